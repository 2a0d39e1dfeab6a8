"""Where does the host-buffer (e2e) path spend its time beyond the device step?
Prints per-call wall-clock medians (us) of several variants of the config-1 layer."""
import ctypes as C
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2003_05328_b200 import _lib, ops  # noqa: E402

Q, P = 576460803525083137, 638977
lib = _lib.lib()
dev = torch.device("cuda", 0)
ctx = ops.Context(n=2048)
L = ops.LayerOps(ctx, ops.ConvSpec(32, 32, 3, 3, True, 16, 16))
g = torch.Generator().manual_seed(1)
x = torch.randint(0, 256, (8, 16, 32, 32), dtype=torch.uint8, generator=g)
w = torch.randint(-128, 128, (16, 16, 3, 3), dtype=torch.int32, generator=g).to(dev)
_, key = ops.secret_sample(ctx, 1)
w_eval = L.prepare_weights(w)
rand = ops.Randomness(seed=1)
h_x = x.pin_memory()
h_out = torch.empty((8, 16, 32, 32), dtype=torch.int32).pin_memory()
ws_h = L.workspace(8, host=True, in_dtype=_lib.IN_U8)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
x_d = x.to(dev)
out_d = torch.empty((8, 16, 32, 32), dtype=torch.int32, device=dev)
ws = L.workspace(8)


def timeit(fn, reps=50, do_flush=True):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    acc = []
    for _ in range(reps):
        if do_flush:
            flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        acc.append((time.perf_counter() - t0) * 1e6)
    return statistics.median(acc)


rs = rand.struct()
args = (ctx.h, C.byref(L.d), ops._ptr(key), ops._ptr(w_eval), C.c_void_p(h_x.data_ptr()), _lib.IN_U8, 8,
        C.byref(rs), ops._ptr(ws_h), C.c_void_p(h_out.data_ptr()))
s_user = torch.cuda.Stream()
res = {}
res["forward_host (bench path)"] = timeit(lambda: L.forward_host(key, w_eval, h_x, rand, ws_h, h_out))
res["direct C call, legacy stream"] = timeit(lambda: lib.ensei_gpu_conv_layer_host(*args, None))
res["direct C call, user stream"] = timeit(lambda: lib.ensei_gpu_conv_layer_host(*args, C.c_void_p(s_user.cuda_stream)))
res["direct C call, no flush"] = timeit(lambda: lib.ensei_gpu_conv_layer_host(*args, None), do_flush=False)
graph = torch.cuda.CUDAGraph()
for _ in range(2):
    L.forward(key, w_eval, x_d, rand, ws=ws, out=out_d)
torch.cuda.synchronize()
with torch.cuda.graph(graph):
    L.forward(key, w_eval, x_d, rand, ws=ws, out=out_d)


def dev_graph():
    graph.replay()
    torch.cuda.synchronize()


res["device graph replay + sync (wall)"] = timeit(dev_graph)
res["device graph + H2D/D2H memcpy + sync"] = timeit(lambda: (x_d.copy_(h_x, non_blocking=True), graph.replay(),
                                                              h_out.copy_(out_d, non_blocking=True),
                                                              torch.cuda.synchronize()))
res["abi_version() call"] = timeit(lambda: lib.ensei_gpu_abi_version(), do_flush=False)
res["sync idle"] = timeit(lambda: torch.cuda.synchronize(), do_flush=False)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
acc = []
for _ in range(20):
    flush.zero_()
    a.record()
    graph.replay()
    b.record()
    b.synchronize()
    acc.append(a.elapsed_time(b) * 1e3)
res["device graph (events)"] = statistics.median(acc)
acc = []
for _ in range(20):
    flush.zero_()
    a.record()
    lib.ensei_gpu_conv_layer_host(*args, None)
    b.record()
    b.synchronize()
    acc.append(a.elapsed_time(b) * 1e3)
res["host entry (events on legacy stream)"] = statistics.median(acc)
for k, v in res.items():
    print(f"{k:45s} {v:9.1f} us")
