"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck), one
tool per run: the fused conv layer at n = 2048 (smoke shape, staged twiddles, PDL),
the host-buffer entry (CUDA graph), the tcgen05 ElementMult (TMEM, mbarriers, bulk
copies) and its transpose, the RNS layer at n = 8192 (exact CRT decryption), the
activation / pool kernel and the wire encode / decode kernels.

    compute-sanitizer --tool memcheck python tools/sanitize_run.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2003_05328_b200 import ops, protocol as GP, wire as Wr  # noqa: E402
from paper_2003_05328_b200._lib import check, lib  # noqa: E402

dev = torch.device("cuda", 0)
g = torch.Generator().manual_seed(5)
ctx = ops.Context(n=2048)
# fused layer, smoke shape
L = ops.LayerOps(ctx, ops.ConvSpec(16, 16, 3, 3, True, 4, 3))
_, key = ops.secret_sample(ctx, 1)
w = torch.randint(-128, 128, (3, 4, 3, 3), dtype=torch.int32, generator=g).to(dev)
x = torch.randint(0, 256, (2, 4, 16, 16), dtype=torch.uint8, generator=g)
we = L.prepare_weights(w)
out = L.forward(key, we, x.to(dev), ops.Randomness(seed=1))
h_out = torch.empty_like(out.cpu()).pin_memory()
L.forward_host(key, we, x.pin_memory(), ops.Randomness(seed=1), L.workspace(2, host=True), h_out)
# tcgen05 ElementMult (forced) on a 40-channel layer, 32 images
check(lib().ensei_gpu_set_mac_variant(5))
L2 = ops.LayerOps(ctx, ops.ConvSpec(8, 8, 3, 3, True, 40, 20))
w2 = torch.randint(-128, 128, (20, 40, 3, 3), dtype=torch.int32, generator=g).to(dev)
x2 = torch.randint(0, 256, (32, 40, 8, 8), dtype=torch.uint8, generator=g).to(dev)
we2 = L2.prepare_weights(w2)
assert L2.mac_path(32) == "tcgen05"
out2 = L2.forward(key, we2, x2, ops.Randomness(seed=2))
check(lib().ensei_gpu_set_mac_variant(-1))
# RNS layer, n = 8192, one image
c4 = ops.Context(n=8192, q=ops.RNS_DEFAULT)
L4 = ops.LayerOps(c4, ops.ConvSpec(32, 32, 3, 3, True, 2, 2))
_, k4 = ops.secret_sample(c4, 4)
w4 = torch.randint(-128, 128, (2, 2, 3, 3), dtype=torch.int32, generator=g).to(dev)
x4 = torch.randint(0, 256, (1, 2, 32, 32), dtype=torch.uint8, generator=g).to(dev)
out4 = L4.forward(k4, L4.prepare_weights(w4), x4, ops.Randomness(seed=4))
# activation + pool and a two-layer session
sess = GP.Session(ctx, [GP.Conv(3, 3, True, 4, 4), GP.Act(0, True), GP.Conv(1, 1, True, 4, 2)], 16, 16,
                  [torch.randint(-8, 8, (4, 4, 3, 3), dtype=torch.int32, generator=g),
                   torch.randint(-8, 8, (2, 4, 1, 1), dtype=torch.int32, generator=g)])
y = sess.run(key, x.to(dev), lambda li: ops.Randomness(seed=6, layer=li))
# wire frames: encode / decode both directions
ct = L.alice_encrypt(key, x.to(dev), ops.Randomness(seed=7))
fr = Wr.encode_ct_blocks(ctx, Wr.CIPHERTEXT_BLOCKS, 0, ct, Wr.EVALUATION)
back, _, _ = Wr.decode_ct_blocks(ctx, fr, Wr.CIPHERTEXT_BLOCKS, 4, L.B)
assert torch.equal(back, ct)
torch.cuda.synchronize()
print("sanitize workload ok")
