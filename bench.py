#!/usr/bin/env python3
"""bench.py -- B200 benchmark of the oblivious NTT-domain convolution hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 4]

Default workload = BASELINE.json configs[4], the one config defined over 1/2/4/8
B200s and the largest that fits one GPU: one 64 -> 128 3x3 Same conv layer over 1024
images of 64x32x32 uint8 per GPU, int8 weights, ring degree n = 8192 with an RNS
ciphertext modulus of three 60-bit primes, p = 638977, 64x64 padded grid (one block per
channel).  One STEP = the whole oblivious layer for the GPU's 1024 images (Alice Enc ->
Bob HomShare + ElementMult -> Alice Dec -> IDFT2D -> recombine), streamed through the
library's 128-image workspace; weights prepared once (t_setup, excluded like the paper,
reported).  `value` = convolutions (images through the layer) per second over all GPUs
with inputs resident in HBM; `e2e` = the same through the host-buffer C-ABI call
(ensei_gpu_conv_layer_host: 64 MiB of pixels in, 512 MiB of outputs back per step).

Under torchrun (N > 1) every rank runs its own 1024 images (weak scaling; image ids
are global, so every image gets the same randomness as in a 1-GPU run) and both
parties' output shares are all-gathered with NCCL chunk by chunk, overlapped with the
next chunk's compute (paper_2003_05328_b200/shard.py ShareGather).

The CPU baseline / reference arm is the UNMODIFIED reference compiled from its own
sources (oracle/_ref/libensei_ref.so).  Config 4 has no reference counterpart (REF has
no RNS), so its proxy is REF's single-prime n = 8192 path with the 60-bit q on the same
layer: the per-image online operators of a REF session (ntt_2d,
encrypt_freq_direct, mul_plain / add_ct, hom_share, decrypt, intt_2d) on all host
threads, Bob's prepare_plain table built once (oracle/ref_harness.cpp
ref_bench_layer_ops).  `--config 1` keeps the round-1 line (8 images, 16 -> 16, n = 2048).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

P = 638977
Q = 576460803525083137
METRIC = "oblivious NTT-domain conv/sec (1/2/4/8 B200); NTT modmul/s vs roofline"
# IMAD-pipe slots per modmul class, min(SURVEY.md 8(d) constant, our SASS) with
# IMAD.WIDE = 2 slots (measured: 4 fmaheavy cycles per warp vs 2 for IMAD):
#   q-Shoup 5 WIDE + 4 IMAD = 14 > 10 -> 10;  Karatsuba MAC 3 WIDE = 6 < 8 -> 6;
#   p-Shoup 1 WIDE + 2 IMAD = 4 > 3 -> 3.
C_Q, C_MAC, C_P = 10, 6, 3
# What the SASS can reach with 32-bit multipliers: a Shoup product is 5 IMAD.WIDE (two pipe
# slots each -- ncu: fmaheavy busy exceeds issue active by exactly that weighting) + 4 IMAD
# = 14 slots (DESIGN 4, "NTT engine"); imad fractions against that floor are reported beside
# the survey's c_q = 10.
C_Q_SASS = 14


# profile name -> kernel names it can stand for (the 3-prime RNS layer runs the second-generation
# tile kernels enc3 / share3 / dec3, every other shape the first-generation ones)
NCU_KERNELS = {"enc": ("enc3_kernel", "tile_enc_kernel"), "share": ("share3_kernel", "share_kernel"),
               "mac": ("mac_kara_kernel",), "dec": ("dec_kernel",), "dec_rns": ("dec3_kernel", "dec_rns_kernel"),
               "planes_tc": ("planes_tc_kernel",), "mac_tc": ("mac_tc_kernel",), "mac_out": ("mac_out_kernel",)}


def ncu_traffic(cfg, name):
    """DRAM bytes (read + write) per launch of kernel `name` from the committed ncu --set full
    capture of this workload (profiles/*_ncu_traffic.json, written by tools/ncu_traffic.py);
    None when no capture is committed."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*_ncu_traffic.json")))
    for f in reversed(files):  # the newest round that captured this kernel
        recs = json.load(open(f)).get(cfg, {})
        for k in NCU_KERNELS.get(name, (name,)):
            if k in recs:
                return recs[k]["dram_bytes"]
    return None


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--images", type=int, default=0, help="images per GPU per step (0: the config's own)")
    ap.add_argument("--seed", type=int, default=2003)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-ntt", action="store_true")
    ap.add_argument("--no-side", action="store_true", help="config 4: skip the config-1 / unpacked side lines")
    ap.add_argument("--pack", type=int, default=None,
                    help="images per ciphertext block (config 4 default: 5 on the 39x39 grid, 2 with --grid 0; "
                         "1 = REF geometry); config 3: 1 = unpacked")
    ap.add_argument("--grid", type=int, default=None,
                    help="config 4: padded grid side (default 39, the smallest side dividing p - 1 that holds the "
                         "convolution; 0 = REF's 64x64)")
    ap.add_argument("--no-graph", action="store_true", help="launch the layer eagerly instead of a CUDA graph")
    return ap.parse_args()


# ------------------------------------------------------------------ accounting

def ntt_fwd(n):
    return (n // 2) * (n.bit_length() - 1)


def ntt_inv(n):
    return ntt_fwd(n) + n


def dft2d(L):
    return 2 * L * (L // 2) * (L.bit_length() - 1)


def idft2d(L):
    return dft2d(L) + L * L


def _pfa_factors(L):
    """L = N1 N2 with coprime factors (the device's prime-factor tile transform), or None."""
    for a in range(2, L):
        if L % a == 0 and math.gcd(a, L // a) == 1:
            return a, L // a
    return None


def dft2d_any(L, inverse=False):
    """Modmuls of one L x L tile transform: radix-2 for powers of two, the prime-factor form
    (N1 + N2 products per output, no twiddles) for the non-power-of-two grid override."""
    if L & (L - 1) == 0:
        return idft2d(L) if inverse else dft2d(L)
    n1, n2 = _pfa_factors(L)
    return 2 * L * L * (n1 + n2)


def layer_counts(n, R, L, B, cin, cout, H, W, oh, ow, imgs, pack=1):
    """Algorithmic modmul counts and HBM bytes per kernel per launch for
    `imgs` images; with packing, the ring work is per ciphertext image (pack images each),
    the 2D transforms and pixel / share bytes per image."""
    c = -(-imgs // pack)  # ciphertext images
    k = {}
    k["enc"] = dict(q=c * cin * B * R * (2 * n + ntt_fwd(n)), mac=0, p=imgs * cin * dft2d_any(L) + c * cin * B * ntt_inv(n),
                    bytes=imgs * cin * H * W + c * cin * B * 2 * R * n * 8 + 2 * R * n * 8)
    k["share"] = dict(q=c * cout * B * R * (n + ntt_fwd(n)), mac=0,
                      p=c * cout * B * ntt_inv(n) + imgs * cout * dft2d_any(L, True),
                      bytes=c * cout * B * R * n * 8 + imgs * cout * oh * ow * 4)
    k["mac"] = dict(q=0, mac=c * cin * cout * B * R * 2 * n, p=0,
                    bytes=c * cin * B * 2 * R * n * 8 + cout * cin * B * R * n * 8 + c * cout * B * R * n * 8
                    + c * cout * B * 2 * R * n * 8)
    k["dec"] = dict(q=c * cout * B * R * (n + ntt_inv(n)), mac=0, p=c * cout * B * ntt_fwd(n) + imgs * cout * dft2d_any(L, True),
                    bytes=c * cout * B * 2 * R * n * 8 + 2 * R * n * 8 + imgs * cout * oh * ow * 4 * 3)
    for v in k.values():
        v["imad"] = C_Q * v["q"] + C_MAC * v["mac"] + C_P * v["p"]
        v["modmul"] = v["q"] + v["mac"] + v["p"]
    return k


# ------------------------------------------------------------------ clocks

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------------ reference arm

def ref_layer_bench(images_per_sample, threads, seed):
    """The reference's own CPU protocol (run_inproc) on the config-1 layer, one
    image per session, `threads` concurrent sessions (2 host threads each)."""
    import numpy as np
    import oracle as O
    R = O.ref()
    g = O.MTRng(seed, 0xDA7A)
    img = np.array([g.uniform_below(256) for _ in range(16 * 32 * 32)], np.int64)
    w = np.array([g.uniform_below(256) - 128 for _ in range(16 * 16 * 9)], np.int64)
    desc = np.array([0, 3, 3, 1, 16, 16, 0], np.int32)
    online = O.C.c_double(0)
    wall = R.ref_bench_protocol(P, Q, 2048, 4.0, seed, 32, 32, 1, desc, img, w, images_per_sample, threads,
                                O.C.byref(online))
    if wall < 0:
        raise RuntimeError("reference bench failed: " + R.ref_last_error().decode())
    # online-phase throughput with `threads` sessions overlapped (t_setup excluded)
    value = images_per_sample / (online.value / threads)
    return value, wall, online.value


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def ref_ops_bench(n, q, cin, cout, images, threads, seed):
    """REF's per-image online operators on one 32x32 3x3 Same layer (ref_bench_layer_ops):
    returns (conv/s with `threads` images in flight, wall s, summed online s, setup s)."""
    import numpy as np
    import oracle as O
    g = O.MTRng(seed, 0xDA7A)
    img = np.array([g.uniform_below(256) for _ in range(cin * 32 * 32)], np.int64)
    w = np.array([g.uniform_below(256) - 128 for _ in range(cout * cin * 9)], np.int64)
    online, setup = O.C.c_double(0), O.C.c_double(0)
    wall = O.ref().ref_bench_layer_ops(P, q, n, 4.0, seed, 32, 32, 3, 3, 1, cin, cout, img, w, images, threads,
                                       O.C.byref(online), O.C.byref(setup))
    if wall < 0:
        raise RuntimeError("reference bench failed: " + O.ref().ref_last_error().decode())
    return images / wall, wall, online.value, setup.value


def run_reference(args, rank):
    """The reference arm: REF's own CPU implementation of the path on all host threads,
    on this arm's config / metric / unit; rank 0 only (other ranks exit without work)."""
    if rank != 0:
        return
    cores = host_cores()
    vals, walls = [], []
    if args.config not in (1, 4):
        print(json.dumps({"impl": "reference", "unavailable": "the reference arm covers the bench lines' configs "
                                                              "(4: default headline, 1)"}), flush=True)
        return
    if args.config == 1:
        threads = max(1, cores // 2)
        per = max(threads, 16)
        step = lambda s: ref_layer_bench(per, threads, args.seed + 1000 * s)[0]  # noqa: E731
        workload = ("config1 layer (16->16 3x3 Same @32x32, n=2048, 60-bit q, p=638977), one image per reference "
                    "run_inproc session")
        sample = (f"{per} run_inproc sessions per step, {threads} concurrent (2 threads each); online phase (Alice "
                  "Hello->Done), Bob weight prep excluded")
    else:
        threads = cores
        per = max(16, cores)
        step = lambda s: ref_ops_bench(8192, Q, 64, 128, per, threads, args.seed + 1000 * s)[0]  # noqa: E731
        workload = ("config4 proxy: the 64->128 3x3 Same layer @32x32 at n=8192 with REF's single 60-bit prime "
                    "q=576460803525083137 (REF has no RNS; SURVEY 8(d)), p=638977")
        sample = (f"{per} images per step through REF's per-image online operators (ntt_2d, encrypt_freq_direct, "
                  f"mul_plain/add_ct, hom_share, decrypt, intt_2d; oracle/ref_harness.cpp ref_bench_layer_ops), "
                  f"{threads} host threads over images; Bob's prepare_plain table built once per step, excluded "
                  "(t_setup)")
    for s in range(args.warmup):
        step(-1 - s)
    t0 = time.perf_counter()
    for s in range(args.steps):
        t1 = time.perf_counter()
        vals.append(step(s))
        walls.append(time.perf_counter() - t1)
    elapsed = time.perf_counter() - t0
    value = statistics.median(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "conv/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * elapsed / max(1, args.steps),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": workload, "images_per_step": per, "threads": threads, "config_index": args.config},
        "cpu_baseline": {"value": value, "unit": "conv/s", "cores": threads, "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": "conv/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm

def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank)

    import torch
    import torch.distributed as dist
    from paper_2003_05328_b200 import _lib, ops
    from paper_2003_05328_b200.shard import ImageShard, gather_outputs

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if args.config == 4:
        line = run_config4(args, world, rank, local)
    elif args.config == 1:
        line = run_config1(args, world, rank, local)
    else:
        line = None
        other_config(args, world, rank, local)
    if rank == 0 and line is not None:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_config1(args, world, rank, local, side=False):
    """BASELINE config 1 (8 images, 16 -> 16, n = 2048); side=True: the compact form
    attached to the config-4 line (no CPU baseline / NTT / wire side measurements)."""
    import torch
    import torch.distributed as dist
    from paper_2003_05328_b200 import _lib, ops
    from paper_2003_05328_b200.shard import ImageShard, gather_outputs
    dev = torch.device("cuda", local)
    lib = _lib.lib()
    imgs = (args.images or 8) if not side else 8
    ctx = ops.Context(n=2048, q=(Q,), p=P, device=local)
    spec = ops.ConvSpec(32, 32, 3, 3, True, 16, 16)
    L = ops.LayerOps(ctx, spec)
    g = L.geom
    gen = torch.Generator().manual_seed(args.seed)
    x_all = torch.randint(0, 256, (world * imgs, 16, 32, 32), dtype=torch.uint8, generator=gen)
    wts = torch.randint(-128, 128, (16, 16, 3, 3), dtype=torch.int32, generator=gen).to(dev)
    shard = ImageShard(world * imgs, world, rank)  # contiguous image shards, global image ids
    x = shard.take(x_all).contiguous().to(dev)
    _, key = ops.secret_sample(ctx, args.seed)
    w_eval = L.prepare_weights(wts)  # t_setup (not timed)
    rand = ops.Randomness(seed=args.seed, image_base=shard.start)
    ws = L.workspace(imgs)
    out = torch.empty((imgs, 16, g.oh, g.ow), dtype=torch.int32, device=dev)
    gathered = torch.empty((world * imgs, 16, g.oh, g.ow), dtype=torch.int32, device=dev) if world > 1 else None
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def layer():
        return L.forward(key, w_eval, x, rand, ws=ws, out=out)

    # The layer's launches (share on the aux stream || Enc, then ElementMult, Dec) are
    # captured once into a CUDA graph and replayed per step; inputs stay in place.
    for _ in range(2):
        layer()
    torch.cuda.synchronize()
    graph = None
    if not args.no_graph:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            layer()
        torch.cuda.synchronize()

    def step():
        if graph is not None:
            graph.replay()
        else:
            layer()
        if world > 1:
            gather_outputs(out, shard, gathered)  # NCCL all-gather of the reconstructed outputs
        return out

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    c0 = lib.ensei_gpu_launch_count()
    layer()
    torch.cuda.synchronize()
    kernels_per_layer = lib.ensei_gpu_launch_count() - c0
    launches0 = lib.ensei_gpu_launch_count()
    total_ms = 0.0
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for i in range(args.steps):
        flush.zero_()  # evict L2 between timed steps (untimed)
        ev[i][0].record(stream)
        step()
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    launches = lib.ensei_gpu_launch_count() - launches0
    if graph is not None:  # graph replays do not pass through the launch counter
        launches = args.steps * kernels_per_layer
    total_ms = sum(a.elapsed_time(b) for a, b in ev)
    clk = clocks.stop()
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        dist.barrier()
    ms_step = total_ms / args.steps
    value = world * imgs * args.steps / (total_ms / 1e3)

    # ---- per-kernel breakdown + roofline (separately launched, CUDA events, L2 flushed)
    kcount = layer_counts(2048, 1, g.Lh, g.blocks, 16, 16, 32, 32, g.oh, g.ow, imgs)
    ct_in = L.empty_ct(imgs, 16)
    ct_out = L.empty_ct(imgs, 16)
    bob = torch.empty((imgs, 16, g.oh, g.ow), dtype=torch.int32, device=dev)

    times = {}
    fns = {
        "enc": lambda: _lib.check(lib.ensei_gpu_alice_encrypt(ctx.h, ops.C.byref(L.d), ops._ptr(key), 0,
                                                               ops._ptr(x), _lib.IN_U8, imgs,
                                                               ops.C.byref(rand.struct()), ops._ptr(ct_in),
                                                               ops._stream())),
        "share": lambda: L.bob_share(imgs, rand, ct_out=ct_out, bob=bob),
        "mac": lambda: L.bob_mac(ct_in, w_eval, ct_out),
        "dec": lambda: _lib.check(lib.ensei_gpu_alice_decrypt(ctx.h, ops.C.byref(L.d), ops._ptr(key), 0,
                                                               ops._ptr(ct_out), imgs, ops._ptr(out),
                                                               ops._stream())),
    }
    for name, fn in fns.items():
        for _ in range(3):
            fn()
        acc = []
        for _ in range(10):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            b.synchronize()
            acc.append(a.elapsed_time(b))
        times[name] = statistics.median(acc)
    imad_peak = lib.ensei_gpu_imad_peak(local)  # IMAD-pipe slots/s (mad.lo.u32 chains), live probe
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    dom = max(times, key=times.get)
    kd = kcount[dom]
    t_dom = times[dom] * 1e-3
    imad_ach = kd["imad"] / t_dom / 1e9
    hbm_ach = kd["bytes"] / t_dom / 1e9
    imad_frac = imad_ach / (imad_peak / 1e9)
    hbm_frac = hbm_ach / hbm_peak
    bound = "imad" if imad_frac >= hbm_frac else "hbm"
    roofline = {
        "bound": bound, "kernel": dom,
        "achieved": imad_ach if bound == "imad" else hbm_ach,
        "peak": imad_peak / 1e9 if bound == "imad" else hbm_peak,
        "unit": "GIMAD/s" if bound == "imad" else "GB/s",
        "frac": imad_frac if bound == "imad" else hbm_frac,
        "traffic": ncu_traffic("config1", dom),
        "peak_source": ("live mad.lo.u32 probe (ensei_gpu_imad_peak)" if bound == "imad"
                        else "MEASURED_PEAKS.json hbm_gbs (measured)"),
        "imad": {"achieved_GIMAD_s": imad_ach, "peak_GIMAD_s": imad_peak / 1e9, "frac": imad_frac,
                 "imad_per_launch": kd["imad"], "c_q": C_Q, "c_mac": C_MAC, "c_p": C_P},
        "hbm": {"achieved_GB_s": hbm_ach, "peak_GB_s": hbm_peak, "frac": hbm_frac, "bytes_per_launch": kd["bytes"]},
        "kernel_ms": times,
        "per_kernel": {k: {"ms": times[k],
                           "imad_frac": kcount[k]["imad"] / (times[k] * 1e-3) / imad_peak,
                           "hbm_frac": kcount[k]["bytes"] / (times[k] * 1e-3) / 1e9 / hbm_peak}
                       for k in times},
    }
    total_modmul = sum(v["modmul"] for v in kcount.values())

    # ---- e2e through the host-buffer C-ABI entry point
    h_x = x.cpu().pin_memory()
    h_out = torch.empty((imgs, 16, g.oh, g.ow), dtype=torch.int32).pin_memory()
    ws_h = L.workspace(imgs, host=True, in_dtype=_lib.IN_U8)
    call = L.host_call(key, w_eval, h_x, rand, ws_h, h_out)  # prepared public call (serving loop)
    for _ in range(3):
        call()
    e2e_ms = []
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        call()
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
    e2e_ms_step = statistics.mean(e2e_ms)
    if world > 1:
        t = torch.tensor([e2e_ms_step], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms_step = float(t.item())
    e2e = {"value": world * imgs / (e2e_ms_step / 1e3), "unit": "conv/s", "h2d_bytes_per_step": h_x.numel(),
           "d2h_bytes_per_step": h_out.numel() * 4, "ms_per_step": e2e_ms_step,
           "api": "LayerOps.host_call -> ensei_gpu_conv_layer_host (host pinned buffers, wall clock)"}

    # ---- config 2 side measurement: batched negacyclic NTT/INTT (device layout)
    ntt = None
    if not args.no_ntt and rank == 0 and not side:
        ntt = {}
        for n in (2048, 4096, 8192):
            c2 = ops.Context(n=n, q=(Q,), p=P, device=local)
            cnt = 65536
            buf = torch.randint(0, 1 << 62, (cnt, n), dtype=torch.int64, device=dev).view(torch.uint64)
            buf.copy_((buf.view(torch.int64) % Q).view(torch.uint64))
            res = {}
            for inv in (False, True):
                for _ in range(2):
                    c2.negacyclic(buf, 0, inv, _lib.LAYOUT_BITREV)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                for _ in range(5):
                    c2.negacyclic(buf, 0, inv, _lib.LAYOUT_BITREV)
                b.record(stream)
                b.synchronize()
                ms = a.elapsed_time(b) / 5
                rate = cnt / (ms / 1e3)
                alg = (ntt_inv(n) if inv else ntt_fwd(n))
                res["inv" if inv else "fwd"] = {"transforms_per_s": rate, "ms": ms,
                                                "GB_s": cnt * n * 16 / (ms / 1e3) / 1e9,
                                                "imad_frac": rate * alg * C_Q / imad_peak}
            ntt[str(n)] = res
            del buf, c2
        torch.cuda.empty_cache()

    # ---- wire framing side measurement: the step's AliceShareCiphertexts frames
    # (imgs x 16 channels x 2 blocks records, REF wire layout) built from / parsed into
    # the device layout, device-resident frames (HBM roofline) and page-locked host frames.
    wire = None
    if rank == 0 and not side:
        from paper_2003_05328_b200 import wire as Wr
        fb = Wr.ct_frame_bytes(2048, 16, g.blocks)
        ct_out.copy_((ct_out.view(torch.int64).abs() % Q).view(torch.uint64))
        fr_dev = torch.empty((imgs, fb), dtype=torch.uint8, device=dev)
        fr_host = Wr.pinned_frames(imgs, fb)
        ct_back = torch.empty_like(ct_out)
        wire = {"frame_bytes": fb, "frames": imgs}
        for name, fn in (("encode_device", lambda: Wr.encode_ct_blocks(ctx, Wr.ALICE_SHARE_CIPHERTEXTS, 0, ct_out,
                                                                         out=fr_dev)),
                         ("decode_device", lambda: Wr.decode_ct_blocks(ctx, fr_dev, Wr.ALICE_SHARE_CIPHERTEXTS, 16,
                                                                         g.blocks, out=ct_back)),
                         ("encode_pinned_host", lambda: Wr.encode_ct_blocks(ctx, Wr.ALICE_SHARE_CIPHERTEXTS, 0,
                                                                              ct_out, out=fr_host)),
                         ("decode_pinned_host", lambda: Wr.decode_ct_blocks(ctx, fr_host, Wr.ALICE_SHARE_CIPHERTEXTS,
                                                                              16, g.blocks, out=ct_back))):
            for _ in range(3):
                fn()
            acc = []
            for _ in range(10):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                fn()
                b.record(stream)
                b.synchronize()
                acc.append(a.elapsed_time(b))
            ms = statistics.median(acc)
            nbytes = imgs * fb + ct_out.numel() * 8  # read one side, write the other
            wire[name] = {"ms": ms, "GB_s": nbytes / (ms / 1e3) / 1e9,
                          "hbm_frac": nbytes / (ms / 1e3) / 1e9 / hbm_peak if "device" in name else None}
        assert torch.equal(ct_back, ct_out)

    # ---- CPU baseline (reference, bounded sample, rank 0)
    cpu = None
    if rank == 0 and not args.no_cpu_baseline and not side:
        try:
            cores = host_cores()
            thr = max(1, cores // 2)
            v, wall, online = ref_layer_bench(max(thr, 16), thr, args.seed)
            cpu = {"value": v, "unit": "conv/s", "cores": cores, "kind": "reference",
                   "sample": f"{max(thr, 16)} reference run_inproc sessions (one config-1 image each), {thr} "
                             f"concurrent x 2 threads, online phase only; wall incl. Bob setup {wall:.2f}s"}
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": "conv/s", "cores": host_cores(), "kind": "reference",
                   "sample": f"unavailable: {e}"}

    # ---- the same layer on the 39x39 grid (grid override: one ciphertext block per channel
    # instead of two), device timing, CUDA graph replay
    grid39 = None
    try:
        Lg = ops.LayerOps(ctx, ops.ConvSpec(32, 32, 3, 3, True, 16, 16, 1, 39))
        weg = Lg.prepare_weights(wts)
        wsg = Lg.workspace(imgs)
        outg = torch.empty_like(out)
        for _ in range(2):
            Lg.forward(key, weg, x, rand, ws=wsg, out=outg)
        torch.cuda.synchronize()
        gg = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gg):
            Lg.forward(key, weg, x, rand, ws=wsg, out=outg)
        tg = _time_steps(gg.replay, args.steps, max(3, args.warmup), flush, stream)
        grid39 = {"value": world * imgs * args.steps / (tg / 1e3), "unit": "conv/s", "ms_per_step": tg / args.steps,
                  "outputs_equal": bool(torch.equal(outg, L.forward(key, w_eval, x, rand, ws=ws))),
                  "geometry": "39x39 padded grid (ensei_conv_desc::grid), 1 block per channel"}
    except Exception as e:  # noqa: BLE001
        grid39 = {"value": None, "error": str(e)}

    if side:
        return {"value": value, "unit": "conv/s", "ms_per_step": ms_step, "e2e": e2e, "kernel_ms": times,
                "grid39": grid39,
                "workload": "config1: 8 images/GPU x 16x32x32, 16->16 3x3 Same, n=2048, single 60-bit q, CUDA graph"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "conv/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u64",
            "data": "synthetic: uint8 pixels U[0,256), int8 weights U[-128,128), seeded (no dataset)",
            "config": {"workload": "config1: one conv layer, 8 images/GPU x 16x32x32 uint8, 16x16x3x3 int8, Same, "
                                   "n=2048, q=576460803525083137 (60-bit), p=638977, 64x64 padded grid, 2 blocks/ch",
                       "images_per_gpu": imgs, "global_batch": world * imgs, "parallelism": f"dp{world} (image shards)",
                       "l2": "flushed (256 MB write) between timed steps", "randomness": "Philox4x32-10 device streams",
                       "launch": "eager" if args.no_graph else "CUDA graph replay of the layer (share || enc, mac, dec)",
                       "unit_def": "1 conv = 1 image through the whole 16->16 layer"},
            "roofline": roofline,
            "modmul_per_s": total_modmul * world * args.steps / (total_ms / 1e3),
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk, "ntt_config2": ntt,
            "wire": wire, "grid39": grid39,
        }
        return line
    return None


# ------------------------------------------------------------------ config 4 (the headline)

def i8_peak_tops(peaks, lib=None, device=0):
    """int8 dense tensor peak in TOP/s, measured live: back-to-back tcgen05.mma.kind::i8
    (M = 128, N = 256, K = 32) on every SM (ensei_gpu_tc_i8_peak; 4.58 POPS on this pool,
    above NVIDIA's nominal 4.5).  MEASURED_PEAKS has no int8 entry; if the probe fails, 2 x
    its bf16 GEMM burst (int8 dense = 2x bf16 dense on sm_100a)."""
    if lib is not None:
        v = lib.ensei_gpu_tc_i8_peak(device, 256)
        if v > 0:
            return 2.0 * v / 1e12, "live tcgen05.mma.kind::i8 probe (ensei_gpu_tc_i8_peak, M128 N256 K32)"
    return 2.0 * peaks.get("bf16_tflops", 1590.0), "2 x MEASURED_PEAKS.json bf16_tflops (int8 dense = 2x bf16 dense)"


def config4_counts(imgs, pack=1, n=8192, R=3, L=64, B=1, cin=64, cout=128, H=32, W=32):
    """Per-kernel algorithmic work for one sub-batch of `imgs` images:
    modmuls by class, IMAD slots (c_q, c_mac, c_p), HBM bytes, int8 tensor MACs.  The
    tcgen05 ElementMult is three kernels: planes_tc (ciphertext words -> byte planes),
    mac_tc (tensor cores; reads the ciphertext and weight planes, writes the slot-major
    product Y) and mac_out (Y + the HomShare masks -> the ciphertext layout)."""
    k = layer_counts(n, R, L, B, cin, cout, H, W, H, W, imgs, pack)
    c = -(-imgs // pack)
    ctw = c * cin * B * 2 * R * n * 8  # ciphertext words in, bytes
    ybytes = c * cout * B * 2 * R * n * 8
    k["planes_tc"] = dict(q=0, mac=0, p=0, bytes=2 * ctw, imad=0, modmul=0)
    # 64 u8 x u8 products per modular MAC (byte planes)
    k["mac_tc"] = dict(q=0, mac=k["mac"]["mac"], p=0, i8_mac=64 * k["mac"]["mac"], imad=0,
                       modmul=k["mac"]["mac"], bytes=ctw + cout * cin * B * R * n * 8 + ybytes)
    k["mac_out"] = dict(q=0, mac=0, p=0, imad=0, modmul=0, bytes=ybytes + c * cout * B * R * n * 8 + ybytes)
    k["mac"]["i8_mac"] = 64 * k["mac"]["mac"]
    k["mac"]["imad"] = 0
    return k


def run_config4(args, world, rank, local):
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2003_05328_b200 import _lib, ops
    from paper_2003_05328_b200 import configs as CF
    from paper_2003_05328_b200.shard import ImageShard, ShareGather
    dev = torch.device("cuda", local)
    lib = _lib.lib()
    cfg = CF.CONFIG4
    imgs = args.images or cfg["images"]
    cin, cout = cfg["cin"], cfg["cout"]
    grid = CF.CONFIG4_GRID if args.grid is None else args.grid
    pack = (CF.CONFIG4_GRID_PACK if grid else CF.CONFIG4_PACK) if args.pack is None else args.pack
    ctx = ops.Context(n=cfg["n"], q=cfg["q"], p=P, device=local)
    L = ops.LayerOps(ctx, ops.ConvSpec(32, 32, 3, 3, True, cin, cout, pack, grid))
    g = L.geom
    shard = ImageShard(world * imgs, world, rank)  # contiguous image shards, global image ids
    # this rank's images (seeded per shard: 64 MiB of pixels per GPU), weights from the common seed
    x_h = torch.randint(0, 256, (imgs, cin, 32, 32), dtype=torch.uint8,
                        generator=torch.Generator().manual_seed(args.seed * 7919 + shard.start))
    w_h = torch.randint(-128, 128, (cout, cin, 3, 3), dtype=torch.int32, generator=torch.Generator().manual_seed(args.seed))
    x = x_h.to(dev)
    _, key = ops.secret_sample(ctx, args.seed)
    torch.cuda.synchronize()
    t_s = time.perf_counter()
    we = L.prepare_weights(w_h.to(dev))  # Bob's t_setup (not timed in the step)
    torch.cuda.synchronize()
    setup_ms = (time.perf_counter() - t_s) * 1e3
    # stream ids are per ciphertext: a rank's first image id must be pack-aligned (ranks own whole
    # ciphertexts; ids stay unique across ranks)
    id_base = rank * (-(-imgs // pack)) * pack
    rand = ops.Randomness(seed=args.seed, image_base=id_base)
    chunk = L.chunk_images(imgs)
    ws = L.workspace(imgs)
    shape = (imgs, cout, g.oh, g.ow)
    out = torch.empty(shape, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    if world > 1:
        alice = torch.empty(shape, dtype=torch.int32, device=dev)
        bob = torch.empty(shape, dtype=torch.int32, device=dev)
        g_alice = torch.empty((world * imgs,) + shape[1:], dtype=torch.int32, device=dev)
        g_bob = torch.empty_like(g_alice)
        gather = ShareGather(shard, g_alice, g_bob)

    def step():
        if world == 1:
            L.forward(key, we, x, rand, ws=ws, out=out)
            return
        # chunk by chunk so each chunk's share all-gathers overlap the next chunk's kernels
        for i0 in range(0, imgs, chunk):
            i1 = min(imgs, i0 + chunk)
            L.forward(key, we, x[i0:i1], ops.Randomness(seed=args.seed, image_base=id_base + i0), ws=ws,
                      out=out[i0:i1], want_shares=True, alice=alice[i0:i1], bob=bob[i0:i1])
            gather.post(i0, i1, alice, bob)
        gather.wait()

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    launches0 = lib.ensei_gpu_launch_count()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for i in range(args.steps):
        flush.zero_()  # evict L2 between timed steps (untimed; the step's own traffic is ~100 GB anyway)
        ev[i][0].record(stream)
        step()
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    launches = lib.ensei_gpu_launch_count() - launches0
    total_ms = sum(a.elapsed_time(b) for a, b in ev)
    clk = clocks.stop()
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        dist.barrier()
    ms_step = total_ms / args.steps
    value = world * imgs * args.steps / (total_ms / 1e3)

    # ---- per-kernel CUDA-event times inside the same step (a separate measurement pass:
    # the library brackets every layer launch with events on its own stream)
    _lib.profile(True)
    prof_steps = 2
    for _ in range(prof_steps):
        flush.zero_()
        L.forward(key, we, x, rand, ws=ws, out=out)
    torch.cuda.synchronize()
    prof = _lib.profile_read()
    _lib.profile(False)
    nchunks = -(-imgs // chunk)
    # algorithmic work of an AVERAGE launch: the step's sub-batches differ in size when the
    # sub-batch does not divide the batch (1024 images = 640 + 384 with five images per block),
    # and the event times below are per-launch averages over the same sub-batches
    kc = config4_counts(imgs, pack, L=int(g.Lh))
    for rec_ in kc.values():
        for key_ in list(rec_):
            rec_[key_] = rec_[key_] / nchunks
    imad_peak = lib.ensei_gpu_imad_peak(local)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    i8_peak, i8_src = i8_peak_tops(peaks, lib, local)
    mac_name = next((k for k in prof if k.startswith("mac")), "mac")
    alias = {"enc": "enc", "share": "share", "dec_rns": "dec", "planes_ct": "planes_ct", "planes_w": "planes_w",
             "planes_tc": "planes_tc", "mac_tc": "mac_tc", "mac_out": "mac_out"}
    if mac_name not in alias:
        alias[mac_name] = "mac"
    per_kernel = {}
    for name, (tot, cnt) in prof.items():
        ms = tot / cnt  # per launch = per sub-batch of `chunk` images
        c = kc.get(alias.get(name, name))
        rec = {"ms_per_launch": ms, "launches_per_step": cnt / prof_steps, "share_of_step": tot / prof_steps / ms_step}
        if c:
            t = ms * 1e-3
            rec["hbm_frac"] = c["bytes"] / t / 1e9 / hbm_peak
            rec["alg_bytes_per_launch"] = c["bytes"]
            if c.get("imad"):
                rec["imad_frac"] = c["imad"] / t / imad_peak
                rec["imad_slots_per_launch"] = c["imad"]
                rec["imad_frac_sass_floor"] = (c["imad"] + (C_Q_SASS - C_Q) * c["q"]) / t / imad_peak
            if c.get("i8_mac"):
                rec["tensor_frac"] = 2 * c["i8_mac"] / t / 1e12 / i8_peak
                rec["int8_macs_per_launch"] = c["i8_mac"]
        per_kernel[name] = rec
    dom = max(per_kernel, key=lambda k: per_kernel[k]["ms_per_launch"] * per_kernel[k]["launches_per_step"])
    d = per_kernel[dom]
    legs = {"tensor": d.get("tensor_frac", 0.0), "imad": d.get("imad_frac", 0.0), "hbm": d.get("hbm_frac", 0.0)}
    bound = max(legs, key=legs.get)
    t_dom = d["ms_per_launch"] * 1e-3
    cdom = kc.get(alias.get(dom, dom), {})
    if bound == "tensor":
        ach, peak, unit = 2 * cdom["i8_mac"] / t_dom / 1e12, i8_peak, "TOP/s (int8)"
    elif bound == "imad":
        ach, peak, unit = cdom["imad"] / t_dom / 1e9, imad_peak / 1e9, "GIMAD/s"
    else:
        ach, peak, unit = cdom["bytes"] / t_dom / 1e9, hbm_peak, "GB/s"
    roofline = {
        "bound": "tensor" if bound == "tensor" else ("hbm" if bound == "hbm" else "imad"), "kernel": dom,
        "achieved": ach, "peak": peak, "unit": unit, "frac": ach / peak, "traffic": ncu_traffic("config4", dom),
        "traffic_note": f"ncu dram__bytes of one launch at the full sub-batch ({chunk} images); achieved / peak are per "
                        f"average launch ({imgs / nchunks:g} images)",
        "peak_source": {"tensor": i8_src, "imad": "live mad.lo.u32 probe (ensei_gpu_imad_peak)",
                        "hbm": "MEASURED_PEAKS.json hbm_gbs (measured)"}[bound],
        "legs": legs, "per_kernel": per_kernel,
        "units_per_launch": f"{imgs / nchunks:g} images on average ({nchunks} sub-batches of at most {chunk} images per step: "
                            f"{nchunks} launches of each kernel)",
        "c_q": C_Q, "c_mac": C_MAC, "c_p": C_P, "c_q_sass_floor": C_Q_SASS,
    }
    step_imad = sum(kc[k]["imad"] for k in ("enc", "share", "dec")) * nchunks
    # the same layer in REF's geometry (one image per ciphertext block on the 64x64 grid) and with
    # two 64x64 grids per block, for comparison
    def other_geometry(pk, gr, what):
        L1 = ops.LayerOps(ctx, ops.ConvSpec(32, 32, 3, 3, True, cin, cout, pk, gr))
        we1 = L1.prepare_weights(w_h.to(dev))
        ws1 = L1.workspace(imgs)
        out1 = torch.empty_like(out)
        rand1 = ops.Randomness(seed=args.seed, image_base=rank * (-(-imgs // pk)) * pk)
        t1 = _time_steps(lambda: L1.forward(key, we1, x, rand1, ws=ws1, out=out1), max(3, args.steps // 4), 2, flush,
                         stream)
        rec = {"value": world * imgs * max(3, args.steps // 4) / (t1 / 1e3), "unit": "conv/s", "geometry": what,
               "outputs_equal_headline": bool(torch.equal(out1, out))}
        del ws1, we1
        torch.cuda.empty_cache()
        return rec
    unpacked = pow2_packed = None
    if (pack > 1 or grid) and not args.no_side:
        unpacked = other_geometry(1, 0, "REF's: one image per n = 8192 ciphertext block, 64x64 grid (half the slots "
                                        "empty)")
        if grid:
            pow2_packed = other_geometry(CF.CONFIG4_PACK, 0, "two 64x64 grids per n = 8192 block (round-2 headline "
                                                             "geometry before the grid override)")
    total_modmul = sum(kc[k]["modmul"] for k in ("enc", "share", "mac", "dec")) * nchunks

    # ---- e2e through the host-buffer C-ABI entry point (pinned host buffers, chunked inside)
    h_x = x_h.pin_memory()
    h_out = torch.empty(shape, dtype=torch.int32).pin_memory()
    ws_h = L.workspace(imgs, host=True, in_dtype=_lib.IN_U8)
    call = L.host_call(key, we, h_x, rand, ws_h, h_out)
    for _ in range(max(3, args.warmup)):
        call()
    e2e_ms = []
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        call()
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
    e2e_ms_step = statistics.mean(e2e_ms)
    if world > 1:
        t = torch.tensor([e2e_ms_step], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms_step = float(t.item())
    e2e = {"value": world * imgs / (e2e_ms_step / 1e3), "unit": "conv/s", "h2d_bytes_per_step": h_x.numel(),
           "d2h_bytes_per_step": h_out.numel() * 4, "ms_per_step": e2e_ms_step,
           "api": "LayerOps.host_call -> ensei_gpu_conv_layer_host (pinned host buffers read / written in place, "
                  "wall clock, synchronous)"}
    del ws_h
    torch.cuda.empty_cache()

    # ---- verification: sampled images of the timed step's output (device path and host path)
    # against the plaintext convolution (REF conv_oracle semantics) -- the oracle as checker only
    verify = None
    if rank == 0:
        try:
            from oracle import protocol as OP
            picks = sorted({0, imgs // 2, imgs - 1})
            ok = True
            for i in picks:
                want = OP.plain_protocol([OP.Conv(3, 3, True, cin, cout)], x_h[i].numpy().astype(np.int64),
                                         [w_h.numpy()], Q, P, 2048, OP.default_workers())
                ok &= bool((out[i].cpu().numpy().astype(np.uint64) == want).all())
                ok &= bool((h_out[i].numpy().astype(np.uint64) == want).all())
            verify = {"images": [shard.start + i for i in picks], "ok": ok,
                      "against": "plaintext convolution (oracle eo_conv_direct = REF conv_oracle), device and "
                                 "host-entry outputs"}
        except Exception as e:  # noqa: BLE001
            verify = {"ok": None, "error": str(e)}

    # ---- CPU baseline: REF single-prime n=8192 proxy, 16+ images over all host threads
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        try:
            cores = host_cores()
            nimg = max(16, cores)
            v, wall, online, setup = ref_ops_bench(8192, Q, cin, cout, nimg, cores, args.seed)
            cpu = {"value": v, "unit": "conv/s", "cores": cores, "kind": "reference",
                   "sample": f"{nimg} images of the same 64->128 layer at n=8192 through REF's per-image online "
                             f"operators with REF's single 60-bit prime (RNS proxy, SURVEY 8(d)), {cores} host "
                             f"threads over images ({wall:.1f} s wall; {online / nimg:.2f} s online per image on one "
                             f"thread); Bob's prepare_plain table ({setup:.1f} s on {cores} threads) excluded"}
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": "conv/s", "cores": host_cores(), "kind": "reference",
                   "sample": f"unavailable: {e}"}

    # ---- side lines: config 1 (round-1 headline) and config 2 (n = 8192 NTT)
    side1 = None
    if world == 1 and not args.no_side:
        del ws
        torch.cuda.empty_cache()
        side1 = run_config1(args, world, rank, local, side=True)
    ntt = None
    if rank == 0 and not args.no_ntt:
        ntt = ntt_side(ctx, dev, stream, imad_peak)

    if rank != 0:
        return None
    return {
        "metric": METRIC, "value": value, "unit": "conv/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u64",
        "data": "synthetic: uint8 pixels U[0,256), int8 weights U[-128,128), seeded (no dataset)",
        "config": {"workload": f"config4: one 64->128 3x3 Same conv layer, {imgs} images/GPU x 64x32x32 uint8, int8 "
                               "weights, n=8192, RNS q = 3 x 60-bit primes == 1 mod 16384 p, p=638977, "
                               f"{g.Lh}x{g.Lw} padded grid, {pack} image(s) per ciphertext block, 1 block/channel",
                   "images_per_gpu": imgs, "global_batch": world * imgs, "parallelism": f"dp{world} (image shards)",
                   "sub_batch_images": chunk, "l2": "flushed (256 MB write) between timed steps; each step also "
                   "streams ~100 GB through HBM", "randomness": "Philox4x32-10 device streams",
                   "launch": f"eager ({nchunks} sub-batches x 6 kernels per step)",
                   "gather": "both parties' output shares all-gathered per sub-batch over NCCL, overlapped"
                             if world > 1 else "none (1 GPU)",
                   "unit_def": "1 conv = 1 image through the whole 64->128 layer", "config_index": 4,
                   "mac_path": L.mac_path(chunk),
                   "pack": pack, "grid": int(g.Lh),
                   "packing": (f"{pack} images' {g.Lh}x{g.Lw} DFT grids per n = 8192 ciphertext block (builder "
                               "extension; every slot-wise step unchanged, outputs = REF's)"
                               + ("; grid override: 39 is the smallest side dividing p - 1 = 2^14 39 that holds the "
                                  "34x34 linear convolution (REF pads to 64 for its radix-2 transform), tile "
                                  "transforms in prime-factor form" if grid else ""))
                   if pack > 1 or grid else "REF geometry (one image per block)"},
        "roofline": roofline, "setup_ms": setup_ms,
        "imad_slot_rate": step_imad * args.steps / (total_ms / 1e3), "modmul_per_s": total_modmul * args.steps / (
            total_ms / 1e3),
        "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk, "verify": verify,
        "config1": side1, "ntt_n8192": ntt, "ref_geometry": unpacked, "pow2_packed": pow2_packed,
    }


def ntt_side(ctx, dev, stream, imad_peak):
    """Config 2 side measurement at n = 8192: 8192 polynomials forward / inverse."""
    import torch
    from paper_2003_05328_b200 import _lib
    n = ctx.n
    cnt = 8192
    buf = torch.randint(0, 1 << 62, (cnt, n), dtype=torch.int64, device=dev)
    buf = (buf % Q).view(torch.uint64)
    res = {}
    for inv in (False, True):
        for _ in range(2):
            ctx.negacyclic(buf, 0, inv, _lib.LAYOUT_BITREV)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(5):
            ctx.negacyclic(buf, 0, inv, _lib.LAYOUT_BITREV)
        b.record(stream)
        b.synchronize()
        ms = a.elapsed_time(b) / 5
        rate = cnt / (ms / 1e3)
        alg = ntt_inv(n) if inv else ntt_fwd(n)
        res["inv" if inv else "fwd"] = {"transforms_per_s": rate, "ms": ms, "imad_frac": rate * alg * C_Q / imad_peak,
                                        "imad_frac_sass_floor": rate * alg * C_Q_SASS / imad_peak}
    del buf
    torch.cuda.empty_cache()
    return res


# ------------------------------------------------------------------ configs 0, 2, 3, 4

def _time_steps(fn, steps, warmup, flush, stream):
    import torch
    for _ in range(max(3, warmup)):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for i in range(steps):
        if flush is not None:
            flush.zero_()
        ev[i][0].record(stream)
        fn()
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    return sum(a.elapsed_time(b) for a, b in ev)


def _ref_sessions(desc_rows, H, W, cin, instances, threads, seed, n=2048, q=Q):
    """Reference run_inproc sessions for an arbitrary schedule; online throughput."""
    import numpy as np
    import oracle as O
    g = O.MTRng(seed, 0xDA7A)
    img = np.array([g.uniform_below(256) for _ in range(cin * H * W)], np.int64)
    wcount = sum(d[1] * d[2] * d[4] * d[5] for d in desc_rows if d[0] == 0)
    w = np.array([g.uniform_below(256) - 128 for _ in range(wcount)], np.int64)
    online = O.C.c_double(0)
    wall = O.ref().ref_bench_protocol(P, q, n, 4.0, seed, H, W, len(desc_rows),
                                      np.array(desc_rows, np.int32).reshape(-1), img, w, instances, threads,
                                      O.C.byref(online))
    if wall < 0:
        raise RuntimeError(O.ref().ref_last_error().decode())
    return instances / (online.value / threads), wall, online.value


def other_config(args, world, rank, local):
    import numpy as np
    import torch
    from paper_2003_05328_b200 import _lib, ops
    from paper_2003_05328_b200 import protocol as GP
    from paper_2003_05328_b200.shard import ImageShard, gather_outputs
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    lib = _lib.lib()
    gen = torch.Generator().manual_seed(args.seed)
    cores = host_cores()
    extra = {}
    cpu = None
    if args.config == 0:
        M = args.images or 4096
        ctx = ops.Context(n=2048, device=local)
        L = ops.LayerOps(ctx, ops.ConvSpec(32, 32, 3, 3, True, 1, 1))
        x = torch.randint(0, 256, (M, 1, 32, 32), dtype=torch.uint8, generator=gen).to(dev)
        w = torch.randint(-128, 128, (1, 1, 3, 3), dtype=torch.int32, generator=gen).to(dev)
        _, key = ops.secret_sample(ctx, args.seed)
        we = L.prepare_weights(w)
        ws = L.workspace(M)
        out = torch.empty((M, 1, 32, 32), dtype=torch.int32, device=dev)
        shard = ImageShard(world * M, world, rank)
        rand = ops.Randomness(seed=args.seed, image_base=shard.start)
        gathered = torch.empty((world * M, 1, 32, 32), dtype=torch.int32, device=dev) if world > 1 else None

        def fn():
            L.forward(key, we, x, rand, ws=ws, out=out)
            if world > 1:
                gather_outputs(out, shard, gathered)  # the one collective: NCCL all-gather of outputs
        total = _time_steps(fn, args.steps, args.warmup, flush, stream)
        value = world * M * args.steps / (total / 1e3)
        unit, workload = "conv/s", f"config0: {M} independent 1->1 3x3 Same convs of 32x32 uint8 per step, n=2048"
        if rank == 0 and not args.no_cpu_baseline:
            thr = max(1, cores // 2)
            v, wall, _ = _ref_sessions([[0, 3, 3, 1, 1, 1, 0]], 32, 32, 1, max(thr, 32), thr, args.seed)
            cpu = {"value": v, "unit": unit, "cores": cores, "kind": "reference",
                   "sample": f"{max(thr, 32)} reference run_inproc sessions (config 0), {thr} concurrent, online"}
    elif args.config == 2:
        n = 2048
        ctx = ops.Context(n=n, device=local)
        cnt = 65536
        buf = torch.randint(0, 1 << 62, (cnt, n), dtype=torch.int64, device=dev, generator=torch.Generator(
            device=dev).manual_seed(args.seed))
        buf = (buf % Q).view(torch.uint64)

        def fn():
            ctx.negacyclic(buf, 0, False, _lib.LAYOUT_BITREV)
            ctx.negacyclic(buf, 0, True, _lib.LAYOUT_BITREV)
        total = _time_steps(fn, args.steps, args.warmup, flush, stream)
        value = world * 2 * cnt * args.steps / (total / 1e3)
        unit, workload = "transforms/s", "config2: 65536 x n=2048 negacyclic NTT then INTT (device layout), 60-bit q"
        nat = _time_steps(lambda: (ctx.negacyclic(buf, 0, False, 0), ctx.negacyclic(buf, 0, True, 0)), 5, 2, flush,
                          stream)
        extra["natural_layout_transforms_per_s"] = 2 * cnt * 5 / (nat / 1e3)
        imad_peak = lib.ensei_gpu_imad_peak(local)
        alg = (ntt_fwd(n) + ntt_inv(n)) * C_Q * cnt
        extra["imad_frac"] = alg * args.steps / (total / 1e3) / imad_peak
        extra["imad_frac_sass_floor"] = extra["imad_frac"] * C_Q_SASS / C_Q
        extra["hbm_GB_s"] = 2 * cnt * n * 16 * args.steps / (total / 1e3) / 1e9
        if rank == 0 and not args.no_cpu_baseline:
            import oracle as O
            sample = np.random.default_rng(0).integers(0, Q, size=(4096, n), dtype=np.uint64)
            secs = O.ref().ref_bench_negacyclic(Q, n, sample.reshape(-1), 4096, cores)
            cpu = {"value": 2 * 4096 / secs, "unit": unit, "cores": cores, "kind": "reference",
                   "sample": "4096 polys x REF NegacyclicPlan forward+inverse over all host threads"}
    elif args.config == 3:
        from paper_2003_05328_b200 import configs as CF
        imgs = args.images or CF.CONFIG3_IMAGES
        ctx = ops.Context(n=2048, device=local)
        sched = (CF.CONFIG3_SCHEDULE if args.pack == 1 else
                 CF.CONFIG3_SCHEDULE_PACKED if args.grid == 0 else CF.CONFIG3_SCHEDULE_GRID)
        ws = [torch.randint(-128, 128, s_, dtype=torch.int32, generator=gen) for s_ in CF.CONFIG3_WEIGHTS]
        sess = GP.Session(ctx, sched, 32, 32, ws)
        shard = ImageShard(world * imgs, world, rank)  # contiguous image shards, global image ids
        x_h = torch.randint(0, 256, (imgs, 3, 32, 32), dtype=torch.uint8,
                            generator=torch.Generator().manual_seed(args.seed * 7919 + shard.start))
        x = x_h.to(dev)
        _, key = ops.secret_sample(ctx, args.seed)
        # ids aligned to every layer's pack (3, 12 and 32 images per block: multiples of 96)
        id_base = rank * (-(-imgs // 96)) * 96
        rands = [ops.Randomness(seed=args.seed, layer=li, image_base=id_base) for li in range(len(sched))]
        out3 = {}
        gathered = torch.empty((world * imgs, 16, 8, 8), dtype=torch.int32, device=dev) if world > 1 else None

        def fn():
            out3["y"] = sess.run(key, x, lambda li: rands[li])
            if world > 1:
                gather_outputs(out3["y"], shard, gathered)  # NCCL all-gather of the outputs
        total = _time_steps(fn, args.steps, args.warmup, flush, stream)
        value = world * imgs * args.steps / (total / 1e3)
        unit = "images/s"
        workload = (f"config3: {imgs} images x 3x32x32 through 7 conv layers (3->64, 64->64 @32; 64->128, "
                    "128->128 @16; 128->128 3x3, 128->128 1x1, 128->16 1x1 @8), ReLU, 2x2 max-pool after L2/L4")
        extra["mac_paths"] = [lo.mac_path(imgs) for lo in sess.layers if lo is not None]
        extra["packs"] = [lo.pack for lo in sess.layers if lo is not None]
        extra["grids"] = [int(lo.geom.Lh) for lo in sess.layers if lo is not None]
        if rank == 0:  # sampled outputs of the last timed step vs the plaintext chain (oracle as checker)
            try:
                from oracle import protocol as OP
                osched = [OP.Conv(s_.fh, s_.fw, s_.same, s_.cin, s_.cout) if hasattr(s_, "cin") else
                          OP.Act(s_.fn, s_.pool2) for s_ in sched]
                picks = sorted({0, imgs - 1})
                ok = all(bool((out3["y"][i].cpu().numpy().astype(np.uint64) == OP.plain_protocol(
                    osched, x_h[i].numpy().astype(np.int64), [w.numpy().astype(np.int64) for w in ws], Q, P, 2048,
                    OP.default_workers())).all()) for i in picks)
                extra["verify"] = {"images": [shard.start + i for i in picks], "ok": ok,
                                   "against": "plaintext chain (oracle conv_direct + ReLU + pool; pinned to REF "
                                              "reference_pipeline per segment by tests/test_config3_pin.py)"}
            except Exception as e:  # noqa: BLE001
                extra["verify"] = {"ok": None, "error": str(e)}
        if rank == 0 and not args.no_cpu_baseline:
            thr = max(1, cores // 2)
            nimg = max(8, thr)
            segs = [([[0, 3, 3, 1, 3, 64, 0], [1, 0, 0, 0, 0, 0, 0], [0, 3, 3, 1, 64, 64, 0]], 32, 3),
                    ([[0, 3, 3, 1, 64, 128, 0], [1, 0, 0, 0, 0, 0, 0], [0, 3, 3, 1, 128, 128, 0]], 16, 64),
                    ([[0, 3, 3, 1, 128, 128, 0], [1, 0, 0, 0, 0, 0, 0], [0, 1, 1, 1, 128, 128, 0],
                      [1, 0, 0, 0, 0, 0, 0], [0, 1, 1, 1, 128, 16, 0]], 8, 128)]
            per_img = 0.0
            for rows, Hs, cin in segs:
                _, _, online = _ref_sessions(rows, Hs, Hs, cin, nimg, thr, args.seed)
                per_img += online / nimg
            cpu = {"value": thr / per_img, "unit": unit, "cores": cores, "kind": "reference",
                   "sample": f"{nimg} images through REF run_inproc sessions of the 3 reference-expressible "
                             f"segments, {thr} concurrent sessions (2 threads each); online phase "
                             f"{per_img:.2f} s per image per session, Bob weight prep excluded"}
    else:
        raise SystemExit(f"unknown config {args.config}")
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": unit, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": total / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic, seeded",
                "config": {"workload": workload, "config_index": args.config}, "cpu_baseline": cpu, **extra}
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
