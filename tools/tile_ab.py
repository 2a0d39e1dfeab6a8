"""A/B of the RNS tile kernels (ensei_gpu_set_tile_variant 0 vs 1) at config 4's shape.

    python tools/tile_ab.py [--images 256] [--reps 3] [--pack 2]

For each generation: Enc, HomShare(+MAC), Dec stage by stage on the same inputs, outputs
compared bit for bit (generation 0 is the oracle-checked one, tests/test_gpu_configs.py),
then per-kernel CUDA-event times through ensei_gpu_profile over `reps` fused layers.
Prints one JSON line.
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2003_05328_b200 import _lib, ops  # noqa: E402
from paper_2003_05328_b200.configs import RNS as RNS_PRIMES  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--images", type=int, default=256)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--pack", type=int, default=2)
    ap.add_argument("--cin", type=int, default=64)
    ap.add_argument("--cout", type=int, default=128)
    ap.add_argument("--hw", type=int, default=32)
    ap.add_argument("--grid", type=int, default=0, help="grid override (39): only the second generation runs")
    a = ap.parse_args()
    lib = _lib.lib()
    ctx = ops.Context(n=8192, q=tuple(RNS_PRIMES))
    g = torch.Generator().manual_seed(7)
    x = torch.randint(0, 256, (a.images, a.cin, a.hw, a.hw), dtype=torch.uint8, generator=g).cuda()
    w = torch.randint(-128, 128, (a.cout, a.cin, 3, 3), dtype=torch.int32, generator=g).cuda()
    L = ops.LayerOps(ctx, ops.ConvSpec(a.hw, a.hw, 3, 3, True, a.cin, a.cout, pack=a.pack, grid=a.grid))
    _, key = ops.secret_sample(ctx, 5)
    we = L.prepare_weights(w)
    R = ops.Randomness(seed=5, image_base=64 * a.pack)
    ws = L.workspace(a.images)
    res, out = {}, {}
    for gen in ((1,) if a.grid else (0, 1)):
        _lib.check(lib.ensei_gpu_set_tile_variant(gen))
        ct = L.alice_encrypt(key, x, R)
        ct_out, bob = L.bob_eval(ct.clone(), we, R)
        alice = L.alice_decrypt(key, ct_out)
        fused, fa, fb = L.forward(key, we, x, R, ws=ws, want_shares=True)
        torch.cuda.synchronize()
        out[gen] = (ct, ct_out, bob, alice, fused, fa, fb)
        for _ in range(2):
            L.forward(key, we, x, R, ws=ws)
        torch.cuda.synchronize()
        _lib.profile(True)
        for _ in range(a.reps):
            L.forward(key, we, x, R, ws=ws)
        torch.cuda.synchronize()
        prof = _lib.profile_read()
        _lib.profile(False)
        res[f"gen{gen}_ms"] = {k: round(v[0] / v[1], 4) for k, v in prof.items()}
        # unprofiled wall (PDL + the HomShare fork on)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            L.forward(key, we, x, R, ws=ws)
        e1.record()
        torch.cuda.synchronize()
        res[f"gen{gen}_layer_ms"] = round(e0.elapsed_time(e1) / a.reps, 4)
        _lib.check(lib.ensei_gpu_set_tile_variant(gen + 2))  # HomShare in line (no fork)
        L.forward(key, we, x, R, ws=ws)
        e0.record()
        for _ in range(a.reps):
            L.forward(key, we, x, R, ws=ws)
        e1.record()
        torch.cuda.synchronize()
        res[f"gen{gen}_layer_nofork_ms"] = round(e0.elapsed_time(e1) / a.reps, 4)
    _lib.check(lib.ensei_gpu_set_tile_variant(1))
    names = ("ct_in", "ct_out", "bob", "alice", "out", "fused_alice", "fused_bob")
    if a.grid:
        out[0] = out[1]
    res["equal"] = {n: bool(torch.equal(p, q)) for n, p, q in zip(names, out[0], out[1])}
    res["stagewise_vs_fused"] = bool(torch.equal(out[1][3], out[1][5]) and torch.equal(out[1][2], out[1][6]))
    res["shape"] = vars(a)
    print(json.dumps(res))
    if not all(res["equal"].values()):
        for n, p, q in zip(names, out[0], out[1]):
            if not torch.equal(p, q):
                d = (p != q)
                print(n, "mismatches", int(d.sum()), "of", d.numel(), "first", d.nonzero()[:4].tolist(), file=sys.stderr)
        sys.exit(1)


if __name__ == "__main__":
    main()
