"""Generates tests/golden/golden.json from the COMPILED REFERENCE (oracle/_ref).

Run in the build container (where /root/reference exists and oracle/_ref is
built):  python tests/golden/make_golden.py

Every value here comes out of the unmodified reference library through
oracle/ref_harness.cpp; inputs are derived from fixed seeds (numpy PCG64 or the
reference's own Rng), so the fixture stays small: full vectors for small cases,
FNV-1a-64 digests (over little-endian u64) plus a short prefix for large ones.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

Q = 576460803525083137
P = 638977
RNS = [576460803525083137, 576461033843064833, 576461054781063169]


def fnv(arr) -> str:
    h = 1469598103934665603
    for b in np.ascontiguousarray(arr, dtype="<u8").tobytes():
        h ^= b
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return "%016x" % h


def proto_case(seed, H, W, desc, img_gen, n=2048, q=Q, mode=1, capture=True):
    """Runs the reference protocol; returns digests of everything observable."""
    R = O.ref()
    desc_arr = np.array(desc, dtype=np.int32).reshape(-1)
    convs = [d for d in desc if d[0] == 0]
    wcount = sum(d[1] * d[2] * d[4] * d[5] for d in convs)
    g = O.MTRng(seed, 0xDA7A)
    img = np.array([img_gen(g) for _ in range(convs[0][4] * H * W)], dtype=np.int64)
    w = np.array([g.uniform_below(256) - 128 for _ in range(wcount)], dtype=np.int64)
    # final output size: walk shapes
    h, ww, ch = H, W, convs[0][4]
    for d in desc:
        if d[0] == 0:
            h = h if d[3] else h - d[1] + 1
            ww = ww if d[3] else ww - d[2] + 1
            ch = d[5]
    out = np.zeros(ch * h * ww, np.uint64)
    hashes = np.zeros(6, np.uint64)
    ctrs = np.zeros(8, np.uint64)
    c0 = convs[0]
    L = O.layer(q, P, n, H, W, c0[1], c0[2], c0[3], c0[4], c0[5])
    a2b = np.zeros(c0[4] * L.blocks * 2 * n, np.uint64)
    b2a = np.zeros(c0[5] * L.blocks * 2 * n, np.uint64)
    O.ref_check(R.ref_run_protocol(P, q, n, 4.0, mode, seed, H, W, len(desc), desc_arr, img, w, out,
                                   O._ptr(hashes), O._ptr(ctrs), 0,
                                   O._ptr(a2b) if capture else None,
                                   O._ptr(b2a) if capture else None, None, None))
    pipe = np.zeros_like(out)
    O.ref_check(R.ref_reference_pipeline(P, q, n, H, W, len(desc), desc_arr, img, w, pipe))
    assert (pipe == out).all()
    return {
        "seed": seed, "H": H, "W": W, "n": n, "q": q, "mode": mode, "desc": desc,
        "out_fnv": fnv(out), "out_prefix": [int(v) for v in out[:8]],
        "alice_sent": "%016x" % int(hashes[0]), "alice_recv": "%016x" % int(hashes[1]),
        "alice_bytes_sent": int(hashes[4]), "bob_bytes_sent": int(hashes[5]),
        "counters_alice": [int(v) for v in ctrs[:4]], "counters_bob": [int(v) for v in ctrs[4:]],
        "ct_a2b_fnv": fnv(a2b) if capture else None, "ct_b2a_fnv": fnv(b2a) if capture else None,
    }


def main():
    R = O.ref()
    G = {"p": P, "q": Q, "rns": RNS}
    # --- SPEC KATs, evaluated by the reference code itself (SPEC.md examples)
    kat = {}
    kat["mul_5_7_17"] = int(R.ref_mulmod(5, 7, 17))
    kat["find_prime_12289_1_4096"] = int(R.ref_find_prime(12289, 1, 4096))
    kat["find_prime_36864_1_4096"] = int(R.ref_find_prime(36864, 1, 4096))  # SPEC says 147457; code gives 40961
    x = np.array([0, 1, 0, 0], np.uint64)
    O.ref_check(R.ref_ntt1d(17, 4, x, 4, 0))
    kat["ntt_0100_w4_p17"] = [int(v) for v in x]
    x = np.array([3, 3, 3, 3], np.uint64)
    O.ref_check(R.ref_ntt1d(17, 4, x, 4, 0))
    kat["ntt_3333_w4_p17"] = [int(v) for v in x]
    x = np.array([1, 1, 1, 1], np.uint64)
    O.ref_check(R.ref_ntt1d(17, 4, x, 4, 1))
    kat["intt_1111_w4_p17"] = [int(v) for v in x]
    o = np.zeros(1, np.uint64)
    O.ref_check(R.ref_conv_oracle(17, np.array([1, 2, 3, 4], np.int64), 2, 2,
                                  np.array([1, 0, 0, 1], np.int64), 2, 2, 0, o))
    kat["conv_oracle_valid_2x2"] = int(o[0])
    for (pp, nm) in ((P, "p"), (Q, "q")) + tuple((r, f"rns{i}") for i, r in enumerate(RNS)):
        gen = O.C.c_uint64()
        ta = O.C.c_int32()
        O.ref_check(R.ref_field_info(pp, O.C.byref(gen), O.C.byref(ta)))
        kat[f"generator_{nm}"] = int(gen.value)
        kat[f"two_adicity_{nm}"] = int(ta.value)
    for L in (8, 16, 32, 64):
        kat[f"omega_{L}"] = int(R.ref_root_of_unity(L, P))
    for n in (2048, 4096, 8192):
        psi = O.C.c_uint64()
        O.ref_check(R.ref_plan_psi(Q, n, O.C.byref(psi)))
        kat[f"psi_q_{n}"] = int(psi.value)
        O.ref_check(R.ref_plan_psi(P, n, O.C.byref(psi)))
        kat[f"psi_p_{n}"] = int(psi.value)
    ph, pw = O.C.c_uint32(), O.C.c_uint32()
    for H, f in ((32, 3), (16, 3), (8, 3), (8, 1)):
        O.ref_check(R.ref_geometry(P, H, H, f, f, 1, O.C.byref(ph), O.C.byref(pw)))
        kat[f"padded_{H}_{f}"] = [int(ph.value), int(pw.value)]
    G["kat"] = kat

    # --- negacyclic transforms over q (config 2 and the RNS primes): seeded inputs
    rng = np.random.default_rng(2003_05328)
    neg = []
    for qq in [Q] + RNS[1:]:
        for n in (16, 2048, 4096, 8192):
            if (qq - 1) % (2 * n):
                continue
            x = rng.integers(0, qq, size=(2, n), dtype=np.uint64)
            y = x.copy()
            O.ref_check(R.ref_negacyclic(qq, n, y.reshape(-1), 2, 0))
            z = x.copy()
            O.ref_check(R.ref_negacyclic(qq, n, z.reshape(-1), 2, 1))
            e = {"q": qq, "n": n, "in_fnv": fnv(x), "fwd_fnv": fnv(y), "inv_fnv": fnv(z),
                 "fwd_prefix": [int(v) for v in y[0, :4]], "inv_prefix": [int(v) for v in z[0, :4]]}
            if n == 16:
                e["in"] = [int(v) for v in x.reshape(-1)]
                e["fwd"] = [int(v) for v in y.reshape(-1)]
                e["inv"] = [int(v) for v in z.reshape(-1)]
            neg.append(e)
    G["negacyclic"] = neg
    G["negacyclic_seed"] = 2003_05328

    # --- negacyclic over p (slot encode/decode)
    slots = []
    for n in (2048, 4096, 8192):
        x = rng.integers(0, P, size=n, dtype=np.uint64)
        enc = x.copy()
        O.ref_check(R.ref_slots(P, Q, n, enc, 0))
        dec = x.copy()
        O.ref_check(R.ref_slots(P, Q, n, dec, 1))
        slots.append({"n": n, "in_fnv": fnv(x), "encode_fnv": fnv(enc), "decode_fnv": fnv(dec)})
    G["slots"] = slots

    # --- 2D image transforms over p
    t2 = []
    for Lh in (8, 16, 32, 64):
        x = rng.integers(0, P, size=(2, Lh, Lh), dtype=np.uint64)
        y = x.copy()
        O.ref_check(R.ref_ntt2d(P, Lh, Lh, y.reshape(-1), 2, 0))
        z = x.copy()
        O.ref_check(R.ref_ntt2d(P, Lh, Lh, z.reshape(-1), 2, 1))
        e = {"L": Lh, "in_fnv": fnv(x), "fwd_fnv": fnv(y), "inv_fnv": fnv(z)}
        if Lh == 8:
            e["in"] = [int(v) for v in x.reshape(-1)]
            e["fwd"] = [int(v) for v in y.reshape(-1)]
            e["inv"] = [int(v) for v in z.reshape(-1)]
        t2.append(e)
    G["ntt2d"] = t2

    # --- protocol runs (two parties, in-process, FreqDirect and Baseline)
    pix = lambda g: g.uniform_below(256)  # noqa: E731
    G["proto"] = [
        # Appendix B config-0 golden run (seed 0, 1->1, Same, 32x32, 3x3)
        proto_case(0, 32, 32, [[0, 3, 3, 1, 1, 1, 0]], pix),
        proto_case(0, 32, 32, [[0, 3, 3, 1, 1, 1, 0]], pix, mode=0),
        # a small two-conv stack with ReLU between (exercises HomRec)
        proto_case(7, 8, 8, [[0, 3, 3, 1, 2, 3, 0], [1, 0, 0, 0, 0, 0, 0], [0, 3, 3, 1, 3, 2, 0]], pix),
        # Valid conv, 1x1 filter
        proto_case(11, 8, 8, [[0, 1, 1, 0, 4, 2, 0]], pix),
        # config-1 channel shape on a 16x16 image (one instance)
        proto_case(3, 16, 16, [[0, 3, 3, 1, 16, 16, 0]], pix),
    ]
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
    with open(path, "w") as f:
        json.dump(G, f, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
