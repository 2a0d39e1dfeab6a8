"""CPU: pin the C restatement (oracle/) against the reference's golden vectors.

Golden values in tests/golden/golden.json were produced by the compiled,
unmodified reference (tests/golden/make_golden.py); these tests need only the
C restatement, so they also hold where the reference .so is absent.
"""
import numpy as np
import pytest

import oracle as O
from oracle import protocol as OP
from conftest import fnv

Q = 576460803525083137
P = 638977


def test_kats(golden):
    k = golden["kat"]
    L = O.lib()
    assert L.eo_mulmod(5, 7, 17) == k["mul_5_7_17"] == 1
    assert L.eo_find_prime(12289, 1, 4096) == k["find_prime_12289_1_4096"]
    assert L.eo_find_prime(36864, 1, 4096) == k["find_prime_36864_1_4096"] == 40961
    for name, inv, vec in (("ntt_0100_w4_p17", 0, [0, 1, 0, 0]), ("ntt_3333_w4_p17", 0, [3, 3, 3, 3]),
                           ("intt_1111_w4_p17", 1, [1, 1, 1, 1])):
        x = np.array(vec, np.uint64)
        assert L.eo_ntt_1d(x, 4, 4, 17, inv) == 0
        assert list(x) == k[name]
    for nm, m in (("p", P), ("q", Q)) + tuple((f"rns{i}", r) for i, r in enumerate(golden["rns"])):
        assert L.eo_primitive_root(m) == k[f"generator_{nm}"]
    for Lh in (8, 16, 32, 64):
        assert L.eo_root_of_unity(Lh, P) == k[f"omega_{Lh}"]


def test_padded_geometry(golden):
    for H, f in ((32, 3), (16, 3), (8, 3), (8, 1)):
        Ly = O.layer(Q, P, 2048, H, H, f, f, 1, 1, 1)
        assert [Ly.Lh, Ly.Lw] == golden["kat"][f"padded_{H}_{f}"]


def test_negacyclic_golden(golden):
    rng = np.random.default_rng(golden["negacyclic_seed"])
    for e in golden["negacyclic"]:
        x = rng.integers(0, e["q"], size=(2, e["n"]), dtype=np.uint64)
        assert fnv(x) == e["in_fnv"]
        y = O.negacyclic(x, e["q"])
        z = O.negacyclic(x, e["q"], inverse=True)
        assert fnv(y) == e["fwd_fnv"] and fnv(z) == e["inv_fnv"]
        if "fwd" in e:
            assert [int(v) for v in y.reshape(-1)] == e["fwd"]
        assert (O.negacyclic(y, e["q"], inverse=True) == x).all()


def test_slots_and_2d_golden(golden):
    rng = np.random.default_rng(golden["negacyclic_seed"])
    for e in golden["negacyclic"]:  # replay the generator in fixture order
        rng.integers(0, e["q"], size=(2, e["n"]), dtype=np.uint64)
    for e in golden["slots"]:
        x = rng.integers(0, P, size=e["n"], dtype=np.uint64)
        assert fnv(x) == e["in_fnv"]
        assert fnv(O.negacyclic(x, P, inverse=True)) == e["encode_fnv"]
        assert fnv(O.negacyclic(x, P)) == e["decode_fnv"]
    for e in golden["ntt2d"]:
        x = rng.integers(0, P, size=(2, e["L"], e["L"]), dtype=np.uint64)
        assert fnv(x) == e["in_fnv"]
        assert fnv(O.ntt2d(x, P)) == e["fwd_fnv"]
        assert fnv(O.ntt2d(x, P, inverse=True)) == e["inv_fnv"]


def _proto_inputs(case):
    g = O.MTRng(case["seed"], 0xDA7A)
    convs = [d for d in case["desc"] if d[0] == 0]
    H, W = case["H"], case["W"]
    img = np.array([g.uniform_below(256) for _ in range(convs[0][4] * H * W)], np.int64)
    ws = []
    for d in convs:
        cnt = d[1] * d[2] * d[4] * d[5]
        ws.append(np.array([g.uniform_below(256) - 128 for _ in range(cnt)], np.int64)
                  .reshape(d[5], d[4], d[1], d[2]))
    sched = [OP.Conv(d[1], d[2], bool(d[3]), d[4], d[5]) if d[0] == 0 else OP.Act(d[6]) for d in case["desc"]]
    return img.reshape(convs[0][4], H, W), ws, sched


@pytest.mark.parametrize("idx", range(5))
def test_protocol_golden(golden, idx):
    """Whole-session parity: the restatement, fed the reference's own mt19937_64
    randomness in consumption order, reproduces the reference's wire ciphertexts
    (FreqDirect mode) and reconstructed outputs."""
    case = golden["proto"][idx]
    img, ws, sched = _proto_inputs(case)
    rand = OP.RefRandomness(case["seed"], case["n"], case["q"], P)
    out, trace = OP.run_protocol(sched, img, ws, rand, case["q"], P, case["n"], want=("ct",))
    assert fnv(out) == case["out_fnv"]
    if case["mode"] == 1:
        assert fnv(trace[0]["ct_in"]) == case["ct_a2b_fnv"]
        assert fnv(trace[0]["ct_out"]) == case["ct_b2a_fnv"]


def test_conv_direct_matches_golden(golden):
    case = golden["proto"][0]
    img, ws, _ = _proto_inputs(case)
    L = O.layer(Q, P, 2048, 32, 32, 3, 3, 1, 1, 1)
    out = np.zeros(1024, np.uint64)
    O.lib().eo_conv_direct(O.C.byref(L), (img.reshape(-1) % P).astype(np.uint64), ws[0].reshape(-1), out)
    assert fnv(out) == case["out_fnv"]


def test_philox_kat():
    # Random123 known-answer vectors for Philox4x32-10
    L = O.lib()
    out = np.zeros(4, np.uint32)
    L.eo_philox4x32_10(np.zeros(4, np.uint32), np.zeros(2, np.uint32), out)
    assert [hex(v) for v in out] == ["0x6627e8d5", "0xe169c58d", "0xbc57ac4c", "0x9b00dbd8"]
    L.eo_philox4x32_10(np.full(4, 0xFFFFFFFF, np.uint32), np.full(2, 0xFFFFFFFF, np.uint32), out)
    assert [hex(v) for v in out] == ["0x408f276d", "0x41c83b0e", "0xa20bc7c6", "0x6d5451fd"]
    L.eo_philox4x32_10(np.array([0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344], np.uint32),
                       np.array([0xa4093822, 0x299f31d0], np.uint32), out)
    assert [hex(v) for v in out] == ["0xd16cfe09", "0x94fdcceb", "0x5001e420", "0x24126ea1"]


def test_samplers_ranges():
    key = O.lib().eo_fork_seed(1, 0xA11CE)
    t = O.rand_ternary(key, 5, 4096)
    assert set(np.unique(t)) <= {-1, 0, 1} and abs(t.mean()) < 0.1
    e = O.rand_cbd(key, 6, 1 << 15, 20)
    assert e.min() >= -20 and e.max() <= 20 and abs(e.var() - 10) < 0.5
    a = O.rand_uniform_q(key, 7, 4096, Q)
    assert a.max() < Q and a.min() >= 0 and abs(a.astype(np.float64).mean() / Q - 0.5) < 0.03
    s = O.rand_uniform_p(key, 8, 4096, P)
    assert s.max() < P


def test_philox_protocol_roundtrip():
    """Throughput-mode randomness (ternary/CBD/Philox) still reconstructs the exact
    plaintext convolution (reconstructed outputs are pinned by reference_pipeline)."""
    rng = np.random.default_rng(0)
    img = rng.integers(0, 256, size=(2, 8, 8)).astype(np.int64)
    w = rng.integers(-128, 128, size=(3, 2, 3, 3)).astype(np.int64)
    sched = [OP.Conv(3, 3, True, 2, 3)]
    rand = OP.PhiloxRandomness(99, 0, 2048, Q, P)
    out, _ = OP.run_protocol(sched, img, [w], rand, Q, P, 2048)
    L = O.layer(Q, P, 2048, 8, 8, 3, 3, 1, 2, 3)
    direct = np.zeros(3 * 64, np.uint64)
    O.lib().eo_conv_direct(O.C.byref(L), (img.reshape(-1) % P).astype(np.uint64), w.reshape(-1), direct)
    assert (out.reshape(-1) == direct).all()


def test_crt_round_single_prime_matches_decrypt_rule():
    rng = np.random.default_rng(3)
    for _ in range(200):
        phi = int(rng.integers(0, Q, dtype=np.uint64))
        want = ((P * phi + Q // 2) // Q) % P
        assert O.lib().eo_crt_round(np.array([phi], np.uint64), np.array([Q], np.uint64), 1, P) == want
