"""GPU parity: batched transforms through the C ABI vs the oracle / golden vectors."""
import numpy as np
import pytest
import torch

import oracle as O
from conftest import fnv
from gpu_util import P, Q, RNS, bitrev_perm, to_np, u64

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ops():
    from paper_2003_05328_b200 import ops as _ops
    return _ops


@pytest.mark.parametrize("n", [2048, 4096, 8192])
def test_negacyclic_q_both_layouts(ops, n):
    ctx = ops.Context(n=n)
    rng = np.random.default_rng(n)
    x = rng.integers(0, Q, size=(19, n), dtype=np.uint64)
    want = O.negacyclic(x, Q)
    br = bitrev_perm(n)
    for layout in (0, 1):
        d = u64(x)
        ctx.negacyclic(d, 0, False, layout)
        got = to_np(d)
        assert (got[:, br] == want).all() if layout == 1 else (got == want).all()
        ctx.negacyclic(d, 0, True, layout)
        assert (to_np(d) == x).all()


def test_negacyclic_rns_primes(ops):
    ctx = ops.Context(n=8192, q=RNS)
    rng = np.random.default_rng(3)
    for i, q in enumerate(RNS):
        x = rng.integers(0, q, size=(5, 8192), dtype=np.uint64)
        d = u64(x)
        ctx.negacyclic(d, i, False, 0)
        assert (to_np(d) == O.negacyclic(x, q)).all()
        ctx.negacyclic(d, i, True, 0)
        assert (to_np(d) == x).all()


@pytest.mark.parametrize("n", [2048, 4096, 8192])
def test_slots_encode_decode(ops, n):
    ctx = ops.Context(n=n)
    x = np.random.default_rng(n + 1).integers(0, P, size=(7, n), dtype=np.uint64)
    d = u64(x)
    ctx.encode_slots(d)
    assert (to_np(d) == O.negacyclic(x, P, inverse=True)).all()
    d = u64(x)
    ctx.decode_slots(d)
    assert (to_np(d) == O.negacyclic(x, P)).all()


@pytest.mark.parametrize("L", [1, 2, 4, 8, 16, 32, 64])
def test_ntt2d(ops, L):
    ctx = ops.Context(n=2048)
    x = np.random.default_rng(L).integers(0, P, size=(5, L, L), dtype=np.uint64)
    for inv in (False, True):
        d = u64(x)
        ctx.ntt_2d(d, inverse=inv)
        assert (to_np(d) == O.ntt2d(x, P, inverse=inv)).all()


def test_golden_negacyclic_vectors(ops, golden):
    rng = np.random.default_rng(golden["negacyclic_seed"])
    for e in golden["negacyclic"]:
        x = rng.integers(0, e["q"], size=(2, e["n"]), dtype=np.uint64)
        if e["n"] < 2048:
            continue  # the device path starts at n = 2048
        ctx = ops.Context(n=e["n"], q=(e["q"],))
        d = u64(x)
        ctx.negacyclic(d, 0, False, 0)
        assert fnv(to_np(d)) == e["fwd_fnv"]
        d = u64(x)
        ctx.negacyclic(d, 0, True, 0)
        assert fnv(to_np(d)) == e["inv_fnv"]


def test_golden_2d_vectors(ops, golden):
    ctx = ops.Context(n=2048)
    e = [g for g in golden["ntt2d"] if g["L"] == 8][0]
    x = np.array(e["in"], np.uint64).reshape(2, 8, 8)
    d = u64(x)
    ctx.ntt_2d(d)
    assert [int(v) for v in to_np(d).reshape(-1)] == e["fwd"]


def test_config2_scale_roundtrip(ops):
    """65536 polynomials x n=2048 (config 2): forward then inverse is the identity;
    a random subset matches the CPU NTT bit-exactly."""
    ctx = ops.Context(n=2048)
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randint(0, 2**62, (65536, 2048), dtype=torch.int64, device="cuda", generator=g)
    x = (x % Q).view(torch.uint64)
    ref = x.clone()
    ctx.negacyclic(x, 0, False, 0)
    idx = torch.randperm(65536, generator=torch.Generator().manual_seed(1))[:24]
    sub = to_np(ref.view(torch.int64)[idx.cuda()]).view(np.uint64)
    assert (to_np(x.view(torch.int64)[idx.cuda()]).view(np.uint64) == O.negacyclic(sub, Q)).all()
    ctx.negacyclic(x, 0, True, 0)
    assert torch.equal(x.view(torch.int64), ref.view(torch.int64))


def test_errors_map_to_reference_types(ops):
    from paper_2003_05328_b200 import EnseiError
    with pytest.raises(EnseiError, match="Error"):
        ops.Context(n=2048, q=(576460752303423619,))  # not prime / not 1 mod p
    ctx = ops.Context(n=1024)
    d = u64(np.zeros((1, 1024), np.uint64))
    with pytest.raises(EnseiError, match="Unsupported"):
        ctx.negacyclic(d, 0, False, 0)
    ctx2 = ops.Context(n=2048)
    d = u64(np.zeros((0, 2048), np.uint64))
    ctx2.negacyclic(d, 0, False, 0)  # empty batch is a no-op
    with pytest.raises(EnseiError, match="InvalidArgument"):
        ctx2.negacyclic(u64(np.zeros((1, 2048), np.uint64)), 5, False, 0)
