"""CPU: the C restatement (oracle/) against the LIVE compiled reference
(oracle/_ref/libensei_ref.so) on fresh seeded inputs -- beyond the golden fixtures."""
import numpy as np
import pytest

import oracle as O
from oracle import protocol as OP

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")

Q = 576460803525083137
P = 638977
RNS = [576460803525083137, 576461033843064833, 576461054781063169]


@pytest.mark.parametrize("q", RNS + [P])
@pytest.mark.parametrize("n", [16, 2048, 8192])
def test_negacyclic_vs_reference(q, n):
    rng = np.random.default_rng(n ^ (q & 0xFFFF))
    x = rng.integers(0, q, size=(2, n), dtype=np.uint64)
    for inv in (0, 1):
        y = x.copy()
        O.ref_check(O.ref().ref_negacyclic(q, n, y.reshape(-1), 2, inv))
        assert (O.negacyclic(x, q, inverse=bool(inv)) == y).all()


@pytest.mark.parametrize("L", [2, 4, 8, 16, 32, 64, 3, 12, 13, 24, 39])
def test_ntt2d_vs_reference(L):
    # the non-powers-of-two take REF's O(L^2) ntt_direct (ntt.cpp:35-49): the lengths of the
    # device's grid override (12, 24, 39) and their prime-factor pieces
    rng = np.random.default_rng(L)
    x = rng.integers(0, P, size=(3, L, L), dtype=np.uint64)
    for inv in (0, 1):
        y = x.copy()
        O.ref_check(O.ref().ref_ntt2d(P, L, L, y.reshape(-1), 3, inv))
        assert (O.ntt2d(x, P, inverse=bool(inv)) == y).all()


def _run_both(seed, H, W, desc, n=2048, q=Q):
    R = O.ref()
    g = O.MTRng(seed, 0xDA7A)
    convs = [d for d in desc if d[0] == 0]
    img = np.array([g.uniform_below(256) for _ in range(convs[0][4] * H * W)], np.int64)
    ws = [np.array([g.uniform_below(256) - 128 for _ in range(d[1] * d[2] * d[4] * d[5])], np.int64)
          .reshape(d[5], d[4], d[1], d[2]) for d in convs]
    h, w, ch = H, W, convs[0][4]
    for d in desc:
        if d[0] == 0:
            h, w, ch = (h if d[3] else h - d[1] + 1), (w if d[3] else w - d[2] + 1), d[5]
    out = np.zeros(ch * h * w, np.uint64)
    O.ref_check(R.ref_run_protocol(P, q, n, 4.0, 1, seed, H, W, len(desc), np.array(desc, np.int32).reshape(-1),
                                   img, np.concatenate([x.reshape(-1) for x in ws]), out, None, None, 0, None,
                                   None, None, None))
    sched = [OP.Conv(d[1], d[2], bool(d[3]), d[4], d[5]) if d[0] == 0 else OP.Act(d[6]) for d in desc]
    mine, _ = OP.run_protocol(sched, img.reshape(convs[0][4], H, W), ws, OP.RefRandomness(seed, n, q, P), q, P, n)
    return out, mine.reshape(-1)


@pytest.mark.parametrize("seed", [101, 202])
def test_protocol_relu_stack_vs_reference(seed):
    desc = [[0, 3, 3, 1, 2, 3, 0], [1, 0, 0, 0, 0, 0, 0], [0, 1, 1, 1, 3, 2, 0], [1, 0, 0, 0, 0, 0, 2]]
    ref, mine = _run_both(seed, 8, 8, desc)
    assert (ref == mine).all()


def test_protocol_valid_and_n4096_vs_reference():
    ref, mine = _run_both(5, 12, 12, [[0, 5, 3, 0, 2, 2, 0]], n=4096)
    assert (ref == mine).all()


def test_square_activation_semantics():
    # REF trusted_activation Square (protocol.cpp:252-257): y^2 on the centered lift,
    # RangeOverflow when y^2 > p/2.  (Not run through REF run_inproc: an overflow there
    # throws on Alice's thread and leaves Bob blocked in recv -- a reference behaviour.)
    v = np.array([0, 1, P - 1, 500, P - 565], np.uint64)
    assert O.lib().eo_activation(v, v.size, P, 1) == 0
    assert list(v) == [0, 1, 1, 250000, 319225]
    big = np.array([566], np.uint64)
    assert O.lib().eo_activation(big, 1, P, 1) == -1


def test_reference_rng_restatement():
    for seed, salt in ((0, 0xA11CE), (12345, 0xB0B), (2**63 + 7, 0xDA7A)):
        r = O.MTRng(seed, salt)
        out = np.empty(500, np.int64)
        O.ref_check(O.ref().ref_rng_draw(seed, salt, 1, 2, 0, 4.0, 500, out))
        assert [r.gaussian(4.0) for _ in range(500)] == list(out)
        r = O.MTRng(seed, salt)
        O.ref_check(O.ref().ref_rng_draw(seed, salt, 1, 1, Q, 0.0, 500, out))
        assert [r.uniform_below(Q) for _ in range(500)] == list(out.astype(np.uint64))


@pytest.mark.parametrize("H,grid,pack", [(32, 39, 1), (16, 24, 3), (8, 12, 12)])
def test_oracle_grid_override_layer_recombines_to_ref_conv(H, grid, pack):
    """The oracle's layer restatement on an overridden grid (oracle.protocol.set_grid, the
    checker of the device's ensei_conv_desc::grid) still reconstructs REF's conv_oracle
    output: the padded side only has to hold the linear convolution and divide p - 1."""
    from oracle import protocol as OP
    cin, cout, n = 2, 2, 2048
    rng = np.random.default_rng(grid)
    x = rng.integers(0, 256, size=(pack, cin, H, H)).astype(np.uint64)
    w = rng.integers(-128, 128, size=(cout, cin, 3, 3)).astype(np.int64)
    L = OP.set_grid(O.layer(Q, P, n, H, H, 3, 3, 1, cin, cout), grid)
    L.pack = pack
    assert (L.Lh, L.Lw, L.blocks) == (grid, grid, 1)
    pr = OP.PhiloxRandomness(9, 0, n, Q, P)
    te = OP.secret_eval(L, pr.secret())
    e, a = pr.enc(0, cin, 1)
    r = OP.run_layer(L, te, x if pack > 1 else x[0], None, OP.prepare_weights(L, w), e, a, pr.share(0, cout, 1))
    al = np.asarray(r["alice"]).reshape(pack, -1)
    bo = np.asarray(r["bob"]).reshape(pack, -1)
    for i in range(pack):
        want = np.zeros(cout * H * H, np.int64)
        for o in range(cout):
            acc = np.zeros(H * H, np.int64)
            for c in range(cin):
                y = np.zeros(H * H, np.uint64)
                O.ref_check(O.ref().ref_conv_oracle(P, x[i, c].astype(np.int64).reshape(-1), H, H,
                                                    w[o, c].reshape(-1), 3, 3, 1, y))
                acc = (acc + y.astype(np.int64)) % P
            want[o * H * H:(o + 1) * H * H] = acc
        assert (((al[i] + bo[i]) % np.uint64(P)).astype(np.int64) == want).all(), i
