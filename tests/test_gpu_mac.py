"""ElementMult + channel accumulation (REF protocol.cpp:537-607 conv branch: mul_plain
then add_ct over input channels, ringbfv.cpp:233-263) through ensei_gpu_bob_mac, against
exact Python-integer sums, on the shapes that exercise the kernel's edges: odd K, K
spanning several K-chunks and fold blocks, partial row / column tiles, the small-tile
path, both prime counts, and K past the exact-u128 limit (1008 channels).

ct_out's c1 words carry the HomShare mask on entry (the kernel adds, does not overwrite),
so the test pre-fills them with random residues."""
import numpy as np
import pytest
import torch

from gpu_util import Q, RNS, dev, to_np, u64

pytestmark = pytest.mark.gpu

M30 = (1 << 30) - 1


@pytest.fixture(scope="module")
def ops():
    from paper_2003_05328_b200 import ops as _ops
    return _ops


def _pack(v):
    """Prepared-weight word: (v >> 30) << 32 | (v & (2^30 - 1)) (ensei_gpu.h prepare_weights)."""
    return ((v >> np.uint64(30)) << np.uint64(32)) | (v & np.uint64(M30))


# (n, images, cin, cout, primes): direct kernel for tiny channel counts, small-tile path (rows,
# cols <= 16), large tiles with partial row/col tiles, odd K, K = one fold block + tail, K across
# chunks, K > 1008 (residue carry)
CASES = [
    (2048, 1, 1, 1, 1),           # direct per-slot kernel (cout <= 2, cin <= 4): config 0's 1 -> 1
    (2048, 5, 4, 2, 1),           # direct kernel, several channels
    (8192, 3, 3, 1, 3),           # direct kernel, three primes
    (2048, 3, 5, 7, 1),
    (2048, 8, 16, 16, 1),
    (2048, 3, 13, 36, 1),
    (2048, 3, 40, 36, 1),
    (2048, 9, 64, 20, 1),
    (2048, 2, 1030, 3, 1),
    (8192, 2, 7, 3, 3),
    (8192, 20, 30, 17, 3),
    (2048, 20, 3, 40, 1),         # few input channels, > 16 rows / cols: small tiles, partial ones
    (8192, 9, 12, 20, 3),         # same with three primes, K = 12 (one whole chunk)
]


@pytest.mark.parametrize("n,images,cin,cout,R", CASES)
def test_bob_mac_exact(ops, n, images, cin, cout, R):
    q = (Q,) if R == 1 else RNS
    ctx = ops.Context(n=n, q=q)
    L = ops.LayerOps(ctx, ops.ConvSpec(16, 16, 3, 3, True, cin, cout))
    B = L.B
    rng = np.random.default_rng(n + 7 * cin + cout)
    qs = np.array(q, dtype=np.uint64).reshape(1, 1, 1, 1, R, 1)
    ct = (rng.integers(0, 2**63, size=(images, cin, B, 2, R, n), dtype=np.uint64) % qs)
    w = (rng.integers(0, 2**63, size=(cout, cin, B, R, n), dtype=np.uint64) %
         np.array(q, dtype=np.uint64).reshape(1, 1, 1, R, 1))
    mask = (rng.integers(0, 2**63, size=(images, cout, B, R, n), dtype=np.uint64) %
            np.array(q, dtype=np.uint64).reshape(1, 1, 1, R, 1))
    out = np.zeros((images, cout, B, 2, R, n), dtype=np.uint64)
    out[:, :, :, 1] = mask
    d_out = u64(out)
    L.bob_mac(u64(ct), L.weights_from_words(u64(_pack(w))), d_out)
    torch.cuda.synchronize()
    got = to_np(d_out).view(np.uint64)
    # exact check on a slot sample (all rows and columns; Python integers)
    slots = sorted(set([0, 1, n // 2, n - 1] + list(rng.integers(0, n, size=12))))
    for b in range(B):
        for r in range(R):
            qr = q[r]
            for k in slots:
                xs = ct[:, :, b, :, r, k].astype(object)        # [img][cin][comp]
                ys = w[:, :, b, r, k].astype(object)            # [cout][cin]
                for img in range(images):
                    for comp in range(2):
                        acc = (xs[img, :, comp][None, :] * ys).sum(axis=1)
                        if comp == 1:
                            acc = acc + mask[img, :, b, r, k].astype(object)
                        exp = np.array([int(v) % qr for v in acc], dtype=np.uint64)
                        assert (got[img, :, b, comp, r, k] == exp).all(), (b, r, k, img, comp)


def test_bob_mac_four_product_fallback():
    """The 4-product kernel (fallback for primes outside the Karatsuba headroom) on the same
    edge shapes; selected in a fresh process by ENSEI_MAC_VARIANT=0 (read once per process)."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, ENSEI_MAC_VARIANT="0")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", os.path.join(here, "test_gpu_mac.py"),
                        "-k", "test_bob_mac_exact"], env=env, capture_output=True, text=True, timeout=900,
                       cwd=os.path.dirname(here))
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


I8_CASES = [c for c in CASES if c[2] <= 255] + [
    (2048, 8, 255, 16, 1),        # the int8 path's K limit (T < 2^128)
    (2048, 17, 33, 40, 1),        # one channel past a 32-channel chunk; partial row / col tiles
    (8192, 64, 64, 32, 3),        # config-4 shape class (three primes)
]
TC_CASES = [
    (8192, 64, 64, 128, 3),       # config 4's layer: one K chunk of 64, two 128-row tiles, 8 col tiles
    (2048, 64, 128, 128, 1),      # config 3's 128 -> 128: two K passes (the second adds the first's sums)
    (2048, 40, 33, 20, 1),        # partial row tile (80 rows), K = 33 (padded to 64), partial col tile
    (2048, 32, 255, 16, 1),       # the int8 K limit
    (4096, 48, 48, 40, 1),        # K = 48 in one 64-channel chunk, n = 4096
    # operand swap (out channels on the MMA's 128-row side, ciphertext rows in 16-row tiles):
    (8192, 13, 64, 128, 3),       # 26 rows: one full 16-row tile + a partial one, three primes
    (2048, 5, 40, 120, 1),        # cout = 120 (8 padded channels), 10 rows, K = 40
    (2048, 23, 130, 256, 1),      # two 128-channel blocks, three K passes, 46 rows
    (2048, 1, 32, 128, 1),        # a single ciphertext (2 rows)
]


@pytest.mark.parametrize("n,images,cin,cout,R", I8_CASES)
def test_bob_mac_int8_tensor_cores_exact(ops, n, images, cin, cout, R):
    """The int8 tensor-core ElementMult (mac_i8.cuh, variant 2) on the same exact checks."""
    from paper_2003_05328_b200._lib import check, lib
    check(lib().ensei_gpu_set_mac_variant(2))
    try:
        test_bob_mac_exact(ops, n, images, cin, cout, R)
    finally:
        check(lib().ensei_gpu_set_mac_variant(-1))


@pytest.mark.parametrize("n,images,cin,cout,R", TC_CASES + [c for c in I8_CASES if c[2] >= 32])
def test_bob_mac_tcgen05_exact(ops, n, images, cin, cout, R):
    """The tcgen05 ElementMult (mac_tc.cuh, variant 5: tcgen05.mma kind::i8, TMEM
    accumulators, weight planes built from the packed words) on the exact checks."""
    from paper_2003_05328_b200._lib import check, lib
    check(lib().ensei_gpu_set_mac_variant(5))
    try:
        q = (Q,) if R == 1 else RNS
        L = ops.LayerOps(ops.Context(n=n, q=q), ops.ConvSpec(16, 16, 3, 3, True, cin, cout))
        assert L.mac_path(images) == "tcgen05"
        test_bob_mac_exact(ops, n, images, cin, cout, R)
    finally:
        check(lib().ensei_gpu_set_mac_variant(-1))
