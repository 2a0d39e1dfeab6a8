"""GPU: the two generations of the 3-prime RNS tile kernels at n = 8192 (Enc / HomShare /
Dec; ensei_gpu_set_tile_variant: 1 = csrc/layer_rns.cuh, the default; 0 = csrc/layer.cuh)
produce identical ciphertexts, shares and outputs, stage by stage and fused, on 64x64 and
32x32 grids, packed and unpacked, ragged packs included; outputs equal the plaintext
convolution.  (Both generations are checked against the oracle elsewhere: the default one
by tests/test_gpu_configs.py, test_gpu_packing.py, test_gpu_layer.py; the exact-rounding
fallback of either by test_fallback_both_generations here.)"""
import ctypes as C

import numpy as np
import pytest
import torch

import oracle as O
from gpu_util import P, RNS, dev, to_np

pytestmark = pytest.mark.gpu


@pytest.fixture()
def tile_variant():
    from paper_2003_05328_b200._lib import check, lib

    def set_(v):
        check(lib().ensei_gpu_set_tile_variant(v))
    yield set_
    set_(1)


def _direct(img, w, H, cin, cout):
    Lo = O.layer(RNS[0], P, 2048, H, H, 3, 3, 1, cin, cout)
    out = np.zeros(cout * H * H, np.uint64)
    O.lib().eo_conv_direct(C.byref(Lo), img.astype(np.uint64).reshape(-1), w.astype(np.int64).reshape(-1), out)
    return out


@pytest.mark.parametrize("H,pack,imgs,cin,cout", [(32, 1, 3, 2, 3), (32, 2, 5, 3, 2), (16, 8, 11, 2, 2), (16, 1, 2, 1, 1)])
def test_generations_agree(tile_variant, H, pack, imgs, cin, cout):
    from paper_2003_05328_b200 import ops
    ctx = ops.Context(n=8192, q=RNS)
    g = torch.Generator().manual_seed(1000 + H + pack)
    x = torch.randint(0, 256, (imgs, cin, H, H), dtype=torch.uint8, generator=g)
    w = torch.randint(-128, 128, (cout, cin, 3, 3), dtype=torch.int32, generator=g)
    L = ops.LayerOps(ctx, ops.ConvSpec(H, H, 3, 3, True, cin, cout, pack))
    _, key = ops.secret_sample(ctx, 17)
    we = L.prepare_weights(w.to(dev()))
    R = ops.Randomness(seed=17, image_base=8 * pack)
    got = {}
    for v in (0, 1):
        tile_variant(v)
        ct = L.alice_encrypt(key, x.to(dev()), R)
        ct_out, bob = L.bob_eval(ct.clone(), we, R, images=imgs)
        alice = L.alice_decrypt(key, ct_out, images=imgs)
        out, fa, fb = L.forward(key, we, x.to(dev()), R, want_shares=True)
        torch.cuda.synchronize()
        got[v] = (ct, ct_out, bob, alice, out, fa, fb)
    for a, b in zip(got[0], got[1]):
        assert torch.equal(a, b)
    assert torch.equal(got[1][3], got[1][5]) and torch.equal(got[1][2], got[1][6])
    for i in range(imgs):
        assert (to_np(got[1][4][i]).astype(np.uint64).reshape(-1) == _direct(x[i].numpy(), w.numpy(), H, cin, cout)).all(), i


@pytest.mark.parametrize("pack,grid", [(1, 0), (2, 0), (5, 39)])
def test_homrec_rns_generations(tile_variant, pack, grid):
    """A second RNS layer (HomRec: Bob adds his previous share into the ciphertexts): the
    second-generation HomRec kernel against the first generation (REF's grids) and the
    plaintext convolution of the recombined input (every geometry)."""
    from paper_2003_05328_b200 import ops
    H, imgs, cin, cout = 32, 7, 3, 2
    ctx = ops.Context(n=8192, q=RNS)
    g = torch.Generator().manual_seed(77 + pack)
    x = torch.randint(0, P, (imgs, cin, H, H), dtype=torch.int32, generator=g)
    prev = torch.randint(0, P, (imgs, cin, H, H), dtype=torch.int32, generator=g)
    w = torch.randint(-128, 128, (cout, cin, 3, 3), dtype=torch.int32, generator=g)
    L = ops.LayerOps(ctx, ops.ConvSpec(H, H, 3, 3, True, cin, cout, pack, grid))
    _, key = ops.secret_sample(ctx, 19)
    we = L.prepare_weights(w.to(dev()))
    R = ops.Randomness(seed=19, image_base=4 * pack)
    got = {}
    for v in ((1,) if grid else (0, 1)):
        tile_variant(v)
        got[v] = L.forward(key, we, x.to(dev()), R, bob_prev=prev.to(dev()), want_shares=True)
        torch.cuda.synchronize()
    if not grid:
        for a, b in zip(got[0], got[1]):
            assert torch.equal(a, b)
    for i in range(imgs):
        xin = (x[i].numpy().astype(np.int64) + prev[i].numpy()) % P
        assert (to_np(got[1][0][i]).astype(np.uint64).reshape(-1) == _direct(xin, w.numpy(), H, cin, cout)).all(), i


@pytest.mark.parametrize("variant", [0, 1])
def test_fallback_both_generations(tile_variant, variant):
    """The in-kernel exact-rounding fallback of either generation (crafted ciphertext, 96
    coefficients next to a rounding boundary) against the oracle's exact decryption."""
    import test_gpu_params as T
    tile_variant(variant)
    T.test_rns_decrypt_exact_fallback_in_kernel()
