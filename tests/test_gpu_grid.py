"""GPU: grid override (ensei_conv_desc::grid, builder extension): config 4's layer shape on the
39 x 39 grid (p - 1 = 2^14 39; 32 + 3 - 1 = 34 <= 39) with five images per n = 8192 block.
Prepared weights, both wire directions' ciphertexts and both shares against the oracle's
restatement with the same grid (its transforms take REF's direct O(L^2) path for such
lengths, REF ntt.cpp:35-49); every image's output against the plaintext convolution; ragged
packs; the refusals."""
import ctypes as C

import numpy as np
import pytest
import torch

import oracle as O
from oracle import protocol as OP
from gpu_util import P, RNS, dev, to_np

pytestmark = pytest.mark.gpu
W = OP.default_workers()


def _direct(img, w, H, cin, cout):
    Lo = O.layer(RNS[0], P, 2048, H, H, 3, 3, 1, cin, cout)
    out = np.zeros(cout * H * H, np.uint64)
    O.lib().eo_conv_direct(C.byref(Lo), img.astype(np.uint64).reshape(-1), w.astype(np.int64).reshape(-1), out)
    return out


@pytest.mark.parametrize("imgs,cin,cout,pack", [(7, 3, 2, 5), (3, 2, 2, 2), (5, 1, 1, 1)])
def test_grid39_layer_vs_oracle(imgs, cin, cout, pack):
    from paper_2003_05328_b200 import ops
    n, H, grid = 8192, 32, 39
    ctx = ops.Context(n=n, q=RNS)
    g = torch.Generator().manual_seed(39 + imgs)
    x = torch.randint(0, 256, (imgs, cin, H, H), dtype=torch.uint8, generator=g)
    w = torch.randint(-128, 128, (cout, cin, 3, 3), dtype=torch.int32, generator=g)
    L = ops.LayerOps(ctx, ops.ConvSpec(H, H, 3, 3, True, cin, cout, pack, grid))
    assert (L.geom.Lh, L.geom.Lw, L.geom.blocks, L.geom.pack) == (39, 39, 1, pack)
    t, key = ops.secret_sample(ctx, 61)
    R = ops.Randomness(seed=61, image_base=3 * pack)
    we = L.prepare_weights(w.to(dev()))
    xd = x.to(dev())
    ct = L.alice_encrypt(key, xd, R)
    ct_out, bob = L.bob_eval(ct.clone(), we, R, images=imgs)
    alice = L.alice_decrypt(key, ct_out, images=imgs)
    out, fa, fb = L.forward(key, we, xd, R, want_shares=True)
    torch.cuda.synchronize()
    assert torch.equal(fa, alice) and torch.equal(fb, bob)
    for i in range(imgs):
        assert (to_np(out[i]).astype(np.uint64).reshape(-1) == _direct(x[i].numpy(), w.numpy(), H, cin, cout)).all(), i

    Ls = OP.rns_layers(list(RNS), P, n, H, H, 3, 3, 1, cin, cout, pack, grid)
    wr = [OP.prepare_weights(Lr, w.numpy(), W) for Lr in Ls]
    wd = ops.unpack_limbs(L.weight_words(we).clone())
    ctx.permute(wd)
    wd = to_np(wd)
    for r in range(3):
        assert (wd[:, :, :, r] == wr[r]).all(), r
    ctx.permute(ct)
    ctx.permute(ct_out)
    for c in range(L.cts(imgs)):  # every ciphertext image, the ragged last one included
        pr = OP.PhiloxRandomnessRNS(61, 3 + c, n, list(RNS), P)
        assert (to_np(t) == pr.secret()).all()
        te = [OP.secret_eval(Lr, pr.secret()) for Lr in Ls]
        e, a = pr.enc_rns(0, cin, 1)
        xin = np.zeros((pack, cin, H, H), np.uint64)
        k = min(pack, imgs - c * pack)
        xin[:k] = x[c * pack:c * pack + k].numpy()
        r_ = OP.run_layer_rns(Ls, te, xin if pack > 1 else xin[0], wr, e, a, pr.share(0, cout, 1), W)
        assert (to_np(ct[c]) == r_["ct_in"]).all(), c
        assert (to_np(ct_out[c]) == r_["ct_out"]).all(), c
        al = np.asarray(r_["alice"]).reshape(pack, -1) if pack > 1 else np.asarray(r_["alice"]).reshape(1, -1)
        bo = np.asarray(r_["bob"]).reshape(pack, -1) if pack > 1 else np.asarray(r_["bob"]).reshape(1, -1)
        for pi in range(k):
            assert (to_np(alice[c * pack + pi]).astype(np.uint64).reshape(-1) == al[pi]).all(), (c, pi)
            assert (to_np(bob[c * pack + pi]).astype(np.uint64).reshape(-1) == bo[pi]).all(), (c, pi)


def test_grid_override_refusals():
    from paper_2003_05328_b200 import ops
    from paper_2003_05328_b200._lib import EnseiError
    ctx = ops.Context(n=8192, q=RNS)
    with pytest.raises(EnseiError, match="BadGeometry"):
        ops.LayerOps(ctx, ops.ConvSpec(32, 32, 3, 3, True, 1, 1, 1, 33))  # 33 does not divide p - 1
    with pytest.raises(EnseiError, match="BadGeometry"):
        ops.LayerOps(ctx, ops.ConvSpec(32, 32, 9, 9, True, 1, 1, 1, 39))  # 40 > 39
    with pytest.raises(EnseiError, match="BadGeometry"):
        ops.LayerOps(ctx, ops.ConvSpec(32, 32, 3, 3, True, 1, 1, 6, 39))  # 6 x 1521 > 8192
    # a single-prime context has no grid-override kernels
    ctx1 = ops.Context(n=8192, q=(RNS[0],))
    L = ops.LayerOps(ctx1, ops.ConvSpec(32, 32, 3, 3, True, 1, 1, 1, 39))
    w = torch.zeros((1, 1, 3, 3), dtype=torch.int32, device=dev())
    with pytest.raises(EnseiError, match="Unsupported"):
        L.prepare_weights(w)


def test_config4_grid_full_shape():
    """Config 4's real layer (64 -> 128, tcgen05 ElementMult) on the 39x39 grid with five
    images per block: 163 images = 33 ciphertext images, the last one ragged (3 images).
    Sampled outputs against the plaintext convolution; ciphertexts of both wire directions
    and both shares of one full and of the ragged ciphertext image against the oracle."""
    from paper_2003_05328_b200 import configs as CF
    from paper_2003_05328_b200 import ops
    n, H, cin, cout = 8192, 32, 64, 128
    pack, grid, imgs = CF.CONFIG4_GRID_PACK, CF.CONFIG4_GRID, 163
    ctx = ops.Context(n=n, q=RNS)
    g = torch.Generator().manual_seed(4039)
    x = torch.randint(0, 256, (imgs, cin, H, H), dtype=torch.uint8, generator=g)
    w = torch.randint(-128, 128, (cout, cin, 3, 3), dtype=torch.int32, generator=g)
    L = ops.LayerOps(ctx, ops.ConvSpec(H, H, 3, 3, True, cin, cout, pack, grid))
    assert L.mac_path(imgs) == "tcgen05"
    _, key = ops.secret_sample(ctx, 43)
    R = ops.Randomness(seed=43, image_base=10 * pack)
    we = L.prepare_weights(w.to(dev()))
    xd = x.to(dev())
    ct = L.alice_encrypt(key, xd, R)
    ct_out, bob = L.bob_eval(ct.clone(), we, R, images=imgs)
    alice = L.alice_decrypt(key, ct_out, images=imgs)
    out, fa, fb = L.forward(key, we, xd, R, want_shares=True)
    torch.cuda.synchronize()
    assert torch.equal(fa, alice) and torch.equal(fb, bob)
    for i in list(range(0, imgs, 13)) + [imgs - 1]:
        assert (to_np(out[i]).astype(np.uint64).reshape(-1) == _direct(x[i].numpy(), w.numpy(), H, cin, cout)).all(), i
    Ls = OP.rns_layers(list(RNS), P, n, H, H, 3, 3, 1, cin, cout, pack, grid)
    wr = [OP.prepare_weights(Lr, w.numpy(), W) for Lr in Ls]
    ctx.permute(ct)
    ctx.permute(ct_out)
    for c in (7, L.cts(imgs) - 1):
        pr = OP.PhiloxRandomnessRNS(43, 10 + c, n, list(RNS), P)
        te = [OP.secret_eval(Lr, pr.secret()) for Lr in Ls]
        e, a = pr.enc_rns(0, cin, 1)
        xin = np.zeros((pack, cin, H, H), np.uint64)
        k = min(pack, imgs - c * pack)
        xin[:k] = x[c * pack:c * pack + k].numpy()
        r_ = OP.run_layer_rns(Ls, te, xin, wr, e, a, pr.share(0, cout, 1), W)
        assert (to_np(ct[c]) == r_["ct_in"]).all(), c
        assert (to_np(ct_out[c]) == r_["ct_out"]).all(), c
        al, bo = np.asarray(r_["alice"]).reshape(pack, -1), np.asarray(r_["bob"]).reshape(pack, -1)
        for pi in range(k):
            assert (to_np(alice[c * pack + pi]).astype(np.uint64).reshape(-1) == al[pi]).all(), (c, pi)
            assert (to_np(bob[c * pack + pi]).astype(np.uint64).reshape(-1) == bo[pi]).all(), (c, pi)
