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


# ---------------------------------------------------------------- single prime, n = 2048

def _direct1(img, w, H, fh, cin, cout):
    Lo = O.layer(RNS[0], P, 2048, H, H, fh, fh, 1, cin, cout)
    out = np.zeros(cout * H * H, np.uint64)
    O.lib().eo_conv_direct(C.byref(Lo), img.astype(np.uint64).reshape(-1), w.astype(np.int64).reshape(-1), out)
    return out


@pytest.mark.parametrize("H,grid,pack,imgs,cin,cout", [(32, 39, 1, 2, 3, 2), (16, 24, 3, 7, 2, 3), (8, 12, 12, 14, 2, 2),
                                                       (8, 12, 5, 5, 1, 1)])
def test_single_prime_grid_layer_vs_oracle(H, grid, pack, imgs, cin, cout):
    """Config 3's layer shapes on the overridden grids (n = 2048, REF's single prime):
    ciphertexts, shares (with HomRec: a second layer fed Bob's share) vs the oracle with the
    same grid and pack; outputs vs the plaintext convolution."""
    from paper_2003_05328_b200 import ops
    n, q = 2048, RNS[0]
    ctx = ops.Context(n=n)
    g = torch.Generator().manual_seed(grid * 100 + pack)
    x = torch.randint(0, 256, (imgs, cin, H, H), dtype=torch.uint8, generator=g)
    prev = torch.randint(0, P, (imgs, cin, H, H), dtype=torch.int32, generator=g)
    w = torch.randint(-128, 128, (cout, cin, 3, 3), dtype=torch.int32, generator=g)
    L = ops.LayerOps(ctx, ops.ConvSpec(H, H, 3, 3, True, cin, cout, pack, grid))
    assert (L.geom.Lh, L.geom.blocks, L.geom.pack) == (grid, 1, pack)
    t, key = ops.secret_sample(ctx, 71)
    R = ops.Randomness(seed=71, image_base=2 * pack)
    we = L.prepare_weights(w.to(dev()))
    xd = x.to(dev())
    for bob_prev in (None, prev):
        ct = L.alice_encrypt(key, xd, R)
        ct_out, bob = L.bob_eval(ct.clone(), we, R, bob_prev=None if bob_prev is None else bob_prev.to(dev()),
                                 images=imgs)
        alice = L.alice_decrypt(key, ct_out, images=imgs)
        out = L.forward(key, we, xd, R, bob_prev=None if bob_prev is None else bob_prev.to(dev()))
        torch.cuda.synchronize()
        for i in range(imgs):
            xin = x[i].numpy().astype(np.int64) if bob_prev is None else (x[i].numpy().astype(np.int64) + bob_prev[i].numpy()) % P
            assert (to_np(out[i]).astype(np.uint64).reshape(-1) == _direct1(xin, w.numpy(), H, 3, cin, cout)).all(), i
        Lo = OP.set_grid(O.layer(q, P, n, H, H, 3, 3, 1, cin, cout), grid)
        Lo.pack = pack
        wr = OP.prepare_weights(Lo, w.numpy(), W)
        ctn, con = ct.clone(), ct_out.clone()
        ctx.permute(ctn)
        ctx.permute(con)
        for c in range(L.cts(imgs)):
            pr = OP.PhiloxRandomness(71, 2 + c, n, q, P)
            assert (to_np(t) == pr.secret()).all()
            te = OP.secret_eval(Lo, pr.secret())
            e, a = pr.enc(0, cin, 1)
            k = min(pack, imgs - c * pack)
            xin = np.zeros((pack, cin, H, H), np.uint64)
            xin[:k] = x[c * pack:c * pack + k].numpy()
            bp = None
            if bob_prev is not None:
                bp = np.zeros((pack, cin, H, H), np.uint64)
                bp[:k] = bob_prev[c * pack:c * pack + k].numpy()
            r_ = OP.run_layer(Lo, te, xin if pack > 1 else xin[0], bp if (bp is None or pack > 1) else bp[0], wr, e, a,
                              pr.share(0, cout, 1), ("ct",), W)
            if bob_prev is None:
                assert (to_np(ctn[c])[:, :, :, 0] == r_["ct_in"]).all(), c
            assert (to_np(con[c])[:, :, :, 0] == r_["ct_out"]).all(), c
            al, bo = np.asarray(r_["alice"]).reshape(pack, -1), np.asarray(r_["bob"]).reshape(pack, -1)
            for pi in range(k):
                assert (to_np(alice[c * pack + pi]).astype(np.uint64).reshape(-1) == al[pi]).all(), (c, pi)
                assert (to_np(bob[c * pack + pi]).astype(np.uint64).reshape(-1) == bo[pi]).all(), (c, pi)


def test_config3_grid_stack():
    """Config 3's seven layers on the overridden grids (39 / 24 / 12, packs 1 / 3 / 12; the
    1x1 layers on REF's 8x8 grid): every image's output equals the plaintext chain and the
    run in REF's geometry."""
    from paper_2003_05328_b200 import configs as CF
    from paper_2003_05328_b200 import ops
    from paper_2003_05328_b200 import protocol as GP
    imgs = 26
    ctx = ops.Context(n=2048)
    g = torch.Generator().manual_seed(3039)
    ws = [torch.randint(-128, 128, s, dtype=torch.int32, generator=g) for s in CF.CONFIG3_WEIGHTS]
    x = torch.randint(0, 256, (imgs, 3, 32, 32), dtype=torch.uint8, generator=g)
    _, key = ops.secret_sample(ctx, 35)
    outs = {}
    for name, sched in (("grid", CF.CONFIG3_SCHEDULE_GRID), ("ref", CF.CONFIG3_SCHEDULE)):
        sess = GP.Session(ctx, sched, 32, 32, ws)
        outs[name] = sess.run(key, x.to(dev()), lambda li: ops.Randomness(seed=35, layer=li))
        if name == "grid":
            assert [int(lo.geom.Lh) for lo in sess.layers if lo is not None] == [39, 39, 24, 24, 12, 8, 8]
            assert [lo.pack for lo in sess.layers if lo is not None] == [1, 1, 3, 3, 12, 32, 32]
    torch.cuda.synchronize()
    assert torch.equal(outs["grid"], outs["ref"])
    osched = [OP.Conv(s.fh, s.fw, s.same, s.cin, s.cout) if hasattr(s, "cin") else OP.Act(s.fn, s.pool2)
              for s in CF.CONFIG3_SCHEDULE]
    wnp = [w.numpy().astype(np.int64) for w in ws]
    for i in (0, 11, imgs - 1):
        want = OP.plain_protocol(osched, x[i].numpy().astype(np.int64), wnp, RNS[0], P, 2048, W)
        assert (to_np(outs["grid"][i]).astype(np.uint64) == want).all(), i


@pytest.mark.parametrize("H,fh,same,grid,pack", [(32, 5, True, 39, 1), (32, 7, True, 39, 1), (32, 3, False, 39, 1),
                                                 (16, 5, True, 24, 3), (16, 9, False, 24, 2), (8, 5, True, 12, 12),
                                                 (8, 3, False, 12, 7), (8, 1, True, 12, 3), (20, 3, True, 24, 2)])
def test_grid_override_filter_shapes(H, fh, same, grid, pack):
    """Overridden grids with other filter sizes and Valid convolutions (crop origin, output
    size) at n = 2048: every output equals the plaintext convolution and the run in REF's
    geometry."""
    from paper_2003_05328_b200 import ops
    cin, cout, imgs = 3, 4, 2 * pack + 1
    ctx = ops.Context(n=2048)
    g = torch.Generator().manual_seed(H * 100 + fh * 10 + pack)
    x = torch.randint(0, 256, (imgs, cin, H, H), dtype=torch.uint8, generator=g)
    w = torch.randint(-128, 128, (cout, cin, fh, fh), dtype=torch.int32, generator=g)
    _, key = ops.secret_sample(ctx, 5)
    outs = []
    for gr, pk in ((grid, pack), (0, 1)):
        L = ops.LayerOps(ctx, ops.ConvSpec(H, H, fh, fh, same, cin, cout, pk, gr))
        out = L.forward(key, L.prepare_weights(w.to(dev())), x.to(dev()), ops.Randomness(seed=5, image_base=pk * 3))
        torch.cuda.synchronize()
        outs.append(out)
    assert torch.equal(outs[0], outs[1])
    Lo = O.layer(RNS[0], P, 2048, H, H, fh, fh, int(same), cin, cout)
    for i in range(imgs):
        want = np.zeros(cout * Lo.oh * Lo.ow, np.uint64)
        O.lib().eo_conv_direct(C.byref(Lo), x[i].numpy().astype(np.uint64).reshape(-1),
                               w.numpy().astype(np.int64).reshape(-1), want)
        assert (to_np(outs[0][i]).astype(np.uint64).reshape(-1) == want).all(), i
