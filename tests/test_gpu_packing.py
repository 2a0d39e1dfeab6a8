"""GPU parity of ciphertext packing (ensei_conv_desc::pack, builder extension): several
images' grids in one ciphertext block.  Ciphertexts and both shares vs the oracle's
packed restatement (oracle/ensei_oracle.c, eo_layer::pack), outputs vs the plaintext
convolution (REF conv_oracle semantics -- packing changes no slot-wise step, so the
outputs are REF's), on single- and three-prime rings, partial last packs, HomRec, the
tcgen05 ElementMult, and config 3's stack with every layer packed."""
import numpy as np
import pytest
import torch

import oracle as O
from oracle import protocol as OP
from gpu_util import P, Q, RNS, dev, to_np
from paper_2003_05328_b200 import configs as CF

pytestmark = pytest.mark.gpu
W = OP.default_workers()


@pytest.fixture(scope="module")
def ops():
    from paper_2003_05328_b200 import ops as _ops
    return _ops


def _plain(img, w, H, fh=3, same=True):
    return OP.plain_protocol([OP.Conv(fh, fh, same, img.shape[0], w.shape[0])], img.astype(np.int64),
                             [w.astype(np.int64)], Q, P, 2048, W)


@pytest.mark.parametrize("n,H,fh,pack,imgs,cin,cout", [
    (2048, 16, 3, 2, 5, 4, 3),    # 32x32 grid: two per block; odd image count (partial last pack)
    (2048, 8, 3, 8, 11, 3, 2),    # 16x16 grid: eight per block
    (2048, 8, 1, 32, 33, 2, 2),   # 8x8 grid (1x1 filter): thirty-two per block
    (4096, 16, 3, 4, 4, 2, 3),    # n = 4096
])
def test_packed_layer_vs_oracle(ops, n, H, fh, pack, imgs, cin, cout):
    ctx = ops.Context(n=n)
    g = torch.Generator().manual_seed(n + pack + imgs)
    x = torch.randint(0, 256, (imgs, cin, H, H), dtype=torch.uint8, generator=g)
    w = torch.randint(-128, 128, (cout, cin, fh, fh), dtype=torch.int32, generator=g)
    L = ops.LayerOps(ctx, ops.ConvSpec(H, H, fh, fh, True, cin, cout, pack))
    assert L.pack == pack and L.cts(imgs) == -(-imgs // pack)
    t, key = ops.secret_sample(ctx, 8)
    R = ops.Randomness(seed=8, image_base=2 * pack)  # pack-aligned
    we = L.prepare_weights(w.to(dev()))
    xd = x.to(dev())
    ct = L.alice_encrypt(key, xd, R)
    ct_out, bob = L.bob_eval(ct.clone(), we, R, images=imgs)
    alice = L.alice_decrypt(key, ct_out, images=imgs)
    out = L.forward(key, we, xd, R)
    torch.cuda.synchronize()
    for i in range(imgs):
        assert (to_np(out[i]).astype(np.uint64) == _plain(x[i].numpy(), w.numpy(), H, fh)).all(), i
    Lo = O.layer(Q, P, n, H, H, fh, fh, 1, cin, cout)
    Lo.pack = pack
    te = OP.secret_eval(Lo, to_np(t))
    wo = OP.prepare_weights(Lo, w.numpy())
    ctx.permute(ct)
    ctx.permute(ct_out)
    for k in range(L.cts(imgs)):
        group = np.zeros((pack, cin, H, H), np.uint64)
        nk = min(pack, imgs - k * pack)
        group[:nk] = x[k * pack:k * pack + nk].numpy()
        pr = OP.PhiloxRandomness(8, 2 + k, n, Q, P)  # stream id = image_base / pack + k
        r = OP.run_layer(Lo, te, group, None, wo, *pr.enc(0, cin, 1), pr.share(0, cout, 1), want=("ct",))
        assert (to_np(ct[k]).reshape(cin, 1, 2, n) == r["ct_in"]).all(), k
        assert (to_np(ct_out[k]).reshape(cout, 1, 2, n) == r["ct_out"]).all(), k
        for pi in range(nk):
            assert (to_np(alice[k * pack + pi]).astype(np.uint64) == r["alice"][pi]).all(), (k, pi)
            assert (to_np(bob[k * pack + pi]).astype(np.uint64) == r["bob"][pi]).all(), (k, pi)


def test_packed_homrec_layer(ops):
    """Layer 2 of a session on a packed ring: HomRec with Bob's previous share."""
    ctx = ops.Context(n=2048)
    g = torch.Generator().manual_seed(12)
    imgs, cin, cout, H = 4, 3, 2, 16
    prev = torch.randint(0, P, (imgs, cin, H, H), dtype=torch.int32, generator=g)
    x = torch.randint(0, P, (imgs, cin, H, H), dtype=torch.int32, generator=g)
    w = torch.randint(-128, 128, (cout, cin, 3, 3), dtype=torch.int32, generator=g)
    L = ops.LayerOps(ctx, ops.ConvSpec(H, H, 3, 3, True, cin, cout, 2))
    _, key = ops.secret_sample(ctx, 5)
    we = L.prepare_weights(w.to(dev()))
    out = L.forward(key, we, x.to(dev()), ops.Randomness(seed=5), bob_prev=prev.to(dev()))
    for i in range(imgs):  # HomRec: the layer sees alice + bob_prev
        want = _plain(((x[i].numpy().astype(np.int64) + prev[i].numpy()) % P), w.numpy(), H)
        assert (to_np(out[i]).astype(np.uint64) == want).all(), i


def test_config4_packed_layer(ops):
    """Config 4's layer with two images per n = 8192 block: 64 images = 32 ciphertext
    images (the tcgen05 ElementMult's 64 rows), outputs vs the plaintext convolution,
    ciphertexts and shares of one pack vs the oracle's exact RNS restatement."""
    n, imgs, cin, cout, pack = 8192, 64, 64, 128, CF.CONFIG4_PACK
    ctx = ops.Context(n=n, q=RNS)
    g = torch.Generator().manual_seed(4040)
    x = torch.randint(0, 256, (imgs, cin, 32, 32), dtype=torch.uint8, generator=g)
    w = torch.randint(-128, 128, (cout, cin, 3, 3), dtype=torch.int32, generator=g)
    L = ops.LayerOps(ctx, ops.ConvSpec(32, 32, 3, 3, True, cin, cout, pack))
    assert L.mac_path(imgs) == "tcgen05"
    t, key = ops.secret_sample(ctx, 42)
    R = ops.Randomness(seed=42)
    we = L.prepare_weights(w.to(dev()))
    xd = x.to(dev())
    ct = L.alice_encrypt(key, xd, R)
    ct_out, bob = L.bob_eval(ct.clone(), we, R, images=imgs)
    alice = L.alice_decrypt(key, ct_out, images=imgs)
    out = L.forward(key, we, xd, R)
    torch.cuda.synchronize()
    for i in range(0, imgs, 7):
        assert (to_np(out[i]).astype(np.uint64) == _plain(x[i].numpy(), w.numpy(), 32)).all(), i
    Ls = OP.rns_layers(list(RNS), P, n, 32, 32, 3, 3, 1, cin, cout, pack)
    wr = [OP.prepare_weights(Lr, w.numpy(), W) for Lr in Ls]
    pr = OP.PhiloxRandomnessRNS(42, 5, n, list(RNS), P)
    te = [OP.secret_eval(Lr, pr.secret()) for Lr in Ls]
    e, a = pr.enc_rns(0, cin, 1)
    r = OP.run_layer_rns(Ls, te, x[10:12].numpy().astype(np.uint64), wr, e, a, pr.share(0, cout, 1), W)
    ctx.permute(ct)
    ctx.permute(ct_out)
    assert (to_np(ct[5]) == r["ct_in"]).all()
    assert (to_np(ct_out[5]) == r["ct_out"]).all()
    for pi in range(2):
        assert (to_np(alice[10 + pi]).astype(np.uint64) == r["alice"][pi]).all(), pi
        assert (to_np(bob[10 + pi]).astype(np.uint64) == r["bob"][pi]).all(), pi


def test_config3_packed_stack(ops):
    """Config 3's seven layers with every layer packed as far as the ring allows
    (packs 1, 1, 2, 2, 8, 32, 32): outputs equal the plaintext chain and the unpacked run."""
    from paper_2003_05328_b200 import protocol as GP
    imgs = 40
    ctx = ops.Context(n=2048)
    g = torch.Generator().manual_seed(333)
    ws = [torch.randint(-128, 128, s, dtype=torch.int32, generator=g) for s in CF.CONFIG3_WEIGHTS]
    x = torch.randint(0, 256, (imgs, 3, 32, 32), dtype=torch.uint8, generator=g)
    sess = GP.Session(ctx, CF.CONFIG3_SCHEDULE_PACKED, 32, 32, ws)
    assert [lo.pack for lo in sess.layers if lo is not None] == [1, 1, 2, 2, 8, 32, 32]
    _, key = ops.secret_sample(ctx, 3)
    out = sess.run(key, x.to(dev()), lambda li: ops.Randomness(seed=3, layer=li))
    ref = GP.Session(ctx, CF.CONFIG3_SCHEDULE, 32, 32, ws).run(key, x.to(dev()),
                                                                lambda li: ops.Randomness(seed=3, layer=li))
    osched = [OP.Conv(s.fh, s.fw, s.same, s.cin, s.cout) if hasattr(s, "cin") else OP.Act(s.fn, s.pool2)
              for s in CF.CONFIG3_SCHEDULE]
    bad_p, bad_u = [], []
    for i in range(imgs):
        want = OP.plain_protocol(osched, x[i].numpy().astype(np.int64), [w.numpy().astype(np.int64) for w in ws],
                                 Q, P, 2048, W)
        if not (to_np(out[i]).astype(np.uint64) == want).all():
            bad_p.append(i)
        if not (to_np(ref[i]).astype(np.uint64) == want).all():
            bad_u.append(i)
    assert not bad_p and not bad_u, (bad_p, bad_u)
    assert torch.equal(out, ref)
