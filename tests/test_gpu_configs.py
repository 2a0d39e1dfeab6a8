"""GPU parity at BASELINE's full shapes (configs 3 and 4), through the C ABI.

config 4: 64 images (one full 128-row tile of the automatically selected tcgen05
ElementMult) of the real 64 -> 128 3x3 layer at n = 8192 with the 3-prime RNS
modulus: prepared weights, both wire directions' ciphertexts, both shares (the exact
multi-limb CRT decryption of the oracle) for two images, and every image's
reconstructed output against the plaintext convolution (REF conv_oracle semantics).

config 3: 32 images through the real seven-layer stack (3->64->64 @32, pool,
64->128->128 @16, pool, 128->128 3x3, 128->128 1x1, 128->16 1x1 @8): every image's
output against the plaintext chain (pinned to REF reference_pipeline segment by
segment in tests/test_config3_pin.py), and one image's per-layer Alice and Bob shares
against the oracle's full homomorphic restatement of the session."""
import numpy as np
import pytest
import torch

from oracle import protocol as OP
from gpu_util import P, Q, RNS, dev, to_np
from paper_2003_05328_b200 import configs as CF

pytestmark = pytest.mark.gpu
W = OP.default_workers()


@pytest.fixture(scope="module")
def ops():
    from paper_2003_05328_b200 import ops as _ops
    return _ops


def _oracle_sched(sched):
    return [OP.Conv(s.fh, s.fw, s.same, s.cin, s.cout) if hasattr(s, "cin") else OP.Act(s.fn, s.pool2) for s in sched]


def test_config4_full_layer(ops):
    n, imgs, cin, cout = 8192, 64, 64, 128
    ctx = ops.Context(n=n, q=RNS)
    g = torch.Generator().manual_seed(404)
    x = torch.randint(0, 256, (imgs, cin, 32, 32), dtype=torch.uint8, generator=g)
    w = torch.randint(-128, 128, (cout, cin, 3, 3), dtype=torch.int32, generator=g)
    L = ops.LayerOps(ctx, ops.ConvSpec(32, 32, 3, 3, True, cin, cout))
    path = L.mac_path(imgs)
    assert path == "tcgen05", path  # the tensor-core ElementMult is what runs
    t, key = ops.secret_sample(ctx, 41)
    R = ops.Randomness(seed=41, image_base=1000)
    we = L.prepare_weights(w.to(dev()))
    xd = x.to(dev())
    ct = L.alice_encrypt(key, xd, R)
    ct_out, bob = L.bob_eval(ct.clone(), we, R)
    alice = L.alice_decrypt(key, ct_out)
    fused, fa, fb = L.forward(key, we, xd, R, want_shares=True)
    torch.cuda.synchronize()
    assert torch.equal(fa, alice) and torch.equal(fb, bob)

    # reconstructed outputs of every image == plaintext convolution
    for i in range(imgs):
        want = OP.plain_protocol([OP.Conv(3, 3, True, cin, cout)], x[i].numpy().astype(np.int64), [w.numpy()],
                                 Q, P, 2048, W)
        assert (to_np(fused[i]).astype(np.uint64) == want).all(), i

    # prepared weights, ciphertexts and shares vs the oracle (two images)
    Ls = OP.rns_layers(list(RNS), P, n, 32, 32, 3, 3, 1, cin, cout)
    wr = [OP.prepare_weights(Lr, w.numpy(), W) for Lr in Ls]
    wd = ops.unpack_limbs(L.weight_words(we).clone())
    ctx.permute(wd)
    wd = to_np(wd)  # [cout][cin][B][R][n]
    for r in range(3):
        assert (wd[:, :, :, r] == wr[r]).all(), r
    ctx.permute(ct)
    ctx.permute(ct_out)
    ct_np, co_np = to_np(ct), to_np(ct_out)
    for i in (0, 45):
        pr = OP.PhiloxRandomnessRNS(41, 1000 + i, n, list(RNS), P)
        assert (to_np(t) == pr.secret()).all()
        te = [OP.secret_eval(Lr, pr.secret()) for Lr in Ls]
        e, a = pr.enc_rns(0, cin, Ls[0].blocks)
        r_ = OP.run_layer_rns(Ls, te, x[i].numpy().astype(np.uint64), wr, e, a, pr.share(0, cout, Ls[0].blocks), W)
        assert (ct_np[i] == r_["ct_in"]).all(), i
        assert (co_np[i] == r_["ct_out"]).all(), i
        assert (to_np(alice[i]).astype(np.uint64) == r_["alice"]).all(), i
        assert (to_np(bob[i]).astype(np.uint64) == r_["bob"]).all(), i


def test_config3_full_stack(ops):
    from paper_2003_05328_b200 import protocol as GP
    imgs = 32
    ctx = ops.Context(n=2048)
    g = torch.Generator().manual_seed(303)
    ws = [torch.randint(-128, 128, s, dtype=torch.int32, generator=g) for s in CF.CONFIG3_WEIGHTS]
    x = torch.randint(0, 256, (imgs, 3, 32, 32), dtype=torch.uint8, generator=g)
    sess = GP.Session(ctx, CF.CONFIG3_SCHEDULE, 32, 32, ws)
    # the 64- and 128-channel layers take the tensor-core ElementMult at this batch
    for lo in sess.layers:
        if lo is not None and lo.spec.cin >= 64:
            assert lo.mac_path(imgs) == "tcgen05", (lo.spec, lo.mac_path(imgs))
    _, key = ops.secret_sample(ctx, 33)
    out, trace = sess.run(key, x.to(dev()), lambda li: ops.Randomness(seed=33, layer=li), keep_trace=True)
    torch.cuda.synchronize()
    osched = _oracle_sched(CF.CONFIG3_SCHEDULE)
    wnp = [w.numpy().astype(np.int64) for w in ws]
    for i in range(imgs):
        want = OP.plain_protocol(osched, x[i].numpy().astype(np.int64), wnp, Q, P, 2048, W)
        assert (to_np(out[i]).astype(np.uint64) == want).all(), i

    # one image through the oracle's homomorphic restatement: every conv layer's shares
    i = 9
    w_evals = []
    h = 32
    for s in osched:
        if isinstance(s, OP.Conv):
            Lo = OP.layer(Q, P, 2048, h, h, s.fh, s.fw, int(s.same), s.cin, s.cout)
            w_evals.append(OP.prepare_weights(Lo, wnp[len(w_evals)], W))
            h = Lo.oh
        elif s.pool2:
            h //= 2
    want, otrace = OP.run_protocol(osched, x[i].numpy().astype(np.int64), wnp, OP.PhiloxRandomness(33, i, 2048, Q, P),
                                   Q, P, 2048, workers=W, w_evals=w_evals)
    assert len(otrace) == len(trace) == 7
    for li, (got, ref) in enumerate(zip(trace, otrace)):
        assert (to_np(got["alice"][i]).astype(np.uint64) == ref["alice"]).all(), li
        assert (to_np(got["bob"][i]).astype(np.uint64) == ref["bob"]).all(), li
    assert (to_np(out[i]).astype(np.uint64) == want).all()
