"""GPU parity for the fused conv-layer path (through the C ABI):

* parity mode -- the reference's own randomness injected: ciphertexts on both
  wire directions, both shares and outputs equal the reference's (golden FNV
  digests from the compiled reference, tests/golden/golden.json);
* throughput mode -- Philox streams: shares equal the oracle restatement, outputs
  equal the plaintext convolution (REF conv_oracle / reference_pipeline)."""
import ctypes as C

import numpy as np
import pytest
import torch

import oracle as O
from oracle import protocol as OP
from conftest import fnv
from gpu_util import P, Q, dev, golden_inputs, to_np, u64

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ops():
    from paper_2003_05328_b200 import ops as _ops
    return _ops


def _inject(ops, rand, li, cin, cout, B, n):
    e, a = rand.enc(li, cin, B)
    s = rand.share(li, cout, B)
    return ops.Randomness(layer=li, noise=torch.from_numpy(e.astype(np.int32)).to(dev()).reshape(1, cin, B, n),
                          a_hat=u64(a).reshape(1, cin, B, 1, n),
                          share=torch.from_numpy(s.astype(np.int32)).to(dev()).reshape(1, cout, B, n)), (e, a, s)


@pytest.mark.parametrize("idx", [0, 1, 3, 4])
def test_single_layer_golden_parity(ops, golden, idx):
    case = golden["proto"][idx]
    img, ws, sched = golden_inputs(case)
    conv = sched[0]
    n = case["n"]
    ctx = ops.Context(n=n)
    H, W = case["H"], case["W"]
    L = ops.LayerOps(ctx, ops.ConvSpec(H, W, conv.fh, conv.fw, conv.same, conv.cin, conv.cout))
    rand = OP.RefRandomness(case["seed"], n, Q, P)
    key = ops.secret_from_coeffs(ctx, torch.from_numpy(rand.secret()).to(dev()))
    w_eval = L.prepare_weights(torch.from_numpy(ws[0].astype(np.int32)).to(dev()))
    R, _ = _inject(ops, rand, 0, conv.cin, conv.cout, L.B, n)
    x = torch.from_numpy(img.astype(np.int32)[None]).to(dev())
    ct = L.alice_encrypt(key, x, R)
    ct_out, bob = L.bob_eval(ct.clone(), w_eval, R)
    alice = L.alice_decrypt(key, ct_out)
    out = (to_np(alice).astype(np.uint64) + to_np(bob).astype(np.uint64)) % P
    assert fnv(out.reshape(-1)) == case["out_fnv"]
    if case["mode"] == 1:  # FreqDirect wire ciphertexts (Baseline differs only in ciphertext domain)
        ctx.permute(ct)
        ctx.permute(ct_out)
        assert fnv(to_np(ct).reshape(-1)) == case["ct_a2b_fnv"]
        assert fnv(to_np(ct_out).reshape(-1)) == case["ct_b2a_fnv"]
    fused = L.forward(key, w_eval, x, R)
    assert fnv(to_np(fused).astype(np.uint64).reshape(-1)) == case["out_fnv"]


def test_multilayer_golden_parity_homrec(ops, golden):
    """conv -> ReLU -> conv with HomRec on Bob's share: the reference's session."""
    from paper_2003_05328_b200 import protocol as GP
    case = golden["proto"][2]
    img, ws, sched = golden_inputs(case)
    n = case["n"]
    ctx = ops.Context(n=n)
    gsched = [GP.Conv(s.fh, s.fw, s.same, s.cin, s.cout) if isinstance(s, OP.Conv) else GP.Act(s.fn) for s in sched]
    sess = GP.Session(ctx, gsched, case["H"], case["W"], [torch.from_numpy(w.astype(np.int32)) for w in ws])
    rand = OP.RefRandomness(case["seed"], n, Q, P)
    key = ops.secret_from_coeffs(ctx, torch.from_numpy(rand.secret()).to(dev()))
    cache = {}

    def rnd(li):
        s = sched[li]
        if isinstance(s, OP.Conv):
            return _inject(ops, rand, li, s.cin, s.cout, sess.layers[li].B, n)[0]
        lo = sess.layers[li - 1]
        fresh = rand.reshare(li, s_cout(li), lo.geom.oh * lo.geom.ow)
        return ops.Randomness(layer=li, share=torch.from_numpy(fresh.astype(np.int32)).to(dev()).reshape(-1))

    def s_cout(li):
        return sched[li - 1].cout

    x = torch.from_numpy(img.astype(np.int32)[None]).to(dev())
    out = sess.run(key, x, rnd)
    assert fnv(to_np(out).astype(np.uint64).reshape(-1)) == case["out_fnv"]


def _direct(img, w, H, same=True, fh=3):
    L = O.layer(Q, P, 2048, H, H, fh, fh, int(same), img.shape[0], w.shape[0])
    out = np.zeros(L.cout * L.oh * L.ow, np.uint64)
    O.lib().eo_conv_direct(C.byref(L), (img.astype(np.uint64) % P).reshape(-1), w.astype(np.int64).reshape(-1), out)
    return out.reshape(L.cout, L.oh, L.ow)


def test_config1_philox_vs_oracle_and_direct(ops):
    """BASELINE config 1: 8 images x 16->16 @ 32x32, n=2048."""
    ctx = ops.Context(n=2048)
    g = torch.Generator().manual_seed(5)
    imgs = torch.randint(0, 256, (8, 16, 32, 32), dtype=torch.uint8, generator=g)
    w = torch.randint(-128, 128, (16, 16, 3, 3), dtype=torch.int32, generator=g)
    L = ops.LayerOps(ctx, ops.ConvSpec(32, 32, 3, 3, True, 16, 16))
    t, key = ops.secret_sample(ctx, 11)
    w_eval = L.prepare_weights(w.to(dev()))
    out, alice, bob = L.forward(key, w_eval, imgs.to(dev()), ops.Randomness(seed=11), want_shares=True)
    for i in range(8):
        assert (to_np(out[i]).astype(np.uint64) == _direct(imgs[i].numpy(), w.numpy(), 32)).all()
    prand = OP.PhiloxRandomness(11, 5, 2048, Q, P)
    assert (to_np(t) == prand.secret()).all()
    Lo = O.layer(Q, P, 2048, 32, 32, 3, 3, 1, 16, 16)
    r = OP.run_layer(Lo, OP.secret_eval(Lo, prand.secret()), imgs[5].numpy().astype(np.uint64), None,
                     OP.prepare_weights(Lo, w.numpy()), *prand.enc(0, 16, 2), prand.share(0, 16, 2))
    assert (to_np(alice[5]).astype(np.uint64) == r["alice"]).all()
    assert (to_np(bob[5]).astype(np.uint64) == r["bob"]).all()


def test_sharding_invariance(ops):
    """Splitting a batch with image_base offsets gives the same shares as one batch."""
    ctx = ops.Context(n=2048)
    g = torch.Generator().manual_seed(6)
    imgs = torch.randint(0, 256, (4, 2, 8, 8), dtype=torch.uint8, generator=g).to(dev())
    w = torch.randint(-128, 128, (3, 2, 3, 3), dtype=torch.int32, generator=g).to(dev())
    L = ops.LayerOps(ctx, ops.ConvSpec(8, 8, 3, 3, True, 2, 3))
    _, key = ops.secret_sample(ctx, 3)
    we = L.prepare_weights(w)
    _, a_all, b_all = L.forward(key, we, imgs, ops.Randomness(seed=3), want_shares=True)
    _, a_hi, b_hi = L.forward(key, we, imgs[2:].contiguous(), ops.Randomness(seed=3, image_base=2), want_shares=True)
    assert torch.equal(a_all[2:], a_hi) and torch.equal(b_all[2:], b_hi)


def test_ragged_shards_through_shard_module(ops):
    """The product's ImageShard splits 5 images over 2 and 3 'ranks' (ragged); each shard
    run with image_base = shard.start and gathered (world-size-1 path per shard) equals
    the single batch: outputs and both parties' shares."""
    from paper_2003_05328_b200.shard import ImageShard
    ctx = ops.Context(n=2048)
    g = torch.Generator().manual_seed(11)
    imgs = torch.randint(0, 256, (5, 2, 8, 8), dtype=torch.uint8, generator=g).to(dev())
    w = torch.randint(-128, 128, (3, 2, 3, 3), dtype=torch.int32, generator=g).to(dev())
    L = ops.LayerOps(ctx, ops.ConvSpec(8, 8, 3, 3, True, 2, 3))
    _, key = ops.secret_sample(ctx, 4)
    we = L.prepare_weights(w)
    out_all, a_all, b_all = L.forward(key, we, imgs, ops.Randomness(seed=4), want_shares=True)
    for world in (2, 3):
        outs, al, bo = [], [], []
        for rank in range(world):
            sh = ImageShard(5, world, rank)
            o, a_, b_ = L.forward(key, we, sh.take(imgs).contiguous(), ops.Randomness(seed=4, image_base=sh.start),
                                  want_shares=True)
            outs.append(o)
            al.append(a_)
            bo.append(b_)
        assert torch.equal(torch.cat(outs), out_all), world
        assert torch.equal(torch.cat(al), a_all) and torch.equal(torch.cat(bo), b_all), world


@pytest.mark.parametrize("n,H,fh,same,cin,cout", [
    (2048, 8, 3, True, 3, 5),     # L = 16, one half-empty block
    (2048, 8, 1, True, 4, 4),     # 1x1 filter, L = 8
    (2048, 12, 5, False, 2, 3),   # Valid, L = 16
    (4096, 16, 3, True, 2, 2),    # n = 4096, L = 32
    (8192, 32, 3, True, 2, 3),    # n = 8192, L = 64, one block
    (2048, 16, 3, True, 40, 36),  # > 16 rows/cols: the large MAC tile, 40-channel accumulation
])
def test_layer_shapes_philox(ops, n, H, fh, same, cin, cout):
    ctx = ops.Context(n=n)
    g = torch.Generator().manual_seed(n + H + cin)
    imgs = torch.randint(0, 256, (3, cin, H, H), dtype=torch.uint8, generator=g)
    w = torch.randint(-128, 128, (cout, cin, fh, fh), dtype=torch.int32, generator=g)
    L = ops.LayerOps(ctx, ops.ConvSpec(H, H, fh, fh, same, cin, cout))
    _, key = ops.secret_sample(ctx, 1)
    out = L.forward(key, L.prepare_weights(w.to(dev())), imgs.to(dev()), ops.Randomness(seed=1))
    for i in range(3):
        assert (to_np(out[i]).astype(np.uint64) == _direct(imgs[i].numpy(), w.numpy(), H, same, fh)).all()


def test_host_buffer_entry_equals_device_path(ops):
    ctx = ops.Context(n=2048)
    g = torch.Generator().manual_seed(9)
    imgs = torch.randint(0, 256, (2, 4, 16, 16), dtype=torch.uint8, generator=g)
    w = torch.randint(-128, 128, (4, 4, 3, 3), dtype=torch.int32, generator=g)
    L = ops.LayerOps(ctx, ops.ConvSpec(16, 16, 3, 3, True, 4, 4))
    _, key = ops.secret_sample(ctx, 2)
    we = L.prepare_weights(w.to(dev()))
    d = L.forward(key, we, imgs.to(dev()), ops.Randomness(seed=2))
    h_out = torch.empty((2, 4, 16, 16), dtype=torch.int32).pin_memory()
    h_in, ws = imgs.pin_memory(), L.workspace(2, host=True)
    L.forward_host(key, we, h_in, ops.Randomness(seed=2), ws, h_out)
    assert torch.equal(h_out, d.cpu())
    # same arguments: the cached CUDA graph replays and reads the host buffer's new contents
    imgs2 = torch.randint(0, 256, (2, 4, 16, 16), dtype=torch.uint8, generator=g)
    h_in.copy_(imgs2)
    L.forward_host(key, we, h_in, ops.Randomness(seed=2), ws, h_out)
    assert torch.equal(h_out, L.forward(key, we, imgs2.to(dev()), ops.Randomness(seed=2)).cpu())
    # changed randomness -> re-captured graph; pageable buffers -> uncaptured fallback
    L.forward_host(key, we, h_in, ops.Randomness(seed=3), ws, h_out)
    assert torch.equal(h_out, L.forward(key, we, imgs2.to(dev()), ops.Randomness(seed=3)).cpu())
    out_pageable = torch.empty((2, 4, 16, 16), dtype=torch.int32)
    L.forward_host(key, we, imgs2.clone(), ops.Randomness(seed=3), ws, out_pageable)
    assert torch.equal(out_pageable, h_out)
    # prepared call (the bench's e2e form): same results, re-reads the input buffer each call
    call = L.host_call(key, we, h_in, ops.Randomness(seed=2), ws, h_out)
    h_in.copy_(imgs)
    assert torch.equal(call(), d.cpu())
    h_in.copy_(imgs2)
    assert torch.equal(call(), L.forward(key, we, imgs2.to(dev()), ops.Randomness(seed=2)).cpu())


def test_pooled_relu_stack_vs_oracle(ops):
    """A miniature config-3 segment chain: conv -> ReLU+pool -> conv -> ReLU -> conv."""
    from paper_2003_05328_b200 import protocol as GP
    ctx = ops.Context(n=2048)
    rng = np.random.default_rng(4)
    img = rng.integers(0, 256, size=(3, 16, 16)).astype(np.int64)
    ws = [rng.integers(-8, 8, size=s).astype(np.int64) for s in ((4, 3, 3, 3), (4, 4, 3, 3), (2, 4, 1, 1))]
    osched = [OP.Conv(3, 3, True, 3, 4), OP.Act(0, True), OP.Conv(3, 3, True, 4, 4), OP.Act(0), OP.Conv(1, 1, True, 4, 2)]
    gsched = [GP.Conv(3, 3, True, 3, 4), GP.Act(0, True), GP.Conv(3, 3, True, 4, 4), GP.Act(0), GP.Conv(1, 1, True, 4, 2)]
    want, _ = OP.run_protocol(osched, img, ws, OP.PhiloxRandomness(21, 0, 2048, Q, P), Q, P, 2048)
    sess = GP.Session(ctx, gsched, 16, 16, [torch.from_numpy(w.astype(np.int32)) for w in ws])
    _, key = ops.secret_sample(ctx, 21)
    got = sess.run(key, torch.from_numpy(img.astype(np.uint8)[None]).to(dev()), lambda li: ops.Randomness(seed=21, layer=li))
    assert (to_np(got[0]).astype(np.uint64) == want).all()


def test_geometry_errors(ops):
    from paper_2003_05328_b200 import EnseiError
    ctx = ops.Context(n=2048)
    with pytest.raises(EnseiError, match="BadGeometry"):
        ops.LayerOps(ctx, ops.ConvSpec(2, 2, 3, 3, False, 1, 1))
    with pytest.raises(EnseiError, match="Unsupported"):
        ops.LayerOps(ctx, ops.ConvSpec(64, 64, 3, 3, True, 1, 1))  # 128x128 grid


def test_rns_config4_shape_vs_oracle(ops):
    """Config 4 arithmetic: n = 8192, three 60-bit primes (RNS), 64x64 grid (B = 1):
    ciphertexts per prime, both shares (CRT decryption) vs the oracle's exact CRT."""
    from gpu_util import RNS
    n = 8192
    ctx = ops.Context(n=n, q=RNS)
    rng = np.random.default_rng(44)
    img = rng.integers(0, 256, size=(2, 32, 32)).astype(np.int64)
    w = rng.integers(-128, 128, size=(3, 2, 3, 3)).astype(np.int64)
    L = ops.LayerOps(ctx, ops.ConvSpec(32, 32, 3, 3, True, 2, 3))
    t, key = ops.secret_sample(ctx, 5)
    R = ops.Randomness(seed=5)
    we = L.prepare_weights(torch.from_numpy(w.astype(np.int32)).to(dev()))
    x = torch.from_numpy(img.astype(np.uint8)[None]).to(dev())
    ct = L.alice_encrypt(key, x, R)
    ct_out, bob = L.bob_eval(ct.clone(), we, R)
    alice = L.alice_decrypt(key, ct_out)
    Ls = OP.rns_layers(list(RNS), P, n, 32, 32, 3, 3, 1, 2, 3)
    pr = OP.PhiloxRandomnessRNS(5, 0, n, list(RNS), P)
    assert (to_np(t) == pr.secret()).all()
    te = [OP.secret_eval(Lr, pr.secret()) for Lr in Ls]
    wr = [OP.prepare_weights(Lr, w) for Lr in Ls]
    e, a = pr.enc_rns(0, 2, Ls[0].blocks)
    r = OP.run_layer_rns(Ls, te, img.astype(np.uint64), wr, e, a, pr.share(0, 3, Ls[0].blocks))
    ctx.permute(ct)
    assert (to_np(ct[0]) == r["ct_in"]).all()
    ctx.permute(ct_out)
    assert (to_np(ct_out[0]) == r["ct_out"]).all()
    assert (to_np(alice[0]).astype(np.uint64) == r["alice"]).all()
    assert (to_np(bob[0]).astype(np.uint64) == r["bob"]).all()
    out = L.forward(key, we, x, R)
    assert (to_np(out[0]).astype(np.uint64) == _direct(img, w, 32)).all()
