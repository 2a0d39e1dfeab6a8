"""GPU: device wire framing (ensei_gpu_wire_*) against the compiled reference's own
wire code (oracle/_ref: write_ciphertext / encode_frame / read_ciphertext / decode_frame)
-- frames byte-identical, decoding identical, every REF error reproduced in kind and
message -- and whole two-party sessions over transports whose transcript hashes,
byte counts and transform counters equal the reference's (tests/golden/golden.json)."""
import ctypes as C
import struct

import numpy as np
import pytest
import torch

import oracle as O
from conftest import fnv
from gpu_util import P, Q, dev, golden_inputs, to_np
from oracle import protocol as OP

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def W():
    from paper_2003_05328_b200 import wire
    return wire


@pytest.fixture(scope="module")
def ops():
    from paper_2003_05328_b200 import ops as _ops
    return _ops


_CTX = {}


def ctx_for(ops, n):
    if n not in _CTX:
        _CTX[n] = ops.Context(n=n)
    return _CTX[n]


def perm(n):
    bits = n.bit_length() - 1
    return np.array([int(format(i, f"0{bits}b")[::-1], 2) for i in range(n)])


def ref_ct_frame(W, msg, layer, n, cts_nat, tag):
    """REF encode_frame(encode_ct_blocks(...)) of natural-order cts [ch][B][2][n]."""
    ch, B = cts_nat.shape[:2]
    cap = W.ct_frame_bytes(n, ch, B)
    out = np.zeros(cap, np.uint8)
    ln = C.c_size_t()
    assert O.ref().ref_wire_ct_frame(msg, layer, n, ch, B, tag, np.ascontiguousarray(cts_nat, np.uint64).reshape(-1),
                                     out.ctypes.data, cap, C.byref(ln)) == 0
    assert ln.value == cap
    return out


def ref_ct_decode(W, frame, msg, n, ch, B):
    cts = np.zeros(ch * B * 2 * n, np.uint64)
    tags = np.zeros(max(ch * B, 1), np.uint8)
    layer = C.c_uint32()
    rc = O.ref().ref_wire_ct_decode(frame.ctypes.data, frame.size, msg, P, Q, n, ch, B, C.byref(layer), cts,
                                    tags.ctypes.data)
    kind = {0: None, 14: "MalformedPayload", 12: "ProtocolOrderViolation"}[rc]
    return kind, O.ref().ref_last_error().decode(), cts.reshape(ch, B, 2, n), tags, layer.value


def device_ct(ops, ctx, nat):
    """natural-order cts [img][ch][B][2][n] -> device layout tensor [img][ch][B][2][1][n]"""
    n = nat.shape[-1]
    t = torch.from_numpy(np.ascontiguousarray(nat[..., perm(n)], np.uint64)).to(dev())
    return t.reshape(*nat.shape[:-1], 1, n).contiguous()


@pytest.mark.parametrize("n,ch,B,imgs", [(2048, 3, 2, 3), (4096, 1, 1, 2), (8192, 2, 1, 1), (2048, 16, 2, 8)])
@pytest.mark.parametrize("where", ["pinned", "device"])
def test_encode_ct_frames_byte_identical(W, ops, n, ch, B, imgs, where):
    ctx = ctx_for(ops, n)
    rng = np.random.default_rng(n + ch + imgs)
    nat = rng.integers(0, Q, size=(imgs, ch, B, 2, n), dtype=np.uint64)
    nat[0, 0, 0, 0, :3] = [0, Q - 1, 1]
    ct = device_ct(ops, ctx, nat)
    fb = W.ct_frame_bytes(n, ch, B)
    stride = fb + 5  # odd stride: every frame starts at a different alignment
    if where == "pinned":
        buf = torch.full((imgs, stride), 0xAB, dtype=torch.uint8).pin_memory()
    else:
        buf = torch.full((imgs, stride), 0xAB, dtype=torch.uint8, device=dev())
    W.encode_ct_blocks(ctx, W.CIPHERTEXT_BLOCKS, 7, ct, out=buf)
    torch.cuda.synchronize()
    got = buf.cpu().numpy()
    for i in range(imgs):
        assert (got[i, :fb] == ref_ct_frame(W, W.CIPHERTEXT_BLOCKS, 7, n, nat[i], 1)).all(), i
        assert (got[i, fb:] == 0xAB).all()  # nothing written past the frame
    # decode back (device-resident frames too), through the odd stride
    out, layers, ncoef = W.decode_ct_blocks(ctx, buf[:, :fb] if where == "device" else buf.narrow(1, 0, fb),
                                            W.CIPHERTEXT_BLOCKS, ch, B)
    assert layers == [7] * imgs and ncoef == 0
    assert (to_np(out) == to_np(ct)).all()


def test_decode_reference_frames(W, ops):
    n, ch, B = 2048, 2, 2
    ctx = ctx_for(ops, n)
    rng = np.random.default_rng(11)
    nat = rng.integers(0, Q, size=(ch, B, 2, n), dtype=np.uint64)
    f = ref_ct_frame(W, W.ALICE_SHARE_CIPHERTEXTS, 4, n, nat, 1)
    kind, _, cts, tags, layer = ref_ct_decode(W, f, W.ALICE_SHARE_CIPHERTEXTS, n, ch, B)
    assert kind is None and layer == 4 and (cts == nat).all()
    fr = torch.from_numpy(f).reshape(1, -1).pin_memory()
    out, layers, _ = W.decode_ct_blocks(ctx, fr, W.ALICE_SHARE_CIPHERTEXTS, ch, B)
    assert layers == [4]
    assert (to_np(out)[0, ..., 0, :][..., perm(n)] == nat).all()


def test_coefficient_records_enter_evaluation_domain(W, ops):
    """Baseline-mode records (tag 0) are moved to the evaluation domain on decode, as REF's
    BobSession does with to_evaluation_domain; mixed tags in one batch too."""
    n, ch, B = 2048, 2, 1
    ctx = ctx_for(ops, n)
    rng = np.random.default_rng(12)
    nat = rng.integers(0, Q, size=(2, ch, B, 2, n), dtype=np.uint64)
    frames = [ref_ct_frame(W, W.CIPHERTEXT_BLOCKS, 0, n, nat[0], 0),  # all Coefficient
              ref_ct_frame(W, W.CIPHERTEXT_BLOCKS, 0, n, nat[1], 1)]  # all Evaluation
    fr = torch.from_numpy(np.stack(frames)).pin_memory()
    out, _, ncoef = W.decode_ct_blocks(ctx, fr, W.CIPHERTEXT_BLOCKS, ch, B)
    assert ncoef == ch * B
    got = to_np(out)[..., 0, :][..., perm(n)]
    ev = O.negacyclic(nat[0].reshape(-1, n), Q).reshape(nat[0].shape)  # REF NegacyclicPlan::forward (pinned)
    assert (got[0] == ev).all()
    assert (got[1] == nat[1]).all()
    # Coefficient-domain encode (REF Baseline encrypt output) is written as-is with tag 0
    ct0 = torch.from_numpy(nat[:1].reshape(1, ch, B, 2, 1, n)).to(dev())
    enc = W.encode_ct_blocks(ctx, W.CIPHERTEXT_BLOCKS, 0, ct0, domain=W.COEFFICIENT)
    torch.cuda.synchronize()
    assert (enc.numpy()[0] == frames[0]).all()


def _corruptions(W, f, n, ch, B, q=Q):
    rb = 9 + 16 * n
    hdr = 26

    def setb(buf, off, val):
        b = buf.copy()
        b[off] = val
        return b

    def setu64(buf, off, v):
        b = buf.copy()
        b[off:off + 8] = np.frombuffer(struct.pack("<Q", v), np.uint8)
        return b

    def setlen(buf):  # header length consistent with the (shortened / extended) frame
        return setu64(buf, 6, buf.size - 14)

    last = hdr + (ch * B - 1) * rb
    return {
        "magic": setb(f, 0, ord("X")),
        "version": setb(f, 4, 2),
        "type": setb(f, 5, 9),
        "cap": setu64(f, 6, (1 << 30) + 1),
        "length": f[:-3].copy(),
        "peer_error": np.frombuffer(W.error_frame("bob gave up"), np.uint8).copy(),
        "unexpected": setb(f, 5, W.ACTIVATION_SHARE_UP),
        "short_payload_hdr": setlen(f[:20].copy()),
        "layout_channels": setb(f, 18, ch + 1),
        "layout_blocks": setb(f, 22, B + 1),
        "tag_first": setb(f, hdr, 2),
        "tag_last": setb(f, last, 7),
        "ring_dim": setu64(f, hdr + rb + 1 if ch * B > 1 else hdr + 1, n // 2),
        "coef_eq_q": setu64(f, hdr + 9 + 8 * 5, q),
        "coef_last_max": setu64(f, last + 9 + 8 * (2 * n - 1), (1 << 64) - 1),
        "two_errors_order": setu64(setb(f, last, 3), hdr + 9, q + 1),  # earlier position wins
        "truncated": setlen(f[:-8].copy()),
        "trailing": setlen(np.concatenate([f, np.zeros(5, np.uint8)])),
    }


@pytest.mark.parametrize("n,ch,B", [(2048, 2, 2), (4096, 1, 1)])
def test_decode_errors_match_reference(W, ops, n, ch, B):
    ctx = ctx_for(ops, n)
    rng = np.random.default_rng(n)
    nat = rng.integers(0, Q, size=(ch, B, 2, n), dtype=np.uint64)
    f = ref_ct_frame(W, W.CIPHERTEXT_BLOCKS, 1, n, nat, 1)
    for name, bad in _corruptions(W, f, n, ch, B).items():
        kind, msg, *_ = ref_ct_decode(W, bad, W.CIPHERTEXT_BLOCKS, n, ch, B)
        assert kind is not None, name
        for where in ("pinned", "device"):
            t = torch.from_numpy(bad).reshape(1, -1)
            t = t.pin_memory() if where == "pinned" else t.to(dev())
            with pytest.raises(W.EnseiError) as e:
                W.decode_ct_blocks(ctx, t, W.CIPHERTEXT_BLOCKS, ch, B)
            assert e.value.kind == kind, (name, where, str(e.value), msg)
            assert msg in str(e.value), (name, where, str(e.value), msg)
    # an error in the third frame of a batch is reported for that frame
    good = torch.from_numpy(np.stack([f, f, _corruptions(W, f, n, ch, B)["coef_eq_q"]])).pin_memory()
    with pytest.raises(W.EnseiError, match=r"coefficient out of range \(frame 2\)"):
        W.decode_ct_blocks(ctx, good, W.CIPHERTEXT_BLOCKS, ch, B)


def _ref_share_frame(W, msg, layer, v):
    ch, r, c = v.shape
    cap = W.share_frame_bytes(ch, r, c)
    out = np.zeros(cap, np.uint8)
    ln = C.c_size_t()
    assert O.ref().ref_wire_share_frame(msg, layer, ch, r, c, np.ascontiguousarray(v, np.uint64).reshape(-1),
                                        out.ctypes.data, cap, C.byref(ln)) == 0
    return out


@pytest.mark.parametrize("shape,imgs", [((3, 5, 7), 3), ((16, 32, 32), 8), ((1, 1, 1), 2)])
def test_shares_frames_vs_reference(W, ops, shape, imgs):
    ctx = ctx_for(ops, 2048)
    rng = np.random.default_rng(sum(shape))
    v = rng.integers(0, P, size=(imgs, *shape), dtype=np.uint64)
    t = torch.from_numpy(v.astype(np.int32)).to(dev())
    fb = W.share_frame_bytes(*shape)
    buf = torch.full((imgs, fb + 3), 0xCD, dtype=torch.uint8).pin_memory()
    W.encode_shares(ctx, W.ACTIVATION_SHARE_UP, 5, t, out=buf)
    torch.cuda.synchronize()
    g = buf.numpy()
    for i in range(imgs):
        assert (g[i, :fb] == _ref_share_frame(W, W.ACTIVATION_SHARE_UP, 5, v[i])).all()
        assert (g[i, fb:] == 0xCD).all()
    back, layers = W.decode_shares(ctx, buf.narrow(1, 0, fb), W.ACTIVATION_SHARE_UP, *shape, P)
    assert layers == [5] * imgs and (to_np(back).astype(np.uint64) == v).all()
    # errors: out-of-range value, layout mismatch, unexpected type -- as REF decode_shares
    f = _ref_share_frame(W, W.ACTIVATION_SHARE_UP, 5, v[0])
    cases = {"range": f.copy(), "layout": f.copy(), "type": f.copy()}
    cases["range"][30 + 8 * (v[0].size - 1):30 + 8 * v[0].size] = np.frombuffer(struct.pack("<Q", P), np.uint8)
    cases["layout"][26] += 1
    cases["type"][5] = W.ACTIVATION_SHARE_DOWN
    for name, bad in cases.items():
        layer = C.c_uint32()
        tmp = np.zeros(v[0].size, np.uint64)
        rc = O.ref().ref_wire_share_decode(bad.ctypes.data, bad.size, W.ACTIVATION_SHARE_UP, *shape, P,
                                           C.byref(layer), tmp)
        kind = {14: "MalformedPayload", 12: "ProtocolOrderViolation"}[rc]
        msg = O.ref().ref_last_error().decode()
        with pytest.raises(W.EnseiError) as e:
            W.decode_shares(ctx, torch.from_numpy(bad).reshape(1, -1).pin_memory(), W.ACTIVATION_SHARE_UP,
                            *shape, P)
        assert e.value.kind == kind and msg in str(e.value), (name, str(e.value), msg)


def _inject(ops, rand, li, cin, cout, B, n):
    e, a = rand.enc(li, cin, B)
    s = rand.share(li, cout, B)
    from gpu_util import u64
    return ops.Randomness(layer=li, noise=torch.from_numpy(e.astype(np.int32)).to(dev()).reshape(1, cin, B, n),
                          a_hat=u64(a).reshape(1, cin, B, 1, n),
                          share=torch.from_numpy(s.astype(np.int32)).to(dev()).reshape(1, cout, B, n))


@pytest.mark.parametrize("idx", [0, 1, 2, 3, 4])
def test_wire_session_transcripts_equal_reference(W, ops, golden, idx):
    """REF run_inproc over real frames: Alice/Bob transcript FNV chains, bytes sent,
    TransformCounters and the output equal the reference's (FreqDirect and Baseline)."""
    from paper_2003_05328_b200 import protocol as GP
    case = golden["proto"][idx]
    img, ws, sched = golden_inputs(case)
    n = case["n"]
    ctx = ctx_for(ops, n)
    gs = [GP.Conv(s.fh, s.fw, s.same, s.cin, s.cout) if isinstance(s, OP.Conv) else GP.Act(s.fn) for s in sched]
    sess = GP.Session(ctx, gs, case["H"], case["W"], [torch.from_numpy(w.astype(np.int32)) for w in ws])
    rand = OP.RefRandomness(case["seed"], n, Q, P)
    key = ops.secret_from_coeffs(ctx, torch.from_numpy(rand.secret()).to(dev()))

    def rnd(li):
        s = sched[li]
        if isinstance(s, OP.Conv):
            return _inject(ops, rand, li, s.cin, s.cout, sess.layers[li].B, n)
        lo = sess.layers[li - 1]
        fresh = rand.reshare(li, sched[li - 1].cout, lo.geom.oh * lo.geom.ow)
        return ops.Randomness(layer=li, share=torch.from_numpy(fresh.astype(np.int32)).to(dev()).reshape(-1))

    x = torch.from_numpy(img.astype(np.int32)[None]).to(dev())
    alice, bob = GP.run_inproc(sess, key, x, rnd, seed=case["seed"], freq_direct=bool(case["mode"]))
    assert fnv(to_np(alice.output).astype(np.uint64).reshape(-1)) == case["out_fnv"]
    ta, tb = alice.transcripts[0], bob.transcripts[0]
    assert "%016x" % ta.content_hash_sent == case["alice_sent"]
    assert "%016x" % ta.content_hash_recv == case["alice_recv"]
    assert ta.total_bytes("sent") == case["alice_bytes_sent"]
    assert tb.total_bytes("sent") == case["bob_bytes_sent"]
    assert tb.content_hash_recv == ta.content_hash_sent and tb.content_hash_sent == ta.content_hash_recv
    order = ["ct_ntt", "ring_ntt", "image_ntt", "hadamard"]
    assert [alice.counters[k] for k in order] == case["counters_alice"]
    assert [bob.counters[k] for k in order] == case["counters_bob"]


def test_wire_session_batched_philox(W, ops):
    """Batched sessions (4 images, one transport each) in throughput mode: outputs equal the
    plaintext convolution, and the same images run without the wire give the same shares."""
    from paper_2003_05328_b200 import protocol as GP
    ctx = ctx_for(ops, 2048)
    g = torch.Generator().manual_seed(9)
    x = torch.randint(0, 256, (4, 3, 16, 16), dtype=torch.uint8, generator=g)
    w1 = torch.randint(-128, 128, (4, 3, 3, 3), dtype=torch.int32, generator=g)
    w2 = torch.randint(-128, 128, (2, 4, 1, 1), dtype=torch.int32, generator=g)
    sess = GP.Session(ctx, [GP.Conv(3, 3, True, 3, 4), GP.Act(0), GP.Conv(1, 1, True, 4, 2)], 16, 16, [w1, w2])
    _, key = ops.secret_sample(ctx, 3)
    rnd = lambda li: ops.Randomness(seed=3, layer=li)  # noqa: E731
    alice, bob = GP.run_inproc(sess, key, x.to(dev()), rnd, seed=3)
    direct = sess.run(key, x.to(dev()), rnd)
    assert (to_np(alice.output) == to_np(direct)).all()
    hs = {t.content_hash_sent for t in alice.transcripts}
    assert len(hs) == 4  # four distinct sessions
    # REF PhaseTimings on both parties (protocol.hpp:80-87)
    ta, tb = alice.timings, bob.timings
    assert ta.online_seconds > 0 and ta.encrypt_seconds > 0 and ta.decrypt_seconds > 0
    assert ta.encrypt_seconds + ta.decrypt_seconds <= ta.online_seconds
    assert tb.setup_seconds > 0 and tb.filter_seconds > 0 and tb.filter_seconds <= tb.online_seconds


def _ref_run(seed, H, Wd, desc, img, ws, mode=1, n=2048):
    hashes = np.zeros(6, np.uint64)
    h, w, ch = H, Wd, desc[0][4]
    for d in desc:
        if d[0] == 0:
            h, w, ch = (h if d[3] else h - d[1] + 1), (w if d[3] else w - d[2] + 1), d[5]
    out = np.zeros(ch * h * w, np.uint64)
    O.ref_check(O.ref().ref_run_protocol(P, Q, n, 4.0, mode, seed, H, Wd, len(desc),
                                         np.array(desc, np.int32).reshape(-1), img.reshape(-1).astype(np.int64),
                                         np.concatenate([x.reshape(-1) for x in ws]).astype(np.int64), out,
                                         hashes.ctypes.data, None, 0, None, None, None, None))
    return out, hashes


@pytest.mark.parametrize("idx", [1, 2])
def test_product_parity_mode_from_json_schedule(W, ops, golden, idx):
    """Product-only REF-compatible run: a JSON schedule (schedule.py), REF's fixture draws
    and per-party streams from the product's RefRng (refrand.py), frames over transports:
    the transcripts equal the reference's golden ones -- no oracle code on this path."""
    import json
    from paper_2003_05328_b200 import protocol as GP
    from paper_2003_05328_b200 import refrand as RR
    from paper_2003_05328_b200 import schedule as S
    case = golden["proto"][idx]
    layers = [{"kind": "conv", "filter_h": d[1], "filter_w": d[2], "conv_type": "same" if d[3] else "valid",
               "channels_in": d[4], "channels_out": d[5]} if d[0] == 0 else {"kind": "activation",
                                                                                "fn": S.FN_NAME[d[6]]}
              for d in case["desc"]]
    sf = S.parse_schedule(json.dumps({"layers": layers}))
    H, Wd, n = case["H"], case["W"], case["n"]
    g = RR.RefRng(case["seed"], 0xDA7A)
    cin = sf.schedule[0].cin
    img = g.uniform_below(256, cin * H * Wd).astype(np.int64).reshape(cin, H, Wd)
    ws = [(g.uniform_below(256, s.cout * s.cin * s.fh * s.fw).astype(np.int64) - 128).reshape(s.cout, s.cin, s.fh,
                                                                                               s.fw)
          for s in sf.schedule if isinstance(s, GP.Conv)]
    ctx = ctx_for(ops, n)
    sess = GP.Session(ctx, sf.schedule, H, Wd, [torch.from_numpy(w.astype(np.int32)) for w in ws])
    sr = RR.SessionRandomness(ctx, [case["seed"]])
    key = sr.keys()[0]
    x = torch.from_numpy(img.astype(np.int32)[None]).to(dev())
    alice, bob = GP.run_inproc(sess, key, x, sr.for_session(sess), seed=case["seed"], freq_direct=bool(case["mode"]))
    ta = alice.transcripts[0]
    assert "%016x" % ta.content_hash_sent == case["alice_sent"]
    assert "%016x" % ta.content_hash_recv == case["alice_recv"]
    assert fnv(to_np(alice.output).astype(np.uint64).reshape(-1)) == case["out_fnv"]


def test_product_parity_mode_batched_sessions(W, ops):
    """Three image sessions with their own seeds and keys in one batched run (key_stride):
    every session's transcripts and output equal an independent reference run."""
    from paper_2003_05328_b200 import protocol as GP
    from paper_2003_05328_b200 import refrand as RR
    desc = [[0, 3, 3, 1, 2, 3, 0], [1, 0, 0, 0, 0, 0, 1], [0, 1, 1, 0, 3, 2, 0]]
    sched = [GP.Conv(3, 3, True, 2, 3), GP.Act(1), GP.Conv(1, 1, False, 3, 2)]
    H = Wd = 8
    ctx = ctx_for(ops, 2048)
    rng = np.random.default_rng(77)
    imgs = rng.integers(0, 4, size=(3, 2, H, Wd)).astype(np.int64)  # small: keeps Square in range
    ws = [rng.integers(-2, 3, size=(3, 2, 3, 3)).astype(np.int64), rng.integers(-2, 3, size=(2, 3, 1, 1))]
    seeds = [101, 5, 999]
    sess = GP.Session(ctx, sched, H, Wd, [torch.from_numpy(w.astype(np.int32)) for w in ws])
    sr = RR.SessionRandomness(ctx, seeds)
    keys = sr.keys()
    x = torch.from_numpy(imgs.astype(np.int32)).to(dev())
    alice, bob = GP.run_inproc(sess, keys, x, sr.for_session(sess), seed=seeds, key_stride=keys.shape[1])
    out = to_np(alice.output).astype(np.uint64)
    for i, s in enumerate(seeds):
        ref_out, h = _ref_run(s, H, Wd, desc, imgs[i], ws)
        assert (out[i].reshape(-1) == ref_out).all(), i
        assert alice.transcripts[i].content_hash_sent == int(h[0]) and alice.transcripts[i].content_hash_recv == int(h[1])
        assert bob.transcripts[i].content_hash_sent == int(h[2]) and bob.transcripts[i].content_hash_recv == int(h[3])
        assert alice.transcripts[i].total_bytes("sent") == int(h[4])
        assert bob.transcripts[i].total_bytes("sent") == int(h[5])


def test_concurrent_decodes_keep_their_own_status(W, ops):
    """The two parties of run_inproc decode from two host threads on one context: each
    decode must report its own frames' errors (the status block is per-context)."""
    import threading
    n, ch, B = 2048, 2, 1
    ctx = ctx_for(ops, n)
    rng = np.random.default_rng(21)
    nat = rng.integers(0, Q, size=(ch, B, 2, n), dtype=np.uint64)
    good = ref_ct_frame(W, W.CIPHERTEXT_BLOCKS, 0, n, nat, 1)
    bad = _corruptions(W, good, n, ch, B)["coef_eq_q"]
    res = {"good": [], "bad": []}

    def run(name, frame):
        t = torch.from_numpy(frame).reshape(1, -1).pin_memory()
        for _ in range(40):
            try:
                W.decode_ct_blocks(ctx, t, W.CIPHERTEXT_BLOCKS, ch, B)
                res[name].append(None)
            except W.EnseiError as e:
                res[name].append(e.kind)

    th = [threading.Thread(target=run, args=("good", good)), threading.Thread(target=run, args=("bad", bad))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert res["good"] == [None] * 40
    assert res["bad"] == ["MalformedPayload"] * 40
