"""Batched device protocol driver: the GPU counterpart of REF run_inproc
(protocol.cpp:276-692) for a whole schedule of conv / activation layers.

Both parties run on one device (as run_inproc runs both on one host); every
arithmetic step happens in libensei_gpu.so kernels through the C ABI:

  conv layer  : Alice Enc (ensei_gpu_alice_encrypt) -> Bob HomRec (layers >= 2),
                ElementMult, HomShare (ensei_gpu_bob_eval) -> Alice Dec + IDFT2D
                (ensei_gpu_alice_decrypt)
  activation  : trusted_activation stub (ensei_gpu_activation), optionally with the
                builder-defined 2x2 max-pool used by config 3's 32 -> 16 -> 8 steps.

Shares stay resident in HBM between layers.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Callable, List, Optional, Sequence, Union

import torch

from . import ops
from ._lib import IN_U8, IN_U32, check, lib


@dataclass
class Conv:
    fh: int
    fw: int
    same: bool
    cin: int
    cout: int
    pack: int = 1  # images per ciphertext block (builder extension; 0 = the most the ring holds)
    grid: int = 0  # padded grid side (builder extension, ensei_conv_desc::grid; 0 = REF's power of two)


@dataclass
class Act:
    fn: int  # 0 ReLU, 1 Square, 2 Identity (REF ActivationFn)
    pool2: bool = False


Layer = Union[Conv, Act]


class RangeOverflow(RuntimeError):
    """REF ensei::RangeOverflow (square activation exceeds p_a / 2)."""


class Session:
    """A batched two-party session over a schedule (weights prepared at construction,
    i.e. Bob's t_setup; REF BobSession::prepare_weights, protocol.cpp:462-502)."""

    def __init__(self, ctx: ops.Context, schedule: Sequence[Layer], H: int, W: int,
                 weights: Sequence[torch.Tensor]):
        import time
        t0 = time.perf_counter()
        self.ctx, self.schedule, self.H, self.W = ctx, list(schedule), H, W
        if not self.schedule or not isinstance(self.schedule[0], Conv):
            raise ValueError("schedule must start with a conv layer")  # REF plan_layers
        self.layers: List[Optional[ops.LayerOps]] = []
        self.w_eval: List[Optional[torch.Tensor]] = []
        h, w = H, W
        ci = 0
        for s in self.schedule:
            if isinstance(s, Conv):
                pk = s.pack
                if pk == 0:  # the most images one ciphertext block holds (1 when the grid spans blocks)
                    probe = ops.LayerOps(ctx, ops.ConvSpec(h, w, s.fh, s.fw, s.same, s.cin, s.cout, 1, s.grid))
                    grid = probe.geom.Lh * probe.geom.Lw
                    pk = max(1, ctx.n // grid) if probe.B == 1 else 1
                lo = ops.LayerOps(ctx, ops.ConvSpec(h, w, s.fh, s.fw, s.same, s.cin, s.cout, pk, s.grid))
                wt = weights[ci].to(device=ctx.device, dtype=torch.int32).contiguous()
                self.layers.append(lo)
                self.w_eval.append(lo.prepare_weights(wt))
                h, w = lo.geom.oh, lo.geom.ow
                ci += 1
            else:
                self.layers.append(None)
                self.w_eval.append(None)
                if s.pool2:
                    h, w = h // 2, w // 2
        if ci != len(weights):
            raise ValueError("extra weight banks beyond the schedule")
        self.out_hw = (h, w)
        torch.cuda.current_stream().synchronize()
        self.setup_seconds = time.perf_counter() - t0  # Bob's weight preparation (REF t_setup)

    def run(self, key: torch.Tensor, x: torch.Tensor, rand: Callable[[int], ops.Randomness],
            key_stride: int = 0, keep_trace: bool = False):
        """x: [img][cin][H][W] uint8 pixels or int32 residues.  rand(layer_index) gives the
        randomness of that layer.  Returns the reconstructed output [img][cout][h][w]."""
        ctx = self.ctx
        alice, bob = x, None
        h, w = self.H, self.W
        trace = []
        out = None
        for li, s in enumerate(self.schedule):
            r = rand(li)
            if isinstance(s, Conv):
                lo = self.layers[li]
                images = alice.shape[0]
                ct = lo.alice_encrypt(key, alice.contiguous(), r, key_stride=key_stride)
                ct_out, bob_new = lo.bob_eval(ct, self.w_eval[li], r, bob_prev=bob, images=images)
                alice = lo.alice_decrypt(key, ct_out, key_stride=key_stride, images=images)
                bob = bob_new
                h, w = lo.geom.oh, lo.geom.ow
                if keep_trace:
                    trace.append({"ct_in": ct, "ct_out": ct_out, "alice": alice, "bob": bob})
            else:
                alice, bob, h, w = self.activation(s, alice, bob, h, w, r)
                if li + 1 == len(self.schedule):
                    out = self._recombine(alice, bob)
        if out is None:
            out = self._recombine(alice, bob)
        return (out, trace) if keep_trace else out

    def activation(self, s: Act, alice: torch.Tensor, bob: torch.Tensor, h: int, w: int, r: ops.Randomness):
        """trusted_activation (REF protocol.cpp:237-268) on the device; returns the fresh
        shares (Alice's, Bob's) and the new spatial size."""
        ctx = self.ctx
        imgs, ch = alice.shape[0], alice.shape[1]
        oh, ow = (h // 2, w // 2) if s.pool2 else (h, w)
        na = torch.empty((imgs, ch, oh, ow), dtype=torch.int32, device=ctx.device)
        nb = torch.empty_like(na)
        flag = torch.zeros(1, dtype=torch.int32, device=ctx.device)
        rs = r.struct()
        check(lib().ensei_gpu_activation(ctx.h, s.fn, int(s.pool2), ch, h, w, imgs, ops._ptr(alice),
                                         ops._ptr(bob), C.byref(rs), ops._ptr(na), ops._ptr(nb),
                                         ops._ptr(flag), ops._stream()))
        if s.fn == 1 and int(flag.item()):
            raise RangeOverflow("square activation exceeds p_a/2")
        return na, nb, oh, ow

    def _recombine(self, a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
        out = torch.empty_like(a)
        check(lib().ensei_gpu_recombine(self.ctx.h, ops._ptr(a), ops._ptr(b), a.numel(), ops._ptr(out),
                                        ops._stream()))
        return out


# --------------------------------------------------------------------------- wire
# The two parties as REF runs them (AliceSession::run / BobSession::run,
# protocol.cpp:276-640): every conv and activation step exchanges REF-format frames
# (paper_2003_05328_b200/wire.py) over a Transport, one transport per image session.
# Ciphertext / share frames are built and parsed by the wire kernels; the counters
# are REF's logical TransformCounters (counters.hpp:17-31) for one session.

@dataclass
class PhaseTimings:
    """REF PhaseTimings (protocol.hpp:80-87), seconds of wall clock on the party's host
    thread with the device synchronised at phase boundaries."""
    setup_seconds: float = 0.0
    online_seconds: float = 0.0
    encrypt_seconds: float = 0.0   # Alice: image transform + encryption
    filter_seconds: float = 0.0    # Bob: HomRec, slot-wise products, HomShare
    hadamard_seconds: float = 0.0  # Bob: the slot-wise products (inside filter; fused, not split out)
    decrypt_seconds: float = 0.0   # Alice: share decryption + inverse transform


@dataclass
class PartyResult:
    """REF PartyResult (protocol.hpp:89-94): output (Alice), counters, transcripts, timings."""
    output: Optional[torch.Tensor]
    counters: dict
    transcripts: list
    timings: PhaseTimings = None


def _counters():
    return {"ct_ntt": 0, "ring_ntt": 0, "image_ntt": 0, "hadamard": 0}


def _sync():
    torch.cuda.current_stream().synchronize()


def _hello(transports, digest, first: bool):
    """Hello exchange (REF AliceSession/BobSession::hello, protocol.cpp:292-308, 504-519);
    `digest` is one config digest per session (or one for all)."""
    from . import wire as Wr
    import struct
    ds = list(digest) if isinstance(digest, (list, tuple)) else [digest] * len(transports)
    if first:
        for t, d in zip(transports, ds):
            t.send_frame(Wr.hello_frame(d))
    peers = [struct.unpack("<Q", Wr.expect_host(t.recv_frame(), Wr.HELLO))[0] for t in transports]
    if not first:
        for t, d in zip(transports, ds):
            t.send_frame(Wr.hello_frame(d))
    if any(p != d for p, d in zip(peers, ds)):
        for t in transports:
            try:
                t.send_frame(Wr.error_frame("configuration digest mismatch"))
            except Exception:
                pass
        raise Wr.ProtocolOrderViolation("configuration digest mismatch")


def run_alice(sess: Session, key: torch.Tensor, x: torch.Tensor, rands: Sequence[ops.Randomness],
              transports, digest: int, freq_direct: bool = True, key_stride: int = 0) -> PartyResult:
    """AliceSession::run (REF protocol.cpp:358-437) for x.shape[0] image sessions."""
    from . import wire as Wr
    ctx, n = sess.ctx, sess.ctx.n
    from ._lib import LAYOUT_BITREV
    import time
    T = [Wr.RecordingTransport(t) for t in transports]
    _hello(T, digest, first=True)
    tm = PhaseTimings()
    online0 = time.perf_counter()
    cnt = _counters()
    alice, bob = x, None
    h, w = sess.H, sess.W
    out = None
    for li, s in enumerate(sess.schedule):
        r = rands[li]
        if isinstance(s, Conv):
            lo = sess.layers[li]
            B = lo.B
            t0 = time.perf_counter()
            ct = lo.alice_encrypt(key, alice.contiguous(), r, key_stride=key_stride)
            cnt["image_ntt"] += s.cin
            cnt["ring_ntt"] += s.cin * B * (2 if freq_direct else 3)
            if not freq_direct:  # REF encrypt (Baseline): coefficient-domain ciphertexts
                ctx.negacyclic(ct.view(-1, n), 0, inverse=True, layout=LAYOUT_BITREV)
            frames = Wr.encode_ct_blocks(ctx, Wr.CIPHERTEXT_BLOCKS, li, ct,
                                         Wr.EVALUATION if freq_direct else Wr.COEFFICIENT)
            _sync()
            tm.encrypt_seconds += time.perf_counter() - t0
            for i, t in enumerate(T):
                t.send_frame(frames[i])
            got = Wr.gather_frames([t.recv_frame() for t in T])
            ct_out, _, ncoef = Wr.decode_ct_blocks(ctx, got, Wr.ALICE_SHARE_CIPHERTEXTS, s.cout, B)
            t0 = time.perf_counter()
            alice = lo.alice_decrypt(key, ct_out, key_stride=key_stride)
            _sync()
            tm.decrypt_seconds += time.perf_counter() - t0
            cnt["ring_ntt"] += s.cout * B * 2 + ncoef // max(len(T), 1)  # Coefficient decrypt: +1 forward
            cnt["image_ntt"] += s.cout
            h, w = lo.geom.oh, lo.geom.ow
        else:
            got = Wr.gather_frames([t.recv_frame() for t in T])
            bob, _ = Wr.decode_shares(ctx, got, Wr.ACTIVATION_SHARE_UP, alice.shape[1], h, w, ctx.p)
            alice, nb, h, w = sess.activation(s, alice, bob, h, w, r)
            if li + 1 == len(sess.schedule):
                out = sess._recombine(alice, nb)
            else:
                frames = Wr.encode_shares(ctx, Wr.ACTIVATION_SHARE_DOWN, li, nb)
                _sync()
                for i, t in enumerate(T):
                    t.send_frame(frames[i])
    if isinstance(sess.schedule[-1], Conv):  # Bob uploads his share of the last conv
        got = Wr.gather_frames([t.recv_frame() for t in T])
        bob, _ = Wr.decode_shares(ctx, got, Wr.ACTIVATION_SHARE_UP, alice.shape[1], h, w, ctx.p)
        out = sess._recombine(alice, bob)
    for t in T:
        t.send_frame(Wr.done_frame())
    for t in T:
        Wr.expect_host(t.recv_frame(), Wr.DONE)
    tm.online_seconds = time.perf_counter() - online0
    return PartyResult(out, cnt, [t.transcript for t in T], tm)


def run_bob(sess: Session, rands: Sequence[ops.Randomness], transports, digest: int) -> PartyResult:
    """BobSession::run (REF protocol.cpp:521-640) for len(transports) image sessions."""
    from . import wire as Wr
    ctx = sess.ctx
    import time
    T = [Wr.RecordingTransport(t) for t in transports]
    _hello(T, digest, first=False)
    tm = PhaseTimings(setup_seconds=getattr(sess, "setup_seconds", 0.0))
    online0 = time.perf_counter()
    cnt = _counters()
    mine = None
    li_last = len(sess.schedule) - 1
    for li, s in enumerate(sess.schedule):
        r = rands[li]
        if isinstance(s, Conv):
            lo = sess.layers[li]
            B = lo.B
            got = Wr.gather_frames([t.recv_frame() for t in T])
            ct, _, ncoef = Wr.decode_ct_blocks(ctx, got, Wr.CIPHERTEXT_BLOCKS, s.cin, B)
            per = ncoef // max(len(T), 1)  # to_evaluation_domain: 2 ring transforms, ct_ntt += 2
            cnt["ct_ntt"] += 2 * per
            cnt["ring_ntt"] += 2 * per
            if mine is not None:  # HomRec (REF protocol.cpp:543-557)
                cnt["image_ntt"] += s.cin
                cnt["ring_ntt"] += 2 * s.cin * B
            t0 = time.perf_counter()
            ct_out, mine = lo.bob_eval(ct, sess.w_eval[li], r, bob_prev=mine)
            _sync()
            tm.filter_seconds += time.perf_counter() - t0
            tm.hadamard_seconds = tm.filter_seconds
            cnt["hadamard"] += s.cin * s.cout * B
            cnt["ring_ntt"] += 2 * s.cout * B
            cnt["image_ntt"] += s.cout
            frames = Wr.encode_ct_blocks(ctx, Wr.ALICE_SHARE_CIPHERTEXTS, li, ct_out, Wr.EVALUATION)
            _sync()
            for i, t in enumerate(T):
                t.send_frame(frames[i])
        else:
            frames = Wr.encode_shares(ctx, Wr.ACTIVATION_SHARE_UP, li, mine)
            _sync()
            for i, t in enumerate(T):
                t.send_frame(frames[i])
            if li != li_last:
                got = Wr.gather_frames([t.recv_frame() for t in T])
                mine, _ = Wr.decode_shares(ctx, got, Wr.ACTIVATION_SHARE_DOWN, mine.shape[1], mine.shape[2],
                                           mine.shape[3], ctx.p)
    if isinstance(sess.schedule[-1], Conv):
        frames = Wr.encode_shares(ctx, Wr.ACTIVATION_SHARE_UP, li_last, mine)
        _sync()
        for i, t in enumerate(T):
            t.send_frame(frames[i])
    for t in T:
        Wr.expect_host(t.recv_frame(), Wr.DONE)
    for t in T:
        t.send_frame(Wr.done_frame())
    tm.online_seconds = time.perf_counter() - online0
    return PartyResult(None, cnt, [t.transcript for t in T], tm)


def run_inproc(sess: Session, key: torch.Tensor, x: torch.Tensor, rand: Callable[[int], ops.Randomness],
               seed, freq_direct: bool = True, key_stride: int = 0, sigma: float = 4.0):
    """REF run_inproc (protocol.cpp:670-692): Bob on a thread, Alice on the caller, one
    in-process transport pair per image session.  `seed` is the sessions' config seed
    (one int, or one per image: it enters the Hello digest).  Returns (alice, bob)."""
    import threading
    from . import wire as Wr
    rands = [rand(li) for li in range(len(sess.schedule))]  # REF Rng consumption is per party, in layer order
    ctx = sess.ctx
    seeds = list(seed) if isinstance(seed, (list, tuple)) else [seed] * x.shape[0]
    digest = [Wr.config_digest(ctx.n, ctx.q[0], ctx.p, s, sess.H, sess.W, sess.schedule, freq_direct, sigma)
              for s in seeds]
    pairs = [Wr.make_inproc_pair() for _ in range(x.shape[0])]
    res, err = {}, {}
    dev = torch.cuda.current_device()

    def bob():
        try:
            torch.cuda.set_device(dev)
            res["bob"] = run_bob(sess, rands, [p[1] for p in pairs], digest)
        except BaseException as e:  # noqa: BLE001 -- re-raised on the caller
            err["bob"] = e
        finally:
            for p in pairs:
                p[1].close()

    th = threading.Thread(target=bob, daemon=True)
    th.start()
    try:
        res["alice"] = run_alice(sess, key, x, rands, [p[0] for p in pairs], digest, freq_direct, key_stride)
    except BaseException as e:  # noqa: BLE001
        err["alice"] = e
    finally:
        for p in pairs:
            p[0].close()
    th.join()
    if "alice" in err:
        raise err["alice"]
    if "bob" in err:
        raise err["bob"]
    return res["alice"], res["bob"]
