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
        self.ctx, self.schedule, self.H, self.W = ctx, list(schedule), H, W
        if not self.schedule or not isinstance(self.schedule[0], Conv):
            raise ValueError("schedule must start with a conv layer")  # REF plan_layers
        self.layers: List[Optional[ops.LayerOps]] = []
        self.w_eval: List[Optional[torch.Tensor]] = []
        h, w = H, W
        ci = 0
        for s in self.schedule:
            if isinstance(s, Conv):
                lo = ops.LayerOps(ctx, ops.ConvSpec(h, w, s.fh, s.fw, s.same, s.cin, s.cout))
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
                ct = lo.alice_encrypt(key, alice.contiguous(), r, key_stride=key_stride)
                ct_out, bob_new = lo.bob_eval(ct, self.w_eval[li], r, bob_prev=bob)
                alice = lo.alice_decrypt(key, ct_out, key_stride=key_stride)
                bob = bob_new
                h, w = lo.geom.oh, lo.geom.ow
                if keep_trace:
                    trace.append({"ct_in": ct, "ct_out": ct_out, "alice": alice, "bob": bob})
            else:
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
                alice, bob = na, nb
                h, w = oh, ow
                if li + 1 == len(self.schedule):
                    out = self._recombine(alice, bob)
        if out is None:
            out = self._recombine(alice, bob)
        return (out, trace) if keep_trace else out

    def _recombine(self, a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
        out = torch.empty_like(a)
        check(lib().ensei_gpu_recombine(self.ctx.h, ops._ptr(a), ops._ptr(b), a.numel(), ops._ptr(out),
                                        ops._stream()))
        return out
