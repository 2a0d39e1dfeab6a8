"""The reference's randomness as a product feature ("parity mode").

REF draws every random value from per-party mt19937_64 streams (Rng, modfield.hpp:
104-130): Alice = Rng(seed).fork(0xA11CE) (keygen Gaussians, then per conv layer and
[channel][block] n Gaussians + n uniforms mod q, per activation n fresh shares),
Bob = Rng(seed).fork(0xB0B) (per conv layer and [out][block] n uniforms mod p).
RefRng runs that stream in libensei_gpu.so (ensei_gpu_ref_rng_*); SessionRandomness
replays it in REF's consumption order for a batch of image sessions and hands the
draws to the batched kernels through ops.Randomness's injected tensors, so device
ciphertexts, shares and transcripts equal the reference's for the same seeds.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Sequence

import numpy as np
import torch

from . import ops
from ._lib import check, lib

SALT_ALICE, SALT_BOB = 0xA11CE, 0xB0B


class RefRng:
    """REF Rng; RefRng(seed) or RefRng(seed, salt) == Rng(seed).fork(salt)."""

    def __init__(self, seed: int, salt: int | None = None):
        h = C.c_void_p()
        check(lib().ensei_gpu_ref_rng_create(seed, int(salt is not None), salt or 0, C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().ensei_gpu_ref_rng_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def next_u64(self, count: int) -> np.ndarray:
        out = np.empty(count, np.uint64)
        check(lib().ensei_gpu_ref_rng_next_u64(self.h, out.ctypes.data, count))
        return out

    def uniform_below(self, bound: int, count: int) -> np.ndarray:
        out = np.empty(count, np.uint64)
        check(lib().ensei_gpu_ref_rng_uniform_below(self.h, bound, out.ctypes.data, count))
        return out

    def gaussian(self, sigma: float, count: int) -> np.ndarray:
        out = np.empty(count, np.int64)
        check(lib().ensei_gpu_ref_rng_gaussian(self.h, sigma, out.ctypes.data, count))
        return out


def random_weights(schedule, magnitude: int, rng: RefRng) -> List[np.ndarray]:
    """REF random_weights (protocol.cpp:752-767): per conv layer [out][in][fh][fw] int64
    drawn as uniform_below(2m+1) - m."""
    out = []
    for s in schedule:
        if not hasattr(s, "cin"):
            continue
        cnt = s.cout * s.cin * s.fh * s.fw
        v = rng.uniform_below(2 * magnitude + 1, cnt).astype(np.int64) - magnitude
        out.append(v.reshape(s.cout, s.cin, s.fh, s.fw))
    return out


class SessionRandomness:
    """REF's per-party streams for a batch of image sessions, session i seeded seeds[i]."""

    def __init__(self, ctx: ops.Context, seeds: Sequence[int], sigma: float = 4.0):
        if ctx.R != 1:
            raise ValueError("REF's randomness is defined for single-prime q only")
        self.ctx, self.seeds, self.sigma = ctx, list(seeds), sigma
        self.alice = [RefRng(s, SALT_ALICE) for s in self.seeds]
        self.bob = [RefRng(s, SALT_BOB) for s in self.seeds]

    def keys(self) -> torch.Tensor:
        """keygen (REF ringbfv.cpp:95-107) per session; returns the key blobs
        [img][ENSEI_KEY_WORDS] (pass key_stride = blob.shape[1], or 0 for one image)."""
        n = self.ctx.n
        blobs = []
        for a in self.alice:
            t = torch.from_numpy(a.gaussian(self.sigma, n)).to(self.ctx.device)
            blobs.append(ops.secret_from_coeffs(self.ctx, t))
        return torch.stack(blobs)

    def conv(self, layer: int, cin: int, cout: int, blocks: int) -> ops.Randomness:
        """Alice's Enc draws ([c][b]: n Gaussians, then n uniforms mod q) and Bob's
        HomShare draws ([o][b]: n uniforms mod p) of one conv layer."""
        n, q, p = self.ctx.n, self.ctx.q[0], self.ctx.p
        imgs = len(self.seeds)
        e = np.empty((imgs, cin, blocks, n), np.int32)
        a = np.empty((imgs, cin, blocks, 1, n), np.uint64)
        s = np.empty((imgs, cout, blocks, n), np.int32)
        for i in range(imgs):
            for c in range(cin):
                for b in range(blocks):
                    e[i, c, b] = self.alice[i].gaussian(self.sigma, n)
                    a[i, c, b, 0] = self.alice[i].uniform_below(q, n)
            for o in range(cout):
                for b in range(blocks):
                    s[i, o, b] = self.bob[i].uniform_below(p, n).astype(np.int32)
        dev = self.ctx.device
        return ops.Randomness(layer=layer, noise=torch.from_numpy(e).to(dev), a_hat=torch.from_numpy(a).to(dev),
                              share=torch.from_numpy(s).to(dev))

    def activation(self, layer: int, channels: int, count: int) -> ops.Randomness:
        """trusted_activation's fresh shares (REF protocol.cpp:237-268) from Alice's stream."""
        p = self.ctx.p
        s = np.stack([self.alice[i].uniform_below(p, channels * count).astype(np.int32)
                      for i in range(len(self.seeds))])
        return ops.Randomness(layer=layer, share=torch.from_numpy(s).to(self.ctx.device).reshape(-1))

    def for_session(self, sess) -> "callable":
        """rand(layer_index) for protocol.Session.run / run_inproc in REF's order."""
        def rnd(li):
            s = sess.schedule[li]
            if hasattr(s, "cin"):
                return self.conv(li, s.cin, s.cout, sess.layers[li].B)
            prev = sess.layers[li - 1]
            return self.activation(li, sess.schedule[li - 1].cout, prev.geom.oh * prev.geom.ow)
        return rnd
