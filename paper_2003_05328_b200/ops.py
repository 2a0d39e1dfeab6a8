"""Python mirror of the reference operator surface over the C ABI.

Names follow REF (ntt_2d / intt_2d, NegacyclicPlan.forward / inverse,
encode_slots / decode_slots, prepare_plain, encrypt_freq_direct, mul_plain,
hom_share, hom_rec, decrypt, run_inproc).  torch is used only for device memory
and streams; every operation runs in libensei_gpu.so kernels.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import (ConvDesc, CtxInfo, ENSEI_MOD_P, IN_U8, IN_U32, LAYOUT_BITREV, LAYOUT_NATURAL,
                   LayerGeom, RAND_INJECTED, RAND_PHILOX, Randomness, check, lib)

P_DEFAULT = 638977
Q_DEFAULT = 576460803525083137
RNS_DEFAULT = (576460803525083137, 576461033843064833, 576461054781063169)
SALT_ALICE, SALT_BOB = 0xA11CE, 0xB0B


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def mix64(x: int) -> int:
    """splitmix64 finalizer (REF modfield.cpp:79-85)."""
    M = (1 << 64) - 1
    x = (x + 0x9E3779B97F4A7C15) & M
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M
    return x ^ (x >> 31)


def fork_seed(seed: int, salt: int) -> int:
    """Rng(seed).fork(salt) seed derivation (REF modfield.cpp:221-223)."""
    return mix64(seed ^ mix64(salt))


class Context:
    """RlweParams + ModulusChain (unified p) on one device (REF ringbfv.cpp:65-87)."""

    def __init__(self, n: int = 2048, q=(Q_DEFAULT,), p: int = P_DEFAULT, device: int = 0):
        if isinstance(q, int):
            q = (q,)
        arr = (C.c_uint64 * len(q))(*q)
        h = C.c_void_p()
        torch.cuda.set_device(device)
        check(lib().ensei_gpu_ctx_create(device, n, arr, len(q), p, C.byref(h)))
        self.h = h
        info = CtxInfo()
        check(lib().ensei_gpu_ctx_query(h, C.byref(info)))
        self.info = info
        self.n, self.p, self.R = n, p, len(q)
        self.q = tuple(q)
        self.device = torch.device("cuda", device)

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().ensei_gpu_ctx_destroy(self.h)
                self.h = None
        except Exception:
            pass

    # ---- single transforms (config 2 / boundary ops)
    def negacyclic(self, x: torch.Tensor, modulus: int = 0, inverse: bool = False,
                   layout: int = LAYOUT_NATURAL, stream=None) -> torch.Tensor:
        """In-place NegacyclicPlan::forward/inverse on rows of a uint64 tensor [..., n]."""
        assert x.dtype == torch.uint64 and x.is_cuda and x.is_contiguous() and x.shape[-1] == self.n
        check(lib().ensei_gpu_negacyclic(self.h, modulus, int(inverse), layout, _ptr(x),
                                         x.numel() // self.n, _stream(stream)))
        return x

    def encode_slots(self, x, stream=None):
        return self.negacyclic(x, ENSEI_MOD_P, inverse=True, stream=stream)

    def decode_slots(self, x, stream=None):
        return self.negacyclic(x, ENSEI_MOD_P, inverse=False, stream=stream)

    def ntt_2d(self, x: torch.Tensor, inverse: bool = False, stream=None) -> torch.Tensor:
        """In-place ntt_2d / intt_2d on uint64 tiles [..., rows, cols]."""
        assert x.dtype == torch.uint64 and x.is_cuda and x.is_contiguous()
        rows, cols = x.shape[-2:]
        check(lib().ensei_gpu_ntt2d(self.h, int(inverse), rows, cols, _ptr(x), x.numel() // (rows * cols),
                                    _stream(stream)))
        return x

    def intt_2d(self, x, stream=None):
        return self.ntt_2d(x, inverse=True, stream=stream)

    def permute(self, x: torch.Tensor, stream=None) -> torch.Tensor:
        check(lib().ensei_gpu_permute(self.h, 1, _ptr(x), x.numel() // self.n, _stream(stream)))
        return x
