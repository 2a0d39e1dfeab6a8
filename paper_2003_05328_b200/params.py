"""Parameter selection over the C ABI: REF params.cpp (min_pntt, build_params, derive_q,
preset_params) plus the RNS extension for large channel accumulation (ensei_gpu.h,
"parameters").  The result feeds ops.Context(n=..., q=ps.q_primes, p=ps.p)."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Tuple

from ._lib import ParamSet as _PS
from ._lib import PrecisionProfile as _Prof
from ._lib import check, lib

UNIFIED, SPLIT_PAPER = 0, 1  # REF ChainMode


@dataclass(frozen=True)
class Profile:
    """REF PrecisionProfile (params.hpp:11-17)."""
    input_bits: int
    filter_bits: int
    f_h: int
    f_w: int

    def c(self) -> _Prof:
        return _Prof(self.input_bits, self.filter_bits, self.f_h, self.f_w)


@dataclass(frozen=True)
class ParamSet:
    """REF ParamSet (params.hpp:27-34); q_primes has one entry (REF) or several (RNS)."""
    p_n: int
    p_a: int
    p_e: int
    n: int
    q_primes: Tuple[int, ...]
    sigma: float
    log2_q_min: float
    mode: int
    insecure: bool
    profile: Profile

    @property
    def p(self) -> int:
        return self.p_e

    @property
    def q(self) -> int:
        out = 1
        for x in self.q_primes:
            out *= x
        return out


def _wrap(ps: _PS) -> ParamSet:
    pr = ps.profile
    return ParamSet(ps.p_n, ps.p_a, ps.p_e, ps.n, tuple(ps.q[i] for i in range(ps.num_q)), ps.sigma, ps.log2_q_min,
                    ps.mode, bool(ps.insecure), Profile(pr.input_bits, pr.filter_bits, pr.f_h, pr.f_w))


def min_pntt(profile: Profile) -> int:
    out = C.c_uint64()
    check(lib().ensei_gpu_min_pntt(C.byref(profile.c()), C.byref(out)))
    return out.value


def build_params(profile: Profile, n: int, mode: int = UNIFIED, accum_channels: int = 1, p_n_floor: int = 0,
                 sigma: float = 4.0, max_primes: int = 1, min_primes: int = 1) -> ParamSet:
    """REF build_params; max_primes > 1 allows an RNS q where REF's single prime runs out."""
    ps = _PS()
    check(lib().ensei_gpu_build_params(C.byref(profile.c()), n, mode, accum_channels, p_n_floor, sigma, max_primes,
                                       min_primes, C.byref(ps)))
    return _wrap(ps)


def preset_params(name: str, accum_channels: int = 1, max_primes: int = 1) -> ParamSet:
    ps = _PS()
    check(lib().ensei_gpu_preset_params(name.encode(), accum_channels, max_primes, C.byref(ps)))
    return _wrap(ps)


def preset_names():
    return ["binary", "medium", "high", "toy"]
