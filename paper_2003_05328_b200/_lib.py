"""ctypes binding of the C ABI (include/ensei_gpu.h) -> libensei_gpu.so.

This is the ONLY way the Python side reaches the device path.  There is no CPU
fallback: if the in-tree .so is missing or fails to load, every call raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(HERE, "libensei_gpu.so")

ENSEI_MAX_PRIMES = 4
ENSEI_MOD_P = 0xFFFFFFFF
LAYOUT_NATURAL, LAYOUT_BITREV = 0, 1
RAND_PHILOX, RAND_INJECTED = 0, 1
IN_U32, IN_U8 = 0, 1

STATUS_NAMES = {
    1: "Error", 2: "OrderNotDividing", 3: "SearchExhausted", 4: "BadRoot", 5: "BadGeometry",
    6: "GeometryMismatch", 7: "DomainMismatch", 8: "NoiseExhausted", 9: "ChainViolation",
    10: "LengthMismatch", 11: "RangeViolation", 12: "ProtocolOrderViolation", 13: "RangeOverflow",
    14: "MalformedPayload", 15: "TransportError", 100: "CudaError", 101: "Unsupported",
    102: "InvalidArgument",
}


class EnseiError(RuntimeError):
    """Mirror of ensei::Error; .kind names the reference subclass (errors.hpp:7-37)."""

    def __init__(self, code: int, msg: str):
        self.code = code
        self.kind = STATUS_NAMES.get(code, "Error")
        super().__init__(f"[{self.kind}] {msg}")


class CtxInfo(C.Structure):
    _fields_ = [
        ("n", C.c_uint32), ("num_q", C.c_uint32),
        ("q", C.c_uint64 * ENSEI_MAX_PRIMES), ("p", C.c_uint64),
        ("delta", C.c_uint64 * ENSEI_MAX_PRIMES), ("psi_q", C.c_uint64 * ENSEI_MAX_PRIMES),
        ("psi_p", C.c_uint64), ("device", C.c_int), ("sm_count", C.c_int),
    ]


class ConvDesc(C.Structure):
    _fields_ = [("H", C.c_uint32), ("W", C.c_uint32), ("fh", C.c_uint32), ("fw", C.c_uint32),
                ("same", C.c_uint32), ("cin", C.c_uint32), ("cout", C.c_uint32), ("pack", C.c_uint32),
                ("grid", C.c_uint32)]


class LayerGeom(C.Structure):
    _fields_ = [("Lh", C.c_uint32), ("Lw", C.c_uint32), ("blocks", C.c_uint32), ("oh", C.c_uint32),
                ("ow", C.c_uint32), ("r0", C.c_uint32), ("c0", C.c_uint32), ("pack", C.c_uint32)]


class Randomness(C.Structure):
    _fields_ = [("mode", C.c_uint32), ("layer", C.c_uint32), ("image_base", C.c_uint32),
                ("cbd_k", C.c_uint32), ("alice_key", C.c_uint64), ("bob_key", C.c_uint64),
                ("d_noise", C.c_void_p), ("d_a_hat", C.c_void_p), ("d_share", C.c_void_p)]


class PrecisionProfile(C.Structure):
    _fields_ = [("input_bits", C.c_int32), ("filter_bits", C.c_int32), ("f_h", C.c_int32), ("f_w", C.c_int32)]


class ParamSet(C.Structure):
    _fields_ = [("p_n", C.c_uint64), ("p_a", C.c_uint64), ("p_e", C.c_uint64), ("n", C.c_uint32),
                ("num_q", C.c_uint32), ("q", C.c_uint64 * ENSEI_MAX_PRIMES), ("sigma", C.c_double),
                ("log2_q_min", C.c_double), ("mode", C.c_uint32), ("insecure", C.c_uint32),
                ("profile", PrecisionProfile)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(SO_PATH):
            raise RuntimeError(f"{SO_PATH} is missing: run __graft_entry__.build() "
                               "(python -m paper_2003_05328_b200.build); there is no CPU fallback")
        L = C.CDLL(SO_PATH)
        vp, sz, u32, u64, i32 = C.c_void_p, C.c_size_t, C.c_uint32, C.c_uint64, C.c_int
        sig = {
            "ensei_gpu_last_error": (C.c_char_p, []),
            "ensei_gpu_abi_version": (i32, []),
            "ensei_gpu_ctx_create": (i32, [i32, u32, C.POINTER(u64), u32, u64, C.POINTER(vp)]),
            "ensei_gpu_ctx_destroy": (None, [vp]),
            "ensei_gpu_ctx_query": (i32, [vp, C.POINTER(CtxInfo)]),
            "ensei_gpu_negacyclic": (i32, [vp, u32, i32, i32, vp, sz, vp]),
            "ensei_gpu_ntt2d": (i32, [vp, i32, u32, u32, vp, sz, vp]),
            "ensei_gpu_permute": (i32, [vp, i32, vp, sz, vp]),
            "ensei_gpu_layer_geometry": (i32, [vp, C.POINTER(ConvDesc), C.POINTER(LayerGeom)]),
            "ensei_gpu_secret_from_coeffs": (i32, [vp, vp, vp, vp]),
            "ensei_gpu_secret_sample": (i32, [vp, u64, vp, vp, vp]),
            "ensei_gpu_prepare_weights": (i32, [vp, C.POINTER(ConvDesc), vp, vp, vp]),
            "ensei_gpu_prepared_weights_bytes": (sz, [vp, C.POINTER(ConvDesc)]),
            "ensei_gpu_prepare_weight_planes": (i32, [vp, C.POINTER(ConvDesc), vp, vp]),
            "ensei_gpu_alice_encrypt": (i32, [vp, C.POINTER(ConvDesc), vp, u32, vp, i32, u32,
                                              C.POINTER(Randomness), vp, vp]),
            "ensei_gpu_bob_eval": (i32, [vp, C.POINTER(ConvDesc), vp, vp, vp, u32, C.POINTER(Randomness),
                                         vp, vp, vp]),
            "ensei_gpu_bob_share": (i32, [vp, C.POINTER(ConvDesc), u32, C.POINTER(Randomness), vp, vp, vp]),
            "ensei_gpu_bob_mac": (i32, [vp, C.POINTER(ConvDesc), vp, vp, u32, vp, vp]),
            "ensei_gpu_alice_decrypt": (i32, [vp, C.POINTER(ConvDesc), vp, u32, vp, u32, vp, vp]),
            "ensei_gpu_activation": (i32, [vp, i32, i32, u32, u32, u32, u32, vp, vp, C.POINTER(Randomness),
                                           vp, vp, vp, vp]),
            "ensei_gpu_recombine": (i32, [vp, vp, vp, sz, vp, vp]),
            "ensei_gpu_crt_round": (i32, [vp, vp, sz, vp, vp]),
            "ensei_gpu_ops_workspace_bytes": (sz, [vp, sz]),
            "ensei_gpu_encrypt_freq_direct": (i32, [vp, vp, vp, vp, vp, sz, vp, vp, vp]),
            "ensei_gpu_decrypt": (i32, [vp, vp, vp, sz, vp, vp, vp]),
            "ensei_gpu_prepare_plain": (i32, [vp, vp, sz, vp, vp, vp, vp]),
            "ensei_gpu_mul_plain": (i32, [vp, vp, vp, sz, i32, vp, vp]),
            "ensei_gpu_add_ct": (i32, [vp, vp, vp, sz, vp, vp]),
            "ensei_gpu_add_plain": (i32, [vp, vp, vp, i32, sz, vp, vp]),
            "ensei_gpu_set_mac_variant": (i32, [i32]),
            "ensei_gpu_set_tile_variant": (i32, [i32]),
            "ensei_gpu_mac_path": (i32, [vp, C.POINTER(ConvDesc), u32, C.POINTER(i32)]),
            "ensei_gpu_conv_workspace_bytes": (sz, [vp, C.POINTER(ConvDesc), u32]),
            "ensei_gpu_conv_chunk_images": (u32, [vp, C.POINTER(ConvDesc), u32]),
            "ensei_gpu_conv_layer": (i32, [vp, C.POINTER(ConvDesc), vp, u32, vp, vp, i32, vp, u32,
                                           C.POINTER(Randomness), vp, vp, vp, vp, vp]),
            "ensei_gpu_conv_host_workspace_bytes": (sz, [vp, C.POINTER(ConvDesc), u32, i32]),
            "ensei_gpu_conv_layer_host": (i32, [vp, C.POINTER(ConvDesc), vp, vp, vp, i32, u32,
                                                C.POINTER(Randomness), vp, vp, vp]),
            "ensei_gpu_wire_ct_frame_bytes": (sz, [u32, u32, u32]),
            "ensei_gpu_wire_share_frame_bytes": (sz, [u32, u32, u32]),
            "ensei_gpu_wire_encode_ct_blocks": (i32, [vp, u32, u32, u32, u32, u32, vp, u32, vp, sz, vp]),
            "ensei_gpu_wire_decode_ct_blocks": (i32, [vp, vp, sz, sz, u32, u32, u32, u32, vp, vp, vp, vp]),
            "ensei_gpu_wire_encode_shares": (i32, [vp, u32, u32, u32, u32, u32, vp, u32, vp, sz, vp]),
            "ensei_gpu_wire_decode_shares": (i32, [vp, vp, sz, sz, u32, u32, u32, u32, u32, u64, vp, vp, vp]),
            "ensei_gpu_fnv1a": (u64, [vp, sz, u64]),
            "ensei_gpu_ref_rng_create": (i32, [u64, i32, u64, C.POINTER(vp)]),
            "ensei_gpu_ref_rng_destroy": (None, [vp]),
            "ensei_gpu_ref_rng_next_u64": (i32, [vp, vp, sz]),
            "ensei_gpu_ref_rng_uniform_below": (i32, [vp, u64, vp, sz]),
            "ensei_gpu_ref_rng_gaussian": (i32, [vp, C.c_double, vp, sz]),
            "ensei_gpu_min_pntt": (i32, [C.POINTER(PrecisionProfile), C.POINTER(u64)]),
            "ensei_gpu_build_params": (i32, [C.POINTER(PrecisionProfile), u32, u32, u64, u64, C.c_double, u32, u32,
                                             C.POINTER(ParamSet)]),
            "ensei_gpu_preset_params": (i32, [C.c_char_p, u64, u32, C.POINTER(ParamSet)]),
            "ensei_gpu_launch_count": (u64, []),
            "ensei_gpu_profile": (i32, [i32]),
            "ensei_gpu_profile_read": (i32, [u32, vp, vp, vp, C.POINTER(u32)]),
            "ensei_gpu_imad_peak": (C.c_double, [i32]),
            "ensei_gpu_tc_i8_peak": (C.c_double, [i32, u32]),
        }
        for name, (res, args) in sig.items():
            if not hasattr(L, name):  # reported by tests/test_capi.py::test_exports
                continue
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def profile(enable: bool) -> None:
    """Per-kernel event timing on/off (ensei_gpu_profile)."""
    check(lib().ensei_gpu_profile(int(enable)))


def profile_read(max_kernels: int = 64) -> dict:
    """{kernel name: (total ms, launches)} recorded since profile(True)."""
    import numpy as np
    names = C.create_string_buffer(32 * max_kernels)
    ms = np.zeros(max_kernels, np.float64)
    cnt = np.zeros(max_kernels, np.uint32)
    nk = C.c_uint32()
    check(lib().ensei_gpu_profile_read(max_kernels, names, ms.ctypes.data_as(C.c_void_p),
                                       cnt.ctypes.data_as(C.c_void_p), C.byref(nk)))
    out = {}
    for k in range(min(nk.value, max_kernels)):
        nm = names.raw[32 * k:32 * k + 32].split(b"\0", 1)[0].decode()
        out[nm] = (float(ms[k]), int(cnt[k]))
    return out


def exported_symbols():
    """Names the header declares (checked by the CPU test suite)."""
    import re
    hdr = os.path.join(os.path.dirname(HERE), "include", "ensei_gpu.h")
    text = open(hdr).read()
    return sorted(set(re.findall(r"\b(ensei_gpu_[a-z0-9_]+)\s*\(", text)))


def check(rc: int) -> None:
    if rc != 0:
        raise EnseiError(rc, lib().ensei_gpu_last_error().decode())
