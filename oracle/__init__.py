"""CPU ORACLE -- test infrastructure only.

Python (ctypes + numpy) access to the two checkers built by ``oracle/Makefile``:

* ``C``   -- ``oracle/build/libensei_oracle.so``, the plain-C restatement of the
  reference hot path (``oracle/ensei_oracle.c``; every function cites the
  reference file:line it restates);
* ``REF`` -- ``oracle/_ref/libensei_ref.so``, the unmodified reference sources
  compiled with our extern "C" harness (``oracle/ref_harness.cpp``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
import this package.  The product path (``paper_2003_05328_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "build", "libensei_oracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libensei_ref.so")

u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
u32p = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")

_c = None
_ref = None


def build() -> None:
    """Builds both checkers (make; the reference half only where /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE, "-j8"], check=True)


class Layer(C.Structure):
    _fields_ = [
        ("q", C.c_uint64), ("p", C.c_uint64), ("n", C.c_uint32),
        ("H", C.c_uint32), ("W", C.c_uint32), ("fh", C.c_uint32), ("fw", C.c_uint32),
        ("same", C.c_uint32), ("cin", C.c_uint32), ("cout", C.c_uint32),
        ("Lh", C.c_uint32), ("Lw", C.c_uint32), ("blocks", C.c_uint32),
        ("oh", C.c_uint32), ("ow", C.c_uint32), ("r0", C.c_uint32), ("c0", C.c_uint32),
        ("delta", C.c_uint64), ("pack", C.c_uint32),
    ]


class MT(C.Structure):
    _fields_ = [("mt", C.c_uint64 * 312), ("idx", C.c_uint32), ("seed", C.c_uint64)]


def lib():
    """The C restatement (built on demand)."""
    global _c
    if _c is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        U64, U32, I64 = C.c_uint64, C.c_uint32, C.c_int64
        sig = {
            "eo_mulmod": (U64, [U64, U64, U64]),
            "eo_powmod": (U64, [U64, U64, U64]),
            "eo_invmod": (U64, [U64, U64]),
            "eo_is_prime": (C.c_int, [U64]),
            "eo_primitive_root": (U64, [U64]),
            "eo_root_of_unity": (U64, [U64, U64]),
            "eo_find_prime": (U64, [U64, U64, U64]),
            "eo_encode_signed": (U64, [I64, U64]),
            "eo_decode_signed": (I64, [U64, U64]),
            "eo_ntt_1d": (C.c_int, [u64p, C.c_size_t, U64, U64, C.c_int]),
            "eo_ntt_2d": (C.c_int, [u64p, C.c_size_t, C.c_size_t, U64, C.c_int]),
            "eo_negacyclic": (C.c_int, [u64p, U32, U64, C.c_int, C.c_size_t]),
            "eo_philox4x32_10": (None, [u32p, u32p, u32p]),
            "eo_mix64": (U64, [U64]),
            "eo_fork_seed": (U64, [U64, U64]),
            "eo_stream_id": (U64, [U32, U32, U32, U32, U32]),
            "eo_rand_ternary": (None, [U64, U64, U32, i64p]),
            "eo_rand_cbd": (None, [U64, U64, U32, U32, i64p]),
            "eo_rand_uniform_q": (None, [U64, U64, U32, U64, u64p]),
            "eo_rand_uniform_p": (None, [U64, U64, U32, U64, u64p]),
            "eo_mt_seed": (None, [C.POINTER(MT), U64]),
            "eo_mt_next": (U64, [C.POINTER(MT)]),
            "eo_mt_fork": (None, [C.POINTER(MT), U64, C.POINTER(MT)]),
            "eo_mt_uniform_below": (U64, [C.POINTER(MT), U64]),
            "eo_mt_gaussian": (I64, [C.POINTER(MT), C.c_double]),
            "eo_layer_init": (C.c_int, [C.POINTER(Layer), U64, U64, U32, U32, U32, U32, U32, U32, U32, U32]),
            "eo_secret_eval": (None, [C.POINTER(Layer), i64p, u64p]),
            "eo_prepare_weights": (None, [C.POINTER(Layer), i64p, u64p]),
            "eo_alice_encrypt": (None, [C.POINTER(Layer), u64p, u64p, i64p, u64p, u64p]),
            "eo_bob_eval": (None, [C.POINTER(Layer), u64p, u64p, C.c_void_p, u64p, u64p, u64p]),
            "eo_alice_decrypt": (None, [C.POINTER(Layer), u64p, u64p, u64p]),
            "eo_conv_direct": (None, [C.POINTER(Layer), u64p, i64p, u64p]),
            "eo_activation": (C.c_int, [u64p, C.c_size_t, U64, C.c_int]),
            "eo_crt_round": (U64, [u64p, u64p, U32, U64]),
            "eo_alice_decrypt_rns": (None, [C.c_void_p, U32, u64p, u64p, u64p]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _c = L
    return _c


def ref_available() -> bool:
    return os.path.exists(REF_PATH)


def ref():
    """The compiled reference + harness (prebuilt .so; travels to the GPU box)."""
    global _ref
    if _ref is None:
        if not os.path.exists(REF_PATH):
            build()
        R = C.CDLL(REF_PATH)
        U64, U32 = C.c_uint64, C.c_uint32
        vp = C.c_void_p
        sig = {
            "ref_last_error": (C.c_char_p, []),
            "ref_field_info": (C.c_int, [U64, C.POINTER(U64), C.POINTER(C.c_int32)]),
            "ref_mulmod": (U64, [U64, U64, U64]),
            "ref_find_prime": (U64, [U64, U64, U64]),
            "ref_root_of_unity": (U64, [U64, U64]),
            "ref_negacyclic": (C.c_int, [U64, U32, u64p, C.c_size_t, C.c_int]),
            "ref_plan_psi": (C.c_int, [U64, U32, C.POINTER(U64)]),
            "ref_ntt2d": (C.c_int, [U64, U32, U32, u64p, C.c_size_t, C.c_int]),
            "ref_ntt1d": (C.c_int, [U64, U64, u64p, C.c_size_t, C.c_int]),
            "ref_conv_oracle": (C.c_int, [U64, i64p, U32, U32, i64p, U32, U32, C.c_int, u64p]),
            "ref_geometry": (C.c_int, [U64, U32, U32, U32, U32, C.c_int, C.POINTER(U32), C.POINTER(U32)]),
            "ref_slots": (C.c_int, [U64, U64, U32, u64p, C.c_int]),
            "ref_rng_draw": (C.c_int, [U64, U64, C.c_int, C.c_int, U64, C.c_double, C.c_size_t, i64p]),
            "ref_session_key": (C.c_int, [U64, U64, U32, C.c_double, U64, i64p, u64p]),
            "ref_encrypt_freq_direct": (C.c_int, [U64, U64, U32, C.c_double, u64p, u64p, U64, u64p]),
            "ref_decrypt": (C.c_int, [U64, U64, U32, u64p, u64p, u64p]),
            "ref_prepare_plain": (C.c_int, [U64, U64, U32, u64p, u64p, C.POINTER(C.c_double)]),
            "ref_run_protocol": (C.c_int, [U64, U64, U32, C.c_double, C.c_int, U64, U32, U32, U32,
                                           i32p, i64p, i64p, u64p, vp, vp, U32, vp, vp, vp, vp]),
            "ref_reference_pipeline": (C.c_int, [U64, U64, U32, U32, U32, U32, i32p, i64p, i64p, u64p]),
            "ref_bench_protocol": (C.c_double, [U64, U64, U32, C.c_double, U64, U32, U32, U32, i32p,
                                                i64p, i64p, U32, U32, C.POINTER(C.c_double)]),
            "ref_bench_negacyclic": (C.c_double, [U64, U32, u64p, C.c_size_t, U32]),
            "ref_bench_layer_ops": (C.c_double, [U64, U64, U32, C.c_double, U64, U32, U32, U32, U32, C.c_int, U32,
                                                 U32, i64p, i64p, U32, U32, C.POINTER(C.c_double),
                                                 C.POINTER(C.c_double)]),
            "ref_wire_ct_frame": (C.c_int, [U32, U32, U32, U32, U32, C.c_int, u64p, vp, C.c_size_t,
                                            C.POINTER(C.c_size_t)]),
            "ref_wire_ct_decode": (C.c_int, [vp, C.c_size_t, U32, U64, U64, U32, U32, U32, C.POINTER(U32), u64p,
                                             vp]),
            "ref_wire_share_frame": (C.c_int, [U32, U32, U32, U32, U32, u64p, vp, C.c_size_t,
                                               C.POINTER(C.c_size_t)]),
            "ref_wire_share_decode": (C.c_int, [vp, C.c_size_t, U32, U32, U32, U32, U64, C.POINTER(U32), u64p]),
            "ref_min_pntt": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(U64)]),
            "ref_build_params": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, U32, C.c_int, U64, U64, C.c_double,
                                           u64p]),
            "ref_preset_params": (C.c_int, [C.c_char_p, U64, u64p]),
            "ref_random_weights": (C.c_int, [U32, i32p, C.c_int64, U64, C.c_int, U64, i64p]),
            "ref_config_digest": (U64, [U64, U64, U32, C.c_double, C.c_int, U64, U32, U32, U32, i32p]),
        }
        for name, (res, args) in sig.items():
            f = getattr(R, name)
            f.restype = res
            f.argtypes = args
        _ref = R
    return _ref


def ref_check(rc: int) -> None:
    if rc != 0:
        raise RuntimeError("reference raised: " + ref().ref_last_error().decode())


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# ----------------------------------------------------------------- helpers

def layer(q, p, n, H, W, fh, fw, same, cin, cout) -> Layer:
    L = Layer()
    rc = lib().eo_layer_init(C.byref(L), q, p, n, H, W, fh, fw, same, cin, cout)
    if rc != 0:
        raise ValueError(f"eo_layer_init failed ({rc})")
    return L


def negacyclic(x: np.ndarray, q: int, inverse: bool = False) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.uint64).copy()
    n = x.shape[-1]
    rc = lib().eo_negacyclic(x.reshape(-1), n, q, int(inverse), x.size // n)
    assert rc == 0
    return x


def ntt2d(x: np.ndarray, p: int, inverse: bool = False) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.uint64).copy()
    rows, cols = x.shape[-2:]
    flat = x.reshape(-1, rows * cols)
    for t in flat:
        t2 = np.ascontiguousarray(t)
        assert lib().eo_ntt_2d(t2, rows, cols, p, int(inverse)) == 0
        t[:] = t2
    return flat.reshape(x.shape)


def rand_ternary(key, stream, n):
    out = np.empty(n, np.int64)
    lib().eo_rand_ternary(key, stream, n, out)
    return out


def rand_cbd(key, stream, n, k=20):
    out = np.empty(n, np.int64)
    lib().eo_rand_cbd(key, stream, n, k, out)
    return out


def rand_uniform_q(key, stream, n, q):
    out = np.empty(n, np.uint64)
    lib().eo_rand_uniform_q(key, stream, n, q, out)
    return out


def rand_uniform_p(key, stream, n, p):
    out = np.empty(n, np.uint64)
    lib().eo_rand_uniform_p(key, stream, n, p, out)
    return out


def stream_id(purpose, layer_idx, image, channel, block):
    return lib().eo_stream_id(purpose, layer_idx, image, channel, block)


PURPOSE_SECRET, PURPOSE_NOISE, PURPOSE_AHAT, PURPOSE_SHARE, PURPOSE_RESHARE = 1, 2, 3, 4, 5
SALT_ALICE, SALT_BOB = 0xA11CE, 0xB0B


class MTRng:
    """The reference Rng (mt19937_64 + samplers) restated in C."""

    def __init__(self, seed: int, salt: int | None = None):
        self.s = MT()
        lib().eo_mt_seed(C.byref(self.s), seed)
        if salt is not None:
            child = MT()
            lib().eo_mt_fork(C.byref(self.s), salt, C.byref(child))
            self.s = child

    def next_u64(self):
        return lib().eo_mt_next(C.byref(self.s))

    def uniform_below(self, bound):
        return lib().eo_mt_uniform_below(C.byref(self.s), bound)

    def gaussian(self, sigma):
        return lib().eo_mt_gaussian(C.byref(self.s), sigma)
