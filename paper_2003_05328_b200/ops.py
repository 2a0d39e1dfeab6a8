"""Python mirror of the reference operator surface over the C ABI.

Names follow REF (ntt_2d / intt_2d, NegacyclicPlan.forward / inverse,
encode_slots / decode_slots, prepare_plain, encrypt_freq_direct, mul_plain,
hom_share, hom_rec, decrypt, run_inproc).  torch is used only for device memory
and streams; every operation runs in libensei_gpu.so kernels.
"""
from __future__ import annotations

import ctypes as C
import functools
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


@functools.lru_cache(maxsize=256)
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


# ------------------------------------------------------------------ conv layers

@dataclass
class ConvSpec:
    """One conv layer (REF LayerSpec + image dims, protocol.hpp:23-31)."""
    H: int
    W: int
    fh: int
    fw: int
    same: bool
    cin: int
    cout: int
    pack: int = 1  # images per ciphertext block (builder extension; 1 = REF geometry)
    grid: int = 0  # padded grid side (builder extension; 0 = REF's next power of two)

    def desc(self) -> ConvDesc:
        return ConvDesc(self.H, self.W, self.fh, self.fw, int(self.same), self.cin, self.cout, self.pack, self.grid)


def unpack_limbs(t: torch.Tensor) -> torch.Tensor:
    """Packed prepared-weight words -> canonical residues (device layout kept)."""
    s = t.view(torch.int64)  # values < 2^62: int64 shifts are exact
    return (((s >> 32) << 30) | (s & ((1 << 30) - 1))).view(torch.uint64)


class Randomness:
    """ensei_randomness: Philox streams keyed by party seeds, or injected draws."""

    def __init__(self, seed: int = 0, layer: int = 0, image_base: int = 0, cbd_k: int = 20,
                 noise=None, a_hat=None, share=None):
        self.seed, self.layer, self.image_base, self.cbd_k = seed, layer, image_base, cbd_k
        self.noise, self.a_hat, self.share = noise, a_hat, share

    def struct(self) -> Randomness_:
        # cached per field values: a hot host-entry loop re-passes the same randomness
        k = (self.seed, self.layer, self.image_base, self.cbd_k, _tid(self.noise), _tid(self.a_hat), _tid(self.share))
        if getattr(self, "_key", None) == k:
            return self._struct
        inj = self.noise is not None or self.a_hat is not None or self.share is not None
        r = Randomness_()
        r.mode = RAND_INJECTED if inj else RAND_PHILOX
        r.layer, r.image_base, r.cbd_k = self.layer, self.image_base, self.cbd_k
        r.alice_key = fork_seed(self.seed, SALT_ALICE)
        r.bob_key = fork_seed(self.seed, SALT_BOB)
        r.d_noise = None if self.noise is None else self.noise.data_ptr()
        r.d_a_hat = None if self.a_hat is None else self.a_hat.data_ptr()
        r.d_share = None if self.share is None else self.share.data_ptr()
        self._key, self._struct = k, r
        return r


def _tid(t):
    return None if t is None else (id(t), t.data_ptr())


Randomness_ = _lib.Randomness


class LayerOps:
    """Batched per-layer operations of the protocol over one Context."""

    def __init__(self, ctx: Context, spec: ConvSpec):
        self.ctx, self.spec = ctx, spec
        self.d = spec.desc()
        g = LayerGeom()
        check(lib().ensei_gpu_layer_geometry(ctx.h, C.byref(self.d), C.byref(g)))
        self.geom = g
        self.B = g.blocks
        self.pack = g.pack

    def cts(self, images: int) -> int:
        """Ciphertext images of a batch (pack images per ciphertext block)."""
        return -(-images // self.pack)

    def empty_ct(self, images: int, channels: int) -> torch.Tensor:
        n, R = self.ctx.n, self.ctx.R
        return torch.empty((self.cts(images), channels, self.B, 2, R, n), dtype=torch.uint64, device=self.ctx.device)

    def prepared_words(self) -> int:
        """uint64 words of a prepared-weights buffer (ABI 2: packed words + tcgen05 planes)."""
        return lib().ensei_gpu_prepared_weights_bytes(self.ctx.h, C.byref(self.d)) // 8

    def prepare_weights(self, w: torch.Tensor, stream=None) -> torch.Tensor:
        """w[cout][cin][fh][fw] int32 (device) -> the prepared-weights buffer (1-D uint64:
        the packed device-layout words [cout][cin][B][R][n], then the tcgen05 byte planes
        when the layer can use them); weight_words() views the first part."""
        s = self.spec
        assert w.dtype == torch.int32 and w.is_cuda and tuple(w.shape) == (s.cout, s.cin, s.fh, s.fw)
        out = torch.empty(self.prepared_words(), dtype=torch.uint64, device=w.device)
        check(lib().ensei_gpu_prepare_weights(self.ctx.h, C.byref(self.d), _ptr(w), _ptr(out), _stream(stream)))
        return out

    def weight_words(self, prepared: torch.Tensor) -> torch.Tensor:
        """The packed words [cout][cin][B][R][n] of a prepared-weights buffer (a view)."""
        s = self.spec
        k = s.cout * s.cin * self.B * self.ctx.R * self.ctx.n
        return prepared[:k].view(s.cout, s.cin, self.B, self.ctx.R, self.ctx.n)

    def weights_from_words(self, words: torch.Tensor, stream=None) -> torch.Tensor:
        """A prepared-weights buffer from caller-made packed words (planes rebuilt)."""
        out = torch.zeros(self.prepared_words(), dtype=torch.uint64, device=words.device)
        out[:words.numel()].copy_(words.reshape(-1))
        check(lib().ensei_gpu_prepare_weight_planes(self.ctx.h, C.byref(self.d), _ptr(out), _stream(stream)))
        return out

    def alice_encrypt(self, key, x: torch.Tensor, rand: Randomness, key_stride: int = 0, stream=None):
        images = x.shape[0]
        in_t = IN_U8 if x.dtype == torch.uint8 else IN_U32
        assert x.dtype in (torch.uint8, torch.int32, torch.uint32) and x.is_contiguous()
        ct = self.empty_ct(images, self.spec.cin)
        r = rand.struct()
        check(lib().ensei_gpu_alice_encrypt(self.ctx.h, C.byref(self.d), _ptr(key), key_stride, _ptr(x), in_t,
                                            images, C.byref(r), _ptr(ct), _stream(stream)))
        return ct

    def bob_eval(self, ct: torch.Tensor, w_eval: torch.Tensor, rand: Randomness, bob_prev=None, stream=None,
                 images=None):
        images = ct.shape[0] * self.pack if images is None else images
        g = self.geom
        ct_out = self.empty_ct(images, self.spec.cout)
        bob = torch.empty((images, self.spec.cout, g.oh, g.ow), dtype=torch.int32, device=ct.device)
        r = rand.struct()
        check(lib().ensei_gpu_bob_eval(self.ctx.h, C.byref(self.d), _ptr(ct), _ptr(w_eval), _ptr(bob_prev), images,
                                       C.byref(r), _ptr(ct_out), _ptr(bob), _stream(stream)))
        return ct_out, bob

    def bob_share(self, images: int, rand: Randomness, ct_out=None, bob=None, stream=None):
        g = self.geom
        ct_out = self.empty_ct(images, self.spec.cout) if ct_out is None else ct_out
        bob = torch.empty((images, self.spec.cout, g.oh, g.ow), dtype=torch.int32,
                          device=self.ctx.device) if bob is None else bob
        r = rand.struct()
        check(lib().ensei_gpu_bob_share(self.ctx.h, C.byref(self.d), images, C.byref(r), _ptr(ct_out), _ptr(bob),
                                        _stream(stream)))
        return ct_out, bob

    def bob_mac(self, ct, w_eval, ct_out, stream=None):
        check(lib().ensei_gpu_bob_mac(self.ctx.h, C.byref(self.d), _ptr(ct), _ptr(w_eval), ct.shape[0] * self.pack,
                                      _ptr(ct_out), _stream(stream)))
        return ct_out

    def alice_decrypt(self, key, ct_out: torch.Tensor, key_stride: int = 0, stream=None, images=None):
        images = ct_out.shape[0] * self.pack if images is None else images
        g = self.geom
        a = torch.empty((images, self.spec.cout, g.oh, g.ow), dtype=torch.int32, device=ct_out.device)
        check(lib().ensei_gpu_alice_decrypt(self.ctx.h, C.byref(self.d), _ptr(key), key_stride, _ptr(ct_out), images,
                                            _ptr(a), _stream(stream)))
        return a

    MAC_PATHS = {0: "imad4", 1: "karatsuba", 2: "int8_planes", 3: "int8_direct", 4: "direct", 5: "tcgen05"}

    def mac_path(self, images: int) -> str:
        """The ElementMult kernel a batch of `images` takes (ensei_gpu_mac_path)."""
        v = C.c_int()
        check(lib().ensei_gpu_mac_path(self.ctx.h, C.byref(self.d), images, C.byref(v)))
        return self.MAC_PATHS.get(v.value, str(v.value))

    def workspace(self, images: int, host: bool = False, in_dtype: int = IN_U8) -> torch.Tensor:
        if host:
            nb = lib().ensei_gpu_conv_host_workspace_bytes(self.ctx.h, C.byref(self.d), images, in_dtype)
        else:
            nb = lib().ensei_gpu_conv_workspace_bytes(self.ctx.h, C.byref(self.d), images)
        return torch.empty(nb, dtype=torch.uint8, device=self.ctx.device)

    def chunk_images(self, images: int) -> int:
        """Images per sub-batch of the layer entry points (the workspace holds that many)."""
        return int(lib().ensei_gpu_conv_chunk_images(self.ctx.h, C.byref(self.d), images))

    def forward(self, key, w_eval, x: torch.Tensor, rand: Randomness, ws=None, bob_prev=None, key_stride: int = 0,
                want_shares: bool = False, stream=None, out=None, alice=None, bob=None):
        """The whole oblivious conv layer for a batch; returns the reconstructed output
        (and the two shares when want_shares; `alice` / `bob` may be given buffers)."""
        images = x.shape[0]
        g = self.geom
        in_t = IN_U8 if x.dtype == torch.uint8 else IN_U32
        ws = self.workspace(images) if ws is None else ws
        shape = (images, self.spec.cout, g.oh, g.ow)
        out = torch.empty(shape, dtype=torch.int32, device=x.device) if out is None else out
        a = (torch.empty(shape, dtype=torch.int32, device=x.device) if alice is None else alice) if want_shares else None
        b = (torch.empty(shape, dtype=torch.int32, device=x.device) if bob is None else bob) if want_shares else None
        r = rand.struct()
        check(lib().ensei_gpu_conv_layer(self.ctx.h, C.byref(self.d), _ptr(key), key_stride, _ptr(w_eval), _ptr(x),
                                         in_t, _ptr(bob_prev), images, C.byref(r), _ptr(ws), _ptr(a), _ptr(b),
                                         _ptr(out), _stream(stream)))
        return (out, a, b) if want_shares else out

    def host_call(self, key, w_eval, h_x: torch.Tensor, rand: Randomness, ws, h_out: torch.Tensor, stream=None):
        """A prepared host-buffer layer call: every argument marshalled once; calling the
        returned function runs the layer (H2D, Enc, Bob, Dec, D2H, synchronous) again on
        the same buffers -- the serving loop's form of forward_host."""
        r = rand.struct()
        st = (stream if stream is not None else torch.cuda.current_stream()).cuda_stream
        in_t = IN_U8 if h_x.dtype == torch.uint8 else IN_U32
        args = (self.ctx.h, C.byref(self.d), _ptr(key), _ptr(w_eval), C.c_void_p(h_x.data_ptr()), in_t, h_x.shape[0],
                C.byref(r), _ptr(ws), C.c_void_p(h_out.data_ptr()), C.c_void_p(st))
        fn = lib().ensei_gpu_conv_layer_host
        keep = (key, w_eval, h_x, rand, r, ws, h_out)  # buffers stay alive with the call

        def call():
            rc = fn(*args)
            if rc:
                check(rc)
            return keep[6]
        return call

    def forward_host(self, key, w_eval, h_x: torch.Tensor, rand: Randomness, ws, h_out: torch.Tensor, stream=None):
        """Host-buffer entry point (pinned h_x / h_out): H2D, layer, D2H, synchronous.
        The marshalled ctypes arguments are cached while the buffers are unchanged."""
        r = rand.struct()
        st = (stream if stream is not None else torch.cuda.current_stream()).cuda_stream
        k = (key.data_ptr(), w_eval.data_ptr(), h_x.data_ptr(), h_x.dtype, h_x.shape[0], id(r), ws.data_ptr(),
             h_out.data_ptr(), st)
        if getattr(self, "_host_key", None) != k:
            in_t = IN_U8 if h_x.dtype == torch.uint8 else IN_U32
            self._host_args = (self.ctx.h, C.byref(self.d), _ptr(key), _ptr(w_eval), C.c_void_p(h_x.data_ptr()),
                               in_t, h_x.shape[0], C.byref(r), _ptr(ws), C.c_void_p(h_out.data_ptr()),
                               C.c_void_p(st))
            self._host_key = k
        check(lib().ensei_gpu_conv_layer_host(*self._host_args))
        return h_out


def key_words(ctx: Context) -> int:
    return 2 * ctx.R * ctx.n


def secret_from_coeffs(ctx: Context, t: torch.Tensor, stream=None) -> torch.Tensor:
    """keygen evaluation form (REF ringbfv.cpp:95-107) from signed coefficients t[n] (int64, device)."""
    key = torch.empty(key_words(ctx), dtype=torch.uint64, device=ctx.device)
    check(lib().ensei_gpu_secret_from_coeffs(ctx.h, _ptr(t), _ptr(key), _stream(stream)))
    return key


def secret_sample(ctx: Context, seed: int, stream=None):
    """Ternary secret from Alice's Philox stream; returns (t, key blob)."""
    key = torch.empty(key_words(ctx), dtype=torch.uint64, device=ctx.device)
    t = torch.empty(ctx.n, dtype=torch.int64, device=ctx.device)
    check(lib().ensei_gpu_secret_sample(ctx.h, fork_seed(seed, SALT_ALICE), _ptr(t), _ptr(key), _stream(stream)))
    return t, key
