"""CPU ORACLE protocol driver -- test infrastructure only.

Runs a schedule of conv / activation layers for one image through the C
restatement (oracle/ensei_oracle.c), mirroring AliceSession/BobSession
(REF protocol.cpp:276-640) on one thread: Alice Enc -> Bob HomRec/ElementMult/
HomShare -> Alice Dec, activations via trusted_activation semantics
(REF protocol.cpp:237-268).

Randomness comes from one of two providers that hand out per-polynomial arrays:

* ``RefRandomness``    -- the reference's own mt19937_64 streams in the exact
  consumption order of a reference session (Alice = Rng(seed).fork(0xA11CE):
  keygen n Gaussians, then per conv layer per [channel][block] n Gaussians + n
  uniform mod q, then per activation layer per element 1 uniform mod p;
  Bob = Rng(seed).fork(0xB0B): per conv layer per [out][block] n uniform mod p).
  Ciphertexts produced with it are bit-identical to the reference's wire frames.
* ``PhiloxRandomness`` -- the counter-based streams the GPU kernels generate
  (keyed by party seed; counter = (index, 0, stream id)); ternary secret,
  CBD(k=20) noise (builder extension: no reference counterpart).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import (Layer, MTRng, PURPOSE_AHAT, PURPOSE_NOISE, PURPOSE_RESHARE, PURPOSE_SECRET,
               PURPOSE_SHARE, SALT_ALICE, SALT_BOB, layer, lib, rand_cbd, rand_ternary,
               rand_uniform_p, rand_uniform_q, stream_id)


@dataclass
class Conv:
    fh: int
    fw: int
    same: bool
    cin: int
    cout: int


@dataclass
class Act:
    fn: int  # 0 ReLU, 1 Square, 2 Identity
    pool2: bool = False  # builder-defined 2x2 max-pool on centered lifts (config 3)


def desc_rows(schedule):
    """ref_harness layer descriptors: {kind, fh, fw, same, cin, cout, fn}."""
    rows = []
    for s in schedule:
        if isinstance(s, Conv):
            rows.append([0, s.fh, s.fw, int(s.same), s.cin, s.cout, 0])
        else:
            rows.append([1, 0, 0, 0, 0, 0, s.fn])
    return rows


class RefRandomness:
    """Reference Rng streams (one session per image, seed = base + image)."""

    def __init__(self, seed: int, n: int, q: int, p: int, sigma: float = 4.0):
        self.alice = MTRng(seed, SALT_ALICE)
        self.bob = MTRng(seed, SALT_BOB)
        self.n, self.q, self.p, self.sigma = n, q, p, sigma

    def secret(self):
        return np.array([self.alice.gaussian(self.sigma) for _ in range(self.n)], np.int64)

    def enc(self, layer_idx, cin, blocks):
        e = np.empty((cin, blocks, self.n), np.int64)
        a = np.empty((cin, blocks, self.n), np.uint64)
        for c in range(cin):
            for b in range(blocks):
                e[c, b] = [self.alice.gaussian(self.sigma) for _ in range(self.n)]
                a[c, b] = [self.alice.uniform_below(self.q) for _ in range(self.n)]
        return e, a

    def share(self, layer_idx, cout, blocks):
        s = np.empty((cout, blocks, self.n), np.uint64)
        for o in range(cout):
            for b in range(blocks):
                s[o, b] = [self.bob.uniform_below(self.p) for _ in range(self.n)]
        return s

    def reshare(self, layer_idx, ch, count):
        return np.array([[self.alice.uniform_below(self.p) for _ in range(count)]
                         for _ in range(ch)], np.uint64)


class PhiloxRandomness:
    """Counter-based streams (what the device kernels draw in throughput mode)."""

    def __init__(self, seed: int, image: int, n: int, q: int, p: int, cbd_k: int = 20):
        self.ka = lib().eo_fork_seed(seed, SALT_ALICE)
        self.kb = lib().eo_fork_seed(seed, SALT_BOB)
        self.image, self.n, self.q, self.p, self.k = image, n, q, p, cbd_k

    def secret(self):
        return rand_ternary(self.ka, stream_id(PURPOSE_SECRET, 0, 0, 0, 0), self.n)

    def enc(self, layer_idx, cin, blocks):
        e = np.empty((cin, blocks, self.n), np.int64)
        a = np.empty((cin, blocks, self.n), np.uint64)
        for c in range(cin):
            for b in range(blocks):
                e[c, b] = rand_cbd(self.ka, stream_id(PURPOSE_NOISE, layer_idx, self.image, c, b), self.n, self.k)
                a[c, b] = rand_uniform_q(self.ka, stream_id(PURPOSE_AHAT, layer_idx, self.image, c, b), self.n, self.q)
        return e, a

    def share(self, layer_idx, cout, blocks):
        s = np.empty((cout, blocks, self.n), np.uint64)
        for o in range(cout):
            for b in range(blocks):
                s[o, b] = rand_uniform_p(self.kb, stream_id(PURPOSE_SHARE, layer_idx, self.image, o, b), self.n, self.p)
        return s

    def reshare(self, layer_idx, ch, count):
        return np.stack([rand_uniform_p(self.ka, stream_id(PURPOSE_RESHARE, layer_idx, self.image, c, 0), count, self.p)
                         for c in range(ch)])


def default_workers() -> int:
    """Host threads for the parallel oracle drivers (ctypes releases the GIL, so the
    C restatement runs concurrently on disjoint output channels)."""
    import os
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except Exception:
        return os.cpu_count() or 1


def _pmap(fn, items, workers):
    items = list(items)
    if workers <= 1 or len(items) <= 1:
        return [fn(x) for x in items]
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(min(workers, len(items))) as ex:
        return list(ex.map(fn, items))


def _ranges(total, workers):
    """Contiguous [lo, hi) ranges covering `total` (about 3 per worker for balance)."""
    parts = max(1, min(total, 3 * workers))
    step = (total + parts - 1) // parts
    return [(lo, min(total, lo + step)) for lo in range(0, total, step)]


def _sub(L, cout):
    """The same layer restricted to `cout` output channels (every oracle per-layer call
    indexes its outputs by o, so a contiguous output-channel slice is a smaller layer)."""
    S = Layer.from_buffer_copy(L)
    S.cout = cout
    return S


def secret_eval(L, t):
    te = np.zeros(L.n, np.uint64)
    lib().eo_secret_eval(C.byref(L), np.ascontiguousarray(t, np.int64), te)
    return te


def prepare_weights(L, w, workers=1):
    """prepare_plain for a layer's filter bank; `workers` host threads over output-channel
    slices (identical results)."""
    out = np.zeros((L.cout, L.cin, L.blocks, L.n), np.uint64)
    w = np.ascontiguousarray(w, np.int64).reshape(L.cout, -1)

    def job(r):
        o0, o1 = r
        sub = np.zeros((o1 - o0) * L.cin * L.blocks * L.n, np.uint64)
        lib().eo_prepare_weights(C.byref(_sub(L, o1 - o0)), np.ascontiguousarray(w[o0:o1]).reshape(-1), sub)
        out[o0:o1] = sub.reshape(o1 - o0, L.cin, L.blocks, L.n)
    _pmap(job, _ranges(L.cout, workers), workers)
    return out


def _pk(L):
    return max(1, int(L.pack))


def bob_eval(L, ct, w_eval, bob_prev, s_b, workers=1):
    """BobSession conv step (HomRec, ElementMult + channel sum, HomShare, Bob's share IDFT2D)
    for one image (one ciphertext image of L.pack images when packed), over output-channel
    slices on `workers` threads.  Bob's shares: [pack][cout][oh * ow] flattened."""
    n, B, pk = L.n, L.blocks, _pk(L)
    ct_out = np.zeros((L.cout, B * 2 * n), np.uint64)
    bob_sh = np.zeros((pk, L.cout, L.oh * L.ow), np.uint64)
    w_eval = np.ascontiguousarray(w_eval, np.uint64).reshape(L.cout, -1)
    s_b = np.ascontiguousarray(s_b, np.uint64).reshape(L.cout, -1)
    prev = None if bob_prev is None else np.ascontiguousarray(bob_prev, np.uint64).reshape(-1)

    def job(r):
        o0, o1 = r
        co = np.zeros((o1 - o0) * B * 2 * n, np.uint64)
        bs = np.zeros(pk * (o1 - o0) * L.oh * L.ow, np.uint64)
        lib().eo_bob_eval(C.byref(_sub(L, o1 - o0)), ct, np.ascontiguousarray(w_eval[o0:o1]).reshape(-1),
                          None if prev is None else prev.ctypes.data_as(C.c_void_p),
                          np.ascontiguousarray(s_b[o0:o1]).reshape(-1), co, bs)
        ct_out[o0:o1] = co.reshape(o1 - o0, -1)
        bob_sh[:, o0:o1] = bs.reshape(pk, o1 - o0, -1)
    _pmap(job, _ranges(L.cout, workers), workers)
    return ct_out.reshape(-1), bob_sh.reshape(-1)


def alice_decrypt(L, t_eval, ct_out, workers=1):
    n, B, pk = L.n, L.blocks, _pk(L)
    ct_out = np.ascontiguousarray(ct_out, np.uint64).reshape(L.cout, -1)
    al = np.zeros((pk, L.cout, L.oh * L.ow), np.uint64)

    def job(r):
        o0, o1 = r
        a_ = np.zeros(pk * (o1 - o0) * L.oh * L.ow, np.uint64)
        lib().eo_alice_decrypt(C.byref(_sub(L, o1 - o0)), t_eval, np.ascontiguousarray(ct_out[o0:o1]).reshape(-1), a_)
        al[:, o0:o1] = a_.reshape(pk, o1 - o0, -1)
    _pmap(job, _ranges(L.cout, workers), workers)
    return al.reshape(-1)


def run_layer(L, t_eval, alice_in, bob_prev, w_eval, e, a, s_b, want=(), workers=1):
    """One conv layer for one image. Returns dict with alice/bob shares (+ cts)."""
    lb = lib()
    n, B = L.n, L.blocks
    ct = np.zeros(L.cin * B * 2 * n, np.uint64)
    lb.eo_alice_encrypt(C.byref(L), t_eval, np.ascontiguousarray(alice_in, np.uint64).reshape(-1),
                        np.ascontiguousarray(e, np.int64).reshape(-1),
                        np.ascontiguousarray(a, np.uint64).reshape(-1), ct)
    ct_out, bob_sh = bob_eval(L, ct, w_eval, bob_prev, s_b, workers)
    al_sh = alice_decrypt(L, t_eval, ct_out, workers)
    if _pk(L) > 1:  # packed: [pack][cout][oh][ow]
        r = {"alice": al_sh.reshape(_pk(L), L.cout, L.oh, L.ow), "bob": bob_sh.reshape(_pk(L), L.cout, L.oh, L.ow)}
    else:
        r = {"alice": al_sh.reshape(L.cout, L.oh, L.ow), "bob": bob_sh.reshape(L.cout, L.oh, L.ow)}
    if "ct" in want:
        r["ct_in"] = ct.reshape(L.cin, B, 2, n)
        r["ct_out"] = ct_out.reshape(L.cout, B, 2, n)
    return r


def run_protocol(schedule, image, weights, rand, q, p, n, want=(), workers=1, w_evals=None):
    """Full schedule for one image. image: [cin][H][W] signed ints; weights: list of
    [cout][cin][fh][fw] arrays (one per conv). Returns (output, trace).  `w_evals`
    (optional) = the prepared weights of every conv (prepare_weights), reused across
    images; `workers` host threads split each layer by output channels."""
    t = rand.secret()
    H, W = image.shape[1:]
    alice = np.array([[[int(v) % p for v in row] for row in ch] for ch in image], np.uint64)
    bob = None
    t_eval = None
    conv_i = 0
    trace = []
    out = None
    for li, s in enumerate(schedule):
        if isinstance(s, Conv):
            L = layer(q, p, n, H, W, s.fh, s.fw, int(s.same), s.cin, s.cout)
            if t_eval is None:
                t_eval = secret_eval(L, t)
            w_eval = w_evals[conv_i] if w_evals is not None else prepare_weights(L, weights[conv_i], workers)
            e, a = rand.enc(li, s.cin, L.blocks)
            s_b = rand.share(li, s.cout, L.blocks)
            r = run_layer(L, t_eval, alice, bob, w_eval, e, a, s_b, want, workers)
            trace.append(r)
            alice, bob = r["alice"], r["bob"]
            H, W = L.oh, L.ow
            conv_i += 1
        else:
            rec = (alice + bob) % np.uint64(p)
            flat = np.ascontiguousarray(rec.reshape(-1))
            if lib().eo_activation(flat, flat.size, p, s.fn) != 0:
                raise OverflowError("square activation exceeds p_a/2")
            val = flat.reshape(rec.shape)
            if getattr(s, "pool2", False):
                cen = np.where(val > p // 2, val.astype(np.int64) - p, val.astype(np.int64))
                C_, H_, W_ = cen.shape
                cen = cen.reshape(C_, H_ // 2, 2, W_ // 2, 2).max(axis=(2, 4))
                val = np.where(cen < 0, cen + p, cen).astype(np.uint64)
                H, W = H // 2, W // 2
            fresh = rand.reshare(li, val.shape[0], H * W).reshape(val.shape)
            if li + 1 == len(schedule):
                out = val
            alice = (val + np.uint64(p) - fresh) % np.uint64(p)
            bob = fresh
    if out is None:
        out = (alice + bob) % np.uint64(p)
    return out, trace


def plain_protocol(schedule, image, weights, q, p, n, workers=1):
    """The plaintext ground truth of a schedule for one image: conv_oracle per conv
    layer (REF ntt.cpp:187-226, channel-summed mod p) and trusted_activation semantics
    (REF protocol.cpp:237-268) plus the builder's 2x2 max-pool -- REF reference_pipeline
    (protocol.cpp:694-750) extended by the pool.  Returns [cout][h][w] residues."""
    x = np.ascontiguousarray(np.asarray(image, np.int64) % p, np.uint64)
    H, W = x.shape[1:]
    ci = 0
    for s in schedule:
        if isinstance(s, Conv):
            L = layer(q, p, n, H, W, s.fh, s.fw, int(s.same), s.cin, s.cout)
            w = np.ascontiguousarray(weights[ci], np.int64).reshape(s.cout, -1)
            out = np.zeros((s.cout, L.oh * L.ow), np.uint64)
            xf = x.reshape(-1)

            def job(r, L=L, w=w, out=out, xf=xf):
                o0, o1 = r
                o = np.zeros((o1 - o0) * L.oh * L.ow, np.uint64)
                lib().eo_conv_direct(C.byref(_sub(L, o1 - o0)), xf, np.ascontiguousarray(w[o0:o1]).reshape(-1), o)
                out[o0:o1] = o.reshape(o1 - o0, -1)
            _pmap(job, _ranges(s.cout, workers), workers)
            x = out.reshape(s.cout, L.oh, L.ow)
            H, W = L.oh, L.ow
            ci += 1
        else:
            flat = np.ascontiguousarray(x.reshape(-1))
            if lib().eo_activation(flat, flat.size, p, s.fn) != 0:
                raise OverflowError("square activation exceeds p_a/2")
            x = flat.reshape(x.shape)
            if getattr(s, "pool2", False):
                cen = np.where(x > p // 2, x.astype(np.int64) - p, x.astype(np.int64))
                C_, H_, W_ = cen.shape
                cen = cen.reshape(C_, H_ // 2, 2, W_ // 2, 2).max(axis=(2, 4))
                x = np.where(cen < 0, cen + p, cen).astype(np.uint64)
                H, W = H // 2, W // 2
    return x


# ------------------------------------------------------------------ RNS (config 4)

def rns_delta(qs, p):
    """floor(Q/p) mod q_r for Q = prod q_r (every q_r == 1 mod p, so Q == 1 mod p)."""
    Q = 1
    for q in qs:
        Q *= q
    return [((Q - 1) // p) % q for q in qs]


def set_grid(L, grid):
    """Grid override (the device's ensei_conv_desc::grid): a padded side that holds the
    linear convolution and divides p - 1, like the lengths REF's choose_padded_len falls
    back to (ntt.cpp:51-61); the C restatement's transforms take any such length (direct
    O(L^2) path, REF ntt.cpp:35-49)."""
    if grid:
        assert grid >= L.H + L.fh - 1 and grid >= L.W + L.fw - 1 and (L.p - 1) % grid == 0
        L.Lh = L.Lw = grid
        L.blocks = -(-grid * grid // L.n)
    return L


def rns_layers(qs, p, n, H, W, fh, fw, same, cin, cout, pack=1, grid=0):
    Ls = []
    for q, d in zip(qs, rns_delta(qs, p)):
        L = set_grid(layer(q, p, n, H, W, fh, fw, same, cin, cout), grid)
        L.delta = d
        L.pack = pack
        Ls.append(L)
    return Ls


class PhiloxRandomnessRNS(PhiloxRandomness):
    """Per-prime a^ streams (block field | prime << 12), shared noise and shares."""

    def __init__(self, seed, image, n, qs, p, cbd_k=20):
        super().__init__(seed, image, n, qs[0], p, cbd_k)
        self.qs = qs

    def enc_rns(self, layer_idx, cin, blocks):
        R = len(self.qs)
        e = np.empty((cin, blocks, self.n), np.int64)
        a = np.empty((cin, blocks, R, self.n), np.uint64)
        for c in range(cin):
            for b in range(blocks):
                e[c, b] = rand_cbd(self.ka, stream_id(PURPOSE_NOISE, layer_idx, self.image, c, b), self.n, self.k)
                for r, q in enumerate(self.qs):
                    a[c, b, r] = rand_uniform_q(self.ka, stream_id(PURPOSE_AHAT, layer_idx, self.image, c, b | (r << 12)),
                                                self.n, q)
        return e, a


def run_layer_rns(Ls, t_evals, alice_in, w_evals, e, a, s_b, workers=1):
    """One RNS conv layer (first layer: no HomRec) for one image; per-prime Enc /
    ElementMult / HomShare with the single-prime restatement, CRT decryption; `workers`
    host threads over (prime, output-channel slice)."""
    R = len(Ls)
    L0 = Ls[0]
    n, B = L0.n, L0.blocks
    ct_in = np.zeros((L0.cin, B, 2, R, n), np.uint64)
    ct_out = np.zeros((L0.cout, B, 2, R, n), np.uint64)
    cts = [None] * R

    def enc(r):
        ct = np.zeros(Ls[r].cin * B * 2 * n, np.uint64)
        lib().eo_alice_encrypt(C.byref(Ls[r]), t_evals[r], np.ascontiguousarray(alice_in, np.uint64).reshape(-1),
                               np.ascontiguousarray(e, np.int64).reshape(-1),
                               np.ascontiguousarray(a[:, :, r], np.uint64).reshape(-1), ct)
        cts[r] = ct
        ct_in[:, :, :, r] = ct.reshape(L0.cin, B, 2, n)
    _pmap(enc, range(R), workers)
    pk = _pk(L0)
    bob = np.zeros((pk, L0.cout, L0.oh * L0.ow), np.uint64)
    s_b = np.ascontiguousarray(s_b, np.uint64).reshape(L0.cout, -1)
    jobs = [(r, rg) for r in range(R) for rg in _ranges(L0.cout, max(1, workers // R))]

    def mac(job):
        r, (o0, o1) = job
        w = np.ascontiguousarray(w_evals[r], np.uint64).reshape(L0.cout, -1)
        co = np.zeros((o1 - o0) * B * 2 * n, np.uint64)
        bs = np.zeros(pk * (o1 - o0) * L0.oh * L0.ow, np.uint64)
        lib().eo_bob_eval(C.byref(_sub(Ls[r], o1 - o0)), cts[r], np.ascontiguousarray(w[o0:o1]).reshape(-1), None,
                          np.ascontiguousarray(s_b[o0:o1]).reshape(-1), co, bs)
        ct_out[o0:o1, :, :, r] = co.reshape(o1 - o0, B, 2, n)
        if r == 0:
            bob[:, o0:o1] = bs.reshape(pk, o1 - o0, -1)
    _pmap(mac, jobs, workers)
    al = np.zeros((pk, L0.cout, L0.oh * L0.ow), np.uint64)
    te = np.ascontiguousarray(np.stack(t_evals), np.uint64).reshape(-1)

    def dec(rg):
        o0, o1 = rg
        arr = (Layer * R)(*[_sub(L, o1 - o0) for L in Ls])
        a_ = np.zeros(pk * (o1 - o0) * L0.oh * L0.ow, np.uint64)
        lib().eo_alice_decrypt_rns(C.cast(arr, C.c_void_p), R, te, np.ascontiguousarray(ct_out[o0:o1]).reshape(-1), a_)
        al[:, o0:o1] = a_.reshape(pk, o1 - o0, -1)
    _pmap(dec, _ranges(L0.cout, workers), workers)
    shape = (pk, L0.cout, L0.oh, L0.ow) if pk > 1 else (L0.cout, L0.oh, L0.ow)
    return {"alice": al.reshape(shape), "bob": bob.reshape(shape), "ct_in": ct_in, "ct_out": ct_out}
