// layer_rns.cuh -- second-generation tile kernels (Enc / HomRec, HomShare, Dec, weight
// preparation), templates over the ring degree, the prime count and the padded-grid policy.
// Instantiated for the 3-prime RNS layer at n = 8192 (config 4: 512-thread CTAs, two per SM)
// and for single-prime layers at n = 2048 on overridden grids (configs 3 / 1: 256-thread
// CTAs, four per SM).
//
// The first-generation kernels (layer.cuh) give every (ciphertext image, channel) tile at
// n = 8192 a 1024-thread CTA that fills an SM's register file: all 32 warps are in the same
// fused stage at the same time, so the load-bound stages (Dec's first INTT pass straight from
// HBM, Enc's a^ draw, the global stores) never overlap the FMA-bound butterfly passes
// (ncu, profiles/r02a_ncu_summary_first_generation.md: issue active 42-56 %, one CTA per SM).
// Here a tile is owned by at most 512 threads that run every radix-8 pass in rounds of n / 8
// virtual threads (same registers per thread, same shared-memory traffic), and the working
// set is cut to <= 113 KB at n = 8192 by aliasing buffers whose lifetimes do not overlap, so
// two CTAs in different stages share an SM (an Enc and a HomShare CTA co-reside too).
//
// One block per channel (B = 1): at n = 8192 every supported grid (<= 64 x 64) fits; at
// n = 2048 the overridden grids do (39^2, 3 x 24^2, 12 x 12^2 <= 2048).
//
//   enc3_kernel     Alice Enc, REF protocol.cpp:310-329 + ringbfv.cpp:180-201 per prime;
//                   HOMREC: Bob's HomRec, REF protocol.cpp:543-557, hss.cpp:51-62
//   share3_kernel   Bob HomShare masks + his share, REF hss.cpp:22-49, protocol.cpp:587-603
//   dec3_kernel     Alice Dec (REF ringbfv.cpp:203-231; three primes: exact CRT rounding over
//                   Q = q0 q1 q2) -> merge -> IDFT2D -> crop (+ recombine), REF protocol.cpp:332-355
//   weights3_kernel Bob's prepare_plain on an overridden grid, REF protocol.cpp:462-502
#pragma once
#include "layer.cuh"

namespace ensei_gpu {

// Thread geometry of a second-generation tile kernel for ring degree 2^LOGN: n / 8 virtual
// threads (8 coefficients each, radix-8 passes) run by at most 512 real threads in rounds.
template <int LOGN>
struct Ring {
  static constexpr int N = 1 << LOGN, NV = N >> 3;
  static constexpr int NT = NV < 512 ? NV : 512;  // threads per CTA
  static constexpr int RD = NV / NT;              // rounds per pass
  static constexpr int MINB = 1024 / NT;          // CTAs per SM the 64-register budget allows
};
constexpr int kRnsLogN = 13;  // the 3-prime RNS layer's ring degree
constexpr int kRnsThreads = Ring<kRnsLogN>::NT;

// One pass of a transform run as RD rounds of virtual threads; in place or between disjoint
// buffers (no SPLIT: a virtual thread stores exactly where it loaded, or where nobody loads).
template <int LOGN, class F, class T, int I, bool INV, class Src, class Dst, bool CORR = false>
EG_DEV void rns_pass(const F& f, const TwPair<T>* __restrict__ tw, int tid, Src& src, Dst& dst, uint32_t cred = 0) {
  const CtaBar bar;
#pragma unroll 1
  for (int rd = 0; rd < Ring<LOGN>::RD; ++rd)
    run_pass<F, T, LOGN, 3, I, INV, 0, false, Src, Dst, CtaBar, CORR>(f, tw, tid + rd * Ring<LOGN>::NT, src, dst, bar,
                                                                     cred);
}

// forward: pass 0 (src -> sm), the middle passes (sm), the last (sm -> dst); no barrier before
// the first pass or after the last; a warp barrier between the two block-local last passes
// (ntt_core.cuh pass_sync: rounds keep a block's sets on the same 8 lanes).  B_IN bounds the
// inputs in units of q.
template <int LOGN, class F, class T, int B_IN, int I, class Src, class Dst>
EG_DEV void rns_forward_from(const F& f, const TwPair<T>* __restrict__ tw, T* sm, int tid, Src& src, Dst& dst,
                             uint32_t cred) {
  using FB = FwdBounds<F, 0, LOGN, 3, B_IN>;
  constexpr int L = PassPlan<LOGN, 3>::npass - 1;
  SmemRW<T> s{sm};
  if constexpr (I == L) {
    rns_pass<LOGN, F, T, L, false, SmemRW<T>, Dst, FB::corr(L)>(f, tw, tid, s, dst, cred);
  } else {
    if constexpr (I == 0) rns_pass<LOGN, F, T, 0, false, Src, SmemRW<T>, FB::corr(0)>(f, tw, tid, src, s, cred);
    else rns_pass<LOGN, F, T, I, false, SmemRW<T>, SmemRW<T>, FB::corr(I)>(f, tw, tid, s, s, cred);
    pass_sync<LOGN, 3, I>(CtaBar{});
    rns_forward_from<LOGN, F, T, B_IN, I + 1, Src, Dst>(f, tw, sm, tid, src, dst, cred);
  }
}
template <int LOGN, class F, class T, int B_IN, class Src, class Dst>
EG_DEV void rns_forward(const F& f, const TwPair<T>* __restrict__ tw, T* sm, int tid, Src src, Dst dst,
                        uint32_t cred = 0) {
  static_assert(PassPlan<LOGN, 3>::npass >= 2, "at least two passes");
  rns_forward_from<LOGN, F, T, B_IN, 0, Src, Dst>(f, tw, sm, tid, src, dst, cred);
}

// inverse passes L (src -> sm) down to 1 (sm), a barrier after each; the caller runs pass 0
template <int LOGN, class F, class T, int I, class Src>
EG_DEV void rns_inverse_from(const F& f, const TwPair<T>* __restrict__ tw, T* sm, int tid, Src& src) {
  constexpr int L = PassPlan<LOGN, 3>::npass - 1;
  SmemRW<T> s{sm};
  if constexpr (I == L) {
    rns_pass<LOGN, F, T, L, true, Src, SmemRW<T>>(f, tw, tid, src, s);
    pass_sync<LOGN, 3, L - 1>(CtaBar{});  // passes L and L - 1: the two block-local passes
  } else {
    rns_pass<LOGN, F, T, I, true, SmemRW<T>, SmemRW<T>>(f, tw, tid, s, s);
    __syncthreads();
  }
  if constexpr (I > 1) rns_inverse_from<LOGN, F, T, I - 1, Src>(f, tw, sm, tid, src);
}
template <int LOGN, class F, class T, class Src>
EG_DEV void rns_inverse_head(const F& f, const TwPair<T>* __restrict__ tw, T* sm, int tid, Src src) {
  static_assert(PassPlan<LOGN, 3>::npass >= 2, "at least two passes");
  rns_inverse_from<LOGN, F, T, PassPlan<LOGN, 3>::npass - 1, Src>(f, tw, sm, tid, src);
}
template <int LOGN, class F, class T, class Src, class Dst>
EG_DEV void rns_inverse(const F& f, const TwPair<T>* __restrict__ tw, T* sm, int tid, Src src, Dst dst) {
  rns_inverse_head<LOGN, F, T, Src>(f, tw, sm, tid, src);
  SmemRW<T> s{sm};
  rns_pass<LOGN, F, T, 0, true, SmemRW<T>, Dst>(f, tw, tid, s, dst);
}

// floor(x C / 2^64) from three wide products (the low x low product and the middle carries
// are dropped): at most 2 below the exact floor.
EG_DEV uint64_t mulhi64_approx(uint64_t x, uint64_t c) {
  const uint32_t x0 = lo32(x), x1 = hi32(x), c0 = lo32(c), c1 = hi32(c);
  return mulw(x1, c1) + hi32(mulw(x0, c1)) + hi32(mulw(x1, c0));
}

// x w mod q in [0, 4q) for a small x < 2^32 (the lifts Delta m): Q' = hi32(x w1') drops
// x w0' / 2^64 < 1, so Q - Q' <= 2; 3 wide + 2 plain IMADs instead of 5 + 4.
EG_DEV uint64_t mul_shoup_small(const Field64& f, uint32_t x, uint64_t w, uint64_t wp) {
  const uint32_t Q = hi32(mulw(x, hi32(wp)));
  const uint64_t a = mulw(x, lo32(w)) + ((uint64_t)(x * hi32(w)) << 32);
  const uint64_t b = mulw(Q, lo32(f.q)) + ((uint64_t)(Q * hi32(f.q)) << 32);
  return a - b;
}

// uniform mod q from 128 bits, floor(x q / 2^128), exact (= philox.cuh uniform_q_from) from
// eight full-rate wide products (the generic __umul64hi costs ~20 IMAD slots).
EG_DEV uint64_t uniform_q_from_fast(const Philox4& r, uint64_t q) {
  const uint64_t x0 = ((uint64_t)r.y << 32) | r.x, x1 = ((uint64_t)r.w << 32) | r.z;
  const uint64_t h0 = mulhi64(x0, q);
  uint64_t hi, lo;
  mul128(x1, q, hi, lo);
  const uint64_t s = lo + h0;
  return hi + (s < lo ? 1 : 0);
}

// In-place 2D transforms of `nt` tiles (TS words apart) at once: every pass covers the
// lines of all tiles before its barrier (a 64 x 64 tile is one radix-8 set per thread of a
// 512-thread CTA: per-tile passes were barrier-latency-bound, ncu: 28 % of HomShare's
// samples for 12 % of its instructions).  Inverse: values are left in [0, 2p) -- the caller
// reduces what it crops (kernels.cuh tile_transform_2d spends a whole pass on that).
template <bool INV, int LOGH, int LOGW>
EG_DEV void rns_tiles_2d(const Field32& f, uint32_t cred, const TwPair<uint32_t>* twc, uint32_t* S, int LS, int TS,
                         int nt) {
  constexpr int Lh = 1 << LOGH, Lw = 1 << LOGW;
  constexpr int EW = LOGW < 3 ? LOGW : 3, EH = LOGH < 3 ? LOGH : 3;
  auto rows = [=](int l) { return TileRow{S + (l >> LOGH) * TS, (l & (Lh - 1)) * LS}; };
  tile_lines_all<INV, LOGW, EW, 0>(f, twc + Lw, rows, nt * Lh);
  if constexpr (!INV) {
    auto cols = [=](int l) {
      return ReduceOnStore<TileCol>{TileCol{S + (l >> LOGW) * TS, l & (Lw - 1), LS}, f, cred};
    };
    tile_lines_all<INV, LOGH, EH, 0>(f, twc + Lh, cols, nt * Lw);
  } else {
    auto cols = [=](int l) { return TileCol{S + (l >> LOGW) * TS, l & (Lw - 1), LS}; };
    tile_lines_all<INV, LOGH, EH, 0>(f, twc + Lh, cols, nt * Lw);
  }
}

// ------------------------------------------------------------ padded-grid policies
// The tile side of a layer: how its DFT2D / IDFT2D run in shared memory and where the
// frequency (r, c) of a transformed tile lives.
//   GridPow2<LOG>  REF's choice (next power of two): radix-8 passes, frequencies in
//                  bit-reversed positions (kernels.cuh conventions).
//   GridPFA<N1,N2> a side L = N1 N2 dividing p - 1 (ensei_conv_desc::grid): REF runs its
//                  O(L^2) ntt_direct for such lengths (ntt.cpp:35-49); here the same
//                  transform as a prime-factor one; natural order throughout; L^-1 per
//                  dimension folded into the inverse tables.
template <int LOG>
struct GridPow2 {
  static constexpr int L = 1 << LOG, LS = L + 1, G = L * L;
  static constexpr int TS = tile_words<LOG, LOG>();
  static constexpr bool kScratch = false;
  EG_DEV static int px(int r, int c) { return r * LS + c; }                        // pixel (r, c)
  EG_DEV static int fq(int r, int c) { return brev(r, LOG) * LS + brev(c, LOG); }  // frequency (r, c)
  EG_DEV static void split(int flat, int& pi, int& r, int& c) {  // natural slot -> (image of the pack, r, c)
    pi = flat >> (2 * LOG);
    r = (flat >> LOG) & (L - 1);
    c = flat & (L - 1);
  }
  template <bool INV>
  EG_DEV static void transform(const LayerArgs& a, uint32_t* S, uint32_t*, int nt) {
    rns_tiles_2d<INV, LOG, LOG>(a.pp.f, a.pp.cred, INV ? a.twc_inv : a.twc_fwd, S, LS, TS, nt);
  }
};

// modular inverse of a mod m for small compile-time values
constexpr int small_inv(int a, int m) {
  for (int x = 1; x < m; ++x)
    if ((a * x) % m == 1) return x;
  return 0;
}

// L = N1 N2 with coprime factors (39 = 3 x 13): Good-Thomas prime-factor transform.  With
// n = (N2 n1 + N1 n2) mod L and k = (A1 k1 + A2 k2) mod L (A1 = N2 (N2^-1 mod N1),
// A2 = N1 (N1^-1 mod N2)) the L-point transform is a twiddle-free N1 x N2 one:
//   X[k] = sum_n1 w1^(n1 k1) sum_n2 x[n] w2^(n2 k2),  w1 = w^N2, w2 = w^N1,
// N2 + N1 products per output instead of L.  One thread per (line, k2): N1 lazy 64-bit
// sums over the N2-point matrix row in shared memory, reduced, then the N1-point stage
// from registers; rows from S into the scratch copy, columns back.
template <int N1, int N2>
struct GridPFA {
  static constexpr int L = N1 * N2, LS = (L & 1) ? L : L + 1, G = L * L;  // odd row stride: conflict-free columns
  static constexpr int TS = (int)((((size_t)L * LS * 4 + 127) & ~(size_t)127) / 4);
  static constexpr bool kScratch = true;
  static constexpr int A1 = (N2 * small_inv(N2 % N1, N1)) % L, A2 = (N1 * small_inv(N1 % N2, N2)) % L;
  static_assert(small_inv(N2 % N1, N1) && small_inv(N1 % N2, N2), "coprime factors");
  static_assert(N1 <= 16 && N2 <= 16, "lazy sums of at most 16 products (red64)");
  EG_DEV static int px(int r, int c) { return r * LS + c; }
  EG_DEV static int fq(int r, int c) { return r * LS + c; }
  EG_DEV static void split(int flat, int& pi, int& r, int& c) {
    pi = flat / G;
    const int rem = flat - pi * G;
    r = rem / L;
    c = rem - r * L;
  }
  // z < 2^zb (zb = grid_zbits: N2 p^2 fits) -> canonical.  Barrett with one wide product:
  // q^ = ((z >> (bp - 1)) mu) >> (zb - bp + 1), mu = floor(2^zb / p), bp = bits(p): at most 2
  // below the quotient, so z - q^ p < 3p (the generic 64-bit reduction took four wide products)
  EG_DEV static uint32_t red64(const LayerArgs& a, uint64_t z) {
    const uint32_t qh = (uint32_t)((mulw((uint32_t)(z >> a.grid_s1), a.grid_mu)) >> a.grid_s2);
    uint32_t r = (uint32_t)z - qh * a.pp.f.q;
    if (r >= a.pp.f.q2) r -= a.pp.f.q2;
    return a.pp.f.reduce_once(r);
  }
  template <bool COLS>
  EG_DEV static void lines(const LayerArgs& a, const uint32_t* M2, const uint32_t* M1, const uint32_t* in,
                           uint32_t* out, int nt) {
    constexpr int ST = COLS ? LS : 1;
    for (int it = threadIdx.x; it < nt * L * N2; it += blockDim.x) {
      const int t = it / (L * N2), rem = it - t * (L * N2), ln = rem / N2, k2 = rem - ln * N2;
      const uint32_t* x = in + t * TS + (COLS ? ln : ln * LS);
      const uint32_t* m2 = M2 + k2 * N2;
      uint32_t y[N1];
#pragma unroll
      for (int n1 = 0; n1 < N1; ++n1) {
        uint64_t acc = 0;
#pragma unroll
        for (int n2 = 0; n2 < N2; ++n2) acc = madw(x[((N2 * n1 + N1 * n2) % L) * ST], m2[n2], acc);
        y[n1] = red64(a, acc);
      }
      const int kb = (A2 * k2) % L;
#pragma unroll
      for (int k1 = 0; k1 < N1; ++k1) {
        uint64_t acc = 0;
#pragma unroll
        for (int n1 = 0; n1 < N1; ++n1) acc = madw(y[n1], M1[k1 * N1 + n1], acc);
        int k = kb + A1 * k1;
        k = k >= L ? k - L : k;  // kb < L, A1 k1 < L for k1 < N1
        k = k >= L ? k - L : k;
        out[t * TS + (COLS ? k * LS + ln : ln * LS + k)] = red64(a, acc);
      }
    }
  }
  template <bool INV>
  EG_DEV static void transform(const LayerArgs& a, uint32_t* S, uint32_t* scratch, int nt) {
    __shared__ uint32_t M2[N2 * N2], M1[N1 * N1];
    const Field32 f = a.pp.f;
    auto pw = [&](uint32_t b, int e) {
      uint32_t r = 1;
      for (; e; e >>= 1) {
        if (e & 1) r = f.mul(r, b, a.pp.m64);
        b = f.mul(b, b, a.pp.m64);
      }
      return r;
    };
    const uint32_t w = INV ? a.grid_winv : a.grid_w;
    for (int i = threadIdx.x; i < N2 * N2 + N1 * N1; i += blockDim.x) {
      if (i < N2 * N2) {
        M2[i] = pw(pw(w, N1), ((i / N2) * (i % N2)) % N2);
      } else {
        const int j = i - N2 * N2;
        const uint32_t v = pw(pw(w, N2), ((j / N1) * (j % N1)) % N1);
        M1[j] = INV ? f.mul(v, a.grid_linv, a.pp.m64) : v;  // L^-1 per dimension
      }
    }
    __syncthreads();
    lines<false>(a, M2, M1, S, scratch, nt);
    __syncthreads();
    lines<true>(a, M2, M1, scratch, S, nt);
    __syncthreads();
  }
};

// -------------------------------------------------------------------- Enc
// shared: [ qbuf n u64 | pbuf n u32 (padded) | noise n int8 ]; the pk DFT2D tiles alias
// qbuf (dead once encode_slots' first pass has gathered them).
template <int LOGN>
constexpr size_t enc3_smem() {
  return (size_t)(1 << LOGN) * 8 + ssize<uint32_t>(1 << LOGN) * 4 + (1 << LOGN);
}
// tiles (and the direct transform's scratch copy) that must fit in qbuf's space
template <class GR>
constexpr size_t grid_tile_bytes(int nt) {
  return (size_t)nt * GR::TS * 4 * (GR::kScratch ? 2 : 1);
}

// slot value at ring position j (natural slot brev(j)); 0 past the packed grids.  TILE0:
// every pack position reads tile 0 (prepared weights, replicated across the pack)
template <int LOGN, class GR, bool TILE0 = false>
EG_DEV uint32_t grid_gather(const uint32_t* S, int j, int pk) {
  int pi, r, c;
  GR::split(brev(j, LOGN), pi, r, c);
  return pi >= pk ? 0u : S[(TILE0 ? 0 : pi) * GR::TS + GR::fq(r, c)];
}

template <int LOGN, int R, class GR, int IN_T, bool HOMREC = false>
__global__ void __launch_bounds__(Ring<LOGN>::NT, Ring<LOGN>::MINB)
    enc3_kernel(const __grid_constant__ LayerArgs a, const uint64_t* __restrict__ key, uint32_t key_stride,
                const void* __restrict__ in, uint64_t* __restrict__ out) {
  constexpr int N = 1 << LOGN, NT = Ring<LOGN>::NT;
  constexpr int TS = GR::TS;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint64_t* qbuf = reinterpret_cast<uint64_t*>(smem_raw);
  uint32_t* S = reinterpret_cast<uint32_t*>(smem_raw);  // tiles alias qbuf
  uint32_t* pbuf = reinterpret_cast<uint32_t*>(qbuf + N);
  int8_t* ebuf = reinterpret_cast<int8_t*>(pbuf + ssize<uint32_t>(N));
  const int tid = threadIdx.x;
  const Field32 pf = a.pp.f;
  const int item = blockIdx.x;
  const int ch = item % a.cin, img = item / a.cin;
  const int npk = a.pk;
  pdl_trigger();

  // 1. pad into the tiles (REF pad_image, ntt.cpp:155-185), pk images
  for (int e = tid; e < npk * GR::G; e += NT) {
    const int pi = e / GR::G, i = e - pi * GR::G;
    const int r = i / GR::L, c = i - r * GR::L;
    uint32_t v = 0;
    if (r < a.H && c < a.W && img * npk + pi < a.num_images) {
      const size_t src = ((size_t)((img * npk + pi) * a.cin + ch) * a.H + r) * a.W + c;
      if constexpr (IN_T == ENSEI_IN_U8) v = static_cast<const uint8_t*>(in)[src];
      else v = static_cast<const uint32_t*>(in)[src] % pf.q;
    }
    S[pi * TS + GR::px(r, c)] = v;
  }
  // Enc noise e0, two CBD draws per Philox call
  const int gimg = a.image_base / a.pk + img;
  if constexpr (!HOMREC) {
    const uint32_t mask = a.cbd_k >= 32 ? 0xFFFFFFFFu : ((1u << a.cbd_k) - 1u);
    const uint64_t sid = stream_id(PURPOSE_NOISE, a.layer, gimg, ch, 0);
    for (int i2 = tid; i2 < N / 2; i2 += NT) {
      const Philox4 rr = philox(a.alice_key, sid, i2);
      const int e0 = cbd_from(rr.x, rr.y, mask), e1 = cbd_from(rr.z, rr.w, mask);
      *reinterpret_cast<uint16_t*>(ebuf + 2 * i2) = (uint16_t)((e0 & 0xFF) | ((e1 & 0xFF) << 8));
    }
  }
  __syncthreads();
  // 2. DFT2D of each tile
  GR::template transform<false>(a, S, S + npk * TS, npk);
  // 3. encode_slots: INTT_p of the slots gathered from the tiles
  {
    auto src = [&](int j) { return grid_gather<LOGN, GR>(S, j, a.pk); };
    SmemRW<uint32_t> praw{pbuf};
    auto dst = [&](int i, uint32_t v) { praw(i, Bfly<Field32, 0>::fin_gs(pf, v)); };
    rns_inverse<LOGN, Field32, uint32_t>(pf, a.twp_inv, pbuf, tid, src, dst);
  }
  __syncthreads();
  const uint64_t* kimg = key + (size_t)img * key_stride;
  uint64_t* ob = out + (size_t)item * ct_words<R>(N);
#pragma unroll 1
  for (int r = 0; r < R; ++r) {
    const PrimeConst pc = a.pc[r];
    const Field64 f = pc.f;
    // 4. Delta m + e, lazy in [0, 3q)
    auto src = [&](int i) -> uint64_t {
      uint64_t x = mul_shoup_small(f, pbuf[sidx<uint32_t>(i)], pc.delta, pc.delta_shoup);  // < 4q
      if (x >= f.q2) x -= f.q2;
      if constexpr (HOMREC) return x;
      else return x + signed_mod(ebuf[i], f.q);
    };
    SmemRW<uint64_t> qs{qbuf};
    rns_forward<LOGN, Field64, uint64_t, 3>(f, a.twq_fwd[r], qbuf, tid, src, qs, pc.cred);
    __syncthreads();
    // 5. c0 = -a^, c1 = a^ t^ + NTT(Delta m + e); two slots per step, 16-byte accesses
    uint64_t* c0 = ob + (size_t)r * N;
    uint64_t* c1 = ob + (size_t)(R + r) * N;
    const uint64_t* tk = kimg + (size_t)(2 * r) * N;
    const uint64_t* tkp = tk + N;
    const uint64_t sid = stream_id(PURPOSE_AHAT, a.layer, gimg, ch, r << 12);
    for (int j2 = tid; j2 < N / 2; j2 += NT) {
      const int j = 2 * j2;
      const ulonglong2 xv = *reinterpret_cast<const ulonglong2*>(qbuf + sidx<uint64_t>(j));
      if constexpr (HOMREC) {  // HomRec (REF hss.cpp:51-62): c1 += NTT_q(Delta INTT_p(DFT2D(Bob's share)))
        const ulonglong2 cv = *reinterpret_cast<const ulonglong2*>(c1 + j);
        const uint64_t y0 = cv.x + Bfly<Field64, 0>::fin_ct(f, xv.x, pc.cred);
        const uint64_t y1 = cv.y + Bfly<Field64, 0>::fin_ct(f, xv.y, pc.cred);
        *reinterpret_cast<ulonglong2*>(c1 + j) = make_ulonglong2(y0 >= f.q ? y0 - f.q : y0, y1 >= f.q ? y1 - f.q : y1);
        continue;
      }
      const ulonglong2 tv = __ldg(reinterpret_cast<const ulonglong2*>(tk + j));
      const ulonglong2 tpv = __ldg(reinterpret_cast<const ulonglong2*>(tkp + j));
      const int k = brev(j, LOGN);  // natural slot index keys the a^ stream; slot j + 1 -> k + n/2
      const uint64_t ah0 = uniform_q_from_fast(philox(a.alice_key, sid, k), f.q);
      const uint64_t ah1 = uniform_q_from_fast(philox(a.alice_key, sid, k + N / 2), f.q);
      auto fin = [&](uint64_t x, uint64_t ah, uint64_t t, uint64_t tp) {
        uint64_t v = Bfly<Field64, 0>::corr(f, x, pc.cred) + f.mul_shoup_approx(ah, t, tp);  // < 7q
        if (v >= f.q4) v -= f.q4;
        if (v >= f.q2) v -= f.q2;
        return v >= f.q ? v - f.q : v;
      };
      *reinterpret_cast<ulonglong2*>(c0 + j) = make_ulonglong2(ah0 ? f.q - ah0 : 0, ah1 ? f.q - ah1 : 0);
      *reinterpret_cast<ulonglong2*>(c1 + j) = make_ulonglong2(fin(xv.x, ah0, tv.x, tpv.x), fin(xv.y, ah1, tv.y, tpv.y));
    }
    __syncthreads();
  }
}

// ------------------------------------------------------- HomShare + Bob share
// shared: [ qbuf n u64 | pbuf n u32 (padded) ]; pbuf first holds s_B in evaluation
// (bit-reversed) order, Bob's share tile aliases qbuf.
template <int LOGN>
constexpr size_t share3_smem() {
  return (size_t)(1 << LOGN) * 8 + ssize<uint32_t>(1 << LOGN) * 4;
}

template <int LOGN, int R, class GR>
__global__ void __launch_bounds__(Ring<LOGN>::NT, Ring<LOGN>::MINB)
    share3_kernel(const __grid_constant__ LayerArgs a, uint64_t* __restrict__ mask, uint32_t* __restrict__ bob_share) {
  constexpr int N = 1 << LOGN, NT = Ring<LOGN>::NT;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint64_t* qbuf = reinterpret_cast<uint64_t*>(smem_raw);
  uint32_t* S = reinterpret_cast<uint32_t*>(smem_raw);
  uint32_t* pbuf = reinterpret_cast<uint32_t*>(qbuf + N);
  const int tid = threadIdx.x;
  const Field32 pf = a.pp.f;
  const uint32_t p = pf.q;
  const int item = blockIdx.x;  // ciphertext image * cout + o
  const int o = item % a.cout, img = item / a.cout;
  const int gimg = a.image_base / a.pk + img;
  // 1. s_B (natural slot i -> evaluation position brev(i))
  {
    const uint64_t sid = stream_id(PURPOSE_SHARE, a.layer, gimg, o, 0);
    for (int i2 = tid; i2 < N / 2; i2 += NT) {
      const Philox4 rr = philox(a.bob_key, sid, i2);
      const int j = brev(2 * i2, LOGN);  // slot 2 i2 + 1 -> j + n/2
      pbuf[sidx<uint32_t>(j)] = uniform_p_from(rr.x, rr.y, p);
      pbuf[sidx<uint32_t>(j + N / 2)] = uniform_p_from(rr.z, rr.w, p);
    }
  }
  // 2. Bob's share of every image of the pack: crop(IDFT2D(its part of the s_B grid))
  // (REF protocol.cpp:593-602); as many tiles at once as fit in qbuf's space
  {
    constexpr int TS = GR::TS;
    constexpr int TB = (int)(((size_t)N * 8) / grid_tile_bytes<GR>(1));  // tiles per batch
    const int npi = min(a.pk, a.num_images - img * a.pk);
    for (int p0 = 0; p0 < npi; p0 += TB) {
      const int nb = min(TB, npi - p0);
      __syncthreads();
      for (int e = tid; e < nb * GR::G; e += NT) {
        const int pi = e / GR::G, i = e - pi * GR::G;
        const int r = i / GR::L, c = i - r * GR::L;
        S[pi * TS + GR::fq(r, c)] = pbuf[sidx<uint32_t>(brev((p0 + pi) * GR::G + i, LOGN))];
      }
      __syncthreads();
      GR::template transform<true>(a, S, S + nb * TS, nb);
      for (int e = tid; e < nb * a.oh * a.ow; e += NT) {
        const int pi = e / (a.oh * a.ow), i = e % (a.oh * a.ow);
        const int r = i / a.ow, c = i % a.ow;
        bob_share[((size_t)(img * a.pk + p0 + pi) * a.cout + o) * a.oh * a.ow + i] =
            pf.reduce_once(S[pi * TS + GR::px(r + a.r0, c + a.c0)]);
      }
    }
  }
  __syncthreads();
  // 3. INTT_p of (p_A - s_B) mod p_E (REF hss.cpp:33-35), in place
  {
    SmemRW<uint32_t> praw{pbuf};
    auto src = [&](int j) {
      const uint32_t s = praw(j);
      return s == 0 ? 0u : p - s;
    };
    auto dst = [&](int i, uint32_t v) { praw(i, Bfly<Field32, 0>::fin_gs(pf, v)); };
    // in place: the first pass negates on load, every virtual thread stores where it loaded
    rns_inverse<LOGN, Field32, uint32_t>(pf, a.twp_inv, pbuf, tid, src, dst);
  }
  __syncthreads();
  // 4. masks NTT_q(Delta m) land where c1 of the output ciphertext lives
#pragma unroll 1
  for (int r = 0; r < R; ++r) {
    const PrimeConst pc = a.pc[r];
    const Field64 f = pc.f;
    auto qsrc = [&](int i) {
      const uint64_t x = mul_shoup_small(f, pbuf[sidx<uint32_t>(i)], pc.delta, pc.delta_shoup);  // < 4q
      return x >= f.q2 ? x - f.q2 : x;
    };
    uint64_t* mo = mask + (size_t)item * ct_words<R>(N) + (size_t)(R + r) * N;
    GlobalOut64Fwd outw{mo, f, pc.cred};
    rns_forward<LOGN, Field64, uint64_t, 2>(f, a.twq_fwd[r], qbuf, tid, qsrc, outw, pc.cred);
    __syncthreads();
  }
}

// -------------------------------------------------------------------- Dec
// L2 prefetch of `bytes` (multiple of 16) from `g` by the calling thread (TMA bulk prefetch)
EG_DEV void prefetch_l2_bulk(const void* g, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(g), "r"(bytes) : "memory");
}

// The exact decision for one coefficient whose fixed-point CRT sum is ambiguous: the three
// phi_r by direct evaluation, exact E_r, 192-bit compare (layer.cuh).  Returns m.
template <int LOGN>
__device__ __noinline__ uint32_t dec3_exact(const LayerArgs& a, const uint64_t* cb, const uint64_t* kimg, int i) {
  constexpr int N = 1 << LOGN, R = 3;
  const uint32_t p = a.pp.f.q;
  uint64_t E[3];
  uint32_t Isum = 0;
  for (int r = 0; r < 3; ++r) {
    uint32_t I;
    uint64_t F;
    crt_part(a.pc[r], p,
             phi_direct<LOGN>(a.pc[r], a.psi_q[r], cb + (size_t)r * N, cb + (size_t)(R + r) * N,
                              kimg + (size_t)(2 * r) * N, i),
             I, E[r], F);
    Isum += I;
  }
  uint32_t v = Isum + crt_round_t(a.crt, E, 0, true);  // < 3p + 3
  if (v >= 2 * p) v -= 2 * p;
  if (v >= p) v -= p;
  return v;
}

// shared: [ qbuf n u64 | acc_lo n u32 | acc_hi n u16 ]: the CRT accumulator
// A = sum_r floor(y_r p 2^k / q_r) (y_r = phi_r (Q/q_r)^-1 mod q_r as the lazy value in
// [0, 4 q_r) the transform leaves, k = dec_kbits fraction bits, A < 12p 2^k <= 2^48) per
// coefficient; m = floor((A + 2^(k-1)) / 2^k) mod p unless the low bits sit within 16 of a
// multiple of 2^k (each term is at most 3.3 below its exact value), where dec3_exact
// decides.  y_r comes out of the INTT itself: (Q/q_r)^-1 is folded
// into the n^-1 constants of its last stage (PrimeConst::dec_*).  m overwrites acc_lo, the
// p-side transform then runs in qbuf's space and scatters into the tiles (over acc).
template <int LOGN, class GR>
constexpr size_t dec3_smem(int pk) {
  const size_t acc = (size_t)(1 << LOGN) * 6, tiles = (size_t)pk * GR::TS * 4;
  return (size_t)(1 << LOGN) * 8 + (acc > tiles ? acc : tiles);
}

template <int LOGN, int R, class GR>
__global__ void __launch_bounds__(Ring<LOGN>::NT, Ring<LOGN>::MINB)
    dec3_kernel(const __grid_constant__ LayerArgs a, const uint64_t* __restrict__ key, uint32_t key_stride, const uint64_t* __restrict__ ct,
                uint32_t* __restrict__ alice_share, const uint32_t* __restrict__ bob_share,
                uint32_t* __restrict__ outp, int ahead) {
  constexpr int N = 1 << LOGN, NT = Ring<LOGN>::NT;
  constexpr int TS = GR::TS;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint64_t* qbuf = reinterpret_cast<uint64_t*>(smem_raw);
  uint32_t* acc_lo = reinterpret_cast<uint32_t*>(qbuf + N);
  uint16_t* acc_hi = reinterpret_cast<uint16_t*>(acc_lo + N);
  uint32_t* pbuf = reinterpret_cast<uint32_t*>(qbuf);
  uint32_t* S = acc_lo;  // pk tiles, TS words apart
  const int tid = threadIdx.x;
  const Field32 pf = a.pp.f;
  const uint32_t p = pf.q;
  const int item = blockIdx.x;
  const int img = item / a.cout, o = item % a.cout;
  const uint64_t* kimg = key + (size_t)img * key_stride;
  const uint64_t* cb = ct + (size_t)item * ct_words<R>(N);
  const int kb = a.dec_kbits;
  __shared__ __align__(8) uint64_t c1_bar;
  if (tid == 0) mbar_init(&c1_bar, 1);
  __syncthreads();
#pragma unroll 1
  for (int r = 0; r < R; ++r) {
    const PrimeConst pc = a.pc[r];
    const Field64 f = pc.f;
    // phi = c0 t^ + c1 as a streaming pre-pass: c1 arrives in qbuf by TMA bulk copies (no
    // registers), c0 / t^ / t^' by 16-byte loads issued two steps ahead of their use; a warp
    // covers whole 128-byte rows per step (8 lanes x 16 B), reads the row's c1 pairs and
    // writes phi into the swizzled positions of the same row.  (Fused into the first INTT
    // pass the loads were serialised behind its butterflies by the 64-register budget:
    // four exposed L2 / HBM round trips per round, ncu: 46 % long-scoreboard stalls there.)
    const uint64_t* c0g = cb + (size_t)r * N;
    const uint64_t* tg = kimg + (size_t)(2 * r) * N;
    if (tid == 0) {
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // qbuf: generic reads/writes -> TMA writes
      mbar_expect_tx(&c1_bar, N * 8);
      const uint8_t* c1g = reinterpret_cast<const uint8_t*>(cb + (size_t)(R + r) * N);
      constexpr uint32_t kCopy = N * 8 < 32768 ? N * 8 : 32768;
      for (uint32_t off = 0; off < N * 8; off += kCopy)
        tma_bulk_g2s(reinterpret_cast<uint8_t*>(qbuf) + off, c1g + off, kCopy, &c1_bar);
      // the next prime's words (or the first prime's of the tile this SM slot runs next)
      // into L2 while this prime's passes run
      const uint64_t* nb = r + 1 < R ? cb : cb + (size_t)ahead * ct_words<R>(N);
      const int nr = r + 1 < R ? r + 1 : 0;
      if (r + 1 < R || item + ahead < (int)gridDim.x) {
        prefetch_l2_bulk(nb + (size_t)nr * N, N * 8);
        prefetch_l2_bulk(nb + (size_t)(R + nr) * N, N * 8);
      }
    }
#pragma unroll 1
    for (int b = 0; b < N / 2 / NT / 2; ++b) {
      ulonglong2 A[2], W[2], WP[2], C[2];
#pragma unroll
      for (int s2 = 0; s2 < 2; ++s2) {
        const int j = 2 * ((2 * b + s2) * NT + tid);
        A[s2] = *reinterpret_cast<const ulonglong2*>(c0g + j);
        W[s2] = __ldg(reinterpret_cast<const ulonglong2*>(tg + j));
        WP[s2] = __ldg(reinterpret_cast<const ulonglong2*>(tg + N + j));
      }
      if (b == 0) mbar_wait(&c1_bar, (uint32_t)(r & 1));
#pragma unroll
      for (int s2 = 0; s2 < 2; ++s2) C[s2] = *reinterpret_cast<const ulonglong2*>(qbuf + 2 * ((2 * b + s2) * NT + tid));
      __syncwarp();
#pragma unroll
      for (int s2 = 0; s2 < 2; ++s2) {
        const int j = 2 * ((2 * b + s2) * NT + tid);
        uint64_t x = f.mul_shoup_approx(A[s2].x, W[s2].x, WP[s2].x) + C[s2].x;  // < 5q
        uint64_t y = f.mul_shoup_approx(A[s2].y, W[s2].y, WP[s2].y) + C[s2].y;
        x = hi32(x) > hi32(f.q4) ? x - f.q4 : x;  // < 4q + 2^32: the Gentleman-Sande input bound
        y = hi32(y) > hi32(f.q4) ? y - f.q4 : y;
        *reinterpret_cast<ulonglong2*>(qbuf + sidx<uint64_t>(j)) = make_ulonglong2(x, y);
      }
    }
    __syncthreads();
    SmemRW<uint64_t> src{qbuf};
    rns_inverse_head<LOGN, Field64, uint64_t>(f, a.twq_inv[r], qbuf, tid, src);
    if constexpr (R == 1) {
      // one prime: the last pass rounds exactly, floor((p phi + floor(q/2)) / q) mod p (REF
      // ringbfv.cpp:224-229; the estimate floor(phi cp / 2^64) is at most 2 below, so the
      // remainder is < 3q and exact in 64 bits), m in natural order into acc_lo
      const uint64_t cp = pc.cp, h = f.q >> 1;
      auto dst = [&](int i, uint64_t v) {
        const uint64_t phi = Bfly<Field64, 0>::fin_gs(f, v);
        const uint64_t Qe = mulhi64(phi, cp);
        const uint64_t rem = (uint64_t)p * phi + h - Qe * f.q;
        const uint32_t Qs = (uint32_t)Qe + (rem >= f.q) + (rem >= f.q2);
        acc_lo[i] = Qs >= p ? Qs - p : Qs;
      };
      SmemRW<uint64_t> qs{qbuf};
      rns_pass<LOGN, Field64, uint64_t, 0, true>(f, a.twq_inv[0], tid, qs, dst);
      __syncthreads();
      continue;
    }
    static_assert(R == 1 || LOGN == 13, "the CRT last stage below is written for the 1 + 3 + 3 + 3 + 3 pass plan");
    // last stage (coefficients i, i + n/2) with the CRT constants folded in, then the
    // accumulator
    const TwPair<uint64_t> t1{pc.dec_t1, pc.dec_t1_shoup}, ni{pc.dec_ni, pc.dec_ni_shoup};
#pragma unroll 1
    for (int i = tid; i < N / 2; i += NT) {
      uint64_t u = qbuf[sidx<uint64_t>(i)], v = qbuf[sidx<uint64_t>(i + N / 2)];
      Bfly<Field64, 0>::gs_last(f, u, v, t1, ni);
      // lazy y = y_r + j q_r (j <= 3) only adds j p to the integer part of its term
      const uint64_t y[2] = {u, v};
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int idx = i + h * (N / 2);
        uint64_t A = mulhi64_approx(y[h], pc.dec_c);
        if (r > 0) A += (uint64_t)acc_lo[idx] | ((uint64_t)acc_hi[idx] << 32);
        if (r < R - 1) {
          acc_lo[idx] = (uint32_t)A;
          acc_hi[idx] = (uint16_t)(A >> 32);
        } else {
          A += 1ull << (kb - 1);
          const uint64_t low = A & ((1ull << kb) - 1);
          uint32_t m;
          if (low < 16 || low > (1ull << kb) - 16) m = dec3_exact<LOGN>(a, cb, kimg, idx);
          else m = reduce_lazy(pf, (uint32_t)(A >> kb), a.pp.cred);  // A >> kb <= 12p
          acc_lo[idx] = m;
        }
      }
    }
    __syncthreads();
  }
  // decode_slots (NTT_p): m (acc_lo, natural order) -> qbuf's space -> tiles over acc
  {
    auto psrc = [&](int i) { return acc_lo[i]; };
    auto pdst = [&](int j, uint32_t v) {
      int pi, r, c;
      GR::split(brev(j, LOGN), pi, r, c);
      if (pi < a.pk) S[pi * TS + GR::fq(r, c)] = reduce_lazy(pf, v, a.pp.cred);
    };
    rns_forward<LOGN, Field32, uint32_t, 1>(pf, a.twp_fwd, pbuf, tid, psrc, pdst);
  }
  __syncthreads();
  {  // IDFT2D of every image of the pack at once, crop (+ recombine)
    const int npi = min(a.pk, a.num_images - img * a.pk);
    GR::template transform<true>(a, S, pbuf, npi);  // (scratch: qbuf's space, free after the p-side transform)
    for (int e = tid; e < npi * a.oh * a.ow; e += NT) {
      const int pi = e / (a.oh * a.ow), i = e % (a.oh * a.ow);
      const int r = i / a.ow, c = i % a.ow;
      const uint32_t s = pf.reduce_once(S[pi * TS + GR::px(r + a.r0, c + a.c0)]);
      const size_t at = ((size_t)(img * a.pk + pi) * a.cout + o) * a.oh * a.ow + i;
      if (alice_share) alice_share[at] = s;
      if (outp) {
        const uint32_t y = s + bob_share[at];
        outp[at] = y >= p ? y - p : y;
      }
    }
  }
}

// -------------------------------------------------------------------- weights
// Bob's setup for layers with a grid override (REF protocol.cpp:462-502,
// ringbfv.cpp:265-280): one CTA per (out, in) filter: pad -> DFT2D -> replicate across the
// pack -> encode_slots -> centered lift -> NTT_q -> packed 30-bit limbs [cout][cin][1][R][n]
// (the layout of tile_enc_kernel<TILE_WEIGHTS>, layer.cuh).  Shared memory as Enc.
template <int LOGN, int R, class GR>
__global__ void __launch_bounds__(Ring<LOGN>::NT, Ring<LOGN>::MINB)
    weights3_kernel(const __grid_constant__ LayerArgs a, const int32_t* __restrict__ w, uint64_t* __restrict__ out) {
  constexpr int N = 1 << LOGN, NT = Ring<LOGN>::NT;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint64_t* qbuf = reinterpret_cast<uint64_t*>(smem_raw);
  uint32_t* S = reinterpret_cast<uint32_t*>(smem_raw);
  uint32_t* pbuf = reinterpret_cast<uint32_t*>(qbuf + N);
  const int tid = threadIdx.x;
  const Field32 pf = a.pp.f;
  const uint32_t p = pf.q;
  const int item = blockIdx.x;  // o * cin + ci
  for (int e = tid; e < GR::G; e += NT) {
    const int r = e / GR::L, c = e - r * GR::L;
    uint32_t v = 0;
    if (r < a.fh && c < a.fw) {
      const int64_t m = (int64_t)w[((size_t)item * a.fh + r) * a.fw + c] % (int64_t)p;
      v = (uint32_t)(m < 0 ? m + p : m);  // encode_signed
    }
    S[GR::px(r, c)] = v;
  }
  __syncthreads();
  GR::template transform<false>(a, S, S + GR::TS, 1);
  {
    auto src = [&](int j) { return grid_gather<LOGN, GR, true>(S, j, a.pk); };
    SmemRW<uint32_t> praw{pbuf};
    auto dst = [&](int i, uint32_t v) { praw(i, Bfly<Field32, 0>::fin_gs(pf, v)); };
    rns_inverse<LOGN, Field32, uint32_t>(pf, a.twp_inv, pbuf, tid, src, dst);
  }
  __syncthreads();
#pragma unroll 1
  for (int r = 0; r < R; ++r) {
    const PrimeConst pc = a.pc[r];
    const Field64 f = pc.f;
    auto src = [&](int i) -> uint64_t {  // encode_signed(decode_signed(m)) over q_r
      const uint32_t m = pbuf[sidx<uint32_t>(i)];
      return m > p / 2 ? f.q - (uint64_t)(p - m) : (uint64_t)m;
    };
    SmemRW<uint64_t> qs{qbuf};
    rns_forward<LOGN, Field64, uint64_t, 1>(f, a.twq_fwd[r], qbuf, tid, src, qs, pc.cred);
    __syncthreads();
    uint64_t* ob = out + ((size_t)item * R + r) * N;
    for (int j = tid; j < N; j += NT) {
      const uint64_t x = Bfly<Field64, 0>::fin_ct(f, qbuf[sidx<uint64_t>(j)], pc.cred);
      ob[j] = ((x >> 30) << 32) | (x & 0x3FFFFFFFull);
    }
    __syncthreads();
  }
}

}  // namespace ensei_gpu
