// layer.cuh -- fused kernels of one oblivious conv layer (templates).
//
//   tile_enc_kernel   Alice Enc (REF protocol.cpp:310-329 + ringbfv.cpp:180-201):
//                     pad -> DFT2D -> split -> encode (INTT_p) -> Delta*m + e -> NTT_q
//                     -> c0 = -a^, c1 = a^ t^ + payload.   Variants: HomRec (Bob adds
//                     NTT_q(Delta*INTT_p(DFT2D(share))) into c1, REF hss.cpp:51-62) and
//                     weight preparation (REF protocol.cpp:462-502, ringbfv.cpp:265-280).
//   share_kernel      Bob HomShare masks NTT_q(Delta*INTT_p(p - s_B)) (REF hss.cpp:22-49)
//                     and Bob's time-domain share crop(IDFT2D(s_B)) (REF protocol.cpp:587-603).
//   mac_kernel        ElementMult + channel accumulation (REF ringbfv.cpp:233-306,
//                     protocol.cpp:570-581) as a tiled per-slot GEMM with lazy 128-bit
//                     accumulation, + the HomShare mask on c1.
//   dec_kernel        Alice Dec (REF ringbfv.cpp:203-231) -> merge -> IDFT2D -> crop
//                     (REF protocol.cpp:332-355) [+ recombine_clear, REF hss.cpp:64-73].
//
// Data never round-trips through HBM inside a kernel: tiles, slot vectors and ring
// polynomials live in shared memory between fused stages.
#pragma once
#include "common.cuh"
#include "kernels.cuh"
#include "philox.cuh"

namespace ensei_gpu {

// log2(coefficients per thread) in the ring transforms of the tile kernels (8 per thread,
// n/8 threads per ring polynomial, radix-8 register passes).  4 per thread at n = 2048
// (twice the threads per tile, 6 passes instead of 4) was measured slower: config 1
// 78.6 -> 86.5 us per step, config 3 -9 %.
__host__ __device__ constexpr int tile_loge(int) { return 3; }
// Tile kernels are latency-bound (one CTA per tile, serial fused stages): capping them
// at 64 registers lets two CTAs share an SM, so Bob's HomShare CTAs co-reside with
// Alice's Enc CTAs and each hides the other's latency.
constexpr int tile_min_blocks(int threads) { return threads >= 1024 ? 1 : 1024 / threads; }

struct LayerArgs {
  // geometry (REF ConvGeometry / LayerPlan)
  int H, W, fh, fw, cin, cout;
  int Lh, Lw, B, oh, ow, r0, c0, G;
  int num_images;
  int pk;       // images per ciphertext block (1: REF geometry)
  int num_cts;  // ciphertext "images" = ceil(num_images / pk): the rows of the ElementMult / 2
  // ring
  PrimeConst pc[ENSEI_MAX_PRIMES];
  uint64_t psi_q[ENSEI_MAX_PRIMES];  // canonical 2n-th roots (direct-evaluation fallback)
  CrtConst crt;
  int dec_kbits;  // layer_rns.cuh: fraction bits of the packed CRT accumulator
  // grid override (layer_rns.cuh GridPFA): primitive L-th root of unity mod p (REF's
  // canonical root, g^((p-1)/L)), its inverse, and L^-1 mod p
  uint32_t grid_w, grid_winv, grid_linv;
  // Barrett reduction of the tile transforms' lazy sums (< 2^zb): shifts and floor(2^zb / p)
  uint32_t grid_mu, grid_s1, grid_s2;
  PConst pp;
  const TwPair<uint64_t>* twq_fwd[ENSEI_MAX_PRIMES];
  const TwPair<uint64_t>* twq_inv[ENSEI_MAX_PRIMES];
  const TwPair<uint32_t>* twp_fwd;
  const TwPair<uint32_t>* twp_inv;
  const TwPair<uint32_t>* twc_fwd;
  const TwPair<uint32_t>* twc_inv;
  // randomness
  uint32_t rand_mode, layer, image_base, cbd_k;
  uint64_t alice_key, bob_key;
  const int32_t* inj_noise;
  const uint64_t* inj_ahat;
  const uint32_t* inj_share;
};

// ---------------------------------------------------------------- helpers

// Packing: a ciphertext block carries `pk` images' grids back to back (slots
// [pi G, (pi + 1) G) hold image pi of the pack; pk = 1 is REF's geometry, one image per
// block with the tail zero-filled, REF protocol.cpp:18-29).  The pk DFT2D tiles live at
// S + pi * TS (TS words apart), each bit-reversed in both dimensions
// (S[brev(r)][brev(c)] = G[r][c]).
// slot value at ring position j of block b; 0 past the packed grids.  TILE0: every pack
// position reads tile 0 (prepared weights, replicated across the pack)
template <int LOGN, int LOGH, int LOGW, bool TILE0 = false>
EG_DEV uint32_t gather_slot(const uint32_t* S, int b, int j, int pk, int TS) {
  const int flat = (b << LOGN) + brev(j, LOGN);
  const int pi = flat >> (LOGH + LOGW);
  if (pi >= pk) return 0;
  const int r = (flat >> LOGW) & ((1 << LOGH) - 1), c = flat & ((1 << LOGW) - 1);
  return S[(TILE0 ? 0 : pi) * TS + brev(r, LOGH) * ((1 << LOGW) + 1) + brev(c, LOGW)];
}

// scatter of a decoded slot (ring position j of block b) into its bit-reversed tile
template <int LOGN, int LOGH, int LOGW>
EG_DEV void scatter_slot(uint32_t* S, int b, int j, int pk, int TS, uint32_t v) {
  const int flat = (b << LOGN) + brev(j, LOGN);
  const int pi = flat >> (LOGH + LOGW);
  if (pi >= pk) return;
  const int r = (flat >> LOGW) & ((1 << LOGH) - 1), c = flat & ((1 << LOGW) - 1);
  S[pi * TS + brev(r, LOGH) * ((1 << LOGW) + 1) + brev(c, LOGW)] = v;
}

// words per tile slot of the tile region (128-byte aligned)
template <int LOGH, int LOGW>
__host__ __device__ constexpr int tile_words() {
  return (int)((((size_t)(1 << LOGH) * ((1 << LOGW) + 1) * 4 + 127) & ~(size_t)127) / 4);
}

// Delta_r * m mod q_r for m < p (R == 1: exact product, Delta*(p-1) < q)
template <int R>
EG_DEV uint64_t delta_mul(const PrimeConst& pc, uint32_t m) {
  if constexpr (R == 1) {
    return mulw(lo32(pc.delta), m) + ((uint64_t)(hi32(pc.delta) * m) << 32);
  } else {
    return Bfly<Field64, 0>::fin_gs(pc.f, pc.f.mul_shoup_approx(m, pc.delta, pc.delta_shoup));
  }
}

EG_DEV uint64_t signed_mod(int32_t e, uint64_t q) { return e < 0 ? q - (uint64_t)(-(int64_t)e) : (uint64_t)e; }

template <int R>
__host__ __device__ constexpr int ct_words(int n) {
  return 2 * R * n;
}

// phi = c0 t^ + c1 (device layout) as the input view of the decryption INTT;
// reduced to [0, 4q + 2^32) for the Gentleman-Sande bounds.
struct PhiSrc {
  const uint64_t *c0, *c1, *t, *tp;
  Field64 f;
  static constexpr bool kVec = true;
  EG_DEV uint64_t at(int j) const {
    uint64_t x = f.mul_shoup_approx(c0[j], t[j], tp[j]) + c1[j];  // < 5q
    return hi32(x) > hi32(f.q4) ? x - f.q4 : x;
  }
  EG_DEV uint64_t operator()(int j) const { return at(j); }
  EG_DEV void ld2(int j, uint64_t& x, uint64_t& y) const {
    x = at(j);
    y = at(j + 1);
  }
};

// Same as PhiSrc with c0, c1, t^, t^' staged in shared memory (swizzled u64 layout,
// 16-byte paired reads).
struct PhiSrcS {
  const uint64_t *c0, *c1, *t, *tp;
  Field64 f;
  static constexpr bool kVec = true;
  EG_DEV uint64_t at(int j) const {
    const int s = sidx<uint64_t>(j);
    uint64_t x = f.mul_shoup_approx(c0[s], t[s], tp[s]) + c1[s];  // < 5q
    return hi32(x) > hi32(f.q4) ? x - f.q4 : x;
  }
  EG_DEV uint64_t operator()(int j) const { return at(j); }
  EG_DEV void ld2(int j, uint64_t& x, uint64_t& y) const {
    const int s = sidx<uint64_t>(j);
    const ulonglong2 a = *reinterpret_cast<const ulonglong2*>(c0 + s);
    const ulonglong2 b = *reinterpret_cast<const ulonglong2*>(c1 + s);
    const ulonglong2 w = *reinterpret_cast<const ulonglong2*>(t + s);
    const ulonglong2 wp = *reinterpret_cast<const ulonglong2*>(tp + s);
    x = f.mul_shoup_approx(a.x, w.x, wp.x) + b.x;
    y = f.mul_shoup_approx(a.y, w.y, wp.y) + b.y;
    x = hi32(x) > hi32(f.q4) ? x - f.q4 : x;
    y = hi32(y) > hi32(f.q4) ? y - f.q4 : y;
  }
};

// ------------------------------------------------------------ tile -> ring

// Barrier over the NT threads of thread group g (literal ids keep ptxas' barrier
// budget at 3, so several CTAs fit per SM).
struct GroupBar {
  int g, count;
  EG_DEV void sync() const {
    if (g == 0) asm volatile("bar.sync 1, %0;" ::"r"(count) : "memory");
    else asm volatile("bar.sync 2, %0;" ::"r"(count) : "memory");
  }
};

enum TileMode { TILE_ENC = 0, TILE_HOMREC = 1, TILE_WEIGHTS = 2 };

// Programmatic dependent launch (the layer's Enc -> ElementMult -> Dec chain): a kernel
// launched with programmatic stream serialization may start while its predecessor in
// the stream still runs; pdl_wait() blocks until that predecessor grid has completed
// and its writes are visible, so everything before it (table staging, key loads,
// weight tiles, launch latency) overlaps the predecessor's tail.  pdl_trigger() lets
// the dependent grid launch once every CTA of this grid has called it.  Both are no-ops
// for ordinary launches.
EG_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
EG_DEV void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Twiddle staging (TWS): a tile kernel walks three read-only tables -- the n-point
// negacyclic table over q, the one over p and the 64-point cyclic table of its 2D
// transform.  Read through L1 they were the top stall reason of the latency-bound tile
// kernels (long_scoreboard on the IMADs consuming twiddles, ~20% of Enc/Dec samples).
// With TWS one thread issues TMA bulk copies into shared memory at kernel start (one
// mbarrier), overlapping the CTA's first loads; every thread waits on the barrier before
// the first transform.  TWS = 1 stages the q table only (32 KB at n = 2048: Enc and
// HomShare CTAs still co-reside), TWS = 2 all three (49 KB: Dec).  n = 2048 only.
// Layout: q [N] x 16 B | p [N] x 8 B | cyclic [128] x 8 B.
template <int LOGN, int TWS>
__host__ __device__ constexpr size_t tw_stage_bytes() {
  return TWS == 0 ? 0 : TWS == 1 ? (size_t)(1 << LOGN) * 16 : (size_t)(1 << LOGN) * 24 + 128 * 8;
}
struct TwStage {
  const TwPair<uint64_t>* q;
  const TwPair<uint32_t>* p;
  const TwPair<uint32_t>* c;
};
template <int LOGN, int TWS>
EG_DEV TwStage tw_stage_issue(uint8_t* dst, uint64_t* bar, const TwPair<uint64_t>* q, const TwPair<uint32_t>* p,
                              const TwPair<uint32_t>* c) {
  constexpr uint32_t N = 1u << LOGN;
  TwStage s{reinterpret_cast<const TwPair<uint64_t>*>(dst), p, c};
  if constexpr (TWS == 2) {
    s.p = reinterpret_cast<const TwPair<uint32_t>*>(dst + N * 16);
    s.c = reinterpret_cast<const TwPair<uint32_t>*>(dst + N * 24);
  }
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_expect_tx(bar, (uint32_t)tw_stage_bytes<LOGN, TWS>());
    for (uint32_t off = 0; off < N * 16; off += 32768u)
      tma_bulk_g2s(dst + off, reinterpret_cast<const uint8_t*>(q) + off, min(32768u, N * 16 - off), bar);
    if constexpr (TWS == 2) {
      tma_bulk_g2s(dst + N * 16, p, N * 8, bar);
      tma_bulk_g2s(dst + N * 24, c, 128 * 8, bar);
    }
  }
  return s;
}

// One CTA per (image, channel) [ENC / HOMREC] or (out, in) filter [WEIGHTS], G thread
// groups of NT = n/8 threads; group g handles blocks b = g, g+G, ... concurrently.
// Shared: tile S (u32) + per group a ring buffer over p (u32), one over q (u64) and the
// block's Enc noise (int8, drawn two per Philox call).  The q-side epilogue (a^ draw,
// a^ t^, stores) runs as a separate coalesced loop after the NTT, not inside its
// unrolled last pass, to keep register pressure low.
// ALIAS (the fully staged single-prime variant): the p-side ring buffer lives inside
// the q-side one -- the q transform's first pass loads all of it before its first store.
template <int LOGN, int LOGH, int LOGW, int G, bool ALIAS = false>
constexpr size_t tile_enc_smem(int pk = 1) {
  return (size_t)pk * tile_words<LOGH, LOGW>() * 4 +
         G * ((((size_t)(1 << LOGN) * 8 + (ALIAS ? 0 : ssize<uint32_t>(1 << LOGN) * 4) + (1 << LOGN)) + 127) &
              ~(size_t)127);
}

template <int LOGN, int LOGH, int LOGW, int R, int TM, bool INJ, int IN_T, int G, int TWS = 0>
__global__ void __launch_bounds__(G*((1 << LOGN) >> tile_loge(LOGN)), tile_min_blocks(G*((1 << LOGN) >> tile_loge(LOGN))))
    tile_enc_kernel(LayerArgs a, const uint64_t* __restrict__ key, uint32_t key_stride,
                    const void* __restrict__ in, uint64_t* __restrict__ out) {
  static_assert(!TWS || R == 1, "twiddle staging: single prime");
  constexpr int N = 1 << LOGN, NT = N >> tile_loge(LOGN);
  constexpr int Lh = 1 << LOGH, Lw = 1 << LOGW, LS = Lw + 1;
  constexpr bool ALIAS = TWS == 2;
  static_assert(!ALIAS || R == 1, "aliased p buffer: one q transform per block");
  constexpr size_t GROUP_BYTES = (size_t)N * 8 + (ALIAS ? 0 : ssize<uint32_t>(N) * 4) + N;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  constexpr int TS = tile_words<LOGH, LOGW>();
  const int npk = TM == TILE_WEIGHTS ? 1 : a.pk;  // tiles loaded (weights: one, replicated by gather_slot)
  uint32_t* S = reinterpret_cast<uint32_t*>(smem_raw);
  const int g = threadIdx.x / NT, tid = threadIdx.x % NT;
  uint8_t* gbase = smem_raw + (size_t)npk * TS * 4 + g * ((GROUP_BYTES + 127) & ~(size_t)127);
  uint64_t* qbuf = reinterpret_cast<uint64_t*>(gbase);
  uint32_t* pbuf = ALIAS ? reinterpret_cast<uint32_t*>(qbuf) : reinterpret_cast<uint32_t*>(qbuf + N);
  int8_t* ebuf = ALIAS ? reinterpret_cast<int8_t*>(qbuf + N) : reinterpret_cast<int8_t*>(pbuf + ssize<uint32_t>(N));
  const GroupBar bar{g, NT};
  const Field32 pf = a.pp.f;
  const uint32_t p = pf.q;

  const int item = blockIdx.x;
  const int ch = item % a.cin;
  const int img = item / a.cin;  // ciphertext image (pk images from img * pk), or output channel for WEIGHTS
  const int th = TM == TILE_WEIGHTS ? a.fh : a.H, tw = TM == TILE_WEIGHTS ? a.fw : a.W;
  pdl_trigger();  // the ElementMult may launch now; its pdl_wait() covers this grid's writes
  __shared__ uint64_t tw_bar;
  TwStage tws{a.twq_fwd[0], a.twp_inv, a.twc_fwd};
  if constexpr (TWS)
    tws = tw_stage_issue<LOGN, TWS>(smem_raw + tile_enc_smem<LOGN, LOGH, LOGW, G, ALIAS>(npk), &tw_bar, a.twq_fwd[0],
                                    a.twp_inv, a.twc_fwd);

  // 1. pad into the tiles (REF pad_image / pad_residues, ntt.cpp:155-185), pk images
  for (int e = threadIdx.x; e < npk * Lh * Lw; e += blockDim.x) {
    const int pi = e >> (LOGH + LOGW), i = e & (Lh * Lw - 1);
    const int r = i >> LOGW, c = i & (Lw - 1);
    const int src_item = TM == TILE_WEIGHTS ? item : (img * npk + pi) * a.cin + ch;
    uint32_t v = 0;
    if (r < th && c < tw && (TM == TILE_WEIGHTS || img * npk + pi < a.num_images)) {
      const size_t src = ((size_t)src_item * th + r) * tw + c;
      if constexpr (TM == TILE_WEIGHTS) {
        const int32_t w = static_cast<const int32_t*>(in)[src];
        int64_t m = (int64_t)w % (int64_t)p;
        v = (uint32_t)(m < 0 ? m + p : m);  // encode_signed
      } else if constexpr (IN_T == ENSEI_IN_U8) {
        v = static_cast<const uint8_t*>(in)[src];
      } else {
        v = static_cast<const uint32_t*>(in)[src] % p;
      }
    }
    S[pi * TS + r * LS + c] = v;
  }
  __syncthreads();
  if constexpr (TWS) mbar_wait(&tw_bar, 0);
  // 2. DFT2D of each tile (rows then columns; output bit-reversed in both dims)
  for (int pi = 0; pi < npk; ++pi) tile_transform_2d<false, LOGH, LOGW>(pf, a.pp.cred, tws.c, S + pi * TS, LS);

  const uint64_t* kimg = key + (size_t)(TM == TILE_ENC ? img : 0) * key_stride;
  const int gimg = a.image_base / a.pk + img;  // stream id of the ciphertext (= the image when pk = 1)
  for (int b = g; b < a.B; b += G) {
    if constexpr (TM == TILE_ENC) {  // Enc noise e0 for this block, two CBD draws per call
      const size_t nb = (((size_t)img * a.cin + ch) * a.B + b) * N;
      const uint32_t mask = a.cbd_k >= 32 ? 0xFFFFFFFFu : ((1u << a.cbd_k) - 1u);
      for (int i2 = tid; i2 < N / 2; i2 += NT) {
        int32_t e0, e1;
        if constexpr (INJ) {
          e0 = a.inj_noise[nb + 2 * i2];
          e1 = a.inj_noise[nb + 2 * i2 + 1];
        } else {
          const Philox4 rr = philox(a.alice_key, stream_id(PURPOSE_NOISE, a.layer, gimg, ch, b), i2);
          e0 = cbd_from(rr.x, rr.y, mask);
          e1 = cbd_from(rr.z, rr.w, mask);
        }
        ebuf[2 * i2] = (int8_t)e0;
        ebuf[2 * i2 + 1] = (int8_t)e1;
      }
    }
    // 3. encode_slots: INTT_p of the block's slots (gathered from the tile)
    {
      auto src = [&](int j) { return gather_slot<LOGN, LOGH, LOGW, TM == TILE_WEIGHTS>(S, b, j, a.pk, TS); };
      SmemRW<uint32_t> dst_raw{pbuf};
      auto dst = [&](int i, uint32_t v) { dst_raw(i, Bfly<Field32, 0>::fin_gs(pf, v)); };
      ntt_inverse<Field32, uint32_t, LOGN, tile_loge(LOGN), 0, false, false>(pf, tws.p, pbuf, tid, src, dst, bar);
    }
    bar.sync();
#pragma unroll 1
    for (int r = 0; r < R; ++r) {
      const PrimeConst pc = a.pc[r];
      const Field64 f = pc.f;
      // 4. lift to q_r: Delta*m + e (ENC), Delta*m (HOMREC), centered lift (WEIGHTS)
      auto src = [&](int i) -> uint64_t {
        const uint32_t m = pbuf[sidx<uint32_t>(i)];
        if constexpr (TM == TILE_WEIGHTS) {
          return m > p / 2 ? f.q - (uint64_t)(p - m) : (uint64_t)m;  // encode_signed(decode_signed(m))
        } else {
          uint64_t x = delta_mul<R>(pc, m);
          if constexpr (TM == TILE_ENC) {
            x += signed_mod(ebuf[i], f.q);
            if (x >= f.q) x -= f.q;
          }
          return x;
        }
      };
      // 5. NTT_q in place (lazy values stay in qbuf), then the epilogue
      SmemRW<uint64_t> qs{qbuf};
      ntt_forward<Field64, uint64_t, LOGN, tile_loge(LOGN), 0, ALIAS, false>(f, TWS ? tws.q : a.twq_fwd[r], qbuf, tid,
                                                                         src, qs, bar, pc.cred);
      bar.sync();
      if constexpr (TM == TILE_WEIGHTS) {
        uint64_t* ob = out + ((((size_t)img * a.cin + ch) * a.B + b) * R + r) * N;
        for (int j = tid; j < N; j += NT) {
          const uint64_t x = Bfly<Field64, 0>::fin_ct(f, qbuf[sidx<uint64_t>(j)], pc.cred);
          ob[j] = ((x >> 30) << 32) | (x & 0x3FFFFFFFull);  // 30-bit limbs for the MAC
        }
      } else {
        uint64_t* ob = out + (((size_t)img * a.cin + ch) * a.B + b) * ct_words<R>(N);
        uint64_t* c0 = ob + (size_t)r * N;
        uint64_t* c1 = ob + (size_t)(R + r) * N;
        const uint64_t* tk = kimg + (size_t)(2 * r) * N;
        const uint64_t* tkp = tk + N;
        const uint64_t sid = stream_id(PURPOSE_AHAT, a.layer, gimg, ch, b | (r << 12));
        const size_t ab = ((((size_t)img * a.cin + ch) * a.B + b) * R + r) * N;
        for (int j = tid; j < N; j += NT) {
          const uint64_t x = Bfly<Field64, 0>::fin_ct(f, qbuf[sidx<uint64_t>(j)], pc.cred);
          if constexpr (TM == TILE_HOMREC) {
            const uint64_t y = c1[j] + x;
            c1[j] = y >= f.q ? y - f.q : y;
          } else {
            const int k = brev(j, LOGN);  // natural slot index keys the a^ stream
            const uint64_t ah = INJ ? a.inj_ahat[ab + k] : draw_uniform_q(a.alice_key, sid, k, f.q);
            uint64_t v1 = Bfly<Field64, 0>::fin_gs(f, f.mul_shoup_approx(ah, tk[j], tkp[j])) + x;
            c0[j] = ah ? f.q - ah : 0;
            c1[j] = v1 >= f.q ? v1 - f.q : v1;
          }
        }
      }
      bar.sync();
    }
  }
}


// ------------------------------------------------------- HomShare + Bob share

// One CTA per (image, out channel), G groups over the blocks.  s_B for every block is
// drawn once (two per Philox call) into shared memory; masks
// NTT_q(Delta*INTT_p(p - s_B)) go to the c1 words of the output ciphertext (device
// layout) and Bob's share = crop(IDFT2D(merge(s_B))).
template <int LOGN, int LOGH, int LOGW, int G, bool ALIAS = false>
constexpr size_t share_smem(int B) {
  return (size_t)tile_words<LOGH, LOGW>() * 4 + (size_t)B * (1 << LOGN) * 4 +
         G * ((((size_t)(1 << LOGN) * 8 + (ALIAS ? 0 : ssize<uint32_t>(1 << LOGN) * 4)) + 127) & ~(size_t)127);
}

template <int LOGN, int LOGH, int LOGW, int R, bool INJ, int G, int TWS = 0>
__global__ void __launch_bounds__(G*((1 << LOGN) >> tile_loge(LOGN)), tile_min_blocks(G*((1 << LOGN) >> tile_loge(LOGN))))
    share_kernel(LayerArgs a, uint64_t* __restrict__ mask, uint32_t* __restrict__ bob_share) {
  static_assert(!TWS || R == 1, "twiddle staging: single prime");
  constexpr int N = 1 << LOGN, NT = N >> tile_loge(LOGN);
  constexpr int Lh = 1 << LOGH, Lw = 1 << LOGW, LS = Lw + 1;
  constexpr bool ALIAS = TWS != 0;  // p buffer inside the q buffer (see tile_enc_smem)
  constexpr size_t GROUP_BYTES = (size_t)N * 8 + (ALIAS ? 0 : ssize<uint32_t>(N) * 4);
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint32_t* S = reinterpret_cast<uint32_t*>(smem_raw);
  uint32_t* sbuf = S + tile_words<LOGH, LOGW>();  // [B][N] shares
  const int g = threadIdx.x / NT, tid = threadIdx.x % NT;
  uint8_t* gbase = reinterpret_cast<uint8_t*>(sbuf + (size_t)a.B * N) + g * ((GROUP_BYTES + 127) & ~(size_t)127);
  uint64_t* qbuf = reinterpret_cast<uint64_t*>(gbase);
  uint32_t* pbuf = ALIAS ? reinterpret_cast<uint32_t*>(qbuf) : reinterpret_cast<uint32_t*>(qbuf + N);
  const GroupBar bar{g, NT};
  const Field32 pf = a.pp.f;
  const uint32_t p = pf.q;
  const int item = blockIdx.x;  // ciphertext image * cout + o
  const int o = item % a.cout, img = item / a.cout;
  const int gimg = a.image_base / a.pk + img;
  __shared__ uint64_t tw_bar;
  TwStage tws{a.twq_fwd[0], a.twp_inv, a.twc_inv};
  if constexpr (TWS)  // tables after the working buffers
    tws = tw_stage_issue<LOGN, TWS>(smem_raw + share_smem<LOGN, LOGH, LOGW, G, ALIAS>(a.B), &tw_bar, a.twq_fwd[0],
                                    a.twp_inv,
                                    a.twc_inv);
  // 1. s_B for all blocks (natural slot order)
  for (int e = threadIdx.x; e < a.B * N / 2; e += blockDim.x) {
    const int b = e / (N / 2), i2 = e % (N / 2);
    uint32_t s0, s1;
    if constexpr (INJ) {
      const size_t base = (((size_t)img * a.cout + o) * a.B + b) * N + 2 * i2;
      s0 = a.inj_share[base];
      s1 = a.inj_share[base + 1];
    } else {
      const Philox4 rr = philox(a.bob_key, stream_id(PURPOSE_SHARE, a.layer, gimg, o, b), i2);
      s0 = uniform_p_from(rr.x, rr.y, p);
      s1 = uniform_p_from(rr.z, rr.w, p);
    }
    sbuf[b * N + 2 * i2] = s0;
    sbuf[b * N + 2 * i2 + 1] = s1;
  }
  __syncthreads();
  if constexpr (TWS) mbar_wait(&tw_bar, 0);
  for (int b = g; b < a.B; b += G) {
    auto src = [&](int j) {
      const uint32_t s = sbuf[b * N + brev(j, LOGN)];
      return s == 0 ? 0u : p - s;  // (p_A - s_B) mod p_E  (REF hss.cpp:33-35)
    };
    SmemRW<uint32_t> dst_raw{pbuf};
    auto dst = [&](int i, uint32_t v) { dst_raw(i, Bfly<Field32, 0>::fin_gs(pf, v)); };
    ntt_inverse<Field32, uint32_t, LOGN, tile_loge(LOGN), 0, false, false>(pf, tws.p, pbuf, tid, src, dst, bar);
    bar.sync();
#pragma unroll 1
    for (int r = 0; r < R; ++r) {
      const PrimeConst pc = a.pc[r];
      const Field64 f = pc.f;
      auto qsrc = [&](int i) { return delta_mul<R>(pc, pbuf[sidx<uint32_t>(i)]); };
      // mask lands where c1 of the output ciphertext (img, o, b) lives
      uint64_t* mo = mask + ((size_t)item * a.B + b) * ct_words<R>(N) + (size_t)(R + r) * N;
      GlobalOut64Fwd outw{mo, f, pc.cred};
      ntt_forward<Field64, uint64_t, LOGN, tile_loge(LOGN), 0, ALIAS, false>(f, TWS ? tws.q : a.twq_fwd[r], qbuf, tid,
                                                                         qsrc, outw, bar, pc.cred);
      bar.sync();
    }
  }
  // 2. Bob's share of every image of the pack: IDFT2D of its part of the merged s_B grid,
  // cropped (REF protocol.cpp:593-602)
  for (int pi = 0; pi < a.pk && img * a.pk + pi < a.num_images; ++pi) {
    __syncthreads();
    for (int i = threadIdx.x; i < Lh * Lw; i += blockDim.x) {
      const int r = i >> LOGW, c = i & (Lw - 1);
      S[brev(r, LOGH) * LS + brev(c, LOGW)] = sbuf[pi * Lh * Lw + i];  // natural grid position i = r*Lw + c
    }
    __syncthreads();
    tile_transform_2d<true, LOGH, LOGW>(pf, a.pp.cred, tws.c, S, LS);
    uint32_t* bs = bob_share + ((size_t)(img * a.pk + pi) * a.cout + o) * a.oh * a.ow;
    for (int i = threadIdx.x; i < a.oh * a.ow; i += blockDim.x) {
      const int r = i / a.ow, c = i % a.ow;
      bs[i] = S[(r + a.r0) * LS + c + a.c0];
    }
  }
}


// Exact RNS decryption rounding (REF ringbfv.cpp:224-229 over Q = q_0 q_1 q_2): with
// y_r = phi_r (Q/q_r)^-1 mod q_r, phi = sum_r y_r M_r - k Q (M_r = Q / q_r), and
// p y_r = I_r q_r + E_r (0 <= E_r < q_r),
//   floor((p phi + floor(Q/2)) / Q) = sum_r I_r - k p + floor(F + 1/2 - 1/(2Q)),  F = sum_r E_r / q_r,
// so m = (sum_r I_r + t) mod p with t = #{t in 1..3 : 2 sum_r E_r M_r > (2t - 1) Q} (Q odd:
// no ties).  F is summed in 2^-62 fixed point (|error| < 8 ulp); only when that lands
// within 8 ulp of a rounding boundary (never for a correctly decrypting ciphertext:
// there F is within p |e| / Q of an integer) t is decided by the exact 192-bit compare.
EG_DEV uint32_t crt_round_t(const CrtConst& cc, const uint64_t (&E)[3], uint64_t Fsum, bool exact = false) {
  const uint64_t G = Fsum + (1ull << 61);
  const uint64_t low = G & ((1ull << 62) - 1);
  const uint32_t t = (uint32_t)(G >> 62);
  if (!exact && low >= 8 && low <= (1ull << 62) - 8) return t;
  uint32_t N[7] = {0, 0, 0, 0, 0, 0, 0};  // sum_r E_r M_r (< 2^182)
#pragma unroll 1
  for (int r = 0; r < 3; ++r) {
    const uint32_t e[2] = {lo32(E[r]), hi32(E[r])};
#pragma unroll 1
    for (int i = 0; i < 2; ++i) {
      uint64_t carry = 0;
#pragma unroll 1
      for (int j = 0; j < 4; ++j) {
        const uint64_t v = (uint64_t)e[i] * cc.M[r][j] + N[i + j] + carry;
        N[i + j] = (uint32_t)v;
        carry = v >> 32;
      }
      for (int k = i + 4; carry && k < 7; ++k) {
        const uint64_t v = (uint64_t)N[k] + carry;
        N[k] = (uint32_t)v;
        carry = v >> 32;
      }
    }
  }
  uint32_t N2[6];  // 2 N (< 2^183)
#pragma unroll
  for (int k = 5; k >= 0; --k) N2[k] = (N[k] << 1) | (k ? N[k - 1] >> 31 : 0);
  uint32_t tt = 0;
#pragma unroll 1
  for (int s = 0; s < 3; ++s) {
    int cmp = 0;
    for (int k = 5; k >= 0 && !cmp; --k) cmp = N2[k] > cc.T[s][k] ? 1 : (N2[k] < cc.T[s][k] ? -1 : 0);
    tt += cmp > 0;
  }
  return tt;
}

// phi_r -> (I_r, E_r, E_r / q_r in 2^-62) for one prime; phi canonical
EG_DEV void crt_part(const PrimeConst& pc, uint32_t p, uint64_t phi, uint32_t& I, uint64_t& E, uint64_t& F) {
  const Field64& f = pc.f;
  const uint64_t y = Bfly<Field64, 0>::fin_gs(f, f.mul_shoup_approx(phi, pc.crt_inv, pc.crt_inv_shoup));
  const uint64_t I0 = mulhi64(y, pc.cp);  // floor(y p / q) - {0, 1, 2}
  uint64_t rem = (uint64_t)p * y - I0 * f.q;  // < 3q, exact in 64 bits
  const uint32_t c1 = rem >= f.q, c2 = rem >= f.q2;
  rem -= (uint64_t)(c1 + c2) * f.q;
  I = (uint32_t)I0 + c1 + c2;  // < p: y < q
  E = rem;
  F = mulhi64(rem << 4, pc.crt_c);
}

// phi_r[i] = INTT_{q_r}(c0 t^ + c1)[i] by direct evaluation, O(n):
//   phi[i] = n^-1 sum_k X[k] psi^-(2k+1) i,  X[k] = c0 t^ + c1 at slot k (device layout:
// position brev(k)).  The exact-rounding fallback of dec_rns_kernel for coefficients whose
// fixed-point CRT sum lands next to a rounding boundary (never for a correctly
// decrypting ciphertext; a few milliseconds of one thread when it happens).
EG_DEV uint64_t powmod64(const PrimeConst& pc, uint64_t b, uint64_t e) {
  uint64_t r = 1;
  while (e) {
    if (e & 1) r = pc.f.mul(r, b, pc.mu_hi, pc.mu_lo);
    b = pc.f.mul(b, b, pc.mu_hi, pc.mu_lo);
    e >>= 1;
  }
  return r;
}
template <int LOGN>
EG_DEV uint64_t phi_direct(const PrimeConst& pc, uint64_t psi, const uint64_t* c0, const uint64_t* c1, const uint64_t* t,
                           int i) {
  constexpr int N = 1 << LOGN;
  const Field64& f = pc.f;
  const uint64_t q = f.q;
  const uint64_t psi_inv = powmod64(pc, psi, 2 * (uint64_t)N - 1);    // psi^-1
  uint64_t pw = powmod64(pc, psi_inv, (uint64_t)i);                  // psi^-i
  const uint64_t step = f.mul(pw, pw, pc.mu_hi, pc.mu_lo);           // psi^-2i
  uint64_t acc = 0;
  for (int k = 0; k < N; ++k) {
    const int j = brev(k, LOGN);
    const uint64_t x = f.add(f.mul(c0[j], t[j], pc.mu_hi, pc.mu_lo), c1[j]);
    acc = f.add(acc, f.mul(x, pw, pc.mu_hi, pc.mu_lo));
    pw = f.mul(pw, step, pc.mu_hi, pc.mu_lo);
  }
  const uint64_t n_inv = powmod64(pc, (uint64_t)N, q - 2);
  return f.mul(acc, n_inv, pc.mu_hi, pc.mu_lo);
}

// RNS decryption (config 4): per prime r, phi_r = INTT_{q_r}(c0 t^ + c1); per coefficient
// the CRT parts accumulate in shared memory (sum I_r: u32, sum E_r / q_r: 2^-62 fixed point,
// u64); then the exact rounding above -> m (slots) -> decode (NTT_p) -> tile -> IDFT2D ->
// crop.  Coefficients whose fixed-point sum is ambiguous recompute their three phi_r by
// direct evaluation (phi_direct) and take the 192-bit comparison.  Builder extension:
// REF has no RNS; pinned by the oracle's exact multi-limb rounding
// (eo_crt_round) and by ensei_gpu_crt_round's boundary tests.
template <int LOGN, int LOGH, int LOGW, int R>
__global__ void __launch_bounds__((1 << LOGN) >> tile_loge(LOGN))
    dec_rns_kernel(LayerArgs a, const uint64_t* __restrict__ key, uint32_t key_stride,
                   const uint64_t* __restrict__ ct, uint32_t* __restrict__ alice_share,
                   const uint32_t* __restrict__ bob_share, uint32_t* __restrict__ outp) {
  static_assert(R == 3, "exact CRT rounding: three primes");
  constexpr int N = 1 << LOGN, NT = N >> tile_loge(LOGN);
  constexpr int Lh = 1 << LOGH, Lw = 1 << LOGW, LS = Lw + 1;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  constexpr int TS = tile_words<LOGH, LOGW>();
  uint64_t* qbuf = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* fsum = qbuf + N;                                  // sum_r E_r / q_r, 2^-62
  uint32_t* pbuf = reinterpret_cast<uint32_t*>(fsum + N);     // sum_r I_r, then m
  uint32_t* S = pbuf + ssize<uint32_t>(N);                    // pk tiles, TS words apart
  const int tid = threadIdx.x;
  const CtaBar bar;
  const Field32 pf = a.pp.f;
  const uint32_t p = pf.q;
  const int item = blockIdx.x;
  const int img = item / a.cout;
  const uint64_t* kimg = key + (size_t)img * key_stride;
  for (int i = tid; i < a.pk * TS; i += NT) S[i] = 0;
  for (int b = 0; b < a.B; ++b) {
    const uint64_t* cb = ct + ((size_t)item * a.B + b) * ct_words<R>(N);
    for (int i = tid; i < N; i += NT) {
      pbuf[sidx<uint32_t>(i)] = 0;
      fsum[i] = 0;
    }
    __syncthreads();
#pragma unroll 1
    for (int r = 0; r < R; ++r) {
      const PrimeConst pc = a.pc[r];
      const Field64 f = pc.f;
      PhiSrc src{cb + (size_t)r * N, cb + (size_t)(R + r) * N, kimg + (size_t)(2 * r) * N,
                 kimg + (size_t)(2 * r + 1) * N, f};
      auto dst = [&](int i, uint64_t v) {
        uint32_t I;
        uint64_t E, F;
        crt_part(pc, p, Bfly<Field64, 0>::fin_gs(f, v), I, E, F);
        pbuf[sidx<uint32_t>(i)] += I;  // < 3p
        fsum[i] += F;
      };
      ntt_inverse<Field64, uint64_t, LOGN, tile_loge(LOGN), 0, false, false>(f, a.twq_inv[r], qbuf, tid, src, dst, bar);
      __syncthreads();
    }
    for (int i = tid; i < N; i += NT) {
      const uint64_t G = fsum[i] + (1ull << 61), low = G & ((1ull << 62) - 1);
      uint32_t t = (uint32_t)(G >> 62);
      if (low < 8 || low > (1ull << 62) - 8) {  // ambiguous: exact phi_r, exact compare
        uint64_t E[3];
        for (int r = 0; r < 3; ++r) {
          uint32_t I;
          uint64_t F;
          crt_part(a.pc[r], p,
                   phi_direct<LOGN>(a.pc[r], a.psi_q[r], cb + (size_t)r * N, cb + (size_t)(R + r) * N,
                                    kimg + (size_t)(2 * r) * N, i),
                   I, E[r], F);
        }
        t = crt_round_t(a.crt, E, 0, true);
      }
      uint32_t v = pbuf[sidx<uint32_t>(i)] + t;  // < 3p + 3
      if (v >= 2 * p) v -= 2 * p;
      if (v >= p) v -= p;
      pbuf[sidx<uint32_t>(i)] = v;
    }
    __syncthreads();
    SmemRW<uint32_t> psrc{pbuf};
    auto pdst = [&](int j, uint32_t v) {
      scatter_slot<LOGN, LOGH, LOGW>(S, b, j, a.pk, TS, reduce_lazy(pf, v, a.pp.cred));
    };
    ntt_forward<Field32, uint32_t, LOGN, tile_loge(LOGN), 0, false, false>(pf, a.twp_fwd, pbuf, tid, psrc, pdst, bar);
    __syncthreads();
  }
  const int o = item % a.cout;
  for (int pi = 0; pi < a.pk && img * a.pk + pi < a.num_images; ++pi) {  // every image of the pack
    uint32_t* St = S + pi * TS;
    tile_transform_2d<true, LOGH, LOGW>(pf, a.pp.cred, a.twc_inv, St, LS);
    const size_t base = ((size_t)(img * a.pk + pi) * a.cout + o) * a.oh * a.ow;
    for (int i = tid; i < a.oh * a.ow; i += NT) {
      const int r = i / a.ow, c = i % a.ow;
      const uint32_t s = St[(r + a.r0) * LS + c + a.c0];
      if (alice_share) alice_share[base + i] = s;
      if (outp) {
        uint32_t y = s + bob_share[base + i];
        outp[base + i] = y >= p ? y - p : y;
      }
    }
  }
}

template <int LOGN, int LOGH, int LOGW>
constexpr size_t dec_rns_smem(int pk = 1) {
  return (size_t)(1 << LOGN) * 16 + ssize<uint32_t>(1 << LOGN) * 4 + (size_t)pk * tile_words<LOGH, LOGW>() * 4;
}

// Standalone exact CRT rounding (ensei_gpu_crt_round, for the boundary tests): residues
// [count][R] -> m = round(p phi / Q) mod p, the same code path as dec_rns_kernel.
template <int R>
__global__ void crt_round_kernel(LayerArgs a, const uint64_t* __restrict__ res, size_t count,
                                 uint32_t* __restrict__ out) {
  static_assert(R == 3, "exact CRT rounding: three primes");
  const uint32_t p = a.pp.f.q;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t Isum = 0;
    uint64_t Fsum = 0, E[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      uint32_t I;
      uint64_t Fr;
      crt_part(a.pc[r], p, res[i * 3 + r], I, E[r], Fr);
      Isum += I;
      Fsum += Fr;
    }
    uint32_t v = Isum + crt_round_t(a.crt, E, Fsum);
    if (v >= 2 * p) v -= 2 * p;
    if (v >= p) v -= p;
    out[i] = v;
  }
}

// ---------------------------------------------------------------- decrypt

// One CTA per (image, out channel), G groups over the blocks: phi = c0 t^ + c1 ->
// INTT_q -> round(p phi / q) -> decode (NTT_p) -> scatter into the tile; then all
// threads: IDFT2D -> crop (-> + Bob's share).
template <int LOGN, int LOGH, int LOGW, int G>
constexpr size_t dec_smem(int pk = 1) {
  return (size_t)pk * tile_words<LOGH, LOGW>() * 4 +
         G * ((((size_t)(1 << LOGN) * 8 + ssize<uint32_t>(1 << LOGN) * 4) + 127) & ~(size_t)127);
}

// STG: the CTA's ciphertext blocks and the key are staged into shared memory with
// cp.async (swizzled) before the first INTT pass, instead of per-thread dependent global
// loads inside it (the pass was 30% of the kernel's stall samples at n = 2048).
template <int LOGN, int LOGH, int LOGW, int G, bool STG, int TWS = 0>
__global__ void __launch_bounds__(G*((1 << LOGN) >> tile_loge(LOGN)))
    dec_kernel(LayerArgs a, const uint64_t* __restrict__ key, uint32_t key_stride,
               const uint64_t* __restrict__ ct, uint32_t* __restrict__ alice_share,
               const uint32_t* __restrict__ bob_share, uint32_t* __restrict__ outp) {
  constexpr int N = 1 << LOGN, NT = N >> tile_loge(LOGN);
  constexpr int Lh = 1 << LOGH, Lw = 1 << LOGW, LS = Lw + 1;
  constexpr size_t GROUP_BYTES = (size_t)N * 8 + ssize<uint32_t>(N) * 4;
  constexpr int TS = tile_words<LOGH, LOGW>();
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint32_t* S = reinterpret_cast<uint32_t*>(smem_raw);  // pk tiles, TS words apart
  const int g = threadIdx.x / NT, tid = threadIdx.x % NT;
  uint8_t* gbase = smem_raw + (size_t)a.pk * TS * 4 + g * ((GROUP_BYTES + 127) & ~(size_t)127);
  uint64_t* qbuf = reinterpret_cast<uint64_t*>(gbase);
  uint32_t* pbuf = reinterpret_cast<uint32_t*>(qbuf + N);
  const GroupBar bar{g, NT};
  const Field32 pf = a.pp.f;
  const uint32_t p = pf.q;
  const int item = blockIdx.x;  // ciphertext image * cout + o
  const int img = item / a.cout, o = item % a.cout;
  const uint64_t* kimg = key + (size_t)img * key_stride;
  const PrimeConst pc = a.pc[0];
  const Field64 f = pc.f;
  const uint64_t cp = pc.cp, h = f.q >> 1;  // floor(p 2^64 / q), floor(q / 2)
  uint64_t* kst = reinterpret_cast<uint64_t*>(smem_raw + dec_smem<LOGN, LOGH, LOGW, G>(a.pk));  // [t^][t^'][B][c0][c1]
  __shared__ uint64_t tw_bar;
  // Bob's share for the final recombination, fetched now: HomShare finished before the
  // ElementMult started, so it is visible here, and the load latency hides behind the
  // transforms instead of stalling the crop loop (unpacked layers)
  constexpr int kBobPre = 4;
  const size_t obase = (size_t)item * a.oh * a.ow;
  uint32_t bob_pre[kBobPre];
#pragma unroll
  for (int k = 0; k < kBobPre; ++k) {
    const int i = threadIdx.x + k * blockDim.x;
    bob_pre[k] = (outp && a.pk == 1 && i < a.oh * a.ow) ? __ldg(bob_share + obase + i) : 0u;
  }
  TwStage tws{a.twq_inv[0], a.twp_fwd, a.twc_inv};
  if constexpr (TWS)  // tables after the staged arrays
    tws = tw_stage_issue<LOGN, TWS>(reinterpret_cast<uint8_t*>(kst + (STG ? (size_t)(2 + 2 * a.B) * N : 0)), &tw_bar,
                               a.twq_inv[0], a.twp_fwd, a.twc_inv);
  if constexpr (STG) {
    const uint64_t* cg = ct + (size_t)item * a.B * ct_words<1>(N);
    const int narr = 2 + 2 * a.B;  // N-word arrays: t^, t^', then c0, c1 per block
    for (int e = threadIdx.x; e < 2 * (N / 2); e += blockDim.x) {  // the key: independent of the MAC
      const int arr = e / (N / 2), c = e % (N / 2);
      cp_async16(kst + (size_t)arr * N + sidx<uint64_t>(2 * c), kimg + (size_t)arr * N + 2 * c);
    }
    cp_async_commit();
    pdl_wait();  // the ElementMult's output ciphertexts
    for (int e = threadIdx.x + 2 * (N / 2); e < narr * (N / 2); e += blockDim.x) {
      const int arr = e / (N / 2), c = e % (N / 2);
      cp_async16(kst + (size_t)arr * N + sidx<uint64_t>(2 * c), cg + (size_t)(arr - 2) * N + 2 * c);
    }
    cp_async_commit();
    cp_async_wait_all();
  } else {
    pdl_wait();
  }
  __syncthreads();
  if constexpr (TWS) mbar_wait(&tw_bar, 0);
  for (int b = g; b < a.B; b += G) {
    const uint64_t* cb = ct + ((size_t)item * a.B + b) * ct_words<1>(N);
    auto run_inv = [&](auto& src) {
    auto dst = [&](int i, uint64_t v) {
      const uint64_t phi = Bfly<Field64, 0>::fin_gs(f, v);
      // exact floor((p phi + floor(q/2)) / q) (REF ringbfv.cpp:224-229): the estimate
      // Q = floor(phi cp / 2^64) is at most 2 below, so the remainder is < 3q and exact
      // in 64-bit arithmetic; the correction is [rem >= q] + [rem >= 2q].  phi < q bounds
      // the rounded quotient by p, so Q mod p is one conditional subtraction (the generic
      // 64-bit % p was a divergent reciprocal / division-call sequence per coefficient).
      const uint64_t Q = mulhi64(phi, cp);
      const uint64_t rem = (uint64_t)p * phi + h - Q * f.q;
      const uint32_t Qs = (uint32_t)Q + (rem >= f.q) + (rem >= f.q2);
      pbuf[sidx<uint32_t>(i)] = Qs >= p ? Qs - p : Qs;
    };
    ntt_inverse<Field64, uint64_t, LOGN, tile_loge(LOGN), 0, false, false>(f, tws.q, qbuf, tid, src, dst, bar);
    };
    if constexpr (STG) {
      PhiSrcS src{kst + (size_t)(2 + 2 * b) * N, kst + (size_t)(3 + 2 * b) * N, kst, kst + N, f};
      run_inv(src);
    } else {
      PhiSrc src{cb, cb + N, kimg, kimg + N, f};
      run_inv(src);
    }
    bar.sync();
    // decode_slots (NTT_p) -> scatter into the bit-reversed tile
    SmemRW<uint32_t> psrc{pbuf};
    auto pdst = [&](int j, uint32_t v) {
      scatter_slot<LOGN, LOGH, LOGW>(S, b, j, a.pk, TS, reduce_lazy(pf, v, a.pp.cred));
    };
    ntt_forward<Field32, uint32_t, LOGN, tile_loge(LOGN), 0, false, false>(pf, tws.p, pbuf, tid, psrc, pdst, bar);
    bar.sync();
  }
  __syncthreads();
  if (a.pk > 1) {  // packed: IDFT2D + crop (+ recombine) of every image of the pack
    for (int pi = 0; pi < a.pk && img * a.pk + pi < a.num_images; ++pi) {
      uint32_t* St = S + pi * TS;
      tile_transform_2d<true, LOGH, LOGW>(pf, a.pp.cred, tws.c, St, LS);
      const size_t base = ((size_t)(img * a.pk + pi) * a.cout + o) * a.oh * a.ow;
      for (int i = threadIdx.x; i < a.oh * a.ow; i += blockDim.x) {
        const int r = i / a.ow, c = i % a.ow;
        const uint32_t s = St[(r + a.r0) * LS + c + a.c0];
        if (alice_share) alice_share[base + i] = s;
        if (outp) {
          uint32_t y = s + bob_share[base + i];
          outp[base + i] = y >= p ? y - p : y;
        }
      }
    }
    return;
  }
  // IDFT2D + crop (+ recombine with Bob's share)
  tile_transform_2d<true, LOGH, LOGW>(pf, a.pp.cred, tws.c, S, LS);
  int k = 0;
  for (int i = threadIdx.x; i < a.oh * a.ow; i += blockDim.x, ++k) {
    const int r = i / a.ow, c = i % a.ow;
    const uint32_t s = S[(r + a.r0) * LS + c + a.c0];
    if (alice_share) alice_share[obase + i] = s;
    if (outp) {
      uint32_t bv = bob_pre[0];
#pragma unroll
      for (int u = 1; u < kBobPre; ++u)
        if (k == u) bv = bob_pre[u];
      if (k >= kBobPre) bv = bob_share[obase + i];
      uint32_t y = s + bv;
      outp[obase + i] = y >= p ? y - p : y;
    }
  }
}


// ------------------------------------------------------------ ElementMult

// Z = A2 2^60 + A1 2^30 + A0 (A0, A1 < 2^63, A2 < 2^63) -> Z mod q, canonical.
// Z = hi 2^64 + lo; lo -> [0,3q) by corr, hi * (2^64 mod q) by Shoup (< 4q).
EG_DEV uint64_t mac_reduce(const Field64& f, const PrimeConst& pc, uint64_t a0, uint64_t a1, uint64_t a2) {
  constexpr uint64_t M30 = (1ull << 30) - 1;
  a1 += a0 >> 30;
  a0 &= M30;
  a2 += a1 >> 30;
  a1 &= M30;
  const uint64_t lo = (a2 << 60) | (a1 << 30) | a0, hi = a2 >> 4;
  uint64_t x = Bfly<Field64, 0>::corr(f, lo, pc.cred);
  if (hi) x += f.mul_shoup_approx(hi, pc.c64, pc.c64p);  // < 7q
  return Bfly<Field64, 0>::fin_ct(f, x, pc.cred);
}

// Per slot s (ring position of one (block, prime)), the rows (img, comp) times
// cols (out channel) product over K = cin:  out = sum_c ct[img][c][comp] w[o][c]
// (mod q), + the HomShare mask already sitting in out's c1 words.  Lazy accumulation
// with 30-bit limbs: for x, y < 2^60, x = x1 2^30 + x0, y = y1 2^30 + y0;
// A0 += x0 y0, A1 += x0 y1 + x1 y0, A2 += x1 y1 (four full-rate mad.wide per MAC, no
// carries), folded every 7 channels, fully reduced every a2_chunk channels, reduced
// once per output.  CTA tile = S slots x MT rows x NT cols; shared tiles [k][row][slot]
// (slot-contiguous) are filled with 16-byte cp.async, double-buffered over K chunks,
// so every ct / weight word crosses HBM once per CTA.
template <int R, int S, int MT, int NT, int KT, int TM, int TN>
__global__ void __launch_bounds__(S*(MT / TM) * (NT / TN))
    mac_kernel(LayerArgs a, int logn, const uint64_t* __restrict__ ct, const uint64_t* __restrict__ w,
               int has_mask, uint64_t* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  constexpr int NTH = S * (MT / TM) * (NT / TN);
  constexpr int SV = S / 2;  // 16-byte chunks per (k, row)
  extern __shared__ __align__(16) uint64_t smac[];
  uint64_t* As = smac;                     // [2][KT][MT][S]
  uint64_t* Bs = smac + 2 * KT * MT * S;   // [2][KT][NT][S]
  const int n = 1 << logn;
  const int s0 = blockIdx.x * S;           // first slot of this CTA over B*R*n
  const int bp = s0 >> logn;               // (block, prime) pair index
  const int b = bp / R, r = bp % R;
  const int k0 = s0 & (n - 1);
  const int rows = 2 * a.num_images, cols = a.cout, K = a.cin;
  const int row0 = blockIdx.y * MT, col0 = blockIdx.z * NT;
  const int tid = threadIdx.x;
  const int sl = tid % S, tm = (tid / S) % (MT / TM), tn = tid / (S * (MT / TM));
  const PrimeConst pc = a.pc[r];
  const Field64 f = pc.f;
  const size_t ctw = (size_t)ct_words<R>(n);
  const size_t chan_stride = (size_t)a.B * ctw;        // ct: next channel
  const size_t w_chan = (size_t)a.B * R * n;            // w: next input channel
  constexpr uint64_t M30 = (1ull << 30) - 1;

  auto load_chunk = [&](int buf, int kc) {
    uint64_t* Ab = As + buf * KT * MT * S;
    uint64_t* Bb = Bs + buf * KT * NT * S;
    for (int e = tid; e < KT * MT * SV; e += NTH) {
      const int v = e % SV, row = (e / SV) % MT, kk = e / (SV * MT);
      const int gr = row0 + row, c = kc + kk;
      uint64_t* dst = Ab + (kk * MT + row) * S + 2 * v;
      if (gr < rows && c < K) {
        const uint64_t* src = ct + ((size_t)(gr >> 1) * a.cin + c) * chan_stride + (size_t)b * ctw +
                              (size_t)((gr & 1) * R + r) * n + k0 + 2 * v;
        cp_async16(dst, src);
      } else {
        dst[0] = 0;
        dst[1] = 0;
      }
    }
    for (int e = tid; e < KT * NT * SV; e += NTH) {
      const int v = e % SV, col = (e / SV) % NT, kk = e / (SV * NT);
      const int go = col0 + col, c = kc + kk;
      uint64_t* dst = Bb + (kk * NT + col) * S + 2 * v;
      if (go < cols && c < K) {
        cp_async16(dst, w + ((size_t)go * a.cin + c) * w_chan + (size_t)bp * n + k0 + 2 * v);
      } else {
        dst[0] = 0;
        dst[1] = 0;
      }
    }
    cp_async_commit();
  };

  uint64_t A0[TM][TN], A1[TM][TN], A2[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) A0[i][j] = A1[i][j] = A2[i][j] = 0;
  int since_fold = 0, since_full = 0;
  const int nchunks = (K + KT - 1) / KT;
  load_chunk(0, 0);
  for (int ch = 0; ch < nchunks; ++ch) {
    const int buf = ch & 1;
    if (ch + 1 < nchunks) {
      load_chunk(buf ^ 1, (ch + 1) * KT);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    } else {
      cp_async_wait_all();
    }
    __syncthreads();
    const uint64_t* Ab = As + buf * KT * MT * S;
    const uint64_t* Bb = Bs + buf * KT * NT * S;
    const int kmax = min(KT, K - ch * KT);
    for (int kk = 0; kk < kmax; ++kk) {
      uint32_t x0[TM], x1[TM], y0[TN], y1[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) {
        const uint64_t v = Ab[(kk * MT + tm * TM + i) * S + sl];
        x0[i] = (uint32_t)(v & M30);
        x1[i] = (uint32_t)(v >> 30);
      }
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const uint64_t v = Bb[(kk * NT + tn * TN + j) * S + sl];
        y0[j] = lo32(v);
        y1[j] = hi32(v);
      }
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) {
          // accumulate in place (one IMAD.WIDE.U32 each, accumulator stays a register pair)
          asm("mad.wide.u32 %0, %3, %5, %0;\n\t"
              "mad.wide.u32 %1, %3, %6, %1;\n\t"
              "mad.wide.u32 %1, %4, %5, %1;\n\t"
              "mad.wide.u32 %2, %4, %6, %2;"
              : "+l"(A0[i][j]), "+l"(A1[i][j]), "+l"(A2[i][j])
              : "r"(x0[i]), "r"(x1[i]), "r"(y0[j]), "r"(y1[j]));
        }
      ++since_fold;
      ++since_full;
      if (since_fold == 7) {  // A1 gains < 2^61 per channel: fold before overflow
        since_fold = 0;
        if (since_full >= (int)pc.a2_chunk) {  // top limb near capacity: reduce mod q
          since_full = 0;
#pragma unroll
          for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < TN; ++j) {
              const uint64_t z = mac_reduce(f, pc, A0[i][j], A1[i][j], A2[i][j]);
              A0[i][j] = z & M30;
              A1[i][j] = z >> 30;
              A2[i][j] = 0;
            }
        } else {
#pragma unroll
          for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < TN; ++j) {
              A1[i][j] += A0[i][j] >> 30;
              A0[i][j] &= M30;
              A2[i][j] += A1[i][j] >> 30;
              A1[i][j] &= M30;
            }
        }
      }
    }
    __syncthreads();  // this buffer is refilled two chunks later
  }
  const int k = k0 + sl;
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int gr = row0 + tm * TM + i;
    if (gr >= rows) continue;
    const int img = gr >> 1, comp = gr & 1;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int go = col0 + tn * TN + j;
      if (go >= cols) continue;
      uint64_t x = mac_reduce(f, pc, A0[i][j], A1[i][j], A2[i][j]);
      const size_t oa = ((size_t)img * a.cout + go) * chan_stride + (size_t)b * ctw + (size_t)(comp * R + r) * n + k;
      if (comp == 1 && has_mask) {  // HomShare mask written in place by share_kernel
        x += out[oa];
        x = x >= f.q ? x - f.q : x;
      }
      out[oa] = x;
    }
  }
}

// Karatsuba ElementMult (the production MAC).  Same per-slot product as mac_kernel,
// three IMAD.WIDE per MAC instead of four: with x = x1 2^30 + x0, y = y1 2^30 + y0,
//   x y = P0 + 2^30 (Pm - P0 - P2) + 2^60 P2,  P0 = x0 y0, P2 = x1 y1,
//   Pm = (x0 + x1)(y0 + y1)  (< 2.27 2^60 since x1, y1 < 2^29.01 for q < 2^59.01).
// Each of S0 = sum P0, Sm = sum Pm, S2 = sum P2 is kept exactly as H 2^50 + L (L a
// 64-bit accumulator, H a 32-bit word: H < K 2^11.2): products accumulate into L, and
// L's bits >= 50 move into H every 6 / 12 / 60 channels for Sm / S0 / S2 (headroom
// after a fold: 2^50 + 6 Pm, 12 P0, 60 P2 all < 2^64).  The epilogue rebuilds the
// exact u128 sum T = sum x y (< 2^128 while K <= 1008) and reduces it once; longer K
// flushes T mod q into the output word every 1008 channels and accumulates there.
// Measured on B200: IMAD.WIDE costs 4 fmaheavy cycles per warp, IADD3 2 ALU cycles, the
// pipes co-issue, so the fmaheavy floor drops from 20 to 12 cycles per MAC.
//
// Work: tiles = (S-slot group) x (MT-row tile) x (NT-col tile), rows/cols fastest so
// concurrently running CTAs share the slot group's ct and weight words in L2.  The grid
// is persistent; each CTA walks its tiles' K chunks as one flat sequence with a
// STAGES-deep cp.async ring, so the next tile's loads overlap this tile's epilogue
// (small-K layers are otherwise pure load latency).
constexpr int kKaraMaxK = 1008;
constexpr uint64_t kKaraLowBits = 50;  // S = H 2^50 + L: L < 2^50 after a fold, H < K 2^11.2

// T = S0 + 2^30 (Sm - S0 - S2) + 2^60 S2 (exact, < 2^128 while K <= 1008) from the split
// sums S = H 2^50 + L (L = lh:ll), as four 32-bit limbs with explicit carry chains --
// S0, Sm, S2 and D = Sm - S0 - S2 take three limbs (< 2^82), the shifts are funnel
// shifts -- then T mod q = corr(T_lo) + Shoup(T_hi, 2^64 mod q), made canonical.
// ~60 instructions; the generic u128 expression compiled to ~115.
EG_DEV uint64_t kara_T_mod(const Field64& f, const PrimeConst& pc, uint32_t l0l, uint32_t l0h, uint32_t h0,
                           uint32_t lml, uint32_t lmh, uint32_t hm, uint32_t l2l, uint32_t l2h, uint32_t h2) {
  uint32_t t0, t1, t2, t3;
  asm("{\n\t"
      ".reg .u32 a1, a2, m1, m2, b1, b2, d0, d1, d2, e0, e1, e2, e3, f1, f2, f3, u;\n\t"
      // S0 = [%4, a1, a2], Sm = [%7, m1, m2], S2 = [%10, b1, b2]: H 2^50 = limb1 += H << 18, limb2 += H >> 14
      "shl.b32 u, %5, 18;\n\t"
      "add.cc.u32 a1, %6, u;\n\t"
      "shr.b32 u, %5, 14;\n\t"
      "addc.u32 a2, u, 0;\n\t"
      "shl.b32 u, %8, 18;\n\t"
      "add.cc.u32 m1, %9, u;\n\t"
      "shr.b32 u, %8, 14;\n\t"
      "addc.u32 m2, u, 0;\n\t"
      "shl.b32 u, %11, 18;\n\t"
      "add.cc.u32 b1, %12, u;\n\t"
      "shr.b32 u, %11, 14;\n\t"
      "addc.u32 b2, u, 0;\n\t"
      // D = Sm - S0 - S2 (>= 0: the cross terms x0 y1 + x1 y0)
      "sub.cc.u32 d0, %7, %4;\n\t"
      "subc.cc.u32 d1, m1, a1;\n\t"
      "subc.u32 d2, m2, a2;\n\t"
      "sub.cc.u32 d0, d0, %10;\n\t"
      "subc.cc.u32 d1, d1, b1;\n\t"
      "subc.u32 d2, d2, b2;\n\t"
      // E = D << 30 (D < 2^71), F = S2 << 60 (S2 < 2^68)
      "shl.b32 e0, d0, 30;\n\t"
      "shf.l.clamp.b32 e1, d0, d1, 30;\n\t"
      "shf.l.clamp.b32 e2, d1, d2, 30;\n\t"
      "shr.b32 e3, d2, 2;\n\t"
      "shl.b32 f1, %10, 28;\n\t"
      "shf.l.clamp.b32 f2, %10, b1, 28;\n\t"
      "shf.l.clamp.b32 f3, b1, b2, 28;\n\t"
      // T = S0 + E + F
      "add.cc.u32 %0, %4, e0;\n\t"
      "addc.cc.u32 %1, a1, e1;\n\t"
      "addc.cc.u32 %2, a2, e2;\n\t"
      "addc.u32 %3, e3, 0;\n\t"
      "add.cc.u32 %1, %1, f1;\n\t"
      "addc.cc.u32 %2, %2, f2;\n\t"
      "addc.u32 %3, %3, f3;\n\t"
      "}"
      : "=r"(t0), "=r"(t1), "=r"(t2), "=r"(t3)
      : "r"(l0l), "r"(h0), "r"(l0h), "r"(lml), "r"(hm), "r"(lmh), "r"(l2l), "r"(h2), "r"(l2h));
  const uint64_t lo = ((uint64_t)t1 << 32) | t0, hi = ((uint64_t)t3 << 32) | t2;
  const uint64_t x = Bfly<Field64, 0>::corr(f, lo, pc.cred) + f.mul_shoup_approx(hi, pc.c64, pc.c64p);  // < 7q
  return Bfly<Field64, 0>::fin_ct(f, x, pc.cred);
}

template <int S, int MT, int NT, int KT, int STAGES>
constexpr size_t mac_kara_smem() {
  return (size_t)STAGES * KT * (MT + NT) * S * sizeof(uint64_t);
}

template <int R, int S, int MT, int NT, int KT, int TM, int TN, int STAGES>
__global__ void __launch_bounds__(S*(MT / TM) * (NT / TN), (512 / (S * (MT / TM) * (NT / TN))) > 1 ? 512 / (S * (MT / TM) * (NT / TN)) : 1)
    mac_kara_kernel(LayerArgs a, int logn, const uint64_t* __restrict__ ct, const uint64_t* __restrict__ w,
                    int has_mask, uint64_t* __restrict__ out, uint32_t zero) {
  static_assert(KT % 6 == 0 && kKaraMaxK % KT == 0, "K chunk: whole fold blocks dividing 1008");
  static_assert(TM == 2, "thread rows = the two components of one image");
  constexpr int NTH = S * (MT / TM) * (NT / TN);
  constexpr int SV = S / 2;
  constexpr int STAGE_WORDS = KT * (MT + NT) * S;
  extern __shared__ __align__(16) uint64_t smac[];
  const int n = 1 << logn;
  const int rows = 2 * a.num_images, cols = a.cout, K = a.cin;
  const int nrt = (rows + MT - 1) / MT, nct = (cols + NT - 1) / NT;
  const int tiles_per_group = nrt * nct;
  const int ntiles = (a.B * R * n / S) * tiles_per_group;
  const int nchunks = (K + KT - 1) / KT;
  const int my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int nsteps = my_tiles * nchunks;
  pdl_wait();     // ciphertexts from Enc / HomRec, masks from HomShare
  pdl_trigger();  // Dec may launch and stage its tables and key meanwhile
  const int tid = threadIdx.x;
  const int sl = tid % S, tm = (tid / S) % (MT / TM), tn = tid / (S * (MT / TM));
  const size_t ctw = (size_t)ct_words<R>(n);
  const size_t chan_stride = (size_t)a.B * ctw;
  const size_t w_chan = (size_t)a.B * R * n;
  constexpr uint64_t M30 = (1ull << 30) - 1;
  constexpr uint64_t kLowMask = (1ull << kKaraLowBits) - 1;

  struct Tile {
    int b, r, k0, row0, col0;
    const uint64_t* a_base;  // ct words of (row0, channel 0, block b, prime r, slot k0)
    const uint64_t* w_base;  // weight words of (col0, channel 0, pair bp, slot k0)
  };
  // tile decode (runtime divisions): once per tile on each side, not per K chunk
  auto tile_of = [&](int j) {
    const int t = blockIdx.x + j * gridDim.x;
    const int g = t / tiles_per_group, rem = t % tiles_per_group;
    const int s0 = g * S, bp = s0 >> logn;
    Tile tl;
    tl.b = bp / R;
    tl.r = bp % R;
    tl.k0 = s0 & (n - 1);
    tl.row0 = (rem % nrt) * MT;
    tl.col0 = (rem / nrt) * NT;
    tl.a_base = ct + (size_t)(tl.row0 >> 1) * a.cin * chan_stride + (size_t)tl.b * ctw + (size_t)tl.r * n + tl.k0;
    tl.w_base = w + (size_t)tl.col0 * a.cin * w_chan + (size_t)bp * n + tl.k0;
    return tl;
  };
  Tile ld = tile_of(0);
  int ld_j = 0, ld_c = 0;  // next (tile, chunk) to load
  // Each thread's 16-byte copies: fixed (row, v) and (col, v), channel kk0 + m*KSTEP, so a
  // step's addresses are one base pointer plus a per-channel stride (no index decoding).
  constexpr int A_KSTEP = NTH / (SV * MT), B_KSTEP = NTH / (SV * NT);
  static_assert(NTH % (SV * MT) == 0 && NTH % (SV * NT) == 0, "copy mapping");
  const int a_v = tid % SV, a_row = (tid / SV) % MT, a_kk0 = tid / (SV * MT);
  const int b_col = (tid / SV) % NT, b_kk0 = tid / (SV * NT);
  const size_t a_off = (size_t)((a_row >> 1) * a.cin + a_kk0) * chan_stride + (a_row & 1) * R * n + 2 * a_v;
  const size_t b_off = (size_t)(b_col * a.cin + b_kk0) * w_chan + 2 * a_v;
  auto load_step = [&](int step) {
    if (step < nsteps) {
      const int kc = ld_c * KT;
      uint64_t* Ab = smac + (step % STAGES) * STAGE_WORDS;
      uint64_t* Bb = Ab + KT * MT * S;
      const bool a_ok = ld.row0 + a_row < rows, b_ok = ld.col0 + b_col < cols;
      const uint64_t* as = ld.a_base + (size_t)kc * chan_stride + a_off;
      const uint64_t* ws = ld.w_base + (size_t)kc * w_chan + b_off;
#pragma unroll
      for (int kk = a_kk0, m = 0; m < (KT + A_KSTEP - 1) / A_KSTEP; ++m, kk += A_KSTEP) {
        if (kk >= KT) break;  // KT need not be a multiple of the copy stride
        uint64_t* dst = Ab + (kk * MT + a_row) * S + 2 * a_v;
        if (a_ok && kc + kk < K) {
          cp_async16(dst, as + (size_t)m * A_KSTEP * chan_stride);
        } else {
          dst[0] = 0;
          dst[1] = 0;
        }
      }
#pragma unroll
      for (int kk = b_kk0, m = 0; m < (KT + B_KSTEP - 1) / B_KSTEP; ++m, kk += B_KSTEP) {
        if (kk >= KT) break;
        uint64_t* dst = Bb + (kk * NT + b_col) * S + 2 * a_v;
        if (b_ok && kc + kk < K) {
          cp_async16(dst, ws + (size_t)m * B_KSTEP * w_chan);
        } else {
          dst[0] = 0;
          dst[1] = 0;
        }
      }
      if (++ld_c == nchunks) {
        ld_c = 0;
        if (++ld_j < my_tiles) ld = tile_of(ld_j);
      }
    }
    cp_async_commit();  // empty groups keep the wait_group count uniform
  };

  // L split into 32-bit halves (not a register pair): the carry-chained multiply-add
  // then updates the accumulator in place, with no pair-rotation moves
  uint32_t L0l[TM][TN], L0h[TM][TN], Lml[TM][TN], Lmh[TM][TN], L2l[TM][TN], L2h[TM][TN];
  uint32_t H0[TM][TN], Hm[TM][TN], H2[TM][TN];
  auto zero_acc = [&]() {
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        L0l[i][j] = L0h[i][j] = Lml[i][j] = Lmh[i][j] = L2l[i][j] = L2h[i][j] = 0;
        H0[i][j] = Hm[i][j] = H2[i][j] = 0;
      }
  };
  // exact T = sum x y from the split sums, reduced mod q (kara_T_mod: 32-bit limb chains)
  auto reduce_T = [&](const Field64& f, const PrimeConst& pc, int i, int j) -> uint64_t {
    return kara_T_mod(f, pc, L0l[i][j], L0h[i][j], H0[i][j], Lml[i][j], Lmh[i][j], Hm[i][j], L2l[i][j], L2h[i][j],
                      H2[i][j]);
  };

#pragma unroll 1
  for (int st = 0; st < STAGES - 1; ++st) load_step(st);
  zero_acc();
  int blocks = 0, kdone = 0, flushes = 0;
  Tile cm = tile_of(0);
  int cm_j = 0, cm_c = 0;  // (tile, chunk) being computed
#pragma unroll 1
  for (int step = 0; step < nsteps; ++step) {
    load_step(step + STAGES - 1);
    asm volatile("cp.async.wait_group %0;\n" ::"n"(STAGES - 1) : "memory");
    __syncthreads();
    const uint64_t* Ab = smac + (step % STAGES) * STAGE_WORDS;
    const uint64_t* Bb = Ab + KT * MT * S;
    const int kmax = min(KT, K - cm_c * KT);
    // one channel pair: six products per output into the three split sums
    auto pair = [&](int kk) {
      uint32_t xl[2][TM], xh[2][TM], xs[2][TM], yl[2][TN], yh[2][TN], ys[2][TN];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
#pragma unroll
        for (int i = 0; i < TM; ++i) {
          const uint64_t v = Ab[((kk + u) * MT + tm * TM + i) * S + sl];
          xl[u][i] = (uint32_t)(v & M30);
          xh[u][i] = (uint32_t)(v >> 30);
          xs[u][i] = xl[u][i] + xh[u][i] + zero;  // 3-input: an ALU IADD3, not an fmaheavy IMAD
        }
#pragma unroll
        for (int j = 0; j < TN; ++j) {
          const uint64_t v = Bb[((kk + u) * NT + tn * TN + j) * S + sl];
          yl[u][j] = lo32(v);
          yh[u][j] = hi32(v);
          ys[u][j] = yl[u][j] + yh[u][j] + zero;
        }
      }
      // k-parity outer: consecutive updates of one accumulator are 3*TM*TN products
      // apart, so ptxas keeps IMAD.WIDE with the accumulator as addend (2 register
      // reads per bank, no 3-input IADD3 of pair-aligned words)
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j)
            asm("mad.lo.cc.u32 %0, %6, %7, %0;\n\tmadc.hi.u32 %1, %6, %7, %1;\n\t"
                "mad.lo.cc.u32 %2, %8, %9, %2;\n\tmadc.hi.u32 %3, %8, %9, %3;\n\t"
                "mad.lo.cc.u32 %4, %10, %11, %4;\n\tmadc.hi.u32 %5, %10, %11, %5;"
                : "+r"(L0l[i][j]), "+r"(L0h[i][j]), "+r"(Lml[i][j]), "+r"(Lmh[i][j]), "+r"(L2l[i][j]), "+r"(L2h[i][j])
                : "r"(xl[u][i]), "r"(yl[u][j]), "r"(xs[u][i]), "r"(ys[u][j]), "r"(xh[u][i]), "r"(yh[u][j]));
    };
    int kk = 0;
#pragma unroll 1
    for (; kk + 6 <= kmax; kk += 6) {  // Sm headroom: 7 products -> fold every 6 channels
#pragma unroll
      for (int u = 0; u < 3; ++u) pair(kk + 2 * u);
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) {
          Hm[i][j] += Lmh[i][j] >> (kKaraLowBits - 32);
          Lmh[i][j] &= (uint32_t)(kLowMask >> 32);
        }
      if (++blocks % 2 == 0) {  // S0: 15 products
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) {
            H0[i][j] += L0h[i][j] >> (kKaraLowBits - 32);
            L0h[i][j] &= (uint32_t)(kLowMask >> 32);
          }
        if (blocks == 10) {  // S2: 63 products
          blocks = 0;
#pragma unroll
          for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < TN; ++j) {
              H2[i][j] += L2h[i][j] >> (kKaraLowBits - 32);
              L2h[i][j] &= (uint32_t)(kLowMask >> 32);
            }
        }
      }
    }
    // last chunk only: < 3 pairs, zero-filled odd tail; straight-line (a rolled loop here
    // rotates every accumulator pair through IMAD.MOV at each back edge)
    if (kk < kmax) pair(kk);
    if (kk + 2 < kmax) pair(kk + 2);
    if (kk + 4 < kmax) pair(kk + 4);
    kdone += KT;
    const bool last = cm_c == nchunks - 1;
    if (last || kdone == kKaraMaxK) {  // flush: out = (mask | previous partial) + T mod q
      const PrimeConst pc = a.pc[cm.r];
      const Field64 f = pc.f;
      // rows row0 + 2 tm + i: image row0/2 + tm, component i (TM == 2)
      const int img = (cm.row0 >> 1) + tm, go0 = cm.col0 + tn * TN;
      uint64_t* ob = out + ((size_t)img * a.cout + go0) * chan_stride + (size_t)cm.b * ctw + (size_t)cm.r * n +
                     cm.k0 + sl;
      const bool row_ok = 2 * img < rows;
      uint64_t prev[TM][TN];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) {
          prev[i][j] = 0;
          if (row_ok && go0 + j < cols && (flushes > 0 || (i == 1 && has_mask)))
            prev[i][j] = ob[(size_t)j * chan_stride + (size_t)i * R * n];
        }
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j)
          if (row_ok && go0 + j < cols) ob[(size_t)j * chan_stride + (size_t)i * R * n] = f.add(reduce_T(f, pc, i, j), prev[i][j]);
      zero_acc();
      blocks = 0;
      kdone = 0;
      flushes = last ? 0 : flushes + 1;
    }
    if (++cm_c == nchunks) {
      cm_c = 0;
      if (++cm_j < my_tiles) cm = tile_of(cm_j);
    }
    __syncthreads();  // this stage's buffer is refilled STAGES-1 steps later
  }
  cp_async_wait_all();
}

// ElementMult for tiny channel counts (config 0's 1 -> 1 layer): the tile GEMM would leave
// most of its 16-column tiles and its 12/24-channel K chunks empty and pay the u128
// epilogue per single product.  One thread per (image, block, prime, slot) computes every
// (out channel, component) output of that slot directly: exact u128 sum of cin products
// (cin (q-1)^2 < 2^128), one reduction, + the HomShare mask on c1.  Consecutive threads
// touch consecutive slots (coalesced); the kernel is HBM-bound.
template <int R>
__global__ void __launch_bounds__(256)
    mac_direct_kernel(LayerArgs a, int logn, const uint64_t* __restrict__ ct, const uint64_t* __restrict__ w,
                      int has_mask, uint64_t* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  typedef unsigned __int128 u128;
  const int n = 1 << logn;
  const size_t slots = (size_t)a.B * R * n;  // per image: (block, prime, slot)
  const size_t total = (size_t)a.num_images * slots;
  const size_t ctw = (size_t)ct_words<R>(n);
  const size_t chan_stride = (size_t)a.B * ctw;
  for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (size_t)gridDim.x * blockDim.x) {
    const size_t img = t / slots, rem = t % slots;
    const int bp = (int)(rem >> logn), sl = (int)(rem & (n - 1));
    const int b = bp / R, r = bp % R;
    const PrimeConst pc = a.pc[r];
    const Field64 f = pc.f;
    const uint64_t* xb = ct + img * a.cin * chan_stride + (size_t)b * ctw + (size_t)r * n + sl;
    const uint64_t* wb = w + (size_t)bp * n + sl;
    uint64_t* ob = out + img * a.cout * chan_stride + (size_t)b * ctw + (size_t)r * n + sl;
    for (int o = 0; o < a.cout; ++o) {
      u128 T0 = 0, T1 = 0;
      for (int c = 0; c < a.cin; ++c) {
        const uint64_t v = wb[((size_t)o * a.cin + c) * a.B * R * n];
        const uint64_t y = (v & 0x3FFFFFFFull) | ((v >> 32) << 30);  // unpack the MAC limb format
        T0 += (u128)xb[(size_t)c * chan_stride] * y;
        T1 += (u128)xb[(size_t)c * chan_stride + (size_t)R * n] * y;
      }
      uint64_t res[2];
      const u128 T[2] = {T0, T1};
#pragma unroll
      for (int comp = 0; comp < 2; ++comp) {
        uint64_t x = Bfly<Field64, 0>::corr(f, (uint64_t)T[comp], pc.cred);
        const uint64_t hi = (uint64_t)(T[comp] >> 64);
        if (hi) x += f.mul_shoup_approx(hi, pc.c64, pc.c64p);
        res[comp] = Bfly<Field64, 0>::fin_ct(f, x, pc.cred);
      }
      uint64_t* oo = ob + (size_t)o * chan_stride;
      oo[0] = res[0];
      oo[(size_t)R * n] = has_mask ? f.add(res[1], oo[(size_t)R * n]) : res[1];
    }
  }
}

template <int S, int MT, int NT, int KT>
constexpr size_t mac_smem() {
  return (size_t)2 * KT * (MT + NT) * S * sizeof(uint64_t);
}

}  // namespace ensei_gpu
