// layer_launch.cuh -- host launchers of the fused layer kernels, templated on the
// ring degree and instantiated once per degree (layer_n11.cu / n12 / n13) so the
// heavy template code compiles in parallel.
#pragma once
#include "layer_rns.cuh"

namespace ensei_gpu {

struct LayerRun {
  const ensei_gpu_ctx* ctx;
  LayerArgs a;
  int logL;  // square padded grid, log2 side
  int R;
  cudaStream_t st;
  int gridL = 0;     // grid override (ensei_conv_desc::grid): the non-power-of-two side, else 0
  int tile_gen = 1;  // RNS tile kernels: 1 = layer_rns.cuh (512 threads, two CTAs per SM), 0 = layer.cuh
};

// Launch with programmatic stream serialization (layer.cuh, pdl_wait / pdl_trigger):
// the kernel may start while its stream predecessor still runs.  Falls back to an
// ordinary launch where the attribute is refused.
template <class... KArgs, class... Args>
static void launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, k, args...) != cudaSuccess) {
    cudaGetLastError();
    k<<<grid, block, smem, st>>>(args...);
  }
}

template <class K>
static void set_smem(K k, size_t smem) {
  if (smem > 48 * 1024) EG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
}
// Kernels meant to share an SM with another kernel's CTAs (Enc + HomShare) ask for the
// full shared-memory carveout: the driver otherwise sizes the SM's carveout for the
// first kernel placed there (e.g. 132 KB for a 114 KB CTA) and the second cannot join.
template <class K>
static void set_smem_shared_sm(K k, size_t smem) {
  set_smem(k, smem);
  EG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared));
}

// ---- tile -> ring (Enc / HomRec / weights / secret) ----
// thread groups per CTA: the blocks of one tile run concurrently when they fit
template <int LOGN>
constexpr bool kTwoGroups = LOGN <= 12;
inline int groups_for(int logn, int B) { return (B >= 2 && logn <= 12) ? 2 : 1; }

template <int LOGN, int LOGL, int R, int TM, bool INJ, int IN_T, int G, int TWS>
static void enc_go_t(const LayerRun& r, const uint64_t* key, uint32_t key_stride, const void* in, uint64_t* out,
                     int items) {
  auto k = tile_enc_kernel<LOGN, LOGL, LOGL, R, TM, INJ, IN_T, G, TWS>;
  const size_t smem = tile_enc_smem<LOGN, LOGL, LOGL, G, TWS == 2>(TM == TILE_WEIGHTS ? 1 : r.a.pk) +
                      tw_stage_bytes<LOGN, TWS>();
  set_smem_shared_sm(k, smem);
  k<<<items, G * ((1 << LOGN) >> tile_loge(LOGN)), smem, r.st>>>(r.a, key, key_stride, in, out);
  check_launch("tile_enc_kernel");
}

// Twiddle staging (layer.cuh, TWS = 2, with the p buffer aliased into the q buffer) at
// n = 2048 for single-wave launches: 49 KB of tables cost occupancy once CTAs queue
// behind each other, but are free when the launch has at most one tile per SM (an Enc
// and a HomShare CTA still co-reside: 102 + 114 KB).
template <int LOGN, int LOGL, int R, int TM, bool INJ, int IN_T, int G>
static void enc_go_g(const LayerRun& r, const uint64_t* key, uint32_t key_stride, const void* in, uint64_t* out,
                     int items) {
  if constexpr (LOGN == 11 && R == 1 && TM != TILE_WEIGHTS) {
    // two groups: registers already hold the kernel to 2 CTAs per SM, and two staged
    // CTAs (2 x 103 KB) still fit -- staging is free at any launch size
    if (G == 2 || items <= r.ctx->sm_count)
      return enc_go_t<LOGN, LOGL, R, TM, INJ, IN_T, G, 2>(r, key, key_stride, in, out, items);
  }
  enc_go_t<LOGN, LOGL, R, TM, INJ, IN_T, G, 0>(r, key, key_stride, in, out, items);
}

template <int LOGN, int LOGL, int R, int TM, bool INJ, int IN_T>
static void enc_go(const LayerRun& r, const uint64_t* key, uint32_t key_stride, const void* in, uint64_t* out,
                   int items) {
  if constexpr (kTwoGroups<LOGN>) {
    if (groups_for(LOGN, r.a.B) == 2) return enc_go_g<LOGN, LOGL, R, TM, INJ, IN_T, 2>(r, key, key_stride, in, out, items);
  }
  enc_go_g<LOGN, LOGL, R, TM, INJ, IN_T, 1>(r, key, key_stride, in, out, items);
}

template <int LOGN, int LOGL, int R>
static void enc_dispatch_l(const LayerRun& r, int tm, bool inj, int in_t, const uint64_t* key, uint32_t ks,
                           const void* in, uint64_t* out, int items) {
  if (tm == TILE_WEIGHTS) return enc_go<LOGN, LOGL, R, TILE_WEIGHTS, false, 0>(r, key, ks, in, out, items);
  if (tm == TILE_HOMREC) return enc_go<LOGN, LOGL, R, TILE_HOMREC, false, 0>(r, key, ks, in, out, items);
  if constexpr (R == 1) {
    if (inj) {
      if (in_t == ENSEI_IN_U8) return enc_go<LOGN, LOGL, R, TILE_ENC, true, ENSEI_IN_U8>(r, key, ks, in, out, items);
      return enc_go<LOGN, LOGL, R, TILE_ENC, true, ENSEI_IN_U32>(r, key, ks, in, out, items);
    }
  } else {
    if (inj) fail(ENSEI_ERR_UNSUPPORTED, "injected randomness is single-prime only (REF has no RNS)");
  }
  if (in_t == ENSEI_IN_U8) return enc_go<LOGN, LOGL, R, TILE_ENC, false, ENSEI_IN_U8>(r, key, ks, in, out, items);
  return enc_go<LOGN, LOGL, R, TILE_ENC, false, ENSEI_IN_U32>(r, key, ks, in, out, items);
}

template <int LOGN, int R>
static void enc_dispatch_r(const LayerRun& r, int tm, bool inj, int in_t, const uint64_t* key, uint32_t ks,
                           const void* in, uint64_t* out, int items) {
  switch (r.logL) {
    case 1: return enc_dispatch_l<LOGN, 1, R>(r, tm, inj, in_t, key, ks, in, out, items);
    case 2: return enc_dispatch_l<LOGN, 2, R>(r, tm, inj, in_t, key, ks, in, out, items);
    case 3: return enc_dispatch_l<LOGN, 3, R>(r, tm, inj, in_t, key, ks, in, out, items);
    case 4: return enc_dispatch_l<LOGN, 4, R>(r, tm, inj, in_t, key, ks, in, out, items);
    case 5: return enc_dispatch_l<LOGN, 5, R>(r, tm, inj, in_t, key, ks, in, out, items);
    case 6: return enc_dispatch_l<LOGN, 6, R>(r, tm, inj, in_t, key, ks, in, out, items);
  }
  fail(ENSEI_ERR_UNSUPPORTED, "padded grid side must be a power of two <= 64 on this path");
}

// ---- second-generation tile kernels (layer_rns.cuh): the 3-prime RNS layer at n = 8192 on
// 32x32 / 64x64 grids (REF's geometry) or the 39x39 override, and single-prime layers at
// n = 2048 on an overridden grid (39, 24 or 12: ensei_conv_desc::grid) ----
template <int LOGN, int R, class GR, int IN_T, bool HOMREC>
static void enc3_go(const LayerRun& r, const uint64_t* key, uint32_t ks, const void* in, uint64_t* out, int items) {
  auto k = enc3_kernel<LOGN, R, GR, IN_T, HOMREC>;
  constexpr size_t smem = enc3_smem<LOGN>();
  set_smem_shared_sm(k, smem);
  k<<<items, Ring<LOGN>::NT, smem, r.st>>>(r.a, key, ks, in, out);
  check_launch("enc3_kernel");
}
template <int LOGN, int R, class GR>
static bool enc3_try(const LayerRun& r, int tm, int in_t, const uint64_t* key, uint32_t ks, const void* in,
                     uint64_t* out, int items) {
  if (grid_tile_bytes<GR>(r.a.pk) > (size_t)(1 << LOGN) * 8) return false;  // tiles alias qbuf
  if (tm == TILE_HOMREC) enc3_go<LOGN, R, GR, ENSEI_IN_U32, true>(r, key, ks, in, out, items);
  else if (in_t == ENSEI_IN_U8) enc3_go<LOGN, R, GR, ENSEI_IN_U8, false>(r, key, ks, in, out, items);
  else enc3_go<LOGN, R, GR, ENSEI_IN_U32, false>(r, key, ks, in, out, items);
  return true;
}
template <int LOGN, int R, class GR>
static void share3_go(const LayerRun& r, uint64_t* mask, uint32_t* bob_share, int items) {
  auto k = share3_kernel<LOGN, R, GR>;
  constexpr size_t smem = share3_smem<LOGN>();
  set_smem_shared_sm(k, smem);
  k<<<items, Ring<LOGN>::NT, smem, r.st>>>(r.a, mask, bob_share);
  check_launch("share3_kernel");
}
template <int LOGN, int R, class GR>
static bool dec3_try(const LayerRun& r, const uint64_t* key, uint32_t ks, const uint64_t* ct, uint32_t* alice,
                     const uint32_t* bob, uint32_t* out, int items) {
  const size_t smem = dec3_smem<LOGN, GR>(r.a.pk);
  if (smem > 113 * 1024 || grid_tile_bytes<GR>(r.a.pk) / (GR::kScratch ? 2 : 1) > (size_t)(1 << LOGN) * 8 ||
      (size_t)r.a.pk * GR::TS * 4 > (size_t)(1 << LOGN) * 6)
    return false;
  auto k = dec3_kernel<LOGN, R, GR>;
  set_smem_shared_sm(k, smem);
  k<<<items, Ring<LOGN>::NT, smem, r.st>>>(r.a, key, ks, ct, alice, bob, out, Ring<LOGN>::MINB * r.ctx->sm_count);
  check_launch("dec3_kernel");
  return true;
}
template <int LOGN, int R, class GR>
static bool weights3_try(const LayerRun& r, const int32_t* w, uint64_t* out, int items) {
  if (grid_tile_bytes<GR>(1) > (size_t)(1 << LOGN) * 8) return false;
  auto k = weights3_kernel<LOGN, R, GR>;
  constexpr size_t smem = enc3_smem<LOGN>();
  set_smem_shared_sm(k, smem);
  k<<<items, Ring<LOGN>::NT, smem, r.st>>>(r.a, w, out);
  check_launch("weights3_kernel");
  return true;
}
[[noreturn]] inline void grid_fail() {
  fail(ENSEI_ERR_UNSUPPORTED,
       "grid override: 3-prime RNS layers at n = 8192 with grid 39, single-prime layers at n = 2048 with grid 39, 24 "
       "or 12; Philox randomness; pack x grid^2 <= n and the pack's tiles within the kernels' shared memory");
}
// the grid sides compiled in, as (LOGN, R, factors): p - 1 = 2^14 x 3 x 13 for the default p
#define EG_GRID_CASES(X)  \
  X(13, 3, 39, 3, 13)     \
  X(11, 1, 39, 3, 13)     \
  X(11, 1, 24, 3, 8)      \
  X(11, 1, 12, 3, 4)

template <int LOGN>
void launch_tile(const LayerRun& r, int tm, bool inj, int in_t, const uint64_t* key, uint32_t ks, const void* in,
                 uint64_t* out, int items) {
  if (items == 0) return;
  if (r.gridL) {  // grid override: second-generation kernels only
    if (!inj) {
#define EG_X(LN, RR, LL, N1, N2)                                                                              \
  if constexpr (LOGN == LN) {                                                                                 \
    if (r.R == RR && r.gridL == LL) {                                                                         \
      if (tm == TILE_WEIGHTS) {                                                                               \
        if (weights3_try<LN, RR, GridPFA<N1, N2>>(r, static_cast<const int32_t*>(in), out, items)) return;    \
      } else if (enc3_try<LN, RR, GridPFA<N1, N2>>(r, tm, in_t, key, ks, in, out, items)) {                   \
        return;                                                                                               \
      }                                                                                                       \
    }                                                                                                         \
  }
      EG_GRID_CASES(EG_X)
#undef EG_X
    }
    grid_fail();
  }
  if (r.R == 1) return enc_dispatch_r<LOGN, 1>(r, tm, inj, in_t, key, ks, in, out, items);
  if constexpr (LOGN == 13) {
    if (r.R == 3 && r.tile_gen && (tm == TILE_ENC || tm == TILE_HOMREC) && !inj) {
      if (r.logL == 6 && enc3_try<13, 3, GridPow2<6>>(r, tm, in_t, key, ks, in, out, items)) return;
      if (r.logL == 5 && enc3_try<13, 3, GridPow2<5>>(r, tm, in_t, key, ks, in, out, items)) return;
    }
    if (r.R == 3) return enc_dispatch_r<LOGN, 3>(r, tm, inj, in_t, key, ks, in, out, items);
  }
  fail(ENSEI_ERR_UNSUPPORTED, "RNS chains are supported with 3 primes at n = 8192");
}

// ---- HomShare masks + Bob share ----
template <int LOGN, int LOGL, int R, bool INJ, int G, int TWS>
static void share_go_t(const LayerRun& r, uint64_t* ct_out, uint32_t* bob_share, int items) {
  auto k = share_kernel<LOGN, LOGL, LOGL, R, INJ, G, TWS>;
  const size_t smem = share_smem<LOGN, LOGL, LOGL, G, TWS != 0>(r.a.B) + tw_stage_bytes<LOGN, TWS>();
  set_smem_shared_sm(k, smem);
  k<<<items, G * ((1 << LOGN) >> tile_loge(LOGN)), smem, r.st>>>(r.a, ct_out, bob_share);
  check_launch("share_kernel");
}

template <int LOGN, int LOGL, int R, bool INJ, int G>
static void share_go_g(const LayerRun& r, uint64_t* ct_out, uint32_t* bob_share, int items) {
  if constexpr (LOGN == 11 && R == 1) {  // q-table staging for single-wave launches (as Enc)
    if (items <= r.ctx->sm_count) return share_go_t<LOGN, LOGL, R, INJ, G, 2>(r, ct_out, bob_share, items);
    // multi-wave, two groups: the q table alone keeps two CTAs per SM (2 x 97 KB)
    if (G == 2) return share_go_t<LOGN, LOGL, R, INJ, G, 1>(r, ct_out, bob_share, items);
  }
  share_go_t<LOGN, LOGL, R, INJ, G, 0>(r, ct_out, bob_share, items);
}

template <int LOGN, int LOGL, int R, bool INJ>
static void share_go(const LayerRun& r, uint64_t* ct_out, uint32_t* bob_share, int items) {
  if constexpr (kTwoGroups<LOGN>) {
    if (groups_for(LOGN, r.a.B) == 2) return share_go_g<LOGN, LOGL, R, INJ, 2>(r, ct_out, bob_share, items);
  }
  share_go_g<LOGN, LOGL, R, INJ, 1>(r, ct_out, bob_share, items);
}

template <int LOGN, int R, bool INJ>
static void share_dispatch(const LayerRun& r, uint64_t* m, uint32_t* bs, int items) {
  switch (r.logL) {
    case 1: return share_go<LOGN, 1, R, INJ>(r, m, bs, items);
    case 2: return share_go<LOGN, 2, R, INJ>(r, m, bs, items);
    case 3: return share_go<LOGN, 3, R, INJ>(r, m, bs, items);
    case 4: return share_go<LOGN, 4, R, INJ>(r, m, bs, items);
    case 5: return share_go<LOGN, 5, R, INJ>(r, m, bs, items);
    case 6: return share_go<LOGN, 6, R, INJ>(r, m, bs, items);
  }
  fail(ENSEI_ERR_UNSUPPORTED, "padded grid side must be a power of two <= 64 on this path");
}

// The mask for (img, o, b, r) is written where c1 of the output ciphertext will
// live; mac_kernel reads it back before overwriting (same thread, same word).
template <int LOGN>
void launch_share(const LayerRun& r, bool inj, uint64_t* mask, uint32_t* bob_share, int items) {
  if (items == 0) return;
  if (r.gridL) {
    if (!inj) {
#define EG_X(LN, RR, LL, N1, N2)                                                             \
  if constexpr (LOGN == LN) {                                                                \
    if (r.R == RR && r.gridL == LL) return share3_go<LN, RR, GridPFA<N1, N2>>(r, mask, bob_share, items); \
  }
      EG_GRID_CASES(EG_X)
#undef EG_X
    }
    grid_fail();
  }
  if (r.R == 1) {
    if (inj) return share_dispatch<LOGN, 1, true>(r, mask, bob_share, items);
    return share_dispatch<LOGN, 1, false>(r, mask, bob_share, items);
  }
  if constexpr (LOGN == 13) {
    if (r.R == 3 && !inj && r.tile_gen) {
      if (r.logL == 6) return share3_go<13, 3, GridPow2<6>>(r, mask, bob_share, items);
      if (r.logL == 5) return share3_go<13, 3, GridPow2<5>>(r, mask, bob_share, items);
    }
    if (r.R == 3 && !inj) return share_dispatch<LOGN, 3, false>(r, mask, bob_share, items);
  }
  fail(ENSEI_ERR_UNSUPPORTED, "HomShare: unsupported prime count / randomness mode");
}

// ---- decrypt ----
template <int LOGN, int LOGL, int G>
static void dec_go_g(const LayerRun& r, const uint64_t* key, uint32_t ks, const uint64_t* ct, uint32_t* alice,
                     const uint32_t* bob, uint32_t* out, int items) {
  const size_t base = dec_smem<LOGN, LOGL, LOGL, G>(r.a.pk);
  const size_t staged = base + (size_t)(2 + 2 * r.a.B) * (1 << LOGN) * 8;  // + t^, t^', c0/c1 per block
  constexpr size_t twb = tw_stage_bytes<LOGN, 2>();
  // + staged twiddles (TWS): free when registers allow one CTA per SM anyway (G = 2)
  if (LOGN == 11 && (G == 2 || items <= r.ctx->sm_count) && staged + twb <= 227 * 1024) {
    auto k = dec_kernel<LOGN, LOGL, LOGL, G, true, LOGN == 11 ? 2 : 0>;
    set_smem(k, staged + twb);
    launch_pdl(k, items, G * ((1 << LOGN) >> tile_loge(LOGN)), staged + twb, r.st, r.a, key, ks, ct, alice, bob, out);
  } else if (staged <= 227 * 1024) {
    auto k = dec_kernel<LOGN, LOGL, LOGL, G, true>;
    set_smem(k, staged);
    launch_pdl(k, items, G * ((1 << LOGN) >> tile_loge(LOGN)), staged, r.st, r.a, key, ks, ct, alice, bob, out);
  } else {
    auto k = dec_kernel<LOGN, LOGL, LOGL, G, false>;
    set_smem(k, base);
    launch_pdl(k, items, G * ((1 << LOGN) >> tile_loge(LOGN)), base, r.st, r.a, key, ks, ct, alice, bob, out);
  }
  check_launch("dec_kernel");
}

template <int LOGN, int LOGL>
static void dec_go(const LayerRun& r, const uint64_t* key, uint32_t ks, const uint64_t* ct, uint32_t* alice,
                   const uint32_t* bob, uint32_t* out, int items) {
  if constexpr (kTwoGroups<LOGN>) {
    if (groups_for(LOGN, r.a.B) == 2) return dec_go_g<LOGN, LOGL, 2>(r, key, ks, ct, alice, bob, out, items);
  }
  dec_go_g<LOGN, LOGL, 1>(r, key, ks, ct, alice, bob, out, items);
}

template <int LOGN, int LOGL>
static void dec_rns_go(const LayerRun& r, const uint64_t* key, uint32_t ks, const uint64_t* ct, uint32_t* alice,
                       const uint32_t* bob, uint32_t* out, int items) {
  auto k = dec_rns_kernel<LOGN, LOGL, LOGL, 3>;
  const size_t smem = dec_rns_smem<LOGN, LOGL, LOGL>(r.a.pk);
  set_smem(k, smem);
  k<<<items, (1 << LOGN) >> tile_loge(LOGN), smem, r.st>>>(r.a, key, ks, ct, alice, bob, out);
  check_launch("dec_rns_kernel");
}

template <int LOGN>
void launch_dec(const LayerRun& r, const uint64_t* key, uint32_t ks, const uint64_t* ct, uint32_t* alice,
                const uint32_t* bob, uint32_t* out, int items) {
  if (items == 0) return;
  if (r.gridL) {
#define EG_X(LN, RR, LL, N1, N2)                                                                         \
  if constexpr (LOGN == LN) {                                                                            \
    if (r.R == RR && r.gridL == LL && (RR == 1 || r.a.dec_kbits) &&                                      \
        dec3_try<LN, RR, GridPFA<N1, N2>>(r, key, ks, ct, alice, bob, out, items))                       \
      return;                                                                                            \
  }
    EG_GRID_CASES(EG_X)
#undef EG_X
    grid_fail();
  }
  if (r.R != 1) {
    if constexpr (LOGN == 13) {
      if (r.R == 3 && r.tile_gen && r.a.dec_kbits) {
        if (r.logL == 6 && dec3_try<13, 3, GridPow2<6>>(r, key, ks, ct, alice, bob, out, items)) return;
        if (r.logL == 5 && dec3_try<13, 3, GridPow2<5>>(r, key, ks, ct, alice, bob, out, items)) return;
      }
      if (r.R == 3) {
        switch (r.logL) {
          case 5: return dec_rns_go<LOGN, 5>(r, key, ks, ct, alice, bob, out, items);
          case 6: return dec_rns_go<LOGN, 6>(r, key, ks, ct, alice, bob, out, items);
        }
      }
    }
    fail(ENSEI_ERR_UNSUPPORTED, "RNS decryption: 3 primes at n = 8192 with a 32x32 or 64x64 grid");
  }
  switch (r.logL) {
    case 1: return dec_go<LOGN, 1>(r, key, ks, ct, alice, bob, out, items);
    case 2: return dec_go<LOGN, 2>(r, key, ks, ct, alice, bob, out, items);
    case 3: return dec_go<LOGN, 3>(r, key, ks, ct, alice, bob, out, items);
    case 4: return dec_go<LOGN, 4>(r, key, ks, ct, alice, bob, out, items);
    case 5: return dec_go<LOGN, 5>(r, key, ks, ct, alice, bob, out, items);
    case 6: return dec_go<LOGN, 6>(r, key, ks, ct, alice, bob, out, items);
  }
  fail(ENSEI_ERR_UNSUPPORTED, "padded grid side must be a power of two <= 64 on this path");
}

// ---- secret key: t -> (t_eval, Shoup companion) per prime, device layout ----
template <int LOGN>
__global__ void __launch_bounds__((1 << LOGN) >> tile_loge(LOGN))
    secret_kernel(LayerArgs a, const int64_t* t_in, int64_t* t_out, uint64_t* key, int sample) {
  constexpr int N = 1 << LOGN, NT = N >> tile_loge(LOGN);
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint64_t* qbuf = reinterpret_cast<uint64_t*>(smem_raw);
  const int r = blockIdx.x;
  const PrimeConst pc = a.pc[r];
  const Field64 f = pc.f;
  const CtaBar bar;
  auto coeff = [&](int i) -> int64_t {
    return sample ? (int64_t)draw_ternary(a.alice_key, stream_id(PURPOSE_SECRET, 0, 0, 0, 0), i) : t_in[i];
  };
  if (sample && t_out && r == 0)
    for (int i = threadIdx.x; i < N; i += NT) t_out[i] = coeff(i);
  auto src = [&](int i) -> uint64_t {
    const int64_t t = coeff(i);
    const int64_t m = t % (int64_t)f.q;
    return m < 0 ? (uint64_t)(m + (int64_t)f.q) : (uint64_t)m;
  };
  uint64_t* kr = key + (size_t)(2 * r) * N;
  auto dst = [&](int j, uint64_t v) {
    const uint64_t x = Bfly<Field64, 0>::fin_ct(f, v, pc.cred);
    kr[j] = x;
    kr[N + j] = (uint64_t)(((unsigned __int128)x << 64) / f.q);
  };
  ntt_forward<Field64, uint64_t, LOGN, tile_loge(LOGN), 0, false, false>(f, a.twq_fwd[r], qbuf, threadIdx.x, src, dst, bar,
                                                               pc.cred);
}

template <int LOGN>
void launch_secret(const LayerRun& r, const int64_t* t_in, int64_t* t_out, uint64_t* key, bool sample) {
  auto k = secret_kernel<LOGN>;
  constexpr size_t smem = (size_t)(1 << LOGN) * 8;
  set_smem(k, smem);
  k<<<r.R, (1 << LOGN) >> tile_loge(LOGN), smem, r.st>>>(r.a, t_in, t_out, key, sample ? 1 : 0);
  check_launch("secret_kernel");
}

#define EG_INSTANTIATE_LAYER(LOGN)                                                                               \
  template void launch_tile<LOGN>(const LayerRun&, int, bool, int, const uint64_t*, uint32_t, const void*,      \
                                  uint64_t*, int);                                                               \
  template void launch_share<LOGN>(const LayerRun&, bool, uint64_t*, uint32_t*, int);                            \
  template void launch_dec<LOGN>(const LayerRun&, const uint64_t*, uint32_t, const uint64_t*, uint32_t*,         \
                                 const uint32_t*, uint32_t*, int);                                               \
  template void launch_secret<LOGN>(const LayerRun&, const int64_t*, int64_t*, uint64_t*, bool);

}  // namespace ensei_gpu
