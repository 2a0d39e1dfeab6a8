// ntt_kernels.cu -- boundary transforms of the C ABI:
//   * ensei_gpu_negacyclic : batched NegacyclicPlan::forward/inverse over q_i or p
//                            (REF ringbfv.cpp:49-59, 109-125); config 2 hot path
//   * ensei_gpu_ntt2d      : batched ntt_2d / intt_2d over p (REF ntt.cpp:112-153)
//   * ensei_gpu_permute    : natural <-> bit-reversed slot order
#include "common.cuh"
#include "kernels.cuh"
#include "ntt_batch.cuh"
#include "layer_rns.cuh"

namespace ensei_gpu {

// ------------------------------------------------------------------- launch

template <int LOGN, int LOGE, int MODE, bool INV, bool NATURAL, bool TW_SMEM, int G>
static void launch_q(const ensei_gpu_ctx* ctx, int prime, uint64_t* d, size_t count, cudaStream_t st) {
  auto k = negacyclic_q_kernel<LOGN, LOGE, MODE, INV, NATURAL, TW_SMEM, G>;
  constexpr int NT = G * ((1 << LOGN) >> LOGE);
  constexpr size_t smem = negacyclic_q_smem<LOGN, LOGE, TW_SMEM, G>();
  static int per_sm = -1;
  if (per_sm < 0) {
    EG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    EG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, NT, smem));
  }
  size_t grid = std::min<size_t>((count + G - 1) / G, (size_t)std::max(per_sm, 1) * ctx->sm_count);
  const TwPair<uint64_t>* tw = INV ? ctx->tab.tw_q_inv[prime] : ctx->tab.tw_q_fwd[prime];
  k<<<(unsigned)grid, NT, smem, st>>>(ctx->pc[prime], tw, d, count);
  check_launch("negacyclic_q_kernel");
}

// n = 8192, device layout, lazy (MODE 0) butterflies: the tile kernels' form of the transform
// (layer_rns.cuh): 512 threads run every pass in two rounds, one 64 KB buffer, two CTAs per SM
// out of step with each other instead of one 1024-thread CTA with a prefetch buffer.
struct GlobalIn64 {
  const uint64_t* g;
  static constexpr bool kVec = true;
  EG_DEV uint64_t operator()(int i) const { return g[i]; }
  EG_DEV void ld2(int i, uint64_t& a, uint64_t& b) const {
    const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(g + i);
    a = v.x;
    b = v.y;
  }
};
template <bool INV>
__global__ void __launch_bounds__(kRnsThreads, 2)
    negacyclic_q13_kernel(PrimeConst pc, const TwPair<uint64_t>* __restrict__ tw, uint64_t* data, size_t count) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint64_t* qbuf = reinterpret_cast<uint64_t*>(smem_raw);
  const int tid = threadIdx.x;
  const Field64 f = pc.f;
  for (size_t poly = blockIdx.x; poly < count; poly += gridDim.x) {
    uint64_t* g = data + poly * (size_t)(1 << kRnsLogN);
    GlobalIn64 src{g};
    if constexpr (!INV) {
      GlobalOut64<0, true> out{g, f, pc.cred};
      rns_forward<kRnsLogN, Field64, uint64_t, 1>(f, tw, qbuf, tid, src, out, pc.cred);
    } else {
      auto dst = [&](int i, uint64_t v) { g[i] = Bfly<Field64, 0>::fin_gs(f, v); };
      rns_inverse<kRnsLogN, Field64, uint64_t>(f, tw, qbuf, tid, src, dst);
    }
    __syncthreads();
  }
}
template <bool INV>
static void launch_q13(const ensei_gpu_ctx* ctx, int prime, uint64_t* d, size_t count, cudaStream_t st) {
  auto k = negacyclic_q13_kernel<INV>;
  constexpr size_t smem = (size_t)(1 << kRnsLogN) * 8;
  static bool once = false;
  if (!once) {
    EG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    once = true;
  }
  const size_t grid = std::min<size_t>(count, (size_t)2 * ctx->sm_count);
  k<<<(unsigned)grid, kRnsThreads, smem, st>>>(ctx->pc[prime], INV ? ctx->tab.tw_q_inv[prime] : ctx->tab.tw_q_fwd[prime],
                                               d, count);
  check_launch("negacyclic_q13_kernel");
}

template <int LOGN, bool INV, bool NATURAL>
static void launch_q_dispatch(const ensei_gpu_ctx* ctx, int prime, uint64_t* d, size_t count, cudaStream_t st) {
  constexpr bool TWS = LOGN <= 12;  // tools/tune_ntt.cu sweep: TMA-staged twiddles win up to n = 4096
  // G = 2 (two polynomials per CTA sharing the staged table: 32 resident warps instead of 24 at
  // n = 2048, 16 at n = 4096) measured slower: 57.8 vs 65.5 M forward transforms/s at n = 2048,
  // 26.7 vs 29.3 M at n = 4096 (the 64-register cap and the per-group barriers cost more than
  // the extra warps bring)
  constexpr int G = 1;
  if constexpr (LOGN == 13 && !NATURAL) {
    if (ctx->approx_ok) return launch_q13<INV>(ctx, prime, d, count, st);
  }
  if (ctx->approx_ok) launch_q<LOGN, 3, 0, INV, NATURAL, TWS, G>(ctx, prime, d, count, st);
  else launch_q<LOGN, 3, 1, INV, NATURAL, TWS, G>(ctx, prime, d, count, st);
}

template <int LOGN, bool INV, bool NATURAL>
static void launch_p(const ensei_gpu_ctx* ctx, uint64_t* d, size_t count, cudaStream_t st) {
  auto k = negacyclic_p_kernel<LOGN, 3, INV, NATURAL>;
  constexpr int NT = (1 << LOGN) >> 3;
  const size_t smem = ssize<uint32_t>(1 << LOGN) * sizeof(uint32_t);
  size_t grid = std::min<size_t>(count, (size_t)ctx->sm_count * 8);
  const TwPair<uint32_t>* tw = INV ? ctx->tab.tw_p_inv : ctx->tab.tw_p_fwd;
  k<<<(unsigned)grid, NT, smem, st>>>(ctx->pp, tw, d, count);
  check_launch("negacyclic_p_kernel");
}

void negacyclic(const ensei_gpu_ctx* ctx, uint32_t modulus, bool inverse, bool natural, uint64_t* d,
                size_t count, cudaStream_t st) {
  if (count == 0) return;
  const int logn = (int)ctx->logn;
#define EG_Q(LN)                                                                   \
  case LN:                                                                         \
    if (inverse) {                                                                 \
      if (natural) launch_q_dispatch<LN, true, true>(ctx, modulus, d, count, st);  \
      else launch_q_dispatch<LN, true, false>(ctx, modulus, d, count, st);         \
    } else {                                                                       \
      if (natural) launch_q_dispatch<LN, false, true>(ctx, modulus, d, count, st); \
      else launch_q_dispatch<LN, false, false>(ctx, modulus, d, count, st);        \
    }                                                                              \
    return;
#define EG_P(LN)                                                          \
  case LN:                                                                \
    if (inverse) {                                                        \
      if (natural) launch_p<LN, true, true>(ctx, d, count, st);           \
      else launch_p<LN, true, false>(ctx, d, count, st);                  \
    } else {                                                              \
      if (natural) launch_p<LN, false, true>(ctx, d, count, st);          \
      else launch_p<LN, false, false>(ctx, d, count, st);                \
    }                                                                     \
    return;
  if (modulus == ENSEI_MOD_P) {
    switch (logn) { EG_P(11) EG_P(12) EG_P(13) }
  } else {
    switch (logn) { EG_Q(11) EG_Q(12) EG_Q(13) }
  }
#undef EG_Q
#undef EG_P
  fail(ENSEI_ERR_UNSUPPORTED, "ring degree must be 2048, 4096 or 8192 on this path");
}

void permute(const ensei_gpu_ctx* ctx, uint64_t* d, size_t count, cudaStream_t st) {
  if (count == 0) return;
  size_t grid = std::min<size_t>(count, (size_t)ctx->sm_count * 8);
  const size_t smem = ssize<uint64_t>(ctx->n) * sizeof(uint64_t);
  EG_CUDA(cudaFuncSetAttribute(permute_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  permute_kernel<<<(unsigned)grid, 256, smem, st>>>(d, count, (int)ctx->logn);
  check_launch("permute_kernel");
}

template <int LH, int LW>
static void launch_2d(const ensei_gpu_ctx* ctx, bool inv, uint64_t* d, size_t count, cudaStream_t st) {
  size_t grid = std::min<size_t>(count, (size_t)ctx->sm_count * 8);
  if (inv) ntt2d_kernel<LH, LW, true><<<(unsigned)grid, 256, 0, st>>>(ctx->pp, ctx->tab.tw_c_inv, d, count);
  else ntt2d_kernel<LH, LW, false><<<(unsigned)grid, 256, 0, st>>>(ctx->pp, ctx->tab.tw_c_fwd, d, count);
  check_launch("ntt2d_kernel");
}

void ntt2d(const ensei_gpu_ctx* ctx, bool inv, int logh, int logw, uint64_t* d, size_t count, cudaStream_t st) {
  if (count == 0) return;
  if (logh != logw) fail(ENSEI_ERR_UNSUPPORTED, "ntt2d: square tiles only on this path");
  switch (logh) {
    case 1: return launch_2d<1, 1>(ctx, inv, d, count, st);
    case 2: return launch_2d<2, 2>(ctx, inv, d, count, st);
    case 3: return launch_2d<3, 3>(ctx, inv, d, count, st);
    case 4: return launch_2d<4, 4>(ctx, inv, d, count, st);
    case 5: return launch_2d<5, 5>(ctx, inv, d, count, st);
    case 6: return launch_2d<6, 6>(ctx, inv, d, count, st);
  }
  fail(ENSEI_ERR_UNSUPPORTED, "ntt2d: tile side must be a power of two <= 64");
}

}  // namespace ensei_gpu
