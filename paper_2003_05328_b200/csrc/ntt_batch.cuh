// ntt_batch.cuh -- batched boundary-transform kernels (templates), shared by
// ntt_kernels.cu and the tuning benchmark (tools/tune_ntt.cu).
#pragma once
#include <type_traits>

#include "common.cuh"
#include "kernels.cuh"

namespace ensei_gpu {

// Prefetch one length-N u64 polynomial into a swizzled smem buffer (cp.async 16B).
template <int N>
EG_DEV void prefetch_poly(uint64_t* sm, const uint64_t* g, int tid, int nthreads) {
  for (int c = tid; c < N / 2; c += nthreads) cp_async16(sm + sidx<uint64_t>(2 * c), g + 2 * c);
  cp_async_commit();
}

// Barrier over the NT threads of thread group g of a CTA (literal ids: ptxas budgets barriers
// by the largest id it sees)
struct BatchGroupBar {
  int g, count;
  EG_DEV void sync() const {
    if (g == 0) asm volatile("bar.sync 1, %0;" ::"r"(count) : "memory");
    else asm volatile("bar.sync 2, %0;" ::"r"(count) : "memory");
  }
};

// One length-N transform per thread group and iteration (NT = N/E threads per group, G groups
// per CTA), persistent grid-stride over polynomials.  The next polynomial streams into the
// group's second smem buffer with cp.async while the current one is transformed; twiddles
// are staged once per CTA by a TMA bulk copy (TW_SMEM) or read through L1.  G = 2 lets two
// polynomials share one staged table: 96 KB per 512-thread CTA at n = 2048 (two CTAs = 32
// warps per SM instead of three 64 KB CTAs = 24), 192 KB per 1024-thread CTA at n = 4096
// (32 warps instead of 16); the groups run out of step behind their own named barriers.
template <int LOGN, int LOGE, int MODE, bool INV, bool NATURAL, bool TW_SMEM, int G = 1>
__global__ void __launch_bounds__(G * ((1 << LOGN) >> LOGE), (G * ((1 << LOGN) >> LOGE) <= 512 && G == 2) ? 2 : 1)
    negacyclic_q_kernel(PrimeConst pc, const TwPair<uint64_t>* __restrict__ tw_g, uint64_t* data,
                        size_t count) {
  constexpr int N = 1 << LOGN, NT = N >> LOGE;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  __shared__ uint64_t mbar;
  TwPair<uint64_t>* tw_s = reinterpret_cast<TwPair<uint64_t>*>(smem_raw);
  const int g = G == 1 ? 0 : threadIdx.x / NT, tid = G == 1 ? threadIdx.x : threadIdx.x % NT;
  uint64_t* buf0 = reinterpret_cast<uint64_t*>(smem_raw + (TW_SMEM ? N * sizeof(TwPair<uint64_t>) : 0)) + g * 2 * N;
  const BatchGroupBar bar{g, NT};
  const Field64 f = pc.f;
  const TwPair<uint64_t>* tw = tw_g;
  size_t poly = (size_t)blockIdx.x * G + g;
  const size_t stride = (size_t)gridDim.x * G;
  if (poly < count) prefetch_poly<N>(buf0, data + poly * N, tid, NT);
  if constexpr (TW_SMEM) {
    stage_table(tw_s, tw_g, N * sizeof(TwPair<uint64_t>), &mbar);
    tw = tw_s;
  }
  int cur = 0;
  for (; poly < count; poly += stride) {
    cp_async_wait_all();
    bar.sync();
    const size_t next = poly + stride;
    if (next < count) prefetch_poly<N>(buf0 + (cur ^ 1) * N, data + next * N, tid, NT);
    uint64_t* sm = buf0 + cur * N;
    uint64_t* gp = data + poly * N;
    SmemRW<uint64_t> s{sm};
    if constexpr (!INV) {
      if constexpr (!NATURAL) {
        GlobalOut64<MODE, true> out{gp, f, pc.cred};
        ntt_forward<Field64, uint64_t, LOGN, LOGE, MODE, false, false>(f, tw, sm, tid, s, out, bar, pc.cred);
      } else {
        auto dst = [&](int i, uint64_t v) {
          sm[sidx<uint64_t>(brev(i, LOGN))] = Bfly<Field64, MODE>::fin_ct(f, v, pc.cred);
        };
        ntt_forward<Field64, uint64_t, LOGN, LOGE, MODE, false, true>(f, tw, sm, tid, s, dst, bar, pc.cred);
        bar.sync();
        for (int c = tid; c < N / 2; c += NT)
          *reinterpret_cast<ulonglong2*>(gp + 2 * c) = *reinterpret_cast<const ulonglong2*>(sm + sidx<uint64_t>(2 * c));
      }
    } else {
      GlobalOut64<MODE, false> out{gp, f, pc.cred};
      if constexpr (!NATURAL) {
        ntt_inverse<Field64, uint64_t, LOGN, LOGE, MODE, false, false>(f, tw, sm, tid, s, out, bar);
      } else {
        auto src = [&](int i) { return sm[sidx<uint64_t>(brev(i, LOGN))]; };
        ntt_inverse<Field64, uint64_t, LOGN, LOGE, MODE, true, false>(f, tw, sm, tid, src, out, bar);
      }
    }
    cur ^= 1;
  }
  cp_async_wait_all();
}

template <int LOGN, int LOGE, bool TW_SMEM, int G = 1>
constexpr size_t negacyclic_q_smem() {
  return (TW_SMEM ? (1 << LOGN) * sizeof(TwPair<uint64_t>) : 0) + (size_t)G * 2 * (1 << LOGN) * sizeof(uint64_t);
}

// Same structure over the 32-bit modulus p, uint64 storage (REF Residue).
template <int LOGN, int LOGE, bool INV, bool NATURAL>
__global__ void __launch_bounds__((1 << LOGN) >> LOGE)
    negacyclic_p_kernel(PConst pc, const TwPair<uint32_t>* __restrict__ tw, uint64_t* data,
                        size_t count) {
  constexpr int N = 1 << LOGN, NT = N >> LOGE;
  extern __shared__ __align__(16) uint32_t smem_p[];
  uint32_t* sm = smem_p;
  const int tid = threadIdx.x;
  const CtaBar bar;
  const Field32 f = pc.f;
  using B = Bfly<Field32, 0>;
  for (size_t poly = blockIdx.x; poly < count; poly += gridDim.x) {
    uint64_t* g = data + poly * N;
    auto gsrc = [&](int i) { return (uint32_t)g[i]; };
    if constexpr (!INV) {
      if constexpr (!NATURAL) {
        auto dst = [&](int i, uint32_t v) { g[i] = reduce_lazy(f, v, pc.cred); };
        ntt_forward<Field32, uint32_t, LOGN, LOGE, 0, false, false>(f, tw, sm, tid, gsrc, dst, bar);
      } else {
        auto dst = [&](int i, uint32_t v) { sm[sidx<uint32_t>(brev(i, LOGN))] = reduce_lazy(f, v, pc.cred); };
        ntt_forward<Field32, uint32_t, LOGN, LOGE, 0, false, true>(f, tw, sm, tid, gsrc, dst, bar);
        bar.sync();
        for (int i = tid; i < N; i += NT) g[i] = sm[sidx<uint32_t>(i)];
      }
    } else {
      auto dst = [&](int i, uint32_t v) { g[i] = B::fin_gs(f, v); };
      if constexpr (!NATURAL) {
        ntt_inverse<Field32, uint32_t, LOGN, LOGE, 0, false, false>(f, tw, sm, tid, gsrc, dst, bar);
      } else {
        for (int i = tid; i < N; i += NT) sm[sidx<uint32_t>(i)] = (uint32_t)g[i];
        bar.sync();
        auto src = [&](int i) { return sm[sidx<uint32_t>(brev(i, LOGN))]; };
        ntt_inverse<Field32, uint32_t, LOGN, LOGE, 0, true, false>(f, tw, sm, tid, src, dst, bar);
      }
    }
    bar.sync();
  }
}

// ----------------------------------------------------------------- permute

__global__ void permute_kernel(uint64_t* data, size_t count, int logn) {
  extern __shared__ __align__(16) uint64_t smem_perm[];
  const int n = 1 << logn;
  for (size_t poly = blockIdx.x; poly < count; poly += gridDim.x) {
    uint64_t* g = data + poly * n;
    for (int i = threadIdx.x; i < n; i += blockDim.x) smem_perm[sidx<uint64_t>(i)] = g[i];
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) g[i] = smem_perm[sidx<uint64_t>(brev(i, logn))];
    __syncthreads();
  }
}

// -------------------------------------------------------------------- 2D

// ntt_2d / intt_2d of one Lh x Lw tile per CTA iteration, natural order in/out.
template <int LOGH, int LOGW, bool INV>
__global__ void __launch_bounds__(256) ntt2d_kernel(PConst pc, const TwPair<uint32_t>* __restrict__ twc,
                                                    uint64_t* data, size_t count) {
  constexpr int Lh = 1 << LOGH, Lw = 1 << LOGW;
  __shared__ uint32_t S[Lh * (Lw + 1)];
  const Field32 f = pc.f;
  for (size_t t = blockIdx.x; t < count; t += gridDim.x) {
    uint64_t* g = data + t * Lh * Lw;
    for (int i = threadIdx.x; i < Lh * Lw; i += blockDim.x) {
      int r = i >> LOGW, c = i & (Lw - 1);
      if (!INV) S[r * (Lw + 1) + c] = (uint32_t)g[i];
      else S[brev(r, LOGH) * (Lw + 1) + brev(c, LOGW)] = (uint32_t)g[i];
    }
    __syncthreads();
    tile_transform_2d<INV, LOGH, LOGW>(f, pc.cred, twc, S, Lw + 1);
    for (int i = threadIdx.x; i < Lh * Lw; i += blockDim.x) {
      int r = i >> LOGW, c = i & (Lw - 1);
      if (!INV) g[i] = S[brev(r, LOGH) * (Lw + 1) + brev(c, LOGW)];
      else g[i] = S[r * (Lw + 1) + c];
    }
    __syncthreads();
  }
}

}  // namespace ensei_gpu
