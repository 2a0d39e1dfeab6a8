// tools/tune_ntt.cu -- sweep launch shapes of the batched negacyclic q-transform
// (config 2) and report throughput.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -o scratch/tune_ntt tools/tune_ntt.cu
#include <cstdio>
#include <vector>
#include "../paper_2003_05328_b200/csrc/ntt_batch.cuh"
#include "../paper_2003_05328_b200/csrc/host_field.hpp"
using namespace ensei_gpu;
std::atomic<uint64_t> ensei_gpu::g_launches{0};

static const uint64_t Q = 576460803525083137ULL;

template <int LOGN, int LOGE, bool INV, bool TWS>
void run(PrimeConst pc, TwPair<uint64_t>* tw, uint64_t* d, size_t count, int sms) {
  auto k = negacyclic_q_kernel<LOGN, LOGE, 0, INV, false, TWS>;
  constexpr int NT = (1 << LOGN) >> LOGE;
  size_t smem = negacyclic_q_smem<LOGN, LOGE, TWS>();
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, NT, smem);
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, k);
  size_t grid = std::min<size_t>(count, (size_t)std::max(per_sm, 1) * sms);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int it = 0; it < 6; ++it) {
    cudaEventRecord(e0);
    k<<<grid, NT, smem>>>(pc, tw, d, count);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (it >= 1) best = std::min(best, ms);
  }
  double n = 1 << LOGN, bfly = n / 2 * LOGN;
  double rate = count / (best * 1e-3);
  printf("n=%5d %s LOGE=%d TWS=%d regs=%3d spill=%zu occ=%d/SM smem=%zu  %.3f ms  %7.1f M transforms/s  %6.0f GB/s  %.2f Gbfly/s  %s\n",
         1 << LOGN, INV ? "inv" : "fwd", LOGE, (int)TWS, fa.numRegs, fa.localSizeBytes, per_sm, smem, best, rate / 1e6,
         count * n * 16 / (best * 1e-3) / 1e9, rate * bfly / 1e9, cudaGetErrorString(cudaGetLastError()));
}

template <int LOGN>
void sweep(int sms) {
  using namespace host;
  const uint64_t n = 1 << LOGN;
  TwiddleValues tv = make_twiddles(Q, n, true);
  std::vector<TwPair<uint64_t>> hf(n), hi(n);
  for (uint64_t k = 0; k < n; ++k) { hf[k] = {tv.fwd[k], shoup64(tv.fwd[k], Q)}; hi[k] = {tv.inv[k], shoup64(tv.inv[k], Q)}; }
  TwPair<uint64_t> *df, *di; cudaMalloc(&df, n * 16); cudaMalloc(&di, n * 16);
  cudaMemcpy(df, hf.data(), n * 16, cudaMemcpyHostToDevice); cudaMemcpy(di, hi.data(), n * 16, cudaMemcpyHostToDevice);
  size_t count = 65536;
  uint64_t* d; cudaMalloc(&d, count * n * 8); cudaMemset(d, 0, count * n * 8);
  PrimeConst pc; pc.f = Field64{Q, 2 * Q, 0 - Q, 4 * Q}; pc.cred = (uint32_t)(((unsigned __int128)1 << 64) / Q);
  run<LOGN, 3, false, false>(pc, df, d, count, sms); run<LOGN, 4, false, false>(pc, df, d, count, sms);
  run<LOGN, 3, true, false>(pc, di, d, count, sms); run<LOGN, 4, true, false>(pc, di, d, count, sms);
  if constexpr (LOGN <= 12) {
    run<LOGN, 3, false, true>(pc, df, d, count, sms); run<LOGN, 4, false, true>(pc, df, d, count, sms);
    run<LOGN, 3, true, true>(pc, di, d, count, sms); run<LOGN, 4, true, true>(pc, di, d, count, sms);
  }
  cudaFree(d); cudaFree(df); cudaFree(di);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  sweep<11>(sms); sweep<12>(sms); sweep<13>(sms);
}
