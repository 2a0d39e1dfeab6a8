// tools/mma_i8_probe.cu -- legacy int8 mma.sync (m16n8k32 u8) throughput on B200; build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scratch/mma_i8_probe tools/mma_i8_probe.cu
#include <cstdio>
#include <cstdint>
__global__ void probe(int iters, int* out) {
  uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
  int c[8][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < 8; ++t)
      asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+r"(c[t][0]), "+r"(c[t][1]), "+r"(c[t][2]), "+r"(c[t][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  int s = 0;
  for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1] + c[t][2] + c[t][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int* d; cudaMalloc(&d, 148 * 16 * 512 * 4);
  int iters = 4096;
  for (int warps : {4, 8, 16}) {
    for (int bps : {1, 2, 4}) {
      dim3 g(148 * bps), b(32 * warps);
      probe<<<g, b>>>(16, d);
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      probe<<<g, b>>>(iters, d);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double macs = (double)g.x * warps * iters * 8 * 16 * 8 * 32;
      printf("warps/CTA %2d CTAs/SM %d: %.1f T int8 MAC/s (%.1f TOPS)\n", warps, bps, macs / ms / 1e9, 2 * macs / ms / 1e9);
    }
  }
  return 0;
}
