// common.cuh -- context layout, error plumbing and launch bookkeeping shared by the
// kernels and the C ABI (include/ensei_gpu.h).
#pragma once
#include <vector>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <mutex>
#include <stdexcept>
#include <string>

#include "../../include/ensei_gpu.h"
#include "ntt_core.cuh"

namespace ensei_gpu {

// A C++ exception carrying an ensei_status; the ABI layer converts it to a code.
struct Status : std::runtime_error {
  int code;
  Status(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& m) { throw Status(code, m); }
inline void require(bool ok, int code, const char* m) {
  if (!ok) fail(code, m);
}
#define EG_CUDA(x)                                                                      \
  do {                                                                                  \
    cudaError_t e_ = (x);                                                               \
    if (e_ != cudaSuccess)                                                              \
      ::ensei_gpu::fail(ENSEI_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

extern std::atomic<uint64_t> g_launches;
inline void count_launch(uint64_t n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }
inline void check_launch(const char* what) {
  cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) fail(ENSEI_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  count_launch();
}

// Per-kernel CUDA-event timing (ensei_gpu_profile): off by default.  When on, each layer
// kernel launch is bracketed by two events recorded on its own stream (skipped while
// the stream is being captured), and ensei_gpu_profile_read() sums the durations per
// kernel.  For a measurement pass outside the timed region (the events serialise PDL).
bool prof_on();
void prof_record(const char* name, cudaStream_t st, bool begin);
struct ProfScope {
  const char* name;
  cudaStream_t st;
  bool on;
  ProfScope(const char* n, cudaStream_t s) : name(n), st(s), on(prof_on()) {
    if (on) prof_record(name, st, true);
  }
  ~ProfScope() {
    if (on) prof_record(name, st, false);
  }
};

// Per-prime constants for Field64 kernels.
struct PrimeConst {
  Field64 f;
  uint32_t cred;  // floor(2^64 / q) (fits 32 bits for q > 2^32), for reduce_lazy
  uint64_t mu_hi, mu_lo;  // floor(2^128 / q)
  uint64_t delta;         // floor(Q / p) mod q_i
  uint64_t delta_shoup;   // Shoup companion of delta
  uint64_t cp;            // floor(p * 2^64 / q), decryption rounding estimate
  uint32_t a2_chunk;      // MAC: channels per full reduction of the top limb
  uint64_t c64, c64p;     // 2^64 mod q and its Shoup companion
  uint64_t crt_inv, crt_inv_shoup;  // (Q/q_i)^-1 mod q_i (RNS decryption)
  uint64_t crt_c;                   // floor(2^122 / q_i): E / q_i in 2^-62 fixed point
  // second-generation RNS decryption (layer_rns.cuh): the last-stage constants of the
  // inverse transform with (Q/q_i)^-1 folded in (n^-1 crt_inv, and twi[1] crt_inv), and
  // floor(p 2^(dec_kbits + 64) / q_i)
  uint64_t dec_ni, dec_ni_shoup, dec_t1, dec_t1_shoup, dec_c;
};

// Exact CRT rounding constants (RNS decryption, layer.cuh crt_round): M_i = Q / q_i and
// the thresholds T_t = (2t - 1) Q, t = 1..3, as little-endian 32-bit limbs.
struct CrtConst {
  uint32_t M[ENSEI_MAX_PRIMES][4];
  uint32_t T[3][6];
};

struct PConst {
  Field32 f;
  uint32_t cred;  // floor(2^32 / p)
  uint64_t m64;   // floor(2^64 / p)
};

// Device twiddle tables (TwPair = value + Shoup companion), see ntt_core.cuh for
// the conventions.  Cyclic tables for L = 2^1 .. 2^6 live at offset L in tw_c_*.
struct DeviceTables {
  TwPair<uint64_t>* tw_q_fwd[ENSEI_MAX_PRIMES] = {};
  TwPair<uint64_t>* tw_q_inv[ENSEI_MAX_PRIMES] = {};
  TwPair<uint32_t>* tw_p_fwd = nullptr;  // negacyclic n-point over p
  TwPair<uint32_t>* tw_p_inv = nullptr;
  TwPair<uint32_t>* tw_c_fwd = nullptr;  // cyclic L-point over p, L <= 64
  TwPair<uint32_t>* tw_c_inv = nullptr;
};

constexpr int kMaxTile = 64;  // largest supported padded grid side

}  // namespace ensei_gpu

struct ensei_gpu_ctx {
  int device = 0;
  int sm_count = 0;
  uint32_t n = 0, logn = 0, R = 0;
  uint64_t q[ENSEI_MAX_PRIMES] = {};
  uint64_t p = 0;
  uint64_t psi_q[ENSEI_MAX_PRIMES] = {};
  uint64_t psi_p = 0;
  ensei_gpu::PrimeConst pc[ENSEI_MAX_PRIMES];
  ensei_gpu::CrtConst crt;
  ensei_gpu::PConst pp;
  ensei_gpu::DeviceTables tab;
  void* table_mem = nullptr;
  bool approx_ok = true;  // every 31 q_i < 2^64: approximate-quotient butterflies (MODE 0); the layer path needs it
  uint32_t i8_kmax = 255;  // int8 tensor-core MAC: largest K with K (q_i - 1)^2 < 2^128 for every prime
  bool kara_ok = true;    // every q_i within the Karatsuba MAC's headroom (layer.cuh)
  // layer_rns.cuh: fraction bits of the packed CRT accumulator (12p 2^k <= 2^48); 0 when the
  // chain cannot use it (then the first-generation kernels run)
  uint32_t dec_kbits = 0;
  // fork/join helpers: Bob's input-independent HomShare work runs concurrently
  // with Alice's encryption on an auxiliary stream (capturable in CUDA graphs)
  cudaStream_t aux = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // ensei_gpu_conv_layer_host: H2D + layer + D2H captured once into a CUDA graph and
  // replayed while every argument is unchanged (key = the arguments' bytes).
  cudaStream_t host_st = nullptr;  // capture/replay stream when the caller passes the legacy stream
  cudaEvent_t host_ev = nullptr;
  cudaGraphExec_t host_graph = nullptr;
  uint64_t host_graph_kernels = 0;  // kernels per replay (for ensei_gpu_launch_count)
  std::vector<uint8_t> host_graph_key;
  // wire decoding (wire.cu): mapped pinned status block [first-error key, domain flags,
  // per-record domain tags], grown on demand; read by the host after the decode kernels
  // (one decode at a time per context: the two parties of an in-process session decode
  // from two host threads)
  uint8_t* wire_status = nullptr;
  size_t wire_status_cap = 0;
  std::mutex wire_mu;
  // int8 tensor-core ElementMult: byte-plane operands (mac_i8.cuh), grown on demand
  void* i8_scratch = nullptr;
  size_t i8_scratch_cap = 0;

};
