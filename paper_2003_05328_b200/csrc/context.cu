// context.cu -- C ABI: context creation (RlweParams/ModulusChain equivalent),
// error mapping and the single-transform entry points.
#include <algorithm>
#include <memory>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "host_field.hpp"
#include "kernels.cuh"

namespace ensei_gpu {

std::atomic<uint64_t> g_launches{0};
static thread_local std::string g_last_error;

template <class Fn>
static int guarded(Fn&& fn) {
  try {
    fn();
    return ENSEI_OK;
  } catch (const Status& s) {
    g_last_error = s.what();
    return s.code;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    return ENSEI_ERR_INVALID_ARGUMENT;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return ENSEI_ERR_GENERIC;
  }
}

// ---- per-kernel event timing (ProfScope, common.cuh)
namespace {
struct ProfRec {
  std::string name;
  cudaEvent_t a, b;
};
std::mutex g_prof_mu;
std::atomic<bool> g_prof{false};
std::vector<ProfRec> g_prof_recs;
std::vector<cudaEvent_t> g_prof_pool;
cudaEvent_t prof_event() {
  if (!g_prof_pool.empty()) {
    cudaEvent_t e = g_prof_pool.back();
    g_prof_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  EG_CUDA(cudaEventCreate(&e));
  return e;
}
}  // namespace

bool prof_on() { return g_prof.load(std::memory_order_relaxed); }
void prof_record(const char* name, cudaStream_t st, bool begin) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  if (begin) {
    g_prof_recs.push_back({name, prof_event(), nullptr});
    EG_CUDA(cudaEventRecord(g_prof_recs.back().a, st));
  } else {
    for (auto it = g_prof_recs.rbegin(); it != g_prof_recs.rend(); ++it)
      if (!it->b && it->name == name) {
        it->b = prof_event();
        EG_CUDA(cudaEventRecord(it->b, st));
        break;
      }
  }
}

// exported for the other translation units
int run_guarded(void (*fn)(void*), void* arg) {
  return guarded([&] { fn(arg); });
}
void set_last_error(const std::string& s) { g_last_error = s; }

static void build_tables(ensei_gpu_ctx* c) {
  using namespace host;
  const uint64_t n = c->n;
  // layout: per prime fwd[n], inv[n] (16 B each) | p fwd[n], inv[n] (8 B) | cyclic fwd[128], inv[128]
  size_t bytes_q = (size_t)c->R * 2 * n * sizeof(TwPair<uint64_t>);
  size_t bytes_p = 2 * n * sizeof(TwPair<uint32_t>);
  size_t bytes_c = 2 * 128 * sizeof(TwPair<uint32_t>);
  std::vector<uint8_t> h(bytes_q + bytes_p + bytes_c);
  auto* hq = reinterpret_cast<TwPair<uint64_t>*>(h.data());
  for (uint32_t i = 0; i < c->R; ++i) {
    TwiddleValues tv = make_twiddles(c->q[i], n, true);
    for (uint64_t k = 0; k < n; ++k) {
      hq[(2 * i) * n + k] = {tv.fwd[k], shoup64(tv.fwd[k], c->q[i])};
      hq[(2 * i + 1) * n + k] = {tv.inv[k], shoup64(tv.inv[k], c->q[i])};
    }
    c->psi_q[i] = root_of_unity(2 * n, c->q[i]);
    // RNS decryption, second generation: y_i = phi_i (Q/q_i)^-1 comes out of the inverse
    // transform itself when its last stage multiplies by n^-1 crt_inv / twi[1] crt_inv
    PrimeConst& pc = c->pc[i];
    pc.dec_ni = mulmod(tv.inv[0], pc.crt_inv, c->q[i]);
    pc.dec_ni_shoup = shoup64(pc.dec_ni, c->q[i]);
    pc.dec_t1 = mulmod(tv.inv[1], pc.crt_inv, c->q[i]);
    pc.dec_t1_shoup = shoup64(pc.dec_t1, c->q[i]);
  }
  auto* hp = reinterpret_cast<TwPair<uint32_t>*>(h.data() + bytes_q);
  {
    TwiddleValues tv = make_twiddles(c->p, n, true);
    for (uint64_t k = 0; k < n; ++k) {
      hp[k] = {(uint32_t)tv.fwd[k], (uint32_t)shoup32(tv.fwd[k], c->p)};
      hp[n + k] = {(uint32_t)tv.inv[k], (uint32_t)shoup32(tv.inv[k], c->p)};
    }
    c->psi_p = root_of_unity(2 * n, c->p);
  }
  auto* hc = reinterpret_cast<TwPair<uint32_t>*>(h.data() + bytes_q + bytes_p);
  for (uint64_t L = 2; L <= (uint64_t)kMaxTile; L <<= 1) {
    if ((c->p - 1) % L) continue;
    TwiddleValues tv = make_twiddles(c->p, L, false);
    for (uint64_t k = 0; k < L; ++k) {
      hc[L + k] = {(uint32_t)tv.fwd[k], (uint32_t)shoup32(tv.fwd[k], c->p)};
      hc[128 + L + k] = {(uint32_t)tv.inv[k], (uint32_t)shoup32(tv.inv[k], c->p)};
    }
  }
  EG_CUDA(cudaMalloc(&c->table_mem, h.size()));
  EG_CUDA(cudaMemcpy(c->table_mem, h.data(), h.size(), cudaMemcpyHostToDevice));
  auto* dq = reinterpret_cast<TwPair<uint64_t>*>(c->table_mem);
  for (uint32_t i = 0; i < c->R; ++i) {
    c->tab.tw_q_fwd[i] = dq + (2 * i) * n;
    c->tab.tw_q_inv[i] = dq + (2 * i + 1) * n;
  }
  auto* dp = reinterpret_cast<TwPair<uint32_t>*>(static_cast<uint8_t*>(c->table_mem) + bytes_q);
  c->tab.tw_p_fwd = dp;
  c->tab.tw_p_inv = dp + n;
  auto* dc = reinterpret_cast<TwPair<uint32_t>*>(static_cast<uint8_t*>(c->table_mem) + bytes_q + bytes_p);
  c->tab.tw_c_fwd = dc;
  c->tab.tw_c_inv = dc + 128;
}

static void ctx_create(int device, uint32_t n, const uint64_t* qs, uint32_t R, uint64_t p,
                       ensei_gpu_ctx** out) {
  using namespace host;
  require(out != nullptr && qs != nullptr, ENSEI_ERR_INVALID_ARGUMENT, "null argument");
  require(R >= 1 && R <= ENSEI_MAX_PRIMES, ENSEI_ERR_INVALID_ARGUMENT, "num_q must be 1..4");
  require(n >= 2 && (n & (n - 1)) == 0, ENSEI_ERR_GENERIC, "lattice dimension must be a power of two");
  require(p >= 3 && p < (1ull << 30) && is_prime(p), ENSEI_ERR_GENERIC, "p must be a prime below 2^30");
  require((p - 1) % (2 * (uint64_t)n) == 0, ENSEI_ERR_GENERIC, "p_e must be 1 mod 2n");
  auto c = std::make_unique<ensei_gpu_ctx>();
  c->device = device;
  c->n = n;
  c->logn = (uint32_t)ilog2(n);
  c->R = R;
  c->p = p;
  for (uint32_t i = 0; i < R; ++i) {
    uint64_t q = qs[i];
    require(q > p && q < (1ull << 62) && is_prime(q), ENSEI_ERR_GENERIC, "q_i must be a prime in (p, 2^62)");
    require((q - 1) % (2 * (uint64_t)n) == 0, ENSEI_ERR_GENERIC, "q must be 1 mod 2n");
    require(q % p == 1, ENSEI_ERR_GENERIC, "q must be 1 mod p_e (keeps the plaintext-wrap term small)");
    require(q > (1ull << 32), ENSEI_ERR_UNSUPPORTED, "q_i below 2^32 not supported on this path");
    c->q[i] = q;
    // MODE-0 (approximate-quotient, uncorrected CT) butterflies let forward values grow
    // to Bfly<Field64, 0>::kMaxBound * q = 31 q before the pass-boundary correction, and
    // the GS side reaches u - v + 8q < 12 q + 2^33: exact only while 31 q < 2^64
    // (q < 2^59.04).  Larger primes take MODE 1 (exact Shoup, q < 2^62) in the batched
    // transforms; the fused layer kernels are MODE 0 only and refuse them.
    if ((unsigned __int128)q * Bfly<Field64, 0>::kMaxBound >= ((unsigned __int128)1 << 64)) c->approx_ok = false;
    {  // int8 tensor-core ElementMult: the 15 byte-plane sums rebuild T = sum x y exactly
       // only while T < 2^128, i.e. K (q - 1)^2 < 2^128
      const unsigned __int128 qq = (unsigned __int128)(q - 1) * (q - 1);
      const unsigned __int128 kmax = (~(unsigned __int128)0) / qq;
      c->i8_kmax = std::min<uint32_t>(c->i8_kmax, kmax > 255 ? 255u : (uint32_t)kmax);
    }
    {  // Karatsuba MAC headroom: 2^50 + 6 Pm, 2^50 + 60 P2 < 2^64, 1008 (q-1)^2 < 2^128
      typedef unsigned __int128 u128;
      const u128 x1 = (q - 1) >> 30, xs = (u128)((1ull << 30) - 1) + x1;
      const u128 lim64 = ((u128)1 << 64) - ((u128)1 << 50);
      const u128 qq = (u128)(q - 1) * (q - 1);
      if (6 * xs * xs >= lim64 || 60 * x1 * x1 >= lim64 || qq > (~(u128)0) / 1008) c->kara_ok = false;
    }
  }
  // Delta = floor(Q / p) mod q_i.  Q == 1 mod p for every chain here (each q_i == 1 mod p),
  // so Delta = (Q - 1) / p exactly; computed per prime without big integers:
  // Delta mod q_i = -(p^-1) mod q_i  (since Delta*p = Q - 1 == -1 mod q_i).
  for (uint32_t i = 0; i < R; ++i) {
    uint64_t q = c->q[i];
    uint64_t d = (R == 1) ? q / p : (q - invmod(p % q, q)) % q;
    PrimeConst& pc = c->pc[i];
    pc.f = Field64{q, 2 * q, (uint64_t)(0 - q), 4 * q};
    pc.cred = (uint32_t)(((unsigned __int128)1 << 64) / q);
    unsigned __int128 mu = ~(unsigned __int128)0 / q;
    pc.mu_hi = (uint64_t)(mu >> 64);
    pc.mu_lo = (uint64_t)mu;
    pc.delta = d;
    pc.delta_shoup = shoup64(d, q);
    pc.cp = (uint64_t)(((unsigned __int128)p << 64) / q);
    // A2 accumulates x1*y1 < ((q >> 30) + 1)^2 per channel; stay below 2^63
    unsigned __int128 top = (unsigned __int128)((q >> 30) + 1) * ((q >> 30) + 1);
    uint64_t cap = (uint64_t)(((unsigned __int128)1 << 63) / top);
    uint64_t qi_prod = 1;
    for (uint32_t j = 0; j < R; ++j)
      if (j != i) qi_prod = mulmod(qi_prod, c->q[j] % q, q);
    pc.crt_inv = invmod(qi_prod, q);
    pc.crt_inv_shoup = shoup64(pc.crt_inv, q);
    pc.crt_c = (uint64_t)(((unsigned __int128)1 << 122) / q);
    pc.c64 = (uint64_t)(0 - q) % q;
    pc.c64p = shoup64(pc.c64, q);
    pc.a2_chunk = (uint32_t)std::max<uint64_t>(7, std::min<uint64_t>(56, cap / 7 * 7));
  }
  {  // exact CRT rounding constants: M_i = Q / q_i (<= 3 primes: 4 limbs), T_t = (2t - 1) Q (6 limbs)
    auto mul_small = [](std::vector<uint32_t>& v, uint64_t m) {  // v *= m (m < 2^62), little-endian limbs
      unsigned __int128 carry = 0;
      for (auto& w : v) {
        const unsigned __int128 t = (unsigned __int128)w * m + carry;
        w = (uint32_t)t;
        carry = t >> 32;
      }
      while (carry) {
        v.push_back((uint32_t)carry);
        carry >>= 32;
      }
    };
    std::memset(&c->crt, 0, sizeof(c->crt));
    if (R <= 3) {
      std::vector<uint32_t> Q{1};
      for (uint32_t i = 0; i < R; ++i) mul_small(Q, c->q[i]);
      for (uint32_t i = 0; i < R; ++i) {
        std::vector<uint32_t> M{1};
        for (uint32_t j = 0; j < R; ++j)
          if (j != i) mul_small(M, c->q[j]);
        for (size_t k = 0; k < M.size() && k < 4; ++k) c->crt.M[i][k] = M[k];
      }
      for (int t = 1; t <= 3; ++t) {
        std::vector<uint32_t> T = Q;
        mul_small(T, 2 * t - 1);
        for (size_t k = 0; k < T.size() && k < 6; ++k) c->crt.T[t - 1][k] = T[k];
      }
    }
  }
  if (R == 3) {  // packed CRT accumulator of layer_rns.cuh: A < 12p 2^k <= 2^48, floor(p 2^(k+64) / q_i) < 2^64
    uint32_t k = 48;
    while (k && (unsigned __int128)(12 * p) << k > ((unsigned __int128)1 << 48)) --k;
    bool ok = k >= 18 && 12 * p + 1 < (1ull << 32);
    for (uint32_t i = 0; i < R && ok; ++i) ok = ((unsigned __int128)p << k) < c->q[i];
    if (ok) {
      c->dec_kbits = k;
      for (uint32_t i = 0; i < R; ++i) c->pc[i].dec_c = (uint64_t)(((unsigned __int128)p << (k + 64)) / c->q[i]);
    }
  }
  c->pp.f = Field32{(uint32_t)p, (uint32_t)(2 * p)};
  c->pp.cred = (uint32_t)((1ull << 32) / p);
  c->pp.m64 = (uint64_t)(((unsigned __int128)1 << 64) / p);
  EG_CUDA(cudaSetDevice(device));
  EG_CUDA(cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device));
  build_tables(c.get());
  EG_CUDA(cudaStreamCreateWithFlags(&c->aux, cudaStreamNonBlocking));
  EG_CUDA(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
  EG_CUDA(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
  *out = c.release();
}

}  // namespace ensei_gpu

using namespace ensei_gpu;

extern "C" {

const char* ensei_gpu_last_error(void) { return g_last_error.c_str(); }

int ensei_gpu_profile(int enable) {
  return guarded([&] {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    for (auto& r : g_prof_recs) {
      g_prof_pool.push_back(r.a);
      if (r.b) g_prof_pool.push_back(r.b);
    }
    g_prof_recs.clear();
    g_prof.store(enable != 0);
  });
}

int ensei_gpu_profile_read(uint32_t max_kernels, char* names, double* total_ms, uint32_t* launches,
                           uint32_t* num_kernels) {
  return guarded([&] {
    require(names && total_ms && launches && num_kernels, ENSEI_ERR_INVALID_ARGUMENT, "null argument");
    std::lock_guard<std::mutex> lk(g_prof_mu);
    std::vector<std::string> order;
    std::vector<double> ms;
    std::vector<uint32_t> cnt;
    for (auto& r : g_prof_recs) {
      if (!r.b) continue;
      EG_CUDA(cudaEventSynchronize(r.b));
      float t = 0.f;
      EG_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
      size_t k = std::find(order.begin(), order.end(), r.name) - order.begin();
      if (k == order.size()) {
        order.push_back(r.name);
        ms.push_back(0.0);
        cnt.push_back(0);
      }
      ms[k] += t;
      cnt[k] += 1;
    }
    *num_kernels = (uint32_t)order.size();
    for (uint32_t k = 0; k < order.size() && k < max_kernels; ++k) {
      std::strncpy(names + 32 * k, order[k].c_str(), 31);
      names[32 * k + 31] = 0;
      total_ms[k] = ms[k];
      launches[k] = cnt[k];
    }
  });
}
int ensei_gpu_abi_version(void) { return ENSEI_GPU_ABI_VERSION; }
uint64_t ensei_gpu_launch_count(void) { return g_launches.load(); }

int ensei_gpu_ctx_create(int device, uint32_t n, const uint64_t* q_primes, uint32_t num_q, uint64_t p,
                         ensei_gpu_ctx** out) {
  return guarded([&] { ctx_create(device, n, q_primes, num_q, p, out); });
}

void ensei_gpu_ctx_destroy(ensei_gpu_ctx* ctx) {
  if (!ctx) return;
  if (ctx->table_mem) cudaFree(ctx->table_mem);
  if (ctx->aux) cudaStreamDestroy(ctx->aux);
  if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
  if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
  if (ctx->host_graph) cudaGraphExecDestroy(ctx->host_graph);
  if (ctx->host_st) cudaStreamDestroy(ctx->host_st);
  if (ctx->host_ev) cudaEventDestroy(ctx->host_ev);
  if (ctx->wire_status) cudaFree(ctx->wire_status);
  if (ctx->i8_scratch) cudaFree(ctx->i8_scratch);
  delete ctx;
}

int ensei_gpu_ctx_query(const ensei_gpu_ctx* ctx, ensei_ctx_info* info) {
  return guarded([&] {
    require(ctx && info, ENSEI_ERR_INVALID_ARGUMENT, "null argument");
    std::memset(info, 0, sizeof(*info));
    info->n = ctx->n;
    info->num_q = ctx->R;
    info->p = ctx->p;
    info->psi_p = ctx->psi_p;
    for (uint32_t i = 0; i < ctx->R; ++i) {
      info->q[i] = ctx->q[i];
      info->delta[i] = ctx->pc[i].delta;
      info->psi_q[i] = ctx->psi_q[i];
    }
    info->device = ctx->device;
    info->sm_count = ctx->sm_count;
  });
}

int ensei_gpu_negacyclic(ensei_gpu_ctx* ctx, uint32_t modulus, int inverse, int eval_layout,
                         uint64_t* d_data, size_t count, void* stream) {
  return guarded([&] {
    require(ctx && (d_data || count == 0), ENSEI_ERR_INVALID_ARGUMENT, "null argument");
    require(modulus == ENSEI_MOD_P || modulus < ctx->R, ENSEI_ERR_INVALID_ARGUMENT, "bad modulus index");
    require(eval_layout == ENSEI_LAYOUT_NATURAL || eval_layout == ENSEI_LAYOUT_BITREV,
            ENSEI_ERR_INVALID_ARGUMENT, "bad layout");
    negacyclic(ctx, modulus, inverse != 0, eval_layout == ENSEI_LAYOUT_NATURAL, d_data, count,
               (cudaStream_t)stream);
  });
}

int ensei_gpu_ntt2d(ensei_gpu_ctx* ctx, int inverse, uint32_t rows, uint32_t cols, uint64_t* d_data,
                    size_t count, void* stream) {
  return guarded([&] {
    require(ctx && (d_data || count == 0), ENSEI_ERR_INVALID_ARGUMENT, "null argument");
    auto lg = [](uint32_t v) {
      int l = 0;
      while ((1u << l) < v) ++l;
      return l;
    };
    require(rows && cols && (rows & (rows - 1)) == 0 && (cols & (cols - 1)) == 0 && rows <= 64 && cols <= 64,
            ENSEI_ERR_UNSUPPORTED, "tile sides must be powers of two <= 64 on this path");
    require((ctx->p - 1) % rows == 0 && (ctx->p - 1) % cols == 0, ENSEI_ERR_BAD_GEOMETRY,
            "tensor dims must divide p-1");
    if (rows == 1 && cols == 1) return;  // identity
    ntt2d(ctx, inverse != 0, lg(rows), lg(cols), d_data, count, (cudaStream_t)stream);
  });
}

int ensei_gpu_permute(ensei_gpu_ctx* ctx, int to_natural, uint64_t* d_data, size_t count, void* stream) {
  (void)to_natural;  // bit reversal is an involution
  return guarded([&] {
    require(ctx && (d_data || count == 0), ENSEI_ERR_INVALID_ARGUMENT, "null argument");
    permute(ctx, d_data, count, (cudaStream_t)stream);
  });
}

}  // extern "C"

// ------------------------------------------------------------ IMAD peak probe
// Issue-slot rate of the integer multiply (fmaheavy) pipe: dependent mad.lo.u32 chains
// whose operands change every iteration (8 independent chains per thread, full
// occupancy).  IMAD.WIDE / IMAD.HI occupy two of these slots each (measured ~31/clk/SM
// vs ~61/clk/SM for IMAD), which is why the roofline counts c_* in IMAD slots.
namespace ensei_gpu {
__global__ void imad_probe_kernel(uint64_t* sink, uint32_t seed, int iters) {
  uint32_t a[8], b[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    a[i] = seed * (threadIdx.x + i) + 1;
    b[i] = a[i] ^ 0x9e3779b9u;
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(b[i]), "r"(b[(i + 1) & 7]));
  }
  uint64_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s ^= a[i];
  if (s == 0x12345) sink[0] = s;
}
}  // namespace ensei_gpu

extern "C" double ensei_gpu_imad_peak(int device) {
  double out = -1.0;
  guarded([&] {
    EG_CUDA(cudaSetDevice(device));
    int sms = 0;
    EG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    uint64_t* sink;
    EG_CUDA(cudaMalloc(&sink, 64));
    cudaEvent_t e0, e1;
    EG_CUDA(cudaEventCreate(&e0));
    EG_CUDA(cudaEventCreate(&e1));
    const int blocks = sms * 8, threads = 256, iters = 4096;
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
      EG_CUDA(cudaEventRecord(e0));
      imad_probe_kernel<<<blocks, threads>>>(sink, 3, iters);
      EG_CUDA(cudaEventRecord(e1));
      EG_CUDA(cudaEventSynchronize(e1));
      float ms;
      EG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      if (rep) best = std::min(best, ms);
    }
    count_launch(4);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(sink);
    out = (double)blocks * threads * iters * 8 / (best * 1e-3);
  });
  return out;
}

// ------------------------------------------------------- tcgen05 int8 peak probe
#include "mac_tc.cuh"
namespace ensei_gpu {
template <int N>
static float tc_probe_ms(int blocks, int iters, uint32_t* sink) {
  auto k = mma_i8_peak_kernel<N>;
  EG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
  cudaEvent_t e0, e1;
  EG_CUDA(cudaEventCreate(&e0));
  EG_CUDA(cudaEventCreate(&e1));
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    EG_CUDA(cudaEventRecord(e0));
    k<<<blocks, 128, 64 * 1024>>>(iters, sink);
    EG_CUDA(cudaEventRecord(e1));
    EG_CUDA(cudaEventSynchronize(e1));
    EG_CUDA(cudaGetLastError());
    float ms;
    EG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    if (rep) best = std::min(best, ms);
  }
  count_launch(3);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return best;
}
}  // namespace ensei_gpu

extern "C" double ensei_gpu_tc_i8_peak(int device, uint32_t n_cols) {
  double out = -1.0;
  guarded([&] {
    EG_CUDA(cudaSetDevice(device));
    int sms = 0;
    EG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    uint32_t* sink;
    EG_CUDA(cudaMalloc(&sink, 64));
    const int iters = 4096;
    float ms;
    switch (n_cols) {
      case 16: ms = tc_probe_ms<16>(sms, iters, sink); break;
      case 32: ms = tc_probe_ms<32>(sms, iters, sink); break;
      case 64: ms = tc_probe_ms<64>(sms, iters, sink); break;
      case 128: ms = tc_probe_ms<128>(sms, iters, sink); break;
      case 256: ms = tc_probe_ms<256>(sms, iters, sink); break;
      default: fail(ENSEI_ERR_INVALID_ARGUMENT, "n_cols must be 16, 32, 64, 128 or 256");
    }
    cudaFree(sink);
    out = (double)sms * iters * 8 * 128.0 * n_cols * 32.0 / (ms * 1e-3);
  });
  return out;
}
