// params.cu -- parameter selection (host code): REF params.cpp restated, with an RNS
// extension where REF's single-prime q runs out (include/ensei_gpu.h, "parameters").
//
// REF: min_pntt / checked_bound (params.cpp:35-45, 79-89), derive_q (:49-60),
// assemble (:62-74), build_params (:91-117), preset_params (:119-144), find_prime
// (modfield.cpp:173-183), FieldSpec::make range (modfield.cpp:120-124),
// make_rlwe_params invariants (ringbfv.cpp:65-87), ModulusChain::make (hss.cpp:7-16).
//
// Extension: when derive_q's requirement reaches 2^62 -- REF
// throws SearchExhausted from about 100-way channel accumulation at n = 2048 -- and
// the caller allows max_primes > 1, q becomes a product of R primes, the smallest
// ones >= 2^59 that are == 1 (mod 2n p_e) (each keeps every REF invariant: prime,
// < 2^62, == 1 mod 2n, == 1 mod p_e, so Q == 1 mod p_e and Delta = (Q-1)/p_e), with R
// minimal (or min_primes) such that Q >= q_min.  Below the cap the result is REF's q.
#include <cmath>
#include <cstring>
#include <string>

#include "common.cuh"
#include "host_field.hpp"

namespace ensei_gpu {

int run_guarded(void (*fn)(void*), void* arg);

namespace {

template <class Fn>
int guarded(Fn&& fn) {
  struct Box {
    Fn* f;
  } box{&fn};
  return run_guarded([](void* p) { (*static_cast<Box*>(p)->f)(); }, &box);
}

using host::u128;
using host::u64;
constexpr u64 kMaxModulus = 1ull << 62;

u64 find_prime(u64 min_value, u64 residue, u64 modulus) {
  require(modulus != 0, ENSEI_ERR_GENERIC, "find_prime: zero modulus");
  residue %= modulus;
  u64 c = min_value < 2 ? 2 : min_value;
  u64 rem = c % modulus;
  if (rem != residue) c += (residue >= rem ? residue - rem : modulus - rem + residue);
  for (; c < kMaxModulus; c += modulus)
    if (host::is_prime(c)) return c;
  fail(ENSEI_ERR_SEARCH_EXHAUSTED, "find_prime: no prime below 2^62 ceiling");
}

u64 checked_bound(u64 max_u, u64 max_w, u64 f_h, u64 f_w) {
  u128 b = (u128)max_u * max_w;
  b *= f_h;
  b *= f_w;
  if (b >= ((u128)1 << 62)) fail(ENSEI_ERR_RANGE_VIOLATION, "dynamic-range bound exceeds the 62-bit modulus cap");
  return (u64)b;
}

u64 min_pntt(const ensei_precision_profile& p) {
  if (p.input_bits <= 0 || p.filter_bits <= 0 || p.f_h <= 0 || p.f_w <= 0)
    fail(ENSEI_ERR_RANGE_VIOLATION, "profile fields must be positive");
  if (p.input_bits > 32 || p.filter_bits > 32) fail(ENSEI_ERR_RANGE_VIOLATION, "bit widths above 32 are unsupported");
  return checked_bound(1ull << p.input_bits, 1ull << p.filter_bits, (u64)p.f_h, (u64)p.f_w);
}

void field_check(u64 m) {  // FieldSpec::make
  if (m < 2 || m >= kMaxModulus) fail(ENSEI_ERR_GENERIC, "FieldSpec: modulus out of range [2, 2^62)");
  if (!host::is_prime(m)) fail(ENSEI_ERR_GENERIC, "FieldSpec: modulus is not prime");
}

// derive_q's requirement: one full-range plaintext product, accum-way accumulation,
// the share masks, one spare bit.
double q_min_of(u64 p_e, uint32_t n, double sigma, uint64_t accum) {
  double a = (double)(accum < 1 ? 1 : accum);
  double w_inf = (double)p_e / 2.0;
  double factor = (double)n * w_inf;
  double bound_after = a * factor * (6.0 * sigma + 1.0);
  double mass_after = a * factor * 4.0 + 8.0;
  return 4.0 * (double)p_e * (bound_after + mass_after);
}

void assemble(u64 p_n, u64 p_a, u64 p_e, uint32_t n, uint32_t mode, uint64_t accum,
              const ensei_precision_profile& prof, double sigma, uint32_t max_primes, uint32_t min_primes,
              ensei_param_set* out) {
  field_check(p_n);
  field_check(p_a);
  field_check(p_e);
  if (!(p_e >= p_a && p_a >= p_n)) fail(ENSEI_ERR_CHAIN_VIOLATION, "moduli must satisfy p_e >= p_a >= p_n");
  require(max_primes >= 1 && max_primes <= ENSEI_MAX_PRIMES && min_primes <= max_primes, ENSEI_ERR_INVALID_ARGUMENT,
          "prime counts must satisfy 1 <= min_primes <= max_primes <= ENSEI_MAX_PRIMES");
  std::memset(out, 0, sizeof(*out));
  const double qmin = q_min_of(p_e, n, sigma, accum);
  const u64 step = (u64)(2ull * n) * p_e;
  out->log2_q_min = std::log2(qmin);
  if (qmin < std::ldexp(1.0, 62) && min_primes <= 1) {
    out->q[0] = find_prime((u64)qmin + 1, 1, step);
    out->num_q = 1;
  } else {
    if (max_primes <= 1) fail(ENSEI_ERR_SEARCH_EXHAUSTED, "required ciphertext modulus exceeds 2^62");
    double log2_Q = 0;
    u64 c = 1ull << 59;
    uint32_t r = 0;
    while (r < max_primes && (r < min_primes || log2_Q < out->log2_q_min)) {
      c = find_prime(c, 1, step);
      out->q[r++] = c;
      log2_Q += std::log2((double)c);
      c += step;
    }
    if (log2_Q < out->log2_q_min)
      fail(ENSEI_ERR_SEARCH_EXHAUSTED, "required ciphertext modulus exceeds max_primes RNS primes");
    out->num_q = r;
  }
  // make_rlwe_params invariants, per prime
  require((n & (n - 1)) == 0 && n, ENSEI_ERR_GENERIC, "lattice dimension must be a power of two");
  for (uint32_t i = 0; i < out->num_q; ++i) {
    const u64 q = out->q[i];
    if (q <= p_e) fail(ENSEI_ERR_GENERIC, "q must exceed p_e");
    field_check(q);
    if ((q - 1) % (2ull * n)) fail(ENSEI_ERR_GENERIC, "q must be 1 mod 2n");
    if (q % p_e != 1) fail(ENSEI_ERR_GENERIC, "q must be 1 mod p_e (keeps the plaintext-wrap term small)");
  }
  if ((p_e - 1) % (2ull * n)) fail(ENSEI_ERR_GENERIC, "p_e must be 1 mod 2n");
  if (out->num_q == 1 && out->q[0] / p_e < 2) fail(ENSEI_ERR_GENERIC, "floor(q/p_e) must be at least 2");
  out->p_n = p_n;
  out->p_a = p_a;
  out->p_e = p_e;
  out->n = n;
  out->sigma = sigma;
  out->mode = mode;
  out->insecure = n < 1024;
  out->profile = prof;
}

struct Preset {
  const char* name;
  u64 p_n, p_e;
  ensei_precision_profile profile;
};
// REF kPresets (params.cpp:22-27): the published candidate sets, run unified at p = p_e
const Preset kPresets[] = {
    {"binary", 2311, 12289, {8, 1, 3, 3}},
    {"medium", 147457, 147457, {8, 4, 3, 3}},
    {"high", 2359303, 2363393, {12, 6, 3, 3}},
};

}  // namespace
}  // namespace ensei_gpu

using namespace ensei_gpu;

extern "C" {

int ensei_gpu_min_pntt(const ensei_precision_profile* profile, uint64_t* out) {
  return guarded([&] {
    require(profile && out, ENSEI_ERR_INVALID_ARGUMENT, "null argument");
    *out = min_pntt(*profile);
  });
}

int ensei_gpu_build_params(const ensei_precision_profile* profile, uint32_t n, uint32_t mode, uint64_t accum_channels,
                           uint64_t p_n_floor, double sigma, uint32_t max_primes, uint32_t min_primes,
                           ensei_param_set* out) {
  return guarded([&] {
    require(profile && out, ENSEI_ERR_INVALID_ARGUMENT, "null argument");
    require(mode == ENSEI_CHAIN_UNIFIED || mode == ENSEI_CHAIN_SPLIT_PAPER, ENSEI_ERR_INVALID_ARGUMENT, "bad mode");
    const u64 bound = std::max<u64>(min_pntt(*profile), p_n_floor);
    if (mode == ENSEI_CHAIN_UNIFIED) {
      const u64 p = find_prime(std::max<u64>(bound, 2ull * n + 1), 1, 2ull * n);
      assemble(p, p, p, n, mode, accum_channels, *profile, sigma, max_primes, min_primes, out);
      return;
    }
    const u64 pn = find_prime(bound, 1, 4096);
    const u64 pe = find_prime(std::max<u64>(pn, 2ull * n + 1), 1, 2ull * n);
    const u128 peak = (u128)(pn - 1) * (pn - 1) + pn;
    if (peak > pe) fail(ENSEI_ERR_RANGE_VIOLATION, "split-moduli no-wrap violated: (p_n-1)^2 + p_n exceeds p_e");
    assemble(pn, pn, pe, n, mode, accum_channels, *profile, sigma, max_primes, min_primes, out);
  });
}

int ensei_gpu_preset_params(const char* name, uint64_t accum_channels, uint32_t max_primes, ensei_param_set* out) {
  return guarded([&] {
    require(name && out, ENSEI_ERR_INVALID_ARGUMENT, "null argument");
    const std::string nm(name);
    if (nm == "toy") {
      ensei_precision_profile prof{2, 2, 2, 2};
      assemble(97, 97, 97, 16, ENSEI_CHAIN_UNIFIED, std::max<uint64_t>(accum_channels, 4), prof, 4.0, max_primes, 1,
               out);
      return;
    }
    for (const Preset& r : kPresets) {
      if (nm != r.name) continue;
      assemble(r.p_e, r.p_e, r.p_e, 2048, ENSEI_CHAIN_UNIFIED, accum_channels, r.profile, 4.0, max_primes, 1, out);
      return;
    }
    fail(ENSEI_ERR_RANGE_VIOLATION, "unknown preset: " + nm);
  });
}

}  // extern "C"
