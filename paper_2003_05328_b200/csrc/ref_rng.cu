// ref_rng.cu -- REF's sequential random stream (host code), so that "parity mode"
// runs are a product feature: a caller that switches from the reference with the same
// seed gets the reference's keys, noise, masks, shares and random weights, hence
// bit-identical ciphertexts and transcripts (include/ensei_gpu.h, "reference
// randomness").
//
// REF: Rng (modfield.hpp:104-130): std::mt19937_64 seeded with the seed, fork(salt) =
// Rng(mix64(seed ^ mix64(salt))) (modfield.cpp:221-223), uniform_below by masked
// rejection (:198-207), sample_gaussian by uniform-k + exp acceptance with a 6 sigma
// tail (:209-219), next_double = 53-bit (modfield.hpp:116-118).  The stream is
// inherently sequential (one Mersenne Twister per party); the batched device kernels
// consume its draws through ensei_randomness's injected pointers.
#include <cmath>
#include <random>

#include "common.cuh"

struct ensei_ref_rng {
  std::mt19937_64 engine;
  uint64_t seed;
};

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

uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

uint64_t uniform_below(ensei_ref_rng* r, uint64_t bound) {
  if (bound == 0) fail(ENSEI_ERR_GENERIC, "uniform_below: zero bound");
  if (bound == 1) return 0;
  const int bits = 64 - __builtin_clzll(bound - 1);
  const uint64_t mask = bits == 64 ? ~0ull : ((1ull << bits) - 1);
  for (;;) {
    const uint64_t v = r->engine() & mask;
    if (v < bound) return v;
  }
}

int64_t gaussian(ensei_ref_rng* r, double sigma) {
  if (sigma <= 0) fail(ENSEI_ERR_GENERIC, "sample_gaussian: sigma must be positive");
  const int64_t tail = (int64_t)std::floor(6.0 * sigma);
  const uint64_t range = (uint64_t)(2 * tail + 1);
  const double inv2s2 = 1.0 / (2.0 * sigma * sigma);
  for (;;) {
    const int64_t k = (int64_t)uniform_below(r, range) - tail;
    const double accept = std::exp(-(double)k * (double)k * inv2s2);
    const double u = (double)(r->engine() >> 11) * 0x1.0p-53;
    if (u < accept) return k;
  }
}

}  // namespace
}  // namespace ensei_gpu

using namespace ensei_gpu;

extern "C" {

int ensei_gpu_ref_rng_create(uint64_t seed, int use_fork, uint64_t salt, ensei_ref_rng** out) {
  return guarded([&] {
    require(out != nullptr, ENSEI_ERR_INVALID_ARGUMENT, "null argument");
    const uint64_t s = use_fork ? mix64(seed ^ mix64(salt)) : seed;
    *out = new ensei_ref_rng{std::mt19937_64(s), s};
  });
}

void ensei_gpu_ref_rng_destroy(ensei_ref_rng* rng) { delete rng; }

int ensei_gpu_ref_rng_uniform_below(ensei_ref_rng* rng, uint64_t bound, uint64_t* out, size_t count) {
  return guarded([&] {
    require(rng && (out || !count), ENSEI_ERR_INVALID_ARGUMENT, "null argument");
    for (size_t i = 0; i < count; ++i) out[i] = uniform_below(rng, bound);
  });
}

int ensei_gpu_ref_rng_gaussian(ensei_ref_rng* rng, double sigma, int64_t* out, size_t count) {
  return guarded([&] {
    require(rng && (out || !count), ENSEI_ERR_INVALID_ARGUMENT, "null argument");
    for (size_t i = 0; i < count; ++i) out[i] = gaussian(rng, sigma);
  });
}

int ensei_gpu_ref_rng_next_u64(ensei_ref_rng* rng, uint64_t* out, size_t count) {
  return guarded([&] {
    require(rng && (out || !count), ENSEI_ERR_INVALID_ARGUMENT, "null argument");
    for (size_t i = 0; i < count; ++i) out[i] = rng->engine();
  });
}

}  // extern "C"
