// philox.cuh -- counter-based randomness for Enc noise, a^ and HomShare shares.
//
// Philox4x32-10 (Salmon et al., SC'11), key = party seed (REF Rng::fork seed of
// Alice 0xA11CE / Bob 0xB0B, modfield.cpp:221-223), counter = (index, 0, stream id).
// Stream ids are keyed by (purpose, layer, GLOBAL image, channel, block) and the
// index by the NATURAL slot / coefficient number, so results do not depend on the
// device layout, the launch shape or how images are sharded across GPUs.  The
// test oracle restates the same streams (eo_rand_* in the oracle directory).
#pragma once
#include "modarith.cuh"

namespace ensei_gpu {

enum : uint32_t { PURPOSE_SECRET = 1, PURPOSE_NOISE = 2, PURPOSE_AHAT = 3, PURPOSE_SHARE = 4, PURPOSE_RESHARE = 5 };

__host__ __device__ inline uint64_t stream_id(uint32_t purpose, uint32_t layer, uint32_t image, uint32_t channel,
                                              uint32_t block) {
  return ((uint64_t)(purpose & 0xF) << 60) | ((uint64_t)(layer & 0xFF) << 52) | ((uint64_t)(image & 0xFFFFF) << 32) |
         ((uint64_t)(channel & 0xFFFF) << 16) | (uint64_t)(block & 0xFFFF);
}

struct Philox4 {
  uint32_t x, y, z, w;
};

EG_DEV Philox4 philox(uint64_t key, uint64_t stream, uint32_t index) {
  uint32_t c0 = index, c1 = 0, c2 = (uint32_t)stream, c3 = (uint32_t)(stream >> 32);
  uint32_t k0 = (uint32_t)key, k1 = (uint32_t)(key >> 32);
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint64_t p0 = mulw(0xD2511F53u, c0);
    uint64_t p1 = mulw(0xCD9E8D57u, c2);
    uint32_t n0 = hi32(p1) ^ c1 ^ k0;
    uint32_t n2 = hi32(p0) ^ c3 ^ k1;
    c1 = lo32(p1);
    c3 = lo32(p0);
    c0 = n0;
    c2 = n2;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return {c0, c1, c2, c3};
}

// uniform mod q from 128 bits: floor(x * q / 2^128)  (x = w:z:y:x little-endian)
EG_DEV uint64_t uniform_q_from(const Philox4& r, uint64_t q) {
  uint64_t x0 = ((uint64_t)r.y << 32) | r.x;
  uint64_t x1 = ((uint64_t)r.w << 32) | r.z;
  uint64_t h0 = mulhi64(x0, q);  // floor(x0 q / 2^64)
  // (x1 * q + h0) >> 64
  uint64_t lo = x1 * q;
  uint64_t hi = __umul64hi(x1, q);
  uint64_t s = lo + h0;
  return hi + (s < lo ? 1 : 0);
}

// uniform mod p from 64 bits: floor(x * p / 2^64)
EG_DEV uint32_t uniform_p_from(uint32_t lo, uint32_t hi, uint32_t p) {
  uint64_t x = ((uint64_t)hi << 32) | lo;
  return (uint32_t)mulhi64(x, (uint64_t)p);
}

EG_DEV int32_t cbd_from(uint32_t a, uint32_t b, uint32_t mask) {
  return (int32_t)__popc(a & mask) - (int32_t)__popc(b & mask);
}

// i-th draw of each sampler (matches eo_rand_* in the oracle)
EG_DEV uint64_t draw_uniform_q(uint64_t key, uint64_t stream, uint32_t i, uint64_t q) {
  return uniform_q_from(philox(key, stream, i), q);
}
EG_DEV uint32_t draw_uniform_p(uint64_t key, uint64_t stream, uint32_t i, uint32_t p) {
  Philox4 r = philox(key, stream, i >> 1);
  return (i & 1) ? uniform_p_from(r.z, r.w, p) : uniform_p_from(r.x, r.y, p);
}
EG_DEV int32_t draw_cbd(uint64_t key, uint64_t stream, uint32_t i, uint32_t k) {
  Philox4 r = philox(key, stream, i >> 1);
  uint32_t mask = k >= 32 ? 0xFFFFFFFFu : ((1u << k) - 1u);
  return (i & 1) ? cbd_from(r.z, r.w, mask) : cbd_from(r.x, r.y, mask);
}
EG_DEV int32_t draw_ternary(uint64_t key, uint64_t stream, uint32_t i) {
  Philox4 r = philox(key, stream, i >> 2);
  uint32_t w = (i & 2) ? ((i & 1) ? r.w : r.z) : ((i & 1) ? r.y : r.x);
  return (int32_t)hi32(mulw(w, 3u)) - 1;
}

}  // namespace ensei_gpu
