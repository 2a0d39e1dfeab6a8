/*
 * ensei_oracle.c -- CPU ORACLE.  TEST INFRASTRUCTURE ONLY (see ensei_oracle.h).
 *
 * Plain-C restatement of the reference algorithms, written from the reference's
 * behaviour (citations "REF file:line" point into /root/reference/proj/core).
 * Deliberately simple: scalar unsigned __int128 arithmetic, no SIMD, no threads.
 */
#include "ensei_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

/* ------------------------------------------------------------------ L0 */

uint64_t eo_mulmod(uint64_t a, uint64_t b, uint64_t m) { return (uint64_t)(((u128)a * b) % m); }

/* REF modfield.hpp:35-39: single conditional correction, overflow-safe */
uint64_t eo_addmod(uint64_t a, uint64_t b, uint64_t m) {
  uint64_t s = a + b;
  if (s >= m || s < a) s -= m;
  return s;
}

/* REF modfield.hpp:40-42 */
uint64_t eo_submod(uint64_t a, uint64_t b, uint64_t m) { return a >= b ? a - b : a + m - b; }

uint64_t eo_powmod(uint64_t b, uint64_t e, uint64_t m) {
  uint64_t acc = 1 % m;
  b %= m;
  while (e) {
    if (e & 1) acc = eo_mulmod(acc, b, m);
    b = eo_mulmod(b, b, m);
    e >>= 1;
  }
  return acc;
}

uint64_t eo_invmod(uint64_t a, uint64_t m) { return eo_powmod(a, m - 2, m); }

/* deterministic Miller-Rabin for 64-bit inputs (REF modfield.cpp:89-112) */
int eo_is_prime(uint64_t n) {
  static const uint64_t bases[12] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  if (n < 2) return 0;
  for (int i = 0; i < 12; ++i)
    if (n % bases[i] == 0) return n == bases[i];
  uint64_t d = n - 1;
  int r = 0;
  while ((d & 1) == 0) { d >>= 1; ++r; }
  for (int i = 0; i < 12; ++i) {
    uint64_t x = eo_powmod(bases[i], d, n);
    if (x == 1 || x == n - 1) continue;
    int composite = 1;
    for (int k = 1; k < r; ++k) {
      x = eo_mulmod(x, x, n);
      if (x == n - 1) { composite = 0; break; }
    }
    if (composite) return 0;
  }
  return 1;
}

static uint64_t gcd_u64(uint64_t a, uint64_t b) {
  while (b) { uint64_t t = a % b; a = b; b = t; }
  return a;
}

/* Pollard rho with Floyd cycle detection; 0 on failure for this c */
static uint64_t rho(uint64_t n, uint64_t c) {
  uint64_t x = 2, y = 2, d = 1;
  while (d == 1) {
    x = (uint64_t)(((u128)x * x + c) % n);
    y = (uint64_t)(((u128)y * y + c) % n);
    y = (uint64_t)(((u128)y * y + c) % n);
    d = gcd_u64(x > y ? x - y : y - x, n);
  }
  return d == n ? 0 : d;
}

static void add_factor(uint64_t* out, int* cnt, uint64_t f) {
  for (int i = 0; i < *cnt; ++i) if (out[i] == f) return;
  out[(*cnt)++] = f;
}

static void factor_rec(uint64_t n, uint64_t* out, int* cnt) {
  if (n == 1) return;
  if (eo_is_prime(n)) { add_factor(out, cnt, n); return; }
  for (uint64_t p = 2; p < 100000 && p * p <= n; ++p) {
    if (n % p == 0) {
      add_factor(out, cnt, p);
      while (n % p == 0) n /= p;
      factor_rec(n, out, cnt);
      return;
    }
  }
  uint64_t d = 0;
  for (uint64_t c = 1; d == 0; ++c) d = rho(n, c);
  factor_rec(d, out, cnt);
  while (n % d == 0) n /= d;
  factor_rec(n, out, cnt);
}

/* smallest g whose order is p-1 (REF modfield.cpp:143-152) */
uint64_t eo_primitive_root(uint64_t p) {
  if (p == 2) return 1;
  uint64_t f[64];
  int cnt = 0;
  factor_rec(p - 1, f, &cnt);
  for (uint64_t g = 2; g < p; ++g) {
    int ok = 1;
    for (int i = 0; i < cnt && ok; ++i)
      if (eo_powmod(g, (p - 1) / f[i], p) == 1) ok = 0;
    if (ok) return g;
  }
  return 0;
}

uint64_t eo_root_of_unity(uint64_t order, uint64_t p) {
  if (order == 0 || (p - 1) % order != 0) return 0;
  return eo_powmod(eo_primitive_root(p), (p - 1) / order, p);
}

uint64_t eo_find_prime(uint64_t min_value, uint64_t residue, uint64_t modulus) {
  if (modulus == 0) return 0;
  residue %= modulus;
  uint64_t c = min_value < 2 ? 2 : min_value;
  uint64_t rem = c % modulus;
  if (rem != residue) c += residue >= rem ? residue - rem : modulus - rem + residue;
  for (; c < ((uint64_t)1 << 62); c += modulus)
    if (eo_is_prime(c)) return c;
  return 0;
}

uint64_t eo_encode_signed(int64_t v, uint64_t p) {
  int64_t r = v % (int64_t)p;
  if (r < 0) r += (int64_t)p;
  return (uint64_t)r;
}

int64_t eo_decode_signed(uint64_t r, uint64_t p) {
  return r > p / 2 ? (int64_t)r - (int64_t)p : (int64_t)r;
}

/* ------------------------------------------------------------------ L1 */

/* bit-reverse permutation then iterative DIT, twiddle wtab[j*(n/len)]
   (REF ntt_kernel.hpp:11-33) */
void eo_ntt_pow2(uint64_t* x, size_t n, const uint64_t* wtab, uint64_t m) {
  for (size_t i = 1, j = 0; i < n; ++i) {
    size_t bit = n >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) { uint64_t t = x[i]; x[i] = x[j]; x[j] = t; }
  }
  for (size_t len = 2; len <= n; len <<= 1) {
    size_t half = len / 2, step = n / len;
    for (size_t i = 0; i < n; i += len)
      for (size_t j = 0; j < half; ++j) {
        uint64_t u = x[i + j];
        uint64_t v = eo_mulmod(x[i + j + half], wtab[j * step], m);
        x[i + j] = eo_addmod(u, v, m);
        x[i + j + half] = eo_submod(u, v, m);
      }
  }
}

static int is_pow2(size_t n) { return n && !(n & (n - 1)); }

/* REF ntt.cpp:14-22: omega must be a primitive n-th root */
static int check_primitive(uint64_t omega, size_t n, uint64_t m) {
  if ((m - 1) % n != 0 || eo_powmod(omega, n, m) != 1) return -1;
  uint64_t f[64];
  int cnt = 0;
  factor_rec(n, f, &cnt);
  for (int i = 0; i < cnt; ++i)
    if (eo_powmod(omega, n / f[i], m) == 1) return -1;
  return 0;
}

int eo_ntt_1d(uint64_t* x, size_t n, uint64_t omega, uint64_t m, int inverse) {
  if (n == 0 || check_primitive(omega, n, m)) return -1;
  uint64_t w = inverse ? eo_invmod(omega, m) : omega;
  if (is_pow2(n)) {
    uint64_t* wtab = (uint64_t*)malloc(sizeof(uint64_t) * (n / 2 + 1));
    wtab[0] = 1;
    for (size_t k = 1; k < n / 2; ++k) wtab[k] = eo_mulmod(wtab[k - 1], w, m);
    eo_ntt_pow2(x, n, wtab, m);
    free(wtab);
  } else { /* O(L^2) direct path (REF ntt.cpp:35-49) */
    uint64_t* y = (uint64_t*)calloc(n, sizeof(uint64_t));
    uint64_t* wp = (uint64_t*)malloc(sizeof(uint64_t) * n);
    wp[0] = 1;
    for (size_t k = 1; k < n; ++k) wp[k] = eo_mulmod(wp[k - 1], w, m);
    for (size_t k = 0; k < n; ++k) {
      uint64_t acc = 0;
      for (size_t i = 0; i < n; ++i) acc = eo_addmod(acc, eo_mulmod(x[i], wp[(i * k) % n], m), m);
      y[k] = acc;
    }
    memcpy(x, y, n * sizeof(uint64_t));
    free(y);
    free(wp);
  }
  if (inverse) {
    uint64_t ninv = eo_invmod(n % m, m);
    for (size_t i = 0; i < n; ++i) x[i] = eo_mulmod(x[i], ninv, m);
  }
  return 0;
}

/* rows with omega_cols, then columns with omega_rows (REF ntt.cpp:112-135) */
int eo_ntt_2d(uint64_t* x, size_t rows, size_t cols, uint64_t m, int inverse) {
  if ((m - 1) % rows != 0 || (m - 1) % cols != 0) return -1;
  uint64_t wr = eo_root_of_unity(rows, m), wc = eo_root_of_unity(cols, m);
  for (size_t r = 0; r < rows; ++r)
    if (eo_ntt_1d(x + r * cols, cols, wc, m, inverse)) return -1;
  uint64_t* line = (uint64_t*)malloc(sizeof(uint64_t) * rows);
  for (size_t c = 0; c < cols; ++c) {
    for (size_t r = 0; r < rows; ++r) line[r] = x[r * cols + c];
    if (eo_ntt_1d(line, rows, wr, m, inverse)) { free(line); return -1; }
    for (size_t r = 0; r < rows; ++r) x[r * cols + c] = line[r];
  }
  free(line);
  return 0;
}

struct eo_plan {
  uint64_t m, psi;
  uint32_t n;
  uint64_t *psi_pow, *psi_inv_pow, *wtab_fwd, *wtab_inv;
};

static void power_table(uint64_t* t, uint64_t base, size_t count, uint64_t m) {
  if (!count) return;
  t[0] = 1;
  for (size_t i = 1; i < count; ++i) t[i] = eo_mulmod(t[i - 1], base, m);
}

/* REF ringbfv.cpp:30-47 */
eo_plan* eo_plan_create(uint64_t m, uint32_t n) {
  if (!is_pow2(n) || (m - 1) % (2 * (uint64_t)n) != 0) return NULL;
  eo_plan* p = (eo_plan*)calloc(1, sizeof(eo_plan));
  p->m = m;
  p->n = n;
  p->psi = eo_root_of_unity(2 * (uint64_t)n, m);
  uint64_t omega = eo_mulmod(p->psi, p->psi, m);
  p->psi_pow = (uint64_t*)malloc(8 * (size_t)n);
  p->psi_inv_pow = (uint64_t*)malloc(8 * (size_t)n);
  p->wtab_fwd = (uint64_t*)malloc(8 * (size_t)(n / 2 + 1));
  p->wtab_inv = (uint64_t*)malloc(8 * (size_t)(n / 2 + 1));
  power_table(p->psi_pow, p->psi, n, m);
  power_table(p->psi_inv_pow, eo_invmod(p->psi, m), n, m);
  uint64_t ninv = eo_invmod(n % m, m);
  for (uint32_t i = 0; i < n; ++i) p->psi_inv_pow[i] = eo_mulmod(p->psi_inv_pow[i], ninv, m);
  power_table(p->wtab_fwd, omega, n / 2, m);
  power_table(p->wtab_inv, eo_invmod(omega, m), n / 2, m);
  return p;
}

void eo_plan_destroy(eo_plan* p) {
  if (!p) return;
  free(p->psi_pow);
  free(p->psi_inv_pow);
  free(p->wtab_fwd);
  free(p->wtab_inv);
  free(p);
}

uint64_t eo_plan_psi(const eo_plan* p) { return p->psi; }

/* REF ringbfv.cpp:49-53 */
void eo_plan_forward(const eo_plan* p, uint64_t* x) {
  for (uint32_t j = 0; j < p->n; ++j) x[j] = eo_mulmod(x[j], p->psi_pow[j], p->m);
  eo_ntt_pow2(x, p->n, p->wtab_fwd, p->m);
}

/* REF ringbfv.cpp:55-59 */
void eo_plan_inverse(const eo_plan* p, uint64_t* x) {
  eo_ntt_pow2(x, p->n, p->wtab_inv, p->m);
  for (uint32_t j = 0; j < p->n; ++j) x[j] = eo_mulmod(x[j], p->psi_inv_pow[j], p->m);
}

int eo_negacyclic(uint64_t* x, uint32_t n, uint64_t m, int inverse, size_t count) {
  eo_plan* p = eo_plan_create(m, n);
  if (!p) return -1;
  for (size_t i = 0; i < count; ++i) {
    if (inverse) eo_plan_inverse(p, x + i * (size_t)n);
    else eo_plan_forward(p, x + i * (size_t)n);
  }
  eo_plan_destroy(p);
  return 0;
}

/* ------------------------------------------------------------------ PRNG */

/* Philox4x32-10 (Salmon et al., SC'11), the counter-based generator the
   device kernels use; key = 2 x 32 bits, counter = 4 x 32 bits. */
void eo_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int r = 0; r < 10; ++r) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
    uint32_t n1 = (uint32_t)p1;
    uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
    uint32_t n3 = (uint32_t)p0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* splitmix64 finalizer (REF modfield.cpp:79-85) */
uint64_t eo_mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

/* Rng::fork seed (REF modfield.cpp:221-223) */
uint64_t eo_fork_seed(uint64_t seed, uint64_t salt) { return eo_mix64(seed ^ eo_mix64(salt)); }

uint64_t eo_stream_id(uint32_t purpose, uint32_t layer, uint32_t image, uint32_t channel,
                      uint32_t block) {
  return ((uint64_t)(purpose & 0xF) << 60) | ((uint64_t)(layer & 0xFF) << 52) |
         ((uint64_t)(image & 0xFFFFF) << 32) | ((uint64_t)(channel & 0xFFFF) << 16) |
         (uint64_t)(block & 0xFFFF);
}

static void draw(uint64_t key, uint64_t stream, uint32_t index, uint32_t out[4]) {
  uint32_t ctr[4] = {index, 0u, (uint32_t)stream, (uint32_t)(stream >> 32)};
  uint32_t k[2] = {(uint32_t)key, (uint32_t)(key >> 32)};
  eo_philox4x32_10(ctr, k, out);
}

/* 4 draws per call: t = floor(3w / 2^32) - 1 in {-1, 0, 1} */
void eo_rand_ternary(uint64_t key, uint64_t stream, uint32_t n, int64_t* out) {
  uint32_t w[4];
  for (uint32_t i = 0; i < n; ++i) {
    if ((i & 3) == 0) draw(key, stream, i >> 2, w);
    out[i] = (int64_t)(((uint64_t)w[i & 3] * 3u) >> 32) - 1;
  }
}

/* centered binomial CBD(k): popc(a & mask) - popc(b & mask), 2 draws per call */
void eo_rand_cbd(uint64_t key, uint64_t stream, uint32_t n, uint32_t k, int64_t* out) {
  uint32_t w[4];
  uint32_t mask = k >= 32 ? 0xFFFFFFFFu : ((1u << k) - 1u);
  for (uint32_t i = 0; i < n; ++i) {
    if ((i & 1) == 0) draw(key, stream, i >> 1, w);
    uint32_t j = (i & 1) * 2;
    out[i] = (int64_t)__builtin_popcount(w[j] & mask) - (int64_t)__builtin_popcount(w[j + 1] & mask);
  }
}

/* uniform mod q from 128 bits: floor(x * q / 2^128), 1 draw per call */
void eo_rand_uniform_q(uint64_t key, uint64_t stream, uint32_t n, uint64_t q, uint64_t* out) {
  uint32_t w[4];
  for (uint32_t i = 0; i < n; ++i) {
    draw(key, stream, i, w);
    uint64_t x0 = ((uint64_t)w[1] << 32) | w[0];
    uint64_t x1 = ((uint64_t)w[3] << 32) | w[2];
    u128 t = (u128)x1 * q + (uint64_t)(((u128)x0 * q) >> 64);
    out[i] = (uint64_t)(t >> 64);
  }
}

/* uniform mod p from 64 bits: floor(x * p / 2^64), 2 draws per call */
void eo_rand_uniform_p(uint64_t key, uint64_t stream, uint32_t n, uint64_t p, uint64_t* out) {
  uint32_t w[4];
  for (uint32_t i = 0; i < n; ++i) {
    if ((i & 1) == 0) draw(key, stream, i >> 1, w);
    uint32_t j = (i & 1) * 2;
    uint64_t x = ((uint64_t)w[j + 1] << 32) | w[j];
    out[i] = (uint64_t)(((u128)x * p) >> 64);
  }
}

/* ---------------------------------------------- mt19937_64 (reference Rng) */

void eo_mt_seed(eo_mt* r, uint64_t seed) {
  r->seed = seed;
  r->mt[0] = seed;
  for (uint32_t i = 1; i < 312; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + i;
  r->idx = 312;
}

uint64_t eo_mt_next(eo_mt* r) {
  if (r->idx >= 312) {
    for (uint32_t i = 0; i < 312; ++i) {
      uint64_t x = (r->mt[i] & 0xFFFFFFFF80000000ULL) | (r->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t xa = x >> 1;
      if (x & 1) xa ^= 0xB5026F5AA96619E9ULL;
      r->mt[i] = r->mt[(i + 156) % 312] ^ xa;
    }
    r->idx = 0;
  }
  uint64_t y = r->mt[r->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

void eo_mt_fork(const eo_mt* parent, uint64_t salt, eo_mt* child) {
  eo_mt_seed(child, eo_fork_seed(parent->seed, salt));
}

/* masked rejection (REF modfield.cpp:198-207) */
uint64_t eo_mt_uniform_below(eo_mt* r, uint64_t bound) {
  if (bound <= 1) return 0;
  int bits = 64 - __builtin_clzll(bound - 1);
  uint64_t mask = bits == 64 ? ~(uint64_t)0 : (((uint64_t)1 << bits) - 1);
  for (;;) {
    uint64_t v = eo_mt_next(r) & mask;
    if (v < bound) return v;
  }
}

/* rejection-sampled discrete Gaussian, 6-sigma tail (REF modfield.cpp:209-219) */
int64_t eo_mt_gaussian(eo_mt* r, double sigma) {
  int64_t tail = (int64_t)floor(6.0 * sigma);
  uint64_t range = (uint64_t)(2 * tail + 1);
  double inv2s2 = 1.0 / (2.0 * sigma * sigma);
  for (;;) {
    int64_t k = (int64_t)eo_mt_uniform_below(r, range) - tail;
    double accept = exp(-(double)k * (double)k * inv2s2);
    double u = (double)(eo_mt_next(r) >> 11) * 0x1.0p-53;
    if (u < accept) return k;
  }
}

/* ------------------------------------------------------------------ L2/L3 */

/* REF ntt.cpp:51-61 */
static uint32_t choose_padded_len(uint32_t min_len, uint64_t p) {
  uint64_t order = p - 1;
  uint32_t p2 = 1;
  while (p2 < min_len) p2 <<= 1;
  if (order % p2 == 0) return p2;
  uint64_t cap = order < (1u << 20) ? order : (1u << 20);
  for (uint64_t l = min_len; l <= cap; ++l)
    if (order % l == 0) return (uint32_t)l;
  return 0;
}

int eo_layer_init(eo_layer* L, uint64_t q, uint64_t p, uint32_t n, uint32_t H, uint32_t W,
                  uint32_t fh, uint32_t fw, uint32_t same, uint32_t cin, uint32_t cout) {
  memset(L, 0, sizeof(*L));
  if (!H || !W || !fh || !fw || !cin || !cout || !is_pow2(n)) return -1;
  if (!same && (fh > H || fw > W)) return -1;
  /* make_rlwe_params invariants (REF ringbfv.cpp:65-87) */
  if (q <= p || (q - 1) % (2 * (uint64_t)n) || (p - 1) % (2 * (uint64_t)n) || q % p != 1) return -2;
  L->q = q; L->p = p; L->n = n; L->H = H; L->W = W; L->fh = fh; L->fw = fw;
  L->same = same; L->cin = cin; L->cout = cout;
  L->Lh = choose_padded_len(H + fh - 1, p);
  L->Lw = choose_padded_len(W + fw - 1, p);
  if (!L->Lh || !L->Lw) return -3;
  L->blocks = (L->Lh * L->Lw + n - 1) / n;
  L->oh = same ? H : H - fh + 1;
  L->ow = same ? W : W - fw + 1;
  L->r0 = same ? (fh - 1) / 2 : fh - 1;
  L->c0 = same ? (fw - 1) / 2 : fw - 1;
  L->delta = q / p;
  L->pack = 1;
  return 0;
}

static uint32_t pack_of(const eo_layer* L) { return L->pack > 1 ? L->pack : 1; }

void eo_secret_eval(const eo_layer* L, const int64_t* t, uint64_t* t_eval) {
  eo_plan* pq = eo_plan_create(L->q, L->n);
  for (uint32_t i = 0; i < L->n; ++i) t_eval[i] = eo_encode_signed(t[i], L->q);
  eo_plan_forward(pq, t_eval);
  eo_plan_destroy(pq);
}

/* pad a residue tile at the grid origin, 2D NTT, flatten, split into zero-filled
   blocks (REF ntt.cpp:155-185, protocol.cpp:18-29).  Packed layers: the pack's tiles
   (tile of image i at tile + i * stride; stride 0 = one tile replicated, the weights)
   land at slots [i G, (i + 1) G) */
static void grid_forward(const eo_layer* L, const uint64_t* tile, uint32_t th, uint32_t tw,
                         uint64_t* blocks /* [B][n] */, size_t stride) {
  size_t G = (size_t)L->Lh * L->Lw;
  uint64_t* g = (uint64_t*)calloc(G, 8);
  memset(blocks, 0, 8 * (size_t)L->blocks * L->n);
  for (uint32_t k = 0; k < pack_of(L); ++k) {
    const uint64_t* t = tile + (size_t)k * stride;
    memset(g, 0, 8 * G);
    for (uint32_t r = 0; r < th; ++r)
      for (uint32_t c = 0; c < tw; ++c) g[(size_t)r * L->Lw + c] = t[(size_t)r * tw + c] % L->p;
    eo_ntt_2d(g, L->Lh, L->Lw, L->p, 0);
    memcpy(blocks + (size_t)k * G, g, 8 * G);
  }
  free(g);
}

/* merge blocks to the grid, IDFT2D, crop (REF protocol.cpp:31-53); packed: the grid of
   image k at slots [k G, (k + 1) G) -> out + k * stride */
static void grid_inverse_crop(const eo_layer* L, const uint64_t* blocks, uint64_t* out, size_t stride) {
  size_t G = (size_t)L->Lh * L->Lw;
  uint64_t* g = (uint64_t*)malloc(8 * G);
  for (uint32_t k = 0; k < pack_of(L); ++k) {
    for (size_t i = 0; i < G; ++i) g[i] = blocks[(size_t)k * G + i] % L->p;
    eo_ntt_2d(g, L->Lh, L->Lw, L->p, 1);
    for (uint32_t r = 0; r < L->oh; ++r)
      for (uint32_t c = 0; c < L->ow; ++c)
        out[(size_t)k * stride + (size_t)r * L->ow + c] = g[(size_t)(r + L->r0) * L->Lw + (c + L->c0)];
  }
  free(g);
}

/* add_plain(ct, m, +1) in the evaluation domain (REF ringbfv.cpp:248-263) */
static void add_plain_eval(const eo_layer* L, const eo_plan* pq, const eo_plan* pp,
                           const uint64_t* slots, uint64_t* c1) {
  uint32_t n = L->n;
  uint64_t* enc = (uint64_t*)malloc(8 * (size_t)n);
  memcpy(enc, slots, 8 * (size_t)n);
  eo_plan_inverse(pp, enc);
  for (uint32_t i = 0; i < n; ++i) enc[i] = eo_mulmod(enc[i] % L->q, L->delta % L->q, L->q);
  eo_plan_forward(pq, enc);
  for (uint32_t i = 0; i < n; ++i) c1[i] = eo_addmod(c1[i], enc[i], L->q);
  free(enc);
}

void eo_prepare_weights(const eo_layer* L, const int64_t* w, uint64_t* w_eval) {
  uint32_t n = L->n, B = L->blocks;
  eo_plan* pq = eo_plan_create(L->q, n);
  eo_plan* pp = eo_plan_create(L->p, n);
  uint64_t* tile = (uint64_t*)malloc(8 * (size_t)L->fh * L->fw);
  uint64_t* blk = (uint64_t*)malloc(8 * (size_t)B * n);
  for (uint32_t o = 0; o < L->cout; ++o)
    for (uint32_t c = 0; c < L->cin; ++c) {
      const int64_t* f = w + ((size_t)o * L->cin + c) * L->fh * L->fw;
      for (uint32_t i = 0; i < L->fh * L->fw; ++i) tile[i] = eo_encode_signed(f[i], L->p);
      grid_forward(L, tile, L->fh, L->fw, blk, 0); /* packed: replicated across the pack */
      for (uint32_t b = 0; b < B; ++b) {
        uint64_t* dst = w_eval + (((size_t)o * L->cin + c) * B + b) * n;
        memcpy(dst, blk + (size_t)b * n, 8 * (size_t)n);
        eo_plan_inverse(pp, dst); /* encode_slots */
        for (uint32_t i = 0; i < n; ++i)
          dst[i] = eo_encode_signed(eo_decode_signed(dst[i], L->p), L->q); /* centered lift */
        eo_plan_forward(pq, dst);
      }
    }
  free(tile);
  free(blk);
  eo_plan_destroy(pq);
  eo_plan_destroy(pp);
}

void eo_alice_encrypt(const eo_layer* L, const uint64_t* t_eval, const uint64_t* in,
                      const int64_t* e, const uint64_t* a_hat, uint64_t* ct) {
  uint32_t n = L->n, B = L->blocks;
  uint64_t q = L->q;
  eo_plan* pq = eo_plan_create(q, n);
  eo_plan* pp = eo_plan_create(L->p, n);
  uint64_t* blk = (uint64_t*)malloc(8 * (size_t)B * n);
  for (uint32_t c = 0; c < L->cin; ++c) {
    grid_forward(L, in + (size_t)c * L->H * L->W, L->H, L->W, blk, (size_t)L->cin * L->H * L->W);
    for (uint32_t b = 0; b < B; ++b) {
      size_t rb = ((size_t)c * B + b) * n;
      uint64_t* m = blk + (size_t)b * n;
      eo_plan_inverse(pp, m); /* encode_slots */
      for (uint32_t i = 0; i < n; ++i) /* scale_message (REF ringbfv.cpp:130-139) */
        m[i] = eo_addmod(eo_mulmod(m[i] % q, L->delta % q, q), eo_encode_signed(e[rb + i], q), q);
      eo_plan_forward(pq, m);
      uint64_t* c0 = ct + ((size_t)c * B + b) * 2 * n;
      uint64_t* c1 = c0 + n;
      for (uint32_t i = 0; i < n; ++i) {
        uint64_t a = a_hat[rb + i];
        c0[i] = a == 0 ? 0 : q - a;
        c1[i] = eo_addmod(eo_mulmod(a, t_eval[i], q), m[i], q);
      }
    }
  }
  free(blk);
  eo_plan_destroy(pq);
  eo_plan_destroy(pp);
}

void eo_bob_eval(const eo_layer* L, const uint64_t* ct_in, const uint64_t* w_eval,
                 const uint64_t* bob_prev, const uint64_t* s_b, uint64_t* ct_out,
                 uint64_t* bob_share) {
  uint32_t n = L->n, B = L->blocks;
  uint64_t q = L->q, p = L->p;
  size_t ctw = (size_t)2 * n;
  eo_plan* pq = eo_plan_create(q, n);
  eo_plan* pp = eo_plan_create(p, n);
  uint64_t* cts = (uint64_t*)malloc(8 * (size_t)L->cin * B * ctw);
  memcpy(cts, ct_in, 8 * (size_t)L->cin * B * ctw);
  uint64_t* blk = (uint64_t*)malloc(8 * (size_t)B * n);
  if (bob_prev) { /* HomRec with Bob's transformed share (REF protocol.cpp:543-557, hss.cpp:51-62) */
    for (uint32_t c = 0; c < L->cin; ++c) {
      grid_forward(L, bob_prev + (size_t)c * L->H * L->W, L->H, L->W, blk, (size_t)L->cin * L->H * L->W);
      for (uint32_t b = 0; b < B; ++b)
        add_plain_eval(L, pq, pp, blk + (size_t)b * n, cts + ((size_t)c * B + b) * ctw + n);
    }
  }
  uint64_t* mask = (uint64_t*)malloc(8 * (size_t)n);
  uint64_t* merged = (uint64_t*)malloc(8 * (size_t)B * n);
  for (uint32_t o = 0; o < L->cout; ++o) {
    for (uint32_t b = 0; b < B; ++b) {
      uint64_t* acc = ct_out + ((size_t)o * B + b) * ctw;
      memset(acc, 0, 8 * ctw);
      for (uint32_t c = 0; c < L->cin; ++c) { /* mul_plain + add_ct (REF ringbfv.cpp:233-306) */
        const uint64_t* x = cts + ((size_t)c * B + b) * ctw;
        const uint64_t* wv = w_eval + (((size_t)o * L->cin + c) * B + b) * n;
        for (uint32_t i = 0; i < n; ++i) {
          acc[i] = eo_addmod(acc[i], eo_mulmod(x[i], wv[i], q), q);
          acc[n + i] = eo_addmod(acc[n + i], eo_mulmod(x[n + i], wv[i], q), q);
        }
      }
      /* HomShare: mask = (p_A - s_B) mod p_E (REF hss.cpp:22-41) */
      const uint64_t* sb = s_b + ((size_t)o * B + b) * n;
      for (uint32_t i = 0; i < n; ++i) mask[i] = (p - sb[i]) % p;
      add_plain_eval(L, pq, pp, mask, acc + n);
      memcpy(merged + (size_t)b * n, sb, 8 * (size_t)n);
    }
    grid_inverse_crop(L, merged, bob_share + (size_t)o * L->oh * L->ow, (size_t)L->cout * L->oh * L->ow);
  }
  free(mask);
  free(merged);
  free(blk);
  free(cts);
  eo_plan_destroy(pq);
  eo_plan_destroy(pp);
}

void eo_alice_decrypt(const eo_layer* L, const uint64_t* t_eval, const uint64_t* ct_out,
                      uint64_t* alice_share) {
  uint32_t n = L->n, B = L->blocks;
  uint64_t q = L->q, p = L->p;
  eo_plan* pq = eo_plan_create(q, n);
  eo_plan* pp = eo_plan_create(p, n);
  uint64_t* merged = (uint64_t*)malloc(8 * (size_t)B * n);
  for (uint32_t o = 0; o < L->cout; ++o) {
    for (uint32_t b = 0; b < B; ++b) {
      const uint64_t* c0 = ct_out + ((size_t)o * B + b) * 2 * n;
      const uint64_t* c1 = c0 + n;
      uint64_t* phi = merged + (size_t)b * n;
      for (uint32_t i = 0; i < n; ++i) phi[i] = eo_addmod(eo_mulmod(c0[i], t_eval[i], q), c1[i], q);
      eo_plan_inverse(pq, phi);
      for (uint32_t i = 0; i < n; ++i) { /* exact rounding (REF ringbfv.cpp:222-229) */
        u128 num = (u128)p * phi[i] + q / 2;
        phi[i] = (uint64_t)((num / q) % p);
      }
      eo_plan_forward(pp, phi); /* decode_slots */
    }
    grid_inverse_crop(L, merged, alice_share + (size_t)o * L->oh * L->ow, (size_t)L->cout * L->oh * L->ow);
  }
  free(merged);
  eo_plan_destroy(pq);
  eo_plan_destroy(pp);
}

void eo_conv_direct(const eo_layer* L, const uint64_t* in, const int64_t* w, uint64_t* out) {
  uint64_t p = L->p;
  uint32_t fullh = L->H + L->fh - 1, fullw = L->W + L->fw - 1;
  uint64_t* full = (uint64_t*)malloc(8 * (size_t)fullh * fullw);
  for (uint32_t o = 0; o < L->cout; ++o) {
    uint64_t* dst = out + (size_t)o * L->oh * L->ow;
    memset(dst, 0, 8 * (size_t)L->oh * L->ow);
    for (uint32_t c = 0; c < L->cin; ++c) {
      const uint64_t* img = in + (size_t)c * L->H * L->W;
      const int64_t* f = w + ((size_t)o * L->cin + c) * L->fh * L->fw;
      memset(full, 0, 8 * (size_t)fullh * fullw);
      for (uint32_t i = 0; i < L->H; ++i)
        for (uint32_t j = 0; j < L->W; ++j) {
          uint64_t u = img[(size_t)i * L->W + j] % p;
          if (!u) continue;
          for (uint32_t a = 0; a < L->fh; ++a)
            for (uint32_t b = 0; b < L->fw; ++b) {
              uint64_t* y = &full[(size_t)(i + a) * fullw + (j + b)];
              *y = eo_addmod(*y, eo_mulmod(u, eo_encode_signed(f[a * L->fw + b], p), p), p);
            }
        }
      for (uint32_t r = 0; r < L->oh; ++r)
        for (uint32_t cc = 0; cc < L->ow; ++cc) {
          uint64_t* d = &dst[(size_t)r * L->ow + cc];
          *d = eo_addmod(*d, full[(size_t)(r + L->r0) * fullw + (cc + L->c0)], p);
        }
    }
  }
  free(full);
}

int eo_activation(uint64_t* v, size_t len, uint64_t p, int fn) {
  int64_t half = (int64_t)(p / 2);
  for (size_t i = 0; i < len; ++i) {
    int64_t y = eo_decode_signed(v[i] % p, p), o = y;
    if (fn == 0) o = y > 0 ? y : 0;
    else if (fn == 1) {
      __int128 sq = (__int128)y * y;
      if (sq > half) return -1;
      o = (int64_t)sq;
    }
    v[i] = eo_encode_signed(o, p);
  }
  return 0;
}

/* ------------------------------------------------------------------ RNS */

/* little-endian 64-bit limb helpers, at most 4 limbs */
static void big_mul_small(uint64_t* a, int na, uint64_t s) {
  u128 carry = 0;
  for (int i = 0; i < na; ++i) {
    u128 t = (u128)a[i] * s + carry;
    a[i] = (uint64_t)t;
    carry = t >> 64;
  }
}
static void big_add(uint64_t* a, const uint64_t* b, int na) {
  u128 carry = 0;
  for (int i = 0; i < na; ++i) {
    u128 t = (u128)a[i] + b[i] + carry;
    a[i] = (uint64_t)t;
    carry = t >> 64;
  }
}
static int big_cmp(const uint64_t* a, const uint64_t* b, int na) {
  for (int i = na - 1; i >= 0; --i) {
    if (a[i] != b[i]) return a[i] > b[i] ? 1 : -1;
  }
  return 0;
}
static void big_sub(uint64_t* a, const uint64_t* b, int na) {
  uint64_t borrow = 0;
  for (int i = 0; i < na; ++i) {
    uint64_t bi = b[i] + borrow;
    uint64_t nb = (bi < borrow) || (a[i] < bi);
    a[i] -= bi;
    borrow = nb;
  }
}
static void big_shl1(uint64_t* a, int na) {
  for (int i = na - 1; i > 0; --i) a[i] = (a[i] << 1) | (a[i - 1] >> 63);
  a[0] <<= 1;
}
static void big_shr1(uint64_t* a, int na) {
  for (int i = 0; i < na - 1; ++i) a[i] = (a[i] >> 1) | (a[i + 1] << 63);
  a[na - 1] >>= 1;
}

/* phi = CRT(res) in [0, Q); returns floor((p*phi + floor(Q/2)) / Q) mod p */
uint64_t eo_crt_round(const uint64_t* res, const uint64_t* qs, uint32_t R, uint64_t p) {
  enum { NL = 5 };
  uint64_t Q[NL] = {1, 0, 0, 0, 0}, phi[NL] = {0};
  for (uint32_t i = 0; i < R; ++i) big_mul_small(Q, NL, qs[i]);
  for (uint32_t i = 0; i < R; ++i) {
    /* term = res_i * (Q/q_i) * ((Q/q_i)^-1 mod q_i) */
    uint64_t Qi[NL] = {1, 0, 0, 0, 0};
    uint64_t inv = 1;
    for (uint32_t j = 0; j < R; ++j)
      if (j != i) {
        big_mul_small(Qi, NL, qs[j]);
        inv = eo_mulmod(inv, qs[j] % qs[i], qs[i]);
      }
    inv = eo_invmod(inv, qs[i]);
    big_mul_small(Qi, NL, eo_mulmod(res[i] % qs[i], inv, qs[i]));
    big_add(phi, Qi, NL);
  }
  while (big_cmp(phi, Q, NL) >= 0) big_sub(phi, Q, NL);
  /* num = p*phi + floor(Q/2) */
  uint64_t num[NL], half[NL];
  memcpy(num, phi, sizeof num);
  big_mul_small(num, NL, p);
  memcpy(half, Q, sizeof half);
  big_shr1(half, NL);
  big_add(num, half, NL);
  /* quotient by shift-subtract; quotient < 2^64 */
  uint64_t D[NL];
  memcpy(D, Q, sizeof D);
  int shift = 0;
  while (big_cmp(D, num, NL) <= 0 && !(D[NL - 1] >> 63)) { big_shl1(D, NL); ++shift; }
  uint64_t quo = 0;
  for (int s = shift; s >= 0; --s) {
    if (big_cmp(num, D, NL) >= 0) { big_sub(num, D, NL); quo |= (uint64_t)1 << s; }
    big_shr1(D, NL);
  }
  return quo % p;
}

void eo_alice_decrypt_rns(const eo_layer* Ls, uint32_t R, const uint64_t* t_evals,
                          const uint64_t* ct_out, uint64_t* alice_share) {
  const eo_layer* L = &Ls[0];
  uint32_t n = L->n, B = L->blocks;
  uint64_t p = L->p;
  uint64_t qs[8];
  eo_plan* pq[8];
  for (uint32_t r = 0; r < R; ++r) {
    qs[r] = Ls[r].q;
    pq[r] = eo_plan_create(qs[r], n);
  }
  eo_plan* pp = eo_plan_create(p, n);
  uint64_t* phi = (uint64_t*)malloc(8 * (size_t)R * n);
  uint64_t* merged = (uint64_t*)malloc(8 * (size_t)B * n);
  for (uint32_t o = 0; o < L->cout; ++o) {
    for (uint32_t b = 0; b < B; ++b) {
      const uint64_t* base = ct_out + ((size_t)o * B + b) * 2 * R * n;
      for (uint32_t r = 0; r < R; ++r) { /* phi_r = INTT(c0 t + c1) mod q_r (REF ringbfv.cpp:208-212) */
        const uint64_t* c0 = base + (size_t)r * n;
        const uint64_t* c1 = base + (size_t)(R + r) * n;
        uint64_t* ph = phi + (size_t)r * n;
        for (uint32_t i = 0; i < n; ++i)
          ph[i] = eo_addmod(eo_mulmod(c0[i], t_evals[(size_t)r * n + i], qs[r]), c1[i], qs[r]);
        eo_plan_inverse(pq[r], ph);
      }
      uint64_t* m = merged + (size_t)b * n;
      uint64_t res[8];
      for (uint32_t i = 0; i < n; ++i) {
        for (uint32_t r = 0; r < R; ++r) res[r] = phi[(size_t)r * n + i];
        m[i] = eo_crt_round(res, qs, R, p);
      }
      eo_plan_forward(pp, m); /* decode_slots */
    }
    grid_inverse_crop(L, merged, alice_share + (size_t)o * L->oh * L->ow, (size_t)L->cout * L->oh * L->ow);
  }
  free(phi);
  free(merged);
  for (uint32_t r = 0; r < R; ++r) eo_plan_destroy(pq[r]);
  eo_plan_destroy(pp);
}
