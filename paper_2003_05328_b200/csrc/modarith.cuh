// modarith.cuh -- modular arithmetic for the two moduli of the ENSEI hot path.
//
//   Field64: the 60-bit ciphertext modulus q (any prime q < 2^62 works; the lazy
//            forward transform additionally needs (2*log2(n)+1)*q < 2^64).
//   Field32: the ~20-bit image/plaintext modulus p (p < 2^30).
//
// Semantics follow FieldSpec::mul/add/sub (REF modfield.hpp:35-69): results are
// exact residues; only the *representation* of intermediates is lazy ([0, 2q) or
// [0, k*q)), and every value that leaves a kernel is canonical in [0, q).
//
// Shoup multiplication by a precomputed constant w (companion w' = floor(w*2^64/q))
// is built ONLY from mad.wide.u32 / mad.lo.u32, which issue at the full IMAD rate
// on sm_100a (61 op/clk/SM measured), while mad.hi.u32 issues at ~25 op/clk/SM and
// the compiler's generic __umul64hi path costs ~20 IMAD slots per modmul.
// Count per Shoup product: 6 IMAD.WIDE + 4 IMAD + 6 IADD3 exact, or 5 IMAD.WIDE +
// 4 IMAD + 2 IADD3 with the approximate quotient (survey c_q = 10).
#pragma once
#include <cstdint>

namespace ensei_gpu {

#define EG_DEV __device__ __forceinline__

EG_DEV uint32_t lo32(uint64_t x) { return (uint32_t)x; }
EG_DEV uint32_t hi32(uint64_t x) { return (uint32_t)(x >> 32); }
EG_DEV uint64_t mulw(uint32_t a, uint32_t b) { return (uint64_t)a * b; }                // IMAD.WIDE.U32
EG_DEV uint64_t madw(uint32_t a, uint32_t b, uint64_t c) { return (uint64_t)a * b + c; }  // IMAD.WIDE.U32 (acc)

// floor(x * wp / 2^64), exact, four full-rate wide multiplies.
EG_DEV uint64_t mulhi64(uint64_t x, uint64_t wp) {
  uint32_t x0 = lo32(x), x1 = hi32(x), w0 = lo32(wp), w1 = hi32(wp);
  uint64_t t = mulw(x0, w0);
  uint64_t m = madw(x0, w1, hi32(t));       // <= (2^32-1)^2 + 2^32-1 < 2^64
  uint64_t m2 = madw(x1, w0, lo32(m));      // same bound
  uint64_t h = madw(x1, w1, hi32(m));
  return h + hi32(m2);
}

// lo64(x*w + y*z) with y < 2^32 known small is not assumed: full 64x64 low products.
EG_DEV uint64_t mullo64(uint64_t x, uint64_t w) {
  uint32_t x0 = lo32(x), x1 = hi32(x), w0 = lo32(w), w1 = hi32(w);
  uint64_t t = mulw(x0, w0);
  uint32_t h = hi32(t) + x0 * w1 + x1 * w0;
  return ((uint64_t)h << 32) | lo32(t);
}

struct Field64 {
  uint64_t q;   // modulus
  uint64_t q2;  // 2q
  uint64_t nq;  // 2^64 - q  (so x*w - Q*q == x*w + Q*nq mod 2^64)
  uint64_t q4;  // 4q

  EG_DEV uint64_t reduce_once(uint64_t x) const { return x >= q ? x - q : x; }
  EG_DEV uint64_t reduce2(uint64_t x) const { return x >= q2 ? x - q2 : x; }
  EG_DEV uint64_t add(uint64_t a, uint64_t b) const { return reduce_once(a + b); }
  EG_DEV uint64_t sub(uint64_t a, uint64_t b) const { return a >= b ? a - b : a + q - b; }
  EG_DEV uint64_t neg(uint64_t a) const { return a == 0 ? 0 : q - a; }

  // x*w mod q in [0, 2q) for ANY x < 2^64 (Shoup; wp = floor(w*2^64/q), w < q).
  // Q = hi64(x*wp) from four mul.wide + a carry chain, r = lo64(x*w + Q*(2^64-q)).
  // SASS: 6 IMAD.WIDE.U32 + 4 IMAD + ~6 IADD3 (no IMAD.HI, no zeroing moves).
  EG_DEV uint64_t mul_shoup_lazy(uint64_t x, uint64_t w, uint64_t wp) const {
    uint64_t r;
    asm("{\n\t"
        ".reg .u32 x0, x1, w0, w1, p0, p1, n0, n1, a, b, c, d, e, f, g, z;\n\t"
        ".reg .u64 t;\n\t"
        "mov.b64 {x0, x1}, %1;\n\t"
        "mov.b64 {w0, w1}, %2;\n\t"
        "mov.b64 {p0, p1}, %3;\n\t"
        "mov.b64 {n0, n1}, %4;\n\t"
        "mul.wide.u32 t, x0, p0;\n\t"
        "mov.b64 {z, a}, t;\n\t"
        "mul.wide.u32 t, x0, p1;\n\t"
        "mov.b64 {b, c}, t;\n\t"
        "mul.wide.u32 t, x1, p0;\n\t"
        "mov.b64 {d, e}, t;\n\t"
        "mul.wide.u32 t, x1, p1;\n\t"
        "mov.b64 {f, g}, t;\n\t"
        "add.cc.u32 a, a, b;\n\t"
        "addc.cc.u32 f, f, c;\n\t"
        "addc.u32 g, g, 0;\n\t"
        "add.cc.u32 a, a, d;\n\t"
        "addc.cc.u32 f, f, e;\n\t"
        "addc.u32 g, g, 0;\n\t"
        "mul.wide.u32 t, x0, w0;\n\t"
        "mov.b64 {a, b}, t;\n\t"
        "mad.lo.u32 b, x0, w1, b;\n\t"
        "mad.lo.u32 b, x1, w0, b;\n\t"
        "mov.b64 t, {a, b};\n\t"
        "mad.wide.u32 t, f, n0, t;\n\t"
        "mov.b64 {a, b}, t;\n\t"
        "mad.lo.u32 b, f, n1, b;\n\t"
        "mad.lo.u32 b, g, n0, b;\n\t"
        "mov.b64 %0, {a, b};\n\t"
        "}"
        : "=l"(r)
        : "l"(x), "l"(w), "l"(wp), "l"(nq));
    return r;
  }
  // Approximate-quotient Shoup: Q' = hi(x1 w1') + hi32(x0 w1') + hi32(x1 w0') drops the
  // low partial product and the middle carries, so Q - Q' in {0,1,2} and the result
  // x*w - Q'*q lies in [0, 4q) (any x < 2^64).  9 IMAD (5 IMAD.WIDE) + 2 IADD3.
  EG_DEV uint64_t mul_shoup_approx(uint64_t x, uint64_t w, uint64_t wp) const {
    uint64_t r;
    asm("{\n\t"
        ".reg .u32 x0, x1, w0, w1, p0, p1, n0, n1, a, b, c, e, f, g;\n\t"
        ".reg .u64 t;\n\t"
        "mov.b64 {x0, x1}, %1;\n\t"
        "mov.b64 {w0, w1}, %2;\n\t"
        "mov.b64 {p0, p1}, %3;\n\t"
        "mov.b64 {n0, n1}, %4;\n\t"
        "mul.wide.u32 t, x0, p1;\n\t"
        "mov.b64 {b, c}, t;\n\t"
        "mul.wide.u32 t, x1, p0;\n\t"
        "mov.b64 {b, e}, t;\n\t"
        "mul.wide.u32 t, x1, p1;\n\t"
        "mov.b64 {f, g}, t;\n\t"
        "add.cc.u32 f, f, c;\n\t"
        "addc.u32 g, g, 0;\n\t"
        "add.cc.u32 f, f, e;\n\t"
        "addc.u32 g, g, 0;\n\t"
        "mul.wide.u32 t, x0, w0;\n\t"
        "mov.b64 {a, b}, t;\n\t"
        "mad.lo.u32 b, x0, w1, b;\n\t"
        "mad.lo.u32 b, x1, w0, b;\n\t"
        "mov.b64 t, {a, b};\n\t"
        "mad.wide.u32 t, f, n0, t;\n\t"
        "mov.b64 {a, b}, t;\n\t"
        "mad.lo.u32 b, f, n1, b;\n\t"
        "mad.lo.u32 b, g, n0, b;\n\t"
        "mov.b64 %0, {a, b};\n\t"
        "}"
        : "=l"(r)
        : "l"(x), "l"(w), "l"(wp), "l"(nq));
    return r;
  }
  EG_DEV uint64_t mul_shoup(uint64_t x, uint64_t w, uint64_t wp) const {
    return reduce_once(mul_shoup_lazy(x, w, wp));
  }
  // a*b mod q for two variables (128-bit product, Barrett with mu = floor(2^128/q)).
  // Used off the butterfly path (pointwise products with non-constant operands).
  EG_DEV uint64_t mul(uint64_t a, uint64_t b, uint64_t mu_hi, uint64_t mu_lo) const;
};

// 128-bit product a*b as (hi, lo) from four wide multiplies.
EG_DEV void mul128(uint64_t a, uint64_t b, uint64_t& hi, uint64_t& lo) {
  uint32_t a0 = lo32(a), a1 = hi32(a), b0 = lo32(b), b1 = hi32(b);
  uint64_t t = mulw(a0, b0);
  uint64_t m = madw(a0, b1, hi32(t));
  uint64_t m2 = madw(a1, b0, lo32(m));
  hi = madw(a1, b1, hi32(m)) + hi32(m2);
  lo = ((uint64_t)lo32(m2) << 32) | lo32(t);
}

// Reduces z = hi*2^64 + lo (< q * 2^64) mod q with mu = floor(2^128 / q) (hi:lo words),
// the same constant FieldSpec keeps (REF modfield.cpp:129-131); result canonical.
EG_DEV uint64_t barrett128(uint64_t zh, uint64_t zl, uint64_t q, uint64_t nq, uint64_t mu_hi,
                           uint64_t mu_lo) {
  // qhat = floor(z * mu / 2^128) approximated from the three significant partial
  // products; underestimates by at most 3 -> a few conditional subtractions.
  uint64_t a = mulhi64(zl, mu_hi);
  uint64_t b = mulhi64(zh, mu_lo);
  uint64_t c = mullo64(zh, mu_hi);
  uint64_t qhat = a + b + c;
  uint64_t r = zl + mullo64(qhat, nq);  // zl - qhat*q mod 2^64
  while (r >= q) r -= q;
  return r;
}

EG_DEV uint64_t Field64::mul(uint64_t a, uint64_t b, uint64_t mu_hi, uint64_t mu_lo) const {
  uint64_t h, l;
  mul128(a, b, h, l);
  return barrett128(h, l, q, nq, mu_hi, mu_lo);
}

struct Field32 {
  uint32_t q;
  uint32_t q2;
  EG_DEV uint32_t reduce_once(uint32_t x) const { return x >= q ? x - q : x; }
  EG_DEV uint32_t reduce2(uint32_t x) const { return x >= q2 ? x - q2 : x; }
  EG_DEV uint32_t add(uint32_t a, uint32_t b) const { return reduce_once(a + b); }
  EG_DEV uint32_t sub(uint32_t a, uint32_t b) const { return a >= b ? a - b : a + q - b; }
  // x*w mod p in [0, 2p), any x < 2^32; wp = floor(w*2^32/p). hi via IMAD.WIDE (full rate).
  EG_DEV uint32_t mul_shoup_lazy(uint32_t x, uint32_t w, uint32_t wp) const {
    // asm: the compiler folds hi32(x * wp) into mul.hi (IMAD.HI, ~0.4x the IMAD.WIDE rate)
    uint32_t Q;
    asm("{\n\t.reg .u64 t;\n\t.reg .u32 l;\n\tmul.wide.u32 t, %1, %2;\n\tmov.b64 {l, %0}, t;\n\t}" : "=r"(Q) : "r"(x), "r"(wp));
    return x * w - Q * q;
  }
  EG_DEV uint32_t mul_shoup(uint32_t x, uint32_t w, uint32_t wp) const {
    return reduce_once(mul_shoup_lazy(x, w, wp));
  }
  // general product, p < 2^30: 64-bit product reduced with m = floor(2^64/p)
  EG_DEV uint32_t mul(uint32_t a, uint32_t b, uint64_t m64) const {
    uint64_t z = mulw(a, b);
    uint64_t qt = mulhi64(z, m64);
    uint32_t r = (uint32_t)(z - qt * q);
    return reduce_once(r);
  }
};

}  // namespace ensei_gpu
