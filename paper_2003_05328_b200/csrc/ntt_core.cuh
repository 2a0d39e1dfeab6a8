// ntt_core.cuh -- CTA-cooperative number-theoretic transforms held in shared memory.
//
// One transform of length N = 2^LOGN is owned by NT = N / E threads; every thread
// keeps E elements in registers and runs up to log2(E) butterfly stages per "pass"
// (radix-2^k in registers), exchanging through swizzled shared memory between passes.
//
// Forward = merged-psi Cooley-Tukey (natural-order input -> bit-reversed output):
//   stage s (2^s groups, half-span N>>(s+1)) multiplies the upper half of group g by
//   tw[2^s + g] = psi^bitrev(2^s + g) (negacyclic) or omega^((N/2^(s+1)) * bitrev_s(g))
//   (cyclic).  Equivalent to REF NegacyclicPlan::forward (ringbfv.cpp:49-53: psi^j
//   twist + natural-order radix-2 DIT of ntt_kernel.hpp:11-33) up to the output
//   permutation; the device evaluation layout is bit-reversed (like SEAL's), and
//   boundary entry points permute to the reference's natural slot order.
// Inverse = merged-psi Gentleman-Sande (bit-reversed input -> natural output) with
//   the n^-1 scale folded into the last stage (twi[0] = n^-1, twi[1] pre-scaled);
//   equals REF NegacyclicPlan::inverse (ringbfv.cpp:55-59).
//
// Lazy reduction (Bfly<F, MODE>): values stay in [0, 8q) through the forward and in
// [0, 4q) through the inverse with the approximate-quotient Shoup product (MODE 0,
// q < 2^61), or [0, 4q) / [0, 2q) with exact Shoup (MODE 1, q < 2^62).  Every value
// that leaves the engine through fin_*() is canonical.
#pragma once
#include <type_traits>

#include "modarith.cuh"

namespace ensei_gpu {

template <class T>
struct alignas(2 * sizeof(T)) TwPair {
  T w, wp;
};

// ------------------------------------------------------------ smem layouts
// u64: XOR swizzle of 16-byte pairs inside every 128-byte row (no padding; keeps
//      (2m, 2m+1) adjacent and 16B aligned so cp.async 16B / LDS.128 work).
// u32: one spare word every 32.
// Both are bank-conflict free for every pass pattern used here except one pass of
// the u32 transforms.
template <class T>
EG_DEV int sidx(int i);
template <>
EG_DEV int sidx<uint64_t>(int i) { return i ^ (((i >> 4) & 7) << 1); }
template <>
EG_DEV int sidx<uint32_t>(int i) { return i + (i >> 5); }
template <class T>
__host__ __device__ constexpr int ssize(int n) {
  return sizeof(T) == 8 ? n : n + (n >> 5);
}

EG_DEV int brev(int x, int bits) { return bits ? (int)(__brev((unsigned)x) >> (32 - bits)) : 0; }

// ---------------------------------------------------------------- butterflies

template <class F, int MODE>
struct Bfly;

// MODE 0: approximate Shoup ([0,4q)), q < 2^59.9.  Forward butterflies do not
// correct: values grow by < 4q per stage and the pass driver inserts corr() (to
// [0,3q)) at the pass boundary where the compile-time bound would exceed 31q.
// GS keeps values < 4q + 2^32 with a hi-word compare and a predicated subtract.
template <>
struct Bfly<Field64, 0> {
  static constexpr int kGrowth = 4;   // forward bound growth per stage (units of q)
  static constexpr int kMaxBound = 31;
  static EG_DEV void ct(const Field64& f, uint64_t& u, uint64_t& v, const TwPair<uint64_t>& t) {
    uint64_t m = f.mul_shoup_approx(v, t.w, t.wp);
    v = u - m + f.q4;
    u = u + m;
  }
  static EG_DEV void gs(const Field64& f, uint64_t& u, uint64_t& v, const TwPair<uint64_t>& t) {
    uint64_t s = u + v;
    if (hi32(s) > hi32(f.q4)) s -= f.q4;
    uint64_t d = u - v + f.q4 + f.q4;
    v = f.mul_shoup_approx(d, t.w, t.wp);
    u = s;
  }
  static EG_DEV void gs_last(const Field64& f, uint64_t& u, uint64_t& v, const TwPair<uint64_t>& t,
                             const TwPair<uint64_t>& ni) {
    uint64_t s = u + v;
    uint64_t d = u - v + f.q4 + f.q4;
    v = f.mul_shoup_approx(d, t.w, t.wp);
    u = f.mul_shoup_approx(s, ni.w, ni.wp);
  }
  // x < 2^64 -> [0, 3q): x - floor(hi32(x) * floor(2^64/q) / 2^32) * q   (3 IMAD)
  static EG_DEV uint64_t corr(const Field64& f, uint64_t x, uint32_t cred) {
    uint32_t k = hi32(mulw(hi32(x), cred));
    return x + mullo64((uint64_t)k, f.nq);
  }
  static EG_DEV uint64_t fin_ct(const Field64& f, uint64_t x, uint32_t cred) {  // -> canonical
    x = corr(f, x, cred);
    if (x >= f.q2) x -= f.q2;
    if (x >= f.q) x -= f.q;
    return x;
  }
  static EG_DEV uint64_t fin_gs(const Field64& f, uint64_t x) {  // < 4q + 2^32 -> canonical
    if (x >= f.q2) x -= f.q2;
    if (x >= f.q) x -= f.q;
    if (x >= f.q) x -= f.q;
    return x;
  }
};

// MODE 1: exact Shoup ([0,2q)), Harvey: CT values < 4q, GS values < 2q.  q < 2^62.
template <>
struct Bfly<Field64, 1> {
  static constexpr int kGrowth = 0;  // Harvey: bounded every stage
  static constexpr int kMaxBound = 1 << 30;
  static EG_DEV uint64_t corr(const Field64& f, uint64_t x, uint32_t) { return x; }
  static EG_DEV void ct(const Field64& f, uint64_t& u, uint64_t& v, const TwPair<uint64_t>& t) {
    u = f.reduce2(u);
    uint64_t m = f.mul_shoup_lazy(v, t.w, t.wp);
    v = u - m + f.q2;
    u = u + m;
  }
  static EG_DEV void gs(const Field64& f, uint64_t& u, uint64_t& v, const TwPair<uint64_t>& t) {
    uint64_t s = f.reduce2(u + v);
    uint64_t d = u - v + f.q2;
    v = f.mul_shoup_lazy(d, t.w, t.wp);
    u = s;
  }
  static EG_DEV void gs_last(const Field64& f, uint64_t& u, uint64_t& v, const TwPair<uint64_t>& t,
                             const TwPair<uint64_t>& ni) {
    uint64_t s = u + v;
    uint64_t d = u - v + f.q2;
    v = f.mul_shoup_lazy(d, t.w, t.wp);
    u = f.mul_shoup_lazy(s, ni.w, ni.wp);
  }
  static EG_DEV uint64_t fin_ct(const Field64& f, uint64_t x, uint32_t) {
    x = f.reduce2(x);
    return f.reduce_once(x);
  }
  static EG_DEV uint64_t fin_gs(const Field64& f, uint64_t x) { return f.reduce_once(x); }
};

// Field32 (p < 2^26 for the lazy forward): CT values grow by 2p per stage without
// correction (< 27p after 13 stages); GS values < 2p (Harvey).
template <int MODE>
struct Bfly<Field32, MODE> {
  static constexpr int kGrowth = 0;  // p < 2^26: (2*13+1) p < 2^32, never corrected
  static constexpr int kMaxBound = 1 << 30;
  static EG_DEV uint32_t corr(const Field32&, uint32_t x, uint32_t) { return x; }
  static EG_DEV void ct(const Field32& f, uint32_t& u, uint32_t& v, const TwPair<uint32_t>& t) {
    uint32_t m = f.mul_shoup_lazy(v, t.w, t.wp);
    v = u - m + f.q2;
    u = u + m;
  }
  static EG_DEV void gs(const Field32& f, uint32_t& u, uint32_t& v, const TwPair<uint32_t>& t) {
    uint32_t s = f.reduce2(u + v);
    uint32_t d = u - v + f.q2;
    v = f.mul_shoup_lazy(d, t.w, t.wp);
    u = s;
  }
  static EG_DEV void gs_last(const Field32& f, uint32_t& u, uint32_t& v, const TwPair<uint32_t>& t,
                             const TwPair<uint32_t>& ni) {
    uint32_t s = u + v;
    uint32_t d = u - v + f.q2;
    v = f.mul_shoup_lazy(d, t.w, t.wp);
    u = f.mul_shoup_lazy(s, ni.w, ni.wp);
  }
  static EG_DEV uint32_t fin_gs(const Field32& f, uint32_t x) { return f.reduce_once(x); }
};

// canonical reduction of a lazily reduced value x < 2^64 (c = floor(2^64/q) < 2^32)
EG_DEV uint64_t reduce_lazy(const Field64& f, uint64_t x, uint32_t c) {
  uint32_t k = hi32(mulw(hi32(x), c));
  uint64_t r = x + mullo64((uint64_t)k, f.nq);  // x - k*q, in [0, 3q)
  r = f.reduce_once(r);
  return f.reduce_once(r);
}
EG_DEV uint32_t reduce_lazy(const Field32& f, uint32_t x, uint32_t c) {
  uint32_t k = hi32(mulw(x, c));
  uint32_t r = x - k * f.q;  // [0, 2q)
  return f.reduce_once(r);
}

// ------------------------------------------------------------- register passes

// Stages S0 .. S0+P-1 of the forward transform on one element set x[0 .. 2^P).
template <int S0, int P, int MODE, class F, class T>
EG_DEV void ct_set(const F& f, const TwPair<T>* __restrict__ tw, T (&x)[1 << P], int g) {
#pragma unroll
  for (int l = 0; l < P; ++l) {
    const int half = (1 << P) >> (l + 1);
#pragma unroll
    for (int h = 0; h < (1 << l); ++h) {
      const TwPair<T> t = tw[(1 << (S0 + l)) + (g << l) + h];
#pragma unroll
      for (int i = 0; i < half; ++i) Bfly<F, MODE>::ct(f, x[2 * h * half + i], x[2 * h * half + i + half], t);
    }
  }
}

// Stages S0+P-1 down to S0 of the inverse transform on one element set.
template <int S0, int P, int MODE, class F, class T>
EG_DEV void gs_set(const F& f, const TwPair<T>* __restrict__ tw, T (&x)[1 << P], int g) {
#pragma unroll
  for (int l = P - 1; l >= 0; --l) {
    const int half = (1 << P) >> (l + 1);
#pragma unroll
    for (int h = 0; h < (1 << l); ++h) {
      const TwPair<T> t = tw[(1 << (S0 + l)) + (g << l) + h];
      if (S0 + l == 0) {
        const TwPair<T> ni = tw[0];
#pragma unroll
        for (int i = 0; i < half; ++i)
          Bfly<F, MODE>::gs_last(f, x[2 * h * half + i], x[2 * h * half + i + half], t, ni);
      } else {
#pragma unroll
        for (int i = 0; i < half; ++i) Bfly<F, MODE>::gs(f, x[2 * h * half + i], x[2 * h * half + i + half], t);
      }
    }
  }
}

// Pass plan: forward passes are [rem, LOGE, LOGE, ...] (remainder first), the
// inverse runs the same passes in reverse order.
template <int LOGN, int LOGE>
struct PassPlan {
  static constexpr int rem = LOGN % LOGE;
  static constexpr int npass = LOGN / LOGE + (rem ? 1 : 0);
  __host__ __device__ static constexpr int p_of(int i) { return (rem && i == 0) ? rem : LOGE; }
  __host__ __device__ static constexpr int s0_of(int i) { return i == 0 ? 0 : (rem ? rem + (i - 1) * LOGE : i * LOGE); }
};

// Element index of member k of set j for a pass (S0, P) of an N-point transform.
template <int LOGN, int S0, int P>
EG_DEV int set_index(int j, int k) {
  constexpr int R = 1 << (LOGN - S0 - P);
  return (j / R) * (1 << (LOGN - S0)) + (j % R) + k * R;
}

// Accessor concept: operator()(i) -> T, operator()(i, T); optionally
//   static constexpr bool kVec = true;  ld2(i, a, b) / st2(i, a, b) for an aligned pair.
template <class A, class = void>
struct HasVec : std::false_type {};
template <class A>
struct HasVec<A, std::void_t<decltype(A::kVec)>> : std::integral_constant<bool, A::kVec> {};

// Runs pass I of the plan for every set owned by thread `tid` of the NT threads of
// one transform: loads all sets (Src), runs the butterflies, optionally syncs
// (SPLIT: needed when Dst permutes in place), then stores (Dst).  Contiguous sets
// (R == 1) use paired (16-byte) accesses when the accessor offers them.
template <class F, class T, int LOGN, int LOGE, int I, bool INV, int MODE, bool SPLIT, class Src,
          class Dst, class Bar, bool CORR = false>
EG_DEV void run_pass(const F& f, const TwPair<T>* __restrict__ tw, int tid, Src& src, Dst& dst,
                     const Bar& bar, uint32_t cred = 0) {
  using Plan = PassPlan<LOGN, LOGE>;
  constexpr int P = Plan::p_of(I), S0 = Plan::s0_of(I);
  constexpr int NT = (1 << LOGN) >> LOGE;
  constexpr int SETS = (1 << LOGE) >> P;  // sets per thread this pass
  constexpr int R = 1 << (LOGN - S0 - P);
  T x[SETS][1 << P];
#pragma unroll
  for (int u = 0; u < SETS; ++u) {
    const int j = tid + u * NT;
    if constexpr (R == 1 && P >= 1 && HasVec<Src>::value) {
#pragma unroll
      for (int k = 0; k < (1 << P); k += 2) src.ld2(j * (1 << P) + k, x[u][k], x[u][k + 1]);
    } else {
#pragma unroll
      for (int k = 0; k < (1 << P); ++k) x[u][k] = src(set_index<LOGN, S0, P>(j, k));
    }
    if constexpr (CORR) {
#pragma unroll
      for (int k = 0; k < (1 << P); ++k) x[u][k] = Bfly<F, MODE>::corr(f, x[u][k], cred);
    }
    if constexpr (INV) gs_set<S0, P, MODE>(f, tw, x[u], j / R);
    else ct_set<S0, P, MODE>(f, tw, x[u], j / R);
  }
  if constexpr (SPLIT) bar.sync();
#pragma unroll
  for (int u = 0; u < SETS; ++u) {
    const int j = tid + u * NT;
    if constexpr (R == 1 && P >= 1 && HasVec<Dst>::value) {
#pragma unroll
      for (int k = 0; k < (1 << P); k += 2) dst.st2(j * (1 << P) + k, x[u][k], x[u][k + 1]);
    } else {
#pragma unroll
      for (int k = 0; k < (1 << P); ++k) dst(set_index<LOGN, S0, P>(j, k), x[u][k]);
    }
  }
}

// Shared-memory accessors (swizzled / padded layout).
template <class T>
struct SmemRW {
  T* s;
  EG_DEV T operator()(int i) const { return s[sidx<T>(i)]; }
  EG_DEV void operator()(int i, T v) const { s[sidx<T>(i)] = v; }
};
template <>
struct SmemRW<uint64_t> {
  uint64_t* s;
  static constexpr bool kVec = true;
  EG_DEV uint64_t operator()(int i) const { return s[sidx<uint64_t>(i)]; }
  EG_DEV void operator()(int i, uint64_t v) const { s[sidx<uint64_t>(i)] = v; }
  EG_DEV void ld2(int i, uint64_t& a, uint64_t& b) const {
    ulonglong2 v = *reinterpret_cast<const ulonglong2*>(s + sidx<uint64_t>(i));
    a = v.x;
    b = v.y;
  }
  EG_DEV void st2(int i, uint64_t a, uint64_t b) const {
    *reinterpret_cast<ulonglong2*>(s + sidx<uint64_t>(i)) = make_ulonglong2(a, b);
  }
};

// Barrier over the NT threads owning one transform (named barrier `id`).
struct NamedBar {
  int id, count;
  EG_DEV void sync() const { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory"); }
};
struct CtaBar {
  EG_DEV void sync() const { __syncthreads(); }
};

// Compile-time bound tracking for the forward transform (units of q): does pass I
// need its inputs corrected, given the input bound B_IN?
template <class F, int MODE, int LOGN, int LOGE, int B_IN>
struct FwdBounds {
  using Plan = PassPlan<LOGN, LOGE>;
  static constexpr int G = Bfly<F, MODE>::kGrowth, M = Bfly<F, MODE>::kMaxBound;
  static constexpr bool corr(int i) {
    int b = B_IN;
    for (int k = 0; k <= i; ++k) {
      bool c = b + G * Plan::p_of(k) > M;
      if (c) b = 3;
      if (k == i) return c;
      b += G * Plan::p_of(k);
    }
    return false;
  }
};

// Barrier between pass I and pass I + 1 of a transform.  The last two passes (2 LOGE stages)
// work inside blocks of 2^(2 LOGE) consecutive elements, and with LOGE = 3 a block's sets
// belong to the same 8 consecutive threads in both passes (set j of the last pass =
// elements [8j, 8j + 8); of the one before = block j / 8): a warp barrier is enough there.
template <int LOGN, int LOGE, int I, class Bar>
EG_DEV void pass_sync(const Bar& bar) {
  using Plan = PassPlan<LOGN, LOGE>;
  if constexpr (LOGE == 3 && I == Plan::npass - 2 && Plan::npass >= 3 && Plan::p_of(I) == 3 && LOGN - 3 >= 5)
    __syncwarp();
  else
    bar.sync();
}

template <class F, class T, int LOGN, int LOGE, int MODE, int B_IN, int I, class Bar>
EG_DEV void fwd_middle(const F& f, const TwPair<T>* __restrict__ tw, int tid, SmemRW<T>& s, const Bar& bar,
                       uint32_t cred) {
  if constexpr (I < PassPlan<LOGN, LOGE>::npass - 1) {
    constexpr bool C = FwdBounds<F, MODE, LOGN, LOGE, B_IN>::corr(I);
    run_pass<F, T, LOGN, LOGE, I, false, MODE, false, SmemRW<T>, SmemRW<T>, Bar, C>(f, tw, tid, s, s, bar, cred);
    pass_sync<LOGN, LOGE, I>(bar);
    fwd_middle<F, T, LOGN, LOGE, MODE, B_IN, I + 1>(f, tw, tid, s, bar, cred);
  }
}

template <class F, class T, int LOGN, int LOGE, int MODE, int I, class Bar>
EG_DEV void inv_middle(const F& f, const TwPair<T>* __restrict__ tw, int tid, SmemRW<T>& s, const Bar& bar) {
  if constexpr (I >= 1) {
    run_pass<F, T, LOGN, LOGE, I, true, MODE, false>(f, tw, tid, s, s, bar);
    bar.sync();
    inv_middle<F, T, LOGN, LOGE, MODE, I - 1>(f, tw, tid, s, bar);
  }
}

// Full forward transform.  src feeds pass 0; dst receives the last pass (LAZY values,
// computational = bit-reversed order; apply Bfly::fin_ct or reduce_lazy).
// Intermediate passes live in `sm` (swizzled).  SPLIT_FIRST / SPLIT_LAST insert a
// barrier between the loads and the stores of the first / last pass (required when
// src / dst alias `sm` through a permutation).  No barrier before the first pass or
// after the last.  B_IN bounds the inputs (units of q; 1 = canonical).
template <class F, class T, int LOGN, int LOGE, int MODE, bool SPLIT_FIRST, bool SPLIT_LAST, class Src,
          class Dst, class Bar, int B_IN = 1>
EG_DEV void ntt_forward(const F& f, const TwPair<T>* __restrict__ tw, T* sm, int tid, Src src, Dst dst,
                        const Bar& bar, uint32_t cred = 0) {
  using Plan = PassPlan<LOGN, LOGE>;
  using FB = FwdBounds<F, MODE, LOGN, LOGE, B_IN>;
  SmemRW<T> s{sm};
  if constexpr (Plan::npass == 1) {
    run_pass<F, T, LOGN, LOGE, 0, false, MODE, SPLIT_FIRST || SPLIT_LAST, Src, Dst, Bar, FB::corr(0)>(
        f, tw, tid, src, dst, bar, cred);
  } else {
    run_pass<F, T, LOGN, LOGE, 0, false, MODE, SPLIT_FIRST, Src, SmemRW<T>, Bar, FB::corr(0)>(f, tw, tid, src, s,
                                                                                          bar, cred);
    pass_sync<LOGN, LOGE, 0>(bar);
    fwd_middle<F, T, LOGN, LOGE, MODE, B_IN, 1>(f, tw, tid, s, bar, cred);
    run_pass<F, T, LOGN, LOGE, Plan::npass - 1, false, MODE, SPLIT_LAST, SmemRW<T>, Dst, Bar,
             FB::corr(Plan::npass - 1)>(f, tw, tid, s, dst, bar, cred);
  }
}

// Full inverse transform: src is read in computational (bit-reversed) order by the
// first pass, dst receives natural-order LAZY values (apply Bfly::fin_gs).
template <class F, class T, int LOGN, int LOGE, int MODE, bool SPLIT_FIRST, bool SPLIT_LAST, class Src,
          class Dst, class Bar>
EG_DEV void ntt_inverse(const F& f, const TwPair<T>* __restrict__ tw, T* sm, int tid, Src src, Dst dst,
                        const Bar& bar) {
  using Plan = PassPlan<LOGN, LOGE>;
  SmemRW<T> s{sm};
  constexpr int L = Plan::npass - 1;
  if constexpr (Plan::npass == 1) {
    run_pass<F, T, LOGN, LOGE, 0, true, MODE, SPLIT_FIRST || SPLIT_LAST>(f, tw, tid, src, dst, bar);
  } else {
    run_pass<F, T, LOGN, LOGE, L, true, MODE, SPLIT_FIRST>(f, tw, tid, src, s, bar);
    pass_sync<LOGN, LOGE, L - 1>(bar);  // passes L and L - 1: the same two block-local passes
    inv_middle<F, T, LOGN, LOGE, MODE, L - 1>(f, tw, tid, s, bar);
    run_pass<F, T, LOGN, LOGE, 0, true, MODE, SPLIT_LAST>(f, tw, tid, s, dst, bar);
  }
}

// ------------------------------------------------------------ async copies

EG_DEV uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// cp.async 16-byte global -> shared (LDGSTS), L2-only (.cg)
EG_DEV void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
EG_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
EG_DEV void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// TMA bulk copy (cp.async.bulk, SASS UBLKCP) global -> shared completing on an mbarrier.
EG_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
EG_DEV void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
EG_DEV void tma_bulk_g2s(void* smem, const void* gmem, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(smem)),
               "l"(gmem), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
EG_DEV void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// Stage `bytes` (multiple of 16) of a read-only table into shared memory with TMA
// bulk copies (<= 32 KiB per copy).  Called by all threads; ends with the data
// visible to the whole CTA.  `bar` is a shared mbarrier (consumed: phase 0).
EG_DEV void stage_table(void* smem, const void* gmem, uint32_t bytes, uint64_t* bar) {
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    mbar_init(bar, 1);
    mbar_expect_tx(bar, bytes);
    for (uint32_t off = 0; off < bytes; off += 32768u) {
      uint32_t c = bytes - off < 32768u ? bytes - off : 32768u;
      tma_bulk_g2s(static_cast<uint8_t*>(smem) + off, static_cast<const uint8_t*>(gmem) + off, c, bar);
    }
  }
  __syncthreads();
  mbar_wait(bar, 0);
}

}  // namespace ensei_gpu
