// ensei_b200.hpp -- header-only C++ host mirror of the REF operator surface over the
// C ABI (include/ensei_gpu.h).  Same names / argument meaning / exception types as
// REF (namespace ensei -> ensei_b200), batched where REF works one block at a time:
//   REF ringbfv.hpp:82-121  keygen, encrypt_freq_direct, decrypt, add_ct, add_plain,
//                           prepare_plain, mul_plain (+ its static NoiseExhausted check)
//   REF hss.hpp:34-49       hom_share, hom_share_with, hom_rec, recombine_clear
//   REF counters.hpp:17-31  TransformCounters with REF's logical counts
//   REF protocol.hpp:80-109 PhaseTimings / PartyResult of a batched conv-layer run
// Value types mirror REF's (natural slot order, uint64 residues); the arithmetic runs in
// libensei_gpu.so kernels (device buffers are made per call: this is the convenience
// surface -- the batched C ABI entry points are the allocation-free hot path).
// Link: -lensei_gpu (paper_2003_05328_b200/libensei_gpu.so) -lcudart.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../../include/ensei_gpu.h"

namespace ensei_b200 {

// REF errors.hpp:7-37, thrown from the C status codes
struct Error : std::runtime_error { using std::runtime_error::runtime_error; };
struct OrderNotDividing : Error { using Error::Error; };
struct SearchExhausted : Error { using Error::Error; };
struct BadRoot : Error { using Error::Error; };
struct BadGeometry : Error { using Error::Error; };
struct GeometryMismatch : Error { using Error::Error; };
struct DomainMismatch : Error { using Error::Error; };
struct NoiseExhausted : Error { using Error::Error; };
struct ChainViolation : Error { using Error::Error; };
struct LengthMismatch : Error { using Error::Error; };
struct RangeViolation : Error { using Error::Error; };
struct ProtocolOrderViolation : Error { using Error::Error; };
struct RangeOverflow : Error { using Error::Error; };
struct MalformedPayload : Error { using Error::Error; };
struct TransportError : Error { using Error::Error; };
struct DeviceError : Error { using Error::Error; };

inline void check(int rc) {
  if (rc == ENSEI_OK) return;
  std::string m = ensei_gpu_last_error();
  switch (rc) {
    case ENSEI_ERR_ORDER_NOT_DIVIDING: throw OrderNotDividing(m);
    case ENSEI_ERR_SEARCH_EXHAUSTED: throw SearchExhausted(m);
    case ENSEI_ERR_BAD_ROOT: throw BadRoot(m);
    case ENSEI_ERR_BAD_GEOMETRY: throw BadGeometry(m);
    case ENSEI_ERR_GEOMETRY_MISMATCH: throw GeometryMismatch(m);
    case ENSEI_ERR_DOMAIN_MISMATCH: throw DomainMismatch(m);
    case ENSEI_ERR_NOISE_EXHAUSTED: throw NoiseExhausted(m);
    case ENSEI_ERR_CHAIN_VIOLATION: throw ChainViolation(m);
    case ENSEI_ERR_LENGTH_MISMATCH: throw LengthMismatch(m);
    case ENSEI_ERR_RANGE_VIOLATION: throw RangeViolation(m);
    case ENSEI_ERR_PROTOCOL_ORDER: throw ProtocolOrderViolation(m);
    case ENSEI_ERR_RANGE_OVERFLOW: throw RangeOverflow(m);
    case ENSEI_ERR_MALFORMED_PAYLOAD: throw MalformedPayload(m);
    case ENSEI_ERR_TRANSPORT: throw TransportError(m);
    // no REF counterpart (device faults, shapes this path does not take, bad arguments)
    case ENSEI_ERR_CUDA: case ENSEI_ERR_UNSUPPORTED: case ENSEI_ERR_INVALID_ARGUMENT: throw DeviceError(m);
    default: throw Error(m);
  }
}

template <class T>
struct DeviceBuffer {
  T* p = nullptr;
  size_t n = 0;
  explicit DeviceBuffer(size_t count) : n(count) {
    if (count && cudaMalloc(&p, count * sizeof(T)) != cudaSuccess) throw DeviceError("cudaMalloc failed");
  }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  ~DeviceBuffer() { if (p) cudaFree(p); }
  void upload(const T* h, size_t count) { cudaMemcpy(p, h, count * sizeof(T), cudaMemcpyHostToDevice); }
  void download(T* h, size_t count) const { cudaMemcpy(h, p, count * sizeof(T), cudaMemcpyDeviceToHost); }
};

// RlweParams + ModulusChain::unified on one device (REF ringbfv.cpp:65-87)
class Context {
 public:
  Context(uint32_t n, std::vector<uint64_t> q, uint64_t p, int device = 0) : n_(n) {
    check(ensei_gpu_ctx_create(device, n, q.data(), (uint32_t)q.size(), p, &h_));
  }
  ~Context() { ensei_gpu_ctx_destroy(h_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  ensei_gpu_ctx* get() const { return h_; }
  uint32_t n() const { return n_; }

  // NegacyclicPlan::forward / inverse (REF ringbfv.cpp:49-59) on `polys` = k*n
  // residues mod q_i (natural order both sides, REF layout).
  void negacyclic_forward(std::vector<uint64_t>& polys, uint32_t prime = 0) const { transform(polys, prime, 0); }
  void negacyclic_inverse(std::vector<uint64_t>& polys, uint32_t prime = 0) const { transform(polys, prime, 1); }
  // encode_slots / decode_slots (REF ringbfv.cpp:109-125)
  void encode_slots(std::vector<uint64_t>& v) const { transform(v, ENSEI_MOD_P, 1); }
  void decode_slots(std::vector<uint64_t>& v) const { transform(v, ENSEI_MOD_P, 0); }
  // ntt_2d / intt_2d (REF ntt.cpp:139-153) on k rows x cols tiles
  void ntt_2d(std::vector<uint64_t>& tiles, uint32_t rows, uint32_t cols, bool inverse = false) const {
    DeviceBuffer<uint64_t> d(tiles.size());
    d.upload(tiles.data(), tiles.size());
    check(ensei_gpu_ntt2d(h_, inverse ? 1 : 0, rows, cols, d.p, tiles.size() / ((size_t)rows * cols), nullptr));
    d.download(tiles.data(), tiles.size());
  }

 private:
  void transform(std::vector<uint64_t>& v, uint32_t modulus, int inverse) const {
    if (v.size() % n_) throw LengthMismatch("vector length must be a multiple of n");
    DeviceBuffer<uint64_t> d(v.size());
    d.upload(v.data(), v.size());
    check(ensei_gpu_negacyclic(h_, modulus, inverse, ENSEI_LAYOUT_NATURAL, d.p, v.size() / n_, nullptr));
    d.download(v.data(), v.size());
  }
  ensei_gpu_ctx* h_ = nullptr;
  uint32_t n_;
};


// ===================================================================== operators
using Residue = uint64_t;

// REF counters.hpp:17-31: per-thread logical counts (one per REF transform call, even
// where the device fuses them)
struct TransformCounters {
  uint64_t ct_ntt = 0, ring_ntt = 0, image_ntt = 0, hadamard = 0;
  TransformCounters operator-(const TransformCounters& o) const {
    return {ct_ntt - o.ct_ntt, ring_ntt - o.ring_ntt, image_ntt - o.image_ntt, hadamard - o.hadamard};
  }
};
inline TransformCounters& transform_counters() {
  static thread_local TransformCounters c;
  return c;
}
inline void reset_transform_counters() { transform_counters() = TransformCounters{}; }

// REF Rng (modfield.hpp:104-130): mt19937_64, REF's samplers, REF's fork
class Rng {
 public:
  explicit Rng(uint64_t seed) { check(ensei_gpu_ref_rng_create(seed, 0, 0, &h_)); seed_ = seed; }
  Rng(Rng&& o) noexcept : h_(o.h_), seed_(o.seed_) { o.h_ = nullptr; }
  Rng(const Rng&) = delete;
  ~Rng() { if (h_) ensei_gpu_ref_rng_destroy(h_); }
  uint64_t next_u64() { uint64_t v; check(ensei_gpu_ref_rng_next_u64(h_, &v, 1)); return v; }
  uint64_t uniform_below(uint64_t bound) { uint64_t v; check(ensei_gpu_ref_rng_uniform_below(h_, bound, &v, 1)); return v; }
  Residue uniform_residue(uint64_t modulus) { return uniform_below(modulus); }
  int64_t sample_gaussian(double sigma) { int64_t v; check(ensei_gpu_ref_rng_gaussian(h_, sigma, &v, 1)); return v; }
  void uniform_below(uint64_t bound, uint64_t* out, size_t k) { check(ensei_gpu_ref_rng_uniform_below(h_, bound, out, k)); }
  void sample_gaussian(double sigma, int64_t* out, size_t k) { check(ensei_gpu_ref_rng_gaussian(h_, sigma, out, k)); }
  Rng fork(uint64_t salt) const { return Rng(seed_, salt); }

 private:
  Rng(uint64_t seed, uint64_t salt) { check(ensei_gpu_ref_rng_create(seed, 1, salt, &h_)); seed_ = h_seed(seed, salt); }
  static uint64_t mix64(uint64_t x) {  // REF modfield.cpp:79-85
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
  }
  static uint64_t h_seed(uint64_t seed, uint64_t salt) { return mix64(seed ^ mix64(salt)); }
  ensei_ref_rng* h_ = nullptr;
  uint64_t seed_ = 0;
};

enum class RingDomain : uint8_t { Coefficient = 0, Evaluation = 1 };
struct RingElem {
  std::vector<Residue> coeffs;
  RingDomain domain = RingDomain::Coefficient;
};
struct PlainVec {
  std::vector<Residue> slots;
  bool operator==(const PlainVec&) const = default;
};

// REF RlweParams (ringbfv.hpp:29-45), single prime as REF; the device context rides along
struct RlweParams {
  size_t n = 0;
  uint64_t q = 0, p_e = 0;
  double sigma = 0;
  uint64_t delta = 0;
  std::shared_ptr<Context> ctx;
  double noise_cap() const { return (double)q / (2.0 * (double)p_e); }
  double fresh_noise_bound() const { return 6.0 * sigma + 1.0; }
};
inline RlweParams make_rlwe_params(size_t n, uint64_t q, uint64_t p_e, double sigma, int device = 0) {
  RlweParams p;
  p.n = n;
  p.q = q;
  p.p_e = p_e;
  p.sigma = sigma;
  p.ctx = std::make_shared<Context>((uint32_t)n, std::vector<uint64_t>{q}, p_e, device);  // REF's invariants
  p.delta = q / p_e;
  return p;
}

struct SecretKey {
  RingElem t, t_eval;
  std::shared_ptr<DeviceBuffer<uint64_t>> blob;  // device key blob (ENSEI_KEY_WORDS)
};
struct Ciphertext {
  RingElem c0, c1;
  double noise_bound = 0.0, plain_mass = 0.0;
  RingDomain domain() const { return c0.domain; }
};
struct PreparedPlain {
  RingElem w_eval;
  double w_inf = 0;
  std::vector<uint64_t> packed;  // device prepared words (bit-reversed, packed limbs)
};
struct ModulusChain {
  uint64_t p_n = 0, p_a = 0, p_e = 0;
  static ModulusChain unified(uint64_t p) { return {p, p, p}; }
};
struct SharePair {
  Ciphertext alice_ct;
  PlainVec bob_share;
  uint64_t share_modulus = 0;
};

namespace detail {
inline ensei_gpu_ctx* h(const RlweParams& p) { return p.ctx->get(); }
struct Work {
  DeviceBuffer<uint8_t> w;
  Work(const RlweParams& p, size_t count) : w(ensei_gpu_ops_workspace_bytes(h(p), count)) {}
};
// host ciphertexts (REF natural order) <-> device [count][2][1][n] (bit-reversed)
inline void upload_cts(const RlweParams& p, const std::vector<const Ciphertext*>& cts, DeviceBuffer<uint64_t>& d) {
  const size_t n = p.n;
  std::vector<uint64_t> hv(cts.size() * 2 * n);
  for (size_t b = 0; b < cts.size(); ++b) {
    if (cts[b]->domain() != RingDomain::Evaluation) throw DomainMismatch("the device path takes evaluation-domain ciphertexts");
    if (cts[b]->c0.coeffs.size() != n || cts[b]->c1.coeffs.size() != n) throw LengthMismatch("ciphertext length must equal n");
    std::copy(cts[b]->c0.coeffs.begin(), cts[b]->c0.coeffs.end(), hv.begin() + b * 2 * n);
    std::copy(cts[b]->c1.coeffs.begin(), cts[b]->c1.coeffs.end(), hv.begin() + b * 2 * n + n);
  }
  d.upload(hv.data(), hv.size());
  check(ensei_gpu_permute(h(p), 0, d.p, 2 * cts.size(), nullptr));
}
inline void download_ct(const RlweParams& p, DeviceBuffer<uint64_t>& d, size_t b, Ciphertext& ct) {
  const size_t n = p.n;
  std::vector<uint64_t> hv(2 * n);
  cudaMemcpy(hv.data(), d.p + b * 2 * n, 2 * n * sizeof(uint64_t), cudaMemcpyDeviceToHost);
  ct.c0.coeffs.assign(hv.begin(), hv.begin() + n);
  ct.c1.coeffs.assign(hv.begin() + n, hv.end());
  ct.c0.domain = ct.c1.domain = RingDomain::Evaluation;
}
inline void upload_slots(const RlweParams& p, const std::vector<const PlainVec*>& v, DeviceBuffer<uint64_t>& d) {
  std::vector<uint64_t> hv(v.size() * p.n);
  for (size_t b = 0; b < v.size(); ++b) {
    if (v[b]->slots.size() != p.n) throw Error("slot count must equal n");  // REF encode_slots
    std::copy(v[b]->slots.begin(), v[b]->slots.end(), hv.begin() + b * p.n);
  }
  d.upload(hv.data(), hv.size());
}
}  // namespace detail

// keygen (REF ringbfv.cpp:95-107): n discrete Gaussians of the REF Rng, t_eval = NTT_q(t)
inline SecretKey keygen(const RlweParams& p, Rng& rng) {
  std::vector<int64_t> t(p.n);
  rng.sample_gaussian(p.sigma, t.data(), p.n);
  SecretKey sk;
  sk.t.domain = RingDomain::Coefficient;
  sk.t.coeffs.resize(p.n);
  for (size_t i = 0; i < p.n; ++i) sk.t.coeffs[i] = t[i] < 0 ? p.q - (uint64_t)(-t[i]) : (uint64_t)t[i];
  DeviceBuffer<int64_t> dt(p.n);
  dt.upload(t.data(), p.n);
  sk.blob = std::make_shared<DeviceBuffer<uint64_t>>(ENSEI_KEY_WORDS(p.n, 1));
  check(ensei_gpu_secret_from_coeffs(detail::h(p), dt.p, sk.blob->p, nullptr));
  sk.t_eval.coeffs.resize(p.n);
  DeviceBuffer<uint64_t> te(p.n);
  cudaMemcpy(te.p, sk.blob->p, p.n * sizeof(uint64_t), cudaMemcpyDeviceToDevice);
  check(ensei_gpu_permute(detail::h(p), 1, te.p, 1, nullptr));
  te.download(sk.t_eval.coeffs.data(), p.n);
  sk.t_eval.domain = RingDomain::Evaluation;
  transform_counters().ring_ntt += 1;
  return sk;
}

// encrypt_freq_direct (REF ringbfv.cpp:180-201), batched: per block REF's draw order
// (n Gaussians, then n uniforms mod q), noise_bound = 6 sigma + 1, plain_mass = 1
inline std::vector<Ciphertext> encrypt_freq_direct(const std::vector<PlainVec>& m, const SecretKey& sk,
                                                   const RlweParams& p, Rng& rng) {
  const size_t k = m.size(), n = p.n;
  std::vector<int64_t> e(k * n);
  std::vector<uint64_t> a(k * n);
  for (size_t b = 0; b < k; ++b) {
    rng.sample_gaussian(p.sigma, e.data() + b * n, n);
    rng.uniform_below(p.q, a.data() + b * n, n);
  }
  std::vector<const PlainVec*> mv;
  for (const auto& x : m) mv.push_back(&x);
  DeviceBuffer<uint64_t> ds(k * n), da(k * n), dct(k * 2 * n);
  DeviceBuffer<int64_t> de(k * n);
  detail::upload_slots(p, mv, ds);
  de.upload(e.data(), e.size());
  da.upload(a.data(), a.size());
  detail::Work w(p, k);
  check(ensei_gpu_encrypt_freq_direct(detail::h(p), ds.p, sk.blob->p, de.p, da.p, k, dct.p, w.w.p, nullptr));
  check(ensei_gpu_permute(detail::h(p), 1, dct.p, 2 * k, nullptr));
  std::vector<Ciphertext> out(k);
  for (size_t b = 0; b < k; ++b) {
    detail::download_ct(p, dct, b, out[b]);
    out[b].noise_bound = p.fresh_noise_bound();
    out[b].plain_mass = 1.0;
  }
  transform_counters().ring_ntt += 2 * k;
  return out;
}
inline Ciphertext encrypt_freq_direct(const PlainVec& m, const SecretKey& sk, const RlweParams& p, Rng& rng) {
  return encrypt_freq_direct(std::vector<PlainVec>{m}, sk, p, rng)[0];
}

// decrypt (REF ringbfv.cpp:203-231), batched, evaluation-domain ciphertexts
inline std::vector<PlainVec> decrypt(const std::vector<Ciphertext>& cts, const SecretKey& sk, const RlweParams& p) {
  const size_t k = cts.size();
  std::vector<const Ciphertext*> cv;
  for (const auto& c : cts) cv.push_back(&c);
  DeviceBuffer<uint64_t> dct(k * 2 * p.n), ds(k * p.n);
  detail::upload_cts(p, cv, dct);
  detail::Work w(p, k);
  check(ensei_gpu_decrypt(detail::h(p), dct.p, sk.blob->p, k, ds.p, w.w.p, nullptr));
  std::vector<uint64_t> hv(k * p.n);
  ds.download(hv.data(), hv.size());
  std::vector<PlainVec> out(k);
  for (size_t b = 0; b < k; ++b) out[b].slots.assign(hv.begin() + b * p.n, hv.begin() + (b + 1) * p.n);
  transform_counters().ring_ntt += 2 * k;
  return out;
}
inline PlainVec decrypt(const Ciphertext& ct, const SecretKey& sk, const RlweParams& p) {
  return decrypt(std::vector<Ciphertext>{ct}, sk, p)[0];
}

// prepare_plain (REF ringbfv.cpp:265-280), batched
inline std::vector<PreparedPlain> prepare_plain(const std::vector<PlainVec>& w, const RlweParams& p) {
  const size_t k = w.size(), n = p.n;
  std::vector<const PlainVec*> wv;
  for (const auto& x : w) wv.push_back(&x);
  DeviceBuffer<uint64_t> ds(k * n), dw(k * n);
  detail::upload_slots(p, wv, ds);
  detail::Work wk(p, k);
  std::vector<double> winf(k);
  check(ensei_gpu_prepare_plain(detail::h(p), ds.p, k, dw.p, winf.data(), wk.w.p, nullptr));
  std::vector<uint64_t> packed(k * n);
  dw.download(packed.data(), packed.size());
  // the natural-order canonical copy REF's PreparedPlain::w_eval holds
  DeviceBuffer<uint64_t> nat(k * n);
  std::vector<uint64_t> canon(k * n);
  for (size_t i = 0; i < canon.size(); ++i) canon[i] = ((packed[i] >> 32) << 30) | (packed[i] & 0x3FFFFFFFull);
  nat.upload(canon.data(), canon.size());
  check(ensei_gpu_permute(detail::h(p), 1, nat.p, k, nullptr));
  nat.download(canon.data(), canon.size());
  std::vector<PreparedPlain> out(k);
  for (size_t b = 0; b < k; ++b) {
    out[b].w_eval.domain = RingDomain::Evaluation;
    out[b].w_eval.coeffs.assign(canon.begin() + b * n, canon.begin() + (b + 1) * n);
    out[b].packed.assign(packed.begin() + b * n, packed.begin() + (b + 1) * n);
    out[b].w_inf = winf[b];
  }
  transform_counters().ring_ntt += 2 * k;
  return out;
}
inline PreparedPlain prepare_plain(const PlainVec& w, const RlweParams& p) { return prepare_plain(std::vector<PlainVec>{w}, p)[0]; }

// REF mul_plain's static check (ringbfv.cpp:284-288), identical doubles and message
inline void mul_plain_check(const Ciphertext& ct, const PreparedPlain& w, const RlweParams& p, double& bound,
                            double& mass) {
  const double factor = (double)p.n * w.w_inf;
  bound = ct.noise_bound * factor;
  mass = ct.plain_mass * factor;
  if (bound + mass >= p.noise_cap()) throw NoiseExhausted("plaintext multiplication would exhaust the noise budget");
}

// add_ct(acc, mul_plain(ct_c, w_c)) over c -- REF's channel sum (protocol.cpp:570-581)
// as one device accumulation; the noise bookkeeping is REF's, term by term
inline Ciphertext mul_plain_sum(const std::vector<const Ciphertext*>& cts, const std::vector<const PreparedPlain*>& ws,
                                const RlweParams& p) {
  if (cts.size() != ws.size() || cts.empty()) throw LengthMismatch("one prepared plain per ciphertext");
  Ciphertext out;
  double nb = 0, pm = 0;
  for (size_t c = 0; c < cts.size(); ++c) {
    double b, m;
    mul_plain_check(*cts[c], *ws[c], p, b, m);
    nb += b;  // add_ct sums (REF ringbfv.cpp:243-244)
    pm += m;
  }
  const size_t k = cts.size(), n = p.n;
  DeviceBuffer<uint64_t> dct(k * 2 * n), dw(k * n), dout(2 * n);
  detail::upload_cts(p, cts, dct);
  std::vector<uint64_t> packed(k * n);
  for (size_t c = 0; c < k; ++c) std::copy(ws[c]->packed.begin(), ws[c]->packed.end(), packed.begin() + c * n);
  dw.upload(packed.data(), packed.size());
  for (size_t c = 0; c < k; ++c)
    check(ensei_gpu_mul_plain(detail::h(p), dct.p + c * 2 * n, dw.p + c * n, 1, c > 0 ? 1 : 0, dout.p, nullptr));
  check(ensei_gpu_permute(detail::h(p), 1, dout.p, 2, nullptr));
  detail::download_ct(p, dout, 0, out);
  out.noise_bound = nb;
  out.plain_mass = pm;
  transform_counters().hadamard += k;
  return out;
}
inline Ciphertext mul_plain(const Ciphertext& ct, const PreparedPlain& w, const RlweParams& p) {
  return mul_plain_sum({&ct}, {&w}, p);
}

inline Ciphertext add_ct(const Ciphertext& a, const Ciphertext& b, const RlweParams& p) {  // REF ringbfv.cpp:233-246
  if (a.domain() != b.domain()) throw DomainMismatch("ciphertext domains differ");
  if (a.c0.coeffs.size() != b.c0.coeffs.size()) throw DomainMismatch("ciphertext sizes differ");
  DeviceBuffer<uint64_t> d(4 * p.n);
  detail::upload_cts(p, {&a, &b}, d);
  check(ensei_gpu_add_ct(detail::h(p), d.p, d.p + 2 * p.n, 1, d.p, nullptr));
  check(ensei_gpu_permute(detail::h(p), 1, d.p, 2, nullptr));
  Ciphertext out;
  detail::download_ct(p, d, 0, out);
  out.noise_bound = a.noise_bound + b.noise_bound;
  out.plain_mass = a.plain_mass + b.plain_mass;
  return out;
}

inline Ciphertext add_plain(const Ciphertext& ct, const PlainVec& m, int sign, const RlweParams& p) {  // REF :248-263
  DeviceBuffer<uint64_t> d(2 * p.n), ds(p.n);
  detail::upload_cts(p, {&ct}, d);
  detail::upload_slots(p, {&m}, ds);
  detail::Work w(p, 1);
  check(ensei_gpu_add_plain(detail::h(p), d.p, ds.p, sign, 1, w.w.p, nullptr));
  check(ensei_gpu_permute(detail::h(p), 1, d.p, 2, nullptr));
  Ciphertext out;
  detail::download_ct(p, d, 0, out);
  out.noise_bound = ct.noise_bound;
  out.plain_mass = ct.plain_mass + 1.0;
  transform_counters().ring_ntt += 2;
  return out;
}

// REF hss.cpp:22-62
inline SharePair hom_share_with(const Ciphertext& ct, PlainVec s_b, const ModulusChain& chain, const RlweParams& p) {
  if (chain.p_a > p.p_e) throw ChainViolation("share modulus exceeds plaintext modulus");
  if (s_b.slots.size() != p.n) throw LengthMismatch("share length must equal slot count");
  PlainVec mask;
  mask.slots.resize(p.n);
  for (size_t i = 0; i < p.n; ++i) {
    if (s_b.slots[i] >= chain.p_a) throw ChainViolation("share entry not reduced mod p_a");
    mask.slots[i] = (chain.p_a - s_b.slots[i]) % p.p_e;
  }
  return SharePair{add_plain(ct, mask, +1, p), std::move(s_b), chain.p_a};
}
inline SharePair hom_share(const Ciphertext& ct, const ModulusChain& chain, const RlweParams& p, Rng& rng) {
  PlainVec s_b;
  s_b.slots.resize(p.n);
  rng.uniform_below(chain.p_a, s_b.slots.data(), p.n);
  return hom_share_with(ct, std::move(s_b), chain, p);
}
inline Ciphertext hom_rec(const Ciphertext& alice_ct, const PlainVec& bob_share, const ModulusChain& chain,
                          const RlweParams& p) {
  if (chain.p_a > p.p_e) throw ChainViolation("share modulus exceeds plaintext modulus");
  if (bob_share.slots.size() != p.n) throw LengthMismatch("share length must equal slot count");
  PlainVec reduced;
  reduced.slots.resize(p.n);
  for (size_t i = 0; i < p.n; ++i) reduced.slots[i] = bob_share.slots[i] % p.p_e;
  return add_plain(alice_ct, reduced, +1, p);
}
inline std::vector<Residue> recombine_clear(const std::vector<Residue>& a, const std::vector<Residue>& b, uint64_t p_a) {
  if (a.size() != b.size()) throw LengthMismatch("share vectors differ in length");
  std::vector<Residue> out(a.size());
  for (size_t i = 0; i < a.size(); ++i) out[i] = (a[i] % p_a + b[i] % p_a) % p_a;
  return out;
}

// ============================================= batched conv layer (run_inproc)
// REF PhaseTimings / PartyResult (protocol.hpp:80-94) for one batched conv layer run
// through the fused device path (REF run_inproc, protocol.cpp:670-692, one conv step):
// setup = Bob's weight preparation, online = the layer, its phases timed with the
// library's per-kernel CUDA events (encrypt = Enc, filter = ElementMult + HomShare,
// decrypt = Dec + IDFT2D + recombination).
struct PhaseTimings {
  double setup_seconds = 0, online_seconds = 0, encrypt_seconds = 0, filter_seconds = 0, hadamard_seconds = 0,
         decrypt_seconds = 0;
};
struct PartyResult {
  std::vector<uint32_t> output;  // [img][cout][oh][ow], mod p_a
  TransformCounters online_counters;
  PhaseTimings timings;
};
inline PartyResult run_inproc_layer(Context& ctx, const ensei_conv_desc& desc, const std::vector<uint8_t>& images,
                                    uint32_t num_images, const std::vector<int32_t>& weights, uint64_t seed) {
  ensei_layer_geom g;
  check(ensei_gpu_layer_geometry(ctx.get(), &desc, &g));
  PartyResult res;
  auto t0 = std::chrono::steady_clock::now();
  DeviceBuffer<int32_t> dw(weights.size());
  dw.upload(weights.data(), weights.size());
  DeviceBuffer<uint8_t> dwe(ensei_gpu_prepared_weights_bytes(ctx.get(), &desc));
  check(ensei_gpu_prepare_weights(ctx.get(), &desc, dw.p, reinterpret_cast<uint64_t*>(dwe.p), nullptr));
  cudaDeviceSynchronize();
  res.timings.setup_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  ensei_ctx_info info;
  check(ensei_gpu_ctx_query(ctx.get(), &info));
  DeviceBuffer<uint64_t> key(ENSEI_KEY_WORDS(info.n, info.num_q));
  auto mix = [](uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
  };
  ensei_randomness rnd{};
  rnd.mode = ENSEI_RAND_PHILOX;
  rnd.alice_key = mix(seed ^ mix(0xA11CEull));
  rnd.bob_key = mix(seed ^ mix(0xB0Bull));
  check(ensei_gpu_secret_sample(ctx.get(), rnd.alice_key, nullptr, key.p, nullptr));
  DeviceBuffer<uint8_t> din(images.size()), ws(ensei_gpu_conv_workspace_bytes(ctx.get(), &desc, num_images));
  din.upload(images.data(), images.size());
  const size_t nout = (size_t)num_images * desc.cout * g.oh * g.ow;
  DeviceBuffer<uint32_t> dout(nout);
  cudaDeviceSynchronize();
  check(ensei_gpu_profile(1));
  auto t1 = std::chrono::steady_clock::now();
  check(ensei_gpu_conv_layer(ctx.get(), &desc, key.p, 0, reinterpret_cast<uint64_t*>(dwe.p), din.p, ENSEI_IN_U8,
                             nullptr, num_images, &rnd, ws.p, nullptr, nullptr, dout.p, nullptr));
  cudaDeviceSynchronize();
  res.timings.online_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count();
  char names[64 * 32];
  double ms[64];
  uint32_t cnt[64], nk = 0;
  check(ensei_gpu_profile_read(64, names, ms, cnt, &nk));
  check(ensei_gpu_profile(0));
  for (uint32_t i = 0; i < nk && i < 64; ++i) {
    const std::string nm(names + 32 * i);
    const double s = ms[i] * 1e-3;
    if (nm == "enc" || nm == "homrec") res.timings.encrypt_seconds += s;
    else if (nm == "dec" || nm == "dec_rns") res.timings.decrypt_seconds += s;
    else {
      res.timings.filter_seconds += s;
      if (nm.rfind("mac", 0) == 0 || nm.rfind("planes", 0) == 0) res.timings.hadamard_seconds += s;
    }
  }
  res.output.resize(nout);
  dout.download(res.output.data(), nout);
  // REF's logical counts for the batch (FreqDirect; protocol.cpp:310-355, 537-607)
  const uint64_t B = g.blocks;
  res.online_counters.image_ntt = (uint64_t)num_images * (desc.cin + 2 * desc.cout);
  res.online_counters.ring_ntt = (uint64_t)num_images * B * (2 * desc.cin + 2 * desc.cout + 2 * desc.cout);
  res.online_counters.hadamard = (uint64_t)num_images * B * desc.cin * desc.cout;
  return res;
}

}  // namespace ensei_b200
