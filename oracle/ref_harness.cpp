// ref_harness.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" harness over the UNMODIFIED reference library, compiled
// from the read-only sources under /root/reference/proj/core by
// oracle/Makefile into oracle/_ref/libensei_ref.so.  It never copies reference
// code: it includes the reference headers and calls the reference's public
// API (FieldSpec, NegacyclicPlan, ntt_2d/intt_2d, make_rlwe_params, keygen,
// encrypt_freq_direct, decrypt, run_alice/run_bob, reference_pipeline).
//
// Uses: (1) pinning the C restatement (oracle/ensei_oracle.c) and the GPU path
// bit-exactly, (2) the CPU baseline legs of bench.py.
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "ensei/counters.hpp"
#include "ensei/hss.hpp"
#include "ensei/modfield.hpp"
#include "ensei/ntt.hpp"
#include "ensei/params.hpp"
#include "ensei/protocol.hpp"
#include "ensei/ringbfv.hpp"
#include "ensei/wire.hpp"

using namespace ensei;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  return -1;
}

// Captures every frame crossing a party's transport (both directions).
struct CaptureTransport : Transport {
  Transport* inner;
  std::vector<Frame> sent, recv;
  explicit CaptureTransport(Transport* t) : inner(t) {}
  void send_frame(const Frame& f) override {
    sent.push_back(f);
    inner->send_frame(f);
  }
  Frame recv_frame() override {
    Frame f = inner->recv_frame();
    recv.push_back(f);
    return f;
  }
};

ParamSet make_paramset(uint64_t p, uint64_t q, uint32_t n, double sigma) {
  ParamSet ps;
  FieldSpec f = FieldSpec::make(p);
  ps.chain = ModulusChain::unified(f);
  ps.rlwe = make_rlwe_params(n, q, p, sigma);
  ps.mode = ChainMode::Unified;
  ps.insecure = n < 1024;
  return ps;
}

struct ProtoArgs {
  ProtocolConfig cfg;
  std::vector<Mat> image;
  NetworkWeights weights;
};

// layer_desc: 7 ints per layer {kind(0 conv,1 act), fh, fw, same, cin, cout, fn}
ProtoArgs make_proto(uint64_t p, uint64_t q, uint32_t n, double sigma, int freq_direct,
                     uint64_t seed, uint32_t H, uint32_t W, uint32_t nlayers,
                     const int32_t* desc, const int64_t* image, const int64_t* weights) {
  ProtoArgs a;
  a.cfg.params = make_paramset(p, q, n, sigma);
  a.cfg.mode = freq_direct ? PipelineMode::FreqDirect : PipelineMode::Baseline;
  a.cfg.seed = seed;
  a.cfg.image_h = H;
  a.cfg.image_w = W;
  size_t woff = 0;
  uint32_t cin0 = 0;
  for (uint32_t l = 0; l < nlayers; ++l) {
    const int32_t* d = desc + 7 * l;
    LayerSpec s;
    if (d[0] == 0) {
      s.kind = LayerKind::Conv;
      s.filter_h = d[1];
      s.filter_w = d[2];
      s.conv_type = d[3] ? ConvType::Same : ConvType::Valid;
      s.channels_in = d[4];
      s.channels_out = d[5];
      if (!cin0) cin0 = d[4];
      LayerWeights bank(d[5], std::vector<Mat>(d[4], Mat(d[1], d[2])));
      for (auto& row : bank)
        for (Mat& m : row)
          for (auto& v : m.data) v = weights ? weights[woff++] : 0;
      a.weights.push_back(std::move(bank));
    } else {
      s.kind = LayerKind::Activation;
      s.fn = static_cast<ActivationFn>(d[6]);
    }
    a.cfg.schedule.layers.push_back(s);
  }
  for (uint32_t c = 0; c < cin0; ++c) {
    Mat m(H, W);
    for (size_t i = 0; i < (size_t)H * W; ++i) m.data[i] = image ? image[(size_t)c * H * W + i] : 0;
    a.image.push_back(std::move(m));
  }
  return a;
}

// Parses a CiphertextBlocks / AliceShareCiphertexts payload into [ch][blk][2][n].
void parse_ct_frame(const Frame& f, uint64_t* out) {
  const uint8_t* b = f.payload.data();
  auto u32 = [&](size_t off) { uint32_t v; std::memcpy(&v, b + off, 4); return v; };
  uint32_t ch = u32(4), blocks = u32(8);
  size_t off = 12;
  size_t k = 0;
  for (uint32_t i = 0; i < ch * blocks; ++i) {
    off += 1;  // domain tag
    uint64_t n;
    std::memcpy(&n, b + off, 8);
    off += 8;
    std::memcpy(out + k, b + off, 16 * n);
    off += 16 * n;
    k += 2 * n;
  }
}

void parse_share_frame(const Frame& f, uint64_t* out) {
  const uint8_t* b = f.payload.data();
  uint32_t ch, r, c;
  std::memcpy(&ch, b + 4, 4);
  std::memcpy(&r, b + 8, 4);
  std::memcpy(&c, b + 12, 4);
  std::memcpy(out, b + 16, 8ull * ch * r * c);
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_field_info(uint64_t p, uint64_t* generator, int32_t* two_adicity) {
  try {
    FieldSpec f = FieldSpec::make(p);
    *generator = f.generator();
    *two_adicity = f.two_adicity();
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

uint64_t ref_mulmod(uint64_t a, uint64_t b, uint64_t p) { return FieldSpec::make(p).mul(a, b); }

uint64_t ref_find_prime(uint64_t min_value, uint64_t residue, uint64_t modulus) {
  try { return find_prime(min_value, residue, modulus); } catch (const std::exception& e) { fail(e); return 0; }
}

uint64_t ref_root_of_unity(uint64_t order, uint64_t p) {
  try { return find_root_of_unity(order, FieldSpec::make(p)); } catch (const std::exception& e) { fail(e); return 0; }
}

// NegacyclicPlan::forward/inverse over `count` contiguous polynomials
int ref_negacyclic(uint64_t q, uint32_t n, uint64_t* data, size_t count, int inverse) {
  try {
    NegacyclicPlan plan = NegacyclicPlan::make(FieldSpec::make(q), n);
    std::vector<Residue> x(n);
    for (size_t i = 0; i < count; ++i) {
      std::memcpy(x.data(), data + i * n, 8ull * n);
      if (inverse) plan.inverse(x); else plan.forward(x);
      std::memcpy(data + i * n, x.data(), 8ull * n);
    }
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

int ref_plan_psi(uint64_t q, uint32_t n, uint64_t* psi) {
  try { *psi = NegacyclicPlan::make(FieldSpec::make(q), n).psi; return 0; }
  catch (const std::exception& e) { return fail(e); }
}

// ntt_2d / intt_2d on `count` rows x cols tiles
int ref_ntt2d(uint64_t p, uint32_t rows, uint32_t cols, uint64_t* data, size_t count, int inverse) {
  try {
    FieldSpec f = FieldSpec::make(p);
    for (size_t i = 0; i < count; ++i) {
      FreqTensor t;
      t.rows = rows;
      t.cols = cols;
      t.field = f;
      t.domain = inverse ? TensorDomain::Frequency : TensorDomain::Time;
      t.data.assign(data + i * rows * cols, data + (i + 1) * rows * cols);
      FreqTensor o = inverse ? intt_2d(t) : ntt_2d(t);
      std::memcpy(data + i * rows * cols, o.data.data(), 8ull * rows * cols);
    }
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

int ref_ntt1d(uint64_t p, uint64_t omega, uint64_t* data, size_t len, int inverse) {
  try {
    FieldSpec f = FieldSpec::make(p);
    std::vector<Residue> x(data, data + len);
    std::vector<Residue> y = inverse ? intt_1d(x, omega, f) : ntt_1d(x, omega, f);
    std::memcpy(data, y.data(), 8 * len);
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

int ref_conv_oracle(uint64_t p, const int64_t* image, uint32_t H, uint32_t W, const int64_t* filt,
                    uint32_t fh, uint32_t fw, int same, uint64_t* out) {
  try {
    FieldSpec f = FieldSpec::make(p);
    ConvGeometry g = make_geometry(H, W, fh, fw, same ? ConvType::Same : ConvType::Valid, f);
    Mat u(H, W), w(fh, fw);
    for (size_t i = 0; i < (size_t)H * W; ++i) u.data[i] = image[i];
    for (size_t i = 0; i < (size_t)fh * fw; ++i) w.data[i] = filt[i];
    std::vector<Residue> r = conv_oracle(u, w, g, f);
    std::memcpy(out, r.data(), 8 * r.size());
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

int ref_geometry(uint64_t p, uint32_t H, uint32_t W, uint32_t fh, uint32_t fw, int same,
                 uint32_t* padded_h, uint32_t* padded_w) {
  try {
    ConvGeometry g = make_geometry(H, W, fh, fw, same ? ConvType::Same : ConvType::Valid,
                                   FieldSpec::make(p));
    *padded_h = (uint32_t)g.padded_h;
    *padded_w = (uint32_t)g.padded_w;
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

// encode_slots (inverse=0 -> slots to coefficients) / decode_slots
int ref_slots(uint64_t p, uint64_t q, uint32_t n, uint64_t* data, int decode) {
  try {
    RlweParams prm = make_rlwe_params(n, q, p, 4.0);
    if (!decode) {
      PlainVec v;
      v.slots.assign(data, data + n);
      RingElem m = encode_slots(v, prm);
      std::memcpy(data, m.coeffs.data(), 8ull * n);
    } else {
      RingElem m;
      m.coeffs.assign(data, data + n);
      m.domain = RingDomain::Coefficient;
      PlainVec v = decode_slots(m, prm);
      std::memcpy(data, v.slots.data(), 8ull * n);
    }
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

// Rng draws (reference stream): kind 0 = next_u64, 1 = uniform_below(bound), 2 = gaussian(sigma)
int ref_rng_draw(uint64_t seed, uint64_t salt, int use_fork, int kind, uint64_t bound,
                 double sigma, size_t count, int64_t* out) {
  try {
    Rng r = use_fork ? Rng(seed).fork(salt) : Rng(seed);
    for (size_t i = 0; i < count; ++i) {
      if (kind == 0) out[i] = (int64_t)r.next_u64();
      else if (kind == 1) out[i] = (int64_t)r.uniform_below(bound);
      else out[i] = r.sample_gaussian(sigma);
    }
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

// Alice's session key exactly as AliceSession builds it (protocol.cpp:284-290)
int ref_session_key(uint64_t p, uint64_t q, uint32_t n, double sigma, uint64_t seed,
                    int64_t* t_signed, uint64_t* t_eval) {
  try {
    RlweParams prm = make_rlwe_params(n, q, p, sigma);
    Rng rng = Rng(seed).fork(0xA11CE);
    SecretKey sk = keygen(prm, rng);
    for (uint32_t i = 0; i < n; ++i) t_signed[i] = decode_signed(sk.t.coeffs[i], prm.q);
    std::memcpy(t_eval, sk.t_eval.coeffs.data(), 8ull * n);
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

// One encrypt_freq_direct with a fresh Rng(seed) (no fork); ct = [2][n]
int ref_encrypt_freq_direct(uint64_t p, uint64_t q, uint32_t n, double sigma,
                            const uint64_t* t_eval, const uint64_t* slots, uint64_t seed,
                            uint64_t* ct) {
  try {
    RlweParams prm = make_rlwe_params(n, q, p, sigma);
    SecretKey sk;
    sk.t_eval.coeffs.assign(t_eval, t_eval + n);
    sk.t_eval.domain = RingDomain::Evaluation;
    PlainVec m;
    m.slots.assign(slots, slots + n);
    Rng rng(seed);
    Ciphertext c = encrypt_freq_direct(m, sk, prm, rng);
    std::memcpy(ct, c.c0.coeffs.data(), 8ull * n);
    std::memcpy(ct + n, c.c1.coeffs.data(), 8ull * n);
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

int ref_decrypt(uint64_t p, uint64_t q, uint32_t n, const uint64_t* t_eval, const uint64_t* ct,
                uint64_t* slots) {
  try {
    RlweParams prm = make_rlwe_params(n, q, p, 4.0);
    SecretKey sk;
    sk.t_eval.coeffs.assign(t_eval, t_eval + n);
    sk.t_eval.domain = RingDomain::Evaluation;
    Ciphertext c;
    c.c0.coeffs.assign(ct, ct + n);
    c.c1.coeffs.assign(ct + n, ct + 2 * n);
    c.c0.domain = c.c1.domain = RingDomain::Evaluation;
    PlainVec v = decrypt(c, sk, prm);
    std::memcpy(slots, v.slots.data(), 8ull * n);
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

int ref_prepare_plain(uint64_t p, uint64_t q, uint32_t n, const uint64_t* slots, uint64_t* w_eval,
                      double* w_inf) {
  try {
    RlweParams prm = make_rlwe_params(n, q, p, 4.0);
    PlainVec v;
    v.slots.assign(slots, slots + n);
    PreparedPlain pp = prepare_plain(v, prm);
    std::memcpy(w_eval, pp.w_eval.coeffs.data(), 8ull * n);
    *w_inf = pp.w_inf;
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

// Full two-party protocol (run_alice/run_bob on two threads over an in-process
// pair, like run_inproc) with frame capture.  capture_conv selects which conv
// layer's ciphertext frames are returned.
int ref_run_protocol(uint64_t p, uint64_t q, uint32_t n, double sigma, int freq_direct,
                     uint64_t seed, uint32_t H, uint32_t W, uint32_t nlayers,
                     const int32_t* desc, const int64_t* image, const int64_t* weights,
                     uint64_t* out, uint64_t* hashes, uint64_t* counters, uint32_t capture_conv,
                     uint64_t* ct_a2b, uint64_t* ct_b2a, uint64_t* bob_up, double* timings) {
  try {
    ProtoArgs a = make_proto(p, q, n, sigma, freq_direct, seed, H, W, nlayers, desc, image, weights);
    auto [ta, tb] = make_inproc_pair();
    CaptureTransport ca(ta.get()), cb(tb.get());
    PartyResult ra, rb;
    std::exception_ptr eb, ea;
    std::thread bob([&] {
      try { rb = run_bob(a.cfg, a.weights, cb); } catch (...) { eb = std::current_exception(); }
    });
    try { ra = run_alice(a.cfg, a.image, ca); } catch (...) { ea = std::current_exception(); }
    bob.join();
    if (ea) std::rethrow_exception(ea);
    if (eb) std::rethrow_exception(eb);
    size_t k = 0;
    for (const ResMat& m : ra.output)
      for (Residue v : m.v) out[k++] = v;
    if (hashes) {
      hashes[0] = ra.transcript.content_hash_sent;
      hashes[1] = ra.transcript.content_hash_recv;
      hashes[2] = rb.transcript.content_hash_sent;
      hashes[3] = rb.transcript.content_hash_recv;
      hashes[4] = ra.transcript.total_bytes(Direction::Sent);
      hashes[5] = rb.transcript.total_bytes(Direction::Sent);
    }
    if (counters) {
      const TransformCounters* cs[2] = {&ra.online_counters, &rb.online_counters};
      for (int i = 0; i < 2; ++i) {
        counters[4 * i + 0] = cs[i]->ct_ntt;
        counters[4 * i + 1] = cs[i]->ring_ntt;
        counters[4 * i + 2] = cs[i]->image_ntt;
        counters[4 * i + 3] = cs[i]->hadamard;
      }
    }
    uint32_t conv_seen = 0;
    for (const Frame& f : ca.sent)
      if (f.type == MsgType::CiphertextBlocks) {
        if (conv_seen++ == capture_conv && ct_a2b) parse_ct_frame(f, ct_a2b);
      }
    conv_seen = 0;
    for (const Frame& f : ca.recv)
      if (f.type == MsgType::AliceShareCiphertexts) {
        if (conv_seen++ == capture_conv && ct_b2a) parse_ct_frame(f, ct_b2a);
      }
    if (bob_up) {  // Bob's first ActivationShareUp after the captured conv layer
      conv_seen = 0;
      bool armed = false;
      for (const Frame& f : cb.sent) {
        if (f.type == MsgType::AliceShareCiphertexts && conv_seen++ == capture_conv) armed = true;
        if (armed && f.type == MsgType::ActivationShareUp) { parse_share_frame(f, bob_up); break; }
      }
    }
    if (timings) {
      timings[0] = ra.timings.setup_seconds;
      timings[1] = ra.timings.online_seconds;
      timings[2] = rb.timings.setup_seconds;
      timings[3] = rb.timings.online_seconds;
    }
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

int ref_reference_pipeline(uint64_t p, uint64_t q, uint32_t n, uint32_t H, uint32_t W,
                           uint32_t nlayers, const int32_t* desc, const int64_t* image,
                           const int64_t* weights, uint64_t* out) {
  try {
    ProtoArgs a = make_proto(p, q, n, 4.0, 1, 0, H, W, nlayers, desc, image, weights);
    std::vector<ResMat> r = reference_pipeline(a.cfg, a.image, a.weights);
    size_t k = 0;
    for (const ResMat& m : r)
      for (Residue v : m.v) out[k++] = v;
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

// CPU baseline: `instances` independent run_inproc sessions (seed + i) spread
// over `threads` host threads; returns wall seconds (the reference's own
// concurrency model: independent ciphertext workers).
// online_sum (optional) receives the sum over sessions of Alice's online seconds
// (REF PhaseTimings::online_seconds: Hello done -> Done, i.e. excluding Bob's weight
// preparation, the paper's t_setup).  Each session runs on 2 threads (run_inproc).
double ref_bench_protocol(uint64_t p, uint64_t q, uint32_t n, double sigma, uint64_t seed,
                          uint32_t H, uint32_t W, uint32_t nlayers, const int32_t* desc,
                          const int64_t* image, const int64_t* weights, uint32_t instances,
                          uint32_t threads, double* online_sum) {
  try {
    ProtoArgs a = make_proto(p, q, n, sigma, 1, seed, H, W, nlayers, desc, image, weights);
    std::atomic<uint32_t> next{0};
    std::atomic<int> bad{0};
    std::vector<double> online(instances, 0.0);
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (uint32_t t = 0; t < threads; ++t)
      pool.emplace_back([&] {
        for (;;) {
          uint32_t i = next++;
          if (i >= instances) break;
          ProtocolConfig cfg = a.cfg;
          cfg.seed = seed + i;
          try {
            InprocRun r = run_inproc(cfg, a.image, a.weights);
            online[i] = r.alice.timings.online_seconds;
          } catch (...) { bad++; }
        }
      });
    for (auto& th : pool) th.join();
    if (online_sum) {
      double acc = 0;
      for (double v : online) acc += v;
      *online_sum = acc;
    }
    double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return bad ? -1.0 : s;
  } catch (const std::exception& e) { fail(e); return -1.0; }
}

// CPU baseline at the operator level: the per-image online work of one conv step of a
// REF session -- Alice pad_image -> ntt_2d -> flatten -> encrypt_freq_direct per block;
// Bob mul_plain / add_ct per (out, block) over the input channels, hom_share, merge ->
// intt_2d -> crop (his share); Alice decrypt -> merge -> intt_2d -> crop -- made of the
// same REF calls AliceSession / BobSession make (protocol.cpp:310-355, 537-603), without
// the in-process transport, and with Bob's prepare_plain table built ONCE for the batch
// (REF rebuilds it in every session: 8192 prepare_plain at n = 8192 for config 4, ~20 s
// per image, which would make a bounded sample impossible).  Per image the Rng streams
// are a session's: Rng(seed + i).fork(0xA11CE) (keygen, Enc) and .fork(0xB0B) (shares).
// Single layer; `threads` host threads over images (and over output channels for the
// setup).  Returns the wall seconds of the online phase; *online_sum = the sum over
// images of the per-image online seconds; *setup_s = the prepare_plain wall time.
namespace {
std::vector<PlainVec> h_split(const std::vector<Residue>& flat, size_t n) {
  std::vector<PlainVec> out((flat.size() + n - 1) / n);
  for (size_t i = 0; i < out.size() * n; ++i) {
    if (i % n == 0) out[i / n].slots.assign(n, 0);
    if (i < flat.size()) out[i / n].slots[i % n] = flat[i];
  }
  return out;
}
std::vector<Residue> h_merge(const std::vector<PlainVec>& blocks, size_t len) {
  std::vector<Residue> out(len);
  for (size_t i = 0; i < len; ++i) out[i] = blocks[i / blocks[0].slots.size()].slots[i % blocks[0].slots.size()];
  return out;
}
}  // namespace

double ref_bench_layer_ops(uint64_t p, uint64_t q, uint32_t n, double sigma, uint64_t seed, uint32_t H,
                           uint32_t W, uint32_t fh, uint32_t fw, int same, uint32_t cin, uint32_t cout,
                           const int64_t* image, const int64_t* weights, uint32_t images, uint32_t threads,
                           double* online_sum, double* setup_s) {
  try {
    const ParamSet ps = make_paramset(p, q, n, sigma);
    const RlweParams& params = ps.rlwe;
    const FieldSpec& pn = ps.chain.p_n;
    const ConvGeometry g = make_geometry(H, W, fh, fw, same ? ConvType::Same : ConvType::Valid, pn);
    const size_t grid = g.padded_h * g.padded_w, B = (grid + n - 1) / n;
    ConvGeometry fg = g;
    std::swap(fg.image_h, fg.filter_h);
    std::swap(fg.image_w, fg.filter_w);
    // Bob's setup (REF BobSession::prepare_weights, protocol.cpp:462-502)
    std::vector<std::vector<std::vector<PreparedPlain>>> prep(cout, std::vector<std::vector<PreparedPlain>>(cin));
    auto t0 = std::chrono::steady_clock::now();
    {
      std::atomic<uint32_t> next{0};
      std::vector<std::thread> pool;
      for (uint32_t t = 0; t < threads; ++t)
        pool.emplace_back([&] {
          for (uint32_t o; (o = next++) < cout;)
            for (uint32_t c = 0; c < cin; ++c) {
              Mat filt(fh, fw);
              for (size_t k = 0; k < (size_t)fh * fw; ++k) filt.data[k] = weights[((size_t)o * cin + c) * fh * fw + k];
              for (PlainVec& blk : h_split(flatten(ntt_2d(pad_image(filt, fg, pn))), n)) {
                for (Residue& v : blk.slots) v = params.p_e.reduce(v);
                prep[o][c].push_back(prepare_plain(blk, params));
              }
            }
        });
      for (auto& th : pool) th.join();
    }
    if (setup_s) *setup_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::vector<Mat> img(cin, Mat(H, W));
    for (uint32_t c = 0; c < cin; ++c)
      for (size_t k = 0; k < (size_t)H * W; ++k) img[c].data[k] = image[(size_t)c * H * W + k];
    std::vector<double> online(images, 0.0);
    std::atomic<uint32_t> next{0};
    std::atomic<int> bad{0};
    auto t1 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (uint32_t t = 0; t < threads; ++t)
      pool.emplace_back([&] {
        for (uint32_t i; (i = next++) < images;) {
          try {
            Rng root(seed + i);
            Rng alice = root.fork(0xA11CE), bob = root.fork(0xB0B);
            SecretKey sk = keygen(params, alice);
            auto s0 = std::chrono::steady_clock::now();
            std::vector<std::vector<Ciphertext>> cts(cin);
            for (uint32_t c = 0; c < cin; ++c)
              for (PlainVec& blk : h_split(flatten(ntt_2d(pad_image(img[c], g, pn))), n))
                cts[c].push_back(encrypt_freq_direct(blk, sk, params, alice));
            std::vector<ResMat> bob_share, alice_share;
            for (uint32_t o = 0; o < cout; ++o) {
              std::vector<PlainVec> mine, dec;
              for (size_t b = 0; b < B; ++b) {
                Ciphertext acc = mul_plain(cts[0][b], prep[o][0][b], params);
                for (uint32_t c = 1; c < cin; ++c) acc = add_ct(acc, mul_plain(cts[c][b], prep[o][c][b], params), params);
                SharePair sp = hom_share(acc, ps.chain, params, bob);
                mine.push_back(std::move(sp.bob_share));
                dec.push_back(decrypt(sp.alice_ct, sk, params));
              }
              for (auto* v : {&mine, &dec}) {
                std::vector<Residue> flat = h_merge(*v, grid);
                for (Residue& x : flat) x = pn.reduce(x);
                FreqTensor tt = intt_2d(unflatten(flat, g.padded_h, g.padded_w, pn, TensorDomain::Frequency));
                ResMat m(g.out_h(), g.out_w());
                for (size_t r = 0; r < m.rows; ++r)
                  for (size_t cc = 0; cc < m.cols; ++cc) m.at(r, cc) = tt.at(r + g.crop_r0(), cc + g.crop_c0());
                (v == &mine ? bob_share : alice_share).push_back(std::move(m));
              }
            }
            online[i] = std::chrono::duration<double>(std::chrono::steady_clock::now() - s0).count();
          } catch (...) {
            bad++;
          }
        }
      });
    for (auto& th : pool) th.join();
    if (online_sum) {
      double acc = 0;
      for (double v : online) acc += v;
      *online_sum = acc;
    }
    if (bad) return -1.0;
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count();
  } catch (const std::exception& e) {
    fail(e);
    return -1.0;
  }
}

// CPU baseline for config 2: `count` polynomials, forward then inverse, over `threads`.
double ref_bench_negacyclic(uint64_t q, uint32_t n, uint64_t* data, size_t count, uint32_t threads) {
  try {
    NegacyclicPlan plan = NegacyclicPlan::make(FieldSpec::make(q), n);
    std::atomic<size_t> next{0};
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (uint32_t t = 0; t < threads; ++t)
      pool.emplace_back([&] {
        std::vector<Residue> x(n);
        for (;;) {
          size_t i = next++;
          if (i >= count) break;
          std::memcpy(x.data(), data + i * n, 8ull * n);
          plan.forward(x);
          plan.inverse(x);
          std::memcpy(data + i * n, x.data(), 8ull * n);
        }
      });
    for (auto& th : pool) th.join();
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  } catch (const std::exception& e) { fail(e); return -1.0; }
}

// ---------------------------------------------------------------- wire framing
// REF's message layouts through its PUBLIC wire API (ByteWriter / write_ciphertext /
// encode_frame, decode_frame / ByteReader / read_ciphertext, wire.cpp:44-144); the
// payload walk is the one of the file-local encode_ct_blocks / decode_ct_blocks /
// encode_shares / decode_shares and recv_expect (protocol.cpp:55-150).
static int wire_code(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const MalformedPayload*>(&e)) return 14;
  if (dynamic_cast<const ProtocolOrderViolation*>(&e)) return 12;
  return -1;
}

static Frame expect_frame(const uint8_t* bytes, size_t len, uint32_t expect) {
  Frame f = decode_frame(std::vector<uint8_t>(bytes, bytes + len));
  if (f.type == MsgType::Error)
    throw ProtocolOrderViolation("peer aborted: " + std::string(f.payload.begin(), f.payload.end()));
  if (f.type != static_cast<MsgType>(expect))
    throw ProtocolOrderViolation(std::string("expected ") + msg_type_name(static_cast<MsgType>(expect)) +
                                 ", got " + msg_type_name(f.type));
  return f;
}

int ref_wire_ct_frame(uint32_t type, uint32_t layer, uint32_t n, uint32_t channels, uint32_t blocks, int tag,
                      const uint64_t* cts, uint8_t* out, size_t cap, size_t* len) {
  try {
    ByteWriter w;
    w.put_u32(layer);
    w.put_u32(channels);
    w.put_u32(channels ? blocks : 0);
    for (size_t r = 0; r < (size_t)channels * blocks; ++r) {
      Ciphertext ct;
      ct.c0.domain = ct.c1.domain = static_cast<RingDomain>(tag);
      ct.c0.coeffs.assign(cts + 2 * r * n, cts + (2 * r + 1) * n);
      ct.c1.coeffs.assign(cts + (2 * r + 1) * n, cts + (2 * r + 2) * n);
      write_ciphertext(w, ct);
    }
    Frame f;
    f.type = static_cast<MsgType>(type);
    f.payload = std::move(w.buf);
    std::vector<uint8_t> b = encode_frame(f);
    *len = b.size();
    if (b.size() > cap) return -2;
    std::memcpy(out, b.data(), b.size());
    return 0;
  } catch (const std::exception& e) { return wire_code(e); }
}

int ref_wire_ct_decode(const uint8_t* bytes, size_t len, uint32_t expect, uint64_t p, uint64_t q, uint32_t n,
                       uint32_t channels, uint32_t blocks, uint32_t* layer, uint64_t* cts, uint8_t* tags) {
  try {
    RlweParams prm = make_rlwe_params(n, q, p, 4.0);
    Frame f = expect_frame(bytes, len, expect);
    ByteReader r(f.payload);
    *layer = r.get_u32();
    uint32_t ch = r.get_u32(), bl = r.get_u32();
    if (ch != channels || bl != blocks) throw ProtocolOrderViolation("ciphertext block layout mismatch");
    for (size_t k = 0; k < (size_t)ch * bl; ++k) {
      Ciphertext ct = read_ciphertext(r, prm);
      tags[k] = static_cast<uint8_t>(ct.domain());
      std::memcpy(cts + 2 * k * n, ct.c0.coeffs.data(), 8ull * n);
      std::memcpy(cts + (2 * k + 1) * n, ct.c1.coeffs.data(), 8ull * n);
    }
    r.expect_end();
    return 0;
  } catch (const std::exception& e) { return wire_code(e); }
}

int ref_wire_share_frame(uint32_t type, uint32_t layer, uint32_t channels, uint32_t rows, uint32_t cols,
                         const uint64_t* v, uint8_t* out, size_t cap, size_t* len) {
  try {
    ByteWriter w;
    w.put_u32(layer);
    w.put_u32(channels);
    w.put_u32(channels ? rows : 0);
    w.put_u32(channels ? cols : 0);
    for (size_t i = 0; i < (size_t)channels * rows * cols; ++i) w.put_u64(v[i]);
    Frame f;
    f.type = static_cast<MsgType>(type);
    f.payload = std::move(w.buf);
    std::vector<uint8_t> b = encode_frame(f);
    *len = b.size();
    if (b.size() > cap) return -2;
    std::memcpy(out, b.data(), b.size());
    return 0;
  } catch (const std::exception& e) { return wire_code(e); }
}

int ref_wire_share_decode(const uint8_t* bytes, size_t len, uint32_t expect, uint32_t channels, uint32_t rows,
                          uint32_t cols, uint64_t max_value, uint32_t* layer, uint64_t* v) {
  try {
    Frame f = expect_frame(bytes, len, expect);
    ByteReader r(f.payload);
    *layer = r.get_u32();
    uint32_t ch = r.get_u32(), ro = r.get_u32(), co = r.get_u32();
    if (ch != channels || ro != rows || co != cols) throw ProtocolOrderViolation("share layout mismatch");
    for (size_t i = 0; i < (size_t)ch * ro * co; ++i) {
      uint64_t x = r.get_u64();
      if (x >= max_value) throw MalformedPayload("share value out of range");
      v[i] = x;
    }
    r.expect_end();
    return 0;
  } catch (const std::exception& e) { return wire_code(e); }
}

uint64_t ref_config_digest(uint64_t p, uint64_t q, uint32_t n, double sigma, int freq_direct, uint64_t seed,
                           uint32_t H, uint32_t W, uint32_t nlayers, const int32_t* desc) {
  try {
    ProtoArgs a = make_proto(p, q, n, sigma, freq_direct, seed, H, W, nlayers, desc, nullptr, nullptr);
    return config_digest(a.cfg);
  } catch (const std::exception& e) { fail(e); return 0; }
}

// ------------------------------------------------------------------ parameters
static int param_code(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const SearchExhausted*>(&e)) return 3;
  if (dynamic_cast<const RangeViolation*>(&e)) return 11;
  if (dynamic_cast<const ChainViolation*>(&e)) return 9;
  return 1;
}

static void put_params(const ParamSet& ps, uint64_t* out) {
  out[0] = ps.chain.p_n.modulus();
  out[1] = ps.chain.p_a.modulus();
  out[2] = ps.chain.p_e.modulus();
  out[3] = ps.rlwe.q.modulus();
  out[4] = ps.rlwe.n;
  out[5] = ps.insecure ? 1 : 0;
}

int ref_min_pntt(int ib, int fb, int fh, int fw, uint64_t* out) {
  try {
    *out = min_pntt(PrecisionProfile{ib, fb, fh, fw});
    return 0;
  } catch (const std::exception& e) { return param_code(e); }
}

int ref_build_params(int ib, int fb, int fh, int fw, uint32_t n, int split, uint64_t accum, uint64_t floor_,
                     double sigma, uint64_t* out) {
  try {
    put_params(build_params(PrecisionProfile{ib, fb, fh, fw}, n, split ? ChainMode::SplitPaper : ChainMode::Unified,
                            accum, floor_, sigma), out);
    return 0;
  } catch (const std::exception& e) { return param_code(e); }
}

int ref_preset_params(const char* name, uint64_t accum, uint64_t* out) {
  try {
    put_params(preset_params(name, accum), out);
    return 0;
  } catch (const std::exception& e) { return param_code(e); }
}

// REF random_weights (protocol.cpp:752-767) with Rng(seed) or Rng(seed).fork(salt)
int ref_random_weights(uint32_t nlayers, const int32_t* desc, int64_t magnitude, uint64_t seed, int use_fork,
                       uint64_t salt, int64_t* out) {
  try {
    ProtoArgs a = make_proto(638977, 576460803525083137ull, 2048, 4.0, 1, 0, 8, 8, nlayers, desc, nullptr, nullptr);
    Rng r = use_fork ? Rng(seed).fork(salt) : Rng(seed);
    NetworkWeights w = random_weights(a.cfg.schedule, magnitude, r);
    size_t k = 0;
    for (auto& bank : w)
      for (auto& row : bank)
        for (Mat& m : row)
          for (int64_t v : m.data) out[k++] = v;
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

}  // extern "C"
