// tools/cpp_mirror_check.cpp -- the C++ host mirror used the way a REF maintainer
// would: REF's operators next to ensei_b200's with the same inputs and the same Rng
// seeds, compared value by value -- NegacyclicPlan, ntt_2d, keygen,
// encrypt_freq_direct, decrypt, prepare_plain (+ w_inf), mul_plain / add_ct (+ the
// noise bookkeeping and REF's NoiseExhausted trigger), add_plain, hom_share,
// hom_share_with, hom_rec, the TransformCounters deltas, and a batched conv layer's
// PartyResult / PhaseTimings.  Built by oracle/Makefile, run by
// tests/test_gpu_cpp_mirror.py (links oracle/_ref for REF).
#include <cstdio>
#include <cstring>
#include <random>
#include <string>

#include "../paper_2003_05328_b200/csrc/host/ensei_b200.hpp"
#include "ensei/counters.hpp"
#include "ensei/errors.hpp"
#include "ensei/hss.hpp"
#include "ensei/modfield.hpp"
#include "ensei/ntt.hpp"
#include "ensei/ringbfv.hpp"

static int fails = 0;
#define EXPECT(cond, what)                     \
  do {                                         \
    if (!(cond)) {                             \
      std::printf("MISMATCH: %s\n", what);     \
      ++fails;                                 \
    }                                          \
  } while (0)

static bool same_ct(const ensei::Ciphertext& r, const ensei_b200::Ciphertext& b) {
  return r.c0.coeffs == b.c0.coeffs && r.c1.coeffs == b.c1.coeffs && r.noise_bound == b.noise_bound &&
         r.plain_mass == b.plain_mass && (int)r.domain() == (int)b.domain();
}

int main() {
  const uint64_t q = 576460803525083137ULL, p = 638977;
  const uint32_t n = 2048;
  std::mt19937_64 g(7);
  std::vector<uint64_t> x(4 * n);
  for (auto& v : x) v = g() % q;
  // ---- transforms
  ensei::NegacyclicPlan plan = ensei::NegacyclicPlan::make(ensei::FieldSpec::make(q), n);
  std::vector<uint64_t> want = x;
  for (int i = 0; i < 4; ++i) {
    std::vector<ensei::Residue> poly(want.begin() + i * n, want.begin() + (i + 1) * n);
    plan.forward(poly);
    std::copy(poly.begin(), poly.end(), want.begin() + i * n);
  }
  ensei_b200::Context ctx(n, {q}, p);
  std::vector<uint64_t> got = x;
  ctx.negacyclic_forward(got);
  EXPECT(got == want, "negacyclic forward");
  ctx.negacyclic_inverse(got);
  EXPECT(got == x, "negacyclic roundtrip");
  std::vector<uint64_t> tile(64 * 64);
  for (auto& v : tile) v = g() % p;
  ensei::FreqTensor t;
  t.rows = t.cols = 64;
  t.field = ensei::FieldSpec::make(p);
  t.data = tile;
  ensei::FreqTensor f = ensei::ntt_2d(t);
  ctx.ntt_2d(tile, 64, 64);
  EXPECT(tile == f.data, "ntt_2d");
  try {
    ensei_b200::Context bad(n, {q + 2}, p);
    EXPECT(false, "bad q accepted");
  } catch (const ensei_b200::Error&) {
  }

  // ---- operators, same seeds on both sides
  ensei::RlweParams rp = ensei::make_rlwe_params(n, q, p, 4.0);
  ensei_b200::RlweParams bp = ensei_b200::make_rlwe_params(n, q, p, 4.0);
  ensei::ModulusChain rch = ensei::ModulusChain::unified(ensei::FieldSpec::make(p));
  ensei_b200::ModulusChain bch = ensei_b200::ModulusChain::unified(p);
  ensei::Rng rr = ensei::Rng(2026).fork(0xA11CE);
  ensei_b200::Rng br = ensei_b200::Rng(2026).fork(0xA11CE);
  ensei::reset_transform_counters();
  ensei_b200::reset_transform_counters();
  ensei::SecretKey rsk = ensei::keygen(rp, rr);
  ensei_b200::SecretKey bsk = ensei_b200::keygen(bp, br);
  EXPECT(rsk.t.coeffs == bsk.t.coeffs && rsk.t_eval.coeffs == bsk.t_eval.coeffs, "keygen");
  ensei::PlainVec rm;
  ensei_b200::PlainVec bm;
  std::vector<ensei::PlainVec> rws;
  std::vector<ensei_b200::PlainVec> bws;
  for (int k = 0; k < 3; ++k) {
    rm.slots.resize(n);
    for (auto& v : rm.slots) v = g() % p;
    bm.slots = rm.slots;
    ensei::PlainVec w;
    w.slots.resize(n);
    for (auto& v : w.slots) v = (g() % 256 + p - 128) % p;  // small signed taps
    rws.push_back(w);
    bws.push_back(ensei_b200::PlainVec{w.slots});
  }
  std::vector<ensei::Ciphertext> rct;
  std::vector<ensei_b200::PlainVec> bms;
  for (int k = 0; k < 3; ++k) {
    ensei::PlainVec m;
    m.slots.resize(n);
    for (auto& v : m.slots) v = g() % p;
    rct.push_back(ensei::encrypt_freq_direct(m, rsk, rp, rr));
    bms.push_back(ensei_b200::PlainVec{m.slots});
  }
  std::vector<ensei_b200::Ciphertext> bct = ensei_b200::encrypt_freq_direct(bms, bsk, bp, br);  // batched
  for (int k = 0; k < 3; ++k) EXPECT(same_ct(rct[k], bct[k]), "encrypt_freq_direct");
  std::vector<ensei::PreparedPlain> rpp;
  for (auto& w : rws) rpp.push_back(ensei::prepare_plain(w, rp));
  std::vector<ensei_b200::PreparedPlain> bpp = ensei_b200::prepare_plain(bws, bp);
  for (int k = 0; k < 3; ++k)
    EXPECT(rpp[k].w_eval.coeffs == bpp[k].w_eval.coeffs && rpp[k].w_inf == bpp[k].w_inf, "prepare_plain / w_inf");
  // channel sum: add_ct(add_ct(mul(ct0, w0), mul(ct1, w1)), mul(ct2, w2))
  ensei::Ciphertext racc = ensei::mul_plain(rct[0], rpp[0], rp);
  for (int k = 1; k < 3; ++k) racc = ensei::add_ct(racc, ensei::mul_plain(rct[k], rpp[k], rp), rp);
  ensei_b200::Ciphertext bacc = ensei_b200::mul_plain_sum({&bct[0], &bct[1], &bct[2]}, {&bpp[0], &bpp[1], &bpp[2]}, bp);
  EXPECT(same_ct(racc, bacc), "mul_plain + add_ct channel sum (values, noise_bound, plain_mass)");
  ensei_b200::Ciphertext bsum = ensei_b200::add_ct(ensei_b200::mul_plain(bct[0], bpp[0], bp),
                                                   ensei_b200::mul_plain(bct[1], bpp[1], bp), bp);
  ensei::Ciphertext rsum = ensei::add_ct(ensei::mul_plain(rct[0], rpp[0], rp), ensei::mul_plain(rct[1], rpp[1], rp), rp);
  EXPECT(same_ct(rsum, bsum), "add_ct");
  // HomShare / HomRec on Bob's stream
  ensei::Rng rbob = ensei::Rng(2026).fork(0xB0B);
  ensei_b200::Rng bbob = ensei_b200::Rng(2026).fork(0xB0B);
  ensei::SharePair rsp = ensei::hom_share(racc, rch, rp, rbob);
  ensei_b200::SharePair bsp = ensei_b200::hom_share(bacc, bch, bp, bbob);
  EXPECT(rsp.bob_share.slots == bsp.bob_share.slots && same_ct(rsp.alice_ct, bsp.alice_ct), "hom_share");
  ensei::PlainVec zeros;
  zeros.slots.assign(n, 0);
  EXPECT(same_ct(ensei::hom_share_with(racc, zeros, rch, rp).alice_ct,
                 ensei_b200::hom_share_with(bacc, ensei_b200::PlainVec{zeros.slots}, bch, bp).alice_ct),
         "hom_share_with");
  EXPECT(same_ct(ensei::hom_rec(rsp.alice_ct, rsp.bob_share, rch, rp),
                 ensei_b200::hom_rec(bsp.alice_ct, bsp.bob_share, bch, bp)),
         "hom_rec");
  EXPECT(same_ct(ensei::add_plain(racc, rm, -1, rp), ensei_b200::add_plain(bacc, bm, -1, bp)), "add_plain (-1)");
  // decryption of every stage
  EXPECT(ensei::decrypt(rsp.alice_ct, rsk, rp).slots == ensei_b200::decrypt(bsp.alice_ct, bsk, bp).slots,
         "decrypt (HomShare output)");
  std::vector<ensei_b200::PlainVec> bdec = ensei_b200::decrypt(bct, bsk, bp);
  for (int k = 0; k < 3; ++k) EXPECT(ensei::decrypt(rct[k], rsk, rp).slots == bdec[k].slots, "decrypt (batched)");
  // REF's static noise check: a second product on an already multiplied ciphertext
  std::string rmsg, bmsg;
  try {
    ensei::mul_plain(racc, rpp[0], rp);
  } catch (const ensei::NoiseExhausted& e) {
    rmsg = e.what();
  }
  try {
    ensei_b200::mul_plain(bacc, bpp[0], bp);
  } catch (const ensei_b200::NoiseExhausted& e) {
    bmsg = e.what();
  }
  EXPECT(!rmsg.empty() && rmsg == bmsg, "NoiseExhausted (thrown by both, same message)");
  ensei::TransformCounters rc = ensei::transform_counters();
  ensei_b200::TransformCounters bc = ensei_b200::transform_counters();
  EXPECT(rc.ring_ntt == bc.ring_ntt && rc.hadamard == bc.hadamard && rc.ct_ntt == bc.ct_ntt, "TransformCounters");
  if (rc.ring_ntt != bc.ring_ntt || rc.hadamard != bc.hadamard)
    std::printf("  counters REF ring %lu had %lu | b200 ring %lu had %lu\n", (unsigned long)rc.ring_ntt,
                (unsigned long)rc.hadamard, (unsigned long)bc.ring_ntt, (unsigned long)bc.hadamard);

  // ---- batched conv layer: output == REF's plaintext convolution, PhaseTimings filled
  {
    ensei_conv_desc d{16, 16, 3, 3, 1, 4, 3};
    const uint32_t imgs = 2;
    std::vector<uint8_t> im(imgs * 4 * 16 * 16);
    for (auto& v : im) v = (uint8_t)(g() % 256);
    std::vector<int32_t> w(3 * 4 * 9);
    for (auto& v : w) v = (int32_t)(g() % 256) - 128;
    ensei_b200::PartyResult res = ensei_b200::run_inproc_layer(ctx, d, im, imgs, w, 11);
    for (uint32_t i = 0; i < imgs; ++i) {
      std::vector<ensei::Mat> image(4, ensei::Mat(16, 16));
      for (int c = 0; c < 4; ++c)
        for (int k = 0; k < 256; ++k) image[c].data[k] = im[(i * 4 + c) * 256 + k];
      for (int o = 0; o < 3; ++o) {
        std::vector<uint64_t> acc(256, 0);
        for (int c = 0; c < 4; ++c) {
          ensei::Mat filt(3, 3);
          for (int k = 0; k < 9; ++k) filt.data[k] = w[(o * 4 + c) * 9 + k];
          const ensei::FieldSpec fp = ensei::FieldSpec::make(p);
          std::vector<ensei::Residue> r =
              ensei::conv_oracle(image[c], filt, ensei::make_geometry(16, 16, 3, 3, ensei::ConvType::Same, fp), fp);
          for (int k = 0; k < 256; ++k) acc[k] = (acc[k] + r[k]) % p;
        }
        for (int k = 0; k < 256; ++k)
          EXPECT(res.output[(i * 3 + o) * 256 + k] == acc[k], "run_inproc_layer output vs REF conv_oracle");
      }
    }
    EXPECT(res.timings.online_seconds > 0 && res.timings.encrypt_seconds > 0 && res.timings.filter_seconds > 0 &&
               res.timings.decrypt_seconds > 0 && res.timings.setup_seconds > 0,
           "PhaseTimings filled");
    EXPECT(res.online_counters.hadamard == (uint64_t)imgs * 1 * 4 * 3, "layer counters");
  }
  if (fails) return 1;
  std::printf("cpp mirror ok\n");
  return 0;
}
