// tools/cpp_mirror_check.cpp -- the C++ host mirror used the way a REF maintainer
// would: REF's NegacyclicPlan / ntt_2d next to ensei_b200's, same inputs, compare.
// Built and run by tests/test_gpu_cpp_mirror.py (links oracle/_ref for REF).
#include <cstdio>
#include <random>

#include "../paper_2003_05328_b200/csrc/host/ensei_b200.hpp"
#include "ensei/modfield.hpp"
#include "ensei/ntt.hpp"
#include "ensei/ringbfv.hpp"

int main() {
  const uint64_t q = 576460803525083137ULL, p = 638977;
  const uint32_t n = 2048;
  std::mt19937_64 g(7);
  std::vector<uint64_t> x(4 * n);
  for (auto& v : x) v = g() % q;
  // REF
  ensei::NegacyclicPlan plan = ensei::NegacyclicPlan::make(ensei::FieldSpec::make(q), n);
  std::vector<uint64_t> want = x;
  for (int i = 0; i < 4; ++i) {
    std::vector<ensei::Residue> poly(want.begin() + i * n, want.begin() + (i + 1) * n);
    plan.forward(poly);
    std::copy(poly.begin(), poly.end(), want.begin() + i * n);
  }
  // B200
  ensei_b200::Context ctx(n, {q}, p);
  std::vector<uint64_t> got = x;
  ctx.negacyclic_forward(got);
  if (got != want) { std::printf("negacyclic mismatch\n"); return 1; }
  ctx.negacyclic_inverse(got);
  if (got != x) { std::printf("roundtrip mismatch\n"); return 1; }
  // 2D
  std::vector<uint64_t> tile(64 * 64);
  for (auto& v : tile) v = g() % p;
  ensei::FreqTensor t;
  t.rows = t.cols = 64;
  t.field = ensei::FieldSpec::make(p);
  t.data = tile;
  ensei::FreqTensor f = ensei::ntt_2d(t);
  ctx.ntt_2d(tile, 64, 64);
  if (tile != f.data) { std::printf("ntt_2d mismatch\n"); return 1; }
  try {
    ensei_b200::Context bad(n, {q + 2}, p);
    std::printf("expected an error\n");
    return 1;
  } catch (const ensei_b200::Error&) {
  }
  std::printf("cpp mirror ok\n");
  return 0;
}
