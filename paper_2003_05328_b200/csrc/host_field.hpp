// host_field.hpp -- host-side prime-field setup for the device tables.
//
// Roots must be the reference's CANONICAL ones so device transforms are
// bit-identical to REF: generator = smallest primitive root (REF modfield.cpp:
// 143-152), omega_L = g^((p-1)/L) (REF modfield.cpp:167-171), psi = g^((q-1)/2n)
// (REF ringbfv.cpp:35).  Primality: deterministic Miller-Rabin; factoring of p-1:
// trial division + Pollard rho.
#pragma once
#include <cstdint>
#include <stdexcept>
#include <vector>

namespace ensei_gpu {
namespace host {

using u64 = uint64_t;
using u128 = unsigned __int128;

inline u64 mulmod(u64 a, u64 b, u64 m) { return (u64)((u128)a * b % m); }
inline u64 powmod(u64 b, u64 e, u64 m) {
  u64 r = 1 % m;
  b %= m;
  while (e) {
    if (e & 1) r = mulmod(r, b, m);
    b = mulmod(b, b, m);
    e >>= 1;
  }
  return r;
}
inline u64 invmod(u64 a, u64 m) { return powmod(a, m - 2, m); }

inline bool is_prime(u64 n) {
  static const u64 bases[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  if (n < 2) return false;
  for (u64 b : bases)
    if (n % b == 0) return n == b;
  u64 d = n - 1;
  int r = 0;
  while (!(d & 1)) { d >>= 1; ++r; }
  for (u64 a : bases) {
    u64 x = powmod(a, d, n);
    if (x == 1 || x == n - 1) continue;
    bool comp = true;
    for (int i = 1; i < r && comp; ++i) {
      x = mulmod(x, x, n);
      if (x == n - 1) comp = false;
    }
    if (comp) return false;
  }
  return true;
}

inline u64 gcd(u64 a, u64 b) {
  while (b) { u64 t = a % b; a = b; b = t; }
  return a;
}

inline void factor(u64 n, std::vector<u64>& out) {
  auto push = [&](u64 f) {
    for (u64 g : out) if (g == f) return;
    out.push_back(f);
  };
  if (n == 1) return;
  if (is_prime(n)) { push(n); return; }
  for (u64 p = 2; p < 100000 && p * p <= n; ++p)
    if (n % p == 0) {
      push(p);
      while (n % p == 0) n /= p;
      factor(n, out);
      return;
    }
  u64 d = 0;
  for (u64 c = 1; !d; ++c) {  // Pollard rho (Floyd)
    u64 x = 2, y = 2, g = 1;
    while (g == 1) {
      x = (u64)(((u128)x * x + c) % n);
      y = (u64)(((u128)y * y + c) % n);
      y = (u64)(((u128)y * y + c) % n);
      g = gcd(x > y ? x - y : y - x, n);
    }
    d = g == n ? 0 : g;
  }
  factor(d, out);
  while (n % d == 0) n /= d;
  factor(n, out);
}

inline u64 primitive_root(u64 p) {
  if (p == 2) return 1;
  std::vector<u64> f;
  factor(p - 1, f);
  for (u64 g = 2; g < p; ++g) {
    bool ok = true;
    for (u64 r : f)
      if (powmod(g, (p - 1) / r, p) == 1) { ok = false; break; }
    if (ok) return g;
  }
  throw std::runtime_error("no primitive root");
}

inline u64 root_of_unity(u64 order, u64 p) {
  if (order == 0 || (p - 1) % order) throw std::invalid_argument("root order does not divide p-1");
  return powmod(primitive_root(p), (p - 1) / order, p);
}

inline int ilog2(u64 n) {
  int l = 0;
  while ((1ull << l) < n) ++l;
  return l;
}
inline u64 bitrev(u64 x, int bits) {
  u64 r = 0;
  for (int i = 0; i < bits; ++i) r |= ((x >> i) & 1) << (bits - 1 - i);
  return r;
}

// Shoup companion for a constant w: floor(w * 2^B / m), B = 64 or 32
inline u64 shoup64(u64 w, u64 m) { return (u64)(((u128)w << 64) / m); }
inline u64 shoup32(u64 w, u64 m) { return (u64)(((u128)w << 32) / m); }

// Twiddle values (no companions) for the device transform conventions of
// ntt_core.cuh.  negacyclic: fwd[k] = psi^brv(k), inv[k] = psi^-brv(k);
// cyclic: fwd[m+i] = omega^((N/2m) brv_{log m}(i)).  inv[1] pre-scaled by N^-1,
// inv[0] = N^-1.
struct TwiddleValues {
  std::vector<u64> fwd, inv;
};

inline TwiddleValues make_twiddles(u64 m, u64 N, bool negacyclic) {
  TwiddleValues t;
  t.fwd.assign(N, 0);
  t.inv.assign(N, 0);
  int lg = ilog2(N);
  u64 ninv = invmod(N % m, m);
  if (negacyclic) {
    u64 psi = root_of_unity(2 * N, m), psii = invmod(psi, m);
    for (u64 k = 0; k < N; ++k) {
      u64 e = bitrev(k, lg);
      t.fwd[k] = powmod(psi, e, m);
      t.inv[k] = powmod(psii, e, m);
    }
  } else {
    u64 w = root_of_unity(N, m), wi = invmod(w, m);
    for (u64 mm = 1; mm < N; mm <<= 1) {
      int lm = ilog2(mm);
      for (u64 i = 0; i < mm; ++i) {
        u64 e = (N / (2 * mm)) * bitrev(i, lm);
        t.fwd[mm + i] = powmod(w, e, m);
        t.inv[mm + i] = powmod(wi, e, m);
      }
    }
  }
  t.inv[1] = mulmod(t.inv[1], ninv, m);
  t.inv[0] = ninv;
  t.fwd[0] = 1;
  return t;
}

}  // namespace host
}  // namespace ensei_gpu
