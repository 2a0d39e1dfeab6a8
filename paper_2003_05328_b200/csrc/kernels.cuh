// kernels.cuh -- device helpers shared by the kernel files + host launcher prototypes.
#pragma once
#include "common.cuh"

namespace ensei_gpu {

// Row / column views of a padded u32 tile in shared memory.
struct TileRow {
  uint32_t* s;
  int base;
  EG_DEV uint32_t operator()(int i) const { return s[base + i]; }
  EG_DEV void operator()(int i, uint32_t v) const { s[base + i] = v; }
};
struct TileCol {
  uint32_t* s;
  int base, stride;
  EG_DEV uint32_t operator()(int i) const { return s[base + i * stride]; }
  EG_DEV void operator()(int i, uint32_t v) const { s[base + i * stride] = v; }
};
template <class Inner>
struct ReduceOnStore {  // canonical reduction of lazy forward outputs on store
  Inner in;
  Field32 f;
  uint32_t cred;
  EG_DEV uint32_t operator()(int i) const { return in(i); }
  EG_DEV void operator()(int i, uint32_t v) const { in(i, reduce_lazy(f, v, cred)); }
};

template <bool INV, int LOGL, int LOGE, int I, class View>
EG_DEV void tile_lines_pass(const Field32& f, const TwPair<uint32_t>* tw, View make_view, int lines) {
  constexpr int NT = (1 << LOGL) >> LOGE;
  const CtaBar bar;
  for (int it = threadIdx.x; it < lines * NT; it += blockDim.x) {
    auto v = make_view(it / NT);
    run_pass<Field32, uint32_t, LOGL, LOGE, I, INV, 0, false>(f, tw, it % NT, v, v, bar);
  }
}

template <bool INV, int LOGL, int LOGE, int I, class MakeView>
EG_DEV void tile_lines_all(const Field32& f, const TwPair<uint32_t>* tw, MakeView mk, int lines) {
  using Plan = PassPlan<LOGL, LOGE>;
  if constexpr (I < Plan::npass) {
    constexpr int PI = INV ? Plan::npass - 1 - I : I;
    tile_lines_pass<INV, LOGL, LOGE, PI>(f, tw, mk, lines);
    __syncthreads();
    tile_lines_all<INV, LOGL, LOGE, I + 1>(f, tw, mk, lines);
  }
}

// In-place 2D transform of an Lh x Lw tile (row stride LS) over p.
//   forward: CT rows then columns; natural order in -> bit-reversed x bit-reversed
//            out, canonical residues (REF ntt_2d computes rows then columns too).
//   inverse: GS rows then columns; bit-reversed x bit-reversed in -> natural out.
// Ends with __syncthreads().  twc: cyclic tables, length-L table at twc + L.
template <bool INV, int LOGH, int LOGW>
EG_DEV void tile_transform_2d(const Field32& f, uint32_t cred, const TwPair<uint32_t>* twc,
                              uint32_t* S, int LS) {
  constexpr int Lh = 1 << LOGH, Lw = 1 << LOGW;
  constexpr int EW = LOGW < 3 ? LOGW : 3, EH = LOGH < 3 ? LOGH : 3;
  if constexpr (LOGW > 0) {
    auto rows = [=](int r) { return TileRow{S, r * LS}; };
    tile_lines_all<INV, LOGW, EW, 0>(f, twc + Lw, rows, Lh);
  }
  if constexpr (LOGH > 0) {
    if constexpr (!INV) {
      auto cols = [=](int c) { return ReduceOnStore<TileCol>{TileCol{S, c, LS}, f, cred}; };
      tile_lines_all<INV, LOGH, EH, 0>(f, twc + Lh, cols, Lw);
    } else {
      auto cols = [=](int c) { return TileCol{S, c, LS}; };
      tile_lines_all<INV, LOGH, EH, 0>(f, twc + Lh, cols, Lw);
    }
  }
  // canonical outputs: forward columns reduce on store above; inverse values are
  // in [0, 2p) -> one conditional subtraction
  if constexpr (INV) {
    for (int i = threadIdx.x; i < Lh * Lw; i += blockDim.x) {
      int r = i >> LOGW, c = i & (Lw - 1);
      S[r * LS + c] = f.reduce_once(S[r * LS + c]);
    }
    __syncthreads();
  } else if constexpr (LOGH == 0) {
    for (int i = threadIdx.x; i < Lw; i += blockDim.x) S[i] = reduce_lazy(f, S[i], cred);
    __syncthreads();
  }
}

// Global store of lazy transform outputs with the canonical reduction applied.
template <int MODE, bool FWD>
struct GlobalOut64 {
  uint64_t* g;
  Field64 f;
  uint32_t cred;
  static constexpr bool kVec = true;
  EG_DEV uint64_t fin(uint64_t v) const {
    return FWD ? Bfly<Field64, MODE>::fin_ct(f, v, cred) : Bfly<Field64, MODE>::fin_gs(f, v);
  }
  EG_DEV void operator()(int i, uint64_t v) const { g[i] = fin(v); }
  EG_DEV void st2(int i, uint64_t a, uint64_t b) const {
    *reinterpret_cast<ulonglong2*>(g + i) = make_ulonglong2(fin(a), fin(b));
  }
};
using GlobalOut64Fwd = GlobalOut64<0, true>;

// host launchers (ntt_kernels.cu)
void negacyclic(const ensei_gpu_ctx* ctx, uint32_t modulus, bool inverse, bool natural, uint64_t* d,
                size_t count, cudaStream_t st);
void permute(const ensei_gpu_ctx* ctx, uint64_t* d, size_t count, cudaStream_t st);
void ntt2d(const ensei_gpu_ctx* ctx, bool inv, int logh, int logw, uint64_t* d, size_t count, cudaStream_t st);

}  // namespace ensei_gpu
