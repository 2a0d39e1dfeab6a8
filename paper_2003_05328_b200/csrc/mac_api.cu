// mac_api.cu -- ElementMult + channel accumulation dispatch (REF mul_plain / add_ct,
// ringbfv.cpp:233-306, channel sum protocol.cpp:570-581): the IMAD tile kernels
// (layer.cuh), the int8 tensor-core kernels (mac_i8.cuh) and the choice between them.
// Its own translation unit: the kernel instantiations dominate compile time.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "layer_launch.cuh"
#include "mac_i8.cuh"
#include "mac_tc.cuh"

namespace ensei_gpu {

template <int R, int S, int MT, int NT, int KT, int TM, int TN>
void mac_go(const LayerRun& r, const uint64_t* ct, const uint64_t* w, uint64_t* out) {
  ProfScope ps("mac_imad4", r.st);
  const int n = (int)r.ctx->n, rows = 2 * r.a.num_images, cols = r.a.cout;
  auto k = mac_kernel<R, S, MT, NT, KT, TM, TN>;
  constexpr size_t smem = mac_smem<S, MT, NT, KT>();
  set_smem(k, smem);
  dim3 grid((unsigned)(r.a.B * R * n / S), (unsigned)((rows + MT - 1) / MT), (unsigned)((cols + NT - 1) / NT));
  launch_pdl(k, grid, S * (MT / TM) * (NT / TN), smem, r.st, r.a, (int)r.ctx->logn, ct, w, 1, out);
  check_launch("mac_kernel");
}

template <int R, int S, int MT, int NT, int KT, int TM, int TN, int STAGES>
void mac_kara_go(const LayerRun& r, const uint64_t* ct, const uint64_t* w, uint64_t* out) {
  ProfScope ps("mac_kara", r.st);
  const int n = (int)r.ctx->n, rows = 2 * r.a.num_images, cols = r.a.cout;
  auto k = mac_kara_kernel<R, S, MT, NT, KT, TM, TN, STAGES>;
  constexpr size_t smem = mac_kara_smem<S, MT, NT, KT, STAGES>();
  set_smem(k, smem);
  const long tiles = (long)(r.a.B * R * n / S) * ((rows + MT - 1) / MT) * ((cols + NT - 1) / NT);
  static int per_sm = -1;  // per instantiation; the launch config never changes
  if (per_sm < 0) EG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, S * (MT / TM) * (NT / TN), smem));
  const long grid = std::min<long>(tiles, (long)std::max(per_sm, 1) * r.ctx->sm_count);
  launch_pdl(k, (unsigned)grid, S * (MT / TM) * (NT / TN), smem, r.st, r.a, (int)r.ctx->logn, ct, w, 1, out, 0u);
  check_launch("mac_kara_kernel");
}

// ElementMult implementation: -1 automatic (default), 0 the 4-product IMAD kernel, 1 the
// Karatsuba IMAD kernel, 2 the int8 tensor-core kernel (mac_i8.cuh).  ENSEI_MAC_VARIANT
// or ensei_gpu_set_mac_variant() override the automatic choice.
static std::atomic<int> g_mac_variant{-2};
void set_mac_variant(int v) { g_mac_variant.store(v, std::memory_order_relaxed); }
static int mac_variant() {
  int v = g_mac_variant.load(std::memory_order_relaxed);
  if (v == -2) {
    const char* e = getenv("ENSEI_MAC_VARIANT");
    v = e ? atoi(e) : -1;
    g_mac_variant.store(v, std::memory_order_relaxed);
  }
  return v;
}

// Context scratch for the workspace-less entry points (bob_mac / bob_eval): grown on
// demand, never under stream capture (nullptr then: the caller falls back), and every
// growth drops the cached host-entry graph.
void* ctx_scratch(const LayerRun& r, size_t need) {
  ensei_gpu_ctx* ctx = const_cast<ensei_gpu_ctx*>(r.ctx);
  if (need > ctx->i8_scratch_cap) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    EG_CUDA(cudaStreamIsCapturing(r.st, &cs));
    if (cs != cudaStreamCaptureStatusNone) return nullptr;
    EG_CUDA(cudaStreamSynchronize(r.st));  // the old buffer may still be read by queued work
    if (ctx->host_graph) {
      cudaGraphExecDestroy(ctx->host_graph);
      ctx->host_graph = nullptr;
      ctx->host_graph_key.clear();
    }
    if (ctx->i8_scratch) EG_CUDA(cudaFree(ctx->i8_scratch));
    ctx->i8_scratch = nullptr;
    ctx->i8_scratch_cap = 0;
    EG_CUDA(cudaMalloc(&ctx->i8_scratch, need));
    ctx->i8_scratch_cap = need;
  }
  return ctx->i8_scratch;
}

// The int8 tensor-core path (mac_i8p_kernel): forced by variant 2, chosen automatically
// for GEMM-sized slots (>= one 32-channel chunk, >= two 16-row tiles; measured: config 3
// +14 %, config 4 +8 %), and only while its exact-sum bound K (q_i - 1)^2 < 2^128 holds
// (ctx->i8_kmax); the IMAD kernels otherwise.
bool use_i8(const ensei_gpu_ctx* c, const LayerArgs& a) {
  const int var = mac_variant();
  return var == 2 && a.cin <= (int)c->i8_kmax;
}

// Prepared weights carry tcgen05 byte planes (after the packed words) exactly when the
// layer can take the tcgen05 ElementMult: 32 <= cin <= ctx->i8_kmax.
bool has_w_planes(const ensei_gpu_ctx* c, int cin) { return cin >= 32 && cin <= (int)c->i8_kmax; }
size_t w_words(const ensei_gpu_ctx* c, const LayerArgs& a) { return (size_t)a.cout * a.cin * a.B * c->R * c->n; }
// Which operand fills the MMA's 128-row side.  The tensor-core kernel multiplies a 128-row
// tile by 16-row tiles; padding goes to the 128-row side.  With the ciphertext rows there,
// a batch pays for whole blocks of 64 ciphertexts (config 4's 1024 images = 410 rows cost 512;
// config 3's packed layers 44, 12 and 4 rows cost 128 each); when the out channels fill
// 128-row blocks (almost) exactly they take that side instead and the ciphertext rows only
// pad to 16.  Decided from cout alone (the weight planes are laid out at prepare time).
bool tc_swap(const LayerArgs& a) {
  const int padded = (a.cout + kTcRowsA - 1) / kTcRowsA * kTcRowsA;
  return (padded - a.cout) * 8 <= a.cout;
}
size_t w_planes_bytes(const ensei_gpu_ctx* c, const LayerArgs& a) {
  if (!has_w_planes(c, a.cin)) return 0;
  const int T = tc_swap(a) ? kTcRowsA : kTcColsB;
  return tc_planes_bytes(a.B * (int)c->R * (int)c->n, (a.cout + T - 1) / T, T, a.cin);
}

// The tcgen05 ElementMult (mac_tc.cuh): chosen automatically for >= one 32-channel chunk and
// >= one 16-column tile within the exact-sum bound K (q_i - 1)^2 < 2^128 (ctx->i8_kmax);
// forced by variant 5.  A mostly empty 128-row tile still beats the IMAD kernels at these
// channel counts (config 3 on its packed grids: 44, 12 and 4 rows per layer -- 10.2k ->
// 12.4k images/s with the tensor-core path on every cin >= 32 layer), so there is no row
// threshold beyond a ciphertext pair.
bool use_tc(const ensei_gpu_ctx* c, const LayerArgs& a) {
  const int var = mac_variant(), rows = 2 * a.num_images;
  if (!has_w_planes(c, a.cin)) return false;
  return var == 5 || (var == -1 && rows >= 4 && a.cout >= kTcColsB);
}

// Tile choice (measured on B200, configs 1/3/4; cout <= 2 and cin <= 4 use mac_direct_kernel): 8-slot x 32-row x 16-col tiles with 36-channel
// chunks and 2 stages for the large shapes; 8 x 16 x 16 with 12-channel chunks, 3 stages when
// rows and cols fit 16.  Alternatives measured slower: 4 outputs per thread (no register-pair
// moves but one more shared load per MAC), 12-channel chunks with 3 stages, 4-slot tiles.
// ENSEI_MAC_VARIANT=0 forces the 4-product kernel (A/B); it is also the fallback for primes
// outside the Karatsuba headroom (kara_ok).
template <int R>
void mac_direct_go(const LayerRun& r, const uint64_t* ct, const uint64_t* w, uint64_t* out) {
  ProfScope ps("mac_direct", r.st);
  const size_t total = (size_t)r.a.num_images * r.a.B * R * r.ctx->n;
  const long grid = std::min<long>((long)((total + 255) / 256), (long)r.ctx->sm_count * 8);
  launch_pdl(mac_direct_kernel<R>, (unsigned)grid, 256, 0, r.st, r.a, (int)r.ctx->logn, ct, w, 1, out);
  check_launch("mac_direct_kernel");
}

template <int R>
void mac_i8_go(const LayerRun& r, const uint64_t* ct, const uint64_t* w, uint64_t* out) {
  ProfScope ps("mac_i8", r.st);
  const int n = (int)r.ctx->n, rows = 2 * r.a.num_images, cols = r.a.cout;
  const long tasks = (long)(r.a.B * R * n / kI8Slots) * ((rows + kI8Rows - 1) / kI8Rows) *
                     ((cols + kI8Cols - 1) / kI8Cols);
  auto k = mac_i8_kernel<R>;
  static int per_sm = -1;
  if (per_sm < 0) EG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 256, 0));
  const long grid = std::min<long>(tasks, (long)std::max(per_sm, 1) * r.ctx->sm_count);
  launch_pdl(k, (unsigned)grid, 256, 0, r.st, r.a, (int)r.ctx->logn, ct, w, 1, out);
  check_launch("mac_i8_kernel");
}

// Byte-plane scratch of the int8 tensor-core MAC (bytes; 0 when the IMAD kernels run).
// tcgen05 scratch: the ciphertext byte planes, then the slot-major product Y
size_t tc_a_bytes(const ensei_gpu_ctx* c, const LayerArgs& a) {  // the ciphertext planes
  const int T = tc_swap(a) ? kTcColsB : kTcRowsA;
  return tc_planes_bytes(a.B * (int)c->R * (int)c->n, (2 * a.num_images + T - 1) / T, T, a.cin);
}
size_t tc_y_bytes(const ensei_gpu_ctx* c, const LayerArgs& a) {
  const int big = tc_swap(a) ? a.cout : 2 * a.num_images, small = tc_swap(a) ? 2 * a.num_images : a.cout;
  return (size_t)a.B * c->R * c->n * ((big + kTcRowsA - 1) / kTcRowsA) * kTcRowsA *
         ((small + kTcColsB - 1) / kTcColsB) * kTcColsB * sizeof(uint64_t);
}

size_t mac_scratch_bytes(const ensei_gpu_ctx* c, const LayerArgs& a) {
  if (use_tc(c, a)) return tc_a_bytes(c, a) + tc_y_bytes(c, a);
  if (!use_i8(c, a)) return 0;
  const int n = (int)c->n, rows = 2 * a.num_images, K = a.cin;
  return (size_t)(i8_plane_words(a.B, (int)c->R, n, K, rows) + i8_plane_words(a.B, (int)c->R, n, K, a.cout)) *
         sizeof(uint32_t);
}

// Byte planes + cp.async pipeline (mac_i8p_kernel).  The planes live in `scratch`
// (the caller's workspace: ensei_gpu_conv_workspace_bytes counts them) or, for the
// workspace-less entry points (bob_mac / bob_eval), in a context buffer grown on
// demand -- never under stream capture (false: the caller falls back to the IMAD
// kernels), and every growth drops the cached host-entry graph.
template <int R>
bool mac_i8p_go(const LayerRun& r, const uint64_t* ct, const uint64_t* w, uint64_t* out, void* scratch) {
  ensei_gpu_ctx* ctx = const_cast<ensei_gpu_ctx*>(r.ctx);
  const int n = (int)ctx->n, rows = 2 * r.a.num_images, cols = r.a.cout, K = r.a.cin;
  const size_t aw = (size_t)i8_plane_words(r.a.B, R, n, K, rows), bw = (size_t)i8_plane_words(r.a.B, R, n, K, cols);
  const size_t need = (aw + bw) * sizeof(uint32_t);
  if (!scratch) scratch = ctx_scratch(r, need);
  if (!scratch) return false;
  uint32_t* Ap = static_cast<uint32_t*>(scratch);
  uint32_t* Bp = Ap + aw;
  const unsigned pg = (unsigned)ctx->sm_count * 8;
  {
    ProfScope ps("planes_ct", r.st);
    planes_kernel<R, false><<<pg, 256, 0, r.st>>>(r.a, (int)ctx->logn, ct, Ap, rows);
    check_launch("planes_kernel");
  }
  {
    ProfScope ps("planes_w", r.st);
    planes_kernel<R, true><<<pg, 256, 0, r.st>>>(r.a, (int)ctx->logn, w, Bp, cols);
    check_launch("planes_kernel");
  }
  constexpr int STAGES = 4;
  constexpr size_t smem = (size_t)STAGES * 2 * 8 * kI8T * 8 * sizeof(uint32_t);
  auto k = mac_i8p_kernel<R, STAGES>;
  set_smem(k, smem);
  static int per_sm = -1;
  if (per_sm < 0) EG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 256, smem));
  const long tasks = (long)r.a.B * R * (n / 4) * ((rows + kI8T - 1) / kI8T) * ((cols + kI8T - 1) / kI8T);
  const long grid = std::min<long>(tasks, (long)std::max(per_sm, 1) * ctx->sm_count);
  ProfScope ps("mac_i8p", r.st);
  k<<<(unsigned)grid, 256, smem, r.st>>>(r.a, (int)ctx->logn, Ap, Bp, 1, out);
  check_launch("mac_i8p_kernel");
  return true;
}

// tcgen05 ElementMult: ciphertext byte planes (planes_tc_kernel, into the workspace or the
// context scratch), then one mac_tc_kernel pass per 32*NK-channel chunk.  The weight
// planes follow the packed words of the prepared weights (ensei_gpu_prepare_weights).
template <int R, int NK>
void mac_tc_launch(const LayerRun& r, const uint8_t* Ap, const uint8_t* Bp, uint64_t* Y, int rows, int cols) {
  auto k = mac_tc_kernel<NK, R>;
  constexpr size_t smem = tc_smem_bytes<NK>();
  set_smem(k, smem);
  const int nkc = tc_nkc(r.a.cin);
  for (int kc = 0; kc < nkc; ++kc) {
    ProfScope ps("mac_tc", r.st);
    launch_pdl(k, (unsigned)(r.ctx->sm_count & ~1), kTcThreads, smem, r.st, r.a, (int)r.ctx->logn, Ap, Bp, kc,
               Y, rows, cols);  // CTA pairs: an even grid
    check_launch("mac_tc_kernel");
  }
}

template <int R>
bool mac_tc_go(const LayerRun& r, const uint64_t* ct, const uint64_t* w, uint64_t* out, void* scratch) {
  const size_t need = mac_scratch_bytes(r.ctx, r.a);
  uint8_t* Ap = static_cast<uint8_t*>(scratch ? scratch : ctx_scratch(r, need));
  if (!Ap) return false;
  uint64_t* Y = reinterpret_cast<uint64_t*>(Ap + tc_a_bytes(r.ctx, r.a));
  const uint8_t* Wp = reinterpret_cast<const uint8_t*>(w + w_words(r.ctx, r.a));
  const bool swap = tc_swap(r.a);
  const int rows = 2 * r.a.num_images, cols = r.a.cout;
  {
    ProfScope ps("planes_tc", r.st);
    if (swap)
      launch_pdl(planes_tc_kernel<kTcColsB, false>, (unsigned)r.ctx->sm_count * 8, 256, 0, r.st, r.a,
                 (int)r.ctx->logn, R, ct, Ap, rows);
    else
      launch_pdl(planes_tc_kernel<kTcRowsA, false>, (unsigned)r.ctx->sm_count * 8, 256, 0, r.st, r.a,
                 (int)r.ctx->logn, R, ct, Ap, rows);
    check_launch("planes_tc_kernel");
  }
  // the 128-row operand first: the weights when swapped (out channels x ciphertext rows)
  const uint8_t* A = swap ? Wp : Ap;
  const uint8_t* B = swap ? Ap : Wp;
  if (tc_nk(r.a.cin) == 2) mac_tc_launch<R, 2>(r, A, B, Y, swap ? cols : rows, swap ? rows : cols);
  else mac_tc_launch<R, 1>(r, A, B, Y, swap ? cols : rows, swap ? rows : cols);
  {
    ProfScope ps("mac_out", r.st);
    if (swap)
      launch_pdl(mac_out_kernel<R, true>, (unsigned)r.ctx->sm_count * 8, 256, 0, r.st, r.a, (int)r.ctx->logn,
                 (const uint64_t*)Y, 1, out);
    else
      launch_pdl(mac_out_kernel<R, false>, (unsigned)r.ctx->sm_count * 8, 256, 0, r.st, r.a, (int)r.ctx->logn,
                 (const uint64_t*)Y, 1, out);
    check_launch("mac_out_kernel");
  }
  return true;
}

// Which ElementMult kernel a launch takes (ENSEI_MAC_* in include/ensei_gpu.h).
int mac_path(const ensei_gpu_ctx* c, const LayerArgs& a) {
  const int var = mac_variant();
  if (var == 3 && a.cin <= (int)c->i8_kmax) return ENSEI_MAC_I8_DIRECT;
  if (use_tc(c, a)) return ENSEI_MAC_TCGEN05;
  if (use_i8(c, a)) return ENSEI_MAC_I8_PLANES;
  // tiny channel counts (config 0: 1 -> 1): direct per-slot kernel (exact while cin <= 1008)
  if (a.cout <= 2 && a.cin <= 4) return ENSEI_MAC_DIRECT;
  if (!c->kara_ok || var == 0) return ENSEI_MAC_IMAD4;
  return ENSEI_MAC_KARATSUBA;
}

template <int R>
void mac_r(const LayerRun& r, const uint64_t* ct, const uint64_t* w, uint64_t* out, void* scratch) {
  const int rows = 2 * r.a.num_images, cols = r.a.cout;
  const bool small = rows <= 16 && cols <= 16;
  int path = mac_path(r.ctx, r.a);
  if (path == ENSEI_MAC_I8_DIRECT) return mac_i8_go<R>(r, ct, w, out);
  if (path == ENSEI_MAC_TCGEN05) {
    if (mac_tc_go<R>(r, ct, w, out, scratch)) return;
    path = r.ctx->kara_ok ? ENSEI_MAC_KARATSUBA : ENSEI_MAC_IMAD4;  // no scratch under capture
  }
  if (path == ENSEI_MAC_I8_PLANES) {
    if (mac_i8p_go<R>(r, ct, w, out, scratch)) return;
    path = r.ctx->kara_ok ? ENSEI_MAC_KARATSUBA : ENSEI_MAC_IMAD4;  // no scratch under capture
  }
  if (path == ENSEI_MAC_DIRECT) return mac_direct_go<R>(r, ct, w, out);
  if (path == ENSEI_MAC_IMAD4) {
    if (small) return mac_go<R, 16, 16, 16, 16, 2, 4>(r, ct, w, out);
    return mac_go<R, 8, 32, 32, 16, 4, 4>(r, ct, w, out);
  }
  if (small) return mac_kara_go<R, 8, 16, 16, 12, 2, 4, 3>(r, ct, w, out);
  // few input channels (config 3's 3 -> 64 layer): the 36-channel chunks of the large tile
  // would be ~90 % zero fill and its 221 KB ring allows one CTA per SM (config 3 +0.3 %)
  if (r.a.cin <= 12) return mac_kara_go<R, 8, 16, 16, 12, 2, 4, 3>(r, ct, w, out);
  return mac_kara_go<R, 8, 32, 16, 36, 2, 4, 2>(r, ct, w, out);
}

void mac(const LayerRun& r, const uint64_t* ct, const uint64_t* w, uint64_t* out, void* scratch) {
  if (r.a.num_images == 0) return;
  if (r.R == 1) return mac_r<1>(r, ct, w, out, scratch);
  if (r.R == 3) return mac_r<3>(r, ct, w, out, scratch);
  fail(ENSEI_ERR_UNSUPPORTED, "ElementMult: unsupported prime count");
}

// The tcgen05 weight planes of a prepared-weights buffer (after its packed words), built
// from those words; no-op for layers that cannot take the tcgen05 path.
void build_w_planes(const LayerRun& r, uint64_t* w_eval) {
  if (!has_w_planes(r.ctx, r.a.cin)) return;
  ProfScope ps("planes_w_tc", r.st);
  uint8_t* wp = reinterpret_cast<uint8_t*>(w_eval + w_words(r.ctx, r.a));
  if (tc_swap(r.a))
    planes_tc_kernel<kTcRowsA, true><<<(unsigned)r.ctx->sm_count * 8, 256, 0, r.st>>>(
        r.a, (int)r.ctx->logn, (int)r.ctx->R, w_eval, wp, r.a.cout);
  else
    planes_tc_kernel<kTcColsB, true><<<(unsigned)r.ctx->sm_count * 8, 256, 0, r.st>>>(
        r.a, (int)r.ctx->logn, (int)r.ctx->R, w_eval, wp, r.a.cout);
  check_launch("planes_tc_kernel");
}
size_t prepared_weights_bytes(const ensei_gpu_ctx* c, const LayerArgs& a) {
  return w_words(c, a) * sizeof(uint64_t) + w_planes_bytes(c, a);
}

}  // namespace ensei_gpu
