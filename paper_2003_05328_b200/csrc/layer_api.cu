// layer_api.cu -- C ABI of the conv-layer path (include/ensei_gpu.h): geometry,
// keys, weight preparation, Alice Enc, Bob eval, Alice Dec, recombination and the
// whole-layer / host-buffer entry points.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>

#include "host_field.hpp"
#include "layer_launch.cuh"

namespace ensei_gpu {

int run_guarded(void (*fn)(void*), void* arg);

template <int LOGN>
void launch_tile(const LayerRun&, int, bool, int, const uint64_t*, uint32_t, const void*, uint64_t*, int);
template <int LOGN>
void launch_share(const LayerRun&, bool, uint64_t*, uint32_t*, int);
template <int LOGN>
void launch_dec(const LayerRun&, const uint64_t*, uint32_t, const uint64_t*, uint32_t*, const uint32_t*, uint32_t*,
                int);
template <int LOGN>
void launch_secret(const LayerRun&, const int64_t*, int64_t*, uint64_t*, bool);

extern template void launch_tile<11>(const LayerRun&, int, bool, int, const uint64_t*, uint32_t, const void*,
                                     uint64_t*, int);
extern template void launch_tile<12>(const LayerRun&, int, bool, int, const uint64_t*, uint32_t, const void*,
                                     uint64_t*, int);
extern template void launch_tile<13>(const LayerRun&, int, bool, int, const uint64_t*, uint32_t, const void*,
                                     uint64_t*, int);
#define EG_EXTERN_LAYER(LOGN)                                                                                  \
  extern template void launch_share<LOGN>(const LayerRun&, bool, uint64_t*, uint32_t*, int);                  \
  extern template void launch_dec<LOGN>(const LayerRun&, const uint64_t*, uint32_t, const uint64_t*, uint32_t*, \
                                        const uint32_t*, uint32_t*, int);                                      \
  extern template void launch_secret<LOGN>(const LayerRun&, const int64_t*, int64_t*, uint64_t*, bool);
EG_EXTERN_LAYER(11)
EG_EXTERN_LAYER(12)
EG_EXTERN_LAYER(13)

// ElementMult dispatch (mac_api.cu)
void mac(const LayerRun& r, const uint64_t* ct, const uint64_t* w, uint64_t* out, void* scratch = nullptr);
int mac_path(const ensei_gpu_ctx* c, const LayerArgs& a);
size_t mac_scratch_bytes(const ensei_gpu_ctx* c, const LayerArgs& a);
void set_mac_variant(int v);
void build_w_planes(const LayerRun& r, uint64_t* w_eval);
size_t prepared_weights_bytes(const ensei_gpu_ctx* c, const LayerArgs& a);

namespace {

template <class Fn>
int guarded(Fn&& fn) {
  struct Box {
    Fn* f;
  } box{&fn};
  return run_guarded([](void* p) { (*static_cast<Box*>(p)->f)(); }, &box);
}

struct Geo {
  uint32_t Lh, Lw, logL, B, oh, ow, r0, c0, G;
  uint32_t pk = 1;  // images per ciphertext block
  uint32_t gridL = 0;  // grid override in force (a non-power-of-two side), else 0
  uint32_t cts(uint32_t imgs) const { return (imgs + pk - 1) / pk; }
};

int ilog2u(uint32_t v) {
  int l = 0;
  while ((1u << l) < v) ++l;
  return l;
}

// make_geometry (REF ntt.cpp:65-81) + blocks per channel (REF protocol.cpp:180)
Geo geometry(const ensei_gpu_ctx* c, const ensei_conv_desc* d) {
  require(c && d, ENSEI_ERR_INVALID_ARGUMENT, "null argument");
  require(d->H && d->W && d->fh && d->fw, ENSEI_ERR_BAD_GEOMETRY, "zero dimension");
  require(d->cin && d->cout, ENSEI_ERR_BAD_GEOMETRY, "conv layer needs channel counts");
  require(d->same || (d->fh <= d->H && d->fw <= d->W), ENSEI_ERR_BAD_GEOMETRY,
          "valid convolution needs filter <= image");
  auto padded = [&](uint32_t min_len) -> uint32_t {
    uint32_t p2 = 1;
    while (p2 < min_len) p2 <<= 1;
    if ((c->p - 1) % p2 == 0) return p2;
    fail(ENSEI_ERR_UNSUPPORTED, "non-power-of-two transform length (REF direct O(L^2) path) not on the GPU path");
  };
  Geo g;
  if (d->grid && (d->grid & (d->grid - 1))) {
    // grid override (builder extension): any side holding the linear convolution that
    // divides p - 1, as REF's own fallback lengths do (choose_padded_len, ntt.cpp:51-61)
    require(d->grid >= d->H + d->fh - 1 && d->grid >= d->W + d->fw - 1, ENSEI_ERR_BAD_GEOMETRY,
            "grid override smaller than the linear convolution");
    require((c->p - 1) % d->grid == 0, ENSEI_ERR_BAD_GEOMETRY, "grid override must divide p - 1");
    g.Lh = g.Lw = g.gridL = d->grid;
  } else {
    g.Lh = padded(d->grid ? std::max(d->grid, d->H + d->fh - 1) : d->H + d->fh - 1);
    g.Lw = padded(d->grid ? std::max(d->grid, d->W + d->fw - 1) : d->W + d->fw - 1);
  }
  require(g.Lh == g.Lw, ENSEI_ERR_UNSUPPORTED, "rectangular padded grids are not on the GPU path");
  require(g.Lh <= (uint32_t)kMaxTile && g.Lh >= 2, ENSEI_ERR_UNSUPPORTED, "padded grid side must be in [2, 64]");
  g.logL = ilog2u(g.Lh);
  g.G = g.Lh * g.Lw;
  g.B = (g.G + c->n - 1) / c->n;
  // packing (builder extension, ensei_conv_desc::pack): pk images' grids per block
  g.pk = d->pack > 1 ? d->pack : 1;
  if (g.pk > 1) {
    require(g.B == 1 && (uint64_t)g.pk * g.G <= c->n, ENSEI_ERR_BAD_GEOMETRY,
            "packing needs pack * padded grid <= n (one block per channel)");
    require(g.gridL || (g.pk & (g.pk - 1)) == 0, ENSEI_ERR_UNSUPPORTED,
            "pack must be a power of two (any pack with a grid override)");
  }
  g.oh = d->same ? d->H : d->H - d->fh + 1;
  g.ow = d->same ? d->W : d->W - d->fw + 1;
  g.r0 = d->same ? (d->fh - 1) / 2 : d->fh - 1;
  g.c0 = d->same ? (d->fw - 1) / 2 : d->fw - 1;
  return g;
}

// RNS tile kernel generation (ensei_gpu_set_tile_variant): 1 = layer_rns.cuh, 0 = layer.cuh
std::atomic<int> g_tile_gen{1};
std::atomic<int> g_no_fork{0};  // tuning: HomShare in line instead of forked onto the aux stream

LayerRun make_run(const ensei_gpu_ctx* c, const ensei_conv_desc* d, const Geo& g, uint32_t num_images,
                  const ensei_randomness* rand, void* stream) {
  require(c->approx_ok, ENSEI_ERR_UNSUPPORTED,
          "the fused layer kernels need 31 q_i < 2^64 for every prime (q_i < 2^59.04); larger primes run only through "
          "ensei_gpu_negacyclic");
  LayerRun r;
  r.ctx = c;
  r.logL = (int)g.logL;
  r.R = (int)c->R;
  r.st = (cudaStream_t)stream;
  r.tile_gen = g_tile_gen.load(std::memory_order_relaxed);
  r.gridL = (int)g.gridL;
  LayerArgs& a = r.a;
  std::memset(&a, 0, sizeof(a));
  a.H = d->H;
  a.W = d->W;
  a.fh = d->fh;
  a.fw = d->fw;
  a.cin = d->cin;
  a.cout = d->cout;
  a.Lh = g.Lh;
  a.Lw = g.Lw;
  a.B = g.B;
  a.oh = g.oh;
  a.ow = g.ow;
  a.r0 = g.r0;
  a.c0 = g.c0;
  a.G = g.G;
  a.num_images = num_images;
  a.pk = (int)g.pk;
  a.num_cts = (int)g.cts(num_images);
  for (uint32_t i = 0; i < c->R; ++i) {
    a.pc[i] = c->pc[i];
    a.psi_q[i] = c->psi_q[i];
    a.twq_fwd[i] = c->tab.tw_q_fwd[i];
    a.twq_inv[i] = c->tab.tw_q_inv[i];
  }
  a.crt = c->crt;
  a.dec_kbits = (int)c->dec_kbits;
  if (g.gridL) {
    const uint64_t w = host::root_of_unity(g.gridL, c->p);
    a.grid_w = (uint32_t)w;
    a.grid_winv = (uint32_t)host::invmod(w, c->p);
    a.grid_linv = (uint32_t)host::invmod(g.gridL % c->p, c->p);
    // lazy sums of at most 16 products of residues: z < 16 p^2 < 2^zb
    uint32_t bp = 0;
    while ((c->p >> bp) != 0) ++bp;
    const uint32_t zb = 2 * bp + 4;
    require(zb <= 62 && zb - bp + 1 < 32 + bp, ENSEI_ERR_UNSUPPORTED, "grid override: p too large for the tile transform");
    a.grid_s1 = bp - 1;
    a.grid_s2 = zb - bp + 1;
    a.grid_mu = (uint32_t)((((unsigned __int128)1) << zb) / c->p);
  }
  a.pp = c->pp;
  a.twp_fwd = c->tab.tw_p_fwd;
  a.twp_inv = c->tab.tw_p_inv;
  a.twc_fwd = c->tab.tw_c_fwd;
  a.twc_inv = c->tab.tw_c_inv;
  if (rand) {
    require(rand->mode == ENSEI_RAND_PHILOX || rand->mode == ENSEI_RAND_INJECTED, ENSEI_ERR_INVALID_ARGUMENT,
            "bad randomness mode");
    require(g.pk == 1 || (rand->mode == ENSEI_RAND_PHILOX && rand->image_base % g.pk == 0), ENSEI_ERR_UNSUPPORTED,
            "packed layers: Philox streams with a pack-aligned image_base");
    a.rand_mode = rand->mode;
    a.layer = rand->layer;
    a.image_base = rand->image_base;
    a.cbd_k = rand->cbd_k ? rand->cbd_k : 20;
    require(a.cbd_k <= 31, ENSEI_ERR_INVALID_ARGUMENT, "cbd_k must be <= 31");
    a.alice_key = rand->alice_key;
    a.bob_key = rand->bob_key;
    a.inj_noise = rand->d_noise;
    a.inj_ahat = rand->d_a_hat;
    a.inj_share = rand->d_share;
  }
  return r;
}

bool injected(const ensei_randomness* r) { return r && r->mode == ENSEI_RAND_INJECTED; }

// The ElementMult sees ciphertexts, not images: its rows are the ciphertext images
LayerRun mac_run(const LayerRun& r) {
  LayerRun m = r;
  m.a.num_images = r.a.num_cts;
  return m;
}

void tile(const LayerRun& r, int tm, bool inj, int in_t, const uint64_t* key, uint32_t ks, const void* in,
          uint64_t* out, int items) {
  ProfScope ps(tm == TILE_ENC ? "enc" : tm == TILE_HOMREC ? "homrec" : "weights", r.st);
  switch (r.ctx->logn) {
    case 11: return launch_tile<11>(r, tm, inj, in_t, key, ks, in, out, items);
    case 12: return launch_tile<12>(r, tm, inj, in_t, key, ks, in, out, items);
    case 13: return launch_tile<13>(r, tm, inj, in_t, key, ks, in, out, items);
  }
  fail(ENSEI_ERR_UNSUPPORTED, "ring degree must be 2048, 4096 or 8192 on this path");
}
void share(const LayerRun& r, bool inj, uint64_t* ct_out, uint32_t* bob_share, int items) {
  ProfScope ps("share", r.st);
  switch (r.ctx->logn) {
    case 11: return launch_share<11>(r, inj, ct_out, bob_share, items);
    case 12: return launch_share<12>(r, inj, ct_out, bob_share, items);
    case 13: return launch_share<13>(r, inj, ct_out, bob_share, items);
  }
  fail(ENSEI_ERR_UNSUPPORTED, "ring degree must be 2048, 4096 or 8192 on this path");
}
void dec(const LayerRun& r, const uint64_t* key, uint32_t ks, const uint64_t* ct, uint32_t* alice,
         const uint32_t* bob, uint32_t* out, int items) {
  ProfScope ps(r.R == 1 ? "dec" : "dec_rns", r.st);
  switch (r.ctx->logn) {
    case 11: return launch_dec<11>(r, key, ks, ct, alice, bob, out, items);
    case 12: return launch_dec<12>(r, key, ks, ct, alice, bob, out, items);
    case 13: return launch_dec<13>(r, key, ks, ct, alice, bob, out, items);
  }
  fail(ENSEI_ERR_UNSUPPORTED, "ring degree must be 2048, 4096 or 8192 on this path");
}
void secret(const LayerRun& r, const int64_t* t_in, int64_t* t_out, uint64_t* key, bool sample) {
  switch (r.ctx->logn) {
    case 11: return launch_secret<11>(r, t_in, t_out, key, sample);
    case 12: return launch_secret<12>(r, t_in, t_out, key, sample);
    case 13: return launch_secret<13>(r, t_in, t_out, key, sample);
  }
  fail(ENSEI_ERR_UNSUPPORTED, "ring degree must be 2048, 4096 or 8192 on this path");
}

__global__ void recombine_kernel(const uint32_t* a, const uint32_t* b, size_t count, uint32_t p, uint32_t* out) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t y = a[i] % p + b[i] % p;
    out[i] = y >= p ? y - p : y;
  }
}

__global__ void activation_kernel(const uint32_t* a, const uint32_t* b, int fn, int pool, int C, int H, int W,
                                  size_t total, uint32_t p, uint32_t layer, uint32_t image_base, uint64_t key,
                                  const uint32_t* inj, uint32_t* na, uint32_t* nb, int* overflow) {
  const int oh = pool ? H / 2 : H, ow = pool ? W / 2 : W;
  const int64_t half = p / 2;
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
    const int i = (int)(idx % ((size_t)oh * ow));
    const size_t ic = idx / ((size_t)oh * ow);  // img * C + c
    const int c = (int)(ic % C), img = (int)(ic / C);
    const int r = i / ow, col = i % ow;
    int64_t best = 0;
    const int np = pool ? 4 : 1;
    for (int t = 0; t < np; ++t) {
      const int rr = pool ? 2 * r + (t >> 1) : r, cc = pool ? 2 * col + (t & 1) : col;
      const size_t src = ic * (size_t)H * W + (size_t)rr * W + cc;
      uint32_t rec = a[src] % p + b[src] % p;
      rec = rec >= p ? rec - p : rec;
      int64_t y = rec > p / 2 ? (int64_t)rec - (int64_t)p : (int64_t)rec;  // decode_signed
      int64_t o = y;
      if (fn == 0) o = y > 0 ? y : 0;
      else if (fn == 1) {
        o = y * y;
        if (o > half && overflow) atomicOr(overflow, 1);
      }
      best = t == 0 ? o : (o > best ? o : best);
    }
    int64_t m = best % (int64_t)p;
    const uint32_t v = (uint32_t)(m < 0 ? m + p : m);  // encode_signed
    const uint32_t fresh = inj ? inj[idx] : draw_uniform_p(key, stream_id(PURPOSE_RESHARE, layer, image_base + img, c, 0), i, p);
    nb[idx] = fresh;
    na[idx] = v >= fresh ? v - fresh : v + p - fresh;
  }
}

struct Workspace {
  uint64_t* ct_in;
  uint64_t* ct_out;
  uint32_t* bob;
  void* mac;  // ElementMult scratch (int8 byte planes), nullptr when none is needed
  uint8_t* stage_in;
  uint32_t* stage_out;
};

size_t mac_bytes(const ensei_gpu_ctx* c, const ensei_conv_desc* d, const Geo& g, uint32_t imgs) {
  LayerArgs a;
  std::memset(&a, 0, sizeof(a));
  a.cin = (int)d->cin;
  a.cout = (int)d->cout;
  a.B = (int)g.B;
  a.num_images = (int)g.cts(imgs);  // the ElementMult's rows are ciphertexts
  return (mac_scratch_bytes(c, a) + 255) & ~(size_t)255;
}

size_t ct_bytes(const ensei_gpu_ctx* c, const Geo& g, uint32_t ch, uint32_t imgs) {
  imgs = g.cts(imgs);  // ciphertexts hold pk images each
  return (size_t)imgs * ch * g.B * 2 * c->R * c->n * sizeof(uint64_t);
}
size_t share_bytes(const Geo& g, uint32_t cout, uint32_t imgs) {
  return ((size_t)imgs * cout * g.oh * g.ow * sizeof(uint32_t) + 255) & ~(size_t)255;
}
size_t in_bytes(const ensei_conv_desc* d, uint32_t imgs, int in_dtype) {
  return ((size_t)imgs * d->cin * d->H * d->W * (in_dtype == ENSEI_IN_U8 ? 1 : 4) + 255) & ~(size_t)255;
}

Workspace carve(const ensei_gpu_ctx* c, const ensei_conv_desc* d, const Geo& g, uint32_t imgs, void* ws,
                int in_dtype, bool host) {
  Workspace w{};
  uint8_t* p = static_cast<uint8_t*>(ws);
  w.ct_in = reinterpret_cast<uint64_t*>(p);
  p += ct_bytes(c, g, d->cin, imgs);
  w.ct_out = reinterpret_cast<uint64_t*>(p);
  p += ct_bytes(c, g, d->cout, imgs);
  w.bob = reinterpret_cast<uint32_t*>(p);
  p += share_bytes(g, d->cout, imgs);
  const size_t mb = mac_bytes(c, d, g, imgs);
  w.mac = mb ? p : nullptr;
  p += mb;
  if (host) {
    w.stage_in = p;
    p += in_bytes(d, imgs, in_dtype);
    w.stage_out = reinterpret_cast<uint32_t*>(p);
  }
  return w;
}

// Images per sub-batch: the workspace holds the ciphertexts (both parties) and the
// ElementMult planes of at most this many images (<= 12 GiB of ciphertexts, a multiple
// of 64 images -- one 128-row ElementMult tile -- once that many fit).  Larger batches
// stream through it chunk by chunk (config 4: 1024 images in 8 chunks of 128).
uint32_t chunk_images(const ensei_gpu_ctx* c, const ensei_conv_desc* d, const Geo& g, uint32_t imgs) {
  const size_t per = ct_bytes(c, g, d->cin, 1) + ct_bytes(c, g, d->cout, 1);  // one ciphertext image
  uint64_t k = std::max<uint64_t>(1, ((size_t)12 << 30) / per);
  if (k >= 64) k = k / 64 * 64;
  k *= g.pk;  // images (a multiple of pk: stream ids stay pack-aligned across sub-batches)
  return (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(k, imgs));
}

// One sub-batch of the layer on stream `st` (aux stream `aux` for Bob's masks):
// share || (Enc [+ HomRec]) -> ElementMult -> Dec (+ recombine).  in / bob_prev / key /
// alice_share / bob_share / out point at the sub-batch's first image already; i0 is its
// index in the caller's batch (randomness stream ids, injected draws); the workspace is
// sub-batch local.
void layer_chain(ensei_gpu_ctx* ctx, const ensei_conv_desc* desc, const Geo& g, const uint64_t* key, uint32_t ks,
                 const uint64_t* w_eval, const void* in, int in_dtype, const uint32_t* bob_prev, uint32_t i0,
                 uint32_t imgs, const ensei_randomness* rand, const Workspace& w, uint32_t* alice_share,
                 uint32_t* bob_share, uint32_t* out, cudaStream_t st, cudaStream_t aux, cudaEvent_t fork,
                 cudaEvent_t join) {
  ensei_randomness rc{};
  if (rand) {
    rc = *rand;
    rc.image_base += i0;
    const size_t nwords = (size_t)ctx->n, B = g.B;
    if (rc.d_noise) rc.d_noise += (size_t)i0 * desc->cin * B * nwords;
    if (rc.d_a_hat) rc.d_a_hat += (size_t)i0 * desc->cin * B * ctx->R * nwords;
    if (rc.d_share) rc.d_share += (size_t)i0 * desc->cout * B * nwords;
  }
  LayerRun r = make_run(ctx, desc, g, imgs, rand ? &rc : nullptr, st);
  uint32_t* bs = bob_share ? bob_share : w.bob;
  const bool inj = injected(rand);
  // Bob's HomShare masks depend only on his randomness: fork them onto the aux stream
  // so they overlap Alice's encryption; join before the ElementMult consumes them.  In a
  // per-kernel timing pass (ensei_gpu_profile) they run in line, so that every kernel's
  // event span is its own.
  const bool fork_share = !prof_on() && !g_no_fork.load(std::memory_order_relaxed);
  LayerRun ra = r;
  if (fork_share) {
    EG_CUDA(cudaEventRecord(fork, st));
    EG_CUDA(cudaStreamWaitEvent(aux, fork, 0));
    ra.st = aux;
  }
  const int cts = r.a.num_cts;  // ciphertext images (pk images each)
  share(ra, inj, w.ct_out, bs, cts * (int)desc->cout);
  if (fork_share) EG_CUDA(cudaEventRecord(join, aux));
  tile(r, TILE_ENC, inj, in_dtype, key, ks, in, w.ct_in, cts * (int)desc->cin);
  if (bob_prev) tile(r, TILE_HOMREC, false, ENSEI_IN_U32, key, 0, bob_prev, w.ct_in, cts * (int)desc->cin);
  if (fork_share) EG_CUDA(cudaStreamWaitEvent(st, join, 0));
  mac(mac_run(r), w.ct_in, w_eval, w.ct_out, w.mac);
  dec(r, key, ks, w.ct_out, alice_share, bs, out, cts * (int)desc->cout);
}

// The whole batch through the chunk-sized workspace.  in_at(i0, cnt) gives the device
// address of image i0's input (and may enqueue its staging copy), out_at(i0) the address
// its output goes to (nullptr: none); out_done(i0, cnt) runs after a chunk's output is
// written (staging copy back); all on `st`.
template <class InAt, class OutAt, class OutDone>
void chunked(ensei_gpu_ctx* ctx, const ensei_conv_desc* desc, const Geo& g, const uint64_t* key, uint32_t ks,
             const uint64_t* w_eval, int in_dtype, const uint32_t* bob_prev, uint32_t imgs,
             const ensei_randomness* rand, const Workspace& w, uint32_t* alice_share, uint32_t* bob_share,
             cudaStream_t st, InAt in_at, OutAt out_at, OutDone out_done) {
  const uint32_t chunk = chunk_images(ctx, desc, g, imgs);
  const size_t tin = (size_t)desc->cin * desc->H * desc->W, tout = (size_t)desc->cout * g.oh * g.ow;
  for (uint32_t i0 = 0; i0 < imgs; i0 += chunk) {
    const uint32_t cnt = std::min(chunk, imgs - i0);
    layer_chain(ctx, desc, g, key + (size_t)i0 * ks, ks, w_eval, in_at(i0, cnt), in_dtype,
                bob_prev ? bob_prev + (size_t)i0 * tin : nullptr, i0, cnt, rand, w,
                alice_share ? alice_share + (size_t)i0 * tout : nullptr,
                bob_share ? bob_share + (size_t)i0 * tout : nullptr, out_at(i0), st,
                ctx->aux, ctx->ev_fork, ctx->ev_join);
    out_done(i0, cnt);
  }
}

void conv_layer(ensei_gpu_ctx* ctx, const ensei_conv_desc* desc, const uint64_t* key, uint32_t ks,
                const uint64_t* w_eval, const void* in, int in_dtype, const uint32_t* bob_prev, uint32_t imgs,
                const ensei_randomness* rand, void* ws, uint32_t* alice_share, uint32_t* bob_share, uint32_t* out,
                void* stream) {
  require(ctx && desc && key && w_eval && in && ws, ENSEI_ERR_INVALID_ARGUMENT, "null argument");
  Geo g = geometry(ctx, desc);
  Workspace w = carve(ctx, desc, g, chunk_images(ctx, desc, g, imgs), ws, in_dtype, false);
  const size_t esz = in_dtype == ENSEI_IN_U8 ? 1 : 4, tin = (size_t)desc->cin * desc->H * desc->W;
  const size_t tout = (size_t)desc->cout * g.oh * g.ow;
  chunked(ctx, desc, g, key, ks, w_eval, in_dtype, bob_prev, imgs, rand, w, alice_share, bob_share,
          (cudaStream_t)stream,
          [&](uint32_t i0, uint32_t) { return static_cast<const void*>(static_cast<const uint8_t*>(in) + i0 * tin * esz); },
          [&](uint32_t i0) { return out ? out + (size_t)i0 * tout : nullptr; }, [](uint32_t, uint32_t) {});
}

}  // namespace
}  // namespace ensei_gpu

using namespace ensei_gpu;

extern "C" {

int ensei_gpu_layer_geometry(const ensei_gpu_ctx* ctx, const ensei_conv_desc* desc, ensei_layer_geom* geom) {
  return guarded([&] {
    require(geom != nullptr, ENSEI_ERR_INVALID_ARGUMENT, "null argument");
    Geo g = geometry(ctx, desc);
    *geom = {g.Lh, g.Lw, g.B, g.oh, g.ow, g.r0, g.c0, g.pk};
  });
}

int ensei_gpu_secret_from_coeffs(ensei_gpu_ctx* ctx, const int64_t* d_t, uint64_t* d_key, void* stream) {
  return guarded([&] {
    require(ctx && d_t && d_key, ENSEI_ERR_INVALID_ARGUMENT, "null argument");
    ensei_conv_desc d{2, 2, 1, 1, 1, 1, 1};
    Geo g{2, 2, 1, 1, 2, 2, 0, 0, 4};
    secret(make_run(ctx, &d, g, 0, nullptr, stream), d_t, nullptr, d_key, false);
  });
}

int ensei_gpu_secret_sample(ensei_gpu_ctx* ctx, uint64_t alice_key, int64_t* d_t, uint64_t* d_key, void* stream) {
  return guarded([&] {
    require(ctx && d_key, ENSEI_ERR_INVALID_ARGUMENT, "null argument");
    ensei_conv_desc d{2, 2, 1, 1, 1, 1, 1};
    Geo g{2, 2, 1, 1, 2, 2, 0, 0, 4};
    ensei_randomness rnd{};
    rnd.mode = ENSEI_RAND_PHILOX;
    rnd.alice_key = alice_key;
    secret(make_run(ctx, &d, g, 0, &rnd, stream), nullptr, d_t, d_key, true);
  });
}

int ensei_gpu_prepare_weights(ensei_gpu_ctx* ctx, const ensei_conv_desc* desc, const int32_t* d_w,
                              uint64_t* d_w_eval, void* stream) {
  return guarded([&] {
    require(d_w && d_w_eval, ENSEI_ERR_INVALID_ARGUMENT, "null argument");
    Geo g = geometry(ctx, desc);
    LayerRun r = make_run(ctx, desc, g, 0, nullptr, stream);
    tile(r, TILE_WEIGHTS, false, 0, nullptr, 0, d_w, d_w_eval, (int)(desc->cout * desc->cin));
    build_w_planes(r, d_w_eval);
  });
}

size_t ensei_gpu_prepared_weights_bytes(const ensei_gpu_ctx* ctx, const ensei_conv_desc* desc) {
  size_t out = 0;
  guarded([&] {
    Geo g = geometry(ctx, desc);
    out = prepared_weights_bytes(ctx, make_run(ctx, desc, g, 0, nullptr, nullptr).a);
  });
  return out;
}

int ensei_gpu_prepare_weight_planes(ensei_gpu_ctx* ctx, const ensei_conv_desc* desc, uint64_t* d_w_eval,
                                    void* stream) {
  return guarded([&] {
    require(d_w_eval, ENSEI_ERR_INVALID_ARGUMENT, "null argument");
    Geo g = geometry(ctx, desc);
    build_w_planes(make_run(ctx, desc, g, 0, nullptr, stream), d_w_eval);
  });
}

int ensei_gpu_alice_encrypt(ensei_gpu_ctx* ctx, const ensei_conv_desc* desc, const uint64_t* d_key,
                            uint32_t key_stride, const void* d_in, int in_dtype, uint32_t num_images,
                            const ensei_randomness* rand, uint64_t* d_ct, void* stream) {
  return guarded([&] {
    require(d_key && d_in && d_ct, ENSEI_ERR_INVALID_ARGUMENT, "null argument");
    require(in_dtype == ENSEI_IN_U32 || in_dtype == ENSEI_IN_U8, ENSEI_ERR_INVALID_ARGUMENT, "bad input dtype");
    Geo g = geometry(ctx, desc);
    LayerRun r = make_run(ctx, desc, g, num_images, rand, stream);
    require(g.pk == 1 || key_stride == 0, ENSEI_ERR_UNSUPPORTED, "packed layers share one key per ciphertext");
    tile(r, TILE_ENC, injected(rand), in_dtype, d_key, key_stride, d_in, d_ct, r.a.num_cts * (int)desc->cin);
  });
}

int ensei_gpu_bob_eval(ensei_gpu_ctx* ctx, const ensei_conv_desc* desc, uint64_t* d_ct, const uint64_t* d_w_eval,
                       const uint32_t* d_bob_prev, uint32_t num_images, const ensei_randomness* rand,
                       uint64_t* d_ct_out, uint32_t* d_bob_share, void* stream) {
  return guarded([&] {
    require(d_ct && d_w_eval && d_ct_out && d_bob_share, ENSEI_ERR_INVALID_ARGUMENT, "null argument");
    Geo g = geometry(ctx, desc);
    LayerRun r = make_run(ctx, desc, g, num_images, rand, stream);
    share(r, injected(rand), d_ct_out, d_bob_share, r.a.num_cts * (int)desc->cout);
    if (d_bob_prev) tile(r, TILE_HOMREC, false, ENSEI_IN_U32, nullptr, 0, d_bob_prev, d_ct, r.a.num_cts * (int)desc->cin);
    mac(mac_run(r), d_ct, d_w_eval, d_ct_out);
  });
}

int ensei_gpu_bob_share(ensei_gpu_ctx* ctx, const ensei_conv_desc* desc, uint32_t num_images,
                        const ensei_randomness* rand, uint64_t* d_ct_out, uint32_t* d_bob_share, void* stream) {
  return guarded([&] {
    require(d_ct_out && d_bob_share, ENSEI_ERR_INVALID_ARGUMENT, "null argument");
    Geo g = geometry(ctx, desc);
    LayerRun r = make_run(ctx, desc, g, num_images, rand, stream);
    share(r, injected(rand), d_ct_out, d_bob_share, r.a.num_cts * (int)desc->cout);
  });
}

int ensei_gpu_bob_mac(ensei_gpu_ctx* ctx, const ensei_conv_desc* desc, const uint64_t* d_ct,
                      const uint64_t* d_w_eval, uint32_t num_images, uint64_t* d_ct_out, void* stream) {
  return guarded([&] {
    require(d_ct && d_w_eval && d_ct_out, ENSEI_ERR_INVALID_ARGUMENT, "null argument");
    Geo g = geometry(ctx, desc);
    LayerRun r = make_run(ctx, desc, g, num_images, nullptr, stream);
    mac(mac_run(r), d_ct, d_w_eval, d_ct_out);
  });
}

int ensei_gpu_alice_decrypt(ensei_gpu_ctx* ctx, const ensei_conv_desc* desc, const uint64_t* d_key,
                            uint32_t key_stride, const uint64_t* d_ct_out, uint32_t num_images,
                            uint32_t* d_alice_share, void* stream) {
  return guarded([&] {
    require(d_key && d_ct_out && d_alice_share, ENSEI_ERR_INVALID_ARGUMENT, "null argument");
    Geo g = geometry(ctx, desc);
    LayerRun r = make_run(ctx, desc, g, num_images, nullptr, stream);
    require(g.pk == 1 || key_stride == 0, ENSEI_ERR_UNSUPPORTED, "packed layers share one key per ciphertext");
    dec(r, d_key, key_stride, d_ct_out, d_alice_share, nullptr, nullptr, r.a.num_cts * (int)desc->cout);
  });
}

int ensei_gpu_activation(ensei_gpu_ctx* ctx, int fn, int pool2, uint32_t channels, uint32_t H, uint32_t W,
                         uint32_t num_images, const uint32_t* d_a, const uint32_t* d_b, const ensei_randomness* rand,
                         uint32_t* d_new_a, uint32_t* d_new_b, int* d_overflow, void* stream) {
  return guarded([&] {
    require(ctx && d_a && d_b && d_new_a && d_new_b, ENSEI_ERR_INVALID_ARGUMENT, "null argument");
    require(fn >= 0 && fn <= 2, ENSEI_ERR_INVALID_ARGUMENT, "bad activation fn");
    require(!pool2 || (H % 2 == 0 && W % 2 == 0), ENSEI_ERR_BAD_GEOMETRY, "2x2 pooling needs even dims");
    const size_t total = (size_t)num_images * channels * (pool2 ? (H / 2) * (W / 2) : H * W);
    if (!total) return;
    const bool inj = rand && rand->mode == ENSEI_RAND_INJECTED;
    size_t grid = std::min<size_t>((total + 255) / 256, (size_t)ctx->sm_count * 16);
    activation_kernel<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(
        d_a, d_b, fn, pool2, (int)channels, (int)H, (int)W, total, (uint32_t)ctx->p, rand ? rand->layer : 0,
        rand ? rand->image_base : 0, rand ? rand->alice_key : 0, inj ? rand->d_share : nullptr, d_new_a, d_new_b,
        d_overflow);
    check_launch("activation_kernel");
  });
}

int ensei_gpu_mac_path(const ensei_gpu_ctx* ctx, const ensei_conv_desc* desc, uint32_t num_images, int* path) {
  return guarded([&] {
    require(path != nullptr, ENSEI_ERR_INVALID_ARGUMENT, "null argument");
    Geo g = geometry(ctx, desc);
    LayerArgs a;
    std::memset(&a, 0, sizeof(a));
    a.cin = (int)desc->cin;
    a.cout = (int)desc->cout;
    a.B = (int)g.B;
    a.num_images = (int)g.cts(num_images);  // ElementMult rows: ciphertexts
    *path = mac_path(ctx, a);
  });
}

int ensei_gpu_set_mac_variant(int variant) {
  return guarded([&] {
    require(variant >= -1 && variant <= 5 && variant != 4, ENSEI_ERR_INVALID_ARGUMENT, "variant must be -1, 0, 1, 2, 3 or 5");
    set_mac_variant(variant);
  });
}

int ensei_gpu_set_tile_variant(int variant) {
  return guarded([&] {
    require(variant >= 0 && variant <= 3, ENSEI_ERR_INVALID_ARGUMENT, "variant must be 0..3");
    g_tile_gen.store(variant & 1, std::memory_order_relaxed);
    g_no_fork.store(variant >> 1, std::memory_order_relaxed);
  });
}

int ensei_gpu_crt_round(ensei_gpu_ctx* ctx, const uint64_t* d_res, size_t count, uint32_t* d_out, void* stream) {
  return guarded([&] {
    require(ctx && (count == 0 || (d_res && d_out)), ENSEI_ERR_INVALID_ARGUMENT, "null argument");
    require(ctx->R == 3, ENSEI_ERR_UNSUPPORTED, "exact CRT rounding: three-prime contexts");
    if (!count) return;
    ensei_conv_desc d{2, 2, 1, 1, 1, 1, 1};
    Geo g{2, 2, 1, 1, 2, 2, 0, 0, 4};
    LayerRun r = make_run(ctx, &d, g, 0, nullptr, stream);
    const size_t grid = std::min<size_t>((count + 255) / 256, (size_t)ctx->sm_count * 8);
    crt_round_kernel<3><<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(r.a, d_res, count, d_out);
    check_launch("crt_round_kernel");
  });
}

int ensei_gpu_recombine(ensei_gpu_ctx* ctx, const uint32_t* d_a, const uint32_t* d_b, size_t count, uint32_t* d_out,
                        void* stream) {
  return guarded([&] {
    require(ctx && d_a && d_b && d_out, ENSEI_ERR_INVALID_ARGUMENT, "null argument");
    if (!count) return;
    size_t grid = std::min<size_t>((count + 255) / 256, (size_t)ctx->sm_count * 8);
    recombine_kernel<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(d_a, d_b, count, (uint32_t)ctx->p, d_out);
    check_launch("recombine_kernel");
  });
}

uint32_t ensei_gpu_conv_chunk_images(const ensei_gpu_ctx* ctx, const ensei_conv_desc* desc, uint32_t num_images) {
  uint32_t out = 0;
  guarded([&] { out = chunk_images(ctx, desc, geometry(ctx, desc), num_images); });
  return out;
}

size_t ensei_gpu_conv_workspace_bytes(const ensei_gpu_ctx* ctx, const ensei_conv_desc* desc, uint32_t num_images) {
  size_t out = 0;
  guarded([&] {
    Geo g = geometry(ctx, desc);
    num_images = chunk_images(ctx, desc, g, num_images);
    out = ct_bytes(ctx, g, desc->cin, num_images) + ct_bytes(ctx, g, desc->cout, num_images) +
          share_bytes(g, desc->cout, num_images) + mac_bytes(ctx, desc, g, num_images);
  });
  return out;
}

int ensei_gpu_conv_layer(ensei_gpu_ctx* ctx, const ensei_conv_desc* desc, const uint64_t* d_key, uint32_t key_stride,
                         const uint64_t* d_w_eval, const void* d_in, int in_dtype, const uint32_t* d_bob_prev,
                         uint32_t num_images, const ensei_randomness* rand, void* d_workspace,
                         uint32_t* d_alice_share, uint32_t* d_bob_share, uint32_t* d_out, void* stream) {
  return guarded([&] {
    conv_layer(ctx, desc, d_key, key_stride, d_w_eval, d_in, in_dtype, d_bob_prev, num_images, rand, d_workspace,
               d_alice_share, d_bob_share, d_out, stream);
  });
}

size_t ensei_gpu_conv_host_workspace_bytes(const ensei_gpu_ctx* ctx, const ensei_conv_desc* desc,
                                           uint32_t num_images, int in_dtype) {
  size_t out = 0;
  guarded([&] {
    Geo g = geometry(ctx, desc);
    num_images = chunk_images(ctx, desc, g, num_images);
    out = ct_bytes(ctx, g, desc->cin, num_images) + ct_bytes(ctx, g, desc->cout, num_images) +
          share_bytes(g, desc->cout, num_images) + mac_bytes(ctx, desc, g, num_images) +
          in_bytes(desc, num_images, in_dtype) + share_bytes(g, desc->cout, num_images);
  });
  return out;
}

int ensei_gpu_conv_layer_host(ensei_gpu_ctx* ctx, const ensei_conv_desc* desc, const uint64_t* d_key,
                              const uint64_t* d_w_eval, const void* h_in, int in_dtype, uint32_t num_images,
                              const ensei_randomness* rand, void* d_workspace, uint32_t* h_out, void* stream) {
  return guarded([&] {
    require(ctx && desc && h_in && h_out && d_workspace && rand, ENSEI_ERR_INVALID_ARGUMENT, "null argument");
    Geo g = geometry(ctx, desc);
    Workspace w = carve(ctx, desc, g, chunk_images(ctx, desc, g, num_images), d_workspace, in_dtype, true);
    const size_t tin = (size_t)desc->cin * desc->H * desc->W * (in_dtype == ENSEI_IN_U8 ? 1 : 4);
    const size_t tout = (size_t)desc->cout * g.oh * g.ow * sizeof(uint32_t);
    cudaStream_t user = (cudaStream_t)stream;
    // the legacy stream cannot be captured: run on the context's own stream, ordered after
    // the caller's prior work by an event
    if (!ctx->host_st) {
      EG_CUDA(cudaStreamCreateWithFlags(&ctx->host_st, cudaStreamNonBlocking));
      EG_CUDA(cudaEventCreateWithFlags(&ctx->host_ev, cudaEventDisableTiming));
    }
    cudaStream_t st = user ? user : ctx->host_st;
    if (!user) {
      EG_CUDA(cudaEventRecord(ctx->host_ev, 0));
      EG_CUDA(cudaStreamWaitEvent(st, ctx->host_ev, 0));
    }
    // Pinned (page-locked) host buffers are device-addressable: Enc then reads the pixels
    // and Dec writes the outputs across the host link directly (zero-copy), so the
    // transfers overlap the kernels instead of being two serial memcpys with their own
    // fixed latency.  Pageable buffers go through the workspace staging copies.
    auto mapped = [](const void* h) -> void* {
      cudaPointerAttributes at{};
      if (cudaPointerGetAttributes(&at, h) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
      }
      return at.type == cudaMemoryTypeHost ? at.devicePointer : nullptr;
    };
    const void* din = mapped(h_in);
    uint32_t* dout = static_cast<uint32_t*>(mapped(h_out));
    // chunk by chunk: pinned buffers are read / written in place, pageable ones staged
    // through the (chunk-sized) workspace with one copy each way per chunk
    auto enqueue = [&] {
      chunked(ctx, desc, g, d_key, 0, d_w_eval, in_dtype, nullptr, num_images, rand, w, nullptr, nullptr, st,
              [&](uint32_t i0, uint32_t cnt) -> const void* {
                if (din) return static_cast<const uint8_t*>(din) + i0 * tin;
                EG_CUDA(cudaMemcpyAsync(w.stage_in, static_cast<const uint8_t*>(h_in) + i0 * tin, cnt * tin,
                                        cudaMemcpyHostToDevice, st));
                return w.stage_in;
              },
              [&](uint32_t i0) { return dout ? dout + i0 * (tout / sizeof(uint32_t)) : w.stage_out; },
              [&](uint32_t i0, uint32_t cnt) {
                if (!dout)
                  EG_CUDA(cudaMemcpyAsync(reinterpret_cast<uint8_t*>(h_out) + i0 * tout, w.stage_out, cnt * tout,
                                          cudaMemcpyDeviceToHost, st));
              });
    };
    // graph key: every argument that shapes the launches (pointers, sizes, randomness)
    std::vector<uint8_t> key;
    auto put = [&](const void* p, size_t n) {
      const uint8_t* b = static_cast<const uint8_t*>(p);
      key.insert(key.end(), b, b + n);
    };
    put(desc, sizeof(*desc));
    put(rand, sizeof(*rand));
    const void* ptrs[] = {d_key, d_w_eval, h_in, d_workspace, h_out, st};
    put(ptrs, sizeof(ptrs));
    put(&in_dtype, sizeof(in_dtype));
    put(&num_images, sizeof(num_images));
    if (!(ctx->host_graph && key == ctx->host_graph_key)) {
      if (ctx->host_graph) {
        cudaGraphExecDestroy(ctx->host_graph);
        ctx->host_graph = nullptr;
      }
      ctx->host_graph_key.clear();
      cudaGraph_t graph = nullptr;
      bool ok = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
      const uint64_t before = g_launches.load();
      if (ok) {
        try {
          enqueue();
        } catch (...) {
          cudaStreamEndCapture(st, &graph);
          if (graph) cudaGraphDestroy(graph);
          throw;
        }
        ctx->host_graph_kernels = g_launches.load() - before;
        g_launches.fetch_sub(ctx->host_graph_kernels);  // captured, not launched: counted at replay
        ok = cudaStreamEndCapture(st, &graph) == cudaSuccess && graph;
        ok = ok && cudaGraphInstantiate(&ctx->host_graph, graph, 0) == cudaSuccess;
        if (graph) cudaGraphDestroy(graph);
      }
      if (!ok) {  // not capturable (e.g. pageable host memory): plain launches
        cudaGetLastError();
        ctx->host_graph = nullptr;
        enqueue();
        EG_CUDA(cudaStreamSynchronize(st));
        return;
      }
      ctx->host_graph_key = key;
    }
    EG_CUDA(cudaGraphLaunch(ctx->host_graph, st));
    count_launch(ctx->host_graph_kernels);
    EG_CUDA(cudaStreamSynchronize(st));
  });
}

}  // extern "C"
