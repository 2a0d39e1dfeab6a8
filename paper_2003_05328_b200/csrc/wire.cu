// wire.cu -- device-side wire framing: the reference's message layouts built and
// parsed by kernels straight from / into the device layouts (include/ensei_gpu.h,
// "wire framing").
//
// REF: frame header wire.cpp:44-79 ("ENSE" | 0x01 | type | u64 LE length), ciphertext
// record wire.cpp:112-144 (tag | n | c0 | c1), ciphertext-blocks payload
// protocol.cpp:83-117, shares payload protocol.cpp:119-150, recv_expect
// protocol.cpp:55-65.
//
// Records are 9 + 16n bytes, so every record after the first starts at a different
// byte alignment.  Each CTA owns one record (ciphertexts) or one slice of values
// (shares): the polynomial is staged through shared memory (coalesced on both sides
// of the bit-reversal; XOR swizzle keeps the bit-reversed accesses conflict-free),
// and every aligned 8-byte output word inside the record is one funnel shift of two
// neighbouring coefficients -- full-width coalesced stores.  The few words a record
// shares with its neighbours (and the 9-byte record header) are written bytewise.
// Decoding runs the same map backwards with one aligned load per word plus a warp
// shuffle for the neighbour, validates every field and records the FIRST violation
// in REF's read order as a per-batch atomicMin over (frame, position) keys.
#include <algorithm>
#include <cstring>
#include <string>

#include "common.cuh"

namespace ensei_gpu {

int run_guarded(void (*fn)(void*), void* arg);

namespace {

template <class Fn>
int guarded(Fn&& fn) {
  struct Box {
    Fn* f;
  } box{&fn};
  return run_guarded([](void* p) { (*static_cast<Box*>(p)->f)(); }, &box);
}

constexpr uint64_t kFrameHdr = 14;                 // REF kFrameHeaderBytes (wire.hpp:40)
constexpr uint64_t kMaxPayload = 1ull << 30;       // REF kMaxPayloadBytes (wire.hpp:41)
constexpr uint64_t kCtHdr = kFrameHdr + 12;        // + layer, channels, blocks
constexpr uint64_t kShareHdr = kFrameHdr + 16;     // + layer, channels, rows, cols
constexpr int kThreads = 256;

// Per-frame error positions, ordered as REF reads a frame (smaller = earlier).
enum : uint32_t {
  E_MAGIC = 1,      // MalformedPayload "bad magic"
  E_VERSION,        // "unsupported version"
  E_TYPE,           // "unknown message type"
  E_CAP,            // "payload length exceeds cap"
  E_LENGTH,         // "payload length mismatch"
  E_PEER,           // ProtocolOrderViolation "peer aborted: ..."
  E_UNEXPECTED,     // ProtocolOrderViolation "expected X, got Y"
  E_TRUNC_HDR,      // MalformedPayload "truncated payload" (payload header)
  E_LAYOUT,         // ProtocolOrderViolation "... layout mismatch"
  E_RECORDS = 16    // + record / value positions
};

// device status block: [0] first-error key, [1] domain flags, u32 layers[frames], u8 tags[...]
struct StatusView {
  unsigned long long* key;
  unsigned long long* flags;
  uint32_t* layers;
  uint8_t* tags;
};

EG_DEV int swz(int x, int sh) { return x ^ ((x >> sh) & 15); }

EG_DEV void report(unsigned long long* key, uint64_t frame_key, uint32_t f, uint64_t local) {
  atomicMin(key, (unsigned long long)(f * frame_key + local));
}

EG_DEV void put_frame_header(uint8_t* F, uint8_t type, uint64_t payload) {
  F[0] = 'E';
  F[1] = 'N';
  F[2] = 'S';
  F[3] = 'E';
  F[4] = 0x01;
  F[5] = type;
  for (int i = 0; i < 8; ++i) F[6 + i] = (uint8_t)(payload >> (8 * i));
}
EG_DEV void put_u32(uint8_t* p, uint32_t v) {
  for (int i = 0; i < 4; ++i) p[i] = (uint8_t)(v >> (8 * i));
}
EG_DEV uint32_t get_u32(const uint8_t* p) {
  uint32_t v = 0;
  for (int i = 0; i < 4; ++i) v |= (uint32_t)p[i] << (8 * i);
  return v;
}

// decode_frame + recv_expect + the payload's count fields (REF wire.cpp:57-79,
// protocol.cpp:55-65 and 99-108 / 134-143).  Returns 0 or the local error position.
EG_DEV uint32_t check_header(const uint8_t* F, size_t frame_len, uint32_t expect_type, uint64_t payload_hdr,
                             const uint32_t* expect, int n_expect, uint32_t* layer) {
  if (F[0] != 'E' || F[1] != 'N' || F[2] != 'S' || F[3] != 'E') return E_MAGIC;
  if (F[4] != 0x01) return E_VERSION;
  if (F[5] < 0x01 || F[5] > 0x07) return E_TYPE;
  uint64_t len = 0;
  for (int i = 0; i < 8; ++i) len |= (uint64_t)F[6 + i] << (8 * i);
  if (len > kMaxPayload) return E_CAP;
  if (frame_len != kFrameHdr + len) return E_LENGTH;
  if (F[5] == ENSEI_MSG_ERROR) return E_PEER;
  if (F[5] != expect_type) return E_UNEXPECTED;
  if (frame_len < payload_hdr) return E_TRUNC_HDR;
  *layer = get_u32(F + kFrameHdr);
  for (int i = 0; i < n_expect; ++i)
    if (get_u32(F + kFrameHdr + 4 + 4 * i) != expect[i]) return E_LAYOUT;
  return 0;
}

// ------------------------------------------------------------------ ciphertexts

__global__ void __launch_bounds__(kThreads) wire_encode_ct_kernel(const uint64_t* __restrict__ src, uint8_t* frames,
                                                                  size_t stride, uint32_t logn, uint32_t recs,
                                                                  int bitrev, uint8_t tag, uint8_t type,
                                                                  uint32_t layer, uint32_t C, uint32_t B) {
  extern __shared__ uint64_t sm[];
  const uint32_t n = 1u << logn, k = blockIdx.x, f = blockIdx.y;
  const int sh = (int)logn - 4;
  const uint64_t* s = src + ((size_t)f * recs + k) * 2 * n;
  for (uint32_t i = threadIdx.x; i < 2 * n; i += kThreads)
    sm[((i >> logn) << logn) + swz(i & (n - 1), sh)] = __ldcs(s + i);
  uint8_t* F = frames + (size_t)f * stride;
  const uint64_t rb = 9 + 16ull * n;
  if (k == 0 && threadIdx.x == 0) {
    put_frame_header(F, type, 12 + (uint64_t)recs * rb);
    put_u32(F + kFrameHdr, layer);
    put_u32(F + kFrameHdr + 4, C);
    put_u32(F + kFrameHdr + 8, B);
  }
  __syncthreads();
  // natural coefficient i of (c0 || c1) from the staged device-layout polynomial
  auto coef = [&](uint32_t i) -> uint64_t {
    uint32_t j = i & (n - 1);
    uint32_t x = bitrev ? (uint32_t)brev((int)j, (int)logn) : j;
    return sm[((i >> logn) << logn) + swz((int)x, sh)];
  };
  const uintptr_t r0 = (uintptr_t)(F + kCtHdr + (uint64_t)k * rb), r1 = r0 + rb, body = r0 + 9;
  const uintptr_t a0 = r0 & ~(uintptr_t)7;
  const uint32_t words = (uint32_t)((((r1 + 7) & ~(uintptr_t)7) - a0) >> 3);
  const uint32_t b = (uint32_t)((a0 - body) & 7);  // shift of every interior word
  for (uint32_t w = threadIdx.x; w < words; w += kThreads) {
    const uintptr_t a = a0 + 8ull * w;
    if (a >= body && a + 8 <= r1) {
      uint32_t i = (uint32_t)((a - body) >> 3);
      uint64_t v = coef(i);
      if (b) v = (v >> (8 * b)) | (coef(i + 1) << (64 - 8 * b));
      *reinterpret_cast<uint64_t*>(a) = v;
    } else {
      const bool full = a >= r0 && a + 8 <= r1;
      uint64_t v = 0;
      for (int t = 0; t < 8; ++t) {
        const uintptr_t o = a + t;
        if (o < r0 || o >= r1) continue;
        const uint64_t off = o - r0;
        uint8_t by;
        if (off == 0)
          by = tag;
        else if (off < 9)
          by = (uint8_t)((uint64_t)n >> (8 * (off - 1)));
        else
          by = (uint8_t)(coef((uint32_t)((off - 9) >> 3)) >> (8 * ((off - 9) & 7)));
        if (full)
          v |= (uint64_t)by << (8 * t);
        else
          *reinterpret_cast<uint8_t*>(o) = by;
      }
      if (full) *reinterpret_cast<uint64_t*>(a) = v;
    }
  }
}

__global__ void __launch_bounds__(kThreads) wire_decode_ct_kernel(const uint8_t* frames, size_t frame_len,
                                                                  size_t stride, uint32_t logn, uint32_t recs,
                                                                  uint32_t avail, uint32_t expect_type, uint32_t C,
                                                                  uint32_t B, uint64_t q, StatusView st,
                                                                  uint64_t frame_key, uint64_t* __restrict__ dst) {
  extern __shared__ uint64_t sm[];
  __shared__ uint32_t s_tag;
  const uint32_t n = 1u << logn, k = blockIdx.x, f = blockIdx.y;
  const int sh = (int)logn - 4;
  const uint8_t* F = frames + (size_t)f * stride;
  const uint64_t rb = 9 + 16ull * n;
  const uint8_t* R = F + kCtHdr + (uint64_t)k * rb;
  const uint64_t rec_key = E_RECORDS + (uint64_t)k * (2 * n + 2);
  if (threadIdx.x == 0) {
    if (k == 0) {
      uint32_t expect[2] = {C, B}, layer = 0;
      uint32_t e = check_header(F, frame_len, expect_type, kCtHdr, expect, 2, &layer);
      if (e) report(st.key, frame_key, f, e);
      st.layers[f] = layer;
    }
    uint32_t tag = 0;
    if (k < avail) {
      tag = R[0];
      uint64_t nn = 0;
      for (int i = 0; i < 8; ++i) nn |= (uint64_t)R[1 + i] << (8 * i);
      if (tag > 1)
        report(st.key, frame_key, f, rec_key);
      else if (nn != n)
        report(st.key, frame_key, f, rec_key + 1);
      st.tags[(size_t)f * recs + k] = (uint8_t)tag;
      atomicOr(st.flags, tag == 0 ? 2ull : 1ull);
    }
    s_tag = tag;
  }
  __syncthreads();
  if (k >= avail) return;
  const bool eval = s_tag == 1;
  const uintptr_t body = (uintptr_t)(R + 9);
  const uint32_t b = (uint32_t)(body & 7);
  const uint64_t* A = reinterpret_cast<const uint64_t*>(body - b);
  const uint32_t lane = threadIdx.x & 31;
  for (uint32_t i0 = 0; i0 < 2 * n; i0 += kThreads) {  // 2n is a multiple of kThreads
    const uint32_t i = i0 + threadIdx.x;
    uint64_t v = A[i];
    if (b) {
      uint64_t hi = __shfl_down_sync(0xffffffffu, v, 1);
      if (lane == 31) {
        if (i + 1 < 2 * n) {
          hi = A[i + 1];
        } else {  // the record's last word: only its first b bytes belong to the record
          const uint8_t* t = reinterpret_cast<const uint8_t*>(A + i + 1);
          hi = 0;
          for (uint32_t u = 0; u < b; ++u) hi |= (uint64_t)t[u] << (8 * u);
        }
      }
      v = (v >> (8 * b)) | (hi << (64 - 8 * b));
    }
    if (v >= q) report(st.key, frame_key, f, rec_key + 2 + i);
    const uint32_t j = i & (n - 1);
    const uint32_t x = eval ? (uint32_t)brev((int)j, (int)logn) : j;
    sm[((i >> logn) << logn) + swz((int)x, sh)] = v;
  }
  __syncthreads();
  uint64_t* d = dst + ((size_t)f * recs + k) * 2 * n;
  for (uint32_t i = threadIdx.x; i < 2 * n; i += kThreads) d[i] = sm[((i >> logn) << logn) + swz(i & (n - 1), sh)];
}

// ----------------------------------------------------------------------- shares

__global__ void __launch_bounds__(kThreads) wire_encode_shares_kernel(const uint32_t* __restrict__ src,
                                                                      uint8_t* frames, size_t stride, uint64_t cnt,
                                                                      uint8_t type, uint32_t layer, uint32_t C,
                                                                      uint32_t rows, uint32_t cols) {
  const uint32_t f = blockIdx.y;
  uint8_t* F = frames + (size_t)f * stride;
  const uint32_t* s = src + (size_t)f * cnt;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    put_frame_header(F, type, 16 + 8 * cnt);
    put_u32(F + kFrameHdr, layer);
    put_u32(F + kFrameHdr + 4, C);
    put_u32(F + kFrameHdr + 8, rows);
    put_u32(F + kFrameHdr + 12, cols);
  }
  const uintptr_t body = (uintptr_t)(F + kShareHdr), r1 = body + 8 * cnt;
  const uintptr_t a0 = body & ~(uintptr_t)7;
  const uint64_t words = (((r1 + 7) & ~(uintptr_t)7) - a0) >> 3;
  const uint32_t b = (uint32_t)((a0 - body) & 7);
  for (uint64_t w = (uint64_t)blockIdx.x * kThreads + threadIdx.x; w < words; w += (uint64_t)gridDim.x * kThreads) {
    const uintptr_t a = a0 + 8 * w;
    if (a >= body && a + 8 <= r1) {
      uint64_t i = (a - body) >> 3;
      uint64_t v = __ldcs(s + i);
      if (b) v = (v >> (8 * b)) | ((uint64_t)__ldcs(s + i + 1) << (64 - 8 * b));
      *reinterpret_cast<uint64_t*>(a) = v;
    } else {
      for (int t = 0; t < 8; ++t) {
        const uintptr_t o = a + t;
        if (o < body || o >= r1) continue;
        const uint64_t off = o - body;
        *reinterpret_cast<uint8_t*>(o) = (uint8_t)((uint64_t)s[off >> 3] >> (8 * (off & 7)));
      }
    }
  }
}

__global__ void __launch_bounds__(kThreads) wire_decode_shares_kernel(const uint8_t* frames, size_t frame_len,
                                                                      size_t stride, uint64_t cnt, uint64_t avail,
                                                                      uint32_t expect_type, uint32_t C, uint32_t rows,
                                                                      uint32_t cols, uint64_t max_value, StatusView st,
                                                                      uint64_t frame_key, uint32_t* __restrict__ dst) {
  const uint32_t f = blockIdx.y;
  const uint8_t* F = frames + (size_t)f * stride;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    uint32_t expect[3] = {C, rows, cols}, layer = 0;
    uint32_t e = check_header(F, frame_len, expect_type, kShareHdr, expect, 3, &layer);
    if (e) report(st.key, frame_key, f, e);
    st.layers[f] = layer;
  }
  const uintptr_t body = (uintptr_t)(F + kShareHdr);
  const uint32_t b = (uint32_t)(body & 7);
  const uint64_t* A = reinterpret_cast<const uint64_t*>(body - b);
  const uint32_t lane = threadIdx.x & 31;
  uint32_t* d = dst + (size_t)f * cnt;
  for (uint64_t base = (uint64_t)blockIdx.x * kThreads; base < avail; base += (uint64_t)gridDim.x * kThreads) {
    const uint64_t i = base + threadIdx.x;
    const bool ok = i < avail;
    uint64_t v = ok ? A[i] : 0;
    if (b) {
      uint64_t hi = __shfl_down_sync(0xffffffffu, v, 1);
      if (ok && (lane == 31 || i + 1 >= avail)) {
        if (i + 1 < avail) {
          hi = A[i + 1];
        } else {
          const uint8_t* t = reinterpret_cast<const uint8_t*>(A + i + 1);
          hi = 0;
          for (uint32_t u = 0; u < b; ++u) hi |= (uint64_t)t[u] << (8 * u);
        }
      }
      v = (v >> (8 * b)) | (hi << (64 - 8 * b));
    }
    if (ok) {
      if (v >= max_value) report(st.key, frame_key, f, E_RECORDS + i);
      __stcs(d + i, (uint32_t)v);
    }
  }
}

// ------------------------------------------------------------------------ host

void require_accessible(const void* p, const char* what) {
  cudaPointerAttributes a;
  cudaError_t e = cudaPointerGetAttributes(&a, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    fail(ENSEI_ERR_INVALID_ARGUMENT, std::string(what) + ": not a CUDA-visible pointer");
  }
  if (a.type == cudaMemoryTypeUnregistered)
    fail(ENSEI_ERR_INVALID_ARGUMENT, std::string(what) + " must be device or page-locked host memory");
}

StatusView status_view(ensei_gpu_ctx* c, uint32_t frames, uint64_t tags) {
  size_t need = 16 + 4 * (size_t)frames + tags;
  need = (need + 255) & ~(size_t)255;
  if (need > c->wire_status_cap) {
    if (c->wire_status) EG_CUDA(cudaFree(c->wire_status));
    c->wire_status = nullptr;
    c->wire_status_cap = 0;
    EG_CUDA(cudaMalloc(&c->wire_status, need));
    c->wire_status_cap = need;
  }
  StatusView v;
  v.key = reinterpret_cast<unsigned long long*>(c->wire_status);
  v.flags = v.key + 1;
  v.layers = reinterpret_cast<uint32_t*>(c->wire_status + 16);
  v.tags = c->wire_status + 16 + 4 * (size_t)frames;
  return v;
}

void reset_status(ensei_gpu_ctx* c, cudaStream_t st) {
  EG_CUDA(cudaMemsetAsync(c->wire_status, 0xFF, 8, st));
  EG_CUDA(cudaMemsetAsync(c->wire_status + 8, 0, 8, st));
}

const char* msg_name(uint32_t t) {  // REF msg_type_name (wire.cpp:31-42)
  switch (t) {
    case 1: return "Hello";
    case 2: return "CiphertextBlocks";
    case 3: return "AliceShareCiphertexts";
    case 4: return "ActivationShareUp";
    case 5: return "ActivationShareDown";
    case 6: return "Done";
    case 7: return "Error";
  }
  return "?";
}

// Throws the REF exception for the first violation (if any).  `record` maps a
// record-area position to its message.
template <class RecordMsg>
void raise_first(uint64_t key, uint64_t frame_key, const uint8_t* frames, size_t stride, const char* layout_msg,
                 RecordMsg record) {
  if (key == ~0ull) return;
  const uint64_t f = key / frame_key, local = key % frame_key;
  const uint8_t* F = frames + f * stride;
  std::string where = " (frame " + std::to_string(f) + ")";
  switch (local) {
    case E_MAGIC: fail(ENSEI_ERR_MALFORMED_PAYLOAD, "bad magic" + where);
    case E_VERSION: fail(ENSEI_ERR_MALFORMED_PAYLOAD, "unsupported version" + where);
    case E_TYPE: fail(ENSEI_ERR_MALFORMED_PAYLOAD, "unknown message type" + where);
    case E_CAP: fail(ENSEI_ERR_MALFORMED_PAYLOAD, "payload length exceeds cap" + where);
    case E_LENGTH: fail(ENSEI_ERR_MALFORMED_PAYLOAD, "payload length mismatch" + where);
    case E_PEER: {
      uint64_t len = 0;
      uint8_t hdr[kFrameHdr];
      EG_CUDA(cudaMemcpy(hdr, F, kFrameHdr, cudaMemcpyDefault));
      for (int i = 0; i < 8; ++i) len |= (uint64_t)hdr[6 + i] << (8 * i);
      std::string msg(std::min<uint64_t>(len, 4096), '\0');
      if (!msg.empty()) EG_CUDA(cudaMemcpy(&msg[0], F + kFrameHdr, msg.size(), cudaMemcpyDefault));
      fail(ENSEI_ERR_PROTOCOL_ORDER, "peer aborted: " + msg);
    }
    case E_UNEXPECTED: {
      uint8_t t = 0;
      EG_CUDA(cudaMemcpy(&t, F + 5, 1, cudaMemcpyDefault));
      fail(ENSEI_ERR_PROTOCOL_ORDER, std::string("expected ") + record(~0ull) + ", got " + msg_name(t) + where);
    }
    case E_TRUNC_HDR: fail(ENSEI_ERR_MALFORMED_PAYLOAD, "truncated payload" + where);
    case E_LAYOUT: fail(ENSEI_ERR_PROTOCOL_ORDER, layout_msg + where);
    default: fail(ENSEI_ERR_MALFORMED_PAYLOAD, record(local - E_RECORDS) + where);
  }
}

void check_type(uint32_t t) {
  require(t >= 1 && t <= 7, ENSEI_ERR_INVALID_ARGUMENT, "unknown message type");
}

}  // namespace
}  // namespace ensei_gpu

using namespace ensei_gpu;

extern "C" {

uint64_t ensei_gpu_fnv1a(const uint8_t* data, size_t len, uint64_t seed) {
  uint64_t h = seed;
  for (size_t i = 0; i < len; ++i) {
    h ^= data[i];
    h *= 1099511628211ull;
  }
  return h;
}

size_t ensei_gpu_wire_ct_frame_bytes(uint32_t n, uint32_t channels, uint32_t blocks) {
  return kCtHdr + (size_t)channels * blocks * (9 + 16ull * n);
}

size_t ensei_gpu_wire_share_frame_bytes(uint32_t channels, uint32_t rows, uint32_t cols) {
  return kShareHdr + 8ull * channels * rows * cols;
}

int ensei_gpu_wire_encode_ct_blocks(ensei_gpu_ctx* ctx, uint32_t msg_type, uint32_t layer, uint32_t channels,
                                    uint32_t blocks, uint32_t domain, const uint64_t* d_ct, uint32_t num_frames,
                                    uint8_t* frames, size_t frame_stride, void* stream) {
  return guarded([&] {
    require(ctx && d_ct && frames, ENSEI_ERR_INVALID_ARGUMENT, "null argument");
    check_type(msg_type);
    require(domain <= 1, ENSEI_ERR_INVALID_ARGUMENT, "domain must be Coefficient (0) or Evaluation (1)");
    require(ctx->R == 1, ENSEI_ERR_UNSUPPORTED, "REF's wire format carries single-prime ciphertexts only");
    const size_t fb = ensei_gpu_wire_ct_frame_bytes(ctx->n, channels, blocks);
    require(frame_stride >= fb, ENSEI_ERR_INVALID_ARGUMENT, "frame_stride smaller than the frame");
    require(fb - kFrameHdr <= kMaxPayload, ENSEI_ERR_MALFORMED_PAYLOAD, "payload exceeds 1 GiB cap");
    const uint32_t recs = channels * blocks;
    if (!num_frames) return;
    require_accessible(frames, "frames");
    const cudaStream_t st = (cudaStream_t)stream;
    const size_t smem = 16ull * ctx->n;
    if (!recs) {  // header-only frames
      fail(ENSEI_ERR_UNSUPPORTED, "empty ciphertext-blocks messages are host-side frames");
    }
    EG_CUDA(cudaFuncSetAttribute(wire_encode_ct_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    wire_encode_ct_kernel<<<dim3(recs, num_frames), kThreads, smem, st>>>(
        d_ct, frames, frame_stride, ctx->logn, recs, domain == ENSEI_DOMAIN_EVALUATION, (uint8_t)domain,
        (uint8_t)msg_type, layer, channels, blocks);
    check_launch("wire_encode_ct_kernel");
  });
}

int ensei_gpu_wire_decode_ct_blocks(ensei_gpu_ctx* ctx, const uint8_t* frames, size_t frame_len,
                                    size_t frame_stride, uint32_t num_frames, uint32_t expect_type,
                                    uint32_t expect_channels, uint32_t expect_blocks, uint32_t* layer_out,
                                    uint64_t* d_ct, uint32_t* coeff_records, void* stream) {
  return guarded([&] {
    require(ctx && frames && d_ct, ENSEI_ERR_INVALID_ARGUMENT, "null argument");
    check_type(expect_type);
    require(ctx->R == 1, ENSEI_ERR_UNSUPPORTED, "REF's wire format carries single-prime ciphertexts only");
    require(num_frames <= 1 || frame_stride >= frame_len, ENSEI_ERR_INVALID_ARGUMENT,
            "frame_stride smaller than frame_len");
    if (coeff_records) *coeff_records = 0;
    if (!num_frames) return;
    require(frame_len >= kFrameHdr, ENSEI_ERR_MALFORMED_PAYLOAD, "frame shorter than header");
    const uint32_t recs = expect_channels * expect_blocks;
    require(recs > 0, ENSEI_ERR_UNSUPPORTED, "empty ciphertext-blocks messages are host-side frames");
    require_accessible(frames, "frames");
    const uint32_t n = ctx->n;
    const uint64_t rb = 9 + 16ull * n;
    const uint64_t avail = frame_len >= kCtHdr ? std::min<uint64_t>(recs, (frame_len - kCtHdr) / rb) : 0;
    const uint64_t frame_key = E_RECORDS + (uint64_t)recs * (2 * n + 2);
    const cudaStream_t st = (cudaStream_t)stream;
    std::lock_guard<std::mutex> lock(ctx->wire_mu);
    StatusView sv = status_view(ctx, num_frames, (uint64_t)num_frames * recs);
    reset_status(ctx, st);
    const size_t smem = 16ull * n;
    EG_CUDA(cudaFuncSetAttribute(wire_decode_ct_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    wire_decode_ct_kernel<<<dim3((unsigned)std::max<uint64_t>(avail, 1), num_frames), kThreads, smem, st>>>(
        frames, frame_len, frame_stride, ctx->logn, recs, (uint32_t)avail, expect_type, expect_channels,
        expect_blocks, ctx->q[0], sv, frame_key, d_ct);
    check_launch("wire_decode_ct_kernel");
    std::vector<uint8_t> head(16 + 4ull * num_frames);
    EG_CUDA(cudaMemcpyAsync(head.data(), ctx->wire_status, head.size(), cudaMemcpyDeviceToHost, st));
    EG_CUDA(cudaStreamSynchronize(st));
    uint64_t key, flags;
    std::memcpy(&key, head.data(), 8);
    std::memcpy(&flags, head.data() + 8, 8);
    const std::string layout = "ciphertext block layout mismatch";
    raise_first(key, frame_key, frames, frame_stride, layout.c_str(), [&](uint64_t pos) -> std::string {
      if (pos == ~0ull) return msg_name(expect_type);
      const uint64_t r = pos % (2 * n + 2);
      if (r == 0) return "bad domain tag";
      if (r == 1) return "ring dimension mismatch";
      return "coefficient out of range";
    });
    const uint64_t expect_len = ensei_gpu_wire_ct_frame_bytes(n, expect_channels, expect_blocks);
    if (frame_len < expect_len) fail(ENSEI_ERR_MALFORMED_PAYLOAD, "truncated payload");
    if (frame_len > expect_len) fail(ENSEI_ERR_MALFORMED_PAYLOAD, "trailing bytes in payload");
    if (layer_out) std::memcpy(layer_out, head.data() + 16, 4ull * num_frames);
    if (flags & 2) {  // Coefficient-domain records: to_evaluation_domain (REF ringbfv.cpp:308-324)
      const size_t total = (size_t)num_frames * recs;
      uint32_t nc = 0;
      if (!(flags & 1)) {
        int rc = ensei_gpu_negacyclic(ctx, 0, 0, ENSEI_LAYOUT_BITREV, d_ct, 2 * total, stream);
        if (rc) fail(rc, ensei_gpu_last_error());
        nc = (uint32_t)total;
      } else {
        std::vector<uint8_t> tags(total);
        EG_CUDA(cudaMemcpy(tags.data(), sv.tags, total, cudaMemcpyDeviceToHost));
        for (size_t r = 0; r < total;) {
          if (tags[r]) {
            ++r;
            continue;
          }
          size_t e = r;
          while (e < total && !tags[e]) ++e;
          int rc = ensei_gpu_negacyclic(ctx, 0, 0, ENSEI_LAYOUT_BITREV, d_ct + r * 2 * n, 2 * (e - r), stream);
          if (rc) fail(rc, ensei_gpu_last_error());
          nc += (uint32_t)(e - r);
          r = e;
        }
      }
      if (coeff_records) *coeff_records = nc;
    }
  });
}

int ensei_gpu_wire_encode_shares(ensei_gpu_ctx* ctx, uint32_t msg_type, uint32_t layer, uint32_t channels,
                                 uint32_t rows, uint32_t cols, const uint32_t* d_shares, uint32_t num_frames,
                                 uint8_t* frames, size_t frame_stride, void* stream) {
  return guarded([&] {
    require(ctx && frames, ENSEI_ERR_INVALID_ARGUMENT, "null argument");
    check_type(msg_type);
    const uint64_t cnt = (uint64_t)channels * rows * cols;
    require(cnt == 0 || d_shares, ENSEI_ERR_INVALID_ARGUMENT, "null argument");
    const size_t fb = ensei_gpu_wire_share_frame_bytes(channels, rows, cols);
    require(frame_stride >= fb, ENSEI_ERR_INVALID_ARGUMENT, "frame_stride smaller than the frame");
    require(fb - kFrameHdr <= kMaxPayload, ENSEI_ERR_MALFORMED_PAYLOAD, "payload exceeds 1 GiB cap");
    if (!num_frames) return;
    require_accessible(frames, "frames");
    const uint64_t words = cnt + 2;
    const unsigned gx = (unsigned)std::max<uint64_t>(
        1, std::min<uint64_t>((words + kThreads - 1) / kThreads, (uint64_t)ctx->sm_count * 8));
    wire_encode_shares_kernel<<<dim3(gx, num_frames), kThreads, 0, (cudaStream_t)stream>>>(
        d_shares, frames, frame_stride, cnt, (uint8_t)msg_type, layer, channels, rows, cols);
    check_launch("wire_encode_shares_kernel");
  });
}

int ensei_gpu_wire_decode_shares(ensei_gpu_ctx* ctx, const uint8_t* frames, size_t frame_len, size_t frame_stride,
                                 uint32_t num_frames, uint32_t expect_type, uint32_t expect_channels,
                                 uint32_t expect_rows, uint32_t expect_cols, uint64_t max_value,
                                 uint32_t* layer_out, uint32_t* d_shares, void* stream) {
  return guarded([&] {
    require(ctx && frames, ENSEI_ERR_INVALID_ARGUMENT, "null argument");
    check_type(expect_type);
    require(max_value <= (1ull << 32), ENSEI_ERR_INVALID_ARGUMENT, "max_value must be <= 2^32 (uint32 shares)");
    require(num_frames <= 1 || frame_stride >= frame_len, ENSEI_ERR_INVALID_ARGUMENT,
            "frame_stride smaller than frame_len");
    if (!num_frames) return;
    require(frame_len >= kFrameHdr, ENSEI_ERR_MALFORMED_PAYLOAD, "frame shorter than header");
    const uint64_t cnt = (uint64_t)expect_channels * expect_rows * expect_cols;
    require(cnt == 0 || d_shares, ENSEI_ERR_INVALID_ARGUMENT, "null argument");
    require_accessible(frames, "frames");
    const uint64_t avail = frame_len >= kShareHdr ? std::min<uint64_t>(cnt, (frame_len - kShareHdr) / 8) : 0;
    const uint64_t frame_key = E_RECORDS + cnt + 1;
    const cudaStream_t st = (cudaStream_t)stream;
    std::lock_guard<std::mutex> lock(ctx->wire_mu);
    StatusView sv = status_view(ctx, num_frames, 0);
    reset_status(ctx, st);
    const unsigned gx = (unsigned)std::max<uint64_t>(
        1, std::min<uint64_t>((avail + kThreads - 1) / kThreads, (uint64_t)ctx->sm_count * 8));
    wire_decode_shares_kernel<<<dim3(gx, num_frames), kThreads, 0, st>>>(
        frames, frame_len, frame_stride, cnt, avail, expect_type, expect_channels, expect_rows, expect_cols,
        max_value, sv, frame_key, d_shares);
    check_launch("wire_decode_shares_kernel");
    std::vector<uint8_t> head(16 + 4ull * num_frames);
    EG_CUDA(cudaMemcpyAsync(head.data(), ctx->wire_status, head.size(), cudaMemcpyDeviceToHost, st));
    EG_CUDA(cudaStreamSynchronize(st));
    uint64_t key;
    std::memcpy(&key, head.data(), 8);
    raise_first(key, frame_key, frames, frame_stride, "share layout mismatch", [&](uint64_t pos) -> std::string {
      if (pos == ~0ull) return msg_name(expect_type);
      return "share value out of range";
    });
    const uint64_t expect_len = ensei_gpu_wire_share_frame_bytes(expect_channels, expect_rows, expect_cols);
    if (frame_len < expect_len) fail(ENSEI_ERR_MALFORMED_PAYLOAD, "truncated payload");
    if (frame_len > expect_len) fail(ENSEI_ERR_MALFORMED_PAYLOAD, "trailing bytes in payload");
    if (layer_out) std::memcpy(layer_out, head.data() + 16, 4ull * num_frames);
  });
}

}  // extern "C"
