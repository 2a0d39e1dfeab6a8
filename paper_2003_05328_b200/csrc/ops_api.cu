// ops_api.cu -- C ABI of the per-block operators (REF ringbfv.hpp / hss.hpp, one call
// for `count` blocks): encrypt_freq_direct, decrypt, prepare_plain, mul_plain, add_ct,
// add_plain.  The conv-layer entry points (layer_api.cu) fuse these into whole-layer
// kernels; these are the drop-in surface for a host that drives REF's operator calls
// itself (csrc/host/ensei_b200.hpp mirrors REF's signatures on top of them).
//
// Layouts: slot vectors and coefficient vectors are REF's natural order, uint64
// residues; ciphertexts [count][2 (c0, c1)][R][n] and prepared plains [count][R][n]
// (packed limbs, as ensei_gpu_prepare_weights) are the device evaluation layout
// (bit-reversed), ensei_gpu_permute converts.  Workspace: ensei_gpu_ops_workspace_bytes.
#include <algorithm>
#include <cstring>

#include "kernels.cuh"
#include "layer.cuh"

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

struct OpsConst {
  PrimeConst pc[ENSEI_MAX_PRIMES];
  CrtConst crt;
  uint32_t p, R, logn;
};

OpsConst ops_const(const ensei_gpu_ctx* c) {
  OpsConst k;
  std::memset(&k, 0, sizeof(k));
  for (uint32_t r = 0; r < c->R; ++r) k.pc[r] = c->pc[r];
  k.crt = c->crt;
  k.p = (uint32_t)c->p;
  k.R = c->R;
  k.logn = c->logn;
  return k;
}

unsigned grid_for(const ensei_gpu_ctx* c, size_t work) {
  return (unsigned)std::max<size_t>(1, std::min<size_t>((work + 255) / 256, (size_t)c->sm_count * 16));
}

#define OPS_LOOP(total) \
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < (total); idx += (size_t)gridDim.x * blockDim.x)

// Work buffers of R polynomials per block are prime-major, [r][b][n], so one batched
// transform call per prime covers every block.
// x[r][b][i] = Delta_r m[b][i] (+ e[b][i]) mod q_r, m = encode_slots output (< p), natural
// coefficient order (REF scale_message ringbfv.cpp:130-138 / add_plain's mask, :248-263)
__global__ void lift_kernel(OpsConst k, const uint64_t* m, const int64_t* e, int sign, size_t count, uint64_t* x) {
  const size_t n = (size_t)1 << k.logn;
  OPS_LOOP(count * k.R * n) {
    const size_t i = idx % n, b = (idx / n) % count, r = idx / (n * count);
    const Field64& f = k.pc[r].f;
    uint64_t v = f.mul(m[b * n + i] % k.p, k.pc[r].delta, k.pc[r].mu_hi, k.pc[r].mu_lo);
    if (sign < 0) v = f.neg(v);
    if (e) {
      const int64_t ev = e[b * n + i];
      v = f.add(v, ev < 0 ? f.q - (uint64_t)(-ev) % f.q : (uint64_t)ev % f.q);
    }
    x[idx] = v;
  }
}

// encrypt_freq_direct's last step (REF ringbfv.cpp:180-201), device layout: c0 = -a^,
// c1 = a^ t^ + x  (a^ given in natural slot order, position j = brev(k))
__global__ void enc_combine_kernel(OpsConst k, const uint64_t* key, const uint64_t* a_hat, const uint64_t* xs,
                                   size_t count, uint64_t* ct) {
  const size_t n = (size_t)1 << k.logn;
  OPS_LOOP(count * k.R * n) {
    const size_t j = idx % n, b = (idx / n) % count, r = idx / (n * count);
    const PrimeConst& pc = k.pc[r];
    const uint64_t a = a_hat[(b * k.R + r) * n + brev((int)j, (int)k.logn)];
    uint64_t* cb = ct + b * 2 * k.R * n;
    const uint64_t x = xs[idx];  // NTT_q(Delta m + e), device layout
    const uint64_t* tk = key + (2 * r) * n;
    const uint64_t at = Bfly<Field64, 0>::fin_gs(pc.f, pc.f.mul_shoup_approx(a, tk[j], tk[n + j]));
    cb[r * n + j] = pc.f.neg(a);
    cb[(k.R + r) * n + j] = pc.f.add(at, x);
  }
}

// phi_r = c0 t^ + c1 (device layout) into work[r][b][n]
__global__ void phi_kernel(OpsConst k, const uint64_t* ct, const uint64_t* key, size_t count, uint64_t* work) {
  const size_t n = (size_t)1 << k.logn;
  OPS_LOOP(count * k.R * n) {
    const size_t j = idx % n, b = (idx / n) % count, r = idx / (n * count);
    const PrimeConst& pc = k.pc[r];
    const uint64_t* cb = ct + b * 2 * k.R * n;
    const uint64_t* tk = key + (2 * r) * n;
    const uint64_t v = Bfly<Field64, 0>::fin_gs(pc.f, pc.f.mul_shoup_approx(cb[r * n + j], tk[j], tk[n + j]));
    work[idx] = pc.f.add(v, cb[(k.R + r) * n + j]);
  }
}

// round(p phi / Q) mod p per coefficient (REF ringbfv.cpp:222-229; RNS: the exact CRT
// rounding of layer.cuh -- every phi_r is at hand here, so its exact compare needs no
// recomputation)
__global__ void round_kernel(OpsConst k, const uint64_t* work, size_t count, uint64_t* out) {
  const size_t n = (size_t)1 << k.logn;
  OPS_LOOP(count * n) {
    const size_t i = idx % n, b = idx / n;
    if (k.R == 1) {
      const PrimeConst& pc = k.pc[0];
      const uint64_t phi = work[b * n + i];
      const uint64_t Q = mulhi64(phi, pc.cp);
      const uint64_t rem = (uint64_t)k.p * phi + (pc.f.q >> 1) - Q * pc.f.q;
      uint32_t v = (uint32_t)Q + (rem >= pc.f.q) + (rem >= pc.f.q2);
      out[idx] = v >= k.p ? v - k.p : v;
    } else {
      uint32_t Isum = 0;
      uint64_t Fsum = 0, E[3];
      for (int r = 0; r < 3; ++r) {
        uint32_t I;
        uint64_t F;
        crt_part(k.pc[r], k.p, work[((size_t)r * count + b) * n + i], I, E[r], F);
        Isum += I;
        Fsum += F;
      }
      uint32_t v = Isum + crt_round_t(k.crt, E, Fsum);
      if (v >= 2 * k.p) v -= 2 * k.p;
      if (v >= k.p) v -= k.p;
      out[idx] = v;
    }
  }
}

// prepare_plain's lift (REF ringbfv.cpp:265-280): centered integer of the p coefficient,
// embedded mod q_r; max |c| -> *winf (per block)
__global__ void plain_lift_kernel(OpsConst k, const uint64_t* m, size_t count, uint64_t* x, uint32_t* winf) {
  const size_t n = (size_t)1 << k.logn;
  OPS_LOOP(count * k.R * n) {
    const size_t i = idx % n, b = (idx / n) % count, r = idx / (n * count);
    const uint64_t v = m[b * n + i] % k.p;
    const bool neg = v > k.p / 2;
    const uint64_t mag = neg ? k.p - v : v;
    x[idx] = neg ? k.pc[r].f.q - mag : mag;
    if (r == 0) atomicMax(winf + b, (uint32_t)mag);
  }
}

// [r][b][n] canonical -> prepared-plain words [b][r][n], packed 30-bit limbs
__global__ void pack_kernel(OpsConst k, const uint64_t* x, size_t count, uint64_t* w) {
  const size_t n = (size_t)1 << k.logn;
  OPS_LOOP(count * k.R * n) {
    const size_t j = idx % n, b = (idx / n) % count, r = idx / (n * count);
    const uint64_t v = x[idx];
    w[(b * k.R + r) * n + j] = ((v >> 30) << 32) | (v & 0x3FFFFFFFull);
  }
}

// out = [out +] ct o w (both components; w packed limbs), REF mul_plain + add_ct
__global__ void mul_plain_kernel(OpsConst k, const uint64_t* ct, const uint64_t* w, size_t count, int accumulate,
                                 uint64_t* out) {
  const size_t n = (size_t)1 << k.logn;
  OPS_LOOP(count * 2 * k.R * n) {
    const size_t j = idx % n, r = (idx / n) % k.R, comp = (idx / (n * k.R)) % 2, b = idx / (2 * n * k.R);
    const PrimeConst& pc = k.pc[r];
    const uint64_t wp = w[(b * k.R + r) * n + j];
    const uint64_t wv = ((wp >> 32) << 30) | (wp & 0x3FFFFFFFull);
    uint64_t v = pc.f.mul(ct[idx], wv, pc.mu_hi, pc.mu_lo);
    if (accumulate) v = pc.f.add(v, out[idx]);
    (void)comp;
    out[idx] = v;
  }
}

__global__ void add_ct_kernel(OpsConst k, const uint64_t* a, const uint64_t* b, size_t count, uint64_t* out) {
  const size_t n = (size_t)1 << k.logn;
  OPS_LOOP(count * 2 * k.R * n) {
    const size_t r = (idx / n) % k.R;
    out[idx] = k.pc[r].f.add(a[idx], b[idx]);
  }
}

// c1 += x (device layout), add_plain's last step
__global__ void add_c1_kernel(OpsConst k, const uint64_t* x, size_t count, uint64_t* ct) {
  const size_t n = (size_t)1 << k.logn;
  OPS_LOOP(count * k.R * n) {
    const size_t j = idx % n, b = (idx / n) % count, r = idx / (n * count);
    uint64_t* c1 = ct + (b * 2 * k.R + k.R + r) * n;
    c1[j] = k.pc[r].f.add(c1[j], x[idx]);
  }
}

// encode_slots of `count` slot vectors into work (natural coefficients mod p, u64)
void encode(ensei_gpu_ctx* ctx, const uint64_t* slots, size_t count, uint64_t* work, cudaStream_t st) {
  EG_CUDA(cudaMemcpyAsync(work, slots, count * ctx->n * sizeof(uint64_t), cudaMemcpyDeviceToDevice, st));
  negacyclic(ctx, ENSEI_MOD_P, true, true, work, count, st);
}

// NTT_q (device layout on the evaluation side) of a prime-major [r][count][n] buffer
void ntt_q(ensei_gpu_ctx* ctx, uint64_t* x, size_t count, bool inverse, cudaStream_t st) {
  for (uint32_t r = 0; r < ctx->R; ++r) negacyclic(ctx, r, inverse, false, x + (size_t)r * count * ctx->n, count, st);
}

}  // namespace
}  // namespace ensei_gpu

using namespace ensei_gpu;

extern "C" {

size_t ensei_gpu_ops_workspace_bytes(const ensei_gpu_ctx* ctx, size_t count) {
  return ctx ? count * (ctx->R + 1) * ctx->n * sizeof(uint64_t) + ((count * sizeof(uint32_t) + 255) & ~(size_t)255) : 0;
}

int ensei_gpu_encrypt_freq_direct(ensei_gpu_ctx* ctx, const uint64_t* d_slots, const uint64_t* d_key,
                                  const int64_t* d_noise, const uint64_t* d_a_hat, size_t count, uint64_t* d_ct,
                                  void* d_work, void* stream) {
  return guarded([&] {
    require(ctx && d_key && d_noise && d_a_hat && (count == 0 || (d_slots && d_ct && d_work)),
            ENSEI_ERR_INVALID_ARGUMENT, "null argument");
    if (!count) return;
    cudaStream_t st = (cudaStream_t)stream;
    OpsConst k = ops_const(ctx);
    uint64_t* m = static_cast<uint64_t*>(d_work);
    encode(ctx, d_slots, count, m, st);
    // x = NTT_q(Delta m + e), prime-major, then c0 = -a^, c1 = a^ t^ + x
    uint64_t* x = m + count * ctx->n;
    lift_kernel<<<grid_for(ctx, count * ctx->R * ctx->n), 256, 0, st>>>(k, m, d_noise, 1, count, x);
    check_launch("lift_kernel");
    ntt_q(ctx, x, count, false, st);
    enc_combine_kernel<<<grid_for(ctx, count * ctx->R * ctx->n), 256, 0, st>>>(k, d_key, d_a_hat, x, count, d_ct);
    check_launch("enc_combine_kernel");
  });
}

int ensei_gpu_decrypt(ensei_gpu_ctx* ctx, const uint64_t* d_ct, const uint64_t* d_key, size_t count,
                      uint64_t* d_slots, void* d_work, void* stream) {
  return guarded([&] {
    require(ctx && d_key && (count == 0 || (d_ct && d_slots && d_work)), ENSEI_ERR_INVALID_ARGUMENT, "null argument");
    require(ctx->R == 1 || ctx->R == 3, ENSEI_ERR_UNSUPPORTED, "decrypt: one or three primes");
    if (!count) return;
    cudaStream_t st = (cudaStream_t)stream;
    OpsConst k = ops_const(ctx);
    uint64_t* phi = static_cast<uint64_t*>(d_work);
    phi_kernel<<<grid_for(ctx, count * ctx->R * ctx->n), 256, 0, st>>>(k, d_ct, d_key, count, phi);
    check_launch("phi_kernel");
    ntt_q(ctx, phi, count, true, st);  // device layout in, natural coefficients out
    round_kernel<<<grid_for(ctx, count * ctx->n), 256, 0, st>>>(k, phi, count, d_slots);
    check_launch("round_kernel");
    negacyclic(ctx, ENSEI_MOD_P, false, true, d_slots, count, st);  // decode_slots
  });
}

int ensei_gpu_prepare_plain(ensei_gpu_ctx* ctx, const uint64_t* d_slots, size_t count, uint64_t* d_w_eval,
                            double* h_w_inf, void* d_work, void* stream) {
  return guarded([&] {
    require(ctx && (count == 0 || (d_slots && d_w_eval && d_work)), ENSEI_ERR_INVALID_ARGUMENT, "null argument");
    if (!count) return;
    cudaStream_t st = (cudaStream_t)stream;
    OpsConst k = ops_const(ctx);
    uint64_t* m = static_cast<uint64_t*>(d_work);
    encode(ctx, d_slots, count, m, st);
    uint64_t* x = m + count * ctx->n;
    uint32_t* winf = reinterpret_cast<uint32_t*>(x + count * ctx->R * ctx->n);
    EG_CUDA(cudaMemsetAsync(winf, 0, count * sizeof(uint32_t), st));
    plain_lift_kernel<<<grid_for(ctx, count * ctx->R * ctx->n), 256, 0, st>>>(k, m, count, x, winf);
    check_launch("plain_lift_kernel");
    ntt_q(ctx, x, count, false, st);
    pack_kernel<<<grid_for(ctx, count * ctx->R * ctx->n), 256, 0, st>>>(k, x, count, d_w_eval);
    check_launch("pack_kernel");
    if (h_w_inf) {
      std::vector<uint32_t> w(count);
      EG_CUDA(cudaMemcpyAsync(w.data(), winf, count * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
      EG_CUDA(cudaStreamSynchronize(st));
      for (size_t b = 0; b < count; ++b) h_w_inf[b] = std::max(1.0, (double)w[b]);  // REF: max(w_inf, 1)
    }
  });
}

int ensei_gpu_mul_plain(ensei_gpu_ctx* ctx, const uint64_t* d_ct, const uint64_t* d_w_eval, size_t count,
                        int accumulate, uint64_t* d_out, void* stream) {
  return guarded([&] {
    require(ctx && (count == 0 || (d_ct && d_w_eval && d_out)), ENSEI_ERR_INVALID_ARGUMENT, "null argument");
    if (!count) return;
    OpsConst k = ops_const(ctx);
    mul_plain_kernel<<<grid_for(ctx, count * 2 * ctx->R * ctx->n), 256, 0, (cudaStream_t)stream>>>(
        k, d_ct, d_w_eval, count, accumulate, d_out);
    check_launch("mul_plain_kernel");
  });
}

int ensei_gpu_add_ct(ensei_gpu_ctx* ctx, const uint64_t* d_a, const uint64_t* d_b, size_t count, uint64_t* d_out,
                     void* stream) {
  return guarded([&] {
    require(ctx && (count == 0 || (d_a && d_b && d_out)), ENSEI_ERR_INVALID_ARGUMENT, "null argument");
    if (!count) return;
    OpsConst k = ops_const(ctx);
    add_ct_kernel<<<grid_for(ctx, count * 2 * ctx->R * ctx->n), 256, 0, (cudaStream_t)stream>>>(k, d_a, d_b, count,
                                                                                                   d_out);
    check_launch("add_ct_kernel");
  });
}

int ensei_gpu_add_plain(ensei_gpu_ctx* ctx, uint64_t* d_ct, const uint64_t* d_slots, int sign, size_t count,
                        void* d_work, void* stream) {
  return guarded([&] {
    require(ctx && (count == 0 || (d_ct && d_slots && d_work)), ENSEI_ERR_INVALID_ARGUMENT, "null argument");
    if (!count) return;
    cudaStream_t st = (cudaStream_t)stream;
    OpsConst k = ops_const(ctx);
    uint64_t* m = static_cast<uint64_t*>(d_work);
    encode(ctx, d_slots, count, m, st);
    uint64_t* x = m + count * ctx->n;
    lift_kernel<<<grid_for(ctx, count * ctx->R * ctx->n), 256, 0, st>>>(k, m, nullptr, sign, count, x);
    check_launch("lift_kernel");
    ntt_q(ctx, x, count, false, st);
    add_c1_kernel<<<grid_for(ctx, count * ctx->R * ctx->n), 256, 0, st>>>(k, x, count, d_ct);
    check_launch("add_c1_kernel");
  });
}

}  // extern "C"
