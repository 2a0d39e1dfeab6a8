/*
 * ensei_oracle.h -- CPU ORACLE.  TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference ENSEI hot path
 * (/root/reference/proj/core, "REF" below) used as the CHECKER for the
 * B200 product path.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  The product library
 * (paper_2003_05328_b200/libensei_gpu.so) never links or calls it.
 *
 * Parity pins:
 *   - every transform, Enc/Dec/ElementMult/HomShare/HomRec step is checked
 *     bit-exactly against the compiled reference (oracle/_ref/libensei_ref.so,
 *     built from the read-only REF sources by oracle/Makefile) and against the
 *     committed golden fixtures in tests/golden/;
 *   - the mt19937_64 stream and samplers are checked against REF's Rng so the
 *     "parity mode" randomness injected into the GPU path is the reference's
 *     own randomness;
 *   - the counter-based (Philox4x32-10) samplers, CBD noise, ternary secret and
 *     RNS/CRT decryption are builder extensions with no REF counterpart
 *     ("parity unpinned" for ciphertext bits in those modes; the reconstructed
 *     convolution outputs are still pinned by REF's reference_pipeline).
 *
 * Layouts: every array is dense row-major uint64_t (Residue), exactly the
 * reference's std::vector<Residue> layouts; evaluation-domain polynomials are
 * in the reference's NATURAL slot order (slot k = x(psi^(2k+1))).
 */
#ifndef ENSEI_ORACLE_H
#define ENSEI_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- L0: prime-field arithmetic (REF modfield.hpp:35-69, modfield.cpp) ---- */
uint64_t eo_mulmod(uint64_t a, uint64_t b, uint64_t m);
uint64_t eo_addmod(uint64_t a, uint64_t b, uint64_t m);
uint64_t eo_submod(uint64_t a, uint64_t b, uint64_t m);
uint64_t eo_powmod(uint64_t b, uint64_t e, uint64_t m);
uint64_t eo_invmod(uint64_t a, uint64_t m);
int eo_is_prime(uint64_t n);
/* smallest primitive root (REF modfield.cpp:143-152) */
uint64_t eo_primitive_root(uint64_t p);
/* canonical g^((p-1)/order); 0 if order does not divide p-1 (REF modfield.cpp:167-171) */
uint64_t eo_root_of_unity(uint64_t order, uint64_t p);
/* smallest prime >= min with prime == residue mod modulus; 0 if none < 2^62 (REF modfield.cpp:173-183) */
uint64_t eo_find_prime(uint64_t min_value, uint64_t residue, uint64_t modulus);
uint64_t eo_encode_signed(int64_t v, uint64_t p);   /* REF modfield.cpp:185-190 */
int64_t eo_decode_signed(uint64_t r, uint64_t p);   /* REF modfield.cpp:192-196 */

/* ---- L1: transforms ---- */
/* natural-in/natural-out radix-2 DIT with wtab[k] = omega^k (REF ntt_kernel.hpp:11-33) */
void eo_ntt_pow2(uint64_t* x, size_t n, const uint64_t* wtab, uint64_t m);
/* y_k = sum x_i omega^{ik}; inverse scales by L^-1 (REF ntt.cpp:83-108). 0 ok, <0 error */
int eo_ntt_1d(uint64_t* x, size_t n, uint64_t omega, uint64_t m, int inverse);
/* separable 2D transform rows-then-columns with canonical roots (REF ntt.cpp:112-153) */
int eo_ntt_2d(uint64_t* x, size_t rows, size_t cols, uint64_t m, int inverse);
/* psi-twisted negacyclic transform, natural order both sides (REF ringbfv.cpp:30-59) */
typedef struct eo_plan eo_plan;
eo_plan* eo_plan_create(uint64_t m, uint32_t n);
void eo_plan_destroy(eo_plan* p);
uint64_t eo_plan_psi(const eo_plan* p);
void eo_plan_forward(const eo_plan* p, uint64_t* x);
void eo_plan_inverse(const eo_plan* p, uint64_t* x);
/* convenience: builds a plan per call */
int eo_negacyclic(uint64_t* x, uint32_t n, uint64_t m, int inverse, size_t count);

/* ---- randomness: counter-based Philox4x32-10 (builder extension) ---- */
void eo_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
/* splitmix64 finalizer and Rng::fork seed derivation (REF modfield.cpp:79-85, 221-223) */
uint64_t eo_mix64(uint64_t x);
uint64_t eo_fork_seed(uint64_t seed, uint64_t salt);
/* stream id of one polynomial's worth of draws */
uint64_t eo_stream_id(uint32_t purpose, uint32_t layer, uint32_t image, uint32_t channel, uint32_t block);
enum { EO_PURPOSE_SECRET = 1, EO_PURPOSE_NOISE = 2, EO_PURPOSE_AHAT = 3, EO_PURPOSE_SHARE = 4, EO_PURPOSE_RESHARE = 5 };
void eo_rand_ternary(uint64_t key, uint64_t stream, uint32_t n, int64_t* out);
void eo_rand_cbd(uint64_t key, uint64_t stream, uint32_t n, uint32_t k, int64_t* out);
void eo_rand_uniform_q(uint64_t key, uint64_t stream, uint32_t n, uint64_t q, uint64_t* out);
void eo_rand_uniform_p(uint64_t key, uint64_t stream, uint32_t n, uint64_t p, uint64_t* out);

/* ---- reference Rng restatement: mt19937_64 + samplers (REF modfield.hpp:104-130, modfield.cpp:198-223) ---- */
typedef struct {
  uint64_t mt[312];
  uint32_t idx;
  uint64_t seed;
} eo_mt;
void eo_mt_seed(eo_mt* r, uint64_t seed);
uint64_t eo_mt_next(eo_mt* r);
void eo_mt_fork(const eo_mt* parent, uint64_t salt, eo_mt* child);
uint64_t eo_mt_uniform_below(eo_mt* r, uint64_t bound);
int64_t eo_mt_gaussian(eo_mt* r, double sigma);

/* ---- L2/L3: one conv layer of the protocol (builder batched restatement) ---- */
typedef struct {
  uint64_t q, p;            /* ciphertext modulus, unified p = p_N = p_A = p_E */
  uint32_t n;               /* ring degree */
  uint32_t H, W, fh, fw;    /* image and filter dims */
  uint32_t same;            /* 1 = ConvType::Same, 0 = Valid */
  uint32_t cin, cout;
  /* derived by eo_layer_init (REF ntt.cpp:51-81, protocol.cpp:162-193) */
  uint32_t Lh, Lw, blocks, oh, ow, r0, c0;
  uint64_t delta;           /* floor(q / p) (REF ringbfv.cpp:80) */
  /* packing (builder extension, the device's ensei_conv_desc::pack): images per
     ciphertext block, 1 = REF geometry.  With pack = k > 1 (one block per channel,
     k Lh Lw <= n) image i of a pack owns slots [i Lh Lw, (i + 1) Lh Lw); the per-image
     arrays below (in, bob_prev, bob_share, alice_share) then hold k images
     ([k][channels][..]) and the filter grid is replicated across the pack. */
  uint32_t pack;
} eo_layer;
int eo_layer_init(eo_layer* L, uint64_t q, uint64_t p, uint32_t n, uint32_t H, uint32_t W,
                  uint32_t fh, uint32_t fw, uint32_t same, uint32_t cin, uint32_t cout);

/* t (signed coeffs) -> t_eval = NTT_q(t) (REF ringbfv.cpp:95-107) */
void eo_secret_eval(const eo_layer* L, const int64_t* t, uint64_t* t_eval);
/* w[cout][cin][fh][fw] signed -> w_eval[cout][cin][B][n] (REF protocol.cpp:462-502, ringbfv.cpp:265-280) */
void eo_prepare_weights(const eo_layer* L, const int64_t* w, uint64_t* w_eval);
/* Alice, one image: in[cin][H][W] residues mod p; e[cin][B][n], a_hat[cin][B][n];
   ct[cin][B][2][n] (REF protocol.cpp:310-329, ringbfv.cpp:180-201) */
void eo_alice_encrypt(const eo_layer* L, const uint64_t* t_eval, const uint64_t* in,
                      const int64_t* e, const uint64_t* a_hat, uint64_t* ct);
/* Bob, one image: optional HomRec with bob_prev[cin][H][W] (NULL for layer 0), ElementMult
   + channel add, HomShare with s_b[cout][B][n]; ct_out[cout][B][2][n],
   bob_share[cout][oh][ow] (REF protocol.cpp:537-607, hss.cpp:22-62) */
void eo_bob_eval(const eo_layer* L, const uint64_t* ct_in, const uint64_t* w_eval,
                 const uint64_t* bob_prev, const uint64_t* s_b, uint64_t* ct_out,
                 uint64_t* bob_share);
/* Alice, one image: decrypt + merge + IDFT2D + crop (REF protocol.cpp:332-355, ringbfv.cpp:203-231) */
void eo_alice_decrypt(const eo_layer* L, const uint64_t* t_eval, const uint64_t* ct_out,
                      uint64_t* alice_share);
/* plaintext ground truth for one image: conv_oracle + channel sum mod p
   (REF ntt.cpp:197-226, protocol.cpp:705-730) */
void eo_conv_direct(const eo_layer* L, const uint64_t* in, const int64_t* w, uint64_t* out);
/* activation on centered lifts: fn 0 = ReLU, 1 = Square, 2 = Identity (REF protocol.cpp:731-747) */
int eo_activation(uint64_t* v, size_t len, uint64_t p, int fn);

/* ---- RNS (config 4; builder extension, unpinned) ---- */
/* Alice decrypt over an RNS chain: Ls[r] = the layer with q = q_r (delta unused),
   t_evals[r][n], ct_out[cout][B][2][R][n] (natural order); exact CRT rounding. */
void eo_alice_decrypt_rns(const eo_layer* Ls, uint32_t R, const uint64_t* t_evals,
                          const uint64_t* ct_out, uint64_t* alice_share);
/* exact CRT rounding: m = round(p * phi / Q) mod p for phi given by residues mod q_i */
uint64_t eo_crt_round(const uint64_t* res, const uint64_t* qs, uint32_t R, uint64_t p);

#ifdef __cplusplus
}
#endif
#endif
