/*
 * ensei_gpu.h -- C ABI of the B200-native ENSEI hot path (libensei_gpu.so).
 *
 * The reference (/root/reference/proj/core, "REF") exposes a C++ operator API in
 * namespace ensei; it has no C ABI and no GPU code.  This header is the thin
 * extern "C" layer the C++ host mirror (paper_2003_05328_b200/csrc/host/
 * ensei_b200.hpp) and the Python ctypes binding call.  Every entry point names
 * the REF interface it replaces.  Conventions:
 *
 *  - Plain pointers and sizes only.  Pointers named d_* are DEVICE pointers
 *    (caller-allocated, caller-owned; no hidden allocations on hot calls);
 *    h_* are host pointers.  `stream` is a cudaStream_t (NULL = legacy stream).
 *  - Return value: 0 on success, else an ensei_status code that maps 1:1 onto
 *    the REF exception hierarchy (REF errors.hpp:7-37); ensei_gpu_last_error()
 *    gives the message (thread-local).
 *  - Residues mod p travel as uint32 (p < 2^30); residues mod q as uint64.
 *  - Evaluation-domain polynomials mod q live on the device in BIT-REVERSED slot
 *    order ("device layout", like SEAL's NTT form).  ensei_gpu_permute() converts
 *    to/from REF's natural slot order (slot k = x(psi^(2k+1))), which is what the
 *    wire format and REF's ciphertexts use.
 *  - Ciphertext array layout: [... ][2 (c0,c1)][R primes][n].  With R = 1 this is
 *    REF's (c0 || c1) wire payload (REF wire.cpp:112-117) minus the tag and n.
 */
#ifndef ENSEI_GPU_H
#define ENSEI_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ENSEI_GPU_ABI_VERSION 3

typedef enum {
  ENSEI_OK = 0,
  ENSEI_ERR_GENERIC = 1,            /* ensei::Error */
  ENSEI_ERR_ORDER_NOT_DIVIDING = 2, /* ensei::OrderNotDividing */
  ENSEI_ERR_SEARCH_EXHAUSTED = 3,   /* ensei::SearchExhausted */
  ENSEI_ERR_BAD_ROOT = 4,           /* ensei::BadRoot */
  ENSEI_ERR_BAD_GEOMETRY = 5,       /* ensei::BadGeometry */
  ENSEI_ERR_GEOMETRY_MISMATCH = 6,  /* ensei::GeometryMismatch */
  ENSEI_ERR_DOMAIN_MISMATCH = 7,    /* ensei::DomainMismatch */
  ENSEI_ERR_NOISE_EXHAUSTED = 8,    /* ensei::NoiseExhausted */
  ENSEI_ERR_CHAIN_VIOLATION = 9,    /* ensei::ChainViolation */
  ENSEI_ERR_LENGTH_MISMATCH = 10,   /* ensei::LengthMismatch */
  ENSEI_ERR_RANGE_VIOLATION = 11,   /* ensei::RangeViolation */
  ENSEI_ERR_PROTOCOL_ORDER = 12,    /* ensei::ProtocolOrderViolation */
  ENSEI_ERR_RANGE_OVERFLOW = 13,    /* ensei::RangeOverflow */
  ENSEI_ERR_MALFORMED_PAYLOAD = 14, /* ensei::MalformedPayload */
  ENSEI_ERR_TRANSPORT = 15,         /* ensei::TransportError */
  ENSEI_ERR_CUDA = 100,             /* CUDA runtime / launch failure */
  ENSEI_ERR_UNSUPPORTED = 101,      /* valid for REF, not (yet) on this path */
  ENSEI_ERR_INVALID_ARGUMENT = 102  /* null pointer, bad enum */
} ensei_status;

const char* ensei_gpu_last_error(void);
int ensei_gpu_abi_version(void);

/* ------------------------------------------------------------- context */
typedef struct ensei_gpu_ctx ensei_gpu_ctx;

#define ENSEI_MAX_PRIMES 4
#define ENSEI_MOD_P 0xFFFFFFFFu /* selects the plaintext/image modulus p */

/* RlweParams + ModulusChain::unified (REF ringbfv.cpp:65-87, hss.cpp:7-20):
 * q = product of num_q NTT-friendly primes (num_q = 1 is REF's single-prime q;
 * num_q > 1 is the RNS extension for large runs), p = p_N = p_A = p_E.
 * Checks REF's invariants: every prime q_i and p are prime, == 1 mod 2n,
 * q_i == 1 mod p, q > p; throws (returns) ENSEI_ERR_GENERIC otherwise.
 * Builds canonical-root twiddle tables on `device`.
 * Threading: a context owns an auxiliary stream, fork / join events, the cached host-entry
 * graph and the wire status block; calls on ONE context must not overlap in time (two host
 * threads, or two streams whose work can run concurrently).  Use one context per
 * concurrently working party / stream; contexts are independent of each other. */
int ensei_gpu_ctx_create(int device, uint32_t n, const uint64_t* q_primes, uint32_t num_q,
                         uint64_t p, ensei_gpu_ctx** out);
void ensei_gpu_ctx_destroy(ensei_gpu_ctx* ctx);

typedef struct {
  uint32_t n, num_q;
  uint64_t q[ENSEI_MAX_PRIMES];
  uint64_t p;
  uint64_t delta[ENSEI_MAX_PRIMES]; /* floor(Q/p) mod q_i  (REF ringbfv.cpp:80, Q = prod q_i) */
  uint64_t psi_q[ENSEI_MAX_PRIMES]; /* canonical 2n-th roots (REF NegacyclicPlan::psi) */
  uint64_t psi_p;
  int device, sm_count;
} ensei_ctx_info;
int ensei_gpu_ctx_query(const ensei_gpu_ctx* ctx, ensei_ctx_info* info);

/* ---------------------------------------------------- single transforms */
#define ENSEI_LAYOUT_NATURAL 0 /* REF slot order */
#define ENSEI_LAYOUT_BITREV 1  /* device evaluation layout */

/* NegacyclicPlan::forward / ::inverse (REF ringbfv.cpp:49-59) over `count`
 * contiguous length-n polynomials, in place.  modulus = prime index i < num_q
 * (uint64 residues mod q_i) or ENSEI_MOD_P (uint64 residues mod p; this is
 * encode_slots/decode_slots, REF ringbfv.cpp:109-125).  eval_layout selects the
 * order of the evaluation side (output of forward, input of inverse).
 * Inputs must be canonical residues; outputs are canonical. */
int ensei_gpu_negacyclic(ensei_gpu_ctx* ctx, uint32_t modulus, int inverse, int eval_layout,
                         uint64_t* d_data, size_t count, void* stream);

/* ntt_2d / intt_2d (REF ntt.cpp:139-153): separable 2D cyclic transform over p
 * with canonical roots, natural order on both sides, `count` rows x cols tiles
 * (uint64 residues), in place.  rows, cols: powers of two in [1, 64]. */
int ensei_gpu_ntt2d(ensei_gpu_ctx* ctx, int inverse, uint32_t rows, uint32_t cols,
                    uint64_t* d_data, size_t count, void* stream);

/* natural <-> bit-reversed order of `count` length-n uint64 polynomials */
int ensei_gpu_permute(ensei_gpu_ctx* ctx, int to_natural, uint64_t* d_data, size_t count,
                      void* stream);

/* ------------------------------------------------------- conv layers */
typedef struct {
  uint32_t H, W;   /* input tile (REF ConvGeometry image_h/w) */
  uint32_t fh, fw; /* filter */
  uint32_t same;   /* 1 = ConvType::Same, 0 = Valid */
  uint32_t cin, cout;
  /* Ciphertext packing (builder extension; 0 or 1 = REF's geometry, one image per
   * ciphertext block).  pack = k (a power of two) puts k images' padded grids into one
   * block, slots [i G, (i + 1) G) = image i of the pack (needs one block per channel and
   * k G <= n); weights are replicated across the pack.  Every slot-wise step (ElementMult,
   * channel sum, HomShare, Dec) is unchanged, so the outputs are REF's; the ciphertexts
   * are the oracle's packed restatement.  Arrays of ciphertexts then hold
   * ceil(num_images / k) "ciphertext images"; image arrays stay per image.  Packed layers
   * take Philox randomness with a pack-aligned image_base and one shared key. */
  uint32_t pack;
  /* Padded grid side (builder extension, ABI 3; 0 = REF's choice, choose_padded_len: the
   * next power of two).  REF pads H + fh - 1 to a power of two for its own radix-2
   * transform; any length L >= max(H + fh - 1, W + fw - 1) dividing p - 1 holds the linear
   * convolution (REF itself falls back to such lengths, with its O(L^2) ntt_direct, when no
   * power of two divides p - 1: ntt.cpp:51-61).  A non-power-of-two grid runs the direct
   * transform on the device too and lets more images share a block (32x32 images, 3x3
   * filter, p - 1 = 2^14 39: L = 39, five images per n = 8192 block instead of two).
   * Outputs are REF's; ciphertexts are the oracle's restatement with the same grid.
   * Supported: the 3-prime RNS layer at n = 8192 with L = 39, and single-prime layers at
   * n = 2048 with L = 39, 24 or 12 (HomRec included); Philox randomness; any pack with
   * pack L^2 <= n whose tiles fit the kernels' shared memory (12 images of a 12x12 grid). */
  uint32_t grid;
} ensei_conv_desc;

typedef struct {
  uint32_t Lh, Lw;   /* padded grid (REF make_geometry, ntt.cpp:65-81) */
  uint32_t blocks;   /* ciphertext blocks per channel, ceil(Lh*Lw/n) (REF protocol.cpp:180) */
  uint32_t oh, ow;   /* output tile */
  uint32_t r0, c0;   /* crop origin (REF ntt.hpp:44-49) */
  uint32_t pack;     /* images per ciphertext block (1: REF geometry) */
} ensei_layer_geom;

/* make_geometry + plan_layers' block count. ENSEI_ERR_BAD_GEOMETRY as REF. */
int ensei_gpu_layer_geometry(const ensei_gpu_ctx* ctx, const ensei_conv_desc* desc,
                             ensei_layer_geom* geom);

#define ENSEI_RAND_PHILOX 0   /* device counter-based streams (throughput mode) */
#define ENSEI_RAND_INJECTED 1 /* caller-supplied draws (parity mode: REF's Rng stream) */

typedef struct {
  uint32_t mode;
  uint32_t layer;      /* layer field of the stream ids */
  uint32_t image_base; /* global index of the batch's first image (sharding-invariant) */
  uint32_t cbd_k;      /* centered-binomial parameter for Enc noise (Philox mode) */
  uint64_t alice_key;  /* Philox key of Alice's streams (Rng(seed).fork(0xA11CE) seed) */
  uint64_t bob_key;    /* Philox key of Bob's streams   (Rng(seed).fork(0xB0B) seed) */
  /* injected mode (natural slot order, per image / channel / block):           */
  const int32_t* d_noise;  /* e0   [img][cin][B][n]   signed                    */
  const uint64_t* d_a_hat; /* a^   [img][cin][B][R][n] canonical mod q_i        */
  const uint32_t* d_share; /* s_B  [img][cout][B][n]  canonical mod p           */
} ensei_randomness;

/* Secret-key blob: ENSEI_KEY_WORDS(n, R) uint64 = per prime [t_eval (device layout),
 * Shoup companions floor(t_eval 2^64 / q_i)].  keygen's t_eval = NTT_q(t)
 * (REF ringbfv.cpp:95-107) from signed coefficients d_t[n]: */
#define ENSEI_KEY_WORDS(n, R) (2u * (uint32_t)(R) * (uint32_t)(n))
int ensei_gpu_secret_from_coeffs(ensei_gpu_ctx* ctx, const int64_t* d_t, uint64_t* d_key,
                                 void* stream);
/* ternary secret sampled from Philox (key = Alice key) -> t (optional) and the blob */
int ensei_gpu_secret_sample(ensei_gpu_ctx* ctx, uint64_t alice_key, int64_t* d_t,
                            uint64_t* d_key, void* stream);

/* BobSession::prepare_weights + prepare_plain (REF protocol.cpp:462-502,
 * ringbfv.cpp:265-280) for one layer: d_w[cout][cin][fh][fw] signed int32
 * filter taps -> d_w_eval[cout][cin][B][R][n] uint64 in device layout (bit-reversed
 * slots; each word packs the canonical value v as (v >> 30) << 32 | (v & (2^30-1)),
 * the limb split the ElementMult accumulator uses).  t_setup, not on the online path. */
int ensei_gpu_prepare_weights(ensei_gpu_ctx* ctx, const ensei_conv_desc* desc, const int32_t* d_w,
                              uint64_t* d_w_eval, void* stream);
/* ABI 2: the prepared-weights buffer is the packed words above FOLLOWED, for layers with
 * 32 <= cin <= the context's int8 K limit, by the byte planes of the tcgen05 ElementMult
 * (built once here, at t_setup, instead of on every call).  Its size: */
size_t ensei_gpu_prepared_weights_bytes(const ensei_gpu_ctx* ctx, const ensei_conv_desc* desc);
/* (Re)build the byte planes of a prepared-weights buffer from its packed words -- for
 * callers that write the words themselves. */
int ensei_gpu_prepare_weight_planes(ensei_gpu_ctx* ctx, const ensei_conv_desc* desc, uint64_t* d_w_eval,
                                    void* stream);

#define ENSEI_IN_U32 0 /* residues mod p */
#define ENSEI_IN_U8 1  /* raw pixels (encode_signed of a non-negative value) */

/* ------------------------------------------------ per-block operators
 * REF's ringbfv / hss operators for `count` independent blocks per call (REF calls them
 * one block at a time; csrc/host/ensei_b200.hpp wraps them with REF's C++ signatures).
 * Slot / coefficient vectors: uint64 residues, REF natural order, [count][n].
 * Ciphertexts: [count][2][R][n] device layout (ensei_gpu_permute <-> REF order).
 * Prepared plains: [count][R][n] packed words (as ensei_gpu_prepare_weights).
 * d_work: ensei_gpu_ops_workspace_bytes(ctx, count). */
size_t ensei_gpu_ops_workspace_bytes(const ensei_gpu_ctx* ctx, size_t count);
/* encrypt_freq_direct (REF ringbfv.cpp:180-201): c0 = -a^, c1 = a^ t^ + NTT_q(Delta
 * encode(m) + e); e (d_noise [count][n] signed) and a^ (d_a_hat [count][R][n], natural
 * slot order, canonical) are the caller's draws (REF's Rng: n Gaussians, then n
 * uniform mod q per block). */
int ensei_gpu_encrypt_freq_direct(ensei_gpu_ctx* ctx, const uint64_t* d_slots, const uint64_t* d_key,
                                  const int64_t* d_noise, const uint64_t* d_a_hat, size_t count, uint64_t* d_ct,
                                  void* d_work, void* stream);
/* decrypt (REF ringbfv.cpp:203-231), evaluation-domain ciphertexts; three-prime contexts
 * round with the exact CRT of the RNS decryption */
int ensei_gpu_decrypt(ensei_gpu_ctx* ctx, const uint64_t* d_ct, const uint64_t* d_key, size_t count,
                      uint64_t* d_slots, void* d_work, void* stream);
/* prepare_plain (REF ringbfv.cpp:265-280): d_w_eval [count][R][n] packed words; h_w_inf
 * (nullable, host, [count]) = REF's w_inf (max |centered coefficient|, at least 1) --
 * synchronous on `stream` when given */
int ensei_gpu_prepare_plain(ensei_gpu_ctx* ctx, const uint64_t* d_slots, size_t count, uint64_t* d_w_eval,
                            double* h_w_inf, void* d_work, void* stream);
/* mul_plain's slot-wise product (REF ringbfv.cpp:282-306; the static noise check is the
 * host's, see ensei_b200.hpp): d_out = [d_out +] d_ct o w -- with accumulate = 1 this
 * is add_ct(acc, mul_plain(ct, w)), REF's channel sum (protocol.cpp:570-581) */
int ensei_gpu_mul_plain(ensei_gpu_ctx* ctx, const uint64_t* d_ct, const uint64_t* d_w_eval, size_t count,
                        int accumulate, uint64_t* d_out, void* stream);
/* add_ct (REF ringbfv.cpp:233-246): d_out = d_a + d_b */
int ensei_gpu_add_ct(ensei_gpu_ctx* ctx, const uint64_t* d_a, const uint64_t* d_b, size_t count, uint64_t* d_out,
                     void* stream);
/* add_plain (REF ringbfv.cpp:248-263), evaluation domain, in place: c1 +- NTT_q(Delta
 * encode(m)); with m = (p_A - s_B) mod p_e this is hom_share_with, with m = s_B hom_rec
 * (REF hss.cpp:22-62) */
int ensei_gpu_add_plain(ensei_gpu_ctx* ctx, uint64_t* d_ct, const uint64_t* d_slots, int sign, size_t count,
                        void* d_work, void* stream);

/* AliceSession::send_encrypted for `num_images` images (REF protocol.cpp:310-329):
 * pad -> DFT2D -> flatten/split -> encrypt_freq_direct (REF ringbfv.cpp:180-201),
 * fused in one kernel.  d_in[img][cin][H][W]; d_key = key blob(s), key_stride = 0
 * (one key) or ENSEI_KEY_WORDS (per-image keys); d_ct[img][cin][B][2][R][n] in
 * device layout. */
int ensei_gpu_alice_encrypt(ensei_gpu_ctx* ctx, const ensei_conv_desc* desc,
                            const uint64_t* d_t_eval, uint32_t key_stride, const void* d_in,
                            int in_dtype, uint32_t num_images, const ensei_randomness* rand,
                            uint64_t* d_ct, void* stream);

/* BobSession conv branch (REF protocol.cpp:537-607): optional HomRec with Bob's
 * previous share d_bob_prev[img][cin][H][W] (NULL for the first layer), then
 * ElementMult + channel accumulation (mul_plain/add_ct, REF ringbfv.cpp:233-306)
 * with lazy 128-bit accumulation, then HomShare (REF hss.cpp:22-49) and Bob's
 * share IDFT2D + crop.  d_ct_out[img][cout][B][2][R][n] (device layout),
 * d_bob_share[img][cout][oh][ow].  With d_bob_prev, HomRec updates d_ct in place
 * (as REF's BobSession updates its received blocks, protocol.cpp:552-555). */
int ensei_gpu_bob_eval(ensei_gpu_ctx* ctx, const ensei_conv_desc* desc, uint64_t* d_ct,
                       const uint64_t* d_w_eval, const uint32_t* d_bob_prev, uint32_t num_images,
                       const ensei_randomness* rand, uint64_t* d_ct_out, uint32_t* d_bob_share,
                       void* stream);

/* The two halves of ensei_gpu_bob_eval, separately: hom_share batched over
 * (img, out channel, block) -- writes the HomShare masks NTT_q(Delta*INTT_p(p - s_B))
 * into the c1 words of d_ct_out and Bob's cropped share into d_bob_share
 * (REF hss.cpp:22-49, protocol.cpp:587-603) -- and the ElementMult + channel
 * accumulation that adds the products onto those masks (REF ringbfv.cpp:233-306). */
int ensei_gpu_bob_share(ensei_gpu_ctx* ctx, const ensei_conv_desc* desc, uint32_t num_images,
                        const ensei_randomness* rand, uint64_t* d_ct_out, uint32_t* d_bob_share,
                        void* stream);
int ensei_gpu_bob_mac(ensei_gpu_ctx* ctx, const ensei_conv_desc* desc, const uint64_t* d_ct,
                      const uint64_t* d_w_eval, uint32_t num_images, uint64_t* d_ct_out,
                      void* stream);

/* AliceSession::receive_shares (REF protocol.cpp:332-355): decrypt (REF
 * ringbfv.cpp:203-231) -> merge -> IDFT2D -> crop, fused.  d_alice_share
 * [img][cout][oh][ow]. */
int ensei_gpu_alice_decrypt(ensei_gpu_ctx* ctx, const ensei_conv_desc* desc,
                            const uint64_t* d_t_eval, uint32_t key_stride, const uint64_t* d_ct_out,
                            uint32_t num_images, uint32_t* d_alice_share, void* stream);

/* trusted_activation (REF protocol.cpp:237-268) for a batch of share tensors
 * [img][channels][H][W]: recombine mod p, centered lift, fn (0 ReLU, 1 Square,
 * 2 Identity), optional 2x2 max-pool (pool2 = 1: builder extension for the 32->16->8
 * spatial steps of config 3; output [img][channels][H/2][W/2]), re-share with fresh
 * randomness (Alice's reshare stream, or rand->d_share injected [img][ch][out]).
 * Square overflow (|y|^2 > p/2, REF RangeOverflow) sets *d_overflow != 0 (nullable). */
int ensei_gpu_activation(ensei_gpu_ctx* ctx, int fn, int pool2, uint32_t channels, uint32_t H,
                         uint32_t W, uint32_t num_images, const uint32_t* d_a, const uint32_t* d_b,
                         const ensei_randomness* rand, uint32_t* d_new_a, uint32_t* d_new_b,
                         int* d_overflow, void* stream);

/* ElementMult implementation (tuning / A-B testing; results are identical):
 * -1 automatic (default), 0 the 4-product IMAD kernel, 1 the Karatsuba IMAD kernel,
 * 2 the int8 mma.sync kernel on byte planes, 3 the same with in-kernel planes, 5 the
 * tcgen05 kernel (the int8 paths: exact byte-plane products, cin <= the context's
 * K (q_i - 1)^2 < 2^128 limit; 5 also needs 32 <= cin). */
int ensei_gpu_set_mac_variant(int variant);

/* Tile kernels (Enc / HomShare / Dec) of the 3-prime RNS layer at n = 8192 (tuning / A-B
 * testing; results are identical): 1 (default) the 512-thread kernels, two CTAs per SM
 * (csrc/layer_rns.cuh); 0 the first-generation 1024-thread kernels (csrc/layer.cuh). */
int ensei_gpu_set_tile_variant(int variant);

/* Which ElementMult kernel a conv layer of `num_images` images takes on this context
 * (the automatic choice, or the forced variant): */
#define ENSEI_MAC_IMAD4 0       /* 4-product IMAD tile kernel (mac_kernel) */
#define ENSEI_MAC_KARATSUBA 1   /* Karatsuba IMAD tile kernel (mac_kara_kernel) */
#define ENSEI_MAC_I8_PLANES 2   /* int8 tensor cores on byte planes (planes_kernel + mac_i8p_kernel) */
#define ENSEI_MAC_I8_DIRECT 3   /* int8 tensor cores, in-kernel plane split (mac_i8_kernel) */
#define ENSEI_MAC_DIRECT 4      /* per-slot direct kernel for 1-4 channels (mac_direct_kernel) */
#define ENSEI_MAC_TCGEN05 5     /* tcgen05.mma kind::i8, TMEM accumulators (planes_tc_kernel + mac_tc_kernel) */
int ensei_gpu_mac_path(const ensei_gpu_ctx* ctx, const ensei_conv_desc* desc, uint32_t num_images, int* path);

/* The RNS decryption rounding alone (three-prime contexts): for `count` residue triples
 * d_res[count][3] (phi mod q_0, q_1, q_2, canonical) -> d_out = round(p phi / Q) mod p
 * exactly as REF's decrypt rounds (ringbfv.cpp:224-229, floor((p phi + floor(Q/2)) / Q)),
 * by the same device code the RNS decryption kernel runs (test hook for the exactness
 * of its fixed-point fast path + multi-limb fallback). */
int ensei_gpu_crt_round(ensei_gpu_ctx* ctx, const uint64_t* d_res, size_t count, uint32_t* d_out, void* stream);

/* recombine_clear (REF hss.cpp:64-73): out = (a + b) mod p */
int ensei_gpu_recombine(ensei_gpu_ctx* ctx, const uint32_t* d_a, const uint32_t* d_b, size_t count,
                        uint32_t* d_out, void* stream);

/* Whole oblivious conv layer for a batch (Alice Enc -> Bob -> Alice Dec ->
 * recombine), the batched equivalent of one conv step of run_inproc
 * (REF protocol.cpp:670-692).  Workspace: ensei_gpu_conv_workspace_bytes() -- both
 * parties' ciphertexts, Bob's share and the ElementMult scratch (int8 byte planes), so
 * a call (or a CUDA graph captured around it) touches no context-owned buffer that can
 * be reallocated.  The workspace-less entry points (ensei_gpu_bob_eval / _bob_mac)
 * keep their byte planes in a context buffer grown on demand outside stream capture.
 * Threading: a context (its auxiliary stream, fork/join events, scratch and wire status
 * block) serves one conv-layer call at a time; concurrent calls from several host
 * threads need one context each (the wire decoders alone are serialised internally). */
size_t ensei_gpu_conv_workspace_bytes(const ensei_gpu_ctx* ctx, const ensei_conv_desc* desc,
                                      uint32_t num_images);
/* Batches larger than this stream through the workspace in sub-batches of this many
 * images (<= 12 GiB of ciphertexts; a multiple of 64 once that many fit: config 4 runs
 * 1024 images as 8 x 128); the workspace functions size for one sub-batch. */
uint32_t ensei_gpu_conv_chunk_images(const ensei_gpu_ctx* ctx, const ensei_conv_desc* desc, uint32_t num_images);
int ensei_gpu_conv_layer(ensei_gpu_ctx* ctx, const ensei_conv_desc* desc, const uint64_t* d_t_eval,
                         uint32_t key_stride, const uint64_t* d_w_eval, const void* d_in,
                         int in_dtype, const uint32_t* d_bob_prev, uint32_t num_images,
                         const ensei_randomness* rand, void* d_workspace, uint32_t* d_alice_share,
                         uint32_t* d_bob_share, uint32_t* d_out, void* stream);

/* Same with HOST buffers, synchronous on `stream`.  Pinned (page-locked) buffers
 * are read / written by the kernels in place across the host link (zero-copy:
 * the transfers overlap the layer); pageable buffers are staged through
 * d_workspace, which must hold the staging input/output
 * (ensei_gpu_conv_host_workspace_bytes()).  The launch sequence is captured
 * into a CUDA graph on first use and replayed while every argument is
 * unchanged. */
size_t ensei_gpu_conv_host_workspace_bytes(const ensei_gpu_ctx* ctx, const ensei_conv_desc* desc,
                                           uint32_t num_images, int in_dtype);
int ensei_gpu_conv_layer_host(ensei_gpu_ctx* ctx, const ensei_conv_desc* desc,
                              const uint64_t* d_t_eval, const uint64_t* d_w_eval, const void* h_in,
                              int in_dtype, uint32_t num_images, const ensei_randomness* rand,
                              void* d_workspace, uint32_t* h_out, void* stream);

/* --------------------------------------------------- reference randomness */
/* REF Rng (modfield.hpp:104-130, modfield.cpp:198-223) on the host: mt19937_64,
 * fork(salt) = Rng(mix64(seed ^ mix64(salt))) (AliceSession salt 0xA11CE, BobSession
 * 0xB0B, protocol.cpp:285,454), masked-rejection uniform_below, 6-sigma-tail discrete
 * Gaussian.  Feeding its draws, in REF's consumption order, through
 * ensei_randomness's injected pointers reproduces the reference bit for bit. */
typedef struct ensei_ref_rng ensei_ref_rng;
int ensei_gpu_ref_rng_create(uint64_t seed, int use_fork, uint64_t salt, ensei_ref_rng** out);
void ensei_gpu_ref_rng_destroy(ensei_ref_rng* rng);
int ensei_gpu_ref_rng_next_u64(ensei_ref_rng* rng, uint64_t* h_out, size_t count);
int ensei_gpu_ref_rng_uniform_below(ensei_ref_rng* rng, uint64_t bound, uint64_t* h_out,
                                    size_t count);
int ensei_gpu_ref_rng_gaussian(ensei_ref_rng* rng, double sigma, int64_t* h_out, size_t count);

/* ------------------------------------------------------------ parameters */
/* REF PrecisionProfile (params.hpp:11-17) */
typedef struct {
  int32_t input_bits, filter_bits, f_h, f_w;
} ensei_precision_profile;

#define ENSEI_CHAIN_UNIFIED 0     /* REF ChainMode::Unified */
#define ENSEI_CHAIN_SPLIT_PAPER 1 /* REF ChainMode::SplitPaper */

/* REF ParamSet (params.hpp:27-34): ModulusChain + RlweParams moduli.  num_q = 1 is
 * REF's single-prime q; num_q > 1 is the RNS extension (q = product of q[0..num_q)). */
typedef struct {
  uint64_t p_n, p_a, p_e;
  uint32_t n, num_q;
  uint64_t q[ENSEI_MAX_PRIMES];
  double sigma;
  double log2_q_min; /* derive_q's requirement (REF params.cpp:49-60), log2 */
  uint32_t mode, insecure;
  ensei_precision_profile profile;
} ensei_param_set;

/* min_pntt (REF params.cpp:79-89); ENSEI_ERR_RANGE_VIOLATION as REF */
int ensei_gpu_min_pntt(const ensei_precision_profile* profile, uint64_t* out);

/* build_params (REF params.cpp:91-117) + derive_q.  max_primes = 1 reproduces REF
 * exactly (ENSEI_ERR_SEARCH_EXHAUSTED when q would reach 2^62, e.g. >= ~100-way channel
 * accumulation at n = 2048); max_primes > 1 switches to an RNS chain of the smallest
 * primes >= 2^59 that are == 1 (mod 2n p_e) when -- and only when -- REF's single
 * prime runs out (min_primes forces at least that many RNS primes). */
int ensei_gpu_build_params(const ensei_precision_profile* profile, uint32_t n, uint32_t mode,
                           uint64_t accum_channels, uint64_t p_n_floor, double sigma,
                           uint32_t max_primes, uint32_t min_primes, ensei_param_set* out);

/* preset_params (REF params.cpp:119-144): "binary", "medium", "high", "toy" */
int ensei_gpu_preset_params(const char* name, uint64_t accum_channels, uint32_t max_primes,
                            ensei_param_set* out);

/* ---------------------------------------------------------- wire framing */
/* REF wire format (wire.hpp:17-80, wire.cpp:44-144, protocol.cpp:83-150):
 *   frame  = "ENSE" | 0x01 | type (1) | payload length (8, LE) | payload
 *   ciphertext-blocks payload (encode_ct_blocks) = layer (4) | channels (4) |
 *            blocks (4) | per [channel][block]: domain tag (1) | n (8) |
 *            c0 (n x 8) | c1 (n x 8), natural slot order
 *   shares payload (encode_shares) = layer (4) | channels (4) | rows (4) |
 *            cols (4) | channels x rows x cols residues (8 each)
 * all little-endian.  The frames are built / parsed by kernels straight from / into
 * the device layouts above, so a frame never takes a host-side serialisation pass;
 * `frames` may be device memory or page-locked host memory (read / written in place
 * across the host link), never pageable memory.  Batched: `num_frames` frames (one
 * per image session) at a fixed byte stride. */
#define ENSEI_MSG_HELLO 0x01
#define ENSEI_MSG_CIPHERTEXT_BLOCKS 0x02
#define ENSEI_MSG_ALICE_SHARE_CIPHERTEXTS 0x03
#define ENSEI_MSG_ACTIVATION_SHARE_UP 0x04
#define ENSEI_MSG_ACTIVATION_SHARE_DOWN 0x05
#define ENSEI_MSG_DONE 0x06
#define ENSEI_MSG_ERROR 0x07
#define ENSEI_DOMAIN_COEFFICIENT 0 /* REF RingDomain::Coefficient (ringbfv.hpp:10) */
#define ENSEI_DOMAIN_EVALUATION 1  /* REF RingDomain::Evaluation */

/* whole-frame sizes (header included) */
size_t ensei_gpu_wire_ct_frame_bytes(uint32_t n, uint32_t channels, uint32_t blocks);
size_t ensei_gpu_wire_share_frame_bytes(uint32_t channels, uint32_t rows, uint32_t cols);

/* encode_frame(encode_ct_blocks(type, layer, cts)) (REF protocol.cpp:83-97,
 * wire.cpp:44-55,112-117) for num_frames messages of channels x blocks ciphertexts
 * (single prime).  d_ct[frame][channel][block][2][n]: with domain =
 * ENSEI_DOMAIN_EVALUATION the polynomials are in device layout (bit-reversed) and
 * are written in REF's natural slot order; with ENSEI_DOMAIN_COEFFICIENT they are
 * coefficient-domain polynomials in natural order (REF Baseline-mode ciphertexts,
 * e.g. after ensei_gpu_negacyclic inverse) and are written as they are. */
int ensei_gpu_wire_encode_ct_blocks(ensei_gpu_ctx* ctx, uint32_t msg_type, uint32_t layer,
                                    uint32_t channels, uint32_t blocks, uint32_t domain,
                                    const uint64_t* d_ct, uint32_t num_frames, uint8_t* frames,
                                    size_t frame_stride, void* stream);

/* decode_frame + recv_expect + decode_ct_blocks (REF wire.cpp:57-79,119-144,
 * protocol.cpp:55-65,99-117) of num_frames frames of frame_len bytes each, into
 * d_ct[frame][channel][block][2][n] in device layout (evaluation domain).  Records
 * tagged Coefficient (REF Baseline mode) are moved to the evaluation domain on the
 * way in (REF BobSession's to_evaluation_domain, protocol.cpp:562-566, ringbfv.cpp:
 * 308-324); *coeff_records (nullable) = how many there were (REF counts 2 ct_ntt
 * each).  Synchronous on `stream`.  Errors exactly as REF: MalformedPayload (header,
 * domain tag, ring dimension, coefficient >= q, truncated / trailing bytes),
 * ProtocolOrderViolation (Error frame from the peer, unexpected type, layout
 * mismatch); the first violation in REF's read order wins.  layer_out[num_frames]
 * (nullable, host) receives each frame's layer field. */
int ensei_gpu_wire_decode_ct_blocks(ensei_gpu_ctx* ctx, const uint8_t* frames, size_t frame_len,
                                    size_t frame_stride, uint32_t num_frames, uint32_t expect_type,
                                    uint32_t expect_channels, uint32_t expect_blocks,
                                    uint32_t* layer_out, uint64_t* d_ct, uint32_t* coeff_records,
                                    void* stream);

/* encode_frame(encode_shares(type, layer, mats)) (REF protocol.cpp:119-132):
 * d_shares[frame][channels][rows][cols] uint32 residues -> u64 LE on the wire. */
int ensei_gpu_wire_encode_shares(ensei_gpu_ctx* ctx, uint32_t msg_type, uint32_t layer,
                                 uint32_t channels, uint32_t rows, uint32_t cols,
                                 const uint32_t* d_shares, uint32_t num_frames, uint8_t* frames,
                                 size_t frame_stride, void* stream);

/* decode_frame + recv_expect + decode_shares (REF protocol.cpp:134-150): values
 * must be < max_value (<= 2^32; REF passes p_a) else MalformedPayload("share value
 * out of range").  Synchronous on `stream`. */
int ensei_gpu_wire_decode_shares(ensei_gpu_ctx* ctx, const uint8_t* frames, size_t frame_len,
                                 size_t frame_stride, uint32_t num_frames, uint32_t expect_type,
                                 uint32_t expect_channels, uint32_t expect_rows,
                                 uint32_t expect_cols, uint64_t max_value, uint32_t* layer_out,
                                 uint32_t* d_shares, void* stream);

/* Host helper: REF fnv1a (wire.cpp:409-416), the transcript hash RecordingTransport
 * chains over every encoded frame (wire.cpp:336-352).  `data` is host memory. */
uint64_t ensei_gpu_fnv1a(const uint8_t* data, size_t len, uint64_t seed);

/* ------------------------------------------------------------ utilities */
/* Per-kernel CUDA-event timing of the layer kernels (a measurement pass: the events
 * are recorded on each kernel's own stream around every launch, never inside stream
 * capture, and serialise programmatic dependent launch).  enable = 1 clears and starts
 * recording, 0 stops; _read synchronises and returns, per kernel name (32-byte slots
 * in `names`), the summed milliseconds and the launch count. */
int ensei_gpu_profile(int enable);
int ensei_gpu_profile_read(uint32_t max_kernels, char* names, double* total_ms, uint32_t* launches,
                           uint32_t* num_kernels);

/* number of this library's kernels launched so far in the process */
uint64_t ensei_gpu_launch_count(void);
/* IMAD-pipe peak probe: returns IMAD slots/s (dependent mad.lo.u32 chains) measured on `device` */
double ensei_gpu_imad_peak(int device);
/* int8 tensor-core peak probe: u8 x u8 multiply-accumulates per second of back-to-back
 * tcgen05.mma.kind::i8 (M = 128, N = n_cols, K = 32) on every SM of `device` */
double ensei_gpu_tc_i8_peak(int device, uint32_t n_cols);

#ifdef __cplusplus
}
#endif
#endif /* ENSEI_GPU_H */
