// mac_tc.cuh -- ElementMult + channel accumulation on the 5th-generation tensor cores
// (tcgen05.mma.kind::i8, accumulators in tensor memory).
//
// Same result as mac_kara_kernel / mac_i8p_kernel (REF mul_plain / add_ct,
// ringbfv.cpp:233-306, channel sum protocol.cpp:570-581, + the HomShare mask on c1):
// per slot s, out[row][col] = sum_k ct[row][k] w[k][col] mod q, rows = (image,
// component), cols = out channels, k = in channels.  Exact integer arithmetic by byte
// planes: x = sum_i x_i 2^(8i), y = sum_j y_j 2^(8j) (8 planes of u8 for residues < 2^64),
//     T = sum_k x y = sum_{d=0..14} 2^(8d) D_d,   D_d = sum_{i+j=d} sum_k x_i y_j,
// every D_d one u8 x u8 -> s32 tensor-core accumulation (8 K 255^2 < 2^31 for K <= 4127;
// T < 2^128 while K (q - 1)^2 < 2^128: ctx->i8_kmax).  64 byte-plane products per MAC.
//
// Operands (byte-plane tiles in the UMMA canonical K-major layout, SWIZZLE_NONE):
//   tile of T rows x 32*NK channel bytes, per plane [T/8 row groups][2*NK k16][8 rows][16 B]
//   -> core matrix (8 rows x 16 B) contiguous, LBO (next 16 k-bytes) = 128 B,
//      SBO (next 8 rows) = 2*NK*128 B; the 8 planes follow each other.
//   A (ciphertexts, planes_tc_kernel<128, false> once per call): blocks
//     ((kc * S + s) * nrb + rb), 128 rows (64 images x 2 components) per block;
//   B (weights, planes_tc_kernel<16, true> once at prepare time, stored after the packed
//     weight words): blocks ((kc * S + s) * nct + ct), 16 out channels per block.
//   S = B * R * n slots; kc = 32*NK-channel chunk of K (one chunk per launch).
//
// mac_tc_kernel: persistent, one CTA per SM, warp-specialised.
//   warp 0      producer: cp.async.bulk (TMA bulk copies, mbarrier completion) of a
//               unit's two A tiles and its 2 nct B tiles (ring of kTcBSt);
//   warp 1      allocates 512 TMEM columns; one elected lane issues tcgen05.mma: per
//               (slot, 16-column tile) 8 shifted-window MMAs x NK (128 x 128 x 32, the
//               first 128 x 240 x 32) into 15 diagonal blocks of 16 columns (240 columns;
//               two buffers, one per slot of the pair);
//   warps 2..17 epilogue: tcgen05.ld (32x32b.x4) of 15 diagonals x 4 columns (row = TMEM
//               lane; 4 warps per lane quarter), release the buffer, rebuild T, reduce
//               mod q_r once, add the mask / previous partial sum, one 16-byte store per
//               (row, column) and slot pair.
// unit = (128-row block, slot quad), quads fastest; CTA pairs walk the same contiguous
// range, one slot pair of each quad each.
#pragma once
#include "mac_i8.cuh"

namespace ensei_gpu {

constexpr int kTcRowsA = 128;  // rows of an A tile (UMMA M)
constexpr int kTcColsB = 16;   // out channels of a B tile (UMMA N)
constexpr int kTcDiag = 15;    // byte-product diagonals
constexpr int kTcBSt = 4;      // B ring depth
constexpr int kTcEpiWarps = 16;  // 4 per TMEM lane quarter, 4 of a tile's 16 columns each
constexpr int kTcThreads = 32 * (2 + kTcEpiWarps);

__host__ __device__ constexpr size_t tc_tile_bytes(int T, int nk) { return (size_t)8 * T * 32 * nk; }
__host__ __device__ constexpr int tc_nk(int K) { return K >= 64 ? 2 : (K + 31) / 32; }
__host__ __device__ constexpr int tc_nkc(int K) { return (K + 32 * tc_nk(K) - 1) / (32 * tc_nk(K)); }
__host__ __device__ inline size_t tc_planes_bytes(int S, int ntiles, int T, int K) {
  return (size_t)tc_nkc(K) * S * ntiles * tc_tile_bytes(T, tc_nk(K));
}

// ------------------------------------------------------------------ PTX wrappers
EG_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
EG_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
EG_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
EG_DEV void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
               : "memory");
}
// D[tmem] (+)= A[smem] x B[smem]^T, u8 x u8 -> s32; acc = 0 overwrites D
EG_DEV void tc_mma_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
// UMMA shared-memory descriptor: K-major, SWIZZLE_NONE, version 1 (sm_100)
EG_DEV uint64_t tc_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
// instruction descriptor: D s32, A/B u8, both K-major, M = 128, N = 16
__host__ __device__ constexpr uint32_t tc_idesc_i8(int M, int N) {
  return (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
EG_DEV void tc_ld8(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr));
}
EG_DEV void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }

// ------------------------------------------------------------------ byte planes
// One thread: 4 consecutive slots x 8 channels of one row (or out channel) -> for each
// slot and plane the 8 channel bytes, one 8-byte store (lanes cover whole core matrices).
// WEIGHTS: source = packed prepared weights [cout][cin][B][R][n]; else ciphertexts
// [img][cin][B][2][R][n] with row = 2 img + component.  Rows / channels past the ends
// are zero.  T = tile rows (128: A, 16: B); tiles indexed as documented above.
template <int T, bool WEIGHTS>
__global__ void __launch_bounds__(256) planes_tc_kernel(LayerArgs a, int logn, int R, const uint64_t* __restrict__ src,
                                                        uint8_t* __restrict__ dst, int nrc) {
  const int n = 1 << logn, K = a.cin, nk = tc_nk(K), nkc = tc_nkc(K);
  const long S = (long)a.B * R * n;
  const int ntiles = (nrc + T - 1) / T;
  const int octs = 4 * nk;  // 8-channel groups per chunk
  const long per_tile = (long)T * octs;
  const long total = (S / 4) * ntiles * nkc * per_tile;
  const size_t ctw = (size_t)2 * R * n, chan_stride = (size_t)a.B * ctw, w_chan = (size_t)a.B * R * n;
  const size_t tile_bytes = tc_tile_bytes(T, nk), plane_bytes = tile_bytes / 8;
  const uint32_t sbo = 2u * nk * 128u;
  constexpr uint64_t M30 = (1ull << 30) - 1;
  pdl_wait();  // launched programmatically after Enc / HomRec: their ciphertexts
  pdl_trigger();
  for (long it = (long)blockIdx.x * 256 + threadIdx.x; it < total; it += (long)gridDim.x * 256) {
    // lane-friendly decomposition: slot-quad parity, row%8, octet%2 | row/8, octet/2, tile,
    // slot-quad pair, chunk.  A store instruction covers two whole 128-byte core matrices,
    // and the two lanes of a slot-quad pair read one contiguous 64-byte run per (row,
    // channel) (32-byte reads cost a 64-byte DRAM access each: 2x read traffic, measured)
    long rest = it;
    const int sq0 = (int)(rest & 1);
    rest >>= 1;
    const int m8 = (int)(rest & 7);
    rest >>= 3;
    const int o2 = (int)(rest & 1);
    rest >>= 1;
    const int mg = (int)(rest % (T / 8));
    rest /= (T / 8);
    const int oh = (int)(rest % (octs / 2));
    rest /= (octs / 2);
    const int tile = (int)(rest % ntiles);
    rest /= ntiles;
    const long sq = (rest % (S / 8)) * 2 + sq0;
    const int kc = (int)(rest / (S / 8));
    const int m = mg * 8 + m8, o = oh * 2 + o2;
    const int rc = tile * T + m;             // global row (or out channel)
    const long s0 = sq * 4;                  // first of 4 slots (same bp: n % 4 == 0)
    const int bp = (int)(s0 >> logn), b = bp / R, r = bp % R, j0 = (int)(s0 & (n - 1));
    uint32_t lo[8][4], hi[8][4];
#pragma unroll
    for (int c8 = 0; c8 < 8; ++c8) {
      const int c = kc * 32 * nk + o * 8 + c8;
      ulonglong2 v0 = make_ulonglong2(0, 0), v1 = make_ulonglong2(0, 0);
      const bool ok = rc < nrc && c < K;
      if (ok) {
        const uint64_t* p = WEIGHTS ? src + ((size_t)rc * a.cin + c) * w_chan + (size_t)bp * n + j0
                                    : src + ((size_t)(rc >> 1) * a.cin + c) * chan_stride + (size_t)b * ctw +
                                          (size_t)((rc & 1) * R + r) * n + j0;
        v0 = __ldg(reinterpret_cast<const ulonglong2*>(p));
        v1 = __ldg(reinterpret_cast<const ulonglong2*>(p) + 1);
        if constexpr (WEIGHTS) {  // packed 30-bit limbs -> canonical value
          v0.x = ((v0.x >> 32) << 30) | (v0.x & M30);
          v0.y = ((v0.y >> 32) << 30) | (v0.y & M30);
          v1.x = ((v1.x >> 32) << 30) | (v1.x & M30);
          v1.y = ((v1.y >> 32) << 30) | (v1.y & M30);
        }
      }
      lo[c8][0] = lo32(v0.x), hi[c8][0] = hi32(v0.x);
      lo[c8][1] = lo32(v0.y), hi[c8][1] = hi32(v0.y);
      lo[c8][2] = lo32(v1.x), hi[c8][2] = hi32(v1.x);
      lo[c8][3] = lo32(v1.y), hi[c8][3] = hi32(v1.y);
    }
    const size_t off = (size_t)mg * sbo + (size_t)(o >> 1) * 128 + (size_t)m8 * 16 + (size_t)(o & 1) * 8;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint8_t* t = dst + (((size_t)kc * S + s0 + q) * ntiles + tile) * tile_bytes + off;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint32_t w0 = i < 4 ? plane_word(lo[0][q], lo[1][q], lo[2][q], lo[3][q], i)
                                  : plane_word(hi[0][q], hi[1][q], hi[2][q], hi[3][q], i - 4);
        const uint32_t w1 = i < 4 ? plane_word(lo[4][q], lo[5][q], lo[6][q], lo[7][q], i)
                                  : plane_word(hi[4][q], hi[5][q], hi[6][q], hi[7][q], i - 4);
        *reinterpret_cast<uint2*>(t + (size_t)i * plane_bytes) = make_uint2(w0, w1);
      }
    }
  }
}

// ------------------------------------------------------------------ the MAC
struct TcShared {
  uint64_t a_full, a_empty;
  uint64_t b_full[kTcBSt], b_empty[kTcBSt];
  uint64_t t_full[2], t_empty[2];
  uint32_t tmem_base;
};

// B stage = the 8 planes of a tile (128 rows of the shifted-window operand, see the MMA
// loop) + 7 planes' worth of zero rows (the 240-row operand of the first MMA)
template <int NK>
constexpr size_t tc_bstage_bytes() {
  return tc_tile_bytes(kTcColsB, NK) / 8 * (2 * 8 - 1);
}
template <int NK>
constexpr size_t tc_smem_bytes() {
  return 1024 + 2 * tc_tile_bytes(kTcRowsA, NK) + kTcBSt * tc_bstage_bytes<NK>();
}

EG_DEV void ld_v2(const uint64_t* p, uint64_t& x, uint64_t& y) {
  const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(p);
  x = v.x;
  y = v.y;
}
EG_DEV void tc_ld4(uint32_t taddr, uint32_t* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
               : "r"(taddr));
}

// T = P0 + 2^32 P1 + 2^64 P2 + 2^96 P3 (P_L = sum_q 2^(8q) D_(4L+q) < 2^51) -> T mod q_r,
// canonical (T < 2^128)
EG_DEV uint64_t tc_reduce(const Field64& f, const PrimeConst& pc, uint64_t P0, uint64_t P1, uint64_t P2, uint64_t P3) {
  uint64_t c64 = P0;
  const uint32_t t0 = lo32(c64);
  c64 = (c64 >> 32) + P1;
  const uint32_t t1 = lo32(c64);
  c64 = (c64 >> 32) + P2;
  const uint32_t t2 = lo32(c64);
  c64 = (c64 >> 32) + P3;
  const uint32_t t3 = lo32(c64);
  const uint64_t lo = ((uint64_t)t1 << 32) | t0, hi = ((uint64_t)t3 << 32) | t2;
  const uint64_t x = Bfly<Field64, 0>::corr(f, lo, pc.cred) + f.mul_shoup_approx(hi, pc.c64, pc.c64p);  // < 7q
  return Bfly<Field64, 0>::fin_ct(f, x, pc.cred);
}

// One launch = one 32*NK-channel chunk kc of K.  unit = (128-row block rb, slot pair):
// both slots' A tiles are resident (single buffer); per 16-column tile ct the two slots
// run back to back into the two TMEM buffers.  Output: the slot-major product
// Y[s][rb][128 rows][nct*16 cols] (T mod q), every unit one contiguous 128-row block --
// the ciphertext layout's slot-innermost order made the epilogue's stores scattered
// 8-byte (or 16-byte) writes, DRAM-bound at ~40 G sectors/s (measured: 18-45 ms per
// config-4 chunk).  mac_out_kernel transposes Y into that layout and adds the HomShare
// mask.  Later K chunks (kc > 0) add onto Y.
template <int NK, int R>
__global__ void __launch_bounds__(kTcThreads, 1)
    mac_tc_kernel(LayerArgs a, int logn, const uint8_t* __restrict__ Ap, const uint8_t* __restrict__ Bp, int kc,
                  uint64_t* __restrict__ Y, int rows, int cols) {
  extern __shared__ __align__(1024) uint8_t tc_smem[];
  TcShared& sh = *reinterpret_cast<TcShared*>(tc_smem);
  constexpr size_t A_BYTES = tc_tile_bytes(kTcRowsA, NK), B_BYTES = tc_tile_bytes(kTcColsB, NK);
  constexpr size_t BST = tc_bstage_bytes<NK>();
  constexpr uint32_t A_PLANE = (uint32_t)A_BYTES / 8;
  constexpr uint32_t SBO = 2u * NK * 128u, LBO = 128u;
  // shifted-window MMAs: A_i x [B_0 .. B_7] (N = 128) lands plane pair (i, j) in column
  // block i + j when D starts at block i -- one MMA per A plane instead of eight
  constexpr uint32_t IDESC128 = tc_idesc_i8(kTcRowsA, 8 * kTcColsB);
  constexpr uint32_t IDESC240 = tc_idesc_i8(kTcRowsA, kTcDiag * kTcColsB);
  constexpr int TCOLS = kTcDiag * kTcColsB;  // 240 TMEM columns per accumulator buffer
  uint8_t* a_buf = tc_smem + 1024;            // [slot of the pair][A tile]
  uint8_t* b_buf = a_buf + 2 * A_BYTES;
  const int n = 1 << logn;
  const long S = (long)a.B * R * n, SQ = S / 4;
  // rows = the A operand's side (128-row tiles), cols = the B operand's (16-row tiles): the
  // ciphertext rows and the out channels, or the other way round (mac_api.cu tc_swap)
  const int nrb = (rows + kTcRowsA - 1) / kTcRowsA, nct = (cols + kTcColsB - 1) / kTcColsB;
  // CTA pairs (2k, 2k+1) walk the same range of (row block, slot quad) units, CTA 2k the
  // quad's first slot pair, 2k+1 its second: the two halves of every 32-byte output sector
  // are written at about the same time (one CTA per slot quad left half-written sectors
  // in L2 long enough to be evicted: 2x DRAM write traffic, measured)
  const int npair = gridDim.x / 2, pi = blockIdx.x >> 1, half_q = blockIdx.x & 1;
  const long units = SQ * nrb;
  const long u0 = units * pi / npair, u1 = units * (pi + 1) / npair;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  for (int st = 0; st < kTcBSt; ++st)  // the zero rows after every B stage's tile (never overwritten)
    for (uint32_t off = threadIdx.x * 16; off < BST - B_BYTES; off += kTcThreads * 16)
      *reinterpret_cast<uint4*>(b_buf + st * BST + B_BYTES + off) = make_uint4(0, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic-proxy zeros -> tensor-core reads
  if (threadIdx.x == 0) {
    mbar_init(&sh.a_full, 1);
    mbar_init(&sh.a_empty, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sh.t_full[i], 1);
      mbar_init(&sh.t_empty[i], kTcEpiWarps);
    }
    for (int i = 0; i < kTcBSt; ++i) {
      mbar_init(&sh.b_full[i], 1);
      mbar_init(&sh.b_empty[i], 1);
    }
  }
  if (warp == 1) {  // whole warp: allocate 512 TMEM columns (two 240-column buffers)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&sh.tmem_base))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sh.tmem_base;
  pdl_wait();  // ciphertext planes (and masks) from the preceding kernels
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {  // ---- producer
      long bc = 0;
      for (long u = u0; u < u1; ++u) {
        const long s0 = 4 * (u % SQ) + 2 * half_q;
        const int rb = (int)(u / SQ);
        mbar_wait(&sh.a_empty, (uint32_t)(((u - u0) & 1) ^ 1));
        mbar_expect_tx(&sh.a_full, (uint32_t)(2 * A_BYTES));
        for (int p = 0; p < 2; ++p) {
          const uint8_t* asrc = Ap + (((size_t)kc * S + s0 + p) * nrb + rb) * A_BYTES;
          for (uint32_t off = 0; off < A_BYTES; off += 32768u)
            tma_bulk_g2s(a_buf + p * A_BYTES + off, asrc + off, (uint32_t)min((size_t)32768u, A_BYTES - off),
                         &sh.a_full);
        }
        for (int ct = 0; ct < nct; ++ct)
          for (int p = 0; p < 2; ++p, ++bc) {
            const int st = (int)(bc % kTcBSt);
            mbar_wait(&sh.b_empty[st], (uint32_t)(((bc / kTcBSt) & 1) ^ 1));
            mbar_expect_tx(&sh.b_full[st], (uint32_t)B_BYTES);
            tma_bulk_g2s(b_buf + st * BST, Bp + (((size_t)kc * S + s0 + p) * nct + ct) * B_BYTES, (uint32_t)B_BYTES,
                         &sh.b_full[st]);
          }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer
      long bc = 0, tc = 0;
      const uint32_t a_base = smem_u32(a_buf), b_base = smem_u32(b_buf);
      for (long u = u0; u < u1; ++u) {
        mbar_wait(&sh.a_full, (uint32_t)((u - u0) & 1));
        for (int ct = 0; ct < nct; ++ct)
          for (int p = 0; p < 2; ++p, ++bc, ++tc) {
            const int st = (int)(bc % kTcBSt), tb = (int)(tc & 1);
            mbar_wait(&sh.b_full[st], (uint32_t)((bc / kTcBSt) & 1));
            mbar_wait(&sh.t_empty[tb], (uint32_t)(((tc >> 1) & 1) ^ 1));
            tc_fence_after();
            const uint32_t acc0 = tmem + (uint32_t)(tb * TCOLS);
            const uint32_t a0 = a_base + p * (uint32_t)A_BYTES, b0 = b_base + st * (uint32_t)BST;
            // plane 0 first, over all 240 columns (B_0..B_7 then zero rows): initialises every
            // diagonal block; planes 1..7 accumulate into their shifted 128-column windows
#pragma unroll
            for (int kk = 0; kk < NK; ++kk)
              tc_mma_i8(acc0, tc_desc(a0 + kk * 256u, LBO, SBO), tc_desc(b0 + kk * 256u, LBO, SBO), IDESC240,
                        kk > 0 ? 1u : 0u);
#pragma unroll
            for (int i = 1; i < 8; ++i)
#pragma unroll
              for (int kk = 0; kk < NK; ++kk)
                tc_mma_i8(acc0 + (uint32_t)(i * kTcColsB), tc_desc(a0 + i * A_PLANE + kk * 256u, LBO, SBO),
                          tc_desc(b0 + kk * 256u, LBO, SBO), IDESC128, 1u);
            tc_commit(&sh.b_empty[st]);
            tc_commit(&sh.t_full[tb]);
          }
        tc_commit(&sh.a_empty);
      }
    }
  } else {  // ---- epilogue: warps 2..17
    const int ew = warp - 2, quarter = warp & 3, c4 = ew >> 2;  // TMEM lanes 32*quarter.., cols 4*c4..
    const int m = 32 * quarter + lane;
    long tc = 0;
    for (long u = u0; u < u1; ++u) {
      const long s0 = 4 * (u % SQ) + 2 * half_q;
      const int rb = (int)(u / SQ);
      const int r = (int)((s0 >> logn) % R);
      const PrimeConst pc = a.pc[r];
      const Field64 f = pc.f;
      for (int ct = 0; ct < nct; ++ct) {
        const int col0 = ct * kTcColsB + c4 * 4;
#pragma unroll
        for (int p = 0; p < 2; ++p, ++tc) {
          const int tb = (int)(tc & 1);
          // Y row (slot, row block, row): 32 contiguous bytes per thread, a tile row per warp
          uint64_t* y = Y + (((size_t)(s0 + p) * nrb + rb) * kTcRowsA + m) * nct * kTcColsB + col0;
          uint64_t prev[4] = {0, 0, 0, 0};
          if (kc > 0) {  // later K chunks: add this launch's sums to the previous chunks'
            ld_v2(y, prev[0], prev[1]);
            ld_v2(y + 2, prev[2], prev[3]);
          }
          mbar_wait(&sh.t_full[tb], (uint32_t)((tc >> 1) & 1));
          tc_fence_after();
          const uint32_t taddr = tmem + ((uint32_t)(32 * quarter) << 16) + (uint32_t)(tb * TCOLS + c4 * 4);
          // stream the 15 diagonals in rounds of 3 into P[L][c] = sum_q 2^(8q) D_(4L+q)
          // (a 15 x 4 register tile spilled at this kernel's 96-register budget)
          uint64_t P[4][4];
#pragma unroll
          for (int L = 0; L < 4; ++L)
#pragma unroll
            for (int c = 0; c < 4; ++c) P[L][c] = 0;
#pragma unroll
          for (int dg = 0; dg < kTcDiag / 3; ++dg) {
            uint32_t D[3][4];
#pragma unroll
            for (int k = 0; k < 3; ++k) tc_ld4(taddr + (uint32_t)((3 * dg + k) * kTcColsB), D[k]);
            tc_wait_ld();
#pragma unroll
            for (int k = 0; k < 3; ++k) {
              const int d = 3 * dg + k;
#pragma unroll
              for (int c = 0; c < 4; ++c) P[d >> 2][c] = madw(D[k][c], 1u << (8 * (d & 3)), P[d >> 2][c]);
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&sh.t_empty[tb]);  // buffer read: back to the MMA warp
          uint64_t x[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) x[c] = f.add(tc_reduce(f, pc, P[0][c], P[1][c], P[2][c], P[3][c]), prev[c]);
          *reinterpret_cast<ulonglong2*>(y) = make_ulonglong2(x[0], x[1]);
          *reinterpret_cast<ulonglong2*>(y + 2) = make_ulonglong2(x[2], x[3]);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem) : "memory");
  }
}

// Y (slot-major MAC product) -> the ciphertext layout out[img][cout][B][2][R][n], + the
// HomShare mask already in out's c1 words (has_mask).  CTA tile = 64 consecutive slots
// (same block and prime) x 4 rows x 16 out channels through shared memory (SWAP: 16 rows x 4
// channels -- Y then is [slot][128-channel block][channel][row], the ElementMult having run
// with the weights as its 128-row operand): reads are contiguous runs of Y, writes (and mask
// reads) 512-byte slot runs per (row, channel).
constexpr int kTrSlots = 64;
template <int R, bool SWAP>
__global__ void __launch_bounds__(256, 4) mac_out_kernel(LayerArgs a, int logn, const uint64_t* __restrict__ Y,
                                                      int has_mask, uint64_t* __restrict__ out) {
  constexpr int TR = SWAP ? 16 : 4, TC = SWAP ? 4 : 16;  // tile rows / out channels
  __shared__ uint64_t t[TR * TC][kTrSlots + 1];
  pdl_wait();
  pdl_trigger();
  const int n = 1 << logn;
  const long S = (long)a.B * R * n;
  const int rows = 2 * a.num_images, cols = a.cout;
  // Y's row blocks (of its 128-row operand) and row length (its 16-row operand, padded)
  const int nab = ((SWAP ? cols : rows) + kTcRowsA - 1) / kTcRowsA;
  const int ylen = (((SWAP ? rows : cols) + kTcColsB - 1) / kTcColsB) * kTcColsB;
  const int nrg = (rows + TR - 1) / TR, ncg = (cols + TC - 1) / TC;
  const long tiles = (S / kTrSlots) * nrg * ncg;
  const size_t ctw = (size_t)2 * R * n, chan_stride = (size_t)a.B * ctw;
  for (long tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int cg = (int)(tile % ncg), rg = (int)((tile / ncg) % nrg);
    const long s0 = tile / ((long)ncg * nrg) * kTrSlots;
    // gather: thread -> (slot, index along Y's rows, 16-byte pair along Y's row length); every
    // load of the tile is issued before the first shared store (8 x 16 B in flight per thread)
    constexpr int GATHER = kTrSlots * 4 * 8 / 256;
    ulonglong2 v[GATHER];
#pragma unroll
    for (int u = 0; u < GATHER; ++u) {
      const int e = threadIdx.x + u * 256;
      const int cp = e % 8, oth = (e / 8) % 4, sl = e / 32;  // pair along the 16-side, index along the 4-side
      const int row = rg * TR + (SWAP ? 2 * cp : oth), col = cg * TC + (SWAP ? oth : 2 * cp);
      const int ya = SWAP ? col : row, yb = SWAP ? row : col;  // Y[(slot, block of ya)][ya % 128][yb]
      v[u] = make_ulonglong2(0, 0);
      if (row < rows && col < cols && yb < ylen)
        v[u] = __ldg(reinterpret_cast<const ulonglong2*>(
            Y + (((size_t)(s0 + sl) * nab + ya / kTcRowsA) * kTcRowsA + ya % kTcRowsA) * ylen + yb));
    }
#pragma unroll
    for (int u = 0; u < GATHER; ++u) {
      const int e = threadIdx.x + u * 256;
      const int cp = e % 8, oth = (e / 8) % 4, sl = e / 32;
      if (SWAP) {  // the pair = rows 2 cp, 2 cp + 1 of channel oth
        t[(2 * cp) * TC + oth][sl] = v[u].x;
        t[(2 * cp + 1) * TC + oth][sl] = v[u].y;
      } else {  // the pair = channels 2 cp, 2 cp + 1 of row oth
        t[oth * TC + 2 * cp][sl] = v[u].x;
        t[oth * TC + 2 * cp + 1][sl] = v[u].y;
      }
    }
    __syncthreads();
    const int bp = (int)(s0 >> logn), b = bp / R, r = bp % R, j0 = (int)(s0 & (n - 1));
    const PrimeConst pc = a.pc[r];
    // scatter: a warp per (row, column) run of 64 slots, 2 slots per lane (16 bytes); the
    // mask loads of the thread's c1 runs are issued first
    constexpr int SCATTER = TR * TC * (kTrSlots / 2) / 256;
    ulonglong2 mk[SCATTER];
    uint64_t* dst[SCATTER];
#pragma unroll
    for (int u = 0; u < SCATTER; ++u) {
      const int e = threadIdx.x + u * 256;
      const int sp = e % (kTrSlots / 2), rc = e / (kTrSlots / 2);
      const int rr = rc / TC, cc = rc % TC;
      const int row = rg * TR + rr, col = cg * TC + cc;
      const int img = row >> 1, comp = row & 1;
      dst[u] = (row < rows && col < cols)
                   ? out + ((size_t)img * a.cout + col) * chan_stride + (size_t)b * ctw + (size_t)(comp * R + r) * n +
                         j0 + 2 * sp
                   : nullptr;
      mk[u] = make_ulonglong2(0, 0);
      if (dst[u] && comp == 1 && has_mask) mk[u] = *reinterpret_cast<const ulonglong2*>(dst[u]);
    }
#pragma unroll
    for (int u = 0; u < SCATTER; ++u) {
      if (!dst[u]) continue;
      const int e = threadIdx.x + u * 256;
      const int sp = e % (kTrSlots / 2), rc = e / (kTrSlots / 2);
      *reinterpret_cast<ulonglong2*>(dst[u]) =
          make_ulonglong2(pc.f.add(t[rc][2 * sp], mk[u].x), pc.f.add(t[rc][2 * sp + 1], mk[u].y));
    }
    __syncthreads();
  }
}

// Throughput probe: one elected thread issues back-to-back 128 x 16 x 32 (or 128 x N)
// u8 MMAs from (uninitialised) shared memory into TMEM; ensei_gpu_tc_i8_peak times it.
template <int N>
__global__ void __launch_bounds__(128, 1) mma_i8_peak_kernel(int iters, uint32_t* sink) {
  extern __shared__ __align__(1024) uint8_t pk_smem[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t done;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) mbar_init(&done, 1);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&tbase))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  if (threadIdx.x == 0) {
    const uint32_t sa = smem_u32(pk_smem), sb = sa + 16384;
    const uint64_t ad = tc_desc(sa, 128, 256), bd = tc_desc(sb, 128, 256);
    constexpr uint32_t ID = tc_idesc_i8(128, N);
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int d = 0; d < 8; ++d) tc_mma_i8(tmem + (uint32_t)((d * N) & 511), ad, bd, ID, 1u);
    tc_commit(&done);
    mbar_wait(&done, 0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    uint32_t v[8];
    tc_ld8(tmem, v);
    tc_wait_ld();
    if (v[0] == 0x12345678u) sink[0] = v[1];
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem) : "memory");
  }
}

}  // namespace ensei_gpu
