// mac_i8.cuh -- ElementMult + channel accumulation on the int8 tensor cores.
//
// Same result as mac_kara_kernel (REF mul_plain / add_ct, ringbfv.cpp:233-306, channel
// sum protocol.cpp:570-581, + the HomShare mask on c1): per slot, out[row][col] =
// sum_k ct[row][k] w[k][col] mod q, rows = (image, component), cols = out channels,
// k = in channels.  Exact integer arithmetic on the tensor cores by byte planes: with
// x = sum_i x_i 2^(8i), y = sum_j y_j 2^(8j) (x_i, y_j bytes, 8 planes for 60-bit
// residues),
//     T = sum_k x y = sum_{d=0..14} 2^(8d) D_d,   D_d = sum_{i+j=d} sum_k x_i y_j,
// and every D_d is one s32 tensor-core accumulation (u8 x u8 -> s32 mma.sync
// m16n8k32, SASS IMMA.16832.U8.U8): 8 K 255^2 < 2^31 for K <= 4127, and T < 2^128 for
// K <= 255.  The epilogue rebuilds T from the fifteen partial sums and reduces it
// once (as kara_T_mod).  64 byte products per MAC at the measured 565 T int8 MAC/s of
// the legacy path (tools/mma_i8_probe.cu) is 2.8x the IMAD pipe's MAC rate.
//
// Work: task = (4 consecutive slots) x (16 rows) x (16 cols); 8 warps, warp w owns
// slot w/2 and the 8-column half w%2 -> one 16x8 tile with 15 x 4 s32 accumulators.
// K chunks of 32 channels: 128 threads stage the ciphertext words (4 slots = one
// 32-byte sector per (row, channel)), 128 the weight words, each splitting 4 channels x
// 4 slots into byte planes with PRMT: shared [slot][plane][row|col][32 channel bytes],
// 16-byte rows XOR-swizzled by (row & 7) so every fragment load is conflict-free.
// Persistent grid; tasks ordered slot group outermost so concurrent CTAs share the
// group's sectors in L2.
#pragma once
#include "layer.cuh"

namespace ensei_gpu {

constexpr int kI8Slots = 4, kI8Rows = 16, kI8Cols = 16, kI8K = 32;
constexpr int kI8MaxK = 255;                                            // T < 2^128
constexpr int kI8PlaneWords = kI8Rows * (kI8K / 4);                      // 128 words per (slot, plane)
constexpr int kI8TileWords = kI8Slots * 8 * kI8PlaneWords;               // 4096 words = 16 KB

EG_DEV uint32_t plane_word(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3, int byte) {
  // bytes `byte` of w0..w3 -> one word (little-endian: w0's byte lowest)
  const uint32_t sel = (uint32_t)byte | ((uint32_t)(byte + 4) << 4);
  const uint32_t x01 = __byte_perm(w0, w1, sel);
  const uint32_t x23 = __byte_perm(w2, w3, sel);
  return __byte_perm(x01, x23, 0x5410);
}

EG_DEV void mma_u8(uint32_t (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <int R>
__global__ void __launch_bounds__(256, 2)
    mac_i8_kernel(LayerArgs a, int logn, const uint64_t* __restrict__ ct, const uint64_t* __restrict__ w,
                  int has_mask, uint64_t* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  __shared__ __align__(16) uint32_t As[kI8TileWords];
  __shared__ __align__(16) uint32_t Bs[kI8TileWords];
  const int n = 1 << logn;
  const int rows = 2 * a.num_images, cols = a.cout, K = a.cin;
  const int nrt = (rows + kI8Rows - 1) / kI8Rows, nct = (cols + kI8Cols - 1) / kI8Cols;
  const long ntasks = (long)(a.B * R * n / kI8Slots) * nrt * nct;
  const int nchunks = (K + kI8K - 1) / kI8K;
  const size_t ctw = (size_t)2 * R * n;            // ciphertext words per (image, channel, block)
  const size_t chan_stride = (size_t)a.B * ctw;    // ct: next channel
  const size_t w_chan = (size_t)a.B * R * n;       // w: next input channel
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;           // mma fragment coordinates
  const int ws = warp >> 1, wn = warp & 1;         // this warp's slot and column half
  constexpr uint64_t M30 = (1ull << 30) - 1;

  for (long task = blockIdx.x; task < ntasks; task += gridDim.x) {
    const long grp = task / (nrt * nct);
    const int rem = (int)(task % (nrt * nct));
    const int row0 = (rem % nrt) * kI8Rows, col0 = (rem / nrt) * kI8Cols;
    const long s0 = grp * kI8Slots;
    const int bp = (int)(s0 >> logn), b = bp / R, r = bp % R, j0 = (int)(s0 & (n - 1));
    uint32_t acc[15][4];
#pragma unroll
    for (int d = 0; d < 15; ++d) acc[d][0] = acc[d][1] = acc[d][2] = acc[d][3] = 0;

    for (int ch = 0; ch < nchunks; ++ch) {
      const int kc = ch * kI8K;
      // ---- stage byte planes: threads 0..127 ciphertexts, 128..255 weights
      {
        const int half = tid >> 7, u = tid & 127;
        const int rc = u >> 3, q = u & 7;  // row (or col) within the tile, channel quad
        uint32_t lo[4][kI8Slots], hi[4][kI8Slots];
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          const int c = kc + 4 * q + m;
          ulonglong2 v01 = make_ulonglong2(0, 0), v23 = make_ulonglong2(0, 0);
          if (half == 0) {
            const int row = row0 + rc;
            if (row < rows && c < K) {
              const uint64_t* src = ct + ((size_t)(row >> 1) * a.cin + c) * chan_stride + (size_t)b * ctw +
                                    (size_t)((row & 1) * R + r) * n + j0;
              v01 = __ldg(reinterpret_cast<const ulonglong2*>(src));
              v23 = __ldg(reinterpret_cast<const ulonglong2*>(src) + 1);
            }
          } else {
            const int col = col0 + rc;
            if (col < cols && c < K) {
              const uint64_t* src = w + ((size_t)col * a.cin + c) * w_chan + (size_t)bp * n + j0;
              v01 = __ldg(reinterpret_cast<const ulonglong2*>(src));
              v23 = __ldg(reinterpret_cast<const ulonglong2*>(src) + 1);
              // prepared weights pack the 30-bit limbs as (v >> 30) << 32 | (v & (2^30 - 1))
              v01.x = ((v01.x >> 32) << 30) | (v01.x & M30);
              v01.y = ((v01.y >> 32) << 30) | (v01.y & M30);
              v23.x = ((v23.x >> 32) << 30) | (v23.x & M30);
              v23.y = ((v23.y >> 32) << 30) | (v23.y & M30);
            }
          }
          lo[m][0] = lo32(v01.x), hi[m][0] = hi32(v01.x);
          lo[m][1] = lo32(v01.y), hi[m][1] = hi32(v01.y);
          lo[m][2] = lo32(v23.x), hi[m][2] = hi32(v23.x);
          lo[m][3] = lo32(v23.y), hi[m][3] = hi32(v23.y);
        }
        uint32_t* dst = half == 0 ? As : Bs;
        const int word = rc * 8 + (q ^ (rc & 7));
#pragma unroll
        for (int s = 0; s < kI8Slots; ++s)
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const uint32_t wv = i < 4 ? plane_word(lo[0][s], lo[1][s], lo[2][s], lo[3][s], i)
                                      : plane_word(hi[0][s], hi[1][s], hi[2][s], hi[3][s], i - 4);
            dst[(s * 8 + i) * kI8PlaneWords + word] = wv;
          }
      }
      __syncthreads();
      // ---- 64 byte-plane products per channel: D_(i+j) += A_i B_j
      {
        const uint32_t* as = As + ws * 8 * kI8PlaneWords;
        const uint32_t* bs = Bs + ws * 8 * kI8PlaneWords;
        const int bc = wn * 8 + g;  // this lane's B column within the tile
        uint32_t bf[8][2];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          bf[j][0] = bs[j * kI8PlaneWords + bc * 8 + (t ^ (bc & 7))];
          bf[j][1] = bs[j * kI8PlaneWords + bc * 8 + ((t + 4) ^ (bc & 7))];
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          uint32_t af[4];
          af[0] = as[i * kI8PlaneWords + g * 8 + (t ^ g)];
          af[1] = as[i * kI8PlaneWords + (g + 8) * 8 + (t ^ g)];
          af[2] = as[i * kI8PlaneWords + g * 8 + ((t + 4) ^ g)];
          af[3] = as[i * kI8PlaneWords + (g + 8) * 8 + ((t + 4) ^ g)];
#pragma unroll
          for (int j = 0; j < 8; ++j) mma_u8(acc[i + j], af, bf[j][0], bf[j][1]);
        }
      }
      __syncthreads();
    }

    // ---- epilogue: T = sum_d 2^(8d) D_d, reduced mod q_r, + the HomShare mask on c1
    const PrimeConst pc = a.pc[r];
    const Field64 f = pc.f;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int row = row0 + g + ((e >> 1) << 3), col = col0 + wn * 8 + 2 * t + (e & 1);
      if (row >= rows || col >= cols) continue;
      uint64_t P[4];
#pragma unroll
      for (int L = 0; L < 4; ++L) {
        uint64_t v = 0;
#pragma unroll
        for (int m = 0; m < 4; ++m)
          if (4 * L + m < 15) v += (uint64_t)acc[4 * L + m][e] << (8 * m);
        P[L] = v;
      }
      uint64_t c64 = P[0];
      const uint32_t t0 = lo32(c64);
      c64 = (c64 >> 32) + P[1];
      const uint32_t t1 = lo32(c64);
      c64 = (c64 >> 32) + P[2];
      const uint32_t t2 = lo32(c64);
      c64 = (c64 >> 32) + P[3];
      const uint32_t t3 = lo32(c64);
      const uint64_t lo = ((uint64_t)t1 << 32) | t0, hi = ((uint64_t)t3 << 32) | t2;
      uint64_t x = Bfly<Field64, 0>::corr(f, lo, pc.cred) + f.mul_shoup_approx(hi, pc.c64, pc.c64p);  // < 7q
      x = Bfly<Field64, 0>::fin_ct(f, x, pc.cred);
      const int img = row >> 1, comp = row & 1;
      uint64_t* o = out + ((size_t)img * a.cout + col) * chan_stride + (size_t)b * ctw + (size_t)(comp * R + r) * n +
                    j0 + ws;
      if (comp == 1 && has_mask) x = f.add(x, *o);
      *o = x;
    }
  }
}

}  // namespace ensei_gpu

namespace ensei_gpu {

// ---------------------------------------------------------------------------------
// Byte-plane operands prepared once per call (planes_kernel), then a cp.async
// pipeline feeding the tensor cores (mac_i8p_kernel).  Global plane layout, for the
// ciphertexts (rc = row = image x component) and the weights (rc = out channel):
//   [bp][slot][32-channel chunk kc][rc (padded to 32)][plane][8 words]
// (8 words = 32 channel bytes), so a task's chunk -- 32 rows (or cols) x 8 planes of
// one slot -- is one contiguous 8 KB block.  The pre-pass reads 4 slots (a 32-byte
// sector) per (row, channel) and scatters them to their slots.  Conversions: each ciphertext word once
// (instead of once per column tile) and each weight once per call (instead of once per
// row tile); the MAC kernel does no conversion, only 16-byte copies, MMA and epilogue.

constexpr int kI8T = 32;  // rows and cols per task of mac_i8p_kernel

__host__ __device__ inline long i8_plane_words(int B, int R, int n, int K, int nrc) {
  const long nkc = (K + kI8K - 1) / kI8K, rcp = (nrc + kI8T - 1) / kI8T * kI8T;
  return (long)B * R * n * nkc * rcp * 64;
}

template <int R, bool WEIGHTS>
__global__ void __launch_bounds__(256) planes_kernel(LayerArgs a, int logn, const uint64_t* __restrict__ src,
                                                     uint32_t* __restrict__ dst, int nrc) {
  // one thread: 4 channels x 8 slots (one 64-byte segment per channel) -> 8 x 8 words
  constexpr int SG = 8;
  const int n = 1 << logn, K = a.cin;
  const long nsg = n / SG, nkc = (K + kI8K - 1) / kI8K;
  const int rcp = (nrc + kI8T - 1) / kI8T * kI8T;
  const long total = (long)a.B * R * nsg * nkc * rcp * 8;
  const size_t ctw = (size_t)2 * R * n, chan_stride = (size_t)a.B * ctw, w_chan = (size_t)a.B * R * n;
  constexpr uint64_t M30 = (1ull << 30) - 1;
  for (long it = (long)blockIdx.x * 256 + threadIdx.x; it < total; it += (long)gridDim.x * 256) {
    const int q = (int)(it & 7);
    long rest = it >> 3;
    const int rc = (int)(rest % rcp);
    rest /= rcp;
    const int kc = (int)(rest % nkc);
    rest /= nkc;
    const long sg = rest % nsg;
    const int bp = (int)(rest / nsg), b = bp / R, r = bp % R;
    const int j0 = (int)(sg * SG);
    uint32_t lo[4][SG], hi[4][SG];
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const int c = kc * kI8K + 4 * q + m;
      ulonglong2 v[SG / 2];
#pragma unroll
      for (int h = 0; h < SG / 2; ++h) v[h] = make_ulonglong2(0, 0);
      if (rc < nrc && c < K) {
        const uint64_t* p = WEIGHTS ? src + ((size_t)rc * a.cin + c) * w_chan + (size_t)bp * n + j0
                                    : src + ((size_t)(rc >> 1) * a.cin + c) * chan_stride + (size_t)b * ctw +
                                          (size_t)((rc & 1) * R + r) * n + j0;
#pragma unroll
        for (int h = 0; h < SG / 2; ++h) v[h] = __ldg(reinterpret_cast<const ulonglong2*>(p) + h);
        if constexpr (WEIGHTS) {  // packed 30-bit limbs -> canonical value
#pragma unroll
          for (int h = 0; h < SG / 2; ++h) {
            v[h].x = ((v[h].x >> 32) << 30) | (v[h].x & M30);
            v[h].y = ((v[h].y >> 32) << 30) | (v[h].y & M30);
          }
        }
      }
#pragma unroll
      for (int h = 0; h < SG / 2; ++h) {
        lo[m][2 * h] = lo32(v[h].x), hi[m][2 * h] = hi32(v[h].x);
        lo[m][2 * h + 1] = lo32(v[h].y), hi[m][2 * h + 1] = hi32(v[h].y);
      }
    }
#pragma unroll
    for (int s = 0; s < SG; ++s) {
      uint32_t* o = dst + ((((long)bp * n + j0 + s) * nkc + kc) * rcp + rc) * 64;
#pragma unroll
      for (int i = 0; i < 8; ++i)
        o[i * 8 + q] = i < 4 ? plane_word(lo[0][s], lo[1][s], lo[2][s], lo[3][s], i)
                             : plane_word(hi[0][s], hi[1][s], hi[2][s], hi[3][s], i - 4);
    }
  }
}

template <int R, int STAGES>
__global__ void __launch_bounds__(256, 2)
    mac_i8p_kernel(LayerArgs a, int logn, const uint32_t* __restrict__ Ap, const uint32_t* __restrict__ Bp,
                   int has_mask, uint64_t* __restrict__ out) {
  // task = (slot, 32-row tile, 32-col tile); warp w owns the 16x8 tile at rows
  // 16 (w >> 2), cols 8 (w & 3) of it.  Stage = A [plane][32 rows][8 words] | B same.
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) uint32_t sm_i8[];
  constexpr int PL = kI8T * 8;           // words per plane of a tile
  constexpr int TILE = 8 * PL, STAGE = 2 * TILE;
  const int n = 1 << logn;
  const int rows = 2 * a.num_images, cols = a.cout, K = a.cin;
  const int nrt = (rows + kI8T - 1) / kI8T, nct = (cols + kI8T - 1) / kI8T;
  const int nkc = (K + kI8K - 1) / kI8K;
  constexpr int SPT = 4;  // slots per task: their outputs share 32-byte sectors, written back to back
  const long ntasks = (long)a.B * R * (n / SPT) * nrt * nct;
  const int my_tasks = blockIdx.x < ntasks ? (int)((ntasks - 1 - blockIdx.x) / gridDim.x + 1) : 0;
  const long nsteps = (long)my_tasks * SPT * nkc;
  const size_t ctw = (size_t)2 * R * n, chan_stride = (size_t)a.B * ctw;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3, wr = warp >> 2, wc = warp & 3;
  const long rows_p = (long)nrt * kI8T, cols_p = (long)nct * kI8T;

  auto task_of = [&](long j, int sub, long& slot, int& rt, int& ctile) {
    const long tk = blockIdx.x + j * gridDim.x;
    slot = tk / (nrt * nct) * SPT + sub;  // over B * R * n: (bp, slot) with the slot fastest
    const int rem = (int)(tk % (nrt * nct));
    rt = rem % nrt;
    ctile = rem / nrt;
  };
  // Copy addressing: a task's SPT * nkc steps read consecutive (slot, chunk) blocks of the
  // plane arrays ((slot * nkc + c) * rows_p + row0) * 64, so each step advances one pointer
  // pair by a fixed stride and only a new task decodes (tk -> slot, tiles: two divisions).
  // The per-thread source / destination offsets of the four 16-byte copies are fixed.
  const long a_step = rows_p * 64, b_step = cols_p * 64;
  const int task_steps = SPT * nkc;
  int src_off[4], dst_off[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int e = tid + u * 256;  // 0..1023: operand, rc, plane, 16-byte half
    const int op = e >> 9, rc = (e >> 4) & 31, pl = (e >> 1) & 7, hf = e & 1;
    src_off[u] = rc * 64 + pl * 8 + hf * 4;
    dst_off[u] = op * TILE + pl * PL + rc * 8 + ((hf ^ ((rc >> 2) & 1)) << 2);
  }
  long ld_j = 0;
  int ld_k = 0;  // step within the task being loaded
  const uint32_t* ag = nullptr;
  const uint32_t* bg = nullptr;
  auto task_ptrs = [&](long j) {
    long slot;
    int rt, ctile;
    task_of(j, 0, slot, rt, ctile);
    ag = Ap + (slot * nkc * rows_p + (long)rt * kI8T) * 64;
    bg = Bp + (slot * nkc * cols_p + (long)ctile * kI8T) * 64;
  };
  if (my_tasks > 0) task_ptrs(0);
  auto load_step = [&](long step) {
    if (step < nsteps) {
      uint32_t* As = sm_i8 + (step % STAGES) * STAGE;
#pragma unroll
      for (int u = 0; u < 4; ++u) cp_async16(As + dst_off[u], (u < 2 ? ag : bg) + src_off[u]);
      ag += a_step;
      bg += b_step;
      if (++ld_k == task_steps) {
        ld_k = 0;
        if (++ld_j < my_tasks) task_ptrs(ld_j);
      }
    }
    cp_async_commit();
  };

  for (int st = 0; st < STAGES - 1; ++st) load_step(st);
  uint32_t acc[15][4];
#pragma unroll
  for (int d = 0; d < 15; ++d) acc[d][0] = acc[d][1] = acc[d][2] = acc[d][3] = 0;
  long cm_j = 0;
  int cm_c = 0, cm_s = 0;
  const int ra = wr * 16 + g, cb = wc * 8 + g;                  // fragment row / col in the tile
  const int sa = ((g >> 2) & 1) << 2;                           // 16-byte half swizzle (rows and cols)
  for (long step = 0; step < nsteps; ++step) {
    // one barrier per step: after it every warp has finished the previous step, so the
    // buffer that step read can be refilled right away (STAGES-2 groups stay in flight)
    asm volatile("cp.async.wait_group %0;\n" ::"n"(STAGES - 2) : "memory");
    __syncthreads();
    load_step(step + STAGES - 1);
    {
      const uint32_t* as = sm_i8 + (step % STAGES) * STAGE;
      const uint32_t* bs = as + TILE;
      uint32_t bf[8][2];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        bf[j][0] = bs[j * PL + cb * 8 + (sa ^ 0) + t];
        bf[j][1] = bs[j * PL + cb * 8 + (sa ^ 4) + t];
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        uint32_t af[4];
        af[0] = as[i * PL + ra * 8 + (sa ^ 0) + t];
        af[1] = as[i * PL + (ra + 8) * 8 + (sa ^ 0) + t];
        af[2] = as[i * PL + ra * 8 + (sa ^ 4) + t];
        af[3] = as[i * PL + (ra + 8) * 8 + (sa ^ 4) + t];
#pragma unroll
        for (int j = 0; j < 8; ++j) mma_u8(acc[i + j], af, bf[j][0], bf[j][1]);
      }
    }
    if (++cm_c == nkc) {  // task complete: T = sum_d 2^(8d) D_d mod q_r (+ mask on c1)
      long slot;
      int rt, ctile;
      task_of(cm_j, cm_s, slot, rt, ctile);
      const int bp = (int)(slot >> logn), b = bp / R, r = bp % R, j = (int)(slot & (n - 1));
      const PrimeConst pc = a.pc[r];
      const Field64 f = pc.f;
      // the four HomShare-mask reads first (one latency for all four, overlapping the
      // reconstruction below); c1 rows are the odd ones: g odd
      uint64_t mv[4] = {0, 0, 0, 0};
      const bool c1 = has_mask && (ra & 1);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int row = rt * kI8T + ra + ((e >> 1) << 3), col = ctile * kI8T + wc * 8 + 2 * t + (e & 1);
        if (c1 && row < rows && col < cols)
          mv[e] = out[((size_t)(row >> 1) * a.cout + col) * chan_stride + (size_t)b * ctw + (size_t)(R + r) * n + j];
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int row = rt * kI8T + ra + ((e >> 1) << 3), col = ctile * kI8T + wc * 8 + 2 * t + (e & 1);
        if (row < rows && col < cols) {
          uint64_t P[4];
#pragma unroll
          for (int L = 0; L < 4; ++L) {
            uint64_t v = 0;
#pragma unroll
            for (int m = 0; m < 4; ++m)
              if (4 * L + m < 15) v += (uint64_t)acc[4 * L + m][e] << (8 * m);
            P[L] = v;
          }
          uint64_t c64 = P[0];
          const uint32_t t0 = lo32(c64);
          c64 = (c64 >> 32) + P[1];
          const uint32_t t1 = lo32(c64);
          c64 = (c64 >> 32) + P[2];
          const uint32_t t2 = lo32(c64);
          c64 = (c64 >> 32) + P[3];
          const uint32_t t3 = lo32(c64);
          const uint64_t lo = ((uint64_t)t1 << 32) | t0, hi = ((uint64_t)t3 << 32) | t2;
          uint64_t x = Bfly<Field64, 0>::corr(f, lo, pc.cred) + f.mul_shoup_approx(hi, pc.c64, pc.c64p);
          x = Bfly<Field64, 0>::fin_ct(f, x, pc.cred);
          const int img = row >> 1, comp = row & 1;
          uint64_t* o = out + ((size_t)img * a.cout + col) * chan_stride + (size_t)b * ctw +
                        (size_t)(comp * R + r) * n + j;
          if (comp == 1 && has_mask) x = f.add(x, mv[e]);
          *o = x;
        }
      }
#pragma unroll
      for (int d = 0; d < 15; ++d) acc[d][0] = acc[d][1] = acc[d][2] = acc[d][3] = 0;
      cm_c = 0;
      if (++cm_s == SPT) {
        cm_s = 0;
        ++cm_j;
      }
    }
  }
  cp_async_wait_all();
}

}  // namespace ensei_gpu
