// ozaki.cuh -- exact-integer tensor-core contractions for the CoFEM hot path.
//
// Phi is stored ONCE as a 32-bit fixed-point matrix split into four signed
// base-256 digit planes (4 bytes / entry -- the same HBM bytes as fp32):
//   Phi[i][j] = r_i c_j 2^-30 sum_a 256^(3-a) D_a[i][j],  D_a in [-128, 127]
// with power-of-two row / column scales r_i, c_j (|Phi / (r c)| <= 1).  The
// skinny operand (P for Phi P, V for Phi^T V) is split the same way per
// column q at every PCG step (k_quantize_cols).  One tcgen05.mma.kind::i8
// (M = 128, N = 4 QW, K = 32) multiplies digit plane a of Phi with ALL four
// digit planes of the operand at once (the planes are concatenated along N),
// accumulating exactly in int32 TMEM; the epilogue recombines the 16 digit
// products in fp64.  The contraction is therefore exact up to the 30-bit
// quantisation of the two factors (~1e-9 relative to the row / column max),
// which is what lets an fp32-sized Phi stream reproduce the float64
// reference, at int8 tensor-core rate.
//
// Phi P (FWD): A = digit plane, K-major (rows i, k = j), TMA box {64 j, 128 i, 4 planes}
// Phi^T V (BWD): A = digit plane, MN-major (m = j, k = i), TMA boxes {64 j, 64 i, 4} x 2
// B (both): operand digit planes [4][QW][K], K-major, TMA box {64 k, QW, 4}
// SWIZZLE_64B everywhere; 5-stage TMA -> smem ring; persistent CTAs
// (warp 0 TMA producer, warp 1 MMA issuer, warps 2..9 TMEM epilogue: warp w
// reads lane quarter w % 4, and the 8-column groups of parity (w - 2) / 4).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.cuh"
#include "pcg.cuh"

namespace cofem {
namespace oz {

#ifndef OZ_VARIANT
// band_kernel timing builds (scratch/build_variants.sh; results in DESIGN.md):
// 1 = no MMAs, 2 = epilogue without math / stores, 3 = no epilogue,
// 4 = no epilogue and no operand loads (pure MMA), 5 = no operand loads
#define OZ_VARIANT 0
#endif
constexpr int KT = 64;           // K bytes per stage (one SWIZZLE_64B row)
constexpr int BM = 128;          // output rows per tile (UMMA M)
constexpr int STAGES = 5;
constexpr int EPI_WARPS = 8;     // two epilogue warps per TMEM lane quarter (column halves)
constexpr int NTHREADS = 64 + 32 * EPI_WARPS;  // warp 0 TMA, warp 1 MMA, warps 2..9 epilogue
constexpr int A_STAGE = 4 * BM * KT;  // 32 KB: four digit planes
constexpr double SCALE30 = 1073741824.0;  // 2^30

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nLAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra LAB_WAIT;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
// operand planes live K-blocked in HBM: [k / 64][4 planes][ncols][64 k], so
// the {64 k, QW cols, 4 planes} box of one stage is 4 contiguous runs of 64 QW
// bytes (not 4 QW rows of 64 B a whole column apart); c3 = k / 64
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                            int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
// byte offset of digit plane a, column col, K index k in the K-blocked layout
__host__ __device__ __forceinline__ int64_t kb_offset(int64_t ncols, int a, int64_t col, int64_t k) {
  return ((((k >> 6) * 4 + a) * ncols + col) << 6) + (k & 63);
}
__device__ __forceinline__ void tma_prefetch(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}

// shared-memory matrix descriptor, SWIZZLE_64B (layout type 4), sm100 version bit
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) | ((uint64_t)4 << 61);
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

#define OZ_LD32(addr, r)                                                                                        \
  asm volatile(                                                                                                 \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"          \
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                                \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),         \
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),   \
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), \
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])  \
      : "r"(addr))

// Digit plane a of Phi is multiplied with operand planes b <= 4 - a only.
// The three dropped pairs (a + b >= 5) sit ~1e-10 below the result -- under
// the 2^-30 quantisation of the factors -- and trimming them cuts a sixth of
// the tensor work (and power: the contraction runs at the 1 kW cap); dropping
// also a + b = 4 was measured to cost 2.6e-8, so those stay.
//
// Significance-aligned accumulation: the MMA for plane a writes its N = QW
// nb(a) columns at TMEM offset a QW, so operand plane b lands in column block
// s = a + b and every product of equal significance accumulates in the same
// block.  Five blocks (s = 0..4) hold the whole result; columns past block 4
// (from rounding N up to the UMMA granularity of 16) only ever collect pruned
// s >= 5 products and are never read.  A set is <= 160 columns, so TMEM holds
// two sets and the epilogue of one tile overlaps the MMAs of the next.  The
// epilogue zeroes its set with tcgen05.st after reading it, so every MMA just
// accumulates.  Exactness: |block| <= 4 pairs * 2^14 * K < 2^31 for K <= 2^15.
template <int QW, int NPA = 4>
struct Cfg {
  static constexpr int NB = 4 * QW;  // B tile rows: the four operand planes side by side
  static constexpr int A_ST = NPA * BM * KT;  // NPA digit planes of Phi per stage
  static constexpr int B_STAGE = NB * KT;
  static constexpr int STAGE = A_ST + B_STAGE;
  static constexpr size_t SMEM = (size_t)STAGES * STAGE + 1024 + 1280;
  __host__ __device__ static constexpr int nb_of(int a) { return a <= 1 ? 4 : 5 - a; }  // operand planes used
  __host__ __device__ static constexpr int n_of(int a) { return ((QW * nb_of(a) + 15) / 16) * 16; }
  static constexpr int SET_COLS = 256;  // TMEM columns per accumulator set (two sets)
  static_assert(QW % 8 == 0 && QW <= 32, "QW in {8,16,24,32}");
  static_assert(NPA >= 2 && NPA <= 4, "2..4 digit planes of Phi");
  static_assert(STAGE % 1024 == 0, "stages must stay 1024-B aligned for the swizzle atoms");
  static_assert(2 * QW + ((QW * 3 + 15) / 16) * 16 <= SET_COLS && 5 * QW <= SET_COLS, "set must fit");
};
constexpr int MAX_K_PER_ITEM = 1 << 15;

// one K=64 stage: 2 k-steps x NPA digit planes of A against the operand tile
template <int QW, bool MN_MAJOR, int NPA = 4>
__device__ __forceinline__ void issue_stage(uint32_t sa, uint32_t sb, uint32_t tset, uint32_t idesc0) {
  using C = Cfg<QW, NPA>;
#pragma unroll
  for (int kk = 0; kk < 2; ++kk) {
    const uint64_t db = sdesc(sb + kk * 32, 16, 512);
#pragma unroll
    for (int a = 0; a < NPA; ++a) {
      uint64_t da;
      if (!MN_MAJOR) da = sdesc(sa + a * (BM * KT) + kk * 32, 16, 512);
      else da = sdesc(sa + a * (64 * KT) + kk * (32 * KT), C::A_ST / 2, 512);
      const uint32_t idesc = idesc0 | ((uint32_t)(C::n_of(a) >> 3) << 17);
      mma_i8(tset + a * QW, da, db, idesc, 1u);
    }
  }
}

// zero both accumulator sets of this warp's TMEM lane quarter (prologue)
__device__ __forceinline__ void tmem_zero_all(uint32_t tmem, int quarter) {
  const uint32_t base = tmem + ((uint32_t)(quarter * 32) << 16);
#pragma unroll 1
  for (int c = 0; c < 512; c += 8)
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(base + c), "r"(0));
  asm volatile("tcgen05.wait::st.sync.aligned;");
}

// 256-bit global accesses (sm_100): an epilogue thread owns one output row, so
// a warp instruction touches 32 rows; moving a whole 32-B sector per thread
// keeps every requested sector fully used (16-B accesses fetched each sector
// twice and, for streamed reads, let L2 evict it in between)
__device__ __forceinline__ void st_v4(double* p, double a, double b, double c, double d) {
  asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}
__device__ __forceinline__ void ld_v4(const double* p, double& a, double& b, double& c, double& d) {
  asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}

// Epilogue of one tile for the calling thread's row: read the five
// significance blocks, re-zero them, combine exactly in int64 and write
// out[q] = value * scale * op_scale[q].  With TRACK the thread keeps running
// per-column maxima of |out| in registers (bit patterns of non-negative
// doubles order like unsigned integers, NaN above everything); they are
// folded across the warp and the CTA once, at the end of the kernel.
template <int QW, bool TRACK, int HALF>
__device__ __forceinline__ void epilogue_row(uint32_t tset_lane, double scale, const double* __restrict__ op_scale,
                                             double* o, unsigned long long (&cm)[QW]) {
#pragma unroll
  for (int q0 = HALF * 8; q0 < QW; q0 += 16) {
    // scale * op_scale: both powers of two, so the products below are exact
    double f[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) f[t] = scale * __ldg(op_scale + q0 + t);
    uint32_t r[5][8];
#pragma unroll
    for (int sb = 0; sb < 5; ++sb)
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(r[sb][0]), "=r"(r[sb][1]), "=r"(r[sb][2]), "=r"(r[sb][3]), "=r"(r[sb][4]),
                     "=r"(r[sb][5]), "=r"(r[sb][6]), "=r"(r[sb][7])
                   : "r"(tset_lane + sb * QW + q0));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
    for (int sb = 0; sb < 5; ++sb)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(
                       tset_lane + sb * QW + q0),
                   "r"(0));
    double v[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      // value = 2^16 (S0 2^32 + S1 2^24 + S2 2^16 + S3 2^8 + S4), |S1 2^24 + ...| < 2^57
      const long long lo = ((long long)(int32_t)r[1][t] << 24) + ((long long)(int32_t)r[2][t] << 16) +
                           ((long long)(int32_t)r[3][t] << 8) + (long long)(int32_t)r[4][t];
      v[t] = fma((double)(int32_t)r[0][t], 4294967296.0, (double)lo) * f[t];
    }
    st_v4(o + q0, v[0], v[1], v[2], v[3]);
    st_v4(o + q0 + 4, v[4], v[5], v[6], v[7]);
    if (TRACK) {
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        // |v| as a bit pattern: clear the sign bit on the integer side (no FP64 op)
        const unsigned long long m = (unsigned long long)__double_as_longlong(v[t]) & 0x7fffffffffffffffull;
        cm[q0 + t] = m > cm[q0 + t] ? m : cm[q0 + t];
      }
    }
  }
}

// the calling epilogue warp's share of one tile row (column groups of parity half)
template <int QW>
__device__ __forceinline__ void epilogue_part(int half, bool track, uint32_t tset_lane, double scale,
                                              const double* __restrict__ op_scale, double* o,
                                              unsigned long long (&cm)[QW]) {
  if (half == 0) {
    if (track) epilogue_row<QW, true, 0>(tset_lane, scale, op_scale, o, cm);
    else epilogue_row<QW, false, 0>(tset_lane, scale, op_scale, o, cm);
  } else {
    if (track) epilogue_row<QW, true, 1>(tset_lane, scale, op_scale, o, cm);
    else epilogue_row<QW, false, 1>(tset_lane, scale, op_scale, o, cm);
  }
}

// fold the per-lane column maxima over the warp into this warp's smem slice
template <int QW>
__device__ __forceinline__ void warp_fold_max(unsigned long long (&cm)[QW], unsigned long long* slice) {
#pragma unroll
  for (int q = 0; q < QW; ++q) {
    unsigned long long m = cm[q];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const unsigned long long x = __shfl_xor_sync(0xffffffffu, m, off);
      m = x > m ? x : m;
    }
    if ((threadIdx.x & 31) == 0) slice[q] = m;
  }
}

// Persistent contraction.  Work item w (< n_items) = (mb = w % n_mblocks,
// split s = w / n_mblocks): output rows [mb*128, +128), K range
// [s*k_per_split, min(+k_per_split, k_total)).  Writes fp64
// out[s][row][0:QW] = sum_k Phi(.)[row][k] * op[k][q] (already scaled).
//   MODE_FWD : rows are i, K is j; row scale r_i (A = digit planes, K-major)
//   MODE_BWD : rows are j, K is i; row scale c_j (A = the same planes, MN-major)
//   MODE_BAND: banded Toeplitz operator streamed from L2 (long filters; see
//     band_kernel for the smem-resident version): every output tile sees the
//     same 128 x k_per_split band, so A's TMA coordinate is relative to the
//     tile: K range [mb*128 + band_offset, + k_per_split); operand rows outside
//     [0, K) arrive as TMA zero fill.
// Rows >= rows_real are written as zeros; out_colmax (may be null) collects
// the column maxima of |out| for the next quantisation (single-split modes).
// Wide operands (n_items > n_mblocks * n_split): item w also selects column
// chunk nc = w / (n_mblocks * n_split) of an operand with out_ld columns
// (B TMA row coordinate nc * QW, op_scale / out offset nc * QW).
enum { MODE_FWD = 0, MODE_BWD = 1, MODE_BAND = 2 };
template <int QW, int MODE, int NPA = 4>
__global__ void __launch_bounds__(NTHREADS, 1)
    contract_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                    int n_mblocks, int n_items, int k_per_split, int k_total, int band_offset,
                    const double* __restrict__ row_scale, const double* __restrict__ op_scale,
                    double* __restrict__ out, int64_t out_rows, int64_t rows_real,
                    unsigned long long* __restrict__ out_colmax, const Status* __restrict__ st, int n_split = 1,
                    int out_ld = QW) {
  constexpr bool BWD = MODE == MODE_BWD;
  using C = Cfg<QW, NPA>;
  if (st && st->done) return;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* sm = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + STAGES * C::STAGE);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;  // [2]
  uint64_t* tempty = tfull + 2;      // [2]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);
  // [EPI_WARPS][QW] column maxima, folded after the last tile: aliases the
  // stage ring, which every MMA has finished reading by then
  unsigned long long* cmax = reinterpret_cast<unsigned long long*>(sm);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 32 * EPI_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    tma_prefetch(&map_a);
    tma_prefetch(&map_b);
  }
  (void)0;
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_holder;
  if (warp >= 2 && warp < 6) tmem_zero_all(tmem, warp & 3);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      int stage = 0;
      uint32_t phase = 0;
      for (int w = blockIdx.x; w < n_items; w += gridDim.x) {
        const int mb = w % n_mblocks, s = (w / n_mblocks) % n_split, nc = w / (n_mblocks * n_split);
        const int k0 = MODE == MODE_BAND ? mb * BM + band_offset : s * k_per_split;
        const int k1 = MODE == MODE_BAND ? k0 + k_per_split : min(k0 + k_per_split, k_total);
        for (int k = k0; k < k1; k += KT) {
          mbar_wait(&empty[stage], phase ^ 1);
          unsigned char* sa = sm + stage * C::STAGE;
          unsigned char* sb = sa + C::A_ST;
          mbar_expect_tx(&full[stage], C::STAGE);
          if (MODE == MODE_BAND) {
            tma_load_3d(sa, &map_a, &full[stage], k - k0, 0, 0);
          } else if (!BWD) {
            tma_load_3d(sa, &map_a, &full[stage], k, mb * BM, 0);
          } else {
            tma_load_3d(sa, &map_a, &full[stage], mb * BM, k, 0);
            tma_load_3d(sa + C::A_ST / 2, &map_a, &full[stage], mb * BM + 64, k, 0);
          }
          tma_load_4d(sb, &map_b, &full[stage], 0, nc * QW, 0, k >> 6);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer (single thread) ----------------
      // idesc: D s32 (bits 4-5 = 2), A,B signed s8 (bits 7, 10), A major (bit 15),
      // N >> 3 (bits 17..22), M >> 4 (bits 24..28)
      const uint32_t idesc0 = (2u << 4) | (1u << 7) | (1u << 10) | ((BWD ? 1u : 0u) << 15) |
                              ((uint32_t)(BM >> 4) << 24);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int w = blockIdx.x; w < n_items; w += gridDim.x, ++it) {
        const int mb = w % n_mblocks, s = (w / n_mblocks) % n_split;
        const int k0 = MODE == MODE_BAND ? mb * BM + band_offset : s * k_per_split;
        const int k1 = MODE == MODE_BAND ? k0 + k_per_split : min(k0 + k_per_split, k_total);
        const int buf = it & 1;
        mbar_wait(&tempty[buf], ((it >> 1) & 1) ^ 1);  // this set has been drained and re-zeroed
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t tset = tmem + buf * C::SET_COLS;
        for (int k = k0; k < k1; k += KT) {
          mbar_wait(&full[stage], phase);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t sa = smem_u32(sm + stage * C::STAGE);
          issue_stage<QW, BWD, NPA>(sa, sa + C::A_ST, tset, idesc0);
          mma_commit(&empty[stage]);  // frees the smem slot once these MMAs retire
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit(&tfull[buf]);  // accumulators complete
      }
    }
  } else {
    // ---------------- epilogue: warps 2..9 -> TMEM lane quarter warp % 4, column half ----------------
    const int quarter = warp & 3, half = (warp - 2) >> 2;
    const int row_in_tile = quarter * 32 + lane;
    unsigned long long cm[QW];
#pragma unroll
    for (int q = 0; q < QW; ++q) cm[q] = 0ull;
    int it = 0;
    for (int w = blockIdx.x; w < n_items; w += gridDim.x, ++it) {
      const int mb = w % n_mblocks, s = (w / n_mblocks) % n_split, nc = w / (n_mblocks * n_split);
      const int buf = it & 1;
      const int64_t row = (int64_t)mb * BM + row_in_tile;
      // the row scale load is issued before the wait so its latency hides behind the MMAs
      const double scale = row < rows_real ? row_scale[row] * (65536.0 / (SCALE30 * SCALE30)) : 0.0;
      mbar_wait(&tfull[buf], (it >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      double* orow = out + ((int64_t)s * out_rows + row) * out_ld + nc * QW;
      epilogue_part<QW>(half, out_colmax != nullptr, tmem + buf * C::SET_COLS + ((uint32_t)(quarter * 32) << 16),
                        scale, op_scale + nc * QW, orow, cm);
      asm volatile("tcgen05.wait::st.sync.aligned;");
      asm volatile("tcgen05.fence::before_thread_sync;");
      mbar_arrive(&tempty[buf]);
    }
    if (out_colmax) warp_fold_max<QW>(cm, cmax + (warp - 2) * QW);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (out_colmax && threadIdx.x < QW) {
    unsigned long long m = cmax[threadIdx.x];
    for (int w = 1; w < EPI_WARPS; ++w) m = cmax[w * QW + threadIdx.x] > m ? cmax[w * QW + threadIdx.x] : m;
    atomicMax(&out_colmax[threadIdx.x], m);
  }
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// Band-resident Toeplitz contraction (convolution dictionaries).  The whole
// 128 x nk band (NPA digit planes, nk = 128 + lpad bytes per row) is loaded
// into shared memory ONCE per CTA; the TMA ring then carries only the operand
// windows (4 QW x 64 B per stage), so the L2 -> SM traffic per output tile is
// the window alone.  Same significance-aligned accumulation as
// contract_kernel (NPA = 3: the 24-bit taps of COFEM_OZAKI24, one MMA per
// k-step less -- the kernel is MMA-issue bound).
constexpr int BSTAGES = 4;
// band_kernel accumulator sets: 5 significance blocks of QW <= 32 columns
// (160 TMEM columns); three sets in the 512-column allocation, so the MMA
// issuer can run two tiles ahead of a slow epilogue
#ifndef BAND_SETS_OVERRIDE
constexpr int BAND_SETS = 3;
#else
constexpr int BAND_SETS = BAND_SETS_OVERRIDE;
#endif
constexpr int BAND_SET_COLS = 160;
constexpr int BAND_EPI_WARPS = 16;                      // 4 lane quarters x 4 column groups of 8
constexpr int BAND_NTHREADS = 64 + 32 * BAND_EPI_WARPS;  // warp 0 TMA, warp 1 MMA, warps 2..17 epilogue
template <int QW, int NPA = 4>
struct BandCfg {
  static constexpr int B_STAGE = 4 * QW * KT;
  static size_t smem(int nk) { return (size_t)nk * NPA * BM + (size_t)BSTAGES * B_STAGE + 1024 + 1280; }
};

// band_kernel epilogues
//   EPI_PLAIN: out = Phi(.) op, optional column maxima of |out|
//   EPI_COMB : the Phi^T V launch of a PCG step: out = Psi = beta Phi^T V +
//              alpha .* P and pi = <P, Psi> (k_combine fused)
//   EPI_FWD  : the Phi P launch of the fused convolution step: out = V, the
//              column maxima of |V| and vv = ||V||^2 per column (block
//              partials + last-block fold), so pi = beta ||V||^2 + <P, alpha P>
//              is known before Phi^T V runs
//   EPI_UPD  : the Phi^T V launch of the fused convolution step: no Psi block
//              and no k_update -- each row applies R -= gamma (beta Phi^T V +
//              alpha .* P) (gamma = rho / pi, pi from EPI_FWD's vv and the
//              direction kernel's <P, alpha P>) and accumulates <R, M^-1 R>,
//              ||R||^2 (block partials + last-block fold) and the column
//              maxima of |M^-1 R| (the next direction's quantisation bound)
enum { EPI_PLAIN = 0, EPI_COMB = 1, EPI_FWD = 2, EPI_UPD = 3 };

// extra arguments of the fused-step epilogues
struct BandStep {
  const double* P;         // [rows][ld] current direction (EPI_COMB / EPI_UPD)
  double* R;               // [rows][ld] residual, updated in place (EPI_UPD)
  int ld;
  int q_real;
  int printed;             // printed recursion: the bound tracks |R| instead of |M^-1 R|
  const double* alpha;     // [rows]
  const double* minv;      // [rows * ngroups]
  const int* groups;       // column -> preconditioner group (nullptr: one group)
  int ngroups;
  double beta;
  const double* rho;       // rho of P(u) (EPI_UPD)
  const double* vv;        // ||Phi P||^2 (EPI_UPD)
  const double* pap;       // <P, alpha P> (EPI_UPD)
  double* gam_out;         // gamma per column, for the direction kernel's X update (EPI_UPD)
  int* frozen;             // breakdown flags (EPI_UPD)
  unsigned long long* wmax;   // column maxima of |M^-1 R| (EPI_UPD, atomicMax)
  unsigned long long* reset;  // zeroed by block 0 (the next direction's |P| maxima)
  double* out0;            // fold outputs: pi (COMB) / vv (FWD) / rho_new (UPD)
  double* out1;            // rn2 (UPD)
  double* partials;        // [grid][2][QW]
  unsigned* ticket;
};

template <int QW>
__device__ __forceinline__ void tmem_rows4(uint32_t tl, int q0, uint32_t (&r)[5][4]) {
#pragma unroll
  for (int sb = 0; sb < 5; ++sb)
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[sb][0]), "=r"(r[sb][1]), "=r"(r[sb][2]), "=r"(r[sb][3])
                 : "r"(tl + sb * QW + q0));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
  for (int sb = 0; sb < 5; ++sb)
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%1,%1,%1};" ::"r"(tl + sb * QW + q0), "r"(0));
}
template <int NC>
__device__ __forceinline__ double combine5n(const uint32_t (&r)[5][NC], int t) {
  const long long lo = ((long long)(int32_t)r[1][t] << 24) + ((long long)(int32_t)r[2][t] << 16) +
                       ((long long)(int32_t)r[3][t] << 8) + (long long)(int32_t)r[4][t];
  return fma((double)(int32_t)r[0][t], 4294967296.0, (double)lo);
}
template <int QW>
__device__ __forceinline__ void tmem_rows8(uint32_t tl, int q0, uint32_t (&r)[5][8]) {
#pragma unroll
  for (int sb = 0; sb < 5; ++sb)
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[sb][0]), "=r"(r[sb][1]), "=r"(r[sb][2]), "=r"(r[sb][3]), "=r"(r[sb][4]), "=r"(r[sb][5]),
                   "=r"(r[sb][6]), "=r"(r[sb][7])
                 : "r"(tl + sb * QW + q0));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
  for (int sb = 0; sb < 5; ++sb)
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(tl + sb * QW + q0),
                 "r"(0));
}
__device__ __forceinline__ double combine5(const uint32_t (&r)[5][8], int t) {
  const long long lo = ((long long)(int32_t)r[1][t] << 24) + ((long long)(int32_t)r[2][t] << 16) +
                       ((long long)(int32_t)r[3][t] << 8) + (long long)(int32_t)r[4][t];
  return fma((double)(int32_t)r[0][t], 4294967296.0, (double)lo);
}
__device__ __forceinline__ void ld_v4_rw(const double* p, double& a, double& b, double& c, double& d) {
  asm volatile("ld.global.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}
// streamed read-only rows: no L1 allocation (the stream would evict the few
// spilled registers of a 96-register epilogue from L1)
__device__ __forceinline__ void ld_v4_stream(const double* p, double& a, double& b, double& c, double& d) {
  asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}

// L2 prefetch of a contiguous global range (bulk, no registers / smem)
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
// Transposed warp reduction of 8 per-lane values (8 columns): 9 shuffles
// instead of 40; the result for column c = 4 b4 + 2 b3 + b2 (bits of the
// lane index) ends up in the four lanes of that group.  Fixed pattern, so
// deterministic.
template <bool MAX>
__device__ __forceinline__ double treduce8(const double (&v)[8]) {
  const int l = threadIdx.x & 31;
  const bool b4 = l & 16, b3 = l & 8, b2 = l & 4;
  auto op = [](double a, double b) { return MAX ? fmax(a, b) : a + b; };
  double w[4], x[2];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const double send = b4 ? v[i] : v[i + 4], keep = b4 ? v[i + 4] : v[i];
    w[i] = op(keep, __shfl_xor_sync(0xffffffffu, send, 16));
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const double send = b3 ? w[i] : w[i + 2], keep = b3 ? w[i + 2] : w[i];
    x[i] = op(keep, __shfl_xor_sync(0xffffffffu, send, 8));
  }
  double y = op(b2 ? x[1] : x[0], __shfl_xor_sync(0xffffffffu, b2 ? x[0] : x[1], 4));
  y = op(y, __shfl_xor_sync(0xffffffffu, y, 2));
  return op(y, __shfl_xor_sync(0xffffffffu, y, 1));
}
__device__ __forceinline__ int treduce8_col() {
  const int l = threadIdx.x & 31;
  return ((l >> 4) & 1) * 4 + ((l >> 3) & 1) * 2 + ((l >> 2) & 1);
}

template <int QW, int EPI = EPI_PLAIN, int NPA = 4>
__global__ void __launch_bounds__(BAND_NTHREADS, 1)
    band_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                int n_mblocks, int nk, int band_offset, const double* __restrict__ row_scale,
                const double* __restrict__ op_scale, double* __restrict__ out, int64_t rows_real,
                unsigned long long* __restrict__ out_colmax, const Status* __restrict__ st,
                const __grid_constant__ BandStep bs) {
  using BC = BandCfg<QW, NPA>;
  constexpr int A_ST = NPA * BM * KT;
  if (st && st->done) return;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* sm = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int nst = nk / KT;                          // band stages
  unsigned char* band = sm;                         // [nst][NPA planes][128][64]
  unsigned char* ring = sm + (size_t)nst * A_ST;    // [BSTAGES][4 QW][64]
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + BSTAGES * BC::B_STAGE);
  uint64_t* empty = full + BSTAGES;
  uint64_t* band_full = empty + BSTAGES;
  uint64_t* tfull = band_full + 1;  // [BAND_SETS]
  uint64_t* tempty = tfull + BAND_SETS;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + BAND_SETS);
  double* gam_s = reinterpret_cast<double*>(tempty + BAND_SETS + 1);  // [QW] gamma (EPI_UPD)
  // after the last tile: [BAND_EPI_WARPS][2][QW] per-warp folds (the ring is idle by then)
  unsigned long long* cmax = reinterpret_cast<unsigned long long*>(ring);
  double* fold = reinterpret_cast<double*>(ring) + BAND_EPI_WARPS * QW;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < BSTAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(band_full, 1);
    for (int b = 0; b < BAND_SETS; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 32 * BAND_EPI_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    tma_prefetch(&map_a);
    tma_prefetch(&map_b);
  }
  if (EPI == EPI_UPD && threadIdx.x >= 64 && threadIdx.x < 64 + QW) {
    const int q = threadIdx.x - 64;
    const double pi = bs.beta * bs.vv[q] + bs.pap[q];
    const double g = pi != 0.0 ? bs.rho[q] / pi : 0.0;  // safe_ratio
    gam_s[q] = g;
    if (blockIdx.x == 0) {
      bs.gam_out[q] = g;
      if (q < bs.q_real && pi == 0.0) bs.frozen[q] = 1;
      bs.reset[q] = 0ull;
    }
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_holder;
  if (warp >= 2 && warp < 6) tmem_zero_all(tmem, warp & 3);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");

  if (warp == 0) {
    if (lane == 0) {
      // band once, then the operand windows of every tile
      mbar_expect_tx(band_full, (uint32_t)(nst * A_ST));
      for (int s = 0; s < nst; ++s) tma_load_3d(band + (size_t)s * A_ST, &map_a, band_full, s * KT, 0, 0);
      int stage = 0;
      uint32_t phase = 0;
      for (int mb = blockIdx.x; mb < n_mblocks; mb += gridDim.x) {
        const int k0 = mb * BM + band_offset;
        if (EPI == EPI_COMB || EPI == EPI_UPD) {
          // the tile's P (and R) rows are one contiguous block: pull them into L2
          // now, a tile or more before the epilogue loads them
          prefetch_l2(bs.P + (int64_t)mb * BM * bs.ld, (uint32_t)(BM * bs.ld * sizeof(double)));
          if (EPI == EPI_UPD) prefetch_l2(bs.R + (int64_t)mb * BM * bs.ld, (uint32_t)(BM * bs.ld * sizeof(double)));
        }
        for (int s = 0; s < nst; ++s) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (OZ_VARIANT >= 4) {
            mbar_arrive(&full[stage]);  // timing variants: no operand loads
          } else {
            mbar_expect_tx(&full[stage], BC::B_STAGE);
            tma_load_4d(ring + stage * BC::B_STAGE, &map_b, &full[stage], 0, 0, 0, (k0 + s * KT) >> 6);
          }
          if (++stage == BSTAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc0 = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BM >> 4) << 24);
      mbar_wait(band_full, 0);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int mb = blockIdx.x; mb < n_mblocks; mb += gridDim.x, ++it) {
        const int buf = it % BAND_SETS;
        mbar_wait(&tempty[buf], ((it / BAND_SETS) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t tset = tmem + buf * BAND_SET_COLS;
        for (int s = 0; s < nst; ++s) {
          mbar_wait(&full[stage], phase);
          asm volatile("tcgen05.fence::after_thread_sync;");
          if (OZ_VARIANT != 1)
            issue_stage<QW, false, NPA>(smem_u32(band + (size_t)s * A_ST), smem_u32(ring + stage * BC::B_STAGE),
                                        tset, idesc0);
          mma_commit(&empty[stage]);
          if (++stage == BSTAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit(&tfull[buf]);
      }
    }
  } else {
    const int quarter = warp & 3, grp = (warp - 2) >> 2;
    const int q0 = grp * 8;
    const bool active = q0 < QW;  // QW < 32: the surplus column groups only keep the barrier phases
    const int row_in_tile = quarter * 32 + lane;
    unsigned long long cm[8];
    double acc0[8], acc1[8];
    // EPI_UPD: running per-column values of this lane's column treduce8_col()
    // (a NaN residual stops the solve through ||R||^2 before the bound is used)
    double acc_rho = 0.0, acc_rn = 0.0, acc_w = 0.0;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      cm[t] = 0ull;
      acc0[t] = 0.0;
      acc1[t] = 0.0;
    }
    // the band's output rows all carry the same power-of-two scale (hrows holds
    // copies): one load before the loop, not a dependent load per tile (ncu:
    // a quarter of the Phi P launch's stall samples sat on that load)
    const double band_scale = row_scale[0] * (65536.0 / (SCALE30 * SCALE30));
    int it = 0;
    for (int mb = blockIdx.x; mb < n_mblocks; mb += gridDim.x, ++it) {
      const int buf = it % BAND_SETS;
      const int64_t row = (int64_t)mb * BM + row_in_tile;
      const double scale = row < rows_real ? band_scale : 0.0;
      double pv[8], rr[8];
      double alpha_j = 0.0, mv = 0.0;
      if ((EPI == EPI_COMB || EPI == EPI_UPD) && active) {
        alpha_j = bs.alpha[row];
        const double* prow = bs.P + row * bs.ld + q0;
        ld_v4_stream(prow, pv[0], pv[1], pv[2], pv[3]);
        ld_v4_stream(prow + 4, pv[4], pv[5], pv[6], pv[7]);
      }
      if (EPI == EPI_UPD && active) {
        mv = bs.minv[row * bs.ngroups];
        const double* rrow = bs.R + row * bs.ld + q0;
        ld_v4_rw(rrow, rr[0], rr[1], rr[2], rr[3]);
        ld_v4_rw(rrow + 4, rr[4], rr[5], rr[6], rr[7]);
      }
      mbar_wait(&tfull[buf], (it / BAND_SETS) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t tl = tmem + buf * BAND_SET_COLS + ((uint32_t)(quarter * 32) << 16);
      if (EPI == EPI_UPD && active && OZ_VARIANT != 3 && OZ_VARIANT != 4) {
        // two passes of 4 columns (register budget: 18 warps -> 96 per thread)
        double wm[8];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint32_t r4[5][4];
          tmem_rows4<QW>(tl, q0 + 4 * h, r4);
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const int q = q0 + 4 * h + t;
            const double u = combine5n<4>(r4, t) * (scale * __ldg(op_scale + q));
            const double psi = bs.beta * u + alpha_j * pv[4 * h + t];
            const double rn = rr[4 * h + t] - psi * gam_s[q];
            rr[4 * h + t] = rn;
            wm[4 * h + t] = fabs(bs.printed ? rn : (q < bs.q_real ? rn * mv : 0.0));
          }
        }
        double* rrow = bs.R + row * bs.ld + q0;
        st_v4(rrow, rr[0], rr[1], rr[2], rr[3]);
        st_v4(rrow + 4, rr[4], rr[5], rr[6], rr[7]);
        // per-tile column reductions, transposed across the warp; one lane per
        // 4 keeps the running value of its column (c = treduce8_col())
        const double m8 = treduce8<true>(wm);
        acc_w = fmax(acc_w, m8);
#pragma unroll
        for (int t = 0; t < 8; ++t) rr[t] = rr[t] * rr[t];
        acc_rn += treduce8<false>(rr);
#pragma unroll
        for (int t = 0; t < 8; ++t) rr[t] = (q0 + t < bs.q_real) ? rr[t] * mv : 0.0;
        acc_rho += treduce8<false>(rr);
      } else if (active && OZ_VARIANT != 3 && OZ_VARIANT != 4) {
        uint32_t r[5][8];
        tmem_rows8<QW>(tl, q0, r);
        double v[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const double u = combine5(r, t) * (scale * __ldg(op_scale + q0 + t));
          if (EPI == EPI_COMB) {
            v[t] = bs.beta * u + alpha_j * pv[t];
            acc0[t] += pv[t] * v[t];
          } else {
            v[t] = u;
            if (EPI == EPI_FWD) acc0[t] += u * u;
            if (EPI == EPI_FWD || out_colmax) {
              const unsigned long long m = (unsigned long long)__double_as_longlong(u) & 0x7fffffffffffffffull;
              cm[t] = m > cm[t] ? m : cm[t];
            }
          }
        }
        double* o = out + row * (EPI == EPI_COMB ? bs.ld : QW) + q0;
        st_v4(o, v[0], v[1], v[2], v[3]);
        st_v4(o + 4, v[4], v[5], v[6], v[7]);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;");
      asm volatile("tcgen05.fence::before_thread_sync;");
      mbar_arrive(&tempty[buf]);
    }
    // per-warp folds of the owned columns into this warp's smem slices (zeros elsewhere)
    const bool want_max = out_colmax || EPI == EPI_FWD || EPI == EPI_UPD;
    const int nsum = EPI == EPI_UPD ? 2 : (EPI == EPI_PLAIN ? 0 : 1);
    unsigned long long* slice = cmax + (warp - 2) * QW;
    double* fsl = fold + (warp - 2) * 2 * QW;
    for (int q = lane; q < QW; q += 32) {
      slice[q] = 0ull;
      fsl[q] = 0.0;
      fsl[QW + q] = 0.0;
    }
    __syncwarp();
    if (EPI == EPI_UPD) {  // lanes 4 c hold column c of this warp's group
      const int cc = treduce8_col();
      if ((lane & 3) == 0 && active) {
        slice[q0 + cc] = (unsigned long long)__double_as_longlong(acc_w);
        fsl[q0 + cc] = acc_rho;
        fsl[QW + q0 + cc] = acc_rn;
      }
    }
#pragma unroll
    for (int t = 0; t < 8 && EPI != EPI_UPD; ++t) {
      unsigned long long m = cm[t];
      double a = acc0[t], b = acc1[t];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        if (want_max) {
          const unsigned long long x = __shfl_xor_sync(0xffffffffu, m, off);
          m = x > m ? x : m;
        }
        if (nsum >= 1) a += __shfl_xor_sync(0xffffffffu, a, off);
        if (nsum >= 2) b += __shfl_xor_sync(0xffffffffu, b, off);
      }
      if (lane == 0 && active) {
        slice[q0 + t] = m;
        fsl[q0 + t] = a;
        fsl[QW + q0 + t] = b;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  unsigned long long* maxout = EPI == EPI_UPD ? bs.wmax : out_colmax;
  if (maxout && threadIdx.x < QW) {
    unsigned long long m = cmax[threadIdx.x];
    for (int w = 1; w < BAND_EPI_WARPS; ++w) m = cmax[w * QW + threadIdx.x] > m ? cmax[w * QW + threadIdx.x] : m;
    atomicMax(&maxout[threadIdx.x], m);
  }
  if (EPI != EPI_PLAIN) {
    const int nsum = EPI == EPI_UPD ? 2 : 1;
    if (threadIdx.x < nsum * QW) {
      const int v = threadIdx.x / QW, q = threadIdx.x % QW;
      double a = 0.0;
      for (int w = 0; w < BAND_EPI_WARPS; ++w) a += fold[w * 2 * QW + v * QW + q];  // fixed warp order
      bs.partials[((int64_t)blockIdx.x * nsum + v) * QW + q] = a;
    }
    double* outs[2] = {bs.out0, bs.out1};
    // fold scratch after the per-warp slices (the ring is idle)
    last_block_reduce(bs.ticket, bs.partials, QW, nsum, outs, fold + BAND_EPI_WARPS * 2 * QW);
  }
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// smallest power of two >= m (m > 0, finite), exact via frexp
__device__ __forceinline__ double pow2_ceil(double m) {
  int e;
  const double f = frexp(m, &e);  // m = f 2^e, f in [0.5, 1)
  return f == 0.5 ? ldexp(1.0, e - 1) : ldexp(1.0, e);
}

// ---------------------------------------------------------------------------
// operand quantisation: column q of  M[k][qoff+q] * pre[k]  (k < k_real) ->
// signed base-256 digits of round(x / s_q * 2^30), planes [4][QW][k_pad].
// s_q = 2^ceil(log2 max_k |M pre|); a non-finite column max makes s_q NaN so
// divergence still surfaces in the contraction output.
__device__ __forceinline__ void digits4(double x, int8_t d[4]) {
  long long v = llrint(x);
#pragma unroll
  for (int a = 3; a >= 0; --a) {
    const int8_t lo = (int8_t)(v & 0xFF);
    d[a] = lo;
    v = (v - lo) >> 8;
  }
}

// explicit column max (operands that did not come out of a fused producer)
template <typename T>
__global__ void k_colmax(int64_t k_real, int ldm, int qoff, int qw, const T* __restrict__ M,
                         const double* __restrict__ pre, unsigned long long* __restrict__ colmax,
                         const Status* __restrict__ st) {
  if (st && st->done) return;
  extern __shared__ double sm_cm[];
  const int rpb = blockDim.x / qw;
  const int q = threadIdx.x % qw;
  double m = 0.0;
  for (int64_t k = (int64_t)blockIdx.x * rpb + threadIdx.x / qw; k < k_real; k += (int64_t)gridDim.x * rpb) {
    const double v = fabs(pre ? (double)M[k * ldm + qoff + q] * pre[k] : (double)M[k * ldm + qoff + q]);
    m = (v > m || v != v) ? v : m;
  }
  sm_cm[threadIdx.x] = m;
  __syncthreads();
  if (threadIdx.x < qw) {
    double mm = 0.0;
    for (int r = threadIdx.x; r < (int)blockDim.x; r += qw) {
      const double x = sm_cm[r];
      mm = (x > mm || x != x) ? x : mm;
    }
    atomicMax(&colmax[threadIdx.x], (unsigned long long)__double_as_longlong(mm));
  }
}

__device__ __forceinline__ double col_scale(unsigned long long bits) {
  const double m = __longlong_as_double((long long)bits);
  if (!(m <= 1.7976931348623157e308)) return __longlong_as_double(0x7ff8000000000000ll);  // NaN / inf column
  return m == 0.0 ? 1.0 : pow2_ceil(m);
}

// Operand quantisation, one warp per 16-row K chunk: lane q < QW owns column
// q, loads its 16 values (each warp load is one contiguous row of the block),
// splits them into signed base-256 digits and stores 16 K bytes per digit
// plane (one 16-B store per plane into the K-blocked layout).  No shared
// memory, 16 independent loads in flight per lane.  The column maxima come
// fused out of the producing kernel.  `reset` (may be null) is zeroed by
// block 0 for the next fused column max.
constexpr int QCHUNK_K = 16;
template <typename T, int QW>
__global__ void __launch_bounds__(256, 3)
    k_quantize(int64_t k_real, int64_t k_pad, int ldm, int qoff, const T* __restrict__ M,
               const double* __restrict__ pre, const unsigned long long* __restrict__ colmax,
               double* __restrict__ scale_out, int8_t* __restrict__ planes, unsigned long long* __restrict__ reset,
               const Status* __restrict__ st) {
  if (st && st->done) return;
  if (blockIdx.x == 0 && threadIdx.x < QW) scale_out[threadIdx.x] = col_scale(colmax[threadIdx.x]);
  if (blockIdx.x == 0 && reset && threadIdx.x < 32) reset[threadIdx.x] = 0ull;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool act = lane < QW;
  const double is = act ? SCALE30 / col_scale(colmax[lane]) : 0.0;  // NaN for a non-finite column
  // the block's 8 warps cover 128 rows = two K-blocks; their digit words are
  // staged in smem in the K-blocked layout (64-B rows padded to 80 B) and
  // leave as whole 64-B lines (a 16-B store per lane leaves half-written
  // sectors that L2 has to merge or read-modify-write)
  __shared__ uint4 stage[2 * 4 * QW * 5];
  const int64_t ngroups = k_pad / 128;
  for (int64_t g = blockIdx.x; g < ngroups; g += gridDim.x) {
    const int64_t k0 = g * 128 + warp * QCHUNK_K;
    if (act) {
      double x[QCHUNK_K];
      if (k0 + QCHUNK_K <= k_real) {  // full chunk: 16 independent loads in flight
        const T* mp = M + k0 * ldm + qoff + lane;
#pragma unroll
        for (int r = 0; r < QCHUNK_K; ++r) x[r] = (double)mp[r * ldm];
        if (pre) {
#pragma unroll
          for (int r = 0; r < QCHUNK_K; ++r) x[r] *= __ldg(pre + k0 + r);
        }
      } else {
#pragma unroll
        for (int r = 0; r < QCHUNK_K; ++r) {
          const int64_t k = k0 + r;
          x[r] = k < k_real ? (double)M[k * ldm + qoff + lane] * (pre ? __ldg(pre + k) : 1.0) : 0.0;
        }
      }
      // |x is| <= 2^30, so v fits int32 and its four balanced base-256 digits
      // (those of digits4) are the bytes of (v + 0x80808080) ^ 0x80808080; a
      // 4 x 4 byte transpose per 4 rows packs them plane by plane
      uint32_t w[4][QCHUNK_K / 4];
      const bool ok = is == is;
#pragma unroll
      for (int j = 0; j < QCHUNK_K / 4; ++j) {
        uint32_t u[4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
          u[i] = ok ? (((uint32_t)__double2int_rn(x[4 * j + i] * is) + 0x80808080u) ^ 0x80808080u) : 0u;
        const uint32_t A = __byte_perm(u[0], u[1], 0x5140), B = __byte_perm(u[0], u[1], 0x7362);
        const uint32_t C = __byte_perm(u[2], u[3], 0x5140), E = __byte_perm(u[2], u[3], 0x7362);
        w[3][j] = __byte_perm(A, C, 0x5410);  // byte 0 (least significant digit)
        w[2][j] = __byte_perm(A, C, 0x7632);
        w[1][j] = __byte_perm(B, E, 0x5410);
        w[0][j] = __byte_perm(B, E, 0x7632);  // byte 3 (most significant digit)
      }
      const int kb = warp >> 2, part = warp & 3;  // K-block of the group, 16-B quarter of its 64-B rows
#pragma unroll
      for (int a = 0; a < 4; ++a) stage[((kb * 4 + a) * QW + lane) * 5 + part] = make_uint4(w[a][0], w[a][1], w[a][2], w[a][3]);
    }
    __syncthreads();
    uint4* dst = reinterpret_cast<uint4*>(planes + kb_offset(QW, 0, 0, g * 128));
    for (int i = threadIdx.x; i < 2 * 4 * QW * 4; i += blockDim.x) dst[i] = stage[(i >> 2) * 5 + (i & 3)];
    __syncthreads();
  }
}

// Direction update of the fused convolution step (one column chunk, ldq ==
// QW, one preconditioner group) with the NEXT Phi P operand quantised on the
// fly: the stopping test, the paired X updates and P(u+1) = eta P(u) + M^-1 R
// exactly as k_direction, and P(u+1)'s K-blocked digit planes, written
// through a smem stage as whole 64-B lines like k_quantize -- so the separate
// quantiser launch and its 1 GB re-read of P per convolution step are gone.
// The column scale must be known before any P(u+1) value exists: it is the
// power of two above the bound |eta| max|P(u)| + max|M^-1 R(u+1)| (max|P(u)|
// from the previous launch, max|M^-1 R| from the EPI_UPD band epilogue), at
// most one bit coarser than the exact column maximum.  Also emitted: the
// exact column maxima of |P(u+1)| (the next bound) and <P(u+1), alpha
// P(u+1)> (fixed-order block partials + last-block fold) for pi of the next
// step.  Each warp owns 16 rows of a 128-row group, lane = column.
template <int QW>
__global__ void __launch_bounds__(256, 2)
    k_direction_q(int64_t rows, int q_real, int step, int max_steps, double tol, int printed,
                  double* __restrict__ P, const double* __restrict__ R, const double* __restrict__ minv,
                  const double* __restrict__ alpha, Scalars sc, const unsigned long long* __restrict__ pmax_cur,
                  unsigned long long* __restrict__ pmax_next, const unsigned long long* __restrict__ wmax,
                  unsigned long long* __restrict__ reset, double* __restrict__ scale_out,
                  int8_t* __restrict__ planes, double* __restrict__ pap, unsigned* ticket, Status* st,
                  Status* mirror, double* X, double* Pdst, const double* Pprev) {
  {
    // finished by an EARLIER step: nothing to do (see k_direction)
    const volatile Status* vs = st;
    const int done = vs->done;
    __threadfence();
    const int sdone = vs->steps;
    if (done && !(step >= 1 && sdone == step)) {
      if (mirror && blockIdx.x == 0 && threadIdx.x == 0) {
        *mirror = *st;
        __threadfence_system();
      }
      return;
    }
  }
  __shared__ uint4 stage[2 * 4 * QW * 5];
  __shared__ double red[8][2][QW];
  __shared__ double fold_sm[256];
  const int cur = step & 1, nxt = (step + 1) & 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool act = lane < QW;
  const int q = lane;
  if (step == 0) {
    double b2 = 0.0;
    for (int c = 0; c < QW; ++c) b2 += sc.bn2[c];
    if (blockIdx.x == 0 && threadIdx.x == 0) st->bnorm = sqrt(b2);
  } else {
    double r2 = 0.0, b2 = 0.0;
    for (int c = 0; c < QW; ++c) r2 += sc.rn2[c];
    for (int c = 0; c < QW; ++c) b2 += sc.bn2[c];
    const double delta = sqrt(r2) / sqrt(b2);
    const bool finite = isfinite(delta);
    const bool conv = finite && delta <= tol;
    const bool stop = !finite || conv || step >= max_steps;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      volatile Status* vs = st;
      vs->steps = step;
      vs->delta = delta;
      vs->converged = conv ? 1 : 0;
      vs->diverged = finite ? 0 : 1;
      __threadfence();
      if (stop) vs->done = 1;
      if (mirror) {
        *mirror = *st;
        __threadfence_system();
      }
    }
    if (stop) {  // the pending solution updates
      const bool pair = (step & 1) == 0 && Pprev;
      for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < rows * QW;
           e += (int64_t)gridDim.x * blockDim.x) {
        const int qq = (int)(e % QW);
        double x = X[e];
        if (pair) x = x + Pprev[e] * sc.gam[nxt][qq];
        X[e] = x + P[e] * sc.gam[cur][qq];
      }
      return;
    }
  }
  double eta = 0.0, is = 0.0, gm = 0.0, gp = 0.0;
  const bool upd_x = X && step >= 1 && (!Pprev || (step & 1) == 0);
  const bool pair = upd_x && Pprev;
  if (act) {
    eta = safe_ratio(sc.rho_new[q], sc.rho[cur][q]);
    const double bound = fabs(eta) * __longlong_as_double((long long)pmax_cur[q]) +
                         __longlong_as_double((long long)wmax[q]);
    const double s = !(bound <= 1.7976931348623157e308) ? __longlong_as_double(0x7ff8000000000000ll)
                                                         : (bound == 0.0 ? 1.0 : pow2_ceil(bound));
    is = SCALE30 / s;
    if (blockIdx.x == 0) scale_out[q] = s;
    if (upd_x) gm = sc.gam[cur][q];
    if (pair) gp = sc.gam[nxt][q];
  }
  if (!Pdst) Pdst = P;
  const bool ok = is == is;
  double pmx = 0.0, pacc = 0.0;
  const int64_t ngrp = rows / 128;
  for (int64_t g = blockIdx.x; g < ngrp; g += gridDim.x) {
    const int64_t k0 = g * 128 + warp * QCHUNK_K;
    if (act) {
      uint32_t w[4][QCHUNK_K / 4];
#pragma unroll
      for (int sub = 0; sub < QCHUNK_K / 4; ++sub) {
        double r[4], p[4], x[4], pp[4], mv[4], al[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int64_t j = k0 + 4 * sub + i, e = j * QW + q;
          r[i] = R[e];
          p[i] = P[e];
          if (upd_x) x[i] = X[e];
          if (pair) pp[i] = Pprev[e];
          mv[i] = __ldg(minv + j);
          al[i] = __ldg(alpha + j);
        }
        uint32_t u[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int64_t j = k0 + 4 * sub + i, e = j * QW + q;
          if (upd_x) X[e] = (pair ? x[i] + pp[i] * gp : x[i]) + p[i] * gm;
          const double wv = (q < q_real) ? r[i] * mv[i] : 0.0;
          const double pn = p[i] * eta + (printed ? r[i] : wv);
          Pdst[e] = pn;
          const double a = fabs(pn);
          pmx = (a > pmx || a != a) ? a : pmx;
          pacc += pn * (al[i] * pn);
          u[i] = ok ? (((uint32_t)__double2int_rn(pn * is) + 0x80808080u) ^ 0x80808080u) : 0u;
        }
        const uint32_t A = __byte_perm(u[0], u[1], 0x5140), B = __byte_perm(u[0], u[1], 0x7362);
        const uint32_t C = __byte_perm(u[2], u[3], 0x5140), E = __byte_perm(u[2], u[3], 0x7362);
        w[3][sub] = __byte_perm(A, C, 0x5410);
        w[2][sub] = __byte_perm(A, C, 0x7632);
        w[1][sub] = __byte_perm(B, E, 0x5410);
        w[0][sub] = __byte_perm(B, E, 0x7632);
      }
      const int kb = warp >> 2, part = warp & 3;
#pragma unroll
      for (int a = 0; a < 4; ++a) stage[((kb * 4 + a) * QW + lane) * 5 + part] = make_uint4(w[a][0], w[a][1], w[a][2], w[a][3]);
    }
    __syncthreads();
    uint4* dst = reinterpret_cast<uint4*>(planes + kb_offset(QW, 0, 0, g * 128));
    for (int i = threadIdx.x; i < 2 * 4 * QW * 4; i += blockDim.x) dst[i] = stage[(i >> 2) * 5 + (i & 3)];
    __syncthreads();
  }
  if (act) {
    red[warp][0][q] = pmx;
    red[warp][1][q] = pacc;
  }
  __syncthreads();
  if (threadIdx.x < QW) {
    double m = 0.0, a = 0.0;
    for (int ww = 0; ww < 8; ++ww) {
      const double x = red[ww][0][threadIdx.x];
      m = (x > m || x != x) ? x : m;
      a += red[ww][1][threadIdx.x];  // fixed warp order
    }
    atomicMax(&pmax_next[threadIdx.x], (unsigned long long)__double_as_longlong(m));
    sc.partials[(int64_t)blockIdx.x * QW + threadIdx.x] = a;
  }
  if (blockIdx.x == 0 && threadIdx.x < QW) {
    sc.rho[nxt][threadIdx.x] = sc.rho_new[threadIdx.x];
    if (reset) reset[threadIdx.x] = 0ull;
  }
  double* outs[1] = {pap};
  last_block_reduce(ticket, sc.partials, QW, 1, outs, fold_sm);
}

// ---- dictionary conversion (once per dictionary) ---------------------------
// row scales r_i = 2^ceil(log2 max_j |Phi_ij|)
template <typename PT>
__global__ void k_phi_rowscale(const PT* __restrict__ phi, int64_t ld, int64_t n_real, int64_t d_real,
                               double* __restrict__ rs, bool raw = false) {
  const int64_t i = blockIdx.x;
  double m = 0.0;
  for (int64_t j = threadIdx.x; j < d_real; j += blockDim.x) m = fmax(m, fabs((double)phi[i * ld + j]));
  __shared__ double red[256];
  red[threadIdx.x] = m;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) rs[i] = raw ? red[0] : ((i < n_real && red[0] > 0) ? pow2_ceil(red[0]) : 1.0);
}

// raw row maxima (max-reduced over the column shards) -> power-of-two scales
__global__ void k_rows_pow2(int64_t n_real, int64_t n_pad, double* __restrict__ rs) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_pad; i += (int64_t)gridDim.x * blockDim.x)
    rs[i] = (i < n_real && rs[i] > 0) ? pow2_ceil(rs[i]) : 1.0;
}

// column scales c_j = 2^ceil(log2 max_i |Phi_ij| / r_i)
template <typename PT>
__global__ void k_phi_colscale(const PT* __restrict__ phi, int64_t ld, int64_t n_real, int64_t d_pad,
                               const double* __restrict__ rs, double* __restrict__ cs) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= d_pad) return;
  double m = 0.0;
  for (int64_t i = 0; i < n_real; ++i) m = fmax(m, fabs((double)phi[i * ld + j]) / rs[i]);
  cs[j] = m > 0 ? pow2_ceil(m) : 1.0;
}

// K-major copy of the digit planes for Phi^T V: planesT[a][j][i] = planes[a][i][j]
// (64 x 64-byte tiles; each thread transposes one 4 x 4 byte block in
// registers, a padded word tile in smem turns it into 16-B row stores).
// rows = Np, cols = Dp (multiples of 64); grid.z = plane.
__global__ void __launch_bounds__(256) k_planes_transpose(const int8_t* __restrict__ planes, int64_t rows,
                                                          int64_t cols, int8_t* __restrict__ planesT) {
  __shared__ uint32_t tile[64][17];  // transposed tile: 64 rows (j) x 16 words (64 i-bytes), padded
  const int64_t plane = blockIdx.z;
  const int8_t* src = planes + plane * rows * cols;
  int8_t* dst = planesT + plane * rows * cols;
  const int t = threadIdx.x;
  for (int64_t tb = blockIdx.x; tb < (rows / 64) * (cols / 64); tb += gridDim.x) {
    const int64_t i0 = (tb / (cols / 64)) * 64, j0 = (tb % (cols / 64)) * 64;
    const int br = t >> 4, bc = t & 15;  // 4 x 4 block (rows 4 br.., bytes 4 bc..)
    uint32_t w[4];
#pragma unroll
    for (int r = 0; r < 4; ++r)
      w[r] = *reinterpret_cast<const uint32_t*>(src + (i0 + 4 * br + r) * cols + j0 + 4 * bc);
    // byte transpose: out word c holds byte c of w[0..3]
    const uint32_t A = __byte_perm(w[0], w[1], 0x5140), B = __byte_perm(w[0], w[1], 0x7362);
    const uint32_t C = __byte_perm(w[2], w[3], 0x5140), E = __byte_perm(w[2], w[3], 0x7362);
    __syncthreads();  // the previous tile's reads are done
    tile[4 * bc + 0][br] = __byte_perm(A, C, 0x5410);
    tile[4 * bc + 1][br] = __byte_perm(A, C, 0x7632);
    tile[4 * bc + 2][br] = __byte_perm(B, E, 0x5410);
    tile[4 * bc + 3][br] = __byte_perm(B, E, 0x7632);
    __syncthreads();
    const int jj = t >> 2, part = t & 3;  // row jj of the transposed tile, words 4 part ..
    const uint4 v = make_uint4(tile[jj][4 * part], tile[jj][4 * part + 1], tile[jj][4 * part + 2],
                               tile[jj][4 * part + 3]);
    *reinterpret_cast<uint4*>(dst + (j0 + jj) * rows + i0 + 16 * part) = v;
  }
}

// digit planes [npa][Np][Dp] of round(Phi / (r c) * 2^(8 npa - 2)): npa = 4 is
// the 32-bit fixed-point dictionary, npa = 3 the 24-bit one (COFEM_OZAKI24).
// Dropping the low plane scales both the digits and the epilogue's 2^-30
// factor by 2^8, so the contraction kernels' epilogue constant is unchanged.
template <typename PT>
__global__ void k_phi_planes(const PT* __restrict__ phi, int64_t ld, int64_t np, int64_t dp,
                             const double* __restrict__ rs, const double* __restrict__ cs, int8_t* __restrict__ planes,
                             int npa) {
  const int64_t n = np * dp;
  const double sc = ldexp(1.0, 8 * npa - 2);
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / dp, j = e % dp;
    long long v = llrint((double)phi[i * ld + j] / (rs[i] * cs[j]) * sc);
    for (int a = npa - 1; a >= 0; --a) {
      const int8_t lo = (int8_t)(v & 0xFF);
      planes[(int64_t)a * n + e] = lo;
      v = (v - lo) >> 8;
    }
  }
}

}  // namespace oz
}  // namespace cofem
