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

// Epilogue with the PCG combine fused in (the conv Phi^T V launch): instead of
// U = Phi^T V the row writes Psi = beta U + alpha_j P_j (k_combine's formula)
// and accumulates p * psi per column for pi = <P, Psi>.
// P values of the row's column groups (group g of this half at pv[8 g ..]),
// loaded before the accumulator wait
template <int QW>
__host__ __device__ constexpr int comb_pv() { return (QW + 15) / 16 * 8; }
template <int QW, int HALF>
__device__ __forceinline__ void comb_prefetch(const double* __restrict__ prow, double (&pv)[comb_pv<QW>()]) {
#pragma unroll
  for (int q0 = HALF * 8, g = 0; q0 < QW; q0 += 16, ++g)
#pragma unroll
    for (int t = 0; t < 8; t += 4) ld_v4(prow + q0 + t, pv[8 * g + t], pv[8 * g + t + 1], pv[8 * g + t + 2], pv[8 * g + t + 3]);
}

template <int QW, int HALF>
__device__ __forceinline__ void epilogue_row_comb(uint32_t tset_lane, double scale, const double* __restrict__ op_scale,
                                                  double* o, const double (&pv)[comb_pv<QW>()], double alpha_j,
                                                  double beta, double (&pacc)[QW]) {
#pragma unroll
  for (int q0 = HALF * 8, g = 0; q0 < QW; q0 += 16, ++g) {
    double f[8], p[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      f[t] = scale * __ldg(op_scale + q0 + t);
      p[t] = pv[8 * g + t];
    }
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
      const long long lo = ((long long)(int32_t)r[1][t] << 24) + ((long long)(int32_t)r[2][t] << 16) +
                           ((long long)(int32_t)r[3][t] << 8) + (long long)(int32_t)r[4][t];
      const double u = fma((double)(int32_t)r[0][t], 4294967296.0, (double)lo) * f[t];
      v[t] = beta * u + alpha_j * p[t];
      pacc[q0 + t] += p[t] * v[t];
    }
    st_v4(o + q0, v[0], v[1], v[2], v[3]);
    st_v4(o + q0 + 4, v[4], v[5], v[6], v[7]);
  }
}

// band_kernel epilogue: 16 warps, warp (quarter, group) owns TMEM lane
// quarter `quarter` (32 rows) and the 8 columns [q0, q0 + 8) -- twice the
// warps of the contraction kernels' epilogue, so TMEM-load / global-memory
// latency of one warp hides behind the others.
template <int QW, bool TRACK>
__device__ __forceinline__ void epi8(uint32_t tl, int q0, double scale, const double* __restrict__ op_scale,
                                     double* o, unsigned long long (&cm)[8]) {
  uint32_t r[5][8];
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
  double v[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const long long lo = ((long long)(int32_t)r[1][t] << 24) + ((long long)(int32_t)r[2][t] << 16) +
                         ((long long)(int32_t)r[3][t] << 8) + (long long)(int32_t)r[4][t];
    v[t] = fma((double)(int32_t)r[0][t], 4294967296.0, (double)lo) * (scale * __ldg(op_scale + q0 + t));
  }
  st_v4(o + q0, v[0], v[1], v[2], v[3]);
  st_v4(o + q0 + 4, v[4], v[5], v[6], v[7]);
  if (TRACK) {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const unsigned long long m = (unsigned long long)__double_as_longlong(v[t]) & 0x7fffffffffffffffull;
      cm[t] = m > cm[t] ? m : cm[t];
    }
  }
}

template <int QW>
__device__ __forceinline__ void epi8_comb(uint32_t tl, int q0, double scale, const double* __restrict__ op_scale,
                                          double* o, const double (&p)[8], double alpha_j, double beta,
                                          double (&pacc)[8]) {
  uint32_t r[5][8];
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
  double v[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const long long lo = ((long long)(int32_t)r[1][t] << 24) + ((long long)(int32_t)r[2][t] << 16) +
                         ((long long)(int32_t)r[3][t] << 8) + (long long)(int32_t)r[4][t];
    const double u = fma((double)(int32_t)r[0][t], 4294967296.0, (double)lo) * (scale * __ldg(op_scale + q0 + t));
    v[t] = beta * u + alpha_j * p[t];
    pacc[t] += p[t] * v[t];
  }
  st_v4(o + q0, v[0], v[1], v[2], v[3]);
  st_v4(o + q0 + 4, v[4], v[5], v[6], v[7]);
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
// 128 x nk band (4 digit planes, nk = 128 + lpad bytes per row) is loaded into
// shared memory ONCE per CTA; the TMA ring then carries only the operand
// windows (4 QW x 64 B per stage), so the L2 -> SM traffic per output tile is
// the window alone.  Same significance-aligned, double-buffered accumulation
// and epilogue as contract_kernel.
constexpr int BSTAGES = 4;
// band_kernel accumulator sets: 5 significance blocks of QW <= 32 columns
// (160 TMEM columns), three sets in the 512-column allocation so the MMA
// issuer can run two tiles ahead of a slow epilogue
#ifndef BAND_SETS_OVERRIDE
constexpr int BAND_SETS = 3;
#else
constexpr int BAND_SETS = BAND_SETS_OVERRIDE;
#endif
constexpr int BAND_SET_COLS = 160;
constexpr int BAND_EPI_WARPS = 16;                      // 4 lane quarters x 4 column groups of 8
constexpr int BAND_NTHREADS = 64 + 32 * BAND_EPI_WARPS;  // warp 0 TMA, warp 1 MMA, warps 2..17 epilogue
template <int QW>
struct BandCfg {
  static constexpr int B_STAGE = 4 * QW * KT;
  static size_t smem(int nk) { return (size_t)nk * 4 * BM + (size_t)BSTAGES * B_STAGE + 1024 + 1280; }
};

// COMB (the Phi^T V launch of a PCG step): out = Psi = beta Phi^T V + alpha .* P
// (P / out row stride p_ld, column offset of the chunk already applied) and
// pi_out[q] = <P_q, Psi_q> through fixed-order block partials + last-block fold.
template <int QW, bool COMB = false>
__global__ void __launch_bounds__(BAND_NTHREADS, 1)
    band_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                int n_mblocks, int nk, int band_offset, const double* __restrict__ row_scale,
                const double* __restrict__ op_scale, double* __restrict__ out, int64_t rows_real,
                unsigned long long* __restrict__ out_colmax, const Status* __restrict__ st,
                const double* __restrict__ Pc = nullptr, int p_ld = 0, const double* __restrict__ alpha = nullptr,
                double beta = 0.0, double* pi_out = nullptr, double* partials = nullptr, unsigned* ticket = nullptr) {
  using C = Cfg<QW>;
  using BC = BandCfg<QW>;
  if (st && st->done) return;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* sm = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int nst = nk / KT;                          // band stages
  unsigned char* band = sm;                         // [nst][4 planes][128][64]
  unsigned char* ring = sm + (size_t)nst * A_STAGE; // [BSTAGES][4 QW][64]
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + BSTAGES * BC::B_STAGE);
  uint64_t* empty = full + BSTAGES;
  uint64_t* band_full = empty + BSTAGES;
  uint64_t* tfull = band_full + 1;  // [BAND_SETS]
  uint64_t* tempty = tfull + BAND_SETS;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + BAND_SETS);
  unsigned long long* cmax = reinterpret_cast<unsigned long long*>(ring);  // [BAND_EPI_WARPS][QW], after the last tile

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
      // band once, then the operand windows of every tile
      mbar_expect_tx(band_full, (uint32_t)(nst * A_STAGE));
      for (int s = 0; s < nst; ++s) tma_load_3d(band + (size_t)s * A_STAGE, &map_a, band_full, s * KT, 0, 0);
      int stage = 0;
      uint32_t phase = 0;
      for (int mb = blockIdx.x; mb < n_mblocks; mb += gridDim.x) {
        const int k0 = mb * BM + band_offset;
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
            issue_stage<QW, false>(smem_u32(band + (size_t)s * A_STAGE), smem_u32(ring + stage * BC::B_STAGE), tset,
                                   idesc0);
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
    double pacc[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      cm[t] = 0ull;
      pacc[t] = 0.0;
    }
    int it = 0;
    for (int mb = blockIdx.x; mb < n_mblocks; mb += gridDim.x, ++it) {
      const int buf = it % BAND_SETS;
      const int64_t row = (int64_t)mb * BM + row_in_tile;
      const double scale = row < rows_real ? row_scale[row] * (65536.0 / (SCALE30 * SCALE30)) : 0.0;
      double pv[8];
      double alpha_j = 0.0;
      if (COMB && active) {
        alpha_j = alpha[row];
        const double* prow = Pc + row * p_ld + q0;
        ld_v4(prow, pv[0], pv[1], pv[2], pv[3]);
        ld_v4(prow + 4, pv[4], pv[5], pv[6], pv[7]);
      }
      mbar_wait(&tfull[buf], (it / BAND_SETS) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t tl = tmem + buf * BAND_SET_COLS + ((uint32_t)(quarter * 32) << 16);
      if (active && OZ_VARIANT != 3 && OZ_VARIANT != 4) {
        if (COMB)
          epi8_comb<QW>(tl, q0, scale, op_scale, out + row * p_ld, pv, alpha_j, beta, pacc);
        else if (out_colmax)
          epi8<QW, true>(tl, q0, scale, op_scale, out + row * QW, cm);
        else
          epi8<QW, false>(tl, q0, scale, op_scale, out + row * QW, cm);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;");
      asm volatile("tcgen05.fence::before_thread_sync;");
      mbar_arrive(&tempty[buf]);
    }
    // per-warp folds of the owned columns into this warp's [QW] smem slice (zeros elsewhere)
    if (out_colmax) {
      unsigned long long* slice = cmax + (warp - 2) * QW;
      for (int q = lane; q < QW; q += 32) slice[q] = 0ull;
      __syncwarp();
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        unsigned long long m = cm[t];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          const unsigned long long x = __shfl_xor_sync(0xffffffffu, m, off);
          m = x > m ? x : m;
        }
        if (lane == 0 && active) slice[q0 + t] = m;
      }
    }
    if (COMB) {
      double* psl = reinterpret_cast<double*>(cmax) + (warp - 2) * QW;
      for (int q = lane; q < QW; q += 32) psl[q] = 0.0;
      __syncwarp();
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        double v = pacc[t];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        if (lane == 0 && active) psl[q0 + t] = v;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (out_colmax && threadIdx.x < QW) {
    unsigned long long m = cmax[threadIdx.x];
    for (int w = 1; w < BAND_EPI_WARPS; ++w) m = cmax[w * QW + threadIdx.x] > m ? cmax[w * QW + threadIdx.x] : m;
    atomicMax(&out_colmax[threadIdx.x], m);
  }
  if (COMB) {
    const double* psl = reinterpret_cast<const double*>(cmax);
    if (threadIdx.x < QW) {
      double v = 0.0;
      for (int w = 0; w < BAND_EPI_WARPS; ++w) v += psl[w * QW + threadIdx.x];  // fixed warp order
      partials[(int64_t)blockIdx.x * QW + threadIdx.x] = v;
    }
    double* outs[1] = {pi_out};
    last_block_reduce(ticket, partials, QW, 1, outs, reinterpret_cast<double*>(cmax) + BAND_EPI_WARPS * QW);
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
