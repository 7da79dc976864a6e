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
// (warp 0 TMA producer, warp 1 MMA issuer, warps 2..5 TMEM epilogue).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.cuh"

namespace cofem {
namespace oz {

constexpr int KT = 64;           // K bytes per stage (one SWIZZLE_64B row)
constexpr int BM = 128;          // output rows per tile (UMMA M)
constexpr int STAGES = 5;
constexpr int NTHREADS = 192;    // 6 warps
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
// The three dropped pairs (a + b >= 5) are worth <= 2^(8*1) / 2^(8*6) per
// digit product; with full-range low digits against leading digits of a few
// bits they still sit ~1e-10 below the result -- under the 2^-30
// quantisation of the factors -- while trimming a sixth of the tensor work
// (and with it power: the contraction runs at the 1 kW cap).  Dropping the
// a + b = 4 pairs as well measured 2.6e-8 relative error, so they stay.
// N_a = QW * min(4, 5 - a) rounded up to the UMMA granularity of 16 (the few
// extra B rows are real smem rows of the next plane; their accumulator
// columns are never read).
template <int QW>
struct Cfg {
  static constexpr int NB = 4 * QW;  // B tile rows: the four operand planes side by side
  static constexpr int B_STAGE = NB * KT;
  static constexpr int STAGE = A_STAGE + B_STAGE;
  static constexpr size_t SMEM = (size_t)STAGES * STAGE + 1024 + 256;
  __host__ __device__ static constexpr int nb_of(int a) { return a <= 1 ? 4 : 5 - a; }  // operand planes used
  __host__ __device__ static constexpr int n_of(int a) { return ((QW * nb_of(a) + 15) / 16) * 16; }
  __host__ __device__ static constexpr int col_of(int a) {
    return a == 0 ? 0 : a == 1 ? n_of(0) : a == 2 ? n_of(0) + n_of(1) : n_of(0) + n_of(1) + n_of(2);
  }
  static constexpr int TMEM_COLS = col_of(3) + n_of(3);
  static_assert(QW % 8 == 0 && QW <= 32, "QW in {8,16,24,32}");
  static_assert(STAGE % 1024 == 0, "stages must stay 1024-B aligned for the swizzle atoms");
  static_assert(TMEM_COLS <= 512, "accumulators must fit TMEM");
};

// Persistent contraction.  Work item w (< n_items) = (mb = w % n_mblocks,
// split s = w / n_mblocks): output rows [mb*128, +128), K range
// [s*k_per_split, min(+k_per_split, k_total)).  Writes fp64
// out[s][row][0:QW] = sum_k Phi(.)[row][k] * op[k][q] (already scaled).
//   MODE_FWD : rows are i, K is j; row scale r_i (A = digit planes, K-major)
//   MODE_BWD : rows are j, K is i; row scale c_j (A = the same planes, MN-major)
//   MODE_BAND: banded Toeplitz operator (convolution dictionaries): every
//     output tile sees the same 128 x k_per_split band matrix, so A's TMA
//     coordinate is relative to the tile: K range [mb*128 + band_offset,
//     + k_per_split); operand rows outside [0, K) arrive as TMA zero fill.
// Rows >= rows_real are written as zeros; out_colmax (may be null) collects
// the column maxima of |out| for the next quantisation (single-split modes).
enum { MODE_FWD = 0, MODE_BWD = 1, MODE_BAND = 2 };
template <int QW, int MODE>
__global__ void __launch_bounds__(NTHREADS, 1)
    contract_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                    int n_mblocks, int n_items, int k_per_split, int k_total, int band_offset,
                    const double* __restrict__ row_scale, const double* __restrict__ op_scale,
                    double* __restrict__ out, int64_t out_rows, int64_t rows_real,
                    unsigned long long* __restrict__ out_colmax, const Status* __restrict__ st) {
  constexpr bool BWD = MODE == MODE_BWD;
  using C = Cfg<QW>;
  if (st && st->done) return;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* sm = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + STAGES * C::STAGE);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 128);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    tma_prefetch(&map_a);
    tma_prefetch(&map_b);
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

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      int stage = 0;
      uint32_t phase = 0;
      for (int w = blockIdx.x; w < n_items; w += gridDim.x) {
        const int mb = w % n_mblocks, s = w / n_mblocks;
        const int k0 = MODE == MODE_BAND ? mb * BM + band_offset : s * k_per_split;
        const int k1 = MODE == MODE_BAND ? k0 + k_per_split : min(k0 + k_per_split, k_total);
        for (int k = k0; k < k1; k += KT) {
          mbar_wait(&empty[stage], phase ^ 1);
          unsigned char* sa = sm + stage * C::STAGE;
          unsigned char* sb = sa + A_STAGE;
          mbar_expect_tx(&full[stage], C::STAGE);
          if (MODE == MODE_BAND) {
            tma_load_3d(sa, &map_a, &full[stage], k - k0, 0, 0);
          } else if (!BWD) {
            tma_load_3d(sa, &map_a, &full[stage], k, mb * BM, 0);
          } else {
            tma_load_3d(sa, &map_a, &full[stage], mb * BM, k, 0);
            tma_load_3d(sa + A_STAGE / 2, &map_a, &full[stage], mb * BM + 64, k, 0);
          }
          tma_load_3d(sb, &map_b, &full[stage], k, 0, 0);
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
      uint32_t phase = 0, tphase = 0;
      for (int w = blockIdx.x; w < n_items; w += gridDim.x) {
        const int mb = w % n_mblocks, s = w / n_mblocks;
        const int k0 = MODE == MODE_BAND ? mb * BM + band_offset : s * k_per_split;
        const int k1 = MODE == MODE_BAND ? k0 + k_per_split : min(k0 + k_per_split, k_total);
        mbar_wait(tempty, tphase ^ 1);  // epilogue has drained the accumulators
        tphase ^= 1;
        asm volatile("tcgen05.fence::after_thread_sync;");
        for (int k = k0; k < k1; k += KT) {
          mbar_wait(&full[stage], phase);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t sa = smem_u32(sm + stage * C::STAGE);
          const uint32_t sb = sa + A_STAGE;
#pragma unroll
          for (int kk = 0; kk < 2; ++kk) {
            const uint64_t db = sdesc(sb + kk * 32, 16, 512);
#pragma unroll
            for (int a = 0; a < 4; ++a) {
              uint64_t da;
              if (!BWD) da = sdesc(sa + a * (BM * KT) + kk * 32, 16, 512);
              else da = sdesc(sa + a * (64 * KT) + kk * (32 * KT), A_STAGE / 2, 512);
              const uint32_t idesc = idesc0 | ((uint32_t)(C::n_of(a) >> 3) << 17);
              mma_i8(tmem + C::col_of(a), da, db, idesc, (k > k0 || kk > 0) ? 1u : 0u);
            }
          }
          mma_commit(&empty[stage]);  // frees the smem slot once these MMAs retire
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit(tfull);  // accumulators complete
      }
    }
  } else {
    // ---------------- epilogue: warps 2..5 -> TMEM lane quarters (warp % 4) ----------------
    const int quarter = warp & 3;
    const int row_in_tile = quarter * 32 + lane;
    uint32_t tphase = 0;
    for (int w = blockIdx.x; w < n_items; w += gridDim.x) {
      const int mb = w % n_mblocks, s = w / n_mblocks;
      mbar_wait(tfull, tphase);
      tphase ^= 1;
      asm volatile("tcgen05.fence::after_thread_sync;");
      double acc[QW];
#pragma unroll
      for (int q = 0; q < QW; ++q) acc[q] = 0.0;
      const uint32_t base = tmem + ((uint32_t)(quarter * 32) << 16);
#pragma unroll
      for (int a = 0; a < 4; ++a) {
#pragma unroll
        for (int b = 0; b < C::nb_of(a); ++b) {
          // digit weights 256^(3-a) * 256^(3-b) relative to 2^48
          const double wgt = (double)(1ull << (8 * (6 - a - b)));
#pragma unroll
          for (int q0 = 0; q0 < QW; q0 += 8) {
            uint32_t r[8];
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                           "=r"(r[7])
                         : "r"(base + C::col_of(a) + b * QW + q0));
            asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
            for (int t = 0; t < 8; ++t) acc[q0 + t] = fma((double)(int32_t)r[t], wgt, acc[q0 + t]);
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      mbar_arrive(tempty);
      const int64_t row = (int64_t)mb * BM + row_in_tile;
      const double rs = row < rows_real ? row_scale[row] * (1.0 / (SCALE30 * SCALE30)) : 0.0;
      double* o = out + ((int64_t)s * out_rows + row) * QW;
#pragma unroll
      for (int q = 0; q < QW; q += 2) {
        const double v0 = acc[q] * rs * op_scale[q], v1 = acc[q + 1] * rs * op_scale[q + 1];
        *reinterpret_cast<double2*>(o + q) = make_double2(v0, v1);
        if (out_colmax) {  // warp max over its 32 rows, one atomic per warp and column
          double m0 = fabs(v0), m1 = fabs(v1);
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) {
            const double o0 = __shfl_xor_sync(0xffffffffu, m0, off), o1 = __shfl_xor_sync(0xffffffffu, m1, off);
            m0 = (o0 > m0 || o0 != o0) ? o0 : m0;
            m1 = (o1 > m1 || o1 != o1) ? o1 : m1;
          }
          if (lane == 0) {
            atomicMax(&out_colmax[q], (unsigned long long)__double_as_longlong(m0));
            atomicMax(&out_colmax[q + 1], (unsigned long long)__double_as_longlong(m1));
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
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
    const double v = fabs((double)M[k * ldm + qoff + q] * pre[k]);
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

// Block-tiled quantisation: a 128-row x QW tile of M is staged through smem
// with coalesced loads, then each thread packs 4 rows of one column into one
// 32-bit word per digit plane (stores coalesced along k).  `reset` (may be
// null) is zeroed by block 0 for the next fused column max.
constexpr int QTILE = 128;
template <typename T, int QW>
__global__ void __launch_bounds__(256)
    k_quantize(int64_t k_real, int64_t k_pad, int ldm, int qoff, const T* __restrict__ M,
               const double* __restrict__ pre, const unsigned long long* __restrict__ colmax,
               double* __restrict__ scale_out, int8_t* __restrict__ planes, unsigned long long* __restrict__ reset,
               const Status* __restrict__ st) {
  if (st && st->done) return;
  __shared__ double inv_s[QW];
  __shared__ double tile[QTILE][QW + 1];
  if (threadIdx.x < QW) {
    const double sc = col_scale(colmax[threadIdx.x]);
    inv_s[threadIdx.x] = SCALE30 / sc;  // NaN for a non-finite column
    if (blockIdx.x == 0) scale_out[threadIdx.x] = sc;
  }
  if (blockIdx.x == 0 && reset && threadIdx.x < 32) reset[threadIdx.x] = 0ull;
  const int64_t ntile = k_pad / QTILE;
  for (int64_t tb = blockIdx.x; tb < ntile; tb += gridDim.x) {
    const int64_t k0 = tb * QTILE;
    __syncthreads();
    for (int e = threadIdx.x; e < QTILE * QW; e += blockDim.x) {
      const int r = e / QW, q = e % QW;
      const int64_t k = k0 + r;
      tile[r][q] = (k < k_real) ? (double)M[k * ldm + qoff + q] * pre[k] : 0.0;
    }
    __syncthreads();
    for (int w = threadIdx.x; w < (QTILE / 4) * QW; w += blockDim.x) {
      const int quad = w % (QTILE / 4), q = w / (QTILE / 4);
      const double is = inv_s[q];
      uint32_t word[4] = {0u, 0u, 0u, 0u};
      if (is == is) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          int8_t d[4];
          digits4(tile[quad * 4 + r][q] * is, d);
#pragma unroll
          for (int a = 0; a < 4; ++a) word[a] |= (uint32_t)(uint8_t)d[a] << (8 * r);
        }
      }
#pragma unroll
      for (int a = 0; a < 4; ++a)
        *reinterpret_cast<uint32_t*>(planes + ((int64_t)a * QW + q) * k_pad + k0 + quad * 4) = word[a];
    }
  }
}

// ---- dictionary conversion (once per dictionary) ---------------------------
// row scales r_i = 2^ceil(log2 max_j |Phi_ij|)
__global__ void k_phi_rowscale(const float* __restrict__ phi, int64_t ld, int64_t n_real, int64_t d_real,
                               double* __restrict__ rs) {
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
  if (threadIdx.x == 0) rs[i] = (i < n_real && red[0] > 0) ? pow2_ceil(red[0]) : 1.0;
}

// column scales c_j = 2^ceil(log2 max_i |Phi_ij| / r_i)
__global__ void k_phi_colscale(const float* __restrict__ phi, int64_t ld, int64_t n_real, int64_t d_pad,
                               const double* __restrict__ rs, double* __restrict__ cs) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= d_pad) return;
  double m = 0.0;
  for (int64_t i = 0; i < n_real; ++i) m = fmax(m, fabs((double)phi[i * ld + j]) / rs[i]);
  cs[j] = m > 0 ? pow2_ceil(m) : 1.0;
}

// digit planes [4][Np][Dp] of round(Phi / (r c) * 2^30)
__global__ void k_phi_planes(const float* __restrict__ phi, int64_t ld, int64_t np, int64_t dp,
                             const double* __restrict__ rs, const double* __restrict__ cs, int8_t* __restrict__ planes) {
  const int64_t n = np * dp;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / dp, j = e % dp;
    int8_t d[4];
    digits4((double)phi[i * ld + j] / (rs[i] * cs[j]) * SCALE30, d);
#pragma unroll
    for (int a = 0; a < 4; ++a) planes[(int64_t)a * n + e] = d[a];
  }
}

}  // namespace oz
}  // namespace cofem
