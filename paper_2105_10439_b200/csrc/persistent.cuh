// persistent.cuh -- a whole dense PCG solve in ONE cooperative launch.
//
// The multi-kernel step (quantise P, Phi P, sum the splits, quantise V,
// Phi^T V, combine, update, direction: 8 launches, ~130 us of tail and launch
// gaps around 2 x 0.68 ms of contraction at the headline size) becomes seven
// phases of one persistent kernel, separated by grid-wide barriers:
//
//   A  quantise P(u) (column scales from the fused maxima of the previous H)
//   B  Phi P on the int8 tensor cores (warp-specialised, as contract_kernel):
//      fp64 split-K partials
//   C  V = sum of the splits, column maxima of |r V|, ||V||^2 partials
//   D  quantise V; pi = beta ||V||^2 + <P, alpha P> (= <P, A P> without
//      forming A P), gamma = rho / pi
//   E  Phi^T V (K-major transposed planes): fp64 split-K partials
//   F  Psi = beta sum(splits) + alpha P on the fly (never stored),
//      R -= gamma Psi, per-column <R, M^-1 R> / ||R||^2 partials
//   H  stopping test (cg.py:141-148) on the folded ||R||; X += gamma P in
//      pairs of steps; P(u+1) = eta P(u) + M^-1 R (kernels.py step_direction),
//      the column maxima of |c P(u+1)| and <P(u+1), alpha P(u+1)> for the
//      next step
//
// The streaming phases (A, C, D, F, H) move whole 32-B sectors per thread
// (4 columns of a row) through L2 with all 16 warps; each thread owns a fixed
// set of rows, so every per-column partial has a fixed place in the fold.
// (Measured and dropped: finishing each 128-row block's C / F work on the
// epilogue warps of the CTA whose tile completes the block -- the fix-up
// lengthened the contraction tails more than it saved, and the block -> CTA
// assignment, hence the fold order, became timing dependent.)
//
// Every per-column scalar is folded from fixed-order per-CTA partials by
// EVERY CTA (identical sums, no broadcast round), so the whole solve is
// deterministic; the grid is one CTA per SM (cooperative launch: all
// co-resident), the stage ring doubles as the streaming phases' staging
// memory, and mutable data written by other CTAs is read through L2
// (ld.global.cg).  A barrier spin that exceeds 20 s traps instead of hanging
// the GPU.  Used for single-GPU dense dictionaries in the ozaki mode with
// K + 1 <= 32 right-hand sides; every other case runs the multi-kernel step.
#pragma once
#include "ozaki.cuh"

namespace cofem {
namespace oz {

// 16 warps: warp 0 TMA, warp 1 MMA, warps 2..9 epilogue in the contraction
// phases; all 16 stream in A / C / D / F / H (latency-bound passes over
// L2 / HBM: the extra warps are memory-level parallelism)
constexpr int PS_THREADS = 512;
constexpr int PS_WARPS = PS_THREADS / 32;
constexpr int PS_UNR = 4;             // rows per thread per loop trip in the streaming phases
constexpr int PS_VU = 1;              // rows per loop trip of the vector-mapped phases F / H
constexpr int PS_CTRL = 256;          // mbarriers + TMEM holder
constexpr int PS_STATE = 12 * 32 * 8; // per-column scalars (12 arrays of <= 32 doubles)
constexpr int PS_TIMES = 16;          // phase stamps per step: [0, 8) phase starts, [8, 16) CTA 0's work ends

template <int QW, int NPA = 4>
struct PsCfg {
  static constexpr size_t SMEM = (size_t)STAGES * Cfg<QW, NPA>::STAGE + 1024 + PS_CTRL + PS_STATE;
};

struct PcgPersistArgs {
  int64_t Np, Dp, N, D;
  int q_real;
  int f_mblocks, f_items, f_kps;  // Phi P: Np / 128 row blocks, (block, split) items, K per split (K = Dp)
  int b_mblocks, b_items, b_kps;  // Phi^T V: Dp / 128, items, K per split (K = Np)
  int f_nsplit, b_nsplit;
  const double* rowscale;  // r_i (Np)
  const double* colscale;  // c_j (Dp)
  double* P0;              // P(1) on entry; P(u) alternates P0 / P1
  double* P1;
  double* X;
  double* R;
  const double* minv;
  const double* alpha;
  double* vpart;  // [f_nsplit][Np][QW]
  double* ppart;  // [b_nsplit][Dp][QW]
  double* V;      // [Np][QW]
  int8_t* pq;     // K-blocked digit planes of diag(c) P
  int8_t* vq;     // K-blocked digit planes of diag(r) V
  unsigned long long* colmax_p;  // [32], valid for P(1) on entry
  unsigned long long* colmax_v;  // [32]
  double* red;                   // [grid][4][QW] per-CTA partials
  const double* rho1;            // rho of P(1)
  const double* bn2;             // ||B_q||^2
  int* frozen;
  double beta, tol;
  int max_steps, printed;
  Status* st;
  unsigned* bar;                 // [0] arrivals, [1] generation
  unsigned long long* times;     // optional [(max_steps + 1) * PS_TIMES] globaltimer stamps (CTA 0)
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

// grid-wide barrier over co-resident CTAs (sense by generation counter)
__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned arrived = atomicAdd(bar, 1u);
    if (arrived == gridDim.x - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(bar + 1), "r"(gen + 1) : "memory");
    } else {
      const unsigned long long t0 = gtimer();
      while (ld_acquire_u32(bar + 1) == gen) {
        if (gtimer() - t0 > 20000000000ull) __trap();  // a lost CTA: fail the launch, never hang the GPU
      }
    }
    __threadfence();
  }
  ++gen;
  __syncthreads();
}


// 32-B (4 x f64) accesses through L2: the streaming phases move whole sectors
// per thread (4x fewer memory instructions than per-column 8-B accesses)
__device__ __forceinline__ void ld4(const double* p, double (&v)[4]) {
  asm volatile("ld.global.cg.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p));
}
__device__ __forceinline__ void st4(double* p, const double (&v)[4]) {
  asm volatile("st.global.cg.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(v[0]), "d"(v[1]), "d"(v[2]), "d"(v[3])
               : "memory");
}

// vector thread map: thread t owns columns 4 (t % G) .. + 3 of rows
// blockIdx.x RPBV + t / G + k gridDim.x RPBV  (G = QW / 4 column groups)
template <int QW>
struct VMap {
  static constexpr int G = QW / 4;
  static constexpr int RPBV = PS_THREADS / G;
  bool on;
  int c0;
  int64_t r0, rstep;
  __device__ __forceinline__ VMap() {
    const int t = threadIdx.x;
    on = t < RPBV * G;
    c0 = 4 * (t % G);
    r0 = (int64_t)blockIdx.x * RPBV + t / G;
    rstep = (int64_t)gridDim.x * RPBV;
  }
};

// per-column fold of the vector map's per-thread 4-column values ->
// red[cta][slot + v][q] (fixed row order through smem; smr holds nv x 4 x 512)
template <int QW, int NV>
__device__ __forceinline__ void cta_col_sums4(double* smr, const double (&vals)[NV][4], double* red, int slot) {
  using M = VMap<QW>;
  const int t = threadIdx.x, nt = blockDim.x;
  constexpr int nv = NV;
  __syncthreads();
#pragma unroll
  for (int v = 0; v < nv; ++v)
#pragma unroll
    for (int c = 0; c < 4; ++c) smr[(v * 4 + c) * nt + t] = t < M::RPBV * M::G ? vals[v][c] : 0.0;
  __syncthreads();
  if (t < nv * QW) {
    const int v = t / QW, q = t % QW;
    double s = 0.0;
    for (int r = 0; r < M::RPBV; ++r) s += smr[(v * 4 + (q & 3)) * nt + r * M::G + (q >> 2)];
    __stcg(red + ((int64_t)blockIdx.x * 4 + slot + v) * QW + q, s);
  }
}

// column maxima of the vector map's per-thread 4-column maxima -> atomicMax(colmax)
template <int QW>
__device__ __forceinline__ void cta_col_max4(double* smr, const double (&m4)[4], unsigned long long* colmax) {
  using M = VMap<QW>;
  const int t = threadIdx.x, nt = blockDim.x;
  __syncthreads();
#pragma unroll
  for (int c = 0; c < 4; ++c) smr[c * nt + t] = t < M::RPBV * M::G ? m4[c] : 0.0;
  __syncthreads();
  if (t < QW) {
    double m = 0.0;
    for (int r = 0; r < M::RPBV; ++r) {
      const double x = smr[(t & 3) * nt + r * M::G + (t >> 2)];
      m = (x > m || x != x) ? x : m;
    }
    atomicMax(colmax + t, (unsigned long long)__double_as_longlong(m));
  }
}

__device__ __forceinline__ double nanmax(double m, double v) { return (v > m || v != v) ? v : m; }

// per-column fold of a CTA's per-thread values -> red[cta][slot + v][q]
// (thread t owns column t % QW; fixed row order through smem)
template <int QW>
__device__ __forceinline__ void cta_col_sums(double* smr, int nv, const double* vals, double* red, int slot) {
  const int t = threadIdx.x, nt = blockDim.x;
  constexpr int RPB = PS_THREADS / QW;
  __syncthreads();
  for (int v = 0; v < nv; ++v) smr[v * nt + t] = vals[v];
  __syncthreads();
  if (t < nv * QW) {
    const int v = t / QW, q = t % QW;
    double s = 0.0;
    for (int r = 0; r < RPB; ++r) s += smr[v * nt + r * QW + q];
    __stcg(red + ((int64_t)blockIdx.x * 4 + slot + v) * QW + q, s);
  }
}

// every CTA folds red[0..grid)[slot + v][q] for v < nv in the same fixed
// order: out[v * QW + q] (smem).  Groups of threads sum interleaved CTA
// subsets with 4 accumulators, then the groups combine in group order.
template <int QW>
__device__ __forceinline__ void fold_all(const double* red, int slot, int nv, double* smr, double* out) {
  const int t = threadIdx.x, nt = blockDim.x;
  const int npair = nv * QW;
  const int groups = nt / npair;
  const int g = t / npair, p = t % npair;
  double s = 0.0;
  if (g < groups) {
    const int v = p / QW, q = p % QW;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    const double* base = red + (int64_t)(slot + v) * QW + q;
    const int64_t st = (int64_t)groups * 4 * QW;  // one CTA stride of the subset
    int b = g;
    for (; b + 3 * groups < (int)gridDim.x; b += 4 * groups) {
      const double* p0 = base + (int64_t)b * 4 * QW;
      a0 += __ldcg(p0);
      a1 += __ldcg(p0 + st);
      a2 += __ldcg(p0 + 2 * st);
      a3 += __ldcg(p0 + 3 * st);
    }
    for (; b < (int)gridDim.x; b += groups) a0 += __ldcg(base + (int64_t)b * 4 * QW);
    s = (a0 + a1) + (a2 + a3);
  }
  __syncthreads();
  smr[t] = s;
  __syncthreads();
  if (t < npair) {
    double tot = 0.0;
    for (int gg = 0; gg < groups; ++gg) tot += smr[gg * npair + t];
    out[t] = tot;
  }
  __syncthreads();
}

// Phase A / D: quantise rows [0, k_pad) of M (QW columns, row stride QW),
// x = M pre -> K-blocked digit planes with scale 2^30 / s_q (s_q from the
// column maxima in s_scale).  A round is 256 rows (four K-blocks): warp w
// takes rows 16 w .. 16 w + 15, lanes q < QW one column each, all loads of
// the round (M, pre, alpha) issued up front; the digit words are staged in
// smem and leave as whole 64-B lines.
template <int QW>
__device__ __forceinline__ void quantize_phase(const double* __restrict__ M, int64_t k_real, int64_t k_pad,
                                               const double* __restrict__ pre, const double* s_scale,
                                               int8_t* __restrict__ planes, uint4* stage) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool act = lane < QW;
  const double is = act ? SCALE30 / s_scale[lane] : 0.0;
  const bool ok = is == is;
  const int64_t nround = (k_pad + 255) / 256;
  for (int64_t g = blockIdx.x; g < nround; g += gridDim.x) {
    const int64_t k0 = g * 256 + warp * QCHUNK_K;
    if (act && k0 < k_pad) {
      double x[QCHUNK_K], pr[QCHUNK_K];
#pragma unroll
      for (int r = 0; r < QCHUNK_K; ++r) {
        const int64_t k = k0 + r;
        const bool in = k < k_real;
        x[r] = in ? __ldcg(M + k * QW + lane) : 0.0;
        pr[r] = in ? __ldg(pre + k) : 0.0;
      }
#pragma unroll
      for (int r = 0; r < QCHUNK_K; ++r) x[r] *= pr[r];
      uint32_t w[4][QCHUNK_K / 4];
#pragma unroll
      for (int j = 0; j < QCHUNK_K / 4; ++j) {
        uint32_t u[4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
          u[i] = ok ? (((uint32_t)__double2int_rn(x[4 * j + i] * is) + 0x80808080u) ^ 0x80808080u) : 0u;
        const uint32_t A = __byte_perm(u[0], u[1], 0x5140), B = __byte_perm(u[0], u[1], 0x7362);
        const uint32_t C = __byte_perm(u[2], u[3], 0x5140), E = __byte_perm(u[2], u[3], 0x7362);
        w[3][j] = __byte_perm(A, C, 0x5410);
        w[2][j] = __byte_perm(A, C, 0x7632);
        w[1][j] = __byte_perm(B, E, 0x5410);
        w[0][j] = __byte_perm(B, E, 0x7632);
      }
      const int kb = warp >> 2, part = warp & 3;  // K-block of the round, 16-B quarter of its 64-B rows
#pragma unroll
      for (int a = 0; a < 4; ++a)
        stage[((kb * 4 + a) * QW + lane) * 5 + part] = make_uint4(w[a][0], w[a][1], w[a][2], w[a][3]);
    }
    __syncthreads();
    const int64_t left = (k_pad - g * 256) / 64;
    const int nkb = left < 4 ? (int)left : 4;  // K-blocks of this round
    uint4* dst = reinterpret_cast<uint4*>(planes + kb_offset(QW, 0, 0, g * 256));
    for (int i = threadIdx.x; i < nkb * 4 * QW * 4; i += blockDim.x) dst[i] = stage[(i >> 2) * 5 + (i & 3)];
    __syncthreads();
  }
}

// (Measured and dropped: an L2 evict-first policy on the Phi plane boxes kept
// the PCG blocks in L2 -- streaming phases C / F 3 us faster -- but cost the
// contractions ~100 us each: a 128-B line is read as two 64-B swizzled boxes
// one k-step apart, and evict-first drops it in between.)

// one split-K contraction phase, warp-specialised exactly like contract_kernel
// (MODE_FWD: A K-major), with the ring / TMEM pipeline counters carried across
// phases.  out[s][row][q] = sum_k A[row][k] B[k][q] * row_scale[row] * s_ops[q].
// items are (row block, split): w -> mb = w % n_mblocks, s = w / n_mblocks
template <int QW, int NPA>
__device__ __forceinline__ void contract_phase(const CUtensorMap* map_a, const CUtensorMap* map_b, int n_mblocks,
                                               int nsplit, int kps, int k_total, int64_t rows_real,
                                               const double* __restrict__ row_scale, const double* s_ops,
                                               double* __restrict__ out, int64_t out_rows, unsigned char* sm,
                                               uint64_t* full, uint64_t* empty, uint64_t* tfull, uint64_t* tempty,
                                               uint32_t tmem, int& stage, uint32_t& phase, int& it) {
  const int n_items = n_mblocks * nsplit;
  using C = Cfg<QW, NPA>;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    if (lane == 0) {
      fence_proxy_async();  // operand planes were written by generic stores before the barrier
      for (int w = blockIdx.x; w < n_items; w += gridDim.x) {
        const int mb = w % n_mblocks, s = w / n_mblocks;
        const int k0 = s * kps, k1 = min(k0 + kps, k_total);
        for (int k = k0; k < k1; k += KT) {
          mbar_wait(&empty[stage], phase ^ 1);
          unsigned char* sa = sm + stage * C::STAGE;
          mbar_expect_tx(&full[stage], C::STAGE);
          tma_load_3d(sa, map_a, &full[stage], k, mb * BM, 0);
          tma_load_4d(sa + C::A_ST, map_b, &full[stage], 0, 0, 0, k >> 6);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc0 = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BM >> 4) << 24);
      for (int w = blockIdx.x; w < n_items; w += gridDim.x, ++it) {
        const int s = w / n_mblocks;
        const int k0 = s * kps, k1 = min(k0 + kps, k_total);
        const int buf = it & 1;
        mbar_wait(&tempty[buf], ((it >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t tset = tmem + buf * C::SET_COLS;
        for (int k = k0; k < k1; k += KT) {
          mbar_wait(&full[stage], phase);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t sa = smem_u32(sm + stage * C::STAGE);
          issue_stage<QW, false, NPA>(sa, sa + C::A_ST, tset, idesc0);
          mma_commit(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit(&tfull[buf]);
      }
    }
  } else if (warp < 2 + EPI_WARPS) {
    const int quarter = warp & 3, half = (warp - 2) >> 2;
    const int row_in_tile = quarter * 32 + lane;
    for (int w = blockIdx.x; w < n_items; w += gridDim.x, ++it) {
      const int mb = w % n_mblocks, s = w / n_mblocks;
      const int buf = it & 1;
      const int64_t row = (int64_t)mb * BM + row_in_tile;
      const double scale = row < rows_real ? __ldg(row_scale + row) * (65536.0 / (SCALE30 * SCALE30)) : 0.0;
      mbar_wait(&tfull[buf], (it >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      double* o = out + ((int64_t)s * out_rows + row) * QW;
      const uint32_t tl = tmem + buf * C::SET_COLS + ((uint32_t)(quarter * 32) << 16);
#pragma unroll
      for (int q0 = 0; q0 < QW; q0 += 16) {
        const int qb = q0 + half * 8;
        if (qb < QW) {
          uint32_t r[5][8];
#pragma unroll
          for (int sb = 0; sb < 5; ++sb)
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(r[sb][0]), "=r"(r[sb][1]), "=r"(r[sb][2]), "=r"(r[sb][3]), "=r"(r[sb][4]),
                           "=r"(r[sb][5]), "=r"(r[sb][6]), "=r"(r[sb][7])
                         : "r"(tl + sb * QW + qb));
          asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
          for (int sb = 0; sb < 5; ++sb)
            asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(tl + sb * QW +
                                                                                                        qb),
                         "r"(0));
          double v[8];
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            const long long lo = ((long long)(int32_t)r[1][t] << 24) + ((long long)(int32_t)r[2][t] << 16) +
                                 ((long long)(int32_t)r[3][t] << 8) + (long long)(int32_t)r[4][t];
            v[t] = fma((double)(int32_t)r[0][t], 4294967296.0, (double)lo) * (scale * s_ops[qb + t]);
          }
          st_v4(o + qb, v[0], v[1], v[2], v[3]);
          st_v4(o + qb + 4, v[4], v[5], v[6], v[7]);
        }
      }
      asm volatile("tcgen05.wait::st.sync.aligned;");
      asm volatile("tcgen05.fence::before_thread_sync;");
      mbar_arrive(&tempty[buf]);
    }
  }
}


// acc[uu] = sum_s part[s][j0 + uu rstep][q] for the UNR rows of a loop trip, in
// split order; the loads of up to PS_MAXS splits x UNR rows are all in flight
// before the first add
template <int UNR, int MAXS>
__device__ __forceinline__ void sum_splits(const double* __restrict__ part, int64_t n, int nsplit, int64_t j0,
                                           int64_t rstep, int64_t rows, int q, int qw, double (&acc)[UNR]) {
  double v[MAXS][UNR];
#pragma unroll
  for (int s = 0; s < MAXS; ++s)
#pragma unroll
    for (int uu = 0; uu < UNR; ++uu) {
      const int64_t j = j0 + uu * rstep;
      v[s][uu] = (s < nsplit && j < rows) ? __ldcg(part + (int64_t)s * n + j * qw + q) : 0.0;
    }
#pragma unroll
  for (int uu = 0; uu < UNR; ++uu) {
    double t = v[0][uu];
#pragma unroll
    for (int s = 1; s < MAXS; ++s)
      if (s < nsplit) t += v[s][uu];
    acc[uu] = t;
  }
  for (int s = MAXS; s < nsplit; ++s)
#pragma unroll
    for (int uu = 0; uu < UNR; ++uu) {
      const int64_t j = j0 + uu * rstep;
      if (j < rows) acc[uu] += __ldcg(part + (int64_t)s * n + j * qw + q);
    }
}

template <int QW, int NPA = 4>
__global__ void __launch_bounds__(PS_THREADS, 1)
    pcg_persistent(const __grid_constant__ CUtensorMap map_af, const __grid_constant__ CUtensorMap map_bf,
                   const __grid_constant__ CUtensorMap map_ab, const __grid_constant__ CUtensorMap map_bb,
                   const __grid_constant__ PcgPersistArgs a) {
  using C = Cfg<QW, NPA>;
  constexpr int RPB = PS_THREADS / QW;  // rows per loop trip of the streaming phases
  extern __shared__ unsigned char smem_raw[];
  unsigned char* sm = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  unsigned char* ctrl = sm + STAGES * C::STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(ctrl);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);
  double* sv = reinterpret_cast<double*>(ctrl + PS_CTRL);
  double* s_rho = sv;             // rho of P(u)
  double* s_pi = sv + 32;         // pi of step u
  double* s_gam = sv + 64;        // gamma_u
  double* s_gprev = sv + 96;      // gamma_{u-1} (paired X updates)
  double* s_ops_p = sv + 128;     // column scales of diag(c) P(u)
  double* s_ops_v = sv + 160;     // column scales of diag(r) V
  double* s_fold = sv + 192;      // folded partials (up to 2 x 32)
  // the stage ring doubles as the streaming phases' scratch (idle outside B / E)
  double* smr = reinterpret_cast<double*>(sm);                          // reductions: up to 2 x 4 x 512 doubles
  uint4* qstage = reinterpret_cast<uint4*>(sm + 65536);                 // quantiser staging (<= 40 KB)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, t = threadIdx.x;
  if (t == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 32 * EPI_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    tma_prefetch(&map_af);
    tma_prefetch(&map_bf);
    tma_prefetch(&map_ab);
    tma_prefetch(&map_bb);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t < 32) {
    s_rho[t] = t < QW ? a.rho1[t] : 0.0;
    s_gprev[t] = 0.0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_holder;
  if (warp >= 2 && warp < 6) tmem_zero_all(tmem, warp & 3);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");

  double b2 = 0.0;  // ||B||_F^2 in k_direction's column order
  for (int c = 0; c < QW; ++c) b2 += a.bn2[c];
  unsigned gen = *((volatile unsigned*)a.bar + 1);
  int stage = 0, it = 0;
  uint32_t phase = 0;
  const int q = t % QW;
  const bool colthr = t < RPB * QW;  // owns column q of rows r0 + k RPB gridDim (streaming phases)
  const VMap<QW> vm;                 // 4-column vector map of the streaming phases
  const int64_t r0 = (int64_t)blockIdx.x * RPB + t / QW;
  const int64_t rstep = (int64_t)gridDim.x * RPB;
  auto stamp = [&](int u, int ph) {
    if (a.times && blockIdx.x == 0 && t == 0 && u <= a.max_steps) a.times[(int64_t)u * PS_TIMES + ph] = gtimer();
  };

  int u = 1;
  for (;; ++u) {
    double* Pc = (u & 1) ? a.P0 : a.P1;  // P(u)
    double* Pn = (u & 1) ? a.P1 : a.P0;  // P(u - 1) in, P(u + 1) out
    // ---- A: quantise P(u); <P, alpha P> partials ------------------------------
    stamp(u, 0);
    if (t < QW) s_ops_p[t] = col_scale(__ldcg(a.colmax_p + t));
    __syncthreads();
    quantize_phase<QW>(Pc, a.D, a.Dp, a.colscale, s_ops_p, a.pq, qstage);
    if (u == 1) {  // <P(1), alpha P(1)> (later steps get it from H)
      double psq = 0.0;
      if (colthr)
        for (int64_t j = r0; j < a.Dp; j += rstep) {
          const double pv = __ldcg(Pc + j * QW + q);
          psq += __ldg(a.alpha + j) * (pv * pv);
        }
      cta_col_sums<QW>(smr, 1, &psq, a.red, 0);
    }
    if (blockIdx.x == 0 && t < 32) a.colmax_v[t] = 0ull;  // last read in D of the previous step
    fence_proxy_async();
    stamp(u, 8);
    grid_sync(a.bar, gen);

    // ---- B: Phi P -> vpart ---------------------------------------------------
    stamp(u, 1);
    contract_phase<QW, NPA>(&map_af, &map_bf, a.f_mblocks, a.f_nsplit, a.f_kps, (int)a.Dp, a.N, a.rowscale, s_ops_p,
                       a.vpart, a.Np, sm, full, empty, tfull, tempty, tmem, stage, phase, it);
    stamp(u, 9);
    grid_sync(a.bar, gen);

    // ---- C: V = sum of the splits; max |r V|; ||V||^2 --------------------------
    stamp(u, 2);
    if (blockIdx.x == 0 && t < 32) a.colmax_p[t] = 0ull;  // read in A, refilled in H
    {
      double vmax[4] = {0.0, 0.0, 0.0, 0.0}, vsq[1][4] = {{0.0, 0.0, 0.0, 0.0}};
      if (vm.on) {
        const int64_t n = a.Np * QW;
        for (int64_t j = vm.r0; j < a.Np; j += vm.rstep) {
          const int64_t e = j * QW + vm.c0;
          const double rs = __ldg(a.rowscale + j);
          double acc[4] = {0.0, 0.0, 0.0, 0.0};
          for (int s0 = 0; s0 < a.f_nsplit; s0 += 4) {  // four split partials in flight, added in split order
            double v[4][4];
#pragma unroll
            for (int s = 0; s < 4; ++s)
              if (s0 + s < a.f_nsplit) ld4(a.vpart + (int64_t)(s0 + s) * n + e, v[s]);
#pragma unroll
            for (int s = 0; s < 4; ++s)
              if (s0 + s < a.f_nsplit)
#pragma unroll
                for (int c = 0; c < 4; ++c) acc[c] = s0 + s == 0 ? v[s][c] : acc[c] + v[s][c];
          }
          st4(a.V + e, acc);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            vsq[0][c] += acc[c] * acc[c];
            vmax[c] = nanmax(vmax[c], fabs(acc[c] * rs));
          }
        }
      }
      cta_col_sums4<QW, 1>(smr, vsq, a.red, 1);
      cta_col_max4<QW>(smr, vmax, a.colmax_v);
    }
    stamp(u, 10);
    grid_sync(a.bar, gen);

    // ---- D: quantise V; pi, gamma -------------------------------------------
    stamp(u, 3);
    if (t < QW) s_ops_v[t] = col_scale(__ldcg(a.colmax_v + t));
    __syncthreads();
    quantize_phase<QW>(a.V, a.Np, a.Np, a.rowscale, s_ops_v, a.vq, qstage);
    fold_all<QW>(a.red, 0, 2, smr, s_fold);  // <P, alpha P> | ||V||^2
    if (t < QW) {
      const double pi = a.beta * s_fold[QW + t] + s_fold[t];
      s_pi[t] = pi;
      s_gam[t] = safe_ratio(s_rho[t], pi);
      if (blockIdx.x == 0 && t < a.q_real && pi == 0.0) a.frozen[t] = 1;
    }
    fence_proxy_async();
    stamp(u, 11);
    grid_sync(a.bar, gen);

    // ---- E: Phi^T V -> ppart ---------------------------------------------------
    stamp(u, 4);
    contract_phase<QW, NPA>(&map_ab, &map_bb, a.b_mblocks, a.b_nsplit, a.b_kps, (int)a.Np, a.D, a.colscale, s_ops_v,
                       a.ppart, a.Dp, sm, full, empty, tfull, tempty, tmem, stage, phase, it);
    stamp(u, 12);
    grid_sync(a.bar, gen);

    // ---- F: R -= gamma (beta Phi^T V + alpha P); rho_new, ||R||^2 ----------------
    stamp(u, 5);
    {
      double sums[2][4] = {{0.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.0, 0.0}};  // rho_new | ||R||^2
      if (vm.on) {
        double gm[4], live[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          gm[c] = s_gam[vm.c0 + c];
          live[c] = vm.c0 + c < a.q_real ? 1.0 : 0.0;
        }
        const int64_t n = a.Dp * QW;
        for (int64_t j = vm.r0; j < a.Dp; j += vm.rstep) {
          const int64_t e = j * QW + vm.c0;
          double v[4][4], p[4], r[4];
#pragma unroll
          for (int s = 0; s < 4; ++s)
            if (s < a.b_nsplit) ld4(a.ppart + (int64_t)s * n + e, v[s]);
          ld4(Pc + e, p);
          ld4(a.R + e, r);
          const double al = __ldg(a.alpha + j), mv = __ldg(a.minv + j);
          double acc[4] = {v[0][0], v[0][1], v[0][2], v[0][3]};
#pragma unroll
          for (int s = 1; s < 4; ++s)
            if (s < a.b_nsplit)
#pragma unroll
              for (int c = 0; c < 4; ++c) acc[c] += v[s][c];
          for (int s = 4; s < a.b_nsplit; ++s) {
            double w[4];
            ld4(a.ppart + (int64_t)s * n + e, w);
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[c] += w[c];
          }
          double rn[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const double psi = a.beta * acc[c] + al * p[c];
            rn[c] = r[c] - psi * gm[c];
            sums[1][c] += rn[c] * rn[c];
            sums[0][c] += live[c] * (rn[c] * (rn[c] * mv));
          }
          st4(a.R + e, rn);
        }
      }
      cta_col_sums4<QW, 2>(smr, sums, a.red, 2);
    }
    stamp(u, 13);
    grid_sync(a.bar, gen);

    // ---- H: stopping test; X updates; P(u+1) ---------------------------------
    stamp(u, 6);
    fold_all<QW>(a.red, 2, 2, smr, s_fold);  // rho_new | ||R||^2
    double r2 = 0.0;
    for (int c = 0; c < QW; ++c) r2 += s_fold[QW + c];
    const double delta = sqrt(r2) / sqrt(b2);
    const bool finite = isfinite(delta);
    const bool conv = finite && delta <= a.tol;
    const bool stop = !finite || conv || u >= a.max_steps;
    if (blockIdx.x == 0 && t == 0) {
      volatile Status* vs = a.st;
      vs->steps = u;
      vs->delta = delta;
      vs->converged = conv ? 1 : 0;
      vs->diverged = finite ? 0 : 1;
      vs->bnorm = sqrt(b2);
      __threadfence();
      if (stop) vs->done = 1;
    }
    const bool pair = (u & 1) == 0;  // odd steps defer X += gamma P; even steps apply both
    if (stop) {
      if (vm.on) {
        double gm[4], gp[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          gm[c] = s_gam[vm.c0 + c];
          gp[c] = pair ? s_gprev[vm.c0 + c] : 0.0;
        }
        for (int64_t j = vm.r0; j < a.Dp; j += vm.rstep) {
          const int64_t e = j * QW + vm.c0;
          double x[4], pc[4], pp[4];
          ld4(a.X + e, x);
          ld4(Pc + e, pc);
          if (pair) ld4(Pn + e, pp);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            if (pair) x[c] = x[c] + pp[c] * gp[c];
            x[c] = x[c] + pc[c] * gm[c];
          }
          st4(a.X + e, x);
        }
      }
      break;
    }
    {
      double pmax[4] = {0.0, 0.0, 0.0, 0.0}, psq[1][4] = {{0.0, 0.0, 0.0, 0.0}};
      if (vm.on) {
        double eta[4], gm[4], gp[4], live[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          eta[c] = safe_ratio(s_fold[vm.c0 + c], s_rho[vm.c0 + c]);
          gm[c] = pair ? s_gam[vm.c0 + c] : 0.0;
          gp[c] = pair ? s_gprev[vm.c0 + c] : 0.0;
          live[c] = vm.c0 + c < a.q_real ? 1.0 : 0.0;
        }
        for (int64_t j0 = vm.r0; j0 < a.Dp; j0 += PS_VU * vm.rstep) {
          double r[PS_VU][4], p[PS_VU][4], x[PS_VU][4], pp[PS_VU][4], mv[PS_VU], al[PS_VU], cs[PS_VU];
#pragma unroll
          for (int uu = 0; uu < PS_VU; ++uu) {
            const int64_t j = j0 + uu * vm.rstep;
            if (j < a.Dp) {
              const int64_t e = j * QW + vm.c0;
              ld4(a.R + e, r[uu]);
              ld4(Pc + e, p[uu]);
              if (pair) {
                ld4(a.X + e, x[uu]);
                ld4(Pn + e, pp[uu]);
              }
              mv[uu] = __ldg(a.minv + j);
              al[uu] = __ldg(a.alpha + j);
              cs[uu] = __ldg(a.colscale + j);
            }
          }
#pragma unroll
          for (int uu = 0; uu < PS_VU; ++uu) {
            const int64_t j = j0 + uu * vm.rstep;
            if (j < a.Dp) {
              const int64_t e = j * QW + vm.c0;
              if (pair) {
                double xn[4];
#pragma unroll
                for (int c = 0; c < 4; ++c) xn[c] = (x[uu][c] + pp[uu][c] * gp[c]) + p[uu][c] * gm[c];
                st4(a.X + e, xn);
              }
              double pn[4];
#pragma unroll
              for (int c = 0; c < 4; ++c) {
                const double w = live[c] * (r[uu][c] * mv[uu]);
                pn[c] = p[uu][c] * eta[c] + (a.printed ? r[uu][c] : w);
                psq[0][c] += al[uu] * (pn[c] * pn[c]);
                pmax[c] = nanmax(pmax[c], fabs(pn[c] * cs[uu]));
              }
              st4(Pn + e, pn);
            }
          }
        }
      }
      cta_col_max4<QW>(smr, pmax, a.colmax_p);
      cta_col_sums4<QW, 1>(smr, psq, a.red, 0);  // <P(u+1), alpha P(u+1)> for the next pi
      __syncthreads();
      if (t < QW) {
        s_rho[t] = s_fold[t];
        s_gprev[t] = s_gam[t];
      }
    }
    stamp(u, 14);
    grid_sync(a.bar, gen);
  }
  if (a.times && blockIdx.x == 0 && t == 0) a.times[(int64_t)u * PS_TIMES + 7] = gtimer();
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

}  // namespace oz
}  // namespace cofem
