// kernels.cuh -- sm_100a kernels of the CoFEM hot path (CUDA-core path).
//
// Layouts (HBM):
//   Phi   : Np x Dp row-major, zero padded (Np % 128 == 0, Dp % 128 == 0);
//           float32 (PhiT = float), or float64 (PhiT = double) when a float64
//           dictionary is set in the fp64 mode (exact entries, no rounding)
//   blocks: Dp x ldq of T (float or double) row-major -- coordinate j's Q
//           right-hand-side entries contiguous (the reference's (D, Q) C order)
//   V     : Np x ldq of T (Phi P)
//
// The two skinny contractions stream Phi once each per PCG step:
//   fwd : Vpart[s] = Phi[:, k-split s] * P[k-split s, :]        (split-K over D)
//   bwd : Psipart[s] = Phi[n-split s, :]^T * V[n-split s, :]    (split-K over N)
// Tiles are staged global->smem with cp.async (16 B, L2-only .cg) in a
// multi-stage pipeline; each thread keeps an R x QP (fwd) or C x QP (bwd)
// accumulator block in registers and reads the small operand (P or V rows)
// as warp-wide smem broadcasts.  Split partials are summed in a fixed order
// by a separate pass, so every result is bitwise reproducible.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace cofem {

struct Status {
  int done;        // 1 once converged / diverged / max steps reached
  int steps;       // PCG steps taken
  int converged;
  int diverged;
  double delta;    // ||R||_F / ||B||_F after the last step
  double bnorm;    // ||B||_F
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// four consecutive dictionary entries from shared memory (16 B or 2 x 16 B)
__device__ __forceinline__ void load4(const float* p, float f[4]) {
  const float4 v = *reinterpret_cast<const float4*>(p);
  f[0] = v.x; f[1] = v.y; f[2] = v.z; f[3] = v.w;
}
__device__ __forceinline__ void load4(const double* p, double f[4]) {
  const double2 a = *reinterpret_cast<const double2*>(p), b = *reinterpret_cast<const double2*>(p + 2);
  f[0] = a.x; f[1] = a.y; f[2] = b.x; f[3] = b.y;
}
template <int CC>
__device__ __forceinline__ void loadc(const float* p, float f[CC]) {
  if constexpr (CC == 4) {
    load4(p, f);
  } else {
    const float2 v = *reinterpret_cast<const float2*>(p);
    f[0] = v.x; f[1] = v.y;
  }
}
template <int CC>
__device__ __forceinline__ void loadc(const double* p, double f[CC]) {
  if constexpr (CC == 4) {
    load4(p, f);
  } else {
    const double2 v = *reinterpret_cast<const double2*>(p);
    f[0] = v.x; f[1] = v.y;
  }
}

template <typename T>
struct Vec4;  // 16-byte vector of T
template <>
struct Vec4<float> {
  static constexpr int W = 4;
};
template <>
struct Vec4<double> {
  static constexpr int W = 2;
};

// ---------------------------------------------------------------------------
// fwd: Vpart[blockIdx.y] (BM x QP) = Phi[m0:m0+BM, k-range] * P[k-range, qoff:qoff+QP]
//
// Thread (warp w = wk*WM + wm, lane l) owns rows m0 + wm*32R + r*32 + l
// (r < R) and the column sub-slice wk of every BK-wide tile; the WK partial
// sums are folded through smem at the end.
template <typename T, int QP, int R, int WM, int WK, int BK, int STAGES, typename PhiT = float>
struct FwdCfg {
  static constexpr int BM = 32 * R * WM;
  static constexpr int NT = 32 * WM * WK;
  static constexpr int SROW = BK + 16 / (int)sizeof(PhiT);  // +16 B: 16-B row reads are conflict-free
  static constexpr int PHI_STAGE = BM * SROW;                // PhiT entries
  static constexpr int P_STAGE = BK * QP;                    // T
  static constexpr size_t STAGE_BYTES = PHI_STAGE * sizeof(PhiT) + P_STAGE * sizeof(T);
  static constexpr size_t RED_BYTES = (size_t)(WK - 1) * BM * QP * sizeof(T);
  static constexpr size_t SMEM = (STAGES * STAGE_BYTES > RED_BYTES) ? STAGES * STAGE_BYTES : RED_BYTES;
  static_assert(BK % (4 * WK) == 0, "each k group needs whole float4 columns");
  static_assert((QP * sizeof(T)) % 16 == 0, "QP row must be a multiple of 16 B");
};

template <typename T, int QP, int R, int WM, int WK, int BK, int STAGES, typename PhiT = float>
__global__ void __launch_bounds__(32 * WM * WK)
    fwd_kernel(const PhiT* __restrict__ phi, int64_t ldphi, const T* __restrict__ P, int ldq, int qoff,
               int k_per_split, int64_t kmax, T* __restrict__ vpart, int64_t np, const Status* __restrict__ st) {
  using C = FwdCfg<T, QP, R, WM, WK, BK, STAGES, PhiT>;
  if (st && st->done) return;
  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp % WM, wk = warp / WM;
  const int64_t m0 = (int64_t)blockIdx.x * C::BM;
  const int64_t k0 = (int64_t)blockIdx.y * k_per_split;
  int64_t k1 = k0 + k_per_split;
  if (k1 > kmax) k1 = kmax;
  const int ntiles = (int)((k1 - k0) / BK);

  constexpr int EPC = 16 / (int)sizeof(PhiT);  // dictionary entries per 16-B chunk
  auto stage_phi = [&](int s) { return reinterpret_cast<PhiT*>(smem + s * C::STAGE_BYTES); };
  auto stage_p = [&](int s) {
    return reinterpret_cast<T*>(smem + s * C::STAGE_BYTES + C::PHI_STAGE * sizeof(PhiT));
  };

  auto load_tile = [&](int s, int t) {
    const int64_t kt = k0 + (int64_t)t * BK;
    PhiT* sphi = stage_phi(s);
    constexpr int CPR = BK / EPC;  // 16-B chunks per tile row
    for (int c = tid; c < C::BM * CPR; c += C::NT) {
      const int row = c / CPR, ch = c % CPR;
      cp_async16(sphi + row * C::SROW + ch * EPC, phi + (m0 + row) * ldphi + kt + ch * EPC);
    }
    T* sp = stage_p(s);
    constexpr int PCH = QP * sizeof(T) / 16;  // chunks per P row
    for (int c = tid; c < BK * PCH; c += C::NT) {
      const int row = c / PCH, ch = c % PCH;
      cp_async16(reinterpret_cast<unsigned char*>(sp + row * QP) + ch * 16,
                 reinterpret_cast<const unsigned char*>(P + (kt + row) * ldq + qoff) + ch * 16);
    }
  };

  T acc[R][QP];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int q = 0; q < QP; ++q) acc[r][q] = T(0);

#pragma unroll
  for (int t = 0; t < STAGES - 1; ++t) {
    if (t < ntiles) load_tile(t, t);
    cp_async_commit();
  }
  constexpr int KW = BK / WK;  // columns of a tile owned by one k group
  for (int t = 0; t < ntiles; ++t) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int tn = t + STAGES - 1;
      if (tn < ntiles) load_tile(tn % STAGES, tn);
      cp_async_commit();
    }
    const PhiT* sphi = stage_phi(t % STAGES);
    const T* sp = stage_p(t % STAGES);
#pragma unroll
    for (int jj = wk * KW; jj < (wk + 1) * KW; jj += 4) {
      PhiT f[R][4];
#pragma unroll
      for (int r = 0; r < R; ++r) load4(sphi + (wm * 32 * R + r * 32 + lane) * C::SROW + jj, f[r]);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const T* prow = sp + (jj + kk) * QP;
#pragma unroll
        for (int q = 0; q < QP; ++q) {
          const T pv = prow[q];
#pragma unroll
          for (int r = 0; r < R; ++r) acc[r][q] = fma(T(f[r][kk]), pv, acc[r][q]);
        }
      }
    }
  }
  cp_async_wait<0>();
  __syncthreads();
  if constexpr (WK > 1) {
    T* red = reinterpret_cast<T*>(smem);
    if (wk > 0) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int row = wm * 32 * R + r * 32 + lane;
#pragma unroll
        for (int q = 0; q < QP; ++q) red[((wk - 1) * C::BM + row) * QP + q] = acc[r][q];
      }
    }
    __syncthreads();
    if (wk == 0) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int row = wm * 32 * R + r * 32 + lane;
        for (int g = 0; g < WK - 1; ++g)
#pragma unroll
          for (int q = 0; q < QP; ++q) acc[r][q] += red[(g * C::BM + row) * QP + q];
      }
    }
  }
  if (wk == 0) {
    T* out = vpart + (int64_t)blockIdx.y * np * QP;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int64_t row = m0 + wm * 32 * R + r * 32 + lane;
#pragma unroll
      for (int q = 0; q < QP; q += Vec4<T>::W) {
        if constexpr (sizeof(T) == 4) {
          *reinterpret_cast<float4*>(out + row * QP + q) =
              make_float4(acc[r][q], acc[r][q + 1], acc[r][q + 2], acc[r][q + 3]);
        } else {
          *reinterpret_cast<double2*>(out + row * QP + q) = make_double2(acc[r][q], acc[r][q + 1]);
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// bwd: Psipart[blockIdx.y] (BN x QP) = Phi[n-range, n0:n0+BN]^T * V[n-range, qoff:qoff+QP]
//
// Warp w = wk*WN + wn, lane l owns columns n0 + wn*32C + l*C + c (c < C) and
// the tile rows i with i % WK == wk.
template <typename T, int QP, int CC, int WN, int WK, int BK, int STAGES, typename PhiT = float>
struct BwdCfg {
  static constexpr int BN = 32 * CC * WN;
  static constexpr int NT = 32 * WN * WK;
  static constexpr int PHI_STAGE = BK * BN;  // PhiT entries
  static constexpr int V_STAGE = BK * QP;    // T
  static constexpr size_t STAGE_BYTES = PHI_STAGE * sizeof(PhiT) + V_STAGE * sizeof(T);
  static constexpr size_t RED_BYTES = (size_t)(WK - 1) * BN * QP * sizeof(T);
  static constexpr size_t SMEM = (STAGES * STAGE_BYTES > RED_BYTES) ? STAGES * STAGE_BYTES : RED_BYTES;
  static_assert(CC == 4 || CC == 2, "columns per thread");
  static_assert(BK % WK == 0, "row interleave");
};

template <typename T, int QP, int CC, int WN, int WK, int BK, int STAGES, typename PhiT = float>
__global__ void __launch_bounds__(32 * WN * WK)
    bwd_kernel(const PhiT* __restrict__ phi, int64_t ldphi, const T* __restrict__ V, int ldv, int qoff,
               int n_per_split, int64_t nmax, T* __restrict__ ppart, int64_t dp, const Status* __restrict__ st) {
  using C = BwdCfg<T, QP, CC, WN, WK, BK, STAGES, PhiT>;
  if (st && st->done) return;
  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wn = warp % WN, wk = warp / WN;
  const int64_t c0 = (int64_t)blockIdx.x * C::BN;
  const int64_t r0 = (int64_t)blockIdx.y * n_per_split;
  int64_t r1 = r0 + n_per_split;
  if (r1 > nmax) r1 = nmax;
  const int ntiles = (int)((r1 - r0) / BK);

  constexpr int EPC = 16 / (int)sizeof(PhiT);  // dictionary entries per 16-B chunk
  auto stage_phi = [&](int s) { return reinterpret_cast<PhiT*>(smem + s * C::STAGE_BYTES); };
  auto stage_v = [&](int s) {
    return reinterpret_cast<T*>(smem + s * C::STAGE_BYTES + C::PHI_STAGE * sizeof(PhiT));
  };

  auto load_tile = [&](int s, int t) {
    const int64_t rt = r0 + (int64_t)t * BK;
    PhiT* sphi = stage_phi(s);
    constexpr int CPR = C::BN / EPC;
    for (int c = tid; c < BK * CPR; c += C::NT) {
      const int row = c / CPR, ch = c % CPR;
      cp_async16(sphi + row * C::BN + ch * EPC, phi + (rt + row) * ldphi + c0 + ch * EPC);
    }
    T* sv = stage_v(s);
    constexpr int VCH = QP * sizeof(T) / 16;
    for (int c = tid; c < BK * VCH; c += C::NT) {
      const int row = c / VCH, ch = c % VCH;
      cp_async16(reinterpret_cast<unsigned char*>(sv + row * QP) + ch * 16,
                 reinterpret_cast<const unsigned char*>(V + (rt + row) * ldv + qoff) + ch * 16);
    }
  };

  T acc[CC][QP];
#pragma unroll
  for (int c = 0; c < CC; ++c)
#pragma unroll
    for (int q = 0; q < QP; ++q) acc[c][q] = T(0);

#pragma unroll
  for (int t = 0; t < STAGES - 1; ++t) {
    if (t < ntiles) load_tile(t, t);
    cp_async_commit();
  }
  for (int t = 0; t < ntiles; ++t) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int tn = t + STAGES - 1;
      if (tn < ntiles) load_tile(tn % STAGES, tn);
      cp_async_commit();
    }
    const PhiT* sphi = stage_phi(t % STAGES);
    const T* sv = stage_v(t % STAGES);
#pragma unroll 4
    for (int i = wk; i < BK; i += WK) {
      PhiT f[CC];
      loadc<CC>(sphi + i * C::BN + wn * 32 * CC + lane * CC, f);
      const T* vrow = sv + i * QP;
#pragma unroll
      for (int q = 0; q < QP; ++q) {
        const T vv = vrow[q];
#pragma unroll
        for (int c = 0; c < CC; ++c) acc[c][q] = fma(T(f[c]), vv, acc[c][q]);
      }
    }
  }
  cp_async_wait<0>();
  __syncthreads();
  if constexpr (WK > 1) {
    T* red = reinterpret_cast<T*>(smem);
    if (wk > 0) {
#pragma unroll
      for (int c = 0; c < CC; ++c) {
        const int col = wn * 32 * CC + lane * CC + c;
#pragma unroll
        for (int q = 0; q < QP; ++q) red[((wk - 1) * C::BN + col) * QP + q] = acc[c][q];
      }
    }
    __syncthreads();
    if (wk == 0) {
#pragma unroll
      for (int c = 0; c < CC; ++c) {
        const int col = wn * 32 * CC + lane * CC + c;
        for (int g = 0; g < WK - 1; ++g)
#pragma unroll
          for (int q = 0; q < QP; ++q) acc[c][q] += red[(g * C::BN + col) * QP + q];
      }
    }
  }
  if (wk == 0) {
    T* out = ppart + (int64_t)blockIdx.y * dp * QP;
#pragma unroll
    for (int c = 0; c < CC; ++c) {
      const int64_t col = c0 + wn * 32 * CC + lane * CC + c;
#pragma unroll
      for (int q = 0; q < QP; q += Vec4<T>::W) {
        if constexpr (sizeof(T) == 4) {
          *reinterpret_cast<float4*>(out + col * QP + q) =
              make_float4(acc[c][q], acc[c][q + 1], acc[c][q + 2], acc[c][q + 3]);
        } else {
          *reinterpret_cast<double2*>(out + col * QP + q) = make_double2(acc[c][q], acc[c][q + 1]);
        }
      }
    }
  }
}

}  // namespace cofem
