// dct.cuh -- 2-D partial-DCT dictionaries (BASELINE config 4) on the int8
// tensor-core contraction.
//
// Phi = M * DCT2 (orthonormal 2-D DCT-II of an n x n image, then the rows of
// the coefficient grid selected by the mask M), so Phi^T Phi P = DCT2^T (M .*
// DCT2 P) and one PCG apply is four dense stages against the fixed n x n DCT
// matrix C (Y = C X C^T, Z = C^T U C), each an ozaki contraction over the
// stacked images of all Q columns.  The digit planes of C are read K-major for
// the C stages and MN-major (C^T) for the adjoint stages -- one copy.
//
// Layouts (ldq = padded column count, Q images side by side):
//   PCG block  P[(i n + j) ldq + q]                 (pixel-major, as every block)
//   stage buffers B[r][(h ldq + q)], r, h < n        (n x n ldq row-major)
//   operand planes K-blocked [n / 64][4][n ldq][64] (oz::kb_offset): column c = h ldq + q, K index t
// Operand element (t, c = h ldq + lo) lives at src[t st + h sh + lo].
#pragma once
#include "ozaki.cuh"

namespace cofem {
namespace dct {

// digit planes of the columns.  One block owns a strip of 64 columns: pass 1
// folds the column maxima (4 K-rows x 64 columns per sweep, coalesced along
// the columns), pass 2 re-reads the strip (L2-hot) in 32 x 64 smem tiles and
// stores one 32-bit word (4 K rows) per digit plane, coalesced along K.
constexpr int TT = 32, TC = 64;
__global__ void __launch_bounds__(256)
    k_cq_quantize(int K, int NC, int ldq, int64_t st, int64_t sh, const double* __restrict__ src,
                  const double* __restrict__ pre, double* __restrict__ scale_out, int8_t* __restrict__ planes,
                  const Status* __restrict__ stt) {
  if (stt && stt->done) return;
  __shared__ double tile[TT][TC + 1];
  __shared__ double inv_s[TC];
  __shared__ unsigned long long red[4][TC];
  const int ntc = NC / TC;
  for (int strip = blockIdx.x; strip < ntc; strip += gridDim.x) {
    const int c0 = strip * TC;
    {
      const int cc = threadIdx.x % TC, tt = threadIdx.x / TC;  // 4 x 64
      const int c = c0 + cc;
      const int64_t base = (int64_t)(c / ldq) * sh + (c % ldq);
      double m = 0.0;
      for (int t = tt; t < K; t += 4) {
        const double v = fabs(src[base + (int64_t)t * st] * pre[t]);
        m = (v > m || v != v) ? v : m;
      }
      __syncthreads();
      red[tt][cc] = (unsigned long long)__double_as_longlong(m);
      __syncthreads();
      if (threadIdx.x < TC) {
        unsigned long long mm = red[0][threadIdx.x];
        for (int r = 1; r < 4; ++r) mm = red[r][threadIdx.x] > mm ? red[r][threadIdx.x] : mm;
        const double sc = oz::col_scale(mm);
        inv_s[threadIdx.x] = oz::SCALE30 / sc;
        scale_out[c0 + threadIdx.x] = sc;
      }
    }
    for (int t0 = 0; t0 < K; t0 += TT) {
      __syncthreads();
      for (int e = threadIdx.x; e < TT * TC; e += blockDim.x) {
        const int r = e / TC, cc = e % TC;
        const int c = c0 + cc, t = t0 + r;
        tile[r][cc] = src[(int64_t)t * st + (int64_t)(c / ldq) * sh + (c % ldq)] * pre[t];
      }
      __syncthreads();
      for (int w = threadIdx.x; w < TC * (TT / 4); w += blockDim.x) {
        const int quad = w % (TT / 4), cc = w / (TT / 4);
        const double is = inv_s[cc];
        uint32_t word[4] = {0u, 0u, 0u, 0u};
        if (is == is) {
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            int8_t d[4];
            oz::digits4(tile[quad * 4 + r][cc] * is, d);
#pragma unroll
            for (int a = 0; a < 4; ++a) word[a] |= (uint32_t)(uint8_t)d[a] << (8 * r);
          }
        }
#pragma unroll
        for (int a = 0; a < 4; ++a)
          *reinterpret_cast<uint32_t*>(planes + oz::kb_offset(NC, a, c0 + cc, t0 + quad * 4)) = word[a];
      }
    }
  }
}

// U = M .* Y on the coefficient grid; the stage buffer holds Y^T as
// [l][(k ldq + q)], the mask is the n x n 0/1 grid [k][l]
__global__ void k_apply_mask(int n, int ldq, double* __restrict__ buf, const uint8_t* __restrict__ grid,
                             const Status* __restrict__ stt) {
  if (stt && stt->done) return;
  const int64_t total = (int64_t)n * n * ldq;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = e / ((int64_t)n * ldq);
    const int k = (int)((e / ldq) % n);
    if (!grid[(int64_t)k * n + l]) buf[e] = 0.0;
  }
}

// final transpose: out[(i n + j) ldq + q] = buf[j][(i ldq + q)], tiles of
// 8 j x 16 i x ldq staged through smem (contiguous along (i, q) on load and
// along (j, q) on store)
constexpr int FJ = 8, FI = 16;
__global__ void k_finish(int n, int ldq, const double* __restrict__ buf, double* __restrict__ out,
                         const Status* __restrict__ stt) {
  if (stt && stt->done) return;
  extern __shared__ double ftile[];  // [FJ][FI * ldq]
  const int nti = n / FI, ntj = n / FJ;
  const int row = FI * ldq;
  for (int tb = blockIdx.x; tb < nti * ntj; tb += gridDim.x) {
    const int ib = tb % nti, jb = tb / nti;
    __syncthreads();
    for (int e = threadIdx.x; e < FJ * row; e += blockDim.x) {
      const int jj = e / row, r = e % row;  // r = ii * ldq + q
      ftile[jj * row + r] = buf[((int64_t)(jb * FJ + jj) * n + ib * FI) * ldq + r];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < FJ * row; e += blockDim.x) {
      const int ii = e / (FJ * ldq), r = e % (FJ * ldq);  // r = jj * ldq + q
      const int jj = r / ldq, q = r % ldq;
      out[((int64_t)(ib * FI + ii) * n + jb * FJ) * ldq + r] = ftile[jj * row + ii * ldq + q];
    }
  }
}

// measurement gather / scatter for the explicit apply / adjoint utilities
__global__ void k_gather(int64_t nm, int n, int ldq, const int64_t* __restrict__ mask, const double* __restrict__ buf,
                         double* __restrict__ v) {
  const int64_t total = nm * ldq;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = e / ldq;
    const int q = (int)(e % ldq);
    const int64_t kl = mask[m];
    const int64_t k = kl / n, l = kl % n;
    v[e] = buf[(l * n + k) * ldq + q];  // buf = Y^T [l][(k ldq + q)]
  }
}

__global__ void k_scatter(int64_t nm, int n, int ldq, const int64_t* __restrict__ mask, const double* __restrict__ v,
                          double* __restrict__ buf) {
  const int64_t total = nm * ldq;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = e / ldq;
    const int q = (int)(e % ldq);
    const int64_t kl = mask[m];
    const int64_t k = kl / n, l = kl % n;
    buf[(l * n + k) * ldq + q] = v[e];
  }
}

}  // namespace dct
}  // namespace cofem
