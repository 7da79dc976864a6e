// dct1.cuh -- the reference's SubsampledDctOperator (operators.py:132-179) in
// O(D log D): Phi = M Omega^{-1}, the rows `mask` of the orthonormal inverse
// DCT-II (= DCT-III) of length D, any D.
//
// Makhoul's reduction for every column, two real columns per complex
// length-D FFT (the FFTs themselves are cuFFT double complex, batched over
// the ldq / 2 column pairs of a PCG block; this operator is not on the
// BASELINE hot path).  With sigma(m) = 2m (m < ceil(D/2)), 2(D-1-m)+1 else --
// v = x o sigma is the even/odd reordering:
//   DCT-II:  X_k = c_k Re(e^{-i pi k / 2D} FFT(v)_k)
//   DCT-III: v = IFFT_unnormalised(W), W_k = e^{i pi k / 2D} (X_k / c_k - i X_{D-k} / c_{D-k}) / D
// and for Phi^T Phi the two reorderings cancel: mask .* x in v order is
// v .* (mask o sigma), so Phi^T Phi P = post(FFT(mask_v .* IFFT(pre(P)))).
// The packed pair (a, b) rides as a + i b; V_a / V_b are separated from
// Z_k and Z_{D-k} in the post pass.  Layouts: real blocks [rows][ldq], the
// complex work buffer [D][ldq / 2] (column pair c = columns 2c, 2c + 1).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace cofem {
namespace dct1 {

__device__ __forceinline__ int64_t sig_inv(int64_t i, int64_t D) { return (i & 1) ? D - 1 - (i >> 1) : (i >> 1); }
__device__ __forceinline__ double ck(int64_t k, int64_t D) { return k == 0 ? sqrt(1.0 / (double)D) : sqrt(2.0 / (double)D); }
// e^{-i pi k / 2D}
__device__ __forceinline__ double2 twm(int64_t k, int64_t D) {
  double s, c;
  sincospi((double)k / (2.0 * (double)D), &s, &c);
  return make_double2(c, -s);
}

// W (complex [D][hc]) = spec(X_{2c}) + i spec(X_{2c+1}) of the real block X
// ([>= D][ldq]): the DCT-III input of every column pair
__global__ void k_pre(int64_t D, int ldq, const double* __restrict__ X, double2* __restrict__ W) {
  const int hc = ldq / 2;
  const double inv_d = 1.0 / (double)D;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < D * hc; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = e / hc;
    const int c = (int)(e % hc);
    const int64_t nk = k == 0 ? 0 : D - k;
    const double2 xk = *reinterpret_cast<const double2*>(X + k * ldq + 2 * c);
    const double2 xn = *reinterpret_cast<const double2*>(X + nk * ldq + 2 * c);
    const double ick = 1.0 / ck(k, D), icn = 1.0 / ck(nk, D);
    const double2 t = twm(k, D);  // conj: e^{+i pi k / 2D} = (t.x, -t.y)
    // spec(x)_k = e^{i pi k/2D} (x_k / c_k - i x_nk / c_nk) / D  (x_nk term absent at k = 0)
    auto spec = [&](double a_k, double a_n) {
      const double re = a_k * ick, im = k == 0 ? 0.0 : -a_n * icn;
      return make_double2((t.x * re + t.y * im) * inv_d, (t.x * im - t.y * re) * inv_d);
    };
    const double2 sa = spec(xk.x, xn.x), sb = spec(xk.y, xn.y);
    W[e] = make_double2(sa.x - sb.y, sa.y + sb.x);
  }
}

// V *= mask in v order (the Phi^T Phi middle step)
__global__ void k_vmask(int64_t D, int hc, double2* __restrict__ V, const uint8_t* __restrict__ mask_v) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < D * hc; e += (int64_t)gridDim.x * blockDim.x)
    if (!mask_v[e / hc]) V[e] = make_double2(0.0, 0.0);
}

// Y ([rows][ldq] real, rows >= D zero-filled) = orthonormal DCT-II of the
// column pairs whose reordered vectors were FFT'd into Z (complex [D][hc])
__global__ void k_post(int64_t D, int64_t rows, int ldq, const double2* __restrict__ Z, double* __restrict__ Y) {
  const int hc = ldq / 2;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < rows * hc; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = e / hc;
    const int c = (int)(e % hc);
    double2 out = make_double2(0.0, 0.0);
    if (k < D) {
      const int64_t nk = k == 0 ? 0 : D - k;
      const double2 zk = Z[k * hc + c], zn = Z[nk * hc + c];
      // V_a = (Z_k + conj Z_nk) / 2, V_b = (Z_k - conj Z_nk) / 2i
      const double2 va = make_double2(0.5 * (zk.x + zn.x), 0.5 * (zk.y - zn.y));
      const double2 vb = make_double2(0.5 * (zk.y + zn.y), -0.5 * (zk.x - zn.x));
      const double2 t = twm(k, D);
      const double s = ck(k, D);
      out = make_double2(s * (t.x * va.x - t.y * va.y), s * (t.x * vb.x - t.y * vb.y));
    }
    *reinterpret_cast<double2*>(Y + k * ldq + 2 * c) = out;
  }
}

// Phi V rows: out[r][q] = x[mask[r]][q], x = v o sigma^{-1} (v = the DCT-III
// output in v order, complex [D][hc]); rows >= nm of out are zeroed
__global__ void k_gather(int64_t nm, int64_t rows, int64_t D, int ldq, const int64_t* __restrict__ mask,
                         const double2* __restrict__ V, double* __restrict__ out) {
  const int hc = ldq / 2;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < rows * hc; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / hc;
    const int c = (int)(e % hc);
    const double2 v = r < nm ? V[sig_inv(mask[r], D) * hc + c] : make_double2(0.0, 0.0);
    *reinterpret_cast<double2*>(out + r * ldq + 2 * c) = v;
  }
}

// Phi^T U input: V (complex [D][hc], zeroed by the caller) at v(sigma^{-1}(mask[r])) = U[r]
__global__ void k_scatter(int64_t nm, int64_t D, int ldq, const int64_t* __restrict__ mask,
                          const double* __restrict__ U, double2* __restrict__ V) {
  const int hc = ldq / 2;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nm * hc; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / hc;
    const int c = (int)(e % hc);
    V[sig_inv(mask[r], D) * hc + c] = *reinterpret_cast<const double2*>(U + r * ldq + 2 * c);
  }
}

}  // namespace dct1
}  // namespace cofem
