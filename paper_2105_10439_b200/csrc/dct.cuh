// dct.cuh -- 2-D partial-DCT dictionaries (BASELINE config 4) as fused
// float64 FFT passes.
//
// Phi = M * DCT2: orthonormal 2-D DCT-II of an n x n image, then the
// coefficients selected by the mask M.  One PCG apply needs
//   Psi = beta DCT2^T (M .* DCT2 P) + alpha .* P
// for the Q = ldq column images of P at once, which is three passes over HBM:
//   row pass    DCT-II along j                        P    -> T1
//   column pass DCT-II along i, mask, DCT-III along i  T1   -> T2  (fused)
//   row pass    DCT-III along j                        T2   -> Z
// then either the streaming PCG combine Psi = beta Z + alpha .* P, pi = <P, Psi>
// (k_combine), or -- the Psi-free step, n >= 512 -- the last pass also returns
// ||Z||^2 per column (= ||Phi P||^2: orthonormal rows) and k_update_psi
// (pcg.cuh) updates the residual straight from Z.
// Each pass streams one n^2 x ldq float64 block in and one out,
// O(log n) arithmetic per element (a dense C X C^T would be O(n)); measured
// latency-bound at 12 warps / SM (0.33 of HBM on the column pass).
//
// Every 1-D transform is Makhoul's: DCT-II of real x is Re(e^{-i pi k / 2n}
// FFT_n(v)[k]) of the even/odd reordering v, and DCT-III inverts it with an
// inverse FFT of e^{i pi k / 2n}(X[k] - i X[n-k]).  Two real vectors ride in
// one complex FFT (real / imaginary part); the pre / post steps work once per
// coefficient pair (k, n - k) (pair_op).  The length-n FFT is a four-step
// N1 x N2 decomposition: register DFTs of size N2 and N1, one twiddle
// multiply and two padded shared-memory transposes.
//
// Block layout (ldq = padded column count, Q images interleaved):
//   P[(i n + j) ldq + q]       pixel-major, as every PCG block
//   T1[(i n + l) ldq + q]      after the row pass (l = j frequency)
//   Y[(k n + l) ldq + q]       coefficient grid after the column pass
// A pass item is (outer index o, q-group of 2 FPI = 4 columns): FPI = 2 complex FFTs,
// one warp each at n >= 512.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.cuh"
#include "pcg.cuh"

namespace cofem {
namespace dctf {

__constant__ double2 c_w64[64];  // e^{-2 pi i j / 64}

#ifndef DCT_STORE
#define DCT_STORE 0  // timing builds: 0 streaming (.cs), 1 default write-back, 2 write-through
#endif
__device__ __forceinline__ void st_out(double2* p, double2 v) {
  if (DCT_STORE == 0) __stcs(p, v);
  else if (DCT_STORE == 1) *p = v;
  else __stwt(p, v);
}

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 conj2(double2 a) { return make_double2(a.x, -a.y); }

__host__ __device__ constexpr int ilog2(int v) { return v <= 1 ? 0 : 1 + ilog2(v / 2); }
// bit reversal of the low `bits` bits; iterative so that unrolled loops fold it
__host__ __device__ __forceinline__ constexpr int brev(int k, int bits) {
  int r = 0;
#pragma unroll
  for (int b = 0; b < 6; ++b)
    if (b < bits) r |= ((k >> b) & 1) << (bits - 1 - b);
  return r;
}

// In-register DFT of size R (power of two <= 64), decimation in frequency:
// natural-order input, bit-reversed output (X[k] = x[brev(k)]).  SIGN = -1
// forward, +1 inverse (unnormalised).
template <int R, int SIGN>
__device__ __forceinline__ void dft_reg(double2 (&x)[R]) {
#pragma unroll
  for (int s = R; s >= 2; s >>= 1) {
#pragma unroll
    for (int b = 0; b < R; b += s) {
#pragma unroll
      for (int j = 0; j < s / 2; ++j) {
        const double2 a = x[b + j], c = x[b + j + s / 2];
        x[b + j] = cadd(a, c);
        const double2 d = csub(a, c);
        const int tj = j * (64 / s);  // twiddle e^{-+ 2 pi i tj / 64}
        if (tj == 0) {
          x[b + j + s / 2] = d;
        } else if (tj == 16) {  // -i (forward), +i (inverse): no multiplication
          x[b + j + s / 2] = SIGN < 0 ? make_double2(d.y, -d.x) : make_double2(-d.y, d.x);
        } else {
          const double2 w = c_w64[tj];
          x[b + j + s / 2] = cmul(d, SIGN < 0 ? w : conj2(w));
        }
      }
    }
  }
}

// Length-N (= N1 N2) FFT of one region z (natural order in, natural order
// out) by the TPF = N2 threads lt of its group.  Input x[n1 + N1 n2]; step 1
// DFTs over n2 (thread n1), twiddle w_N^{n1 k2}, step 3 DFTs over n1
// (thread k2) -> X[k2 + N2 k1].  The intermediate uses the padded stride
// N2 + 1 (conflict-free transposes).  Contains __syncthreads: every thread of
// the block must call it.
// Step-1 twiddles w_N^{lt k2} of one thread: the table value every 8th k2,
// powers of the thread constant w1 = w_N^{lt} in between (<= 7 products).
// With TABLE every twiddle comes from the lane-contiguous table
// wT[k2 * N1 + lt] instead (independent L1 loads; see DCT_TWT).
template <int N2>
struct Tw1 {
  double2 w1;
  const double2* wN;
  const double2* wT;
};

// a group of N2 = 32 threads is one warp and the region is its own: warp-level barriers inside
template <int N2>
__device__ __forceinline__ void group_sync() {
  if (N2 == 32) __syncwarp();
  else __syncthreads();
}

template <int N1, int N2, int SIGN, bool TABLE = false>
__device__ __forceinline__ void fft4step(double2* z, int lt, const Tw1<N2>& tw1) {
  constexpr int B2 = ilog2(N2), B1 = ilog2(N1);
  {
    double2 r[N2];
    if (lt < N1) {
#pragma unroll
      for (int n2 = 0; n2 < N2; ++n2) r[n2] = z[lt + N1 * n2];
      dft_reg<N2, SIGN>(r);
    }
    group_sync<N2>();
    if (lt < N1) {
      const double2 w1 = SIGN < 0 ? tw1.w1 : conj2(tw1.w1);
      double2 cur = make_double2(1.0, 0.0);
#pragma unroll
      for (int k2 = 0; k2 < N2; ++k2) {
        if (TABLE) {
          if (k2 > 0) {
            const double2 w = __ldg(tw1.wT + k2 * N1 + lt);
            cur = SIGN < 0 ? w : conj2(w);
          }
        } else if (k2 % 8 == 0) {
          const double2 w = __ldg(tw1.wN + lt * k2);
          cur = SIGN < 0 ? w : conj2(w);
        } else {
          cur = cmul(cur, w1);
        }
        const double2 v = r[brev(k2, B2)];
        z[lt * (N2 + 1) + k2] = k2 == 0 ? v : cmul(v, cur);
      }
    }
    group_sync<N2>();
  }
  double2 s[N1];
#pragma unroll
  for (int n1 = 0; n1 < N1; ++n1) s[n1] = z[n1 * (N2 + 1) + lt];
  dft_reg<N1, SIGN>(s);
  group_sync<N2>();
#pragma unroll
  for (int k1 = 0; k1 < N1; ++k1) z[lt + N2 * k1] = s[brev(k1, B1)];
  __syncthreads();
}

enum { P_FWD = 0, P_INV = 1, P_FMI = 2 };  // DCT-II; DCT-III; DCT-II -> mask -> DCT-III

__device__ __forceinline__ double2 cmulc(double2 a, double2 t) {  // a conj(t)
  return make_double2(fma(a.x, t.x, a.y * t.y), fma(a.y, t.x, -a.x * t.y));
}

// The Makhoul pre / post step on one coefficient pair (k, n - k) of the two
// real vectors packed in a complex FFT; z = value at k, y = value at n - k,
// t = e^{-i pi k / 2n} / sqrt(2n) (c_k / 2 = 1 / (c_k n) = 1 / sqrt(2n) for k >= 1).
//   P_FWD: spectrum Z -> orthonormal DCT-II coefficients (X_a, X_b) at k and n - k:
//          V_a = (Z[k] + conj Z[n-k]) / 2, V_b = (Z[k] - conj Z[n-k]) / 2i,
//          X[k] = c_k Re(e^{..} V[k]), X[n-k] = -c_k Im(e^{..} V[k])
//   P_INV: coefficients -> input W of the unnormalised inverse FFT,
//          W[k] = conj(t) ((a_k + b_{n-k}) + i (b_k - a_{n-k})), W[n-k] = t ((a_k - b_{n-k}) + i (a_{n-k} + b_k))
//   P_FMI: both with the mask in between.  c_k cancels, and with u = t (2 V[k]):
//          W_a[k] = conj(t) (m_k Re u_a, m_{n-k} Im u_a), W[n-k] = conj(W[k]) per vector
// (derivation and a lane-level emulation against scipy: tools/dctw_emul.py).
template <int MODE>
__device__ __forceinline__ void pair_op(double2 z, double2 y, double2 t, bool mk, bool mnk, double2& ok, double2& onk) {
  if (MODE == P_INV) {
    const double2 p = make_double2(z.x + y.y, z.y - y.x), q = make_double2(z.x - y.y, y.x + z.y);
    ok = cmulc(p, t);
    onk = cmul(q, t);
    return;
  }
  const double2 sa = make_double2(z.x + y.x, z.y - y.y), sb = make_double2(z.y + y.y, y.x - z.x);
  if (MODE == P_FWD) {
    ok = make_double2(fma(t.x, sa.x, -t.y * sa.y), fma(t.x, sb.x, -t.y * sb.y));
    onk = make_double2(-fma(t.y, sa.x, t.x * sa.y), -fma(t.y, sb.x, t.x * sb.y));
    return;
  }
  double2 ua = cmul(sa, t), ub = cmul(sb, t);
  if (!mk) ua.x = ub.x = 0.0;
  if (!mnk) ua.y = ub.y = 0.0;
  const double2 wa = cmulc(ua, t), wb = cmulc(ub, t);
  ok = make_double2(wa.x - wb.y, wa.y + wb.x);
  onk = make_double2(wa.x + wb.y, wb.x - wa.y);
}

// complex entries per FFT region: the padded transpose, plus 4 so that the
// FPI regions start 16 banks apart (adjacent lanes of the pair loops work on
// the same k in adjacent regions)
__host__ __device__ constexpr int region_entries(int n1, int n2) { return n1 * (n2 + 1) + 4; }

// One pass over an (nouter x n x ldq) float64 block: item (o, g) transforms
// the 8 vectors src[o stride_o + g 8 + m stride_m + v], v < 8, m < n.
//   P_FWD: dst = DCT-II;  P_INV: dst = DCT-III;  P_FMI: dst = DCT-III(mask .* DCT-II)
//   with the transposed 0/1 grid gridT[o n + k] (outer index o, coefficient k along m)
// The last row pass of a PCG apply can also return vv_q = ||Z_q||^2 per column (VV): with
// orthonormal rows, ||Phi^T Phi P||^2 = ||Phi P||^2, so pi = beta vv + <P, alpha P> is known
// before Psi exists and the residual update needs no Psi block (k_update_psi, pcg.cuh).
// A thread's columns are (4 g + 2 f, + 1) with f = lane parity and g changing per item: an
// item ends with a shuffle fold over the lanes of equal parity into the warp's accumulators
// in shared memory; the block folds its warps in order and writes partials[block][q]; the
// consumer (k_update_psi) folds the blocks in order (deterministic: the item -> block map is
// static; a last-block fold by this kernel's 64-thread blocks cost 20 us of serial tail).
constexpr int VV_MAXQ = 32;
struct VvArgs {
  double* partials = nullptr;  // [grid][ldq]
  int ldq = 0;
};
// fold v over the lanes of this lane's parity
__device__ __forceinline__ double parity_fold(double v) {
#pragma unroll
  for (int d = 16; d >= 2; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
  return v;
}

#ifndef DCT_TWT
#define DCT_TWT false  // true: every step twiddle from the lane-contiguous table -- measured 13 % slower (column
                       // pass 0.189 vs 0.167 ms): 31 more L1 loads per FFT cost more than the 28 complex products
#endif
#ifndef DCT_FPI
#define DCT_FPI 2  // complex FFTs (column pairs) per item / block: 2 measured best (4: -7 %, 1: -16 %)
#endif
template <int N1, int N2, int MODE, int FPI = DCT_FPI, bool VV = false>
__global__ void __launch_bounds__(FPI * N2, (N2 >= 32 ? 12 / FPI : 16 / FPI))
    k_dct_pass(const double* __restrict__ src, double* __restrict__ dst, int64_t stride_o, int64_t stride_m,
               int nouter, int ngroups, const double2* __restrict__ wN, const double2* __restrict__ tws,
               const uint8_t* __restrict__ grid, const Status* __restrict__ stt, const double2* __restrict__ wT,
               VvArgs vv = VvArgs()) {
  constexpr int N = N1 * N2, TPF = N2, NT = FPI * TPF;
  constexpr int ZS = region_entries(N1, N2);
  constexpr int NW = (NT + 31) / 32;
  static_assert(!VV || (MODE == P_INV && FPI == 2 && NT % 32 == 0), "vv: last row pass, f = lane parity");
  if (stt && stt->done) return;
  extern __shared__ double2 zsm[];  // [FPI][ZS], then the item's mask column (P_FMI) / the vv accumulators
  uint8_t* mcol = reinterpret_cast<uint8_t*>(zsm + FPI * ZS);
  double* wacc = reinterpret_cast<double*>(mcol);  // [NW][VV_MAXQ] (VV: the mask column is unused)
  const int t = threadIdx.x;
  const int f_own = t / TPF, lt = t % TPF;
  if (VV)
    for (int i = t; i < NW * VV_MAXQ; i += NT) wacc[i] = 0.0;  // visible after the first item's barriers
  // thread constants: step-1 twiddles; the scaled Makhoul twiddles tws[k] = e^{-i pi k / 2n} / sqrt(2n)
  // come from their (L1-resident) table
  Tw1<N2> tw1;
  tw1.w1 = __ldg(wN + (lt < N1 ? lt : 0));
  tw1.wN = wN;
  tw1.wT = wT;
  const double dc = 1.0 / sqrt((double)N);  // c_0 = 1 / (c_0 n); folds at compile time
  for (int item = blockIdx.x; item < nouter * ngroups; item += gridDim.x) {
    const int o = item / ngroups, g = item % ngroups;
    const int64_t base = (int64_t)o * stride_o + g * (2 * FPI);
    __syncthreads();  // the previous item is done with shared memory
    // ---- load: 4 consecutive threads copy one contiguous 64-B row of the item;
    // cp.async keeps every copy of the thread in flight without registers
#pragma unroll 8
    for (int e = t; e < FPI * N; e += NT) {
      const int f = e % FPI, m = e / FPI;
      const int dst_i = MODE == P_INV ? m : ((m & 1) ? N - 1 - (m >> 1) : (m >> 1));  // Makhoul reorder
      cp_async16(zsm + f * ZS + dst_i, src + base + m * stride_m + 2 * f);
    }
    if (MODE == P_FMI)  // gridT[o n + k]: this item's mask column, n bytes
      for (int b = t; b < N / 16; b += NT) cp_async16(mcol + 16 * b, grid + (int64_t)o * N + 16 * b);
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    // The pair loops: slot e = (f, kk), kk < n / 2; kk >= 1 is the pair (kk, n - kk), kk = 0
    // carries the two unpaired coefficients k = 0 and k = n / 2.  In place (pairs are disjoint).
    if (MODE == P_INV) {
#pragma unroll(N1 * N2 >= 1024 ? 4 : 2)
      for (int e = t; e < FPI * (N / 2); e += NT) {
        const int f = e % FPI, kk = e / FPI;
        double2* z = zsm + f * ZS;
        const int k = kk == 0 ? N / 2 : kk, nk = N - k;
        double2 ok, onk;
        pair_op<P_INV>(z[k], z[nk], __ldg(tws + k), true, true, ok, onk);
        z[k] = ok;
        if (kk == 0) z[0] = make_double2(dc * z[0].x, dc * z[0].y);
        else z[nk] = onk;
      }
      __syncthreads();
    }
    fft4step<N1, N2, (MODE == P_INV) ? 1 : -1, DCT_TWT>(zsm + f_own * ZS, lt, tw1);
    if (MODE == P_FWD) {
#pragma unroll(N1 * N2 >= 1024 ? 4 : 2)
      for (int e = t; e < FPI * (N / 2); e += NT) {
        const int f = e % FPI, kk = e / FPI;
        const double2* z = zsm + f * ZS;
        const int k = kk == 0 ? N / 2 : kk, nk = N - k;
        double2 ok, onk;
        pair_op<P_FWD>(z[k], z[nk], __ldg(tws + k), true, true, ok, onk);
        st_out(reinterpret_cast<double2*>(dst + base + k * stride_m + 2 * f), ok);
        if (kk == 0) onk = make_double2(dc * z[0].x, dc * z[0].y);
        st_out(reinterpret_cast<double2*>(dst + base + (kk == 0 ? 0 : nk) * stride_m + 2 * f), onk);
      }
      continue;
    }
    if (MODE == P_FMI) {
      // spectrum -> coefficients -> mask -> inverse-FFT input, in place per pair
      const double dcm = 1.0 / N;
#pragma unroll(N1 * N2 >= 1024 ? 4 : 2)
      for (int e = t; e < FPI * (N / 2); e += NT) {
        const int f = e % FPI, kk = e / FPI;
        double2* z = zsm + f * ZS;
        const int k = kk == 0 ? N / 2 : kk, nk = N - k;
        double2 ok, onk;
        pair_op<P_FMI>(z[k], z[nk], __ldg(tws + k), mcol[k] != 0, mcol[nk] != 0, ok, onk);
        z[k] = ok;
        if (kk == 0) {
          const double m0 = mcol[0] ? dcm : 0.0;
          z[0] = make_double2(m0 * z[0].x, m0 * z[0].y);
        } else {
          z[nk] = onk;
        }
      }
      __syncthreads();
      fft4step<N1, N2, 1, DCT_TWT>(zsm + f_own * ZS, lt, tw1);
    }
    // ---- DCT-III output: x[m] = v[p(m)] (real part: vector 2f, imaginary: 2f + 1)
    double sqa = 0.0, sqb = 0.0;
#pragma unroll 4
    for (int e = t; e < FPI * N; e += NT) {
      const int f = e % FPI, m = e / FPI;
      const double2 v = zsm[f * ZS + ((m & 1) ? N - 1 - (m >> 1) : (m >> 1))];
      if (VV) {
        sqa = fma(v.x, v.x, sqa);
        sqb = fma(v.y, v.y, sqb);
        *reinterpret_cast<double2*>(dst + base + m * stride_m + 2 * f) = v;  // read again right away: no streaming hint
      } else {
        st_out(reinterpret_cast<double2*>(dst + base + m * stride_m + 2 * f), v);
      }
    }
    if (VV) {
      sqa = parity_fold(sqa);
      sqb = parity_fold(sqb);
      if ((t & 31) < 2) {  // lane = f
        double* a = wacc + (t >> 5) * VV_MAXQ + g * (2 * FPI) + 2 * (t & 31);
        a[0] += sqa;
        a[1] += sqb;
      }
    }
  }
  if (VV) {
    __syncthreads();
    for (int q = t; q < vv.ldq; q += NT) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < NW; ++w) s += wacc[w * VV_MAXQ + q];
      vv.partials[(int64_t)blockIdx.x * vv.ldq + q] = s;
    }
  }
}

// measurement gather / scatter on the coefficient grid Y[(k n + l) ldq + q]
__global__ void k_gather(int64_t nm, int ldq, const int64_t* __restrict__ mask, const double* __restrict__ grid_buf,
                         double* __restrict__ v) {
  const int64_t total = nm * ldq;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = e / ldq;
    v[e] = grid_buf[mask[m] * ldq + (e % ldq)];
  }
}

__global__ void k_scatter(int64_t nm, int ldq, const int64_t* __restrict__ mask, const double* __restrict__ v,
                          double* __restrict__ grid_buf) {
  const int64_t total = nm * ldq;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = e / ldq;
    grid_buf[mask[m] * ldq + (e % ldq)] = v[e];
  }
}

}  // namespace dctf
}  // namespace cofem

// ---------------------------------------------------------------------------
// Convolution dictionaries on the same FFT machinery: overlap-save with
// 1024-point blocks.  Phi x (causal conv with h, L taps) and Phi^T x (the
// correlation) are both "circular convolution of a 1024-sample window with a
// fixed spectrum, keep samples [L-1, 1024)": window start b V - (L - 1) with
// the spectrum of h (Phi), or b V with the spectrum of reversed h (Phi^T),
// V = 1024 - (L - 1) outputs per block.  Two real columns ride in one complex
// FFT (h is real, so the packed pair convolves independently), and the
// spectrum carries the 1/1024 of the inverse transform.  Float64 throughout.
namespace cofem {
namespace dctf {

template <int N1, int N2, int FPI = DCT_FPI>
__global__ void __launch_bounds__(FPI * N2, (N2 >= 32 ? 12 / FPI : 16 / FPI))
    k_conv_fft_pass(const double* __restrict__ src, double* __restrict__ dst, int64_t rows, int ldq, int ngroups,
                    int nblocks, int valid, int in_shift, int keep0, const double2* __restrict__ spec,
                    const double2* __restrict__ wN, const Status* __restrict__ stt) {
  constexpr int N = N1 * N2, TPF = N2, NT = FPI * TPF;
  constexpr int ZS = region_entries(N1, N2);
  if (stt && stt->done) return;
  extern __shared__ double2 zsm[];
  const int t = threadIdx.x;
  const int f_own = t / TPF, lt = t % TPF;
  Tw1<N2> tw1;
  tw1.w1 = __ldg(wN + (lt < N1 ? lt : 0));
  tw1.wN = wN;
  tw1.wT = nullptr;
  for (int item = blockIdx.x; item < nblocks * ngroups; item += gridDim.x) {
    const int b = item / ngroups, g = item % ngroups;
    const int64_t w0 = (int64_t)b * valid - in_shift;  // first window row
    __syncthreads();
#pragma unroll 8
    for (int e = t; e < FPI * N; e += NT) {
      const int f = e % FPI, m = e / FPI;
      const int64_t row = w0 + m;
      if (row >= 0 && row < rows) cp_async16(zsm + f * ZS + m, src + row * ldq + g * (2 * FPI) + 2 * f);
      else zsm[f * ZS + m] = make_double2(0.0, 0.0);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    fft4step<N1, N2, -1>(zsm + f_own * ZS, lt, tw1);
    for (int e = t; e < FPI * N; e += NT) {
      const int f = e % FPI, k = e / FPI;
      zsm[f * ZS + k] = cmul(zsm[f * ZS + k], __ldg(spec + k));
    }
    __syncthreads();
    fft4step<N1, N2, 1>(zsm + f_own * ZS, lt, tw1);
    // outputs rows b V + m', m' < valid, from circular samples keep0 + m'
    const int64_t o0 = (int64_t)b * valid;
    for (int e = t; e < FPI * valid; e += NT) {
      const int f = e % FPI, mm = e / FPI;
      const int64_t row = o0 + mm;
      if (row < rows) st_out(reinterpret_cast<double2*>(dst + row * ldq + g * (2 * FPI) + 2 * f), zsm[f * ZS + keep0 + mm]);
    }
  }
}

}  // namespace dctf
}  // namespace cofem
