// dct1024.cuh -- the 2-D DCT passes of dct.cuh at n = 1024 (BASELINE config
// 5), one warp per complex FFT with the data resident in registers.
//
// dct.cuh's passes keep an item (two packed real vectors = one complex
// length-1024 FFT) in shared memory and walk it five times per transform; at
// 12 warps / SM they are bound by shared-memory latency and block barriers.
// Here a warp owns its item end to end:
//   * lane lt holds the 32 complex values of indices lt + 32 r (128 registers);
//     global loads land in those registers directly (the Makhoul even/odd
//     reordering is an address computation), stores leave from them;
//   * the four-step FFT is DFT-32 in registers (compile-time twiddles: the
//     multiplications by 1 and -i vanish), twiddle from a lane-contiguous
//     table, one padded shared-memory transpose (the only shared-memory
//     traffic of a transform), DFT-32 in registers;
//   * the Makhoul post / pre steps pair coefficient k with n - k.  k = lt +
//     32 r lives in lane lt slot r and n - k in lane 32 - lt slot 31 - r, so
//     the pair meets through one shuffle each way; every pair is computed
//     once (slots r < 16 own it).  Lane 0 (k = 32 j pairs with 32 (32 - j) in
//     the same lane, k = 0 and 512 with themselves) goes through 33 words of
//     the idle transpose region;
//   * the fused column pass (DCT-II, mask, DCT-III) never leaves registers
//     between its two FFTs; with c_k cancelling, the masked pair step is
//     W = conj(t) (m_k Re(t V), m_{n-k} Im(t V)), t = e^{-i pi k / 2n};
//   * no block barriers after the prologue: one 12-warp block per SM, every
//     warp with its own transpose region, walks its own items; the step
//     twiddles (16 KB, lane-contiguous) and the lanes' Makhoul twiddles sit in
//     shared memory next to the regions (the L1 left beside 220 KB of shared
//     memory cannot hold them against the streaming loads).
// Outputs agree with dct.cuh's to a few ulp (same FFT factorisation, other
// operation order); tests compare both with scipy to 1e-12.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "dct.cuh"

namespace cofem {
namespace dctw {

using dctf::P_FMI;
using dctf::P_FWD;
using dctf::P_INV;

constexpr int NN = 1024;
constexpr int ZT = 33 * 32;                         // padded 32 x 32 transpose region, double2 entries
#ifndef DCTW_WARPS
#define DCTW_WARPS 12
#endif
constexpr int WARPS = DCTW_WARPS;                   // 168 registers x 32 lanes x 12 = the register file
constexpr int TWS = 1024 + 64;                      // step twiddles [k2][lt], then e^{-i pi k / 2n} at k = lt and k = 32 j
constexpr size_t SMEM = (size_t)(TWS + WARPS * ZT) * sizeof(double2);  // 17408 + 12 x 16896 B

// cos(2 pi j / 128), j = 0..32; the switch folds once the callers' loops unroll
__host__ __device__ __forceinline__ constexpr double cos128(int j) {
  switch (j) {
    case 0: return 1.0;
    case 1: return 0.9987954562051724;
    case 2: return 0.9951847266721969;
    case 3: return 0.989176509964781;
    case 4: return 0.9807852804032304;
    case 5: return 0.970031253194544;
    case 6: return 0.9569403357322088;
    case 7: return 0.9415440651830208;
    case 8: return 0.9238795325112867;
    case 9: return 0.9039892931234433;
    case 10: return 0.881921264348355;
    case 11: return 0.8577286100002721;
    case 12: return 0.8314696123025452;
    case 13: return 0.8032075314806449;
    case 14: return 0.773010453362737;
    case 15: return 0.7409511253549591;
    case 16: return 0.7071067811865476;
    case 17: return 0.6715589548470183;
    case 18: return 0.6343932841636455;
    case 19: return 0.5956993044924335;
    case 20: return 0.5555702330196023;
    case 21: return 0.5141027441932217;
    case 22: return 0.4713967368259978;
    case 23: return 0.4275550934302822;
    case 24: return 0.38268343236508984;
    case 25: return 0.33688985339222005;
    case 26: return 0.29028467725446233;
    case 27: return 0.24298017990326398;
    case 28: return 0.19509032201612833;
    case 29: return 0.14673047445536175;
    case 30: return 0.09801714032956077;
    case 31: return 0.049067674327418126;
    default: return 0.0;
  }
}
// e^{-2 pi i j / 128} for j in [0, 64]
__host__ __device__ __forceinline__ constexpr double wre128(int j) { return j <= 32 ? cos128(j) : -cos128(64 - j); }
__host__ __device__ __forceinline__ constexpr double wim128(int j) { return j <= 32 ? -cos128(32 - j) : -cos128(j - 32); }

__host__ __device__ __forceinline__ constexpr int brev5(int k) {
  return ((k & 1) << 4) | ((k & 2) << 2) | (k & 4) | ((k & 8) >> 2) | ((k & 16) >> 4);
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cmulc(double2 a, double2 t) {  // a * conj(t)
  return make_double2(fma(a.x, t.x, a.y * t.y), fma(a.y, t.x, -a.x * t.y));
}
__device__ __forceinline__ double2 shfl2(double2 v, int src) {
  return make_double2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}

// DFT-32 in registers, decimation in frequency: natural-order input,
// bit-reversed output (X[k] = x[brev5(k)]).  SIGN = -1 forward, +1 inverse.
template <int SIGN>
__device__ __forceinline__ void dft32(double2 (&x)[32]) {
#pragma unroll
  for (int s = 32; s >= 2; s >>= 1) {
#pragma unroll
    for (int b = 0; b < 32; b += s) {
#pragma unroll
      for (int j = 0; j < s / 2; ++j) {
        const double2 a = x[b + j], c = x[b + j + s / 2];
        x[b + j] = make_double2(a.x + c.x, a.y + c.y);
        const double dx = a.x - c.x, dy = a.y - c.y;
        const int tj = j * (128 / s);  // twiddle e^{-+ 2 pi i tj / 128}, tj < 64
        if (tj == 0) {
          x[b + j + s / 2] = make_double2(dx, dy);
        } else if (tj == 32) {  // -i (forward), +i (inverse)
          x[b + j + s / 2] = SIGN < 0 ? make_double2(dy, -dx) : make_double2(-dy, dx);
        } else {
          const double wr = wre128(tj), wi = SIGN < 0 ? wim128(tj) : -wim128(tj);
          x[b + j + s / 2] = make_double2(fma(dx, wr, -dy * wi), fma(dx, wi, dy * wr));
        }
      }
    }
  }
}

// Length-1024 FFT of one warp: lane lt holds x[lt + 32 r] in r[], and ends
// with X[lt + 32 r] in r[] (natural slots).  tws[k2 * 32 + lt] = the forward
// step twiddle w^{lt k2} (shared memory); the inverse multiplies by its
// conjugate.  Unnormalised both ways.
struct NoPrefetch {
  __device__ __forceinline__ void operator()() const {}
};
// `mid` runs between the transpose and the second DFT-32: loads issued there
// (the pair-mask bytes) are covered by the DFT without living through the first
template <int SIGN, class Mid = NoPrefetch>
__device__ __forceinline__ void fft1024(double2 (&r)[32], double2* zt, const double2* tws, int lt, Mid mid = Mid()) {
  dft32<SIGN>(r);
  __syncwarp();  // earlier readers of the region are done
#pragma unroll
  for (int k2 = 0; k2 < 32; ++k2) {
    double2 v = r[brev5(k2)];
    if (k2 != 0) v = SIGN < 0 ? cmul(v, tws[k2 * 32 + lt]) : cmulc(v, tws[k2 * 32 + lt]);
    zt[lt * 33 + k2] = v;
  }
  __syncwarp();
#pragma unroll
  for (int n1 = 0; n1 < 32; ++n1) r[n1] = zt[n1 * 33 + lt];
  mid();
  dft32<SIGN>(r);
#pragma unroll
  for (int k1 = 0; k1 < 32; ++k1) {
    if (k1 < brev5(k1)) {
      const double2 t = r[k1];
      r[k1] = r[brev5(k1)];
      r[brev5(k1)] = t;
    }
  }
}

// One coefficient pair (k, n - k) of the two packed vectors; z = value at k,
// y = value at n - k, t = the mode's scaled Makhoul twiddle at k.
// With t = 2^-5.5 e^{-i pi k / 2n} in every mode (c_k / 2 = 1 / (c_k n) = 1 / sqrt(2 n) = 2^-5.5 at n = 1024):
//   P_FWD: spectrum -> orthonormal DCT-II coefficients
//   P_FMI: spectrum -> masked input of the (unnormalised) inverse FFT
//   P_INV: coefficients -> input of the inverse FFT
template <int MODE>
__device__ __forceinline__ void pair_op(double2 z, double2 y, double2 t, unsigned mbits, double2& ok, double2& onk) {
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
  if (!(mbits & 1u)) ua.x = ub.x = 0.0;
  if (!(mbits & 2u)) ua.y = ub.y = 0.0;
  const double2 wa = cmulc(ua, t), wb = cmulc(ub, t);
  ok = make_double2(wa.x - wb.y, wa.y + wb.x);
  onk = make_double2(wa.x + wb.y, wb.x - wa.y);
}

// The Makhoul pair step over a warp's registers (see the header comment).
// tmk = the scaled twiddles (shared memory: [lt] at k = lt, [32 + j] at k = 32 j),
// mb = the lane's 16 pair-mask bytes, mb0 = lane 0's byte for pair j = lt.
template <int MODE>
__device__ __forceinline__ void pair_step(double2 (&r)[32], double2* zt, const double2* tmk, int lt, uint4 mb,
                                          unsigned mb0) {
  const int pl = (32 - lt) & 31;
  const double2 tl = tmk[lt];
  __syncwarp();
  if (lt == 0) {
#pragma unroll
    for (int j = 0; j < 32; ++j) zt[j] = r[j];
  }
  __syncwarp();
#pragma unroll
  for (int k1 = 0; k1 < 16; ++k1) {
    const double2 y = shfl2(r[31 - k1], pl);
    // e^{-i pi (lt + 32 k1) / 2n} = tl e^{-2 pi i k1 / 128}
    const double2 t = k1 == 0 ? tl : cmul(tl, make_double2(wre128(k1), wim128(k1)));
    const unsigned w = k1 < 4 ? mb.x : k1 < 8 ? mb.y : k1 < 12 ? mb.z : mb.w;
    double2 ok, onk;
    pair_op<MODE>(r[k1], y, t, w >> (8 * (k1 & 3)), ok, onk);
    r[k1] = ok;
    r[31 - k1] = shfl2(onk, pl);
  }
  if (lt <= 16) {  // lane 0's column: pair j = lt
    const double2 z = zt[lt], y = zt[(32 - lt) & 31];
    double2 ok, onk;
    pair_op<MODE>(z, y, tmk[32 + lt], mb0, ok, onk);
    if (lt == 0) {  // k = 0: unpaired; c_0 = 1 / (c_0 n) = 1 / 32, masked identity 1 / n
      const double f = MODE == P_FMI ? ((mb0 & 1u) ? 0.0009765625 : 0.0) : 0.03125;
      ok = make_double2(f * z.x, f * z.y);
    }
    zt[lt] = ok;
    if (lt >= 1 && lt < 16) zt[32 - lt] = onk;
  }
  __syncwarp();
  if (lt == 0) {
#pragma unroll
    for (int j = 0; j < 32; ++j) r[j] = zt[j];
  }
}

// streamed once: keep it out of the small L1 beside the shared-memory carve-out
__device__ __forceinline__ double2 ld_in(const double2* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
#ifndef DCTW_STORE
#define DCTW_STORE 1  // 0 streaming (.cs), 1 write-back: the two column pairs of a 32-B sector are stored by two warps
#endif
__device__ __forceinline__ void st_out(double2* p, double2 v) {
  if (DCTW_STORE == 0) __stcs(p, v);
  else *p = v;
}

// One pass over an (nouter x 1024 x ldq) float64 block, as dctf::k_dct_pass:
// item (o, p) transforms the two vectors src[o stride_o + 2 p + m stride_m + {0, 1}], m < 1024;
// so2 / sm2 = the strides in 16-byte units (32-bit: a row address is one wide multiply-add,
// cheap enough that the compiler recomputes it instead of keeping 32 loop-invariant offsets).
//   twF[k2 * 32 + lt]: forward step twiddles; tw: e^{-i pi k / 2n} / sqrt(2n);
//   pm[(o 32 + lt) 16 + k1]: bit 0 = mask at k = lt + 32 k1 of outer index o,
//   bit 1 = mask at n - k; pm[(o 32) 16] bit 2 = mask at k = 512.
template <int MODE>
__global__ void __launch_bounds__(32 * WARPS, 1)
    k_pass(const double* __restrict__ src, double* __restrict__ dst, int so2, int sm2, int nouter,
           int npairs, const double2* __restrict__ twF, const double2* __restrict__ tw, const uint8_t* __restrict__ pm,
           const Status* __restrict__ stt) {
  if (stt && stt->done) return;
  extern __shared__ double2 dsm[];
  double2* tws = dsm;
  double2* tmk = dsm + 1024;
  const int lt = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double2* zt = dsm + TWS + warp * ZT;
  for (int i = threadIdx.x; i < 1024; i += 32 * WARPS) tws[i] = __ldg(twF + i);
  volatile int* sm2v = reinterpret_cast<volatile int*>(dsm + 1024 + 49);
  if (threadIdx.x == 0) *sm2v = sm2;
  if (threadIdx.x < 49) {
    tmk[threadIdx.x] = __ldg(tw + (threadIdx.x < 32 ? threadIdx.x : 32 * (threadIdx.x - 32)));
  }
  __syncthreads();
  const int nitems = nouter * npairs;
  for (int item = blockIdx.x * WARPS + warp; item < nitems; item += gridDim.x * WARPS) {
    const int o = item / npairs, p = item % npairs;
    // the row stride re-read from shared memory (volatile) per use: a row address is one wide
    // multiply-add, but with a stride the compiler can see through it hoists the 32
    // loop-invariant row offsets out of the item loop, shares them between the loads and the
    // stores, and spills them
    const int sm2l = *sm2v;
    const double2* s0 = reinterpret_cast<const double2*>(src) + ((int64_t)o * so2 + p);
    double2* d0 = reinterpret_cast<double2*>(dst) + ((int64_t)o * so2 + p);
    uint4 mb = make_uint4(0, 0, 0, 0);
    unsigned mb0 = 0;
    auto load_mask = [&]() {
      if (MODE == P_FMI) {
        mb = __ldg(reinterpret_cast<const uint4*>(pm + ((int64_t)o * 32 + lt) * 16));
        mb0 = __ldg(pm + (int64_t)o * 512 + (lt & 15));
      }
    };
    double2 r[32];
    if (MODE == P_INV) {
#pragma unroll
      for (int k1 = 0; k1 < 32; ++k1) r[k1] = ld_in(s0 + (int64_t)(lt + 32 * k1) * sm2l);
      pair_step<P_INV>(r, zt, tmk, lt, mb, mb0);
    } else {
      // v[n] = x[2n] (n < 512), x[2047 - 2n] (n >= 512) at n = lt + 32 r
#pragma unroll
      for (int n2 = 0; n2 < 32; ++n2) {
        const int m = n2 < 16 ? 2 * lt + 64 * n2 : 2047 - 2 * lt - 64 * n2;
        r[n2] = ld_in(s0 + (int64_t)m * sm2l);
      }
      fft1024<-1>(r, zt, tws, lt, load_mask);
      if (lt == 16) mb0 = ((mb0 >> 2) & 1u) * 3u;
      pair_step<MODE>(r, zt, tmk, lt, mb, mb0);
      if (MODE == P_FWD) {
#pragma unroll
        const int sm2s = *sm2v;
#pragma unroll
        for (int k1 = 0; k1 < 32; ++k1) st_out(d0 + (int64_t)(lt + 32 * k1) * sm2s, r[k1]);
        continue;
      }
    }
    fft1024<1>(r, zt, tws, lt);
    const int sm2s = *sm2v;
#pragma unroll
    for (int n2 = 0; n2 < 32; ++n2) {
      const int m = n2 < 16 ? 2 * lt + 64 * n2 : 2047 - 2 * lt - 64 * n2;
      st_out(d0 + (int64_t)m * sm2s, r[n2]);
    }
  }
}

}  // namespace dctw
}  // namespace cofem
