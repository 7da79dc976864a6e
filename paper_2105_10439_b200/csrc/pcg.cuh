// pcg.cuh -- fused elementwise passes of the blocked PCG and the EM updates.
//
// All per-column reductions (pi, ||R||^2, rho = <R, M^-1 R>, ||B||^2) are
// accumulated in double: a thread owns one column q for the whole
// grid-stride loop (blockDim and grid stride are multiples of ldq), the block
// folds its rows through smem, and the last block to finish (atomic ticket)
// sums the per-block partials in block order -- deterministic, no float
// atomics.  Per-column scalars live in device memory; every consumer block
// re-derives gamma / eta / delta from them, so no host round trip is needed
// inside the PCG loop.
#pragma once
#include "kernels.cuh"

namespace cofem {

struct Scalars {
  // per column (ldq entries each)
  double* rho[2];   // rho of the current direction, double-buffered by step parity
  double* rho_new;  // <R, M^-1 R> after the latest residual update
  double* rn2;      // ||R_q||^2 (contiguous after rho_new: one allreduce)
  double* pi;       // <P_q, A P_q>
  double* bn2;      // ||B_q||^2
  int* frozen;      // breakdown flags
  double* partials; // nblocks x 2 x ldq scratch
  unsigned* ticket; // last-block counters (one per reduction site)
};

template <typename T>
__device__ __forceinline__ double dd(T v) { return (double)v; }

// block-level fold of per-thread column sums; returns via `out` (thread q < ldq)
__device__ __forceinline__ void block_col_reduce(double* sm, int ldq, int nvals, const double* vals,
                                                 double* partials_blk) {
  // sm: nvals x blockDim doubles
  const int t = threadIdx.x, nt = blockDim.x;
  for (int v = 0; v < nvals; ++v) sm[v * nt + t] = vals[v];
  __syncthreads();
  if (t < ldq) {
    for (int v = 0; v < nvals; ++v) {
      double s = 0.0;
      for (int r = t; r < nt; r += ldq) s += sm[v * nt + r];
      partials_blk[v * ldq + t] = s;
    }
  }
}

// last-block reduction of partials[nblk][nvals][ldq] -> outs[v][q]
__device__ __forceinline__ bool last_block_reduce(unsigned* ticket, const double* partials, int ldq, int nvals,
                                                  double* const* outs) {
  __shared__ int is_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned tk = atomicAdd(ticket, 1u);
    is_last = (tk == gridDim.x - 1);
  }
  __syncthreads();
  if (!is_last) return false;
  __threadfence();
  for (int idx = threadIdx.x; idx < nvals * ldq; idx += blockDim.x) {
    const int v = idx / ldq, q = idx % ldq;
    double s = 0.0;
    for (int b = 0; b < (int)gridDim.x; ++b) s += ((volatile const double*)partials)[(b * nvals + v) * ldq + q];
    outs[v][q] = s;
  }
  if (threadIdx.x == 0) *ticket = 0u;
  return true;
}

__device__ __forceinline__ double safe_ratio(double num, double den) { return den != 0.0 ? num / den : 0.0; }

// ---- init: X = 0, P = 0, bn2 = ||R||^2, rho_new = <R, M^-1 R> (R already holds B)
template <typename T>
__global__ void k_pcg_init(int64_t rows, int ldq, int q_real, T* X, T* P, const T* R, const double* minv, int ngroups,
                           const int* group_of_col, Scalars sc) {
  extern __shared__ double sm_init[];
  const int64_t n = rows * ldq;
  const int q = threadIdx.x % ldq;
  const int g = group_of_col ? group_of_col[q] : 0;
  double s_bn = 0.0, s_rho = 0.0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / ldq;
    X[e] = T(0);
    P[e] = T(0);
    const double r = dd(R[e]);
    const double w = (q < q_real) ? r * minv[j * ngroups + g] : 0.0;
    s_bn += r * r;
    s_rho += r * w;
  }
  double vals[2] = {s_bn, s_rho};
  block_col_reduce(sm_init, ldq, 2, vals, sc.partials + (int64_t)blockIdx.x * 2 * ldq);
  double* outs[2] = {sc.bn2, sc.rho_new};
  last_block_reduce(sc.ticket + 0, sc.partials, ldq, 2, outs);
}

// ---- combine: Psi = beta * sum_s Psipart[s] + alpha .* P ; pi_q = <P_q, Psi_q>
// (chunk of QPc columns at column offset qoff; partial buffer is dense QPc)
template <typename T>
__global__ void k_combine(int64_t rows, int ldq, int qoff, int qpc, int nsplit, const T* ppart, double beta,
                          const double* alpha, const T* P, T* Psi, Scalars sc, const Status* st) {
  if (st && st->done) return;
  extern __shared__ double sm_comb[];
  const int64_t n = rows * qpc;
  double s_pi = 0.0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / qpc;
    const int q = (int)(e % qpc);
    T acc = ppart[e];
    for (int s = 1; s < nsplit; ++s) acc += ppart[(int64_t)s * n + e];
    const int64_t idx = j * ldq + qoff + q;
    const T p = P[idx];
    const T psi = T(beta) * acc + T(alpha[j]) * p;
    Psi[idx] = psi;
    s_pi += dd(p) * dd(psi);
  }
  block_col_reduce(sm_comb, qpc, 1, &s_pi, sc.partials + (int64_t)blockIdx.x * qpc);
  double* outs[1] = {sc.pi + qoff};
  last_block_reduce(sc.ticket + 1, sc.partials, qpc, 1, outs);
}

// ---- V = sum_s Vpart[s]  (chunk, dense QPc layout -> V dense QPc)
template <typename T>
__global__ void k_sum_splits(int64_t n, int nsplit, const T* part, T* out, const Status* st) {
  if (st && st->done) return;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    T acc = part[e];
    for (int s = 1; s < nsplit; ++s) acc += part[(int64_t)s * n + e];
    out[e] = acc;
  }
}

// ---- solution update (kernels.py step_solution) fused with the residual
// norms and the next direction's rho:  gamma = rho/pi (0 when pi == 0),
// X += P gamma, R -= Psi gamma, rn2 = ||R||^2, rho_new = <R, M^-1 R>
template <typename T>
__global__ void k_update(int64_t rows, int ldq, int q_real, int parity, T* X, T* R, const T* P, const T* Psi,
                         const double* minv, int ngroups, const int* group_of_col, Scalars sc, const Status* st) {
  if (st && st->done) return;
  extern __shared__ double sm_upd[];
  const int q = threadIdx.x % ldq;
  const int g = group_of_col ? group_of_col[q] : 0;
  const double pi = sc.pi[q];
  const double gamma = safe_ratio(sc.rho[parity][q], pi);
  if (blockIdx.x == 0 && threadIdx.x < ldq && q < q_real && pi == 0.0) sc.frozen[q] = 1;
  const T gm = T(gamma);
  const int64_t n = rows * ldq;
  double s_rn = 0.0, s_rho = 0.0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / ldq;
    X[e] = X[e] + P[e] * gm;
    const T r = R[e] - Psi[e] * gm;
    R[e] = r;
    const double rd = dd(r);
    s_rn += rd * rd;
    if (q < q_real) s_rho += rd * (rd * minv[j * ngroups + g]);
  }
  double vals[2] = {s_rho, s_rn};
  block_col_reduce(sm_upd, ldq, 2, vals, sc.partials + (int64_t)blockIdx.x * 2 * ldq);
  double* outs[2] = {sc.rho_new, sc.rn2};
  last_block_reduce(sc.ticket + 2, sc.partials, ldq, 2, outs);
}

// ---- convergence test (cg.py:141-148) + direction update (kernels.py
// step_direction): eta = rho_new / rho (0 when rho == 0), P = P eta + W
// (or R for the printed recursion), rho <- rho_new.  step == 0 is the
// initialisation pass (no convergence test).
template <typename T>
__global__ void k_direction(int64_t rows, int ldq, int q_real, int step, int max_steps, double tol, int printed,
                            T* P, const T* R, const double* minv, int ngroups, const int* group_of_col, Scalars sc,
                            Status* st) {
  if (st->done) return;
  const int cur = step & 1, nxt = (step + 1) & 1;
  if (step == 0) {
    double b2 = 0.0;
    for (int c = 0; c < ldq; ++c) b2 += sc.bn2[c];
    if (blockIdx.x == 0 && threadIdx.x == 0) st->bnorm = sqrt(b2);
  } else {
    double r2 = 0.0;
    for (int c = 0; c < ldq; ++c) r2 += sc.rn2[c];
    double b2 = 0.0;
    for (int c = 0; c < ldq; ++c) b2 += sc.bn2[c];
    const double delta = sqrt(r2) / sqrt(b2);
    const bool finite = isfinite(delta);
    const bool conv = finite && delta <= tol;
    const bool stop = !finite || conv || step >= max_steps;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      st->steps = step;
      st->delta = delta;
      st->converged = conv ? 1 : 0;
      st->diverged = finite ? 0 : 1;
      if (stop) st->done = 1;
    }
    if (stop) return;
  }
  const int q = threadIdx.x % ldq;
  const int g = group_of_col ? group_of_col[q] : 0;
  const double eta = safe_ratio(sc.rho_new[q], sc.rho[cur][q]);
  const T et = T(eta);
  const int64_t n = rows * ldq;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / ldq;
    const T r = R[e];
    const T w = (q < q_real) ? T(dd(r) * minv[j * ngroups + g]) : T(0);
    P[e] = P[e] * et + (printed ? r : w);
  }
  if (blockIdx.x == 0 && threadIdx.x < ldq) sc.rho[nxt][threadIdx.x] = sc.rho_new[threadIdx.x];
}

// ---- EM glue ---------------------------------------------------------------

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// Rademacher sign of (seed, iteration, global coordinate, probe)
__device__ __forceinline__ int8_t device_probe(uint64_t seed, int iter, int64_t jg, int k) {
  const uint64_t h = splitmix64(seed ^ splitmix64(((uint64_t)iter << 40) ^ ((uint64_t)jg << 8) ^ (uint64_t)k));
  return (h >> 63) ? int8_t(1) : int8_t(-1);
}

// R = [probes | aty | 0-pad] ; probes int8 D x K (host-drawn) or device-drawn
template <typename T>
__global__ void k_build_rhs(int64_t d_real, int64_t rows, int ldq, int K, const int8_t* probes, uint64_t dseed,
                            int iter, int64_t col_offset, const double* aty, T* R, int8_t* probe_store) {
  const int64_t n = rows * ldq;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / ldq;
    const int q = (int)(e % ldq);
    T v = T(0);
    if (j < d_real) {
      if (q < K) {
        int8_t p;
        if (probes) p = probes[j * K + q];
        else p = device_probe(dseed, iter, col_offset + j, q);
        probe_store[j * K + q] = p;
        v = T(p);
      } else if (q == K) {
        v = T(aty[j]);
      }
    }
    R[e] = v;
  }
}

// E-step read-out (cofem.py:98-100) fused with the M-step (cofem.py:103/:120)
// and the next preconditioner m = beta theta + alpha (cg.py:108).
template <typename T>
__global__ void k_em_finish(int64_t d_real, int ldq, int K, double beta, const T* X, const int8_t* probes, double* mu,
                            double* s, double* alpha, double* minv, const double* theta, int theta_policy, int do_update,
                            int variant, double floor_eps, double clamp_max) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < d_real; j += (int64_t)gridDim.x * blockDim.x) {
    const T* xr = X + j * ldq;
    const double m = beta * dd(xr[K]);
    double acc = 0.0;
    for (int k = 0; k < K; ++k) acc += (double)probes[j * K + k] * dd(xr[k]);
    const double sv = acc / (double)K;
    mu[j] = m;
    s[j] = sv;
    if (do_update) {
      double second;
      if (variant == 1) {
        // rectified second moment mu^2 + s + mu sqrt(s/pi) / erfcx(-xi)
        const double sf = fmax(sv, floor_eps);
        const double xi = m / sqrt(2.0 * sf);
        const double corr = m * sqrt(sf / 3.141592653589793) / erfcx(-xi);
        second = m * m + sf + corr;
      } else {
        second = m * m + sv;
      }
      const double a = fmin(1.0 / fmax(second, floor_eps), clamp_max);
      alpha[j] = a;
      const double th = theta_policy == 0 ? 1.0 : (theta_policy == 2 ? 0.0 : theta[j]);
      minv[j] = theta_policy == 2 ? 1.0 : 1.0 / (beta * th + a);
    }
  }
}

// minv = 1 / (beta theta + alpha) (or 1 for policy "none"); padded rows get 0
__global__ void k_make_minv(int64_t d_real, int64_t rows, double beta, const double* alpha, const double* theta,
                            int theta_policy, double* minv) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < rows; j += (int64_t)gridDim.x * blockDim.x) {
    if (j >= d_real) {
      minv[j] = 0.0;
      continue;
    }
    const double th = theta_policy == 0 ? 1.0 : (theta_policy == 2 ? 0.0 : theta[j]);
    minv[j] = theta_policy == 2 ? 1.0 : 1.0 / (beta * th + alpha[j]);
  }
}

// ---- dictionary utilities ---------------------------------------------------

__device__ __forceinline__ void philox_round(uint32_t& c0, uint32_t& c1, uint32_t& c2, uint32_t& c3, uint32_t k0,
                                             uint32_t k1) {
  const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
  const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
  const uint32_t h0 = (uint32_t)(p0 >> 32), l0 = (uint32_t)p0;
  const uint32_t h1 = (uint32_t)(p1 >> 32), l1 = (uint32_t)p1;
  const uint32_t n0 = h1 ^ c1 ^ k0, n2 = h0 ^ c3 ^ k1;
  c0 = n0; c1 = l1; c2 = n2; c3 = l0;
}

// Philox4x32-10 keyed by seed, counter = (row, global column pair index)
__device__ __forceinline__ void philox4(uint64_t seed, uint64_t ctr_hi, uint64_t ctr_lo, uint32_t out[4]) {
  uint32_t c0 = (uint32_t)ctr_lo, c1 = (uint32_t)(ctr_lo >> 32), c2 = (uint32_t)ctr_hi, c3 = (uint32_t)(ctr_hi >> 32);
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    philox_round(c0, c1, c2, c3, k0, k1);
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

// Phi[i][j] = scale * N(0,1); four normals per Philox call (Box-Muller)
__global__ void k_gen_gaussian(float* phi, int64_t ld, int64_t n_real, int64_t d_real, int64_t col_offset,
                               uint64_t seed, double scale) {
  const int64_t quads_per_row = (d_real + 3) / 4;
  const int64_t total = n_real * quads_per_row;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / quads_per_row, jq = e % quads_per_row;
    const int64_t jg = col_offset / 4 + jq;  // shards start at multiples of 4 columns
    uint32_t r[4];
    philox4(seed, (uint64_t)i, (uint64_t)jg, r);
    float z[4];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const double u1 = ((double)r[2 * h] + 1.0) * (1.0 / 4294967296.0);
      const double u2 = (double)r[2 * h + 1] * (1.0 / 4294967296.0);
      const double rad = sqrt(-2.0 * log(u1));
      double sn, cs;
      sincospi(2.0 * u2, &sn, &cs);
      z[2 * h] = (float)(scale * rad * cs);
      z[2 * h + 1] = (float)(scale * rad * sn);
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int64_t j = jq * 4 + c;
      if (j < d_real) phi[i * ld + j] = z[c];
    }
  }
}

// column squared norms in double (operators.py:128-129)
__global__ void k_colsq(const float* phi, int64_t ld, int64_t n_real, int64_t d_real, double* out) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= d_real) return;
  double s = 0.0;
  for (int64_t i = 0; i < n_real; ++i) {
    const double v = phi[i * ld + j];
    s += v * v;
  }
  out[j] = s;
}

}  // namespace cofem
