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
  double* gam[2];   // gamma = rho / pi of the step, by step parity (batched X updates)
  int* frozen;      // breakdown flags
  double* partials; // nblocks x 2 x ldq scratch
  unsigned* ticket; // last-block counters (one per reduction site)
  // Row sweep of k_combine and k_direction: descending when set.  For blocks larger than L2
  // (the 2-D DCT's 201 MB) the passes alternate direction -- row pass 3 writes Z ascending,
  // k_combine reads it descending, k_update reads Psi ascending (k_combine finished at the low
  // rows), k_direction reads R descending, the next row pass reads P ascending -- so every
  // kernel starts on the rows its producer wrote last (the part of them still in L2:
  // measured +0.6 % on dct-large, 39.4 -> 39.6 EM it/s; write-back instead of streaming
  // stores in the passes changes nothing).
  int rev_rows;
};

template <typename T>
__device__ __forceinline__ double dd(T v) { return (double)v; }

// Thread -> (row, column) map of the column-block kernels: blockDim is a
// multiple of ldq, thread t owns column q = t % ldq and visits rows
// j = blockIdx.x * rpb + t / ldq + k * gridDim.x * rpb (no index division
// inside the loop); consecutive threads touch consecutive elements.
constexpr int UNR = 4;  // rows per thread per loop trip: independent loads in flight

struct ColMap {
  int q, r0, rstep;
  __device__ __forceinline__ ColMap(int ldq) {
    const int rpb = blockDim.x / ldq;
    q = threadIdx.x % ldq;
    r0 = blockIdx.x * rpb + threadIdx.x / ldq;
    rstep = gridDim.x * rpb;
  }
};

// block-level fold of per-thread column sums into partials[blk][v][ldq]
__device__ __forceinline__ void block_col_reduce(double* sm, int ldq, int nvals, const double* vals,
                                                 double* partials_blk) {
  const int t = threadIdx.x, nt = blockDim.x;
  for (int v = 0; v < nvals; ++v) sm[v * nt + t] = vals[v];
  __syncthreads();
  for (int idx = t; idx < nvals * ldq; idx += nt) {
    const int v = idx / ldq, q = idx % ldq;
    double s = 0.0;
    for (int r = q; r < nt; r += ldq) s += sm[v * nt + r];
    partials_blk[v * ldq + q] = s;
  }
}

// Last-block reduction of partials[nblk][nvals*ldq] -> outs[v][q].  All
// threads of the last block take part: pair p = (v, q) is summed by `groups`
// threads over a fixed block stride, then folded in group order through smem
// -- deterministic, and the partial loads (__ldcg, L2) are independent.
__device__ __forceinline__ bool last_block_reduce(unsigned* ticket, const double* partials, int ldq, int nvals,
                                                  double* const* outs, double* sm) {
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
  const int npair = nvals * ldq;
  const int groups = blockDim.x >= npair ? blockDim.x / npair : 1;
  const int t = threadIdx.x;
  for (int p0 = 0; p0 < npair; p0 += blockDim.x) {
    double s = 0.0;
    const int p = p0 + t % npair;
    const int g = t / npair;
    if (g < groups && p < npair) {
      // 8 independent accumulators keep 8 L2 loads in flight per thread
      double a8[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      int b = g;
      const int nb = (int)gridDim.x;
      for (; b + 7 * groups < nb; b += 8 * groups) {
#pragma unroll
        for (int u = 0; u < 8; ++u) a8[u] += __ldcg(partials + (size_t)(b + u * groups) * npair + p);
      }
      for (int u = 0; b < nb; b += groups, ++u) a8[u] += __ldcg(partials + (size_t)b * npair + p);
      s = ((a8[0] + a8[1]) + (a8[2] + a8[3])) + ((a8[4] + a8[5]) + (a8[6] + a8[7]));
    }
    __syncthreads();
    sm[t] = s;
    __syncthreads();
    if (t < npair && p0 + t < npair) {
      double tot = 0.0;
      for (int gg = 0; gg < groups; ++gg) tot += sm[gg * npair + t];
      const int pp = p0 + t;
      outs[pp / ldq][pp % ldq] = tot;
    }
    if (groups > 1) break;  // all pairs handled in one sweep
  }
  if (threadIdx.x == 0) *ticket = 0u;
  return true;
}

// per-block column max of non-negative values (or NaN) -> atomicMax on the
// bit patterns (order independent, so deterministic)
__device__ __forceinline__ void block_col_max(double* sm, int ldq, double v, unsigned long long* colmax) {
  const int t = threadIdx.x, nt = blockDim.x;
  __syncthreads();
  sm[t] = v;
  __syncthreads();
  if (t < ldq) {
    double m = 0.0;
    for (int r = t; r < nt; r += ldq) {
      const double x = sm[r];
      m = (x > m || x != x) ? x : m;
    }
    atomicMax(&colmax[t], (unsigned long long)__double_as_longlong(m));
  }
}

__device__ __forceinline__ double safe_ratio(double num, double den) { return den != 0.0 ? num / den : 0.0; }

// ---- init: X = 0, P = 0, bn2 = ||R||^2, rho_new = <R, M^-1 R> (R already holds B)
template <typename T>
__global__ void k_pcg_init(int64_t rows, int ldq, int q_real, T* X, T* P, const T* R, const double* minv, int ngroups,
                           const int* group_of_col, Scalars sc) {
  extern __shared__ double sm_init[];
  const ColMap m(ldq);
  const int g = group_of_col ? group_of_col[m.q] : 0;
  double s_bn = 0.0, s_rho = 0.0;
  for (int64_t j = m.r0; j < rows; j += m.rstep) {
    const int64_t e = j * ldq + m.q;
    X[e] = T(0);
    P[e] = T(0);
    const double r = dd(R[e]);
    const double w = (m.q < q_real) ? r * minv[j * ngroups + g] : 0.0;
    s_bn += r * r;
    s_rho += r * w;
  }
  double vals[2] = {s_bn, s_rho};
  block_col_reduce(sm_init, ldq, 2, vals, sc.partials + (int64_t)blockIdx.x * 2 * ldq);
  double* outs[2] = {sc.bn2, sc.rho_new};
  last_block_reduce(sc.ticket + 0, sc.partials, ldq, 2, outs, sm_init);
}

// ---- combine: Psi = beta * sum_s Psipart[s] + alpha .* P ; pi_q = <P_q, Psi_q>
// (chunk of QPc columns at column offset qoff; partial buffer is dense QPc)
template <typename T>
__global__ void k_combine(int64_t rows, int ldq, int qoff, int qpc, int nsplit, const T* ppart, double beta,
                          const double* alpha, const T* P, T* Psi, Scalars sc, const Status* st) {
  if (st && st->done) return;
  extern __shared__ double sm_comb[];
  const ColMap m(qpc);
  const int64_t n = rows * qpc;
  double s_pi = 0.0;
  for (int64_t j0 = m.r0; j0 < rows; j0 += UNR * (int64_t)m.rstep) {
    T acc[UNR], p[UNR];
    double al[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {  // issue every load of UNR rows first
      const int64_t ja = j0 + (int64_t)u * m.rstep, j = sc.rev_rows ? rows - 1 - ja : ja;
      if (ja < rows) {
        const int64_t e = j * qpc + m.q;
        acc[u] = ppart[e];
        for (int s = 1; s < nsplit; ++s) acc[u] += ppart[(int64_t)s * n + e];
        p[u] = P[j * ldq + qoff + m.q];
        al[u] = alpha[j];
      }
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int64_t ja = j0 + (int64_t)u * m.rstep, j = sc.rev_rows ? rows - 1 - ja : ja;
      if (ja < rows) {
        const T psi = T(beta) * acc[u] + T(al[u]) * p[u];
        Psi[j * ldq + qoff + m.q] = psi;
        s_pi += dd(p[u]) * dd(psi);
      }
    }
  }
  block_col_reduce(sm_comb, qpc, 1, &s_pi, sc.partials + (int64_t)blockIdx.x * qpc);
  double* outs[1] = {sc.pi + qoff};
  last_block_reduce(sc.ticket + 1, sc.partials, qpc, 1, outs, sm_comb);
}

// ---- V = sum_s Vpart[s] (dense rows x qw).  With `colmax` set, also the
// per-column max of |pre_i V_iq| that the next quantisation needs.
template <typename T>
__global__ void k_sum_splits(int64_t rows, int qw, int nsplit, const T* part, T* out, const double* pre,
                             unsigned long long* colmax, const Status* st) {
  if (st && st->done) return;
  extern __shared__ double sm_sum[];
  const ColMap m(qw);
  const int64_t n = rows * qw;
  double vmax = 0.0;
  for (int64_t j = m.r0; j < rows; j += m.rstep) {
    const int64_t e = j * qw + m.q;
    T acc = part[e];
    for (int s = 1; s < nsplit; ++s) acc += part[(int64_t)s * n + e];
    out[e] = acc;
    if (colmax) {
      const double v = fabs(dd(acc) * pre[j]);
      vmax = (v > vmax || v != v) ? v : vmax;
    }
  }
  if (colmax) block_col_max(sm_sum, qw, vmax, colmax);
}

// ---- residual update (kernels.py step_solution) fused with the residual
// norms and the next direction's rho:  gamma = rho/pi (0 when pi == 0),
// R -= Psi gamma, rn2 = ||R||^2, rho_new = <R, M^-1 R>.  With X == nullptr
// the solution update X += P gamma is left to k_direction, which reads P
// anyway (one D x ldq block less per step); otherwise it is done here.
template <typename T>
__global__ void k_update(int64_t rows, int ldq, int q_real, int parity, T* X, T* R, const T* P, const T* Psi,
                         const double* minv, int ngroups, const int* group_of_col, Scalars sc,
                         unsigned long long* colmax_reset, const Status* st) {
  if (st && st->done) return;
  extern __shared__ double sm_upd[];
  const ColMap m(ldq);
  const int q = m.q;
  const int g = group_of_col ? group_of_col[q] : 0;
  const double pi = sc.pi[q];
  const double gamma = safe_ratio(sc.rho[parity][q], pi);
  if (blockIdx.x == 0 && threadIdx.x < ldq) {
    if (q < q_real && pi == 0.0) sc.frozen[q] = 1;
    if (colmax_reset) colmax_reset[threadIdx.x] = 0ull;  // consumed by k_direction below
    sc.gam[parity][q] = gamma;                           // k_direction's (batched) X update
  }
  const T gm = T(gamma);
  double s_rn = 0.0, s_rho = 0.0;
  for (int64_t j0 = m.r0; j0 < rows; j0 += UNR * (int64_t)m.rstep) {
    T x[UNR], p[UNR], r[UNR], ps[UNR];
    double mv[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int64_t j = j0 + (int64_t)u * m.rstep;
      if (j < rows) {
        const int64_t e = j * ldq + q;
        if (X) {
          x[u] = X[e];
          p[u] = P[e];
        }
        r[u] = R[e];
        ps[u] = Psi[e];
        mv[u] = minv[j * ngroups + g];
      }
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int64_t j = j0 + (int64_t)u * m.rstep;
      if (j < rows) {
        const int64_t e = j * ldq + q;
        if (X) X[e] = x[u] + p[u] * gm;
        const T rn = r[u] - ps[u] * gm;
        R[e] = rn;
        const double rd = dd(rn);
        s_rn += rd * rd;
        if (q < q_real) s_rho += rd * (rd * mv[u]);
      }
    }
  }
  double vals[2] = {s_rho, s_rn};
  block_col_reduce(sm_upd, ldq, 2, vals, sc.partials + (int64_t)blockIdx.x * 2 * ldq);
  double* outs[2] = {sc.rho_new, sc.rn2};
  last_block_reduce(sc.ticket + 2, sc.partials, ldq, 2, outs, sm_upd);
}

// ---- the Psi-free residual update of dictionaries with orthonormal rows (the 2-D DCT).
// pi = beta vv + pap with vv = ||Phi^T Phi P||^2 = ||Phi P||^2 (per-block sums of Z^2 from the
// last FFT pass, folded here in block order by every block: no serial fold at the pass's end) and
// pap = <P, alpha P>, carried by the direction recurrence P(u+1) = eta P(u) + W(u):
//   pap(u+1) = eta^2 pap(u) + 2 eta <P(u), alpha W(u)> + <W(u), alpha W(u)>
// whose two inner products this kernel returns (it holds P, the new R and alpha anyway; W =
// M^-1 R, or R for the printed recursion), so the direction kernel is unchanged.  Then
// gamma = rho / pi and, in ONE pass over Z, P and R:  R -= gamma (beta Z + alpha .* P), rn2,
// rho_new -- what k_combine (Psi, pi) and k_update do in two passes and a D x ldq round trip.
// State `ps` (per column, stride PSQ): pap by step parity [0], [1]; s1 [2]; s2 [3].
constexpr int PSQ = 32;
template <typename T>
__global__ void k_update_psi(int64_t rows, int ldq, int q_real, int step, int printed, T* R, const T* P, const T* Z,
                             double beta, const double* alpha, const double* minv, int ngroups,
                             const int* group_of_col, const double* vv_partials, int vv_blocks, double* ps,
                             double* partials4, Scalars sc, const Status* st) {
  if (st && st->done) return;
  extern __shared__ double sm_upd[];
  const ColMap m(ldq);
  const int q = m.q, parity = step & 1;
  const int g = group_of_col ? group_of_col[q] : 0;
  // vv_q: the pass's block partials, thread-row rs sums blocks rs, rs + rpb, ..., then the rows in order
  {
    const int rpb = blockDim.x / ldq, rs = threadIdx.x / ldq;
    double a8[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // 8 independent L2 loads in flight
    int b2 = rs;
    for (; b2 + 7 * rpb < vv_blocks; b2 += 8 * rpb) {
#pragma unroll
      for (int u = 0; u < 8; ++u) a8[u] += __ldcg(vv_partials + (int64_t)(b2 + u * rpb) * ldq + q);
    }
    for (int u = 0; b2 < vv_blocks; b2 += rpb, ++u) a8[u] += __ldcg(vv_partials + (int64_t)b2 * ldq + q);
    sm_upd[threadIdx.x] = ((a8[0] + a8[1]) + (a8[2] + a8[3])) + ((a8[4] + a8[5]) + (a8[6] + a8[7]));
    __syncthreads();
    double v = 0.0;
    for (int r2 = 0; r2 < rpb; ++r2) v += sm_upd[r2 * ldq + q];
    __syncthreads();
    sm_upd[threadIdx.x] = v;  // every thread of column q holds vv_q
  }
  const double vvq = sm_upd[threadIdx.x];
  __syncthreads();
  // eta of the previous direction step: rho(u) / rho(u-1), both still in the parity buffers
  const double eta = safe_ratio(sc.rho[parity][q], sc.rho[parity ^ 1][q]);
  const double pap = step == 1 ? ps[3 * PSQ + q] : (eta * eta) * ps[(parity ^ 1) * PSQ + q] + (2.0 * eta) * ps[2 * PSQ + q] + ps[3 * PSQ + q];
  const double pi = beta * vvq + pap;
  const double gamma = safe_ratio(sc.rho[parity][q], pi);
  if (blockIdx.x == 0 && threadIdx.x < ldq) {
    if (q < q_real && pi == 0.0) sc.frozen[q] = 1;
    sc.pi[q] = pi;
    sc.gam[parity][q] = gamma;  // k_direction's (batched) X update
    ps[parity * PSQ + q] = pap;
  }
  const T gm = T(gamma);
  double s_rn = 0.0, s_rho = 0.0, s1 = 0.0, s2 = 0.0;
  for (int64_t j0 = m.r0; j0 < rows; j0 += UNR * (int64_t)m.rstep) {
    T p[UNR], r[UNR], z[UNR];
    double mv[UNR], al[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int64_t ja = j0 + (int64_t)u * m.rstep, j = sc.rev_rows ? rows - 1 - ja : ja;
      if (ja < rows) {
        const int64_t e = j * ldq + q;
        p[u] = P[e];
        r[u] = R[e];
        z[u] = Z[e];
        al[u] = alpha[j];
        mv[u] = minv[j * ngroups + g];
      }
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int64_t ja = j0 + (int64_t)u * m.rstep, j = sc.rev_rows ? rows - 1 - ja : ja;
      if (ja < rows) {
        const T psi = T(beta) * z[u] + T(al[u]) * p[u];
        const T rn = r[u] - psi * gm;
        R[j * ldq + q] = rn;
        const double rd = dd(rn);
        s_rn += rd * rd;
        const double w = q < q_real ? rd * mv[u] : 0.0;
        s_rho += rd * w;
        const double wd = printed ? rd : w, aw = al[u] * wd;
        s1 += dd(p[u]) * aw;
        s2 += wd * aw;
      }
    }
  }
  double vals[4] = {s_rho, s_rn, s1, s2};
  block_col_reduce(sm_upd, ldq, 4, vals, partials4 + (int64_t)blockIdx.x * 4 * ldq);
  double* outs[4] = {sc.rho_new, sc.rn2, ps + 2 * PSQ, ps + 3 * PSQ};
  last_block_reduce(sc.ticket + 2, partials4, ldq, 4, outs, sm_upd);
}

// start of a Psi-free solve: s2 = <W, alpha W> of W = M^-1 B (B for the printed recursion), the
// first direction; pap(0) = s1 = 0
template <typename T>
__global__ void k_pap_init(int64_t rows, int ldq, int q_real, int printed, const T* R, const double* alpha,
                           const double* minv, int ngroups, const int* group_of_col, double* ps, double* partials4,
                           Scalars sc) {
  extern __shared__ double sm_upd[];
  const ColMap m(ldq);
  const int q = m.q;
  const int g = group_of_col ? group_of_col[q] : 0;
  double s2 = 0.0;
  for (int64_t j = m.r0; j < rows; j += m.rstep) {
    const double rd = dd(R[j * ldq + q]);
    const double wd = printed ? rd : (q < q_real ? rd * minv[j * ngroups + g] : 0.0);
    s2 += wd * (alpha[j] * wd);
  }
  if (blockIdx.x == 0 && threadIdx.x < ldq) ps[q] = ps[PSQ + q] = ps[2 * PSQ + q] = 0.0;
  block_col_reduce(sm_upd, ldq, 1, &s2, partials4 + (int64_t)blockIdx.x * ldq);
  double* outs[1] = {ps + 3 * PSQ};
  last_block_reduce(sc.ticket + 5, partials4, ldq, 1, outs, sm_upd);
}

// ---- convergence test (cg.py:141-148) + direction update (kernels.py
// step_direction): eta = rho_new / rho (0 when rho == 0), P = P eta + W
// (or R for the printed recursion), rho <- rho_new.  step == 0 is the
// initialisation pass (no convergence test).  With `colmax` set, also the
// per-column max of |pre_j P_jq| for the next Phi P quantisation.
// With X set (step >= 1) the kernel also applies the solution updates
// X += P(u) gamma_u (gamma_u = rho/pi as k_update stored it), in pairs: an odd
// step defers its update, the next (even) step applies both,
//   X = (X + P(u-1) gamma_{u-1}) + P(u) gamma_u
// (the order of the one-step-at-a-time recursion, so the bits are the same)
// with P(u-1) still intact in Pprev -- one read-modify-write of X per two
// steps.  The stopping step applies whatever is pending.  P(u+1) goes to
// Pdst (nullptr: in place); the host swaps the two direction buffers, so at
// an even step Pdst == Pprev (each element read before it is overwritten).
template <typename T>
__global__ void k_direction(int64_t rows, int ldq, int q_real, int step, int max_steps, double tol, int printed,
                            T* P, const T* R, const double* minv, int ngroups, const int* group_of_col, Scalars sc,
                            const double* pre, unsigned long long* colmax, Status* st,
                            const double* agg = nullptr, Status* mirror = nullptr, T* X = nullptr,
                            T* Pdst = nullptr, const T* Pprev = nullptr) {
  // agg (multi-task solves): {sum ||R||^2, sum ||B||^2} over every task's columns
  // mirror: host-mapped status slot the host polls (no copy in the stream)
  {
    // a solve finished by an EARLIER step: nothing to do.  (Block 0 of this
    // very launch may already have set `done` for this step -- then the X
    // update below must still run: steps is published before done.)
    const volatile Status* vs = st;
    const int done = vs->done;
    __threadfence();
    const int sdone = vs->steps;
    if (done && !(X && step >= 1 && sdone == step)) {
      if (mirror && blockIdx.x == 0 && threadIdx.x == 0) {
        *mirror = *st;
        __threadfence_system();
      }
      return;
    }
  }
  extern __shared__ double sm_dir[];
  const int cur = step & 1, nxt = (step + 1) & 1;
  if (step == 0) {
    double b2 = 0.0;
    for (int c = 0; c < ldq; ++c) b2 += sc.bn2[c];
    if (agg) b2 = agg[1];
    if (blockIdx.x == 0 && threadIdx.x == 0) st->bnorm = sqrt(b2);
  } else {
    double r2 = 0.0;
    for (int c = 0; c < ldq; ++c) r2 += sc.rn2[c];
    double b2 = 0.0;
    for (int c = 0; c < ldq; ++c) b2 += sc.bn2[c];
    if (agg) {
      r2 = agg[0];
      b2 = agg[1];
    }
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
    if (stop) {
      if (X) {  // the pending solution updates
        const ColMap m(ldq);
        const T gm = T(sc.gam[cur][m.q]);
        const bool pair = (step & 1) == 0 && Pprev;
        const T gp = pair ? T(sc.gam[nxt][m.q]) : T(0);
        for (int64_t j = m.r0; j < rows; j += m.rstep) {
          const int64_t e = j * ldq + m.q;
          T x = X[e];
          if (pair) x = x + Pprev[e] * gp;
          X[e] = x + P[e] * gm;
        }
      }
      return;
    }
  }
  if (!Pdst) Pdst = P;
  const ColMap m(ldq);
  const int q = m.q;
  const int g = group_of_col ? group_of_col[q] : 0;
  const double eta = safe_ratio(sc.rho_new[q], sc.rho[cur][q]);
  const T et = T(eta);
  // X updates: every step without Pprev (one-step mode), even steps in pairs
  const bool upd_x = X && step >= 1 && (!Pprev || (step & 1) == 0);
  const bool pair = upd_x && Pprev;
  const T gm = upd_x ? T(sc.gam[cur][q]) : T(0);
  const T gp = pair ? T(sc.gam[nxt][q]) : T(0);
  double pmax = 0.0;
  for (int64_t j0 = m.r0; j0 < rows; j0 += UNR * (int64_t)m.rstep) {
    T r[UNR], p[UNR], x[UNR], pp[UNR];
    double mv[UNR], pr[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int64_t ja = j0 + (int64_t)u * m.rstep, j = sc.rev_rows ? rows - 1 - ja : ja;
      if (ja < rows) {
        const int64_t e = j * ldq + q;
        r[u] = R[e];
        p[u] = P[e];
        if (upd_x) x[u] = X[e];
        if (pair) pp[u] = Pprev[e];
        mv[u] = minv[j * ngroups + g];
        pr[u] = colmax ? pre[j] : 0.0;
      }
    }
    if (upd_x) {
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const int64_t ja = j0 + (int64_t)u * m.rstep, j = sc.rev_rows ? rows - 1 - ja : ja;
        if (ja < rows) X[j * ldq + q] = (pair ? x[u] + pp[u] * gp : x[u]) + p[u] * gm;
      }
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int64_t ja = j0 + (int64_t)u * m.rstep, j = sc.rev_rows ? rows - 1 - ja : ja;
      if (ja < rows) {
        const T w = (q < q_real) ? T(dd(r[u]) * mv[u]) : T(0);
        const T pn = p[u] * et + (printed ? r[u] : w);
        Pdst[j * ldq + q] = pn;
        if (colmax) {
          const double v = fabs(dd(pn) * pr[u]);
          pmax = (v > pmax || v != v) ? v : pmax;
        }
      }
    }
  }
  if (blockIdx.x == 0 && threadIdx.x < ldq) sc.rho[nxt][threadIdx.x] = sc.rho_new[threadIdx.x];
  if (colmax) block_col_max(sm_dir, ldq, pmax, colmax);
}

// ---- multi-task glue (cofem.py:160-214) -------------------------------------
// agg = {sum_l sum_q rn2_l[q], sum_l sum_q bn2_l[q]} in task order
__global__ void k_sum_tasks(int L, int ldq, const double* const* rn2, const double* const* bn2, double* agg) {
  // one sequential pass over the concatenated columns, like the single-task
  // reduction in k_direction (so L = 1 reproduces run_cofem bit for bit)
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  double r = 0.0, b = 0.0;
  for (int l = 0; l < L; ++l)
    for (int q = 0; q < ldq; ++q) {
      r += rn2[l][q];
      b += bn2[l][q];
    }
  agg[0] = r;
  agg[1] = b;
}

// shared precision update: alpha = min(L / max(sum_l (mu_l^2 + s_l), floor), clamp),
// written into every task together with its next M^-1 (task beta_l)
__global__ void k_multitask_alpha(int64_t d_real, int L, const double* betas, const double* const* mu,
                                  const double* const* s, double* const* alpha, double* const* minv,
                                  const double* const* theta, int theta_policy, double floor_eps, double clamp_max) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < d_real; j += (int64_t)gridDim.x * blockDim.x) {
    double tot = 0.0;
    for (int l = 0; l < L; ++l) tot = tot + (mu[l][j] * mu[l][j] + s[l][j]);
    const double a = fmin((double)L / fmax(tot, floor_eps), clamp_max);
    for (int l = 0; l < L; ++l) {
      alpha[l][j] = a;
      const double th = theta_policy == 0 ? 1.0 : (theta_policy == 2 ? 0.0 : theta[l][j]);
      minv[l][j] = theta_policy == 2 ? 1.0 : 1.0 / (betas[l] * th + a);
    }
  }
}

// ---- EM glue ---------------------------------------------------------------

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// ---- the reference's probe stream on the device ------------------------------
// numpy's Generator(PCG64).integers(0, 2, size=(D, K)) (probes.py:13-17, the
// reference's draw_rademacher) takes, for element e of the row-major D x K
// draw, the top bit of the next 32-bit value of the generator -- Lemire's
// bounded draw for a range of 2 never rejects -- and the generator hands out
// 32-bit values as the low then the high half of each raw PCG64 output,
// buffering an unused high half across calls.  So the probes of all draws
// form one stream of 32-bit halves u_0, u_1, ... (u_{2r} = low(raw_r),
// u_{2r+1} = high(raw_r)) and EM iteration t uses u_{t D K + e}.  PCG64 is a
// 128-bit LCG (state = state M + inc, then output the new state) with the
// XSL-RR output; threads jump ahead in O(log n).
typedef unsigned __int128 u128;
constexpr uint64_t PCG_MULT_HI = 0x2360ED051FC65DA4ull, PCG_MULT_LO = 0x4385DF649FCCF645ull;

__host__ __device__ __forceinline__ uint64_t pcg64_output(u128 s) {
  const uint64_t x = (uint64_t)(s >> 64) ^ (uint64_t)s;
  const unsigned rot = (unsigned)(s >> 122);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}
// state after `delta` LCG steps
__host__ __device__ __forceinline__ u128 pcg64_advance(u128 s, u128 inc, uint64_t delta) {
  u128 cur_mult = ((u128)PCG_MULT_HI << 64) | PCG_MULT_LO, cur_plus = inc;
  u128 acc_mult = 1, acc_plus = 0;
  while (delta) {
    if (delta & 1) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  return acc_mult * s + acc_plus;
}

// rows [row0, row0 + rows) of the row-major D x K sign matrix whose element 0
// is 32-bit half `half_base` of the stream that starts at state (hi, lo).
// Each thread produces the elements of 32 consecutive raw outputs.
__global__ void k_pcg64_rademacher(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                                   uint64_t half_base, int64_t row0, int64_t rows, int K, int8_t* __restrict__ out) {
  constexpr int RCH = 32;
  const u128 s0 = ((u128)state_hi << 64) | state_lo, inc = ((u128)inc_hi << 64) | inc_lo;
  const u128 mult = ((u128)PCG_MULT_HI << 64) | PCG_MULT_LO;
  const uint64_t h_begin = half_base + (uint64_t)(row0 * K), h_end = h_begin + (uint64_t)(rows * K);
  const uint64_t r_begin = h_begin >> 1, r_end = (h_end + 1) >> 1;
  const int64_t nchunk = (int64_t)((r_end - r_begin + RCH - 1) / RCH);
  for (int64_t ch = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; ch < nchunk; ch += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t r0 = r_begin + (uint64_t)ch * RCH;
    u128 st = pcg64_advance(s0, inc, r0);  // state before raw output r0
#pragma unroll 4
    for (int i = 0; i < RCH; ++i) {
      st = st * mult + inc;
      const uint64_t v = pcg64_output(st);
      const uint64_t h = 2 * (r0 + i);
      if (h >= h_begin && h < h_end) out[h - h_begin] = ((v >> 31) & 1) ? int8_t(1) : int8_t(-1);
      if (h + 1 >= h_begin && h + 1 < h_end) out[h + 1 - h_begin] = ((v >> 63) & 1) ? int8_t(1) : int8_t(-1);
    }
  }
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
template <typename PT>
__global__ void k_colsq(const PT* phi, int64_t ld, int64_t n_real, int64_t d_real, double* out) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= d_real) return;
  double s = 0.0;
  for (int64_t i = 0; i < n_real; ++i) {
    const double v = phi[i * ld + j];
    s += v * v;
  }
  out[j] = s;
}

// ---- Phi^T y staging: y (n doubles) -> column 0 of an (rows x ld) block
// (other columns and the padding rows zero), and column 0 back out
template <typename T>
__global__ void k_put_col0(const double* __restrict__ y, int64_t n, int64_t rows, int ld, T* __restrict__ V) {
  const int64_t total = rows * ld;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / ld;
    V[e] = (e % ld == 0 && i < n) ? T(y[i]) : T(0);
  }
}
template <typename T>
__global__ void k_get_col0(const T* __restrict__ src, int64_t n, int64_t rows, int ld, double* __restrict__ dst) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = i < n ? (double)src[i * ld] : 0.0;
}

// ---- in-process shard group (cofem_group): element-wise reduction over the
// ranks' buffers, in rank order so every rank gets the same bits.  op 0 sum,
// 1 max (used on non-negative doubles' bit patterns as uint64).
constexpr int GROUP_MAX = 8;
struct GroupPtrs {
  const void* p[GROUP_MAX];
};
template <typename T>
__global__ void k_group_reduce(GroupPtrs src, int n, int64_t count, int op, T* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    T a = ((const T*)src.p[0])[i];
    for (int r = 1; r < n; ++r) {
      const T b = ((const T*)src.p[r])[i];
      a = op ? (b > a ? b : a) : a + b;
    }
    out[i] = a;
  }
}

}  // namespace cofem
