// CholeskyQR factor as an explicit triangular T (Y T has orthonormal columns),
// one CTA of 1024 threads, one block barrier per column.
//
// Right-looking elimination of the equilibrated Gram S = D G D (D = diag(dsc),
// dsc_i = G_ii^{-1/2}) with the inverse of the unit lower factor accumulated
// alongside: for pivot k, every entry with row a > k is updated
//   S_ab -= (S_ka / S_kk) S_kb      (a, b > k: Schur complement, kept symmetric)
//   W_ab -= (S_ka / S_kk) W_kb      (b <= k < a, W_kk = 1: W = L^{-1})
// so that S = L diag(d) L^T, R = diag(d)^{1/2} L^T and
//   T = D R^{-1} = D W^T diag(d)^{-1/2}
// without a separate triangular inversion. Row k is only read during step k
// and rows > k are only written, so one barrier per pivot suffices.
//
// Column drop (the rank reveal of QR-CP, reading R4): a
// pivot whose equilibrated Schur diagonal is <= tol (relative to the column's
// own squared norm) eliminates nothing and gets a zero column in T; the other
// columns of T then have zero coefficients on it (W_ic = 0 for dropped c).
//
// Range propagation (reading R11): with r = *r_dev > 0
// the input is Y = [Q~ | Y_p], Q~ (r columns) orthonormal. Its Gram block is
// taken as I, so R12 = G12 = Q~^T Y_p and only the Schur complement
//   S22 = G22 - G12^T G12   (p = l - r, the fresh columns)
// is factored, equilibrated by the fresh columns' own norms (so the drop test
// is relative to |y_j|, as in the full factorisation). The output is the
// l x p apply matrix Tp = [-G12 T22 ; T22] (columns p..l-1 zero):
// Y Tp = (Y_p - Q~ G12) T22 spans the fresh directions (classical Gram-Schmidt
// against Q~ followed by CholeskyQR, P:179 with reading R11); the caller keeps
// Q~ as the first r columns.
#pragma once
#include "common.cuh"

namespace frsvt {

constexpr int CI_THREADS = 1024;
constexpr int CI_LD = FRSVT_LMAX;  // row stride (doubles) of the p x p work matrix

__host__ __device__ constexpr size_t chol_inv_smem_bytes() {
  // M (LMAX x CI_LD) + G12 (<= (LMAX/2)^2 when r, p > 0) + dsc + sd + 32 pivot rows + 32 pivot
  // inverses + LMAX row barriers
  return ((size_t)FRSVT_LMAX * CI_LD + (size_t)(FRSVT_LMAX / 2) * (FRSVT_LMAX / 2) + 2 * FRSVT_LMAX +
          32 * (size_t)FRSVT_LMAX + 32 + FRSVT_LMAX) *
         sizeof(double);
}

__device__ __forceinline__ void ci_bar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)) : "memory");
}
__device__ __forceinline__ void ci_bar_arrive(uint64_t* bar) {
  asm volatile("{\n.reg .b64 st;\nmbarrier.arrive.release.cta.shared.b64 st, [%0];\n}" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(bar))
               : "memory");
}
__device__ __forceinline__ void ci_bar_wait0(uint64_t* bar) {  // phase 0 completion (each barrier is used once)
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.test_wait.parity.acquire.cta.shared::cta.b64 p, [%1], 0;\nselp.b32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(a)
        : "memory");
  } while (!ok);
}
// 1 / d for d in (tol, ~1]: fp32 reciprocal + two Newton steps (~1 ulp)
__device__ __forceinline__ double ci_rcp(double d) {
  double r = (double)__frcp_rn((float)d);
  r = fma(r, fma(-d, r, 1.0), r);
  r = fma(r, fma(-d, r, 1.0), r);
  return r;
}

// Storage during the elimination (before step k), M = the p x p work matrix:
//   a, b >= k          : the current Schur complement, both triangles (symmetric)
//   a > b, b < k       : W_ab
//   a < b, a < k       : row a of the Schur complement at its own step (R up to scaling)
// Step k touches only rows a > k, all with one formula (u_a = S_ka / S_kk):
//   M_ab -= u_a M_kb   (b != k: Schur update for b > k, W update for b < k)
//   M_ak  = -u_a       (W_ak; written as M_ak - u_a (S_kk + 1), since M_ak = S_ak = S_ka)
// Thread (warp w, lane L) keeps the 4 x 4 entries (w + 32 i, L + 32 j) in
// registers. Step k needs only row k, so there is no block barrier: the owner
// warp of row k + 1 updates that row first in step k, publishes it (and
// 1 / S_{k+1,k+1}) to ring slot (k + 1) mod 32 and arrives on the row's
// one-shot mbarrier; every warp waits on row k's barrier before step k. A
// slot is rewritten 32 rows later by the same warp, which by then waited on
// rows published by all 31 other warps after their step k: no reader of row k
// is left.
template <typename Tq>
__global__ void __launch_bounds__(CI_THREADS, 1)
chol_inv_kernel(const double* __restrict__ G, int l, const int* __restrict__ r_dev, double tol, Tq* __restrict__ T,
                int64_t ldt, int* __restrict__ s_out, int* __restrict__ flags, const int* __restrict__ skip,
                unsigned long long* __restrict__ prof = nullptr) {
  if (skip && *skip) return;
  // prof (test hook, nullable): %globaltimer at phase boundaries
#define CI_STAMP(q)                                          \
  do {                                                       \
    if (prof && threadIdx.x == 0) {                          \
      unsigned long long t_;                                 \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); \
      prof[q] = t_;                                          \
    }                                                        \
  } while (0)
  CI_STAMP(0);
  extern __shared__ double cis[];
  double* M = cis;                               // p x p (row stride CI_LD)
  double* X = M + (size_t)FRSVT_LMAX * CI_LD;    // G12, r x p row-major (X[c * p + i])
  double* dsc = X + (FRSVT_LMAX / 2) * (FRSVT_LMAX / 2);
  double* sd = dsc + FRSVT_LMAX;
  double* rowbuf = sd + FRSVT_LMAX;              // 32 x LMAX ring of pivot rows
  double* invbuf = rowbuf + 32 * FRSVT_LMAX;     // 32 pivot inverses
  uint64_t* rbar = reinterpret_cast<uint64_t*>(invbuf + 32);  // LMAX one-shot row barriers
  const int tid = threadIdx.x, w = tid >> 5, L = tid & 31;
  const int r = r_dev ? min(max(*r_dev, 0), l) : 0;
  const int p = l - r;

  // (1) fresh columns' norms, G12
  for (int i = tid; i < p; i += CI_THREADS) {
    const double g = G[(size_t)(r + i) * (l + 1)];
    if (!isfinite(g)) atomicOr(flags, FLAG_NONFINITE);
    dsc[i] = (g > 0.0 && isfinite(g)) ? 1.0 / sqrt(g) : 0.0;
  }
  for (int idx = tid; idx < r * p; idx += CI_THREADS) {
    const int c = idx % r, i = idx / r;
    X[c * p + i] = G[c + (size_t)(r + i) * l];
  }
  __syncthreads();
  CI_STAMP(1);
  // (2) equilibrated Schur complement, both triangles
  for (int idx = tid; idx < p * p; idx += CI_THREADS) {
    const int i = idx / p, j = idx - i * p;
    if (j >= i) {
      double s = G[(r + j) + (size_t)(r + i) * l];  // G symmetric: coalesced along j
      for (int c = 0; c < r; ++c) s = fma(-X[c * p + i], X[c * p + j], s);
      double v = s * dsc[i] * dsc[j];
      if (!isfinite(v)) v = 0.0;
      M[i * CI_LD + j] = v;
      M[j * CI_LD + i] = v;
    }
  }
  __syncthreads();
  double m[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int a = w + 32 * i, b = L + 32 * j;
      m[i][j] = (a < p && b < p) ? M[a * CI_LD + b] : 0.0;
    }
  for (int i = tid; i < FRSVT_LMAX; i += CI_THREADS) ci_bar_init(&rbar[i]);
  __syncthreads();
  if (w == 0 && p > 0) {  // row 0
#pragma unroll
    for (int j = 0; j < 4; ++j) rowbuf[L + 32 * j] = m[0][j];
    if (L == 0) invbuf[0] = m[0][0] > tol ? ci_rcp(m[0][0]) : 0.0;
    __syncwarp();
    if (L == 0) ci_bar_arrive(&rbar[0]);
  }

  CI_STAMP(2);
  // (3) elimination
  for (int k = 0; k < p; ++k) {
    ci_bar_wait0(&rbar[k]);
    const double* rk = rowbuf + (k & 31) * FRSVT_LMAX;
    const double inv = invbuf[k & 31];
    const double d = rk[k];
    double v[4], u[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int b = L + 32 * j;
      v[j] = (b == k) ? d + 1.0 : rk[b];
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int a = w + 32 * i;
      u[i] = (a > k && a < p) ? rk[a] * inv : 0.0;
    }
    const int k1 = k + 1;
    const bool owner = k1 < p && w == (k1 & 31);
    const int i1 = k1 >> 5;
    // row i is updated when active; the owner's row k + 1 first, then published
#pragma unroll
    for (int pass = 0; pass < 2; ++pass) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int a = w + 32 * i;
        const bool first = owner && i == i1;
        if (a > k && a < p && (pass == 0) == first) {
          if (inv != 0.0) {
#pragma unroll
            for (int j = 0; j < 4; ++j) m[i][j] = fma(-u[i], v[j], m[i][j]);
          } else {  // dropped pivot: no elimination, W_ak = 0
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (L + 32 * j == k) m[i][j] = 0.0;
          }
        }
        if (pass == 0 && first) {
          double* rn = rowbuf + (k1 & 31) * FRSVT_LMAX;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            rn[L + 32 * j] = m[i][j];
            if (j == i1 && L == (k1 & 31)) invbuf[k1 & 31] = m[i][j] > tol ? ci_rcp(m[i][j]) : 0.0;
          }
          __syncwarp();
          if (L == 0) ci_bar_arrive(&rbar[k1]);
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int a = w + 32 * i, b = L + 32 * j;
      if (a < p && b < p) M[a * CI_LD + b] = m[i][j];
    }
  __syncthreads();
  CI_STAMP(3);
  // (4) T22 (upper, in place of S): T22[c][i] = dsc_c W_ic / sqrt(d_i), kept i
  for (int i = tid; i < p; i += CI_THREADS) {
    const double d = M[i * CI_LD + i];
    sd[i] = d > tol ? 1.0 / sqrt(d) : 0.0;
  }
  __syncthreads();
  for (int idx = tid; idx < p * p; idx += CI_THREADS) {
    const int c = idx / p, i = idx - c * p;
    if (i >= c) M[c * CI_LD + i] = dsc[c] * (i == c ? 1.0 : M[i * CI_LD + c]) * sd[i];
  }
  __syncthreads();

  CI_STAMP(4);
  // (5) output, column-major with leading dimension ldt
  for (int idx = tid; idx < l * l; idx += CI_THREADS) {
    const int j = idx / l, c = idx - j * l;  // T[c + j ldt]: consecutive threads along c
    double v = 0.0;
    if (j < p) {
      if (c >= r) {
        const int cc = c - r;
        v = cc <= j ? M[cc * CI_LD + j] : 0.0;
      } else {
        for (int i = 0; i <= j; ++i) v = fma(-X[c * p + i], M[i * CI_LD + j], v);
      }
    }
    T[c + (int64_t)j * ldt] = (Tq)v;
  }
  CI_STAMP(5);
#undef CI_STAMP
  if (tid == 0) {
    int s = r;
    for (int i = 0; i < p; ++i) s += (sd[i] > 0.0);
    *s_out = s;
  }
}

}  // namespace frsvt
