// CholeskyQR first pass without an explicit inverse (fp32 handles):
//   chol_rows_kernel : R' of the equilibrated Gram, one CTA, register resident
//   trsm_rows_kernel : Q1 = Y R'^{-1}, one thread per row of Y, 32-column blocks
//
// The factor ("QR_CP", reading R4): unpivoted Cholesky
// of S = diag(dsc) G diag(dsc), dsc_i = G_ii^{-1/2}, with column drop: a
// column whose Schur diagonal is <= tol (relative to its own norm^2) gets a
// zero row in R (a zero column in Q1). Only the span of Q1 matters downstream
// (Prop. 1). R' = R diag(dsc)^{-1}, so Y R'^{-1} = Y diag(dsc) R^{-1}.
//
// chol_rows_kernel: each of the 1024 threads owns <= 9 entries (i <= j) of the
// upper triangle of S in registers. Step k reads row k of the current Schur
// complement from a double-buffered shared row, every thread forms
// 1/S_kk itself, updates its entries with i > k by S_ij -= S_ki S_kj / S_kk,
// and the owners of row k+1 publish it: one block barrier per step. The owner
// of (k, j) writes R'_kj = S_kj / sqrt(S_kk) / dsc_j at step k.
#pragma once
#include "common.cuh"

namespace frsvt {

constexpr int CHR_THREADS = 1024;
constexpr int CHR_PER = (FRSVT_LMAX * (FRSVT_LMAX + 1) / 2 + CHR_THREADS - 1) / CHR_THREADS;  // 9

__global__ void __launch_bounds__(CHR_THREADS, 1)
chol_rows_kernel(const double* __restrict__ G, int l, double tol, double* __restrict__ Rp, int* __restrict__ s_out,
                 int* __restrict__ flags, const int* __restrict__ skip) {
  if (skip && *skip) return;
  __shared__ double dsc[FRSVT_LMAX];
  __shared__ double row[2][FRSVT_LMAX];
  const int tid = threadIdx.x;
  for (int i = tid; i < l; i += CHR_THREADS) {
    const double g = G[i + (size_t)i * l];
    if (!isfinite(g)) atomicOr(flags, FLAG_NONFINITE);
    dsc[i] = (g > 0.0 && isfinite(g)) ? rsqrt(g) : 0.0;
  }
  __syncthreads();
  // owned entries: e = tid + CHR_THREADS q of the row-major upper triangle
  double s[CHR_PER];
  int ij[CHR_PER];  // (i << 16) | j, or -1
  const int ntri = l * (l + 1) / 2;
#pragma unroll
  for (int q = 0; q < CHR_PER; ++q) {
    const int e = tid + CHR_THREADS * q;
    int i = -1, j = -1;
    if (e < ntri) {
      // row i starts at base(i) = i l - i (i - 1) / 2; invert the prefix sum
      const double b2 = 2.0 * l + 1.0;
      int ri = (int)floor(0.5 * (b2 - sqrt(b2 * b2 - 8.0 * e)));
      ri = max(0, min(l - 1, ri));
      while (ri > 0 && ri * l - ri * (ri - 1) / 2 > e) --ri;
      while (ri + 1 < l && (ri + 1) * l - (ri + 1) * ri / 2 <= e) ++ri;
      i = ri;
      j = ri + (e - (ri * l - ri * (ri - 1) / 2));
    }
    ij[q] = i >= 0 ? ((i << 16) | j) : -1;
    double v = 0.0;
    if (i >= 0) {
      v = G[i + (size_t)j * l] * dsc[i] * dsc[j];
      if (!isfinite(v)) v = 0.0;
      if (i == 0) row[0][j] = v;
    }
    s[q] = v;
  }
  __syncthreads();
  int kept = 0;
  for (int k = 0; k < l; ++k) {
    const double* rk = row[k & 1];
    double* rn = row[(k + 1) & 1];
    const double d = rk[k];
    const bool ok = d > tol;
    const double dinv = ok ? 1.0 / d : 0.0;
    const double rin = ok ? rsqrt(d) : 0.0;
    if (tid == 0) kept += ok ? 1 : 0;
#pragma unroll
    for (int q = 0; q < CHR_PER; ++q) {
      const int i = ij[q] >= 0 ? (ij[q] >> 16) : -1, j = ij[q] & 0xFFFF;
      if (i == k) {  // row k of R' (final)
        Rp[(size_t)k * l + j] = (ok && dsc[j] > 0.0) ? s[q] * rin / dsc[j] : 0.0;
      } else if (i > k) {
        s[q] = fma(-rk[i] * dinv, rk[j], s[q]);
        if (i == k + 1) rn[j] = s[q];
      }
    }
    __syncthreads();
  }
  // lower triangle of R' is zero
  for (int idx = tid; idx < l * l; idx += CHR_THREADS) {
    const int i = idx / l, j = idx % l;
    if (j < i) Rp[idx] = 0.0;
  }
  if (tid == 0) *s_out = kept;
}

// Q (rows x l) = Y R'^{-1}: q R' = y by forward substitution, one thread per
// row. The row is processed in NB blocks of 32 columns (fully unrolled); a
// solved block is stored and re-read as one batch of loads when a later block
// needs it (register pressure, occupancy). R' (fp32 copy, row-major,
// zero padded) and 1/R'_ii are broadcast from shared memory (LDS.128 for the
// off-diagonal block updates). Rows of R' with a zero diagonal are dropped
// columns (q = 0).
template <int NB>
__global__ void __launch_bounds__(128)
trsm_rows_kernel(const float* __restrict__ Y, int64_t rows, int64_t ldy, const double* __restrict__ Rp, int l,
                 float* __restrict__ Q, int64_t ldq) {
  constexpr int LP = 32 * NB;
  extern __shared__ float trs[];
  float* R = trs;             // [LP][LP]
  float* rin = trs + LP * LP;
  for (int idx = threadIdx.x; idx < LP * LP; idx += blockDim.x) {
    const int i = idx / LP, j = idx % LP;
    R[idx] = (i < l && j < l) ? (float)Rp[(size_t)i * l + j] : 0.f;
  }
  for (int i = threadIdx.x; i < LP; i += blockDim.x) {
    const double d = i < l ? Rp[(size_t)i * l + i] : 0.0;
    rin[i] = d != 0.0 ? (float)(1.0 / d) : 0.f;
  }
  __syncthreads();
  const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (row >= rows) return;
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    float acc[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) acc[c] = (32 * b + c < l) ? Y[row + (int64_t)(32 * b + c) * ldy] : 0.f;
#pragma unroll 1
    for (int bp = 0; bp < b; ++bp) {
      // the already solved block bp, re-read as one batch of independent loads
      // (this thread wrote it; L1/L2 hits) instead of holding all q in registers
      float qb[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) qb[k] = (32 * bp + k < l) ? Q[row + (int64_t)(32 * bp + k) * ldq] : 0.f;
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const float qk = qb[k];
        const float4* r4 = reinterpret_cast<const float4*>(R + (32 * bp + k) * LP + 32 * b);
#pragma unroll
        for (int c4 = 0; c4 < 8; ++c4) {
          const float4 rv = r4[c4];
          acc[4 * c4 + 0] = fmaf(-qk, rv.x, acc[4 * c4 + 0]);
          acc[4 * c4 + 1] = fmaf(-qk, rv.y, acc[4 * c4 + 1]);
          acc[4 * c4 + 2] = fmaf(-qk, rv.z, acc[4 * c4 + 2]);
          acc[4 * c4 + 3] = fmaf(-qk, rv.w, acc[4 * c4 + 3]);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const float qi = acc[i] * rin[32 * b + i];
      acc[i] = qi;
#pragma unroll
      for (int c = i + 1; c < 32; ++c) acc[c] = fmaf(-qi, R[(32 * b + i) * LP + 32 * b + c], acc[c]);
    }
#pragma unroll
    for (int c = 0; c < 32; ++c)
      if (32 * b + c < l) Q[row + (int64_t)(32 * b + c) * ldq] = acc[c];
  }
}

}  // namespace frsvt
