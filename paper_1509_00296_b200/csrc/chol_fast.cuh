// CholeskyQR first pass without an explicit inverse (fp32 handles,
// FRSVT_FASTCHOL=1; the default is chol_inv.cuh + a tensor-core apply):
//   trsm_rows_kernel : Q1 = Y R'^{-1}, one thread per row of Y, 32-column blocks,
// with R' from orth_chol_kernel's R mode ("QR_CP",
// reading R4): R' = R diag(dsc)^{-1} of the equilibrated Gram's Cholesky factor
// with column drop, so Y R'^{-1} = Y diag(dsc) R^{-1}. Only the span of Q1
// matters downstream (Prop. 1).
#pragma once
#include "common.cuh"

namespace frsvt {

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
