// Warm start of the small SVD under range propagation (reading R16).
//
// With a carry of r columns the basis is Q = [Q~-derived columns | p fresh
// columns]. The carried columns come out of the power step
// nearly aligned with the singular directions of B (their Gram block G_cc is
// nearly diagonal and G_cf is small), while the p fresh columns are a random
// basis of the rest: G_ff is a dense p x p block. The one-sided Jacobi then
// spends its sweeps resolving G_ff. Diagonalising G_ff first (a 24- or
// 32-column Jacobi on [[G_ff, 0], [0, c I]], c > lambda_max(G_ff)) and rotating G by
// V = blockdiag(I_r, V_f) leaves a nearly diagonal G2 = V^T G V, which the
// full solve resolves in a few sweeps; U_B = V U2. Same eigenvalues, same
// invariant subspaces (an exact similarity), so X is unchanged up to rounding.
// All decisions are on the device (r is a device scalar): outside
// 2 <= p <= 32 (or r = 0) the kernels copy G / do nothing.
#pragma once
#include "common.cuh"

namespace frsvt {

constexpr int EW_P = 32;  // largest fresh block handled

// Gpad (W x W, column-major) = [[G_ff, 0], [0, c I]], W = 24 when p <= 24
// else 32 (fewer Jacobi rounds for the usual small p); flags[0] = W (0 when
// the warm start does not apply), flags[1] = (W == 24), flags[2] = (W == 32)
__global__ void __launch_bounds__(256) eig_fresh_pack_kernel(const double* __restrict__ G, int l,
                                                              const int* __restrict__ r_dev, double* __restrict__ Gpad,
                                                              int* __restrict__ flags) {
  const int r = min(max(*r_dev, 0), l), p = l - r;
  const bool on = r > 0 && p >= 2 && p <= EW_P;
  const int W = !on ? 0 : (p <= 24 ? 24 : EW_P);
  if (threadIdx.x == 0) {
    flags[0] = W;
    flags[1] = W == 24 ? 1 : 0;
    flags[2] = W == EW_P ? 1 : 0;
  }
  if (!on) return;
  __shared__ double tr;
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < p; ++i) t += fabs(G[(size_t)(r + i) * (l + 1)]);
    tr = 2.0 * t + 1.0;  // > lambda_max(G_ff) (G_ff is PSD: lambda_max <= trace)
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < W * W; idx += blockDim.x) {
    const int i = idx % W, j = idx / W;
    double v = 0.0;
    if (i < p && j < p) v = G[(r + i) + (size_t)(r + j) * l];
    else if (i == j) v = tr;
    Gpad[idx] = v;
  }
}

// G2 = V^T G V, V = blockdiag(I_r, V_f), V_f = Uf[0:p, W-p:W] (the padding
// eigenvalue c sorts first; Uf is W x W); a copy of G when the warm start is off
__global__ void __launch_bounds__(256) eig_fresh_rotate_kernel(const double* __restrict__ G, int l,
                                                                const int* __restrict__ r_dev,
                                                                const double* __restrict__ Uf,
                                                                const int* __restrict__ flag,
                                                                double* __restrict__ G2) {
  __shared__ double Vf[EW_P * EW_P];
  const int W = *flag;
  const bool on = W != 0;
  const int r = min(max(*r_dev, 0), l), p = l - r;
  if (on) {
    for (int idx = threadIdx.x; idx < EW_P * EW_P; idx += blockDim.x) {
      const int i = idx % EW_P, j = idx / EW_P;  // Vf[i + j * 32]
      Vf[idx] = (i < p && j < p) ? Uf[i + (size_t)(W - p + j) * W] : 0.0;
    }
  }
  __syncthreads();
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < l * l; idx += gridDim.x * blockDim.x) {
    const int a = idx % l, b = idx / l;
    if (!on || (a < r && b < r)) {
      G2[idx] = G[idx];
      continue;
    }
    double v = 0.0;
    if (a < r) {  // (G_cf V_f)[a, b - r]
      for (int k = 0; k < p; ++k) v = fma(G[a + (size_t)(r + k) * l], Vf[k + (b - r) * EW_P], v);
    } else if (b < r) {  // (V_f^T G_fc)[a - r, b]
      for (int k = 0; k < p; ++k) v = fma(Vf[k + (a - r) * EW_P], G[(r + k) + (size_t)b * l], v);
    } else {  // (V_f^T G_ff V_f)[a - r, b - r]
      for (int k = 0; k < p; ++k) {
        double t = 0.0;
        for (int q = 0; q < p; ++q) t = fma(G[(r + k) + (size_t)(r + q) * l], Vf[q + (b - r) * EW_P], t);
        v = fma(Vf[k + (a - r) * EW_P], t, v);
      }
    }
    G2[idx] = v;
  }
}

// U_B[r:, :] <- V_f U_B[r:, :] (one thread per column)
__global__ void __launch_bounds__(128) eig_fresh_back_kernel(double* __restrict__ UB, int l,
                                                              const int* __restrict__ r_dev,
                                                              const double* __restrict__ Uf,
                                                              const int* __restrict__ flag) {
  const int W = *flag;
  if (!W) return;
  const int r = min(max(*r_dev, 0), l), p = l - r;
  __shared__ double Vf[EW_P * EW_P];
  for (int idx = threadIdx.x; idx < EW_P * EW_P; idx += blockDim.x) {
    const int i = idx % EW_P, j = idx / EW_P;
    Vf[idx] = (i < p && j < p) ? Uf[i + (size_t)(W - p + j) * W] : 0.0;
  }
  __syncthreads();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= l) return;
  double u[EW_P];
#pragma unroll
  for (int k = 0; k < EW_P; ++k) u[k] = k < p ? UB[(r + k) + (size_t)c * l] : 0.0;
  for (int i = 0; i < p; ++i) {
    double v = 0.0;
#pragma unroll
    for (int k = 0; k < EW_P; ++k) v = fma(Vf[i + k * EW_P], u[k], v);
    UB[(r + i) + (size_t)c * l] = v;
  }
}

}  // namespace frsvt
