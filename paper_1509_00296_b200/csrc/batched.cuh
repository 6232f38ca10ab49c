// Batched FRSVT of many small independent matrices (
// PAPER.md P:23 / P:48: WNNM's weighted SVT of many patch-group matrices,
// per-window problems): ONE CTA per matrix runs the whole of
// Algorithm 1 in shared memory, so a batch is one launch whose
// bound is the SM (shared memory and FMA pipes), not HBM.
//
// Per matrix (A m x n fp32, column-major; l <= BT_LMAX; shared Omega n x l):
//   Y = A Omega                                   (fp32 FMA, Alg. 1 line 3)
//   Q = orth(Y)                                   CGS2 in fp64 with rank reveal
//   q x { Z = orth(A^T Q); Q = orth(A Z) }        power iteration (lines 13-15)
//   W = A^T Q  (= B^T)                            (line 16)
//   one-sided Jacobi on the columns of W:  W V = V_B Sigma, V accumulates U_B
//                                                 (the SVD of B, lines 16-18; reading Z8)
//   d_i = max(sigma_i - t_i, 0), t_i = tau or w_i (weighted SVT, fn. 1 P:48)
//   X = (Q V diag(d / sigma)) (W V)^T             Eq. (6)
// Products of A with the small operands are fp32 sums of at most
// max(m, n) terms (~1e-6 relative), the orthonormalisation and the Jacobi
// fp64. Thread block: 256 threads (8 warps).
#pragma once
#include "common.cuh"

namespace frsvt {

constexpr int BT_THREADS = 256;
constexpr int BT_WARPS = BT_THREADS / 32;
constexpr int BT_LMAX = 16;

__host__ __device__ inline size_t batched_smem_bytes(int m, int n, int l) {
  // Q (m x l) and W (n x l) fp64, V (l x l) fp64, per-warp scratch, A fp32
  return ((size_t)(m + n) * l + (size_t)l * l + (size_t)BT_WARPS * BT_LMAX + 4 * BT_LMAX) * sizeof(double) +
         (size_t)m * n * sizeof(float) + 64;
}

// Out (rows x l, fp64) = A * In (AX) or A^T * In (ATQ), A in shared memory
// (m x n fp32, column-major); fp32 accumulation
__device__ __forceinline__ void bt_ax(const float* __restrict__ sA, int m, int n, int l,
                                      const double* __restrict__ In, double* __restrict__ Out) {
  for (int idx = threadIdx.x; idx < m * l; idx += BT_THREADS) {
    const int i = idx % m, c = idx / m;
    float acc = 0.f;
    for (int j = 0; j < n; ++j) acc = fmaf(sA[i + j * m], (float)In[j + c * n], acc);
    Out[idx] = acc;
  }
}
__device__ __forceinline__ void bt_atx(const float* __restrict__ sA, int m, int n, int l,
                                       const double* __restrict__ In, double* __restrict__ Out) {
  // one warp per output (j, c): lanes split the m rows, shuffle reduction
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int o = warp; o < n * l; o += BT_WARPS) {
    const int j = o % n, c = o / n;
    float acc = 0.f;
    for (int i = lane; i < m; i += 32) acc = fmaf(sA[i + j * m], (float)In[i + c * m], acc);
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
    if (lane == 0) Out[o] = acc;
  }
}

// CTA sum of one value per thread (fp64); every thread gets the result
__device__ __forceinline__ double bt_sum(double v, double* scratch) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) v += __shfl_xor_sync(0xffffffffu, v, s);
  __syncthreads();
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  double t = 0.0;
#pragma unroll
  for (int w = 0; w < BT_WARPS; ++w) t += scratch[w];
  return t;
}

// Orthonormal columns for Y (rows x l, fp64, in place) by classical
// Gram-Schmidt with one re-orthogonalisation (CGS2); a column whose residual
// is <= tol of its original norm is numerically dependent and becomes zero
// (the rank reveal of P:163, reading R4). Returns the kept count.
__device__ int bt_orth(double* __restrict__ Y, int rows, int l, double tol, double* scratch, double* coef) {
  int kept = 0;
  for (int j = 0; j < l; ++j) {
    double* y = Y + (size_t)j * rows;
    double loc = 0.0;
    for (int i = threadIdx.x; i < rows; i += BT_THREADS) loc = fma(y[i], y[i], loc);
    const double n0 = sqrt(bt_sum(loc, scratch));
    for (int pass = 0; pass < 2; ++pass) {
      // coef[k] = Q_k . y for k < j: warp w handles k = w, w + 8, ...
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
      for (int k = warp; k < j; k += BT_WARPS) {
        const double* qk = Y + (size_t)k * rows;
        double s = 0.0;
        for (int i = lane; i < rows; i += 32) s = fma(qk[i], y[i], s);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) coef[k] = s;
      }
      __syncthreads();
      for (int i = threadIdx.x; i < rows; i += BT_THREADS) {
        double v = y[i];
        for (int k = 0; k < j; ++k) v = fma(-coef[k], Y[i + (size_t)k * rows], v);
        y[i] = v;
      }
      __syncthreads();
    }
    loc = 0.0;
    for (int i = threadIdx.x; i < rows; i += BT_THREADS) loc = fma(y[i], y[i], loc);
    const double nr = sqrt(bt_sum(loc, scratch));
    const bool keep = n0 > 0.0 && nr > tol * n0;
    const double inv = keep ? 1.0 / nr : 0.0;
    for (int i = threadIdx.x; i < rows; i += BT_THREADS) y[i] *= inv;
    kept += keep ? 1 : 0;
    __syncthreads();
  }
  return kept;
}

// wmode 0: t_i = tau (scalar, or tau_b[b] when given); 1: t_i = w[i] (host
// weights copied to the device, length l, shared by the batch)
__global__ void __launch_bounds__(BT_THREADS)
batched_frsvt_kernel(int m, int n, int l, int q, const float* __restrict__ Ab, int64_t lda, int64_t strideA,
                     const float* __restrict__ Om, int64_t ldo, int wmode, double tau,
                     const double* __restrict__ tau_b, const double* __restrict__ w, float* __restrict__ Xb,
                     int64_t ldx, int64_t strideX, int* __restrict__ r_b, double* __restrict__ sig_b) {
  extern __shared__ double bsm[];
  double* Q = bsm;                               // m x l
  double* W = Q + (size_t)m * l;                 // n x l: Z, then B^T = A^T Q, then W V
  double* V = W + (size_t)n * l;                 // l x l
  double* scratch = V + (size_t)l * l;           // BT_WARPS x BT_LMAX
  double* coef = scratch + BT_WARPS * BT_LMAX;   // BT_LMAX
  double* sg = coef + BT_LMAX;                   // sigma (l)
  double* fd = sg + BT_LMAX;                     // d / sigma (l)
  float* sA = reinterpret_cast<float*>(fd + 2 * BT_LMAX);
  const int b = blockIdx.x;
  const float* A = Ab + (int64_t)b * strideA;
  const int tid = threadIdx.x;
  const double tol = 1e-6;  // fp32 data: a sample whose residual is below 1e-6 of its norm carries no direction
  for (int idx = tid; idx < m * n; idx += BT_THREADS) {
    const int i = idx % m, j = idx / m;
    sA[idx] = A[i + (int64_t)j * lda];
  }
  // Omega (n x l) into W as fp64, then Y = A Omega into Q
  for (int idx = tid; idx < n * l; idx += BT_THREADS) W[idx] = Om[idx % n + (int64_t)(idx / n) * ldo];
  __syncthreads();
  bt_ax(sA, m, n, l, W, Q);
  __syncthreads();
  bt_orth(Q, m, l, tol, scratch, coef);
  for (int it = 0; it < q; ++it) {
    bt_atx(sA, m, n, l, Q, W);
    __syncthreads();
    bt_orth(W, n, l, tol, scratch, coef);
    bt_ax(sA, m, n, l, W, Q);
    __syncthreads();
    bt_orth(Q, m, l, tol, scratch, coef);
  }
  bt_atx(sA, m, n, l, Q, W);  // W = B^T
  for (int idx = tid; idx < l * l; idx += BT_THREADS) V[idx] = (idx % l == idx / l) ? 1.0 : 0.0;
  __syncthreads();
  // one-sided Jacobi on the columns of W (n x l): round-robin pairs, warp w
  // takes pair w of the round; V accumulates the rotations (U_B)
  const int warp = tid >> 5, lane = tid & 31;
  const int L2 = (l + 1) & ~1;
  for (int sweep = 0; sweep < 30; ++sweep) {
    int rotated = 0;
    for (int rnd = 0; rnd < L2 - 1; ++rnd) {
      for (int pr = warp; pr < L2 / 2; pr += BT_WARPS) {
        // circle ordering: position 0 fixed, the others rotate by rnd
        const int a0 = pr == 0 ? 0 : 1 + (pr - 1 + rnd) % (L2 - 1);
        const int b0 = 1 + (L2 - 2 - pr + rnd) % (L2 - 1);
        const int pcol = min(a0, b0), qcol = max(a0, b0);
        if (qcol >= l) continue;
        double* wp = W + (size_t)pcol * n;
        double* wq = W + (size_t)qcol * n;
        double al = 0.0, be = 0.0, g = 0.0;
        for (int i = lane; i < n; i += 32) {
          al = fma(wp[i], wp[i], al);
          be = fma(wq[i], wq[i], be);
          g = fma(wp[i], wq[i], g);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          al += __shfl_xor_sync(0xffffffffu, al, o);
          be += __shfl_xor_sync(0xffffffffu, be, o);
          g += __shfl_xor_sync(0xffffffffu, g, o);
        }
        if (g != 0.0 && fabs(g) > 1e-15 * sqrt(al * be)) {
          rotated = 1;
          const double zeta = (be - al) / (2.0 * g);
          const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
          for (int i = lane; i < n; i += 32) {
            const double x = wp[i], y = wq[i];
            wp[i] = c * x - s * y;
            wq[i] = s * x + c * y;
          }
          for (int i = lane; i < l; i += 32) {
            const double x = V[i + pcol * l], y = V[i + qcol * l];
            V[i + pcol * l] = c * x - s * y;
            V[i + qcol * l] = s * x + c * y;
          }
        }
      }
      __syncthreads();
    }
    if (!__syncthreads_or(rotated)) break;
  }
  // sigma_i = |W_i|, shrink
  for (int i = warp; i < l; i += BT_WARPS) {
    double s2 = 0.0;
    for (int k = lane; k < n; k += 32) s2 = fma(W[k + i * n], W[k + i * n], s2);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    if (lane == 0) sg[i] = sqrt(s2);
  }
  __syncthreads();
  if (tid == 0) {
    // thresholds on sigma sorted descending (rank positions)
    int r = 0;
    for (int i = 0; i < l; ++i) {
      int pos = 0;
      for (int k = 0; k < l; ++k) pos += (sg[k] > sg[i]) || (sg[k] == sg[i] && k < i);
      const double t = wmode == 1 ? w[pos] : (tau_b ? tau_b[b] : tau);
      const double d = fmax(sg[i] - t, 0.0);
      fd[i] = (d > 0.0 && sg[i] > 0.0) ? d / sg[i] : 0.0;
      r += d > 0.0;
      if (sig_b) sig_b[(int64_t)b * l + pos] = sg[i];
    }
    if (r_b) r_b[b] = r;
  }
  __syncthreads();
  // P = Q V diag(d / sigma) into Q's place (row by row: each thread owns rows)
  for (int i = tid; i < m; i += BT_THREADS) {
    double row[BT_LMAX];
#pragma unroll
    for (int c = 0; c < BT_LMAX; ++c) row[c] = 0.0;
    for (int k = 0; k < l; ++k) {
      const double qk = Q[i + (size_t)k * m];
#pragma unroll
      for (int c = 0; c < BT_LMAX; ++c)
        if (c < l) row[c] = fma(qk, V[k + c * l], row[c]);
    }
#pragma unroll
    for (int c = 0; c < BT_LMAX; ++c)
      if (c < l) Q[i + (size_t)c * m] = row[c] * fd[c];
  }
  __syncthreads();
  // X = P W^T (W = B^T V = V_B Sigma)
  float* X = Xb + (int64_t)b * strideX;
  for (int idx = tid; idx < m * n; idx += BT_THREADS) {
    const int i = idx % m, j = idx / m;
    double acc = 0.0;
    for (int c = 0; c < l; ++c) acc = fma(Q[i + (size_t)c * m], W[j + (size_t)c * n], acc);
    X[i + (int64_t)j * ldx] = (float)acc;
  }
}

}  // namespace frsvt
