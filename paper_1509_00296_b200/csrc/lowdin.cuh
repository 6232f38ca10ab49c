// Second CholeskyQR pass by symmetric (Loewdin) orthogonalisation.
//
// After the first pass Q1 = Y T1 is nearly orthonormal: G2 = Q1^T Q1 = I + E
// with |E| ~ u32 kappa(Y). Any T2 with T2^T G2 T2 = I and the same span
// finishes orth(Y) (only the span of the basis enters Alg. 1, Prop. 1
// P:103-111). T2 = G2^{-1/2} is a short series in E:
//   (I + E)^{-1/2} = I - E/2 + 3/8 E^2 - 5/16 E^3 + 35/128 E^4 + O(E^5),
// i.e. three l x l products, spread over many CTAs, instead of a serial
// l-step Cholesky and triangular inverse on one SM. Used when max|E_ij| <=
// 0.05 (truncation <= 63/256 * 0.05^5 ~ 8e-8 per entry); otherwise the flag
// stays 0 and the Cholesky path (orth_chol_kernel with `skip` = this flag)
// produces T2. Columns that pass 1 dropped (zero in Q1, G2_dd ~ 0) are kept
// out of E and mapped to zero.
#pragma once
#include "common.cuh"

namespace frsvt {

// Shared-memory staging: LWD_T rows (or columns) x l of an l x l fp64 matrix per block.
constexpr int LWD_THREADS = 256;
constexpr int LWD_T = 16;  // output tile LWD_T x LWD_T per block, one output per thread (several accumulator chains)
__host__ __device__ constexpr size_t lowdin_smem_bytes(int l) { return (size_t)3 * LWD_T * l * sizeof(double); }

// E(i, j) of G2 (column-major): G2 - I on kept columns, 0 elsewhere
__device__ __forceinline__ double lowdin_e(const double* __restrict__ G2, int l, int i, int j) {
  const double gi = G2[i + (size_t)i * l], gj = G2[j + (size_t)j * l];
  if (!(gi > 0.25) || !(gj > 0.25)) return 0.0;
  const double e = G2[i + (size_t)j * l] - (i == j ? 1.0 : 0.0);
  return isfinite(e) ? e : 1e300;
}

// Block (bx, by) of an LWD_T x LWD_T tiling: E2 tile = (E E)(rows, cols of the tile), and
// max|E| over its row panel folded into *emax (atomicMax on the bit pattern of a non-negative double)
__global__ void __launch_bounds__(LWD_THREADS) lowdin_sq_kernel(const double* __restrict__ G2, int l,
                                                                double* __restrict__ E2,
                                                                unsigned long long* __restrict__ emax) {
  extern __shared__ double lws[];
  double* Ar = lws;              // [T][l]: E(i0 + a, k)
  double* Bc = lws + LWD_T * l;  // [l][T]: E(k, j0 + b) stored Bc[k * T + b]
  const int i0 = blockIdx.x * LWD_T, j0 = blockIdx.y * LWD_T;
  double mx = 0.0;
  for (int idx = threadIdx.x; idx < LWD_T * l; idx += blockDim.x) {
    const int a = idx % LWD_T, k = idx / LWD_T;  // consecutive threads: consecutive rows
    const double ea = (i0 + a < l) ? lowdin_e(G2, l, i0 + a, k) : 0.0;
    Ar[a * l + k] = ea;
    mx = fmax(mx, fabs(ea));
    Bc[k * LWD_T + a] = (j0 + a < l) ? lowdin_e(G2, l, k, j0 + a) : 0.0;
  }
  if (blockIdx.y == 0) {
    mx = warp_max(mx);
    if ((threadIdx.x & 31) == 0) atomicMax(emax, __double_as_longlong(mx));
  }
  __syncthreads();
  const int a = threadIdx.x / LWD_T, b = threadIdx.x % LWD_T;
  if (i0 + a < l && j0 + b < l) {
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    int k = 0;
    for (; k + 3 < l; k += 4) {
#pragma unroll
      for (int u = 0; u < 4; ++u) s[u] = fma(Ar[a * l + k + u], Bc[(k + u) * LWD_T + b], s[u]);
    }
    for (; k < l; ++k) s[0] = fma(Ar[a * l + k], Bc[k * LWD_T + b], s[0]);
    E2[(i0 + a) + (size_t)(j0 + b) * l] = (s[0] + s[1]) + (s[2] + s[3]);
  }
}

// T2 = I - E/2 + 3/8 E2 - 5/16 E E2 + 35/128 E2 E2 on kept columns (0 on
// dropped ones); *ok = (max|E| <= 0.05), written by block (0, 0)
template <typename Tq>
__global__ void __launch_bounds__(LWD_THREADS) lowdin_series_kernel(const double* __restrict__ G2,
                                                                    const double* __restrict__ E2, int l,
                                                                    const unsigned long long* __restrict__ emax,
                                                                    int* __restrict__ ok, Tq* __restrict__ T) {
  const bool good = __longlong_as_double((long long)*emax) <= 0.05;
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) *ok = good ? 1 : 0;
  if (!good) return;
  extern __shared__ double lws[];
  double* Er = lws;                  // [T][l]  E(i0 + a, k)
  double* Fr = lws + LWD_T * l;      // [T][l]  E2(i0 + a, k)
  double* Fc = lws + 2 * LWD_T * l;  // [l][T]  E2(k, j0 + b)
  const int i0 = blockIdx.x * LWD_T, j0 = blockIdx.y * LWD_T;
  for (int idx = threadIdx.x; idx < LWD_T * l; idx += blockDim.x) {
    const int a = idx % LWD_T, k = idx / LWD_T;
    const bool ri = i0 + a < l, cj = j0 + a < l;
    Er[a * l + k] = ri ? lowdin_e(G2, l, i0 + a, k) : 0.0;
    Fr[a * l + k] = ri ? E2[(i0 + a) + (size_t)k * l] : 0.0;
    Fc[k * LWD_T + a] = cj ? E2[k + (size_t)(j0 + a) * l] : 0.0;
  }
  __syncthreads();
  const int a = threadIdx.x / LWD_T, b = threadIdx.x % LWD_T;
  const int i = i0 + a, j = j0 + b;
  if (i < l && j < l) {
    double e3[2] = {0.0, 0.0}, e4[2] = {0.0, 0.0};
    int k = 0;
    for (; k + 1 < l; k += 2) {
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const double f = Fc[(k + u) * LWD_T + b];
        e3[u] = fma(Er[a * l + k + u], f, e3[u]);
        e4[u] = fma(Fr[a * l + k + u], f, e4[u]);
      }
    }
    for (; k < l; ++k) {
      const double f = Fc[k * LWD_T + b];
      e3[0] = fma(Er[a * l + k], f, e3[0]);
      e4[0] = fma(Fr[a * l + k], f, e4[0]);
    }
    const double gi = G2[i + (size_t)i * l], gj = G2[j + (size_t)j * l];
    double t = (i == j ? 1.0 : 0.0) - 0.5 * Er[a * l + j] + 0.375 * Fr[a * l + j] - 0.3125 * (e3[0] + e3[1]) +
               0.2734375 * (e4[0] + e4[1]);
    if (!(gi > 0.25) || !(gj > 0.25)) t = 0.0;
    T[i + (size_t)j * l] = (Tq)t;
  }
}

// C (M x N) = op(A) op(B), fp64 inputs, column-major, K <= FRSVT_LMAX; one
// LWD_T x LWD_T tile of C per block (one output per thread, 4 accumulator
// chains); the A rows / B columns the tile needs are staged in shared memory
// first. op(X) = X or X^T (trans flags). Used for the l x l products that
// fold the second CholeskyQR factor into the small SVD.
template <typename Tout>
__global__ void __launch_bounds__(LWD_THREADS) sgemm64_kernel(int M, int N, int K, const double* __restrict__ A,
                                                              int lda, int ta, const double* __restrict__ B, int ldb,
                                                              int tb, Tout* __restrict__ C, int ldc) {
  extern __shared__ double lws[];
  double* As = lws;              // [T][K]: op(A)(i0 + a, k)
  double* Bs = lws + LWD_T * K;  // [K][T]: op(B)(k, j0 + b)
  const int i0 = blockIdx.x * LWD_T, j0 = blockIdx.y * LWD_T;
  for (int idx = threadIdx.x; idx < LWD_T * K; idx += blockDim.x) {
    int a, k;
    if (ta) { a = idx / K; k = idx % K; } else { a = idx % LWD_T; k = idx / LWD_T; }
    const int i = i0 + a;
    As[a * K + k] = (i < M) ? (ta ? A[k + (size_t)i * lda] : A[i + (size_t)k * lda]) : 0.0;
  }
  for (int idx = threadIdx.x; idx < LWD_T * K; idx += blockDim.x) {
    int b, k;
    if (tb) { b = idx % LWD_T; k = idx / LWD_T; } else { b = idx / K; k = idx % K; }
    const int j = j0 + b;
    Bs[k * LWD_T + b] = (j < N) ? (tb ? B[j + (size_t)k * ldb] : B[k + (size_t)j * ldb]) : 0.0;
  }
  __syncthreads();
  const int a = threadIdx.x / LWD_T, b = threadIdx.x % LWD_T;
  if (i0 + a >= M || j0 + b >= N) return;
  double s[4] = {0.0, 0.0, 0.0, 0.0};
  int k = 0;
  for (; k + 3 < K; k += 4) {
#pragma unroll
    for (int u = 0; u < 4; ++u) s[u] = fma(As[a * K + k + u], Bs[(k + u) * LWD_T + b], s[u]);
  }
  for (; k < K; ++k) s[0] = fma(As[a * K + k], Bs[k * LWD_T + b], s[0]);
  C[(i0 + a) + (size_t)(j0 + b) * ldc] = (Tout)((s[0] + s[1]) + (s[2] + s[3]));
}

}  // namespace frsvt
