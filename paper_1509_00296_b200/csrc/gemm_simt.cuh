// Generic SIMT skinny GEMM  C(M x N) = A(M x K) * B(K x N)  for the passes of
// Algorithm 1 where one dimension is the sketch width l:
//   Y  = A * X        (A m x n, X n x l)        A M-contiguous, B K-contiguous
//   Z  = A^T * Q      (split-K over the m rows)  A K-contiguous, B K-contiguous
//   G  = Y^T * Y      (fp64 accumulate, split-K) A K-contiguous, B K-contiguous
//   Y' = Y * T        (T l x l)                  A M-contiguous, B K-contiguous
//   L  = Qt * Wt^T    (reconstruction, K = r)    A M-contiguous, B N-contiguous
// Tiles: BM x BN x BK with a TM x TN register tile per thread, 256 threads.
// Rows of a thread are strided by BM/TM so a warp touches consecutive rows
// (coalesced column-major epilogue, conflict-free A reads from shared memory).
// The epilogue is a functor called per output element; functors with
// kReduce = true return a double that is block-reduced into part[block].
#pragma once
#include "common.cuh"

namespace frsvt {

template <typename Tin, typename Tacc, int BM, int BN, int BK, int TM, int TN,
          bool A_MC, bool B_KC, class Epi>
__global__ void __launch_bounds__(256)
gemm_simt_kernel(int M, int N, int K, int kchunk,
                 const Tin* __restrict__ A, int64_t lda,
                 const Tin* __restrict__ B, int64_t ldb,
                 const int* __restrict__ kdev, Epi epi) {
  constexpr int NT = 256;
  constexpr int TXN = BM / TM;
  static_assert(TXN * (BN / TN) == NT, "tile/thread mismatch");
  __shared__ Tacc As[BK][BM + 4];
  __shared__ Tacc Bs[BK][BN + 4];
  __shared__ double red_scratch[NT / 32];

  const int tid = threadIdx.x;
  const int tx = tid % TXN, ty = tid / TXN;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int kbeg = blockIdx.z * kchunk;
  int kend = min(K, kbeg + kchunk);
  if (kdev != nullptr) kend = min(kend, *kdev);

  Tacc acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = Tacc(0);

  for (int k0 = kbeg; k0 < kend; k0 += BK) {
#pragma unroll 4
    for (int idx = tid; idx < BM * BK; idx += NT) {
      int i, k;
      if (A_MC) { i = idx % BM; k = idx / BM; } else { k = idx % BK; i = idx / BK; }
      const int gi = m0 + i, gk = k0 + k;
      Tacc v = Tacc(0);
      if (gi < M && gk < kend)
        v = (Tacc)(A_MC ? A[gi + (int64_t)gk * lda] : A[gk + (int64_t)gi * lda]);
      As[k][i] = v;
    }
#pragma unroll 4
    for (int idx = tid; idx < BK * BN; idx += NT) {
      int k, j;
      if (B_KC) { k = idx % BK; j = idx / BK; } else { j = idx % BN; k = idx / BN; }
      const int gk = k0 + k, gj = n0 + j;
      Tacc v = Tacc(0);
      if (gj < N && gk < kend)
        v = (Tacc)(B_KC ? B[gk + (int64_t)gj * ldb] : B[gj + (int64_t)gk * ldb]);
      Bs[k][j] = v;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      Tacc a[TM], b[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) a[i] = As[k][tx + i * TXN];
#pragma unroll
      for (int j = 0; j < TN; ++j) b[j] = Bs[k][ty * TN + j];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }

  double red = 0.0;
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int gi = m0 + tx + i * TXN;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int gj = n0 + ty * TN + j;
      if (gi < M && gj < N) red += epi(gi, gj, acc[i][j], (int)blockIdx.z);
    }
  }
  if (Epi::kReduce) {
    double s = block_sum(red, red_scratch);
    if (tid == 0)
      epi.part[blockIdx.x + (int64_t)gridDim.x * (blockIdx.y + (int64_t)gridDim.y * blockIdx.z)] = s;
  }
}

// ---- epilogues -------------------------------------------------------------
template <typename Tout>
struct EpiStore {  // C[z*zstride + i + j*ldc] = v
  Tout* C;
  int64_t ldc, zstride;
  double* part = nullptr;
  static constexpr bool kReduce = false;
  template <typename Tacc>
  __device__ __forceinline__ double operator()(int i, int j, Tacc v, int z) const {
    C[(int64_t)z * zstride + i + (int64_t)j * ldc] = (Tout)v;
    return 0.0;
  }
};

template <typename Tout>
struct EpiStoreAdd {  // C = v + Add   (range propagation: Y = A*Omega' + Q~)
  Tout* C;
  int64_t ldc;
  const Tout* Add;
  int64_t ldadd;
  double* part = nullptr;
  static constexpr bool kReduce = false;
  template <typename Tacc>
  __device__ __forceinline__ double operator()(int i, int j, Tacc v, int) const {
    C[i + (int64_t)j * ldc] = (Tout)(v + (Tacc)Add[i + (int64_t)j * ldadd]);
    return 0.0;
  }
};

// Fused iALM epilogue (S:449 order):
// given the tile value L_{k+1}(i,j) of the reconstruction,
//   resid += (D - L - E)^2                 (E = E_{k+1})
//   Y_{k+1}/mu_{k+1} = (A_k - L) * mu_k/mu_{k+1}
//   E_{k+2} = S_{lambda/mu_{k+1}}(D - L + Y_{k+1}/mu_{k+1})
//   A_{k+1} = D - E_{k+2} + Y_{k+1}/mu_{k+1}
// finalize: write L, leave D/E/A untouched.
template <typename T>
struct EpiAlm {
  const T* D;
  T* Aop;
  T* E;
  T* L;
  int64_t ld;
  const double* mu;  // device {mu_k, mu_bar}
  double rho, lambda;
  int finalize;
  double* part;
  static constexpr bool kReduce = true;
  template <typename Tacc>
  __device__ __forceinline__ double operator()(int i, int j, Tacc v, int) const {
    const int64_t o = i + (int64_t)j * ld;
    const T Lv = (T)v;
    const T d = D[o];
    const T e = E[o];
    const T res = d - Lv - e;
    if (finalize) {
      L[o] = Lv;
    } else {
      const double mu0 = __ldg(mu);
      const double mu1 = fmin(rho * mu0, __ldg(mu + 1));
      const T ratio = (T)(mu0 / mu1);
      const T thr = (T)(lambda / mu1);
      const T a = Aop[o];
      const T rr = (a - Lv) * ratio;
      const T en = soft<T>(d - Lv + rr, thr);
      E[o] = en;
      Aop[o] = d - en + rr;
    }
    return (double)res * (double)res;
  }
};

}  // namespace frsvt
