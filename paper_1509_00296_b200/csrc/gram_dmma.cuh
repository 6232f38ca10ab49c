// fp64 Gram G = Y^T Y of a tall m x l matrix (first CholeskyQR pass, PAPER.md
// P:130/P:163; the small-SVD Gram B B^T = Z'^T Z') on the fp64 tensor cores.
//
// fp32 inputs are widened to fp64 (their products are exact in fp64) and
// accumulated in fp64 by mma.sync.m8n8k4.f64 (DMMA): G is tiled into 8 x 8
// blocks and only the upper-triangular ones are computed (symmetry halves the
// work). Each CTA takes a contiguous range of rows, stages 32-row chunks in
// shared memory (coalesced column reads), and its 16 warps own disjoint sets
// of 8 x 8 blocks, accumulating in registers; one fp64 partial per CTA (both
// triangles written), summed over CTAs by splitk_reduce_wide_kernel.
#pragma once
#include "common.cuh"

namespace frsvt {

constexpr int GD_THREADS = 512;
constexpr int GD_ROWS = 32;                 // rows per staged chunk
constexpr int GD_LD = FRSVT_LMAX + 4;       // padded row stride (doubles) of the staged chunk
constexpr int GD_WARPS = GD_THREADS / 32;
constexpr int GD_MAXB = 9;                  // 8x8 blocks per warp: 16*17/2 = 136 for l = 128 over 16 warps

__device__ __forceinline__ void dmma_m8n8k4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <typename Tin>
__global__ void __launch_bounds__(GD_THREADS)
gram_dmma_kernel(const Tin* __restrict__ Y, int64_t rows, int64_t ldy, int l, int64_t rows_per_cta,
                 double* __restrict__ part, const int* __restrict__ r_dev = nullptr) {
  // r_dev (nullable, range propagation): only the 8 x 8 blocks whose column
  // block reaches the fresh columns [r, l) are formed (G12 and G22, the
  // entries chol_inv_kernel reads); the rest of the partial is left stale.
  __shared__ double sY[GD_ROWS * GD_LD];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nb8 = (l + 7) >> 3;
  const int nblk = nb8 * (nb8 + 1) / 2;
  const int jb0 = r_dev ? (min(max(*r_dev, 0), l) >> 3) : 0;
  // this warp's blocks: q = warp + GD_WARPS t, (bi <= bj) in row-major upper order
  int bi[GD_MAXB], bj[GD_MAXB];
  double acc0[GD_MAXB], acc1[GD_MAXB];
#pragma unroll
  for (int t = 0; t < GD_MAXB; ++t) {
    int q = warp + GD_WARPS * t, i = 0;
    if (q < nblk) {
      while (q >= nb8 - i) {
        q -= nb8 - i;
        ++i;
      }
      bi[t] = i;
      bj[t] = i + q;
      if (bj[t] < jb0) bi[t] = bj[t] = -1;
    } else {
      bi[t] = -1;
      bj[t] = -1;
    }
    acc0[t] = 0.0;
    acc1[t] = 0.0;
  }
  const int64_t r0 = blockIdx.x * rows_per_cta;
  const int64_t r1 = min(rows, r0 + rows_per_cta);
  const int kq = lane & 3, g = lane >> 2;
  // software pipeline: the next 32-row chunk is loaded into registers while
  // the current one is multiplied (all of a thread's loads in flight at once)
  constexpr int PER = GD_ROWS * FRSVT_LMAX / GD_THREADS;  // 8 elements per thread
  Tin pre[PER];
  auto load_chunk = [&](int64_t rc) {
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int idx = threadIdx.x + GD_THREADS * u;
      const int rr = idx & (GD_ROWS - 1), c = idx >> 5;
      const int64_t r = rc + rr;
      pre[u] = (c < l && r < r1) ? Y[r + (int64_t)c * ldy] : Tin(0);
    }
  };
  if (r0 < r1) load_chunk(r0);
  for (int64_t rc = r0; rc < r1; rc += GD_ROWS) {
    __syncthreads();
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int idx = threadIdx.x + GD_THREADS * u;
      const int rr = idx & (GD_ROWS - 1), c = idx >> 5;
      sY[rr * GD_LD + c] = (double)pre[u];  // columns >= l are zero (padding of the last 8-block)
    }
    __syncthreads();
    if (rc + GD_ROWS < r1) load_chunk(rc + GD_ROWS);
#pragma unroll 2
    for (int k = 0; k < GD_ROWS; k += 4) {
      const double* rowp = sY + (k + kq) * GD_LD + g;
#pragma unroll
      for (int t = 0; t < GD_MAXB; ++t) {
        if (bi[t] >= 0) {
          const double a = rowp[8 * bi[t]];
          const double b = rowp[8 * bj[t]];
          dmma_m8n8k4(acc0[t], acc1[t], a, b);
        }
      }
    }
  }
  // partial (l x l, column-major), both triangles
  double* P = part + (int64_t)blockIdx.x * l * l;
#pragma unroll
  for (int t = 0; t < GD_MAXB; ++t) {
    if (bi[t] < 0) continue;
    const int i = 8 * bi[t] + g, j0 = 8 * bj[t] + 2 * kq;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int j = j0 + e;
      const double v = e ? acc1[t] : acc0[t];
      if (i < l && j < l) {
        P[i + (int64_t)j * l] = v;
        P[j + (int64_t)i * l] = v;
      }
    }
  }
}

}  // namespace frsvt
