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
  constexpr int CR = GD_ROWS, LDC = GD_LD;
  __shared__ double sY[CR * LDC];
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
  constexpr int PER = CR * (LDC - 4) / GD_THREADS;  // 8 elements per thread
  Tin pre[PER];
  auto load_chunk = [&](int64_t rc) {
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int idx = threadIdx.x + GD_THREADS * u;
      const int rr = idx % CR, c = idx / CR;
      const int64_t r = rc + rr;
      pre[u] = (c < l && r < r1) ? Y[r + (int64_t)c * ldy] : Tin(0);
    }
  };
  if (r0 < r1) load_chunk(r0);
  for (int64_t rc = r0; rc < r1; rc += CR) {
    __syncthreads();
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int idx = threadIdx.x + GD_THREADS * u;
      const int rr = idx % CR, c = idx / CR;
      sY[rr * LDC + c] = (double)pre[u];  // columns >= l are zero (padding of the last 8-block)
    }
    __syncthreads();
    if (rc + CR < r1) load_chunk(rc + CR);
#pragma unroll 2
    for (int k = 0; k < CR; k += 4) {
      const double* rowp = sY + (k + kq) * LDC + g;
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

// Gram of a tall NARROW matrix (l <= 16, e.g. BASELINE c3's l = 10 over
// 76800 rows): the 8 x 8 DMMA blocks would leave most warps idle and chain
// dependent MMAs, so here threads own entries (i <= j) of the upper triangle
// and accumulate them in fp64 over 256-row chunks staged in shared memory.
// Thread t loads row t of the chunk (all l columns, issued together: one
// memory latency per chunk, not one per element); with at most 64 entries
// (l <= 10) four threads share an entry, each over a quarter of the rows,
// and their sums are added in a fixed order. One partial per CTA (both
// triangles), summed over CTAs by splitk_reduce_wide_kernel.
constexpr int GS_THREADS = 256;
constexpr int GS_ROWS = 256;
constexpr int GS_LMAX = 16;
constexpr int GS_LD = GS_ROWS + 1;  // odd column stride (doubles): the lanes of a warp read
                                    // different columns at the same row without bank conflicts
template <typename Tin>
__global__ void __launch_bounds__(GS_THREADS)
gram_small_kernel(const Tin* __restrict__ Y, int64_t rows, int64_t ldy, int l, int64_t rows_per_cta,
                  double* __restrict__ part) {
  static_assert(GS_ROWS == GS_THREADS, "one row per thread");
  __shared__ double sY[GS_LMAX * GS_LD];  // column-major chunk
  __shared__ double red[3][64];
  const int ne = l * (l + 1) / 2;
  const int ks_n = ne <= 64 ? 4 : 1;          // threads per entry
  const int ei = ks_n == 4 ? (threadIdx.x & 63) : threadIdx.x;
  const int ks = ks_n == 4 ? (threadIdx.x >> 6) : 0;
  const int kr = GS_ROWS / ks_n;              // rows of the chunk per thread
  int ii = 0, jj = 0;
  if (ei < ne) {
    int q = ei;
    while (q >= l - ii) {
      q -= l - ii;
      ++ii;
    }
    jj = ii + q;
  }
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  const int64_t r0 = blockIdx.x * rows_per_cta;
  const int64_t r1 = min(rows, r0 + rows_per_cta);
  for (int64_t rc = r0; rc < r1; rc += GS_ROWS) {
    const int64_t r = rc + threadIdx.x;
    Tin v[GS_LMAX];
#pragma unroll
    for (int c = 0; c < GS_LMAX; ++c) v[c] = (c < l && r < r1) ? Y[r + (int64_t)c * ldy] : Tin(0);
    __syncthreads();  // the previous chunk is consumed
#pragma unroll
    for (int c = 0; c < GS_LMAX; ++c)
      if (c < l) sY[c * GS_LD + threadIdx.x] = (double)v[c];
    __syncthreads();
    if (ei < ne) {
      const double* yi = sY + ii * GS_LD + ks * kr;
      const double* yj = sY + jj * GS_LD + ks * kr;
#pragma unroll 4
      for (int k = 0; k < kr; k += 4) {
        a0 = fma(yi[k], yj[k], a0);
        a1 = fma(yi[k + 1], yj[k + 1], a1);
        a2 = fma(yi[k + 2], yj[k + 2], a2);
        a3 = fma(yi[k + 3], yj[k + 3], a3);
      }
    }
  }
  double v = (a0 + a1) + (a2 + a3);
  if (ks_n == 4) {
    if (ks > 0 && ei < ne) red[ks - 1][ei] = v;
    __syncthreads();
    if (ks == 0 && ei < ne) v = ((v + red[0][ei]) + red[1][ei]) + red[2][ei];
  }
  if (ks == 0 && ei < ne) {
    double* P = part + (int64_t)blockIdx.x * l * l;
    P[ii + (int64_t)jj * l] = v;
    P[jj + (int64_t)ii * l] = v;
  }
}

}  // namespace frsvt
