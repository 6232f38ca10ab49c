// CholeskyQR factor for orth(Y): blocked, unpivoted Cholesky of the
// equilibrated fp64 Gram with column drop, and T = diag(dsc) R^{-1}, in one CTA.
//
// Y T spans range(Y) with orthonormal columns ("QR_CP(Y)",
// P:141 "QR(A A^T Q)"); numerically dependent columns are dropped: a
// column whose Schur diagonal (equilibrated, i.e. relative to its own norm^2)
// falls to <= tol gets a zero row in R and a zero column in T. This is the
// rank reveal of QR-CP realised without pivoting (reading R4); only the span
// matters downstream (Prop. 1), so the column order is irrelevant.
//
// 16-column panels: the 16 x 16 diagonal block is factored by one warp
// (warp-synchronous, no block barrier), the panel's rows are completed by a
// triangular solve (one thread per trailing column), and the trailing matrix
// gets a rank-16 update from a 16 x 16 thread grid — three block barriers per
// panel instead of two per column. T~ = R^{-1} by 16 x 16 blocks.
#pragma once
#include "common.cuh"

namespace frsvt {

constexpr int OC_THREADS = 256;

__host__ __device__ constexpr size_t orth_chol_smem_bytes(int l) {
  // S (l*l) + packed T~ (l(l+1)/2) + dsc (l) doubles; keep (l) ints
  return ((size_t)l * l + (size_t)l * (l + 1) / 2 + (size_t)l) * sizeof(double) + (size_t)l * sizeof(int) + 64;
}

__device__ __forceinline__ int oc_pk(int i, int j) { return j * (j + 1) / 2 + i; }  // packed upper, i <= j

template <typename Tq>
__global__ void __launch_bounds__(OC_THREADS, 1)
orth_chol_kernel(const double* __restrict__ G, int l, double tol, Tq* __restrict__ T, int* __restrict__ s_out,
                 int* __restrict__ flags) {
  extern __shared__ double ocs[];
  double* S = ocs;                                  // l*l row-major; R overwrites the upper triangle
  double* Tt = S + (size_t)l * l;                   // packed T~
  double* dsc = Tt + (size_t)l * (l + 1) / 2;
  int* keep = (int*)(dsc + l);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tx = tid & 15, ty = tid >> 4;

  for (int i = tid; i < l; i += OC_THREADS) {
    const double g = G[i + (size_t)i * l];
    if (!isfinite(g)) atomicOr(flags, FLAG_NONFINITE);
    dsc[i] = (g > 0.0 && isfinite(g)) ? rsqrt(g) : 0.0;
  }
  __syncthreads();
  for (int idx = tid; idx < l * l; idx += OC_THREADS) {
    const int i = idx / l, c = idx % l;
    double v = G[i + (size_t)c * l] * dsc[i] * dsc[c];
    S[idx] = isfinite(v) ? v : 0.0;
  }
  __syncthreads();

  const int nb = (l + 15) >> 4;
  for (int P = 0; P < nb; ++P) {
    const int k0 = 16 * P, k1 = min(k0 + 16, l);
    // (1) diagonal block, warp 0, in registers: lane c (< 16) holds column
    //     k0 + c of the block; rows are broadcast with shuffles.
    if (warp == 0) {
      const int c = lane & 15;
      double col[16];
#pragma unroll
      for (int r = 0; r < 16; ++r)
        col[r] = (k0 + r < k1 && k0 + c < k1) ? S[(size_t)(k0 + r) * l + k0 + c] : 0.0;
      int kp = 0;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        if (k0 + j < k1) {
          const double d = __shfl_sync(0xffffffffu, col[j], j);  // Schur diagonal (k0+j, k0+j)
          const bool drop = !(d > tol);
          const double rin = drop ? 0.0 : rsqrt(d);
          if (c == j) col[j] = drop ? 0.0 : d * rin;
          else if (c > j) col[j] *= rin;                         // R[j][c]
          if (c == j) kp = drop ? 0 : 1;
#pragma unroll
          for (int r = j + 1; r < 16; ++r) {
            const double rjr = __shfl_sync(0xffffffffu, col[j], r);  // R[j][r]
            if (c >= r) col[r] = fma(-rjr, col[j], col[r]);
          }
        }
      }
      if (lane < 16 && k0 + c < k1) {
#pragma unroll
        for (int r = 0; r < 16; ++r)
          if (k0 + r < k1 && r <= c) S[(size_t)(k0 + r) * l + k0 + c] = col[r];
        keep[k0 + c] = kp;
      }
    }
    __syncthreads();
    // (2) panel rows over the trailing columns, one thread per column, in
    //     registers: R[j][c] = (S[j][c] - sum_{k0<=t<j} R[t][j] R[t][c]) / R[j][j]
    for (int c = k1 + tid; c < l; c += OC_THREADS) {
      double v[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = (k0 + j < k1) ? S[(size_t)(k0 + j) * l + c] : 0.0;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        if (k0 + j < k1) {
          double acc = v[j];
#pragma unroll
          for (int t = 0; t < j; ++t) acc = fma(-S[(size_t)(k0 + t) * l + k0 + j], v[t], acc);
          const double rjj = S[(size_t)(k0 + j) * l + k0 + j];
          v[j] = keep[k0 + j] ? acc / rjj : 0.0;
        }
      }
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (k0 + j < k1) S[(size_t)(k0 + j) * l + c] = v[j];
    }
    __syncthreads();
    // (3) trailing update (upper triangle): S[c1][c2] -= sum_{t in panel} R[t][c1] R[t][c2]
    const int w = l - k1;
    if (w > 0) {
      for (int a0 = 0; a0 < w; a0 += 16 * 8) {
        double acc[8][8];
        int c1s[8], c2s[8];
#pragma unroll
        for (int a = 0; a < 8; ++a) {
          c1s[a] = k1 + a0 + ty + 16 * a;
#pragma unroll
          for (int b = 0; b < 8; ++b) acc[a][b] = 0.0;
        }
#pragma unroll
        for (int b = 0; b < 8; ++b) c2s[b] = k1 + tx + 16 * b;
        for (int t = k0; t < k1; ++t) {
          double r1[8], r2[8];
#pragma unroll
          for (int a = 0; a < 8; ++a) r1[a] = c1s[a] < l ? S[(size_t)t * l + c1s[a]] : 0.0;
#pragma unroll
          for (int b = 0; b < 8; ++b) r2[b] = c2s[b] < l ? S[(size_t)t * l + c2s[b]] : 0.0;
#pragma unroll
          for (int a = 0; a < 8; ++a)
#pragma unroll
            for (int b = 0; b < 8; ++b) acc[a][b] = fma(r1[a], r2[b], acc[a][b]);
        }
#pragma unroll
        for (int a = 0; a < 8; ++a)
#pragma unroll
          for (int b = 0; b < 8; ++b)
            if (c1s[a] < l && c2s[b] < l && c2s[b] >= c1s[a]) S[(size_t)c1s[a] * l + c2s[b]] -= acc[a][b];
      }
    }
    __syncthreads();
  }

  // T~ = R^{-1} on the kept set (dropped rows/columns are zero): 16 x 16 blocks.
  for (int I = warp; I < nb; I += OC_THREADS / 32) {
    // lane c (< 16) owns column j = 16 I + c of T~_II, kept in registers;
    // R_II rows are broadcast reads from shared memory
    const int c = lane & 15, i0 = 16 * I;
    const int j = i0 + c;
    double tcol[16];
#pragma unroll
    for (int r = 15; r >= 0; --r) {
      const int i = i0 + r;
      double u = (r == c) ? 1.0 : 0.0;
#pragma unroll
      for (int t = r + 1; t < 16; ++t)
        if (t <= c && i0 + t < l) u = fma(-S[(size_t)i * l + i0 + t], tcol[t], u);
      const bool ok = (r <= c) && (j < l) && (i < l) && keep[i] && keep[j];
      tcol[r] = ok ? u / S[(size_t)i * l + i] : 0.0;
    }
    if (lane < 16 && j < l) {
#pragma unroll
      for (int r = 0; r < 16; ++r)
        if (r <= c) Tt[oc_pk(i0 + r, j)] = tcol[r];
    }
  }
  __syncthreads();
  for (int d = 1; d < nb; ++d) {
    for (int I = 0; I + d < nb; ++I) {
      const int J = I + d;
      const int gi = 16 * I + ty, gj = 16 * J + tx;
      double wv = 0.0;
      if (gi < l && gj < l) {
        // W = sum_{t = 16(I+1)}^{gj} R[gi][t] T~[t][gj]
        double w1 = 0.0, w2 = 0.0, w3 = 0.0;
        int t = 16 * (I + 1);
        for (; t + 3 <= gj; t += 4) {
          wv = fma(S[(size_t)gi * l + t], Tt[oc_pk(t, gj)], wv);
          w1 = fma(S[(size_t)gi * l + t + 1], Tt[oc_pk(t + 1, gj)], w1);
          w2 = fma(S[(size_t)gi * l + t + 2], Tt[oc_pk(t + 2, gj)], w2);
          w3 = fma(S[(size_t)gi * l + t + 3], Tt[oc_pk(t + 3, gj)], w3);
        }
        for (; t <= gj; ++t) wv = fma(S[(size_t)gi * l + t], Tt[oc_pk(t, gj)], wv);
        wv = (wv + w1) + (w2 + w3);
      }
      __syncthreads();
      if (gi < l && gj < l) Tt[oc_pk(gi, gj)] = wv;
      __syncthreads();
      double v = 0.0;
      if (gi < l && gj < l) {
        const int i1 = min(16 * I + 16, l);
        for (int t = gi; t < i1; ++t) v = fma(Tt[oc_pk(gi, t)], Tt[oc_pk(t, gj)], v);
      }
      __syncthreads();
      if (gi < l && gj < l) Tt[oc_pk(gi, gj)] = keep[gj] ? -v : 0.0;
      __syncthreads();
    }
  }
  for (int idx = tid; idx < l * l; idx += OC_THREADS) {
    const int o = idx % l, j = idx / l;  // T[o + j*l]
    T[idx] = (Tq)((o <= j) ? dsc[o] * Tt[oc_pk(o, j)] : 0.0);
  }
  if (tid == 0) {
    int s = 0;
    for (int i = 0; i < l; ++i) s += keep[i];
    *s_out = s;
  }
}

}  // namespace frsvt
