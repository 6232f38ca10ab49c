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
  // S (l*(l+1): Schur complement, then the dense inverse with stride l+1) +
  // packed R (l(l+1)/2) + dsc (l) + W scratch (3 x 32 x 32) doubles; keep (l) ints
  return ((size_t)l * (l + 1) + (size_t)l * (l + 1) / 2 + (size_t)l + 3 * 1024) * sizeof(double) +
         (size_t)l * sizeof(int) + 64;
}

__device__ __forceinline__ int oc_pk(int i, int j) { return j * (j + 1) / 2 + i; }  // packed upper, i <= j

template <typename Tq>
__global__ void __launch_bounds__(OC_THREADS, 1)
orth_chol_kernel(const double* __restrict__ G, int l, double tol, Tq* __restrict__ T, int* __restrict__ s_out,
                 int* __restrict__ flags, unsigned long long* __restrict__ prof = nullptr,
                 const int* __restrict__ skip = nullptr, double* __restrict__ Rout = nullptr) {
  // Rout (nullable): stop after the factorisation and write R' = R diag(dsc)^{-1}
  // (l x l row-major upper, fp64; dropped rows and diagonals 0) for the
  // row-parallel TRSM apply Y R'^{-1} = Y diag(dsc) R^{-1}; T is not written.
  // skip (nullable): a device flag set when the Loewdin path already produced T
  if (skip && *skip) return;
  // prof (test hook, nullable): %globaltimer stamps at phase boundaries
#define OC_STAMP(k)                                                                  \
  do {                                                                               \
    if (prof && threadIdx.x == 0) {                                                  \
      unsigned long long t_;                                                         \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                         \
      prof[k] = t_;                                                                  \
    }                                                                                \
  } while (0)
  OC_STAMP(0);
  extern __shared__ double ocs[];
  double* S = ocs;                                  // l*l row-major; R overwrites the upper triangle
  double* Tt = S + (size_t)l * (l + 1);             // packed R (after the factorisation)
  double* dsc = Tt + (size_t)l * (l + 1) / 2;
  double* Wsc = dsc + l;                            // 3 x 32 x 32 block products
  int* keep = (int*)(Wsc + 3 * 1024);
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

  OC_STAMP(1);
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
    if (P == 0) OC_STAMP(2);
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
    if (P == 0) OC_STAMP(3);
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

  OC_STAMP(4);
  if (Rout) {
    for (int idx = tid; idx < l * l; idx += OC_THREADS) {
      const int i = idx / l, j = idx % l;
      double v = 0.0;
      if (j >= i && keep[i] && dsc[j] > 0.0) v = S[(size_t)i * l + j] / dsc[j];
      Rout[idx] = v;
    }
    if (tid == 0) {
      int s = 0;
      for (int i = 0; i < l; ++i) s += keep[i];
      *s_out = s;
    }
    return;
  }
  // T~ = R^{-1} on the kept set (dropped rows/columns are zero), by 32 x 32
  // blocks: (A) the diagonal blocks, one warp each, back substitution in
  // registers (lane = column); (B) block diagonals d = 1.. in parallel:
  // W_IJ = sum_{I<K<=J} R_IK T_KJ, T_IJ = -T_II W_IJ. R is first moved to
  // packed storage so that S can hold the dense inverse (row stride l + 1).
  for (int idx = tid; idx < l * l; idx += OC_THREADS) {
    const int i = idx / l, j = idx % l;
    if (j >= i) Tt[oc_pk(i, j)] = keep[i] ? S[(size_t)i * l + j] : 0.0;
  }
  __syncthreads();
  double* Tn = S;  // dense inverse, Tn[i * (l + 1) + j]
  const int ldt = l + 1;
  for (int idx = tid; idx < l * ldt; idx += OC_THREADS) Tn[idx] = 0.0;
  __syncthreads();
  const int NB = (l + 31) >> 5;
  if (warp < NB) {
    const int c = lane, w0 = 32 * warp, j = w0 + c;
    double x[32];
#pragma unroll
    for (int r = 31; r >= 0; --r) {
      const int i = w0 + r;
      double v = 0.0;
      if (i < l && keep[i] && r <= c && j < l && keep[j]) {
        double s0 = (r == c) ? 1.0 : 0.0, s1 = 0.0;
#pragma unroll
        for (int k = r + 1; k < 32; k += 2) {
          if (w0 + k < l) s0 = fma(-Tt[oc_pk(i, w0 + k)], x[k], s0);
          if (k + 1 < 32 && w0 + k + 1 < l) s1 = fma(-Tt[oc_pk(i, w0 + k + 1)], x[k + 1], s1);
        }
        v = (s0 + s1) / Tt[oc_pk(i, i)];
      }
      x[r] = v;
    }
    if (j < l) {
#pragma unroll
      for (int r = 0; r < 32; ++r)
        if (w0 + r < l) Tn[(size_t)(w0 + r) * ldt + j] = x[r];
    }
  }
  __syncthreads();
  OC_STAMP(5);
  for (int d = 1; d < NB; ++d) {
    const int npairs = NB - d;
    // (B1) W_IJ = sum_{K = I+1..J} R_IK T_KJ  (thread: b fastest -> broadcast R, stride-1 T)
    for (int o = tid; o < npairs * 1024; o += OC_THREADS) {
      const int pr = o >> 10, a = (o >> 5) & 31, b = o & 31;
      const int I = pr, J = pr + d;
      const int gi = 32 * I + a, gj = 32 * J + b;
      double w = 0.0, w2 = 0.0;
      if (gi < l && gj < l) {
        const int t1 = min(gj, l - 1);
        int t = 32 * (I + 1);
        for (; t + 1 <= t1; t += 2) {
          w = fma(Tt[oc_pk(gi, t)], Tn[(size_t)t * ldt + gj], w);
          w2 = fma(Tt[oc_pk(gi, t + 1)], Tn[(size_t)(t + 1) * ldt + gj], w2);
        }
        if (t <= t1) w = fma(Tt[oc_pk(gi, t)], Tn[(size_t)t * ldt + gj], w);
      }
      Wsc[pr * 1024 + a * 32 + b] = w + w2;
    }
    __syncthreads();
    // (B2) T_IJ = -T_II W_IJ
    for (int o = tid; o < npairs * 1024; o += OC_THREADS) {
      const int pr = o >> 10, a = (o >> 5) & 31, b = o & 31;
      const int I = pr, J = pr + d;
      const int gi = 32 * I + a, gj = 32 * J + b;
      if (gi < l && gj < l) {
        double v = 0.0, v2 = 0.0;
        for (int t = a; t < 32; t += 2) {
          v = fma(Tn[(size_t)gi * ldt + 32 * I + t], Wsc[pr * 1024 + t * 32 + b], v);
          if (t + 1 < 32) v2 = fma(Tn[(size_t)gi * ldt + 32 * I + t + 1], Wsc[pr * 1024 + (t + 1) * 32 + b], v2);
        }
        Tn[(size_t)gi * ldt + gj] = -(v + v2);
      }
    }
    __syncthreads();
  }
  OC_STAMP(6);
  for (int idx = tid; idx < l * l; idx += OC_THREADS) {
    const int o = idx % l, j = idx / l;  // T[o + j*l]
    T[idx] = (Tq)((o <= j) ? dsc[o] * Tn[(size_t)o * ldt + j] : 0.0);
  }
  OC_STAMP(7);
  if (tid == 0) {
    int s = 0;
    for (int i = 0; i < l; ++i) s += keep[i];
    *s_out = s;
  }
}

}  // namespace frsvt
