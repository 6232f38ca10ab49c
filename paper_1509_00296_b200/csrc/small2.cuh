// Single-CTA small-matrix kernels on the l x l fp64 Gram (l <= 128), 1024
// threads, the Schur complement held in registers (thread (ty, tx) owns the
// entries (ty + 32a, tx + 32b), a, b < 4) so each pivot step costs two
// block barriers and 16 register FMAs per thread.
//
// Pivoted Cholesky with logical pivoting (no row/column swaps): step k picks
// the largest remaining Schur diagonal p, writes row k of R over the original
// column index (zero on already-pivoted columns) and updates the complement.
// A pivot <= tol * ref truncates the factorisation at s = k: the rank reveal of
// QR-CP ("estimating the rank ... by QR decomposition with
// Column Pivoting"), realised on the Gram.
//
// MODE_ORTH: equilibrated Gram (unit diagonal); also builds T~ = R~^{-1}
//   column by column (T~[0:k, k] = -T~[0:k,0:k] R~[0:k,k] / R~[k,k], warp
//   reductions, packed in shared memory) and writes T (l x l) with
//   Y T = orthonormal basis of range(Y) (CholeskyQR step).
// MODE_EIG: Gram G = B B^T of the projected matrix B = Q^T A (Alg. 1 line 16).
//   G = M M^T with M = R^T (columns = rows of R, original coordinates), and a
//   one-sided Jacobi on the s columns of M gives M J = U_B diag(sigma): the
//   small SVD of B (sigma_i(B), left vectors U_B) without accumulating J. The
//   pivoted Cholesky is the QR preconditioning of Drmac-Veselic, which cuts
//   the Jacobi sweep count. Replaces Alg. 1 lines 16-18 (QR, Newton polar,
//   eigendecomposition; reading Z8).
#pragma once
#include "common.cuh"

namespace frsvt {

constexpr int SM2_ORTH = 0;
constexpr int SM2_EIG = 1;

__host__ __device__ constexpr size_t small2_smem_bytes(int l, int mode) {
  // R (l*l) + packed T~ (l(l+1)/2, ORTH) + dsc, nrm (2l) doubles; piv, ipiv, dn (3l) ints; cand 2x32 (val, idx)
  return ((size_t)l * l + (mode == SM2_ORTH ? (size_t)l * (l + 1) / 2 : 0) + 2 * (size_t)l + 64) * sizeof(double) +
         (3 * (size_t)l + 64) * sizeof(int);
}

__device__ __forceinline__ int pk_col(int i, int j) { return j * (j + 1) / 2 + i; }  // packed upper, i <= j

template <int MODE, typename Tq>
__global__ void __launch_bounds__(1024, 1)
small2_kernel(const double* __restrict__ G, int l, double tol, Tq* __restrict__ T, double* __restrict__ sigma,
              double* __restrict__ UB, int* __restrict__ s_out, int* __restrict__ sweeps_out,
              int* __restrict__ flags, int max_sweeps) {
  extern __shared__ double sm2[];
  double* R = sm2;                                     // l*l, row k = R[k*l + c]
  double* Tt = R + (size_t)l * l;                      // packed T~ (ORTH)
  double* dsc = Tt + (MODE == SM2_ORTH ? (size_t)l * (l + 1) / 2 : 0);
  double* nrm = dsc + l;
  double* cval = nrm + l;                              // 2 x 32
  int* piv = (int*)(cval + 64);
  int* ipiv = piv + l;
  int* dn = ipiv + l;
  int* cidx = dn + l;                                  // 2 x 32
  __shared__ double refmax;
  __shared__ int s_sh;

  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;

  for (int i = tid; i < l; i += 1024) {
    const double g = G[i + (size_t)i * l];
    if (!isfinite(g)) atomicOr(flags, FLAG_NONFINITE);
    dsc[i] = (MODE == SM2_ORTH) ? ((g > 0.0 && isfinite(g)) ? 1.0 / sqrt(g) : 0.0) : 1.0;
    dn[i] = 0;
    ipiv[i] = l;
  }
  if (tid == 0) {
    double mx = 0.0;
    for (int i = 0; i < l; ++i) {
      const double g = G[i + (size_t)i * l];
      if (isfinite(g)) mx = fmax(mx, g);
    }
    refmax = (MODE == SM2_ORTH) ? 1.0 : mx;
    s_sh = l;
  }
  __syncthreads();

  double S[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int i = ty + 32 * a, c = tx + 32 * b;
      double v = 0.0;
      if (i < l && c < l) {
        v = G[i + (size_t)c * l] * dsc[i] * dsc[c];
        if (!isfinite(v)) v = 0.0;
      }
      S[a][b] = v;
    }
  const double thr = tol * refmax;

  int k = 0;
  for (; k < l; ++k) {
    const int buf = k & 1;
    if (tx == ty) {
      double best = -1.0;
      int bj = l;
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int j = ty + 32 * a;
        if (j < l && !dn[j] && S[a][a] > best) { best = S[a][a]; bj = j; }
      }
      cval[buf * 32 + ty] = best;
      cidx[buf * 32 + ty] = bj;
    }
    __syncthreads();  // S1
    double best = cval[buf * 32 + tx];
    int bj = cidx[buf * 32 + tx];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
      if (ob > best || (ob == best && oj < bj)) { best = ob; bj = oj; }
    }
    if (!(best > thr) || bj >= l) break;  // uniform across the block
    const int p = bj;
    const double rkk = sqrt(best);
    if (ty == (p & 31)) {
      const int ap = p >> 5;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int c = tx + 32 * b;
        if (c < l) {
          double rv;
          if (c == p) rv = rkk;
          else if (dn[c]) rv = 0.0;
          else {
            // compile-time row select keeps S in registers
            const double spb = ap == 0 ? S[0][b] : (ap == 1 ? S[1][b] : (ap == 2 ? S[2][b] : S[3][b]));
            rv = spb / rkk;
          }
          R[(size_t)k * l + c] = rv;
        }
      }
    }
    if (tid == 0) {
      piv[k] = p;
      ipiv[p] = k;
      dn[p] = 1;  // (readers of dn[c != p] above touch other words)
    }
    __syncthreads();  // S2: R row k and dn[p] visible
    double ri[4], rc[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int i = ty + 32 * a;
      ri[a] = (i < l) ? R[(size_t)k * l + i] : 0.0;
    }
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int c = tx + 32 * b;
      rc[b] = (c < l) ? R[(size_t)k * l + c] : 0.0;
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) S[a][b] -= ri[a] * rc[b];
    if (MODE == SM2_ORTH) {
      // T~[i][k] = -(sum_{i<=t<k} T~[i][t] R[t][p]) / rkk for i < k; T~[k][k] = 1/rkk
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int i = ty + 32 * a;
        double u = 0.0;
        if (i < k) {
          for (int t = i + tx; t < k; t += 32) u += Tt[pk_col(i, t)] * R[(size_t)t * l + p];
        }
        u = warp_sum(u);
        if (i < k && tx == 0) Tt[pk_col(i, k)] = -u / rkk;
      }
      if (tid == 0) Tt[pk_col(k, k)] = 1.0 / rkk;
    }
  }
  if (tid == 0) s_sh = k;
  __syncthreads();
  const int s = s_sh;

  if (MODE == SM2_ORTH) {
    for (int idx = tid; idx < l * l; idx += 1024) {
      const int o = idx % l, j = idx / l;  // T[o + j*l]
      const int kk = ipiv[o];
      double v = 0.0;
      if (j < s && kk <= j) v = dsc[o] * Tt[pk_col(kk, j)];
      T[idx] = (Tq)v;
    }
    if (tid == 0) *s_out = s;
    return;
  }

  // ---------------- MODE_EIG: one-sided Jacobi on the s columns of M = R^T ----
  const int L2 = (s + 1) & ~1;
  const int h = L2 / 2;
  const int lane = tx, warp = ty;
  int sweep = 0;
  bool converged = (s <= 1);
  for (sweep = 0; sweep < max_sweeps && !converged; ++sweep) {
    // exact column norms at the start of each sweep
    for (int c = warp; c < s; c += 32) {
      double a2 = 0.0;
      for (int i = lane; i < l; i += 32) {
        const double x = R[(size_t)c * l + i];
        a2 += x * x;
      }
      a2 = warp_sum(a2);
      if (lane == 0) nrm[c] = a2;
    }
    __syncthreads();
    int rotated = 0;
    for (int rnd = 0; rnd < L2 - 1; ++rnd) {
      for (int q = warp; q < h; q += 32) {
        const int pa = q, pb = L2 - 1 - q;
        int p1 = pa == 0 ? 0 : 1 + ((pa - 1 + rnd) % (L2 - 1));
        int p2 = pb == 0 ? 0 : 1 + ((pb - 1 + rnd) % (L2 - 1));
        if (p1 > p2) { const int t = p1; p1 = p2; p2 = t; }
        if (p2 >= s) continue;
        double* x = R + (size_t)p1 * l;
        double* y = R + (size_t)p2 * l;
        double xv[4], yv[4];
        double g = 0.0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int i = lane + 32 * e;
          xv[e] = i < l ? x[i] : 0.0;
          yv[e] = i < l ? y[i] : 0.0;
          g += xv[e] * yv[e];
        }
        g = warp_sum(g);
        const double al = nrm[p1], be = nrm[p2];
        if (fabs(g) > 1e-15 * sqrt(al * be) && fabs(g) > 1e-300) {
          const double zeta = (be - al) / (2.0 * g);
          const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double cs = 1.0 / sqrt(1.0 + t * t), sn = cs * t;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int i = lane + 32 * e;
            if (i < l) {
              x[i] = cs * xv[e] - sn * yv[e];
              y[i] = sn * xv[e] + cs * yv[e];
            }
          }
          __syncwarp();
          if (lane == 0) {
            nrm[p1] = al - t * g;
            nrm[p2] = be + t * g;
          }
          rotated = 1;
        }
      }
      __syncthreads();
    }
    converged = !__syncthreads_or(rotated);
  }
  // sigma_k = ||m_k||, U_B(:, k) = m_k / sigma_k, sorted descending
  for (int c = warp; c < s; c += 32) {
    double a2 = 0.0;
    for (int i = lane; i < l; i += 32) {
      const double x = R[(size_t)c * l + i];
      a2 += x * x;
    }
    a2 = warp_sum(a2);
    if (lane == 0) nrm[c] = sqrt(a2);
  }
  __syncthreads();
  for (int c = tid; c < l; c += 1024) {
    if (c >= s) {
      sigma[c] = 0.0;
      for (int i = 0; i < l; ++i) UB[i + (size_t)c * l] = 0.0;
    }
  }
  for (int c = warp; c < s; c += 32) {
    const double sc = nrm[c];
    int rank = 0;
    for (int j = 0; j < s; ++j) {
      const double sj = nrm[j];
      rank += (sj > sc) || (sj == sc && j < c);
    }
    if (lane == 0) sigma[rank] = sc;
    const double inv = sc > 0.0 ? 1.0 / sc : 0.0;
    for (int i = lane; i < l; i += 32) UB[i + (size_t)rank * l] = R[(size_t)c * l + i] * inv;
  }
  if (tid == 0) {
    *sweeps_out = sweep;
    if (!converged) atomicOr(flags, FLAG_NOCONV);
  }
}

}  // namespace frsvt
