// Single-CTA small-matrix kernels on the l x l fp64 Gram (l <= 128), 256
// threads. The Schur complement lives in registers: thread (ty, tx) of a
// 16 x 16 grid owns the entries (ty + 16a, tx + 16b), a, b < 8, so a pivot
// step is 64 register FMAs per thread and two block barriers.
//
// Pivoted Cholesky with logical pivoting (no row/column swaps): step k picks
// the largest remaining Schur diagonal p, writes row k of R over the original
// column index (zero on already-pivoted columns) and updates the complement.
// A pivot <= tol * ref truncates the factorisation at s = k: the rank reveal of
// QR-CP ("estimating the rank ... by QR decomposition with
// Column Pivoting"), realised on the Gram.
//
// MODE_ORTH: equilibrated Gram (unit diagonal); then T~ = R~^{-1} (column
//   sweep, one thread per row, R~ = R with columns in pivot order) and the
//   output T (l x l) with Y T = orthonormal basis of range(Y) (CholeskyQR).
// MODE_EIG: Gram G = B B^T of the projected matrix B = Q^T A (Alg. 1 line 16).
//   G = M M^T with M = R^T (columns = rows of R, original coordinates); a
//   one-sided Jacobi on the s columns of M gives M J = U_B diag(sigma), the
//   small SVD of B (sigma_i(B), left vectors U_B), without accumulating J. The
//   pivoted Cholesky is the QR preconditioning of Drmac-Veselic. Replaces Alg. 1
//   lines 16-18 (QR, Newton polar, eigendecomposition; reading Z8).
#pragma once
#include "common.cuh"

namespace frsvt {

constexpr int SM2_ORTH = 0;
constexpr int SM2_EIG = 1;
constexpr int SM2_THREADS = 256;

__host__ __device__ constexpr size_t small2_smem_bytes(int l, int mode) {
  // R (l*l) + packed T~ (l(l+1)/2, ORTH) + dsc, nrm (2l) + cand (32) doubles; piv, ipiv, dn (3l) + cand (32) ints
  return ((size_t)l * l + (mode == SM2_ORTH ? (size_t)l * (l + 1) / 2 : 0) + 2 * (size_t)l + 32) * sizeof(double) +
         (3 * (size_t)l + 32) * sizeof(int);
}

__device__ __forceinline__ int pk_col(int i, int j) { return j * (j + 1) / 2 + i; }  // packed upper, i <= j

template <int MODE, typename Tq>
__global__ void __launch_bounds__(SM2_THREADS, 1)
small2_kernel(const double* __restrict__ G, int l, double tol, Tq* __restrict__ T, double* __restrict__ sigma,
              double* __restrict__ UB, int* __restrict__ s_out, int* __restrict__ sweeps_out,
              int* __restrict__ flags, int max_sweeps, double jtol) {
  extern __shared__ double sm2[];
  double* R = sm2;                                     // l*l, row k = R[k*l + c]
  double* Tt = R + (size_t)l * l;                      // packed T~ (ORTH)
  double* dsc = Tt + (MODE == SM2_ORTH ? (size_t)l * (l + 1) / 2 : 0);
  double* nrm = dsc + l;
  double* cval = nrm + l;                              // 2 x 16
  int* piv = (int*)(cval + 32);
  int* ipiv = piv + l;
  int* dn = ipiv + l;
  int* cidx = dn + l;                                  // 2 x 16
  __shared__ double refmax;
  __shared__ int s_sh;

  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int lane = tid & 31, warp = tid >> 5;

  for (int i = tid; i < l; i += SM2_THREADS) {
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

  double S[8][8];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const int i = ty + 16 * a, c = tx + 16 * b;
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
      for (int a = 0; a < 8; ++a) {
        const int j = ty + 16 * a;
        if (j < l && !dn[j] && S[a][a] > best) { best = S[a][a]; bj = j; }
      }
      cval[buf * 16 + ty] = best;
      cidx[buf * 16 + ty] = bj;
    }
    __syncthreads();  // S1
    // every thread scans the 16 candidates (broadcast loads, no shuffle chain)
    double best = cval[buf * 16];
    int bj = cidx[buf * 16];
#pragma unroll
    for (int c = 1; c < 16; ++c) {
      const double ob = cval[buf * 16 + c];
      const int oj = cidx[buf * 16 + c];
      if (ob > best || (ob == best && oj < bj)) { best = ob; bj = oj; }
    }
    if (!(best > thr) || bj >= l) break;  // uniform across the block
    const int p = bj;
    const double rinv = rsqrt(best);
    const double rkk = best * rinv;
    if (ty == (p & 15)) {
      const int ap = p >> 4;
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        const int c = tx + 16 * b;
        if (c < l) {
          double spb = S[0][b];
#pragma unroll
          for (int a = 1; a < 8; ++a)
            if (a == ap) spb = S[a][b];
          R[(size_t)k * l + c] = (c == p) ? rkk : (dn[c] ? 0.0 : spb * rinv);
        }
      }
    }
    if (tid == 0) {
      piv[k] = p;
      ipiv[p] = k;
      dn[p] = 1;  // (the row writers above read dn[c != p] only)
    }
    __syncthreads();  // S2: R row k and dn[p] visible
    double ri[8], rc[8];
#pragma unroll
    for (int a = 0; a < 8; ++a) {
      const int i = ty + 16 * a;
      ri[a] = (i < l) ? R[(size_t)k * l + i] : 0.0;
    }
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const int c = tx + 16 * b;
      rc[b] = (c < l) ? R[(size_t)k * l + c] : 0.0;
    }
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
      for (int b = 0; b < 8; ++b) S[a][b] = fma(-ri[a], rc[b], S[a][b]);
  }
  if (tid == 0) s_sh = k;
  __syncthreads();
  const int s = s_sh;

  if (MODE == SM2_ORTH) {
    // T~ = R~^{-1}, R~[t][j] = R[t][piv_j] (upper triangular, s x s), by 16 x 16
    // blocks: (1) the diagonal blocks, one warp each (lane = column, back
    // substitution); (2) block diagonals d = 1..: T~_IJ = -T~_II sum_{I<t<=J}
    // R~_It T~_tJ, one element per thread of the 16 x 16 grid. Packed storage.
    const int nb = (s + 15) >> 4;
    for (int I = warp; I < nb; I += SM2_THREADS / 32) {
      const int j = 16 * I + (lane & 15);
      if (lane < 16 && j < s) {
        const int i0 = 16 * I;
        for (int i = j; i >= i0; --i) {  // T~[i][j], i = j .. i0 within the block
          double u = (i == j) ? 1.0 : 0.0;
          for (int t = i + 1; t <= j; ++t) u = fma(-R[(size_t)i * l + piv[t]], Tt[pk_col(t, j)], u);
          Tt[pk_col(i, j)] = u / R[(size_t)i * l + piv[i]];
        }
      }
    }
    __syncthreads();
    for (int d = 1; d < nb; ++d) {
      for (int I = 0; I + d < nb; ++I) {
        const int J = I + d;
        const int a = ty, b = tx;          // element (16I + a, 16J + b)
        const int gi = 16 * I + a, gj = 16 * J + b;
        double w = 0.0;
        if (gi < s && gj < s) {
          // W[a][b] = sum_{t = 16(I+1)}^{gj} R~[gi][t] T~[t][gj]
          for (int t = 16 * (I + 1); t <= gj; ++t) w = fma(R[(size_t)gi * l + piv[t]], Tt[pk_col(t, gj)], w);
        }
        __syncthreads();
        // stash W in the (still unused) block (I, J) of T~, then multiply by T~_II
        if (gi < s && gj < s) Tt[pk_col(gi, gj)] = w;
        __syncthreads();
        double v = 0.0;
        if (gi < s && gj < s) {
          const int i1 = min(16 * I + 16, s);
          for (int t = gi; t < i1; ++t) v = fma(Tt[pk_col(gi, t)], Tt[pk_col(t, gj)], v);
        }
        __syncthreads();
        if (gi < s && gj < s) Tt[pk_col(gi, gj)] = -v;
        __syncthreads();
      }
    }
    for (int idx = tid; idx < l * l; idx += SM2_THREADS) {
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
  constexpr int NW = SM2_THREADS / 32;
  int sweep = 0;
  bool converged = (s <= 1);
  for (sweep = 0; sweep < max_sweeps && !converged; ++sweep) {
    for (int c = warp; c < s; c += NW) {  // exact column norms at the start of each sweep
      double a2 = 0.0;
      for (int i = lane; i < l; i += 32) {
        const double x = R[(size_t)c * l + i];
        a2 = fma(x, x, a2);
      }
      a2 = warp_sum(a2);
      if (lane == 0) nrm[c] = a2;
    }
    __syncthreads();
    int rotated = 0;
    for (int rnd = 0; rnd < L2 - 1; ++rnd) {
      // each warp handles 4 disjoint pairs at once (independent dependency
      // chains: loads, warp reductions and rotation parameters interleave)
      for (int q0 = warp * 4; q0 < h; q0 += NW * 4) {
        int P1[4], P2[4];
        bool ok[4];
        double xv[4][4], yv[4][4], g[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int q = q0 + j;
          // circle method: position 0 fixed, positions 1..L2-1 rotate by rnd
          int p1 = 0, p2;
          if (q > 0) {
            p1 = q - 1 + rnd;
            if (p1 >= L2 - 1) p1 -= L2 - 1;
            ++p1;
          }
          p2 = L2 - 2 - q + rnd;
          if (p2 >= L2 - 1) p2 -= L2 - 1;
          ++p2;
          if (p1 > p2) { const int t = p1; p1 = p2; p2 = t; }
          ok[j] = (q < h) && (p2 < s);
          P1[j] = ok[j] ? p1 : 0;
          P2[j] = ok[j] ? p2 : 0;
          g[j] = 0.0;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int i = lane + 32 * e;
            xv[j][e] = (ok[j] && i < l) ? R[(size_t)P1[j] * l + i] : 0.0;
            yv[j][e] = (ok[j] && i < l) ? R[(size_t)P2[j] * l + i] : 0.0;
            g[j] = fma(xv[j][e], yv[j][e], g[j]);
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
          for (int j = 0; j < 4; ++j) g[j] += __shfl_xor_sync(0xffffffffu, g[j], o);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (!ok[j]) continue;
          const double al = nrm[P1[j]], be = nrm[P2[j]];
          const double gj = g[j];
          if (gj * gj > jtol * jtol * al * be && fabs(gj) > 1e-300) {
            // t = tan(theta) solving t^2 + 2 zeta t - 1 = 0, zeta = (be - al) / (2 g):
            // t = sgn(u) g / (|u| + sqrt(u^2 + g^2)), u = (be - al)/2 (one sqrt, one divide)
            const double u = 0.5 * (be - al);
            const double den = fabs(u) + sqrt(fma(u, u, gj * gj));
            const double t = (u >= 0.0 ? gj : -gj) / den;
            const double cs = rsqrt(fma(t, t, 1.0)), sn = cs * t;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int i = lane + 32 * e;
              if (i < l) {
                R[(size_t)P1[j] * l + i] = cs * xv[j][e] - sn * yv[j][e];
                R[(size_t)P2[j] * l + i] = sn * xv[j][e] + cs * yv[j][e];
              }
            }
            if (lane == 0) {  // exact for the (c, s) actually applied
              const double c2 = cs * cs, s2 = sn * sn, cs2 = 2.0 * cs * sn * gj;
              nrm[P1[j]] = fma(c2, al, fma(s2, be, -cs2));
              nrm[P2[j]] = fma(s2, al, fma(c2, be, cs2));
            }
            rotated = 1;
          }
        }
      }
      __syncthreads();
    }
    converged = !__syncthreads_or(rotated);
  }
  // sigma_k = ||m_k||, U_B(:, k) = m_k / sigma_k, sorted descending
  for (int c = warp; c < s; c += NW) {
    double a2 = 0.0;
    for (int i = lane; i < l; i += 32) {
      const double x = R[(size_t)c * l + i];
      a2 = fma(x, x, a2);
    }
    a2 = warp_sum(a2);
    if (lane == 0) nrm[c] = sqrt(a2);
  }
  __syncthreads();
  for (int c = s + warp; c < l; c += NW) {
    if (lane == 0) sigma[c] = 0.0;
    for (int i = lane; i < l; i += 32) UB[i + (size_t)c * l] = 0.0;
  }
  for (int c = warp; c < s; c += NW) {
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
