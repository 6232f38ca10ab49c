// CholeskyQR factor as an explicit triangular T (Y T has orthonormal columns),
// one CTA (8 warps up to l = 64, 16 above), no block barrier per column.
//
// Right-looking elimination of the equilibrated Gram S = D G D (D = diag(dsc),
// dsc_i = G_ii^{-1/2}) with the inverse of the unit lower factor accumulated
// alongside: for pivot k, every entry with row a > k is updated
//   S_ab -= (S_ka / S_kk) S_kb      (a, b > k: Schur complement, kept symmetric)
//   W_ab -= (S_ka / S_kk) W_kb      (b <= k < a, W_kk = 1: W = L^{-1})
// so that S = L diag(d) L^T, R = diag(d)^{1/2} L^T and
//   T = D R^{-1} = D W^T diag(d)^{-1/2}
// without a separate triangular inversion. Row k is only read during step k
// and rows > k are only written, so one barrier per pivot suffices.
//
// Column drop (the rank reveal of QR-CP, reading R4): a
// pivot whose equilibrated Schur diagonal is <= tol (relative to the column's
// own squared norm) eliminates nothing and gets a zero column in T; the other
// columns of T then have zero coefficients on it (W_ic = 0 for dropped c).
//
// Range propagation (reading R11): with r = *r_dev > 0
// the input is Y = [Q~ | Y_p], Q~ (r columns) orthonormal. Its Gram block is
// taken as I, so R12 = G12 = Q~^T Y_p and only the Schur complement
//   S22 = G22 - G12^T G12   (p = l - r, the fresh columns)
// is factored, equilibrated by the fresh columns' own norms (so the drop test
// is relative to |y_j|, as in the full factorisation). The output is the
// l x p apply matrix Tp = [-G12 T22 ; T22] (columns p..l-1 zero):
// Y Tp = (Y_p - Q~ G12) T22 spans the fresh directions (classical Gram-Schmidt
// against Q~ followed by CholeskyQR, P:179 with reading R11); the caller keeps
// Q~ as the first r columns.
#pragma once
#include "common.cuh"

namespace frsvt {

constexpr int CI_THREADS = 512;    // l > 64: 16 warps, 8 x 4 entries each (128 x 128)
constexpr int CI_THREADS_S = 256;  // l <= 64: 8 warps, 8 x 2 entries each (64 x 64)
#ifndef CI_PROF
#define CI_PROF 0  // phase stamps (the test hook's `stamps`): build with -DCI_PROF=1
#endif
constexpr int CI_LD = FRSVT_LMAX + 1;  // row stride (doubles) of the p x p work matrix: odd, so
                                       // column-wise accesses (consecutive rows) are conflict free
constexpr int CI_XMAX = (FRSVT_LMAX / 2 + 1) * (FRSVT_LMAX / 2 + 1);  // r x (p | 1) <= this

__host__ __device__ constexpr size_t chol_inv_smem_bytes() {
  // M (LMAX x CI_LD) + G12 (r x (p | 1) <= CI_XMAX when r, p > 0) + dsc + sd + pivot inverses + ready flags
  return ((size_t)FRSVT_LMAX * CI_LD + (size_t)CI_XMAX + 4 * FRSVT_LMAX + 2) *
         sizeof(double);
}

// Storage during the elimination, M = the p x p work matrix:
//   a, b >= k          : the current Schur complement, both triangles (symmetric)
//   a > b, b < k       : W_ab
//   a < b, a < k       : row a of the Schur complement at its own step (R up to scaling)
// Step k touches only rows a > k, all with one formula (u_a = S_ka / S_kk):
//   M_ab -= u_a M_kb   (b != k: Schur update for b > k, W update for b < k)
//   M_ak  = -u_a       (W_ak; written as M_ak - u_a (S_kk + 1), since M_ak = S_ak = S_ka)
// Thread (warp w, lane L) keeps the TI x TJ entries (w + NW i, L + 32 j) in
// registers. Row k is final once step k - 1 has updated it (later steps touch
// only rows > k), so its owner warp publishes it straight into M (with
// 1 / S_kk) and arrives on a per-row ready mbarrier (release / acquire at CTA
// scope).
// There is no block barrier per pivot: each warp runs the pivots in order,
// waiting only for the flag of the pivot row it needs, and the owner of row
// k + 1 updates that row FIRST at step k (lookahead) and publishes it before
// its bulk update, so the pivot chain costs one row update + one flag hand-off
// per step while the bulk updates of different warps overlap it. (The
// previous design, one block barrier per pivot with the whole update between
// barriers, measured ~600 ns per pivot at l = 120; this one ~480 ns: the
// per-warp instruction issue of the bulk updates, not the hand-off, now bounds
// it.)
// per-row ready signal: an mbarrier of count 1 per row (arrive = release,
// try_wait = acquire at CTA scope); measured on B200 at l = 120: 63 us per
// factor vs 70 us with st.release / ld.acquire flags (a fence per publish)
// 1/x for a pivot x > tol (> 0, finite): rcp.approx seed (~2^-23) and two
// Newton steps (~2^-46 -> below one ulp after the second), shorter on the
// pivot chain than the IEEE division's slow-path-guarded sequence
__device__ __forceinline__ double ci_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  r = fma(r, fma(-x, r, 1.0), r);
  r = fma(r, fma(-x, r, 1.0), r);
  return r;
}

__device__ __forceinline__ void ci_flag_release(uint64_t* f) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"((unsigned)__cvta_generic_to_shared(f))
               : "memory");
}
__device__ __forceinline__ int ci_flag_acquire(uint64_t* f) {
  int v;
  asm volatile(
      "{\n.reg .pred p;\nmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], 0;\nselp.b32 %0, 1, 0, p;\n}"
      : "=r"(v)
      : "r"((unsigned)__cvta_generic_to_shared(f))
      : "memory");
  return v;
}

template <typename Tq, int NW = 16>
__global__ void __launch_bounds__(NW * 32, 1)
chol_inv_kernel(const double* __restrict__ G, int l, const int* __restrict__ r_dev, double tol, Tq* __restrict__ T,
                int64_t ldt, int* __restrict__ s_out, int* __restrict__ flags, const int* __restrict__ skip,
                unsigned long long* __restrict__ prof = nullptr, double* __restrict__ resid_last = nullptr) {
  // resid_last (nullable): ||(I - Q Q^T) y||, y the last nonzero sample and Q
  // a basis of the carry and the samples before it (the
  // by-product behind the Prop. 4 estimate varsigma)
  if (skip && *skip) return;
  // prof (test hook, nullable): %globaltimer at phase boundaries
#define CI_STAMP(q)                                          \
  do {                                                       \
    if (CI_PROF && prof && threadIdx.x == 0) {               \
      unsigned long long t_;                                 \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); \
      prof[q] = t_;                                          \
    }                                                        \
  } while (0)
  CI_STAMP(0);
  extern __shared__ double cis[];
  double* M = cis;                               // p x p (row stride CI_LD)
  double* X = M + (size_t)FRSVT_LMAX * CI_LD;    // G12, r x p row-major (X[c * xld + i], xld = p | 1)
  double* dsc = X + CI_XMAX;
  double* sd = dsc + FRSVT_LMAX;
  double* invp = sd + FRSVT_LMAX;                // 1 / S_kk of each published row (0: dropped)
  uint64_t* rdy = reinterpret_cast<uint64_t*>(invp + FRSVT_LMAX);  // per-row ready mbarriers
  // rows w + NW i, columns L + 32 j: 16 warps 8 x 4 (128 x 128); 8 warps 8 x 2 (64 x 64)
  constexpr int TI = NW == 32 ? 4 : 8, TJ = NW == 8 ? 2 : 4;
  static_assert(NW * TI == FRSVT_LMAX || NW * TI == FRSVT_LMAX / 2, "tile");
  constexpr int NT = NW * 32;
  const int tid = threadIdx.x, w = tid >> 5, L = tid & 31;
  const int r = r_dev ? min(max(*r_dev, 0), l) : 0;
  const int p = l - r;
  const int xld = p | 1;  // odd: the output phase reads X down a column

  // (1) fresh columns' norms, G12, ready flags
  for (int i = tid; i < p; i += NT) {
    const double g = G[(size_t)(r + i) * (l + 1)];
    if (!isfinite(g)) atomicOr(flags, FLAG_NONFINITE);
    dsc[i] = (g > 0.0 && isfinite(g)) ? 1.0 / sqrt(g) : 0.0;
  }
  for (int idx = tid; idx < r * p; idx += NT) {
    const int c = idx % r, i = idx / r;
    X[c * xld + i] = G[c + (size_t)(r + i) * l];
  }
  for (int i = tid; i < FRSVT_LMAX; i += NT)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(rdy + i)) : "memory");
  __syncthreads();
  CI_STAMP(1);
  // (2) equilibrated Schur complement S = D (G22 - G12^T G12) D straight into
  // the register tiles (all of a thread's loads issued together)
  double m[TI][TJ];
#pragma unroll
  for (int i = 0; i < TI; ++i)
#pragma unroll
    for (int j = 0; j < TJ; ++j) {
      const int a = w + NW * i, b = L + 32 * j;
      m[i][j] = (a < p && b < p) ? G[(r + b) + (size_t)(r + a) * l] : 0.0;
    }
  if (r > 0) {
#pragma unroll
    for (int i = 0; i < TI; ++i) {
      const int a = w + NW * i;
      if (a >= p) continue;
#pragma unroll
      for (int j = 0; j < TJ; ++j) {
        const int b = L + 32 * j;
        if (b >= p) continue;
        double s = m[i][j];
        for (int c = 0; c < r; ++c) s = fma(-X[c * xld + a], X[c * xld + b], s);
        m[i][j] = s;
      }
    }
  }
#pragma unroll
  for (int i = 0; i < TI; ++i)
#pragma unroll
    for (int j = 0; j < TJ; ++j) {
      const int a = w + NW * i, b = L + 32 * j;
      double v = (a < p && b < p) ? m[i][j] * (dsc[a] * dsc[b]) : 0.0;
      m[i][j] = isfinite(v) ? v : 0.0;
    }
  CI_STAMP(2);
  // (3) elimination (see above): publish row 0, then the pivots in order
  if (w == 0 && p > 0) {
#pragma unroll
    for (int j = 0; j < TJ; ++j) M[L + 32 * j] = m[0][j];
    if (L == 0) invp[0] = m[0][0] > tol ? ci_rcp(m[0][0]) : 0.0;
    __syncwarp();
    if (L == 0) ci_flag_release(rdy);
  }
  // the last row this warp owns: steps >= it update nothing here
  const int last = w < p ? w + NW * ((p - 1 - w) / NW) : -1;
  for (int k = 0; k < last; ++k) {
    while (ci_flag_acquire(rdy + k) == 0) {
    }
    const double* rk = M + (size_t)k * CI_LD;
    const double inv = invp[k];
    const double d = rk[k];
    double v[TJ];
#pragma unroll
    for (int j = 0; j < TJ; ++j) {
      const int b = L + 32 * j;
      v[j] = (b == k) ? d + 1.0 : rk[b];  // column k: M_ak - u_a (S_kk + 1) = -u_a
    }
    const int k1 = k + 1;
    const bool own1 = (k1 % NW) == w;  // k1 <= last < p
    const int i1 = k1 / NW;
    if (own1) {  // lookahead: row k + 1 first, then publish it
#pragma unroll
      for (int i = 0; i < TI; ++i) {
        if (i != i1) continue;
        if (inv != 0.0) {
          const double u = rk[k1] * inv;
#pragma unroll
          for (int j = 0; j < TJ; ++j) m[i][j] = fma(-u, v[j], m[i][j]);
        } else {
#pragma unroll
          for (int j = 0; j < TJ; ++j)
            if (L + 32 * j == k) m[i][j] = 0.0;
        }
        double* rn = M + (size_t)k1 * CI_LD;
#pragma unroll
        for (int j = 0; j < TJ; ++j) {
          rn[L + 32 * j] = m[i][j];
          if (L + 32 * j == k1) invp[k1] = m[i][j] > tol ? ci_rcp(m[i][j]) : 0.0;
        }
      }
      __syncwarp();
      if (L == 0) ci_flag_release(rdy + k1);
    }
    // bulk: the other rows > k
    if (inv != 0.0) {
#pragma unroll
      for (int i = 0; i < TI; ++i) {
        const int a = w + NW * i;
        if (a > k && a < p && !(own1 && i == i1)) {
          const double u = rk[a] * inv;
#pragma unroll
          for (int j = 0; j < TJ; ++j) m[i][j] = fma(-u, v[j], m[i][j]);
        }
      }
    } else {  // dropped pivot: no elimination, W_ak = 0
#pragma unroll
      for (int i = 0; i < TI; ++i) {
        const int a = w + NW * i;
        if (a > k && a < p) {
#pragma unroll
          for (int j = 0; j < TJ; ++j)
            if (L + 32 * j == k) m[i][j] = 0.0;
        }
      }
    }
  }
  __syncthreads();  // every row published (= its final values) in M
  CI_STAMP(3);
  // (4) T22 (upper, in place of S): T22[c][i] = dsc_c W_ic / sqrt(d_i), kept i
  for (int i = tid; i < p; i += NT) {
    const double d = M[i * CI_LD + i];
    sd[i] = d > tol ? 1.0 / sqrt(d) : 0.0;
  }
  __syncthreads();
  for (int idx = tid; idx < p * p; idx += NT) {
    const int c = idx / p, i = idx - c * p;
    if (i >= c) M[c * CI_LD + i] = dsc[c] * (i == c ? 1.0 : M[i * CI_LD + c]) * sd[i];
  }
  __syncthreads();

  CI_STAMP(4);
  // (5) output, column-major with leading dimension ldt
  for (int idx = tid; idx < l * l; idx += NT) {
    const int j = idx / l, c = idx - j * l;  // T[c + j ldt]: consecutive threads along c
    double v = 0.0;
    if (j < p) {
      if (c >= r) {
        const int cc = c - r;
        v = cc <= j ? M[cc * CI_LD + j] : 0.0;
      } else {
        for (int i = 0; i <= j; ++i) v = fma(-X[c * xld + i], M[i * CI_LD + j], v);
      }
    }
    T[c + (int64_t)j * ldt] = (Tq)v;
  }
  CI_STAMP(5);
#undef CI_STAMP
  if (tid == 0) {
    int s = r;
    for (int i = 0; i < p; ++i) s += (sd[i] > 0.0);
    *s_out = s;
    if (resid_last) {
      double res = 0.0;
      for (int i = p - 1; i >= 0; --i)
        if (dsc[i] > 0.0) {  // the last nonzero sample: its Schur diagonal, unequilibrated
          res = sd[i] > 0.0 ? 1.0 / (sd[i] * dsc[i]) : 0.0;  // sqrt(d) / dsc (a dropped sample: ~0)
          break;
        }
      *resid_last = res;
    }
  }
}

}  // namespace frsvt
