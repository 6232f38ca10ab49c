// Small SVD of B from its l x l fp64 Gram G = B B^T (Alg. 1 lines 16-18,
// reading Z8): a single-CTA one-sided (Hestenes) Jacobi on the columns of G
// itself, register resident.
//
// G is symmetric positive semidefinite, so a rotation sequence V that makes
// the columns of M = G V mutually orthogonal gives G V = V Lambda: the
// column norms are lambda_i = sigma_i(B)^2 and the normalised columns are the
// left singular vectors U_B. (The Gram already carries the squared condition
// number; factoring it first, e.g. by Cholesky, adds no accuracy and costs a
// serial l-step phase, so the sweep runs on G directly.)
//
// Parallel ordering: the round-robin "circle" tournament on L2 (even) column
// positions, L2 - 1 rounds per sweep, L2/2 disjoint pairs per round: T[0]
// stays, the ring T[1] -> ... -> T[h-1] -> B[h-1] -> ... -> B[0] -> T[1]
// advances one position per round, and pair q is (T[q], B[q]). Column c >= 1
// starts at ring index c - 1, so the column in every slot at every round is
// a closed form (eig_col_at). Warp w owns the 8 pairs q = 8w .. 8w + 7; lane
// j holds rows j, j+32, j+64, j+96 of its 16 columns in registers (8 warps of
// up to 255 registers at l = 120: fewer warps issuing the per-round parameter
// chain than 4 pairs per warp on 15 warps). Advancing the ring is a register
// renaming inside a warp (eig_round); only two columns per warp cross to a
// neighbour warp, through a double-buffered shared-memory mailbox (one block
// barrier per round).
//
// Per round and warp: 8 partial dots, a reduce-scatter that leaves the dot of
// pair p in lanes 4p .. 4p+3, the rotation parameters of the 8 pairs computed
// lane-parallel (branch-free), then the rotations. Rotations are applied in scaled form
// (column c is stored as x~ with true column d_c x~): x~' = x~ - a y~,
// y~' = y~ + b x~ with a = t d_y / d_x, b = t d_x / d_y, d' = c d — two FMAs
// per element pair instead of four. The per-column metadata (true squared
// norm, d, 1/d) lives in shared memory indexed by column, so it never moves.
// Scales are folded back into the data at the start of every sweep, where the
// norms are also recomputed exactly.
//
// A pair rotates when |g| > tol_rot sqrt(|m_p|^2 |m_q|^2), g = m_p . m_q.
// The solve stops after a sweep with no rotation, or (tol_stop > 0) after a
// sweep whose largest measured off-diagonal was <= tol_stop, measured as
// g^2 / (|m_p|^2 |m_q|^2) (relative to both columns), except for a pair whose
// smaller column is clearly below the scalar threshold t (sigma < t/2,
// t_mode != 0): there g^2 / max(|m_p|^2, |m_q|^2)^2. With m = G v ~ lambda v,
// an unresolved g perturbs the pair's eigenvectors by ~g / (lambda_p^2 -
// lambda_q^2), which both measures bound, and over-estimates the smaller
// eigenvalue by ~g^2 / lambda_p^2: relative to a kept eigenvalue that needs the
// two-sided measure, while a clearly sub-threshold one stays below t. So a
// kept column paired with a near-null one (fp32 rounding noise in B once the
// revealed rank drops) no longer holds the solve open. Jacobi sweeps converge
// quadratically: the sweep that measured tol_stop leaves off-diagonals near
// tol_stop^2 (fp32 handles: tol_stop 1e-4).
//
// Exact shortcut (t_mode != 0): if the Gershgorin bound max_i sum_j |G_ij| is
// <= t_min^2, every sigma_i <= t_min and every shrunk value
// max(sigma_i - t_i, 0) is zero, so the thresholded result (X = 0, r = 0) is
// known without the decomposition; sigma then reports sqrt(G_ii) (each
// <= t_min), U_B the matching unit vectors, sweeps 0.
#pragma once
#include "common.cuh"

namespace frsvt {

// pairs per warp: 8 (two renaming halves of 4; 8 warps of up to 255
// registers at l = 120) above l = 40, else 4 (fewer rounds for small l: the
// sweep has 2 * PPW * warps - 1 rounds)
__host__ __device__ constexpr int eig_ppw(int l) { return l > 40 ? 8 : 4; }

struct EigJacobi {
  static int warps(int l) {
    const int per = 2 * eig_ppw(l);
    return (l + per - 1) / per;
  }
  // mailbox [2][nw][2][128] + metadata [128][4] + a/b [nw][PPW][2]
  static size_t smem_bytes(int l) {
    const int nw = warps(l);
    return ((size_t)2 * nw * 2 * 128 + (size_t)FRSVT_LMAX * 4 + (size_t)nw * eig_ppw(l) * 2) * sizeof(double) + 64;
  }
};

__device__ __forceinline__ double eig_rcp_approx(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  return r;
}
__device__ __forceinline__ double eig_rsqrt_approx(double x) {
  double r;
  asm("rsqrt.approx.f64 %0, %1;" : "=d"(r) : "d"(x));
  return r;
}

// column in slot T[q] (top) / B[q] (bottom) at round k
__device__ __forceinline__ int eig_col_at(bool top, int q, int k, int L2) {
  const int R = L2 - 1;
  if (top && q == 0) return 0;
  const int rho = top ? q - 1 : L2 - 2 - q;
  int c = rho - (k % R);
  if (c < 0) c += R;
  return c + 1;
}

// Per-launch state of the round body (see eig_jacobi_kernel).
struct EigRoundCtx {
  double* meta;
  double* abuf;
  double* mbox;
  double tol2, tsmall, tstop2;
  int l, nw, warp, lane, pj, Rr;
  bool b4, b3, b2;
  int rho_x, rho_y;  // ring indices of this lane's parameter pair
  bool bigoff;       // an off-diagonal above tol_stop was measured this sweep
  bool rotated;
  bool precise;      // fp64-level tolerance: c to full precision (two Newton steps)
};

// One round of the sweep at ring phase t (compile time). The PPW top / PPW
// bottom slots of a warp are PPW / 4 halves of 4; inside a half the ring advance
// is a register renaming, not a copy: logical top slot j lives in
// x[(j & 4) + (((j & 3) - t) & 3)] and bottom slot j in
// y[(j & 4) + (((j & 3) + t) & 3)], so per round only the two columns that
// cross between the halves are copied (the round loop is unrolled by 4; the
// sweep ends at phase 3 and is renamed back once). Warp 0 (the fixed column
// T[0]) and the last warp (T[h-1] -> B[h-1]) copy one more column each.
template <int t, int PPW>
__device__ __forceinline__ void eig_round(double (&X)[PPW][4], double (&Y)[PPW][4], EigRoundCtx& c, int rnd) {
  static_assert(PPW == 4 || PPW == 8, "renaming halves of 4 pairs");
  constexpr int H = PPW / 4;
#define XL(j) X[((j) & 4) + ((((j) & 3) - t) & 3)]
#define YL(j) Y[((j) & 4) + ((((j) & 3) + t) & 3)]
  const int lane = c.lane, warp = c.warp;
  // partial dots, then a reduce-scatter: the (32 / PPW)-lane group p ends
  // with the full (stored) dot of pair p
  double gp[PPW];
#pragma unroll
  for (int j = 0; j < PPW; ++j) {
    double s = XL(j)[0] * YL(j)[0];
#pragma unroll
    for (int e = 1; e < 4; ++e) s = fma(XL(j)[e], YL(j)[e], s);
    gp[j] = s;
  }
  double gm;
  if constexpr (PPW == 8) {
    double k4[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      k4[i] = c.b4 ? gp[4 + i] : gp[i];
      k4[i] += __shfl_xor_sync(0xffffffffu, c.b4 ? gp[i] : gp[4 + i], 16);
    }
    double k2[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      k2[i] = c.b3 ? k4[2 + i] : k4[i];
      k2[i] += __shfl_xor_sync(0xffffffffu, c.b3 ? k4[i] : k4[2 + i], 8);
    }
    gm = c.b2 ? k2[1] : k2[0];
    gm += __shfl_xor_sync(0xffffffffu, c.b2 ? k2[0] : k2[1], 4);
  } else {
    double k2[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      k2[i] = c.b4 ? gp[2 + i] : gp[i];
      k2[i] += __shfl_xor_sync(0xffffffffu, c.b4 ? gp[i] : gp[2 + i], 16);
    }
    gm = c.b3 ? k2[1] : k2[0];
    gm += __shfl_xor_sync(0xffffffffu, c.b3 ? k2[0] : k2[1], 8);
    gm += __shfl_xor_sync(0xffffffffu, gm, 4);
  }
  gm += __shfl_xor_sync(0xffffffffu, gm, 2);
  gm += __shfl_xor_sync(0xffffffffu, gm, 1);
  // rotation parameters of pair pj, lane-parallel over the PPW pairs
  {
    const int cx = c.rho_x + 1, cy = c.rho_y + 1;  // column = (ring index - round) mod R, + 1
    if (c.rho_x >= 0) c.rho_x = (c.rho_x == 0) ? c.Rr - 1 : c.rho_x - 1;
    c.rho_y = (c.rho_y == 0) ? c.Rr - 1 : c.rho_y - 1;
    double* meta = c.meta;
    const double2 mx01 = *reinterpret_cast<const double2*>(meta + 4 * cx);
    const double2 my01 = *reinterpret_cast<const double2*>(meta + 4 * cy);
    const double dinx = meta[4 * cx + 2], diny = meta[4 * cy + 2];
    const double al = mx01.x, be = my01.x, dxv = mx01.y, dyv = my01.y;
    const double g = gm * dxv * dyv;  // true dot
    const double abv = al * be, gg = g * g;
    const bool rot = (cx < c.l) && (cy < c.l) && al > 0.0 && be > 0.0 && gg > c.tol2 * abv;
    // branch-free: every lane evaluates the rotation (safe operands where it
    // does not rotate, t = 0 there), so the warp never splits
    // convergence measure (see the header): relative to the larger
    // column when the smaller one is clearly below the threshold
    const double mxn = fmax(al, be);
    const double den = fmin(al, be) >= c.tsmall ? abv : mxn * mxn;
    c.bigoff |= rot && gg > c.tstop2 * den;
    // t = tan(theta) = sgn(zeta) / (|zeta| + sqrt(1 + zeta^2)), zeta = (be - al)/(2g),
    // in fp32 (~1e-7 relative) for |zeta| <= 1e4, else t = 1/(2|zeta|) in fp64
    // (relative error < 1e-8 + that of the approximate reciprocal): any t
    // defines an exact rotation once c, s are consistent with it, an
    // approximate angle only leaves a ~1e-7 fraction of g for the next sweep
    const double zeta = 0.5 * (be - al) * eig_rcp_approx(rot ? g : 1.0);
    const double azd = fabs(zeta);
    const float az = (float)fmin(azd, 1e4);
    const float z1 = fmaf(az, az, 1.0f);
    float tf;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(tf) : "f"(fmaf(z1, rsqrtf(z1), az)));
    const double tt = azd <= 1e4 ? (double)tf : 0.5 * eig_rcp_approx(fmax(azd, 1e4));
    const double tn = rot ? (zeta >= 0.0 ? tt : -tt) : 0.0;
    // c = 1/sqrt(1 + t^2) consistent with t: fp32 seed and one Newton step
    // (~2^-45), a second for fp64 handles (c only scales the column: its error
    // reaches sigma, not U_B)
    const double q1 = fma(tn, tn, 1.0), hq = -0.5 * q1;
    double cs = (double)rsqrtf((float)q1);
    cs = cs * fma(hq * cs, cs, 1.5);
    if (c.precise) cs = cs * fma(hq * cs, cs, 1.5);
    const double sn = cs * tn, ic = q1 * cs;  // ic = 1/c
    const double a = tn * dyv * dinx;
    const double b = tn * dxv * diny;
    c.rotated |= rot;
    if ((lane & (32 / PPW - 1)) == 0) {
      if (rot) {
        const double c2 = cs * cs, s2 = sn * sn, cs2 = 2.0 * cs * sn * g;
        meta[4 * cx + 0] = fma(c2, al, fma(s2, be, -cs2));
        meta[4 * cx + 1] = cs * dxv;
        meta[4 * cx + 2] = ic * dinx;
        meta[4 * cy + 0] = fma(s2, al, fma(c2, be, cs2));
        meta[4 * cy + 1] = cs * dyv;
        meta[4 * cy + 2] = ic * diny;
      }
      c.abuf[(warp * PPW + c.pj) * 2 + 0] = a;
      c.abuf[(warp * PPW + c.pj) * 2 + 1] = b;
    }
  }
  __syncwarp();
#pragma unroll
  for (int j = 0; j < PPW; ++j) {
    const double2 abj = *reinterpret_cast<const double2*>(c.abuf + (warp * PPW + j) * 2);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const double xv = XL(j)[e], yv = YL(j)[e];
      XL(j)[e] = fma(-abj.x, yv, xv);
      YL(j)[e] = fma(abj.y, xv, yv);
    }
  }
  // ---- advance the ring by one position --------------------------------
  // registers of phase t (half hh): top slot 4hh + 3 = X[4hh + ((3 - t) & 3)],
  // top 0 = X[(-t) & 3]; bottom slot 4hh = Y[4hh + (t & 3)]. At phase t + 1
  // the register of old top 4hh + 3 is new top 4hh (<- old top 4hh - 1, or
  // warp - 1 for hh = 0) and that of old bottom 4hh is new bottom 4hh + 3
  // (<- old bottom 4hh + 4, or warp + 1 for the last half).
  constexpr int X3 = (3 - t) & 3, X0 = (0 - t) & 3, Y0 = t & 3;
  constexpr int XL7 = 4 * (H - 1) + X3, YL4 = 4 * (H - 1) + Y0;  // last half's top out / bottom in
  const int nw = c.nw;
  double* mb = c.mbox + (size_t)(rnd & 1) * nw * 2 * 128;
  double x7[4], y0[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    x7[e] = X[XL7][e];
    y0[e] = Y[Y0][e];
  }
  if (warp + 1 < nw) {  // last top slot -> warp + 1
    double* outT = mb + (size_t)(warp * 2 + 0) * 128;
#pragma unroll
    for (int e = 0; e < 4; ++e) outT[32 * e + lane] = x7[e];
  }
  if (warp > 0) {  // first bottom slot -> warp - 1
    double* outB = mb + (size_t)(warp * 2 + 1) * 128;
#pragma unroll
    for (int e = 0; e < 4; ++e) outB[32 * e + lane] = y0[e];
  }
#pragma unroll
  for (int hh = H - 1; hh >= 1; --hh)
#pragma unroll
    for (int e = 0; e < 4; ++e) X[4 * hh + X3][e] = X[4 * (hh - 1) + X3][e];  // top 4hh - 1 -> top 4hh
#pragma unroll
  for (int hh = 0; hh + 1 < H; ++hh)
#pragma unroll
    for (int e = 0; e < 4; ++e) Y[4 * hh + Y0][e] = Y[4 * (hh + 1) + Y0][e];  // bottom 4hh + 4 -> bottom 4hh + 3
  if (warp == 0) {  // T[0] stays, B[0] -> T[1]
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      X[X3][e] = X[X0][e];
      X[X0][e] = y0[e];
    }
  }
  if (warp == nw - 1) {  // T[h-1] -> B[h-1]
#pragma unroll
    for (int e = 0; e < 4; ++e) Y[YL4][e] = x7[e];
  }
  __syncthreads();
  if (warp > 0) {  // new top slot 0 <- warp - 1's last top slot
    const double* inT = mb + (size_t)((warp - 1) * 2 + 0) * 128;
#pragma unroll
    for (int e = 0; e < 4; ++e) X[X3][e] = inT[32 * e + lane];
  }
  if (warp + 1 < nw) {  // new last bottom slot <- warp + 1's first bottom slot
    const double* inB = mb + (size_t)((warp + 1) * 2 + 1) * 128;
#pragma unroll
    for (int e = 0; e < 4; ++e) Y[YL4][e] = inB[32 * e + lane];
  }
#undef XL
#undef YL
}

template <int PPW>
__global__ void __launch_bounds__(PPW == 8 ? 256 : 512, 1)
eig_jacobi_kernel(const double* __restrict__ G, int l, const double* __restrict__ t_dev, double t_host,
                  int t_mode, double tol_rot, double tol_stop, int max_sweeps, double* __restrict__ sigma,
                  double* __restrict__ UB, int* __restrict__ sweeps_out, int* __restrict__ flags,
                  const int* __restrict__ run_if = nullptr) {
  if (run_if && !*run_if) return;  // (warm-start block solve, eig_warm.cuh) not needed
  extern __shared__ double esm[];
  const int nw = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = nw * PPW;  // pairs per round
  const int L2 = 2 * h;    // positions (>= l; columns >= l are empty)
  double* mbox = esm;                                // [2][nw][2][128]
  double* meta = esm + (size_t)2 * nw * 2 * 128;     // [128][4]: N (true |col|^2), d, 1/d, -
  double* abuf = meta + (size_t)FRSVT_LMAX * 4;      // [nw][PPW][2]: a, b of this round
  __shared__ double red_d[16];
  __shared__ int red_i[16];
  __shared__ int stop_sh, early_sh;

  // ---- exact shortcut: Gershgorin bound vs the smallest threshold --------
  double t2 = -1.0;
  if (t_mode == 1) t2 = t_host * t_host;
  if (t_mode == 2) t2 = (*t_dev) * (*t_dev);
  {
    double rs = 0.0;
    int bad = 0;
    for (int c = warp; c < l; c += nw) {
      double a = 0.0;
      for (int i = lane; i < l; i += 32) a += fabs(G[i + (size_t)c * l]);
      a = warp_sum(a);
      rs = fmax(rs, a);
      if (lane == 0 && !isfinite(G[c + (size_t)c * l])) bad = 1;
    }
    if (lane == 0) red_d[warp] = rs;
    if (bad) atomicOr(flags, FLAG_NONFINITE);
    __syncthreads();
    if (threadIdx.x == 0) {
      double mx = 0.0;
      for (int w = 0; w < nw; ++w) mx = fmax(mx, red_d[w]);
      early_sh = (t2 >= 0.0 && mx <= t2) ? 1 : 0;
    }
    __syncthreads();
  }
  if (early_sh) {
    for (int c = threadIdx.x; c < l; c += blockDim.x) {
      const double gc = fmax(G[c + (size_t)c * l], 0.0);
      int rank = 0;
      for (int j = 0; j < l; ++j) {
        const double gj = fmax(G[j + (size_t)j * l], 0.0);
        rank += (gj > gc) || (gj == gc && j < c);
      }
      sigma[rank] = sqrt(gc);
      for (int i = 0; i < l; ++i) UB[i + (size_t)rank * l] = (i == c) ? 1.0 : 0.0;
    }
    if (threadIdx.x == 0) *sweeps_out = 0;
    return;
  }

  // ---- load (round-0 placement of the closed form) ------------------------
  double x[PPW][4], y[PPW][4];  // stored top / bottom slot columns
  const int q0 = warp * PPW;
#pragma unroll
  for (int j = 0; j < PPW; ++j) {
    const int ct = eig_col_at(true, q0 + j, 0, L2), cb = eig_col_at(false, q0 + j, 0, L2);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int i = lane + 32 * e;
      const double vx = (ct < l && i < l) ? G[i + (size_t)ct * l] : 0.0;
      const double vy = (cb < l && i < l) ? G[i + (size_t)cb * l] : 0.0;
      x[j][e] = isfinite(vx) ? vx : 0.0;
      y[j][e] = isfinite(vy) ? vy : 0.0;
    }
  }
  for (int c = threadIdx.x; c < FRSVT_LMAX; c += blockDim.x) {
    meta[4 * c + 0] = 0.0;
    meta[4 * c + 1] = 1.0;
    meta[4 * c + 2] = 1.0;
    meta[4 * c + 3] = 0.0;
  }

  EigRoundCtx ctx;
  ctx.meta = meta;
  ctx.abuf = abuf;
  ctx.mbox = mbox;
  ctx.tol2 = tol_rot * tol_rot;
  ctx.precise = tol_rot < 1e-12;
  // |m|^2 below which a column is clearly under the threshold (sigma < t/2,
  // |G v|^2 = lambda^2 < t^4/16); 0 without a scalar threshold
  ctx.tsmall = t2 > 0.0 ? t2 * t2 * (1.0 / 16.0) : 0.0;
  ctx.tstop2 = tol_stop > 0.0 ? tol_stop * tol_stop : 0.0;
  ctx.l = l;
  ctx.nw = nw;
  ctx.warp = warp;
  ctx.lane = lane;
  ctx.pj = lane / (32 / PPW);  // the pair this lane computes parameters for
  ctx.b4 = (lane & 16) != 0;
  ctx.b3 = (lane & 8) != 0;
  ctx.b2 = (lane & 4) != 0;
  ctx.Rr = L2 - 1;
  int sweep = 0;
  bool converged = false;
  int rnd_base = 0;  // rounds elapsed (ring offset)
  for (; sweep < max_sweeps; ++sweep) {
    __syncthreads();  // metadata of the previous sweep complete
    // fold the scales into the data and recompute exact norms
    {
      double a[2 * PPW];
#pragma unroll
      for (int j = 0; j < PPW; ++j) {
        const int ct = eig_col_at(true, q0 + j, rnd_base, L2), cb = eig_col_at(false, q0 + j, rnd_base, L2);
        const double dxv = meta[4 * ct + 1], dyv = meta[4 * cb + 1];
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          x[j][e] *= dxv;
          y[j][e] *= dyv;
          s0 = fma(x[j][e], x[j][e], s0);
          s1 = fma(y[j][e], y[j][e], s1);
        }
        a[2 * j] = s0;
        a[2 * j + 1] = s1;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int j = 0; j < 2 * PPW; ++j) a[j] += __shfl_xor_sync(0xffffffffu, a[j], o);
      __syncthreads();  // every warp has read the old scales
      if (lane == 0) {
#pragma unroll
        for (int j = 0; j < PPW; ++j) {
          const int ct = eig_col_at(true, q0 + j, rnd_base, L2), cb = eig_col_at(false, q0 + j, rnd_base, L2);
          meta[4 * ct + 0] = ct < l ? a[2 * j] : 0.0;
          meta[4 * ct + 1] = 1.0;
          meta[4 * ct + 2] = 1.0;
          meta[4 * cb + 0] = cb < l ? a[2 * j + 1] : 0.0;
          meta[4 * cb + 1] = 1.0;
          meta[4 * cb + 2] = 1.0;
        }
      }
      __syncthreads();
    }
    ctx.bigoff = false;
    ctx.rotated = false;
    {
      const int pj = ctx.pj, Rr = ctx.Rr, k = rnd_base % Rr;
      int rho_x = (q0 + pj == 0) ? -1 : q0 + pj - 1, rho_y = L2 - 2 - (q0 + pj);
      if (rho_x >= 0) rho_x = (rho_x - k + Rr) % Rr;
      rho_y = (rho_y - k + Rr) % Rr;
      ctx.rho_x = rho_x;
      ctx.rho_y = rho_y;
    }
    // L2 - 1 = 8 nw - 1 rounds = G4 groups of 4, the last one cut after 3
    const int G4 = L2 / 4;
    for (int g4 = 0; g4 < G4; ++g4) {
      const int rnd = rnd_base + 4 * g4;
      eig_round<0, PPW>(x, y, ctx, rnd);
      eig_round<1, PPW>(x, y, ctx, rnd + 1);
      eig_round<2, PPW>(x, y, ctx, rnd + 2);
      if (g4 == G4 - 1) break;
      eig_round<3, PPW>(x, y, ctx, rnd + 3);
    }
    // phase 3 -> 0: in each half, top slot j is x[(j + 1) & 3], bottom slot j is y[(j + 3) & 3]
#pragma unroll
    for (int hh = 0; hh < PPW; hh += 4)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const double x0 = x[hh][e], y3 = y[hh + 3][e];
        x[hh][e] = x[hh + 1][e];
        x[hh + 1][e] = x[hh + 2][e];
        x[hh + 2][e] = x[hh + 3][e];
        x[hh + 3][e] = x0;
        y[hh + 3][e] = y[hh + 2][e];
        y[hh + 2][e] = y[hh + 1][e];
        y[hh + 1][e] = y[hh][e];
        y[hh][e] = y3;
      }
    rnd_base += L2 - 1;
    // ---- sweep verdict -----------------------------------------------------
    const int big = __any_sync(0xffffffffu, ctx.bigoff);
    const int rotated = __any_sync(0xffffffffu, ctx.rotated);
    if (lane == 0) {
      red_i[warp] = rotated | (big << 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int any = 0;
      for (int w = 0; w < nw; ++w) any |= red_i[w];
      stop_sh = !(any & 1) || (tol_stop > 0.0 && !(any & 2));
    }
    __syncthreads();
    if (stop_sh) {
      converged = true;
      ++sweep;
      break;
    }
  }

  // ---- sigma = sqrt(d |x~|), U_B = x~ / |x~|, sorted descending ------------
  __syncthreads();
  double nrm[2 * PPW];
#pragma unroll
  for (int j = 0; j < PPW; ++j) {
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      s0 = fma(x[j][e], x[j][e], s0);
      s1 = fma(y[j][e], y[j][e], s1);
    }
    nrm[j] = s0;
    nrm[PPW + j] = s1;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int j = 0; j < 2 * PPW; ++j) nrm[j] += __shfl_xor_sync(0xffffffffu, nrm[j], o);
  double* lam = mbox;  // reuse the mailbox: lambda per column
  int cols[2 * PPW];
  double lams[2 * PPW];
#pragma unroll
  for (int j = 0; j < 2 * PPW; ++j) {
    const int c = eig_col_at(j < PPW, q0 + (j < PPW ? j : j - PPW), rnd_base, L2);
    cols[j] = c;
    nrm[j] = sqrt(nrm[j]);
    lams[j] = (c < l) ? fabs(meta[4 * c + 1]) * nrm[j] : 0.0;
  }
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int j = 0; j < 2 * PPW; ++j)
      if (cols[j] < l) lam[cols[j]] = lams[j];
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < 2 * PPW; ++j) {
    const int c = cols[j];
    if (c >= l) continue;
    const double lc = lams[j];
    int rank = 0;
    for (int k = lane; k < l; k += 32) {
      const double lk = lam[k];
      rank += (lk > lc) || (lk == lc && k < c);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) rank += __shfl_xor_sync(0xffffffffu, rank, o);
    const double inv = nrm[j] > 0.0 ? 1.0 / nrm[j] : 0.0;
    if (lane == 0) sigma[rank] = sqrt(lc);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int i = lane + 32 * e;
      if (i < l) UB[i + (size_t)rank * l] = ((j < PPW) ? x[j][e] : y[j - PPW][e]) * inv;
    }
  }
  if (threadIdx.x == 0) {
    *sweeps_out = sweep;
    if (!converged) atomicOr(flags, FLAG_NOCONV);
  }
}

// host launcher: the pairs-per-warp instance of l (eig_ppw), one CTA on st
inline void eig_jacobi_launch(cudaStream_t st, const double* G, int l, const double* t_dev, double t_host, int t_mode,
                              double tol_rot, double tol_stop, int max_sweeps, double* sigma, double* UB,
                              int* sweeps_out, int* flags, const int* run_if = nullptr) {
  const int nw = EigJacobi::warps(l);
  const size_t smem = EigJacobi::smem_bytes(l);
  if (eig_ppw(l) == 8)
    eig_jacobi_kernel<8><<<1, 32 * nw, smem, st>>>(G, l, t_dev, t_host, t_mode, tol_rot, tol_stop, max_sweeps, sigma,
                                                     UB, sweeps_out, flags, run_if);
  else
    eig_jacobi_kernel<4><<<1, 32 * nw, smem, st>>>(G, l, t_dev, t_host, t_mode, tol_rot, tol_stop, max_sweeps, sigma,
                                                     UB, sweeps_out, flags, run_if);
}

}  // namespace frsvt
