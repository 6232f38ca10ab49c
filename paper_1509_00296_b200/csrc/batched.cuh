// Small FRSVT in one CTA (PAPER.md P:23 / P:48:
// WNNM's weighted SVT of many patch-group matrices: per-window
// problems; BASELINE c1: one 200 x 100 fp64 call). ONE CTA per matrix runs the
// whole of Algorithm 1 with A resident in shared memory, so a
// call is one launch and a batch is one launch of `batch` CTAs.
//
// Per matrix (A m x n, T = fp32 or fp64, column-major; l <= 16 padded with
// zero columns to LC in {4, 8, 12, 16}; Omega n x l shared by a batch):
//   Y = A Omega                                   (FMA in T, Alg. 1 line 3)
//   Q = orth(Y)                                   CGS2 in fp64 with rank reveal
//   q x { Z = orth(A^T Q); Q = orth(A Z) }        power iteration (lines 13-15)
//   W = A^T Q  (= B^T)                            (line 16)
//   G = W^T W = B B^T = U_B diag(.) U_B^T         cyclic Jacobi (lines 16-18; reading Z8)
//   sigma_i = || W u_i ||                         (columns of W U_B = V_B Sigma)
//   d_i = max(sigma_i - t_i, 0), t_i = tau or w_i (weighted SVT, fn. 1 P:48)
//   X = (Q U_B diag(d / sigma)) (W U_B)^T         Eq. (6)
//
// Layout: threads own ROWS. Thread t holds rows t, t + 256, ... (RM of them)
// of the current m x LC (Y, Q) or n x LC (Z, W) block in registers, so the
// products are row-parallel FMA streams against a broadcast shared-memory
// row of the small operand, and CGS2 is per-thread partial dot products
// followed by one block reduction per pass. A sits in shared memory
// column-major with an odd leading dimension, so both the row-parallel
// (A X) and the column-parallel (A^T Q) reads are bank-conflict free.
// The LC x LC eigenproblem runs in one warp, lane k holding row k of G and of
// U_B in registers; the round-robin pair schedule is unrolled so every
// register index is static.
#pragma once
#include "common.cuh"
#include "small.cuh"  // philox_normal (the Omega generator)

namespace frsvt {

constexpr int BT_THREADS = 256;
constexpr int BT_WARPS = BT_THREADS / 32;
constexpr int BT_LMAX = 16;

// padded width and rows per thread (0: the problem does not fit the design)
__host__ __device__ inline int bt_lc(int l) { return l <= 4 ? 4 : l <= 8 ? 8 : l <= 12 ? 12 : 16; }
__host__ __device__ inline int bt_rm(int64_t m, int64_t n) {
  const int64_t r = m > n ? m : n;
  return r <= BT_THREADS ? 1 : r <= 4 * BT_THREADS ? 4 : 0;
}

// reduction width: LC rounded up to a power of two
__host__ __device__ constexpr int bt_kp(int lc) { return lc <= 4 ? 4 : lc <= 8 ? 8 : 16; }

// shared-memory carve-up (bytes, 16-aligned pieces)
struct BtSmem {
  int lds, lc;
  size_t oA, oQ, oW, oGp, oRed, oV, oMisc, total;
  __host__ __device__ BtSmem(int m, int n, int l, int esz) {
    lc = bt_lc(l);
    lds = m | 1;
    const int kp = bt_kp(lc), ng = lc * (lc + 1) / 2;
    auto al = [](size_t x) { return (x + 15) & ~(size_t)15; };
    oA = 0;
    oQ = al(oA + (size_t)lds * n * esz);                     // m x LC (T), row-major: Q
    oW = al(oQ + (size_t)m * lc * esz);                      // n x LC (T), row-major: Omega, Z, W U_B
    oGp = al(oW + (size_t)n * lc * esz);                     // BT_WARPS x LC (LC + 1) / 2 fp64: Gram partials
    oRed = al(oGp + (size_t)BT_WARPS * ng * 8);              // 2 x (BT_WARPS + 1) x KP fp64: block reductions
    oV = al(oRed + (size_t)2 * (BT_WARPS + 1) * kp * 8);     // LC x LC fp64 (U_B)
    oMisc = al(oV + (size_t)lc * lc * 8);                    // sigma, d/sigma (LC each)
    total = al(oMisc + (size_t)2 * lc * 8);
  }
};

__host__ __device__ inline size_t batched_smem_bytes(int m, int n, int l, int esz = 4) {
  return BtSmem(m, n, l, esz).total;
}

struct BtArgs {
  int m, n, l, q;
  const void* A;
  int64_t lda, strideA;
  const void* Om;         // n x l test matrix; nullptr: drawn in the kernel (om_seed, om_stream)
  int64_t ldo;
  uint64_t om_seed;
  uint32_t om_stream;
  int wmode;
  double tau;
  const double* tau_b;    // per-matrix thresholds (wmode 0, nullable)
  const double* tau_dev;  // one device threshold (wmode 0, nullable)
  const double* w;        // explicit weights by rank position (wmode 1, device)
  void* X;
  int64_t ldx, strideX;
  int* r_b;               // kept rank
  double* sig_b;          // sigma by rank position (l per matrix)
  double* d_b;            // shrunk values by rank position
  int* s_b;               // revealed rank of the sketch
  int* sweeps_b;          // Jacobi sweeps
  double* vs_b;           // residual norm of the last sketch sample (Prop. 4)
  int* flags;             // FLAG_NONFINITE / FLAG_NOCONV (atomicOr; flags_store: written, batch 1)
  int flags_store;
  int stop_after;         // test hook (phase timing): 0 = run everything, k = return after phase k (1..6)
};

// Warp-level transposed reduction of KP values (KP a power of two <= 16):
// at every level each lane keeps half of its values and adds the partner's
// copy of them (KP - 1 shuffles instead of 5 KP); afterwards v[0] of a lane
// holds the warp sum of value bt_tr_idx<KP>(lane).
template <int KP>
__device__ __forceinline__ int bt_tr_idx(int lane) {
  int idx = 0, o = 16;
#pragma unroll
  for (int h = KP / 2; h >= 1; h >>= 1, o >>= 1) idx += (lane & o) ? h : 0;
  return idx;
}
template <int KP>
__device__ __forceinline__ void bt_warp_tr(double (&v)[KP]) {
  const int lane = threadIdx.x & 31;
  int o = 16;
#pragma unroll
  for (int h = KP / 2; h >= 1; h >>= 1, o >>= 1) {
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int k = 0; k < h; ++k) {
      const double send = up ? v[k] : v[k + h];
      const double keep = up ? v[k + h] : v[k];
      v[k] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
#pragma unroll
  for (; o >= 1; o >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
}

// sum over the CTA of v[0..KP) (unused entries zero); every thread gets the
// sums. Two alternating buffers (BT_WARPS partial rows + the final row), so
// reductions may follow each other without an extra barrier.
template <int KP>
__device__ __forceinline__ void bt_reduce(double (&v)[KP], double* red, int& rb) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* part = red + (rb & 1) * (BT_WARPS + 1) * KP;
  double* fin = part + BT_WARPS * KP;
  ++rb;
  bt_warp_tr<KP>(v);
  if ((lane & (32 / KP - 1)) == 0) part[warp * KP + bt_tr_idx<KP>(lane)] = v[0];
  __syncthreads();
  if (warp == 0 && lane < KP) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < BT_WARPS; ++w) s += part[w * KP + lane];
    fin[lane] = s;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < KP; k += 2) {
    const double2 t = *reinterpret_cast<const double2*>(fin + k);
    v[k] = t.x;
    v[k + 1] = t.y;
  }
}

// broadcast load of one LC-wide row of a small operand (T, 16-aligned)
template <typename T, int LC>
__device__ __forceinline__ void bt_row(const T* __restrict__ p, T (&b)[LC]) {
  if constexpr (sizeof(T) == 8) {
#pragma unroll
    for (int c = 0; c < LC; c += 2) {
      const double2 v = *reinterpret_cast<const double2*>(p + c);
      b[c] = v.x;
      b[c + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int c = 0; c < LC; c += 4) {
      const float4 v = *reinterpret_cast<const float4*>(p + c);
      b[c] = v.x;
      b[c + 1] = v.y;
      b[c + 2] = v.z;
      b[c + 3] = v.w;
    }
  }
}

// y (rows tid + 256 r of an m x LC block) = A In, In: n x LC row-major in smem
template <typename T, int LC, int RM>
__device__ __forceinline__ void bt_ax(const T* __restrict__ sA, int lds, int m, int n, const T* __restrict__ sIn,
                                      double (&y)[RM][LC]) {
  T acc[RM][LC];
#pragma unroll
  for (int r = 0; r < RM; ++r)
#pragma unroll
    for (int c = 0; c < LC; ++c) acc[r][c] = T(0);
  const int t = threadIdx.x;
#pragma unroll 2
  for (int j = 0; j < n; ++j) {
    T b[LC];
    bt_row<T, LC>(sIn + (size_t)j * LC, b);
#pragma unroll
    for (int r = 0; r < RM; ++r) {
      const int i = t + r * BT_THREADS;
      const T a = i < m ? sA[i + (size_t)j * lds] : T(0);
#pragma unroll
      for (int c = 0; c < LC; ++c) acc[r][c] = fma(a, b[c], acc[r][c]);
    }
  }
#pragma unroll
  for (int r = 0; r < RM; ++r)
#pragma unroll
    for (int c = 0; c < LC; ++c) y[r][c] = (double)acc[r][c];
}

// z (rows tid + 256 r of an n x LC block) = A^T In, In: m x LC row-major in smem
template <typename T, int LC, int RM>
__device__ __forceinline__ void bt_atx(const T* __restrict__ sA, int lds, int m, int n, const T* __restrict__ sIn,
                                       double (&z)[RM][LC]) {
  T acc[RM][LC];
#pragma unroll
  for (int r = 0; r < RM; ++r)
#pragma unroll
    for (int c = 0; c < LC; ++c) acc[r][c] = T(0);
  const int t = threadIdx.x;
#pragma unroll 2
  for (int i = 0; i < m; ++i) {
    T b[LC];
    bt_row<T, LC>(sIn + (size_t)i * LC, b);
#pragma unroll
    for (int r = 0; r < RM; ++r) {
      const int j = t + r * BT_THREADS;
      const T a = j < n ? sA[i + (size_t)j * lds] : T(0);
#pragma unroll
      for (int c = 0; c < LC; ++c) acc[r][c] = fma(a, b[c], acc[r][c]);
    }
  }
#pragma unroll
  for (int r = 0; r < RM; ++r)
#pragma unroll
    for (int c = 0; c < LC; ++c) z[r][c] = (double)acc[r][c];
}

// Orthonormal columns for the register-resident block y (rows x LC) by
// classical Gram-Schmidt, column by column, re-orthogonalised when needed
// ("twice is enough": a second pass only when the first removed more than
// half of the column's squared norm); a column whose residual is <= tol of its
// original norm is numerically dependent and becomes zero (the rank reveal of
// P:163, reading R4). Columns >= l are zero padding. Returns the kept count;
// *last_nr gets the residual norm of column l - 1 (Prop. 4). One block
// reduction per pass carries (q_k . y for k < j, y . y); the residual norm is
// ||y||^2 - sum_k c_k^2 (the q_k orthonormal).
template <int LC, int RM>
__device__ __forceinline__ int bt_orth(double (&y)[RM][LC], int l, double tol, double* red, int& rb,
                                       double* last_nr) {
  constexpr int KP = bt_kp(LC);
  int kept = 0;
#pragma unroll
  for (int j = 0; j < LC; ++j) {
    if (j >= l) break;
    double n0sq = 0.0, s2 = 0.0;
#pragma unroll
    for (int pass = 0; pass < 2; ++pass) {
      double v[KP];
#pragma unroll
      for (int k = 0; k < KP; ++k) {
        double s = 0.0;
        if (k <= j) {
#pragma unroll
          for (int r = 0; r < RM; ++r) s = fma(y[r][k], y[r][j], s);
        }
        v[k] = s;
      }
      bt_reduce<KP>(v, red, rb);
      // y_j -= sum_{k<j} v_k q_k  (v_j is y_j . y_j)
#pragma unroll
      for (int r = 0; r < RM; ++r)
#pragma unroll
        for (int k = 0; k < j; ++k) y[r][j] = fma(-v[k], y[r][k], y[r][j]);
      s2 = v[j];
#pragma unroll
      for (int k = 0; k < j; ++k) s2 = fma(-v[k], v[k], s2);
      if (pass == 0) n0sq = v[j];
      if (pass == 0 && s2 > 0.5 * n0sq) break;  // little cancellation: one pass suffices
    }
    const double nr = sqrt(fmax(s2, 0.0));
    const double n0 = sqrt(n0sq);
    const bool keep = n0 > 0.0 && nr > tol * n0;
    const double inv = keep ? 1.0 / nr : 0.0;
#pragma unroll
    for (int r = 0; r < RM; ++r) y[r][j] *= inv;
    kept += keep ? 1 : 0;
    if (j == l - 1) *last_nr = nr;
  }
  return kept;
}

// store the register block (rows tid + 256 r < rows) to a row-major LC-wide smem array
template <typename T, int LC, int RM>
__device__ __forceinline__ void bt_store(const double (&y)[RM][LC], int rows, T* __restrict__ s) {
#pragma unroll
  for (int r = 0; r < RM; ++r) {
    const int i = threadIdx.x + r * BT_THREADS;
    if (i < rows) {
#pragma unroll
      for (int c = 0; c < LC; ++c) s[(size_t)i * LC + c] = (T)y[r][c];
    }
  }
}

// Circle-method ring on JC slots (pair q = slots (2q, 2q + 1)): slot 0 stays,
// the others advance T[1] -> T[2] -> ... -> T[h-1] -> B[h-1] -> ... -> B[0] ->
// T[1] (T[q] = slot 2q, B[q] = slot 2q + 1). After JC - 1 rounds every pair
// of columns has met once and the ring is back at its start.
template <int JC, int LC, typename V>
__device__ __forceinline__ void bt_ring(V (&a)[LC]) {
  if constexpr (JC > 2) {
    constexpr int h = JC / 2;
    V o[JC];
#pragma unroll
    for (int k = 0; k < JC; ++k) o[k] = a[k];
#pragma unroll
    for (int q = 1; q < h - 1; ++q) a[2 * (q + 1)] = o[2 * q];
    a[2 * (h - 1) + 1] = o[2 * (h - 1)];
#pragma unroll
    for (int q = 0; q < h - 1; ++q) a[2 * q + 1] = o[2 * (q + 1) + 1];
    a[2] = o[1];
  }
}

// Cyclic Jacobi on the symmetric JC x JC matrix held by one warp (entries
// >= JC are zero padding). Lane k < JC holds row k of G and of U, their
// columns in SLOT order: g[s] = G[k][col(s)], u[s] = U[k][col(s)], U
// starting at I. Pair q of a round is the columns in slots (2q, 2q + 1); the
// slots advance on the circle-method ring after each round (register moves
// with static indices), so the round body is one compact loop iteration. G is
// first scaled by 1 / trace (eigenvectors unchanged; the 1e-17 floor below is
// then relative to the trace). Per round: lane q computes the
// rotation of pair q = (p, p') (p = col(2q)), every lane applies all of them
// to its row's columns (G <- G J, U <- U J), rows p and p' exchange through
// shuffles (G <- J^T G), and the rotated off-diagonal is set to exactly 0. A
// pair rotates while g_pp'^2 > tol^2 |g_pp g_p'p'| and |g_pp'| > 1e-17 (below
// that lies the Gram's own rounding). Returns the sweeps; *conv: a sweep
// without a rotation was reached.
template <int JC, int LC>
__device__ __forceinline__ int bt_jacobi(double (&g)[LC], double (&u)[LC], double tol, bool* conv) {
  constexpr int h = JC / 2;
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  double tr = 0.0;
#pragma unroll
  for (int k = 0; k < JC; ++k) tr += __shfl_sync(full, g[k], k);
  const double sc = tr > 0.0 ? 1.0 / tr : 1.0;
#pragma unroll
  for (int k = 0; k < JC; ++k) g[k] *= sc;
  const double fl = 1e-17, tol2 = tol * tol;
  int colv[LC];
#pragma unroll
  for (int k = 0; k < LC; ++k) colv[k] = k;
  int sweep = 0;
  *conv = false;
  for (; sweep < 30; ++sweep) {
    bool anyl = false;
#pragma unroll 1
    for (int rnd = 0; rnd < JC - 1; ++rnd) {
      // the three entries of pair q, gathered in lane q
      double dg = 0.0, off = 0.0, dq = 0.0;
      int myslot = 0;
#pragma unroll
      for (int q = 0; q < h; ++q) {
        const int p = colv[2 * q], pp = colv[2 * q + 1];
        const double a0 = __shfl_sync(full, g[2 * q], p);
        const double a1 = __shfl_sync(full, g[2 * q + 1], p);
        const double a2 = __shfl_sync(full, g[2 * q + 1], pp);
        if (lane == q) { dg = a0; off = a1; dq = a2; }
        if (lane == p) myslot = 2 * q;
        if (lane == pp) myslot = 2 * q + 1;
      }
      double c = 1.0, s = 0.0;
      bool rot = false;
      if (lane < h && off * off > tol2 * fabs(dg * dq) && fabs(off) > fl) {
        // t = tan(theta), the smaller root of t^2 + 2 zeta t - 1 = 0,
        // zeta = (g_qq - g_pp) / (2 g_pq): t = sgn(zeta) 2|g_pq| / (|dif| + sqrt(dif^2 + 4 g_pq^2))
        const double dif = dq - dg;
        const double sg = ((dif >= 0.0) == (off >= 0.0)) ? 1.0 : -1.0;
        // (IEEE sqrt and division: ~100 and ~80 cycles of latency on B200, less
        // than fp32-seeded Newton sequences with their fp64<->fp32 conversions)
        const double h = sqrt(fma(dif, dif, 4.0 * off * off));
        const double t = sg * 2.0 * fabs(off) / (fabs(dif) + h);
        c = 1.0 / sqrt(fma(t, t, 1.0));
        s = c * t;
        rot = true;
      }
      anyl |= rot;
      // columns: G <- G J, U <- U J; this row's own pair parameters on the way
      double myc = 1.0, mys = 0.0;
      bool myrot = false;
#pragma unroll
      for (int q = 0; q < h; ++q) {
        const double cc = __shfl_sync(full, c, q), ss = __shfl_sync(full, s, q);
        const double gp = g[2 * q], gq = g[2 * q + 1];
        g[2 * q] = cc * gp - ss * gq;
        g[2 * q + 1] = ss * gp + cc * gq;
        const double up = u[2 * q], uq = u[2 * q + 1];
        u[2 * q] = cc * up - ss * uq;
        u[2 * q + 1] = ss * up + cc * uq;
        if ((myslot >> 1) == q) { myc = cc; mys = ss; }
      }
      myrot = __shfl_sync(full, rot ? 1 : 0, myslot >> 1) != 0;
      // rows: G <- J^T G (the row of the slot partner through shuffles)
      int partner = 0;
#pragma unroll
      for (int k = 0; k < JC; ++k)
        if (k == (myslot ^ 1)) partner = colv[k];
      const bool isp = (myslot & 1) == 0;
#pragma unroll
      for (int k = 0; k < JC; ++k) {
        const double o = __shfl_sync(full, g[k], partner);
        g[k] = isp ? (myc * g[k] - mys * o) : (mys * o + myc * g[k]);
      }
      // the rotated pair's off-diagonal is zero by construction
      if (myrot) {
#pragma unroll
        for (int k = 0; k < JC; ++k)
          if (k == (myslot ^ 1)) g[k] = 0.0;
      }
      bt_ring<JC, LC>(g);
      bt_ring<JC, LC>(u);
      bt_ring<JC, LC>(colv);
    }
    if (!__any_sync(full, anyl)) {
      ++sweep;
      *conv = true;
      break;
    }
  }
  return sweep;
}

template <typename T, int LC, int RM>
__global__ void __launch_bounds__(BT_THREADS, 1) batched_frsvt_kernel(BtArgs a) {
  extern __shared__ __align__(16) unsigned char bsm_raw[];
  const int m = a.m, n = a.n, l = a.l;
  const BtSmem L(m, n, l, (int)sizeof(T));
  T* sA = reinterpret_cast<T*>(bsm_raw + L.oA);
  T* sQ = reinterpret_cast<T*>(bsm_raw + L.oQ);
  T* sW = reinterpret_cast<T*>(bsm_raw + L.oW);
  double* sGp = reinterpret_cast<double*>(bsm_raw + L.oGp);
  double* red = reinterpret_cast<double*>(bsm_raw + L.oRed);
  double* sV = reinterpret_cast<double*>(bsm_raw + L.oV);
  double* sg = reinterpret_cast<double*>(bsm_raw + L.oMisc);
  double* fd = sg + LC;
  const int lds = L.lds;
  const int b = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const T* A = reinterpret_cast<const T*>(a.A) + (int64_t)b * a.strideA;
  const T* Om = reinterpret_cast<const T*>(a.Om);
  // a sample whose residual is below this fraction of its norm carries no
  // direction (fp32 data 1e-6, fp64 data 1e-13; reading R4)
  const double tol = sizeof(T) == 4 ? 1e-6 : 1e-13;
  // A into shared memory with asynchronous copies (every element in flight at once)
  for (int idx = tid; idx < m * n; idx += BT_THREADS) {
    const int i = idx % m, j = idx / m;
    const unsigned dst = (unsigned)__cvta_generic_to_shared(sA + i + (size_t)j * lds);
    const T* src = A + i + (int64_t)j * a.lda;
    if constexpr (sizeof(T) == 8)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
    else
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  // Omega (n x l) into sW row-major, zero padded to LC columns (drawn here
  // while A is in flight when no explicit Omega is given: element (j, c) is
  // normal number c n + j of the Philox stream, as omega_kernel)
  for (int idx = tid; idx < n * LC; idx += BT_THREADS) {
    const int j = idx / LC, c = idx % LC;
    T v = T(0);
    if (c < l) v = Om ? Om[j + (int64_t)c * a.ldo] : (T)philox_normal(a.om_seed, a.om_stream, (uint64_t)c * n + j);
    sW[idx] = v;
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  if (a.stop_after == 1) return;
  int rb = 0;
  double vs_raw = 0.0;
  int s_kept = 0;
  double y[RM][LC];
  // phase 0: Q = orth(A Omega); then per power step Z = orth(A^T Q) (odd
  // phases), Q = orth(A Z) (even phases). One call site of the (unrolled)
  // orthonormalisation keeps the kernel's code compact.
#pragma unroll 1
  for (int ph = 0; ph <= 2 * a.q; ++ph) {
    const bool ax = (ph & 1) == 0;
    if (ax) bt_ax<T, LC, RM>(sA, lds, m, n, sW, y);
    else bt_atx<T, LC, RM>(sA, lds, m, n, sQ, y);
    double nr_last = 0.0;
    const int kept = bt_orth<LC, RM>(y, l, tol, red, rb, &nr_last);
    if (ph == 0) vs_raw = nr_last;
    if (ax) {
      s_kept = kept;
      bt_store<T, LC, RM>(y, m, sQ);
    } else {
      bt_store<T, LC, RM>(y, n, sW);
    }
    __syncthreads();
    if (ph == 0 && a.stop_after == 2) return;
  }
  if (a.stop_after == 3) return;
  // W = A^T Q (= B^T) in registers; per-warp partials of G = W^T W (upper
  // triangle, row-major packed, entry e(p, q) = p LC - p (p - 1) / 2 + q - p),
  // 16 entries per transposed warp reduction
  bt_atx<T, LC, RM>(sA, lds, m, n, sQ, y);
  constexpr int NG = LC * (LC + 1) / 2;
  {
    double* gp = sGp + (size_t)warp * NG;
#pragma unroll
    for (int c0 = 0; c0 < NG; c0 += 16) {
      double v[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) v[e] = 0.0;
      int e = 0;
#pragma unroll
      for (int p = 0; p < LC; ++p) {
#pragma unroll
        for (int q2 = p; q2 < LC; ++q2, ++e) {
          if (e >= c0 && e < c0 + 16) {
            double s = 0.0;
#pragma unroll
            for (int r = 0; r < RM; ++r) s = fma(y[r][p], y[r][q2], s);
            v[e - c0] = s;
          }
        }
      }
      bt_warp_tr<16>(v);
      const int eo = c0 + bt_tr_idx<16>(lane);
      if ((lane & 1) == 0 && eo < NG) gp[eo] = v[0];
    }
  }
  __syncthreads();
  if (a.stop_after == 4) return;
  int sweeps = 0;
  bool conv = true;
  if (warp == 0) {
    double g[LC], u[LC];
    const int k = lane < LC ? lane : 0;
#pragma unroll
    for (int c = 0; c < LC; ++c) {
      const int p = k < c ? k : c, q2 = k < c ? c : k;
      const int e = p * LC - p * (p - 1) / 2 + q2 - p;
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < BT_WARPS; ++w) s += sGp[(size_t)w * NG + e];
      g[c] = s;
      u[c] = c == k ? 1.0 : 0.0;
    }
    const double jtol = sizeof(T) == 8 ? 1e-15 : 1e-9;
    // the rounds run over l rounded up to even (JC = LC - 2 when that covers l)
    if constexpr (LC > 4) {
      if (l <= LC - 2) sweeps = bt_jacobi<LC - 2, LC>(g, u, jtol, &conv);
      else sweeps = bt_jacobi<LC, LC>(g, u, jtol, &conv);
    } else {
      if (l <= 2) sweeps = bt_jacobi<2, LC>(g, u, jtol, &conv);
      else sweeps = bt_jacobi<LC, LC>(g, u, jtol, &conv);
    }
    if (lane < LC) {
#pragma unroll
      for (int c = 0; c < LC; ++c) sV[lane * LC + c] = u[c];
    }
  }
  __syncthreads();
  if (a.stop_after == 5) return;
  // W U_B in place (rows in registers), sigma_c = || (W U_B)_c ||
#pragma unroll
  for (int r = 0; r < RM; ++r) {
    double t[LC];
#pragma unroll
    for (int c = 0; c < LC; ++c) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < LC; ++k) s = fma(y[r][k], sV[k * LC + c], s);
      t[c] = s;
    }
#pragma unroll
    for (int c = 0; c < LC; ++c) y[r][c] = t[c];
  }
  {
    constexpr int KP = bt_kp(LC);
    double v[KP];
#pragma unroll
    for (int c = 0; c < KP; ++c) {
      double s = 0.0;
      if (c < LC) {
#pragma unroll
        for (int r = 0; r < RM; ++r) s = fma(y[r][c], y[r][c], s);
      }
      v[c] = s;
    }
    bt_reduce<KP>(v, red, rb);
#pragma unroll
    for (int c = 0; c < LC; ++c)
      if (tid == c) sg[c] = sqrt(v[c]);
  }
  bt_store<T, LC, RM>(y, n, sW);
  __syncthreads();
  if (warp == 0) {
    // thresholds on sigma sorted descending (rank positions; padding sorts
    // last); lane i handles sigma_i
    const int i = lane;
    bool bad = false, pos_ok = false;
    double d = 0.0;
    if (i < LC) {
      const double si = sg[i];
      bad = !isfinite(si);
      int pos = 0;
#pragma unroll
      for (int k = 0; k < LC; ++k) {
        const double sk = sg[k];
        pos += (sk > si) || (sk == si && k < i);
      }
      pos_ok = pos < l;
      double t;
      if (a.wmode == 1) t = pos_ok ? a.w[pos] : 0.0;
      else t = a.tau_b ? a.tau_b[b] : (a.tau_dev ? *a.tau_dev : a.tau);
      d = pos_ok ? fmax(si - t, 0.0) : 0.0;
      fd[i] = (d > 0.0 && si > 0.0) ? d / si : 0.0;
      if (pos_ok) {
        if (a.sig_b) a.sig_b[(int64_t)b * l + pos] = si;
        if (a.d_b) a.d_b[(int64_t)b * l + pos] = d;
      }
    }
    const int r = __popc(__ballot_sync(0xffffffffu, d > 0.0));
    const bool anybad = __any_sync(0xffffffffu, bad);
    if (lane == 0) {
      if (a.r_b) a.r_b[b] = r;
      if (a.s_b) a.s_b[b] = s_kept;
      if (a.vs_b) a.vs_b[b] = vs_raw;
      if (a.sweeps_b) a.sweeps_b[b] = sweeps;
      const int fl = (anybad ? FLAG_NONFINITE : 0) | (conv ? 0 : FLAG_NOCONV);
      if (a.flags && a.flags_store) *a.flags = fl;
      else if (a.flags && fl) atomicOr(a.flags, fl);
    }
  }
  __syncthreads();
  if (a.stop_after == 6) return;
  // X = P (W U_B)^T, P = Q U_B diag(d / sigma); thread = row i of X (coalesced stores)
  T* X = reinterpret_cast<T*>(a.X) + (int64_t)b * a.strideX;
#pragma unroll
  for (int r = 0; r < RM; ++r) {
    const int i = tid + r * BT_THREADS;
    if (i >= m) continue;
    T qrow[LC];
    bt_row<T, LC>(sQ + (size_t)i * LC, qrow);
    T pr[LC];
#pragma unroll
    for (int c = 0; c < LC; ++c) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < LC; ++k) s = fma((double)qrow[k], sV[k * LC + c], s);
      pr[c] = (T)(s * fd[c]);
    }
#pragma unroll 2
    for (int j = 0; j < n; ++j) {
      T wr[LC];
      bt_row<T, LC>(sW + (size_t)j * LC, wr);
      T acc = T(0);
#pragma unroll
      for (int c = 0; c < LC; ++c) acc = fma(pr[c], wr[c], acc);
      X[i + (int64_t)j * a.ldx] = acc;
    }
  }
}

// eligibility of a problem for the one-CTA design
__host__ inline bool bt_fits(int64_t m, int64_t n, int l, int esz) {
  return l >= 1 && l <= BT_LMAX && m >= 1 && n >= 1 && bt_rm(m, n) != 0 &&
         batched_smem_bytes((int)m, (int)n, l, esz) <= 227 * 1024;
}

template <typename T, int LC, int RM>
__host__ inline cudaError_t bt_launch_t(const BtArgs& a, int batch, cudaStream_t st) {
  const size_t smem = batched_smem_bytes(a.m, a.n, a.l, (int)sizeof(T));
  batched_frsvt_kernel<T, LC, RM><<<(unsigned)batch, BT_THREADS, smem, st>>>(a);
  return cudaGetLastError();
}

// launch (the caller checked bt_fits and set the shared-memory attributes)
template <typename T>
__host__ inline cudaError_t bt_launch(const BtArgs& a, int batch, cudaStream_t st) {
  const int lc = bt_lc(a.l);
  const int rm = bt_rm(a.m, a.n);
#define BT_CASE(LCV, RMV) \
  if (lc == LCV && rm == RMV) return bt_launch_t<T, LCV, RMV>(a, batch, st);
  BT_CASE(4, 1) BT_CASE(8, 1) BT_CASE(12, 1) BT_CASE(16, 1)
  BT_CASE(4, 4) BT_CASE(8, 4) BT_CASE(12, 4) BT_CASE(16, 4)
#undef BT_CASE
  return cudaErrorInvalidValue;
}

template <typename T>
__host__ inline cudaError_t bt_set_attrs() {
  const int mx = 227 * 1024;
  cudaError_t e = cudaSuccess;
#define BT_ATTR(LCV, RMV) \
  if (e == cudaSuccess)   \
    e = cudaFuncSetAttribute(batched_frsvt_kernel<T, LCV, RMV>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  BT_ATTR(4, 1) BT_ATTR(8, 1) BT_ATTR(12, 1) BT_ATTR(16, 1)
  BT_ATTR(4, 4) BT_ATTR(8, 4) BT_ATTR(12, 4) BT_ATTR(16, 4)
#undef BT_ATTR
  return e;
}

}  // namespace frsvt
