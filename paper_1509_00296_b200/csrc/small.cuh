// Small-matrix and elementwise kernels of libfrsvt (sm_100a).
//   omega_kernel     : Gaussian test matrix Omega
//   shrink_kernel    : thresholds t_i, d_i = max(sigma_i - t_i, 0), kept set,
//                      the l x l factors of Eq. (6)
//   reductions, ALM init, split-K reduce.
#pragma once
#include "common.cuh"

namespace frsvt {

// ---- Philox4x32-10 + Box-Muller (same stream layout as synth/philox.py) ----
__device__ __forceinline__ void philox10(uint32_t& c0, uint32_t& c1, uint32_t& c2, uint32_t& c3,
                                         uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
  }
}
__device__ __forceinline__ double u53(uint32_t x0, uint32_t x1) {
  return ((double)(x0 >> 5) * 67108864.0 + (double)(x1 >> 6)) * (1.0 / 9007199254740992.0);
}
__device__ __forceinline__ double philox_normal(uint64_t seed, uint32_t stream, uint64_t e) {
  const uint64_t t = e >> 1;
  uint32_t c0 = (uint32_t)t, c1 = (uint32_t)(t >> 32), c2 = stream, c3 = 0u;
  philox10(c0, c1, c2, c3, (uint32_t)seed, (uint32_t)(seed >> 32));
  const double ua = u53(c0, c1), ub = u53(c2, c3);
  const double rad = sqrt(-2.0 * log1p(-ua));
  const double ang = 6.283185307179586 * ub;
  return (e & 1) ? rad * sin(ang) : rad * cos(ang);
}

// Omega' (n x l, ld n): columns [r, r+p) hold columns [0, p) of Omega of this
// call (p = l - r, RP reading Z6), columns < r are zero so that
// A * Omega' + Q~ = [Q~ | A Omega_p]. r = 0 without a carry. With front != 0
// the p fresh columns sit at [0, p) instead (the stream-K sketch multiplies
// only them and writes them behind the carried columns). pmax_dev (nullable,
// adaptive rank prediction P:204-215): at most *pmax_dev fresh columns, the
// rest zero (a zero sample is dropped by the rank reveal, so the basis has
// r + p columns: the sketch width of Eq. (7)). tf32 (fp32 only,
// FRSVT_OPT_TF32_OMEGA): drawn entries rounded to tf32 (rna).
template <typename T>
__global__ void omega_kernel(T* __restrict__ Om, int64_t n, int l, const int* __restrict__ r_dev,
                             int use_r, uint64_t seed, uint32_t stream,
                             const T* __restrict__ override_om, int64_t ldo, int front = 0,
                             const int* __restrict__ pmax_dev = nullptr, int tf32 = 0) {
  const int r = use_r ? *r_dev : 0;
  const int p = pmax_dev ? min(l - r, max(*pmax_dev, 0)) : l - r;
  const int64_t total = n * (int64_t)l;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx % n;
    const int c = (int)(idx / n);
    T v = T(0);
    if (front ? (c < p) : (c >= r && c < r + p)) {
      const int src = front ? c : c - r;
      if (override_om) v = override_om[i + src * ldo];
      else {
        v = (T)philox_normal(seed, stream, (uint64_t)src * (uint64_t)n + (uint64_t)i);
        if constexpr (sizeof(T) == 4) {  // FRSVT_OPT_TF32_OMEGA: rna to tf32
          if (tf32) v = __uint_as_float((__float_as_uint((float)v) + 0x1000u) & 0xFFFFE000u);
        }
      }
    }
    Om[idx] = v;
  }
}

// ---- narrow apply: Out (rows x ncols) = In (rows x l) M, l <= 16 -----------
// M l x l column-major (ld l) in shared memory, one thread per row, FMA in T
// (a tensor-core pass with K = l would spend its ~10 us of fixed set-up on a
// 2 x rows x l x 4-byte stream). r_dev (range propagation, in place, reading
// R11): columns [r, l) of Out = In Tp[:, 0 .. l-r), columns < r untouched.
constexpr int AR_LMAX = 16;
template <typename T, int L>
__global__ void __launch_bounds__(128) apply_rows_kernel(const T* __restrict__ In, int64_t ldin, int64_t rows, int l,
                                                         const T* __restrict__ M, T* Out, int64_t ldout,
                                                         const int* __restrict__ r_dev) {
  __shared__ T sM[L * L];  // zero padded to L x L, row k = M[k, :]
  for (int idx = threadIdx.x; idx < L * L; idx += blockDim.x) {
    const int k = idx / L, c = idx % L;
    sM[idx] = (k < l && c < l) ? M[k + c * l] : T(0);
  }
  __syncthreads();
  const int rsh = r_dev ? min(max(*r_dev, 0), l) : 0;
  const int nact = l - rsh;
  // one row per thread (grid = rows / 128): no row loop, so the compiler keeps
  // sM in shared memory instead of hoisting all L^2 values into registers
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= rows) return;
  T v[L];
#pragma unroll
  for (int k = 0; k < L; ++k) v[k] = k < l ? In[i + (int64_t)k * ldin] : T(0);
#pragma unroll
  for (int c = 0; c < L; ++c) {
    T acc = T(0);
#pragma unroll
    for (int k = 0; k < L; ++k) acc = fma(v[k], sM[k * L + c], acc);
    if (c < nact) Out[i + (int64_t)(rsh + c) * ldout] = acc;
  }
}

// ---- split-K reduction (fixed order => deterministic) ----------------------
template <typename Tp, typename Tout>
__global__ void splitk_reduce_kernel(const Tp* __restrict__ part, int S, int M, int N,
                                     Tout* __restrict__ C, int64_t ldc) {
  const int64_t MN = (int64_t)M * N;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < MN;
       idx += (int64_t)gridDim.x * blockDim.x) {
    Tp s = Tp(0);
    for (int z = 0; z < S; ++z) s += part[z * MN + idx];
    const int i = (int)(idx % M), j = (int)(idx / M);
    C[i + (int64_t)j * ldc] = (Tout)s;
  }
}

// split-K reduction for few outputs / many partials: each block owns 32
// consecutive outputs, its 8 warps stride over z (coalesced 128-byte rows),
// a fixed-order shared-memory fold => deterministic.
template <typename Tp, typename Tout>
__global__ void __launch_bounds__(256) splitk_reduce_wide_kernel(const Tp* __restrict__ part, int S, int M, int N,
                                                                 Tout* __restrict__ C, int64_t ldc) {
  __shared__ double acc[8][33];
  const int64_t MN = (int64_t)M * N;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t idx = (int64_t)blockIdx.x * 32 + lane;
  double s = 0.0;
  if (idx < MN)
    for (int z = warp; z < S; z += 8) s += (double)part[z * MN + idx];
  acc[warp][lane] = s;
  __syncthreads();
  if (warp == 0 && idx < MN) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += acc[w][lane];
    const int i = (int)(idx % M), j = (int)(idx / M);
    C[i + (int64_t)j * ldc] = (Tout)t;
  }
}


// ---- shrinkage and the l x l factors of Eq. (6) ----------------------------
// wmode: 0 tau (scalar: tau_dev ? *tau_dev : tau), 1 explicit w (device, l),
//        2 reciprocal C/(sigma+eps), 3 reweighted C/(d_prev+eps) (falls back
//        to 2 when no previous call).
// Kept set K = {i : d_i > 0} (compacted, ascending). Outputs (ld l):
//   Mc[:, j] = U_B[:, K_j]            (carry Q~ = Q Mc, Alg. 1 line 21)
//   Mp[:, j] = U_B[:, K_j] * d_{K_j}/sigma_{K_j}   (so Wt = B^T Mp = V_K diag(d))
// and the report vector rep = {sigma[l], d[l]}; ints {r, flags}.
template <typename Tq>
__global__ void shrink_kernel(const double* __restrict__ sigma, const double* __restrict__ UB,
                              int l, const int* __restrict__ s_dev, int wmode, double tau,
                              const double* __restrict__ tau_dev, const double* __restrict__ w,
                              double C, double eps, double* __restrict__ d_prev, int* have_prev,
                              Tq* __restrict__ Mc, Tq* __restrict__ Mp, int* __restrict__ r_dev,
                              int* __restrict__ flags, double* __restrict__ rep, int keep = 0) {
  // keep (wmode 0): partial SVT, the first `keep` singular values are not
  // thresholded (t_i = 0, the truncated nuclear norm of Type B)
  __shared__ double d_sh[FRSVT_LMAX], f_sh[FRSVT_LMAX];
  __shared__ int kept[FRSVT_LMAX];
  __shared__ int r_sh;
  const int tid = threadIdx.x;
  const int s = *s_dev;
  const int prev_ok = *have_prev;
  for (int i = tid; i < l; i += blockDim.x) {
    const double sg = sigma[i];
    double t;
    if (wmode == 0) t = i < keep ? 0.0 : (tau_dev ? *tau_dev : tau);
    else if (wmode == 1) t = w[i];
    else if (wmode == 3 && prev_ok) t = C / (d_prev[i] + eps);
    else t = C / (sg + eps);
    double d = (i < s) ? fmax(sg - t, 0.0) : 0.0;
    if (!isfinite(d)) d = 0.0;
    d_sh[i] = d;
    f_sh[i] = (d > 0.0 && sg > 0.0) ? d / sg : 0.0;
    rep[i] = sg;
    rep[FRSVT_LMAX + i] = d;
    if (wmode == 1 && i + 1 < l && w[i + 1] < w[i]) atomicOr(flags, FLAG_NONMONOTONE_W);
  }
  __syncthreads();
  if (tid == 0) {
    int r = 0;
    for (int i = 0; i < l; ++i)
      if (d_sh[i] > 0.0) kept[r++] = i;
    r_sh = r;
    *r_dev = r;
    *have_prev = 1;
  }
  __syncthreads();
  for (int i = tid; i < l; i += blockDim.x) d_prev[i] = d_sh[i];
  const int r = r_sh;
#pragma unroll 4
  for (int idx = tid; idx < l * l; idx += blockDim.x) {
    const int row = idx % l, j = idx / l;
    double vc = 0.0, vp = 0.0;
    if (j < r) {
      const int src = kept[j];
      vc = UB[row + (int64_t)src * l];
      vp = vc * f_sh[src];
    }
    Mc[idx] = (Tq)vc;
    Mp[idx] = (Tq)vp;
  }
}

// ---- reductions over an m x n column-major matrix --------------------------
// (4 consecutive rows per thread when the layout allows 16-byte loads)
template <typename T>
__global__ void absmax_sumsq_kernel(const T* __restrict__ X, int64_t m, int64_t n, int64_t ld,
                                    double* __restrict__ part_max, double* __restrict__ part_ss) {
  __shared__ double scratch[32];
  double mx = 0.0, ss = 0.0;
  const bool vec = sizeof(T) == 4 && (m % 4) == 0 && (ld % 4) == 0 && ((uintptr_t)X % 16) == 0;
  if (vec) {
    const int64_t m4 = m / 4, total = m4 * n;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
      const int64_t i4 = idx % m4, j = idx / m4;
      const float4 v = __ldcs(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(X) + j * ld) + i4);
      mx = fmax(mx, fmax(fmax(fabs((double)v.x), fabs((double)v.y)), fmax(fabs((double)v.z), fabs((double)v.w))));
      ss += (double)v.x * v.x + (double)v.y * v.y + (double)v.z * v.z + (double)v.w * v.w;
    }
  } else {
    const int64_t total = m * n;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
      const int64_t i = idx % m, j = idx / m;
      const double v = (double)X[i + j * ld];
      mx = fmax(mx, fabs(v));
      ss += v * v;
    }
  }
  const double bm = block_max(mx, scratch);
  const double bs = block_sum(ss, scratch);
  if (threadIdx.x == 0) { part_max[blockIdx.x] = bm; part_ss[blockIdx.x] = bs; }
}

// single block: fold partial maxima / sums (fixed order)
__global__ void fold_kernel(const double* __restrict__ part_max, const double* __restrict__ part_ss,
                            int nparts, double* __restrict__ out_max, double* __restrict__ out_ss) {
  __shared__ double scratch[32];
  double mx = 0.0, ss = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) {
    if (part_max) mx = fmax(mx, part_max[i]);
    if (part_ss) ss += part_ss[i];
  }
  mx = block_max(mx, scratch);
  ss = block_sum(ss, scratch);
  if (threadIdx.x == 0) {
    if (out_max) *out_max = mx;
    if (out_ss) *out_ss = ss;
  }
}

// ALM scalars after the init reductions:
//   norm2 = supplied or sqrt(lambda_max) of the block-power estimate,
//   mu0 = supplied or 1.25/norm2, mu_bar = factor*mu0,
//   J = max(norm2, ||D||_inf / lambda); scal = {mu0, mu_bar, 1/J, norm2, ||D||_F^2 ...}
__global__ void alm_scalars_kernel(double norm2_supplied, const double* __restrict__ sigma_est,
                                   double mu0_supplied, double mu_factor, double lambda,
                                   const double* __restrict__ dmax, double* __restrict__ mu,
                                   double* __restrict__ scal) {
  const double n2 = norm2_supplied > 0.0 ? norm2_supplied : sigma_est[0];
  const double mu0 = mu0_supplied > 0.0 ? mu0_supplied : 1.25 / n2;
  mu[0] = mu0;
  mu[1] = mu_factor * mu0;
  const double J = fmax(n2, *dmax / lambda);
  scal[0] = 1.0 / J;
  scal[1] = n2;
}

// E_1 = S_{lambda/mu_0}(D + Y_0/mu_0), A_1 = D - E_1 + Y_0/mu_0 with Y_0 = D/J
// (L_0 = E_0 = 0).
template <typename T>
__global__ void alm_init_kernel(const T* __restrict__ D, T* __restrict__ E, T* __restrict__ A,
                                int64_t m, int64_t n, int64_t ld, const double* __restrict__ mu,
                                const double* __restrict__ scal, double lambda) {
  const double mu0 = mu[0];
  const T yscale = (T)(scal[0] / mu0);  // (1/J)/mu0
  const T thr = (T)(lambda / mu0);
  const bool vec = sizeof(T) == 4 && (m % 4) == 0 && (ld % 4) == 0 && ((uintptr_t)D % 16) == 0 &&
                   ((uintptr_t)E % 16) == 0 && ((uintptr_t)A % 16) == 0;
  if (vec) {
    const int64_t m4 = m / 4, total = m4 * n;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
      const int64_t o = (idx % m4) * 4 + (idx / m4) * ld;
      const float4 d = __ldcs(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(D) + o));
      float4 e, a;
      const float ys = (float)yscale, th = (float)thr;
      e.x = soft<float>(d.x + d.x * ys, th); a.x = d.x - e.x + d.x * ys;
      e.y = soft<float>(d.y + d.y * ys, th); a.y = d.y - e.y + d.y * ys;
      e.z = soft<float>(d.z + d.z * ys, th); a.z = d.z - e.z + d.z * ys;
      e.w = soft<float>(d.w + d.w * ys, th); a.w = d.w - e.w + d.w * ys;
      __stcs(reinterpret_cast<float4*>(reinterpret_cast<float*>(E) + o), e);
      __stcs(reinterpret_cast<float4*>(reinterpret_cast<float*>(A) + o), a);
    }
    return;
  }
  const int64_t total = m * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = (idx % m) + (idx / m) * ld;
    const T d = D[o];
    const T y = d * yscale;
    const T e = soft<T>(d + y, thr);
    E[o] = e;
    A[o] = d - e + y;
  }
}

// after the fused ALM epilogue: fold the residual partials (local sum)
__global__ void fold_sum_kernel(const double* __restrict__ part, int nparts, double* __restrict__ out) {
  __shared__ double scratch[32];
  double ss = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) ss += part[i];
  ss = block_sum(ss, scratch);
  if (threadIdx.x == 0) *out = ss;
}

// relative residual ||D - L - E||_F / ||D||_F and mu_{k+1} = min(rho mu_k, mu_bar)
__global__ void alm_mu_kernel(double rho, int finalize, double* __restrict__ mu,
                              const double* __restrict__ dss, double* __restrict__ resid) {
  resid[1] = sqrt(resid[0] / fmax(*dss, 1e-300));
  if (!finalize) mu[0] = fmin(rho * mu[0], mu[1]);
}

// tau = 1/mu (device) for the SVT of the ALM step
__global__ void tau_from_mu_kernel(const double* __restrict__ mu, double* __restrict__ tau) {
  *tau = 1.0 / mu[0];
}

}  // namespace frsvt
