// tcgen05 composition X = Q~ Wt^T (Eq. (6); Alg. 1 line 19)
// for fp32 handles, fused with its consumer:
//   EPI_STORE   : X (m x n) = L                          (frsvt_apply*)
//   EPI_ALM     : the iALM update of rpca_alm_step
//                 resid += (D - L - E)^2; rr = (A - L) mu_k/mu_{k+1};
//                 E' = S_{lambda/mu_{k+1}}(D - L + rr); A' = D - E' + rr
//   EPI_FINAL   : L stored, resid += (D - L - E)^2       (finalize step)
// K = r (the kept rank, read on the device) is tiny, so the MMA work is far
// below the HBM time of the epilogue's 20 bytes/element: the kernel is built
// to stream D, A, E at bandwidth while the tensor core produces L tiles.
//
// Operands (3xTF32, pre-split, K-major, zero-padded to Kp = 32*ceil(l/32)):
//   QtT_hi/lo (Kp x m)   Wt_hi/lo^T (Kp x n)
// One CTA owns a 128-row block and a range of 128-column tiles:
//   warp 0     TMA: its Q~ block (resident, all K) once, then Wt K-chunks of
//              every column tile through a 2-stage ring
//   warp 1     MMA (SS, both operands from shared memory), accumulator
//              double-buffered in TMEM (2 x 128 columns)
//   warp 2     TMEM allocator
//   warps 4-19 epilogue: tcgen05.ld its 32 rows x 32 columns, then the
//              element-wise update with coalesced column accesses
#pragma once
#include "tc_pass.cuh"

namespace frsvt {
namespace tc {

constexpr int EPI_STORE = 0;
constexpr int EPI_ALM = 1;
constexpr int EPI_FINAL = 2;
constexpr int CMP_THREADS = 640;   // 4 role warps + 16 epilogue warps
constexpr int CMP_EPI_WARPS = 16;
constexpr int CMP_KMAX_CHUNKS = 4;   // Kp <= 128
constexpr int CMP_WSTAGES = 2;

struct ComposeSmem {
  static constexpr uint32_t chunk_bytes = 128u * BK * 4u;  // 128 rows x 32 K fp32 = 16 KB
  static constexpr size_t total() {
    return 1024 + (size_t)CMP_KMAX_CHUNKS * 2 * chunk_bytes + (size_t)CMP_WSTAGES * 2 * chunk_bytes + 512;
  }
};

__device__ __forceinline__ void mma_tf32_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(
          d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

template <int EPI>
__global__ void __launch_bounds__(CMP_THREADS, 1)
tc_compose_kernel(const __grid_constant__ CUtensorMap mapQh, const __grid_constant__ CUtensorMap mapQl,
                  const __grid_constant__ CUtensorMap mapWh, const __grid_constant__ CUtensorMap mapWl, int m, int n,
                  const int* __restrict__ r_dev, int nfull, int sp, float* __restrict__ X, int64_t ldx,
                  const float* __restrict__ D, float* __restrict__ Aop, float* __restrict__ E, int64_t ld,
                  const double* __restrict__ mu, double rho, double lambda, double* __restrict__ part) {
  constexpr uint32_t CB = ComposeSmem::chunk_bytes;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sQh = smem;                              // CMP_KMAX_CHUNKS x CB
  uint8_t* sQl = sQh + CMP_KMAX_CHUNKS * CB;
  uint8_t* sWh = sQl + CMP_KMAX_CHUNKS * CB;        // CMP_WSTAGES x CB
  uint8_t* sWl = sWh + CMP_WSTAGES * CB;
  uint64_t* qfull = (uint64_t*)(sWl + CMP_WSTAGES * CB);
  uint64_t* wfull = qfull + 1;
  uint64_t* wempty = wfull + CMP_WSTAGES;
  uint64_t* accfull = wempty + CMP_WSTAGES;
  uint64_t* accempty = accfull + 2;
  uint32_t* tslot = (uint32_t*)(accempty + 2);
  __shared__ double red[CMP_THREADS / 32];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // CTA -> work: the first nfull CTAs take one whole 128-row block each (full
  // waves, all CTAs of a wave sweep the same column tiles in step: long
  // contiguous DRAM runs per column); the remaining row blocks are split into
  // sp column ranges so the last wave is not a tail of a few CTAs
  const int ntiles = (n + 127) / 128;
  int rb, jt0, jt1;
  if ((int)blockIdx.x < nfull) {
    rb = blockIdx.x;
    jt0 = 0;
    jt1 = ntiles;
  } else {
    const int e = blockIdx.x - nfull;
    const int tpc = (ntiles + sp - 1) / sp;
    rb = nfull + e / sp;
    jt0 = (e % sp) * tpc;
    jt1 = min(ntiles, jt0 + tpc);
  }
  const int r = *r_dev;
  const int nk = (r + BK - 1) / BK;                // K chunks actually used (r <= Kp)

  if (threadIdx.x == 0) {
    mbar_init(qfull, 1);
    for (int s = 0; s < CMP_WSTAGES; ++s) {
      mbar_init(&wfull[s], 1);
      mbar_init(&wempty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&accfull[b], 1);
      mbar_init(&accempty[b], CMP_EPI_WARPS);
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    tmem_alloc(tslot, 256);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;

  if (warp == 0) {
    if (lane == 0 && nk > 0) {
      prefetch_tmap(&mapQh);
      prefetch_tmap(&mapQl);
      prefetch_tmap(&mapWh);
      prefetch_tmap(&mapWl);
      const uint64_t wpol = l2_policy_evict_last();  // Wt tiles are re-read by every row block
      mbar_expect_tx(qfull, 2 * CB * nk);
      for (int kc = 0; kc < nk; ++kc) {
        tma_load_2d(sQh + kc * CB, &mapQh, qfull, kc * BK, rb * 128);
        tma_load_2d(sQl + kc * CB, &mapQl, qfull, kc * BK, rb * 128);
      }
      int it = 0;
      for (int jt = jt0; jt < jt1; ++jt) {
        for (int kc = 0; kc < nk; ++kc, ++it) {
          const int s = it % CMP_WSTAGES;
          const uint32_t ph = (it / CMP_WSTAGES) & 1;
          mbar_wait(&wempty[s], ph ^ 1);
          mbar_expect_tx(&wfull[s], 2 * CB);
          tma_load_2d_hint(sWh + s * CB, &mapWh, &wfull[s], kc * BK, jt * 128, wpol);
          tma_load_2d_hint(sWl + s * CB, &mapWl, &wfull[s], kc * BK, jt * 128, wpol);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && nk > 0) {
      constexpr uint32_t idesc = idesc_tf32(128, 128);
      mbar_wait(qfull, 0);
      int it = 0;
      for (int jt = jt0; jt < jt1; ++jt) {
        const int tl = jt - jt0;
        const int b = tl & 1;
        mbar_wait(&accempty[b], ((tl >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t acc = tbase + 128 * b;
        for (int kc = 0; kc < nk; ++kc, ++it) {
          const int s = it % CMP_WSTAGES;
          const uint32_t ph = (it / CMP_WSTAGES) & 1;
          mbar_wait(&wfull[s], ph);
          tc_fence_after();
          const uint64_t qh = desc_kmajor_sw128(smem_u32(sQh + kc * CB));
          const uint64_t ql = desc_kmajor_sw128(smem_u32(sQl + kc * CB));
          const uint64_t wh = desc_kmajor_sw128(smem_u32(sWh + s * CB));
          const uint64_t wl = desc_kmajor_sw128(smem_u32(sWl + s * CB));
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk) {
            const uint64_t ko = (uint64_t)(kk * 32) >> 4;
            mma_tf32_ss(acc, qh + ko, wh + ko, idesc, (kc > 0 || kk > 0) ? 1u : 0u);
            mma_tf32_ss(acc, qh + ko, wl + ko, idesc, 1u);
            mma_tf32_ss(acc, ql + ko, wh + ko, idesc, 1u);
          }
          tc_commit(&wempty[s]);
        }
        tc_commit(&accfull[b]);
      }
    }
  } else if (warp >= 4) {
    const int ew = warp - 4;               // 0..15
    const int wq = warp & 3;               // TMEM lane quarter (warp % 4)
    const int col0 = (ew >> 2) * 32;       // 32-column quarter of the tile
    const int row = rb * 128 + wq * 32 + lane;
    const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
    double ratio = 1.0, thr = 0.0;
    if (EPI == EPI_ALM) {
      const double mu0 = mu[0];
      const double mu1 = fmin(rho * mu0, mu[1]);
      ratio = mu0 / mu1;
      thr = lambda / mu1;
    }
    const float fratio = (float)ratio, fthr = (float)thr;
    double resid = 0.0;
    for (int jt = jt0; jt < jt1; ++jt) {
      const int tl = jt - jt0;
      const int b = tl & 1;
      if (nk > 0) {
        mbar_wait(&accfull[b], (tl >> 1) & 1);
        tc_fence_after();
      }
      const int c0 = jt * 128 + col0;
      // two 16-column groups; each TMEM load is followed by all of the group's
      // D/E/A loads before any store (E/A stores would otherwise block the
      // next loads: no proof of non-aliasing across columns)
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        uint32_t v[16];
        if (nk > 0) {
          tmem_ld16(tbase + 128 * b + col0 + 16 * g + lane_off, v);
          tc_wait_ld();
          if (g == 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&accempty[b]);
          }
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = 0u;
        }
        if (row < m) {
          if (EPI == EPI_STORE) {
#pragma unroll
            for (int jj = 0; jj < 16; ++jj) {
              const int c = c0 + 16 * g + jj;
              if (c < n) X[row + (int64_t)c * ldx] = __uint_as_float(v[jj]);
            }
          } else {
            float dv[16], ev[16], av[16];
#pragma unroll
            for (int jj = 0; jj < 16; ++jj) {
              const int c = c0 + 16 * g + jj;
              const int64_t o = row + (int64_t)min(c, n - 1) * ld;
              dv[jj] = __ldg(D + o);
              ev[jj] = __ldcs(E + o);
              if (EPI == EPI_ALM) av[jj] = __ldcs(Aop + o);
            }
#pragma unroll
            for (int jj = 0; jj < 16; ++jj) {
              const int c = c0 + 16 * g + jj;
              if (c < n) {
                const float Lv = __uint_as_float(v[jj]);
                const int64_t o = row + (int64_t)c * ld;
                const float res = dv[jj] - Lv - ev[jj];
                resid += (double)res * (double)res;
                if (EPI == EPI_FINAL) {
                  X[row + (int64_t)c * ldx] = Lv;
                } else {
                  const float rr = (av[jj] - Lv) * fratio;
                  const float en = soft<float>(dv[jj] - Lv + rr, fthr);
                  __stcs(E + o, en);
                  __stcs(Aop + o, dv[jj] - en + rr);
                }
              }
            }
          }
        }
      }
    }
    if (EPI != EPI_STORE) {
      resid = warp_sum(resid);
      if (lane == 0) red[warp] = resid;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (EPI != EPI_STORE && threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 4; w < CMP_THREADS / 32; ++w) s += red[w];
    part[blockIdx.x] = s;
  }
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tbase, 256);
  }
}

// split + transpose: Out_hi/lo (Kp x rows, ld Kp) from In (rows x l, ld ldi),
// zero for l <= k < Kp. 32 x 32 tiles through shared memory.
__global__ void split_transpose_kernel(const float* __restrict__ In, int64_t rows, int l, int64_t ldi, int Kp,
                                       float* __restrict__ Hi, float* __restrict__ Lo) {
  __shared__ float t[32][33];
  const int64_t r0 = (int64_t)blockIdx.x * 32;
  const int k0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8 threads
  for (int yy = ty; yy < 32; yy += 8) {
    const int k = k0 + yy;
    const int64_t rr = r0 + tx;
    t[yy][tx] = (k < l && rr < rows) ? In[rr + (int64_t)k * ldi] : 0.f;
  }
  __syncthreads();
  for (int yy = ty; yy < 32; yy += 8) {
    const int64_t rr = r0 + yy;
    const int k = k0 + tx;
    if (rr < rows && k < Kp) {
      const float x = t[tx][yy];
      const uint32_t h = rna_tf32(x);
      Hi[k + rr * Kp] = __uint_as_float(h);
      Lo[k + rr * Kp] = x - __uint_as_float(h);
    }
  }
}

}  // namespace tc
}  // namespace frsvt
