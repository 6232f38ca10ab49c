// tcgen05 composition fused with the iALM epilogue, version 2 (default for
// EPI_ALM / EPI_FINAL): the same arithmetic as tc_compose_kernel
// (tc_compose.cuh: X = Q~ Wt^T, Eq. (6)), with
// the streamed operands D, A, E moved by TMA instead of per-thread loads.
//
// Why: the first version's 16 epilogue warps held at most ~50 KB of D/E/A
// loads in flight per SM (register-bound at 640 threads), and ncu showed the
// kernel stalled on long scoreboard at 4.9 TB/s. Here the resident Q~ block
// lives in TMEM as the MMA A operand (hi/lo, up to 2 x 128 columns next to
// the 2 x 128-column accumulator), which frees the shared memory for a
// 12-stage TMA ring of 8-column D/A/E slices (144 KB in flight per SM).
//
// Roles (640 threads):
//   warp 0     TMA: the Q~ block (hi/lo, once, into the ring area), then Wt
//              K-chunks of every column tile through a 2-stage ring
//   warp 1     MMA: 3xTF32 with A = Q~ from TMEM, B = Wt from shared memory
//   warp 2     TMEM allocator (512 columns)
//   warp 3     TMA: D/A/E 8-column slices (128 rows each) into the ring,
//              after Q~ has been moved to TMEM
//   warps 4-19 epilogue, 4 groups of 4 warps (one per TMEM lane quarter);
//              group g takes the slices s = g (mod 4): tcgen05.ld of the 8
//              accumulator columns, D/A/E from shared memory, the update,
//              direct stores of E', A' (or L)
#pragma once
#include "tc_compose.cuh"
#include "tc_pass2.cuh"

namespace frsvt {
namespace tc {

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr)
               : "memory");
}

constexpr int C2_RING = 12;                     // D/A/E slice stages
constexpr uint32_t C2_SLICE = 128u * 8u * 4u;  // one array, 128 rows x 8 columns = 4 KB

struct Compose2Smem {
  static constexpr uint32_t chunk_bytes = 128u * BK * 4u;  // 16 KB (Wt / Q~ chunk)
  __host__ __device__ static constexpr size_t ring_bytes() { return (size_t)C2_RING * 3 * C2_SLICE; }  // 144 KB >= Q~ staging (128 KB)
  __host__ __device__ static constexpr size_t total() {
    return 1024 + ring_bytes() + (size_t)CMP_WSTAGES * 2 * chunk_bytes + 1024;
  }
};

template <int EPI>
__global__ void __launch_bounds__(CMP_THREADS, 1)
tc_compose2_kernel(const __grid_constant__ CUtensorMap mapQh, const __grid_constant__ CUtensorMap mapQl,
                   const __grid_constant__ CUtensorMap mapWh, const __grid_constant__ CUtensorMap mapWl,
                   const __grid_constant__ CUtensorMap mapD, const __grid_constant__ CUtensorMap mapA,
                   const __grid_constant__ CUtensorMap mapE, int m, int n, const int* __restrict__ r_dev, int nfull,
                   int sp, float* __restrict__ X, int64_t ldx, float* __restrict__ Aop, float* __restrict__ E,
                   int64_t ld, const double* __restrict__ mu, double rho, double lambda, double* __restrict__ part) {
  static_assert(EPI == EPI_ALM || EPI == EPI_FINAL, "compose2 streams D/E(/A)");
  constexpr uint32_t CB = Compose2Smem::chunk_bytes;
  constexpr int NARR = EPI == EPI_ALM ? 3 : 2;  // D, E (, A)
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* ring = smem;                                   // C2_RING x 3 slices; first Q~ staging
  uint8_t* sWh = ring + Compose2Smem::ring_bytes();       // CMP_WSTAGES x CB
  uint8_t* sWl = sWh + CMP_WSTAGES * CB;
  uint64_t* qfull = (uint64_t*)(sWl + CMP_WSTAGES * CB);
  uint64_t* qready = qfull + 1;
  uint64_t* wfull = qready + 1;
  uint64_t* wempty = wfull + CMP_WSTAGES;
  uint64_t* accfull = wempty + CMP_WSTAGES;
  uint64_t* accempty = accfull + 2;
  uint64_t* sfull = accempty + 2;
  uint64_t* sempty = sfull + C2_RING;
  uint32_t* tslot = (uint32_t*)(sempty + C2_RING);
  __shared__ double red[CMP_THREADS / 32];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
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
  const int nk = (r + BK - 1) / BK;  // K chunks actually used (r <= Kp <= 128)
  const int nsl = (jt1 - jt0) * 16;  // 8-column slices of this CTA

  if (threadIdx.x == 0) {
    mbar_init(qfull, 1);
    mbar_init(qready, 4);
    for (int s = 0; s < CMP_WSTAGES; ++s) {
      mbar_init(&wfull[s], 1);
      mbar_init(&wempty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&accfull[b], 1);
      mbar_init(&accempty[b], CMP_EPI_WARPS);
    }
    for (int s = 0; s < C2_RING; ++s) {
      mbar_init(&sfull[s], 1);
      mbar_init(&sempty[s], 4);
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    tmem_alloc(tslot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  const uint32_t t_qh = tbase + 256, t_ql = tbase + 384;  // Q~ hi / lo, K along columns

  if (warp == 0) {
    if (lane == 0) {
      prefetch_tmap(&mapQh);
      prefetch_tmap(&mapQl);
      prefetch_tmap(&mapWh);
      prefetch_tmap(&mapWl);
      if (nk > 0) {
        mbar_expect_tx(qfull, 2 * CB * nk);
        for (int kc = 0; kc < nk; ++kc) {
          tma_load_2d(ring + kc * CB, &mapQh, qfull, kc * BK, rb * 128);
          tma_load_2d(ring + (4 + kc) * CB, &mapQl, qfull, kc * BK, rb * 128);
        }
        const uint64_t wpol = l2_policy_evict_last();  // Wt tiles are re-read by every row block
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
    }
  } else if (warp == 3) {
    if (lane == 0) {
      prefetch_tmap(&mapD);
      prefetch_tmap(&mapE);
      if (EPI == EPI_ALM) prefetch_tmap(&mapA);
      const uint64_t pol = l2_policy_evict_first();
      if (nk > 0) mbar_wait(qready, 0);  // Q~ staging in the ring has been consumed
      for (int i = 0; i < nsl; ++i) {
        const int s = i % C2_RING;
        const uint32_t ph = (i / C2_RING) & 1;
        mbar_wait(&sempty[s], ph ^ 1);
        const int c0 = jt0 * 128 + 8 * i;
        uint8_t* st = ring + (size_t)s * 3 * C2_SLICE;
        mbar_expect_tx(&sfull[s], NARR * C2_SLICE);
        tma_load_2d_hint(st, &mapD, &sfull[s], rb * 128, c0, pol);
        tma_load_2d_hint(st + C2_SLICE, &mapE, &sfull[s], rb * 128, c0, pol);
        if (EPI == EPI_ALM) tma_load_2d_hint(st + 2 * C2_SLICE, &mapA, &sfull[s], rb * 128, c0, pol);
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && nk > 0) {
      constexpr uint32_t idesc = idesc_tf32(128, 128);
      mbar_wait(qready, 0);
      tc_fence_after();
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
          const uint64_t wh = desc_kmajor_sw128(smem_u32(sWh + s * CB));
          const uint64_t wl = desc_kmajor_sw128(smem_u32(sWl + s * CB));
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk) {
            const uint64_t ko = (uint64_t)(kk * 32) >> 4;
            const uint32_t qa = (uint32_t)(kc * BK + kk * 8);
            mma_tf32_ts(acc, t_qh + qa, wh + ko, idesc, (kc > 0 || kk > 0) ? 1u : 0u);
            mma_tf32_ts(acc, t_qh + qa, wl + ko, idesc, 1u);
            mma_tf32_ts(acc, t_ql + qa, wh + ko, idesc, 1u);
          }
          tc_commit(&wempty[s]);
        }
        tc_commit(&accfull[b]);
      }
    }
  } else if (warp >= 4) {
    const int wq = warp & 3;         // TMEM lane quarter
    const int grp = (warp - 4) >> 2;  // slice group
    const int rloc = wq * 32 + lane;
    const int row = rb * 128 + rloc;
    const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
    // Q~ (hi/lo) of this row: staging (128B-swizzled K-major chunks) -> TMEM
    if (grp == 0 && nk > 0) {
      mbar_wait(qfull, 0);
#pragma unroll 1
      for (int q = 0; q < 2 * nk; ++q) {
        const int hl = q & 1, kc = q >> 1;
        const uint32_t a_s = smem_u32(ring + (hl * 4 + kc) * CB);
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          uint32_t x[16];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int cc = 4 * half + c;
            lds_u32x4(a_s + (uint32_t)(rloc * 128 + ((cc ^ (rloc & 7)) * 16)), x[4 * c], x[4 * c + 1], x[4 * c + 2],
                      x[4 * c + 3]);
          }
          tmem_st16((hl ? t_ql : t_qh) + (uint32_t)(kc * BK + 16 * half) + lane_off, x);
        }
      }
      tc_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(qready);
    }
    double ratio = 1.0, thr = 0.0;
    if (EPI == EPI_ALM) {
      const double mu0 = mu[0];
      const double mu1 = fmin(rho * mu0, mu[1]);
      ratio = mu0 / mu1;
      thr = lambda / mu1;
    }
    const float fratio = (float)ratio, fthr = (float)thr;
    double resid = 0.0;
    for (int i = grp; i < nsl; i += 4) {
      const int tl = i >> 4, cc = i & 15, b = tl & 1;
      const int s = i % C2_RING;
      uint32_t v[8];
      if (nk > 0) {
        if (cc < 4) {  // this group's first slice of the tile
          mbar_wait(&accfull[b], (tl >> 1) & 1);
          tc_fence_after();
        }
        tmem_ld8(tbase + 128 * b + 8 * cc + lane_off, v);
        tc_wait_ld();
        if (cc >= 12) {  // last slice of the tile for this group
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&accempty[b]);
        }
      } else {
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) v[jj] = 0u;
      }
      mbar_wait(&sfull[s], (i / C2_RING) & 1);
      const float* st = reinterpret_cast<const float*>(ring + (size_t)s * 3 * C2_SLICE);
      float dv[8], ev[8], av[8];
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) {
        dv[jj] = st[jj * 128 + rloc];
        ev[jj] = st[1024 + jj * 128 + rloc];
        av[jj] = EPI == EPI_ALM ? st[2048 + jj * 128 + rloc] : 0.f;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sempty[s]);
      if (row < m) {
        const int c0 = (jt0 + tl) * 128 + 8 * cc;
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          const int c = c0 + jj;
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
    resid = warp_sum(resid);
    if (lane == 0) red[warp] = resid;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 4; w < CMP_THREADS / 32; ++w) s += red[w];
    part[blockIdx.x] = s;
  }
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tbase, 512);
  }
}

}  // namespace tc
}  // namespace frsvt
