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
//   warp 0     TMA: the Q~ block (once, into the ring area; split into
//              hi/lo by the epilogue warps on its way to TMEM), then Wt
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
#include "tc_util.cuh"

namespace frsvt {
namespace tc {

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr)
               : "memory");
}

// d = a * b + c on fp32 pairs (FFMA2)
__device__ __forceinline__ uint64_t ffma2_u64(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

// Omega^T (rows 0..n-1, FS_PMAX columns each, zero past l) for the fused sketch's TMA slices
__global__ void omega_t24_kernel(const float* __restrict__ Om, int64_t n, int l, float* __restrict__ OmT) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= n * 24) return;
  const int64_t c = idx / 24;
  const int j = (int)(idx - c * 24);
  OmT[idx] = j < l ? Om[c + (int64_t)j * n] : 0.f;
}

constexpr int C2_RING = 12;                     // D/A/E slice stages
constexpr uint32_t C2_SLICE = 128u * 8u * 4u;  // one array, 128 rows x 8 columns = 4 KB
constexpr int FS_PMAX = 24;                     // fused next sketch: at most this many fresh columns
constexpr uint32_t C2_OM = 8u * FS_PMAX * 4u;   // Omega rows of a slice: 8 x 24 fp32 = 768 B
constexpr uint32_t C2_STAGE = 3 * C2_SLICE + C2_OM;

struct Compose2Smem {
  static constexpr uint32_t chunk_bytes = 128u * BK * 4u;  // 16 KB (Wt / Q~ chunk)
  __host__ __device__ static constexpr size_t ring_bytes() { return (size_t)C2_RING * C2_STAGE; }  // 153 KB >= Q~ staging (128 KB)
  __host__ __device__ static constexpr size_t total() {
    return 1024 + ring_bytes() + (size_t)CMP_WSTAGES * 2 * chunk_bytes + 1024;
  }
};

// FS (EPI_ALM only): also form the next call's fresh sketch Y_p = A' Omega_p
// (Alg. 1 line 4 / the RP branch P:132-135 for the next iALM iteration;
// SURVEY §8(a)-a9 "optional partial A' Omega'_p") from the A' values this
// epilogue computes anyway, when p = l - r <= FS_PMAX: fp32 FMAs over the
// CTA's columns, one partial row block per CTA in fspart (summed in CTA order
// by fs_finish_kernel); *fs_done says whether it was formed.
template <int EPI, bool FS>
__global__ void __launch_bounds__(CMP_THREADS, 1)
tc_compose2_kernel(const __grid_constant__ CUtensorMap mapQ, const __grid_constant__ CUtensorMap mapWh, const __grid_constant__ CUtensorMap mapWl,
                   const __grid_constant__ CUtensorMap mapD, const __grid_constant__ CUtensorMap mapA,
                   const __grid_constant__ CUtensorMap mapE, const __grid_constant__ CUtensorMap mapOm, int m, int n,
                   int l, const int* __restrict__ r_dev, int nfull, int sp, float* __restrict__ X, int64_t ldx,
                   float* __restrict__ Aop, float* __restrict__ E, int64_t ld, const double* __restrict__ mu,
                   double rho, double lambda, double* __restrict__ part, float* __restrict__ fspart,
                   int* __restrict__ fs_done) {
  // EPI_STORE: X = Q~ Wt^T only (the FRSVT call's composition, Eq. (6)); no
  // streamed operands, the epilogue writes X from the accumulator
  constexpr uint32_t CB = Compose2Smem::chunk_bytes;
  constexpr int NARR = EPI == EPI_ALM ? 3 : (EPI == EPI_FINAL ? 2 : 0);  // D, E (, A)
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
  const int pfs = l - r;             // fresh columns of the next sketch
  const bool fs = FS && EPI == EPI_ALM && pfs >= 1 && pfs <= FS_PMAX;

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
      prefetch_tmap(&mapQ);
      prefetch_tmap(&mapWh);
      prefetch_tmap(&mapWl);
      if (nk > 0) {
        // Q~ (m x l column-major): K-chunk kc = box {128 rows, 32 columns}, column-major in smem
        mbar_expect_tx(qfull, CB * nk);
        for (int kc = 0; kc < nk; ++kc) tma_load_2d(ring + kc * CB, &mapQ, qfull, rb * 128, kc * BK);
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
    if (lane == 0 && NARR > 0) {
      prefetch_tmap(&mapD);
      prefetch_tmap(&mapE);
      if (EPI == EPI_ALM) prefetch_tmap(&mapA);
      if (fs) prefetch_tmap(&mapOm);
      const uint64_t pol = l2_policy_evict_first();
      if (nk > 0) mbar_wait(qready, 0);  // Q~ staging in the ring has been consumed
      for (int i = 0; i < nsl; ++i) {
        const int s = i % C2_RING;
        const uint32_t ph = (i / C2_RING) & 1;
        mbar_wait(&sempty[s], ph ^ 1);
        const int c0 = jt0 * 128 + 8 * i;
        uint8_t* st = ring + (size_t)s * C2_STAGE;
        mbar_expect_tx(&sfull[s], NARR * C2_SLICE + (fs ? C2_OM : 0u));
        tma_load_2d_hint(st, &mapD, &sfull[s], rb * 128, c0, pol);
        tma_load_2d_hint(st + C2_SLICE, &mapE, &sfull[s], rb * 128, c0, pol);
        if (EPI == EPI_ALM) tma_load_2d_hint(st + 2 * C2_SLICE, &mapA, &sfull[s], rb * 128, c0, pol);
        if (fs) tma_load_2d(st + 3 * C2_SLICE, &mapOm, &sfull[s], 0, c0);  // Omega^T: rows c0..c0+7, 24 columns each
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
    // Q~ of this row: staging (column-major chunks) -> split into tf32 hi and
    // the fp32 remainder lo (the 3xTF32 A operands) -> TMEM
    if (grp == 0 && nk > 0) {
      mbar_wait(qfull, 0);
#pragma unroll 1
      for (int kc = 0; kc < nk; ++kc) {
        const float* qs = reinterpret_cast<const float*>(ring + kc * CB);
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          uint32_t hi[16], lo[16];
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            const float x = qs[(16 * half + c) * 128 + rloc];
            const uint32_t hx = rna_tf32(x);
            hi[c] = hx;
            lo[c] = __float_as_uint(x - __uint_as_float(hx));
          }
          tmem_st16(t_qh + (uint32_t)(kc * BK + 16 * half) + lane_off, hi);
          tmem_st16(t_ql + (uint32_t)(kc * BK + 16 * half) + lane_off, lo);
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
    uint64_t ys[FS ? FS_PMAX / 2 : 1];  // fp32 pairs (j = 2q, 2q + 1)
#pragma unroll
    for (int q = 0; q < (FS ? FS_PMAX / 2 : 1); ++q) ys[q] = 0ull;
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
      if (EPI == EPI_STORE) {
        if (row < m) {
          const int c0 = (jt0 + tl) * 128 + 8 * cc;
#pragma unroll
          for (int jj = 0; jj < 8; ++jj)
            if (c0 + jj < n) __stcs(X + row + (int64_t)(c0 + jj) * ldx, __uint_as_float(v[jj]));
        }
        continue;
      }
      mbar_wait(&sfull[s], (i / C2_RING) & 1);
      const float* st = reinterpret_cast<const float*>(ring + (size_t)s * C2_STAGE);
      float dv[8], ev[8], av[8];
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) {
        dv[jj] = st[jj * 128 + rloc];
        ev[jj] = st[1024 + jj * 128 + rloc];
        av[jj] = EPI == EPI_ALM ? st[2048 + jj * 128 + rloc] : 0.f;
      }
      if (!fs) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&sempty[s]);
      }
      float an[8];  // A' of this slice (fused sketch)
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
              an[jj] = dv[jj] - en + rr;
              __stcs(E + o, en);
              __stcs(Aop + o, an[jj]);
            }
          } else {
            an[jj] = 0.f;
          }
        }
      } else {
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) an[jj] = 0.f;
      }
      if (FS && fs) {
        // ys[j] += sum_jj A'(row, c0 + jj) Omega(c0 + jj, j): packed fp32 pairs
        // (FFMA2), Omega^T rows of the slice in shared memory ([jj][24], zero
        // past n)
        const float* om = st + 3 * 1024;
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          const float2 a2 = make_float2(an[jj], an[jj]);
          const uint64_t a = *reinterpret_cast<const uint64_t*>(&a2);
#pragma unroll
          for (int t = 0; t < FS_PMAX / 4; ++t) {
            if (4 * t < pfs) {
              const float4 o = *reinterpret_cast<const float4*>(om + jj * FS_PMAX + 4 * t);
              const float2 o01 = make_float2(o.x, o.y), o23 = make_float2(o.z, o.w);
              ys[2 * t] = ffma2_u64(a, *reinterpret_cast<const uint64_t*>(&o01), ys[2 * t]);
              ys[2 * t + 1] = ffma2_u64(a, *reinterpret_cast<const uint64_t*>(&o23), ys[2 * t + 1]);
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sempty[s]);
      }
    }
    if (FS && fs) {
      // the four groups' partial rows -> this CTA's slot: ring reused as scratch
      // once every epilogue warp is past its last slice
      asm volatile("bar.sync 1, 512;" ::: "memory");
      float* scr = reinterpret_cast<float*>(ring);  // [grp][j][128]
#pragma unroll
      for (int q = 0; q < FS_PMAX / 2; ++q) {
        const float2 y = *reinterpret_cast<const float2*>(&ys[q]);
        if (2 * q < pfs) scr[(grp * FS_PMAX + 2 * q) * 128 + rloc] = y.x;
        if (2 * q + 1 < pfs) scr[(grp * FS_PMAX + 2 * q + 1) * 128 + rloc] = y.y;
      }
      asm volatile("bar.sync 1, 512;" ::: "memory");
      if (grp == 0) {
        float* dst = fspart + (size_t)blockIdx.x * FS_PMAX * 128;
        for (int j = 0; j < pfs; ++j)
          dst[j * 128 + rloc] = ((scr[(0 * FS_PMAX + j) * 128 + rloc] + scr[(1 * FS_PMAX + j) * 128 + rloc]) +
                                 scr[(2 * FS_PMAX + j) * 128 + rloc]) + scr[(3 * FS_PMAX + j) * 128 + rloc];
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
    if (FS && blockIdx.x == 0) *fs_done = fs ? 1 : 0;
  }
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tbase, 512);
  }
}

// Y[:, r + j] (j < p) = sum of the covering CTAs' partial rows, in CTA order
// (the compose2 grid: CTA rb for rb < nfull, else nfull + (rb - nfull) sp + e).
__global__ void __launch_bounds__(128) fs_finish_kernel(const float* __restrict__ fspart, int m, int l,
                                                        const int* __restrict__ r_dev, int nfull, int sp,
                                                        float* __restrict__ Y, const int* __restrict__ fs_done) {
  if (!*fs_done) return;
  const int r = *r_dev, p = l - r;
  const int rb = blockIdx.x, rloc = threadIdx.x, row = rb * 128 + rloc;
  const int c0 = rb < nfull ? rb : nfull + (rb - nfull) * sp;
  const int nc = rb < nfull ? 1 : sp;
  for (int j = 0; j < p; ++j) {
    float y = 0.f;
    for (int e = 0; e < nc; ++e) y += fspart[((size_t)(c0 + e) * FS_PMAX + j) * 128 + rloc];
    if (row < m) Y[row + (int64_t)(r + j) * m] = y;
  }
}

}  // namespace tc
}  // namespace frsvt
