// Persistent stream-K streaming pass over the m x n operand A on CTA PAIRS
// (tcgen05 cta_group::2): the GEMM-shaped steps of Algorithm 1 (PAPER.md
// P:128 sketch, P:141 power iteration, P:143/P:177 B = Q^T A).
//   MODE_AX : Y (m x l) = A (m x n) X (n x l)      M = rows of A, K = n
//   MODE_ATQ: Z (n x l) = A^T (n x m) Q (m x l)    M = columns of A, K = m
//
// Why this shape. A streams from HBM once per pass; the small operand B (X or
// Q, split into tensor-core formats) is re-read from L2 for every row tile.
// With one CTA per 128-row tile, B cost 2 bytes of shared-memory fill and ~2
// bytes of MMA operand reads per byte of A (round 1, profiles/r1_*): the SM's
// shared-memory bandwidth and the L2->SM delivery, not HBM, bound the pass.
// Here the two CTAs of a cluster issue ONE M = 256 MMA (cta_group::2): each
// CTA holds its 128 A rows in its own TMEM and HALF of every B stage (N/2
// rows) in its shared memory, so B costs each SM half the fill and half the
// operand reads, and the pair fetches B from L2 once.
//
// Products (fp32-level; 1xTF32 misses 1e-4), with
// a_h = rna_tf32(a), a_l = a - a_h, b_h = rna_tf32(b), b_l = b - b_h:
//   TERMS = 3 (exact):     a b ~= a_h b_h + [bf16 a_h | bf16 a_l] . [bf16 b_l ; bf16 b_h]
//                          4 tf32 MMAs (K = 8) + 4 bf16 MMAs (K = 16) per 32-wide K chunk
//   TERMS = 2 (span-only): a b_h ~= a_h b_h + bf16(a_l) bf16(b_h)
//                          4 tf32 + 2 bf16 MMAs: the product of the EXACT A with the
//                          tf32-rounded small operand (reading R17: used only where the
//                          small operand is a basis whose span alone matters next)
// The bf16 roundings cost ~2^-19 |a b| per term; measured pass error ~1e-6.
//
// Work: M tile pairs x K chunks flattened pair-major and cut into G
// contiguous ranges, one per cluster (stream-K): every SM streams the same
// number of chunks. A pair range covering a whole tile writes it; a tile
// split between clusters leaves partials in per-CTA slots and the CTA that
// completes it last (per-tile arrival counter) sums them in CTA order.
//
// Roles per CTA (640 threads):
//   warp 0      A producer: 16 KB chunks of this CTA's 128 rows, AST-deep ring
//   warp 3      B producer: this CTA's N/2-row half of each B stage; the
//               completion is counted on the LEADER's barrier (cta_group::2 TMA)
//   warp 1      MMA issuer, leader CTA only (one elected thread)
//   warp 2      TMEM allocator (cta_group::2: both CTAs, same columns)
//   warps 4..11 converters (two groups of four, alternate chunks): A chunk ->
//               a_h (tf32) and bf16 parts -> own TMEM ring; arrive on the
//               leader's stage barrier (remote arrive for the peer CTA)
//   warps 12..19 flush: accumulator pieces (<= 8 chunks, never across a
//               tile) -> fp32 registers -> output / partial slot
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include "tc_util.cuh"

namespace frsvt {
namespace tc {

constexpr int P3_THREADS = 640;
constexpr int P3_SLOTS = 2;  // partial-tile slots per CTA
#ifndef P3_SEG_CH
#define P3_SEG_CH 8
#endif
#ifndef P3_BST_WIDE
#define P3_BST_WIDE 6
#endif
#ifndef P3_AST_WIDE
#define P3_AST_WIDE 6
#endif
constexpr int P3_SEG = P3_SEG_CH;  // chunks accumulated in TMEM before a flush

// A ring (16 KB stages) and B ring depth of an instance
__host__ __device__ constexpr int p3_astages(int np, int terms) {
  return np <= 32 ? 8 : (terms == 2 ? P3_AST_WIDE + 1 : P3_AST_WIDE);
}
__host__ __device__ constexpr int p3_bstages(int np, int terms) { return np <= 32 ? 8 : P3_BST_WIDE; }

// the chunk range of a cluster as accumulator pieces of <= P3_SEG chunks,
// never crossing a tile (all roles iterate it identically)
struct P3Walk {
  int64_t g, g1;  // next chunk, end of range
  int nch;        // chunks per tile
  __device__ __forceinline__ bool next(int& tile, int& k0, int& k1, bool& tile_first, bool& tile_last,
                                       int64_t& seg_begin) {
    if (g >= g1) return false;
    tile = (int)(g / nch);
    k0 = (int)(g - (int64_t)tile * nch);
    const int64_t end = min(g1, (int64_t)(tile + 1) * nch);
    tile_first = (g == seg_begin);
    k1 = (int)min((int64_t)(k0 + P3_SEG), end - (int64_t)tile * nch);
    g = (int64_t)tile * nch + k1;
    tile_last = (g == end);
    if (tile_last) seg_begin = g;
    return true;
  }
};
// TMEM A ring: stage stride in columns, number of stages (accumulators use 0..255)
__host__ __device__ constexpr int p3_tstride(int terms) { return terms == 3 ? 64 : 48; }
__host__ __device__ constexpr int p3_tstages(int terms) { return terms == 3 ? 4 : 5; }

struct Pass3Smem {
  static constexpr uint32_t a_bytes = 128u * BK * 4u;  // 16 KB
  // one B stage of this CTA: nh = N/2 rows of tf32 (128 B) + bf16 (128 B [b_l|b_h] or 64 B b_h)
  __host__ __device__ static constexpr uint32_t bh_bytes(int np) { return (uint32_t)(np / 2) * 128u; }
  __host__ __device__ static constexpr uint32_t bx_bytes(int np, int terms) {
    return (uint32_t)(np / 2) * (terms == 3 ? 128u : 64u);
  }
  __host__ __device__ static constexpr uint32_t b_stage(int np, int terms) { return bh_bytes(np) + bx_bytes(np, terms); }
  __host__ __device__ static constexpr size_t total(int np, int terms) {
    return 1024 + (size_t)p3_astages(np, terms) * a_bytes + (size_t)p3_bstages(np, terms) * b_stage(np, terms) + 512;
  }
};

__device__ __forceinline__ uint32_t mapa_u32(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
// arrive on the barrier at the same offset in CTA `rank` of the cluster. The
// data handed over this way lives in TMEM (ordered by tcgen05.wait::st and
// tcgen05.fence::before_thread_sync on the arriving side, fence::after on the
// MMA side) or is a TMEM read that completed (tcgen05.wait::ld), so the
// default CTA-scope release suffices; a .release.cluster arrive measured
// ~0.7 us per arrival on B200 (a cluster-scope fence per call).
__device__ __forceinline__ void mbar_arrive_rank(uint64_t* bar, uint32_t rank) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(mapa_u32(smem_u32(bar), rank)) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* b, uint32_t parity) { mbar_wait(b, parity); }
// TMA 2D load into this CTA's shared memory whose transaction bytes complete
// on the barrier at cluster address `bar_cluster` (the leader CTA's)
__device__ __forceinline__ void tma_load_2d_cg2(void* dst, const CUtensorMap* map, uint32_t bar_cluster, int c0, int c1,
                                                uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(bar_cluster), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tmem_alloc_cg2(uint32_t* slot, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void tmem_relinquish_cg2() {
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc_cg2(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void mma_tf32_ts_cg2(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                                uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(
          d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_bf16_ts_cg2(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                                uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(
          d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// MMA completion -> the barrier at the same offset in both CTAs of the pair
__device__ __forceinline__ void tc_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)0x3)
      : "memory");
}
// the same arrivals without an MMA (pipeline probes): both CTAs' barriers
__device__ __forceinline__ void arrive_pair(uint64_t* bar) {
  mbar_arrive(bar);
  mbar_arrive_rank(bar, 1);
}

// dbg (test hook only, 0 in production): bit 0 no MMA, bit 1 no conversion,
// bit 2 no B loads, bit 4 no accumulator reads (flush), bit 8 whole work
// tiles per cluster (small K, set by the host)
template <int MODE, int NP, int TERMS>
__global__ void __launch_bounds__(P3_THREADS, 1)
tc_pass3_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapBh,
                const __grid_constant__ CUtensorMap mapBx, int Mtot, int Ktot, int Nvalid,
                float* __restrict__ out, int64_t ldo, const float* __restrict__ add, int64_t ldadd,
                float* __restrict__ part, const int* __restrict__ rp_dev, int dbg,
                unsigned int* __restrict__ tile_cnt, const int* __restrict__ skip_dev) {
  // skip_dev (nullable): the output was already formed (fused next sketch, or
  // the other instance of a device-side width choice)
  if (skip_dev && *skip_dev) return;
  // rp_dev (MODE_AX, range propagation): r = *rp_dev carried columns; only the
  // p = Nvalid - r fresh columns are multiplied (B holds them at [0, p)) and
  // land in out[:, r + c]; out[:, :r] is a copy of add[:, :r] (the carry Q~).
  static_assert(NP == 32 || NP == 64 || NP == 128, "N tile (cta_group::2 TS: N % 32 == 0)");
  static_assert(TERMS == 2 || TERMS == 3, "product terms");
  constexpr int CL = 2;
  constexpr int AST = p3_astages(NP, TERMS);
  constexpr int BST = p3_bstages(NP, TERMS);
  constexpr int TST = p3_tstages(TERMS);
  constexpr int TSTR = p3_tstride(TERMS);
  constexpr uint32_t A_BYTES = Pass3Smem::a_bytes;
  constexpr uint32_t BH_BYTES = Pass3Smem::bh_bytes(NP);
  constexpr uint32_t B_BYTES = Pass3Smem::b_stage(NP, TERMS);
  constexpr int NH = NP / 2;   // B rows per CTA
  constexpr int HALF = NP / 2; // accumulator columns per flush warp
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + AST * A_BYTES;
  uint64_t* fulla = (uint64_t*)(sB + BST * B_BYTES);
  uint64_t* emptya = fulla + AST;
  uint64_t* fullb = emptya + AST;
  uint64_t* emptyb = fullb + BST;
  uint64_t* tfull = emptyb + BST;
  uint64_t* tempty = tfull + TST;
  uint64_t* accfull = tempty + TST;
  uint64_t* accempty = accfull + 2;
  uint32_t* tslot = (uint32_t*)(accempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = cluster_ctarank();
  const bool leader = crank == 0;
  const int rsh = rp_dev ? min(max(*rp_dev, 0), Nvalid) : 0;  // output column shift
  const int nact = Nvalid - rsh;                              // multiplied columns
  const int nmma = min(NP, max(32, ((rp_dev ? nact : Nvalid) + 31) & ~31));
  const int nch = (Ktot + BK - 1) / BK;
  const int mtiles = (Mtot + 127) / 128;
  const int mgroups = (mtiles + CL - 1) / CL;
  const int64_t total = (int64_t)mgroups * nch;
  const int G = gridDim.x / CL, cta = blockIdx.x, cgrp = blockIdx.x / CL;
  const bool talign = (dbg & 256) != 0;
  const int64_t g0 = talign ? ((int64_t)mgroups * cgrp / G) * nch : sk_range_begin(total, G, cgrp);
  const int64_t g1 = talign ? ((int64_t)mgroups * (cgrp + 1) / G) * nch : sk_range_begin(total, G, cgrp + 1);
  const int nloc = (int)(g1 - g0);

  if (threadIdx.x == 0) {
    for (int s = 0; s < AST; ++s) {
      mbar_init(&fulla[s], 1);
      mbar_init(&emptya[s], 4);
    }
    for (int s = 0; s < BST; ++s) {
      mbar_init(&fullb[s], 1);   // leader: its expect_tx arrive (+ both CTAs' bytes)
      mbar_init(&emptyb[s], 1);  // the leader's MMA commit
    }
    for (int t = 0; t < TST; ++t) {
      mbar_init(&tfull[t], 8);   // leader: 4 converter warps of each CTA
      mbar_init(&tempty[t], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&accfull[b], 1);
      mbar_init(&accempty[b], 16);  // leader: 8 flush warps of each CTA
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    tmem_alloc_cg2(tslot, 512);
    tmem_relinquish_cg2();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // barriers of both CTAs initialised, TMEM allocated in both
  tc_fence_after();
  const uint32_t tbase = *tslot;
  const uint32_t t_acc0 = tbase;     // accumulator buffer b at columns [128 b, 128 b + NP)
  const uint32_t t_a = tbase + 256;  // A ring: stage t at 256 + TSTR t

  if (warp == 0) {
    // A producer (HBM stream) of this CTA's 128 rows
    if (lane == 0 && nloc > 0) {
      prefetch_tmap(&mapA);
      const uint64_t pol = l2_policy_evict_first();
      for (int i = 0; i < nloc; ++i) {
        const int64_t g = g0 + i;
        const int grp = (int)(g / nch), kc = (int)(g - (int64_t)grp * nch) * BK;
        const int tile = grp * CL + (int)crank;
        const int s = i % AST;
        mbar_wait(&emptya[s], ((i / AST) & 1) ^ 1);
        mbar_expect_tx(&fulla[s], A_BYTES);
        if (MODE == MODE_AX)
          tma_load_2d_hint(sA + s * A_BYTES, &mapA, &fulla[s], tile * 128, kc, pol);
        else
          tma_load_2d_hint(sA + s * A_BYTES, &mapA, &fulla[s], kc, tile * 128, pol);
      }
    }
  } else if (warp == 3) {
    // B producer: this CTA's NH-row half of every stage, counted on the leader's barrier
    if (lane == 0 && nloc > 0) {
      prefetch_tmap(&mapBh);
      prefetch_tmap(&mapBx);
      const uint64_t pol = l2_policy_evict_last();
      constexpr uint32_t btx = 2u * B_BYTES;  // both halves (out-of-bounds rows are zero-filled and counted)
      for (int i = 0; i < nloc; ++i) {
        const int64_t g = g0 + i;
        const int grp = (int)(g / nch), kc = (int)(g - (int64_t)grp * nch) * BK;
        const int s = i % BST;
        mbar_wait(&emptyb[s], ((i / BST) & 1) ^ 1);
        if (dbg & 4) {
          if (leader) mbar_arrive(&fullb[s]);
          continue;
        }
        if (leader) mbar_expect_tx(&fullb[s], btx);
        const uint32_t bar = mapa_u32(smem_u32(&fullb[s]), 0);
        tma_load_2d_cg2(sB + s * B_BYTES, &mapBh, bar, kc, NH * (int)crank, pol);
        tma_load_2d_cg2(sB + s * B_BYTES + BH_BYTES, &mapBx, bar, TERMS == 3 ? 2 * kc : kc, NH * (int)crank, pol);
      }
    }
  } else if (warp == 1) {
    // MMA issuer (leader CTA): one M = 256 MMA per K step covers both CTAs' rows
    if (leader && nloc > 0) {
      const uint32_t id_tf = idesc_tf32(256, nmma);
      const uint32_t id_bf = idesc_bf16(256, nmma);
      const bool elected = elect_one();
      P3Walk wk{g0, g1, nch};
      int64_t sb = g0;
      int tile, k0, k1;
      bool tf, tl;
      int i = 0, piece = 0;
      const uint32_t sB_u = smem_u32(sB);
      while (wk.next(tile, k0, k1, tf, tl, sb)) {
        const int b = piece & 1;
        mbar_wait_cluster(&accempty[b], ((piece >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t acc = t_acc0 + 128 * b;
        for (int kc = k0; kc < k1; ++kc, ++i) {
          const int s = i % BST;
          const int t = i % TST;
          mbar_wait_cluster(&fullb[s], (i / BST) & 1);
          mbar_wait_cluster(&tfull[t], (i / TST) & 1);
          tc_fence_after();
          if (elected) {
            if (dbg & 1) {
              arrive_pair(&emptyb[s]);
              arrive_pair(&tempty[t]);
            } else {
              const uint32_t st = sB_u + (uint32_t)s * B_BYTES;
              const uint64_t bh = desc_kmajor_sw128(st);
              const uint32_t a_hi = t_a + t * TSTR, a_x = a_hi + 32;
#pragma unroll
              for (int kk = 0; kk < BK / 8; ++kk)  // a_h b_h: 8 tf32 = 32 bytes along K
                mma_tf32_ts_cg2(acc, a_hi + kk * 8, bh + ((uint64_t)(kk * 32) >> 4), id_tf,
                                (kc > k0 || kk > 0) ? 1u : 0u);
              if (TERMS == 3) {
                const uint64_t bx = desc_kmajor_sw128(st + BH_BYTES);
#pragma unroll
                for (int kk = 0; kk < 2 * BK / 16; ++kk)  // [a_h | a_l] . [b_l ; b_h], 16 bf16 = 32 bytes along K'
                  mma_bf16_ts_cg2(acc, a_x + kk * 8, bx + ((uint64_t)(kk * 32) >> 4), id_bf, 1u);
              } else {
                const uint64_t bx = desc_kmajor_sw64(st + BH_BYTES);
#pragma unroll
                for (int kk = 0; kk < BK / 16; ++kk)  // a_l b_h
                  mma_bf16_ts_cg2(acc, a_x + kk * 8, bx + ((uint64_t)(kk * 32) >> 4), id_bf, 1u);
              }
              tc_commit_pair(&emptyb[s]);  // frees B stage s in both CTAs
              tc_commit_pair(&tempty[t]);  // frees A stage t in both CTAs' TMEM
            }
          }
          __syncwarp();
        }
        if (elected) {
          if (dbg & 1) arrive_pair(&accfull[b]);
          else tc_commit_pair(&accfull[b]);
        }
        __syncwarp();
        ++piece;
      }
    }
  } else if (warp >= 4 && warp < 12) {
    // converters: A chunk in shared memory -> a_h (tf32) and bf16 parts -> TMEM ring
    const int wq = warp & 3, grp = (warp - 4) >> 2;
    const int row = wq * 32 + lane;
    const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
    for (int i = grp; i < nloc; i += 2) {
      const int s = i % AST;
      const int t = i % TST;
      const uint32_t tph = (i / TST) & 1;
      mbar_wait(&fulla[s], (i / AST) & 1);
      if (dbg & 2) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&emptya[s]);
        mbar_wait(&tempty[t], tph ^ 1);
        __syncwarp();
        if (lane == 0) mbar_arrive_rank(&tfull[t], 0);
        continue;
      }
      const uint32_t a_s = smem_u32(sA + s * A_BYTES);
      uint32_t x[32], hb[16], lb[16];
      if (MODE == MODE_AX) {
        // box {128 rows, 32 cols}, no swizzle: (row, k) at (k*128 + row)*4
#pragma unroll
        for (int k = 0; k < 32; ++k) x[k] = lds_u32(a_s + (uint32_t)((k * 128 + row) * 4));
      } else {
        // box {32 rows (K), 128 cols (M)}, 128B swizzle: (j, k) at j*128 + ((k/4 ^ j%8) * 16) + (k%4)*4
#pragma unroll
        for (int c = 0; c < 8; ++c)
          lds_u32x4(a_s + (uint32_t)(row * 128 + ((c ^ (row & 7)) * 16)), x[4 * c], x[4 * c + 1], x[4 * c + 2],
                    x[4 * c + 3]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&emptya[s]);  // the A stage is free once its values are in registers
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const uint32_t x0 = x[2 * k], x1 = x[2 * k + 1];
        const uint32_t h0 = (x0 + 0x1000u) & 0xFFFFE000u, h1 = (x1 + 0x1000u) & 0xFFFFE000u;  // rna tf32
        const __nv_bfloat162 lp = __floats2bfloat162_rn(__uint_as_float(x0) - __uint_as_float(h0),
                                                        __uint_as_float(x1) - __uint_as_float(h1));
        lb[k] = *reinterpret_cast<const uint32_t*>(&lp);
        if (TERMS == 3) {
          const __nv_bfloat162 hp = __floats2bfloat162_rn(__uint_as_float(h0), __uint_as_float(h1));
          hb[k] = *reinterpret_cast<const uint32_t*>(&hp);
        }
        x[2 * k] = h0;
        x[2 * k + 1] = h1;
      }
      mbar_wait(&tempty[t], tph ^ 1);
      // stage: [0, 32) a_h tf32; TERMS 3: [32, 48) bf16 a_h pairs (K' 0..31), [48, 64) bf16 a_l
      // pairs (K' 32..63); TERMS 2: [32, 48) bf16 a_l pairs
      const uint32_t ta = t_a + t * TSTR + lane_off;
      tmem_st16(ta, *reinterpret_cast<const uint32_t(*)[16]>(&x[0]));
      tmem_st16(ta + 16, *reinterpret_cast<const uint32_t(*)[16]>(&x[16]));
      if (TERMS == 3) {
        tmem_st16(ta + 32, hb);
        tmem_st16(ta + 48, lb);
      } else {
        tmem_st16(ta + 32, lb);
      }
      tc_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (leader) mbar_arrive(&tfull[t]);
        else mbar_arrive_rank(&tfull[t], 0);
      }
    }
  } else if (warp >= 12) {
    // flush warps: accumulator pieces -> fp32 registers -> output / partial slot
    const int wq = warp & 3;
    const int col0 = ((warp - 12) >> 2) * HALF;
    const int row = wq * 32 + lane;
    const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
    float sum[HALF];
#pragma unroll
    for (int j = 0; j < HALF; ++j) sum[j] = 0.f;
    P3Walk wk{g0, g1, nch};
    int64_t sb = g0;
    int tile, k0, k1;
    bool tf, tl;
    int piece = 0, seg = 0;
    int tile_k0 = 0;
    while (wk.next(tile, k0, k1, tf, tl, sb)) {
      if (tf) tile_k0 = k0;
      const int b = piece & 1;
      mbar_wait(&accfull[b], (piece >> 1) & 1);
      tc_fence_after();
      if (!(dbg & 16)) {
#pragma unroll
        for (int cb = 0; cb < HALF; cb += 16) {
          uint32_t v[16];
          tmem_ld16(t_acc0 + 128 * b + col0 + cb + lane_off, v);
          tc_wait_ld();
#pragma unroll
          for (int j = 0; j < 16; ++j) sum[cb + j] += __uint_as_float(v[j]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (leader) mbar_arrive(&accempty[b]);
        else mbar_arrive_rank(&accempty[b], 0);
      }
      ++piece;
      if (tl) {
        const bool whole = (tile_k0 == 0) && (k1 == nch);
        const int gm = (tile * CL + (int)crank) * 128 + row;
        if (whole) {
          if (gm < Mtot) {
#pragma unroll
            for (int j = 0; j < HALF; ++j) {
              const int c = col0 + j;
              if (rp_dev) {
                if (c < nact) out[gm + (int64_t)(rsh + c) * ldo] = sum[j];
                if (add && c < rsh) out[gm + (int64_t)c * ldo] = add[gm + (int64_t)c * ldadd];
              } else if (c < Nvalid) {
                float xv = sum[j];
                if (add) xv += add[gm + (int64_t)c * ldadd];
                out[gm + (int64_t)c * ldo] = xv;
              }
            }
          }
        } else {
          // slot 0: the range's first (partial) segment, slot 1: its last
          const int slot = (seg == 0) ? 0 : 1;
          float* p = part + ((int64_t)cta * P3_SLOTS + slot) * 128 * NP;
#pragma unroll
          for (int j = 0; j < HALF; ++j) p[(int64_t)(col0 + j) * 128 + row] = sum[j];
          // covering clusters of this work tile, and whether this CTA is the last to finish
          // (tile_cnt == nullptr: p3_fixup_kernel sums the slots after the pass)
          __shared__ int s_last;
          __shared__ int s_c0, s_c1;
          if (tile_cnt) {
          __threadfence();
          asm volatile("bar.sync 1, 256;" ::: "memory");  // the 8 flush warps
          if (warp == 12 && lane == 0) {
            const int64_t t0 = (int64_t)tile * nch, t1 = t0 + nch;
            int c0 = (int)((t0 * G) / total);
            while (c0 > 0 && sk_range_begin(total, G, c0) > t0) --c0;
            while (sk_range_begin(total, G, c0 + 1) <= t0) ++c0;
            int c1 = c0;
            while (c1 + 1 < G && sk_range_begin(total, G, c1 + 1) < t1) ++c1;
            int nc = 0;
            for (int cc = c0; cc <= c1; ++cc) nc += (sk_range_begin(total, G, cc + 1) > sk_range_begin(total, G, cc));
            const int atile = tile * CL + (int)crank;
            const unsigned int old = atomicAdd(&tile_cnt[atile], 1u);
            s_last = (old + 1 == (unsigned int)nc) ? 1 : 0;
            if (s_last) tile_cnt[atile] = 0u;  // re-arm for the next pass
            s_c0 = c0;
            s_c1 = c1;
          }
          asm volatile("bar.sync 1, 256;" ::: "memory");
          if (s_last) {
            __threadfence();
            const int64_t t0 = (int64_t)tile * nch;
            float* acc = sum;  // this CTA's own partial is re-read from its slot like the others
#pragma unroll
            for (int j = 0; j < HALF; ++j) acc[j] = 0.f;
            for (int cc = s_c0; cc <= s_c1; ++cc) {
              const int64_t bg = sk_range_begin(total, G, cc);
              if (sk_range_begin(total, G, cc + 1) <= bg) continue;
              const int sl = (bg >= t0) ? 0 : 1;
              const float* q = part + ((int64_t)(cc * CL + (int)crank) * P3_SLOTS + sl) * 128 * NP;
#pragma unroll
              for (int j = 0; j < HALF; ++j) acc[j] += __ldcg(q + (int64_t)(col0 + j) * 128 + row);
            }
            if (gm < Mtot) {
#pragma unroll
              for (int j = 0; j < HALF; ++j) {
                const int c = col0 + j;
                if (rp_dev) {
                  if (c < nact) out[gm + (int64_t)(rsh + c) * ldo] = acc[j];
                  if (add && c < rsh) out[gm + (int64_t)c * ldo] = add[gm + (int64_t)c * ldadd];
                } else if (c < Nvalid) {
                  float xv = acc[j];
                  if (add) xv += add[gm + (int64_t)c * ldadd];
                  out[gm + (int64_t)c * ldo] = xv;
                }
              }
            }
          }
          }  // tile_cnt
        }
#pragma unroll
        for (int j = 0; j < HALF; ++j) sum[j] = 0.f;
        ++seg;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // every MMA of the pair done, every TMEM read done, no more remote arrivals
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_cg2(tbase, 512);
  }
}

// Tiles split between MANY clusters (a pass with few output tiles, e.g. the
// A^T Q of a tall matrix with a narrow n): out = sum of the covering CTAs'
// partial slots in cluster order (+ add), one block per (row tile, fx_c <=
// P3_FX_C output columns) so the reduction runs on many SMs instead of in the
// last covering CTA. The same slots as the in-kernel fixup, summed in a fixed order
// (four interleaved slot groups, then the groups): deterministic. Grid (row
// tiles, column groups), 512 threads (128 rows x 4 slot groups; G <= 512).
constexpr int P3_FX_C = 8;
template <int NP>
__global__ void __launch_bounds__(512) p3_fixup_kernel(int Mtot, int Ktot, int Nvalid, int G,
                                                       const float* __restrict__ part, float* __restrict__ out,
                                                       int64_t ldo, const float* __restrict__ add, int64_t ldadd,
                                                       const int* __restrict__ rp_dev,
                                                       const int* __restrict__ skip_dev, int fx_c) {
  if (skip_dev && *skip_dev) return;  // the pass was skipped: nothing to sum
  constexpr int CL = 2;
  __shared__ int64_t soff[256];
  __shared__ int wcnt[16];
  const int nch = (Ktot + BK - 1) / BK;
  const int mtiles = (Mtot + 127) / 128;
  const int mgroups = (mtiles + CL - 1) / CL;
  const int64_t total = (int64_t)mgroups * nch;
  const int tile = blockIdx.x;
  const int wt = tile / CL, crank = tile % CL;
  // the slots covering this tile, in cluster order: thread cc examines
  // cluster cc's stream-K range [b0, b1) (G <= blockDim), then an ordered
  // compaction (a serial scan by one thread costs two 64-bit divisions per
  // cluster, ~15 us for 74 clusters)
  const int64_t t0 = (int64_t)wt * nch, t1 = t0 + nch;
  const int cc = threadIdx.x, wp = threadIdx.x >> 5, ln = threadIdx.x & 31;
  bool has = false, whole = false;
  int64_t off = 0;
  if (cc < G) {
    const int64_t b0 = sk_range_begin(total, G, cc), b1 = sk_range_begin(total, G, cc + 1);
    has = b1 > b0 && b0 < t1 && b1 > t0;
    whole = has && b0 <= t0 && b1 >= t1;
    off = ((int64_t)(cc * CL + crank) * P3_SLOTS + ((b0 >= t0) ? 0 : 1)) * 128 * NP;
  }
  const unsigned bal = __ballot_sync(0xffffffffu, has);
  if (ln == 0) wcnt[wp] = __popc(bal);
  const int anywhole = __syncthreads_or(whole ? 1 : 0);
  int kbase = 0, nc = 0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
    if (w < wp) kbase += wcnt[w];
    nc += wcnt[w];
  }
  if (has) soff[kbase + __popc(bal & ((1u << ln) - 1u))] = off;
  __syncthreads();
  if (anywhole) nc = 0;
  if (nc == 0) return;  // written directly by the pass
  const int rsh = rp_dev ? min(max(*rp_dev, 0), Nvalid) : 0;
  // fx_c output columns per block (the slot scan above is paid once per
  // block, not per column; the launch picks fx_c so that ~2 waves of blocks
  // remain); thread (g, row): row of the tile, slot group g of
  // FX_G (slots g, g + FX_G, ...), the groups summed in order afterwards
  // (deterministic). With ~150 slots per tile (narrow A^T Q: every cluster
  // touches the few tiles) the per-thread chain is nc / FX_G loads, 8 in flight.
  constexpr int FX_G = 4;
  __shared__ float gsum[FX_G - 1][128];
  const int row = threadIdx.x & 127, g = threadIdx.x >> 7, gm = tile * 128 + row;
  const bool live = gm < Mtot;
  for (int cj = 0; cj < fx_c; ++cj) {
    const int c = blockIdx.y * fx_c + cj;  // block-uniform
    if (c >= Nvalid) break;
    if (rp_dev && c < rsh) {  // carried column (copied unless the output is in place)
      if (g == 0 && live && add) out[gm + (int64_t)c * ldo] = add[gm + (int64_t)c * ldadd];
      continue;
    }
    const float* base = part + (int64_t)(c - rsh) * 128 + row;
    float acc = 0.f;
    if (live) {
      int k = g;
      for (; k + 7 * FX_G < nc; k += 8 * FX_G) {
        float v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldcg(base + soff[k + u * FX_G]);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += v[u];
      }
      for (; k < nc; k += FX_G) acc += __ldcg(base + soff[k]);
    }
    if (g > 0) gsum[g - 1][row] = acc;
    __syncthreads();
    if (g == 0 && live) {
#pragma unroll
      for (int q = 0; q < FX_G - 1; ++q) acc += gsum[q][row];
      if (add && !rp_dev) acc += add[gm + (int64_t)c * ldadd];
      out[gm + (int64_t)c * ldo] = acc;
    }
    __syncthreads();  // gsum is reused by the next column
  }
}

// B operand split of a TERMS = 2 pass: Bh = rna_tf32(x) (fp32, ld ldh) and
// Bb = bf16(Bh) (K-major rows of bf16, ld ldb, zero past `rows` up to a
// multiple of 32). One thread per two rows of a column.
__global__ void __launch_bounds__(256) split_tf32_bf16_kernel(const float* __restrict__ X, int64_t rows,
                                                              int64_t ldx_in, float* __restrict__ Bh, int64_t ldh,
                                                              __nv_bfloat16* __restrict__ Bb, int64_t ldb) {
  const int j = blockIdx.y;
  const int64_t k = ((int64_t)blockIdx.x * 256 + threadIdx.x) * 2;
  const int64_t kpad = ((rows + 31) / 32) * 32;
  if (k >= kpad) return;
  const float* xc = X + j * ldx_in;
  const float x0 = k < rows ? xc[k] : 0.f;
  const float x1 = k + 1 < rows ? xc[k + 1] : 0.f;
  const float h0 = __uint_as_float((__float_as_uint(x0) + 0x1000u) & 0xFFFFE000u);
  const float h1 = __uint_as_float((__float_as_uint(x1) + 0x1000u) & 0xFFFFE000u);
  float* bh = Bh + j * ldh;
  if (k < rows) bh[k] = h0;
  if (k + 1 < rows) bh[k + 1] = h1;
  *reinterpret_cast<__nv_bfloat162*>(Bb + k + j * ldb) = __floats2bfloat162_rn(h0, h1);
}

}  // namespace tc
}  // namespace frsvt
