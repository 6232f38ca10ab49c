// Persistent stream-K tcgen05 streaming pass over the m x n operand A (fp32
// handles): the GEMM-shaped steps of Algorithm 1 (PAPER.md P:128 sketch,
// P:141 power iteration, P:143/P:177 B = Q^T A).
//   MODE_AX : Y (m x l) = A (m x n) X (n x l)      M = rows of A, K = n
//   MODE_ATQ: Z (n x l) = A^T (n x m) Q (m x l)    M = columns of A, K = m
//
// Why this shape (measured on B200, profiles/r1_summary.md): A streams from
// HBM once per pass, but the small operand B (X or Q) is re-read from L2 for
// every 128-row tile. With B as fp32 hi + lo that is 2 bytes of L2 traffic
// per byte of A, and the L2 slice throughput (~6300 B/cycle chip-wide, the
// guide's LTS cap) was one bound of the old passes; here B is tf32 b_h (4 B)
// + bf16 [b_l | b_h] (4 B) per element, re-read from L2 per tile.
//
// Products (fp32-level: 1xTF32 misses 1e-4):
//   a b ~= a_h b_h + bf16(a_h) bf16(b_l) + bf16(a_l) bf16(b_h)
// with a_h = rna_tf32(a), a_l = a - a_h, b_h = rna_tf32(b), b_l = b - b_h.
// The dropped a_l b_l is ~2^-22 |ab|, the bf16 roundings of the two cross
// terms ~2^-19 |ab| each; measured relative error of a pass ~1e-6
// (tests/test_gpu_tc.py). The two cross terms are one bf16 product over a
// doubled K: [bf16(a_h) | bf16(a_l)] . [bf16(b_l) ; bf16(b_h)]. Per 32-wide K
// chunk: 4 tf32 MMAs (K = 8) + 4 bf16 MMAs (K = 16); measured on B200 (all
// SMs busy, scripts/mma_rate.py) 70 and 81.5 cycles each, 606 tensor cycles
// per 16 KB of A (3xTF32: 840). Under the 1 kW cap the SM clock settles near
// 1.35 GHz during a pass, so tensor cycles, not HBM, bound these passes.
//
// Work: the M tiles x K chunks of the pass are flattened tile-major and cut
// into gridDim.x contiguous ranges, one per CTA (stream-K): every SM streams
// the same number of chunks, no wave tail. A range covering a whole tile
// writes it directly; a tile split between CTAs leaves partial sums in a
// per-CTA slot (first or last segment of the range), and the CTA that
// finishes a split tile last (per-tile arrival counter) adds all its slots in
// CTA order (deterministic). Small K (the l x l applies): whole tiles per CTA.
//
// Roles per CTA (640 threads; 2-CTA clusters multicast the B stages):
//   warp 0      TMA producer of A (16 KB chunks, 4-deep ring, released as soon as
//               the converters hold the values in registers)
//   warp 3      TMA producer of B_h (tf32) + B_x (bf16 [b_l | b_h]), both
//               128B swizzle, 5-deep ring released by the MMAs of both CTAs
//   warp 1      MMA issuer (one thread); A operands from TMEM, B from smem
//   warp 2      TMEM allocator
//   warps 4..11 converters, two groups of four (one warp per TMEM lane
//               quarter) on alternate chunks: A chunk -> a_h (tf32) and bf16
//               [a_h | a_l] pairs -> TMEM ring (thread = TMEM lane = M row)
//   warps 12..19 flush: double-buffered TMEM accumulator pieces (<= SEG
//               chunks, never across a tile) -> fp32 registers -> output
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include "tc_pass.cuh"

namespace frsvt {
namespace tc {

#ifndef P2_AST
#define P2_AST 4
#endif
#ifndef P2_BST
#define P2_BST 5
#endif
constexpr int P2_ASTAGES = P2_AST;  // A ring (16 KB stages; released by the converters; even)
// the A ring of an NP-column instance: the narrow (NP <= 32) B stages leave room for 8 stages
__host__ __device__ constexpr int p2_astages(int np) { return np <= 32 ? 8 : P2_ASTAGES; }
// B ring: released by the MMA. Its depth must cover MMA completion (~700
// cycles) + the L2 latency of the small operand under the A stream (~1900
// cycles, clock64 stamps): 5 stages of (roundup8(l) rows x 256 B)
constexpr int P2_BSTAGES = P2_BST;
constexpr int P2_TSTAGES = 4;  // TMEM A ring (64 columns per stage: a_h tf32 | bf16 a_h | bf16 a_l)
constexpr int P2_SEG = 8;      // chunks accumulated in TMEM before a flush
constexpr int P2_THREADS = 640;
constexpr int P2_SLOTS = 2;    // partial-tile slots per CTA

struct Pass2Smem {
  static constexpr uint32_t a_bytes = 128u * BK * 4u;         // 16 KB
  static constexpr uint32_t bh_bytes = 128u * BK * 4u;        // 16 KB (N <= 128 rows)
  static constexpr uint32_t bx_bytes = 128u * 2 * BK * 2u;    // 16 KB: bf16 [b_l | b_h], 64 K per row
  static constexpr uint32_t b_bytes = bh_bytes + bx_bytes;    // 32 KB
  // one B stage for nb valid rows (128B-swizzle atoms are 8 rows = 1 KB)
  __host__ __device__ static constexpr uint32_t b_stage(int nb) { return 2u * (uint32_t)((nb + 7) / 8) * 1024u; }
  __host__ __device__ static constexpr size_t total(int nb, int ast = P2_ASTAGES) {
    return 1024 + (size_t)ast * a_bytes + (size_t)P2_BSTAGES * b_stage(nb) + 512;
  }
};

// Shared-memory descriptor: K-major, 64-byte swizzle (bf16 rows of 32 K), 8-row groups 512 B apart.
__device__ __forceinline__ uint64_t desc_kmajor_sw64(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1u << 16) | ((uint64_t)(512u >> 4) << 32) |
         ((uint64_t)1u << 46) | ((uint64_t)4u << 61);
}
// Instruction descriptor: D fp32, A/B bf16 (kind::f16), both K-major, M x N.
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(
          d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
               "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t saddr) {
  uint32_t v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(saddr) : "memory");
  return v;
}
__device__ __forceinline__ void lds_u32x4(uint32_t saddr, uint32_t& a, uint32_t& b, uint32_t& c, uint32_t& d) {
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "r"(saddr) : "memory");
}

__device__ __forceinline__ uint64_t p2_gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// per-CTA global-timer stamps (dbg bit 6): [cta][0] entry, [1] producer done, [2] flush done, [3] exit
__device__ __forceinline__ void p2_cta_stamp(int dbg, float* out, int ev) {
  if (dbg & 64) reinterpret_cast<uint64_t*>(out)[40000 + blockIdx.x * 4 + ev] = p2_gtime();
}
__device__ __forceinline__ void p2_stamp(int dbg, float* out, int ev, int i, int nloc) {
  if ((dbg & 32) && blockIdx.x == 0 && i < 4096) {
    uint64_t* t = reinterpret_cast<uint64_t*>(out);
    t[(int64_t)ev * 4096 + i] = clock64();
  }
}

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// TMA 2D load multicast to the CTAs in ctaMask (same smem offset in each; each
// destination's mbarrier at the same offset receives the complete_tx)
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                               uint16_t mask, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster.L2::cache_hint "
      "[%0], [%1, {%3, %4}], [%2], %5, %6;" ::"r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tc_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                   smem_u32(bar)),
               "h"(mask)
               : "memory");
}
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n.reg .pred p;\nelect.sync _|p, 0xffffffff;\nselp.u32 %0, 1, 0, p;\n}" : "=r"(pred));
  return pred != 0;
}

// Chunk range of CTA c: [c * total / G, (c + 1) * total / G).
__host__ __device__ __forceinline__ int64_t p2_range_begin(int64_t total, int G, int c) {
  return (total * c) / G;
}

// Walks the CTA's chunk range as a sequence of accumulator pieces: at most
// P2_SEG chunks, never crossing a tile. All roles iterate it identically.
struct P2Walk {
  int64_t g, g1;   // next chunk, end of range
  int nch;         // chunks per tile
  __device__ __forceinline__ bool next(int& tile, int& k0, int& k1, bool& tile_first, bool& tile_last,
                                       int64_t& seg_begin) {
    if (g >= g1) return false;
    tile = (int)(g / nch);
    k0 = (int)(g - (int64_t)tile * nch);
    const int64_t tile_end = (int64_t)(tile + 1) * nch;
    const int64_t end = min(g1, tile_end);
    tile_first = (g == seg_begin);
    int kk = k0 + P2_SEG;
    k1 = (int)min((int64_t)kk, end - (int64_t)tile * nch);
    g = (int64_t)tile * nch + k1;
    tile_last = (g == end);
    if (tile_last) seg_begin = g;
    return true;
  }
};

// CL = 2: the CTAs of a 2-CTA cluster take the two 128-row tiles of a
// 256-row pair over the same K chunks; each loads half of every B stage and
// multicasts it to both (halving the B traffic through L2, which the passes
// were bound by: A + B re-reads ~ 2.9x A at the ~12 TB/s LTS cap), and a
// B stage is reused only after both CTAs' MMAs consumed it.
template <int MODE, int NP, int CL>
__global__ void __launch_bounds__(P2_THREADS, 1)
tc_pass2_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapBh,
                const __grid_constant__ CUtensorMap mapBl, int Mtot, int Ktot, int Nvalid, int nbrows,
                float* __restrict__ out, int64_t ldo, const float* __restrict__ add, int64_t ldadd,
                float* __restrict__ part, const int* __restrict__ rp_dev, int dbg,
                unsigned int* __restrict__ tile_cnt, const int* __restrict__ skip_dev) {
  // skip_dev (nullable): the output was already formed (fused next sketch)
  if (skip_dev && *skip_dev) return;
  // tile_cnt (nullable, >= mtiles zeros): in-kernel stream-K fixup. The CTA
  // that completes the last partial segment of a split tile sums all its
  // partial slots in CTA order (deterministic), writes the tile and re-arms
  // the counter (tile_cnt is required whenever a tile can be split).
  // rp_dev (MODE_AX, range propagation): r = *rp_dev carried columns; only the
  // p = Nvalid - r fresh columns are multiplied (B holds them at [0, p), the
  // MMA runs with N = roundup16(p)) and land in out[:, r + c]; out[:, :r] is a
  // copy of add[:, :r] (the carry Q~).
  // dbg (test hook only, 0 in production): bit 0 no MMA, bit 1 no conversion, bit 2 no B loads,
  // bit 3 no bf16 MMAs, bit 4 no a_lo MMAs, bit 5 clock64 stamps of CTA 0 into out (output invalid)
  static_assert(NP % 16 == 0 && NP >= 32 && NP <= 128, "N tile");
  constexpr int AST = p2_astages(NP);
  constexpr uint32_t A_BYTES = Pass2Smem::a_bytes;
  const uint32_t B_BYTES = Pass2Smem::b_stage(CL > 1 ? NP : nbrows);  // Bh | Bx, each rows x 128 B
  const uint32_t BHB = B_BYTES / 2;
  constexpr int HALF = NP / 2;  // columns per flush warp
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;                                   // AST x 16 KB
  uint8_t* sB = smem + AST * A_BYTES;            // P2_BSTAGES x B_BYTES
  uint64_t* fulla = (uint64_t*)(sB + P2_BSTAGES * B_BYTES);
  uint64_t* emptya = fulla + AST;
  uint64_t* fullb = emptya + AST;
  uint64_t* emptyb = fullb + P2_BSTAGES;
  uint64_t* tfull = emptyb + P2_BSTAGES;
  uint64_t* tempty = tfull + P2_TSTAGES;
  uint64_t* accfull = tempty + P2_TSTAGES;
  uint64_t* accempty = accfull + 2;
  uint32_t* tslot = (uint32_t*)(accempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) p2_cta_stamp(dbg, out, 0);
  const int rsh = rp_dev ? min(max(*rp_dev, 0), Nvalid) : 0;   // output column shift
  const int nact = Nvalid - rsh;                               // multiplied columns
  // MMA N: the valid columns rounded up to 8 (N steps of 8 are legal at
  // cta_group::1; measured 60 cycles at N = 120 vs 64 at 128)
  const int nmma = min(NP, max(16, ((rp_dev ? nact : Nvalid) + 7) & ~7));
  const int nch = (Ktot + BK - 1) / BK;
  const int mtiles = (Mtot + 127) / 128;
  const int mgroups = (mtiles + CL - 1) / CL;  // work tiles: CL row tiles each
  const int64_t total = (int64_t)mgroups * nch;
  const int crank = CL > 1 ? (int)cluster_ctarank() : 0;
  const int G = gridDim.x / CL, cta = blockIdx.x, cgrp = blockIdx.x / CL;
  // dbg bit 8 (small K): ranges of whole work tiles, so no tile is split and
  // no partial slots or fixup are needed
  const bool talign = (dbg & 256) != 0;
  const int64_t g0 = talign ? ((int64_t)mgroups * cgrp / G) * nch : p2_range_begin(total, G, cgrp);
  const int64_t g1 = talign ? ((int64_t)mgroups * (cgrp + 1) / G) * nch : p2_range_begin(total, G, cgrp + 1);
  const int nloc = (int)(g1 - g0);
  // expected TMA bytes per B stage (CL = 1: boxes of nbrows rows; CL = 2: both
  // CTAs' 64-row halves, out-of-bounds rows zero-filled and counted)
  const uint32_t brows = CL > 1 ? (uint32_t)NP : (uint32_t)nbrows;
  const uint32_t btx = brows * BK * 4u + brows * 2 * BK * 2u;

  if (threadIdx.x == 0) {
    for (int s = 0; s < AST; ++s) {
      mbar_init(&fulla[s], 1);
      mbar_init(&emptya[s], 4);
    }
    for (int s = 0; s < P2_BSTAGES; ++s) {
      mbar_init(&fullb[s], 1);
      mbar_init(&emptyb[s], CL);
    }
    for (int t = 0; t < P2_TSTAGES; ++t) {
      mbar_init(&tfull[t], 4);
      mbar_init(&tempty[t], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&accfull[b], 1);
      mbar_init(&accempty[b], 8);
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    tmem_alloc(tslot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  if (CL > 1) cluster_sync_all();  // barriers initialised before the partner multicasts into them
  tc_fence_after();
  const uint32_t tbase = *tslot;
  const uint32_t t_acc0 = tbase;     // accumulator buffer b at columns [128 b, 128 b + NP)
  const uint32_t t_a = tbase + 256;  // A ring: stage t at 256 + 64 t

  if (warp == 0) {
    // A producer (HBM stream, deep ring)
    if (lane == 0 && nloc > 0) {
      prefetch_tmap(&mapA);
      const uint64_t pol = l2_policy_evict_first();
      for (int i = 0; i < nloc; ++i) {
        const int64_t g = g0 + i;
        const int grp = (int)(g / nch), kc = (int)(g - (int64_t)grp * nch) * BK;
        const int tile = grp * CL + crank;
        const int s = i % AST;
        const uint32_t ph = (i / AST) & 1;
        mbar_wait(&emptya[s], ph ^ 1);
        p2_stamp(dbg, out, 0, i, nloc);
        mbar_expect_tx(&fulla[s], A_BYTES);
        if (MODE == MODE_AX)
          tma_load_2d_hint(sA + s * A_BYTES, &mapA, &fulla[s], tile * 128, kc, pol);
        else
          tma_load_2d_hint(sA + s * A_BYTES, &mapA, &fulla[s], kc, tile * 128, pol);
      }
      p2_cta_stamp(dbg, out, 1);
    }
  } else if (warp == 3) {
    // B producer (L2-resident small operand)
    if (lane == 0 && nloc > 0) {
      prefetch_tmap(&mapBh);
      prefetch_tmap(&mapBl);
      const uint64_t pol = l2_policy_evict_last();
      for (int i = 0; i < nloc; ++i) {
        const int64_t g = g0 + i;
        const int grp = (int)(g / nch), kc = (int)(g - (int64_t)grp * nch) * BK;
        const int s = i % P2_BSTAGES;
        const uint32_t ph = (i / P2_BSTAGES) & 1;
        mbar_wait(&emptyb[s], ph ^ 1);
        p2_stamp(dbg, out, 6, i, nloc);
        if (dbg & 4) {
          mbar_arrive(&fullb[s]);
          continue;
        }
        mbar_expect_tx(&fullb[s], btx);
        if (CL > 1) {  // my NP/2-row half of the stage, into both CTAs
          const uint32_t ho = (uint32_t)crank * (uint32_t)(NP / 2) * 128u;
          tma_load_2d_mc(sB + s * B_BYTES + ho, &mapBh, &fullb[s], kc, (NP / 2) * crank, 0x3, pol);
          tma_load_2d_mc(sB + s * B_BYTES + BHB + ho, &mapBl, &fullb[s], 2 * kc, (NP / 2) * crank, 0x3, pol);
        } else {
          tma_load_2d_hint(sB + s * B_BYTES, &mapBh, &fullb[s], kc, 0, pol);
          tma_load_2d_hint(sB + s * B_BYTES + BHB, &mapBl, &fullb[s], 2 * kc, 0, pol);
        }
      }
    }
  } else if (warp == 1) {
    // The whole warp walks the schedule (warp-uniform values stay in uniform
    // registers); one elected lane issues the tcgen05 instructions.
    if (nloc > 0) {
      const uint32_t id_tf = idesc_tf32(128, nmma);
      const uint32_t id_bf = idesc_bf16(128, nmma);
      const bool leader = elect_one();
      P2Walk wk{g0, g1, nch};
      int64_t sb = g0;
      int tile, k0, k1;
      bool tf, tl;
      int i = 0, piece = 0;
      const uint32_t sB_u = smem_u32(sB);
      while (wk.next(tile, k0, k1, tf, tl, sb)) {
        const int b = piece & 1;
        mbar_wait(&accempty[b], ((piece >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t acc = t_acc0 + 128 * b;
        for (int kc = k0; kc < k1; ++kc, ++i) {
          const int s = i % P2_BSTAGES;
          const uint32_t ph = (i / P2_BSTAGES) & 1;
          const int t = i % P2_TSTAGES;
          const uint32_t tph = (i / P2_TSTAGES) & 1;
          mbar_wait(&fullb[s], ph);
          if (leader) p2_stamp(dbg, out, 7, i, nloc);
          mbar_wait(&tfull[t], tph);
          tc_fence_after();
          if (leader) p2_stamp(dbg, out, 4, i, nloc);
          if (dbg & 1) {
            if (leader) {
              if (CL > 1) tc_commit_mc(&emptyb[s], 0x3);
              else mbar_arrive(&emptyb[s]);
              mbar_arrive(&tempty[t]);
            }
            __syncwarp();
            continue;
          }
          const uint32_t st = sB_u + (uint32_t)s * B_BYTES;
          const uint64_t bh = desc_kmajor_sw128(st);
          const uint64_t bx = desc_kmajor_sw128(st + BHB);
          const uint32_t a_hi = t_a + t * 64, a_x = a_hi + 32;
          if (leader) {
#pragma unroll
            for (int kk = 0; kk < BK / 8; ++kk) {
              const uint64_t koff = (uint64_t)(kk * 32) >> 4;  // 8 tf32 = 32 bytes along K
              mma_tf32_ts(acc, a_hi + kk * 8, bh + koff, id_tf, (kc > k0 || kk > 0) ? 1u : 0u);
            }
            if (!(dbg & 8)) {
#pragma unroll
              for (int kk = 0; kk < 2 * BK / 16; ++kk) {
                const uint64_t koff = (uint64_t)(kk * 32) >> 4;  // 16 bf16 = 32 bytes along K'
                mma_bf16_ts(acc, a_x + kk * 8, bx + koff, id_bf, 1u);
              }
            }
            if (CL > 1) tc_commit_mc(&emptyb[s], 0x3);  // frees stage s in both CTAs
            else tc_commit(&emptyb[s]);
            tc_commit(&tempty[t]);
            p2_stamp(dbg, out, 5, i, nloc);
          }
          __syncwarp();
        }
        if (leader) {
          if (dbg & 1) mbar_arrive(&accfull[b]);
          else tc_commit(&accfull[b]);
        }
        __syncwarp();
        ++piece;
      }
    }
  } else if (warp >= 4 && warp < 12) {
    // converters: A chunk in shared memory -> a_h, a_l, bf16(a_h) -> TMEM ring.
    // Two groups of four warps (one per TMEM lane quarter) take alternate
    // chunks, each warp converting all 32 K of its 32 rows, so two chunks
    // are in conversion at once (the load -> convert -> tcgen05.st -> wait
    // chain of one chunk overlaps the other's).
    const int wq = warp & 3, grp = (warp - 4) >> 2;
    const int row = wq * 32 + lane;
    const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
    for (int i = grp; i < nloc; i += 2) {
      const int s = i % AST;
      const uint32_t ph = (i / AST) & 1;
      const int t = i % P2_TSTAGES;
      const uint32_t tph = (i / P2_TSTAGES) & 1;
      mbar_wait(&fulla[s], ph);
      if (warp == 4 && lane == 0) p2_stamp(dbg, out, 1, i, nloc);
      if (dbg & 2) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&emptya[s]);
        mbar_wait(&tempty[t], tph ^ 1);
        __syncwarp();
        if (lane == 0) mbar_arrive(&tfull[t]);
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
      // the A stage is free once its values are in registers
      __syncwarp();
      if (lane == 0) mbar_arrive(&emptya[s]);
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const uint32_t x0 = x[2 * k], x1 = x[2 * k + 1];
        const uint32_t h0 = (x0 + 0x1000u) & 0xFFFFE000u, h1 = (x1 + 0x1000u) & 0xFFFFE000u;  // rna tf32
        const __nv_bfloat162 hp = __floats2bfloat162_rn(__uint_as_float(h0), __uint_as_float(h1));
        const __nv_bfloat162 lp = __floats2bfloat162_rn(__uint_as_float(x0) - __uint_as_float(h0),
                                                        __uint_as_float(x1) - __uint_as_float(h1));
        hb[k] = *reinterpret_cast<const uint32_t*>(&hp);
        lb[k] = *reinterpret_cast<const uint32_t*>(&lp);
        x[2 * k] = h0;
        x[2 * k + 1] = h1;
      }
      mbar_wait(&tempty[t], tph ^ 1);
      if (warp == 4 && lane == 0) p2_stamp(dbg, out, 2, i, nloc);
      // stage layout: [0, 32) a_h tf32; [32, 48) bf16 a_h pairs (K' 0..31); [48, 64) bf16 a_l pairs (K' 32..63)
      const uint32_t ta = t_a + t * 64 + lane_off;
      tmem_st16(ta, *reinterpret_cast<const uint32_t(*)[16]>(&x[0]));
      tmem_st16(ta + 16, *reinterpret_cast<const uint32_t(*)[16]>(&x[16]));
      tmem_st16(ta + 32, hb);
      tmem_st16(ta + 48, lb);
      tc_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tfull[t]);
      if (warp == 4 && lane == 0) p2_stamp(dbg, out, 3, i, nloc);
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
    P2Walk wk{g0, g1, nch};
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
#pragma unroll
      for (int cb = 0; cb < HALF; cb += 16) {
        uint32_t v[16];
        tmem_ld16(t_acc0 + 128 * b + col0 + cb + lane_off, v);
        tc_wait_ld();
#pragma unroll
        for (int j = 0; j < 16; ++j) sum[cb + j] += __uint_as_float(v[j]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&accempty[b]);
      ++piece;
      if (tl && !(dbg & 96)) {
        const bool whole = (tile_k0 == 0) && (k1 == nch);
        const int gm = (tile * CL + crank) * 128 + row;
        if (whole) {
          if (gm < Mtot) {
#pragma unroll
            for (int j = 0; j < HALF; ++j) {
              const int c = col0 + j;
              if (rp_dev) {
                if (c < nact) out[gm + (int64_t)(rsh + c) * ldo] = sum[j];
                if (add && c < rsh) out[gm + (int64_t)c * ldo] = add[gm + (int64_t)c * ldadd];
              } else if (c < Nvalid) {
                float x = sum[j];
                if (add) x += add[gm + (int64_t)c * ldadd];
                out[gm + (int64_t)c * ldo] = x;
              }
            }
          }
        } else {
          // slot 0: the range's first (partial) segment, slot 1: its last
          const int slot = (seg == 0) ? 0 : 1;
          float* p = part + ((int64_t)cta * P2_SLOTS + slot) * 128 * NP;
#pragma unroll
          for (int j = 0; j < HALF; ++j) p[(int64_t)(col0 + j) * 128 + row] = sum[j];
          if (tile_cnt) {
            // covering work groups of this work tile, and whether this CTA is the last to finish
            __shared__ int s_last;
            __shared__ int s_c0, s_c1;
            __threadfence();
            asm volatile("bar.sync 1, 256;" ::: "memory");  // the 8 flush warps
            if (warp == 12 && lane == 0) {
              const int64_t t0 = (int64_t)tile * nch, t1 = t0 + nch;
              int c0 = (int)((t0 * G) / total);
              while (c0 > 0 && p2_range_begin(total, G, c0) > t0) --c0;
              while (p2_range_begin(total, G, c0 + 1) <= t0) ++c0;
              int c1 = c0;
              while (c1 + 1 < G && p2_range_begin(total, G, c1 + 1) < t1) ++c1;
              int nc = 0;
              for (int cc = c0; cc <= c1; ++cc) nc += (p2_range_begin(total, G, cc + 1) > p2_range_begin(total, G, cc));
              const int atile = tile * CL + crank;
              const unsigned int old = atomicAdd(&tile_cnt[atile], 1u);
              s_last = (old + 1 == (unsigned int)nc) ? 1 : 0;
              if (s_last) tile_cnt[atile] = 0u;  // re-arm for the next pass
              s_c0 = c0;
              s_c1 = c1;
            }
            asm volatile("bar.sync 1, 256;" ::: "memory");
            if (s_last) {
              __threadfence();
              const int gm = (tile * CL + crank) * 128 + row;
              const int64_t t0 = (int64_t)tile * nch;
              float* acc = sum;  // this CTA's own partial is re-read from its slot like the others
#pragma unroll
              for (int j = 0; j < HALF; ++j) acc[j] = 0.f;
              for (int cc = s_c0; cc <= s_c1; ++cc) {
                const int64_t b = p2_range_begin(total, G, cc);
                if (p2_range_begin(total, G, cc + 1) <= b) continue;
                const int sl = (b >= t0) ? 0 : 1;
                const float* q = part + ((int64_t)(cc * CL + crank) * P2_SLOTS + sl) * 128 * NP;
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
                    float x = acc[j];
                    if (add) x += add[gm + (int64_t)c * ldadd];
                    out[gm + (int64_t)c * ldo] = x;
                  }
                }
              }
            }
          }
        }
#pragma unroll
        for (int j = 0; j < HALF; ++j) sum[j] = 0.f;
        ++seg;
      }
    }
  }
  if (warp == 12 && lane == 0) p2_cta_stamp(dbg, out, 2);
  tc_fence_before();
  __syncthreads();
  if (CL > 1) cluster_sync_all();  // the partner no longer multicasts into this CTA
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tbase, 512);
  }
  if (threadIdx.x == 0) p2_cta_stamp(dbg, out, 3);
}

// B operand split: Bh = rna_tf32(x) (fp32, rows x cols, ld ldh) and Bx (bf16,
// (2 * roundup32(rows)) x cols, ld ldx): for K chunk c, Bx rows 64c + j hold
// bf16(x - Bh) at K = 32c + j (j < 32) and bf16(Bh) at K = 32c + j - 32
// (j >= 32), zero past `rows`. One thread per two rows of a column, writing both halves.
__global__ void __launch_bounds__(256) split_tf32_bf16x2_kernel(const float* __restrict__ X, int64_t rows, int64_t cols,
                                                                  int64_t ldx_in, float* __restrict__ Bh, int64_t ldh,
                                                                  __nv_bfloat16* __restrict__ Bx, int64_t ldx) {
  // grid (chunks of 512 rows, cols): thread = rows k, k + 1 of column j
  // (packed bf16x2 / float2 stores; X, Bh column starts are 8-byte aligned
  // when ldx_in, ldh are even, else the scalar path)
  const int j = blockIdx.y;
  const int64_t k = ((int64_t)blockIdx.x * 256 + threadIdx.x) * 2;
  const int64_t kpad = ((rows + 31) / 32) * 32;
  if (k >= kpad) return;
  float x0 = 0.f, x1 = 0.f;
  const float* xc = X + j * ldx_in;
  if (k + 1 < rows && ((ldx_in | ldh) & 1) == 0) {
    const float2 v = *reinterpret_cast<const float2*>(xc + k);
    x0 = v.x;
    x1 = v.y;
  } else {
    if (k < rows) x0 = xc[k];
    if (k + 1 < rows) x1 = xc[k + 1];
  }
  const float h0 = k < rows ? __uint_as_float((__float_as_uint(x0) + 0x1000u) & 0xFFFFE000u) : 0.f;
  const float h1 = k + 1 < rows ? __uint_as_float((__float_as_uint(x1) + 0x1000u) & 0xFFFFE000u) : 0.f;
  float* bh = Bh + j * ldh;
  if (k + 1 < rows && ((ldx_in | ldh) & 1) == 0) {
    *reinterpret_cast<float2*>(bh + k) = make_float2(h0, h1);
  } else {
    if (k < rows) bh[k] = h0;
    if (k + 1 < rows) bh[k + 1] = h1;
  }
  const int64_t base = (k >> 5) * 64 + (k & 31) + j * ldx;  // k even: (k, k+1) in the same 32-chunk
  *reinterpret_cast<__nv_bfloat162*>(Bx + base) = __floats2bfloat162_rn(x0 - h0, x1 - h1);
  *reinterpret_cast<__nv_bfloat162*>(Bx + base + 32) = __floats2bfloat162_rn(h0, h1);
}

}  // namespace tc
}  // namespace frsvt
