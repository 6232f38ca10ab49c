// tcgen05 (5th-gen tensor core) streaming passes over the m x n operand A for
// fp32 handles, in 3xTF32 (split) precision:
//   MODE_AX : Y (m x l) = A (m x n) * X (n x l)      M = rows of A, K = n
//   MODE_ATQ: Z (n x l) = A^T (n x m) * Q (m x l)    M = columns of A, K = m (split-K)
// These are the GEMM-shaped steps of Algorithm 1 (PAPER.md P:128 sketch,
// P:141 power iteration, P:143/P:177 B = Q^T A). fp32-level products are
// required on every pass (1xTF32 misses 1e-4), so each product
// is a_hi*b_hi + a_hi*b_lo + a_lo*b_hi with hi = rna_tf32(x), lo = x - hi.
//
// Per CTA: one 128-row M tile, N = NP (l rounded up to 16), K streamed in
// 32-wide chunks.
//   warp 0      TMA producer: raw A tile (16 KB) + B_hi/B_lo tiles (K-major,
//               128B swizzle) into a 4-stage shared-memory ring
//   warp 1      MMA issuer (one thread): 3 x tcgen05.mma.kind::tf32 per K=8
//               step, A operand from TMEM, B from shared memory, fp32
//               accumulator in TMEM
//   warp 2      TMEM allocator
//   warps 4..7  converters: shared A tile -> (hi, lo) -> tcgen05.st into a
//               4-stage TMEM ring (thread = TMEM lane = M row)
//   warps 8..15 flush + epilogue: double-buffered TMEM accumulator segments
//               -> fp32 registers (tcgen05.ld) -> global
// A passes through shared memory once (TMA write + one LDS per element) and
// never through the MMA's shared-memory read port, which keeps the 3xTF32
// split off the shared-memory bandwidth roofline.
#pragma once
#include <cuda.h>

#include "common.cuh"

namespace frsvt {
namespace tc {

constexpr int MODE_AX = 0;
constexpr int MODE_ATQ = 1;
constexpr int BK = 32;      // K per stage (one 128-byte swizzle atom of fp32)
constexpr int STAGES = 4;   // shared-memory ring depth
constexpr int TSTAGES = 4;  // TMEM A ring depth

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("{\n.reg .b64 st;\nmbarrier.arrive.shared::cta.b64 st, [%0];\n}" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("{\n.reg .b64 st;\nmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  const uint32_t a = smem_u32(b);
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.b32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"((uint64_t)map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
// TMA load with an L2 eviction-priority policy (createpolicy): the streamed
// big operand is marked evict_first, the re-read small operands evict_last,
// so the 2 GB stream does not flush the L2-resident small operand
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tma_load_2d_hint(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                                 uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, "
      "%4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)m) : "memory");
}
__device__ __forceinline__ void tmem_alloc(uint32_t* slot, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void tmem_relinquish() {
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// D[tmem] (+)= A[tmem] * B[smem desc], kind::tf32, fp32 accumulate
__device__ __forceinline__ void mma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(
          d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Instruction descriptor: D fp32, A/B tf32, both K-major, M x N.
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
// Shared-memory descriptor: K-major, 128-byte swizzle, 8-row groups 1024 B apart.
__device__ __forceinline__ uint64_t desc_kmajor_sw128(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1u << 16) | ((uint64_t)(1024u >> 4) << 32) |
         ((uint64_t)1u << 46) | ((uint64_t)2u << 61);
}

__device__ __forceinline__ uint32_t rna_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

#define FRSVT_R32(v)                                                                                     \
  "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),     \
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),     \
      "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),    \
      "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
#define FRSVT_W32(v)                                                                                     \
  "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),         \
      "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),           \
      "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),         \
      "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),         \
      "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
#define FRSVT_ARGS32                                                                                     \
  "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, " \
  "%23, %24, %25, %26, %27, %28, %29, %30, %31, %32}"
#define FRSVT_OUTS32                                                                                     \
  "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, " \
  "%22, %23, %24, %25, %26, %27, %28, %29, %30, %31}"

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], " FRSVT_ARGS32 ";" ::"r"(taddr), FRSVT_R32(v)
               : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 " FRSVT_OUTS32 ", [%32];" : FRSVT_W32(v) : "r"(taddr)
               : "memory");
}

struct PassSmem {
  static constexpr uint32_t a_bytes = 128u * BK * 4u;
  __host__ __device__ static constexpr uint32_t b_bytes(int np) { return (uint32_t)np * BK * 4u; }
  __host__ __device__ static constexpr size_t total(int np) {
    return 1024 + (size_t)STAGES * (a_bytes + 2 * b_bytes(np)) + 256;
  }
};

constexpr int SEG = 8;            // K chunks accumulated in TMEM before a flush
constexpr int PASS_THREADS = 512; // 16 warps

// out[z*zstride + row + c*ldo] = D(row, c) (+ add[row + c*ldadd]) for row < Mtot, c < Nvalid
//
// Accuracy: the tensor core adds each MMA result into the fp32 accumulator
// with truncation, so its error grows with the number of accumulations
// (measured: ~2e-6 relative per 256 of K). The accumulator is therefore
// double-buffered in TMEM and flushed every SEG chunks (K = 256) into fp32
// registers of 8 flush warps (round-to-nearest adds), which keeps a pass over
// K = 65536 at the error of a K = 256 product.
template <int MODE, int NP>
__global__ void __launch_bounds__(PASS_THREADS, 1)
tc_pass_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapBhi,
               const __grid_constant__ CUtensorMap mapBlo, int Mtot, int Ktot, int chunks_per_split,
               int Nvalid, float* __restrict__ out, int64_t ldo, int64_t zstride,
               const float* __restrict__ add, int64_t ldadd) {
  static_assert(NP % 16 == 0 && NP >= 32 && NP <= 128, "N tile");
  constexpr uint32_t A_BYTES = PassSmem::a_bytes;
  constexpr uint32_t B_BYTES = PassSmem::b_bytes(NP);
  constexpr int HALF = NP / 2;  // columns per flush warp
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  float* sA = (float*)smem;
  uint8_t* sBh = smem + STAGES * A_BYTES;
  uint8_t* sBl = sBh + STAGES * B_BYTES;
  uint64_t* full = (uint64_t*)(sBl + STAGES * B_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + TSTAGES;
  uint64_t* accfull = tempty + TSTAGES;
  uint64_t* accempty = accfull + 2;
  uint32_t* tslot = (uint32_t*)(accempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mt = blockIdx.x, z = blockIdx.y;
  const int nchunks = (Ktot + BK - 1) / BK;
  const int c_begin = z * chunks_per_split;
  const int c_end = min(nchunks, c_begin + chunks_per_split);
  const int nch = max(0, c_end - c_begin);
  const int nseg = (nch + SEG - 1) / SEG;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1 + 4);
    }
    for (int t = 0; t < TSTAGES; ++t) {
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
  tc_fence_after();
  const uint32_t tbase = *tslot;
  const uint32_t t_acc0 = tbase;        // accumulator buffer b at columns [128 b, 128 b + NP)
  const uint32_t t_a = tbase + 256;     // A ring: stage t at 256 + 64 t (hi), +32 (lo)

  if (warp == 0) {
    if (lane == 0) {
      prefetch_tmap(&mapA);
      prefetch_tmap(&mapBhi);
      prefetch_tmap(&mapBlo);
      for (int i = 0; i < nch; ++i) {
        const int s = i % STAGES;
        const uint32_t ph = (i / STAGES) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        mbar_expect_tx(&full[s], A_BYTES + 2 * B_BYTES);
        const int kc = (c_begin + i) * BK;
        if (MODE == MODE_AX)
          tma_load_2d(sA + s * (A_BYTES / 4), &mapA, &full[s], mt * 128, kc);
        else
          tma_load_2d(sA + s * (A_BYTES / 4), &mapA, &full[s], kc, mt * 128);
        tma_load_2d(sBh + s * B_BYTES, &mapBhi, &full[s], kc, 0);
        tma_load_2d(sBl + s * B_BYTES, &mapBlo, &full[s], kc, 0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_tf32(128, NP);
      for (int i = 0; i < nch; ++i) {
        const int s = i % STAGES;
        const uint32_t ph = (i / STAGES) & 1;
        const int t = i % TSTAGES;
        const uint32_t tph = (i / TSTAGES) & 1;
        const int g = i / SEG, b = g & 1;
        const bool seg_first = (i % SEG) == 0;
        const bool seg_last = ((i % SEG) == SEG - 1) || (i == nch - 1);
        if (seg_first) mbar_wait(&accempty[b], ((g >> 1) & 1) ^ 1);
        mbar_wait(&full[s], ph);
        mbar_wait(&tfull[t], tph);
        tc_fence_after();
        const uint32_t acc = t_acc0 + 128 * b;
        const uint32_t a_hi = t_a + t * 64, a_lo = a_hi + 32;
        const uint64_t bh = desc_kmajor_sw128(smem_u32(sBh + s * B_BYTES));
        const uint64_t bl = desc_kmajor_sw128(smem_u32(sBl + s * B_BYTES));
#pragma unroll
        for (int kk = 0; kk < BK / 8; ++kk) {
          const uint64_t koff = (uint64_t)(kk * 32) >> 4;  // 8 tf32 = 32 bytes along K
          mma_tf32_ts(acc, a_hi + kk * 8, bh + koff, idesc, (!seg_first || kk > 0) ? 1u : 0u);
          mma_tf32_ts(acc, a_hi + kk * 8, bl + koff, idesc, 1u);
          mma_tf32_ts(acc, a_lo + kk * 8, bh + koff, idesc, 1u);
        }
        tc_commit(&empty[s]);
        tc_commit(&tempty[t]);
        if (seg_last) tc_commit(&accfull[b]);
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // converters: shared A tile -> (hi, lo) -> TMEM ring
    const int wq = warp & 3;
    const int row = wq * 32 + lane;
    const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
    for (int i = 0; i < nch; ++i) {
      const int s = i % STAGES;
      const uint32_t ph = (i / STAGES) & 1;
      const int t = i % TSTAGES;
      const uint32_t tph = (i / TSTAGES) & 1;
      mbar_wait(&full[s], ph);
      mbar_wait(&tempty[t], tph ^ 1);
      const float* a = sA + s * (A_BYTES / 4);
      uint32_t hi[32], lo[32];
      if (MODE == MODE_AX) {
        // box {128 rows, 32 cols}, no swizzle: (row, k) at k*128 + row
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const float v = a[k * 128 + row];
          const uint32_t h = rna_tf32(v);
          hi[k] = h;
          lo[k] = __float_as_uint(v - __uint_as_float(h));
        }
      } else {
        // box {32 rows (K), 128 cols (M)}, 128B swizzle: (row=j, k) at
        // j*128 + ((k/4 ^ j%8) * 16) + (k%4)*4 bytes
        const float4* a4 = reinterpret_cast<const float4*>(a) + row * 8;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const float4 v4 = a4[c ^ (row & 7)];
          const float vv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const uint32_t h = rna_tf32(vv[e]);
            hi[c * 4 + e] = h;
            lo[c * 4 + e] = __float_as_uint(vv[e] - __uint_as_float(h));
          }
        }
      }
      tmem_st32(t_a + t * 64 + lane_off, hi);
      tmem_st32(t_a + t * 64 + 32 + lane_off, lo);
      tc_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&tfull[t]);
        mbar_arrive(&empty[s]);
      }
    }
  } else if (warp >= 8) {
    // flush warps: TMEM accumulator segments -> fp32 registers -> global
    const int wq = warp & 3;
    const int col0 = ((warp - 8) >> 2) * HALF;
    const int row = wq * 32 + lane;
    const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
    float sum[HALF];
#pragma unroll
    for (int j = 0; j < HALF; ++j) sum[j] = 0.f;
    for (int g = 0; g < nseg; ++g) {
      const int b = g & 1;
      mbar_wait(&accfull[b], (g >> 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int cb = 0; cb < HALF; cb += 32) {
        uint32_t v[32];
        tmem_ld32(t_acc0 + 128 * b + col0 + cb + lane_off, v);
        tc_wait_ld();
#pragma unroll
        for (int j = 0; j < 32; ++j) sum[cb + j] += __uint_as_float(v[j]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&accempty[b]);
    }
    const int gm = mt * 128 + row;
    if (gm < Mtot) {
      float* o = out + (int64_t)z * zstride;
#pragma unroll
      for (int j = 0; j < HALF; ++j) {
        const int c = col0 + j;
        if (c < Nvalid) {
          float x = sum[j];
          if (add) x += add[gm + (int64_t)c * ldadd];
          o[gm + (int64_t)c * ldo] = x;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tbase, 512);
  }
}

// hi = rna_tf32(x), lo = x - hi for a rows x cols column-major matrix (ld in/out)
__global__ void split_tf32_kernel(const float* __restrict__ X, int64_t rows, int64_t cols, int64_t ldx,
                                  float* __restrict__ Hi, float* __restrict__ Lo, int64_t ldo) {
  const int64_t total = rows * cols;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx % rows, j = idx / rows;
    const float x = X[i + j * ldx];
    const uint32_t h = rna_tf32(x);
    Hi[i + j * ldo] = __uint_as_float(h);
    Lo[i + j * ldo] = x - __uint_as_float(h);
  }
}

}  // namespace tc
}  // namespace frsvt
