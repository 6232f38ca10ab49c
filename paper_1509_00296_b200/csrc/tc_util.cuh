// Shared tcgen05 / TMA / cluster helpers of the tensor-core kernels (sm_100a):
// UMMA shared-memory and instruction descriptors, TMEM stores, cluster
// barriers and multicast TMA, the stream-K range partition, and the split of
// a small operand B into the tensor-core formats of the streaming passes
// (tc_pass3.cuh): b_h = rna_tf32(b) and bf16 [b_l | b_h].
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include "tc_pass.cuh"

namespace frsvt {
namespace tc {

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
__host__ __device__ __forceinline__ int64_t sk_range_begin(int64_t total, int G, int c) {
  return (total * c) / G;
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
