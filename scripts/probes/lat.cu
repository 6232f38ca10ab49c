// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/probes/lat scripts/probes/lat.cu
// Latency probes (one warp unless noted): dependent DFMA chain, DMUL, fp64
// division, MUFU rcp + Newton, mbarrier arrive -> wait ping-pong between two
// warps, __syncthreads with 1024 threads.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k_dfma(double* out, long long* cyc, int n) {
  double a = out[0], b = 1.0000001, c = 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = fma(a, b, c);
  long long t1 = clock64();
  out[1] = a; cyc[0] = (t1 - t0);
}
__global__ void k_div(double* out, long long* cyc, int n) {
  double a = out[0] + 1.5;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = 1.0 / a + 0.5;
  long long t1 = clock64();
  out[1] = a; cyc[0] = (t1 - t0);
}
__global__ void k_rcp(double* out, long long* cyc, int n) {
  double a = out[0] + 1.5;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    double r = (double)__frcp_rn((float)a);
    r = fma(r, fma(-a, r, 1.0), r);
    r = fma(r, fma(-a, r, 1.0), r);
    a = r + 0.5;
  }
  long long t1 = clock64();
  out[1] = a; cyc[0] = (t1 - t0);
}
__global__ void k_sync(long long* cyc, int n) {
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__device__ __forceinline__ void arrive(uint32_t a) {
  asm volatile("{\n.reg .b64 st;\nmbarrier.arrive.release.cta.shared::cta.b64 st, [%0];\n}" ::"r"(a) : "memory");
}
__device__ __forceinline__ void waitp(uint32_t a, uint32_t ph, int test) {
  uint32_t ok = 0;
  do {
    if (test)
      asm volatile("{\n.reg .pred p;\nmbarrier.test_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\nselp.b32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(a), "r"(ph) : "memory");
    else
      asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\nselp.b32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(a), "r"(ph) : "memory");
  } while (!ok);
}
// two warps ping-pong n times through two mbarriers
__global__ void k_pingpong(long long* cyc, int n, int test) {
  __shared__ uint64_t bar[2];
  uint32_t b0 = (uint32_t)__cvta_generic_to_shared(&bar[0]);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(b0));
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(b0 + 8));
  }
  __syncthreads();
  const int w = threadIdx.x >> 5, L = threadIdx.x & 31;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if (w == 0) {
      if (L == 0) arrive(b0);
      waitp(b0 + 8, i & 1, test);
    } else if (w == 1) {
      waitp(b0, i & 1, test);
      if (L == 0) arrive(b0 + 8);
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* d; long long* c; long long h;
  cudaMalloc(&d, 64); cudaMalloc(&c, 64); cudaMemset(d, 0, 64);
  const int n = 10000;
  k_dfma<<<1, 32>>>(d, c, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("dfma dependent: %.1f cycles\n", (double)h / n);
  k_div<<<1, 32>>>(d, c, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("1.0/x + add dependent: %.1f cycles\n", (double)h / n);
  k_rcp<<<1, 32>>>(d, c, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("frcp+2 newton + add: %.1f cycles\n", (double)h / n);
  k_sync<<<1, 1024>>>(c, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("syncthreads 1024: %.1f cycles\n", (double)h / n);
  k_sync<<<1, 256>>>(c, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("syncthreads 256: %.1f cycles\n", (double)h / n);
  k_pingpong<<<1, 64>>>(c, n, 0); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("mbarrier ping-pong round trip (try_wait): %.1f cycles\n", (double)h / n);
  k_pingpong<<<1, 64>>>(c, n, 1); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("mbarrier ping-pong round trip (test_wait): %.1f cycles\n", (double)h / n);
  k_pingpong<<<1, 1024>>>(c, n, 0); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("ping-pong with 30 idle warps: %.1f cycles\n", (double)h / n);
  return 0;
}
