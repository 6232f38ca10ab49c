// Probe library (not product code): phase timing of the one-CTA FRSVT kernel
// (event-timed runs that stop after phase k) and the FP64 FMA issue rate of one SM / the whole GPU.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC \
//        -I include -I paper_1509_00296_b200/csrc scripts/probes/bt_probe.cu -o scripts/probes/libbtprobe.so
// Also: latencies of single dependent operations (lat_probe).
#include "../../include/frsvt.h"
#include "common.cuh"
#include "batched.cuh"

using namespace frsvt;

extern "C" int bt_probe_run(int f64, int m, int n, int l, int q, const void* A, long lda, const void* Om,
                            void* X, double tau, int* r, double* sig, int stop_after, int* sweeps,
                            int* flags, void* stream) {
  BtArgs a{};
  a.m = m; a.n = n; a.l = l; a.q = q; a.A = A; a.lda = lda; a.Om = Om; a.ldo = n; a.tau = tau;
  a.X = X; a.ldx = m; a.r_b = r; a.sig_b = sig; a.stop_after = stop_after; a.sweeps_b = sweeps; a.flags = flags;
  a.flags_store = 1;
  cudaError_t e = f64 ? bt_set_attrs<double>() : bt_set_attrs<float>();
  if (e != cudaSuccess) return (int)e;
  e = f64 ? bt_launch<double>(a, 1, (cudaStream_t)stream) : bt_launch<float>(a, 1, (cudaStream_t)stream);
  return (int)e;
}

// 8 independent DFMA chains per thread, `iters` steps
__global__ void dfma_rate_kernel(int iters, double* out, unsigned long long* cyc) {
  double x[8];
  for (int k = 0; k < 8; ++k) x[k] = 1.0 + 1e-9 * (threadIdx.x + k);
  const double a = 0.999999999, b = 1e-9;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  double s = 0;
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.0) out[0] = s;
  if (threadIdx.x == 0 && cyc) cyc[blockIdx.x] = t1 - t0;
}

extern "C" int dfma_rate(int blocks, int threads, int iters, double* out, unsigned long long* cyc, void* stream) {
  dfma_rate_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(iters, out, cyc);
  return (int)cudaGetLastError();
}

// latency probes: one CTA; thread 0 reports clock64 cycles per step
__device__ __forceinline__ double lat_rsqrt(double x) {
  double r = rsqrtf((float)x);
  r = r * fma(-0.5 * x * r, r, 1.5);
  r = r * fma(-0.5 * x * r, r, 1.5);
  return r;
}
__global__ void lat_kernel(int n, double* out, long long* res) {
  __shared__ double sh[1024];
  __shared__ int chase[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) { sh[i] = 1.0; chase[i] = (i * 7 + 1) & 1023; }
  __syncthreads();
  double x = 1.0 + threadIdx.x * 1e-9;
  float xf = 1.0f + threadIdx.x * 1e-7f;
  long long t0, t1;
  // (0) dependent DFMA
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, 0.999999, 1e-7);
  t1 = clock64(); if (threadIdx.x == 0) res[0] = (t1 - t0);
  // (1) dependent FFMA
  t0 = clock64();
  for (int i = 0; i < n; ++i) xf = fmaf(xf, 0.999999f, 1e-7f);
  t1 = clock64(); if (threadIdx.x == 0) res[1] = (t1 - t0);
  // (2) dependent 64-bit shuffles
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1) + 1e-9;
  t1 = clock64(); if (threadIdx.x == 0) res[2] = (t1 - t0);
  // (3) dependent fast rsqrt (fp32 seed + 2 Newton)
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = lat_rsqrt(x) + 1.0;
  t1 = clock64(); if (threadIdx.x == 0) res[3] = (t1 - t0);
  // (4) dependent IEEE double division
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = 1.0 / x + 1.0;
  t1 = clock64(); if (threadIdx.x == 0) res[4] = (t1 - t0);
  // (5) dependent double sqrt
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = sqrt(x) + 1.0;
  t1 = clock64(); if (threadIdx.x == 0) res[5] = (t1 - t0);
  // (6) __syncthreads
  t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  t1 = clock64(); if (threadIdx.x == 0) res[6] = (t1 - t0);
  // (7) dependent shared loads (pointer chase)
  int c = threadIdx.x & 1023;
  t0 = clock64();
  for (int i = 0; i < n; ++i) c = chase[c];
  t1 = clock64(); if (threadIdx.x == 0) res[7] = (t1 - t0);
  // (8) dependent DADD
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = x + 1e-9;
  t1 = clock64(); if (threadIdx.x == 0) res[8] = (t1 - t0);
  // (9) dependent double shared load + add
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = sh[((int)x) & 1023] + x * 1e-30;
  t1 = clock64(); if (threadIdx.x == 0) res[9] = (t1 - t0);
  // (10) rsqrt.approx.f64 (MUFU) alone
  t0 = clock64();
  for (int i = 0; i < n; ++i) { double r; asm("rsqrt.approx.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r + 1.0; }
  t1 = clock64(); if (threadIdx.x == 0) res[10] = (t1 - t0);
  // (11) rcp.approx.ftz.f64 alone
  t0 = clock64();
  for (int i = 0; i < n; ++i) { double r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r + 1.0; }
  t1 = clock64(); if (threadIdx.x == 0) res[11] = (t1 - t0);
  // (12) F2F f64 -> f32 -> f64 round trip
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = (double)(float)x + 1e-9;
  t1 = clock64(); if (threadIdx.x == 0) res[12] = (t1 - t0);
  // (13) 32-bit shuffle
  t0 = clock64();
  for (int i = 0; i < n; ++i) xf = __shfl_xor_sync(0xffffffffu, xf, 1) + 1e-7f;
  t1 = clock64(); if (threadIdx.x == 0) res[13] = (t1 - t0);
  if (x == 12345.0 || xf == 1.5f || c == -1) out[0] = x + xf + c;
}
extern "C" int lat_probe(int threads, int n, double* out, long long* res, void* stream) {
  lat_kernel<<<1, threads, 0, (cudaStream_t)stream>>>(n, out, res);
  return (int)cudaGetLastError();
}

