// Probe library (not product code): phase timing of the one-CTA FRSVT kernel
// (clock64 stamps) and the FP64 FMA issue rate of one SM / the whole GPU.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC \
//        -I include -I paper_1509_00296_b200/csrc scripts/probes/bt_probe.cu -o scripts/probes/libbtprobe.so
#include "../../include/frsvt.h"
#include "common.cuh"
#include "batched.cuh"

using namespace frsvt;

extern "C" int bt_probe_run(int f64, int m, int n, int l, int q, const void* A, long lda, const void* Om,
                            void* X, double tau, int* r, double* sig, unsigned long long* stamps, int* sweeps,
                            int* flags, void* stream) {
  BtArgs a{};
  a.m = m; a.n = n; a.l = l; a.q = q; a.A = A; a.lda = lda; a.Om = Om; a.ldo = n; a.tau = tau;
  a.X = X; a.ldx = m; a.r_b = r; a.sig_b = sig; a.stamps = stamps; a.sweeps_b = sweeps; a.flags = flags;
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
