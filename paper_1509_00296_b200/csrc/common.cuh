// Shared device helpers for libfrsvt (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>

#ifndef FRSVT_LMAX
#define FRSVT_LMAX 128
#endif

namespace frsvt {

// ---- warp reductions -------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-wide sum of one double per thread; result valid in thread 0.
// `scratch` must hold blockDim.x/32 doubles.
__device__ __forceinline__ double block_sum(double v, double* scratch) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  double r = 0.0;
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    r = lane < nw ? scratch[lane] : 0.0;
    r = warp_sum(r);
  }
  __syncthreads();
  return r;
}
__device__ __forceinline__ double block_max(double v, double* scratch) {
  v = warp_max(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  double r = 0.0;
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    r = lane < nw ? scratch[lane] : 0.0;
    r = warp_max(r);
  }
  __syncthreads();
  return r;
}

template <typename T> __device__ __forceinline__ T soft(T x, T t) {
  // S_t(x) = sgn(x) max(|x| - t, 0)  (Definition 1)
  T a = fabs(x) - t;
  return a > T(0) ? copysign(a, x) : T(0);
}

// flag bits (mirror frsvt.h)
constexpr int FLAG_NONFINITE = 1;
constexpr int FLAG_NOCONV = 2;
constexpr int FLAG_NONMONOTONE_W = 4;

}  // namespace frsvt
