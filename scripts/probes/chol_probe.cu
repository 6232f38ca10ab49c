// Timing probe for chol_inv_kernel: mean
// kernel time over back-to-back launches on a random SPD Gram, plus a
// check of T^T G T = I. Not part of libfrsvt.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include "chol_inv.cuh"
using namespace frsvt;
int main(int argc, char** argv) {
  const int l = argc > 1 ? atoi(argv[1]) : 120, r = argc > 2 ? atoi(argv[2]) : 0;
  const int m = 4 * l;
  std::vector<double> Y((size_t)m * l), G((size_t)l * l);
  srand(1);
  for (auto& v : Y) v = (rand() / (double)RAND_MAX - 0.5);
  for (int j = 0; j < l; ++j) for (int i = 0; i < m; ++i) Y[i + (size_t)j * m] *= pow(10.0, -3.0 * j / l);
  for (int a = 0; a < l; ++a) for (int b = 0; b < l; ++b) {
    double s = 0; for (int i = 0; i < m; ++i) s += Y[i + (size_t)a * m] * Y[i + (size_t)b * m];
    G[a + (size_t)b * l] = s;
  }
  double *dG; float* dT; int *ds, *df, *dr;
  cudaMalloc(&dG, sizeof(double) * l * l); cudaMalloc(&dT, sizeof(float) * l * l);
  cudaMalloc(&ds, 4); cudaMalloc(&df, 4); cudaMalloc(&dr, 4);
  cudaMemcpy(dG, G.data(), sizeof(double) * l * l, cudaMemcpyHostToDevice);
  cudaMemcpy(dr, &r, 4, cudaMemcpyHostToDevice);
  cudaMemset(df, 0, 4);
  auto kern = l <= 64 ? chol_inv_kernel<float, 8> : chol_inv_kernel<float, 16>;
  const int thr = l <= 64 ? 256 : 512;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)chol_inv_smem_bytes());
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int it = 0; it < 5; ++it) kern<<<1, thr, chol_inv_smem_bytes()>>>(dG, l, dr, 1e-12, dT, l, ds, df, nullptr, nullptr, nullptr);
  const int N = 200;
  cudaEventRecord(e0);
  for (int it = 0; it < N; ++it) kern<<<1, thr, chol_inv_smem_bytes()>>>(dG, l, dr, 1e-12, dT, l, ds, df, nullptr, nullptr, nullptr);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  std::vector<float> T((size_t)l * l);
  cudaMemcpy(T.data(), dT, sizeof(float) * l * l, cudaMemcpyDeviceToHost);
  int s; cudaMemcpy(&s, ds, 4, cudaMemcpyDeviceToHost);
  // |T^T G T - I|_F
  double err = 0;
  for (int a = 0; a < l; ++a) for (int b = 0; b < l; ++b) {
    double v = 0;
    for (int i = 0; i < l; ++i) { double gi = 0; for (int j = 0; j < l; ++j) gi += G[i + (size_t)j * l] * T[j + (size_t)b * l]; v += T[i + (size_t)a * l] * gi; }
    if (r == 0) { double d = v - (a == b); err += d * d; }
  }
  printf("l=%d r=%d: %.2f us per launch (back-to-back), s=%d, |T^T G T - I|=%.2e, err=%s\n", l, r,
         1e3 * ms / N, s, sqrt(err), cudaGetErrorString(cudaGetLastError()));
  return 0;
}
