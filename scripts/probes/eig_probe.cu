// Timing probe for eig_jacobi_kernel: mean kernel time over back-to-back
// launches on the Gram of a random l x 2l matrix with a decaying spectrum,
// a fixed number of sweeps (tol_stop = 0), and the residuals
// |G U - U diag(sigma^2)| / |G| and |U^T U - I|. Not part of libfrsvt.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include "eig_jacobi.cuh"
using namespace frsvt;
int main(int argc, char** argv) {
  const int l = argc > 1 ? atoi(argv[1]) : 120, sweeps = argc > 2 ? atoi(argv[2]) : 3;
  const int kind = argc > 3 ? atoi(argv[3]) : 0;  // 1: clustered spectrum, nearly diagonal (tol_stop 0, <= 40 sweeps)
  const int n = 2 * l;
  std::vector<double> B((size_t)l * n), G((size_t)l * l);
  srand(7);
  for (int i = 0; i < l; ++i)
    for (int j = 0; j < n; ++j) B[i + (size_t)j * l] = (rand() / (double)RAND_MAX - 0.5) * pow(10.0, -2.0 * i / l);
  for (int a = 0; a < l; ++a) for (int b = 0; b < l; ++b) {
    double s = 0; for (int j = 0; j < n; ++j) s += B[a + (size_t)j * l] * B[b + (size_t)j * l];
    G[a + (size_t)b * l] = s;
  }
  if (kind == 1) {  // Q = GS(I + K - K^T), K ~ 0.02 U(-1,1); s: 5/6 in [0.3, 0.4], rest ~7e-4
    std::vector<double> Q((size_t)l * l), sv(l);
    for (int a = 0; a < l; ++a) for (int b = 0; b < l; ++b) Q[a + (size_t)b * l] = (a == b);
    for (int a = 0; a < l; ++a) for (int b = 0; b < a; ++b) {
      const double k = 0.02 * (rand() / (double)RAND_MAX - 0.5);
      Q[a + (size_t)b * l] += k; Q[b + (size_t)a * l] -= k;
    }
    for (int j = 0; j < l; ++j) {
      for (int i = 0; i < j; ++i) {
        double d = 0; for (int r = 0; r < l; ++r) d += Q[r + (size_t)i * l] * Q[r + (size_t)j * l];
        for (int r = 0; r < l; ++r) Q[r + (size_t)j * l] -= d * Q[r + (size_t)i * l];
      }
      double nn = 0; for (int r = 0; r < l; ++r) nn += Q[r + (size_t)j * l] * Q[r + (size_t)j * l];
      for (int r = 0; r < l; ++r) Q[r + (size_t)j * l] /= sqrt(nn);
    }
    for (int i = 0; i < l; ++i) sv[i] = i < 5 * l / 6 ? 0.3 + 0.1 * rand() / (double)RAND_MAX : 6e-4 + 2e-4 * rand() / (double)RAND_MAX;
    for (int a = 0; a < l; ++a) for (int b = 0; b < l; ++b) {
      double s = 0; for (int i = 0; i < l; ++i) s += Q[a + (size_t)i * l] * sv[i] * sv[i] * Q[b + (size_t)i * l];
      G[a + (size_t)b * l] = s;
    }
  }
  double *dG, *dsig, *dU; int *dsw, *df;
  cudaMalloc(&dG, 8 * l * l); cudaMalloc(&dU, 8 * l * l); cudaMalloc(&dsig, 8 * l);
  cudaMalloc(&dsw, 4); cudaMalloc(&df, 4); cudaMemset(df, 0, 4);
  cudaMemcpy(dG, G.data(), 8 * l * l, cudaMemcpyHostToDevice);
  auto run = [&]() {
    eig_jacobi_launch(0, dG, l, nullptr, 0.0, 0, 1e-15, 0.0, kind == 1 ? 40 : sweeps, dsig, dU, dsw, df, nullptr);
  };
  for (int i = 0; i < 3; ++i) run();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int N = 50;
  cudaEventRecord(e0);
  for (int i = 0; i < N; ++i) run();
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  std::vector<double> U((size_t)l * l), sig(l);
  int sw; cudaMemcpy(&sw, dsw, 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(U.data(), dU, 8 * l * l, cudaMemcpyDeviceToHost);
  cudaMemcpy(sig.data(), dsig, 8 * l, cudaMemcpyDeviceToHost);
  double r1 = 0, r2 = 0, gn = 0;
  for (int a = 0; a < l; ++a) for (int b = 0; b < l; ++b) {
    double gu = 0, uu = 0;
    for (int i = 0; i < l; ++i) { gu += G[a + (size_t)i * l] * U[i + (size_t)b * l]; uu += U[i + (size_t)a * l] * U[i + (size_t)b * l]; }
    gu -= U[a + (size_t)b * l] * sig[b] * sig[b];
    r1 += gu * gu; r2 += (uu - (a == b)) * (uu - (a == b)); gn += G[a + (size_t)b * l] * G[a + (size_t)b * l];
  }
  printf("l=%d: %.1f us per launch, %d sweeps, %.2f us per sweep; |GU-U S^2|/|G|=%.2e |U^TU-I|=%.2e sig0=%.6e sig_last=%.6e %s\n",
         l, 1e3 * ms / N, sw, 1e3 * ms / N / sw, sqrt(r1 / gn), sqrt(r2), sig[0], sig[l - 1], cudaGetErrorString(cudaGetLastError()));
  return 0;
}
