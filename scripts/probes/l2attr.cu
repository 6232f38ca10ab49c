// prints the L2 persisting-cache limits of device 0
#include <cstdio>
#include <cuda_runtime.h>
int main() {
  int a = 0, b = 0, c = 0;
  cudaDeviceGetAttribute(&a, cudaDevAttrMaxPersistingL2CacheSize, 0);
  cudaDeviceGetAttribute(&b, cudaDevAttrMaxAccessPolicyWindowSize, 0);
  cudaDeviceGetAttribute(&c, cudaDevAttrL2CacheSize, 0);
  printf("L2 %d B, max persisting %d B, max access policy window %d B\n", c, a, b);
  return 0;
}
