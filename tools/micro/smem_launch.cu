// Launch cost of a 148 x 1024 grid vs its dynamic shared memory, alone and
// alternating with a small-smem kernel (carveout switches).  Probe only.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void big(int* p) {
  extern __shared__ int s[];
  s[threadIdx.x] = threadIdx.x;
  __syncthreads();
  if (threadIdx.x == 0 && s[5] == 77) p[0] = 1;
}
__global__ void small_k(int* p) {
  __shared__ int s[256];
  s[threadIdx.x & 255] = threadIdx.x;
  __syncthreads();
  if (threadIdx.x == 0 && s[5] == 77) p[1] = 1;
}
int main() {
  int* p;
  cudaMalloc(&p, 64);
  cudaFuncSetAttribute(big, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int sizes[] = {4096, 16 * 1024, 48 * 1024, 96 * 1024, 128 * 1024, 177 * 1024, 200 * 1024};
  for (int alt = 0; alt < 2; ++alt)
    for (int sz : sizes) {
      for (int i = 0; i < 10; ++i) big<<<148, 1024, sz>>>(p);
      cudaEventRecord(a);
      for (int i = 0; i < 200; ++i) {
        big<<<148, 1024, sz>>>(p);
        if (alt) small_k<<<148 * 4, 256>>>(p);
      }
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("alt=%d smem=%6d  %.2f us per iteration\n", alt, sz, ms * 1000 / 200);
    }
  float ms;
  cudaEventRecord(a);
  for (int i = 0; i < 200; ++i) small_k<<<148 * 4, 256>>>(p);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf("small alone %.2f us\n", ms * 1000 / 200);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
