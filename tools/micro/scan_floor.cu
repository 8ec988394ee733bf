// Microbenchmark: the integer floor of the Bloom positive scan on B200.
// K1 hash only (h_a + probe-0 position), K2 + an L2 word load, K3 + a smem load,
// K4 the expected full per-key work without control flow (3.5 mix64, 2 mods, 2 loads).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ULL; z ^= z >> 27; z *= 0x94D049BB133111EBULL; return z ^ (z >> 31);
}
__device__ __forceinline__ uint32_t fmod_small(uint64_t x, uint64_t minv, uint32_t m) {
  const uint32_t q = static_cast<uint32_t>(__umul64hi(x, minv));
  const uint32_t r = static_cast<uint32_t>(x) - q * m;
  return r >= m ? r - m : r;
}

template <int kMode>
__global__ void __launch_bounds__(256) floor_kernel(const uint32_t* __restrict__ words, uint32_t d, uint32_t m,
                                                   uint64_t minv, uint64_t sa, uint64_t sb, uint32_t* out) {
  extern __shared__ uint32_t sw[];
  if (kMode == 3) {
    for (uint32_t i = threadIdx.x; i < (m + 31) / 32 && i < 12 * 1024; i += blockDim.x) sw[i] = words[i];
    __syncthreads();
  }
  uint32_t acc = 0;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t x0 = blockIdx.x * blockDim.x + threadIdx.x; x0 < d; x0 += 4 * stride) {
    uint32_t p[4], q[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint64_t x = x0 + u * stride;
      const uint64_t a = mix64(x ^ sa);
      p[u] = fmod_small(mix64(a), minv, m);
      if (kMode == 4) {
        const uint64_t b = mix64(x ^ sb);
        q[u] = fmod_small(mix64(a + b), minv, m);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (kMode == 1) acc += p[u];
      if (kMode == 2 || kMode == 4) acc += words[p[u] >> 5] >> (p[u] & 31);
      if (kMode == 4) acc += words[q[u] >> 5] >> (q[u] & 31);
      if (kMode == 3) acc += sw[(p[u] >> 5) % (12 * 1024)] >> (p[u] & 31);
    }
  }
  if (acc == 0x12345678u) out[0] = acc;
}

int main() {
  const uint32_t d = 25557032, m = 3674481;
  const uint64_t minv = ~0ULL / m;
  uint32_t *words, *out;
  cudaMalloc(&words, (m / 32 + 1) * 4);
  cudaMemset(words, 0x5a, (m / 32 + 1) * 4);
  cudaMalloc(&out, 4);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(floor_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const char* names[] = {"", "hash only (2 mix64 + mod)", "+ L2 word load", "+ smem word load",
                         "4 mix64 + 2 mod + 2 L2 loads"};
  for (int mode = 1; mode <= 4; ++mode) {
    for (int bpsm : {4, 8}) {
      const int grid = sms * bpsm;
      float best = 1e9f;
      for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(a);
        switch (mode) {
          case 1: floor_kernel<1><<<grid, 256>>>(words, d, m, minv, 1, 2, out); break;
          case 2: floor_kernel<2><<<grid, 256>>>(words, d, m, minv, 1, 2, out); break;
          case 3: floor_kernel<3><<<grid, 256, 48 * 1024>>>(words, d, m, minv, 1, 2, out); break;
          case 4: floor_kernel<4><<<grid, 256>>>(words, d, m, minv, 1, 2, out); break;
        }
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
      }
      printf("mode %d (%s), %d blocks/SM: %.4f ms  (%.1f G keys/s)\n", mode, names[mode], bpsm, best, d / best / 1e6);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
