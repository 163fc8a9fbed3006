// lat_gen_probe.cu -- dependent latency of shared-memory loads through LDS vs generic LD (tool).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __noinline__ int* pick(int* a, int* b, int sel) { return sel ? a : b; }
__global__ void k(long long* out, int* gbuf, int n, int sel) {
  __shared__ int idx[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) idx[i] = (i * 37 + 11) & 255;
  __syncthreads();
  int j = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) j = idx[j];
  long long t1 = clock64();
  out[0] = (t1 - t0) / n;
  int* g = pick(idx, gbuf, sel);  // generic pointer (to shared when sel != 0)
  t0 = clock64();
  for (int i = 0; i < n; ++i) j = g[j];
  t1 = clock64();
  out[1] = (t1 - t0) / n;
  out[2] = j;
}
int main() {
  long long* d; int* g;
  cudaMalloc(&d, 64); cudaMalloc(&g, 1024);
  for (int r = 0; r < 2; ++r) k<<<1, 32>>>(d, g, 1000, 1);
  cudaDeviceSynchronize();
  long long h[3]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  printf("LDS chase %lld cycles | generic LD (to shared) chase %lld cycles\n", h[0], h[1]);
  return 0;
}
