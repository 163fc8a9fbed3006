// lat64_probe.cu -- dependent-latency of fp64 / fp32 / int ops on this GPU (measurement tool).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(long long* out, double* sd, float* sf, int n) {
  double a = sd[0], b = sd[1];
  float x = sf[0], y = sf[1];
  unsigned u = (unsigned)n;
  long long t0, t1;
  t0 = clock64();
  for (int i = 0; i < n; ++i) a = fma(a, b, 0.5);
  t1 = clock64(); out[0] = (t1 - t0) / n;
  t0 = clock64();
  for (int i = 0; i < n; ++i) a = a + b;
  t1 = clock64(); out[1] = (t1 - t0) / n;
  t0 = clock64();
  for (int i = 0; i < n; ++i) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a)); a = r + 1.0; }
  t1 = clock64(); out[2] = (t1 - t0) / n;
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = fmaf(x, y, 0.5f);
  t1 = clock64(); out[3] = (t1 - t0) / n;
  t0 = clock64();
  for (int i = 0; i < n; ++i) u = u * 3u + 1u;
  t1 = clock64(); out[4] = (t1 - t0) / n;
  t0 = clock64();
  for (int i = 0; i < n; ++i) a = __shfl_xor_sync(0xffffffffu, a, 1);
  t1 = clock64(); out[5] = (t1 - t0) / n;
  sd[2] = a; sf[2] = x; sd[3] = u;
}
__global__ void lat_smem(long long* out, int n) {
  __shared__ double arr[256];
  __shared__ int idx[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) { arr[i] = i; idx[i] = (i * 37 + 11) & 255; }
  __syncthreads();
  int j = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) j = idx[j];
  long long t1 = clock64(); if (threadIdx.x == 0) out[6] = (t1 - t0) / n;
  double a = 0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) { a = arr[(int)a & 255] + 1.0; }
  t1 = clock64(); if (threadIdx.x == 0) out[7] = (t1 - t0) / n;
  if (a == -1) out[8] = j;
}
int main() {
  long long* d; double* sd; float* sf;
  cudaMalloc(&d, 64 * 8); cudaMalloc(&sd, 64); cudaMalloc(&sf, 64);
  double h0[2] = {1.0000001, 0.9999999}; float f0[2] = {1.0f, 0.999f};
  cudaMemcpy(sd, h0, 16, cudaMemcpyHostToDevice); cudaMemcpy(sf, f0, 8, cudaMemcpyHostToDevice);
  for (int r = 0; r < 2; ++r) { lat<<<1, 32>>>(d, sd, sf, 1000); lat_smem<<<1, 32>>>(d, 1000); }
  cudaDeviceSynchronize();
  long long h[9]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  printf("dependent latency (cycles): DFMA %lld | DADD %lld | MUFU.RCP64H+DADD %lld | FFMA %lld | IMAD %lld | SHFL.f64 %lld | LDS.32 chase %lld | LDS.64+I2F+DADD chain %lld\n",
         h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7]);
  return 0;
}
