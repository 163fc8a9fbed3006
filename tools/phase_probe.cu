// phase_probe.cu -- cost of solver-like phases on the B200 (measurement tool).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double rcp_fast(double x) {
  double r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0); r = fma(r, e, r); e = fma(-x, r, 1.0); return fma(r, e, r);
}
__global__ void phases(long long* out, double* sink, int n) {
  __shared__ double red[8][8];
  __shared__ double arr[2048];
  __shared__ int idx[2048];
  const int tid = threadIdx.x;
  for (int i = tid; i < 2048; i += blockDim.x) { arr[i] = 1.0 + i; idx[i] = (i * 37 + 11) & 2047; }
  if (tid < 64) red[tid / 8][tid % 8] = tid;
  __syncthreads();
  double acc = 0;
  long long t0, t1;
  t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  t1 = clock64(); if (tid == 0) out[0] = (t1 - t0) / n;
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    double a = 0; for (int w = 0; w < 8; ++w) a += red[i & 7][w];
    acc += rcp_fast(a + 1.0);
    __syncthreads();
  }
  t1 = clock64(); if (tid == 0) out[1] = (t1 - t0) / n;
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    double v = acc + i;
    for (int d = 16; d >= 1; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    if ((tid & 31) == 0) red[i & 7][tid >> 5] = v;
    __syncthreads();
    double a = 0; for (int w = 0; w < 8; ++w) a += red[i & 7][w];
    acc += a * 1e-30;
  }
  t1 = clock64(); if (tid == 0) out[2] = (t1 - t0) / n;
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    int j = (tid + i) & 2047;
    double a = 0;
    for (int k = 0; k < 8; ++k) { j = idx[j]; a += arr[j]; }
    acc += a * 1e-30;
    __syncthreads();
  }
  t1 = clock64(); if (tid == 0) out[3] = (t1 - t0) / n;
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    const int j = (tid * 8 + i) & 2047;
    double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
    for (int k = 0; k < 8; k += 4) { a0 += arr[(j + k) & 2047]; a1 += arr[(j + k + 1) & 2047]; a2 += arr[(j + k + 2) & 2047]; a3 += arr[(j + k + 3) & 2047]; }
    acc += (a0 + a1 + a2 + a3) * 1e-30;
    __syncthreads();
  }
  t1 = clock64(); if (tid == 0) out[4] = (t1 - t0) / n;
  sink[tid] = acc;
}
int main() {
  long long* d; double* s;
  cudaMalloc(&d, 64 * 8); cudaMalloc(&s, 1024 * 8);
  for (int th : {32, 256}) {
    phases<<<1, th>>>(d, s, 200); phases<<<1, th>>>(d, s, 200);
    cudaDeviceSynchronize();
    long long h[8]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("threads=%d: barrier %lld | slotsum+rcp+bar %lld | shfl-reduce+bar+sum %lld | 8 dep (LDS,LDS,DADD)+bar %lld | 8 indep LDS.64+bar %lld cycles\n",
           th, h[0], h[1], h[2], h[3], h[4]);
  }
  return 0;
}
