// tail_probe.cu -- cycles of solver sub-steps in isolation (measurement tool): the Eq. 20 row
// walk (row_runs) on one warp, with generic and shared-window pointers.
#include <cstdio>
#include "../paper_2510_21100_b200/csrc/solve_dev.cuh"
using namespace hr;
__global__ void probe(long long* out, double* sink, int nR, int nL, int rep) {
  __shared__ uint8_t kc[8192];
  __shared__ double hL[256], D[4096];
  const int tid = threadIdx.x;
  for (int i = tid; i < nR * nL; i += blockDim.x) { const int a = i / nL, c = i - a * nL; kc[i] = (uint8_t)(((a * 9 + 3) * c + 127) / 255); }
  for (int i = tid; i < 256; i += blockDim.x) hL[i] = 1.0 + i;
  for (int i = tid; i < 4096; i += blockDim.x) D[i] = 0.0;
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < rep; ++r) {
    if (tid < nR) row_runs(kc + tid * nL, nL, hL, 1.5 + r, D, tid * 64);
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) out[0] = (t1 - t0) / rep;
  // dependent fp64 chain: 64 DADDs
  double a = tid;
  t0 = clock64();
  for (int r = 0; r < rep; ++r) {
#pragma unroll
    for (int m = 0; m < 64; ++m) a = a + 1.25;
  }
  t1 = clock64();
  if (tid == 0) out[1] = (t1 - t0) / rep;
  // select + add chain like the walk
  int k = tid;
  t0 = clock64();
  for (int r = 0; r < rep; ++r) {
#pragma unroll
    for (int m = 0; m < 64; ++m) { a = ((k ^ m) & 1 ? 0.0 : a) + 1.25; k = k * 3 + m; }
  }
  t1 = clock64();
  if (tid == 0) out[2] = (t1 - t0) / rep;
  sink[tid] = a + k + D[tid];
}
int main() {
  long long* d; double* s;
  cudaMalloc(&d, 64 * 8); cudaMalloc(&s, 1024 * 8);
  for (int th : {32, 256}) {
    probe<<<1, th>>>(d, s, 27, 75, 50); probe<<<1, th>>>(d, s, 27, 75, 50);
    cudaDeviceSynchronize();
    long long h[8]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("threads=%d: row walk nL=75 %lld | 64 dependent DADD %lld | 64 x (select + DADD) %lld cycles (%s)\n", th, h[0], h[1], h[2], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
