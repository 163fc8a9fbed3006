// imad_probe.cu -- issue cost of IMAD.HI against IMAD / FFMA / PRMT on the B200 (measurement tool):
// 256 operations in 8 independent chains per thread, 16 warps per SM (4 per scheduler).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int OP>
__global__ void probe(long long* out, uint32_t* sink, uint32_t seed) {
  uint32_t x[8];
  float f[8];
  for (int i = 0; i < 8; ++i) { x[i] = seed + threadIdx.x * 7 + i; f[i] = (float)x[i]; }
  __syncthreads();
  const long long t0 = clock64();
#pragma unroll 1
  for (int r = 0; r < 32; ++r) {
#pragma unroll
    for (int m = 0; m < 64; ++m) {
      const int i = m & 7;
      if (OP == 0) x[i] = x[i] * 0x9E3779B1u + seed;                 // IMAD
      if (OP == 1) x[i] = __umulhi(x[i], 0x9E3779B1u) + seed;        // IMAD.HI
      if (OP == 2) f[i] = fmaf(f[i], 1.0000001f, 0.5f);              // FFMA
      if (OP == 3) x[i] = __byte_perm(x[i], seed, 0x3210u + (m & 3)); // PRMT
      if (OP == 4) { x[i] = x[i] * 0x9E3779B1u + seed; x[(i + 1) & 7] = __byte_perm(x[(i + 1) & 7], seed, 0x2103u); }  // IMAD + PRMT
      if (OP == 5) { x[i] = __umulhi(x[i], 0x9E3779B1u) + seed; x[(i + 1) & 7] = __byte_perm(x[(i + 1) & 7], seed, 0x2103u); }  // IMAD.HI + PRMT
    }
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[OP] = (t1 - t0);
  uint32_t a = 0;
  for (int i = 0; i < 8; ++i) a += x[i] + (uint32_t)f[i];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = a;
}
int main() {
  long long* d; uint32_t* s;
  cudaMalloc(&d, 64 * 8); cudaMalloc(&s, 148 * 512 * 4);
  probe<0><<<148, 512>>>(d, s, 3); probe<1><<<148, 512>>>(d, s, 3); probe<2><<<148, 512>>>(d, s, 3);
  probe<3><<<148, 512>>>(d, s, 3); probe<4><<<148, 512>>>(d, s, 3); probe<5><<<148, 512>>>(d, s, 3);
  cudaDeviceSynchronize();
  long long h[8]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  const double n = 32.0 * 64 * 4;  // warp instructions per scheduler (4 warps each)
  printf("cycles per warp instruction per scheduler (16 warps/SM): IMAD %.2f | IMAD.HI %.2f | FFMA %.2f | PRMT %.2f | IMAD+PRMT pair %.2f | IMAD.HI+PRMT pair %.2f\n",
         h[0] / n, h[1] / n, h[2] / n, h[3] / n, h[4] / n, h[5] / n);
  return 0;
}
