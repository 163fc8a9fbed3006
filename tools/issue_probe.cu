// issue_probe.cu -- what one solver-like phase costs per warp on the B200 (measurement tool):
// a chunk phase (2 x LDS.128 descriptors -> 16 gathered LDS.64 -> 8 DMUL -> tree -> STS) timed on
// warp 0 for 1..16 resident warps, with shared-window generic loads or LDS, and a gather walk
// (key LDS.U8 -> LDS.64 gather -> DFMA) like the R phase.
#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>
template <bool GENERIC>
__global__ void probe(long long* out, double* sink, int n, const double* gh) {
  __shared__ __align__(16) uint32_t desc[8 * 512];
  __shared__ double hr[256], hl[258], pv[512], rho[256];
  __shared__ uint8_t kc[8192];
  const int tid = threadIdx.x, T = blockDim.x;
  for (int i = tid; i < 8 * 512; i += T) desc[i] = (uint32_t)(8 * ((i / 64) & 31)) | ((uint32_t)(8 * (i & 63)) << 16);
  for (int i = tid; i < 256; i += T) { hr[i] = 1.0 + i; hl[i] = 2.0 + i; rho[i] = 1.0 / (1 + i); }
  for (int i = tid; i < 8192; i += T) kc[i] = (uint8_t)((i * 7 / 64) & 255);
  __syncthreads();
  const unsigned char* hrb = GENERIC ? (const unsigned char*)(gh ? (const double*)hr : gh) : (const unsigned char*)hr;
  const unsigned char* hlb = (const unsigned char*)hl;
  double acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < n; ++it) {
    const uint4* cd = GENERIC ? reinterpret_cast<const uint4*>(gh ? (const void*)gh : (const void*)desc) : reinterpret_cast<const uint4*>(desc);
    const int p = tid;
    const uint4 q0 = cd[2 * p], q1 = cd[2 * p + 1];
    const uint32_t d[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
    double x[8];
#pragma unroll
    for (int m = 0; m < 8; ++m)
      x[m] = *reinterpret_cast<const double*>(hrb + (d[m] & 0xFFFFu)) * *reinterpret_cast<const double*>(hlb + (d[m] >> 16));
#pragma unroll
    for (int w = 1; w < 8; w <<= 1)
#pragma unroll
      for (int m = 0; m + w < 8; m += 2 * w) x[m] += x[m + w];
    (GENERIC ? (gh ? const_cast<double*>(gh) + 4096 : pv) : pv)[p] = x[0] + acc;
    __syncthreads();
    acc += pv[(p + 1) % T] * 1e-300;
  }
  long long t1 = clock64();
  if (tid == 0) out[0] = (t1 - t0) / n;
  // gather walk: 8 cells per lane, 4 per step
  t0 = clock64();
  for (int it = 0; it < n; ++it) {
    const uint8_t* kr = kc + (tid >> 3) * 64;
    double A0 = 0, A1 = 0, A2 = 0, A3 = 0;
    int c = tid & 7;
    for (; c + 24 < 64; c += 32) {
      const int k0 = kr[c], k1 = kr[c + 8], k2 = kr[c + 16], k3 = kr[c + 24];
      A0 = fma(hl[c], rho[k0], A0); A1 = fma(hl[c + 8], rho[k1], A1);
      A2 = fma(hl[c + 16], rho[k2], A2); A3 = fma(hl[c + 24], rho[k3], A3);
    }
    double A = (A0 + A1) + (A2 + A3);
    for (int d = 4; d >= 1; d >>= 1) A += __shfl_xor_sync(0xffffffffu, A, d);
    if ((tid & 7) == 0) hr[tid >> 3] = A + acc * 1e-300 + 1.0;
    __syncthreads();
  }
  t1 = clock64();
  if (tid == 0) out[1] = (t1 - t0) / n;
  // pure dependent ALU chain of 64 IMADs (issue latency reference)
  t0 = clock64();
  int z = tid;
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int m = 0; m < 64; ++m) z = z * 3 + m;
  }
  t1 = clock64();
  if (tid == 0) out[2] = (t1 - t0) / n;
  // 64 independent-ish DFMAs in 8 chains
  t0 = clock64();
  double f[8] = {1, 2, 3, 4, 5, 6, 7, 8};
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int m = 0; m < 64; ++m) f[m & 7] = fma(f[m & 7], 1.0000001, 0.5);
  }
  t1 = clock64();
  if (tid == 0) out[3] = (t1 - t0) / n;
  sink[tid] = acc + z + f[0] + f[1] + f[2] + f[3] + f[4] + f[5] + f[6] + f[7];
}
int main() {
  long long* d; double* s;
  cudaMalloc(&d, 64 * 8); cudaMalloc(&s, 1024 * 8);
  for (int grid : {1, 2})
    for (int th : {32, 96, 256}) {
      if (grid == 1) { probe<false><<<1, th>>>(d, s, 200, nullptr); probe<false><<<1, th>>>(d, s, 200, nullptr); }
      else { probe<true><<<1, th>>>(d, s, 200, nullptr); probe<true><<<1, th>>>(d, s, 200, nullptr); }
      cudaDeviceSynchronize();
      long long h[8]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
      printf("grid=%3d threads=%3d: chunk phase+bar %lld | gather walk+shfl+bar %lld | 64 dep IMAD %lld | 64 DFMA in 8 chains %lld cycles\n",
             grid, th, h[0], h[1], h[2], h[3]);
    }
  return 0;
}
