// walk_probe.cu -- the solver's R-phase row walk in isolation (measurement tool): the current
// loop (4 cells per step + remainders) against a fully predicated form with every load issued
// before the first use, on a 256-thread CTA with C3-like supports (nR = 27, nL = 75).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void probe(long long* out, double* sink, int nR, int nL, int rep) {
  __shared__ uint8_t kc[8192];
  __shared__ double q2[256], rho[256], res[256];
  const int tid = threadIdx.x, T = blockDim.x;
  for (int i = tid; i < nR * nL; i += T) { const int a = i / nL, c = i - a * nL; kc[i] = (uint8_t)(((a * 9 + 3) * c + 127) / 255); }
  for (int i = tid; i < 256; i += T) { q2[i] = 1.0 + i; rho[i] = 1.0 / (1 + i); }
  __syncthreads();
  const int lgR = nR <= T / 8 ? 3 : nR <= T / 4 ? 2 : nR <= T / 2 ? 1 : 0, TPR = 1 << lgR;
  const int a = tid >> lgR, p = tid & (TPR - 1);
  double sum = 0;
  long long t0 = clock64();
  for (int r = 0; r < rep; ++r) {  // ---- current form
    double A0 = 0.0, A1 = 0.0;
    if (a < nR) {
      const uint8_t* kr = kc + a * nL;
      int c = p;
      double A2 = 0.0, A3 = 0.0;
      for (; c + 3 * TPR < nL; c += 4 * TPR) {
        const int k0 = kr[c], k1 = kr[c + TPR], k2 = kr[c + 2 * TPR], k3 = kr[c + 3 * TPR];
        A0 = fma(q2[c], rho[k0], A0); A1 = fma(q2[c + TPR], rho[k1], A1);
        A2 = fma(q2[c + 2 * TPR], rho[k2], A2); A3 = fma(q2[c + 3 * TPR], rho[k3], A3);
      }
      if (c < nL) A0 = fma(q2[c], rho[kr[c]], A0);
      if (c + TPR < nL) A1 = fma(q2[c + TPR], rho[kr[c + TPR]], A1);
      if (c + 2 * TPR < nL) A2 = fma(q2[c + 2 * TPR], rho[kr[c + 2 * TPR]], A2);
      A0 += A2; A1 += A3;
    }
    double A = A0 + A1;
    for (int d = TPR >> 1; d >= 1; d >>= 1) A += __shfl_xor_sync(0xffffffffu, A, d);
    if (a < nR && p == 0) res[a] = A + sum;
    __syncthreads();
    sum += res[0] * 1e-300;
  }
  long long t1 = clock64();
  if (tid == 0) out[0] = (t1 - t0) / rep;
  t0 = clock64();
  for (int r = 0; r < rep; ++r) {  // ---- predicated batches of 8 cells, loads first
    double A0 = 0.0, A1 = 0.0, A2 = 0.0, A3 = 0.0;
    if (a < nR) {
      const uint8_t* kr = kc + a * nL;
      for (int c0 = p; c0 < nL; c0 += 8 * TPR) {
        int k[8]; double q[8], g[8];
#pragma unroll
        for (int m = 0; m < 8; ++m) { const int c = c0 + m * TPR; const bool in = c < nL; k[m] = in ? kr[c] : 0; q[m] = in ? q2[c] : 0.0; }
#pragma unroll
        for (int m = 0; m < 8; ++m) g[m] = rho[k[m]];
        A0 = fma(q[0], g[0], A0); A1 = fma(q[1], g[1], A1); A2 = fma(q[2], g[2], A2); A3 = fma(q[3], g[3], A3);
        A0 = fma(q[4], g[4], A0); A1 = fma(q[5], g[5], A1); A2 = fma(q[6], g[6], A2); A3 = fma(q[7], g[7], A3);
      }
    }
    double A = (A0 + A1) + (A2 + A3);
    for (int d = TPR >> 1; d >= 1; d >>= 1) A += __shfl_xor_sync(0xffffffffu, A, d);
    if (a < nR && p == 0) res[a] = A + sum;
    __syncthreads();
    sum += res[0] * 1e-300;
  }
  t1 = clock64();
  if (tid == 0) out[1] = (t1 - t0) / rep;
  t0 = clock64();
  for (int r = 0; r < rep; ++r) {  // ---- contiguous cells per lane: 4-byte key loads, 16-B q2 loads
    double A0 = 0.0, A1 = 0.0, A2 = 0.0, A3 = 0.0;
    if (a < nR) {
      const uint8_t* kr = kc + a * nL;
      const int per = (nL + TPR - 1) / TPR, cb = p * per, ce = min(nL, cb + per);
      for (int c0 = cb; c0 < ce; c0 += 4) {
        int k[4]; double q[4], g[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) { const bool in = c0 + m < ce; k[m] = in ? kr[c0 + m] : 0; q[m] = in ? q2[c0 + m] : 0.0; }
#pragma unroll
        for (int m = 0; m < 4; ++m) g[m] = rho[k[m]];
        A0 = fma(q[0], g[0], A0); A1 = fma(q[1], g[1], A1); A2 = fma(q[2], g[2], A2); A3 = fma(q[3], g[3], A3);
      }
    }
    double A = (A0 + A1) + (A2 + A3);
    for (int d = TPR >> 1; d >= 1; d >>= 1) A += __shfl_xor_sync(0xffffffffu, A, d);
    if (a < nR && p == 0) res[a] = A + sum;
    __syncthreads();
    sum += res[0] * 1e-300;
  }
  t1 = clock64();
  if (tid == 0) out[2] = (t1 - t0) / rep;
  sink[tid] = sum;
}
int main() {
  long long* d; double* s;
  cudaMalloc(&d, 64 * 8); cudaMalloc(&s, 1024 * 8);
  for (int nL : {22, 75, 200}) {
    probe<<<1, 256>>>(d, s, 27, nL, 50); probe<<<1, 256>>>(d, s, 27, nL, 50);
    cudaDeviceSynchronize();
    long long h[8]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("nR=27 nL=%d: current %lld | predicated 8-batches %lld | contiguous 4-batches %lld cycles (walk + shuffles + barrier)\n", nL, h[0], h[1], h[2]);
  }
  return 0;
}
