// lut_probe.cu -- cycles of the CDF + LUT tail (cdf_lut) in isolation (measurement tool).
#include <cstdio>
#include "../paper_2510_21100_b200/csrc/solve_dev.cuh"
using namespace hr;
__global__ void probe(long long* out, uint8_t* lut, int rep, double* gscratch) {
  __shared__ uint32_t hSi[256];
  __shared__ __align__(16) double Tt_[256], Pt_[256], Ct_[256], Cs_[256];
  __shared__ int wscr[8];
  // gscratch == nullptr at run time, but the compiler cannot know: the arrays are reached through
  // generic pointers, as in k_solve (state struct carved from dynamic shared memory)
  double* Tt = gscratch ? gscratch : Tt_;
  double* Pt = gscratch ? gscratch + 256 : Pt_;
  double* Ct = gscratch ? gscratch + 512 : Ct_;
  double* Cs = gscratch ? gscratch + 768 : Cs_;
  const int tid = threadIdx.x;
  hSi[tid] = tid < 80 ? 1000 + 37 * tid : 0;
  Tt[tid] = tid < 200 ? 1.0 + 0.01 * tid * tid : 0.0;
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < rep; ++r) {
    cdf_lut<256>(hSi, Tt, Pt, Ct, Cs, wscr, lut, nullptr);
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) out[0] = (t1 - t0) / rep;
}
int main() {
  long long* d; uint8_t* l;
  cudaMalloc(&d, 64 * 8); cudaMalloc(&l, 256);
  probe<<<1, 256>>>(d, l, 20, nullptr); probe<<<1, 256>>>(d, l, 20, nullptr);
  cudaDeviceSynchronize();
  long long h[8]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  uint8_t hl[256]; cudaMemcpy(hl, l, 256, cudaMemcpyDeviceToHost);
  unsigned sum = 0; for (int i = 0; i < 256; ++i) sum = sum * 31 + hl[i];
  printf("cdf_lut: %lld cycles, lut checksum %u (%s)\n", h[0], sum, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
