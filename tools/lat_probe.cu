// lat_probe.cu -- dependent-chain latencies on the B200 (measurement tool; not product code).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lat_probe tools/lat_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void probe(long long* out, double* dsink, int* isink, int n) {
  __shared__ double sd[256];
  __shared__ int si[256];
  __shared__ unsigned su[256];
  const int tid = threadIdx.x;
  sd[tid] = 1.0 + tid * 1e-9;
  si[tid] = (tid * 7 + 1) & 255;
  su[tid] = 0;
  __syncthreads();
  long long t0, t1;
  double x = sd[tid], y = 1.0000001;
  int j = tid;
  int k = 0;
  // DADD chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = x + y;
  t1 = clock64();
  if (tid == 0) out[0] = (t1 - t0);
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, y, 1e-12);
  t1 = clock64();
  if (tid == 0) out[1] = (t1 - t0);
  // FADD chain
  float f = (float)x;
  t0 = clock64();
  for (int i = 0; i < n; ++i) f = f + 1.0001f;
  t1 = clock64();
  if (tid == 0) out[2] = (t1 - t0);
  // LDS pointer chase
  t0 = clock64();
  for (int i = 0; i < n; ++i) j = si[j];
  t1 = clock64();
  if (tid == 0) out[3] = (t1 - t0);
  // LDS double chase (load value then add)
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = x + sd[(int)(x) & 255];
  t1 = clock64();
  if (tid == 0) out[4] = (t1 - t0);
  // SHFL double chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1);
  t1 = clock64();
  if (tid == 0) out[5] = (t1 - t0);
  // drcp chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __drcp_rn(x + 1.0);
  t1 = clock64();
  if (tid == 0) out[6] = (t1 - t0);
  // ddiv chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = 3.0 / (x + 1.0);
  t1 = clock64();
  if (tid == 0) out[7] = (t1 - t0);
  // bar.sync
  t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  t1 = clock64();
  if (tid == 0) out[8] = (t1 - t0);
  // match.any
  t0 = clock64();
  for (int i = 0; i < n; ++i) k += __match_any_sync(0xffffffffu, (k + tid) & 7);
  t1 = clock64();
  if (tid == 0) out[9] = (t1 - t0);
  // atoms.or same word (warp-wide)
  t0 = clock64();
  for (int i = 0; i < n; ++i) atomicOr(&su[i & 3], 1u << (tid & 31));
  t1 = clock64();
  if (tid == 0) out[10] = (t1 - t0);
  // IMAD chain
  int q = tid;
  t0 = clock64();
  for (int i = 0; i < n; ++i) q = q * 3 + 1;
  t1 = clock64();
  if (tid == 0) out[11] = (t1 - t0);
  // global load chain (L2 hit)
  dsink[tid] = x + f;
  isink[tid] = j + k + q;
}

int main() {
  long long* d;
  double* ds;
  int* is;
  cudaMalloc(&d, 64 * sizeof(long long));
  cudaMalloc(&ds, 1024 * sizeof(double));
  cudaMalloc(&is, 1024 * sizeof(int));
  const int n = 1000;
  const char* names[] = {"DADD", "DFMA", "FADD", "LDS chase", "LDS+DADD", "SHFL.64", "drcp_rn", "ddiv",
                         "bar.sync(8w)", "match.any", "atoms.or same", "IMAD"};
  for (int warps : {1, 8}) {
    probe<<<1, 32 * warps>>>(d, ds, is, n);
    probe<<<1, 32 * warps>>>(d, ds, is, n);
    cudaDeviceSynchronize();
    long long h[12];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("warps=%d\n", warps);
    for (int i = 0; i < 12; ++i) printf("  %-16s %7.1f cycles/op\n", names[i], (double)h[i] / n);
  }
  return 0;
}
