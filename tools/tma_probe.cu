// tma_probe.cu -- read bandwidth of per-warp cp.async.bulk pipelines vs copy size (measurement
// tool; not product code).  Each warp streams its share of a 2 GiB buffer through a KST-stage
// shared-memory ring with copies of S bytes and touches one word per copy (no other work).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_probe tools/tma_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const unsigned char* __restrict__ src, size_t n, int S, int KST, unsigned* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, NW = blockDim.x >> 5;
  unsigned char* ring = sm + (size_t)w * KST * S;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + (size_t)NW * KST * S) + w * KST;
  if (lane == 0) {
    for (int k = 0; k < KST; ++k) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(bar + k)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const size_t nchunks = n / S;
  const size_t gw = (size_t)blockIdx.x * NW + w, GW = (size_t)gridDim.x * NW;
  const size_t mine = nchunks > gw ? (nchunks - gw + GW - 1) / GW : 0;
  auto issue = [&](size_t i) {
    const int st = (int)(i % KST);
    const unsigned char* g = src + (gw + i * GW) * (size_t)S;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(bar + st)), "r"(S) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su(ring + (size_t)st * S)),
                 "l"(g), "r"(S), "r"(su(bar + st))
                 : "memory");
  };
  if (lane == 0)
    for (size_t i = 0; i < (size_t)KST && i < mine; ++i) issue(i);
  unsigned acc = 0;
  for (size_t i = 0; i < mine; ++i) {
    const int st = (int)(i % KST);
    const uint32_t ph = (uint32_t)((i / KST) & 1);
    asm volatile(
        "{\n .reg .pred P1;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n @!P1 bra W_%=;\n}\n" ::"r"(
            su(bar + st)),
        "r"(ph)
        : "memory");
    acc += *reinterpret_cast<const unsigned*>(ring + (size_t)st * S + 4 * lane);
    __syncwarp();
    if (lane == 0 && i + KST < mine) issue(i + KST);
  }
  if (acc == 0x12345678u) *sink = acc;
}

int main() {
  const size_t n = 2ull << 30;
  unsigned char* d;
  unsigned* sink;
  cudaMalloc(&d, n);
  cudaMalloc(&sink, 4);
  cudaMemset(d, 1, n);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int sizes[] = {1536, 3072, 6144, 12288, 24576};
  const int warps[] = {4, 8, 16, 32};
  printf("S_bytes warps/SM stages  GB/s  copies/us/SM\n");
  for (int S : sizes)
    for (int NW : warps)
      for (int KST : {2, 3, 4, 6}) {
        const size_t smem = (size_t)NW * KST * S + NW * KST * 8;
        if (smem > 200 * 1024) continue;
        probe<<<sms, NW * 32, smem>>>(d, n, S, KST, sink);
        cudaEventRecord(a);
        for (int r = 0; r < 3; ++r) probe<<<sms, NW * 32, smem>>>(d, n, S, KST, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double sec = ms / 3 / 1e3;
        const cudaError_t e = cudaGetLastError();
        printf("%6d %4d %3d %8.1f %8.2f %s\n", S, NW, KST, n / sec / 1e9, n / (double)S / sec / 1e6 / sms,
               e ? cudaGetErrorString(e) : "");
      }
  return 0;
}
