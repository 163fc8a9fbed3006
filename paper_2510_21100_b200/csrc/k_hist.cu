// k_hist.cu -- kernel (a): fused colour convert + gradient + privatised histograms.
//
// PAPER.md Alg. 1 lines "Compute the histogram of the low-light image H_C(S)" and
// "Compute the histogram of the gradient image H_C(grad S)", Eq. 3.
// The per-segment device body (value channel, gradient, lane-private counters, flush) is in
// hist_dev.cuh; this file holds the launch.
//
// Design (B200): persistent grid of 2 CTAs/SM x 512 threads.  Each CTA owns a contiguous
// range of global rows (all images concatenated), split at image boundaries into segments;
// one flush per (CTA, image) segment with global integer atomics -> exact, deterministic.
#include <algorithm>
#include <cstdlib>

#include "hist_dev.cuh"

namespace hr {
namespace {

// done (nullable): after each flushed segment of image b, add its row count to done[b] (fence,
// then atomic: a release), so that k_solve's CTA for image b can start as soon as all H rows of
// image b are flushed -- images finish at staggered times because image boundaries fall at
// spread-out points of the CTA ranges.
template <int SW, int VEC, int NT>
__global__ void __launch_bounds__(NT, 1024 / NT)
k_hist(const uint8_t* __restrict__ rgb, int64_t B, int H, int W, uint32_t* __restrict__ hist_s,
       uint32_t* __restrict__ hist_graw, uint32_t* __restrict__ done, int nowait) {
  extern __shared__ __align__(16) uint32_t sm[];
  TRACE_T0();
  if (!nowait) pdl_wait();
  pdl_trigger();
  const int64_t R = B * (int64_t)H;
  const int64_t r_begin = R * blockIdx.x / gridDim.x;
  const int64_t r_end = R * (blockIdx.x + 1) / gridDim.x;
  const size_t imgBytes = (size_t)H * (size_t)W * 3;
  for (int64_t r = r_begin; r < r_end;) {
    const int64_t b = r / H;
    const int y0 = (int)(r - b * H);
    const int y1 = (int)min((int64_t)H, (int64_t)y0 + (r_end - r));
    r += y1 - y0;
    hist_zero<NT>(sm);
    __syncthreads();
    hist_segment<SW, VEC, NT>(rgb + (size_t)b * imgBytes, H, W, y0, y1, sm, hist_s + b * kLevels,
                              hist_graw + b * kGradSlots);
    if (done) {
      __threadfence();
      if (threadIdx.x == 0) atomicAdd(done + b, (uint32_t)(y1 - y0));
    }
  }
  TRACE_END(1u, (uint32_t)((uintptr_t)hist_s >> 8), 0ull);  // aux: which launch (group)
}

template <int SW, int VEC>
cudaError_t launch_v(const uint8_t* rgb, int64_t B, int32_t H, int32_t W, uint32_t* hs, uint32_t* hg, int grid,
                     uint32_t* done, cudaStream_t st, bool nowait, int nt) {
  if (nt == 1024)
    return launch_pdl(k_hist<SW, VEC, 1024>, dim3(grid), dim3(1024), kHistDevSmem, st, rgb, B, H, W, hs, hg, done,
                      (int)nowait);
  return launch_pdl(k_hist<SW, VEC, kHistThreads>, dim3(grid), dim3(kHistThreads), kHistDevSmem, st, rgb, B, H, W,
                    hs, hg, done, (int)nowait);
}

__global__ void __launch_bounds__(256) k_zero(uint4* __restrict__ p, size_t n16) {
  pdl_wait();
  pdl_trigger();
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
    p[i] = make_uint4(0u, 0u, 0u, 0u);
}

}  // namespace

cudaError_t trace_bind_hist(void* buf, uint32_t* n, uint32_t cap) { return trace_bind_tu(buf, n, cap); }

cudaError_t launch_zero(void* p, size_t n, cudaStream_t st) {
  const size_t n16 = n / 16;
  if (n16 == 0) return cudaSuccess;
  const size_t grid = std::min<size_t>((n16 + 255) / 256, 1024);
  return launch_pdl(k_zero, dim3((unsigned)grid), dim3(256), 0, st, reinterpret_cast<uint4*>(p), n16);
}

int hist_grid_clamped(int64_t B, int32_t H, int grid) {
  const int64_t rows = B * (int64_t)H;
  if (grid > rows) grid = (int)rows;
  return grid < 1 ? 1 : grid;
}

cudaError_t init_attrs_hist() {
  cudaError_t e = cudaSuccess;
  for (auto k : {k_hist<16, 16, kHistThreads>, k_hist<8, 8, kHistThreads>, k_hist<16, 1, kHistThreads>,
                 k_hist<16, 16, 1024>, k_hist<8, 8, 1024>, k_hist<16, 1, 1024>})
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kHistDevSmem);
  return e;
}

cudaError_t launch_hist(const uint8_t* rgb, int64_t B, int32_t H, int32_t W, uint32_t* hist_s,
                        uint32_t* hist_graw, int grid, cudaStream_t st, uint32_t* done, bool nowait, int nt) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(rgb);
  grid = hist_grid_clamped(B, H, grid);
  if (a % 16 == 0 && W % 16 == 0) return launch_v<16, 16>(rgb, B, H, W, hist_s, hist_graw, grid, done, st, nowait, nt);
  // 8-B aligned rows (W % 16 == 8, e.g. C5's 600-px rows: a 1,800-B stride alternates between 0
  // and 8 mod 16): 8-px strips of three 8-B loads (C5 58 vs 61 us with the round-1 16-px strips
  // of mixed 16/8-B loads plus half-strip walkers, which needed 20 B of spills)
  if (a % 8 == 0 && W % 8 == 0) return launch_v<8, 8>(rgb, B, H, W, hist_s, hist_graw, grid, done, st, nowait, nt);
  return launch_v<16, 1>(rgb, B, H, W, hist_s, hist_graw, grid, done, st, nowait, nt);
}

}  // namespace hr
