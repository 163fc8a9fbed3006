// k_hist.cu -- kernel (a): fused colour convert + gradient + privatised histograms.
//
// PAPER.md Alg. 1 lines "Compute the histogram of the low-light image H_C(S)" and
// "Compute the histogram of the gradient image H_C(grad S)", Eq. 3.
// The per-segment device body (value channel, gradient, lane-private counters, flush) is in
// hist_dev.cuh; this kernel is the standalone launch used by hr_histogram and the serial /
// chunk-pipelined hr_enhance paths.
//
// Design (B200): persistent grid of 2 CTAs/SM x 512 threads.  Each CTA owns a contiguous
// range of global rows (all images concatenated), split at image boundaries into segments;
// one flush per (CTA, image) segment with global integer atomics -> exact, deterministic.
#include <algorithm>
#include <cstdlib>

#include "hist_dev.cuh"

namespace hr {
namespace {

// done (nullable): after each flushed segment of image b, count it in done[b] (fence, then
// atomic: a release), so that k_solve's CTA for image b can start as soon as every CTA range
// overlapping image b has flushed it (hist_segments_of) -- images finish at staggered times
// because image boundaries fall at spread-out points of the CTA ranges.
template <int SW, int VEC, int NT>
__global__ void __launch_bounds__(NT, 1024 / NT)
k_hist(const uint8_t* __restrict__ rgb, int64_t B, int H, int W, uint32_t* __restrict__ hist_s,
       uint32_t* __restrict__ hist_graw, uint32_t* __restrict__ done) {
  extern __shared__ __align__(16) uint32_t sm[];
  pdl_wait();
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
      if (threadIdx.x == 0) atomicAdd(done + b, 1u);
    }
  }
}

template <int SW, int VEC, int NT>
cudaError_t launch_v(const uint8_t* rgb, int64_t B, int32_t H, int32_t W, uint32_t* hs, uint32_t* hg, int grid,
                     uint32_t* done, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e =
        cudaFuncSetAttribute(k_hist<SW, VEC, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, kHistDevSmem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  return launch_pdl(k_hist<SW, VEC, NT>, dim3(grid), dim3(NT), kHistDevSmem, st, rgb, B, H, W, hs, hg, done);
}

template <int SW, int VEC>
cudaError_t launch_nt(const uint8_t* rgb, int64_t B, int32_t H, int32_t W, uint32_t* hs, uint32_t* hg, int grid,
                      int nt, uint32_t* done, cudaStream_t st) {
  return nt == 256 ? launch_v<SW, VEC, 256>(rgb, B, H, W, hs, hg, grid, done, st)
                   : launch_v<SW, VEC, kHistThreads>(rgb, B, H, W, hs, hg, grid, done, st);
}

bool hist_w8_strip16() {  // measurement switch: HR_HIST_W8=8 keeps the 8-px strips
  static const int v = [] {
    const char* e = getenv("HR_HIST_W8");
    return e ? atoi(e) : 16;
  }();
  return v != 8;
}

__global__ void __launch_bounds__(256) k_zero(uint4* __restrict__ p, size_t n16) {
  pdl_wait();
  pdl_trigger();
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
    p[i] = make_uint4(0u, 0u, 0u, 0u);
}

}  // namespace

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

cudaError_t launch_hist(const uint8_t* rgb, int64_t B, int32_t H, int32_t W, uint32_t* hist_s,
                        uint32_t* hist_graw, int grid, cudaStream_t st, int nt, uint32_t* done) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(rgb);
  grid = hist_grid_clamped(B, H, grid);
  if (a % 16 == 0 && W % 16 == 0) return launch_nt<16, 16>(rgb, B, H, W, hist_s, hist_graw, grid, nt, done, st);
  // 8-B aligned rows: 16-px strips of six 8-B loads (the W % 16 == 8 remainder is the scalar tail)
  if (a % 8 == 0 && W % 8 == 0 && W >= 16 && hist_w8_strip16())
    return launch_nt<16, 8>(rgb, B, H, W, hist_s, hist_graw, grid, nt, done, st);
  if (a % 8 == 0 && W % 8 == 0) return launch_nt<8, 8>(rgb, B, H, W, hist_s, hist_graw, grid, nt, done, st);
  return launch_nt<16, 1>(rgb, B, H, W, hist_s, hist_graw, grid, nt, done, st);
}

}  // namespace hr
