// hr_common.cuh -- shared device-side definitions of the HistRetinex CUDA path (sm_100a).
//
// Product code.  Shares nothing with oracle/ (the CPU test oracle).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <utility>

#include "../../include/histretinex.h"

namespace hr {

// ---- invariant checks (checked builds only: -DHR_CHECKS; tools/build_measure_libs.sh) ----
// compute-sanitizer is not available on the GPU pool, so a checked build asserts the indexing
// invariants the kernels rely on and the whole GPU suite runs against it (HR_LIB=...).
#ifdef HR_CHECKS
#define HR_CHECK(cond)                                                                       \
  do {                                                                                       \
    if (!(cond)) {                                                                           \
      printf("HR_CHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__, \
             (int)blockIdx.x, (int)threadIdx.x);                                             \
      asm volatile("trap;");                                                                 \
    }                                                                                        \
  } while (0)
#else
#define HR_CHECK(cond) \
  do {                 \
  } while (0)
#endif

// ---- programmatic dependent launch (PDL) ----
// Kernels of a step are launched with programmatic stream serialization: a kernel's launch
// (CTA rasterisation, shared-memory carve-out) overlaps its predecessor's tail.  Every such
// kernel calls pdl_wait() before touching memory, which returns once the predecessor grid has
// completed and its writes are visible (a no-op for a normal launch), then pdl_trigger() so
// that its own successor may launch early.  HR_PDL=0 disables the attribute (A/B timing).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" :::); }
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("HR_PDL");
    return !(e && atoi(e) == 0);
  }();
  return on;
}
// gpu-scope acquire / release on a 32-bit flag (LUT-ready handshakes between CTAs and grids)
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

constexpr int kLevels = 256;     // l (the only level count of this build)
constexpr int kGradSlots = 512;  // raw gradient |dx|+|dy| in [0, 510]
constexpr int kMaxGrad = 510;

// ---------------------------------------------------------------- k_hist
constexpr int kHistThreads = 512;  // 16 warps; 2 CTAs per SM (96 KB smem each)
constexpr int kLanes = 32;
// Lane-private sub-histograms: counter for bin v of lane l at word v*32 + l, so every
// smem atomic of a warp hits 32 distinct banks whatever the data skew.
constexpr int kHistSmemBytes = (kLevels + kGradSlots) * kLanes * 4;  // 98,304 B

// ---------------------------------------------------------------- k_solve
constexpr int kSolveThreads = 256;  // one thread per level for the per-bin phases
constexpr int kSolveWarps = kSolveThreads / 32;

// ---------------------------------------------------------------- k_apply
constexpr int kApplyThreads = 256;

// Launch helpers implemented in the kernel translation units.
// nt: threads per CTA (512, or 256 to leave room for a solver CTA); done (nullable): per-image
// counts of flushed segments (see hist_segments_of)
cudaError_t launch_hist(const uint8_t* rgb, int64_t B, int32_t H, int32_t W, uint32_t* hist_s,
                        uint32_t* hist_graw, int grid, cudaStream_t st, int nt = kHistThreads,
                        uint32_t* done = nullptr);
int hist_grid_clamped(int64_t B, int32_t H, int grid);  // the grid launch_hist actually uses
// number of k_hist CTA row ranges [R c / G, R (c+1) / G) overlapping image b's rows [bH, (b+1)H)
__host__ __device__ inline int hist_segments_of(int64_t b, int64_t H, int64_t R, int64_t G) {
  const int64_t first = ((b * H + 1) * G + R - 1) / R - 1;      // min c with R (c+1) / G > bH
  int64_t last = ((b + 1) * H * G + R - 1) / R - 1;             // max c with R c / G < (b+1) H
  if (last > G - 1) last = G - 1;
  return (int)(last - first + 1);
}
cudaError_t launch_remap(const uint32_t* hist_graw, int64_t B, int32_t grad_norm, uint32_t* hist_g,
                         cudaStream_t st);


struct SolveArgs {
  const uint32_t* hist_s;   // [B][256]
  const uint32_t* hist_g;   // [B][256] remapped gradient histogram, or NULL -> use graw
  const uint32_t* graw;     // [B][512] raw gradient histogram (used when hist_g == NULL)
  int32_t grad_norm;        // remap mode when reading graw
  hr_params p;
  double* hL;               // [B][256] nullable
  double* hR;               // [B][256] nullable
  double* target;           // [B][256] nullable
  int32_t* iters;           // [B] nullable
  uint8_t* lut;             // [B][256] nullable (fused CDF + LUT tail)
  int32_t* status;          // [B] nullable
  unsigned char* cells_ws;  // [B][kArenaGlobal] run arenas of images whose runs exceed shared memory
  const uint8_t* idx1_tab;  // [256][256] index_1(i, j) for params.gamma (launch_idx1_table)
  const int32_t* only_deferred;  // k_solve: when set, images with only_deferred[b] == 0 are skipped
  uint32_t* ready;               // [B] nullable (k_solve): released (= 1) once image b's LUT is written
  uint32_t* queue;               // [B] nullable (k_solve): completion queue, queue[i] = (i-th finished b) + 1
  uint32_t* queue_tail;          // ... its tail counter
  const uint32_t* hist_done;     // [B] nullable (k_solve): start image b once all its segments flushed
  int32_t hist_grid;             // ... k_hist's grid (the segment count follows from it)
  int32_t hist_H;                // ... rows per image
  int32_t arena_bytes;           // shared run arena per CTA (0: the default 80 KB)
  double* trace;                 // [B][trace_stride] nullable: Eq. 10 objective, 3 values per update
  int32_t trace_stride;
};
// warp-per-image solver for nR <= 32; flags the other images in deferred[b] (then run k_solve)
cudaError_t launch_solve_warp(const SolveArgs& a, int64_t B, int32_t* deferred, cudaStream_t st);
cudaError_t launch_idx1_table(double gamma, uint8_t* tab, cudaStream_t st);
cudaError_t launch_solve(const SolveArgs& a, int64_t B, int cpsm, cudaStream_t st);
size_t solve_smem_bytes(int arena_bytes = 0);
size_t solve_cells_ws_bytes(int64_t B);

cudaError_t launch_match(const uint32_t* hist_s, const double* target, int64_t B, uint8_t* lut,
                         int32_t* status, cudaStream_t st);

// ready (nullable): per-image LUT-ready flags released by k_solve; when given, the TMA apply
// does not wait for the solver grid to finish but acquires ready[b] before image b's table
cudaError_t launch_apply(const uint8_t* in, const uint8_t* lut, int64_t B, int32_t H, int32_t W,
                         uint8_t* out, int grid_ctas, cudaStream_t st, const uint32_t* ready = nullptr);
// dynamic apply: warps take groups of GS chunks of the images in LUT-completion order (queue
// filled by k_solve); false when the shape needs the scalar path (then use launch_apply)
bool apply_dyn_supported(const uint8_t* in, const uint8_t* out, int64_t B, int32_t H, int32_t W);
cudaError_t launch_apply_dyn(const uint8_t* in, const uint8_t* lut, int64_t B, int32_t H, int32_t W, uint8_t* out,
                             int grid_ctas, const uint32_t* queue, uint32_t* ticket, int GS, cudaStream_t st);
// second workload (k_quality.cu): HE LUT per image (Eq. 4-5) and the quality metrics
cudaError_t launch_he_lut(const uint32_t* hist_s, int64_t B, uint8_t* lut, cudaStream_t st);
size_t quality_ws_bytes(int64_t B, int32_t H, int32_t W);
cudaError_t launch_quality(const uint8_t* a, const uint8_t* b, int64_t B, int32_t H, int32_t W, double* psnr,
                           double* ssim, double* loe, void* ws, cudaStream_t st);
// zero n bytes (n % 16 == 0, 16-B aligned) -- replaces cudaMemsetAsync inside the PDL chain
cudaError_t launch_zero(void* p, size_t n, cudaStream_t st);

// Persistent fused kernel (k_fused.cu): histograms -> per-image solve + LUT -> apply.
constexpr int kCtlHeader = 32;  // control words before done[B]
// control block: [header | done[B] | ready[B] | queue[B]]; header word 2 = completion-queue
// tail, word 3 = dynamic-apply ticket
inline size_t fused_ctl_bytes(int64_t B) { return (size_t)(kCtlHeader + 3 * B) * sizeof(uint32_t); }
struct FusedArgs {
  const uint8_t* in;  // [B][H][W][3]
  uint8_t* out;       // [B][H][W][3]
  int64_t B;
  int32_t H, W;
  uint32_t* hist_s;   // [B][256]  zeroed accumulators
  uint32_t* graw;     // [B][512]  zeroed accumulators
  uint32_t* ctl;      // [kCtlHeader + 2B] zeroed: [0] band ticket, [1] apply ticket, done[B], ready[B]
  SolveArgs sa;       // solver view: hist_s/graw (as above), lut, params, idx1 table, cells_ws
  int32_t KB;         // histogram bands per image
  uint32_t cpi;       // apply chunks per image (set by launch_fused)
  uint32_t GS;        // chunks per apply ticket
};
bool fused_supported(const uint8_t* in, const uint8_t* out, int64_t B, int32_t H, int32_t W);
size_t fused_smem_bytes();
cudaError_t launch_fused(FusedArgs a, int grid, cudaStream_t st);

}  // namespace hr
