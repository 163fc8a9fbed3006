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

// ---- step timeline (measurement builds only: -DHR_STEP_TRACE; tools/step_trace.py) ----
// Thread 0 of every CTA of k_hist / k_solve / k_apply appends {kernel, CTA, SM, aux, start, end}
// (globaltimer ns) to a host-bound buffer; aux = the image a solver CTA solved (its wait for the
// image's histogram ends at `mid`).  Each translation unit holds its own pointer copies, bound
// by hr_debug_trace_bind.
#ifdef HR_STEP_TRACE
struct TraceRec {
  uint32_t kind, cta, sm, aux;
  unsigned long long t0, mid, t1, pad;
};
namespace {
__device__ TraceRec* g_trace = nullptr;
__device__ uint32_t* g_trace_n = nullptr;
__device__ uint32_t g_trace_cap = 0;
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint32_t smid() {
  uint32_t s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  return s;
}
__device__ __forceinline__ void trace_rec(uint32_t kind, uint32_t aux, unsigned long long t0, unsigned long long mid) {
  if (threadIdx.x == 0 && g_trace) {
    const uint32_t i = atomicAdd(g_trace_n, 1u);
    if (i < g_trace_cap) g_trace[i] = TraceRec{kind, blockIdx.x, smid(), aux, t0, mid, gtime(), 0ull};
  }
}
inline void trace_bind_tu(void* buf, uint32_t* n, uint32_t cap) {
  cudaMemcpyToSymbol(g_trace, &buf, sizeof(void*));
  cudaMemcpyToSymbol(g_trace_n, &n, sizeof(void*));
  cudaMemcpyToSymbol(g_trace_cap, &cap, sizeof(uint32_t));
}
}  // namespace
#define TRACE_T0() const unsigned long long tr_t0_ = gtime()
#define TRACE_MID(v) v = gtime()
#define TRACE_END(kind, aux, mid) trace_rec((kind), (aux), tr_t0_, (mid))
#else
#define TRACE_T0() \
  do {             \
  } while (0)
#define TRACE_MID(v) \
  do {               \
  } while (0)
#define TRACE_END(kind, aux, mid) \
  do {                            \
  } while (0)
#endif
void trace_bind_hist(void* buf, uint32_t* n, uint32_t cap);
void trace_bind_solve(void* buf, uint32_t* n, uint32_t cap);
void trace_bind_apply(void* buf, uint32_t* n, uint32_t cap);

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
// counts of flushed rows (a segment of image b adds its row count to done[b] after its flush);
// tma: use the TMA-staged kernel when the shape allows it (tma_hist_supported): one CTA per SM
// (grid / 2), and with done: 512 threads at <= 64 registers in image waves
// (hist_wave_images), leaving registers and shared memory for one solver CTA per SM
cudaError_t launch_hist(const uint8_t* rgb, int64_t B, int32_t H, int32_t W, uint32_t* hist_s,
                        uint32_t* hist_graw, int grid, cudaStream_t st, int nt = kHistThreads,
                        uint32_t* done = nullptr, int tma = 1, bool nowait = false, uint32_t* cq = nullptr,
                        uint32_t* cq_tail = nullptr);
// cq, cq_tail (with done; direct-load kernel): the segment that completes image b appends b + 1
// to cq at atomicAdd(cq_tail) (release), i.e. images in histogram-completion order
// nowait: the kernel does not wait for its stream predecessor (griddepcontrol.wait); only for a
// predecessor it shares no data with (the grouped step's histograms of group k >= 1 follow the
// solver of group k - 1)
int hist_grid_clamped(int64_t B, int32_t H, int grid);  // the grid launch_hist actually uses
bool tma_hist_supported(const uint8_t* rgb, int64_t B, int32_t H, int32_t W);
// Wave order of the TMA histogram kernel with per-image completion counts: images
// [w k, min(B, (w + 1) k)) form wave w and CTA c of G takes rows [R_w c / G, R_w (c + 1) / G) of
// the wave (R_w = its images x H), so the images of wave w are complete once every CTA has
// passed wave w.  Returns the images per wave for a target of ~rows_per_cta rows per CTA.
__host__ __device__ inline int64_t hist_wave_images(int64_t B, int64_t H, int64_t G, int64_t rows_per_cta) {
  int64_t k = (rows_per_cta * G + H - 1) / H;
  if (k < 1) k = 1;
  return k < B ? k : B;
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
  const uint32_t* hist_done;     // [B] nullable (k_solve): start image b once all its rows are flushed
  int32_t hist_H;                // ... rows per image: image b is complete when hist_done[b] == hist_H
  int32_t arena_bytes;           // shared run arena per CTA (0: the default 80 KB)
  double* trace;                 // [B][trace_stride] nullable: Eq. 10 objective, 3 values per update
  int32_t trace_stride;
  int64_t nimg;                  // > 0: images solved by a grid of fewer CTAs (CTA c: c, c + grid, ...);
                                 // 0: one image per CTA
  const uint32_t* cq;            // nullable (with hist_done): histogram-completion queue (k_hist); each
  uint32_t* cq_head;             // CTA solves the image at cq[atomicAdd(cq_head)] - 1 (acquire)
};
// warp-per-image solver for nR <= 32; flags the other images in deferred[b] (then run k_solve)
cudaError_t launch_solve_warp(const SolveArgs& a, int64_t B, int32_t* deferred, cudaStream_t st);
cudaError_t launch_idx1_table(double gamma, uint8_t* tab, cudaStream_t st);
// max_ctas > 0: at most that many CTAs, each solving images c, c + grid, ... in turn (releasing
// each image's ready flag as it completes)
// wide (with cpsm == 1): 512-thread CTAs (large supports: C4 103 vs 121 us per image; small ones
// are faster at 256 threads: C2 37 vs 43 us)
cudaError_t launch_solve(const SolveArgs& a, int64_t B, int cpsm, cudaStream_t st, int max_ctas = 0,
                         bool wide = false);
size_t solve_smem_bytes(int arena_bytes = 0);
size_t solve_cells_ws_bytes(int64_t B);

cudaError_t launch_match(const uint32_t* hist_s, const double* target, int64_t B, uint8_t* lut,
                         int32_t* status, cudaStream_t st);

// ready (nullable): per-image LUT-ready flags released by k_solve; when given, the TMA apply
// does not wait for the solver grid to finish but acquires ready[b] before image b's table
cudaError_t launch_apply(const uint8_t* in, const uint8_t* lut, int64_t B, int32_t H, int32_t W,
                         uint8_t* out, int grid_ctas, cudaStream_t st, const uint32_t* ready = nullptr,
                         int64_t b_last = 0, uint32_t* ticket = nullptr, int GS = 8, int tail_pct = 0);
// b_last (0 < b_last < B): every CTA first takes its share of images [0, b_last), then its share
// of [b_last, B) (the grouped step: the last group's LUTs complete last); with ticket (zeroed
// counter), images [b_last, B) go by CTA tickets of 8 * GS chunks instead of static shares
// dynamic apply: warps take groups of GS chunks of the images in LUT-completion order (queue
// filled by k_solve); false when the shape needs the scalar path (then use launch_apply)
bool apply_dyn_supported(const uint8_t* in, const uint8_t* out, int64_t B, int32_t H, int32_t W);
cudaError_t launch_apply_dyn(const uint8_t* in, const uint8_t* lut, int64_t B, int32_t H, int32_t W, uint8_t* out,
                             int grid_ctas, const uint32_t* queue, uint32_t* ticket, int GS, cudaStream_t st,
                             const uint32_t* ready = nullptr, int64_t b_last = 0);
// (ready given, queue NULL, 0 < b_last < B: images [0, b_last) split statically per CTA, images
// [b_last, B) by tickets)
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
// control block: header, done[B], ready[B], LUT queue[B], histogram-completion queue[B], and per
// group (<= 64) the completion queue's tail and head counters
inline size_t fused_ctl_bytes(int64_t B) { return (size_t)(kCtlHeader + 4 * B + 128) * sizeof(uint32_t); }
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
