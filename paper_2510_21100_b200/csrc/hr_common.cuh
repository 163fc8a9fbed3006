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

// ---- step timeline (measurement: hr_trace_bind; bench.py's in-step kernel durations) ----
// While a record buffer is bound, thread 0 of every CTA of k_hist / k_solve / k_apply appends
// {kernel, CTA, SM, aux, start, mid, end} (%globaltimer ns); aux tells launches of one kernel
// apart (hist/solve: the group's hist_s address >> 8), mid = when a solver CTA's image was
// complete (its wait ends).  Unbound (the default) a CTA only tests one pointer at its start.
// Each translation unit holds its own pointer copies, bound by hr_trace_bind.
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
  if (t0 != 0ull && threadIdx.x == 0) {
    const uint32_t i = atomicAdd(g_trace_n, 1u);
    if (i < g_trace_cap) g_trace[i] = TraceRec{kind, blockIdx.x, smid(), aux, t0, mid, gtime(), 0ull};
  }
}
inline cudaError_t trace_bind_tu(void* buf, uint32_t* n, uint32_t cap) {
  cudaError_t e = cudaMemcpyToSymbol(g_trace, &buf, sizeof(void*));
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_trace_n, &n, sizeof(void*));
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_trace_cap, &cap, sizeof(uint32_t));
  return e;
}
}  // namespace
#define TRACE_T0() const unsigned long long tr_t0_ = (threadIdx.x == 0 && g_trace) ? gtime() : 0ull
#define TRACE_MID(v) \
  if (tr_t0_) v = gtime()
#define TRACE_END(kind, aux, mid) trace_rec((kind), (aux), tr_t0_, (mid))
cudaError_t trace_bind_hist(void* buf, uint32_t* n, uint32_t cap);
cudaError_t trace_bind_solve(void* buf, uint32_t* n, uint32_t cap);
cudaError_t trace_bind_apply(void* buf, uint32_t* n, uint32_t cap);

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

constexpr int kHistThreads = 512;  // k_hist: 16 warps, 2 CTAs per SM
constexpr int kApplyThreads = 256; // k_apply: 8 warps, 2 CTAs per SM

// Spin-wait bound for the cross-grid flags (k_solve waiting for its image's histogram rows,
// k_apply for a LUT): a wall-clock bound from %globaltimer, far above any real wait.  Reaching
// it is a logic error: the checked build traps, the product build stops waiting.
constexpr unsigned long long kSpinLimitNs = 30ull * 1000 * 1000 * 1000;
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// wait until *p >= need (acquire); returns false on timeout
__device__ __forceinline__ bool wait_flag_geq(const uint32_t* p, uint32_t need, unsigned sleep_ns) {
  if (ld_acquire(p) >= need) return true;
  const unsigned long long t0 = global_ns();
  for (;;) {
    __nanosleep(sleep_ns);
    if (ld_acquire(p) >= need) return true;
    if (global_ns() - t0 > kSpinLimitNs) {
#ifdef HR_CHECKS
      printf("HR_CHECK: flag wait timed out (block %d)\n", (int)blockIdx.x);
      asm volatile("trap;");
#endif
      return false;
    }
  }
}

// Launch helpers implemented in the kernel translation units.
// Kernel attributes (dynamic shared memory opt-in, carve-out) are per device: hr_create calls
// init_kernel_attrs() once per device (std::call_once), with that device current.
cudaError_t init_attrs_hist();
cudaError_t init_attrs_solve();
cudaError_t init_attrs_apply();
// grid: CTAs (2 per SM by default); done (nullable): per-image counts of flushed rows (a segment
// of image b adds its row count to done[b] after its flush, a release);
// nowait: the kernel does not wait for its stream predecessor (griddepcontrol.wait) -- only for a
// predecessor it shares no data with (the grouped step's histograms of group k >= 1 follow the
// solver of group k - 1)
cudaError_t launch_hist(const uint8_t* rgb, int64_t B, int32_t H, int32_t W, uint32_t* hist_s,
                        uint32_t* hist_graw, int grid, cudaStream_t st, uint32_t* done = nullptr,
                        bool nowait = false, int nt = kHistThreads);
int hist_grid_clamped(int64_t B, int32_t H, int grid);  // the grid launch_hist actually uses
cudaError_t launch_remap(const uint32_t* hist_graw, int64_t B, int32_t grad_norm, uint32_t* hist_g,
                         cudaStream_t st);

struct SolveArgs {
  const uint32_t* hist_s;   // [B][256]
  const uint32_t* hist_g;   // [B][256] remapped gradient histogram, or NULL -> use graw
  uint32_t* hist_g_out;     // [B][256] nullable: the remapped gradient histogram (debug output)
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
  uint32_t* ready;               // [B] nullable (k_solve): released (= 1) once image b's LUT is written
  const uint32_t* hist_done;     // [B] nullable (k_solve): start image b once all its rows are flushed
  int32_t hist_H;                // ... rows per image: image b is complete when hist_done[b] == hist_H
  int32_t arena_bytes;           // shared run arena per CTA (0: the default 80 KB)
  double* trace;                 // [B][trace_stride] nullable: Eq. 10 objective, 3 values per update
  int32_t trace_stride;
};
cudaError_t launch_idx1_table(double gamma, uint8_t* tab, cudaStream_t st);
// cpsm: solver CTAs per SM the launch is sized for (1: the shared memory a lone CTA reserves
// goes to the run arena); wide (with cpsm == 1): 512-thread CTAs (large supports: C4 103 vs
// 121 us per image; small ones are faster at 256 threads: C2 37 vs 43 us)
cudaError_t launch_solve(const SolveArgs& a, int64_t B, int cpsm, cudaStream_t st, bool wide = false);
size_t solve_smem_bytes(int arena_bytes = 0);
// the cluster solver (one image per cluster of kClusterCS CTAs; large single images)
constexpr int kClusterCS = 16;   // largest cluster (ranks with their own global arenas)
constexpr int kClusterMaxB = 9;  // images per cluster launch (148 SMs / 16)
// variant: 1 = 8 CTAs x 256 threads, 2 = 8 x 512, 3 = 16 x 256, 4 = 16 x 512
cudaError_t launch_solve_cluster(const SolveArgs& a, int64_t B, cudaStream_t st, int variant);
size_t solve_cells_ws_bytes(int64_t B);

cudaError_t launch_match(const uint32_t* hist_s, const double* target, int64_t B, uint8_t* lut,
                         int32_t* status, cudaStream_t st);

// ready (nullable): per-image LUT-ready flags released by k_solve; when given, the TMA apply
// does not wait for the solver grid to finish but acquires ready[b] before image b's table.
// b_last (0 < b_last < B): every CTA first takes its share of images [0, b_last); with ticket
// (a zeroed counter) images [b_last, B) go by CTA tickets of 8 * GS chunks (the grouped step:
// the last group's LUTs complete last), else by static shares
cudaError_t launch_apply(const uint8_t* in, const uint8_t* lut, int64_t B, int32_t H, int32_t W,
                         uint8_t* out, int grid_ctas, cudaStream_t st, const uint32_t* ready = nullptr,
                         int64_t b_last = 0, uint32_t* ticket = nullptr, int GS = 8);
// second workload (k_quality.cu): HE LUT per image (Eq. 4-5) and the quality metrics
cudaError_t launch_he_lut(const uint32_t* hist_s, int64_t B, uint8_t* lut, cudaStream_t st);
size_t quality_ws_bytes(int64_t B, int32_t H, int32_t W);
cudaError_t launch_quality(const uint8_t* a, const uint8_t* b, int64_t B, int32_t H, int32_t W, double* psnr,
                           double* ssim, double* loe, void* ws, cudaStream_t st);
// zero n bytes (n % 16 == 0, 16-B aligned) -- replaces cudaMemsetAsync inside the PDL chain
cudaError_t launch_zero(void* p, size_t n, cudaStream_t st);

// Control block of hr_enhance (zeroed every step): [header | done[B] | ready[B]]; header word 3
// = the apply's ticket counter.
constexpr int kCtlHeader = 32;
inline size_t ctl_bytes(int64_t B) { return (size_t)(kCtlHeader + 2 * B) * sizeof(uint32_t); }

}  // namespace hr
