// hr_api.cu -- the C-ABI boundary (include/histretinex.h): validation, context, launches.
//
// Every entry point validates synchronously and enqueues nothing on error.  No exception
// or exit() crosses the boundary.
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <new>
#include <vector>

#include "hr_common.cuh"

struct hr_ctx {
  int device = 0;
  int num_sms = 148;
  int l2_bytes = 0;
  char last_error[512] = {0};
  // index_1 tables of Eqs. 17-19, one per gamma (64 KB each, built on first use, stream-ordered)
  static constexpr int kTab = 8;
  uint8_t* idx1_tab[kTab] = {};
  double idx1_gamma[kTab] = {};
  int idx1_next = 0;
  // execution policy of hr_enhance (defaults chosen from B200 measurements; HR_* env overrides)
  int chunks = 1;         // >1: fork/join pipeline over image chunks (hist | solve | apply streams)
  int hist_cpsm = 2;      // k_hist CTAs per SM
  int apply_cpsm = 2;     // k_apply CTAs per SM
  int warp_solver = 0;    // 1: k_solve_warp for nR <= 32, k_solve for the rest; 0: k_solve only
  int fused_min_b = 0;    // hr_enhance: persistent fused kernel for B >= this (0: never) ...
  int fused_max_b = 0;    // ... and B <= this (0: auto = SMs / 2: the solves' CTA slots stay cheap)
  int fused_cpsm = 2;     // k_fused CTAs per SM
  int fused_bands = 2;    // histogram band items per CTA (sets bands per image)
  int fused_gs = 8;       // 1024-px chunks per apply ticket
  int solve_cpsm = 0;     // k_solve CTAs per SM: 1, 2, or 0 = auto (1 when B <= SMs)
  int apply_gs = 8;       // dynamic apply: 1024-px chunks per warp ticket
  int apply_dyn = 0;      // separate kernels: 1 = the apply takes images in LUT-completion order,
                          // 2 = natural order after the solver grid, 3 = natural order gated by the
                          // per-image LUT-ready flags; warp tickets balancing the work
                          // (off: per-warp tickets scatter the streams; C3 0.364 vs 0.269 ms)
  int hist_tma = 0;       // k_hist: TMA-staged rows where the shape allows (off: measured no faster)
  int hist_overlap = 0;   // separate kernels: solves start per image beside a 2x256-thread histogram pass
                          // (off: the 16-warp histogram pass costs more than the overlap saves)
  int solve_queue = 0;    // grouped step: solver CTAs take images in histogram-completion order
  int group_apply = 2;    // grouped step's apply: 0 = static shares of groups 0..G-2, then of the
                          // last group; 1 = last group by warp-ring CTA tickets (k_apply_dyn,
                          // measured slower); 2 = last group by CTA tickets taken at barriers
                          // (k_apply_tma; C3 0.250-0.252 vs 0.254-0.259, C5 0.168 vs 0.168-0.173)
  int solve_wide_px = 4 << 20;  // hr_enhance: 512-thread solver CTAs (one per SM) for H*W >= this (0: never)
  int solve_waves = 0;    // separate kernels, B > SMs: one solver CTA per SM solving images in turn
  int solve_waves_ag = 1; // ... apply CTAs per SM launched beside it
  int apply_tail_pct = 0;   // grouped step, group_apply 2: % of the first groups' chunks also ticketed
  int group_first_pct = -1;  // grouped step, G = 2: first group's share of the images in % (0: half;
                             // -1: auto = 38 for B <= SMs / 2 -- a short hist(0) lets solve(0) hide
                             // under the longer hist(1), C3 24 + 40 images 0.254 ms vs 32 + 32 0.261 --
                             // and 90 for larger batches -- the last group's few solves overlap the
                             // first group's apply, C5 230 + 26 images 0.167 vs 0.177 ungrouped)
  int groups = -1;        // grouped step (>= 2): histograms of group k+1 run beside the solves of
                          // group k, the apply beside the last group's solves (0/1: off)
  int64_t launches = 0;   // kernels launched through this context (hr_kernel_launches)
  int last_path = -1;     // hr_last_path: 0 separate kernels, 1 fused, 2 chunk pipeline, 3 grouped
  cudaStream_t sH = nullptr, sS = nullptr, sA = nullptr;
  std::vector<cudaEvent_t> pev;  // pipeline events
  cudaStream_t sIn = nullptr, sOut = nullptr;  // hr_enhance_host copy streams
  std::vector<cudaEvent_t> hev;                // hr_enhance_host events
  // stage timing (hr_profile_*)
  bool prof = false;
  int prof_used = 0;
  std::vector<cudaEvent_t> prof_ev;  // 4 per recorded call
};

namespace {

using hr::kGradSlots;
using hr::kLevels;

size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

constexpr int kOverlapArena = 40 * 1024;  // solver shared arena when it runs beside the histograms

// count a successful kernel launch
inline cudaError_t counted(hr_ctx* c, cudaError_t e) {
  if (e == cudaSuccess) ++c->launches;
  return e;
}

struct WsLayout {
  size_t hist_s, graw, ctl, lut, iters, target, deferred, cells, total;
};

WsLayout ws_layout(int64_t B) {
  WsLayout L;
  size_t o = 0;
  L.hist_s = o;
  o = align_up(o + (size_t)B * kLevels * sizeof(uint32_t));
  L.graw = o;
  o = align_up(o + (size_t)B * kGradSlots * sizeof(uint32_t));
  L.ctl = o;  // fused-kernel control block, right after graw: one memset clears all three
  o = align_up(o + hr::fused_ctl_bytes(B));
  L.lut = o;
  o = align_up(o + (size_t)B * kLevels);
  L.iters = o;
  o = align_up(o + (size_t)B * sizeof(int32_t));
  L.target = o;
  o = align_up(o + (size_t)B * kLevels * sizeof(double));
  L.deferred = o;
  o = align_up(o + (size_t)B * sizeof(int32_t));
  L.cells = o;
  o = align_up(o + hr::solve_cells_ws_bytes(B));
  L.total = o;
  return L;
}

hr_status set_err(hr_ctx* c, hr_status s, const char* msg) {
  if (c) snprintf(c->last_error, sizeof c->last_error, "%s", msg);
  return s;
}

hr_status cuda_err(hr_ctx* c, cudaError_t e, const char* where) {
  if (e == cudaSuccess) return HR_OK;
  if (c) snprintf(c->last_error, sizeof c->last_error, "%s: %s", where, cudaGetErrorString(e));
  return HR_ECUDA;
}

hr_status check_shape(hr_ctx* c, int64_t B, int32_t H, int32_t W) {
  if (B < 1 || H < 0 || W < 0) return set_err(c, HR_EINVAL, "B must be >= 1 and H, W >= 0");
  if ((int64_t)H * W == 0) return set_err(c, HR_EEMPTY, "empty image (H*W == 0)");
  if (B > (1 << 30) || (int64_t)H * W > (int64_t)1 << 32) return set_err(c, HR_EINVAL, "size too large");
  return HR_OK;
}

hr_status check_params(hr_ctx* c, const hr_params* p) {
  if (!p) return set_err(c, HR_EINVAL, "params is NULL");
  if (p->levels != 256) return set_err(c, HR_EUNSUPPORTED, "levels must be 256");
  if (!(p->alpha > 0) || !(p->beta > 0)) return set_err(c, HR_EINVAL, "alpha and beta must be > 0");
  if (!(p->gamma >= 1.0)) return set_err(c, HR_EINVAL, "gamma must be >= 1");
  if (!(p->epsilon > 0)) return set_err(c, HR_EINVAL, "epsilon must be > 0");
  if (p->max_iter < 1) return set_err(c, HR_EINVAL, "max_iter must be >= 1");
  if (p->use_epsilon != 0 && p->use_epsilon != 1) return set_err(c, HR_EINVAL, "use_epsilon must be 0/1");
  if (p->update_form != 0 && p->update_form != 1) return set_err(c, HR_EINVAL, "update_form must be 0/1");
  if (p->grad_norm != 0 && p->grad_norm != 1) return set_err(c, HR_EINVAL, "grad_norm must be 0/1");
  if (p->reserved != 0) return set_err(c, HR_EINVAL, "reserved must be 0");
  return HR_OK;
}

hr_status activate(hr_ctx* c) {
  int cur = -1;
  cudaError_t e = cudaGetDevice(&cur);
  if (e != cudaSuccess) return cuda_err(c, e, "cudaGetDevice");
  if (cur != c->device) {
    e = cudaSetDevice(c->device);
    if (e != cudaSuccess) return cuda_err(c, e, "cudaSetDevice");
  }
  return HR_OK;
}

int hist_grid(const hr_ctx* c) { return c->hist_cpsm * c->num_sms; }

// index_1 table for gamma, building it on `st` when it is not cached (round-robin over kTab)
cudaError_t idx1_table(hr_ctx* c, double gamma, cudaStream_t st, const uint8_t** out) {
  for (int i = 0; i < hr_ctx::kTab; ++i)
    if (c->idx1_tab[i] && c->idx1_gamma[i] == gamma) {
      *out = c->idx1_tab[i];
      return cudaSuccess;
    }
  const int i = c->idx1_next;
  c->idx1_next = (i + 1) % hr_ctx::kTab;
  if (!c->idx1_tab[i]) {
    cudaError_t e = cudaMalloc(&c->idx1_tab[i], 256 * 256);
    if (e != cudaSuccess) return e;
  }
  c->idx1_gamma[i] = gamma;
  *out = c->idx1_tab[i];
  return counted(c, hr::launch_idx1_table(gamma, c->idx1_tab[i], st));
}
int apply_grid(const hr_ctx* c) { return c->apply_cpsm * c->num_sms; }
int solve_cpsm_for(const hr_ctx* c, int64_t B) { return c->solve_cpsm ? c->solve_cpsm : (B <= c->num_sms ? 1 : 2); }

}  // namespace

extern "C" {

hr_status hr_default_params(hr_params* p) {
  if (!p) return HR_EINVAL;
  p->levels = 256;
  p->max_iter = 10;
  p->alpha = 0.1;
  p->beta = 1e-3;
  p->gamma = 2.2;
  p->epsilon = 1e-3;
  p->use_epsilon = 0;
  p->update_form = 0;
  p->grad_norm = 0;
  p->reserved = 0;
  return HR_OK;
}

hr_status hr_create(hr_ctx** out, int device) {
  if (!out) return HR_EINVAL;
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n) {
    cudaGetLastError();
    return HR_ECUDA;
  }
  hr_ctx* c = new (std::nothrow) hr_ctx();
  if (!c) return HR_ECUDA;
  c->device = device;
  if (cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess ||
      cudaDeviceGetAttribute(&c->l2_bytes, cudaDevAttrL2CacheSize, device) != cudaSuccess) {
    cudaGetLastError();
    delete c;
    return HR_ECUDA;
  }
  if (const char* v = getenv("HR_CHUNKS")) c->chunks = atoi(v) > 0 ? atoi(v) : 1;
  if (const char* v = getenv("HR_HIST_CPSM")) c->hist_cpsm = atoi(v) > 0 ? atoi(v) : 2;
  if (const char* v = getenv("HR_APPLY_CPSM")) c->apply_cpsm = atoi(v) > 0 ? atoi(v) : 2;
  if (const char* v = getenv("HR_WARP_SOLVER")) c->warp_solver = atoi(v) != 0;
  if (const char* v = getenv("HR_FUSED_MIN_B")) c->fused_min_b = atoi(v) >= 0 ? atoi(v) : 0;
  if (const char* v = getenv("HR_FUSED_MAX_B")) c->fused_max_b = atoi(v) >= 0 ? atoi(v) : 0;
  if (const char* v = getenv("HR_FUSED_CPSM")) c->fused_cpsm = atoi(v) > 0 ? atoi(v) : 2;
  if (const char* v = getenv("HR_FUSED_BANDS")) c->fused_bands = atoi(v) > 0 ? atoi(v) : 2;
  if (const char* v = getenv("HR_FUSED_GS")) c->fused_gs = atoi(v) > 0 ? atoi(v) : 8;
  if (const char* v = getenv("HR_SOLVE_CPSM")) c->solve_cpsm = atoi(v) >= 0 && atoi(v) <= 2 ? atoi(v) : 0;
  if (const char* v = getenv("HR_HIST_OVERLAP")) c->hist_overlap = atoi(v) != 0;
  if (const char* v = getenv("HR_HIST_TMA")) c->hist_tma = atoi(v) != 0;
  if (const char* v = getenv("HR_APPLY_DYN")) c->apply_dyn = atoi(v) >= 0 && atoi(v) <= 3 ? atoi(v) : 0;
  if (const char* v = getenv("HR_APPLY_GS")) c->apply_gs = atoi(v) > 0 ? atoi(v) : 8;
  if (const char* v = getenv("HR_SOLVE_QUEUE")) c->solve_queue = atoi(v) != 0;
  if (const char* v = getenv("HR_GROUP_APPLY")) c->group_apply = atoi(v) >= 0 && atoi(v) <= 2 ? atoi(v) : 2;
  if (const char* v = getenv("HR_SOLVE_WAVES")) c->solve_waves = atoi(v) != 0;
  if (const char* v = getenv("HR_SOLVE_WIDE_PX")) c->solve_wide_px = atoi(v) >= 0 ? atoi(v) : 4 << 20;
  if (const char* v = getenv("HR_SOLVE_WAVES_AG")) c->solve_waves_ag = atoi(v) == 2 ? 2 : 1;
  if (const char* v = getenv("HR_APPLY_TAIL_PCT")) c->apply_tail_pct = atoi(v) >= 0 && atoi(v) <= 100 ? atoi(v) : 0;
  if (const char* v = getenv("HR_GROUP_FIRST_PCT")) c->group_first_pct = atoi(v) >= -1 && atoi(v) < 100 ? atoi(v) : -1;
  if (const char* v = getenv("HR_GROUPS")) c->groups = atoi(v) >= -1 && atoi(v) <= 64 ? atoi(v) : -1;
  *out = c;
  return HR_OK;
}

hr_status hr_destroy(hr_ctx* c) {
  if (c) {
    for (cudaEvent_t e : c->prof_ev) cudaEventDestroy(e);
    for (cudaEvent_t e : c->pev) cudaEventDestroy(e);
    if (c->sH) cudaStreamDestroy(c->sH);
    if (c->sS) cudaStreamDestroy(c->sS);
    if (c->sA) cudaStreamDestroy(c->sA);
    for (cudaEvent_t e : c->hev) cudaEventDestroy(e);
    if (c->sIn) cudaStreamDestroy(c->sIn);
    if (c->sOut) cudaStreamDestroy(c->sOut);
    for (int i = 0; i < hr_ctx::kTab; ++i)
      if (c->idx1_tab[i]) cudaFree(c->idx1_tab[i]);
  }
  delete c;
  return HR_OK;
}

hr_status hr_profile_enable(hr_ctx* c, int32_t on) {
  if (!c) return HR_EINVAL;
  c->prof = on != 0;
  c->prof_used = 0;
  return HR_OK;
}

int64_t hr_kernel_launches(const hr_ctx* c) { return c ? c->launches : -1; }
int32_t hr_last_path(const hr_ctx* c) { return c ? c->last_path : -1; }

namespace {
struct Knob {
  const char* name;
  int* field;
  int64_t lo, hi;
};
// the policy knob named key (nullptr if unknown)
const Knob* find_knob(hr_ctx* c, const char* key, Knob* out) {
  const Knob knobs[] = {
      {"fused_min_b", &c->fused_min_b, 0, 1 << 30}, {"fused_max_b", &c->fused_max_b, 0, 1 << 30},
      {"fused_cpsm", &c->fused_cpsm, 1, 2},
      {"fused_bands", &c->fused_bands, 1, 1 << 20}, {"fused_gs", &c->fused_gs, 1, 1 << 30},
      {"chunks", &c->chunks, 1, 1 << 16},           {"hist_cpsm", &c->hist_cpsm, 1, 2},
      {"apply_cpsm", &c->apply_cpsm, 1, 2},         {"warp_solver", &c->warp_solver, 0, 1},
      {"solve_cpsm", &c->solve_cpsm, 0, 2},         {"hist_overlap", &c->hist_overlap, 0, 1},
      {"apply_dyn", &c->apply_dyn, 0, 3},           {"apply_gs", &c->apply_gs, 1, 1 << 20},
      {"hist_tma", &c->hist_tma, 0, 1},             {"groups", &c->groups, -1, 64},
      {"group_apply", &c->group_apply, 0, 2},       {"group_first_pct", &c->group_first_pct, -1, 99},
      {"apply_tail_pct", &c->apply_tail_pct, 0, 100}, {"solve_queue", &c->solve_queue, 0, 1},       {"solve_waves", &c->solve_waves, 0, 1},
      {"solve_waves_ag", &c->solve_waves_ag, 1, 2}, {"solve_wide_px", &c->solve_wide_px, 0, 1 << 30},
  };
  for (const Knob& k : knobs)
    if (strcmp(k.name, key) == 0) {
      *out = k;
      return out;
    }
  return nullptr;
}
}  // namespace

hr_status hr_set_policy(hr_ctx* c, const char* key, int64_t v) {
  if (!c) return HR_EINVAL;
  if (!key) return set_err(c, HR_EINVAL, "NULL key");
  Knob k;
  if (!find_knob(c, key, &k)) return set_err(c, HR_EINVAL, "unknown policy key");
  if (v < k.lo || v > k.hi) return set_err(c, HR_EINVAL, "policy value out of range");
  *k.field = (int)v;
  return HR_OK;
}

hr_status hr_get_policy(hr_ctx* c, const char* key, int64_t* value) {
  if (!c) return HR_EINVAL;
  if (!key || !value) return set_err(c, HR_EINVAL, "NULL key or value");
  Knob k;
  if (!find_knob(c, key, &k)) return set_err(c, HR_EINVAL, "unknown policy key");
  *value = *k.field;
  return HR_OK;
}

hr_status hr_profile_collect(hr_ctx* c, double* stage_ms, int32_t* steps) {
  if (!c || !stage_ms) return HR_EINVAL;
  hr_status s = activate(c);
  if (s) return s;
  double acc[3] = {0.0, 0.0, 0.0};
  for (int i = 0; i < c->prof_used; ++i) {
    cudaEvent_t* e = &c->prof_ev[4 * i];
    cudaError_t err = cudaEventSynchronize(e[3]);
    if (err != cudaSuccess) return cuda_err(c, err, "hr_profile_collect");
    for (int k = 0; k < 3; ++k) {
      float ms = 0.f;
      err = cudaEventElapsedTime(&ms, e[k], e[k + 1]);
      if (err != cudaSuccess) return cuda_err(c, err, "hr_profile_collect");
      acc[k] += ms;
    }
  }
  for (int k = 0; k < 3; ++k) stage_ms[k] = acc[k];
  if (steps) *steps = c->prof_used;
  c->prof_used = 0;
  return HR_OK;
}

const char* hr_status_string(hr_status s) {
  switch (s) {
    case HR_OK: return "ok";
    case HR_EINVAL: return "invalid argument";
    case HR_EEMPTY: return "empty input";
    case HR_EDEGENERATE: return "degenerate histogram";
    case HR_ECUDA: return "CUDA error";
    case HR_EUNSUPPORTED: return "unsupported";
  }
  return "unknown status";
}

const char* hr_last_error(const hr_ctx* c) { return c ? c->last_error : ""; }

const char* hr_version(void) { return "histretinex-b200 0.1 sm_100a"; }

size_t hr_workspace_bytes(int64_t B, int32_t H, int32_t W) {
  if (B < 1 || H < 0 || W < 0) return 0;
  (void)H;
  (void)W;
  return ws_layout(B).total;
}

hr_status hr_histogram(hr_ctx* c, const uint8_t* rgb, int64_t B, int32_t H, int32_t W, int32_t grad_norm,
                       uint32_t* hist_s, uint32_t* hist_g, uint32_t* hist_g_raw, void* ws, void* stream) {
  if (!c) return HR_EINVAL;
  hr_status s = check_shape(c, B, H, W);
  if (s) return s;
  if (!rgb || !hist_s || !hist_g || !ws) return set_err(c, HR_EINVAL, "NULL pointer");
  if (grad_norm != 0 && grad_norm != 1) return set_err(c, HR_EINVAL, "grad_norm must be 0/1");
  if ((s = activate(c))) return s;
  cudaStream_t st = (cudaStream_t)stream;
  const WsLayout L = ws_layout(B);
  uint32_t* graw = hist_g_raw ? hist_g_raw : reinterpret_cast<uint32_t*>((char*)ws + L.graw);
  cudaError_t e = cudaMemsetAsync(hist_s, 0, (size_t)B * kLevels * sizeof(uint32_t), st);
  if (e == cudaSuccess) e = cudaMemsetAsync(graw, 0, (size_t)B * kGradSlots * sizeof(uint32_t), st);
  if (e == cudaSuccess) e = counted(c, hr::launch_hist(rgb, B, H, W, hist_s, graw, hist_grid(c), st, hr::kHistThreads, nullptr, c->hist_tma));
  if (e == cudaSuccess) e = counted(c, hr::launch_remap(graw, B, grad_norm, hist_g, st));
  return cuda_err(c, e, "hr_histogram");
}

static hr_status solve_impl(hr_ctx* c, const uint32_t* hist_s, const uint32_t* hist_g, int64_t B, const hr_params* p,
                            double* hL, double* hR, double* target, int32_t* iters, double* trace,
                            int32_t trace_stride, void* ws, void* stream) {
  if (!c) return HR_EINVAL;
  if (!hist_s || !hist_g || !hL || !hR || !target || !ws) return set_err(c, HR_EINVAL, "NULL pointer");
  if (B < 1 || B > (1 << 30)) return set_err(c, HR_EINVAL, "B must be >= 1");
  hr_status s = check_params(c, p);
  if (s) return s;
  if ((s = activate(c))) return s;
  hr::SolveArgs a{};
  a.cells_ws = reinterpret_cast<unsigned char*>((char*)ws + ws_layout(B).cells);
  {
    cudaError_t e = idx1_table(c, p->gamma, (cudaStream_t)stream, &a.idx1_tab);
    if (e != cudaSuccess) return cuda_err(c, e, "hr_solve (index_1 table)");
  }
  int32_t* deferred = reinterpret_cast<int32_t*>((char*)ws + ws_layout(B).deferred);
  a.hist_s = hist_s;
  a.hist_g = hist_g;
  a.graw = nullptr;
  a.grad_norm = p->grad_norm;
  a.p = *p;
  a.hL = hL;
  a.hR = hR;
  a.target = target;
  a.iters = iters;
  a.lut = nullptr;
  a.status = nullptr;
  a.trace = trace;
  a.trace_stride = trace_stride;
  cudaError_t e = cudaSuccess;
  if (c->warp_solver && !trace) {  // (the warp solver has no objective trace)
    e = counted(c, hr::launch_solve_warp(a, B, deferred, (cudaStream_t)stream));
    a.only_deferred = deferred;
  }
  if (e == cudaSuccess) e = counted(c, hr::launch_solve(a, B, solve_cpsm_for(c, B), (cudaStream_t)stream));
  return cuda_err(c, e, trace ? "hr_solve_trace" : "hr_solve");
}

hr_status hr_solve(hr_ctx* c, const uint32_t* hist_s, const uint32_t* hist_g, int64_t B, const hr_params* p,
                   double* hL, double* hR, double* target, int32_t* iters, void* ws, void* stream) {
  return solve_impl(c, hist_s, hist_g, B, p, hL, hR, target, iters, nullptr, 0, ws, stream);
}

hr_status hr_solve_trace(hr_ctx* c, const uint32_t* hist_s, const uint32_t* hist_g, int64_t B, const hr_params* p,
                         double* hL, double* hR, double* target, int32_t* iters, double* trace,
                         int32_t trace_stride, void* ws, void* stream) {
  if (!c) return HR_EINVAL;
  if (!trace) return set_err(c, HR_EINVAL, "NULL trace");
  if (p && trace_stride < 3 * p->max_iter) return set_err(c, HR_EINVAL, "trace_stride < 3 * max_iter");
  return solve_impl(c, hist_s, hist_g, B, p, hL, hR, target, iters, trace, trace_stride, ws, stream);
}

hr_status hr_match(hr_ctx* c, const uint32_t* hist_s, const double* target, int64_t B, uint8_t* lut,
                   int32_t* img_status, void* stream) {
  if (!c) return HR_EINVAL;
  if (!hist_s || !target || !lut) return set_err(c, HR_EINVAL, "NULL pointer");
  if (B < 1 || B > (1 << 30)) return set_err(c, HR_EINVAL, "B must be >= 1");
  hr_status s = activate(c);
  if (s) return s;
  return cuda_err(c, counted(c, hr::launch_match(hist_s, target, B, lut, img_status, (cudaStream_t)stream)), "hr_match");
}

hr_status hr_apply(hr_ctx* c, const uint8_t* in, const uint8_t* lut, int64_t B, int32_t H, int32_t W, uint8_t* out,
                   void* stream) {
  if (!c) return HR_EINVAL;
  hr_status s = check_shape(c, B, H, W);
  if (s) return s;
  if (!in || !lut || !out) return set_err(c, HR_EINVAL, "NULL pointer");
  if ((s = activate(c))) return s;
  return cuda_err(c, counted(c, hr::launch_apply(in, lut, B, H, W, out, apply_grid(c), (cudaStream_t)stream)), "hr_apply");
}

hr_status hr_enhance_debug(hr_ctx* c, const uint8_t* in, int64_t B, int32_t H, int32_t W, const hr_params* p,
                           uint8_t* out, void* ws, uint32_t* hist_s_dbg, uint8_t* lut_dbg, int32_t* iters_dbg,
                           void* stream) {
  if (!c) return HR_EINVAL;
  hr_status s = check_shape(c, B, H, W);
  if (s) return s;
  if ((s = check_params(c, p))) return s;
  if (!in || !out || !ws) return set_err(c, HR_EINVAL, "NULL pointer");
  if (in == out) return set_err(c, HR_EINVAL, "rgb_out must not alias rgb_in");
  if ((s = activate(c))) return s;
  cudaStream_t st = (cudaStream_t)stream;
  cudaEvent_t* ev = nullptr;
  if (c->prof) {
    if (c->prof_used >= 4096) return set_err(c, HR_EINVAL, "profile buffer full: call hr_profile_collect");
    while ((int)c->prof_ev.size() < 4 * (c->prof_used + 1)) {
      cudaEvent_t e;
      cudaError_t err = cudaEventCreate(&e);
      if (err != cudaSuccess) return cuda_err(c, err, "cudaEventCreate");
      c->prof_ev.push_back(e);
    }
    ev = &c->prof_ev[4 * c->prof_used];
    c->prof_used++;
  }
  auto mark = [&](int k) -> cudaError_t { return ev ? cudaEventRecord(ev[k], st) : cudaSuccess; };
  const WsLayout L = ws_layout(B);
  uint32_t* hs = hist_s_dbg ? hist_s_dbg : reinterpret_cast<uint32_t*>((char*)ws + L.hist_s);
  uint32_t* graw = reinterpret_cast<uint32_t*>((char*)ws + L.graw);
  uint8_t* lut = lut_dbg ? lut_dbg : reinterpret_cast<uint8_t*>((char*)ws + L.lut);
  double* target = reinterpret_cast<double*>((char*)ws + L.target);
  int32_t* deferred = reinterpret_cast<int32_t*>((char*)ws + L.deferred);
  unsigned char* cells = reinterpret_cast<unsigned char*>((char*)ws + L.cells);
  const uint8_t* tab = nullptr;
  cudaError_t e = idx1_table(c, p->gamma, st, &tab);
  const size_t img = (size_t)H * W * 3;
  // one chunk of images [b0, b0 + nb): histograms | solve + LUT | apply, each on its stream
  auto hist_chunk = [&](int64_t b0, int64_t nb, cudaStream_t s) -> cudaError_t {
    cudaError_t r = counted(c, hr::launch_zero(hs + b0 * kLevels, (size_t)nb * kLevels * sizeof(uint32_t), s));
    if (r == cudaSuccess) r = counted(c, hr::launch_zero(graw + b0 * kGradSlots, (size_t)nb * kGradSlots * sizeof(uint32_t), s));
    if (r == cudaSuccess) r = counted(c, hr::launch_hist(in + b0 * img, nb, H, W, hs + b0 * kLevels, graw + b0 * kGradSlots, hist_grid(c), s, hr::kHistThreads, nullptr, c->hist_tma));
    return r;
  };
  auto solve_chunk = [&](int64_t b0, int64_t nb, cudaStream_t s, uint32_t* ready = nullptr,
                         const uint32_t* hist_done = nullptr, int hist_bands = 0, uint32_t* queue = nullptr,
                         uint32_t* queue_tail = nullptr, int cpsm = 0, int max_ctas = 0,
                         const uint32_t* cq = nullptr, uint32_t* cq_head = nullptr) -> cudaError_t {
    hr::SolveArgs a{};
    a.cq = c->warp_solver ? nullptr : cq;
    a.cq_head = cq_head;
    a.ready = c->warp_solver ? nullptr : ready;
    a.queue = c->warp_solver ? nullptr : queue;
    a.queue_tail = queue_tail;
    a.hist_done = c->warp_solver ? nullptr : hist_done;
    a.hist_H = H;
    a.arena_bytes = hist_done ? kOverlapArena : 0;  // fits beside two histogram CTAs
    if (max_ctas > 0 && !hist_done) {
      // one solver CTA per SM beside one apply CTA: too large for two solvers on an SM (113.5 KB
      // + 1 KB reserved each > 228 KB), small enough for a solver and an apply CTA
      a.arena_bytes = 116224 - (int)(hr::solve_smem_bytes(1) - 1);
    }
    a.idx1_tab = tab;
    a.hist_s = hs + b0 * kLevels;
    a.hist_g = nullptr;
    a.graw = graw + b0 * kGradSlots;
    a.grad_norm = p->grad_norm;
    a.p = *p;
    a.iters = iters_dbg ? iters_dbg + b0 : nullptr;
    a.cells_ws = cells + (size_t)b0 * (hr::solve_cells_ws_bytes(1));
    cudaError_t r = cudaSuccess;
    if (c->warp_solver) {  // the warp solver writes the target; k_match then builds every LUT
      a.target = target + b0 * kLevels;
      r = counted(c, hr::launch_solve_warp(a, nb, deferred + b0, s));
      a.only_deferred = deferred + b0;
      if (r == cudaSuccess) r = counted(c, hr::launch_solve(a, nb, solve_cpsm_for(c, nb), s));
      if (r == cudaSuccess) r = counted(c, hr::launch_match(a.hist_s, a.target, nb, lut + b0 * kLevels, nullptr, s));
      return r;
    }
    a.lut = lut + b0 * kLevels;  // CDF + LUT tail fused into the solver CTA (no target round trip)
    // 512-thread solver CTAs for large images (their supports, and so the cell loops, tend to be
    // large: C4 33 MP 8,480 cells; C2 0.66 MP 1,334 cells)
    const bool wide = c->solve_wide_px > 0 && (int64_t)H * W >= c->solve_wide_px;
    return counted(c, hr::launch_solve(a, nb, hist_done ? 2 : cpsm ? cpsm : solve_cpsm_for(c, nb), s, max_ctas, wide));
  };
  auto apply_chunk = [&](int64_t b0, int64_t nb, cudaStream_t s, const uint32_t* ready = nullptr) -> cudaError_t {
    return counted(c, hr::launch_apply(in + b0 * img, lut + b0 * kLevels, nb, H, W, out + b0 * img, apply_grid(c), s,
                                       c->warp_solver ? nullptr : ready));
  };
  // persistent fused kernel: hist -> per-image solve + LUT -> apply, solves overlapped
  const int64_t fmax = c->fused_max_b > 0 ? c->fused_max_b : std::max(1, c->num_sms / 2);
  if (c->fused_min_b > 0 && B >= c->fused_min_b && B <= fmax && hr::fused_supported(in, out, B, H, W)) {
    uint32_t* ctl = reinterpret_cast<uint32_t*>((char*)ws + L.ctl);
    if (e == cudaSuccess && hs != reinterpret_cast<uint32_t*>((char*)ws + L.hist_s))
      e = counted(c, hr::launch_zero(hs, (size_t)B * kLevels * sizeof(uint32_t), st));
    const size_t z0 = hs == reinterpret_cast<uint32_t*>((char*)ws + L.hist_s) ? L.hist_s : L.graw;
    if (e == cudaSuccess) e = mark(0);
    if (e == cudaSuccess) e = counted(c, hr::launch_zero((char*)ws + z0, align_up(L.ctl + hr::fused_ctl_bytes(B)) - z0, st));
    if (e == cudaSuccess) e = mark(1);
    hr::FusedArgs f{};
    f.in = in;
    f.out = out;
    f.B = B;
    f.H = H;
    f.W = W;
    f.hist_s = hs;
    f.graw = graw;
    f.ctl = ctl;
    f.sa.hist_s = hs;
    f.sa.graw = graw;
    f.sa.grad_norm = p->grad_norm;
    f.sa.p = *p;
    f.sa.iters = iters_dbg;
    f.sa.lut = lut;
    f.sa.cells_ws = cells;
    f.sa.idx1_tab = tab;
    const int grid = c->fused_cpsm * c->num_sms;
    const int64_t kb = (c->fused_bands * (int64_t)grid + B - 1) / B;
    f.KB = (int32_t)std::max<int64_t>(1, std::min<int64_t>(kb, std::max(1, H / 16)));
    f.GS = (uint32_t)c->fused_gs;
    if (e == cudaSuccess) e = counted(c, hr::launch_fused(f, grid, st));
    c->last_path = 1;
    if (e == cudaSuccess) e = mark(2);
    if (e == cudaSuccess) e = mark(3);
    return cuda_err(c, e, "hr_enhance");
  }
  // grouped step: images in G groups; one stream, every kernel launched early (programmatic
  // dependent launch):  zero | hist(0) | solve(0) | hist(1) | solve(1) | ... | solve(G-1) | apply.
  // No kernel after hist(0) waits for its predecessor grid (griddepcontrol.wait waits for
  // everything earlier in the stream, which would serialise the solves): hist(k), k >= 1, shares
  // no data with solve(k-1), so the streaming pass runs on the slots the earlier solves leave
  // free; each solver CTA acquires its image's flushed-row count (all H rows: histograms
  // complete); the apply acquires each image's LUT-ready flag and takes every CTA's share
  // of groups 0..G-2 before its share of group G-1, so it overlaps the last solves.  The
  // streaming grids are sized to the slots left beside the resident solver CTAs (a solver CTA
  // takes one streaming CTA's registers).
  const bool ready_ok = [] {
    const char* v = getenv("HR_READY");
    return !(v && atoi(v) == 0);
  }();
  // groups < 0 (default): 2 groups for every batch (B >= 2), split by group_first_pct: C3 0.255
  // vs 0.270 ms ungrouped, C5 0.167 vs 0.177 (equal halves were slower on C5: 0.193)
  const int ngroups = c->groups >= 0 ? c->groups : (B >= 2 ? 2 : 0);
  if (ngroups >= 2 && B >= 2 && !c->warp_solver && ready_ok) {
    const int64_t G = std::min<int64_t>(ngroups, B);
    uint32_t* ctl = reinterpret_cast<uint32_t*>((char*)ws + L.ctl);
    uint32_t* done = ctl + hr::kCtlHeader;  // rows flushed per image (k_hist -> k_solve)
    uint32_t* ready = ctl + hr::kCtlHeader + B;
    c->last_path = 3;
    if (e == cudaSuccess) e = mark(0);
    if (e == cudaSuccess) e = counted(c, hr::launch_zero(hs, (size_t)B * kLevels * sizeof(uint32_t), st));
    if (e == cudaSuccess) e = counted(c, hr::launch_zero(graw, (size_t)B * kGradSlots * sizeof(uint32_t), st));
    if (e == cudaSuccess) e = counted(c, hr::launch_zero((char*)ws + L.ctl, align_up(hr::fused_ctl_bytes(B)), st));
    if (e == cudaSuccess) e = mark(1);
    // group boundaries: equal groups, or (G = 2) a first group of group_first_pct % of the images
    auto gstart = [&](int64_t k) -> int64_t {
      if (k <= 0) return 0;
      if (k >= G) return B;
      const int pct = c->group_first_pct >= 0 ? c->group_first_pct : (B <= c->num_sms / 2 ? 38 : 90);
      if (G == 2 && pct > 0) return std::min<int64_t>(B - 1, std::max<int64_t>(1, (B * pct + 50) / 100));
      return B * k / G;
    };
    const int slots = hist_grid(c);
    int64_t prev_nb = 0;
    for (int64_t k = 0; k < G && e == cudaSuccess; ++k) {
      const int64_t b0 = gstart(k), nb = gstart(k + 1) - b0;
      const int grid = (int)std::max<int64_t>(c->num_sms, slots - std::min<int64_t>(prev_nb, slots / 2));
      // histogram-completion queue of this group (solver CTAs take images in the order they complete)
      uint32_t* cq = c->solve_queue ? ctl + hr::kCtlHeader + 3 * B + b0 : nullptr;
      uint32_t* cqc = ctl + hr::kCtlHeader + 4 * B + 2 * k;  // [0] tail, [1] head
      e = counted(c, hr::launch_hist(in + b0 * img, nb, H, W, hs + b0 * kLevels, graw + b0 * kGradSlots, grid, st,
                                     hr::kHistThreads, done + b0, 0, k > 0, cq, cq ? cqc : nullptr));
      if (e == cudaSuccess)
        e = solve_chunk(b0, nb, st, ready + b0, done + b0, 0, nullptr, nullptr, 2, 0, cq, cq ? cqc + 1 : nullptr);
      prev_nb = nb;
    }
    if (e == cudaSuccess) e = mark(2);
    static const int ag_sub = [] {  // measurement switch: apply slots given up per last-group solve
      const char* v = getenv("HR_GROUP_AG_SUB");
      return v ? atoi(v) : 1;
    }();
    const int ag = (int)std::max<int64_t>(c->num_sms, apply_grid(c) - std::min<int64_t>(ag_sub * prev_nb, apply_grid(c) / 2));
    const int64_t b_last = gstart(G - 1);
    if (e == cudaSuccess)
      e = c->group_apply == 1 && hr::apply_dyn_supported(in, out, B, H, W)
              ? counted(c, hr::launch_apply_dyn(in, lut, B, H, W, out, ag, nullptr, ctl + 3, c->apply_gs, st, ready,
                                                b_last))
              : counted(c, hr::launch_apply(in, lut, B, H, W, out, ag, st, ready, b_last,
                                            c->group_apply == 2 ? ctl + 3 : nullptr, c->apply_gs, c->apply_tail_pct));
    if (e == cudaSuccess) e = mark(3);
    return cuda_err(c, e, "hr_enhance");
  }
  const int K = (int)std::min<int64_t>(c->chunks, B);
  c->last_path = K <= 1 ? 0 : 2;
  if (K <= 1) {  // serial on the caller's stream (stage-timed: hist | solve + LUT | apply)
    // per-image LUT-ready flags (in the zeroed control block) let the apply grid, launched
    // early under PDL, start on images whose LUT is done while the solver grid finishes
    static const bool use_ready = [] {
      const char* v = getenv("HR_READY");
      return !(v && atoi(v) == 0);
    }();
    uint32_t* ready = use_ready ? reinterpret_cast<uint32_t*>((char*)ws + L.ctl) + hr::kCtlHeader + B : nullptr;
    const bool own_hs = hs == reinterpret_cast<uint32_t*>((char*)ws + L.hist_s);
    const size_t z0 = own_hs ? L.hist_s : L.graw;
    // zeroing as separate launches per region: measured faster in the PDL chain than one launch
    // over [hist_s | graw | ctl] (C5 0.165 vs 0.174 ms; HR_ZERO2=0 selects the single launch)
    static const bool zero2 = [] {
      const char* v = getenv("HR_ZERO2");
      return !(v && atoi(v) == 0);
    }();
    if (e == cudaSuccess) e = mark(0);
    if (zero2) {
      if (e == cudaSuccess) e = counted(c, hr::launch_zero(hs, (size_t)B * kLevels * sizeof(uint32_t), st));
      if (e == cudaSuccess) e = counted(c, hr::launch_zero(graw, (size_t)B * kGradSlots * sizeof(uint32_t), st));
      if (e == cudaSuccess && ready)  // the whole (256-B aligned) control block holding ready[]
        e = counted(c, hr::launch_zero((char*)ws + L.ctl, align_up(hr::fused_ctl_bytes(B)), st));
    } else {
      if (e == cudaSuccess && !own_hs) e = counted(c, hr::launch_zero(hs, (size_t)B * kLevels * sizeof(uint32_t), st));
      if (e == cudaSuccess)
        e = counted(c, hr::launch_zero((char*)ws + z0, align_up(L.ctl + hr::fused_ctl_bytes(B)) - z0, st));
    }
    // histograms counting flushed rows per image (TMA-staged kernel in image waves, 512 threads
    // per SM; else the direct-load kernel at 2 x 256 threads per SM): each solver CTA, resident
    // beside them, starts once its image is complete (needs the zeroed control block)
    const bool overlap = c->hist_overlap && ready && !c->warp_solver;
    uint32_t* ctl = reinterpret_cast<uint32_t*>((char*)ws + L.ctl);
    const int HG = hr::hist_grid_clamped(B, H, 2 * c->num_sms);
    if (e == cudaSuccess)
      e = overlap ? counted(c, hr::launch_hist(in, B, H, W, hs, graw, HG, st, 256, ctl + hr::kCtlHeader, c->hist_tma))
                  : counted(c, hr::launch_hist(in, B, H, W, hs, graw, hist_grid(c), st, hr::kHistThreads, nullptr, c->hist_tma));
    if (e == cudaSuccess) e = mark(1);
    // completion-order apply: k_solve appends each finished image to a queue in the control block
    const bool dyn = c->apply_dyn && ready && !c->warp_solver && hr::apply_dyn_supported(in, out, B, H, W);
    uint32_t* queue = dyn && c->apply_dyn == 1 ? ctl + hr::kCtlHeader + 2 * B : nullptr;
    // solve waves (B > #SMs): one solver CTA per SM solving its images in turn (the first wave's
    // LUTs complete early), the apply at one CTA per SM beside it, every apply CTA taking its share
    // of the first wave's images first
    const bool waves = c->solve_waves && ready && !overlap && !dyn && B > c->num_sms;
    if (e == cudaSuccess)
      e = solve_chunk(0, B, st, ready, overlap ? ctl + hr::kCtlHeader : nullptr, overlap ? HG : 0, queue,
                      queue ? ctl + 2 : nullptr, waves ? 2 : 0, waves ? c->num_sms : 0);
    if (e == cudaSuccess) e = mark(2);
    if (e == cudaSuccess)
      e = dyn ? counted(c, hr::launch_apply_dyn(in, lut, B, H, W, out, apply_grid(c), queue, ctl + 3, c->apply_gs, st,
                                                c->apply_dyn == 3 ? ready : nullptr, c->apply_dyn == 3 ? B / 2 : 0))
              : waves ? counted(c, hr::launch_apply(in, lut, B, H, W, out, c->solve_waves_ag * c->num_sms, st, ready,
                                                    c->num_sms))
                      : apply_chunk(0, B, st, ready);
    if (e == cudaSuccess) e = mark(3);
    return cuda_err(c, e, "hr_enhance");
  }
  // fork/join pipeline: solve(c) overlaps hist(c+1) and apply(c-1)
  if (!c->sH) {
    for (cudaStream_t* q : {&c->sH, &c->sS, &c->sA})
      if (e == cudaSuccess) e = cudaStreamCreateWithFlags(q, cudaStreamNonBlocking);
  }
  while (e == cudaSuccess && (int)c->pev.size() < 2 * K + 4) {
    cudaEvent_t x;
    e = cudaEventCreateWithFlags(&x, cudaEventDisableTiming);
    if (e == cudaSuccess) c->pev.push_back(x);
  }
  cudaEvent_t* E = c->pev.data();  // [0] fork, [1..3] joins, [4..4+K) hist done, [4+K..4+2K) solve done
  // stage-timed: the whole pipeline is one stage (stage_ms = [0, 0, total])
  if (e == cudaSuccess) e = mark(0);
  if (e == cudaSuccess) e = mark(1);
  if (e == cudaSuccess) e = mark(2);
  if (e == cudaSuccess) e = cudaEventRecord(E[0], st);
  for (cudaStream_t q : {c->sH, c->sS, c->sA})
    if (e == cudaSuccess) e = cudaStreamWaitEvent(q, E[0], 0);
  for (int k = 0; k < K && e == cudaSuccess; ++k) {
    const int64_t b0 = B * k / K, nb = B * (k + 1) / K - b0;
    e = hist_chunk(b0, nb, c->sH);
    if (e == cudaSuccess) e = cudaEventRecord(E[4 + k], c->sH);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(c->sS, E[4 + k], 0);
    if (e == cudaSuccess) e = solve_chunk(b0, nb, c->sS);
    if (e == cudaSuccess) e = cudaEventRecord(E[4 + K + k], c->sS);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(c->sA, E[4 + K + k], 0);
    if (e == cudaSuccess) e = apply_chunk(b0, nb, c->sA);
  }
  int j = 1;
  for (cudaStream_t q : {c->sH, c->sS, c->sA}) {
    if (e == cudaSuccess) e = cudaEventRecord(E[j], q);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, E[j], 0);
    ++j;
  }
  if (e == cudaSuccess) e = mark(3);
  return cuda_err(c, e, "hr_enhance");
}

hr_status hr_enhance(hr_ctx* c, const uint8_t* in, int64_t B, int32_t H, int32_t W, const hr_params* p,
                     uint8_t* out, void* ws, void* stream) {
  return hr_enhance_debug(c, in, B, H, W, p, out, ws, nullptr, nullptr, nullptr, stream);
}

hr_status hr_he(hr_ctx* c, const uint8_t* in, int64_t B, int32_t H, int32_t W, uint8_t* out, uint8_t* lut_dbg,
                void* ws, void* stream) {
  if (!c) return HR_EINVAL;
  hr_status s = check_shape(c, B, H, W);
  if (s) return s;
  if (!in || !out || !ws) return set_err(c, HR_EINVAL, "NULL pointer");
  if (in == out) return set_err(c, HR_EINVAL, "rgb_out must not alias rgb_in");
  if ((s = activate(c))) return s;
  cudaStream_t st = (cudaStream_t)stream;
  const WsLayout L = ws_layout(B);
  uint32_t* hs = reinterpret_cast<uint32_t*>((char*)ws + L.hist_s);
  uint32_t* graw = reinterpret_cast<uint32_t*>((char*)ws + L.graw);
  uint8_t* lut = lut_dbg ? lut_dbg : reinterpret_cast<uint8_t*>((char*)ws + L.lut);
  cudaError_t e = counted(c, hr::launch_zero(hs, (size_t)B * kLevels * sizeof(uint32_t), st));
  if (e == cudaSuccess) e = counted(c, hr::launch_zero(graw, (size_t)B * kGradSlots * sizeof(uint32_t), st));
  if (e == cudaSuccess) e = counted(c, hr::launch_hist(in, B, H, W, hs, graw, hist_grid(c), st, hr::kHistThreads, nullptr, c->hist_tma));
  if (e == cudaSuccess) e = counted(c, hr::launch_he_lut(hs, B, lut, st));
  if (e == cudaSuccess) e = counted(c, hr::launch_apply(in, lut, B, H, W, out, apply_grid(c), st));
  return cuda_err(c, e, "hr_he");
}

size_t hr_quality_workspace_bytes(int64_t B, int32_t H, int32_t W) {
  if (B <= 0 || H <= 0 || W <= 0) return 0;
  return hr::quality_ws_bytes(B, H, W);
}

hr_status hr_quality(hr_ctx* c, const uint8_t* a, const uint8_t* b, int64_t B, int32_t H, int32_t W, double* psnr,
                     double* ssim, double* loe, void* ws, void* stream) {
  if (!c) return HR_EINVAL;
  hr_status s = check_shape(c, B, H, W);
  if (s) return s;
  if (!a || !b || !ws) return set_err(c, HR_EINVAL, "NULL pointer");
  if (!psnr && !ssim && !loe) return set_err(c, HR_EINVAL, "no metric requested");
  if ((s = activate(c))) return s;
  return cuda_err(c, hr::launch_quality(a, b, B, H, W, psnr, ssim, loe, ws, (cudaStream_t)stream), "hr_quality");
}

hr_status hr_enhance_host(hr_ctx* c, const uint8_t* in_h, int64_t B, int32_t H, int32_t W, const hr_params* p,
                          uint8_t* out_h, uint8_t* in_d, uint8_t* out_d, void* ws, int32_t chunks, void* stream) {
  if (!c) return HR_EINVAL;
  hr_status s = check_shape(c, B, H, W);
  if (s) return s;
  if ((s = check_params(c, p))) return s;
  if (!in_h || !out_h || !in_d || !out_d || !ws) return set_err(c, HR_EINVAL, "NULL pointer");
  if (in_h == out_h || in_d == out_d) return set_err(c, HR_EINVAL, "output must not alias input");
  if (chunks < 0) return set_err(c, HR_EINVAL, "chunks must be >= 0");
  if ((s = activate(c))) return s;
  const int K = (int)std::min<int64_t>(chunks > 0 ? chunks : 8, B);
  const size_t img = (size_t)H * W * 3;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaSuccess;
  if (!c->sIn) e = cudaStreamCreateWithFlags(&c->sIn, cudaStreamNonBlocking);
  if (e == cudaSuccess && !c->sOut) e = cudaStreamCreateWithFlags(&c->sOut, cudaStreamNonBlocking);
  while (e == cudaSuccess && (int)c->hev.size() < 2 * K + 2) {
    cudaEvent_t x;
    e = cudaEventCreateWithFlags(&x, cudaEventDisableTiming);
    if (e == cudaSuccess) c->hev.push_back(x);
  }
  if (e != cudaSuccess) return cuda_err(c, e, "hr_enhance_host");
  cudaEvent_t* E = c->hev.data();  // [0] fork, [1] join, [2, 2+K) copied in, [2+K, 2+2K) enhanced
  e = cudaEventRecord(E[0], st);  // everything earlier on `stream` (incl. the previous call) first
  if (e == cudaSuccess) e = cudaStreamWaitEvent(c->sIn, E[0], 0);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(c->sOut, E[0], 0);
  for (int k = 0; k < K && e == cudaSuccess; ++k) {  // all host->device copies, in order
    const int64_t b0 = B * k / K, nb = B * (k + 1) / K - b0;
    e = cudaMemcpyAsync(in_d + b0 * img, in_h + b0 * img, nb * img, cudaMemcpyHostToDevice, c->sIn);
    if (e == cudaSuccess) e = cudaEventRecord(E[2 + k], c->sIn);
  }
  for (int k = 0; k < K && e == cudaSuccess; ++k) {  // enhance chunk k once it is in, then copy it out
    const int64_t b0 = B * k / K, nb = B * (k + 1) / K - b0;
    e = cudaStreamWaitEvent(st, E[2 + k], 0);
    if (e != cudaSuccess) break;
    const hr_status r = hr_enhance_debug(c, in_d + b0 * img, nb, H, W, p, out_d + b0 * img, ws, nullptr, nullptr,
                                         nullptr, stream);
    if (r != HR_OK) return r;
    e = cudaEventRecord(E[2 + K + k], st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(c->sOut, E[2 + K + k], 0);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(out_h + b0 * img, out_d + b0 * img, nb * img, cudaMemcpyDeviceToHost, c->sOut);
  }
  if (e == cudaSuccess) e = cudaEventRecord(E[1], c->sOut);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(st, E[1], 0);
  return cuda_err(c, e, "hr_enhance_host");
}

}  // extern "C"

#ifdef HR_STEP_TRACE
// measurement-only (tools/step_trace.py; not part of histretinex.h): bind the step-timeline buffer
extern "C" int hr_debug_trace_bind(void* buf, uint32_t* n, uint32_t cap) {
  hr::trace_bind_hist(buf, n, cap);
  hr::trace_bind_solve(buf, n, cap);
  hr::trace_bind_apply(buf, n, cap);
  return (int)cudaGetLastError();
}
#endif
