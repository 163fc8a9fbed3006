// hr_api.cu -- the C-ABI boundary (include/histretinex.h): validation, context, launches.
//
// Every entry point validates synchronously and enqueues nothing on error.  No exception
// or exit() crosses the boundary.
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <mutex>
#include <new>
#include <vector>

#include "hr_common.cuh"

struct hr_ctx {
  int device = 0;
  int num_sms = 148;
  int l2_bytes = 0;
  char last_error[512] = {0};
  // index_1 tables of Eqs. 17-19, one per gamma (64 KB each).  Built on first use on a private
  // stream and synchronised before use (so any stream may read them); a slot is reused (after
  // kTab distinct gammas) only after its last-use event -- recorded after every launch that
  // reads it -- has completed.
  static constexpr int kTab = 64;
  uint8_t* idx1_tab[kTab] = {};
  double idx1_gamma[kTab] = {};
  bool idx1_valid[kTab] = {};
  cudaEvent_t idx1_used[kTab] = {};
  int idx1_next = 0;
  cudaStream_t sTab = nullptr;
  // execution policy of hr_enhance (performance only; defaults chosen from B200 measurements;
  // HR_<KEY> environment variables override them at hr_create)
  int hist_cpsm = 2;        // k_hist CTAs per SM
  int apply_cpsm = 2;       // k_apply CTAs per SM
  int solve_cpsm = 0;       // k_solve CTAs per SM: 1, 2, or 0 = auto (1 when B <= SMs)
  int solve_wide_px = 4 << 20;  // one-CTA-per-SM solves: 512-thread CTAs for H*W >= this (0: never)
  int groups = -1;          // grouped step (>= 2): histograms of group k+1 run beside the solves of
                            // group k, the apply beside the last group's solves (0/1: off; -1: auto
                            // = 2 when B >= 2)
  int group_first_pct = -1; // grouped step, G = 2: first group's share of the images in % (0: equal
                            // groups; -1: auto = 47 for B <= SMs / 2 -- solve(0) hides under hist(1)
                            // and the last group stays the larger one (the apply then takes every
                            // slot): C3 30 + 34 images 0.2332 ms, 24 + 40 0.2370, 32 + 32 0.2436 --
                            // and 90 for larger batches -- the last group's few solves
                            // overlap the first group's apply, C5 230 + 26 images 0.167 vs 0.177)
  int apply_gs = 8;         // grouped step's apply: 1024-px chunks per warp in a CTA ticket
  int apply_full_grid = -1; // grouped step's apply grid: 1 every slot, 0 the slots the last group's
                            // solvers leave, -1 auto (every slot when the last group is the larger)
  int solve_cluster = 1;    // large images (H*W >= solve_wide_px, <= 9 per launch, separate kernels):
                            // one cluster per image (solve_cluster_dev.cuh): 1 = 8 CTAs x 256
                            // threads (C4 solve 119 -> 77 us), 2 = 8 x 512 (88), 3 = 16 x 256
                            // (88), 4 = 16 x 512 (113); 0: one 512-thread CTA
  int graph_b1 = 1;         // hr_enhance of one image: replay a cached CUDA graph of the step
                            // (C1 0.0629 -> 0.0614 ms, C2 0.0777 -> 0.0757, C4 0.2063 -> 0.2048;
                            // batches lose the PDL overlap between consecutive steps, so B >= 2
                            // launches directly: C3 0.2490 vs 0.2507, C5 0.1625 vs 0.1643)
  // cached single-image step graphs, keyed by every argument of the call (LRU)
  struct GraphEntry {
    const uint8_t* in;
    uint8_t* out;
    void* ws;
    cudaStream_t st;
    int32_t H, W;
    hr_params p;
    cudaGraphExec_t exec;
    int slot;         // the index_1 table slot the graph reads
    int64_t kernels;  // kernels one replay launches (hr_kernel_launches)
    uint64_t used;
  };
  static constexpr int kGraphs = 8;
  GraphEntry graphs[kGraphs] = {};
  uint64_t graph_clock = 0;
  int64_t launches = 0;     // kernels launched through this context (hr_kernel_launches)
  int last_path = -1;       // hr_last_path: 0 separate kernels, 3 grouped step
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

// count a successful kernel launch (HR_SYNC_CHECK=1, debugging: synchronise after every launch
// and report which launch faulted)
const char* g_launch_label = "";
inline cudaError_t counted(hr_ctx* c, cudaError_t e) {
  if (e == cudaSuccess) ++c->launches;
  static const bool sync_check = [] {
    const char* v = getenv("HR_SYNC_CHECK");
    return v && atoi(v) != 0;
  }();
  if (sync_check && e == cudaSuccess) {
    e = cudaDeviceSynchronize();
    if (e != cudaSuccess) fprintf(stderr, "HR_SYNC_CHECK: launch #%lld (%s) faulted: %s\n", (long long)c->launches, g_launch_label, cudaGetErrorString(e));
  }
  return e;
}

struct WsLayout {
  size_t hist_s, graw, ctl, lut, iters, target, cells, total;
};

WsLayout ws_layout(int64_t B) {
  WsLayout L;
  size_t o = 0;
  L.hist_s = o;
  o = align_up(o + (size_t)B * kLevels * sizeof(uint32_t));
  L.graw = o;
  o = align_up(o + (size_t)B * kGradSlots * sizeof(uint32_t));
  L.ctl = o;  // control block (done[], ready[], ticket)
  o = align_up(o + hr::ctl_bytes(B));
  L.lut = o;
  o = align_up(o + (size_t)B * kLevels);
  L.iters = o;
  o = align_up(o + (size_t)B * sizeof(int32_t));
  L.target = o;
  o = align_up(o + (size_t)B * kLevels * sizeof(double));
  L.cells = o;
  o = align_up(o + hr::solve_cells_ws_bytes(B));
  L.total = o;
  return L;
}

// kernel attributes once per device (cudaFuncSetAttribute applies to the current device only)
constexpr int kMaxDevices = 64;
std::once_flag g_attr_once[kMaxDevices];
cudaError_t g_attr_err[kMaxDevices];
cudaError_t init_kernel_attrs(int device) {
  if (device < 0 || device >= kMaxDevices) return cudaErrorInvalidDevice;
  std::call_once(g_attr_once[device], [device] {
    int cur = -1;
    cudaError_t e = cudaGetDevice(&cur);
    if (e == cudaSuccess && cur != device) e = cudaSetDevice(device);
    if (e == cudaSuccess) e = hr::init_attrs_hist();
    if (e == cudaSuccess) e = hr::init_attrs_solve();
    if (e == cudaSuccess) e = hr::init_attrs_apply();
    if (cur >= 0 && cur != device) cudaSetDevice(cur);
    g_attr_err[device] = e;
  });
  return g_attr_err[device];
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
  // uint32 histogram bins: a constant image of 2^32 pixels would wrap its bin to 0
  if (B > (1 << 30) || (int64_t)H * W >= (int64_t)1 << 32) return set_err(c, HR_EINVAL, "size too large");
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
int hist_nt(const hr_ctx* c) { return c->hist_cpsm == 1 ? 1024 : hr::kHistThreads; }  // 1 CTA/SM: 1024 threads
int apply_grid(const hr_ctx* c) { return c->apply_cpsm * c->num_sms; }
int solve_cpsm_for(const hr_ctx* c, int64_t B) { return c->solve_cpsm ? c->solve_cpsm : (B <= c->num_sms ? 1 : 2); }

// index_1 table for gamma (slot *slot): cached, or built now on the context's table stream and
// synchronised (the first call with a new gamma blocks the host for one small kernel)
cudaError_t idx1_table(hr_ctx* c, double gamma, const uint8_t** out, int* slot) {
  for (int i = 0; i < hr_ctx::kTab; ++i)
    if (c->idx1_valid[i] && c->idx1_gamma[i] == gamma) {
      *out = c->idx1_tab[i];
      *slot = i;
      return cudaSuccess;
    }
  const int i = c->idx1_next;
  cudaError_t e = cudaSuccess;
  if (c->idx1_valid[i]) e = cudaEventSynchronize(c->idx1_used[i]);  // in-flight readers are done
  for (auto& g : c->graphs)  // cached step graphs that read this slot
    if (g.exec && g.slot == i) {
      cudaGraphExecDestroy(g.exec);
      g = hr_ctx::GraphEntry{};
    }
  if (e == cudaSuccess && !c->idx1_tab[i]) e = cudaMalloc(&c->idx1_tab[i], 256 * 256);
  if (e == cudaSuccess && !c->idx1_used[i]) e = cudaEventCreateWithFlags(&c->idx1_used[i], cudaEventDisableTiming);
  if (e == cudaSuccess && !c->sTab) e = cudaStreamCreateWithFlags(&c->sTab, cudaStreamNonBlocking);
  if (e != cudaSuccess) return e;
  c->idx1_valid[i] = false;
  e = hr::launch_idx1_table(gamma, c->idx1_tab[i], c->sTab);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->sTab);
  if (e != cudaSuccess) return e;
  ++c->launches;
  c->idx1_gamma[i] = gamma;
  c->idx1_valid[i] = true;
  c->idx1_next = (i + 1) % hr_ctx::kTab;
  *out = c->idx1_tab[i];
  *slot = i;
  return cudaSuccess;
}
// after the launches that read table `slot` on `st` (skipped while `st` is being captured
// into a graph: a captured graph keeps reading the table, which stays cached for the ctx)
cudaError_t idx1_mark_used(hr_ctx* c, int slot, cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaError_t e = cudaStreamIsCapturing(st, &cs);
  if (e != cudaSuccess || cs != cudaStreamCaptureStatusNone) return e;
  return cudaEventRecord(c->idx1_used[slot], st);
}

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
  if (init_kernel_attrs(device) != cudaSuccess) {
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
  auto env = [](const char* k, int& field, int lo, int hi) {
    if (const char* v = getenv(k)) {
      const int x = atoi(v);
      if (x >= lo && x <= hi) field = x;
    }
  };
  env("HR_HIST_CPSM", c->hist_cpsm, 1, 2);
  env("HR_APPLY_CPSM", c->apply_cpsm, 1, 2);
  env("HR_SOLVE_CPSM", c->solve_cpsm, 0, 2);
  env("HR_SOLVE_WIDE_PX", c->solve_wide_px, 0, 1 << 30);
  env("HR_GROUPS", c->groups, -1, 64);
  env("HR_GROUP_FIRST_PCT", c->group_first_pct, -1, 99);
  env("HR_APPLY_GS", c->apply_gs, 1, 1 << 20);
  env("HR_APPLY_FULL_GRID", c->apply_full_grid, -1, 1);
  env("HR_GRAPH_B1", c->graph_b1, 0, 1);
  env("HR_SOLVE_CLUSTER", c->solve_cluster, 0, 4);
  *out = c;
  return HR_OK;
}

hr_status hr_destroy(hr_ctx* c) {
  if (c) {
    for (cudaEvent_t e : c->prof_ev) cudaEventDestroy(e);
    for (cudaEvent_t e : c->hev) cudaEventDestroy(e);
    for (auto& g : c->graphs)
      if (g.exec) cudaGraphExecDestroy(g.exec);
    if (c->sIn) cudaStreamDestroy(c->sIn);
    if (c->sOut) cudaStreamDestroy(c->sOut);
    for (int i = 0; i < hr_ctx::kTab; ++i) {
      if (c->idx1_used[i]) {
        cudaEventSynchronize(c->idx1_used[i]);
        cudaEventDestroy(c->idx1_used[i]);
      }
      if (c->idx1_tab[i]) cudaFree(c->idx1_tab[i]);
    }
    if (c->sTab) cudaStreamDestroy(c->sTab);
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
      {"hist_cpsm", &c->hist_cpsm, 1, 2},          {"apply_cpsm", &c->apply_cpsm, 1, 2},
      {"solve_cpsm", &c->solve_cpsm, 0, 2},        {"solve_wide_px", &c->solve_wide_px, 0, 1 << 30},
      {"groups", &c->groups, -1, 64},              {"group_first_pct", &c->group_first_pct, -1, 99},
      {"apply_gs", &c->apply_gs, 1, 1 << 20},      {"graph_b1", &c->graph_b1, 0, 1},
      {"apply_full_grid", &c->apply_full_grid, -1, 1},
      {"solve_cluster", &c->solve_cluster, 0, 4},
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
  if (e == cudaSuccess) e = counted(c, hr::launch_hist(rgb, B, H, W, hist_s, graw, hist_grid(c), st, nullptr, false, hist_nt(c)));
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
  int slot = 0;
  {
    cudaError_t e = idx1_table(c, p->gamma, &a.idx1_tab, &slot);
    if (e != cudaSuccess) return cuda_err(c, e, "hr_solve (index_1 table)");
  }
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
  cudaError_t e = counted(c, hr::launch_solve(a, B, solve_cpsm_for(c, B), (cudaStream_t)stream));
  if (e == cudaSuccess) e = idx1_mark_used(c, slot, (cudaStream_t)stream);
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
                           uint8_t* out, void* ws, const hr_debug_out* dbg, void* stream) {
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
  const hr_debug_out none{};
  const hr_debug_out& D = dbg ? *dbg : none;
  uint32_t* hs = D.hist_s ? D.hist_s : reinterpret_cast<uint32_t*>((char*)ws + L.hist_s);
  uint32_t* graw = reinterpret_cast<uint32_t*>((char*)ws + L.graw);
  uint32_t* ctl = reinterpret_cast<uint32_t*>((char*)ws + L.ctl);
  uint32_t* done = ctl + hr::kCtlHeader;  // rows flushed per image (k_hist -> k_solve)
  uint32_t* ready = done + B;             // LUT written per image (k_solve -> k_apply)
  uint8_t* lut = D.lut ? D.lut : reinterpret_cast<uint8_t*>((char*)ws + L.lut);
  unsigned char* cells = reinterpret_cast<unsigned char*>((char*)ws + L.cells);
  const uint8_t* tab = nullptr;
  int slot = 0;
  cudaError_t e = idx1_table(c, p->gamma, &tab, &slot);
  const size_t img = (size_t)H * W * 3;
  // solves of images [b0, b0 + nb): per-image LUT-ready flags; with wait_done each CTA first
  // acquires its image's flushed-row count instead of waiting for the grid before it
  auto solve_group = [&](int64_t b0, int64_t nb, int cpsm, bool wait_done) -> cudaError_t {
    hr::SolveArgs a{};
    a.ready = ready + b0;
    a.hist_done = wait_done ? done + b0 : nullptr;
    a.hist_H = H;
    // grouped step: a solver CTA runs beside histogram CTAs, so its shared run arena is smaller
    // (runs that do not fit go to the global arena)
    a.arena_bytes = wait_done ? 40 * 1024 : 0;
    a.idx1_tab = tab;
    a.hist_s = hs + b0 * kLevels;
    a.hist_g = nullptr;
    a.graw = graw + b0 * kGradSlots;
    a.grad_norm = p->grad_norm;
    a.p = *p;
    a.iters = D.iters ? D.iters + b0 : nullptr;
    a.hist_g_out = D.hist_g ? D.hist_g + b0 * kLevels : nullptr;
    a.hL = D.hL ? D.hL + b0 * kLevels : nullptr;
    a.hR = D.hR ? D.hR + b0 * kLevels : nullptr;
    a.target = D.target ? D.target + b0 * kLevels : nullptr;
    a.lut = lut + b0 * kLevels;  // CDF + LUT tail fused into the solver CTA (no target round trip)
    a.cells_ws = cells + (size_t)b0 * hr::solve_cells_ws_bytes(1);
    // 512-thread solver CTAs for large images (their supports, and so the cell loops, tend to be
    // large: C4 33 MP 8,480 cells; C2 0.66 MP 1,334 cells)
    const bool wide = c->solve_wide_px > 0 && (int64_t)H * W >= c->solve_wide_px;
    if (wide && c->solve_cluster && nb <= hr::kClusterMaxB && !wait_done) {
      g_launch_label = "solve_cluster";
      return counted(c, hr::launch_solve_cluster(a, nb, st, c->solve_cluster));
    }
    g_launch_label = "solve";
    return counted(c, hr::launch_solve(a, nb, cpsm, st, wide));
  };
  auto zero = [&](void* q, size_t n) -> cudaError_t {
    g_launch_label = "zero";
    return counted(c, hr::launch_zero(q, n, st));
  };
  const int ngroups = c->groups >= 0 ? c->groups : (B >= 2 ? 2 : 0);
  if (e == cudaSuccess) e = mark(0);
  // the accumulators and the control block are contiguous in the workspace: one zeroing launch
  // (three launches, one per region, were 2 us slower per step: C1 0.0570 vs 0.0551 ms, C3 0.2328
  // vs 0.2310, C5 0.1531 vs 0.1509)
  if (D.hist_s) {  // hr_enhance_debug with the caller's hist_s buffer: that one on its own
    if (e == cudaSuccess) e = zero(hs, (size_t)B * kLevels * sizeof(uint32_t));
    if (e == cudaSuccess) e = zero(graw, (size_t)(L.ctl - L.graw) + align_up(hr::ctl_bytes(B)));
  } else if (e == cudaSuccess) {
    e = zero(hs, (size_t)(L.ctl - L.hist_s) + align_up(hr::ctl_bytes(B)));
  }
  if (ngroups >= 2 && B >= 2) {
    // grouped step: images in G groups; one stream, every kernel launched early (programmatic
    // dependent launch):  zero | hist(0) | solve(0) | hist(1) | solve(1) | ... | solve(G-1) | apply.
    // No kernel after hist(0) waits for its predecessor grid (griddepcontrol.wait waits for
    // everything earlier in the stream, which would serialise the solves): hist(k), k >= 1, shares
    // no data with solve(k-1), so the streaming pass runs on the slots the earlier solves leave
    // free; each solver CTA acquires its image's flushed-row count (all H rows: histograms
    // complete); the apply acquires each image's LUT-ready flag and takes every CTA's share of
    // groups 0..G-2 before the last group, by CTA tickets, so it overlaps the last solves.  The
    // streaming grids are sized to the slots left beside the resident solver CTAs (a solver CTA
    // takes one streaming CTA's registers).
    const int64_t G = std::min<int64_t>(ngroups, B);
    c->last_path = 3;
    if (e == cudaSuccess) e = mark(1);
    // group boundaries: equal groups, or (G = 2) a first group of group_first_pct % of the images
    auto gstart = [&](int64_t k) -> int64_t {
      if (k <= 0) return 0;
      if (k >= G) return B;
      const int pct = c->group_first_pct >= 0 ? c->group_first_pct : (B <= c->num_sms / 2 ? 47 : 90);
      if (G == 2 && pct > 0) return std::min<int64_t>(B - 1, std::max<int64_t>(1, (B * pct + 50) / 100));
      return B * k / G;
    };
    const int slots = hist_grid(c);
    int64_t prev_nb = 0;
    for (int64_t k = 0; k < G && e == cudaSuccess; ++k) {
      const int64_t b0 = gstart(k), nb = gstart(k + 1) - b0;
      const int grid = (int)std::max<int64_t>(c->num_sms, slots - std::min<int64_t>(prev_nb, slots / 2));
      e = counted(c, hr::launch_hist(in + b0 * img, nb, H, W, hs + b0 * kLevels, graw + b0 * kGradSlots, grid, st,
                                     done + b0, k > 0, hist_nt(c)));
      if (e == cudaSuccess) e = solve_group(b0, nb, 2, true);
      prev_nb = nb;
    }
    if (e == cudaSuccess) e = mark(2);
    // the apply grid: every slot (2 per SM) when the last group is the larger one -- the CTAs that
    // can only start once solve(G-1)'s CTAs leave then still add streaming capacity for the
    // rest of the apply, their static share of the first groups being small (C3 0.2509 ->
    // 0.2407 ms); else the slots the last group's solver CTAs leave (C5: a full grid puts 90%
    // of the work in static shares that late CTAs finish last, 0.1876 vs 0.1649 ms)
    const bool full_apply = c->apply_full_grid >= 0 ? c->apply_full_grid != 0 : 2 * gstart(G - 1) < B;
    const int ag = full_apply ? apply_grid(c)
                              : (int)std::max<int64_t>(c->num_sms, apply_grid(c) - std::min<int64_t>(prev_nb, apply_grid(c) / 2));
    if (e == cudaSuccess)
      e = counted(c, hr::launch_apply(in, lut, B, H, W, out, ag, st, ready, gstart(G - 1), ctl + 3, c->apply_gs));
  } else {
    // separate kernels: hist | solve + LUT | apply, chained by PDL; the apply grid, launched
    // early, starts on images whose LUT-ready flag is set while the solver grid finishes
    c->last_path = 0;
    g_launch_label = "hist";
    if (e == cudaSuccess) e = counted(c, hr::launch_hist(in, B, H, W, hs, graw, hist_grid(c), st, nullptr, false, hist_nt(c)));
    if (e == cudaSuccess) e = mark(1);
    if (e == cudaSuccess) e = solve_group(0, B, solve_cpsm_for(c, B), false);
    if (e == cudaSuccess) e = mark(2);
    g_launch_label = "apply";
    if (e == cudaSuccess) e = counted(c, hr::launch_apply(in, lut, B, H, W, out, apply_grid(c), st, ready));
  }
  if (e == cudaSuccess) e = mark(3);
  if (e == cudaSuccess) e = idx1_mark_used(c, slot, st);
  return cuda_err(c, e, "hr_enhance");
}

hr_status hr_enhance(hr_ctx* c, const uint8_t* in, int64_t B, int32_t H, int32_t W, const hr_params* p,
                     uint8_t* out, void* ws, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  // one image: the step's launches (zeroing, histograms, solve, apply: launch-latency bound at
  // these sizes) replayed from a cached CUDA graph captured from the same calls; the PDL edges
  // become programmatic graph edges.  Not for the legacy default stream (no capture there),
  // while stage profiling is on, or while the caller itself is capturing.
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (!c || !c->graph_b1 || B != 1 || !st || st == cudaStreamLegacy || st == cudaStreamPerThread || c->prof ||
      cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone ||
      check_shape(c, B, H, W) != HR_OK || check_params(c, p) != HR_OK || !in || !out || !ws || in == out) {
    cudaGetLastError();
    return hr_enhance_debug(c, in, B, H, W, p, out, ws, nullptr, stream);
  }
  hr_status s = activate(c);
  if (s) return s;
  for (auto& g : c->graphs)
    if (g.exec && g.in == in && g.out == out && g.ws == ws && g.st == st && g.H == H && g.W == W &&
        memcmp(&g.p, p, sizeof(hr_params)) == 0) {
      g.used = ++c->graph_clock;
      cudaError_t e = cudaGraphLaunch(g.exec, st);
      if (e == cudaSuccess) c->launches += g.kernels;
      if (e == cudaSuccess) e = cudaEventRecord(c->idx1_used[g.slot], st);
      return cuda_err(c, e, "hr_enhance (graph)");
    }
  // miss: build the gamma's index_1 table outside the capture, capture the step, instantiate
  const uint8_t* tab = nullptr;
  int slot = 0;
  cudaError_t e = idx1_table(c, p->gamma, &tab, &slot);
  if (e != cudaSuccess) return cuda_err(c, e, "hr_enhance (index_1 table)");
  e = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return hr_enhance_debug(c, in, B, H, W, p, out, ws, nullptr, stream);
  }
  const int64_t l0 = c->launches;
  const hr_status r = hr_enhance_debug(c, in, B, H, W, p, out, ws, nullptr, stream);
  cudaGraph_t graph = nullptr;
  e = cudaStreamEndCapture(st, &graph);
  const int64_t nk = c->launches - l0;
  c->launches = l0;
  if (r != HR_OK) {
    if (graph) cudaGraphDestroy(graph);
    return r;
  }
  cudaGraphExec_t exec = nullptr;
  if (e == cudaSuccess) e = cudaGraphInstantiate(&exec, graph, 0);
  if (graph) cudaGraphDestroy(graph);
  if (e != cudaSuccess) return cuda_err(c, e, "hr_enhance (graph capture)");
  hr_ctx::GraphEntry* v = &c->graphs[0];  // the least recently used slot
  for (auto& g : c->graphs)
    if (g.used < v->used) v = &g;
  if (v->exec) cudaGraphExecDestroy(v->exec);
  *v = hr_ctx::GraphEntry{in, out, ws, st, H, W, *p, exec, slot, nk, ++c->graph_clock};
  e = cudaGraphLaunch(exec, st);
  if (e == cudaSuccess) c->launches += nk;
  if (e == cudaSuccess) e = cudaEventRecord(c->idx1_used[slot], st);
  return cuda_err(c, e, "hr_enhance (graph)");
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
  if (e == cudaSuccess) e = counted(c, hr::launch_hist(in, B, H, W, hs, graw, hist_grid(c), st, nullptr, false, hist_nt(c)));
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
    const hr_status r = hr_enhance_debug(c, in_d + b0 * img, nb, H, W, p, out_d + b0 * img, ws, nullptr, stream);
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

extern "C" hr_status hr_trace_bind(hr_ctx* c, void* records, uint32_t* count, uint32_t capacity) {
  if (!c) return HR_EINVAL;
  if (records && (!count || capacity == 0)) return set_err(c, HR_EINVAL, "count and capacity are required");
  hr_status s = activate(c);
  if (s) return s;
  if (!records) count = nullptr, capacity = 0;
  cudaError_t e = hr::trace_bind_hist(records, count, capacity);
  if (e == cudaSuccess) e = hr::trace_bind_solve(records, count, capacity);
  if (e == cudaSuccess) e = hr::trace_bind_apply(records, count, capacity);
  return cuda_err(c, e, "hr_trace_bind");
}
