/*
 * histretinex.h -- C-ABI of the B200-native HistRetinex hot path (sm_100a).
 *
 * The library computes, for a batch of 8-bit RGB low-light images, the per-image
 * pipeline of HistRetinex (arXiv 2510.21100, /root/reference/PAPER.md, "P:<line>"):
 *
 *   RGB8 -> value channel S and gradient image -> 256-bin count histograms (Eq. 3)
 *        -> histogram-domain Retinex solve, Algorithm 1 (Eqs. 6-15)
 *        -> gamma-reprocessed enhanced histogram (Eqs. 17-20)
 *        -> histogram matching LUT -> per-pixel LUT apply + colour.
 *
 * Readings of the paper where it is silent or garbled are DESIGN.md section 3
 * (R1..R21); they are named at each entry point below.
 *
 * Conventions for every call
 * --------------------------
 *  - Pointers named *_dev / device arrays are CUDA device pointers owned by the
 *    caller; the library never allocates caller-visible memory and never frees
 *    caller memory.  Host pointers appear only in hr_enhance_host.
 *  - Images are contiguous uint8 [B][H][W][3] (HWC, RGB), per-image stride
 *    H*W*3 bytes.  Any base alignment is accepted; 16-byte aligned bases with
 *    W % 16 == 0 take the vectorised path.
 *  - Histograms are uint32 [B][256]; raw gradient histograms uint32 [B][512]
 *    (bins 0..510 used, bin 511 always 0).  Float histograms are double [B][256].
 *  - `stream` is a cudaStream_t (passed as void* so this header needs no CUDA
 *    include); NULL means the legacy default stream.  All device calls are
 *    asynchronous on `stream`; they never synchronise the host.
 *  - Validation is synchronous and happens before anything is launched: on any
 *    error nothing is enqueued and the status is returned.  Asynchronous CUDA
 *    faults surface on a later call or on stream synchronisation.
 *  - Outputs are bit-identical run to run (deterministic reductions, integer
 *    histogram atomics only).
 *  - A context is not thread-safe: use one hr_ctx per host thread.
 *  - No C++ exception or exit() crosses this boundary.
 */
#ifndef HISTRETINEX_H
#define HISTRETINEX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HR_OK = 0,
  HR_EINVAL = 1,        /* null pointer, B < 1, negative size, parameter out of range */
  HR_EEMPTY = 2,        /* H*W == 0 (an image has no pixels) */
  HR_EDEGENERATE = 3,   /* all-zero target histogram in hr_match (per image, see img_status) */
  HR_ECUDA = 4,         /* a CUDA runtime call failed; text in hr_last_error() */
  HR_EUNSUPPORTED = 5   /* valid for the paper but not for this build (levels != 256) */
} hr_status;

/* Parameters of Algorithm 1 ("Input: ... error threshold eps, maximum iteration T,
   weight parameter alpha and beta") and of the reprocessing (Eq. 17 gamma). */
typedef struct hr_params {
  int32_t levels;      /* number of gray levels l; must be 256 (HR_EUNSUPPORTED otherwise) */
  int32_t max_iter;    /* T >= 1 (Alg. 1); the paper's timing runs use 10 */
  double alpha;        /* > 0, weight of the illumination prior (Eq. 10) */
  double beta;         /* > 0, weight of the reflectance (gradient) prior (Eq. 10) */
  double gamma;        /* >= 1, Eq. 17 gamma on the illumination location vector (R13) */
  double epsilon;      /* > 0, stop threshold RELATIVE to N^2: ||dh||^2 <= epsilon*N^2 (R11) */
  int32_t use_epsilon; /* 0: exactly max_iter iterations; 1: Alg. 1 stop rule (R11) */
  int32_t update_form; /* 0: gradient-consistent Eqs. 12-13 (R7, default); 1: as printed */
  int32_t grad_norm;   /* 0: MAXNORM gradient levels (R14, default); 1: RAW_CLAMP min(g,255) */
  int32_t reserved;    /* must be 0 */
} hr_params;

/* Fills the defaults: levels 256, T 10, alpha 0.1, beta 1e-3, gamma 2.2, epsilon 1e-3,
   use_epsilon 0, update_form 0, grad_norm 0 (R12-R14).  HR_EINVAL on NULL. */
hr_status hr_default_params(hr_params* p);

typedef struct hr_ctx hr_ctx;

/* Creates a context bound to CUDA device `device` (queries SM count, L2 size; builds no
   tables).  *ctx is set to NULL on failure. */
hr_status hr_create(hr_ctx** ctx, int device);
/* Destroys a context (NULL is a no-op).  Does not synchronise caller streams. */
hr_status hr_destroy(hr_ctx* ctx);

const char* hr_status_string(hr_status s);
/* Last error text of this context (never NULL; "" when none). */
const char* hr_last_error(const hr_ctx* ctx);
/* Library version string, e.g. "histretinex-b200 0.1 sm_100a". */
const char* hr_version(void);

/* Device workspace bytes needed by hr_enhance / hr_histogram / hr_solve for a batch
   of B images of H x W (0 on invalid sizes).  The caller allocates it (e.g. torch). */
size_t hr_workspace_bytes(int64_t B, int32_t H, int32_t W);

/* Step (1): value channel S = max(R,G,B) ("S is the value channel ... in the HSV";
   R15) and its gradient image g = |dx| + |dy| with forward differences, 0 on the last
   column / row (R14), reduced to count histograms (Eq. 3):
     hist_s[b][v]     = #{pixels of image b with S == v}                 (256 bins)
     hist_g_raw[b][g] = #{pixels of image b with raw gradient == g}      (512 slots)
     hist_g[b][k]     = #{pixels whose gradient level is k}              (256 bins)
   where the gradient level is MAXNORM: (510*g + gmax) / (2*gmax) (integer division,
   gmax = largest raw gradient of the image, all 0 if gmax == 0) or RAW_CLAMP: min(g,255),
   chosen by grad_norm (0/1).  hist_g_raw may be NULL.  Sums equal H*W exactly.
   Workspace: hr_workspace_bytes(B,H,W) bytes, device. */
hr_status hr_histogram(hr_ctx* ctx, const uint8_t* rgb_dev, int64_t B, int32_t H, int32_t W,
                       int32_t grad_norm, uint32_t* hist_s_dev, uint32_t* hist_g_dev,
                       uint32_t* hist_g_raw_dev, void* ws_dev, void* stream);

/* Step (2): Algorithm 1 on each image's histograms, fp64:
   H_C(R)^0 = hist_g, H_C(L)^0 = hist_s (R9); repeat Eq. 13, Eq. 12 (raw new R, frozen K,
   R10), Eq. 15, Eq. 14, Eq. 11 until the stop rule (R11).  Then Eqs. 17-20 give the
   enhanced histogram target[b][k] = sum over index_1(i,j)==k of hR_i hL_j / N (N = sum
   hist_s).  Outputs (device, [B][256] doubles; iters [B] nullable): final hL, hR
   (renormalised, sum N, exactly 0 off the supports of hist_s / hist_g), target.
   Images with N == 0 get all-zero outputs and iters 0.
   Workspace: hr_workspace_bytes(B,1,1) bytes or more, device. */
hr_status hr_solve(hr_ctx* ctx, const uint32_t* hist_s_dev, const uint32_t* hist_g_dev, int64_t B,
                   const hr_params* params, double* hL_dev, double* hR_dev, double* target_dev,
                   int32_t* iters_dev, void* ws_dev, void* stream);

/* hr_solve with the Eq. 10 objective trace (diagnostics):
   three values per update t, K frozen at the state of update t (Eq. 11):
   trace[b][3t]   = F(hR^t,  hL^t),   before Eq. 13
   trace[b][3t+1] = F(hR',   hL^t),   after Eq. 13 (raw, before renormalisation)
   trace[b][3t+2] = F(hR',   hL'),    after Eq. 12 (raw)
   F = sum_ij (hR_i hL_j / N - K_ij hS_index(i,j))^2 + alpha |hL - hS|^2 + beta |hR - hG|^2.
   trace_dev: double [B][trace_stride], trace_stride >= 3 * params->max_iter; entries from
   3 * iters on are zero.  Slower than hr_solve (one more pass over the cells per value). */
hr_status hr_solve_trace(hr_ctx* ctx, const uint32_t* hist_s_dev, const uint32_t* hist_g_dev, int64_t B,
                         const hr_params* params, double* hL_dev, double* hR_dev, double* target_dev,
                         int32_t* iters_dev, double* trace_dev, int32_t trace_stride, void* ws_dev,
                         void* stream);

/* Step (3): histogram matching (R16).  Cs(v) = Ps(v)/N with Ps the integer prefix
   of hist_s; Pt(k) = Pt(k-1) + target(k) (plateau-preserving), Ct(k) = Pt(k)/Pt(255);
   lut[b][v] = smallest k minimising |Ct(k) - Cs(v)| (monotone non-decreasing in v).
   img_status[b] (nullable) = HR_OK, or HR_EDEGENERATE when Pt(255) <= 0 or N == 0 (lut
   is then the identity). */
hr_status hr_match(hr_ctx* ctx, const uint32_t* hist_s_dev, const double* target_dev, int64_t B,
                   uint8_t* lut_dev, int32_t* img_status_dev, void* stream);

/* Step (4): per-pixel LUT application and colour reconstruction (R17):
   V = max(R,G,B), V' = lut[b][V]; each channel c -> floor((2*c*V' + V) / (2*V)), i.e.
   V replaced in exact hexcone HSV with H and S kept, rounded half up; V == 0 -> (V',V',V').
   rgb_out may equal rgb_in (in place). */
hr_status hr_apply(hr_ctx* ctx, const uint8_t* rgb_in_dev, const uint8_t* lut_dev, int64_t B,
                   int32_t H, int32_t W, uint8_t* rgb_out_dev, void* stream);

/* Steps (1)-(4) for the whole batch ("matching its histogram with the one provided by
   HistRetinex") on `stream`.  One image (or policy groups = 0): the histogram, solve + LUT and
   apply kernels in order, chained by programmatic dependent launch, the apply acquiring each
   image's LUT-ready flag (so it overlaps the solver's tail).  B >= 2: the grouped step (two
   image groups, policy "groups": the second group's histograms run beside the first group's
   solves, the apply beside the second group's solves).  One image on a non-default stream
   (policy graph_b1): the step's launches are captured once into a CUDA graph, cached per
   call arguments, and replayed.  Every policy gives bit-identical outputs.  The first call with a new gamma builds its index_1 table (Eqs. 17-19) and waits for
   it (host-blocking, once per gamma per context).  Intermediate results: hr_enhance_debug.
   rgb_out must not alias rgb_in.
   Workspace: hr_workspace_bytes(B,H,W), device. */
hr_status hr_enhance(hr_ctx* ctx, const uint8_t* rgb_in_dev, int64_t B, int32_t H, int32_t W,
                     const hr_params* params, uint8_t* rgb_out_dev, void* ws_dev, void* stream);

/* Steps (1)-(4) from HOST memory to HOST memory, pipelined over image chunks: chunk k's
   host->device copy overlaps chunk k-1's enhancement (hr_enhance on `stream`) and chunk
   k-2's device->host copy (PCIe is full duplex; the copies run on two library streams).
   rgb_in_host, rgb_out_host: [B][H][W][3] host buffers, page-locked (cudaHostAlloc /
   cudaHostRegister) for the copies to be asynchronous -- pageable memory still works but the
   copies then serialise.  in_dev, out_dev: caller-owned device staging buffers of B*H*W*3
   bytes each (reused across calls); ws_dev: hr_workspace_bytes(B, H, W).  chunks: number of
   image chunks, 1..B (0 = min(B, 8)).  Enqueued on `stream`: rgb_out_host is complete when
   `stream` reaches this point (e.g. after cudaStreamSynchronize).  The outputs are
   bit-identical to hr_enhance on the same images.  rgb_out_host must not alias rgb_in_host. */
hr_status hr_enhance_host(hr_ctx* ctx, const uint8_t* rgb_in_host, int64_t B, int32_t H, int32_t W,
                          const hr_params* params, uint8_t* rgb_out_host, uint8_t* in_dev, uint8_t* out_dev,
                          void* ws_dev, int32_t chunks, void* stream);

/* hr_enhance with intermediate results (parity tests): every non-NULL field receives, for the
   same schedule and launch configuration as hr_enhance, the image's hist_s / hist_g (the
   gradient levels of R14) [B][256] uint32, lut [B][256], iters [B], and the solver's final hL,
   hR and Eq. 20 target [B][256] double (device pointers, caller-owned).  dbg may be NULL. */
typedef struct hr_debug_out {
  uint32_t* hist_s;
  uint32_t* hist_g;
  uint8_t* lut;
  int32_t* iters;
  double* hL;
  double* hR;
  double* target;
} hr_debug_out;
hr_status hr_enhance_debug(hr_ctx* ctx, const uint8_t* rgb_in_dev, int64_t B, int32_t H, int32_t W,
                           const hr_params* params, uint8_t* rgb_out_dev, void* ws_dev,
                           const hr_debug_out* dbg, void* stream);

/* ---- Second workload: the HE baseline and the quality metrics ---- */

/* HE baseline (Eq. 5): V -> t_V = floor(255 c_V + 0.5), c the running sum of
   hS_u / N (Eq. 4), with the R17 colour reconstruction of hr_apply.  lut_dev (nullable):
   the [B][256] HE tables.  Workspace: hr_workspace_bytes(B, H, W).  rgb_out must not alias
   rgb_in.  Bit-exact with the oracle. */
hr_status hr_he(hr_ctx* ctx, const uint8_t* rgb_in_dev, int64_t B, int32_t H, int32_t W,
                uint8_t* rgb_out_dev, uint8_t* lut_dev, void* ws_dev, void* stream);

/* Bytes of device workspace hr_quality needs (0 for empty shapes). */
size_t hr_quality_workspace_bytes(int64_t B, int32_t H, int32_t W);

/* Quality metrics of image pairs a[b], b[b] (P:311 names them; SPEC.md metrics module defines
   them): PSNR = 10 log10(255^2 / MSE) over all channels (+inf if equal); SSIM on luma
   0.299R + 0.587G + 0.114B with an 11x11 Gaussian (sigma 1.5), valid windows, C1 = (0.01*255)^2,
   C2 = (0.03*255)^2, the mean of the map (NaN if H or W < 11); LOE = (1/m) sum over pairs of
   sampled pixels of [(L(x) >= L(y)) xor (L'(x) >= L'(y))], L = max(R,G,B) on a
   min(H,100) x min(W,100) nearest-neighbour grid (row (i H)/mh, column (j W)/mw), a = original.
   Outputs: double [B] each, nullable (at least one).  Workspace: hr_quality_workspace_bytes.
   fp64; deterministic.  LOE is exact; PSNR and SSIM equal the oracle up to rounding order. */
hr_status hr_quality(hr_ctx* ctx, const uint8_t* a_dev, const uint8_t* b_dev, int64_t B, int32_t H,
                     int32_t W, double* psnr_dev, double* ssim_dev, double* loe_dev, void* ws_dev,
                     void* stream);

/* Stage timing (measurement only).  While enabled, every hr_enhance records four CUDA
   events on its stream.  Separate-kernel path: before the histogram kernel, after it,
   after the solver + LUT, after the apply kernel -> stage_ms[0] histogram incl. its
   zeroing, [1] solve + LUT, [2] apply.
   hr_profile_collect waits for the recorded events, returns the summed milliseconds over
   the *steps calls since the last collect, and resets the counters.  Grouped step: before the
   accumulator zeroing, after it, after the last solver launch, after the apply -> stage_ms[0]
   zeroing, [1] histograms + solves of all groups, [2] the apply (stages overlap on the device,
   so only the sum is a step time).  At most 4096 calls
   are kept between collects (HR_EINVAL beyond). */
hr_status hr_profile_enable(hr_ctx* ctx, int32_t on);
hr_status hr_profile_collect(hr_ctx* ctx, double* stage_ms, int32_t* steps);

/* Step timeline (measurement only).  Binds a device record buffer for every later launch on
   this context's device (NULL records unbinds; count and capacity are then ignored): thread 0
   of each CTA of the histogram, solver and apply kernels appends one 48-byte record
     { uint32 kind (1 histogram, 3 solver, 4 apply), cta, sm, aux;
       uint64 start_ns, mid_ns, end_ns, pad }
   at records[atomicAdd(count, 1)] while that index is below capacity (%globaltimer
   nanoseconds; aux = (hist_s address of the launch's first image) >> 8 for the histogram and
   solver kernels, so launches of one step are told apart; mid_ns = when a solver CTA's image
   histograms were complete).  The caller zeroes *count (device uint32) and owns both buffers.
   Outputs of every entry point are unchanged while bound. */
hr_status hr_trace_bind(hr_ctx* ctx, void* records_dev, uint32_t* count_dev, uint32_t capacity);

/* Execution policy of hr_enhance (performance only: results never depend on it).  Keys:
     "hist_cpsm", "apply_cpsm"  streaming kernels' CTAs per SM (1..2)          default 2
     "solve_cpsm"   solver CTAs per SM: 1, 2, 0 = auto (1 when B <= #SMs)      default 0
     "solve_wide_px" one solver CTA per SM (B <= #SMs): 512-thread CTAs for     default 4194304
                    images of H*W >= value pixels (0: never; large images have
                    large supports: C4 103 vs 121 us per image, while small
                    supports are faster at 256 threads: C2 37 vs 43 us)
     "groups"       grouped step (>= 2): images in G groups, launched in order  default -1
                    hist(0) solve(0) hist(1) solve(1) ... solve(G-1) apply; the
                    histograms of group k+1 run beside the solves of group k (they
                    do not wait for them), the apply (every CTA: groups 0..G-2
                    first, the last group by CTA tickets) beside the last group's
                    solves; streaming grids sized to the slots the resident solver
                    CTAs leave.  0/1: off (separate kernels); -1: auto = 2 when B >= 2
     "group_first_pct" grouped step with 2 groups: the first group's share of  default -1
                    the batch in % (0: equal groups; -1: auto = 47 for B <= #SMs / 2,
                    the first solves hidden under the second histogram pass and the
                    last group still the larger one, C3 0.233 vs 0.244 ms at 50; 90
                    for larger batches, the last group's few solves beside the first
                    group's apply, C5 0.154 vs 0.177 ms ungrouped)
     "apply_gs"     grouped step's apply: 1024-pixel chunks per warp in one CTA  default 8
                    ticket of the last group (>= 1)
     "apply_full_grid" grouped step's apply grid: 1 every slot (2 per SM; CTAs  default -1
                    that start once the last solver CTAs leave add capacity), 0 the
                    slots the last group's solver CTAs leave, -1 auto = every slot
                    when the last group is the larger (C3 0.2407 vs 0.2509 ms; C5,
                    a 90% first group, keeps the reduced grid: 0.1649 vs 0.1876)
     "solve_cluster" images of H*W >= solve_wide_px (<= 9 per call, separate   default 1
                    kernels): each solved by a thread-block cluster exchanging
                    partial sums through distributed shared memory: 1 = 8 CTAs x
                    256 threads, 2 = 8 x 512, 3 = 16 x 256, 4 = 16 x 512; 0: one
                    512-thread CTA (C4: 77 us vs 119 us per image)
     "graph_b1"     hr_enhance with B == 1 on a non-default stream: the step is     default 1
                    captured once into a CUDA graph (cached per call arguments,
                    8 entries, LRU) and replayed (C1/C2/C4 1.5-2 us faster; batches
                    launch directly: they lose the PDL overlap of consecutive steps
                    in a graph)
   The environment variables HR_<KEY upper-cased> set the initial values at hr_create.
   Returns HR_EINVAL for an unknown key or an out-of-range value (nothing changes). */
hr_status hr_set_policy(hr_ctx* ctx, const char* key, int64_t value);
/* Current value of a policy key (same keys as hr_set_policy) into *value.  HR_EINVAL for a
   NULL ctx / key / value or an unknown key (*value untouched). */
hr_status hr_get_policy(hr_ctx* ctx, const char* key, int64_t* value);

/* Number of CUDA kernels this context has launched so far (all entry points, including the
   accumulator-zeroing kernel; driver memsets are not counted).  -1 for a NULL ctx. */
int64_t hr_kernel_launches(const hr_ctx* ctx);

/* Execution path of the last hr_enhance on this context: 0 separate kernels (histogram |
   solve + LUT | apply), 3 the grouped step (policy "groups"); -1 none yet or a NULL ctx. */
int32_t hr_last_path(const hr_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* HISTRETINEX_H */
