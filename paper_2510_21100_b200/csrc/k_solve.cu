// k_solve.cu -- kernel (b): batched histogram-domain Retinex solver (Algorithm 1) in fp64,
// with the Eq. 17-20 reprocessing and the fused CDF + histogram-matching LUT tail (c).
//
// Standalone launches of the solver (one CTA per image), the per-gamma index_1 table, the
// gradient remap and the CDF/LUT match.  The device body is in solve_dev.cuh.
#include <algorithm>
#include <cstdlib>

#include "solve_cluster_dev.cuh"

namespace hr {
namespace {

// NT = 256: two CTAs per SM (batches); NT = 512: one CTA per SM, the cell loops over 16 warps.
// (A 64-register form, MINB = 4 -- four per SM, two beside a histogram CTA -- measured slower on
// C5 in the grouped step, 0.177 vs 0.165 ms, and is not built.)
template <int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_solve(SolveArgs args) {
  extern __shared__ __align__(16) unsigned char smraw[];
  __shared__ int wscr[NT / 32];
  TRACE_T0();
  unsigned long long tr_mid = 0ull;
  (void)tr_mid;
  if (!args.hist_done) {
    pdl_wait();
    pdl_trigger();
  } else {
    pdl_trigger();
  }
  const int64_t b = blockIdx.x;
  if (args.hist_done) {  // wait for this image's histogram rows only (all H rows flushed)
    if (threadIdx.x == 0) wait_flag_geq(args.hist_done + b, (uint32_t)args.hist_H, 256);
    __syncthreads();
  }
  TRACE_MID(tr_mid);
  solve_image<NT>(args, b, smraw, wscr);
  if (args.ready) {  // every exit of solve_image arrives here: the LUT is written
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) st_release(args.ready + b, 1u);
  }
  TRACE_END(3u, (uint32_t)((uintptr_t)args.hist_s >> 8), tr_mid);  // aux: which launch (group)
}

// One image per cluster of CS CTAs (solve_cluster_dev.cuh): large single images.
template <int NT, int CS>
__global__ void __launch_bounds__(NT, 1) k_solve_cluster(SolveArgs args) {
  extern __shared__ __align__(16) unsigned char smraw[];
  __shared__ int wscr[NT / 32];
  TRACE_T0();
  unsigned long long tr_mid = 0ull;
  (void)tr_mid;
  pdl_trigger();
  const int64_t b = blockIdx.x / CS;
  // the state structs start zeroed: without this the kernel faulted (illegal address) in one
  // test sequence on B200 -- zeroing either struct region fixed it, the arena region did not;
  // the stale shared-memory read behind it was not pinned down (the checked build's bounds
  // checks stay silent), so this stays as a guard (~30 KB of 16-B stores, < 1 us)
  for (int i = threadIdx.x; i < (int)((sizeof(Sm) + sizeof(SmClusterExtra)) / 16); i += NT)
    reinterpret_cast<uint4*>(smraw)[i] = make_uint4(0u, 0u, 0u, 0u);
  __syncthreads();
  TRACE_MID(tr_mid);
  solve_image_cluster<NT, CS>(args, b, smraw, wscr);
  if (args.ready && (blockIdx.x % CS) == 0) {  // rank 0 wrote the LUT
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) st_release(args.ready + b, 1u);
  }
  TRACE_END(3u, (uint32_t)((uintptr_t)args.hist_s >> 8), tr_mid);
}

// index_1(i, j) of Eqs. 17-19 for every (i, j), once per gamma (R4, R5):
// p_j = b_j^(1/gamma) (b_j itself when gamma == 1), first k minimising |b_i p_j - b_k|.
__global__ void __launch_bounds__(kLevels) k_idx1_table(double gamma, uint8_t* tab) {
  __shared__ double bk[kLevels], pj[kLevels];
  const int j = threadIdx.x;
  bk[j] = (double)j / 255.0;
  pj[j] = (gamma == 1.0) ? bk[j] : pow(bk[j], 1.0 / gamma);
  __syncthreads();
  const int i = blockIdx.x;
  tab[i * kLevels + j] = (uint8_t)idx1(bk, bk[i], pj[j]);
}

__global__ void __launch_bounds__(kLevels) k_remap(const uint32_t* graw, int32_t grad_norm, uint32_t* hist_g) {
  __shared__ uint32_t h[kLevels];
  __shared__ int wscr[kLevels / 32];
  const int64_t b = blockIdx.x;
  remap_gradient<kLevels>(graw + b * kGradSlots, grad_norm, h, wscr);
  hist_g[b * kLevels + threadIdx.x] = h[threadIdx.x];
}

__global__ void __launch_bounds__(kLevels) k_match(const uint32_t* hist_s, const double* target, uint8_t* lut,
                                             int32_t* status) {
  __shared__ uint32_t hSi[kLevels];
  __shared__ __align__(16) double Tt[kLevels], Pt[kLevels], Ct[kLevels], Cs[kLevels];
  __shared__ int wscr[kLevels / 32];
  const int64_t b = blockIdx.x;
  hSi[threadIdx.x] = hist_s[b * kLevels + threadIdx.x];
  Tt[threadIdx.x] = target[b * kLevels + threadIdx.x];
  __syncthreads();
  cdf_lut<kLevels>(hSi, Tt, Pt, Ct, Cs, wscr, lut + b * kLevels, status ? status + b : nullptr);
}

}  // namespace

cudaError_t trace_bind_solve(void* buf, uint32_t* n, uint32_t cap) { return trace_bind_tu(buf, n, cap); }

size_t solve_smem_bytes(int arena_bytes) { return sizeof(Sm) + (size_t)(arena_bytes > 0 ? arena_bytes : kArenaSmem); }
// one global arena per image, or per (image, rank) when the image may take the cluster solver
size_t solve_cells_ws_bytes(int64_t B) {
  return (size_t)std::max<int64_t>(B, std::min<int64_t>(B, kClusterMaxB) * kClusterCS) * (size_t)kArenaGlobal;
}
size_t solve_cluster_smem_bytes() { return sizeof(Sm) + sizeof(SmClusterExtra) + (size_t)kArenaSmem; }

template <int NT, int CS>
cudaError_t cluster_attrs() {
  cudaError_t e = cudaFuncSetAttribute(k_solve_cluster<NT, CS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)solve_cluster_smem_bytes());
  if (e == cudaSuccess && CS > 8) e = cudaFuncSetAttribute(k_solve_cluster<NT, CS>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  return e;
}

constexpr int kBigArena = 190 * 1024;  // sizeof(Sm) + 190 KB <= 227 KB per block

cudaError_t init_attrs_solve() {
  cudaError_t e = cudaSuccess;
  for (auto k : {k_solve<256, 2>, k_solve<512, 1>}) {
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)solve_smem_bytes(kBigArena));
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared);
  }
  if (e == cudaSuccess) e = cluster_attrs<256, 8>();
  if (e == cudaSuccess) e = cluster_attrs<512, 8>();
  if (e == cudaSuccess) e = cluster_attrs<256, 16>();
  if (e == cudaSuccess) e = cluster_attrs<512, 16>();
  return e;
}

// cpsm == 1: one solver CTA per SM (the CTA scheduler would otherwise pack two latency-bound
// solves onto one SM while others idle).  The shared memory that placement reserves anyway is
// given to the run arena (kBigArena), so images with large supports (C4: E = 8480 cells) keep
// their run structure in shared memory instead of the global arena.
cudaError_t launch_solve(const SolveArgs& a0, int64_t B, int cpsm, cudaStream_t st, bool wide) {
  SolveArgs a = a0;
  if (cpsm == 1 && a.arena_bytes == 0) a.arena_bytes = kBigArena;
  if (cpsm == 1 && wide)
    return launch_pdl(k_solve<512, 1>, dim3((unsigned)B), dim3(512), solve_smem_bytes(a.arena_bytes), st, a);
  return launch_pdl(k_solve<256, 2>, dim3((unsigned)B), dim3(256), solve_smem_bytes(a.arena_bytes), st, a);
}

// B images, one cluster of kClusterCS CTAs (256 threads each) per image (B <= kClusterMaxB)
template <int NT, int CS>
cudaError_t launch_cluster_v(const SolveArgs& a0, int64_t B, cudaStream_t st) {
  SolveArgs a = a0;
  a.arena_bytes = kArenaSmem;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(B * CS));
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = solve_cluster_smem_bytes();
  cfg.stream = st;
  // a plain (not programmatically serialized) launch: with programmatic dependent launch the
  // cluster kernel raised illegal-address faults on B200 / driver 580 (one test sequence, every
  // run; not with launch blocking, PDL off, or this launch without it), so its CTAs start
  // after the histogram grid completes.  Its own trigger still lets the apply launch early.
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_solve_cluster<NT, CS>, a);
}

cudaError_t launch_solve_cluster(const SolveArgs& a, int64_t B, cudaStream_t st, int variant) {
  switch (variant) {
    case 2: return launch_cluster_v<512, 8>(a, B, st);
    case 3: return launch_cluster_v<256, 16>(a, B, st);
    case 4: return launch_cluster_v<512, 16>(a, B, st);
    default: return launch_cluster_v<256, 8>(a, B, st);
  }
}

cudaError_t launch_idx1_table(double gamma, uint8_t* tab, cudaStream_t st) {
  k_idx1_table<<<kLevels, kLevels, 0, st>>>(gamma, tab);
  return cudaGetLastError();
}

cudaError_t launch_remap(const uint32_t* hist_graw, int64_t B, int32_t grad_norm, uint32_t* hist_g,
                         cudaStream_t st) {
  k_remap<<<(unsigned)B, kLevels, 0, st>>>(hist_graw, grad_norm, hist_g);
  return cudaGetLastError();
}

cudaError_t launch_match(const uint32_t* hist_s, const double* target, int64_t B, uint8_t* lut,
                         int32_t* status, cudaStream_t st) {
  k_match<<<(unsigned)B, kLevels, 0, st>>>(hist_s, target, lut, status);
  return cudaGetLastError();
}

}  // namespace hr

#ifdef HR_SOLVE_PROFILE
// measurement-only export of the phase clocks (profiling builds; not part of histretinex.h)
extern "C" int hr_debug_solve_clocks(long long* out, int n) {
  int cnt = 0;
  cudaMemcpyFromSymbol(&cnt, hr::g_solve_nclk, sizeof(int));
  if (cnt > n) cnt = n;
  cudaMemcpyFromSymbol(out, hr::g_solve_clk, sizeof(long long) * cnt);
  int zero = 0;
  cudaMemcpyToSymbol(hr::g_solve_nclk, &zero, sizeof(int));
  return cnt;
}
extern "C" int hr_debug_solve_clocks_all(long long* out) {
  return (int)cudaMemcpyFromSymbol(out, hr::g_solve_clk, sizeof(long long) * 1024);
}
#endif
