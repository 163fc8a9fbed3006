// k_fused.cu -- the whole hot path of a batch in ONE persistent kernel:
//   histograms (kernel (a) body, hist_dev.cuh) -> per-image Algorithm 1 solve + Eq. 20 +
//   CDF/LUT (kernel (b)+(c) body, solve_dev.cuh) -> LUT apply (kernel (d), apply_dev.cuh).
//
// Why: the solve is latency-bound (~70 us per image, one CTA each).  Run serially between the
// two streaming passes it adds its whole latency to the step; here it overlaps them.
//
// Work queue (one global ticket per phase, taken in order):
//   phase 1  items (b, band) image-major: CTA histograms rows [H band/KB, H (band+1)/KB) of
//            image b, flushes with integer atomics, then counts the band in done[b].  The CTA
//            that completes image b's LAST band solves image b right away (fence -> ticket ->
//            fence, the threadfence-reduction pattern) and publishes ready[b] (release).
//   phase 2  entered when the phase-1 queue is exhausted: every WARP pulls groups of GS
//            512-px chunks (image-major) from the apply ticket into its own 5-stage TMA
//            bulk-copy pipeline, and before the first chunk of an image acquires ready[b].
// Deadlock freedom: a warp waits only on ready[b] of an image whose bands were all ticketed
// before phase 2 began (single queue order); each such band is held by a running CTA that
// waits on nothing, and the CTA that finishes the last one solves before taking new work.
// No co-residency assumption: a serialised execution (e.g. under a profiler) also finishes.
//
// Results are bit-identical to the separate kernels: the histogram counts are integers, the
// solve and LUT are the same device code on the same inputs, the apply is per pixel.
#include <algorithm>

#include "apply_dev.cuh"
#include "hist_dev.cuh"
#include "solve_dev.cuh"

namespace hr {
namespace {

constexpr int kFT = 256;  // threads per CTA (== kSolveThreads == kApplyThreads)
static_assert(kFT == kSolveThreads && kFT == kApplyThreads, "fused roles share the CTA shape");
constexpr size_t kFusedSmem =
    std::max(std::max((size_t)kHistDevSmem, sizeof(Sm) + (size_t)kArenaSmem), sizeof(ApplySmem));
constexpr uint32_t kEnd = 0xFFFFFFFFu;

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Timeline trace (measurement builds only: -DHR_FUSED_TRACE; tools/fused_trace.py).
#ifdef HR_FUSED_TRACE
struct TraceRec {
  uint32_t kind, cta, b, aux;  // kind: 0 hist band, 1 solve, 2 apply warp span, 3 ready wait, 4 CTA start
  unsigned long long t0, t1;   // %globaltimer ns
};
constexpr unsigned kTraceCap = 1u << 17;
__device__ TraceRec g_trace[kTraceCap];
__device__ unsigned g_ntrace;
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TRACE_T(v) const unsigned long long v = gtime()
#define TRACE(kind, b, aux, t0, t1)                                                               \
  do {                                                                                            \
    const unsigned i_ = atomicAdd(&g_ntrace, 1u);                                                 \
    if (i_ < kTraceCap) g_trace[i_] = TraceRec{(kind), blockIdx.x, (uint32_t)(b), (uint32_t)(aux), (t0), (t1)}; \
  } while (0)
#else
#define TRACE_T(v) \
  do {             \
  } while (0)
#define TRACE(kind, b, aux, t0, t1) \
  do {                              \
  } while (0)
#endif

template <int SW, int VEC>
__global__ void __launch_bounds__(kFT, 2) k_fused(const FusedArgs a) {
  extern __shared__ __align__(128) unsigned char smraw[];
  __shared__ int wscr[kFT / 32];
  __shared__ uint32_t meta[kWarps][kStages];
  __shared__ int sh;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int H = a.H, W = a.W, KB = a.KB;
  const int64_t HW = (int64_t)H * W;
  const size_t imgBytes = (size_t)HW * 3;
  uint32_t* done = a.ctl + kCtlHeader;
  uint32_t* ready = done + a.B;
  pdl_wait();
  pdl_trigger();
#ifdef HR_FUSED_TRACE
  if (tid == 0) {
    TRACE_T(tk);
    TRACE(4u, 0, 0, tk, tk);
  }
#endif

  // ---------------- phase 1: histogram bands; the last band of an image triggers its solve
  const int64_t NH = a.B * (int64_t)KB;
  uint32_t* hsm = reinterpret_cast<uint32_t*>(smraw);
  for (;;) {
    if (tid == 0) sh = (int)atomicAdd(a.ctl + 0, 1u);
    __syncthreads();
    const int64_t item = sh;
    if (item >= NH) break;  // CTA-uniform
#ifdef HR_FUSED_TRACE
    TRACE_T(th0);
#endif
    const int64_t b = item / KB;
    const int band = (int)(item - b * KB);
    const int y0 = (int)((int64_t)H * band / KB), y1 = (int)((int64_t)H * (band + 1) / KB);
    hist_zero<kFT>(hsm);
    __syncthreads();
    hist_segment<SW, VEC, kFT>(a.in + (size_t)b * imgBytes, H, W, y0, y1, hsm, a.hist_s + b * kLevels,
                               a.graw + b * kGradSlots);
    __threadfence();  // this CTA's flush atomics before its done[b] ticket
    __syncthreads();
    if (tid == 0) sh = (atomicAdd(done + b, 1u) == (uint32_t)(KB - 1)) ? 1 : 0;
#ifdef HR_FUSED_TRACE
    if (tid == 0) {
      TRACE_T(th1);
      TRACE(0u, b, band, th0, th1);
    }
#endif
    __syncthreads();
    if (sh) {  // image b complete: Algorithm 1 + Eq. 20 + LUT, then publish
#ifdef HR_FUSED_TRACE
      TRACE_T(ts0);
#endif
      __threadfence();
      solve_image<kFT>(a.sa, b, smraw, wscr);
      __threadfence();
      __syncthreads();
      if (tid == 0) st_release(ready + b, 1u);
#ifdef HR_FUSED_TRACE
      if (tid == 0) {
        TRACE_T(ts1);
        TRACE(1u, b, 0, ts0, ts1);
      }
#endif
    }
    __syncthreads();
  }

  // ---------------- phase 2: per-warp TMA pipelines over dynamically ticketed chunk groups
  ApplySmem& s = *reinterpret_cast<ApplySmem*>(smraw);
  if (lane == 0) {
    for (int k = 0; k < kStages; ++k) mbar_init(&s.bar[w][k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const uint32_t cpi = a.cpi, GS = a.GS;
  const uint32_t total = (uint32_t)(a.B * (int64_t)cpi);  // < 2^31 (host-checked)
  const uint32_t ngroups = (total + GS - 1) / GS;
  const uint64_t pol = policy_evict_first();
  uint2* tab = s.tab[w];
  // loader state (lane 0): next chunk, end of its group, prefetched next group ticket
  uint32_t ldc = 0, lde = 0, nxt = 0;
  if (lane == 0) nxt = atomicAdd(a.ctl + 1, 1u);
  auto next_chunk = [&]() -> uint32_t {
    if (ldc >= lde) {
      if (nxt >= ngroups) return kEnd;
      ldc = nxt * GS;
      lde = min(ldc + GS, total);
      nxt = atomicAdd(a.ctl + 1, 1u);
    }
    return ldc++;
  };
  auto locate = [&](uint32_t c, uint32_t& bimg, uint64_t& off, uint32_t& bytes) {
    bimg = c / cpi;
    const uint32_t px0 = (c - bimg * cpi) * kChunkPx;
    const uint32_t npx = min((uint32_t)kChunkPx, (uint32_t)(HW - px0));
    off = ((uint64_t)bimg * (uint64_t)HW + px0) * 3u;
    bytes = npx * 3u;
  };
  // LUT prefetch: when the loader reaches the first chunk of a new image (kAhead chunks before
  // the compute does), the warp acquires ready[b] and every lane loads its 8 LUT bytes into
  // registers, so the table rebuild at the image switch needs no memory access.  At most one
  // image is pending; a second switch inside the window takes the synchronous path.
  uint32_t ld_img = kEnd;  // image of the last issued chunk
  uint32_t pend_img = kEnd;
  uint2 pend = make_uint2(0u, 0u);
  auto issue = [&](uint32_t i) {  // all lanes (warp-uniform); lane 0 fills stage i % kStages
    const int st = (int)(i % kStages);
    uint32_t c = 0;
    if (lane == 0) c = next_chunk();
    c = __shfl_sync(0xffffffffu, c, 0);
    if (lane == 0) meta[w][st] = c;
    if (c == kEnd) {
      if (lane == 0) mbar_arrive(&s.bar[w][st]);
      return;
    }
    uint32_t bimg, bytes;
    uint64_t off;
    locate(c, bimg, off, bytes);
    if (bimg != ld_img) {
      ld_img = bimg;
      if (pend_img == kEnd) {
        uint32_t rdy = 0;
        if (lane == 0) rdy = ld_acquire(ready + bimg);
        __syncwarp();  // orders lane 0's acquire before the other lanes' LUT loads
        if (__shfl_sync(0xffffffffu, rdy, 0)) {
          pend = __ldcg(reinterpret_cast<const uint2*>(a.sa.lut + (uint64_t)bimg * kLevels) + lane);
          pend_img = bimg;
        }
      }
    }
    if (lane == 0) {
      mbar_expect_tx(&s.bar[w][st], bytes);
      bulk_load(s.stage[w][st], a.in + off, bytes, &s.bar[w][st], pol);
    }
  };

#ifdef HR_FUSED_TRACE
  TRACE_T(ta0);
#endif
  for (uint32_t i = 0; i < (uint32_t)kAhead; ++i) issue(i);
  int64_t cur_img = -1;
  int st = 0;
  uint32_t ph = 0;
  for (uint32_t i = 0;; ++i) {
    if (lane == 0 && i >= 2) bulk_wait_read<1>();  // the store of chunk i-2 has left stage (i+kAhead)%kStages
    __syncwarp();
    issue(i + kAhead);
    mbar_wait(&s.bar[w][st], ph);
    const uint32_t c = meta[w][st];
    if (c == kEnd) break;  // warp-uniform
    uint32_t bimg, bytes;
    uint64_t off;
    locate(c, bimg, off, bytes);
    HR_CHECK(c < total && bimg < a.B && bytes > 0 && bytes <= (uint32_t)kChunkBytes);
    if ((int64_t)bimg != cur_img) {  // image switch: rebuild the per-warp (e, M) table
      __syncwarp();
      if (bimg == pend_img) {
        build_tab_regs(tab, pend, lane);
        pend_img = kEnd;
      } else {
        if (lane == 0) {
#ifdef HR_FUSED_TRACE
          if (ld_acquire(ready + bimg) == 0u) {
            TRACE_T(tw0);
            while (ld_acquire(ready + bimg) == 0u) __nanosleep(200);
            TRACE_T(tw1);
            TRACE(3u, bimg, w, tw0, tw1);
          }
#else
          while (ld_acquire(ready + bimg) == 0u) __nanosleep(200);
#endif
        }
        __syncwarp();
        build_tab(tab, a.sa.lut + (uint64_t)bimg * kLevels, lane);
      }
      __syncwarp();
      cur_img = bimg;
    }
    uint8_t* p = s.stage[w][st];
    apply_chunk_smem(p, bytes, tab, lane);
    fence_async_smem();
    __syncwarp();
    if (lane == 0) {
      bulk_store(a.out + off, p, bytes, pol);
      bulk_commit();
    }
    if (++st == kStages) {
      st = 0;
      ph ^= 1u;
    }
  }
  if (lane == 0) bulk_wait<0>();
#ifdef HR_FUSED_TRACE
  if (lane == 0) {
    TRACE_T(ta1);
    TRACE(2u, 0, w, ta0, ta1);
  }
#endif
}

template <int SW, int VEC>
cudaError_t launch_fv(const FusedArgs& a, int grid, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_fused<SW, VEC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFusedSmem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  return launch_pdl(k_fused<SW, VEC>, dim3(grid), dim3(kFT), kFusedSmem, st, a);
}

}  // namespace

bool fused_supported(const uint8_t* in, const uint8_t* out, int64_t B, int32_t H, int32_t W) {
  const int64_t HW = (int64_t)H * W;
  return reinterpret_cast<uintptr_t>(in) % 16 == 0 && reinterpret_cast<uintptr_t>(out) % 16 == 0 && HW % 16 == 0 &&
         B * ((HW + kChunkPx - 1) / kChunkPx) < (1LL << 31) && B * (int64_t)H < (1LL << 31);
}

size_t fused_smem_bytes() { return kFusedSmem; }

cudaError_t launch_fused(FusedArgs a, int grid, cudaStream_t st) {
  const int64_t HW = (int64_t)a.H * a.W;
  a.cpi = (uint32_t)((HW + kChunkPx - 1) / kChunkPx);
  if (a.GS < 1) a.GS = 8;
  if (a.KB < 1) a.KB = 1;
  if (a.KB > a.H) a.KB = a.H;
  if (grid < 1) grid = 1;
  const uintptr_t p = reinterpret_cast<uintptr_t>(a.in);
  if (p % 16 == 0 && a.W % 16 == 0) return launch_fv<16, 16>(a, grid, st);
  if (p % 8 == 0 && a.W % 8 == 0 && a.W >= 16) return launch_fv<16, 8>(a, grid, st);
  if (p % 8 == 0 && a.W % 8 == 0) return launch_fv<8, 8>(a, grid, st);
  return launch_fv<16, 1>(a, grid, st);
}

}  // namespace hr

#ifdef HR_FUSED_TRACE
// measurement-only export of the fused-kernel timeline (trace builds; not part of histretinex.h)
extern "C" int hr_debug_fused_trace(void* out, int max_recs) {
  unsigned n = 0;
  if (cudaMemcpyFromSymbol(&n, hr::g_ntrace, sizeof(unsigned)) != cudaSuccess) return -1;
  if (n > hr::kTraceCap) n = hr::kTraceCap;
  if ((int)n > max_recs) n = (unsigned)max_recs;
  if (n && cudaMemcpyFromSymbol(out, hr::g_trace, sizeof(hr::TraceRec) * n) != cudaSuccess) return -1;
  const unsigned zero = 0;
  cudaMemcpyToSymbol(hr::g_ntrace, &zero, sizeof(unsigned));
  return (int)n;
}
#endif
