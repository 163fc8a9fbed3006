// k_apply.cu -- kernel (d): streaming LUT application + colour reconstruction.
//
// Standalone launch of the LUT application (hr_apply, serial / chunk-pipelined hr_enhance);
// the helpers are in apply_dev.cuh.
// P:308 ("we utilize the histogram matching to estimate the enhanced image") and P:59
// (S is the HSV value channel): V = max(R,G,B), V' = LUT[V]; replacing V in hexcone HSV
// scales every channel by V'/V (reading R17), rounded half up:
//     out_c = floor((2 c V' + V) / (2 V)),  V = 0 -> (V', V', V').
// Exact integer form: out_c = umulhi(c * e + V, M[V]) + (e >> 16) with the per-level entry
//     V >= 1: e = 2 LUT[V],  M = floor(2^32 / (2V)) + 1   (exact for every numerator <= 130305)
//     V == 0: e = LUT[0] << 16 (then c = 0, the numerator is 0 and the addend gives LUT[0]),
// i.e. one IMAD and one IMAD.HI (with addend) per channel.
//
// B200 design: every warp runs its own TMA bulk-copy pipeline over 512-pixel chunks
// (1,536 B): cp.async.bulk global->smem completes on a per-stage mbarrier, the 32 lanes
// transform their 16 pixels in place (three conflict-free 16-B LDS/STS at a 48-B lane
// stride), and cp.async.bulk smem->global writes whole lines back -- no partial-sector
// stores (the v1 per-thread 48-B STG pattern sent 1.4x the bytes to L2).  M lives in a
// lane-private table (word 32v + lane: conflict-free), (A | Bv << 16) in a per-warp table
// rebuilt when the warp's chunk changes image, so warps never synchronise with each other.
// Chunks never straddle images; images whose pixel count is not a multiple of 16 (or
// unaligned buffers) take the scalar fallback kernel.
#include "apply_dev.cuh"

namespace hr {
namespace {

__global__ void __launch_bounds__(kApplyThreads, 2)
k_apply_tma(const uint8_t* __restrict__ in, const uint8_t* __restrict__ lut, int64_t B, int64_t HW,
            uint8_t* __restrict__ out, const uint32_t* __restrict__ ready, int64_t b_last,
            uint32_t* __restrict__ ticket, uint32_t GS, uint32_t tail_pct) {
  extern __shared__ __align__(128) unsigned char smraw[];
  ApplySmem& s = *reinterpret_cast<ApplySmem*>(smraw);
  __shared__ uint32_t tk_s;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  TRACE_T0();
  if (!ready) pdl_wait();  // with per-image flags only the LUTs depend on the solver grid
  pdl_trigger();
  if (lane == 0) {
    for (int k = 0; k < kStages; ++k) mbar_init(&s.bar[w][k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const uint32_t cpi = (uint32_t)((HW + kChunkPx - 1) / kChunkPx);  // chunks per image
  // chunk space in two parts: images [0, b_last) then [b_last, B) (b_last = B: one part); this
  // CTA takes a contiguous share of each part, part A first.  With `ticket`, part B is not
  // split statically: the CTA takes tickets of kWarps * GS contiguous chunks of it (all warps of
  // the CTA stream a ticket together, warp w taking chunks w, w + kWarps, ...), so CTAs that
  // started late or run beside a solver CTA take fewer
  if (b_last <= 0 || b_last > B) b_last = B;
  const uint32_t GA0 = (uint32_t)(b_last * (int64_t)cpi), GB0 = (uint32_t)(B * (int64_t)cpi) - GA0;  // < 2^31
  const bool dynB = ticket != nullptr && GB0 > 0;
  // with tickets, the last tail_pct % of part A joins the ticketed part (natural order)
  const uint32_t GA = dynB ? GA0 - (uint32_t)((uint64_t)GA0 * min(tail_pct, 100u) / 100u) : GA0;
  const uint32_t GB = GA0 + GB0 - GA;
  const uint32_t a0 = (uint32_t)((uint64_t)GA * blockIdx.x / gridDim.x), a1 = (uint32_t)((uint64_t)GA * (blockIdx.x + 1) / gridDim.x);
  const uint32_t c0 = GA + (dynB ? 0u : (uint32_t)((uint64_t)GB * blockIdx.x / gridDim.x));
  const uint32_t c1 = GA + (dynB ? 0u : (uint32_t)((uint64_t)GB * (blockIdx.x + 1) / gridDim.x));
  // this warp's chunks: a0 + w, a0 + w + kWarps, ... < a1, then c0 + w, ... < c1
  auto cnt = [&](uint32_t lo, uint32_t hi) { return (hi - lo > (uint32_t)w) ? (int)((hi - lo - w + kWarps - 1) / kWarps) : 0; };
  const int nA = cnt(a0, a1);
  const uint64_t pol = policy_evict_first();
  uint2* tab = s.tab[w];
  int64_t cur_img = -1;
  uint32_t nIss = 0, nComp = 0;  // chunks issued / computed by this warp so far (stage and parity)

  auto where = [&](uint32_t g, uint64_t& off, uint32_t& bytes, uint32_t& b) {
    b = g / cpi;
    const uint32_t px0 = (g - b * cpi) * kChunkPx;
    const uint32_t npx = min((uint32_t)kChunkPx, (uint32_t)(HW - px0));
    off = ((uint64_t)b * (uint64_t)HW + px0) * 3u;
    bytes = npx * 3u;
  };
  auto issue = [&](uint32_t g) {  // lane 0
    uint64_t off;
    uint32_t bytes, b;
    where(g, off, bytes, b);
    const int st = (int)(nIss % kStages);
    mbar_expect_tx(&s.bar[w][st], bytes);
    bulk_load(s.stage[w][st], in + off, bytes, &s.bar[w][st], pol);
    ++nIss;
  };
  // this warp's per-chunk pipeline over `count` chunks, chunk i = global chunk index chunk(i)
  auto pipeline = [&](int count, auto&& chunk) {
    if (lane == 0)
      for (int i = 0; i < min(kAhead, count); ++i) issue(chunk(i));
    for (int i = 0; i < count; ++i) {
      uint64_t off;
      uint32_t bytes, b;
      where(chunk(i), off, bytes, b);
      if ((int64_t)b != cur_img) {  // per-warp LUT table for this image
        __syncwarp();
        if (ready && lane == 0)
          while (ld_acquire(ready + b) == 0u) __nanosleep(100);
        __syncwarp();
        build_tab(tab, lut + (uint64_t)b * kLevels, lane);
        __syncwarp();
        cur_img = b;
      }
      // prefetch chunk i + kAhead into the stage of chunk i - 2, whose bulk store (committed
      // two iterations ago) has finished reading shared memory once all but the latest
      // store group have
      if (lane == 0 && i + kAhead < count) {
        if (nComp >= 2) bulk_wait_read<1>();
        issue(chunk(i + kAhead));
      }
      HR_CHECK(bytes > 0 && bytes <= (uint32_t)kChunkBytes && bytes % 48 == 0 && off + bytes <= (uint64_t)B * HW * 3);
      const int st = (int)(nComp % kStages);
      mbar_wait(&s.bar[w][st], (nComp / kStages) & 1u);
      uint8_t* p = s.stage[w][st];
      apply_chunk_smem(p, bytes, tab, lane);
      fence_async_smem();
      __syncwarp();
      if (lane == 0) {
        bulk_store(out + off, p, bytes, pol);
        bulk_commit();
      }
      ++nComp;
    }
    if (lane == 0) bulk_wait_read<0>();  // the stages are free for the next call's prologue
    __syncwarp();
  };

  // static shares: part A, then (without tickets) part B
  pipeline(nA + cnt(c0, c1), [&](int i) {
    return i < nA ? a0 + (uint32_t)w + (uint32_t)i * kWarps : c0 + (uint32_t)w + (uint32_t)(i - nA) * kWarps;
  });
  if (dynB) {  // part B by CTA tickets
    const uint32_t CT = (uint32_t)kWarps * GS, nT = (GB + CT - 1) / CT;
    for (;;) {
      __syncthreads();
      if (tid == 0) tk_s = atomicAdd(ticket, 1u);
      __syncthreads();
      const uint32_t t = tk_s;
      if (t >= nT) break;
      const uint32_t lo = GA + t * CT, hi = min(GA + GB, lo + CT);
      pipeline(cnt(lo, hi), [&](int i) { return lo + (uint32_t)w + (uint32_t)i * kWarps; });
    }
  }
  if (lane == 0) bulk_wait<0>();
  TRACE_END(4u, 0u, 0ull);
}

// ---------------------------------------------------------------- dynamic (ticketed) apply
// The same per-warp TMA pipeline, fed by tickets over (image position, group of GS chunks),
// each warp's next ticket fetched while it works on the current one.  With a completion queue
// the loader lane acquires queue[pos] (k_solve released it after writing that image's LUT), so
// warps always work on images whose LUT is done and the apply starts with the first finished
// solve; without one (queue == NULL) images go in natural order after the whole solver grid
// (griddepcontrol.wait) -- the tickets then only balance the streaming work across warps
// whatever their start times (CTAs that become resident late take fewer tickets).  Each new image's LUT is loaded into registers when its first chunk is issued
// (kAhead chunks before it is computed).  Deadlock-free: launched (PDL) only once every solver
// CTA is resident, and each solve fills one queue slot.
struct DynSmem {
  static constexpr int kRing = 4;
  uint2 meta[kWarps][kStages];
  uint32_t ring_t[kRing];
  int ring_tag[kRing], ring_read[kWarps], ring_claim;
};

__global__ void __launch_bounds__(kApplyThreads, 2)
k_apply_dyn(const uint8_t* __restrict__ in, const uint8_t* __restrict__ lut, int64_t B, int64_t HW,
            uint8_t* __restrict__ out, const uint32_t* __restrict__ queue, uint32_t* __restrict__ ticket, uint32_t GS,
            const uint32_t* __restrict__ ready, int64_t b_last) {
  extern __shared__ __align__(128) unsigned char smraw[];
  ApplySmem& s = *reinterpret_cast<ApplySmem*>(smraw);
  // all shared memory is dynamic: a static block before it would push the 128-B aligned
  // dynamic block to the next 1 KB and leave room for only one CTA per SM
  DynSmem& x = *reinterpret_cast<DynSmem*>(smraw + sizeof(ApplySmem));
  auto& meta = x.meta;  // (image, chunk) of each stage, image = kEndImg: end
  constexpr uint32_t kEndImg = 0xFFFFFFFFu;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  TRACE_T0();
  // with the completion queue there is no grid-wide wait: LUTs arrive through the queue; with
  // per-image ready flags (natural order) each image's LUT is acquired before its first group;
  // with neither every LUT is read after the solver grid has completed
  if (!queue && !ready) pdl_wait();
  pdl_trigger();
  if (lane == 0) {
    for (int k = 0; k < kStages; ++k) mbar_init(&s.bar[w][k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t cpi = (uint32_t)((HW + kChunkPx - 1) / kChunkPx);
  const uint32_t gpi = (cpi + GS - 1) / GS;
  // hybrid form (0 < b_last < B, natural order with ready flags): images [0, b_last) are split
  // statically (this CTA's contiguous share, its warps interleaved chunk by chunk, as in
  // k_apply_tma) and only images [b_last, B) go by tickets, so CTAs that became resident late
  // or run slower take fewer of them
  if (queue || b_last <= 0 || b_last > B) b_last = 0;
  const uint32_t GA = (uint32_t)(b_last * (int64_t)cpi);
  const uint32_t a0 = (uint32_t)((uint64_t)GA * blockIdx.x / gridDim.x), a1 = (uint32_t)((uint64_t)GA * (blockIdx.x + 1) / gridDim.x);
  const uint32_t nA = (a1 - a0 > (uint32_t)w) ? (a1 - a0 - w + kWarps - 1) / kWarps : 0u;
  uint32_t sA = 0;  // static chunks issued so far
  const uint64_t ngroups = (uint64_t)(B - b_last) * gpi;
  // hybrid form, part B: CTA tickets of kWarps * GS contiguous chunks (all warps of the CTA
  // stream one ticket together, warp w taking chunks w, w + kWarps, ... as in the static part:
  // per-warp tickets scatter the DRAM streams and measured far slower).  The CTA's k-th ticket
  // is fetched by the first warp that needs it and published in a ring of kRing slots; a slot
  // is refilled only after every warp has read its previous ticket (no lag limit otherwise).
  constexpr int kRing = DynSmem::kRing;
  uint32_t* ring_t = x.ring_t;
  int *ring_tag = x.ring_tag, *ring_read = x.ring_read;
  int& ring_claim = x.ring_claim;
  const uint32_t GB = (uint32_t)((B - b_last) * (int64_t)cpi), CT = (uint32_t)kWarps * GS;
  const uint32_t nT = (GB + CT - 1) / CT;
  if (tid < kRing) ring_tag[tid] = -1;
  if (tid < kWarps) ring_read[tid] = 0;
  if (tid == 0) ring_claim = 0;
  __syncthreads();
  int tix = -1;           // CTA ticket index this warp is on
  uint32_t tcur = 0, tm = GS;  // its global ticket, chunks taken from it
  auto cta_ticket = [&](int i) -> uint32_t {  // lane 0: the CTA's i-th ticket
    volatile int* tag = ring_tag;
    volatile uint32_t* rt = ring_t;
    for (;;) {
      if (tag[i % kRing] == i) break;
      if (*(volatile int*)&ring_claim == i && atomicCAS(&ring_claim, i, i + 1) == i) {
        for (bool ok = false; !ok;) {  // every warp has read ticket i - kRing (slot free)
          ok = true;
          for (int u = 0; u < kWarps; ++u) ok = ok && ((volatile int*)ring_read)[u] > i - kRing;
        }
        rt[i % kRing] = atomicAdd(ticket, 1u);
        __threadfence_block();
        tag[i % kRing] = i;
        break;
      }
      __nanosleep(20);
    }
    const uint32_t t = rt[i % kRing];
    __threadfence_block();
    ((volatile int*)ring_read)[w] = i + 1;
    return t;
  };
  const uint64_t pol = policy_evict_first();
  uint2* tab = s.tab[w];
  // loader state (lane 0): image and chunk range of the current group, prefetched next ticket
  uint32_t lb = 0, lc = 0, le = 0, nxt = 0, rd_img = kEndImg;
  if (lane == 0 && b_last == 0) nxt = atomicAdd(ticket, 1u);
  auto next_chunk = [&](uint32_t& b, uint32_t& c) -> bool {
    if (sA < nA) {  // static part
      const uint32_t g = a0 + (uint32_t)w + sA * kWarps;
      ++sA;
      b = g / cpi;
      c = g - b * cpi;
      if (ready && b != rd_img) {
        while (ld_acquire(ready + b) == 0u) __nanosleep(100);
        rd_img = b;
      }
      return true;
    }
    if (b_last > 0) {  // part B: CTA tickets
      for (;;) {
        if (tm >= GS) {
          tcur = cta_ticket(++tix);
          tm = 0;
        }
        if (tcur >= nT) {
          ((volatile int*)ring_read)[w] = 1 << 30;  // never blocks a refill again
          return false;
        }
        const uint32_t g = tcur * CT + (uint32_t)w + tm * kWarps;
        ++tm;
        if (g >= GB) {
          tm = GS;
          continue;
        }
        b = (uint32_t)b_last + g / cpi;
        c = g % cpi;
        break;
      }
      if (ready && b != rd_img) {
        while (ld_acquire(ready + b) == 0u) __nanosleep(100);
        rd_img = b;
      }
      return true;
    }
    if (lc >= le) {
      if (nxt >= ngroups) return false;
      const uint32_t q = (uint32_t)b_last + nxt / gpi, g = nxt % gpi;
      if (queue) {
        uint32_t v;
        while ((v = ld_acquire(queue + q)) == 0u) __nanosleep(100);
        lb = v - 1u;
      } else {
        lb = q;
        if (ready && q != rd_img) {  // natural order gated by the image's LUT-ready flag
          while (ld_acquire(ready + q) == 0u) __nanosleep(100);
          rd_img = q;
        }
      }
      lc = g * GS;
      le = min(lc + GS, cpi);
      nxt = atomicAdd(ticket, 1u);
    }
    b = lb;
    c = lc++;
    return true;
  };
  uint32_t ld_img = kEndImg, pend_img = kEndImg;
  uint2 pend = make_uint2(0u, 0u);
  auto issue = [&](uint32_t i) {  // all lanes; lane 0 fills stage i % kStages
    const int st = (int)(i % kStages);
    uint32_t b = kEndImg, c = 0;
    if (lane == 0 && !next_chunk(b, c)) b = kEndImg;
    b = __shfl_sync(0xffffffffu, b, 0);
    c = __shfl_sync(0xffffffffu, c, 0);
    __syncwarp();  // lane 0's queue acquire before the other lanes read this image's LUT
    if (lane == 0) meta[w][st] = make_uint2(b, c);
    if (b == kEndImg) {
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&s.bar[w][st])) : "memory");
      return;
    }
    if (b != ld_img) {
      ld_img = b;
      if (pend_img == kEndImg) {
        pend = __ldcg(reinterpret_cast<const uint2*>(lut + (uint64_t)b * kLevels) + lane);
        pend_img = b;
      }
    }
    if (lane == 0) {
      const uint32_t px0 = c * kChunkPx, npx = min((uint32_t)kChunkPx, (uint32_t)(HW - px0));
      const uint64_t off = ((uint64_t)b * (uint64_t)HW + px0) * 3u;
      mbar_expect_tx(&s.bar[w][st], npx * 3u);
      bulk_load(s.stage[w][st], in + off, npx * 3u, &s.bar[w][st], pol);
    }
  };
  for (uint32_t i = 0; i < (uint32_t)kAhead; ++i) issue(i);
  uint32_t cur_img = kEndImg;
  int st = 0;
  uint32_t ph = 0;
  for (uint32_t i = 0;; ++i) {
    if (lane == 0 && i >= 2) bulk_wait_read<1>();
    __syncwarp();
    issue(i + kAhead);
    mbar_wait(&s.bar[w][st], ph);
    const uint2 m = meta[w][st];
    if (m.x == kEndImg) break;  // warp-uniform
    const uint32_t b = m.x, px0 = m.y * kChunkPx;
    const uint32_t bytes = min((uint32_t)kChunkPx, (uint32_t)(HW - px0)) * 3u;
    const uint64_t off = ((uint64_t)b * (uint64_t)HW + px0) * 3u;
    HR_CHECK(b < B && bytes > 0 && bytes <= (uint32_t)kChunkBytes);
    if (b != cur_img) {
      __syncwarp();
      if (b == pend_img) {
        build_tab_regs(tab, pend, lane);
        pend_img = kEndImg;
      } else {
        build_tab(tab, lut + (uint64_t)b * kLevels, lane);  // queue order implies the LUT is done
      }
      __syncwarp();
      cur_img = b;
    }
    uint8_t* p = s.stage[w][st];
    apply_chunk_smem(p, bytes, tab, lane);
    fence_async_smem();
    __syncwarp();
    if (lane == 0) {
      bulk_store(out + off, p, bytes, pol);
      bulk_commit();
    }
    if (++st == kStages) {
      st = 0;
      ph ^= 1u;
    }
  }
  if (lane == 0) bulk_wait<0>();
  TRACE_END(5u, 0u, 0ull);
}

// ---------------------------------------------------------------- scalar fallback
__device__ __forceinline__ void apply_scalar(const uint8_t* __restrict__ in, uint8_t* __restrict__ out, int64_t q,
                                             const uint32_t* ab) {
  const uint32_t r = in[3 * q], g = in[3 * q + 1], b = in[3 * q + 2];
  const uint32_t v = __vimax3_u32(r, g, b);
  const uint32_t e = ab[v], M = magic_of((int)v), F = e >> 16;
  out[3 * q] = (uint8_t)chan(r, e, v, M, F);
  out[3 * q + 1] = (uint8_t)chan(g, e, v, M, F);
  out[3 * q + 2] = (uint8_t)chan(b, e, v, M, F);
}

__global__ void __launch_bounds__(kApplyThreads)
k_apply_scalar(const uint8_t* __restrict__ in, const uint8_t* __restrict__ lut, int64_t B, int64_t HW,
               uint8_t* __restrict__ out) {
  __shared__ uint32_t ab[kLevels];
  const int tid = threadIdx.x;
  const int64_t P = B * HW;
  const int64_t q0 = P * blockIdx.x / gridDim.x, q1 = P * (blockIdx.x + 1) / gridDim.x;
  for (int64_t q = q0; q < q1;) {
    const int64_t b = q / HW;
    const int64_t qe = min(q1, (b + 1) * HW);
    __syncthreads();
    ab[tid] = ab_of(tid, lut[b * kLevels + tid]);
    __syncthreads();
    for (int64_t p = q + tid; p < qe; p += kApplyThreads) apply_scalar(in, out, p, ab);
    q = qe;
  }
}

}  // namespace

void trace_bind_apply(void* buf, uint32_t* n, uint32_t cap) {
#ifdef HR_STEP_TRACE
  trace_bind_tu(buf, n, cap);
#else
  (void)buf, (void)n, (void)cap;
#endif
}

bool apply_dyn_supported(const uint8_t* in, const uint8_t* out, int64_t B, int32_t H, int32_t W) {
  const int64_t HW = (int64_t)H * W;
  return reinterpret_cast<uintptr_t>(in) % 16 == 0 && reinterpret_cast<uintptr_t>(out) % 16 == 0 && HW % 16 == 0 &&
         B * ((HW + kChunkPx - 1) / kChunkPx) < (1LL << 31);
}

cudaError_t launch_apply_dyn(const uint8_t* in, const uint8_t* lut, int64_t B, int32_t H, int32_t W, uint8_t* out,
                             int grid_ctas, const uint32_t* queue, uint32_t* ticket, int GS, cudaStream_t st,
                             const uint32_t* ready, int64_t b_last) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_apply_dyn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(sizeof(ApplySmem) + sizeof(DynSmem)));
    // the whole carve-out: without it the driver may configure less shared memory than two
    // CTAs need, halving the resident warps (measured 1.5x slower)
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_apply_dyn, cudaFuncAttributePreferredSharedMemoryCarveout,
                               (int)cudaSharedmemCarveoutMaxShared);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int64_t HW = (int64_t)H * W;
  return launch_pdl(k_apply_dyn, dim3((unsigned)(grid_ctas < 1 ? 1 : grid_ctas)), dim3(kApplyThreads),
                    sizeof(ApplySmem) + sizeof(DynSmem), st, in, lut, B, HW, out, queue, ticket, (uint32_t)(GS < 1 ? 1 : GS), ready, b_last);
}

cudaError_t launch_apply(const uint8_t* in, const uint8_t* lut, int64_t B, int32_t H, int32_t W, uint8_t* out,
                         int grid_ctas, cudaStream_t st, const uint32_t* ready, int64_t b_last, uint32_t* ticket,
                         int GS, int tail_pct) {
  const int64_t HW = (int64_t)H * W;
  const bool tma = (reinterpret_cast<uintptr_t>(in) % 16 == 0) && (reinterpret_cast<uintptr_t>(out) % 16 == 0) &&
                   (HW % 16 == 0) && B * ((HW + kChunkPx - 1) / kChunkPx) < (1LL << 31);
  if (tma) {
    static bool attr = false;
    if (!attr) {
      cudaError_t e = cudaFuncSetAttribute(k_apply_tma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)sizeof(ApplySmem));
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_apply_tma, cudaFuncAttributePreferredSharedMemoryCarveout,
                                 (int)cudaSharedmemCarveoutMaxShared);
      if (e != cudaSuccess) return e;
      attr = true;
    }
    const int64_t chunks = B * ((HW + kChunkPx - 1) / kChunkPx);
    int64_t grid = grid_ctas;
    if (grid > (chunks + kWarps - 1) / kWarps) grid = (chunks + kWarps - 1) / kWarps;
    if (grid < 1) grid = 1;
    return launch_pdl(k_apply_tma, dim3((unsigned)grid), dim3(kApplyThreads), sizeof(ApplySmem), st, in, lut, B, HW,
                      out, ready, b_last, ticket, (uint32_t)(GS < 1 ? 1 : GS), (uint32_t)(tail_pct < 0 ? 0 : tail_pct));
  } else {
    int64_t grid = 4LL * grid_ctas;
    const int64_t P = B * HW;
    if (grid > (P + kApplyThreads - 1) / kApplyThreads) grid = (P + kApplyThreads - 1) / kApplyThreads;
    if (grid < 1) grid = 1;
    k_apply_scalar<<<(unsigned)grid, kApplyThreads, 0, st>>>(in, lut, B, HW, out);
  }
  return cudaGetLastError();
}

}  // namespace hr
