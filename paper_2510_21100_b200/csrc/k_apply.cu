// k_apply.cu -- kernel (d): streaming LUT application + colour reconstruction.
//
// The LUT application of hr_apply and hr_enhance; the helpers are in apply_dev.cuh.
// P:308 ("we utilize the histogram matching to estimate the enhanced image") and P:59
// (S is the HSV value channel): V = max(R,G,B), V' = LUT[V]; replacing V in hexcone HSV
// scales every channel by V'/V (reading R17), rounded half up:
//     out_c = floor((2 c V' + V) / (2 V)),  V = 0 -> (V', V', V').
// The streaming kernel evaluates it in fp32, out_c = rn(c alpha + beta) with alpha = fl(V'/V) and
// beta = fl(1/(4V)) per level (exact: apply_dev.cuh); the scalar fallback kernel in integers,
// out_c = umulhi(c * e + V, M[V]) + (e >> 16), e = 2 LUT[V], M = floor(2^32 / (2V)) + 1.
//
// B200 design: every warp runs its own TMA bulk-copy pipeline over 1024-pixel chunks
// (3,072 B): cp.async.bulk global->smem completes on a per-stage mbarrier, the 32 lanes
// transform the chunk in place as two 512-px sub-blocks (lane l owns 16 px of each: three
// conflict-free 16-B LDS/STS at a 48-B lane stride), and cp.async.bulk smem->global writes whole
// lines back -- no partial-sector stores (the v1 per-thread 48-B STG pattern sent 1.4x the
// bytes to L2).  Per pixel one 8-B LDS fetches (alpha, beta) from a per-warp table rebuilt when
// the warp's chunk changes image, so warps never synchronise with each other.  Chunks never
// straddle images; images whose pixel count is not a multiple of 16 (or unaligned buffers) take
// the scalar fallback kernel.
#include "apply_dev.cuh"

namespace hr {
namespace {

__global__ void __launch_bounds__(kApplyThreads, 2)
k_apply_tma(const uint8_t* __restrict__ in, const uint8_t* __restrict__ lut, int64_t B, int64_t HW,
            uint8_t* __restrict__ out, const uint32_t* __restrict__ ready, int64_t b_last,
            uint32_t* __restrict__ ticket, uint32_t GS) {
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
  const uint32_t GA = GA0, GB = GB0;
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

  // A chunk cursor: image b and chunk li within it.  A warp's chunks are kWarps apart, so a cursor
  // advances by an add and a compare (no division per chunk); every lane keeps the same cursors
  // and counters (warp-uniform bookkeeping), lane 0 alone issues the bulk copies.
  struct Cur {
    uint32_t b, li;
  };
  auto cur_at = [&](uint32_t g) {
    Cur c;
    c.b = g / cpi;
    c.li = g - c.b * cpi;
    return c;
  };
  auto cur_step = [&](Cur& c) {
    c.li += (uint32_t)kWarps;
    while (c.li >= cpi) {
      c.li -= cpi;
      ++c.b;
    }
  };
  auto span = [&](const Cur& c, uint64_t& off, uint32_t& bytes) {
    const uint32_t px0 = c.li * kChunkPx;
    const uint32_t npx = min((uint32_t)kChunkPx, (uint32_t)(HW - px0));
    off = ((uint64_t)c.b * (uint64_t)HW + px0) * 3u;
    bytes = npx * 3u;
  };
  auto issue = [&](const Cur& c) {  // every lane: the stage bookkeeping; lane 0: the copy
    uint64_t off;
    uint32_t bytes;
    span(c, off, bytes);
    const int st = (int)(nIss % kStages);
    if (lane == 0) {
      mbar_expect_tx(&s.bar[w][st], bytes);
      bulk_load(s.stage[w][st], in + off, bytes, &s.bar[w][st], pol);
    }
    ++nIss;
  };
  // this warp's per-chunk pipeline over two runs of chunks: gA, gA + kWarps, ... (nA_ chunks),
  // then gB, gB + kWarps, ... (nB_ chunks)
  auto pipeline = [&](uint32_t gA, int nA_, uint32_t gB, int nB_) {
    const int count = nA_ + nB_;
    if (count <= 0) return;
    Cur ci = cur_at(nA_ > 0 ? gA : gB), cc = ci;  // issue cursor (kAhead ahead), compute cursor
    int ii = 0;                                   // index of the issue cursor's chunk
    auto advance = [&](Cur& c, int& idx) {
      ++idx;
      if (idx == nA_ && nB_ > 0)
        c = cur_at(gB);
      else
        cur_step(c);
    };
    for (int i = 0; i < min(kAhead, count); ++i) {
      issue(ci);
      advance(ci, ii);
    }
    for (int i = 0; i < count;) {
      uint64_t off;
      uint32_t bytes;
      span(cc, off, bytes);
      const uint32_t b = cc.b;
      if ((int64_t)b != cur_img) {  // per-warp LUT table for this image
        __syncwarp();
        if (ready && lane == 0) wait_flag_geq(ready + b, 1u, 100);
        __syncwarp();
        build_tab(tab, lut + (uint64_t)b * kLevels, lane);
        __syncwarp();
        cur_img = b;
      }
      // prefetch chunk i + kAhead into the stage of chunk i - 2, whose bulk store (committed
      // two iterations ago) has finished reading shared memory once all but the latest
      // store group have
      if (ii < count) {
        if (lane == 0 && nComp >= 2) bulk_wait_read<1>();
        issue(ci);
        advance(ci, ii);
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
      advance(cc, i);
    }
    if (lane == 0) bulk_wait_read<0>();  // the stages are free for the next call's prologue
    __syncwarp();
  };

  // round 0: the static shares (part A, then -- without tickets -- part B); further rounds: part B
  // by CTA tickets.  One call site, so the pipeline body exists once in the kernel (the code of a
  // step timed after an L2 flush is fetched from DRAM).
  const uint32_t CT = (uint32_t)kWarps * GS, nT = dynB ? (GB + CT - 1) / CT : 0u;
  for (int round = 0;; ++round) {
    uint32_t gA_ = a0 + (uint32_t)w, gB_ = c0 + (uint32_t)w;
    int nA_ = nA, nB_ = cnt(c0, c1);
    if (round > 0) {
      if (!dynB) break;
      __syncthreads();
      if (tid == 0) tk_s = atomicAdd(ticket, 1u);
      __syncthreads();
      const uint32_t t = tk_s;
      if (t >= nT) break;
      const uint32_t lo = GA + t * CT, hi = min(GA + GB, lo + CT);
      gA_ = lo + (uint32_t)w;
      nA_ = cnt(lo, hi);
      gB_ = 0u;
      nB_ = 0;
    }
    pipeline(gA_, nA_, gB_, nB_);
  }
  if (lane == 0) bulk_wait<0>();
  TRACE_END(4u, 0u, 0ull);
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

cudaError_t trace_bind_apply(void* buf, uint32_t* n, uint32_t cap) { return trace_bind_tu(buf, n, cap); }

cudaError_t init_attrs_apply() {
  cudaError_t e = cudaFuncSetAttribute(k_apply_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(ApplySmem));
  // the whole carve-out: without it the driver may configure less shared memory than two CTAs
  // need, halving the resident warps (measured 1.5x slower)
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_apply_tma, cudaFuncAttributePreferredSharedMemoryCarveout,
                             (int)cudaSharedmemCarveoutMaxShared);
  return e;
}

cudaError_t launch_apply(const uint8_t* in, const uint8_t* lut, int64_t B, int32_t H, int32_t W, uint8_t* out,
                         int grid_ctas, cudaStream_t st, const uint32_t* ready, int64_t b_last, uint32_t* ticket,
                         int GS) {
  const int64_t HW = (int64_t)H * W;
  const bool tma = (reinterpret_cast<uintptr_t>(in) % 16 == 0) && (reinterpret_cast<uintptr_t>(out) % 16 == 0) &&
                   (HW % 16 == 0) && B * ((HW + kChunkPx - 1) / kChunkPx) < (1LL << 31);
  if (tma) {
    const int64_t chunks = B * ((HW + kChunkPx - 1) / kChunkPx);
    int64_t grid = grid_ctas;
    if (grid > (chunks + kWarps - 1) / kWarps) grid = (chunks + kWarps - 1) / kWarps;
    if (grid < 1) grid = 1;
    return launch_pdl(k_apply_tma, dim3((unsigned)grid), dim3(kApplyThreads), sizeof(ApplySmem), st, in, lut, B, HW,
                      out, ready, b_last, ticket, (uint32_t)(GS < 1 ? 1 : GS));
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
