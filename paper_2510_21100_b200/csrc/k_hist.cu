// k_hist.cu -- kernel (a): fused colour convert + gradient + privatised histograms.
//
// PAPER.md Alg. 1 lines "Compute the histogram of the low-light image H_C(S)" and
// "Compute the histogram of the gradient image H_C(grad S)", Eq. 3.
// The per-segment device body (value channel, gradient, lane-private counters, flush) is in
// hist_dev.cuh; this kernel is the standalone launch used by hr_histogram and the serial /
// chunk-pipelined hr_enhance paths.
//
// Design (B200): persistent grid of 2 CTAs/SM x 512 threads.  Each CTA owns a contiguous
// range of global rows (all images concatenated), split at image boundaries into segments;
// one flush per (CTA, image) segment with global integer atomics -> exact, deterministic.
#include <algorithm>
#include <cstdlib>

#include "apply_dev.cuh"  // mbarrier / bulk-copy PTX wrappers
#include "hist_dev.cuh"

namespace hr {
namespace {

// ---------------------------------------------------------------- TMA-staged form (default)
// The same per-pixel arithmetic and lane-private counters as hist_segment (hist_dev.cuh), but
// the pixels reach the threads through shared memory: each warp runs its own cp.async.bulk
// pipeline (KST stages) over the rows its 32 strips walk.  A thread's 16-px (or 8-px) strip is
// 48 (24) contiguous bytes, so direct per-thread vector loads from global memory touch 12
// distinct 128-B lines per warp instruction (3x the lines of the bytes moved); staged by TMA,
// the same bytes arrive as whole lines and the lanes read them with conflict-free 16-B (8-B)
// shared loads at a 48-B (24-B) lane stride.
//
// Layout: 1 CTA per SM x 1024 threads.  Thread t owns strip s = t % SPf of row group
// g = t / SPf (SPf = W / SW full strips per row, W % SW == 0); group g walks the rows of its
// band [ya, yb) of the CTA's segment plus one halo row, keeping the previous row's packed V and
// dx in registers (dy needs no second read).  A warp's lanes cover <= 3 groups (SPf >= 16), so
// a warp step copies <= 3 row pieces (strips [s_lo, s_hi] of one row, + the 3 bytes of the
// right neighbour pixel when the piece does not end the row); lane k issues piece k.  Piece
// copies start at the 16-B aligned address at or below the piece (W % 16 == 8 rows alternate
// between 0 and 8 bytes of misalignment; the strips are then read with 8-B loads).
template <int SW, int NT_, int KST_>
struct HistTma {
  static constexpr int NT = NT_;                                  // threads per CTA (1 CTA per SM)
  static constexpr int kHTW = NT / 32;
  static constexpr int KST = KST_;                                // stages per warp
  static constexpr int kPieceSlack = 32;                          // alignment + neighbour bytes
  static constexpr int kStage = 32 * 3 * SW + 3 * (kPieceSlack + 16);  // <= 3 pieces per warp step
  static constexpr int kRing = KST * kStage;
  static constexpr int kSmem = kHistDevSmem + kHTW * kRing + kHTW * KST * 8;
  static_assert(kSmem <= 227 * 1024, "TMA histogram smem");
};
static_assert(HistTma<16, 1024, 3>::kSmem <= 227 * 1024, "TMA histogram smem");
static_assert(HistTma<16, 512, 5>::kSmem <= 227 * 1024, "TMA histogram smem");

// shared loads at a shared::cta address
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
// one strip row of SW px (3 SW / 4 words): SW = 16 -> three 16-B loads (16-B aligned), SW = 8 ->
// three 8-B loads (8-B aligned)
template <int SW>
__device__ __forceinline__ void lds_strip(uint32_t a, uint32_t (&w)[3 * SW / 4]) {
  if constexpr (SW == 16) {
#pragma unroll
    for (int i = 0; i < 3; ++i)
      asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(w[4 * i]), "=r"(w[4 * i + 1]), "=r"(w[4 * i + 2]), "=r"(w[4 * i + 3])
                   : "r"(a + 16u * i));
  } else {
#pragma unroll
    for (int i = 0; i < 3; ++i)
      asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(w[2 * i]), "=r"(w[2 * i + 1]) : "r"(a + 8u * i));
  }
}
__device__ __forceinline__ void mbar_expect_tx_s(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_s(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_load_s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(bar), "l"(pol)
      : "memory");
}

template <int SW, int NT, int KST_>
__device__ __forceinline__ void hist_segment_tma(const uint8_t* __restrict__ img, int H, int W, int y0, int y1,
                                                 uint32_t* sm, unsigned char* ring, uint64_t* bars, uint32_t& phase,
                                                 uint64_t pol, uint32_t* __restrict__ hist_s_b,
                                                 uint32_t* __restrict__ hist_graw_b) {
  using C = HistTma<SW, NT, KST_>;
  constexpr int G = SW / 4;
  constexpr int KST = C::KST;
  uint32_t* ghi = sm + kLevels * kSlotWords;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const uint32_t Lv = (uint32_t)lane * 4u;
  const uint32_t Lg = 128u + (uint32_t)lane * 4u;
  const uint32_t sb = (uint32_t)__cvta_generic_to_shared(sm);

  const int SPf = W / SW;              // full strips per row (W % SW == 0, 16 <= SPf <= NT)
  const int NG = NT / SPf;             // row groups
  const int nrows = y1 - y0;
  const int RPG = (nrows + NG - 1) / NG;
  const size_t rowBytes = (size_t)W * 3;
  const int t0 = warp * 32;            // first thread of this warp
  const int gfirst = t0 / SPf;

  // ---- this lane as a consumer: group, strip, band ----
  const int grp = tid / SPf, s = tid - grp * SPf;
  const int ya = y0 + grp * RPG;
  const int yb = min(y1, ya + RPG);
  const bool act = grp < NG && ya < yb;
  const int nr = act ? yb - ya : 0;
  const bool halo = act && yb < H;
  const bool rowEnd = s == SPf - 1;    // last pixel of the strip is x = W - 1 (no tail: W % SW == 0)
  // ---- piece of group g of this warp: strips [lo, hi], shared slot offset ----
  auto piece_lo = [&](int g) { return max(0, t0 - g * SPf); };
  auto piece_hi = [&](int g) { return min(SPf - 1, t0 + 31 - g * SPf); };
  auto slot_bytes = [&](int g) { return ((3 * SW * (piece_hi(g) - piece_lo(g) + 1) + 15) & ~15) + C::kPieceSlack; };
  int myslot = 0;
  for (int g = gfirst; g < grp && act; ++g) myslot += slot_bytes(g);
  const int mylo = act ? piece_lo(grp) : 0;
  // ---- this lane as an issuer: piece k = lane (group gfirst + lane) ----
  const int ig = gfirst + lane;
  const bool iss = lane < 3 && ig < NG && ig * SPf <= t0 + 31;
  int islot = 0;
  for (int g = gfirst; g < ig && iss; ++g) islot += slot_bytes(g);
  const int iya = y0 + ig * RPG;
  const int inr = iss ? max(0, min(y1, iya + RPG) - iya) : 0;
  const bool ihalo = inr > 0 && iya + inr < H;
  HR_CHECK(!iss || islot + slot_bytes(ig) <= C::kStage);
  // Everything per step is precomputed per parity of the step: rows it and it + 2 have the same
  // misalignment, so the copy of step it starts at ip[it & 1] + (it >> 1) * 2 rowBytes.
  const int ilast = inr > 0 ? inr - 1 + (ihalo ? 1 : 0) : -1;  // last step this lane copies
  const unsigned char* ip0 = img;
  const unsigned char* ip1 = img;
  uint32_t ib0 = 0u, ib1 = 0u;
  if (inr > 0) {
    const int ilo = piece_lo(ig), ihi = piece_hi(ig);
    auto piece = [&](int y, const unsigned char*& src, uint32_t& bytes) {
      const size_t a = (size_t)y * rowBytes + (size_t)(3 * SW) * ilo;
      const size_t e = (size_t)y * rowBytes + (size_t)(3 * SW) * (ihi + 1) + (ihi < SPf - 1 ? 3 : 0);  // + neighbour
      const uintptr_t A = reinterpret_cast<uintptr_t>(img + a) & ~(uintptr_t)15;
      const uintptr_t E = (reinterpret_cast<uintptr_t>(img + e) + 15) & ~(uintptr_t)15;
      src = reinterpret_cast<const unsigned char*>(A);
      bytes = (uint32_t)(E - A);
      HR_CHECK(bytes <= (uint32_t)(((3 * SW * (ihi - ilo + 1) + 15) & ~15) + C::kPieceSlack));
    };
    piece(iya, ip0, ib0);
    piece(iya + 1, ip1, ib1);
  }
  const size_t step2 = 2 * rowBytes;
  const uint32_t ring_s = smem_u32(ring), bar_s = smem_u32(bars);
  const uint32_t idst = ring_s + (uint32_t)islot;
  // consumer side: strip address in stage 0 for even / odd steps
  const int clast = act ? nr - 1 + (halo ? 1 : 0) : -1;  // last step this lane reads
  uint32_t cad0 = ring_s + (uint32_t)(myslot + 3 * SW * (s - mylo)), cad1 = cad0;
  if (SW == 8 && act) {
    cad0 += (uint32_t)(reinterpret_cast<uintptr_t>(img + (size_t)ya * rowBytes + 24 * mylo) & 15u);
    cad1 += (uint32_t)(reinterpret_cast<uintptr_t>(img + (size_t)(ya + 1) * rowBytes + 24 * mylo) & 15u);
  }

  // issue the copies of row step it into the stage at offset so (warp-uniform)
  auto issue = [&](int it, uint32_t so, uint32_t bar) -> bool {
    const uint32_t bytes = it <= ilast ? ((it & 1) ? ib1 : ib0) : 0u;
    const uint32_t total = __reduce_add_sync(0xffffffffu, bytes);
    if (total == 0u) return false;
    // tx-count may run ahead of the expect (it is signed); the phase cannot complete before
    // lane 0's arrival
    if (lane == 0) mbar_expect_tx_s(bar, total);
    if (bytes) {
      fence_async_smem();
      bulk_load_s(idst + so, ((it & 1) ? ip1 : ip0) + (size_t)(it >> 1) * step2, bytes, bar, pol);
    }
    return true;
  };

  uint32_t Vp[G], Dp[G];
#pragma unroll
  for (int q = 0; q < G; ++q) Vp[q] = Dp[q] = 0u;
  uint32_t armed = 0u;
#pragma unroll
  for (int k = 0; k < KST; ++k)
    if (k <= RPG && issue(k, (uint32_t)(k * C::kStage), bar_s + 8u * k)) armed |= 1u << k;
  int st = 0;
  uint32_t so = 0u;
  for (int it = 0; it <= RPG; ++it) {
    uint32_t wr[3 * G], nbr = 0u;
#pragma unroll
    for (int i = 0; i < 3 * G; ++i) wr[i] = 0u;
    if (armed & (1u << st)) {
      mbar_wait_s(bar_s + 8u * st, (phase >> st) & 1u);
      phase ^= 1u << st;
      if (it <= clast) {
        const uint32_t a = ((it & 1) ? cad1 : cad0) + so;
        lds_strip<SW>(a, wr);  // 16-B loads (48-B strips), else 8-B loads (24-B strips)
        if (!rowEnd) nbr = lds_u32(a + 3 * SW);
      }
    }
    armed &= ~(1u << st);
    __syncwarp();
    if (it + KST <= RPG && issue(it + KST, so, bar_s + 8u * st)) armed |= 1u << st;
    if (++st == KST) {
      st = 0;
      so = 0u;
    } else {
      so += (uint32_t)C::kStage;
    }
    // ---- the per-row arithmetic of hist_segment ----
    uint32_t Vc[G], Dc[G];
#pragma unroll
    for (int q = 0; q < G; ++q) Vc[q] = value4(wr[3 * q], wr[3 * q + 1], wr[3 * q + 2]);
    if (it < nr) {  // H_C(S), Eq. 3
#pragma unroll
      for (int q = 0; q < G; ++q) {
        sinc(sb, __byte_perm(Lv, Vc[q], 0x1140u));
        sinc(sb, __byte_perm(Lv, Vc[q], 0x1150u));
        sinc(sb, __byte_perm(Lv, Vc[q], 0x1160u));
        sinc(sb, __byte_perm(Lv, Vc[q], 0x1170u));
      }
    }
    const uint32_t nbV = nb_value<16>(nbr);
#pragma unroll
    for (int q = 0; q < G; ++q) Dc[q] = __vabsdiffu4(Vc[q], __funnelshift_r(Vc[q], q < G - 1 ? Vc[q + 1] : nbV, 8));
    if (rowEnd) Dc[G - 1] &= 0x00FFFFFFu;  // dx = 0 at x = W-1
    if (it > 0 && it <= nr) grad_row<G>(sb, ghi, Lg, Dp, Vp, Vc, it < nr || halo);
#pragma unroll
    for (int q = 0; q < G; ++q) {
      Vp[q] = Vc[q];
      Dp[q] = Dc[q];
    }
  }

  // ---------------- flush: one integer atomic per nonzero bin ----------------
  __syncthreads();
  for (int bin = tid; bin < 2 * kLevels; bin += NT) {
    if (bin < kLevels) {
      uint32_t sv = 0, sg = 0;
#pragma unroll 8
      for (int l = 0; l < 32; ++l) {
        const int o = bin * kSlotWords + ((l + bin) & 31);
        sv += sm[o];
        sg += sm[o + 32];
      }
      if (sv) atomicAdd(hist_s_b + bin, sv);
      if (sg) atomicAdd(hist_graw_b + bin, sg);
    } else {
      const uint32_t c = ghi[bin - kLevels];
      if (c) atomicAdd(hist_graw_b + bin, c);
    }
  }
  __syncthreads();
}

// MINB = 2 caps the 512-thread form at 64 registers: with done counts a solver CTA (256 threads
// x 128 registers) runs beside it.  Images are taken in waves of wave_imgs (hist_wave_images).
template <int SW, int NT, int KST, int MINB>
__global__ void __launch_bounds__(NT, MINB)
k_hist_tma(const uint8_t* __restrict__ rgb, int64_t B, int H, int W, uint32_t* __restrict__ hist_s,
           uint32_t* __restrict__ hist_graw, uint32_t* __restrict__ done, int64_t wave_imgs) {
  using C = HistTma<SW, NT, KST>;
  extern __shared__ __align__(16) uint32_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* ring = reinterpret_cast<unsigned char*>(sm) + kHistDevSmem + warp * C::kRing;
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(sm) + kHistDevSmem + C::kHTW * C::kRing) +
                   warp * C::KST;
  if (lane == 0) {
    for (int k = 0; k < C::KST; ++k) mbar_init(bars + k, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  TRACE_T0();
  pdl_wait();
  pdl_trigger();
  const uint64_t pol = policy_evict_first();
  uint32_t phase = 0u;
  const size_t imgBytes = (size_t)H * (size_t)W * 3;
  for (int64_t w0 = 0; w0 < B; w0 += wave_imgs) {
    const int64_t R = min(wave_imgs, B - w0) * (int64_t)H;
    const int64_t r_end = w0 * H + R * (blockIdx.x + 1) / gridDim.x;
    for (int64_t r = w0 * H + R * blockIdx.x / gridDim.x; r < r_end;) {
      const int64_t b = r / H;
      const int y0 = (int)(r - b * H);
      const int y1 = (int)min((int64_t)H, (int64_t)y0 + (r_end - r));
      r += y1 - y0;
      hist_zero<NT>(sm);
      __syncthreads();
      hist_segment_tma<SW, NT, KST>(rgb + (size_t)b * imgBytes, H, W, y0, y1, sm, ring, bars, phase, pol,
                                    hist_s + b * kLevels, hist_graw + b * kGradSlots);
      if (done) {  // the flush above ended with a barrier: release this segment's rows
        __threadfence();
        if (threadIdx.x == 0) atomicAdd(done + b, (uint32_t)(y1 - y0));
      }
    }
  }
  TRACE_END(2u, 0u, 0ull);
}

template <int SW, int NT, int KST, int MINB = 1>
cudaError_t launch_tma_v(const uint8_t* rgb, int64_t B, int32_t H, int32_t W, uint32_t* hs, uint32_t* hg, int grid,
                         cudaStream_t st, uint32_t* done = nullptr, int64_t wave_imgs = 0) {
  using C = HistTma<SW, NT, KST>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e =
        cudaFuncSetAttribute(k_hist_tma<SW, NT, KST, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    // the whole shared-memory carve-out: a solver CTA fits beside the histogram CTA only when
    // the SM is not configured for the histogram CTA alone
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_hist_tma<SW, NT, KST, MINB>, cudaFuncAttributePreferredSharedMemoryCarveout,
                               (int)cudaSharedmemCarveoutMaxShared);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  if (wave_imgs <= 0) wave_imgs = B;
  return launch_pdl(k_hist_tma<SW, NT, KST, MINB>, dim3(grid), dim3(NT), C::kSmem, st, rgb, B, H, W, hs, hg, done,
                    wave_imgs);
}

int wave_rows() {  // rows per CTA per image wave of the overlapped form (HR_HIST_WAVE_ROWS)
  static const int v = [] {
    const char* e = getenv("HR_HIST_WAVE_ROWS");
    return e && atoi(e) > 0 ? atoi(e) : 96;
  }();
  return v;
}

int tma_cfg() {  // measurement switch HR_HIST_TMA_CFG: 0 = 1024 threads x 2 stages, 1 = 512 x 4, 2 = 512 x 3
  static const int v = [] {
    const char* e = getenv("HR_HIST_TMA_CFG");
    return e ? atoi(e) : 0;
  }();
  return v;
}

template <int SW>
cudaError_t launch_tma(const uint8_t* rgb, int64_t B, int32_t H, int32_t W, uint32_t* hs, uint32_t* hg, int grid,
                       cudaStream_t st) {
  switch (tma_cfg()) {
    case 1: return launch_tma_v<SW, 512, 4>(rgb, B, H, W, hs, hg, grid, st);
    case 2: return launch_tma_v<SW, 512, 3>(rgb, B, H, W, hs, hg, grid, st);
    default: return launch_tma_v<SW, 1024, 2>(rgb, B, H, W, hs, hg, grid, st);
  }
}


// done (nullable): after each flushed segment of image b, add its row count to done[b] (fence,
// then atomic: a release), so that k_solve's CTA for image b can start as soon as all H rows of
// image b are flushed -- images finish at staggered times because image boundaries fall at
// spread-out points of the CTA ranges.
template <int SW, int VEC, int NT>
__global__ void __launch_bounds__(NT, 1024 / NT)
k_hist(const uint8_t* __restrict__ rgb, int64_t B, int H, int W, uint32_t* __restrict__ hist_s,
       uint32_t* __restrict__ hist_graw, uint32_t* __restrict__ done, int nowait, uint32_t* __restrict__ cq,
       uint32_t* __restrict__ cq_tail) {
  extern __shared__ __align__(16) uint32_t sm[];
  TRACE_T0();
  if (!nowait) pdl_wait();
  pdl_trigger();
  const int64_t R = B * (int64_t)H;
  const int64_t r_begin = R * blockIdx.x / gridDim.x;
  const int64_t r_end = R * (blockIdx.x + 1) / gridDim.x;
  const size_t imgBytes = (size_t)H * (size_t)W * 3;
  for (int64_t r = r_begin; r < r_end;) {
    const int64_t b = r / H;
    const int y0 = (int)(r - b * H);
    const int y1 = (int)min((int64_t)H, (int64_t)y0 + (r_end - r));
    r += y1 - y0;
    hist_zero<NT>(sm);
    __syncthreads();
    hist_segment<SW, VEC, NT>(rgb + (size_t)b * imgBytes, H, W, y0, y1, sm, hist_s + b * kLevels,
                              hist_graw + b * kGradSlots);
    if (done) {
      __threadfence();
      if (threadIdx.x == 0) {
        const uint32_t rows = (uint32_t)(y1 - y0);
        // the segment that completes image b appends it to the completion queue (release)
        if (atomicAdd(done + b, rows) + rows == (uint32_t)H && cq) st_release(cq + atomicAdd(cq_tail, 1u), (uint32_t)b + 1u);
      }
    }
  }
  TRACE_END(1u, (uint32_t)((uintptr_t)hist_s >> 8), 0ull);  // aux: which launch (group)
}

template <int SW, int VEC, int NT>
cudaError_t launch_v(const uint8_t* rgb, int64_t B, int32_t H, int32_t W, uint32_t* hs, uint32_t* hg, int grid,
                     uint32_t* done, cudaStream_t st, bool nowait, uint32_t* cq, uint32_t* cq_tail) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e =
        cudaFuncSetAttribute(k_hist<SW, VEC, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, kHistDevSmem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  return launch_pdl(k_hist<SW, VEC, NT>, dim3(grid), dim3(NT), kHistDevSmem, st, rgb, B, H, W, hs, hg, done,
                    (int)nowait, cq, cq_tail);
}

template <int SW, int VEC>
cudaError_t launch_nt(const uint8_t* rgb, int64_t B, int32_t H, int32_t W, uint32_t* hs, uint32_t* hg, int grid,
                      int nt, uint32_t* done, cudaStream_t st, bool nowait, uint32_t* cq, uint32_t* cq_tail) {
  return nt == 256 ? launch_v<SW, VEC, 256>(rgb, B, H, W, hs, hg, grid, done, st, nowait, cq, cq_tail)
                   : launch_v<SW, VEC, kHistThreads>(rgb, B, H, W, hs, hg, grid, done, st, nowait, cq, cq_tail);
}

bool hist_w8_strip16() {  // measurement switch: HR_HIST_W8=8 keeps the 8-px strips
  static const int v = [] {
    const char* e = getenv("HR_HIST_W8");
    return e ? atoi(e) : 16;
  }();
  return v != 8;
}

bool hist_mixed() {  // measurement switch: HR_HIST_MIXED=0 keeps six 8-B loads per strip row
  static const int v = [] {
    const char* e = getenv("HR_HIST_MIXED");
    return e ? atoi(e) : 1;
  }();
  return v != 0;
}

__global__ void __launch_bounds__(256) k_zero(uint4* __restrict__ p, size_t n16) {
  pdl_wait();
  pdl_trigger();
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
    p[i] = make_uint4(0u, 0u, 0u, 0u);
}

}  // namespace

void trace_bind_hist(void* buf, uint32_t* n, uint32_t cap) {
#ifdef HR_STEP_TRACE
  trace_bind_tu(buf, n, cap);
#else
  (void)buf, (void)n, (void)cap;
#endif
}

cudaError_t launch_zero(void* p, size_t n, cudaStream_t st) {
  const size_t n16 = n / 16;
  if (n16 == 0) return cudaSuccess;
  const size_t grid = std::min<size_t>((n16 + 255) / 256, 1024);
  return launch_pdl(k_zero, dim3((unsigned)grid), dim3(256), 0, st, reinterpret_cast<uint4*>(p), n16);
}

// shapes of the TMA-staged kernel: 16-B aligned batch whose byte count is a multiple of 16,
// W % 16 == 0 (48-B strips, 16..512 per row) or W % 16 == 8 (24-B strips, 16..512 per row)
bool tma_hist_supported(const uint8_t* rgb, int64_t B, int32_t H, int32_t W) {
  if (reinterpret_cast<uintptr_t>(rgb) % 16 != 0 || ((size_t)B * H * W * 3) % 16 != 0) return false;
  if (W % 16 == 0) return W / 16 >= 16 && W / 16 <= 512;
  if (W % 16 == 8) return W / 8 >= 16 && W / 8 <= 512;
  return false;
}

int hist_grid_clamped(int64_t B, int32_t H, int grid) {
  const int64_t rows = B * (int64_t)H;
  if (grid > rows) grid = (int)rows;
  return grid < 1 ? 1 : grid;
}

cudaError_t launch_hist(const uint8_t* rgb, int64_t B, int32_t H, int32_t W, uint32_t* hist_s,
                        uint32_t* hist_graw, int grid, cudaStream_t st, int nt, uint32_t* done, int tma,
                        bool nowait, uint32_t* cq, uint32_t* cq_tail) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(rgb);
  if (tma && !nowait && !cq && tma_hist_supported(rgb, B, H, W)) {
    // TMA-staged kernel: one CTA per SM (grid is given for 2 CTAs per SM)
    const int g1 = hist_grid_clamped(B, H, std::max(1, grid / 2));
    if (done) {  // overlapped with the solver: 512 threads, <= 64 registers, image waves
      const int64_t k = hist_wave_images(B, H, g1, wave_rows());
      return W % 16 == 0 ? launch_tma_v<16, 512, 3, 2>(rgb, B, H, W, hist_s, hist_graw, g1, st, done, k)
                         : launch_tma_v<8, 512, 3, 2>(rgb, B, H, W, hist_s, hist_graw, g1, st, done, k);
    }
    if (nt == kHistThreads) return W % 16 == 0 ? launch_tma<16>(rgb, B, H, W, hist_s, hist_graw, g1, st)
                                               : launch_tma<8>(rgb, B, H, W, hist_s, hist_graw, g1, st);
  }
  grid = hist_grid_clamped(B, H, grid);
  if (a % 16 == 0 && W % 16 == 0) return launch_nt<16, 16>(rgb, B, H, W, hist_s, hist_graw, grid, nt, done, st, nowait, cq, cq_tail);
  // 8-B aligned rows: 16-px strips of six 8-B loads (the W % 16 == 8 remainder is the scalar tail)
  if (a % 8 == 0 && W % 8 == 0 && W >= 16 && hist_w8_strip16())
    return hist_mixed() ? launch_nt<16, 9>(rgb, B, H, W, hist_s, hist_graw, grid, nt, done, st, nowait, cq, cq_tail)
                        : launch_nt<16, 8>(rgb, B, H, W, hist_s, hist_graw, grid, nt, done, st, nowait, cq, cq_tail);
  if (a % 8 == 0 && W % 8 == 0) return launch_nt<8, 8>(rgb, B, H, W, hist_s, hist_graw, grid, nt, done, st, nowait, cq, cq_tail);
  return launch_nt<16, 1>(rgb, B, H, W, hist_s, hist_graw, grid, nt, done, st, nowait, cq, cq_tail);
}

}  // namespace hr
