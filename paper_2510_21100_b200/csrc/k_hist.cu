// k_hist.cu -- kernel (a): fused colour convert + gradient + privatised histograms.
//
// PAPER.md Alg. 1 lines "Compute the histogram of the low-light image H_C(S)" and
// "Compute the histogram of the gradient image H_C(grad S)", Eq. 3.
// S = max(R,G,B) (HSV value, reading R15); gradient = |dx|+|dy| forward
// differences, 0 on the last column/row (reading R14).  The raw gradient
// (0..510) is histogrammed so that every gradient reading is an exact remap of the
// histogram (k_remap / the solver prologue), never a second pixel pass.
//
// Design (B200): persistent grid of 2 CTAs/SM x 512 threads.  Each CTA owns a contiguous
// range of global rows (all images concatenated), split at image boundaries into
// segments.  A thread owns a 16-pixel strip (48 B, 3 x 16-B vector loads when W % 16 == 0)
// and walks DOWN its rows keeping the previous row's packed V and dx in registers, so dy
// needs no re-read; only one halo row per thread group is re-read (L2 hit).  Neighbour V
// for dx comes from lane+1 by shuffle.  V = VIMNMX3 of the three channels; dx/dy via
// VABSDIFF4.U8 on packed bytes; gradient pairs g0|g2 / g1|g3 in u16x2 lanes so one IMAD
// gives two smem addresses.  Histograms are LANE-PRIVATE (counter of bin v for lane l at
// word v*32+l): every ATOMS of a warp hits 32 distinct banks regardless of data skew (the
// dark configs put >90% of pixels in 16 bins).  One flush per (CTA, image) segment with
// global integer atomics -> deterministic exact counts.
#include "hr_common.cuh"

namespace hr {
namespace {

__device__ __forceinline__ uint32_t bx(uint32_t w, int k) {
  return __byte_perm(w, 0u, 0x4440u | (uint32_t)k);  // zero-extended byte k
}

template <int VEC>
__device__ __forceinline__ void load48(const uint8_t* __restrict__ p, uint32_t (&w)[12]) {
  if constexpr (VEC == 16) {
    const uint4* q = reinterpret_cast<const uint4*>(p);
    const uint4 a = __ldg(q), b = __ldg(q + 1), c = __ldg(q + 2);
    w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w;
    w[4] = b.x; w[5] = b.y; w[6] = b.z; w[7] = b.w;
    w[8] = c.x; w[9] = c.y; w[10] = c.z; w[11] = c.w;
  } else if constexpr (VEC == 8) {
    const uint2* q = reinterpret_cast<const uint2*>(p);
#pragma unroll
    for (int i = 0; i < 6; ++i) {
      const uint2 a = __ldg(q + i);
      w[2 * i] = a.x;
      w[2 * i + 1] = a.y;
    }
  } else if constexpr (VEC == 4) {
    const uint32_t* q = reinterpret_cast<const uint32_t*>(p);
#pragma unroll
    for (int i = 0; i < 12; ++i) w[i] = __ldg(q + i);
  } else {
#pragma unroll
    for (int i = 0; i < 12; ++i)
      w[i] = (uint32_t)__ldg(p + 4 * i) | ((uint32_t)__ldg(p + 4 * i + 1) << 8) |
             ((uint32_t)__ldg(p + 4 * i + 2) << 16) | ((uint32_t)__ldg(p + 4 * i + 3) << 24);
  }
}

// Ragged strip (npx < 16 pixels left in the row): byte loads, zero fill.
__device__ __forceinline__ void load_partial(const uint8_t* __restrict__ p, int npx, uint32_t (&w)[12]) {
  const int nb = 3 * npx;
#pragma unroll
  for (int i = 0; i < 12; ++i) w[i] = 0;
#pragma unroll
  for (int k = 0; k < 48; ++k)
    if (k < nb) w[k >> 2] |= (uint32_t)__ldg(p + k) << (8 * (k & 3));
}

__device__ __forceinline__ uint32_t pack4(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  return __byte_perm(__byte_perm(a, b, 0x0040u), __byte_perm(c, d, 0x0040u), 0x5410u);
}

template <int VEC>
__global__ void __launch_bounds__(kHistThreads, 2)
k_hist(const uint8_t* __restrict__ rgb, int64_t B, int H, int W, uint32_t* __restrict__ hist_s,
       uint32_t* __restrict__ hist_graw) {
  extern __shared__ __align__(16) uint32_t sm[];
  uint32_t* hv = sm;                   // [256][32]
  uint32_t* hg = sm + kLevels * kLanes;  // [512][32]
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const uint32_t lane4 = (uint32_t)lane * 4u;
  const uint32_t lane4x2 = lane4 | (lane4 << 16);
  constexpr int kWords = (kLevels + kGradSlots) * kLanes;

  for (int i = tid; i < kWords / 4; i += kHistThreads)
    reinterpret_cast<uint4*>(sm)[i] = make_uint4(0u, 0u, 0u, 0u);
  __syncthreads();

  const int64_t R = B * (int64_t)H;
  const int64_t r_begin = R * blockIdx.x / gridDim.x;
  const int64_t r_end = R * (blockIdx.x + 1) / gridDim.x;
  const int SP = (W + 15) >> 4;                 // strips per row
  const int SPt = SP < kHistThreads ? SP : kHistThreads;
  const int NG = SP < kHistThreads ? kHistThreads / SP : 1;  // row groups per CTA
  const int ntile = (SP + kHistThreads - 1) / kHistThreads;
  const int grp = tid / SPt;
  const int sl = tid - grp * SPt;
  const size_t rowBytes = (size_t)W * 3;

  for (int64_t r = r_begin; r < r_end;) {
    const int64_t b = r / H;
    const int y0 = (int)(r - b * H);
    const int y1 = (int)min((int64_t)H, (int64_t)y0 + (r_end - r));
    r += y1 - y0;
    const uint8_t* img = rgb + (size_t)b * (size_t)H * rowBytes;
    const int nrows = y1 - y0;
    const int RPG = (nrows + NG - 1) / NG;
    const int ya = y0 + grp * RPG;
    const int yb = min(y1, ya + RPG);

    for (int tile = 0; tile < ntile; ++tile) {
      const int s = tile * kHistThreads + sl;
      const bool active = (grp < NG) && (s < SP) && (ya < yb);
      const int x0 = s << 4;
      const int npx = active ? min(16, W - x0) : 0;
      const bool lastStrip = (s == SP - 1);
      // lane+1 holds strip s+1 of the same row unless we are lane 31 or the tile's end.
      const bool needNbLoad = active && !lastStrip && (lane == 31 || sl == SPt - 1);
      uint32_t Vp[4] = {0u, 0u, 0u, 0u}, Dp[4] = {0u, 0u, 0u, 0u};

      for (int it = 0; it <= RPG; ++it) {
        const int y = ya + it;
        const bool inBand = active && y < yb;
        const bool haveRow = inBand || (active && y == yb && yb < H);  // halo row
        const uint8_t* rowp = img + (size_t)y * rowBytes + (size_t)x0 * 3;
        uint32_t w[12];
        if (haveRow) {
          if (npx == 16)
            load48<VEC>(rowp, w);
          else
            load_partial(rowp, npx, w);
        } else {
#pragma unroll
          for (int i = 0; i < 12; ++i) w[i] = 0u;
        }
        uint32_t v[16];
#pragma unroll
        for (int p = 0; p < 16; ++p) {
          const int o = 3 * p;
          v[p] = __vimax3_u32(bx(w[o >> 2], o & 3), bx(w[(o + 1) >> 2], (o + 1) & 3),
                              bx(w[(o + 2) >> 2], (o + 2) & 3));
        }
        // H_C(S) for rows of this band (Eq. 3)
        if (inBand) {
          if (npx == 16) {
#pragma unroll
            for (int p = 0; p < 16; ++p) atomicAdd(hv + ((v[p] << 5) | lane), 1u);
          } else {
#pragma unroll
            for (int p = 0; p < 16; ++p)
              if (p < npx) atomicAdd(hv + ((v[p] << 5) | lane), 1u);
          }
        }
        uint32_t Vc[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) Vc[q] = pack4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        uint32_t nb = __shfl_down_sync(0xffffffffu, v[0], 1);
        if (needNbLoad && haveRow) {
          const uint8_t* qn = rowp + 48;
          nb = __vimax3_u32(__ldg(qn), __ldg(qn + 1), __ldg(qn + 2));
        }
        uint32_t Dc[4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
          Dc[q] = __vabsdiffu4(Vc[q], __funnelshift_r(Vc[q], q < 3 ? Vc[q + 1] : nb, 8));
        if (lastStrip) {  // dx = 0 at x = W-1 (forward difference, last column)
          const int pl = npx - 1;
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (q == (pl >> 2)) Dc[q] &= ~(0xFFu << (8 * (pl & 3)));
        }
        // gradient of row y-1: g = dx(y-1) + |V(y) - V(y-1)|  (dy = 0 on the last row)
        if (active && it > 0 && y - 1 < yb) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint32_t dy = haveRow ? __vabsdiffu4(Vp[q], Vc[q]) : 0u;
            const uint32_t ge = __byte_perm(Dp[q], 0u, 0x4240u) + __byte_perm(dy, 0u, 0x4240u);
            const uint32_t go = __byte_perm(Dp[q], 0u, 0x4341u) + __byte_perm(dy, 0u, 0x4341u);
            const uint32_t ae = ge * 128u + lane4x2;  // byte offsets of pixels 4q, 4q+2
            const uint32_t ao = go * 128u + lane4x2;  // pixels 4q+1, 4q+3
            char* hgb = reinterpret_cast<char*>(hg);
            if (npx == 16) {
              atomicAdd(reinterpret_cast<uint32_t*>(hgb + (ae & 0xFFFFu)), 1u);
              atomicAdd(reinterpret_cast<uint32_t*>(hgb + (ao & 0xFFFFu)), 1u);
              atomicAdd(reinterpret_cast<uint32_t*>(hgb + (ae >> 16)), 1u);
              atomicAdd(reinterpret_cast<uint32_t*>(hgb + (ao >> 16)), 1u);
            } else {
              if (4 * q < npx) atomicAdd(reinterpret_cast<uint32_t*>(hgb + (ae & 0xFFFFu)), 1u);
              if (4 * q + 1 < npx) atomicAdd(reinterpret_cast<uint32_t*>(hgb + (ao & 0xFFFFu)), 1u);
              if (4 * q + 2 < npx) atomicAdd(reinterpret_cast<uint32_t*>(hgb + (ae >> 16)), 1u);
              if (4 * q + 3 < npx) atomicAdd(reinterpret_cast<uint32_t*>(hgb + (ao >> 16)), 1u);
            }
          }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          Vp[q] = Vc[q];
          Dp[q] = Dc[q];
        }
      }
    }
    // flush this image's sub-histograms: one integer atomic per nonzero bin
    __syncthreads();
    for (int bin = tid; bin < kLevels + kGradSlots; bin += kHistThreads) {
      uint32_t acc = 0;
#pragma unroll 8
      for (int l = 0; l < kLanes; ++l) acc += sm[bin * kLanes + ((l + bin) & 31)];  // conflict-free
      if (acc) {
        if (bin < kLevels)
          atomicAdd(hist_s + b * kLevels + bin, acc);
        else
          atomicAdd(hist_graw + b * kGradSlots + (bin - kLevels), acc);
      }
    }
    __syncthreads();
    if (r < r_end) {
      for (int i = tid; i < kWords / 4; i += kHistThreads)
        reinterpret_cast<uint4*>(sm)[i] = make_uint4(0u, 0u, 0u, 0u);
      __syncthreads();
    }
  }
}

template <int VEC>
cudaError_t launch_vec(const uint8_t* rgb, int64_t B, int32_t H, int32_t W, uint32_t* hs, uint32_t* hg,
                       int grid, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_hist<VEC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kHistSmemBytes);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  k_hist<VEC><<<grid, kHistThreads, kHistSmemBytes, st>>>(rgb, B, H, W, hs, hg);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_hist(const uint8_t* rgb, int64_t B, int32_t H, int32_t W, uint32_t* hist_s,
                        uint32_t* hist_graw, int grid, cudaStream_t st) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(rgb);
  const int64_t rows = B * (int64_t)H;
  if (grid > rows) grid = (int)rows;
  if (grid < 1) grid = 1;
  if (a % 16 == 0 && W % 16 == 0) return launch_vec<16>(rgb, B, H, W, hist_s, hist_graw, grid, st);
  if (a % 8 == 0 && W % 8 == 0) return launch_vec<8>(rgb, B, H, W, hist_s, hist_graw, grid, st);
  if (a % 4 == 0 && W % 4 == 0) return launch_vec<4>(rgb, B, H, W, hist_s, hist_graw, grid, st);
  return launch_vec<1>(rgb, B, H, W, hist_s, hist_graw, grid, st);
}

}  // namespace hr
