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
// segments.  A thread owns an SW-pixel strip (SW = 16: three 16-B loads; SW = 8: three
// 8-B loads, chosen so that W % SW == 0 on the configs) and walks DOWN its rows keeping the
// previous row's packed V and dx in registers, so dy needs no re-read; one halo row per
// thread group is re-read (an L2 hit).  Columns left over when W % SW != 0 go through a
// scalar tail phase.
//
// Per 4 pixels (three words w0 w1 w2 = r0 g0 b0 r1 | g1 b1 r2 g2 | b2 r3 g3 b3):
//   * value channel: PRMT gathers (r0,K,r2,K) (g0,K,g2,K) (b0,K,b2,K) with the SAME filler
//     byte K in each u16 lane, so one VIMNMX3.U16x2 yields max(r,g,b) of two pixels in
//     the low bytes; 6 PRMT + 2 VIMNMX3 for 4 pixels;
//   * dx, dy: VABSDIFF4.U8 on packed V bytes (dy against the previous row's registers);
//   * counters are LANE-PRIVATE: bin v of lane l at word 64v + l (V) and 64v + 32 + l
//     (gradient < 256), so every smem atomic of a warp hits 32 distinct banks whatever the
//     skew (C5 puts 99.8% of pixels in 16 bins), and the byte address (v << 8) | 4l is a
//     single PRMT of the packed value byte with the lane offset;
//   * gradients >= 256 (a byte of dx or dy >= 128: strong edges only) take a checked slow
//     path into a small shared table.
// One flush per (CTA, image) segment with global integer atomics -> exact, deterministic.
#include "hr_common.cuh"

namespace hr {
namespace {

constexpr int kSlotWords = 64;  // words per bin row: 32 V lanes + 32 gradient lanes

__device__ __forceinline__ uint32_t bx(uint32_t w, int k) {
  return __byte_perm(w, 0u, 0x4440u | (uint32_t)k);  // zero-extended byte k
}

template <int SW, int VEC>
__device__ __forceinline__ void load_strip(const uint8_t* __restrict__ p, uint32_t (&w)[3 * SW / 4]) {
  constexpr int NWD = 3 * SW / 4;
  if constexpr (VEC == 16) {
    static_assert(NWD % 4 == 0, "");
    const uint4* q = reinterpret_cast<const uint4*>(p);
#pragma unroll
    for (int i = 0; i < NWD / 4; ++i) {
      const uint4 a = __ldg(q + i);
      w[4 * i] = a.x;
      w[4 * i + 1] = a.y;
      w[4 * i + 2] = a.z;
      w[4 * i + 3] = a.w;
    }
  } else if constexpr (VEC == 8) {
    const uint2* q = reinterpret_cast<const uint2*>(p);
#pragma unroll
    for (int i = 0; i < NWD / 2; ++i) {
      const uint2 a = __ldg(q + i);
      w[2 * i] = a.x;
      w[2 * i + 1] = a.y;
    }
  } else {
#pragma unroll
    for (int i = 0; i < NWD; ++i)
      w[i] = (uint32_t)__ldg(p + 4 * i) | ((uint32_t)__ldg(p + 4 * i + 1) << 8) |
             ((uint32_t)__ldg(p + 4 * i + 2) << 16) | ((uint32_t)__ldg(p + 4 * i + 3) << 24);
  }
}

__device__ __forceinline__ uint32_t vmax3_px(const uint8_t* __restrict__ p) {
  return __vimax3_u32(__ldg(p), __ldg(p + 1), __ldg(p + 2));
}

// value channel of 4 pixels packed as bytes [V0 V1 V2 V3]
__device__ __forceinline__ uint32_t value4(uint32_t w0, uint32_t w1, uint32_t w2) {
  const uint32_t m02 = __vimax3_u16x2(__byte_perm(w0, w1, 0x0600u), __byte_perm(w0, w1, 0x0701u),
                                      __byte_perm(w0, w2, 0x0402u));
  const uint32_t m13 = __vimax3_u16x2(__byte_perm(w0, w2, 0x4543u), __byte_perm(w1, w2, 0x4640u),
                                      __byte_perm(w1, w2, 0x4741u));
  return __byte_perm(m02, m13, 0x6240u);
}

__device__ __forceinline__ void inc(char* base, uint32_t byteoff) {
  atomicAdd(reinterpret_cast<uint32_t*>(base + byteoff), 1u);
}

template <int SW, int VEC>
__global__ void __launch_bounds__(kHistThreads, 2)
k_hist(const uint8_t* __restrict__ rgb, int64_t B, int H, int W, uint32_t* __restrict__ hist_s,
       uint32_t* __restrict__ hist_graw) {
  constexpr int G = SW / 4;  // 4-pixel groups per strip
  extern __shared__ __align__(16) uint32_t sm[];
  uint32_t* ghi = sm + kLevels * kSlotWords;  // gradients 256..511 (shared, rare)
  char* cb = reinterpret_cast<char*>(sm);
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const uint32_t Lv = (uint32_t)lane * 4u;          // byte offset of this lane's V counter
  const uint32_t Lg = 128u + (uint32_t)lane * 4u;   // ... of its gradient counter
  constexpr int kWords = kLevels * kSlotWords + kLevels;

  for (int i = tid; i < kWords / 4; i += kHistThreads)
    reinterpret_cast<uint4*>(sm)[i] = make_uint4(0u, 0u, 0u, 0u);
  __syncthreads();

  const int64_t R = B * (int64_t)H;
  const int64_t r_begin = R * blockIdx.x / gridDim.x;
  const int64_t r_end = R * (blockIdx.x + 1) / gridDim.x;
  const int SPf = W / SW;                       // full strips per row
  const int xt = SPf * SW;                      // first column of the scalar tail
  const int SPt = SPf < kHistThreads ? SPf : kHistThreads;
  const int NG = SPf == 0 ? 0 : (SPf < kHistThreads ? kHistThreads / SPf : 1);  // row groups
  const int ntile = (SPf + kHistThreads - 1) / kHistThreads;
  const int grp = SPt ? tid / SPt : 0;
  const int sl = SPt ? tid - grp * SPt : 0;
  const size_t rowBytes = (size_t)W * 3;

  for (int64_t r = r_begin; r < r_end;) {
    const int64_t b = r / H;
    const int y0 = (int)(r - b * H);
    const int y1 = (int)min((int64_t)H, (int64_t)y0 + (r_end - r));
    r += y1 - y0;
    const uint8_t* img = rgb + (size_t)b * (size_t)H * rowBytes;

    // ---------------- main walk over the full strips ----------------
    if (NG > 0) {
      const int nrows = y1 - y0;
      const int RPG = (nrows + NG - 1) / NG;
      const int ya = y0 + grp * RPG;
      const int yb = min(y1, ya + RPG);
      for (int tile = 0; tile < ntile; ++tile) {
        const int s = tile * kHistThreads + sl;
        const bool active = (grp < NG) && (s < SPf) && (ya < yb);
        const int x0 = s * SW;
        const bool rowEnd = (s == SPf - 1) && (xt == W);  // last pixel of this strip is x = W-1
        // lane+1 holds strip s+1 of the same row unless we are lane 31 or the tile's end
        const bool needNb = active && !rowEnd && (lane == 31 || sl == SPt - 1 || s == SPf - 1);
        uint32_t Vp[G], Dp[G];
#pragma unroll
        for (int q = 0; q < G; ++q) Vp[q] = Dp[q] = 0u;

#pragma unroll 2
        for (int it = 0; it <= RPG; ++it) {
          const int y = ya + it;
          const bool inBand = active && y < yb;
          const bool haveRow = inBand || (active && y == yb && yb < H);  // halo row
          const uint8_t* rowp = img + (size_t)y * rowBytes + (size_t)x0 * 3;
          uint32_t w[3 * G];
          if (haveRow) {
            load_strip<SW, VEC>(rowp, w);
          } else {
#pragma unroll
            for (int i = 0; i < 3 * G; ++i) w[i] = 0u;
          }
          uint32_t Vc[G];
#pragma unroll
          for (int q = 0; q < G; ++q) Vc[q] = value4(w[3 * q], w[3 * q + 1], w[3 * q + 2]);
          if (inBand) {  // H_C(S), Eq. 3
#pragma unroll
            for (int q = 0; q < G; ++q) {
              inc(cb, __byte_perm(Lv, Vc[q], 0x1140u));
              inc(cb, __byte_perm(Lv, Vc[q], 0x1150u));
              inc(cb, __byte_perm(Lv, Vc[q], 0x1160u));
              inc(cb, __byte_perm(Lv, Vc[q], 0x1170u));
            }
          }
          uint32_t nb = __shfl_down_sync(0xffffffffu, Vc[0], 1) & 0xFFu;
          if (needNb && haveRow) nb = vmax3_px(rowp + 3 * SW);
          uint32_t Dc[G];
#pragma unroll
          for (int q = 0; q < G; ++q)
            Dc[q] = __vabsdiffu4(Vc[q], __funnelshift_r(Vc[q], q < G - 1 ? Vc[q + 1] : nb, 8));
          if (rowEnd) Dc[G - 1] &= 0x00FFFFFFu;  // dx = 0 at x = W-1
          // gradient of row y-1: g = dx(y-1) + |V(y) - V(y-1)|  (dy = 0 on the last row)
          if (active && it > 0 && y - 1 < yb) {
#pragma unroll
            for (int q = 0; q < G; ++q) {
              const uint32_t dy = haveRow ? __vabsdiffu4(Vp[q], Vc[q]) : 0u;
              if (((Dp[q] | dy) & 0x80808080u) == 0u) {
                const uint32_t gw = Dp[q] + dy;  // byte-wise: no carries (all bytes < 256)
                inc(cb, __byte_perm(Lg, gw, 0x1140u));
                inc(cb, __byte_perm(Lg, gw, 0x1150u));
                inc(cb, __byte_perm(Lg, gw, 0x1160u));
                inc(cb, __byte_perm(Lg, gw, 0x1170u));
              } else {
#pragma unroll
                for (int p = 0; p < 4; ++p) {
                  const uint32_t g = bx(Dp[q], p) + bx(dy, p);
                  if (g < 256u)
                    inc(cb, (g << 8) | Lg);
                  else
                    atomicAdd(ghi + (g - 256u), 1u);
                }
              }
            }
          }
#pragma unroll
          for (int q = 0; q < G; ++q) {
            Vp[q] = Vc[q];
            Dp[q] = Dc[q];
          }
        }
      }
    }

    // ---------------- scalar tail: columns [xt, W) of rows [y0, y1) ----------------
    if (xt < W) {
      const int tw = W - xt;
      const int n = (y1 - y0) * tw;
      for (int i = tid; i < n; i += kHistThreads) {
        const int y = y0 + i / tw;
        const int x = xt + i % tw;
        const uint8_t* p = img + (size_t)y * rowBytes + (size_t)x * 3;
        const uint32_t v = vmax3_px(p);
        const uint32_t vr = (x + 1 < W) ? vmax3_px(p + 3) : v;
        const uint32_t vd = (y + 1 < H) ? vmax3_px(p + rowBytes) : v;
        const uint32_t g = (uint32_t)abs((int)vr - (int)v) + (uint32_t)abs((int)vd - (int)v);
        inc(cb, (v << 8) | Lv);
        if (g < 256u)
          inc(cb, (g << 8) | Lg);
        else
          atomicAdd(ghi + (g - 256u), 1u);
      }
    }

    // ---------------- flush: one integer atomic per nonzero bin ----------------
    __syncthreads();
    for (int bin = tid; bin < 2 * kLevels; bin += kHistThreads) {
      if (bin < kLevels) {
        uint32_t sv = 0, sg = 0;
#pragma unroll 8
        for (int l = 0; l < 32; ++l) {
          const int o = bin * kSlotWords + ((l + bin) & 31);  // rotated: conflict-free
          sv += sm[o];
          sg += sm[o + 32];
        }
        if (sv) atomicAdd(hist_s + b * kLevels + bin, sv);
        if (sg) atomicAdd(hist_graw + b * kGradSlots + bin, sg);
      } else {
        const uint32_t c = ghi[bin - kLevels];
        if (c) atomicAdd(hist_graw + b * kGradSlots + bin, c);
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

template <int SW, int VEC>
cudaError_t launch_v(const uint8_t* rgb, int64_t B, int32_t H, int32_t W, uint32_t* hs, uint32_t* hg, int grid,
                     cudaStream_t st) {
  constexpr int smem = (kLevels * kSlotWords + kLevels) * 4;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_hist<SW, VEC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  k_hist<SW, VEC><<<grid, kHistThreads, smem, st>>>(rgb, B, H, W, hs, hg);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_hist(const uint8_t* rgb, int64_t B, int32_t H, int32_t W, uint32_t* hist_s,
                        uint32_t* hist_graw, int grid, cudaStream_t st) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(rgb);
  const int64_t rows = B * (int64_t)H;
  if (grid > rows) grid = (int)rows;
  if (grid < 1) grid = 1;
  if (a % 16 == 0 && W % 16 == 0) return launch_v<16, 16>(rgb, B, H, W, hist_s, hist_graw, grid, st);
  if (a % 8 == 0 && W % 8 == 0) return launch_v<8, 8>(rgb, B, H, W, hist_s, hist_graw, grid, st);
  return launch_v<16, 1>(rgb, B, H, W, hist_s, hist_graw, grid, st);
}

}  // namespace hr
