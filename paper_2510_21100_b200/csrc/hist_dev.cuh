// hist_dev.cuh -- device body of kernel (a): fused colour convert + gradient + privatised
// histograms over one image segment, launched by k_hist (k_hist.cu).
//
// PAPER.md Alg. 1 lines "Compute the histogram of the low-light image H_C(S)" and
// "Compute the histogram of the gradient image H_C(grad S)", Eq. 3.
// S = max(R,G,B) (HSV value, reading R15); gradient = |dx|+|dy| forward
// differences, 0 on the last column/row (reading R14).  The raw gradient
// (0..510) is histogrammed so that every gradient reading is an exact remap of the
// histogram (k_remap / the solver prologue), never a second pixel pass.
//
// A thread owns an SW-pixel strip (SW = 16: three 16-B loads; SW = 8: three 8-B loads,
// chosen so that W % SW == 0 on the configs) and walks DOWN its rows keeping the previous
// row's packed V and dx in registers, so dy needs no re-read; one halo row per thread group
// is re-read (an L2 hit).  Row y+1 is loaded before row y is processed (two rows in flight
// per thread) and the strip's right neighbour is one extra 4-byte load, so threads never
// exchange data and each walks its own rows.  Columns left over when W % SW != 0 go through
// a scalar tail.
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
// One flush per segment with global integer atomics -> exact, deterministic.
#pragma once
#include "hr_common.cuh"

namespace hr {
namespace {

constexpr int kSlotWords = 64;                                   // 32 V lanes + 32 gradient lanes
constexpr int kHistWords = kLevels * kSlotWords + kLevels;       // + gradients 256..511
constexpr int kHistDevSmem = kHistWords * 4;                     // 66,560 B

__device__ __forceinline__ uint32_t hbx(uint32_t w, int k) {
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

__device__ __forceinline__ void hinc(char* base, uint32_t byteoff) {
  atomicAdd(reinterpret_cast<uint32_t*>(base + byteoff), 1u);
}
// +1 at shared::cta address sbase + byteoff (sbase hoisted out of the loops: one register
// add folded into the ATOMS address, no generic->shared conversion per increment)
__device__ __forceinline__ void sinc(uint32_t sbase, uint32_t byteoff) {
  asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(sbase + byteoff) : "memory");
}

// The 4 bytes at the first pixel of the next strip (r, g, b in bytes 0..2); VEC == 1: the
// value channel itself (byte loads, any alignment).
template <int VEC>
__device__ __forceinline__ uint32_t load_nb(const uint8_t* __restrict__ p) {
  if constexpr (VEC == 1) {
    return vmax3_px(p);
  } else {
    return __ldg(reinterpret_cast<const uint32_t*>(p));  // 8- or 16-B aligned (x0 * 3 + 3 SW)
  }
}
template <int VEC>
__device__ __forceinline__ uint32_t nb_value(uint32_t nb) {
  if constexpr (VEC == 1) {
    return nb;
  } else {
    return __vimax3_u32(hbx(nb, 0), hbx(nb, 1), hbx(nb, 2));
  }
}

// H_C(grad S) counts of one strip row: g = dx + dy per pixel byte, dx of that row in D,
// dy = |V - Vn| against the row below (dy = 0 when !below).  Bytes never carry when every
// dx, dy < 128 (one check per row); otherwise the checked per-pixel path (g up to 510).
template <int G>
__device__ __forceinline__ void grad_row(uint32_t sb, uint32_t* ghi, uint32_t Lg, const uint32_t (&D)[G],
                                         const uint32_t (&V)[G], const uint32_t (&Vn)[G], bool below) {
  uint32_t dy[G], any = 0u;
#pragma unroll
  for (int q = 0; q < G; ++q) {
    dy[q] = below ? __vabsdiffu4(V[q], Vn[q]) : 0u;
    any |= D[q] | dy[q];
  }
  if ((any & 0x80808080u) == 0u) {
#pragma unroll
    for (int q = 0; q < G; ++q) {
      const uint32_t gw = D[q] + dy[q];  // byte-wise: no carries (all bytes < 256)
      sinc(sb, __byte_perm(Lg, gw, 0x1140u));
      sinc(sb, __byte_perm(Lg, gw, 0x1150u));
      sinc(sb, __byte_perm(Lg, gw, 0x1160u));
      sinc(sb, __byte_perm(Lg, gw, 0x1170u));
    }
  } else {
#pragma unroll
    for (int q = 0; q < G; ++q) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t g = hbx(D[q], k) + hbx(dy[q], k);
        if (g < 256u)
          sinc(sb, (g << 8) | Lg);
        else
          atomicAdd(ghi + (g - 256u), 1u);
      }
    }
  }
}

// L2 prefetch of the image rows a few rows ahead of the walk: the walk's own loads (one row
// ahead, registers) then hit L2 instead of DRAM.
#ifndef HR_HIST_PF
#define HR_HIST_PF 2
#endif
// One 128-B line per lane: the first ceil(rowBytes / 128) threads of a row group each prefetch one
// line of the row (p = the line's address in the row the walk is at; lines past the image's end
// are skipped), two instructions per row instead of a bulk-prefetch descriptor built by one lane.
__device__ __forceinline__ void prefetch_line_l2(const uint8_t* p, uintptr_t img_end) {
  if (reinterpret_cast<uintptr_t>(p) < img_end) asm volatile("prefetch.global.L2 [%0];" ::"l"(p) : "memory");
}

// Zero the counters (all NT threads; caller synchronises before use).
template <int NT>
__device__ __forceinline__ void hist_zero(uint32_t* sm) {
  for (int i = threadIdx.x; i < kHistWords / 4; i += NT) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0u, 0u, 0u, 0u);
}

// One thread's walk down a G-group (4 G px) strip: rows ya .. ya + nr - 1 of the band (+ the
// halo row when `halo`), starting at p (the strip's first byte in row ya).  rowEnd: the strip's
// last pixel is x = W - 1 (dx = 0 there, no neighbour load).  RPG + 1 row steps for every lane
// (a warp-uniform trip count); lanes with nr == 0 only mask their counts.
// pfp (nullable): this thread prefetches one 128-B line of each of its group's rows into L2,
// HR_HIST_PF rows ahead (pfp = its line in row ya; img_end = the end of the image).
template <int G, int VEC>
__device__ __forceinline__ void walk_strip(const uint8_t* __restrict__ p, size_t rowBytes, int RPG, int nr,
                                           bool halo, bool rowEnd, uint32_t sb, uint32_t* ghi, uint32_t Lv,
                                           uint32_t Lg, const uint8_t* pfp = nullptr, uintptr_t img_end = 0) {
  const bool pf = pfp != nullptr;  // pfp: this thread's line of the group's first row
  uint32_t Vp[G], Dp[G];
#pragma unroll
  for (int q = 0; q < G; ++q) Vp[q] = Dp[q] = 0u;
  auto need = [&](int it) { return it < nr || (it == nr && halo); };  // row ya+it is read
  auto load_row = [&](const uint8_t* pr, uint32_t (&wr)[3 * G], uint32_t& nbr) {
    load_strip<4 * G, VEC>(pr, wr);
    nbr = rowEnd ? 0u : load_nb<VEC>(pr + 12 * G);
  };
  // step it: row ya+it -> value channel, H_C(S) counts, dx; gradient of row ya+it-1
  auto step = [&](const uint32_t (&wr)[3 * G], uint32_t nbr, int it) {
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
    const uint32_t nbV = nb_value<VEC>(nbr);
#pragma unroll
    for (int q = 0; q < G; ++q)
      Dc[q] = __vabsdiffu4(Vc[q], __funnelshift_r(Vc[q], q < G - 1 ? Vc[q + 1] : nbV, 8));
    if (rowEnd) Dc[G - 1] &= 0x00FFFFFFu;  // dx = 0 at x = W-1
    if (it > 0 && it <= nr) grad_row<G>(sb, ghi, Lg, Dp, Vp, Vc, it < nr || halo);  // dy = 0 on the last row
#pragma unroll
    for (int q = 0; q < G; ++q) {
      Vp[q] = Vc[q];
      Dp[q] = Dc[q];
    }
  };
  // two register sets alternate: row it+1 is in flight while row it is processed
  uint32_t wa[3 * G], wb[3 * G], na = 0u, nb = 0u;
#pragma unroll
  for (int i = 0; i < 3 * G; ++i) wa[i] = wb[i] = 0u;
  if (pf)
    for (int r = 1; r < HR_HIST_PF; ++r)
      if (need(r)) prefetch_line_l2(pfp + r * rowBytes, img_end);
  if (need(0)) load_row(p, wa, na);
  for (int it = 0; it <= RPG; it += 2) {
    if (pf) {  // rows it + PF and it + PF + 1 (this step pair's loads are rows it + 1, it + 2)
      if (need(it + HR_HIST_PF)) prefetch_line_l2(pfp + HR_HIST_PF * rowBytes, img_end);
      if (need(it + HR_HIST_PF + 1)) prefetch_line_l2(pfp + (HR_HIST_PF + 1) * rowBytes, img_end);
      pfp += 2 * rowBytes;
    }
    if (need(it + 1)) load_row(p + rowBytes, wb, nb);
    step(wa, na, it);
    if (it + 1 > RPG) break;
    if (need(it + 2)) load_row(p + 2 * rowBytes, wa, na);
    step(wb, nb, it + 1);
    p += 2 * rowBytes;
  }
}

// Histogram rows [y0, y1) of one H x W image `img` into the (zeroed) lane-private counters
// `sm`, then flush them with integer atomics into hist_s_b[256] / hist_graw_b[512].  All NT
// threads call it; it ends with a barrier (the counters are then free for reuse, not zero).
template <int SW, int VEC, int NT>
__device__ __forceinline__ void hist_segment(const uint8_t* __restrict__ img, int H, int W, int y0, int y1,
                                             uint32_t* sm, uint32_t* __restrict__ hist_s_b,
                                             uint32_t* __restrict__ hist_graw_b) {
  constexpr int G = SW / 4;  // 4-pixel groups per strip
  uint32_t* ghi = sm + kLevels * kSlotWords;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const uint32_t Lv = (uint32_t)lane * 4u;         // byte offset of this lane's V counter
  const uint32_t Lg = 128u + (uint32_t)lane * 4u;  // ... of its gradient counter
  const uint32_t sb = (uint32_t)__cvta_generic_to_shared(sm);

  const int SPf = W / SW;   // full strips per row
  const int xt = SPf * SW;  // first column of the scalar tail
  const int SPt = SPf < NT ? SPf : NT;
  const int NG = SPf == 0 ? 0 : (SPf < NT ? NT / SPf : 1);  // row groups
  const int ntile = (SPf + NT - 1) / NT;
  const int grp = SPt ? tid / SPt : 0;
  const int sl = SPt ? tid - grp * SPt : 0;
  const size_t rowBytes = (size_t)W * 3;

  // ---------------- main walk over the full strips ----------------
  // No shuffles: the right neighbour of the strip's last pixel comes from one extra 4-byte
  // load at the strip end (the same L1 line as the neighbouring thread's strip), and row
  // y+1 is loaded before row y is processed, so two rows of loads are in flight per thread.
  if (NG > 0) {
    const int nrows = y1 - y0;
    const int RPG = (nrows + NG - 1) / NG;
    for (int tile = 0; tile < ntile; ++tile) {
      const int s = tile * NT + sl;
      const bool act = (grp < NG) && (s < SPf) && (y0 + grp * RPG < min(y1, y0 + grp * RPG + RPG));
      const int ya = y0 + grp * RPG;
      const int yb = min(y1, ya + RPG);
      const int nr = act ? yb - ya : 0;  // rows of this thread's band
      const bool halo = act && yb < H;   // row yb exists: the gradient of row yb-1 needs it
      const int x0 = act ? s * SW : 0;
      const bool rowEnd = (s == SPf - 1) && (xt == W);  // last pixel of this strip is x = W-1
      const uint8_t* p = img + (size_t)(act ? ya : 0) * rowBytes + (size_t)x0 * 3;
      // the first strips of each row group prefetch the group's rows into L2, one 128-B line each
      const uintptr_t img_end = reinterpret_cast<uintptr_t>(img) + (size_t)H * rowBytes;
      const bool pfl = act && HR_HIST_PF > 0 && (size_t)s * 128 < rowBytes;
      const uint8_t* pfp = pfl ? img + (size_t)ya * rowBytes + (size_t)s * 128 : nullptr;
      walk_strip<G, VEC>(p, rowBytes, RPG, nr, halo, rowEnd, sb, ghi, Lv, Lg, pfp, img_end);
    }
  }

  // ---------------- scalar tail: columns [xt, W) of rows [y0, y1) ----------------
  if (xt < W) {
    const int tw = W - xt;
    const int n = (y1 - y0) * tw;
    for (int i = tid; i < n; i += NT) {
      const int y = y0 + i / tw;
      const int x = xt + i % tw;
      const uint8_t* p = img + (size_t)y * rowBytes + (size_t)x * 3;
      const uint32_t v = vmax3_px(p);
      const uint32_t vr = (x + 1 < W) ? vmax3_px(p + 3) : v;
      const uint32_t vd = (y + 1 < H) ? vmax3_px(p + rowBytes) : v;
      const uint32_t g = (uint32_t)abs((int)vr - (int)v) + (uint32_t)abs((int)vd - (int)v);
      sinc(sb, (v << 8) | Lv);
      if (g < 256u)
        sinc(sb, (g << 8) | Lg);
      else
        atomicAdd(ghi + (g - 256u), 1u);
    }
  }

  // ---------------- flush: one integer atomic per nonzero bin ----------------
  __syncthreads();
  for (int bin = tid; bin < 2 * kLevels; bin += NT) {
    if (bin < kLevels) {
      uint32_t sv = 0, sg = 0;
#pragma unroll 8
      for (int l = 0; l < 32; ++l) {
        const int o = bin * kSlotWords + ((l + bin) & 31);  // rotated: conflict-free
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

}  // namespace
}  // namespace hr
