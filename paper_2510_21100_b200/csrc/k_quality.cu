// k_quality.cu -- the second workload: the HE baseline (Eq. 5) and the
// quality metrics of §IV (PSNR, SSIM, LOE) on the GPU, batched over images.
//
// Definitions: PAPER.md Eq. 5 for HE; SPEC.md's metrics module for the
// metrics, which PAPER.md names without formulas:
//   HE    t_v = floor(255 c_v + 0.5), c_v = running sum of hS_u / N over u <= v (Eq. 4), applied
//         to V with the R17 colour reconstruction (the k_apply kernel);
//   PSNR  10 log10(255^2 / MSE), MSE over all channels (exact integer SSE); +inf if equal;
//   SSIM  on luma 0.299 R + 0.587 G + 0.114 B, 11x11 Gaussian (sigma 1.5), valid windows,
//         C1 = (0.01 * 255)^2, C2 = (0.03 * 255)^2, mean of the map; NaN if H or W < 11;
//   LOE   lightness max(R,G,B) sampled on a min(H,100) x min(W,100) nearest-neighbour grid,
//         (1/m) sum_x sum_y [(L(x) >= L(y)) xor (L'(x) >= L'(y))].
// Exactness: HE LUTs and LOE counts are bit-exact with the oracle (same fp64 operation order,
// explicit round-to-nearest ops; integer counts).  PSNR and SSIM are fp64 and deterministic
// (integer atomics; per-tile partials summed in a fixed order), equal to the oracle up to
// rounding order.  These kernels serve diagnostics; they are not on the enhancement hot path.
#include <algorithm>

#include "hr_common.cuh"

namespace hr {
namespace {

constexpr int kT = 256;

// ---------------------------------------------------------------- HE LUT (Eq. 4-5)
__global__ void __launch_bounds__(kT) k_he_lut(const uint32_t* __restrict__ hist_s, uint8_t* __restrict__ lut) {
  __shared__ double q[kLevels];
  __shared__ unsigned long long Np[kT / 32];
  const int tid = threadIdx.x;
  const int64_t b = blockIdx.x;
  const uint32_t h = hist_s[b * kLevels + tid];
  unsigned long long v = h;
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
  if ((tid & 31) == 0) Np[tid >> 5] = v;
  __syncthreads();
  unsigned long long N = 0;
  for (int u = 0; u < kT / 32; ++u) N += Np[u];
  q[tid] = N ? __ddiv_rn((double)h, (double)N) : 0.0;  // hS_u / N, correctly rounded
  __syncthreads();
  if (tid == 0) {  // the running sum in the oracle's order (no contraction)
    double c = 0.0;
    for (int i = 0; i < kLevels; ++i) {
      c = __dadd_rn(c, q[i]);
      const double t = floor(__dadd_rn(__dmul_rn(255.0, c), 0.5));
      lut[b * kLevels + i] = (uint8_t)(N ? (t < 0.0 ? 0.0 : (t > 255.0 ? 255.0 : t)) : i);
    }
  }
}

// ---------------------------------------------------------------- PSNR: integer SSE
__global__ void __launch_bounds__(kT) k_sse(const uint8_t* __restrict__ a, const uint8_t* __restrict__ b, int64_t n3,
                                             unsigned long long* __restrict__ sse) {
  const int64_t img = blockIdx.y;
  const uint8_t* pa = a + img * n3;
  const uint8_t* pb = b + img * n3;
  unsigned long long acc = 0;
  for (int64_t i = blockIdx.x * (int64_t)kT + threadIdx.x; i < n3; i += (int64_t)gridDim.x * kT) {
    const int d = (int)pa[i] - (int)pb[i];
    acc += (unsigned long long)(d * d);
  }
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, d);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(sse + img, acc);
}

// ---------------------------------------------------------------- SSIM: separable fp64 tiles
constexpr int kR = 5, kWin = 2 * kR + 1;
constexpr int kTW = 32, kTH = 8;                         // output tile (columns x rows)
constexpr int kIW = kTW + 2 * kR, kIH = kTH + 2 * kR;    // input tile with halo

__device__ __forceinline__ double luma(const uint8_t* p) {
  return __dadd_rn(__dadd_rn(__dmul_rn(0.299, (double)p[0]), __dmul_rn(0.587, (double)p[1])),
                   __dmul_rn(0.114, (double)p[2]));
}

__global__ void __launch_bounds__(kT) k_ssim_tiles(const uint8_t* __restrict__ a, const uint8_t* __restrict__ b,
                                                    int H, int W, int tiles_x, int tiles_y,
                                                    double* __restrict__ partial) {
  __shared__ double ya[kIH][kIW], yb[kIH][kIW];
  __shared__ double hs[5][kIH][kTW];  // horizontal sums: mu_a, mu_b, a^2, b^2, ab
  __shared__ double g[kWin];
  __shared__ double red[kT / 32];
  const int tid = threadIdx.x;
  const int64_t img = blockIdx.y;
  const int tile = blockIdx.x, tx = tile % tiles_x, ty = tile / tiles_x;
  const int ox = kR + tx * kTW, oy = kR + ty * kTH;  // first output centre of this tile
  const size_t n3 = (size_t)H * W * 3;
  const uint8_t* pa = a + img * n3;
  const uint8_t* pb = b + img * n3;
  if (tid < kWin) {
    double gs = 0.0;
    for (int k = -kR; k <= kR; ++k) gs += exp(-(double)(k * k) / (2.0 * 1.5 * 1.5));
    g[tid] = exp(-(double)((tid - kR) * (tid - kR)) / (2.0 * 1.5 * 1.5)) / gs;
  }
  for (int i = tid; i < kIH * kIW; i += kT) {
    const int r = i / kIW, c = i - r * kIW;
    const int y = oy - kR + r, x = ox - kR + c;
    const bool in = y < H && x < W;
    ya[r][c] = in ? luma(pa + 3 * ((size_t)y * W + x)) : 0.0;
    yb[r][c] = in ? luma(pb + 3 * ((size_t)y * W + x)) : 0.0;
  }
  __syncthreads();
  for (int i = tid; i < kIH * kTW; i += kT) {
    const int r = i / kTW, c = i - r * kTW;
    double s0 = 0, s1 = 0, s2 = 0, s3 = 0, s4 = 0;
#pragma unroll
    for (int k = 0; k < kWin; ++k) {
      const double w = g[k], va = ya[r][c + k], vb = yb[r][c + k];
      s0 += w * va;
      s1 += w * vb;
      s2 += w * va * va;
      s3 += w * vb * vb;
      s4 += w * va * vb;
    }
    hs[0][r][c] = s0;
    hs[1][r][c] = s1;
    hs[2][r][c] = s2;
    hs[3][r][c] = s3;
    hs[4][r][c] = s4;
  }
  __syncthreads();
  const double C1 = (0.01 * 255.0) * (0.01 * 255.0), C2 = (0.03 * 255.0) * (0.03 * 255.0);
  double acc = 0.0;
  for (int i = tid; i < kTH * kTW; i += kT) {
    const int r = i / kTW, c = i - r * kTW;
    if (oy + r >= H - kR || ox + c >= W - kR) continue;  // valid centres only
    double m0 = 0, m1 = 0, m2 = 0, m3 = 0, m4 = 0;
#pragma unroll
    for (int k = 0; k < kWin; ++k) {
      const double w = g[k];
      m0 += w * hs[0][r + k][c];
      m1 += w * hs[1][r + k][c];
      m2 += w * hs[2][r + k][c];
      m3 += w * hs[3][r + k][c];
      m4 += w * hs[4][r + k][c];
    }
    const double va = m2 - m0 * m0, vb = m3 - m1 * m1, cov = m4 - m0 * m1;
    acc += ((2.0 * m0 * m1 + C1) * (2.0 * cov + C2)) / ((m0 * m0 + m1 * m1 + C1) * (va + vb + C2));
  }
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, d);
  if ((tid & 31) == 0) red[tid >> 5] = acc;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int u = 0; u < kT / 32; ++u) t += red[u];
    partial[img * (int64_t)(tiles_x * tiles_y) + tile] = t;
  }
}

// ---------------------------------------------------------------- LOE
constexpr int kLoeMax = 100;

__global__ void __launch_bounds__(kT) k_loe_sample(const uint8_t* __restrict__ a, const uint8_t* __restrict__ b,
                                                    int H, int W, uint8_t* __restrict__ La, uint8_t* __restrict__ Lb) {
  const int64_t img = blockIdx.y;
  const int mh = H < kLoeMax ? H : kLoeMax, mw = W < kLoeMax ? W : kLoeMax, m = mh * mw;
  const size_t n3 = (size_t)H * W * 3;
  for (int s = blockIdx.x * kT + threadIdx.x; s < m; s += gridDim.x * kT) {
    const int i = s / mw, j = s - i * mw;
    const int64_t y = (int64_t)i * H / mh, x = (int64_t)j * W / mw;
    const uint8_t* p = a + img * n3 + 3 * (y * W + x);
    const uint8_t* q = b + img * n3 + 3 * (y * W + x);
    La[img * (kLoeMax * kLoeMax) + s] = (uint8_t)__vimax3_u32(p[0], p[1], p[2]);
    Lb[img * (kLoeMax * kLoeMax) + s] = (uint8_t)__vimax3_u32(q[0], q[1], q[2]);
  }
}

__global__ void __launch_bounds__(kT) k_loe_count(const uint8_t* __restrict__ La, const uint8_t* __restrict__ Lb,
                                                   int m, unsigned long long* __restrict__ cnt) {
  __shared__ uint8_t sa[2048], sb[2048];
  const int64_t img = blockIdx.y;
  const uint8_t* A = La + img * (kLoeMax * kLoeMax);
  const uint8_t* Bv = Lb + img * (kLoeMax * kLoeMax);
  const int x = blockIdx.x * kT + threadIdx.x;
  const uint32_t lx = x < m ? A[x] : 0u, lex = x < m ? Bv[x] : 0u;
  uint32_t c = 0;
  for (int y0 = 0; y0 < m; y0 += 2048) {
    const int ny = min(2048, m - y0);
    __syncthreads();
    for (int i = threadIdx.x; i < ny; i += kT) {
      sa[i] = A[y0 + i];
      sb[i] = Bv[y0 + i];
    }
    __syncthreads();
    if (x < m)
      for (int y = 0; y < ny; ++y) c += (uint32_t)((lx >= sa[y]) != (lex >= sb[y]));
  }
  unsigned long long v = c;
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(cnt + img, v);
}

// ---------------------------------------------------------------- finals
__global__ void k_metrics_final(const unsigned long long* __restrict__ sse, const double* __restrict__ ssim_part,
                                const unsigned long long* __restrict__ loe_cnt, int64_t B, int64_t npix, int H, int W,
                                int ntiles, double* psnr, double* ssim, double* loe) {
  const int64_t img = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (img >= B) return;
  if (psnr) {
    const unsigned long long s = sse[img];
    psnr[img] = s == 0 ? __longlong_as_double(0x7FF0000000000000LL)
                       : 10.0 * log10(255.0 * 255.0 / ((double)s / (double)(3 * npix)));
  }
  if (ssim) {
    if (H < kWin || W < kWin) {
      ssim[img] = __longlong_as_double(0x7FF8000000000000LL);
    } else {
      double t = 0.0;
      for (int i = 0; i < ntiles; ++i) t += ssim_part[img * (int64_t)ntiles + i];
      ssim[img] = t / ((double)(H - 2 * kR) * (double)(W - 2 * kR));
    }
  }
  if (loe) {
    const int mh = H < kLoeMax ? H : kLoeMax, mw = W < kLoeMax ? W : kLoeMax;
    loe[img] = (double)loe_cnt[img] / (double)(mh * mw);
  }
}

}  // namespace

cudaError_t launch_he_lut(const uint32_t* hist_s, int64_t B, uint8_t* lut, cudaStream_t st) {
  k_he_lut<<<(unsigned)B, kT, 0, st>>>(hist_s, lut);
  return cudaGetLastError();
}

size_t quality_ws_bytes(int64_t B, int32_t H, int32_t W) {
  const int tx = W > 2 * kR ? (W - 2 * kR + kTW - 1) / kTW : 1, ty = H > 2 * kR ? (H - 2 * kR + kTH - 1) / kTH : 1;
  const size_t nt = (size_t)tx * ty;
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  return al(B * 8) + al(B * 8) + al(B * nt * 8) + 2 * al((size_t)B * kLoeMax * kLoeMax);
}

cudaError_t launch_quality(const uint8_t* a, const uint8_t* b, int64_t B, int32_t H, int32_t W, double* psnr,
                           double* ssim, double* loe, void* ws, cudaStream_t st) {
  const int tx = W > 2 * kR ? (W - 2 * kR + kTW - 1) / kTW : 1, ty = H > 2 * kR ? (H - 2 * kR + kTH - 1) / kTH : 1;
  const int nt = tx * ty;
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  char* w = static_cast<char*>(ws);
  auto* sse = reinterpret_cast<unsigned long long*>(w);
  auto* cnt = reinterpret_cast<unsigned long long*>(w + al(B * 8));
  auto* part = reinterpret_cast<double*>(w + 2 * al(B * 8));
  auto* La = reinterpret_cast<uint8_t*>(w + 2 * al(B * 8) + al(B * (size_t)nt * 8));
  auto* Lb = La + al((size_t)B * kLoeMax * kLoeMax);
  cudaError_t e = cudaMemsetAsync(w, 0, 2 * al(B * 8), st);
  const int64_t npix = (int64_t)H * W;
  if (e == cudaSuccess && psnr) {
    const int gx = (int)std::min<int64_t>((3 * npix + kT * 64 - 1) / (kT * 64), 64);
    k_sse<<<dim3(gx, (unsigned)B), kT, 0, st>>>(a, b, 3 * npix, sse);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess && ssim && H >= kWin && W >= kWin) {
    k_ssim_tiles<<<dim3(nt, (unsigned)B), kT, 0, st>>>(a, b, H, W, tx, ty, part);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess && loe) {
    const int mh = H < kLoeMax ? H : kLoeMax, mw = W < kLoeMax ? W : kLoeMax, m = mh * mw;
    k_loe_sample<<<dim3((m + kT - 1) / kT, (unsigned)B), kT, 0, st>>>(a, b, H, W, La, Lb);
    e = cudaGetLastError();
    if (e == cudaSuccess) {
      k_loe_count<<<dim3((m + kT - 1) / kT, (unsigned)B), kT, 0, st>>>(La, Lb, m, cnt);
      e = cudaGetLastError();
    }
  }
  if (e == cudaSuccess) {
    k_metrics_final<<<(unsigned)((B + 127) / 128), 128, 0, st>>>(sse, part, cnt, B, npix, H, W, nt, psnr, ssim, loe);
    e = cudaGetLastError();
  }
  return e;
}

}  // namespace hr
