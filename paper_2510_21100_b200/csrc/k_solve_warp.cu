// k_solve_warp.cu -- kernel (b), warp-per-image form: Algorithm 1 (Eqs. 6-15) and the
// Eq. 20 target for images whose gradient support has at most 32 levels (nR <= 32: every
// batched config; C4 and dense parity inputs go to the CTA kernel k_solve).
//
// One warp owns one image; lane a owns compacted reflectance row a (its state hR, hG, the
// raw update and the L-weight live in registers).  There is no block barrier anywhere: the
// phases are separated by __syncwarp and every reduction is a fixed-order shuffle tree, so
// results are bit-identical run to run.  Same mathematics and readings as k_solve.cu (see
// its header): factored Eq. 13 / Eq. 12 with rho_k = hS_k / EstRaw_k, supports frozen,
// EstRaw_k = sum over the runs of bin k of hR_a * (sum of hL over the run) in row order
// (a run = maximal stretch of a row with one index(i,j)), renormalisation folded into the
// next run-sum phase.  With nR <= 32 a bin's row set is one 32-bit word, built by one ballot.
// Images with nR > 32 or more than kRunCap runs are flagged (deferred[b] = 1) and left to
// k_solve.  Outputs: hL, hR (dense), target (Eq. 20), iters; the LUT comes from k_match.
#include "hr_common.cuh"

namespace hr {
namespace {

constexpr int kWPC = 4;        // warps (images) per CTA

#ifdef HR_SOLVE_PROFILE
__device__ long long g_wclk[64];
#define WMARK(i) do { if (blockIdx.x == 0 && threadIdx.x == 0) { const long long c_ = clock64(); wacc[i] += c_ - wt0; wt0 = c_; } } while (0)
#else
#define WMARK(i) do { } while (0)
#endif
constexpr int kRunCap = 512;   // runs per image handled in shared memory

struct __align__(16) WarpSm {
  double hL[kLevels];      // renormalised illumination state (compacted columns)
  double rho[kLevels];     // rho_k (GC) or sigma_k (paper-literal)
  double runE[kRunCap];    // bin order: hR_a * sum(hL over the run)
  double runS2[kRunCap];   // bin order: sum(hL^2 over the run)
  double wsm[32];          // L-weights of the rows
  uint32_t hSi[kLevels], hGi[kLevels];
  uint32_t rr[kRunCap];    // run descriptors k | lo << 8 | hi << 16 | a << 24 (bin order)
  uint32_t mask[kLevels];  // bit a: row a has a run of bin k
  uint16_t keyStart[kLevels + 1];
  uint16_t rowRun[kRunCap];  // run slots in row order
  uint8_t listL[kLevels], posL[kLevels], listR[32];
};

__device__ __forceinline__ int idx0(int i, int j) { return (int)(((uint32_t)(i * j + 127) * 32897u) >> 23); }

__device__ __forceinline__ double rcp_fast(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
  return v;
}
__device__ __forceinline__ void wsum3(double& a, double& b, double& c) {
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, d);
    b += __shfl_xor_sync(0xffffffffu, b, d);
    c += __shfl_xor_sync(0xffffffffu, c, d);
  }
}

// per-bin row words from each lane's 256-bit bin set; keyStart = exclusive scan of popcounts
// (bin-ordered slots).  Returns the number of runs.
__device__ __forceinline__ int warp_masks(WarpSm& s, const uint32_t (&set)[8], int kmax) {
  const int lane = threadIdx.x & 31;
  const int kw = (kmax >> 5) + 1;
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    if (u < kw) {
      for (int bit = 0; bit < 32; ++bit) {
        const uint32_t m = __ballot_sync(0xffffffffu, (set[u] >> bit) & 1u);
        if (lane == bit) s.mask[u * 32 + bit] = m;
      }
    } else {
      s.mask[u * 32 + lane] = 0u;
    }
  }
  __syncwarp();
  // keys 8*lane .. 8*lane+7 are contiguous per lane: local prefix + warp scan of lane totals
  int loc[8], tot = 0;
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    loc[u] = tot;
    tot += __popc(s.mask[8 * lane + u]);
  }
  int inc = tot;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int o = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc += o;
  }
  const int base = inc - tot;
#pragma unroll
  for (int u = 0; u < 8; ++u) s.keyStart[8 * lane + u] = (uint16_t)(base + loc[u]);
  const int RR = __shfl_sync(0xffffffffu, inc, 31);
  if (lane == 0) s.keyStart[kLevels] = (uint16_t)min(RR, 65535);
  __syncwarp();
  return RR;
}

__device__ __forceinline__ void set_bit8(uint32_t (&set)[8], int k) {
#pragma unroll
  for (int u = 0; u < 8; ++u) set[u] |= (u == (k >> 5)) ? (1u << (k & 31)) : 0u;
}

__global__ void __launch_bounds__(32 * kWPC, 2) k_solve_warp(SolveArgs args, int64_t B, int32_t* deferred) {
  extern __shared__ __align__(16) unsigned char smraw[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  WarpSm& s = reinterpret_cast<WarpSm*>(smraw)[wid];
  const int64_t b = (int64_t)blockIdx.x * kWPC + wid;
  if (b >= B) return;
  const hr_params& P = args.p;
  const unsigned full = 0xffffffffu;
#ifdef HR_SOLVE_PROFILE
  long long wacc[16] = {0}, wt0 = clock64();
#endif

  // ---- histograms (Alg. 1 init) and the gradient levels (R14) ----
  for (int v = lane; v < kLevels; v += 32) {
    s.hSi[v] = args.hist_s[b * kLevels + v];
    s.hGi[v] = args.hist_g ? args.hist_g[b * kLevels + v] : 0u;
  }
  if (!args.hist_g) {
    const uint32_t* graw = args.graw + b * kGradSlots;
    uint32_t cnt[16];
    int gmax = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      cnt[j] = graw[lane + 32 * j];
      if (cnt[j]) gmax = lane + 32 * j;
    }
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) gmax = max(gmax, __shfl_xor_sync(full, gmax, d));
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const uint32_t g = lane + 32 * j;
      if (cnt[j]) {
        const int lev = args.grad_norm == 1 ? (g < 255u ? (int)g : 255)
                                            : (gmax == 0 ? 0 : (int)((510u * g + (uint32_t)gmax) / (2u * (uint32_t)gmax)));
        atomicAdd(&s.hGi[lev], cnt[j]);  // integer: order-independent
      }
    }
  }
  __syncwarp();
  WMARK(0);

  // ---- supports (fixed for all t) and N ----
  int nL = 0, nR = 0;
  unsigned long long nsum = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int v = 32 * j + lane;
    const uint32_t hs = s.hSi[v], hg = s.hGi[v];
    nsum += hs;
    const uint32_t mL = __ballot_sync(full, hs != 0u), mR = __ballot_sync(full, hg != 0u);
    const int pl = nL + __popc(mL & ((1u << lane) - 1u)), pr = nR + __popc(mR & ((1u << lane) - 1u));
    if (hs) {
      s.listL[pl] = (uint8_t)v;
      s.posL[v] = (uint8_t)pl;
    }
    if (hg && pr < 32) s.listR[pr] = (uint8_t)v;
    nL += __popc(mL);
    nR += __popc(mR);
  }
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) nsum += __shfl_xor_sync(full, nsum, d);
  const double N = (double)nsum;
  __syncwarp();
  if (nR > 32 || nR == 0 || nsum == 0) {  // not for this kernel (k_solve handles it)
    if (lane == 0) deferred[b] = 1;
    return;
  }
  const bool row = lane < nR;
  const int ia = row ? s.listR[lane] : 0;
  WMARK(1);

  // ---- runs of index(i,j) along the rows (fixed for all t) ----
  uint32_t set[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
  int cntR = 0, kmax = 0;
  if (row) {
    int prev = -1;
    for (int c = 0; c < nL; ++c) {
      const int k = idx0(ia, s.listL[c]);
      if (k != prev) {
        set_bit8(set, k);
        ++cntR;
        prev = k;
      }
    }
    kmax = prev;
  }
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) kmax = max(kmax, __shfl_xor_sync(full, kmax, d));
  const int RR = warp_masks(s, set, kmax);
  if (RR > kRunCap) {
    if (lane == 0) deferred[b] = 1;
    return;
  }
  int rs = cntR;  // exclusive scan of the runs per row -> first rowRun index of this row
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int o = __shfl_up_sync(full, rs, d);
    if (lane >= d) rs += o;
  }
  rs -= cntR;
  if (row) {
    const uint32_t below = (1u << lane) - 1u;
    int prev = idx0(ia, s.listL[0]), lo = 0, i = rs;
    for (int c = 1; c <= nL; ++c) {
      const int k = c < nL ? idx0(ia, s.listL[c]) : -1;
      if (k != prev) {
        const int slot = s.keyStart[prev] + __popc(s.mask[prev] & below);
        s.rr[slot] = (uint32_t)prev | ((uint32_t)lo << 8) | ((uint32_t)(c - 1) << 16) | ((uint32_t)lane << 24);
        s.rowRun[i++] = (uint16_t)slot;
        prev = k;
        lo = c;
      }
    }
  }
  __syncwarp();
  WMARK(2);

  // ---- state: hR^0 = hG, hL^0 = hS (R9) as raw iterates with sums N ----
  const double hGa = row ? (double)s.hGi[ia] : 0.0;
  double hR = hGa, hR1 = hGa;
  double hL1[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int c = lane + 32 * j;
    hL1[j] = c < nL ? (double)s.hSi[s.listL[c]] : 0.0;
    if (c < nL) s.hL[c] = hL1[j];
  }
  const int form = P.update_form;
  const double invN = 1.0 / N, invN2 = invN * invN;
  double SR1 = N, SL1 = N;
  int t = 0;
  for (;;) {
    // ======== E1: renormalise (Eqs. 15, 14) + run sums (Eqs. 6, 8) ========
    const double cR = N * rcp_fast(SR1), cL = N * rcp_fast(SL1);
    double dr = 0.0, dl = 0.0, q = 0.0;
    {
      const double n = cR * hR1;
      if (row) dr = (n - hR) * (n - hR);
      hR = row ? n : 0.0;
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int c = lane + 32 * j;
      if (c < nL) {
        const double n = cL * hL1[j];
        const double o = s.hL[c];
        dl += (n - o) * (n - o);
        s.hL[c] = n;
        q += n * n;
      }
    }
    __syncwarp();
    if (row) {
      for (int i = rs; i < rs + cntR; ++i) {
        const int slot = s.rowRun[i];
        const uint32_t d = s.rr[slot];
        const int lo = (d >> 8) & 255, hi = (d >> 16) & 255;
        double s0 = 0.0, s1 = 0.0, q0 = 0.0, q1 = 0.0;
        int c = lo;
        for (; c + 1 <= hi; c += 2) {
          const double x0 = s.hL[c], x1 = s.hL[c + 1];
          s0 += x0;
          s1 += x1;
          q0 = fma(x0, x0, q0);
          q1 = fma(x1, x1, q1);
        }
        if (c <= hi) {
          const double x0 = s.hL[c];
          s0 += x0;
          q0 = fma(x0, x0, q0);
        }
        s.runE[slot] = hR * (s0 + s1);
        s.runS2[slot] = q0 + q1;
      }
    }
    WMARK(3);
    wsum3(dr, dl, q);
    __syncwarp();
    WMARK(4);
    if (t > 0) {  // stop rule (R11) on the renormalised iterates of update t
      const double eps = P.epsilon * N * N;
      if ((P.use_epsilon && dr <= eps && dl <= eps) || t >= P.max_iter) break;
    }
    // ======== EstRaw_k over the runs of bin k (row order) and rho_k (Eq. 11 folded) ========
#pragma unroll 2
    for (int u = 0; u < 8; ++u) {
      const int k = lane + 32 * u;
      const int k0 = s.keyStart[k], k1 = s.keyStart[k + 1];
      if (k0 < k1) {
        double e0 = 0.0, e1 = 0.0, e2 = 0.0, e3 = 0.0;
        int j = k0;
        for (; j + 3 < k1; j += 4) {
          e0 += s.runE[j];
          e1 += s.runE[j + 1];
          e2 += s.runE[j + 2];
          e3 += s.runE[j + 3];
        }
        for (; j < k1; ++j) e0 += s.runE[j];
        const double e = (e0 + e1) + (e2 + e3);
        s.rho[k] = form == 0 ? (e > 0.0 ? (double)s.hSi[k] * rcp_fast(e) : 0.0) : (double)s.hSi[k] * e;
      }
    }
    __syncwarp();
    WMARK(5);
    // ======== Eq. 13 (lane = row) ========
    {
      const double invDenR = rcp_fast(q * invN2 + P.beta);
      double A = 0.0;
      if (row) {
        for (int i = rs; i < rs + cntR; ++i) {
          const int slot = s.rowRun[i];
          const uint32_t d = s.rr[slot];
          const double r = s.rho[d & 255];
          A = form == 0 ? fma(r, s.runS2[slot], A) : fma(r, (double)(((d >> 16) & 255) - ((d >> 8) & 255) + 1), A);
        }
        const double num = form == 0 ? hR * A * invN : A * rcp_fast(N * hR);
        double v = (num + P.beta * hGa) * invDenR;
        hR1 = v > 0.0 ? v : 0.0;
        s.wsm[lane] = form == 0 ? hR1 * hR : hR1 * rcp_fast(hR);
      } else {
        hR1 = 0.0;
      }
    }
    WMARK(6);
    double sr1 = hR1, sr2 = hR1 * hR1, unused = 0.0;
    wsum3(sr1, sr2, unused);
    __syncwarp();
    WMARK(7);
    // ======== Eq. 12, frozen K (lane = columns lane + 32j) ========
    {
      const double invDenL = rcp_fast(sr2 * invN2 + P.alpha);
      double sl1 = 0.0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int c = lane + 32 * j;
        if (c < nL) {
          const int jc = s.listL[c];
          double b0 = 0.0, b1 = 0.0;
          int a = 0;
          for (; a + 1 < nR; a += 2) {
            b0 = fma(s.wsm[a], s.rho[idx0(s.listR[a], jc)], b0);
            b1 = fma(s.wsm[a + 1], s.rho[idx0(s.listR[a + 1], jc)], b1);
          }
          if (a < nR) b0 = fma(s.wsm[a], s.rho[idx0(s.listR[a], jc)], b0);
          const double Bv = b0 + b1, hl = s.hL[c];
          const double num = form == 0 ? hl * Bv * invN : Bv * rcp_fast(N * hl);
          double u = (num + P.alpha * (double)s.hSi[jc]) * invDenL;
          u = u > 0.0 ? u : 0.0;
          hL1[j] = u;
          sl1 += u;
        }
      }
      WMARK(8);
      SL1 = wsum(sl1);
    }
    SR1 = sr1;
    ++t;
    __syncwarp();
    WMARK(9);
  }
  WMARK(10);

  // ---- outputs hL, hR (dense, zero off support), iteration count ----
  for (int v = lane; v < kLevels; v += 32) {
    if (args.hL) args.hL[b * kLevels + v] = s.hSi[v] ? s.hL[s.posL[v]] : 0.0;
    if (args.hR) args.hR[b * kLevels + v] = 0.0;
  }
  __syncwarp();
  if (args.hR && row) args.hR[b * kLevels + ia] = hR;
  if (args.iters && lane == 0) args.iters[b] = t;

  // ---- Eq. 20: runs of index_1 (table) along the rows, summed per bin in row order ----
  uint32_t set1[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
  int cnt1 = 0, kmax1 = 0;
  const uint8_t* tab = args.idx1_tab + ia * kLevels;
  if (row) {
    int prev = -1;
    for (int c = 0; c < nL; ++c) {
      const int k = __ldg(tab + s.listL[c]);
      if (k != prev) {
        set_bit8(set1, k);
        ++cnt1;
        prev = k;
      }
    }
    kmax1 = prev;
  }
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) kmax1 = max(kmax1, __shfl_xor_sync(full, kmax1, d));
  __syncwarp();
  const int RT = warp_masks(s, set1, kmax1);
  if (RT > kRunCap) {
    if (lane == 0) deferred[b] = 1;
    return;
  }
  double* Tv = s.runE;
  if (row) {
    const uint32_t below = (1u << lane) - 1u;
    int prev = __ldg(tab + s.listL[0]);
    double acc = 0.0;
    for (int c = 0; c <= nL; ++c) {
      const int k = c < nL ? __ldg(tab + s.listL[c]) : -1;
      if (k != prev) {
        Tv[s.keyStart[prev] + __popc(s.mask[prev] & below)] = hR * acc;
        prev = k;
        acc = 0.0;
      }
      if (c < nL) acc += s.hL[c];
    }
  }
  __syncwarp();
  for (int k = lane; k < kLevels; k += 32) {
    const int k0 = s.keyStart[k], k1 = s.keyStart[k + 1];
    double e0 = 0.0, e1 = 0.0;
    int j = k0;
    for (; j + 1 < k1; j += 2) {
      e0 += Tv[j];
      e1 += Tv[j + 1];
    }
    if (j < k1) e0 += Tv[j];
    args.target[b * kLevels + k] = (e0 + e1) * invN;
  }
  if (lane == 0) deferred[b] = 0;
  WMARK(11);
#ifdef HR_SOLVE_PROFILE
  if (blockIdx.x == 0 && threadIdx.x == 0)
    for (int i = 0; i < 16; ++i) g_wclk[i] = wacc[i];
#endif
}

}  // namespace

#ifdef HR_SOLVE_PROFILE
}  // namespace hr
extern "C" int hr_debug_solve_warp_clocks(long long* out) {
  return (int)cudaMemcpyFromSymbol(out, hr::g_wclk, sizeof(long long) * 16);
}
namespace hr {
#endif

cudaError_t launch_solve_warp(const SolveArgs& a, int64_t B, int32_t* deferred, cudaStream_t st) {
  static bool attr = false;
  const size_t smem = sizeof(WarpSm) * kWPC;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_solve_warp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  k_solve_warp<<<(unsigned)((B + kWPC - 1) / kWPC), 32 * kWPC, smem, st>>>(a, B, deferred);
  return cudaGetLastError();
}

}  // namespace hr
