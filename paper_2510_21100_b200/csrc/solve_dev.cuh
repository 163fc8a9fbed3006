// solve_dev.cuh -- device body of kernel (b): one image of the histogram-domain Retinex
// solver (Algorithm 1, fp64) + Eq. 20 + the CDF/LUT tail (c).  Shared by k_solve (k_solve.cu)
// and the persistent fused kernel (k_fused.cu).
//
//
// One CTA (256 threads) per image, 2 CTAs per SM.  PAPER.md references:
//   Eq. 6  count matrix  C_ij = hR_i hL_j / N          -- never materialised
//   Eq. 7  location matrix b_i b_j (R1, R2)            -- constant: idx(i,j)
//   P:192           index(i,j) = nearest bin of b_i b_j          = (i*j + 127) div 255
//   Eq. 8  Est_k = sum_{idx(i,j)=k} C_ij (R3)
//   Eq. 11  K_ij = C_ij / Est_idx(i,j) (R8)
//   Eq. 13, Eq. 12, Eqs. 15, 14, Alg. 1 loop
//   Eqs. 17-20 enhanced histogram with index_1 (R4, R5)
//   P:308 histogram matching (R16)
//
// Factored form.  With rho_k = hS_k / EstRaw_k (EstRaw = N Est):
//   Eq. 13 (gradient-consistent, R7): hR'_i = (hR_i A_i / N + beta hG_i) / (sum hL^2/N^2 + beta),
//        A_i = sum_j hL_j^2 rho_idx(i,j)
//   Eq. 12: hL'_j = (hL_j B_j / N + alpha hS_j) / (sum hR'^2/N^2 + alpha),
//        B_j = sum_i hR'_i hR_i rho_idx(i,j)         (K frozen at iteration t, R10)
//   Paper-literal form (K_ij as a divisor): A_i = sum_j sigma_k / hR_i, sigma_k = hS_k EstRaw_k,
//        B_j = sum_i (hR'_i / hR_i) sigma_k / hL_j   (both divided by N).
// Supports never change (hR stays 0 off supp(hG), hL off supp(hS)), so all work runs over the
// nR x nL compacted cells only.
//
// Run structure.  index(i,j) is monotone in j, so each compacted row splits into a few RUNS
// of equal output bin k (found once per image by a row walk).  EstRaw_k is the sum over the
// runs of bin k of hR_a * (sum of hL over the run); a run's slot in the bin-ordered array is
// fixed by a per-bin bitmask of rows (rank = popc of the bits below its row), so every
// per-bin sum runs in row order: deterministic, no floating-point atomics, bit-identical run
// to run.  The R- and L-updates are thread-per-row / thread-per-column walks (no combine).
// The renormalisation of iteration t is folded into the run-sum phase of iteration t+1, so
// an iteration is four phases / four barriers:  E1 (renorm + run sums) | E2 (EstRaw, rho)
// | R (Eq. 13) | L (Eq. 12).  Eq. 20 reuses the run machinery with index_1.
#pragma once
#include "hr_common.cuh"

namespace hr {
namespace {

constexpr int T = kSolveThreads;
constexpr int NW = kSolveWarps;
// run arena: rr (u32 descriptor, bin order) + rowRun (u16) + runE, runS2 (double) per run
constexpr int kMaxRuns = 32896;              // sum_{i<256} (i + 1): bound on the runs of any image
constexpr int kMaskBytes = kLevels * 8 * 4;  // per-bin row bitmask (8 words per bin)
constexpr int kArenaSmem = 80 * 1024;
constexpr int kArenaGlobal = 720 * 1024;  // descriptors + row slots + run sums (22 B per run)
static_assert(kArenaGlobal >= 22 * kMaxRuns + 64, "global arena too small");

// Phase clock marks (measurement builds only: -DHR_SOLVE_PROFILE; block kProfBlock, thread 0).
#ifdef HR_SOLVE_PROFILE
__device__ long long g_solve_clk[1024];
__device__ int g_solve_nclk;
constexpr int kProfBlock = 0;
// thread 0 keeps the count in a register: a mark is a clock read and a fire-and-forget store
#define PROF_MARK()                                                                  \
  do {                                                                               \
    if (blockIdx.x == kProfBlock && threadIdx.x == 0 && prof_n < 1024) {             \
      g_solve_clk[prof_n++] = clock64();                                             \
      g_solve_nclk = prof_n;                                                         \
    }                                                                                \
  } while (0)
#else
#define PROF_MARK() \
  do {              \
  } while (0)
#endif

// slots of the block-reduction scratch
enum { R_SL2 = 0, R_SR1, R_SR2, R_SL1, R_DR, R_DL, kSlots };

struct __align__(16) Sm {
  double hR[kLevels], hL[kLevels];    // renormalised state (index a over sR, c over sL)
  double hR1[kLevels], hL1[kLevels];  // raw updates (Eq. 13 / Eq. 12 outputs)
  double hSc[kLevels], hGc[kLevels];  // priors at the support entries
  double hL2[kLevels];                // hL_c^2
  double wgt[kLevels];                // per-row weight of the L-walk
  double hSd[kLevels];                // dense hS as double
  double rho[kLevels];                // rho_k (GC) or sigma_k (paper-literal)
  double bk[kLevels];                 // b_k = k/255 (R1)
  double red[kSlots][NW];
  uint32_t hSi[kLevels], hGi[kLevels];
  int rowStart[kLevels + 1];  // run offsets per row
  int keyStart[kLevels + 1];  // run offsets per bin (bin order)
  uint8_t listR[kLevels], listL[kLevels];
  unsigned long long nw[NW];
  uint32_t bunion[8];  // union of the row bin sets (run_build)
};

__device__ __forceinline__ int idx0(int i, int j) {  // P:192 index(i,j) for l = 256
  return (int)(((uint32_t)(i * j + 127) * 32897u) >> 23);
}

// Sum over warps in fixed order (call after a barrier that follows the slot writes).
__device__ __forceinline__ double slot_sum(const Sm& s, int slot) {
  double a = 0.0;
#pragma unroll
  for (int w = 0; w < NW; ++w) a += s.red[slot][w];
  return a;
}

// Fixed-order warp reductions of up to three values at once (independent shuffle trees
// interleave, so three sums cost about the latency of one).
__device__ __forceinline__ void slot_put3(Sm& s, int s0, double v0, int s1, double v1, int s2, double v2) {
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) {
    v0 += __shfl_xor_sync(0xffffffffu, v0, d);
    v1 += __shfl_xor_sync(0xffffffffu, v1, d);
    v2 += __shfl_xor_sync(0xffffffffu, v2, d);
  }
  if ((threadIdx.x & 31) == 0) {
    const int w = threadIdx.x >> 5;
    s.red[s0][w] = v0;
    if (s1 >= 0) s.red[s1][w] = v1;
    if (s2 >= 0) s.red[s2][w] = v2;
  }
}


__device__ int block_scan_excl(int x, int* total, int* wscratch) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int v = x;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, v, d);
    if (lane >= d) v += u;
  }
  if (lane == 31) wscratch[w] = v;
  __syncthreads();
  int off = 0, tot = 0;
  for (int u = 0; u < NW; ++u) {
    if (u < w) off += wscratch[u];
    tot += wscratch[u];
  }
  __syncthreads();
  *total = tot;
  return off + v - x;
}


// index_1(i,j) of Eqs. 17-19: first k minimising |b_i p_j - b_k|, p_j = b_j^(1/gamma).
__device__ __forceinline__ int idx1(const double* bk, double bi, double pj) {
  const double x = __dmul_rn(bi, pj);  // rounded product (no contraction into the compare)
  int k0 = (int)floor(x * 255.0);
  int best = -1;
  double bd = 0.0;
#pragma unroll
  for (int d = -1; d <= 1; ++d) {
    const int k = k0 + d;
    if (k < 0 || k > 255) continue;
    const double dist = fabs(x - bk[k]);
    if (best < 0 || dist < bd) {
      bd = dist;
      best = k;
    }
  }
  return best;
}

// CDF + LUT (R16), shared by the solver tail and k_match.  T: dense target [256] in
// smem, hSi: dense counts in smem.  Uses Pt/Ct/Cs scratch (3 x 256 doubles).
__device__ void cdf_lut(const uint32_t* hSi, const double* Tt, double* Pt, double* Ct, double* Cs,
                        int* wscr, uint8_t* lut_out, int32_t* status_out) {
  const int tid = threadIdx.x, lane = tid & 31;
  // integer prefix of hS (exact in any order)
  unsigned long long v = hSi[tid];
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const unsigned long long u = __shfl_up_sync(0xffffffffu, v, d);
    if (lane >= d) v += u;
  }
  __shared__ unsigned long long wtot[NW];
  if (lane == 31) wtot[tid >> 5] = v;
  __syncthreads();
  unsigned long long off = 0, Ntot = 0;
  for (int u = 0; u < NW; ++u) {
    if (u < (tid >> 5)) off += wtot[u];
    Ntot += wtot[u];
  }
  const unsigned long long Ps = off + v;
  Cs[tid] = Ntot ? (double)Ps / (double)Ntot : 0.0;
  // plateau-preserving prefix of the target: lane-sequential blocks of 8, sequential carry
  if (tid < 32) {
    double loc[8];
    double acc = 0.0;
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      acc = (m == 0) ? Tt[8 * tid] : acc + Tt[8 * tid + m];
      loc[m] = acc;
    }
    // carry_l = carry_{l-1} + total_{l-1}, strictly sequential over lanes
    double carry = 0.0;
    for (int l = 0; l < 32; ++l) {
      const double tot = __shfl_sync(0xffffffffu, acc, l);
      if (l < tid) carry = carry + tot;  // carry for lane tid: sum in lane order
    }
#pragma unroll
    for (int m = 0; m < 8; ++m) Pt[8 * tid + m] = (tid == 0) ? loc[m] : carry + loc[m];
  }
  __syncthreads();
  const double last = Pt[kLevels - 1];
  const bool degenerate = !(last > 0.0) || Ntot == 0;
  Ct[tid] = degenerate ? 0.0 : Pt[tid] / last;
  __syncthreads();
  int res = tid;
  if (!degenerate) {
    const double x = Cs[tid];
    // k* = first k with Ct[k] >= x
    int lo = 0, hi = kLevels;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (Ct[mid] >= x) hi = mid; else lo = mid + 1;
    }
    const int ks = lo;  // <= 255 because Ct[255] == 1 >= x
    res = ks;
    if (ks > 0) {
      const double cprev = Ct[ks - 1];
      // first index of the plateau holding Ct[ks-1]
      int l2 = 0, h2 = ks - 1;
      while (l2 < h2) {
        const int mid = (l2 + h2) >> 1;
        if (Ct[mid] >= cprev) h2 = mid; else l2 = mid + 1;
      }
      const double d0 = fabs(cprev - x);
      const double d1 = fabs(Ct[ks] - x);
      if (d0 <= d1) res = l2;  // ties -> smallest k
    }
  }
  if (lut_out) lut_out[tid] = (uint8_t)res;
  if (status_out && tid == 0) *status_out = degenerate ? (int32_t)HR_EDEGENERATE : (int32_t)HR_OK;
  (void)wscr;
}

__device__ void remap_gradient(const uint32_t* graw, int grad_norm, uint32_t* hGi, int* wscr) {
  const int tid = threadIdx.x, lane = tid & 31;
  const uint32_t c0 = __ldcg(graw + tid), c1 = __ldcg(graw + tid + T);
  int m = c1 ? tid + T : (c0 ? tid : 0);
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, d));
  if (lane == 0) wscr[tid >> 5] = m;
  hGi[tid] = 0u;
  __syncthreads();
  int gmax = 0;
  for (int u = 0; u < NW; ++u) gmax = max(gmax, wscr[u]);
  auto level = [&](int g) -> int {
    if (grad_norm == 1) return g < 255 ? g : 255;                         // RAW_CLAMP
    return gmax == 0 ? 0 : (int)((510u * (uint32_t)g + (uint32_t)gmax) / (2u * (uint32_t)gmax));  // MAXNORM
  };
  if (c0) atomicAdd(&hGi[level(tid)], c0);
  if (c1) atomicAdd(&hGi[level(tid + T)], c1);
  __syncthreads();
}


// rank of row a among the rows whose bit is set in a bin's 8-word mask (bits below a)
__device__ __forceinline__ int mask_rank(const uint32_t* m, int a) {
  int r = 0;
  const int w = a >> 5;
  for (int u = 0; u < w; ++u) r += __popc(m[u]);
  return r + __popc(m[w] & ((1u << (a & 31)) - 1u));
}

// Run structure from the cached keys kc[a * nL + c] (monotone in c).  Per-bin row bitmasks:
// bit a of mask[k*8 + a/32] is set iff row a has a run of bin k.  Each row records its key
// set (8 words, owned by the row's thread: no atomics); the warp of rows 32w..32w+31 then
// transposes the 256 x 32 bit matrix with one ballot per bin.  keyStart = exclusive scan of
// the per-bin popcounts (bin-ordered run slots), rowStart = exclusive scan of the runs per
// row.  Returns the number of runs.
__device__ int run_build(Sm& s, int nR, int nL, const uint8_t* kc, uint32_t* mask, uint32_t* rowset, int* wscr) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid < 8) s.bunion[tid] = 0u;
  int kmax = 0, cnt = 0;
  if (tid < nR) {
    uint32_t* rs = rowset + tid * 8;
#pragma unroll
    for (int u = 0; u < 8; ++u) rs[u] = 0u;
    const uint8_t* kr = kc + tid * nL;
    int prev = -1;
    for (int c = 0; c < nL; ++c) {
      const int k = kr[c];
      if (k != prev) {
        rs[k >> 5] |= 1u << (k & 31);
        prev = k;
        ++cnt;
      }
    }
    kmax = prev;  // keys are non-decreasing along the row
  }
  int RR;
  const int rs0 = block_scan_excl(cnt, &RR, wscr);
  s.rowStart[tid] = rs0;
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, d));
  if (lane == 0) wscr[w] = kmax;
  __syncthreads();
  for (int u = 0; u < NW; ++u) kmax = max(kmax, wscr[u]);
  // transpose: the warp of rows 32w..32w+31 ballots each bin present in any row of the CTA
  // (the union of the row sets, 8 words, via shared memory); all other bins get 0 words
  {
    const int a = w * 32 + lane;
    uint32_t set[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) set[u] = (a < nR) ? rowset[a * 8 + u] : 0u;
    uint32_t uni[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      uint32_t x = set[u];
#pragma unroll
      for (int d = 16; d >= 1; d >>= 1) x |= __shfl_xor_sync(0xffffffffu, x, d);
      uni[u] = x;
    }
    if (lane == 0) {
#pragma unroll
      for (int u = 0; u < 8; ++u) atomicOr(&s.bunion[u], uni[u]);
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t all = s.bunion[u];
      mask[(u * 32 + lane) * 8 + w] = 0u;  // default; bins present are overwritten below
      __syncwarp();
      uint32_t rem = all;
      while (rem) {
        const int bit = __ffs(rem) - 1;
        rem &= rem - 1u;
        const uint32_t m = __ballot_sync(0xffffffffu, (set[u] >> bit) & 1u);
        if (lane == 0) mask[(u * 32 + bit) * 8 + w] = m;
      }
    }
  }
  (void)kmax;
  __syncthreads();
  int kcount = 0;
#pragma unroll
  for (int u = 0; u < 8; ++u) kcount += __popc(mask[tid * 8 + u]);
  int RK;
  const int ks = block_scan_excl(kcount, &RK, wscr);
  s.keyStart[tid] = ks;
  if (tid == 0) {
    s.keyStart[kLevels] = RK;
    s.rowStart[kLevels] = RR;
  }
  __syncthreads();
  return RR;
}

// slot of row a's run of bin k in the bin-ordered run array
__device__ __forceinline__ int run_slot(const Sm& s, const uint32_t* mask, int k, int a) {
  return s.keyStart[k] + mask_rank(mask + k * 8, a);
}

__host__ __device__ constexpr int align16(int x) { return (x + 15) & ~15; }

// fast fp64 reciprocal: MUFU.RCP64H seed and two Newton steps (within ~1 ulp)
__device__ __forceinline__ double rcp_fast(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// Algorithm 1 iterations over the run arena (SM: arena in shared memory).  Returns t.
// Arena: rr (descriptors, bin order) | rowRun (slots in row order) | runE | runS2.
// Four phases per update, each closed by a barrier:
//   E1  renormalise the raw iterates of the previous update (Eqs. 15, 14) and, one thread per
//       run, the run sums hR_a * sum(hL) and sum(hL^2) over the run (Eqs. 6, 8)
//   E2  one thread per bin: EstRaw_k over the bin's runs in row order, rho_k (Eq. 11 folded)
//   R   one thread per row: A_a over the row's runs, Eq. 13
//   L   one thread per column: B_c over the rows, Eq. 12 with the frozen K
template <bool SM>
__device__ __forceinline__ int iterate(Sm& s, const hr_params& P, int nR, int nL, int RR, double N,
                                       unsigned char* arena, int off) {
  const int tid = threadIdx.x;
  const uint32_t* rr = reinterpret_cast<const uint32_t*>(arena + off);
  const uint16_t* rowRun = reinterpret_cast<const uint16_t*>(arena + off + align16(4 * RR));
  double* runE = reinterpret_cast<double*>(arena + off + align16(4 * RR) + align16(2 * RR));
  double* runS2 = runE + RR;
  const int form = P.update_form;
  const double invN = 1.0 / N, invN2 = invN * invN;
  double SR1 = N, SL1 = N;  // sums of the raw iterates (initially exactly N)
  int t = 0;
#ifdef HR_SOLVE_PROFILE
  long long pacc[6] = {0, 0, 0, 0, 0, 0}, pt0 = clock64(), pt1;
#define PHASE(i) do { pt1 = clock64(); pacc[i] += pt1 - pt0; pt0 = pt1; } while (0)
#else
#define PHASE(i) do { } while (0)
#endif
  for (;;) {
    // ======== E1: renormalise (Eqs. 15, 14); run sums of hL and hL^2 (Eqs. 6, 8) ========
    {
      const double cR = N * rcp_fast(SR1), cL = N * rcp_fast(SL1), cRL = cR * cL, cL2 = cL * cL;
      double dr = 0.0, dl = 0.0, q = 0.0;
      if (tid < nR) {
        const double n = cR * s.hR1[tid];
        dr = (n - s.hR[tid]) * (n - s.hR[tid]);
        s.hR[tid] = n;
      }
      if (tid < nL) {
        const double n = cL * s.hL1[tid];
        dl = (n - s.hL[tid]) * (n - s.hL[tid]);
        s.hL[tid] = n;
        s.hL2[tid] = n * n;
        q = n * n;
      }
      for (int r = tid; r < RR; r += T) {
        const uint32_t d = rr[r];
        const int lo = (d >> 8) & 255, hi = (d >> 16) & 255, ra = d >> 24;
        double s0 = 0.0, s1 = 0.0, q0 = 0.0, q1 = 0.0;
        int c = lo;
        for (; c + 1 <= hi; c += 2) {
          const double x0 = s.hL1[c], x1 = s.hL1[c + 1];
          s0 += x0;
          s1 += x1;
          q0 = fma(x0, x0, q0);
          q1 = fma(x1, x1, q1);
        }
        if (c <= hi) {
          const double x0 = s.hL1[c];
          s0 += x0;
          q0 = fma(x0, x0, q0);
        }
        runE[r] = s.hR1[ra] * (s0 + s1) * cRL;
        runS2[r] = (q0 + q1) * cL2;
      }
      slot_put3(s, R_DR, dr, R_DL, dl, R_SL2, q);
    }
    __syncthreads();
    PHASE(0);
    if (t > 0) {  // stop rule (R11) on the renormalised iterates of update t
      const double eps = P.epsilon * N * N;
      const bool conv = P.use_epsilon && slot_sum(s, R_DR) <= eps && slot_sum(s, R_DL) <= eps;
      if (conv || t >= P.max_iter) break;
    }
    // ======== E2: EstRaw_k over the bin's runs in row order; rho_k (Eq. 11 folded) ========
    {
      const int k = tid, k0 = s.keyStart[k], k1 = s.keyStart[k + 1];
      if (k0 < k1) {
        double e0 = 0.0, e1 = 0.0;
        int j = k0;
        for (; j + 1 < k1; j += 2) {
          e0 += runE[j];
          e1 += runE[j + 1];
        }
        if (j < k1) e0 += runE[j];
        const double e = e0 + e1;  // EstRaw_k (Eqs. 6, 8)
        s.rho[k] = form == 0 ? (e > 0.0 ? s.hSd[k] * rcp_fast(e) : 0.0) : s.hSd[k] * e;
      }
    }
    const double invDenR = rcp_fast(slot_sum(s, R_SL2) * invN2 + P.beta);
    __syncthreads();
    PHASE(1);
    // ======== R: Eq. 13, one thread per row walking the row's cells ========
    {
      double v = 0.0;
      if (tid < nR) {
        const int ia = s.listR[tid];
        double a0 = 0.0, a1 = 0.0;
        int c = 0;
        if (form == 0) {
          for (; c + 1 < nL; c += 2) {
            a0 = fma(s.hL2[c], s.rho[idx0(ia, s.listL[c])], a0);
            a1 = fma(s.hL2[c + 1], s.rho[idx0(ia, s.listL[c + 1])], a1);
          }
          if (c < nL) a0 = fma(s.hL2[c], s.rho[idx0(ia, s.listL[c])], a0);
        } else {
          for (; c + 1 < nL; c += 2) {
            a0 += s.rho[idx0(ia, s.listL[c])];
            a1 += s.rho[idx0(ia, s.listL[c + 1])];
          }
          if (c < nL) a0 += s.rho[idx0(ia, s.listL[c])];
        }
        const double A = a0 + a1, hr = s.hR[tid];
        const double num = form == 0 ? hr * A * invN : A * rcp_fast(N * hr);
        v = (num + P.beta * s.hGc[tid]) * invDenR;
        v = v > 0.0 ? v : 0.0;
        s.hR1[tid] = v;
        s.wgt[tid] = form == 0 ? v * hr : v * rcp_fast(hr);
      }
      slot_put3(s, R_SR1, v, R_SR2, v * v, -1, 0.0);
    }
    __syncthreads();
    PHASE(2);
    // ======== L: Eq. 12 (frozen K), one thread per column over the rows ========
    {
      const double invDenL = rcp_fast(slot_sum(s, R_SR2) * invN2 + P.alpha);
      double u = 0.0;
      if (tid < nL) {
        const int jc = s.listL[tid];
        double b0 = 0.0, b1 = 0.0;
        int a = 0;
        for (; a + 1 < nR; a += 2) {
          b0 = fma(s.wgt[a], s.rho[idx0(s.listR[a], jc)], b0);
          b1 = fma(s.wgt[a + 1], s.rho[idx0(s.listR[a + 1], jc)], b1);
        }
        if (a < nR) b0 = fma(s.wgt[a], s.rho[idx0(s.listR[a], jc)], b0);
        const double Bv = b0 + b1, hl = s.hL[tid];
        const double num = form == 0 ? hl * Bv * invN : Bv * rcp_fast(N * hl);
        u = (num + P.alpha * s.hSc[tid]) * invDenL;
        u = u > 0.0 ? u : 0.0;
        s.hL1[tid] = u;
      }
      slot_put3(s, R_SL1, u, -1, 0.0, -1, 0.0);
    }
    __syncthreads();
    PHASE(3);
    ++t;
    SR1 = slot_sum(s, R_SR1);
    SL1 = slot_sum(s, R_SL1);
  }
#ifdef HR_SOLVE_PROFILE
  if (blockIdx.x == kProfBlock && threadIdx.x == 0)
    for (int i = 0; i < 6; ++i) g_solve_clk[512 + i] = pacc[i];
#endif
#undef PHASE
  return t;
}

// Eq. 20 run values Tv (bin order) from the cached index_1 keys kc1, then the dense target.
template <bool SM>
__device__ __forceinline__ void target_runs(Sm& s, int nR, int nL, const uint8_t* kc1, const uint32_t* mask,
                                            double* Tv, double invN, double* Tt) {
  const int tid = threadIdx.x;
  if (tid < nR) {  // every run of row a: hR_a * sum(hL over the run) at its bin-order slot
    const double hr = s.hR[tid];
    const uint8_t* kr = kc1 + tid * nL;
    int prev = kr[0];
    double acc = s.hL[0];
    for (int c = 1; c < nL; ++c) {
      const int k = kr[c];
      if (k != prev) {
        Tv[run_slot(s, mask, prev, tid)] = hr * acc;
        prev = k;
        acc = 0.0;
      }
      acc += s.hL[c];
    }
    Tv[run_slot(s, mask, prev, tid)] = hr * acc;
  }
  __syncthreads();
  const int k = tid, k0 = s.keyStart[k], k1 = s.keyStart[k + 1];
  double e0 = 0.0, e1 = 0.0;
  int j = k0;
  for (; j + 1 < k1; j += 2) {
    e0 += Tv[j];
    e1 += Tv[j + 1];
  }
  if (j < k1) e0 += Tv[j];
  Tt[k] = (e0 + e1) * invN;
}

// One image of Algorithm 1 + Eq. 20 + the CDF/LUT tail, by all T threads of the CTA.
// smraw: solve_smem_bytes() of shared memory; wscr: NW ints of shared scratch.  Every exit is
// CTA-uniform.  Histograms are read through L2 (__ldcg): in the fused kernel they were
// accumulated by other CTAs' atomics during this launch.
__device__ __forceinline__ void solve_image(const SolveArgs& args, const int64_t b, unsigned char* smraw, int* wscr) {
#ifdef HR_SOLVE_PROFILE
  int prof_n = 0;
#endif
  PROF_MARK();
  Sm& s = *reinterpret_cast<Sm*>(smraw);
  unsigned char* arenaS = smraw + sizeof(Sm);
  // shared arena tail: [ ... | rowset 8 KB | mask 8 KB ]
  uint32_t* mask = reinterpret_cast<uint32_t*>(arenaS + kArenaSmem - kMaskBytes);
  uint32_t* rowset = reinterpret_cast<uint32_t*>(arenaS + kArenaSmem - 2 * kMaskBytes);
  const int tid = threadIdx.x;
  const hr_params& P = args.p;
  if (args.only_deferred && args.only_deferred[b] == 0) return;  // solved by k_solve_warp

  // ---- histograms (Alg. 1 init) ----
  s.hSi[tid] = __ldcg(args.hist_s + b * kLevels + tid);
  if (args.hist_g) {
    s.hGi[tid] = __ldcg(args.hist_g + b * kLevels + tid);
  } else {
    remap_gradient(args.graw + b * kGradSlots, args.grad_norm, s.hGi, wscr);
  }
  s.bk[tid] = (double)tid / 255.0;
  s.hSd[tid] = (double)s.hSi[tid];
  __syncthreads();
  PROF_MARK();

  // ---- supports (fixed for all t) ----
  const bool fL = s.hSi[tid] != 0u, fR = s.hGi[tid] != 0u;
  int nL, nR;
  const int pL = block_scan_excl(fL ? 1 : 0, &nL, wscr);
  const int pR = block_scan_excl(fR ? 1 : 0, &nR, wscr);
  if (fL) s.listL[pL] = (uint8_t)tid;
  if (fR) s.listR[pR] = (uint8_t)tid;
  {
    unsigned long long v = s.hSi[tid];
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    if ((tid & 31) == 0) s.nw[tid >> 5] = v;
  }
  __syncthreads();
  PROF_MARK();
  unsigned long long Nint = 0;
  for (int u = 0; u < NW; ++u) Nint += s.nw[u];
  const double N = (double)Nint;
  if (Nint == 0 || nR == 0) {  // empty image: zero outputs (never for validated inputs)
    if (args.hL) args.hL[b * kLevels + tid] = 0.0;
    if (args.hR) args.hR[b * kLevels + tid] = 0.0;
    if (args.target) args.target[b * kLevels + tid] = 0.0;
    if (args.lut) args.lut[b * kLevels + tid] = (uint8_t)tid;
    if (tid == 0) {
      if (args.iters) args.iters[b] = 0;
      if (args.status) args.status[b] = HR_EDEGENERATE;
    }
    return;
  }

  // ---- initial state: hR^0 = hG, hL^0 = hS (R9), as raw iterates whose sums are N ----
  if (tid < nL) {
    const double v = s.hSd[s.listL[tid]];
    s.hL1[tid] = v;
    s.hSc[tid] = v;
    s.hL[tid] = v;
  }
  if (tid < nR) {
    const double v = (double)s.hGi[s.listR[tid]];
    s.hR1[tid] = v;
    s.hGc[tid] = v;
    s.hR[tid] = v;
  }

  // ---- runs of index(i,j) along each compacted row (fixed for all t) ----
  // keys kc (u8 per cell, always fits: E <= 65536 <= arena - 16 KB) at the arena start
  const int E = nR * nL;
  uint8_t* kc = arenaS;
  for (int e = tid; e < E; e += T) {
    const int a = e / nL, c = e - a * nL;
    kc[e] = (uint8_t)idx0(s.listR[a], s.listL[c]);
  }
  __syncthreads();
  const int RR = run_build(s, nR, nL, kc, mask, rowset, wscr);
  // rr | rowRun after kc, clear of the live mask; runE | runS2 may overlap the mask
  const int rrBytes = align16(4 * RR) + align16(2 * RR);
  const bool inSmem = align16(E) + rrBytes <= kArenaSmem - kMaskBytes &&
                      align16(E) + rrBytes + 16 * RR <= kArenaSmem;
  unsigned char* arena = inSmem ? arenaS : args.cells_ws + b * (int64_t)kArenaGlobal;
  const int off = inSmem ? align16(E) : 0;
  {
    uint32_t* rr = reinterpret_cast<uint32_t*>(arena + off);
    uint16_t* rowRun = reinterpret_cast<uint16_t*>(arena + off + align16(4 * RR));
    if (tid < nR) {  // descriptor k | lo << 8 | hi << 16 | a << 24 at the run's bin-order slot
      const uint8_t* kr = kc + tid * nL;
      int prev = kr[0], lo = 0, i = s.rowStart[tid];
      for (int c = 1; c < nL; ++c) {
        const int k = kr[c];
        if (k != prev) {
          const int slot = run_slot(s, mask, prev, tid);
          rr[slot] = (uint32_t)prev | ((uint32_t)lo << 8) | ((uint32_t)(c - 1) << 16) | ((uint32_t)tid << 24);
          rowRun[i++] = (uint16_t)slot;
          prev = k;
          lo = c;
        }
      }
      const int slot = run_slot(s, mask, prev, tid);
      rr[slot] = (uint32_t)prev | ((uint32_t)lo << 8) | ((uint32_t)(nL - 1) << 16) | ((uint32_t)tid << 24);
      rowRun[i] = (uint16_t)slot;
    }
  }
  __syncthreads();
  PROF_MARK();

  const int t = inSmem ? iterate<true>(s, P, nR, nL, RR, N, arenaS, off)
                       : iterate<false>(s, P, nR, nL, RR, N, arena, off);
  PROF_MARK();

  // ---- outputs hL, hR (dense, zero off support) ----
  if (args.hL) args.hL[b * kLevels + tid] = fL ? s.hL[pL] : 0.0;
  if (args.hR) args.hR[b * kLevels + tid] = fR ? s.hR[pR] : 0.0;
  if (args.iters && tid == 0) args.iters[b] = t;

  // ---- Eq. 20: runs of index_1 (Eqs. 17-19) along each row, summed per bin in row order ----
  // index_1 of every cell from the per-gamma table (built once per gamma by k_idx1_table)
  uint8_t* kc1 = arenaS;
  for (int e = tid; e < E; e += T) {
    const int a = e / nL, c = e - a * nL;
    kc1[e] = __ldg(args.idx1_tab + s.listR[a] * kLevels + s.listL[c]);
  }
  __syncthreads();
  const int RT = run_build(s, nR, nL, kc1, mask, rowset, wscr);
  double* Tt = s.rho;  // dense target
  if (align16(E) + 8 * RT <= kArenaSmem - kMaskBytes)
    target_runs<true>(s, nR, nL, kc1, mask, reinterpret_cast<double*>(arenaS + align16(E)), 1.0 / N, Tt);
  else
    target_runs<false>(s, nR, nL, kc1, mask, reinterpret_cast<double*>(args.cells_ws + b * (int64_t)kArenaGlobal),
                       1.0 / N, Tt);
  if (args.target) args.target[b * kLevels + tid] = Tt[tid];
  __syncthreads();
  PROF_MARK();
  if (args.lut || args.status)
    cdf_lut(s.hSi, Tt, s.hL1, s.wgt, s.hL2, wscr, args.lut ? args.lut + b * kLevels : nullptr,
            args.status ? args.status + b : nullptr);
}


}  // namespace
}  // namespace hr
