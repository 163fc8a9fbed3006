// solve_dev.cuh -- device body of kernel (b): one image of the histogram-domain Retinex
// solver (Algorithm 1, fp64) + Eq. 20 + the CDF/LUT tail (c), launched by k_solve (k_solve.cu).
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
// Chunk structure.  index(i,j) is monotone in j, so each compacted row splits into a few RUNS
// of equal output bin k.  The cells are laid out in BIN order (bin, then row, then column; a
// run's place among its bin's runs is fixed by a per-bin bitmask of rows: rank = popc of the
// bits below its row) and cut into chunks of 8 cells that never straddle a bin.  EstRaw_k is the
// sum of the bin's chunk sums in that order: deterministic, no floating-point atomics,
// bit-identical run to run.  The R- and L-updates are walks over a row / a column by 1-8 lanes.
// The iterates stay raw; the renormalisation factors of Eqs. 15, 14 are scalars applied where a
// renormalised value enters, so an iteration is four phases / four barriers:
//   E1 (chunk sums of the cell products) | E2 (EstRaw, rho) | R (Eq. 13) | L (Eq. 12).
// Eq. 20 sums hR_a hL_c per index_1 key by dense per-row run sums (no second chunk structure).
#pragma once
#include "hr_common.cuh"

namespace hr {
namespace {

// Thread count T of a solver CTA is a template parameter: 256 (batched; 2 CTAs per SM) or 512
// (few images: one CTA per SM, the cell loops spread over twice the warps).  Bin-indexed steps
// use threads 0..255 (thread k <-> bin k); the others only join the cell loops and barriers.
constexpr int kMaxSW = 16;  // warps of the widest solver CTA
// Chunk arena (per image): runs = maximal equal-key segments of a compacted row; the cells in BIN
// order (bin, then row, then column), kChunk per chunk, a bin's last chunk padded:
//   pDesc [8 P] u32  per cell: (byte offset of hR1_a) | (byte offset of hL1_c) << 16; an unused
//                    slot points at hL1[256] = 0                                  (persistent)
//   pVal  [P] f64    chunk sums                   (persistent; build scratch before that:
//                    runDesc [RR] u32 row order k | lo << 8 | hi << 16 | a << 24, and the
//                    bin-ordered per-run cell counts / offsets [RR] u32)
//   s.keyStart[k] = first chunk of bin k
constexpr int kMaxRuns = 32896;                        // sum_{i<256} (i + 1): runs of any image
constexpr int kChunk = 8;                              // cells per chunk
constexpr int kMaxChunks = 65536 / kChunk + 256;       // each bin's last chunk may be partial
constexpr int kMaskBytes = kLevels * 8 * 4;            // per-bin row bitmask (8 words per bin)
constexpr int kArenaSmem = 80 * 1024;  // default shared arena: keys (E bytes) + run arena + mask tail
constexpr int kKeysGlobal = 65536;      // keys of images whose keys do not fit the shared arena
// per-image global arena: descriptors + max(values, build scratch), then keys
constexpr int kArenaRun = 4 * kChunk * kMaxChunks + 8 * kMaxRuns + 256;
constexpr int kArenaGlobal = kArenaRun + kKeysGlobal;

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
// fixed-slot marks (run_build steps, Eq. 20 steps): g_solve_clk[600 + slot]
#define SLOT_MARK(slot)                                                                \
  do {                                                                                 \
    if (blockIdx.x == kProfBlock && threadIdx.x == 0) g_solve_clk[600 + (slot)] = clock64(); \
  } while (0)
#else
#define PROF_MARK() \
  do {              \
  } while (0)
#define SLOT_MARK(slot) \
  do {                  \
  } while (0)
#endif

// slots of the block-reduction scratch
enum { R_SL2 = 0, R_SR1, R_SR2, R_SL1, R_DR, R_DL, R_QL1, R_OBJ, kSlots };

struct __align__(16) Sm {
  double hR[kLevels], hL[kLevels];    // renormalised state (index a over sR, c over sL)
  double hR1[kLevels], hL1[kLevels + 2];  // raw updates (Eq. 13 / Eq. 12 outputs); hL1[256] = 0: the
                                          // factor of a chunk's unused cell slots
  double hSc[kLevels], hGc[kLevels];  // priors at the support entries
  double hL2[kLevels];                // hL_c^2
  double wgt[kLevels];                // per-row weight of the L-walk
  double hSd[kLevels];                // dense hS as double
  double rho[kLevels];                // rho_k (GC) or sigma_k (paper-literal)
  double bk[kLevels];                 // b_k = k/255 (R1)
  double red[kSlots][kMaxSW];
  uint32_t hSi[kLevels], hGi[kLevels];
  int keyStart[kLevels + 1];  // chunk offsets per bin (bin order)
  alignas(16) int pStart[kLevels];      // run_build (chunks): a bin's first chunk; Eq. 20: packed row ranges
  int cBase[kLevels];                   // run_build (chunks): a bin's first cell
  uint8_t listR[kLevels], listL[kLevels];
  uint8_t binList[kLevels];   // the bins holding chunks, ascending (E2: lanes per bin)
  int nBins;
  unsigned long long nw[kMaxSW];
};

__device__ __forceinline__ int idx0(int i, int j) {  // P:192 index(i,j) for l = 256
  return (int)(((uint32_t)(i * j + 127) * 32897u) >> 23);
}

// Sum over warps in fixed order (call after a barrier that follows the slot writes).
template <int T>
__device__ __forceinline__ double slot_sum(const Sm& s, int slot) {
  constexpr int NW = T / 32;
  static_assert(NW % 2 == 0, "pairs of warp partials");
  double x[NW];
#pragma unroll
  for (int w = 0; w < NW; w += 2) {  // 16-B loads, then a pairwise tree in warp order
    const double2 v = *reinterpret_cast<const double2*>(&s.red[slot][w]);
    x[w] = v.x;
    x[w + 1] = v.y;
  }
#pragma unroll
  for (int d = 1; d < NW; d <<= 1)
#pragma unroll
    for (int w = 0; w + d < NW; w += 2 * d) x[w] += x[w + d];
  return x[0];
}

// Fixed-order warp reductions of up to three values at once (independent shuffle trees
// interleave, so three sums cost about the latency of one).
// (from > 1: only lanes that are multiples of `from` hold values -- the others hold copies or
// zero -- so the levels below `from` are skipped)
__device__ __forceinline__ void slot_put3(Sm& s, int s0, double v0, int s1, double v1, int s2, double v2,
                                          int from = 1) {
  for (int d = 16; d >= from; d >>= 1) {
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


template <int T>
__device__ int block_scan_excl(int x, int* total, int* wscratch) {
  constexpr int NW = T / 32;
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
template <int T>
__device__ void cdf_lut(const uint32_t* hSi, const double* Tt, double* Pt, double* Ct, double* Cs,
                        int* wscr, uint8_t* lut_out, int32_t* status_out) {
  constexpr int NB = kLevels / 32;  // warps holding bins (thread k <-> bin k)
  const int tid = threadIdx.x, lane = tid & 31;
  const bool bin = tid < kLevels;
  // integer prefix of hS (exact in any order)
  unsigned long long v = bin ? hSi[tid] : 0ull;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const unsigned long long u = __shfl_up_sync(0xffffffffu, v, d);
    if (lane >= d) v += u;
  }
  __shared__ unsigned long long wtot[NB];
  if (lane == 31 && bin) wtot[tid >> 5] = v;
  __syncthreads();
  unsigned long long off = 0, Ntot = 0;
  for (int u = 0; u < NB; ++u) {
    if (u < (tid >> 5)) off += wtot[u];
    Ntot += wtot[u];
  }
  const unsigned long long Ps = off + v;
  if (bin) Cs[tid] = Ntot ? (double)Ps / (double)Ntot : 0.0;
  // plateau-preserving prefix of the target: lane-sequential blocks of 8, sequential carry
  if (tid < 32) {
    double loc[8];
    double acc = 0.0;
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      acc = (m == 0) ? Tt[8 * tid] : acc + Tt[8 * tid + m];
      loc[m] = acc;
    }
    // carry_l = carry_{l-1} + total_{l-1}, strictly sequential over lanes: lane 0 adds the 32
    // totals in order (loads first, then one dependent add per lane) -- Ct is free until the
    // barrier below: [0, 32) the totals, [32, 64) the carries
    Ct[tid] = acc;
    __syncwarp();
    if (tid == 0) {
      double tot[32];
#pragma unroll
      for (int l = 0; l < 32; ++l) tot[l] = Ct[l];
      double c = 0.0;
#pragma unroll
      for (int l = 0; l < 32; ++l) {
        Ct[32 + l] = c;
        c = c + tot[l];
      }
    }
    __syncwarp();
    const double carry = Ct[32 + tid];
#pragma unroll
    for (int m = 0; m < 8; ++m) Pt[8 * tid + m] = (tid == 0) ? loc[m] : carry + loc[m];
  }
  __syncthreads();
  const double last = Pt[kLevels - 1];
  const bool degenerate = !(last > 0.0) || Ntot == 0;
  if (bin) Ct[tid] = degenerate ? 0.0 : Pt[tid] / last;
  __syncthreads();
  int res = tid;
  if (bin && !degenerate) {
    const double x = Cs[tid];
    // first k with Ct[k] >= y (Ct non-decreasing, Ct[255] >= y): a 16-ary search, two rounds of
    // 16 independent loads instead of 8 dependent ones
    auto lower = [&](double y) -> int {
      int j = 0;
#pragma unroll
      for (int i = 0; i < 16; ++i) j += Ct[16 * i + 15] < y ? 1 : 0;
      j = j < 15 ? j : 15;
      const double2* seg = reinterpret_cast<const double2*>(Ct + 16 * j);
      int n = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const double2 v = seg[i];
        n += (v.x < y ? 1 : 0) + (v.y < y ? 1 : 0);
      }
      return 16 * j + (n < 15 ? n : 15);
    };
    const int ks = lower(x);  // <= 255 because Ct[255] == 1 >= x
    res = ks;
    if (ks > 0) {
      const double cprev = Ct[ks - 1];
      const int l2 = lower(cprev);  // first index of the plateau holding Ct[ks-1] (<= ks - 1)
      const double d0 = fabs(cprev - x);
      const double d1 = fabs(Ct[ks] - x);
      if (d0 <= d1) res = l2;  // ties -> smallest k
    }
  }
  if (lut_out && bin) lut_out[tid] = (uint8_t)res;
  if (status_out && tid == 0) *status_out = degenerate ? (int32_t)HR_EDEGENERATE : (int32_t)HR_OK;
  (void)wscr;
}

template <int T>
__device__ void remap_gradient(const uint32_t* graw, int grad_norm, uint32_t* hGi, int* wscr) {
  constexpr int NW = T / 32;
  static_assert(2 * 256 == kGradSlots && (T == 256 || T == 512), "gradient slots per thread");
  const int tid = threadIdx.x, lane = tid & 31;
  // slots tid and tid + 256 (T = 256) or tid (T = 512)
  const uint32_t c0 = __ldcg(graw + tid), c1 = T == 256 ? __ldcg(graw + tid + 256) : 0u;
  int m = c1 ? tid + 256 : (c0 ? tid : 0);
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, d));
  if (lane == 0) wscr[tid >> 5] = m;
  if (tid < kLevels) hGi[tid] = 0u;
  __syncthreads();
  int gmax = 0;
  for (int u = 0; u < NW; ++u) gmax = max(gmax, wscr[u]);
  auto level = [&](int g) -> int {
    if (grad_norm == 1) return g < 255 ? g : 255;                         // RAW_CLAMP
    return gmax == 0 ? 0 : (int)((510u * (uint32_t)g + (uint32_t)gmax) / (2u * (uint32_t)gmax));  // MAXNORM
  };
  if (c0) atomicAdd(&hGi[level(tid)], c0);
  if (c1) atomicAdd(&hGi[level(tid + 256)], c1);
  __syncthreads();
}


// rank of row a among the rows whose bit is set in a bin's 8-word mask (bits below a)
__device__ __forceinline__ int mask_rank(const uint32_t* m, int a) {
  int r = 0;
  const int w = a >> 5;
  for (int u = 0; u < w; ++u) r += __popc(m[u]);
  return r + __popc(m[w] & ((1u << (a & 31)) - 1u));
}

__host__ __device__ constexpr int align16(int x) { return (x + 15) & ~15; }

// (row, column) of the cells e = tid, tid + T, ... of an n-column matrix without a division per
// cell (an integer division by a run-time value is ~25 instructions with two conversions)
template <int T>
struct CellCursor {
  int a, c, da, dc, n;
  __device__ CellCursor(int tid, int n_) : n(n_) {
    a = tid / n_;
    c = tid - a * n_;
    da = T / n_;
    dc = T - da * n_;
  }
  __device__ __forceinline__ void step() {
    a += da;
    c += dc;
    if (c >= n) {
      c -= n;
      ++a;
    }
  }
};

struct RunArena {
  uint32_t* pDesc;
  double* pVal;
  int RR, P;
};

// Run + chunk structure of the keys keys[a * nL + c] (non-decreasing in c), built in
// parallel over cells: thread t owns cells [E t / T, E (t+1) / T).  A cell starts a run when
// c == 0 or its key differs from the left neighbour; a block scan numbers the runs in row
// order.  Each run sets its row's bit in the bin's mask (atomicOr: the result is order-free);
// its bin-ordered slot = (runs of smaller bins) + rank of its row among the bin's rows.  A
// scan of the per-slot run lengths gives every run's first cell in bin order, a scan of the
// bins' chunk counts each bin's first chunk: the CELLS are written in bin order (bin, then row,
// then column), kChunk per chunk, chunks never straddling a bin (a bin's last chunk is padded
// with slots whose factor is hL1[256] = 0): chunk p = pDesc[8p .. 8p + 8), a cell = (byte offset
// of hR1_a) | (byte offset of hL1_c) << 16; s.keyStart = chunk offsets per bin.  The E1 phase is
// then one chunk (8 independent products, a fixed tree) per thread with ~E / 8 + (bins) chunks
// in all -- pieces of single runs are mostly 1-2 cells long when the rows are sparse (a MAXNORM
// gradient support): ~5 per thread on C3.  Placement: after the keys in shared memory when it
// fits (mask tail excluded), else arenaG.
template <int T>
__device__ void run_build(Sm& s, int nR, int nL, const uint8_t* keys, uint32_t* mask, unsigned char* arenaS,
                          int arenaBytes, bool keysInSmem, unsigned char* arenaG, RunArena& A, int* wscr,
                          int pslot = 0) {
  const int tid = threadIdx.x;
  SLOT_MARK(pslot + 0);
  const int E = nR * nL;
  for (int i = tid; i < kLevels * 8; i += T) mask[i] = 0u;
  const int e0 = (int)((long long)E * tid / T), e1 = (int)((long long)E * (tid + 1) / T);
  int cnt = 0;
  {
    int c = e0 % nL;
    int prev = (e0 < e1 && c > 0) ? keys[e0 - 1] : -1;
    for (int e = e0; e < e1; ++e) {
      const int k = keys[e];
      cnt += (c == 0 || k != prev) ? 1 : 0;
      prev = k;
      if (++c == nL) c = 0;
    }
  }
  int RR;
  int r = block_scan_excl<T>(cnt, &RR, wscr);
  SLOT_MARK(pslot + 1);
  const int Pmax = E / kChunk + kLevels;
  HR_CHECK(RR >= nR && RR <= E && RR <= kMaxRuns);
  const int keysS = keysInSmem ? align16(E) : 0;
  const int descB = align16(4 * kChunk * Pmax);
  const int valB = 8 * (Pmax > RR ? Pmax : RR);  // chunk sums; the build scratch before that
  const bool sm = keysS + descB + valB <= arenaBytes - kMaskBytes;
  unsigned char* base = sm ? arenaS + keysS : arenaG;
  A.pDesc = reinterpret_cast<uint32_t*>(base);
  A.pVal = reinterpret_cast<double*>(base + descB);
  A.RR = RR;
  uint32_t* runDesc = reinterpret_cast<uint32_t*>(A.pVal);  // build scratch under pVal
  uint32_t* slotN = runDesc + RR;                           // bin order: cell counts, then offsets
  {  // descriptors with hi provisional (fixed below)
    int a = e0 / nL, c = e0 - a * nL;
    int prev = (e0 < e1 && c > 0) ? keys[e0 - 1] : -1;
    for (int e = e0; e < e1; ++e) {
      const int k = keys[e];
      if (c == 0 || k != prev) runDesc[r++] = (uint32_t)k | ((uint32_t)c << 8) | ((uint32_t)a << 24);
      prev = k;
      if (++c == nL) {
        c = 0;
        ++a;
      }
    }
  }
  __syncthreads();
  SLOT_MARK(pslot + 2);
  // hi = next run's lo - 1 in the same row (else nL - 1); bin masks
  const int r0 = (int)((long long)RR * tid / T), r1 = (int)((long long)RR * (tid + 1) / T);
  for (int q = r0; q < r1; ++q) {
    const uint32_t d = runDesc[q];
    const int a = d >> 24, k = d & 255;
    int hi = nL - 1;
    if (q + 1 < RR) {
      const uint32_t dn = runDesc[q + 1];
      if ((int)(dn >> 24) == a) hi = (int)((dn >> 8) & 255) - 1;
    }
    runDesc[q] = d | ((uint32_t)hi << 16);
    atomicOr(&mask[k * 8 + (a >> 5)], 1u << (a & 31));
  }
  __syncthreads();
  int kcount = 0;
#pragma unroll
  for (int u = 0; u < 8; ++u) kcount += tid < kLevels ? __popc(mask[tid * 8 + u]) : 0;
  SLOT_MARK(pslot + 3);
  int RK;
  const int kfirst = block_scan_excl<T>(kcount, &RK, wscr);  // first run slot of bin tid
  if (tid < kLevels) s.keyStart[tid] = kfirst;
  __syncthreads();
  for (int q = r0; q < r1; ++q) {  // cell count at the run's bin-order slot
    const uint32_t d = runDesc[q];
    const int a = d >> 24, lo = (d >> 8) & 255, hi = (d >> 16) & 255, k = d & 255;
    HR_CHECK(lo <= hi && hi < nL && a < nR);
    HR_CHECK(s.keyStart[k] + mask_rank(mask + k * 8, a) < RR);
    slotN[s.keyStart[k] + mask_rank(mask + k * 8, a)] = (uint32_t)(hi - lo + 1);
  }
  __syncthreads();
  SLOT_MARK(pslot + 4);
  int np = 0;  // exclusive scan of the bin-ordered cell counts -> cell offsets
  for (int q = r0; q < r1; ++q) np += (int)slotN[q];
  int P;
  int off = block_scan_excl<T>(np, &P, wscr);
  for (int q = r0; q < r1; ++q) {
    const int n = (int)slotN[q];
    slotN[q] = (uint32_t)off;
    off += n;
  }
  A.P = P;
  HR_CHECK(RK == RR && P == E);
  __syncthreads();
  SLOT_MARK(pslot + 5);
  {
    // cells per bin -> chunks per bin -> chunk offsets (a scan over the bins)
    int nc = 0, cs = 0;
    if (tid < kLevels) {
      cs = kfirst < RK ? (int)slotN[kfirst] : P;
      const int kn = kfirst + kcount;  // the next bin's first run slot
      nc = ((kn < RK ? (int)slotN[kn] : P) - cs + kChunk - 1) / kChunk;
    }
    int PC;
    const int ps = block_scan_excl<T>(nc, &PC, wscr);
    HR_CHECK(PC <= Pmax);
    if (tid < kLevels) {
      s.pStart[tid] = ps;
      s.cBase[tid] = cs;
    }
    for (int i = tid; i < kChunk * PC; i += T) A.pDesc[i] = (uint32_t)(8 * kLevels) << 16;  // unused: hR1_0 * hL1[256]
    __syncthreads();
    for (int q = r0; q < r1; ++q) {  // the cells of each run at its bin-order position
      const uint32_t d = runDesc[q];
      const int a = d >> 24, lo = (d >> 8) & 255, hi = (d >> 16) & 255, k = d & 255;
      int p = kChunk * s.pStart[k] + (int)slotN[s.keyStart[k] + mask_rank(mask + k * 8, a)] - s.cBase[k];
      HR_CHECK(p >= 0 && p + hi - lo < kChunk * PC);
      for (int l = lo; l <= hi; ++l, ++p) A.pDesc[p] = (uint32_t)(8 * a) | ((uint32_t)(8 * l) << 16);
    }
    __syncthreads();
    if (tid < kLevels) s.keyStart[tid] = s.pStart[tid];  // run slots -> chunk offsets
    if (tid == 0) s.keyStart[kLevels] = PC;
    A.P = PC;
  }
  __syncthreads();
  {  // the bins holding chunks, ascending
    const bool has = tid < kLevels && s.keyStart[tid] < s.keyStart[tid + 1];
    int nb;
    const int pos = block_scan_excl<T>(has ? 1 : 0, &nb, wscr);
    if (has) s.binList[pos] = (uint8_t)tid;
    if (tid == 0) s.nBins = nb;
  }
  __syncthreads();
  SLOT_MARK(pslot + 6);
}

// One row's Eq. 20 run sums (keys kr[0..nL) non-decreasing): D[off + k - k0] = hra * (sum of
// hL over the row's cells of key k), in column order.  Branch-free: every cell stores the
// running sum of its run (the run's last cell stores the complete sum), so lanes walking
// different rows do not diverge at their run boundaries; keys and hL are loaded 8 cells at a
// time (all in flight together).  Entries of keys the row skips are not written (zeroed before).
__device__ __forceinline__ void row_runs(const uint8_t* __restrict__ kr, int nL, const double* __restrict__ hL,
                                         double hra, double* __restrict__ D, int off) {
  const int k0 = kr[0], klast = kr[nL - 1];
  double acc = 0.0;
  int kprev = k0;
  D += off - k0;
  for (int c0 = 0; c0 < nL; c0 += 8) {
    int kk[8];
    double hv[8], g[8];
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      const bool in = c0 + m < nL;
      kk[m] = in ? (int)kr[c0 + m] : klast;  // a slot past the row's end continues the last run with + 0
      hv[m] = in ? hL[c0 + m] : 0.0;
    }
    // The issue is in order, so the batch has no branch and one dependent operation per cell:
    // acc = acc * g + h with g = 0 where a run starts, else 1 (both exact), the flags computed
    // from neighbouring keys ahead of the chain; the multiplies and stores follow independently.
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      HR_CHECK(kk[m] >= (m ? kk[m - 1] : kprev));
      g[m] = kk[m] != (m ? kk[m - 1] : kprev) ? 0.0 : 1.0;
    }
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      acc = fma(acc, g[m], hv[m]);
      D[kk[m]] = hra * acc;
    }
    kprev = kk[7];
  }
}

// sum over bin k of its chunk sums (contiguous, bin order; the cluster solver's E2)
// (eight accumulators, eight loads in flight per step)
__device__ __forceinline__ double bin_sum(const Sm& s, const RunArena& A, int k) {
  double e[8];
#pragma unroll
  for (int m = 0; m < 8; ++m) e[m] = 0.0;
  int j = s.keyStart[k];
  const int j1 = s.keyStart[k + 1];
  const double* __restrict__ pv = A.pVal;
  for (; j + 7 < j1; j += 8) {
    double x[8];
#pragma unroll
    for (int m = 0; m < 8; ++m) x[m] = pv[j + m];
#pragma unroll
    for (int m = 0; m < 8; ++m) e[m] += x[m];
  }
#pragma unroll
  for (int m = 0; m < 7; ++m)
    if (j + m < j1) e[m] += pv[j + m];
  return ((e[0] + e[1]) + (e[2] + e[3])) + ((e[4] + e[5]) + (e[6] + e[7]));
}

// fast fp64 reciprocal: MUFU.RCP64H seed and two Newton steps (within ~1 ulp)
__device__ __forceinline__ double rcp_fast(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// Eq. 10 objective with K frozen at the current state (s.hR, s.hL, rho of this
// update): F = sum_cells (X_a Y_c / N - K_ac hS_k)^2 + alpha sum (Y - hS)^2 + beta sum (X - hG)^2,
// K_ac hS_k = hR_a hL_c hS_k / EstRaw_k (Eq. 11); X, Y the evaluated reflectance / illumination.
// Cells off the supports contribute 0.  Diagnostics only (hr_solve_trace): one more pass over the
// cells and one block reduction per value; every thread returns the total.
template <int T>
__device__ double objective(Sm& s, const hr_params& P, int nR, int nL, double N, const uint8_t* kc,
                            const double* X, const double* Y) {
  const int tid = threadIdx.x;
  double acc = 0.0;
  for (int e = tid; e < nR * nL; e += T) {
    const int a = e / nL, c = e - a * nL, k = kc[e];
    const double hsk = s.hSd[k];
    const double rho = P.update_form == 0 ? s.rho[k] : (s.rho[k] > 0.0 ? hsk * hsk / s.rho[k] : 0.0);
    const double r = X[a] * Y[c] / N - s.hR[a] * s.hL[c] * rho;
    acc = fma(r, r, acc);
  }
  if (tid < nL) {
    const double dl = Y[tid] - s.hSc[tid];
    acc += P.alpha * dl * dl;
  }
  if (tid < nR) {
    const double dr = X[tid] - s.hGc[tid];
    acc += P.beta * dr * dr;
  }
  slot_put3(s, R_OBJ, acc, -1, 0.0, -1, 0.0);
  __syncthreads();
  const double F = slot_sum<T>(s, R_OBJ);
  __syncthreads();
  return F;
}

// Algorithm 1 iterations over the chunk arena A (run_build with chunks: the cells in bin order,
// 8 per chunk).  Returns t; s.hR, s.hL then hold the renormalised final iterates (barrier done).
// The iterates stay RAW (s.hR1, s.hL1, the outputs of Eqs. 13 / 12); the factors of Eqs. 15, 14,
// cR = N / sum hR1 and cL = N / sum hL1, are applied as scalars where a renormalised value
// enters, so no phase waits for a renormalisation pass.
// Four phases per update, each closed by a barrier:
//   E1  one chunk per thread: the sum of its 8 cell products hR1_a hL1_c (Eqs. 6, 8)
//   E2  TPB lanes per occupied bin: EstRaw_k = cR cL sum of the bin's chunks; rho_k (Eq. 11 folded)
//   R   TPR threads per row: A_a over the row's cells (cached keys kc), Eq. 13
//   L   TPC threads per column: B_c over the rows, Eq. 12 with the frozen K
// Before the call: s.hR1 = s.hR = hG, s.hL1 = s.hL = hS (support entries), s.hL2 = hS^2, slot
// R_QL1 = per-warp partials of sum hS^2 (barrier done).
// kTrace: the Eq. 10 objective trace (hr_solve_trace) is compiled into a separate instance, so
// the product loop stays small.  kForm: P.update_form as a compile-time constant.
template <int T, bool kTrace, int kForm>
__device__ __forceinline__ int iterate(Sm& s, const hr_params& P, int nR, int nL, double N, const uint8_t* kc,
                                       const RunArena& A, double* trace = nullptr, int trace_cap = 0) {
  const int tid = threadIdx.x;
  // threads per row (R) / per column (L): the largest power of two with all rows / columns
  // covered by the T threads; each group sums its cells in a fixed order (deterministic)
  const int lgR = nR <= T / 8 ? 3 : nR <= T / 4 ? 2 : nR <= T / 2 ? 1 : 0, TPR = 1 << lgR;
  const int lgL = nL <= T / 8 ? 3 : nL <= T / 4 ? 2 : nL <= T / 2 ? 1 : 0, TPC = 1 << lgL;
  const int nBins = s.nBins;
  int lgB = 5;
  while (lgB > 0 && (nBins << lgB) > T) --lgB;
  const int TPB = 1 << lgB;
  constexpr int form = kForm;
  const double invN = 1.0 / N, invN2 = invN * invN;
  // this thread's share of the E2 phase: lane qb of the TPB lanes of bin kb (fixed for all t)
  const int jb = tid >> lgB, qb = tid & (TPB - 1);
  int kb = 0, pbeg = 0, pend = 0;
  if (jb < nBins) {
    kb = s.binList[jb];
    pbeg = s.keyStart[kb] + qb;
    pend = s.keyStart[kb + 1];
  }
  const double hSk = s.hSd[kb];
  const bool diffs = P.use_epsilon || kTrace;  // the renormalised iterates are needed every update
  double SR1 = N, SL1 = N;  // sums of the raw iterates (initially exactly N)
  double QL1 = slot_sum<T>(s, R_QL1);
  int t = 0;
#ifdef HR_SOLVE_PROFILE
  long long pacc[16] = {0}, pt0 = clock64(), pt1;
#define PHASE(i) do { pt1 = clock64(); pacc[i] += pt1 - pt0; pt0 = pt1; } while (0)
#else
#define PHASE(i) do { } while (0)
#endif
  for (;;) {
    if (t > 0 && !P.use_epsilon && t >= P.max_iter) break;
    // Eqs. 15, 14 as scalars: hR = cR hR1, hL = cL hL1
    const double cR = N * rcp_fast(SR1), cL = N * rcp_fast(SL1);
    // ======== E1: one chunk per thread: 8 cell products (Eqs. 6, 8) in flight, a fixed tree ========
    {
      const uint4* __restrict__ cd = reinterpret_cast<const uint4*>(A.pDesc);
      double* __restrict__ pv = A.pVal;
      const unsigned char* __restrict__ hrb = reinterpret_cast<const unsigned char*>(s.hR1);
      const unsigned char* __restrict__ hlb = reinterpret_cast<const unsigned char*>(s.hL1);
      for (int p = tid; p < A.P; p += T) {
        const uint4 q0 = cd[2 * p], q1 = cd[2 * p + 1];
        const uint32_t d[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
        double x[8];
#pragma unroll
        for (int m = 0; m < 8; ++m)
          x[m] = *reinterpret_cast<const double*>(hrb + (d[m] & 0xFFFFu)) *
                 *reinterpret_cast<const double*>(hlb + (d[m] >> 16));
#pragma unroll
        for (int w = 1; w < 8; w <<= 1)
#pragma unroll
          for (int m = 0; m + w < 8; m += 2 * w) x[m] += x[m + w];
        pv[p] = x[0];
      }
      PHASE(8);
      if (diffs && t > 0) {  // stop rule (R11): the renormalised iterates of update t against t-1
        double dr = 0.0, dl = 0.0;
        if (tid < nR) {
          const double n = cR * s.hR1[tid];
          dr = (n - s.hR[tid]) * (n - s.hR[tid]);
          s.hR[tid] = n;
        }
        if (tid < nL) {
          const double n = cL * s.hL1[tid];
          dl = (n - s.hL[tid]) * (n - s.hL[tid]);
          s.hL[tid] = n;
        }
        if (P.use_epsilon) slot_put3(s, R_DR, dr, R_DL, dl, -1, 0.0);
      }
    }
    PHASE(9);
    __syncthreads();
    PHASE(0);
    if (P.use_epsilon && t > 0) {
      const double eps = P.epsilon * N * N;
      if ((slot_sum<T>(s, R_DR) <= eps && slot_sum<T>(s, R_DL) <= eps) || t >= P.max_iter) break;
    }
    // ======== E2: EstRaw_k = cR cL (sum of the bin's cell products, bin order); rho_k (Eq. 11) ========
    // TPB lanes per occupied bin (the largest power of two <= 32 with every bin covered), each
    // summing every TPB-th product, then a fixed shuffle tree over the TPB lanes
    {
      const double* __restrict__ pv = A.pVal;
      double e0 = 0.0, e1 = 0.0, e2 = 0.0, e3 = 0.0;
      int i = pbeg;
      for (; i + 3 * TPB < pend; i += 4 * TPB) {
        e0 += pv[i];
        e1 += pv[i + TPB];
        e2 += pv[i + 2 * TPB];
        e3 += pv[i + 3 * TPB];
      }
      if (i < pend) e0 += pv[i];
      if (i + TPB < pend) e1 += pv[i + TPB];
      if (i + 2 * TPB < pend) e2 += pv[i + 2 * TPB];
      double e = (e0 + e1) + (e2 + e3);
      for (int d = 1; d < TPB; d <<= 1) e += __shfl_xor_sync(0xffffffffu, e, d);
      PHASE(15);
      if (jb < nBins && qb == 0) {
        const double er = e * (cR * cL);  // EstRaw_k of the renormalised iterates
        s.rho[kb] = form == 0 ? (er > 0.0 ? hSk * rcp_fast(er) : 0.0) : hSk * er;
      }
    }
    PHASE(10);
    __syncthreads();
    PHASE(1);
    if (kTrace) {  // before Eq. 13
      const double F = objective<T>(s, P, nR, nL, N, kc, s.hR, s.hL);
      if (tid == 0 && 3 * t < trace_cap) trace[3 * t] = F;
    }
    // ======== R: Eq. 13, TPR threads per row walking every TPR-th cell, fixed-order reduce ========
    const double cL2 = cL * cL;
    {
      const double invDenR = rcp_fast(cL2 * QL1 * invN2 + P.beta);
      double A0 = 0.0, A1 = 0.0;
      const int a = tid >> lgR, p = tid & (TPR - 1);
      if (a < nR) {
        const uint8_t* __restrict__ kr = kc + a * nL;
        const double* __restrict__ q2 = s.hL2;
        const double* __restrict__ rho = s.rho;
        int c = p;
        if (form == 0) {  // four cells per step: keys, then rho and hL1^2, all in flight
          double A2 = 0.0, A3 = 0.0;
          for (; c + 3 * TPR < nL; c += 4 * TPR) {
            const int k0 = kr[c], k1 = kr[c + TPR], k2 = kr[c + 2 * TPR], k3 = kr[c + 3 * TPR];
            A0 = fma(q2[c], rho[k0], A0);
            A1 = fma(q2[c + TPR], rho[k1], A1);
            A2 = fma(q2[c + 2 * TPR], rho[k2], A2);
            A3 = fma(q2[c + 3 * TPR], rho[k3], A3);
          }
          if (c < nL) A0 = fma(q2[c], rho[kr[c]], A0);
          if (c + TPR < nL) A1 = fma(q2[c + TPR], rho[kr[c + TPR]], A1);
          if (c + 2 * TPR < nL) A2 = fma(q2[c + 2 * TPR], rho[kr[c + 2 * TPR]], A2);
          A0 += A2;
          A1 += A3;
        } else {
          for (; c + TPR < nL; c += 2 * TPR) {
            A0 += rho[kr[c]];
            A1 += rho[kr[c + TPR]];
          }
          if (c < nL) A0 += rho[kr[c]];
        }
      }
      PHASE(4);
      double Av = A0 + A1;
      for (int d = TPR >> 1; d >= 1; d >>= 1) Av += __shfl_xor_sync(0xffffffffu, Av, d);
      double v = 0.0;
      if (a < nR && p == 0) {
        const double hr = cR * s.hR1[a];  // renormalised hR_a of update t
        const double num = form == 0 ? hr * (cL2 * Av) * invN : Av * rcp_fast(N * hr);
        v = (num + P.beta * s.hGc[a]) * invDenR;
        v = v > 0.0 ? v : 0.0;
        s.hR1[a] = v;
        s.wgt[a] = form == 0 ? v * hr : v * rcp_fast(hr);
      }
      PHASE(5);
      slot_put3(s, R_SR1, v, R_SR2, v * v, -1, 0.0, TPR);
    }
    PHASE(6);
    __syncthreads();
    PHASE(2);
    if (kTrace) {  // after Eq. 13 (raw hR', current hL)
      const double F = objective<T>(s, P, nR, nL, N, kc, s.hR1, s.hL);
      if (tid == 0 && 3 * t + 1 < trace_cap) trace[3 * t + 1] = F;
    }
    // ======== L: Eq. 12 (frozen K), TPC threads per column over every TPC-th row ========
    {
      const double invDenL = rcp_fast(slot_sum<T>(s, R_SR2) * invN2 + P.alpha);
      double B0 = 0.0, B1 = 0.0;
      const int c = tid >> lgL, p = tid & (TPC - 1);
      if (c < nL) {
        const uint8_t* __restrict__ kq = kc + c;
        const double* __restrict__ wg = s.wgt;
        const double* __restrict__ rho = s.rho;
        int a = p;
        double B2 = 0.0, B3 = 0.0;
        for (; a + 3 * TPC < nR; a += 4 * TPC) {  // four cells per step, keys first
          const int k0 = kq[a * nL], k1 = kq[(a + TPC) * nL], k2 = kq[(a + 2 * TPC) * nL], k3 = kq[(a + 3 * TPC) * nL];
          B0 = fma(wg[a], rho[k0], B0);
          B1 = fma(wg[a + TPC], rho[k1], B1);
          B2 = fma(wg[a + 2 * TPC], rho[k2], B2);
          B3 = fma(wg[a + 3 * TPC], rho[k3], B3);
        }
        if (a < nR) B0 = fma(wg[a], rho[kq[a * nL]], B0);
        if (a + TPC < nR) B1 = fma(wg[a + TPC], rho[kq[(a + TPC) * nL]], B1);
        if (a + 2 * TPC < nR) B2 = fma(wg[a + 2 * TPC], rho[kq[(a + 2 * TPC) * nL]], B2);
        B0 += B2;
        B1 += B3;
      }
      PHASE(11);
      double Bv = B0 + B1;
      for (int d = TPC >> 1; d >= 1; d >>= 1) Bv += __shfl_xor_sync(0xffffffffu, Bv, d);
      double u = 0.0;
      if (c < nL && p == 0) {
        const double hl = cL * s.hL1[c];  // renormalised hL_c of update t
        const double num = form == 0 ? hl * Bv * invN : Bv * rcp_fast(N * hl);
        u = (num + P.alpha * s.hSc[c]) * invDenL;
        u = u > 0.0 ? u : 0.0;
        s.hL1[c] = u;
        s.hL2[c] = u * u;
      }
      PHASE(12);
      slot_put3(s, R_SL1, u, R_QL1, u * u, -1, 0.0, TPC);
    }
    PHASE(13);
    SR1 = slot_sum<T>(s, R_SR1);
    __syncthreads();
    PHASE(3);
    if (kTrace) {  // after Eq. 12 (raw hR', raw hL')
      const double F = objective<T>(s, P, nR, nL, N, kc, s.hR1, s.hL1);
      if (tid == 0 && 3 * t + 2 < trace_cap) trace[3 * t + 2] = F;
    }
    ++t;
    SL1 = slot_sum<T>(s, R_SL1);
    QL1 = slot_sum<T>(s, R_QL1);
  }
  {  // the renormalised final iterates (Eqs. 15, 14)
    const double cR = N * rcp_fast(SR1), cL = N * rcp_fast(SL1);
    if (tid < nR) s.hR[tid] = cR * s.hR1[tid];
    if (tid < nL) s.hL[tid] = cL * s.hL1[tid];
  }
  __syncthreads();
#ifdef HR_SOLVE_PROFILE
  if (blockIdx.x == kProfBlock && threadIdx.x == 0)
    for (int i = 0; i < 16; ++i) g_solve_clk[512 + i] = pacc[i];
#endif
#undef PHASE
  return t;
}

// One image of Algorithm 1 + Eq. 20 + the CDF/LUT tail, by all T threads of the CTA.
// smraw: solve_smem_bytes() of shared memory; wscr: NW ints of shared scratch.  Every exit is
// CTA-uniform.  Histograms are read through L2 (__ldcg): in the grouped step they were
// accumulated by other grids' atomics while this grid was already running.
template <int T>
__device__ __forceinline__ void solve_image(const SolveArgs& args, const int64_t b, unsigned char* smraw, int* wscr) {
#ifdef HR_SOLVE_PROFILE
  int prof_n = 0;
#endif
  PROF_MARK();
  Sm& s = *reinterpret_cast<Sm*>(smraw);
  unsigned char* arenaS = smraw + sizeof(Sm);
  // shared arena: [ keys (E bytes) | run arena (when it fits) | ... | mask 8 KB ]
  const int AB = args.arena_bytes > 0 ? args.arena_bytes : kArenaSmem;
  uint32_t* mask = reinterpret_cast<uint32_t*>(arenaS + AB - kMaskBytes);
  const int tid = threadIdx.x;
  const hr_params& P = args.p;

  // ---- histograms (Alg. 1 init) ----
  constexpr int NW = T / 32;
  const bool binT = tid < kLevels;  // thread tid <-> bin tid
  if (binT) s.hSi[tid] = __ldcg(args.hist_s + b * kLevels + tid);
  if (args.hist_g) {
    if (binT) s.hGi[tid] = __ldcg(args.hist_g + b * kLevels + tid);
  } else {
    remap_gradient<T>(args.graw + b * kGradSlots, args.grad_norm, s.hGi, wscr);
  }
  if (binT) {
    s.bk[tid] = (double)tid / 255.0;
    s.hSd[tid] = (double)s.hSi[tid];
    if (args.hist_g_out) args.hist_g_out[b * kLevels + tid] = s.hGi[tid];
  }
  __syncthreads();
  PROF_MARK();

  // ---- supports (fixed for all t) ----
  const bool fL = binT && s.hSi[tid] != 0u, fR = binT && s.hGi[tid] != 0u;
  int nL, nR;
  const int pL = block_scan_excl<T>(fL ? 1 : 0, &nL, wscr);
  const int pR = block_scan_excl<T>(fR ? 1 : 0, &nR, wscr);
  if (fL) s.listL[pL] = (uint8_t)tid;
  if (fR) s.listR[pR] = (uint8_t)tid;
  {
    unsigned long long v = binT ? s.hSi[tid] : 0ull;
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
    if (binT) {
      if (args.hL) args.hL[b * kLevels + tid] = 0.0;
      if (args.hR) args.hR[b * kLevels + tid] = 0.0;
      if (args.target) args.target[b * kLevels + tid] = 0.0;
      if (args.lut) args.lut[b * kLevels + tid] = (uint8_t)tid;
    }
    if (tid == 0) {
      if (args.iters) args.iters[b] = 0;
      if (args.status) args.status[b] = HR_EDEGENERATE;
    }
    return;
  }

  // ---- initial state: hR^0 = hG, hL^0 = hS (R9), as raw iterates whose sums are N ----
  double q0 = 0.0;
  if (tid < nL) {
    const double v = s.hSd[s.listL[tid]];
    s.hL1[tid] = v;
    s.hSc[tid] = v;
    s.hL[tid] = v;
    s.hL2[tid] = v * v;
    q0 = v * v;
  }
  if (tid == 0) s.hL1[kLevels] = 0.0;         // the factor of unused chunk slots
  slot_put3(s, R_QL1, q0, -1, 0.0, -1, 0.0);  // sum hS^2: the first Eq. 13's denominator
  if (tid < nR) {
    const double v = (double)s.hGi[s.listR[tid]];
    s.hR1[tid] = v;
    s.hGc[tid] = v;
    s.hR[tid] = v;
  }

  // ---- runs of index(i,j) along each compacted row (fixed for all t) ----
  // keys kc (u8 per cell) at the shared arena start, or at the end of the global arena when
  // E does not fit (only with a reduced shared arena: the default holds E = 65536)
  const int E = nR * nL;
  unsigned char* arenaG = args.cells_ws + b * (int64_t)kArenaGlobal;
  const bool keysS = E <= AB - kMaskBytes;
  uint8_t* kc = keysS ? arenaS : arenaG + (kArenaGlobal - kKeysGlobal);
  {
    CellCursor<T> cur(tid, nL);
    for (int e = tid; e < E; e += T, cur.step()) kc[e] = (uint8_t)idx0(s.listR[cur.a], s.listL[cur.c]);
  }
  __syncthreads();
  RunArena A;
  run_build<T>(s, nR, nL, kc, mask, arenaS, AB, keysS, arenaG, A, wscr);  // bin-ordered cell chunks
  PROF_MARK();
  // the index_1 rows of the support rows (Eqs. 17-19 table) for Eq. 20: copied asynchronously
  // into the (now dead) bin-mask region while the iterations run (nR <= 32: 8 KB)
  const bool tabS = nR * kLevels <= kMaskBytes;
  if (tabS) {
    const uint32_t dst = (uint32_t)__cvta_generic_to_shared(mask);
    for (int i = tid; i < nR * (kLevels / 16); i += T) {
      const int a = i >> 4, j = i & 15;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + a * kLevels + j * 16),
                   "l"(args.idx1_tab + (size_t)s.listR[a] * kLevels + j * 16)
                   : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }

  double* tr = args.trace ? args.trace + b * (int64_t)args.trace_stride : nullptr;
  const int t = tr ? (P.update_form == 0 ? iterate<T, true, 0>(s, P, nR, nL, N, kc, A, tr, args.trace_stride)
                                         : iterate<T, true, 1>(s, P, nR, nL, N, kc, A, tr, args.trace_stride))
              : P.update_form == 0 ? iterate<T, false, 0>(s, P, nR, nL, N, kc, A, nullptr, 0)
                                   : iterate<T, false, 1>(s, P, nR, nL, N, kc, A, nullptr, 0);
  if (tr && tid == 0)
    for (int i = 3 * t; i < args.trace_stride; ++i) tr[i] = 0.0;
  PROF_MARK();

  // ---- outputs hL, hR (dense, zero off support) ----
  if (args.hL && binT) args.hL[b * kLevels + tid] = fL ? s.hL[pL] : 0.0;
  if (args.hR && binT) args.hR[b * kLevels + tid] = fR ? s.hR[pR] : 0.0;
  if (args.iters && tid == 0) args.iters[b] = t;

  // ---- Eq. 20: runs of index_1 (Eqs. 17-19) along each row, summed per bin in row order ----
  // index_1 of every cell from the per-gamma table (built once per gamma by k_idx1_table)
  uint8_t* kc1 = kc;
  SLOT_MARK(10);
  if (tabS) {
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    const uint8_t* tab = reinterpret_cast<const uint8_t*>(mask);
    CellCursor<T> cur(tid, nL);
    for (int e = tid; e < E; e += T, cur.step()) kc1[e] = tab[cur.a * kLevels + s.listL[cur.c]];
  } else {
    CellCursor<T> cur(tid, nL);
    for (int e = tid; e < E; e += T, cur.step())
      kc1[e] = __ldg(args.idx1_tab + s.listR[cur.a] * kLevels + s.listL[cur.c]);
  }
  // index_1 is non-decreasing along a row (b_i p_j increases with j), so row a's keys cover the
  // range [kmin_a, kmax_a]; D holds, per row, hR_a * (sum of hL over the cells of key k) for k in
  // that range (zero where no cell has key k), rows at offsets rowOff[a] (a block scan of the
  // widths).  Then T_k = (1/N) sum over the rows, in row order, of D[a][k]: deterministic, and no
  // second chunk structure to build (that build cost more than the sums themselves).
  __syncthreads();
  SLOT_MARK(11);
  const int wr = tid < nR ? (int)kc1[tid * nL + nL - 1] - (int)kc1[tid * nL] + 1 : 0;
  int Wtot;
  const int offr = block_scan_excl<T>(wr, &Wtot, wscr);
  // per row: kmin | kmax << 8 | offset << 16 (offset < Wtot <= 65536), padded to a multiple of 4
  // rows with empty ranges (kmin > kmax)
  uint32_t* rowPack = reinterpret_cast<uint32_t*>(s.pStart);
  if (tid < ((nR + 3) & ~3))
    rowPack[tid] = tid < nR ? (uint32_t)kc1[tid * nL] | ((uint32_t)kc1[tid * nL + nL - 1] << 8) | ((uint32_t)offr << 16)
                            : 1u;
  const bool dS = keysS && align16(E) + 8 * Wtot <= AB - kMaskBytes;
  double* D = dS ? reinterpret_cast<double*>(arenaS + align16(E)) : reinterpret_cast<double*>(arenaG);
  HR_CHECK(dS || 8 * Wtot <= kArenaRun);
  for (int i = tid; i < Wtot; i += T) D[i] = 0.0;
  __syncthreads();
  SLOT_MARK(12);
  if (tid < nR) row_runs(kc1 + tid * nL, nL, s.hL, s.hR[tid], D, offr);  // row a = tid
  __syncthreads();
  SLOT_MARK(13);
  double* Tt = s.rho;  // dense target
  if (binT) {  // rows in order; four rows' ranges (one 16-B load) and entries in flight per step
    double e0 = 0.0;
    const uint4* __restrict__ rp = reinterpret_cast<const uint4*>(rowPack);
    for (int a = 0; a < nR; a += 4) {
      const uint4 q = rp[a >> 2];
      const uint32_t r[4] = {q.x, q.y, q.z, q.w};
      double v[4];
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const int lo = r[m] & 255, hi = (r[m] >> 8) & 255;
        v[m] = (tid >= lo && tid <= hi) ? D[(int)(r[m] >> 16) + tid - lo] : 0.0;
      }
#pragma unroll
      for (int m = 0; m < 4; ++m) e0 += v[m];  // + 0 for the rows without this key
    }
    Tt[tid] = e0 / N;
  }
  __syncthreads();
  SLOT_MARK(14);
  if (args.target && binT) args.target[b * kLevels + tid] = Tt[tid];
  __syncthreads();
  PROF_MARK();
  SLOT_MARK(15);
  if (args.lut || args.status)
    cdf_lut<T>(s.hSi, Tt, s.hL1, s.wgt, s.hL2, wscr, args.lut ? args.lut + b * kLevels : nullptr,
            args.status ? args.status + b : nullptr);
  SLOT_MARK(16);
}


}  // namespace
}  // namespace hr
