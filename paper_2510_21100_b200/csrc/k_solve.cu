// k_solve.cu -- kernel (b): batched histogram-domain Retinex solver (Algorithm 1) in fp64,
// with the Eq. 17-20 reprocessing and the fused CDF + histogram-matching LUT tail (c).
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
// Supports never change (hR stays 0 off supp(hG), hL off supp(hS)), so every pass runs over
// the E = nR x nL compacted cells only.
//
// Each of the three passes (E: cells grouped by output bin k; R: row-major, key = row;
// L: column-major, key = column) is a segmented sum whose segment boundaries are known in
// advance.  Thread t sums the fixed slice [t*S, t*S+S) of the pass's cell order: segments
// wholly inside its slice are finalised by the thread itself; a segment spanning several
// slices leaves a partial in pf[t] (its part at the slice start) / pl[t] (at the slice end),
// and after one barrier the segment's owner adds those partials in slice order.  Two
// barriers per pass, no floating-point atomics, a fixed summation order: bit-identical run
// to run.
#include "hr_common.cuh"

namespace hr {
namespace {

constexpr int T = kSolveThreads;
constexpr int NW = kSolveWarps;
constexpr int kMaxCells = kLevels * kLevels;
constexpr int kSmemCells = 32768;  // cell list capacity in shared memory (64 KB)

// slots of the block-reduction scratch
enum { R_SL2 = 0, R_SR1, R_SR2, R_SL1, R_DR, R_DL, kSlots };

struct __align__(16) Sm {
  double hR[kLevels], hL[kLevels];    // compacted state (index a over sR, c over sL)
  double hR1[kLevels], hL1[kLevels];  // raw updates (Eq. 13 / Eq. 12 outputs)
  double hSc[kLevels], hGc[kLevels];  // priors at the support entries
  double hL2[kLevels];                // hL_c^2
  double wgt[kLevels];                // per-row weight of the L-pass
  double hSd[kLevels];                // dense hS as double
  double est[kLevels];                // EstRaw_k (= N Est_k)
  double rho[kLevels];                // rho_k (GC) or sigma_k (paper-literal)
  double bk[kLevels];                 // b_k = k/255 (R1)
  double pf[T], pl[T];                // slice-boundary partials
  double red[kSlots][NW];
  uint32_t hSi[kLevels], hGi[kLevels];
  uint32_t rcp[kLevels];              // ceil(2^32 / i)
  int cstart[kLevels + 1];
  uint16_t posL[kLevels + 1];
  uint8_t listR[kLevels], listL[kLevels];
  int nR, nL, E;
  unsigned long long Nint;
  unsigned long long nw[NW];
};

__device__ __forceinline__ int idx0(int i, int j) {  // P:192 index(i,j) for l = 256
  return (int)(((uint32_t)(i * j + 127) * 32897u) >> 23);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
  return v;
}

// Sum over warps in fixed order (call after a barrier that follows the slot writes).
__device__ __forceinline__ double slot_sum(const Sm& s, int slot) {
  double a = 0.0;
#pragma unroll
  for (int w = 0; w < NW; ++w) a += s.red[slot][w];
  return a;
}

__device__ __forceinline__ void slot_put(Sm& s, int slot, double v) {
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) s.red[slot][threadIdx.x >> 5] = v;
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

// c-range [lo, hi] of the compacted columns whose index(i, j) == k (idx monotone in j).
// Divisions by i use the exact reciprocal magic floor(x / i) = umulhi(x, ceil(2^32 / i))
// (x <= 65152, i <= 255: error x (ceil - 2^32/i) / 2^32 < 1/i).
__device__ __forceinline__ int div_i(const Sm& s, uint32_t x, int i) {
  return i == 1 ? (int)x : (int)__umulhi(x, s.rcp[i]);
}
__device__ __forceinline__ void crange(const Sm& s, int i, int k, int& lo, int& hi) {
  if (i == 0) {  // index(0, j) = 0 for all j
    lo = 0;
    hi = (k == 0) ? s.nL - 1 : -1;
    return;
  }
  // (i*j + 127) div 255 == k  <=>  255k - 127 <= i*j <= 255k + 127
  const int a = 255 * k - 127, bnd = 255 * k + 127;
  const int jlo = a <= 0 ? 0 : div_i(s, (uint32_t)(a + i - 1), i);
  int jhi = div_i(s, (uint32_t)bnd, i);
  if (jhi > 255) jhi = 255;
  if (jlo > jhi) {
    lo = 0;
    hi = -1;
    return;
  }
  lo = s.posL[jlo];
  hi = (int)s.posL[jhi + 1] - 1;
}

// index_1(i,j) of Eqs. 17-19: first k minimising |b_i p_j - b_k|, p_j = b_j^(1/gamma).
__device__ __forceinline__ int idx1(const Sm& s, double bi, double pj) {
  const double x = __dmul_rn(bi, pj);  // rounded product (no contraction into the compare)
  int k0 = (int)floor(x * 255.0);
  int best = -1;
  double bd = 0.0;
#pragma unroll
  for (int d = -1; d <= 1; ++d) {
    const int k = k0 + d;
    if (k < 0 || k > 255) continue;
    const double dist = fabs(x - s.bk[k]);
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
  const uint32_t c0 = graw[tid], c1 = graw[tid + T];
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

// Sum of the partials of a segment [ks, ke) that spans slices t1 < t2 (slice size S).
__device__ __forceinline__ double span_sum(const Sm& s, int ks, int ke, int S) {
  const int t1 = ks / S, t2 = (ke - 1) / S;
  double acc = s.pl[t1];
  for (int t = t1 + 1; t < t2; ++t) acc += s.pf[t];
  return acc + s.pf[t2];
}

__device__ __forceinline__ bool spans(int ks, int ke, int S) { return ks / S != (ke - 1) / S; }

__global__ void __launch_bounds__(T, 2) k_solve(SolveArgs args) {
  extern __shared__ __align__(16) unsigned char smraw[];
  Sm& s = *reinterpret_cast<Sm*>(smraw);
  uint16_t* cells = reinterpret_cast<uint16_t*>(smraw + sizeof(Sm));
  __shared__ int wscr[NW];
  const int tid = threadIdx.x;
  const int64_t b = blockIdx.x;
  const hr_params& P = args.p;

  // ---- histograms (Alg. 1 init) ----
  s.hSi[tid] = args.hist_s[b * kLevels + tid];
  if (args.hist_g) {
    s.hGi[tid] = args.hist_g[b * kLevels + tid];
  } else {
    remap_gradient(args.graw + b * kGradSlots, args.grad_norm, s.hGi, wscr);
  }
  s.bk[tid] = (double)tid / 255.0;
  s.hSd[tid] = (double)s.hSi[tid];
  s.rcp[tid] = tid <= 1 ? 0u : (uint32_t)((0x100000000ull + (uint64_t)tid - 1) / (uint64_t)tid);
  s.est[tid] = 0.0;
  __syncthreads();

  // ---- supports (fixed for all t) ----
  const bool fL = s.hSi[tid] != 0u, fR = s.hGi[tid] != 0u;
  int nL, nR;
  const int pL = block_scan_excl(fL ? 1 : 0, &nL, wscr);
  const int pR = block_scan_excl(fR ? 1 : 0, &nR, wscr);
  if (fL) s.listL[pL] = (uint8_t)tid;
  if (fR) s.listR[pR] = (uint8_t)tid;
  s.posL[tid] = (uint16_t)pL;
  {
    unsigned long long v = s.hSi[tid];
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    if ((tid & 31) == 0) s.nw[tid >> 5] = v;
  }
  if (tid == 0) {
    s.posL[kLevels] = (uint16_t)nL;
    s.nL = nL;
    s.nR = nR;
  }
  __syncthreads();
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

  // ---- compacted state: hR^0 = hG, hL^0 = hS (R9) ----
  double l2 = 0.0;
  if (tid < nL) {
    const double v = s.hSd[s.listL[tid]];
    s.hL[tid] = v;
    s.hSc[tid] = v;
    s.hL2[tid] = v * v;
    l2 = v * v;
  }
  if (tid < nR) {
    const double v = (double)s.hGi[s.listR[tid]];
    s.hR[tid] = v;
    s.hGc[tid] = v;
  }
  slot_put(s, R_SL2, l2);

  // ---- cells grouped by output bin k = index(i,j): one thread per k ----
  const int E = nR * nL;  // every cell of sR x sL has exactly one k
  uint16_t* cl = (E <= kSmemCells || args.cells_ws == nullptr) ? cells : args.cells_ws + b * kMaxCells;
  {
    const int k = tid;
    int cnt = 0;
    for (int a = 0; a < nR; ++a) {
      int lo, hi;
      crange(s, s.listR[a], k, lo, hi);
      if (hi >= lo) cnt += hi - lo + 1;
    }
    int Etot;
    const int start = block_scan_excl(cnt, &Etot, wscr);
    s.cstart[k] = start;
    if (tid == 0) s.cstart[kLevels] = Etot;
    int pos = start;
    for (int a = 0; a < nR && pos < start + cnt; ++a) {
      int lo, hi;
      crange(s, s.listR[a], k, lo, hi);
      for (int c = lo; c <= hi; ++c) cl[pos++] = (uint16_t)((a << 8) | c);
    }
  }
  __syncthreads();

  const double N2 = N * N;
  const int form = P.update_form;
  const int S = (E + T - 1) / T;            // slice length, identical for the three passes
  const int e0 = min(E, tid * S), e1 = min(E, e0 + S);
  const bool has = e0 < e1;
  int kstart = 0;                           // bin of cell e0 in the k-grouped order
  if (has) {
    int lo = 0, hi = kLevels + 1;           // upper_bound(cstart, e0) - 1
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (s.cstart[mid] <= e0) lo = mid + 1; else hi = mid;
    }
    kstart = lo - 1;
  }
  const int astart = has ? e0 / nL : 0;     // row of cell e0 (row-major)
  const int cstart0 = has ? e0 / nR : 0;    // column of cell e0 (column-major)

  double SL2 = slot_sum(s, R_SL2);
  int t = 0;
  for (;;) {
    // ======== E-pass: EstRaw_k = sum_{idx=k} hR_a hL_c  (Eqs. 6, 8 with N folded) ========
    if (has) {
      int k = kstart;
      for (;;) {
        const int ks = s.cstart[k], ke = s.cstart[k + 1];
        const int lo = max(ks, e0), hi = min(ke, e1);
        double acc = 0.0;
        for (int e = lo; e < hi; ++e) {
          const uint32_t x = cl[e];
          acc += s.hR[x >> 8] * s.hL[x & 255u];
        }
        if (ks >= e0 && ke <= e1) {
          s.est[k] = acc;
          s.rho[k] = form == 0 ? (acc > 0.0 ? s.hSd[k] / acc : 0.0) : s.hSd[k] * acc;
        } else {
          if (ks < e0) s.pf[tid] = acc;
          if (ke > e1) s.pl[tid] = acc;
        }
        if (ke >= e1) break;
        do { ++k; } while (s.cstart[k + 1] == s.cstart[k]);
      }
    }
    __syncthreads();
    {
      const int k = tid, ks = s.cstart[k], ke = s.cstart[k + 1];
      if (ks < ke && spans(ks, ke, S)) {
        const double e = span_sum(s, ks, ke, S);
        s.est[k] = e;
        s.rho[k] = form == 0 ? (e > 0.0 ? s.hSd[k] / e : 0.0) : s.hSd[k] * e;
      }
    }
    __syncthreads();

    // ======== R-pass (Eq. 13): A_a over row-major cells ========
    double sr1 = 0.0, sr2 = 0.0;
    const double denR = SL2 / N2 + P.beta;
    auto finR = [&](int a, double A) {
      const double hr = s.hR[a];
      const double num = form == 0 ? hr * A / N : A / (N * hr);
      double v = (num + P.beta * s.hGc[a]) / denR;
      v = v > 0.0 ? v : 0.0;
      s.hR1[a] = v;
      s.wgt[a] = form == 0 ? v * hr : v / hr;
      sr1 += v;
      sr2 += v * v;
    };
    if (has) {
      int a = astart;
      for (;;) {
        const int as = a * nL, ae = as + nL;
        const int lo = max(as, e0), hi = min(ae, e1);
        const int ia = s.listR[a];
        double acc = 0.0;
        for (int e = lo; e < hi; ++e) {
          const int c = e - as;
          const double r = s.rho[idx0(ia, s.listL[c])];
          acc += form == 0 ? s.hL2[c] * r : r;
        }
        if (as >= e0 && ae <= e1) {
          finR(a, acc);
        } else {
          if (as < e0) s.pf[tid] = acc;
          if (ae > e1) s.pl[tid] = acc;
        }
        if (ae >= e1) break;
        ++a;
      }
    }
    __syncthreads();
    if (tid < nR) {
      const int as = tid * nL, ae = as + nL;
      if (spans(as, ae, S)) finR(tid, span_sum(s, as, ae, S));
    }
    slot_put(s, R_SR1, sr1);
    slot_put(s, R_SR2, sr2);
    __syncthreads();

    // ======== L-pass (Eq. 12, frozen K): B_c over column-major cells ========
    const double SR2 = slot_sum(s, R_SR2);
    const double denL = SR2 / N2 + P.alpha;
    double sl1 = 0.0;
    auto finL = [&](int c, double Bv) {
      const double hl = s.hL[c];
      const double num = form == 0 ? hl * Bv / N : Bv / (N * hl);
      double u = (num + P.alpha * s.hSc[c]) / denL;
      u = u > 0.0 ? u : 0.0;
      s.hL1[c] = u;
      sl1 += u;
    };
    if (has) {
      int c = cstart0;
      for (;;) {
        const int cs = c * nR, ce = cs + nR;
        const int lo = max(cs, e0), hi = min(ce, e1);
        const int jc = s.listL[c];
        double acc = 0.0;
        for (int e = lo; e < hi; ++e) {
          const int a = e - cs;
          acc += s.wgt[a] * s.rho[idx0(s.listR[a], jc)];
        }
        if (cs >= e0 && ce <= e1) {
          finL(c, acc);
        } else {
          if (cs < e0) s.pf[tid] = acc;
          if (ce > e1) s.pl[tid] = acc;
        }
        if (ce >= e1) break;
        ++c;
      }
    }
    __syncthreads();
    if (tid < nL) {
      const int cs = tid * nR, ce = cs + nR;
      if (spans(cs, ce, S)) finL(tid, span_sum(s, cs, ce, S));
    }
    slot_put(s, R_SL1, sl1);
    __syncthreads();

    // ======== Eqs. 15, 14: renormalise; stop test (R11); Eq. 11 refresh is implicit ========
    {
      const double SR1 = slot_sum(s, R_SR1), SL1 = slot_sum(s, R_SL1);
      double dr = 0.0, dl = 0.0, q = 0.0;
      if (tid < nR) {
        const double n = N * s.hR1[tid] / SR1;
        dr = (n - s.hR[tid]) * (n - s.hR[tid]);
        s.hR[tid] = n;
      }
      if (tid < nL) {
        const double n = N * s.hL1[tid] / SL1;
        dl = (n - s.hL[tid]) * (n - s.hL[tid]);
        s.hL[tid] = n;
        s.hL2[tid] = n * n;
        q = n * n;
      }
      slot_put(s, R_DR, dr);
      slot_put(s, R_DL, dl);
      slot_put(s, R_SL2, q);
    }
    __syncthreads();
    ++t;
    SL2 = slot_sum(s, R_SL2);
    const double eps = P.epsilon * N2;
    const bool conv = P.use_epsilon && slot_sum(s, R_DR) <= eps && slot_sum(s, R_DL) <= eps;
    if (conv || t >= P.max_iter) break;
  }

  // ---- outputs hL, hR (dense, zero off support) ----
  if (args.hL) args.hL[b * kLevels + tid] = fL ? s.hL[pL] : 0.0;
  if (args.hR) args.hR[b * kLevels + tid] = fR ? s.hR[pR] : 0.0;
  if (args.iters && tid == 0) args.iters[b] = t;

  // ---- Eq. 20 with index_1 (Eqs. 17-19): warp per row, segmented by k, warp-private sums ----
  double* pj = s.hR1;                                   // p_j = b_j^(1/gamma)   (Eq. 17)
  double* Twarp = reinterpret_cast<double*>(cells);     // 8 x 256 doubles = 16 KB (cells dead)
  {
    const double bj = s.bk[tid];
    pj[tid] = (P.gamma == 1.0) ? bj : pow(bj, 1.0 / P.gamma);
    for (int w = 0; w < NW; ++w) Twarp[w * kLevels + tid] = 0.0;
  }
  __syncthreads();
  {
    const int lane = tid & 31, w = tid >> 5;
    for (int a = w; a < nR; a += NW) {
      const double bi = s.bk[s.listR[a]];
      const double vr = s.hR[a];
      for (int c0 = 0; c0 < nL; c0 += 32) {
        const int c = c0 + lane;
        const bool valid = c < nL;
        const int k = valid ? idx1(s, bi, pj[s.listL[c]]) : 256 + lane;  // keys non-decreasing
        double v = valid ? vr * s.hL[c] : 0.0;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const double vu = __shfl_up_sync(0xffffffffu, v, d);
          const int ku = __shfl_up_sync(0xffffffffu, k, d);
          if (lane >= d && ku == k) v += vu;
        }
        const int kn = __shfl_down_sync(0xffffffffu, k, 1);
        if (valid && (lane == 31 || kn != k)) Twarp[w * kLevels + k] += v;
      }
    }
  }
  __syncthreads();
  double* Tt = s.est;  // dense target
  {
    double acc = 0.0;
    for (int w = 0; w < NW; ++w) acc += Twarp[w * kLevels + tid];
    Tt[tid] = acc / N;
    if (args.target) args.target[b * kLevels + tid] = Tt[tid];
  }
  __syncthreads();
  if (args.lut || args.status)
    cdf_lut(s.hSi, Tt, s.hL1, s.rho, s.wgt, wscr, args.lut ? args.lut + b * kLevels : nullptr,
            args.status ? args.status + b : nullptr);
}

__global__ void __launch_bounds__(T) k_remap(const uint32_t* graw, int32_t grad_norm, uint32_t* hist_g) {
  __shared__ uint32_t h[kLevels];
  __shared__ int wscr[NW];
  const int64_t b = blockIdx.x;
  remap_gradient(graw + b * kGradSlots, grad_norm, h, wscr);
  hist_g[b * kLevels + threadIdx.x] = h[threadIdx.x];
}

__global__ void __launch_bounds__(T) k_match(const uint32_t* hist_s, const double* target, uint8_t* lut,
                                             int32_t* status) {
  __shared__ uint32_t hSi[kLevels];
  __shared__ double Tt[kLevels], Pt[kLevels], Ct[kLevels], Cs[kLevels];
  __shared__ int wscr[NW];
  const int64_t b = blockIdx.x;
  hSi[threadIdx.x] = hist_s[b * kLevels + threadIdx.x];
  Tt[threadIdx.x] = target[b * kLevels + threadIdx.x];
  __syncthreads();
  cdf_lut(hSi, Tt, Pt, Ct, Cs, wscr, lut + b * kLevels, status ? status + b : nullptr);
}

}  // namespace

size_t solve_smem_bytes() { return sizeof(Sm) + (size_t)kSmemCells * sizeof(uint16_t); }
size_t solve_cells_ws_bytes(int64_t B) { return (size_t)B * kMaxCells * sizeof(uint16_t); }

cudaError_t launch_solve(const SolveArgs& a, int64_t B, cudaStream_t st) {
  static bool attr = false;
  const size_t smem = solve_smem_bytes();
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  k_solve<<<(unsigned)B, T, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_remap(const uint32_t* hist_graw, int64_t B, int32_t grad_norm, uint32_t* hist_g,
                         cudaStream_t st) {
  k_remap<<<(unsigned)B, T, 0, st>>>(hist_graw, grad_norm, hist_g);
  return cudaGetLastError();
}

cudaError_t launch_match(const uint32_t* hist_s, const double* target, int64_t B, uint8_t* lut,
                         int32_t* status, cudaStream_t st) {
  k_match<<<(unsigned)B, T, 0, st>>>(hist_s, target, lut, status);
  return cudaGetLastError();
}

}  // namespace hr
