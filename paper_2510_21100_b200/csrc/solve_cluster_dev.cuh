// solve_cluster_dev.cuh -- kernel (b) for one LARGE image on a thread-block cluster (SURVEY
// §8(f) NEXT #3): the same Algorithm 1 (fp64, factored, support-compacted) as solve_dev.cuh,
// with the cells split over the CS CTAs of a cluster and the partial results exchanged through
// distributed shared memory (DSMEM).
//
// PAPER.md: Eqs. 6-15 and Algorithm 1, Eqs. 17-20, P:308 (matching);
// readings R1-R21 exactly as in solve_dev.cuh.
//
// Split (rank r of CS): rows a in [aB, aE) = [nR r / CS, nR (r+1) / CS) for the E and R passes
// (their keys index(i,j), runs and cell chunks are built from those rows only), columns c in
// [cB, cE) = [nL r / CS, nL (r+1) / CS) for the L pass (over all rows).  Every CTA keeps the
// FULL state vectors (hR, hL, raw hR', hL', L-pass row weights) in its own shared memory.
// One iteration:
//   E1  renormalise the full raw iterates (Eqs. 15, 14; identical arithmetic in every CTA),
//       chunk sums of the local cells
//   E2  per bin, the local rows' EstRaw partial  -> cluster barrier
//   E3  EstRaw_k = sum over ranks, in rank order, of the partials (DSMEM loads), rho_k
//   R   Eq. 13 for the local rows; hR'_a and the L weight stored into EVERY CTA (DSMEM
//       stores); the CTA's partial sums of hR' and hR'^2 likewise -> cluster barrier
//   L   Eq. 12 for the local columns (all rows, frozen K); hL'_c into every CTA, partial sums
//       -> cluster barrier
// Every cross-CTA sum runs in rank order and every per-CTA sum in a fixed order: the results
// are deterministic and identical in all CTAs (so the stop rule is decided alike everywhere).
// Eq. 20: each CTA sums its rows' cells per bin (dense per-row run sums, as solve_dev.cuh);
// rank 0 adds the CS partials in rank order and builds the LUT.
#pragma once
#include <cooperative_groups.h>

#include "solve_dev.cuh"

namespace hr {
namespace {

namespace cg = cooperative_groups;

constexpr int kMaxCS = 16;

struct __align__(16) SmClusterExtra {
  double est[kLevels];       // this CTA's EstRaw partial (E2), then its Eq. 20 partial (tail)
  double part[4][kMaxCS];    // per-rank partial sums: hR', hR'^2, hL', hL'^2
};

// phase clocks (measurement builds, -DHR_SOLVE_PROFILE): rank 0 of block 0, thread 0;
// g_solve_clk[700 + i]: 0 start, 1 supports, 2 keys, 3 runs, 4 iterations, 5 Eq. 20 + LUT;
// [720 + j] per-phase sums over the iterations: E1, E2, E3, R, L (each to its closing barrier);
// 6-10: the tail's steps (tools/cluster_scan.py)
#ifdef HR_SOLVE_PROFILE
#define CMARK(i)                                                    \
  do {                                                              \
    if (blockIdx.x == 0 && threadIdx.x == 0) g_solve_clk[700 + (i)] = clock64(); \
  } while (0)
#define CPH_T0() long long cph_t0_ = clock64()
#define CPH(j)                                                                         \
  do {                                                                                 \
    if (blockIdx.x == 0 && threadIdx.x == 0) {                                         \
      const long long t1_ = clock64();                                                 \
      g_solve_clk[720 + (j)] += t1_ - cph_t0_;                                         \
      cph_t0_ = t1_;                                                                   \
    }                                                                                  \
  } while (0)
#else
#define CMARK(i) \
  do {           \
  } while (0)
#define CPH_T0() \
  do {           \
  } while (0)
#define CPH(j) \
  do {         \
  } while (0)
#endif

// cluster-wide barrier (release / acquire: the DSMEM stores before it are visible after it).
// Not the .aligned form: that one requires every warp to arrive converged, which the compiler
// does not guarantee after the data-dependent loops that precede some calls.
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire;\n" ::: "memory");
}

template <int T, int CS, int kForm>
__device__ int iterate_cluster(Sm& s, SmClusterExtra& x, cg::cluster_group& cl, int rank, const hr_params& P,
                               int nR, int nL, int aB, int nRl, int cB, int nLl, double N, const uint8_t* kcR,
                               const uint8_t* kcL, const RunArena& A) {
  const int tid = threadIdx.x;
  // threads per local row (R) / per local column (L), as solve_dev.cuh
  const int lgR = nRl <= T / 8 ? 3 : nRl <= T / 4 ? 2 : nRl <= T / 2 ? 1 : 0, TPR = 1 << lgR;
  const int lgL = nLl <= T / 8 ? 3 : nLl <= T / 4 ? 2 : nLl <= T / 2 ? 1 : 0, TPC = 1 << lgL;
  const double invN = 1.0 / N, invN2 = invN * invN;
  double SR1 = N, SL1 = N, QL1 = 0.0;
  // remote (DSMEM) views of the arrays every CTA writes into every other CTA
  double* rR1[CS];
  double* rW[CS];
  double* rL1[CS];
  double* rPart[CS];
#pragma unroll
  for (int q = 0; q < CS; ++q) {
    rR1[q] = cl.map_shared_rank(s.hR1, q);
    rW[q] = cl.map_shared_rank(s.wgt, q);
    rL1[q] = cl.map_shared_rank(s.hL1, q);
    rPart[q] = cl.map_shared_rank(&x.part[0][0], q);
  }
  int t = 0;
#ifdef HR_SOLVE_PROFILE
  if (blockIdx.x == 0 && threadIdx.x == 0)
    for (int j = 0; j < 5; ++j) g_solve_clk[720 + j] = 0;
#endif
  CPH_T0();
  for (;;) {
    // ======== E1: renormalise (Eqs. 15, 14), local chunk sums (Eqs. 6, 8) ========
    const double cL = SL1 == N ? 1.0 : N * rcp_fast(SL1);
    const double cR = SR1 == N ? 1.0 : N * rcp_fast(SR1), cRL = cR * cL;
    {
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
      // one chunk of 8 bin-ordered local cells per thread (run_build with chunks)
      const uint4* __restrict__ cd = reinterpret_cast<const uint4*>(A.pDesc);
      double* __restrict__ pv = A.pVal;
      const unsigned char* __restrict__ hrb = reinterpret_cast<const unsigned char*>(s.hR1 + aB);
      const unsigned char* __restrict__ hlb = reinterpret_cast<const unsigned char*>(s.hL1);
      for (int p = tid; p < A.P; p += T) {
        const uint4 q0 = cd[2 * p], q1 = cd[2 * p + 1];
        const uint32_t d[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
        double xv[8];
#pragma unroll
        for (int m = 0; m < 8; ++m) {
          HR_CHECK((int)(d[m] & 0xFFFFu) < 8 * (nRl > 0 ? nRl : 1) && (int)(d[m] >> 16) <= 8 * kLevels);
          xv[m] = *reinterpret_cast<const double*>(hrb + (d[m] & 0xFFFFu)) *
                  *reinterpret_cast<const double*>(hlb + (d[m] >> 16));
        }
#pragma unroll
        for (int w = 1; w < 8; w <<= 1)
#pragma unroll
          for (int m = 0; m + w < 8; m += 2 * w) xv[m] += xv[m + w];
        pv[p] = xv[0] * cRL;
      }
      if (t == 0 || P.use_epsilon) slot_put3(s, R_DR, dr, R_DL, dl, R_SL2, q);
    }
    __syncthreads();
    CPH(0);
    if (t > 0) {  // stop rule (R11): the same full vectors in every CTA, the same decision
      const double eps = P.epsilon * N * N;
      const bool conv = P.use_epsilon && slot_sum<T>(s, R_DR) <= eps && slot_sum<T>(s, R_DL) <= eps;
      if (conv || t >= P.max_iter) break;
    }
    // ======== E2: the local rows' EstRaw partial per bin ========
    if (tid < kLevels) x.est[tid] = s.keyStart[tid] < s.keyStart[tid + 1] ? bin_sum(s, A, tid) : 0.0;
    const double invDenR = rcp_fast((t == 0 ? slot_sum<T>(s, R_SL2) : cL * cL * QL1) * invN2 + P.beta);
    cluster_sync_all();
    CPH(1);
    // ======== E3: EstRaw_k over the ranks (rank order), rho_k (Eq. 11) ========
    if (tid < kLevels) {
      double e = 0.0;
#pragma unroll
      for (int q = 0; q < CS; ++q) e += cl.map_shared_rank(x.est, q)[tid];
      s.rho[tid] = kForm == 0 ? (e > 0.0 ? s.hSd[tid] * rcp_fast(e) : 0.0) : s.hSd[tid] * e;
    }
    __syncthreads();
    CPH(2);
    // ======== R: Eq. 13 for the local rows; hR' and the L weight into every CTA ========
    {
      double A0 = 0.0, A1 = 0.0;
      const int al = tid >> lgR, p = tid & (TPR - 1);
      if (al < nRl) {
        const uint8_t* kr = kcR + al * nL;
        int c = p;
        if (kForm == 0) {
          double A2 = 0.0, A3 = 0.0;
          for (; c + 3 * TPR < nL; c += 4 * TPR) {
            const int k0 = kr[c], k1 = kr[c + TPR], k2 = kr[c + 2 * TPR], k3 = kr[c + 3 * TPR];
            A0 = fma(s.hL2[c], s.rho[k0], A0);
            A1 = fma(s.hL2[c + TPR], s.rho[k1], A1);
            A2 = fma(s.hL2[c + 2 * TPR], s.rho[k2], A2);
            A3 = fma(s.hL2[c + 3 * TPR], s.rho[k3], A3);
          }
          if (c < nL) A0 = fma(s.hL2[c], s.rho[kr[c]], A0);
          if (c + TPR < nL) A1 = fma(s.hL2[c + TPR], s.rho[kr[c + TPR]], A1);
          if (c + 2 * TPR < nL) A2 = fma(s.hL2[c + 2 * TPR], s.rho[kr[c + 2 * TPR]], A2);
          A0 += A2;
          A1 += A3;
        } else {
          for (; c + TPR < nL; c += 2 * TPR) {
            A0 += s.rho[kr[c]];
            A1 += s.rho[kr[c + TPR]];
          }
          if (c < nL) A0 += s.rho[kr[c]];
        }
      }
      double Av = A0 + A1;
      for (int d = TPR >> 1; d >= 1; d >>= 1) Av += __shfl_xor_sync(0xffffffffu, Av, d);
      double v = 0.0;
      if (al < nRl && p == 0) {
        const int a = aB + al;
        const double hr = s.hR[a];
        const double num = kForm == 0 ? hr * Av * invN : Av * rcp_fast(N * hr);
        v = (num + P.beta * s.hGc[a]) * invDenR;
        v = v > 0.0 ? v : 0.0;
        const double w = kForm == 0 ? v * hr : v * rcp_fast(hr);
        HR_CHECK(a < nR);
#pragma unroll
        for (int q = 0; q < CS; ++q) {
          rR1[q][a] = v;
          rW[q][a] = w;
        }
      }
      slot_put3(s, R_SR1, v, R_SR2, v * v, -1, 0.0);
    }
    __syncthreads();
    if (tid < CS) {  // this CTA's partial sums, into rank `rank` of every CTA's table
      rPart[tid][0 * kMaxCS + rank] = slot_sum<T>(s, R_SR1);
      rPart[tid][1 * kMaxCS + rank] = slot_sum<T>(s, R_SR2);
    }
    cluster_sync_all();
    CPH(3);
    // ======== L: Eq. 12 (frozen K) for the local columns over all rows ========
    {
      double sr2 = 0.0;
#pragma unroll
      for (int q = 0; q < CS; ++q) sr2 += x.part[1][q];
      const double invDenL = rcp_fast(sr2 * invN2 + P.alpha);
      double B0 = 0.0, B1 = 0.0;
      const int cl_ = tid >> lgL, p = tid & (TPC - 1);
      if (cl_ < nLl) {
        const uint8_t* kq = kcL + cl_ * nR;
        int a = p;
        double B2 = 0.0, B3 = 0.0;
        for (; a + 3 * TPC < nR; a += 4 * TPC) {
          const int k0 = kq[a], k1 = kq[a + TPC], k2 = kq[a + 2 * TPC], k3 = kq[a + 3 * TPC];
          B0 = fma(s.wgt[a], s.rho[k0], B0);
          B1 = fma(s.wgt[a + TPC], s.rho[k1], B1);
          B2 = fma(s.wgt[a + 2 * TPC], s.rho[k2], B2);
          B3 = fma(s.wgt[a + 3 * TPC], s.rho[k3], B3);
        }
        if (a < nR) B0 = fma(s.wgt[a], s.rho[kq[a]], B0);
        if (a + TPC < nR) B1 = fma(s.wgt[a + TPC], s.rho[kq[a + TPC]], B1);
        if (a + 2 * TPC < nR) B2 = fma(s.wgt[a + 2 * TPC], s.rho[kq[a + 2 * TPC]], B2);
        B0 += B2;
        B1 += B3;
      }
      double Bv = B0 + B1;
      for (int d = TPC >> 1; d >= 1; d >>= 1) Bv += __shfl_xor_sync(0xffffffffu, Bv, d);
      double u = 0.0;
      if (cl_ < nLl && p == 0) {
        const int c = cB + cl_;
        const double hl = s.hL[c];
        const double num = kForm == 0 ? hl * Bv * invN : Bv * rcp_fast(N * hl);
        u = (num + P.alpha * s.hSc[c]) * invDenL;
        u = u > 0.0 ? u : 0.0;
        HR_CHECK(c < nL);
#pragma unroll
        for (int q = 0; q < CS; ++q) rL1[q][c] = u;
      }
      slot_put3(s, R_SL1, u, R_QL1, u * u, -1, 0.0);
    }
    __syncthreads();
    if (tid < CS) {
      rPart[tid][2 * kMaxCS + rank] = slot_sum<T>(s, R_SL1);
      rPart[tid][3 * kMaxCS + rank] = slot_sum<T>(s, R_QL1);
    }
    cluster_sync_all();
    CPH(4);
    ++t;
    SR1 = 0.0, SL1 = 0.0, QL1 = 0.0;
#pragma unroll
    for (int q = 0; q < CS; ++q) {
      SR1 += x.part[0][q];
      SL1 += x.part[2][q];
      QL1 += x.part[3][q];
    }
  }
  return t;
}

// One image on the CS CTAs of a cluster (rank = %cluster_ctarank).  smraw: sizeof(Sm) +
// sizeof(SmClusterExtra) + arena_bytes of shared memory.  Rank 0 writes every output.
template <int T, int CS>
__device__ __forceinline__ void solve_image_cluster(const SolveArgs& args, const int64_t b, unsigned char* smraw,
                                                    int* wscr) {
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  HR_CHECK((int)cl.num_blocks() == CS && rank == (int)(blockIdx.x % CS) && blockDim.x == T);
  Sm& s = *reinterpret_cast<Sm*>(smraw);
  SmClusterExtra& x = *reinterpret_cast<SmClusterExtra*>(smraw + sizeof(Sm));
  unsigned char* arenaS = smraw + sizeof(Sm) + sizeof(SmClusterExtra);
  const int AB = args.arena_bytes > 0 ? args.arena_bytes : kArenaSmem;
  const int tid = threadIdx.x;
  const hr_params& P = args.p;
  const bool out0 = rank == 0;
  CMARK(0);

  // ---- histograms, supports, N: computed alike in every CTA ----
  constexpr int NW = T / 32;
  const bool binT = tid < kLevels;
  if (binT) s.hSi[tid] = __ldcg(args.hist_s + b * kLevels + tid);
  if (args.hist_g) {
    if (binT) s.hGi[tid] = __ldcg(args.hist_g + b * kLevels + tid);
  } else {
    remap_gradient<T>(args.graw + b * kGradSlots, args.grad_norm, s.hGi, wscr);
  }
  if (binT) {
    s.bk[tid] = (double)tid / 255.0;
    s.hSd[tid] = (double)s.hSi[tid];
    if (out0 && args.hist_g_out) args.hist_g_out[b * kLevels + tid] = s.hGi[tid];
  }
  __syncthreads();
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
  unsigned long long Nint = 0;
  for (int u = 0; u < NW; ++u) Nint += s.nw[u];
  const double N = (double)Nint;
  if (Nint == 0 || nR == 0) {  // empty image (never for validated inputs): every CTA exits here
    if (out0 && binT) {
      if (args.hL) args.hL[b * kLevels + tid] = 0.0;
      if (args.hR) args.hR[b * kLevels + tid] = 0.0;
      if (args.target) args.target[b * kLevels + tid] = 0.0;
      if (args.lut) args.lut[b * kLevels + tid] = (uint8_t)tid;
    }
    if (out0 && tid == 0) {
      if (args.iters) args.iters[b] = 0;
      if (args.status) args.status[b] = HR_EDEGENERATE;
    }
    return;
  }
  if (tid < nL) {
    const double v = s.hSd[s.listL[tid]];
    s.hL1[tid] = v;
    s.hSc[tid] = v;
    s.hL[tid] = v;
  }
  if (tid == 0) s.hL1[kLevels] = 0.0;  // the factor of unused chunk slots
  if (tid < nR) {
    const double v = (double)s.hGi[s.listR[tid]];
    s.hR1[tid] = v;
    s.hGc[tid] = v;
    s.hR[tid] = v;
  }
  CMARK(1);
  const int aB = (int)((long long)nR * rank / CS), aE = (int)((long long)nR * (rank + 1) / CS), nRl = aE - aB;
  const int cB = (int)((long long)nL * rank / CS), cE = (int)((long long)nL * (rank + 1) / CS), nLl = cE - cB;

  // ---- keys: local rows (row-major, E and R passes), local columns (column-major, L pass);
  // arena: [ kcR | run arena | ... | kcL | mask 8 KB ] ----
  const int El = nRl * nL, EL = nLl * nR;
  const int kcLb = align16(EL);
  uint32_t* mask = reinterpret_cast<uint32_t*>(arenaS + AB - kMaskBytes);
  unsigned char* arenaG = args.cells_ws + (b * CS + rank) * (int64_t)kArenaGlobal;
  HR_CHECK(El <= AB - kMaskBytes - kcLb && kcLb + kMaskBytes <= AB);
  uint8_t* kcR = arenaS;
  uint8_t* kcL = arenaS + AB - kMaskBytes - kcLb;
  {
    CellCursor<T> cur(tid, nL);
    for (int e = tid; e < El; e += T, cur.step()) kcR[e] = (uint8_t)idx0(s.listR[aB + cur.a], s.listL[cur.c]);
    CellCursor<T> cuc(tid, nR);  // column-major copy: (local column, row)
    for (int e = tid; e < EL; e += T, cuc.step()) kcL[e] = (uint8_t)idx0(s.listR[cuc.c], s.listL[cB + cuc.a]);
  }
  __syncthreads();
  CMARK(2);
  RunArena A;
  if (nRl > 0) {
    run_build<T>(s, nRl, nL, kcR, mask, arenaS, AB - kcLb, true, arenaG, A, wscr);  // bin-ordered chunks
  } else {  // more ranks than rows: no local chunks
    A.P = 0;
    A.RR = 0;
    A.pDesc = nullptr;
    A.pVal = nullptr;
    if (tid <= kLevels) s.keyStart[tid] = 0;
    __syncthreads();
  }
  cluster_sync_all();  // every CTA's state is initialised before any remote store
  CMARK(3);
  // the index_1 rows of the local rows (Eq. 20) copied asynchronously into the dead bin-mask
  // region while the iterations run (as in solve_image)
  const bool tabS = nRl * kLevels <= kMaskBytes;
  if (tabS) {
    const uint32_t dst = (uint32_t)__cvta_generic_to_shared(mask);
    for (int i = tid; i < nRl * (kLevels / 16); i += T) {
      const int a = i >> 4, j = i & 15;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + a * kLevels + j * 16),
                   "l"(args.idx1_tab + (size_t)s.listR[aB + a] * kLevels + j * 16)
                   : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }

  const int t = P.update_form == 0 ? iterate_cluster<T, CS, 0>(s, x, cl, rank, P, nR, nL, aB, nRl, cB, nLl, N, kcR, kcL, A)
                                   : iterate_cluster<T, CS, 1>(s, x, cl, rank, P, nR, nL, aB, nRl, cB, nLl, N, kcR, kcL, A);

  CMARK(4);
  if (out0) {
    if (args.hL && binT) args.hL[b * kLevels + tid] = fL ? s.hL[pL] : 0.0;
    if (args.hR && binT) args.hR[b * kLevels + tid] = fR ? s.hR[pR] : 0.0;
    if (args.iters && tid == 0) args.iters[b] = t;
  }

  // ---- Eq. 20 on the local rows: dense per-row run sums (solve_dev.cuh), summed per bin ----
  uint8_t* kc1 = kcR;
  if (tabS) {
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    const uint8_t* tab = reinterpret_cast<const uint8_t*>(mask);
    CellCursor<T> cur(tid, nL);
    for (int e = tid; e < El; e += T, cur.step()) kc1[e] = tab[cur.a * kLevels + s.listL[cur.c]];
  } else {
    CellCursor<T> cur(tid, nL);
    for (int e = tid; e < El; e += T, cur.step())
      kc1[e] = __ldg(args.idx1_tab + s.listR[aB + cur.a] * kLevels + s.listL[cur.c]);
  }
  __syncthreads();
  CMARK(6);
  const int wr = tid < nRl ? (int)kc1[tid * nL + nL - 1] - (int)kc1[tid * nL] + 1 : 0;
  int Wtot;
  const int offr = block_scan_excl<T>(wr, &Wtot, wscr);
  // per local row: kmin | kmax << 8 | offset << 16, padded to a multiple of 4 rows with empty ranges
  uint32_t* rowPack = reinterpret_cast<uint32_t*>(s.pStart);
  if (tid < ((nRl + 3) & ~3))
    rowPack[tid] = tid < nRl ? (uint32_t)kc1[tid * nL] | ((uint32_t)kc1[tid * nL + nL - 1] << 8) | ((uint32_t)offr << 16)
                             : 1u;
  const bool dS = align16(El) + 8 * Wtot <= AB - kMaskBytes - kcLb;
  HR_CHECK(dS || 8LL * Wtot <= kArenaGlobal);
  double* D = dS ? reinterpret_cast<double*>(arenaS + align16(El)) : reinterpret_cast<double*>(arenaG);
  for (int i = tid; i < Wtot; i += T) D[i] = 0.0;
  __syncthreads();
  if (tid < nRl) row_runs(kc1 + tid * nL, nL, s.hL, s.hR[aB + tid], D, offr);  // local row tid
  __syncthreads();
  CMARK(7);
  if (binT) {  // local rows in order; four rows' ranges (one 16-B load) and entries in flight per step
    double e0 = 0.0;
    const uint4* __restrict__ rp = reinterpret_cast<const uint4*>(rowPack);
    for (int a = 0; a < nRl; a += 4) {
      const uint4 q = rp[a >> 2];
      const uint32_t r[4] = {q.x, q.y, q.z, q.w};
      double v[4];
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const int lo = r[m] & 255, hi = (r[m] >> 8) & 255;
        v[m] = (tid >= lo && tid <= hi) ? D[(int)(r[m] >> 16) + tid - lo] : 0.0;
      }
#pragma unroll
      for (int m = 0; m < 4; ++m) e0 += v[m];
    }
    x.est[tid] = e0;
  }
  cluster_sync_all();
  CMARK(8);
  if (out0) {
    double* Tt = s.rho;
    if (binT) {
      double e = 0.0;
#pragma unroll
      for (int q = 0; q < CS; ++q) e += cl.map_shared_rank(x.est, q)[tid];
      Tt[tid] = e / N;
    }
    __syncthreads();
    CMARK(9);
    if (args.target && binT) args.target[b * kLevels + tid] = Tt[tid];
    if (args.lut || args.status)
      cdf_lut<T>(s.hSi, Tt, s.hL1, s.wgt, s.hL2, wscr, args.lut ? args.lut + b * kLevels : nullptr,
                 args.status ? args.status + b : nullptr);
  }
  CMARK(10);
  cluster_sync_all();  // rank 0's DSMEM reads are done before any CTA exits
  CMARK(5);
}

}  // namespace
}  // namespace hr
