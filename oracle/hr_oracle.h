/*
 * hr_oracle.h -- plain, slow, fp64 CPU oracle for the HistRetinex hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_2510_21100_b200/) never links, imports or calls it,
 * and this file shares no code, header, table or constant with the CUDA path.
 *
 * Every function follows /root/reference/PAPER.md ("P:<line>") literally, in
 * the paper's order and notation; where the paper is silent or garbled the
 * reading R<n> of DESIGN.md section 3 (== SURVEY.md section 8(c)) is named.
 * Arithmetic: fp64, every sum left to right in index order, compiled with
 * -O2 -ffp-contract=off (no FMA contraction, no fast-math).
 *
 * Conventions: l = number of levels (general l >= 2 unless stated), bins are
 * indexed 0..l-1 (R6), b_k = k/(l-1) (R1).  Matrices are row-major l x l with
 * row index i = reflectance level, column index j = illumination level (R4).
 * Return codes: 0 ok, 1 invalid argument, 2 empty input, 3 degenerate.
 */
#ifndef HR_ORACLE_H
#define HR_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Parameters of Algorithm 1 + reprocessing (readings R7,R11-R14). */
typedef struct {
  int32_t levels;      /* l >= 2 */
  double alpha, beta;  /* > 0, Eq. 10 prior weights */
  double gamma;        /* >= 1, Eq. 17 */
  double epsilon;      /* stop threshold, RELATIVE: ||dh||^2 <= epsilon * N^2 (R11) */
  int32_t max_iter;    /* T >= 1 */
  int32_t use_epsilon; /* 0: exactly T iterations; 1: Alg. 1 stop rule (R11) */
  int32_t update_form; /* 0 gradient-consistent (R7 default), 1 paper-literal (printed Eqs. 12-13) */
  int32_t grad_norm;   /* 0 MAXNORM, 1 RAW_CLAMP (R14) */
} ho_params;

/* O1: value channel S of HSV, quantised to l levels:
   S = round_half_up(max(R,G,B) * (l-1) / 255); for l = 256 this is max(R,G,B). */
int ho_value_channel(const uint8_t* rgb, int64_t npix, int32_t levels, int32_t* S);

/* O2: gradient image (reading R14).  Forward differences,
   dx = S(y,x+1)-S(y,x) (0 in the last column), dy = S(y+1,x)-S(y,x) (0 in the
   last row), raw magnitude g = |dx|+|dy| in [0, 2(l-1)]. */
int ho_gradient_raw(const int32_t* S, int32_t H, int32_t W, int32_t* g);

/* O2: quantise the raw gradient image to l levels (R14):
   grad_norm 0 (MAXNORM): g' = round_half_up((l-1) * g / gmax), gmax = max g (0 -> all 0)
   grad_norm 1 (RAW_CLAMP): g' = min(g, l-1). */
int ho_gradient_levels(const int32_t* g, int64_t n, int32_t levels, int32_t grad_norm, int32_t* gq);

/* Eq. 3: count histogram h[k] = #{p : x[p] == k}, k in [0, nbins). */
int ho_count_histogram(const int32_t* x, int64_t n, int32_t nbins, uint64_t* h);

/* O3 (R1): location vector b[k] = k/(l-1). */
int ho_locations(int32_t levels, double* b);

/* O4/O5: index map (P:192 below Eq. 10; Eqs. 17-19).
   idx[i][j] = first k minimising |b_i * pow(b_j, 1/gamma) - b_k| (R5: smallest k on ties).
   gamma == 1 gives index(i,j) of Eq. 10 (pow is skipped, so b_j is used exactly). */
int ho_index_map(int32_t levels, double gamma, int32_t* idx);

/* Eq. 6: count matrix C[i][j] = hR[i] * hL[j] / N. */
int ho_pair_count(const double* hR, const double* hL, int32_t levels, double N, double* C);

/* Eq. 8 (reading R3): estimate est[k] = sum over (i,j), idx[i][j]==k, of C[i][j]. */
int ho_estimate(const double* C, const int32_t* idx, int32_t levels, double* est);

/* Eq. 11: K[i][j] = C[i][j] / est[idx[i][j]]; 0 when est == 0 (R8). */
int ho_weights(const double* C, const int32_t* idx, const double* est, int32_t levels, double* K);

/* Eq. 10 (R6): J = sum_ij (hR_i hL_j / N - K_ij hS_idx(i,j))^2
   + alpha sum_j (hL_j - hS_j)^2 + beta sum_i (hR_i - hG_i)^2. */
double ho_objective(const double* hR, const double* hL, const double* hS, const double* hG,
                    const double* K, const int32_t* idx, int32_t levels, double N,
                    double alpha, double beta);

/* Eq. 13: reflectance update with K frozen.  form 0 (R7, the stationary
   point of Eq. 10 in hR_i):
     hR'_i = (sum_j hL_j K_ij hS_idx / N + beta hG_i) / (sum_j hL_j^2 / N^2 + beta)
   form 1 (as printed): the K_ij factor is a divisor, /(N K_ij), over cells with K_ij != 0.
   Output clamped at >= 0. */
int ho_update_reflectance(const double* hL, const double* hS, const double* hG, const double* K,
                          const int32_t* idx, int32_t levels, double N, double beta,
                          int32_t form, double* hR_out);

/* Eq. 12: illumination update with K frozen, mirror of Eq. 13
   (hR is the just-updated, not yet renormalised reflectance; reading R10). */
int ho_update_illumination(const double* hR, const double* hS, const double* K,
                           const int32_t* idx, int32_t levels, double N, double alpha,
                           int32_t form, double* hL_out);

/* Eqs. 14-15: out[k] = N * h[k] / sum h.  Returns 3 if sum h <= 0. */
int ho_renormalize(const double* h, int32_t levels, double N, double* out);

/* Algorithm 1.  hS, hG: count histograms (as doubles) with sum N.
   Outputs hL, hR (final renormalised iterates), iteration count, and optionally the
   objective trace: 3 values per iteration (before Eq. 13, after Eq. 13, after Eq. 12),
   K frozen, written up to trace_cap entries. */
int ho_decompose(const double* hS, const double* hG, const ho_params* p,
                 double* hL, double* hR, int32_t* iters, double* trace, int32_t trace_cap);

/* Eq. 20: T[k] = sum over (i,j) with idx1[i][j]==k of hR_i hL_j / N. */
int ho_enhanced_histogram(const double* hR, const double* hL, const int32_t* idx1,
                          int32_t levels, double N, double* T);

/* Histogram matching (reading R16).  Cs(v) = Ps(v)/N with Ps the integer prefix of
   hS; Pt(k) = Pt(k-1) + T(k), Ct(k) = Pt(k)/Pt(l-1); lut[v] = first k minimising
   |Ct(k) - Cs(v)|.  margin[v] (nullable) = second-smallest distinct distance - smallest.
   Returns 3 if Pt(l-1) <= 0. */
int ho_match_lut(const uint64_t* hS, const double* T, int32_t levels, int32_t* lut, double* margin);

/* Eq. 5: HE transform t_i = round((l-1) * sum_{j<=i} hS_j / N). */
int ho_he_transform(const uint64_t* hS, int32_t levels, int32_t* t);

/* O11 (reading R17): replace V in exact hexcone HSV, round half up, per pixel.
   Vnew[p] is the new 8-bit value.  Exact rational arithmetic. */
int ho_reconstruct(const uint8_t* rgb, int64_t npix, const int32_t* Vnew, uint8_t* out);

/* Whole pipeline for one 8-bit RGB image, l must be 256.  Any output pointer may be NULL.
   hS, hG: [256] histograms; hgraw: [511]; hL, hR, T: [256]; lut: [256]. */
int ho_enhance(const uint8_t* rgb, int32_t H, int32_t W, const ho_params* p, uint8_t* out,
               uint64_t* hS, uint64_t* hG, uint64_t* hgraw, double* hL, double* hR, double* T,
               int32_t* lut, int32_t* iters, double* lut_margin);

/* Same for a batch [B][H][W][3], images processed by nthreads host threads (>= 1).
   Per-image outputs are laid out [B][...]. */
int ho_enhance_batch(const uint8_t* rgb, int64_t B, int32_t H, int32_t W, const ho_params* p,
                     uint8_t* out, uint64_t* hS, uint64_t* hG, double* hL, double* hR,
                     double* T, int32_t* lut, int32_t* iters, int32_t nthreads);

/* ---------------------------------------------------------------------------------------
   Second workload: the HE baseline and the quality metrics of §IV.
   Definitions are SPEC.md's metrics module, which fixes what PAPER.md leaves
   open (P:311 names PSNR [40], SSIM [41], LOE [15] without formulas).
   --------------------------------------------------------------------------------------- */

/* HE baseline (Eq. 5): V -> t_V with t from ho_he_transform, colour by R17. */
int ho_he_enhance(const uint8_t* rgb, int32_t H, int32_t W, uint8_t* out);

/* PSNR: 10 log10(255^2 / MSE), MSE over all three channels; identical -> +inf. */
double ho_psnr(const uint8_t* a, const uint8_t* b, int64_t npix);

/* SSIM: luma Y = 0.299 R + 0.587 G + 0.114 B; 11x11 Gaussian window, sigma 1.5,
   normalised; valid windows only ((H-10) x (W-10) centres); C1 = (0.01*255)^2,
   C2 = (0.03*255)^2; the mean of the SSIM map.  Needs H, W >= 11 (else NaN). */
double ho_ssim(const uint8_t* a, const uint8_t* b, int32_t H, int32_t W);

/* LOE: lightness L = max(R,G,B); both images sampled to mh x mw = min(H,100) x
   min(W,100) by nearest neighbour (row i <- (i*H)/mh, column j <- (j*W)/mw); LOE =
   (1/m) sum_x sum_y [(L(x) >= L(y)) xor (L'(x) >= L'(y))], m = mh * mw. */
double ho_loe(const uint8_t* orig, const uint8_t* enh, int32_t H, int32_t W);

#ifdef __cplusplus
}
#endif
#endif
