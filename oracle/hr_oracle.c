/*
 * hr_oracle.c -- plain, slow, fp64 CPU oracle for the HistRetinex hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see hr_oracle.h).  Literal transcription of
 * PAPER.md Eqs. 3-20 and Algorithm 1 in the paper's order; no blocking, no
 * factoring, no reordering.  Every sum runs left to right in index order.
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -fPIC -shared -pthread.
 *
 * parity pins: see tests/test_oracle_*.py (each function is pinned against a
 * brute force, closed form, invariant or textbook special case; DESIGN.md s.3).
 */
#include "hr_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define HO_OK 0
#define HO_EINVAL 1
#define HO_EEMPTY 2
#define HO_EDEGENERATE 3

/* ------------------------------------------------------------------ pixels */

/* O1, "S is the value channel of the test image I in the HSV":
   v = max(R,G,B)/255, level = round(v*(l-1)) (round half away from zero). */
int ho_value_channel(const uint8_t* rgb, int64_t npix, int32_t levels, int32_t* S) {
  if (!rgb || !S || levels < 2) return HO_EINVAL;
  if (npix <= 0) return HO_EEMPTY;
  for (int64_t p = 0; p < npix; ++p) {
    int r = rgb[3 * p + 0], g = rgb[3 * p + 1], b = rgb[3 * p + 2];
    int mx = r;
    if (g > mx) mx = g;
    if (b > mx) mx = b;
    double v = (double)mx / 255.0;
    S[p] = (int32_t)floor(v * (double)(levels - 1) + 0.5);
  }
  return HO_OK;
}

/* O2, P:73 / P:246 (reading R14): forward differences, L1 magnitude. */
int ho_gradient_raw(const int32_t* S, int32_t H, int32_t W, int32_t* g) {
  if (!S || !g || H < 0 || W < 0) return HO_EINVAL;
  if ((int64_t)H * W == 0) return HO_EEMPTY;
  for (int32_t y = 0; y < H; ++y) {
    for (int32_t x = 0; x < W; ++x) {
      int64_t p = (int64_t)y * W + x;
      int32_t dx = (x + 1 < W) ? S[p + 1] - S[p] : 0;
      int32_t dy = (y + 1 < H) ? S[p + W] - S[p] : 0;
      g[p] = abs(dx) + abs(dy);
    }
  }
  return HO_OK;
}

/* O2, reading R14: MAXNORM normalises the gradient image by its maximum to [0,1]
   and quantises to l levels, round half up; RAW_CLAMP clamps to l-1. */
int ho_gradient_levels(const int32_t* g, int64_t n, int32_t levels, int32_t grad_norm, int32_t* gq) {
  if (!g || !gq || levels < 2 || (grad_norm != 0 && grad_norm != 1)) return HO_EINVAL;
  if (n <= 0) return HO_EEMPTY;
  if (grad_norm == 1) {
    for (int64_t p = 0; p < n; ++p) gq[p] = g[p] < levels - 1 ? g[p] : levels - 1;
    return HO_OK;
  }
  int32_t gmax = 0;
  for (int64_t p = 0; p < n; ++p)
    if (g[p] > gmax) gmax = g[p];
  for (int64_t p = 0; p < n; ++p) {
    if (gmax == 0) {
      gq[p] = 0;
    } else {
      /* (l-1)*g is an exact integer; the quotient is correctly rounded, so an exact
         .5 tie stays exact and rounds up (round half up). */
      double q = ((double)(levels - 1) * (double)g[p]) / (double)gmax;
      gq[p] = (int32_t)floor(q + 0.5);
    }
  }
  return HO_OK;
}

/* Eq. 3: H_C(S)_i = n_i. */
int ho_count_histogram(const int32_t* x, int64_t n, int32_t nbins, uint64_t* h) {
  if (!x || !h || nbins < 1) return HO_EINVAL;
  for (int32_t k = 0; k < nbins; ++k) h[k] = 0;
  if (n <= 0) return HO_EEMPTY;
  for (int64_t p = 0; p < n; ++p) {
    if (x[p] < 0 || x[p] >= nbins) return HO_EINVAL;
    h[x[p]] += 1;
  }
  return HO_OK;
}

/* ------------------------------------------------------ histogram domain */

/* R1 (P:159 names H_B without values): b_k = k/(l-1). */
int ho_locations(int32_t levels, double* b) {
  if (!b || levels < 2) return HO_EINVAL;
  for (int32_t k = 0; k < levels; ++k) b[k] = (double)k / (double)(levels - 1);
  return HO_OK;
}

/* P:192 index(i,j) = argmin_k |H_B(L,R)_ij - H_B(S)_k| with H_B(L,R)_ij = b_i b_j
   (Eq. 7 without the printed /N, R2); Eqs. 17-19: index_1 uses b_j^(1/gamma) for the
   illumination factor (R4).  Ties -> smallest k (R5). */
int ho_index_map(int32_t levels, double gamma, int32_t* idx) {
  if (!idx || levels < 2 || !(gamma >= 1.0)) return HO_EINVAL;
  double* b = (double*)malloc(sizeof(double) * (size_t)levels);
  double* p = (double*)malloc(sizeof(double) * (size_t)levels);
  if (!b || !p) {
    free(b);
    free(p);
    return HO_EINVAL;
  }
  ho_locations(levels, b);
  for (int32_t j = 0; j < levels; ++j) p[j] = (gamma == 1.0) ? b[j] : pow(b[j], 1.0 / gamma); /* Eq. 17 */
  for (int32_t i = 0; i < levels; ++i) {
    for (int32_t j = 0; j < levels; ++j) {
      double loc = b[i] * p[j]; /* Eq. 7 / Eq. 18 cell */
      int32_t best = 0;
      double bestd = fabs(loc - b[0]);
      for (int32_t k = 1; k < levels; ++k) {
        double d = fabs(loc - b[k]);
        if (d < bestd) {
          bestd = d;
          best = k;
        }
      }
      idx[(int64_t)i * levels + j] = best;
    }
  }
  free(b);
  free(p);
  return HO_OK;
}

/* Eq. 6: H_C(L,R) = H_C(L) x H_C(R)^T / N, stored [i=R][j=L] (R4). */
int ho_pair_count(const double* hR, const double* hL, int32_t levels, double N, double* C) {
  if (!hR || !hL || !C || levels < 2 || !(N > 0)) return HO_EINVAL;
  for (int32_t i = 0; i < levels; ++i)
    for (int32_t j = 0; j < levels; ++j) C[(int64_t)i * levels + j] = hR[i] * hL[j] / N;
  return HO_OK;
}

/* Eq. 8, P:161-168 (R3: without the printed extra /N): sum of the count-matrix cells
   classified to bin k. */
int ho_estimate(const double* C, const int32_t* idx, int32_t levels, double* est) {
  if (!C || !idx || !est || levels < 2) return HO_EINVAL;
  for (int32_t k = 0; k < levels; ++k) est[k] = 0.0;
  for (int32_t i = 0; i < levels; ++i)
    for (int32_t j = 0; j < levels; ++j) {
      int64_t c = (int64_t)i * levels + j;
      est[idx[c]] += C[c];
    }
  return HO_OK;
}

/* Eq. 11: K_ij = H_C(L,R)_ij / sum_{k in dN_index(i,j)} H_C(L,R)_k; 0 if that is 0 (R8). */
int ho_weights(const double* C, const int32_t* idx, const double* est, int32_t levels, double* K) {
  if (!C || !idx || !est || !K || levels < 2) return HO_EINVAL;
  for (int64_t c = 0; c < (int64_t)levels * levels; ++c) {
    double d = est[idx[c]];
    K[c] = (d > 0.0) ? C[c] / d : 0.0;
  }
  return HO_OK;
}

/* Eq. 10, sums over 0..l-1 (R6). */
double ho_objective(const double* hR, const double* hL, const double* hS, const double* hG,
                    const double* K, const int32_t* idx, int32_t levels, double N,
                    double alpha, double beta) {
  double fid = 0.0;
  for (int32_t i = 0; i < levels; ++i)
    for (int32_t j = 0; j < levels; ++j) {
      int64_t c = (int64_t)i * levels + j;
      double r = hR[i] * hL[j] / N - K[c] * hS[idx[c]];
      fid += r * r;
    }
  double pl = 0.0;
  for (int32_t j = 0; j < levels; ++j) pl += (hL[j] - hS[j]) * (hL[j] - hS[j]);
  double pr = 0.0;
  for (int32_t i = 0; i < levels; ++i) pr += (hR[i] - hG[i]) * (hR[i] - hG[i]);
  return fid + alpha * pl + beta * pr;
}

/* Eq. 13. */
int ho_update_reflectance(const double* hL, const double* hS, const double* hG, const double* K,
                          const int32_t* idx, int32_t levels, double N, double beta,
                          int32_t form, double* hR_out) {
  if (!hL || !hS || !hG || !K || !idx || !hR_out || levels < 2 || !(N > 0) || !(beta > 0))
    return HO_EINVAL;
  double den = 0.0;
  for (int32_t j = 0; j < levels; ++j) den += hL[j] * hL[j] / (N * N);
  den += beta;
  for (int32_t i = 0; i < levels; ++i) {
    double num = 0.0;
    for (int32_t j = 0; j < levels; ++j) {
      int64_t c = (int64_t)i * levels + j;
      if (form == 0) {
        num += hL[j] * K[c] * hS[idx[c]] / N; /* K in the numerator (R7) */
      } else if (K[c] != 0.0) {
        num += hL[j] * hS[idx[c]] / (N * K[c]); /* as printed */
      }
    }
    double v = (num + beta * hG[i]) / den;
    hR_out[i] = v > 0.0 ? v : 0.0;
  }
  return HO_OK;
}

/* Eq. 12. */
int ho_update_illumination(const double* hR, const double* hS, const double* K,
                           const int32_t* idx, int32_t levels, double N, double alpha,
                           int32_t form, double* hL_out) {
  if (!hR || !hS || !K || !idx || !hL_out || levels < 2 || !(N > 0) || !(alpha > 0))
    return HO_EINVAL;
  double den = 0.0;
  for (int32_t i = 0; i < levels; ++i) den += hR[i] * hR[i] / (N * N);
  den += alpha;
  for (int32_t j = 0; j < levels; ++j) {
    double num = 0.0;
    for (int32_t i = 0; i < levels; ++i) {
      int64_t c = (int64_t)i * levels + j;
      if (form == 0) {
        num += hR[i] * K[c] * hS[idx[c]] / N;
      } else if (K[c] != 0.0) {
        num += hR[i] * hS[idx[c]] / (N * K[c]);
      }
    }
    double v = (num + alpha * hS[j]) / den;
    hL_out[j] = v > 0.0 ? v : 0.0;
  }
  return HO_OK;
}

/* Eqs. 14-15. */
int ho_renormalize(const double* h, int32_t levels, double N, double* out) {
  if (!h || !out || levels < 1) return HO_EINVAL;
  double s = 0.0;
  for (int32_t k = 0; k < levels; ++k) s += h[k];
  if (!(s > 0.0)) return HO_EDEGENERATE;
  for (int32_t k = 0; k < levels; ++k) out[k] = N * h[k] / s;
  return HO_OK;
}

static int check_params(const ho_params* p) {
  if (!p) return HO_EINVAL;
  if (p->levels < 2 || !(p->alpha > 0) || !(p->beta > 0) || !(p->gamma >= 1.0) ||
      !(p->epsilon > 0) || p->max_iter < 1 || (p->update_form != 0 && p->update_form != 1) ||
      (p->grad_norm != 0 && p->grad_norm != 1))
    return HO_EINVAL;
  return HO_OK;
}

/* Algorithm 1 with a precomputed index map. */
static int decompose_idx(const double* hS, const double* hG, const ho_params* p, const int32_t* idx,
                         double* hL_out, double* hR_out, int32_t* iters, double* trace,
                         int32_t trace_cap) {
  const int32_t l = p->levels;
  const size_t L = (size_t)l, LL = L * L;
  double N = 0.0;
  for (int32_t k = 0; k < l; ++k) N += hS[k];
  if (!(N > 0.0)) return HO_EEMPTY;
  double* hR = (double*)malloc(sizeof(double) * L);
  double* hL = (double*)malloc(sizeof(double) * L);
  double* hR1 = (double*)malloc(sizeof(double) * L);
  double* hL1 = (double*)malloc(sizeof(double) * L);
  double* hRt = (double*)malloc(sizeof(double) * L);
  double* hLt = (double*)malloc(sizeof(double) * L);
  double* est = (double*)malloc(sizeof(double) * L);
  double* C = (double*)malloc(sizeof(double) * LL);
  double* K = (double*)malloc(sizeof(double) * LL);
  int rc = HO_OK;
  if (!hR || !hL || !hR1 || !hL1 || !hRt || !hLt || !est || !C || !K) {
    rc = HO_EINVAL;
    goto done;
  }
  /* Initialisation: H_C(R)^(0) = H_C(grad S); H_C(L)^(0) = H_C(S) (R9). */
  for (int32_t k = 0; k < l; ++k) {
    hR[k] = hG[k];
    hL[k] = hS[k];
  }
  /* K^(0) by Eq. 11 from the count matrix of Eq. 6. */
  ho_pair_count(hR, hL, l, N, C);
  ho_estimate(C, idx, l, est);
  ho_weights(C, idx, est, l, K);
  const double eps = p->epsilon * N * N; /* R11: epsilon is relative to N^2 */
  int32_t t = 0;
  int32_t nt = 0;
  for (;;) {
    if (trace && nt < trace_cap)
      trace[nt++] = ho_objective(hR, hL, hS, hG, K, idx, l, N, p->alpha, p->beta);
    /* Update H_C(R)^(t+1) by Eq. (13) */
    ho_update_reflectance(hL, hS, hG, K, idx, l, N, p->beta, p->update_form, hR1);
    if (trace && nt < trace_cap)
      trace[nt++] = ho_objective(hR1, hL, hS, hG, K, idx, l, N, p->alpha, p->beta);
    /* Update H_C(L)^(t+1) by Eq. (12) -- uses the raw H_C(R)^(t+1) and the frozen K^(t) (R10) */
    ho_update_illumination(hR1, hS, K, idx, l, N, p->alpha, p->update_form, hL1);
    if (trace && nt < trace_cap)
      trace[nt++] = ho_objective(hR1, hL1, hS, hG, K, idx, l, N, p->alpha, p->beta);
    /* Eq. (15) then Eq. (14) */
    rc = ho_renormalize(hR1, l, N, hRt);
    if (rc) goto done;
    rc = ho_renormalize(hL1, l, N, hLt);
    if (rc) goto done;
    double dR = 0.0, dL = 0.0;
    for (int32_t k = 0; k < l; ++k) dR += (hRt[k] - hR[k]) * (hRt[k] - hR[k]);
    for (int32_t k = 0; k < l; ++k) dL += (hLt[k] - hL[k]) * (hLt[k] - hL[k]);
    for (int32_t k = 0; k < l; ++k) {
      hR[k] = hRt[k];
      hL[k] = hLt[k];
    }
    /* Update K^(t+1) by Eq. (11) */
    ho_pair_count(hR, hL, l, N, C);
    ho_estimate(C, idx, l, est);
    ho_weights(C, idx, est, l, K);
    t = t + 1;
    /* until (R11): (||dR||^2 <= eps and ||dL||^2 <= eps) or t >= T */
    if ((p->use_epsilon && dR <= eps && dL <= eps) || t >= p->max_iter) break;
  }
  for (int32_t k = 0; k < l; ++k) {
    hL_out[k] = hL[k];
    hR_out[k] = hR[k];
  }
  if (iters) *iters = t;
done:
  free(hR);
  free(hL);
  free(hR1);
  free(hL1);
  free(hRt);
  free(hLt);
  free(est);
  free(C);
  free(K);
  return rc;
}

int ho_decompose(const double* hS, const double* hG, const ho_params* p, double* hL, double* hR,
                 int32_t* iters, double* trace, int32_t trace_cap) {
  int rc = check_params(p);
  if (rc) return rc;
  if (!hS || !hG || !hL || !hR) return HO_EINVAL;
  const size_t LL = (size_t)p->levels * (size_t)p->levels;
  int32_t* idx = (int32_t*)malloc(sizeof(int32_t) * LL);
  if (!idx) return HO_EINVAL;
  ho_index_map(p->levels, 1.0, idx);
  rc = decompose_idx(hS, hG, p, idx, hL, hR, iters, trace, trace_cap);
  free(idx);
  return rc;
}

/* Eq. 20: H_C(S~)_k = sum over index_1(i,j) == k of H_C(R,L)_ij. */
int ho_enhanced_histogram(const double* hR, const double* hL, const int32_t* idx1,
                          int32_t levels, double N, double* T) {
  if (!hR || !hL || !idx1 || !T || levels < 2 || !(N > 0)) return HO_EINVAL;
  for (int32_t k = 0; k < levels; ++k) T[k] = 0.0;
  for (int32_t i = 0; i < levels; ++i)
    for (int32_t j = 0; j < levels; ++j) T[idx1[(int64_t)i * levels + j]] += hR[i] * hL[j] / N;
  return HO_OK;
}

/* P:308 histogram matching (R16). */
int ho_match_lut(const uint64_t* hS, const double* T, int32_t levels, int32_t* lut, double* margin) {
  if (!hS || !T || !lut || levels < 2) return HO_EINVAL;
  const size_t L = (size_t)levels;
  double* Cs = (double*)malloc(sizeof(double) * L);
  double* Pt = (double*)malloc(sizeof(double) * L);
  double* Ct = (double*)malloc(sizeof(double) * L);
  int rc = HO_OK;
  if (!Cs || !Pt || !Ct) {
    rc = HO_EINVAL;
    goto done;
  }
  uint64_t N = 0;
  for (int32_t k = 0; k < levels; ++k) N += hS[k];
  if (N == 0) {
    rc = HO_EEMPTY;
    goto done;
  }
  uint64_t Ps = 0;
  for (int32_t v = 0; v < levels; ++v) {
    Ps += hS[v];
    Cs[v] = (double)Ps / (double)N;
  }
  Pt[0] = T[0];
  for (int32_t k = 1; k < levels; ++k) Pt[k] = Pt[k - 1] + T[k];
  if (!(Pt[levels - 1] > 0.0)) {
    rc = HO_EDEGENERATE;
    goto done;
  }
  for (int32_t k = 0; k < levels; ++k) Ct[k] = Pt[k] / Pt[levels - 1];
  for (int32_t v = 0; v < levels; ++v) {
    int32_t best = 0;
    double bestd = fabs(Ct[0] - Cs[v]);
    for (int32_t k = 1; k < levels; ++k) {
      double d = fabs(Ct[k] - Cs[v]);
      if (d < bestd) {
        bestd = d;
        best = k;
      }
    }
    lut[v] = best;
    if (margin) {
      double second = INFINITY;
      for (int32_t k = 0; k < levels; ++k) {
        double d = fabs(Ct[k] - Cs[v]);
        if (d > bestd && d < second) second = d;
      }
      margin[v] = second - bestd;
    }
  }
done:
  free(Cs);
  free(Pt);
  free(Ct);
  return rc;
}

/* Eq. 5. */
int ho_he_transform(const uint64_t* hS, int32_t levels, int32_t* t) {
  if (!hS || !t || levels < 2) return HO_EINVAL;
  uint64_t N = 0;
  for (int32_t k = 0; k < levels; ++k) N += hS[k];
  if (N == 0) return HO_EEMPTY;
  double c = 0.0;
  for (int32_t i = 0; i < levels; ++i) {
    c += (double)hS[i] / (double)N; /* Eq. 4 */
    t[i] = (int32_t)floor((double)(levels - 1) * c + 0.5);
  }
  return HO_OK;
}

/* ------------------------------------------- exact hexcone HSV (O11, R17) */

typedef struct {
  int64_t n, d; /* value n/d, d > 0, reduced */
} rat;

static int64_t gcd64(int64_t a, int64_t b) {
  if (a < 0) a = -a;
  while (b) {
    int64_t t = a % b;
    a = b;
    b = t;
  }
  return a ? a : 1;
}
static rat R(int64_t n, int64_t d) {
  if (d < 0) {
    n = -n;
    d = -d;
  }
  int64_t g = gcd64(n, d);
  rat r = {n / g, d / g};
  return r;
}
static rat radd(rat a, rat b) { return R(a.n * b.d + b.n * a.d, a.d * b.d); }
static rat rsub(rat a, rat b) { return R(a.n * b.d - b.n * a.d, a.d * b.d); }
static rat rmul(rat a, rat b) { return R(a.n * b.n, a.d * b.d); }
static rat rdiv(rat a, rat b) { return R(a.n * b.d, a.d * b.n); }
static int64_t rfloor(rat a) { return a.n >= 0 ? a.n / a.d : -((-a.n + a.d - 1) / a.d); }
/* round half up of a >= 0 */
static int64_t rround(rat a) { return rfloor(radd(a, R(1, 2))); }

/* Standard hexcone conversion (rgb_to_hsv / hsv_to_rgb) in exact arithmetic; the
   value channel v is replaced by vnew/255 and each channel rounded half up to 8 bits. */
static void hexcone_replace_v(int r8, int g8, int b8, int vnew8, uint8_t* out) {
  rat r = R(r8, 255), g = R(g8, 255), b = R(b8, 255);
  int mx8 = r8 > g8 ? (r8 > b8 ? r8 : b8) : (g8 > b8 ? g8 : b8);
  int mn8 = r8 < g8 ? (r8 < b8 ? r8 : b8) : (g8 < b8 ? g8 : b8);
  rat maxc = R(mx8, 255), minc = R(mn8, 255);
  rat h = R(0, 1), s = R(0, 1);
  /* rgb -> hsv */
  if (mx8 != mn8) {
    s = rdiv(rsub(maxc, minc), maxc);
    rat span = rsub(maxc, minc);
    rat rc = rdiv(rsub(maxc, r), span);
    rat gc = rdiv(rsub(maxc, g), span);
    rat bc = rdiv(rsub(maxc, b), span);
    if (r8 == mx8)
      h = rsub(bc, gc);
    else if (g8 == mx8)
      h = radd(R(2, 1), rsub(rc, bc));
    else
      h = radd(R(4, 1), rsub(gc, rc));
    h = rdiv(h, R(6, 1));
    h = rsub(h, R(rfloor(h), 1)); /* h mod 1.0 */
  }
  rat v = R(vnew8, 255);
  rat c[3];
  /* hsv -> rgb */
  if (s.n == 0) {
    c[0] = c[1] = c[2] = v;
  } else {
    rat h6 = rmul(h, R(6, 1));
    int64_t i = rfloor(h6);
    rat f = rsub(h6, R(i, 1));
    rat one = R(1, 1);
    rat p = rmul(v, rsub(one, s));
    rat q = rmul(v, rsub(one, rmul(s, f)));
    rat t = rmul(v, rsub(one, rmul(s, rsub(one, f))));
    switch (i % 6) {
      case 0: c[0] = v; c[1] = t; c[2] = p; break;
      case 1: c[0] = q; c[1] = v; c[2] = p; break;
      case 2: c[0] = p; c[1] = v; c[2] = t; break;
      case 3: c[0] = p; c[1] = q; c[2] = v; break;
      case 4: c[0] = t; c[1] = p; c[2] = v; break;
      default: c[0] = v; c[1] = p; c[2] = q; break;
    }
  }
  for (int k = 0; k < 3; ++k) out[k] = (uint8_t)rround(rmul(c[k], R(255, 1)));
}

int ho_reconstruct(const uint8_t* rgb, int64_t npix, const int32_t* Vnew, uint8_t* out) {
  if (!rgb || !Vnew || !out) return HO_EINVAL;
  if (npix <= 0) return HO_EEMPTY;
  for (int64_t p = 0; p < npix; ++p) {
    if (Vnew[p] < 0 || Vnew[p] > 255) return HO_EINVAL;
    hexcone_replace_v(rgb[3 * p], rgb[3 * p + 1], rgb[3 * p + 2], Vnew[p], out + 3 * p);
  }
  return HO_OK;
}

/* ---------------------------------------------------------------- pipeline */

static int enhance_idx(const uint8_t* rgb, int32_t H, int32_t W, const ho_params* p,
                       const int32_t* idx, const int32_t* idx1, uint8_t* out, uint64_t* hS_o,
                       uint64_t* hG_o, uint64_t* hgraw_o, double* hL_o, double* hR_o,
                       double* T_o, int32_t* lut_o, int32_t* iters_o, double* margin_o) {
  const int32_t l = 256;
  const int64_t n = (int64_t)H * W;
  if (n <= 0) return HO_EEMPTY;
  int rc = HO_OK;
  int32_t* S = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  int32_t* g = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  int32_t* gq = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  int32_t* Vn = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  uint64_t hS[256], hG[256], hgraw[511];
  double dS[256], dG[256], hL[256], hR[256], T[256], margin[256];
  int32_t lut[256], iters = 0;
  if (!S || !g || !gq || !Vn) {
    rc = HO_EINVAL;
    goto done;
  }
  /* Alg. 1 lines 1-2: histograms of S and of the gradient image. */
  if ((rc = ho_value_channel(rgb, n, l, S))) goto done;
  if ((rc = ho_gradient_raw(S, H, W, g))) goto done;
  if ((rc = ho_gradient_levels(g, n, l, p->grad_norm, gq))) goto done;
  if ((rc = ho_count_histogram(S, n, l, hS))) goto done;
  if ((rc = ho_count_histogram(gq, n, l, hG))) goto done;
  if ((rc = ho_count_histogram(g, n, 2 * l - 1, hgraw))) goto done;
  for (int32_t k = 0; k < l; ++k) {
    dS[k] = (double)hS[k];
    dG[k] = (double)hG[k];
  }
  /* Algorithm 1 */
  if ((rc = decompose_idx(dS, dG, p, idx, hL, hR, &iters, NULL, 0))) goto done;
  /* Eqs. 17-20 */
  if ((rc = ho_enhanced_histogram(hR, hL, idx1, l, (double)n, T))) goto done;
  /* P:308 histogram matching */
  if ((rc = ho_match_lut(hS, T, l, lut, margin_o ? margin : NULL))) goto done;
  for (int64_t q = 0; q < n; ++q) Vn[q] = lut[S[q]];
  if (out && (rc = ho_reconstruct(rgb, n, Vn, out))) goto done;
  for (int32_t k = 0; k < l; ++k) {
    if (hS_o) hS_o[k] = hS[k];
    if (hG_o) hG_o[k] = hG[k];
    if (hL_o) hL_o[k] = hL[k];
    if (hR_o) hR_o[k] = hR[k];
    if (T_o) T_o[k] = T[k];
    if (lut_o) lut_o[k] = lut[k];
    if (margin_o) margin_o[k] = margin[k];
  }
  if (hgraw_o)
    for (int32_t k = 0; k < 2 * l - 1; ++k) hgraw_o[k] = hgraw[k];
  if (iters_o) *iters_o = iters;
done:
  free(S);
  free(g);
  free(gq);
  free(Vn);
  return rc;
}

int ho_enhance(const uint8_t* rgb, int32_t H, int32_t W, const ho_params* p, uint8_t* out,
               uint64_t* hS, uint64_t* hG, uint64_t* hgraw, double* hL, double* hR, double* T,
               int32_t* lut, int32_t* iters, double* lut_margin) {
  int rc = check_params(p);
  if (rc) return rc;
  if (p->levels != 256 || !rgb || H < 0 || W < 0) return HO_EINVAL;
  if ((int64_t)H * W == 0) return HO_EEMPTY;
  int32_t* idx = (int32_t*)malloc(sizeof(int32_t) * 65536);
  int32_t* idx1 = (int32_t*)malloc(sizeof(int32_t) * 65536);
  if (!idx || !idx1) {
    free(idx);
    free(idx1);
    return HO_EINVAL;
  }
  ho_index_map(256, 1.0, idx);
  ho_index_map(256, p->gamma, idx1);
  rc = enhance_idx(rgb, H, W, p, idx, idx1, out, hS, hG, hgraw, hL, hR, T, lut, iters, lut_margin);
  free(idx);
  free(idx1);
  return rc;
}

typedef struct {
  const uint8_t* rgb;
  int64_t B;
  int32_t H, W;
  const ho_params* p;
  const int32_t *idx, *idx1;
  uint8_t* out;
  uint64_t *hS, *hG;
  double *hL, *hR, *T;
  int32_t *lut, *iters;
  int64_t next; /* guarded by mu */
  pthread_mutex_t mu;
  int rc;
} batch_job;

static void* batch_worker(void* arg) {
  batch_job* J = (batch_job*)arg;
  const int64_t npx = (int64_t)J->H * J->W;
  for (;;) {
    pthread_mutex_lock(&J->mu);
    int64_t b = J->next++;
    pthread_mutex_unlock(&J->mu);
    if (b >= J->B) break;
    int rc = enhance_idx(J->rgb + b * npx * 3, J->H, J->W, J->p, J->idx, J->idx1,
                         J->out ? J->out + b * npx * 3 : NULL, J->hS ? J->hS + b * 256 : NULL,
                         J->hG ? J->hG + b * 256 : NULL, NULL, J->hL ? J->hL + b * 256 : NULL,
                         J->hR ? J->hR + b * 256 : NULL, J->T ? J->T + b * 256 : NULL,
                         J->lut ? J->lut + b * 256 : NULL, J->iters ? J->iters + b : NULL, NULL);
    if (rc) {
      pthread_mutex_lock(&J->mu);
      J->rc = rc;
      pthread_mutex_unlock(&J->mu);
    }
  }
  return NULL;
}

int ho_enhance_batch(const uint8_t* rgb, int64_t B, int32_t H, int32_t W, const ho_params* p,
                     uint8_t* out, uint64_t* hS, uint64_t* hG, double* hL, double* hR,
                     double* T, int32_t* lut, int32_t* iters, int32_t nthreads) {
  int rc = check_params(p);
  if (rc) return rc;
  if (p->levels != 256 || !rgb || B < 1 || H < 0 || W < 0 || nthreads < 1) return HO_EINVAL;
  if ((int64_t)H * W == 0) return HO_EEMPTY;
  batch_job J;
  memset(&J, 0, sizeof J);
  J.rgb = rgb;
  J.B = B;
  J.H = H;
  J.W = W;
  J.p = p;
  J.out = out;
  J.hS = hS;
  J.hG = hG;
  J.hL = hL;
  J.hR = hR;
  J.T = T;
  J.lut = lut;
  J.iters = iters;
  int32_t* idx = (int32_t*)malloc(sizeof(int32_t) * 65536);
  int32_t* idx1 = (int32_t*)malloc(sizeof(int32_t) * 65536);
  if (!idx || !idx1) {
    free(idx);
    free(idx1);
    return HO_EINVAL;
  }
  ho_index_map(256, 1.0, idx);
  ho_index_map(256, p->gamma, idx1);
  J.idx = idx;
  J.idx1 = idx1;
  pthread_mutex_init(&J.mu, NULL);
  if (nthreads == 1) {
    batch_worker(&J);
  } else {
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
    int32_t started = 0;
    for (int32_t t = 0; t < nthreads; ++t)
      if (pthread_create(&th[started], NULL, batch_worker, &J) == 0) ++started;
    if (started == 0) batch_worker(&J);
    for (int32_t t = 0; t < started; ++t) pthread_join(th[t], NULL);
    free(th);
  }
  pthread_mutex_destroy(&J.mu);
  free(idx);
  free(idx1);
  return J.rc;
}

/* ============================ second workload: HE baseline and quality metrics (NEXT #4) */

int ho_he_enhance(const uint8_t* rgb, int32_t H, int32_t W, uint8_t* out) {
  if (!rgb || !out || H <= 0 || W <= 0) return HO_EINVAL;
  const int64_t n = (int64_t)H * W;
  uint64_t hS[256];
  int32_t t[256];
  memset(hS, 0, sizeof hS);
  for (int64_t p = 0; p < n; ++p) {
    uint8_t v = rgb[3 * p];
    if (rgb[3 * p + 1] > v) v = rgb[3 * p + 1];
    if (rgb[3 * p + 2] > v) v = rgb[3 * p + 2];
    hS[v]++;
  }
  int rc = ho_he_transform(hS, 256, t);
  if (rc) return rc;
  int32_t* Vn = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  if (!Vn) return HO_EINVAL;
  for (int64_t p = 0; p < n; ++p) {
    uint8_t v = rgb[3 * p];
    if (rgb[3 * p + 1] > v) v = rgb[3 * p + 1];
    if (rgb[3 * p + 2] > v) v = rgb[3 * p + 2];
    Vn[p] = t[v];
  }
  rc = ho_reconstruct(rgb, n, Vn, out);
  free(Vn);
  return rc;
}

double ho_psnr(const uint8_t* a, const uint8_t* b, int64_t npix) {
  uint64_t sse = 0;
  for (int64_t i = 0; i < 3 * npix; ++i) {
    const int64_t d = (int64_t)a[i] - (int64_t)b[i];
    sse += (uint64_t)(d * d);
  }
  if (sse == 0) return INFINITY;
  const double mse = (double)sse / (double)(3 * npix);
  return 10.0 * log10(255.0 * 255.0 / mse);
}

double ho_ssim(const uint8_t* a, const uint8_t* b, int32_t H, int32_t W) {
  if (H < 11 || W < 11) return NAN;
  const int R = 5;
  double g[11], gs = 0.0;
  for (int k = -R; k <= R; ++k) {
    g[k + R] = exp(-(double)(k * k) / (2.0 * 1.5 * 1.5));
    gs += g[k + R];
  }
  for (int k = 0; k < 11; ++k) g[k] /= gs;
  const double C1 = (0.01 * 255.0) * (0.01 * 255.0), C2 = (0.03 * 255.0) * (0.03 * 255.0);
  const size_t n = (size_t)H * W;
  double* ya = (double*)malloc(sizeof(double) * n);
  double* yb = (double*)malloc(sizeof(double) * n);
  if (!ya || !yb) {
    free(ya);
    free(yb);
    return NAN;
  }
  for (size_t p = 0; p < n; ++p) {
    ya[p] = 0.299 * a[3 * p] + 0.587 * a[3 * p + 1] + 0.114 * a[3 * p + 2];
    yb[p] = 0.299 * b[3 * p] + 0.587 * b[3 * p + 1] + 0.114 * b[3 * p + 2];
  }
  double sum = 0.0;
  for (int y = R; y < H - R; ++y)
    for (int x = R; x < W - R; ++x) {
      double ma = 0.0, mb = 0.0, saa = 0.0, sbb = 0.0, sab = 0.0;
      for (int dy = -R; dy <= R; ++dy)
        for (int dx = -R; dx <= R; ++dx) {
          const double w = g[dy + R] * g[dx + R];
          const size_t q = (size_t)(y + dy) * W + (x + dx);
          ma += w * ya[q];
          mb += w * yb[q];
          saa += w * ya[q] * ya[q];
          sbb += w * yb[q] * yb[q];
          sab += w * ya[q] * yb[q];
        }
      const double va = saa - ma * ma, vb = sbb - mb * mb, cov = sab - ma * mb;
      sum += ((2.0 * ma * mb + C1) * (2.0 * cov + C2)) / ((ma * ma + mb * mb + C1) * (va + vb + C2));
    }
  free(ya);
  free(yb);
  return sum / ((double)(H - 2 * R) * (double)(W - 2 * R));
}

double ho_loe(const uint8_t* orig, const uint8_t* enh, int32_t H, int32_t W) {
  if (!orig || !enh || H <= 0 || W <= 0) return NAN;
  const int mh = H < 100 ? H : 100, mw = W < 100 ? W : 100;
  const int m = mh * mw;
  uint8_t* L = (uint8_t*)malloc((size_t)m);
  uint8_t* Le = (uint8_t*)malloc((size_t)m);
  if (!L || !Le) {
    free(L);
    free(Le);
    return NAN;
  }
  for (int i = 0; i < mh; ++i)
    for (int j = 0; j < mw; ++j) {
      const int64_t y = (int64_t)i * H / mh, x = (int64_t)j * W / mw;
      const uint8_t* p = orig + 3 * (y * W + x);
      const uint8_t* q = enh + 3 * (y * W + x);
      uint8_t l = p[0], le = q[0];
      if (p[1] > l) l = p[1];
      if (p[2] > l) l = p[2];
      if (q[1] > le) le = q[1];
      if (q[2] > le) le = q[2];
      L[i * mw + j] = l;
      Le[i * mw + j] = le;
    }
  uint64_t cnt = 0;
  for (int x = 0; x < m; ++x)
    for (int y = 0; y < m; ++y) cnt += (uint64_t)((L[x] >= L[y]) != (Le[x] >= Le[y]));
  free(L);
  free(Le);
  return (double)cnt / (double)m;
}
