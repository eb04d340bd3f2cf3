/*
 * fbs_oracle.c — CPU ORACLE for the fast bilateral stereo (FBS) hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the plain, slow, obviously-correct
 * double-precision definition of what the B200 path computes.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load it.  It shares no code, header, table or constant generator with
 * the CUDA path (paper_1807_02044_b200/csrc), and neither side includes the
 * other.
 *
 * Every function cites the PAPER.md passage it follows ("P:Lnn" = line of
 * /root/reference/PAPER.md; equation numbers are the LaTeX ordinals, see
 * DESIGN.md §2).  Where the paper is silent the reading taken is the one
 * listed in DESIGN.md §3 ("R#k").
 *
 * Conventions:
 *   images    uint8 grayscale, row-major [H][W]                       (R#3)
 *   volumes   double, index ((v*W+u)*D + d-d_min)   (SPEC cost_volume_index)
 *   SENT      -2.0 marks an undefined cost / aggregated cost          (R#7)
 *   INVALID   -1 (int maps) / -1.0 (subpixel map)                     (R#23)
 * Arithmetic: double, no contraction (-ffp-contract=off), no fast-math.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_SENT (-2.0)
#define ORACLE_INVALID (-1)
#define ORACLE_RHO_NCC 1        /* ϱ = 1, "ϱ is set to 1 in this paper"          */
#define ORACLE_N 9              /* n = (2ϱ+1)^2                                   */
#define ORACLE_SIGMA_FLOOR 1e-6 /* textureless block => NCC undefined (R#7)              */
#define ORACLE_LRC_TOL 1        /* R#17                                                  */
#define ORACLE_SUBPIX_EPS 1e-9  /* R#21                                                  */

/* ------------------------------------------------------------------------- */
/* Eq.(2)(3): mean μ and standard deviation σ of the (2ϱ+1)^2 block
 * centred at (u,v).  Population form: σ = sqrt(Σ i^2 / n − μ^2)  (R#4).
 * Returns 0 (undefined) when the block does not fit in the image (R#7). */
static int block_stat(const uint8_t* I, int W, int H, int u, int v, double* mu, double* sigma) {
  if (u - ORACLE_RHO_NCC < 0 || u + ORACLE_RHO_NCC > W - 1 || v - ORACLE_RHO_NCC < 0 ||
      v + ORACLE_RHO_NCC > H - 1)
    return 0;
  double s = 0.0, q = 0.0;
  for (int y = v - ORACLE_RHO_NCC; y <= v + ORACLE_RHO_NCC; ++y)
    for (int x = u - ORACLE_RHO_NCC; x <= u + ORACLE_RHO_NCC; ++x) {
      double i = (double)I[y * W + x];
      s += i;
      q += i * i;
    }
  double m = s / ORACLE_N;
  double var = q / ORACLE_N - m * m;
  if (var < 0.0) var = 0.0; /* guards a -0 from rounding; exact integers make it >= 0 */
  *mu = m;
  *sigma = sqrt(var);
  return 1;
}

void oracle_block_stats(const uint8_t* I, int W, int H, double* mu, double* sigma, uint8_t* defined) {
  for (int v = 0; v < H; ++v)
    for (int u = 0; u < W; ++u) {
      double m = 0.0, s = 0.0;
      int ok = block_stat(I, W, H, u, v, &m, &s);
      mu[v * W + u] = ok ? m : 0.0;
      sigma[v * W + u] = ok ? s : 0.0;
      if (defined) defined[v * W + u] = (uint8_t)ok;
    }
}

/* ------------------------------------------------------------------------- */
/* Eq.(1): NCC between the left block centred at (u,v) and the right
 * block centred at (u-d,v):
 *   c = (Σ i_l(x,y) i_r(x-d,y) − n μ_l μ_r) / (n σ_l σ_r),  clamped to [-1,1] (R#8).
 * μ, σ are the pre-calculated block statistics.
 * SENT when either block is undefined (border / right block outside the image)
 * or either σ is below the floor (R#7). */
static double ncc(const uint8_t* IL, const uint8_t* IR, int W, int H, int u, int v, int d,
                  double mu_l, double sig_l, int def_l, double mu_r, double sig_r, int def_r) {
  (void)H;
  if (!def_l || !def_r) return ORACLE_SENT;
  if (sig_l < ORACLE_SIGMA_FLOOR || sig_r < ORACLE_SIGMA_FLOOR) return ORACLE_SENT;
  double dot = 0.0;
  for (int y = v - ORACLE_RHO_NCC; y <= v + ORACLE_RHO_NCC; ++y)
    for (int x = u - ORACLE_RHO_NCC; x <= u + ORACLE_RHO_NCC; ++x)
      dot += (double)IL[y * W + x] * (double)IR[y * W + (x - d)];
  double c = (dot - ORACLE_N * mu_l * mu_r) / (ORACLE_N * sig_l * sig_r);
  if (c > 1.0) c = 1.0;
  if (c < -1.0) c = -1.0;
  return c;
}

/* NCC at (u,v,d) from the raw images (statistics computed on the spot). */
double oracle_ncc_at(const uint8_t* IL, const uint8_t* IR, int W, int H, int u, int v, int d) {
  double ml = 0, sl = 0, mr = 0, sr = 0;
  int dl = block_stat(IL, W, H, u, v, &ml, &sl);
  int dr = (u - d >= 0) ? block_stat(IR, W, H, u - d, v, &mr, &sr) : 0;
  return ncc(IL, IR, W, H, u, v, d, ml, sl, dl, mr, sr, dr);
}

/* "The calculated correlation costs c are simultaneously stored
 * in the left and right 3-D cost volumes ... the value of c at (u,v,d) in the
 * left cost volume is the same as that at (u-d,v,d) in the right cost volume."
 * One evaluation, written twice; right entries never written stay SENT. */
void oracle_cost_volumes(const uint8_t* IL, const uint8_t* IR, int W, int H, int d_min, int d_max,
                         double* cost_l, double* cost_r, int nthreads) {
  const int D = d_max - d_min + 1;
  const size_t npix = (size_t)W * H;
  double* mu_l = (double*)malloc(npix * sizeof(double));
  double* sg_l = (double*)malloc(npix * sizeof(double));
  double* mu_r = (double*)malloc(npix * sizeof(double));
  double* sg_r = (double*)malloc(npix * sizeof(double));
  uint8_t* df_l = (uint8_t*)malloc(npix);
  uint8_t* df_r = (uint8_t*)malloc(npix);
  oracle_block_stats(IL, W, H, mu_l, sg_l, df_l);
  oracle_block_stats(IR, W, H, mu_r, sg_r, df_r);
  for (size_t i = 0; i < npix * D; ++i) {
    cost_l[i] = ORACLE_SENT;
    cost_r[i] = ORACLE_SENT;
  }
  /* rows are independent; the right-volume write (u-d,v) stays in row v */
#pragma omp parallel for schedule(static) num_threads(nthreads)
  for (int v = 0; v < H; ++v)
    for (int u = 0; u < W; ++u)
      for (int d = d_min; d <= d_max; ++d) {
        const int ur = u - d;
        double c = ORACLE_SENT;
        if (ur >= 0)
          c = ncc(IL, IR, W, H, u, v, d, mu_l[v * W + u], sg_l[v * W + u], df_l[v * W + u],
                  mu_r[v * W + ur], sg_r[v * W + ur], df_r[v * W + ur]);
        cost_l[((size_t)v * W + u) * D + (d - d_min)] = c;
        if (ur >= 0 && c != ORACLE_SENT) cost_r[((size_t)v * W + ur) * D + (d - d_min)] = c;
      }
  free(mu_l); free(sg_l); free(mu_r); free(sg_r); free(df_l); free(df_r);
}

/* ------------------------------------------------------------------------- */
/* Eq.(7): ω_d = exp{-((x-u)^2 + (y-v)^2) / γ_d^2}; table indexed
 * [(dy+ρ)(2ρ+1) + (dx+ρ)] (R#10: γ used verbatim, no 2σ^2). */
void oracle_spatial_weights(int rho, double gamma_d, double* wd) {
  const int K1 = 2 * rho + 1;
  for (int dy = -rho; dy <= rho; ++dy)
    for (int dx = -rho; dx <= rho; ++dx)
      wd[(dy + rho) * K1 + (dx + rho)] = exp(-((double)(dx * dx + dy * dy)) / (gamma_d * gamma_d));
}

/* Eq.(8): ω_r = exp{-(i(x,y) - i(u,v))^2 / γ_r^2} for |Δ| = 0..255. */
void oracle_range_weights(double gamma_r, double* wr) {
  for (int a = 0; a < 256; ++a) wr[a] = exp(-((double)a * (double)a) / (gamma_r * gamma_r));
}

/* Eq.(6): c_agg(u,v,d) = Σ ω_d ω_r c / Σ ω_d ω_r over the (2ρ+1)^2
 * window of (u,v); the guide i is the volume's own image (R#11).  Window
 * truncated to the image, SENT taps excluded from both sums, SENT if none is
 * left (R#12).  Summation order: dy-major, dx-minor. */
static double bilateral_at(const double* cost, const uint8_t* guide, int W, int H, int D, int u, int v,
                           int di, int rho, const double* wd, const double* wr) {
  const int K1 = 2 * rho + 1;
  const int gp = guide[v * W + u];
  double num = 0.0, den = 0.0;
  int any = 0;
  for (int y = v - rho; y <= v + rho; ++y) {
    if (y < 0 || y >= H) continue;
    for (int x = u - rho; x <= u + rho; ++x) {
      if (x < 0 || x >= W) continue;
      const double c = cost[((size_t)y * W + x) * D + di];
      if (c == ORACLE_SENT) continue;
      const double w = wd[(y - v + rho) * K1 + (x - u + rho)] * wr[abs((int)guide[y * W + x] - gp)];
      num += w * c;
      den += w;
      any = 1;
    }
  }
  if (!any) return ORACLE_SENT;
  return num / den;
}

void oracle_aggregate(const double* cost, const uint8_t* guide, int W, int H, int D, int rho,
                      double gamma_d, double gamma_r, double* agg, int nthreads) {
  const int K1 = 2 * rho + 1;
  double* wd = (double*)malloc((size_t)K1 * K1 * sizeof(double));
  double wr[256];
  oracle_spatial_weights(rho, gamma_d, wd);
  oracle_range_weights(gamma_r, wr);
#pragma omp parallel for schedule(static) num_threads(nthreads)
  for (int v = 0; v < H; ++v)
    for (int u = 0; u < W; ++u)
      for (int di = 0; di < D; ++di)
        agg[((size_t)v * W + u) * D + di] = bilateral_at(cost, guide, W, H, D, u, v, di, rho, wd, wr);
  free(wd);
}

/* ------------------------------------------------------------------------- */
/* WTA: "each SP searches for the highest correlation cost
 * c_agg between (u,v,d_min) and (u,v,d_max)".  Ascending scan, strictly-greater
 * update => ties go to the smallest d (R#15); all-SENT => INVALID.
 * Also reports the best and second-best values (near-tie logging, R#30). */
static int wta_column(const double* col, int D, int d_min, double* best_out, double* second_out) {
  int best = ORACLE_INVALID;
  double bv = ORACLE_SENT, sv = ORACLE_SENT;
  for (int di = 0; di < D; ++di) {
    const double c = col[di];
    if (c == ORACLE_SENT) continue;
    if (best == ORACLE_INVALID || c > bv) {
      if (best != ORACLE_INVALID) sv = bv;
      bv = c;
      best = d_min + di;
    } else if (sv == ORACLE_SENT || c > sv) {
      sv = c;
    }
  }
  if (best_out) *best_out = bv;
  if (second_out) *second_out = sv;
  return best;
}

void oracle_wta(const double* agg, int W, int H, int d_min, int d_max, int32_t* disp, double* best,
                double* second) {
  const int D = d_max - d_min + 1;
  for (size_t p = 0; p < (size_t)W * H; ++p) {
    double b, s;
    disp[p] = wta_column(agg + p * D, D, d_min, &b, &s);
    if (best) best[p] = b;
    if (second) second[p] = s;
  }
}

/* Eq.(9): ℓ^lf(u,v) = ℓ^rt(u − ℓ^lf(u,v), v), left image as
 * reference, tolerance 1 on integer maps (R#17). */
static int lrc_ok(const int32_t* dl, const int32_t* dr, int W, int u, int v) {
  const int d = dl[v * W + u];
  if (d == ORACLE_INVALID) return 0;
  const int ur = u - d;
  if (ur < 0) return 0;
  const int e = dr[v * W + ur];
  if (e == ORACLE_INVALID) return 0;
  return abs(d - e) <= ORACLE_LRC_TOL;
}

void oracle_lrc(const int32_t* dl, const int32_t* dr, int W, int H, uint8_t* valid) {
  for (int v = 0; v < H; ++v)
    for (int u = 0; u < W; ++u) valid[v * W + u] = (uint8_t)lrc_ok(dl, dr, W, u, v);
}

/* Eq.(10): d^s = d + (c(d-1) − c(d+1)) / (2c(d-1) + 2c(d+1) − 4c(d)),
 * on the aggregated costs (R#19), interior d with defined neighbours only,
 * |den| >= 1e-9, offset clamped to ±0.5 (R#21).  Returns also the denominator. */
static double subpixel(const double* col, int D, int d_min, int d, double* den_out) {
  const int di = d - d_min;
  if (den_out) *den_out = 0.0;
  if (di <= 0 || di >= D - 1) return (double)d;
  const double cm = col[di - 1], c0 = col[di], cp = col[di + 1];
  if (cm == ORACLE_SENT || cp == ORACLE_SENT) return (double)d;
  const double den = 2.0 * cm + 2.0 * cp - 4.0 * c0;
  if (den_out) *den_out = den;
  if (fabs(den) < ORACLE_SUBPIX_EPS) return (double)d;
  double delta = (cm - cp) / den;
  if (delta > 0.5) delta = 0.5;
  if (delta < -0.5) delta = -0.5;
  return (double)d + delta;
}

void oracle_subpixel(const double* agg_l, const int32_t* dl, const uint8_t* valid, int W, int H,
                     int d_min, int d_max, double* disp_s, double* den) {
  const int D = d_max - d_min + 1;
  for (size_t p = 0; p < (size_t)W * H; ++p) {
    double dd = 0.0;
    if (!valid[p]) {
      disp_s[p] = (double)ORACLE_INVALID;
    } else {
      disp_s[p] = subpixel(agg_l + p * D, D, d_min, dl[p], &dd);
    }
    if (den) den[p] = dd;
  }
}

/* ------------------------------------------------------------------------- */
/* The whole method in Fig. 1 order: cost → aggregation
 * → WTA (both) → LRC → subpixel.  Every intermediate may be exported; NULL
 * outputs are allocated internally. */
int oracle_fbs(const uint8_t* IL, const uint8_t* IR, int W, int H, int d_min, int d_max, int rho,
               double gamma_d, double gamma_r, int nthreads, double* cost_l, double* cost_r,
               double* agg_l, double* agg_r, int32_t* disp_l, int32_t* disp_r, uint8_t* valid,
               double* disp_s, double* best_l, double* second_l, double* sub_den) {
  if (W < 3 || H < 3 || d_min < 0 || d_max <= d_min || rho < 0 || !(gamma_d > 0) || !(gamma_r > 0))
    return -1;
  const int D = d_max - d_min + 1;
  const size_t nvol = (size_t)W * H * D, npix = (size_t)W * H;
  double *cl = cost_l, *cr = cost_r, *al = agg_l, *ar = agg_r;
  int32_t *dl = disp_l, *dr = disp_r;
  uint8_t* vm = valid;
  if (!cl) cl = (double*)malloc(nvol * sizeof(double));
  if (!cr) cr = (double*)malloc(nvol * sizeof(double));
  if (!al) al = (double*)malloc(nvol * sizeof(double));
  if (!ar) ar = (double*)malloc(nvol * sizeof(double));
  if (!dl) dl = (int32_t*)malloc(npix * sizeof(int32_t));
  if (!dr) dr = (int32_t*)malloc(npix * sizeof(int32_t));
  if (!vm) vm = (uint8_t*)malloc(npix);
  if (!cl || !cr || !al || !ar || !dl || !dr || !vm) return -6;

  oracle_cost_volumes(IL, IR, W, H, d_min, d_max, cl, cr, nthreads);
  oracle_aggregate(cl, IL, W, H, D, rho, gamma_d, gamma_r, al, nthreads);
  oracle_aggregate(cr, IR, W, H, D, rho, gamma_d, gamma_r, ar, nthreads);
  oracle_wta(al, W, H, d_min, d_max, dl, best_l, second_l);
  oracle_wta(ar, W, H, d_min, d_max, dr, NULL, NULL);
  oracle_lrc(dl, dr, W, H, vm);
  if (disp_s) oracle_subpixel(al, dl, vm, W, H, d_min, d_max, disp_s, sub_den);

  if (cl != cost_l) free(cl);
  if (cr != cost_r) free(cr);
  if (al != agg_l) free(al);
  if (ar != agg_r) free(ar);
  if (dl != disp_l) free(dl);
  if (dr != disp_r) free(dr);
  if (vm != valid) free(vm);
  return 0;
}

/* ------------------------------------------------------------------------- */
/* Sampled pixels for frames whose volumes are too large to materialise
 * (BASELINE configs 4-5).  Same definitions, evaluated locally:
 *   agg_l(p,·)  from the NCC of every tap q in p's window     (Eq.(1),(6))
 *   d_L(p)      WTA of that column
 *   agg_r(p',·) at p' = (u − d_L, v) from c_R(q',d) = c_L(q'+d, d)
 *   d_R(p'), LRC, subpixel                                  (Eq.(9),(10))
 * Because block_stat / ncc / the tap order are the same functions as the
 * full-frame path, results are bit-identical to oracle_fbs at those pixels. */
static void agg_column_local(const uint8_t* IL, const uint8_t* IR, int W, int H, int d_min, int d_max,
                             int rho, const double* wd, const double* wr, int side, int u, int v,
                             double* col) {
  const int K1 = 2 * rho + 1;
  const uint8_t* guide = side == 0 ? IL : IR;
  const int gp = guide[v * W + u];
  for (int d = d_min; d <= d_max; ++d) {
    double num = 0.0, den = 0.0;
    int any = 0;
    for (int y = v - rho; y <= v + rho; ++y) {
      if (y < 0 || y >= H) continue;
      for (int x = u - rho; x <= u + rho; ++x) {
        if (x < 0 || x >= W) continue;
        /* left volume entry (x,y,d); right volume entry (x,y,d) = left (x+d,y,d) */
        const int xl = side == 0 ? x : x + d;
        double c = ORACLE_SENT;
        if (xl < W) c = oracle_ncc_at(IL, IR, W, H, xl, y, d);
        if (c == ORACLE_SENT) continue;
        const double w = wd[(y - v + rho) * K1 + (x - u + rho)] * wr[abs((int)guide[y * W + x] - gp)];
        num += w * c;
        den += w;
        any = 1;
      }
    }
    col[d - d_min] = any ? num / den : ORACLE_SENT;
  }
}

int oracle_fbs_pixels(const uint8_t* IL, const uint8_t* IR, int W, int H, int d_min, int d_max, int rho,
                      double gamma_d, double gamma_r, int npts, const int32_t* us, const int32_t* vs,
                      int nthreads, double* disp_s, int32_t* disp_l, int32_t* disp_r_at, double* best_l,
                      double* second_l, double* sub_den, double* agg_col_l) {
  if (W < 3 || H < 3 || d_min < 0 || d_max <= d_min || rho < 0 || !(gamma_d > 0) || !(gamma_r > 0))
    return -1;
  const int D = d_max - d_min + 1;
  const int K1 = 2 * rho + 1;
  double* wd = (double*)malloc((size_t)K1 * K1 * sizeof(double));
  double wr[256];
  oracle_spatial_weights(rho, gamma_d, wd);
  oracle_range_weights(gamma_r, wr);
#pragma omp parallel for schedule(dynamic) num_threads(nthreads)
  for (int i = 0; i < npts; ++i) {
    const int u = us[i], v = vs[i];
    double* coll = (double*)malloc((size_t)D * sizeof(double));
    double* colr = (double*)malloc((size_t)D * sizeof(double));
    agg_column_local(IL, IR, W, H, d_min, d_max, rho, wd, wr, 0, u, v, coll);
    double b, s, den = 0.0;
    const int dl = wta_column(coll, D, d_min, &b, &s);
    int dr = ORACLE_INVALID, ok = 0;
    if (dl != ORACLE_INVALID && u - dl >= 0) {
      agg_column_local(IL, IR, W, H, d_min, d_max, rho, wd, wr, 1, u - dl, v, colr);
      dr = wta_column(colr, D, d_min, NULL, NULL);
      ok = dr != ORACLE_INVALID && abs(dl - dr) <= ORACLE_LRC_TOL;
    }
    disp_s[i] = ok ? subpixel(coll, D, d_min, dl, &den) : (double)ORACLE_INVALID;
    if (disp_l) disp_l[i] = dl;
    if (disp_r_at) disp_r_at[i] = dr;
    if (best_l) best_l[i] = b;
    if (second_l) second_l[i] = s;
    if (sub_den) sub_den[i] = den;
    if (agg_col_l) memcpy(agg_col_l + (size_t)i * D, coll, (size_t)D * sizeof(double));
    free(coll);
    free(colr);
  }
  free(wd);
  return 0;
}
