/*
 * oracle.c — serial CPU restatement of the reference CCD hot path.
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Compiled with -ffp-contract=off
 * like the reference core (src/CMakeLists.txt:11-13) so that products are not
 * fused into FMAs.
 *
 * Strata: the reference has none; every per-stratum loop below evaluates the
 * reference algorithm on the stratum's rows as if they were their own dataset
 * and sums the results (composition).
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define XBETA_BOUND 700.0   /* src/engine.cpp:12 */
#define HW_FLOOR 1e-300     /* src/ccd.cpp:13 */

/* [s, e) row range of the stratum that starts at row s. */
static int64_t stratum_end(const orc_data* d, int64_t s) {
  int64_t e = s + 1;
  if (!d->stratum_start) return d->n;
  while (e < d->n && !d->stratum_start[e]) ++e;
  return e;
}

static int any_competing(const orc_data* d) {
  for (int64_t i = 0; i < d->n; ++i)
    if (d->status[i] == 2) return 1;
  return 0;
}

/* Maximal runs of equal time inside a stratum (src/dataset.cpp:190-204):
 * count_at_end[k] = number of status==1 rows in the block if k is the block's
 * last row, else 0. */
int orc_block_counts(const orc_data* d, double* cnt) {
  for (int64_t s = 0; s < d->n;) {
    const int64_t e = stratum_end(d, s);
    for (int64_t start = s; start < e;) {
      int64_t end = start;
      while (end + 1 < e && d->times[end + 1] == d->times[start]) ++end;
      double c = 0.0;
      for (int64_t k = start; k <= end; ++k) {
        c += d->status[k] == 1 ? 1.0 : 0.0;
        cnt[k] = 0.0;
      }
      cnt[end] = c;
      start = end + 1;
    }
    s = e;
  }
  return ORC_OK;
}

/* KM of the censoring distribution, failures before censorings on ties, and
 * the per-row weights u = 1/G(Y-) (competing rows), g = G(Y-)
 * (src/censoring.cpp:39-90).  Walking blocks in ascending time, G(t-) of a
 * block equals the survival product accumulated over all earlier jumps,
 * which is what CensoringCurve::before() looks up (src/censoring.cpp:32-37). */
int orc_ipcw(const orc_data* d, double* u, double* g) {
  for (int64_t s = 0; s < d->n;) {
    const int64_t e = stratum_end(d, s);
    /* collect block ends of this stratum (local positions) */
    int64_t nb = 0;
    int64_t* ends = (int64_t*)malloc(sizeof(int64_t) * (size_t)(e - s));
    for (int64_t start = s; start < e;) {
      int64_t end = start;
      while (end + 1 < e && d->times[end + 1] == d->times[start]) ++end;
      ends[nb++] = end;
      start = end + 1;
    }
    double surv = 1.0;
    for (int64_t b = nb; b-- > 0;) {
      const int64_t end = ends[b];
      const int64_t start = b == 0 ? s : ends[b - 1] + 1;
      const double before = surv; /* G(t-) for this block's time */
      int64_t censored = 0, failed = 0;
      for (int64_t i = start; i <= end; ++i) {
        if (d->status[i] == 0) ++censored; else ++failed;
        g[i] = before;
        u[i] = 0.0;
        if (d->status[i] == 2) {
          if (!(before > 0.0)) { free(ends); return ORC_DEGENERATE; }
          u[i] = 1.0 / before;
        }
      }
      if (censored) {
        const double at_risk = (double)(end - s + 1 - failed);
        surv *= 1.0 - (double)censored / at_risk;
      }
    }
    free(ends);
    s = e;
  }
  return ORC_OK;
}

/* src/engine.cpp:76-101 (event mask dotted with each column). */
void orc_fixed_terms(const orc_data* d, double* fixed) {
  for (int64_t j = 0; j < d->p; ++j) {
    double acc = 0.0;
    for (int64_t k = d->col_ptr[j]; k < d->col_ptr[j + 1]; ++k) {
      const double m = d->status[d->row_idx[k]] == 1 ? 1.0 : 0.0;
      acc += d->col_indicator[j] ? m : m * d->vals[k];
    }
    fixed[j] = acc;
  }
}

int orc_init(const orc_data* d, orc_state* s) {
  if (s->recompute_interval < 1) return ORC_DOMAIN;
  if (!s->fine_gray && any_competing(d)) return ORC_DOMAIN; /* engine.cpp:110-112 */
  if (s->fine_gray) {
    const int rc = orc_ipcw(d, s->u, s->g);
    if (rc) return rc;
  }
  for (int64_t j = 0; j < d->p; ++j) s->beta[j] = 0.0;
  for (int64_t i = 0; i < d->n; ++i) { s->eta[i] = 0.0; s->e[i] = 1.0; }
  orc_fixed_terms(d, s->fixed);
  s->accepted = s->refreshes = 0;
  return ORC_OK;
}

/* Engine::load_beta (src/engine.cpp:120-154): column-order accumulation,
 * validate every row before committing anything. */
int orc_load_beta(const orc_data* d, orc_state* s, const double* beta) {
  for (int64_t j = 0; j < d->p; ++j)
    if (!isfinite(beta[j])) return ORC_DOMAIN;
  double* fresh = (double*)calloc((size_t)d->n + 1, sizeof(double));
  for (int64_t j = 0; j < d->p; ++j) {
    const double bj = beta[j];
    if (bj == 0.0) continue;
    for (int64_t k = d->col_ptr[j]; k < d->col_ptr[j + 1]; ++k) {
      const int32_t i = d->row_idx[k];
      fresh[i] += d->col_indicator[j] ? bj : bj * d->vals[k];
    }
  }
  for (int64_t i = 0; i < d->n; ++i)
    if (fabs(fresh[i]) > XBETA_BOUND) { free(fresh); return ORC_OVERFLOW; }
  memcpy(s->beta, beta, sizeof(double) * (size_t)d->p);
  for (int64_t i = 0; i < d->n; ++i) { s->eta[i] = fresh[i]; s->e[i] = exp(fresh[i]); }
  free(fresh);
  return ORC_OK;
}

/* Engine::update_xbeta_sparse (src/engine.cpp:162-218). */
int orc_update(const orc_data* d, orc_state* s, int64_t j, double delta) {
  if (j < 0 || j >= d->p) return ORC_INVALID_COLUMN;
  if (!isfinite(delta)) return ORC_DOMAIN;
  if (delta == 0.0) return ORC_OK;
  const int ind = d->col_indicator[j];
  for (int64_t k = d->col_ptr[j]; k < d->col_ptr[j + 1]; ++k) {
    const double x = ind ? 1.0 : d->vals[k];
    if (fabs(s->eta[d->row_idx[k]] + x * delta) > XBETA_BOUND) return ORC_OVERFLOW;
  }
  if (ind) {
    const double factor = exp(delta);
    for (int64_t k = d->col_ptr[j]; k < d->col_ptr[j + 1]; ++k) {
      const int32_t i = d->row_idx[k];
      s->eta[i] += delta;
      s->e[i] *= factor;
    }
  } else {
    for (int64_t k = d->col_ptr[j]; k < d->col_ptr[j + 1]; ++k) {
      const int32_t i = d->row_idx[k];
      s->eta[i] += d->vals[k] * delta;
      s->e[i] = exp(s->eta[i]);
    }
  }
  s->beta[j] += delta;
  if (++s->accepted % s->recompute_interval == 0) {
    double* b = (double*)malloc(sizeof(double) * (size_t)d->p);
    memcpy(b, s->beta, sizeof(double) * (size_t)d->p);
    const int rc = orc_load_beta(d, s, b);
    free(b);
    if (rc) return rc;
    ++s->refreshes;
  }
  return ORC_OK;
}

/* Serial fused scan -> block-end transform -> reduce for column j over one
 * stratum [s, e) (include/survscan/scan_kernels.hpp:74-214 with a single
 * chunk).  x_j is walked with a cursor like ColumnSource (src/engine.cpp:16-73). */
static int grad_hess_stratum(const orc_data* d, const orc_state* st, int64_t j,
                             int weighted, int64_t s, int64_t e, const double* cnt,
                             double* gsum, double* hsum) {
  const int64_t m = e - s;
  double* sa = NULL; double* sb = NULL; double* sc = NULL;
  const int ind = d->col_indicator[j];
  const int64_t kb = d->col_ptr[j], ke = d->col_ptr[j + 1];
  if (weighted) {
    /* inclusive u-weighted suffix of the lanes, right to left (:143-159);
     * slot m holds the (zero) suffix past the end */
    sa = (double*)calloc((size_t)m + 1, sizeof(double));
    sb = (double*)calloc((size_t)m + 1, sizeof(double));
    sc = (double*)calloc((size_t)m + 1, sizeof(double));
    double ra = 0.0, rb = 0.0, rc = 0.0;
    int64_t cur = ke;
    while (cur > kb && d->row_idx[cur - 1] >= e) --cur;
    for (int64_t k = e; k-- > s;) {
      const double ev = st->e[k];
      double x = 0.0;
      if (cur > kb && d->row_idx[cur - 1] == k) { --cur; x = ind ? 1.0 : d->vals[cur]; }
      const double ex = ev * x;
      const double uk = st->u[k];
      ra += uk * ev; rb += uk * ex; rc += uk * (ex * x);
      sa[k - s] = ra; sb[k - s] = rb; sc[k - s] = rc;
    }
  }
  int64_t cur = kb;
  while (cur < ke && d->row_idx[cur] < s) ++cur;
  double pa = 0.0, pb = 0.0, pc = 0.0, lg = 0.0, lh = 0.0;
  int bad = 0;
  for (int64_t k = s; k < e; ++k) {
    const double ev = st->e[k];
    double x = 0.0;
    if (cur < ke && d->row_idx[cur] == k) { x = ind ? 1.0 : d->vals[cur]; ++cur; }
    const double ex = ev * x;
    pa += ev; pb += ex; pc += ex * x;
    if (cnt[k] > 0.0) {
      double den = pa, n1 = pb, n2 = pc;
      if (weighted) {
        const double gk = st->g[k];
        den += gk * sa[k + 1 - s];
        n1 += gk * sb[k + 1 - s];
        n2 += gk * sc[k + 1 - s];
      }
      if (!(den > 0.0)) { bad = 1; }
      else {
        const double G = n1 / den, H = n2 / den;
        lg += cnt[k] * G;
        lh += cnt[k] * (H - G * G);
      }
    }
  }
  free(sa); free(sb); free(sc);
  *gsum += lg; *hsum += lh;
  return bad ? ORC_NONPOS_DEN : ORC_OK;
}

int orc_grad_hessian(const orc_data* d, const orc_state* st, int64_t j,
                     double* grad, double* hess, double* fixed_term,
                     double* grad_sum, double* hess_sum) {
  if (j < 0 || j >= d->p) return ORC_INVALID_COLUMN;
  const int weighted = st->fine_gray && any_competing(d); /* engine.cpp:237 */
  double* cnt = (double*)malloc(sizeof(double) * ((size_t)d->n + 1));
  orc_block_counts(d, cnt);
  double gs = 0.0, hs = 0.0;
  int rc = ORC_OK;
  for (int64_t s = 0; s < d->n;) {
    const int64_t e = stratum_end(d, s);
    const int r = grad_hess_stratum(d, st, j, weighted, s, e, cnt, &gs, &hs);
    if (r) rc = r;
    s = e;
  }
  free(cnt);
  if (rc) return rc;
  /* Engine::finish (src/engine.cpp:220-230) */
  double g = st->fixed[j] - gs;
  double h = -hs;
  if (h > 0.0) h = 0.0;
  if (!isfinite(g) || !isfinite(h)) return ORC_NONPOS_DEN;
  *grad = g; *hess = h; *fixed_term = st->fixed[j];
  if (grad_sum) *grad_sum = gs;
  if (hess_sum) *hess_sum = hs;
  return ORC_OK;
}

/* Engine::log_likelihood = masked_dot(delta, eta) - fused_log_denominator
 * (src/engine.cpp:331-341; src/scan.cpp:233-250, 275-367). */
int orc_log_likelihood(const orc_data* d, const orc_state* st, double* out) {
  const int weighted = st->fine_gray && any_competing(d);
  double* cnt = (double*)malloc(sizeof(double) * ((size_t)d->n + 1));
  orc_block_counts(d, cnt);
  double fixed = 0.0, logden = 0.0;
  int bad = 0;
  for (int64_t i = 0; i < d->n; ++i)
    fixed += (d->status[i] == 1 ? 1.0 : 0.0) * st->eta[i];
  for (int64_t s = 0; s < d->n;) {
    const int64_t e = stratum_end(d, s);
    double* ls = NULL;
    if (weighted) {
      ls = (double*)calloc((size_t)(e - s) + 1, sizeof(double));
      double run = 0.0;
      for (int64_t k = e; k-- > s;) { run += st->u[k] * st->e[k]; ls[k - s] = run; }
    }
    double run = 0.0, part = 0.0;
    for (int64_t k = s; k < e; ++k) {
      run += st->e[k];
      if (cnt[k] > 0.0) {
        double den = run;
        if (weighted) den += st->g[k] * ls[k + 1 - s];
        if (!(den > 0.0)) bad = 1;
        else part += cnt[k] * log(den);
      }
    }
    logden += part;
    free(ls);
    s = e;
  }
  free(cnt);
  if (bad) return ORC_NONPOS_DEN;
  *out = fixed - logden;
  return ORC_OK;
}

static double sgn(double x) { return x > 0.0 ? 1.0 : (x < 0.0 ? -1.0 : 0.0); }

/* coordinate_step (src/ccd.cpp:71-129). */
void orc_coordinate_step(double beta_j, double grad, double hess, int kind,
                         double strength, int penalized, double hw,
                         double* new_beta, double* applied, double* new_hw,
                         int* skipped) {
  double geff = grad, heff = hess;
  int at_zero_l1 = 0;
  if (penalized) {
    if (kind == 2) { geff -= beta_j / strength; heff -= 1.0 / strength; }
    else if (kind == 1) {
      if (beta_j != 0.0) geff -= strength * sgn(beta_j);
      else at_zero_l1 = 1;
    }
  }
  *new_beta = beta_j; *applied = 0.0; *new_hw = hw; *skipped = 0;
  if (at_zero_l1) {
    if (fabs(geff) <= strength) { *new_hw = fmax(hw / 2.0, HW_FLOOR); return; }
    geff -= strength * sgn(geff);
  }
  if (!(heff < 0.0)) {
    if (geff != 0.0) { *skipped = 1; return; }
    *new_hw = fmax(hw / 2.0, HW_FLOOR);
    return;
  }
  double raw = -geff / heff;
  if (penalized && kind == 1 && beta_j != 0.0 && sgn(beta_j + raw) != sgn(beta_j))
    raw = -beta_j;
  const double a = sgn(raw) * fmin(fabs(raw), hw);
  *applied = a;
  *new_beta = beta_j + a;
  *new_hw = fmax(fmax(2.0 * fabs(a), hw / 2.0), HW_FLOOR);
}

static double penalty_value(const orc_data* d, const double* beta, int kind,
                            double strength, const uint8_t* exempt) {
  if (kind == 0) return 0.0;
  double acc = 0.0;
  for (int64_t j = 0; j < d->p; ++j) {
    if (exempt && exempt[j]) continue;
    acc += kind == 1 ? strength * fabs(beta[j]) : beta[j] * beta[j] / (2.0 * strength);
  }
  return acc;
}

/* fit_with_engine (src/ccd.cpp:131-184). */
int orc_fit(const orc_data* d, orc_state* s, int kind, double strength,
            const uint8_t* exempt, double tol, int64_t max_cycles,
            double trust_init, double* trace, orc_fit_result* out) {
  const int64_t p = d->p;
  double* zero = (double*)calloc((size_t)p + 1, sizeof(double));
  int rc = orc_load_beta(d, s, zero);
  free(zero);
  if (rc) return rc;
  double* hw = (double*)malloc(sizeof(double) * ((size_t)p + 1));
  for (int64_t j = 0; j < p; ++j) hw[j] = trust_init;
  memset(out, 0, sizeof(*out));
  double ll;
  rc = orc_log_likelihood(d, s, &ll);
  if (rc) { free(hw); return rc; }
  double prev = ll - penalty_value(d, s->beta, kind, strength, exempt);
  trace[0] = prev;
  int converged = p == 0;
  int64_t cycle;
  for (cycle = 1; !converged && cycle <= max_cycles; ++cycle) {
    for (int64_t j = 0; j < p; ++j) {
      double g, h, f;
      rc = orc_grad_hessian(d, s, j, &g, &h, &f, NULL, NULL);
      if (rc) { free(hw); return rc; }
      const int pen = kind != 0 && !(exempt && exempt[j]);
      double nb, a, nh; int sk;
      orc_coordinate_step(s->beta[j], g, h, kind, strength, pen, hw[j], &nb, &a, &nh, &sk);
      if (sk) { ++out->skipped; continue; }
      if (a != 0.0) {
        rc = orc_update(d, s, j, a);
        if (rc) { free(hw); return rc; }
      }
      hw[j] = nh;
    }
    out->cycles = cycle;
    rc = orc_log_likelihood(d, s, &ll);
    if (rc) { free(hw); return rc; }
    const double obj = ll - penalty_value(d, s->beta, kind, strength, exempt);
    trace[cycle] = obj;
    if (obj < prev - 1e-10) ++out->violations;
    if (fabs(obj - prev) / fmax(1.0, fabs(obj)) < tol) converged = 1;
    prev = obj;
  }
  out->converged = converged;
  out->objective = prev;
  for (int64_t j = 0; j < p; ++j) out->nonzero += s->beta[j] != 0.0;
  free(hw);
  return ORC_OK;
}
