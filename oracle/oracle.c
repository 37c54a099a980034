/*
 * oracle.c -- plain, slow, obviously-correct fp64 CPU oracle of FastDOG's
 * Alg. "Parallel Deferred Min-Marginal Averaging" (arXiv 2111.10270,
 * P:620-656) with the BDD min-marginal passes of P:307-342.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Shares no code with the product.
 *
 * Structure follows the paper's order and notation:
 *   - compile_row():  constraint row -> weighted BDD (Def. BDD P:241-257,
 *     canonical form P:273-277; readings A12).  Compiler "A": enumerate the
 *     partial sums sum_{t<h} a_t x_t top-down, keep states that can still
 *     be completed, then merge equal (s0, s1) signatures bottom-up.
 *   - oracle_create(): J_i, I_j, lambda init (P:622,
 *     original form A9), mbar = 0, shp(v,T) by a backward DP.
 *   - forward_pass()/backward_pass(): Alg. forward_pass_mm (with
 *     the arc cost lambda_{i-1} of the weighted BDD P:292-296, reading A4)
 *     and Alg. backward_pass_mm; min-marginals by Eq.
 *     (min-marginal-via-shortest-path) P:310-313; dual update P:641 (A1, A16).
 *   - deferred swap mbar <- m after every pass (A2).
 *   - lower bound: lifted bound of A7 = sum_j E^j(lambda^j) +
 *     sum_slots min(delta_bar, 0) + sum_free min(c_i, 0).
 *   - finalize: P:650-652 (per-slot, A11).
 *
 * No blocking, fusion or reordering: per BDD, per hop, per node, literally.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define O_OK 0
#define O_EINVAL 1
#define O_EINFEASIBLE 2
#define O_ENOMEM 3
#define O_ESTATE 6

#define BOT (-1)
#define TOP (-2)

typedef struct {
  int32_t k;          /* |I_j|                                     */
  int32_t n_nodes;    /* non-terminal nodes                        */
  int32_t *vars;      /* I_j ascending (global indices)            */
  int32_t *hop_start; /* k+1: P_h = nodes [hop_start[h], hop_start[h+1]) */
  int32_t *lo, *hi;   /* s^0(v), s^1(v): node index, BOT or TOP    */
  double *cfr;        /* shp(r, v)                                 */
  double *ctt;        /* shp(v, T)                                 */
  int64_t slot0;      /* first canonical slot of this BDD          */
} obdd;

struct oracle_solver {
  int32_t n_vars, n_cons;
  double *cost;
  double clamp;
  int n_threads;
  obdd *bdd;
  int64_t n_slots;
  int32_t *slot_var;   /* i of slot (j, h)                         */
  int32_t *slot_bdd;   /* j of slot (j, h)                         */
  double *lambda;      /* lambda_i^j per slot                      */
  double *delta_bar;   /* omega * d of the last pass (deferred)    */
  double *delta_new;   /* this pass                                */
  double *m0, *m1;     /* min-marginals recorded in the last pass  */
  /* J_i as CSR over slots, j ascending (A1: sum over k in J_i). */
  int64_t *var_ptr;
  int64_t *var_slots;
  double *avg;         /* (1/|J_i|) sum_k delta_bar_ik           */
  double *energy;      /* E^j per BDD (scratch for the bound)      */
  double free_term;    /* sum over free variables of min(c_i, 0) (A13) */
  double lb;
  int passes;
  /* which stored distances are valid for the current lambda: the incremental
   * reuse of P:315-316 holds when forward and backward passes alternate; any
   * other sequence recomputes them from their definition */
  int ctt_ok, cfr_ok;
  /* lifted representation (oracle_set_lifted): lambda holds
   * lambda^{j,1}, lam0 holds lambda^{j,0} (the 0-arc costs) */
  int lifted;
  double *lam0;
  double *avg0;        /* (1/|J_i|) sum_k max(-delta_bar_ik, 0)     */
};

/* ------------------------------------------------------------------ */
/* small growable int64 array                                          */
typedef struct {
  int64_t *v;
  int64_t n, cap;
} vec64;

static int vec_push(vec64 *a, int64_t x) {
  if (a->n == a->cap) {
    int64_t nc = a->cap ? 2 * a->cap : 16;
    int64_t *nv = (int64_t *)realloc(a->v, (size_t)nc * sizeof(int64_t));
    if (!nv) return 0;
    a->v = nv;
    a->cap = nc;
  }
  a->v[a->n++] = x;
  return 1;
}

static int cmp64(const void *a, const void *b) {
  int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
  return (x > y) - (x < y);
}

/* index of x in sorted array, or -1 */
static int64_t find64(const int64_t *a, int64_t n, int64_t x) {
  int64_t lo = 0, hi = n - 1;
  while (lo <= hi) {
    int64_t mid = (lo + hi) / 2;
    if (a[mid] == x) return mid;
    if (a[mid] < x) lo = mid + 1; else hi = mid - 1;
  }
  return -1;
}

static int row_sat(int64_t s, int rel, int64_t b) {
  if (rel < 0) return s <= b;
  if (rel > 0) return s >= b;
  return s == b;
}

/* Could partial sum s at level h still be completed to a satisfying
 * assignment?  Necessary condition only (sound pruning of states that are
 * certainly dead); exact deadness is decided bottom-up below. */
static int may_complete(int64_t s, int rel, int64_t b, int64_t sufmin, int64_t sufmax) {
  if (rel < 0) return s + sufmin <= b;
  if (rel > 0) return s + sufmax >= b;
  return s + sufmin <= b && s + sufmax >= b;
}

/* Compile row (a_0..a_{k-1}) rel b into a quasi-reduced ordered BDD.
 * Returns O_OK, O_EINFEASIBLE (empty X_j) or O_ENOMEM. */
static int compile_row(int32_t k, const int32_t *coef, int rel, int64_t b, obdd *out) {
  int rc = O_ENOMEM;
  int64_t *sufmin = (int64_t *)calloc((size_t)k + 1, sizeof(int64_t));
  int64_t *sufmax = (int64_t *)calloc((size_t)k + 1, sizeof(int64_t));
  vec64 *lev = (vec64 *)calloc((size_t)k + 1, sizeof(vec64));  /* states per level */
  int32_t **cls = (int32_t **)calloc((size_t)k + 1, sizeof(int32_t *)); /* state -> class */
  int32_t *ncls = (int32_t *)calloc((size_t)k + 1, sizeof(int32_t));
  int32_t **cls_lo = (int32_t **)calloc((size_t)k + 1, sizeof(int32_t *));
  int32_t **cls_hi = (int32_t **)calloc((size_t)k + 1, sizeof(int32_t *));
  if (!sufmin || !sufmax || !lev || !cls || !ncls || !cls_lo || !cls_hi) goto done;
  for (int32_t h = k - 1; h >= 0; --h) {
    sufmin[h] = sufmin[h + 1] + (coef[h] < 0 ? coef[h] : 0);
    sufmax[h] = sufmax[h + 1] + (coef[h] > 0 ? coef[h] : 0);
  }
  /* top-down: reachable partial sums */
  if (!may_complete(0, rel, b, sufmin[0], sufmax[0])) { rc = O_EINFEASIBLE; goto done; }
  if (!vec_push(&lev[0], 0)) goto done;
  for (int32_t h = 0; h < k; ++h) {
    vec64 *nx = &lev[h + 1];
    for (int64_t t = 0; t < lev[h].n; ++t) {
      int64_t s = lev[h].v[t];
      if (may_complete(s, rel, b, sufmin[h + 1], sufmax[h + 1]) && !vec_push(nx, s)) goto done;
      int64_t s1 = s + coef[h];
      if (may_complete(s1, rel, b, sufmin[h + 1], sufmax[h + 1]) && !vec_push(nx, s1)) goto done;
    }
    if (nx->n) {
      qsort(nx->v, (size_t)nx->n, sizeof(int64_t), cmp64);
      int64_t u = 1;
      for (int64_t t = 1; t < nx->n; ++t)
        if (nx->v[t] != nx->v[u - 1]) nx->v[u++] = nx->v[t];
      nx->n = u;
    }
  }
  /* bottom-up: class of every state = merged (s0, s1) signature; dead -> BOT */
  for (int32_t h = k - 1; h >= 0; --h) {
    int64_t n = lev[h].n;
    cls[h] = (int32_t *)malloc((size_t)(n ? n : 1) * sizeof(int32_t));
    cls_lo[h] = (int32_t *)malloc((size_t)(n ? n : 1) * sizeof(int32_t));
    cls_hi[h] = (int32_t *)malloc((size_t)(n ? n : 1) * sizeof(int32_t));
    if (!cls[h] || !cls_lo[h] || !cls_hi[h]) goto done;
    ncls[h] = 0;
    for (int64_t t = 0; t < n; ++t) {
      int64_t s = lev[h].v[t];
      int32_t c0, c1;
      if (h == k - 1) {
        c0 = row_sat(s, rel, b) ? TOP : BOT;
        c1 = row_sat(s + coef[h], rel, b) ? TOP : BOT;
      } else {
        int64_t i0 = find64(lev[h + 1].v, lev[h + 1].n, s);
        int64_t i1 = find64(lev[h + 1].v, lev[h + 1].n, s + coef[h]);
        c0 = i0 < 0 ? BOT : cls[h + 1][i0];
        c1 = i1 < 0 ? BOT : cls[h + 1][i1];
      }
      if (c0 == BOT && c1 == BOT) { cls[h][t] = BOT; continue; }
      int32_t c = -1;
      for (int32_t q = 0; q < ncls[h]; ++q)
        if (cls_lo[h][q] == c0 && cls_hi[h][q] == c1) { c = q; break; }
      if (c < 0) {
        c = ncls[h]++;
        cls_lo[h][c] = c0;
        cls_hi[h][c] = c1;
      }
      cls[h][t] = c;
    }
  }
  if (k == 0 || cls[0][0] == BOT) { rc = O_EINFEASIBLE; goto done; }
  /* Every class is reachable from the root (its state was generated
   * top-down from a live parent), so the classes are the nodes.  Lay the
   * partitions out contiguously, P_1 first. */
  {
    int32_t total = 0;
    out->k = k;
    out->hop_start = (int32_t *)malloc(((size_t)k + 1) * sizeof(int32_t));
    if (!out->hop_start) goto done;
    for (int32_t h = 0; h < k; ++h) { out->hop_start[h] = total; total += ncls[h]; }
    out->hop_start[k] = total;
    out->n_nodes = total;
    out->lo = (int32_t *)malloc((size_t)total * sizeof(int32_t));
    out->hi = (int32_t *)malloc((size_t)total * sizeof(int32_t));
    out->cfr = (double *)malloc((size_t)total * sizeof(double));
    out->ctt = (double *)malloc((size_t)total * sizeof(double));
    if (!out->lo || !out->hi || !out->cfr || !out->ctt) goto done;
    for (int32_t h = 0; h < k; ++h)
      for (int32_t q = 0; q < ncls[h]; ++q) {
        int32_t v = out->hop_start[h] + q;
        int32_t c0 = cls_lo[h][q], c1 = cls_hi[h][q];
        out->lo[v] = (c0 >= 0) ? out->hop_start[h + 1] + c0 : c0;
        out->hi[v] = (c1 >= 0) ? out->hop_start[h + 1] + c1 : c1;
      }
    rc = O_OK;
  }
done:
  for (int32_t h = 0; h <= k; ++h) {
    if (lev) free(lev[h].v);
    if (cls) free(cls[h]);
    if (cls_lo) free(cls_lo[h]);
    if (cls_hi) free(cls_hi[h]);
  }
  free(sufmin); free(sufmax); free(lev); free(cls); free(ncls); free(cls_lo); free(cls_hi);
  return rc;
}

/* ------------------------------------------------------------------ */
/* Weighted-BDD shortest paths                             */

/* shp(w, T) of a successor code w: T -> 0, bottom -> +inf */
static double ctt_of(const obdd *d, int32_t w) {
  if (w == TOP) return 0.0;
  if (w == BOT) return INFINITY;
  return d->ctt[w];
}

/* Backward DP over all partitions with the current lambda, no updates:
 * shp(v,T) = min{shp(s0 v, T), shp(s1 v, T) + lambda_h}. */
static void backward_dp(obdd *d, const double *lam) {
  for (int32_t h = d->k - 1; h >= 0; --h)
    for (int32_t v = d->hop_start[h]; v < d->hop_start[h + 1]; ++v) {
      double a = ctt_of(d, d->lo[v]);
      double b = lam[h] + ctt_of(d, d->hi[v]);
      d->ctt[v] = a < b ? a : b;
    }
}

/* Forward DP over all partitions with the current lambda, no updates:
 * shp(r,v) = min over parents (arc cost lambda_{h-1}, A4). */
static void forward_dp(obdd *d, const double *lam) {
  if (d->k == 0) return;
  d->cfr[0] = 0.0;
  for (int32_t h = 1; h < d->k; ++h)
    for (int32_t v = d->hop_start[h]; v < d->hop_start[h + 1]; ++v) {
      double best = INFINITY;
      for (int32_t u = d->hop_start[h - 1]; u < d->hop_start[h]; ++u) {
        if (d->lo[u] == v && d->cfr[u] < best) best = d->cfr[u];
        if (d->hi[u] == v && d->cfr[u] + lam[h - 1] < best) best = d->cfr[u] + lam[h - 1];
      }
      d->cfr[v] = best;
    }
}

/* E^j(lambda^j) = min_{x in X_j} x^T lambda^j = shp(r, T). */
static double energy_of(const obdd *d, const double *lam) {
  /* fresh DP into a temporary so the stored distances are untouched */
  double *t = (double *)malloc((size_t)(d->n_nodes ? d->n_nodes : 1) * sizeof(double));
  if (!t) return NAN;
  for (int32_t h = d->k - 1; h >= 0; --h)
    for (int32_t v = d->hop_start[h]; v < d->hop_start[h + 1]; ++v) {
      double a = d->lo[v] == TOP ? 0.0 : d->lo[v] == BOT ? INFINITY : t[d->lo[v]];
      double b = lam[h] + (d->hi[v] == TOP ? 0.0 : d->hi[v] == BOT ? INFINITY : t[d->hi[v]]);
      t[v] = a < b ? a : b;
    }
  double e = t[0];
  free(t);
  return e;
}

/* Eq. (min-marginal-via-shortest-path) P:312 for hop h, using the stored
 * shp(r, v) of P_h and shp(s^beta(v), T). */
static void min_marginals_at(const obdd *d, const double *lam, int32_t h, double *m0, double *m1) {
  double b0 = INFINITY, b1 = INFINITY;
  for (int32_t v = d->hop_start[h]; v < d->hop_start[h + 1]; ++v) {
    if (d->lo[v] != BOT) {
      double x = d->cfr[v] + ctt_of(d, d->lo[v]);
      if (x < b0) b0 = x;
    }
    if (d->hi[v] != BOT) {
      double x = (d->cfr[v] + lam[h]) + ctt_of(d, d->hi[v]);
      if (x < b1) b1 = x;
    }
  }
  *m0 = b0;
  *m1 = b1;
}

/* d = m1 - m0, with an infinite side replaced by the clamp (A5). */
static double mm_difference(double m1, double m0, double clamp) {
  if (isinf(m1) && isinf(m0)) return 0.0; /* impossible for X_j != {} */
  if (isinf(m1)) return clamp;
  if (isinf(m0)) return -clamp;
  return m1 - m0;
}

/* Dual update P:641 (A1/A16): lambda <- lambda - omega*(m1-m0) + avg_i,
 * avg_i = (omega/|J_i|) sum_k (mbar1_ik - mbar0_ik) = mean of delta_bar. */
static void update_slot(oracle_solver *s, int64_t slot, double *lam_h, double m0, double m1,
                        double omega) {
  double d = mm_difference(m1, m0, s->clamp);
  s->m0[slot] = m0;
  s->m1[slot] = m1;
  *lam_h = *lam_h - omega * d + s->avg[s->slot_var[slot]];
  s->delta_new[slot] = omega * d;
}

/* Forward pass with Alg. forward_pass_mm. */
static void forward_pass(oracle_solver *s, obdd *d, double omega) {
  double *lam = s->lambda + d->slot0;
  for (int32_t h = 0; h < d->k; ++h) {
    if (h == 0) {
      d->cfr[0] = 0.0; /* shp(r, r) */
    } else {
      /* for v in P_h: shp(r,v) = min{ min_{u: s0(u)=v} shp(r,u),
       *                               min_{u: s1(u)=v} shp(r,u) + lambda_{h-1} } (A4) */
      for (int32_t v = d->hop_start[h]; v < d->hop_start[h + 1]; ++v) {
        double best = INFINITY;
        for (int32_t u = d->hop_start[h - 1]; u < d->hop_start[h]; ++u) {
          if (d->lo[u] == v && d->cfr[u] < best) best = d->cfr[u];
          if (d->hi[u] == v && d->cfr[u] + lam[h - 1] < best) best = d->cfr[u] + lam[h - 1];
        }
        d->cfr[v] = best;
      }
    }
    double m0, m1;
    min_marginals_at(d, lam, h, &m0, &m1);
    update_slot(s, d->slot0 + h, &lam[h], m0, m1, omega);
  }
}

/* Backward pass with Alg. backward_pass_mm. */
static void backward_pass(oracle_solver *s, obdd *d, double omega) {
  double *lam = s->lambda + d->slot0;
  for (int32_t h = d->k - 1; h >= 0; --h) {
    /* shp(v, T) for v in P_{h+1} was recomputed in the previous step with
     * the updated lambda_{h+1}; for h = k-1 the successors are terminals. */
    double m0, m1;
    min_marginals_at(d, lam, h, &m0, &m1);
    update_slot(s, d->slot0 + h, &lam[h], m0, m1, omega);
    for (int32_t v = d->hop_start[h]; v < d->hop_start[h + 1]; ++v) {
      double a = ctt_of(d, d->lo[v]);
      double b = lam[h] + ctt_of(d, d->hi[v]);
      d->ctt[v] = a < b ? a : b;
    }
  }
}

/* sum_j E^j + free term (raw dual energy at the current lambda) */
static double raw_energy(const oracle_solver *s) {
  const int32_t m = s->n_cons;
  int j;
#pragma omp parallel for num_threads(s->n_threads) schedule(dynamic, 256)
  for (j = 0; j < m; ++j) s->energy[j] = energy_of(&s->bdd[j], s->lambda + s->bdd[j].slot0);
  double e = 0.0;
  for (int32_t q = 0; q < m; ++q) e += s->energy[q]; /* fixed order */
  return e + s->free_term;
}

/* ------------------------------------------------------------------ */

static void free_solver(oracle_solver *s) {
  if (!s) return;
  if (s->bdd) {
    for (int32_t j = 0; j < s->n_cons; ++j) {
      free(s->bdd[j].vars); free(s->bdd[j].hop_start); free(s->bdd[j].lo); free(s->bdd[j].hi);
      free(s->bdd[j].cfr); free(s->bdd[j].ctt);
    }
  }
  free(s->bdd); free(s->cost); free(s->slot_var); free(s->slot_bdd); free(s->lambda); free(s->delta_bar);
  free(s->delta_new); free(s->m0); free(s->m1); free(s->var_ptr); free(s->var_slots);
  free(s->avg); free(s->energy); free(s->lam0); free(s->avg0);
  free(s);
}

int oracle_create(const oracle_problem *p, double clamp, int n_threads, oracle_solver **out) {
  if (!p || !out || p->n_vars < 0 || p->n_cons < 0) return O_EINVAL;
  if (p->n_vars > 0 && !p->cost) return O_EINVAL;
  if (p->n_cons > 0 && (!p->row_ptr || !p->rel || !p->rhs)) return O_EINVAL;
  *out = NULL;
  oracle_solver *s = (oracle_solver *)calloc(1, sizeof(oracle_solver));
  if (!s) return O_ENOMEM;
  s->n_vars = p->n_vars;
  s->n_cons = p->n_cons;
  s->clamp = clamp;
#ifdef _OPENMP
  s->n_threads = n_threads > 0 ? n_threads : omp_get_max_threads();
#else
  s->n_threads = 1;
#endif
  int rc = O_ENOMEM;
  s->cost = (double *)malloc((size_t)(p->n_vars ? p->n_vars : 1) * sizeof(double));
  s->bdd = (obdd *)calloc((size_t)(p->n_cons ? p->n_cons : 1), sizeof(obdd));
  s->energy = (double *)calloc((size_t)(p->n_cons ? p->n_cons : 1), sizeof(double));
  if (!s->cost || !s->bdd || !s->energy) goto fail;
  if (p->n_vars) memcpy(s->cost, p->cost, (size_t)p->n_vars * sizeof(double));
  /* validate rows: ascending variables, nonzero coefficients */
  for (int32_t j = 0; j < p->n_cons; ++j) {
    int64_t a = p->row_ptr[j], b = p->row_ptr[j + 1];
    if (b < a || b - a > 0x7fffffff) { rc = O_EINVAL; goto fail; }
    if (p->rel[j] < -1 || p->rel[j] > 1) { rc = O_EINVAL; goto fail; }
    for (int64_t q = a; q < b; ++q) {
      if (p->col_var[q] < 0 || p->col_var[q] >= p->n_vars || p->col_coef[q] == 0) { rc = O_EINVAL; goto fail; }
      if (q > a && p->col_var[q] <= p->col_var[q - 1]) { rc = O_EINVAL; goto fail; }
    }
  }
  /* compile each row (rows with no variables: I_j empty, drop unless infeasible) */
  {
    int bad = O_OK;
    int j;
#pragma omp parallel for num_threads(s->n_threads) schedule(dynamic, 64)
    for (j = 0; j < p->n_cons; ++j) {
      int64_t a = p->row_ptr[j];
      int32_t k = (int32_t)(p->row_ptr[j + 1] - a);
      obdd *d = &s->bdd[j];
      if (k == 0) {
        if (!row_sat(0, p->rel[j], p->rhs[j])) {
#pragma omp critical
          bad = O_EINFEASIBLE;
        }
        continue;
      }
      int r = compile_row(k, p->col_coef + a, p->rel[j], p->rhs[j], d);
      if (r == O_OK) {
        d->vars = (int32_t *)malloc((size_t)k * sizeof(int32_t));
        if (!d->vars) r = O_ENOMEM;
        else memcpy(d->vars, p->col_var + a, (size_t)k * sizeof(int32_t));
      }
      if (r != O_OK) {
#pragma omp critical
        bad = r;
      }
    }
    if (bad != O_OK) { rc = bad; goto fail; }
  }
  /* slots (j asc, h asc), J_i CSR with j ascending, |J_i| */
  s->n_slots = 0;
  for (int32_t j = 0; j < p->n_cons; ++j) { s->bdd[j].slot0 = s->n_slots; s->n_slots += s->bdd[j].k; }
  {
    int64_t S = s->n_slots ? s->n_slots : 1;
    s->slot_var = (int32_t *)malloc((size_t)S * sizeof(int32_t));
    s->slot_bdd = (int32_t *)malloc((size_t)S * sizeof(int32_t));
    s->lambda = (double *)malloc((size_t)S * sizeof(double));
    s->delta_bar = (double *)calloc((size_t)S, sizeof(double));
    s->delta_new = (double *)calloc((size_t)S, sizeof(double));
    s->m0 = (double *)calloc((size_t)S, sizeof(double));
    s->m1 = (double *)calloc((size_t)S, sizeof(double));
    s->var_ptr = (int64_t *)calloc((size_t)p->n_vars + 1, sizeof(int64_t));
    s->var_slots = (int64_t *)malloc((size_t)S * sizeof(int64_t));
    s->avg = (double *)calloc((size_t)(p->n_vars ? p->n_vars : 1), sizeof(double));
    if (!s->slot_var || !s->slot_bdd || !s->lambda || !s->delta_bar || !s->delta_new || !s->m0 || !s->m1 ||
        !s->var_ptr || !s->var_slots || !s->avg)
      goto fail;
  }
  for (int32_t j = 0; j < p->n_cons; ++j)
    for (int32_t h = 0; h < s->bdd[j].k; ++h) {
      int32_t i = s->bdd[j].vars[h];
      s->slot_var[s->bdd[j].slot0 + h] = i;
      s->slot_bdd[s->bdd[j].slot0 + h] = j;
      s->var_ptr[i + 1]++;
    }
  for (int32_t i = 0; i < p->n_vars; ++i) s->var_ptr[i + 1] += s->var_ptr[i];
  {
    int64_t *fill = (int64_t *)calloc((size_t)(p->n_vars ? p->n_vars : 1), sizeof(int64_t));
    if (!fill) goto fail;
    for (int32_t j = 0; j < p->n_cons; ++j) /* j ascending -> J_i ascending */
      for (int32_t h = 0; h < s->bdd[j].k; ++h) {
        int32_t i = s->bdd[j].vars[h];
        s->var_slots[s->var_ptr[i] + fill[i]++] = s->bdd[j].slot0 + h;
      }
    free(fill);
  }
  /* lambda_i^j = c_i / |J_i| (P:622 via A9); free variables add min(c_i,0) (A13) */
  s->free_term = 0.0;
  for (int32_t i = 0; i < p->n_vars; ++i) {
    int64_t deg = s->var_ptr[i + 1] - s->var_ptr[i];
    if (deg == 0) { s->free_term += s->cost[i] < 0 ? s->cost[i] : 0.0; continue; }
    for (int64_t q = s->var_ptr[i]; q < s->var_ptr[i + 1]; ++q)
      s->lambda[s->var_slots[q]] = s->cost[i] / (double)deg;
  }
  /* shp(v, T) under the initial lambda, so the first forward pass can use it;
   * shp(r, v) too, for a caller that starts with a backward pass */
  for (int32_t j = 0; j < p->n_cons; ++j) {
    backward_dp(&s->bdd[j], s->lambda + s->bdd[j].slot0);
    forward_dp(&s->bdd[j], s->lambda + s->bdd[j].slot0);
  }
  s->lb = raw_energy(s);
  s->passes = 0;
  s->ctt_ok = s->cfr_ok = 1;
  *out = s;
  return O_OK;
fail:
  free_solver(s);
  return rc;
}

void oracle_destroy(oracle_solver *s) { free_solver(s); }

static int lifted_pass(oracle_solver *s, int forward, double omega);
static double lifted_bound(const oracle_solver *s);

int oracle_pass(oracle_solver *s, int forward, double omega) {
  if (!s) return O_EINVAL;
  if (!(omega > 0.0 && omega <= 1.0)) return O_EINVAL; /* A14 */
  if (s->lifted) return lifted_pass(s, forward, omega);
  /* deferred averaging from the previous pass's delta_bar (A1, A2) */
  for (int32_t i = 0; i < s->n_vars; ++i) {
    int64_t deg = s->var_ptr[i + 1] - s->var_ptr[i];
    if (deg == 0) { s->avg[i] = 0.0; continue; }
    double sum = 0.0;
    for (int64_t q = s->var_ptr[i]; q < s->var_ptr[i + 1]; ++q) sum += s->delta_bar[s->var_slots[q]];
    s->avg[i] = sum / (double)deg;
  }
  /* stored distances of the opposite direction must match the current lambda */
  if (forward && !s->ctt_ok)
    for (int32_t q = 0; q < s->n_cons; ++q) backward_dp(&s->bdd[q], s->lambda + s->bdd[q].slot0);
  if (!forward && !s->cfr_ok)
    for (int32_t q = 0; q < s->n_cons; ++q) forward_dp(&s->bdd[q], s->lambda + s->bdd[q].slot0);
  /* for j in J in parallel */
  int j;
#pragma omp parallel for num_threads(s->n_threads) schedule(dynamic, 256)
  for (j = 0; j < s->n_cons; ++j) {
    if (s->bdd[j].k == 0) continue;
    if (forward) forward_pass(s, &s->bdd[j], omega);
    else backward_pass(s, &s->bdd[j], omega);
  }
  /* mbar <- m */
  double *t = s->delta_bar;
  s->delta_bar = s->delta_new;
  s->delta_new = t;
  /* lifted lower bound (A7) */
  double e = raw_energy(s);
  double neg = 0.0;
  for (int64_t q = 0; q < s->n_slots; ++q) neg += s->delta_bar[q] < 0 ? s->delta_bar[q] : 0.0;
  s->lb = e + neg;
  s->passes++;
  s->ctt_ok = !forward; /* a forward pass leaves shp(r,v) valid, a backward pass shp(v,T) */
  s->cfr_ok = forward;
  return O_OK;
}

/* ------------------------------------------------------------------ */
/* Non-deferred min-marginal averaging ("If mbar <- m, then    */
/* (dual_update) matches the update from [lange2021efficient]"; the      */
/* sequential scheme the deferral replaces).                  */
/*                                                                       */
/* Variables are visited one at a time, in ascending (forward) or        */
/* descending (backward) global index.  At variable i every subproblem   */
/* j in J_i computes m_ij at its current lambda^j (via P:312),    */
/* then all of them update at once:                                      */
/*   lambda_i^j <- lambda_i^j - omega d_ij + (1/|J_i|) sum_k omega d_ik   */
/* (the update of Alg. parallel-mma line 'lambda-update' with mbar = m;  */
/* d = clamp(m1 - m0), A5).  Each BDD orders its variables ascending     */
/* (A12), so BDD j reaches hop h exactly when variable I_j[h] is visited */
/* and the incremental shortest paths of P:315-342 apply unchanged.      */
/* sum_j lambda_i^j = c_i after every variable, so no deferred term       */
/* remains (delta_bar = 0) and sum_j E^j is the bound.                   */
int oracle_pass_seq(oracle_solver *s, int forward, double omega) {
  if (!s) return O_EINVAL;
  if (s->lifted) return O_ESTATE;
  if (!(omega > 0.0 && omega <= 1.0)) return O_EINVAL; /* A14 */
  /* a pending deferred correction is not part of this scheme */
  for (int64_t q = 0; q < s->n_slots; ++q)
    if (s->delta_bar[q] != 0.0) return O_ESTATE;
  if (forward && !s->ctt_ok)
    for (int32_t q = 0; q < s->n_cons; ++q) backward_dp(&s->bdd[q], s->lambda + s->bdd[q].slot0);
  if (!forward && !s->cfr_ok)
    for (int32_t q = 0; q < s->n_cons; ++q) forward_dp(&s->bdd[q], s->lambda + s->bdd[q].slot0);
  double *dl = s->delta_new; /* omega * d_ij of the current variable's slots */
  for (int32_t t = 0; t < s->n_vars; ++t) {
    const int32_t i = forward ? t : s->n_vars - 1 - t;
    const int64_t q0 = s->var_ptr[i], q1 = s->var_ptr[i + 1];
    if (q0 == q1) continue;
    /* min-marginals of i in every j in J_i (ascending j) */
    for (int64_t q = q0; q < q1; ++q) {
      const int64_t slot = s->var_slots[q];
      obdd *d = &s->bdd[s->slot_bdd[slot]];
      double *lam = s->lambda + d->slot0;
      const int32_t h = (int32_t)(slot - d->slot0);
      if (forward) {
        if (h == 0) {
          d->cfr[0] = 0.0; /* shp(r, r) */
        } else {
          /* shp(r, v), v in P_h, from P_{h-1} with the updated lambda_{h-1} (A4) */
          for (int32_t v = d->hop_start[h]; v < d->hop_start[h + 1]; ++v) {
            double best = INFINITY;
            for (int32_t u = d->hop_start[h - 1]; u < d->hop_start[h]; ++u) {
              if (d->lo[u] == v && d->cfr[u] < best) best = d->cfr[u];
              if (d->hi[u] == v && d->cfr[u] + lam[h - 1] < best) best = d->cfr[u] + lam[h - 1];
            }
            d->cfr[v] = best;
          }
        }
      }
      double m0, m1;
      min_marginals_at(d, lam, h, &m0, &m1);
      s->m0[slot] = m0;
      s->m1[slot] = m1;
      dl[slot] = omega * mm_difference(m1, m0, s->clamp);
    }
    /* the averaging of the same min-marginals (j ascending, A1) */
    double sum = 0.0;
    for (int64_t q = q0; q < q1; ++q) sum += dl[s->var_slots[q]];
    const double avg = sum / (double)(q1 - q0);
    for (int64_t q = q0; q < q1; ++q) {
      const int64_t slot = s->var_slots[q];
      obdd *d = &s->bdd[s->slot_bdd[slot]];
      double *lam = s->lambda + d->slot0;
      const int32_t h = (int32_t)(slot - d->slot0);
      lam[h] = lam[h] - dl[slot] + avg;
      if (!forward) /* shp(v, T), v in P_h, with the updated lambda_h */
        for (int32_t v = d->hop_start[h]; v < d->hop_start[h + 1]; ++v) {
          double a = ctt_of(d, d->lo[v]);
          double b = lam[h] + ctt_of(d, d->hi[v]);
          d->ctt[v] = a < b ? a : b;
        }
    }
  }
  for (int64_t q = 0; q < s->n_slots; ++q) s->delta_bar[q] = 0.0;
  s->lb = raw_energy(s);
  s->passes++;
  s->ctt_ok = !forward;
  s->cfr_ok = forward;
  return O_OK;
}

int oracle_iterate_seq(oracle_solver *s, int n_iter, double omega) {
  if (!s || n_iter < 0) return O_EINVAL;
  for (int t = 0; t < n_iter; ++t) {
    int rc = oracle_pass_seq(s, 1, omega);
    if (rc) return rc;
    rc = oracle_pass_seq(s, 0, omega);
    if (rc) return rc;
  }
  return O_OK;
}

int oracle_iterate(oracle_solver *s, int n_iter, double omega) {
  if (!s || n_iter < 0) return O_EINVAL;
  for (int t = 0; t < n_iter; ++t) {
    int rc = oracle_pass(s, 1, omega);
    if (rc) return rc;
    rc = oracle_pass(s, 0, omega);
    if (rc) return rc;
  }
  return O_OK;
}

int oracle_lower_bound(const oracle_solver *s, double *out) {
  if (!s || !out) return O_EINVAL;
  *out = s->lb;
  return O_OK;
}

int oracle_dual_energy(const oracle_solver *s, double *out) {
  if (!s || !out) return O_EINVAL;
  if (s->lifted) return O_ESTATE;
  *out = raw_energy(s);
  return O_OK;
}

int oracle_finalize(oracle_solver *s) {
  if (!s) return O_EINVAL;
  if (s->lifted) {
    /* lambda^{j,b} += omega max(mbar^b - mbar^{1-b}, 0) (lifted form) */
    for (int64_t q = 0; q < s->n_slots; ++q) {
      const double x = s->delta_bar[q];
      s->lambda[q] += x > 0 ? x : 0.0;
      s->lam0[q] += x < 0 ? -x : 0.0;
      s->delta_bar[q] = 0.0;
    }
    s->lb = lifted_bound(s);
    return O_OK;
  }
  /* lambda_i^j += omega (mbar1_ij - mbar0_ij)  (per slot, A11) */
  for (int64_t q = 0; q < s->n_slots; ++q) {
    s->lambda[q] += s->delta_bar[q];
    s->delta_bar[q] = 0.0;
  }
  for (int32_t j = 0; j < s->n_cons; ++j) {
    backward_dp(&s->bdd[j], s->lambda + s->bdd[j].slot0);
    forward_dp(&s->bdd[j], s->lambda + s->bdd[j].slot0);
  }
  s->lb = raw_energy(s);
  s->ctt_ok = s->cfr_ok = 1;
  return O_OK;
}

/* Final correction read as "a min-marginal averaging step" (reading
 * A11 alternative): lambda_i^j += (1/|J_i|) sum_k delta_bar_ik, delta_bar = 0.
 * Dual feasible like the per-slot form: sum_j [lambda + avg] = c_i. */
int oracle_finalize_avg(oracle_solver *s) {
  if (!s) return O_EINVAL;
  if (s->lifted) return O_ESTATE;
  for (int32_t i = 0; i < s->n_vars; ++i) {
    int64_t deg = s->var_ptr[i + 1] - s->var_ptr[i];
    if (deg == 0) continue;
    double sum = 0.0;
    for (int64_t q = s->var_ptr[i]; q < s->var_ptr[i + 1]; ++q) sum += s->delta_bar[s->var_slots[q]];
    double avg = sum / (double)deg;
    for (int64_t q = s->var_ptr[i]; q < s->var_ptr[i + 1]; ++q) s->lambda[s->var_slots[q]] += avg;
  }
  for (int64_t q = 0; q < s->n_slots; ++q) s->delta_bar[q] = 0.0;
  for (int32_t j = 0; j < s->n_cons; ++j) {
    backward_dp(&s->bdd[j], s->lambda + s->bdd[j].slot0);
    forward_dp(&s->bdd[j], s->lambda + s->bdd[j].slot0);
  }
  s->lb = raw_energy(s);
  s->ctt_ok = s->cfr_ok = 1;
  return O_OK;
}

int oracle_num_slots(const oracle_solver *s, int64_t *out) {
  if (!s || !out) return O_EINVAL;
  *out = s->n_slots;
  return O_OK;
}

static int copy_out(const double *src, int64_t n, double *dst, int64_t len) {
  if (!dst || len < n) return O_EINVAL;
  if (n) memcpy(dst, src, (size_t)n * sizeof(double));
  return O_OK;
}

int oracle_get_lambda(const oracle_solver *s, double *out, int64_t len) {
  if (!s) return O_EINVAL;
  int rc = copy_out(s->lambda, s->n_slots, out, len);
  if (!rc && s->lifted) /* original space: lambda = lambda^1 - lambda^0 */
    for (int64_t q = 0; q < s->n_slots; ++q) out[q] -= s->lam0[q];
  return rc;
}

int oracle_get_deferred(const oracle_solver *s, double *out, int64_t len) {
  if (!s) return O_EINVAL;
  return copy_out(s->delta_bar, s->n_slots, out, len);
}

int oracle_min_marginals(const oracle_solver *s, double *m0, double *m1, int64_t len) {
  if (!s) return O_EINVAL;
  if (s->passes == 0) return O_ESTATE;
  int rc = copy_out(s->m0, s->n_slots, m0, len);
  return rc ? rc : copy_out(s->m1, s->n_slots, m1, len);
}

int oracle_set_lambda(oracle_solver *s, const double *lambda, int64_t len) {
  if (!s || !lambda || len != s->n_slots) return O_EINVAL;
  if (s->lifted) return O_ESTATE;
  memcpy(s->lambda, lambda, (size_t)len * sizeof(double));
  for (int32_t j = 0; j < s->n_cons; ++j) {
    backward_dp(&s->bdd[j], s->lambda + s->bdd[j].slot0);
    forward_dp(&s->bdd[j], s->lambda + s->bdd[j].slot0);
  }
  /* delta_bar is untouched: the lifted bound (A7) keeps its outstanding
   * sum_slots min(delta_bar, 0) term (zero when delta_bar = 0) */
  double neg = 0.0;
  for (int64_t q = 0; q < s->n_slots; ++q) neg += s->delta_bar[q] < 0 ? s->delta_bar[q] : 0.0;
  s->lb = raw_energy(s) + neg;
  s->ctt_ok = s->cfr_ok = 1;
  return O_OK;
}

int oracle_bdd_size(const oracle_solver *s, int32_t j, int32_t *k, int32_t *n_nodes) {
  if (!s || j < 0 || j >= s->n_cons || !k || !n_nodes) return O_EINVAL;
  *k = s->bdd[j].k;
  *n_nodes = s->bdd[j].n_nodes;
  return O_OK;
}

int oracle_bdd_get(const oracle_solver *s, int32_t j, int32_t *vars, int32_t *hop_start,
                   int32_t *lo, int32_t *hi) {
  if (!s || j < 0 || j >= s->n_cons) return O_EINVAL;
  const obdd *d = &s->bdd[j];
  if (d->k == 0) return O_OK;
  memcpy(vars, d->vars, (size_t)d->k * sizeof(int32_t));
  memcpy(hop_start, d->hop_start, ((size_t)d->k + 1) * sizeof(int32_t));
  memcpy(lo, d->lo, (size_t)d->n_nodes * sizeof(int32_t));
  memcpy(hi, d->hi, (size_t)d->n_nodes * sizeof(int32_t));
  return O_OK;
}

int oracle_total_nodes(const oracle_solver *s, int64_t *out) {
  if (!s || !out) return O_EINVAL;
  int64_t n = 0;
  for (int32_t j = 0; j < s->n_cons; ++j) n += s->bdd[j].n_nodes;
  *out = n;
  return O_OK;
}

int oracle_num_threads(const oracle_solver *s) { return s ? s->n_threads : 0; }

/* ------------------------------------------------------------------ */
/* Alg. "Perturbation Primal Rounding"                     */

/* Counter-based uniform in [0, 1): splitmix64 of (seed, round, i).  Both sides
 * (oracle and product) implement this same generator, so they draw the same r
 * (Alg. 2 "Sample r uniformly from [-delta, delta]"). */
static double primal_uniform(uint64_t seed, int64_t round, int64_t i) {
  uint64_t z = seed * 0x9E3779B97F4A7C15ull + (uint64_t)round * 0xBF58476D1CE4E5B9ull +
               (uint64_t)i * 0x94D049BB133111EBull + 1ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return (double)(z >> 11) * (1.0 / 9007199254740992.0);
}

/* sign of m1 - m0 with the clamp of A5 */
static int mm_sign(double m1, double m0, double clamp) {
  double d = mm_difference(m1, m0, clamp);
  return (d > 0) - (d < 0);
}

/* One classification + perturbation step of Alg. 2 over the min-marginals
 * recorded in the last pass.  Returns the number of undecided variables
 * (subproblems not all strictly favouring one value -- the loop guard, P:204,
 * read with P:193/P:197, reading R1); perturbs lambda only if that number is > 0.  x (length n_vars, may be NULL) receives the
 * labeling read off the signs: 1 if m1 < m0 in every subproblem, else 0;
 * free variables x_i = [c_i < 0]. */
int oracle_primal_step(oracle_solver *s, int32_t round, double delta, uint64_t seed, int64_t *conflicts,
                       uint8_t *x) {
  if (!s || !conflicts) return O_EINVAL;
  if (s->passes == 0 || s->lifted) return O_ESTATE;
  int64_t nc = 0;
  for (int32_t i = 0; i < s->n_vars; ++i) {
    int64_t a = s->var_ptr[i], b = s->var_ptr[i + 1];
    if (a == b) {
      if (x) x[i] = s->cost[i] < 0;
      continue;
    }
    int pos = 1, neg = 1, zero = 1;
    for (int64_t q = a; q < b; ++q) {
      int sg = mm_sign(s->m1[s->var_slots[q]], s->m0[s->var_slots[q]], s->clamp);
      pos &= sg > 0;
      neg &= sg < 0;
      zero &= sg == 0;
    }
    if (x) x[i] = (uint8_t)neg;
    /* undecided unless every subproblem strictly favours the same value:
     * P:193 "agree and favor a single variable", P:197 ties are perturbed
     * (reading R1); the literal guard of P:204 would stop on ties */
    (void)zero;
    if (!(pos || neg)) nc++;
  }
  *conflicts = nc;
  if (nc == 0) return O_OK;
  for (int32_t i = 0; i < s->n_vars; ++i) {
    int64_t a = s->var_ptr[i], b = s->var_ptr[i + 1];
    if (a == b) continue;
    int pos = 1, neg = 1, zero = 1;
    double dsum = 0.0; /* d_i = sum_j (m1_ij - m0_ij), clamped (A5) */
    for (int64_t q = a; q < b; ++q) {
      int64_t sl = s->var_slots[q];
      int sg = mm_sign(s->m1[sl], s->m0[sl], s->clamp);
      pos &= sg > 0;
      neg &= sg < 0;
      zero &= sg == 0;
      dsum += mm_difference(s->m1[sl], s->m0[sl], s->clamp);
    }
    double r = delta * (2.0 * primal_uniform(seed, round, i) - 1.0); /* r ~ U[-delta, delta] */
    double step;
    if (pos) step = delta;
    else if (neg) step = -delta;
    else if (zero) step = r * delta;
    else step = (double)((dsum > 0) - (dsum < 0)) * fabs(r) * delta;
    for (int64_t q = a; q < b; ++q) s->lambda[s->var_slots[q]] += step;
  }
  /* lambda changed: stored distances must be recomputed before the next pass */
  s->ctt_ok = s->cfr_ok = 0;
  return O_OK;
}

/* Alg. 2 driver: while some variable's min-marginals disagree in sign,
 * perturb (delta, then delta *= alpha) and reoptimise with `inner`
 * iterations of Alg. 1.  On success x holds the labeling, *rounds the
 * number of perturbation rounds; returns 7 if max_rounds is exhausted. */
int oracle_round_primal(oracle_solver *s, double delta0, double alpha, int32_t inner, int32_t max_rounds,
                        uint64_t seed, double omega, uint8_t *x, int32_t *rounds) {
  if (!s || !x || !rounds || !(delta0 > 0) || !(alpha >= 1) || inner < 1 || max_rounds < 0) return O_EINVAL;
  if (s->passes == 0) {
    int rc = oracle_iterate(s, inner, omega);
    if (rc) return rc;
  }
  double delta = delta0;
  for (int32_t round = 0;; ++round) {
    int64_t nc = 0;
    int rc = oracle_primal_step(s, round, delta, seed, &nc, x);
    if (rc) return rc;
    if (nc == 0) {
      *rounds = round;
      return O_OK;
    }
    if (round + 1 > max_rounds) {
      *rounds = round;
      return 7;
    }
    delta *= alpha;
    rc = oracle_iterate(s, inner, omega);
    if (rc) return rc;
  }
}

/* ------------------------------------------------------------------ */
/* Lifted representation: every BDD j keeps two costs per     */
/* variable, lambda^{j,0} on 0-arcs and lambda^{j,1} on 1-arcs, so      */
/* E^j = min over paths of sum_h lambda^{j, x_h}_h and the bound is the */
/* plain sum of per-BDD shortest paths (the appendix's lifted energy).  */
/* Initialisation lambda^{j,beta} = beta c_i / |J_i|.  Update,  */
/* reading A8 (P:53-56 with max(., 0)):                                 */
/*   lambda^{j,b} <- lambda^{j,b} - omega max(m^b - m^{1-b}, 0)         */
/*                  + (omega/|J_i|) sum_k max(mbar^b_ik - mbar^{1-b}_ik, 0) */
/* with m^1 - m^0 clamped as A5 (d = clamp(m1 - m0); omega max(d, 0) =  */
/* max(delta, 0) for delta = omega d, and omega max(-d, 0) =            */
/* max(-delta, 0)).  lambda^1 - lambda^0 follows the original-space      */
/* update P:641.  Each pass recomputes the opposite-direction  */
/* distances from their definition at its start, then walks */
/* the hops as Alg. forward_pass_mm / backward_pass_mm with */
/* the two arc costs.                                                   */

/* shp(v, T) with lifted arc costs */
static void lifted_backward_dp(obdd *d, const double *l0, const double *l1) {
  for (int32_t h = d->k - 1; h >= 0; --h)
    for (int32_t v = d->hop_start[h]; v < d->hop_start[h + 1]; ++v) {
      double a = l0[h] + ctt_of(d, d->lo[v]);
      double b = l1[h] + ctt_of(d, d->hi[v]);
      d->ctt[v] = a < b ? a : b;
    }
}

/* shp(r, v) of P_h from P_{h-1} with lifted arc costs (A4) */
static void lifted_relax_into(obdd *d, const double *l0, const double *l1, int32_t h) {
  for (int32_t v = d->hop_start[h]; v < d->hop_start[h + 1]; ++v) {
    double best = INFINITY;
    for (int32_t u = d->hop_start[h - 1]; u < d->hop_start[h]; ++u) {
      if (d->lo[u] == v && d->cfr[u] + l0[h - 1] < best) best = d->cfr[u] + l0[h - 1];
      if (d->hi[u] == v && d->cfr[u] + l1[h - 1] < best) best = d->cfr[u] + l1[h - 1];
    }
    d->cfr[v] = best;
  }
}

static void lifted_forward_dp(obdd *d, const double *l0, const double *l1) {
  if (d->k == 0) return;
  d->cfr[0] = 0.0;
  for (int32_t h = 1; h < d->k; ++h) lifted_relax_into(d, l0, l1, h);
}

/* m^beta = min_{v in P_h} shp(r, v) + lambda^{j,beta}_h + shp(s^beta(v), T) */
static void lifted_min_marginals_at(const obdd *d, const double *l0, const double *l1, int32_t h, double *m0,
                                    double *m1) {
  double b0 = INFINITY, b1 = INFINITY;
  for (int32_t v = d->hop_start[h]; v < d->hop_start[h + 1]; ++v) {
    if (d->lo[v] != BOT) {
      double x = (d->cfr[v] + l0[h]) + ctt_of(d, d->lo[v]);
      if (x < b0) b0 = x;
    }
    if (d->hi[v] != BOT) {
      double x = (d->cfr[v] + l1[h]) + ctt_of(d, d->hi[v]);
      if (x < b1) b1 = x;
    }
  }
  *m0 = b0;
  *m1 = b1;
}

static void lifted_update_slot(oracle_solver *s, int64_t slot, double *l0, double *l1, double m0, double m1,
                               double omega) {
  const double d = mm_difference(m1, m0, s->clamp);
  const double delta = omega * d;
  const int32_t i = s->slot_var[slot];
  s->m0[slot] = m0;
  s->m1[slot] = m1;
  *l1 = (*l1 - (delta > 0 ? delta : 0.0)) + s->avg[i];   /* beta = 1 */
  *l0 = (*l0 - (delta < 0 ? -delta : 0.0)) + s->avg0[i]; /* beta = 0 */
  s->delta_new[slot] = delta;
}

static double lifted_energy_of(const obdd *d, const double *l0, const double *l1) {
  double *t = (double *)malloc((size_t)(d->n_nodes ? d->n_nodes : 1) * sizeof(double));
  if (!t) return NAN;
  for (int32_t h = d->k - 1; h >= 0; --h)
    for (int32_t v = d->hop_start[h]; v < d->hop_start[h + 1]; ++v) {
      double a = l0[h] + (d->lo[v] == TOP ? 0.0 : d->lo[v] == BOT ? INFINITY : t[d->lo[v]]);
      double b = l1[h] + (d->hi[v] == TOP ? 0.0 : d->hi[v] == BOT ? INFINITY : t[d->hi[v]]);
      t[v] = a < b ? a : b;
    }
  double e = t[0];
  free(t);
  return e;
}

/* sum_j E_lifted^j + free term: the bound of the lifted representation */
static double lifted_bound(const oracle_solver *s) {
  const int32_t m = s->n_cons;
  int j;
#pragma omp parallel for num_threads(s->n_threads) schedule(dynamic, 256)
  for (j = 0; j < m; ++j) {
    const obdd *d = &s->bdd[j];
    s->energy[j] = d->k ? lifted_energy_of(d, s->lam0 + d->slot0, s->lambda + d->slot0) : 0.0;
  }
  double e = 0.0;
  for (int32_t q = 0; q < m; ++q) e += s->energy[q]; /* fixed order */
  return e + s->free_term;
}

int oracle_set_lifted(oracle_solver *s) {
  if (!s) return O_EINVAL;
  if (s->lifted) return O_OK;
  if (s->passes != 0) return O_ESTATE;
  int64_t S = s->n_slots ? s->n_slots : 1;
  s->lam0 = (double *)calloc((size_t)S, sizeof(double)); /* lambda^{j,0} = 0 */
  s->avg0 = (double *)calloc((size_t)(s->n_vars ? s->n_vars : 1), sizeof(double));
  if (!s->lam0 || !s->avg0) return O_ENOMEM;
  s->lifted = 1; /* lambda^{j,1} = c_i / |J_i| is the lambda set at create */
  s->lb = lifted_bound(s);
  return O_OK;
}

static int lifted_pass(oracle_solver *s, int forward, double omega) {
  /* the two deferred averages from the previous pass (j ascending, A1) */
  for (int32_t i = 0; i < s->n_vars; ++i) {
    int64_t deg = s->var_ptr[i + 1] - s->var_ptr[i];
    double sp = 0.0, sn = 0.0;
    for (int64_t q = s->var_ptr[i]; q < s->var_ptr[i + 1]; ++q) {
      const double x = s->delta_bar[s->var_slots[q]];
      sp += x > 0 ? x : 0.0;
      sn += x < 0 ? -x : 0.0;
    }
    s->avg[i] = deg ? sp / (double)deg : 0.0;
    s->avg0[i] = deg ? sn / (double)deg : 0.0;
  }
  int j;
#pragma omp parallel for num_threads(s->n_threads) schedule(dynamic, 256)
  for (j = 0; j < s->n_cons; ++j) {
    obdd *d = &s->bdd[j];
    if (d->k == 0) continue;
    double *l0 = s->lam0 + d->slot0, *l1 = s->lambda + d->slot0;
    if (forward) {
      lifted_backward_dp(d, l0, l1); /* shp(v, T) at the pass's start */
      for (int32_t h = 0; h < d->k; ++h) {
        if (h == 0) d->cfr[0] = 0.0;
        else lifted_relax_into(d, l0, l1, h); /* with the updated lambda_{h-1} */
        double m0, m1;
        lifted_min_marginals_at(d, l0, l1, h, &m0, &m1);
        lifted_update_slot(s, d->slot0 + h, &l0[h], &l1[h], m0, m1, omega);
      }
    } else {
      lifted_forward_dp(d, l0, l1); /* shp(r, v) at the pass's start */
      for (int32_t h = d->k - 1; h >= 0; --h) {
        double m0, m1;
        lifted_min_marginals_at(d, l0, l1, h, &m0, &m1);
        lifted_update_slot(s, d->slot0 + h, &l0[h], &l1[h], m0, m1, omega);
        for (int32_t v = d->hop_start[h]; v < d->hop_start[h + 1]; ++v) {
          double a = l0[h] + ctt_of(d, d->lo[v]);
          double b = l1[h] + ctt_of(d, d->hi[v]);
          d->ctt[v] = a < b ? a : b;
        }
      }
    }
  }
  double *t = s->delta_bar; /* mbar <- m */
  s->delta_bar = s->delta_new;
  s->delta_new = t;
  s->lb = lifted_bound(s);
  s->passes++;
  return O_OK;
}

int oracle_get_lifted(const oracle_solver *s, double *lam0, double *lam1, int64_t len) {
  if (!s || !s->lifted) return O_EINVAL;
  int rc = copy_out(s->lam0, s->n_slots, lam0, len);
  return rc ? rc : copy_out(s->lambda, s->n_slots, lam1, len);
}
