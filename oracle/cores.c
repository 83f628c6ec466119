/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's O(L^3) Wigner-Delta cores, used by
 * tests/ (as the parity checker), __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference arm.  The product path never links or
 * calls this file.
 *
 * Each function follows /root/reference/pkg/src/torusht/kernels/_numba.py
 * statement for statement with the same per-output summation order, so the
 * results match the numba backend bit for bit when compiled with
 * -ffp-contract=off (pinned by tests/test_oracle.py against the golden
 * vectors that tests/golden/make_golden.py produced from the reference).
 *
 * Threading (pthreads team, `nthreads` argument; 1 = serial): only loops
 * whose iterations write disjoint outputs are split, and every output keeps
 * its serial operation order, so any thread count gives identical bits:
 *   - trapani_step: columns m (each column is an independent chain)  :63-71
 *   - risbo half step: rows i                                          :26-41
 *   - fmm_core: rows m' of T                                           :91-104
 *   - flm_core: outputs m                                              :155-165
 *
 * Layout (row-major, complex = interleaved re/im doubles):
 *   flm2d (L, 2L-1), T (L, 2L-1), gfold (2L-1, L), R (L, 2L-1); real: (L, L)
 */
#define _GNU_SOURCE
#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* _numba.py:15: computed as 1/sqrt(2), one ulp below the rounded literal */
#define INV_SQRT2 (1.0 / sqrt(2.0))

/* ------------------------------------------------------------------ team */

typedef struct team {
  int n;
  pthread_barrier_t bar;
  void (*fn)(struct team *, int tid, void *ctx);
  void *ctx;
} team_t;

typedef struct {
  team_t *t;
  int tid;
} team_arg_t;

static void *team_entry(void *p) {
  team_arg_t *a = (team_arg_t *)p;
  a->t->fn(a->t, a->tid, a->t->ctx);
  return NULL;
}

static void team_sync(team_t *t) {
  if (t->n > 1) pthread_barrier_wait(&t->bar);
}

static void team_run(int n, void (*fn)(team_t *, int, void *), void *ctx) {
  if (n < 1) n = 1;
  team_t t = {n, {{0}}, fn, ctx};
  if (n == 1) {
    fn(&t, 0, ctx);
    return;
  }
  pthread_barrier_init(&t.bar, NULL, (unsigned)n);
  pthread_t *th = malloc(sizeof(pthread_t) * n);
  team_arg_t *args = malloc(sizeof(team_arg_t) * n);
  for (int i = 0; i < n; i++) {
    args[i].t = &t;
    args[i].tid = i;
    if (i) pthread_create(&th[i], NULL, team_entry, &args[i]);
  }
  team_entry(&args[0]);
  for (int i = 1; i < n; i++) pthread_join(th[i], NULL);
  pthread_barrier_destroy(&t.bar);
  free(th);
  free(args);
}

/* contiguous share [lo, hi) of [0, n) for thread tid */
static void share(int n, int tid, int nt, int *lo, int *hi) {
  *lo = (int)((long)n * tid / nt);
  *hi = (int)((long)n * (tid + 1) / nt);
}

/* ------------------------------------------------------------ recursions */

/* _numba.py:18-41, rows [i0, i1) of the half step.  Every entry is computed
 * with the reference's expression and operation order (acc = 0.0, then
 * acc += ri*rk*cc*src[..] etc., dst = acc / two_j); the branches on i and k
 * are only hoisted out of the inner loop (boundary rows/columns peeled), so
 * the interior loop vectorises without changing any entry's bits. */
static void risbo_half_rows(const double *src, int ld, double *dst, int two_j, double cc,
                            double ss, const double *rt, int i0, int i1) {
  const double dj = (double)two_j;
  for (int i = i0; i < i1; i++) {
    const double ri = rt[i], ui = rt[two_j - i];
    const double *sp = i > 0 ? src + (long)(i - 1) * ld : NULL;  /* row i-1 */
    const double *sc = i < two_j ? src + (long)i * ld : NULL;    /* row i   */
    double *d = dst + (long)i * ld;
    for (int k = 0; k <= two_j; k++) {
      if (k == 1 && sp && sc && two_j >= 2) {
        /* interior columns 1 <= k < two_j, all four terms */
        const int kend = two_j;
        for (int kk = 1; kk < kend; kk++) {
          const double rk = rt[kk], uk = rt[two_j - kk];
          double acc = 0.0;
          acc += ri * rk * cc * sp[kk - 1];
          acc -= ri * uk * ss * sp[kk];
          acc += ui * rk * ss * sc[kk - 1];
          acc += ui * uk * cc * sc[kk];
          d[kk] = acc / dj;
        }
        k = kend - 1;
        continue;
      }
      const double rk = rt[k], uk = rt[two_j - k];
      double acc = 0.0;
      if (sp) {
        if (k > 0) acc += ri * rk * cc * sp[k - 1];
        if (k < two_j) acc -= ri * uk * ss * sp[k];
      }
      if (sc) {
        if (k > 0) acc += ui * rk * ss * sc[k - 1];
        if (k < two_j) acc += ui * uk * cc * sc[k];
      }
      d[k] = acc / two_j;
    }
  }
}

/* _numba.py:53-71, columns [m0, m1) only (the top row is written by the
 * caller's thread 0 before the team splits the columns). */
static void trapani_top(double *quad, int ld, int ell) {
  for (int m = ell; m > 0; m--)
    quad[ell * ld + m] =
        sqrt(ell * (2.0 * ell - 1.0) / (2.0 * (ell + m) * (ell + m - 1.0))) *
        quad[(ell - 1) * ld + (m - 1)];
  quad[ell * ld + 0] = -sqrt((2.0 * ell - 1.0) / (2.0 * ell)) * quad[(ell - 1) * ld + 0];
}

static void trapani_cols(double *quad, int ld, int ell, int m0, int m1) {
  for (int mu = ell - 1; mu >= 0; mu--) {
    double inv = 1.0 / sqrt((ell + mu + 1.0) * (ell - mu));
    if (mu + 2 <= ell) {
      double c2 = sqrt((ell - mu - 1.0) * (ell + mu + 2.0));
      for (int m = m0; m < m1; m++)
        quad[mu * ld + m] =
            (2.0 * m * quad[(mu + 1) * ld + m] - c2 * quad[(mu + 2) * ld + m]) * inv;
    } else {
      for (int m = m0; m < m1; m++) quad[mu * ld + m] = 2.0 * m * quad[(mu + 1) * ld + m] * inv;
    }
  }
}

/* Shared per-transform state: quadrant + Risbo planes. */
typedef struct {
  int L, use_trapani;
  double *quad, *a, *b, *rt;
} state_t;

static int state_init(state_t *s, int L, int use_trapani) {
  s->L = L;
  s->use_trapani = use_trapani;
  s->quad = calloc((size_t)L * L, sizeof(double));
  s->a = s->b = NULL;
  s->rt = calloc((size_t)2 * L + 2, sizeof(double));
  if (!use_trapani) {
    size_t side = 2 * (size_t)L - 1;
    s->a = calloc(side * side, sizeof(double));
    s->b = calloc(side * side, sizeof(double));
  }
  return s->quad && s->rt && (use_trapani || (s->a && s->b));
}

static void state_free(state_t *s) {
  free(s->quad);
  free(s->a);
  free(s->b);
  free(s->rt);
}

/* Advance every thread's view to degree el (_numba.py:82-88, 44-50).
 * Ends with a team barrier: s->quad holds the degree-el quadrant. */
static void state_step(team_t *t, int tid, state_t *s, int el) {
  int L = s->L, lo, hi;
  if (s->use_trapani) {
    if (el == 0) {
      if (tid == 0) s->quad[0] = 1.0;
      team_sync(t);
      return;
    }
    if (tid == 0) trapani_top(s->quad, L, el);
    team_sync(t);
    share(el + 1, tid, t->n, &lo, &hi);
    trapani_cols(s->quad, L, el, lo, hi);
    team_sync(t);
    return;
  }
  int side = 2 * L - 1;
  if (el == 0) {
    if (tid == 0) s->a[0] = 1.0, s->quad[0] = 1.0;
    team_sync(t);
    return;
  }
  if (tid == 0)
    for (int i = 0; i <= 2 * el; i++) s->rt[i] = sqrt((double)i);
  team_sync(t);
  share(2 * el, tid, t->n, &lo, &hi);
  risbo_half_rows(s->a, side, s->b, 2 * el - 1, INV_SQRT2, INV_SQRT2, s->rt, lo, hi);
  team_sync(t);
  share(2 * el + 1, tid, t->n, &lo, &hi);
  risbo_half_rows(s->b, side, s->a, 2 * el, INV_SQRT2, INV_SQRT2, s->rt, lo, hi);
  team_sync(t);
  share(el + 1, tid, t->n, &lo, &hi);
  for (int mp = lo; mp < hi; mp++)
    for (int m = 0; m <= el; m++) s->quad[mp * L + m] = s->a[(el + mp) * side + el + m];
  team_sync(t);
}

/* Single-threaded recursion hooks (kernel-level parity tests). */
void oracle_trapani_step(double *quad, int ld, int ell) {
  if (ell == 0) {
    quad[0] = 1.0;
    return;
  }
  trapani_top(quad, ld, ell);
  trapani_cols(quad, ld, ell, 0, ell + 1);
}

void oracle_risbo_step_into(double *a, double *b, int side, int ell) {
  if (ell == 0) {
    a[0] = 1.0;
    return;
  }
  double *rt = malloc(sizeof(double) * (2 * ell + 1));
  for (int i = 0; i <= 2 * ell; i++) rt[i] = sqrt((double)i);
  risbo_half_rows(a, side, b, 2 * ell - 1, INV_SQRT2, INV_SQRT2, rt, 0, 2 * ell);
  risbo_half_rows(b, side, a, 2 * ell, INV_SQRT2, INV_SQRT2, rt, 0, 2 * ell + 1);
  free(rt);
}

/* ----------------------------------------------------------------- cores */

typedef struct {
  state_t s;
  const double *in, *cl;
  double *out, *dsrow;
  int L, spin;
} core_ctx_t;

/* _numba.py:74-105 */
static void fmm_worker(team_t *t, int tid, void *p) {
  core_ctx_t *c = (core_ctx_t *)p;
  int L = c->L, N = 2 * L - 1, spin = c->spin, cs = abs(spin), lo, hi;
  for (int el = 0; el < L; el++) {
    state_step(t, tid, &c->s, el);
    if (el < cs) continue;
    const double *q = c->s.quad;
    share(el + 1, tid, t->n, &lo, &hi);
    for (int mp = lo; mp < hi; mp++) {
      double sgn = ((el + mp) & 1) ? -1.0 : 1.0;
      double ds = q[mp * L + cs];
      if (spin > 0) ds *= sgn;
      double w = c->cl[el] * ds;
      double *Trow = c->out + 2 * (size_t)mp * N;
      const double *frow = c->in + 2 * (size_t)el * N;
      for (int m = 0; m <= el; m++) {
        double x = w * q[mp * L + m];
        Trow[2 * (L - 1 + m)] += x * frow[2 * (L - 1 + m)];
        Trow[2 * (L - 1 + m) + 1] += x * frow[2 * (L - 1 + m) + 1];
      }
      double ws = w * sgn;
      for (int m = 1; m <= el; m++) {
        double x = ws * q[mp * L + m];
        Trow[2 * (L - 1 - m)] += x * frow[2 * (L - 1 - m)];
        Trow[2 * (L - 1 - m) + 1] += x * frow[2 * (L - 1 - m) + 1];
      }
    }
    /* the next state_step starts with a barrier-protected write by tid 0
       only to the top row / rt, which no thread reads here */
    team_sync(t);
  }
}

/* _numba.py:108-128 */
static void fmm_real_worker(team_t *t, int tid, void *p) {
  core_ctx_t *c = (core_ctx_t *)p;
  int L = c->L, lo, hi;
  for (int el = 0; el < L; el++) {
    state_step(t, tid, &c->s, el);
    const double *q = c->s.quad;
    share(el + 1, tid, t->n, &lo, &hi);
    for (int mp = lo; mp < hi; mp++) {
      double w = c->cl[el] * q[mp * L + 0];
      if (w == 0.0) continue;
      double *Trow = c->out + 2 * (size_t)mp * L;
      const double *frow = c->in + 2 * (size_t)el * L;
      for (int m = 0; m <= el; m++) {
        double x = w * q[mp * L + m];
        Trow[2 * m] += x * frow[2 * m];
        Trow[2 * m + 1] += x * frow[2 * m + 1];
      }
    }
    team_sync(t);
  }
}

/* _numba.py:131-166 */
static void flm_worker(team_t *t, int tid, void *p) {
  core_ctx_t *c = (core_ctx_t *)p;
  int L = c->L, N = 2 * L - 1, spin = c->spin, cs = abs(spin), lo, hi;
  for (int el = 0; el < L; el++) {
    state_step(t, tid, &c->s, el);
    if (el < cs) continue;
    const double *q = c->s.quad;
    if (tid == 0)
      for (int mp = 0; mp <= el; mp++) {
        double sgn = ((el + mp) & 1) ? -1.0 : 1.0;
        double ds = q[mp * L + cs];
        if (spin > 0) ds *= sgn;
        c->dsrow[mp] = ds;
      }
    team_sync(t);
    share(el + 1, tid, t->n, &lo, &hi);
    for (int m = lo; m < hi; m++) {
      double ar = 0.0, ai = 0.0;
      const double *g = c->in + 2 * (size_t)(L - 1 + m) * L;
      for (int mp = 0; mp <= el; mp++) {
        double x = c->dsrow[mp] * q[mp * L + m];
        ar += x * g[2 * mp];
        ai += x * g[2 * mp + 1];
      }
      c->out[2 * ((size_t)el * N + L - 1 + m)] = ar;
      c->out[2 * ((size_t)el * N + L - 1 + m) + 1] = ai;
    }
    share(el, tid, t->n, &lo, &hi);
    for (int m = lo + 1; m < hi + 1; m++) {
      double ar = 0.0, ai = 0.0;
      const double *g = c->in + 2 * (size_t)(L - 1 - m) * L;
      for (int mp = 0; mp <= el; mp++) {
        double sgn = ((el + mp) & 1) ? -1.0 : 1.0;
        double x = c->dsrow[mp] * sgn * q[mp * L + m];
        ar += x * g[2 * mp];
        ai += x * g[2 * mp + 1];
      }
      c->out[2 * ((size_t)el * N + L - 1 - m)] = ar;
      c->out[2 * ((size_t)el * N + L - 1 - m) + 1] = ai;
    }
    team_sync(t);
  }
}

/* _numba.py:169-188 */
static void flm_real_worker(team_t *t, int tid, void *p) {
  core_ctx_t *c = (core_ctx_t *)p;
  int L = c->L, lo, hi;
  for (int el = 0; el < L; el++) {
    state_step(t, tid, &c->s, el);
    const double *q = c->s.quad;
    share(el + 1, tid, t->n, &lo, &hi);
    for (int m = lo; m < hi; m++) {
      double ar = 0.0, ai = 0.0;
      const double *g = c->in + 2 * (size_t)m * L;
      for (int mp = 0; mp <= el; mp++) {
        double x = q[mp * L + 0] * q[mp * L + m];
        ar += x * g[2 * mp];
        ai += x * g[2 * mp + 1];
      }
      c->out[2 * ((size_t)el * L + m)] = ar;
      c->out[2 * ((size_t)el * L + m) + 1] = ai;
    }
    team_sync(t);
  }
}

static int run_core(void (*fn)(team_t *, int, void *), const double *in, const double *cl,
                    int L, int spin, int use_trapani, double *out, size_t out_doubles,
                    int nthreads) {
  core_ctx_t c;
  memset(&c, 0, sizeof(c));
  if (L < 1) return -2;
  if (!state_init(&c.s, L, use_trapani)) return -1;
  c.in = in;
  c.cl = cl;
  c.out = out;
  c.L = L;
  c.spin = spin;
  c.dsrow = calloc((size_t)L, sizeof(double));
  memset(out, 0, sizeof(double) * out_doubles);
  if (nthreads > L) nthreads = L;
  team_run(nthreads, fn, &c);
  free(c.dsrow);
  state_free(&c.s);
  return 0;
}

int oracle_fmm_core(const double *flm2d, const double *cl, int L, int spin, int use_trapani,
                    double *T, int nthreads) {
  return run_core(fmm_worker, flm2d, cl, L, spin, use_trapani, T,
                  2 * (size_t)L * (2 * L - 1), nthreads);
}

int oracle_fmm_core_real(const double *flm2d, const double *cl, int L, int use_trapani,
                         double *T, int nthreads) {
  return run_core(fmm_real_worker, flm2d, cl, L, 0, use_trapani, T, 2 * (size_t)L * L,
                  nthreads);
}

int oracle_flm_core(const double *gfold, int L, int spin, int use_trapani, double *R,
                    int nthreads) {
  return run_core(flm_worker, gfold, NULL, L, spin, use_trapani, R,
                  2 * (size_t)L * (2 * L - 1), nthreads);
}

int oracle_flm_core_real(const double *gfold, int L, int use_trapani, double *R,
                         int nthreads) {
  return run_core(flm_real_worker, gfold, NULL, L, 0, use_trapani, R, 2 * (size_t)L * L,
                  nthreads);
}
