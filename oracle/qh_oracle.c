/*
 * ORACLE -- test infrastructure only.  Nothing in the product path
 * (paper_1201_2936_b200/) links, loads or calls this file; only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * leg use it, and only as the checker / CPU baseline.
 *
 * Plain-C restatement of the reference's flat-array Quickhull drivers
 * (/root/reference/pkg/src/seghull/quickhull.py) for the hot path:
 *   quickhull_2d   quickhull.py:167-279
 *   quickhull_3d   quickhull.py:282-446 (main loop; the post-loop candidate
 *                  filter _extreme_vertex_mask :136-164 is NOT restated here,
 *                  the loop's candidate list is returned instead)
 *
 * The segment bookkeeping follows the reference exactly: segments live in
 * one flat array in flag_permute order ((parent, state) groups, stable,
 * primitives.py:91-117), compact preserves order (primitives.py:120-148),
 * so vertices come out in the reference's discovery order and the result
 * can be compared byte-for-byte with the reference's `vertices`.
 *
 * Arithmetic: every product and sum is rounded separately (the Makefile
 * builds with -ffp-contract=off and no -march), in the operation order of
 * geometry.py; edge lengths use libm hypot, which is what np.hypot calls.
 *
 * Parity of this restatement is pinned by tests/test_oracle.py against
 * golden vectors produced by the reference itself (tests/golden/, made by
 * tests/golden/make_golden.py) and against the reference's own KATs.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OQ_OK 0
#define OQ_EMPTY 2
#define OQ_DEGENERATE 3
#define OQ_ROUND_GUARD 4
#define OQ_NOMEM 5

/* flags */
#define OQ_WARN_COLLINEAR 1

static double cross2(double ax, double ay, double bx, double by, double qx, double qy) {
  /* geometry.py:121 */
  return ax * (by - qy) + bx * (qy - ay) + qx * (ay - by);
}

static double edge_length(double ax, double ay, double bx, double by) {
  return hypot(bx - ax, by - ay); /* geometry.py:124-127 */
}

/* quickhull.py:75-84: lexicographic extreme over (coords..., index); the
 * minimum takes the lowest index among full ties, the maximum the highest. */
static int64_t lex_extreme(const double* const* c, int dim, int64_t n, int want_max) {
  int64_t best = 0;
  for (int64_t i = 1; i < n; i++) {
    int cmp = 0;
    for (int a = 0; a < dim && cmp == 0; a++) {
      if (c[a][i] < c[a][best]) cmp = -1;
      else if (c[a][i] > c[a][best]) cmp = 1;
    }
    if (want_max) {
      if (cmp >= 0) best = i; /* ties: later (higher) index wins */
    } else {
      if (cmp < 0) best = i; /* ties: keep the lower index */
    }
  }
  return best;
}

/* geometry.py:79-83 */
static double effective_eps(const double* const* c, int dim, int64_t n, double eps_rel) {
  if (n == 0) return 0.0;
  double acc = 0.0;
  for (int a = 0; a < dim; a++) {
    double lo = c[a][0], hi = c[a][0];
    for (int64_t i = 1; i < n; i++) {
      if (c[a][i] < lo) lo = c[a][i];
      if (c[a][i] > hi) hi = c[a][i];
    }
    double span = hi - lo;
    acc = (a == 0) ? span : hypot(acc, span); /* np.hypot.reduce */
  }
  return eps_rel * acc;
}

/* ------------------------------------------------------------------------ */
/* 2D                                                                        */
/* ------------------------------------------------------------------------ */

typedef struct { double ax, ay, bx, by; } edge2;

/*
 * out_idx: capacity n, receives original indices of the hull vertices in the
 * reference's discovery order.  trace (optional): 3 int64 per round
 * (live entering, kept after compact, segments).  Returns a status code.
 */
int oq_hull2d(const double* x0, const double* y0, int64_t n, double eps_rel, double eps_abs,
              int64_t* out_idx, int64_t* out_h, int64_t* out_iters, int32_t* out_flags,
              int64_t* trace, int64_t trace_cap, int64_t* out_trace_len) {
  *out_h = 0;
  *out_iters = 0;
  *out_flags = 0;
  if (out_trace_len) *out_trace_len = 0;
  if (n == 0) return OQ_EMPTY;
  const double* cs[2] = {x0, y0};
  /* eps_abs (not NaN): a sharded run's global eps (paper_1201_2936_b200/sharded.py) */
  double eps = isnan(eps_abs) ? effective_eps(cs, 2, n, eps_rel) : eps_abs;
  int64_t h = 0;
  int64_t imin = lex_extreme(cs, 2, n, 0);
  int64_t imax = lex_extreme(cs, 2, n, 1);
  double pminx = x0[imin], pminy = y0[imin], pmaxx = x0[imax], pmaxy = y0[imax];
  if (pminx == pmaxx && pminy == pmaxy) { /* quickhull.py:195-197 */
    out_idx[h++] = imin;
    *out_h = h;
    return OQ_OK;
  }
  out_idx[h++] = imin;
  out_idx[h++] = imax;

  /* first split, quickhull.py:200-222 */
  double* X = (double*)malloc(sizeof(double) * (size_t)n);
  double* Y = (double*)malloc(sizeof(double) * (size_t)n);
  int64_t* I = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  double* X2 = (double*)malloc(sizeof(double) * (size_t)n);
  double* Y2 = (double*)malloc(sizeof(double) * (size_t)n);
  int64_t* I2 = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  signed char* st = (signed char*)malloc((size_t)n);
  int64_t* segstart = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 2));
  int64_t* segstart2 = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 2));
  edge2* tab = (edge2*)malloc(sizeof(edge2) * (size_t)(n + 2));
  edge2* tab2 = (edge2*)malloc(sizeof(edge2) * (size_t)(n + 2));
  int64_t* far = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 2));
  int status = OQ_OK;
  if (!X || !Y || !I || !X2 || !Y2 || !I2 || !st || !segstart || !segstart2 || !tab || !tab2 || !far) {
    status = OQ_NOMEM;
    goto done;
  }
  {
    double thr = eps * edge_length(pminx, pminy, pmaxx, pmaxy);
    int64_t m = 0, c0 = 0;
    for (int64_t i = 0; i < n; i++) {
      if (i == imin || i == imax) continue;
      double d = cross2(pminx, pminy, pmaxx, pmaxy, x0[i], y0[i]);
      if (fabs(d) > thr) {
        X2[m] = x0[i];
        Y2[m] = y0[i];
        I2[m] = i;
        st[m] = d < 0 ? 1 : 0;
        c0 += st[m] == 0;
        m++;
      }
    }
    if (m == 0) {
      if (n - 2 > 0) *out_flags |= OQ_WARN_COLLINEAR;
      goto done;
    }
    /* flag_permute(states, s, 2): stable, side 0 first */
    int64_t w0 = 0, w1 = c0;
    for (int64_t i = 0; i < m; i++) {
      int64_t p = st[i] == 0 ? w0++ : w1++;
      X[p] = X2[i];
      Y[p] = Y2[i];
      I[p] = I2[i];
    }
    int64_t nseg = 0;
    if (c0 > 0) {
      segstart[nseg] = 0;
      tab[nseg] = (edge2){pminx, pminy, pmaxx, pmaxy};
      nseg++;
    }
    if (m - c0 > 0) {
      segstart[nseg] = c0;
      tab[nseg] = (edge2){pmaxx, pmaxy, pminx, pminy};
      nseg++;
    }
    segstart[nseg] = m;

    int64_t iters = 0;
    while (m > 0) { /* quickhull.py:225 */
      iters++;
      if (iters > n + 1) { status = OQ_ROUND_GUARD; break; }
      /* farthest per segment: first max (lowest position) */
      for (int64_t s = 0; s < nseg; s++) {
        edge2 e = tab[s];
        int64_t best = -1;
        double bd = 0;
        for (int64_t i = segstart[s]; i < segstart[s + 1]; i++) {
          double d = cross2(e.ax, e.ay, e.bx, e.by, X[i], Y[i]) + 0.0;
          if (best < 0 || d > bd) { best = i; bd = d; }
        }
        far[s] = best;
        out_idx[h++] = I[best];
      }
      /* keep + classify + permute; child segments in (parent, state) order */
      int64_t m2 = 0, nseg2 = 0, kept = 0;
      for (int64_t s = 0; s < nseg; s++) {
        edge2 e = tab[s];
        double fx = X[far[s]], fy = Y[far[s]];
        double t_ab = -eps * edge_length(e.ax, e.ay, e.bx, e.by);
        double t_bf = -eps * edge_length(e.bx, e.by, fx, fy);
        double t_fa = -eps * edge_length(fx, fy, e.ax, e.ay);
        int64_t cnt[2] = {0, 0};
        int64_t base = m2;
        /* pass 1: count per state among survivors */
        for (int64_t i = segstart[s]; i < segstart[s + 1]; i++) {
          double qx = X[i], qy = Y[i];
          int inside = cross2(e.ax, e.ay, e.bx, e.by, qx, qy) >= t_ab;
          inside &= cross2(e.bx, e.by, fx, fy, qx, qy) >= t_bf;
          inside &= cross2(fx, fy, e.ax, e.ay, qx, qy) >= t_fa;
          if (inside || i == far[s]) { st[i] = -1; continue; }
          /* classify_two_edges(a, far, b, q), geometry.py:178-189 */
          double c0v = cross2(e.ax, e.ay, fx, fy, qx, qy);
          double c1v = cross2(fx, fy, e.bx, e.by, qx, qy);
          int one_sided = (c0v > 0) != (c1v > 0);
          int state = one_sided ? (c1v > 0 ? 1 : 0) : (c1v > c0v ? 1 : 0);
          st[i] = (signed char)state;
          cnt[state]++;
        }
        kept += cnt[0] + cnt[1];
        int64_t w[2] = {base, base + cnt[0]};
        for (int64_t i = segstart[s]; i < segstart[s + 1]; i++) {
          if (st[i] < 0) continue;
          int64_t p = w[(int)st[i]]++;
          X2[p] = X[i];
          Y2[p] = Y[i];
          I2[p] = I[i];
        }
        if (cnt[0]) {
          segstart2[nseg2] = base;
          tab2[nseg2] = (edge2){e.ax, e.ay, fx, fy};
          nseg2++;
        }
        if (cnt[1]) {
          segstart2[nseg2] = base + cnt[0];
          tab2[nseg2] = (edge2){fx, fy, e.bx, e.by};
          nseg2++;
        }
        m2 += cnt[0] + cnt[1];
      }
      if (trace && *out_trace_len < trace_cap) {
        trace[3 * *out_trace_len + 0] = m;
        trace[3 * *out_trace_len + 1] = kept;
        trace[3 * *out_trace_len + 2] = nseg;
        (*out_trace_len)++;
      }
      segstart2[nseg2] = m2;
      double* tx = X; X = X2; X2 = tx;
      double* ty = Y; Y = Y2; Y2 = ty;
      int64_t* ti = I; I = I2; I2 = ti;
      int64_t* ts = segstart; segstart = segstart2; segstart2 = ts;
      edge2* tt = tab; tab = tab2; tab2 = tt;
      m = m2;
      nseg = nseg2;
    }
    *out_iters = iters;
  }
done:
  *out_h = h;
  free(X); free(Y); free(I); free(X2); free(Y2); free(I2); free(st);
  free(segstart); free(segstart2); free(tab); free(tab2); free(far);
  return status;
}

/* ------------------------------------------------------------------------ */
/* 3D                                                                        */
/* ------------------------------------------------------------------------ */

typedef struct {
  double c[3][3]; /* corners a, b, c */
  double n[3];    /* (b-a) x (c-a) */
  double nlen;
} face3;

static void cross3(double ux, double uy, double uz, double vx, double vy, double vz, double* o) {
  o[0] = uy * vz - uz * vy; /* geometry.py:131 */
  o[1] = uz * vx - ux * vz;
  o[2] = ux * vy - uy * vx;
}

static double norm3(const double* v) { return sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]); }

static face3 make_face(const double* a, const double* b, const double* c) {
  /* FaceTable.from_corners, quickhull.py:68-72 */
  face3 f;
  for (int k = 0; k < 3; k++) {
    f.c[0][k] = a[k];
    f.c[1][k] = b[k];
    f.c[2][k] = c[k];
  }
  cross3(b[0] - a[0], b[1] - a[1], b[2] - a[2], c[0] - a[0], c[1] - a[1], c[2] - a[2], f.n);
  f.nlen = norm3(f.n);
  return f;
}

static double pdist(const face3* f, double qx, double qy, double qz) {
  /* geometry.py:147 / quickhull.py:376-377 */
  return f->n[0] * (qx - f->c[0][0]) + f->n[1] * (qy - f->c[0][1]) + f->n[2] * (qz - f->c[0][2]);
}

/*
 * Loop of quickhull_3d; out_idx receives the candidate vertices (before the
 * reference's _extreme_vertex_mask filter) in discovery order.  flat_counts
 * (optional, per round) receives the near-coplanar segment drop counts that
 * the reference turns into warnings (quickhull.py:386-389).
 * Returns OQ_DEGENERATE for the coplanar case (quickhull.py:349-351).
 * out_filter = 1 when the reference would run the candidate filter
 * (normal loop exit), 0 for the early returns (result(0)).
 */
int oq_hull3d(const double* x0, const double* y0, const double* z0, int64_t n, double eps_rel,
              double eps_abs, int64_t* out_idx, int64_t* out_h, int64_t* out_iters, int32_t* out_flags,
              int32_t* out_filter, int64_t* flat_counts, int64_t flat_cap,
              int64_t* trace, int64_t trace_cap, int64_t* out_trace_len) {
  *out_h = 0;
  *out_iters = 0;
  *out_flags = 0;
  *out_filter = 0;
  if (out_trace_len) *out_trace_len = 0;
  if (n == 0) return OQ_EMPTY;
  const double* cs[3] = {x0, y0, z0};
  double eps = isnan(eps_abs) ? effective_eps(cs, 3, n, eps_rel) : eps_abs;
  int64_t h = 0;
  int64_t imin = lex_extreme(cs, 3, n, 0);
  int64_t imax = lex_extreme(cs, 3, n, 1);
  double pa[3] = {x0[imin], y0[imin], z0[imin]};
  double pb[3] = {x0[imax], y0[imax], z0[imax]};
  if (pa[0] == pb[0] && pa[1] == pb[1] && pa[2] == pb[2]) {
    out_idx[h++] = imin;
    *out_h = h;
    return OQ_OK;
  }
  out_idx[h++] = imin;
  out_idx[h++] = imax;
  if (n - 2 == 0) { *out_h = h; return OQ_OK; }

  /* third corner: farthest from the extrema line (first argmax), :330-335 */
  double u[3] = {pb[0] - pa[0], pb[1] - pa[1], pb[2] - pa[2]};
  int64_t far_i = -1;
  double best = 0;
  for (int64_t i = 0; i < n; i++) {
    if (i == imin || i == imax) continue;
    double c[3];
    cross3(x0[i] - pa[0], y0[i] - pa[1], z0[i] - pa[2], u[0], u[1], u[2], c);
    double d2 = c[0] * c[0] + c[1] * c[1] + c[2] * c[2];
    if (far_i < 0 || d2 > best) { far_i = i; best = d2; }
  }
  /* np.linalg.norm(pb - pa) (:336) is sqrt(ddot(u, u)); on the reference
   * host OpenBLAS's ddot evaluates it as fma(u2,u2, fma(u1,u1, u0*u0))
   * (matched 100000/100000 random vectors). */
  double line_len = sqrt(fma(u[2], u[2], fma(u[1], u[1], u[0] * u[0])));
  if (sqrt(best) <= eps * line_len) {
    *out_flags |= OQ_WARN_COLLINEAR;
    *out_h = h;
    return OQ_OK;
  }
  double pc[3] = {x0[far_i], y0[far_i], z0[far_i]};
  out_idx[h++] = far_i;
  if (n - 3 == 0) { *out_h = h; return OQ_OK; }

  double nn[3];
  cross3(pb[0] - pa[0], pb[1] - pa[1], pb[2] - pa[2], pc[0] - pa[0], pc[1] - pa[1], pc[2] - pa[2], nn);
  double nlen = sqrt(nn[0] * nn[0] + nn[1] * nn[1] + nn[2] * nn[2]);

  double *X = malloc(8 * (size_t)n), *Y = malloc(8 * (size_t)n), *Z = malloc(8 * (size_t)n);
  double *X2 = malloc(8 * (size_t)n), *Y2 = malloc(8 * (size_t)n), *Z2 = malloc(8 * (size_t)n);
  int64_t *I = malloc(8 * (size_t)n), *I2 = malloc(8 * (size_t)n);
  signed char* st = malloc((size_t)n);
  int64_t* segstart = malloc(8 * (size_t)(n + 2));
  int64_t* segstart2 = malloc(8 * (size_t)(n + 2));
  face3* tab = malloc(sizeof(face3) * (size_t)(n + 2));
  face3* tab2 = malloc(sizeof(face3) * (size_t)(n + 2));
  int64_t* far = malloc(8 * (size_t)(n + 2));
  signed char* flat = malloc((size_t)(n + 2));
  int status = OQ_OK;
  if (!X || !Y || !Z || !X2 || !Y2 || !Z2 || !I || !I2 || !st || !segstart || !segstart2 || !tab ||
      !tab2 || !far || !flat) {
    status = OQ_NOMEM;
    goto done3;
  }
  {
    double dmax = 0;
    int64_t m = 0, c0 = 0;
    double nthr = -eps * nlen;
    for (int64_t i = 0; i < n; i++) {
      if (i == imin || i == imax || i == far_i) continue;
      double d = nn[0] * (x0[i] - pa[0]) + nn[1] * (y0[i] - pa[1]) + nn[2] * (z0[i] - pa[2]);
      if (fabs(d) > dmax) dmax = fabs(d);
      X2[m] = x0[i]; Y2[m] = y0[i]; Z2[m] = z0[i]; I2[m] = i;
      st[m] = d < nthr ? 1 : 0;
      c0 += st[m] == 0;
      m++;
    }
    if (dmax <= eps * nlen) { status = OQ_DEGENERATE; goto done3; }
    int64_t w0 = 0, w1 = c0;
    for (int64_t i = 0; i < m; i++) {
      int64_t p = st[i] == 0 ? w0++ : w1++;
      X[p] = X2[i]; Y[p] = Y2[i]; Z[p] = Z2[i]; I[p] = I2[i];
    }
    int64_t nseg = 0;
    if (c0 > 0) { segstart[nseg] = 0; tab[nseg++] = make_face(pa, pb, pc); }
    if (m - c0 > 0) { segstart[nseg] = c0; tab[nseg++] = make_face(pa, pc, pb); }
    segstart[nseg] = m;

    int64_t iters = 0;
    while (m > 0) {
      iters++;
      if (iters > n + 1) { status = OQ_ROUND_GUARD; break; }
      int64_t nflat = 0;
      for (int64_t s = 0; s < nseg; s++) {
        const face3* f = &tab[s];
        int64_t b = -1;
        double bd = 0;
        for (int64_t i = segstart[s]; i < segstart[s + 1]; i++) {
          double d = pdist(f, X[i], Y[i], Z[i]) + 0.0;
          if (b < 0 || d > bd) { b = i; bd = d; }
        }
        far[s] = b;
        flat[s] = bd <= eps * f->nlen;
        if (flat[s]) nflat++;
        else out_idx[h++] = I[b];
      }
      if (flat_counts && iters - 1 < flat_cap) flat_counts[iters - 1] = nflat;
      int64_t m2 = 0, nseg2 = 0, kept = 0;
      for (int64_t s = 0; s < nseg; s++) {
        const face3* f = &tab[s];
        if (flat[s]) continue;
        double fp[3] = {X[far[s]], Y[far[s]], Z[far[s]]};
        face3 ch[3] = {make_face(f->c[0], f->c[1], fp), make_face(f->c[1], f->c[2], fp),
                       make_face(f->c[2], f->c[0], fp)};
        double tb = -eps * f->nlen;
        double tch[3] = {eps * ch[0].nlen, eps * ch[1].nlen, eps * ch[2].nlen};
        int64_t cnt[3] = {0, 0, 0};
        int64_t base = m2;
        for (int64_t i = segstart[s]; i < segstart[s + 1]; i++) {
          double qx = X[i], qy = Y[i], qz = Z[i];
          double D[3];
          for (int j = 0; j < 3; j++) D[j] = pdist(&ch[j], qx, qy, qz);
          int inside = pdist(f, qx, qy, qz) >= tb;
          for (int j = 0; j < 3; j++) inside &= D[j] <= tch[j];
          if (inside || i == far[s]) { st[i] = -1; continue; }
          /* classify_three_faces: first argmax of D_j / |N_j| (np.argmax) */
          double q0 = D[0] / ch[0].nlen, q1 = D[1] / ch[1].nlen, q2 = D[2] / ch[2].nlen;
          int state = 0;
          double qb = q0;
          if (q1 > qb) { state = 1; qb = q1; }
          if (q2 > qb) { state = 2; qb = q2; }
          st[i] = (signed char)state;
          cnt[state]++;
        }
        kept += cnt[0] + cnt[1] + cnt[2];
        int64_t w[3] = {base, base + cnt[0], base + cnt[0] + cnt[1]};
        for (int64_t i = segstart[s]; i < segstart[s + 1]; i++) {
          if (st[i] < 0) continue;
          int64_t p = w[(int)st[i]]++;
          X2[p] = X[i]; Y2[p] = Y[i]; Z2[p] = Z[i]; I2[p] = I[i];
        }
        int64_t off = base;
        for (int j = 0; j < 3; j++) {
          if (cnt[j]) {
            segstart2[nseg2] = off;
            tab2[nseg2] = ch[j];
            nseg2++;
          }
          off += cnt[j];
        }
        m2 += cnt[0] + cnt[1] + cnt[2];
      }
      if (trace && *out_trace_len < trace_cap) {
        trace[3 * *out_trace_len + 0] = m;
        trace[3 * *out_trace_len + 1] = kept;
        trace[3 * *out_trace_len + 2] = nseg;
        (*out_trace_len)++;
      }
      segstart2[nseg2] = m2;
      double* t;
      t = X; X = X2; X2 = t;
      t = Y; Y = Y2; Y2 = t;
      t = Z; Z = Z2; Z2 = t;
      int64_t* ti = I; I = I2; I2 = ti;
      int64_t* ts = segstart; segstart = segstart2; segstart2 = ts;
      face3* tt = tab; tab = tab2; tab2 = tt;
      m = m2;
      nseg = nseg2;
    }
    *out_iters = iters;
    *out_filter = 1;
  }
done3:
  *out_h = h;
  free(X); free(Y); free(Z); free(X2); free(Y2); free(Z2); free(I); free(I2); free(st);
  free(segstart); free(segstart2); free(tab); free(tab2); free(far); free(flat);
  return status;
}

/* hull2_giftwrap (reference seghull/oracle module lines 20-52): sequential
 * scan in index order, coordinates compared as tuples.  Writes the index of
 * the first occurrence of each hull vertex, CCW from the lexicographic
 * minimum; returns the vertex count (or -1 when cap is too small). */
int64_t oq_giftwrap2d(const double* x, const double* y, int64_t n, double eps, int64_t* out, int64_t cap) {
  if (n <= 0 || cap < 1) return -1;
  int64_t s = 0;
  for (int64_t i = 1; i < n; i++)
    if (x[i] < x[s] || (x[i] == x[s] && y[i] < y[s])) s = i;
  int64_t h = 0;
  out[h++] = s;
  int64_t cur = s;
  for (int64_t step = 0; step <= n; step++) {
    const double cx = x[cur], cy = y[cur];
    int64_t cand = -1;
    for (int64_t q = 0; q < n; q++) {
      if (x[q] == cx && y[q] == cy) continue;
      if (cand < 0) {
        cand = q;
        continue;
      }
      const double ax = x[cand] - cx, ay = y[cand] - cy, qx = x[q] - cx, qy = y[q] - cy;
      const double cr = ax * qy - ay * qx;
      const double limit = eps * hypot(ax, ay);
      if (cr < -limit)
        cand = q;
      else if (cr <= limit && qx * qx + qy * qy > ax * ax + ay * ay)
        cand = q;
    }
    if (cand < 0 || (x[cand] == x[s] && y[cand] == y[s])) break;
    if (h >= cap) return -1;
    /* first occurrence of the coordinates (the reference keeps tuples) */
    int64_t f = cand;
    for (int64_t q = 0; q < cand; q++)
      if (x[q] == x[cand] && y[q] == y[cand]) {
        f = q;
        break;
      }
    out[h++] = f;
    cur = cand;
  }
  return h;
}
