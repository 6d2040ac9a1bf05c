// Exact orientation predicates with symbolic perturbation, for the 3D facet
// output (sh_facets3.cuh).
//
// The reference returns only the hull's vertex set (quickhull.py:282-446).
// The facet triples asked for by the north star (and pinned against Qhull's
// simplices) must be a consistent triangulation even
// when four or more vertices are coplanar (cube corners, lattices), so the
// facet builder decides every orientation exactly:
//
//   orient2d(a,b,c)   = det [[ax ay 1] [bx by 1] [cx cy 1]]
//   orient3d(a,b,c,d) = det [[ax ay az 1] ... [dx dy dz 1]]
//                     = det3(a-d, b-d, c-d)
//
//   1. fp64 evaluation with a forward error bound (Shewchuk's filter);
//   2. if that is inconclusive: the exact determinant in expansion
//      arithmetic (sums of non-overlapping doubles, two_sum / two_prod);
//   3. if that is exactly zero: Simulation of Simplicity (Edelsbrunner &
//      Muecke 1990).  Coordinate c of the point with index i is perturbed by
//      eps^(2^(d*i + d-1-c)); the sign of the perturbed determinant is the
//      sign of the first non-zero signed minor in the order of increasing
//      perturbation exponent.  The order only depends on the relative order
//      of the point indices, so every predicate sees one fixed perturbed,
//      general-position point set and the wrap yields a valid triangulation.
// Coordinates whose pairwise products underflow or overflow are outside the
// exactness guarantee (as for any fp64 predicate library).
#pragma once

#include "sh_numerics.cuh"

namespace sh {

// ------------------------------------------------------------ expansions
SH_HD void two_sum(double a, double b, double& x, double& y) {
  x = add(a, b);
  const double bv = sub(x, a);
  const double av = sub(x, bv);
  y = add(sub(a, av), sub(b, bv));
}

SH_HD void two_prod(double a, double b, double& x, double& y) {
  x = mul(a, b);
#if defined(__CUDA_ARCH__)
  y = __fma_rn(a, b, -x);
#else
  y = fma(a, b, -x);
#endif
}

// h = e + b (e non-overlapping, increasing magnitude); zero components
// dropped.  Returns the length of h (h may alias nothing).
SH_HD int grow_expansion(int elen, const double* e, double b, double* h) {
  double q = b;
  int k = 0;
  for (int i = 0; i < elen; i++) {
    double s, t;
    two_sum(q, e[i], s, t);
    q = s;
    if (t != 0.0) h[k++] = t;
  }
  if (q != 0.0 || k == 0) h[k++] = q;
  return k;
}

// h = e * b
SH_HD int scale_expansion(int elen, const double* e, double b, double* h) {
  int k = 0;
  double q, t;
  two_prod(e[0], b, q, t);
  if (t != 0.0) h[k++] = t;
  for (int i = 1; i < elen; i++) {
    double p1, p0, s, u;
    two_prod(e[i], b, p1, p0);
    two_sum(q, p0, s, u);
    if (u != 0.0) h[k++] = u;
    // fast_two_sum(p1, s): |p1| >= |s|
    q = add(p1, s);
    u = sub(s, sub(q, p1));
    if (u != 0.0) h[k++] = u;
  }
  if (q != 0.0 || k == 0) h[k++] = q;
  return k;
}

// h = h + f in place (h has room for hlen + flen components): growing an
// expansion writes component k only after reading component k, so the
// output may overwrite the input.
SH_HD int expansion_add(int hlen, double* h, int flen, const double* f) {
  for (int j = 0; j < flen; j++) hlen = grow_expansion(hlen, h, f[j], h);
  return hlen;
}

SH_HD int expansion_sign(int len, const double* e) {
  const double v = e[len - 1];  // most significant component
  return (v > 0.0) - (v < 0.0);
}

// ------------------------------------------------------- exact determinants
// m: k x k row-major, k <= 4.  Returns the exact sign.
SH_HD int det2_exact(double a, double b, double c, double d, double* out) {
  // a*d - b*c
  double x1, y1, x2, y2;
  two_prod(a, d, x1, y1);
  two_prod(b, c, x2, y2);
  double e[2] = {y1, x1};
  double t[4];
  int l = grow_expansion(2, e, -y2, t);
  return grow_expansion(l, t, -x2, out);
}

SH_HD int det3_exact(const double* m, double* out) {
  // along the first row: m00*C00 - m01*C01 + m02*C02 (out: >= 24 doubles)
  double d[4], sc[8];
  int al = 0;
  for (int j = 0; j < 3; j++) {
    const int c0 = (j == 0) ? 1 : 0, c1 = (j == 2) ? 1 : 2;
    const double f = (j == 1) ? -m[j] : m[j];
    if (f == 0.0) continue;
    const int dl = det2_exact(m[3 + c0], m[3 + c1], m[6 + c0], m[6 + c1], d);
    const int sl = scale_expansion(dl, d, f, sc);
    if (al == 0) {
      for (int i = 0; i < sl; i++) out[i] = sc[i];
      al = sl;
    } else {
      al = expansion_add(al, out, sl, sc);
    }
  }
  if (al == 0) {
    out[0] = 0.0;
    return 1;
  }
  return al;
}

// Exact sign of det(m), m k x k row-major, k <= 4.  For k == 4 the last
// column must be all ones (the orientation matrices): the determinant is
// expanded along it, a signed sum of four 3x3 coordinate determinants.
SH_HD int det_sign_exact(int k, const double* m) {
  if (k == 1) return (m[0] > 0.0) - (m[0] < 0.0);
  if (k == 2) {
    double o[4];
    int l = det2_exact(m[0], m[1], m[2], m[3], o);
    return expansion_sign(l, o);
  }
  if (k == 3) {
    double o[24];
    int l = det3_exact(m, o);
    return expansion_sign(l, o);
  }
  double acc[96], d3[24], minor[9];
  int al = 0;
  for (int r = 0; r < 4; r++) {
    int rr = 0;
    for (int i = 0; i < 4; i++) {
      if (i == r) continue;
      for (int c = 0; c < 3; c++) minor[rr * 3 + c] = m[i * 4 + c];
      rr++;
    }
    int dl = det3_exact(minor, d3);
    if ((r & 1) == 0)  // cofactor sign (-1)^(r + 3)
      for (int i = 0; i < dl; i++) d3[i] = -d3[i];
    if (al == 0) {
      for (int i = 0; i < dl; i++) acc[i] = d3[i];
      al = dl;
    } else {
      al = expansion_add(al, acc, dl, d3);
    }
  }
  return expansion_sign(al, acc);
}

// ------------------------------------------------- Simulation of Simplicity
// A perturbation term is a partial matching S of (row, coordinate column)
// pairs (distinct rows, distinct columns).  Its magnitude is
// eps^key(S), key(S) = sum of 2^(d*r + d-1-c); its coefficient in
// det(M + E) is (-1)^(sum r + sum c) * sgn(column order) * det(M minus the
// rows and columns of S) (generalised Laplace expansion).
struct SosTerm {
  uint8_t n;      // pairs in S
  uint8_t r[3];
  uint8_t c[3];
  int8_t sign;
  uint16_t key;
};

template <int D>
struct SosTable {
  static constexpr int kMax = (D == 3) ? 72 : 12;
  SosTerm t[kMax];
  int count;
};

template <int D>
constexpr SosTable<D> make_sos() {
  SosTable<D> T{};
  int cnt = 0;
  const int R = D + 1;
  // enumerate matchings of size 1..D: each row picks a column or none
  // (encode choice per row as 0 = none, 1 + c)
  int total = 1;
  for (int i = 0; i < R; i++) total *= (D + 1);
  for (int code = 1; code < total; code++) {
    int ch[4] = {0, 0, 0, 0};
    int x = code;
    for (int i = 0; i < R; i++) {
      ch[i] = x % (D + 1);
      x /= (D + 1);
    }
    bool ok = true;
    int used = 0, n = 0;
    for (int i = 0; i < R && ok; i++) {
      if (!ch[i]) continue;
      int bit = 1 << (ch[i] - 1);
      if (used & bit) ok = false;
      used |= bit;
      n++;
    }
    if (!ok || n == 0 || n > D) continue;
    SosTerm s{};
    s.n = (uint8_t)n;
    int k = 0, key = 0, par = 0;
    for (int i = 0; i < R; i++) {
      if (!ch[i]) continue;
      const int c = ch[i] - 1;
      s.r[k] = (uint8_t)i;
      s.c[k] = (uint8_t)c;
      key += 1 << (D * i + D - 1 - c);
      par += i + c;
      k++;
    }
    // sign of the column sequence (rows ascending) as a permutation
    int inv = 0;
    for (int a = 0; a < n; a++)
      for (int b = a + 1; b < n; b++)
        if (s.c[a] > s.c[b]) inv++;
    s.sign = (int8_t)((((par + inv) & 1) == 0) ? 1 : -1);
    s.key = (uint16_t)key;
    T.t[cnt++] = s;
  }
  // insertion sort by key (ascending = decreasing magnitude)
  for (int i = 1; i < cnt; i++) {
    SosTerm v = T.t[i];
    int j = i - 1;
    while (j >= 0 && T.t[j].key > v.key) {
      T.t[j + 1] = T.t[j];
      j--;
    }
    T.t[j + 1] = v;
  }
  T.count = cnt;
  return T;
}

#if defined(__CUDACC__)
__constant__ SosTable<2> c_sos2 = make_sos<2>();
__constant__ SosTable<3> c_sos3 = make_sos<3>();
#endif
static const SosTable<2> h_sos2 = make_sos<2>();
static const SosTable<3> h_sos3 = make_sos<3>();

template <int D>
SH_HD const SosTable<D>& sos_table() {
#if defined(__CUDA_ARCH__)
  if constexpr (D == 2) return c_sos2;
  else return c_sos3;
#else
  if constexpr (D == 2) return h_sos2;
  else return h_sos3;
#endif
}

// Sign of det [[p_i, 1]] (rows = D+1 points of dimension D, given in any
// order with their global indices) under the perturbation above.  Never 0
// for distinct indices.
template <int D>
#if defined(__CUDACC__)
__host__ __device__ __noinline__
#else
static
#endif
int orient_sos(const double* pts, const int64_t* ids) {
  constexpr int R = D + 1;
  // rows sorted by index; parity of the sort
  int ord[R];
  for (int i = 0; i < R; i++) ord[i] = i;
  int par = 0;
  for (int i = 1; i < R; i++)
    for (int j = i; j > 0 && ids[ord[j - 1]] > ids[ord[j]]; j--) {
      int t = ord[j];
      ord[j] = ord[j - 1];
      ord[j - 1] = t;
      par ^= 1;
    }
  double M[R * R];
  for (int i = 0; i < R; i++) {
    for (int c = 0; c < D; c++) M[i * R + c] = pts[ord[i] * D + c];
    M[i * R + D] = 1.0;
  }
  const int base = par ? -1 : 1;
  int s = det_sign_exact(R, M);
  if (s) return base * s;
  const SosTable<D>& T = sos_table<D>();
  double sub_m[R * R];
  for (int t = 0; t < T.count; t++) {
    const SosTerm& S = T.t[t];
    int rmask = 0, cmask = 0;
    for (int k = 0; k < S.n; k++) {
      rmask |= 1 << S.r[k];
      cmask |= 1 << S.c[k];
    }
    const int k2 = R - S.n;
    int ii = 0;
    for (int i = 0; i < R; i++) {
      if (rmask & (1 << i)) continue;
      int jj = 0;
      for (int c = 0; c < R; c++) {
        if (cmask & (1 << c)) continue;
        sub_m[ii * k2 + jj++] = M[i * R + c];
      }
      ii++;
    }
    s = det_sign_exact(k2, sub_m);
    if (s) return base * S.sign * s;
  }
  return 0;  // identical indices
}

// Filtered orient3d(a, b, c, d) sign with SoS ties (ids: global indices).
SH_HD int orient3d_exact(const double* a, const double* b, const double* c, const double* d, int64_t ia,
                         int64_t ib, int64_t ic, int64_t id) {
  const double adx = sub(a[0], d[0]), ady = sub(a[1], d[1]), adz = sub(a[2], d[2]);
  const double bdx = sub(b[0], d[0]), bdy = sub(b[1], d[1]), bdz = sub(b[2], d[2]);
  const double cdx = sub(c[0], d[0]), cdy = sub(c[1], d[1]), cdz = sub(c[2], d[2]);
  const double bc = sub(mul(bdx, cdy), mul(cdx, bdy));
  const double ca = sub(mul(cdx, ady), mul(adx, cdy));
  const double ab = sub(mul(adx, bdy), mul(bdx, ady));
  const double det = add(add(mul(adz, bc), mul(bdz, ca)), mul(cdz, ab));
  const double perm = add(add(mul(add(fabs(mul(bdx, cdy)), fabs(mul(cdx, bdy))), fabs(adz)),
                              mul(add(fabs(mul(cdx, ady)), fabs(mul(adx, cdy))), fabs(bdz))),
                          mul(add(fabs(mul(adx, bdy)), fabs(mul(bdx, ady))), fabs(cdz)));
  const double err = mul(7.8e-16, perm);  // > (7 + 56 eps) eps
  if (det > err) return 1;
  if (-det > err) return -1;
  double P[12] = {a[0], a[1], a[2], b[0], b[1], b[2], c[0], c[1], c[2], d[0], d[1], d[2]};
  int64_t I[4] = {ia, ib, ic, id};
  return orient_sos<3>(P, I);
}

SH_HD int orient2d_exact(const double* a, const double* b, const double* c, int64_t ia, int64_t ib, int64_t ic) {
  const double l = mul(sub(a[0], c[0]), sub(b[1], c[1]));
  const double r = mul(sub(a[1], c[1]), sub(b[0], c[0]));
  const double det = sub(l, r);
  const double err = mul(3.4e-16, add(fabs(l), fabs(r)));  // > (3 + 16 eps) eps
  if (det > err) return 1;
  if (-det > err) return -1;
  double P[6] = {a[0], a[1], b[0], b[1], c[0], c[1]};
  int64_t I[3] = {ia, ib, ic};
  return orient_sos<2>(P, I);
}

}  // namespace sh
