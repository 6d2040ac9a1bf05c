// Bit-exact fp64 numerics shared by every kernel (and by the host side of
// the library for the self-test entry points).
//
// The reference evaluates its predicates as separate numpy ufunc passes, so
// every product and sum is rounded on its own (no contraction).  This whole
// library is compiled with -fmad=false (device) and -ffp-contract=off (host);
// in addition the predicate helpers below use the explicit _rn intrinsics on
// the device so that a stray flag change can not silently fuse them.
//
// Reference operation orders followed here:
//   cross2         geometry.py:111-121   ax*(by-qy) + bx*(qy-ay) + qx*(ay-by), L->R
//   edge_length    geometry.py:124-127   np.hypot(bx-ax, by-ay) == glibc hypot
//   cross3         geometry.py:130-131   (uy*vz-uz*vy, uz*vx-ux*vz, ux*vy-uy*vx)
//   plane distance geometry.py:141-147   (nx*(qx-ax) + ny*(qy-ay)) + nz*(qz-az)
//   _norm3         geometry.py:159-160   sqrt((x*x + y*y) + z*z)
//   Tolerance      geometry.py:79-83     eps_rel * hypot.reduce(spans)
#pragma once

#include <stdint.h>
#include <math.h>

#if defined(__CUDACC__)
#define SH_HD __host__ __device__ __forceinline__
#else
#define SH_HD static inline
#endif

namespace sh {

#if defined(__CUDA_ARCH__)
SH_HD double mul(double a, double b) { return __dmul_rn(a, b); }
SH_HD double add(double a, double b) { return __dadd_rn(a, b); }
SH_HD double sub(double a, double b) { return __dsub_rn(a, b); }
SH_HD double div_(double a, double b) { return __ddiv_rn(a, b); }
SH_HD double sqrt_(double a) { return __dsqrt_rn(a); }
#else
SH_HD double mul(double a, double b) { volatile double r = a * b; return r; }
SH_HD double add(double a, double b) { volatile double r = a + b; return r; }
SH_HD double sub(double a, double b) { volatile double r = a - b; return r; }
SH_HD double div_(double a, double b) { return a / b; }
SH_HD double sqrt_(double a) { return sqrt(a); }
#endif

// glibc >= 2.35 hypot (sysdeps/ieee754/dbl-64/e_hypot.c, non-FMA kernel:
// Borges, "An Improved Algorithm for hypot(a,b)", corrected variant).  This
// is what np.hypot calls on the reference's host (glibc 2.39); SURVEY.md
// Appendix A.3 describes the port and its 40M-sample agreement.
SH_HD double hypot_kernel(double ax, double ay) {
  double h = sqrt_(add(mul(ax, ax), mul(ay, ay)));
  double t1, t2;
  if (h <= mul(2.0, ay)) {
    double delta = sub(h, ay);
    t1 = mul(ax, sub(mul(2.0, delta), ax));
    t2 = mul(sub(delta, mul(2.0, sub(ax, ay))), delta);
  } else {
    double delta = sub(h, ax);
    t1 = mul(mul(2.0, delta), sub(ax, mul(2.0, ay)));
    t2 = add(mul(sub(mul(4.0, delta), ay), ay), mul(delta, delta));
  }
  return sub(h, div_(add(t1, t2), mul(2.0, h)));
}

SH_HD double glibc_hypot(double x, double y) {
  const double SCALE = 0x1p-600;
  const double LARGE_VAL = 0x1p+511;
  const double TINY_VAL = 0x1p-459;  // keeps the kernel's squares and deltas normal
  const double EPS = 0x1p-54;
  if (!isfinite(x) || !isfinite(y)) {
    if (isinf(x) || isinf(y)) return INFINITY;
    return x + y;
  }
  x = fabs(x);
  y = fabs(y);
  double ax = x < y ? y : x;
  double ay = x < y ? x : y;
  if (ax > LARGE_VAL) {
    if (ay <= mul(ax, EPS)) return add(ax, ay);
    return div_(hypot_kernel(mul(ax, SCALE), mul(ay, SCALE)), SCALE);
  }
  if (ay < TINY_VAL) {
    if (ax >= div_(ay, EPS)) return add(ax, ay);
    return mul(hypot_kernel(div_(ax, SCALE), div_(ay, SCALE)), SCALE);
  }
  if (ay <= mul(ax, EPS)) return add(ax, ay);
  return hypot_kernel(ax, ay);
}

// geometry.py:111-121 -- symmetric three-product form, left to right.
SH_HD double cross2(double ax, double ay, double bx, double by, double qx, double qy) {
  return add(add(mul(ax, sub(by, qy)), mul(bx, sub(qy, ay))), mul(qx, sub(ay, by)));
}

// geometry.py:124-127
SH_HD double edge_length(double ax, double ay, double bx, double by) {
  return glibc_hypot(sub(bx, ax), sub(by, ay));
}

// geometry.py:130-131
SH_HD void cross3(double ux, double uy, double uz, double vx, double vy, double vz,
                  double* ox, double* oy, double* oz) {
  *ox = sub(mul(uy, vz), mul(uz, vy));
  *oy = sub(mul(uz, vx), mul(ux, vz));
  *oz = sub(mul(ux, vy), mul(uy, vx));
}

// geometry.py:134-138 face_normal: (b-a) x (c-a)
SH_HD void face_normal(const double* a, const double* b, const double* c, double* n) {
  cross3(sub(b[0], a[0]), sub(b[1], a[1]), sub(b[2], a[2]),
         sub(c[0], a[0]), sub(c[1], a[1]), sub(c[2], a[2]), &n[0], &n[1], &n[2]);
}

// geometry.py:141-147 / quickhull.py:376-377
SH_HD double plane_dist(const double* n, const double* a, double qx, double qy, double qz) {
  return add(add(mul(n[0], sub(qx, a[0])), mul(n[1], sub(qy, a[1]))), mul(n[2], sub(qz, a[2])));
}

// geometry.py:159-160 (also FaceTable.nlen, quickhull.py:72: identical bits)
SH_HD double norm3(const double* n) {
  return sqrt_(add(add(mul(n[0], n[0]), mul(n[1], n[1])), mul(n[2], n[2])));
}

// Order-preserving map fp64 -> u64 (after canonicalising -0.0 to +0.0, as
// segments.py:197 does with `values + 0.0`).  NaN is not expected: inputs
// are finite (geometry.py:38-40).
SH_HD uint64_t ordered_bits(double d) {
  d = add(d, 0.0);
#if defined(__CUDA_ARCH__)
  uint64_t b = (uint64_t)__double_as_longlong(d);
#else
  union { double f; uint64_t u; } cv; cv.f = d; uint64_t b = cv.u;
#endif
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

SH_HD double from_ordered_bits(uint64_t k) {
  uint64_t b = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
#if defined(__CUDA_ARCH__)
  return __longlong_as_double((long long)b);
#else
  union { double f; uint64_t u; } cv; cv.u = b; return cv.f;
#endif
}

// fl(Db / nb) > fl(Da / na) (nb, na > 0): the reference compares the
// rounded quotients (classify_three_faces, geometry.py:192-208).  When the
// cross products Db*na and Da*nb differ by more than 1e-14 of their size the
// exact quotients differ by far more than a rounding step, so the rounded
// ones compare the same way and no division is needed; otherwise divide.
SH_HD bool quotient_gt(double Db, double nb, double Da, double na) {
  const double p = mul(Db, na), r = mul(Da, nb);
  const double diff = sub(p, r);
  if (fabs(diff) > mul(1e-14, add(fabs(p), fabs(r)))) return diff > 0.0;
  return div_(Db, nb) > div_(Da, na);
}

#ifdef __CUDACC__
// The same, with the (rare) division fallback taken by the warp only when
// one of its lanes needs it: no per-lane divergence on the common path.
__device__ __forceinline__ bool quotient_gt_warp(double Db, double nb, double Da, double na) {
  const double p = mul(Db, na), r = mul(Da, nb);
  const double diff = sub(p, r);
  const bool sure = fabs(diff) > mul(1e-14, add(fabs(p), fabs(r)));
  bool gt = diff > 0.0;
  if (__any_sync(__activemask(), !sure)) gt = sure ? gt : (div_(Db, nb) > div_(Da, na));
  return gt;
}
#endif

}  // namespace sh
