// K4: 3D post-loop candidate filter (reference _extreme_vertex_mask,
// quickhull.py:136-164) and result assembly.
//
// The 3D round loop emits every true hull vertex plus some candidates that
// lie inside the hull (the farthest point of one face's outside set need
// not be extreme for the whole set).  The reference prunes them with a
// direction certificate, an eps-tolerant supporting-plane search and a
// HiGHS LP; its keep rule is, up to eps: keep v iff v is not inside the
// convex hull of the other candidates by more than eps.  On the device:
//
//   F0 k_f_setup    grid size from the candidate count m, reset the cells
//   F1 k_f_gather   candidate coordinates (discovery order) + bbox
//   F2 k_f_count    uniform G^3 grid (G = 4..64, ~4 candidates per cell):
//                   cell of each candidate, tight cell / superblock boxes
//   F3 k_f_scan     cell offsets (one block)
//   F4 k_f_scatter  candidates sorted by cell
//   F5 k_f_test     one warp per candidate:
//                     (1) certificate: no other candidate above the plane
//                         through v with normal v - bbox centre (+eps) -> keep
//                     (2) otherwise GJK on {c - v}: distance from v to the
//                         hull of the other candidates.  Outside -> keep;
//                         a tetrahedron of candidates containing v with
//                         every face farther than eps -> prune; anything
//                         closer than eps -> keep (the reference's
//                         eps-tolerant supporting plane keeps it too).
//                   Both use a branch-and-bound support query over the
//                   grid: a box is skipped when the monotone fp64 upper
//                   bound of d.(c - v) over it can not beat the best value
//                   (IEEE rounding is monotone, so the bound computed with
//                   the point formula's operation order is exact).
//   F6 k_f_compact  kept candidates -> user indices, discovery order kept
//                   (verts[extreme], quickhull.py:311)
// m <= 4 keeps everything (quickhull.py:148-149).
#pragma once

#include "sh_common.cuh"

namespace sh {

constexpr uint32_t ST_CAND_OVERFLOW = 7;
constexpr int FG_MAX = 64;   // grid cells per axis (max)
constexpr int FSB = 4;       // cells per superblock per axis
constexpr int F_TEST_BLOCK = 256;

struct FilterParams {
  uint32_t m, G, GS, ctr_test;
  double lo[3], inv_h[3], ctr[3];
  unsigned long long bb[6];  // candidate bbox, ordered bits: min x,y,z then max x,y,z
  uint32_t ambiguous, gjk_capped, pad0, pad1;
};

struct FilterWs {
  unsigned long long* result;  // [0] kept, [1] facets, [2] filter applied, [3] ambiguous
  int32_t* out_facets;
  int64_t facet_cap;
  uint32_t mcap;
  FilterParams* fp;
  double *cx, *cy, *cz;              // candidates, discovery order
  uint32_t* ccell;
  double *sx, *sy, *sz;              // candidates sorted by cell
  uint32_t* sid;                     // discovery index of sorted entry
  uint32_t *cell_cnt, *cell_start, *cell_cur;
  unsigned long long* cell_box;      // [cell][6] ordered bits
  unsigned long long* sb_box;        // [superblock][6]
  uint8_t* keep;
};

static inline int filter_alloc(FilterWs& f, uint64_t mcap) {
  bool ok = true;
  auto A = [&](void** p, size_t b) { ok &= cudaMalloc(p, b + 64) == cudaSuccess; };
  const size_t cells = (size_t)FG_MAX * FG_MAX * FG_MAX;
  const size_t sbs = cells / (FSB * FSB * FSB);
  A((void**)&f.result, 64);
  A((void**)&f.fp, sizeof(FilterParams));
  A((void**)&f.cx, mcap * 8);
  A((void**)&f.cy, mcap * 8);
  A((void**)&f.cz, mcap * 8);
  A((void**)&f.sx, mcap * 8);
  A((void**)&f.sy, mcap * 8);
  A((void**)&f.sz, mcap * 8);
  A((void**)&f.ccell, mcap * 4);
  A((void**)&f.sid, mcap * 4);
  A((void**)&f.keep, mcap);
  A((void**)&f.cell_cnt, cells * 4);
  A((void**)&f.cell_start, (cells + 1) * 4);
  A((void**)&f.cell_cur, cells * 4);
  A((void**)&f.cell_box, cells * 48);
  A((void**)&f.sb_box, sbs * 48);
  f.mcap = (uint32_t)mcap;
  return ok ? 0 : 1;
}

static inline void filter_free(FilterWs& f) {
  void* ps[] = {f.result, f.fp, f.cx, f.cy, f.cz, f.sx, f.sy, f.sz, f.ccell, f.sid, f.keep,
                f.cell_cnt, f.cell_start, f.cell_cur, f.cell_box, f.sb_box};
  for (void* p : ps)
    if (p) cudaFree(p);
  int32_t* of = f.out_facets;
  int64_t fc = f.facet_cap;
  f = FilterWs{};
  f.out_facets = of;
  f.facet_cap = fc;
}

static inline int filter_set_params(FilterWs& f, int32_t* facets, int64_t cap, cudaStream_t s) {
  (void)s;
  f.out_facets = facets;
  f.facet_cap = cap;
  return 0;
}

__device__ __forceinline__ unsigned long long obits(double d) { return ordered_bits(d); }
__device__ __forceinline__ double ofrom(unsigned long long b) { return from_ordered_bits(b); }

__device__ __forceinline__ uint32_t f_grid_of(uint32_t m) {
  // ~4 candidates per cell, G a multiple of the superblock edge
  double g = cbrt((double)m / 4.0);
  uint32_t G = (uint32_t)(FSB * ceil(g / FSB));
  return G < FSB ? FSB : (G > FG_MAX ? FG_MAX : G);
}

// ------------------------------------------------------------------ F0
__global__ void __launch_bounds__(BLOCK) k_f_setup(Workspace ws, FilterWs f) {
  DevState* st = ws.st;
  uint32_t m = st->h_final;
  if (m > f.mcap) m = 0;  // overflow: reported below, nothing else runs
  const uint32_t G = f_grid_of(m), GS = G / FSB;
  const uint32_t cells = G * G * G, sbs = GS * GS * GS;
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x, T = gridDim.x * blockDim.x;
  for (uint32_t c = tid; c < cells; c += T) {
    f.cell_cnt[c] = 0;
#pragma unroll
    for (int k = 0; k < 3; k++) {
      f.cell_box[(size_t)c * 6 + k] = ~0ull;
      f.cell_box[(size_t)c * 6 + 3 + k] = 0ull;
    }
  }
  for (uint32_t c = tid; c < sbs; c += T) {
#pragma unroll
    for (int k = 0; k < 3; k++) {
      f.sb_box[(size_t)c * 6 + k] = ~0ull;
      f.sb_box[(size_t)c * 6 + 3 + k] = 0ull;
    }
  }
  if (tid == 0) {
    FilterParams* P = f.fp;
    P->m = m;
    P->G = G;
    P->GS = GS;
    P->ctr_test = 0;
    P->ambiguous = 0;
    P->gjk_capped = 0;
    for (int k = 0; k < 3; k++) {
      P->bb[k] = ~0ull;
      P->bb[3 + k] = 0ull;
    }
    if (st->h_final > f.mcap) {
      st->status = ST_CAND_OVERFLOW;
      st->seg_needed = st->h_final;
    }
  }
}

// ------------------------------------------------------------------ F1
__global__ void __launch_bounds__(BLOCK) k_f_gather(Workspace ws, FilterWs f) {
  DevState* st = ws.st;
  const uint32_t m = f.fp->m;
  const int64_t stride = st->stride;
  unsigned long long lo[3] = {~0ull, ~0ull, ~0ull}, hi[3] = {0, 0, 0};
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    uint32_t q = ws.vout[i];
    double c[3] = {ld_coord(st->px, stride, q), ld_coord(st->py, stride, q),
                   ld_coord(st->pz, stride, q)};
    f.cx[i] = c[0];
    f.cy[i] = c[1];
    f.cz[i] = c[2];
#pragma unroll
    for (int k = 0; k < 3; k++) {
      unsigned long long b = obits(c[k]);
      lo[k] = b < lo[k] ? b : lo[k];
      hi[k] = b > hi[k] ? b : hi[k];
    }
  }
#pragma unroll
  for (int k = 0; k < 3; k++) {
    for (int o = 16; o; o >>= 1) {
      unsigned long long a = __shfl_xor_sync(0xFFFFFFFFu, lo[k], o);
      unsigned long long b = __shfl_xor_sync(0xFFFFFFFFu, hi[k], o);
      lo[k] = a < lo[k] ? a : lo[k];
      hi[k] = b > hi[k] ? b : hi[k];
    }
  }
  if ((threadIdx.x & 31) == 0 && lo[0] != ~0ull) {
#pragma unroll
    for (int k = 0; k < 3; k++) {
      atomicMin(&f.fp->bb[k], lo[k]);
      atomicMax(&f.fp->bb[3 + k], hi[k]);
    }
  }
}

// ------------------------------------------------------------------ F2
struct GridGeom {
  double lo[3], inv_h[3];
  uint32_t G, GS;
};

__device__ __forceinline__ GridGeom f_geom(const FilterParams* P) {
  GridGeom g;
  g.G = P->G;
  g.GS = P->GS;
#pragma unroll
  for (int k = 0; k < 3; k++) {
    double lo = ofrom(P->bb[k]), hi = ofrom(P->bb[3 + k]);
    g.lo[k] = lo;
    g.inv_h[k] = (hi > lo) ? (double)g.G / (hi - lo) : 0.0;
  }
  return g;
}

__device__ __forceinline__ uint32_t f_axis_cell(const GridGeom& g, int k, double x) {
  double t = (x - g.lo[k]) * g.inv_h[k];
  int c = (int)t;
  return (uint32_t)(c < 0 ? 0 : (c >= (int)g.G ? (int)g.G - 1 : c));
}

__global__ void __launch_bounds__(BLOCK) k_f_count(Workspace ws, FilterWs f) {
  const FilterParams* P = f.fp;
  const uint32_t m = P->m;
  const GridGeom g = f_geom(P);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    for (int k = 0; k < 3; k++) {
      double lo = ofrom(P->bb[k]), hi = ofrom(P->bb[3 + k]);
      f.fp->lo[k] = lo;
      f.fp->inv_h[k] = g.inv_h[k];
      f.fp->ctr[k] = 0.5 * lo + 0.5 * hi;
    }
  }
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    double c[3] = {f.cx[i], f.cy[i], f.cz[i]};
    uint32_t a[3];
#pragma unroll
    for (int k = 0; k < 3; k++) a[k] = f_axis_cell(g, k, c[k]);
    uint32_t cell = (a[2] * g.G + a[1]) * g.G + a[0];
    uint32_t sb = ((a[2] / FSB) * g.GS + a[1] / FSB) * g.GS + a[0] / FSB;
    f.ccell[i] = cell;
    atomicAdd(&f.cell_cnt[cell], 1u);
#pragma unroll
    for (int k = 0; k < 3; k++) {
      unsigned long long b = obits(c[k]);
      atomicMin(&f.cell_box[(size_t)cell * 6 + k], b);
      atomicMax(&f.cell_box[(size_t)cell * 6 + 3 + k], b);
      atomicMin(&f.sb_box[(size_t)sb * 6 + k], b);
      atomicMax(&f.sb_box[(size_t)sb * 6 + 3 + k], b);
    }
  }
}

// ------------------------------------------------------------------ F3
__global__ void __launch_bounds__(1024) k_f_scan(FilterWs f) {
  __shared__ uint32_t s_w[32];
  __shared__ uint32_t s_carry;
  const uint32_t G = f.fp->G;
  const uint32_t cells = G * G * G;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (uint32_t base = 0; base < cells; base += 1024) {
    uint32_t c = base + threadIdx.x;
    uint32_t v = c < cells ? f.cell_cnt[c] : 0u;
    uint32_t x = v;
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_w[warp] = x;
    __syncthreads();
    if (warp == 0) {
      uint32_t w = s_w[lane], y = w;
      for (int o = 1; o < 32; o <<= 1) {
        uint32_t z = __shfl_up_sync(0xFFFFFFFFu, y, o);
        if (lane >= o) y += z;
      }
      s_w[lane] = y - w;
    }
    __syncthreads();
    uint32_t ex = s_carry + s_w[warp] + x - v;
    if (c < cells) {
      f.cell_start[c] = ex;
      f.cell_cur[c] = ex;
    }
    __syncthreads();
    if (threadIdx.x == 1023) s_carry = ex + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) f.cell_start[cells] = s_carry;
}

// ------------------------------------------------------------------ F4
__global__ void __launch_bounds__(BLOCK) k_f_scatter(FilterWs f) {
  const uint32_t m = f.fp->m;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    uint32_t p = atomicAdd(&f.cell_cur[f.ccell[i]], 1u);
    f.sx[p] = f.cx[i];
    f.sy[p] = f.cy[i];
    f.sz[p] = f.cz[i];
    f.sid[p] = i;
  }
}

// ------------------------------------------------------------------ F5
struct V3 {
  double x, y, z;
};
__device__ __forceinline__ V3 v3(double x, double y, double z) { V3 r; r.x = x; r.y = y; r.z = z; return r; }
__device__ __forceinline__ V3 vsub(V3 a, V3 b) { return v3(sub(a.x, b.x), sub(a.y, b.y), sub(a.z, b.z)); }
__device__ __forceinline__ V3 vadd(V3 a, V3 b) { return v3(add(a.x, b.x), add(a.y, b.y), add(a.z, b.z)); }
__device__ __forceinline__ V3 vscale(V3 a, double s) { return v3(mul(a.x, s), mul(a.y, s), mul(a.z, s)); }
__device__ __forceinline__ double vdot(V3 a, V3 b) {
  return add(add(mul(a.x, b.x), mul(a.y, b.y)), mul(a.z, b.z));
}
__device__ __forceinline__ V3 vcross(V3 u, V3 v) {
  V3 r;
  cross3(u.x, u.y, u.z, v.x, v.y, v.z, &r.x, &r.y, &r.z);
  return r;
}
__device__ __forceinline__ V3 vneg(V3 a) { return v3(-a.x, -a.y, -a.z); }

// max over the box of d.(c - v), evaluated with the point formula's order
__device__ __forceinline__ double box_bound(const unsigned long long* b, V3 d, V3 v) {
  double lo0 = ofrom(b[0]), lo1 = ofrom(b[1]), lo2 = ofrom(b[2]);
  double hi0 = ofrom(b[3]), hi1 = ofrom(b[4]), hi2 = ofrom(b[5]);
  double t0 = fmax(mul(d.x, sub(lo0, v.x)), mul(d.x, sub(hi0, v.x)));
  double t1 = fmax(mul(d.y, sub(lo1, v.y)), mul(d.y, sub(hi1, v.y)));
  double t2 = fmax(mul(d.z, sub(lo2, v.z)), mul(d.z, sub(hi2, v.z)));
  return add(add(t0, t1), t2);
}

struct Sup {
  double val;    // d.(c - v) of the best candidate (-inf if none)
  uint32_t pos;  // sorted position
  uint32_t id;   // discovery index
};

__device__ __forceinline__ void sup_merge(Sup& a, double val, uint32_t pos, uint32_t id) {
  if (val > a.val || (val == a.val && id < a.id)) {
    a.val = val;
    a.pos = pos;
    a.id = id;
  }
}

// Scan the points of one cell (warp-cooperative), updating `best`.
// first_hit: stop at the first value > thr (existence query).
__device__ __forceinline__ bool scan_cell(const FilterWs& f, uint32_t cell, V3 d, V3 v, uint32_t self,
                                          double thr, bool first_hit, Sup& best) {
  const int lane = threadIdx.x & 31;
  const uint32_t s0 = f.cell_start[cell], s1 = f.cell_start[cell + 1];
  for (uint32_t p0 = s0; p0 < s1; p0 += 32) {
    uint32_t p = p0 + lane;
    double val = -INFINITY;
    uint32_t id = 0xFFFFFFFFu;
    if (p < s1) {
      id = f.sid[p];
      if (id != self) {
        V3 c = v3(f.sx[p], f.sy[p], f.sz[p]);
        val = vdot(d, vsub(c, v));
      }
    }
    Sup s;
    s.val = val;
    s.pos = p;
    s.id = id;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      double ov = __shfl_xor_sync(0xFFFFFFFFu, s.val, o);
      uint32_t op = __shfl_xor_sync(0xFFFFFFFFu, s.pos, o);
      uint32_t oi = __shfl_xor_sync(0xFFFFFFFFu, s.id, o);
      sup_merge(s, ov, op, oi);
    }
    sup_merge(best, s.val, s.pos, s.id);
    if (first_hit && best.val > thr) return true;
  }
  return false;
}

__device__ __forceinline__ bool scan_superblock(const FilterWs& f, const GridGeom& g, uint32_t sb, V3 d,
                                                V3 v, uint32_t self, double thr, bool first_hit,
                                                Sup& best) {
  const int lane = threadIdx.x & 31;
  const uint32_t GS = g.GS, G = g.G;
  const uint32_t bx = sb % GS, by = (sb / GS) % GS, bz = sb / (GS * GS);
#pragma unroll 1
  for (int half = 0; half < 2; half++) {
    const uint32_t l = half * 32 + lane;  // 64 cells per superblock
    const uint32_t cell = ((bz * FSB + l / 16) * G + (by * FSB + (l / 4) % 4)) * G + bx * FSB + l % 4;
    double bnd = -INFINITY;
    if (f.cell_box[(size_t)cell * 6] != ~0ull) bnd = box_bound(&f.cell_box[(size_t)cell * 6], d, v);
    const double floor_ = first_hit ? thr : best.val;
    uint32_t mask = __ballot_sync(0xFFFFFFFFu, bnd > floor_ || (!first_hit && bnd == floor_ && bnd > -INFINITY));
    while (mask) {
      const int src = __ffs(mask) - 1;
      mask &= mask - 1;
      const double cb = __shfl_sync(0xFFFFFFFFu, bnd, src);
      const uint32_t cc = __shfl_sync(0xFFFFFFFFu, cell, src);
      if (!first_hit && cb < best.val) continue;
      if (scan_cell(f, cc, d, v, self, thr, first_hit, best)) return true;
    }
  }
  return false;
}

// Branch-and-bound support query: max over candidates c != self of d.(c-v).
__device__ Sup support_query(const FilterWs& f, const GridGeom& g, V3 d, V3 v, uint32_t self, double thr,
                             bool first_hit) {
  const int lane = threadIdx.x & 31;
  const uint32_t nsb = g.GS * g.GS * g.GS;
  Sup best;
  best.val = -INFINITY;
  best.pos = 0xFFFFFFFFu;
  best.id = 0xFFFFFFFFu;
  // pass 1: the superblock with the largest bound first (tightens `best`)
  double mb = -INFINITY;
  uint32_t msb = 0xFFFFFFFFu;
  for (uint32_t s0 = 0; s0 < nsb; s0 += 32) {
    uint32_t sb = s0 + lane;
    double b = -INFINITY;
    if (sb < nsb && f.sb_box[(size_t)sb * 6] != ~0ull) b = box_bound(&f.sb_box[(size_t)sb * 6], d, v);
    if (b > mb) {
      mb = b;
      msb = sb;
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    double ob = __shfl_xor_sync(0xFFFFFFFFu, mb, o);
    uint32_t os = __shfl_xor_sync(0xFFFFFFFFu, msb, o);
    if (ob > mb || (ob == mb && os < msb)) {
      mb = ob;
      msb = os;
    }
  }
  if (msb == 0xFFFFFFFFu) return best;
  if (first_hit && !(mb > thr)) return best;
  if (scan_superblock(f, g, msb, d, v, self, thr, first_hit, best)) return best;
  // pass 2: every other superblock that can still win
  for (uint32_t s0 = 0; s0 < nsb; s0 += 32) {
    uint32_t sb = s0 + lane;
    double b = -INFINITY;
    if (sb < nsb && sb != msb && f.sb_box[(size_t)sb * 6] != ~0ull)
      b = box_bound(&f.sb_box[(size_t)sb * 6], d, v);
    const double floor_ = first_hit ? thr : best.val;
    uint32_t mask = __ballot_sync(0xFFFFFFFFu, b > floor_ || (!first_hit && b == floor_ && b > -INFINITY));
    while (mask) {
      const int src = __ffs(mask) - 1;
      mask &= mask - 1;
      const double bb = __shfl_sync(0xFFFFFFFFu, b, src);
      const uint32_t ss = s0 + src;
      if (!first_hit && bb < best.val) continue;
      if (scan_superblock(f, g, ss, d, v, self, thr, first_hit, best)) return best;
    }
  }
  return best;
}

// Closest point to the origin on segment / triangle (Ericson, Real-Time
// Collision Detection 5.1.2 / 5.1.5 with p = 0).  Keeps in W only the
// vertices of the feature the closest point lies on.
__device__ __forceinline__ V3 closest_seg(V3* W, uint32_t* id, int& n) {
  V3 a = W[0], b = W[1];
  V3 ab = vsub(b, a);
  double t = -vdot(a, ab), den = vdot(ab, ab);
  if (t <= 0.0 || den <= 0.0) {
    n = 1;
    return a;
  }
  if (t >= den) {
    W[0] = b;
    id[0] = id[1];
    n = 1;
    return b;
  }
  return vadd(a, vscale(ab, t / den));
}

__device__ __forceinline__ V3 closest_tri(V3* W, uint32_t* id, int& n) {
  V3 a = W[0], b = W[1], c = W[2];
  V3 ab = vsub(b, a), ac = vsub(c, a), ap = vneg(a);
  double d1 = vdot(ab, ap), d2 = vdot(ac, ap);
  if (d1 <= 0.0 && d2 <= 0.0) {
    n = 1;
    return a;
  }
  V3 bp = vneg(b);
  double d3 = vdot(ab, bp), d4 = vdot(ac, bp);
  if (d3 >= 0.0 && d4 <= d3) {
    W[0] = b;
    id[0] = id[1];
    n = 1;
    return b;
  }
  double vc = d1 * d4 - d3 * d2;
  if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) {
    double t = d1 / (d1 - d3);
    n = 2;
    return vadd(a, vscale(ab, t));
  }
  V3 cp = vneg(c);
  double d5 = vdot(ab, cp), d6 = vdot(ac, cp);
  if (d6 >= 0.0 && d5 <= d6) {
    W[0] = c;
    id[0] = id[2];
    n = 1;
    return c;
  }
  double vb = d5 * d2 - d1 * d6;
  if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {
    double t = d2 / (d2 - d6);
    W[1] = c;
    id[1] = id[2];
    n = 2;
    return vadd(a, vscale(ac, t));
  }
  double va = d3 * d6 - d5 * d4;
  if (va <= 0.0 && (d4 - d3) >= 0.0 && (d5 - d6) >= 0.0) {
    double t = (d4 - d3) / ((d4 - d3) + (d5 - d6));
    W[0] = b;
    id[0] = id[1];
    W[1] = c;
    id[1] = id[2];
    n = 2;
    return vadd(b, vscale(vsub(c, b), t));
  }
  double den = 1.0 / (va + vb + vc);
  n = 3;
  return vadd(a, vadd(vscale(ab, vb * den), vscale(ac, vc * den)));
}

// Tetrahedron: returns true when the origin is inside (W unchanged, n = 4);
// otherwise the closest face feature.  `degenerate` set for a flat tetra.
__device__ __forceinline__ bool closest_tet(V3* W, uint32_t* id, int& n, V3& x, bool& degenerate) {
  const int F[4][4] = {{0, 1, 2, 3}, {0, 2, 3, 1}, {0, 3, 1, 2}, {1, 3, 2, 0}};
  double best = INFINITY;
  V3 bx = x;
  V3 bW[3];
  uint32_t bid[3];
  int bn = 0;
  bool any_out = false;
  degenerate = false;
#pragma unroll 1
  for (int f = 0; f < 4; f++) {
    V3 a = W[F[f][0]], b = W[F[f][1]], c = W[F[f][2]], d = W[F[f][3]];
    V3 nrm = vcross(vsub(b, a), vsub(c, a));
    double sp = -vdot(nrm, a);          // origin side
    double sd = vdot(nrm, vsub(d, a));  // opposite vertex side
    if (sd == 0.0) {
      degenerate = true;
      return false;
    }
    if (sp * sd < 0.0) {
      any_out = true;
      V3 T[3] = {a, b, c};
      uint32_t Ti[3] = {id[F[f][0]], id[F[f][1]], id[F[f][2]]};
      int tn = 3;
      V3 q = closest_tri(T, Ti, tn);
      double dq = vdot(q, q);
      if (dq < best) {
        best = dq;
        bx = q;
        bn = tn;
        for (int k = 0; k < tn; k++) {
          bW[k] = T[k];
          bid[k] = Ti[k];
        }
      }
    }
  }
  if (!any_out) {
    n = 4;
    return true;
  }
  for (int k = 0; k < bn; k++) {
    W[k] = bW[k];
    id[k] = bid[k];
  }
  n = bn;
  x = bx;
  return false;
}

// smallest distance from the origin to a face plane of the tetrahedron W
__device__ __forceinline__ double tet_depth(const V3* W) {
  const int F[4][3] = {{0, 1, 2}, {0, 2, 3}, {0, 3, 1}, {1, 3, 2}};
  double dmin = INFINITY;
  for (int f = 0; f < 4; f++) {
    V3 a = W[F[f][0]], b = W[F[f][1]], c = W[F[f][2]];
    V3 nrm = vcross(vsub(b, a), vsub(c, a));
    double nl = sqrt_(vdot(nrm, nrm));
    double dd = fabs(vdot(nrm, a)) / nl;
    dmin = fmin(dmin, dd);
  }
  return dmin;
}

// 1 keep, 0 prune; *amb set when kept only because v is within eps of the
// boundary of the other candidates' hull (or the iteration cap was hit).
__device__ int f_decide(const FilterWs& f, const GridGeom& g, uint32_t i, V3 v, V3 ctr, double eps,
                        int* amb, int* capped) {
  V3 w0 = vsub(v, ctr);
  double wl = sqrt_(vdot(w0, w0));
  if (!(wl > 0.0)) {
    w0 = v3(1.0, 0.0, 0.0);
    wl = 1.0;
  }
  // (1) certificate along v - centre
  const double thr0 = mul(eps, wl);
  Sup s = support_query(f, g, w0, v, i, thr0, true);
  if (!(s.val > thr0)) return 1;
  // (2) GJK on U = {c - v : c != v}
  V3 W[4];
  uint32_t id[4];
  int n = 1;
  W[0] = vsub(v3(f.sx[s.pos], f.sy[s.pos], f.sz[s.pos]), v);
  id[0] = s.id;
  V3 x = W[0];
#pragma unroll 1
  for (int it = 0; it < 64; it++) {
    double xx = vdot(x, x);
    if (xx <= 0.0) {
      *amb = 1;
      return 1;
    }
    V3 dir = vneg(x);
    Sup q = support_query(f, g, dir, v, i, 0.0, false);
    if (q.pos == 0xFFFFFFFFu) return 1;
    // q.val = max_u (-x).u ; gap = x.x - min_u x.u = xx + q.val
    if (add(xx, q.val) <= 1e-13 * xx) return 1;  // origin outside: v is extreme
    for (int k = 0; k < n; k++)
      if (id[k] == q.id) return 1;               // no progress: outside
    W[n] = vsub(v3(f.sx[q.pos], f.sy[q.pos], f.sz[q.pos]), v);
    id[n] = q.id;
    n++;
    if (n == 2) {
      x = closest_seg(W, id, n);
    } else if (n == 3) {
      x = closest_tri(W, id, n);
    } else {
      bool degen = false;
      if (closest_tet(W, id, n, x, degen)) {
        if (tet_depth(W) > eps) return 0;        // strictly inside: prune
        *amb = 1;
        return 1;
      }
      if (degen) {
        *amb = 1;
        return 1;
      }
    }
    if (sqrt_(vdot(x, x)) <= eps) {
      *amb = 1;                                  // within eps of the boundary
      return 1;
    }
  }
  *capped = 1;
  return 1;
}

__global__ void __launch_bounds__(F_TEST_BLOCK) k_f_test(Workspace ws, FilterWs f) {
  const FilterParams* P = f.fp;
  const uint32_t m = P->m;
  const double eps = ws.st->eps;
  const GridGeom g = f_geom(P);
  const V3 ctr = v3(P->ctr[0], P->ctr[1], P->ctr[2]);
  const int lane = threadIdx.x & 31;
  int amb_count = 0, cap_count = 0;
  for (;;) {
    uint32_t i = 0;
    if (lane == 0) i = atomicAdd(&f.fp->ctr_test, 1u);
    i = __shfl_sync(0xFFFFFFFFu, i, 0);
    if (i >= m) break;
    int keep = 1, amb = 0, capped = 0;
    if (m > 4) keep = f_decide(f, g, i, v3(f.cx[i], f.cy[i], f.cz[i]), ctr, eps, &amb, &capped);
    if (lane == 0) {
      f.keep[i] = (uint8_t)keep;
      amb_count += amb;
      cap_count += capped;
    }
  }
  if (lane == 0 && amb_count) atomicAdd(&f.fp->ambiguous, (uint32_t)amb_count);
  if (lane == 0 && cap_count) atomicAdd(&f.fp->gjk_capped, (uint32_t)cap_count);
}

// ------------------------------------------------------------------ F6
__global__ void __launch_bounds__(1024) k_f_compact(Workspace ws, FilterWs f) {
  __shared__ uint32_t s_w[32];
  __shared__ uint32_t s_carry;
  const uint32_t m = f.fp->m;
  int64_t* out = ws.st->out_idx;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (uint32_t base = 0; base < m; base += 1024) {
    uint32_t i = base + threadIdx.x;
    uint32_t v = (i < m && f.keep[i]) ? 1u : 0u;
    uint32_t bal = __ballot_sync(0xFFFFFFFFu, v);
    if (lane == 0) s_w[warp] = __popc(bal);
    __syncthreads();
    if (warp == 0) {
      uint32_t w = s_w[lane], y = w;
      for (int o = 1; o < 32; o <<= 1) {
        uint32_t z = __shfl_up_sync(0xFFFFFFFFu, y, o);
        if (lane >= o) y += z;
      }
      s_w[lane] = y - w;
    }
    __syncthreads();
    uint32_t pos = s_carry + s_w[warp] + __popc(bal & lanemask_lt());
    if (v) out[pos] = (int64_t)ws.vout[i];
    __syncthreads();
    if (threadIdx.x == 1023) s_carry = pos + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    f.result[0] = s_carry;
    f.result[1] = 0;
    f.result[2] = 1;
    f.result[3] = f.fp->ambiguous;
  }
}

static inline int filter_launch(FilterWs& f, Workspace ws, int nsm, cudaStream_t s) {
  const int grid = nsm * 4;
  k_f_setup<<<grid, BLOCK, 0, s>>>(ws, f);
  k_f_gather<<<grid, BLOCK, 0, s>>>(ws, f);
  k_f_count<<<grid, BLOCK, 0, s>>>(ws, f);
  k_f_scan<<<1, 1024, 0, s>>>(f);
  k_f_scatter<<<grid, BLOCK, 0, s>>>(f);
  k_f_test<<<nsm * 8, F_TEST_BLOCK, 0, s>>>(ws, f);
  k_f_compact<<<1, 1024, 0, s>>>(ws, f);
  return cudaGetLastError() == cudaSuccess ? 0 : 10;
}

// vout (uint32, discovery order) -> user int64 indices (2D; 3D goes through
// the filter's compaction)
template <int DIM>
__global__ void __launch_bounds__(BLOCK) k_output(Workspace ws, FilterWs fw) {
  DevState* st = ws.st;
  uint32_t h = st->h_final;
  int64_t* out = st->out_idx;
  for (uint32_t i = blockIdx.x * BLOCK + threadIdx.x; i < h; i += gridDim.x * BLOCK)
    out[i] = (int64_t)ws.vout[i];
}

}  // namespace sh
