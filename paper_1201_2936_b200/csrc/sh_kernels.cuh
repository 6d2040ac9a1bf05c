// Kernels of the B200 Quickhull path (2D and 3D) around the round kernels,
// see DESIGN.md.
//
//   K0  k_first_reduce  bbox (-> eps, Tolerance.effective geometry.py:79-83)
//                       + lexicographic extremes (_lex_extreme quickhull.py:75-84);
//                       for a sharded hull also the slice's statistics, and
//                       k_shard_apply finishes it with the whole input's
//   K0b k_line_far      3D third corner: farthest from the extrema line
//                       (quickhull.py:329-344)
//   K1  k_first_count   first split (quickhull.py:200-222 / :346-364) as a
//                       counting pass: per side, survivors and farthest point
//   k_stats / k_stats_reduce / k_bbox: per-slice statistics of sharded hulls
//
// The round kernels are k_stream (sh_stream.cuh: round 1 fused with the
// first split, and every long round) and k_round (sh_round.cuh: the short
// rounds); the bookkeeping between rounds is k_book (sh_book.cuh).
#pragma once

#include "sh_common.cuh"

namespace sh {

// ------------------------------------------------------------------ K0
struct LexRec {
  double c[3];
  uint32_t idx;
  uint32_t pad;
};

template <int DIM>
__device__ __forceinline__ bool lex_less(const LexRec& a, const LexRec& b) {
  // a < b over (coords..., idx); fp comparisons, so -0.0 == +0.0 like
  // `vals == best` in _lex_extreme.
#pragma unroll
  for (int k = 0; k < DIM; k++) {
    if (a.c[k] < b.c[k]) return true;
    if (a.c[k] > b.c[k]) return false;
  }
  return a.idx < b.idx;
}

struct FirstRed {
  double lo[3], hi[3];
  LexRec mn, mx;  // lex-min (lowest idx among ties), lex-max (highest idx)
};

template <int DIM>
__device__ __forceinline__ void fr_merge(FirstRed& a, const FirstRed& b) {
#pragma unroll
  for (int k = 0; k < DIM; k++) {
    a.lo[k] = fmin(a.lo[k], b.lo[k]);
    a.hi[k] = fmax(a.hi[k], b.hi[k]);
  }
  if (lex_less<DIM>(b.mn, a.mn)) a.mn = b.mn;
  if (lex_less<DIM>(a.mx, b.mx)) a.mx = b.mx;
}

__device__ __forceinline__ FirstRed ld_cg_fr(const FirstRed* p) {
  FirstRed r;
  const double* s = reinterpret_cast<const double*>(p);
  double* d = reinterpret_cast<double*>(&r);
  for (int i = 0; i < (int)(sizeof(FirstRed) / 8); i++) d[i] = __ldcg(s + i);
  return r;
}

template <class T>
__device__ __forceinline__ T shfl_xor_t(T v, int m) {
  T r;
  const uint32_t* s = reinterpret_cast<const uint32_t*>(&v);
  uint32_t* d = reinterpret_cast<uint32_t*>(&r);
#pragma unroll
  for (int i = 0; i < (int)(sizeof(T) / 4); i++) d[i] = __shfl_xor_sync(0xFFFFFFFFu, s[i], m);
  return r;
}

// parameters of the first split (K1 + the root bookkeeping)
__device__ __forceinline__ void start_first_split(DevState* st) {
  RoundParams rp;
  rp.active = 1;
  rp.root = 1;
  rp.n_live = st->n;
  rp.nseg = 1;
  rp.cur = 0;
  rp.h = st->h_final;
  rp.round = 0;
  rp.n_true = st->n;
  rp.aligned = 0;
  rp.pad = 0;
  st->rp = rp;
}

template <int DIM>
__global__ void __launch_bounds__(BLOCK) k_init(Workspace ws) {
  DevState* st = ws.st;
  // Look-back status words carry a 16-bit launch tag; long before the tag
  // space wraps, zero the status arrays and restart the tags.
  if (st->seq % 65535u >= 32768u) {
    for (uint64_t i = threadIdx.x; i < ws.lb_book_words; i += blockDim.x) ws.lb_book[i] = 0;
    __syncthreads();
    if (threadIdx.x == 0) st->seq = 0;
    __threadfence();
    __syncthreads();
  }
  if (threadIdx.x < 4) ws.cursor[0][threadIdx.x] = 0;  // root children start at 0
  if (threadIdx.x == 0) {
    st->status = ST_OK;
    st->flags = 0;
    st->h_final = 0;
    st->rounds_final = 0;
    st->seg_needed = 0;
    st->first_active = 0;
    st->ctr_book = 0;
    st->arrive_book = 0;
    st->book_small = 1;
    st->nonfinite = 0;
    st->dead_round = 0;
    st->ctr_red = 0;
    st->dmax_bits = 0;
    st->rp.active = 0;
    ws.segstart[0][0] = 0;  // the root "parent" of the first split
    ws.segstart[0][1] = st->n;
  }
}

// K0's conclusion (one thread): eps (Tolerance.effective, geometry.py:
// 79-83; of the whole input's box for a sharded hull), the lexicographic
// extremes (quickhull.py:75-84; the global ones for a sharded hull) and the
// first split's parameters.
template <int DIM>
__device__ void finish_first_reduce(Workspace ws, FirstRed t) {
  DevState* st = ws.st;
  const uint32_t n = st->n;
  if (*(volatile uint32_t*)&st->nonfinite) {  // ContractViolation, nothing else runs
    st->status = ST_NONFINITE;
    st->h_final = 0;
    st->first_active = 0;
    return;
  }
  // Tolerance.effective: eps_rel * np.hypot.reduce(spans) -- of the whole
  // input's box when this is one slice of a sharded hull
  const double* gs = st->gstats;
  const uint32_t sf = gs ? st->shard_flags : 0u;
  double lo[3], hi[3];
#pragma unroll
  for (int k = 0; k < 3; k++) {
    lo[k] = (sf & SHARD_EPS) ? -gs[k] : t.lo[k];
    hi[k] = (sf & SHARD_EPS) ? gs[3 + k] : t.hi[k];
  }
  double acc = sub(hi[0], lo[0]);
#pragma unroll
  for (int k = 1; k < DIM; k++) acc = glibc_hypot(acc, sub(hi[k], lo[k]));
  double eps = st->use_eps_abs ? st->eps_abs : mul(st->eps_rel, acc);
  st->eps = eps;
  if (sf & SHARD_SPLIT) {
    // the first-split line through the global lexicographic extremes (hull
    // vertices of the whole input); one from another slice enters this
    // slice's hull as a virtual point with index n (min) / n + 1 (max)
    const int64_t off = st->gidx_offset;
#pragma unroll
    for (int e = 0; e < 2; e++) {
      const double* g = gs + 6 + 4 * e;
      const long long gi = (long long)g[3];
      LexRec& r = e ? t.mx : t.mn;
      if (gi != off + (long long)r.idx) {
#pragma unroll
        for (int k = 0; k < 3; k++) r.c[k] = g[k];
        r.idx = n + (uint32_t)e;
      }
    }
  }
  st->imin = t.mn.idx;
  st->imax = t.mx.idx;
  bool same = true;
#pragma unroll
  for (int k = 0; k < 3; k++) {
    st->pa[k] = t.mn.c[k];
    st->pb[k] = t.mx.c[k];
    if (k < DIM) same = same && (t.mn.c[k] == t.mx.c[k]);
  }
  ws.vout[0] = t.mn.idx;
  if (same) {  // quickhull.py:195-197 / :320-322 -- every point coincides
    st->h_final = 1;
    return;
  }
  ws.vout[1] = t.mx.idx;
  st->h_final = 2;
  if (DIM == 2) {
    // off_line threshold eps * edge_length(pmin, pmax), quickhull.py:203
    st->thr_line = mul(eps, edge_length(t.mn.c[0], t.mn.c[1], t.mx.c[0], t.mx.c[1]));
    st->first_active = 1;
    start_first_split(st);
  } else {
    st->first_active = (n > 2) ? 2u : 0u;  // 2: K0b runs next
  }
}

// Blocks a pass over the input uses: the whole grid for large inputs, fewer
// for small ones (>= 32 points per thread), so the per-block reductions,
// partials and atomics do not dominate a short pass.
__device__ __forceinline__ uint32_t first_pass_blocks(uint32_t n) {
  const uint32_t want = (uint32_t)(((uint64_t)n + BLOCK * 32u - 1) / (BLOCK * 32u));
  return want < 1u ? 1u : (want < gridDim.x ? want : gridDim.x);
}

template <int DIM>
__global__ void __launch_bounds__(BLOCK) k_first_reduce(Workspace ws) {
  DevState* st = ws.st;
  const uint32_t n = st->n;
  const uint32_t nb = first_pass_blocks(n);
  if (blockIdx.x >= nb) return;
  const int64_t stride = st->stride;
  const double* P[3] = {st->px, st->py, st->pz};
  FirstRed r;
#pragma unroll
  for (int k = 0; k < 3; k++) {
    r.lo[k] = INFINITY;
    r.hi[k] = -INFINITY;
    r.mn.c[k] = INFINITY;
    r.mx.c[k] = -INFINITY;
  }
  r.mn.idx = 0xFFFFFFFFu;
  r.mx.idx = 0;
  r.mn.pad = r.mx.pad = 0;
  // geometry.py:38-40, coordinates must be finite: NaN is caught here, an
  // infinity by the reduced box (below)
  bool nan_seen = false;
  auto visit = [&](const LexRec& q) {
    // x range = the lexicographic extremes' x (set after the loops); only a
    // point at or beyond them can replace them
#pragma unroll
    for (int k = 0; k < DIM; k++) {
      nan_seen |= q.c[k] != q.c[k];
      if (k > 0) {
        r.lo[k] = fmin(r.lo[k], q.c[k]);
        r.hi[k] = fmax(r.hi[k], q.c[k]);
      }
    }
    if (q.c[0] <= r.mn.c[0] && lex_less<DIM>(q, r.mn)) r.mn = q;
    if (q.c[0] >= r.mx.c[0] && lex_less<DIM>(r.mx, q)) r.mx = q;
  };
  const uint32_t G = nb * BLOCK;
  uint32_t i = blockIdx.x * BLOCK + threadIdx.x;
  bool aligned = stride == 1;
#pragma unroll
  for (int k = 0; k < DIM; k++) aligned = aligned && ((reinterpret_cast<uintptr_t>(P[k]) & 15) == 0);
  if (aligned) {
    // structure of arrays: 16-byte loads of point pairs, 4 pairs in flight
    const uint32_t npair = n / 2;
    uint32_t pi = blockIdx.x * BLOCK + threadIdx.x;
    for (; (uint64_t)pi + 3ull * G < npair; pi += 4 * G) {
      double2 v[4][3];
#pragma unroll
      for (int u = 0; u < 4; u++)
#pragma unroll
        for (int k = 0; k < DIM; k++) v[u][k] = __ldcs(reinterpret_cast<const double2*>(P[k]) + pi + u * G);
#pragma unroll
      for (int u = 0; u < 4; u++) {
        LexRec a, b2;
#pragma unroll
        for (int k = 0; k < 3; k++) {
          a.c[k] = (k < DIM) ? v[u][k].x : 0.0;
          b2.c[k] = (k < DIM) ? v[u][k].y : 0.0;
        }
        a.idx = 2 * (pi + u * G);
        b2.idx = a.idx + 1;
        a.pad = b2.pad = 0;
        visit(a);
        visit(b2);
      }
    }
    for (; pi < npair; pi += G) {
#pragma unroll
      for (int h = 0; h < 2; h++) {
        LexRec q;
#pragma unroll
        for (int k = 0; k < 3; k++) q.c[k] = (k < DIM) ? ld_coord(P[k], 1, 2 * pi + h) : 0.0;
        q.idx = 2 * pi + h;
        q.pad = 0;
        visit(q);
      }
    }
    i = (blockIdx.x == 0 && threadIdx.x == 0 && (n & 1)) ? n - 1 : n;  // odd tail
  }
  for (; (uint64_t)i + 3ull * G < n; i += 4 * G) {  // 4 independent loads in flight
    LexRec q[4];
#pragma unroll
    for (int u = 0; u < 4; u++) {
#pragma unroll
      for (int k = 0; k < 3; k++) q[u].c[k] = (k < DIM) ? ld_coord(P[k], stride, i + u * G) : 0.0;
      q[u].idx = i + u * G;
      q[u].pad = 0;
    }
#pragma unroll
    for (int u = 0; u < 4; u++) visit(q[u]);
  }
  for (; i < n; i += G) {
    LexRec q;
#pragma unroll
    for (int k = 0; k < 3; k++) q.c[k] = (k < DIM) ? ld_coord(P[k], stride, i) : 0.0;
    q.idx = i;
    q.pad = 0;
    visit(q);
  }
  if (nan_seen) st->nonfinite = 1;
  if (r.mn.idx != 0xFFFFFFFFu) {  // this thread saw a point
    r.lo[0] = r.mn.c[0];
    r.hi[0] = r.mx.c[0];
  }
  // block reduce
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) {
    FirstRed o = shfl_xor_t(r, m);
    fr_merge<DIM>(r, o);
  }
  __shared__ FirstRed s_w[WARPS];
  __shared__ bool s_last;
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) s_w[warp] = r;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < WARPS; w++) fr_merge<DIM>(s_w[0], s_w[w]);
    FirstRed* parts = reinterpret_cast<FirstRed*>(ws.red);
    parts[blockIdx.x] = s_w[0];
    __threadfence();
    uint32_t done = atomicAdd(&st->ctr_red, 1u);
    s_last = (done == nb - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  {  // last block: parallel reduction of the per-block partials
    const FirstRed* parts = reinterpret_cast<const FirstRed*>(ws.red);
    FirstRed t = r;
    bool any = false;
    for (uint32_t b = threadIdx.x; b < nb; b += BLOCK) {
      FirstRed o = ld_cg_fr(parts + b);
      if (!any) t = o;
      else fr_merge<DIM>(t, o);
      any = true;
    }
    if (!any) t = ld_cg_fr(parts);
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
      FirstRed o = shfl_xor_t(t, m);
      fr_merge<DIM>(t, o);
    }
    __syncthreads();
    if (lane == 0) s_w[warp] = t;
    __syncthreads();
    if (threadIdx.x != 0) return;
    for (int w = 1; w < WARPS; w++) fr_merge<DIM>(s_w[0], s_w[w]);
  }
  FirstRed t = s_w[0];
  st->ctr_red = 0;
#pragma unroll
  for (int k = 0; k < DIM; k++)
    if (!isfinite(t.lo[k]) || !isfinite(t.hi[k])) st->nonfinite = 1;  // an infinity
  __threadfence();
  if (st->stats_out) {  // this slice's statistics (sh_hull_shard_begin)
    double* o = st->stats_out;
    const int64_t off = st->gidx_offset;
#pragma unroll
    for (int k = 0; k < 3; k++) {
      o[k] = k < DIM ? -t.lo[k] : 0.0;
      o[3 + k] = k < DIM ? t.hi[k] : 0.0;
      o[6 + k] = t.mn.c[k];
      o[10 + k] = t.mx.c[k];
    }
    o[9] = (double)(off + (int64_t)t.mn.idx);
    o[13] = (double)(off + (int64_t)t.mx.idx);
  }
  if (st->defer_first) {  // k_shard_apply finishes with the whole input's statistics
#pragma unroll
    for (int k = 0; k < 3; k++) {
      st->keep_lo[k] = t.lo[k];
      st->keep_hi[k] = t.hi[k];
      st->keep_mn[k] = t.mn.c[k];
      st->keep_mx[k] = t.mx.c[k];
    }
    st->keep_imn = t.mn.idx;
    st->keep_imx = t.mx.idx;
    return;
  }
  finish_first_reduce<DIM>(ws, t);
}

// Stage 2 of a two-stage sharded hull: K0's kept reduction + the whole
// input's statistics (st->gstats) -> eps and the first split.
template <int DIM>
__global__ void k_shard_apply(Workspace ws) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  DevState* st = ws.st;
  FirstRed t;
#pragma unroll
  for (int k = 0; k < 3; k++) {
    t.lo[k] = st->keep_lo[k];
    t.hi[k] = st->keep_hi[k];
    t.mn.c[k] = st->keep_mn[k];
    t.mx.c[k] = st->keep_mx[k];
  }
  t.mn.idx = st->keep_imn;
  t.mx.idx = st->keep_imx;
  t.mn.pad = t.mx.pad = 0;
  finish_first_reduce<DIM>(ws, t);
}

// ------------------------------------------------------------------ K1
// The first split (quickhull.py:200-222 / :346-364) as a counting pass:
// per side, the number of points kept and the farthest one (largest
// distance, lowest index among ties).  Nothing per point is written; round
// 1 (k_round<MODE_ROUND1>) re-derives the split from the input.
struct SideAgg {
  uint32_t cnt[2];
  unsigned long long hi[2];
  uint32_t idx[2];
};

template <int DIM>
__global__ void __launch_bounds__(BLOCK) k_first_count(Workspace ws) {
  DevState* st = ws.st;
  const RoundParams rp = st->rp;
  if (!rp.active || !rp.root) return;
  const uint32_t nb = first_pass_blocks(st->n);
  if (blockIdx.x >= nb) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->ctr_book = 0;
    st->arrive_book = 0;
    st->book_small = 1;
  }
  const uint32_t n = st->n;
  const int64_t stride = st->stride;
  const double pa0 = st->pa[0], pa1 = st->pa[1], pa2 = st->pa[2];
  const double pb0 = st->pb[0], pb1 = st->pb[1];
  const double n0 = st->nrm[0], n1 = st->nrm[1], n2 = st->nrm[2];
  const double thr = st->thr_line;
  const uint32_t imin = st->imin, imax = st->imax, ifar = (DIM == 3) ? st->ifar : 0xFFFFFFFFu;
  SideAgg a;
  a.cnt[0] = a.cnt[1] = 0;
  a.hi[0] = a.hi[1] = 0ull;
  a.idx[0] = a.idx[1] = 0xFFFFFFFFu;
  double dmax = 0.0;
  auto visit = [&](uint32_t i, double x, double y, double z) {
    if (i == imin || i == imax || i == ifar) return;
    int s;
    double dn;
    if (DIM == 2) {
      const double d = cross2(pa0, pa1, pb0, pb1, x, y);
      if (!(fabs(d) > thr)) return;
      s = d < 0 ? 1 : 0;
      dn = s ? -d : d;
    } else {
      const double nn[3] = {n0, n1, n2}, pp[3] = {pa0, pa1, pa2};
      const double d = plane_dist(nn, pp, x, y, z);
      dmax = fmax(dmax, fabs(d));
      s = d < thr ? 1 : 0;
      dn = s ? -d : d;
    }
    const unsigned long long k = ordered_bits(dn);
    // indices arrive in increasing order per thread: strict > keeps the lowest
    if (s == 0) {
      a.cnt[0]++;
      if (k > a.hi[0]) { a.hi[0] = k; a.idx[0] = i; }
    } else {
      a.cnt[1]++;
      if (k > a.hi[1]) { a.hi[1] = k; a.idx[1] = i; }
    }
  };
  const double* P[3] = {st->px, st->py, st->pz};
  bool aligned = stride == 1;
#pragma unroll
  for (int k = 0; k < DIM; k++) aligned = aligned && ((reinterpret_cast<uintptr_t>(P[k]) & 15) == 0);
  const uint32_t G = nb * BLOCK;
  uint32_t i = blockIdx.x * BLOCK + threadIdx.x;
  if (aligned) {
    const uint32_t npair = n / 2;
    uint32_t pi = i;
    for (; (uint64_t)pi + G < npair; pi += 2 * G) {  // two pairs in flight
      double2 v[2][3];
#pragma unroll
      for (int u = 0; u < 2; u++)
#pragma unroll
        for (int k = 0; k < DIM; k++) v[u][k] = __ldcs(reinterpret_cast<const double2*>(P[k]) + pi + u * G);
#pragma unroll
      for (int u = 0; u < 2; u++) {
        visit(2 * (pi + u * G), v[u][0].x, v[u][1].x, DIM == 3 ? v[u][2].x : 0.0);
        visit(2 * (pi + u * G) + 1, v[u][0].y, v[u][1].y, DIM == 3 ? v[u][2].y : 0.0);
      }
    }
    for (; pi < npair; pi += G) {
      double2 v[3];
#pragma unroll
      for (int k = 0; k < DIM; k++) v[k] = __ldcs(reinterpret_cast<const double2*>(P[k]) + pi);
      visit(2 * pi, v[0].x, v[1].x, DIM == 3 ? v[2].x : 0.0);
      visit(2 * pi + 1, v[0].y, v[1].y, DIM == 3 ? v[2].y : 0.0);
    }
    i = (blockIdx.x == 0 && threadIdx.x == 0 && (n & 1)) ? n - 1 : n;  // odd tail
  }
  for (; i < n; i += G)
    visit(i, ld_coord(P[0], stride, i), ld_coord(P[1], stride, i), DIM == 3 ? ld_coord(P[2], stride, i) : 0.0);
  // warp + block reduction
  __shared__ SideAgg s_w[WARPS];
  __shared__ double s_d[WARPS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
#pragma unroll
    for (int s = 0; s < 2; s++) {
      a.cnt[s] += __shfl_xor_sync(0xFFFFFFFFu, a.cnt[s], o);
      const unsigned long long oh = __shfl_xor_sync(0xFFFFFFFFu, a.hi[s], o);
      const uint32_t oi = __shfl_xor_sync(0xFFFFFFFFu, a.idx[s], o);
      if (oh > a.hi[s] || (oh == a.hi[s] && oi < a.idx[s])) {
        a.hi[s] = oh;
        a.idx[s] = oi;
      }
    }
    dmax = fmax(dmax, __shfl_xor_sync(0xFFFFFFFFu, dmax, o));
  }
  if (lane == 0) {
    s_w[warp] = a;
    s_d[warp] = dmax;
  }
  __syncthreads();
  if (threadIdx.x < 2) {
    const int s = threadIdx.x;
    uint32_t c = 0;
    unsigned long long h = 0ull;
    uint32_t x = 0xFFFFFFFFu;
    for (int w = 0; w < WARPS; w++) {
      c += s_w[w].cnt[s];
      if (s_w[w].hi[s] > h || (s_w[w].hi[s] == h && s_w[w].idx[s] < x)) {
        h = s_w[w].hi[s];
        x = s_w[w].idx[s];
      }
    }
    if (c) {
      atomicAdd(&ws.cursor[0][s], c);  // root children (0, s): counts = cursor - 0
      atomic_max_key(&ws.slot_key[s], h, x);
    }
  }
  if (DIM == 3 && threadIdx.x == 0) {
    double m = 0.0;
    for (int w = 0; w < WARPS; w++) m = fmax(m, s_d[w]);
    if (m > 0.0) atomicMax((unsigned long long*)&st->dmax_bits, (unsigned long long)__double_as_longlong(m));
  }
}

// ------------------------------------------------------------------ bbox
// Per-axis min / max of a point slice (sharded hulls all-reduce these to
// the global Tolerance.effective, geometry.py:79-83).  Ordered-bits atomics
// into out[0..2*dim): min x[,y[,z]], then max.
__global__ void __launch_bounds__(BLOCK) k_bbox(const double* px, const double* py, const double* pz,
                                                int64_t stride, uint32_t n, int dim,
                                                unsigned long long* out) {
  unsigned long long lo[3] = {~0ull, ~0ull, ~0ull}, hi[3] = {0, 0, 0};
  const double* P[3] = {px, py, pz};
  for (uint32_t i = blockIdx.x * BLOCK + threadIdx.x; i < n; i += gridDim.x * BLOCK) {
#pragma unroll
    for (int k = 0; k < 3; k++) {
      if (k >= dim) break;
      const unsigned long long b = ordered_bits(ld_coord(P[k], stride, i));
      lo[k] = b < lo[k] ? b : lo[k];
      hi[k] = b > hi[k] ? b : hi[k];
    }
  }
#pragma unroll
  for (int k = 0; k < 3; k++) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const unsigned long long a = __shfl_xor_sync(0xFFFFFFFFu, lo[k], o);
      const unsigned long long b = __shfl_xor_sync(0xFFFFFFFFu, hi[k], o);
      lo[k] = a < lo[k] ? a : lo[k];
      hi[k] = b > hi[k] ? b : hi[k];
    }
  }
  if ((threadIdx.x & 31) == 0 && lo[0] != ~0ull) {
    for (int k = 0; k < dim; k++) {
      atomicMin(&out[k], lo[k]);
      atomicMax(&out[dim + k], hi[k]);
    }
  }
}

__global__ void k_bbox_init(unsigned long long* out, int dim) {
  if (threadIdx.x < 2 * dim) out[threadIdx.x] = threadIdx.x < dim ? ~0ull : 0ull;
}

__global__ void k_bbox_final(unsigned long long* out, double* res, int dim) {
  if (threadIdx.x < 2 * dim) res[threadIdx.x] = from_ordered_bits(out[threadIdx.x]);
}

// ------------------------------------------------------------------ stats
// One slice of a sharded hull (sh_stats): bbox and lexicographic extremes
// (quickhull.py:75-84, with global indices) in one pass.  out (SH_STATS
// doubles): -lo[3], hi[3] (one MAX all-reduce merges boxes), lex-min
// (x, y, z, global index), lex-max.  Partials per block, last block merges.
template <int DIM>
__global__ void __launch_bounds__(BLOCK) k_stats(const double* px, const double* py, const double* pz,
                                                 int64_t stride, uint32_t n, int64_t offset, FirstRed* parts,
                                                 uint32_t* counter, double* out) {
  const double* P[3] = {px, py, pz};
  FirstRed r;
#pragma unroll
  for (int k = 0; k < 3; k++) {
    r.lo[k] = INFINITY;
    r.hi[k] = -INFINITY;
    r.mn.c[k] = INFINITY;
    r.mx.c[k] = -INFINITY;
  }
  r.mn.idx = 0xFFFFFFFFu;
  r.mx.idx = 0;
  r.mn.pad = r.mx.pad = 0;
  for (uint32_t i = blockIdx.x * BLOCK + threadIdx.x; i < n; i += gridDim.x * BLOCK) {
    LexRec q;
#pragma unroll
    for (int k = 0; k < 3; k++) q.c[k] = (k < DIM) ? ld_coord(P[k], stride, i) : 0.0;
    q.idx = i;
    q.pad = 0;
#pragma unroll
    for (int k = 0; k < DIM; k++) {
      r.lo[k] = fmin(r.lo[k], q.c[k]);
      r.hi[k] = fmax(r.hi[k], q.c[k]);
    }
    if (lex_less<DIM>(q, r.mn)) r.mn = q;
    if (lex_less<DIM>(r.mx, q)) r.mx = q;
  }
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) {
    FirstRed o = shfl_xor_t(r, m);
    fr_merge<DIM>(r, o);
  }
  __shared__ FirstRed s_w[WARPS];
  __shared__ bool s_last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) s_w[warp] = r;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < WARPS; w++) fr_merge<DIM>(s_w[0], s_w[w]);
    parts[blockIdx.x] = s_w[0];
    __threadfence();
    s_last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last || threadIdx.x != 0) return;
  __threadfence();
  FirstRed t = ld_cg_fr(parts);
  for (uint32_t b = 1; b < gridDim.x; b++) {
    FirstRed o = ld_cg_fr(parts + b);
    fr_merge<DIM>(t, o);
  }
  *counter = 0;
#pragma unroll
  for (int k = 0; k < 3; k++) {
    out[k] = k < DIM ? -t.lo[k] : 0.0;
    out[3 + k] = k < DIM ? t.hi[k] : 0.0;
    out[6 + k] = t.mn.c[k];
    out[10 + k] = t.mx.c[k];
  }
  out[9] = (double)(offset + (int64_t)t.mn.idx);
  out[13] = (double)(offset + (int64_t)t.mx.idx);
}

// The ranks' statistics (gathered: world x SH_STATS) -> the whole input's:
// elementwise max of the boxes, lexicographic min / max of the extreme
// records (coordinates, then global index).
template <int DIM>
__global__ void k_stats_reduce(const double* gathered, int world, double* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double g[STATS_N];
  for (int k = 0; k < STATS_N; k++) g[k] = gathered[k];
  auto less = [](const double* a, const double* b) {
    for (int k = 0; k < DIM; k++) {
      if (a[k] < b[k]) return true;
      if (a[k] > b[k]) return false;
    }
    return a[3] < b[3];
  };
  for (int r = 1; r < world; r++) {
    const double* o = gathered + (size_t)r * STATS_N;
    for (int k = 0; k < 6; k++) g[k] = fmax(g[k], o[k]);
    if (less(o + 6, g + 6))
      for (int k = 0; k < 4; k++) g[6 + k] = o[6 + k];
    if (less(g + 10, o + 10))
      for (int k = 0; k < 4; k++) g[10 + k] = o[10 + k];
  }
  for (int k = 0; k < STATS_N; k++) out[k] = g[k];
}

// ------------------------------------------------------------------ K0b
struct KeyIdx {
  uint64_t hi;
  uint32_t idx;
  uint32_t pad;
};

__device__ __forceinline__ bool ki_better(const KeyIdx& a, const KeyIdx& b) {
  return (a.hi > b.hi) || (a.hi == b.hi && a.idx < b.idx);
}

__global__ void __launch_bounds__(BLOCK) k_line_far(Workspace ws) {
  DevState* st = ws.st;
  if (st->first_active != 2) return;
  const uint32_t n = st->n;
  const uint32_t nb = first_pass_blocks(n);
  if (blockIdx.x >= nb) return;
  const int64_t stride = st->stride;
  const double pa0 = st->pa[0], pa1 = st->pa[1], pa2 = st->pa[2];
  const double ux = sub(st->pb[0], pa0), uy = sub(st->pb[1], pa1), uz = sub(st->pb[2], pa2);
  const uint32_t imin = st->imin, imax = st->imax;
  KeyIdx best;
  best.hi = 0;
  best.idx = 0xFFFFFFFFu;
  best.pad = 0;
  auto visit = [&](uint32_t i, double x, double y, double z) {
    if (i == imin || i == imax) return;
    double cx, cy, cz;
    // quickhull.py:331-334: cross3(q - pa, u), squared norm left to right
    cross3(sub(x, pa0), sub(y, pa1), sub(z, pa2), ux, uy, uz, &cx, &cy, &cz);
    double d2 = add(add(mul(cx, cx), mul(cy, cy)), mul(cz, cz));
    KeyIdx k;
    k.hi = ordered_bits(d2);
    k.idx = i;
    k.pad = 0;
    if (ki_better(k, best)) best = k;
  };
  const uint32_t G = nb * BLOCK;
  uint32_t i = blockIdx.x * BLOCK + threadIdx.x;
  for (; (uint64_t)i + 3ull * G < n; i += 4 * G) {
    double x[4], y[4], z[4];
#pragma unroll
    for (int u = 0; u < 4; u++) {
      x[u] = ld_coord(st->px, stride, i + u * G);
      y[u] = ld_coord(st->py, stride, i + u * G);
      z[u] = ld_coord(st->pz, stride, i + u * G);
    }
#pragma unroll
    for (int u = 0; u < 4; u++) visit(i + u * G, x[u], y[u], z[u]);
  }
  for (; i < n; i += G)
    visit(i, ld_coord(st->px, stride, i), ld_coord(st->py, stride, i), ld_coord(st->pz, stride, i));
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) {
    KeyIdx o = shfl_xor_t(best, m);
    if (ki_better(o, best)) best = o;
  }
  __shared__ KeyIdx s_w[WARPS];
  __shared__ bool s_last;
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) s_w[warp] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < WARPS; w++)
      if (ki_better(s_w[w], s_w[0])) s_w[0] = s_w[w];
    KeyIdx* parts = reinterpret_cast<KeyIdx*>(ws.red);
    parts[blockIdx.x] = s_w[0];
    __threadfence();
    uint32_t done = atomicAdd(&st->ctr_red, 1u);
    s_last = (done == nb - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  KeyIdx t;
  {
    const KeyIdx* parts = reinterpret_cast<const KeyIdx*>(ws.red);
    t.hi = 0;
    t.idx = 0xFFFFFFFFu;
    t.pad = 0;
    for (uint32_t b = threadIdx.x; b < nb; b += BLOCK) {
      KeyIdx o;
      o.hi = __ldcg(&parts[b].hi);
      o.idx = __ldcg(&parts[b].idx);
      o.pad = 0;
      if (ki_better(o, t)) t = o;
    }
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
      KeyIdx o = shfl_xor_t(t, m);
      if (ki_better(o, t)) t = o;
    }
    __syncthreads();
    if (lane == 0) s_w[warp] = t;
    __syncthreads();
    if (threadIdx.x != 0) return;
    for (int w = 0; w < WARPS; w++)
      if (ki_better(s_w[w], t)) t = s_w[w];
  }
  st->ctr_red = 0;
  const double eps = st->eps;
  double d2 = from_ordered_bits(t.hi);
  // np.linalg.norm(pb - pa) == sqrt(ddot(u, u)), OpenBLAS FMA order
  double line_len = sqrt_(__fma_rn(uz, uz, __fma_rn(uy, uy, mul(ux, ux))));
  if (sqrt_(d2) <= mul(eps, line_len)) {  // quickhull.py:337-339
    st->flags |= FL_COLLINEAR;
    st->first_active = 0;
    return;
  }
  uint32_t f = t.idx;
  st->ifar = f;
  double pc[3] = {ld_coord(st->px, stride, f), ld_coord(st->py, stride, f),
                  ld_coord(st->pz, stride, f)};
  for (int k = 0; k < 3; k++) st->pc[k] = pc[k];
  ws.vout[2] = f;
  st->h_final = 3;
  if (n == 3) {  // quickhull.py:343-344
    st->first_active = 0;
    return;
  }
  double nx, ny, nz;  // quickhull.py:346-347
  cross3(sub(st->pb[0], pa0), sub(st->pb[1], pa1), sub(st->pb[2], pa2), sub(pc[0], pa0),
         sub(pc[1], pa1), sub(pc[2], pa2), &nx, &ny, &nz);
  st->nrm[0] = nx;
  st->nrm[1] = ny;
  st->nrm[2] = nz;
  double nv[3] = {nx, ny, nz};
  double nlen = norm3(nv);
  st->nlen = nlen;
  st->thr_line = mul(-eps, nlen);  // states = d < -eps * nlen (:353)
  st->first_active = 1;
  start_first_split(st);
}

}  // namespace sh
