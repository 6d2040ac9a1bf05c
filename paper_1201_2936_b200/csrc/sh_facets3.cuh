// K5: 3D facet output -- the (i, j, k) index triples of the hull's
// triangles, counter-clockwise seen from outside (north star: "3D: point
// array in, hull vertex indices / facet index triples out"; SURVEY.md §8(f)
// rank 3, pinned to Qhull's simplices on general-position inputs).
//
// The reference has no facet output (quickhull.py:282-446 returns the vertex
// set).  The device builds the facets of the hull of the filter's kept
// vertices K by parallel gift wrapping over the filter's Morton-sorted box
// tree (sh_filter3.cuh):
//
//   wrap(a, b): the facet (b, a, p) across the directed hull edge (a, b):
//     p such that every other vertex s has orient3d(b, a, p, s) > 0.
//     "s beats q" <=> orient3d(b, a, q, s) < 0 is a strict total order on
//     the vertices (they all lie in a half-space bounded by a plane through
//     a and b), so p is an argmax: each warp keeps the current best q, scans
//     the 64 sorted neighbours of a and of b, then descends the box tree
//     skipping every box whose points provably cannot beat q (fp64 upper
//     bound of (s - q).((b - q) x (a - q)) plus its rounding-error bound is
//     < 0; once pruned for q a box stays pruned for every better q).  Ties
//     between beating lanes are settled by a warp tournament.
//   Orientations are exact (sh_exact.cuh): fp64 filter, expansion
//   arithmetic, then Simulation of Simplicity on the original point indices,
//   so coplanar vertices (cube corners) still give a valid triangulation.
//
//   F7a k_fac_clear  reset the hash tables / work queue for this m
//   F7b k_fac_init   a0 = the vertex of minimal perturbed x; b0 = its
//                    neighbour on the 2D hull of the xy projection (exact
//                    orient2d with the same perturbation, so (a0, b0) is a
//                    3D hull edge); first facet = wrap(a0, b0) against the
//                    vertical half-plane through a0; its 3 edges seed the
//                    queue
//   F7c k_fac_wrap   persistent work-queue kernel, one warp per edge item:
//                    skip if the twin edge is known, else wrap; the facet
//                    hash set admits each facet once, its directed edges go
//                    into the edge hash set, its two open edges are pushed.
//                    Termination: completed == reserved (read in that order)
//   F7d k_fac_done   facet count -> result[1]
// Facet order in the output is unspecified (Qhull's is too); the set and the
// orientation are deterministic.
#pragma once

#include "sh_exact.cuh"
#include "sh_filter3.cuh"

namespace sh {

constexpr int FAC_BLOCK = 128;
constexpr uint32_t FAC_ID_BITS = 21;  // vertex ids (discovery order) < 2^21
constexpr uint32_t FAC_NONE = 0xFFFFFFFFu;
constexpr unsigned long long FAC_EMPTY = ~0ull;
constexpr uint32_t ST_FAC_TOO_MANY = 1;   // m >= 2^21
constexpr uint32_t ST_FAC_OVERFLOW = 2;   // facet_cap too small

struct FacetCtl {
  unsigned int head, reserved, completed, nfacets;
  unsigned int status, a0, b0, pad;
  unsigned long long fmask, emask, icap;
};

struct FacetWs {
  unsigned long long* ftab;   // facet keys (canonical rotation of discovery ids)
  unsigned long long* etab;   // directed edge keys
  unsigned long long* items;  // work queue: (1 << 63) | a << 21 | b, 0 = not yet written
  FacetCtl* ctl;
  uint64_t fcap, ecap, icap;  // allocated entries
  uint32_t mcap;
};

static inline uint64_t pow2_at_least(uint64_t x) {
  uint64_t p = 1;
  while (p < x) p <<= 1;
  return p;
}

static inline int facet_alloc(FacetWs& w, uint32_t mcap) {
  w.fcap = pow2_at_least(4ull * mcap + 16);
  w.ecap = pow2_at_least(16ull * mcap + 64);
  w.icap = 4ull * mcap + 64;
  bool ok = true;
  ok &= cudaMalloc((void**)&w.ftab, w.fcap * 8) == cudaSuccess;
  ok &= cudaMalloc((void**)&w.etab, w.ecap * 8) == cudaSuccess;
  ok &= cudaMalloc((void**)&w.items, w.icap * 8) == cudaSuccess;
  ok &= cudaMalloc((void**)&w.ctl, sizeof(FacetCtl)) == cudaSuccess;
  w.mcap = mcap;
  return ok ? 0 : 1;
}

static inline void facet_free(FacetWs& w) {
  void* ps[] = {w.ftab, w.etab, w.items, w.ctl};
  for (void* p : ps)
    if (p) cudaFree(p);
  w = FacetWs{};
}

__device__ __forceinline__ unsigned long long fac_mix(unsigned long long k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdull;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ull;
  k ^= k >> 33;
  return k;
}

// true if newly inserted
__device__ bool hset_insert(unsigned long long* tab, unsigned long long mask, unsigned long long key) {
  unsigned long long h = fac_mix(key) & mask;
  for (;;) {
    const unsigned long long old = atomicCAS(&tab[h], FAC_EMPTY, key);
    if (old == FAC_EMPTY) return true;
    if (old == key) return false;
    h = (h + 1) & mask;
  }
}

__device__ bool hset_find(const unsigned long long* tab, unsigned long long mask, unsigned long long key) {
  unsigned long long h = fac_mix(key) & mask;
  for (;;) {
    const unsigned long long v = *(const volatile unsigned long long*)&tab[h];
    if (v == key) return true;
    if (v == FAC_EMPTY) return false;
    h = (h + 1) & mask;
  }
}

__device__ __forceinline__ unsigned long long edge_key(uint32_t u, uint32_t v) {
  return ((unsigned long long)u << FAC_ID_BITS) | v;
}

__device__ __forceinline__ unsigned long long facet_key(uint32_t x, uint32_t y, uint32_t z) {
  // rotate so the smallest id comes first (orientation kept)
  if (y < x && y < z) {
    uint32_t t = x;
    x = y;
    y = z;
    z = t;
  } else if (z < x && z < y) {
    uint32_t t = z;
    z = y;
    y = x;
    x = t;
  }
  return ((unsigned long long)x << (2 * FAC_ID_BITS)) | ((unsigned long long)y << FAC_ID_BITS) | z;
}

// ------------------------------------------------------------------ F7a
__global__ void __launch_bounds__(BLOCK) k_fac_clear(Workspace ws, FilterWs f, FacetWs w) {
  const uint32_t m = f.fp->m;
  const unsigned long long fm = pow2_dev(4ull * m + 16), em = pow2_dev(16ull * m + 64), ic = 4ull * m + 64;
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x, T = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = tid; i < fm; i += T) w.ftab[i] = FAC_EMPTY;
  for (uint64_t i = tid; i < em; i += T) w.etab[i] = FAC_EMPTY;
  for (uint64_t i = tid; i < ic; i += T) w.items[i] = 0ull;
  if (tid == 0) {
    FacetCtl* c = w.ctl;
    c->head = c->reserved = c->completed = c->nfacets = 0;
    c->status = (m >= (1u << FAC_ID_BITS)) ? ST_FAC_TOO_MANY : 0u;
    c->a0 = c->b0 = FAC_NONE;
    c->fmask = fm - 1;
    c->emask = em - 1;
    c->icap = ic;
  }
}

// ------------------------------------------------------------------ wrap
// Warp-uniform state of one wrap query around the directed edge (a, b).
struct Wrap {
  double a[3], b[3];
  int64_t ga, gb;     // original indices (perturbation order)
  uint32_t ia, ib;    // discovery ids
  uint32_t iq;        // current best (FAC_NONE: none yet)
  int64_t gq;
  double q[3];
  double n[3];        // (b - q) x (a - q)
  double P[3];        // |products| of n's components (error bound)
};

__device__ __forceinline__ void wrap_set_q(Wrap& W, uint32_t iq, int64_t gq, const double* q) {
  W.iq = iq;
  W.gq = gq;
  W.q[0] = q[0];
  W.q[1] = q[1];
  W.q[2] = q[2];
  const double bd[3] = {sub(W.b[0], q[0]), sub(W.b[1], q[1]), sub(W.b[2], q[2])};
  const double ad[3] = {sub(W.a[0], q[0]), sub(W.a[1], q[1]), sub(W.a[2], q[2])};
  W.n[0] = sub(mul(bd[1], ad[2]), mul(bd[2], ad[1]));
  W.n[1] = sub(mul(bd[2], ad[0]), mul(bd[0], ad[2]));
  W.n[2] = sub(mul(bd[0], ad[1]), mul(bd[1], ad[0]));
  W.P[0] = add(fabs(mul(bd[1], ad[2])), fabs(mul(bd[2], ad[1])));
  W.P[1] = add(fabs(mul(bd[2], ad[0])), fabs(mul(bd[0], ad[2])));
  W.P[2] = add(fabs(mul(bd[0], ad[1])), fabs(mul(bd[1], ad[0])));
}

// error factor of the fp64 evaluation of (s - q).n incl. the rounded
// differences (> 12 eps; Shewchuk's orient3d bound is 7 eps)
constexpr double WRAP_ERR = 1.5e-15;

// s beats the current best q: orient3d(b, a, q, s) < 0, i.e.
// det3(s - q, b - q, a - q) = (s - q).n > 0
__device__ __forceinline__ bool wrap_beats(const Wrap& W, const double* s, int64_t gs) {
  if (W.iq == FAC_NONE) return true;
  const double sd[3] = {sub(s[0], W.q[0]), sub(s[1], W.q[1]), sub(s[2], W.q[2])};
  const double v = add(add(mul(sd[0], W.n[0]), mul(sd[1], W.n[1])), mul(sd[2], W.n[2]));
  const double perm = add(add(mul(fabs(sd[0]), W.P[0]), mul(fabs(sd[1]), W.P[1])), mul(fabs(sd[2]), W.P[2]));
  const double err = mul(WRAP_ERR, perm);
  if (v > err) return true;
  if (-v > err) return false;
  return orient3d_exact(W.b, W.a, W.q, s, W.gb, W.ga, W.gq, gs) < 0;
}

// y beats x (both real points): orient3d(b, a, x, y) < 0
__device__ __forceinline__ bool wrap_beats_pair(const Wrap& W, const double* x, int64_t gx, const double* y,
                                                int64_t gy) {
  return orient3d_exact(W.b, W.a, x, y, W.gb, W.ga, gx, gy) < 0;
}

struct FacTree {
  const double *sx, *sy, *sz;
  const uint32_t* sid;
  const uint8_t* keep;
  const uint32_t* vout;
};

// One 32-point batch (sorted positions p0 + lane): lanes whose point beats
// q compete in a tournament, the winner becomes the new q.
__device__ __forceinline__ void wrap_batch(Wrap& W, const FacTree& T, uint32_t m, uint32_t p) {
  const int lane = threadIdx.x & 31;
  bool cand = false;
  double s[3] = {0.0, 0.0, 0.0};
  uint32_t id = FAC_NONE;
  int64_t gs = -1;
  if (p < m) {
    id = __ldg(&T.sid[p]);
    if (__ldg(&T.keep[id]) && id != W.ia && id != W.ib && id != W.iq) {
      s[0] = __ldg(&T.sx[p]);
      s[1] = __ldg(&T.sy[p]);
      s[2] = __ldg(&T.sz[p]);
      gs = (int64_t)__ldg(&T.vout[id]);
      cand = wrap_beats(W, s, gs);
    }
  }
  const uint32_t mask = __ballot_sync(0xFFFFFFFFu, cand);
  if (!mask) return;
  if (!cand) id = FAC_NONE;
  // butterfly tournament (strict total order => every lane ends with the max)
#pragma unroll 1
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t oid = __shfl_xor_sync(0xFFFFFFFFu, id, o);
    const int64_t og = __shfl_xor_sync(0xFFFFFFFFu, gs, o);
    double os[3];
    os[0] = __shfl_xor_sync(0xFFFFFFFFu, s[0], o);
    os[1] = __shfl_xor_sync(0xFFFFFFFFu, s[1], o);
    os[2] = __shfl_xor_sync(0xFFFFFFFFu, s[2], o);
    if (oid != FAC_NONE && (id == FAC_NONE || wrap_beats_pair(W, s, gs, os, og))) {
      id = oid;
      gs = og;
      s[0] = os[0];
      s[1] = os[1];
      s[2] = os[2];
    }
  }
  wrap_set_q(W, id, gs, s);
}

// max over the box of (s - q).n in the point formula's operation order,
// plus the error allowance; < 0 => no point of the box beats q
__device__ __forceinline__ bool wrap_box_may_beat(const Wrap& W, const double* bx) {
  if (W.iq == FAC_NONE) return true;
  double bound = 0.0, perm = 0.0;
#pragma unroll
  for (int k = 0; k < 3; k++) {
    const double lo = sub(__ldg(bx + k), W.q[k]), hi = sub(__ldg(bx + 3 + k), W.q[k]);
    const double t = fmax(mul(lo, W.n[k]), mul(hi, W.n[k]));
    bound = (k == 0) ? t : add(bound, t);
    perm = add(perm, mul(fmax(fabs(lo), fabs(hi)), W.P[k]));
  }
  return !(bound < -mul(2.0 * WRAP_ERR, perm));
}

// p of the facet (b, a, p) across the hull edge (a, b); every lane returns it
__device__ uint32_t wrap_query(Wrap& W, const FacTree& T, const FilterParams& P, const FilterWs& f,
                               uint32_t* stk) {
  const int lane = threadIdx.x & 31;
  const uint32_t m = P.m;
  // (1) the sorted neighbourhoods of a and b
  const uint32_t pa = __ldg(&f.spos[W.ia]), pb = __ldg(&f.spos[W.ib]);
#pragma unroll 1
  for (int k = 0; k < 4; k++) {
    const uint32_t c = (k < 2) ? pa : pb;
    const uint32_t lo = c >= 32 ? c - 32 : 0;
    wrap_batch(W, T, m, lo + (k & 1) * 32 + lane);
  }
  // (2) box-tree descent
  if (P.nlev == 0) return W.iq;
  int top = 0;
  stk[0] = ((P.nlev - 1) << 26) | 0u;
  top = 1;
  while (top > 0) {
    top--;
    const uint32_t e = stk[top];
    __syncwarp();
    const uint32_t cl = e >> 26, cn = e & ((1u << 26) - 1);
    if (!wrap_box_may_beat(W, f.nbox + (size_t)(P.loff[cl] + cn) * 6)) continue;
    if (cl == 0) {
      wrap_batch(W, T, m, cn * 32 + lane);
      continue;
    }
    const uint32_t chl = cl - 1, ch = cn * 32 + lane;
    const bool pass = ch < P.lnodes[chl] && wrap_box_may_beat(W, f.nbox + (size_t)(P.loff[chl] + ch) * 6);
    const uint32_t mask = __ballot_sync(0xFFFFFFFFu, pass);
    const uint32_t r = __popc(mask & lanemask_lt());
    if (pass && top + (int)r < F_STACK) stk[top + r] = (chl << 26) | ch;
    top = min(top + __popc(mask), F_STACK);
    __syncwarp();
  }
  return W.iq;
}

__device__ __forceinline__ void load_pt(const FilterWs& f, uint32_t i, double* p) {
  p[0] = f.cx[i];
  p[1] = f.cy[i];
  p[2] = f.cz[i];
}

__device__ __forceinline__ void wrap_begin(Wrap& W, const FilterWs& f, const uint32_t* vout, uint32_t a,
                                           uint32_t b) {
  W.ia = a;
  W.ib = b;
  load_pt(f, a, W.a);
  load_pt(f, b, W.b);
  W.ga = (int64_t)vout[a];
  W.gb = (int64_t)vout[b];
  W.iq = FAC_NONE;
  W.gq = -1;
}

// Record the facet (x, y, z) (discovery ids) if new: output triple of
// original indices, its directed edges into the edge set, and the open
// edges (those whose twin is not known) onto the queue.  Warp-uniform
// arguments; lane 0 does the work.  skip: edge index (0..2) not to push.
__device__ void fac_emit(const FacetWs& w, const uint32_t* vout, int32_t* out, int64_t cap, uint32_t x,
                         uint32_t y, uint32_t z, int skip) {
  if ((threadIdx.x & 31) != 0) return;
  FacetCtl* C = w.ctl;
  if (!hset_insert(w.ftab, C->fmask, facet_key(x, y, z))) return;
  const unsigned int pos = atomicAdd(&C->nfacets, 1u);
  if ((int64_t)pos < cap) {
    out[3 * (size_t)pos + 0] = (int32_t)vout[x];
    out[3 * (size_t)pos + 1] = (int32_t)vout[y];
    out[3 * (size_t)pos + 2] = (int32_t)vout[z];
  }
  const uint32_t u[3] = {x, y, z}, v[3] = {y, z, x};
  for (int k = 0; k < 3; k++) hset_insert(w.etab, C->emask, edge_key(u[k], v[k]));
  unsigned long long push[3];
  int np = 0;
  for (int k = 0; k < 3; k++) {
    if (k == skip) continue;
    if (hset_find(w.etab, C->emask, edge_key(v[k], u[k]))) continue;
    push[np++] = (1ull << 63) | edge_key(u[k], v[k]);
  }
  if (np) {
    const unsigned int base = atomicAdd(&C->reserved, (unsigned int)np);
    for (int k = 0; k < np; k++)
      if (base + k < C->icap) *(volatile unsigned long long*)&w.items[base + k] = push[k];
  }
}

// ------------------------------------------------------------------ F7b
__global__ void __launch_bounds__(1024) k_fac_init(Workspace ws, FilterWs f, FacetWs w) {
  __shared__ FilterParams sP;
  __shared__ uint32_t s_id[32];
  __shared__ uint32_t s_stk[F_STACK];
  __shared__ uint32_t s_a0;
  if (threadIdx.x == 0) sP = *f.fp;
  __syncthreads();
  const FilterParams& P = sP;
  const uint32_t m = P.m;
  FacetCtl* C = w.ctl;
  const uint32_t* vout = ws.vout;
  int32_t* out = ws.st->out_facets;
  if (!out || m < 4 || C->status) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // a0: minimal perturbed x = minimal x, ties -> highest original index
  uint32_t best = FAC_NONE;
  double bx = 0.0;
  int64_t bg = -1;
  for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
    if (!f.keep[i]) continue;
    const double x = f.cx[i];
    const int64_t g = vout[i];
    if (best == FAC_NONE || x < bx || (x == bx && g > bg)) {
      best = i;
      bx = x;
      bg = g;
    }
  }
  for (int o = 16; o; o >>= 1) {
    const uint32_t ob = __shfl_xor_sync(0xFFFFFFFFu, best, o);
    const double ox = __shfl_xor_sync(0xFFFFFFFFu, bx, o);
    const int64_t og = __shfl_xor_sync(0xFFFFFFFFu, bg, o);
    if (ob != FAC_NONE && (best == FAC_NONE || ox < bx || (ox == bx && og > bg))) {
      best = ob;
      bx = ox;
      bg = og;
    }
  }
  if (lane == 0) s_id[warp] = best;
  __syncthreads();
  if (warp == 0) {
    best = s_id[lane];
    bx = best != FAC_NONE ? f.cx[best] : 0.0;
    bg = best != FAC_NONE ? (int64_t)vout[best] : -1;
    for (int o = 16; o; o >>= 1) {
      const uint32_t ob = __shfl_xor_sync(0xFFFFFFFFu, best, o);
      const double ox = __shfl_xor_sync(0xFFFFFFFFu, bx, o);
      const int64_t og = __shfl_xor_sync(0xFFFFFFFFu, bg, o);
      if (ob != FAC_NONE && (best == FAC_NONE || ox < bx || (ox == bx && og > bg))) {
        best = ob;
        bx = ox;
        bg = og;
      }
    }
    if (lane == 0) s_a0 = best;
  }
  __syncthreads();
  const uint32_t a0 = s_a0;
  if (a0 == FAC_NONE) return;
  const double A[2] = {f.cx[a0], f.cy[a0]};
  const int64_t ga = vout[a0];
  // b0: s beats q <=> orient2d(a0, q, s) < 0 (xy projection, same perturbation)
  uint32_t q = FAC_NONE;
  double Q[2] = {0.0, 0.0};
  int64_t gq = -1;
  for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
    if (!f.keep[i] || i == a0) continue;
    const double S[2] = {f.cx[i], f.cy[i]};
    const int64_t gs = vout[i];
    if (q == FAC_NONE || orient2d_exact(A, Q, S, ga, gq, gs) < 0) {
      q = i;
      Q[0] = S[0];
      Q[1] = S[1];
      gq = gs;
    }
  }
  auto tourney = [&]() {
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t oq = __shfl_xor_sync(0xFFFFFFFFu, q, o);
      const double ox = __shfl_xor_sync(0xFFFFFFFFu, Q[0], o), oy = __shfl_xor_sync(0xFFFFFFFFu, Q[1], o);
      const int64_t og = __shfl_xor_sync(0xFFFFFFFFu, gq, o);
      const double O[2] = {ox, oy};
      if (oq != FAC_NONE && (q == FAC_NONE || orient2d_exact(A, Q, O, ga, gq, og) < 0)) {
        q = oq;
        Q[0] = ox;
        Q[1] = oy;
        gq = og;
      }
    }
  };
  tourney();
  if (lane == 0) s_id[warp] = q;
  __syncthreads();
  if (warp != 0) return;
  q = s_id[lane];
  Q[0] = q != FAC_NONE ? f.cx[q] : 0.0;
  Q[1] = q != FAC_NONE ? f.cy[q] : 0.0;
  gq = q != FAC_NONE ? (int64_t)vout[q] : -1;
  tourney();
  const uint32_t b0 = q;
  if (b0 == FAC_NONE) return;
  // first facet: wrap (a0, b0) against the vertical half-plane through a0
  FacTree T{f.sx, f.sy, f.sz, f.sid, f.keep, vout};
  Wrap W;
  wrap_begin(W, f, vout, a0, b0);
  const uint32_t p = wrap_query(W, T, P, f, s_stk);
  if (lane == 0) {
    C->a0 = a0;
    C->b0 = b0;
  }
  if (p == FAC_NONE) return;
  fac_emit(w, vout, out, ws.st->facet_cap, b0, a0, p, -1);
}

// ------------------------------------------------------------------ F7c
__global__ void __launch_bounds__(FAC_BLOCK) k_fac_wrap(Workspace ws, FilterWs f, FacetWs w) {
  __shared__ FilterParams sP;
  __shared__ uint32_t s_stk[FAC_BLOCK / 32][F_STACK];
  if (threadIdx.x == 0) sP = *f.fp;
  __syncthreads();
  const FilterParams& P = sP;
  FacetCtl* C = w.ctl;
  int32_t* out = ws.st->out_facets;
  if (!out || P.m < 4 || C->status) return;
  const int64_t cap = ws.st->facet_cap;
  const uint32_t* vout = ws.vout;
  const int lane = threadIdx.x & 31;
  uint32_t* stk = s_stk[threadIdx.x >> 5];
  const FacTree T{f.sx, f.sy, f.sz, f.sid, f.keep, vout};
  const unsigned long long icap = C->icap, emask = C->emask;
  const uint32_t idm = (1u << FAC_ID_BITS) - 1;
  for (;;) {
    unsigned int idx = 0;
    if (lane == 0) idx = atomicAdd(&C->head, 1u);
    idx = __shfl_sync(0xFFFFFFFFu, idx, 0);
    unsigned long long item = 0;
    int done = 0;
    if (lane == 0) {
      for (;;) {
        if (idx < icap) {
          item = *(volatile unsigned long long*)&w.items[idx];
          if (item) break;
        }
        const unsigned int cdone = *(volatile unsigned int*)&C->completed;
        __threadfence();
        const unsigned int res = *(volatile unsigned int*)&C->reserved;
        if (cdone == res && idx >= res) {
          done = 1;
          break;
        }
        __nanosleep(200);
      }
    }
    done = __shfl_sync(0xFFFFFFFFu, done, 0);
    if (done) return;
    item = __shfl_sync(0xFFFFFFFFu, item, 0);
    __threadfence();
    const uint32_t a = (uint32_t)(item >> FAC_ID_BITS) & idm, b = (uint32_t)item & idm;
    bool known = false;
    if (lane == 0) known = hset_find(w.etab, emask, edge_key(b, a));
    known = __shfl_sync(0xFFFFFFFFu, known, 0);
    if (!known) {
      Wrap W;
      wrap_begin(W, f, vout, a, b);
      const uint32_t p = wrap_query(W, T, P, f, stk);
      if (p != FAC_NONE) fac_emit(w, vout, out, cap, b, a, p, 0);
    }
    __syncwarp();
    if (lane == 0) {
      __threadfence();
      atomicAdd(&C->completed, 1u);
    }
  }
}

// ------------------------------------------------------------------ F7d
__global__ void k_fac_done(Workspace ws, FilterWs f, FacetWs w) {
  if (threadIdx.x != 0) return;
  FacetCtl* C = w.ctl;
  const uint32_t nf = C->nfacets;
  f.result[1] = nf;
  if (!C->status && (int64_t)nf > ws.st->facet_cap) C->status = ST_FAC_OVERFLOW;
  f.result[4] = C->status;
}

static inline int facet_launch(FacetWs& w, FilterWs& f, Workspace ws, int nsm, int wrap_occ, cudaStream_t s) {
  k_fac_clear<<<nsm * 4, BLOCK, 0, s>>>(ws, f, w);
  k_fac_init<<<1, 1024, 0, s>>>(ws, f, w);
  k_fac_wrap<<<nsm * wrap_occ, FAC_BLOCK, 0, s>>>(ws, f, w);
  k_fac_done<<<1, 32, 0, s>>>(ws, f, w);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : 10;
}

}  // namespace sh
