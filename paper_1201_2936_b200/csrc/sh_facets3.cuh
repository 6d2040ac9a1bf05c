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
//   F7b' k_fac_seeds 64 direction seeds (fp64 extreme vertex + virtual
//                    line, facet verified exactly), see below
//   F7b k_fac_init   (only if no direction seed survived)
//                    a0 = the vertex of minimal perturbed x; b0 = its
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
constexpr uint32_t ST_FAC_BROKEN = 3;     // internal: table / queue capacity exceeded

struct FacetCtl {
  unsigned int head, reserved, completed, nfacets;
  unsigned int status, a0, b0, pad;
  unsigned long long fmask, emask, icap;
  // diagnostics (sh_facet_stats)
  unsigned long long queries, batches, beat_batches, nodes, wrap_cycles, wait_cycles, init_cycles;
};

struct FacetWs {
  double *kx, *ky, *kz;       // kept vertices in Morton order (vertex id = position)
  uint32_t* korig;            // their original point indices
  double* knbox;              // box tree over them (layout of FilterWs::nbox)
  double* knvol;              // oriented slabs of its levels 0-1 (FilterWs::nvol)
  FilterParams* kfp;          // its parameters (m = number of kept vertices)
  unsigned long long* ftab;   // facet keys (canonical rotation of vertex ids)
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
  ok &= cudaMalloc((void**)&w.kx, (size_t)mcap * 8 + 64) == cudaSuccess;
  ok &= cudaMalloc((void**)&w.ky, (size_t)mcap * 8 + 64) == cudaSuccess;
  ok &= cudaMalloc((void**)&w.kz, (size_t)mcap * 8 + 64) == cudaSuccess;
  ok &= cudaMalloc((void**)&w.korig, (size_t)mcap * 4 + 64) == cudaSuccess;
  ok &= cudaMalloc((void**)&w.knbox, ((size_t)mcap / 31 + 2 * F_LEVELS + 8) * 48) == cudaSuccess;
  ok &= cudaMalloc((void**)&w.knvol, ((size_t)mcap / 31 + 2 * F_LEVELS + 8) * 72) == cudaSuccess;
  ok &= cudaMalloc((void**)&w.kfp, sizeof(FilterParams)) == cudaSuccess;
  w.mcap = mcap;
  return ok ? 0 : 1;
}

static inline void facet_free(FacetWs& w) {
  void* ps[] = {w.ftab, w.etab, w.items, w.ctl, w.kx, w.ky, w.kz, w.korig, w.knbox, w.knvol, w.kfp};
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

// true if newly inserted; a full table (only possible if the construction
// went wrong) sets *status and reports the key as present
__device__ bool hset_insert(unsigned long long* tab, unsigned long long mask, unsigned long long key,
                            unsigned int* status) {
  unsigned long long h = fac_mix(key) & mask;
  for (unsigned long long probe = 0; probe <= mask; probe++) {
    const unsigned long long old = atomicCAS(&tab[h], FAC_EMPTY, key);
    if (old == FAC_EMPTY) return true;
    if (old == key) return false;
    h = (h + 1) & mask;
  }
  atomicExch(status, ST_FAC_BROKEN);
  return false;
}

__device__ bool hset_find(const unsigned long long* tab, unsigned long long mask, unsigned long long key) {
  unsigned long long h = fac_mix(key) & mask;
  for (unsigned long long probe = 0; probe <= mask; probe++) {
    const unsigned long long v = *(const volatile unsigned long long*)&tab[h];
    if (v == key) return true;
    if (v == FAC_EMPTY) return false;
    h = (h + 1) & mask;
  }
  return true;
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
    c->queries = c->batches = c->beat_batches = c->nodes = 0;
    c->wrap_cycles = c->wait_cycles = c->init_cycles = 0;
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
  uint32_t nb, nbb, nn;  // diagnostics: batches, batches with a beating lane, tree nodes
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

// The kept vertices in Morton order (a subsequence of the filter's sorted
// candidates) with their own box tree: vertex ids in the facet builder are
// positions in this order.
struct KTree {
  const double *x, *y, *z;
  const uint32_t* orig;  // original point index (output, perturbation order)
  const double* nbox;
  const double* nvol;
};

// One 32-vertex batch (positions p = base + lane): lanes whose vertex beats
// q compete in a tournament, the winner becomes the new q.
__device__ __forceinline__ void wrap_batch(Wrap& W, const KTree& T, uint32_t K, uint32_t p) {
  bool cand = false;
  double s[3] = {0.0, 0.0, 0.0};
  uint32_t id = FAC_NONE;
  int64_t gs = -1;
  if (p < K && p != W.ia && p != W.ib && p != W.iq) {
    id = p;
    s[0] = __ldg(&T.x[p]);
    s[1] = __ldg(&T.y[p]);
    s[2] = __ldg(&T.z[p]);
    gs = (int64_t)__ldg(&T.orig[p]);
    cand = wrap_beats(W, s, gs);
  }
  const uint32_t mask = __ballot_sync(0xFFFFFFFFu, cand);
  W.nb++;
  if (!mask) return;
  W.nbb++;
  if (!cand) id = FAC_NONE;
  if (__popc(mask) == 1) {
    const int src = __ffs(mask) - 1;
    id = __shfl_sync(0xFFFFFFFFu, id, src);
    gs = __shfl_sync(0xFFFFFFFFu, gs, src);
    s[0] = __shfl_sync(0xFFFFFFFFu, s[0], src);
    s[1] = __shfl_sync(0xFFFFFFFFu, s[1], src);
    s[2] = __shfl_sync(0xFFFFFFFFu, s[2], src);
    wrap_set_q(W, id, gs, s);
    return;
  }
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
    const double lo = sub(bx[k], W.q[k]), hi = sub(bx[3 + k], W.q[k]);
    const double t = fmax(mul(lo, W.n[k]), mul(hi, W.n[k]));
    bound = (k == 0) ? t : add(bound, t);
    perm = add(perm, mul(fmax(fabs(lo), fabs(hi)), W.P[k]));
  }
  return !(bound < -mul(2.0 * WRAP_ERR, perm));
}

// the same test against a node's oriented slab (levels 0-1)
__device__ __forceinline__ bool wrap_vol_may_beat(const Wrap& W, const double* vol) {
  if (W.iq == FAC_NONE) return true;
  const V3 n = v3(W.n[0], W.n[1], W.n[2]), q = v3(W.q[0], W.q[1], W.q[2]);
  const double vb = vol_bound(vol, n, q);
  const double ext = fabs(__ldg(vol + 0) - q.x) + fabs(__ldg(vol + 1) - q.y) + fabs(__ldg(vol + 2) - q.z) +
                     __ldg(vol + 8) + fmax(fabs(__ldg(vol + 6)), fabs(__ldg(vol + 7)));
  return !(vb < -2.0 * WRAP_ERR * (W.P[0] + W.P[1] + W.P[2]) * ext);
}

__device__ __forceinline__ void load_box(const double* src, double* bx) {
#pragma unroll
  for (int k = 0; k < 6; k++) bx[k] = __ldg(src + k);
}

// p of the facet (b, a, p) across the hull edge (a, b); every lane returns it
__device__ uint32_t wrap_query(Wrap& W, const KTree& T, const FilterParams& P, uint32_t* stk) {
  const int lane = threadIdx.x & 31;
  const uint32_t K = P.m;
  // (1) the Morton neighbourhoods of a and b
#pragma unroll 1
  for (int k = 0; k < 4; k++) {
    const uint32_t c = (k < 2 || W.ib == FAC_NONE) ? W.ia : W.ib;  // ib: virtual in seeding
    const uint32_t lo = c >= 32 ? c - 32 : 0;
    wrap_batch(W, T, K, lo + (k & 1) * 32 + lane);
  }
  // (2) box-tree descent (depth first); passing leaf children are scanned
  // right away, each re-tested against the then current q
  if (P.nlev == 0) return W.iq;
  if (P.nlev == 1) {
    wrap_batch(W, T, K, lane);
    return W.iq;
  }
  int top = 1;
  stk[0] = ((P.nlev - 1) << 26) | 0u;
  __syncwarp();
  while (top > 0) {
    top--;
    const uint32_t e = stk[top];
    __syncwarp();
    const uint32_t cl = e >> 26, cn = e & ((1u << 26) - 1);
    W.nn++;
    double bx[6];
    load_box(T.nbox + (size_t)(P.loff[cl] + cn) * 6, bx);
    if (!wrap_box_may_beat(W, bx)) continue;
    if (cl <= 1 && !wrap_vol_may_beat(W, T.nvol + (size_t)(P.loff[cl] + cn) * 9)) continue;
    const uint32_t chl = cl - 1, ch = cn * 32 + lane;
    bool pass = false;
    if (ch < P.lnodes[chl]) {
      load_box(T.nbox + (size_t)(P.loff[chl] + ch) * 6, bx);
      pass = wrap_box_may_beat(W, bx) &&
             (chl > 1 || wrap_vol_may_beat(W, T.nvol + (size_t)(P.loff[chl] + ch) * 9));
    }
    uint32_t mask = __ballot_sync(0xFFFFFFFFu, pass);
    if (chl == 0) {
      bool first = true;
      while (mask) {
        const int l = __ffs(mask) - 1;
        mask &= mask - 1;
        if (!first && !__shfl_sync(0xFFFFFFFFu, wrap_box_may_beat(W, bx), l)) continue;
        first = false;
        wrap_batch(W, T, K, (cn * 32 + l) * 32 + lane);
      }
      continue;
    }
    const uint32_t r = __popc(mask & lanemask_lt());
    if (pass && top + (int)r < F_STACK) stk[top + r] = (chl << 26) | ch;
    top = min(top + __popc(mask), F_STACK);
    __syncwarp();
  }
  return W.iq;
}

__device__ __forceinline__ void wrap_begin(Wrap& W, const KTree& T, uint32_t a, uint32_t b) {
  W.ia = a;
  W.ib = b;
  W.a[0] = T.x[a];
  W.a[1] = T.y[a];
  W.a[2] = T.z[a];
  W.b[0] = T.x[b];
  W.b[1] = T.y[b];
  W.b[2] = T.z[b];
  W.ga = (int64_t)T.orig[a];
  W.gb = (int64_t)T.orig[b];
  W.iq = FAC_NONE;
  W.gq = -1;
  W.nb = W.nbb = W.nn = 0;
}

// Record the facet (x, y, z) (vertex ids) if new: output triple of original
// indices, its directed edges into the edge set, and the open edges (those
// whose twin is not known) onto the queue.  Warp-uniform arguments; lane 0
// does the work.  skip: edge index (0..2) not to push.
__device__ void fac_emit(const FacetWs& w, const uint32_t* orig, int32_t* out, int64_t cap, uint32_t x,
                         uint32_t y, uint32_t z, int skip) {
  if ((threadIdx.x & 31) != 0) return;
  FacetCtl* C = w.ctl;
  if (!hset_insert(w.ftab, C->fmask, facet_key(x, y, z), &C->status)) return;
  const unsigned int pos = atomicAdd(&C->nfacets, 1u);
  if ((int64_t)pos < cap) {
    out[3 * (size_t)pos + 0] = (int32_t)orig[x];
    out[3 * (size_t)pos + 1] = (int32_t)orig[y];
    out[3 * (size_t)pos + 2] = (int32_t)orig[z];
  }
  const uint32_t u[3] = {x, y, z}, v[3] = {y, z, x};
  for (int k = 0; k < 3; k++) hset_insert(w.etab, C->emask, edge_key(u[k], v[k]), &C->status);
  unsigned long long push[3];
  int np = 0;
  for (int k = 0; k < 3; k++) {
    if (k == skip) continue;
    if (hset_find(w.etab, C->emask, edge_key(v[k], u[k]))) continue;
    push[np++] = (1ull << 63) | edge_key(u[k], v[k]);
  }
  if (np && *(volatile unsigned int*)&C->status == 0) {
    const unsigned int base = atomicAdd(&C->reserved, (unsigned int)np);
    int lost = 0;
    for (int k = 0; k < np; k++) {
      if (base + k < C->icap) *(volatile unsigned long long*)&w.items[base + k] = push[k];
      else lost++;
    }
    if (lost) {  // never written: count them as completed so the queue drains
      atomicExch(&C->status, ST_FAC_BROKEN);
      __threadfence();
      atomicAdd(&C->completed, (unsigned int)lost);
    }
  }
}

// ------------------------------------------------------------------ F7a'
// kept vertices (filter keep mask) in Morton order -> the facet builder's
// vertex arrays, plus the parameters of their box tree
__global__ void __launch_bounds__(1024) k_fac_keep(Workspace ws, FilterWs f, FacetWs w) {
  __shared__ uint32_t s_w[32];
  __shared__ uint32_t s_carry;
  const uint32_t m = f.fp->m;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (!ws.st->out_facets) return;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (uint32_t base = 0; base < m; base += 1024) {
    const uint32_t p = base + threadIdx.x;
    uint32_t id = 0, v = 0;
    if (p < m) {
      id = f.sid[p];
      v = f.keep[id] ? 1u : 0u;
    }
    const uint32_t bal = __ballot_sync(0xFFFFFFFFu, v);
    if (lane == 0) s_w[warp] = __popc(bal);
    __syncthreads();
    if (warp == 0) {
      const uint32_t x = s_w[lane];
      uint32_t y = x;
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t z = __shfl_up_sync(0xFFFFFFFFu, y, o);
        if (lane >= o) y += z;
      }
      s_w[lane] = y - x;
    }
    __syncthreads();
    const uint32_t pos = s_carry + s_w[warp] + __popc(bal & lanemask_lt());
    if (v) {
      w.kx[pos] = f.sx[p];
      w.ky[pos] = f.sy[p];
      w.kz[pos] = f.sz[p];
      w.korig[pos] = ws.vout[id];
    }
    __syncthreads();
    if (threadIdx.x == 1023) s_carry = pos + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    FilterParams* P = w.kfp;
    const uint32_t K = s_carry;
    P->m = K;
    uint32_t nl = K ? (K + 31) / 32 : 0, off = 0, lev = 0;
    for (int l = 0; l < F_LEVELS; l++) {
      P->lnodes[l] = nl;
      P->loff[l] = off;
      if (nl) lev = l + 1;
      off += nl;
      nl = (nl <= 1) ? 0 : (nl + 31) / 32;
    }
    P->nlev = lev;
  }
}

// ------------------------------------------------------------------ F7b
// Seeds: the vertices of minimal / maximal perturbed x and y (xy
// projection, virtual vertical line) and z (xz projection, virtual line
// along y).  Perturbed minimum: smallest value, ties -> largest original
// index (its perturbation is the smallest); maximum: ties -> smallest.
constexpr int FAC_SEEDS = 6;

__device__ __forceinline__ bool seed_better(int s, double v, int64_t g, double bv, int64_t bg) {
  if (s & 1) return v > bv || (v == bv && g < bg);  // maximum
  return v < bv || (v == bv && g > bg);             // minimum
}

__global__ void __launch_bounds__(1024) k_fac_init(Workspace ws, FacetWs w) {
  const long long t_start = clock64();
  __shared__ FilterParams sP;
  __shared__ uint32_t s_best[FAC_SEEDS][32];
  __shared__ uint32_t s_a[FAC_SEEDS], s_b[FAC_SEEDS];
  __shared__ uint32_t s_stk[FAC_SEEDS][F_STACK];
  if (threadIdx.x == 0) sP = *w.kfp;
  __syncthreads();
  const FilterParams& P = sP;
  const uint32_t K = P.m;
  FacetCtl* C = w.ctl;
  int32_t* out = ws.st->out_facets;
  // runs after k_fac_seeds: only needed when no direction seed survived its
  // verification (tiny or degenerate vertex sets)
  if (!out || K < 4 || C->status || C->nfacets) return;
  const KTree T{w.kx, w.ky, w.kz, w.korig, w.knbox, w.knvol};
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // (A) the six perturbed axis extremes
  {
    uint32_t best[FAC_SEEDS];
    double bv[FAC_SEEDS];
    int64_t bg[FAC_SEEDS];
    for (int s = 0; s < FAC_SEEDS; s++) {
      best[s] = FAC_NONE;
      bv[s] = 0.0;
      bg[s] = -1;
    }
    for (uint32_t i = threadIdx.x; i < K; i += blockDim.x) {
      const double c[3] = {T.x[i], T.y[i], T.z[i]};
      const int64_t g = T.orig[i];
      for (int s = 0; s < FAC_SEEDS; s++)
        if (best[s] == FAC_NONE || seed_better(s, c[s >> 1], g, bv[s], bg[s])) {
          best[s] = i;
          bv[s] = c[s >> 1];
          bg[s] = g;
        }
    }
    for (int s = 0; s < FAC_SEEDS; s++) {
      for (int o = 16; o; o >>= 1) {
        const uint32_t ob = __shfl_xor_sync(0xFFFFFFFFu, best[s], o);
        const double ov = __shfl_xor_sync(0xFFFFFFFFu, bv[s], o);
        const int64_t og = __shfl_xor_sync(0xFFFFFFFFu, bg[s], o);
        if (ob != FAC_NONE && (best[s] == FAC_NONE || seed_better(s, ov, og, bv[s], bg[s]))) {
          best[s] = ob;
          bv[s] = ov;
          bg[s] = og;
        }
      }
      if (lane == 0) s_best[s][warp] = best[s];
    }
    __syncthreads();
    if (warp < FAC_SEEDS) {
      const int s = warp;
      uint32_t b = s_best[s][lane];
      double v = b != FAC_NONE ? (s < 2 ? T.x[b] : s < 4 ? T.y[b] : T.z[b]) : 0.0;
      int64_t g = b != FAC_NONE ? (int64_t)T.orig[b] : -1;
      for (int o = 16; o; o >>= 1) {
        const uint32_t ob = __shfl_xor_sync(0xFFFFFFFFu, b, o);
        const double ov = __shfl_xor_sync(0xFFFFFFFFu, v, o);
        const int64_t og = __shfl_xor_sync(0xFFFFFFFFu, g, o);
        if (ob != FAC_NONE && (b == FAC_NONE || seed_better(s, ov, og, v, g))) {
          b = ob;
          v = ov;
          g = og;
        }
      }
      if (lane == 0) s_a[s] = b;
    }
    __syncthreads();
  }
  // (B) per seed (5 warps each): the neighbour b on the projected 2D hull,
  // s beats q <=> orient2d(a, q, s) < 0
  const int sd = warp < 5 * FAC_SEEDS ? warp / 5 : 0;
  const bool xz = sd >= 4;
  const uint32_t a2 = s_a[sd];
  const double A[2] = {T.x[a2], xz ? T.z[a2] : T.y[a2]};
  const int64_t ga = T.orig[a2];
  auto tourney = [&](uint32_t& q, double* Q, int64_t& gq) {
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t oq = __shfl_xor_sync(0xFFFFFFFFu, q, o);
      const double O[2] = {__shfl_xor_sync(0xFFFFFFFFu, Q[0], o), __shfl_xor_sync(0xFFFFFFFFu, Q[1], o)};
      const int64_t og = __shfl_xor_sync(0xFFFFFFFFu, gq, o);
      if (oq != FAC_NONE && (q == FAC_NONE || orient2d_exact(A, Q, O, ga, gq, og) < 0)) {
        q = oq;
        Q[0] = O[0];
        Q[1] = O[1];
        gq = og;
      }
    }
  };
  if (warp < 5 * FAC_SEEDS) {
    const uint32_t gt = threadIdx.x - sd * 160;
    uint32_t q = FAC_NONE;
    double Q[2] = {0.0, 0.0};
    int64_t gq = -1;
    for (uint32_t i = gt; i < K; i += 160) {
      if (i == a2) continue;
      const double S[2] = {T.x[i], xz ? T.z[i] : T.y[i]};
      const int64_t gs = T.orig[i];
      if (q == FAC_NONE || orient2d_exact(A, Q, S, ga, gq, gs) < 0) {
        q = i;
        Q[0] = S[0];
        Q[1] = S[1];
        gq = gs;
      }
    }
    tourney(q, Q, gq);
    if (lane == 0) s_best[sd][warp - 5 * sd] = q;
  }
  __syncthreads();
  if (warp < 5 * FAC_SEEDS && warp == 5 * sd) {
    uint32_t q = lane < 5 ? s_best[sd][lane] : FAC_NONE;
    double Q[2] = {q != FAC_NONE ? T.x[q] : 0.0, q != FAC_NONE ? (xz ? T.z[q] : T.y[q]) : 0.0};
    int64_t gq = q != FAC_NONE ? (int64_t)T.orig[q] : -1;
    tourney(q, Q, gq);
    if (lane == 0) s_b[sd] = q;
  }
  __syncthreads();
  // (C) one warp per seed: the hull facet across the silhouette edge.  In
  // the xy projection the virtual facet is (a, b, a + e_z), so wrap(a, b)
  // gives the facet (b, a, p); in the xz projection it is (b, a, a + e_y)
  // and wrap(b, a) gives (a, b, p).
  if (warp < FAC_SEEDS) {
    const int s = warp;
    const uint32_t a = s_a[s], b = s_b[s];
    if (a == FAC_NONE || b == FAC_NONE) return;
    const uint32_t u = s >= 4 ? b : a, v = s >= 4 ? a : b;
    Wrap W;
    wrap_begin(W, T, u, v);
    const uint32_t p = wrap_query(W, T, P, s_stk[s]);
    if (s == 0 && lane == 0) {
      C->a0 = a;
      C->b0 = b;
      C->init_cycles = (unsigned long long)(clock64() - t_start);
    }
    if (p == FAC_NONE) return;
    fac_emit(w, T.orig, out, ws.st->facet_cap, v, u, p, -1);
  }
}

// ------------------------------------------------------------------ F7b'
// More seeds, spread over the sphere of directions, to shorten the BFS (its
// critical path is the number of dependent wraps from the nearest seed).
// One warp per direction d (Fibonacci sphere):
//   v = the fp64 argmax of d.p over the kept vertices (an extreme vertex);
//   wrap(v, v + L e) with e a unit vector orthogonal to d and v + L e a
//   virtual point (perturbation index -1): the plane through the line
//   supports the hull at v, so the wrap yields a hull edge (v, p);
//   wrap(v, p) then yields the facet (p, v, q).
// The argmax is not exact, so the facet is verified exactly before it is
// used: a second descent starting from q must not find any vertex beating q
// (with q fixed the pruning is exact).  Failed seeds are dropped.
#ifndef SH_FAC_SEEDS
#define SH_FAC_SEEDS 256
#endif
constexpr int FAC_DIR_SEEDS = SH_FAC_SEEDS;

__global__ void __launch_bounds__(128) k_fac_seeds(Workspace ws, FilterWs f, FacetWs w) {
  __shared__ FilterParams sP;
  __shared__ uint32_t s_stk[4][F_STACK];
  if (threadIdx.x == 0) sP = *w.kfp;
  __syncthreads();
  const FilterParams& P = sP;
  const uint32_t K = P.m;
  FacetCtl* C = w.ctl;
  int32_t* out = ws.st->out_facets;
  if (!out || K < 4 || C->status) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t sd = blockIdx.x * 4 + warp;
  if (sd >= (uint32_t)FAC_DIR_SEEDS) return;
  const KTree T{w.kx, w.ky, w.kz, w.korig, w.knbox, w.knvol};
  // direction sd of a Fibonacci sphere
  const double zc = 1.0 - (2.0 * sd + 1.0) / FAC_DIR_SEEDS;
  const double rr = sqrt(fmax(0.0, 1.0 - zc * zc));
  const double ph = 2.399963229728653 * sd;
  const double d[3] = {rr * cos(ph), rr * sin(ph), zc};
  // fp64 argmax of d.p
  double bv = -INFINITY;
  uint32_t bi = FAC_NONE;
  for (uint32_t i = lane; i < K; i += 32) {
    const double v = d[0] * __ldg(&T.x[i]) + d[1] * __ldg(&T.y[i]) + d[2] * __ldg(&T.z[i]);
    if (v > bv) {
      bv = v;
      bi = i;
    }
  }
  for (int o = 16; o; o >>= 1) {
    const double ov = __shfl_xor_sync(0xFFFFFFFFu, bv, o);
    const uint32_t oi = __shfl_xor_sync(0xFFFFFFFFu, bi, o);
    if (ov > bv || (ov == bv && oi < bi)) {
      bv = ov;
      bi = oi;
    }
  }
  const uint32_t v = bi;
  if (v == FAC_NONE) return;
  // e orthogonal to d, scaled to the candidates' extent
  double e[3];
  {
    const double ax[3] = {fabs(d[0]) < 0.9 ? 1.0 : 0.0, fabs(d[0]) < 0.9 ? 0.0 : 1.0, 0.0};
    e[0] = d[1] * ax[2] - d[2] * ax[1];
    e[1] = d[2] * ax[0] - d[0] * ax[2];
    e[2] = d[0] * ax[1] - d[1] * ax[0];
    double span = 0.0;
    for (int k = 0; k < 3; k++)
      span = fmax(span, from_ordered_bits(f.fp->bb[3 + k]) - from_ordered_bits(f.fp->bb[k]));
    const double el = sqrt(e[0] * e[0] + e[1] * e[1] + e[2] * e[2]);
    for (int k = 0; k < 3; k++) e[k] = e[k] / el * (span > 0.0 ? span : 1.0);
  }
  uint32_t* stk = s_stk[warp];
  Wrap W;
  wrap_begin(W, T, v, v);
  W.ib = FAC_NONE;  // virtual second point v + e
  W.gb = -1;
  W.b[0] = W.a[0] + e[0];
  W.b[1] = W.a[1] + e[1];
  W.b[2] = W.a[2] + e[2];
  const uint32_t p = wrap_query(W, T, P, stk);
  if (p == FAC_NONE) return;
  wrap_begin(W, T, v, p);
  const uint32_t q = wrap_query(W, T, P, stk);
  if (q == FAC_NONE) return;
  // exact verification: nothing beats q for the edge (v, p)
  wrap_begin(W, T, v, p);
  {
    double qq[3] = {T.x[q], T.y[q], T.z[q]};
    wrap_set_q(W, q, (int64_t)T.orig[q], qq);
  }
  if (wrap_query(W, T, P, stk) != q) return;
  fac_emit(w, T.orig, out, ws.st->facet_cap, p, v, q, -1);
}

// ------------------------------------------------------------------ F7c
#ifndef SH_FAC_MINB
#define SH_FAC_MINB 4
#endif
__global__ void __launch_bounds__(FAC_BLOCK, SH_FAC_MINB) k_fac_wrap(Workspace ws, FacetWs w) {
  __shared__ FilterParams sP;
  __shared__ uint32_t s_stk[FAC_BLOCK / 32][F_STACK];
  if (threadIdx.x == 0) sP = *w.kfp;
  __syncthreads();
  const FilterParams& P = sP;
  FacetCtl* C = w.ctl;
  int32_t* out = ws.st->out_facets;
  if (!out || P.m < 4 || C->status) return;
  const int64_t cap = ws.st->facet_cap;
  const int lane = threadIdx.x & 31;
  uint32_t* stk = s_stk[threadIdx.x >> 5];
  const KTree T{w.kx, w.ky, w.kz, w.korig, w.knbox, w.knvol};
  const unsigned long long icap = C->icap, emask = C->emask;
  const uint32_t idm = (1u << FAC_ID_BITS) - 1;
  unsigned long long st_q = 0, st_b = 0, st_bb = 0, st_n = 0, st_wrap = 0, st_wait = 0;
  for (;;) {
    const long long t0 = clock64();
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
    const long long t1 = clock64();
    st_wait += (unsigned long long)(t1 - t0);
    if (done) break;
    item = __shfl_sync(0xFFFFFFFFu, item, 0);
    __threadfence();
    const uint32_t a = (uint32_t)(item >> FAC_ID_BITS) & idm, b = (uint32_t)item & idm;
    bool known = false;
    if (lane == 0) known = hset_find(w.etab, emask, edge_key(b, a));
    known = __shfl_sync(0xFFFFFFFFu, known, 0);
    if (!known) {
      Wrap W;
      wrap_begin(W, T, a, b);
      const uint32_t p = wrap_query(W, T, P, stk);
      if (p != FAC_NONE) fac_emit(w, T.orig, out, cap, b, a, p, 0);
      st_q++;
      st_b += W.nb;
      st_bb += W.nbb;
      st_n += W.nn;
    }
    st_wrap += (unsigned long long)(clock64() - t1);
    __syncwarp();
    if (lane == 0) {
      __threadfence();
      atomicAdd(&C->completed, 1u);
    }
  }
  if (lane == 0) {
    atomicAdd(&C->queries, st_q);
    atomicAdd(&C->batches, st_b);
    atomicAdd(&C->beat_batches, st_bb);
    atomicAdd(&C->nodes, st_n);
    atomicAdd(&C->wrap_cycles, st_wrap);
    atomicAdd(&C->wait_cycles, st_wait);
  }
}

// ------------------------------------------------------------------ F7d
__global__ void k_fac_done(Workspace ws, FilterWs f, FacetWs w) {
  if (!ws.st->out_facets) return;
  if (threadIdx.x != 0) return;
  FacetCtl* C = w.ctl;
  const uint32_t nf = C->nfacets;
  f.result[1] = nf;
  if (!C->status && (int64_t)nf > ws.st->facet_cap) C->status = ST_FAC_OVERFLOW;
  f.result[4] = C->status;
}

static inline int facet_launch(FacetWs& w, FilterWs& f, Workspace ws, int nsm, int wrap_occ, cudaStream_t s) {
  // the kept vertices' box tree reuses the filter's box kernels on a view
  FilterWs kv = f;
  kv.fp = w.kfp;
  kv.sx = kv.cx = w.kx;
  kv.sy = kv.cy = w.ky;
  kv.sz = kv.cz = w.kz;
  kv.nbox = w.knbox;
  kv.nvol = w.knvol;
  k_fac_clear<<<nsm * 4, BLOCK, 0, s>>>(ws, f, w);
  k_fac_keep<<<1, 1024, 0, s>>>(ws, f, w);
  k_f_boxes01<<<nsm * 2, 1024, 0, s>>>(kv);
  k_f_boxes_hi<<<1, 1024, 0, s>>>(kv);
  k_f_vols<<<nsm * 4, BLOCK, 0, s>>>(kv);
  k_fac_seeds<<<(FAC_DIR_SEEDS + 3) / 4, 128, 0, s>>>(ws, f, w);
  k_fac_init<<<1, 1024, 0, s>>>(ws, w);
  k_fac_wrap<<<nsm * wrap_occ, FAC_BLOCK, 0, s>>>(ws, w);
  k_fac_done<<<1, 32, 0, s>>>(ws, f, w);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : 10;
}

}  // namespace sh
