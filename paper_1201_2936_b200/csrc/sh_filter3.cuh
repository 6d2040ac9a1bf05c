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
//   F2 k_f_count    uniform G^3 grid (G a power of two <= 64, ~1 candidate
//                   per cell) numbered in Morton order
//   F3 k_f_scan     cell offsets (one block)
//   F4 k_f_scatter  candidates sorted by cell, i.e. along a Morton curve
//   F4b k_f_boxes   a 32-ary box tree over the sorted candidates: level 0 =
//                   32 consecutive candidates, level l+1 = 32 level-l nodes,
//                   tight fp64 boxes
//   F5 k_f_test     one warp per candidate:
//                     (1) certificate: no other candidate above the plane
//                         through v with normal v - bbox centre (+eps) -> keep
//                     (2) otherwise GJK on {c - v}: distance from v to the
//                         hull of the other candidates.  Outside -> keep;
//                         a tetrahedron of candidates containing v with
//                         every face farther than eps -> prune; anything
//                         closer than eps -> keep (the reference's
//                         eps-tolerant supporting plane keeps it too).
//                   Both use a best-first branch-and-bound support query
//                   down the tree: a node is skipped when the fp64 upper
//                   bound of d.(c - v) over its box can not beat the best
//                   value (IEEE rounding is monotone, so the bound computed
//                   with the point formula's operation order is exact).
//   F6 k_f_compact  kept candidates -> user indices, discovery order kept
//                   (verts[extreme], quickhull.py:311)
// m <= 4 keeps everything (quickhull.py:148-149).
#pragma once

#include "sh_common.cuh"

namespace sh {

constexpr uint32_t ST_CAND_OVERFLOW = 7;
constexpr int FG_MAX = 64;   // grid cells per axis (max, power of two)
constexpr int F_LEVELS = 6;  // box-tree levels: 32^6 candidates max
constexpr int F_TEST_BLOCK = 128;
constexpr int F_STACK = 32 * F_LEVELS;  // traversal stack entries per warp
#ifndef SH_FGRID_SLACK
#define SH_FGRID_SLACK 2.0
#endif
#ifndef F_PER_CELL
#define F_PER_CELL 1.0   // target candidates per grid cell
#endif

struct FilterParams {
  uint32_t m, G, nlev, ctr_test;
  uint32_t lnodes[F_LEVELS];   // nodes per tree level
  uint32_t loff[F_LEVELS];     // first node of each level in nbox
  double lo[3], inv_h[3], ctr[3];
  double gsum[3];              // sum of the candidates (deterministic order)
  unsigned long long bb[6];  // candidate bbox, ordered bits: min x,y,z then max x,y,z
  uint32_t ambiguous, gjk_capped, nwl, ctr_wl;  // nwl: work-list length (k_f_cert)
  uint32_t nwl2, ctr_wl2, pad2, nparts;          // second work list (k_f_local); k_f_boxes01's blocks
  uint32_t share_lo, share_hi;                    // discovery indices this launch decides (the others are kept)
  unsigned long long queries, scanned, gjk_iters, certified;  // diagnostics
  unsigned long long local_in, local_out, fallback;
  unsigned long long cyc_cert, cyc_local, cyc_out, cyc_fallback;  // SM cycles per phase (summed over warps)
  // -DSH_FILTER_CYCLES: k_f_test items by wall cycles (log2 buckets from
  // 2^10), and the slowest item's cycles, GJK iterations, queries, scanned
  uint32_t dur_hist[20];
  unsigned long long dur_max, dur_max_iters, dur_max_queries, dur_max_scanned;
};

struct FilterWs {
  unsigned long long* result;  // [0] kept, [1] facets, [2] filter applied, [3] ambiguous, [4] facet status
  uint32_t mcap;
  FilterParams* fp;
  double *cx, *cy, *cz;              // candidates, discovery order
  uint32_t* ccell;
  double *sx, *sy, *sz;              // candidates sorted by cell
  uint32_t* sid;                     // discovery index of sorted entry
  uint32_t* spos;                    // sorted position of discovery index
  uint32_t *cell_cnt, *cell_start, *cell_cur;
  double* nbox;                      // [node][6]: lo x,y,z, hi x,y,z (all levels)
  double* nvol;                      // [node][9]: oriented slab of levels 0-1 (see k_f_vols)
  uint8_t* keep;
  // candidates the first (certificate) query does not settle, for k_f_test
  uint32_t *wl_ps, *wl_pos, *wl_id;
  double* wl_val;
  // candidates the first local GJK (k_f_local) does not prune, for k_f_test:
  // work-list index (| 1 << 31 when the local GJK was inconclusive) and the
  // separating direction it found
  uint32_t* wl2_k;
  double* wl2_sep;
};

static inline int filter_alloc(FilterWs& f, uint64_t mcap) {
  bool ok = true;
  auto A = [&](void** p, size_t b) { ok &= cudaMalloc(p, b + 64) == cudaSuccess; };
  const size_t cells = (size_t)FG_MAX * FG_MAX * FG_MAX;
  const size_t nodes = mcap / 31 + 2 * F_LEVELS + 8;
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
  A((void**)&f.spos, mcap * 4);
  A((void**)&f.keep, mcap);
  A((void**)&f.wl_ps, mcap * 4);
  A((void**)&f.wl_pos, mcap * 4);
  A((void**)&f.wl_id, mcap * 4);
  A((void**)&f.wl_val, mcap * 8);
  A((void**)&f.wl2_k, mcap * 4);
  A((void**)&f.wl2_sep, mcap * 24);
  A((void**)&f.cell_cnt, cells * 4);
  A((void**)&f.cell_start, (cells + 1) * 4);
  A((void**)&f.cell_cur, cells * 4);
  A((void**)&f.nbox, nodes * 48);
  A((void**)&f.nvol, nodes * 72);
  f.mcap = (uint32_t)mcap;
  return ok ? 0 : 1;
}

static inline void filter_free(FilterWs& f) {
  void* ps[] = {f.result, f.fp, f.cx, f.cy, f.cz, f.sx, f.sy, f.sz, f.ccell, f.sid, f.spos, f.keep,
                f.cell_cnt, f.cell_start, f.cell_cur, f.nbox, f.nvol,
                f.wl_ps, f.wl_pos, f.wl_id, f.wl_val, f.wl2_k, f.wl2_sep};
  for (void* p : ps)
    if (p) cudaFree(p);
  f = FilterWs{};
}

// per-warp diagnostics (every lane holds the same values)
// per-phase cycle counters cost ~20% of the filter: compiled in only with
// -DSH_FILTER_CYCLES (diagnostics, sh_filter_stats)
#ifdef SH_FILTER_CYCLES
#define FCLK() clock64()
#else
#define FCLK() 0ll
#endif

struct FStat {
  unsigned long long scanned, queries, iters, certified, local_in, local_out, fallback;
  unsigned long long cyc_cert, cyc_local, cyc_out, cyc_fallback;
};

__device__ __forceinline__ unsigned long long obits(double d) { return ordered_bits(d); }
__device__ __forceinline__ double ofrom(unsigned long long b) { return from_ordered_bits(b); }

__device__ __forceinline__ uint32_t f_grid_of(uint32_t m) {
  // G a power of two with G^3 <= m / F_PER_CELL * SH_FGRID_SLACK (>= ~0.5
  // candidates per cell): finer grids only cost scan time
  double g = (double)m / F_PER_CELL * SH_FGRID_SLACK;
  uint32_t G = 2;
  while (G < FG_MAX && (double)(2 * G) * (2 * G) * (2 * G) <= g) G <<= 1;
  return G;
}

__device__ __forceinline__ uint32_t spread3(uint32_t x) {  // 6 bits -> every third bit
  uint32_t r = 0;
#pragma unroll
  for (int b = 0; b < 6; b++) r |= ((x >> b) & 1u) << (3 * b);
  return r;
}

// ------------------------------------------------------------------ F0
__global__ void __launch_bounds__(BLOCK) k_f_setup(Workspace ws, FilterWs f) {
  DevState* st = ws.st;
  uint32_t m = st->h_final;
  if (m > f.mcap) m = 0;  // overflow: reported below, nothing else runs
  const uint32_t G = f_grid_of(m);
  const uint32_t cells = G * G * G;
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x, T = gridDim.x * blockDim.x;
  for (uint32_t c = tid; c < cells; c += T) f.cell_cnt[c] = 0;
  if (tid == 0) {
    FilterParams* P = f.fp;
    P->m = m;
    P->G = G;
    {  // sh_set_filter_share: a contiguous range of discovery indices (the
       // Morton order within a grid cell depends on atomics, the discovery
       // order does not: every launch of the merge sees the same partition)
      const uint32_t R = st->filter_nshares > 1 ? st->filter_nshares : 1u, r = R > 1 ? st->filter_share : 0u;
      P->share_lo = (uint32_t)(((uint64_t)m * r) / R);
      P->share_hi = (uint32_t)(((uint64_t)m * (r + 1)) / R);
    }
    P->ctr_test = 0;
    P->ambiguous = 0;
    P->gjk_capped = 0;
    P->nwl = 0;
    P->ctr_wl = 0;
    P->nwl2 = 0;
    P->ctr_wl2 = 0;
    P->queries = 0;
    P->scanned = 0;
    P->gjk_iters = 0;
    P->certified = 0;
    P->local_in = 0;
    P->local_out = 0;
    P->fallback = 0;
    P->cyc_cert = P->cyc_local = P->cyc_out = P->cyc_fallback = 0;
    for (int k = 0; k < 20; k++) P->dur_hist[k] = 0;
    P->dur_max = P->dur_max_iters = P->dur_max_queries = P->dur_max_scanned = 0;
    // box tree: level 0 = chunks of 32 candidates, level l+1 = 32 level-l nodes
    uint32_t nl = m ? (m + 31) / 32 : 0, off = 0, lev = 0;
    for (int l = 0; l < F_LEVELS; l++) {
      P->lnodes[l] = nl;
      P->loff[l] = off;
      if (nl) lev = l + 1;
      off += nl;
      nl = (nl <= 1) ? 0 : (nl + 31) / 32;
    }
    P->nlev = lev;
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
    double c[3];
    if (q < st->n) {
      c[0] = ld_coord(st->px, stride, q);
      c[1] = ld_coord(st->py, stride, q);
      c[2] = ld_coord(st->pz, stride, q);
    } else {  // virtual first-split extreme of a sharded hull (k_first_reduce)
      const double* v = q == st->n ? st->pa : st->pb;
      c[0] = v[0];
      c[1] = v[1];
      c[2] = v[2];
    }
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
  uint32_t G;
};

__device__ __forceinline__ GridGeom f_geom(const FilterParams* P) {
  GridGeom g;
  g.G = P->G;
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
    const uint32_t cell = spread3(f_axis_cell(g, 0, f.cx[i])) | (spread3(f_axis_cell(g, 1, f.cy[i])) << 1) |
                          (spread3(f_axis_cell(g, 2, f.cz[i])) << 2);
    f.ccell[i] = cell;
    atomicAdd(&f.cell_cnt[cell], 1u);
  }
}

// ------------------------------------------------------------------ F3
// cell offsets: tiles of 8192 cells (1024 threads x 8 consecutive cells,
// 16-byte loads; G^3 is a multiple of 8).  k_f_scan_tiles: each block the
// total of its tile; k_f_scan: each block the exclusive scan of its tile
// on top of the totals of the tiles before it.
constexpr uint32_t F_SCAN_TILE = 8192;
constexpr uint32_t F_SCAN_GRID = (uint32_t)FG_MAX * FG_MAX * FG_MAX / F_SCAN_TILE;

__device__ __forceinline__ void f_load8(const uint32_t* a, uint32_t c, uint32_t cells, uint32_t* v) {
  if (c < cells) {
    const uint4 x = *reinterpret_cast<const uint4*>(a + c);
    const uint4 y = *reinterpret_cast<const uint4*>(a + c + 4);
    v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
    v[4] = y.x; v[5] = y.y; v[6] = y.z; v[7] = y.w;
  } else {
#pragma unroll
    for (int k = 0; k < 8; k++) v[k] = 0;
  }
}

__global__ void __launch_bounds__(1024) k_f_scan_tiles(FilterWs f) {
  __shared__ uint32_t s_w[32];
  const uint32_t G = f.fp->G, cells = G * G * G;
  const uint32_t base = blockIdx.x * F_SCAN_TILE;
  if (base >= cells) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t v[8];
  f_load8(f.cell_cnt, base + 8 * threadIdx.x, cells, v);
  uint32_t tot = 0;
#pragma unroll
  for (int k = 0; k < 8; k++) tot += v[k];
  tot = __reduce_add_sync(0xFFFFFFFFu, tot);
  if (lane == 0) s_w[warp] = tot;
  __syncthreads();
  if (warp == 0) {
    const uint32_t t = __reduce_add_sync(0xFFFFFFFFu, s_w[lane]);
    if (lane == 0) f.wl_ps[blockIdx.x] = t;  // free until k_f_cert
  }
}

__global__ void __launch_bounds__(1024) k_f_scan(FilterWs f) {
  __shared__ uint32_t s_w[32];
  __shared__ uint32_t s_carry;
  const uint32_t G = f.fp->G, cells = G * G * G;
  const uint32_t base = blockIdx.x * F_SCAN_TILE;
  if (base >= cells) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp == 0) {  // the tiles before this one
    const uint32_t t = lane < blockIdx.x ? f.wl_ps[lane] : 0u;
    const uint32_t c = __reduce_add_sync(0xFFFFFFFFu, t);
    if (lane == 0) s_carry = c;
  }
  const uint32_t c = base + 8 * threadIdx.x;
  uint32_t v[8];
  f_load8(f.cell_cnt, c, cells, v);
  uint32_t tot = 0;
#pragma unroll
  for (int k = 0; k < 8; k++) tot += v[k];
  uint32_t x = tot;
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_w[warp] = x;
  __syncthreads();
  if (warp == 0) {
    const uint32_t w = s_w[lane];
    uint32_t y = w;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t z = __shfl_up_sync(0xFFFFFFFFu, y, o);
      if (lane >= o) y += z;
    }
    s_w[lane] = y - w;
  }
  __syncthreads();
  uint32_t run = s_carry + s_w[warp] + x - tot;
  if (c < cells) {
    uint32_t o[8];
#pragma unroll
    for (int k = 0; k < 8; k++) {
      o[k] = run;
      run += v[k];
    }
    *reinterpret_cast<uint4*>(f.cell_start + c) = make_uint4(o[0], o[1], o[2], o[3]);
    *reinterpret_cast<uint4*>(f.cell_start + c + 4) = make_uint4(o[4], o[5], o[6], o[7]);
    *reinterpret_cast<uint4*>(f.cell_cur + c) = make_uint4(o[0], o[1], o[2], o[3]);
    *reinterpret_cast<uint4*>(f.cell_cur + c + 4) = make_uint4(o[4], o[5], o[6], o[7]);
    if (c + 8 == cells) f.cell_start[cells] = run;
  }
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
    f.spos[i] = p;
  }
}

// ------------------------------------------------------------------ F4b
// levels 0 and 1: a block of 32 warps builds 32 level-0 boxes (one warp
// per 32 sorted candidates) and the level-1 box above them
__global__ void __launch_bounds__(1024) k_f_boxes01(FilterWs f) {
  __shared__ double sbx[32][6];
  const FilterParams* P = f.fp;
  const uint32_t m = P->m, n0 = P->lnodes[0], n1 = P->lnodes[1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  {
    // this block's part of the candidates' sum (discovery order, a fixed
    // slice and reduction tree: deterministic), combined by k_f_boxes_hi
    __shared__ double s_sum[32][3];
    const uint32_t p0 = (uint32_t)(((uint64_t)m * blockIdx.x) / gridDim.x);
    const uint32_t p1 = (uint32_t)(((uint64_t)m * (blockIdx.x + 1)) / gridDim.x);
    double a[3] = {0.0, 0.0, 0.0};
    for (uint32_t p = p0 + threadIdx.x; p < p1; p += 1024) {
      a[0] += f.cx[p];
      a[1] += f.cy[p];
      a[2] += f.cz[p];
    }
#pragma unroll
    for (int k = 0; k < 3; k++)
      for (int o = 16; o; o >>= 1) a[k] += __shfl_xor_sync(0xFFFFFFFFu, a[k], o);
    if (lane == 0)
      for (int k = 0; k < 3; k++) s_sum[warp][k] = a[k];
    __syncthreads();
    if (threadIdx.x < 3) {
      double t = 0.0;
      for (int w = 0; w < 32; w++) t += s_sum[w][threadIdx.x];
      f.wl_val[3 * blockIdx.x + threadIdx.x] = t;  // free until k_f_cert
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) f.fp->nparts = gridDim.x;
  }
  for (uint32_t base = blockIdx.x * 32; base < n0; base += gridDim.x * 32) {
    const uint32_t node = base + warp;
    double b[6] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY};
    const uint32_t p = node * 32 + lane;
    if (node < n0 && p < m) {
      const double c[3] = {f.sx[p], f.sy[p], f.sz[p]};
#pragma unroll
      for (int k = 0; k < 3; k++) {
        b[k] = c[k];
        b[3 + k] = c[k];
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
#pragma unroll
      for (int k = 0; k < 3; k++) {
        b[k] = fmin(b[k], __shfl_xor_sync(0xFFFFFFFFu, b[k], o));
        b[3 + k] = fmax(b[3 + k], __shfl_xor_sync(0xFFFFFFFFu, b[3 + k], o));
      }
    }
    if (lane < 6) {
      double v = b[0];
#pragma unroll
      for (int k = 1; k < 6; k++) v = (lane == k) ? b[k] : v;
      sbx[warp][lane] = v;
      if (node < n0) f.nbox[(size_t)(P->loff[0] + node) * 6 + lane] = v;
    }
    __syncthreads();
    if (warp == 0 && n1 > 0) {
      double c[6];
#pragma unroll
      for (int k = 0; k < 6; k++) c[k] = sbx[lane][k];
#pragma unroll
      for (int o = 16; o; o >>= 1) {
#pragma unroll
        for (int k = 0; k < 3; k++) {
          c[k] = fmin(c[k], __shfl_xor_sync(0xFFFFFFFFu, c[k], o));
          c[3 + k] = fmax(c[3 + k], __shfl_xor_sync(0xFFFFFFFFu, c[3 + k], o));
        }
      }
      if (lane < 6) {
        double v = c[0];
#pragma unroll
        for (int k = 1; k < 6; k++) v = (lane == k) ? c[k] : v;
        f.nbox[(size_t)(P->loff[1] + base / 32) * 6 + lane] = v;
      }
    }
    __syncthreads();
  }
}

// levels 2.. (at most a few hundred nodes): one block, one warp per node;
// the same block also adds up k_f_boxes01's partial sums in order (centroid)
__global__ void __launch_bounds__(1024) k_f_boxes_hi(FilterWs f) {
  const FilterParams* P = f.fp;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x < 3) {  // the parts of k_f_boxes01, in order
    double t = 0.0;
    for (uint32_t b = 0; b < P->nparts; b++) t += f.wl_val[3 * b + threadIdx.x];
    f.fp->gsum[threadIdx.x] = t;
  }
  for (int l = 2; l < (int)P->nlev; l++) {
    const uint32_t nl = P->lnodes[l], nc = P->lnodes[l - 1];
    for (uint32_t node = warp; node < nl; node += 32) {
      double c[6] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY};
      const uint32_t ch = node * 32 + lane;
      if (ch < nc) {
#pragma unroll
        for (int k = 0; k < 6; k++) c[k] = f.nbox[(size_t)(P->loff[l - 1] + ch) * 6 + k];
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
#pragma unroll
        for (int k = 0; k < 3; k++) {
          c[k] = fmin(c[k], __shfl_xor_sync(0xFFFFFFFFu, c[k], o));
          c[3 + k] = fmax(c[3 + k], __shfl_xor_sync(0xFFFFFFFFu, c[3 + k], o));
        }
      }
      if (lane < 6) {
        double v = c[0];
#pragma unroll
        for (int k = 1; k < 6; k++) v = (lane == k) ? c[k] : v;
        f.nbox[(size_t)(P->loff[l] + node) * 6 + lane] = v;
      }
    }
    __syncthreads();
  }
}

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

// ------------------------------------------------------------------ F4c
// Oriented slabs for the nodes of levels 0 and 1 (32 / 1024 candidates).
// The candidates lie near the hull surface, where an axis-aligned box
// overestimates the support d.c by O(patch size) while a slab along the
// patch's outward axis overestimates it by O(patch size^2) (the sagitta):
//   c   = mean of the node's points, u = unit(c - centroid of all),
//   [hmin, hmax] = range of u.(p - c), rho = max |(p - c) - (u.(p - c)) u|,
//   max_p d.(p - v) <= d.(c - v) + max(a hmax, a hmin) + |d_perp| rho,
//   a = d.u, |d_perp| = sqrt(|d|^2 - a^2).
// Stored ranges are widened by 1e-13 of the node's extent and vol_bound
// adds a relative margin, so the fp64 bound is >= every fp64 point value.
__global__ void __launch_bounds__(BLOCK) k_f_vols(FilterWs f) {
  const FilterParams* P = f.fp;
  const uint32_t m = P->m, n0 = P->lnodes[0], n1 = P->nlev > 1 ? P->lnodes[1] : 0;
  const int lane = threadIdx.x & 31;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, W = (gridDim.x * blockDim.x) >> 5;
  const double inv_m = m ? 1.0 / (double)m : 0.0;
  const V3 G = v3(P->gsum[0] * inv_m, P->gsum[1] * inv_m, P->gsum[2] * inv_m);
  for (uint32_t node = gw; node < n0 + n1; node += W) {
    const uint32_t lev = node < n0 ? 0 : 1, j = node < n0 ? node : node - n0;
    const uint32_t span = lev ? 1024u : 32u;
    const uint32_t p0 = j * span, p1 = min(p0 + span, m);
    double sx = 0.0, sy = 0.0, sz = 0.0;
    for (uint32_t p = p0 + lane; p < p1; p += 32) {
      sx += f.sx[p];
      sy += f.sy[p];
      sz += f.sz[p];
    }
    for (int o = 16; o; o >>= 1) {
      sx += __shfl_xor_sync(0xFFFFFFFFu, sx, o);
      sy += __shfl_xor_sync(0xFFFFFFFFu, sy, o);
      sz += __shfl_xor_sync(0xFFFFFFFFu, sz, o);
    }
    const double inv = 1.0 / (double)(p1 - p0);
    const V3 c = v3(sx * inv, sy * inv, sz * inv);
    V3 u = vsub(c, G);
    double ul = sqrt_(vdot(u, u));
    if (!(ul > 0.0)) {
      u = v3(1.0, 0.0, 0.0);
      ul = 1.0;
    }
    u = v3(u.x / ul, u.y / ul, u.z / ul);
    double hmin = INFINITY, hmax = -INFINITY, rho = 0.0, wmax = 0.0;
    for (uint32_t p = p0 + lane; p < p1; p += 32) {
      const V3 w = vsub(v3(f.sx[p], f.sy[p], f.sz[p]), c);
      const double h = vdot(u, w);
      const V3 t = vsub(w, vscale(u, h));
      hmin = fmin(hmin, h);
      hmax = fmax(hmax, h);
      rho = fmax(rho, sqrt_(vdot(t, t)));
      wmax = fmax(wmax, fabs(w.x) + fabs(w.y) + fabs(w.z));
    }
    for (int o = 16; o; o >>= 1) {
      hmin = fmin(hmin, __shfl_xor_sync(0xFFFFFFFFu, hmin, o));
      hmax = fmax(hmax, __shfl_xor_sync(0xFFFFFFFFu, hmax, o));
      rho = fmax(rho, __shfl_xor_sync(0xFFFFFFFFu, rho, o));
      wmax = fmax(wmax, __shfl_xor_sync(0xFFFFFFFFu, wmax, o));
    }
    const double slack = 1e-13 * wmax;
    const double vals[9] = {c.x, c.y, c.z, u.x, u.y, u.z, hmin - slack, hmax + slack, rho + slack};
    if (lane < 9) {
      double v = vals[0];
#pragma unroll
      for (int k = 1; k < 9; k++) v = (lane == k) ? vals[k] : v;
      f.nvol[(size_t)(P->loff[lev] + j) * 9 + lane] = v;
    }
  }
}

// ------------------------------------------------------------------ F5

// max over the box of d.(c - v), evaluated with the point formula's order
__device__ __forceinline__ double box_bound(const double* b, V3 d, V3 v) {
  const double t0 = fmax(mul(d.x, sub(__ldg(b + 0), v.x)), mul(d.x, sub(__ldg(b + 3), v.x)));
  const double t1 = fmax(mul(d.y, sub(__ldg(b + 1), v.y)), mul(d.y, sub(__ldg(b + 4), v.y)));
  const double t2 = fmax(mul(d.z, sub(__ldg(b + 2), v.z)), mul(d.z, sub(__ldg(b + 5), v.z)));
  return add(add(t0, t1), t2);
}

// Upper bound of d.(p - v) over a node with an oriented slab (k_f_vols),
// valid for the fp64 point values (relative margin 1e-12).
__device__ __forceinline__ double vol_bound(const double* vol, V3 d, V3 v) {
  const V3 c = v3(__ldg(vol + 0), __ldg(vol + 1), __ldg(vol + 2));
  const V3 u = v3(__ldg(vol + 3), __ldg(vol + 4), __ldg(vol + 5));
  const double hmin = __ldg(vol + 6), hmax = __ldg(vol + 7), rho = __ldg(vol + 8);
  const V3 cv = vsub(c, v);
  const double dc = vdot(d, cv), al = vdot(d, u), dd = vdot(d, d);
  const double beta = sqrt_(fmax(dd - al * al, 0.0) + 1e-15 * dd);
  const double b = dc + fmax(al * hmax, al * hmin) + beta * rho;
  const double d1 = fabs(d.x) + fabs(d.y) + fabs(d.z);
  return b + 1e-12 * d1 * (fabs(cv.x) + fabs(cv.y) + fabs(cv.z) + rho + fmax(fabs(hmin), fabs(hmax)));
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

struct FStack {
  uint32_t node[F_STACK];  // (level << 26) | node
  double bound[F_STACK];
};

// Best-first branch-and-bound support query down the box tree:
// max over candidates c != self of d.(c - v).  first_hit: stop at the first
// value > thr (existence query).  Warp-cooperative; every lane returns the
// same result.
__device__ Sup support_query(const FilterWs& f, const FilterParams& P, V3 d, V3 v, uint32_t self,
                             double thr, bool first_hit, FStack& stk, FStat& fs) {
  const int lane = threadIdx.x & 31;
  fs.queries++;
  Sup best;
  best.val = -INFINITY;
  best.pos = 0xFFFFFFFFu;
  best.id = 0xFFFFFFFFu;
  if (P.nlev == 0) return best;
  int top = 0;
  uint32_t cl = P.nlev - 1, cn = 0;  // current node: level, index
  double cb = INFINITY;
  bool have = true;
  for (;;) {
    if (!have) {
      if (top == 0) break;
      top--;
      const uint32_t e = stk.node[top];
      cl = e >> 26;
      cn = e & ((1u << 26) - 1);
      cb = stk.bound[top];
      __syncwarp();  // every lane has read the entry before any lane pushes over it
    }
    have = false;
    if (first_hit ? !(cb > thr) : (cb < best.val)) continue;
    if (cl == 0) {
      // leaf: 32 consecutive candidates
      const uint32_t p = cn * 32 + lane;
      double val = -INFINITY;
      uint32_t id = 0xFFFFFFFFu;
      if (p < P.m) {
        id = __ldg(&f.sid[p]);
        if (id != self) val = vdot(d, vsub(v3(__ldg(&f.sx[p]), __ldg(&f.sy[p]), __ldg(&f.sz[p])), v));
      }
      fs.scanned += 32;
      if (first_hit) {
        const uint32_t hit = __ballot_sync(0xFFFFFFFFu, val > thr);
        if (hit) {
          const int src = __ffs(hit) - 1;
          best.val = __shfl_sync(0xFFFFFFFFu, val, src);
          best.pos = __shfl_sync(0xFFFFFFFFu, p, src);
          best.id = __shfl_sync(0xFFFFFFFFu, id, src);
          return best;
        }
        continue;
      }
      if (!__ballot_sync(0xFFFFFFFFu, val >= best.val && val > -INFINITY)) continue;
      Sup sp;
      sp.val = val;
      sp.pos = p;
      sp.id = id;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const double ov = __shfl_xor_sync(0xFFFFFFFFu, sp.val, o);
        const uint32_t op = __shfl_xor_sync(0xFFFFFFFFu, sp.pos, o);
        const uint32_t oi = __shfl_xor_sync(0xFFFFFFFFu, sp.id, o);
        sup_merge(sp, ov, op, oi);
      }
      sup_merge(best, sp.val, sp.pos, sp.id);
      continue;
    }
    // inner node: bounds of its (up to) 32 children at level cl - 1
    const uint32_t chl = cl - 1;
    const uint32_t ch = cn * 32 + lane;
    double b = -INFINITY;
    if (ch < P.lnodes[chl]) {
      b = box_bound(f.nbox + (size_t)(P.loff[chl] + ch) * 6, d, v);
      // the slab only where the box does not already prune the child
      if (chl <= 1 && (first_hit ? b > thr : b >= best.val))
        b = fmin(b, vol_bound(f.nvol + (size_t)(P.loff[chl] + ch) * 9, d, v));
    }
    const bool pass = first_hit ? (b > thr) : (b >= best.val && b > -INFINITY);
    uint32_t mask = __ballot_sync(0xFFFFFFFFu, pass);
    if (!mask) continue;
    // descend into the child with the largest bound, push the others
    double mb = pass ? b : -INFINITY;
    int ml = lane;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double ob = __shfl_xor_sync(0xFFFFFFFFu, mb, o);
      const int oln = __shfl_xor_sync(0xFFFFFFFFu, ml, o);
      if (ob > mb || (ob == mb && oln < ml)) {
        mb = ob;
        ml = oln;
      }
    }
    mask &= ~(1u << ml);
    const uint32_t r = __popc(mask & lanemask_lt());
    if (((mask >> lane) & 1u) && top + (int)r < F_STACK) {
      stk.node[top + r] = (chl << 26) | ch;
      stk.bound[top + r] = b;
    }
    top = min(top + __popc(mask), F_STACK);
    __syncwarp();
    cl = chl;
    cn = cn * 32 + ml;
    cb = mb;
    have = true;
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

// GJK distance test of the origin against conv(U), U given by a support
// oracle sup(dir) -> (value, id, u) maximising dir.u.  Outcomes:
enum { GJK_OUTSIDE = 0, GJK_INSIDE = 1, GJK_AMBIGUOUS = 2, GJK_CAPPED = 3 };
struct SupU {
  double val;
  uint32_t id;  // 0xFFFFFFFF: empty set
  V3 u;
};

template <class SupFn>
__device__ int gjk(SupFn&& sup, SupU first, double eps, V3* sep, int* iters, int max_iters = 64) {
  V3 W[4];
  uint32_t id[4];
  int n = 1;
  W[0] = first.u;
  id[0] = first.id;
  V3 x = W[0];
#pragma unroll 1
  for (int it = 0; it < max_iters; it++) {
    const double xx = vdot(x, x);
    if (xx <= 0.0) return GJK_AMBIGUOUS;
    const V3 dir = vneg(x);
    (*iters)++;
    const SupU q = sup(dir);
    *sep = dir;
    if (q.id == 0xFFFFFFFFu) return GJK_OUTSIDE;
    // q.val = max_u (-x).u ; gap = x.x - min_u x.u = xx + q.val
    if (add(xx, q.val) <= 1e-13 * xx) return GJK_OUTSIDE;
    for (int k = 0; k < n; k++)
      if (id[k] == q.id) return GJK_OUTSIDE;  // no progress
    W[n] = q.u;
    id[n] = q.id;
    n++;
    if (n == 2) {
      x = closest_seg(W, id, n);
    } else if (n == 3) {
      x = closest_tri(W, id, n);
    } else {
      bool degen = false;
      if (closest_tet(W, id, n, x, degen)) return tet_depth(W) > eps ? GJK_INSIDE : GJK_AMBIGUOUS;
      if (degen) return GJK_AMBIGUOUS;
    }
    if (sqrt_(vdot(x, x)) <= eps) return GJK_AMBIGUOUS;  // within eps of the boundary
  }
  return GJK_CAPPED;
}

#ifndef F_LOCAL_N
#define F_LOCAL_N 4
#endif
constexpr int F_LOCAL = F_LOCAL_N;
#ifndef SH_F_EXTRA
#define SH_F_EXTRA 12
#endif
constexpr int F_EXTRA = SH_F_EXTRA;  // global points added to the local set  // local set: F_LOCAL * 32 sorted neighbours of the candidate

// 1 keep, 0 prune; *amb set when kept only because v is within eps of the
// boundary of the other candidates' hull (or the iteration cap was hit).
// direction of the certificate query: v - centre of the candidates' box
__device__ __forceinline__ V3 f_cert_dir(V3 v, V3 ctr, double* len) {
  V3 w0 = vsub(v, ctr);
  double wl = sqrt_(vdot(w0, w0));
  if (!(wl > 0.0)) {
    w0 = v3(1.0, 0.0, 0.0);
    wl = 1.0;
  }
  *len = wl;
  return w0;
}

// offsets of the 27 cells around a cell, nearest first: centre, 6 faces,
// 12 edges, 8 corners
__device__ __forceinline__ void f_nbr27(int t, int* dx, int* dy, int* dz) {
  // code per neighbour: 2 bits per axis (0: -1, 1: 0, 2: +1)
  constexpr unsigned char NB[27] = {0x15, 0x14, 0x16, 0x11, 0x19, 0x05, 0x25,              // centre, faces
                                    0x10, 0x12, 0x18, 0x1a, 0x04, 0x06, 0x24, 0x26,        // edges (x,y) and (x,z)
                                    0x01, 0x09, 0x21, 0x29,                                // edges (y,z)
                                    0x00, 0x02, 0x08, 0x0a, 0x20, 0x22, 0x28, 0x2a};       // corners
  const int c = NB[t];
  *dx = (c & 3) - 1;
  *dy = ((c >> 2) & 3) - 1;
  *dz = ((c >> 4) & 3) - 1;
}

__device__ __forceinline__ uint32_t f_axis_cell_p(const FilterParams& P, int k, double x) {
  const double t = (x - P.lo[k]) * P.inv_h[k];
  const int c = (int)t;
  return (uint32_t)(c < 0 ? 0 : (c >= (int)P.G ? (int)P.G - 1 : c));
}

// (1)-(3) for a candidate whose certificate query (k_f_cert) found the
// candidate s0 above v's radial plane
// mode 0: everything; mode 1: the first local GJK (k_f_local) already
// separated v from the local set along sep_in; mode 2: it was inconclusive,
// go straight to the global GJK; mode 3: the first local GJK only (returns
// 0 = pruned, 1 = separated along *sep_out, 2 = inconclusive)
template <int MODE>
__device__ int f_decide(const FilterWs& f, const FilterParams& P, uint32_t ps, uint32_t i, V3 v, V3 ctr,
                        V3 gsum, double eps, Sup s0, int* amb, int* capped, FStack& stk, FStat& fs,
                        V3 sep_in = V3{0.0, 0.0, 0.0}, V3* sep_out = nullptr) {
  const int lane = threadIdx.x & 31;
  double wl;
  const V3 w0 = f_cert_dir(v, ctr, &wl);
  long long tc = FCLK();
  int iters = 0;
  // (1) local GJK: the candidate's Morton neighbours plus the centroid of
  // all other candidates (a convex combination of them, so any simplex it
  // spans with candidates lies in their hull)
  if (MODE != 2) {
    // the local set: the candidates of the 27 grid cells around v (centre
    // cell, then faces, edges, corners), filled up with v's neighbours in
    // Morton order; F_LOCAL * 32 points
    const uint32_t lo = ps > 16u * F_LOCAL ? ps - 16u * F_LOCAL : 0u;
    uint32_t cstart = 0, ccnt = 0;
    if (lane < 27) {
      int dx, dy, dz;
      f_nbr27((int)lane, &dx, &dy, &dz);
      const int G = (int)P.G;
      const int cx = (int)f_axis_cell_p(P, 0, v.x) + dx, cy = (int)f_axis_cell_p(P, 1, v.y) + dy,
                cz = (int)f_axis_cell_p(P, 2, v.z) + dz;
      if (cx >= 0 && cy >= 0 && cz >= 0 && cx < G && cy < G && cz < G) {
        const uint32_t cell = spread3((uint32_t)cx) | (spread3((uint32_t)cy) << 1) | (spread3((uint32_t)cz) << 2);
        cstart = __ldg(&f.cell_start[cell]);
        ccnt = __ldg(&f.cell_start[cell + 1]) - cstart;
      }
    }
    uint32_t incl = ccnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if (lane >= o) incl += y;
    }
    const uint32_t ncell = __shfl_sync(0xFFFFFFFFu, incl, 31);
    const uint32_t excl = incl - ccnt;
    V3 lu[F_LOCAL];
    uint32_t lid[F_LOCAL];
#pragma unroll
    for (int k = 0; k < F_LOCAL; k++) {
      const uint32_t slot = k * 32 + lane;
      // the cell (lane) whose inclusive prefix first exceeds slot
      uint32_t a = 0;
#pragma unroll
      for (int step = 16; step; step >>= 1) {
        const uint32_t pv = __shfl_sync(0xFFFFFFFFu, incl, (int)(a + step - 1));
        if (pv <= slot) a += step;
      }
      const uint32_t st0 = __shfl_sync(0xFFFFFFFFu, cstart, (int)(a & 31u));
      const uint32_t ex0 = __shfl_sync(0xFFFFFFFFu, excl, (int)(a & 31u));
      const uint32_t p = slot < ncell ? st0 + (slot - ex0) : lo + (slot - ncell);
      lid[k] = 0xFFFFFFFFu;
      lu[k] = v3(0.0, 0.0, 0.0);
      if (p < P.m && p != ps) {
        lid[k] = __ldg(&f.sid[p]);
        lu[k] = vsub(v3(__ldg(&f.sx[p]), __ldg(&f.sy[p]), __ldg(&f.sz[p])), v);
      }
    }
    const double inv = 1.0 / (double)(P.m - 1);
    const V3 g = vsub(v3(mul(sub(gsum.x, v.x), inv), mul(sub(gsum.y, v.y), inv), mul(sub(gsum.z, v.z), inv)), v);
    // points found above a separating plane of the local set join it (one
    // per lane, up to F_EXTRA) and the local GJK is rerun: most candidates
    // the local set can not decide are settled after one or two of these
    // existence queries instead of a global GJK
    V3 ex_u = v3(0.0, 0.0, 0.0);
    uint32_t ex_id = 0xFFFFFFFFu;
    int nex = 0;
    auto local_sup = [&](V3 d) -> SupU {
      double bv = -INFINITY;
      uint32_t bid = 0xFFFFFFFFu;
      int bk = -1;
#pragma unroll
      for (int k = 0; k < F_LOCAL; k++) {
        const double val = vdot(d, lu[k]);
        if (lid[k] != 0xFFFFFFFFu && (val > bv || (val == bv && lid[k] < bid))) {
          bv = val;
          bid = lid[k];
          bk = k;
        }
      }
      if (lane == 0) {  // the centroid, id 0xFFFFFFFE
        const double val = vdot(d, g);
        if (val > bv) {
          bv = val;
          bid = 0xFFFFFFFEu;
          bk = F_LOCAL;
        }
      }
      if (lane < nex) {  // global points found above earlier separating planes
        const double val = vdot(d, ex_u);
        if (val > bv || (val == bv && ex_id < bid)) {
          bv = val;
          bid = ex_id;
          bk = F_LOCAL + 1;
        }
      }
      int bl = lane;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const double ov = __shfl_xor_sync(0xFFFFFFFFu, bv, o);
        const uint32_t oi = __shfl_xor_sync(0xFFFFFFFFu, bid, o);
        const int ol = __shfl_xor_sync(0xFFFFFFFFu, bl, o);
        if (ov > bv || (ov == bv && oi < bid)) {
          bv = ov;
          bid = oi;
          bl = ol;
        }
      }
      const int kk = __shfl_sync(0xFFFFFFFFu, bk, bl);
      V3 u = g;
#pragma unroll
      for (int k = 0; k < F_LOCAL; k++)
        if (kk == k) u = lu[k];
      if (kk == F_LOCAL + 1) u = ex_u;
      SupU r;
      r.val = bv;
      r.id = bid;
      r.u = v3(__shfl_sync(0xFFFFFFFFu, u.x, bl), __shfl_sync(0xFFFFFFFFu, u.y, bl),
               __shfl_sync(0xFFFFFFFFu, u.z, bl));
      return r;
    };
    // start from the candidate above v's radial plane found by (0)
    SupU first;
    first.val = s0.val;
    first.id = s0.id;
    first.u = vsub(v3(f.sx[s0.pos], f.sy[s0.pos], f.sz[s0.pos]), v);
    V3 sep = w0;
#pragma unroll 1
    for (int xr = 0; xr <= F_EXTRA; xr++) {
      iters = 0;
      int r;
      if (MODE == 1 && xr == 0) {
        r = GJK_OUTSIDE;
        sep = sep_in;
      } else {
        r = gjk(local_sup, first, eps, &sep, &iters);
      }
      fs.iters += iters;
      if (MODE == 3) {
        if (r == GJK_INSIDE) fs.local_in++;
        *sep_out = sep;
        return r == GJK_INSIDE ? 0 : (r == GJK_OUTSIDE ? 1 : 2);
      }
      {
        const long long t2 = FCLK();
        fs.cyc_local += (unsigned long long)(t2 - tc);
        tc = t2;
      }
      if (r == GJK_INSIDE) {
        fs.local_in++;
        return 0;  // strictly inside the hull of other candidates
      }
      if (r != GJK_OUTSIDE) break;
      // (2) separated from the local set along sep: one global existence query
      const double thr = mul(eps, sqrt_(vdot(sep, sep)));
      const Sup c = support_query(f, P, sep, v, i, thr, true, stk, fs);
      {
        const long long t2 = FCLK();
        fs.cyc_out += (unsigned long long)(t2 - tc);
        tc = t2;
      }
      if (!(c.val > thr)) {
        fs.local_out++;
        return 1;  // no candidate above the plane: extreme
      }
      if (xr == F_EXTRA) break;
      const V3 cu = vsub(v3(f.sx[c.pos], f.sy[c.pos], f.sz[c.pos]), v);
      if (lane == nex) {
        ex_u = cu;
        ex_id = c.id;
      }
      nex++;
      first.val = c.val;
      first.id = c.id;
      first.u = cu;
    }
  }
  if (MODE == 3) return 2;
  fs.fallback++;
  struct CycGuard {
    FStat& s;
    long long t;
    __device__ ~CycGuard() { s.cyc_fallback += (unsigned long long)(FCLK() - t); }
  } guard{fs, FCLK()};
  // (3) global GJK, started from the candidate farthest along v - centre
  const Sup s = support_query(f, P, w0, v, i, 0.0, false, stk, fs);
  if (s.pos == 0xFFFFFFFFu) return 1;
  // global GJK on U = {c - v : c != v} (branch-and-bound support queries)
  auto global_sup = [&](V3 d) -> SupU {
    const Sup q = support_query(f, P, d, v, i, 0.0, false, stk, fs);
    SupU r;
    r.val = q.val;
    r.id = q.id;
    r.u = q.pos == 0xFFFFFFFFu ? v3(0.0, 0.0, 0.0)
                               : vsub(v3(f.sx[q.pos], f.sy[q.pos], f.sz[q.pos]), v);
    return r;
  };
  SupU first;
  first.val = s.val;
  first.id = s.id;
  first.u = vsub(v3(f.sx[s.pos], f.sy[s.pos], f.sz[s.pos]), v);
  V3 sep;
  iters = 0;
  // the last resort: a generous iteration cap (a capped GJK keeps the
  // candidate, which is conservative; the tests assert it never happens)
  const int r = gjk(global_sup, first, eps, &sep, &iters, 1024);
  fs.iters += iters;
  if (r == GJK_INSIDE) return 0;
  if (r == GJK_AMBIGUOUS) *amb = 1;
  if (r == GJK_CAPPED) *capped = 1;
  return 1;
}

// (0) certificate queries, one warp per candidate (Morton order): a light
// kernel (the support query only) at high occupancy; the candidates it
// does not settle go to a work list for k_f_test
#ifndef SH_FCERT_MINB
#define SH_FCERT_MINB 8
#endif
__global__ void __launch_bounds__(F_TEST_BLOCK, SH_FCERT_MINB) k_f_cert(Workspace ws, FilterWs f) {
  __shared__ FilterParams sP;
  __shared__ FStack s_stk[F_TEST_BLOCK / 32];
  if (threadIdx.x == 0) sP = *f.fp;
  __syncthreads();
  const FilterParams& P = sP;
  const uint32_t m = P.m;
  const double eps = ws.st->eps;
  const V3 ctr = v3(P.ctr[0], P.ctr[1], P.ctr[2]);
  const int lane = threadIdx.x & 31;
  FStack& stk = s_stk[threadIdx.x >> 5];
  FStat fs = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (;;) {
    uint32_t ps = 0;
    if (lane == 0) ps = atomicAdd(&f.fp->ctr_test, 1u);
    ps = __shfl_sync(0xFFFFFFFFu, ps, 0);
    if (ps >= m) break;
    const uint32_t i = __ldg(&f.sid[ps]);
    if (m <= 4 || i < P.share_lo || i >= P.share_hi) {  // quickhull.py:148-149; another share's
      if (lane == 0) f.keep[i] = 1;
      continue;
    }
    const V3 v = v3(f.cx[i], f.cy[i], f.cz[i]);
    double wl;
    const V3 w0 = f_cert_dir(v, ctr, &wl);
    const double thr0 = mul(eps, wl);
    const long long tc = FCLK();
    const Sup s0 = support_query(f, P, w0, v, i, thr0, true, stk, fs);
    fs.cyc_cert += (unsigned long long)(FCLK() - tc);
    if (lane == 0) {
      if (!(s0.val > thr0)) {
        f.keep[i] = 1;
        fs.certified++;
      } else {
        const uint32_t k = atomicAdd(&f.fp->nwl, 1u);
        f.wl_ps[k] = ps;
        f.wl_pos[k] = s0.pos;
        f.wl_id[k] = s0.id;
        f.wl_val[k] = s0.val;
      }
    }
  }
  if (lane == 0 && fs.queries) {
    atomicAdd(&f.fp->queries, fs.queries);
    atomicAdd(&f.fp->scanned, fs.scanned);
    atomicAdd(&f.fp->certified, fs.certified);
    atomicAdd(&f.fp->cyc_cert, fs.cyc_cert);
  }
}

#ifndef SH_FTEST_MINB
#define SH_FTEST_MINB 4
#endif
// the first local GJK for the work list of k_f_cert: pruned candidates are
// settled here, the rest go to a second work list with the outcome
__global__ void __launch_bounds__(F_TEST_BLOCK, SH_FTEST_MINB) k_f_local(Workspace ws, FilterWs f) {
  __shared__ FilterParams sP;
  __shared__ FStack s_stk[F_TEST_BLOCK / 32];
  if (threadIdx.x == 0) sP = *f.fp;
  __syncthreads();
  const FilterParams& P = sP;
  const uint32_t nwl = P.nwl;
  const double eps = ws.st->eps;
  const V3 ctr = v3(P.ctr[0], P.ctr[1], P.ctr[2]);
  const V3 gsum = v3(P.gsum[0], P.gsum[1], P.gsum[2]);
  const int lane = threadIdx.x & 31;
  FStack& stk = s_stk[threadIdx.x >> 5];
  FStat fs = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (;;) {
    uint32_t k = 0;
    if (lane == 0) k = atomicAdd(&f.fp->ctr_wl, 1u);
    k = __shfl_sync(0xFFFFFFFFu, k, 0);
    if (k >= nwl) break;
    const uint32_t ps = f.wl_ps[k];
    const uint32_t i = __ldg(&f.sid[ps]);
    Sup s0;
    s0.pos = f.wl_pos[k];
    s0.id = f.wl_id[k];
    s0.val = f.wl_val[k];
    int amb = 0, capped = 0;
    V3 sep;
    const int r = f_decide<3>(f, P, ps, i, v3(f.cx[i], f.cy[i], f.cz[i]), ctr, gsum, eps, s0, &amb, &capped,
                              stk, fs, V3{0.0, 0.0, 0.0}, &sep);
    if (lane == 0) {
      if (r == 0) {
        f.keep[i] = 0;
      } else {
        const uint32_t j = atomicAdd(&f.fp->nwl2, 1u);
        f.wl2_k[j] = k | (r == 2 ? 0x80000000u : 0u);
        f.wl2_sep[3 * j + 0] = sep.x;
        f.wl2_sep[3 * j + 1] = sep.y;
        f.wl2_sep[3 * j + 2] = sep.z;
      }
    }
  }
  if (lane == 0 && fs.iters) {
    atomicAdd(&f.fp->gjk_iters, fs.iters);
    atomicAdd(&f.fp->local_in, fs.local_in);
  }
}

// (2)-(3) for the candidates the first local GJK separated or could not decide
__global__ void __launch_bounds__(F_TEST_BLOCK, SH_FTEST_MINB) k_f_test(Workspace ws, FilterWs f) {
  __shared__ FilterParams sP;
  __shared__ FStack s_stk[F_TEST_BLOCK / 32];
  if (threadIdx.x == 0) sP = *f.fp;
  __syncthreads();
  const FilterParams& P = sP;
  const uint32_t nwl2 = P.nwl2;
  const double eps = ws.st->eps;
  const V3 ctr = v3(P.ctr[0], P.ctr[1], P.ctr[2]);
  const V3 gsum = v3(P.gsum[0], P.gsum[1], P.gsum[2]);
  const int lane = threadIdx.x & 31;
  FStack& stk = s_stk[threadIdx.x >> 5];
  int amb_count = 0, cap_count = 0;
  FStat fs = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (;;) {
    uint32_t j = 0;
    if (lane == 0) j = atomicAdd(&f.fp->ctr_wl2, 1u);
    j = __shfl_sync(0xFFFFFFFFu, j, 0);
    if (j >= nwl2) break;
#ifdef SH_FILTER_CYCLES
    const long long t_item = clock64();
    const unsigned long long it0 = fs.iters, q0 = fs.queries, sc0 = fs.scanned;
#endif
    const uint32_t kk = f.wl2_k[j];
    const uint32_t k = kk & 0x7FFFFFFFu;
    const uint32_t ps = f.wl_ps[k];
    const uint32_t i = __ldg(&f.sid[ps]);
    Sup s0;
    s0.pos = f.wl_pos[k];
    s0.id = f.wl_id[k];
    s0.val = f.wl_val[k];
    const V3 v = v3(f.cx[i], f.cy[i], f.cz[i]);
    int amb = 0, capped = 0, keep;
    if (kk & 0x80000000u) {
      keep = f_decide<2>(f, P, ps, i, v, ctr, gsum, eps, s0, &amb, &capped, stk, fs);
    } else {
      const V3 sep = v3(f.wl2_sep[3 * j + 0], f.wl2_sep[3 * j + 1], f.wl2_sep[3 * j + 2]);
      keep = f_decide<1>(f, P, ps, i, v, ctr, gsum, eps, s0, &amb, &capped, stk, fs, sep);
    }
    if (lane == 0) {
      f.keep[i] = (uint8_t)keep;
      amb_count += amb;
      cap_count += capped;
#ifdef SH_FILTER_CYCLES
      const unsigned long long dt = (unsigned long long)(clock64() - t_item);
      int bkt = 63 - __clzll((long long)(dt | 1ull)) - 10;
      atomicAdd(&f.fp->dur_hist[bkt < 0 ? 0 : (bkt > 19 ? 19 : bkt)], 1u);
      if (dt > atomicMax(&f.fp->dur_max, dt)) {  // racy record of the slowest item (diagnostics)
        f.fp->dur_max_iters = fs.iters - it0;
        f.fp->dur_max_queries = fs.queries - q0;
        f.fp->dur_max_scanned = fs.scanned - sc0;
      }
#endif
    }
  }
  if (lane == 0 && amb_count) atomicAdd(&f.fp->ambiguous, (uint32_t)amb_count);
  if (lane == 0 && cap_count) atomicAdd(&f.fp->gjk_capped, (uint32_t)cap_count);
  if (lane == 0 && fs.queries) {
    atomicAdd(&f.fp->queries, fs.queries);
    atomicAdd(&f.fp->scanned, fs.scanned);
    atomicAdd(&f.fp->gjk_iters, fs.iters);
    atomicAdd(&f.fp->local_in, fs.local_in);
    atomicAdd(&f.fp->local_out, fs.local_out);
    atomicAdd(&f.fp->fallback, fs.fallback);
    atomicAdd(&f.fp->cyc_local, fs.cyc_local);
    atomicAdd(&f.fp->cyc_out, fs.cyc_out);
    atomicAdd(&f.fp->cyc_fallback, fs.cyc_fallback);
  }
}

// ------------------------------------------------------------------ F6
// Kept candidates -> user indices in discovery order: each block of
// k_f_ccount counts the kept ones of its slice; each block of k_f_compact
// writes its slice at the total of the slices before it.
constexpr uint32_t F_COMPACT_GRID = 128;

__global__ void __launch_bounds__(1024) k_f_ccount(FilterWs f) {
  __shared__ uint32_t s_w[32];
  const uint32_t m = f.fp->m;
  const uint32_t p0 = (uint32_t)(((uint64_t)m * blockIdx.x) / gridDim.x);
  const uint32_t p1 = (uint32_t)(((uint64_t)m * (blockIdx.x + 1)) / gridDim.x);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t c = 0;
  for (uint32_t i = p0 + threadIdx.x; i < p1; i += 1024) c += f.keep[i] ? 1u : 0u;
  c = __reduce_add_sync(0xFFFFFFFFu, c);
  if (lane == 0) s_w[warp] = c;
  __syncthreads();
  if (warp == 0) {
    const uint32_t t = __reduce_add_sync(0xFFFFFFFFu, s_w[lane]);
    if (lane == 0) f.wl_pos[blockIdx.x] = t;  // free after k_f_test
  }
}

__global__ void __launch_bounds__(1024) k_f_compact(Workspace ws, FilterWs f) {
  static_assert(F_COMPACT_GRID <= 1024, "one count per thread");
  __shared__ uint32_t s_w[32], s_b[32], s_a[32];
  __shared__ uint32_t s_carry, s_total;
  const uint32_t m = f.fp->m;
  int64_t* out = ws.st->out_idx;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  {  // kept candidates before this slice and in all slices
    const uint32_t t = threadIdx.x < gridDim.x ? f.wl_pos[threadIdx.x] : 0u;
    const uint32_t before = __reduce_add_sync(0xFFFFFFFFu, threadIdx.x < blockIdx.x ? t : 0u);
    const uint32_t all = __reduce_add_sync(0xFFFFFFFFu, t);
    if (lane == 0) {
      s_b[warp] = before;
      s_a[warp] = all;
    }
    __syncthreads();
    if (warp == 0) {
      const uint32_t b2 = __reduce_add_sync(0xFFFFFFFFu, s_b[lane]);
      const uint32_t a2 = __reduce_add_sync(0xFFFFFFFFu, s_a[lane]);
      if (lane == 0) {
        s_carry = b2;
        s_total = a2;
      }
    }
    __syncthreads();
  }
  const uint32_t p0 = (uint32_t)(((uint64_t)m * blockIdx.x) / gridDim.x);
  const uint32_t p1 = (uint32_t)(((uint64_t)m * (blockIdx.x + 1)) / gridDim.x);
  for (uint32_t base = p0; base < p1; base += 1024) {
    const uint32_t i = base + threadIdx.x;
    const uint32_t v = (i < p1 && f.keep[i]) ? 1u : 0u;
    const uint32_t bal = __ballot_sync(0xFFFFFFFFu, v);
    if (lane == 0) s_w[warp] = __popc(bal);
    __syncthreads();
    if (warp == 0) {
      const uint32_t w = s_w[lane];
      uint32_t y = w;
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t z = __shfl_up_sync(0xFFFFFFFFu, y, o);
        if (lane >= o) y += z;
      }
      s_w[lane] = y - w;
    }
    __syncthreads();
    const uint32_t pos = s_carry + s_w[warp] + __popc(bal & lanemask_lt());
    if (v) out[pos] = (int64_t)ws.vout[i];
    __syncthreads();
    if (threadIdx.x == 1023) s_carry = pos + v;
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    f.result[0] = s_total;
    f.result[1] = 0;
    f.result[2] = 1;
    f.result[3] = f.fp->ambiguous;
    f.result[4] = 0;
  }
}

static inline int filter_launch(FilterWs& f, Workspace ws, int nsm, cudaStream_t s) {
  const int grid = nsm * 4;
  k_f_setup<<<grid, BLOCK, 0, s>>>(ws, f);
  k_f_gather<<<grid, BLOCK, 0, s>>>(ws, f);
  k_f_count<<<grid, BLOCK, 0, s>>>(ws, f);
  k_f_scan_tiles<<<F_SCAN_GRID, 1024, 0, s>>>(f);
  k_f_scan<<<F_SCAN_GRID, 1024, 0, s>>>(f);
  k_f_scatter<<<grid, BLOCK, 0, s>>>(f);
  k_f_boxes01<<<nsm * 2, 1024, 0, s>>>(f);
  k_f_boxes_hi<<<1, 1024, 0, s>>>(f);
  k_f_vols<<<nsm * 4, BLOCK, 0, s>>>(f);
  k_f_cert<<<nsm * 16, F_TEST_BLOCK, 0, s>>>(ws, f);
  k_f_local<<<nsm * 8, F_TEST_BLOCK, 0, s>>>(ws, f);
  k_f_test<<<nsm * 8, F_TEST_BLOCK, 0, s>>>(ws, f);
  k_f_ccount<<<F_COMPACT_GRID, 1024, 0, s>>>(f);
  k_f_compact<<<F_COMPACT_GRID, 1024, 0, s>>>(ws, f);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : 10;
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
