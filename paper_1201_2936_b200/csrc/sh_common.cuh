// Shared device-side types for the B200 Quickhull path.
//
// Data layout in HBM:
//   * live points of a round are structure-of-arrays records
//     (x, y[, z] fp64 + uint32 original index).  Each ping-pong buffer has
//     K = dim "streams" of capacity rcap; child (p, s) -- the survivors of
//     segment p with child state s -- is written to stream s at
//     [segstart[p], segstart[p] + count): disjoint per parent, contiguous per
//     child, gaps between children.  The next round addresses its segments
//     through seg_phys (physical element offset of the segment's first
//     record) and a dense logical numbering (segstart), so it never reads a
//     gap.  Within a child the order is free (original indices are carried).
//   * segments are numbered parent-major (child id e = p*K + s), which is the
//     reference's flat-array segment order (flag_permute's stable (parent,
//     state) grouping, primitives.py:105-116), so vertices come out in the
//     reference's discovery order.
//   * per-segment tables (Seg2 / Seg3) hold everything a point needs to be
//     classified against its segment's simplex, built once per segment by
//     the bookkeeping kernel (K3), never per element (the reference gathers
//     the per-segment edge/face data to every element, quickhull.py:231-233,
//     :373-375).
//   * per child: a write cursor (survivor count = cursor - parent start) and
//     the farthest-point key, both merged with atomics.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "sh_numerics.cuh"

namespace sh {

constexpr int BLOCK = 256;
constexpr int WARPS = BLOCK / 32;
constexpr int ITEMS = 8;             // points per thread per tile (round kernel)
constexpr int TILE = BLOCK * ITEMS;  // 2048 points per tile
constexpr int ITEMS3 = 4;            // children per thread per tile (bookkeeping kernel)
constexpr int TILE3 = BLOCK * ITEMS3;
constexpr int MAX_TRACE = 4096;      // per-round counters kept on device
#ifndef SH_RB
#define SH_RB 128
#endif
#ifndef SH_RITEMS
#define SH_RITEMS 4
#endif
constexpr int RB = SH_RB;            // threads per round-kernel block
constexpr int RITEMS = SH_RITEMS;    // points per thread per round tile
constexpr int RTILE = RB * RITEMS;   // 1024 points per round tile
constexpr int WMAX = 128;            // tile-window segments kept in shared memory
constexpr uint32_t BOOK_SMALL = 1024; // children handled by a single K3 block

// status codes (C ABI, include/seghull_b200.h)
constexpr uint32_t ST_OK = 0;
constexpr uint32_t ST_EMPTY = 2;
constexpr uint32_t ST_DEGENERATE = 3;
constexpr uint32_t ST_ROUND_GUARD = 4;
constexpr uint32_t ST_SEG_OVERFLOW = 6;
constexpr uint32_t ST_NONFINITE = 8;

constexpr uint32_t FL_COLLINEAR = 1;

// sharded hulls: statistics record layout and flags (include/seghull_b200.h)
constexpr int STATS_N = 14;           // -lo[3], hi[3], lexmin[4], lexmax[4] (SH_STATS)
constexpr uint32_t SHARD_EPS = 1;     // eps = eps_rel * hypot(spans of the global bbox)
constexpr uint32_t SHARD_SPLIT = 2;   // first-split line through the global lexicographic extremes

// Original index of a padding record.  The streaming round kernel claims
// output in multiples of 4 records (16-byte aligned runs, written by bulk
// copies) and fills the rest of a claim with DEAD records; the bookkeeping
// kernel pads every segment to a multiple of 4 the same way.  Every round
// kernel drops DEAD records on read, and the per-round traces count live
// records only.  (Original indices are < 2^31.)
constexpr uint32_t DEAD = 0xFFFFFFFFu;

// Farthest-point aggregate of a run of points (one child segment).
// Larger `hi` (order-preserving bits of the distance) wins, ties go to the
// lowest original index (quickhull.py:93-100: first max in a segment whose
// elements are in ascending original-index order).  cnt sums.
// 128-bit farthest-point key in a child slot: (hi, idx) with larger hi
// winning and ties going to the lower index.
struct __align__(16) Key128 {
  unsigned long long hi;
  unsigned long long lo;  // original index
};

struct __align__(16) RunVal {
  uint64_t hi;
  uint32_t idx;
  uint32_t cnt;
};

SH_HD RunVal rv_merge(RunVal a, RunVal b) {
  RunVal r;
  bool take_b = (b.hi > a.hi) || (b.hi == a.hi && b.idx < a.idx);
  r.hi = take_b ? b.hi : a.hi;
  r.idx = take_b ? b.idx : a.idx;
  r.cnt = a.cnt + b.cnt;
  return r;
}

struct __align__(16) Sum3 {
  uint32_t v[4];
};

SH_HD Sum3 s3_identity() { Sum3 s; s.v[0] = s.v[1] = s.v[2] = s.v[3] = 0; return s; }
SH_HD Sum3 s3_combine(Sum3 a, Sum3 b) {
  Sum3 r;
  for (int i = 0; i < 4; i++) r.v[i] = a.v[i] + b.v[i];
  return r;
}

// 2D segment: directed split edge a->b (points lie left of it), its
// farthest point f, the constant terms of the two cross products a point is
// classified with (cross2(a, f, q) and cross2(f, b, q), geometry.py:121:
// ay - fy and fy - by) and the two pre-scaled triangle thresholds
// (-eps)*|edge| of point_in_triangle (geometry.py:150-156).  Pairs are laid
// out for 16-byte shared-memory loads.
struct __align__(16) Seg2 {
  double ax, ay, fx, fy, bx, by;
  double d_af, d_fb;
  double nt_bf, nt_fa;
  uint32_t fidx, pad;
};

// 3D segment: face (a, b, c) with outward normal n = (b-a)x(c-a), far point
// f, and the three side faces (a,b,f), (b,c,f), (c,a,f) of the tetrahedron
// (geometry.py:163-175) with their normals, norms and eps thresholds.
struct __align__(16) Seg3 {
  double a[3], b[3], c[3];
  double n[3];
  double nt_base;  // (-eps) * |n|
  double f[3];
  double N[3][3];
  double nrm[3];   // |N_j|
  double thr[3];   // eps * |N_j|
  uint32_t fidx, flat;
};

// Parameters of one round, read by the round kernel (K2) and the
// bookkeeping kernel (K3) that follows it.  Only K3's finalising tile
// writes the next round's parameters, after every K3 block has read them
// (arrival counter), so no block ever sees a half-updated set.
struct RoundParams {
  uint32_t active;
  uint32_t root;          // 1: the first split (K1)
  uint32_t n_live;        // points entering the round (logical positions)
  uint32_t nseg;          // segments of the round (parents of its children)
  uint32_t cur;           // ping-pong index of the buffers the round reads
  uint32_t h;             // vertices emitted before this round's children
  uint32_t round;         // 0: first split, r: loop round r
  uint32_t n_true;        // live points entering the round (n_live counts DEAD padding too)
  uint32_t aligned;       // segments start 4-record aligned: k_stream may take the round (k_book)
  uint32_t pad;
};

struct DevState {
  // ---- call parameters (host -> device before every launch) ----
  const double* px;
  const double* py;
  const double* pz;
  int64_t stride;         // element stride of the coordinate arrays
  uint32_t n;
  uint32_t dim;
  double eps_rel;
  double eps_abs;
  uint32_t use_eps_abs;
  uint32_t segcap;        // capacity of segment tables
  int64_t* out_idx;       // user output (device), capacity n
  int32_t* out_facets;    // 3D facet triples (device), NULL = not requested
  int64_t facet_cap;      // triples out_facets can hold
  uint32_t long_min_live; // k_stream long-round thresholds (long_round(); env overrides for tests)
  uint32_t long_seg_min;
  uint32_t filter_share, filter_nshares;  // 3D filter decides only sorted candidates of share r of R (sh_set_filter_share)
  // sharded hulls (sh_set_shard): the all-ranks statistics (device, SH_STATS
  // doubles: -lo[3], hi[3], lex-min and lex-max records (x, y, z, global
  // index)), this slice's first global index, SHARD_* flags
  const double* gstats;
  int64_t gidx_offset;
  uint32_t shard_flags;
  uint32_t defer_first;   // two-stage sharded hull: K0 stops after the reduction (k_shard_apply finishes it)
  double* stats_out;      // two-stage sharded hull: K0 writes this slice's statistics here
  // ---- first split (K0/K0b) ----
  double eps;
  uint32_t imin, imax, ifar;
  uint32_t first_active;
  double pa[3], pb[3], pc[3];
  double nrm[3];
  double nlen;
  double thr_line;        // 2D: eps*|pmax-pmin|; 3D: (-eps)*nlen
  uint64_t dmax_bits;     // 3D coplanarity check: max |d| over the first split
  // ---- loop ----
  RoundParams rp;
  uint32_t status;
  uint32_t flags;
  uint32_t h_final;
  uint32_t rounds_final;
  uint32_t seg_needed;    // largest segment count requested (overflow retry)
  uint32_t seq;           // look-back tag of the bookkeeping kernel
  uint32_t ctr_book;      // dynamic tile counter of K3 (reset by K2)
  uint32_t arrive_book;   // K3 blocks that have read rp (reset by K3's finalizer)
  uint32_t ctr_red;       // last-block counter for reductions
  uint32_t book_small;    // K3 runs in one block (few children); set by K2
  uint32_t nonfinite;     // K0 saw a NaN / inf coordinate
  uint32_t dead_round;    // DEAD padding records written by the current round (k_stream)
  // K0's reduction of this slice, kept for k_shard_apply (two-stage hull)
  double keep_lo[3], keep_hi[3], keep_mn[3], keep_mx[3];
  uint32_t keep_imn, keep_imx;
  // ---- traces (per round r, index r-1) ----
  uint32_t tr_live[MAX_TRACE];
  uint32_t tr_kept[MAX_TRACE];
  uint32_t tr_nseg[MAX_TRACE];
  uint32_t tr_flat[MAX_TRACE];
};

// Device buffers of one context (all allocated once, sized for n / segcap).
struct Workspace {
  DevState* st;
  // live records, ping-pong, K streams of capacity rcap each
  double* rx[2];
  double* ry[2];
  double* rz[2];
  uint32_t* ri[2];
  uint64_t rcap;
  // segment tables (ping-pong, dense segment ids)
  void* seg[2];
  uint32_t* segstart[2];   // dense logical start (+ sentinel = n_live)
  uint64_t* seg_phys[2];   // physical element offset of the first record
  // per child (e = parent*K + state) of the round reading buffer b:
  uint32_t* cursor[2];     // write cursor, initialised to the parent's start
  Key128* slot_key;        // farthest key, zero between uses
  // decoupled look-back status words of K3, [tiles][4]
  uint64_t* lb_book;
  uint64_t lb_book_words;
  // vertex output (uint32 original indices)
  uint32_t* vout;
  // reduction partials
  double* red;               // per block partial records
  uint32_t red_blocks;
  uint32_t round_grid;
  uint32_t book_grid;
  uint32_t max_tiles;     // round tiles at capacity
  cudaGraphConditionalHandle cond;
  uint32_t use_cond;
  uint32_t peeled;        // launch outside the WHILE loop (first rounds): k_stream may take the round
  uint32_t slack;         // round 1: extra room before side 1's children (their claims are padded per tile)
  uint32_t stream_grid;   // k_stream launch: CTAs, points per tile
  uint32_t stream_T;
};

// Rounds >= 2 whose segments are long run the streaming kernel
// (k_stream<SRC_REC>, sh_stream.cuh); the others run k_round.  The first
// LONG_PEEL loop rounds are launched outside the CUDA graph's WHILE node as
// the pair (k_stream, k_round), exactly one of which works; inside the WHILE
// node only k_round runs, so the later, short rounds pay no extra launch.
constexpr uint32_t LONG_SEG_MIN = 4096;
constexpr uint32_t LONG_MIN_LIVE = 4u << 20;
#ifndef SH_LONG_PEEL
#define SH_LONG_PEEL 5
#endif
constexpr int LONG_PEEL = SH_LONG_PEEL;  // rounds 2..6 are launched outside the WHILE loop

// ---------------------------------------------------------------- helpers
__device__ __forceinline__ unsigned long long pow2_dev(unsigned long long x) {
  unsigned long long p = 1;
  while (p < x) p <<= 1;
  return p;
}

__device__ __forceinline__ uint64_t ld_volatile_u64(const uint64_t* p) {
  return *(const volatile uint64_t*)p;
}
__device__ __forceinline__ void st_volatile_u64(uint64_t* p, uint64_t v) {
  *(volatile uint64_t*)p = v;
}

template <class T>
__device__ __forceinline__ T ld_cg(const T* p) {
  static_assert(sizeof(T) % 16 == 0, "16B payloads");
  T r;
  const uint4* s = reinterpret_cast<const uint4*>(p);
  uint4* d = reinterpret_cast<uint4*>(&r);
#pragma unroll
  for (int i = 0; i < (int)(sizeof(T) / 16); i++) d[i] = __ldcg(s + i);
  return r;
}

template <class T>
__device__ __forceinline__ void st_cg(T* p, const T& v) {
  static_assert(sizeof(T) % 16 == 0, "16B payloads");
  uint4* d = reinterpret_cast<uint4*>(p);
  const uint4* s = reinterpret_cast<const uint4*>(&v);
#pragma unroll
  for (int i = 0; i < (int)(sizeof(T) / 16); i++) __stcg(d + i, s[i]);
}

__device__ __forceinline__ double ld_coord(const double* p, int64_t stride, uint32_t i) {
  return __ldg(p + (int64_t)i * stride);
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

template <class T>
__device__ __forceinline__ T shfl_up_t(T v, int off) {
  static_assert(sizeof(T) % 4 == 0, "");
  T r;
  const uint32_t* s = reinterpret_cast<const uint32_t*>(&v);
  uint32_t* d = reinterpret_cast<uint32_t*>(&r);
#pragma unroll
  for (int i = 0; i < (int)(sizeof(T) / 4); i++) d[i] = __shfl_up_sync(0xFFFFFFFFu, s[i], off);
  return r;
}

template <class T>
__device__ __forceinline__ T shfl_t(T v, int src) {
  static_assert(sizeof(T) % 4 == 0, "");
  T r;
  const uint32_t* s = reinterpret_cast<const uint32_t*>(&v);
  uint32_t* d = reinterpret_cast<uint32_t*>(&r);
#pragma unroll
  for (int i = 0; i < (int)(sizeof(T) / 4); i++) d[i] = __shfl_sync(0xFFFFFFFFu, s[i], src);
  return r;
}

template <class T>
__device__ __forceinline__ T shfl_down_t(T v, int off) {
  static_assert(sizeof(T) % 4 == 0, "");
  T r;
  const uint32_t* s = reinterpret_cast<const uint32_t*>(&v);
  uint32_t* d = reinterpret_cast<uint32_t*>(&r);
#pragma unroll
  for (int i = 0; i < (int)(sizeof(T) / 4); i++) d[i] = __shfl_down_sync(0xFFFFFFFFu, s[i], off);
  return r;
}

// ------------------------------------------------------------------------
// Count-only decoupled look-back (the hot-path variant).
// One 64-bit status word per (tile, counter): [tag:16][flag:2][count:46].
// The count travels inside the status word, so a reader needs exactly one
// load per predecessor and no memory fence; every counter is an independent
// chained scan.  Tags (1..65535, never 0) separate launches, the arrays are
// zeroed at allocation and re-zeroed by k_init before the tag space wraps.
constexpr uint64_t LB_AGG = 1, LB_INC = 2;

__device__ __forceinline__ uint64_t ld_relaxed_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint64_t lb_word(uint32_t tag, uint64_t flag, uint32_t count) {
  return ((uint64_t)tag << 48) | (flag << 46) | (uint64_t)count;
}

template <int NC>
__device__ __forceinline__ void lb_publish(uint64_t* st, uint32_t tile, uint32_t tag, uint64_t flag,
                                           const uint32_t* cnt) {
#pragma unroll
  for (int c = 0; c < NC; c++) st_relaxed_u64(&st[(size_t)tile * 4 + c], lb_word(tag, flag, cnt[c]));
}

// All threads of the block call this.  On return s_prefix[0..NC) holds the
// exclusive prefix of `tile` for every counter.
template <int NC>
__device__ void lb_lookback(const uint64_t* st, uint32_t tile, uint32_t tag, uint32_t* s_prefix,
                            int* s_stop) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = warp * 32 + lane;
  if (threadIdx.x < NC) s_prefix[threadIdx.x] = 0;
  bool done[NC];
#pragma unroll
  for (int c = 0; c < NC; c++) done[c] = false;
  int64_t pos = (int64_t)tile - 1;
  __syncthreads();
  while (pos >= 0) {
    const int64_t t = pos - g;
    const bool valid = t >= 0;
    uint64_t w[NC];
#pragma unroll
    for (int c = 0; c < NC; c++) {
      w[c] = 0;
      if (valid && !done[c]) {
        do {
          w[c] = ld_relaxed_u64(&st[(size_t)t * 4 + c]);
        } while ((uint32_t)(w[c] >> 48) != tag || ((w[c] >> 46) & 3ull) == 0);
      }
    }
    if (threadIdx.x < NC) s_stop[threadIdx.x] = 1 << 30;
    __syncthreads();
#pragma unroll
    for (int c = 0; c < NC; c++) {
      uint32_t im = __ballot_sync(0xFFFFFFFFu, valid && !done[c] && ((w[c] >> 46) & 3ull) == LB_INC);
      if (lane == 0 && im) atomicMin(&s_stop[c], warp * 32 + (__ffs(im) - 1));
    }
    __syncthreads();
#pragma unroll
    for (int c = 0; c < NC; c++) {
      const int stop = s_stop[c];
      uint32_t v = (valid && !done[c] && g <= stop) ? (uint32_t)(w[c] & ((1ull << 46) - 1)) : 0u;
      v = __reduce_add_sync(0xFFFFFFFFu, v);
      if (lane == 0 && v) atomicAdd(&s_prefix[c], v);
    }
    bool all = true;
#pragma unroll
    for (int c = 0; c < NC; c++) {
      done[c] = done[c] || (s_stop[c] < (1 << 30));
      all = all && done[c];
    }
    __syncthreads();
    if (all) break;
    pos -= 32 * WARPS;
  }
}

__device__ __forceinline__ void atomic_max_key(Key128* p, uint64_t hi, uint32_t idx) {
  // cheap filter: the slot's hi only grows, so a smaller hi can never win
  uint64_t cur_hi = ld_relaxed_u64(reinterpret_cast<const uint64_t*>(p));
  if (hi < cur_hi) return;
  Key128 want;
  want.hi = hi;
  want.lo = idx;
  Key128 cmp;
  cmp.hi = cur_hi;
  cmp.lo = 0;
  for (;;) {
    Key128 old = atomicCAS(p, cmp, want);
    if (old.hi == cmp.hi && old.lo == cmp.lo) return;
    if (!(hi > old.hi || (hi == old.hi && (unsigned long long)idx < old.lo))) return;
    cmp = old;
  }
}

// thresholds come with the call parameters (defaults LONG_MIN_LIVE /
// LONG_SEG_MIN; SH_LONG_MIN_LIVE / SH_LONG_SEG_MIN override them, which the
// tests use to drive every peeled round through k_stream)
__device__ __forceinline__ bool long_round(const RoundParams& rp, const DevState* st) {
  return rp.round >= 2 && rp.aligned && rp.n_live >= st->long_min_live &&
         (uint64_t)rp.n_live >= (uint64_t)st->long_seg_min * rp.nseg;
}

// Decided by the bookkeeping kernel before it lays out the segments of
// round `round_next` (from bounds it knows up front): whether that round may
// run k_stream, i.e. its segments are padded to 4-record alignment.  Padding
// and k_stream's per-tile DEAD claims grow the positions of the rounds
// after it; they must stay within the record streams (rcap).
__device__ __forceinline__ bool stream_eligible(const Workspace& ws, const DevState* st, const RoundParams& bp,
                                                uint32_t round_next, uint32_t K) {
  if (round_next < 2 || round_next > 1u + (uint32_t)LONG_PEEL) return false;
  if (bp.n_true < st->long_min_live || (uint64_t)bp.n_true < (uint64_t)st->long_seg_min * K * bp.nseg) return false;
  const uint64_t nseg_next = (uint64_t)K * bp.nseg;
  const uint64_t u = (uint64_t)bp.n_true + st->dead_round + 3 * nseg_next;  // positions of round_next
  const uint64_t tiles = u / ws.stream_T + nseg_next + 2ull * ws.stream_grid;
  return u + 3ull * (2 * K) * tiles <= ws.rcap;  // + k_stream's DEAD claims
}

}  // namespace sh
