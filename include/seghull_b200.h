/*
 * seghull_b200 -- C ABI of the B200-native Quickhull (drop-in for the hull
 * entry points of the reference package `seghull`).
 *
 * Replaces (reference, /root/reference/pkg/src/seghull/):
 *   quickhull_2d(points, tol) -> HullResult      quickhull.py:167-279
 *   quickhull_3d(points, tol) -> HullResult      quickhull.py:282-446
 *   Tolerance.effective (eps = eps_rel * hypot.reduce(bbox spans))
 *                                                geometry.py:68-83
 *   exceptions ContractViolation / EmptyInputError / DegenerateInputError
 *                                                errors.py:4-15
 *   AssertionError("round count exceeded ...")   quickhull.py:227-228
 * The reference has no FFI layer; its boundary is the Python function pair
 * above.  The Python shim paper_1201_2936_b200/quickhull.py keeps those
 * names and raises the same exception classes from the status codes below.
 *
 * All pointers passed to the hull calls are DEVICE pointers (CUDA), except
 * `res`.  Coordinates are fp64; `stride` is the element distance between
 * consecutive points of one coordinate array (1 for structure-of-arrays,
 * dim for a row-major (n, dim) array).  Indices written to out_idx are
 * original point indices (int64), in discovery order (first-split extremes,
 * then per round per segment).  `stream` is a cudaStream_t (NULL = legacy
 * default stream).  One context per device; a context is not thread-safe.
 */
#ifndef SEGHULL_B200_H
#define SEGHULL_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define SH_OK 0
#define SH_CONTRACT 1     /* ContractViolation (bad arguments)              */
#define SH_EMPTY 2        /* EmptyInputError   (n == 0)                     */
#define SH_DEGENERATE 3   /* DegenerateInputError (3D coplanar input)       */
#define SH_ROUND_GUARD 4  /* AssertionError round count exceeded n + 1      */
#define SH_NOMEM 5        /* device allocation failed                       */
#define SH_CUDA 10        /* CUDA error, see sh_last_error()                */

/* result flags */
#define SH_FLAG_COLLINEAR 1 /* "collinear input: ..." warning (2D :208, 3D :338) */

typedef struct sh_ctx sh_ctx;

typedef struct sh_result {
  int64_t h;          /* vertex indices written to out_idx                   */
  int64_t iterations; /* Quickhull rounds (HullResult.iterations)            */
  int64_t candidates; /* 3D: loop candidates before the extreme filter       */
  int64_t pruned;     /* 3D: candidates removed by the extreme filter        */
  int64_t facets;     /* 3D: facet triples written (0 if not requested)      */
  int32_t status;     /* SH_* status                                         */
  int32_t flags;      /* SH_FLAG_*                                           */
  double eps;         /* effective absolute tolerance used                   */
} sh_result;

/* Context management. */
int sh_create(int device, sh_ctx** out);
void sh_destroy(sh_ctx* ctx);

/* 2D hull.  eps_abs: NaN -> eps = eps_rel * glibc_hypot(bbox spans)
 * (Tolerance.effective); otherwise eps_abs is used as the absolute eps
 * (sharded runs share the global eps).  out_idx: capacity n.
 * Synchronous w.r.t. `stream` (returns after the result is known). */
int sh_hull2d(sh_ctx* ctx, const double* x, const double* y, int64_t stride, int64_t n,
              double eps_rel, double eps_abs, int64_t* out_idx, sh_result* res, void* stream);

/* 3D hull: vertex indices of the extreme points (reference result after
 * _extreme_vertex_mask, quickhull.py:136-164).  out_facets (optional, may
 * be NULL): int32 triples (i, j, k) of original indices, counter-clockwise
 * seen from outside (det[[p_i 1];[p_j 1];[p_k 1];[s 1]] > 0 for every other
 * vertex s), capacity facet_cap triples (2*h - 4 suffice); res->facets = the
 * number written.  The reference has no facet output; these are the facets
 * of the hull of the returned vertices, exact (coplanar vertices are
 * triangulated consistently by symbolic perturbation), in unspecified order.
 * SH_CONTRACT if facet_cap is too small or the loop emitted >= 2^21
 * candidate vertices. */
int sh_hull3d(sh_ctx* ctx, const double* x, const double* y, const double* z, int64_t stride,
              int64_t n, double eps_rel, double eps_abs, int64_t* out_idx, int32_t* out_facets,
              int64_t facet_cap, sh_result* res, void* stream);

/* Asynchronous variants: enqueue the whole hull (one CUDA-graph launch, no
 * host synchronisation inside the round loop) and return immediately;
 * sh_fetch() waits for the stream and fills `res`. */
int sh_hull2d_async(sh_ctx* ctx, const double* x, const double* y, int64_t stride, int64_t n,
                    double eps_rel, double eps_abs, int64_t* out_idx, void* stream);
int sh_hull3d_async(sh_ctx* ctx, const double* x, const double* y, const double* z, int64_t stride,
                    int64_t n, double eps_rel, double eps_abs, int64_t* out_idx, int32_t* out_facets,
                    int64_t facet_cap, void* stream);
int sh_fetch(sh_ctx* ctx, sh_result* res, void* stream);

/* Per-round counters of the last hull on this context (live points
 * entering, survivors, segments, near-coplanar segments dropped); returns
 * the number of rounds written (<= cap). */
int64_t sh_trace(sh_ctx* ctx, int64_t* live, int64_t* kept, int64_t* nseg, int64_t* flat,
                 int64_t cap);

/* Per-axis bounding box of a point slice (device): out (device, 2*dim
 * doubles) = min x[,y[,z]], max x[,y[,z]].  Stream-ordered, no host sync.
 * Sharded hulls all-reduce these boxes (NCCL) and pass the resulting
 * eps = eps_rel * hypot(spans) as eps_abs, so every shard and the final
 * merge use the whole input's Tolerance.effective (geometry.py:79-83). */
int sh_bbox(sh_ctx* ctx, const double* x, const double* y, const double* z, int64_t stride, int64_t n,
            int dim, double* out, void* stream);

/* Sharded hulls (paper_1201_2936_b200/sharded.py).
 *
 * sh_stats: one pass over a slice -> out (device, SH_STATS = 14 doubles):
 * -min x, -min y, -min z, max x, max y, max z (a MAX all-reduce merges the
 * boxes of all slices), then the lexicographic minimum and maximum
 * (quickhull.py:75-84) as (x, y, z, global index = gidx_offset + local),
 * z = 0 in 2D.  Stream-ordered, no host synchronisation.
 * sh_stats_reduce: gathered (device, world x 14, every rank's sh_stats) ->
 * out (device, 14): the whole input's box and lexicographic extremes.
 * sh_set_shard: the next hull calls on this context use the whole input's
 * statistics gstats (device, 14 doubles, read on the device -- the host
 * never waits for them): flag SH_SHARD_EPS: eps = eps_rel * hypot(spans of
 * the global box) (Tolerance.effective of the whole input, geometry.py:
 * 79-83); flag SH_SHARD_SPLIT: the first split uses the global
 * lexicographic extremes; one that lies in another slice enters this
 * slice's hull as a virtual point, reported as local index n (min) or n + 1
 * (max).  gstats = NULL clears the setting. */
#define SH_STATS 14
#define SH_SHARD_EPS 1
#define SH_SHARD_SPLIT 2
int sh_stats(sh_ctx* ctx, const double* x, const double* y, const double* z, int64_t stride, int64_t n, int dim,
             int64_t gidx_offset, double* out, void* stream);
int sh_stats_reduce(sh_ctx* ctx, const double* gathered, int world, int dim, double* out, void* stream);
int sh_set_shard(sh_ctx* ctx, const double* gstats, int64_t gidx_offset, int flags);

/* Sharded merge of a 3D hull: the next sh_hull3d calls decide the extreme
 * filter (quickhull.py:136-164) only for share `share` of `nshares` equal
 * ranges of the candidates (in discovery order) and keep every
 * other candidate.  The vertex lists of all shares, intersected, are the
 * filtered hull (paper_1201_2936_b200/sharded.py splits the rank-0 merge's
 * filter this way).  nshares = 1 restores the whole filter. */
int sh_set_filter_share(sh_ctx* ctx, int share, int nshares);

/* The same sharded hull in two halves around the exchange, without a
 * separate statistics pass: sh_hull_shard_begin launches the hull's own
 * first pass over the slice (bbox + lexicographic extremes), writes the
 * slice's statistics (as sh_stats) to stats_out and returns without waiting;
 * the caller all-gathers them (NCCL, same stream) and reduces them
 * (sh_stats_reduce); sh_hull_shard_end(gstats, flags) runs the rest of the
 * hull with the whole input's statistics (as sh_set_shard) and returns like
 * sh_hull2d / sh_hull3d (out_idx capacity n + 2; no facets).  The two calls
 * belong together: no other hull may run on the context in between. */
int sh_hull_shard_begin(sh_ctx* ctx, int dim, const double* x, const double* y, const double* z, int64_t stride,
                        int64_t n, double eps_rel, double eps_abs, int64_t gidx_offset, double* stats_out,
                        void* stream);
int sh_hull_shard_end(sh_ctx* ctx, const double* gstats, int flags, int64_t* out_idx, sh_result* res,
                      void* stream);

/* order_hull_2d (reference quickhull.py:449-461) on the device: out_perm
 * (device, h int64) = the CCW boundary order of the h vertices (x, y device
 * arrays), starting at the lexicographically smallest, by angle around the
 * centroid (stable sort).  h < 3: the identity. */
int sh_order_hull_2d(sh_ctx* ctx, const double* x, const double* y, int64_t h, int64_t* out_perm, void* stream);

/* The CLI's `verify` check (reference oracle.py:20-52, hull2_giftwrap): gift
 * wrapping from the lexicographic minimum, next vertex = the candidate all
 * other points lie left of, among candidates collinear within
 * eps * |cand - cur| the farthest.  Per vertex: a tree reduction of that
 * rule, a proof that its winner dominates every other point, and an exact
 * replay of the reference's sequential scan when it does not (ties within
 * eps), so the walk visits the reference's coordinates.  out_idx (device,
 * capacity cap) receives the vertex indices in CCW order, *out_h their
 * count; SH_CONTRACT when cap is too small. */
int sh_giftwrap_2d(sh_ctx* ctx, const double* x, const double* y, int64_t n, double eps, int64_t* out_idx,
                   int64_t cap, int64_t* out_h, void* stream);

/* Device bytes the context allocates for `dim`-D hulls of n points with the
 * default table capacities: the ping-pong record streams (2 * dim streams of
 * (8*dim + 4)-byte records, capacity n each) plus segment tables sized for
 * n / 8 segments (C2: 11.3 GB); -1 for bad arguments.  No GPU needed. */
int64_t sh_workspace_bytes(int dim, int64_t n);

/* Reserve workspace for `dim`-D hulls of up to n points (optional). */
int sh_reserve(sh_ctx* ctx, int dim, int64_t n);

/* Host-side self test of the glibc-hypot port used for eps and 2D edge
 * lengths (no GPU needed). */
void sh_hypot_host(const double* x, const double* y, double* out, int64_t n);

/* Host self test of the exact orientation predicates used by the 3D facet
 * builder (no GPU needed): for each of nq queries, dim+1 points of `dim`
 * doubles (pts) with their global indices (ids), out = sign of
 * det [[p_i, 1]] under Simulation of Simplicity (never 0 for distinct ids).
 * exact_only: skip the fp64 filter. */
int sh_orient_host(int dim, const double* pts, const int64_t* ids, int64_t nq, int exact_only, int32_t* out);

/* 0 (default): one CUDA-graph launch per hull, round loop on the device.
 * 1: host-driven round loop (one sync per round) -- for profilers that can
 * not attribute kernels inside conditional graphs.
 * 2: as 1, plus a CUDA event after every kernel launch (sh_launch_times). */
int sh_set_launch_mode(sh_ctx* ctx, int mode);

/* Kernel launches of the last hull run in launch mode 2, in launch order:
 * kernel id (0 init, 1 first reduce, 2 line-far, 3 first-split round,
 * 4 round, 5 bookkeeping, 6 3D filter, 7 output) and device time in ms
 * (event to event on the hull's stream).  Returns the count written. */
int64_t sh_launch_times(sh_ctx* ctx, int32_t* kind, float* ms, int64_t cap);

/* Diagnostics of the last 3D extreme filter: candidates m, grid edge G,
 * candidates kept as within-eps ambiguous, GJK iteration caps, candidates
 * certified by the first query, support queries, points scanned, GJK
 * iterations, pruned by the local GJK, certified after the local GJK,
 * resolved by the global GJK, then SM cycles (summed over warps) spent in
 * the first query, the local GJK, the query after it and the global GJK;
 * then (-DSH_FILTER_CYCLES builds) 20 log2 buckets of k_f_test's per-item
 * wall cycles from 2^10 and the slowest item's cycles, GJK iterations,
 * queries and scanned candidates.  Returns the count written (<= cap,
 * <= 39). */
int sh_filter_stats(sh_ctx* ctx, int64_t* out, int64_t cap);

/* Diagnostics of the last 3D facet build: facets, queue items, wrap
 * queries, 32-point batches scanned, batches with a better candidate, box
 * tree nodes visited, SM cycles in wrap queries / waiting on the queue
 * (summed over warps), cycles of the initial-facet search.  Returns the
 * count written (<= cap, <= 9). */
int sh_facet_stats(sh_ctx* ctx, int64_t* out, int64_t cap);

/* ---- point sources ----
 * Device-side generation of the uniform-box benchmark clouds ("unit
 * square" 2D / "unit cube" 3D; reference splitmix64 stream, datagen.py:
 * 53-71): n points, global indices start..start+n-1 of the seeded cloud,
 * bit-identical to the host generator.  layout 0: structure of arrays
 * (out[c*n + i]); 1: rows (out[i*dim + c]).  Stream-ordered. */
int sh_uniform_points(sh_ctx* ctx, int dim, int64_t n, uint64_t seed, int64_t start, int layout, double* out,
                      void* stream);

/* ---- framework primitives (device arrays) ----
 * Replace segments.segmented_scan (segments.py:201-234), flag_permute
 * (primitives.py:91-117), compact (:120-148) and scatter (:151-176).
 * heads: uint8 segment-head flags (element 0 is always a head).
 * op: 0 sum (int64 only), 1 max, 2 min.  values/out: int64, or fp64 when
 * is_f64 (max/min; -0.0 is canonicalised to +0.0 as segments.py:197). */
int sh_segmented_scan(sh_ctx* ctx, const void* values, int is_f64, const uint8_t* heads, int64_t n, int op,
                      int backward, int exclusive, void* out, void* stream);
/* Stable in-segment grouping by state f in [0, k): destination p (int64,
 * a bijection within each segment) and new heads (uint8, length n). */
int sh_flag_permute(sh_ctx* ctx, const int64_t* f, const uint8_t* heads, int64_t n, int64_t k, int64_t* p,
                    uint8_t* heads_out, void* stream);
/* Keep-mask compaction: p = exclusive count of kept elements (int64),
 * *out_len (host) = number kept, heads_out (uint8, capacity n, first
 * *out_len written) = each surviving segment's head at its first kept
 * element.  Synchronises the stream (the output length is returned). */
int sh_compact(sh_ctx* ctx, const uint8_t* b, const uint8_t* heads, int64_t n, int64_t* p, int64_t* out_len,
               uint8_t* heads_out, void* stream);
/* out[p[i]] = data[i] (rows of row_bytes) for live i (live may be NULL);
 * SH_CONTRACT on colliding or out-of-range destinations (checked before any
 * write).  Synchronises the stream. */
int sh_scatter(sh_ctx* ctx, const void* data, int64_t row_bytes, const int64_t* p, const uint8_t* live,
               int64_t n, int64_t out_len, void* out, void* stream);

const char* sh_last_error(void);
const char* sh_version(void);

#ifdef __cplusplus
}
#endif

#endif /* SEGHULL_B200_H */
