// Host side of the B200 Quickhull: context, workspace, CUDA-graph driver,
// C ABI (include/seghull_b200.h).
//
// One hull call = one CUDA-graph launch:
//   k_init -> K0 k_first_reduce -> [3D: K0b k_line_far] -> K1 k_round<FIRST>
//   -> K3 k_book (root) -> WHILE(live points) { K2 k_round ; K3 k_book }
//   -> [3D: K4 extreme filter] -> k_output
// The WHILE condition is written by the finalising tile of k_book
// (cudaGraphSetConditional), so the round loop never returns to the host
// (the paper's per-iteration "new input size" readback, PAPER.md:292 /
// quickhull.py:225, is gone).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "../../include/seghull_b200.h"
#include "sh_book.cuh"
#include "sh_datagen.cuh"
#include "sh_facets3.cuh"
#include "sh_filter3.cuh"
#include "sh_kernels.cuh"
#include "sh_prims.cuh"
#include "sh_round.cuh"
#include "sh_stream.cuh"
#include "sh_order.cuh"

#include <cub/device/device_radix_sort.cuh>

using namespace sh;

namespace {

thread_local std::string g_last_error;

struct Graph {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
};

}  // namespace

struct sh_ctx {
  int device = 0;
  int nsm = 148;
  cudaStream_t build_stream = nullptr;
  cudaStream_t body_stream = nullptr;
  // workspace
  int dim = 0;           // dim the workspace was sized for (2 or 3), 0 = none
  uint64_t cap_n = 0;    // points
  uint32_t segcap = 0;   // segments
  uint32_t mcap = 0;     // 3D filter: candidates
  unsigned long long* bbox_bits = nullptr;  // sh_bbox scratch
  void* stats_parts = nullptr;                // sh_stats scratch: per-block partials + counter
  // sh_set_shard: applies to every hull call until cleared
  const double* shard_gstats = nullptr;
  int64_t shard_offset = 0;
  uint32_t shard_flags = 0;
  Workspace ws{};
  FilterWs fws{};
  FacetWs facws{};       // 3D facet output (allocated on the first facet request)
  int fac_occ = 1;
  size_t red_bytes = 0;
  // the workspace of the other dimension, parked while this one is active
  // (alternating 2D and 3D hulls neither free nor re-capture anything)
  struct Parked {
    int dim = 0;
    uint64_t cap_n = 0;
    uint32_t segcap = 0, mcap = 0;
    Workspace ws{};
    FilterWs fws{};
    FacetWs facws{};
    Graph g[3][4];
  } parked;
  DevState* st_host = nullptr;  // pinned mirror
  Graph g[3][4];         // [stage: 0 whole hull, 1 / 2 two-stage sharded hull][2 2D, 3 3D, 1 3D + facets]
  // sh_hull_shard_begin: the call it started (sh_hull_shard_end finishes it)
  struct {
    int dim = 0;
    const double *x = nullptr, *y = nullptr, *z = nullptr;
    int64_t stride = 1, n = 0, offset = 0;
    double eps_rel = 0, eps_abs = 0;
    bool open = false;
  } pend;
  double* stage_stats = nullptr;  // stats_out of the current stage-1 launch
  int round_occ2 = 0, round_occ3 = 0, book_occ2 = 0, book_occ3 = 0;
  int stream_occ2 = 1, stream_occ3 = 1;  // k_stream blocks per SM
  uint32_t filter_share = 0, filter_nshares = 1;  // sh_set_filter_share
  uint32_t last_n = 0;
  bool last_facets = false;
  int launch_mode = 0;  // 0: CUDA graph with device-side WHILE; 1: host loop; 2: host loop + events
  // per-launch CUDA events (launch_mode 2): ev0[i] / ev1[i] right before /
  // after launch i, whose kernel is prof_kind[i]
  static constexpr int PROF_CAP = 4096;
  cudaEvent_t ev0[PROF_CAP] = {}, ev1[PROF_CAP] = {};
  int prof_kind[PROF_CAP] = {};
  int prof_n = 0;
  bool prof_on = false;
};

// Kernel ids reported by sh_launch_times (include/seghull_b200.h).
enum { KID_INIT = 0, KID_FIRST_REDUCE, KID_LINE_FAR, KID_ROUND_FIRST, KID_ROUND, KID_BOOK,
       KID_FILTER, KID_OUTPUT, KID_FACETS };

// launch mode 2: bracket the next launch with events
static void prof_begin(sh_ctx* c, cudaStream_t s) {
  if (!c->prof_on || c->prof_n >= sh_ctx::PROF_CAP) return;
  if (!c->ev0[c->prof_n]) cudaEventCreate(&c->ev0[c->prof_n]);
  cudaEventRecord(c->ev0[c->prof_n], s);
}
static void prof_mark(sh_ctx* c, cudaStream_t s, int kind) {
  static const bool dbg = getenv("SH_DEBUG") != nullptr;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (dbg) cudaStreamIsCapturing(s, &cap);
  if (dbg && c->launch_mode != 0 && cap == cudaStreamCaptureStatusNone) {  // debugging aid
    cudaError_t e = cudaStreamSynchronize(s);
    DevState h;
    cudaMemcpy(&h, c->ws.st, offsetof(DevState, tr_live), cudaMemcpyDeviceToHost);
    fprintf(stderr, "[sh] kernel %d done (%s): rp active=%u root=%u n_live=%u nseg=%u cur=%u round=%u status=%u\n",
            kind, cudaGetErrorString(e), h.rp.active, h.rp.root, h.rp.n_live, h.rp.nseg, h.rp.cur, h.rp.round,
            h.status);
  }
  if (!c->prof_on || c->prof_n >= sh_ctx::PROF_CAP) return;
  if (!c->ev1[c->prof_n]) cudaEventCreate(&c->ev1[c->prof_n]);
  c->prof_kind[c->prof_n] = kind;
  cudaEventRecord(c->ev1[c->prof_n], s);
  c->prof_n++;
}

#define CK(x)                                                                     \
  do {                                                                            \
    cudaError_t e_ = (x);                                                         \
    if (e_ != cudaSuccess) {                                                      \
      g_last_error = std::string(#x) + ": " + cudaGetErrorString(e_);             \
      return SH_CUDA;                                                             \
    }                                                                             \
  } while (0)

static int set_err(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

template <class T>
static cudaError_t dalloc(T** p, size_t count) {
  return cudaMalloc((void**)p, count * sizeof(T) + 64);
}

static void free_ws(sh_ctx* c) {
  Workspace& w = c->ws;
  for (int b = 0; b < 2; b++) {
    cudaFree(w.rx[b]);
    cudaFree(w.ry[b]);
    cudaFree(w.rz[b]);
    cudaFree(w.ri[b]);
    cudaFree(w.seg[b]);
    cudaFree(w.segstart[b]);
    cudaFree(w.seg_phys[b]);
    cudaFree(w.cursor[b]);
  }
  cudaFree(w.slot_key);
  cudaFree(w.lb_book);
  cudaFree(w.vout);
  cudaFree(w.red);
  cudaFree(w.st);
  filter_free(c->fws);
  facet_free(c->facws);
  w = Workspace{};
  c->fws = FilterWs{};
  c->facws = FacetWs{};
  for (auto& gs : c->g)
    for (auto& g : gs) {
      if (g.exec) cudaGraphExecDestroy(g.exec);
      if (g.graph) cudaGraphDestroy(g.graph);
      g = Graph{};
    }
  c->dim = 0;
  c->cap_n = 0;
  c->segcap = 0;
  c->mcap = 0;
}

// Round 1 claims its output per tile, padded to 4 records per tile and
// child (sh_stream.cuh); the first-split sides' children are interleaved in
// the input, so side 0's children may outgrow side 0's span by 3 records
// per tile: side 1's children start this much later (a multiple of 4).
static uint32_t round1_slack(int dim, uint64_t n) {
  const uint64_t T = dim == 2 ? StreamCfg<2>::T : StreamCfg<3>::T;
  return (uint32_t)(((3 * ((n + T - 1) / T) + 4) + 3) & ~3ull);
}

// Records per stream: n live points, both sides' round-1 padding, and 1/16
// headroom for the DEAD records of the streamed rounds (k_book only lets
// k_stream take a round whose padding fits, stream_eligible()), rounded to a
// multiple of 16 so every stream starts 64-byte aligned.
static uint64_t record_cap(int dim, uint64_t n) {
  return (n + n / 16 + 4096 + 2 * (uint64_t)round1_slack(dim, n) + 15) & ~15ull;
}

// active workspace <-> parked one
static void swap_parked(sh_ctx* c) {
  auto& p = c->parked;
  std::swap(p.dim, c->dim);
  std::swap(p.cap_n, c->cap_n);
  std::swap(p.segcap, c->segcap);
  std::swap(p.mcap, c->mcap);
  std::swap(p.ws, c->ws);
  std::swap(p.fws, c->fws);
  std::swap(p.facws, c->facws);
  for (int a = 0; a < 3; a++)
    for (int b = 0; b < 4; b++) std::swap(p.g[a][b], c->g[a][b]);
}

static int alloc_ws(sh_ctx* c, int dim, uint64_t n, uint32_t segcap, uint32_t mcap) {
  free_ws(c);
  Workspace& w = c->ws;
  const int K = dim;
  w.slack = round1_slack(dim, n);
  uint64_t rcap = record_cap(dim, n);
  w.rcap = rcap;
  uint64_t max_tiles = (n + RTILE - 1) / RTILE + 4;
  uint64_t book_tiles = ((uint64_t)K * segcap + TILE3 - 1) / TILE3 + 4;
  size_t seg_bytes = (dim == 2) ? sizeof(Seg2) : sizeof(Seg3);
  bool ok = true;
  for (int b = 0; b < 2; b++) {
    ok &= dalloc(&w.rx[b], K * rcap) == cudaSuccess;
    ok &= dalloc(&w.ry[b], K * rcap) == cudaSuccess;
    if (dim == 3) ok &= dalloc(&w.rz[b], K * rcap) == cudaSuccess;
    ok &= dalloc(&w.ri[b], K * rcap) == cudaSuccess;
    ok &= cudaMalloc(&w.seg[b], (size_t)segcap * seg_bytes + 256) == cudaSuccess;
    ok &= dalloc(&w.segstart[b], (size_t)segcap + 4) == cudaSuccess;
    ok &= dalloc(&w.seg_phys[b], (size_t)segcap + 4) == cudaSuccess;
    ok &= dalloc(&w.cursor[b], (size_t)K * segcap + 4) == cudaSuccess;
  }
  ok &= dalloc(&w.slot_key, (size_t)K * segcap + 4) == cudaSuccess;
  ok &= dalloc(&w.lb_book, book_tiles * 4) == cudaSuccess;
  w.lb_book_words = book_tiles * 4;
  ok &= dalloc(&w.vout, n + 8) == cudaSuccess;
  w.red_blocks = (uint32_t)c->nsm * 8;
  ok &= cudaMalloc((void**)&w.red, (size_t)w.red_blocks * 128 + 256) == cudaSuccess;
  ok &= dalloc(&w.st, 1) == cudaSuccess;
  if (ok && dim == 3) ok &= filter_alloc(c->fws, mcap) == 0;
  if (!ok) {
    free_ws(c);
    cudaGetLastError();
    return set_err(SH_NOMEM, "device allocation failed for the hull workspace");
  }
  CK(cudaMemset(w.slot_key, 0, ((size_t)K * segcap + 4) * sizeof(Key128)));
  CK(cudaMemset(w.lb_book, 0, book_tiles * 4 * sizeof(uint64_t)));
  CK(cudaMemset(w.st, 0, sizeof(DevState)));
  w.max_tiles = (uint32_t)max_tiles;
  w.round_grid = (uint32_t)(c->nsm * (dim == 2 ? c->round_occ2 : c->round_occ3));
  w.stream_grid = (uint32_t)(c->nsm * (dim == 2 ? c->stream_occ2 : c->stream_occ3));
  w.stream_T = dim == 2 ? StreamCfg<2>::T : StreamCfg<3>::T;
  w.book_grid = (uint32_t)(c->nsm * (dim == 2 ? c->book_occ2 : c->book_occ3));
  c->dim = dim;
  c->cap_n = n;
  c->segcap = segcap;
  c->mcap = (dim == 3) ? mcap : 0;
  return SH_OK;
}

static uint32_t default_segcap(int dim, uint64_t n) {
  uint64_t s = std::max<uint64_t>(1u << 16, n / 8);
  s = std::min<uint64_t>(s, n + 4);
  return (uint32_t)s;
}

static uint32_t default_mcap(uint64_t n) {
  uint64_t m = std::max<uint64_t>(1u << 16, n / 64);
  return (uint32_t)std::min<uint64_t>(m, n + 4);
}

static int ensure_ws(sh_ctx* c, int dim, uint64_t n, uint32_t segcap_min, uint32_t mcap_min) {
  uint32_t want = std::max(default_segcap(dim, n), segcap_min);
  uint32_t mwant = (dim == 3) ? std::max(default_mcap(n), mcap_min) : 0u;
  if (c->dim != 0 && c->dim != dim) {
    // park the other dimension's workspace (freeing an older parked one of
    // this dimension's kind only if it is the one we are about to replace)
    if (c->parked.dim != dim && c->parked.dim != 0) {
      swap_parked(c);
      free_ws(c);
      swap_parked(c);
    }
    swap_parked(c);  // the parked workspace (this dim, or none) becomes active
  }
  if (c->dim == dim && c->cap_n >= n && c->segcap >= want && c->mcap >= mwant) return SH_OK;
  bool same = c->dim == dim;
  uint64_t cap = std::max<uint64_t>(n, same ? c->cap_n : 0);
  return alloc_ws(c, dim, cap, std::max(want, same ? c->segcap : 0u),
                  std::max(mwant, same ? c->mcap : 0u));
}

// ---------------------------------------------------------------- graph
template <int DIM>
static int launch_body(sh_ctx* c, Workspace ws, cudaStream_t s) {
  size_t dsm = RoundSmem<DIM>::bytes();
  // exactly one of the two round kernels does the work (long_round())
  prof_begin(c, s);
  if (SH_LEAN_LONG && ws.peeled)
    k_stream<DIM, SRC_REC><<<ws.stream_grid, StreamCfg<DIM>::NTHREADS,
                             StreamCfg<DIM>::SMEM, s>>>(ws);
  k_round<DIM, MODE_NORMAL><<<ws.round_grid, RB, dsm, s>>>(ws);
  CK(cudaGetLastError());
  prof_mark(c, s, KID_ROUND);
  prof_begin(c, s);
  k_book<DIM><<<ws.book_grid, BLOCK, 0, s>>>(ws);
  CK(cudaGetLastError());
  prof_mark(c, s, KID_BOOK);
  return SH_OK;
}

// stage 1: K0 over the input (a sharded hull stops here for the exchange)
template <int DIM>
static int launch_stage1(sh_ctx* c, Workspace ws, cudaStream_t s) {
  prof_begin(c, s);
  k_init<DIM><<<1, BLOCK, 0, s>>>(ws);
  CK(cudaGetLastError());
  prof_mark(c, s, KID_INIT);
  prof_begin(c, s);
  k_first_reduce<DIM><<<ws.red_blocks, BLOCK, 0, s>>>(ws);
  CK(cudaGetLastError());
  prof_mark(c, s, KID_FIRST_REDUCE);
  return SH_OK;
}

// stage 2: [the whole input's statistics applied,] the first split, round 1
template <int DIM>
static int launch_stage2(sh_ctx* c, Workspace ws, cudaStream_t s, bool apply) {
  if (apply) {
    prof_begin(c, s);
    k_shard_apply<DIM><<<1, 32, 0, s>>>(ws);
    CK(cudaGetLastError());
    prof_mark(c, s, KID_FIRST_REDUCE);
  }
  if (DIM == 3) {
    prof_begin(c, s);
    k_line_far<<<ws.red_blocks, BLOCK, 0, s>>>(ws);
    CK(cudaGetLastError());
    prof_mark(c, s, KID_LINE_FAR);
  }
  prof_begin(c, s);
  k_first_count<DIM><<<ws.red_blocks, BLOCK, 0, s>>>(ws);
  CK(cudaGetLastError());
  prof_mark(c, s, KID_ROUND_FIRST);
  prof_begin(c, s);
  k_book<DIM><<<ws.book_grid, BLOCK, 0, s>>>(ws);
  CK(cudaGetLastError());
  prof_mark(c, s, KID_BOOK);
  // round 1 re-reads the input and applies the first split on the fly, so
  // the split's survivors are never written
  prof_begin(c, s);
  k_stream<DIM, SRC_INPUT><<<ws.stream_grid, StreamCfg<DIM>::NTHREADS, StreamCfg<DIM>::SMEM, s>>>(ws);
  CK(cudaGetLastError());
  prof_mark(c, s, KID_ROUND);
  prof_begin(c, s);
  k_book<DIM><<<ws.book_grid, BLOCK, 0, s>>>(ws);
  CK(cudaGetLastError());
  prof_mark(c, s, KID_BOOK);
  return SH_OK;
}

template <int DIM>
static int launch_pre(sh_ctx* c, Workspace ws, cudaStream_t s, int stage) {
  int rc = SH_OK;
  if (stage != 2) rc = launch_stage1<DIM>(c, ws, s);
  if (rc || stage == 1) return rc;
  return launch_stage2<DIM>(c, ws, s, stage == 2);
}

template <int DIM>
static int launch_post(sh_ctx* c, Workspace ws, cudaStream_t s, bool facets) {
  if (DIM == 3) {
    prof_begin(c, s);
    int rc = filter_launch(c->fws, ws, c->nsm, s);
    if (rc) return set_err(rc, std::string("3D filter launch: ") + cudaGetErrorString(cudaGetLastError()));
    prof_mark(c, s, KID_FILTER);
    if (facets) {
      prof_begin(c, s);
      rc = facet_launch(c->facws, c->fws, ws, c->nsm, c->fac_occ, s);
      if (rc) return set_err(rc, std::string("3D facet launch: ") + cudaGetErrorString(cudaGetLastError()));
      prof_mark(c, s, KID_FACETS);
    }
    return SH_OK;
  }
  prof_begin(c, s);
  k_output<DIM><<<c->nsm * 4, BLOCK, 0, s>>>(ws, c->fws);
  CK(cudaGetLastError());
  prof_mark(c, s, KID_OUTPUT);
  return SH_OK;
}

// graph slots: [stage][2 = 2D, 3 = 3D vertices, 1 = 3D vertices + facets];
// stage 0 the whole hull, 1 / 2 the two halves of a sharded hull
template <int DIM>
static int build_graph(sh_ctx* c, bool facets = false, int stage = 0) {
  Graph& G = c->g[stage][(DIM == 3 && facets) ? 1 : DIM];
  if (G.exec) return SH_OK;
  cudaStream_t s = c->build_stream;
  if (stage == 1) {  // K0 only: no loop
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    int rc = launch_stage1<DIM>(c, c->ws, s);
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(s, &graph);
    if (rc) return rc;
    CK(e);
    CK(cudaGraphInstantiate(&G.exec, graph, 0));
    G.graph = graph;
    return SH_OK;
  }
  CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  cudaStreamCaptureStatus cs;
  cudaGraph_t cg = nullptr;
  const cudaGraphNode_t* deps = nullptr;
  size_t ndeps = 0;
  CK(cudaStreamGetCaptureInfo(s, &cs, nullptr, &cg, &deps, &ndeps));
  cudaGraphConditionalHandle handle;
  CK(cudaGraphConditionalHandleCreate(&handle, cg, 0, cudaGraphCondAssignDefault));
  Workspace ws = c->ws;
  ws.cond = handle;
  ws.use_cond = 1;
  int rc = launch_pre<DIM>(c, ws, s, stage);
  for (int r = 0; rc == SH_OK && SH_LEAN_LONG && r < LONG_PEEL; r++) {
    Workspace wp = ws;
    wp.peeled = 1;
    rc = launch_body<DIM>(c, wp, s);
  }
  if (rc) {
    cudaGraph_t tmp;
    cudaStreamEndCapture(s, &tmp);
    if (tmp) cudaGraphDestroy(tmp);
    return rc;
  }
  CK(cudaStreamGetCaptureInfo(s, &cs, nullptr, &cg, &deps, &ndeps));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = handle;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t cnode;
  CK(cudaGraphAddNode(&cnode, cg, deps, ndeps, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  CK(cudaStreamUpdateCaptureDependencies(s, &cnode, 1, cudaStreamSetCaptureDependencies));
  rc = launch_post<DIM>(c, ws, s, facets);
  cudaGraph_t graph = nullptr;
  cudaError_t e = cudaStreamEndCapture(s, &graph);
  if (rc) return rc;
  CK(e);
  // loop body
  CK(cudaStreamBeginCaptureToGraph(c->body_stream, body, nullptr, nullptr, 0,
                                   cudaStreamCaptureModeThreadLocal));
  rc = launch_body<DIM>(c, ws, c->body_stream);
  cudaGraph_t bg = nullptr;
  e = cudaStreamEndCapture(c->body_stream, &bg);
  if (rc) return rc;
  CK(e);
  CK(cudaGraphInstantiate(&G.exec, graph, 0));
  G.graph = graph;
  return SH_OK;
}

template <int DIM>
static int hull_async(sh_ctx* c, const double* x, const double* y, const double* z, int64_t stride,
                      int64_t n, double eps_rel, double eps_abs, int64_t* out_idx, int32_t* facets,
                      int64_t facet_cap, cudaStream_t s, uint32_t segcap_min, uint32_t mcap_min, int stage = 0) {
  if (n <= 0) return set_err(SH_EMPTY, "cannot take the hull of an empty point set");
  if (n >= (int64_t)0x7FFFFFF0) return set_err(SH_CONTRACT, "n must be < 2^31");
  if (!x || !y || (DIM == 3 && !z) || (!out_idx && stage != 1)) return set_err(SH_CONTRACT, "null pointer");
  if (stride < 1) return set_err(SH_CONTRACT, "stride must be >= 1");
  if (!(eps_rel >= 0)) return set_err(SH_CONTRACT, "eps_rel must be nonnegative");
  CK(cudaSetDevice(c->device));
  int rc = ensure_ws(c, DIM, (uint64_t)n, segcap_min, mcap_min);
  if (rc) return rc;
  const bool want_facets = DIM == 3 && facets != nullptr;
  if (want_facets && facet_cap < 0) return set_err(SH_CONTRACT, "facet_cap must be >= 0");
  if (want_facets && c->facws.mcap < c->mcap) {
    facet_free(c->facws);
    for (auto& gs : c->g) {
      Graph& g1 = gs[1];
      if (g1.exec) cudaGraphExecDestroy(g1.exec);
      if (g1.graph) cudaGraphDestroy(g1.graph);
      g1 = Graph{};
    }
    if (facet_alloc(c->facws, c->mcap)) {
      facet_free(c->facws);
      cudaGetLastError();
      return set_err(SH_NOMEM, "device allocation failed for the facet workspace");
    }
  }
  rc = build_graph<DIM>(c, want_facets, stage);
  if (rc) return rc;
  // call parameters -> device (pinned mirror, one small async copy)
  DevState* h = c->st_host;
  h->px = x;
  h->py = y;
  h->pz = (DIM == 3) ? z : y;
  h->stride = stride;
  h->n = (uint32_t)n;
  h->dim = DIM;
  h->eps_rel = eps_rel;
  h->use_eps_abs = std::isnan(eps_abs) ? 0u : 1u;
  h->eps_abs = std::isnan(eps_abs) ? 0.0 : eps_abs;
  h->segcap = c->segcap;
  h->out_idx = out_idx;
  {
    const char* e1 = getenv("SH_LONG_MIN_LIVE");
    const char* e2 = getenv("SH_LONG_SEG_MIN");
    h->long_min_live = e1 ? (uint32_t)strtoul(e1, nullptr, 10) : LONG_MIN_LIVE;
    h->long_seg_min = e2 ? (uint32_t)strtoul(e2, nullptr, 10) : LONG_SEG_MIN;
  }
  h->filter_share = c->filter_share;
  h->filter_nshares = c->filter_nshares;
  h->gstats = c->shard_gstats;
  h->gidx_offset = c->shard_offset;
  h->shard_flags = c->shard_gstats ? c->shard_flags : 0u;
  h->defer_first = stage == 1 ? 1u : 0u;
  h->stats_out = stage == 1 ? c->stage_stats : nullptr;
  h->out_facets = want_facets ? facets : nullptr;
  h->facet_cap = want_facets ? facet_cap : 0;
  CK(cudaMemcpyAsync(c->ws.st, h, offsetof(DevState, eps), cudaMemcpyHostToDevice, s));
  c->last_facets = want_facets;
  if (c->launch_mode == 0) {
    CK(cudaGraphLaunch(c->g[stage][want_facets ? 1 : DIM].exec, s));
  } else {
    // host-driven loop: same kernels, one host sync per round (ncu can not
    // attribute kernels inside graphs that contain conditional nodes)
    Workspace ws = c->ws;
    ws.use_cond = 0;
    c->prof_on = (c->launch_mode == 2);
    c->prof_n = 0;
    rc = launch_pre<DIM>(c, ws, s, stage);
    if (rc || stage == 1) {
      c->prof_on = false;
      return rc;
    }
    for (int r = 0;; r++) {
      CK(cudaMemcpyAsync(&h->rp, &c->ws.st->rp, sizeof(RoundParams), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      if (!h->rp.active) break;
      Workspace wr = ws;
      wr.peeled = (SH_LEAN_LONG && r < LONG_PEEL) ? 1u : 0u;
      rc = launch_body<DIM>(c, wr, s);
      if (rc) return rc;
    }
    rc = launch_post<DIM>(c, ws, s, want_facets);
    c->prof_on = false;
    if (rc) return rc;
  }
  c->last_n = (uint32_t)n;
  return SH_OK;
}

static int fetch(sh_ctx* c, sh_result* res, cudaStream_t s) {
  CK(cudaMemcpyAsync(c->st_host, c->ws.st, offsetof(DevState, tr_live), cudaMemcpyDeviceToHost, s));
  uint64_t fres[5] = {0, 0, 0, 0, 0};
  if (c->dim == 3) CK(cudaMemcpyAsync(fres, c->fws.result, sizeof(fres), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  const DevState* h = c->st_host;
  if (res) {
    memset(res, 0, sizeof(*res));
    res->status = (int32_t)h->status;
    res->flags = (int32_t)h->flags;
    res->iterations = h->rounds_final;
    res->eps = h->eps;
    res->h = h->h_final;
    res->candidates = h->h_final;
    if (c->dim == 3) {
      res->h = (int64_t)fres[0];
      res->pruned = (int64_t)h->h_final - (int64_t)fres[0];
      res->facets = c->last_facets ? (int64_t)fres[1] : 0;
    }
  }
  if (c->dim == 3 && c->last_facets && h->status == ST_OK) {
    if (fres[4] == ST_FAC_TOO_MANY)
      return set_err(SH_CONTRACT, "facet output supports fewer than 2^21 candidate vertices");
    if (fres[4] == ST_FAC_BROKEN) return set_err(SH_CUDA, "facet construction exceeded its tables (internal error)");
    if (fres[4] == ST_FAC_OVERFLOW)
      return set_err(SH_CONTRACT, "facet_cap too small: " + std::to_string(fres[1]) + " facets");
  }
  if (h->status == ST_SEG_OVERFLOW || h->status == ST_CAND_OVERFLOW) return SH_OK;  // caller retries
  if (h->status == ST_NONFINITE) return set_err(SH_CONTRACT, "coordinates must be finite");
  if (h->status == ST_DEGENERATE)
    return set_err(SH_DEGENERATE, "all points are coplanar; project to the plane and use the 2D driver");
  if (h->status == ST_ROUND_GUARD) return set_err(SH_ROUND_GUARD, "round count exceeded the input size");
  return SH_OK;
}

template <int DIM>
static int hull_sync(sh_ctx* c, const double* x, const double* y, const double* z, int64_t stride,
                     int64_t n, double eps_rel, double eps_abs, int64_t* out_idx, int32_t* facets,
                     int64_t facet_cap, sh_result* res, cudaStream_t s) {
  uint32_t segmin = 0, mmin = 0;
  for (int attempt = 0; attempt < 8; attempt++) {
    int rc = hull_async<DIM>(c, x, y, z, stride, n, eps_rel, eps_abs, out_idx, facets, facet_cap, s,
                             segmin, mmin);
    if (rc) return rc;
    rc = fetch(c, res, s);
    const uint32_t stt = c->st_host->status;
    if (stt != ST_SEG_OVERFLOW && stt != ST_CAND_OVERFLOW) return rc;
    uint64_t need = (uint64_t)c->st_host->seg_needed * 2 + 1024;
    if (stt == ST_SEG_OVERFLOW) segmin = (uint32_t)std::min<uint64_t>(need, (uint64_t)n + 4);
    else mmin = (uint32_t)std::min<uint64_t>(need, (uint64_t)n + 4);
  }
  return set_err(SH_NOMEM, "segment table capacity retries exhausted");
}

// ---------------------------------------------------------- primitives
static PsView ps_view(const void* vals, const uint8_t* heads, int64_t n, int backward) {
  PsView v;
  memset(&v, 0, sizeof(v));
  v.vals = vals;
  v.heads = heads;
  v.n = n;
  v.backward = backward;
  return v;
}

template <class T>
static int ps_launch(PsView v, int op, int exclusive, T* out, cudaStream_t s) {
  const int64_t ntiles = (v.n + PS_TILE - 1) / PS_TILE;
  PsAgg<T>* scratch = nullptr;
  CK(cudaMallocAsync((void**)&scratch, (size_t)(ntiles + 1) * sizeof(PsAgg<T>), s));
  int rc = ps_run<T>(v, op, exclusive, out, scratch, s);
  cudaFreeAsync(scratch, s);
  if (rc) return set_err(SH_CUDA, std::string("segmented scan launch: ") + cudaGetErrorString(cudaGetLastError()));
  return SH_OK;
}

template <int DIM>
static int shard_end(sh_ctx* c, int64_t* out_idx, sh_result* res, cudaStream_t s) {
  auto& p = c->pend;
  uint32_t segmin = 0, mmin = 0;
  for (int attempt = 0; attempt < 8; attempt++) {
    int rc = SH_OK;
    if (attempt > 0)  // the workspace grew (and was reset): K0 again
      rc = hull_async<DIM>(c, p.x, p.y, p.z, p.stride, p.n, p.eps_rel, p.eps_abs, nullptr, nullptr, 0, s,
                           segmin, mmin, 1);
    if (!rc)
      rc = hull_async<DIM>(c, p.x, p.y, p.z, p.stride, p.n, p.eps_rel, p.eps_abs, out_idx, nullptr, 0, s,
                           segmin, mmin, 2);
    if (rc) return rc;
    rc = fetch(c, res, s);
    const uint32_t stt = c->st_host->status;
    if (stt != ST_SEG_OVERFLOW && stt != ST_CAND_OVERFLOW) return rc;
    uint64_t need = (uint64_t)c->st_host->seg_needed * 2 + 1024;
    if (stt == ST_SEG_OVERFLOW) segmin = (uint32_t)std::min<uint64_t>(need, (uint64_t)p.n + 4);
    else mmin = (uint32_t)std::min<uint64_t>(need, (uint64_t)p.n + 4);
  }
  return set_err(SH_NOMEM, "segment table capacity retries exhausted");
}

// ---------------------------------------------------------------- C ABI
extern "C" {

int sh_create(int device, sh_ctx** out) {
  if (!out) return set_err(SH_CONTRACT, "null out pointer");
  *out = nullptr;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return set_err(SH_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
  sh_ctx* c = new sh_ctx();
  c->device = device;
  cudaDeviceGetAttribute(&c->nsm, cudaDevAttrMultiProcessorCount, device);
  cudaFuncSetAttribute(k_round<2, MODE_NORMAL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)RoundSmem<2>::bytes());
  cudaFuncSetAttribute(k_round<3, MODE_NORMAL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)RoundSmem<3>::bytes());
  int o2 = 0, o3 = 0, ob = 0, ob2 = 0, of = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, k_round<2, MODE_NORMAL>, RB, RoundSmem<2>::bytes());
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o3, k_round<3, MODE_NORMAL>, RB, RoundSmem<3>::bytes());
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ob, k_book<3>, BLOCK, 0);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ob2, k_book<2>, BLOCK, 0);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&of, k_fac_wrap, FAC_BLOCK, 0);
  c->fac_occ = std::max(1, of);
  cudaFuncSetAttribute(k_stream<2, SRC_INPUT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)StreamCfg<2>::SMEM);
  cudaFuncSetAttribute(k_stream<2, SRC_REC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)StreamCfg<2>::SMEM);
  cudaFuncSetAttribute(k_stream<3, SRC_INPUT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)StreamCfg<3>::SMEM);
  cudaFuncSetAttribute(k_stream<3, SRC_REC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)StreamCfg<3>::SMEM);
  {
    int a = 0, b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, k_stream<2, SRC_REC>, StreamCfg<2>::NTHREADS, StreamCfg<2>::SMEM);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_stream<3, SRC_REC>, StreamCfg<3>::NTHREADS, StreamCfg<3>::SMEM);
    c->stream_occ2 = std::max(1, a);
    c->stream_occ3 = std::max(1, b);
  }
  c->round_occ2 = std::max(1, o2);
  c->round_occ3 = std::max(1, o3);
  c->book_occ3 = std::max(1, std::min(ob, 4));
  c->book_occ2 = std::max(1, std::min(ob2, 4));
  e = cudaGetLastError();
  if (e != cudaSuccess) {
    delete c;
    return set_err(SH_CUDA, std::string("kernel setup: ") + cudaGetErrorString(e));
  }
  cudaStreamCreateWithFlags(&c->build_stream, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&c->body_stream, cudaStreamNonBlocking);
  if (cudaMallocHost((void**)&c->st_host, sizeof(DevState)) != cudaSuccess) {
    delete c;
    return set_err(SH_NOMEM, "pinned allocation failed");
  }
  memset(c->st_host, 0, sizeof(DevState));
  *out = c;
  return SH_OK;
}

void sh_destroy(sh_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  free_ws(c);
  swap_parked(c);
  free_ws(c);
  if (c->st_host) cudaFreeHost(c->st_host);
  if (c->bbox_bits) cudaFree(c->bbox_bits);
  if (c->stats_parts) cudaFree(c->stats_parts);
  for (auto& e : c->ev0)
    if (e) cudaEventDestroy(e);
  for (auto& e : c->ev1)
    if (e) cudaEventDestroy(e);
  if (c->build_stream) cudaStreamDestroy(c->build_stream);
  if (c->body_stream) cudaStreamDestroy(c->body_stream);
  delete c;
}

int64_t sh_workspace_bytes(int dim, int64_t n) {
  // mirrors alloc_ws / filter_alloc with the default capacities (the
  // workspace only grows past them when a hull overflows, see hull_sync)
  if ((dim != 2 && dim != 3) || n <= 0) return -1;
  const uint64_t K = dim, rcap = record_cap(dim, (uint64_t)n);
  const uint64_t segcap = default_segcap(dim, (uint64_t)n);
  const uint64_t max_tiles = ((uint64_t)n + RTILE - 1) / RTILE + 4;
  (void)max_tiles;
  const uint64_t book_tiles = (K * segcap + TILE3 - 1) / TILE3 + 4;
  const uint64_t seg_bytes = dim == 2 ? sizeof(Seg2) : sizeof(Seg3);
  uint64_t b = 0;
  b += 2 * (K * rcap * (8 * K + 4));                        // ping-pong records
  b += 2 * (segcap * seg_bytes + 4 * (segcap + 4) + 8 * (segcap + 4) + 4 * (K * segcap + 4));
  b += sizeof(Key128) * (K * segcap + 4) + 8 * book_tiles * 4 + 4 * ((uint64_t)n + 8);
  b += sizeof(DevState);
  if (dim == 3) {
    const uint64_t mcap = default_mcap((uint64_t)n);
    const uint64_t cells = (uint64_t)FG_MAX * FG_MAX * FG_MAX;
    const uint64_t nodes = mcap / 31 + 2 * F_LEVELS + 8;
    b += mcap * (6 * 8 + 4 * 3 + 1 + 3 * 4 + 8 + 4 + 24) + cells * 12 + nodes * (48 + 72);
  }
  return (int64_t)b;
}

int sh_reserve(sh_ctx* c, int dim, int64_t n) {
  if (!c || (dim != 2 && dim != 3) || n <= 0) return set_err(SH_CONTRACT, "bad reserve arguments");
  CK(cudaSetDevice(c->device));
  int rc = ensure_ws(c, dim, (uint64_t)n, 0, 0);
  if (rc) return rc;
  return dim == 2 ? build_graph<2>(c) : build_graph<3>(c);
}

int sh_hull2d(sh_ctx* c, const double* x, const double* y, int64_t stride, int64_t n, double eps_rel,
              double eps_abs, int64_t* out_idx, sh_result* res, void* stream) {
  if (!c) return set_err(SH_CONTRACT, "null context");
  return hull_sync<2>(c, x, y, nullptr, stride, n, eps_rel, eps_abs, out_idx, nullptr, 0, res,
                      (cudaStream_t)stream);
}

int sh_hull3d(sh_ctx* c, const double* x, const double* y, const double* z, int64_t stride, int64_t n,
              double eps_rel, double eps_abs, int64_t* out_idx, int32_t* out_facets, int64_t facet_cap,
              sh_result* res, void* stream) {
  if (!c) return set_err(SH_CONTRACT, "null context");
  return hull_sync<3>(c, x, y, z, stride, n, eps_rel, eps_abs, out_idx, out_facets, facet_cap, res,
                      (cudaStream_t)stream);
}

int sh_hull2d_async(sh_ctx* c, const double* x, const double* y, int64_t stride, int64_t n,
                    double eps_rel, double eps_abs, int64_t* out_idx, void* stream) {
  if (!c) return set_err(SH_CONTRACT, "null context");
  return hull_async<2>(c, x, y, nullptr, stride, n, eps_rel, eps_abs, out_idx, nullptr, 0,
                       (cudaStream_t)stream, 0, 0);
}

int sh_hull3d_async(sh_ctx* c, const double* x, const double* y, const double* z, int64_t stride,
                    int64_t n, double eps_rel, double eps_abs, int64_t* out_idx, int32_t* out_facets,
                    int64_t facet_cap, void* stream) {
  if (!c) return set_err(SH_CONTRACT, "null context");
  return hull_async<3>(c, x, y, z, stride, n, eps_rel, eps_abs, out_idx, out_facets, facet_cap,
                       (cudaStream_t)stream, 0, 0);
}

int sh_fetch(sh_ctx* c, sh_result* res, void* stream) {
  if (!c) return set_err(SH_CONTRACT, "null context");
  int rc = fetch(c, res, (cudaStream_t)stream);
  if (c->st_host->status == ST_SEG_OVERFLOW || c->st_host->status == ST_CAND_OVERFLOW)
    return set_err(SH_NOMEM, "segment/candidate table overflow; use the synchronous call (it retries)");
  return rc;
}

int64_t sh_trace(sh_ctx* c, int64_t* live, int64_t* kept, int64_t* nseg, int64_t* flat, int64_t cap) {
  if (!c || !c->ws.st) return 0;
  static_assert(offsetof(DevState, tr_flat) > offsetof(DevState, tr_live), "layout");
  DevState* h = c->st_host;
  if (cudaMemcpy(h, c->ws.st, sizeof(DevState), cudaMemcpyDeviceToHost) != cudaSuccess) return 0;
  int64_t r = std::min<int64_t>(std::min<int64_t>(h->rounds_final, MAX_TRACE), cap);
  for (int64_t i = 0; i < r; i++) {
    if (live) live[i] = h->tr_live[i];
    if (kept) kept[i] = h->tr_kept[i];
    if (nseg) nseg[i] = h->tr_nseg[i];
    if (flat) flat[i] = (c->dim == 3) ? h->tr_flat[i] : 0;
  }
  return r;
}

void sh_hypot_host(const double* x, const double* y, double* out, int64_t n) {
  for (int64_t i = 0; i < n; i++) out[i] = sh::glibc_hypot(x[i], y[i]);
}

int sh_orient_host(int dim, const double* pts, const int64_t* ids, int64_t nq, int exact_only, int32_t* out) {
  if ((dim != 2 && dim != 3) || nq < 0 || !pts || !ids || !out) return set_err(SH_CONTRACT, "bad arguments");
  const int R = dim + 1;
  for (int64_t q = 0; q < nq; q++) {
    const double* p = pts + q * R * dim;
    const int64_t* I = ids + q * R;
    if (dim == 2)
      out[q] = exact_only ? sh::orient_sos<2>(p, I) : sh::orient2d_exact(p, p + 2, p + 4, I[0], I[1], I[2]);
    else
      out[q] = exact_only ? sh::orient_sos<3>(p, I)
                          : sh::orient3d_exact(p, p + 3, p + 6, p + 9, I[0], I[1], I[2], I[3]);
  }
  return SH_OK;
}

int sh_set_launch_mode(sh_ctx* c, int mode) {
  if (!c || mode < 0 || mode > 2)
    return set_err(SH_CONTRACT, "mode must be 0 (graph), 1 (host loop) or 2 (host loop + events)");
  c->launch_mode = mode;
  return SH_OK;
}

int64_t sh_launch_times(sh_ctx* c, int32_t* kind, float* ms, int64_t cap) {
  if (!c) return 0;
  if (cudaSetDevice(c->device) != cudaSuccess) return 0;
  int64_t n = std::min<int64_t>(c->prof_n, cap);
  for (int64_t i = 0; i < n; i++) {
    if (cudaEventSynchronize(c->ev1[i]) != cudaSuccess) return i;
    float t = 0.f;
    cudaEventElapsedTime(&t, c->ev0[i], c->ev1[i]);
    if (kind) kind[i] = c->prof_kind[i];
    if (ms) ms[i] = t;
  }
  return n;
}

int sh_bbox(sh_ctx* c, const double* x, const double* y, const double* z, int64_t stride, int64_t n,
            int dim, double* out, void* stream) {
  if (!c) return set_err(SH_CONTRACT, "null context");
  if ((dim != 2 && dim != 3) || n <= 0 || !x || !y || (dim == 3 && !z) || !out || stride < 1)
    return set_err(SH_CONTRACT, "bad bbox arguments");
  if (n >= (int64_t)0x7FFFFFF0) return set_err(SH_CONTRACT, "n must be < 2^31");
  CK(cudaSetDevice(c->device));
  cudaStream_t s = (cudaStream_t)stream;
  if (!c->bbox_bits) CK(cudaMalloc((void**)&c->bbox_bits, 64));
  k_bbox_init<<<1, 32, 0, s>>>(c->bbox_bits, dim);
  k_bbox<<<c->nsm * 8, BLOCK, 0, s>>>(x, y, dim == 3 ? z : y, stride, (uint32_t)n, dim, c->bbox_bits);
  k_bbox_final<<<1, 32, 0, s>>>(c->bbox_bits, out, dim);
  CK(cudaGetLastError());
  return SH_OK;
}

int sh_stats(sh_ctx* c, const double* x, const double* y, const double* z, int64_t stride, int64_t n, int dim,
             int64_t gidx_offset, double* out, void* stream) {
  if (!c) return set_err(SH_CONTRACT, "null context");
  if ((dim != 2 && dim != 3) || n <= 0 || !x || !y || (dim == 3 && !z) || !out || stride < 1)
    return set_err(SH_CONTRACT, "bad stats arguments");
  if (n >= (int64_t)0x7FFFFFF0) return set_err(SH_CONTRACT, "n must be < 2^31");
  CK(cudaSetDevice(c->device));
  cudaStream_t s = (cudaStream_t)stream;
  const uint32_t grid = (uint32_t)c->nsm * 4;
  if (!c->stats_parts) {
    CK(cudaMalloc(&c->stats_parts, (size_t)grid * sizeof(FirstRed) + 64));
    CK(cudaMemset(c->stats_parts, 0, (size_t)grid * sizeof(FirstRed) + 64));
  }
  FirstRed* parts = reinterpret_cast<FirstRed*>(c->stats_parts);
  uint32_t* counter = reinterpret_cast<uint32_t*>(parts + grid);
  if (dim == 2)
    k_stats<2><<<grid, BLOCK, 0, s>>>(x, y, y, stride, (uint32_t)n, gidx_offset, parts, counter, out);
  else
    k_stats<3><<<grid, BLOCK, 0, s>>>(x, y, z, stride, (uint32_t)n, gidx_offset, parts, counter, out);
  CK(cudaGetLastError());
  return SH_OK;
}

int sh_stats_reduce(sh_ctx* c, const double* gathered, int world, int dim, double* out, void* stream) {
  if (!c) return set_err(SH_CONTRACT, "null context");
  if ((dim != 2 && dim != 3) || world < 1 || !gathered || !out) return set_err(SH_CONTRACT, "bad stats arguments");
  CK(cudaSetDevice(c->device));
  if (dim == 2) k_stats_reduce<2><<<1, 32, 0, (cudaStream_t)stream>>>(gathered, world, out);
  else k_stats_reduce<3><<<1, 32, 0, (cudaStream_t)stream>>>(gathered, world, out);
  CK(cudaGetLastError());
  return SH_OK;
}

int sh_set_shard(sh_ctx* c, const double* gstats, int64_t gidx_offset, int flags) {
  if (!c) return set_err(SH_CONTRACT, "null context");
  if (flags & ~3) return set_err(SH_CONTRACT, "unknown shard flags");
  c->shard_gstats = gstats;
  c->shard_offset = gidx_offset;
  c->shard_flags = (uint32_t)flags;
  return SH_OK;
}

int sh_set_filter_share(sh_ctx* c, int share, int nshares) {
  if (!c) return set_err(SH_CONTRACT, "null context");
  if (nshares < 1 || share < 0 || share >= nshares) return set_err(SH_CONTRACT, "bad filter share");
  c->filter_share = (uint32_t)share;
  c->filter_nshares = (uint32_t)nshares;
  return SH_OK;
}

int sh_hull_shard_begin(sh_ctx* c, int dim, const double* x, const double* y, const double* z, int64_t stride,
                        int64_t n, double eps_rel, double eps_abs, int64_t gidx_offset, double* stats_out,
                        void* stream) {
  if (!c) return set_err(SH_CONTRACT, "null context");
  if ((dim != 2 && dim != 3) || !stats_out) return set_err(SH_CONTRACT, "bad sharded hull arguments");
  auto& p = c->pend;
  p.dim = dim;
  p.x = x;
  p.y = y;
  p.z = z;
  p.stride = stride;
  p.n = n;
  p.offset = gidx_offset;
  p.eps_rel = eps_rel;
  p.eps_abs = eps_abs;
  c->shard_gstats = nullptr;
  c->shard_offset = gidx_offset;
  c->shard_flags = 0;
  c->stage_stats = stats_out;
  cudaStream_t s = (cudaStream_t)stream;
  int rc = dim == 2 ? hull_async<2>(c, x, y, nullptr, stride, n, eps_rel, eps_abs, nullptr, nullptr, 0, s, 0, 0, 1)
                    : hull_async<3>(c, x, y, z, stride, n, eps_rel, eps_abs, nullptr, nullptr, 0, s, 0, 0, 1);
  c->stage_stats = nullptr;
  p.open = rc == SH_OK;
  return rc;
}

int sh_hull_shard_end(sh_ctx* c, const double* gstats, int flags, int64_t* out_idx, sh_result* res, void* stream) {
  if (!c) return set_err(SH_CONTRACT, "null context");
  if (!c->pend.open) return set_err(SH_CONTRACT, "sh_hull_shard_end without sh_hull_shard_begin");
  if (!gstats || !out_idx || (flags & ~3)) return set_err(SH_CONTRACT, "bad sharded hull arguments");
  c->pend.open = false;
  c->shard_gstats = gstats;
  c->shard_offset = c->pend.offset;
  c->shard_flags = (uint32_t)flags;
  cudaStream_t s = (cudaStream_t)stream;
  int rc = c->pend.dim == 2 ? shard_end<2>(c, out_idx, res, s) : shard_end<3>(c, out_idx, res, s);
  c->shard_gstats = nullptr;
  c->shard_flags = 0;
  return rc;
}

int sh_order_hull_2d(sh_ctx* c, const double* x, const double* y, int64_t h, int64_t* out_perm, void* stream) {
  if (!c) return set_err(SH_CONTRACT, "null context");
  if (h < 0 || (h > 0 && (!x || !y || !out_perm))) return set_err(SH_CONTRACT, "bad order_hull_2d arguments");
  if (h >= (int64_t)0x7FFFFFF0) return set_err(SH_CONTRACT, "h must be < 2^31");
  CK(cudaSetDevice(c->device));
  cudaStream_t s = (cudaStream_t)stream;
  const uint32_t n = (uint32_t)h;
  if (n < 3) {  // quickhull.py:455-456: returned as given
    for (uint32_t i = 0; i < n; i++) {
      const int64_t v = i;
      CK(cudaMemcpyAsync(out_perm + i, &v, 8, cudaMemcpyHostToDevice, s));
    }
    CK(cudaStreamSynchronize(s));
    return SH_OK;
  }
  const uint32_t grid = std::min<uint32_t>((n + BLOCK - 1) / BLOCK, (uint32_t)c->nsm * 4);
  size_t temp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, temp, (unsigned long long*)nullptr, (unsigned long long*)nullptr,
                                  (uint32_t*)nullptr, (uint32_t*)nullptr, (int)n, 0, 64, s);
  const size_t bytes = (size_t)n * 24 + (size_t)grid * 16 + 64 + temp + 256;
  unsigned char* buf = nullptr;
  CK(cudaMallocAsync((void**)&buf, bytes, s));
  unsigned long long* k0 = (unsigned long long*)buf;
  unsigned long long* k1 = k0 + n;
  uint32_t* v0 = (uint32_t*)(k1 + n);
  uint32_t* v1 = v0 + n;
  double* acc = (double*)(((uintptr_t)(v1 + n) + 15) & ~(uintptr_t)15);
  double* mean = acc + 2 * grid;
  uint32_t* counter = (uint32_t*)(mean + 2);
  void* tmp = (void*)(((uintptr_t)(counter + 4) + 255) & ~(uintptr_t)255);
  CK(cudaMemsetAsync(counter, 0, 4, s));
  k_ord_sum<<<grid, BLOCK, 0, s>>>(x, y, n, acc, counter, mean);
  k_ord_keys<<<grid, BLOCK, 0, s>>>(x, y, n, mean, k0, v0);
  cudaError_t e = cub::DeviceRadixSort::SortPairs(tmp, temp, k0, k1, v0, v1, (int)n, 0, 64, s);  // stable
  if (e == cudaSuccess) k_ord_roll<<<1, 1024, 0, s>>>(x, y, n, v1, out_perm);
  cudaFreeAsync(buf, s);
  CK(e);
  CK(cudaGetLastError());
  return SH_OK;
}

int sh_giftwrap_2d(sh_ctx* c, const double* x, const double* y, int64_t n, double eps, int64_t* out_idx,
                   int64_t cap, int64_t* out_h, void* stream) {
  if (!c) return set_err(SH_CONTRACT, "null context");
  if (n <= 0 || !x || !y || !out_idx || !out_h || cap < 1) return set_err(SH_CONTRACT, "bad giftwrap arguments");
  if (n >= (int64_t)0x7FFFFFF0) return set_err(SH_CONTRACT, "n must be < 2^31");
  CK(cudaSetDevice(c->device));
  cudaStream_t s = (cudaStream_t)stream;
  // start: the lexicographic minimum (min(pts) in hull2_giftwrap)
  const uint32_t grid = (uint32_t)std::min<int64_t>((int64_t)c->nsm * 4, (n + BLOCK - 1) / BLOCK);
  unsigned char* buf = nullptr;
  CK(cudaMallocAsync((void**)&buf, (size_t)grid * sizeof(GwBest) + 256 + STATS_N * 8, s));
  GwBest* parts = (GwBest*)buf;
  GwState* st = (GwState*)(((uintptr_t)(parts + grid) + 15) & ~(uintptr_t)15);
  double* dstats = (double*)(((uintptr_t)(st + 1) + 15) & ~(uintptr_t)15);
  int rc = sh_stats(c, x, y, nullptr, 1, n, 2, 0, dstats, stream);
  if (rc) {
    cudaFreeAsync(buf, s);
    return rc;
  }
  double stats[STATS_N];
  CK(cudaMemcpyAsync(stats, dstats, sizeof(stats), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  GwState h0{};
  h0.cur = h0.start = (uint32_t)stats[9];
  h0.h = 1;
  const int64_t first = h0.start;
  CK(cudaMemcpyAsync(out_idx, &first, 8, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(st, &h0, sizeof(h0), cudaMemcpyHostToDevice, s));
  // at most n + 1 steps (the reference's loop bound); poll between batches
  GwState hs{};
  for (int64_t step = 0; step <= n;) {
    const int64_t batch = std::min<int64_t>(step == 0 ? 8 : 256, n + 1 - step);
    for (int64_t k = 0; k < batch; k++) {
      k_gw_step<<<grid, BLOCK, 0, s>>>(x, y, (uint32_t)n, eps, st, parts);
      k_gw_check<<<grid, BLOCK, 0, s>>>(x, y, (uint32_t)n, eps, st);
      k_gw_commit<<<1, 1024, 0, s>>>(x, y, (uint32_t)n, eps, st, out_idx, cap);
    }
    CK(cudaGetLastError());
    step += batch;
    CK(cudaMemcpyAsync(&hs, st, sizeof(hs), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (hs.done) break;
  }
  cudaFreeAsync(buf, s);
  if (hs.done == 2) return set_err(SH_CONTRACT, "giftwrap output capacity exceeded");
  *out_h = hs.h;
  return SH_OK;
}

int sh_uniform_points(sh_ctx* c, int dim, int64_t n, uint64_t seed, int64_t start, int layout, double* out,
                      void* stream) {
  if (!c) return set_err(SH_CONTRACT, "null context");
  if ((dim != 2 && dim != 3) || n < 0 || start < 0 || (layout != 0 && layout != 1) || (n > 0 && !out))
    return set_err(SH_CONTRACT, "bad uniform_points arguments");
  if (n == 0) return SH_OK;
  CK(cudaSetDevice(c->device));
  k_uniform_points<<<c->nsm * 8, BLOCK, 0, (cudaStream_t)stream>>>(dim, (uint64_t)n, (unsigned long long)seed,
                                                                 (uint64_t)start, out, layout);
  CK(cudaGetLastError());
  return SH_OK;
}

int sh_segmented_scan(sh_ctx* c, const void* values, int is_f64, const uint8_t* heads, int64_t n, int op,
                      int backward, int exclusive, void* out, void* stream) {
  if (!c) return set_err(SH_CONTRACT, "null context");
  if (n < 0 || (n > 0 && (!values || !heads || !out)) || op < 0 || op > 2 || (is_f64 && op == PS_SUM))
    return set_err(SH_CONTRACT, "bad segmented scan arguments");
  if (n == 0) return SH_OK;
  CK(cudaSetDevice(c->device));
  PsView v = ps_view(values, heads, n, backward);
  cudaStream_t s = (cudaStream_t)stream;
  return is_f64 ? ps_launch<double>(v, op, exclusive, (double*)out, s)
                : ps_launch<long long>(v, op, exclusive, (long long*)out, s);
}

int sh_flag_permute(sh_ctx* c, const int64_t* f, const uint8_t* heads, int64_t n, int64_t k, int64_t* p,
                    uint8_t* heads_out, void* stream) {
  if (!c) return set_err(SH_CONTRACT, "null context");
  if (n < 0 || k < 1 || (n > 0 && (!f || !heads || !p || !heads_out)))
    return set_err(SH_CONTRACT, "bad flag permute arguments");
  if (n == 0) return SH_OK;
  CK(cudaSetDevice(c->device));
  cudaStream_t s = (cudaStream_t)stream;
  int64_t *seg = nullptr, *rank = nullptr, *seg_start = nullptr;
  unsigned long long* counts = nullptr;
  CK(cudaMallocAsync((void**)&seg, n * 8, s));
  CK(cudaMallocAsync((void**)&rank, n * 8, s));
  CK(cudaMallocAsync((void**)&seg_start, n * 8, s));
  CK(cudaMallocAsync((void**)&counts, (size_t)n * k * 8, s));
  CK(cudaMemsetAsync(counts, 0, (size_t)n * k * 8, s));
  // segment id = inclusive count of heads - 1 (element 0 always heads)
  PsView hv = ps_view(nullptr, nullptr, n, 0);
  hv.u8 = heads;
  hv.force0 = 1;
  int rc = ps_launch<long long>(hv, PS_SUM, 0, (long long*)seg, s);
  const unsigned grid = (unsigned)std::min<int64_t>((n + BLOCK - 1) / BLOCK, 65535);
  if (!rc) {
    k_fp_subone<<<grid, BLOCK, 0, s>>>(seg, n);
    k_fp_counts<<<grid, BLOCK, 0, s>>>(f, seg, n, k, heads, counts, seg_start);
  }
  // stable in-segment rank per state: exclusive segmented count of state j
  for (int64_t j = 0; j < k && !rc; j++) {
    PsView sv = ps_view(nullptr, heads, n, 0);
    sv.states = f;
    sv.state = j;
    rc = ps_launch<long long>(sv, PS_SUM, 1, (long long*)rank, s);
  }
  if (!rc) {
    k_fp_assemble<<<grid, BLOCK, 0, s>>>(f, seg, rank, n, k, counts, seg_start, p, heads_out);
    k_fp_heads<<<grid, BLOCK, 0, s>>>(n, k, counts, seg_start, heads_out);
  }
  cudaFreeAsync(seg, s);
  cudaFreeAsync(rank, s);
  cudaFreeAsync(seg_start, s);
  cudaFreeAsync(counts, s);
  if (rc) return rc;
  CK(cudaPeekAtLastError());
  return SH_OK;
}

int sh_compact(sh_ctx* c, const uint8_t* b, const uint8_t* heads, int64_t n, int64_t* p, int64_t* out_len,
               uint8_t* heads_out, void* stream) {
  if (!c) return set_err(SH_CONTRACT, "null context");
  if (n < 0 || !out_len || (n > 0 && (!b || !heads || !p || !heads_out)))
    return set_err(SH_CONTRACT, "bad compact arguments");
  *out_len = 0;
  if (n == 0) return SH_OK;
  CK(cudaSetDevice(c->device));
  cudaStream_t s = (cudaStream_t)stream;
  // p = exclusive count of kept elements (one segment)
  PsView kv = ps_view(nullptr, nullptr, n, 0);
  kv.u8 = b;
  int rc = ps_launch<long long>(kv, PS_SUM, 1, (long long*)p, s);
  if (rc) return rc;
  int64_t last_p = 0;
  uint8_t last_b = 0;
  CK(cudaMemcpyAsync(&last_p, p + n - 1, 8, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(&last_b, b + n - 1, 1, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  *out_len = last_p + (last_b ? 1 : 0);
  // each head moves to the first kept destination at or after it
  // (backward segmented min scan of kept destinations, primitives.py:141-146)
  int64_t* firsts = nullptr;
  CK(cudaMallocAsync((void**)&firsts, n * 8, s));
  PsView mv = ps_view(nullptr, heads, n, 1);
  mv.keep = b;
  mv.mvals = p;
  rc = ps_launch<long long>(mv, PS_MIN, 0, (long long*)firsts, s);
  if (!rc && *out_len > 0) {
    CK(cudaMemsetAsync(heads_out, 0, *out_len, s));
    const unsigned grid = (unsigned)std::min<int64_t>((n + BLOCK - 1) / BLOCK, 65535);
    k_cp_heads<<<grid, BLOCK, 0, s>>>(firsts, heads, n, heads_out);
  }
  cudaFreeAsync(firsts, s);
  if (rc) return rc;
  CK(cudaPeekAtLastError());
  return SH_OK;
}

int sh_scatter(sh_ctx* c, const void* data, int64_t row_bytes, const int64_t* p, const uint8_t* live, int64_t n,
               int64_t out_len, void* out, void* stream) {
  if (!c) return set_err(SH_CONTRACT, "null context");
  if (n < 0 || out_len < 0 || row_bytes < 1 || (n > 0 && (!data || !p)) || (out_len > 0 && !out))
    return set_err(SH_CONTRACT, "bad scatter arguments");
  CK(cudaSetDevice(c->device));
  cudaStream_t s = (cudaStream_t)stream;
  if (out_len > 0) CK(cudaMemsetAsync(out, 0, (size_t)out_len * row_bytes, s));
  if (n == 0) return SH_OK;
  unsigned int* hits = nullptr;
  unsigned long long* err = nullptr;
  CK(cudaMallocAsync((void**)&hits, (size_t)(out_len + 1) * 4, s));
  CK(cudaMallocAsync((void**)&err, 16, s));
  CK(cudaMemsetAsync(hits, 0, (size_t)(out_len + 1) * 4, s));
  CK(cudaMemsetAsync(err, 0, 16, s));
  const unsigned grid = (unsigned)std::min<int64_t>((n + BLOCK - 1) / BLOCK, 65535);
  k_scatter_check<<<grid, BLOCK, 0, s>>>(p, live, n, out_len, hits, err);
  unsigned long long herr[2] = {0, 0};
  CK(cudaMemcpyAsync(herr, err, 16, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  cudaFreeAsync(hits, s);
  cudaFreeAsync(err, s);
  if (herr[1]) return set_err(SH_CONTRACT, "map destination out of range");
  if (herr[0]) return set_err(SH_CONTRACT, "map destinations collide");
  k_scatter<<<grid, BLOCK, 0, s>>>((const unsigned char*)data, p, live, n, row_bytes, (unsigned char*)out);
  CK(cudaPeekAtLastError());
  return SH_OK;
}

int sh_filter_stats(sh_ctx* c, int64_t* out, int64_t cap) {
  if (!c || !c->fws.fp || cap <= 0) return 0;
  FilterParams P;
  if (cudaMemcpy(&P, c->fws.fp, sizeof(P), cudaMemcpyDeviceToHost) != cudaSuccess) return 0;
  int64_t v[39] = {P.m, P.G, P.ambiguous, P.gjk_capped, (int64_t)P.certified, (int64_t)P.queries,
                   (int64_t)P.scanned, (int64_t)P.gjk_iters, (int64_t)P.local_in, (int64_t)P.local_out,
                   (int64_t)P.fallback, (int64_t)P.cyc_cert, (int64_t)P.cyc_local, (int64_t)P.cyc_out,
                   (int64_t)P.cyc_fallback};
  for (int k = 0; k < 20; k++) v[15 + k] = P.dur_hist[k];
  v[35] = (int64_t)P.dur_max;
  v[36] = (int64_t)P.dur_max_iters;
  v[37] = (int64_t)P.dur_max_queries;
  v[38] = (int64_t)P.dur_max_scanned;
  int64_t n = std::min<int64_t>(cap, 39);
  for (int64_t i = 0; i < n; i++) out[i] = v[i];
  return (int)n;
}

int sh_facet_stats(sh_ctx* c, int64_t* out, int64_t cap) {
  if (!c || !c->facws.ctl || cap <= 0) return 0;
  FacetCtl C;
  if (cudaMemcpy(&C, c->facws.ctl, sizeof(C), cudaMemcpyDeviceToHost) != cudaSuccess) return 0;
  int64_t v[9] = {C.nfacets, C.reserved, (int64_t)C.queries, (int64_t)C.batches, (int64_t)C.beat_batches,
                  (int64_t)C.nodes, (int64_t)C.wrap_cycles, (int64_t)C.wait_cycles, (int64_t)C.init_cycles};
  int64_t n = std::min<int64_t>(cap, 9);
  for (int64_t i = 0; i < n; i++) out[i] = v[i];
  return (int)n;
}

const char* sh_last_error(void) { return g_last_error.c_str(); }
const char* sh_version(void) { return "seghull_b200 0.1 (sm_100a)"; }

}  // extern "C"
