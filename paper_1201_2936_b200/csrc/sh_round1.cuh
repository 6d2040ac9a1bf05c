// K1+K2 for round 1: the first split fused with the first Quickhull round,
// as a barrier-free streaming kernel (quickhull.py:200-266 for 2D,
// :346-437 for 3D).
//
// Round 1 is the largest pass of a hull (it reads the whole input and
// writes every round-1 survivor) and it has at most 2 segments (the two
// sides of the first split) x K states = 2K children, so it does not need
// the general round kernel's per-tile segment windows, shared-memory
// counters and block barriers.  Each warp streams 256-point chunks of the
// input (8 points per lane, lane-interleaved so every load is coalesced):
//   * branch-free classification in the reference's fp64 order: first-split
//     side (cross2 / plane distance against the extreme line or plane), then
//     the side's round-1 segment (classify2 / classify3: discard test, child
//     state, the child's next-round distance);
//   * warp ballots give each survivor its rank among the chunk's survivors
//     of the same child; one lane per child claims the chunk's output range
//     with one global atomicAdd on the child's cursor;
//   * survivors are stored straight from registers (each child's part of a
//     chunk is one contiguous run of its output stream);
//   * every lane keeps its running farthest key per child in registers;
//     they are reduced per warp, then per block, and merged into the child
//     slots with one 128-bit atomicCAS per block and child at the end.
// Same outputs as k_round<DIM, MODE_ROUND1> (child cursors, survivor
// records, slot keys), byte for byte in the records' multiset.
#pragma once

#include <type_traits>

#include "sh_common.cuh"

namespace sh {

constexpr int R1B = 256;     // threads per block
#ifndef SH_R1ITEMS
#define SH_R1ITEMS 4
#endif
constexpr int R1ITEMS = SH_R1ITEMS;  // points per lane per chunk
constexpr int R1CHUNK = 32 * R1ITEMS;
static_assert(R1CHUNK <= 255, "per-child chunk counts are packed 8 bits each");

// classify2 without early returns (same predicates, same operation order)
__device__ __forceinline__ int classify2_bf(const Seg2& g, double qx, double qy, uint32_t qi, double* dnext) {
  const double c0 = cross2(g.ax, g.ay, g.fx, g.fy, qx, qy);  // cross2(a, far, q)
  const double c1 = cross2(g.fx, g.fy, g.bx, g.by, qx, qy);  // cross2(far, b, q)
  const bool inside = (-c1 >= g.nt_bf) & (-c0 >= g.nt_fa);
  const bool one_sided = (c0 > 0) != (c1 > 0);
  const int state = one_sided ? (c1 > 0 ? 1 : 0) : (c1 > c0 ? 1 : 0);
  *dnext = state ? c1 : c0;
  return (inside | (qi == g.fidx)) ? -1 : state;
}

__device__ __forceinline__ int classify3_bf(const Seg3& g, double qx, double qy, double qz, uint32_t qi,
                                            double* dnext) {
  const double D0 = plane_dist(g.N[0], g.a, qx, qy, qz);
  const double D1 = plane_dist(g.N[1], g.b, qx, qy, qz);
  const double D2 = plane_dist(g.N[2], g.c, qx, qy, qz);
  const bool inside = (D0 <= g.thr[0]) & (D1 <= g.thr[1]) & (D2 <= g.thr[2]);
  // first argmax of the rounded quotients D_j / |N_j| (quotient_gt)
  int state = 0;
  double db = D0, nb = g.nrm[0];
  if (quotient_gt(D1, g.nrm[1], db, nb)) {
    state = 1;
    db = D1;
    nb = g.nrm[1];
  }
  if (quotient_gt(D2, g.nrm[2], db, nb)) {
    state = 2;
    db = D2;
  }
  *dnext = db;
  return (inside | (g.flat != 0) | (qi == g.fidx)) ? -1 : state;
}

#ifndef SH_R1_MINB
#define SH_R1_MINB 2
#endif
#ifndef SH_R1_MINB3
#define SH_R1_MINB3 2
#endif
#ifndef SH_RL_MINB3
#define SH_RL_MINB3 1  // 3D long rounds: no spills at one block per SM (measured faster)
#endif
// Ranks of a warp chunk's survivors per child (key < NK; NK <= 8): rank[j]
// = number of earlier survivors of the same child in the chunk (item-major,
// then lane).  Returns the chunk's per-child counts packed 8 bits each
// (child k at bit 8k; a chunk has < 256 points).  3D (6 children), per
// item: REDUX.SUMs of the lanes' 1 << 8*key (the item's packed counts, 4
// children per 32-bit word) and log2(NK) + 1 ballots to find the lanes with
// the same key; 2D (4 children): one ballot per child.
template <int NK, int ITEMS>
__device__ __forceinline__ unsigned long long chunk_ranks(const uint32_t* key, uint32_t* rank) {
  static_assert(NK <= 8, "8-bit fields, two 32-bit words");
  constexpr int NBITS = NK <= 2 ? 1 : (NK <= 4 ? 2 : 3);
  const uint32_t lt = lanemask_lt();
  if constexpr (NK <= 4) {
    // 2D (4 children): one ballot per child is cheaper here (measured)
    unsigned long long packed = 0ull;
#pragma unroll
    for (int j = 0; j < ITEMS; j++) {
      uint32_t r = 0;
      unsigned long long add = 0ull;
#pragma unroll
      for (int k = 0; k < NK; k++) {
        const bool mine = key[j] == (uint32_t)k;
        const uint32_t m = __ballot_sync(0xFFFFFFFFu, mine);
        r += mine ? (uint32_t)__popc(m & lt) : 0u;
        add += (unsigned long long)__popc(m) << (8 * k);
      }
      const uint32_t kj = key[j] < (uint32_t)NK ? key[j] : 0u;
      rank[j] = r + (uint32_t)((packed >> (8 * kj)) & 0xFFull);
      packed += add;
    }
    return packed;
  }
  uint32_t run_lo = 0, run_hi = 0;
#pragma unroll
  for (int j = 0; j < ITEMS; j++) {
    const uint32_t kj = key[j];
    const bool valid = kj < (uint32_t)NK;
    const uint32_t c_lo = __reduce_add_sync(0xFFFFFFFFu, (valid && kj < 4u) ? (1u << (8 * kj)) : 0u);
    const uint32_t c_hi = NK > 4 ? __reduce_add_sync(0xFFFFFFFFu, (valid && kj >= 4u) ? (1u << (8 * (kj - 4))) : 0u) : 0u;
    uint32_t grp = __ballot_sync(0xFFFFFFFFu, valid);
#pragma unroll
    for (int b = 0; b < NBITS; b++) {
      const uint32_t mb = __ballot_sync(0xFFFFFFFFu, (kj >> b) & 1u);
      grp &= ((kj >> b) & 1u) ? mb : ~mb;
    }
    const uint32_t base = kj < 4u ? (run_lo >> (8 * kj)) & 0xFFu : (run_hi >> (8 * ((kj - 4) & 3u))) & 0xFFu;
    rank[j] = __popc(grp & lt) + base;
    run_lo += c_lo;
    run_hi += c_hi;
  }
  return (unsigned long long)run_lo | ((unsigned long long)run_hi << 32);
}

template <int DIM>
__global__ void __launch_bounds__(R1B, DIM == 2 ? SH_R1_MINB : SH_R1_MINB3) k_round1(Workspace ws) {
  constexpr int K = DIM;
  constexpr int NK = 2 * K;  // children: (side segment w, state s) -> w * K + s
  using SegT = typename std::conditional<DIM == 2, Seg2, Seg3>::type;
  __shared__ __align__(16) SegT s_seg[2];
  __shared__ unsigned long long s_hi[R1B / 32][NK];
  __shared__ uint32_t s_idx[R1B / 32][NK];
  __shared__ double s_stage_x[R1B / 32][R1CHUNK];
  __shared__ double s_stage_y[R1B / 32][R1CHUNK];
  __shared__ double s_stage_z[DIM == 3 ? R1B / 32 : 1][DIM == 3 ? R1CHUNK : 1];
  __shared__ uint32_t s_stage_i[R1B / 32][R1CHUNK];
  DevState* st = ws.st;
  const RoundParams rp = st->rp;
  if (!rp.active || rp.root || rp.round != 1) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (blockIdx.x == 0 && tid == 0) {
    st->ctr_book = 0;  // K3's tile counter
    st->arrive_book = 0;
    st->book_small = (uint32_t)K * rp.nseg <= BOOK_SMALL ? 1u : 0u;
  }
  const uint32_t nseg = rp.nseg, cur = rp.cur;
  {
    const unsigned long long* src = reinterpret_cast<const unsigned long long*>(ws.seg[cur]);
    unsigned long long* dst = reinterpret_cast<unsigned long long*>(s_seg);
    for (uint32_t k = tid; k < nseg * (sizeof(SegT) / 8); k += R1B) dst[k] = src[k];
  }
  const uint32_t n = st->n;
  const double* px = st->px;
  const double* py = st->py;
  const double* pz = st->pz;
  const int64_t stride = st->stride;
  double f_pa[3], f_pb[3], f_nrm[3];
#pragma unroll
  for (int k = 0; k < 3; k++) {
    f_pa[k] = st->pa[k];
    f_pb[k] = st->pb[k];
    f_nrm[k] = st->nrm[k];
  }
  const double f_thr = st->thr_line;
  const uint32_t f_imin = st->imin, f_imax = st->imax, f_ifar = (DIM == 3) ? st->ifar : 0xFFFFFFFFu;
  // segment of each first-split side (side 0 is segment 0 when it has
  // survivors; the root children's counts are still in cursor[0])
  const uint32_t side1_seg = ws.cursor[0][0] ? 1u : 0u;
  uint32_t* cursor = ws.cursor[cur];
  double* outx = ws.rx[cur ^ 1u];
  double* outy = ws.ry[cur ^ 1u];
  double* outz = ws.rz[cur ^ 1u];
  uint32_t* outi = ws.ri[cur ^ 1u];
  const uint64_t rcap = ws.rcap;
  __syncthreads();

  unsigned long long bh[NK];
  uint32_t bi[NK];
#pragma unroll
  for (int k = 0; k < NK; k++) {
    bh[k] = 0ull;
    bi[k] = 0xFFFFFFFFu;
  }
  const uint32_t nchunks = (n + R1CHUNK - 1) / R1CHUNK;
  const uint32_t gw = blockIdx.x * (R1B / 32) + warp, nw = gridDim.x * (R1B / 32);
  // per-warp staging of one chunk's survivors, grouped by child
  double* stx = s_stage_x[warp];
  double* sty = s_stage_y[warp];
  double* stz = DIM == 3 ? s_stage_z[warp] : nullptr;
  uint32_t* sti = s_stage_i[warp];
  // the previous chunk's survivors wait in the staging area until its claims
  // have returned (flushed at the top of the next iteration)
  uint32_t pend_base = 0;                // lane k: the claimed base of child k
  unsigned long long pend_off = 0ull;    // staged start of each child (8 bits each)
  unsigned long long pend_cnt = 0ull;    // staged count of each child
  auto flush = [&]() {
    const uint32_t tot = (uint32_t)(((pend_off >> (8 * (NK - 1))) & 0xFFull) + ((pend_cnt >> (8 * (NK - 1))) & 0xFFull));
    for (uint32_t t0 = 0; t0 < tot; t0 += 32) {  // warp-uniform bound
      const uint32_t t = t0 + lane;
      uint32_t k = 0;
#pragma unroll
      for (int kk = 1; kk < NK; kk++) k += t >= (uint32_t)((pend_off >> (8 * kk)) & 0xFFull) ? 1u : 0u;
      const uint32_t kb = __shfl_sync(0xFFFFFFFFu, pend_base, k);
      if (t < tot) {
        const size_t dst = (size_t)(k % K) * rcap + kb + (t - (uint32_t)((pend_off >> (8 * k)) & 0xFFull));
        outx[dst] = stx[t];
        outy[dst] = sty[t];
        if (DIM == 3) outz[dst] = stz[t];
        outi[dst] = sti[t];
      }
    }
    __syncwarp();
  };
  // registers hold the current chunk and the prefetched next one
  double x[R1ITEMS], y[R1ITEMS], z[R1ITEMS], nx[R1ITEMS], ny[R1ITEMS], nz[R1ITEMS];
  auto load_chunk = [&](uint32_t c, double* X, double* Y, double* Z) {
#pragma unroll
    for (int j = 0; j < R1ITEMS; j++) {
      const uint32_t q = min(c * R1CHUNK + j * 32 + lane, n - 1);
      X[j] = ld_coord(px, stride, q);
      Y[j] = ld_coord(py, stride, q);
      if (DIM == 3) Z[j] = ld_coord(pz, stride, q);
    }
  };
  if (gw < nchunks) load_chunk(gw, nx, ny, nz);
  for (uint32_t c = gw; c < nchunks; c += nw) {
    const uint32_t base = c * R1CHUNK;
#pragma unroll
    for (int j = 0; j < R1ITEMS; j++) {
      x[j] = nx[j];
      y[j] = ny[j];
      if (DIM == 3) z[j] = nz[j];
    }
    if (c + nw < nchunks) load_chunk(c + nw, nx, ny, nz);
    uint32_t key[R1ITEMS];
    uint32_t hu[R1ITEMS], hl[R1ITEMS];
#pragma unroll
    for (int j = 0; j < R1ITEMS; j++) {
      const uint32_t q = base + j * 32 + lane;
      bool keep;
      int side;
      if (DIM == 2) {
        // quickhull.py:202-211
        const double d = cross2(f_pa[0], f_pa[1], f_pb[0], f_pb[1], x[j], y[j]);
        keep = (q < n) & (q != f_imin) & (q != f_imax) & (fabs(d) > f_thr);
        side = d < 0 ? 1 : 0;
      } else {
        // quickhull.py:348-353
        const double d = plane_dist(f_nrm, f_pa, x[j], y[j], z[j]);
        keep = (q < n) & (q != f_imin) & (q != f_imax) & (q != f_ifar);
        side = d < f_thr ? 1 : 0;
      }
      const uint32_t w = side ? side1_seg : 0u;
      double dn;
      int s;
      if constexpr (DIM == 2) s = classify2_bf(s_seg[w], x[j], y[j], q, &dn);
      else s = classify3_bf(s_seg[w], x[j], y[j], z[j], q, &dn);
      keep &= s >= 0;
      key[j] = keep ? w * K + (uint32_t)s : 0xFFFFFFFFu;
      // d > 0 for every survivor: the raw bits order like ordered_bits(d)
      hu[j] = (uint32_t)__double2hiint(dn) | 0x80000000u;
      hl[j] = (uint32_t)__double2loint(dn);
    }
    // per-child counts of the chunk (8 bits each, packed) and every
    // survivor's rank among its child's survivors in the chunk
    uint32_t rank[R1ITEMS];
    const unsigned long long packed = chunk_ranks<NK, R1ITEMS>(key, rank);
    // staged start of each child: exclusive prefix of the packed counts
    unsigned long long off = 0ull;
#pragma unroll
    for (int k = 1; k < NK; k++)
      off |= ((((off >> (8 * (k - 1))) & 0xFFull) + ((packed >> (8 * (k - 1))) & 0xFFull)) << (8 * k));
    // the previous chunk's claims have had a whole chunk of work to return
    flush();
    // stage this chunk's survivors grouped by child, then claim their ranges
#pragma unroll
    for (int j = 0; j < R1ITEMS; j++) {
      const uint32_t kj = key[j];
      if (kj < (uint32_t)NK) {
        const uint32_t t = (uint32_t)((off >> (8 * kj)) & 0xFFull) + rank[j];
        stx[t] = x[j];
        sty[t] = y[j];
        if (DIM == 3) stz[t] = z[j];
        sti[t] = base + j * 32 + lane;
      }
    }
    __syncwarp();
    const uint32_t mycnt = lane < NK ? (uint32_t)((packed >> (8 * lane)) & 0xFFull) : 0u;
    pend_base = mycnt ? atomicAdd(&cursor[lane], mycnt) : 0u;
    pend_off = off;
    pend_cnt = packed;
    // farthest keys: only when some survivor reaches its child's running
    // maximum (rare after the first chunks) -- per child, the chunk's
    // maximum by warp REDUX on the key's halves, lowest index among ties
    // (against the smallest running maximum of all children: a per-child
    // select here would be turned into an indexed local-memory array)
    uint32_t thr = 0xFFFFFFFFu;
#pragma unroll
    for (int k = 0; k < NK; k++) thr = min(thr, (uint32_t)(bh[k] >> 32));
    bool cand = false;
#pragma unroll
    for (int j = 0; j < R1ITEMS; j++) cand |= key[j] < (uint32_t)NK && hu[j] >= thr;
    if (__any_sync(0xFFFFFFFFu, cand)) {
#pragma unroll
      for (int k = 0; k < NK; k++) {
        uint32_t tu = 0, tl = 0, ti = 0xFFFFFFFFu;
#pragma unroll
        for (int j = 0; j < R1ITEMS; j++) {
          const bool mine = key[j] == (uint32_t)k;
          const uint32_t q = base + j * 32 + lane;
          const bool better = mine && (hu[j] > tu || (hu[j] == tu && (hl[j] > tl || (hl[j] == tl && q < ti))));
          tu = better ? hu[j] : tu;
          tl = better ? hl[j] : tl;
          ti = better ? q : ti;
        }
        const uint32_t mu = __reduce_max_sync(0xFFFFFFFFu, tu);
        if (mu == 0u || mu < (uint32_t)(bh[k] >> 32)) continue;  // warp-uniform
        const uint32_t ml = __reduce_max_sync(0xFFFFFFFFu, tu == mu ? tl : 0u);
        const unsigned long long h = ((unsigned long long)mu << 32) | ml;
        const uint32_t mi = __reduce_min_sync(0xFFFFFFFFu, (tu == mu && tl == ml) ? ti : 0xFFFFFFFFu);
        if (h > bh[k] || (h == bh[k] && mi < bi[k])) {
          bh[k] = h;
          bi[k] = mi;
        }
      }
    }
  }
  flush();
  // farthest keys (warp-uniform per warp): block, then one merge per block
  // and child
#pragma unroll
  for (int k = 0; k < NK; k++) {
    if (lane == 0) {
      s_hi[warp][k] = bh[k];
      s_idx[warp][k] = bi[k];
    }
  }
  __syncthreads();
  if (tid < NK && tid < (int)(nseg * K)) {
    unsigned long long h = 0ull;
    uint32_t idx = 0xFFFFFFFFu;
#pragma unroll
    for (int w = 0; w < R1B / 32; w++) {
      const unsigned long long h2 = s_hi[w][tid];
      const uint32_t i2 = s_idx[w][tid];
      if (h2 > h || (h2 == h && i2 < idx)) {
        h = h2;
        idx = i2;
      }
    }
    if (h) atomic_max_key(&ws.slot_key[tid], h, idx);
  }
}

}  // namespace sh

namespace sh {

// ------------------------------------------------------------------ K2L
// Rounds >= 2 whose segments are long (the first rounds of every config:
// n_live >= LONG_SEG_MIN * nseg) run the same streaming scheme as round 1.
// Each warp owns a contiguous range of 128-position chunks and walks the
// dense logical positions with a window of the (usually one, at a boundary
// two) segments the chunk overlaps; a chunk that overlaps three or more
// segments (rare here) is handled point by point with global atomics.  The
// per-child farthest keys are kept per warp for the children of the current
// window and merged (128-bit CAS max) when the window moves on.
// The first LONG_PEEL loop rounds are launched outside the CUDA graph's
// WHILE node as the pair (k_round_long, k_round), and exactly one of them
// works (long_round()); inside the WHILE node only k_round runs, so the
// later, short rounds pay no extra launch.
constexpr uint32_t LONG_SEG_MIN = 4096;
constexpr uint32_t LONG_MIN_LIVE = 4u << 20;
constexpr int LONG_PEEL = 3;  // rounds 2..4 are launched outside the WHILE loop

// thresholds come with the call parameters (defaults LONG_MIN_LIVE /
// LONG_SEG_MIN; SH_LONG_MIN_LIVE / SH_LONG_SEG_MIN override them, which the
// tests use to drive every round through this kernel)
__device__ __forceinline__ bool long_round(const RoundParams& rp, const DevState* st) {
  return rp.round >= 2 && rp.n_live >= st->long_min_live &&
         (uint64_t)rp.n_live >= (uint64_t)st->long_seg_min * rp.nseg;
}

template <int DIM>
__global__ void __launch_bounds__(R1B, DIM == 2 ? SH_R1_MINB : SH_RL_MINB3) k_round_long(Workspace ws) {
  constexpr int K = DIM;
  constexpr int NK = 2 * K;  // children of the window: (segment w + k / K, state k % K)
  using SegT = typename std::conditional<DIM == 2, Seg2, Seg3>::type;
  __shared__ __align__(16) SegT s_seg[R1B / 32][2][2];  // [warp][chunk parity][window slot]
  __shared__ double s_stage_x[R1B / 32][R1CHUNK];
  __shared__ double s_stage_y[R1B / 32][R1CHUNK];
  __shared__ double s_stage_z[DIM == 3 ? R1B / 32 : 1][DIM == 3 ? R1CHUNK : 1];
  __shared__ uint32_t s_stage_i[R1B / 32][R1CHUNK];
  DevState* st = ws.st;
  const RoundParams rp = st->rp;
  if (!ws.peeled || !rp.active || rp.root || !long_round(rp, st)) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (blockIdx.x == 0 && tid == 0) {
    st->ctr_book = 0;  // K3's tile counter
    st->arrive_book = 0;
    st->book_small = (uint32_t)K * rp.nseg <= BOOK_SMALL ? 1u : 0u;
  }
  const uint32_t nseg = rp.nseg, cur = rp.cur, n_live = rp.n_live;
  const uint32_t* segstart = ws.segstart[cur];
  const uint64_t* seg_phys = ws.seg_phys[cur];
  const SegT* segtab = reinterpret_cast<const SegT*>(ws.seg[cur]);
  const double* inx = ws.rx[cur];
  const double* iny = ws.ry[cur];
  const double* inz = ws.rz[cur];
  const uint32_t* ini = ws.ri[cur];
  uint32_t* cursor = ws.cursor[cur];
  double* outx = ws.rx[cur ^ 1u];
  double* outy = ws.ry[cur ^ 1u];
  double* outz = ws.rz[cur ^ 1u];
  uint32_t* outi = ws.ri[cur ^ 1u];
  const uint64_t rcap = ws.rcap;
  Key128* slot_key = ws.slot_key;

  const uint32_t nchunks = (n_live + R1CHUNK - 1) / R1CHUNK;
  const uint32_t gw = blockIdx.x * (R1B / 32) + warp, nwarps = gridDim.x * (R1B / 32);
  const uint32_t c0 = (uint32_t)(((uint64_t)nchunks * gw) / nwarps);
  const uint32_t c1 = (uint32_t)(((uint64_t)nchunks * (gw + 1)) / nwarps);
  if (c0 >= c1) return;

  // segment containing logical position q (warp-cooperative 32-ary search)
  auto find_segment = [&](uint32_t q) -> uint32_t {
    uint32_t lo = 0, hi = nseg - 1;
    while (hi - lo > 31u) {
      const uint32_t step = (hi - lo + 32u) / 32u;
      const uint32_t idx = lo + lane * step;
      const uint32_t m = __ballot_sync(0xFFFFFFFFu, idx <= hi && __ldg(&segstart[idx]) <= q);
      const uint32_t L = 31u - __clz(m);
      const uint32_t nlo = lo + L * step;
      hi = min(hi, nlo + step - 1u);
      lo = nlo;
    }
    const uint32_t idx = lo + lane;
    const uint32_t m = __ballot_sync(0xFFFFFFFFu, idx <= hi && __ldg(&segstart[idx]) <= q);
    return lo + (31u - __clz(m));
  };
  auto sstart = [&](uint32_t w) -> uint32_t { return w <= nseg ? __ldg(&segstart[w]) : 0xFFFFFFFFu; };

  // window of a chunk: first segment w, starts sA (of w), sB (of w + 1),
  // sC (of w + 2), physical offsets of w and w + 1
  struct Win {
    uint32_t w, sA, sB, sC;
    uint64_t pA, pB;
  };
  auto make_win = [&](uint32_t w) -> Win {
    Win r;
    r.w = w;
    r.sA = sstart(w);
    r.sB = sstart(w + 1);
    r.sC = sstart(w + 2);
    r.pA = __ldg(&seg_phys[w]);
    r.pB = (w + 1 < nseg) ? __ldg(&seg_phys[w + 1]) : 0ull;
    return r;
  };
  auto advance = [&](const Win& cw, uint32_t base) -> Win {
    uint32_t w = cw.w;
    if (base < cw.sB) return cw;
    if (base < cw.sC) return make_win(w + 1);
    w += 2;
    while (sstart(w + 1) <= base) w++;  // rare: several segments skipped
    return make_win(w);
  };
  auto stage_tables = [&](const Win& wn, int par) {
    // the window's (up to) two segment tables into this warp's smem slot
    const unsigned long long* src = reinterpret_cast<const unsigned long long*>(segtab + wn.w);
    unsigned long long* dst = reinterpret_cast<unsigned long long*>(&s_seg[warp][par][0]);
    const uint32_t words = (wn.w + 1 < nseg ? 2u : 1u) * (uint32_t)(sizeof(SegT) / 8);
    for (uint32_t k = lane; k < words; k += 32) dst[k] = __ldg(&src[k]);
    __syncwarp();
  };

  double* stx = s_stage_x[warp];
  double* sty = s_stage_y[warp];
  double* stz = DIM == 3 ? s_stage_z[warp] : nullptr;
  uint32_t* sti = s_stage_i[warp];
  uint32_t pend_base = 0;
  unsigned long long pend_off = 0ull, pend_cnt = 0ull;
  auto flush = [&]() {
    const uint32_t tot = (uint32_t)(((pend_off >> (8 * (NK - 1))) & 0xFFull) + ((pend_cnt >> (8 * (NK - 1))) & 0xFFull));
    for (uint32_t t0 = 0; t0 < tot; t0 += 32) {
      const uint32_t t = t0 + lane;
      uint32_t k = 0;
#pragma unroll
      for (int kk = 1; kk < NK; kk++) k += t >= (uint32_t)((pend_off >> (8 * kk)) & 0xFFull) ? 1u : 0u;
      const uint32_t kb = __shfl_sync(0xFFFFFFFFu, pend_base, k);
      if (t < tot) {
        const size_t dst = (size_t)(k % K) * rcap + kb + (t - (uint32_t)((pend_off >> (8 * k)) & 0xFFull));
        outx[dst] = stx[t];
        outy[dst] = sty[t];
        if (DIM == 3) outz[dst] = stz[t];
        outi[dst] = sti[t];
      }
    }
    pend_off = pend_cnt = 0ull;
    __syncwarp();
  };
  // running farthest keys of the window's children (warp-uniform)
  unsigned long long bh[NK];
  uint32_t bi[NK];
#pragma unroll
  for (int k = 0; k < NK; k++) {
    bh[k] = 0ull;
    bi[k] = 0xFFFFFFFFu;
  }
  uint32_t rw = 0xFFFFFFFFu;  // segment the running keys refer to
  auto merge_keys = [&](int k0, int k1) {
    if (lane == 0)
      for (int k = k0; k < k1; k++)
        if (bh[k]) atomic_max_key(&slot_key[(size_t)(rw + k / K) * K + k % K], bh[k], bi[k]);
  };
  auto move_keys = [&](uint32_t w) {
    if (w == rw) return;
    if (rw != 0xFFFFFFFFu && w == rw + 1) {
      merge_keys(0, K);
#pragma unroll
      for (int k = 0; k < K; k++) {
        bh[k] = bh[k + K];
        bi[k] = bi[k + K];
        bh[k + K] = 0ull;
        bi[k + K] = 0xFFFFFFFFu;
      }
    } else {
      if (rw != 0xFFFFFFFFu) merge_keys(0, NK);
#pragma unroll
      for (int k = 0; k < NK; k++) {
        bh[k] = 0ull;
        bi[k] = 0xFFFFFFFFu;
      }
    }
    rw = w;
  };

  double x[R1ITEMS], y[R1ITEMS], z[R1ITEMS], nx[R1ITEMS], ny[R1ITEMS], nz[R1ITEMS];
  uint32_t ii[R1ITEMS], ni[R1ITEMS];
  auto load_chunk = [&](uint32_t c, const Win& wn) {
    const uint32_t base = c * R1CHUNK;
#pragma unroll
    for (int j = 0; j < R1ITEMS; j++) {
      const uint32_t q = min(base + j * 32 + lane, n_live - 1);
      const uint64_t p = q < wn.sB ? wn.pA + (q - wn.sA) : wn.pB + (q - wn.sB);
      nx[j] = __ldg(&inx[p]);
      ny[j] = __ldg(&iny[p]);
      if (DIM == 3) nz[j] = __ldg(&inz[p]);
      ni[j] = __ldg(&ini[p]);
    }
  };
  auto fast_chunk = [&](const Win& wn, uint32_t base) {
    return wn.sC >= min(base + (uint32_t)R1CHUNK, n_live);
  };

  Win win = make_win(find_segment(c0 * R1CHUNK));
  stage_tables(win, c0 & 1);
  if (fast_chunk(win, c0 * R1CHUNK)) load_chunk(c0, win);
  for (uint32_t c = c0; c < c1; c++) {
    const uint32_t base = c * R1CHUNK;
    const int par = c & 1;
    const bool fast = fast_chunk(win, base);
#pragma unroll
    for (int j = 0; j < R1ITEMS; j++) {
      x[j] = nx[j];
      y[j] = ny[j];
      if (DIM == 3) z[j] = nz[j];
      ii[j] = ni[j];
    }
    // window of the next chunk; prefetch it when it is a fast chunk
    Win nwin = win;
    if (c + 1 < c1) {
      nwin = advance(win, base + R1CHUNK);
      stage_tables(nwin, par ^ 1);
      if (fast_chunk(nwin, base + R1CHUNK)) load_chunk(c + 1, nwin);
    }
    move_keys(win.w);
    if (!fast) {
      // three or more segments in the chunk: point by point
      flush();
#pragma unroll 1
      for (int j = 0; j < R1ITEMS; j++) {
        const uint32_t q = base + j * 32 + lane;
        if (q >= n_live) continue;
        uint32_t lo = win.w, hi = nseg - 1;  // largest w with segstart[w] <= q
        while (lo < hi) {
          const uint32_t mid = (lo + hi + 1) >> 1;
          if (__ldg(&segstart[mid]) <= q) lo = mid;
          else hi = mid - 1;
        }
        const uint64_t p = __ldg(&seg_phys[lo]) + (q - __ldg(&segstart[lo]));
        const double qx = __ldg(&inx[p]), qy = __ldg(&iny[p]), qz = DIM == 3 ? __ldg(&inz[p]) : 0.0;
        const uint32_t qi = __ldg(&ini[p]);
        const SegT& g = segtab[lo];
        double dn;
        int s;
        if constexpr (DIM == 2) s = classify2_bf(g, qx, qy, qi, &dn);
        else s = classify3_bf(g, qx, qy, qz, qi, &dn);
        if (s < 0) continue;
        const size_t e = (size_t)lo * K + s;
        const uint32_t pos = atomicAdd(&cursor[e], 1u);
        const size_t dst = (size_t)s * rcap + pos;
        outx[dst] = qx;
        outy[dst] = qy;
        if (DIM == 3) outz[dst] = qz;
        outi[dst] = qi;
        atomic_max_key(&slot_key[e], (unsigned long long)__double_as_longlong(dn) | 0x8000000000000000ull, qi);
      }
      __syncwarp();
      win = nwin;
      continue;
    }
    uint32_t key[R1ITEMS], hu[R1ITEMS], hl[R1ITEMS];
#pragma unroll
    for (int j = 0; j < R1ITEMS; j++) {
      const uint32_t q = base + j * 32 + lane;
      const uint32_t wsl = q < win.sB ? 0u : 1u;
      double dn;
      int s;
      if constexpr (DIM == 2) s = classify2_bf(s_seg[warp][par][wsl], x[j], y[j], ii[j], &dn);
      else s = classify3_bf(s_seg[warp][par][wsl], x[j], y[j], z[j], ii[j], &dn);
      const bool keep = (q < n_live) & (s >= 0);
      key[j] = keep ? wsl * K + (uint32_t)s : 0xFFFFFFFFu;
      hu[j] = (uint32_t)__double2hiint(dn) | 0x80000000u;
      hl[j] = (uint32_t)__double2loint(dn);
    }
    uint32_t rank[R1ITEMS];
    const unsigned long long packed = chunk_ranks<NK, R1ITEMS>(key, rank);
    unsigned long long off = 0ull;
#pragma unroll
    for (int k = 1; k < NK; k++)
      off |= ((((off >> (8 * (k - 1))) & 0xFFull) + ((packed >> (8 * (k - 1))) & 0xFFull)) << (8 * k));
    flush();
#pragma unroll
    for (int j = 0; j < R1ITEMS; j++) {
      const uint32_t kj = key[j];
      if (kj < (uint32_t)NK) {
        const uint32_t t = (uint32_t)((off >> (8 * kj)) & 0xFFull) + rank[j];
        stx[t] = x[j];
        sty[t] = y[j];
        if (DIM == 3) stz[t] = z[j];
        sti[t] = ii[j];
      }
    }
    __syncwarp();
    const uint32_t mycnt = lane < NK ? (uint32_t)((packed >> (8 * lane)) & 0xFFull) : 0u;
    pend_base = mycnt ? atomicAdd(&cursor[(size_t)(win.w + lane / K) * K + lane % K], mycnt) : 0u;
    pend_off = off;
    pend_cnt = packed;
    // per child: does any survivor reach its running maximum?  (boolean
    // per child, so the running maxima stay in registers)
    uint32_t need = 0;
#pragma unroll
    for (int k = 0; k < NK; k++) {
      const uint32_t tk = (uint32_t)(bh[k] >> 32);
      bool ck = false;
#pragma unroll
      for (int j = 0; j < R1ITEMS; j++) ck |= (key[j] == (uint32_t)k) & (hu[j] >= tk);
      need |= __any_sync(0xFFFFFFFFu, ck) ? (1u << k) : 0u;
    }
    if (need) {
#pragma unroll
      for (int k = 0; k < NK; k++) {
        if (!((need >> k) & 1u)) continue;
        uint32_t tu = 0, tl = 0, ti = 0xFFFFFFFFu;
#pragma unroll
        for (int j = 0; j < R1ITEMS; j++) {
          const bool mine = key[j] == (uint32_t)k;
          const bool better = mine && (hu[j] > tu || (hu[j] == tu && (hl[j] > tl || (hl[j] == tl && ii[j] < ti))));
          tu = better ? hu[j] : tu;
          tl = better ? hl[j] : tl;
          ti = better ? ii[j] : ti;
        }
        const uint32_t mu = __reduce_max_sync(0xFFFFFFFFu, tu);
        if (mu == 0u || mu < (uint32_t)(bh[k] >> 32)) continue;
        const uint32_t ml = __reduce_max_sync(0xFFFFFFFFu, tu == mu ? tl : 0u);
        const unsigned long long h = ((unsigned long long)mu << 32) | ml;
        const uint32_t mi = __reduce_min_sync(0xFFFFFFFFu, (tu == mu && tl == ml) ? ti : 0xFFFFFFFFu);
        if (h > bh[k] || (h == bh[k] && mi < bi[k])) {
          bh[k] = h;
          bi[k] = mi;
        }
      }
    }
    win = nwin;
  }
  flush();
  if (rw != 0xFFFFFFFFu) merge_keys(0, NK);
}

}  // namespace sh
