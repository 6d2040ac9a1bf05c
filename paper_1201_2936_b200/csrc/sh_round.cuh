// K2: the fused Quickhull round kernel.
//
// One launch processes one whole round over all segments at once, reading
// every live record once and writing every survivor once
// (quickhull.py:229-266 / :372-437).  Round 1 is fused with the first split
// (quickhull.py:200-222 / :346-364): it reads the input and re-derives each
// point's side, so the split's survivors are never materialised
// (MODE_ROUND1; k_first_count only counts the split and finds its apexes).
//
// Work split: persistent blocks, each owning a static contiguous range of
// 512-point tiles.  Tiles are independent -- there is no tile-to-tile
// prefix chain: every child (parent segment p, state s) owns a disjoint
// region of output stream s starting at p's start, and survivors claim
// positions in it with one shared-memory atomic per warp and one global
// atomicAdd per (tile, child).  Order inside a child is free because
// records carry their original index.
//
// Per tile:
//   * the records were prefetched into shared memory with cp.async while the
//     previous tile was processed (double buffering); the tile's segment
//     window (start, physical offset of every segment overlapping the tile)
//     is staged in shared memory;
//   * classification against the segment's simplex in the reference's fp64
//     operation order: discard test, child state, and the child's distance
//     for the next round (the next round's farthest-point key);
//   * per-child counts and farthest keys: warp ballots + REDUX reductions
//     when a 32-point slot lies in one segment (the common case), shared
//     atomics otherwise; then one global cursor claim per child;
//   * survivors are written straight from the staged records;
//   * a child's farthest key is stored directly when the child lies inside
//     one tile, carried to the block's next tile when its segment continues,
//     and merged with a 128-bit atomicCAS when several blocks share it.
// Windows wider than WMAX segments (late rounds of tiny segments) take a
// slow path with per-point global atomics.
#pragma once

#include <type_traits>

#include "sh_common.cuh"

namespace sh {

constexpr uint32_t NOKEY = 0xFFFFFFFFu;

template <int DIM>
struct RoundSmem {
  // one stage: DIM coordinate arrays, original index, window index
  static constexpr size_t stage_bytes() { return (size_t)RTILE * (8 * DIM + 4 + 2); }
  static constexpr size_t bytes() { return 2 * stage_bytes(); }
};

template <int DIM>
struct RoundShared {
  uint32_t wstart[2][WMAX + 2];      // window: dense start of every segment (+ next)
  unsigned long long wphys[2][WMAX + 1];  // window: physical offset of every segment
  uint32_t wlo[2], wn[2], wslow[2], wnext[2];
  uint32_t wslot[2][RTILE / 32];     // window segment of each 32-point slot's first point
  __align__(16) unsigned long long seg0[2][(sizeof(Seg3) + 15) / 16 * 2];  // first segment's table
  uint32_t kcnt[WMAX * DIM];         // per (window segment, state) of the current tile
  uint32_t kbase[WMAX * DIM];
  uint32_t khh[WMAX * DIM];          // farthest key, upper / lower 32 bits
  uint32_t khl[WMAX * DIM];
  uint32_t kidx[WMAX * DIM];
  uint32_t pend_seg[2];              // segment carried into the next tile (by tile parity)
  uint32_t pend_complete[2];         // its aggregate covers it from its first point
  unsigned long long pend_hi[2][DIM];
  uint32_t pend_idx[2][DIM];
  // uniform tiles: per-warp totals / maxima, then per-warp output bases
  uint32_t wtot[RB / 32][2 * DIM];
  unsigned long long whi[RB / 32][2 * DIM];
  uint32_t widx[RB / 32][2 * DIM];
  uint32_t boff[RB / 32][2 * DIM];
  // ROUND1: the block's running farthest keys of round 1's children
  unsigned long long racc_hi[2 * DIM];
  uint32_t racc_idx[2 * DIM];
};

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Classification of one point against its segment (2D), quickhull.py:230-266.
// Returns state in {-1 (discard), 0, 1} and the child's next-round distance.
__device__ __forceinline__ int classify2(const Seg2& g, double qx, double qy, uint32_t qi,
                                         double* dnext) {
  if (qi == g.fidx) return -1;  // keep[far_seg] = False (:244)
  // point_in_triangle(ea, eb, fq, q, eps), geometry.py:150-156, is
  //   d >= (-eps)|ab|  &  cross2(b, far, q) >= (-eps)|bf|  &  cross2(far, a, q) >= (-eps)|fa|
  // with d = cross2(a, b, q) > 0 for every live point (by induction: the
  // first split keeps |d| > eps|pmin pmax| on each side, and a survivor's
  // next distance is a strictly positive c0 or c1, computed with the very
  // operation order the next round uses for d), so the first clause is
  // always true and d is not recomputed.
  // classify_two_edges(a, far, b, q), geometry.py:178-189
  double c0 = cross2(g.ax, g.ay, g.fx, g.fy, qx, qy);  // cross2(a, far, q)
  double c1 = cross2(g.fx, g.fy, g.bx, g.by, qx, qy);  // cross2(far, b, q)
  // cross2(b, far, q) == -c1 and cross2(far, a, q) == -c0 bit-exactly (the
  // symmetric form negates every term exactly, test_geometry.py:35-38)
  bool inside = (-c1 >= g.nt_bf) & (-c0 >= g.nt_fa);
  if (inside) return -1;
  bool one_sided = (c0 > 0) != (c1 > 0);
  int state = one_sided ? (c1 > 0 ? 1 : 0) : (c1 > c0 ? 1 : 0);
  *dnext = state ? c1 : c0;  // next round: cross2(a, far, q) / cross2(far, b, q)
  return state;
}

// 3D, quickhull.py:372-437 with point_in_tetrahedron (geometry.py:163-175)
// and classify_three_faces (geometry.py:192-208).
__device__ __forceinline__ int classify3(const Seg3& g, double qx, double qy, double qz, uint32_t qi,
                                         double* dnext) {
  if (g.flat) return -1;          // keep &= ~flat_seg[ids] (:399)
  if (qi == g.fidx) return -1;    // keep[far_seg] = False (:398)
  // base clause d >= (-eps)|n| of point_in_tetrahedron always holds for a
  // live point (same induction as classify2: side-0 points of the first
  // split have d >= (-eps)*nlen, the same product; every later distance is
  // the positive winning D_j, bit-identical to the next round's d)
  double D0 = plane_dist(g.N[0], g.a, qx, qy, qz);
  double D1 = plane_dist(g.N[1], g.b, qx, qy, qz);
  double D2 = plane_dist(g.N[2], g.c, qx, qy, qz);
  bool inside = (D0 <= g.thr[0]) & (D1 <= g.thr[1]) & (D2 <= g.thr[2]);
  if (inside) return -1;
  // first argmax of D_j / |N_j| (np.argmax over the stacked quotients)
  int state = 0;
  double db = D0, nb = g.nrm[0];
  if (quotient_gt_warp(D1, g.nrm[1], db, nb)) { state = 1; db = D1; nb = g.nrm[1]; }
  if (quotient_gt_warp(D2, g.nrm[2], db, nb)) { state = 2; db = D2; }
  *dnext = db;
  return state;
}

// largest w in [0, n) with start[w] <= q
__device__ __forceinline__ uint32_t win_search(const uint32_t* start, uint32_t n, uint32_t q) {
  uint32_t lo = 0, hi = n - 1;
  while (lo < hi) {
    uint32_t mid = (lo + hi + 1) >> 1;
    if (start[mid] <= q) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// (The first split itself is a read-only counting pass, k_first_count.)
// MODE_ROUND1: round 1 fused with the first split: reads the input, drops
//   what the first split drops, classifies the rest against the side's
//   round-1 segment, writes round 1's survivors.
// MODE_NORMAL: rounds 2.. over the records of the previous round.
constexpr int MODE_ROUND1 = 1, MODE_NORMAL = 2;

template <int DIM, int MODE>
__global__ void __launch_bounds__(RB) k_round(Workspace ws) {
  constexpr int K = DIM;
  constexpr bool R1 = MODE == MODE_ROUND1;
  constexpr bool INPUT = MODE != MODE_NORMAL;  // tiles over the caller's points
  DevState* st = ws.st;
  extern __shared__ __align__(16) unsigned char dsm[];
  __shared__ RoundShared<DIM> S;
  const int tid = threadIdx.x, lane = tid & 31;

  const RoundParams rp = st->rp;
  if (!rp.active || rp.root || R1 != (rp.round == 1)) return;
#ifndef SH_LEAN_LONG
#define SH_LEAN_LONG 1
#endif
  if (!R1 && SH_LEAN_LONG && ws.peeled && long_round(rp, st)) return;  // k_stream (sh_stream.cuh) runs it
  if (blockIdx.x == 0 && tid == 0) {
    st->ctr_book = 0;  // K3's tile counter
    st->arrive_book = 0;
    st->book_small = (uint32_t)K * rp.nseg <= BOOK_SMALL ? 1u : 0u;
  }
  const uint32_t nseg = rp.nseg, cur = rp.cur;
  const uint32_t n_live = INPUT ? st->n : rp.n_live;  // positions the tiles cover
  const uint32_t num_tiles = (n_live + RTILE - 1) / RTILE;
  const uint32_t t0 = (uint32_t)(((uint64_t)num_tiles * blockIdx.x) / gridDim.x);
  const uint32_t t1 = (uint32_t)(((uint64_t)num_tiles * (blockIdx.x + 1)) / gridDim.x);
  if (t0 >= t1) return;
  const uint64_t rcap = ws.rcap;
  const double* inx = ws.rx[cur];
  const double* iny = ws.ry[cur];
  const double* inz = ws.rz[cur];
  const uint32_t* ini = ws.ri[cur];
  double* outx = ws.rx[cur ^ 1u];
  double* outy = ws.ry[cur ^ 1u];
  double* outz = ws.rz[cur ^ 1u];
  uint32_t* outi = ws.ri[cur ^ 1u];
  const uint32_t* segstart = ws.segstart[cur];
  const uint64_t* seg_phys = ws.seg_phys[cur];
  uint32_t* cursor = ws.cursor[cur];

  // first-split constants
  double f_pa[3], f_pb[3], f_nrm[3], f_thr = 0;
  uint32_t f_imin = 0, f_imax = 0, f_ifar = 0xFFFFFFFFu;
  const double* px = st->px;
  const double* py = st->py;
  const double* pz = st->pz;
  const int64_t pstride = st->stride;
  if (INPUT) {
#pragma unroll
    for (int k = 0; k < 3; k++) {
      f_pa[k] = st->pa[k];
      f_pb[k] = st->pb[k];
      f_nrm[k] = st->nrm[k];
    }
    f_thr = st->thr_line;
    f_imin = st->imin;
    f_imax = st->imax;
    if (DIM == 3) f_ifar = st->ifar;
  }
  // ROUND1: segment of each first-split side (side 0 is segment 0 when it
  // has survivors; the root children's counts are still in cursor[0])
  uint32_t side_seg[2] = {0u, 0u};
  if (R1) side_seg[1] = ws.cursor[0][0] ? 1u : 0u;

  auto stage_ptr = [&](uint32_t b) { return dsm + (size_t)b * RoundSmem<DIM>::stage_bytes(); };

  // ---- window of tile t into buffer b (warp 0)
  // segment containing logical position q (warp-cooperative 32-ary search)
  auto find_segment = [&](uint32_t q) -> uint32_t {
    uint32_t lo = 0, hi = nseg - 1;
    while (hi - lo > 31u) {
      const uint32_t step = (hi - lo + 32u) / 32u;  // ceil(range size / 32)
      const uint32_t idx = lo + lane * step;  // probes beyond hi do not vote
      const uint32_t m = __ballot_sync(0xFFFFFFFFu, idx <= hi && segstart[idx] <= q);
      const uint32_t L = 31u - __clz(m);
      const uint32_t nlo = lo + L * step;
      hi = min(hi, nlo + step - 1u);
      lo = nlo;
    }
    const uint32_t idx = lo + lane;
    const uint32_t m = __ballot_sync(0xFFFFFFFFu, idx <= hi && segstart[idx] <= q);
    return lo + (31u - __clz(m));
  };

  // ---- window of tile t into buffer b (warp 0): every segment overlapping
  // the tile, found by scanning segstart forward from the tile's first
  // segment (carried from the previous tile's window; a 32-ary search for a
  // block's first tile)
  auto load_window = [&](uint32_t t, uint32_t b) {
    if (INPUT) {
      // ROUND1: the round-1 segments are the first split's sides,
      // interleaved in input order
      if (lane == 0) {
        S.wlo[b] = 0;
        S.wn[b] = nseg;
        S.wslow[b] = 0;
        S.wstart[b][0] = 0;
        S.wstart[b][1] = 0;
        S.wphys[b][0] = 0;
      }
      return;
    }
    const uint32_t base = t * RTILE, end = min(base + (uint32_t)RTILE, n_live);
    const uint32_t lo = (t == t0) ? find_segment(base) : S.wnext[b ^ 1u];
    // the first 32 segments' physical offsets and segment lo's table, in
    // flight with the scan of their starts (one memory round trip)
    using SegT0 = typename std::conditional<DIM == 2, Seg2, Seg3>::type;
    constexpr uint32_t TW = sizeof(SegT0) / 8;
    static_assert(TW <= 32, "one table word per lane");
    const unsigned long long phys0 = lo + lane < nseg ? seg_phys[lo + lane] : 0ull;
    const unsigned long long tw0 =
        lane < TW ? reinterpret_cast<const unsigned long long*>(ws.seg[cur])[(size_t)lo * TW + lane] : 0ull;
    uint32_t nw = 0, nxt = lo;
    for (uint32_t w0 = 0;; w0 += 32) {
      const uint32_t idx = lo + w0 + lane;
      const uint32_t st_ = idx <= nseg ? segstart[idx] : 0xFFFFFFFFu;  // segstart[nseg] = n_live
      if (w0 + lane <= (uint32_t)WMAX) S.wstart[b][w0 + lane] = st_;
      const uint32_t m = __ballot_sync(0xFFFFFFFFu, st_ < end);
      if (m != 0xFFFFFFFFu) {
        const uint32_t c = __popc(m);  // segments of this batch that start inside the tile
        nw = w0 + c;
        // first position of the next tile: in segment lo+nw-1, or lo+nw when it starts there
        const uint32_t nstart = __shfl_sync(0xFFFFFFFFu, st_, c & 31u);
        nxt = lo + nw - 1 + ((c < 32u && nstart == end) ? 1u : 0u);
        break;
      }
    }
    const bool slow = nw > (uint32_t)WMAX;
    if (!slow) {
      if (lane < nw) S.wphys[b][lane] = phys0;
      for (uint32_t w = 32 + lane; w < nw; w += 32) S.wphys[b][w] = seg_phys[lo + w];
      __syncwarp();
      // one binary search per 32-point slot (all slots at once, one per lane)
      const uint32_t q = base + lane * 32;
      if (lane < RTILE / 32) S.wslot[b][lane] = q < n_live ? win_search(S.wstart[b], nw, q) : 0u;
    }
    if (lane < TW) S.seg0[b][lane] = tw0;
    if (lane == 0) {
      S.wlo[b] = lo;
      S.wn[b] = nw;
      S.wslow[b] = slow ? 1u : 0u;
      S.wnext[b] = nxt;
    }
  };

  // ---- cp.async the records of tile t into stage b (all threads; window b ready)
  auto issue_items = [&](uint32_t t, uint32_t b) {
    unsigned char* sp = stage_ptr(b);
    double* sx = reinterpret_cast<double*>(sp);
    uint32_t* si = reinterpret_cast<uint32_t*>(sx + DIM * RTILE);
    uint16_t* sw = reinterpret_cast<uint16_t*>(si + RTILE);
    const uint32_t base = t * RTILE;
    const uint32_t cnt = min((uint32_t)RTILE, n_live - base);
    const uint32_t lo = S.wlo[b], nw = S.wn[b];
    const bool slow = S.wslow[b] != 0;
    // a full tile inside one segment is one contiguous run of records:
    // 16-byte copies when the run is aligned
    const double *gx = nullptr, *gy = nullptr, *gz = nullptr;
    const uint32_t* gi = nullptr;
    bool contig = false;
    if (INPUT) {
      contig = pstride == 1;
      gx = px + base;
      gy = py + base;
      gz = pz + base;
    } else if (!slow && S.wstart[b][1] >= base + cnt) {
      const uint64_t p0 = S.wphys[b][0] + (base - S.wstart[b][0]);
      contig = true;
      gx = inx + p0;
      gy = iny + p0;
      gz = inz + p0;
      gi = ini + p0;
    }
    auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
    if (contig && cnt == RTILE && al16(gx) && al16(gy) && (DIM == 2 || al16(gz))) {
#pragma unroll
      for (int jp = 0; jp < RITEMS / 2; jp++) {
        const uint32_t e = 2 * (jp * RB + tid);
        cp_async16(&sx[e], gx + e);
        cp_async16(&sx[RTILE + e], gy + e);
        if (DIM == 3) cp_async16(&sx[2 * RTILE + e], gz + e);
      }
      if (!INPUT) {
        if (al16(gi)) {
#pragma unroll
          for (int jq = 0; jq < RITEMS / 4; jq++) {
            const uint32_t e = 4 * (jq * RB + tid);
            cp_async16(&si[e], gi + e);
          }
        } else {
#pragma unroll
          for (int j = 0; j < RITEMS; j++) cp_async4(&si[j * RB + tid], gi + j * RB + tid);
        }
      }
      cp_async_commit();
      return;
    }
#pragma unroll
    for (int j = 0; j < RITEMS; j++) {
      const uint32_t i = j * RB + tid;
      const uint32_t q = base + i;
      uint32_t wfast = 0;
      if (!INPUT && !contig && !slow) {
        // segment of q: the slot's first segment + the starts inside the slot
        const uint32_t wb = S.wslot[b][i >> 5];
        const uint32_t slot0 = base + (i & ~31u);
        const uint32_t k = wb + 1 + lane;
        const uint32_t off = (k <= nw) ? S.wstart[b][k] - slot0 : 32u;
        const uint32_t m = __reduce_or_sync(0xFFFFFFFFu, off < 32u ? (1u << off) : 0u);
        const uint32_t le = (lane == 31) ? 0xFFFFFFFFu : ((2u << lane) - 1u);
        wfast = wb + __popc(m & le);
      }
      if (i >= cnt) continue;
      if (INPUT) {
        const int64_t o = (int64_t)q * pstride;
        cp_async8(&sx[i], px + o);
        cp_async8(&sx[RTILE + i], py + o);
        if (DIM == 3) cp_async8(&sx[2 * RTILE + i], pz + o);
      } else if (contig) {
        cp_async8(&sx[i], gx + i);
        cp_async8(&sx[RTILE + i], gy + i);
        if (DIM == 3) cp_async8(&sx[2 * RTILE + i], gz + i);
        cp_async4(&si[i], gi + i);
      } else {
        uint32_t w;
        uint64_t phys;
        if (!slow) {
          w = wfast;
          phys = S.wphys[b][w] + (q - S.wstart[b][w]);
        } else {
          w = win_search(segstart + lo, nw, q);
          phys = seg_phys[lo + w] + (q - segstart[lo + w]);
        }
        sw[i] = (uint16_t)w;
        cp_async8(&sx[i], inx + phys);
        cp_async8(&sx[RTILE + i], iny + phys);
        if (DIM == 3) cp_async8(&sx[2 * RTILE + i], inz + phys);
        cp_async4(&si[i], ini + phys);
      }
    }
    cp_async_commit();
  };

  // ---- prologue
  if (tid < K * WMAX) {
    for (uint32_t e = tid; e < (uint32_t)(K * WMAX); e += RB) {
      S.kcnt[e] = 0;
      S.khh[e] = 0u;
      S.khl[e] = 0u;
      S.kidx[e] = 0xFFFFFFFFu;
    }
  }
  if (tid < 2) {
    S.pend_seg[tid] = NOKEY;
    S.pend_complete[tid] = 0;
  }
  if (tid < 2 * K) {
    S.racc_hi[tid] = 0ull;
    S.racc_idx[tid] = 0xFFFFFFFFu;
  }
  if (R1) {
    // round 1's (at most two) segment tables, constant for the whole launch
    using SegT = typename std::conditional<DIM == 2, Seg2, Seg3>::type;
    const unsigned long long* src = reinterpret_cast<const unsigned long long*>(ws.seg[cur]);
    for (uint32_t k = tid; k < nseg * (sizeof(SegT) / 8); k += RB)
      S.seg0[k / (sizeof(SegT) / 8)][k % (sizeof(SegT) / 8)] = src[k];
  }
  if (tid < 32) load_window(t0, 0);
  __syncthreads();
  issue_items(t0, 0);

  for (uint32_t t = t0; t < t1; t++) {
    const uint32_t lt = t - t0;
    const uint32_t b = lt & 1u;
    const bool has_next = t + 1 < t1;
    if (has_next && tid < 32) load_window(t + 1, b ^ 1u);
    cp_async_wait_all();
    __syncthreads();  // stage b landed, window b^1 staged
    if (has_next) issue_items(t + 1, b ^ 1u);

    const uint32_t tile_begin = t * RTILE;
    const uint32_t tile_end = min(tile_begin + RTILE, n_live);
    const uint32_t lo = S.wlo[b], nw = S.wn[b];
    const bool slow = S.wslow[b] != 0;
    unsigned char* sp = stage_ptr(b);
    const double* sx = reinterpret_cast<const double*>(sp);
    const uint32_t* si = reinterpret_cast<const uint32_t*>(sx + DIM * RTILE);
    const uint16_t* sw = reinterpret_cast<const uint16_t*>(si + RTILE);
    const uint32_t pin = (lt + 1u) & 1u;  // pending written by the previous tile
    const uint32_t pout = lt & 1u;

    // ---- classify
    const bool uniform = S.wstart[b][1] >= tile_end;  // the whole tile lies in window segment 0
    uint32_t key[RITEMS], rank[RITEMS];
    unsigned long long khi_[RITEMS];
    uint32_t wv[RITEMS];  // window segment of each item
    auto classify_item = [&](int j, bool uni, auto&& seg_of) {
      const uint32_t i = j * RB + tid;
      const uint32_t q = tile_begin + i;
      key[j] = NOKEY;
      rank[j] = 0;
      khi_[j] = 0;
      wv[j] = 0;
      if (q >= tile_end) return;
      const double qx = sx[i], qy = sx[RTILE + i];
      const double qz = (DIM == 3) ? sx[2 * RTILE + i] : 0.0;
      uint32_t w = (uni || INPUT) ? 0u : (uint32_t)sw[i];
      double dn = 0.0;
      int s = -1;
      if (INPUT) {
        if (DIM == 2) {
          if (q != f_imin && q != f_imax) {
            // quickhull.py:202-211
            double d = cross2(f_pa[0], f_pa[1], f_pb[0], f_pb[1], qx, qy);
            if (fabs(d) > f_thr) {
              s = d < 0 ? 1 : 0;
              dn = s ? -d : d;  // cross2(pmax, pmin, q) == -d exactly
            }
          }
        } else {
          if (q != f_imin && q != f_imax && q != f_ifar) {
            // quickhull.py:348-353
            double d = plane_dist(f_nrm, f_pa, qx, qy, qz);
            s = d < f_thr ? 1 : 0;
            dn = s ? -d : d;  // face (pa, pc, pb) has normal -n exactly
          }
        }
        if (R1 && s >= 0) {
          // round 1 on the survivors of the split: the side's segment
          w = side_seg[s];
          if constexpr (DIM == 2) s = classify2(seg_of(w), qx, qy, q, &dn);
          else s = classify3(seg_of(w), qx, qy, qz, q, &dn);
        }
      } else {
        const uint32_t qi = si[i];
        if (qi == DEAD) {  // padding record (sh_common.cuh)
          wv[j] = w;
          return;
        }
        if constexpr (DIM == 2) s = classify2(seg_of(w), qx, qy, qi, &dn);
        else s = classify3(seg_of(w), qx, qy, qz, qi, &dn);
      }
      wv[j] = w;
      if (s >= 0) {
        key[j] = w * K + (uint32_t)s;
        // d > 0 for every live point (see classify2), so the raw bits order
        // like ordered_bits(d)
        khi_[j] = (unsigned long long)__double_as_longlong(dn) | 0x8000000000000000ull;
      }
    };
    using SegT = typename std::conditional<DIM == 2, Seg2, Seg3>::type;
    const SegT* segtab = reinterpret_cast<const SegT*>(ws.seg[cur]);
    if (uniform && !slow && !R1) {
      const SegT g0 = *reinterpret_cast<const SegT*>(S.seg0[b]);  // staged with the window
#pragma unroll
      for (int j = 0; j < RITEMS; j++) classify_item(j, true, [&](uint32_t) -> SegT { return g0; });
    } else if (R1) {
#pragma unroll
      for (int j = 0; j < RITEMS; j++)
        classify_item(j, false, [&](uint32_t w) -> const SegT& { return *reinterpret_cast<const SegT*>(S.seg0[w]); });
    } else {
#pragma unroll
      for (int j = 0; j < RITEMS; j++)
        classify_item(j, false, [&](uint32_t w) -> const SegT& { return segtab[lo + w]; });
    }

    // close, carry or merge child (window segment w, state s) of this tile
    auto close_child = [&](uint32_t w, uint32_t s, unsigned long long hi, uint32_t idx) {
      const uint32_t seg = lo + w;
      const uint32_t segbeg = S.wstart[b][w], segend = S.wstart[b][w + 1];
      bool complete = segbeg >= tile_begin;
      if (w == 0 && S.pend_seg[pin] == seg) {
        const unsigned long long ph = S.pend_hi[pin][s];
        const uint32_t pi = S.pend_idx[pin][s];
        if (ph > hi || (ph == hi && pi < idx)) {
          hi = ph;
          idx = pi;
        }
        complete = S.pend_complete[pin] != 0;
      }
      const bool continues = segend > tile_end;
      if (continues && has_next && w == nw - 1) {
        S.pend_hi[pout][s] = hi;
        S.pend_idx[pout][s] = idx;
        if (s == 0) {
          S.pend_seg[pout] = seg;
          S.pend_complete[pout] = complete ? 1u : 0u;
        }
      } else if (hi) {
        Key128* slot = &ws.slot_key[(size_t)seg * K + s];
        if (complete && !continues) {
          Key128 kv;
          kv.hi = hi;
          kv.lo = idx;
          st_cg(slot, kv);
        } else {
          atomic_max_key(slot, hi, idx);
        }
      }
    };
    const int warp = tid >> 5;

    if (!slow && uniform && !R1) {
      // ---- few keys (one segment's K states; ROUND1: both sides' states):
      // ballots for ranks, register maxima, one claim per key
      constexpr int NK = K;
      const uint32_t nk = (uint32_t)K;
      uint32_t wrun[NK];
      unsigned long long hm[NK];
      uint32_t im[NK];
#pragma unroll
      for (int s = 0; s < NK; s++) {
        wrun[s] = 0;
        hm[s] = 0ull;
        im[s] = 0xFFFFFFFFu;
      }
#pragma unroll
      for (int j = 0; j < RITEMS; j++) {
        uint32_t r = 0;
#pragma unroll
        for (int s = 0; s < NK; s++) {
          const bool mine = key[j] == (uint32_t)s;
          const uint32_t m = __ballot_sync(0xFFFFFFFFu, mine);
          r = mine ? wrun[s] + __popc(m & lanemask_lt()) : r;
          wrun[s] += __popc(m);
          const unsigned long long v = mine ? khi_[j] : 0ull;
          hm[s] = v > hm[s] ? v : hm[s];
        }
        rank[j] = r;
      }
#pragma unroll
      for (int s = 0; s < NK; s++) {
        const uint32_t mu = __reduce_max_sync(0xFFFFFFFFu, (uint32_t)(hm[s] >> 32));
        const uint32_t ml = __reduce_max_sync(0xFFFFFFFFu, ((uint32_t)(hm[s] >> 32) == mu) ? (uint32_t)hm[s] : 0u);
        hm[s] = ((unsigned long long)mu << 32) | ml;
      }
      // lowest original index among the warp's farthest points
#pragma unroll
      for (int j = 0; j < RITEMS; j++) {
        const uint32_t i = j * RB + tid;
        const uint32_t qi = INPUT ? tile_begin + i : si[i];
#pragma unroll
        for (int s = 0; s < NK; s++) {
          const uint32_t c = (key[j] == (uint32_t)s && khi_[j] == hm[s]) ? qi : 0xFFFFFFFFu;
          im[s] = c < im[s] ? c : im[s];
        }
      }
#pragma unroll
      for (int s = 0; s < NK; s++) {
        im[s] = __reduce_min_sync(0xFFFFFFFFu, im[s]);
        if (lane == 0) {
          S.wtot[warp][s] = wrun[s];
          S.whi[warp][s] = hm[s];
          S.widx[warp][s] = im[s];
        }
      }
      __syncthreads();
      if (tid < nk) {
        const uint32_t s = tid;
        uint32_t tot = 0;
        unsigned long long hi = 0ull;
        uint32_t idx = 0xFFFFFFFFu;
#pragma unroll
        for (int w = 0; w < RB / 32; w++) {
          tot += S.wtot[w][s];
          const unsigned long long h2 = S.whi[w][s];
          const uint32_t i2 = S.widx[w][s];
          if (h2 > hi || (h2 == hi && i2 < idx)) {
            hi = h2;
            idx = i2;
          }
        }
        uint32_t base = tot ? atomicAdd(&cursor[(size_t)lo * K + s], tot) : 0u;
#pragma unroll
        for (int w = 0; w < RB / 32; w++) {
          S.boff[w][s] = base;
          base += S.wtot[w][s];
        }
        if (R1) {
          // round 1's children are interleaved over the whole input: fold
          // into the block's running maxima, merged once per block below
          if (hi > S.racc_hi[s] || (hi == S.racc_hi[s] && hi && idx < S.racc_idx[s])) {
            S.racc_hi[s] = hi;
            S.racc_idx[s] = idx;
          }
        } else {
          close_child(0, s, hi, idx);
        }
      }
      __syncthreads();
      size_t wb[NK];
#pragma unroll
      for (int s = 0; s < NK; s++) wb[s] = (size_t)(s % K) * rcap + S.boff[warp][s];
#pragma unroll
      for (int j = 0; j < RITEMS; j++) {
        if (key[j] == NOKEY) continue;
        const uint32_t i = j * RB + tid;
        size_t dst = wb[0];
#pragma unroll
        for (int s = 1; s < NK; s++) dst = key[j] == (uint32_t)s ? wb[s] : dst;
        dst += rank[j];
        outx[dst] = sx[i];
        outy[dst] = sx[RTILE + i];
        if (DIM == 3) outz[dst] = sx[2 * RTILE + i];
        outi[dst] = INPUT ? (tile_begin + i) : si[i];
      }
      if (tid == 0 && !(has_next && S.wstart[b][nw] > tile_end)) S.pend_seg[pout] = NOKEY;
    } else if (!slow) {
      // ---- per (segment, state): tile-local ranks, counts, farthest keys
      // (upper 32 bits of the key by shared atomicMax now, lower 32 bits
      // among the upper-bit winners after the barrier: native 32-bit atomics)
#pragma unroll
      for (int j = 0; j < RITEMS; j++) {
        const uint32_t i = j * RB + tid;
        const bool valid = tile_begin + i < tile_end;
        const uint32_t w = valid ? wv[j] : 0u;
        const uint32_t wmin = __reduce_min_sync(0xFFFFFFFFu, valid ? w : 0xFFFFu);
        const uint32_t wmax = __reduce_max_sync(0xFFFFFFFFu, valid ? w : 0u);
        const uint32_t hu = (uint32_t)(khi_[j] >> 32);
        if (wmin == wmax) {
          // one segment in this 32-point slot: ballots + REDUX per state
#pragma unroll
          for (int s = 0; s < K; s++) {
            const uint32_t kk = wmin * K + s;
            const bool mine = key[j] == kk;
            const uint32_t m = __ballot_sync(0xFFFFFFFFu, mine);
            if (!m) continue;
            const uint32_t mu = __reduce_max_sync(0xFFFFFFFFu, mine ? hu : 0u);
            const int leader = __ffs(m) - 1;
            uint32_t off = 0;
            if (lane == leader) {
              off = atomicAdd(&S.kcnt[kk], (uint32_t)__popc(m));
              atomicMax(&S.khh[kk], mu);
            }
            off = __shfl_sync(0xFFFFFFFFu, off, leader);
            if (mine) rank[j] = off + __popc(m & lanemask_lt());
          }
        } else {
          const uint32_t grp = __match_any_sync(0xFFFFFFFFu, key[j]);
          const int leader = __ffs(grp) - 1;
          uint32_t off = 0;
          if (key[j] != NOKEY && lane == leader) off = atomicAdd(&S.kcnt[key[j]], (uint32_t)__popc(grp));
          off = __shfl_sync(0xFFFFFFFFu, off, leader);
          if (key[j] != NOKEY) {
            rank[j] = off + __popc(grp & lanemask_lt());
            atomicMax(&S.khh[key[j]], hu);
          }
        }
      }
      __syncthreads();
      // ---- lower key bits among the upper-bit winners; one global claim per child
#pragma unroll
      for (int j = 0; j < RITEMS; j++) {
        if (key[j] != NOKEY && (uint32_t)(khi_[j] >> 32) == S.khh[key[j]])
          atomicMax(&S.khl[key[j]], (uint32_t)khi_[j]);
      }
      const uint32_t ne = nw * K;
      for (uint32_t e = tid; e < ne; e += RB) {
        const uint32_t c = S.kcnt[e];
        if (c) S.kbase[e] = atomicAdd(&cursor[(size_t)(lo + e / K) * K + e % K], c);
      }
      __syncthreads();
      // ---- lowest index among the farthest; write the survivors
#pragma unroll
      for (int j = 0; j < RITEMS; j++) {
        if (key[j] == NOKEY) continue;
        const uint32_t i = j * RB + tid;
        const uint32_t kk = key[j];
        const uint32_t qi = INPUT ? (tile_begin + i) : si[i];
        if ((uint32_t)(khi_[j] >> 32) == S.khh[kk] && (uint32_t)khi_[j] == S.khl[kk]) atomicMin(&S.kidx[kk], qi);
        const uint32_t s = kk % K;
        const size_t dst = (size_t)s * rcap + S.kbase[kk] + rank[j];
        outx[dst] = sx[i];
        outy[dst] = sx[RTILE + i];
        if (DIM == 3) outz[dst] = sx[2 * RTILE + i];
        outi[dst] = qi;
      }
      __syncthreads();
      // ---- close, carry or merge every child of the tile
      for (uint32_t e = tid; e < ne; e += RB) {
        const unsigned long long hk = S.kcnt[e] ? (((unsigned long long)S.khh[e] << 32) | S.khl[e]) : 0ull;
        if (R1) {
          // round 1's children are interleaved over the whole input: fold
          // into the block's running maxima, merged once per block below
          if (hk > S.racc_hi[e] || (hk == S.racc_hi[e] && hk && S.kidx[e] < S.racc_idx[e])) {
            S.racc_hi[e] = hk;
            S.racc_idx[e] = S.kidx[e];
          }
        } else {
          close_child(e / K, e % K, hk, S.kidx[e]);
        }
        S.kcnt[e] = 0;
        S.khh[e] = 0u;
        S.khl[e] = 0u;
        S.kidx[e] = 0xFFFFFFFFu;
      }
      if (tid == 0 && !(has_next && S.wstart[b][nw] > tile_end)) S.pend_seg[pout] = NOKEY;
    } else {
      // ---- slow path: per-point global claims (windows wider than WMAX)
      if (tid < K && S.pend_seg[pin] != NOKEY) {
        const unsigned long long ph = S.pend_hi[pin][tid];
        if (ph) atomic_max_key(&ws.slot_key[(size_t)S.pend_seg[pin] * K + tid], ph, S.pend_idx[pin][tid]);
      }
      if (tid == 0) S.pend_seg[pout] = NOKEY;
#pragma unroll
      for (int j = 0; j < RITEMS; j++) {
        if (key[j] == NOKEY) continue;
        const uint32_t i = j * RB + tid;
        const uint32_t s = key[j] % K;
        const size_t e = (size_t)(lo + key[j] / K) * K + s;
        const uint32_t pos = atomicAdd(&cursor[e], 1u);
        const uint32_t qi = si[i];
        atomic_max_key(&ws.slot_key[e], khi_[j], qi);
        const size_t dst = (size_t)s * rcap + pos;
        outx[dst] = sx[i];
        outy[dst] = sx[RTILE + i];
        if (DIM == 3) outz[dst] = sx[2 * RTILE + i];
        outi[dst] = qi;
      }
    }
    __syncthreads();  // stage b, window b and the child arrays are free
  }

  if (R1 && tid < nseg * K && S.racc_hi[tid])
    atomic_max_key(&ws.slot_key[tid], S.racc_hi[tid], S.racc_idx[tid]);
}

}  // namespace sh
