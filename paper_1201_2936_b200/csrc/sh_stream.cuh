// K2S: the streaming Quickhull round kernel (round 1 fused with the first
// split, and every round whose segments are long).
//
// Reference: one round of quickhull_2d / quickhull_3d
// (/root/reference/pkg/src/seghull/quickhull.py:229-266 / :372-437): discard
// the points inside the round's triangle / tetrahedron, classify the rest to
// a child edge / face, regroup them child by child (flag_permute + compact +
// scatter, primitives.py:91-176) and find every child's farthest point
// (_farthest_per_segment, quickhull.py:93-100).  Round 1 also applies the
// first split (quickhull.py:200-222 / :346-364) on the fly, so the split's
// survivors are never written.
//
// One launch does the whole round in one read of the live points and one
// write of the survivors.  Per CTA: one producer warp and NW consumer warps.
//   * The producer walks the CTA's contiguous range of T-point tiles and
//     loads each into a ring of S shared-memory stages with 1D bulk copies
//     (cp.async.bulk, SASS UBLKCP) that complete on the stage's mbarrier.  A
//     tile of live records spans at most two segments ("parts"; each part is
//     one contiguous run of its stream, copied from its 16-byte aligned-down
//     start); the parts' segment tables come with the same transaction.
//     Tiles that span more segments, or inputs that are not unit-stride,
//     fall back to per-point loads.
//   * Consumers classify their IT points per tile from shared memory in the
//     reference's fp64 operation order (cls2 / cls3).  Each survivor gets a
//     child key (part, state); per-thread counts are packed 4 bits per
//     child, one warp scan over 16-bit fields gives every survivor its
//     place, and the survivors are staged child by child in the tile's own
//     stage (in place: the points are in registers by then).
//   * One lane per child claims the tile's output range with one atomicAdd
//     on the child's cursor; the claim is consumed one tile later, so its
//     latency hides behind a whole tile of work: tile j is written out
//     (coalesced) while tile j+1 is processed, then its stage is released
//     to the producer.
//   * Farthest points: every warp keeps the running farthest key (distance
//     bits, lowest original index among ties) of each child of its window in
//     shared memory; a point is a candidate only if its distance reaches the
//     running maximum of its child, and only then does the warp reduce (REDUX)
//     the candidates.  Running keys are merged into the child slots with a
//     128-bit CAS when the window moves on and at the end.
#pragma once

#include <type_traits>

#include "sh_common.cuh"
#include "sh_tma.cuh"

namespace sh {

constexpr int SRC_INPUT = 0;  // round 1: the caller's points + first split
constexpr int SRC_REC = 1;    // rounds >= 2: the live records of the previous round

#ifndef SH_S2_NW
#define SH_S2_NW 7
#endif
#ifndef SH_S2_IT
#define SH_S2_IT 8
#endif
#ifndef SH_S2_S
#define SH_S2_S 3
#endif
#ifndef SH_S2_MINB
#define SH_S2_MINB 2
#endif
#ifndef SH_S3_MINB
#define SH_S3_MINB 2
#endif
#ifndef SH_S3_NW
#define SH_S3_NW 7
#endif
#ifndef SH_S3_IT
#define SH_S3_IT 5
#endif
#ifndef SH_S3_S
#define SH_S3_S 3
#endif

template <int DIM>
struct StreamCfg {
  static constexpr int NW = DIM == 2 ? SH_S2_NW : SH_S3_NW;  // consumer warps
  static constexpr int IT = DIM == 2 ? SH_S2_IT : SH_S3_IT;  // points per consumer thread per tile
  static constexpr int S = DIM == 2 ? SH_S2_S : SH_S3_S;     // pipeline stages
  static constexpr int NT = NW * 32;
  static constexpr int T = NT * IT;                            // points per tile
  static constexpr int NTHREADS = NT + 32;                     // + producer warp
  static constexpr int MINB = DIM == 2 ? SH_S2_MINB : SH_S3_MINB;  // CTAs per SM
  // per array and stage: a tile's records (two parts, each copied from its
  // aligned-down start: + 4 doubles / + 6 uint32) or its survivors with
  // every child run padded to 4 records (+ 3 per child, 6 children in 3D)
  static constexpr int CAPD = T + 32;                          // doubles per array per stage
  static constexpr int CAPI = T + 32;                          // uint32 per stage
  static constexpr size_t STAGE = (size_t)DIM * CAPD * 8 + (size_t)CAPI * 4;
  static constexpr size_t SMEM = (size_t)S * STAGE;
  static_assert(IT <= 15, "per-thread child counts are packed 4 bits each");
  static_assert(T < 65536, "tile positions are packed 16 bits each");
  static_assert(STAGE % 16 == 0, "stages are 16-byte aligned");
};

constexpr uint32_t SM_TMA = 0, SM_LDG = 1, SM_END = 2;

struct StageDesc {
  uint32_t base;    // first position of the tile (input index / logical live position)
  uint32_t count;   // points in the tile
  uint32_t mode;    // SM_TMA, SM_LDG (per-point loads of the input), SM_END (no more tiles)
  uint32_t bound;   // tile-local index where part 1 starts (0xFFFFFFFF: one part)
  uint32_t lo;      // segment of part 0 (records)
  uint32_t sh[2][4];  // stage index of tile point i of part p in array a = i + sh[p][a] (x, y, z, idx)
};

// 2D classification of a live point against its segment (quickhull.py:
// 236-266, geometry.py:150-156 and :178-189): c0 = cross2(a, far, q),
// c1 = cross2(far, b, q) in the reference's operation order; inside the
// triangle iff -c1 >= (-eps)|bf| and -c0 >= (-eps)|fa| (cross2(b, far, q) ==
// -c1 bit-exactly; the (a, b) clause holds for every live point, see
// classify2 in sh_round.cuh).  The far point itself gives c0 = c1 = 0 exactly
// and is dropped by the same test, so no index check is needed.
__device__ __forceinline__ int cls2(const Seg2& g, double qx, double qy, double* dn) {
  const double c0 = add(add(mul(g.ax, sub(g.fy, qy)), mul(g.fx, sub(qy, g.ay))), mul(qx, g.d_af));
  const double c1 = add(add(mul(g.fx, sub(g.by, qy)), mul(g.bx, sub(qy, g.fy))), mul(qx, g.d_fb));
  const bool inside = (-c1 >= g.nt_bf) & (-c0 >= g.nt_fa);
  const bool p0 = c0 > 0.0, p1 = c1 > 0.0;
  const bool st1 = (p0 != p1) ? p1 : (c1 > c0);
  *dn = st1 ? c1 : c0;
  return inside ? -1 : (st1 ? 1 : 0);
}

// 3D (quickhull.py:372-437, geometry.py:163-175, :192-208): the three side
// faces' plane distances, the tetrahedron test, and the first argmax of the
// rounded quotients D_j / |N_j|.
__device__ __forceinline__ int cls3(const Seg3& g, double qx, double qy, double qz, uint32_t qi, double* dn) {
  const double D0 = plane_dist(g.N[0], g.a, qx, qy, qz);
  const double D1 = plane_dist(g.N[1], g.b, qx, qy, qz);
  const double D2 = plane_dist(g.N[2], g.c, qx, qy, qz);
  const bool inside = (D0 <= g.thr[0]) & (D1 <= g.thr[1]) & (D2 <= g.thr[2]);
  int state = 0;
  double db = D0, nb = g.nrm[0];
  if (quotient_gt_warp(D1, g.nrm[1], db, nb)) {
    state = 1;
    db = D1;
    nb = g.nrm[1];
  }
  if (quotient_gt_warp(D2, g.nrm[2], db, nb)) {
    state = 2;
    db = D2;
  }
  *dn = db;
  return (inside | (g.flat != 0) | (qi == g.fidx)) ? -1 : state;
}

template <int DIM, int SRC>
__global__ void __launch_bounds__(StreamCfg<DIM>::NTHREADS, StreamCfg<DIM>::MINB) k_stream(Workspace ws) {
  using C = StreamCfg<DIM>;
  using SegT = typename std::conditional<DIM == 2, Seg2, Seg3>::type;
  constexpr int K = DIM, NK = 2 * K, NW = C::NW, NT = C::NT, IT = C::IT, T = C::T, S = C::S;
  constexpr uint32_t NONE = 0xFFFFFFFFu;
  extern __shared__ __align__(16) unsigned char dsm[];  // the stages (16-byte aligned bulk copies)
  __shared__ __align__(8) uint64_t s_full[S];
  __shared__ __align__(8) uint64_t s_ready[S];  // staged tile + its claims are in place (NW + 1 arrivals)
  __shared__ StageDesc s_desc[S];
  __shared__ __align__(16) SegT s_tab[S][2];
  __shared__ uint32_t s_wtot[2][NW][K];    // per warp: inclusive per-child counts, 16-bit fields
  __shared__ uint32_t s_coff[S][NK + 1];  // per stage: stage offset of each child's run (multiples of 4), total
  __shared__ long long s_gdst[S][NK];      // per stage: global element of the first record of child k's run
  __shared__ unsigned long long s_bh[NW][NK];
  __shared__ uint32_t s_thr[NW][8];        // per warp: running farthest key of child k, upper 32 bits (key 7: never)
  __shared__ uint32_t s_bi[NW][NK];
  __shared__ uint32_t s_rlo[NW];           // per warp: segment of part 0 of the running keys

  DevState* st = ws.st;
  const RoundParams rp = st->rp;
  if (SRC == SRC_INPUT) {
    if (!rp.active || rp.root || rp.round != 1) return;
  } else {
    if (!ws.peeled || !rp.active || rp.root || !long_round(rp, st)) return;
  }
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (blockIdx.x == 0 && tid == 0) {
    st->ctr_book = 0;  // K3's tile counter
    st->arrive_book = 0;
    st->book_small = (uint32_t)K * rp.nseg <= BOOK_SMALL ? 1u : 0u;
  }
  const uint32_t cur = rp.cur, nseg = rp.nseg;
  const uint32_t npos = SRC == SRC_INPUT ? st->n : rp.n_live;
  const uint32_t ntiles = (npos + T - 1) / T;
  const uint32_t t0 = (uint32_t)(((uint64_t)ntiles * blockIdx.x) / gridDim.x);
  const uint32_t t1 = (uint32_t)(((uint64_t)ntiles * (blockIdx.x + 1)) / gridDim.x);
  if (t0 >= t1) return;
  const uint64_t rcap = ws.rcap;
  const SegT* segtab = reinterpret_cast<const SegT*>(ws.seg[cur]);
  // round 1: side 0 of the first split is segment 0 when it has survivors;
  // side 1 is segment 1 then, else 0 (the root children's counts are still
  // in cursor[0])
  const uint32_t side1_seg = SRC == SRC_INPUT ? (ws.cursor[0][0] ? 1u : 0u) : 0u;
  if (SRC == SRC_INPUT) {
    // the two round-1 tables stay in s_tab[0][side] for the whole launch
    constexpr uint32_t W = sizeof(SegT) / 8;
    const unsigned long long* src = reinterpret_cast<const unsigned long long*>(segtab);
    unsigned long long* dst = reinterpret_cast<unsigned long long*>(&s_tab[0][0]);
    for (uint32_t k = tid; k < 2 * W; k += blockDim.x) dst[k] = src[(k < W ? 0u : side1_seg) * W + k % W];
  }
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < S; s++) {
      mbar_init(&s_full[s], 1);
      mbar_init(&s_ready[s], NW + 1);
    }
    fence_mbar_init();
  }
  for (int e = tid; e < NW * NK; e += blockDim.x) {
    (&s_bh[0][0])[e] = 0ull;
    (&s_bi[0][0])[e] = 0xFFFFFFFFu;
  }
  if (tid < NW) s_rlo[tid] = NONE;
  for (int e = tid; e < NW * 8; e += blockDim.x) (&s_thr[0][0])[e] = (e % 8) < NK ? 0u : 0xFFFFFFFFu;
  __syncthreads();

  auto stage_ptr = [&](uint32_t s) { return dsm + (size_t)s * C::STAGE; };
  const double* px = st->px;
  const double* py = st->py;
  const double* pz = st->pz;
  const int64_t pstride = st->stride;
  const uint32_t n_in = st->n;
  const double* inx = ws.rx[cur];
  const double* iny = ws.ry[cur];
  const double* inz = ws.rz[cur];
  const uint32_t* ini = ws.ri[cur];
  const uint32_t* segstart = ws.segstart[cur];
  const uint64_t* seg_phys = ws.seg_phys[cur];

  // ------------------------------------------------------------ producer
  if (warp == NW) {
    if (lane != 0) return;
    const uint64_t pol = policy_evict_first();
    uint32_t w = 0;
    if (SRC == SRC_REC) {  // segment containing the CTA's first position
      uint32_t lo = 0, hi = nseg - 1, q = t0 * T;
      while (lo < hi) {
        const uint32_t mid = (lo + hi + 1) >> 1;
        if (__ldg(&segstart[mid]) <= q) lo = mid;
        else hi = mid - 1;
      }
      w = lo;
    }
    double* outp[3] = {ws.rx[cur ^ 1u], ws.ry[cur ^ 1u], ws.rz[cur ^ 1u]};
    uint32_t* outi = ws.ri[cur ^ 1u];
    // write out the staged survivors of the CTA's u-th tile (its stage's
    // child runs are 4-record aligned in shared memory and in the output
    // streams) and wait until the stage has been read
    auto flush = [&](uint32_t u) {
      const uint32_t su = u % S;
      mbar_wait(&s_ready[su], (u / S) & 1u);
      const unsigned char* sp = stage_ptr(su);
      bool any = false;
#ifdef SH_DIAG_NOFLUSH
      return;
#endif
#pragma unroll 1
      for (int k = 0; k < NK; k++) {
        const uint32_t c0 = s_coff[su][k], n = s_coff[su][k + 1] - c0;
        if (!n) continue;
        const long long g = s_gdst[su][k];
#pragma unroll
        for (int a = 0; a < DIM; a++)
          bulk_s2g(outp[a] + g, sp + ((size_t)a * C::CAPD + c0) * 8, n * 8);
        bulk_s2g(outi + g, sp + (size_t)DIM * C::CAPD * 8 + (size_t)c0 * 4, n * 4);
        any = true;
      }
      if (any) {
        bulk_commit();
#ifndef SH_DIAG_NOWAIT
        bulk_wait_read<0>();
#endif
      }
    };
    // the CTA's positions [t0*T, t1*T): fixed T-point tiles of the input;
    // record tiles are cut at segment starts so that none spans more than
    // two segments (every cut is a multiple of 4: segments start 4-aligned)
    const uint32_t pend_all = min(t1 * T, npos);
    uint32_t pos = t0 * T, j = 0;
    for (; pos < pend_all; j++) {
      const uint32_t s = j % S;
      if (j >= (uint32_t)S) flush(j - S);
      StageDesc d;
      d.base = pos;
      d.count = min((uint32_t)T, pend_all - pos);
      d.bound = NONE;
      d.lo = 0;
#pragma unroll
      for (int p = 0; p < 2; p++)
#pragma unroll
        for (int a = 0; a < 4; a++) d.sh[p][a] = 0;
      unsigned char* sp = stage_ptr(s);
      if (SRC == SRC_INPUT) {
        const double* P[3] = {px, py, pz};
        bool tma = pstride == 1;
        uint32_t bytes = 0;
#pragma unroll
        for (int a = 0; a < DIM; a++) {
          const double* src = P[a] + d.base;
          const uint32_t sh = (uint32_t)((reinterpret_cast<uintptr_t>(src) & 15) >> 3);
          const uint32_t nel = (sh + d.count + 1) & ~1u;
          if (src - sh < P[a] || src - sh + nel > P[a] + n_in) tma = false;
          d.sh[0][a] = sh;
          bytes += nel * 8;
        }
        d.mode = tma ? SM_TMA : SM_LDG;
        s_desc[s] = d;
        if (tma) {
          mbar_arrive_expect_tx(&s_full[s], bytes);
#pragma unroll
          for (int a = 0; a < DIM; a++) {
            const uint32_t sh = d.sh[0][a];
            bulk_g2s(sp + (size_t)a * C::CAPD * 8, P[a] + d.base - sh, ((sh + d.count + 1) & ~1u) * 8, &s_full[s],
                     pol);
          }
        } else {
          mbar_arrive(&s_full[s]);
        }
      } else {
        while (__ldg(&segstart[w + 1]) <= d.base) w++;  // segstart[nseg] = n_live
        const uint32_t s1 = __ldg(&segstart[w + 1]);
        uint32_t np = 1;
        if (s1 < d.base + d.count) {
          np = 2;
          if (w + 2 <= nseg) {
            const uint32_t s2 = __ldg(&segstart[w + 2]);
            if (s2 < d.base + d.count) d.count = s2 - d.base;  // cut before a third segment
          }
          d.bound = s1 - d.base;
        }
        d.lo = w;
        d.mode = SM_TMA;
        // part p: one contiguous run of records, copied from its 16-byte
        // aligned-down start; its points land at stage index i + sh[p][a]
        uint32_t len[2], sd[2], si[2], nd[2], ni[2], od[2], oi[2];
        uint64_t phys[2];
        len[0] = np == 2 ? d.bound : d.count;
        len[1] = d.count - len[0];
        uint32_t dd = 0, di = 0, bytes = np * (uint32_t)sizeof(SegT);
        for (uint32_t p = 0; p < np; p++) {
          const uint32_t ls = p ? s1 : d.base;
          phys[p] = __ldg(&seg_phys[w + p]) + (ls - __ldg(&segstart[w + p]));
          sd[p] = (uint32_t)(phys[p] & 1u);
          si[p] = (uint32_t)(phys[p] & 3u);
          nd[p] = (sd[p] + len[p] + 1) & ~1u;
          ni[p] = (si[p] + len[p] + 3) & ~3u;
          od[p] = dd;
          oi[p] = di;
          const uint32_t off = p ? d.bound : 0u;
          d.sh[p][0] = d.sh[p][1] = d.sh[p][2] = od[p] + sd[p] - off;
          d.sh[p][3] = oi[p] + si[p] - off;
          dd += nd[p];
          di += ni[p];
          bytes += DIM * nd[p] * 8 + ni[p] * 4;
        }
        s_desc[s] = d;
        mbar_arrive_expect_tx(&s_full[s], bytes);
        bulk_g2s(&s_tab[s][0], segtab + w, np * (uint32_t)sizeof(SegT), &s_full[s], policy_evict_last());
        const double* A[3] = {inx, iny, inz};
        for (uint32_t p = 0; p < np; p++) {
#pragma unroll
          for (int a = 0; a < DIM; a++)
            bulk_g2s(sp + ((size_t)a * C::CAPD + od[p]) * 8, A[a] + phys[p] - sd[p], nd[p] * 8, &s_full[s], pol);
          bulk_g2s(sp + (size_t)DIM * C::CAPD * 8 + (size_t)oi[p] * 4, ini + phys[p] - si[p], ni[p] * 4, &s_full[s],
                   pol);
        }
      }
      pos = d.base + d.count;
    }
    {  // end of the CTA's tiles: an empty descriptor
      const uint32_t s = j % S;
      if (j >= (uint32_t)S) flush(j - S);
      StageDesc d;
      d.base = pos;
      d.count = 0;
      d.mode = SM_END;
      s_desc[s] = d;
      mbar_arrive(&s_full[s]);
      j++;
    }
    for (uint32_t u = j > (uint32_t)S ? j - S : 0u; u + 1 < j; u++) flush(u);  // (the last descriptor is the end)
    bulk_wait<0>();
    return;
  }

  // ------------------------------------------------------------ consumers
  Key128* slot_key = ws.slot_key;
  uint32_t* cursor = ws.cursor[cur];
  // first-split constants (round 1)
  double f_pa[3], f_pb[3], f_nrm[3];
#pragma unroll
  for (int k = 0; k < 3; k++) {
    f_pa[k] = st->pa[k];
    f_pb[k] = st->pb[k];
    f_nrm[k] = st->nrm[k];
  }
  const double f_thr = st->thr_line;
  const uint32_t f_imin = st->imin, f_imax = st->imax, f_ifar = DIM == 3 ? st->ifar : NONE;
  auto seg_of_part = [&](uint32_t lo, uint32_t p) -> uint32_t {
    return SRC == SRC_INPUT ? (p ? side1_seg : 0u) : lo + p;
  };
  // merge this warp's running keys of parts [p0, p1) into the child slots (lane 0)
  auto merge_running = [&](uint32_t p0, uint32_t p1) {
    const uint32_t lo = s_rlo[warp];
    for (uint32_t p = p0; p < p1; p++) {
      const uint32_t seg = seg_of_part(lo, p);
      if (SRC == SRC_REC && seg >= nseg) continue;
#pragma unroll
      for (int s = 0; s < K; s++) {
        const uint32_t k = p * K + s;
        if (s_bh[warp][k]) atomic_max_key(&slot_key[(size_t)seg * K + s], s_bh[warp][k], s_bi[warp][k]);
      }
    }
  };

  // classification of point i of a tile (the reference's fp64 order); returns
  // the child key (part * K + state) or 7 (dropped) and the child's distance
  auto classify_pt = [&](const StageDesc& d, const SegT* tab, uint32_t i, double x, double y, double z, uint32_t qi,
                         double* dn, auto one_tag) -> uint32_t {
    constexpr bool ONE = decltype(one_tag)::value;  // the tile is one segment: one table for every point
    bool keep = i < d.count;
    uint32_t part = (!ONE && i >= d.bound) ? 1u : 0u;
    if (SRC == SRC_INPUT) {
      if (DIM == 2) {
        // quickhull.py:202-211: off the extreme line by more than eps
        // (pmin, pmax themselves give d = 0 exactly)
        const double dd = cross2(f_pa[0], f_pa[1], f_pb[0], f_pb[1], x, y);
        keep &= fabs(dd) > f_thr;
        part = dd < 0.0 ? 1u : 0u;
      } else {
        // quickhull.py:348-353
        const double dd = plane_dist(f_nrm, f_pa, x, y, z);
        part = dd < f_thr ? 1u : 0u;
      }
    }
    int sst;
    if constexpr (DIM == 2) sst = cls2(tab[part], x, y, dn);
    else sst = cls3(tab[part], x, y, z, qi, dn);
    keep &= sst >= 0;
    return keep ? part * K + (uint32_t)sst : 7u;
  };

  uint32_t pend = 0;                 // warp 0, lane k < NK: the previous tile's claim of child k
  uint32_t dead = 0;                 // warp 0 lane 0: DEAD padding records claimed by this CTA
  uint32_t j = 0;
  for (;; j++) {
    const uint32_t s = j % S, par = j & 1u;
    mbar_wait(&s_full[s], (j / S) & 1u);
    const StageDesc d = s_desc[s];
    if (d.mode == SM_END) break;
    unsigned char* sp = stage_ptr(s);
    double* sxa = reinterpret_cast<double*>(sp);
    double* sya = sxa + C::CAPD;
    double* sza = sxa + 2 * C::CAPD;
    uint32_t* sia = reinterpret_cast<uint32_t*>(sxa + DIM * C::CAPD);
    const SegT* tab = &s_tab[SRC == SRC_INPUT ? 0 : s][0];

    // per point: coordinates, original index (records), key | local rank << 4
    uint32_t kr[IT], I[IT];
    double X[IT], Y[IT], Z[IT];
    uint32_t nib = 0;  // per-thread counts, 4 bits per child (nibble 7: dropped points)
#pragma unroll
    for (int it = 0; it < IT; it++) kr[it] = 7u;
    {
      if (SRC == SRC_REC && d.lo != s_rlo[warp]) {
        // the window moved: merge the running keys of segments left behind
        if (lane == 0) {
          const uint32_t rlo = s_rlo[warp];
          if (rlo != NONE && d.lo == rlo + 1) {
            merge_running(0, 1);
#pragma unroll
            for (int s2 = 0; s2 < K; s2++) {
              s_bh[warp][s2] = s_bh[warp][K + s2];
              s_bi[warp][s2] = s_bi[warp][K + s2];
              s_thr[warp][s2] = s_thr[warp][K + s2];
              s_bh[warp][K + s2] = 0ull;
              s_bi[warp][K + s2] = 0xFFFFFFFFu;
              s_thr[warp][K + s2] = 0u;
            }
          } else {
            if (rlo != NONE) merge_running(0, 2);
#pragma unroll
            for (int k = 0; k < NK; k++) {
              s_bh[warp][k] = 0ull;
              s_bi[warp][k] = 0xFFFFFFFFu;
              s_thr[warp][k] = 0u;
            }
          }
          s_rlo[warp] = d.lo;
        }
        __syncwarp();
      }
      const uint32_t h0x = d.sh[0][0], h0y = d.sh[0][1], h0z = d.sh[0][2], h0i = d.sh[0][3];
      const uint32_t h1x = d.sh[1][0], h1i = d.sh[1][3];
      uint32_t candmask = 0;
      // classification of the tile's points (TMA: from the stage; LDG: per-
      // point loads of the input, the fallback for non-unit strides)
      auto classify = [&](auto tma_tag, auto one_tag) {
        constexpr bool TMA = decltype(tma_tag)::value;
#pragma unroll
        for (int it = 0; it < IT; it++) {
          const uint32_t i = it * NT + tid;
          if (TMA) {
            if (SRC == SRC_INPUT) {  // one part; every coordinate array has its own shift
              X[it] = sxa[i + h0x];
              Y[it] = sya[i + h0y];
              if (DIM == 3) Z[it] = sza[i + h0z];
              I[it] = d.base + i;
            } else {                 // records: one shift per part for the coordinates
              const bool p = i >= d.bound;
              const uint32_t ix = i + (p ? h1x : h0x);
              X[it] = sxa[ix];
              Y[it] = sya[ix];
              if (DIM == 3) Z[it] = sza[ix];
              I[it] = sia[i + (p ? h1i : h0i)];
            }
          } else {
            const uint32_t q = min(d.base + i, n_in - 1);
            X[it] = ld_coord(px, pstride, q);
            Y[it] = ld_coord(py, pstride, q);
            if (DIM == 3) Z[it] = ld_coord(pz, pstride, q);
            I[it] = d.base + i;
          }
          double dn;
          uint32_t key = classify_pt(d, tab, i, X[it], Y[it], DIM == 3 ? Z[it] : 0.0, I[it], &dn, one_tag);
          if (SRC == SRC_INPUT && DIM == 3) {
            // the extreme points and the third corner are removed before the
            // split (quickhull.py:342)
            if (I[it] == f_imin || I[it] == f_imax || I[it] == f_ifar) key = 7u;
          }
          if (SRC == SRC_REC && I[it] == DEAD) key = 7u;  // padding record
          // dn > 0 for every survivor: the raw bits order like ordered_bits
          const uint32_t hu = (uint32_t)__double2hiint(dn) | 0x80000000u;
          candmask |= (hu >= s_thr[warp][key]) ? (1u << it) : 0u;  // reaches the child's running maximum
          const uint32_t shf = 4u * key;
          kr[it] = key | (((nib >> shf) & 15u) << 4);
          nib += 1u << shf;
        }
      };
      if (SRC == SRC_REC) {
        if (d.bound == NONE) classify(std::true_type{}, std::true_type{});
        else classify(std::true_type{}, std::false_type{});
      } else if (d.mode == SM_TMA) {
        classify(std::true_type{}, std::false_type{});
      } else {
        classify(std::false_type{}, std::false_type{});
      }
      // ---- farthest-point candidates (rare after the first tiles): the
      // candidates are re-classified for their distances, then reduced per
      // child with REDUX (max distance bits, lowest original index)
      if (__any_sync(0xFFFFFFFFu, candmask != 0)) {
        uint32_t cu[IT], cl[IT];
#pragma unroll
        for (int it = 0; it < IT; it++) {
          cu[it] = 0;
          cl[it] = 0;
          if ((candmask >> it) & 1u) {
            double dn;
            classify_pt(d, tab, it * NT + tid, X[it], Y[it], DIM == 3 ? Z[it] : 0.0, I[it], &dn, std::false_type{});
            cu[it] = (uint32_t)__double2hiint(dn) | 0x80000000u;
            cl[it] = (uint32_t)__double2loint(dn);
          }
        }
#pragma unroll 1
        for (int k = 0; k < NK; k++) {
          uint32_t tu = 0, tl = 0, ti = 0xFFFFFFFFu;
#pragma unroll
          for (int it = 0; it < IT; it++) {
            const bool mine = ((candmask >> it) & 1u) && (kr[it] & 7u) == (uint32_t)k;
            const bool better = mine && (cu[it] > tu || (cu[it] == tu && (cl[it] > tl || (cl[it] == tl && I[it] < ti))));
            tu = better ? cu[it] : tu;
            tl = better ? cl[it] : tl;
            ti = better ? I[it] : ti;
          }
          const uint32_t mu = __reduce_max_sync(0xFFFFFFFFu, tu);
          const unsigned long long ch = s_bh[warp][k];
          if (mu == 0u || mu < (uint32_t)(ch >> 32)) continue;  // warp-uniform
          const uint32_t ml = __reduce_max_sync(0xFFFFFFFFu, tu == mu ? tl : 0u);
          const uint32_t mi = __reduce_min_sync(0xFFFFFFFFu, (tu == mu && tl == ml) ? ti : 0xFFFFFFFFu);
          const unsigned long long h = ((unsigned long long)mu << 32) | ml;
          const uint32_t ci = s_bi[warp][k];
          __syncwarp();
          if (lane == 0 && (h > ch || (h == ch && mi < ci))) {
            s_bh[warp][k] = h;
            s_bi[warp][k] = mi;
            s_thr[warp][k] = mu;
          }
          __syncwarp();
        }
      }
    }

    // ---- warp scan of the per-thread counts over 16-bit fields: word c
    // holds children 2c (low) and 2c+1 (high)
    uint32_t incl[K], own[K];
    {
      const uint32_t ev = nib & 0x0F0F0F0Fu, od = (nib >> 4) & 0x0F0F0F0Fu;
#pragma unroll
      for (int c = 0; c < K; c++) {
        own[c] = ((ev >> (8 * c)) & 0xFFu) | (((od >> (8 * c)) & 0xFFu) << 16);
        incl[c] = own[c];
      }
    }
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
#pragma unroll
      for (int c = 0; c < K; c++) {
        const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, incl[c], off);
        if (lane >= off) incl[c] += v;
      }
    }
    if (lane == 31) {
#pragma unroll
      for (int c = 0; c < K; c++) s_wtot[par][warp][c] = incl[c];
    }
    // the previous tile's claims have had a whole tile of work to return:
    // publish them, then the previous tile can be written out (s_ready)
    if (warp == 0 && j > 0) {
      const uint32_t sprev = (j - 1) % S;
      if (lane < NK) s_gdst[sprev][lane] = (long long)((uint32_t)lane % K) * (long long)rcap + (long long)pend;
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_ready[sprev]);
    }
    named_bar(1, NT);  // ---- the one barrier of the tile: per-warp counts, previous claims
    // ---- tile offsets, computed by every warp (no serial section): lane L
    // holds warp L's counts; scan over the warps
    uint32_t coff[NK + 1], pb[K];
    {
      uint32_t v[K], x[K];
#pragma unroll
      for (int c = 0; c < K; c++) {
        v[c] = lane < NW ? s_wtot[par][lane][c] : 0u;
        x[c] = v[c];
      }
#pragma unroll
      for (int off = 1; off < NW; off <<= 1) {
#pragma unroll
        for (int c = 0; c < K; c++) {
          const uint32_t u = __shfl_up_sync(0xFFFFFFFFu, x[c], off);
          if (lane >= off) x[c] += u;
        }
      }
      uint32_t tk[NK];
#pragma unroll
      for (int c = 0; c < K; c++) {
        const uint32_t tot = __shfl_sync(0xFFFFFFFFu, x[c], NW - 1);
        tk[2 * c] = tot & 0xFFFFu;
        tk[2 * c + 1] = tot >> 16;
      }
      // every child's run starts 4-record aligned (DEAD-padded to a multiple
      // of 4: written out by 16-byte bulk copies)
      coff[0] = 0;
#pragma unroll
      for (int k = 0; k < NK; k++) coff[k + 1] = coff[k] + ((tk[k] + 3u) & ~3u);
#pragma unroll
      for (int c = 0; c < K; c++) {
        const uint32_t wex = __shfl_sync(0xFFFFFFFFu, x[c] - v[c], warp);  // this warp's exclusive prefix
        pb[c] = (coff[2 * c] | (coff[2 * c + 1] << 16)) + wex + (incl[c] - own[c]);
      }
      if (warp == 0) {
        if (lane <= NK) {
          uint32_t mc = 0;
#pragma unroll
          for (int k = 0; k <= NK; k++) mc = lane == k ? coff[k] : mc;
          s_coff[s][lane] = mc;
        }
        if (lane < NK) {
          // claim this tile's (padded) output run of child `lane`; the
          // result is consumed one tile later
          uint32_t mt = 0;
#pragma unroll
          for (int k = 0; k < NK; k++) mt = lane == k ? tk[k] : mt;
          const uint32_t pt = (mt + 3u) & ~3u;
          const uint32_t seg = seg_of_part(d.lo, (uint32_t)lane / K);
          pend = pt ? atomicAdd(&cursor[(size_t)seg * K + (uint32_t)lane % K], pt) : 0u;
          dead += pt - mt;
        }
        // DEAD records in the padding slots of the runs
        const uint32_t k = (uint32_t)lane >> 2, r = (uint32_t)lane & 3u;
        uint32_t mt = 0, mc = 0;
#pragma unroll
        for (int kk = 0; kk < NK; kk++) {
          mt = k == (uint32_t)kk ? tk[kk] : mt;
          mc = k == (uint32_t)kk ? coff[kk] : mc;
        }
        if (k < (uint32_t)NK && r < ((4u - (mt & 3u)) & 3u)) sia[mc + mt + r] = DEAD;
      }
    }
    // ---- stage this tile's survivors child by child (in place)
#pragma unroll
    for (int it = 0; it < IT; it++) {
      const uint32_t k = kr[it] & 7u;
      const uint32_t w = K == 2 ? ((k & 2u) ? pb[1] : pb[0]) : (k < 2u ? pb[0] : (k < 4u ? pb[1] : pb[K - 1]));
      // dropped points go to a scratch slot past every staged run (no branch)
      const uint32_t pos = k < (uint32_t)NK ? ((w >> (16 * (k & 1u))) & 0xFFFFu) + (kr[it] >> 4) : C::CAPD - 1;
      sxa[pos] = X[it];
      sya[pos] = Y[it];
      if (DIM == 3) sza[pos] = Z[it];
      sia[pos] = I[it];
    }
    // ---- the staged tile is complete once the claims return (next tile)
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) mbar_arrive(&s_ready[s]);
  }
  // ---- the last tile's claims
  if (warp == 0) {
    const uint32_t sprev = (j - 1) % S;
    if (lane < NK) s_gdst[sprev][lane] = (long long)((uint32_t)lane % K) * (long long)rcap + (long long)pend;
    const uint32_t dsum = __reduce_add_sync(0xFFFFFFFFu, lane < NK ? dead : 0u);
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(&s_ready[sprev]);
      if (dsum) atomicAdd(&st->dead_round, dsum);
    }
  }
  // ---- running farthest keys -> child slots
  if (SRC == SRC_INPUT) {
    // every warp has the same children: reduce over the block first
    if (warp == 0 && lane < NK) {
      unsigned long long h = 0ull;
      uint32_t idx = 0xFFFFFFFFu;
#pragma unroll 1
      for (int w2 = 0; w2 < NW; w2++) {
        const unsigned long long h2 = s_bh[w2][lane];
        const uint32_t i2 = s_bi[w2][lane];
        if (h2 > h || (h2 == h && i2 < idx)) {
          h = h2;
          idx = i2;
        }
      }
      const uint32_t seg = seg_of_part(0, (uint32_t)lane / K);
      if (h) atomic_max_key(&slot_key[(size_t)seg * K + (uint32_t)lane % K], h, idx);
    }
  } else if (lane == 0 && s_rlo[warp] != NONE) {
    merge_running(0, 2);
  }
}

}  // namespace sh
