// K1/K2: the fused Quickhull round kernel.
//
// One persistent launch processes one round over all segments at once.
// Per 2048-point tile (dynamic tile ids, so look-back never waits on an
// unscheduled block):
//   1. coalesced loads of the live records (SoA, K input streams);
//   2. segment lookup (K3 leaves the first segment of every tile in
//      tile_seg; the tile's segment starts are staged in shared memory);
//   3. classification against the segment's simplex -- discard test and
//      child state in the reference's exact fp64 operation order -- and the
//      child's next-round distance (the next round's farthest-point key);
//   4. stable K-way split: warp ballots + a block scan give each survivor
//      its rank inside its stream; survivors are staged in shared memory in
//      output order (stream-major, so every child is one contiguous run);
//   5. reduce-by-key over the staged child keys (warp segmented scans):
//      farthest point (max distance, lowest original index) and count per
//      child run.  Runs that start and end inside the tile are final and
//      written straight to `slots`; the tile's first/last run per stream go
//      into the look-back payload;
//   6. decoupled look-back: stream offsets + the open run carried across
//      tiles (sa_combine), so a child split across tiles is closed by the
//      first tile that sees its end -- no global atomics at all;
//   7. coalesced copy-out of the staged records to the output streams.
#pragma once

#include "sh_common.cuh"

namespace sh {

struct Frag {
  uint32_t has, single, fkey, lkey;
  RunVal fval, lval;
};

template <int DIM>
struct RoundSmem {
  // dynamic part: staging (union with the segment-start window)
  static constexpr size_t bytes() {
    return (size_t)TILE * (8 * DIM + 8 + 4 + 4) + 64;
  }
};

struct RoundShared {
  uint32_t tile;
  uint32_t nwin;
  uint32_t seg_lo;
  uint32_t last;
  uint32_t off[5];
  uint32_t wcnt[ITEMS * WARPS * 3];
  uint32_t fkey[3], lkey[3];
  RunVal first[3], last_run[3];
  uint32_t cnt[4], prefix[4], incl[4];
  int stop[4];
  // per-block pending run per stream, carried across the block's tiles
  uint32_t pend_key[3];
  uint32_t pend_valid[3];
  RunVal pend[3];
  Frag frag[WARPS];
};

__device__ __forceinline__ RunVal rv_ident() {
  RunVal r;
  r.hi = 0;
  r.idx = 0xFFFFFFFFu;
  r.cnt = 0;
  return r;
}

template <int K>
__device__ __forceinline__ void flush_run(RoundShared& sh_, const Workspace& ws, uint32_t nseg,
                                          uint32_t key, RunVal v) {
  uint32_t s = (K == 1) ? 0 : key / nseg;
  bool done = false;
  if (key == sh_.fkey[s]) {
    sh_.first[s] = v;
    done = true;
  }
  if (key == sh_.lkey[s]) {
    sh_.last_run[s] = v;
    done = true;
  }
  if (!done) {
    // a run bounded by other keys inside the tile is the whole child
    Key128 k;
    k.hi = v.hi;
    k.lo = v.idx;
    st_cg(&ws.slot_key[key], k);
    ws.slot_cnt[key] = v.cnt;
  }
}

// Boundary runs of a child that spans tiles: merged with atomics.
__device__ __forceinline__ void flush_atomic(const Workspace& ws, uint32_t key, RunVal v) {
  atomicAdd(&ws.slot_cnt[key], v.cnt);
  atomic_max_key(&ws.slot_key[key], v.hi, v.idx);
}

// Thread 0: fold a boundary run into the block's pending run of its stream.
__device__ __forceinline__ void pend_push(RoundShared& sh_, const Workspace& ws, int s, uint32_t key,
                                          RunVal v) {
  if (sh_.pend_valid[s] && sh_.pend_key[s] == key) {
    sh_.pend[s] = rv_merge(sh_.pend[s], v);
  } else {
    if (sh_.pend_valid[s]) flush_atomic(ws, sh_.pend_key[s], sh_.pend[s]);
    sh_.pend_key[s] = key;
    sh_.pend[s] = v;
    sh_.pend_valid[s] = 1;
  }
}

// Classification of one point against its segment (2D), quickhull.py:230-266.
// Returns state in {-1 (discard), 0, 1} and the child's next-round distance.
__device__ __forceinline__ int classify2(const Seg2& g, double qx, double qy, uint32_t qi,
                                         double* dnext) {
  if (qi == g.fidx) return -1;  // keep[far_seg] = False (:244)
  // point_in_triangle(ea, eb, fq, q, eps), geometry.py:150-156
  double d = cross2(g.ax, g.ay, g.bx, g.by, qx, qy);
  // classify_two_edges(a, far, b, q), geometry.py:178-189
  double c0 = cross2(g.ax, g.ay, g.fx, g.fy, qx, qy);  // cross2(a, far, q)
  double c1 = cross2(g.fx, g.fy, g.bx, g.by, qx, qy);  // cross2(far, b, q)
  // cross2(b, far, q) == -c1 and cross2(far, a, q) == -c0 bit-exactly (the
  // symmetric form negates every term exactly, test_geometry.py:35-38)
  bool inside = (d >= g.nt_ab) & (-c1 >= g.nt_bf) & (-c0 >= g.nt_fa);
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
  double d = plane_dist(g.n, g.a, qx, qy, qz);
  double D0 = plane_dist(g.N[0], g.a, qx, qy, qz);
  double D1 = plane_dist(g.N[1], g.b, qx, qy, qz);
  double D2 = plane_dist(g.N[2], g.c, qx, qy, qz);
  bool inside = (d >= g.nt_base) & (D0 <= g.thr[0]) & (D1 <= g.thr[1]) & (D2 <= g.thr[2]);
  if (inside) return -1;
  // first argmax of D_j / |N_j| (np.argmax over the stacked quotients)
  double q0 = div_(D0, g.nrm[0]), q1 = div_(D1, g.nrm[1]), q2 = div_(D2, g.nrm[2]);
  int state = 0;
  double qb = q0, db = D0;
  if (q1 > qb) { state = 1; qb = q1; db = D1; }
  if (q2 > qb) { state = 2; db = D2; }
  *dnext = db;
  return state;
}

template <int DIM, bool FIRST>
__global__ void __launch_bounds__(BLOCK, 2) k_round(Workspace ws) {
  constexpr int K = DIM;
  DevState* st = ws.st;
  extern __shared__ __align__(16) unsigned char dsm[];
  __shared__ RoundShared sh_;
  double* sx = reinterpret_cast<double*>(dsm);
  double* sy = sx + TILE;
  double* sz = sy + TILE;  // DIM == 3 only
  uint64_t* shi = reinterpret_cast<uint64_t*>(sx + DIM * TILE);
  uint32_t* sidx = reinterpret_cast<uint32_t*>(shi + TILE);
  uint32_t* skey = sidx + TILE;
  uint32_t* swin = reinterpret_cast<uint32_t*>(dsm);  // union with staging

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // ---- launch parameters (own block only, see RoundParams)
  uint32_t n_live, nseg, cur, tag;
  uint32_t cum1 = 0, cum2 = 0;
  if (FIRST) {
    if (st->first_active != 1) return;
    n_live = st->n;
    nseg = 1;
    cur = 0;
    tag = st->rp.tag;
  } else {
    if (!st->rp.active) return;
    n_live = st->rp.n_live;
    nseg = st->rp.nseg;
    cur = st->rp.cur;
    tag = st->rp.tag;
    cum1 = st->rp.cnt_in[0];
    cum2 = cum1 + st->rp.cnt_in[1];
  }
  const uint32_t num_tiles = (n_live + TILE - 1) / TILE;
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
  const uint32_t* tile_seg = ws.tile_seg[cur];
  const Seg2* seg2 = reinterpret_cast<const Seg2*>(ws.seg[cur]);
  const Seg3* seg3 = reinterpret_cast<const Seg3*>(ws.seg[cur]);

  // first-split constants
  double f_pa[3], f_pb[3], f_nrm[3], f_thr = 0;
  uint32_t f_imin = 0, f_imax = 0, f_ifar = 0xFFFFFFFFu;
  if (FIRST) {
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
  double dmax_local = 0.0;
  const uint32_t tag16 = (tag % 65535u) + 1u;
  if (tid < 3) sh_.pend_valid[tid] = 0;

  while (true) {
    if (tid == 0) sh_.tile = atomicAdd(&st->ctr_round, 1u);
    __syncthreads();
    const uint32_t tile = sh_.tile;
    if (tile >= num_tiles) break;
    const uint32_t base = tile * TILE;
    const bool last_tile = (tile == num_tiles - 1);

    // ---- segment window
    if (!FIRST) {
      if (tid == 0) {
        uint32_t lo = tile_seg[tile];
        uint32_t hi = (tile + 1 < num_tiles) ? tile_seg[tile + 1] : nseg - 1;
        sh_.seg_lo = lo;
        sh_.nwin = hi - lo + 1;
      }
      __syncthreads();
      for (uint32_t i = tid; i < sh_.nwin; i += BLOCK) swin[i] = segstart[sh_.seg_lo + i];
      __syncthreads();
    }
    const uint32_t seg_lo = FIRST ? 0u : sh_.seg_lo;
    const uint32_t nwin = FIRST ? 1u : sh_.nwin;

    // ---- load + classify (striped: item j of thread t is base + j*BLOCK + t)
    double qx[ITEMS], qy[ITEMS], qz[ITEMS];
    uint32_t qi[ITEMS], qseg[ITEMS];
    int qs[ITEMS];
    uint64_t qhi[ITEMS];
#pragma unroll
    for (int j = 0; j < ITEMS; j++) {
      uint32_t p = base + j * BLOCK + tid;
      qs[j] = -1;
      qseg[j] = 0;
      qi[j] = p;
      qx[j] = qy[j] = qz[j] = 0.0;
      if (p < n_live) {
        if (FIRST) {
          qx[j] = ld_coord(st->px, st->stride, p);
          qy[j] = ld_coord(st->py, st->stride, p);
          if (DIM == 3) qz[j] = ld_coord(st->pz, st->stride, p);
        } else {
          uint32_t s = (p >= cum1) + (K == 3 ? (p >= cum2) : 0);
          uint32_t o = p - (s == 0 ? 0u : (s == 1 ? cum1 : cum2));
          size_t a = (size_t)s * rcap + o;
          qx[j] = __ldcs(inx + a);
          qy[j] = __ldcs(iny + a);
          if (DIM == 3) qz[j] = __ldcs(inz + a);
          qi[j] = __ldcs(ini + a);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < ITEMS; j++) {
      uint32_t p = base + j * BLOCK + tid;
      if (p >= n_live) continue;
      double dn = 0.0;
      int s = -1;
      if (FIRST) {
        if (DIM == 2) {
          if (p != f_imin && p != f_imax) {
            // quickhull.py:202-211
            double d = cross2(f_pa[0], f_pa[1], f_pb[0], f_pb[1], qx[j], qy[j]);
            if (fabs(d) > f_thr) {
              s = d < 0 ? 1 : 0;
              dn = s ? -d : d;  // cross2(pmax, pmin, q) == -d exactly
            }
          }
        } else {
          if (p != f_imin && p != f_imax && p != f_ifar) {
            // quickhull.py:348-353
            double d = plane_dist(f_nrm, f_pa, qx[j], qy[j], qz[j]);
            dmax_local = fmax(dmax_local, fabs(d));
            s = d < f_thr ? 1 : 0;
            dn = s ? -d : d;  // face (pa, pc, pb) has normal -n exactly
          }
        }
      } else {
        // segment: largest w with swin[w] <= p
        uint32_t lo = 0, hi = nwin - 1;
        while (lo < hi) {
          uint32_t mid = (lo + hi + 1) >> 1;
          if (swin[mid] <= p) lo = mid;
          else hi = mid - 1;
        }
        uint32_t sg = seg_lo + lo;
        qseg[j] = sg;
        if (DIM == 2) s = classify2(seg2[sg], qx[j], qy[j], qi[j], &dn);
        else s = classify3(seg3[sg], qx[j], qy[j], qz[j], qi[j], &dn);
      }
      qs[j] = s;
      qhi[j] = ordered_bits(dn);
    }

    // ---- stable K-way split: ranks inside the tile
    uint32_t lrank[ITEMS];
#pragma unroll
    for (int j = 0; j < ITEMS; j++) {
      lrank[j] = 0;
#pragma unroll
      for (int s = 0; s < K; s++) {
        uint32_t m = __ballot_sync(0xFFFFFFFFu, qs[j] == s);
        if (qs[j] == s) lrank[j] = __popc(m & lanemask_lt());
        if (lane == 0) sh_.wcnt[(j * WARPS + warp) * 3 + s] = __popc(m);
      }
    }
    __syncthreads();
    if (warp == 0) {
      uint32_t tot_prev = 0;
#pragma unroll
      for (int s = 0; s < K; s++) {
        uint32_t a = sh_.wcnt[(2 * lane) * 3 + s];
        uint32_t b = sh_.wcnt[(2 * lane + 1) * 3 + s];
        uint32_t v = a + b;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          uint32_t o = __shfl_up_sync(0xFFFFFFFFu, v, off);
          if (lane >= off) v += o;
        }
        uint32_t ex = v - a - b;
        sh_.wcnt[(2 * lane) * 3 + s] = ex;
        sh_.wcnt[(2 * lane + 1) * 3 + s] = ex + a;
        uint32_t tot = __shfl_sync(0xFFFFFFFFu, v, 31);
        if (lane == 0) sh_.off[s] = tot_prev;
        tot_prev += tot;
      }
      if (lane == 0) sh_.off[K] = tot_prev;
    }
    __syncthreads();

    // ---- stage survivors in output order (the window is no longer needed)
    const uint32_t N = sh_.off[K];
#pragma unroll
    for (int j = 0; j < ITEMS; j++) {
      int s = qs[j];
      if (s < 0) continue;
      uint32_t pos = sh_.off[s] + sh_.wcnt[(j * WARPS + warp) * 3 + s] + lrank[j];
      sx[pos] = qx[j];
      sy[pos] = qy[j];
      if (DIM == 3) sz[pos] = qz[j];
      sidx[pos] = qi[j];
      shi[pos] = qhi[j];
      skey[pos] = (uint32_t)s * nseg + qseg[j];
    }
    __syncthreads();
    if (tid < K) {
      uint32_t a = sh_.off[tid], b = sh_.off[tid + 1];
      sh_.fkey[tid] = (b > a) ? skey[a] : 0xFFFFFFFFu;
      sh_.lkey[tid] = (b > a) ? skey[b - 1] : 0xFFFFFFFFu;
      sh_.first[tid] = rv_ident();
      sh_.last_run[tid] = rv_ident();
    }
    __syncthreads();

    // ---- reduce-by-key over staged child keys (per warp, 32 at a time)
    {
      uint32_t chunk = (((N + WARPS - 1) / WARPS) + 31u) & ~31u;
      uint32_t w0 = min(N, warp * chunk), w1 = min(N, w0 + chunk);
      Frag fr;
      fr.has = (w1 > w0);
      fr.single = 1;
      fr.fkey = fr.lkey = 0;
      fr.fval = fr.lval = rv_ident();
      bool first_open = true, carry_valid = false;
      uint32_t carry_key = 0;
      RunVal carry = rv_ident();
      for (uint32_t cb = w0; cb < w1; cb += 32) {
        uint32_t e = cb + lane;
        bool valid = e < w1;
        uint32_t key = valid ? skey[e] : 0xFFFFFFFFu;
        RunVal v = rv_ident();
        if (valid) {
          v.hi = shi[e];
          v.idx = sidx[e];
          v.cnt = 1;
        }
        uint32_t prevk = __shfl_up_sync(0xFFFFFFFFu, key, 1);
        uint32_t nextk = __shfl_down_sync(0xFFFFFFFFu, key, 1);
        bool head = (lane == 0) || (key != prevk);
        RunVal val = v;
        bool f = head;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          RunVal ov = shfl_up_t(val, off);
          bool of = __shfl_up_sync(0xFFFFFFFFu, f, off);
          if (lane >= off) {
            if (!f) val = rv_merge(ov, val);
            f = f || of;
          }
        }
        int lastl = (int)min(31u, w1 - 1 - cb);
        bool tail = valid && (lane == lastl || nextk != key);
        uint32_t tail_mask = __ballot_sync(0xFFFFFFFFu, tail);
        int first_tail = __ffs(tail_mask) - 1;
        uint32_t k0 = __shfl_sync(0xFFFFFFFFu, key, 0);
        // the chunk's first run continues the carry?
        bool cont = carry_valid && carry_key == k0;
        bool closeA = carry_valid && !cont;
        if (tail && lane == first_tail && cont) val = rv_merge(carry, val);
        uint32_t closeB = __ballot_sync(0xFFFFFFFFu, tail && lane != lastl);
        if (first_open) {
          if (closeA) {
            fr.fkey = carry_key;
            fr.fval = carry;
            first_open = false;
          } else if (closeB) {
            int fl = __ffs(closeB) - 1;
            fr.fkey = __shfl_sync(0xFFFFFFFFu, key, fl);
            fr.fval = shfl_t(val, fl);
            closeB &= closeB - 1;  // that run is recorded, not flushed
            first_open = false;
          }
        } else if (closeA) {
          if (lane == 0) flush_run<K>(sh_, ws, nseg, carry_key, carry);
        }
        if ((closeB >> lane) & 1u) flush_run<K>(sh_, ws, nseg, key, val);
        carry_key = __shfl_sync(0xFFFFFFFFu, key, lastl);
        carry = shfl_t(val, lastl);
        carry_valid = true;
      }
      if (fr.has) {
        fr.lkey = carry_key;
        fr.lval = carry;
        if (first_open) {
          fr.single = 1;
          fr.fkey = carry_key;
          fr.fval = carry;
        } else {
          fr.single = 0;
        }
      }
      if (lane == 0) sh_.frag[warp] = fr;
    }
    __syncthreads();
    if (tid == 0) {
      Frag A = sh_.frag[0];
      for (int w = 1; w < WARPS; w++) {
        Frag F = sh_.frag[w];
        if (!F.has) continue;
        if (!A.has) {
          A = F;
          continue;
        }
        if (A.lkey == F.fkey) {
          RunVal m = rv_merge(A.lval, F.fval);
          if (A.single && F.single) {
            A.fval = m;
            A.lval = m;
          } else if (A.single) {
            A.fval = m;
            A.lkey = F.lkey;
            A.lval = F.lval;
            A.single = 0;
          } else if (F.single) {
            A.lval = m;
          } else {
            flush_run<K>(sh_, ws, nseg, A.lkey, m);
            A.lkey = F.lkey;
            A.lval = F.lval;
          }
        } else {
          if (!A.single) flush_run<K>(sh_, ws, nseg, A.lkey, A.lval);
          if (!F.single) flush_run<K>(sh_, ws, nseg, F.fkey, F.fval);
          A.lkey = F.lkey;
          A.lval = F.lval;
          A.single = 0;
        }
      }
      if (A.has) {
        flush_run<K>(sh_, ws, nseg, A.fkey, A.fval);
        if (!A.single) flush_run<K>(sh_, ws, nseg, A.lkey, A.lval);
      }
    }
    __syncthreads();

    // ---- stream offsets: count-only decoupled look-back (whole block)
    if (tid < K) sh_.cnt[tid] = sh_.off[tid + 1] - sh_.off[tid];
    __syncthreads();
    if (tile > 0) {
      if (tid == 0) lb_publish<K>(ws.lb_round, tile, tag16, LB_AGG, sh_.cnt);
      lb_lookback<K>(ws.lb_round, tile, tag16, sh_.prefix, sh_.stop);
    } else if (tid < K) {
      sh_.prefix[tid] = 0;
    }
    __syncthreads();
    if (tid == 0) {
#pragma unroll
      for (int s = 0; s < K; s++) sh_.incl[s] = sh_.prefix[s] + sh_.cnt[s];
      lb_publish<K>(ws.lb_round, tile, tag16, LB_INC, sh_.incl);
      // tile-boundary runs of children that may span tiles: merge into the
      // block's pending run (children are contiguous, so consecutive tiles
      // of a long child keep hitting the same pending run)
#pragma unroll
      for (int s = 0; s < K; s++) {
        if (sh_.cnt[s] == 0) continue;
        pend_push(sh_, ws, s, sh_.fkey[s], sh_.first[s]);
        if (sh_.lkey[s] != sh_.fkey[s]) pend_push(sh_, ws, s, sh_.lkey[s], sh_.last_run[s]);
      }
      // ---- finalise the launch
      if (last_tile) {
        uint32_t tot = 0;
        BookParams bp;
        bp.active = 1;
        bp.root = FIRST ? 1u : 0u;
        bp.nseg_parent = nseg;
        for (int s = 0; s < 4; s++) bp.cnt_out[s] = (s < K) ? sh_.incl[s] : 0u;
        for (int s = 0; s < K; s++) tot += sh_.incl[s];
        bp.n_out = tot;
        bp.cur = cur;
        bp.h = FIRST ? st->h_final : st->rp.h;
        bp.round = FIRST ? 0u : st->rp.round + 1;
        bp.tag = tag + 1;
        if (!FIRST) {
          uint32_t r = st->rp.round;
          if (r < MAX_TRACE) {
            st->tr_live[r] = n_live;
            st->tr_kept[r] = tot;
            st->tr_nseg[r] = nseg;
          }
          st->rp.active = 0;
        }
        st->bp = bp;
        st->seq = tag + 1;
        st->ctr_book = 0;
      }
    }
    __syncthreads();

    // ---- copy-out (coalesced per stream)
    for (uint32_t e = tid; e < N; e += BLOCK) {
      uint32_t s = (e >= sh_.off[1]) + (K == 3 ? (e >= sh_.off[2]) : 0);
      size_t dst = (size_t)s * rcap + sh_.prefix[s] + (e - sh_.off[s]);
      outx[dst] = sx[e];
      outy[dst] = sy[e];
      if (DIM == 3) outz[dst] = sz[e];
      outi[dst] = sidx[e];
    }
    __syncthreads();
  }
  if (tid == 0) {
    for (int s = 0; s < K; s++)
      if (sh_.pend_valid[s]) flush_atomic(ws, sh_.pend_key[s], sh_.pend[s]);
  }
  if (FIRST && DIM == 3) {
    // coplanarity check input: max |d| of the first split (quickhull.py:349)
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) dmax_local = fmax(dmax_local, __shfl_xor_sync(0xFFFFFFFFu, dmax_local, m));
    if (lane == 0 && dmax_local > 0.0)
      atomicMax((unsigned long long*)&st->dmax_bits, (unsigned long long)__double_as_longlong(dmax_local));
  }
}

}  // namespace sh
