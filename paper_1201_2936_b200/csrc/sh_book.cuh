// K3: per-segment bookkeeping between rounds.
//
// Input: the child results of the round kernel (child id e = parent*K +
// state: farthest key in slot_key, survivor count = write cursor - parent
// start).  One persistent launch, one thread per child:
//   * occupied children (count > 0) get dense ids by a decoupled look-back
//     scan over (occupied, count, emitted) in parent-major order -- the
//     reference's flat-array segment order -- which also gives every new
//     segment its dense start and every emitted vertex its output position;
//   * the new segment's records stay where the round kernel wrote them:
//     stream s at the parent's start (seg_phys), and its children's write
//     cursors are initialised to its own dense start;
//   * child tables are built once per segment (2D: the child edge and the
//     three glibc-exact hypot thresholds, quickhull.py:268-277 and
//     geometry.py:150-156; 3D: face normal, |n|, flat-segment test
//     quickhull.py:384-389, side faces of the next tetrahedron);
//   * the farthest point of every non-flat child is emitted as a hull vertex
//     (quickhull.py:236-240 / :390-391);
//   * the finalising tile writes the next round's launch parameters and the
//     CUDA-graph WHILE condition (live points remain), so the host never
//     synchronises inside the loop (quickhull.py:225 / :367 become a device
//     flag).
#pragma once

#include "sh_common.cuh"

namespace sh {

struct BookShared {
  uint32_t tile;
  uint32_t wsum[ITEMS3 * WARPS * 4];
  Sum3 agg, prefix;
  int stop[4];
};

template <int DIM>
__global__ void __launch_bounds__(BLOCK, DIM == 2 ? 2 : 1) k_book(Workspace ws) {
  constexpr int K = DIM;
  DevState* st = ws.st;
  __shared__ BookShared sb;
  __shared__ RoundParams s_rp;
  __shared__ uint32_t s_seq;
  __shared__ Sum3 s_carry;
  __shared__ uint32_t s_dead, s_status;  // final by now (the round kernel wrote them)
  // few children (flag written by the round kernel): block 0 does everything
  // in tile order with a running prefix -- no look-back, no arrival protocol
  const bool small = st->book_small != 0;
  if (small && blockIdx.x != 0) return;
  if (threadIdx.x == 0) {
    s_rp = st->rp;
    s_seq = st->seq;
    s_dead = st->dead_round;
    s_status = st->status;
    s_carry = s3_identity();
    if (!small) {
      __threadfence();
      atomicAdd(&st->arrive_book, 1u);  // the finaliser waits for every block's read
    }
    sb.tile = 0xFFFFFFFFu;
  }
  __syncthreads();
  const RoundParams bp = s_rp;
  if (!bp.active) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t nsp = bp.nseg;
  const uint32_t E = K * nsp;
  const uint32_t num_tiles = (E + TILE3 - 1) / TILE3;
  const uint32_t tag = s_seq + 1;
  const uint32_t tag16 = (tag % 65535u) + 1u;
  const double eps = st->eps;
  const uint32_t segcap = st->segcap;
  const int64_t stride = st->stride;
  const uint64_t rcap = ws.rcap;
  const uint32_t in_b = bp.cur, out_b = bp.cur ^ 1u;
  const Seg2* par2 = reinterpret_cast<const Seg2*>(ws.seg[in_b]);
  const Seg3* par3 = reinterpret_cast<const Seg3*>(ws.seg[in_b]);
  const uint32_t* par_start = ws.segstart[in_b];
  const uint32_t* cur_in = ws.cursor[in_b];
  // 4-record aligned segments (spans rounded up, DEAD-padded): always for
  // round 1 (k_stream writes it), for later rounds when k_stream may run them
  const bool pad_next = bp.root || stream_eligible(ws, st, bp, bp.round + 1, K);
  Seg2* ch2 = reinterpret_cast<Seg2*>(ws.seg[out_b]);
  Seg3* ch3 = reinterpret_cast<Seg3*>(ws.seg[out_b]);
  uint32_t* segstart = ws.segstart[out_b];
  uint64_t* seg_phys = ws.seg_phys[out_b];
  uint32_t* cur_out = ws.cursor[out_b];

  while (true) {
    if (tid == 0) sb.tile = small ? sb.tile + 1u : atomicAdd(&st->ctr_book, 1u);
    __syncthreads();
    const uint32_t tile = sb.tile;
    if (tile >= num_tiles) break;
    const uint32_t base = tile * TILE3;
    const bool last_tile = tile == num_tiles - 1;

    RunVal v[ITEMS3];
    // counters: occupied, span (records rounded up to 4: the next round's
    // positions, DEAD-padded), emitted vertex, records (incl. DEAD claims)
    uint32_t cval[ITEMS3][4];
    // 3D child face (needed before the scan for the flat test)
    double fa[ITEMS3][3], fb[ITEMS3][3], fc[ITEMS3][3], fn[ITEMS3][3], fnl[ITEMS3];
    // 2D child edge ends (loaded with the counts: one memory round trip)
    double ea[ITEMS3][2], eb[ITEMS3][2];
#pragma unroll
    for (int j = 0; j < ITEMS3; j++) {
      uint32_t e = base + j * BLOCK + tid;
      v[j].hi = 0;
      v[j].idx = 0;
      v[j].cnt = 0;
      if (e < E) {
        const uint32_t p = e / K, s = e - p * K;
        // count, farthest key and (2D) the parent's edge, all in flight at once
        const uint32_t cin = __ldcg(&cur_in[e]), pst = __ldg(&par_start[p]);
        const Key128 k = ld_cg(&ws.slot_key[e]);
        if (DIM == 2) {
          if (bp.root) {  // quickhull.py:217-222
            ea[j][0] = (s == 0) ? st->pa[0] : st->pb[0];
            ea[j][1] = (s == 0) ? st->pa[1] : st->pb[1];
            eb[j][0] = (s == 0) ? st->pb[0] : st->pa[0];
            eb[j][1] = (s == 0) ? st->pb[1] : st->pa[1];
          } else {  // (a, far) / (far, b), quickhull.py:272-277
            const Seg2& P = par2[p];
            ea[j][0] = (s == 0) ? P.ax : P.fx;
            ea[j][1] = (s == 0) ? P.ay : P.fy;
            eb[j][0] = (s == 0) ? P.fx : P.bx;
            eb[j][1] = (s == 0) ? P.fy : P.by;
          }
        }
        v[j].cnt = cin - pst;
        if (v[j].cnt) {
          v[j].hi = k.hi;
          v[j].idx = (uint32_t)k.lo;
          Key128 z;
          z.hi = 0;
          z.lo = 0;
          st_cg(&ws.slot_key[e], z);  // slots are all-zero between uses
        }
      }
      bool occ = v[j].cnt > 0;
      bool emit = occ;
      if (DIM == 3 && occ) {
        uint32_t p = e / K, s = e - p * K;
        const double *A, *B, *C;
        if (bp.root) {  // quickhull.py:359-364
          A = st->pa;
          B = (s == 0) ? st->pb : st->pc;
          C = (s == 0) ? st->pc : st->pb;
        } else {        // children (a,b,f), (b,c,f), (c,a,f), quickhull.py:419-423
          const Seg3& P = par3[p];
          A = (s == 0) ? P.a : (s == 1 ? P.b : P.c);
          B = (s == 0) ? P.b : (s == 1 ? P.c : P.a);
          C = P.f;
        }
#pragma unroll
        for (int k = 0; k < 3; k++) {
          fa[j][k] = A[k];
          fb[j][k] = B[k];
          fc[j][k] = C[k];
        }
        face_normal(fa[j], fb[j], fc[j], fn[j]);
        fnl[j] = norm3(fn[j]);
        // flat_seg = seg_max <= eps * nlen (quickhull.py:385)
        emit = !(from_ordered_bits(v[j].hi) <= mul(eps, fnl[j]));
      }
      cval[j][0] = occ ? 1u : 0u;
      cval[j][1] = pad_next ? (v[j].cnt + 3u) & ~3u : v[j].cnt;
      cval[j][2] = emit ? 1u : 0u;
      cval[j][3] = v[j].cnt;
    }
    // ---- block exclusive scan (striped order) of the three counters
    uint32_t ex[ITEMS3][4];
#pragma unroll
    for (int j = 0; j < ITEMS3; j++) {
#pragma unroll
      for (int q = 0; q < 4; q++) {
        uint32_t x = cval[j][q];
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          uint32_t o = __shfl_up_sync(0xFFFFFFFFu, x, off);
          if (lane >= off) x += o;
        }
        ex[j][q] = x - cval[j][q];
        if (lane == 31) sb.wsum[(j * WARPS + warp) * 4 + q] = x;
      }
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
      for (int q = 0; q < 4; q++) {
        uint32_t w = sb.wsum[lane * 4 + q];
        uint32_t x = w;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          uint32_t o = __shfl_up_sync(0xFFFFFFFFu, x, off);
          if (lane >= off) x += o;
        }
        sb.wsum[lane * 4 + q] = x - w;
        uint32_t tot = __shfl_sync(0xFFFFFFFFu, x, 31);
        if (lane == 0) sb.agg.v[q] = tot;
      }
    }
    __syncthreads();
    if (small) {
      if (tid < 4) sb.prefix.v[tid] = s_carry.v[tid];
    } else if (tile > 0) {
      if (tid == 0) lb_publish<4>(ws.lb_book, tile, tag16, LB_AGG, sb.agg.v);
      lb_lookback<4>(ws.lb_book, tile, tag16, sb.prefix.v, sb.stop);
    } else if (tid < 4) {
      sb.prefix.v[tid] = 0;
    }
    __syncthreads();
    if (tid == 0) {
      Sum3 inc = s3_combine(sb.prefix, sb.agg);
      if (small) s_carry = inc;
      else lb_publish<4>(ws.lb_book, tile, tag16, LB_INC, inc.v);
    }

    // ---- build child tables, emit vertices
#pragma unroll
    for (int j = 0; j < ITEMS3; j++) {
      if (!cval[j][0]) continue;
      uint32_t e = base + j * BLOCK + tid;
      uint32_t p = e / K, s = e - p * K;
      const uint32_t* wo = &sb.wsum[(j * WARPS + warp) * 4];
      uint32_t c = sb.prefix.v[0] + wo[0] + ex[j][0];
      uint32_t start = sb.prefix.v[1] + wo[1] + ex[j][1];
      uint32_t vpos = sb.prefix.v[2] + wo[2] + ex[j][2];
      uint32_t far = v[j].idx;
      if (cval[j][2]) ws.vout[bp.h + vpos] = far;
      if (c >= segcap) continue;  // overflow: reported by the finalising tile
      // round 1 claims output per tile (padded to 4 records per tile and
      // child): room for that padding before the second side's children
      if (bp.root && c > 0) start += ws.slack;
      if (!bp.root && pad_next) {
        // DEAD records from the last record of the segment to its span
        uint32_t* ri = ws.ri[out_b] + (size_t)s * rcap + __ldg(&par_start[p]);
        for (uint32_t r = v[j].cnt; r < cval[j][1]; r++) ri[r] = DEAD;
      }
      segstart[c] = start;
      seg_phys[c] = (uint64_t)s * rcap + __ldg(&par_start[p]);  // where K2 wrote child (p, s)
#pragma unroll
      for (int q = 0; q < K; q++) cur_out[(size_t)c * K + q] = start;
      double F[3];
      F[0] = ld_coord(st->px, stride, far);
      F[1] = ld_coord(st->py, stride, far);
      F[2] = (DIM == 3) ? ld_coord(st->pz, stride, far) : 0.0;
      if (DIM == 2) {
        const double Ax = ea[j][0], Ay = ea[j][1], Bx = eb[j][0], By = eb[j][1];
        Seg2 g;
        g.ax = Ax; g.ay = Ay; g.bx = Bx; g.by = By; g.fx = F[0]; g.fy = F[1];
        // point_in_triangle(a, b, far): -eps * edge_length(.,.) per edge;
        // the (a, b) clause always holds for live points (classify2), so
        // only the two edges to the new apex are needed
        g.d_af = sub(Ay, F[1]);
        g.d_fb = sub(F[1], By);
        g.nt_bf = mul(-eps, edge_length(Bx, By, F[0], F[1]));
        g.nt_fa = mul(-eps, edge_length(F[0], F[1], Ax, Ay));
        g.fidx = far;
        g.pad = 0;
        ch2[c] = g;
      } else {
        Seg3 g;
#pragma unroll
        for (int k = 0; k < 3; k++) {
          g.a[k] = fa[j][k];
          g.b[k] = fb[j][k];
          g.c[k] = fc[j][k];
          g.n[k] = fn[j][k];
          g.f[k] = F[k];
        }
        g.nt_base = mul(-eps, fnl[j]);  // point_in_tetrahedron base test (geometry.py:172)
        g.fidx = far;
        g.flat = cval[j][2] ? 0u : 1u;
        // side faces (a,b,f), (b,c,f), (c,a,f), geometry.py:166-175
        face_normal(g.a, g.b, F, g.N[0]);
        face_normal(g.b, g.c, F, g.N[1]);
        face_normal(g.c, g.a, F, g.N[2]);
#pragma unroll
        for (int q = 0; q < 3; q++) {
          g.nrm[q] = norm3(g.N[q]);
          g.thr[q] = mul(eps, g.nrm[q]);
        }
        ch3[c] = g;
      }
    }

    __syncthreads();

    // ---- finalise the launch: next round's parameters + loop condition
    if (last_tile && tid == 0) {
      Sum3 T = s3_combine(sb.prefix, sb.agg);
      uint32_t nseg_next = T.v[0], n_next = T.v[1], emitted = T.v[2];
      // live points of the next round: records minus the DEAD padding the
      // round kernel claimed (quickhull.py's compact count)
      const uint32_t n_true_next = T.v[3] - s_dead;
      if (bp.root && nseg_next > 1) n_next += ws.slack;
      uint32_t status = s_status;
      uint32_t round_next = bp.round + 1;  // the round the children belong to
      // every block has read this round's parameters before they change
      if (!small)
        while (*(volatile uint32_t*)&st->arrive_book < gridDim.x) {
        }
      if (bp.root && DIM == 3) {
        // quickhull.py:349-351 -- every point within eps of the first plane
        double dmax = __longlong_as_double((long long)st->dmax_bits);
        if (dmax <= mul(eps, st->nlen)) status = ST_DEGENERATE;
      }
      if (bp.root && DIM == 2 && n_next == 0 && st->n > 2) st->flags |= FL_COLLINEAR;  // :206-209
      if (nseg_next > segcap) {
        status = ST_SEG_OVERFLOW;
        st->seg_needed = nseg_next;
      } else {
        segstart[nseg_next] = n_next;
      }
      if (DIM == 3 && round_next - 1 < MAX_TRACE) st->tr_flat[round_next - 1] = nseg_next - emitted;
      if (!bp.root && bp.round - 1 < MAX_TRACE) {  // loop round bp.round: (live, kept, segments)
        st->tr_live[bp.round - 1] = bp.n_true;
        st->tr_kept[bp.round - 1] = n_true_next;
        st->tr_nseg[bp.round - 1] = bp.nseg;
      }
      uint32_t h_next = bp.h + emitted;
      bool cont = (n_next > 0) && status == ST_OK;
      if (cont && (uint64_t)round_next > (uint64_t)st->n + 1) {  // quickhull.py:227-228
        status = ST_ROUND_GUARD;
        cont = false;
      }
      RoundParams rp;
      rp.active = cont ? 1u : 0u;
      rp.root = 0;
      rp.n_live = n_next;
      rp.nseg = nseg_next;
      rp.cur = out_b;
      rp.h = h_next;
      rp.round = round_next;
      rp.n_true = n_true_next;
      rp.aligned = pad_next ? 1u : 0u;
      rp.pad = 0;
      st->dead_round = 0;
      st->rp = rp;
      st->status = status;
      st->h_final = h_next;
      st->rounds_final = bp.round;
      st->seq = tag;
      st->arrive_book = 0;
      if (ws.use_cond) cudaGraphSetConditional(ws.cond, cont ? 1u : 0u);
    }
    __syncthreads();
  }
}

}  // namespace sh
