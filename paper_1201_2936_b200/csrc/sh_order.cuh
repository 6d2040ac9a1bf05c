// Callers of the hull path: the CCW boundary order
// of a 2D hull and the gift-wrapping check of the CLI's `verify` command.
//
// order_hull_2d (reference quickhull.py:449-461): angles around the
// centroid, stable sort, rotation to the lexicographically smallest vertex.
//   k_ord_sum   centroid (fp64 sums, last block divides)
//   k_ord_keys  order-preserving bits of atan2(y - my, x - mx), index values
//   (cub::DeviceRadixSort::SortPairs, stable)
//   k_ord_roll  position of the lexicographic minimum, rotated permutation
// For a strictly convex vertex set no two vertices share an angle from an
// interior point, so the order equals the reference's whatever the last bits
// of the centroid.
//
// Gift wrapping (hull2_giftwrap, reference seghull/oracle module lines 20-52): from the
// current vertex, the next one is the candidate every other point lies
// left of; among collinear candidates (within eps * |cand - cur|) the
// farthest.  The replacement rule is not associative (ties within eps), so
// the result of the reference's sequential scan is reproduced in two tiers:
// k_gw_step reduces the rule over all points in tree order (winner w),
// k_gw_check proves that w dominates every other point (then the scan ends
// at w's first copy in any order), and k_gw_commit replays the scan exactly
// in one block when it does not.  The walk state stays on the device; the
// host polls the done flag between batches of steps.
#pragma once

#include "sh_common.cuh"

namespace sh {

__global__ void __launch_bounds__(BLOCK) k_ord_sum(const double* x, const double* y, uint32_t h, double* acc,
                                                   uint32_t* counter, double* mean) {
  double sx = 0.0, sy = 0.0;
  for (uint32_t i = blockIdx.x * BLOCK + threadIdx.x; i < h; i += gridDim.x * BLOCK) {
    sx += x[i];
    sy += y[i];
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    sx += __shfl_xor_sync(0xFFFFFFFFu, sx, o);
    sy += __shfl_xor_sync(0xFFFFFFFFu, sy, o);
  }
  __shared__ double s[2][WARPS];
  __shared__ bool last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    s[0][warp] = sx;
    s[1][warp] = sy;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < WARPS; w++) {
      a += s[0][w];
      b += s[1][w];
    }
    acc[2 * blockIdx.x] = a;
    acc[2 * blockIdx.x + 1] = b;
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last || threadIdx.x != 0) return;
  __threadfence();
  double a = 0.0, b = 0.0;
  for (uint32_t k = 0; k < gridDim.x; k++) {
    a += __ldcg(&acc[2 * k]);
    b += __ldcg(&acc[2 * k + 1]);
  }
  mean[0] = a / (double)h;
  mean[1] = b / (double)h;
  *counter = 0;
}

__global__ void __launch_bounds__(BLOCK) k_ord_keys(const double* x, const double* y, uint32_t h, const double* mean,
                                                    unsigned long long* keys, uint32_t* vals) {
  const double mx = mean[0], my = mean[1];
  for (uint32_t i = blockIdx.x * BLOCK + threadIdx.x; i < h; i += gridDim.x * BLOCK) {
    keys[i] = ordered_bits(atan2(sub(y[i], my), sub(x[i], mx)));
    vals[i] = i;
  }
}

// one block: the sorted position of the lexicographic minimum (x, y, then
// position, as _lex_extreme), then the rotated permutation
__global__ void __launch_bounds__(1024) k_ord_roll(const double* x, const double* y, uint32_t h, const uint32_t* sorted,
                                                   int64_t* out) {
  __shared__ double s_x[32], s_y[32];
  __shared__ uint32_t s_p[32];
  __shared__ uint32_t s_start;
  double bx = INFINITY, by = INFINITY;
  uint32_t bp = 0xFFFFFFFFu;
  for (uint32_t j = threadIdx.x; j < h; j += blockDim.x) {
    const uint32_t i = sorted[j];
    const double xi = x[i], yi = y[i];
    if (xi < bx || (xi == bx && (yi < by || (yi == by && j < bp)))) {
      bx = xi;
      by = yi;
      bp = j;
    }
  }
  auto better = [](double x1, double y1, uint32_t p1, double x0, double y0, uint32_t p0) {
    return x1 < x0 || (x1 == x0 && (y1 < y0 || (y1 == y0 && p1 < p0)));
  };
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const double ox = __shfl_xor_sync(0xFFFFFFFFu, bx, o), oy = __shfl_xor_sync(0xFFFFFFFFu, by, o);
    const uint32_t op = __shfl_xor_sync(0xFFFFFFFFu, bp, o);
    if (better(ox, oy, op, bx, by, bp)) {
      bx = ox;
      by = oy;
      bp = op;
    }
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    s_x[warp] = bx;
    s_y[warp] = by;
    s_p[warp] = bp;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); w++)
      if (better(s_x[w], s_y[w], s_p[w], bx, by, bp)) {
        bx = s_x[w];
        by = s_y[w];
        bp = s_p[w];
      }
    s_start = bp;
  }
  __syncthreads();
  const uint32_t start = s_start;
  for (uint32_t j = threadIdx.x; j < h; j += blockDim.x) {
    uint32_t k = j + start;
    if (k >= h) k -= h;
    out[j] = (int64_t)sorted[k];
  }
}

// ------------------------------------------------------------ gift wrap
struct GwBest {
  double dx, dy;  // candidate - cur
  uint32_t idx;
  uint32_t pad;
};

// does q (relative to cur) replace cand in hull2_giftwrap's scan?
__device__ __forceinline__ bool gw_beats(double qx, double qy, const GwBest& c, double eps) {
  if (c.idx == 0xFFFFFFFFu) return true;
  const double cross = sub(mul(c.dx, qy), mul(c.dy, qx));
  const double limit = mul(eps, glibc_hypot(c.dx, c.dy));
  if (cross < -limit) return true;  // strictly right of cur -> cand
  if (cross <= limit) return add(mul(qx, qx), mul(qy, qy)) > add(mul(c.dx, c.dx), mul(c.dy, c.dy));  // farthest
  return false;
}

// walk state on the device: cur vertex, tree winner w, hull count, done flag
// (1 = closed, 2 = output capacity exceeded).  The host queues batches of
// steps without synchronising; steps after the walk closes return at once.
struct GwState {
  uint32_t cur, start;
  int64_t h;
  uint32_t done, counter;
  uint32_t w, wmin;  // tree winner, lowest index with w's coordinates
  uint32_t tie, pad;
};

__device__ __forceinline__ void gw_merge(GwBest& a, const GwBest& o, double eps) {
  if (o.idx == 0xFFFFFFFFu) return;
  if (gw_beats(o.dx, o.dy, a, eps)) a = o;
}

__device__ __forceinline__ void gw_warp_reduce(GwBest& b, double eps) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    GwBest t;
    t.dx = __shfl_xor_sync(0xFFFFFFFFu, b.dx, o);
    t.dy = __shfl_xor_sync(0xFFFFFFFFu, b.dy, o);
    t.idx = __shfl_xor_sync(0xFFFFFFFFu, b.idx, o);
    t.pad = 0;
    gw_merge(b, t, eps);
  }
}

// step 1: a winner w by tree reduction of the replacement rule
__global__ void __launch_bounds__(BLOCK) k_gw_step(const double* x, const double* y, uint32_t n, double eps,
                                                   GwState* st, GwBest* parts) {
  if (*(volatile uint32_t*)&st->done) return;
  const uint32_t cur = st->cur;
  const double cx = x[cur], cy = y[cur];
  GwBest b;
  b.idx = 0xFFFFFFFFu;
  b.dx = b.dy = 0.0;
  b.pad = 0;
  for (uint32_t i = blockIdx.x * BLOCK + threadIdx.x; i < n; i += gridDim.x * BLOCK) {
    const double qx = sub(x[i], cx), qy = sub(y[i], cy);
    if (qx == 0.0 && qy == 0.0) continue;  // q == cur
    if (gw_beats(qx, qy, b, eps)) {
      b.dx = qx;
      b.dy = qy;
      b.idx = i;
    }
  }
  gw_warp_reduce(b, eps);
  __shared__ GwBest s[WARPS];
  __shared__ bool last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) s[warp] = b;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < WARPS; w++) gw_merge(s[0], s[w], eps);
    parts[blockIdx.x] = s[0];
    __threadfence();
    last = atomicAdd(&st->counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  b.idx = 0xFFFFFFFFu;
  b.dx = b.dy = 0.0;
  for (uint32_t k = threadIdx.x; k < gridDim.x; k += BLOCK) {
    GwBest o;
    o.dx = __ldcg(&parts[k].dx);
    o.dy = __ldcg(&parts[k].dy);
    o.idx = __ldcg(&parts[k].idx);
    o.pad = 0;
    gw_merge(b, o, eps);
  }
  gw_warp_reduce(b, eps);
  __syncthreads();  // s[] reuse
  if (lane == 0) s[warp] = b;
  __syncthreads();
  if (threadIdx.x != 0) return;
  GwBest r = s[0];
  for (int w = 1; w < WARPS; w++) gw_merge(r, s[w], eps);
  st->counter = 0;
  st->w = r.idx;
  st->wmin = r.idx;
  st->tie = 0;
}

// step 2: does w dominate every other point (w replaces it, it never
// replaces w)?  Then the sequential scan ends at w's first occurrence
// whatever the order: once the scan meets a copy of w no other point
// displaces it, and before that every point is displaced by it.
// Otherwise flag a tie for the exact sequential scan of step 3.
__global__ void __launch_bounds__(BLOCK) k_gw_check(const double* x, const double* y, uint32_t n, double eps,
                                                    GwState* st) {
  if (*(volatile uint32_t*)&st->done) return;
  const uint32_t cur = st->cur, w = st->w;
  if (w == 0xFFFFFFFFu) return;
  const double cx = x[cur], cy = y[cur];
  GwBest bw;
  bw.dx = sub(x[w], cx);
  bw.dy = sub(y[w], cy);
  bw.idx = w;
  bw.pad = 0;
  const double xw = x[w], yw = y[w];
  bool tie = false;
  uint32_t wmin = 0xFFFFFFFFu;
  for (uint32_t i = blockIdx.x * BLOCK + threadIdx.x; i < n; i += gridDim.x * BLOCK) {
    const double xi = x[i], yi = y[i];
    const double qx = sub(xi, cx), qy = sub(yi, cy);
    if (qx == 0.0 && qy == 0.0) continue;
    if (xi == xw && yi == yw) {
      wmin = min(wmin, i);
      continue;
    }
    GwBest bq;
    bq.dx = qx;
    bq.dy = qy;
    bq.idx = i;
    bq.pad = 0;
    if (!gw_beats(bw.dx, bw.dy, bq, eps) || gw_beats(qx, qy, bw, eps)) tie = true;
  }
  wmin = __reduce_min_sync(0xFFFFFFFFu, wmin);
  tie = __any_sync(0xFFFFFFFFu, tie);
  if ((threadIdx.x & 31) == 0) {
    if (wmin < w) atomicMin(&st->wmin, wmin);
    if (tie) st->tie = 1;
  }
}

// step 3 (one block): commit the next vertex.  On a tie, replay the
// reference's scan exactly: with the candidate fixed, test a tile of points
// in parallel, jump to the first one that replaces it, continue after it.
__global__ void __launch_bounds__(1024) k_gw_commit(const double* x, const double* y, uint32_t n, double eps,
                                                    GwState* st, int64_t* out, int64_t cap) {
  if (*(volatile uint32_t*)&st->done) return;
  __shared__ uint32_t s_first;
  __shared__ uint32_t s_r;
  const uint32_t cur = st->cur, start = st->start;
  if (threadIdx.x == 0) s_r = st->w == 0xFFFFFFFFu ? 0xFFFFFFFFu : st->wmin;
  if (*(volatile uint32_t*)&st->tie) {
    const double cx = x[cur], cy = y[cur];
    GwBest c;
    c.idx = 0xFFFFFFFFu;
    c.dx = c.dy = 0.0;
    c.pad = 0;
    for (uint32_t base = 0; base < n; base += blockDim.x) {
      const uint32_t i = base + threadIdx.x;
      const bool valid = i < n;
      const double qx = valid ? sub(x[i], cx) : 0.0, qy = valid ? sub(y[i], cy) : 0.0;
      const bool live = valid && !(qx == 0.0 && qy == 0.0);
      uint32_t after = 0;  // positions <= after in this tile are done
      bool first_pass = true;
      for (;;) {
        const bool hit = live && (first_pass || i > after) && gw_beats(qx, qy, c, eps);
        if (threadIdx.x == 0) s_first = 0xFFFFFFFFu;
        __syncthreads();
        if (hit) atomicMin(&s_first, i);
        __syncthreads();
        const uint32_t f = s_first;
        __syncthreads();
        if (f == 0xFFFFFFFFu) break;
        c.idx = f;
        c.dx = sub(x[f], cx);
        c.dy = sub(y[f], cy);
        after = f;
        first_pass = false;
      }
    }
    if (threadIdx.x == 0) s_r = c.idx;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const uint32_t r = s_r;
  // the walk closes when the candidate has the start's coordinates
  // (`cand == start` on tuples), whichever copy it is
  if (r == 0xFFFFFFFFu || (x[r] == x[start] && y[r] == y[start])) {
    st->done = 1;
  } else if (st->h >= cap) {
    st->done = 2;
  } else {
    out[st->h++] = r;
    st->cur = r;
  }
}

}  // namespace sh
