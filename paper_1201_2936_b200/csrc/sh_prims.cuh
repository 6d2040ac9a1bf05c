// The framework primitives of the paper (§4.1 flag permute, §4.2 compact)
// and the segmented scans they are built from, as public device ops
// (reference segments.py:201-266,
// primitives.py:91-176).  Not on the hull's hot path (the round kernel fuses
// all of this), but the same API as the reference's so its primitive-level
// tests and callers run on the GPU.
//
// Segmented scan: three passes over 1024-element tiles (per-tile
// segmented aggregates, a one-block carry chain over the tiles, a per-tile
// rescan with the carry), for sum (int64, exact), max and min (int64 or
// fp64).  Backward scans run over mirrored indices; exclusive scans emit the
// identity at each segment's starting boundary.  Results are deterministic:
// sums are integer, max/min are selections, -0.0 is canonicalised to +0.0
// (segments.py:10-13, :197).
#pragma once

#include <type_traits>

#include "sh_common.cuh"

namespace sh {

constexpr int PS_ITEMS = 4;
constexpr int PS_TILE = BLOCK * PS_ITEMS;

enum { PS_SUM = 0, PS_MAX = 1, PS_MIN = 2 };

template <class T>
__device__ __forceinline__ T ps_identity(int op);
template <>
__device__ __forceinline__ long long ps_identity<long long>(int op) {
  return op == PS_SUM ? 0ll : (op == PS_MAX ? (long long)0x8000000000000000ull : 0x7FFFFFFFFFFFFFFFll);
}
template <>
__device__ __forceinline__ double ps_identity<double>(int op) {
  return op == PS_SUM ? 0.0 : (op == PS_MAX ? -INFINITY : INFINITY);
}

template <class T>
__device__ __forceinline__ T ps_op(int op, T a, T b) {
  if (op == PS_SUM) return a + b;
  if (op == PS_MAX) return a > b ? a : b;
  return a < b ? a : b;
}

// Element j of the scan order: forward = i, backward = n-1-i.  A head in
// scan order starts a segment in the scan direction: for backward scans
// that is a segment's last element (the next original element is a head).
struct PsView {
  const void* vals;
  const uint8_t* heads;   // null: one segment
  const int64_t* states;  // optional: value = (states[i] == state); only those i are written
  int64_t state;
  const int64_t* mvals;   // optional: value = keep[i] ? mvals[i] : identity
  const uint8_t* keep;
  const uint8_t* u8;      // optional: value = u8[i] (element 0 counts as 1 when force0)
  int force0;
  int64_t n;
  int backward;
};

__device__ __forceinline__ int64_t ps_src(const PsView& v, int64_t j) {
  return v.backward ? v.n - 1 - j : j;
}
__device__ __forceinline__ bool ps_head(const PsView& v, int64_t j) {
  if (j == 0) return true;
  if (!v.heads) return false;
  if (!v.backward) return v.heads[j] != 0;
  return v.heads[v.n - j] != 0;  // original element n-1-j ends its segment
}
template <class T>
__device__ __forceinline__ T ps_val(const PsView& v, int64_t j, int op) {
  const int64_t i = ps_src(v, j);
  if constexpr (sizeof(T) == 8 && std::is_same<T, long long>::value) {
    if (v.states) return (long long)(v.states[i] == v.state);
    if (v.keep) return v.keep[i] ? (long long)v.mvals[i] : ps_identity<long long>(op);
    if (v.u8) return (v.force0 && i == 0) ? 1ll : (long long)(v.u8[i] != 0);
    return reinterpret_cast<const long long*>(v.vals)[i];
  } else {
    return reinterpret_cast<const double*>(v.vals)[i] + 0.0;  // canonical -0.0
  }
}

// segmented aggregate of a run: (has a head, reduction after its last head)
template <class T>
struct PsAgg {
  uint32_t head;
  T val;
};

template <class T>
__device__ __forceinline__ PsAgg<T> ps_combine(int op, PsAgg<T> a, PsAgg<T> b) {
  PsAgg<T> r;
  r.head = a.head | b.head;
  r.val = b.head ? b.val : ps_op(op, a.val, b.val);
  return r;
}

template <class T>
__device__ PsAgg<T> ps_block_scan(int op, PsAgg<T> mine, PsAgg<T>* s_warp, PsAgg<T>* total) {
  // inclusive block scan of per-thread aggregates (thread order)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  PsAgg<T> x = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    PsAgg<T> y;
    y.head = __shfl_up_sync(0xFFFFFFFFu, x.head, o);
    y.val = __shfl_up_sync(0xFFFFFFFFu, x.val, o);
    if (lane >= o) x = ps_combine(op, y, x);
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  if (threadIdx.x == 0) {
    PsAgg<T> acc;
    acc.head = 0;
    acc.val = ps_identity<T>(op);
    for (int w = 0; w < WARPS; w++) {
      PsAgg<T> t = s_warp[w];
      s_warp[w] = acc;  // exclusive prefix of warp w
      acc = ps_combine(op, acc, t);
    }
    *total = acc;
  }
  __syncthreads();
  return ps_combine(op, s_warp[warp], x);
}

// pass 1: per-tile aggregates
template <class T>
__global__ void __launch_bounds__(BLOCK) k_ps_tiles(PsView v, int op, PsAgg<T>* agg) {
  __shared__ PsAgg<T> s_warp[WARPS];
  __shared__ PsAgg<T> total;
  const int64_t base = (int64_t)blockIdx.x * PS_TILE + (int64_t)threadIdx.x * PS_ITEMS;
  PsAgg<T> a;
  a.head = 0;
  a.val = ps_identity<T>(op);
#pragma unroll
  for (int k = 0; k < PS_ITEMS; k++) {
    const int64_t j = base + k;
    if (j >= v.n) break;
    PsAgg<T> e;
    e.head = ps_head(v, j) ? 1u : 0u;
    e.val = ps_val<T>(v, j, op);
    a = ps_combine(op, a, e);
  }
  ps_block_scan(op, a, s_warp, &total);
  if (threadIdx.x == 0) agg[blockIdx.x] = total;
}

// pass 2: carry-in of every tile (one block, sequential over tiles)
template <class T>
__global__ void k_ps_carry(int op, PsAgg<T>* agg, int64_t ntiles) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  PsAgg<T> acc;
  acc.head = 0;
  acc.val = ps_identity<T>(op);
  for (int64_t t = 0; t < ntiles; t++) {
    PsAgg<T> x = agg[t];
    agg[t] = acc;
    acc = ps_combine(op, acc, x);
  }
}

// pass 3: rescan each tile with its carry; exclusive shifts inside segments
template <class T>
__global__ void __launch_bounds__(BLOCK) k_ps_apply(PsView v, int op, int exclusive, const PsAgg<T>* carry,
                                                    T* out) {
  __shared__ PsAgg<T> s_warp[WARPS];
  __shared__ PsAgg<T> total;
  const int64_t base = (int64_t)blockIdx.x * PS_TILE + (int64_t)threadIdx.x * PS_ITEMS;
  PsAgg<T> e[PS_ITEMS];
  PsAgg<T> a;
  a.head = 0;
  a.val = ps_identity<T>(op);
#pragma unroll
  for (int k = 0; k < PS_ITEMS; k++) {
    const int64_t j = base + k;
    e[k].head = 1;
    e[k].val = ps_identity<T>(op);
    if (j < v.n) {
      e[k].head = ps_head(v, j) ? 1u : 0u;
      e[k].val = ps_val<T>(v, j, op);
    }
    a = ps_combine(op, a, e[k]);
  }
  PsAgg<T> incl = ps_block_scan(op, a, s_warp, &total);
  // exclusive prefix of this thread = (tile carry) + (block-exclusive)
  PsAgg<T> ex;
  {
    // block-exclusive = incl with this thread's own aggregate removed: recompute
    // from the warp prefix by re-scanning is costly; use the identity
    // ex = combine(carry, incl_prev) where incl_prev = shuffle of incl
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    PsAgg<T> prev;
    prev.head = __shfl_up_sync(0xFFFFFFFFu, incl.head, 1);
    prev.val = __shfl_up_sync(0xFFFFFFFFu, incl.val, 1);
    if (lane == 0) prev = s_warp[warp];
    ex = ps_combine(op, carry[blockIdx.x], prev);
  }
  T run = ex.val;
#pragma unroll
  for (int k = 0; k < PS_ITEMS; k++) {
    const int64_t j = base + k;
    if (j >= v.n) break;
    const T before = e[k].head ? ps_identity<T>(op) : run;
    run = e[k].head ? e[k].val : ps_op(op, run, e[k].val);
    const int64_t i = ps_src(v, j);
    if (!v.states || v.states[i] == v.state) out[i] = exclusive ? before : run;
  }
}

template <class T>
static int ps_run(PsView v, int op, int exclusive, T* out, PsAgg<T>* scratch, cudaStream_t s) {
  if (v.n <= 0) return 0;
  const int64_t ntiles = (v.n + PS_TILE - 1) / PS_TILE;
  k_ps_tiles<T><<<(unsigned)ntiles, BLOCK, 0, s>>>(v, op, scratch);
  k_ps_carry<T><<<1, 32, 0, s>>>(op, scratch, ntiles);
  k_ps_apply<T><<<(unsigned)ntiles, BLOCK, 0, s>>>(v, op, exclusive, scratch, out);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : 10;
}

// ------------------------------------------------------------ flag permute
__global__ void __launch_bounds__(BLOCK) k_fp_subone(int64_t* seg, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * BLOCK + threadIdx.x; i < n; i += (int64_t)gridDim.x * BLOCK) seg[i] -= 1;
}

// counts[seg*k + j] += 1 per element; head positions per segment
__global__ void __launch_bounds__(BLOCK) k_fp_counts(const int64_t* f, const int64_t* seg, int64_t n, int64_t k,
                                                     const uint8_t* heads, unsigned long long* counts,
                                                     int64_t* seg_start) {
  for (int64_t i = (int64_t)blockIdx.x * BLOCK + threadIdx.x; i < n; i += (int64_t)gridDim.x * BLOCK) {
    atomicAdd(&counts[seg[i] * k + f[i]], 1ull);
    if (i == 0 || heads[i]) seg_start[seg[i]] = i;
  }
}

// p[i] = head + sum_{j < f[i]} counts[seg][j] + rank_i; new heads at every
// occupied (segment, state) group start (primitives.py:105-116)
__global__ void __launch_bounds__(BLOCK) k_fp_assemble(const int64_t* f, const int64_t* seg, const int64_t* rank,
                                                       int64_t n, int64_t k, const unsigned long long* counts,
                                                       const int64_t* seg_start, int64_t* p, uint8_t* heads_out) {
  for (int64_t i = (int64_t)blockIdx.x * BLOCK + threadIdx.x; i < n; i += (int64_t)gridDim.x * BLOCK) {
    const int64_t sg = seg[i], st = f[i];
    int64_t off = 0;
    for (int64_t j = 0; j < st; j++) off += (int64_t)counts[sg * k + j];
    p[i] = seg_start[sg] + off + rank[i];
    heads_out[i] = 0;
  }
}

__global__ void __launch_bounds__(BLOCK) k_fp_heads(int64_t nseg, int64_t k, const unsigned long long* counts,
                                                    const int64_t* seg_start, uint8_t* heads_out) {
  for (int64_t sg = (int64_t)blockIdx.x * BLOCK + threadIdx.x; sg < nseg; sg += (int64_t)gridDim.x * BLOCK) {
    int64_t off = 0;
    for (int64_t j = 0; j < k; j++) {
      const int64_t c = (int64_t)counts[sg * k + j];
      if (c) heads_out[seg_start[sg] + off] = 1;
      off += c;
    }
  }
}

// ------------------------------------------------------------ compact
__global__ void __launch_bounds__(BLOCK) k_cp_heads(const int64_t* firsts, const uint8_t* heads, int64_t n,
                                                    uint8_t* heads_out) {
  for (int64_t i = (int64_t)blockIdx.x * BLOCK + threadIdx.x; i < n; i += (int64_t)gridDim.x * BLOCK) {
    if ((i == 0 || heads[i]) && firsts[i] != 0x7FFFFFFFFFFFFFFFll) heads_out[firsts[i]] = 1;
  }
}

// ------------------------------------------------------------ scatter
// out[p[i]] = data[i] (row of `row` bytes) for live i; counts collisions and
// out-of-range destinations into err[0] / err[1]
__global__ void __launch_bounds__(BLOCK) k_scatter_check(const int64_t* p, const uint8_t* live, int64_t n,
                                                         int64_t out_len, unsigned int* hits,
                                                         unsigned long long* err) {
  for (int64_t i = (int64_t)blockIdx.x * BLOCK + threadIdx.x; i < n; i += (int64_t)gridDim.x * BLOCK) {
    if (live && !live[i]) continue;
    const int64_t d = p[i];
    if (d < 0 || d >= out_len) {
      atomicAdd(&err[1], 1ull);
      continue;
    }
    if (atomicAdd(&hits[d], 1u) != 0) atomicAdd(&err[0], 1ull);
  }
}

__global__ void __launch_bounds__(BLOCK) k_scatter(const unsigned char* data, const int64_t* p, const uint8_t* live,
                                                   int64_t n, int64_t row, unsigned char* out) {
  for (int64_t i = (int64_t)blockIdx.x * BLOCK + threadIdx.x; i < n; i += (int64_t)gridDim.x * BLOCK) {
    if (live && !live[i]) continue;
    const unsigned char* s = data + i * row;
    unsigned char* d = out + p[i] * row;
    for (int64_t b = 0; b < row; b++) d[b] = s[b];
  }
}

}  // namespace sh
