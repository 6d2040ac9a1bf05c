// K4: 3D post-loop candidate filter (reference _extreme_vertex_mask,
// quickhull.py:136-164) and result assembly.
//
// PLACEHOLDER (round-1 bring-up): candidates are passed through unfiltered
// and result[2] = 0 marks "filter not applied"; the Python shim refuses to
// return such a 3D result.  Replaced by the device gift-wrapping filter.
#pragma once

#include "sh_common.cuh"

namespace sh {

struct FilterWs {
  unsigned long long* result;  // [0] vertices kept, [1] facets, [2] filter applied, [3] spare
  int32_t* out_facets;
  int64_t facet_cap;
};

static inline int filter_alloc(FilterWs& f, uint64_t n) {
  (void)n;
  return cudaMalloc((void**)&f.result, 64) == cudaSuccess ? 0 : 1;
}

static inline void filter_free(FilterWs& f) {
  if (f.result) cudaFree(f.result);
  f.result = nullptr;
}

static inline int filter_set_params(FilterWs& f, int32_t* facets, int64_t cap, cudaStream_t s) {
  (void)s;
  f.out_facets = facets;
  f.facet_cap = cap;
  return 0;
}

__global__ void k_filter_passthrough(Workspace ws, FilterWs fw) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    fw.result[0] = ws.st->h_final;
    fw.result[1] = 0;
    fw.result[2] = 0;
  }
}

static inline int filter_launch(FilterWs& f, Workspace ws, int nsm, cudaStream_t s) {
  (void)nsm;
  k_filter_passthrough<<<1, 32, 0, s>>>(ws, f);
  return cudaGetLastError() == cudaSuccess ? 0 : 10;
}

// vout (uint32, discovery order) -> user int64 indices
template <int DIM>
__global__ void __launch_bounds__(BLOCK) k_output(Workspace ws, FilterWs fw) {
  DevState* st = ws.st;
  uint32_t h = st->h_final;
  int64_t* out = st->out_idx;
  for (uint32_t i = blockIdx.x * BLOCK + threadIdx.x; i < h; i += gridDim.x * BLOCK)
    out[i] = (int64_t)ws.vout[i];
}

}  // namespace sh
