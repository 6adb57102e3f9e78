// Deterministic fp64 gosa reduction shared by every stencil kernel.
#pragma once
#include "hp_internal.h"

namespace hp {
namespace {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// Block sum in fixed order; result valid in thread 0.
__device__ double block_sum(double v) {
  __shared__ double warp_part[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) warp_part[w] = v;
  __syncthreads();
  double t = 0.0;
  if (w == 0) {
    t = lane < nw ? warp_part[lane] : 0.0;
    t = warp_sum(t);
  }
  return t;
}

// Every block calls this exactly once with its partial; the last block to
// arrive folds all partials (in block order) into *slot.
__device__ void gosa_commit(const GosaSink& g, double v, int nblocks, int block_id, int reset) {
  __shared__ bool last;
  const double s = block_sum(v);
  if (threadIdx.x == 0) {
    g.partials[block_id] = s;
    __threadfence();
    const unsigned t = atomicAdd(g.ticket, 1u);
    last = (t == (unsigned)nblocks - 1u);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double acc = 0.0;
  for (int b = threadIdx.x; b < nblocks; b += blockDim.x)
    acc += ((volatile double*)g.partials)[b];
  acc = block_sum(acc);
  if (threadIdx.x == 0) {
    *g.slot = reset ? acc : (*g.slot + acc);
    *g.ticket = 0u;
  }
}

}  // namespace
}  // namespace hp
