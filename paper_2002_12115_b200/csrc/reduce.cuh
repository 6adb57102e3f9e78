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

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Persistent kernels with a dynamic unit queue (stencil_tma.cu): which CTA runs
// which unit varies from run to run, so per-CTA partials would make the grid
// total depend on scheduling.  Instead the nw warps that computed a unit
// (warp index wrel among them; all call this, named barrier `bar`) fold their
// sums in warp order into partials[unit], and gosa_commit_units folds the units
// in unit order: gosa is bit-reproducible.  `part` = nw doubles of smem.
__device__ void unit_partial(const GosaSink& g, uint32_t unit, double v, double* part, int wrel,
                             int nw, int bar) {
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) part[wrel] = v;
  named_bar_sync(bar, nw * 32);
  if (wrel == 0 && (threadIdx.x & 31) == 0) {
    double s = 0.0;
    for (int w = 0; w < nw; ++w) s += part[w];
    g.partials[unit] = s;
  }
  named_bar_sync(bar, nw * 32);   // part[] is reused by the next unit
}

// Every thread of every block calls this once at the end of a unit-queue
// kernel; the last block folds partials[0, nunits) in unit order into *slot.
__device__ void gosa_commit_units(const GosaSink& g, uint32_t nunits, int reset) {
  __shared__ bool last_block;
  __threadfence();   // this block's unit partials before its ticket
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned t = atomicAdd(g.ticket, 1u);
    last_block = (t == gridDim.x - 1u);
  }
  __syncthreads();
  if (!last_block) return;
  __threadfence();
  double acc = 0.0;
  for (uint32_t u = threadIdx.x; u < nunits; u += blockDim.x)
    acc += ((volatile double*)g.partials)[u];
  acc = block_sum(acc);
  if (threadIdx.x == 0) {
    *g.slot = reset ? acc : (*g.slot + acc);
    *g.ticket = 0u;
    *g.work = 0u;   // every unit was claimed: the queue is ready for the next launch
  }
}

// Every block calls this exactly once with its partial; the last block to
// arrive folds all partials (in block order) into *slot.
__device__ void gosa_commit(const GosaSink& g, double v, int nblocks, int block_id, int reset) {
  __shared__ bool last;
  const double s = block_sum(v);
  if (nblocks == 1) {
    // single-block launch (a row of an inner-loop gang): no partials / ticket
    // round trip; same sum as the last-block fold of one partial
    if (threadIdx.x == 0) *g.slot = reset ? s : (*g.slot + s);
    return;
  }
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
