// TMA / mbarrier helpers shared by the TMA-pipelined stencil kernels.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "hp_internal.h"

namespace hp {
namespace tma {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Bounded wait: a pipeline bug must abort the kernel (trap -> launch error),
// never hang the GPU.  2^26 polls (each try_wait suspends up to a
// hardware-defined interval) is seconds, far beyond any legitimate wait.
// try_wait suspend-time hint (ns) of mbar_wait: 1000 -> M flow pass 42.4 -> 40.3 us, L
// pass -1..2 %: the polling loops of waiting warps had been ~19 % of the two-step kernel's
// executed instructions (profiles/r02_tb2_experiments_late.md).  0 = no hint.
#ifndef HP_MBAR_HINT_NS
#define HP_MBAR_HINT_NS 1000
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
#if HP_MBAR_HINT_NS > 0
  // suspend-time hint: a waiting warp sleeps until the phase completes (or the hint
  // expires) instead of re-polling, leaving its issue slots to the working warps
#pragma unroll 1
  for (uint32_t n = 0; n < (1u << 26) / (HP_MBAR_HINT_NS / 100 + 1) + 16; ++n) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity), "r"((uint32_t)HP_MBAR_HINT_NS)
        : "memory");
    if (done) return;
  }
#else
#pragma unroll 1
  for (uint32_t n = 0; n < (1u << 26); ++n) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) return;
  }
#endif
  asm volatile("trap;");
}
// try_wait with a short suspend hint (ns): true once the phase has completed
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(done)
      : "r"(smem_u32(bar)), "r"(parity), "r"(100u)
      : "memory");
  return done != 0;
}
// non-blocking: has the phase with this parity completed?
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(done)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return done != 0;
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

// the same with an L2 cache-policy hint (createpolicy): eviction priority of the lines
__device__ __forceinline__ void tma_load_3d_hint(void* dst, const CUtensorMap* map, uint64_t* bar,
                                                 int c0, int c1, int c2, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)),
      "l"(policy)
      : "memory");
}

// ---- device-wide dynamic work queue -----------------------------------------
// The producer lane of each CTA claims unit ids with atomicAdd on a counter
// (reset to 0 before the launch) and hands them to the CTA's consumer warps
// through a small ring in shared memory (full: 1 arrive, empty: one arrive per
// consumer warp).  A claim >= the unit count is published as kNoUnit.
constexpr uint32_t kNoUnit = 0xffffffffu;
constexpr int kUnitRing = 4;
struct UnitRing {
  uint32_t id[kUnitRing];
  uint64_t full[kUnitRing];
  uint64_t empty[kUnitRing];
};

__device__ __forceinline__ void unit_ring_init(UnitRing* r, int consumers);
__device__ __forceinline__ uint32_t unit_publish(UnitRing* r, uint32_t n, unsigned int* counter,
                                                 uint32_t units);
__device__ __forceinline__ uint32_t unit_take(UnitRing* r, uint32_t n, int lane);

__device__ __forceinline__ float fmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float fadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float fsub(float a, float b) { return __fsub_rn(a, b); }

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
    else
      cudaGetLastError();
  }
  return fn;
}

__device__ __forceinline__ void unit_ring_init(UnitRing* r, int consumers) {
  for (int s = 0; s < kUnitRing; ++s) {
    mbar_init(&r->full[s], 1);
    mbar_init(&r->empty[s], consumers);
  }
}
// producer lane: claim the n-th unit of this CTA and publish it; returns the id
__device__ __forceinline__ uint32_t unit_publish(UnitRing* r, uint32_t n, unsigned int* counter,
                                                 uint32_t units) {
  const int slot = n % kUnitRing;
  if (n >= (uint32_t)kUnitRing) mbar_wait(&r->empty[slot], ((n / kUnitRing) - 1) & 1);
  uint32_t u = atomicAdd(counter, 1u);
  if (u >= units) u = kNoUnit;
  r->id[slot] = u;
  mbar_arrive(&r->full[slot]);
  return u;
}
// consumer warp: the n-th unit of this CTA (all lanes), slot released by lane 0
__device__ __forceinline__ uint32_t unit_take(UnitRing* r, uint32_t n, int lane) {
  const int slot = n % kUnitRing;
  mbar_wait(&r->full[slot], (n / kUnitRing) & 1);
  const uint32_t u = *(volatile uint32_t*)&r->id[slot];
  __syncwarp();
  if (lane == 0) mbar_arrive(&r->empty[slot]);
  return u;
}

// L2 promotion of a map: 0 none, 1 64B, 2 128B, 3 256B
inline CUtensorMapL2promotion promo(int code) {
  switch (code) {
    case 0: return CU_TENSOR_MAP_L2_PROMOTION_NONE;
    case 1: return CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
    case 3: return CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    default: return CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
  }
}

inline bool encode(CUtensorMap* m, const DevFields& F, const float* base, uint32_t box_k,
                   uint32_t box_j, int promo_code = 2, int dim_k = 0, int dim_j = 0) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)(dim_k > 0 ? dim_k : F.P),
                              (cuuint64_t)(dim_j > 0 ? dim_j : F.J), (cuuint64_t)F.I};
  const cuuint64_t strides[2] = {(cuuint64_t)F.P * 4, (cuuint64_t)F.plane() * 4};
  const cuuint32_t box[3] = {box_k, box_j, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            promo(promo_code), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}


}  // namespace tma
}  // namespace hp
