// TMA-pipelined full-interior stencil (loops 7-9 body) for sm_100a.
//
// Warp-specialised CTA, one per SM (persistent over a contiguous range of
// (tile, plane) work units -- same partition as k_stencil_3d):
//
//   warp 8 (producer, one elected lane): for every plane i of its units issues
//       cp.async.bulk.tensor.3d loads of
//         * the 12 coefficient tiles  a0..a3 b0..b2 c0..c2 wrk1 bnd, box 128k x 8j
//         * the p tile of plane i+1 with a 1-row / 4-column halo, box 136k x 10j
//           (TMA zero-fills out-of-bounds halo: only masked lanes consume it)
//       into stage s = seq % S of a shared-memory ring, completing on full[s]
//       (mbarrier complete_tx); it first waits empty[s] for the consumers.
//   warps 0..7 (consumers, warp w = row j0+w, lane = k-quad): keep the
//       register queue of p rows (j-1, j, j+1) for planes i-1, i; read the new
//       plane's rows and the coefficients from the stage, release it
//       (one arrive per warp on empty[s]), then compute and store 4 points.
//       k+-1 neighbours: lane shuffles, halo columns 3 / 132 for the edge lanes.
//
// HBM traffic per interior point = 12 coefficient reads + 1 p read (halo rows
// and columns hit in L2) + 1 wrk2 write = 56 B, the algorithmic minimum; the
// ring keeps S x 53 KB in flight per SM, independent of register pressure.
// Arithmetic and gosa handling are identical to k_stencil_3d (bit-exact p).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>

#include "hp_internal.h"
#include "reduce.cuh"

namespace hp {
namespace {

constexpr int TJ = 8;                 // rows per tile = consumer warps
constexpr int TK = 128;               // k per tile (32 lanes x float4)
constexpr int PW = TK + 8;            // p tile row: 4-float halo each side (16-byte aligned)
constexpr int PH = TJ + 2;            // p tile rows: j0-1 .. j0+TJ
constexpr int NCOEF = 12;
constexpr int kThreads = (TJ + 1) * 32;
constexpr uint32_t kPBytes = PW * PH * 4;                    // 5440
constexpr uint32_t kPSlot = (kPBytes + 127) / 128 * 128;     // 5504
constexpr uint32_t kCoefBytes = TK * TJ * 4;                 // 4096
constexpr uint32_t kStageBytes = kPSlot + NCOEF * kCoefBytes;

// coefficient slots in smem order (fields a0..a3 b0..b2 c0..c2 wrk1 bnd)
enum { CA0 = 0, CA1, CA2, CA3, CB0, CB1, CB2, CC0, CC1, CC2, CW1, CBN };

struct __align__(64) StencilMaps {
  CUtensorMap coef[NCOEF];
  CUtensorMap pin;
};

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
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
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
  asm volatile("trap;");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ float fmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float fadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float fsub(float a, float b) { return __fsub_rn(a, b); }

struct Row {            // one p row quad of a lane + its k-1 / k+4 neighbours
  float4 v;
  float left, right;
};

__device__ __forceinline__ float el(const float4& v, int x) {
  return x == 0 ? v.x : (x == 1 ? v.y : (x == 2 ? v.z : v.w));
}
__device__ __forceinline__ float km1(const Row& r, int x) { return x == 0 ? r.left : el(r.v, x - 1); }
__device__ __forceinline__ float kp1(const Row& r, int x) { return x == 3 ? r.right : el(r.v, x + 1); }

// read p tile row `row` (0..PH-1) for this lane from a stage
__device__ __forceinline__ Row load_row(const float* ptile, int row, int lane) {
  const float* base = ptile + row * PW;
  Row r;
  r.v = *reinterpret_cast<const float4*>(base + 4 + lane * 4);
  r.left = __shfl_up_sync(0xffffffffu, r.v.w, 1);
  r.right = __shfl_down_sync(0xffffffffu, r.v.x, 1);
  if (lane == 0) r.left = base[3];
  if (lane == 31) r.right = base[4 + TK];
  return r;
}

struct Unit {           // one contiguous run of planes of one tile
  int kt, jt, ia, ib;
};

// the CTA's segments, identical for producer and consumers
struct Walker {
  long long u, u_end;
  int ni, ktiles;
  __device__ bool next(Unit& s) {
    if (u >= u_end) return false;
    const int t = (int)(u / ni);
    s.ia = (int)(u % ni);
    s.ib = (int)min((long long)ni, (long long)s.ia + (u_end - u));
    u += s.ib - s.ia;
    s.kt = t % ktiles;
    s.jt = t / ktiles;
    return true;
  }
};

template <int S>
__global__ void __launch_bounds__(kThreads, 1)
k_stencil_tma(const __grid_constant__ StencilMaps maps, DevFields F, float* __restrict__ out,
              int i_lo, int i_hi, int j_lo, int j_hi, int k_lo, int k_hi, int ktiles,
              float omega, GosaSink g, int reset) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  // TMA destinations are 128-byte aligned regardless of static smem placement
  unsigned char* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * kStageBytes);
  uint64_t* empty = full + S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ni = i_hi - i_lo;
  const int jtiles = (j_hi - j_lo + TJ - 1) / TJ;
  const long long U = (long long)ktiles * jtiles * ni;
  Walker walk{U * blockIdx.x / gridDim.x, U * (blockIdx.x + 1) / gridDim.x, ni, ktiles};

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], TJ);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  double acc = 0.0;
  if (warp == TJ) {
    // ------------------------------------------------------------- producer
    if (lane == 0) {
      for (int m = 0; m < NCOEF; ++m)
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.coef[m])));
      uint32_t seq = 0;
      Unit s{0, 0, 0, 0};
      auto issue = [&](const Unit& s, int plane_p, int plane_c) {  // plane_c < 0: p-only stage
        const int slot = seq % S;
        if (seq >= (uint32_t)S) mbar_wait(&empty[slot], ((seq / S) - 1) & 1);
        unsigned char* st = smem + slot * kStageBytes;
        const uint32_t bytes = kPBytes + (plane_c >= 0 ? NCOEF * kCoefBytes : 0);
        mbar_expect_tx(&full[slot], bytes);
        tma_load_3d(st, &maps.pin, &full[slot], s.kt * TK - 4, j_lo + s.jt * TJ - 1, plane_p);
        if (plane_c >= 0)
          for (int m = 0; m < NCOEF; ++m)
            tma_load_3d(st + kPSlot + m * kCoefBytes, &maps.coef[m], &full[slot], s.kt * TK,
                        j_lo + s.jt * TJ, plane_c);
        ++seq;
      };
      while (walk.next(s)) {
        const int i0 = i_lo + s.ia, i1 = i_lo + s.ib;
        issue(s, i0 - 1, -1);
        issue(s, i0, -1);
        for (int i = i0; i < i1; ++i) issue(s, i + 1, i);
      }
    }
  } else {
    // ------------------------------------------------------------ consumers
    uint32_t seq = 0;
    Unit s;
    const size_t P = F.P, L = F.plane();
    while (walk.next(s)) {
      const int j = j_lo + s.jt * TJ + warp;
      const bool row_ok = j < j_hi;
      const int kb = s.kt * TK + lane * 4;
      const bool active = row_ok && kb + 3 >= k_lo && kb < k_hi;
      bool ok[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) ok[x] = active && kb + x >= k_lo && kb + x < k_hi;
      const bool whole = ok[0] && ok[1] && ok[2] && ok[3];
      Row lm, l0, lp, mm, m0, mp;
      // warm-up stages: planes i0-1 and i0
      for (int w = 0; w < 2; ++w) {
        const int slot = seq % S;
        mbar_wait(&full[slot], (seq / S) & 1);
        const float* pt = reinterpret_cast<const float*>(smem + slot * kStageBytes);
        const Row a = load_row(pt, warp, lane), b = load_row(pt, warp + 1, lane),
                  c = load_row(pt, warp + 2, lane);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
        if (w == 0) { lm = a; l0 = b; lp = c; }
        else { mm = a; m0 = b; mp = c; }
        ++seq;
      }
      size_t cidx = F.at(i_lo + s.ia, j, kb);
#pragma unroll 1
      for (int i = i_lo + s.ia; i < i_lo + s.ib; ++i, cidx += L) {
        const int slot = seq % S;
        mbar_wait(&full[slot], (seq / S) & 1);
        const unsigned char* st = smem + slot * kStageBytes;
        const float* pt = reinterpret_cast<const float*>(st);
        const Row nm = load_row(pt, warp, lane), n0 = load_row(pt, warp + 1, lane),
                  np = load_row(pt, warp + 2, lane);
        float4 q[NCOEF];
#pragma unroll
        for (int m = 0; m < NCOEF; ++m)
          q[m] = *reinterpret_cast<const float4*>(st + kPSlot + m * kCoefBytes +
                                                  (warp * TK + lane * 4) * 4);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
        ++seq;
        if (row_ok) {
          float r[4];
#pragma unroll
          for (int x = 0; x < 4; ++x) {
            float s0 = fmul(el(q[CA0], x), el(n0.v, x));
            s0 = fadd(s0, fmul(el(q[CA1], x), el(mp.v, x)));
            s0 = fadd(s0, fmul(el(q[CA2], x), kp1(m0, x)));
            s0 = fadd(s0, fmul(el(q[CB0], x),
                               fadd(fsub(fsub(el(np.v, x), el(nm.v, x)), el(lp.v, x)), el(lm.v, x))));
            s0 = fadd(s0, fmul(el(q[CB1], x),
                               fadd(fsub(fsub(kp1(mp, x), kp1(mm, x)), km1(mp, x)), km1(mm, x))));
            s0 = fadd(s0, fmul(el(q[CB2], x),
                               fadd(fsub(fsub(kp1(n0, x), kp1(l0, x)), km1(n0, x)), km1(l0, x))));
            s0 = fadd(s0, fmul(el(q[CC0], x), el(l0.v, x)));
            s0 = fadd(s0, fmul(el(q[CC1], x), el(mm.v, x)));
            s0 = fadd(s0, fmul(el(q[CC2], x), km1(m0, x)));
            s0 = fadd(s0, el(q[CW1], x));
            const float ss = fmul(fsub(fmul(s0, el(q[CA3], x)), el(m0.v, x)), el(q[CBN], x));
            r[x] = fadd(el(m0.v, x), fmul(omega, ss));
            if (ok[x]) acc += (double)fmul(ss, ss);
          }
          if (whole) {
            *reinterpret_cast<float4*>(out + cidx) = make_float4(r[0], r[1], r[2], r[3]);
          } else if (active) {
#pragma unroll
            for (int x = 0; x < 4; ++x)
              if (ok[x]) out[cidx + x] = r[x];
          }
        }
        lm = mm; l0 = m0; lp = mp;
        mm = nm; m0 = n0; mp = np;
      }
      (void)P;
    }
  }
  gosa_commit(g, acc, gridDim.x, blockIdx.x, reset);
}

// ------------------------------------------------------------------ host side

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
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

bool encode(CUtensorMap* m, const DevFields& F, const float* base, uint32_t box_k, uint32_t box_j) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)F.P, (cuuint64_t)F.J, (cuuint64_t)F.I};
  const cuuint64_t strides[2] = {(cuuint64_t)F.P * 4, (cuuint64_t)F.plane() * 4};
  const cuuint32_t box[3] = {box_k, box_j, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

struct TmaState {
  StencilMaps base;          // coefficient maps + p map
  CUtensorMap scratch_map;   // p map of the rotation buffer
  const float* p;
  const float* scratch;
};

}  // namespace

// Build the tensor maps of one context (fields + rotation scratch); nullptr if
// the driver cannot encode them (the caller then uses k_stencil_3d).
void* create_stencil_tma(const DevFields& F, const float* scratch) {
  TmaState* t = new TmaState;
  bool ok = true;
  for (int m = 0; m < NCOEF; ++m) {
    static const int fields[NCOEF] = {HP_F_A0, HP_F_A1, HP_F_A2, HP_F_A3, HP_F_B0, HP_F_B1,
                                      HP_F_B2, HP_F_C0, HP_F_C1, HP_F_C2, HP_F_WRK1, HP_F_BND};
    ok = ok && encode(&t->base.coef[m], F, F.f[fields[m]], TK, TJ);
  }
  ok = ok && encode(&t->base.pin, F, F.f[HP_F_P], PW, PH);
  ok = ok && encode(&t->scratch_map, F, scratch, PW, PH);
  t->p = F.f[HP_F_P];
  t->scratch = scratch;
  if (!ok) {
    delete t;
    return nullptr;
  }
  return t;
}

void destroy_stencil_tma(void* h) { delete static_cast<TmaState*>(h); }

// Launch the TMA stencil with S stages; returns 1, 0 (not applicable: caller
// falls back), or -1 on launch error.
int launch_stencil_tma(const DevFields& F, const void* h, const float* p_in, float* p_out,
                       const LaunchArgs& a, const GosaSink& g, cudaStream_t s, int stages,
                       int sms) {
  const TmaState* t = static_cast<const TmaState*>(h);
  if (!t || (p_in != t->p && p_in != t->scratch)) return 0;
  const int i_lo = a.li_lo, i_hi = a.li_hi, j_lo = 1, j_hi = a.jmax - 1, k_lo = 1,
            k_hi = a.kmax - 1;
  if (i_hi <= i_lo || j_hi <= j_lo || k_hi <= k_lo) return 0;
  StencilMaps maps = t->base;
  if (p_in == t->scratch) maps.pin = t->scratch_map;
  const int ktiles = (k_hi + TK - 1) / TK;
  const int jtiles = (j_hi - j_lo + TJ - 1) / TJ;
  const long long units = (long long)ktiles * jtiles * (i_hi - i_lo);
  long long grid = sms;
  if (grid > units) grid = units;
  if (grid > g.capacity) return -1;
  const size_t smem = 128 + (size_t)stages * kStageBytes + 2 * stages * sizeof(uint64_t);
  static bool attr_set[5] = {};   // per stage count: raise the dynamic smem limit once
  auto launch = [&](auto kern) {
    if (!attr_set[stages]) {
      if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
          cudaSuccess)
        return;
      attr_set[stages] = true;
    }
    kern<<<(int)grid, kThreads, smem, s>>>(maps, F, p_out, i_lo, i_hi, j_lo, j_hi, k_lo, k_hi,
                                           ktiles, a.omega, g, a.gosa_reset);
  };
  switch (stages) {
    case 2: launch(k_stencil_tma<2>); break;
    case 3: launch(k_stencil_tma<3>); break;
    case 4: launch(k_stencil_tma<4>); break;
    default: return 0;
  }
  return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

}  // namespace hp
