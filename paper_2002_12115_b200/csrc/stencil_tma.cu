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
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "hp_internal.h"
#include "reduce.cuh"
#include "tma.cuh"

namespace hp {
namespace {
using namespace tma;

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
// planes per work unit (HIMENO_CHUNK overrides for sweeps)
static int chunk_planes() {
  static int c = 0;
  if (!c) {
    const char* e = getenv("HIMENO_CHUNK");
    c = e ? atoi(e) : 32;
    if (c < 1) c = 32;
  }
  return c;
}

// coefficient slots in smem order (fields a0..a3 b0..b2 c0..c2 wrk1 bnd)
enum { CA0 = 0, CA1, CA2, CA3, CB0, CB1, CB2, CC0, CC1, CC2, CW1, CBN };

struct __align__(64) StencilMaps {
  CUtensorMap coef[NCOEF];
  CUtensorMap pin;
};

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

// Work units = (plane chunk, tile) in chunk-major order, handed out by the
// device-wide queue (tma.cuh): CTAs that are resident together stream
// neighbouring tiles over the same planes at the same time, so the halo rows a
// tile shares with its neighbours are served from L2.
struct Units {
  int ni, ktiles, tiles, len;
  uint32_t count;
  __device__ void decode(uint32_t u, Unit& s) const {
    const int t = (int)(u % (uint32_t)tiles), c = (int)(u / (uint32_t)tiles);
    s.kt = t % ktiles;
    s.jt = t / ktiles;
    s.ia = c * len;
    s.ib = min(ni, s.ia + len);
  }
};

template <int S>
__global__ void __launch_bounds__(kThreads, 1)
k_stencil_tma(const __grid_constant__ StencilMaps maps, DevFields F, float* __restrict__ out,
              int i_lo, int i_hi, int j_lo, int j_hi, int k_lo, int k_hi, int ktiles, int chunk,
              float omega, GosaSink g, int reset) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  // TMA destinations are 128-byte aligned regardless of static smem placement
  unsigned char* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * kStageBytes);
  uint64_t* empty = full + S;
  UnitRing* ring = reinterpret_cast<UnitRing*>(empty + S);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ni = i_hi - i_lo;
  const int jtiles = (j_hi - j_lo + TJ - 1) / TJ;
  Units units{ni, ktiles, ktiles * jtiles, chunk,
              (uint32_t)(ktiles * jtiles * ((ni + chunk - 1) / chunk))};

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], TJ);
    }
    unit_ring_init(ring, TJ);
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
      for (uint32_t n = 0;; ++n) {
        const uint32_t u = unit_publish(ring, n, g.work, units.count);
        if (u == kNoUnit) break;
        units.decode(u, s);
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
    for (uint32_t n = 0;; ++n) {
      const uint32_t u = unit_take(ring, n, lane);
      if (u == kNoUnit) break;
      units.decode(u, s);
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

// ================================================================ two-step kernel
//
// k_stencil_tb2: two Jacobi iterations per pass (temporal blocking).  Output
// tile = TJ2 rows x 128 k; step 1 computes p1 = S(p0) on the tile extended by
// one row / column on each side (R1 = TJ2+2 rows, 130 columns) so that step 2
// can compute p2 = S(p1) on the tile one plane behind.  The 12 coefficient
// arrays are read from HBM once for both iterations: 56 B per point per TWO
// iterations (vs 2 x 56 for two single-step passes).
//
//   producer warp: p0 plane tiles (136k x (R1+2)j) into a 4-slot ring, extended
//     coefficient tiles (136k x R1 j, 12 arrays) into a 3-slot ring.
//   consumer warp w (0..R1-1) <-> row j0-1+w:
//     step 1 (plane m): register queue of p0 rows, lanes = k-quads, lane 0 / 31
//       also the extra columns k0-1 / k0+128 (scalars from the p0 ring);
//       non-interior points copy p0 (boundaries are fixed).  p1 -> smem (2 slots).
//     named barrier among the consumer warps (p1(m) complete)
//     step 2 (plane m-1, warps 1..TJ2): register queue of p1 rows; coefficients
//       of plane m-1 are still resident in the coefficient ring.
// Every product/sum rounds exactly like the single-step kernel: p2 is
// bit-identical to two single steps; gosa (fp64) is that of the second step.
constexpr int TJ2 = 6;                 // output rows per tile
constexpr int R1 = TJ2 + 2;            // step-1 rows = consumer warps
constexpr int kThreads2 = (R1 + 1) * 32;
constexpr uint32_t kP0Bytes = PW * (R1 + 2) * 4;           // 5440
constexpr uint32_t kP0Slot = (kP0Bytes + 127) / 128 * 128;
constexpr uint32_t kCExtBytes = PW * R1 * 4;               // 4352 per array
constexpr uint32_t kCSlot = NCOEF * kCExtBytes;            // 52224
constexpr uint32_t kP1Slot = PW * R1 * 4;                  // 4352
constexpr int SP = 4, SC = 3, SQ = 2;                      // p0 / coef / p1 ring slots
constexpr uint32_t kTb2Smem = SP * kP0Slot + SC * kCSlot + SQ * kP1Slot;

struct __align__(64) Tb2Maps {
  CUtensorMap coef[NCOEF];   // box 136 x R1
  CUtensorMap pin;           // box 136 x (R1+2)
};

// one step of the stencil at element x of lane quads (rows: m* plane i, l* i-1, n* i+1)
__device__ __forceinline__ float ss_point(const float* q, const Row& lm, const Row& l0,
                                          const Row& lp, const Row& mm, const Row& m0,
                                          const Row& mp, const Row& nm, const Row& n0,
                                          const Row& np, int x) {
  float s0 = fmul(q[CA0], el(n0.v, x));
  s0 = fadd(s0, fmul(q[CA1], el(mp.v, x)));
  s0 = fadd(s0, fmul(q[CA2], kp1(m0, x)));
  s0 = fadd(s0, fmul(q[CB0], fadd(fsub(fsub(el(np.v, x), el(nm.v, x)), el(lp.v, x)), el(lm.v, x))));
  s0 = fadd(s0, fmul(q[CB1], fadd(fsub(fsub(kp1(mp, x), kp1(mm, x)), km1(mp, x)), km1(mm, x))));
  s0 = fadd(s0, fmul(q[CB2], fadd(fsub(fsub(kp1(n0, x), kp1(l0, x)), km1(n0, x)), km1(l0, x))));
  s0 = fadd(s0, fmul(q[CC0], el(l0.v, x)));
  s0 = fadd(s0, fmul(q[CC1], el(mm.v, x)));
  s0 = fadd(s0, fmul(q[CC2], km1(m0, x)));
  s0 = fadd(s0, q[CW1]);
  return fmul(fsub(fmul(s0, q[CA3]), el(m0.v, x)), q[CBN]);
}

// the same on scalars read from shared-memory tiles: P(plane, drow, dcol)
template <class PF>
__device__ __forceinline__ float ss_scalar(const float* q, PF P) {
  float s0 = fmul(q[CA0], P(1, 0, 0));
  s0 = fadd(s0, fmul(q[CA1], P(0, 1, 0)));
  s0 = fadd(s0, fmul(q[CA2], P(0, 0, 1)));
  s0 = fadd(s0, fmul(q[CB0], fadd(fsub(fsub(P(1, 1, 0), P(1, -1, 0)), P(-1, 1, 0)), P(-1, -1, 0))));
  s0 = fadd(s0, fmul(q[CB1], fadd(fsub(fsub(P(0, 1, 1), P(0, -1, 1)), P(0, 1, -1)), P(0, -1, -1))));
  s0 = fadd(s0, fmul(q[CB2], fadd(fsub(fsub(P(1, 0, 1), P(-1, 0, 1)), P(1, 0, -1)), P(-1, 0, -1))));
  s0 = fadd(s0, fmul(q[CC0], P(-1, 0, 0)));
  s0 = fadd(s0, fmul(q[CC1], P(0, -1, 0)));
  s0 = fadd(s0, fmul(q[CC2], P(0, 0, -1)));
  s0 = fadd(s0, q[CW1]);
  return fmul(fsub(fmul(s0, q[CA3]), P(0, 0, 0)), q[CBN]);
}

__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__global__ void __launch_bounds__(kThreads2, 1)
k_stencil_tb2(const __grid_constant__ Tb2Maps maps, DevFields F, float* __restrict__ out,
              int i_lo, int i_hi, int j_lo, int j_hi, int k_lo, int k_hi, int ktiles, int chunk,
              float omega, GosaSink g, int reset) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  unsigned char* p0ring = smem;
  unsigned char* cring = p0ring + SP * kP0Slot;
  float* p1ring = reinterpret_cast<float*>(cring + SC * kCSlot);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kTb2Smem);
  uint64_t* pfull = bars;
  uint64_t* pempty = pfull + SP;
  uint64_t* cfull = pempty + SP;
  uint64_t* cempty = cfull + SC;
  UnitRing* ring = reinterpret_cast<UnitRing*>(cempty + SC);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ni = i_hi - i_lo;
  const int jtiles = (j_hi - j_lo + TJ2 - 1) / TJ2;
  Units units{ni, ktiles, ktiles * jtiles, chunk,
              (uint32_t)(ktiles * jtiles * ((ni + chunk - 1) / chunk))};
  if (threadIdx.x == 0) {
    for (int s = 0; s < SP; ++s) { mbar_init(&pfull[s], 1); mbar_init(&pempty[s], R1); }
    for (int s = 0; s < SC; ++s) { mbar_init(&cfull[s], 1); mbar_init(&cempty[s], R1); }
    unit_ring_init(ring, R1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  double acc = 0.0;
  if (warp == R1) {
    // ------------------------------------------------------------- producer
    if (lane == 0) {
      uint32_t sp = 0, sc = 0;
      Unit s{0, 0, 0, 0};
      auto load_p0 = [&](const Unit& u, int plane) {
        const int slot = sp % SP;
        if (sp >= (uint32_t)SP) mbar_wait(&pempty[slot], ((sp / SP) - 1) & 1);
        mbar_expect_tx(&pfull[slot], kP0Bytes);
        tma_load_3d(p0ring + slot * kP0Slot, &maps.pin, &pfull[slot], u.kt * TK - 4,
                    j_lo + u.jt * TJ2 - 2, plane);
        ++sp;
      };
      auto load_c = [&](const Unit& u, int plane) {
        const int slot = sc % SC;
        if (sc >= (uint32_t)SC) mbar_wait(&cempty[slot], ((sc / SC) - 1) & 1);
        mbar_expect_tx(&cfull[slot], NCOEF * kCExtBytes);
        for (int m = 0; m < NCOEF; ++m)
          tma_load_3d(cring + slot * kCSlot + m * kCExtBytes, &maps.coef[m], &cfull[slot],
                      u.kt * TK - 4, j_lo + u.jt * TJ2 - 1, plane);
        ++sc;
      };
      for (uint32_t n = 0;; ++n) {
        const uint32_t u = unit_publish(ring, n, g.work, units.count);
        if (u == kNoUnit) break;
        units.decode(u, s);
        const int ia = i_lo + s.ia, ib = i_lo + s.ib;
        load_p0(s, ia - 2);
        load_p0(s, ia - 1);
        for (int m = ia - 1; m <= ib; ++m) {
          load_p0(s, m + 1);
          load_c(s, m);
        }
      }
    }
  } else {
    // ------------------------------------------------------------ consumers
    uint32_t sp = 0, sc = 0;   // consumed counts of the two rings
    uint32_t it = 0;           // p1 slot counter
    Unit s;
    const int imax1 = i_hi;    // planes [i_lo, i_hi) are the global interior
    for (uint32_t n = 0;; ++n) {
      const uint32_t u = unit_take(ring, n, lane);
      if (u == kNoUnit) break;
      units.decode(u, s);
      const int ia = i_lo + s.ia, ib = i_lo + s.ib;
      const int j1 = j_lo + s.jt * TJ2 - 1 + warp;      // this warp's step-1 row
      const int k0 = s.kt * TK;
      const int kb = k0 + lane * 4;
      const bool row_in = j1 >= j_lo && j1 < j_hi;
      bool in1[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) in1[x] = row_in && kb + x >= k_lo && kb + x < k_hi;
      const bool out_row = warp >= 1 && warp <= TJ2 && row_in;   // step-2 output row
      // p0 queue: planes m-1 (a*), m (b*); p0 slot of plane q = sequence sp0 + (q - (ia-2))
      const uint32_t sp0 = sp;
      Row am, a0, ap, bm, b0, bp;
      for (int w = 0; w < 2; ++w) {
        const int slot = sp % SP;
        mbar_wait(&pfull[slot], (sp / SP) & 1);
        const float* pt = reinterpret_cast<const float*>(p0ring + slot * kP0Slot);
        const Row x0 = load_row(pt, warp, lane), x1 = load_row(pt, warp + 1, lane),
                  x2 = load_row(pt, warp + 2, lane);
        if (w == 0) { am = x0; a0 = x1; ap = x2; } else { bm = x0; b0 = x1; bp = x2; }
        ++sp;
      }
      // first p0 plane (ia-2) is only needed by step1(ia-1)'s scalars: released in-loop
      Row ym, y0, yp, zm, z0, zp;   // p1 queue: planes m-2 (y*), m-1 (z*)
      for (int m = ia - 1; m <= ib; ++m) {
        const int pslot = sp % SP;
        mbar_wait(&pfull[pslot], (sp / SP) & 1);
        const float* pt = reinterpret_cast<const float*>(p0ring + pslot * kP0Slot);
        const Row cm = load_row(pt, warp, lane), c0 = load_row(pt, warp + 1, lane),
                  cp = load_row(pt, warp + 2, lane);
        ++sp;
        const int cslot = sc % SC;
        mbar_wait(&cfull[cslot], (sc / SC) & 1);
        ++sc;
        const float* ct = reinterpret_cast<const float*>(cring + cslot * kCSlot);
        // ---- step 1 at plane m, row j1 -> p1 slot
        float* q1 = p1ring + (it % SQ) * (PW * R1);
        const bool plane_in = m >= i_lo && m < imax1;
        float r[4];
        float qv[4][NCOEF];
#pragma unroll
        for (int c = 0; c < NCOEF; ++c) {
          const float4 t = *reinterpret_cast<const float4*>(ct + c * (PW * R1) + warp * PW + 4 + lane * 4);
          qv[0][c] = t.x; qv[1][c] = t.y; qv[2][c] = t.z; qv[3][c] = t.w;
        }
#pragma unroll
        for (int x = 0; x < 4; ++x)
          r[x] = (plane_in && in1[x]) ? fadd(el(b0.v, x), fmul(omega, ss_point(qv[x], am, a0, ap,
                                                                                  bm, b0, bp, cm,
                                                                                  c0, cp, x)))
                                      : el(b0.v, x);
        *reinterpret_cast<float4*>(q1 + warp * PW + 4 + lane * 4) = make_float4(r[0], r[1], r[2], r[3]);
        if (lane == 0 || lane == 31) {
          // extra column k0-1 (lane 0) / k0+128 (lane 31), scalars from the p0 ring
          const int col = lane == 0 ? 3 : 4 + TK;
          const int k = k0 - 4 + col;
          const float* pl[3];
          for (int d = 0; d < 3; ++d)
            pl[d] = reinterpret_cast<const float*>(p0ring + ((sp0 + (m - (ia - 2)) - 1 + d) % SP) * kP0Slot);
          auto P = [&](int di, int dj, int dk) { return pl[di + 1][(warp + 1 + dj) * PW + col + dk]; };
          float v = P(0, 0, 0);
          if (plane_in && row_in && k >= k_lo && k < k_hi) {
            float qs[NCOEF];
            for (int c = 0; c < NCOEF; ++c) qs[c] = ct[c * (PW * R1) + warp * PW + col];
            v = fadd(v, fmul(omega, ss_scalar(qs, P)));
          }
          q1[warp * PW + col] = v;
        }
        // p0 plane m-1 is no longer needed (scalars of step1(m) were its last use)
        __syncwarp();
        if (lane == 0) mbar_arrive(&pempty[(sp0 + (m - (ia - 2)) - 1) % SP]);
        named_bar(1, R1 * 32);
        // ---- p1(m) rows into the queue; step 2 at plane m-1
        const Row nm = load_row(q1, warp > 0 ? warp - 1 : 0, lane),
                  n0 = load_row(q1, warp, lane),
                  np = load_row(q1, warp < R1 - 1 ? warp + 1 : R1 - 1, lane);
        if (m >= ia + 1 && out_row) {
          const int pc = (sc - 2) % SC;   // coefficient slot of plane m-1
          const float* cq = reinterpret_cast<const float*>(cring + pc * kCSlot);
          float q2[4][NCOEF];
#pragma unroll
          for (int c = 0; c < NCOEF; ++c) {
            const float4 t = *reinterpret_cast<const float4*>(cq + c * (PW * R1) + warp * PW + 4 + lane * 4);
            q2[0][c] = t.x; q2[1][c] = t.y; q2[2][c] = t.z; q2[3][c] = t.w;
          }
          float w2[4];
#pragma unroll
          for (int x = 0; x < 4; ++x) {
            const float ss = ss_point(q2[x], ym, y0, yp, zm, z0, zp, nm, n0, np, x);
            w2[x] = fadd(el(z0.v, x), fmul(omega, ss));
            if (in1[x]) acc += (double)fmul(ss, ss);
          }
          float* o = out + F.at(m - 1, j1, kb);
          if (in1[0] && in1[1] && in1[2] && in1[3]) {
            *reinterpret_cast<float4*>(o) = make_float4(w2[0], w2[1], w2[2], w2[3]);
          } else {
            for (int x = 0; x < 4; ++x)
              if (in1[x]) o[x] = w2[x];
          }
        }
        // release coefficient stages: plane m-1 after its step 2, plane ia-1 / ib after step 1
        __syncwarp();
        if (lane == 0) {
          if (m >= ia + 1) mbar_arrive(&cempty[(sc - 2) % SC]);
          if (m == ia - 1 || m == ib) mbar_arrive(&cempty[(sc - 1) % SC]);
        }
        ym = zm; y0 = z0; yp = zp;
        zm = nm; z0 = n0; zp = np;
        am = bm; a0 = b0; ap = bp;
        bm = cm; b0 = c0; bp = cp;
        ++it;
      }
      // release the p0 planes ib and ib+1 (and nothing else remains)
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&pempty[(sp - 2) % SP]);
        mbar_arrive(&pempty[(sp - 1) % SP]);
      }
    }
  }
  gosa_commit(g, acc, gridDim.x, blockIdx.x, reset);
}

// ------------------------------------------------------------------ host side

struct TmaState {
  StencilMaps base;          // coefficient maps + p map
  CUtensorMap scratch_map;   // p map of the rotation buffer
  Tb2Maps tb2;               // two-step kernel: extended coefficient boxes + p map
  CUtensorMap tb2_scratch;
  const float* p;
  const float* scratch;
};

}  // namespace

// Build the tensor maps of one context (fields + rotation scratch); nullptr if
// the driver cannot encode them (the caller then uses k_stencil_3d).
// HIMENO_TMA_PROMO="a,b,c,d": L2 promotion codes (0 none, 1 64B, 2 128B, 3 256B)
// of the single-step coefficient / p maps and the two-step coefficient / p maps.
static void promo_codes(int* c) {
  c[0] = 2; c[1] = 2; c[2] = 0; c[3] = 0;
  if (const char* e = getenv("HIMENO_TMA_PROMO"))
    sscanf(e, "%d,%d,%d,%d", &c[0], &c[1], &c[2], &c[3]);
}

void* create_stencil_tma(const DevFields& F, const float* scratch) {
  TmaState* t = new TmaState;
  int pc[4];
  promo_codes(pc);
  bool ok = true;
  for (int m = 0; m < NCOEF; ++m) {
    static const int fields[NCOEF] = {HP_F_A0, HP_F_A1, HP_F_A2, HP_F_A3, HP_F_B0, HP_F_B1,
                                      HP_F_B2, HP_F_C0, HP_F_C1, HP_F_C2, HP_F_WRK1, HP_F_BND};
    ok = ok && encode(&t->base.coef[m], F, F.f[fields[m]], TK, TJ, pc[0]);
  }
  ok = ok && encode(&t->base.pin, F, F.f[HP_F_P], PW, PH, pc[1]);
  ok = ok && encode(&t->scratch_map, F, scratch, PW, PH, pc[1]);
  for (int m = 0; m < NCOEF; ++m) {
    static const int fields[NCOEF] = {HP_F_A0, HP_F_A1, HP_F_A2, HP_F_A3, HP_F_B0, HP_F_B1,
                                      HP_F_B2, HP_F_C0, HP_F_C1, HP_F_C2, HP_F_WRK1, HP_F_BND};
    ok = ok && encode(&t->tb2.coef[m], F, F.f[fields[m]], PW, R1, pc[2]);
  }
  ok = ok && encode(&t->tb2.pin, F, F.f[HP_F_P], PW, R1 + 2, pc[3]);
  ok = ok && encode(&t->tb2_scratch, F, scratch, PW, R1 + 2, pc[3]);
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
  const int chunk = chunk_planes();
  const long long units = (long long)ktiles * jtiles * ((i_hi - i_lo + chunk - 1) / chunk);
  long long grid = sms;
  if (grid > units) grid = units;
  if (grid > g.capacity) return -1;
  const size_t smem = 128 + (size_t)stages * kStageBytes + 2 * stages * sizeof(uint64_t) +
                      sizeof(UnitRing);
  if (cudaMemsetAsync(g.work, 0, sizeof(unsigned int), s) != cudaSuccess) return -1;
  static bool attr_set[5] = {};   // per stage count: raise the dynamic smem limit once
  auto launch = [&](auto kern) {
    if (!attr_set[stages]) {
      if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
          cudaSuccess)
        return;
      attr_set[stages] = true;
    }
    kern<<<(int)grid, kThreads, smem, s>>>(maps, F, p_out, i_lo, i_hi, j_lo, j_hi, k_lo, k_hi,
                                           ktiles, chunk, a.omega, g, a.gosa_reset);
  };
  switch (stages) {
    case 2: launch(k_stencil_tma<2>); break;
    case 3: launch(k_stencil_tma<3>); break;
    case 4: launch(k_stencil_tma<4>); break;
    default: return 0;
  }
  return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

// Two-step pass p_in -> p_out (2 Jacobi iterations); returns 1, 0 (not
// applicable: caller runs two single steps), or -1 on launch error.
int launch_stencil_tb2(const DevFields& F, const void* h, const float* p_in, float* p_out,
                       const LaunchArgs& a, const GosaSink& g, cudaStream_t s, int sms) {
  const TmaState* t = static_cast<const TmaState*>(h);
  if (!t || (p_in != t->p && p_in != t->scratch)) return 0;
  const int i_lo = a.li_lo, i_hi = a.li_hi, j_lo = 1, j_hi = a.jmax - 1, k_lo = 1,
            k_hi = a.kmax - 1;
  // full grid only (a slab's halo would need two planes per exchange)
  if (a.i_off != 0 || i_lo != 1 || i_hi != a.imax - 1) return 0;
  if (i_hi <= i_lo || j_hi <= j_lo || k_hi <= k_lo) return 0;
  Tb2Maps maps = t->tb2;
  if (p_in == t->scratch) maps.pin = t->tb2_scratch;
  const int ktiles = (k_hi + TK - 1) / TK;
  const int jtiles = (j_hi - j_lo + TJ2 - 1) / TJ2;
  const int chunk = chunk_planes();
  const long long units = (long long)ktiles * jtiles * ((i_hi - i_lo + chunk - 1) / chunk);
  long long grid = sms;
  if (grid > units) grid = units;
  if (grid > g.capacity) return -1;
  const size_t smem = 128 + (size_t)kTb2Smem + 2 * (SP + SC) * sizeof(uint64_t) +
                      sizeof(UnitRing);
  if (cudaMemsetAsync(g.work, 0, sizeof(unsigned int), s) != cudaSuccess) return -1;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(k_stencil_tb2, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
      return -1;
    attr = true;
  }
  k_stencil_tb2<<<(int)grid, kThreads2, smem, s>>>(maps, F, p_out, i_lo, i_hi, j_lo, j_hi, k_lo,
                                                   k_hi, ktiles, chunk, a.omega, g,
                                                   a.gosa_reset);
  return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

}  // namespace hp
