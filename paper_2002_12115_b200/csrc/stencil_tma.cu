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

#include <algorithm>
#include <array>
#include <atomic>
#include <functional>
#include <map>
#include <mutex>
#include <queue>
#include <vector>
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
// planes per work unit of the single-step kernel: 32 (measured,
// profiles/r01_chunk_sweep.txt); HIMENO_CHUNK overrides it for sweeps.  The
// two-step kernel chooses its own (tb2_choose).
static int chunk_planes(int dflt) {
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("HIMENO_CHUNK");
    env = e ? atoi(e) : 0;
  }
  return env > 0 ? env : dflt;
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

// Work units, handed out by the device-wide queue (tma.cuh) in unit order.  The
// first `full` units are whole tile columns (every plane of tiles 0..full-1);
// the rest are (plane chunk, tile) pairs of the remaining tiles in chunk-major
// order.  Either way the CTAs resident together stream neighbouring tiles over
// the same planes at the same time, so the halo rows a tile shares with its
// neighbours are served from L2, and a whole column pays no chunk boundary
// (the two extra planes a unit loads and computes).
// Two-range mode (r2_hi > r2_lo, two-step kernel only): exactly two plane ranges per
// tile, [0, ni) and [r2_lo, r2_hi) relative to i_lo -- a slab's two boundary plane
// pairs in one launch (decomp.cpp, halo exchange overlapped with the interior).
// Boundary-prefix mode (sw > 0, two-step kernel, decomp.cpp): the first 2 * tiles units
// are the slab's boundary plane blocks [0, sw) and [ni - sw, ni) of every tile -- what the
// neighbouring slabs need -- and the usual whole-column / chunk units follow over the
// interior [sw, ni - sw).  One launch; the boundary units signal as they finish.
struct Units {
  int ni, ktiles, tiles, len, full;
  uint32_t count;
  int r2_lo, r2_hi;
  int sw;        // boundary-prefix width (planes), 0 = off
  uint32_t nb;   // boundary units (2 * tiles when sw > 0)
  __device__ Units(int ni_, int ktiles_, int tiles_, int len_, int full_, int r2_lo_ = 0,
                   int r2_hi_ = 0, int sw_ = 0)
      : ni(ni_), ktiles(ktiles_), tiles(tiles_), len(len_), full(r2_hi_ > r2_lo_ ? 0 : full_),
        count(r2_hi_ > r2_lo_
                  ? (uint32_t)(2 * tiles_)
                  : (uint32_t)((sw_ > 0 ? 2 * tiles_ : 0) + full_ +
                               (tiles_ - full_) * ((ni_ - 2 * sw_ + len_ - 1) / len_))),
        r2_lo(r2_lo_), r2_hi(r2_hi_), sw(sw_), nb(sw_ > 0 ? (uint32_t)(2 * tiles_) : 0u) {}
  __device__ void decode(uint32_t u, Unit& s) const {
    int t, c;
    if (r2_hi > r2_lo) {
      t = (int)(u % (uint32_t)tiles);
      c = (int)(u / (uint32_t)tiles);
      s.ia = c ? r2_lo : 0;
      s.ib = c ? r2_hi : ni;
    } else if (u < nb) {
      t = (int)(u % (uint32_t)tiles);
      c = (int)(u / (uint32_t)tiles);
      s.ia = c ? ni - sw : 0;
      s.ib = c ? ni : sw;
    } else if (u - nb < (uint32_t)full) {
      t = (int)(u - nb);
      s.ia = sw;
      s.ib = ni - sw;
    } else {
      const uint32_t v = u - nb - (uint32_t)full, rest = (uint32_t)(tiles - full);
      t = full + (int)(v % rest);
      c = (int)(v / rest);
      s.ia = sw + c * len;
      s.ib = min(ni - sw, s.ia + len);
    }
    s.kt = t % ktiles;
    s.jt = t / ktiles;
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
  __shared__ double unit_part[TJ];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ni = i_hi - i_lo;
  const int jtiles = (j_hi - j_lo + TJ - 1) / TJ;
  const Units units(ni, ktiles, ktiles * jtiles, chunk, 0);

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
      units.decode(u % units.count, s);
      const int pass = (int)(u / units.count);
      (void)pass;
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
      unit_partial(g, u, acc, unit_part, warp, TJ, 1);
      acc = 0.0;
    }
  }
  gosa_commit_units(g, units.count, reset);
}

// ================================================================ two-step kernel
//
// k_stencil_tb2<LW>: two Jacobi iterations per pass (temporal blocking).  A row
// of a tile is LW lanes x 4 floats = QK columns; a warp carries RPW = 32/LW rows
// (LW = 32: one row per warp, QK = 128; LW = 16: two rows per warp, QK = 64).
// Step 1 computes p1 = S(p0) on R1 = 8*RPW rows x QK columns (k0-4 ..
// k0+QK-5: one float4 quad per lane, uniform SIMT, no scalar halo path); step 2
// computes p2 = S(p1) one plane behind on the TJ2 = R1-2 inner rows, lanes
// 1..LW-2 of each row (the edge lanes only carry the k halo), TK2 = QK-8 output
// columns.  The 12 coefficient arrays are read from HBM once for both
// iterations: 56 B per point per TWO iterations.
//
//   producer warp: p0 plane tiles (QK+8 k x R1+2 j) into an SP-slot ring and the
//     coefficient tiles (QK k x R1 j, 12 arrays) into an SC-slot ring; work units
//     from the device-wide queue (as k_stencil_tma).
//   step-1 warps (8): register queue of p0 rows; non-interior points copy p0
//     (boundaries are fixed); p1 quad -> SQ-slot smem ring (per-thread arrivals).
//   step-2 warps (TJ2/RPW): register queue of p1 rows (k+-1 by shuffles);
//     coefficients of plane m-1 still resident in the ring.
// The narrow variant (LW = 16: 56 x 14 output points per 64 x 16 step-1 tile)
// has less halo work per output than the wide one (120 x 6 per 128 x 8) and
// fits the Himeno k extents (254, 510, 1022) with less tail waste.
// Every product/sum rounds exactly like the single-step kernel: p2 is
// bit-identical to two single steps; gosa (fp64) is that of the second step.
constexpr int SP = 3, SQ = 4;  // p0 / p1 ring slots
#ifndef HP_TB2_ROW_LDS
#define HP_TB2_ROW_LDS 1
#endif

// LW lanes per row, NW1_ step-1 warps, SC_ coefficient ring slots
template <int LW, int NW1_ = 8, int SC_ = 4>
struct Tb2 {
  static constexpr int RPW = 32 / LW;          // rows per warp
  static constexpr int NW1 = NW1_;             // step-1 warps
  static constexpr int SC = SC_;               // coefficient ring slots
  static constexpr int R1 = NW1 * RPW;         // step-1 rows
  static constexpr int TJ2 = R1 - 2;           // output rows per tile
  static constexpr int NW2 = TJ2 / RPW;        // step-2 warps
  static constexpr int QK = LW * 4;            // step-1 columns per tile
  static constexpr int TK2 = QK - 8;           // output columns per tile
  static constexpr int PW0 = QK + 8;           // p0 tile row: k0-8 .. k0+QK-1
  static constexpr int kThreads = (NW1 + NW2 + 1) * 32;
  static constexpr uint32_t kP0Bytes = PW0 * (R1 + 2) * 4;
  static constexpr uint32_t kP0Slot = (kP0Bytes + 127) / 128 * 128;
  static constexpr uint32_t kCExtBytes = QK * R1 * 4;        // one coefficient array
  static constexpr uint32_t kCSlot = NCOEF * kCExtBytes;
  static constexpr uint32_t kP1Slot = QK * R1 * 4;
  static constexpr uint32_t kSmem = SP * kP0Slot + SC * kCSlot + SQ * kP1Slot;
  static_assert(TJ2 % RPW == 0, "output rows must split evenly over step-2 warps");
  // rings + barriers / unit ring / alignment pad + the static gosa scratch <= 227 KB
  static_assert(kSmem + 2560 <= 232448, "rings exceed the 227 KB of shared memory");
  static constexpr size_t smem_bytes() {
    return 128 + (size_t)kSmem + 2 * (SP + SC + SQ) * sizeof(uint64_t) + sizeof(UnitRing);
  }
};

constexpr int kTb2Shapes = 4;

struct __align__(64) Tb2Maps {
  CUtensorMap coef[NCOEF];   // box QK x R1, origin (k0-4, j0-1)
  CUtensorMap pin;           // box QK+8 x (R1+2), origin (k0-8, j0-2): input of even passes
  CUtensorMap pin2;          // the same over the other buffer: input of odd passes (flow)
};

// Several two-step passes in one launch ("flow"): the unit queue is pass-major and
// a unit of pass t (t >= 1) starts once the pass t-1 units of its 3 x 3 tile
// neighbourhood that cover its planes +-2 have completed (per-unit completion tags):
// pass t+1 overlaps the tail of pass t instead of waiting for the whole grid.  The
// dependencies of a unit are claimed before it (pass-major order) by running CTAs,
// so every wait ends.  passes == 1: one classic pass (no tags).
struct Flow {
  int passes;          // two-step passes in this launch
  int upp;             // units per pass
  float* out[2];       // pass t writes out[t & 1] (and reads the other buffer)
  unsigned* done;      // [upp]: unit v of pass t complete <=> done[v] >= tag0 + t + 1
  unsigned tag0;       // launch epoch * 4096
  int split;           // boundary-prefix width (planes) of a signalled slab pass, 0 = off
  unsigned* sig;       // incremented once per finished boundary unit (split > 0)
};

// p0 tile row (PW0 floats): sub-lane quad at column 4 + 4*hl (k0-4+4*hl), edges at
// 3 / QK+4; shuffles stay within the LW-lane segment of the row
template <int LW>
__device__ __forceinline__ Row load_row0(const float* ptile, int row, int hl) {
  constexpr int QK = LW * 4;
  const float* base = ptile + row * (QK + 8);
  Row r;
  r.v = *reinterpret_cast<const float4*>(base + 4 + hl * 4);
#if HP_TB2_ROW_LDS
  // k-1 / k+4 straight from the tile row (the halo columns are in it): two loads,
  // no shuffles or edge predicates
  r.left = base[3 + hl * 4];
  r.right = base[8 + hl * 4];
#else
  r.left = __shfl_up_sync(0xffffffffu, r.v.w, 1, LW);
  r.right = __shfl_down_sync(0xffffffffu, r.v.x, 1, LW);
  if (hl == 0) r.left = base[3];
  if (hl == LW - 1) r.right = base[4 + QK];
#endif
  return r;
}
// p1 tile row (QK floats): k+-1 by shuffles only (edge lanes never output)
template <int LW>
__device__ __forceinline__ Row load_row1(const float* ptile, int row, int hl) {
  Row r;
  r.v = *reinterpret_cast<const float4*>(ptile + row * (LW * 4) + hl * 4);
  r.left = __shfl_up_sync(0xffffffffu, r.v.w, 1, LW);
  r.right = __shfl_down_sync(0xffffffffu, r.v.x, 1, LW);
  return r;
}

// ss for the 4 elements of a lane quad, coefficients streamed term by term
// from the shared-memory tile (ct = tile row base + lane quad, CS = stride
// between the coefficient arrays); same order of operations per element as the
// C program.
template <int CS>
__device__ __forceinline__ void ss_quad(const float* ct, const Row& lm, const Row& l0,
                                        const Row& lp, const Row& mm, const Row& m0,
                                        const Row& mp, const Row& nm, const Row& n0,
                                        const Row& np, float (&ss)[4]) {
  auto Q = [&](int c) { return *reinterpret_cast<const float4*>(ct + c * CS); };
  float s0[4];
  {
    const float4 q = Q(CA0);
#pragma unroll
    for (int x = 0; x < 4; ++x) s0[x] = fmul(el(q, x), el(n0.v, x));
  }
  {
    const float4 q = Q(CA1);
#pragma unroll
    for (int x = 0; x < 4; ++x) s0[x] = fadd(s0[x], fmul(el(q, x), el(mp.v, x)));
  }
  {
    const float4 q = Q(CA2);
#pragma unroll
    for (int x = 0; x < 4; ++x) s0[x] = fadd(s0[x], fmul(el(q, x), kp1(m0, x)));
  }
  {
    const float4 q = Q(CB0);
#pragma unroll
    for (int x = 0; x < 4; ++x)
      s0[x] = fadd(s0[x], fmul(el(q, x), fadd(fsub(fsub(el(np.v, x), el(nm.v, x)), el(lp.v, x)),
                                              el(lm.v, x))));
  }
  {
    const float4 q = Q(CB1);
#pragma unroll
    for (int x = 0; x < 4; ++x)
      s0[x] = fadd(s0[x], fmul(el(q, x), fadd(fsub(fsub(kp1(mp, x), kp1(mm, x)), km1(mp, x)),
                                              km1(mm, x))));
  }
  {
    const float4 q = Q(CB2);
#pragma unroll
    for (int x = 0; x < 4; ++x)
      s0[x] = fadd(s0[x], fmul(el(q, x), fadd(fsub(fsub(kp1(n0, x), kp1(l0, x)), km1(n0, x)),
                                              km1(l0, x))));
  }
  {
    const float4 q = Q(CC0);
#pragma unroll
    for (int x = 0; x < 4; ++x) s0[x] = fadd(s0[x], fmul(el(q, x), el(l0.v, x)));
  }
  {
    const float4 q = Q(CC1);
#pragma unroll
    for (int x = 0; x < 4; ++x) s0[x] = fadd(s0[x], fmul(el(q, x), el(mm.v, x)));
  }
  {
    const float4 q = Q(CC2);
#pragma unroll
    for (int x = 0; x < 4; ++x) s0[x] = fadd(s0[x], fmul(el(q, x), km1(m0, x)));
  }
  {
    const float4 q = Q(CW1);
#pragma unroll
    for (int x = 0; x < 4; ++x) s0[x] = fadd(s0[x], el(q, x));
  }
  const float4 a3 = Q(CA3), bn = Q(CBN);
#pragma unroll
  for (int x = 0; x < 4; ++x) ss[x] = fmul(fsub(fmul(s0[x], el(a3, x)), el(m0.v, x)), el(bn, x));
}

// Paired fp32 (sm_100 FMUL2 / FADD2): two lanes of a quad per instruction, each
// rounded separately -- bit-identical to the scalar ops.  ptxas contracts an
// f32x2 multiply feeding an f32x2 add into FFMA2 even with --fmad=false (measured:
// scratch probe, 25% of results differ), so products only ever feed scalar adds
// here, and f32x2 adds only combine loaded values.
__device__ __forceinline__ unsigned long long pk2(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 up2(unsigned long long r) {
  float2 v;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
  return v;
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk2(a.x, a.y)), "l"(pk2(b.x, b.y)));
  return up2(r);
}
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk2(a.x, a.y)), "l"(pk2(b.x, b.y)));
  return up2(r);
}
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
  unsigned long long r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk2(a.x, a.y)), "l"(pk2(b.x, b.y)));
  return up2(r);
}
__device__ __forceinline__ float2 lo2(const float4& v) { return make_float2(v.x, v.y); }
__device__ __forceinline__ float2 hi2(const float4& v) { return make_float2(v.z, v.w); }

// ss for a lane quad with paired products of the unshifted terms (a0, a1, b0, c0,
// c1, a3, bnd); same per-element order of operations as ss_quad.
template <class QF>
__device__ __forceinline__ void ss_quad2q(const QF& Q, const Row& lm, const Row& l0,
                                          const Row& lp, const Row& mm, const Row& m0,
                                          const Row& mp, const Row& nm, const Row& n0,
                                          const Row& np, float (&ss)[4]) {
  float s0[4];
  auto acc2 = [&](float2 p01, float2 p23) {   // s0 += products (scalar adds)
    s0[0] = fadd(s0[0], p01.x);
    s0[1] = fadd(s0[1], p01.y);
    s0[2] = fadd(s0[2], p23.x);
    s0[3] = fadd(s0[3], p23.y);
  };
  {
    const float4 q = Q(CA0);
    const float2 p01 = mul2(lo2(q), lo2(n0.v)), p23 = mul2(hi2(q), hi2(n0.v));
    s0[0] = p01.x; s0[1] = p01.y; s0[2] = p23.x; s0[3] = p23.y;
  }
  {
    const float4 q = Q(CA1);
    acc2(mul2(lo2(q), lo2(mp.v)), mul2(hi2(q), hi2(mp.v)));
  }
  {
    const float4 q = Q(CA2);
#pragma unroll
    for (int x = 0; x < 4; ++x) s0[x] = fadd(s0[x], fmul(el(q, x), kp1(m0, x)));
  }
  {
    const float4 q = Q(CB0);
    const float2 t01 = add2(sub2(sub2(lo2(np.v), lo2(nm.v)), lo2(lp.v)), lo2(lm.v));
    const float2 t23 = add2(sub2(sub2(hi2(np.v), hi2(nm.v)), hi2(lp.v)), hi2(lm.v));
    acc2(mul2(lo2(q), t01), mul2(hi2(q), t23));
  }
  {
    const float4 q = Q(CB1);
#pragma unroll
    for (int x = 0; x < 4; ++x)
      s0[x] = fadd(s0[x], fmul(el(q, x), fadd(fsub(fsub(kp1(mp, x), kp1(mm, x)), km1(mp, x)),
                                              km1(mm, x))));
  }
  {
    const float4 q = Q(CB2);
#pragma unroll
    for (int x = 0; x < 4; ++x)
      s0[x] = fadd(s0[x], fmul(el(q, x), fadd(fsub(fsub(kp1(n0, x), kp1(l0, x)), km1(n0, x)),
                                              km1(l0, x))));
  }
  {
    const float4 q = Q(CC0);
    acc2(mul2(lo2(q), lo2(l0.v)), mul2(hi2(q), hi2(l0.v)));
  }
  {
    const float4 q = Q(CC1);
    acc2(mul2(lo2(q), lo2(mm.v)), mul2(hi2(q), hi2(mm.v)));
  }
  {
    const float4 q = Q(CC2);
#pragma unroll
    for (int x = 0; x < 4; ++x) s0[x] = fadd(s0[x], fmul(el(q, x), km1(m0, x)));
  }
  {
    const float4 q = Q(CW1);
#pragma unroll
    for (int x = 0; x < 4; ++x) s0[x] = fadd(s0[x], el(q, x));
  }
  const float4 a3 = Q(CA3), bn = Q(CBN);
  // ss = (s0 * a3 - p) * bnd: product -> scalar sub -> paired product
  const float2 u01 = mul2(make_float2(s0[0], s0[1]), lo2(a3));
  const float2 u23 = mul2(make_float2(s0[2], s0[3]), hi2(a3));
  const float2 d01 = make_float2(fsub(u01.x, m0.v.x), fsub(u01.y, m0.v.y));
  const float2 d23 = make_float2(fsub(u23.x, m0.v.z), fsub(u23.y, m0.v.w));
  const float2 r01 = mul2(d01, lo2(bn)), r23 = mul2(d23, hi2(bn));
  ss[0] = r01.x; ss[1] = r01.y; ss[2] = r23.x; ss[3] = r23.y;
}
// coefficients streamed from the shared-memory tile (ct = tile row + lane quad, CS =
// stride between the coefficient arrays)
template <int CS>
__device__ __forceinline__ void ss_quad2(const float* ct, const Row& lm, const Row& l0,
                                         const Row& lp, const Row& mm, const Row& m0,
                                         const Row& mp, const Row& nm, const Row& n0,
                                         const Row& np, float (&ss)[4]) {
  auto Q = [&](int c) { return *reinterpret_cast<const float4*>(ct + c * CS); };
  ss_quad2q(Q, lm, l0, lp, mm, m0, mp, nm, n0, np, ss);
}

// ---- tensor memory as a per-thread stash (two-step kernel, ST variant): 32x32b
// shapes, so thread t of warp w owns TMEM lane 32*(w%4)+t; address (lane<<16)|col
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t cols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "r"(cols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t base, uint32_t cols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "r"(cols)
               : "memory");
}
// 16 consecutive columns of this thread's lane
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16};" ::"r"(taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]),
      "f"(v[8]), "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15])
      : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15}, [%16];"
      : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]),
        "=f"(v[7]), "=f"(v[8]), "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]),
        "=f"(v[14]), "=f"(v[15])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// wait for this thread's tcgen05.ld results; the registers are in/out operands so no
// use of them can be scheduled above the wait
__device__ __forceinline__ void tmem_wait_ld24(float* v) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+f"(v[0]), "+f"(v[1]), "+f"(v[2]), "+f"(v[3]), "+f"(v[4]), "+f"(v[5]),
                 "+f"(v[6]), "+f"(v[7]), "+f"(v[8]), "+f"(v[9]), "+f"(v[10]), "+f"(v[11]),
                 "+f"(v[12]), "+f"(v[13]), "+f"(v[14]), "+f"(v[15]), "+f"(v[16]), "+f"(v[17]),
                 "+f"(v[18]), "+f"(v[19]), "+f"(v[20]), "+f"(v[21]), "+f"(v[22]), "+f"(v[23])
               :
               : "memory");
}
__device__ __forceinline__ void tmem_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// End of a unit for the step-2 warps of a two-step kernel: the gosa partial of the
// last pass's units (only the last iteration's gosa is observable), and in a flow
// launch the unit's completion tag, published after every step-2 thread's stores
// (named barrier, then a gpu-scope fence by the publishing thread).
__device__ void unit_finish(const GosaSink& g, uint32_t u, uint32_t upp, const Flow& fl, double v,
                            double* part, int wrel, int nw, int bar) {
  const uint32_t pass = u / upp, local = u % upp;
  if ((int)pass == fl.passes - 1) {
    unit_partial(g, local, v, part, wrel, nw, bar);
  } else {
    named_bar_sync(bar, nw * 32);
  }
  if (fl.passes > 1 && wrel == 0 && (threadIdx.x & 31) == 0) {
    __threadfence();
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(fl.done + local),
                 "r"(fl.tag0 + pass + 1u)
                 : "memory");
  }
}
// A boundary unit of a signalled slab pass is written: count it.  The halo exchange's
// stream waits for the count (cuStreamWaitValue32) and then copies / sends the planes, so
// the stores must be visible beyond the SMs (copy engines, NCCL): system-scope fence.
// Called by every step-2 thread after unit_finish's named barrier.
__device__ __forceinline__ void boundary_signal(const Flow& fl, bool boundary, int wrel, int nw,
                                                int bar) {
  if (!fl.sig || !boundary) return;
  named_bar_sync(bar, nw * 32);   // every step-2 warp's stores of the unit are issued
  if (wrel == 0 && (threadIdx.x & 31) == 0) {
    __threadfence_system();
    atomicAdd_system(fl.sig, 1u);
  }
}

// CPOL_ is a bit set of variants (instantiations: 0, 1, 4, 12, 13):
//   1  the coefficient TMA loads carry an L2 evict_first policy.  The flow launch
//      (several passes in flight, small grids) runs 2.7 % faster with it on M; on L, whose
//      step-1 halo lines must survive in L2 until the neighbouring tile reads them, it
//      costs 28 % (profiles/r02_flow.md), so per-pass launches go without (no hint at
//      all: an evict_normal hint already costs 0.7 %).
//   4  cross-warp stash (XS, below): step 1 hands the step-2 coefficients over in TMEM.
//   8  (with 4) coefficients-first producer order and late p0 release (ORD, below).
template <int LW, int NW1_, int SC_, bool ST_ = false, int CPOL_ = 0>
__global__ void __launch_bounds__(Tb2<LW, NW1_, SC_>::kThreads, 1)
k_stencil_tb2(const __grid_constant__ Tb2Maps maps, DevFields F, int i_lo, int i_hi, int j_lo,
              int j_hi, int k_lo, int k_hi, int k_org, int ktiles, int chunk, int full, int g_lo,
              int g_hi, float omega, GosaSink g, int reset, Flow fl, int i_lo2, int i_hi2) {
  using T = Tb2<LW, NW1_, SC_>;
  constexpr int RPW = T::RPW, NW1 = T::NW1, NW2 = T::NW2, R1 = T::R1, TJ2 = T::TJ2,
                QK = T::QK, TK2 = T::TK2, SC = T::SC;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  unsigned char* p0ring = smem;
  unsigned char* cring = p0ring + SP * T::kP0Slot;
  float* p1ring = reinterpret_cast<float*>(cring + SC * T::kCSlot);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + T::kSmem);
  uint64_t* pfull = bars;
  uint64_t* pempty = pfull + SP;
  uint64_t* cfull = pempty + SP;
  uint64_t* cempty = cfull + SC;
  uint64_t* qfull = cempty + SC;
  uint64_t* qempty = qfull + SQ;
  UnitRing* ring = reinterpret_cast<UnitRing*>(qempty + SQ);
  __shared__ double unit_part[NW2];
  __shared__ uint32_t tmem_base_s;   // ST: tensor-memory stash of the step-2 coefficients
  // CPOL_ & 4 (XS, "cross-warp stash"): the step-1 warps, which load every coefficient
  // quad from shared memory anyway, write the quads of rows 1..14 into tensor memory and
  // the step-2 warps read them from there -- no second shared-memory read of the
  // coefficients.  Step-1 warp w < 7 takes rows 2w+1, 2w+2 (warp 7 the halo rows 0 and
  // 15), so step-2 warp w2 needs exactly step-1 warp w2's quads, in the same TMEM lanes
  // (warps 8+w2 and w2 share the lane quarter w2 % 4).  Five stash slots per plane ring.
  constexpr bool XS = (CPOL_ & 4) != 0;
  // CPOL_ & 8 (with XS): the producer issues plane m's coefficients before p0(m+1) and
  // step 1 releases the p0 slot together with the coefficient stage, after both loads
  // are in flight (one load-latency stall less per plane).  It lets the columns drift
  // further apart, so it is used where L2 holds many planes (M, L), not on XL
  // (profiles/r02_tb2_experiments_late.md).
  constexpr bool ORD = XS && (CPOL_ & 8) != 0;
  constexpr bool LATE_P = ORD;
  constexpr uint32_t kStashCols = XS ? 512 : 256;
  constexpr int kXSlots = 5;
  static_assert(!ST_ || (NW1 % 4 == 0 && NW2 <= 8), "stash: (warp%4, block) per step-2 warp");
  static_assert(!XS || (ST_ && NW1 == 8 && RPW == 2 && NW2 == 7 && SQ == 4),
                "cross-warp stash: shape (16, 8, 4) with the p1 ring of 4 (WAR via qempty)");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int hl = lane % LW, half = lane / LW;   // lane within the row, row within the warp
  const int ni = i_hi - i_lo;
  const int jtiles = (j_hi - j_lo + TJ2 - 1) / TJ2;
  const Units units(ni, ktiles, ktiles * jtiles, chunk, full, i_lo2 - i_lo, i_hi2 - i_lo, fl.split);
  const uint32_t nunits = units.count * (uint32_t)fl.passes;   // queue: pass-major
  if (threadIdx.x == 0) {
    for (int s = 0; s < SP; ++s) { mbar_init(&pfull[s], 1); mbar_init(&pempty[s], NW1); }
    for (int s = 0; s < SC; ++s) { mbar_init(&cfull[s], 1); mbar_init(&cempty[s], XS ? NW1 : NW1 + NW2); }
    // p1 ring: every thread arrives (no reliance on __syncwarp ordering for the
    // shared-memory rows written / read by other warps)
    for (int s = 0; s < SQ; ++s) { mbar_init(&qfull[s], NW1 * 32); mbar_init(&qempty[s], NW2 * 32); }
    unit_ring_init(ring, NW1 + NW2);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if constexpr (ST_) {
    if (warp == NW1) tmem_alloc(&tmem_base_s, kStashCols);
    tmem_fence_before();
  }
  __syncthreads();
  if constexpr (ST_) tmem_fence_after();
  // launched with programmatic stream serialization: the next pass may be
  // scheduled as SMs free up, but nothing global (queue counter, fields, gosa)
  // is touched before the previous grid has completed and flushed
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  double acc = 0.0;
  if (warp == NW1 + NW2) {
    // ------------------------------------------------------------- producer
    // lane 0 claims units and issues the TMA loads; in a flow launch the whole warp
    // first waits for the unit's dependencies (one completion tag per lane)
    uint64_t cpolicy = 0;
    if constexpr ((CPOL_ & 1) != 0)
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(cpolicy));
    uint32_t sp = 0, sc = 0;
    Unit s{0, 0, 0, 0};
    for (uint32_t n = 0;; ++n) {
      uint32_t u = 0;
      if (lane == 0) u = unit_publish(ring, n, g.work, nunits);
      u = __shfl_sync(0xffffffffu, u, 0);
      if (u == kNoUnit) break;
      const int pass = (int)(u / units.count);
      units.decode(u % units.count, s);
      if (pass > 0) {
        // lane l: neighbour tile l / 3 of the 3 x 3 block, l % 3-th plane chunk
        // overlapping [ia-2, ib+2) (planes the step-1 box reads, and the planes this
        // unit overwrites in the buffer the previous pass read)
        const int d = lane / 3, co = lane % 3;
        if (d < 9) {
          const int jn = s.jt + d / 3 - 1, kn = s.kt + d % 3 - 1;
          if (jn >= 0 && jn < jtiles && kn >= 0 && kn < ktiles) {
            const int tn = jn * ktiles + kn;
            int v = -1;
            if (tn < units.full) {
              if (co == 0) v = tn;
            } else {
              const int c_lo = max(0, s.ia - 2) / units.len;
              const int c_hi = min(ni - 1, s.ib + 1) / units.len;
              if (c_lo + co <= c_hi)
                v = units.full + (c_lo + co) * (units.tiles - units.full) + (tn - units.full);
            }
            if (v >= 0) {
              const unsigned want = fl.tag0 + (unsigned)pass;   // pass - 1 complete
              uint32_t polls = 0;
              while (ld_acquire_u32(fl.done + v) < want) {
                if (++polls > (1u << 26)) asm volatile("trap;");
              }
            }
          }
        }
        __syncwarp();
        // the previous pass's generic-proxy stores before this CTA's TMA (async
        // proxy) reads of them
        asm volatile("fence.proxy.async.global;" ::: "memory");
      }
      if (lane == 0) {
        const int ia = i_lo + s.ia, ib = i_lo + s.ib;
        const int k0 = k_org + s.kt * TK2, j0 = j_lo + s.jt * TJ2;
        const CUtensorMap* pin = (pass & 1) ? &maps.pin2 : &maps.pin;
        auto load_p0 = [&](int plane) {
          const int slot = sp % SP;
          if (sp >= (uint32_t)SP) mbar_wait(&pempty[slot], ((sp / SP) - 1) & 1);
          mbar_expect_tx(&pfull[slot], T::kP0Bytes);
          tma_load_3d(p0ring + slot * T::kP0Slot, pin, &pfull[slot], k0 - 8, j0 - 2, plane);
          ++sp;
        };
        load_p0(ia - 2);
        load_p0(ia - 1);
        for (int m = ia - 1; m <= ib; ++m) {
          if constexpr (!ORD) load_p0(m + 1);
          const int slot = sc % SC;
          if (sc >= (uint32_t)SC) mbar_wait(&cempty[slot], ((sc / SC) - 1) & 1);
          if ((CPOL_ & 1) == 0 && (m < g_lo || m >= g_hi)) {
            // one-pass launches: a plane outside the global interior carries no data (step
            // 1 computes nothing there, step 2 has no output plane); a plain arrive
            // completes the stage
            ++sc;
            mbar_arrive(&cfull[slot]);
            if constexpr (ORD) load_p0(m + 1);
            continue;
          }
          mbar_expect_tx(&cfull[slot], NCOEF * T::kCExtBytes);
          for (int c = 0; c < NCOEF; ++c) {
            if constexpr ((CPOL_ & 1) != 0)
              tma_load_3d_hint(cring + slot * T::kCSlot + c * T::kCExtBytes, &maps.coef[c],
                               &cfull[slot], k0 - 4, j0 - 1, m, cpolicy);
            else
              tma_load_3d(cring + slot * T::kCSlot + c * T::kCExtBytes, &maps.coef[c], &cfull[slot],
                          k0 - 4, j0 - 1, m);
          }
          ++sc;
          // ORD: plane m's coefficients go out before p0(m+1), so a p0 slot still held
          // by step 1 (released with the coefficient stage) delays only the next p0 box
          if constexpr (ORD) load_p0(m + 1);
        }
      }
      __syncwarp();
    }
  } else if (warp < NW1) {
    // ------------------------------------- step-1 warps (tile row r = j0-1+r)
    const int r = XS ? (warp < NW1 - 1 ? 2 * warp + 1 + half : (half ? R1 - 1 : 0)) : warp * RPW + half;
    [[maybe_unused]] const uint32_t xs_tl =
        tmem_base_s + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * (kXSlots * 48));
    uint32_t sc = 0, sq = 0;
    int pslot = 0;          // p0 ring position, advanced incrementally (SP = 3 is not a
    uint32_t pphase = 0;    // power of two: no division per plane)
    Unit s;
    for (uint32_t n = 0;; ++n) {
      const uint32_t u = unit_take(ring, n, lane);
      if (u == kNoUnit) break;
      units.decode(u % units.count, s);
      const int pass = (int)(u / units.count);
      (void)pass;
      const int ia = i_lo + s.ia, ib = i_lo + s.ib;
      const int k0 = k_org + s.kt * TK2, j0 = j_lo + s.jt * TJ2;
      const int j1 = j0 - 1 + r;
      const int kq = k0 - 4 + hl * 4;
      const bool row_in = j1 >= j_lo && j1 < j_hi;
      bool in1[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) in1[x] = row_in && kq + x >= k_lo && kq + x < k_hi;
      Row am, a0, ap, bm, b0, bp;
      auto next_p = [&]() {
        if (++pslot == SP) {
          pslot = 0;
          pphase ^= 1u;
        }
      };
      for (int w = 0; w < 2; ++w) {
        const int slot = pslot;
        mbar_wait(&pfull[slot], pphase);
        const float* pt = reinterpret_cast<const float*>(p0ring + slot * T::kP0Slot);
        const Row x0 = load_row0<LW>(pt, r, hl), x1 = load_row0<LW>(pt, r + 1, hl),
                  x2 = load_row0<LW>(pt, r + 2, hl);
        __syncwarp();
        if (lane == 0) mbar_arrive(&pempty[slot]);
        if (w == 0) { am = x0; a0 = x1; ap = x2; } else { bm = x0; b0 = x1; bp = x2; }
        next_p();
      }
#pragma unroll 1
      for (int m = ia - 1; m <= ib; ++m) {
        const int cur = pslot;
        mbar_wait(&pfull[cur], pphase);
        const float* pt = reinterpret_cast<const float*>(p0ring + cur * T::kP0Slot);
        const Row cm = load_row0<LW>(pt, r, hl), c0 = load_row0<LW>(pt, r + 1, hl),
                  cp = load_row0<LW>(pt, r + 2, hl);
        // flow launches (XS with evict_first): the p0 slot is released together with the
        // coefficient stage, after both stages' loads are in flight (M -2.4 % per pass);
        // per-pass launches release it here, so the producer -- which issues p0(m+1)
        // before the coefficients of plane m -- is not held behind the cfull wait (XL +1.2 %
        // with the late release)
        if constexpr (!LATE_P) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&pempty[cur]);
        }
        next_p();
        const int cslot = sc % SC;
        mbar_wait(&cfull[cslot], (sc / SC) & 1);
        const float* ct = reinterpret_cast<const float*>(cring + cslot * T::kCSlot) + r * QK + hl * 4;
        // planes of the global interior (local indices): in a slab, step 1 also
        // recomputes the neighbours' adjacent planes (two-plane halos)
        const bool plane_in = m >= g_lo && m < g_hi;
        float v[4];
        if constexpr (XS) {
          // p1 ring slot and stash slot of this plane free (qempty: step 2 finished the
          // iteration that read the stash slot's previous plane), then the quads: shared
          // memory -> registers -> tensor memory (planes that carry an output plane)
          const int qslot = sq % SQ;
          if (sq >= (uint32_t)SQ) mbar_wait(&qempty[qslot], ((sq / SQ) - 1) & 1);
          tmem_fence_after();
          float cv[48];
#pragma unroll
          for (int c = 0; c < NCOEF; ++c) {
            const float4 q = *reinterpret_cast<const float4*>(ct + c * (QK * R1));
            cv[4 * c] = q.x; cv[4 * c + 1] = q.y; cv[4 * c + 2] = q.z; cv[4 * c + 3] = q.w;
          }
          __syncwarp();
          if (lane == 0) {
            if constexpr (LATE_P) mbar_arrive(&pempty[cur]);
            mbar_arrive(&cempty[cslot]);
          }
          if (warp < NW1 - 1 && m >= ia && m < ib) {
            const uint32_t ta = xs_tl + (uint32_t)((sc % kXSlots) * 48);
#pragma unroll
            for (int k = 0; k < 3; ++k) {
              float t16[16];
#pragma unroll
              for (int x = 0; x < 16; ++x) t16[x] = cv[16 * k + x];
              tmem_st16(ta + 16 * k, t16);
            }
          }
          if (plane_in && row_in) {
            auto Q = [&](int c) {
              return make_float4(cv[4 * c], cv[4 * c + 1], cv[4 * c + 2], cv[4 * c + 3]);
            };
            float ss[4];
            ss_quad2q(Q, am, a0, ap, bm, b0, bp, cm, c0, cp, ss);
#pragma unroll
            for (int x = 0; x < 4; ++x) v[x] = in1[x] ? fadd(el(b0.v, x), fmul(omega, ss[x])) : el(b0.v, x);
          } else {
#pragma unroll
            for (int x = 0; x < 4; ++x) v[x] = el(b0.v, x);
          }
          ++sc;
          float* q1 = p1ring + qslot * (QK * R1);
          *reinterpret_cast<float4*>(q1 + r * QK + hl * 4) = make_float4(v[0], v[1], v[2], v[3]);
          tmem_wait_st();
          tmem_fence_before();
          mbar_arrive(&qfull[qslot]);   // release: this thread's p1 quad and stash quads
          ++sq;
        } else {
        if (plane_in && row_in) {
          float ss[4];
          ss_quad2<QK * R1>(ct, am, a0, ap, bm, b0, bp, cm, c0, cp, ss);
#pragma unroll
          for (int x = 0; x < 4; ++x) v[x] = in1[x] ? fadd(el(b0.v, x), fmul(omega, ss[x])) : el(b0.v, x);
        } else {
#pragma unroll
          for (int x = 0; x < 4; ++x) v[x] = el(b0.v, x);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&cempty[cslot]);
        ++sc;
        // p1(m) -> ring slot (wait until the step-2 warps released its last use)
        const int qslot = sq % SQ;
        if (sq >= (uint32_t)SQ) mbar_wait(&qempty[qslot], ((sq / SQ) - 1) & 1);
        float* q1 = p1ring + qslot * (QK * R1);
        *reinterpret_cast<float4*>(q1 + r * QK + hl * 4) = make_float4(v[0], v[1], v[2], v[3]);
        mbar_arrive(&qfull[qslot]);   // release: publishes this thread's quad
        ++sq;
        }
        am = bm; a0 = b0; ap = bp;
        bm = cm; b0 = c0; bp = cp;
      }
    }
  } else if constexpr (ST_) {
    // ------------------- step-2 warps, coefficients stashed in tensor memory
    // Each thread copies the 12 coefficient quads it will need for output plane m
    // into its TMEM lane as soon as the stage of plane m lands and releases the
    // stage at once; one iteration later it reads them back.  A stage is then held
    // only while step 1 works on it, and the producer runs a plane further ahead.
    const int w2 = warp - NW1;
    const int r2 = w2 * RPW + half;
    const uint32_t tl = tmem_base_s + ((uint32_t)(32 * (warp & 3)) << 16) +
                        (uint32_t)((w2 >> 2) * (XS ? kXSlots * 48 : 96));
    uint32_t sc = 0, sq = 0;
    Unit s;
    for (uint32_t n = 0;; ++n) {
      const uint32_t u = unit_take(ring, n, lane);
      if (u == kNoUnit) break;
      units.decode(u % units.count, s);
      const int pass = (int)(u / units.count);
      (void)pass;
      const int ia = i_lo + s.ia, ib = i_lo + s.ib;
      const int k0 = k_org + s.kt * TK2, j0 = j_lo + s.jt * TJ2;
      const int j = j0 + r2;
      const int kq = k0 - 4 + hl * 4;
      const bool row_in = j < j_hi;
      bool in2[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) in2[x] = row_in && kq + x >= k_lo && kq + x < k_hi;
      const bool writer = row_in && hl >= 1 && hl <= LW - 2;
      Row ym, y0, yp, zm, z0, zp;   // p1 queue: planes m-2 (y*), m-1 (z*)
#pragma unroll 1
      for (int m = ia - 1; m <= ib; ++m) {
        if constexpr (XS) {
          // the stash of plane m-1 was written by step-1 warp w2 (same lanes) before it
          // released p1(m-1); read it with p1(m), then release the p1 slot
          const int qslot = sq % SQ;
          mbar_wait(&qfull[qslot], (sq / SQ) & 1);
          tmem_fence_after();
          const float* q1 = p1ring + qslot * (QK * R1);
          const Row nm = load_row1<LW>(q1, r2, hl), n0 = load_row1<LW>(q1, r2 + 1, hl),
                    np = load_row1<LW>(q1, r2 + 2, hl);
          float cv[48];
          if (m >= ia + 1) {
            const uint32_t ta = tl + (uint32_t)(((sc - 1) % kXSlots) * 48);
#pragma unroll
            for (int k = 0; k < 3; ++k) {
              float v[16];
              tmem_ld16(ta + 16 * k, v);
#pragma unroll
              for (int x = 0; x < 16; ++x) cv[16 * k + x] = v[x];
            }
            tmem_wait_ld24(cv);
            tmem_wait_ld24(cv + 24);
          }
          tmem_fence_before();
          mbar_arrive(&qempty[qslot]);
          ++sq;
          ++sc;
          if (m >= ia + 1) {
            auto Q = [&](int c) {
              return make_float4(cv[4 * c], cv[4 * c + 1], cv[4 * c + 2], cv[4 * c + 3]);
            };
            float ss[4];
            ss_quad2q(Q, ym, y0, yp, zm, z0, zp, nm, n0, np, ss);
            float w[4];
#pragma unroll
            for (int x = 0; x < 4; ++x) {
              w[x] = fadd(el(z0.v, x), fmul(omega, ss[x]));
              if (writer && in2[x]) acc += (double)fmul(ss[x], ss[x]);
            }
            if (writer) {
              float* o = ((pass & 1) ? fl.out[1] : fl.out[0]) + F.at(m - 1, j, kq);
              if (in2[0] && in2[1] && in2[2] && in2[3]) {
                *reinterpret_cast<float4*>(o) = make_float4(w[0], w[1], w[2], w[3]);
              } else {
                for (int x = 0; x < 4; ++x)
                  if (in2[x]) o[x] = w[x];
              }
            }
          }
          ym = zm; y0 = z0; yp = zp;
          zm = nm; z0 = n0; zp = np;
          continue;
        }
        {
          const int cslot = sc % SC;
          mbar_wait(&cfull[cslot], (sc / SC) & 1);
          if (m >= ia && m < ib) {   // planes that carry an output plane
            const float* ct = reinterpret_cast<const float*>(cring + cslot * T::kCSlot) + (r2 + 1) * QK + hl * 4;
#pragma unroll
            for (int k = 0; k < 3; ++k) {
              float v[16];
#pragma unroll
              for (int c4 = 0; c4 < 4; ++c4) {
                const float4 q = *reinterpret_cast<const float4*>(ct + (4 * k + c4) * (QK * R1));
                v[4 * c4] = q.x; v[4 * c4 + 1] = q.y; v[4 * c4 + 2] = q.z; v[4 * c4 + 3] = q.w;
              }
              tmem_st16(tl + (uint32_t)((m & 1) * 48 + 16 * k), v);
            }
            tmem_wait_st();
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&cempty[cslot]);
          ++sc;
        }
        const int qslot = sq % SQ;
        mbar_wait(&qfull[qslot], (sq / SQ) & 1);
        const float* q1 = p1ring + qslot * (QK * R1);
        const Row nm = load_row1<LW>(q1, r2, hl), n0 = load_row1<LW>(q1, r2 + 1, hl),
                  np = load_row1<LW>(q1, r2 + 2, hl);
        mbar_arrive(&qempty[qslot]);
        ++sq;
        if (m >= ia + 1) {
          float cv[48];
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            float v[16];
            tmem_ld16(tl + (uint32_t)(((m - 1) & 1) * 48 + 16 * k), v);
#pragma unroll
            for (int x = 0; x < 16; ++x) cv[16 * k + x] = v[x];
          }
          tmem_wait_ld24(cv);
          tmem_wait_ld24(cv + 24);
          auto Q = [&](int c) {
            return make_float4(cv[4 * c], cv[4 * c + 1], cv[4 * c + 2], cv[4 * c + 3]);
          };
          float ss[4];
          ss_quad2q(Q, ym, y0, yp, zm, z0, zp, nm, n0, np, ss);
          float w[4];
#pragma unroll
          for (int x = 0; x < 4; ++x) {
            w[x] = fadd(el(z0.v, x), fmul(omega, ss[x]));
            if (writer && in2[x]) acc += (double)fmul(ss[x], ss[x]);
          }
          if (writer) {
            float* o = ((pass & 1) ? fl.out[1] : fl.out[0]) + F.at(m - 1, j, kq);
            if (in2[0] && in2[1] && in2[2] && in2[3]) {
              *reinterpret_cast<float4*>(o) = make_float4(w[0], w[1], w[2], w[3]);
            } else {
              for (int x = 0; x < 4; ++x)
                if (in2[x]) o[x] = w[x];
            }
          }
        }
        ym = zm; y0 = z0; yp = zp;
        zm = nm; z0 = n0; zp = np;
      }
      unit_finish(g, u, units.count, fl, acc, unit_part, warp - NW1, NW2, 1);
      boundary_signal(fl, (u % units.count) < units.nb, warp - NW1, NW2, 1);
      acc = 0.0;
    }
  } else {
    // -------------------------------------- step-2 warps (output row j0+r2)
    const int r2 = (warp - NW1) * RPW + half;
    uint32_t sc = 0, sq = 0;
    Unit s;
    for (uint32_t n = 0;; ++n) {
      const uint32_t u = unit_take(ring, n, lane);
      if (u == kNoUnit) break;
      units.decode(u % units.count, s);
      const int pass = (int)(u / units.count);
      (void)pass;
      const int ia = i_lo + s.ia, ib = i_lo + s.ib;
      const int k0 = k_org + s.kt * TK2, j0 = j_lo + s.jt * TJ2;
      const int j = j0 + r2;
      const int kq = k0 - 4 + hl * 4;
      const bool row_in = j < j_hi;
      bool in2[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) in2[x] = row_in && kq + x >= k_lo && kq + x < k_hi;
      const bool writer = row_in && hl >= 1 && hl <= LW - 2;
      Row ym, y0, yp, zm, z0, zp;   // p1 queue: planes m-2 (y*), m-1 (z*)
#pragma unroll 1
      for (int m = ia - 1; m <= ib; ++m) {
        const int qslot = sq % SQ;
        mbar_wait(&qfull[qslot], (sq / SQ) & 1);
        const float* q1 = p1ring + qslot * (QK * R1);
        const Row nm = load_row1<LW>(q1, r2, hl), n0 = load_row1<LW>(q1, r2 + 1, hl),
                  np = load_row1<LW>(q1, r2 + 2, hl);
        mbar_arrive(&qempty[qslot]);  // this thread's reads of the slot are done
        ++sq;
        // coefficient stage of plane m (sequence sc): used at iteration m+1 for
        // output plane m; stages of planes ia-1 and ib are only released
        if (m >= ia + 1) {
          const int cslot = (sc - 1) % SC;          // stage of plane m-1
          mbar_wait(&cfull[cslot], ((sc - 1) / SC) & 1);
          const float* ct = reinterpret_cast<const float*>(cring + cslot * T::kCSlot) + (r2 + 1) * QK + hl * 4;
          float ss[4];
          ss_quad2<QK * R1>(ct, ym, y0, yp, zm, z0, zp, nm, n0, np, ss);
          float w[4];
#pragma unroll
          for (int x = 0; x < 4; ++x) {
            w[x] = fadd(el(z0.v, x), fmul(omega, ss[x]));
            if (writer && in2[x]) acc += (double)fmul(ss[x], ss[x]);
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&cempty[cslot]);
          if (writer) {
            float* o = ((pass & 1) ? fl.out[1] : fl.out[0]) + F.at(m - 1, j, kq);
            if (in2[0] && in2[1] && in2[2] && in2[3]) {
              *reinterpret_cast<float4*>(o) = make_float4(w[0], w[1], w[2], w[3]);
            } else {
              for (int x = 0; x < 4; ++x)
                if (in2[x]) o[x] = w[x];
            }
          }
        } else if (m == ia) {
          // stage of plane ia-1 carries no output plane: release it unused
          if (lane == 0) mbar_arrive(&cempty[(sc - 1) % SC]);
        }
        ++sc;   // stage of plane m
        ym = zm; y0 = z0; yp = zp;
        zm = nm; z0 = n0; zp = np;
      }
      // stage of plane ib carries no output plane either
      if (lane == 0) mbar_arrive(&cempty[(sc - 1) % SC]);
      unit_finish(g, u, units.count, fl, acc, unit_part, warp - NW1, NW2, 1);
      boundary_signal(fl, (u % units.count) < units.nb, warp - NW1, NW2, 1);
      acc = 0.0;
    }
  }
  if constexpr (ST_) {
    tmem_fence_before();
    __syncthreads();
    if (warp == NW1) {
      tmem_fence_after();
      tmem_dealloc(tmem_base_s, kStashCols);
    }
  }
  gosa_commit_units(g, units.count, reset);
}

#include "stencil_tx.cuh"

// ------------------------------------------------------------------ host side

constexpr int kTxTJ = 7;   // rows per exchange tile (L: 4 x 37 tiles = 148 SMs)

struct TmaState {
  StencilMaps base;          // coefficient maps + p map
  CUtensorMap scratch_map;   // p map of the rotation buffer
  Tb2Maps tb2[kTb2Shapes];   // two-step kernel shapes: coefficient boxes + p map
  CUtensorMap tb2_scratch[kTb2Shapes];
  TxMaps tx;                 // exchange kernel: coefficient boxes 128 x TJ + p map
  CUtensorMap tx_scratch;
  const float* p;
  const float* scratch;
  // exchange buffers (k_stencil_tx), sized for this context's j/k extents
  uint2* xr = nullptr;       // tagged boundary words {value, tag}
  uint2* xc = nullptr;
  size_t nxr = 0, nxc = 0;   // words
  unsigned* err = nullptr;
  int tx_ktiles = 0, tx_jtiles = 0, tx_chunks = 0;   // capacity (0: exchange kernel off)
  unsigned epoch = 0;
  // multi-pass flow launches of k_stencil_tb2: per-unit completion tags
  unsigned* done = nullptr;
  int done_cap = 0;
  unsigned flow_epoch = 0;
  // maps whose k / j extents stop at K-1 / J-1 (HIMENO_TMA_TRIM bits: 1 two-step, 2
  // single-step, 4 exchange kernel); launches need kmax <= K-1 and jmax <= J-1
  int trim = 0;
};

}  // namespace

// integer environment knob, -1 when unset
static int env_int(const char* name) {
  const char* e = getenv(name);
  return e ? atoi(e) : -1;
}

// Build the tensor maps of one context (fields + rotation scratch); nullptr if
// the driver cannot encode them (the caller then uses k_stencil_3d).
// HIMENO_TMA_PROMO="a,b,c,d": L2 promotion codes (0 none, 1 64B, 2 128B, 3 256B)
// of the single-step coefficient / p maps and the two-step coefficient / p maps.
static void promo_codes(int* c) {
  c[0] = 2; c[1] = 2; c[2] = 2; c[3] = 2;
  if (const char* e = getenv("HIMENO_TMA_PROMO"))
    sscanf(e, "%d,%d,%d,%d", &c[0], &c[1], &c[2], &c[3]);
}

void* create_stencil_tma(const DevFields& F, const float* scratch) {
  TmaState* t = new TmaState;
  int pc[4];
  promo_codes(pc);
  // row extent the maps expose: K (columns past it are zero-filled by TMA, never
  // read) or the padded pitch P
  int dk = F.K;
  if (const char* e = getenv("HIMENO_TMA_DIMK")) dk = atoi(e) ? F.K : F.P;
  bool ok = true;
  // The program never touches column K-1 or row J-1 (kmax = K-1, jmax = J-1: its
  // loops and step-1 halos end at K-2 / J-2), but a box reaching the row end would
  // still fetch the 128-byte line that holds column K-1 -- on L one extra line per
  // 16 per row, 0.12 GB of a pass's 1.90 GB DRAM reads (1.11x -> 1.04x algorithmic;
  // L pass -0.6 %, M -0.9 %, XL -5 %; profiles/r02_tb2_experiments_late.md).  Maps end
  // there unless HIMENO_TMA_TRIM clears the bit.
  const int trim_env = env_int("HIMENO_TMA_TRIM");
  t->trim = F.K >= 4 && F.J >= 4 ? (trim_env < 0 ? 7 : trim_env & 7) : 0;
  const int dk1 = (t->trim & 2) ? F.K - 1 : dk, dj1 = (t->trim & 2) ? F.J - 1 : 0;
  for (int m = 0; m < NCOEF; ++m) {
    static const int fields[NCOEF] = {HP_F_A0, HP_F_A1, HP_F_A2, HP_F_A3, HP_F_B0, HP_F_B1,
                                      HP_F_B2, HP_F_C0, HP_F_C1, HP_F_C2, HP_F_WRK1, HP_F_BND};
    ok = ok && encode(&t->base.coef[m], F, F.f[fields[m]], TK, TJ, pc[0], dk1, dj1);
  }
  ok = ok && encode(&t->base.pin, F, F.f[HP_F_P], PW, PH, pc[1], dk1, dj1);
  ok = ok && encode(&t->scratch_map, F, scratch, PW, PH, pc[1], dk1, dj1);
  const int dk2 = (t->trim & 1) ? F.K - 1 : dk, dj2 = (t->trim & 1) ? F.J - 1 : 0;
  auto encode_tb2 = [&](Tb2Maps& maps, CUtensorMap& scr, int qk, int r1) {
    static const int fields[NCOEF] = {HP_F_A0, HP_F_A1, HP_F_A2, HP_F_A3, HP_F_B0, HP_F_B1,
                                      HP_F_B2, HP_F_C0, HP_F_C1, HP_F_C2, HP_F_WRK1, HP_F_BND};
    for (int m = 0; m < NCOEF; ++m)
      ok = ok && encode(&maps.coef[m], F, F.f[fields[m]], qk, r1, pc[2], dk2, dj2);
    ok = ok && encode(&maps.pin, F, F.f[HP_F_P], qk + 8, r1 + 2, pc[3], dk2, dj2);
    ok = ok && encode(&scr, F, scratch, qk + 8, r1 + 2, pc[3], dk2, dj2);
  };
  encode_tb2(t->tb2[0], t->tb2_scratch[0], Tb2<32, 8, 4>::QK, Tb2<32, 8, 4>::R1);
  encode_tb2(t->tb2[1], t->tb2_scratch[1], Tb2<16, 8, 4>::QK, Tb2<16, 8, 4>::R1);
  encode_tb2(t->tb2[2], t->tb2_scratch[2], Tb2<16, 6, 5>::QK, Tb2<16, 6, 5>::R1);
  encode_tb2(t->tb2[3], t->tb2_scratch[3], Tb2<16, 5, 6>::QK, Tb2<16, 5, 6>::R1);
  {
    static const int fields[NCOEF] = {HP_F_A0, HP_F_A1, HP_F_A2, HP_F_A3, HP_F_B0, HP_F_B1,
                                      HP_F_B2, HP_F_C0, HP_F_C1, HP_F_C2, HP_F_WRK1, HP_F_BND};
    const int dk3 = (t->trim & 4) ? F.K - 1 : dk, dj3 = (t->trim & 4) ? F.J - 1 : 0;
    for (int m = 0; m < NCOEF; ++m)
      ok = ok && encode(&t->tx.coef[m], F, F.f[fields[m]], XK, kTxTJ, pc[2], dk3, dj3);
    ok = ok && encode(&t->tx.pin, F, F.f[HP_F_P], XW, kTxTJ + 2, pc[3], dk3, dj3);
    ok = ok && encode(&t->tx_scratch, F, scratch, XW, kTxTJ + 2, pc[3], dk3, dj3);
  }
  t->p = F.f[HP_F_P];
  t->scratch = scratch;
  if (!ok) {
    delete t;
    return nullptr;
  }
  // completion tags of the flow launches: one per unit of a pass (at most the gosa
  // partial capacity, which launch_tb2 enforces)
  {
    const int cap = gosa_capacity_needed(F);
    if (cudaMalloc(&t->done, (size_t)cap * 4) == cudaSuccess &&
        cudaMemset(t->done, 0, (size_t)cap * 4) == cudaSuccess) {
      t->done_cap = cap;
    } else {
      if (t->done) cudaFree(t->done);
      t->done = nullptr;
      cudaGetLastError();   // no flow launches for this context
    }
  }
  // exchange buffers for the j/k extents of this context (slab contexts share the
  // global j/k extents): tiles of 128 k x TJ j over [0, K-2) x [1, J-2), only when
  // every tile can be resident at once
  {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int ktiles = (F.K - 2 + XK - 1) / XK;
    const int jtiles = (F.J - 3 + kTxTJ - 1) / kTxTJ;
    const int tiles = ktiles * jtiles;
    if (tiles >= 1 && sms > 0 && tiles <= sms && F.K >= 4 && F.J >= 4) {
      const int chunks = sms / tiles;
      const size_t xrw = (size_t)XK * ktiles + 8, xcw = ((size_t)kTxTJ * jtiles + 8) * XCP;
      const size_t nxr = (size_t)XRX * chunks * jtiles * 2 * xrw;
      const size_t nxc = (size_t)XRX * chunks * ktiles * 2 * xcw;
      // zeroed: tags start at epoch 1 (4097), so no stale word can match
      if (cudaMalloc(&t->xr, nxr * 8) == cudaSuccess && cudaMalloc(&t->xc, nxc * 8) == cudaSuccess &&
          cudaMalloc(&t->err, 4) == cudaSuccess && cudaMemset(t->xr, 0, nxr * 8) == cudaSuccess &&
          cudaMemset(t->xc, 0, nxc * 8) == cudaSuccess && cudaMemset(t->err, 0, 4) == cudaSuccess) {
        t->nxr = nxr;
        t->nxc = nxc;
        t->tx_ktiles = ktiles;
        t->tx_jtiles = jtiles;
        t->tx_chunks = chunks;
      } else {
        cudaGetLastError();   // no exchange kernel for this context (tb2 runs instead)
      }
    }
  }
  return t;
}

void destroy_stencil_tma(void* h) {
  TmaState* t = static_cast<TmaState*>(h);
  if (!t) return;
  if (t->done) cudaFree(t->done);
  if (t->xr) cudaFree(t->xr);
  if (t->xc) cudaFree(t->xc);
  if (t->err) cudaFree(t->err);
  delete t;
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) changes the kernel in the
// *current device's* context only, so the opt-in is recorded per (kernel, device):
// a process that drives several GPUs (B200Evaluator over every device,
// hp_group_jacobi) raises it on each device before the first launch there.
bool ensure_smem_optin(const void* func, int bytes) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> done;   // (kernel, device) -> bytes
  std::lock_guard<std::mutex> lock(mu);
  int& have = done[{func, dev}];
  if (have >= bytes) return true;
  if (cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) !=
      cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  have = bytes;
  return true;
}

// The large-shared-memory kernels by id (hp_smem_optin): 0..2 = single-step with
// 2..4 stages, 3.. = two-step shapes 0..3, 7 = shape 1 with the tensor-memory stash.
const void* smem_kernel(int id) {
  switch (id) {
    case 0: return (const void*)k_stencil_tma<2>;
    case 1: return (const void*)k_stencil_tma<3>;
    case 2: return (const void*)k_stencil_tma<4>;
    case 3: return (const void*)k_stencil_tb2<32, 8, 4, false>;
    case 4: return (const void*)k_stencil_tb2<16, 8, 4, false>;
    case 5: return (const void*)k_stencil_tb2<16, 6, 5, false>;
    case 6: return (const void*)k_stencil_tb2<16, 5, 6, false>;
    case 7: return (const void*)k_stencil_tb2<16, 8, 4, true>;
    case 8: return (const void*)k_stencil_tx<kTxTJ>;
    case 9: return (const void*)k_stencil_tb2<16, 8, 4, true, 1>;
    case 10: return (const void*)k_stencil_tb2<16, 8, 4, true, 4>;
    case 11: return (const void*)k_stencil_tb2<16, 8, 4, true, 13>;
    case 12: return (const void*)k_stencil_tb2<16, 8, 4, true, 12>;
    default: return nullptr;
  }
}

// Launch the TMA stencil with S stages; returns 1, 0 (not applicable: caller
// falls back), or -1 on launch error.
int launch_stencil_tma(const DevFields& F, const void* h, const float* p_in, float* p_out,
                       const LaunchArgs& a, const GosaSink& g, cudaStream_t s, int stages,
                       int sms) {
  const TmaState* t = static_cast<const TmaState*>(h);
  if (!t || (p_in != t->p && p_in != t->scratch)) return 0;
  if ((t->trim & 2) && (a.kmax > F.K - 1 || a.jmax > F.J - 1)) return 0;
  const int i_lo = a.li_lo, i_hi = a.li_hi, j_lo = 1, j_hi = a.jmax - 1, k_lo = 1,
            k_hi = a.kmax - 1;
  if (i_hi <= i_lo || j_hi <= j_lo || k_hi <= k_lo) return 0;
  StencilMaps maps = t->base;
  if (p_in == t->scratch) maps.pin = t->scratch_map;
  const int ktiles = (k_hi + TK - 1) / TK;
  const int jtiles = (j_hi - j_lo + TJ - 1) / TJ;
  const int chunk = chunk_planes(32);
  const long long units = (long long)ktiles * jtiles * ((i_hi - i_lo + chunk - 1) / chunk);
  long long grid = sms;
  if (grid > units) grid = units;
  if (units > g.capacity) return -1;   // one gosa partial per unit
  const size_t smem = 128 + (size_t)stages * kStageBytes + 2 * stages * sizeof(uint64_t) +
                      sizeof(UnitRing);
  // the work-queue counter is zero: set at context creation, reset by the last CTA
  bool attr_ok = true;
  auto launch = [&](auto kern) {
    // the opt-in is a property of the kernel in the current device's context
    if (!(attr_ok = ensure_smem_optin((const void*)kern, (int)smem))) return;
    kern<<<(int)grid, kThreads, smem, s>>>(maps, F, p_out, i_lo, i_hi, j_lo, j_hi, k_lo, k_hi,
                                           ktiles, chunk, a.omega, g, a.gosa_reset);
  };
  switch (stages) {
    case 2: launch(k_stencil_tma<2>); break;
    case 3: launch(k_stencil_tma<3>); break;
    case 4: launch(k_stencil_tma<4>); break;
    default: return 0;
  }
  if (!attr_ok) return -1;
  return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

// Two-step tile shapes (lanes per row, step-1 warps, coefficient slots):
//   0 = (32, 8, 4): 128 x 8 step-1 tile, 120 x 6 outputs, 48 KB stages
//   1 = (16, 8, 4):  64 x 16 step-1 tile, 56 x 14 outputs, 48 KB stages
//   2 = (16, 6, 5):  64 x 12 step-1 tile, 56 x 10 outputs, 36 KB stages
//   3 = (16, 5, 6):  64 x 10 step-1 tile, 56 x 8 outputs, 30 KB stages
// The shape and the planes per work unit are chosen per pass geometry by a
// scheduling model (tb2_choose below).

// First output column of k-tile 0.  -4 puts every tile's coefficient boxes (origin
// k0-4) on a 32-byte sector boundary: 8 sectors per 64-column row instead of 9
// (HIMENO_TB2_KORG=0 restores tiles starting at column 0).
static int tb2_k_org() {
  static const int v = env_int("HIMENO_TB2_KORG") == 0 ? 0 : -4;
  return v;
}

template <int LW, int NW1, int SC>
static long long tb2_tiles(int nj, int k_hi) {
  using T = Tb2<LW, NW1, SC>;
  return (long long)((k_hi - tb2_k_org() + T::TK2 - 1) / T::TK2) * ((nj + T::TJ2 - 1) / T::TJ2);
}

// Makespan of one pass: the device-wide queue hands the units (`full` whole
// columns, then the chunk-major units of the other tiles) to the first free CTA
// (list scheduling); a unit of n planes takes n + 2 plane steps (two warm-up
// planes) at the shape's per-step cost (microseconds per plane step of one CTA,
// measured on the L grid: profiles/r01_tb2_shapes.txt).
static double tb2_makespan(long long tiles, int ni, int chunk, long long full, int sms,
                           double cost) {
  std::priority_queue<double, std::vector<double>, std::greater<double>> q;
  const long long total = full + (tiles - full) * ((ni + chunk - 1) / chunk);
  for (long long c = 0; c < std::min<long long>(sms, total); ++c) q.push(0.0);
  double end = 0.0;
  auto run = [&](double d) {
    const double f = q.top() + d;
    q.pop();
    q.push(f);
    end = std::max(end, f);
  };
  for (long long t = 0; t < full; ++t) run((double)(ni + 2) * cost);
  for (int c0 = 0; c0 < ni; c0 += chunk) {
    const double d = (double)(std::min(chunk, ni - c0) + 2) * cost;
    for (long long t = full; t < tiles; ++t) run(d);
  }
  return end;
}

// (shape, planes per unit, whole columns) with the least predicted makespan,
// cached per pass geometry; HIMENO_TB2_SHAPE / HIMENO_TB2_CHUNK pin the first
// two for sweeps; HIMENO_TB2_FULL=0 disables whole-column units, =1 leaves them
// to the model, =n >= 2 pins n of them (tests).
struct Tb2Choice {
  int shape, chunk, full;
};
static Tb2Choice tb2_choose(int ni, int nj, int k_hi, int sms) {
  // (16,8,4) runs with the tensor-memory stash unless HIMENO_TB2_STASH=0: 1.005 us
  // per plane step with it, 1.04 without
  const bool stash = env_int("HIMENO_TB2_STASH") != 0;
  const double cost[kTb2Shapes] = {1.03, stash ? 1.005 : 1.04, 0.91, 0.885};
  const int pin_shape = env_int("HIMENO_TB2_SHAPE"), pin_chunk = env_int("HIMENO_TB2_CHUNK");
  const int pin_full = env_int("HIMENO_TB2_FULL");
  // cached per geometry, pins and stash setting (the list-scheduling model is too
  // slow to rerun for every pass)
  static std::mutex mu;
  static std::map<std::array<int, 8>, Tb2Choice> cache;
  const std::array<int, 8> key{ni, nj, k_hi, sms, pin_shape, pin_chunk, pin_full, (int)stash};
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  Tb2Choice best{1, 64, 0};
  double best_t = 1e300;
  for (int v = 0; v < kTb2Shapes; ++v) {
    if (pin_shape >= 0 && pin_shape < kTb2Shapes && v != pin_shape) continue;
    long long tiles = 0;
    switch (v) {
      case 0: tiles = tb2_tiles<32, 8, 4>(nj, k_hi); break;
      case 1: tiles = tb2_tiles<16, 8, 4>(nj, k_hi); break;
      case 2: tiles = tb2_tiles<16, 6, 5>(nj, k_hi); break;
      default: tiles = tb2_tiles<16, 5, 6>(nj, k_hi); break;
    }
    // whole columns: none, or every full wave of tiles (the remainder is chunked)
    long long fulls[2] = {0, pin_full != 0 ? tiles / sms * sms : 0};
    if (pin_full >= 2) fulls[0] = fulls[1] = std::min<long long>(pin_full, tiles);
    for (long long full : fulls) {
      for (int chunk = 16; chunk <= 128; chunk += 8) {
        const int ch = pin_chunk > 0 ? pin_chunk : chunk;
        const double t = tb2_makespan(tiles, ni, ch, full, sms, cost[v]);
        if (t < best_t) { best_t = t; best = {v, ch, (int)full}; }
        if (pin_chunk > 0) break;
      }
    }
  }
  {
    std::lock_guard<std::mutex> lock(mu);
    cache[key] = best;
  }
  return best;
}

struct Range2 {
  int lo = 0, hi = 0;   // second output plane range (two-range launch), empty if hi <= lo
  int grid_cap = 0;     // > 0: at most this many CTAs (SMs left to a concurrent kernel)
  int split = 0;        // > 0: boundary-prefix units of this width (signalled slab pass)
  unsigned* sig = nullptr;
  int* nb_out = nullptr;   // receives the number of boundary units (signal target step)
};

template <int LW, int NW1, int SC, bool ST = false, int CPOL = 0>
static int launch_tb2(const Tb2Maps& maps, const DevFields& F, Flow fl, int i_lo, int i_hi,
                      int j_lo, int j_hi, int k_lo, int k_hi, int g_lo, int g_hi, int chunk,
                      int full, const LaunchArgs& a, const GosaSink& g, cudaStream_t s, int sms,
                      const Range2& r2 = Range2{}) {
  using T = Tb2<LW, NW1, SC>;
  const int k_org = tb2_k_org();
  const int ktiles = (k_hi - k_org + T::TK2 - 1) / T::TK2;
  const int jtiles = (j_hi - j_lo + T::TJ2 - 1) / T::TJ2;
  const long long tiles = (long long)ktiles * jtiles;
  if (full < 0 || full > tiles) full = 0;
  const bool two = r2.hi > r2.lo;
  const int sw = two ? 0 : r2.split;
  const long long units =
      two ? 2 * tiles
          : (sw > 0 ? 2 * tiles : 0) + full + (tiles - full) * ((i_hi - i_lo - 2 * sw + chunk - 1) / chunk);
  if (sw > 0) {
    fl.split = sw;
    fl.sig = r2.sig;
    if (r2.nb_out) *r2.nb_out = (int)(2 * tiles);
  }
  long long grid = sms;
  if (r2.grid_cap > 0 && grid > r2.grid_cap) grid = r2.grid_cap;
  if (grid > units * fl.passes) grid = units * fl.passes;
  if (units > g.capacity) return -1;   // one gosa partial per unit (of the last pass)
  fl.upp = (int)units;
  const size_t smem = T::smem_bytes();
  // the work-queue counter is zero: set at context creation, reset by the last CTA
  if (!ensure_smem_optin((const void*)k_stencil_tb2<LW, NW1, SC, ST, CPOL>, (int)smem)) return -1;
  static const bool pdl = env_int("HIMENO_TB2_PDL") != 0;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute la[1];
  la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  la[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(T::kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = la;
  cfg.numAttrs = pdl ? 1 : 0;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, k_stencil_tb2<LW, NW1, SC, ST, CPOL>, maps, F, i_lo,
                                           i_hi, j_lo, j_hi, k_lo, k_hi, k_org, ktiles, chunk, full,
                                           g_lo, g_hi, a.omega, g, a.gosa_reset, fl,
                                           two ? r2.lo : 0, two ? r2.hi : 0);
  return e == cudaSuccess ? 1 : -1;
}

// ---- exchange kernel launches --------------------------------------------------
// Its CTAs wait on each other, so two exchange launches must never share a device
// at the same time (each could hold part of the SMs the other needs).  Launches
// of different streams on one device are therefore chained in enqueue order: a
// launch on stream s first waits for everything the previously used stream had
// enqueued (an event recorded there).  Consecutive launches on one stream need
// nothing (stream order; PDL keeps overlapping their tails).  Any other kernel
// that overlaps an exchange launch finishes on its own, so the launch's CTAs all
// become resident eventually.
static std::mutex g_tx_mu;
struct TxLane {
  cudaStream_t last = nullptr;
  cudaEvent_t ev = nullptr;
};
static std::map<int, TxLane> g_tx_lanes;

void tx_forget_stream(cudaStream_t s) {
  std::lock_guard<std::mutex> lock(g_tx_mu);
  for (auto& kv : g_tx_lanes)
    if (kv.second.last == s) kv.second.last = nullptr;   // stream is being destroyed
}

// HIMENO_TX: 0 (default) = never, 1 = when tiles x chunks fill at least half the
// SMs, 2 = whenever the tiles fit (tests: small and ragged grids).  Off by default:
// on L it reads 7% fewer DRAM bytes than k_stencil_tb2 but runs 4% slower
// (profiles/r02_tx_experiments.md).  Read per launch so tests can switch it.
static int tx_mode() {
  const int v = env_int("HIMENO_TX");
  return v < 0 ? 0 : v;
}
// planes per chunk at least this many (HIMENO_TX_MINCHUNK; a chunk recomputes two
// planes at each end)
static int tx_min_chunk() {
  const int v = env_int("HIMENO_TX_MINCHUNK");
  return v > 0 ? v : 16;
}

static int launch_tx(TmaState* t, const DevFields& F, const float* p_in, float* p_out, int i_lo,
                     int i_hi, int j_lo, int j_hi, int k_lo, int k_hi, int g_lo, int g_hi,
                     const LaunchArgs& a, const GosaSink& g, cudaStream_t s, int sms) {
  constexpr int TJ = kTxTJ;
  using T = Tx<TJ>;
  const int mode = tx_mode();
  // a pinned two-step shape (sweeps, tests) asks for k_stencil_tb2
  if (mode == 0 || !t->xr || env_int("HIMENO_TB2_SHAPE") >= 0) return 0;
  if ((t->trim & 4) && (a.kmax > F.K - 1 || a.jmax > F.J - 1)) return 0;
  const int ktiles = (k_hi + XK - 1) / XK;
  const int jtiles = (j_hi - j_lo + TJ - 1) / TJ;
  const int tiles = ktiles * jtiles;
  if (ktiles > t->tx_ktiles || jtiles > t->tx_jtiles || tiles > sms) return 0;
  const int ni = i_hi - i_lo;
  int chunks = std::min(t->tx_chunks, sms / tiles);
  chunks = std::max(1, std::min(chunks, ni / tx_min_chunk()));
  const int chunk = (ni + chunks - 1) / chunks;
  chunks = (ni + chunk - 1) / chunk;
  if (chunk + 2 >= (int)kXEpoch) return 0;
  if (mode == 1 && tiles * chunks * 2 < sms) return 0;
  if (tiles * chunks > g.capacity) return 0;
  const size_t smem = T::smem_bytes();
  if (!ensure_smem_optin((const void*)k_stencil_tx<TJ>, (int)smem)) return -1;
  TxMaps maps = t->tx;
  if (p_in == t->scratch) maps.pin = t->tx_scratch;
  XBuf x;
  x.xr = t->xr;
  x.xc = t->xc;
  x.err = t->err;
  x.xrw = XK * ktiles + 8;
  x.xcw = (TJ * jtiles + 8) * XCP;
  x.chunks = chunks;
  x.dbg = std::max(0, env_int("HIMENO_TX_DBG"));
  x.ahead = env_int("HIMENO_TX_AHEAD") > 0 ? std::min(env_int("HIMENO_TX_AHEAD"), XNS - 2) : XNS - 2;
  x.xrx = XRX;
  if (env_int("HIMENO_TX_XRX") > 0) x.xrx = std::min(XRX, env_int("HIMENO_TX_XRX"));
  if (x.xrx < 10 + 2 * x.ahead || (x.xrx & (x.xrx - 1))) x.xrx = XRX;
  x.evl = env_int("HIMENO_TX_EVL") != 0 ? 1 : 0;   // evict_last: default (10% faster)
  x.sleep_ns = env_int("HIMENO_TX_SLEEP") >= 0 ? env_int("HIMENO_TX_SLEEP") : 0;
  std::lock_guard<std::mutex> lock(g_tx_mu);
  if (++t->epoch >= (1u << 20)) {   // tags epoch * 4096 + plane stay in 32 bits
    if (cudaMemsetAsync(t->xr, 0, t->nxr * 8, s) != cudaSuccess ||
        cudaMemsetAsync(t->xc, 0, t->nxc * 8, s) != cudaSuccess)
      return -1;
    t->epoch = 1;
  }
  x.epoch = t->epoch;
  int dev = 0;
  cudaGetDevice(&dev);
  TxLane& lane = g_tx_lanes[dev];
  if (lane.last && lane.last != s) {
    if (!lane.ev && cudaEventCreateWithFlags(&lane.ev, cudaEventDisableTiming) != cudaSuccess)
      return -1;
    if (cudaEventRecord(lane.ev, lane.last) != cudaSuccess ||
        cudaStreamWaitEvent(s, lane.ev, 0) != cudaSuccess)
      return -1;
  }
  lane.last = s;
  static const bool pdl = env_int("HIMENO_TB2_PDL") != 0;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute la[1];
  la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  la[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.gridDim = dim3((unsigned)(tiles * chunks));
  cfg.blockDim = dim3(T::kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = la;
  cfg.numAttrs = pdl ? 1 : 0;
  const cudaError_t e =
      cudaLaunchKernelEx(&cfg, k_stencil_tx<TJ>, maps, F, p_out, i_lo, i_hi, j_lo, j_hi, k_lo, k_hi,
                         ktiles, jtiles, chunk, g_lo, g_hi, a.omega, g, a.gosa_reset, x);
  return e == cudaSuccess ? 1 : -1;
}

// which two-step kernel the last two-step launch used: 1 = k_stencil_tb2 (one
// pass), 2 = k_stencil_tx, 3 = k_stencil_tb2 in a multi-pass flow launch
// (hp_last_two_step_kernel; tests and bench.py name it)
static std::atomic<int> g_last_two_step{0};

int tx_error(const void* h) {
  const TmaState* t = static_cast<const TmaState*>(h);
  if (!t || !t->err) return 0;
  unsigned v = 0;
  if (cudaMemcpy(&v, t->err, 4, cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
  return v ? 1 : 0;
}

// Coefficients-first producer order with late p0 release (CPOL_ & 8) for one-pass
// launches: when L2 holds at least 8 planes of the 14 arrays (L: 17, XL: 4).  With it XL
// read 22 % more DRAM (halo lines evicted between neighbouring columns); L runs 3 %
// faster.  HIMENO_TB2_ORD=0/1 forces it.
static bool tb2_ord(const DevFields& F) {
  const int force = env_int("HIMENO_TB2_ORD");
  if (force >= 0) return force != 0;
  static std::atomic<int> l2_of[64] = {};   // L2 bytes per device (0: not queried yet)
  int dev = 0;
  cudaGetDevice(&dev);
  int l2 = dev >= 0 && dev < 64 ? l2_of[dev].load() : 0;
  if (l2 == 0) {
    if (cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    if (dev >= 0 && dev < 64) l2_of[dev] = l2;
  }
  const double plane = 14.0 * F.J * F.P * 4.0;
  return l2 >= 8.0 * plane;
}

// `passes` two-step passes p_in -> p_out -> p_in ... (2 * passes Jacobi iterations)
// in one launch; the result is in p_out for an odd number of passes, p_in for an
// even one.  Returns 1, 0 (not applicable: the caller runs single steps), or -1.
static int launch_two_step(const DevFields& F, const void* h, const float* p_in, float* p_out,
                           int passes, const LaunchArgs& a, const GosaSink& g, cudaStream_t s,
                           int sms, const Range2& r2 = Range2{}) {
  TmaState* t = const_cast<TmaState*>(static_cast<const TmaState*>(h));
  if (!t || (p_in != t->p && p_in != t->scratch) || passes < 1) return 0;
  if ((t->trim & 1) && (a.kmax > F.K - 1 || a.jmax > F.J - 1)) return 0;
  const int i_lo = a.li_lo, i_hi = a.li_hi, j_lo = 1, j_hi = a.jmax - 1, k_lo = 1,
            k_hi = a.kmax - 1;
  // step 1 reads p0 two planes beyond the planes it updates: the full grid (plane
  // -1 is never used by a computed point) or a slab with two-plane halos
  const bool full = a.i_off == 0 && i_lo == 1 && i_hi == a.imax - 1;
  if (!full && (i_lo < 2 || i_hi > F.I - 2)) return 0;
  if (i_hi <= i_lo || j_hi <= j_lo || k_hi <= k_lo) return 0;
  const int g_lo = 1 - a.i_off, g_hi = a.imax - 1 - a.i_off;
  if (passes > 1 && !t->done) return 0;
  // the exchange kernel (one pass per launch) when enabled and its tiles can all
  // be resident
  if (passes == 1 && r2.hi <= r2.lo && r2.grid_cap == 0) {
    const int r = launch_tx(t, F, p_in, p_out, i_lo, i_hi, j_lo, j_hi, k_lo, k_hi, g_lo, g_hi, a, g,
                            s, sms);
    if (r != 0) {
      g_last_two_step = 2;
      return r;
    }
  }
  g_last_two_step = passes > 1 ? 3 : 1;
  Tb2Choice c = tb2_choose(i_hi - i_lo, j_hi - j_lo, k_hi, sms);
  const int v = c.shape;
  Tb2Maps maps = t->tb2[v];
  const bool from_scratch = p_in == t->scratch;
  maps.pin = from_scratch ? t->tb2_scratch[v] : t->tb2[v].pin;
  maps.pin2 = from_scratch ? t->tb2[v].pin : t->tb2_scratch[v];
  Flow fl{};
  fl.passes = passes;
  fl.out[0] = p_out;
  fl.out[1] = const_cast<float*>(p_in);
  if (passes > 1) {
    // a unit of pass t+1 waits for whole neighbouring units of pass t: chunked units
    // only (whole columns would make every wait a wait for the entire pass), unless
    // HIMENO_FLOW_MODEL=1 keeps the per-pass model's schedule (whole columns + tail)
    const bool keep_model = env_int("HIMENO_FLOW_MODEL") > 0;
    if (!keep_model) c.full = 0;
    // balanced chunks of about 22 planes (M, 126 planes: 6 x 21 -> 43.8 us per pass;
    // 16 -> 45.6, 22 -> 44.1, 24 -> 44.6, 32 -> 48.7; profiles/r02_flow.md)
    const int fc = env_int("HIMENO_FLOW_CHUNK");
    const int ni = i_hi - i_lo;
    const int nch = std::max(1, (ni + 11) / 22);
    if (!keep_model) c.chunk = fc > 0 ? fc : (ni + nch - 1) / nch;
    fl.done = t->done;
    std::lock_guard<std::mutex> lock(g_tx_mu);
    if (++t->flow_epoch >= (1u << 20) - 1u) {   // tags epoch * 4096 + pass + 1 in 32 bits
      if (cudaMemsetAsync(t->done, 0, (size_t)t->done_cap * 4, s) != cudaSuccess) return -1;
      t->flow_epoch = 1;
    }
    if (passes >= 4095) return 0;
    fl.tag0 = t->flow_epoch * 4096u;
  }
#define HP_TB2(LW, NW1, SC) \
  launch_tb2<LW, NW1, SC>(maps, F, fl, i_lo, i_hi, j_lo, j_hi, k_lo, k_hi, g_lo, g_hi, c.chunk, \
                          c.full, a, g, s, sms, r2)
  switch (v) {
    case 1:
      if (env_int("HIMENO_TB2_STASH") != 0) {
        // cross-warp stash (default; HIMENO_TB2_XS=0: each step-2 warp copies its own
        // quads from shared memory): L -1.6..3.6 %, M -2.5 %, XL -1.5..3.6 % per pass
        if (env_int("HIMENO_TB2_XS") != 0) {
          if (passes > 1 && env_int("HIMENO_FLOW_CPOL") != 0)
            return launch_tb2<16, 8, 4, true, 13>(maps, F, fl, i_lo, i_hi, j_lo, j_hi, k_lo, k_hi,
                                                  g_lo, g_hi, c.chunk, c.full, a, g, s, sms, r2);
          if (tb2_ord(F))
            return launch_tb2<16, 8, 4, true, 12>(maps, F, fl, i_lo, i_hi, j_lo, j_hi, k_lo, k_hi,
                                                  g_lo, g_hi, c.chunk, c.full, a, g, s, sms, r2);
          return launch_tb2<16, 8, 4, true, 4>(maps, F, fl, i_lo, i_hi, j_lo, j_hi, k_lo, k_hi,
                                               g_lo, g_hi, c.chunk, c.full, a, g, s, sms, r2);
        }
        if (passes > 1 && env_int("HIMENO_FLOW_CPOL") != 0)
          return launch_tb2<16, 8, 4, true, 1>(maps, F, fl, i_lo, i_hi, j_lo, j_hi, k_lo, k_hi,
                                               g_lo, g_hi, c.chunk, c.full, a, g, s, sms, r2);
        return launch_tb2<16, 8, 4, true>(maps, F, fl, i_lo, i_hi, j_lo, j_hi, k_lo, k_hi, g_lo,
                                          g_hi, c.chunk, c.full, a, g, s, sms, r2);
      }
      return HP_TB2(16, 8, 4);
    case 2: return HP_TB2(16, 6, 5);
    case 3: return HP_TB2(16, 5, 6);
    default: return HP_TB2(32, 8, 4);
  }
#undef HP_TB2
}

// Two-step pass p_in -> p_out (2 Jacobi iterations); returns 1, 0 (not
// applicable: caller runs two single steps), or -1 on launch error.
int launch_stencil_tb2(const DevFields& F, const void* h, const float* p_in, float* p_out,
                       const LaunchArgs& a, const GosaSink& g, cudaStream_t s, int sms) {
  return launch_two_step(F, h, p_in, p_out, 1, a, g, s, sms);
}

// One two-step pass of a slab in parts (decomp.cpp): part 1 = the two boundary plane
// pairs [li_lo, li_lo+2) and [li_hi-2, li_hi) in one launch (what the neighbours need;
// gosa stored), part 2 = the interior [li_lo+2, li_hi-2) on at most sms - reserve CTAs
// (gosa accumulated).  Same arithmetic per point as the whole pass: bit-identical.
// Returns 1, 0 (slab too thin: run the whole pass), or -1.
int launch_stencil_tb2_part(const DevFields& F, const void* h, const float* p_in, float* p_out,
                            const LaunchArgs& a, const GosaSink& g, cudaStream_t s, int sms,
                            int part, int reserve) {
  if (a.li_hi - a.li_lo < 6) return 0;
  LaunchArgs b = a;
  Range2 r2;
  if (part == 1) {
    b.li_hi = a.li_lo + 2;
    r2.lo = a.li_hi - 2;
    r2.hi = a.li_hi;
  } else {
    b.li_lo = a.li_lo + 2;
    b.li_hi = a.li_hi - 2;
    b.gosa_reset = 0;
    r2.grid_cap = reserve > 0 ? std::max(1, sms - reserve) : sms;
  }
  return launch_two_step(F, h, p_in, p_out, 1, b, g, s, sms, r2);
}

// One two-step pass of a slab as ONE launch whose first units are the boundary plane
// pairs (decomp.cpp): each finished boundary unit increments *sig, so the halo exchange
// can start (cuStreamWaitValue32 on the exchange stream) while the interior units run;
// *nb_out = boundary units per pass (the signal target step).  At most sms - reserve
// CTAs.  Returns 1, 0 (slab too thin: caller splits or runs the whole pass), or -1.
int launch_stencil_tb2_signaled(const DevFields& F, const void* h, const float* p_in,
                                float* p_out, const LaunchArgs& a, const GosaSink& g,
                                cudaStream_t s, int sms, int reserve, unsigned* sig, int* nb_out) {
  if (a.li_hi - a.li_lo < 6 || !sig || !nb_out) return 0;
  Range2 r2;
  r2.split = 2;
  r2.sig = sig;
  r2.nb_out = nb_out;
  r2.grid_cap = reserve > 0 ? std::max(1, sms - reserve) : sms;
  *nb_out = 0;
  const int r = launch_two_step(F, h, p_in, p_out, 1, a, g, s, sms, r2);
  if (r > 0 && *nb_out <= 0) return -1;
  return r;
}

// Flow launches pay where the per-pass drain matters: when one pass's tiles fit in
// one wave of the SMs (M: 45 tiles, 50.1 -> 44.6 us per pass); with more tiles (L:
// 190, whole tile columns) the pass-by-pass launches are as fast or faster
// (profiles/r02_flow.md).  HIMENO_TB2_FLOW: 0 = never, 1 = always, unset = that rule.
int stencil_flow_ok(const DevFields& F, const LaunchArgs& a, int sms) {
  const TmaState* t = static_cast<const TmaState*>(F.tma);
  if (!t || !t->done) return 0;
  const int mode = env_int("HIMENO_TB2_FLOW");
  if (mode == 0 || env_int("HIMENO_TX") > 0) return 0;
  if (mode < 0) {
    const int j_hi = a.jmax - 1, k_hi = a.kmax - 1;
    const Tb2Choice c = tb2_choose(a.li_hi - a.li_lo, j_hi - 1, k_hi, sms);
    long long tiles = 0;
    switch (c.shape) {
      case 0: tiles = tb2_tiles<32, 8, 4>(j_hi - 1, k_hi); break;
      case 1: tiles = tb2_tiles<16, 8, 4>(j_hi - 1, k_hi); break;
      case 2: tiles = tb2_tiles<16, 6, 5>(j_hi - 1, k_hi); break;
      default: tiles = tb2_tiles<16, 5, 6>(j_hi - 1, k_hi); break;
    }
    if (tiles > sms) return 0;
  }
  return 1;
}

int launch_stencil_flow(const DevFields& F, const void* h, const float* p_in, float* p_out,
                        int passes, const LaunchArgs& a, const GosaSink& g, cudaStream_t s,
                        int sms) {
  if (h != F.tma || !stencil_flow_ok(F, a, sms)) return 0;
  return launch_two_step(F, h, p_in, p_out, passes, a, g, s, sms);
}

}  // namespace hp

extern "C" int hp_last_two_step_kernel(void) { return hp::g_last_two_step.load(); }

// Diagnostics: the dynamic shared-memory limit kernel `id` has on `device`
// (cudaFuncGetAttributes in that device's context).
extern "C" int hp_smem_optin(int id, int device, int* bytes) {
  const void* f = hp::smem_kernel(id);
  if (!f || !bytes) {
    hp::set_error("hp_smem_optin: bad arguments");
    return HP_ERR_ARG;
  }
  int prev = 0;
  cudaGetDevice(&prev);
  cudaError_t e = cudaSetDevice(device);
  cudaFuncAttributes fa{};
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, f);
  cudaSetDevice(prev);
  if (e != cudaSuccess) return hp::cuda_fail(e, "hp_smem_optin");
  *bytes = fa.maxDynamicSharedSizeBytes;
  return HP_OK;
}
