// sm_100a kernels for the Himeno loop nests (apps/himeno.py loop ids 0-12).
//
// Arithmetic is the C program's, evaluated in the same order with every
// product/sum rounded separately (__fmul_rn/__fadd_rn, and the file is built
// with --fmad=false): the device result is bit-identical to the host loops
// and to the CPU oracle (oracle/himeno_oracle.c), which is what lets any mix
// of host and device loops in a genome reproduce the all-CPU output exactly.
// gosa terms ss*ss are rounded to fp32 (as in `gosa += ss*ss`) and summed in
// fp64; the block/grid reduction order is fixed, so the
// sum is run-to-run deterministic.
//
// Kernel families:
//   k_nest<NEST, MAP>   generic body for any loop-nest box, three mappings
//                       (kernels = collapse, parallel loop = gang, parallel
//                       loop vector = one CTA) -- used for plane/row/partial
//                       anchors and every init/copy nest.
//   k_stencil_3d        tuned full-interior stencil: one warp per (j, k-tile)
//                       row, float4 k-quads, i-marching register queue for
//                       p (2.5-D blocking), k+-1 via warp shuffles, streamed
//                       coefficient loads (ld.global.nc.L1::no_allocate).
//   k_copy_3d           float4 interior copy p = wrk2.
#include <cuda_runtime.h>

#include <cstdio>

#include "hp_internal.h"
#include "reduce.cuh"

namespace hp {
namespace {

constexpr int kNestThreads = 256;
constexpr int kMaxCollapseBlocks = 148 * 16;

__device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }

// ---------------------------------------------------------------- loop bodies

// loop 2 body: zero a[4], b[3], c[3], p, wrk1, bnd (wrk2 untouched)
__device__ __forceinline__ void body_init0(const DevFields& F, size_t c) {
#pragma unroll
  for (int f = 0; f < HP_NFIELDS; ++f)
    if (f != HP_F_WRK2) F.f[f][c] = 0.0f;
}

// loop 5 body: coefficients and p = (float)(i*i)/(float)((imax-1)*(imax-1))
__device__ __forceinline__ void body_init1(const DevFields& F, size_t c, int i, int imax) {
  F.f[HP_F_A0][c] = 1.0f;
  F.f[HP_F_A1][c] = 1.0f;
  F.f[HP_F_A2][c] = 1.0f;
  F.f[HP_F_A3][c] = (float)(1.0 / 6.0);
  F.f[HP_F_B0][c] = 0.0f;
  F.f[HP_F_B1][c] = 0.0f;
  F.f[HP_F_B2][c] = 0.0f;
  F.f[HP_F_C0][c] = 1.0f;
  F.f[HP_F_C1][c] = 1.0f;
  F.f[HP_F_C2][c] = 1.0f;
  F.f[HP_F_P][c] = __fdiv_rn((float)(i * i), (float)((imax - 1) * (imax - 1)));
  F.f[HP_F_WRK1][c] = 0.0f;
  F.f[HP_F_BND][c] = 1.0f;
}

// loop 9 body on explicit neighbour values; returns ss.
// n[] = p at: 0 i+1 | 1 j+1 | 2 k+1 | 3 (i+1,j+1) | 4 (i+1,j-1) | 5 (i-1,j+1)
//   6 (i-1,j-1) | 7 (j+1,k+1) | 8 (j-1,k+1) | 9 (j+1,k-1) | 10 (j-1,k-1)
//   11 (i+1,k+1) | 12 (i-1,k+1) | 13 (i+1,k-1) | 14 (i-1,k-1) | 15 i-1
//   16 j-1 | 17 k-1 | 18 centre
struct Coef { float a0, a1, a2, a3, b0, b1, b2, c0, c1, c2, wrk1, bnd; };

__device__ __forceinline__ float stencil_ss(const Coef& q, const float (&n)[19]) {
  float s0 = mul(q.a0, n[0]);
  s0 = add(s0, mul(q.a1, n[1]));
  s0 = add(s0, mul(q.a2, n[2]));
  s0 = add(s0, mul(q.b0, add(sub(sub(n[3], n[4]), n[5]), n[6])));
  s0 = add(s0, mul(q.b1, add(sub(sub(n[7], n[8]), n[9]), n[10])));
  s0 = add(s0, mul(q.b2, add(sub(sub(n[11], n[12]), n[13]), n[14])));
  s0 = add(s0, mul(q.c0, n[15]));
  s0 = add(s0, mul(q.c1, n[16]));
  s0 = add(s0, mul(q.c2, n[17]));
  s0 = add(s0, q.wrk1);
  return mul(sub(mul(s0, q.a3), n[18]), q.bnd);
}

__device__ __forceinline__ float body_stencil(const DevFields& F, const float* __restrict__ p,
                                              float* __restrict__ out, size_t c, float omega,
                                              double& acc) {
  const size_t P = F.P, L = F.plane();
  Coef q;
  q.a0 = F.f[HP_F_A0][c]; q.a1 = F.f[HP_F_A1][c]; q.a2 = F.f[HP_F_A2][c];
  q.a3 = F.f[HP_F_A3][c]; q.b0 = F.f[HP_F_B0][c]; q.b1 = F.f[HP_F_B1][c];
  q.b2 = F.f[HP_F_B2][c]; q.c0 = F.f[HP_F_C0][c]; q.c1 = F.f[HP_F_C1][c];
  q.c2 = F.f[HP_F_C2][c]; q.wrk1 = F.f[HP_F_WRK1][c]; q.bnd = F.f[HP_F_BND][c];
  const float n[19] = {
      p[c + L], p[c + P], p[c + 1],
      p[c + L + P], p[c + L - P], p[c - L + P], p[c - L - P],
      p[c + P + 1], p[c - P + 1], p[c + P - 1], p[c - P - 1],
      p[c + L + 1], p[c - L + 1], p[c + L - 1], p[c - L - 1],
      p[c - L], p[c - P], p[c - 1], p[c]};
  const float ss = stencil_ss(q, n);
  acc += (double)mul(ss, ss);
  out[c] = add(n[18], mul(omega, ss));
  return ss;
}

// -------------------------------------------------------- generic nest kernel

template <int NEST>
__device__ __forceinline__ void nest_point(const DevFields& F, int i, int j, int k,
                                           const LaunchArgs& a, double& acc) {
  const size_t c = F.at(i, j, k);
  if (NEST == NEST_INIT0) {
    body_init0(F, c);
  } else if (NEST == NEST_INIT1) {
    body_init1(F, c, i + a.i_off, a.imax);
  } else if (NEST == NEST_STENCIL) {
    body_stencil(F, F.f[HP_F_P], F.f[HP_F_WRK2], c, a.omega, acc);
  } else {
    F.f[HP_F_P][c] = F.f[HP_F_WRK2][c];
  }
}

// MAP_COLLAPSE: every warp takes whole (i, j) rows of the box (grid-stride over
//               rows), lanes stride k -- one division per row, coalesced rows.
// MAP_GANG:     block b owns outer index b of the box (i plane, or j row of a
//               plane box); its warps take the rows, lanes stride k.  A row box
//               is gang+vector over k.
// MAP_VECTOR:   one block walks the rows in order, k strips of blockDim
//               separated by barriers (all reads of a strip precede the next).
template <int NEST, int MAP>
__global__ void __launch_bounds__(kNestThreads)
k_nest(DevFields F, Box b, LaunchArgs a, GosaSink g) {
  // launched with programmatic stream serialization: the next launch may be
  // scheduled as soon as every block of this one started, and this one waits for
  // its predecessor's completion (and memory) before touching any data -- the
  // launches of an inner-loop gang (one per outer iteration) overlap their
  // launch latency, never their data.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int nk = (int)b.nk(), nj = (int)b.nj(), ni = (int)b.ni();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  double acc = 0.0;
  if (MAP == MAP_COLLAPSE) {
    const long long rows = (long long)ni * nj;
    const long long wstride = (long long)gridDim.x * nwarps;
    for (long long r = (long long)blockIdx.x * nwarps + warp; r < rows; r += wstride) {
      const int i = (int)(r / nj), j = (int)(r % nj);
      for (int k = lane; k < nk; k += 32)
        nest_point<NEST>(F, b.i0 + i, b.j0 + j, b.k0 + k, a, acc);
    }
  } else if (MAP == MAP_GANG) {
    if (ni > 1) {
      const int i = blockIdx.x;
      for (int j = warp; j < nj; j += nwarps)
        for (int k = lane; k < nk; k += 32)
          nest_point<NEST>(F, b.i0 + i, b.j0 + j, b.k0 + k, a, acc);
    } else if (nj > 1) {
      const int j = blockIdx.x;
      for (int k = threadIdx.x; k < nk; k += blockDim.x)
        nest_point<NEST>(F, b.i0, b.j0 + j, b.k0 + k, a, acc);
    } else {
      const int k = blockIdx.x * blockDim.x + threadIdx.x;
      if (k < nk) nest_point<NEST>(F, b.i0, b.j0, b.k0 + k, a, acc);
    }
  } else {
    for (int i = 0; i < ni; ++i)
      for (int j = 0; j < nj; ++j)
        for (int base = 0; base < nk; base += blockDim.x) {
          const int k = base + threadIdx.x;
          if (k < nk) nest_point<NEST>(F, b.i0 + i, b.j0 + j, b.k0 + k, a, acc);
          __syncthreads();
        }
  }
  if (NEST == NEST_STENCIL) gosa_commit(g, acc, gridDim.x, blockIdx.x, a.gosa_reset);
}

// ------------------------------------------------------- tuned full stencil

constexpr int kTileWarps = 8;          // rows (j) per CTA, one warp per row
constexpr int kQuadsPerWarp = 32;      // 128 k per warp
constexpr int kTargetCtasPerSm = 2;

__device__ __forceinline__ float4 ldg_stream(const float* ptr) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(ptr));
  return r;
}

// VEC consecutive k values held by one lane (VEC = 2 or 4: 8/16-byte accesses)
template <int VEC> struct Vec { float e[VEC]; };

template <int VEC> __device__ __forceinline__ Vec<VEC> ldv(const float* p) {
  Vec<VEC> v;
  if (VEC == 4) {
    const float4 t = *reinterpret_cast<const float4*>(p);
    v.e[0] = t.x; v.e[1] = t.y; v.e[2 % VEC] = t.z; v.e[3 % VEC] = t.w;
  } else {
    const float2 t = *reinterpret_cast<const float2*>(p);
    v.e[0] = t.x; v.e[1] = t.y;
  }
  return v;
}

template <int VEC> __device__ __forceinline__ Vec<VEC> ldv_stream(const float* p) {
  Vec<VEC> v;
  if (VEC == 4) {
    const float4 t = __ldcs(reinterpret_cast<const float4*>(p));
    v.e[0] = t.x; v.e[1] = t.y; v.e[2 % VEC] = t.z; v.e[3 % VEC] = t.w;
  } else {
    const float2 t = __ldcs(reinterpret_cast<const float2*>(p));
    v.e[0] = t.x; v.e[1] = t.y;
  }
  return v;
}

template <int VEC> __device__ __forceinline__ void stv(float* p, const float (&r)[VEC]) {
  if (VEC == 4) *reinterpret_cast<float4*>(p) = make_float4(r[0], r[1], r[2 % VEC], r[3 % VEC]);
  else *reinterpret_cast<float2*>(p) = make_float2(r[0], r[1]);
}

// k-1 neighbour of element 0 and k+1 neighbour of element VEC-1 of a row vector
struct Edge { float left, right; };

template <int VEC>
__device__ __forceinline__ Edge row_edges(const Vec<VEC>& v, const float* row_at, int lane) {
  Edge e;
  e.left = __shfl_up_sync(0xffffffffu, v.e[VEC - 1], 1);
  e.right = __shfl_down_sync(0xffffffffu, v.e[0], 1);
  if (lane == 0) e.left = row_at[-1];
  if (lane == 31) e.right = row_at[VEC];
  return e;
}

template <int VEC>
__device__ __forceinline__ float km1(const Vec<VEC>& v, const Edge& e, int x) {
  return x == 0 ? e.left : v.e[x - 1];
}
template <int VEC>
__device__ __forceinline__ float kp1(const Vec<VEC>& v, const Edge& e, int x) {
  return x == VEC - 1 ? e.right : v.e[x + 1];
}

// One warp-row column: row j, lane vector starting at kb, planes [ia, ib).
// Register queue along i holds rows (j-1, j, j+1) of planes i-1 (l*), i (m*),
// i+1 (n*); k+-1 neighbours come from lane shuffles (+1 scalar load at each
// warp edge).  Coefficients are streamed (ld.global.cs: read once, evict
// first) and consumed term by term in the C program's order.
template <int VEC>
__device__ __forceinline__ void stencil_column(const DevFields& F, const float* __restrict__ pin,
                                               float* __restrict__ out, int ia, int ib, int j,
                                               int kb, int k_lo, int k_hi, float omega, int lane,
                                               double& acc) {
  const size_t P = F.P, L = F.plane();
  const bool active = kb + VEC - 1 >= k_lo && kb < k_hi;  // vector overlaps [k_lo, k_hi)
  bool ok[VEC];
  bool full = true;
#pragma unroll
  for (int x = 0; x < VEC; ++x) {
    ok[x] = active && kb + x >= k_lo && kb + x < k_hi;
    full = full && ok[x];
  }
  size_t c = F.at(ia, j, kb);
  Vec<VEC> l0 = ldv<VEC>(pin + c - L), lm = ldv<VEC>(pin + c - L - P), lp = ldv<VEC>(pin + c - L + P);
  Vec<VEC> m0 = ldv<VEC>(pin + c), mm = ldv<VEC>(pin + c - P), mp = ldv<VEC>(pin + c + P);
#pragma unroll 1
  for (int i = ia; i < ib; ++i, c += L) {
    const Vec<VEC> n0 = ldv<VEC>(pin + c + L), nm = ldv<VEC>(pin + c + L - P),
                   np = ldv<VEC>(pin + c + L + P);
    const Vec<VEC> A0 = ldv_stream<VEC>(F.f[HP_F_A0] + c), A1 = ldv_stream<VEC>(F.f[HP_F_A1] + c);
    const Vec<VEC> A2 = ldv_stream<VEC>(F.f[HP_F_A2] + c), A3 = ldv_stream<VEC>(F.f[HP_F_A3] + c);
    const Vec<VEC> B0 = ldv_stream<VEC>(F.f[HP_F_B0] + c), B1 = ldv_stream<VEC>(F.f[HP_F_B1] + c);
    const Vec<VEC> B2 = ldv_stream<VEC>(F.f[HP_F_B2] + c), C0 = ldv_stream<VEC>(F.f[HP_F_C0] + c);
    const Vec<VEC> C1 = ldv_stream<VEC>(F.f[HP_F_C1] + c), C2 = ldv_stream<VEC>(F.f[HP_F_C2] + c);
    const Vec<VEC> W1 = ldv_stream<VEC>(F.f[HP_F_WRK1] + c), BN = ldv_stream<VEC>(F.f[HP_F_BND] + c);

    const Edge eL = row_edges<VEC>(l0, pin + c - L, lane);
    const Edge eN = row_edges<VEC>(n0, pin + c + L, lane);
    const Edge eM = row_edges<VEC>(m0, pin + c, lane);
    const Edge eMm = row_edges<VEC>(mm, pin + c - P, lane);
    const Edge eMp = row_edges<VEC>(mp, pin + c + P, lane);

    float r[VEC];
#pragma unroll
    for (int x = 0; x < VEC; ++x) {
      float s0 = mul(A0.e[x], n0.e[x]);
      s0 = add(s0, mul(A1.e[x], mp.e[x]));
      s0 = add(s0, mul(A2.e[x], kp1<VEC>(m0, eM, x)));
      s0 = add(s0, mul(B0.e[x], add(sub(sub(np.e[x], nm.e[x]), lp.e[x]), lm.e[x])));
      s0 = add(s0, mul(B1.e[x], add(sub(sub(kp1<VEC>(mp, eMp, x), kp1<VEC>(mm, eMm, x)),
                                         km1<VEC>(mp, eMp, x)), km1<VEC>(mm, eMm, x))));
      s0 = add(s0, mul(B2.e[x], add(sub(sub(kp1<VEC>(n0, eN, x), kp1<VEC>(l0, eL, x)),
                                         km1<VEC>(n0, eN, x)), km1<VEC>(l0, eL, x))));
      s0 = add(s0, mul(C0.e[x], l0.e[x]));
      s0 = add(s0, mul(C1.e[x], mm.e[x]));
      s0 = add(s0, mul(C2.e[x], km1<VEC>(m0, eM, x)));
      s0 = add(s0, W1.e[x]);
      const float ss = mul(sub(mul(s0, A3.e[x]), m0.e[x]), BN.e[x]);
      r[x] = add(m0.e[x], mul(omega, ss));
      if (ok[x]) acc += (double)mul(ss, ss);
    }
    if (full) {
      stv<VEC>(out + c, r);
    } else if (active) {
#pragma unroll
      for (int x = 0; x < VEC; ++x)
        if (ok[x]) out[c + x] = r[x];
    }
    lm = mm; l0 = m0; lp = mp;
    mm = nm; m0 = n0; mp = np;
  }
}

// Interior = i in [i_lo, i_hi), j in [j_lo, j_hi), k in [k_lo, k_hi).
// Work unit = (tile, plane), tile = 8 rows x (32*VEC) k, one warp per row.
// The grid is one wave (SMs x resident CTAs) and CTA b takes the contiguous
// unit range [U*b/G, U*(b+1)/G) in tile-major, plane-minor order, so every
// CTA streams the same number of planes (no tail wave).
template <int VEC, int MINB>
__global__ void __launch_bounds__(kTileWarps * 32, MINB)
k_stencil_3d(DevFields F, const float* __restrict__ pin, float* __restrict__ out,
             int i_lo, int i_hi, int j_lo, int j_hi, int k_lo, int k_hi, int ktiles,
             float omega, GosaSink g, int reset) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int ni = i_hi - i_lo;
  const int jtiles = (j_hi - j_lo + kTileWarps - 1) / kTileWarps;
  const long long U = (long long)ktiles * jtiles * ni;
  long long u = U * blockIdx.x / gridDim.x;
  const long long u_end = U * (blockIdx.x + 1) / gridDim.x;
  double acc = 0.0;
  while (u < u_end) {
    const int t = (int)(u / ni);
    const int ia = (int)(u % ni);
    const int ib = (int)min((long long)ni, (long long)ia + (u_end - u));
    u += ib - ia;
    const int kt = t % ktiles, jt = t / ktiles;
    const int j = j_lo + jt * kTileWarps + w;
    if (j >= j_hi) continue;  // warp-uniform: shuffles inside stay convergent
    const int kb = (kt * 32 + lane) * VEC;
    stencil_column<VEC>(F, pin, out, i_lo + ia, i_lo + ib, j, kb, k_lo, k_hi, omega, lane, acc);
  }
  gosa_commit(g, acc, gridDim.x, blockIdx.x, reset);
}

// p[interior] = src[interior] on float4 quads with masked edges.
__global__ void __launch_bounds__(256)
k_copy_3d(DevFields F, const float* __restrict__ src, float* __restrict__ dst,
          int i_lo, int i_hi, int j_lo, int j_hi, int k_lo, int k_hi) {
  const int nq = (k_hi + 3) / 4;                      // quads covering [0, k_hi)
  const long long rows = (long long)(i_hi - i_lo) * (j_hi - j_lo);
  const long long total = rows * nq;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int q = (int)(t % nq);
    const long long r = t / nq;
    const int j = j_lo + (int)(r % (j_hi - j_lo));
    const int i = i_lo + (int)(r / (j_hi - j_lo));
    const int kb = q * 4;
    if (kb + 3 < k_lo) continue;
    const size_t c = F.at(i, j, kb);
    if (kb >= k_lo && kb + 3 < k_hi) {
      *reinterpret_cast<float4*>(dst + c) = ldg_stream(src + c);
    } else {
      for (int x = 0; x < 4; ++x)
        if (kb + x >= k_lo && kb + x < k_hi) dst[c + x] = src[c + x];
    }
  }
}

// Copy every non-interior point of [0,I)x[0,J)x[0,K) (the faces the stencil
// reads but never writes): whole rows on boundary planes/rows, else the row
// ends k = 0 and k >= kmax-1.  One thread per (i, j) row.
__global__ void k_copy_halo(DevFields F, const float* __restrict__ src, float* __restrict__ dst,
                            int li_lo, int li_hi, int jmax, int kmax) {
  const long long rows = (long long)F.I * F.J;
  for (long long r = (long long)blockIdx.x * blockDim.y + threadIdx.y; r < rows;
       r += (long long)gridDim.x * blockDim.y) {
    const int i = (int)(r / F.J), j = (int)(r % F.J);
    const size_t base = F.at(i, j, 0);
    const bool whole = i < li_lo || i >= li_hi || j == 0 || j >= jmax - 1;
    if (whole) {
      for (int k = threadIdx.x; k < F.K; k += blockDim.x) dst[base + k] = src[base + k];
    } else {
      if (threadIdx.x == 0) dst[base] = src[base];
      for (int k = kmax - 1 + threadIdx.x; k < F.K; k += blockDim.x) dst[base + k] = src[base + k];
    }
  }
}

// 2-D copy between row pitches (elements): host-layout staging <-> pitched field
__global__ void k_repitch(float* __restrict__ dst, size_t dpitch, const float* __restrict__ src,
                          size_t spitch, int width, size_t rows) {
  const size_t total = rows * (size_t)width;
  for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (size_t)gridDim.x * blockDim.x) {
    const size_t r = t / (size_t)width, c = t % (size_t)width;
    dst[r * dpitch + c] = src[r * spitch + c];
  }
}

__global__ void k_fill(float* dst, size_t n, float v) {
  for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (size_t)gridDim.x * blockDim.x)
    dst[t] = v;
}

// Verification mode (HP_FLAG_LITERAL_GOSA): the ss*ss terms of one stencil
// execution over box b, from the same device state and with the same arithmetic
// as the stencil kernel about to run, stored at their program-order position
// [i][j][k] of an unpadded I x J x K buffer (the host sums them sequentially).
__global__ void k_stencil_terms(DevFields F, const float* __restrict__ p, float* __restrict__ terms,
                                Box b) {
  const long long nk = b.nk(), nj = b.nj(), total = b.count();
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int k = b.k0 + (int)(t % nk);
    const int j = b.j0 + (int)((t / nk) % nj);
    const int i = b.i0 + (int)(t / (nk * nj));
    const size_t c = F.at(i, j, k);
    const size_t P = F.P, L = F.plane();
    Coef q;
    q.a0 = F.f[HP_F_A0][c]; q.a1 = F.f[HP_F_A1][c]; q.a2 = F.f[HP_F_A2][c];
    q.a3 = F.f[HP_F_A3][c]; q.b0 = F.f[HP_F_B0][c]; q.b1 = F.f[HP_F_B1][c];
    q.b2 = F.f[HP_F_B2][c]; q.c0 = F.f[HP_F_C0][c]; q.c1 = F.f[HP_F_C1][c];
    q.c2 = F.f[HP_F_C2][c]; q.wrk1 = F.f[HP_F_WRK1][c]; q.bnd = F.f[HP_F_BND][c];
    const float n[19] = {
        p[c + L], p[c + P], p[c + 1],
        p[c + L + P], p[c + L - P], p[c - L + P], p[c - L - P],
        p[c + P + 1], p[c - P + 1], p[c + P - 1], p[c - P - 1],
        p[c + L + 1], p[c - L + 1], p[c + L - 1], p[c - L - 1],
        p[c - L], p[c - P], p[c - 1], p[c]};
    const float ss = stencil_ss(q, n);
    terms[((size_t)i * F.J + j) * F.K + k] = mul(ss, ss);
  }
}

template <int NEST>
int launch_nest_t(Mapping map, const DevFields& F, const Box& b, const LaunchArgs& a,
                  const GosaSink& g, cudaStream_t s) {
  if (b.count() <= 0) {
    return 0;
  }
  int blocks = 1;
  if (map == MAP_COLLAPSE) {
    const long long rows = b.ni() * b.nj();
    const long long need = (rows + kNestThreads / 32 - 1) / (kNestThreads / 32);
    blocks = (int)(need < kMaxCollapseBlocks ? need : kMaxCollapseBlocks);
  } else if (map == MAP_GANG) {
    if (b.ni() > 1) blocks = (int)b.ni();
    else if (b.nj() > 1) blocks = (int)b.nj();
    else blocks = (int)((b.nk() + kNestThreads - 1) / kNestThreads);
  }
  if (NEST == NEST_STENCIL && blocks > g.capacity) return -1;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.gridDim = dim3(map == MAP_VECTOR ? 1 : blocks);
  cfg.blockDim = dim3(kNestThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e;
  if (map == MAP_COLLAPSE) e = cudaLaunchKernelEx(&cfg, k_nest<NEST, MAP_COLLAPSE>, F, b, a, g);
  else if (map == MAP_GANG) e = cudaLaunchKernelEx(&cfg, k_nest<NEST, MAP_GANG>, F, b, a, g);
  else e = cudaLaunchKernelEx(&cfg, k_nest<NEST, MAP_VECTOR>, F, b, a, g);
  return e == cudaSuccess ? 1 : -1;
}

}  // namespace

static int sm_count();

int gosa_capacity_needed(const DevFields& F) {
  const int tiles = ((F.K + 127) / 128) * ((F.J + kTileWarps - 1) / kTileWarps);
  const int want = sm_count() * kTargetCtasPerSm * 2;
  // unit-queue kernels (stencil_tma.cu): one partial per work unit; the finest
  // unit grid is 16 planes x 8 rows x 56 columns
  const int units = ((F.I + 15) / 16) * ((F.J + 7) / 8) * ((F.K + 55) / 56);
  return kMaxCollapseBlocks + F.I + F.J + tiles + want + units + 1024;
}

int launch_nest(Nest nest, Mapping map, const DevFields& F, const Box& box,
                const LaunchArgs& a, const GosaSink& g, cudaStream_t s) {
  switch (nest) {
    case NEST_INIT0: return launch_nest_t<NEST_INIT0>(map, F, box, a, g, s);
    case NEST_INIT1: return launch_nest_t<NEST_INIT1>(map, F, box, a, g, s);
    case NEST_STENCIL: return launch_nest_t<NEST_STENCIL>(map, F, box, a, g, s);
    default: return launch_nest_t<NEST_COPY>(map, F, box, a, g, s);
  }
}

int device_sm_count() { return sm_count(); }

static int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

namespace {
// Tuned-stencil configurations (vector width, min CTAs/SM); selectable at run
// time for sweeps (hp_set_stencil_config), default chosen from measurements.
struct StencilCfg {
  int vec, minb;
  void (*fn)(DevFields, const float*, float*, int, int, int, int, int, int, int, float, GosaSink,
             int);
  int tma_stages;   // > 0: TMA-pipelined kernel (stencil_tma.cu) with this many stages
};
const StencilCfg kStencilCfgs[] = {
    {4, 2, k_stencil_3d<4, 2>, 0}, {4, 1, k_stencil_3d<4, 1>, 0}, {2, 3, k_stencil_3d<2, 3>, 0},
    {2, 4, k_stencil_3d<2, 4>, 0}, {2, 2, k_stencil_3d<2, 2>, 0}, {4, 3, k_stencil_3d<4, 3>, 0},
    {4, 1, nullptr, 2},            {4, 1, nullptr, 3},            {4, 1, nullptr, 4}};
constexpr int kNumStencilCfgs = sizeof(kStencilCfgs) / sizeof(kStencilCfgs[0]);
int g_stencil_cfg = 7;   // TMA, 3 stages: best on M/L/XL (profiles/)

int stencil_grid(int cfg) {
  static int g[kNumStencilCfgs] = {};
  if (!kStencilCfgs[cfg].fn) return sm_count();
  if (!g[cfg]) {
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kStencilCfgs[cfg].fn,
                                                      kTileWarps * 32, 0) != cudaSuccess ||
        per_sm < 1)
      per_sm = 1;
    g[cfg] = sm_count() * per_sm;
  }
  return g[cfg];
}

}  // namespace

int g_temporal_blocking = 1;   // two-step passes (stencil_tma.cu), DESIGN.md §5

// on < 0: query only
int set_temporal_blocking(int on) {
  const int old = g_temporal_blocking;
  if (on >= 0) g_temporal_blocking = on ? 1 : 0;
  return old;
}

int stencil_iterations(const DevFields& F, float* buf0, float* buf1, int nn, const LaunchArgs& a,
                       const GosaSink& g, cudaStream_t s, float** last, int* stencil_launches) {
  float* cur = buf0;
  float* oth = buf1;
  int n = 0, it = 0;
  if (g_temporal_blocking && nn - it >= 4) {
    // every two-step pass in one flow launch (stencil_tma.cu)
    const int passes = (nn - it) / 2;
    const int r = launch_stencil_flow(F, F.tma, cur, oth, passes, a, g, s, sm_count());
    if (r < 0) return -1;
    if (r > 0) {
      n += r;
      it += 2 * passes;
      if (stencil_launches) ++*stencil_launches;
      if (passes & 1) {   // the last pass wrote oth
        float* t = cur;
        cur = oth;
        oth = t;
      }
    }
  }
  while (it < nn) {
    int r = 0;
    if (g_temporal_blocking && nn - it >= 2) {
      r = launch_stencil_tb2(F, F.tma, cur, oth, a, g, s, sm_count());
      if (r > 0) it += 2;
    }
    if (r == 0) {
      r = launch_stencil_rotate(F, cur, oth, a, g, s);
      it += 1;
    }
    if (r < 0) return -1;
    n += r;
    if (stencil_launches) ++*stencil_launches;
    float* t = cur;
    cur = oth;
    oth = t;
  }
  *last = cur;
  return n;
}

int set_stencil_config(int cfg) {
  if (cfg < 0 || cfg >= kNumStencilCfgs) return -1;
  g_stencil_cfg = cfg;
  return kNumStencilCfgs;
}

int launch_stencil_rotate(const DevFields& F, const float* p_in, float* p_out,
                          const LaunchArgs& a, const GosaSink& g, cudaStream_t s) {
  const int i_lo = a.li_lo, i_hi = a.li_hi, j_lo = 1, j_hi = a.jmax - 1;
  const int k_lo = 1, k_hi = a.kmax - 1;
  if (i_hi <= i_lo || j_hi <= j_lo || k_hi <= k_lo) {
    // empty interior: the nest body never runs, gosa keeps (or resets to) 0
    Box b{1, 1, 1, 1, 1, 1};
    return launch_nest(NEST_STENCIL, MAP_VECTOR, F, b, a, g, s);
  }
  if (kStencilCfgs[g_stencil_cfg].tma_stages > 0) {
    const int r = launch_stencil_tma(F, F.tma, p_in, p_out, a, g, s,
                                     kStencilCfgs[g_stencil_cfg].tma_stages, sm_count());
    if (r != 0) return r;           // else: no tensor maps -> register kernel below
  }
  const StencilCfg& cfg = kStencilCfgs[kStencilCfgs[g_stencil_cfg].fn ? g_stencil_cfg : 0];
  const int kspan = 32 * cfg.vec;
  const int ktiles = (k_hi + kspan - 1) / kspan;
  const int jtiles = (j_hi - j_lo + kTileWarps - 1) / kTileWarps;
  const long long units = (long long)ktiles * jtiles * (i_hi - i_lo);
  long long grid = stencil_grid(kStencilCfgs[g_stencil_cfg].fn ? g_stencil_cfg : 0);
  if (grid > units) grid = units;
  if (grid > g.capacity) return -1;
  cfg.fn<<<(int)grid, kTileWarps * 32, 0, s>>>(F, p_in, p_out, i_lo, i_hi, j_lo, j_hi, k_lo, k_hi,
                                              ktiles, a.omega, g, a.gosa_reset);
  return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

int launch_stencil_3d(const DevFields& F, const LaunchArgs& a, const GosaSink& g,
                      cudaStream_t s) {
  return launch_stencil_rotate(F, F.f[HP_F_P], F.f[HP_F_WRK2], a, g, s);
}

static int copy_interior_impl(const DevFields& F, const float* src, float* dst,
                              const LaunchArgs& a, cudaStream_t s) {
  const int i_lo = a.li_lo, i_hi = a.li_hi, j_lo = 1, j_hi = a.jmax - 1, k_lo = 1,
            k_hi = a.kmax - 1;
  if (i_hi <= i_lo || j_hi <= j_lo || k_hi <= k_lo) return 0;
  const long long total = (long long)(i_hi - i_lo) * (j_hi - j_lo) * ((k_hi + 3) / 4);
  long long blocks = (total + 255) / 256;
  const long long cap = (long long)sm_count() * 8;
  if (blocks > cap) blocks = cap;
  k_copy_3d<<<(int)blocks, 256, 0, s>>>(F, src, dst, i_lo, i_hi, j_lo, j_hi, k_lo, k_hi);
  return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

int launch_copy_3d(const DevFields& F, const LaunchArgs& a, cudaStream_t s) {
  return copy_interior_impl(F, F.f[HP_F_WRK2], F.f[HP_F_P], a, s);
}

int launch_copy_halo(const DevFields& F, const float* src, float* dst, const LaunchArgs& a,
                     cudaStream_t s) {
  k_copy_halo<<<sm_count() * 4, dim3(64, 4), 0, s>>>(F, src, dst, a.li_lo, a.li_hi, a.jmax,
                                                     a.kmax);
  return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

int launch_repitch(float* dst, size_t dpitch, const float* src, size_t spitch, int width,
                   size_t rows, cudaStream_t s) {
  k_repitch<<<sm_count() * 8, 256, 0, s>>>(dst, dpitch, src, spitch, width, rows);
  return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

int launch_fill(float* dst, size_t n, float value, cudaStream_t s) {
  k_fill<<<sm_count() * 8, 256, 0, s>>>(dst, n, value);
  return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

int launch_stencil_terms(const DevFields& F, const float* p, float* terms, const Box& b,
                         cudaStream_t s) {
  if (b.count() <= 0) return 0;
  const long long need = (b.count() + 255) / 256;
  const int blocks = (int)(need < (long long)sm_count() * 16 ? need : (long long)sm_count() * 16);
  k_stencil_terms<<<blocks, 256, 0, s>>>(F, p, terms, b);
  return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

// interior copy between arbitrary buffers with the program's interior bounds
int launch_copy_interior_bounds(const DevFields& F, const float* src, float* dst,
                                const LaunchArgs& a, cudaStream_t s) {
  return copy_interior_impl(F, src, dst, a, s);
}

}  // namespace hp
