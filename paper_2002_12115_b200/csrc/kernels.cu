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

// ------------------------------------------------------------- reductions

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

// -------------------------------------------------------- generic nest kernel

template <int NEST>
__device__ __forceinline__ void nest_point(const DevFields& F, int i, int j, int k,
                                           const LaunchArgs& a, double& acc) {
  const size_t c = F.at(i, j, k);
  if (NEST == NEST_INIT0) {
    body_init0(F, c);
  } else if (NEST == NEST_INIT1) {
    body_init1(F, c, i, a.imax);
  } else if (NEST == NEST_STENCIL) {
    body_stencil(F, F.f[HP_F_P], F.f[HP_F_WRK2], c, a.omega, acc);
  } else {
    F.f[HP_F_P][c] = F.f[HP_F_WRK2][c];
  }
}

// MAP_COLLAPSE: grid-stride over the linearised box (k fastest).
// MAP_GANG:     block b owns outer index b of the box, threads stride the rest.
// MAP_VECTOR:   one block strides the whole box in strips separated by barriers.
template <int NEST, int MAP>
__global__ void __launch_bounds__(kNestThreads)
k_nest(DevFields F, Box b, LaunchArgs a, GosaSink g) {
  const unsigned nk = (unsigned)b.nk(), nj = (unsigned)b.nj(), ni = (unsigned)b.ni();
  double acc = 0.0;
  if (MAP == MAP_COLLAPSE) {
    const unsigned long long total = (unsigned long long)ni * nj * nk;
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long t = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
         t < total; t += stride) {
      const unsigned k = (unsigned)(t % nk);
      const unsigned long long r = t / nk;
      const unsigned j = (unsigned)(r % nj);
      const unsigned i = (unsigned)(r / nj);
      nest_point<NEST>(F, b.i0 + i, b.j0 + j, b.k0 + k, a, acc);
    }
  } else if (MAP == MAP_GANG) {
    // outer dimension = first non-degenerate of (i, j); a row box is gang+vector over k
    if (ni > 1) {
      const unsigned i = blockIdx.x;
      for (unsigned t = threadIdx.x; t < nj * nk; t += blockDim.x)
        nest_point<NEST>(F, b.i0 + i, b.j0 + t / nk, b.k0 + t % nk, a, acc);
    } else if (nj > 1) {
      const unsigned j = blockIdx.x;
      for (unsigned t = threadIdx.x; t < nk; t += blockDim.x)
        nest_point<NEST>(F, b.i0, b.j0 + j, b.k0 + t, a, acc);
    } else {
      const unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
      if (t < nk) nest_point<NEST>(F, b.i0, b.j0, b.k0 + t, a, acc);
    }
  } else {
    const unsigned long long total = (unsigned long long)ni * nj * nk;
    for (unsigned long long base = 0; base < total; base += blockDim.x) {
      const unsigned long long t = base + threadIdx.x;
      if (t < total) {
        const unsigned k = (unsigned)(t % nk);
        const unsigned long long r = t / nk;
        nest_point<NEST>(F, b.i0 + (unsigned)(r / nj), b.j0 + (unsigned)(r % nj), b.k0 + k,
                         a, acc);
      }
      __syncthreads();  // strip boundary: all reads of a strip precede the next strip
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

__device__ __forceinline__ float4 ld4(const float* ptr) {
  return *reinterpret_cast<const float4*>(ptr);
}

__device__ __forceinline__ float elem(const float4& v, int e) {
  return e == 0 ? v.x : (e == 1 ? v.y : (e == 2 ? v.z : v.w));
}

// k-1 neighbour of element 0 and k+1 neighbour of element 3 of a row quad
struct Edge { float left, right; };

__device__ __forceinline__ Edge row_edges(const float4& v, const float* row_at_quad, int lane) {
  Edge e;
  e.left = __shfl_up_sync(0xffffffffu, v.w, 1);
  e.right = __shfl_down_sync(0xffffffffu, v.x, 1);
  if (lane == 0) e.left = row_at_quad[-1];
  if (lane == 31) e.right = row_at_quad[4];
  return e;
}

__device__ __forceinline__ float km1(const float4& v, const Edge& e, int x) {
  return x == 0 ? e.left : elem(v, x - 1);
}
__device__ __forceinline__ float kp1(const float4& v, const Edge& e, int x) {
  return x == 3 ? e.right : elem(v, x + 1);
}

// Interior = i in [i_lo, i_hi), j in [j_lo, j_hi), k in [k_lo, k_hi).
// grid: x = k tiles (128 k), y = j tiles (8 rows), z = i chunks.
__global__ void __launch_bounds__(kTileWarps * 32, kTargetCtasPerSm)
k_stencil_3d(DevFields F, const float* __restrict__ pin, float* __restrict__ out,
             int i_lo, int i_hi, int chunk, int j_lo, int j_hi, int k_lo, int k_hi,
             float omega, GosaSink g, int reset) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int quad = blockIdx.x * kQuadsPerWarp + lane;
  const int kb = quad * 4;                         // first k of this thread's quad
  const int j = j_lo + blockIdx.y * kTileWarps + w;
  const int i0 = i_lo + blockIdx.z * chunk;
  const int i1 = min(i0 + chunk, i_hi);
  const size_t P = F.P, L = F.plane();
  double acc = 0.0;

  // whole warp shares j, so this test is warp-uniform and shuffles stay legal
  if (j < j_hi && i0 < i1) {
    const bool active = kb + 3 >= k_lo && kb < k_hi;  // quad overlaps [k_lo, k_hi)
    bool ok[4];
#pragma unroll
    for (int x = 0; x < 4; ++x) ok[x] = active && kb + x >= k_lo && kb + x < k_hi;
    const bool full = ok[0] && ok[1] && ok[2] && ok[3];

    size_t c = F.at(i0, j, kb);
    // register queue along i: rows (j-1, j, j+1) of planes i-1 (l*), i (m*), i+1 (n*)
    float4 l0 = ld4(pin + c - L), lm = ld4(pin + c - L - P), lp = ld4(pin + c - L + P);
    float4 m0 = ld4(pin + c), mm = ld4(pin + c - P), mp = ld4(pin + c + P);
    for (int i = i0; i < i1; ++i, c += L) {
      const float4 n0 = ld4(pin + c + L), nm = ld4(pin + c + L - P), np = ld4(pin + c + L + P);
      const float4 A0 = ldg_stream(F.f[HP_F_A0] + c), A1 = ldg_stream(F.f[HP_F_A1] + c);
      const float4 A2 = ldg_stream(F.f[HP_F_A2] + c), A3 = ldg_stream(F.f[HP_F_A3] + c);
      const float4 B0 = ldg_stream(F.f[HP_F_B0] + c), B1 = ldg_stream(F.f[HP_F_B1] + c);
      const float4 B2 = ldg_stream(F.f[HP_F_B2] + c), C0 = ldg_stream(F.f[HP_F_C0] + c);
      const float4 C1 = ldg_stream(F.f[HP_F_C1] + c), C2 = ldg_stream(F.f[HP_F_C2] + c);
      const float4 W1 = ldg_stream(F.f[HP_F_WRK1] + c), BN = ldg_stream(F.f[HP_F_BND] + c);

      const Edge eL = row_edges(l0, pin + c - L, lane);
      const Edge eN = row_edges(n0, pin + c + L, lane);
      const Edge eM = row_edges(m0, pin + c, lane);
      const Edge eMm = row_edges(mm, pin + c - P, lane);
      const Edge eMp = row_edges(mp, pin + c + P, lane);

      float r[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        Coef q;
        q.a0 = elem(A0, x); q.a1 = elem(A1, x); q.a2 = elem(A2, x); q.a3 = elem(A3, x);
        q.b0 = elem(B0, x); q.b1 = elem(B1, x); q.b2 = elem(B2, x);
        q.c0 = elem(C0, x); q.c1 = elem(C1, x); q.c2 = elem(C2, x);
        q.wrk1 = elem(W1, x); q.bnd = elem(BN, x);
        const float n[19] = {
            elem(n0, x), elem(mp, x), kp1(m0, eM, x),
            elem(np, x), elem(nm, x), elem(lp, x), elem(lm, x),
            kp1(mp, eMp, x), kp1(mm, eMm, x), km1(mp, eMp, x), km1(mm, eMm, x),
            kp1(n0, eN, x), kp1(l0, eL, x), km1(n0, eN, x), km1(l0, eL, x),
            elem(l0, x), elem(mm, x), km1(m0, eM, x), elem(m0, x)};
        const float ss = stencil_ss(q, n);
        r[x] = add(n[18], mul(omega, ss));
        if (ok[x]) acc += (double)mul(ss, ss);
      }
      if (full) {
        *reinterpret_cast<float4*>(out + c) = make_float4(r[0], r[1], r[2], r[3]);
      } else if (active) {
#pragma unroll
        for (int x = 0; x < 4; ++x)
          if (ok[x]) out[c + x] = r[x];
      }
      lm = mm; l0 = m0; lp = mp;
      mm = nm; m0 = n0; mp = np;
    }
  }
  const int nblocks = gridDim.x * gridDim.y * gridDim.z;
  const int bid = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
  gosa_commit(g, acc, nblocks, bid, reset);
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
                            int imax, int jmax, int kmax) {
  const long long rows = (long long)F.I * F.J;
  for (long long r = (long long)blockIdx.x * blockDim.y + threadIdx.y; r < rows;
       r += (long long)gridDim.x * blockDim.y) {
    const int i = (int)(r / F.J), j = (int)(r % F.J);
    const size_t base = F.at(i, j, 0);
    const bool whole = i == 0 || i >= imax - 1 || j == 0 || j >= jmax - 1;
    if (whole) {
      for (int k = threadIdx.x; k < F.K; k += blockDim.x) dst[base + k] = src[base + k];
    } else {
      if (threadIdx.x == 0) dst[base] = src[base];
      for (int k = kmax - 1 + threadIdx.x; k < F.K; k += blockDim.x) dst[base + k] = src[base + k];
    }
  }
}

__global__ void k_fill(float* dst, size_t n, float v) {
  for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (size_t)gridDim.x * blockDim.x)
    dst[t] = v;
}

template <int NEST>
int launch_nest_t(Mapping map, const DevFields& F, const Box& b, const LaunchArgs& a,
                  const GosaSink& g, cudaStream_t s) {
  if (b.count() <= 0) {
    return 0;
  }
  int blocks = 1;
  if (map == MAP_COLLAPSE) {
    const long long need = (b.count() + kNestThreads - 1) / kNestThreads;
    blocks = (int)(need < kMaxCollapseBlocks ? need : kMaxCollapseBlocks);
  } else if (map == MAP_GANG) {
    if (b.ni() > 1) blocks = (int)b.ni();
    else if (b.nj() > 1) blocks = (int)b.nj();
    else blocks = (int)((b.nk() + kNestThreads - 1) / kNestThreads);
  }
  if (NEST == NEST_STENCIL && blocks > g.capacity) return -1;
  if (map == MAP_COLLAPSE) k_nest<NEST, MAP_COLLAPSE><<<blocks, kNestThreads, 0, s>>>(F, b, a, g);
  else if (map == MAP_GANG) k_nest<NEST, MAP_GANG><<<blocks, kNestThreads, 0, s>>>(F, b, a, g);
  else k_nest<NEST, MAP_VECTOR><<<1, kNestThreads, 0, s>>>(F, b, a, g);
  return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

}  // namespace

static int sm_count();

int gosa_capacity_needed(const DevFields& F) {
  const int tiles = ((F.K + 127) / 128) * ((F.J + kTileWarps - 1) / kTileWarps);
  const int want = sm_count() * kTargetCtasPerSm * 2;
  return kMaxCollapseBlocks + F.I + F.J + tiles + want + 1024;
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

int launch_stencil_rotate(const DevFields& F, const float* p_in, float* p_out,
                          const LaunchArgs& a, const GosaSink& g, cudaStream_t s) {
  const int i_lo = 1, i_hi = a.imax - 1, j_lo = 1, j_hi = a.jmax - 1;
  const int k_lo = 1, k_hi = a.kmax - 1;
  if (i_hi <= i_lo || j_hi <= j_lo || k_hi <= k_lo) {
    // empty interior: the nest body never runs, gosa keeps (or resets to) 0
    Box b{1, 1, 1, 1, 1, 1};
    return launch_nest_t<NEST_STENCIL>(MAP_VECTOR, F, b, a, g, s);
  }
  const int ktiles = (k_hi + 4 * kQuadsPerWarp - 1) / (4 * kQuadsPerWarp);
  const int jtiles = (j_hi - j_lo + kTileWarps - 1) / kTileWarps;
  const int ni = i_hi - i_lo;
  const int want = sm_count() * kTargetCtasPerSm * 2;
  int chunks = (want + ktiles * jtiles - 1) / (ktiles * jtiles);
  if (chunks < 1) chunks = 1;
  if (chunks > ni) chunks = ni;
  int chunk = (ni + chunks - 1) / chunks;
  chunks = (ni + chunk - 1) / chunk;
  if ((long long)ktiles * jtiles * chunks > g.capacity) return -1;
  dim3 grid(ktiles, jtiles, chunks);
  k_stencil_3d<<<grid, kTileWarps * 32, 0, s>>>(F, p_in, p_out, i_lo, i_hi, chunk, j_lo, j_hi,
                                               k_lo, k_hi, a.omega, g, a.gosa_reset);
  return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

int launch_stencil_3d(const DevFields& F, const LaunchArgs& a, const GosaSink& g,
                      cudaStream_t s) {
  return launch_stencil_rotate(F, F.f[HP_F_P], F.f[HP_F_WRK2], a, g, s);
}

static int copy_interior_impl(const DevFields& F, const float* src, float* dst, int imax,
                              int jmax, int kmax, cudaStream_t s) {
  const int i_lo = 1, i_hi = imax - 1, j_lo = 1, j_hi = jmax - 1, k_lo = 1, k_hi = kmax - 1;
  if (i_hi <= i_lo || j_hi <= j_lo || k_hi <= k_lo) return 0;
  const long long total = (long long)(i_hi - i_lo) * (j_hi - j_lo) * ((k_hi + 3) / 4);
  long long blocks = (total + 255) / 256;
  const long long cap = (long long)sm_count() * 8;
  if (blocks > cap) blocks = cap;
  k_copy_3d<<<(int)blocks, 256, 0, s>>>(F, src, dst, i_lo, i_hi, j_lo, j_hi, k_lo, k_hi);
  return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

int launch_copy_3d(const DevFields& F, const LaunchArgs& a, cudaStream_t s) {
  return copy_interior_impl(F, F.f[HP_F_WRK2], F.f[HP_F_P], a.imax, a.jmax, a.kmax, s);
}

int launch_copy_halo(const DevFields& F, const float* src, float* dst, int imax, int jmax,
                     int kmax, cudaStream_t s) {
  k_copy_halo<<<sm_count() * 4, dim3(64, 4), 0, s>>>(F, src, dst, imax, jmax, kmax);
  return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

int launch_fill(float* dst, size_t n, float value, cudaStream_t s) {
  k_fill<<<sm_count() * 8, 256, 0, s>>>(dst, n, value);
  return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

// interior copy between arbitrary buffers with the program's interior bounds
int launch_copy_interior_bounds(const DevFields& F, const float* src, float* dst, int imax,
                                int jmax, int kmax, cudaStream_t s) {
  return copy_interior_impl(F, src, dst, imax, jmax, kmax, s);
}

}  // namespace hp
