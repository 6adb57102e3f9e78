// Internal declarations shared by kernels.cu and executor.cpp.
//
// Device layout: each fp32 field is a
// pitched [I][J][P] array, P = round_up(K, 32) floats, so every (i, j) row
// starts on a 128-byte boundary and float4 loads of k-quads are aligned.
// All 14 fields live in one slab, each at a 2 MiB-aligned offset.
// Host copies (the program's static arrays) are unpadded [I][J][K] in pinned
// memory; transfers are 2-D copies (K floats per row).
#pragma once

#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

#include "../../include/himeno_b200.h"

namespace hp {

constexpr int kRowAlign = 32;           // floats per pitch quantum (128 B)

struct DevFields {
  float* f[HP_NFIELDS];                 // device mirrors
  int I, J, K, P;                       // extents and row pitch (floats)
  const void* tma;                      // host handle: TMA tensor maps (stencil_tma.cu)
  __host__ __device__ size_t plane() const { return (size_t)J * (size_t)P; }
  __host__ __device__ size_t at(int i, int j, int k) const {
    return ((size_t)i * (size_t)J + (size_t)j) * (size_t)P + (size_t)k;
  }
};

struct Box {                            // half-open [i0,i1) x [j0,j1) x [k0,k1)
  int i0, i1, j0, j1, k0, k1;
  __host__ __device__ long long ni() const { return i1 > i0 ? i1 - i0 : 0; }
  __host__ __device__ long long nj() const { return j1 > j0 ? j1 - j0 : 0; }
  __host__ __device__ long long nk() const { return k1 > k0 ? k1 - k0 : 0; }
  __host__ __device__ long long count() const { return ni() * nj() * nk(); }
};

// Deterministic gosa reduction target: each block writes a partial, the last
// block to finish sums the partials in block order and adds (or stores, when
// `reset`) the total into *slot (the device copy of jacobi's gosa).
struct GosaSink {
  double* slot;
  double* partials;
  unsigned int* ticket;
  int capacity;                         // number of partial slots
  unsigned int* work;                   // dynamic work-queue counter (TMA kernels)
};

enum Nest { NEST_INIT0 = 0, NEST_INIT1 = 1, NEST_STENCIL = 2, NEST_COPY = 3 };

// Mapping of a loop-nest execution onto the device (selected by hp_kind).
enum Mapping {
  MAP_COLLAPSE = 0,   // kernels: every point of the box is one thread
  MAP_GANG = 1,       // parallel loop: one CTA per iteration of the box's outer dim
  MAP_VECTOR = 2      // parallel loop vector: a single CTA strides the box
};

struct LaunchArgs {
  int imax, jmax, kmax;                 // program scalars (by value; global grid)
  float omega;
  int gosa_reset;                       // stencil: store instead of accumulate
  int i_off;                            // global i of local plane 0 (slab contexts)
  int li_lo, li_hi;                     // local planes of the stencil interior
};

// Full-grid arguments: local == global planes, interior [1, imax-1).
inline LaunchArgs grid_args(int imax, int jmax, int kmax, float omega, int reset) {
  LaunchArgs a;
  a.imax = imax; a.jmax = jmax; a.kmax = kmax; a.omega = omega; a.gosa_reset = reset;
  a.i_off = 0; a.li_lo = 1; a.li_hi = imax - 1;
  return a;
}

// ---- kernels.cu launchers (all enqueue on `s`, no host sync) ----------------
// Returns number of kernels launched (>=0) or -1 on launch error.
int launch_nest(Nest nest, Mapping map, const DevFields& F, const Box& box,
                const LaunchArgs& a, const GosaSink& g, cudaStream_t s);
// Tuned full-interior stencil (2.5-D blocked, float4) and copy.
int launch_stencil_3d(const DevFields& F, const LaunchArgs& a, const GosaSink& g,
                      cudaStream_t s);
int launch_copy_3d(const DevFields& F, const LaunchArgs& a, cudaStream_t s);
// Fused time-loop step: reads p_in, writes p_out (interior) -- wrk2 semantics
// restored at the end of the loop by launch_time_loop_finish.
int launch_stencil_rotate(const DevFields& F, const float* p_in, float* p_out,
                          const LaunchArgs& a, const GosaSink& g, cudaStream_t s);
int launch_fill(float* dst, size_t n, float value, cudaStream_t s);
// ss*ss of each point of box b (stencil over p) -> terms[(i*J + j)*K + k]
int launch_stencil_terms(const DevFields& F, const float* p, float* terms, const Box& b,
                         cudaStream_t s);
// dst[r*dpitch + c] = src[r*spitch + c] for r < rows, c < width (elements)
int launch_repitch(float* dst, size_t dpitch, const float* src, size_t spitch, int width,
                   size_t rows, cudaStream_t s);
// dst = src on every point outside the stencil interior (local planes outside
// [li_lo, li_hi) included whole)
int launch_copy_halo(const DevFields& F, const float* src, float* dst, const LaunchArgs& a,
                     cudaStream_t s);
// dst = src on the interior [li_lo,li_hi) x [1,jmax-1) x [1,kmax-1)
int launch_copy_interior_bounds(const DevFields& F, const float* src, float* dst,
                                const LaunchArgs& a, cudaStream_t s);
int gosa_capacity_needed(const DevFields& F);
// select the tuned-stencil configuration; returns the number of configs or -1
int set_stencil_config(int cfg);
// stencil_tma.cu: tensor maps of one context and the TMA-pipelined stencil
void* create_stencil_tma(const DevFields& F, const float* scratch);
void destroy_stencil_tma(void* h);
int launch_stencil_tma(const DevFields& F, const void* h, const float* p_in, float* p_out,
                       const LaunchArgs& a, const GosaSink& g, cudaStream_t s, int stages,
                       int sms);
// two Jacobi iterations per pass (temporal blocking); 0 = not applicable
int launch_stencil_tb2(const DevFields& F, const void* h, const float* p_in, float* p_out,
                       const LaunchArgs& a, const GosaSink& g, cudaStream_t s, int sms);
// one two-step pass of a slab in two parts (halo exchange overlapped with the
// interior): part 1 = boundary plane pairs, part 2 = interior on <= sms - reserve
// CTAs; 0 = slab too thin
int launch_stencil_tb2_part(const DevFields& F, const void* h, const float* p_in, float* p_out,
                            const LaunchArgs& a, const GosaSink& g, cudaStream_t s, int sms,
                            int part, int reserve);
// one two-step pass of a slab as one launch, boundary units first, each counted in
// *sig as it finishes (*nb_out = boundary units); 0 = slab too thin
int launch_stencil_tb2_signaled(const DevFields& F, const void* h, const float* p_in,
                                float* p_out, const LaunchArgs& a, const GosaSink& g,
                                cudaStream_t s, int sms, int reserve, unsigned* sig, int* nb_out);
// `passes` >= 2 two-step passes in ONE launch (units of pass t+1 start as soon as
// their neighbourhood in pass t is done); result in p_out if passes is odd, else
// p_in; 0 = not applicable (caller launches pass by pass)
int launch_stencil_flow(const DevFields& F, const void* h, const float* p_in, float* p_out,
                        int passes, const LaunchArgs& a, const GosaSink& g, cudaStream_t s,
                        int sms);
// 1 if the device time loop of this geometry runs its two-step passes as one flow
// launch (policy of launch_stencil_flow), else 0
int stencil_flow_ok(const DevFields& F, const LaunchArgs& a, int sms);
int device_sm_count();   // kernels.cu
// run iterations [0, nn) p_in -> ... choosing one- or two-step passes; sets
// *last to the buffer holding p_nn; returns kernels launched or -1
int stencil_iterations(const DevFields& F, float* buf0, float* buf1, int nn, const LaunchArgs& a,
                       const GosaSink& g, cudaStream_t s, float** last, int* stencil_launches);
int set_temporal_blocking(int on);
// raise a kernel's dynamic shared-memory limit on the current device (once per
// kernel and device); false if the runtime refuses
bool ensure_smem_optin(const void* func, int bytes);
// exchange-kernel launches are chained per device across streams (stencil_tma.cu);
// a stream about to be destroyed must be dropped from that chain
void tx_forget_stream(cudaStream_t s);
// 1 if an exchange launch of this context timed out waiting for a neighbour, 0 if
// not, -1 on a CUDA error (synchronous read)
int tx_error(const void* tma);
const void* smem_kernel(int id);   // the opted-in kernels by id (hp_smem_optin)
void set_error(const char* fmt, ...);   // executor.cpp: hp_last_error() text
int cuda_fail(cudaError_t e, const char* what);

// ---- host loop bodies (executor.cpp), same arithmetic as the kernels --------
struct HostFields {
  float* f[HP_NFIELDS];
  int I, J, K;
  size_t at(int i, int j, int k) const {
    return ((size_t)i * (size_t)J + (size_t)j) * (size_t)K + (size_t)k;
  }
};

}  // namespace hp
