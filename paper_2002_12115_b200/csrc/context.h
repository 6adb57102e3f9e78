// The device context behind hp_ctx (shared by executor.cpp and decomp.cpp).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "coherence.h"
#include "hp_internal.h"

namespace hp {
enum { SLOT_BYTES = 8 };
}  // namespace hp

struct hp_ctx {
  int device = 0;
  int I = 0, J = 0, K = 0, P = 0;
  size_t field_elems = 0;        // I*J*P
  size_t field_stride = 0;       // slab offset between fields (2 MiB aligned)
  cudaStream_t stream = nullptr;
  float* slab = nullptr;         // HP_NFIELDS + 1 (rotation scratch) fields
  hp::DevFields dev{};
  float* scratch = nullptr;      // rotation buffer for the fused time loop
  float* host[HP_NFIELDS] = {};  // pinned [I][J][K]
  unsigned char* hscal = nullptr;   // pinned scalar slots
  unsigned char* dscal = nullptr;   // device scalar slots
  double* partials = nullptr;
  unsigned int* ticket = nullptr;
  int capacity = 0;
  std::vector<int32_t> samples;  // i,j,k triples
  // per-run data-manager state
  uint64_t clock = 0;
  uint64_t host_ver[HP_NVARS] = {}, dev_ver[HP_NVARS] = {};
  bool declared[HP_NVARS] = {};
  int refcount[HP_NVARS] = {};
  bool host_dirty[HP_NFIELDS] = {};  // written since the last fresh-process reset
  hp::Coherence coh[HP_NVARS];           // arrays: which side holds the latest data where
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  uint64_t launches = 0;         // kernels launched by this context (all entry points)
  double* pending_gosa = nullptr;  // hp_jacobi_host_async: where hp_sync delivers gosa
  cudaEvent_t h2d_done = nullptr;  // end of this context's last host-input upload
  // hp_jacobi_host uploads: copy stream + second staging buffer, so the H2D copy of one
  // field overlaps the on-device repitch of the previous one (created on first use)
  cudaStream_t up = nullptr;
  float* stage2 = nullptr;
  cudaEvent_t up_start = nullptr, up_ev[2] = {}, rep_ev[2] = {};
  // slab decomposition (decomp.cpp): this context holds global planes
  // [i_off, i_off + I) of a gI-plane grid; stencil interior = local [li_lo, li_hi)
  int gI = 0, i_off = 0, li_lo = 1, li_hi = 0;
  void* dd = nullptr;            // decomposition state (NCCL communicator, ...)
  float* terms = nullptr;        // HP_FLAG_LITERAL_GOSA: last iteration's ss*ss, [I][J][K]

  hp::GosaSink sink() const {
    hp::GosaSink g;
    g.slot = reinterpret_cast<double*>(dscal + HP_V_GOSA * hp::SLOT_BYTES);
    g.partials = partials;
    g.ticket = ticket;
    g.work = ticket + 1;
    g.capacity = capacity;
    return g;
  }
  hp::HostFields hostf() const {
    hp::HostFields h;
    for (int f = 0; f < HP_NFIELDS; ++f) h.f[f] = host[f];
    h.I = I; h.J = J; h.K = K;
    return h;
  }
  template <class T> T& hs(int v) { return *reinterpret_cast<T*>(hscal + v * hp::SLOT_BYTES); }
};


namespace hp {
// Arguments of the device-resident time loop for this context.
inline LaunchArgs ctx_args(const hp_ctx* c, int reset) {
  LaunchArgs a = grid_args(c->gI - 1, c->J - 1, c->K - 1, 0.8f, reset);
  a.i_off = c->i_off;
  a.li_lo = c->li_lo;
  a.li_hi = c->li_hi;
  return a;
}
// Fused time loop in pieces: begin (scratch faces), step `it` (one stencil
// launch p_it -> p_{it+1}), end (final interior into wrk2 and p).  Return the
// number of kernels launched or -1.
int time_loop_begin(hp_ctx* c, const LaunchArgs& a);
int time_loop_step(hp_ctx* c, int it, const LaunchArgs& a);
int time_loop_end(hp_ctx* c, int nn, const LaunchArgs& a);
int time_loop_finish(hp_ctx* c, float* last, const LaunchArgs& a);
float* time_loop_buffer(hp_ctx* c, int it);   // buffer holding p after `it` steps
void dd_destroy(hp_ctx* c);                   // decomp.cpp
// Whole-field host <-> device copies: one contiguous PCIe transfer through the
// rotation scratch buffer (staging) + an on-device repitch, instead of a
// pitched 2-D copy of K-float rows.  Stream-ordered; `host` is [I][J][K].
cudaError_t field_to_device(hp_ctx* c, float* dev_field, const float* host);
cudaError_t field_to_host(hp_ctx* c, float* host, const float* dev_field);
// allocate a context for a local I x J x K field set (no extent checks)
int create_ctx(int device, int I, int J, int K, hp_ctx** out);
void set_error(const char* fmt, ...);
int cuda_fail(cudaError_t e, const char* what);
}  // namespace hp
