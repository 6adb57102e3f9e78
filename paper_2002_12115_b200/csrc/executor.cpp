// Schedule executor + device data manager for the Himeno program (C ABI in
// include/himeno_b200.h).
//
// One hp_run() = one execution of the program the reference would have
// compiled and timed (acctuner/evaluators.py:190-222), under one gene pattern:
//
//   main:   imax = I-1; jmax = J-1; kmax = K-1; omega = 0.8      (host)
//           initmt():  nest(0,1,2) zero, nest(3,4,5) coefficients
//           gosa = jacobi(nn): loop 6 { gosa = 0; nest(7,8,9); nest(10,11,12) }
//           print gosa and the p samples                          (host copies)
//
// Every loop statement is executed by `run_loop`: fire the plan events
// attached before it, then either launch the device kernel variant selected
// by its directive kind (gene = 1: the loop is an anchor), or iterate it on
// the host (gene = 0) -- descending into children only when something below
// needs it (a device anchor or an event), else running the whole sub-nest as
// a tight C++ loop -- and fire the events attached after it.
//
// Data manager: every variable has a host and a
// device copy with a write version each.  Plan events execute literally
// (update device/self, structured data enter/exit with present_or_copy
// reference counts, declare create); kernels touching arrays that are not
// present get implicit present_or_copy around the launch (the per-kernel
// copies the paper's batching removes).  With HP_FLAG_COHERENCE_GUARD a
// transfer whose source copy is older than its destination is skipped and
// counted (n_skipped_stale) instead of clobbering newer data.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "context.h"
#include "host_loops.h"

using namespace hp;

// NVTX ranges (header-only NVTX3: a no-op unless a profiler is attached): one per
// program run, per loop execution (device launch / host nest, by loop id) and per
// transfer, so an nsys/ncu timeline reads in the program's own terms.
namespace {
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
};
const char* loop_range_name(int loop, bool device) {
  static const char* const dev[HP_NLOOPS] = {
      "loop 0 device", "loop 1 device", "loop 2 device", "loop 3 device", "loop 4 device",
      "loop 5 device", "loop 6 device", "loop 7 device", "loop 8 device", "loop 9 device",
      "loop 10 device", "loop 11 device", "loop 12 device"};
  static const char* const host[HP_NLOOPS] = {
      "loop 0 host", "loop 1 host", "loop 2 host", "loop 3 host", "loop 4 host",
      "loop 5 host", "loop 6 host", "loop 7 host", "loop 8 host", "loop 9 host",
      "loop 10 host", "loop 11 host", "loop 12 host"};
  return loop >= 0 && loop < HP_NLOOPS ? (device ? dev[loop] : host[loop]) : "loop";
}
}  // namespace

// ------------------------------------------------------------------ errors

static thread_local std::string g_last_error;

void hp::set_error(const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
}

extern "C" const char* hp_last_error(void) { return g_last_error.c_str(); }
extern "C" int hp_abi_version(void) { return HP_ABI_VERSION; }

extern "C" int hp_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

// --------------------------------------------------------- program tables

namespace {

struct VarInfo {
  const char* name;
  int nfields;          // >0: array var made of fields [f0, f0 + nfields)
  int f0;
  int bytes;            // scalar size (0 for arrays)
};

const VarInfo kVars[HP_NVARS] = {
    {"p", 1, HP_F_P, 0},        {"bnd", 1, HP_F_BND, 0},   {"wrk1", 1, HP_F_WRK1, 0},
    {"wrk2", 1, HP_F_WRK2, 0},  {"a", 4, HP_F_A0, 0},      {"b", 3, HP_F_B0, 0},
    {"c", 3, HP_F_C0, 0},       {"imax", 0, 0, 4},         {"jmax", 0, 0, 4},
    {"kmax", 0, 0, 4},          {"omega", 0, 0, 4},        {"jacobi:nn", 0, 0, 4},
    {"jacobi:gosa", 0, 0, 8},   {"jacobi:s0", 0, 0, 4},    {"jacobi:ss", 0, 0, 4},
    {"main:gosa", 0, 0, 4}};

// loop id -> nest and level; loop 6 is the time loop
constexpr int kNestOf[HP_NLOOPS] = {NEST_INIT0, NEST_INIT0, NEST_INIT0, NEST_INIT1, NEST_INIT1,
                                   NEST_INIT1, -1,         NEST_STENCIL, NEST_STENCIL,
                                   NEST_STENCIL, NEST_COPY, NEST_COPY,   NEST_COPY};
constexpr int kLevelOf[HP_NLOOPS] = {0, 1, 2, 0, 1, 2, -1, 0, 1, 2, 0, 1, 2};
constexpr int kParentOf[HP_NLOOPS] = {-1, 0, 1, -1, 3, 4, -1, 6, 7, 8, 6, 10, 11};
constexpr int kNestLoops[4][3] = {{0, 1, 2}, {3, 4, 5}, {7, 8, 9}, {10, 11, 12}};

// variables each nest's body touches (reads, writes); scalars read by value
struct NestVars { std::vector<int> arrays; std::vector<int> writes; bool gosa; };

const NestVars& nest_vars(int nest) {
  static const NestVars v[4] = {
      {{HP_V_P, HP_V_BND, HP_V_WRK1, HP_V_A, HP_V_B, HP_V_C},
       {HP_V_P, HP_V_BND, HP_V_WRK1, HP_V_A, HP_V_B, HP_V_C}, false},
      {{HP_V_P, HP_V_BND, HP_V_WRK1, HP_V_A, HP_V_B, HP_V_C},
       {HP_V_P, HP_V_BND, HP_V_WRK1, HP_V_A, HP_V_B, HP_V_C}, false},
      {{HP_V_P, HP_V_BND, HP_V_WRK1, HP_V_WRK2, HP_V_A, HP_V_B, HP_V_C}, {HP_V_WRK2}, true},
      {{HP_V_P, HP_V_WRK2}, {HP_V_P}, false}};
  return v[nest];
}

double now_s() {
  using clk = std::chrono::steady_clock;
  return std::chrono::duration<double>(clk::now().time_since_epoch()).count();
}

size_t round_up(size_t x, size_t q) { return (x + q - 1) / q * q; }

}  // namespace

// ------------------------------------------------------------------ context

cudaError_t hp::field_to_device(hp_ctx* c, float* dev_field, const float* host) {
  const size_t n = (size_t)c->I * c->J * c->K;
  cudaError_t e = cudaMemcpyAsync(c->scratch, host, n * sizeof(float), cudaMemcpyHostToDevice,
                                  c->stream);
  if (e != cudaSuccess) return e;
  if (launch_repitch(dev_field, (size_t)c->P, c->scratch, (size_t)c->K, c->K,
                     (size_t)c->I * c->J, c->stream) < 0)
    return cudaGetLastError();
  return cudaSuccess;
}

cudaError_t hp::field_to_host(hp_ctx* c, float* host, const float* dev_field) {
  const size_t n = (size_t)c->I * c->J * c->K;
  if (launch_repitch(c->scratch, (size_t)c->K, dev_field, (size_t)c->P, c->K,
                     (size_t)c->I * c->J, c->stream) < 0)
    return cudaGetLastError();
  return cudaMemcpyAsync(host, c->scratch, n * sizeof(float), cudaMemcpyDeviceToHost, c->stream);
}

// p -> scratch -> p ... ; faces of scratch mirror p's; the final interior goes
// to p (if it ended in scratch) and to wrk2, so p/wrk2/gosa match the unfused loop.
float* hp::time_loop_buffer(hp_ctx* c, int it) {
  return (it & 1) ? c->scratch : c->dev.f[HP_F_P];
}
int hp::time_loop_begin(hp_ctx* c, const LaunchArgs& a) {
  return launch_copy_halo(c->dev, c->dev.f[HP_F_P], c->scratch, a, c->stream);
}
int hp::time_loop_step(hp_ctx* c, int it, const LaunchArgs& a) {
  return launch_stencil_rotate(c->dev, time_loop_buffer(c, it), time_loop_buffer(c, it + 1), a,
                               c->sink(), c->stream);
}
int hp::time_loop_end(hp_ctx* c, int nn, const LaunchArgs& a) {
  return time_loop_finish(c, time_loop_buffer(c, nn), a);
}
int hp::time_loop_finish(hp_ctx* c, float* last, const LaunchArgs& a) {
  int n = 0, r;
  if ((r = launch_copy_interior_bounds(c->dev, last, c->dev.f[HP_F_WRK2], a, c->stream)) < 0)
    return -1;
  n += r;
  if (last != c->dev.f[HP_F_P]) {
    if ((r = launch_copy_interior_bounds(c->dev, last, c->dev.f[HP_F_P], a, c->stream)) < 0)
      return -1;
    n += r;
  }
  return n;
}

int hp::cuda_fail(cudaError_t e, const char* what) {
  set_error("%s: %s", what, cudaGetErrorString(e));
  return e == cudaErrorMemoryAllocation ? HP_ERR_OOM : HP_ERR_DEVICE;
}

#define CK(call, what)                         \
  do {                                         \
    cudaError_t e_ = (call);                   \
    if (e_ != cudaSuccess) return cuda_fail(e_, what); \
  } while (0)

static void forget_upload(hp_ctx* c);

extern "C" void hp_destroy(hp_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  forget_upload(c);
  if (c->h2d_done) cudaEventDestroy(c->h2d_done);
  if (c->up) {
    cudaStreamSynchronize(c->up);
    cudaStreamDestroy(c->up);
  }
  for (cudaEvent_t e : {c->up_start, c->up_ev[0], c->up_ev[1], c->rep_ev[0], c->rep_ev[1]})
    if (e) cudaEventDestroy(e);
  if (c->stage2) cudaFree(c->stage2);
  if (c->dd) dd_destroy(c);
  if (c->dev.tma) destroy_stencil_tma(const_cast<void*>(c->dev.tma));
  if (c->slab) cudaFree(c->slab);
  if (c->dscal) cudaFree(c->dscal);
  if (c->partials) cudaFree(c->partials);
  if (c->ticket) cudaFree(c->ticket);
  if (c->terms) cudaFree(c->terms);
  for (float* h : c->host)
    if (h) cudaFreeHost(h);
  if (c->hscal) cudaFreeHost(c->hscal);
  if (c->stream) {
    tx_forget_stream(c->stream);
    cudaStreamDestroy(c->stream);
  }
  delete c;
}

extern "C" int hp_create(int device, const hp_grid* grid, int flags, hp_ctx** out) {
  (void)flags;
  if (!grid || !out) {
    set_error("hp_create: null argument");
    return HP_ERR_ARG;
  }
  *out = nullptr;
  if (grid->I < 4 || grid->J < 4 || grid->K < 4) {
    set_error("hp_create: extents must be >= 4 (got %d x %d x %d)", grid->I, grid->J, grid->K);
    return HP_ERR_ARG;
  }
  return hp::create_ctx(device, grid->I, grid->J, grid->K, out);
}

int hp::create_ctx(int device, int I, int J, int K, hp_ctx** out) {
  *out = nullptr;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) {
    set_error("no CUDA device available (%s)", cudaGetErrorString(e));
    cudaGetLastError();
    return HP_ERR_DEVICE;
  }
  if (device < 0 || device >= ndev) {
    set_error("device %d out of range (have %d)", device, ndev);
    return HP_ERR_ARG;
  }
  hp_ctx* c = new (std::nothrow) hp_ctx;
  if (!c) {
    set_error("out of host memory");
    return HP_ERR_OOM;
  }
  c->device = device;
  c->I = I; c->J = J; c->K = K;
  c->gI = c->I; c->i_off = 0; c->li_lo = 1; c->li_hi = c->I - 2;
  c->P = (int)round_up((size_t)c->K + 4, kRowAlign);
  c->field_elems = (size_t)c->I * c->J * c->P;
  c->field_stride = round_up(c->field_elems, (size_t)1 << 19);  // 2 MiB of floats
  int rc = HP_OK;
  auto fail = [&](int code) { hp_destroy(c); return code; };
  if ((e = cudaSetDevice(device)) != cudaSuccess) return fail(cuda_fail(e, "cudaSetDevice"));
  if ((e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking)) != cudaSuccess)
    return fail(cuda_fail(e, "cudaStreamCreate"));
  const size_t slab_elems = c->field_stride * (HP_NFIELDS + 1);
  if ((e = cudaMalloc(&c->slab, slab_elems * sizeof(float))) != cudaSuccess)
    return fail(cuda_fail(e, "cudaMalloc(field slab)"));
  c->dev.I = c->I; c->dev.J = c->J; c->dev.K = c->K; c->dev.P = c->P;
  for (int f = 0; f < HP_NFIELDS; ++f) c->dev.f[f] = c->slab + (size_t)f * c->field_stride;
  c->scratch = c->slab + (size_t)HP_NFIELDS * c->field_stride;
  const size_t host_bytes = (size_t)c->I * c->J * c->K * sizeof(float);
  for (int f = 0; f < HP_NFIELDS; ++f) {
    if ((e = cudaHostAlloc(&c->host[f], host_bytes, cudaHostAllocPortable)) != cudaSuccess)
      return fail(cuda_fail(e, "cudaHostAlloc(host field)"));
    memset(c->host[f], 0, host_bytes);
  }
  if ((e = cudaHostAlloc(&c->hscal, HP_NVARS * SLOT_BYTES, cudaHostAllocPortable)) != cudaSuccess)
    return fail(cuda_fail(e, "cudaHostAlloc(scalars)"));
  memset(c->hscal, 0, HP_NVARS * SLOT_BYTES);
  if ((e = cudaMalloc(&c->dscal, HP_NVARS * SLOT_BYTES)) != cudaSuccess)
    return fail(cuda_fail(e, "cudaMalloc(scalars)"));
  c->capacity = gosa_capacity_needed(c->dev);
  if ((e = cudaMalloc(&c->partials, (size_t)c->capacity * sizeof(double))) != cudaSuccess)
    return fail(cuda_fail(e, "cudaMalloc(partials)"));
  // [0]: last-block ticket of the gosa reduction, [1]: work-queue counter
  if ((e = cudaMalloc(&c->ticket, 2 * sizeof(unsigned int))) != cudaSuccess)
    return fail(cuda_fail(e, "cudaMalloc(ticket)"));
  cudaMemsetAsync(c->ticket, 0, 2 * sizeof(unsigned int), c->stream);
  cudaMemsetAsync(c->dscal, 0, HP_NVARS * SLOT_BYTES, c->stream);
  cudaMemsetAsync(c->slab, 0, slab_elems * sizeof(float), c->stream);
  cudaEventCreate(&c->ev0);
  cudaEventCreate(&c->ev1);
  c->dev.tma = create_stencil_tma(c->dev, c->scratch);   // nullptr: register kernel only
  if ((e = cudaStreamSynchronize(c->stream)) != cudaSuccess)
    return fail(cuda_fail(e, "context init"));
  (void)rc;
  *out = c;
  return HP_OK;
}

extern "C" void* hp_stream(hp_ctx* c) { return c ? (void*)c->stream : nullptr; }

extern "C" int hp_set_samples(hp_ctx* c, int n, const int32_t* ijk) {
  if (!c || n < 0 || n > HP_MAX_SAMPLES || (n && !ijk)) {
    set_error("hp_set_samples: bad arguments");
    return HP_ERR_ARG;
  }
  for (int s = 0; s < n; ++s) {
    if (ijk[3 * s] < 0 || ijk[3 * s] >= c->I || ijk[3 * s + 1] < 0 || ijk[3 * s + 1] >= c->J ||
        ijk[3 * s + 2] < 0 || ijk[3 * s + 2] >= c->K) {
      set_error("hp_set_samples: sample %d out of range", s);
      return HP_ERR_ARG;
    }
  }
  c->samples.assign(ijk, ijk + 3 * n);
  return HP_OK;
}

// ------------------------------------------------------------- host loops
// host_loops_tuned.cpp (this library's tuned build) and host_loops_ref.cpp (the
// reference's compile template, gcc -O2); HP_FLAG_HOST_REFERENCE selects the latter.

// ----------------------------------------------------------------- runner

namespace {

struct Runner {
  hp_ctx* C;
  const hp_schedule* S;
  hp_result* R;
  std::vector<const hp_event*> before[HP_NLOOPS], after[HP_NLOOPS];
  bool busy_below[HP_NLOOPS] = {};   // device anchor or event strictly inside
  double t_start = 0, deadline = 0;
  bool guard = true;
  bool pending_h2d = false;
  // the program's literal fp32 gosa: valid while every ss*ss term since the
  // last `gosa = 0.0` was summed on the host, in program order
  float lit32 = 0.0f;
  bool lit_valid = false;
  // HP_FLAG_LITERAL_GOSA: the last iteration's device-side terms (C->terms)
  bool literal = false, terms_valid = false;
  int cur_iter = -1;               // host time loop: current iteration of loop 6
  int status = HP_OK;
  char diag[256] = {0};

  // --- helpers ---------------------------------------------------------------
  bool failed() const { return status != HP_OK; }
  void fail(int code, const char* fmt, ...) {
    if (status != HP_OK) return;
    status = code;
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(diag, sizeof diag, fmt, ap);
    va_end(ap);
  }
  bool check_time() {
    if (deadline > 0 && now_s() > deadline) {
      fail(HP_TIMEOUT, "watchdog: run exceeded %.1f s", S->timeout_s);
      return false;
    }
    return true;
  }
  bool cuda_ok(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return true;
    fail(HP_FAIL_LAUNCH, "%s: %s", what, cudaGetErrorString(e));
    return false;
  }
  int kind(int loop) const { return S->loop_kind[loop]; }
  bool on_device(int loop) const {
    const int k = kind(loop);
    return k == HP_K_KERNELS || k == HP_K_PARALLEL_LOOP || k == HP_K_PLV;
  }
  bool present(int v) const { return C->declared[v] || C->refcount[v] > 0; }
  Box full_box() const { return Box{0, C->I, 0, C->J, 0, C->K}; }
  bool is_array(int v) const { return kVars[v].nfields > 0; }
  void host_write(int v, const Box& b) {
    if (is_array(v)) C->coh[v].write(b, OWN_HOST);
    else C->host_ver[v] = ++C->clock;
    mark_host_dirty(v);
  }
  void host_write(int v) { host_write(v, full_box()); }
  void dev_write(int v, const Box& b) {
    if (is_array(v)) C->coh[v].write(b, OWN_DEV);
    else C->dev_ver[v] = ++C->clock;
  }
  void host_read(int v, const Box& b) {
    const bool stale = is_array(v) ? C->coh[v].newer_in(OWN_DEV, b) : C->host_ver[v] < C->dev_ver[v];
    if (stale) R->n_stale_reads++;
  }
  void host_read(int v) { host_read(v, full_box()); }
  void dev_read(int v, const Box& b) {
    const bool stale = is_array(v) ? C->coh[v].newer_in(OWN_HOST, b) : C->dev_ver[v] < C->host_ver[v];
    if (stale) R->n_stale_reads++;
  }
  // one field box copy in either direction (2-D fast path for the whole array)
  bool copy_box(int fid, const Box& b, cudaMemcpyKind kind) {
    cudaError_t e;
    const size_t K4 = (size_t)C->K * sizeof(float), P4 = (size_t)C->P * sizeof(float);
    if (box_contains(b, full_box())) {
      e = kind == cudaMemcpyHostToDevice ? field_to_device(C, C->dev.f[fid], C->host[fid])
                                         : field_to_host(C, C->host[fid], C->dev.f[fid]);
    } else {
      cudaMemcpy3DParms m = {};
      cudaPitchedPtr d = make_cudaPitchedPtr(C->dev.f[fid], P4, K4, (size_t)C->J);
      cudaPitchedPtr h = make_cudaPitchedPtr(C->host[fid], K4, K4, (size_t)C->J);
      m.srcPtr = kind == cudaMemcpyHostToDevice ? h : d;
      m.dstPtr = kind == cudaMemcpyHostToDevice ? d : h;
      m.srcPos = make_cudaPos((size_t)b.k0 * sizeof(float), (size_t)b.j0, (size_t)b.i0);
      m.dstPos = m.srcPos;
      m.extent = make_cudaExtent((size_t)b.nk() * sizeof(float), (size_t)b.nj(), (size_t)b.ni());
      m.kind = kind;
      e = cudaMemcpy3DAsync(&m, C->stream);
    }
    return cuda_ok(e, kind == cudaMemcpyHostToDevice ? "update device" : "update self");
  }
  void mark_host_dirty(int v) {
    const VarInfo& vi = kVars[v];
    for (int f = 0; f < vi.nfields; ++f) C->host_dirty[vi.f0 + f] = true;
  }

  // --- transfers ---------------------------------------------------------------
  void sync_pending() {
    if (pending_h2d) {
      const double t0 = now_s();
      cuda_ok(cudaStreamSynchronize(C->stream), "sync before host loop");
      R->xfer_s += now_s() - t0;
      pending_h2d = false;
    }
  }
  // Host -> device.  With the guard every point is copied except those whose
  // latest data is on the device (nothing, counted as skipped, when the host
  // copy is entirely stale -- SURVEY.md B.2); without it the whole array is.
  void h2d(int v, bool implicit) {
    if (failed()) return;
    Nvtx range(implicit ? "h2d (implicit)" : "h2d");
    const VarInfo& vi = kVars[v];
    if (vi.nfields) {
      const std::vector<Box> boxes = guard ? C->coh[v].region_excluding(OWN_DEV, full_box())
                                           : std::vector<Box>{full_box()};
      if (boxes.empty()) {
        R->n_skipped_stale++;
        return;
      }
      const double t0 = now_s();
      for (int f = 0; f < vi.nfields; ++f)
        for (const Box& b : boxes) {
          if (!copy_box(vi.f0 + f, b, cudaMemcpyHostToDevice)) return;
          R->h2d_bytes += (uint64_t)b.count() * sizeof(float);
        }
      R->n_h2d += (uint64_t)vi.nfields;
      if (implicit) R->n_implicit++;
      pending_h2d = true;
      R->xfer_s += now_s() - t0;
      if (guard) C->coh[v].mark_synced(OWN_HOST);
      else C->coh[v].all_synced(full_box());
      return;
    }
    if (guard && C->host_ver[v] < C->dev_ver[v]) {
      R->n_skipped_stale++;
      return;
    }
    const double t0 = now_s();
    {
      if (!cuda_ok(cudaMemcpyAsync(C->dscal + v * SLOT_BYTES, C->hscal + v * SLOT_BYTES,
                                   (size_t)vi.bytes, cudaMemcpyHostToDevice, C->stream),
                   "update device (scalar)"))
        return;
      R->h2d_bytes += (uint64_t)vi.bytes;
      R->n_h2d++;
    }
    if (implicit) R->n_implicit++;
    pending_h2d = true;
    R->xfer_s += now_s() - t0;
    C->dev_ver[v] = C->host_ver[v];
  }
  // Device -> host.  With the guard every point is copied back except those
  // whose latest data is on the host -- which includes device memory the
  // program never defined -- so undefined or older device data never reaches
  // the host; without it the whole array is copied, as a literal `update self`.
  void d2h(int v, bool implicit) {
    if (failed()) return;
    Nvtx range(implicit ? "d2h (implicit)" : "d2h");
    const VarInfo& vi = kVars[v];
    const double t0 = now_s();
    if (vi.nfields) {
      const std::vector<Box> boxes = guard ? C->coh[v].region_excluding(OWN_HOST, full_box())
                                           : std::vector<Box>{full_box()};
      if (boxes.empty()) {
        R->n_skipped_stale++;
        return;
      }
      for (int f = 0; f < vi.nfields; ++f)
        for (const Box& b : boxes) {
          if (!copy_box(vi.f0 + f, b, cudaMemcpyDeviceToHost)) return;
          R->d2h_bytes += (uint64_t)b.count() * sizeof(float);
        }
      R->n_d2h += (uint64_t)vi.nfields;
      mark_host_dirty(v);
    } else {
      if (guard && C->dev_ver[v] < C->host_ver[v]) {
        R->n_skipped_stale++;
        return;
      }
      if (!cuda_ok(cudaMemcpyAsync(C->hscal + v * SLOT_BYTES, C->dscal + v * SLOT_BYTES,
                                   (size_t)vi.bytes, cudaMemcpyDeviceToHost, C->stream),
                   "update self (scalar)"))
        return;
      R->d2h_bytes += (uint64_t)vi.bytes;
      R->n_d2h++;
    }
    if (implicit) R->n_implicit++;
    cuda_ok(cudaStreamSynchronize(C->stream), "update self (sync)");
    pending_h2d = false;
    R->xfer_s += now_s() - t0;
    if (vi.nfields) {
      if (guard) C->coh[v].mark_synced(OWN_DEV);
      else C->coh[v].all_synced(full_box());
    } else {
      C->host_ver[v] = C->dev_ver[v];
    }
  }

  // A structured data region (or an implicit per-kernel copy) ends: the device
  // copy is deallocated, its contents undefined from now on.
  void dealloc(int v) {
    if (is_array(v)) C->coh[v].reset(full_box());
    else C->dev_ver[v] = 0;
  }

  // --- plan events ---------------------------------------------------------------
  void fire(const hp_event* e) {
    if (failed()) return;
    const int v = e->var;
    switch (e->op) {
      case HP_EV_DECLARE:
        C->declared[v] = true;
        break;
      case HP_EV_UPDATE_DEVICE:
        h2d(v, false);
        break;
      case HP_EV_UPDATE_SELF:
        d2h(v, false);
        break;
      case HP_EV_DATA_ENTER:
        if (present(v)) {
          if (!C->declared[v]) C->refcount[v]++;
        } else {
          C->refcount[v] = 1;
          if (e->arg) h2d(v, false);
        }
        break;
      case HP_EV_DATA_EXIT:
        if (C->declared[v]) break;
        if (C->refcount[v] > 0 && --C->refcount[v] == 0) {
          if (e->arg) d2h(v, false);
          dealloc(v);
        }
        break;
      case HP_EV_PRESENT:
        if (!present(v))
          fail(HP_FAIL_PRESENT, "present(%s) failed at loop %d: data not on device",
               kVars[v].name, e->loop_id);
        break;
      default:
        fail(HP_FAIL_PATTERN, "unknown event op %d", e->op);
    }
  }
  void fire_all(const std::vector<const hp_event*>& evs) {
    for (const hp_event* e : evs) fire(e);
  }

  // --- kernel launches ---------------------------------------------------------
  LaunchArgs args(int reset) const {
    return grid_args(C->hs<int>(HP_V_IMAX), C->hs<int>(HP_V_JMAX), C->hs<int>(HP_V_KMAX),
                     C->hs<float>(HP_V_OMEGA), reset);
  }

  // implicit present_or_copy for arrays (and the gosa reduction scalar)
  void implicit_vars(int nest, std::vector<int>& out) const {
    out.clear();
    const NestVars& nv = nest_vars(nest);
    for (int v : nv.arrays)
      if (!present(v)) out.push_back(v);
    if (nv.gosa && !present(HP_V_GOSA)) out.push_back(HP_V_GOSA);
  }

  // reads/writes of one nest execution over box b (stencil reads p with a halo of 1)
  void note_device_access(int nest, const Box& b) {
    const NestVars& nv = nest_vars(nest);
    for (int v : nv.arrays) {
      const bool w = std::find(nv.writes.begin(), nv.writes.end(), v) != nv.writes.end();
      const bool r = !(nest == NEST_INIT0 || nest == NEST_INIT1) &&
                     !(nest == NEST_STENCIL && v == HP_V_WRK2) && !(nest == NEST_COPY && v == HP_V_P);
      if (r) dev_read(v, (nest == NEST_STENCIL && v == HP_V_P) ? grow(b, 1) : b);
      if (w) dev_write(v, b);
    }
    if (nv.gosa) {
      dev_read(HP_V_GOSA, b);
      dev_write(HP_V_GOSA, b);
    }
  }

  void launch(int nest, Mapping map, const Box& b, bool full_tuned) {
    if (failed()) return;
    std::vector<int> imp;
    implicit_vars(nest, imp);
    for (int v : imp) h2d(v, true);
    if (failed()) return;
    note_device_access(nest, b);
    int n = 0;
    if (nest == NEST_STENCIL) {
      lit_valid = false;   // terms summed on the device
      if (literal && cur_iter == C->hs<int>(HP_V_NN) - 1) {
        if (launch_stencil_terms(C->dev, C->dev.f[HP_F_P], C->terms, b, C->stream) < 0) {
          fail(HP_FAIL_LAUNCH, "terms kernel: %s", cudaGetErrorString(cudaGetLastError()));
          return;
        }
        terms_valid = true;
      }
    }
    const LaunchArgs a = args(0);
    if (full_tuned && map == MAP_COLLAPSE && nest == NEST_STENCIL)
      n = launch_stencil_3d(C->dev, a, C->sink(), C->stream);
    else if (full_tuned && map == MAP_COLLAPSE && nest == NEST_COPY)
      n = launch_copy_3d(C->dev, a, C->stream);
    else
      n = launch_nest((Nest)nest, map, C->dev, b, a, C->sink(), C->stream);
    if (n < 0) {
      cudaError_t e = cudaGetLastError();
      fail(HP_FAIL_LAUNCH, "launch of nest %d failed: %s", nest, cudaGetErrorString(e));
      return;
    }
    R->n_launch += (uint64_t)n;
    C->launches += (uint64_t)n;
    for (int v : imp) {
      d2h(v, true);
      dealloc(v);
    }
  }

  // --- nests ---------------------------------------------------------------------
  Box nest_box(int nest) const {
    const int imax = C->hs<int>(HP_V_IMAX), jmax = C->hs<int>(HP_V_JMAX),
              kmax = C->hs<int>(HP_V_KMAX);
    switch (nest) {
      case NEST_INIT0: return Box{0, C->I, 0, C->J, 0, C->K};
      case NEST_INIT1: return Box{0, imax, 0, jmax, 0, kmax};
      default: return Box{1, imax - 1, 1, jmax - 1, 1, kmax - 1};
    }
  }

  void host_nest(int nest, const Box& b) {
    if (failed()) return;
    sync_pending();
    const double t0 = now_s();
    const HostFields H = C->hostf();
    const NestVars& nv = nest_vars(nest);
    if (nest == NEST_STENCIL || nest == NEST_COPY)
      for (int v : nv.arrays)
        if (!(nest == NEST_STENCIL && v == HP_V_WRK2) && !(nest == NEST_COPY && v == HP_V_P))
          host_read(v, (nest == NEST_STENCIL && v == HP_V_P) ? grow(b, 1) : b);
    const bool ref = (S->flags & HP_FLAG_HOST_REFERENCE) != 0;
    switch (nest) {
      case NEST_INIT0: ref ? host_ref::init0(H, b) : host_tuned::init0(H, b); break;
      case NEST_INIT1: {
        const int imax = C->hs<int>(HP_V_IMAX);
        ref ? host_ref::init1(H, b, imax) : host_tuned::init1(H, b, imax);
        break;
      }
      case NEST_STENCIL: {
        host_read(HP_V_GOSA);
        const float omega = C->hs<float>(HP_V_OMEGA);
        C->hs<double>(HP_V_GOSA) += ref ? host_ref::stencil(H, b, omega, &lit32)
                                        : host_tuned::stencil(H, b, omega, &lit32);
        host_write(HP_V_GOSA);
        break;
      }
      default: ref ? host_ref::copy(H, b) : host_tuned::copy(H, b); break;
    }
    for (int v : nv.writes) host_write(v, b);
    R->host_s += now_s() - t0;
  }

  Mapping mapping(int loop) const {
    switch (kind(loop)) {
      case HP_K_PARALLEL_LOOP: return MAP_GANG;
      case HP_K_PLV: return MAP_VECTOR;
      default: return MAP_COLLAPSE;
    }
  }

  // Execute loop `level` of `nest` with outer indices fixed in `b`.
  void run_level(int nest, int level, Box b) {
    if (failed()) return;
    const int loop = kNestLoops[nest][level];
    fire_all(before[loop]);
    if (on_device(loop)) {
      Nvtx range(loop_range_name(loop, true));
      launch(nest, mapping(loop), b, level == 0);
    } else if (level < 2 && busy_below[loop]) {
      const int lo = level == 0 ? b.i0 : b.j0, hi = level == 0 ? b.i1 : b.j1;
      for (int x = lo; x < hi && !failed(); ++x) {
        Box inner = b;
        if (level == 0) { inner.i0 = x; inner.i1 = x + 1; }
        else { inner.j0 = x; inner.j1 = x + 1; }
        run_level(nest, level + 1, inner);
        if (level == 0) check_time();
      }
    } else {
      Nvtx range(loop_range_name(loop, false));
      host_nest(nest, b);
      check_time();
    }
    fire_all(after[loop]);
  }

  void run_nest(int nest) { run_level(nest, 0, nest_box(nest)); }

  // device-resident time loop (gene 6 = 1)
  void device_time_loop() {
    if (failed()) return;
    Nvtx range(loop_range_name(6, true));
    // implicit copies for everything the loop body touches
    std::vector<int> imp, tmp;
    implicit_vars(NEST_STENCIL, tmp);
    imp = tmp;
    implicit_vars(NEST_COPY, tmp);
    for (int v : tmp)
      if (std::find(imp.begin(), imp.end(), v) == imp.end()) imp.push_back(v);
    if (!present(HP_V_GOSA) && std::find(imp.begin(), imp.end(), HP_V_GOSA) == imp.end())
      imp.push_back(HP_V_GOSA);
    for (int v : imp) h2d(v, true);
    if (failed()) return;
    const int nn = C->hs<int>(HP_V_NN);
    const int k6 = kind(6);
    if (nn > 0) lit_valid = false;
    const bool fused = (S->flags & HP_FLAG_FUSED_TIME_LOOP) && k6 != HP_K_PLV;
    const Box interior = nest_box(NEST_STENCIL);
    if (nn > 0) note_device_access(NEST_STENCIL, interior);
    int n = 0;
    if (nn > 0) {
      float* terms = literal ? C->terms : nullptr;
      if (fused) {
        n = time_loop_fused(C, nn, args(1), terms, interior);
      } else {
        const Box bs = nest_box(NEST_STENCIL);
        for (int it = 0; it < nn && n >= 0; ++it) {
          const LaunchArgs a = args(1);
          int r1, r2;
          if (terms && it == nn - 1) {
            if (launch_stencil_terms(C->dev, C->dev.f[HP_F_P], terms, bs, C->stream) < 0) {
              n = -1;
              break;
            }
            n += 1;
          }
          if (k6 == HP_K_PLV) {
            r1 = launch_nest(NEST_STENCIL, MAP_VECTOR, C->dev, bs, a, C->sink(), C->stream);
            r2 = launch_nest(NEST_COPY, MAP_VECTOR, C->dev, bs, a, C->sink(), C->stream);
          } else {
            r1 = launch_stencil_3d(C->dev, a, C->sink(), C->stream);
            r2 = launch_copy_3d(C->dev, a, C->stream);
          }
          n = (r1 < 0 || r2 < 0) ? -1 : n + r1 + r2;
        }
      }
    }
    if (n < 0) {
      fail(HP_FAIL_LAUNCH, "time-loop launch failed: %s", cudaGetErrorString(cudaGetLastError()));
      return;
    }
    if (literal && nn > 0) terms_valid = true;
    R->n_launch += (uint64_t)n;
    C->launches += (uint64_t)n;
    if (nn > 0) {
      dev_write(HP_V_WRK2, interior);
      dev_write(HP_V_P, interior);
      dev_write(HP_V_GOSA, interior);
    }
    for (int v : imp) {
      d2h(v, true);
      dealloc(v);
    }
  }

 public:
  // the fused device time loop: one- and two-step passes (temporal blocking)
  // With `terms` (verification mode) the passes stop before the last iteration,
  // whose ss*ss terms are written out from the rotation buffer holding p_{nn-1}.
  static int time_loop_fused(hp_ctx* c, int nn, const LaunchArgs& a, float* terms = nullptr,
                             const Box& interior = Box{}) {
    int n = 0, r;
    if ((r = time_loop_begin(c, a)) < 0) return -1;
    n += r;
    float* last = nullptr;
    if (!terms) {
      if ((r = stencil_iterations(c->dev, c->dev.f[HP_F_P], c->scratch, nn, a, c->sink(),
                                  c->stream, &last, nullptr)) < 0)
        return -1;
      n += r;
    } else {
      float* mid = nullptr;
      if ((r = stencil_iterations(c->dev, c->dev.f[HP_F_P], c->scratch, nn - 1, a, c->sink(),
                                  c->stream, &mid, nullptr)) < 0)
        return -1;
      n += r;
      if ((r = launch_stencil_terms(c->dev, mid, terms, interior, c->stream)) < 0) return -1;
      n += r;
      float* other = mid == c->dev.f[HP_F_P] ? c->scratch : c->dev.f[HP_F_P];
      if ((r = stencil_iterations(c->dev, mid, other, 1, a, c->sink(), c->stream, &last,
                                  nullptr)) < 0)
        return -1;
      n += r;
    }
    if ((r = time_loop_finish(c, last, a)) < 0) return -1;
    return n + r;
  }

  void run_time_loop() {
    fire_all(before[6]);
    if (on_device(6)) {
      device_time_loop();
    } else {
      const int nn = C->hs<int>(HP_V_NN);
      for (int it = 0; it < nn && !failed(); ++it) {
        cur_iter = it;
        C->hs<double>(HP_V_GOSA) = 0.0;  // gosa = 0.0;  (host statement in loop 6)
        host_write(HP_V_GOSA);
        lit32 = 0.0f;
        lit_valid = true;
        terms_valid = false;
        run_nest(NEST_STENCIL);
        run_nest(NEST_COPY);
        check_time();
      }
    }
    fire_all(after[6]);
  }

  // --- setup -------------------------------------------------------------------
  int prepare() {
    if (S->n_loops != HP_NLOOPS) {
      set_error("schedule has %d loops, program has %d", S->n_loops, HP_NLOOPS);
      return HP_ERR_ARG;
    }
    if (S->n_events < 0 || (S->n_events > 0 && !S->events)) {
      set_error("schedule events missing");
      return HP_ERR_ARG;
    }
    for (int l = 0; l < HP_NLOOPS; ++l)
      if (S->loop_kind[l] < HP_K_HOST || S->loop_kind[l] > HP_K_COVERED) {
        set_error("loop %d: bad kind %d", l, S->loop_kind[l]);
        return HP_ERR_ARG;
      }
    // nested compute constructs: reject (reference: compile failure -> penalty)
    for (int l = 0; l < HP_NLOOPS; ++l) {
      if (!on_device(l)) continue;
      for (int a = kParentOf[l]; a >= 0; a = kParentOf[a])
        if (on_device(a)) {
          fail(HP_FAIL_PATTERN, "nested compute construct: loop %d inside device loop %d", l, a);
          return HP_OK;
        }
    }
    for (int n = 0; n < S->n_events; ++n) {
      const hp_event* e = &S->events[n];
      if (e->var < 0 || e->var >= HP_NVARS) {
        set_error("event %d: bad var %d", n, e->var);
        return HP_ERR_ARG;
      }
      if (e->op == HP_EV_DECLARE) continue;
      if (e->loop_id < 0 || e->loop_id >= HP_NLOOPS) {
        set_error("event %d: bad loop %d", n, e->loop_id);
        return HP_ERR_ARG;
      }
      (e->when == HP_BEFORE ? before : after)[e->loop_id].push_back(e);
      for (int a = kParentOf[e->loop_id]; a >= 0; a = kParentOf[a]) busy_below[a] = true;
    }
    for (int l = 0; l < HP_NLOOPS; ++l)
      if (on_device(l))
        for (int a = kParentOf[l]; a >= 0; a = kParentOf[a]) busy_below[a] = true;
    // emitter stacking order: update device (10) < data (20) < present (30);
    // after a statement: data exit / brace (60) < update self (90)
    auto rank = [](const hp_event* e) {
      switch (e->op) {
        case HP_EV_UPDATE_DEVICE: return 10;
        case HP_EV_DATA_ENTER: return 20;
        case HP_EV_PRESENT: return 30;
        case HP_EV_DATA_EXIT: return 60;
        default: return 90;
      }
    };
    for (int l = 0; l < HP_NLOOPS; ++l) {
      std::stable_sort(before[l].begin(), before[l].end(),
                       [&](const hp_event* x, const hp_event* y) { return rank(x) < rank(y); });
      std::stable_sort(after[l].begin(), after[l].end(),
                       [&](const hp_event* x, const hp_event* y) { return rank(x) < rank(y); });
    }
    return HP_OK;
  }

  // Verification mode, after the timed run: the device-side terms of the last
  // iteration summed as the program does (`gosa += ss*ss`, float, i/j/k order).
  void finish_literal() {
    if (failed() || !literal || lit_valid || !terms_valid) return;
    const Box b = nest_box(NEST_STENCIL);
    std::vector<float> t((size_t)C->I * C->J * C->K);
    if (!cuda_ok(cudaMemcpyAsync(t.data(), C->terms, t.size() * sizeof(float),
                                 cudaMemcpyDeviceToHost, C->stream), "terms D2H") ||
        !cuda_ok(cudaStreamSynchronize(C->stream), "terms sync"))
      return;
    const HostFields H = C->hostf();
    float g = 0.0f;
    for (int i = b.i0; i < b.i1; ++i)
      for (int j = b.j0; j < b.j1; ++j) {
        const float* row = t.data() + H.at(i, j, 0);
        for (int k = b.k0; k < b.k1; ++k) g += row[k];
      }
    R->gosa_f32 = g;
    R->gosa_f32_literal = 1;
  }

  void reset_state() {
    C->clock = 1;
    for (int v = 0; v < HP_NVARS; ++v) {
      C->host_ver[v] = 1;   // static storage / declarations: host copy is defined
      C->dev_ver[v] = 0;    // fresh device memory: undefined
      C->declared[v] = false;
      C->refcount[v] = 0;
      C->coh[v].reset(Box{0, C->I, 0, C->J, 0, C->K});
    }
    memset(C->hscal, 0, HP_NVARS * SLOT_BYTES);
  }

  void program() {
    // main: imax = I-1; jmax = J-1; kmax = K-1; omega = 0.8;
    C->hs<int>(HP_V_IMAX) = C->I - 1; host_write(HP_V_IMAX);
    C->hs<int>(HP_V_JMAX) = C->J - 1; host_write(HP_V_JMAX);
    C->hs<int>(HP_V_KMAX) = C->K - 1; host_write(HP_V_KMAX);
    C->hs<float>(HP_V_OMEGA) = 0.8f; host_write(HP_V_OMEGA);
    for (int n = 0; n < S->n_events; ++n)
      if (S->events[n].op == HP_EV_DECLARE) fire(&S->events[n]);
    // initmt()
    run_nest(NEST_INIT0);
    run_nest(NEST_INIT1);
    // gosa = jacobi(nn)
    C->hs<int>(HP_V_NN) = S->nn; host_write(HP_V_NN);
    run_time_loop();
    sync_pending();
    if (!failed()) cuda_ok(cudaStreamSynchronize(C->stream), "program end");
    // main:gosa = jacobi's return value (host copy); printed with the p samples
    host_read(HP_V_GOSA);
    R->gosa = C->hs<double>(HP_V_GOSA);
    R->gosa_f32_literal = lit_valid ? 1 : 0;
    R->gosa_f32 = lit_valid ? lit32 : (float)R->gosa;
    host_read(HP_V_P);
    const int ns = (int)C->samples.size() / 3;
    R->n_samples = ns;
    for (int s = 0; s < ns; ++s)
      R->samples[s] = C->host[HP_F_P][C->hostf().at(C->samples[3 * s], C->samples[3 * s + 1],
                                                   C->samples[3 * s + 2])];
  }
};

}  // namespace

extern "C" int hp_run(hp_ctx* c, const hp_schedule* s, hp_result* r) {
  if (!c || !s || !r) {
    set_error("hp_run: null argument");
    return HP_ERR_ARG;
  }
  memset(r, 0, sizeof *r);
  cudaError_t e = cudaSetDevice(c->device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  Runner run;
  run.C = c;
  run.S = s;
  run.R = r;
  run.guard = (s->flags & HP_FLAG_COHERENCE_GUARD) != 0;
  run.literal = (s->flags & HP_FLAG_LITERAL_GOSA) != 0;
  int rc = run.prepare();
  if (rc != HP_OK) return rc;
  if (run.failed()) {  // rejected pattern: nothing executes
    r->status = run.status;
    memcpy(r->diag, run.diag, sizeof r->diag);
    set_error("%s", run.diag);
    return run.status;
  }
  // fresh process: static arrays zero, device memory undefined (not timed)
  if (s->flags & HP_FLAG_FRESH_PROCESS) {
    // zero the dirty host arrays, one thread per array (up to 8 at a time): the
    // reset sits between two fitness runs of a GA worker slot, so it is kept short
    const size_t bytes = (size_t)c->I * c->J * c->K * sizeof(float);
    std::vector<int> dirty;
    for (int f = 0; f < HP_NFIELDS; ++f)
      if (c->host_dirty[f]) dirty.push_back(f);
    const size_t nt = std::min<size_t>(8, dirty.size());
    std::vector<std::thread> pool;
    for (size_t t = 1; t < nt; ++t)
      pool.emplace_back([&, t] {
        for (size_t x = t; x < dirty.size(); x += nt) memset(c->host[dirty[x]], 0, bytes);
      });
    for (size_t x = 0; nt && x < dirty.size(); x += nt) memset(c->host[dirty[x]], 0, bytes);
    for (std::thread& th : pool) th.join();
    for (int f : dirty) c->host_dirty[f] = false;
  }
  if (s->flags & HP_FLAG_POISON_DEVICE) {
    if (launch_fill(c->slab, c->field_stride * (HP_NFIELDS + 1), nanf(""), c->stream) < 0)
      return cuda_fail(cudaGetLastError(), "poison");
  }
  if (run.literal && !c->terms) {
    e = cudaMalloc(&c->terms, (size_t)c->I * c->J * c->K * sizeof(float));
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(terms)");
  }
  cudaMemsetAsync(c->dscal, 0xff, HP_NVARS * SLOT_BYTES, c->stream);
  e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return cuda_fail(e, "pre-run sync");
  run.reset_state();

  run.t_start = now_s();
  run.deadline = s->timeout_s > 0 ? run.t_start + s->timeout_s : 0;
  {
    Nvtx range("hp_run program");
    run.program();
  }
  if (run.status == HP_TIMEOUT || run.status == HP_FAIL_LAUNCH) cudaStreamSynchronize(c->stream);
  r->wall_s = now_s() - run.t_start;
  run.finish_literal();   // verification mode only; not part of the timed run
  // a sticky device error (illegal address, ...) poisons the context
  e = cudaGetLastError();
  if (e != cudaSuccess && run.status == HP_OK)
    run.fail(HP_FAIL_LAUNCH, "device error: %s", cudaGetErrorString(e));
  r->status = run.status;
  memcpy(r->diag, run.diag, sizeof r->diag);
  if (run.status != HP_OK) set_error("%s", run.diag);
  return run.status;
}

// --------------------------------------------------------- field access

extern "C" int hp_read_field(hp_ctx* c, int field, int side, float* dst, size_t n) {
  if (!c || !dst || field < 0 || field >= HP_NFIELDS || n != (size_t)c->I * c->J * c->K) {
    set_error("hp_read_field: bad arguments");
    return HP_ERR_ARG;
  }
  CK(cudaSetDevice(c->device), "cudaSetDevice");
  if (side == 0) {
    memcpy(dst, c->host[field], n * sizeof(float));
    return HP_OK;
  }
  CK(field_to_host(c, dst, c->dev.f[field]), "read field");
  CK(cudaStreamSynchronize(c->stream), "read field sync");
  return HP_OK;
}

extern "C" int hp_write_field(hp_ctx* c, int field, int side, const float* src, size_t n) {
  if (!c || !src || field < 0 || field >= HP_NFIELDS || n != (size_t)c->I * c->J * c->K) {
    set_error("hp_write_field: bad arguments");
    return HP_ERR_ARG;
  }
  CK(cudaSetDevice(c->device), "cudaSetDevice");
  if (side == 0) {
    memcpy(c->host[field], src, n * sizeof(float));
    c->host_dirty[field] = true;
    return HP_OK;
  }
  CK(field_to_device(c, c->dev.f[field], src), "write field");
  CK(cudaStreamSynchronize(c->stream), "write field sync");
  return HP_OK;
}

extern "C" int hp_read_gosa(hp_ctx* c, int side, double* out) {
  if (!c || !out) {
    set_error("hp_read_gosa: bad arguments");
    return HP_ERR_ARG;
  }
  CK(cudaSetDevice(c->device), "cudaSetDevice");
  if (side == 0) {
    *out = c->hs<double>(HP_V_GOSA);
    return HP_OK;
  }
  CK(cudaMemcpyAsync(out, c->dscal + HP_V_GOSA * SLOT_BYTES, sizeof(double),
                     cudaMemcpyDeviceToHost, c->stream),
     "read gosa");
  CK(cudaStreamSynchronize(c->stream), "read gosa sync");
  return HP_OK;
}

// ------------------------------------------------- device-resident Jacobi

static LaunchArgs default_args(const hp_ctx* c, int reset) { return ctx_args(c, reset); }


extern "C" int hp_init_device(hp_ctx* c) {
  if (!c) return HP_ERR_ARG;
  CK(cudaSetDevice(c->device), "cudaSetDevice");
  const LaunchArgs a = default_args(c, 0);
  GosaSink g = c->sink();
  Box b0{0, c->I, 0, c->J, 0, c->K};
  // initmt nest B over global i < imax: local planes [0, imax - i_off)
  Box b1{std::max(0, -c->i_off), std::min(c->I, a.imax - c->i_off), 0, a.jmax, 0, a.kmax};
  if (launch_fill(c->dev.f[HP_F_WRK2], c->field_elems, 0.0f, c->stream) < 0 ||
      launch_nest(NEST_INIT0, MAP_COLLAPSE, c->dev, b0, a, g, c->stream) < 0 ||
      launch_nest(NEST_INIT1, MAP_COLLAPSE, c->dev, b1, a, g, c->stream) < 0)
    return cuda_fail(cudaGetLastError(), "init launch");
  CK(cudaStreamSynchronize(c->stream), "init sync");
  return HP_OK;
}

extern "C" int hp_jacobi_device(hp_ctx* c, int nn, int variant) {
  if (!c || nn < 0 || (variant != 0 && variant != 1)) {
    set_error("hp_jacobi_device: bad arguments");
    return HP_ERR_ARG;
  }
  CK(cudaSetDevice(c->device), "cudaSetDevice");
  const LaunchArgs a = default_args(c, 1);
  if (variant == 1) {
    if (nn > 0) {
      const int n = Runner::time_loop_fused(c, nn, a);
      if (n < 0) return cuda_fail(cudaGetLastError(), "fused time loop");
      c->launches += (uint64_t)n;
    }
    return HP_OK;
  }
  for (int it = 0; it < nn; ++it) {
    const int r1 = launch_stencil_3d(c->dev, a, c->sink(), c->stream);
    const int r2 = r1 < 0 ? -1 : launch_copy_3d(c->dev, a, c->stream);
    if (r1 < 0 || r2 < 0) return cuda_fail(cudaGetLastError(), "time loop");
    c->launches += (uint64_t)(r1 + r2);
  }
  return HP_OK;
}

extern "C" uint64_t hp_launch_count(hp_ctx* c) { return c ? c->launches : 0; }

extern "C" int hp_set_temporal_blocking(int on) { return set_temporal_blocking(on); }

extern "C" int hp_tx_status(hp_ctx* c) {
  if (!c) return HP_ERR_ARG;
  CK(cudaSetDevice(c->device), "cudaSetDevice");
  const int r = tx_error(c->dev.tma);
  return r < 0 ? cuda_fail(cudaGetLastError(), "hp_tx_status") : r;
}

extern "C" int hp_set_stencil_config(int cfg) {
  const int n = set_stencil_config(cfg);
  if (n < 0) {
    set_error("hp_set_stencil_config: no configuration %d", cfg);
    return HP_ERR_ARG;
  }
  return n;
}

extern "C" int hp_time_steps(hp_ctx* c, int steps, int nn, int variant, double* ms_out) {
  if (!c || !ms_out || steps < 0) {
    set_error("hp_time_steps: bad arguments");
    return HP_ERR_ARG;
  }
  CK(cudaSetDevice(c->device), "cudaSetDevice");
  CK(cudaEventRecord(c->ev0, c->stream), "event record");
  for (int s = 0; s < steps; ++s) {
    const int rc = hp_jacobi_device(c, nn, variant);
    if (rc != HP_OK) return rc;
  }
  CK(cudaEventRecord(c->ev1, c->stream), "event record");
  CK(cudaEventSynchronize(c->ev1), "event sync");
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, c->ev0, c->ev1), "event elapsed");
  *ms_out = ms;
  return HP_OK;
}

extern "C" int hp_time_jacobi(hp_ctx* c, int nn, int variant, hp_kernel_times* out) {
  if (!c || !out || nn < 1 || (variant != 0 && variant != 1)) {
    set_error("hp_time_jacobi: bad arguments");
    return HP_ERR_ARG;
  }
  CK(cudaSetDevice(c->device), "cudaSetDevice");
  memset(out, 0, sizeof *out);
  const LaunchArgs a = default_args(c, 1);
  // one event before every launch and one after the last: launch k spans [k, k+1]
  std::vector<cudaEvent_t> ev;
  std::vector<int> is_stencil;
  auto mark = [&]() -> bool {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return false;
    ev.push_back(e);
    return cudaEventRecord(e, c->stream) == cudaSuccess;
  };
  bool ok = mark();
  float* bufs[2] = {c->dev.f[HP_F_P], c->scratch};
  if (variant == 1) {
    ok = ok && launch_copy_halo(c->dev, bufs[0], bufs[1], a, c->stream) >= 0;
    is_stencil.push_back(0);
    ok = ok && mark();
    float* cur = bufs[0];
    float* oth = bufs[1];
    int it = 0;
    while (ok && it < nn) {
      // one pass at a time (same choice as stencil_iterations), an event after each
      float* last = nullptr;
      int passes = 0;
      // one launch as stencil_iterations would make it: every remaining pair of
      // iterations in one flow launch where that applies, else two iterations per
      // pass when temporal blocking is on (otherwise each single step alone)
      const bool tb = set_temporal_blocking(-1) != 0;
      int step = (nn - it >= 2 && tb) ? 2 : 1;
      if (tb && nn - it >= 4 && stencil_flow_ok(c->dev, a, device_sm_count())) step = (nn - it) / 2 * 2;
      ok = stencil_iterations(c->dev, cur, oth, step, a, c->sink(), c->stream, &last, &passes) >= 0;
      ok = ok && mark();   // (a 2-step request may have run as two single passes)
      is_stencil.push_back(1);
      out->stencil_iters += step;
      it += step;
      cur = last;
      oth = last == bufs[0] ? bufs[1] : bufs[0];
    }
    float* last = cur;
    ok = ok && launch_copy_interior_bounds(c->dev, last, c->dev.f[HP_F_WRK2], a, c->stream) >= 0 && mark();
    is_stencil.push_back(0);
    if (ok && last != c->dev.f[HP_F_P]) {
      ok = launch_copy_interior_bounds(c->dev, last, c->dev.f[HP_F_P], a,
                                       c->stream) >= 0 && mark();
      is_stencil.push_back(0);
    }
  } else {
    for (int it = 0; ok && it < nn; ++it) {
      ok = launch_stencil_3d(c->dev, a, c->sink(), c->stream) >= 0 && mark();
      is_stencil.push_back(1);
      out->stencil_iters += 1;
      ok = ok && launch_copy_3d(c->dev, a, c->stream) >= 0 && mark();
      is_stencil.push_back(0);
    }
  }
  int rc = HP_OK;
  if (!ok || cudaStreamSynchronize(c->stream) != cudaSuccess) {
    rc = cuda_fail(cudaGetLastError(), "hp_time_jacobi");
  } else {
    c->launches += is_stencil.size();
    double st = 0, ot = 0;
    for (size_t k = 0; k + 1 < ev.size(); ++k) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[k], ev[k + 1]);
      if (is_stencil[k]) { st += ms; out->n_stencil++; }
      else { ot += ms; out->n_other++; }
    }
    float total = 0.f;
    cudaEventElapsedTime(&total, ev.front(), ev.back());
    out->total_ms = total;
    out->stencil_ms = out->n_stencil ? st / out->n_stencil : 0.0;
    out->stencil_iters = out->n_stencil ? out->stencil_iters / out->n_stencil : 0.0;
    out->other_ms = out->n_other ? ot / out->n_other : 0.0;
  }
  for (cudaEvent_t e : ev) cudaEventDestroy(e);
  return rc;
}

// Host-input uploads of all contexts on one device are ordered through a
// per-device token: each upload waits for the previous one (cudaStreamWaitEvent)
// and publishes its own completion event.  PCIe is the shared resource, so
// serialising uploads loses nothing, and it staggers concurrent jobs: the next
// job's upload overlaps the current job's device loop instead of splitting the
// link with it and then competing for the SMs at the same time.
namespace {
std::mutex g_upload_mu;
cudaEvent_t g_last_upload[64] = {};
}  // namespace

static void forget_upload(hp_ctx* c) {
  std::lock_guard<std::mutex> lock(g_upload_mu);
  if (c->device >= 0 && c->device < 64 && g_last_upload[c->device] == c->h2d_done)
    g_last_upload[c->device] = nullptr;
}

// Enqueue H2D of the inputs (through the staging buffer, repitched on device),
// the device loop, D2H of p and of gosa into the pinned scalar slot; no host sync.
static int jacobi_host_enqueue(hp_ctx* c, const float* const* fields, int nn, int variant,
                               float* p_out, const char* who) {
  if (!c || !fields || !p_out) {
    set_error("%s: null argument", who);
    return HP_ERR_ARG;
  }
  CK(cudaSetDevice(c->device), "cudaSetDevice");
  for (int f = 0; f < HP_NFIELDS; ++f) {
    if (f != HP_F_WRK2 && !fields[f]) {
      set_error("%s: field %d missing", who, f);
      return HP_ERR_ARG;
    }
  }
  if (!c->h2d_done)
    CK(cudaEventCreateWithFlags(&c->h2d_done, cudaEventDisableTiming), "cudaEventCreate");
  if (!c->up) {
    // copy stream, events and the second staging buffer of the double-buffered upload
    CK(cudaStreamCreateWithFlags(&c->up, cudaStreamNonBlocking), "cudaStreamCreate");
    for (cudaEvent_t* e : {&c->up_start, &c->up_ev[0], &c->up_ev[1], &c->rep_ev[0], &c->rep_ev[1]})
      CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "cudaEventCreate");
    CK(cudaMalloc(&c->stage2, (size_t)c->I * c->J * c->K * sizeof(float)), "cudaMalloc stage");
  }
  {
    // H2D of field i into staging buffer i % 2 on the copy stream, repitch into the
    // field on the compute stream: the link moves field i+1 while field i is repitched
    // (one buffer: the link idled ~0.1 ms per field on L)
    std::lock_guard<std::mutex> lock(g_upload_mu);
    const bool tok = c->device >= 0 && c->device < 64;
    CK(cudaEventRecord(c->up_start, c->stream), "upload start");   // staging buffers free
    CK(cudaStreamWaitEvent(c->up, c->up_start, 0), "upload start");
    if (tok && g_last_upload[c->device])
      CK(cudaStreamWaitEvent(c->up, g_last_upload[c->device], 0), "upload order");
    float* stage[2] = {c->scratch, c->stage2};
    const size_t n = (size_t)c->I * c->J * c->K;
    int i = 0;
    for (int f = 0; f < HP_NFIELDS; ++f) {
      if (f == HP_F_WRK2) continue;
      const int b = i & 1;
      if (i >= 2) CK(cudaStreamWaitEvent(c->up, c->rep_ev[b], 0), "stage reuse");
      CK(cudaMemcpyAsync(stage[b], fields[f], n * sizeof(float), cudaMemcpyHostToDevice, c->up),
         "jacobi H2D");
      CK(cudaEventRecord(c->up_ev[b], c->up), "H2D event");
      CK(cudaStreamWaitEvent(c->stream, c->up_ev[b], 0), "H2D wait");
      if (launch_repitch(c->dev.f[f], (size_t)c->P, stage[b], (size_t)c->K, c->K,
                         (size_t)c->I * c->J, c->stream) < 0)
        CK(cudaGetLastError(), "repitch");
      CK(cudaEventRecord(c->rep_ev[b], c->stream), "repitch event");
      ++i;
    }
    CK(cudaEventRecord(c->h2d_done, c->up), "upload event");
    if (tok) g_last_upload[c->device] = c->h2d_done;
  }
  int rc = hp_jacobi_device(c, nn, variant);
  if (rc != HP_OK) return rc;
  CK(field_to_host(c, p_out, c->dev.f[HP_F_P]), "jacobi D2H p");
  CK(cudaMemcpyAsync(&c->hs<double>(HP_V_GOSA), c->dscal + HP_V_GOSA * SLOT_BYTES,
                     sizeof(double), cudaMemcpyDeviceToHost, c->stream),
     "jacobi D2H gosa");
  return HP_OK;
}

extern "C" int hp_jacobi_host(hp_ctx* c, const float* const* fields, int nn, int variant,
                              float* p_out, double* gosa_out) {
  if (!gosa_out) {
    set_error("hp_jacobi_host: null argument");
    return HP_ERR_ARG;
  }
  const int rc = jacobi_host_enqueue(c, fields, nn, variant, p_out, "hp_jacobi_host");
  if (rc != HP_OK) return rc;
  CK(cudaStreamSynchronize(c->stream), "jacobi sync");
  *gosa_out = c->hs<double>(HP_V_GOSA);
  return HP_OK;
}

extern "C" int hp_jacobi_host_async(hp_ctx* c, const float* const* fields, int nn, int variant,
                                    float* p_out, double* gosa_out) {
  if (!gosa_out) {
    set_error("hp_jacobi_host_async: null argument");
    return HP_ERR_ARG;
  }
  if (c && c->pending_gosa) {
    set_error("hp_jacobi_host_async: previous call not completed by hp_sync");
    return HP_ERR_ARG;
  }
  const int rc = jacobi_host_enqueue(c, fields, nn, variant, p_out, "hp_jacobi_host_async");
  if (rc != HP_OK) return rc;
  c->pending_gosa = gosa_out;
  return HP_OK;
}

extern "C" int hp_sync(hp_ctx* c) {
  if (!c) {
    set_error("hp_sync: null context");
    return HP_ERR_ARG;
  }
  CK(cudaSetDevice(c->device), "cudaSetDevice");
  CK(cudaStreamSynchronize(c->stream), "hp_sync");
  if (c->pending_gosa) {
    *c->pending_gosa = c->hs<double>(HP_V_GOSA);
    c->pending_gosa = nullptr;
  }
  return HP_OK;
}

extern "C" void* hp_host_alloc(size_t bytes) {
  void* p = nullptr;
  if (cudaHostAlloc(&p, bytes, cudaHostAllocPortable) != cudaSuccess) {
    cudaGetLastError();
    set_error("cudaHostAlloc(%zu) failed", bytes);
    return nullptr;
  }
  return p;
}

extern "C" void hp_host_free(void* p) {
  if (p) cudaFreeHost(p);
}
