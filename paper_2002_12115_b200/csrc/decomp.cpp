// Slab decomposition of the device-resident Jacobi over several GPUs.
//
// The interior planes [1, I-2) of the slowest dimension (C `i`) are split into
// contiguous slabs (>= 2 planes), one per rank.  A slab context holds global
// planes [i_begin-2, i_end+2): its interior plus two halo planes on each side
// (global boundary planes at the ends of the grid).  Each pass runs one or two
// Jacobi iterations on the slab -- the two-step kernel's first step also
// recomputes the neighbours' adjacent planes from the two-deep halo -- and then
// exchanges two planes per side: its first two interior planes go to rank-1's
// upper halo, its last two to rank+1's lower halo.  After the last pass the
// per-rank gosa partials (fp64) are summed.  Only the final iteration's gosa is
// observable (jacobi returns it), so one reduction per jacobi call suffices.
//
// Transports:
//  * in-process group (hp_group_jacobi): several slab contexts driven by one
//    host thread; halo planes move by cudaMemcpyPeerAsync on the receiver's
//    stream after a cross-stream event on the sender's stencil.  Used for one
//    process driving several GPUs, and to test the decomposition with virtual
//    ranks on a single GPU.
//  * NCCL (hp_dd_*): one process per GPU; ncclSend/ncclRecv of the halo planes
//    and one ncclAllReduce of gosa, on the context's stream.  libnccl.so.2 is
//    dlopen'ed on first use (the library has no link-time NCCL dependency; an
//    NCCL already loaded by torch is reused).
#include <cuda.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <vector>

#include "context.h"

using namespace hp;

// ---------------------------------------------------------------- geometry

constexpr int kHalo = 2;   // halo planes per side (two-step passes need two)

extern "C" int hp_slab_range(int I, int nranks, int rank, int32_t* i_begin, int32_t* i_end) {
  const int n = I - 3;  // interior planes [1, I-2)
  if (I < 4 || nranks < 1 || rank < 0 || rank >= nranks || (nranks > 1 && nranks > n / kHalo) ||
      nranks > n || !i_begin || !i_end) {
    set_error("hp_slab_range: bad arguments (I=%d nranks=%d rank=%d)", I, nranks, rank);
    return HP_ERR_ARG;
  }
  *i_begin = 1 + (int)((long long)rank * n / nranks);
  *i_end = 1 + (int)((long long)(rank + 1) * n / nranks);
  return HP_OK;
}

extern "C" int hp_create_slab(int device, const hp_grid* global, int i_begin, int i_end,
                              hp_ctx** out) {
  if (!global || !out) {
    set_error("hp_create_slab: null argument");
    return HP_ERR_ARG;
  }
  *out = nullptr;
  const int I = global->I;
  const bool whole = i_begin == 1 && i_end == I - 2;
  if (I < 4 || global->J < 4 || global->K < 4 || i_begin < 1 || i_end > I - 2 ||
      i_end <= i_begin || (!whole && i_end - i_begin < kHalo)) {
    set_error("hp_create_slab: planes [%d, %d) not a slab (>= %d planes) of the interior of "
              "a %d-plane grid", i_begin, i_end, kHalo, I);
    return HP_ERR_ARG;
  }
  hp_ctx* c = nullptr;
  const int rc = create_ctx(device, i_end - i_begin + 2 * kHalo, global->J, global->K, &c);
  if (rc != HP_OK) return rc;
  c->gI = I;
  c->i_off = i_begin - kHalo;
  c->li_lo = kHalo;
  c->li_hi = i_end - i_begin + kHalo;
  *out = c;
  return HP_OK;
}

namespace {

size_t plane_bytes(const hp_ctx* c) { return c->dev.plane() * sizeof(float); }
int sm_count_of(const hp_ctx* c) {
  int n = 0;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, c->device);
  return n > 0 ? n : 148;
}
float* plane_ptr(hp_ctx* c, float* buf, int li) { return buf + (size_t)li * c->dev.plane(); }

}  // namespace

// ------------------------------------------------------- in-process group

// One pass on a slab: two iterations (two-step kernel) when `step` == 2, else
// one; reads `in`, writes `out`.  Returns kernels launched or -1.
static int slab_pass(hp_ctx* c, const float* in, float* out, int step, const LaunchArgs& a) {
  if (step == 2) {
    const int r = launch_stencil_tb2(c->dev, c->dev.tma, in, out, a, c->sink(), c->stream,
                                     sm_count_of(c));
    if (r != 0) return r;
    return -1;   // every slab has two-plane halos: the two-step kernel must apply
  }
  return launch_stencil_rotate(c->dev, in, out, a, c->sink(), c->stream);
}

static float* pass_buffer(hp_ctx* c, int pass) { return (pass & 1) ? c->scratch : c->dev.f[HP_F_P]; }

// iterations of the next pass: two while temporal blocking is on (same on every rank)
static int pass_step(int done, int nn) {
  return (set_temporal_blocking(-1) && nn - done >= 2) ? 2 : 1;
}

// Halo exchange overlapped with the interior (HIMENO_DD_OVERLAP=0 turns it off):
// a two-step pass runs as (1) the slab's two boundary plane pairs, then an event,
// then (2) the interior; the exchange of pass t waits only for (1) and runs on a
// comm stream while (2) computes; pass t+1 waits for it before its own (1) -- its
// interior needs only the slab's own planes.  SMs left free for NCCL's kernels
// during (2): HIMENO_DD_RESERVE (default 8; copy-engine peer copies need none).
static int dd_overlap() {
  const char* e = getenv("HIMENO_DD_OVERLAP");   // read per call (tests switch it)
  return e ? atoi(e) : 1;
}
static int dd_reserve() {
  const char* e = getenv("HIMENO_DD_RESERVE");
  return e ? atoi(e) : 8;
}

// cuStreamWaitValue32 (driver API, via the runtime's entry-point query): the exchange
// stream waits until a device counter reaches a value -- the boundary units of a
// signalled slab pass bump it from inside the running kernel.  nullptr if unavailable.
typedef CUresult (*WaitValue32Fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
static WaitValue32Fn wait_value32() {
  static WaitValue32Fn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<WaitValue32Fn>(p);
    cudaGetLastError();
    return (WaitValue32Fn) nullptr;
  }();
  return fn;
}

// HIMENO_DD_SIGNAL=0: overlapped passes as two launches (boundary, then interior) with an
// event between them instead of one signalled launch.  Read per call (tests switch it).
static bool dd_signal() {
  const char* e = getenv("HIMENO_DD_SIGNAL");
  return !(e && atoi(e) == 0) && wait_value32() != nullptr;
}

// Boundary counter of one slab context (signalled passes): device word + the value the
// next wait targets.  Reset to 0 between passes when the target nears 2^31 (safe then:
// the compute stream has already waited for the previous exchange).
struct Signal {
  unsigned* dev = nullptr;
  unsigned target = 0;
};

// One signalled pass: one launch, boundary units first; returns kernels launched (1), 0
// if not applicable, -1 on error.  On success sig->target is the count to wait for.
static int slab_pass_signaled(hp_ctx* c, const float* in, float* out, const LaunchArgs& a,
                              int reserve, Signal* sig) {
  if (!sig || !sig->dev || !dd_signal()) return 0;
  if (sig->target > (1u << 30)) {
    if (cudaMemsetAsync(sig->dev, 0, sizeof(unsigned), c->stream) != cudaSuccess) return -1;
    sig->target = 0;
  }
  int nb = 0;
  const int r = launch_stencil_tb2_signaled(c->dev, c->dev.tma, in, out, a, c->sink(), c->stream,
                                            sm_count_of(c), reserve, sig->dev, &nb);
  if (r > 0) sig->target += (unsigned)nb;
  return r;
}

// Make `xs` wait for a signalled pass's boundary units (value >= target).
static cudaError_t gate_on_signal(cudaStream_t xs, const Signal& sig) {
  const CUresult r = wait_value32()(reinterpret_cast<CUstream>(xs),
                                    reinterpret_cast<CUdeviceptr>(sig.dev), sig.target,
                                    CU_STREAM_WAIT_VALUE_GEQ);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorUnknown;
}

// One pass on a slab, split into boundary + interior when overlapping; `bdone` is
// recorded on the compute stream after the planes the neighbours need are written.
static int slab_pass_overlapped(hp_ctx* c, const float* in, float* out, int step,
                                const LaunchArgs& a, bool overlap, int reserve, cudaEvent_t bdone) {
  if (overlap && step == 2) {
    const int r1 = launch_stencil_tb2_part(c->dev, c->dev.tma, in, out, a, c->sink(), c->stream,
                                           sm_count_of(c), 1, 0);
    if (r1 < 0) return -1;
    if (r1 > 0) {
      if (cudaEventRecord(bdone, c->stream) != cudaSuccess) return -1;
      const int r2 = launch_stencil_tb2_part(c->dev, c->dev.tma, in, out, a, c->sink(), c->stream,
                                             sm_count_of(c), 2, reserve);
      return r2 > 0 ? 2 : -1;
    }
  }
  const int r = slab_pass(c, in, out, step, a);
  if (r < 0) return -1;
  return cudaEventRecord(bdone, c->stream) == cudaSuccess ? r : -1;
}

extern "C" int hp_group_jacobi(hp_ctx** ctxs, int n, int nn, double* gosa_out) {
  if (!ctxs || n < 1 || nn < 0) {
    set_error("hp_group_jacobi: bad arguments");
    return HP_ERR_ARG;
  }
  for (int r = 0; r < n; ++r) {
    if (!ctxs[r]) {
      set_error("hp_group_jacobi: null context %d", r);
      return HP_ERR_ARG;
    }
    if (r > 0 && ctxs[r]->i_off + ctxs[r]->li_lo != ctxs[r - 1]->i_off + ctxs[r - 1]->li_hi) {
      set_error("hp_group_jacobi: slab %d does not continue slab %d", r, r - 1);
      return HP_ERR_ARG;
    }
  }
  std::vector<cudaEvent_t> done(n, nullptr), hin(n, nullptr);
  std::vector<cudaStream_t> comm(n, nullptr);
  int rc = HP_OK;
  auto fail = [&](cudaError_t e, const char* what) {
    if (rc == HP_OK) rc = cuda_fail(e, what);
  };
  const bool overlap = dd_overlap() != 0 && n > 1;
  // signalled passes (one launch, the exchange waits on a counter the boundary units bump)
  // when every slab is on one device (the counters are then local to every stream)
  bool one_device = true;
  for (int r = 1; r < n; ++r) one_device = one_device && ctxs[r]->device == ctxs[0]->device;
  std::vector<Signal> sig(n);
  const bool signaled = overlap && one_device && dd_signal();
  for (int r = 0; r < n && rc == HP_OK; ++r) {
    cudaSetDevice(ctxs[r]->device);
    cudaError_t e = cudaEventCreateWithFlags(&done[r], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&hin[r], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&comm[r], cudaStreamNonBlocking);
    if (e == cudaSuccess && signaled) e = cudaMalloc(&sig[r].dev, sizeof(unsigned));
    if (e == cudaSuccess && signaled) e = cudaMemset(sig[r].dev, 0, sizeof(unsigned));
    if (e != cudaSuccess) fail(e, "event / stream create");
    else if (time_loop_begin(ctxs[r], ctx_args(ctxs[r], 1)) < 0) fail(cudaGetLastError(), "begin");
  }
  std::vector<char> gated(n, 0);   // this pass's exchange gates on the counter, not `done`
  int pass = 0;
  for (int it = 0; it < nn && rc == HP_OK; ++pass) {
    const int step = pass_step(it, nn);
    for (int r = 0; r < n && rc == HP_OK; ++r) {
      hp_ctx* c = ctxs[r];
      cudaSetDevice(c->device);
      // the halos of the previous pass, before this pass's boundary planes
      if (pass > 0 && n > 1) {
        cudaError_t e = cudaStreamWaitEvent(c->stream, hin[r], 0);
        if (e != cudaSuccess) fail(e, "wait halo");
      }
      int k = 0;
      gated[r] = 0;
      if (signaled && step == 2) {
        k = slab_pass_signaled(c, pass_buffer(c, pass), pass_buffer(c, pass + 1), ctx_args(c, 1),
                               0, &sig[r]);
        gated[r] = k > 0;
      }
      if (k == 0)
        k = slab_pass_overlapped(c, pass_buffer(c, pass), pass_buffer(c, pass + 1), step,
                                 ctx_args(c, 1), overlap, 0, done[r]);
      else if (k > 0 && cudaEventRecord(done[r], c->stream) != cudaSuccess)   // end of pass
        k = -1;
      if (k < 0) fail(cudaGetLastError(), "stencil pass");
      c->launches += k > 0 ? k : 0;
    }
    // halo planes on each receiver's comm stream (copy engines), after the
    // receiver's and the sender's boundary planes of this pass
    for (int r = 0; r < n && rc == HP_OK && n > 1; ++r) {
      hp_ctx* c = ctxs[r];
      cudaSetDevice(c->device);
      float* out = pass_buffer(c, pass + 1);
      // WAR: the receiver's previous pass no longer reads these halo planes once its
      // current pass runs (its boundary units counted / `done` recorded)
      cudaError_t e = gated[r] ? gate_on_signal(comm[r], sig[r])
                               : cudaStreamWaitEvent(comm[r], done[r], 0);
      for (int side = -1; side <= 1 && rc == HP_OK; side += 2) {
        const int q = r + side;
        if (q < 0 || q >= n) continue;
        hp_ctx* nb = ctxs[q];
        float* nb_out = pass_buffer(nb, pass + 1);
        // lower halo <- neighbour's last two interior planes; upper <- its first two
        const int dst_plane = side < 0 ? c->li_lo - kHalo : c->li_hi;
        const int src_plane = side < 0 ? nb->li_hi - kHalo : nb->li_lo;
        if (e == cudaSuccess)
          e = gated[q] ? gate_on_signal(comm[r], sig[q]) : cudaStreamWaitEvent(comm[r], done[q], 0);
        if (e == cudaSuccess)
          e = cudaMemcpyPeerAsync(plane_ptr(c, out, dst_plane), c->device,
                                  plane_ptr(nb, nb_out, src_plane), nb->device,
                                  kHalo * plane_bytes(c), comm[r]);
        if (e != cudaSuccess) fail(e, "halo copy");
      }
      if (e == cudaSuccess) e = cudaEventRecord(hin[r], comm[r]);
      if (e != cudaSuccess) fail(e, "halo event");
    }
    it += step;
  }
  for (int r = 0; r < n && rc == HP_OK && n > 1 && pass > 0; ++r) {
    cudaSetDevice(ctxs[r]->device);
    cudaError_t e = cudaStreamWaitEvent(ctxs[r]->stream, hin[r], 0);
    if (e != cudaSuccess) fail(e, "wait halo");
  }
  for (int r = 0; r < n && rc == HP_OK; ++r) {
    cudaSetDevice(ctxs[r]->device);
    if (time_loop_finish(ctxs[r], pass_buffer(ctxs[r], pass), ctx_args(ctxs[r], 1)) < 0)
      fail(cudaGetLastError(), "end");
  }
  // gosa of the last iteration: sum of the per-slab fp64 partials, in rank order
  double total = 0.0;
  for (int r = 0; r < n && rc == HP_OK; ++r) {
    hp_ctx* c = ctxs[r];
    cudaSetDevice(c->device);
    double part = 0.0;
    cudaError_t e = cudaMemcpyAsync(&part, c->dscal + HP_V_GOSA * SLOT_BYTES, sizeof(double),
                                    cudaMemcpyDeviceToHost, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) fail(e, "gosa partial");
    total += nn > 0 ? part : 0.0;
  }
  for (int r = 0; r < n; ++r) {
    cudaSetDevice(ctxs[r]->device);
    if (comm[r]) {
      cudaStreamSynchronize(comm[r]);
      cudaStreamDestroy(comm[r]);
    }
    if (done[r]) cudaEventDestroy(done[r]);
    if (hin[r]) cudaEventDestroy(hin[r]);
    if (sig[r].dev) cudaFree(sig[r].dev);
  }
  if (rc == HP_OK && gosa_out) *gosa_out = total;
  return rc;
}

// ----------------------------------------------------------------- NCCL

namespace {

struct Nccl {
  void* handle = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

Nccl* nccl() {
  static Nccl lib;
  static bool tried = false;
  if (tried) return lib.handle ? &lib : nullptr;
  tried = true;
  // HIMENO_NCCL_LIB: an explicit library (tests: tests/nccl_shim.cpp runs the NCCL
  // transport with virtual ranks on one GPU); else prefer an NCCL the process already
  // loaded (torch's), else the system one
  void* h = nullptr;
  if (const char* e = getenv("HIMENO_NCCL_LIB")) h = dlopen(e, RTLD_NOW | RTLD_LOCAL);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return nullptr;
  auto sym = [&](const char* n) { return dlsym(h, n); };
  lib.GetUniqueId = reinterpret_cast<decltype(lib.GetUniqueId)>(sym("ncclGetUniqueId"));
  lib.CommInitRank = reinterpret_cast<decltype(lib.CommInitRank)>(sym("ncclCommInitRank"));
  lib.CommDestroy = reinterpret_cast<decltype(lib.CommDestroy)>(sym("ncclCommDestroy"));
  lib.GroupStart = reinterpret_cast<decltype(lib.GroupStart)>(sym("ncclGroupStart"));
  lib.GroupEnd = reinterpret_cast<decltype(lib.GroupEnd)>(sym("ncclGroupEnd"));
  lib.Send = reinterpret_cast<decltype(lib.Send)>(sym("ncclSend"));
  lib.Recv = reinterpret_cast<decltype(lib.Recv)>(sym("ncclRecv"));
  lib.AllReduce = reinterpret_cast<decltype(lib.AllReduce)>(sym("ncclAllReduce"));
  lib.GetErrorString = reinterpret_cast<decltype(lib.GetErrorString)>(sym("ncclGetErrorString"));
  if (!lib.GetUniqueId || !lib.CommInitRank || !lib.CommDestroy || !lib.GroupStart ||
      !lib.GroupEnd || !lib.Send || !lib.Recv || !lib.AllReduce || !lib.GetErrorString)
    return nullptr;
  lib.handle = h;
  return &lib;
}

struct DD {
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
  cudaStream_t xs = nullptr;      // halo exchange stream (overlapped with the interior)
  cudaEvent_t bdone = nullptr;    // boundary planes of the current pass written
  cudaEvent_t hin = nullptr;      // halos of the current pass received
  Signal sig;                     // signalled passes: boundary-unit counter
};

int nccl_fail(ncclResult_t r, const char* what) {
  set_error("%s: %s", what, nccl() ? nccl()->GetErrorString(r) : "nccl unavailable");
  return HP_ERR_DEVICE;
}

}  // namespace

void hp::dd_destroy(hp_ctx* c) {
  DD* d = static_cast<DD*>(c->dd);
  if (d && d->comm && nccl()) nccl()->CommDestroy(d->comm);
  if (d && d->xs) {
    cudaStreamSynchronize(d->xs);
    cudaStreamDestroy(d->xs);
  }
  if (d && d->bdone) cudaEventDestroy(d->bdone);
  if (d && d->hin) cudaEventDestroy(d->hin);
  if (d && d->sig.dev) cudaFree(d->sig.dev);
  delete d;
  c->dd = nullptr;
}

extern "C" int hp_nccl_unique_id(unsigned char* out, size_t n) {
  if (!out || n < NCCL_UNIQUE_ID_BYTES) {
    set_error("hp_nccl_unique_id: need %d bytes", NCCL_UNIQUE_ID_BYTES);
    return HP_ERR_ARG;
  }
  Nccl* l = nccl();
  if (!l) {
    set_error("libnccl.so.2 not available");
    return HP_ERR_DEVICE;
  }
  ncclUniqueId id;
  const ncclResult_t r = l->GetUniqueId(&id);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  memcpy(out, id.internal, NCCL_UNIQUE_ID_BYTES);
  return HP_OK;
}

extern "C" int hp_dd_init(hp_ctx* c, int nranks, int rank, const unsigned char* id, size_t n) {
  if (!c || nranks < 1 || rank < 0 || rank >= nranks || (nranks > 1 && (!id || n < 128))) {
    set_error("hp_dd_init: bad arguments");
    return HP_ERR_ARG;
  }
  if (c->dd) dd_destroy(c);
  DD* d = new DD;
  d->nranks = nranks;
  d->rank = rank;
  // a communicator also for a single rank when an id is given (the NCCL transport
  // then runs its all-reduce over one rank: how it is exercised on a 1-GPU box)
  if (nranks > 1 || (id && n >= NCCL_UNIQUE_ID_BYTES)) {
    Nccl* l = nccl();
    if (!l) {
      delete d;
      set_error("libnccl.so.2 not available");
      return HP_ERR_DEVICE;
    }
    ncclUniqueId uid;
    memcpy(uid.internal, id, NCCL_UNIQUE_ID_BYTES);
    cudaSetDevice(c->device);
    const ncclResult_t r = l->CommInitRank(&d->comm, nranks, uid, rank);
    if (r != ncclSuccess) {
      delete d;
      return nccl_fail(r, "ncclCommInitRank");
    }
  }
  cudaSetDevice(c->device);
  if (cudaStreamCreateWithFlags(&d->xs, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&d->bdone, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&d->hin, cudaEventDisableTiming) != cudaSuccess ||
      cudaMalloc(&d->sig.dev, sizeof(unsigned)) != cudaSuccess ||
      cudaMemset(d->sig.dev, 0, sizeof(unsigned)) != cudaSuccess) {
    c->dd = d;
    dd_destroy(c);
    return cuda_fail(cudaGetLastError(), "hp_dd_init streams");
  }
  c->dd = d;
  return HP_OK;
}

// nn iterations in passes (two-step while temporal blocking is on), two halo
// planes per side exchanged after each pass, then the gosa all-reduce; async.
extern "C" int hp_dd_jacobi(hp_ctx* c, int nn) {
  if (!c || !c->dd || nn < 0) {
    set_error("hp_dd_jacobi: context not initialised for decomposition");
    return HP_ERR_ARG;
  }
  DD* d = static_cast<DD*>(c->dd);
  Nccl* l = d->comm ? nccl() : nullptr;
  cudaSetDevice(c->device);
  const LaunchArgs a = ctx_args(c, 1);
  if (time_loop_begin(c, a) < 0) return cuda_fail(cudaGetLastError(), "begin");
  const size_t count = kHalo * c->dev.plane();
  const bool overlap = dd_overlap() != 0 && l && d->nranks > 1;
  const int reserve = overlap ? dd_reserve() : 0;
  int pass = 0;
  for (int it = 0; it < nn; ++pass) {
    const int step = pass_step(it, nn);
    if (pass > 0 && l) {   // the previous pass's halos before this pass's boundary planes
      const cudaError_t e = cudaStreamWaitEvent(c->stream, d->hin, 0);
      if (e != cudaSuccess) return cuda_fail(e, "wait halo");
    }
    int k = 0;
    bool gated = false;
    if (overlap && step == 2) {   // one launch, the exchange gated on the boundary counter
      k = slab_pass_signaled(c, pass_buffer(c, pass), pass_buffer(c, pass + 1), a, reserve,
                             &d->sig);
      gated = k > 0;
    }
    if (k == 0)
      k = slab_pass_overlapped(c, pass_buffer(c, pass), pass_buffer(c, pass + 1), step, a,
                               overlap, reserve, d->bdone);
    if (k < 0) return cuda_fail(cudaGetLastError(), "stencil pass");
    c->launches += k;
    it += step;
    if (!l) continue;
    // halo exchange on the exchange stream once the boundary planes are written
    cudaError_t e = gated ? gate_on_signal(d->xs, d->sig) : cudaStreamWaitEvent(d->xs, d->bdone, 0);
    if (e != cudaSuccess) return cuda_fail(e, "wait boundary");
    float* out = pass_buffer(c, pass + 1);
    ncclResult_t r = l->GroupStart();
    if (d->rank > 0) {
      if (r == ncclSuccess)
        r = l->Send(plane_ptr(c, out, c->li_lo), count, ncclFloat32, d->rank - 1, d->comm, d->xs);
      if (r == ncclSuccess)
        r = l->Recv(plane_ptr(c, out, c->li_lo - kHalo), count, ncclFloat32, d->rank - 1, d->comm,
                    d->xs);
    }
    if (d->rank < d->nranks - 1) {
      if (r == ncclSuccess)
        r = l->Send(plane_ptr(c, out, c->li_hi - kHalo), count, ncclFloat32, d->rank + 1, d->comm,
                    d->xs);
      if (r == ncclSuccess)
        r = l->Recv(plane_ptr(c, out, c->li_hi), count, ncclFloat32, d->rank + 1, d->comm, d->xs);
    }
    const ncclResult_t r2 = l->GroupEnd();
    if (r != ncclSuccess) return nccl_fail(r, "halo exchange");
    if (r2 != ncclSuccess) return nccl_fail(r2, "ncclGroupEnd");
    if ((e = cudaEventRecord(d->hin, d->xs)) != cudaSuccess) return cuda_fail(e, "halo event");
  }
  if (l && pass > 0) {
    const cudaError_t e = cudaStreamWaitEvent(c->stream, d->hin, 0);
    if (e != cudaSuccess) return cuda_fail(e, "wait halo");
  }
  if (time_loop_finish(c, pass_buffer(c, pass), a) < 0) return cuda_fail(cudaGetLastError(), "end");
  if (l && nn > 0) {
    double* g = reinterpret_cast<double*>(c->dscal + HP_V_GOSA * SLOT_BYTES);
    const ncclResult_t r = l->AllReduce(g, g, 1, ncclFloat64, ncclSum, d->comm, c->stream);
    if (r != ncclSuccess) return nccl_fail(r, "gosa all-reduce");
  }
  return HP_OK;
}

extern "C" int hp_dd_time_steps(hp_ctx* c, int steps, int nn, double* ms_out) {
  if (!c || !ms_out || steps < 0) {
    set_error("hp_dd_time_steps: bad arguments");
    return HP_ERR_ARG;
  }
  cudaSetDevice(c->device);
  cudaError_t e = cudaEventRecord(c->ev0, c->stream);
  if (e != cudaSuccess) return cuda_fail(e, "event record");
  for (int s = 0; s < steps; ++s) {
    const int rc = hp_dd_jacobi(c, nn);
    if (rc != HP_OK) return rc;
  }
  if ((e = cudaEventRecord(c->ev1, c->stream)) != cudaSuccess) return cuda_fail(e, "event record");
  if ((e = cudaEventSynchronize(c->ev1)) != cudaSuccess) return cuda_fail(e, "event sync");
  float ms = 0.f;
  cudaEventElapsedTime(&ms, c->ev0, c->ev1);
  *ms_out = ms;
  return HP_OK;
}
