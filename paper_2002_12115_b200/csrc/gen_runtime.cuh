// Runtime of the generated B200 executors (codegen.py): loop hooks, the
// whole-array device data manager, reductions, the C ABI (include/app_b200.h).
//
// Semantics follow the Himeno library's executor (executor.cpp), at array
// granularity instead of boxes:
//   * every array has a host and a device version (write clock); a guarded
//     transfer is skipped when the destination already holds newer data
//     (SURVEY.md Appendix B.2), otherwise it copies the whole array;
//   * plan events (lower.py) fire before / after their loop statement:
//     declare create, update device / self, structured data enter / exit with
//     present_or_copy reference counts, present assertions;
//   * a kernel launch implicitly copies in (and afterwards out, then frees) every
//     array it touches that is not present -- OpenACC's present_or_copy default;
//   * scalars are host-authoritative: kernels receive them by value
//     (firstprivate), reductions return into the host variable; scalar plan
//     events are counted (bytes, events) but move nothing;
//   * a fresh run zeroes the program's statics (a new process) and treats device
//     memory as undefined;
//   * writes are tracked as boxes on both sides: each launch reports the box of every
//     array it writes and each host-executed loop the box its own statements wrote,
//     computed from the loop bounds (codegen.write_boxes / host_write_boxes); a
//     guarded transfer moves exactly the source side's dirty boxes, or the whole array
//     when the destination copy is undefined or the writes are unbounded -- so
//     undefined or stale memory never lands on newer data (the hazard of the
//     reference's plans on real hardware; the Himeno library's
//     coherence log does the same per box) and a pattern pays only the bytes it changes;
//   * a launch whose write box is not exact first brings an undefined or stale device
//     copy up to date (n_guard_init), so the over-approximated box is safe;
//   * small whole-array uploads go through a pinned staging ring without a host
//     wait; large ones and box copies wait (the host may write the array next).
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "app_b200.h"

namespace hpg {

struct VarDesc {
  const char* name;
  int is_array;
  unsigned long long bytes;
};

enum { ST_OK = 0, ST_PATTERN = 1, ST_LAUNCH = 2, ST_TIMEOUT = 3, ST_PRESENT = 4 };
enum { ERR_DEVICE = -1, ERR_ARG = -2, ERR_OOM = -3 };
enum { EV_UPDATE_DEVICE = 1, EV_UPDATE_SELF, EV_DATA_ENTER, EV_DATA_EXIT, EV_DECLARE, EV_PRESENT };
enum { K_HOST = 0, K_KERNELS = 1, K_PL = 2, K_PLV = 3, K_COVERED = 4 };
enum { FLAG_GUARD = 1, FLAG_FRESH = 2 };

struct Failure {
  int code;
  char msg[256];
};

inline thread_local char g_last_error[512] = "";
inline void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof g_last_error, fmt, ap);
  va_end(ap);
}

inline double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

// Block partial of a reduction slot: warp shuffles then warps in fixed order;
// every thread of the block calls it (same slot sequence).
__device__ inline void block_reduce_store(double v, double* out, int slot, int nslots) {
  __shared__ double part[32];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  __syncthreads();
  if (lane == 0) part[w] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int x = 0; x < nw; ++x) s += part[x];
    out[(size_t)blockIdx.x * nslots + slot] = s;
  }
  __syncthreads();
}

struct Tables {
  int nloops, nvars;
  const VarDesc* vars;
  const unsigned* const* dims;   // per variable: extents (arrays)
  const int* ndims;
  const unsigned long long* elems;
  const int* elig_kind;
  const int* parent;
  const int* const* loop_wr;
  const int* loop_wr_n;
  const int* const* pre_wr;
  const int* pre_wr_n;
};

class Runtime {
 public:
  Tables T{};
  int device = -1;
  bool has_dev = false;
  cudaStream_t stream = nullptr;
  int sms = 148;
  std::vector<void*> host_ptr, dev_ptr;
  // per run
  const hpg_schedule* S = nullptr;
  hpg_result* Rz = nullptr;
  std::vector<std::vector<const hpg_event*>> before_ev, after_ev;
  std::vector<uint64_t> host_ver, dev_ver;
  std::vector<int> refcount;
  std::vector<char> declared;
  uint64_t clock = 1;
  bool guard = true;
  double deadline = 0;
  std::string out;
  double* d_red = nullptr;
  double* h_red = nullptr;
  size_t red_cap = 0;
  std::vector<std::vector<int>> implicit_stack;
  struct Box4 {
    long long lo[4], hi[4];
  };
  std::vector<std::vector<Box4>> dirty;   // per array: device-written boxes since last sync
  std::vector<char> dirty_full;
  std::vector<std::vector<Box4>> hdirty;  // per array: host-written boxes since last sync
  std::vector<char> hdirty_full;
  std::vector<char> dev_defined;          // device copy holds the whole array (a full h2d)

  // pinned staging ring for small host -> device copies: the host copy is snapshotted
  // into the ring and the transfer proceeds asynchronously, so the program keeps
  // running (and may write the array again) while it is in flight
  static constexpr size_t kStageSmall = 256 << 10;
  static constexpr size_t kRingBytes = 64 << 20;
  char* ring = nullptr;
  size_t ring_off = 0;

  ~Runtime() {
    if (ring) cudaFreeHost(ring);
    if (d_red) cudaFree(d_red);
    if (h_red) cudaFreeHost(h_red);
    for (void* p : dev_ptr)
      if (p) cudaFree(p);
    if (stream) cudaStreamDestroy(stream);
  }

  [[noreturn]] void fail(int code, const char* fmt, ...) {
    Failure f;
    f.code = code;
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(f.msg, sizeof f.msg, fmt, ap);
    va_end(ap);
    throw f;
  }
  int vprint(const char* f, va_list ap) {
    char buf[1024];
    const int n = vsnprintf(buf, sizeof buf, f, ap);
    if (n > 0) out.append(buf, std::min<size_t>((size_t)n, sizeof buf - 1));
    return n;
  }
  void cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(ST_LAUNCH, "%s: %s", what, cudaGetErrorString(e));
  }

  // ---- loop hooks ----------------------------------------------------------
  int kind(int L) const { return S->loop_kind[L]; }
  bool dev(int L) const { return kind(L) >= K_KERNELS && kind(L) <= K_PLV; }
  void host_only(int L) {
    if (dev(L)) fail(ST_PATTERN, "loop %d has no device version", L);
  }
  // host statements wrote these arrays somewhere (no box known): host-newer everywhere
  void host_writes(const int* v, int n) {
    for (int x = 0; x < n; ++x) {
      if (v[x] < 0) continue;
      host_ver[v[x]] = ++clock;
      hdirty_full[v[x]] = 1;
      hdirty[v[x]].clear();
    }
  }
  // a host-executed loop reports the box its own statements wrote (codegen.write_boxes
  // on the host version, evaluated after the loop)
  void host_wrote(int v, const long long* lo, const long long* hi, int nd) {
    host_ver[v] = ++clock;
    if (hdirty_full[v]) return;
    Box4 b;
    if (!make_box(v, lo, hi, nd, b)) return;
    if (is_full(v, b) || hdirty[v].size() >= 64) {
      hdirty_full[v] = 1;
      hdirty[v].clear();
    } else if (!hdirty_full[v]) {
      hdirty[v].push_back(b);
    }
  }
  bool on_host(int L) const { return kind(L) == K_HOST; }
  void before(int L) {
    if (deadline > 0 && now_s() > deadline) fail(ST_TIMEOUT, "watchdog: run exceeded %.1f s", S->timeout_s);
    // host statements that ran since the previous hook: the host region right
    // before a top-level loop, or the enclosing host loop's own statements
    if (T.pre_wr[L]) host_writes(T.pre_wr[L], T.pre_wr_n[L]);
    const int p = T.parent[L];
    if (p >= 0 && on_host(p)) host_writes(T.loop_wr[p], T.loop_wr_n[p]);
    for (const hpg_event* e : before_ev[L]) fire(e);
  }
  void after(int L) {
    for (const hpg_event* e : after_ev[L]) fire(e);
  }

  // ---- data manager ----------------------------------------------------------
  // Each array has two dirty sets: boxes the host wrote since the device copy was last
  // brought up to date, and boxes the device wrote since the host copy was.  A guarded
  // transfer moves exactly the source's dirty boxes (both ways), or the whole array
  // when the destination copy is undefined or the source's writes are unbounded; an
  // unguarded one (HP flag off) is the literal whole-array copy.
  bool present(int v) const { return declared[v] || refcount[v] > 0; }
  bool make_box(int v, const long long* lo, const long long* hi, int nd, Box4& b) const {
    const unsigned* dims = T.dims[v];
    for (int d = 0; d < 4; ++d) {
      const long long ext = d < nd ? (long long)dims[d] : 1;
      b.lo[d] = d < nd ? std::max<long long>(0, lo[d]) : 0;
      b.hi[d] = d < nd ? std::min<long long>(ext, hi[d]) : 1;
      if (b.lo[d] >= b.hi[d]) return false;   // empty
    }
    return true;
  }
  bool is_full(int v, const Box4& b) const {
    for (int d = 0; d < T.ndims[v]; ++d)
      if (b.lo[d] != 0 || b.hi[d] != (long long)T.dims[v][d]) return false;
    return true;
  }
  size_t box_bytes(int v, const Box4& b) const {
    size_t n = T.vars[v].bytes / T.elems[v];
    for (int d = 0; d < T.ndims[v]; ++d) n *= (size_t)(b.hi[d] - b.lo[d]);
    return n;
  }
  // boxes are worth it only when few and small: each strided copy costs a call
  // (~10 us) where one contiguous whole-array copy streams at PCIe bandwidth
  bool boxes_pay(int v, const std::vector<Box4>& bs) const {
    if (bs.size() > 4) return false;
    size_t sum = 0;
    for (const Box4& b : bs) sum += box_bytes(v, b);
    return sum * 4 <= T.vars[v].bytes;
  }
  // one box of array v between host and device (innermost three dims per memcpy3D;
  // a box whose inner dimensions are full is one contiguous copy)
  void copy_box(int v, const Box4& b, cudaMemcpyKind kind) {
    {
      const int nd = T.ndims[v];
      int d0 = 0;   // first dim that is not a single index
      while (d0 < nd && b.hi[d0] - b.lo[d0] == 1) ++d0;
      bool contiguous = true;
      for (int d = d0 + 1; d < nd; ++d)
        contiguous = contiguous && b.lo[d] == 0 && b.hi[d] == (long long)T.dims[v][d];
      if (contiguous) {
        const size_t esz = T.vars[v].bytes / T.elems[v];
        size_t off = 0;
        for (int d = 0; d < nd; ++d) off = off * T.dims[v][d] + (size_t)b.lo[d];
        const size_t bytes = box_bytes(v, b);
        const bool up = kind == cudaMemcpyHostToDevice;
        char* h = (char*)host_ptr[v] + off * esz;
        char* dv = (char*)dev_ptr[v] + off * esz;
        cuda(cudaMemcpyAsync(up ? dv : h, up ? h : dv, bytes, kind, stream),
             up ? "h2d box" : "d2h box");
        (up ? Rz->h2d_bytes : Rz->d2h_bytes) += bytes;
        return;
      }
    }
    const int nd = T.ndims[v];
    const unsigned* dims = T.dims[v];
    const size_t esz = T.vars[v].bytes / T.elems[v];
    long long ext[4], lo[4], hi[4];
    for (int d = 0; d < 4; ++d) {   // right-align the dims into 4
      const int sd = d - (4 - nd);
      ext[d] = sd >= 0 ? dims[sd] : 1;
      lo[d] = sd >= 0 ? b.lo[sd] : 0;
      hi[d] = sd >= 0 ? b.hi[sd] : 1;
    }
    const size_t row = (size_t)ext[3] * esz, vol = row * ext[2] * ext[1];
    const bool up = kind == cudaMemcpyHostToDevice;
    for (long long i0 = lo[0]; i0 < hi[0]; ++i0) {
      cudaMemcpy3DParms m = {};
      char* hbase = (char*)host_ptr[v] + i0 * vol;
      char* dbase = (char*)dev_ptr[v] + i0 * vol;
      const cudaPitchedPtr hp = make_cudaPitchedPtr(hbase, row, row, (size_t)ext[2]);
      const cudaPitchedPtr dp = make_cudaPitchedPtr(dbase, row, row, (size_t)ext[2]);
      m.srcPtr = up ? hp : dp;
      m.dstPtr = up ? dp : hp;
      m.srcPos = make_cudaPos((size_t)lo[3] * esz, (size_t)lo[2], (size_t)lo[1]);
      m.dstPos = m.srcPos;
      m.extent = make_cudaExtent((size_t)(hi[3] - lo[3]) * esz, (size_t)(hi[2] - lo[2]),
                                 (size_t)(hi[1] - lo[1]));
      m.kind = kind;
      cuda(cudaMemcpy3DAsync(&m, stream), up ? "h2d box" : "d2h box");
      const uint64_t bytes = (uint64_t)m.extent.width * m.extent.height * m.extent.depth;
      (up ? Rz->h2d_bytes : Rz->d2h_bytes) += bytes;
    }
  }
  void full_h2d(int v) {
    const VarDesc& d = T.vars[v];
    if (d.bytes <= kStageSmall) {
      if (!ring && cudaMallocHost(&ring, kRingBytes) != cudaSuccess) {
        ring = nullptr;
        fail(ST_LAUNCH, "staging ring allocation failed");
      }
      if (ring_off + d.bytes > kRingBytes) {   // wrap: earlier copies out of the ring first
        cuda(cudaStreamSynchronize(stream), "staging ring wrap");
        ring_off = 0;
      }
      std::memcpy(ring + ring_off, host_ptr[v], d.bytes);
      cuda(cudaMemcpyAsync(dev_ptr[v], ring + ring_off, d.bytes, cudaMemcpyHostToDevice, stream),
           "h2d (staged)");
      ring_off = (ring_off + d.bytes + 255) & ~(size_t)255;
    } else {
      cuda(cudaMemcpyAsync(dev_ptr[v], host_ptr[v], d.bytes, cudaMemcpyHostToDevice, stream),
           "h2d");
      cuda(cudaStreamSynchronize(stream), "h2d sync");
    }
    Rz->h2d_bytes += d.bytes;
  }
  void flush_dev_boxes(int v) {   // device-newer boxes -> host (before a whole-array h2d)
    if (dirty[v].empty()) return;
    for (const Box4& b : dirty[v]) copy_box(v, b, cudaMemcpyDeviceToHost);
    cuda(cudaStreamSynchronize(stream), "flush device boxes");
    dirty[v].clear();
  }
  void h2d(int v, bool implicit) {
    const VarDesc& d = T.vars[v];
    if (!d.is_array) {   // host-authoritative scalar: counted only
      Rz->h2d_bytes += d.bytes;
      Rz->n_h2d++;
      return;
    }
    if (!has_dev) fail(ST_LAUNCH, "no device for update device(%s)", d.name);
    const double t0 = now_s();
    if (!guard) {
      full_h2d(v);
      dirty[v].clear();
      dirty_full[v] = 0;
      dev_defined[v] = 1;
    } else if (!dev_defined[v] || hdirty_full[v]) {
      if (dirty_full[v] && dev_ver[v] > host_ver[v]) {   // device newer everywhere: stale update
        Rz->n_skipped_stale++;
        hdirty[v].clear();
        hdirty_full[v] = 0;
        return;
      }
      flush_dev_boxes(v);
      full_h2d(v);
      dev_defined[v] = 1;
    } else if (!hdirty[v].empty()) {
      if (boxes_pay(v, hdirty[v])) {
        for (const Box4& b : hdirty[v]) copy_box(v, b, cudaMemcpyHostToDevice);
        cuda(cudaStreamSynchronize(stream), "h2d boxes");
      } else {
        flush_dev_boxes(v);
        full_h2d(v);
      }
    } else {
      Rz->n_skipped_stale++;   // nothing the device does not already hold
      return;
    }
    hdirty[v].clear();
    hdirty_full[v] = 0;
    Rz->xfer_s += now_s() - t0;
    Rz->n_h2d++;
    if (implicit) Rz->n_implicit++;
    dev_ver[v] = std::max(dev_ver[v], host_ver[v]);
  }
  void dev_wrote(int v, const long long* lo, const long long* hi, int nd) {
    dev_ver[v] = ++clock;
    Box4 b;
    if (!make_box(v, lo, hi, nd, b)) return;
    if (is_full(v, b)) dev_defined[v] = 1;   // the device wrote every element
    if (is_full(v, b) || dirty[v].size() >= 64) {
      dirty_full[v] = 1;
      dirty[v].clear();
    } else if (!dirty_full[v]) {
      dirty[v].push_back(b);
    }
  }
  void d2h(int v, bool implicit) {
    const VarDesc& d = T.vars[v];
    if (!d.is_array) {
      Rz->d2h_bytes += d.bytes;
      Rz->n_d2h++;
      return;
    }
    if (!has_dev) fail(ST_LAUNCH, "no device for update self(%s)", d.name);
    const double t0 = now_s();
    if (!guard || dirty_full[v]) {
      if (guard && hdirty_full[v] && host_ver[v] > dev_ver[v]) {   // host newer everywhere
        Rz->n_skipped_stale++;
        return;
      }
      cuda(cudaMemcpyAsync(host_ptr[v], dev_ptr[v], d.bytes, cudaMemcpyDeviceToHost, stream),
           "d2h");
      Rz->d2h_bytes += d.bytes;
    } else if (!dirty[v].empty()) {
      if (boxes_pay(v, dirty[v]) || !dev_defined[v] || !hdirty[v].empty() || hdirty_full[v]) {
        // (a whole-array copy is only safe when the device copy is complete and the
        // host has no newer data)
        for (const Box4& b : dirty[v]) copy_box(v, b, cudaMemcpyDeviceToHost);
      } else {
        cuda(cudaMemcpyAsync(host_ptr[v], dev_ptr[v], d.bytes, cudaMemcpyDeviceToHost, stream),
             "d2h");
        Rz->d2h_bytes += d.bytes;
      }
    } else {
      Rz->n_skipped_stale++;   // the device wrote nothing since the last synchronisation
      return;
    }
    cuda(cudaStreamSynchronize(stream), "d2h sync");
    Rz->xfer_s += now_s() - t0;
    dirty[v].clear();
    dirty_full[v] = 0;
    Rz->n_d2h++;
    if (implicit) Rz->n_implicit++;
    host_ver[v] = std::max(host_ver[v], dev_ver[v]);
  }
  void dealloc(int v) {
    dev_ver[v] = 0;
    dirty[v].clear();
    dirty_full[v] = 0;
    dev_defined[v] = 0;
  }
  void fire(const hpg_event* e) {
    const int v = e->var;
    switch (e->op) {
      case EV_DECLARE: declared[v] = 1; break;
      case EV_UPDATE_DEVICE: h2d(v, false); break;
      case EV_UPDATE_SELF: d2h(v, false); break;
      case EV_DATA_ENTER:
        if (present(v)) {
          if (!declared[v]) refcount[v]++;
        } else {
          refcount[v] = 1;
          if (e->arg) h2d(v, false);
        }
        break;
      case EV_DATA_EXIT:
        if (declared[v]) break;
        if (refcount[v] > 0 && --refcount[v] == 0) {
          if (e->arg) d2h(v, false);
          dealloc(v);
        }
        break;
      case EV_PRESENT:
        if (!present(v))
          fail(ST_PRESENT, "present(%s) failed at loop %d: data not on device", T.vars[v].name,
               e->loop_id);
        break;
      default: fail(ST_PATTERN, "unknown event op %d", e->op);
    }
  }

  // ---- kernels --------------------------------------------------------------
  // wr: the arrays this launch writes with an inexact (over-approximated) box
  void kernel_enter(int L, const int* arrs, int n, const int* wr, int nw) {
    if (!has_dev) fail(ST_LAUNCH, "loop %d: no CUDA device in this context", L);
    implicit_stack.emplace_back();
    for (int x = 0; x < n; ++x) {
      const int v = arrs[x];
      if (v < 0 || present(v)) continue;
      h2d(v, true);
      implicit_stack.back().push_back(v);
    }
    // an over-approximated write box needs a complete, current device copy (else
    // the later copy-out of the whole box would carry undefined or stale elements)
    for (int x = 0; x < nw; ++x) {
      const int v = wr[x];
      if (v < 0 || !T.vars[v].is_array) continue;
      if (dev_defined[v] && !hdirty_full[v] && hdirty[v].empty()) continue;
      const bool g = guard;
      guard = true;
      h2d(v, false);
      guard = g;
      Rz->n_guard_init++;
    }
  }
  void kernel_exit(int L, const int* arrs, int n, const int* wr, int nw) {
    (void)L;
    (void)arrs;
    (void)n;
    (void)wr;
    (void)nw;
    std::vector<int> imp = std::move(implicit_stack.back());
    implicit_stack.pop_back();
    for (int v : imp) {
      d2h(v, true);
      dealloc(v);
    }
  }
  int grid_for(long long total, int single) const {
    if (single) return 1;
    const long long b = (total + 255) / 256;
    return (int)std::max<long long>(1, std::min<long long>(b, (long long)sms * 8));
  }
  // every generated kernel starts with griddepcontrol.launch_dependents + wait, so it
  // can be launched with programmatic stream serialization: launch N+1 is scheduled
  // while N runs, touches no data before N completed (loop-per-launch patterns)
  template <typename... KArgs, typename... Args>
  void launch(void (*kern)(KArgs...), int grid, int block, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.stream = stream;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cuda(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...), "launch");
  }
  template <typename... KArgs, typename... Args>
  void launch2(void (*kern)(KArgs...), int gx, int gy, int block, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.gridDim = dim3(gx, gy);
    cfg.blockDim = dim3(block);
    cfg.stream = stream;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cuda(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...), "launch");
  }
  // blocks per gang when the vector loops need no barrier: fill about two waves
  int vector_split(long long gangs) const {
    const long long want = (2LL * sms + gangs - 1) / std::max<long long>(1, gangs);
    return (int)std::max<long long>(1, std::min<long long>(want, 64));
  }
  int gang_grid(long long total) const {
    return (int)std::max<long long>(1, std::min<long long>(total, (long long)sms * 16));
  }
  double* red_buffer(int grid, int nslots) {
    const size_t need = (size_t)grid * nslots;
    if (need > red_cap) {
      if (d_red) cudaFree(d_red);
      if (h_red) cudaFreeHost(h_red);
      d_red = nullptr;
      h_red = nullptr;
      red_cap = std::max<size_t>(need, 4096);
      if (cudaMalloc(&d_red, red_cap * sizeof(double)) != cudaSuccess ||
          cudaMallocHost(&h_red, red_cap * sizeof(double)) != cudaSuccess)
        fail(ST_LAUNCH, "reduction buffer allocation failed");
    }
    return d_red;
  }
  void launched(int L) {
    cudaError_t e = cudaPeekAtLastError();
    if (e != cudaSuccess) fail(ST_LAUNCH, "launch of loop %d failed: %s", L, cudaGetErrorString(e));
    Rz->n_launch++;
  }
  // block partials in block order -> per-slot sums (waits for the kernel)
  void fetch_sums(int grid, int nslots, double* out_v) {
    cuda(cudaMemcpyAsync(h_red, d_red, (size_t)grid * nslots * sizeof(double),
                         cudaMemcpyDeviceToHost, stream), "reduction d2h");
    cuda(cudaStreamSynchronize(stream), "reduction sync");
    for (int r = 0; r < nslots; ++r) {
      double s = 0.0;
      for (int b = 0; b < grid; ++b) s += h_red[(size_t)b * nslots + r];
      out_v[r] = s;
    }
  }

  // ---- run setup -------------------------------------------------------------
  void prepare(const hpg_schedule* s, hpg_result* r) {
    S = s;
    Rz = r;
    if (s->n_loops != T.nloops) {
      set_error("schedule has %d loops, program has %d", s->n_loops, T.nloops);
      throw ERR_ARG;
    }
    before_ev.assign(T.nloops + 1, {});
    after_ev.assign(T.nloops + 1, {});
    for (int n = 0; n < s->n_events; ++n) {
      const hpg_event* e = &s->events[n];
      if (e->var < 0 || e->var >= T.nvars || e->loop_id < -1 || e->loop_id >= T.nloops) {
        set_error("event %d out of range", n);
        throw ERR_ARG;
      }
      if (e->op == EV_DECLARE) continue;
      (e->when == 0 ? before_ev : after_ev)[e->loop_id].push_back(e);
    }
    // same intra-hook order as the Himeno executor: updates, enters, present, exits
    auto rank = [](const hpg_event* e) {
      switch (e->op) {
        case EV_UPDATE_DEVICE: return 10;
        case EV_DATA_ENTER: return 20;
        case EV_PRESENT: return 30;
        case EV_DATA_EXIT: return 60;
        default: return 90;
      }
    };
    for (auto& v : before_ev)
      std::stable_sort(v.begin(), v.end(), [&](auto* a, auto* b) { return rank(a) < rank(b); });
    for (auto& v : after_ev)
      std::stable_sort(v.begin(), v.end(), [&](auto* a, auto* b) { return rank(a) < rank(b); });
    for (int L = 0; L < T.nloops; ++L)
      if (dev(L) && T.elig_kind[L] == 0) {
        r->status = ST_PATTERN;
        snprintf(r->diag, sizeof r->diag, "loop %d is not offloadable", L);
      }
    host_ver.assign(T.nvars, 1);
    dev_ver.assign(T.nvars, 0);
    refcount.assign(T.nvars, 0);
    declared.assign(T.nvars, 0);
    dirty.assign(T.nvars, {});
    dirty_full.assign(T.nvars, 0);
    hdirty.assign(T.nvars, {});
    hdirty_full.assign(T.nvars, 1);   // zeroed statics: defined on the host only
    dev_defined.assign(T.nvars, 0);
    clock = 1;
    guard = (s->flags & FLAG_GUARD) != 0;
    out.clear();
    implicit_stack.clear();
    for (int n = 0; n < s->n_events; ++n)
      if (s->events[n].op == EV_DECLARE) declared[s->events[n].var] = 1;
  }
};

}  // namespace hpg

struct hpg_ctx {
  hpg::Runtime R;
  void* P = nullptr;        // the application's Prog (statics + functions)
  size_t prog_bytes = 0;
  bool pinned = false;
};

namespace hpg {

// C ABI of one generated application A (A::Prog, A::kLoops, A::kVars, A::tables(),
// A::bind(Prog*, Runtime&)); instantiated once per shared library.
template <class A>
struct Abi {
  using Prog = typename A::Prog;
  static int create(int device, hpg_ctx** out) {
    if (!out) return ERR_ARG;
    *out = nullptr;
    hpg_ctx* c = new (std::nothrow) hpg_ctx;
    if (!c) return ERR_OOM;
    c->R.T = A::tables();
    c->R.host_ptr.assign(A::kVars, nullptr);
    c->R.dev_ptr.assign(A::kVars, nullptr);
    c->prog_bytes = sizeof(Prog);
    if (device >= 0) {
      int n = 0;
      if (cudaGetDeviceCount(&n) != cudaSuccess || device >= n) {
        cudaGetLastError();
        set_error("hpg_create: no CUDA device %d", device);
        delete c;
        return ERR_DEVICE;
      }
      cudaSetDevice(device);
      c->R.device = device;
      c->R.has_dev = true;
      cudaDeviceGetAttribute(&c->R.sms, cudaDevAttrMultiProcessorCount, device);
      if (cudaStreamCreateWithFlags(&c->R.stream, cudaStreamNonBlocking) != cudaSuccess ||
          cudaMallocHost(&c->P, sizeof(Prog)) != cudaSuccess) {
        set_error("hpg_create: stream / pinned allocation failed: %s",
                  cudaGetErrorString(cudaGetLastError()));
        delete c;
        return ERR_DEVICE;
      }
      c->pinned = true;
    } else {
      c->P = std::aligned_alloc(4096, (sizeof(Prog) + 4095) / 4096 * 4096);
      if (!c->P) {
        delete c;
        return ERR_OOM;
      }
    }
    std::memset(c->P, 0, sizeof(Prog));
    Prog* P = new (c->P) Prog(c->R);
    A::bind(P, c->R);
    if (c->R.has_dev) {
      for (int v = 0; v < A::kVars; ++v)
        if (c->R.T.vars[v].is_array &&
            cudaMalloc(&c->R.dev_ptr[v], c->R.T.vars[v].bytes) != cudaSuccess) {
          set_error("hpg_create: device allocation of %s failed", c->R.T.vars[v].name);
          destroy(c);
          return ERR_OOM;
        }
    }
    *out = c;
    return 0;
  }
  static void destroy(hpg_ctx* c) {
    if (!c) return;
    if (c->R.has_dev) cudaSetDevice(c->R.device);
    if (c->P) {
      static_cast<Prog*>(c->P)->~Prog();
      if (c->pinned) cudaFreeHost(c->P);
      else std::free(c->P);
    }
    delete c;
  }
  static int run(hpg_ctx* c, const hpg_schedule* s, hpg_result* r) {
    if (!c || !s || !r || (s->n_events > 0 && !s->events) || !s->loop_kind) {
      set_error("hpg_run: bad arguments");
      return ERR_ARG;
    }
    std::memset(r, 0, sizeof *r);
    Runtime& R = c->R;
    if (R.has_dev && cudaSetDevice(R.device) != cudaSuccess) {
      set_error("hpg_run: cudaSetDevice failed");
      return ERR_DEVICE;
    }
    try {
      R.prepare(s, r);
    } catch (int rc) {
      return rc;
    }
    if (r->status != ST_OK) {
      set_error("%s", r->diag);
      return r->status;
    }
    Prog* P = static_cast<Prog*>(c->P);
    if (s->flags & FLAG_FRESH) {   // a new process: zeroed statics (not timed)
      P->~Prog();
      std::memset(c->P, 0, sizeof(Prog));
      P = new (c->P) Prog(R);
      A::bind(P, R);
    }
    const double t0 = now_s();
    R.deadline = s->timeout_s > 0 ? t0 + s->timeout_s : 0;
    try {
      P->main_();
      if (R.has_dev) R.cuda(cudaStreamSynchronize(R.stream), "program end");
      r->status = ST_OK;
    } catch (const Failure& f) {
      if (R.has_dev) {
        cudaStreamSynchronize(R.stream);
        cudaGetLastError();
      }
      r->status = f.code;
      snprintf(r->diag, sizeof r->diag, "%s", f.msg);
      set_error("%s", f.msg);
    }
    r->wall_s = now_s() - t0;
    return r->status;
  }
  static size_t output(hpg_ctx* c, char* dst, size_t cap) {
    if (!c) return 0;
    const size_t n = c->R.out.size();
    if (dst && cap) {
      const size_t m = std::min(n, cap - 1);
      std::memcpy(dst, c->R.out.data(), m);
      dst[m] = 0;
    }
    return n;
  }
};

}  // namespace hpg

#define HPG_DEFINE_APP(NS)                                                                   \
  extern "C" int hpg_create(int device, hpg_ctx** out) { return hpg::Abi<NS::App>::create(device, out); } \
  extern "C" void hpg_destroy(hpg_ctx* c) { hpg::Abi<NS::App>::destroy(c); }                 \
  extern "C" int hpg_run(hpg_ctx* c, const hpg_schedule* s, hpg_result* r) {                 \
    return hpg::Abi<NS::App>::run(c, s, r);                                                  \
  }                                                                                          \
  extern "C" size_t hpg_output(hpg_ctx* c, char* d, size_t n) { return hpg::Abi<NS::App>::output(c, d, n); } \
  extern "C" int hpg_n_loops(void) { return NS::App::kLoops; }                               \
  extern "C" int hpg_n_vars(void) { return NS::App::kVars; }                                 \
  extern "C" const char* hpg_var_name(int v) {                                               \
    return v >= 0 && v < NS::App::kVars ? NS::kVarDesc[v].name : nullptr;                    \
  }                                                                                          \
  extern "C" int hpg_loop_kind(int l) {                                                      \
    return l >= 0 && l < NS::App::kLoops ? NS::kEligibleKind[l] : -1;                        \
  }                                                                                          \
  extern "C" const char* hpg_loop_note(int l) {                                              \
    return l >= 0 && l < NS::App::kLoops ? NS::kLoopNote[l] : nullptr;                       \
  }                                                                                          \
  extern "C" const char* hpg_last_error(void) { return hpg::g_last_error; }
