// Test-only stand-in for libnccl.so.2 (the subset decomp.cpp uses), so the library's
// NCCL transport -- hp_dd_init / hp_dd_jacobi with the halo exchange overlapped with
// the interior -- can run with several ranks on ONE GPU (real NCCL refuses two ranks on
// one device).  Ranks are threads of one process, each with its own slab context.
//
// Semantics kept: stream ordering.  ncclSend records an event on the sender's stream;
// the matching ncclRecv (paired per (src, dst) in issue order) makes the receiver's
// stream wait for it and copies device to device on that stream; the sender's stream
// then waits for the copy (the send buffer may be rewritten only after it).  Pairing is
// a host rendezvous at ncclGroupEnd.  ncclAllReduce (double, sum) sums the ranks' values
// on the host in rank order.  Not a performance model.
//
//   g++ -O2 -shared -fPIC -I<cuda>/include tests/nccl_shim.cpp -L<cuda>/lib64 -lcudart
#include <cuda_runtime.h>
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <random>
#include <string>
#include <vector>

namespace {

struct Msg {
  const void* buf;
  size_t bytes;
  cudaEvent_t ready;        // sender's stream reached the send
  cudaEvent_t done = nullptr;   // receiver's copy finished (set by the receiver)
};

struct World {
  int nranks = 0;
  std::mutex mu;
  std::condition_variable cv;
  std::map<std::pair<int, int>, std::deque<std::shared_ptr<Msg>>> q;   // (src, dst)
  // all-reduce rendezvous
  int ar_round = 0, ar_count = 0;
  std::vector<double> ar_vals;
  double ar_total = 0.0;
};

std::mutex g_mu;
std::map<std::string, std::shared_ptr<World>> g_worlds;

struct Op {
  bool send;
  void* buf;
  size_t bytes;
  int peer;
  cudaStream_t stream;
};

}  // namespace

struct ncclComm {
  std::shared_ptr<World> w;
  int rank;
};

static thread_local int t_group = 0;
static thread_local std::vector<std::pair<ncclComm*, Op>> t_ops;

static size_t type_size(ncclDataType_t t) {
  switch (t) {
    case ncclFloat64: case ncclInt64: case ncclUint64: return 8;
    case ncclFloat16: case ncclBfloat16: return 2;
    case ncclInt8: case ncclUint8: return 1;
    default: return 4;
  }
}

static ncclResult_t flush_ops() {
  std::vector<std::pair<ncclComm*, std::shared_ptr<Msg>>> mine;
  for (auto& [comm, op] : t_ops)   // publish the sends
    if (op.send) {
      auto m = std::make_shared<Msg>();
      m->buf = op.buf;
      m->bytes = op.bytes;
      cudaEventCreateWithFlags(&m->ready, cudaEventDisableTiming);
      cudaEventRecord(m->ready, op.stream);
      {
        std::lock_guard<std::mutex> lk(comm->w->mu);
        comm->w->q[{comm->rank, op.peer}].push_back(m);
      }
      comm->w->cv.notify_all();
      mine.push_back({comm, m});
    }
  for (auto& [comm, op] : t_ops)   // receive: copy after the sender's event
    if (!op.send) {
      std::shared_ptr<Msg> m;
      {
        std::unique_lock<std::mutex> lk(comm->w->mu);
        auto& dq = comm->w->q[{op.peer, comm->rank}];
        comm->w->cv.wait(lk, [&] { return !dq.empty(); });
        m = dq.front();
        dq.pop_front();
      }
      if (m->bytes != op.bytes) return ncclInvalidArgument;
      cudaStreamWaitEvent(op.stream, m->ready, 0);
      cudaMemcpyAsync(op.buf, m->buf, op.bytes, cudaMemcpyDeviceToDevice, op.stream);
      cudaEvent_t d;
      cudaEventCreateWithFlags(&d, cudaEventDisableTiming);
      cudaEventRecord(d, op.stream);
      {
        std::lock_guard<std::mutex> lk(comm->w->mu);
        m->done = d;
      }
      comm->w->cv.notify_all();
    }
  for (auto& [comm, m] : mine) {   // the send buffer is free once the copy ran
    std::unique_lock<std::mutex> lk(comm->w->mu);
    comm->w->cv.wait(lk, [&] { return m->done != nullptr; });
    cudaStream_t s = nullptr;
    for (auto& [c2, op] : t_ops)
      if (op.send && c2 == comm && op.buf == m->buf) s = op.stream;
    lk.unlock();
    cudaStreamWaitEvent(s, m->done, 0);
  }
  t_ops.clear();
  return ncclSuccess;
}

extern "C" {

ncclResult_t ncclGetUniqueId(ncclUniqueId* id) {
  std::random_device rd;
  memset(id->internal, 0, sizeof id->internal);
  snprintf(id->internal, sizeof id->internal, "shim-%u-%u", rd(), rd());
  return ncclSuccess;
}

ncclResult_t ncclCommInitRank(ncclComm_t* comm, int nranks, ncclUniqueId id, int rank) {
  const std::string key(id.internal, strnlen(id.internal, sizeof id.internal));
  std::shared_ptr<World> w;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto& slot = g_worlds[key];
    if (!slot) {
      slot = std::make_shared<World>();
      slot->nranks = nranks;
      slot->ar_vals.assign(nranks, 0.0);
    }
    w = slot;
  }
  if (w->nranks != nranks || rank < 0 || rank >= nranks) return ncclInvalidArgument;
  *comm = new ncclComm{w, rank};
  return ncclSuccess;
}

ncclResult_t ncclCommDestroy(ncclComm_t comm) {
  delete comm;
  return ncclSuccess;
}

ncclResult_t ncclGroupStart() {
  ++t_group;
  return ncclSuccess;
}

ncclResult_t ncclGroupEnd() {
  if (--t_group == 0) return flush_ops();
  return ncclSuccess;
}

ncclResult_t ncclSend(const void* buf, size_t count, ncclDataType_t type, int peer, ncclComm_t comm,
                      cudaStream_t stream) {
  t_ops.push_back({comm, Op{true, const_cast<void*>(buf), count * type_size(type), peer, stream}});
  return t_group ? ncclSuccess : flush_ops();
}

ncclResult_t ncclRecv(void* buf, size_t count, ncclDataType_t type, int peer, ncclComm_t comm,
                      cudaStream_t stream) {
  t_ops.push_back({comm, Op{false, buf, count * type_size(type), peer, stream}});
  return t_group ? ncclSuccess : flush_ops();
}

ncclResult_t ncclAllReduce(const void* send, void* recv, size_t count, ncclDataType_t type,
                           ncclRedOp_t op, ncclComm_t comm, cudaStream_t stream) {
  if (type != ncclFloat64 || op != ncclSum || count != 1) return ncclInvalidArgument;
  double v = 0.0;
  cudaMemcpyAsync(&v, send, 8, cudaMemcpyDeviceToHost, stream);
  cudaStreamSynchronize(stream);
  World& w = *comm->w;
  double total;
  {
    std::unique_lock<std::mutex> lk(w.mu);
    const int round = w.ar_round;
    w.ar_vals[comm->rank] = v;
    if (++w.ar_count == w.nranks) {
      double t = 0.0;
      for (double x : w.ar_vals) t += x;   // rank order
      w.ar_total = t;
      w.ar_count = 0;
      ++w.ar_round;
      w.cv.notify_all();
    } else {
      w.cv.wait(lk, [&] { return w.ar_round != round; });
    }
    total = w.ar_total;
  }
  cudaMemcpyAsync(recv, &total, 8, cudaMemcpyHostToDevice, stream);
  cudaStreamSynchronize(stream);
  return ncclSuccess;
}

const char* ncclGetErrorString(ncclResult_t r) { return r == ncclSuccess ? "success" : "nccl shim error"; }

}  // extern "C"
