// NCCL halo transport of libsdrt (see comm.h).  Only the handful of NCCL entry points
// the exchange needs are resolved; the types below are NCCL's public ABI (nccl.h):
// ncclUniqueId = 128 bytes, ncclComm_t = pointer, enums as int.
#include "comm.h"

#include <dlfcn.h>

#include <mutex>
#include <stdexcept>
#include <vector>

namespace sdrt {

namespace {

typedef int ncclResult_t;
typedef void* ncclComm_t;
struct ncclUniqueId_t {
  char internal[128];
};
constexpr int kNcclFloat64 = 8;  // ncclFloat64 / ncclDouble
constexpr int kNcclUint64 = 5;   // ncclUint64
constexpr int kNcclMin = 3;      // ncclMin

struct Api {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId_t*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId_t, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

Api& api() {
  static Api a;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      a.h = dlopen(n, RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);  // the process's copy (torch's)
      if (a.h) break;
    }
    for (const char* n : names) {
      if (a.h) break;
      a.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
    }
    if (!a.h) return;
    auto sym = [&](const char* s) { return dlsym(a.h, s); };
    a.GetUniqueId = (decltype(a.GetUniqueId))sym("ncclGetUniqueId");
    a.CommInitRank = (decltype(a.CommInitRank))sym("ncclCommInitRank");
    a.CommDestroy = (decltype(a.CommDestroy))sym("ncclCommDestroy");
    a.GroupStart = (decltype(a.GroupStart))sym("ncclGroupStart");
    a.GroupEnd = (decltype(a.GroupEnd))sym("ncclGroupEnd");
    a.Send = (decltype(a.Send))sym("ncclSend");
    a.Recv = (decltype(a.Recv))sym("ncclRecv");
    a.AllReduce = (decltype(a.AllReduce))sym("ncclAllReduce");
    a.GetErrorString = (decltype(a.GetErrorString))sym("ncclGetErrorString");
    if (!a.GetUniqueId || !a.CommInitRank || !a.CommDestroy || !a.GroupStart || !a.GroupEnd || !a.Send ||
        !a.Recv || !a.AllReduce)
      a.h = nullptr;
  });
  if (!a.h) throw std::runtime_error("nccl: libnccl.so.2 not found or incomplete");
  return a;
}

void check(ncclResult_t r, const char* what) {
  if (r != 0) {
    const char* s = api().GetErrorString ? api().GetErrorString(r) : "?";
    throw std::runtime_error(std::string("nccl: ") + what + " failed: " + s);
  }
}

}  // namespace

struct NcclComm {
  ncclComm_t comm = nullptr;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev[2] = {nullptr, nullptr};
};

void nccl_unique_id(uint8_t id[128]) {
  ncclUniqueId_t u;
  check(api().GetUniqueId(&u), "ncclGetUniqueId");
  for (int i = 0; i < 128; ++i) id[i] = (uint8_t)u.internal[i];
}

NcclComm* nccl_comm_create(const uint8_t id[128], int rank, int nranks) {
  ncclUniqueId_t u;
  for (int i = 0; i < 128; ++i) u.internal[i] = (char)id[i];
  auto* c = new NcclComm;
  ncclResult_t r = api().CommInitRank(&c->comm, nranks, u, rank);
  if (r != 0) {
    delete c;
    check(r, "ncclCommInitRank");
  }
  if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev[0], cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev[1], cudaEventDisableTiming) != cudaSuccess) {
    nccl_comm_destroy(c);
    throw std::runtime_error("nccl: comm stream / event creation failed");
  }
  return c;
}

void nccl_comm_destroy(NcclComm* c) {
  if (!c) return;
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->comm) api().CommDestroy(c->comm);
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

cudaStream_t nccl_comm_stream(NcclComm* c) { return c->stream; }
cudaEvent_t nccl_comm_event(NcclComm* c, int k) { return c->ev[k]; }

void nccl_exchange(NcclComm* c, int n, const double* const* sbuf, const int64_t* n_send, const int* peer_send,
                   double* const* rbuf, const int64_t* n_recv, const int* peer_recv) {
  Api& a = api();
  check(a.GroupStart(), "ncclGroupStart");
  for (int i = 0; i < n; ++i) {
    if (n_send[i] > 0) check(a.Send(sbuf[i], (size_t)n_send[i], kNcclFloat64, peer_send[i], c->comm, c->stream), "ncclSend");
    if (n_recv[i] > 0) check(a.Recv(rbuf[i], (size_t)n_recv[i], kNcclFloat64, peer_recv[i], c->comm, c->stream), "ncclRecv");
  }
  check(a.GroupEnd(), "ncclGroupEnd");
}

void nccl_allreduce_min_u64(NcclComm* c, unsigned long long* d_val, cudaStream_t st) {
  check(api().AllReduce(d_val, d_val, 1, kNcclUint64, kNcclMin, c->comm, st), "ncclAllReduce");
}

}  // namespace sdrt
