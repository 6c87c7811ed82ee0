// Native NCCL transport of the subdomain-partitioned DDM: the per-macro-step
// trace / ghost exchange as ncclSend / ncclRecv groups and the reductions as ncclAllReduce, issued
// by the library on its solver stream (so partitioned applications stay graph-captured and no host
// code runs between macro-steps). The reference has no counterpart: it deposits traces in shared
// memory (/root/reference/proj/src/sweeper.cpp:295-307, src/transfer.cpp:24-36).
//
// libnccl is loaded at run time (dlopen), not linked: the process may already hold one (PyTorch
// bundles NCCL 2.28; the system has 2.27), and whichever is present serves. The library's
// communicator is its own (ncclCommInitRank from a 128-byte unique id the caller distributes), so
// it never shares state with a framework's communicator.
#include "hs_nccl.hpp"

#include <dlfcn.h>

#include <cstdlib>
#include <mutex>
#include <string>

namespace hsb {

namespace {

struct Api {
  void* h = nullptr;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) =
      nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GetVersion)(int*) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

template <class T>
bool sym(void* h, const char* name, T& fn) {
  fn = reinterpret_cast<T>(dlsym(h, name));
  return fn != nullptr;
}

Api load() {
  Api a;
  // the copy the process already holds, then an explicit path, then the loader's search path
  const char* env = std::getenv("HS_NCCL_LIB");
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h && env) h = dlopen(env, RTLD_NOW | RTLD_LOCAL);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
  if (!h) {
    const char* e = dlerror();
    a.why = std::string("libnccl.so.2 not loadable: ") + (e ? e : "unknown");
    return a;
  }
  bool ok = sym(h, "ncclGetUniqueId", a.GetUniqueId) && sym(h, "ncclCommInitRank", a.CommInitRank) &&
            sym(h, "ncclCommDestroy", a.CommDestroy) && sym(h, "ncclGroupStart", a.GroupStart) &&
            sym(h, "ncclGroupEnd", a.GroupEnd) && sym(h, "ncclSend", a.Send) && sym(h, "ncclRecv", a.Recv) &&
            sym(h, "ncclAllReduce", a.AllReduce) && sym(h, "ncclAllGather", a.AllGather) &&
            sym(h, "ncclGetVersion", a.GetVersion) && sym(h, "ncclGetErrorString", a.GetErrorString);
  if (!ok) {
    a.why = "libnccl.so.2 lacks an expected entry point";
    return a;
  }
  a.h = h;
  return a;
}

const Api& api() {
  static std::once_flag once;
  static Api a;
  std::call_once(once, [] { a = load(); });
  if (!a.h) throw Error(kCuda, "NCCL transport: " + a.why);
  return a;
}

void check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw Error(kCuda, std::string("NCCL ") + what + ": " + api().GetErrorString(r));
}

}  // namespace

int nccl_version() {
  int v = 0;
  check(api().GetVersion(&v), "ncclGetVersion");
  return v;
}

void nccl_unique_id(unsigned char out[NCCL_UNIQUE_ID_BYTES]) {
  ncclUniqueId id;
  check(api().GetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out, id.internal, NCCL_UNIQUE_ID_BYTES);
}

NcclComm::NcclComm(const unsigned char id[NCCL_UNIQUE_ID_BYTES], int rank_, int world_) : rank(rank_), world(world_) {
  ncclUniqueId u;
  std::memcpy(u.internal, id, NCCL_UNIQUE_ID_BYTES);
  check(api().CommInitRank(&comm, world, u, rank), "ncclCommInitRank");
}

NcclComm::~NcclComm() {
  if (comm) api().CommDestroy(comm);
}

void NcclComm::exchange(int npeers, const int* peers, const std::int64_t* soff, const std::int64_t* scnt,
                        const std::int64_t* roff, const std::int64_t* rcnt, const double* send, double* recv,
                        cudaStream_t s) {
  const Api& a = api();
  check(a.GroupStart(), "ncclGroupStart");
  for (int i = 0; i < npeers; ++i) {
    if (scnt[i] > 0) check(a.Send(send + soff[i], static_cast<size_t>(scnt[i]), ncclFloat64, peers[i], comm, s), "ncclSend");
    if (rcnt[i] > 0) check(a.Recv(recv + roff[i], static_cast<size_t>(rcnt[i]), ncclFloat64, peers[i], comm, s), "ncclRecv");
  }
  check(a.GroupEnd(), "ncclGroupEnd");
}

void NcclComm::allreduce(double* buf, std::int64_t count, cudaStream_t s) {
  check(api().AllReduce(buf, buf, static_cast<size_t>(count), ncclFloat64, ncclSum, comm, s), "ncclAllReduce");
}

void NcclComm::allgather(const double* send, double* recv, std::int64_t count, cudaStream_t s) {
  check(api().AllGather(send, recv, static_cast<size_t>(count), ncclFloat64, comm, s), "ncclAllGather");
}

}  // namespace hsb
