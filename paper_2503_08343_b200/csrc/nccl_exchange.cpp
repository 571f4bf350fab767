// Native NCCL transport for the partitioned factorization: a
// gmrf_exchange_fn that posts an exchange point's messages straight on the
// factor's stream — ncclSend / ncclRecv in one group for the Schur complements,
// solve vectors and Σ blocks, ncclAllReduce for the results — with no trip
// through the host language at the exchange points (the torch.distributed
// callback of partition.py stays for the CPU/gloo tests).
//
// NCCL is resolved at run time (dlopen of the library the process already
// carries, e.g. torch's libnccl.so.2): libgmrf_b200.so has no link-time
// dependency on it and single-GPU use never touches it. Only the handful of
// entry points below are used; their prototypes follow nccl.h (2.x ABI).
#include <dlfcn.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "../../include/gmrf_b200.h"
#include "common.hpp"

namespace {

struct NcclId {
  char internal[128];  // ncclUniqueId
};
using Comm = void*;
// ncclDataType_t / ncclRedOp_t values of nccl.h
constexpr int kInt32 = 2, kFloat64 = 8, kSum = 0, kMin = 3;

struct Api {
  void* lib = nullptr;
  int (*GetUniqueId)(NcclId*) = nullptr;
  int (*CommInitRank)(Comm*, int, NcclId, int) = nullptr;
  int (*CommDestroy)(Comm) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  int (*Send)(const void*, size_t, int, int, Comm, void*) = nullptr;
  int (*Recv)(void*, size_t, int, int, Comm, void*) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, Comm, void*) = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
};

Api& api() {
  static Api a;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {std::getenv("GMRF_NCCL_LIB"), "libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      if (!n) continue;
      a.lib = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (a.lib) break;
    }
    if (!a.lib) return;
    auto sym = [&](const char* s) { return dlsym(a.lib, s); };
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
    a.Send = reinterpret_cast<decltype(a.Send)>(sym("ncclSend"));
    a.Recv = reinterpret_cast<decltype(a.Recv)>(sym("ncclRecv"));
    a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(sym("ncclAllReduce"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
  });
  return a;
}

Api& need_api() {
  Api& a = api();
  gmrf::require(a.lib && a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.GroupStart &&
                    a.GroupEnd && a.Send && a.Recv && a.AllReduce,
                gmrf::kCuda, "NCCL not available (libnccl.so.2 could not be loaded; set GMRF_NCCL_LIB)");
  return a;
}

void ck(Api& a, int rc, const char* what) {
  if (rc != 0)
    gmrf::fail(gmrf::kCuda, std::string(what) + ": " +
                                (a.GetErrorString ? a.GetErrorString(rc) : "NCCL error"));
}

// gmrf_exchange_fn: ctx is the ncclComm_t
int nccl_exchange(void* ctx, const gmrf_msg_t* msgs, int32_t count, void* stream) {
  try {
    Api& a = need_api();
    Comm comm = ctx;
    bool p2p = false;
    for (int32_t i = 0; i < count; ++i) p2p = p2p || msgs[i].kind == 0 || msgs[i].kind == 1;
    if (p2p) {
      // every send/recv of the exchange point in one group: progress does not
      // depend on the order the two sides list them in
      ck(a, a.GroupStart(), "ncclGroupStart");
      for (int32_t i = 0; i < count; ++i) {
        const gmrf_msg_t& m = msgs[i];
        if (m.kind == 0)
          ck(a, a.Send(m.dptr, static_cast<size_t>(m.count), kFloat64, m.peer, comm, stream), "ncclSend");
        else if (m.kind == 1)
          ck(a, a.Recv(m.dptr, static_cast<size_t>(m.count), kFloat64, m.peer, comm, stream), "ncclRecv");
      }
      ck(a, a.GroupEnd(), "ncclGroupEnd");
    }
    for (int32_t i = 0; i < count; ++i) {
      const gmrf_msg_t& m = msgs[i];
      if (m.kind == 2)  // disjoint owned entries, zeros elsewhere: the sum is exact in any order
        ck(a, a.AllReduce(m.dptr, m.dptr, static_cast<size_t>(m.count), kFloat64, kSum, comm, stream),
           "ncclAllReduce");
      else if (m.kind == 3)
        ck(a, a.AllReduce(m.dptr, m.dptr, static_cast<size_t>(m.count), kInt32, kMin, comm, stream),
           "ncclAllReduce");
    }
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}

thread_local std::string g_nccl_err;

template <typename F>
int guard(F&& f) {
  try {
    f();
    return GMRF_OK;
  } catch (const gmrf::Error& e) {
    g_nccl_err = e.what();
    return e.status;
  } catch (const std::exception& e) {
    g_nccl_err = e.what();
    return GMRF_ERR_CUDA;
  }
}

}  // namespace

extern "C" {

int gmrf_nccl_unique_id(uint8_t* id128) {
  return guard([&] {
    gmrf::require(id128 != nullptr, gmrf::kContract, "nccl: null id buffer");
    Api& a = need_api();
    NcclId id;
    ck(a, a.GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(id128, id.internal, sizeof(id.internal));
  });
}

int gmrf_nccl_comm_create(int32_t nranks, int32_t rank, const uint8_t* id128, void** comm) {
  return guard([&] {
    gmrf::require(id128 && comm && nranks >= 1 && rank >= 0 && rank < nranks, gmrf::kContract,
                  "nccl: bad communicator arguments");
    Api& a = need_api();
    NcclId id;
    std::memcpy(id.internal, id128, sizeof(id.internal));
    Comm c = nullptr;
    ck(a, a.CommInitRank(&c, nranks, id, rank), "ncclCommInitRank");
    *comm = c;
  });
}

void gmrf_nccl_comm_destroy(void* comm) {
  Api& a = api();
  if (comm && a.CommDestroy) a.CommDestroy(comm);
}

gmrf_exchange_fn gmrf_nccl_exchange(void) { return &nccl_exchange; }

const char* gmrf_nccl_last_error(void) { return g_nccl_err.c_str(); }

}  // extern "C"
