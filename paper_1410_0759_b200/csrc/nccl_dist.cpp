// Native NCCL for the batch-sharded backward-filter: the
// library loads libnccl at run time (dlopen; the process' already-loaded
// copy when there is one, e.g. torch's), so libdnnp.so has no link-time NCCL
// dependency and a C caller can shard a minibatch without any Python or
// torch: dnnp_nccl_unique_id / dnnp_nccl_comm_create (or
// dnnp_set_nccl_comm with the caller's own ncclComm_t) and
// dnnp_convolution_backward_filter_allreduce.  Reductions are enqueued on the
// handle's stream, so they order with the convolution kernels and can be
// captured into a CUDA graph.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "core.h"

namespace dnnp {
namespace nccl {
namespace {

struct Api {
  void* lib = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  std::string why;
};

const Api& api() {
  static Api a;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {getenv("DNNP_NCCL_LIB"), "libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      if (!n || !*n) continue;
      a.lib = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (a.lib) break;
    }
    if (!a.lib) {
      a.why = "libnccl.so.2 not found (set DNNP_NCCL_LIB)";
      return;
    }
    a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(a.lib, "ncclGetUniqueId"));
    a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(a.lib, "ncclCommInitRank"));
    a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(a.lib, "ncclCommDestroy"));
    a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(dlsym(a.lib, "ncclAllReduce"));
    a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(a.lib, "ncclGetErrorString"));
    if (!a.get_unique_id || !a.comm_init_rank || !a.comm_destroy || !a.all_reduce ||
        !a.error_string) {
      a.why = "libnccl is missing an entry point";
      a.lib = nullptr;
    }
  });
  return a;
}

}  // namespace

bool available(const char** why) {
  const Api& a = api();
  if (!a.lib && why) *why = a.why.c_str();
  return a.lib != nullptr;
}

const char* error_string(int r) {
  const Api& a = api();
  return a.lib ? a.error_string(ncclResult_t(r)) : "NCCL unavailable";
}

int unique_id(void* out) {
  const Api& a = api();
  if (!a.lib) return int(ncclSystemError);
  ncclUniqueId id;
  const ncclResult_t r = a.get_unique_id(&id);
  if (r == ncclSuccess) memcpy(out, &id, sizeof id);
  return int(r);
}

int comm_init(void** comm, const void* id, int nranks, int rank) {
  const Api& a = api();
  if (!a.lib) return int(ncclSystemError);
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof uid);
  ncclComm_t c = nullptr;
  const ncclResult_t r = a.comm_init_rank(&c, nranks, uid, rank);
  *comm = c;
  return int(r);
}

int comm_destroy(void* comm) {
  const Api& a = api();
  if (!a.lib || !comm) return int(ncclSuccess);
  return int(a.comm_destroy(static_cast<ncclComm_t>(comm)));
}

int allreduce_sum(const void* send, void* recv, size_t count, bool f64, void* comm,
                  cudaStream_t st) {
  const Api& a = api();
  if (!a.lib) return int(ncclSystemError);
  return int(a.all_reduce(send, recv, count, f64 ? ncclFloat64 : ncclFloat32, ncclSum,
                          static_cast<ncclComm_t>(comm), st));
}

}  // namespace nccl
}  // namespace dnnp
