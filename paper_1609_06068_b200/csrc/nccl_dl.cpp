// NCCL, resolved at run time with dlopen so that single-GPU use has no NCCL
// dependency.  Search order: an NCCL already loaded in the process (torch's,
// RTLD_NOLOAD), $SDP_NCCL_LIB (the binding points it at torch's bundled copy),
// then the soname.  Always RTLD_LOCAL: loading the system libnccl globally
// before torch would make torch bind its newer NCCL symbols to the older one.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "internal.h"

namespace sdp {

namespace {
struct NcclApi {
  void* lib = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
};
NcclApi g_nccl;
std::once_flag g_once;
std::string g_load_error;

void load() {
  g_nccl.lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL | RTLD_NOLOAD);
  const char* env = getenv("SDP_NCCL_LIB");
  if (!g_nccl.lib && env && *env) g_nccl.lib = dlopen(env, RTLD_NOW | RTLD_LOCAL);
  const char* names[] = {"libnccl.so.2", "libnccl.so"};
  for (const char* nm : names) {
    if (g_nccl.lib) break;
    g_nccl.lib = dlopen(nm, RTLD_NOW | RTLD_LOCAL);
  }
  if (!g_nccl.lib) {
    g_load_error = std::string("dlopen(libnccl.so.2) failed: ") + dlerror();
    return;
  }
  g_nccl.getUniqueId = (decltype(g_nccl.getUniqueId))dlsym(g_nccl.lib, "ncclGetUniqueId");
  g_nccl.commInitRank = (decltype(g_nccl.commInitRank))dlsym(g_nccl.lib, "ncclCommInitRank");
  g_nccl.allReduce = (decltype(g_nccl.allReduce))dlsym(g_nccl.lib, "ncclAllReduce");
  g_nccl.commDestroy = (decltype(g_nccl.commDestroy))dlsym(g_nccl.lib, "ncclCommDestroy");
  g_nccl.getErrorString = (decltype(g_nccl.getErrorString))dlsym(g_nccl.lib, "ncclGetErrorString");
  if (!g_nccl.getUniqueId || !g_nccl.commInitRank || !g_nccl.allReduce || !g_nccl.commDestroy)
    g_load_error = "libnccl.so.2 lacks a required symbol";
}

void need() {
  std::call_once(g_once, load);
  if (!g_load_error.empty()) throw Error{SDP_E_NCCL, g_load_error};
}

void check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw Error{SDP_E_NCCL, std::string(what) + ": " + (g_nccl.getErrorString ? g_nccl.getErrorString(r) : "error")};
}
}  // namespace

void nccl_unique_id(void* out128) {
  need();
  ncclUniqueId id;
  check(g_nccl.getUniqueId(&id), "ncclGetUniqueId");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  std::memcpy(out128, &id, sizeof(id));
}

void* nccl_comm_init(const void* id128, int world, int rank) {
  need();
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  ncclComm_t comm = nullptr;
  check(g_nccl.commInitRank(&comm, world, id, rank), "ncclCommInitRank");
  return (void*)comm;
}

void nccl_allreduce_sum(void* comm, double* buf, size_t count, cudaStream_t s) {
  if (count == 0) return;
  check(g_nccl.allReduce(buf, buf, count, ncclFloat64, ncclSum, (ncclComm_t)comm, s), "ncclAllReduce");
}

void nccl_comm_destroy(void* comm) {
  if (comm && g_nccl.commDestroy) g_nccl.commDestroy((ncclComm_t)comm);
}

}  // namespace sdp
