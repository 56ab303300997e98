// Inter-GPU gradient exchange of the stream-sharded data parallelism
// (streams are independent, so each GPU owns a slice of
// them; gradients are raw sums over streams, reference engine.py:593-598).
//
// NCCL (the pip wheel torch links, 2.28.x) is bound at run time with dlopen,
// so the library loads -- and every non-collective entry point works --
// without NCCL present; rgb_comm_init reports its absence.  One communicator
// per process (one process per GPU); the collectives run on the caller's
// stream (rgb_allreduce_*) or, for the bucketed backward, on the plan's
// communication stream forked from / joined into the caller's stream
// (rgb_plan.cu, STEP_AR), which CUDA-graph capture records like any other
// fork/join.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "../../include/rnngraph_b200.h"
#include "rgb_comm.cuh"

namespace {

// the slice of nccl.h this file needs (types are ABI-stable since NCCL 2.0)
typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;
enum { ncclSuccess = 0 };
enum { ncclFloat32 = 7, ncclFloat64 = 8 };
enum { ncclSum = 0, ncclMax = 2 };

struct Nccl {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*GetVersion)(int*) = nullptr;
};

thread_local std::string g_comm_err;

int cfail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_comm_err = buf;
  rgb::set_last_error(buf);
  return code;
}

// libnccl.so.2: already mapped by torch in a PyTorch process (dlopen by
// soname returns it), else RGB_NCCL_LIB, else the loader's search path
Nccl* nccl() {
  static Nccl n;
  static bool tried = false;
  if (tried) return n.h ? &n : nullptr;
  tried = true;
  const char* env = getenv("RGB_NCCL_LIB");
  const char* names[] = {env, "libnccl.so.2", "libnccl.so"};
  for (const char* name : names) {
    if (!name) continue;
    n.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
    if (n.h) break;
  }
  if (!n.h) return nullptr;
  auto sym = [&](const char* s) { return dlsym(n.h, s); };
  n.GetUniqueId = reinterpret_cast<decltype(n.GetUniqueId)>(sym("ncclGetUniqueId"));
  n.CommInitRank = reinterpret_cast<decltype(n.CommInitRank)>(sym("ncclCommInitRank"));
  n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(sym("ncclCommDestroy"));
  n.AllReduce = reinterpret_cast<decltype(n.AllReduce)>(sym("ncclAllReduce"));
  n.GroupStart = reinterpret_cast<decltype(n.GroupStart)>(sym("ncclGroupStart"));
  n.GroupEnd = reinterpret_cast<decltype(n.GroupEnd)>(sym("ncclGroupEnd"));
  n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(sym("ncclGetErrorString"));
  n.GetVersion = reinterpret_cast<decltype(n.GetVersion)>(sym("ncclGetVersion"));
  if (!n.GetUniqueId || !n.CommInitRank || !n.CommDestroy || !n.AllReduce || !n.GroupStart || !n.GroupEnd) {
    dlclose(n.h);
    n.h = nullptr;
    return nullptr;
  }
  return &n;
}

int nccl_rc(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return RGB_OK;
  Nccl* n = nccl();
  return cfail(RGB_ERR_CUDA, "%s: %s", what, n && n->GetErrorString ? n->GetErrorString(r) : "NCCL error");
}

}  // namespace

struct rgb_comm {
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
};

namespace rgb {

// Sum `count` floats at g over all ranks, in place, on stream st.
int comm_allreduce_f32(rgb_comm* c, float* g, size_t count, cudaStream_t st) {
  if (!c || count == 0) return RGB_OK;
  Nccl* n = nccl();
  if (!n) return cfail(RGB_ERR_CUDA, "NCCL not loaded");
  return nccl_rc(n->AllReduce(g, g, count, ncclFloat32, ncclSum, c->comm, st), "ncclAllReduce");
}

int comm_group(bool start) {
  Nccl* n = nccl();
  if (!n) return cfail(RGB_ERR_CUDA, "NCCL not loaded");
  return nccl_rc(start ? n->GroupStart() : n->GroupEnd(), start ? "ncclGroupStart" : "ncclGroupEnd");
}

}  // namespace rgb

extern "C" {

int rgb_comm_unique_id(void* id_out) {
  if (!id_out) return cfail(RGB_ERR_KERNEL, "null argument");
  Nccl* n = nccl();
  if (!n) return cfail(RGB_ERR_CUDA, "NCCL (libnccl.so.2) not found; set RGB_NCCL_LIB");
  ncclUniqueId id;
  int rc = nccl_rc(n->GetUniqueId(&id), "ncclGetUniqueId");
  if (rc) return rc;
  std::memcpy(id_out, &id, sizeof id);
  return RGB_OK;
}

int rgb_comm_init(const void* id_in, int nranks, int rank, rgb_comm** out) {
  if (!id_in || !out) return cfail(RGB_ERR_KERNEL, "null argument");
  if (nranks < 1 || rank < 0 || rank >= nranks) return cfail(RGB_ERR_KERNEL, "rank %d outside [0, %d)", rank, nranks);
  *out = nullptr;
  Nccl* n = nccl();
  if (!n) return cfail(RGB_ERR_CUDA, "NCCL (libnccl.so.2) not found; set RGB_NCCL_LIB");
  ncclUniqueId id;
  std::memcpy(&id, id_in, sizeof id);
  rgb_comm* c = new rgb_comm();
  c->nranks = nranks;
  c->rank = rank;
  int rc = nccl_rc(n->CommInitRank(&c->comm, nranks, id, rank), "ncclCommInitRank");
  if (rc) {
    delete c;
    return rc;
  }
  *out = c;
  return RGB_OK;
}

int rgb_comm_destroy(rgb_comm* c) {
  if (!c) return RGB_OK;
  Nccl* n = nccl();
  int rc = RGB_OK;
  if (n && c->comm) rc = nccl_rc(n->CommDestroy(c->comm), "ncclCommDestroy");
  delete c;
  return rc;
}

int rgb_comm_size(const rgb_comm* c, int* nranks, int* rank) {
  if (!c || !nranks || !rank) return cfail(RGB_ERR_KERNEL, "null argument");
  *nranks = c->nranks;
  *rank = c->rank;
  return RGB_OK;
}

int rgb_allreduce_grads(rgb_comm* c, float* g, int64_t n, void* stream) {
  if (!c || (!g && n > 0) || n < 0) return cfail(RGB_ERR_KERNEL, "bad arguments");
  return rgb::comm_allreduce_f32(c, g, (size_t)n, reinterpret_cast<cudaStream_t>(stream));
}

int rgb_allreduce_f64(rgb_comm* c, double* v, int64_t n, int op_max, void* stream) {
  if (!c || (!v && n > 0) || n < 0) return cfail(RGB_ERR_KERNEL, "bad arguments");
  Nccl* nc = nccl();
  if (!nc) return cfail(RGB_ERR_CUDA, "NCCL not loaded");
  return nccl_rc(nc->AllReduce(v, v, (size_t)n, ncclFloat64, op_max ? ncclMax : ncclSum, c->comm,
                               reinterpret_cast<cudaStream_t>(stream)),
                 "ncclAllReduce");
}

}  // extern "C"
