// nccl_dl.cpp -- minimal run-time binding of the NCCL entry points libciq uses.
#include "nccl_dl.h"

#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <string>

namespace ciq {
namespace {

typedef int (*GetUniqueId_t)(void*);
struct Id128 { char b[128]; };
typedef int (*CommInitRankV_t)(void**, int, Id128, int);
typedef int (*CommDestroy_t)(void*);
typedef int (*AllGather_t)(const void*, void*, size_t, int, void*, cudaStream_t);
typedef int (*AllReduce_t)(const void*, void*, size_t, int, int, void*, cudaStream_t);
typedef const char* (*GetErrorString_t)(int);

struct Nccl {
  void* h = nullptr;
  GetUniqueId_t get_unique_id = nullptr;
  CommInitRankV_t comm_init_rank = nullptr;
  CommDestroy_t comm_destroy = nullptr;
  AllGather_t all_gather = nullptr;
  AllReduce_t all_reduce = nullptr;
  GetErrorString_t err = nullptr;
  std::string last = "NCCL not loaded";
} g;
std::once_flag g_once;

void do_load() {
  const char* names[] = {"libnccl.so.2", "libnccl.so",
                         "/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/lib/libnccl.so.2"};
  for (const char* n : names) {
    g.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
    if (g.h) break;
  }
  if (!g.h) { g.last = std::string("dlopen(libnccl.so.2) failed: ") + dlerror(); return; }
  g.get_unique_id = (GetUniqueId_t)dlsym(g.h, "ncclGetUniqueId");
  g.comm_init_rank = (CommInitRankV_t)dlsym(g.h, "ncclCommInitRank");
  g.comm_destroy = (CommDestroy_t)dlsym(g.h, "ncclCommDestroy");
  g.all_gather = (AllGather_t)dlsym(g.h, "ncclAllGather");
  g.all_reduce = (AllReduce_t)dlsym(g.h, "ncclAllReduce");
  g.err = (GetErrorString_t)dlsym(g.h, "ncclGetErrorString");
  if (!g.get_unique_id || !g.comm_init_rank || !g.all_gather || !g.all_reduce || !g.comm_destroy) {
    g.last = "libnccl.so.2 lacks required symbols";
    g.h = nullptr;
    return;
  }
  g.last = "";
}

bool check(int r) {
  if (r == 0) return true;
  g.last = g.err ? g.err(r) : "NCCL error";
  return false;
}

}  // namespace

bool nccl_load() {
  std::call_once(g_once, do_load);
  return g.h != nullptr;
}
const char* nccl_error() { return g.last.c_str(); }

bool nccl_unique_id(void* out128) {
  if (!nccl_load()) return false;
  return check(g.get_unique_id(out128));
}

void* nccl_comm_init(int world, int rank, const void* id128) {
  if (!nccl_load()) return nullptr;
  Id128 id;
  std::memcpy(id.b, id128, 128);
  void* comm = nullptr;
  if (!check(g.comm_init_rank(&comm, world, id, rank))) return nullptr;
  return comm;
}

void nccl_comm_destroy(void* comm) {
  if (comm && g.comm_destroy) g.comm_destroy(comm);
}

bool nccl_allgather(const void* send, void* recv, size_t count, int dtype, void* comm, cudaStream_t s) {
  return check(g.all_gather(send, recv, count, dtype, comm, s));
}

bool nccl_allreduce_sum(const void* send, void* recv, size_t count, int dtype, void* comm, cudaStream_t s) {
  return check(g.all_reduce(send, recv, count, dtype, /*ncclSum*/ 0, comm, s));
}

}  // namespace ciq
