// collectives.cu — run-time NCCL loader (see collectives.h).
#include "collectives.h"

#include <dlfcn.h>

#include <mutex>
#include <string>

namespace itercur_b200 {
namespace {
NcclApi g_api{};
bool g_ok = false;
std::string g_err = "not loaded";
std::once_flag g_once;

template <class F>
bool sym(void* h, const char* name, F& out) {
  out = reinterpret_cast<F>(dlsym(h, name));
  if (!out) g_err = std::string("libnccl.so.2 lacks ") + name;
  return out != nullptr;
}

void load() {
  // an NCCL already in the process (torch.distributed's) first, then the loader's search path
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    const char* e = dlerror();
    g_err = std::string("cannot load libnccl.so.2: ") + (e ? e : "unknown");
    return;
  }
  g_ok = sym(h, "ncclAllReduce", g_api.AllReduce) && sym(h, "ncclAllGather", g_api.AllGather) &&
         sym(h, "ncclGroupStart", g_api.GroupStart) && sym(h, "ncclGroupEnd", g_api.GroupEnd) &&
         sym(h, "ncclGetUniqueId", g_api.GetUniqueId) && sym(h, "ncclCommInitRank", g_api.CommInitRank) &&
         sym(h, "ncclCommDestroy", g_api.CommDestroy) && sym(h, "ncclCommCount", g_api.CommCount) &&
         sym(h, "ncclCommUserRank", g_api.CommUserRank) && sym(h, "ncclGetErrorString", g_api.GetErrorString);
  if (g_ok) g_err.clear();
}
}  // namespace

const NcclApi* nccl_api() {
  std::call_once(g_once, load);
  return g_ok ? &g_api : nullptr;
}
const char* nccl_load_error() {
  std::call_once(g_once, load);
  return g_err.c_str();
}

}  // namespace itercur_b200
