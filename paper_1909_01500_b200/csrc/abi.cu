// ABI helpers: version, error strings, launch counter (include/rpl.h).
#include "common.cuh"

#include <stdlib.h>
#include <string.h>

namespace rpl {
std::atomic<int64_t> g_launches{0};

bool pdl_enabled() {
  static const bool on = [] {
    const char* v = getenv("RPL_PDL");
    return !(v && strcmp(v, "0") == 0);
  }();
  return on;
}
}

extern "C" const char* rpl_strerror(int status) {
  switch (status) {
    case RPL_OK: return "ok";
    case RPL_EINVAL: return "invalid argument (null pointer, bad shape or parameter)";
    case RPL_ERANGE: return "argument out of range";
    case RPL_EEMPTY: return "empty";
    case RPL_ECUDA: return "CUDA launch or runtime failure";
    case RPL_EUNSUPPORTED: return "unsupported configuration";
    default: return "unknown status";
  }
}

extern "C" int rpl_abi_version(void) { return RPL_ABI_VERSION; }

extern "C" int64_t rpl_launch_count(void) { return rpl::g_launches.load(); }
