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

extern "C" int rpl_peer_access(int32_t peer) {
  int cur = 0, n = 0;
  if (cudaGetDevice(&cur) != cudaSuccess || cudaGetDeviceCount(&n) != cudaSuccess) return RPL_ECUDA;
  if (peer < 0 || peer >= n) return RPL_EINVAL;
  if (peer == cur) return RPL_OK;
  int can = 0;
  if (cudaDeviceCanAccessPeer(&can, cur, peer) != cudaSuccess) return RPL_ECUDA;
  if (!can) return RPL_EUNSUPPORTED;
  const cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    (void)cudaGetLastError();  // clear the sticky-free status the call left
    return RPL_OK;
  }
  return e == cudaSuccess ? RPL_OK : RPL_ECUDA;
}
