// ABI helpers: version, error strings, launch counter (include/rpl.h).
#include "common.cuh"

#include <stdio.h>
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
int carveout_knob() {
  static const int c = [] {
    const char* v = getenv("RPL_CARVEOUT");
    if (!v) return -1;
    const int x = atoi(v);
    return (x < 0 || x > 100) ? -1 : x;
  }();
  return c;
}
void cfg_tree(int* stage_on, int* upd_threads, int* sample_warps, int* stage_words, int* hash_slots);
void cfg_scan(int* variant, int* trigger);
void cfg_gather(int* variant, int* diag, int* diag_build, int* seq_consumers, int* trans_consumers, int* slot_kb,
                int* g_threads);
}  // namespace rpl

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

extern "C" int rpl_config(char* buf, int64_t len) {
  if (!buf || len < 1) return RPL_EINVAL;
  int st, ut, sw, sword, hs, sv, strig, gv, gd, gdb, sc, tc, skb, gt;
  rpl::cfg_tree(&st, &ut, &sw, &sword, &hs);
  rpl::cfg_scan(&sv, &strig);
  rpl::cfg_gather(&gv, &gd, &gdb, &sc, &tc, &skb, &gt);
  const int w = snprintf(buf, (size_t)len,
                         "{\"abi\": %d, \"pdl\": %d, \"pdl_early\": %d, \"tree_stage\": %d, \"upd_threads\": %d, "
                         "\"sample_warps\": %d, \"stage_words\": %d, \"hash_slots\": %d, \"scan_variant\": %d, "
                         "\"scan_trigger\": %d, \"gather_variant\": %d, \"gather_diag\": %d, \"diag_build\": %d, "
                         "\"seq_consumers\": %d, \"trans_consumers\": %d, \"seq_slot_kb\": %d, \"g_threads\": %d, "
                         "\"carveout\": %d}",
                         RPL_ABI_VERSION, rpl::pdl_enabled() ? 1 : 0, (int)RPL_PDL_EARLY, st, ut, sw, sword, hs, sv,
                         strig, gv, gd, gdb, sc, tc, skb, gt, rpl::carveout_knob());
  return (w < 0 || w >= len) ? RPL_ERANGE : RPL_OK;
}
