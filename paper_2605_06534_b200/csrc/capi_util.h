// capi_util.h -- error plumbing shared by the C-ABI translation units.
#pragma once

#include <cuda_runtime.h>

#include <string>

#include "wsync.h"

namespace wsync {

ws_status set_error(ws_status s, const std::string& msg);
ws_status cuda_status(cudaError_t e, const char* what);
bool valid_dtype(int dt);
ws_status check_shard(const int64_t* full, int nd, const ws_shard& d, const char* what);
uint64_t shard_elems(const int64_t* full, int nd, const ws_shard& d);

// Entry points that switch to an engine's GPU restore the caller's current
// device on return (a process may drive several GPUs).
struct DeviceGuard {
  int prev = 0;
  DeviceGuard() { cudaGetDevice(&prev); }
  ~DeviceGuard() { cudaSetDevice(prev); }
};

}  // namespace wsync
