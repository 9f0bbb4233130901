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

}  // namespace wsync
