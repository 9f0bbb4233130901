// exchange.cu -- cross-GPU route of the engine (K3 over NVLink).
#include "capi_util.h"
#include "engine.h"

using namespace wsync;

struct ws_engine::Comm {};

ws_status ws_engine::init_comm(const uint8_t* unique_id) {
  (void)unique_id;
  if (plan_.world() > 1) return set_error(WS_INVALID_ARGUMENT, "multi-GPU exchange not built yet");
  return WS_OK;
}

void ws_engine::destroy_comm() { delete comm_; comm_ = nullptr; }

ws_status ws_engine::exchange(const ws_sync_options&, int, cudaStream_t, uint32_t*) {
  return set_error(WS_INVALID_ARGUMENT, "multi-GPU exchange not built yet");
}

extern "C" ws_status ws_nccl_unique_id(uint8_t out[128]) {
  (void)out;
  return set_error(WS_NCCL, "NCCL not built yet");
}
