// relay_shim.hpp -- binds any reference Relay (relay.hpp:27-35: MemoryRelay,
// ThrottledRelay, the TCP relay client a RelayFactory returns) to the ws_relay
// callbacks of ws_engine_sync_relay (include/wsync.h).  Header-only; compile
// it into the reference side next to codec_shim.cpp.
//
//   coserve::transfer::MemoryRelay relay;
//   ws_relay r = wsync_shim::bind_relay(relay);
//   ws_engine_sync_relay(engine, step, &opts, &relay_opts, &r, &report);
#pragma once

#include <cstring>
#include <string>
#include <vector>

#include "coserve/transfer/relay.hpp"
#include "wsync.h"

namespace wsync_shim {

inline int relay_put(void* ctx, const char* key, uint64_t key_len, const uint8_t* data,
                     uint64_t len) {
  try {
    static_cast<coserve::transfer::Relay*>(ctx)->put(std::string(key, key_len),
                                                     std::vector<uint8_t>(data, data + len));
    return 0;
  } catch (...) {
    return -2;
  }
}

inline int64_t relay_get_any(void* ctx, const char* const* keys, const uint64_t* key_lens, int n,
                             int timeout_ms, int* hit, uint8_t* out, uint64_t cap) {
  try {
    std::vector<std::string> ks;
    for (int i = 0; i < n; ++i) ks.emplace_back(keys[i], key_lens[i]);
    auto kv = static_cast<coserve::transfer::Relay*>(ctx)->get_any(ks, timeout_ms);
    for (int i = 0; i < n; ++i)
      if (ks[i] == kv.first) *hit = i;
    if (kv.second.size() <= cap) std::memcpy(out, kv.second.data(), kv.second.size());
    return static_cast<int64_t>(kv.second.size());
  } catch (const coserve::transfer::RelayTimeout&) {
    return -1;
  } catch (...) {
    return -2;
  }
}

inline ws_relay bind_relay(coserve::transfer::Relay& relay) {
  ws_relay r{};  // no framed transport: the Relay frames (or not) itself
  r.ctx = &relay;
  r.put = &relay_put;
  r.get_any = &relay_get_any;
  return r;
}

}  // namespace wsync_shim
