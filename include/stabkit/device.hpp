// stabkit/device.hpp -- process-wide device context for the stabkit:: host classes.
// One sk_ctx (stabkit_b200.h) per process, created on first use on device STABKIT_DEVICE
// (default 0).  If no CUDA device is usable construction throws stabkit::Error: the host API
// has no CPU fallback for tableau / grouping / transpiler work.
#pragma once
#include <cstdlib>
#include <string>

#include "stabkit/error.hpp"
#include "stabkit_b200.h"

namespace stabkit {

class Device {
  public:
    static Device& instance() { static Device d; return d; }
    sk_ctx* ctx() const { return ctx_; }
    void check(int code) const { if (code != SK_OK) throw_status(code, sk_last_error(ctx_)); }
    void sync() const { check(sk_ctx_sync(ctx_)); }
    sk_counters counters() const { sk_counters c{}; check(sk_get_counters(ctx_, &c)); return c; }
    Device(const Device&) = delete;
    Device& operator=(const Device&) = delete;

  private:
    Device() {
        const char* env = std::getenv("STABKIT_DEVICE");
        const int ordinal = env ? std::atoi(env) : 0;
        if (sk_ctx_create(ordinal, nullptr, &ctx_) != SK_OK)
            throw Error("stabkit: no usable CUDA device " + std::to_string(ordinal) + " (the B200 engine has no CPU fallback)");
    }
    ~Device() { sk_ctx_destroy(ctx_); }
    sk_ctx* ctx_ = nullptr;
};

}  // namespace stabkit
