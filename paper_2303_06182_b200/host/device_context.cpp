#include "device_context.hpp"

#include <stdexcept>

namespace moesim::detail {

namespace {
moe_ctx* g_ctx = nullptr;
}

std::mutex& context_mutex() {
  static std::mutex mu;
  return mu;
}

moe_ctx* context_locked() {
  if (!g_ctx) {
    const int st = moe_ctx_create(0, &g_ctx);
    if (st != MOE_OK) {
      g_ctx = nullptr;
      throw std::runtime_error(std::string("moesim: no usable B200 (") + moe_last_error() + ")");
    }
  }
  return g_ctx;
}

void rethrow(int status) {
  const std::string msg = moe_last_error();
  if (status == MOE_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  throw std::runtime_error("moesim: " + msg);
}

}  // namespace moesim::detail
