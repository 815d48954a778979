#include "runtime.hpp"

#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

#include "orchsim/errors.hpp"

namespace orchsim::b200 {

namespace {

struct ThreadContext {
  orch_ctx* ctx = nullptr;
  int device = -1;
  ~ThreadContext() {
    if (ctx) orch_ctx_destroy(ctx);
  }
};

thread_local ThreadContext g_tc;

}  // namespace

orch_ctx* context() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
  if (g_tc.ctx && g_tc.device == dev) return g_tc.ctx;
  if (g_tc.ctx) orch_ctx_destroy(g_tc.ctx);
  g_tc.ctx = nullptr;
  check(orch_ctx_create(dev, &g_tc.ctx));
  g_tc.device = dev;
  return g_tc.ctx;
}

void check(int code) {
  if (code == ORCH_OK) return;
  const std::string msg = orch_last_error();
  switch (code) {
    case ORCH_INVALID_ARGUMENT:
      throw std::invalid_argument(msg);
    case ORCH_CONFIG_ERROR:
      throw ConfigError(msg);
    case ORCH_SIZE_CAP:
      throw SizeCapError(msg);
    case ORCH_LOGIC_ERROR:
      throw std::logic_error(msg);
    default:
      throw std::runtime_error("orchsim B200 library error " + std::to_string(code) + ": " + msg);
  }
}

}  // namespace orchsim::b200
