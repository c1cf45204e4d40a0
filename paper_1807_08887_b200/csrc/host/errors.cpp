#include <cstring>

#include "common.h"

namespace tofu {
static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
int write_out(const std::string& s, char* out, size_t cap, size_t* len) {
  if (len) *len = s.size();
  if (!out || cap < s.size() + 1) return out ? fail(TOFU_ERR_SPACE, "output buffer too small") : TOFU_OK;
  std::memcpy(out, s.data(), s.size());
  out[s.size()] = 0;
  return TOFU_OK;
}
}  // namespace tofu

extern "C" const char* tofu_last_error(void) { return tofu::g_err.c_str(); }
extern "C" const char* tofu_version(void) { return "libtofu 0.1 (sm_100a)"; }
