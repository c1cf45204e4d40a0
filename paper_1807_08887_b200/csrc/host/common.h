// Host-side shared declarations for libtofu (C++17).
#pragma once
#include <cstdint>
#include <stdexcept>
#include <string>

#include "tofu.h"

namespace tofu {

// Thrown inside the library, converted to an error code at the C boundary.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void set_error(const std::string& msg);
int fail(int code, const std::string& msg);

// Write `s` into a caller buffer (cap bytes) with NUL; always report len.
int write_out(const std::string& s, char* out, size_t cap, size_t* len);

template <class F>
int guard(F&& f) {
  try {
    return f();
  } catch (const Error& e) {
    return fail(e.code, e.what());
  } catch (const std::exception& e) {
    return fail(TOFU_ERR_ARG, e.what());
  }
}

}  // namespace tofu
