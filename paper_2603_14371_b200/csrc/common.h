// Shared error plumbing for the C ABI.
#pragma once

#include <cstdarg>
#include <cstdio>
#include <stdexcept>
#include <string>

#include "../../include/oxygen_b200.h"

namespace oxy {

void set_error(const char *fmt, ...);

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] void fail(int code, const char *fmt, ...);

}  // namespace oxy

// Wrap an ABI body: exceptions become status codes + oxy_last_error().
#define OXY_API_BEGIN try {
#define OXY_API_END                                   \
  return OXY_OK;                                      \
  }                                                   \
  catch (const oxy::Error &e) {                       \
    oxy::set_error("%s", e.what());                   \
    return e.code;                                    \
  }                                                   \
  catch (const std::exception &e) {                   \
    oxy::set_error("internal error: %s", e.what());   \
    return OXY_ESTATE;                                \
  }

#define OXY_REQUIRE(cond, ...) \
  do {                         \
    if (!(cond)) oxy::fail(OXY_EINVAL, __VA_ARGS__); \
  } while (0)
