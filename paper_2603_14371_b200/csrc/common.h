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

// The ABI does not trust caller block tables: every id a call will touch must
// lie inside the pool it was created with (OXY_EINVAL otherwise).
inline void check_block_ids(const int32_t *b, int64_t n, int32_t pool_blocks, const char *what) {
  for (int64_t i = 0; i < n; ++i)
    if (b[i] < 0 || b[i] >= pool_blocks) fail(OXY_EINVAL, "%s: block id %d outside pool of %d", what, b[i], pool_blocks);
}
// copy-on-write triples (src, dst, slots) per row: -1 / -1 / 0 when none
inline void check_cow(const int32_t *cow, int32_t rows, int32_t pool_blocks, int32_t block_size) {
  for (int32_t r = 0; r < rows; ++r) {
    const int32_t s = cow[3 * r], d = cow[3 * r + 1], n = cow[3 * r + 2];
    if (s < 0 && d < 0) continue;
    if (s < 0 || s >= pool_blocks || d < 0 || d >= pool_blocks || n < 0 || n > block_size)
      fail(OXY_EINVAL, "copy-on-write triple (%d, %d, %d) of row %d outside pool of %d", s, d, n, r, pool_blocks);
  }
}

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
