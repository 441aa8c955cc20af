// Deterministic paged-KV block allocator (host side).
//
// The unified KV pool replaces the reference's per-request immutable numpy
// caches (kvweaver/kv_manager.py:35-105) while keeping their value semantics:
// a cache handle is (block ids, seq_len) and only ever reads positions
// [0, seq_len), so handles survive later decodes of the same state
// (kvweaver/verify.py:136-138, 195-205 decode one state twice).
//
// Rules (restated in oracle/paged_alloc.py, bit-exact parity tested):
//   * free blocks come from a min-heap: lowest id first;
//   * every block has a refcount and a fill watermark (slots claimed);
//   * appending at p with p % B != 0 writes in place iff fill[tail] == p % B,
//     otherwise the tail is copied-on-write into a fresh block;
//   * a block whose refcount drops to 0 is returned to the heap, fill = 0.
#include <algorithm>
#include <cstring>
#include <functional>
#include <queue>
#include <vector>

#include "common.h"

namespace oxy {

static thread_local std::string g_err;
unsigned long long g_launches = 0;
unsigned long long g_devbuf_reallocs = 0;

void set_error(const char *fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
}

void fail(int code, const char *fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  throw Error(code, buf);
}

}  // namespace oxy

struct oxy_alloc {
  int32_t num_blocks = 0, bs = 0;
  std::vector<int32_t> ref, fill;
  std::priority_queue<int32_t, std::vector<int32_t>, std::greater<int32_t>> heap;

  int32_t blocks_for(int64_t n) const { return (int32_t)((n + bs - 1) / bs); }

  int32_t take() {
    if (heap.empty()) oxy::fail(OXY_ENOBLOCKS, "KV pool out of blocks (%d in use)", num_blocks);
    int32_t b = heap.top();
    heap.pop();
    ref[b] = 1;
    fill[b] = 0;
    return b;
  }
  void check_id(int32_t b) const {
    if (b < 0 || b >= num_blocks) oxy::fail(OXY_EINVAL, "block id %d outside pool of %d", b, num_blocks);
    if (ref[b] <= 0) oxy::fail(OXY_ESTATE, "block %d is not allocated", b);
  }
  void decref(int32_t b) {
    check_id(b);
    if (--ref[b] == 0) {
      fill[b] = 0;
      heap.push(b);
    }
  }
};

extern "C" {

const char *oxy_last_error(void) { return oxy::g_err.c_str(); }
int oxy_abi_version(void) { return 1; }
int64_t oxy_launch_count(void) { return (int64_t)__atomic_load_n(&oxy::g_launches, __ATOMIC_RELAXED); }

int oxy_alloc_create(int32_t num_blocks, int32_t block_size, oxy_alloc **out) {
  OXY_API_BEGIN
  OXY_REQUIRE(num_blocks > 0 && block_size > 0, "pool needs positive num_blocks/block_size");
  auto *a = new oxy_alloc;
  a->num_blocks = num_blocks;
  a->bs = block_size;
  a->ref.assign(num_blocks, 0);
  a->fill.assign(num_blocks, 0);
  for (int32_t b = 0; b < num_blocks; ++b) a->heap.push(b);
  *out = a;
  OXY_API_END
}

int oxy_alloc_destroy(oxy_alloc *a) {
  delete a;
  return OXY_OK;
}

int oxy_alloc_seq(oxy_alloc *a, int32_t n_tokens, int32_t *blocks_h) {
  OXY_API_BEGIN
  OXY_REQUIRE(a != nullptr, "null allocator handle");
  OXY_REQUIRE(n_tokens >= 1, "sequence needs at least one position");
  int32_t nb = a->blocks_for(n_tokens);
  if ((int32_t)a->heap.size() < nb)
    oxy::fail(OXY_ENOBLOCKS, "KV pool out of blocks: need %d, %zu free", nb, a->heap.size());
  for (int32_t i = 0; i < nb; ++i) {
    int32_t b = a->take();
    a->fill[b] = std::min(a->bs, n_tokens - i * a->bs);
    blocks_h[i] = b;
  }
  OXY_API_END
}

int oxy_alloc_incref(oxy_alloc *a, const int32_t *blocks_h, int32_t n) {
  OXY_API_BEGIN
  OXY_REQUIRE(a != nullptr, "null allocator handle");
  for (int32_t i = 0; i < n; ++i) a->check_id(blocks_h[i]);
  for (int32_t i = 0; i < n; ++i) a->ref[blocks_h[i]]++;
  OXY_API_END
}

int oxy_alloc_decref(oxy_alloc *a, const int32_t *blocks_h, int32_t n) {
  OXY_API_BEGIN
  OXY_REQUIRE(a != nullptr, "null allocator handle");
  for (int32_t i = 0; i < n; ++i) a->decref(blocks_h[i]);
  OXY_API_END
}

int oxy_alloc_reserve(oxy_alloc *a, const int32_t *blocks_h, int32_t seq_len, int32_t n_new,
                      int32_t *new_blocks_h, int32_t *cow_h) {
  OXY_API_BEGIN
  OXY_REQUIRE(a != nullptr, "null allocator handle");
  OXY_REQUIRE(seq_len >= 1 && n_new >= 0, "reserve needs seq_len >= 1 and n_new >= 0");
  const int32_t bs = a->bs;
  const int32_t nb_old = a->blocks_for(seq_len);
  const int32_t nb_new = a->blocks_for((int64_t)seq_len + n_new);
  const int32_t off = seq_len % bs;
  for (int32_t i = 0; i < nb_old; ++i) a->check_id(blocks_h[i]);
  const int32_t tail = blocks_h[nb_old - 1];
  const bool cow = off != 0 && n_new > 0 && a->fill[tail] != off;
  if (off != 0 && a->fill[tail] < off)
    oxy::fail(OXY_ESTATE, "tail block %d holds %d slots, handle needs %d", tail, a->fill[tail], off);
  const int32_t need = (nb_new - nb_old) + (cow ? 1 : 0);
  if ((int32_t)a->heap.size() < need)
    oxy::fail(OXY_ENOBLOCKS, "KV pool out of blocks: need %d, %zu free", need, a->heap.size());

  for (int32_t i = 0; i < nb_old; ++i) {
    new_blocks_h[i] = blocks_h[i];
    a->ref[blocks_h[i]]++;
  }
  cow_h[0] = -1;
  cow_h[1] = -1;
  cow_h[2] = 0;
  if (off != 0 && n_new > 0) {
    int32_t dst = tail;
    if (cow) {
      dst = a->take();
      a->decref(tail);
      new_blocks_h[nb_old - 1] = dst;
      cow_h[0] = tail;
      cow_h[1] = dst;
      cow_h[2] = off;
    }
    a->fill[dst] = std::min(bs, off + n_new);  // claim the slots we may write
  }
  int64_t remaining = (int64_t)seq_len + n_new - (int64_t)nb_old * bs;
  for (int32_t i = nb_old; i < nb_new; ++i) {
    int32_t b = a->take();
    a->fill[b] = (int32_t)std::min<int64_t>(bs, remaining);
    remaining -= bs;
    new_blocks_h[i] = b;
  }
  OXY_API_END
}

int oxy_alloc_reserve_need(const oxy_alloc *a, const int32_t *blocks_h, int32_t seq_len, int32_t n_new,
                           int32_t *need) {
  OXY_API_BEGIN
  OXY_REQUIRE(a != nullptr && need != nullptr, "null allocator handle");
  OXY_REQUIRE(seq_len >= 1 && n_new >= 0, "reserve needs seq_len >= 1 and n_new >= 0");
  const int32_t nb_old = a->blocks_for(seq_len), off = seq_len % a->bs;
  const int32_t tail = blocks_h[nb_old - 1];
  a->check_id(tail);
  const bool cow = off != 0 && n_new > 0 && a->fill[tail] != off;
  *need = a->blocks_for((int64_t)seq_len + n_new) - nb_old + (cow ? 1 : 0);
  OXY_API_END
}

int oxy_alloc_settle(oxy_alloc *a, const int32_t *blocks_h, int32_t seq_len, int32_t n_reserved,
                     int32_t n_actual, int32_t *n_blocks_out) {
  OXY_API_BEGIN
  OXY_REQUIRE(a != nullptr, "null allocator handle");
  OXY_REQUIRE(n_actual >= 0 && n_actual <= n_reserved, "settle: n_actual %d outside [0, %d]",
              n_actual, n_reserved);
  const int32_t nb_res = a->blocks_for((int64_t)seq_len + n_reserved);
  const int32_t nb_act = a->blocks_for((int64_t)seq_len + n_actual);
  for (int32_t i = 0; i < nb_res; ++i) a->check_id(blocks_h[i]);
  for (int32_t i = nb_act; i < nb_res; ++i) a->decref(blocks_h[i]);
  if (n_actual < n_reserved) {
    const int32_t t = blocks_h[nb_act - 1];
    const int32_t nb_old = a->blocks_for(seq_len);
    if (nb_act - 1 >= nb_old - 1 && (nb_act > nb_old || seq_len % a->bs != 0))
      a->fill[t] = seq_len + n_actual - (nb_act - 1) * a->bs;
  }
  *n_blocks_out = nb_act;
  OXY_API_END
}

int oxy_alloc_num_free(const oxy_alloc *a, int32_t *out) {
  OXY_API_BEGIN
  OXY_REQUIRE(a != nullptr && out != nullptr, "null allocator handle");
  *out = (int32_t)a->heap.size();
  OXY_API_END
}

int oxy_alloc_snapshot(const oxy_alloc *a, int32_t *refcount_h, int32_t *fill_h, int32_t *free_h,
                       int32_t *n_free) {
  OXY_API_BEGIN
  OXY_REQUIRE(a != nullptr, "null allocator handle");
  std::memcpy(refcount_h, a->ref.data(), sizeof(int32_t) * a->num_blocks);
  std::memcpy(fill_h, a->fill.data(), sizeof(int32_t) * a->num_blocks);
  int32_t n = 0;
  for (int32_t b = 0; b < a->num_blocks; ++b)
    if (a->ref[b] == 0) free_h[n++] = b;
  *n_free = n;
  if (n != (int32_t)a->heap.size()) oxy::fail(OXY_ESTATE, "free list size %d != heap %zu", n, a->heap.size());
  OXY_API_END
}

int oxy_build_slot_mapping(const int32_t *blocks_h, int32_t block_size, int32_t start,
                           int32_t count, int32_t *slots_h) {
  OXY_API_BEGIN
  OXY_REQUIRE(block_size > 0 && start >= 0 && count >= 0, "bad slot-mapping arguments");
  for (int32_t i = 0; i < count; ++i) {
    int32_t p = start + i;
    slots_h[i] = blocks_h[p / block_size] * block_size + p % block_size;
  }
  OXY_API_END
}

}  // extern "C"
