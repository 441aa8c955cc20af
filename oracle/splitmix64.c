/*
 * ORACLE — test infrastructure only; never linked into the product.
 *
 * C restatement of the reference generator kvweaver/rng.py:18-61
 * (next_u64 31-36, uniform 38-40, below 42-46) and of the toy weight draw
 * -0.1 + 0.2 * uniform() (kvweaver/backend.py:249-254).  Built by
 * oracle/Makefile into oracle/_build/liboracle_splitmix.so; tests check it
 * against the golden vectors of tests/test_rng.py in the reference
 * (seed 0: 0xE220A8397B1DCDAF ...).
 */
#include <stdint.h>

static const uint64_t GAMMA = 0x9E3779B97F4A7C15ULL;

static uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

/* sequential stream: n outputs of SplitMix64(seed).next_u64() */
void oracle_splitmix_u64(uint64_t seed, int64_t n, uint64_t *out) {
  uint64_t s = seed;
  for (int64_t i = 0; i < n; ++i) {
    s += GAMMA;
    out[i] = mix(s);
  }
}

/* weights: draws [start, start+n) mapped to [-0.1, 0.1) the reference way */
void oracle_toy_weights(uint64_t seed, int64_t start, int64_t n, double *out) {
  uint64_t s = seed + (uint64_t)start * GAMMA;
  for (int64_t i = 0; i < n; ++i) {
    s += GAMMA;
    volatile double u = (double)(mix(s) >> 11) * (1.0 / 9007199254740992.0);
    volatile double scaled = 0.2 * u;
    out[i] = -0.1 + scaled;
  }
}

/* below(n) draws: modulo reduction */
void oracle_splitmix_below(uint64_t seed, uint64_t bound, int64_t n, uint64_t *out) {
  uint64_t s = seed;
  for (int64_t i = 0; i < n; ++i) {
    s += GAMMA;
    out[i] = mix(s) % bound;
  }
}
