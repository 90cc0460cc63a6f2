/* mc5gen.c -- the config-5 Monte-Carlo trace recipe (workloads/mc5.py) in C,
 * for host-side parity at full size (all 1M traces vs the oracle).
 *
 * Input generation only: no allocator arithmetic. It implements exactly the
 * recipe documented in workloads/mc5.py (and tested against its numpy form,
 * tests/test_mc5_cpu.py):
 *   c(j)   = j <= n-2 and splitmix64(seed + j + 1) < threshold
 *   swap at j iff c(j) and not c(j-1) and id(j) != id(j+1)
 *   event  = (fixed + per * b, tag) of the source position.
 * Shared by nothing but this generator; the oracle (oracle/) and the CUDA
 * expander (K4) are separate implementations of their own parts.
 */
#include <stdint.h>

static inline uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* Writes trace t (template tpl[t], batch size b[t], seed seed[t]) to
 * out_bytes/out_tag at out_off[t]. Returns 0, or -1 if an output span does not
 * match its template's length. */
int mc5_instantiate(const int64_t* fixed, const int64_t* per, const uint32_t* tag,
                    const int64_t* tpl_off, const uint32_t* tpl, const uint32_t* b,
                    const uint64_t* seed, int64_t n_traces, uint64_t threshold,
                    const int64_t* out_off, int64_t* out_bytes, uint32_t* out_tag) {
  for (int64_t t = 0; t < n_traces; ++t) {
    const int64_t base = tpl_off[tpl[t]];
    const int64_t n = tpl_off[tpl[t] + 1] - base;
    if (out_off[t + 1] - out_off[t] != n) return -1;
    const int64_t bs = (int64_t)b[t];
    int64_t* ob = out_bytes + out_off[t];
    uint32_t* ot = out_tag + out_off[t];
    int c_prev = 0;
    int64_t j = 0;
    while (j < n) {
      const int cj = j < n - 1 && splitmix64(seed[t] + (uint64_t)j + 1u) < threshold;
      const int swap = cj && !c_prev &&
                       (tag[base + j] & 0x0FFFFFFFu) != (tag[base + j + 1] & 0x0FFFFFFFu);
      if (swap) {
        ob[j] = fixed[base + j + 1] + per[base + j + 1] * bs;
        ot[j] = tag[base + j + 1];
        ob[j + 1] = fixed[base + j] + per[base + j] * bs;
        ot[j + 1] = tag[base + j];
        /* c(j+1) is needed for position j+2 */
        c_prev = j + 1 < n - 1 && splitmix64(seed[t] + (uint64_t)j + 2u) < threshold;
        j += 2;
      } else {
        ob[j] = fixed[base + j] + per[base + j] * bs;
        ot[j] = tag[base + j];
        c_prev = cj;
        j += 1;
      }
    }
  }
  return 0;
}
