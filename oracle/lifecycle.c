/*
 * oracle/lifecycle.c -- ORACLE. TEST INFRASTRUCTURE ONLY (see oracle/xmo.c).
 *
 * Lifecycle reconstruction, the Analyzer step two before the Simulator
 * (SURVEY.md §8(f) NEXT-3): "It processes the event stream sequentially,
 * systematically pairing allocation and deallocation events based on address
 * tracking and timing to determine the size, CPU allocation time, and CPU
 * deallocation time for each distinct memory block while correctly handling
 * address reuse. Blocks lacking a deallocation event are considered
 * persistent for the trace duration." (§3.2), with SPEC.md's
 * reconstruct_blocks contract: an allocation (+bytes at
 * addr) opens a block; a deallocation (-bytes at addr) closes the most
 * recently opened still-open block at that address (D1, LIFO per address);
 * none open -> orphan free (tallied, SPEC D4); |bytes| != the block's size ->
 * mismatch (tallied; the block is closed with its own size). S:107's "whose
 * size matches" clause is read as in DESIGN.md Q22: the LIFO top closes
 * whatever its size (otherwise S:107's own mismatch clause could never fire).
 *
 * Plain sequential C: a per-address stack of open blocks (linked through the
 * alloc events' indices) found through an open-addressing hash map.
 *
 * Outputs for one trace of n instants in time order:
 *   partner[i]  alloc: index of the free that closes it, -1 = persistent;
 *               free: index of the alloc it closes, -1 = orphan
 *   mismatch[i] 1 on a free whose |bytes| differs from its block's size
 *   tallies[6]  n_blocks, n_orphan, n_mismatch, n_persistent, n_kept
 *               (= allocs + matched frees), max_open (most blocks open at once)
 * Returns 0, -1 for a zero-byte instant, -5 out of host memory.
 *
 * Parity status: pinned (tests/test_oracle_lifecycle.py: SPEC.md:109-111
 * examples, the conservation invariant SPEC.md:133, an O(n^2) brute force).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct { uint64_t addr; int64_t top; int32_t used; } LSlot;

int xmo_reconstruct(const uint64_t* addr, const int64_t* bytes, int64_t n, int64_t* partner,
                    uint8_t* mismatch, uint64_t* tallies) {
  memset(tallies, 0, 6 * sizeof(uint64_t));
  uint64_t cap = 16;
  while (cap < (uint64_t)(2 * n + 2)) cap *= 2;
  LSlot* map = (LSlot*)calloc(cap, sizeof(LSlot));
  int64_t* below = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
  if (!map || !below) { free(map); free(below); return -5; }
  uint64_t open = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (bytes[i] == 0) { free(map); free(below); return -1; }
    partner[i] = -1;
    mismatch[i] = 0;
    uint64_t h = (addr[i] * 0x9E3779B97F4A7C15ull) & (cap - 1);
    while (map[h].used && map[h].addr != addr[i]) h = (h + 1) & (cap - 1);
    LSlot* s = &map[h];
    if (bytes[i] > 0) {                       /* allocation: open a block, push it */
      if (!s->used) { s->used = 1; s->addr = addr[i]; s->top = -1; }
      below[i] = s->top;
      s->top = i;
      tallies[0] += 1;
      open += 1;
      if (open > tallies[5]) tallies[5] = open;
    } else if (!s->used || s->top < 0) {      /* nothing open at this address */
      tallies[1] += 1;
    } else {                                  /* close the most recent open block */
      int64_t b = s->top;
      s->top = below[b];
      partner[i] = b;
      partner[b] = i;
      if (bytes[b] != -bytes[i]) { mismatch[i] = 1; tallies[2] += 1; }
      open -= 1;
    }
  }
  tallies[3] = open;
  tallies[4] = tallies[0] + (tallies[0] - open);
  free(map);
  free(below);
  return 0;
}
