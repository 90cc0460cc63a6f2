/*
 * oracle/xmo.c -- ORACLE. TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, single-threaded CPU re-statement of xMem's Simulator
 * (§3.4) with the caching-allocator rules the paper defers
 * to ("The segment's allocation strategy follows the PyTorch Official
 * implementation", PAPER.md:257 footnote) and SPEC.md's allocator_sim module
 * (SPEC.md:205-294).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this file.  It shares no code,
 * header, table or constant with paper_2510_21048_b200/ (the CUDA product),
 * and nothing here is derived from that path.
 *
 * Data structures are the obvious ones: an arena of blocks with explicit
 * address-order prev/next links inside each segment (SPEC.md:214 Segment,
 * "blocks tile the segment exactly"), an UNORDERED array of free blocks that
 * every allocation scans linearly for the best fit ("free-block
 * index ... ordered by size then address" -- a linear min-scan is the plain
 * definition of the first element of that order), and a hash map from block
 * id to block.  Addresses come from a bump pointer that is never reused
 * (reading Q4), so (size, addr) order == SPEC D2's
 * (size, segment_id, offset) order.
 *
 * Readings of the paper taken here (all listed in DESIGN.md §Readings):
 *   Q1 large-pool split iff remainder > small_size (torch strict), configurable
 *   Q2 both "allocated" definitions are reported
 *   Q3 reclamation releases every whole-segment free block, retries once
 *   Q5 per-stream pools: stream is an exact-match filter
 *   Q6 array order is replay order, Q7 first index reaching a peak
 *   Q9 OOM stops the trace; Q10 refuse iff reserved + size > capacity
 *   Q19, Q20, Q26, Q27 allocator variants (NEXT-4), off by default
 *
 * Parity status: every function below is pinned by tests/test_oracle_*.py
 * (SPEC worked examples, paper examples, closed forms H1-H7, invariants
 * after every event, and an independent gap-model brute force).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---- error codes (call-level contract violations) ---- */
#define XMO_E_ZERO      (-1)  /* zero-byte request ("zero request -> contract violation") */
#define XMO_E_DUP       (-2)  /* alloc of an id that is live */
#define XMO_E_NOTLIVE   (-3)  /* free of an id that is not live */
#define XMO_E_SIZE      (-4)  /* free whose |bytes| differs from the alloc's request */
#define XMO_E_NOMEM     (-5)  /* host malloc failed */
#define XMO_E_INVARIANT (-6)  /* invariant check failed (check mode only) */

/* ---- per-trace status (a result, not an error: SPEC.md:284 D4) ---- */
#define XMO_T_OK  0
#define XMO_T_OOM 1

/* ---- output record: XMO_NF uint64 fields per trace (names in oracle/__init__.py) ---- */
enum {
  F_PEAK_ALLOC = 0, F_PEAK_ALLOC_IDX, F_PEAK_BLK, F_PEAK_BLK_IDX, F_PEAK_RES, F_PEAK_RES_IDX,
  F_FINAL_RES, F_NSEG_ALLOC, F_NSEG_RELEASE, F_MAX_LIVE_SEG, F_EVENTS_DONE, F_STATUS,
  F_NFREE_END, F_FINAL_ALLOC, F_FINAL_BLK, XMO_NF
};

typedef struct {
  uint64_t min_block;        /* 512      PAPER.md:154, 256 (i) "multiple of 512 bytes" */
  uint64_t small_size;       /* 1 MiB    small-pool threshold (SPEC.md:210 small_alloc_threshold) */
  uint64_t small_buffer;     /* 2 MiB    PAPER.md:169 "requesting 2MB for a 1MB tensor" */
  uint64_t large_buffer;     /* 20 MiB   PAPER.md:654 "a 20MB block for a 10MB tensor" */
  uint64_t min_large_alloc;  /* 10 MiB   SPEC.md:211 min_large_alloc */
  uint64_t round_large;      /* 2 MiB    SPEC.md:211 large_round */
  uint64_t capacity;         /* device capacity; UINT64_MAX = unlimited */
  int32_t  large_split_strict; /* 1: split iff rem > small_size (torch); 0: rem >= */
  int32_t  roundup_power2_divisions; /* NEXT-4 variant: torch PYTORCH_CUDA_ALLOC_CONF          */
                                     /* roundup_power2_divisions:N (uniform N); 0/1 = off      */
  int32_t  reclaim_policy;           /* 0: torch release all cached segments (reading Q3);     */
                                     /* 1: SPEC.md:283 D3 largest first until capacity suffices */
  int32_t  _pad;
  /* NEXT-4 variants, torch PYTORCH_CUDA_ALLOC_CONF knobs (PAPER.md:257 defers to
   * the PyTorch allocator; readings Q26, Q27):                                  */
  uint64_t max_split_size;           /* max_split_size_mb:N -> N MiB; UINT64_MAX = off  */
  uint64_t max_non_split_rounding;   /* max_non_split_rounding_mb (default 20 MiB)      */
  double   gc_threshold;             /* garbage_collection_threshold:x, 0 = off; acts   */
                                     /* only with a finite capacity ("set_fraction")     */
} xmo_config;

/* ------------------------------------------------------------------------ */
/* The three sizing rules, written out.                                      */
/* ------------------------------------------------------------------------ */

/* SPEC.md:227-235 round_size: smallest multiple of min_block >= request.
 * PAPER.md:256 (i) "rounded up to the nearest hardware-required multiple". */
uint64_t xmo_round_size(uint64_t request, const xmo_config* c) {
  /* Variant (reading Q15): torch's roundup_power2_divisions:N.
   * A request above min_block * N is rounded up to the next multiple of
   * 2^k / N, where 2^k is the largest power of two <= the request (N equal
   * divisions of [2^k, 2^(k+1))); a power of two is kept as is. */
  uint64_t div = c->roundup_power2_divisions > 1 ? (uint64_t)c->roundup_power2_divisions : 0;
  if (div && request > c->min_block * div) {
    uint64_t p2 = 1;
    while (p2 <= request / 2) p2 *= 2;
    if (p2 == request) return request;
    uint64_t step = p2 / div;
    uint64_t k = request / step;
    if (k * step < request) k += 1;
    return k * step;
  }
  uint64_t q = request / c->min_block;
  if (q * c->min_block < request) q += 1;
  if (q == 0) q = 1;
  return q * c->min_block;
}

/* Pool choice: small pool iff rounded size <= small_size. */
int xmo_is_small(uint64_t s, const xmo_config* c) { return s <= c->small_size; }

/* SPEC.md:236-244 segment_size_for; PAPER.md:257 (ii), 169, 654. */
uint64_t xmo_segment_size(uint64_t s, const xmo_config* c) {
  if (s <= c->small_size) return c->small_buffer;
  if (s < c->min_large_alloc) return c->large_buffer;
  uint64_t q = s / c->round_large;
  if (q * c->round_large < s) q += 1;
  return q * c->round_large;
}

/* Split rule (PAPER.md:258 (iii) "splitting blocks when an exact match is
 * unavailable"; reading Q1). */
int xmo_should_split(int small_pool, uint64_t remaining, const xmo_config* c) {
  if (small_pool) return remaining >= c->min_block;
  if (c->large_split_strict) return remaining > c->small_size;
  return remaining >= c->small_size;
}

/* ------------------------------------------------------------------------ */
/* Simulator state                                                           */
/* ------------------------------------------------------------------------ */
typedef struct {
  uint64_t addr, size;
  int64_t prev, next;   /* address-order neighbours in the same segment, -1 = none */
  int64_t seg;
  int32_t stream, small, allocated, alive;
  uint64_t gc_base;     /* its pool's free-block-search count when it entered the free index */
} Block;

typedef struct {
  uint64_t base, size;
  int32_t stream, small, alive, _pad;
} Segment;

typedef struct { uint32_t id; int32_t used; int64_t block; uint64_t request; } Slot;

typedef struct {
  Block* blk; int64_t nblk, capblk;
  Segment* seg; int64_t nseg, capseg;
  int64_t* fr; int64_t nfr, capfr;     /* unordered free-block index */
  Slot* map; uint64_t mapcap;          /* open-addressing hash: id -> live block */
  uint64_t next_base;
  uint64_t reserved, alloc_blk, alloc_tensor;
  int64_t live_segs;
  uint64_t searches[2];                /* free-block searches per pool [large, small] (GC ages) */
} State;

static int grow(void** p, int64_t* cap, int64_t need, size_t elem) {
  if (need <= *cap) return 0;
  int64_t nc = *cap ? *cap : 16;
  while (nc < need) nc *= 2;
  void* q = realloc(*p, (size_t)nc * elem);
  if (!q) return XMO_E_NOMEM;
  *p = q; *cap = nc;
  return 0;
}

static Slot* map_find(State* S, uint32_t id, int insert) {
  uint64_t h = ((uint64_t)id * 0x9E3779B97F4A7C15ull) & (S->mapcap - 1);
  for (;;) {
    Slot* s = &S->map[h];
    if (!s->used) {
      if (!insert) return NULL;
      s->used = 1; s->id = id; s->block = -1; s->request = 0;
      return s;
    }
    if (s->id == id) return s;
    h = (h + 1) & (S->mapcap - 1);
  }
}

static int64_t new_block(State* S) {
  if (grow((void**)&S->blk, &S->capblk, S->nblk + 1, sizeof(Block))) return -1;
  memset(&S->blk[S->nblk], 0, sizeof(Block));
  S->blk[S->nblk].prev = S->blk[S->nblk].next = -1;
  S->blk[S->nblk].alive = 1;
  return S->nblk++;
}

static int free_index_add(State* S, int64_t b) {
  if (grow((void**)&S->fr, &S->capfr, S->nfr + 1, sizeof(int64_t))) return XMO_E_NOMEM;
  S->fr[S->nfr++] = b;
  /* torch BlockPool::insert_into_blocks: gc_count_base = the pool's
   * get_free_blocks_call_count, so the block's age counts from now */
  S->blk[b].gc_base = S->searches[S->blk[b].small];
  return 0;
}

/* Return a whole-segment free block's segment to the device (torch
 * release_block). The caller removes it from the free index. */
static void release_segment_of(State* S, Block* b, uint64_t* out) {
  Segment* g = &S->seg[b->seg];
  g->alive = 0;
  S->reserved -= g->size;
  S->live_segs -= 1;
  out[F_NSEG_RELEASE] += 1;
  b->alive = 0;
}

static void free_index_remove(State* S, int64_t b) {
  for (int64_t k = 0; k < S->nfr; ++k)
    if (S->fr[k] == b) { S->fr[k] = S->fr[S->nfr - 1]; S->nfr--; return; }
}

/* torch release_cached_blocks (reading Q3; PAPER.md:259 (iv) "Cached blocks
 * persist until the framework allocator needs more memory, but the device
 * indicates an OOM error"; (v) "even after attempting the reclamation of cached
 * segments"): every free block that spans its whole segment is returned. */
static void release_cached(State* S, uint64_t* out) {
  int64_t k = 0;
  while (k < S->nfr) {
    Block* b = &S->blk[S->fr[k]];
    if (b->prev < 0 && b->next < 0) {
      Segment* g = &S->seg[b->seg];
      g->alive = 0;
      S->reserved -= g->size;
      S->live_segs -= 1;
      out[F_NSEG_RELEASE] += 1;
      b->alive = 0;
      S->fr[k] = S->fr[S->nfr - 1];
      S->nfr--;
    } else {
      ++k;
    }
  }
}

/* Variant: SPEC.md:283 D3 "Reclamation releases only
 * fully-free segments, both pools, largest first, stopping when capacity
 * suffices" (ties in size: lowest address first -- a reading, Q19). */
static void release_largest_first(State* S, uint64_t need, uint64_t capacity, uint64_t* out) {
  while (S->reserved + need > capacity) {
    int64_t best = -1;
    for (int64_t k = 0; k < S->nfr; ++k) {
      Block* b = &S->blk[S->fr[k]];
      if (b->prev >= 0 || b->next >= 0) continue;        /* not a whole segment */
      if (best < 0 || b->size > S->blk[S->fr[best]].size ||
          (b->size == S->blk[S->fr[best]].size && b->addr < S->blk[S->fr[best]].addr))
        best = k;
    }
    if (best < 0) return;
    Block* b = &S->blk[S->fr[best]];
    Segment* g = &S->seg[b->seg];
    g->alive = 0;
    S->reserved -= g->size;
    S->live_segs -= 1;
    out[F_NSEG_RELEASE] += 1;
    b->alive = 0;
    S->fr[best] = S->fr[S->nfr - 1];
    S->nfr--;
  }
}

/* Variant (NEXT-4, reading Q26): torch release_available_cached_blocks, run
 * only when max_split_size is set, when the device refuses a new segment and
 * before release_cached. key = max(s, max_split_size). In the request's pool
 * and stream, the smallest free block with size >= key (lowest address on a
 * tie) is released if there is one; otherwise the free blocks of that pool
 * and stream with size >= max_split_size are released from the largest down
 * (torch walks its (stream, size, address) set backwards: equal sizes go
 * highest address first) until at least key bytes are released. Blocks of
 * max_split_size or more are never split, so each is a whole segment (checked:
 * XMO_E_INVARIANT otherwise). Returns 1 when it released the one block or at
 * least key bytes (torch then retries the device), 0 otherwise (torch goes on
 * to release_cached straight away; the releases made stand), <0 on error. */
static int release_available(State* S, const xmo_config* c, uint64_t s, int small, int32_t stream,
                             uint64_t* out) {
  if (c->max_split_size == UINT64_MAX) return 0;
  uint64_t key = s < c->max_split_size ? c->max_split_size : s;
  int64_t best = -1;
  for (int64_t k = 0; k < S->nfr; ++k) {
    Block* B = &S->blk[S->fr[k]];
    if (B->small != small || B->stream != stream || B->size < key) continue;
    if (best < 0 || B->size < S->blk[S->fr[best]].size ||
        (B->size == S->blk[S->fr[best]].size && B->addr < S->blk[S->fr[best]].addr))
      best = k;
  }
  if (best >= 0) {
    Block* B = &S->blk[S->fr[best]];
    if (B->prev >= 0 || B->next >= 0) return XMO_E_INVARIANT;
    release_segment_of(S, B, out);
    S->fr[best] = S->fr[S->nfr - 1];
    S->nfr--;
    return 1;
  }
  uint64_t released = 0;
  while (released < key) {
    int64_t top = -1;                     /* largest (size, addr) below key */
    for (int64_t k = 0; k < S->nfr; ++k) {
      Block* B = &S->blk[S->fr[k]];
      if (B->small != small || B->stream != stream) continue;
      if (top < 0 || B->size > S->blk[S->fr[top]].size ||
          (B->size == S->blk[S->fr[top]].size && B->addr > S->blk[S->fr[top]].addr))
        top = k;
    }
    if (top < 0) break;
    Block* B = &S->blk[S->fr[top]];
    if (B->size < c->max_split_size) break;
    if (B->prev >= 0 || B->next >= 0) return XMO_E_INVARIANT;
    released += B->size;
    release_segment_of(S, B, out);
    S->fr[top] = S->fr[S->nfr - 1];
    S->nfr--;
  }
  return released >= key ? 1 : 0;
}

/* Variant (NEXT-4, reading Q27): torch garbage_collect_cached_blocks, run on
 * every free-block search that found nothing while garbage_collection_threshold
 * is set and the capacity is finite. Acts only when reserved exceeds
 * threshold * capacity; then, over the LARGE pool's whole-segment free blocks
 * (all streams), repeatedly: the mean age (double(total age) / count) is the
 * bar, and every block at least that old is released (in one pass, without
 * stopping at the target), until reserved has dropped by the excess or a pass
 * releases nothing. Age = large-pool searches since the block entered the free
 * index (torch gc_count). */
static void garbage_collect(State* S, const xmo_config* c, uint64_t* out) {
  uint64_t gc_bytes = (uint64_t)(c->gc_threshold * (double)c->capacity);
  if (S->reserved <= gc_bytes) return;
  uint64_t target = S->reserved - gc_bytes, reclaimed = 0, total_age = 0;
  int64_t freeable = 0;
  for (int64_t k = 0; k < S->nfr; ++k) {
    Block* B = &S->blk[S->fr[k]];
    if (B->small || B->prev >= 0 || B->next >= 0) continue;
    total_age += S->searches[0] - B->gc_base;
    freeable++;
  }
  if (freeable == 0) return;
  int freed = 1;
  while (reclaimed < target && freed && freeable > 0) {
    double age_threshold = (double)total_age / (double)freeable;
    freed = 0;
    int64_t k = 0;
    while (k < S->nfr) {
      Block* B = &S->blk[S->fr[k]];
      uint64_t age = S->searches[0] - B->gc_base;
      if (!B->small && B->prev < 0 && B->next < 0 && (double)age >= age_threshold) {
        freed = 1;
        reclaimed += B->size;
        total_age -= age;
        freeable--;
        release_segment_of(S, B, out);
        S->fr[k] = S->fr[S->nfr - 1];
        S->nfr--;
      } else {
        ++k;
      }
    }
  }
}

/* Invariants (SPEC.md:272-279 plus DESIGN.md §Invariants), checked after every
 * event in check mode. Returns 0 or XMO_E_INVARIANT. */
static int check_state(State* S, const xmo_config* c) {
  uint64_t res = 0, blk = 0;
  int64_t nfree = 0, nlive = 0;
  for (int64_t g = 0; g < S->nseg; ++g) {
    Segment* G = &S->seg[g];
    if (!G->alive) continue;
    nlive++;
    res += G->size;
    int64_t first = -1;
    for (int64_t i = 0; i < S->nblk; ++i)
      if (S->blk[i].alive && S->blk[i].seg == g && S->blk[i].prev < 0) {
        if (first >= 0) return XMO_E_INVARIANT;  /* two heads */
        first = i;
      }
    if (first < 0) return XMO_E_INVARIANT;
    uint64_t a = G->base, sum = 0;
    int prev_free = 0;
    for (int64_t i = first; i >= 0; i = S->blk[i].next) {
      Block* B = &S->blk[i];
      if (!B->alive || B->seg != g) return XMO_E_INVARIANT;
      if (B->addr != a) return XMO_E_INVARIANT;                 /* tiling */
      if (B->size == 0 || B->size % c->min_block) return XMO_E_INVARIANT; /* alignment */
      if (B->stream != G->stream || B->small != G->small) return XMO_E_INVARIANT;
      if (!B->allocated && prev_free) return XMO_E_INVARIANT;   /* coalescing maximality */
      if (B->next >= 0 && S->blk[B->next].prev != i) return XMO_E_INVARIANT;
      prev_free = !B->allocated;
      if (B->allocated) blk += B->size; else nfree++;
      a += B->size; sum += B->size;
    }
    if (sum != G->size) return XMO_E_INVARIANT;                 /* tiling */
  }
  if (nlive != S->live_segs || res != S->reserved || blk != S->alloc_blk) return XMO_E_INVARIANT;
  if (nfree != S->nfr) return XMO_E_INVARIANT;                  /* index mirrors free blocks */
  for (int64_t k = 0; k < S->nfr; ++k) {
    Block* B = &S->blk[S->fr[k]];
    if (!B->alive || B->allocated) return XMO_E_INVARIANT;
  }
  if (!(S->alloc_tensor <= S->alloc_blk && S->alloc_blk <= S->reserved)) return XMO_E_INVARIANT;
  if (S->reserved > c->capacity) return XMO_E_INVARIANT;
  return 0;
}

static void state_free(State* S) {
  free(S->blk); free(S->seg); free(S->fr); free(S->map);
  memset(S, 0, sizeof(*S));
}

/* ------------------------------------------------------------------------ */
/* simulate(seq, cfg) -> outcome  ("processes   */
/* the orchestrated memory event sequence chronologically")                  */
/* ------------------------------------------------------------------------ */
int xmo_simulate(const int64_t* bytes, const uint32_t* tag, int64_t n,
                 const xmo_config* c, uint64_t capacity, uint64_t* out,
                 uint64_t* curve, int check) {
  State S;
  memset(&S, 0, sizeof(S));
  memset(out, 0, sizeof(uint64_t) * XMO_NF);
  xmo_config cc = *c;
  cc.capacity = capacity;
  int rc = 0;

  int64_t nalloc = 0;
  for (int64_t i = 0; i < n; ++i) nalloc += bytes[i] > 0;
  S.mapcap = 16;
  while (S.mapcap < (uint64_t)(2 * nalloc + 2)) S.mapcap *= 2;
  S.map = (Slot*)calloc(S.mapcap, sizeof(Slot));
  if (!S.map) return XMO_E_NOMEM;

  uint64_t status = XMO_T_OK;
  int64_t i;
  for (i = 0; i < n; ++i) {
    uint32_t id = tag[i] & 0x0FFFFFFFu;
    int32_t stream = (int32_t)(tag[i] >> 28);
    if (bytes[i] == 0) { rc = XMO_E_ZERO; goto done; }

    if (bytes[i] > 0) {
      /* ---------------- ALLOC ("attempts to secure memory") -- */
      uint64_t req = (uint64_t)bytes[i];
      Slot* sl = map_find(&S, id, 1);
      if (sl->block >= 0) { rc = XMO_E_DUP; goto done; }
      uint64_t s = xmo_round_size(req, &cc);
      int small = xmo_is_small(s, &cc);

      /* torch get_free_block counts its calls per pool while GC is on */
      int gc_on = cc.gc_threshold > 0.0 && cc.capacity != UINT64_MAX;
      if (gc_on) S.searches[small] += 1;

      /* best fit: min (size, addr) over free blocks of this pool and stream */
      int64_t best = -1;
      for (int64_t k = 0; k < S.nfr; ++k) {
        Block* B = &S.blk[S.fr[k]];
        if (B->small != small || B->stream != stream || B->size < s) continue;
        if (best < 0 || B->size < S.blk[best].size ||
            (B->size == S.blk[best].size && B->addr < S.blk[best].addr))
          best = S.fr[k];
      }

      /* max_split_size variant (reading Q26; torch get_free_block): "Do not
       * return an oversized block" -- for a request below max_split_size, a
       * best fit of max_split_size or more; for a larger request, a best fit
       * of s + max_non_split_rounding or more. Nothing else is searched. */
      if (best >= 0) {
        uint64_t bs = S.blk[best].size;
        if (s < cc.max_split_size && bs >= cc.max_split_size) best = -1;
        else if (s >= cc.max_split_size && bs >= s + cc.max_non_split_rounding) best = -1;
      }

      int64_t b;
      if (best >= 0) {
        free_index_remove(&S, best);
        b = best;
      } else {
        if (gc_on) garbage_collect(&S, &cc, out);     /* GC variant (Q27)      */
        /* New segment from the device level (PAPER.md:259 (iv) "New segments
         * are requested from the GPU only if this cache is insufficient"). */
        uint64_t a = xmo_segment_size(s, &cc);
        if (S.reserved + a > cc.capacity) {           /* device refuses (Q10) */
          if (cc.reclaim_policy == 1) {
            release_largest_first(&S, a, cc.capacity, out);  /* SPEC D3 variant */
          } else {
            /* torch: alloc_block || (release_available && alloc_block) ||
             * (release_cached && alloc_block) */
            int e = release_available(&S, &cc, s, small, stream, out);   /* Q26 */
            if (e < 0) { rc = e; goto done; }
            if (e == 0 || S.reserved + a > cc.capacity)
              release_cached(&S, out);                /* reclaim (Q3)          */
          }
          if (S.reserved + a > cc.capacity) {         /* retry refused: OOM    */
            status = XMO_T_OOM;                       /* PAPER.md:260 (v)      */
            break;
          }
        }
        if (grow((void**)&S.seg, &S.capseg, S.nseg + 1, sizeof(Segment))) { rc = XMO_E_NOMEM; goto done; }
        int64_t g = S.nseg++;
        S.seg[g].base = S.next_base; S.seg[g].size = a;
        S.seg[g].stream = stream; S.seg[g].small = small; S.seg[g].alive = 1;
        S.next_base += a;
        S.reserved += a;
        S.live_segs += 1;
        out[F_NSEG_ALLOC] += 1;
        if ((uint64_t)S.live_segs > out[F_MAX_LIVE_SEG]) out[F_MAX_LIVE_SEG] = (uint64_t)S.live_segs;
        b = new_block(&S);
        if (b < 0) { rc = XMO_E_NOMEM; goto done; }
        S.blk[b].addr = S.seg[g].base; S.blk[b].size = a; S.blk[b].seg = g;
        S.blk[b].stream = stream; S.blk[b].small = small;
        sl = map_find(&S, id, 1);  /* (arena realloc does not move the map) */
      }

      /* split: the request takes the low end, the remainder stays free; with
       * max_split_size set a large-pool request of that size or more is never
       * split (torch should_split: size < max_split_size && remaining > ...) */
      uint64_t rem = S.blk[b].size - s;
      if (xmo_should_split(small, rem, &cc) && (small || s < cc.max_split_size)) {
        int64_t r = new_block(&S);
        if (r < 0) { rc = XMO_E_NOMEM; goto done; }
        Block* B = &S.blk[b];
        Block* R = &S.blk[r];
        R->addr = B->addr + s; R->size = rem; R->seg = B->seg;
        R->stream = B->stream; R->small = B->small; R->allocated = 0;
        R->prev = b; R->next = B->next;
        if (B->next >= 0) S.blk[B->next].prev = r;
        B->next = r;
        B->size = s;
        if (free_index_add(&S, r)) { rc = XMO_E_NOMEM; goto done; }
      }
      S.blk[b].allocated = 1;
      S.alloc_blk += S.blk[b].size;
      S.alloc_tensor += s;
      sl->block = b;
      sl->request = req;
    } else {
      /* ---------------- FREE ("marks the block as free ...
       * which may trigger coalescing"; reserved unchanged, PAPER.md:259 (iv)) */
      uint64_t req = (uint64_t)(-bytes[i]);
      Slot* sl = map_find(&S, id, 0);
      if (!sl || sl->block < 0) { rc = XMO_E_NOTLIVE; goto done; }
      if (sl->request != req) { rc = XMO_E_SIZE; goto done; }
      int64_t b = sl->block;
      sl->block = -1;
      Block* B = &S.blk[b];
      S.alloc_blk -= B->size;
      S.alloc_tensor -= xmo_round_size(req, &cc);
      B->allocated = 0;
      /* merge with the previous block, then the next one, when free */
      int64_t p = B->prev;
      if (p >= 0 && !S.blk[p].allocated) {
        Block* P = &S.blk[p];
        free_index_remove(&S, p);
        B->addr = P->addr;
        B->size += P->size;
        B->prev = P->prev;
        if (P->prev >= 0) S.blk[P->prev].next = b;
        P->alive = 0;
      }
      int64_t q = B->next;
      if (q >= 0 && !S.blk[q].allocated) {
        Block* Q = &S.blk[q];
        free_index_remove(&S, q);
        B->size += Q->size;
        B->next = Q->next;
        if (Q->next >= 0) S.blk[Q->next].prev = b;
        Q->alive = 0;
      }
      if (free_index_add(&S, b)) { rc = XMO_E_NOMEM; goto done; }
    }

    /* time series and peaks ("The Estimated Peak Memory is then
     * identified as the maximum value in this time series"; first index, Q7) */
    if (S.alloc_tensor > out[F_PEAK_ALLOC]) { out[F_PEAK_ALLOC] = S.alloc_tensor; out[F_PEAK_ALLOC_IDX] = (uint64_t)i; }
    if (S.alloc_blk > out[F_PEAK_BLK]) { out[F_PEAK_BLK] = S.alloc_blk; out[F_PEAK_BLK_IDX] = (uint64_t)i; }
    if (S.reserved > out[F_PEAK_RES]) { out[F_PEAK_RES] = S.reserved; out[F_PEAK_RES_IDX] = (uint64_t)i; }
    if (curve) { curve[3 * i] = S.alloc_tensor; curve[3 * i + 1] = S.alloc_blk; curve[3 * i + 2] = S.reserved; }
    if (check && check_state(&S, &cc)) { rc = XMO_E_INVARIANT; out[F_EVENTS_DONE] = (uint64_t)i; goto done; }
  }
  if (check && check_state(&S, &cc)) { rc = XMO_E_INVARIANT; goto done; }
  out[F_EVENTS_DONE] = (uint64_t)i;
  out[F_STATUS] = status;
  out[F_FINAL_RES] = S.reserved;
  out[F_NFREE_END] = (uint64_t)S.nfr;
  out[F_FINAL_ALLOC] = S.alloc_tensor;
  out[F_FINAL_BLK] = S.alloc_blk;
done:
  state_free(&S);
  return rc;
}

/* Batch driver: traces are independent (one after another, no shared state).
 * Returns 0, or the first error with *bad_trace set. */
int xmo_simulate_batch(const int64_t* bytes, const uint32_t* tag, const int64_t* off,
                       int64_t n_traces, const xmo_config* c, const uint64_t* capacity,
                       uint64_t* out, int check, int64_t* bad_trace) {
  *bad_trace = -1;
  for (int64_t t = 0; t < n_traces; ++t) {
    int64_t a = off[t], b = off[t + 1];
    int rc = xmo_simulate(bytes + a, tag + a, b - a, c, capacity ? capacity[t] : c->capacity,
                          out + (size_t)t * XMO_NF, NULL, check);
    if (rc) { *bad_trace = t; return rc; }
  }
  return 0;
}

int xmo_nfields(void) { return XMO_NF; }
