// replay.cu -- K2: batched caching-allocator replay, one warp per trace (sm_100a).
//
// Computes xMem's Simulator (§3.4) for every trace of a
// batch: (i) round-up, (ii) segment sizing, (iii) best-fit-with-coalescing
// search / split / merge, (iv) caching, (v) two-level OOM with reclamation,
// plus the time-series peaks. Rules and readings: DESIGN.md
// §2 (Q1-Q18); per-step citations inline.
//
// Execution model (DESIGN.md §6 K2):
//  * persistent grid, one CTA per SM, 16 warps per CTA, one trace per warp;
//    traces are pulled longest-first (host LPT order) from one atomic counter;
//  * each CTA owns a shared-memory HEAP (all of the SM's 227 KB, 512 B pages).
//    A warp sizes a region for its trace's state (id space + a free-list
//    guess), takes it FIFO (ticket lock) from the heap, replays, frees it. So
//    occupancy adapts: few warps hold the big early traces, many hold the
//    small later ones. A free list that outgrows its guess restarts the trace
//    in a 4x larger region; a trace larger than the heap runs in a
//    global-memory arena sized to the exact bound (never overflows);
//  * events stream through registers in 32-event tiles (coalesced streaming
//    loads, next tile prefetched); round-up and the allocated-bytes prefix
//    scan of a tile are lane-parallel (a2, a3);
//  * the serial state machine is warp-uniform (every lane computes the same
//    scalars, so no broadcasts); the best-fit search scans the free list
//    lane-strided with ONE packed 32-bit key per entry (class in the top 5
//    bits, saturated size below) and __reduce_min_sync; exact (size, pos)
//    tie-breaking falls back to a full compare only when needed (a5).
//
// State (structure of arrays):
//  A[id]  allocated block of dense id: pos u64, size u32, prev u32, next u32, cls u8
//  F[f]   free block f (unordered, nf entries): pos u64, key u32, size u32, prev u32, next u32
//  pos  = segment_index << 32 | offset_in_units  (bump addresses never reused:
//         (size, pos) order == SPEC D2's (size, segment, offset), reading Q4)
//  prev/next = address-order neighbours in the segment: kNone, an id, or kF|f
//  cls  = stream << 1 | small_pool ;  key = cls << 27 | min(size, 2^27-1)
#include <cuda_runtime.h>

#include <algorithm>

#include "xm_internal.h"

#ifdef XM_DEBUG
#include <cstdio>
#define XM_CHECK(cond, ...)                                   \
  do {                                                        \
    if (!(cond)) {                                            \
      printf("XM_CHECK %s:%d: ", __FILE__, __LINE__);         \
      printf(__VA_ARGS__);                                    \
      __trap();                                               \
    }                                                         \
  } while (0)
#else
#define XM_CHECK(cond, ...) do {} while (0)
#endif

namespace {

constexpr uint32_t kNone = 0xFFFFFFFFu;
constexpr uint32_t kF = 0x80000000u;
constexpr uint32_t kIdMask = 0x07FFFFFFu;
constexpr uint32_t kAllocBit = 0x08000000u;
constexpr uint32_t kKeyBits = 27;
constexpr uint32_t kKeyMax = (1u << kKeyBits) - 1u;
constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr int kStatusOk = XM_T_OK, kStatusOom = XM_T_OOM, kStatusOverflow = XM_T_OVERFLOW;

// shared-memory heap geometry
constexpr uint32_t kPage = 512;
constexpr uint32_t kHdrBytes = 128;
constexpr uint32_t kMaxDynSmem = 232448;  // 227 KB, the sm_100 per-CTA maximum
constexpr uint32_t kMaxPages = (kMaxDynSmem - kHdrBytes) / kPage;  // 453
constexpr uint32_t kBitmapWords = (kMaxPages + 31) / 32;          // 15
static_assert(8 + 4 * kBitmapWords <= kHdrBytes, "heap header");

struct HeapHdr {
  int ticket;
  int serving;
  uint32_t bitmap[kBitmapWords];
};

struct KParams {
  const int64_t* __restrict__ bytes;
  const uint32_t* __restrict__ tag;
  const int64_t* __restrict__ off;
  const uint32_t* __restrict__ n_ids;
  const uint32_t* __restrict__ order;
  const uint64_t* __restrict__ capacity;
  uint64_t cap_default;
  int64_t n_traces;
  xm_internal::UnitConfig u;
  uint32_t heap_pages;       // pages per CTA heap
  uint32_t* counter;         // [0] work counter; [1..] arena claim bitmap
  unsigned char* arena;
  size_t arena_bytes;        // bytes per arena slot
  uint32_t n_arena;
  uint32_t arena_ids, arena_free;
  xm_result* out;
};

struct State {
  uint64_t* A_pos;
  uint32_t* A_size;
  uint32_t* A_prev;
  uint32_t* A_next;
  uint8_t* A_cls;
  uint64_t* F_pos;
  uint32_t* F_key;
  uint32_t* F_size;
  uint32_t* F_prev;
  uint32_t* F_next;
  uint32_t cap_f;
};

__host__ __device__ inline size_t state_bytes(uint32_t na, uint32_t nf) {
  return size_t(na) * 21 + size_t(nf) * 24 + 16;
}

__device__ inline State carve(unsigned char* base, uint32_t na, uint32_t nf) {
  State S;
  unsigned char* p = base;
  S.A_pos = reinterpret_cast<uint64_t*>(p); p += size_t(na) * 8;
  S.F_pos = reinterpret_cast<uint64_t*>(p); p += size_t(nf) * 8;
  S.A_size = reinterpret_cast<uint32_t*>(p); p += size_t(na) * 4;
  S.A_prev = reinterpret_cast<uint32_t*>(p); p += size_t(na) * 4;
  S.A_next = reinterpret_cast<uint32_t*>(p); p += size_t(na) * 4;
  S.F_key = reinterpret_cast<uint32_t*>(p); p += size_t(nf) * 4;
  S.F_size = reinterpret_cast<uint32_t*>(p); p += size_t(nf) * 4;
  S.F_prev = reinterpret_cast<uint32_t*>(p); p += size_t(nf) * 4;
  S.F_next = reinterpret_cast<uint32_t*>(p); p += size_t(nf) * 4;
  S.A_cls = p;
  S.cap_f = nf;
  return S;
}

__device__ __forceinline__ uint32_t make_key(uint32_t cls, uint32_t size) {
  return (cls << kKeyBits) | (size < kKeyMax ? size : kKeyMax);
}

__device__ __forceinline__ void set_next(const State& S, uint32_t ref, uint32_t v) {
  if (ref == kNone) return;
  XM_CHECK(!(ref & kF) || (ref & ~kF) < S.cap_f, "set_next ref=%x cap=%u\n", ref, S.cap_f);
  if (ref & kF) S.F_next[ref & ~kF] = v;
  else S.A_next[ref] = v;
}

__device__ __forceinline__ void set_prev(const State& S, uint32_t ref, uint32_t v) {
  if (ref == kNone) return;
  XM_CHECK(!(ref & kF) || (ref & ~kF) < S.cap_f, "set_prev ref=%x cap=%u\n", ref, S.cap_f);
  if (ref & kF) S.F_prev[ref & ~kF] = v;
  else S.A_prev[ref] = v;
}

// Remove free entry f by moving the last entry into its slot (warp-uniform).
__device__ __forceinline__ void f_remove(const State& S, uint32_t f, uint32_t& nf) {
  XM_CHECK(nf >= 1 && f < nf, "f_remove f=%u nf=%u\n", f, nf);
  const uint32_t L = nf - 1;
  if (f != L) {
    const uint32_t k = S.F_key[L], sz = S.F_size[L], pv = S.F_prev[L], nx = S.F_next[L];
    const uint64_t pos = S.F_pos[L];
    S.F_key[f] = k; S.F_size[f] = sz; S.F_pos[f] = pos; S.F_prev[f] = pv; S.F_next[f] = nx;
    set_next(S, pv, kF | f);
    set_prev(S, nx, kF | f);
  }
  nf = L;
}

__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

__device__ __forceinline__ int64_t warp_max_i64(int64_t v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    int64_t w = __shfl_xor_sync(kFull, v, o);
    v = w > v ? w : v;
  }
  return v;
}

// Reclamation (reading Q3; PAPER.md:259 (iv) "Cached blocks persist until the
// framework allocator needs more memory, but the device indicates an OOM
// error"): release every free block that spans a whole segment, in all pools
// and streams. Warp-parallel stable compaction of the free list.
__device__ __forceinline__ void reclaim(const State& S, uint32_t& nf, uint64_t& reserved,
                                     uint32_t& n_release, uint32_t& live_segs) {
  const uint32_t lane = threadIdx.x & 31;
  uint32_t newn = 0, cnt = 0;
  uint64_t freed = 0;
  for (uint32_t base = 0; base < nf; base += 32) {
    const uint32_t f = base + lane;
    const bool valid = f < nf;
    uint32_t k = 0, sz = 0, pv = kNone, nx = kNone;
    uint64_t pos = 0;
    if (valid) {
      k = S.F_key[f]; sz = S.F_size[f]; pv = S.F_prev[f]; nx = S.F_next[f]; pos = S.F_pos[f];
    }
    const bool whole = valid && pv == kNone && nx == kNone;
    const bool keep = valid && !whole;
    const unsigned km = __ballot_sync(kFull, keep);
    const unsigned wm = __ballot_sync(kFull, whole);
    const uint64_t fs = warp_sum_u64(whole ? uint64_t(sz) : 0ull);
    const uint32_t dst = newn + __popc(km & ((1u << lane) - 1u));
    __syncwarp();
    if (keep && dst != f) {
      S.F_key[dst] = k; S.F_size[dst] = sz; S.F_pos[dst] = pos; S.F_prev[dst] = pv; S.F_next[dst] = nx;
      set_next(S, pv, kF | dst);
      set_prev(S, nx, kF | dst);
    }
    __syncwarp();
    newn += __popc(km);
    cnt += __popc(wm);
    freed += fs;
  }
  nf = newn;
  reserved -= freed;
  n_release += cnt;
  live_segs -= cnt;
}

// Exact best fit: min (size, pos) over entries of class cls with size >= s.
// Used when the packed-key search cannot decide (ties, saturated sizes).
__device__ __forceinline__ uint32_t best_fit_exact(const State& S, uint32_t nf, uint32_t cls,
                                                uint32_t s) {
  const uint32_t lane = threadIdx.x & 31;
  uint32_t bsz = kNone, bf = kNone;
  uint64_t bpos = ~0ull;
  for (uint32_t f = lane; f < nf; f += 32) {
    const uint32_t k = S.F_key[f];
    if ((k >> kKeyBits) != cls) continue;
    const uint32_t sz = S.F_size[f];
    if (sz < s) continue;
    const uint64_t pos = S.F_pos[f];
    if (sz < bsz || (sz == bsz && pos < bpos)) { bsz = sz; bpos = pos; bf = f; }
  }
  __syncwarp();
  const uint32_t m = __reduce_min_sync(kFull, bsz);
  if (m == kNone) return kNone;
  const bool c1 = bsz == m;
  const uint32_t hi = c1 ? uint32_t(bpos >> 32) : kNone;
  const uint32_t mh = __reduce_min_sync(kFull, hi);
  const uint32_t lo = (c1 && hi == mh) ? uint32_t(bpos) : kNone;
  const uint32_t ml = __reduce_min_sync(kFull, lo);
  const int wl = __ffs(__ballot_sync(kFull, c1 && hi == mh && uint32_t(bpos) == ml)) - 1;
  return __shfl_sync(kFull, bf, wl);
}

// Replays events [e0, e0+n) of one trace on state S. Returns the status; on
// XM_T_OVERFLOW the caller restarts the trace with a larger free list.
//
// Warp-uniform execution: every lane runs the same bookkeeping on the same
// values (loads of the same address are broadcasts; stores of the same value
// to the same address are benign), so no broadcasts are needed. This is only
// correct while the warp is CONVERGED: a split lane group would re-read state
// another group already updated. The only lane-dependent branches are the
// best-fit scan loop (reconverges before the reduction) and lane-0 regions in
// the caller, each closed by __syncwarp(); every event also ends with one.
__device__ __forceinline__ int replay_trace(const KParams& P, const State& S, int64_t e0,
                                            uint32_t n, uint64_t cap_u, xm_result& R) {
  const uint32_t lane = threadIdx.x & 31;
  const xm_internal::UnitConfig& u = P.u;
  const uint64_t unit_m1 = (1ull << u.unit_shift) - 1;
  const long long* __restrict__ by = reinterpret_cast<const long long*>(P.bytes) + e0;
  const uint32_t* __restrict__ tg = P.tag + e0;

  uint32_t nf = 0, nseg = 0, live_segs = 0, max_live = 0, n_release = 0;
  uint64_t reserved = 0, blk = 0;
  int64_t tensor = 0;
  uint64_t pk_tensor = 0, pk_blk = 0, pk_res = 0;
  uint32_t ix_tensor = 0, ix_blk = 0, ix_res = 0;
  int status = kStatusOk;
  uint32_t done_total = 0;

  int64_t b_nx = 0;
  uint32_t t_nx = 0;
  if (lane < n) { b_nx = __ldcs(by + lane); t_nx = __ldcs(tg + lane); }
  for (uint32_t base = 0; base < n; base += 32) {
    const int64_t bc = b_nx;
    const uint32_t tc = t_nx;
    const uint32_t cnt = min(32u, n - base);
    if (base + 32 + lane < n) { b_nx = __ldcs(by + base + 32 + lane); t_nx = __ldcs(tg + base + 32 + lane); }
    __syncwarp();                                       // reconverge after the lane-dependent branch
    // ---- a2: round-up of this lane's event (PAPER.md:256 (i)) ----
    const bool is_alloc = bc > 0;
    const uint64_t mag = is_alloc ? uint64_t(bc) : uint64_t(-bc);
    const uint32_t su = uint32_t((mag + unit_m1) >> u.unit_shift);
    // ---- a3: tile prefix-scan of +-s (allocated tensor bytes) ----
    int64_t d = lane < cnt ? (is_alloc ? int64_t(su) : -int64_t(su)) : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(kFull, d, o);
      if (lane >= uint32_t(o)) d += y;
    }
    const int64_t cur = tensor + d;
    const uint32_t w1 = (tc & 0xF0000000u) | (tc & kIdMask) | (is_alloc ? kAllocBit : 0u);

    uint32_t j = 0;
    for (; j < cnt; ++j) {
      const uint32_t s = __shfl_sync(kFull, su, j);
      const uint32_t w = __shfl_sync(kFull, w1, j);
      const uint32_t id = w & kIdMask;
      if (w & kAllocBit) {
        // ================= ALLOC =================
        const uint32_t small = s <= u.small_u;                     // a4: pool
        const uint32_t cls = ((w >> 28) << 1) | small;             // per-stream pools (Q5)
        // a5: best fit = min (size, pos) over free blocks of class cls with
        // size >= s. Candidate iff key in [cls<<27 | min(s,max), cls<<27 | max];
        // equal keys are ordered by pos, loaded only on a tie.
        const uint32_t lo = make_key(cls, s);
        const uint32_t span = (cls << kKeyBits | kKeyMax) - lo;
        uint32_t best = kNone, bf = kNone;
        uint64_t bpos = ~0ull;          // valid iff bpos_ok
        bool bpos_ok = false;
        for (uint32_t f = lane; f < nf; f += 32) {
          const uint32_t k = S.F_key[f];
          if (k - lo <= span) {
            if (k < best) {
              best = k; bf = f; bpos_ok = false;
            } else if (k == best) {
              if (!bpos_ok) { bpos = S.F_pos[bf]; bpos_ok = true; }
              const uint64_t pos = S.F_pos[f];
              if (pos < bpos) { bf = f; bpos = pos; }
            }
          }
        }
        __syncwarp();                                   // reconverge after the scan
        const bool has = bf != kNone;
        const uint32_t m = __reduce_min_sync(kFull, has ? best : kNone);
        uint32_t fsel = kNone;
        if (m != kNone || __any_sync(kFull, has)) {
          if ((m & kKeyMax) == kKeyMax) {
            fsel = best_fit_exact(S, nf, cls, s);          // saturated sizes: exact compare
          } else {
            const bool c1 = has && best == m;
            const unsigned win = __ballot_sync(kFull, c1);
            int wl;
            if ((win & (win - 1u)) == 0u) {
              wl = __ffs(win) - 1;
            } else {                                       // size tie across lanes: min pos
              if (c1 && !bpos_ok) bpos = S.F_pos[bf];
              __syncwarp();
              const uint32_t hi = c1 ? uint32_t(bpos >> 32) : kNone;
              const uint32_t mh = __reduce_min_sync(kFull, hi);
              const uint32_t lo2 = (c1 && hi == mh) ? uint32_t(bpos) : kNone;
              const uint32_t ml = __reduce_min_sync(kFull, lo2);
              wl = __ffs(__ballot_sync(kFull, c1 && hi == mh && uint32_t(bpos) == ml)) - 1;
            }
            fsel = __shfl_sync(kFull, bf, wl);
          }
        }
        uint32_t bsize, bprev, bnext;
        uint64_t bposu;
        if (fsel == kNone) {
          // a4/a6: new segment from the device level (PAPER.md:259 (iv), 169, 654)
          uint32_t a;
          if (small) a = u.sbuf_u;
          else if (s < u.minlarge_u) a = u.lbuf_u;
          else a = uint32_t((uint64_t(s) + u.rlarge_u - 1) / u.rlarge_u * u.rlarge_u);
          if (reserved + a > cap_u) {                          // device level refuses (Q10)
            reclaim(S, nf, reserved, n_release, live_segs);    // reclaim cached segments (Q3)
            if (reserved + a > cap_u) { status = kStatusOom; break; }  // both levels failed
          }
          bsize = a;
          bprev = kNone;
          bnext = kNone;
          bposu = uint64_t(nseg) << 32;
          nseg += 1;
          live_segs += 1;
          max_live = max(max_live, live_segs);
          reserved += a;
          if (reserved > pk_res) { pk_res = reserved; ix_res = base + j; }
        } else {
          bsize = S.F_size[fsel];
          bprev = S.F_prev[fsel];
          bnext = S.F_next[fsel];
          bposu = S.F_pos[fsel];
        }
        // a7: split (PAPER.md:258 (iii); reading Q1)
        const uint32_t rem = bsize - s;
        const bool split = small ? (rem >= 1u) : (u.strict ? (rem > u.small_u) : (rem >= u.small_u));
        uint32_t asize;
        if (split) {
          uint32_t r;
          if (fsel != kNone) {
            r = fsel;                                  // remainder keeps the free entry
          } else {
            if (nf >= S.cap_f) { status = kStatusOverflow; break; }
            r = nf++;
            S.F_next[r] = kNone;                       // new segment: no right neighbour
          }
          S.F_pos[r] = bposu + s;
          S.F_key[r] = make_key(cls, rem);
          S.F_size[r] = rem;
          S.F_prev[r] = id;
          S.A_next[id] = kF | r;
          asize = s;
        } else {
          S.A_next[id] = bnext;
          set_prev(S, bnext, id);
          if (fsel != kNone) f_remove(S, fsel, nf);
          asize = bsize;
        }
        S.A_size[id] = asize;
        S.A_pos[id] = bposu;
        S.A_prev[id] = bprev;
        S.A_cls[id] = uint8_t(cls);
        set_next(S, bprev, id);
        blk += asize;
        // a9: the block peak only moves up on allocs, first index (Q7)
        if (blk > pk_blk) { pk_blk = blk; ix_blk = base + j; }
      } else {
        // ================= FREE =================
        const uint32_t sz = S.A_size[id];
        const uint32_t p = S.A_prev[id];
        const uint32_t q = S.A_next[id];
        const bool pf = p != kNone && (p & kF);
        const bool qf = q != kNone && (q & kF);
        // a8: coalesce with free neighbours; reserved unchanged (PAPER.md:259 (iv))
        if (pf) {
          const uint32_t P_ = p & ~kF;
          uint32_t nsz = S.F_size[P_] + sz;
          uint32_t nn = q;
          if (qf) {
            const uint32_t N_ = q & ~kF;
            nsz += S.F_size[N_];
            nn = S.F_next[N_];
          }
          S.F_size[P_] = nsz;
          S.F_key[P_] = make_key(S.A_cls[id], nsz);
          S.F_next[P_] = nn;
          set_prev(S, nn, p);
          if (qf) f_remove(S, q & ~kF, nf);
        } else if (qf) {
          const uint32_t N_ = q & ~kF;
          const uint32_t nsz = S.F_size[N_] + sz;
          S.F_pos[N_] = S.A_pos[id];
          S.F_size[N_] = nsz;
          S.F_key[N_] = make_key(S.A_cls[id], nsz);
          S.F_prev[N_] = p;
          set_next(S, p, q);
        } else {
          if (nf >= S.cap_f) { status = kStatusOverflow; break; }
          const uint32_t r = nf++;
          S.F_pos[r] = S.A_pos[id];
          S.F_size[r] = sz;
          S.F_key[r] = make_key(S.A_cls[id], sz);
          S.F_prev[r] = p;
          S.F_next[r] = q;
          set_next(S, p, kF | r);
          set_prev(S, q, kF | r);
        }
        blk -= sz;
      }
      __syncwarp();
    }
    __syncwarp();
    // a3: allocated-tensor peak over the processed prefix of this tile
    const int64_t v = lane < j ? cur : INT64_MIN;
    const int64_t mx = warp_max_i64(v);
    if (j > 0 && mx > int64_t(pk_tensor)) {
      const unsigned bm = __ballot_sync(kFull, v == mx);
      pk_tensor = uint64_t(mx);
      ix_tensor = base + __ffs(bm) - 1;
    }
    tensor = __shfl_sync(kFull, cur, 31);
    done_total = base + j;
    XM_CHECK(nf <= S.cap_f, "nf=%u cap=%u base=%u\n", nf, S.cap_f, base);
    if (status != kStatusOk) break;
  }
  const uint32_t sh = u.unit_shift;
  R.peak_allocated = pk_tensor << sh;
  R.peak_allocated_blk = pk_blk << sh;
  R.peak_reserved = pk_res << sh;
  R.final_reserved = reserved << sh;
  R.peak_allocated_idx = ix_tensor;
  R.peak_allocated_blk_idx = ix_blk;
  R.peak_reserved_idx = ix_res;
  R.n_seg_alloc = nseg;
  R.n_seg_release = n_release;
  R.max_live_segments = max_live;
  R.events_done = status == kStatusOk ? n : done_total;
  R.status = uint16_t(status);
  R.n_free_blocks_end = uint16_t(nf > 0xFFFFu ? 0xFFFFu : nf);
  return status;
}

// ---- shared-memory heap (one per CTA) --------------------------------------
// All heap and arena routines are called by the WHOLE warp with warp-uniform
// control flow: single-lane work is predicated and its result broadcast, and
// every wait loop tests a broadcast (uniform) condition. A lane-0-only branch
// around a spinning call would leave the warp split into lane groups for the
// rest of the trace, which breaks the warp-uniform replay (see replay_trace).
__device__ __forceinline__ uint32_t bitmap_word(const HeapHdr* h, uint32_t w) {
  return reinterpret_cast<const volatile uint32_t*>(h->bitmap)[w];
}

// Is [p, p+np) free? (reads the bitmap word by word)
__device__ __forceinline__ bool run_free(const HeapHdr* h, uint32_t p, uint32_t np) {
  const uint32_t e = p + np;
  for (uint32_t q = p; q < e;) {
    const uint32_t w = q >> 5, b0 = q & 31;
    const uint32_t nb = min(32u - b0, e - q);
    const uint32_t mask = (nb == 32 ? 0xFFFFFFFFu : ((1u << nb) - 1u)) << b0;
    if (bitmap_word(h, w) & mask) return false;
    q += nb;
  }
  return true;
}

// stats: [0] restarts, [1] arena runs, [2] heap wait rounds, [3] ticket wait rounds
__device__ uint32_t heap_alloc(HeapHdr* h, uint32_t total, uint32_t np, uint32_t* stats) {
  const uint32_t lane = threadIdx.x & 31;
  int t = 0;
  if (lane == 0) t = atomicAdd(&h->ticket, 1);
  t = __shfl_sync(kFull, t, 0);
  uint32_t tw = 0, hw = 0;
  for (;;) {                                                   // FIFO: wait for our ticket
    const int srv = __shfl_sync(kFull, *(volatile int*)&h->serving, 0);
    if (srv == t) break;
    __nanosleep(128);
    ++tw;
  }
  uint32_t start;
  for (;;) {                                                   // first fit, lane-parallel
    uint32_t cand = kNone;
    for (uint32_t p = lane; p + np <= total; p += 32)
      if (run_free(h, p, np)) { cand = p; break; }
    __syncwarp();
    start = __reduce_min_sync(kFull, cand);
    if (start != kNone) break;
    __nanosleep(512);
    ++hw;
  }
  // claim: lane k sets word (start>>5)+k of the range
  const uint32_t w0 = start >> 5, w1 = (start + np - 1) >> 5;
  for (uint32_t w = w0 + lane; w <= w1; w += 32) {
    const uint32_t lo = max(start, w << 5), hi = min(start + np, (w + 1) << 5);
    const uint32_t nb = hi - lo;
    const uint32_t mask = (nb == 32 ? 0xFFFFFFFFu : ((1u << nb) - 1u)) << (lo & 31);
    const uint32_t old = atomicOr(&h->bitmap[w], mask);
    XM_CHECK((old & mask) == 0, "heap overlap start=%u np=%u\n", start, np);
    (void)old;
  }
  __syncwarp();
  __threadfence_block();
  if (lane == 0) {
    atomicAdd(&h->serving, 1);
    if (tw) atomicAdd(stats + 3, tw);
    if (hw) atomicAdd(stats + 2, hw);
  }
  __syncwarp();
  return start;
}

__device__ void heap_free(HeapHdr* h, uint32_t start, uint32_t np) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t w0 = start >> 5, w1 = (start + np - 1) >> 5;
  __syncwarp();
  for (uint32_t w = w0 + lane; w <= w1; w += 32) {
    const uint32_t lo = max(start, w << 5), hi = min(start + np, (w + 1) << 5);
    const uint32_t nb = hi - lo;
    const uint32_t mask = (nb == 32 ? 0xFFFFFFFFu : ((1u << nb) - 1u)) << (lo & 31);
    atomicAnd(&h->bitmap[w], ~mask);
  }
  __syncwarp();
}

// Claim a global arena slot (whole warp; spins while all are busy).
__device__ uint32_t arena_claim(uint32_t* bits, uint32_t n) {
  const uint32_t lane = threadIdx.x & 31;
  for (;;) {
    uint32_t got = kNone;
    if (lane == 0) {
      for (uint32_t i = 0; i < n; ++i) {
        const uint32_t m = 1u << (i & 31);
        if (!(atomicOr(&bits[i >> 5], m) & m)) { got = i; break; }
      }
    }
    got = __shfl_sync(kFull, got, 0);
    if (got != kNone) return got;
    __nanosleep(1024);
  }
}

__global__ void __launch_bounds__(512, 1) k_replay(KParams P) {
  extern __shared__ __align__(128) unsigned char smem[];
  HeapHdr* hdr = reinterpret_cast<HeapHdr*>(smem);
  unsigned char* pages = smem + kHdrBytes;
  const uint32_t lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    hdr->ticket = 0;
    hdr->serving = 0;
    for (uint32_t i = 0; i < kBitmapWords; ++i) hdr->bitmap[i] = 0;
  }
  __syncthreads();
  for (;;) {
    uint32_t k = 0;
    if (lane == 0) k = atomicAdd(P.counter, 1u);
    k = __shfl_sync(kFull, k, 0);
    if (int64_t(k) >= P.n_traces) break;
    const uint32_t t = P.order[k];
    const int64_t e0 = P.off[t];
    const uint32_t n = uint32_t(P.off[t + 1] - e0);
    const uint32_t na = P.n_ids[t];
    const uint64_t cap = P.capacity ? P.capacity[t] : P.cap_default;
    const uint64_t cap_u = cap >> P.u.unit_shift;
    xm_result R;
    const uint32_t nf_exact = n + 1;              // nf <= events
    uint32_t nfc = min(nf_exact, na / 4 + 96);
    int st = kStatusOverflow;
    for (;;) {
      const uint32_t np = uint32_t((state_bytes(na, nfc) + kPage - 1) / kPage);
      if (np > P.heap_pages) break;
      const uint32_t start = heap_alloc(hdr, P.heap_pages, np, P.counter + 32);
      const State S = carve(pages + size_t(start) * kPage, na, nfc);
      st = replay_trace(P, S, e0, n, cap_u, R);
      heap_free(hdr, start, np);
      if (st != kStatusOverflow || nfc >= nf_exact) break;
      if (lane == 0) atomicAdd(P.counter + 32, 1u);
      nfc = min(nf_exact, nfc * 4);
    }
    if (st == kStatusOverflow) {
      // global arena, exact bound: cannot overflow
      const uint32_t slot = arena_claim(P.counter + 1, P.n_arena);
      if (lane == 0) atomicAdd(P.counter + 33, 1u);
      const State S = carve(P.arena + size_t(slot) * P.arena_bytes, na, nf_exact);
      st = replay_trace(P, S, e0, n, cap_u, R);
      __syncwarp();
      __threadfence();
      if (lane == 0) atomicAnd(P.counter + 1 + (slot >> 5), ~(1u << (slot & 31)));
    }
    if (lane == 0) P.out[t] = R;
    __syncwarp();
  }
}

}  // namespace

namespace xm_internal {

ReplayPlan plan_replay(const xm_batch* b, const xm_config* cfg) {
  ReplayPlan p{};
  int dev = 0, sms = 148;
  if (cuda_usable() && cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaGetLastError();
  p.warps_per_cta = cfg->warps_per_cta ? int(cfg->warps_per_cta) : 16;
  if (p.warps_per_cta > 16) p.warps_per_cta = 16;
  if (p.warps_per_cta < 1) p.warps_per_cta = 1;
  // heap: the whole per-CTA maximum unless capped (smem_per_warp x warps)
  size_t heap = size_t(kMaxPages) * kPage;
  if (cfg->smem_per_warp) heap = std::min(heap, size_t(cfg->smem_per_warp) * p.warps_per_cta);
  if (heap < kPage) heap = kPage;
  p.heap_pages = uint32_t(heap / kPage);
  p.ctas = sms;
  const int64_t warps_total = int64_t(p.ctas) * p.warps_per_cta;
  if (b->n_traces < warps_total) {
    p.ctas = int((b->n_traces + p.warps_per_cta - 1) / p.warps_per_cta);
    if (p.ctas < 1) p.ctas = 1;
  }
  // global arenas (exact bound): a pool of slots, claimed only by traces whose
  // state cannot live in shared memory
  p.arena_ids = b->max_ids;
  p.arena_free = b->max_events + 1;
  p.arena_per_warp = (state_bytes(p.arena_ids, p.arena_free) + 255) & ~size_t(255);
  const int64_t tw = int64_t(p.ctas) * p.warps_per_cta;
  const uint32_t n_arena = uint32_t(std::min<int64_t>(std::min<int64_t>(tw, 64),
                                                      std::max<int64_t>(1, b->n_traces)));
  p.n_arena = n_arena;
  p.scratch_bytes = 256 + size_t(n_arena) * p.arena_per_warp;
  return p;
}

int launch_replay(const xm_batch* b, const xm_config* cfg, const UnitConfig& u,
                  const ReplayPlan& plan, void* d_scratch, xm_result* d_out, void* stream,
                  int* n_launches) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  KParams P{};
  P.bytes = b->bytes;
  P.tag = b->tag;
  P.off = b->off;
  P.n_ids = b->n_ids;
  P.order = b->order;
  P.capacity = b->capacity;
  P.cap_default = cfg->capacity;
  P.n_traces = b->n_traces;
  P.u = u;
  P.heap_pages = plan.heap_pages;
  P.counter = static_cast<uint32_t*>(d_scratch);
  P.arena = static_cast<unsigned char*>(d_scratch) + 256;
  P.arena_bytes = plan.arena_per_warp;
  P.n_arena = plan.n_arena;
  P.arena_ids = plan.arena_ids;
  P.arena_free = plan.arena_free;
  P.out = d_out;
  cudaError_t e = cudaMemsetAsync(d_scratch, 0, 256, st);
  if (e != cudaSuccess) return int(e);
  const size_t smem = kHdrBytes + size_t(plan.heap_pages) * kPage;
  e = cudaFuncSetAttribute(k_replay, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return int(e);
  k_replay<<<plan.ctas, plan.warps_per_cta * 32, smem, st>>>(P);
  *n_launches += 1;
  return int(cudaGetLastError());
}

}  // namespace xm_internal
