// lifecycle.cu -- K5: batched lifecycle reconstruction,
// the Analyzer step two before the Simulator: "pairing allocation and
// deallocation events based on address tracking and timing ... while
// correctly handling address reuse. Blocks lacking a deallocation event are
// considered persistent" (§3.2); SPEC.md:104-112 (LIFO per
// address, orphan and mismatch tallies). Its output is also the replay's
// input: the kept events (allocations + matched frees) in the xm_batch wire
// format with dense block ids, so profiler instants go to k_replay without a
// host round trip.
//
//   k_reconstruct  one warp per trace (persistent grid), 32-instant tiles:
//     * allocations take dense ids at the tile start from a per-warp free-id
//       stack (ids freed in earlier tiles; then fresh ids), so an id is never
//       reused while its block is open and n_ids <= max open + 31;
//     * matching: a per-warp open-addressing hash table in global memory maps
//       address -> top of that address's stack of open blocks (linked through
//       the allocations' event indices); each trace clears and uses the
//       first 2^ceil(log2 (n+1)) slots of its warp's region. Each allocation
//       writes one 16-byte record (stack link, dense id | stream, request
//       bytes), so a matching free reads everything it needs about its
//       allocation from one sector. When the tile's addresses are distinct (the common
//       case: __match_any_sync) every lane does its own lookup, insertions are
//       resolved by a read phase / claim phase loop; instants sharing an
//       address inside a tile are applied in rounds (round r: every
//       address's r-th instant);
//     * per instant: partner (alloc <-> free, -1 persistent / orphan),
//       mismatch flag; kept events are written compacted within the trace at
//       its input offset (staging), ids of matched blocks go back on the stack;
//   k_wire_offsets  one CTA: exclusive scan of the kept counts -> wire offsets;
//   k_wire_compact  one warp per trace: staging -> dense wire arrays, n_ids.
// HBM (algorithmic): 17 B/instant read, 5 B written (partner, mismatch) + 12 B
// staging write and read + 12 B wire write. Measured DRAM traffic is ~5x that
// (round 1 ncu): the random per-instant sectors (hash probes, records, the
// partner write of a matched allocation) mostly miss L2.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

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

constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr int kWarps = 16;                // per CTA; scratch is per warp slot
constexpr int kCtasPerSm = 4;

struct Slot {                             // 16 B hash slot
  unsigned long long addr;
  unsigned int gen;                       // trace index + 1 that owns it (0 = never)
  int top;                                // local index of the top open block, -1 none
};

struct __align__(16) ARec {                 // what a matching free needs, in one sector
  int below;                              // the address's previous open allocation (-1)
  uint32_t tag;                           // dense id | stream << 28
  long long bytes;                        // the allocation's request bytes
};

struct LParams {
  const uint32_t* __restrict__ tag;       // loader mode (xm_simulate_raw): raw block id |
                                          // stream << 28 stands for (addr, stream); else null
  const uint64_t* __restrict__ addr;
  const int64_t* __restrict__ bytes;
  const uint8_t* __restrict__ stream;
  const int64_t* __restrict__ off;
  int64_t n_traces;
  uint32_t hbits;                         // log2 slots per warp table
  Slot* tables;                           // [n_slots][1 << hbits]
  uint32_t* idstacks;                     // [n_slots][max_events]
  uint32_t max_events;
  ARec* arec;                             // [n_events] per allocation: stack link,
                                          // dense id | stream << 28, request bytes
  int64_t* st_bytes;                      // [n_events] staging (trace-compacted wire)
  uint32_t* st_tag;
  int32_t* partner;
  uint8_t* mismatch;
  xm_lifecycle* rec;
  unsigned int* work;
  const int64_t* wire_off;                // loader mode, direct wire output: the wire
  const uint32_t* pos;                    // offsets (stored order), caller -> stored
  uint32_t* w_nids;                       // index, n_ids out (0 = invalid); or null
  const uint32_t* chunk_first;            // loader mode, streamed input: [n_chunks + 1]
  const uint32_t* chunk_flag;             // first trace of each upload chunk; [0], [1]
                                          // the chunks landed so far on copy stream 0 / 1
                                          // (written stream-ordered after them), [2 + c]
                                          // chunk c's stream << 31 | its rank in that
                                          // stream's copy order; or null
  int n_chunks;
  const uint32_t* pull;                   // loader mode, overlapped replay: traces are
                                          // pulled in stored order (pull[k] = caller
                                          // trace of stored k); or null (caller order)
  uint32_t* stall;                        // overlapped mode: set when a chunk never lands
                                          // (or the replay gave up); every waiter bails
  const uint32_t* pull_count;             // with pull: the number of entries (device), or null
  uint32_t* loaded;                       // ... and each finished trace is appended to
                                          // a completion queue: loaded[n_traces] is its
                                          // tail, loaded[i] = stored index + 1 (release)
                                          // once its wire events and n_ids are written
};

__device__ __forceinline__ uint32_t hash_addr(uint64_t a, uint32_t bits) {
  return uint32_t((a * 0x9E3779B97F4A7C15ull) >> (64 - bits));
}

template <int kW>
__global__ void __launch_bounds__(32 * kW) k_reconstruct(LParams P) {
  const uint32_t lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const uint32_t slot = blockIdx.x * kW + (threadIdx.x >> 5);
  Slot* T = P.tables + (size_t(slot) << P.hbits);
  uint32_t* ids = P.idstacks + size_t(slot) * P.max_events;
  for (;;) {
    unsigned k = 0;
    if (lane == 0) k = atomicAdd(P.work, 1u);
    k = __shfl_sync(kFull, k, 0);
    if (int64_t(k) >= P.n_traces || (P.pull_count && k >= *P.pull_count)) break;
    const unsigned t = P.pull ? P.pull[k] : k;   // the caller's trace
    if (P.chunk_flag) {                     // wait until trace t's chunk has landed
      int lo = 0, hi = P.n_chunks - 1;      // the chunk c with first[c] <= t < first[c+1]
      while (lo < hi) {
        const int m = (lo + hi + 1) >> 1;
        if (P.chunk_first[m] <= t) lo = m; else hi = m - 1;
      }
      // chunk lo's copy stream (bit 31) and its rank in that stream's order
      const uint32_t cr = P.chunk_flag[2 + lo];
      const uint32_t need = cr & 0x7FFFFFFFu;
      const uint32_t* landed = P.chunk_flag + (cr >> 31);
      uint32_t nap = 256;
      unsigned long long t0 = 0;
      bool gave_up = false;
      for (;;) {
        uint32_t r = 0;
        if (lane == 0)
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(r) : "l"(landed) : "memory");
        if (__shfl_sync(kFull, r, 0) > need) break;   // chunks landed so far > its rank
        if (P.stall) {                      // overlapped: bounded wait (XM_LOADED_TIMEOUT_NS)
          unsigned long long now;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
          now = __shfl_sync(kFull, now, 0);
          const uint32_t sv = __shfl_sync(kFull, *(volatile uint32_t*)P.stall, 0);
          if (t0 == 0) t0 = now;
          if (sv != 0 || now - t0 > 4000000000ull) {
            if (lane == 0) atomicExch(P.stall, 1u);
            gave_up = true;
            break;
          }
        }
        __nanosleep(nap);
        nap = min(nap * 2, 4096u);
      }
      __syncwarp();
      if (gave_up) break;
    }
    const unsigned gen = t + 1;
    const int64_t e0 = P.off[t];
    const uint32_t sk = P.pull ? k : (P.wire_off ? P.pos[t] : 0u);
    const int64_t wire0 = P.wire_off ? P.wire_off[sk] : 0;
    const int n = int(P.off[t + 1] - e0);
    // this trace's table: the first 2^hb slots of the warp's region, 2^hb > n
    // (at most n distinct addresses, so a free slot always exists; with about
    // half the instants allocations and addresses reused, the load stays well
    // below 1/2 in practice); other traces' entries carry other generations
    uint32_t hb = 6;
    while ((1u << hb) < uint32_t(n) + 1u && hb < P.hbits) ++hb;
    const uint32_t hmask = (1u << hb) - 1u;
    // clear this trace's slots (16-byte stores), so no per-call memset of the
    // tables is needed
    for (uint32_t h = lane; h <= hmask; h += 32)
      reinterpret_cast<uint4*>(T)[h] = make_uint4(0u, 0u, 0u, 0u);
    __syncwarp();
    uint32_t top = 0, fresh = 0, max_open = 0, open = 0;
    unsigned long long n_blocks = 0, n_orphan = 0, n_mism = 0, n_matched = 0, n_kept = 0, n_inv = 0,
                       n_reopen = 0;
    // the tile's instants are loaded one tile ahead (registers), so a tile's
    // matching does not start behind its own loads
    const long long* __restrict__ ib = reinterpret_cast<const long long*>(P.bytes) + e0;
    const unsigned long long* __restrict__ ia =
        P.tag ? nullptr : reinterpret_cast<const unsigned long long*>(P.addr) + e0;
    const uint32_t* __restrict__ ig = P.tag ? P.tag + e0 : nullptr;
    const uint8_t* __restrict__ is = P.stream ? P.stream + e0 : nullptr;
    // (address or raw tag, bytes, stream) of instant i
#define XM_K5_LOAD(i, A, B, S)                                              \
    do {                                                                   \
      B = __ldcg(ib + (i));                                                \
      if (ig) {                                                            \
        const uint32_t g_ = __ldcg(ig + (i));                              \
        A = uint64_t(g_ & 0x0FFFFFFFu);                                    \
        S = g_ >> 28;                                                      \
      } else {                                                             \
        A = __ldcg(ia + (i));                                              \
        S = is ? uint32_t(__ldcg(is + (i))) : 0u;                          \
      }                                                                    \
    } while (0)
    uint64_t a_nx = 0;
    int64_t b_nx = 0;
    uint32_t s_nx = 0;
    if (int(lane) < n) XM_K5_LOAD(int(lane), a_nx, b_nx, s_nx);
    for (int base = 0; base < n; base += 32) {
      const int li = base + int(lane);
      const bool valid = li < n;
      uint64_t a = valid ? a_nx : ~0ull - lane;
      int64_t b = valid ? b_nx : 0;
      uint32_t s = valid ? s_nx : 0u;
      if (li + 32 < n) XM_K5_LOAD(li + 32, a_nx, b_nx, s_nx);
      // |bytes| >= XM_MAX_REQUEST is out of the replay's range: invalid like 0
      if (b >= int64_t(XM_MAX_REQUEST) || b <= -int64_t(XM_MAX_REQUEST)) b = 0;
      const bool is_alloc = b > 0, is_free = b < 0;
      // ---- dense ids for this tile's allocations (ids freed before the tile) ----
      const unsigned am = __ballot_sync(kFull, is_alloc);
      const uint32_t na = __popc(am), ka = __popc(am & lt);
      const uint32_t take = min(na, top);
      uint32_t my_tag = 0;                  // an allocation's dense id | stream << 28
      if (is_alloc) {
        const uint32_t id = ka < take ? ids[top - 1 - ka] : fresh + (ka - take);
        my_tag = id | (s << 28);
        if (P.partner) {
          P.partner[e0 + li] = -1;
          P.mismatch[e0 + li] = 0;
        }
      }
      top -= take;
      fresh += na - take;
      __syncwarp();
      // ---- matching (LIFO per address) ----
      bool matched = false, reopened = false;
      int blk = -1;
      uint32_t blk_tag = 0;                 // the matched allocation's record
      long long blk_bytes = 0;
      // Lanes with the same address form a group; its instants must be
      // applied in time order, different addresses touch different keys. So
      // round r applies every group's r-th instant at once (one round when
      // the tile's addresses are distinct, the common case).
      const unsigned grp = __match_any_sync(kFull, a);
      const uint32_t my_rank = __popc(grp & lt);
      const uint32_t rounds = __reduce_max_sync(kFull, valid ? uint32_t(__popc(grp)) : 0u);
      for (uint32_t r = 0; r < rounds; ++r) {
        const bool act = valid && b != 0 && my_rank == r;
        // read phase: find my key or the first free slot of my probe sequence
        uint32_t h = hash_addr(a, hb);
        bool found = false;
        if (act) {
          for (;;) {
            if (T[h].gen != gen) break;
            if (T[h].addr == a) { found = true; break; }
            h = (h + 1) & hmask;
          }
        }
        // claim phase for allocations at new addresses: lanes aiming at the
        // same free slot -> the lowest wins, the others probe on
        bool pend = act && is_alloc && !found;
        while (__any_sync(kFull, pend)) {
          const unsigned same = __match_any_sync(kFull, pend ? h : 0xFFFFFFFFu);
          const bool win = pend && (__ffs(same) - 1) == int(lane);
          __syncwarp();
          if (win) { T[h].addr = a; T[h].gen = gen; T[h].top = -1; }
          __syncwarp();
          if (pend && !win) {
            h = (h + 1) & hmask;
            for (;;) {                       // next free slot (or, never, my key)
              if (T[h].gen != gen) break;
              h = (h + 1) & hmask;
            }
          }
          pend = pend && !win;
        }
        __syncwarp();
        if (act) {
          if (is_alloc) {
            reopened = found && T[h].top >= 0;           // its address still has an open block
            // one 16-byte store / load per record
            const unsigned long long ub = static_cast<unsigned long long>(b);
            reinterpret_cast<int4*>(P.arec)[e0 + li] =
                make_int4(T[h].top, int(my_tag), int(uint32_t(ub)), int(uint32_t(ub >> 32)));
            T[h].top = li;
          } else if (found && T[h].top >= 0) {
            blk = T[h].top;
            const int4 r = reinterpret_cast<const int4*>(P.arec)[e0 + blk];
            T[h].top = r.x;
            blk_tag = uint32_t(r.y);
            blk_bytes = static_cast<long long>((static_cast<unsigned long long>(uint32_t(r.w)) << 32) |
                                               uint32_t(r.z));
            matched = true;
          }
        }
        __syncwarp();
      }
      __syncwarp();
      // ---- per-instant outputs ----
      bool mism = false;
      if (is_free && matched) mism = blk_bytes != -b;
      if (P.partner) {                      // (the loader mode needs the tallies only)
        if (is_free) {
          P.partner[e0 + li] = matched ? blk : -1;
          if (matched) P.partner[e0 + blk] = li;
          P.mismatch[e0 + li] = mism ? 1 : 0;
        } else if (valid && b == 0) {
          P.partner[e0 + li] = -1;
          P.mismatch[e0 + li] = 0;
        }
      }
      __syncwarp();
      // ---- matched blocks' ids go back on the stack ----
      const unsigned mm = __ballot_sync(kFull, matched);
      if (matched) ids[top + __popc(mm & lt)] = blk_tag & 0x0FFFFFFFu;
      top += __popc(mm);
      // ---- staging: kept events, compacted within the trace ----
      const bool kept = is_alloc || matched;
      const unsigned km = __ballot_sync(kFull, kept);
      if (kept) {
        // staging at the trace's input offset, or (direct wire output) at
        // its final place in the stored-order wire arrays
        const int64_t dst = (P.wire_off ? wire0 : e0) + int64_t(n_kept) + __popc(km & lt);
        if (is_alloc) {
          P.st_bytes[dst] = b;
          P.st_tag[dst] = my_tag;
        } else {
          P.st_bytes[dst] = -blk_bytes;                  // the block's size
          P.st_tag[dst] = blk_tag;                       // its id and stream
        }
      }
      // ---- open count (max open = the minimal id space) ----
      int d = is_alloc ? 1 : (matched ? -1 : 0);
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(kFull, d, o);
        if (int(lane) >= o) d += y;
      }
      const uint32_t mo = __reduce_max_sync(kFull, uint32_t(int(open) + d));
      max_open = max(max_open, mo);
      open = uint32_t(int(open) + __shfl_sync(kFull, d, 31));
      n_blocks += na;
      n_matched += __popc(mm);
      n_kept += __popc(km);
      n_orphan += __popc(__ballot_sync(kFull, is_free && !matched));
      n_mism += __popc(__ballot_sync(kFull, mism));
      n_inv += __popc(__ballot_sync(kFull, valid && b == 0));
      n_reopen += __popc(__ballot_sync(kFull, reopened));
      __syncwarp();
    }
    if (lane == 0) {
      xm_lifecycle r;
      r.n_blocks = n_blocks;
      r.n_orphan = n_orphan;
      r.n_mismatch = n_mism;
      r.n_persistent = n_blocks - n_matched;
      r.n_kept = n_kept;
      r.n_invalid = n_inv;
      r.max_open = max_open;
      r.n_ids = fresh;
      r.n_reopened = n_reopen;
      P.rec[t] = r;
      // direct wire output: a trace with any verdict (its wire events are not
      // the trace) gets n_ids 0, which the replay refuses (XM_T_INVALID)
      if (P.w_nids)
        P.w_nids[sk] = (n_orphan | n_mism | n_inv | n_reopen) || fresh > (1u << 27) ? 0u : fresh;
    }
    __syncwarp();
    if (P.loaded) {
      // publish: every lane's wire stores (and lane 0's n_ids) before the
      // queue entry
      __threadfence();
      __syncwarp();
      if (lane == 0) {
        const uint32_t at = atomicAdd(P.loaded + P.n_traces, 1u);
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(P.loaded + at), "r"(sk + 1u) : "memory");
      }
      __syncwarp();
    }
  }
}

// ---- k_reconstruct_smem: K5 with its per-trace state in shared memory --------
// The same matching as k_reconstruct (general mode: addresses, LIFO stacks per
// address, the same dense-id assignment and outputs), but each warp's hash
// table (address -> top open block), block records and free-id stack live in
// shared memory, so the probes and record reads are shared-memory round trips
// and the only global traffic is the instants, the per-instant outputs and
// the staging. Records are indexed by dense id (at most one open block per
// id): w0 = block below (id + 1, 0 none) | stream << 28, w1 = its event index,
// w2/w3 = its request bytes. The table is never cleared: a slot belongs to the
// current trace iff its generation does (a warp-local count, cleared once at
// start). A trace needing more than kSRecs dense ids or more than 3/4 of the
// table's slots stops and is queued (ovf) for k_reconstruct, which rewrites
// every output of it.
constexpr int kSW = 4;                      // warps per CTA (one CTA per SM)
constexpr uint32_t kSTable = 2048;          // table slots per warp (16 B)
constexpr uint32_t kSRecs = 1024;           // dense ids per warp (16 B records + 4 B stack)
constexpr size_t kSWarpBytes = size_t(kSTable) * 16 + size_t(kSRecs) * 20;
constexpr size_t kSSmem = kSW * kSWarpBytes;

__global__ void __launch_bounds__(32 * kSW, 1) k_reconstruct_smem(LParams P, uint32_t* ovf,
                                                                  uint32_t* ovf_count) {
  extern __shared__ __align__(16) unsigned char sm[];
  const uint32_t lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const uint32_t w = threadIdx.x >> 5;
  uint4* T = reinterpret_cast<uint4*>(sm + size_t(w) * kSWarpBytes);
  uint4* Rr = T + kSTable;
  uint32_t* ids = reinterpret_cast<uint32_t*>(Rr + kSRecs);
  for (uint32_t h = lane; h < kSTable; h += 32) T[h] = make_uint4(0u, 0u, 0u, 0u);
  __syncwarp();
  uint32_t gen = 0;
  const uint32_t hb = 11;                   // log2 kSTable
  const uint32_t hmask = kSTable - 1u;
  for (;;) {
    unsigned k = 0;
    if (lane == 0) k = atomicAdd(P.work, 1u);
    k = __shfl_sync(kFull, k, 0);
    if (int64_t(k) >= P.n_traces) break;
    const unsigned t = k;
    ++gen;
    const int64_t e0 = P.off[t];
    const int n = int(P.off[t + 1] - e0);
    uint32_t top = 0, fresh = 0, max_open = 0, open = 0, ndist = 0;
    bool overflow = false;
    unsigned long long n_blocks = 0, n_orphan = 0, n_mism = 0, n_matched = 0, n_kept = 0, n_inv = 0,
                       n_reopen = 0;
    const long long* __restrict__ ib = reinterpret_cast<const long long*>(P.bytes) + e0;
    const unsigned long long* __restrict__ ia = reinterpret_cast<const unsigned long long*>(P.addr) + e0;
    const uint32_t* __restrict__ ig = nullptr;
    const uint8_t* __restrict__ is = P.stream ? P.stream + e0 : nullptr;
    uint64_t a_nx = 0;
    int64_t b_nx = 0;
    uint32_t s_nx = 0;
    if (int(lane) < n) XM_K5_LOAD(int(lane), a_nx, b_nx, s_nx);
    for (int base = 0; base < n; base += 32) {
      const int li = base + int(lane);
      const bool valid = li < n;
      uint64_t a = valid ? a_nx : ~0ull - lane;
      int64_t b = valid ? b_nx : 0;
      uint32_t s = valid ? s_nx : 0u;
      if (li + 32 < n) XM_K5_LOAD(li + 32, a_nx, b_nx, s_nx);
      if (b >= int64_t(XM_MAX_REQUEST) || b <= -int64_t(XM_MAX_REQUEST)) b = 0;
      const bool is_alloc = b > 0, is_free = b < 0;
      // ---- dense ids for this tile's allocations (ids freed before the tile) ----
      const unsigned am = __ballot_sync(kFull, is_alloc);
      const uint32_t na = __popc(am), ka = __popc(am & lt);
      const uint32_t take = min(na, top);
      if (fresh + (na - take) > kSRecs) { overflow = true; break; }   // (warp-uniform)
      uint32_t my_id = 0, my_tag = 0;
      if (is_alloc) {
        my_id = ka < take ? ids[top - 1 - ka] : fresh + (ka - take);
        my_tag = my_id | (s << 28);
        P.partner[e0 + li] = -1;
        P.mismatch[e0 + li] = 0;
      }
      top -= take;
      fresh += na - take;
      __syncwarp();
      // ---- matching (LIFO per address), rounds as in k_reconstruct ----
      bool matched = false, reopened = false;
      int blk = -1;
      uint32_t blk_tag = 0;
      long long blk_bytes = 0;
      const unsigned grp = __match_any_sync(kFull, a);
      const uint32_t my_rank = __popc(grp & lt);
      const uint32_t rounds = __reduce_max_sync(kFull, valid ? uint32_t(__popc(grp)) : 0u);
      for (uint32_t r = 0; r < rounds; ++r) {
        const bool act = valid && b != 0 && my_rank == r;
        uint32_t h = hash_addr(a, hb);
        bool found = false;
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        if (act) {
          for (;;) {
            v = T[h];
            if (v.w != gen) break;
            if ((uint64_t(v.y) << 32 | v.x) == a) { found = true; break; }
            h = (h + 1) & hmask;
          }
        }
        bool pend = act && is_alloc && !found;
        ndist += __popc(__ballot_sync(kFull, pend));
        if (ndist > kSTable / 4 * 3) { overflow = true; break; }   // (warp-uniform)
        while (__any_sync(kFull, pend)) {
          const unsigned same = __match_any_sync(kFull, pend ? h : 0xFFFFFFFFu);
          const bool win = pend && (__ffs(same) - 1) == int(lane);
          __syncwarp();
          if (win) T[h] = make_uint4(uint32_t(a), uint32_t(a >> 32), 0u, gen);
          __syncwarp();
          if (pend && !win) {
            h = (h + 1) & hmask;
            for (;;) {
              if (T[h].w != gen) break;
              h = (h + 1) & hmask;
            }
          }
          pend = pend && !win;
        }
        __syncwarp();
        if (act) {
          const uint32_t tp = found ? v.z : 0u;          // top open block (id + 1)
          if (is_alloc) {
            reopened = tp != 0u;
            const unsigned long long ub = static_cast<unsigned long long>(b);
            Rr[my_id] = make_uint4(tp | (s << 28), uint32_t(li), uint32_t(ub), uint32_t(ub >> 32));
            T[h].z = my_id + 1u;
          } else if (tp != 0u) {
            const uint4 rr = Rr[tp - 1u];
            T[h].z = rr.x & 0x0FFFFFFFu;
            blk = int(rr.y);
            blk_tag = (tp - 1u) | (rr.x & 0xF0000000u);
            blk_bytes = static_cast<long long>((static_cast<unsigned long long>(rr.w) << 32) | rr.z);
            matched = true;
          }
        }
        __syncwarp();
      }
      if (overflow) break;
      __syncwarp();
      // ---- per-instant outputs ----
      bool mism = false;
      if (is_free && matched) mism = blk_bytes != -b;
      if (is_free) {
        P.partner[e0 + li] = matched ? blk : -1;
        if (matched) P.partner[e0 + blk] = li;
        P.mismatch[e0 + li] = mism ? 1 : 0;
      } else if (valid && b == 0) {
        P.partner[e0 + li] = -1;
        P.mismatch[e0 + li] = 0;
      }
      __syncwarp();
      // ---- matched blocks' ids go back on the stack ----
      const unsigned mm = __ballot_sync(kFull, matched);
      if (matched) ids[top + __popc(mm & lt)] = blk_tag & 0x0FFFFFFFu;
      top += __popc(mm);
      // ---- staging: kept events, compacted within the trace ----
      const bool kept = is_alloc || matched;
      const unsigned km = __ballot_sync(kFull, kept);
      if (kept) {
        const int64_t dst = e0 + int64_t(n_kept) + __popc(km & lt);
        if (is_alloc) {
          P.st_bytes[dst] = b;
          P.st_tag[dst] = my_tag;
        } else {
          P.st_bytes[dst] = -blk_bytes;
          P.st_tag[dst] = blk_tag;
        }
      }
      int d = is_alloc ? 1 : (matched ? -1 : 0);
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(kFull, d, o);
        if (int(lane) >= o) d += y;
      }
      const uint32_t mo = __reduce_max_sync(kFull, uint32_t(int(open) + d));
      max_open = max(max_open, mo);
      open = uint32_t(int(open) + __shfl_sync(kFull, d, 31));
      n_blocks += na;
      n_matched += __popc(mm);
      n_kept += __popc(km);
      n_orphan += __popc(__ballot_sync(kFull, is_free && !matched));
      n_mism += __popc(__ballot_sync(kFull, mism));
      n_inv += __popc(__ballot_sync(kFull, valid && b == 0));
      n_reopen += __popc(__ballot_sync(kFull, reopened));
      __syncwarp();
    }
    __syncwarp();
    if (overflow) {                          // k_reconstruct redoes this trace
      if (lane == 0) ovf[atomicAdd(ovf_count, 1u)] = t;
      __syncwarp();
      continue;
    }
    if (lane == 0) {
      xm_lifecycle r;
      r.n_blocks = n_blocks;
      r.n_orphan = n_orphan;
      r.n_mismatch = n_mism;
      r.n_persistent = n_blocks - n_matched;
      r.n_kept = n_kept;
      r.n_invalid = n_inv;
      r.max_open = max_open;
      r.n_ids = fresh;
      r.n_reopened = n_reopen;
      P.rec[t] = r;
    }
    __syncwarp();
  }
}

#undef XM_K5_LOAD

// ---- k_load: the device loader of xm_simulate_raw ------------------------------
// The loader mode of k_reconstruct, specialised: the key is the raw block id,
// and a valid trace has at most one open block per key, so
// the hash slot itself holds the open block's record -- no per-allocation
// records, no stacks of blocks per key -- and a valid trace keeps every event,
// so event i's wire form goes straight to wire0 + i. The next tile's events
// are loaded while the current one is matched. Slot (16 B, one load per probe
// step): w0 raw id, w1 generation (trace + 1, 24 bits) | request bits 32-39
// << 24, w2 dense id | stream << 28, w3 request bits 0-31; open iff the
// request is nonzero (a close stores 0). Verdicts and tallies as k_reconstruct
// (invalid: zero or >= 2^40 bytes; reopened: alloc of an open id; orphan: free
// of a key with no open block; mismatch: free bytes != the alloc's).
template <int kW>
__global__ void __launch_bounds__(32 * kW) k_load(LParams P) {
  const uint32_t lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const uint32_t slot = blockIdx.x * kW + (threadIdx.x >> 5);
  uint4* T = reinterpret_cast<uint4*>(P.tables + (size_t(slot) << P.hbits));
  uint32_t* ids = P.idstacks + size_t(slot) * P.max_events;
  const long long* by = reinterpret_cast<const long long*>(P.bytes);
  for (;;) {
    unsigned k = 0;
    if (lane == 0) k = atomicAdd(P.work, 1u);
    k = __shfl_sync(kFull, k, 0);
    if (int64_t(k) >= P.n_traces) break;
    const unsigned t = P.pull ? P.pull[k] : k;   // the caller's trace
    if (P.chunk_flag) {                     // wait until trace t's chunk has landed
      int lo = 0, hi = P.n_chunks - 1;
      while (lo < hi) {
        const int m = (lo + hi + 1) >> 1;
        if (P.chunk_first[m] <= t) lo = m; else hi = m - 1;
      }
      // chunk lo's copy stream (bit 31) and its rank in that stream's order
      const uint32_t cr = P.chunk_flag[2 + lo];
      const uint32_t need = cr & 0x7FFFFFFFu;
      const uint32_t* landed = P.chunk_flag + (cr >> 31);
      uint32_t nap = 256;
      unsigned long long t0 = 0;
      bool gave_up = false;
      for (;;) {
        uint32_t r = 0;
        if (lane == 0)
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(r) : "l"(landed) : "memory");
        if (__shfl_sync(kFull, r, 0) > need) break;   // chunks landed so far > its rank
        if (P.stall) {                      // overlapped: bounded wait
          unsigned long long now;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
          now = __shfl_sync(kFull, now, 0);
          const uint32_t sv = __shfl_sync(kFull, *(volatile uint32_t*)P.stall, 0);
          if (t0 == 0) t0 = now;
          if (sv != 0 || now - t0 > 4000000000ull) {
            if (lane == 0) atomicExch(P.stall, 1u);
            gave_up = true;
            break;
          }
        }
        __nanosleep(nap);
        nap = min(nap * 2, 4096u);
      }
      __syncwarp();
      if (gave_up) break;
    }
    const uint32_t gen = (t + 1u) & 0xFFFFFFu;    // the host keeps T < 2^24 here
    const int64_t e0 = P.off[t];
    const uint32_t sk = P.pull ? k : P.pos[t];
    const int64_t wire0 = P.wire_off[sk];
    const int n = int(P.off[t + 1] - e0);
    uint32_t hb = 6;
    while ((1u << hb) < uint32_t(n) + 1u && hb < P.hbits) ++hb;
    const uint32_t hmask = (1u << hb) - 1u;
    for (uint32_t h = lane; h <= hmask; h += 32) T[h] = make_uint4(0u, 0u, 0u, 0u);
    __syncwarp();
    uint32_t top = 0, fresh = 0, max_open = 0, open = 0;
    unsigned long long n_blocks = 0, n_orphan = 0, n_mism = 0, n_matched = 0, n_inv = 0, n_reopen = 0;
    // the first tile's events; each tile loads the next one's
    long long b_nx = 0;
    uint32_t g_nx = 0;
    if (int(lane) < n) {
      b_nx = __ldcg(by + e0 + lane);
      g_nx = __ldcg(P.tag + e0 + lane);
    }
    for (int base = 0; base < n; base += 32) {
      const int li = base + int(lane);
      const bool valid = li < n;
      long long b = b_nx;
      const uint32_t g = g_nx;
      if (li + 32 < n) {
        b_nx = __ldcg(by + e0 + li + 32);
        g_nx = __ldcg(P.tag + e0 + li + 32);
      }
      if (b >= (long long)(XM_MAX_REQUEST) || b <= -(long long)(XM_MAX_REQUEST)) b = 0;
      const uint32_t key = valid ? (g & 0x0FFFFFFFu) : (0xF0000000u | lane);   // never a raw id
      const uint32_t s = g >> 28;
      const bool is_alloc = valid && b > 0, is_free = valid && b < 0;
      // ---- dense ids for this tile's allocations (ids freed before the tile) ----
      const unsigned am = __ballot_sync(kFull, is_alloc);
      const uint32_t na = __popc(am), ka = __popc(am & lt);
      const uint32_t take = min(na, top);
      uint32_t my_tag = 0;
      XM_CHECK(top <= P.max_events, "k_load: id stack %u > %u\n", top, P.max_events);
      if (is_alloc) my_tag = (ka < take ? ids[top - 1 - ka] : fresh + (ka - take)) | (s << 28);
      top -= take;
      fresh += na - take;
      __syncwarp();
      // ---- matching: one open block per key; a key's instants in this tile
      // are applied in time order (round r: every key's r-th instant) ----
      bool matched = false, reopened = false, mism = false;
      uint32_t blk_tag = 0;
      const unsigned grp = __match_any_sync(kFull, key);
      const uint32_t my_rank = __popc(grp & lt);
      const uint32_t rounds = __reduce_max_sync(kFull, valid ? uint32_t(__popc(grp)) : 0u);
      const unsigned long long ub = static_cast<unsigned long long>(b);
      for (uint32_t r = 0; r < rounds; ++r) {
        const bool act = valid && b != 0 && my_rank == r;
        uint32_t h = hash_addr(key, hb);
        bool found = false;
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        if (act) {
          uint32_t steps = 0;
          (void)steps;
          for (;;) {                         // read phase: my key or the first free slot
            XM_CHECK(++steps <= hmask + 1u, "k_load: probe wrapped the table (2^%u slots)\n", hb);
            v = T[h];
            if ((v.y & 0xFFFFFFu) != gen) break;
            if (v.x == key) { found = true; break; }
            h = (h + 1) & hmask;
          }
        }
        // claim phase for allocations of new keys: lanes aiming at the same
        // free slot -> the lowest wins, the others probe on
        bool pend = act && is_alloc && !found;
        while (__any_sync(kFull, pend)) {
          const unsigned same = __match_any_sync(kFull, pend ? h : 0xFFFFFFFFu);
          const bool win = pend && (__ffs(same) - 1) == int(lane);
          __syncwarp();
          if (win) T[h] = make_uint4(key, gen | (uint32_t(ub >> 32) << 24), my_tag, uint32_t(ub));
          __syncwarp();
          if (pend && !win) {
            h = (h + 1) & hmask;
            for (;;) {
              if ((T[h].y & 0xFFFFFFu) != gen) break;
              h = (h + 1) & hmask;
            }
          }
          pend = pend && !win;
        }
        __syncwarp();
        if (act) {
          const bool is_open = found && ((v.y >> 24) | v.w) != 0u;
          if (is_alloc) {
            if (found) {                      // a known key: (re)opened with this block
              reopened = is_open;
              T[h] = make_uint4(key, gen | (uint32_t(ub >> 32) << 24), my_tag, uint32_t(ub));
            }
          } else if (is_open) {
            matched = true;
            blk_tag = v.z;
            const unsigned long long ab = (static_cast<unsigned long long>(v.y >> 24) << 32) | v.w;
            mism = ab != static_cast<unsigned long long>(-b);
            T[h] = make_uint4(key, gen, v.z, 0u);    // closed
          }
        }
        __syncwarp();
      }
      __syncwarp();
      // ---- matched blocks' ids go back on the stack ----
      const unsigned mm = __ballot_sync(kFull, matched);
      if (matched) ids[top + __popc(mm & lt)] = blk_tag & 0x0FFFFFFFu;
      top += __popc(mm);
      XM_CHECK(top <= P.max_events, "k_load: id stack %u > %u\n", top, P.max_events);
      // ---- the wire event in place (a valid trace keeps every event) ----
      XM_CHECK(!valid || wire0 + li < P.wire_off[sk + 1], "k_load: wire index past trace %u\n", sk);
      if (valid) {
        P.st_bytes[wire0 + li] = b;
        P.st_tag[wire0 + li] = is_alloc ? my_tag : blk_tag;
      }
      // ---- open count and tallies ----
      int d = is_alloc ? 1 : (matched ? -1 : 0);
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(kFull, d, o);
        if (int(lane) >= o) d += y;
      }
      const uint32_t mo = __reduce_max_sync(kFull, uint32_t(int(open) + d));
      max_open = max(max_open, mo);
      open = uint32_t(int(open) + __shfl_sync(kFull, d, 31));
      n_blocks += na;
      n_matched += __popc(mm);
      n_orphan += __popc(__ballot_sync(kFull, is_free && !matched));
      n_mism += __popc(__ballot_sync(kFull, mism));
      n_inv += __popc(__ballot_sync(kFull, valid && b == 0));
      n_reopen += __popc(__ballot_sync(kFull, reopened));
      __syncwarp();
    }
    if (lane == 0) {
      xm_lifecycle r;
      r.n_blocks = n_blocks;
      r.n_orphan = n_orphan;
      r.n_mismatch = n_mism;
      r.n_persistent = n_blocks - n_matched;
      r.n_kept = n_blocks + n_matched;
      r.n_invalid = n_inv;
      r.max_open = max_open;
      r.n_ids = fresh;
      r.n_reopened = n_reopen;
      P.rec[t] = r;
      P.w_nids[sk] = (n_orphan | n_mism | n_inv | n_reopen) || fresh > (1u << 27) ? 0u : fresh;
    }
    __syncwarp();
    if (P.loaded) {                         // publish (see k_reconstruct)
      __threadfence();
      __syncwarp();
      if (lane == 0) {
        const uint32_t at = atomicAdd(P.loaded + P.n_traces, 1u);
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(P.loaded + at), "r"(sk + 1u) : "memory");
      }
      __syncwarp();
    }
  }
}

// exclusive scan of rec[order[k]].n_kept over stored k -> woff[T+1] (one CTA)
__global__ void __launch_bounds__(1024) k_wire_offsets(const xm_lifecycle* rec,
                                                       const uint32_t* order, int64_t T,
                                                       int64_t* woff) {
  __shared__ long long part[1024];
  const int tid = threadIdx.x;
  const int64_t per = (T + 1023) / 1024;
  const int64_t a = min(T, int64_t(tid) * per), z = min(T, a + per);
  long long s = 0;
  for (int64_t t = a; t < z; ++t) s += (long long)rec[order ? order[t] : t].n_kept;
  part[tid] = s;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {            // Hillis-Steele inclusive scan
    const long long v = tid >= o ? part[tid - o] : 0;
    __syncthreads();
    part[tid] += v;
    __syncthreads();
  }
  long long run = part[tid] - s;
  for (int64_t t = a; t < z; ++t) {
    woff[t] = run;
    run += (long long)rec[order ? order[t] : t].n_kept;
  }
  if (tid == 1023) woff[T] = part[1023];
}

__global__ void k_wire_compact(const int64_t* __restrict__ off, const int64_t* __restrict__ woff,
                               const xm_lifecycle* __restrict__ rec, const uint32_t* order,
                               const int64_t* st_bytes, const uint32_t* st_tag, int64_t T,
                               int64_t* w_bytes, uint32_t* w_tag, uint32_t* w_nids) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t k = w0; k < T; k += nw) {               // stored trace k
    const int64_t t = order ? order[k] : k;
    const int64_t src = off[t], dst = woff[k], m = woff[k + 1] - dst;
    for (int64_t j = lane; j < m; j += 32) {
      w_bytes[dst + j] = st_bytes[src + j];
      w_tag[dst + j] = st_tag[src + j];
    }
    if (lane == 0) w_nids[k] = rec[t].n_ids;
  }
}

struct Layout {
  uint32_t hbits, n_slots, ctas;
  size_t tables, stacks, arec, st_bytes, st_tag, ovf, total;
};

Layout layout(const xm_instants* in) {
  Layout L{};
  int dev = 0, sms = 148;
  if (xm_internal::cuda_usable() && cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaGetLastError();
  const int64_t want_ctas = (in->n_traces + kWarps - 1) / kWarps;
  uint32_t hb = 6;
  while ((1ull << hb) < uint64_t(in->max_events) + 1) ++hb;
  L.hbits = hb;
  // as many CTAs as fit (kCtasPerSm per SM) within a 2 GiB budget for the
  // per-warp hash tables (long traces -> fewer, larger tables)
  const int64_t per_cta = int64_t(kWarps) * int64_t(sizeof(Slot)) << hb;
  const int64_t budget_ctas = std::max<int64_t>(1, (int64_t(2) << 30) / per_cta);
  const int64_t cap_ctas = std::min<int64_t>(int64_t(sms) * kCtasPerSm, budget_ctas);
  L.ctas = uint32_t(want_ctas < cap_ctas ? (want_ctas > 0 ? want_ctas : 1) : cap_ctas);
  if (const char* v = getenv("XM_K5_CTAS")) {        // tooling: cap the concurrency
    const long c = strtol(v, nullptr, 10);
    if (c > 0 && uint32_t(c) < L.ctas) L.ctas = uint32_t(c);
  }
  L.n_slots = L.ctas * kWarps;
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  size_t o = 256;                                   // header: work counter
  L.tables = o; o += al((size_t(L.n_slots) << hb) * sizeof(Slot));
  L.stacks = o; o += al(size_t(L.n_slots) * (in->max_events ? in->max_events : 1) * 4);
  const size_t E = size_t(in->n_events > 0 ? in->n_events : 1);
  L.arec = o; o += al(E * sizeof(ARec));
  L.st_bytes = o; o += al(E * 8);
  L.st_tag = o; o += al(E * 4);
  L.ovf = o; o += al(size_t(in->n_traces > 0 ? in->n_traces : 1) * 4);   // k_reconstruct_smem overflow
  L.total = o;
  return L;
}

}  // namespace

using namespace xm_internal;

extern "C" size_t xm_reconstruct_scratch_bytes(const xm_instants* in) {
  if (!in || in->n_traces < 0 || in->n_events < 0) return 0;
  return layout(in).total;
}

extern "C" int xm_reconstruct(const xm_instants* in, void* d_scratch, size_t scratch_bytes,
                              int32_t* d_partner, uint8_t* d_mismatch, xm_lifecycle* d_rec,
                              void* stream) {
  launch_counter() = 0;
  if (!in || in->n_traces < 0 || in->n_events < 0)
    return set_error(XM_EINVAL, "xm_reconstruct: bad arguments");
  if (in->n_events > 0x7FFFFFFFll || in->max_events > 0x7FFFFFFFu)
    return set_error(XM_ERANGE, "xm_reconstruct: trace longer than 2^31-1 instants");
  if (in->n_traces == 0) return XM_OK;
  if (!in->off || (in->n_events > 0 && (!in->addr || !in->bytes)) || !d_partner || !d_mismatch ||
      !d_rec || !d_scratch)
    return set_error(XM_EINVAL, "xm_reconstruct: null pointer");
  const Layout L = layout(in);
  if (scratch_bytes < L.total) return set_error(XM_ENOMEM, "xm_reconstruct: scratch too small");
  if (!cuda_usable()) return set_error(XM_ECUDA, "no CUDA device");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char* base = static_cast<char*>(d_scratch);
  // zero the header (work counter); each warp clears its table per trace
  cudaError_t e = cudaMemsetAsync(base, 0, 256, st);
  if (e != cudaSuccess) return set_error(XM_ECUDA, cudaGetErrorString(e));
  LParams P{};
  P.addr = in->addr;
  P.bytes = in->bytes;
  P.stream = in->stream;
  P.off = in->off;
  P.n_traces = in->n_traces;
  P.hbits = L.hbits;
  P.tables = reinterpret_cast<Slot*>(base + L.tables);
  P.idstacks = reinterpret_cast<uint32_t*>(base + L.stacks);
  P.max_events = in->max_events ? in->max_events : 1;
  P.arec = reinterpret_cast<ARec*>(base + L.arec);
  P.st_bytes = reinterpret_cast<int64_t*>(base + L.st_bytes);
  P.st_tag = reinterpret_cast<uint32_t*>(base + L.st_tag);
  P.partner = d_partner;
  P.mismatch = d_mismatch;
  P.rec = d_rec;
  P.work = reinterpret_cast<unsigned int*>(base);
  // XM_K5=smem: the shared-memory pass first (one CTA per SM), then
  // k_reconstruct over the traces it could not hold (header word 1 counts
  // them, word 2 is the second pass's work counter)
  const char* k5 = getenv("XM_K5");
  if (k5 && k5[0] == 's') {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    e = cudaFuncSetAttribute(k_reconstruct_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSSmem));
    if (e != cudaSuccess) return set_error(XM_ECUDA, std::string("xm_reconstruct: ") + cudaGetErrorString(e));
    uint32_t* hdr = reinterpret_cast<uint32_t*>(base);
    uint32_t* ovf = reinterpret_cast<uint32_t*>(base + L.ovf);
    const int64_t g = std::min<int64_t>(sms, (in->n_traces + kSW - 1) / kSW);
    k_reconstruct_smem<<<unsigned(g > 0 ? g : 1), 32 * kSW, kSSmem, st>>>(P, ovf, hdr + 1);
    LParams Q = P;
    Q.pull = ovf;
    Q.pull_count = hdr + 1;
    Q.work = hdr + 2;
    k_reconstruct<kWarps><<<L.ctas, 32 * kWarps, 0, st>>>(Q);
    launch_counter() = 2;
  } else {
    k_reconstruct<kWarps><<<L.ctas, 32 * kWarps, 0, st>>>(P);
    launch_counter() = 1;
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(XM_ECUDA, std::string("xm_reconstruct: ") + cudaGetErrorString(e));
  return XM_OK;
}

extern "C" int xm_reconstruct_wire(const xm_instants* in, const void* d_scratch,
                                   size_t scratch_bytes, const xm_lifecycle* d_rec,
                                   const uint32_t* d_order, int64_t* d_wire_bytes,
                                   uint32_t* d_wire_tag, int64_t* d_wire_off,
                                   uint32_t* d_wire_nids, void* stream) {
  launch_counter() = 0;
  if (!in || in->n_traces < 0 || in->n_events < 0)
    return set_error(XM_EINVAL, "xm_reconstruct_wire: bad arguments");
  if (in->n_traces == 0) return XM_OK;
  if (!in->off || !d_rec || !d_scratch || !d_wire_bytes || !d_wire_tag || !d_wire_off || !d_wire_nids)
    return set_error(XM_EINVAL, "xm_reconstruct_wire: null pointer");
  const Layout L = layout(in);
  if (scratch_bytes < L.total) return set_error(XM_ENOMEM, "xm_reconstruct_wire: scratch too small");
  if (!cuda_usable()) return set_error(XM_ECUDA, "no CUDA device");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const char* base = static_cast<const char*>(d_scratch);
  k_wire_offsets<<<1, 1024, 0, st>>>(d_rec, d_order, in->n_traces, d_wire_off);
  const int64_t want = (in->n_traces + 7) / 8;
  const int g = int(want < int64_t(L.ctas) * 8 ? want : int64_t(L.ctas) * 8);
  k_wire_compact<<<g > 0 ? g : 1, 256, 0, st>>>(
      in->off, d_wire_off, d_rec, d_order, reinterpret_cast<const int64_t*>(base + L.st_bytes),
      reinterpret_cast<const uint32_t*>(base + L.st_tag), in->n_traces, d_wire_bytes, d_wire_tag,
      d_wire_nids);
  launch_counter() = 2;
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(XM_ECUDA, std::string("xm_reconstruct_wire: ") + cudaGetErrorString(e));
  return XM_OK;
}

// ---- reconstruction -> orchestrator input --------------------------------------
namespace {

// One warp per trace: the blocks of trace t in allocation order at
// boff[t] + ordinal: allocation time, free time (-1 = persistent), size,
// stream -- the Analyzer's block list for xm_orchestrate.
__global__ void k_blocks(const int64_t* __restrict__ ts, const int64_t* __restrict__ bytes,
                         const uint8_t* __restrict__ stream, const int64_t* __restrict__ off,
                         const int32_t* __restrict__ partner, const int64_t* __restrict__ boff,
                         int64_t T, int64_t* a_ts, int64_t* f_ts, int64_t* size, uint8_t* st) {
  const unsigned lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const int64_t w0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t t = w0; t < T; t += nw) {
    const int64_t e0 = off[t];
    const int n = int(off[t + 1] - e0);
    int64_t ord = boff[t];
    for (int base = 0; base < n; base += 32) {
      const int i = base + int(lane);
      const int64_t b = i < n ? bytes[e0 + i] : 0;
      const bool al = b > 0;
      const unsigned am = __ballot_sync(0xFFFFFFFFu, al);
      if (al) {
        const int64_t o = ord + __popc(am & lt);
        const int p = partner[e0 + i];
        a_ts[o] = ts[e0 + i];
        f_ts[o] = p >= 0 ? ts[e0 + p] : -1;
        size[o] = b;
        st[o] = stream ? stream[e0 + i] : 0;
      }
      ord += __popc(am);
    }
  }
}

}  // namespace

extern "C" int xm_blocks_from_instants(const xm_instants* in, const int64_t* d_ts,
                                       const int32_t* d_partner, const int64_t* d_boff,
                                       int64_t* d_alloc_ts, int64_t* d_free_ts, int64_t* d_size,
                                       uint8_t* d_stream, void* stream) {
  launch_counter() = 0;
  if (!in || in->n_traces < 0) return set_error(XM_EINVAL, "xm_blocks_from_instants: bad arguments");
  if (in->n_traces == 0) return XM_OK;
  if (!in->off || !d_boff || (in->n_events > 0 && (!in->bytes || !d_ts || !d_partner)) ||
      !d_alloc_ts || !d_free_ts || !d_size || !d_stream)
    return set_error(XM_EINVAL, "xm_blocks_from_instants: null pointer");
  if (!cuda_usable()) return set_error(XM_ECUDA, "no CUDA device");
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (in->n_traces + 7) / 8;
  const int g = int(std::min<int64_t>(std::max<int64_t>(want, 1), int64_t(sms) * 8));
  k_blocks<<<g, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      d_ts, in->bytes, in->stream, in->off, d_partner, d_boff, in->n_traces, d_alloc_ts, d_free_ts,
      d_size, d_stream);
  launch_counter() = 1;
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(XM_ECUDA, std::string("k_blocks: ") + cudaGetErrorString(e));
  return XM_OK;
}

// ---- device loader (xm_simulate_raw): K5 keyed by raw block ids ------------------
namespace xm_internal {

// Loads the loader kernels' module now (see preload_replay).
int preload_loader() {
  cudaFuncAttributes a;
  cudaError_t e = cudaFuncGetAttributes(&a, k_reconstruct<32>);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, k_reconstruct<kWarps>);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, k_load<32>);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, k_load<kWarps>);
  return int(e);
}

// Scratch of the loader mode for T traces / E events / the longest trace.
size_t loader_scratch_bytes(int64_t T, int64_t E, uint32_t max_events) {
  xm_instants in{};
  in.n_traces = T;
  in.n_events = E;
  in.max_events = max_events;
  return layout(&in).total;
}

// Validation + dense renumbering of raw traces on the device: k_reconstruct with
// the raw block id as the matching key (one open block per id in a valid trace,
// SPEC.md:249/258), tallies only (no partner output), then the wire arrays
// stored in `d_order`. A trace is valid iff its n_orphan, n_mismatch, n_invalid
// and n_reopened are 0; then its wire form is the trace itself with dense ids.
int launch_loader(const int64_t* d_bytes, const uint32_t* d_tag, const int64_t* d_off, int64_t T,
                  int64_t E, uint32_t max_events, void* d_scratch, xm_lifecycle* d_rec,
                  const uint32_t* d_order, int64_t* w_bytes, uint32_t* w_tag, int64_t* w_off,
                  uint32_t* w_nids, void* stream, int* n_launches, const uint32_t* chunk_first,
                  const uint32_t* chunk_flag, int n_chunks, const uint32_t* d_pos,
                  uint32_t* loaded, int loader_sms, uint32_t* stall) {
  xm_instants in{};
  in.n_traces = T;
  in.n_events = E;
  in.max_events = max_events;
  in.off = d_off;
  in.bytes = d_bytes;
  const Layout L = layout(&in);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char* base = static_cast<char*>(d_scratch);
  cudaError_t e = cudaMemsetAsync(base, 0, 256, st);
  if (e != cudaSuccess) return int(e);
  LParams P{};
  P.tag = d_tag;
  P.bytes = d_bytes;
  P.off = d_off;
  P.n_traces = T;
  P.hbits = L.hbits;
  P.tables = reinterpret_cast<Slot*>(base + L.tables);
  P.idstacks = reinterpret_cast<uint32_t*>(base + L.stacks);
  P.max_events = max_events ? max_events : 1;
  P.arec = reinterpret_cast<ARec*>(base + L.arec);
  P.st_bytes = reinterpret_cast<int64_t*>(base + L.st_bytes);
  P.st_tag = reinterpret_cast<uint32_t*>(base + L.st_tag);
  P.rec = d_rec;
  P.work = reinterpret_cast<unsigned int*>(base);
  if (d_pos) {                                      // direct wire output (w_off given)
    P.wire_off = w_off;
    P.pos = d_pos;
    P.w_nids = w_nids;
    P.st_bytes = w_bytes;
    P.st_tag = w_tag;
  }
  P.chunk_first = chunk_first;
  P.chunk_flag = chunk_flag;
  P.n_chunks = n_chunks;
  // k_load where it applies (direct wire output, generations fit 24 bits;
  // XM_LOADER=k5 forces k_reconstruct, tooling), else k_reconstruct
  const char* lk = std::getenv("XM_LOADER");
  const bool lean = d_pos && T < (int64_t(1) << 24) && !(lk && lk[0] == 'k');
  if (loaded && d_pos) {
    // overlapped with the replay (xm_simulate_raw): pulled in stored order,
    // each finished trace appended to the completion queue, on `loader_sms`
    // SMs -- one 32-warp CTA per SM (a whole SM's registers: no replay CTA
    // fits beside it, nor a second one)
    P.pull = d_order;
    P.loaded = loaded;
    P.stall = stall;
    const uint32_t g = std::min<uint32_t>(uint32_t(std::max(loader_sms, 1)), L.n_slots / 32);
    if (g >= 1) {
      if (lean) k_load<32><<<g, 32 * 32, 0, st>>>(P);
      else k_reconstruct<32><<<g, 32 * 32, 0, st>>>(P);
    } else {
      if (lean) k_load<kWarps><<<1, 32 * kWarps, 0, st>>>(P);
      else k_reconstruct<kWarps><<<1, 32 * kWarps, 0, st>>>(P);
    }
    *n_launches += 1;
    return int(cudaGetLastError());
  }
  if (lean) {
    k_load<kWarps><<<L.ctas, 32 * kWarps, 0, st>>>(P);
    *n_launches += 1;
    return int(cudaGetLastError());
  }
  k_reconstruct<kWarps><<<L.ctas, 32 * kWarps, 0, st>>>(P);
  if (d_pos) {                                      // written in place: no compaction
    *n_launches += 1;
    return int(cudaGetLastError());
  }
  k_wire_offsets<<<1, 1024, 0, st>>>(d_rec, d_order, T, w_off);
  const int64_t want = (T + 7) / 8;
  const int g = int(want < int64_t(L.ctas) * 8 ? want : int64_t(L.ctas) * 8);
  k_wire_compact<<<g > 0 ? g : 1, 256, 0, st>>>(d_off, w_off, d_rec, d_order, P.st_bytes, P.st_tag, T,
                                               w_bytes, w_tag, w_nids);
  *n_launches += 3;
  return int(cudaGetLastError());
}

}  // namespace xm_internal
