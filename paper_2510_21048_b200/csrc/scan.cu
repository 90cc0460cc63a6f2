// scan.cu -- K1: allocated-bytes peak as a segmented prefix-scan/max (sm_100a).
//
// For every trace, peak_allocated = max over events i of sum_{k<=i} +-s_k with
// s_k the 512 B round-up of event k's request (PAPER.md:256 (i)
// "allocated_bytes changes by exactly the rounded request"; "the
// maximum value in this time series"), and its first index (reading Q7). No
// allocator state is needed for this quantity, so it is exact whenever no OOM
// truncates the trace (the mode requires unlimited capacity).
//
// Batches whose traces are all at most 65536 events long (every paper-shaped
// config) take K1t, one CTA per trace (below). Otherwise the flat,
// trace-oblivious decomposition, so that long traces never bound the launch
// (DESIGN.md §6 K1):
//   K1z  row_trace[r] = trace owning the first event of 16-event row r
//   K1a  persistent CTAs over 4096-event tiles (cp.async double-buffered in
//        shared memory), 16 contiguous events per thread. A tile
//        with no trace start inside (the common case) is one piece: plain
//        scan + argmax. Otherwise a segmented scan of the monoid (sum,
//        max-prefix, argmax); traces wholly inside the tile are finished here
//        and the tile's first/last pieces are stored for crossing traces
//   K1b  one thread per crossing trace folds its pieces (~len/4096 of them)
// HBM traffic: 8 B/event read once + 0.5 B/event row map + 48 B/tile + 64 B/trace.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "rounding.cuh"
#include "xm_internal.h"

namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr int kThreads = 256;
constexpr int kPer = 16;                     // events per thread
constexpr int kTile = kThreads * kPer;       // 4096 events per CTA
constexpr int kWarps = kThreads / 32;
constexpr int64_t kNeg = INT64_MIN;

// piece monoid as stored between kernels: sum of deltas, max prefix (relative
// to the piece start, kNeg if empty), flat index of its first occurrence
struct Mono {
  int64_t sum, mx, arg;
};

// register form: tile-relative argmax; tr = trace of the head the piece
// starts at (meaningful only for pieces that start at a head in this tile)
struct MonoR {
  int64_t sum, mx;
  int32_t arg;
  uint32_t tr;
};

__device__ __forceinline__ MonoR mono_id() { return MonoR{0, kNeg, -1, 0}; }

// A then B (strict >: the earlier index wins ties)
__device__ __forceinline__ MonoR combine(const MonoR& a, const MonoR& b) {
  MonoR r;
  r.sum = a.sum + b.sum;
  const int64_t cand = a.sum + b.mx;
  const bool take_b = b.mx != kNeg && cand > a.mx;
  r.mx = take_b ? cand : a.mx;
  r.arg = take_b ? b.arg : a.arg;
  r.tr = a.tr;
  return r;
}

__device__ __forceinline__ Mono combine_g(const Mono& a, const Mono& b) {
  Mono r;
  r.sum = a.sum + b.sum;
  const int64_t cand = a.sum + b.mx;
  const bool take_b = b.mx != kNeg && cand > a.mx;
  r.mx = take_b ? cand : a.mx;
  r.arg = take_b ? b.arg : a.arg;
  return r;
}

// +ceil(b/2^sh) for an alloc (b > 0), -ceil(-b/2^sh) = floor(b/2^sh) for a free:
// one arithmetic shift either way
__device__ __forceinline__ int64_t rounded_delta(int64_t b, uint32_t sh) {
  return (b + (b > 0 ? int64_t((1ull << sh) - 1) : 0)) >> sh;
}

// a packed event word (xm_batch.packed) -> signed request bytes
__device__ __forceinline__ int64_t unpack_bytes(int64_t v) {
  const int64_t m = v & ((1ll << 41) - 1);
  return (v >> 41) & 1 ? m : -m;
}

// with the roundup_power2_divisions variant (NEXT-4): the shared a2 rule
__device__ __forceinline__ int64_t rounded_delta(int64_t b, const xm_internal::UnitConfig& u) {
  if (!u.div_shift) return rounded_delta(b, u.unit_shift);
  const int64_t r = int64_t(xm_internal::round_units(uint64_t(b > 0 ? b : -b), u));
  return b > 0 ? r : -r;
}

struct SParams {
  const int64_t* __restrict__ bytes;      // signed request bytes, or the packed words
  bool packed;                            // bytes holds xm_batch.packed words
  const int64_t* __restrict__ off;
  const uint32_t* __restrict__ order;   // caller index of each stored trace
  int64_t n_traces, n_events;
  uint32_t unit_shift;
  xm_internal::UnitConfig u;
  int64_t n_tiles;
  uint32_t* row_trace;      // [n_tiles * kThreads] trace owning each thread row's first event
  Mono* tile_first;         // [n_tiles] piece before the tile's first trace start
  Mono* tile_last;          // [n_tiles] piece from the tile's last trace start
  xm_result* out;
  unsigned int* work;       // trace counter of k_scan_trace
};

__device__ __forceinline__ Mono to_global(const MonoR& m, int64_t t0e) {
  return Mono{m.sum, m.mx, m.arg < 0 ? -1 : t0e + m.arg};
}

__device__ __forceinline__ void write_result(const SParams& P, uint32_t t, int64_t mx,
                                             int64_t arg_flat) {
  const int64_t o = P.off[t];
  xm_result R{};
  R.peak_allocated = mx > 0 ? uint64_t(mx) << P.unit_shift : 0ull;
  R.peak_allocated_idx = mx > 0 ? uint32_t(arg_flat - o) : 0u;
  R.events_done = uint32_t(P.off[t + 1] - o);
  R.status = XM_T_OK;
  P.out[P.order[t]] = R;
}

__device__ __forceinline__ MonoR shfl_up_mono(const MonoR& m, int o) {
  return MonoR{__shfl_up_sync(kFull, m.sum, o), __shfl_up_sync(kFull, m.mx, o),
               __shfl_up_sync(kFull, m.arg, o), __shfl_up_sync(kFull, m.tr, o)};
}

// segmented op: (fa, A) (+) (fb, B) = (fa | fb, fb ? B : A.B)
__device__ __forceinline__ void seg_combine(bool& fa, MonoR& a, bool fb, const MonoR& b) {
  a = fb ? b : combine(a, b);
  fa = fa || fb;
}

// K1z: row_trace[r] = trace owning event r*kPer (one warp per trace, lanes stride
// over its rows, so a long trace does not serialise)
__global__ void k_row_map(SParams P) {
  const int64_t t = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= P.n_traces) return;
  const int64_t a = P.off[t], b = P.off[t + 1];
  if (b <= a) return;
  for (int64_t r = (a + kPer - 1) / kPer + lane; r * kPer < b; r += 32) P.row_trace[r] = uint32_t(t);
}

__device__ __forceinline__ void stage_tile(const SParams& P, unsigned char* buf, int64_t c) {
  const int tid = threadIdx.x;
  const int64_t t0e = c * kTile;
  const int64_t t1e = min(t0e + kTile, P.n_events);
  const int nchunks = int((t1e - t0e + 1) / 2);                   // 16 B = 2 events
  const uint32_t sbase = uint32_t(__cvta_generic_to_shared(buf));
  const long long* by = reinterpret_cast<const long long*>(P.bytes);
#pragma unroll
  for (int r = 0; r < kTile / 2 / kThreads; ++r) {
    const int ch = tid + r * kThreads;
    if (ch < nchunks) {
      const uint32_t dst = sbase + uint32_t(ch * 16 + (ch >> 3) * 16);
      const long long* src = by + t0e + 2 * ch;
      if (t0e + 2 * ch + 1 < t1e) {
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src));
      } else {                                                    // odd tail: one event
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(src));
      }
    }
  }
}

// K1a: persistent; tiles are staged in shared memory with coalesced cp.async
// (16 B per thread per round), padded by 16 B every 128 B so that each
// thread's 16-event (128 B) row reads back without bank conflicts; the next
// tile is in flight while the current one is scanned (double buffer).
__global__ void __launch_bounds__(kThreads) k_scan_tiles(SParams P) {
  extern __shared__ __align__(16) unsigned char dsm[];
  __shared__ bool wflag[kWarps];
  __shared__ MonoR wagg[kWarps];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int kStage = kTile * 8 + kTile / 16 * 16;           // 36 KB per stage

  int64_t c = blockIdx.x;
  if (c < P.n_tiles) stage_tile(P, dsm, c);
  asm volatile("cp.async.commit_group;\n" ::);
  for (int k = 0; c < P.n_tiles; ++k, c += gridDim.x) {
    unsigned char* cur_buf = dsm + (k & 1) * kStage;
    const int64_t cn = c + gridDim.x;
    if (cn < P.n_tiles) stage_tile(P, dsm + ((k + 1) & 1) * kStage, cn);
    asm volatile("cp.async.commit_group;\n" ::);

    const int64_t t0e = c * kTile;
    const int64_t t1e = min(t0e + kTile, P.n_events);
    const int rel0 = tid * kPer;
    const int64_t g0 = t0e + rel0;
    const int64_t left = t1e - g0;
    const int nvalid = left <= 0 ? 0 : (left >= kPer ? kPer : int(left));
    // which trace owns this thread's first event, and does a trace start in its row?
    uint32_t tcur = 0;
    int64_t end_cur = INT64_MAX;
    bool head0 = false;
    if (nvalid > 0) {
      tcur = P.row_trace[c * kThreads + tid];
      end_cur = P.off[tcur + 1];
      head0 = P.off[tcur] == g0;
    }
    const bool any_head = __syncthreads_or(head0 || (nvalid > 0 && end_cur < g0 + nvalid));

    asm volatile("cp.async.wait_group 1;\n" ::);
    __syncthreads();
    int64_t d[kPer];
    {
      const longlong2* row = reinterpret_cast<const longlong2*>(cur_buf + tid * 144);
#pragma unroll
      for (int i = 0; i < kPer / 2; ++i) {
        const longlong2 x = row[i];
        d[2 * i] = x.x;
        d[2 * i + 1] = x.y;
      }
    }
    __syncthreads();                          // the buffer is refilled next iteration

    if (!any_head) {
      // ===== fast path: the whole tile is one piece of one trace =====
      int64_t run = 0, mx = kNeg;
      int32_t arg = -1;
#pragma unroll
      for (int i = 0; i < kPer; ++i) {
        if (i < nvalid) {
          run += rounded_delta(P.packed ? unpack_bytes(d[i]) : d[i], P.u);
          if (run > mx) { mx = run; arg = rel0 + i; }
        }
      }
      int64_t incl = run;                     // warp exclusive prefix of run
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += y;
      }
      const int64_t excl = incl - run;
      int64_t v = mx == kNeg ? kNeg : excl + mx;
      int32_t va = arg;
#pragma unroll
      for (int o = 16; o; o >>= 1) {          // argmax, earlier index on ties
        const int64_t w = __shfl_xor_sync(kFull, v, o);
        const int32_t wa = __shfl_xor_sync(kFull, va, o);
        if (w > v || (w == v && wa < va && w != kNeg)) { v = w; va = wa; }
      }
      if (lane == 31) wagg[warp] = MonoR{incl, v, va, 0};
      __syncthreads();
      if (tid == 0) {
        MonoR m = wagg[0];
        for (int w = 1; w < kWarps; ++w) m = combine(m, wagg[w]);
        const Mono g = to_global(m, t0e);
        P.tile_first[c] = g;
        P.tile_last[c] = g;
      }
      __syncthreads();
      continue;
    }

    // ===== general path: segmented scan; pieces carry the trace of their head =====
    MonoR cur = mono_id(), first_piece = mono_id();
    bool seen = false;
    int64_t run = 0;
    int hnext = int(min(end_cur - g0, int64_t(kPer)));     // row offset of the next head
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      if (i < nvalid) {
        const bool head = (i == 0) ? head0 : (i == hnext);
        if (head) {
          if (i > 0) {                        // step to the trace starting here (skip empties)
            const int64_t pos = g0 + i;
            ++tcur;
            while (P.off[tcur + 1] == pos) ++tcur;
            end_cur = P.off[tcur + 1];
            hnext = int(min(end_cur - g0, int64_t(kPer)));
          }
          if (!seen) {
            first_piece = cur;
            seen = true;
          } else {
            write_result(P, cur.tr, cur.mx, t0e + cur.arg);   // trace wholly inside this row
          }
          cur = mono_id();
          cur.tr = tcur;
          run = 0;
        }
        run += rounded_delta(P.packed ? unpack_bytes(d[i]) : d[i], P.u);
        cur.sum = run;
        if (run > cur.mx) { cur.mx = run; cur.arg = rel0 + i; }
      }
    }
    // ---- CTA exclusive segmented scan of (seen, cur) ----
    bool f = seen;
    MonoR a = cur;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const MonoR b = shfl_up_mono(a, o);
      const bool fb = __shfl_up_sync(kFull, f, o);
      if (lane >= o) {          // (fb, b) precedes (f, a)
        MonoR x = b;
        bool fx = fb;
        seg_combine(fx, x, f, a);
        a = x;
        f = fx;
      }
    }
    if (lane == 31) { wflag[warp] = f; wagg[warp] = a; }
    __syncthreads();
    bool cf = false;
    MonoR cw = mono_id();
    for (int w = 0; w < warp; ++w) seg_combine(cf, cw, wflag[w], wagg[w]);
    MonoR ex = shfl_up_mono(a, 1);
    bool exf = __shfl_up_sync(kFull, f, 1);
    if (lane == 0) { ex = mono_id(); exf = false; }
    bool carry_f = cf;
    MonoR carry = cw;
    seg_combine(carry_f, carry, exf, ex);   // everything before this thread

    if (seen) {
      const MonoR done = combine(carry, first_piece);
      if (carry_f) write_result(P, carry.tr, done.mx, t0e + done.arg);   // started at a head here
      else P.tile_first[c] = to_global(done, t0e);   // prefix piece of a trace that crossed in
    }
    const int last_tid = int((t1e - t0e - 1) / kPer);   // owns the tile's tail piece
    if (tid == last_tid) {
      bool lf = carry_f;
      MonoR lm = carry;
      seg_combine(lf, lm, seen, cur);
      if (P.off[lm.tr + 1] <= t1e) write_result(P, lm.tr, lm.mx, t0e + lm.arg);  // ends in tile
      else P.tile_last[c] = to_global(lm, t0e);
    }
    __syncthreads();                          // wflag/wagg reused next tile
  }
  asm volatile("cp.async.wait_group 0;\n" ::);
}

// K1b: fold pieces of traces that cross tile boundaries; empty traces -> zeros
__global__ void k_scan_combine(SParams P) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= P.n_traces) return;
  const int64_t a = P.off[t], b = P.off[t + 1];
  if (b <= a) {
    xm_result R{};
    P.out[P.order[t]] = R;
    return;
  }
  const int64_t ca = a / kTile, cb = (b - 1) / kTile;
  if (ca == cb) return;                     // finished by k_scan_tiles
  Mono m = P.tile_last[ca];
  for (int64_t c = ca + 1; c <= cb; ++c) m = combine_g(m, P.tile_first[c]);
  write_result(P, uint32_t(t), m.mx, m.arg);
}

// K1t: one CTA (kTWarps warps) per trace, persistent over the stored (longest-first)
// order -- the path for batches of traces up to kTraceMax events (all of the
// paper-shaped configs). A step covers kStep = kTWarps x 32 lanes x kPerLane
// events: each lane takes kPerLane CONSECUTIVE events with 16-byte loads (the
// next step's loads are in flight meanwhile), scans them serially (sum, max
// prefix, first argmax), the warp combines its lanes with one exclusive scan
// and one arg-max reduction, and warp 0 folds the warp pieces in order onto
// the running prefix. 8 B read per event, 2 barriers per step.
constexpr int kTraceMax = 1 << 16;
#ifndef XM_K1_WARPS
#define XM_K1_WARPS 4
#endif
#ifndef XM_K1_PER_LANE
#define XM_K1_PER_LANE 8
#endif
#ifndef XM_K1_MINB
#define XM_K1_MINB 8            // launch bound: 8 resident CTAs per SM (64 registers)
#endif
constexpr int kTWarps = XM_K1_WARPS;
constexpr int kTThreads = 32 * kTWarps;
constexpr int kPerLane = XM_K1_PER_LANE;
constexpr int kWarpSpan = 32 * kPerLane;
constexpr int kStep = kTWarps * kWarpSpan;

// a2 for K1t: the plain 512 B rule as one shift, or the divisions variant
template <bool kDiv>
__device__ __forceinline__ int64_t k1_delta(int64_t b, const SParams& P) {
  if constexpr (kDiv) return rounded_delta(b, P.u);
  else return rounded_delta(b, P.unit_shift);
}

template <bool kPacked, bool kDiv>
__global__ void __launch_bounds__(kTThreads, XM_K1_MINB) k_scan_trace(SParams P) {
  __shared__ long long s_sum[kTWarps], s_mx[kTWarps];
  __shared__ int s_arg[kTWarps];
  __shared__ unsigned int s_k;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const long long* by = reinterpret_cast<const long long*>(P.bytes);
  // the grid is exactly the resident CTAs: CTA i starts on stored trace i
  // (the longest-first order's first wave) without touching the counter,
  // then pulls gridDim.x + counter
  for (bool first = true;; first = false) {
    if (tid == 0) s_k = first ? blockIdx.x : gridDim.x + atomicAdd(P.work, 1u);
    __syncthreads();
    const unsigned k = s_k;
    __syncthreads();                        // s_k is rewritten by the next pull
    if (int64_t(k) >= P.n_traces) break;
    const int64_t e0 = P.off[k];
    const int n = int(P.off[k + 1] - e0);
    // positions relative to the 16-byte aligned event pair holding e0
    const int sh = int(e0 & 1);
    const long long* b2 = by + (e0 - sh);
    const int m = n + sh;
    long long carry = 0, best = kNeg;       // warp 0 (uniform across its lanes)
    int barg = -1;
    longlong2 cur[kPerLane / 2], nxt[kPerLane / 2];
    const int p0 = kWarpSpan * w + kPerLane * lane;     // this lane's first position
    auto load = [&](longlong2* dst, int base) {
#pragma unroll
      for (int q = 0; q < kPerLane / 2; ++q) {
        const int p = base + p0 + 2 * q;
        if (p + 1 < m) dst[q] = __ldcs(reinterpret_cast<const longlong2*>(b2 + p));
        else dst[q] = make_longlong2(p < m ? __ldcs(b2 + p) : 0, 0);
      }
    };
    load(cur, 0);
    for (int base = 0; base < m; base += kStep) {
      load(nxt, base + kStep);
      long long run = 0, lmx = kNeg;
      int larg = -1;
      if ((base > 0 || sh == 0) && base + kStep <= m) {    // every position valid
#pragma unroll
        for (int q = 0; q < kPerLane; ++q) {
          const long long raw = (q & 1) ? cur[q >> 1].y : cur[q >> 1].x;
          run += k1_delta<kDiv>(kPacked ? unpack_bytes(raw) : raw, P);
          if (run > lmx) { lmx = run; larg = base + p0 + q - sh; }
        }
      } else {
#pragma unroll
        for (int q = 0; q < kPerLane; ++q) {
          const int idx = base + p0 + q - sh;           // event index in the trace
          const long long raw = (q & 1) ? cur[q >> 1].y : cur[q >> 1].x;
          if (idx >= 0 && idx < n) {
            run += k1_delta<kDiv>(kPacked ? unpack_bytes(raw) : raw, P);
            if (run > lmx) { lmx = run; larg = idx; }
          }
        }
      }
      long long ex = run;                     // exclusive scan of the lane sums
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(kFull, ex, o);
        if (lane >= o) ex += y;
      }
      const long long wsum = __shfl_sync(kFull, ex, 31);
      ex -= run;
      // first argmax of the warp: lanes hold increasing index ranges, so it
      // is the lowest lane with the maximum; the maximum by two 32-bit
      // reductions of the order-preserving unsigned image (kNeg -> 0)
      const unsigned long long ukey =
          static_cast<unsigned long long>(lmx == kNeg ? kNeg : ex + lmx) ^ 0x8000000000000000ull;
      const unsigned khi = unsigned(ukey >> 32), klo = unsigned(ukey);
      const unsigned mh = __reduce_max_sync(kFull, khi);
      const unsigned ml = __reduce_max_sync(kFull, khi == mh ? klo : 0u);
      const int src = __ffs(__ballot_sync(kFull, khi == mh && klo == ml)) - 1;
      const int ca = __shfl_sync(kFull, larg, src);
      const long long c =
          static_cast<long long>(((static_cast<unsigned long long>(mh) << 32) | ml) ^ 0x8000000000000000ull);
      if (lane == 0) { s_sum[w] = wsum; s_mx[w] = c; s_arg[w] = ca; }
      __syncthreads();
      if (w == 0) {                           // fold the warp pieces in order
        const long long ps = lane < kTWarps ? s_sum[lane] : 0;
        const long long pm = lane < kTWarps ? s_mx[lane] : kNeg;
        const int pa = lane < kTWarps ? s_arg[lane] : -1;
        long long pe = ps;
#pragma unroll
        for (int o = 1; o < kTWarps; o <<= 1) {
          const long long y = __shfl_up_sync(kFull, pe, o);
          if (lane >= o) pe += y;
        }
        pe -= ps;
        // first argmax over the warp pieces (lowest lane among ties), as above
        const unsigned long long uk =
            static_cast<unsigned long long>(pm == kNeg ? kNeg : carry + pe + pm) ^ 0x8000000000000000ull;
        const unsigned fhi = unsigned(uk >> 32), flo = unsigned(uk);
        const unsigned fmh = __reduce_max_sync(kFull, fhi);
        const unsigned fml = __reduce_max_sync(kFull, fhi == fmh ? flo : 0u);
        const int fsrc = __ffs(__ballot_sync(kFull, fhi == fmh && flo == fml)) - 1;
        const int cca = __shfl_sync(kFull, pa, fsrc);
        const long long cc =
            static_cast<long long>(((static_cast<unsigned long long>(fmh) << 32) | fml) ^ 0x8000000000000000ull);
        if (cc != kNeg && cc > best) { best = cc; barg = cca; }
        carry += __shfl_sync(kFull, pe + ps, kTWarps - 1);
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < kPerLane / 2; ++q) cur[q] = nxt[q];
    }
    if (tid == 0) {
      xm_result R{};
      R.peak_allocated = best > 0 ? uint64_t(best) << P.unit_shift : 0ull;
      R.peak_allocated_idx = best > 0 ? uint32_t(barg) : 0u;
      R.events_done = uint32_t(n);
      R.status = XM_T_OK;
      P.out[P.order[k]] = R;
    }
  }
}


// ---- K1c: contiguous event chunks streamed by TMA -----------------------------
//
// The same quantity as K1t (max prefix sum of +-s per trace and its first
// index), but trace-oblivious: the batch's events are cut into contiguous
// chunks of whole tiles, one per WARP of a persistent grid, so every warp
// streams an equal share no matter how long the traces are, no trace start
// waits on a work counter, and no barrier couples the warps of a CTA while
// they stream. Each warp's tiles arrive by TMA (cp.async.bulk.tensor.2d; the
// events viewed as rows of 16 words with the 128-byte swizzle, so each lane's
// consecutive events read back without bank conflicts) into the warp's own
// kCStages-deep mbarrier ring, kCStages tiles ahead, issued by lane 0. A tile
// without a trace start (the common case) is one piece: a warp scan + arg-max
// folded onto the warp's running piece. Otherwise a segmented scan of
// (starts-here flag, piece, trace): traces that start and end inside the
// warp's chunk are finished in place. Each chunk leaves its head piece (events
// before its first trace start) and tail piece (from its last start); warp 0
// folds its CTA's chunk records into one, and the last CTA to finish folds
// the CTA records (the same segmented scan).
// HBM: 8 B/event read once + 64 B/trace written.
#ifndef XM_K1C_PER
#define XM_K1C_PER 8
#endif
#ifndef XM_K1C_STAGES
#define XM_K1C_STAGES 3
#endif
#ifndef XM_K1C_CTAS_PER_SM
#define XM_K1C_CTAS_PER_SM 3
#endif
#ifndef XM_K1C_THREADS
#define XM_K1C_THREADS 256
#endif
constexpr int kCThreads = XM_K1C_THREADS;
constexpr int kCWarps = kCThreads / 32;
constexpr int kCPer = XM_K1C_PER;                  // consecutive events per lane (8 or 16)
constexpr int kCTile = 32 * kCPer;                 // events per warp tile (16 per 128-byte row)
constexpr int kCRows = kCTile / 16;                // TMA box rows
constexpr int kCTileBytes = kCTile * 8;            // a multiple of 1024 (the swizzle atom)
constexpr int kCStages = XM_K1C_STAGES;
constexpr int kCSmem = kCWarps * kCStages * kCTileBytes + 1024;   // + the swizzle alignment
constexpr int kCList = kCTile + 64;                // trace starts listed per (re)fill: a refill
                                                   // from a tile's first start covers the tile
static_assert(kCPer == 8 || kCPer == 16, "K1c: 8 or 16 events per lane");
static_assert(kCTileBytes % 1024 == 0, "K1c: swizzle atom");

// segmented-scan element: a piece (sum, max prefix or kNeg if empty, global
// index of its first maximum), whether a trace starts inside it (f), and the
// trace of its last start (tr, when f)
struct SegE {
  int64_t sum, mx, arg;
  int32_t tr;
  bool f;
};

__device__ __forceinline__ SegE seg_id() { return SegE{0, kNeg, -1, -1, false}; }

// a then b
__device__ __forceinline__ SegE seg_op(const SegE& a, const SegE& b) {
  if (b.f) return b;
  SegE r;
  r.sum = a.sum + b.sum;
  const int64_t cand = a.sum + b.mx;
  const bool take = b.mx != kNeg && cand > a.mx;       // strict: the first index wins
  r.mx = take ? cand : a.mx;
  r.arg = take ? b.arg : a.arg;
  r.tr = a.tr;
  r.f = a.f;
  return r;
}

__device__ __forceinline__ SegE shfl_up_seg(const SegE& e, int o) {
  SegE r;
  r.sum = __shfl_up_sync(kFull, e.sum, o);
  r.mx = __shfl_up_sync(kFull, e.mx, o);
  r.arg = __shfl_up_sync(kFull, e.arg, o);
  r.tr = __shfl_up_sync(kFull, e.tr, o);
  r.f = __shfl_up_sync(kFull, int(e.f), o) != 0;
  return r;
}

__device__ __forceinline__ SegE shfl_seg(const SegE& e, int src) {
  SegE r;
  r.sum = __shfl_sync(kFull, e.sum, src);
  r.mx = __shfl_sync(kFull, e.mx, src);
  r.arg = __shfl_sync(kFull, e.arg, src);
  r.tr = __shfl_sync(kFull, e.tr, src);
  r.f = __shfl_sync(kFull, int(e.f), src) != 0;
  return r;
}

// inclusive warp segmented scan
__device__ __forceinline__ SegE warp_seg_scan(SegE x, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const SegE y = shfl_up_seg(x, o);
    if (lane >= o) x = seg_op(y, x);
  }
  return x;
}

struct __align__(16) ChunkSum {   // one per chunk (K1c), in scratch; 64 B
  int64_t h_sum, h_mx, h_arg;      // head piece: events before the chunk's first trace start
  int64_t t_sum, t_mx, t_arg;      // tail piece: from its last trace start to its end
  int32_t t_tr;                    // trace of the last start
  int32_t has;                     // a trace starts inside the chunk
  int64_t pad;
};
static_assert(sizeof(ChunkSum) == 64, "ChunkSum");

// another CTA's record (L2, not a possibly stale L1 line)
__device__ __forceinline__ ChunkSum load_chunk(const ChunkSum* p) {
  ChunkSum r;
  const longlong2* s = reinterpret_cast<const longlong2*>(p);
  longlong2* d = reinterpret_cast<longlong2*>(&r);
#pragma unroll
  for (int i = 0; i < 4; ++i) d[i] = __ldcg(s + i);
  return r;
}

struct CParams {
  const int64_t* __restrict__ bytes;    // events (signed bytes or packed words)
  const int64_t* __restrict__ off;
  const uint32_t* __restrict__ order;
  int64_t n_traces, n_events;
  int64_t rows;                         // full 16-event rows covered by the tensor map
  int64_t n_tiles;
  uint32_t unit_shift;
  xm_internal::UnitConfig u;
  ChunkSum* chunks;
  unsigned int* done;
  xm_result* out;
};

__device__ __forceinline__ void c_write(const CParams& P, int32_t tr, int64_t mx, int64_t arg) {
  const int64_t o = P.off[tr];
  xm_result R{};
  R.peak_allocated = mx > 0 ? uint64_t(mx) << P.unit_shift : 0ull;
  R.peak_allocated_idx = mx > 0 ? uint32_t(arg - o) : 0u;
  R.events_done = uint32_t(P.off[tr + 1] - o);
  R.status = XM_T_OK;
  P.out[P.order[tr]] = R;
}

template <bool kPacked, bool kDiv>
__device__ __forceinline__ int64_t c_delta(int64_t raw, const CParams& P) {
  if constexpr (kPacked && !kDiv) {
    // |request| in bits 0-40, allocation bit 41: ceil(|b| / 2^sh) with the sign
    // of the event (the same value as rounded_delta(unpack_bytes(raw), sh))
    const uint64_t m = uint64_t(raw) & ((1ull << 41) - 1);
    const int64_t u = int64_t((m + ((1ull << P.unit_shift) - 1)) >> P.unit_shift);
    return (raw >> 41) & 1 ? u : -u;
  }
  const int64_t b = kPacked ? unpack_bytes(raw) : raw;
  if constexpr (kDiv) return rounded_delta(b, P.u);
  else return rounded_delta(b, P.unit_shift);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return uint32_t(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar), "r"(parity) : "memory");
}

// Last CTA: fold the chunk pieces (segmented scan over the G chunk elements).
__device__ void c_fixup(const CParams& P, int G, SegE* s_w) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  SegE carry = seg_id();
  for (int base = 0; base < G; base += kCThreads) {
    const int c = base + tid;
    SegE e = seg_id();
    ChunkSum cs{};
    if (c < G) {
      cs = load_chunk(P.chunks + c);
      e = cs.has ? SegE{cs.t_sum, cs.t_mx, cs.t_arg, cs.t_tr, true}
                 : SegE{cs.h_sum, cs.h_mx, cs.h_arg, -1, false};
    }
    const SegE inc = warp_seg_scan(e, lane);
    if (lane == 31) s_w[w] = inc;
    __syncthreads();
    SegE pre = carry;
    for (int k = 0; k < w; ++k) pre = seg_op(pre, s_w[k]);
    SegE ex = shfl_up_seg(inc, 1);
    if (lane == 0) ex = seg_id();
    const SegE cin = seg_op(pre, ex);               // everything before chunk c
    if (c < G && cs.has && cin.f) {                 // chunk c ends the trace open at its start
      const SegE h{cs.h_sum, cs.h_mx, cs.h_arg, -1, false};
      const SegE d = seg_op(cin, h);
      c_write(P, cin.tr, d.mx, d.arg);
    }
    SegE tot = carry;
    for (int k = 0; k < kCWarps; ++k) tot = seg_op(tot, s_w[k]);
    carry = tot;
    __syncthreads();
  }
  if (tid == 0 && carry.f) c_write(P, carry.tr, carry.mx, carry.arg);   // ends at the last event
}

// one warp: list the distinct trace starts at or after trace jn (the last trace
// of a run of equal offsets; the earlier ones are empty) below `end`, up to
// kCList of them, as chunk-relative positions; returns (count, next jn) and
// whether every start below `end` is listed
__device__ __forceinline__ void list_starts(const CParams& P, int64_t& jn, int64_t c0, int64_t end,
                                            uint32_t* pos, int32_t* tr, int& cnt, bool& all) {
  const int lane = threadIdx.x & 31;
  cnt = 0;
  all = false;
  for (;;) {
    if (cnt > kCList - 32) return;                 // full: refilled later
    const int64_t x = jn + lane;
    const int64_t v = x < P.n_traces ? P.off[x] : INT64_MAX;
    const int64_t vn = x < P.n_traces ? P.off[x + 1] : INT64_MAX;
    const bool in = v < end;
    const bool keep = in && vn != v;
    const unsigned km = __ballot_sync(kFull, keep);
    if (keep) {
      const int d = cnt + __popc(km & ((1u << lane) - 1u));
      pos[d] = uint32_t(v - c0);
      tr[d] = int32_t(x);
    }
    cnt += __popc(km);
    const int nin = __popc(__ballot_sync(kFull, in));
    jn += nin;
    if (nin < 32) { all = true; return; }
  }
}

// the pieces of a run of records (chunk heads and tails) in order: the traces
// that end inside the run are finished; returns the run's own record. One warp,
// n <= 32 records, the carry-in of the run is the identity.
__device__ ChunkSum fold_records(const CParams& P, const ChunkSum* rec, int n) {
  const int lane = threadIdx.x & 31;
  ChunkSum cs{};
  SegE e = seg_id(), h = seg_id();
  if (lane < n) {
    cs = rec[lane];
    h = SegE{cs.h_sum, cs.h_mx, cs.h_arg, -1, false};
    e = cs.has ? SegE{cs.t_sum, cs.t_mx, cs.t_arg, cs.t_tr, true} : h;
  }
  const SegE inc = warp_seg_scan(e, lane);
  SegE cin = shfl_up_seg(inc, 1);
  if (lane == 0) cin = seg_id();
  const SegE dn = seg_op(cin, h);
  const bool has = lane < n && cs.has;
  if (has && cin.f) c_write(P, cin.tr, dn.mx, dn.arg);   // ends at this record's first start
  const unsigned hm = __ballot_sync(kFull, has && !cin.f);   // the run's first start
  const SegE tot = shfl_seg(inc, 31);
  ChunkSum r{};
  if (hm) {
    const SegE hh = shfl_seg(dn, __ffs(hm) - 1);
    r = ChunkSum{hh.sum, hh.mx, hh.arg, tot.sum, tot.mx, tot.arg, tot.tr, 1, 0};
  } else {
    r = ChunkSum{tot.sum, tot.mx, tot.arg, 0, kNeg, -1, -1, 0, 0};
  }
  return r;
}

template <bool kPacked, bool kDiv>
__global__ void __launch_bounds__(kCThreads, XM_K1C_CTAS_PER_SM) k_scan_chunks(const __grid_constant__ CUtensorMap tm,
                                                           CParams P) {
  extern __shared__ unsigned char c_dsm[];
  __shared__ __align__(8) unsigned long long s_bar[kCWarps][kCStages];
  __shared__ uint32_t s_pos[kCWarps][kCList];    // each warp's listed trace starts (chunk-relative)
  __shared__ int32_t s_tr[kCWarps][kCList];      // ... and the trace starting there
  __shared__ ChunkSum s_rec[kCWarps];
  __shared__ SegE s_w[kCWarps];
  __shared__ bool s_last;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  // this warp's stages, as a shared-window address (1024-aligned: the swizzle atom)
  const uint32_t ring = ((smem_u32(c_dsm) + 1023u) & ~1023u) + uint32_t(w * kCStages * kCTileBytes);
  uint32_t* pos = s_pos[w];
  int32_t* trs = s_tr[w];
  const int G = gridDim.x;
  const int64_t NW = int64_t(G) * kCWarps;
  const int64_t u = int64_t(blockIdx.x) * kCWarps + w;              // this warp's chunk
  const int64_t k0 = u * P.n_tiles / NW, k1 = (u + 1) * P.n_tiles / NW;
  const int nk = int(k1 - k0);
  const int64_t c0 = k0 * kCTile;                                   // first event
  const int64_t c1 = min(k1 * kCTile, P.n_events);                  // past the last

  if (lane == 0) {
    for (int st = 0; st < kCStages; ++st)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&s_bar[w][st])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncwarp();
  auto issue = [&](int k, int st) {                // tile k0+k into stage st (= k % kCStages)
    const uint32_t bar = smem_u32(&s_bar[w][st]);
    const int64_t row = (k0 + k) * kCRows;
    if (row < P.rows) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                   "r"(kCTileBytes) : "memory");
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3}], [%4];" ::"r"(ring + uint32_t(st * kCTileBytes)),
          "l"(reinterpret_cast<uint64_t>(&tm)), "r"(0), "r"(int(row)), "r"(bar)
          : "memory");
    } else {                                       // past the tensor: read from global
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
    }
  };
  if (lane == 0)
    for (int k = 0; k < kCStages && k < nk; ++k) issue(k, k);
  for (int64_t t = int64_t(blockIdx.x) * kCThreads + tid; t < P.n_traces;
       t += int64_t(G) * kCThreads)
    if (P.off[t + 1] == P.off[t]) P.out[P.order[t]] = xm_result{};   // empty trace
  // jn = first trace with off[jn] >= c0 (a 32-ary search), then the chunk's starts
  int64_t jn;
  {
    int64_t lo = 0, hi = P.n_traces;               // answer in [lo, hi]
    while (hi - lo > 32) {
      const int64_t step = (hi - lo + 31) / 32;
      const int64_t x = lo + int64_t(lane) * step;
      const bool below = x < hi && P.off[x] < c0;
      const int nbl = __popc(__ballot_sync(kFull, below));   // lanes 0..nbl-1 are below
      const int64_t nlo = nbl == 0 ? lo : lo + int64_t(nbl - 1) * step + 1;
      const int64_t nhi = min(hi, lo + int64_t(nbl) * step);
      lo = nlo;
      hi = nhi;
    }
    const int64_t x = lo + lane;
    const bool below = x < hi && P.off[x] < c0;
    jn = lo + __popc(__ballot_sync(kFull, below));
  }
  int cnt = 0;
  bool all = true;
  if (nk > 0) list_starts(P, jn, c0, c1, pos, trs, cnt, all);
  __syncwarp();
  int bi = 0;                                      // first listed start not yet passed

  SegE run = seg_id();                             // this warp's chunk so far (warp-uniform)
  SegE head = seg_id();                            // (the lane that closed the head piece)
  bool head_here = false;
  int st = 0;                                      // stage of tile k, and its phase
  uint32_t phase = 0;
  for (int k = 0; k < nk; ++k) {
    const int64_t ts = (k0 + k) * kCTile;
    const int64_t te = min(ts + kCTile, P.n_events);
    const uint32_t rte = uint32_t(te - c0);
    if (!all && (bi == cnt || pos[cnt - 1] < rte)) {
      // (rare) unlisted starts may lie in this tile: relist from its first start
      int64_t j = bi < cnt ? int64_t(trs[bi]) : jn;
      __syncwarp();
      list_starts(P, j, c0, c1, pos, trs, cnt, all);
      __syncwarp();
      jn = j;
      bi = 0;
    }
    // starts in this tile: listed entries [bi, bi + nb)
    int nb = 0;
    for (;;) {
      const int i = bi + nb + lane;
      const bool in = i < cnt && pos[i] < rte;
      const int m = __popc(__ballot_sync(kFull, in));
      nb += m;
      if (m < 32) break;
    }
    mbar_wait(smem_u32(&s_bar[w][st]), phase);
    const int64_t p0 = ts + int64_t(lane) * kCPer; // this lane's first event
    const uint32_t sb = ring + uint32_t(st * kCTileBytes);
    // 128-byte swizzle: 16-byte chunk j of row r sits at chunk j ^ (r & 7)
    auto load_stage = [&](int64_t* d) {
      const int r = (lane * kCPer) >> 4;
      const int j0 = (lane * kCPer & 15) >> 1;
#pragma unroll
      for (int q = 0; q < kCPer / 2; ++q) {
        const uint32_t a = sb + uint32_t(r * 128 + (((j0 + q) ^ (r & 7)) << 4));
        long long x, y;
        asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(x), "=l"(y) : "r"(a));
        d[2 * q] = x;
        d[2 * q + 1] = y;
      }
    };
    // the warp's tile is whole and staged (every tile but the batch's last)
    const bool full = te - ts == kCTile && ts + kCTile <= P.rows * 16;
    int64_t d[kCPer];
    bool done = false;
    if constexpr (!kDiv) {
      if (full && nb == 0) {
        // ===== the common tile: no trace starts, no ragged end =====
        // a2 in 32 bits (sh = log2 min_block < 32): |request| < 2^40
        // (XM_MAX_REQUEST); the low word of b >> sh is one funnel shift of
        // (hi, lo), plus one for an allocation with a remainder (ceil).
        // Tier 32 (8 events per lane): every |b| < 2^31, so |delta| <= 2^22
        // and the warp's 256 sums stay within int32, warp scan included.
        // Tier 35: every |b| < 2^35 (|delta| <= 2^26): lane sums in int32,
        // the warp scan in 64 bits. Else the 64-bit path.
        load_stage(d);
        const uint32_t sh = P.unit_shift;
        const uint32_t msk = (1u << sh) - 1u;
        int32_t v[kCPer];
        uint32_t g32 = 0, g35 = 0;           // tier 32 iff g32 == 0, tier 35 iff g35 < 16
#pragma unroll
        for (int q = 0; q < kCPer; ++q) {
          const uint32_t lo = uint32_t(uint64_t(d[q]));
          int32_t hi = int32_t(uint64_t(d[q]) >> 32);
          bool pos;
          if constexpr (kPacked) {           // |b| in bits 0-40, allocation bit 41
            pos = (hi >> 9) & 1;
            hi &= 0x1FF;
          } else {
            pos = hi >= 0;
          }
          const uint32_t qv = __funnelshift_r(lo, uint32_t(hi), sh);
          if constexpr (kPacked) {           // ceil of the magnitude, then the sign
            const int32_t u = int32_t(qv) + ((lo & msk) ? 1 : 0);
            v[q] = pos ? u : -u;
            g32 |= uint32_t(hi) | (lo >> 31);                           // m < 2^31
          } else {                           // ceil for allocations, floor for frees
            v[q] = int32_t(qv) + ((pos && (lo & msk)) ? 1 : 0);
            g32 |= uint32_t(hi ^ (int32_t(lo) >> 31));                 // b fits int32
          }
          g35 |= uint32_t(hi + 8);
        }
        int ai = 0;
        if (kCPer == 8 && sh < 32 && !__any_sync(kFull, g32 != 0u)) {
          // ---- tier 32 ----
          int32_t s32 = v[0], m32 = v[0];
#pragma unroll
          for (int q = 1; q < kCPer; ++q) {
            s32 += v[q];
            if (s32 > m32) { m32 = s32; ai = q; }
          }
          int32_t incl = s32;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int32_t y = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += y;
          }
          const int32_t key = incl - s32 + m32;
          const int32_t wm = __reduce_max_sync(kFull, key);
          const int src = __ffs(__ballot_sync(kFull, key == wm)) - 1;
          const int64_t warg = ts + int64_t(src) * kCPer + __shfl_sync(kFull, ai, src);
          const int32_t wsum = __shfl_sync(kFull, incl, 31);
          run = seg_op(run, SegE{int64_t(wsum), int64_t(wm), warg, -1, false});
        } else {
          int64_t sum, mx;
          if (sh < 32 && !__any_sync(kFull, g35 >= 16u)) {
            // ---- tier 35 ----
            int32_t s32 = v[0], m32 = v[0];
#pragma unroll
            for (int q = 1; q < kCPer; ++q) {
              s32 += v[q];
              if (s32 > m32) { m32 = s32; ai = q; }
            }
            sum = s32;
            mx = m32;
          } else {
            sum = c_delta<kPacked, kDiv>(d[0], P);
            mx = sum;
#pragma unroll
            for (int q = 1; q < kCPer; ++q) {
              sum += c_delta<kPacked, kDiv>(d[q], P);
              if (sum > mx) { mx = sum; ai = q; }
            }
          }
          int64_t incl = sum;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int64_t y = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += y;
          }
          const unsigned long long uk = static_cast<unsigned long long>(incl - sum + mx) ^ 0x8000000000000000ull;
          const unsigned khi = unsigned(uk >> 32), klo = unsigned(uk);
          const unsigned mh = __reduce_max_sync(kFull, khi);
          const unsigned ml = __reduce_max_sync(kFull, khi == mh ? klo : 0u);
          const int src = __ffs(__ballot_sync(kFull, khi == mh && klo == ml)) - 1;
          const int64_t wmx = static_cast<int64_t>((static_cast<unsigned long long>(mh) << 32 | ml) ^
                                                   0x8000000000000000ull);
          const int64_t warg = ts + int64_t(src) * kCPer + __shfl_sync(kFull, ai, src);
          const int64_t wsum = __shfl_sync(kFull, incl, 31);
          run = seg_op(run, SegE{wsum, wmx, warg, -1, false});
        }
        done = true;
      }
    }
    if (!done) {
    if (full || p0 + kCPer <= P.rows * 16) {
      load_stage(d);
    } else {
#pragma unroll
      for (int q = 0; q < kCPer; ++q)
        d[q] = p0 + q < te ? reinterpret_cast<const long long*>(P.bytes)[p0 + q] : 0;
    }
    const int nv = int(max(int64_t(0), min(int64_t(kCPer), te - p0)));
#pragma unroll
    for (int q = 0; q < kCPer; ++q) d[q] = q < nv ? c_delta<kPacked, kDiv>(d[q], P) : 0;
    // this lane's starts: listed entries [b, bi + nb) below r0 + kCPer
    const uint32_t r0 = uint32_t(p0 - c0);
    int b = bi + nb;
    if (nb) {
      int lo = bi, hi = bi + nb;                   // first start at or after r0
      while (lo < hi) {
        const int m = (lo + hi) >> 1;
        if (pos[m] < r0) lo = m + 1; else hi = m;
      }
      b = lo;
    }
    const bool mine = b < bi + nb && pos[b] < r0 + kCPer;
    const bool wany = __any_sync(kFull, mine);    // warp-uniform
    if (!wany) {
      // ===== no trace starts in this tile: one piece =====
      int64_t sum = 0, mx = kNeg;
      int ai = -1;
#pragma unroll
      for (int q = 0; q < kCPer; ++q) {
        sum += d[q];
        if (q < nv && sum > mx) { mx = sum; ai = q; }
      }
      int64_t incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += y;
      }
      const unsigned long long uk =
          static_cast<unsigned long long>(mx == kNeg ? kNeg : incl - sum + mx) ^ 0x8000000000000000ull;
      const unsigned khi = unsigned(uk >> 32), klo = unsigned(uk);
      const unsigned mh = __reduce_max_sync(kFull, khi);
      const unsigned ml = __reduce_max_sync(kFull, khi == mh ? klo : 0u);
      const int src = __ffs(__ballot_sync(kFull, khi == mh && klo == ml)) - 1;
      const int64_t wmx = static_cast<int64_t>((static_cast<unsigned long long>(mh) << 32 | ml) ^
                                               0x8000000000000000ull);
      const int64_t warg = p0 + __shfl_sync(kFull, ai, src) - (int64_t(lane) - src) * kCPer;
      const int64_t wsum = __shfl_sync(kFull, incl, 31);
      run = seg_op(run, SegE{wsum, wmx, wmx == kNeg ? -1 : warg, -1, false});
    } else {
      // ===== pieces split at the starts; traces wholly inside a lane are finished =====
      SegE cur = seg_id(), hd = seg_id();
      if (!mine) {
        int64_t sum = 0, mx = kNeg;
        int ai = -1;
#pragma unroll
        for (int q = 0; q < kCPer; ++q) {
          sum += d[q];
          if (q < nv && sum > mx) { mx = sum; ai = q; }
        }
        cur = SegE{sum, mx, ai < 0 ? -1 : p0 + ai, -1, false};
      } else {
        const int bend = bi + nb;
        uint32_t nxt = pos[b];
        bool seen = false;
#pragma unroll
        for (int q = 0; q < kCPer; ++q) {
          if (q < nv) {
            if (r0 + q == nxt) {
              if (!seen) hd = cur;
              else c_write(P, cur.tr, cur.mx, cur.arg);
              seen = true;
              cur = SegE{0, kNeg, -1, trs[b], true};
              ++b;
              nxt = b < bend ? pos[b] : 0xFFFFFFFFu;
            }
            cur.sum += d[q];
            if (cur.sum > cur.mx) { cur.mx = cur.sum; cur.arg = p0 + q; }
          }
        }
      }
      const SegE inc = warp_seg_scan(cur, lane);
      const SegE ex = shfl_up_seg(inc, 1);
      if (mine) {
        // finish the trace open at this lane's first start
        const SegE cin = lane ? seg_op(run, ex) : run;
        const SegE dn = seg_op(cin, SegE{hd.sum, hd.mx, hd.arg, -1, false});
        if (cin.f) {
          c_write(P, cin.tr, dn.mx, dn.arg);       // started in this chunk: finished here
        } else {                                   // the chunk's head piece (one lane)
          head = dn;
          head_here = true;
        }
      }
      run = seg_op(run, shfl_seg(inc, 31));
    }
    }
    __syncwarp();                                  // every lane has read the stage
    if (lane == 0 && k + kCStages < nk) issue(k + kCStages, st);
    if (++st == kCStages) { st = 0; phase ^= 1u; }
    bi += nb;
  }
  // this warp's chunk record, then the CTA's, then (last CTA) the grid's
  const unsigned hm = __ballot_sync(kFull, head_here);
  if (lane == 0) {
    ChunkSum cs;
    if (run.f) {
      cs = ChunkSum{0, kNeg, -1, run.sum, run.mx, run.arg, run.tr, 1, 0};
    } else {
      cs = ChunkSum{run.sum, run.mx, run.arg, 0, kNeg, -1, -1, 0, 0};
    }
    s_rec[w] = cs;
  }
  if (hm) {
    const SegE h = shfl_seg(head, __ffs(hm) - 1);
    if (lane == 0) { s_rec[w].h_sum = h.sum; s_rec[w].h_mx = h.mx; s_rec[w].h_arg = h.arg; }
  }
  __syncthreads();
  if (w == 0) {
    const ChunkSum cs = fold_records(P, s_rec, kCWarps);
    if (lane == 0) {
      P.chunks[blockIdx.x] = cs;
      __threadfence();
      s_last = atomicAdd(P.done, 1u) == unsigned(G - 1);
    }
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    c_fixup(P, G, s_w);
  }
}

}  // namespace

namespace xm_internal {

static int64_t n_tiles_of(const xm_batch* b) { return (b->n_events + kTile - 1) / kTile; }

size_t scan_scratch_bytes(const xm_batch* b) {
  const int64_t nt = n_tiles_of(b);
  const size_t flat = 256 + size_t(nt) * (2 * sizeof(Mono) + 4 * kThreads) + 256;
  const size_t chunks = 256 + size_t(1024) * XM_K1C_CTAS_PER_SM * sizeof(ChunkSum);   // <= 512 SMs
  return std::max(flat, chunks);
}

// K1c's tensor map: the events as rows of 16 x 8-byte words, 128-row boxes,
// 128-byte swizzle. cuTensorMapEncodeTiled comes from the driver through the
// runtime's entry-point query (no link against libcuda).
static bool encode_event_map(const void* base, int64_t rows, CUtensorMap* tm) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  if (!enc) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn) {
      cudaGetLastError();
      return false;
    }
    enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const cuuint64_t dims[2] = {16, cuuint64_t(rows)};
  const cuuint64_t strides[1] = {128};
  const cuuint32_t box[2] = {16, cuuint32_t(kCRows)};   // one warp tile
  const cuuint32_t es[2] = {1, 1};
  return enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// K1 path: K1t when every trace fits one CTA's trace loop (<= kTraceMax
// events; measured faster there), else K1c; env XM_K1 = c | t | f(lat)
// forces one for tooling and tests
static char k1_path(const xm_batch* b) {
  const char* e = getenv("XM_K1");
  if (e && (e[0] == 't' || e[0] == 'f' || e[0] == 'c')) return e[0];
  return b->max_events <= uint32_t(kTraceMax) ? 't' : 'c';
}

static int launch_chunks(const xm_batch* b, const UnitConfig& u, void* d_scratch, xm_result* d_out,
                         cudaStream_t st, int* n_launches, bool* used) {
  *used = false;
  const void* ev = b->packed ? static_cast<const void*>(b->packed) : static_cast<const void*>(b->bytes);
  if (b->n_events <= 0 || (reinterpret_cast<uintptr_t>(ev) & 15)) return 0;
  const int64_t rows = b->n_events / 16;
  CUtensorMap tm;
  memset(&tm, 0, sizeof(tm));
  if (rows > 0 && !encode_event_map(ev, rows, &tm)) return 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  CParams P{};
  P.bytes = static_cast<const int64_t*>(ev);
  P.off = b->off;
  P.order = b->order;
  P.n_traces = b->n_traces;
  P.n_events = b->n_events;
  P.rows = rows;
  P.n_tiles = (b->n_events + kCTile - 1) / kCTile;
  P.unit_shift = u.unit_shift;
  P.u = u;
  P.done = static_cast<unsigned int*>(d_scratch) + 1;
  P.chunks = reinterpret_cast<ChunkSum*>(static_cast<char*>(d_scratch) + 256);
  P.out = d_out;
  const int64_t by_tiles = (P.n_tiles + kCWarps - 1) / kCWarps;          // >= 1 tile per warp
  const int G = int(std::max<int64_t>(1, std::min<int64_t>(by_tiles,
                                                           int64_t(std::min(sms, 1024)) * XM_K1C_CTAS_PER_SM)));
  cudaError_t e = cudaMemsetAsync(d_scratch, 0, 8, st);
  if (e != cudaSuccess) return int(e);
  const bool dv = u.div_shift != 0;
  auto kern = b->packed ? (dv ? k_scan_chunks<true, true> : k_scan_chunks<true, false>)
                        : (dv ? k_scan_chunks<false, true> : k_scan_chunks<false, false>);
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kCSmem);
  if (e != cudaSuccess) return int(e);
  kern<<<G, kCThreads, kCSmem, st>>>(tm, P);
  *n_launches += 1;
  *used = true;
  return int(cudaGetLastError());
}

int launch_scan(const xm_batch* b, const UnitConfig& u, void* d_scratch, size_t,
                xm_result* d_out, void* stream, int* n_launches) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  SParams P{};
  P.packed = b->packed != nullptr;
  P.bytes = b->packed ? reinterpret_cast<const int64_t*>(b->packed) : b->bytes;
  P.off = b->off;
  P.order = b->order;
  P.n_traces = b->n_traces;
  P.n_events = b->n_events;
  P.unit_shift = u.unit_shift;
  P.u = u;
  P.n_tiles = n_tiles_of(b);
  char* s = static_cast<char*>(d_scratch) + 256;
  P.tile_first = reinterpret_cast<Mono*>(s);
  s += size_t(P.n_tiles) * sizeof(Mono);
  P.tile_last = reinterpret_cast<Mono*>(s);
  s += size_t(P.n_tiles) * sizeof(Mono);
  P.row_trace = reinterpret_cast<uint32_t*>(s);
  P.out = d_out;
  P.work = static_cast<unsigned int*>(d_scratch);
  const char path = k1_path(b);
  if (path == 'c') {
    bool used = false;
    const int e = launch_chunks(b, u, d_scratch, d_out, st, n_launches, &used);
    if (e || used) return e;
  }
  if (path != 'f' && b->max_events <= uint32_t(kTraceMax)) {
    // every trace is short enough for one CTA: the trace-per-CTA path
    cudaError_t e = cudaMemsetAsync(d_scratch, 0, 4, st);
    if (e != cudaSuccess) return int(e);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // persistent grid = the CTAs resident at once (a CTA launched only when a
    // first-wave one exits would find the work gone and only delay the end)
    const bool dv = u.div_shift != 0;
    static int per_sm[4] = {0, 0, 0, 0};
    const int vi = (P.packed ? 2 : 0) + (dv ? 1 : 0);
    if (!per_sm[vi]) {
      const void* fn = P.packed ? (dv ? (const void*)k_scan_trace<true, true> : (const void*)k_scan_trace<true, false>)
                                : (dv ? (const void*)k_scan_trace<false, true> : (const void*)k_scan_trace<false, false>);
      int nb = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, kTThreads, 0) != cudaSuccess || nb < 1) nb = 1;
      per_sm[vi] = nb;
    }
    const int64_t grid = std::min<int64_t>(std::max<int64_t>(b->n_traces, 1), int64_t(sms) * per_sm[vi]);
    if (P.packed) {
      if (dv) k_scan_trace<true, true><<<unsigned(grid), kTThreads, 0, st>>>(P);
      else k_scan_trace<true, false><<<unsigned(grid), kTThreads, 0, st>>>(P);
    } else {
      if (dv) k_scan_trace<false, true><<<unsigned(grid), kTThreads, 0, st>>>(P);
      else k_scan_trace<false, false><<<unsigned(grid), kTThreads, 0, st>>>(P);
    }
    *n_launches += 1;
    return int(cudaGetLastError());
  }
  const int tb = 256;
  const int gt = int((b->n_traces + tb - 1) / tb);
  if (P.n_tiles > 0) {
    const int dsm = 2 * (kTile * 8 + kTile / 16 * 16);       // two staged tiles, 72 KB
    cudaError_t e = cudaFuncSetAttribute(k_scan_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, dsm);
    if (e != cudaSuccess) return int(e);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t grid = std::min<int64_t>(P.n_tiles, int64_t(sms) * 3);   // 3 CTAs/SM fit
    k_row_map<<<int((b->n_traces * 32 + tb - 1) / tb), tb, 0, st>>>(P);
    k_scan_tiles<<<unsigned(grid), kThreads, dsm, st>>>(P);
    *n_launches += 2;
  }
  k_scan_combine<<<gt > 0 ? gt : 1, tb, 0, st>>>(P);
  *n_launches += 1;
  return int(cudaGetLastError());
}

}  // namespace xm_internal
