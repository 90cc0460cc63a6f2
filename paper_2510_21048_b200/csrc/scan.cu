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
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

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
__global__ void __launch_bounds__(kTThreads) k_scan_trace(SParams P) {
  __shared__ long long s_sum[kTWarps], s_mx[kTWarps];
  __shared__ int s_arg[kTWarps];
  __shared__ unsigned int s_k;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const long long* by = reinterpret_cast<const long long*>(P.bytes);
  for (;;) {
    if (tid == 0) s_k = atomicAdd(P.work, 1u);
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

}  // namespace

namespace xm_internal {

static int64_t n_tiles_of(const xm_batch* b) { return (b->n_events + kTile - 1) / kTile; }

size_t scan_scratch_bytes(const xm_batch* b) {
  const int64_t nt = n_tiles_of(b);
  return 256 + size_t(nt) * (2 * sizeof(Mono) + 4 * kThreads) + 256;
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
  if (b->max_events <= uint32_t(kTraceMax)) {
    // every trace is short enough for one CTA: the trace-per-CTA path
    cudaError_t e = cudaMemsetAsync(d_scratch, 0, 4, st);
    if (e != cudaSuccess) return int(e);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t grid = std::min<int64_t>(std::max<int64_t>(b->n_traces, 1), int64_t(sms) * (64 / kTWarps));
    const bool dv = u.div_shift != 0;
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
