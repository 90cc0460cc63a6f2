// scan.cu -- K1: allocated-bytes peak as a segmented prefix-scan/max (sm_100a).
//
// For every trace, peak_allocated = max over events i of sum_{k<=i} +-s_k with
// s_k the 512 B round-up of event k's request (PAPER.md:256 (i)
// "allocated_bytes changes by exactly the rounded request"; "the
// maximum value in this time series"), and its first index (reading Q7). No
// allocator state is needed for this quantity, so it is exact whenever no OOM
// truncates the trace (the mode requires unlimited capacity).
//
// Flat, trace-oblivious decomposition so that long traces never bound the
// launch (DESIGN.md §6 K1):
//   K1z  tile_trace[c] = trace owning the first event of tile c   (T threads)
//   K1a  one CTA per TILE-event tile: 8 contiguous events per thread, a
//        segmented scan of the monoid (sum, max-prefix, argmax) across the
//        CTA; traces wholly inside a tile are finished here, the tile's first
//        and last pieces are stored for the traces that cross tile edges
//   K1b  one thread per crossing trace folds its pieces (~len/TILE of them)
// HBM traffic: 8 B/event read once + ~52 B/tile + 64 B/trace written.
#include <cuda_runtime.h>

#include <cstdint>

#include "xm_internal.h"

namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr int kThreads = 256;
constexpr int kPer = 8;                      // events per thread
constexpr int kTile = kThreads * kPer;       // 2048 events per CTA
constexpr int kWarps = kThreads / 32;
constexpr int64_t kNeg = INT64_MIN;

// piece monoid: sum of deltas, max prefix (relative to the piece start), its
// flat event index. Identity: (0, kNeg, -1). combine(A, B) = A then B.
struct Mono {
  int64_t sum, mx, arg;
};

__device__ __forceinline__ Mono mono_id() { return Mono{0, kNeg, -1}; }

__device__ __forceinline__ Mono combine(const Mono& a, const Mono& b) {
  Mono r;
  r.sum = a.sum + b.sum;
  if (b.mx != kNeg && (a.mx == kNeg || a.sum + b.mx > a.mx)) {   // strict: first index wins
    r.mx = a.sum + b.mx;
    r.arg = b.arg;
  } else {
    r.mx = a.mx;
    r.arg = a.arg;
  }
  return r;
}

__device__ __forceinline__ int64_t rounded_delta(int64_t b, uint32_t sh) {
  const uint64_t mag = b > 0 ? uint64_t(b) : uint64_t(-b);
  const int64_t s = int64_t((mag + ((1ull << sh) - 1)) >> sh);
  return b > 0 ? s : -s;
}

struct SParams {
  const int64_t* __restrict__ bytes;
  const int64_t* __restrict__ off;
  int64_t n_traces, n_events;
  uint32_t unit_shift;
  int64_t n_tiles;
  uint32_t* tile_trace;     // [n_tiles]
  Mono* tile_first;         // [n_tiles] piece before the tile's first head
  Mono* tile_last;          // [n_tiles] piece from the tile's last head
  xm_result* out;
};

__device__ __forceinline__ void write_result(const SParams& P, uint32_t t, const Mono& m) {
  const int64_t o = P.off[t];
  xm_result R{};
  const int64_t mx = m.mx > 0 ? m.mx : 0;
  R.peak_allocated = uint64_t(mx) << P.unit_shift;
  R.peak_allocated_idx = m.mx > 0 ? uint32_t(m.arg - o) : 0u;
  R.events_done = uint32_t(P.off[t + 1] - o);
  R.status = XM_T_OK;
  P.out[t] = R;
}

// K1z: tile c's first event (c*kTile) lies in trace t iff off[t] <= c*kTile < off[t+1]
__global__ void k_tile_map(SParams P) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= P.n_traces) return;
  const int64_t a = P.off[t], b = P.off[t + 1];
  if (b <= a) return;
  for (int64_t c = (a + kTile - 1) / kTile; c * kTile < b; ++c) P.tile_trace[c] = uint32_t(t);
}

__device__ __forceinline__ Mono shfl_up_mono(const Mono& m, int o) {
  return Mono{__shfl_up_sync(kFull, m.sum, o), __shfl_up_sync(kFull, m.mx, o),
              __shfl_up_sync(kFull, m.arg, o)};
}

// segmented op: (fa, A) (+) (fb, B) = (fa | fb, fb ? B : A.B)
__device__ __forceinline__ void seg_combine(bool& fa, Mono& a, bool fb, const Mono& b) {
  a = fb ? b : combine(a, b);
  fa = fa || fb;
}

__global__ void __launch_bounds__(kThreads) k_scan_tiles(SParams P) {
  __shared__ int32_t head_pos[kTile];       // tile-relative positions of heads (sorted)
  __shared__ uint32_t head_trace[kTile];
  __shared__ int n_heads_s;
  __shared__ bool wflag[kWarps];
  __shared__ Mono wagg[kWarps];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t c = blockIdx.x;
  const int64_t t0e = c * kTile;
  const int64_t t1e = min(t0e + kTile, P.n_events);
  const uint32_t tf = P.tile_trace[c];

  // ---- load this thread's 8 contiguous events first (latency overlaps the head search) ----
  const int64_t g0 = t0e + int64_t(tid) * kPer;
  int64_t d[kPer];
  const long long* by = reinterpret_cast<const long long*>(P.bytes);
  if (g0 + kPer <= t1e) {
    const longlong2* v = reinterpret_cast<const longlong2*>(by + g0);
#pragma unroll
    for (int i = 0; i < kPer / 2; ++i) {
      const longlong2 x = __ldcs(v + i);
      d[2 * i] = x.x;                       // raw bytes; rounded in the local pass
      d[2 * i + 1] = x.y;
    }
  } else {
#pragma unroll
    for (int i = 0; i < kPer; ++i)
      d[i] = (g0 + i < t1e) ? __ldcs(by + g0 + i) : 0;
  }
  // ---- heads: starts of non-empty traces inside [t0e, t1e) ----
  if (tid == 0) n_heads_s = 0;
  __syncthreads();
  {
    const bool first_is_head = P.off[tf] == t0e;
    int64_t tb = first_is_head ? tf : int64_t(tf) + 1;
    for (;;) {
      const int64_t t = tb + tid;
      bool head = false;
      bool past = true;
      int64_t a = 0;
      if (t < P.n_traces) {
        a = P.off[t];
        past = a >= t1e;
        head = !past && P.off[t + 1] > a;
      }
      const unsigned hm = __ballot_sync(kFull, head);
      int base = 0;
      if (lane == 0 && hm) base = atomicAdd(&n_heads_s, __popc(hm));
      base = __shfl_sync(kFull, base, 0);
      if (head) {
        const int k = base + __popc(hm & ((1u << lane) - 1u));
        head_pos[k] = int32_t(a - t0e);
        head_trace[k] = uint32_t(t);
      }
      // more traces may start in this tile iff the chunk's last one did not pass it
      const int any_more = __syncthreads_or(tid == kThreads - 1 && !past);
      if (!any_more) break;
      tb += kThreads;
    }
  }
  __syncthreads();
  const int nh = n_heads_s;
  // warps appended in arbitrary order: sort heads by position (few; insertion
  // sort by one thread is fine when nh is small, else a simple parallel rank)
  if (nh > 1) {
    __shared__ int32_t tmp_pos[kTile];
    __shared__ uint32_t tmp_tr[kTile];
    for (int k = tid; k < nh; k += kThreads) { tmp_pos[k] = head_pos[k]; tmp_tr[k] = head_trace[k]; }
    __syncthreads();
    for (int k = tid; k < nh; k += kThreads) {
      const int32_t p = tmp_pos[k];
      int r = 0;
      for (int q = 0; q < nh; ++q) r += tmp_pos[q] < p;   // positions are distinct
      head_pos[r] = p;
      head_trace[r] = tmp_tr[k];
    }
    __syncthreads();
  }

  // heads inside [rel0, rel0 + kPer)
  const int rel0 = tid * kPer;
  int h0 = 0;                               // first head index with pos >= rel0
  {
    int lo = 0, hi = nh;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (head_pos[mid] < rel0) lo = mid + 1; else hi = mid;
    }
    h0 = lo;
  }
  unsigned hb = 0;
  for (int k = h0; k < nh && head_pos[k] < rel0 + kPer; ++k) hb |= 1u << (head_pos[k] - rel0);

  // ---- thread-local segmented pass ----
  Mono cur = mono_id(), first_piece = mono_id();
  bool seen = false;
  int hk = h0;                              // index of the next head in this thread
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    if ((hb >> i) & 1u) {
      if (!seen) {
        first_piece = cur;
        seen = true;
      } else {
        write_result(P, head_trace[hk - 1], cur);  // trace wholly inside this thread
      }
      ++hk;
      cur = mono_id();
    }
    if (g0 + i < t1e) {
      const int64_t x = rounded_delta(d[i], P.unit_shift);
      cur = combine(cur, Mono{x, x, g0 + i});
    }
  }
  // ---- CTA exclusive segmented scan of (seen, cur) ----
  bool f = seen;
  Mono a = cur;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const Mono b = shfl_up_mono(a, o);
    const bool fb = __shfl_up_sync(kFull, f, o);
    if (lane >= o) {            // (fb, b) precedes (f, a)
      Mono x = b;
      bool fx = fb;
      seg_combine(fx, x, f, a);
      a = x;
      f = fx;
    }
  }
  if (lane == 31) { wflag[warp] = f; wagg[warp] = a; }
  __syncthreads();
  // carry into this warp: fold of warps before it
  bool cf = false;
  Mono cw = mono_id();
  for (int w = 0; w < warp; ++w) seg_combine(cf, cw, wflag[w], wagg[w]);
  // exclusive within warp
  Mono ex = Mono{__shfl_up_sync(kFull, a.sum, 1), __shfl_up_sync(kFull, a.mx, 1),
                 __shfl_up_sync(kFull, a.arg, 1)};
  bool exf = __shfl_up_sync(kFull, f, 1);
  if (lane == 0) { ex = mono_id(); exf = false; }
  bool carry_f = cf;
  Mono carry = cw;
  seg_combine(carry_f, carry, exf, ex);     // carry = everything before this thread

  if (seen) {
    const Mono done = combine(carry, first_piece);
    if (carry_f) {
      // the piece ending at this thread's first head started at a head in this tile
      if (h0 > 0) write_result(P, head_trace[h0 - 1], done);
    } else {
      P.tile_first[c] = done;               // tile prefix piece (trace crossed in)
    }
  }
  // last thread with events owns the tile's tail piece
  const int last_tid = int((t1e - t0e - 1) / kPer);
  if (tid == last_tid) {
    bool lf = carry_f;
    Mono lm = carry;
    seg_combine(lf, lm, seen, cur);
    if (nh == 0) {
      P.tile_first[c] = lm;                 // no head: the whole tile is one piece
      P.tile_last[c] = lm;
    } else {
      const uint32_t tl = head_trace[nh - 1];
      if (P.off[tl + 1] <= t1e) write_result(P, tl, lm);   // last trace ends in tile
      else P.tile_last[c] = lm;
    }
  }
}

// K1b: fold pieces of traces that cross tile boundaries; empty traces -> zeros
__global__ void k_scan_combine(SParams P) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= P.n_traces) return;
  const int64_t a = P.off[t], b = P.off[t + 1];
  if (b <= a) {
    xm_result R{};
    P.out[t] = R;
    return;
  }
  const int64_t ca = a / kTile, cb = (b - 1) / kTile;
  if (ca == cb) return;                     // finished by k_scan_tiles
  Mono m = P.tile_last[ca];
  for (int64_t c = ca + 1; c <= cb; ++c) m = combine(m, P.tile_first[c]);
  write_result(P, uint32_t(t), m);
}

}  // namespace

namespace xm_internal {

static int64_t n_tiles_of(const xm_batch* b) { return (b->n_events + kTile - 1) / kTile; }

size_t scan_scratch_bytes(const xm_batch* b) {
  const int64_t nt = n_tiles_of(b);
  return 256 + size_t(nt) * (4 + 2 * sizeof(Mono)) + 256;
}

int launch_scan(const xm_batch* b, const UnitConfig& u, void* d_scratch, size_t,
                xm_result* d_out, void* stream, int* n_launches) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  SParams P{};
  P.bytes = b->bytes;
  P.off = b->off;
  P.n_traces = b->n_traces;
  P.n_events = b->n_events;
  P.unit_shift = u.unit_shift;
  P.n_tiles = n_tiles_of(b);
  char* s = static_cast<char*>(d_scratch) + 256;
  P.tile_first = reinterpret_cast<Mono*>(s);
  s += size_t(P.n_tiles) * sizeof(Mono);
  P.tile_last = reinterpret_cast<Mono*>(s);
  s += size_t(P.n_tiles) * sizeof(Mono);
  P.tile_trace = reinterpret_cast<uint32_t*>(s);
  P.out = d_out;
  const int tb = 256;
  const int gt = int((b->n_traces + tb - 1) / tb);
  if (P.n_tiles > 0) {
    k_tile_map<<<gt, tb, 0, st>>>(P);
    k_scan_tiles<<<unsigned(P.n_tiles), kThreads, 0, st>>>(P);
    *n_launches += 2;
  }
  k_scan_combine<<<gt > 0 ? gt : 1, tb, 0, st>>>(P);
  *n_launches += 1;
  return int(cudaGetLastError());
}

}  // namespace xm_internal
