// replay.cu -- K2: batched caching-allocator replay, one warp per trace (sm_100a).
//
// Computes xMem's Simulator (§3.4) for every trace of a
// batch: (i) round-up, (ii) segment sizing, (iii) best-fit-with-coalescing
// search / split / merge, (iv) caching, (v) two-level OOM with reclamation,
// plus the time-series peaks. Rules and readings: DESIGN.md
// §Readings; per-step citations inline.
//
// Execution model:
//  * persistent grid, one trace per warp, traces pulled longest-first from a
//    global atomic work counter (host LPT order);
//  * a trace's allocator state lives in the warp's shared-memory slot when it
//    fits, else (or when the free list outgrows the slot) in the warp's
//    global-memory arena, sized so it cannot overflow;
//  * events stream through registers in 32-event tiles (coalesced loads,
//    next tile prefetched while the current one is replayed); the allocated
//    peak of each tile is a warp prefix-scan/max (a3);
//  * the serial state machine is warp-uniform; the best-fit search is a
//    warp-strided scan of the free list + ballot/__reduce_min_sync (a5).
//
// State (structure of arrays; 21 B per record):
//  A[id]  allocated block of dense id: pos u64, size u32, prev u32, next u32, cls u8
//  F[f]   free block f (unordered list, nf entries): same fields
//  pos  = segment_index << 32 | offset_in_units  (bump addresses never reused:
//         (size, pos) order == SPEC D2's (size, segment, offset), reading Q4)
//  prev/next = address-order neighbours in the segment: kNone, an id, or kF|f
//  cls  = stream << 1 | small_pool
#include <cuda_runtime.h>

#include "xm_internal.h"

namespace {

constexpr uint32_t kNone = 0xFFFFFFFFu;
constexpr uint32_t kF = 0x80000000u;
constexpr uint32_t kIdMask = 0x07FFFFFFu;
constexpr uint32_t kAllocBit = 0x08000000u;
constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr int kStatusOk = XM_T_OK, kStatusOom = XM_T_OOM, kStatusOverflow = XM_T_OVERFLOW;

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
  uint32_t smem_per_warp;
  uint32_t* counter;
  unsigned char* arena;
  size_t arena_per_warp;
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
  uint32_t* F_size;
  uint32_t* F_prev;
  uint32_t* F_next;
  uint8_t* F_cls;
  uint32_t cap_f;
};

constexpr size_t kRecordBytes = 21;

__host__ __device__ inline size_t state_bytes(uint32_t na, uint32_t nf) {
  return size_t(na + nf) * kRecordBytes + 16;
}

__host__ __device__ inline uint32_t free_cap(size_t budget, uint32_t na) {
  size_t need = size_t(na) * kRecordBytes + 16;
  if (budget <= need) return 0;
  size_t c = (budget - need) / kRecordBytes;
  return c > 0x7FFFFFFFu ? 0x7FFFFFFFu : uint32_t(c);
}

__device__ inline State carve(unsigned char* base, uint32_t na, uint32_t nf) {
  State S;
  unsigned char* p = base;
  S.A_pos = reinterpret_cast<uint64_t*>(p); p += size_t(na) * 8;
  S.F_pos = reinterpret_cast<uint64_t*>(p); p += size_t(nf) * 8;
  S.A_size = reinterpret_cast<uint32_t*>(p); p += size_t(na) * 4;
  S.A_prev = reinterpret_cast<uint32_t*>(p); p += size_t(na) * 4;
  S.A_next = reinterpret_cast<uint32_t*>(p); p += size_t(na) * 4;
  S.F_size = reinterpret_cast<uint32_t*>(p); p += size_t(nf) * 4;
  S.F_prev = reinterpret_cast<uint32_t*>(p); p += size_t(nf) * 4;
  S.F_next = reinterpret_cast<uint32_t*>(p); p += size_t(nf) * 4;
  S.A_cls = p; p += na;
  S.F_cls = p;
  S.cap_f = nf;
  return S;
}

__device__ __forceinline__ void set_next(const State& S, uint32_t ref, uint32_t v) {
  if (ref == kNone) return;
  if (ref & kF) S.F_next[ref & ~kF] = v;
  else S.A_next[ref] = v;
}

__device__ __forceinline__ void set_prev(const State& S, uint32_t ref, uint32_t v) {
  if (ref == kNone) return;
  if (ref & kF) S.F_prev[ref & ~kF] = v;
  else S.A_prev[ref] = v;
}

// Remove free entry f by moving the last entry into its slot (warp-uniform).
__device__ __forceinline__ void f_remove(const State& S, uint32_t f, uint32_t& nf) {
  const uint32_t L = nf - 1;
  if (f != L) {
    const uint32_t sz = S.F_size[L], pv = S.F_prev[L], nx = S.F_next[L];
    const uint64_t pos = S.F_pos[L];
    const uint8_t c = S.F_cls[L];
    S.F_size[f] = sz; S.F_pos[f] = pos; S.F_prev[f] = pv; S.F_next[f] = nx; S.F_cls[f] = c;
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
__device__ void reclaim(const State& S, uint32_t& nf, uint64_t& reserved, uint32_t& n_release,
                        uint32_t& live_segs) {
  const uint32_t lane = threadIdx.x & 31;
  uint32_t newn = 0, cnt = 0;
  uint64_t freed = 0;
  for (uint32_t base = 0; base < nf; base += 32) {
    const uint32_t f = base + lane;
    const bool valid = f < nf;
    uint32_t sz = 0, pv = kNone, nx = kNone;
    uint64_t pos = 0;
    uint8_t c = 0;
    if (valid) {
      sz = S.F_size[f]; pv = S.F_prev[f]; nx = S.F_next[f]; pos = S.F_pos[f]; c = S.F_cls[f];
    }
    const bool whole = valid && pv == kNone && nx == kNone;
    const bool keep = valid && !whole;
    const unsigned km = __ballot_sync(kFull, keep);
    const unsigned wm = __ballot_sync(kFull, whole);
    const uint64_t fs = warp_sum_u64(whole ? uint64_t(sz) : 0ull);
    const uint32_t dst = newn + __popc(km & ((1u << lane) - 1u));
    __syncwarp();
    if (keep && dst != f) {
      S.F_size[dst] = sz; S.F_pos[dst] = pos; S.F_prev[dst] = pv; S.F_next[dst] = nx; S.F_cls[dst] = c;
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

struct Peaks {
  uint64_t tensor_pk, blk_pk, res_pk;
  uint32_t tensor_ix, blk_ix, res_ix;
};

// Replays events [e0, e0+n) of one trace on state S. Returns status; on
// XM_T_OVERFLOW the caller restarts the trace on a larger arena.
__device__ int replay_trace(const KParams& P, const State& S, int64_t e0, uint32_t n,
                            uint64_t cap_u, xm_result& R) {
  const uint32_t lane = threadIdx.x & 31;
  const xm_internal::UnitConfig& u = P.u;
  const uint64_t unit_m1 = (1ull << u.unit_shift) - 1;

  uint32_t nf = 0, nseg = 0, live_segs = 0, max_live = 0, n_release = 0;
  uint64_t reserved = 0, blk = 0;
  int64_t tensor = 0;
  Peaks pk{0, 0, 0, 0, 0, 0};
  int status = kStatusOk;
  uint32_t done_total = 0;

  // tile prefetch registers
  int64_t b_nx = 0;
  uint32_t t_nx = 0;
  if (lane < n) {
    b_nx = __ldcs(reinterpret_cast<const long long*>(P.bytes) + e0 + lane);
    t_nx = __ldcs(P.tag + e0 + lane);
  }
  for (uint32_t base = 0; base < n; base += 32) {
    const int64_t bc = b_nx;
    const uint32_t tc = t_nx;
    const uint32_t cnt = min(32u, n - base);
    if (base + 32 + lane < n) {
      b_nx = __ldcs(reinterpret_cast<const long long*>(P.bytes) + e0 + base + 32 + lane);
      t_nx = __ldcs(P.tag + e0 + base + 32 + lane);
    }
    // ---- a2: round-up of this lane's event (PAPER.md:256 (i)) ----
    const bool valid = lane < cnt;
    const bool is_alloc = bc > 0;
    const uint64_t mag = is_alloc ? uint64_t(bc) : uint64_t(-bc);
    const uint32_t su = uint32_t((mag + unit_m1) >> u.unit_shift);
    // ---- a3: tile prefix-scan of +-s (allocated tensor bytes) ----
    int64_t d = valid ? (is_alloc ? int64_t(su) : -int64_t(su)) : 0;
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
        const uint32_t small = s <= u.small_u;                  // a4: pool
        const uint8_t cls = uint8_t(((w >> 28) << 1) | small);  // per-stream pools (Q5)
        // a5: best fit = min (size, pos) over free blocks of this class with size >= s
        uint32_t bsz = kNone, bf = kNone;
        uint64_t bpos = ~0ull;
        for (uint32_t f = lane; f < nf; f += 32) {
          const uint32_t sz = S.F_size[f];
          const uint8_t c = S.F_cls[f];
          if (c == cls && sz >= s) {
            const uint64_t pos = S.F_pos[f];
            if (sz < bsz || (sz == bsz && pos < bpos)) { bsz = sz; bpos = pos; bf = f; }
          }
        }
        const uint32_t m = __reduce_min_sync(kFull, bsz);
        uint32_t fsel = kNone;
        if (m != kNone) {
          const unsigned tie = __ballot_sync(kFull, bsz == m);
          int wl;
          if ((tie & (tie - 1u)) == 0u) {
            wl = __ffs(tie) - 1;
          } else {
            const uint32_t hi = bsz == m ? uint32_t(bpos >> 32) : kNone;
            const uint32_t mh = __reduce_min_sync(kFull, hi);
            const uint32_t lo = (bsz == m && hi == mh) ? uint32_t(bpos) : kNone;
            const uint32_t ml = __reduce_min_sync(kFull, lo);
            wl = __ffs(__ballot_sync(kFull, bsz == m && hi == mh && uint32_t(bpos) == ml)) - 1;
          }
          fsel = __shfl_sync(kFull, bf, wl);
        }
        uint32_t bsize, bprev, bnext;
        uint64_t bposu;
        if (fsel == kNone) {
          // a4/a6: new segment from the device level (PAPER.md:259 (iv), 169, 654)
          uint32_t a;
          if (small) a = u.sbuf_u;
          else if (s < u.minlarge_u) a = u.lbuf_u;
          else a = uint32_t((uint64_t(s) + u.rlarge_u - 1) / u.rlarge_u * u.rlarge_u);
          if (reserved + a > cap_u) {                 // device level refuses (Q10)
            reclaim(S, nf, reserved, n_release, live_segs);   // reclaim cached segments (Q3)
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
        } else {
          bsize = S.F_size[fsel];
          bprev = S.F_prev[fsel];
          bnext = S.F_next[fsel];
          bposu = S.F_pos[fsel];
        }
        // a7: split (PAPER.md:258 (iii); reading Q1)
        const uint32_t rem = bsize - s;
        const bool split = small ? (rem >= 1u) : (u.strict ? (rem > u.small_u) : (rem >= u.small_u));
        if (split) {
          uint32_t r;
          if (fsel != kNone) {
            r = fsel;                                // remainder keeps the free entry
          } else {
            if (nf >= S.cap_f) { status = kStatusOverflow; break; }
            r = nf++;
            S.F_next[r] = kNone;                     // new segment: no right neighbour
            S.F_cls[r] = cls;
          }
          S.F_pos[r] = bposu + s;
          S.F_size[r] = rem;
          S.F_prev[r] = id;
          S.A_size[id] = s;
          S.A_next[id] = kF | r;
        } else {
          S.A_size[id] = bsize;
          S.A_next[id] = bnext;
          set_prev(S, bnext, id);
          if (fsel != kNone) f_remove(S, fsel, nf);
        }
        S.A_pos[id] = bposu;
        S.A_prev[id] = bprev;
        S.A_cls[id] = cls;
        set_next(S, bprev, id);
        blk += split ? s : bsize;
      } else {
        // ================= FREE =================
        const uint32_t sz = S.A_size[id];
        const uint32_t p = S.A_prev[id];
        const uint32_t q = S.A_next[id];
        const uint64_t pos = S.A_pos[id];
        const uint8_t cls = S.A_cls[id];
        blk -= sz;
        const bool pf = p != kNone && (p & kF);
        const bool qf = q != kNone && (q & kF);
        // a8: coalesce with free neighbours; reserved unchanged (PAPER.md:259 (iv))
        if (pf && qf) {
          const uint32_t P_ = p & ~kF, N_ = q & ~kF;
          const uint32_t nn = S.F_next[N_];
          S.F_size[P_] = S.F_size[P_] + sz + S.F_size[N_];
          S.F_next[P_] = nn;
          set_prev(S, nn, p);
          f_remove(S, N_, nf);
        } else if (pf) {
          const uint32_t P_ = p & ~kF;
          S.F_size[P_] = S.F_size[P_] + sz;
          S.F_next[P_] = q;
          set_prev(S, q, p);
        } else if (qf) {
          const uint32_t N_ = q & ~kF;
          S.F_pos[N_] = pos;
          S.F_size[N_] = S.F_size[N_] + sz;
          S.F_prev[N_] = p;
          set_next(S, p, q);
        } else {
          if (nf >= S.cap_f) { status = kStatusOverflow; break; }
          const uint32_t r = nf++;
          S.F_pos[r] = pos; S.F_size[r] = sz; S.F_prev[r] = p; S.F_next[r] = q; S.F_cls[r] = cls;
          set_next(S, p, kF | r);
          set_prev(S, q, kF | r);
        }
      }
      // a9: time series peaks, first index (Q7)
      const uint32_t ev = base + j;
      if (blk > pk.blk_pk) { pk.blk_pk = blk; pk.blk_ix = ev; }
      if (reserved > pk.res_pk) { pk.res_pk = reserved; pk.res_ix = ev; }
      __syncwarp();
    }
    // a3: allocated-tensor peak over the processed prefix of this tile
    const int64_t v = lane < j ? cur : INT64_MIN;
    const int64_t mx = warp_max_i64(v);
    if (j > 0 && mx > int64_t(pk.tensor_pk)) {
      const unsigned bm = __ballot_sync(kFull, v == mx);
      pk.tensor_pk = uint64_t(mx);
      pk.tensor_ix = base + __ffs(bm) - 1;
    }
    tensor = __shfl_sync(kFull, cur, 31);
    done_total = base + j;
    if (status != kStatusOk) break;
  }
  const uint32_t sh = u.unit_shift;
  R.peak_allocated = pk.tensor_pk << sh;
  R.peak_allocated_blk = pk.blk_pk << sh;
  R.peak_reserved = pk.res_pk << sh;
  R.final_reserved = reserved << sh;
  R.peak_allocated_idx = pk.tensor_ix;
  R.peak_allocated_blk_idx = pk.blk_ix;
  R.peak_reserved_idx = pk.res_ix;
  R.n_seg_alloc = nseg;
  R.n_seg_release = n_release;
  R.max_live_segments = max_live;
  R.events_done = status == kStatusOk ? n : done_total;
  R.status = uint16_t(status);
  R.n_free_blocks_end = uint16_t(nf > 0xFFFFu ? 0xFFFFu : nf);
  return status;
}

__global__ void __launch_bounds__(256) k_replay(KParams P) {
  extern __shared__ __align__(16) unsigned char smem[];
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warp = threadIdx.x >> 5;
  const uint32_t gwarp = blockIdx.x * (blockDim.x >> 5) + warp;
  unsigned char* my_smem = smem + size_t(warp) * P.smem_per_warp;
  unsigned char* my_arena = P.arena + size_t(gwarp) * P.arena_per_warp;
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
    int st = kStatusOverflow;
    const uint32_t fc = free_cap(P.smem_per_warp, na);
    if (fc >= 32) {
      const State S = carve(my_smem, na, fc);
      st = replay_trace(P, S, e0, n, cap_u, R);
    }
    if (st == kStatusOverflow && na <= P.arena_ids) {
      const State S = carve(my_arena, na, P.arena_free);
      st = replay_trace(P, S, e0, n, cap_u, R);
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
  p.warps_per_cta = cfg->warps_per_cta ? int(cfg->warps_per_cta) : 4;
  if (p.warps_per_cta > 8) p.warps_per_cta = 8;
  uint32_t spw = cfg->smem_per_warp;
  if (spw == 0) {
    // enough for the largest id space plus a free list of 512 entries, capped so
    // that 4 warps fit in one SM's 227 KB
    size_t want = state_bytes(b->max_ids, 512);
    size_t capb = (227u * 1024u) / size_t(p.warps_per_cta);
    spw = uint32_t(want < capb ? want : capb);
    if (spw < 4096) spw = 4096;
  }
  spw = (spw + 15u) & ~15u;
  p.smem_per_warp = spw;
  const size_t smem_cta = size_t(spw) * p.warps_per_cta;
  int per_sm = smem_cta ? int((227u * 1024u) / smem_cta) : 8;
  if (per_sm < 1) per_sm = 1;
  if (per_sm * p.warps_per_cta > 64) per_sm = 64 / p.warps_per_cta;
  p.ctas = sms * per_sm;
  const int64_t warps_total = int64_t(p.ctas) * p.warps_per_cta;
  if (b->n_traces < warps_total) {
    p.ctas = int((b->n_traces + p.warps_per_cta - 1) / p.warps_per_cta);
    if (p.ctas < 1) p.ctas = 1;
  }
  // global arena: exact bound (nf <= n_events, SPEC invariants; K2)
  p.arena_ids = b->max_ids;
  p.arena_free = b->max_events + 1;
  p.arena_per_warp = (state_bytes(p.arena_ids, p.arena_free) + 255) & ~size_t(255);
  p.scratch_bytes = 256 + size_t(p.ctas) * p.warps_per_cta * p.arena_per_warp;
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
  P.smem_per_warp = plan.smem_per_warp;
  P.counter = static_cast<uint32_t*>(d_scratch);
  P.arena = static_cast<unsigned char*>(d_scratch) + 256;
  P.arena_per_warp = plan.arena_per_warp;
  P.arena_ids = plan.arena_ids;
  P.arena_free = plan.arena_free;
  P.out = d_out;
  cudaError_t e = cudaMemsetAsync(d_scratch, 0, 256, st);
  if (e != cudaSuccess) return int(e);
  const size_t smem = size_t(plan.smem_per_warp) * plan.warps_per_cta;
  e = cudaFuncSetAttribute(k_replay, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return int(e);
  k_replay<<<plan.ctas, plan.warps_per_cta * 32, smem, st>>>(P);
  *n_launches += 1;
  return int(cudaGetLastError());
}

}  // namespace xm_internal
