// orchestrate.cu -- K6: batched Memory Orchestrator (
// PAPER.md:239-248 §3.3), the step directly before the
// Simulator: classify the Analyzer's blocks by the training-loop windows,
// re-time them for the analysis iteration and emit the ordered sequence
// (ts, Free before Alloc, block) that k_replay consumes. Rules and readings:
// DESIGN.md §2 (Q22-Q25), restated in include/xmem.h.
//
//   k_orchestrate  one CTA (16 warps) per trace, persistent:
//     1. parameters (persistent, allocated before the first iteration) and
//        optimizer-step candidates are listed (CTA-wide atomics);
//     2. a candidate is optimizer state iff fewer than 2 x (#parameters of
//        its size) earlier candidates have its size (the quota consumed in
//        allocation order, SPEC D3): candidates sorted by (size, block) and
//        parameter sizes sorted (bitonic), then binary searches;
//     3. every block: class (priority Parameter > OptState > Gradient >
//        BatchData > Activation > Other), re-timed allocation / free, and
//        64-bit keys (ts - Ws) << 32 | kind << 31 | block;
//     4. bitonic sort of the keys in shared memory (global scratch for traces
//        of more than 4096 blocks; two CTAs per SM);
//     5. warp 0 walks the sorted keys in 32-event tiles, assigns dense block
//        ids (allocations take ids freed before the tile, else fresh ids) and
//        stages the wire events at the trace's 2 x block offset;
//   k_owire_offsets / k_owire_compact  stored (e.g. longest-first) order ->
//        dense xm_batch arrays.
#include <cuda_runtime.h>

#include <cstring>

#include "xm_internal.h"

namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr int kThreads = 512;
#ifndef XM_ORCH_SMEM_KEYS
#define XM_ORCH_SMEM_KEYS 8192    // 64 KB: two CTAs per SM (the register limit at 512 threads)
#endif
constexpr int kSmemKeys = XM_ORCH_SMEM_KEYS;  // keys in shared memory (8 B each)
constexpr int kCtasPerSm = kSmemKeys > 8192 ? 1 : 2;
constexpr int kBlockBits = 23;            // quota keys: size << 23 | block (< 2^23 blocks,
constexpr uint64_t kBlockMask = (1ull << kBlockBits) - 1;   // sizes < 2^41 bytes)
enum { kParam = 0, kState, kGrad, kData, kAct, kOther };
enum { wIt = 0, wData, wFw, wBw, wZg, wOpt };

struct OParams {
  const int64_t* __restrict__ alloc_ts;
  const int64_t* __restrict__ free_ts;
  const int64_t* __restrict__ size;
  const uint8_t* __restrict__ stream;
  const int64_t* __restrict__ boff;
  const int64_t* __restrict__ win;        // [iters][6][2]
  const int64_t* __restrict__ woff;
  int64_t n_traces;
  uint32_t analysis;
  uint32_t max_blocks;
  // per-CTA scratch regions
  uint32_t* cand;                         // [ctas][max_blocks] candidate block indices
  int64_t* psize;                         // [ctas][max_blocks] parameter sizes
  uint32_t* id_of;                        // [ctas][max_blocks]
  uint32_t* idstack;                      // [ctas][max_blocks]
  unsigned long long* gkeys;              // [ctas][keys_cap] (large traces)
  uint32_t keys_cap;
  // outputs
  uint8_t* cls;                           // [n_blocks]
  unsigned long long* seq;                // [2 n_blocks] sorted keys at 2 boff[t]
  xm_orchestrated* rec;
  int64_t* st_bytes;                      // [2 n_blocks] staged wire events
  uint32_t* st_tag;
  unsigned int* work;
};

__device__ __forceinline__ bool inside(int64_t ts, const int64_t* w) {
  return w[0] >= 0 && w[0] <= ts && ts <= w[1];
}

// in-place ascending bitonic sort of n (power of two) keys, CTA-wide
__device__ void bitonic(unsigned long long* k, uint32_t n) {
  for (uint32_t len = 2; len <= n; len <<= 1) {
    for (uint32_t j = len >> 1; j > 0; j >>= 1) {
      for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        const uint32_t p = i ^ j;
        if (p > i) {
          const bool up = (i & len) == 0;
          const unsigned long long a = k[i], b = k[p];
          if ((a > b) == up) { k[i] = b; k[p] = a; }
        }
      }
      __syncthreads();
    }
  }
}

__global__ void __launch_bounds__(kThreads, kCtasPerSm) k_orchestrate(OParams P) {
  extern __shared__ __align__(16) unsigned long long skeys[];
  __shared__ unsigned int s_trace, s_ncand, s_npar, s_nkeys, s_bad;
  __shared__ unsigned int s_ncls[6];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t* cand = P.cand + size_t(blockIdx.x) * P.max_blocks;
  int64_t* psize = P.psize + size_t(blockIdx.x) * P.max_blocks;
  uint32_t* id_of = P.id_of + size_t(blockIdx.x) * P.max_blocks;
  uint32_t* ids = P.idstack + size_t(blockIdx.x) * P.max_blocks;
  for (;;) {
    if (tid == 0) {
      s_trace = atomicAdd(P.work, 1u);
      s_ncand = s_npar = s_nkeys = s_bad = 0;
      for (int c = 0; c < 6; ++c) s_ncls[c] = 0;
    }
    __syncthreads();
    const unsigned t = s_trace;
    if (int64_t(t) >= P.n_traces) break;
    const int64_t b0 = P.boff[t];
    const int n = int(P.boff[t + 1] - b0);
    const int64_t* W = P.win + 12 * P.woff[t];
    const int nit = int(P.woff[t + 1] - P.woff[t]);
    const int64_t* A = P.alloc_ts + b0;
    const int64_t* F = P.free_ts + b0;
    const int64_t* S = P.size + b0;
    xm_orchestrated R{};
    if (nit < int(P.analysis) + 1) {                    // SPEC.md:166 needs >= 2 iterations
      if (tid == 0) { R.status = XM_O_FEW_ITERATIONS; P.rec[t] = R; }
      __syncthreads();
      continue;
    }
    const int64_t first = W[12 * 0 + 2 * wIt];
    const int64_t* Wa = W + 12 * P.analysis;
    const int64_t Ws = Wa[2 * wIt], We = Wa[2 * wIt + 1];
    const int64_t zg_end = Wa[2 * wZg] >= 0 ? Wa[2 * wZg + 1] : -1;
    // ---- 1. parameters and optimizer-step candidates ----
    for (int i = tid; i < n; i += kThreads) {
      const int64_t a = A[i];
      if (S[i] <= 0 || uint64_t(S[i]) >= XM_MAX_REQUEST) atomicExch(&s_bad, 1u);   // sizes in (0, 2^40): the replay's bound
      if (F[i] == -1 && a < first) {
        psize[atomicAdd(&s_npar, 1u)] = S[i];
      } else {
        bool in_opt = false;
        for (int k = 0; k < nit; ++k) in_opt |= inside(a, W + 12 * k + 2 * wOpt);
        if (in_opt) {
          cand[atomicAdd(&s_ncand, 1u)] = uint32_t(i);
          P.cls[b0 + i] = kOther;                       // step 2 may mark it kState
        }
      }
    }
    __syncthreads();
    const uint32_t nc = s_ncand, np = s_npar;
    // ---- 2. the quota: a candidate is state iff fewer than 2 x (parameters of
    // its size) earlier candidates have its size. Sort the candidates by
    // (size, block) and the parameter sizes (bitonic, in the key buffer); a
    // candidate's rank in its size run and the run length of its size among
    // the parameters are then two binary searches. ----
    const bool big = 2 * n > kSmemKeys;
    unsigned long long* keys = big ? P.gkeys + size_t(blockIdx.x) * P.keys_cap : skeys;
    {
      uint32_t cpow = 1, ppow = 1;
      while (cpow < nc) cpow <<= 1;
      while (ppow < np) ppow <<= 1;
      unsigned long long* ck = keys;
      unsigned long long* pk = keys + cpow;
      for (uint32_t c = tid; c < cpow; c += kThreads)
        ck[c] = c < nc ? (uint64_t(S[cand[c]]) << kBlockBits) | cand[c] : ~0ull;
      for (uint32_t q = tid; q < ppow; q += kThreads) pk[q] = q < np ? uint64_t(psize[q]) : ~0ull;
      __syncthreads();
      if (nc > 1) bitonic(ck, cpow);
      if (np > 1) bitonic(pk, ppow);
      for (uint32_t c = tid; c < nc; c += kThreads) {
        const unsigned long long key = ck[c];
        const uint64_t sz = key >> kBlockBits;
        uint32_t lo = 0, hi = c;                         // first candidate of this size
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if ((ck[mid] >> kBlockBits) < sz) lo = mid + 1; else hi = mid;
        }
        const uint32_t rank = c - lo;
        uint32_t a0 = 0, a1 = np;                        // parameters of this size
        while (a0 < a1) {
          const uint32_t mid = (a0 + a1) >> 1;
          if (pk[mid] < sz) a0 = mid + 1; else a1 = mid;
        }
        uint32_t b1 = a0, b2 = np;
        while (b1 < b2) {
          const uint32_t mid = (b1 + b2) >> 1;
          if (pk[mid] <= sz) b1 = mid + 1; else b2 = mid;
        }
        if (rank < 2 * (b1 - a0)) P.cls[b0 + uint32_t(key & kBlockMask)] = kState;
      }
      __syncthreads();
    }
    // ---- 3. classes, re-timing, keys ----
    for (int i = tid; i < n; i += kThreads) {
      const int64_t a = A[i];
      int64_t f = F[i];
      const bool param = f == -1 && a < first;
      bool state = false;
      if (!param) {
        bool in_opt = false;
        for (int k = 0; k < nit; ++k) in_opt |= inside(a, W + 12 * k + 2 * wOpt);
        state = in_opt && P.cls[b0 + i] == kState;      // (set in step 2, else stale)
      }
      int c = kOther;
      int64_t it_end = -1;
      bool grad = false, data = false, act = false;
      for (int k = 0; k < nit; ++k) {
        const int64_t* w = W + 12 * k;
        if (inside(a, w + 2 * wBw) && (f == -1 || f > w[2 * wBw + 1])) grad = true;
        if (inside(a, w + 2 * wData)) data = true;
        if (inside(a, w + 2 * wFw) || inside(a, w + 2 * wBw)) act = true;
        if (w[2 * wIt] <= a && a <= w[2 * wIt + 1] && it_end < 0) it_end = w[2 * wIt + 1];
      }
      if (param) c = kParam;
      else if (state) c = kState;
      else if (grad) c = kGrad;
      else if (data) c = kData;
      else if (act) c = kAct;
      P.cls[b0 + i] = uint8_t(c);
      atomicAdd(&s_ncls[c], 1u);
      if (a >= We) continue;
      if (c == kData && it_end >= 0 && (f == -1 || f > it_end)) f = it_end;
      int64_t a2, f2;
      bool has_free = true;
      if (a < Ws) {
        if (!(f == -1 || f > Ws)) continue;             // not alive in W
        a2 = Ws;
        if (c == kParam || c == kState) has_free = false, f2 = 0;
        else if (c == kGrad) f2 = zg_end >= 0 ? zg_end : We;
        else f2 = (f != -1 && f < We) ? f : We;
      } else {
        a2 = a;
        if (c == kParam || c == kState) {
          has_free = f != -1 && f < We;
          f2 = f;
        } else if (c == kGrad) {
          f2 = We;
        } else {
          f2 = (f != -1 && f < We) ? f : We;
        }
      }
      if (has_free && f2 < a2 + 1) f2 = a2 + 1;
      const uint32_t m = has_free ? 2u : 1u;
      const uint32_t p = atomicAdd(&s_nkeys, m);
      const unsigned long long ra = (unsigned long long)(a2 - Ws);
      if (ra > 0xFFFFFFFFull || (has_free && (unsigned long long)(f2 - Ws) > 0xFFFFFFFFull))
        atomicExch(&s_bad, 1u);
      keys[p] = (ra << 32) | (1ull << 31) | uint32_t(i);
      if (has_free) keys[p + 1] = ((unsigned long long)(f2 - Ws) << 32) | uint32_t(i);
    }
    __syncthreads();
    const uint32_t nk = s_nkeys;
    uint32_t npow = 1;
    while (npow < nk) npow <<= 1;
    for (uint32_t i = nk + tid; i < npow; i += kThreads) keys[i] = ~0ull;
    __syncthreads();
    // ---- 4. sort ----
    bitonic(keys, npow);
    // ---- 5. outputs: sequence, dense ids, staged wire events ----
    unsigned long long* seq = P.seq + 2 * b0;
    for (uint32_t i = tid; i < nk; i += kThreads) seq[i] = keys[i];
    __syncthreads();                                    // warp 0 rewrites keys[] below
    int64_t* ob = P.st_bytes + 2 * b0;
    uint32_t* ot = P.st_tag + 2 * b0;
    if (warp == 0) {
      const unsigned lt = (1u << lane) - 1u;
      uint32_t top = 0, fresh = 0;
      // the serial part only assigns the dense ids (kept in the high half of
      // each key); the block sizes and streams are gathered by the whole CTA
      // afterwards, off the serial chain
      for (uint32_t base = 0; base < nk; base += 32) {
        const uint32_t j = base + lane;
        const bool v = j < nk;
        const unsigned long long key = v ? keys[j] : 0ull;
        const bool al = v && ((key >> 31) & 1ull);
        const bool fr = v && !al;
        const uint32_t blk = uint32_t(key & 0x7FFFFFFFu);
        const unsigned am = __ballot_sync(kFull, al);
        const uint32_t na = __popc(am), ka = __popc(am & lt), take = min(na, top);
        uint32_t id = 0;
        if (al) {
          id = ka < take ? ids[top - 1 - ka] : fresh + (ka - take);
          id_of[blk] = id;
        }
        top -= take;
        fresh += na - take;
        __syncwarp();
        if (fr) id = id_of[blk];
        const unsigned fm = __ballot_sync(kFull, fr);
        if (fr) ids[top + __popc(fm & lt)] = id;
        top += __popc(fm);
        if (v) keys[j] = (static_cast<unsigned long long>(id) << 32) | (key & 0xFFFFFFFFull);
        __syncwarp();
      }
      if (lane == 0) {
        R.ws = Ws;
        R.we = We;
        R.n_events = nk;
        R.n_ids = fresh;
        R.status = s_bad ? XM_O_TS_RANGE : XM_O_OK;
        for (int c = 0; c < 6; ++c) R.n_class[c] = s_ncls[c];
        P.rec[t] = R;
      }
    }
    __syncthreads();
    // staged wire events: (size, dense id | stream << 28) of each sequence entry
    for (uint32_t j = tid; j < nk; j += kThreads) {
      const unsigned long long key = keys[j];
      const uint32_t blk = uint32_t(key & 0x7FFFFFFFu);
      const bool al = (key >> 31) & 1ull;
      const uint32_t st = P.stream ? P.stream[b0 + blk] : 0u;
      ob[j] = al ? S[blk] : -S[blk];
      ot[j] = uint32_t(key >> 32) | (st << 28);
    }
    __syncthreads();
  }
}

// exclusive scan of rec[order[k]].n_events over stored k -> woff (one CTA)
__global__ void __launch_bounds__(1024) k_owire_offsets(const xm_orchestrated* rec,
                                                        const uint32_t* order, int64_t T,
                                                        int64_t* woff) {
  __shared__ long long part[1024];
  const int tid = threadIdx.x;
  const int64_t per = (T + 1023) / 1024;
  const int64_t a = min(T, int64_t(tid) * per), z = min(T, a + per);
  long long s = 0;
  for (int64_t k = a; k < z; ++k) s += (long long)rec[order ? order[k] : k].n_events;
  part[tid] = s;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    const long long v = tid >= o ? part[tid - o] : 0;
    __syncthreads();
    part[tid] += v;
    __syncthreads();
  }
  long long run = part[tid] - s;
  for (int64_t k = a; k < z; ++k) {
    woff[k] = run;
    run += (long long)rec[order ? order[k] : k].n_events;
  }
  if (tid == 1023) woff[T] = part[1023];
}

__global__ void k_owire_compact(const int64_t* __restrict__ boff, const int64_t* __restrict__ woff,
                                const xm_orchestrated* __restrict__ rec, const uint32_t* order,
                                const int64_t* st_bytes, const uint32_t* st_tag, int64_t T,
                                int64_t* w_bytes, uint32_t* w_tag, uint32_t* w_nids) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t k = w0; k < T; k += nw) {
    const int64_t t = order ? order[k] : k;
    const int64_t src = 2 * boff[t], dst = woff[k], m = woff[k + 1] - dst;
    for (int64_t j = lane; j < m; j += 32) {
      w_bytes[dst + j] = st_bytes[src + j];
      w_tag[dst + j] = st_tag[src + j];
    }
    if (lane == 0) w_nids[k] = rec[t].n_ids;
  }
}

struct OLayout {
  uint32_t ctas, keys_cap;
  size_t cand, psize, id_of, idstack, gkeys, st_bytes, st_tag, total;
};

OLayout olayout(const xm_profiles* in) {
  OLayout L{};
  int dev = 0, sms = 148;
  if (xm_internal::cuda_usable() && cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaGetLastError();
  const int64_t max_ctas = int64_t(sms) * kCtasPerSm;
  L.ctas = uint32_t(in->n_traces < max_ctas ? (in->n_traces > 0 ? in->n_traces : 1) : max_ctas);
  const size_t mb = in->max_blocks ? in->max_blocks : 1;
  uint32_t cap = 1;
  while (cap < 2 * mb) cap <<= 1;
  L.keys_cap = 2 * mb > size_t(kSmemKeys) ? cap : 0;
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  size_t o = 256;
  L.cand = o; o += al(L.ctas * mb * 4);
  L.psize = o; o += al(L.ctas * mb * 8);
  L.id_of = o; o += al(L.ctas * mb * 4);
  L.idstack = o; o += al(L.ctas * mb * 4);
  L.gkeys = o; o += al(size_t(L.ctas) * L.keys_cap * 8);
  const size_t E2 = 2 * size_t(in->n_blocks > 0 ? in->n_blocks : 1);
  L.st_bytes = o; o += al(E2 * 8);
  L.st_tag = o; o += al(E2 * 4);
  L.total = o;
  return L;
}

}  // namespace

using namespace xm_internal;

extern "C" size_t xm_orchestrate_scratch_bytes(const xm_profiles* in) {
  if (!in || in->n_traces < 0 || in->n_blocks < 0) return 0;
  return olayout(in).total;
}

extern "C" int xm_orchestrate(const xm_profiles* in, uint32_t analysis_iter, void* d_scratch,
                              size_t scratch_bytes, uint8_t* d_class, uint64_t* d_seq,
                              xm_orchestrated* d_rec, void* stream) {
  launch_counter() = 0;
  if (!in || in->n_traces < 0 || in->n_blocks < 0)
    return set_error(XM_EINVAL, "xm_orchestrate: bad arguments");
  if (in->max_blocks > (1u << kBlockBits))
    return set_error(XM_ERANGE, "xm_orchestrate: more than 2^23 blocks in a trace");
  if (in->n_traces == 0) return XM_OK;
  if (!in->boff || !in->win || !in->woff || (in->n_blocks > 0 && (!in->alloc_ts || !in->free_ts ||
      !in->size)) || !d_class || !d_seq || !d_rec || !d_scratch)
    return set_error(XM_EINVAL, "xm_orchestrate: null pointer");
  const OLayout L = olayout(in);
  if (scratch_bytes < L.total) return set_error(XM_ENOMEM, "xm_orchestrate: scratch too small");
  if (!cuda_usable()) return set_error(XM_ECUDA, "no CUDA device");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char* base = static_cast<char*>(d_scratch);
  cudaError_t e = cudaMemsetAsync(base, 0, 256, st);
  if (e != cudaSuccess) return set_error(XM_ECUDA, cudaGetErrorString(e));
  OParams P{};
  P.alloc_ts = in->alloc_ts;
  P.free_ts = in->free_ts;
  P.size = in->size;
  P.stream = in->stream;
  P.boff = in->boff;
  P.win = in->win;
  P.woff = in->woff;
  P.n_traces = in->n_traces;
  P.analysis = analysis_iter;
  P.max_blocks = in->max_blocks ? in->max_blocks : 1;
  P.cand = reinterpret_cast<uint32_t*>(base + L.cand);
  P.psize = reinterpret_cast<int64_t*>(base + L.psize);
  P.id_of = reinterpret_cast<uint32_t*>(base + L.id_of);
  P.idstack = reinterpret_cast<uint32_t*>(base + L.idstack);
  P.gkeys = reinterpret_cast<unsigned long long*>(base + L.gkeys);
  P.keys_cap = L.keys_cap;
  P.cls = d_class;
  P.seq = reinterpret_cast<unsigned long long*>(d_seq);
  P.rec = d_rec;
  P.st_bytes = reinterpret_cast<int64_t*>(base + L.st_bytes);
  P.st_tag = reinterpret_cast<uint32_t*>(base + L.st_tag);
  P.work = reinterpret_cast<unsigned int*>(base);
  const int smem = kSmemKeys * 8;
  e = cudaFuncSetAttribute(k_orchestrate, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return set_error(XM_ECUDA, cudaGetErrorString(e));
  k_orchestrate<<<L.ctas, kThreads, smem, st>>>(P);
  launch_counter() = 1;
  e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(XM_ECUDA, std::string("xm_orchestrate: ") + cudaGetErrorString(e));
  return XM_OK;
}

extern "C" int xm_orchestrate_wire(const xm_profiles* in, const void* d_scratch,
                                   size_t scratch_bytes, const xm_orchestrated* d_rec,
                                   const uint32_t* d_order, int64_t* d_wire_bytes,
                                   uint32_t* d_wire_tag, int64_t* d_wire_off,
                                   uint32_t* d_wire_nids, void* stream) {
  launch_counter() = 0;
  if (!in || in->n_traces < 0) return set_error(XM_EINVAL, "xm_orchestrate_wire: bad arguments");
  if (in->n_traces == 0) return XM_OK;
  if (!in->boff || !d_rec || !d_scratch || !d_wire_bytes || !d_wire_tag || !d_wire_off || !d_wire_nids)
    return set_error(XM_EINVAL, "xm_orchestrate_wire: null pointer");
  const OLayout L = olayout(in);
  if (scratch_bytes < L.total) return set_error(XM_ENOMEM, "xm_orchestrate_wire: scratch too small");
  if (!cuda_usable()) return set_error(XM_ECUDA, "no CUDA device");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const char* base = static_cast<const char*>(d_scratch);
  k_owire_offsets<<<1, 1024, 0, st>>>(d_rec, d_order, in->n_traces, d_wire_off);
  const int64_t want = (in->n_traces + 7) / 8;
  const int g = int(want < int64_t(L.ctas) * 8 ? want : int64_t(L.ctas) * 8);
  k_owire_compact<<<g > 0 ? g : 1, 256, 0, st>>>(
      in->boff, d_wire_off, d_rec, d_order, reinterpret_cast<const int64_t*>(base + L.st_bytes),
      reinterpret_cast<const uint32_t*>(base + L.st_tag), in->n_traces, d_wire_bytes, d_wire_tag,
      d_wire_nids);
  launch_counter() = 2;
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(XM_ECUDA, std::string("xm_orchestrate_wire: ") + cudaGetErrorString(e));
  return XM_OK;
}
