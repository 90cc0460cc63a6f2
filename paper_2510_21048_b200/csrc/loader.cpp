// loader.cpp -- host side of the boundary: validate, renumber and pack traces.
//
// xm_load_traces (include/xmem.h) checks the contract violations SPEC.md lists
// for the simulator's input (zero request S:231, duplicate live id S:249, free
// of a non-live id or of the wrong size S:258), renumbers block ids densely so a
// trace's id space equals its maximum number of live blocks (the device keeps
// one state record per id), and computes the longest-first processing order
// the persistent replay kernel pulls work from, storing the traces in that
// order. Traces are processed in parallel on host threads. None of the allocator arithmetic lives here.
#include <algorithm>
#include <cmath>
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#include "xmem.h"
#include "xm_internal.h"

struct xm_traces {
  int64_t n_traces = 0, n_events = 0;
  int64_t* bytes = nullptr;
  uint32_t* tag = nullptr;
  int64_t* off = nullptr;
  uint32_t* n_ids = nullptr;
  uint32_t* order = nullptr;
  uint32_t max_ids = 0, max_events = 0;
  uint32_t* chunk_end = nullptr;   // [kUploadChunks] pinned, see xm_simulate_host
  int n_chunks = 0;
  uint64_t* packed = nullptr;      // compact events (xm_batch.packed), or null
  std::vector<void*> blocks;
  std::vector<bool> pinned;
};

namespace {

void* host_alloc(xm_traces* tr, size_t n) {
  if (n == 0) n = 8;
  void* p = nullptr;
  if (xm_internal::cuda_usable() && cudaHostAlloc(&p, n, cudaHostAllocMapped) == cudaSuccess) {
    tr->blocks.push_back(p);
    tr->pinned.push_back(true);
    return p;
  }
  cudaGetLastError();  // clear a sticky "no device" error
  p = std::malloc(n);
  if (p) {
    tr->blocks.push_back(p);
    tr->pinned.push_back(false);
  }
  return p;
}

struct Slot {
  uint32_t key;
  uint32_t dense;  // kNone when not live
  int64_t req;
  uint32_t used;
  uint32_t stream;  // of the live block's alloc
};
constexpr uint32_t kNone = 0xFFFFFFFFu;

struct Renumberer {
  std::vector<Slot> table;
  std::vector<uint32_t> free_ids;
  uint64_t mask = 0;

  Slot* find(uint32_t key) {
    uint64_t h = (uint64_t(key) * 0x9E3779B97F4A7C15ull) >> 20 & mask;
    for (;;) {
      Slot& s = table[h];
      if (!s.used || s.key == key) return &s;
      h = (h + 1) & mask;
    }
  }

  // returns 0 or an error code with *msg set; writes renumbered tags and n_ids
  int run(const int64_t* bytes, const uint32_t* tag, int64_t n, uint32_t* out_tag,
          uint32_t* n_ids, const char** msg) {
    int64_t nalloc = 0;
    for (int64_t i = 0; i < n; ++i) nalloc += bytes[i] > 0;
    uint64_t cap = 16;
    while (cap < uint64_t(2 * nalloc + 2)) cap <<= 1;
    table.assign(cap, Slot{0, kNone, 0, 0, 0});
    mask = cap - 1;
    free_ids.clear();
    uint32_t next = 0;
    for (int64_t i = 0; i < n; ++i) {
      int64_t b = bytes[i];
      uint32_t raw = tag[i] & ((1u << XM_ID_BITS) - 1);
      const uint32_t stream = tag[i] >> XM_STREAM_SHIFT;
      if (b == 0) { *msg = "zero-byte event (SPEC.md:231)"; return XM_EINVAL; }
      uint64_t mag = b > 0 ? uint64_t(b) : uint64_t(-(b + 1)) + 1;
      if (mag >= XM_MAX_REQUEST) { *msg = "request >= 2^40 bytes"; return XM_ERANGE; }
      Slot* s = find(raw);
      if (b > 0) {
        if (s->used && s->dense != kNone) { *msg = "alloc of a live id (SPEC.md:249)"; return XM_EINVAL; }
        uint32_t d;
        if (!free_ids.empty()) { d = free_ids.back(); free_ids.pop_back(); }
        else {
          d = next++;
          if (next > (1u << 27)) { *msg = "more than 2^27 live blocks"; return XM_ERANGE; }
        }
        s->used = 1; s->key = raw; s->dense = d; s->req = b; s->stream = stream;
        out_tag[i] = d | (stream << XM_STREAM_SHIFT);
      } else {
        if (!s->used || s->dense == kNone) { *msg = "free of a non-live id (SPEC.md:258)"; return XM_EINVAL; }
        if (s->req != -b) { *msg = "free size differs from the alloc's request (SPEC.md:258)"; return XM_EINVAL; }
        // a block returns to its own pool (PAPER.md:259 (iv)): the free carries
        // the stream of the block's alloc, whatever stream the trace records
        out_tag[i] = s->dense | (s->stream << XM_STREAM_SHIFT);
        free_ids.push_back(s->dense);
        s->dense = kNone;
      }
    }
    *n_ids = next;
    return XM_OK;
  }
};

}  // namespace

extern "C" int xm_load_traces(const int64_t* bytes, const uint32_t* tag, const int64_t* off,
                              int64_t n_traces, xm_traces** out, int64_t* bad_trace) {
  using xm_internal::set_error;
  if (bad_trace) *bad_trace = -1;
  if (!out || n_traces < 0 || !off || (n_traces > 0 && (!bytes || !tag)))
    return set_error(XM_EINVAL, "xm_load_traces: null argument or negative n_traces");
  *out = nullptr;
  if (off[0] != 0) return set_error(XM_EINVAL, "xm_load_traces: off[0] != 0");
  for (int64_t t = 0; t < n_traces; ++t) {
    if (off[t + 1] < off[t]) {
      if (bad_trace) *bad_trace = t;
      return set_error(XM_EINVAL, "xm_load_traces: offsets not monotone");
    }
    if (off[t + 1] - off[t] >= int64_t(0xFFFFFFFFu)) {
      if (bad_trace) *bad_trace = t;
      return set_error(XM_ERANGE, "xm_load_traces: trace longer than 2^32-2 events");
    }
  }
  const int64_t E = off[n_traces];
  xm_traces* tr = new (std::nothrow) xm_traces();
  if (!tr) return set_error(XM_ENOMEM, "xm_load_traces: out of host memory");
  tr->n_traces = n_traces;
  tr->n_events = E;
  tr->bytes = (int64_t*)host_alloc(tr, sizeof(int64_t) * E);
  tr->tag = (uint32_t*)host_alloc(tr, sizeof(uint32_t) * E);
  tr->off = (int64_t*)host_alloc(tr, sizeof(int64_t) * (n_traces + 1));
  tr->n_ids = (uint32_t*)host_alloc(tr, sizeof(uint32_t) * n_traces);
  tr->order = (uint32_t*)host_alloc(tr, sizeof(uint32_t) * n_traces);
  tr->chunk_end = (uint32_t*)host_alloc(tr, sizeof(uint32_t) * xm_internal::kUploadChunks);
  if (!tr->bytes || !tr->tag || !tr->off || !tr->n_ids || !tr->order || !tr->chunk_end) {
    xm_free_traces(tr);
    return set_error(XM_ENOMEM, "xm_load_traces: out of host memory");
  }
  // storage order = processing order: longest first (LPT), stable (ties keep
  // caller order). order[i] = caller index of stored trace i; off is the
  // storage prefix sum. Storing the longest traces first lets the host entry
  // point stream the batch to the device in chunks the kernel starts on as
  // they land (xm_simulate_host).
  for (int64_t i = 0; i < n_traces; ++i) tr->order[i] = uint32_t(i);
  std::stable_sort(tr->order, tr->order + n_traces, [&](uint32_t a, uint32_t b) {
    return off[a + 1] - off[a] > off[b + 1] - off[b];
  });
  tr->off[0] = 0;
  for (int64_t i = 0; i < n_traces; ++i) {
    const uint32_t t = tr->order[i];
    tr->off[i + 1] = tr->off[i] + (off[t + 1] - off[t]);
  }
  const int64_t* soff = tr->off;

  // parallel over stored traces: contiguous ranges of roughly equal event counts
  unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  int nth = int(std::min<int64_t>(hw, std::max<int64_t>(1, E / 65536)));
  nth = std::max(1, std::min<int>(nth, int(std::max<int64_t>(1, n_traces))));
  // first_bad = the smallest CALLER index of an invalid trace
  std::atomic<int64_t> first_bad{INT64_MAX};
  std::vector<int> codes(nth, XM_OK);
  std::vector<const char*> msgs(nth, nullptr);
  std::vector<int64_t> bads(nth, INT64_MAX);
  std::vector<int64_t> bounds(nth + 1);
  bounds[0] = 0;
  for (int k = 1; k < nth; ++k)
    bounds[k] = std::max(bounds[k - 1], int64_t(std::lower_bound(soff, soff + n_traces, E * k / nth) - soff));
  bounds[nth] = n_traces;
  auto work2 = [&](int k) {
    Renumberer R;
    for (int64_t i = bounds[k]; i < bounds[k + 1]; ++i) {
      const int64_t t = tr->order[i];
      if (t >= first_bad.load(std::memory_order_relaxed)) continue;
      const int64_t a = off[t], n = off[t + 1] - a, d = soff[i];
      std::memcpy(tr->bytes + d, bytes + a, sizeof(int64_t) * n);
      const char* m = nullptr;
      int rc = R.run(bytes + a, tag + a, n, tr->tag + d, tr->n_ids + i, &m);
      if (rc) {
        if (t < bads[k]) { codes[k] = rc; msgs[k] = m; bads[k] = t; }
        int64_t cur = first_bad.load();
        while (t < cur && !first_bad.compare_exchange_weak(cur, t)) {}
      }
    }
  };
  if (nth == 1) {
    work2(0);
  } else {
    std::vector<std::thread> th;
    for (int k = 0; k < nth; ++k) th.emplace_back(work2, k);
    for (auto& x : th) x.join();
  }
  int64_t fb = first_bad.load();
  if (fb != INT64_MAX) {
    int rc = XM_EINVAL;
    const char* m = "invalid trace";
    for (int k = 0; k < nth; ++k)
      if (bads[k] == fb) { rc = codes[k]; m = msgs[k]; }
    if (bad_trace) *bad_trace = fb;
    xm_free_traces(tr);
    return set_error(rc, std::string("xm_load_traces: trace ") + std::to_string(fb) + ": " + m);
  }
  uint32_t mi = 0;
  for (int64_t i = 0; i < n_traces; ++i) mi = std::max(mi, tr->n_ids[i]);
  tr->max_ids = mi;
  // compact 8-byte events for the host entry point's upload (2/3 of the bytes)
  if (mi <= (1u << XM_PACKED_ID_BITS) && E > 0) {
    tr->packed = (uint64_t*)host_alloc(tr, sizeof(uint64_t) * E);
    if (tr->packed) {
      auto pack = [&](int k) {
        for (int64_t e = soff[bounds[k]]; e < soff[bounds[k + 1]]; ++e) {
          const int64_t b = tr->bytes[e];
          const uint32_t g = tr->tag[e];
          tr->packed[e] = uint64_t(b > 0 ? b : -b) | (uint64_t(b > 0) << 41) |
                          (uint64_t(g >> XM_STREAM_SHIFT) << 42) |
                          (uint64_t(g & ((1u << XM_STREAM_SHIFT) - 1u)) << 46);
        }
      };
      if (nth == 1) {
        pack(0);
      } else {
        std::vector<std::thread> th;
        for (int k = 0; k < nth; ++k) th.emplace_back(pack, k);
        for (auto& x : th) x.join();
      }
    }
  }
  tr->max_events = n_traces ? uint32_t(soff[1] - soff[0]) : 0u;
  // upload chunks for the streamed host entry point: chunk c = stored traces
  // [chunk_end[c-1], chunk_end[c]), cut at trace boundaries; chunk sizes grow
  // geometrically (x1.15) so that the first, longest traces land -- and start
  // -- early while later chunks stay few
  tr->n_chunks = 0;
  if (tr->chunk_end) {
    int64_t prev = 0;
    const double r = 1.15, rn = std::pow(r, double(xm_internal::kUploadChunks));
    for (int c = 1; c <= xm_internal::kUploadChunks && prev < n_traces; ++c) {
      const double frac = (std::pow(r, double(c)) - 1.0) / (rn - 1.0);
      const int64_t target = int64_t(double(E) * frac);
      int64_t e = int64_t(std::lower_bound(soff, soff + n_traces + 1, target) - soff);
      if (c == xm_internal::kUploadChunks) e = n_traces;
      if (e <= prev) continue;
      tr->chunk_end[tr->n_chunks++] = uint32_t(e);
      prev = e;
    }
  }
  *out = tr;
  xm_internal::clear_error();
  return XM_OK;
}

extern "C" int xm_traces_views(const xm_traces* tr, const int64_t** bytes, const uint32_t** tag,
                               const int64_t** off, const uint32_t** n_ids, const uint32_t** order,
                               int64_t* n_traces, int64_t* n_events, uint32_t* max_ids,
                               uint32_t* max_events) {
  if (!tr) return xm_internal::set_error(XM_EINVAL, "xm_traces_views: null traces");
  if (bytes) *bytes = tr->bytes;
  if (tag) *tag = tr->tag;
  if (off) *off = tr->off;
  if (n_ids) *n_ids = tr->n_ids;
  if (order) *order = tr->order;
  if (n_traces) *n_traces = tr->n_traces;
  if (n_events) *n_events = tr->n_events;
  if (max_ids) *max_ids = tr->max_ids;
  if (max_events) *max_events = tr->max_events;
  return XM_OK;
}

extern "C" int xm_traces_packed(const xm_traces* tr, const uint64_t** packed) {
  if (!tr || !packed) return xm_internal::set_error(XM_EINVAL, "xm_traces_packed: null argument");
  *packed = tr->packed;
  return XM_OK;
}

extern "C" void xm_free_traces(xm_traces* tr) {
  if (!tr) return;
  for (size_t i = 0; i < tr->blocks.size(); ++i) {
    if (tr->pinned[i]) cudaFreeHost(tr->blocks[i]);
    else std::free(tr->blocks[i]);
  }
  delete tr;
}

// ---- helpers for the host entry point (capi.cu) ----
namespace xm_internal {
const xm_traces_info traces_info(const xm_traces* tr) {
  return xm_traces_info{tr->bytes,   tr->tag,      tr->off,      tr->n_ids,    tr->order,
                        tr->n_traces, tr->n_events, tr->max_ids, tr->max_events,
                        tr->chunk_end, tr->n_chunks, tr->packed};
}
}  // namespace xm_internal
