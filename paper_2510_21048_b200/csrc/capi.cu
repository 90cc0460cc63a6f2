// capi.cu -- the extern "C" entry points of libxmem.so (include/xmem.h) that
// are not the loader: configuration, scratch sizing, the device and host
// simulate calls, result download and error reporting.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "xm_internal.h"

namespace xm_internal {

namespace {
thread_local std::string g_err;
thread_local int g_launches = 0;
}  // namespace

int set_error(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

void clear_error() { g_err.clear(); }

bool cuda_usable() {
  static int state = -1;  // -1 unknown, 0 no, 1 yes
  if (state < 0) {
    int n = 0;
    state = (cudaGetDeviceCount(&n) == cudaSuccess && n > 0) ? 1 : 0;
    cudaGetLastError();
  }
  return state == 1;
}

static bool is_pow2(uint64_t x) { return x && !(x & (x - 1)); }

int make_unit_config(const xm_config* c, UnitConfig* u) {
  if (!is_pow2(c->min_block) || c->min_block > (1u << 20))
    return set_error(XM_EINVAL, "xm_config: min_block must be a power of two <= 1 MiB");
  const uint64_t m = c->min_block;
  const uint64_t v[5] = {c->small_size, c->small_buffer, c->large_buffer, c->min_large_alloc,
                         c->round_large};
  for (uint64_t x : v)
    if (x == 0 || x % m || x / m > 0x7FFFFFFFull)
      return set_error(XM_EINVAL, "xm_config: sizes must be non-zero multiples of min_block");
  if (c->small_buffer < c->small_size || c->large_buffer <= c->small_size)
    return set_error(XM_EINVAL, "xm_config: segment sizes must cover the small threshold");
  // SPEC.md:211-213 / torch's constants: small_size < min_large_alloc <=
  // large_buffer, so a request between them fits its large_buffer segment
  // (otherwise the remainder bsize - s underflows) and narrow keys never saturate
  if (c->min_large_alloc <= c->small_size || c->min_large_alloc > c->large_buffer)
    return set_error(XM_EINVAL, "xm_config: need small_size < min_large_alloc <= large_buffer");
  if (c->mode != XM_FULL && c->mode != XM_ALLOCATED_ONLY)
    return set_error(XM_EINVAL, "xm_config: unknown mode");
  const uint32_t dv = c->roundup_power2_divisions;
  if (dv > 1 && (dv & (dv - 1) || dv > 64))
    return set_error(XM_EINVAL, "xm_config: roundup_power2_divisions must be a power of two <= 64");
  if (c->reclaim_policy != XM_RECLAIM_ALL && c->reclaim_policy != XM_RECLAIM_LARGEST_FIRST)
    return set_error(XM_EINVAL, "xm_config: unknown reclaim_policy");
  if (c->host_input > XM_HOST_INPUT_COPY) return set_error(XM_EINVAL, "xm_config: unknown host_input");
  if (c->max_split_size != XM_UNLIMITED &&
      (c->max_split_size == 0 || c->max_split_size % m || c->max_split_size / m > 0x7FFFFFFFull))
    return set_error(XM_EINVAL, "xm_config: max_split_size must be a non-zero multiple of min_block");
  if (c->max_non_split_rounding % m || c->max_non_split_rounding / m > 0x7FFFFFFFull)
    return set_error(XM_EINVAL, "xm_config: max_non_split_rounding must be a multiple of min_block");
  if (!(c->garbage_collection_threshold >= 0.0 && c->garbage_collection_threshold < 1.0))
    return set_error(XM_EINVAL, "xm_config: garbage_collection_threshold must be in [0, 1)");
  int sh = 0;
  while ((1ull << sh) < m) ++sh;
  u->unit_shift = uint32_t(sh);
  u->small_u = uint32_t(c->small_size / m);
  u->sbuf_u = uint32_t(c->small_buffer / m);
  u->lbuf_u = uint32_t(c->large_buffer / m);
  u->minlarge_u = uint32_t(c->min_large_alloc / m);
  u->rlarge_u = uint32_t(c->round_large / m);
  u->strict = c->large_split_strict ? 1u : 0u;
  u->div_shift = 0;
  while (dv > 1 && (1u << u->div_shift) < dv) ++u->div_shift;
  u->reclaim_d3 = c->reclaim_policy == XM_RECLAIM_LARGEST_FIRST ? 1u : 0u;
  u->msplit_u = c->max_split_size == XM_UNLIMITED ? 0xFFFFFFFFu : uint32_t(c->max_split_size / m);
  u->nsr_u = uint32_t(c->max_non_split_rounding / m);
  u->gc_threshold = c->garbage_collection_threshold;
  return XM_OK;
}

int& launch_counter() { return g_launches; }

}  // namespace xm_internal

using namespace xm_internal;

extern "C" void xm_config_default(xm_config* c) {
  if (!c) return;
  std::memset(c, 0, sizeof(*c));
  c->min_block = 512;
  c->small_size = 1ull << 20;
  c->small_buffer = 2ull << 20;
  c->large_buffer = 20ull << 20;
  c->min_large_alloc = 10ull << 20;
  c->round_large = 2ull << 20;
  c->capacity = XM_UNLIMITED;
  c->large_split_strict = 1;
  c->mode = XM_FULL;
  c->max_split_size = XM_UNLIMITED;
  c->max_non_split_rounding = 20ull << 20;
  c->garbage_collection_threshold = 0.0;
}

extern "C" const char* xm_last_error(void) { return g_err.c_str(); }

extern "C" int xm_last_launch_count(void) { return launch_counter(); }

static int check_batch(const xm_batch* b) {
  if (!b) return set_error(XM_EINVAL, "null batch");
  if (b->n_traces < 0 || b->n_events < 0) return set_error(XM_EINVAL, "negative sizes");
  if (b->n_traces > 0x7FFFFFFFll) return set_error(XM_ERANGE, "more than 2^31-1 traces");
  if (b->n_traces > 0 && (!b->off || !b->n_ids || !b->order))
    return set_error(XM_EINVAL, "null device array in batch");
  if (b->n_events > 0 && !b->packed && (!b->bytes || !b->tag))
    return set_error(XM_EINVAL, "null event arrays");
  return XM_OK;
}

extern "C" size_t xm_scratch_bytes(const xm_batch* b, const xm_config* cfg) {
  if (!b || !cfg) return 0;
  if (cfg->mode == XM_ALLOCATED_ONLY) return scan_scratch_bytes(b);
  return plan_replay(b, cfg).scratch_bytes;
}

// ready: streamed-input counter (xm_simulate_host) or null
static int simulate(const xm_batch* b, const xm_config* cfg, void* d_scratch, size_t scratch_bytes,
                    xm_result* d_out, void* stream, const uint32_t* ready) {
  launch_counter() = 0;
  if (!cfg) return set_error(XM_EINVAL, "null config");
  UnitConfig u;
  int rc = make_unit_config(cfg, &u);
  if (rc) return rc;
  if ((rc = check_batch(b))) return rc;
  if (b->n_traces == 0) return XM_OK;
  if (!d_out || !d_scratch) return set_error(XM_EINVAL, "null output or scratch");
  if (!cuda_usable()) return set_error(XM_ECUDA, "no CUDA device");
  int e;
  if (cfg->mode == XM_ALLOCATED_ONLY) {
    if (cfg->capacity != XM_UNLIMITED || b->capacity)
      return set_error(XM_EINVAL, "XM_ALLOCATED_ONLY requires unlimited capacity");
    if (b->curve) return set_error(XM_EINVAL, "the memory curve needs XM_FULL");
    if (ready) return set_error(XM_EINVAL, "streamed input needs XM_FULL");
    if (scratch_bytes < scan_scratch_bytes(b)) return set_error(XM_ENOMEM, "scratch too small");
    e = launch_scan(b, u, d_scratch, scratch_bytes, d_out, stream, &launch_counter());
  } else {
    ReplayPlan plan = plan_replay(b, cfg);
    if (scratch_bytes < plan.scratch_bytes)
      return set_error(XM_ENOMEM, "scratch smaller than xm_scratch_bytes()");
    e = launch_replay(b, cfg, u, plan, d_scratch, d_out, stream, &launch_counter(), ready);
  }
  if (e != 0)
    return set_error(XM_ECUDA, std::string("launch failed: ") + cudaGetErrorString(cudaError_t(e)));
  clear_error();
  return XM_OK;
}

extern "C" int xm_simulate_batch(const xm_batch* b, const xm_config* cfg, void* d_scratch,
                                 size_t scratch_bytes, xm_result* d_out, void* stream) {
  return simulate(b, cfg, d_scratch, scratch_bytes, d_out, stream, nullptr);
}

extern "C" int xm_peaks(const xm_result* d_res, int64_t n, xm_result* h_out, xm_summary* h_sum,
                        uint64_t capacity_for_eq1, void* stream) {
  if (n < 0 || (n > 0 && !d_res)) return set_error(XM_EINVAL, "xm_peaks: bad arguments");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  xm_result* h = h_out;
  xm_result* tmp = nullptr;
  if (!h && h_sum && n > 0) {
    tmp = static_cast<xm_result*>(std::malloc(sizeof(xm_result) * size_t(n)));
    if (!tmp) return set_error(XM_ENOMEM, "xm_peaks: host allocation failed");
    h = tmp;
  }
  if (h && n > 0) {
    cudaError_t e = cudaMemcpyAsync(h, d_res, sizeof(xm_result) * size_t(n), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
      std::free(tmp);
      return set_error(XM_ECUDA, std::string("xm_peaks: ") + cudaGetErrorString(e));
    }
  }
  if (h_sum) {
    std::memset(h_sum, 0, sizeof(*h_sum));
    h_sum->n_traces = uint64_t(n);
    for (int64_t i = 0; i < n; ++i) {
      const xm_result& r = h[i];
      h_sum->events_done += r.events_done;
      h_sum->n_oom += r.status == XM_T_OOM;
      h_sum->n_overflow += r.status == XM_T_OVERFLOW;
      h_sum->max_peak_reserved = std::max(h_sum->max_peak_reserved, r.peak_reserved);
      h_sum->max_peak_allocated = std::max(h_sum->max_peak_allocated, r.peak_allocated);
      h_sum->sum_peak_reserved += r.peak_reserved;
      // Eq. 1: OOM_hat = [M_peak > M_max], strict
      h_sum->n_predicted_oom += (r.status == XM_T_OOM) || (r.peak_reserved > capacity_for_eq1);
    }
  }
  std::free(tmp);
  clear_error();
  return XM_OK;
}

namespace {
struct HostLayout {
  size_t bytes, tag, packed, off, n_ids, order, cap, out, ready, scratch, total;
};
size_t al(size_t x) { return (x + 255) & ~size_t(255); }

HostLayout host_layout(const xm_traces_info& I, const xm_config* cfg, bool with_cap) {
  HostLayout L{};
  size_t p = 0;
  // events: the packed 8-byte form when the loader built it, else bytes + tag
  if (I.packed) {
    L.packed = p; p += al(sizeof(uint64_t) * I.n_events);
  } else {
    L.bytes = p; p += al(sizeof(int64_t) * I.n_events);
    L.tag = p; p += al(sizeof(uint32_t) * I.n_events);
  }
  L.off = p; p += al(sizeof(int64_t) * (I.n_traces + 1));
  L.n_ids = p; p += al(sizeof(uint32_t) * I.n_traces);
  L.order = p; p += al(sizeof(uint32_t) * I.n_traces);
  L.cap = p; p += with_cap ? al(sizeof(uint64_t) * I.n_traces) : 0;
  L.out = p; p += al(sizeof(xm_result) * I.n_traces);
  L.ready = p; p += 256;
  L.scratch = p;
  xm_batch b{};
  b.n_traces = I.n_traces;
  b.n_events = I.n_events;
  b.max_ids = I.max_ids;
  b.max_events = I.max_events;
  p += al(xm_scratch_bytes(&b, cfg));
  L.total = p;
  return L;
}

// Per-thread copy stream + events of the streamed host entry point (created
// on first use per device and kept for the thread's lifetime).
struct Pipe {
  int dev = -1;
  cudaStream_t cs = nullptr;        // copies
  cudaStream_t cs2 = nullptr;       // xm_simulate_raw's second copy stream (chunks alternate)
  cudaStream_t ls = nullptr;        // xm_simulate_raw's loader (overlapped with the replay)
  cudaEvent_t start = nullptr, copied = nullptr, meta = nullptr, ldone = nullptr, copied2 = nullptr;
};
thread_local Pipe g_pipe;

cudaError_t get_pipe(Pipe** out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  Pipe& p = g_pipe;
  if (p.dev != dev) {
    Pipe q;
    q.dev = dev;
    if ((e = cudaStreamCreateWithFlags(&q.cs, cudaStreamNonBlocking)) != cudaSuccess) return e;
    if ((e = cudaEventCreateWithFlags(&q.start, cudaEventDisableTiming)) != cudaSuccess) return e;
    if ((e = cudaEventCreateWithFlags(&q.copied, cudaEventDisableTiming)) != cudaSuccess) return e;
    if ((e = cudaStreamCreateWithFlags(&q.ls, cudaStreamNonBlocking)) != cudaSuccess) return e;
    if ((e = cudaEventCreateWithFlags(&q.meta, cudaEventDisableTiming)) != cudaSuccess) return e;
    if ((e = cudaEventCreateWithFlags(&q.ldone, cudaEventDisableTiming)) != cudaSuccess) return e;
    if ((e = cudaStreamCreateWithFlags(&q.cs2, cudaStreamNonBlocking)) != cudaSuccess) return e;
    if ((e = cudaEventCreateWithFlags(&q.copied2, cudaEventDisableTiming)) != cudaSuccess) return e;
    p = q;   // a previous device's objects are leaked, not destroyed under another context
  }
  *out = &p;
  return cudaSuccess;
}

// cuStreamWriteValue32 (driver API, a stream-ordered 4-byte write with
// memory-barrier semantics: the writes of earlier copies in the stream are
// visible before it), resolved at run time so that libxmem needs no -lcuda.
typedef int (*WriteValue32Fn)(cudaStream_t, unsigned long long, unsigned int, unsigned int);
WriteValue32Fn write_value32() {
  static WriteValue32Fn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    cudaGetLastError();
    return reinterpret_cast<WriteValue32Fn>(f);
  }();
  return fn;
}
}  // namespace

extern "C" size_t xm_host_ws_bytes(const xm_traces* tr, const xm_config* cfg) {
  if (!tr || !cfg) return 0;
  return host_layout(traces_info(tr), cfg, true).total;
}

// Streamed end-to-end replay. The packed batch is stored longest-first
// (xm_load_traces), so the upload is cut into chunks of whole traces in that
// order: the metadata goes first on `stream`, the event chunks follow on a
// second (copy) stream, each chunk followed by a stream-ordered write of the
// number of stored traces now resident, and the replay kernel, launched on
// `stream` without waiting for the copies, starts each trace as soon as its
// chunk has landed (wait_ready in replay.cu). The H2D transfer thereby
// overlaps the replay instead of preceding it. XM_ALLOCATED_ONLY (K1 reads the
// batch as one flat array) copies everything first.
extern "C" int xm_simulate_host(const xm_traces* tr, const uint64_t* capacity,
                                const xm_config* cfg, void* d_ws, size_t ws_bytes,
                                xm_result* h_out, void* stream) {
  if (!tr || !cfg || !d_ws || !h_out) return set_error(XM_EINVAL, "xm_simulate_host: null argument");
  const xm_traces_info I = traces_info(tr);
  const HostLayout L = host_layout(I, cfg, true);
  if (ws_bytes < L.total) return set_error(XM_ENOMEM, "xm_simulate_host: workspace too small");
  if (!cuda_usable()) return set_error(XM_ECUDA, "no CUDA device");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char* w = static_cast<char*>(d_ws);
  cudaError_t e = cudaSuccess;
  auto cp = [&](size_t o, const void* src, size_t n, cudaStream_t s) {
    if (e == cudaSuccess && n) e = cudaMemcpyAsync(w + o, src, n, cudaMemcpyHostToDevice, s);
  };
  // event input (include/xmem.h): DIRECT (the default when the packed host
  // array is device-mapped) = the replaying warps load the events in place
  // from host memory over PCIe, nothing staged in HBM; STREAM = chunked copies
  // on a copy stream overlapping the replay; COPY = everything copied first.
  // cfg->host_input chooses; env XM_HOST_INPUT=direct|stream|copy overrides,
  // XM_NO_STREAM=1 = copy.
  uint32_t hin = cfg->host_input;
  if (const char* v = std::getenv("XM_HOST_INPUT")) {
    if (!std::strcmp(v, "direct")) hin = XM_HOST_INPUT_DIRECT;
    else if (!std::strcmp(v, "stream")) hin = XM_HOST_INPUT_STREAM;
    else if (!std::strcmp(v, "copy")) hin = XM_HOST_INPUT_COPY;
  }
  if (std::getenv("XM_NO_STREAM")) hin = XM_HOST_INPUT_COPY;
  if (hin > XM_HOST_INPUT_COPY) return set_error(XM_EINVAL, "xm_config: unknown host_input");
  const bool want_copy = hin == XM_HOST_INPUT_COPY;
  const uint64_t* h_direct = nullptr;        // device-usable pointer of I.packed
  if (cfg->mode == XM_FULL && I.packed && I.n_events > 0 &&
      (hin == XM_HOST_INPUT_AUTO || hin == XM_HOST_INPUT_DIRECT)) {
    void* dp = nullptr;
    if (cudaHostGetDevicePointer(&dp, const_cast<uint64_t*>(I.packed), 0) == cudaSuccess)
      h_direct = static_cast<const uint64_t*>(dp);
    else
      cudaGetLastError();        // not page-locked (loaded without CUDA): stream instead
  }
  const bool streamed = !h_direct && cfg->mode == XM_FULL && I.n_chunks > 0 && !want_copy;
  cp(L.off, I.off, sizeof(int64_t) * (I.n_traces + 1), st);
  cp(L.n_ids, I.n_ids, sizeof(uint32_t) * I.n_traces, st);
  cp(L.order, I.order, sizeof(uint32_t) * I.n_traces, st);
  if (capacity) cp(L.cap, capacity, sizeof(uint64_t) * I.n_traces, st);
  uint32_t* ready = reinterpret_cast<uint32_t*>(w + L.ready);
  if (h_direct) {
    // DIRECT: nothing staged (h2d traffic = the events, read by the kernel)
  } else if (!streamed) {
    if (I.packed) {
      cp(L.packed, I.packed, sizeof(uint64_t) * I.n_events, st);
    } else {
      cp(L.bytes, I.bytes, sizeof(int64_t) * I.n_events, st);
      cp(L.tag, I.tag, sizeof(uint32_t) * I.n_events, st);
    }
  } else {
    Pipe* pp = nullptr;
    if (e == cudaSuccess) e = cudaMemsetAsync(ready, 0, sizeof(uint32_t), st);
    if (e == cudaSuccess) e = get_pipe(&pp);
    // the copy stream starts after everything already queued on `stream`
    // (earlier users of this workspace, the counter reset)
    if (e == cudaSuccess) e = cudaEventRecord(pp->start, st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(pp->cs, pp->start, 0);
    const WriteValue32Fn wv = write_value32();
    int64_t ev0 = 0;
    for (int c = 0; c < I.n_chunks && e == cudaSuccess; ++c) {
      // chunk ends are rounded up to 32 events (>= 128 B of each array) so no
      // cache sector holds events of two chunks
      int64_t ev1 = I.off[I.chunk_end[c]];
      if (c + 1 < I.n_chunks) ev1 = std::min<int64_t>(I.n_events, (ev1 + 31) & ~int64_t(31));
      else ev1 = I.n_events;
      if (ev1 > ev0) {
        if (I.packed) {
          cp(L.packed + sizeof(uint64_t) * ev0, I.packed + ev0, sizeof(uint64_t) * (ev1 - ev0), pp->cs);
        } else {
          cp(L.bytes + sizeof(int64_t) * ev0, I.bytes + ev0, sizeof(int64_t) * (ev1 - ev0), pp->cs);
          cp(L.tag + sizeof(uint32_t) * ev0, I.tag + ev0, sizeof(uint32_t) * (ev1 - ev0), pp->cs);
        }
        ev0 = ev1;
      }
      if (e != cudaSuccess) break;
      if (wv) {
        if (wv(pp->cs, reinterpret_cast<unsigned long long>(ready), I.chunk_end[c], 0) != 0)
          e = cudaErrorUnknown;
      } else {
        cp(L.ready, I.chunk_end + c, sizeof(uint32_t), pp->cs);
      }
    }
    // every copy and counter write is queued before the kernel that waits on
    // them is launched
    if (e == cudaSuccess) e = cudaEventRecord(pp->copied, pp->cs);
  }
  if (e != cudaSuccess) return set_error(XM_ECUDA, std::string("H2D: ") + cudaGetErrorString(e));
  xm_batch b{};
  b.bytes = I.packed ? nullptr : reinterpret_cast<const int64_t*>(w + L.bytes);
  b.tag = I.packed ? nullptr : reinterpret_cast<const uint32_t*>(w + L.tag);
  b.packed = h_direct ? h_direct : I.packed ? reinterpret_cast<const uint64_t*>(w + L.packed) : nullptr;
  b.off = reinterpret_cast<const int64_t*>(w + L.off);
  b.n_ids = reinterpret_cast<const uint32_t*>(w + L.n_ids);
  b.order = reinterpret_cast<const uint32_t*>(w + L.order);
  b.capacity = capacity ? reinterpret_cast<const uint64_t*>(w + L.cap) : nullptr;
  b.n_traces = I.n_traces;
  b.n_events = I.n_events;
  b.max_ids = I.max_ids;
  b.max_events = I.max_events;
  xm_result* d_out = reinterpret_cast<xm_result*>(w + L.out);
  int rc = simulate(&b, cfg, w + L.scratch, L.total - L.scratch, d_out, stream,
                    streamed ? ready : nullptr);
  // `stream` resumes (result download, the caller's later work) only after
  // the copies too, also when the launch failed
  if (streamed) {
    const cudaError_t e2 = cudaStreamWaitEvent(st, g_pipe.copied, 0);
    if (!rc && e2 != cudaSuccess)
      return set_error(XM_ECUDA, std::string("stream wait: ") + cudaGetErrorString(e2));
  }
  if (rc) return rc;
  return xm_peaks(d_out, I.n_traces, h_out, nullptr, XM_UNLIMITED, stream);
}

// ---- raw host traces -> device loader -> replay (xm_simulate_raw) -----------------
namespace {
struct RawLayout {
  size_t bytes, tag, off, order, cap, rec, k5, wbytes, wtag, woff, wnids, out, ready, pos, loaded, scratch,
      total;
};

constexpr int kRawChunks = 256;         // most upload chunks of xm_simulate_raw (ready area)
constexpr int kRawDefaultChunks = 48;   // upload chunks by default (tuned, config 4)
constexpr int kRawLoaderSms = 16;       // SMs of the overlapped loader by default (tuned)
constexpr int kRawFlagEvery = 1;        // landed count published after every n-th chunk
constexpr int64_t kRawOverlapMinTraces = 16;   // smallest batch run overlapped (measured)
constexpr int kRawCopyStreams = 1;      // copy streams the upload chunks alternate over

struct RawShape {
  int64_t T, E;
  uint32_t max_events, max_ids;
};

RawLayout raw_layout(const RawShape& R, const xm_config* cfg) {
  RawLayout L{};
  size_t p = 0;
  const size_t E = size_t(R.E > 0 ? R.E : 1), T = size_t(R.T > 0 ? R.T : 1);
  L.bytes = p; p += al(8 * E);
  L.tag = p; p += al(4 * E);
  L.off = p; p += al(8 * (T + 1));
  L.order = p; p += al(4 * T);
  L.cap = p; p += al(8 * T);
  L.rec = p; p += al(sizeof(xm_lifecycle) * T);
  L.k5 = p; p += al(loader_scratch_bytes(R.T, R.E, R.max_events));
  L.wbytes = p; p += al(8 * E);
  L.wtag = p; p += al(4 * E);
  L.woff = p; p += al(8 * (T + 1));
  L.wnids = p; p += al(4 * T);
  L.out = p; p += al(sizeof(xm_result) * T);
  L.ready = p; p += al(sizeof(uint32_t) * (2 * kRawChunks + 3));   // chunk firsts, 2 landed counts, ranks
  L.pos = p; p += al(4 * T);                                        // caller -> stored index
  L.loaded = p; p += al(4 * (T + 1));                               // completion queue + tail
  L.scratch = p;
  xm_batch b{};
  b.n_traces = R.T;
  b.n_events = R.E;
  b.max_ids = R.max_ids;
  b.max_events = R.max_events;
  p += al(xm_scratch_bytes(&b, cfg));
  L.total = p;
  return L;
}

// host checks of the offsets (the per-event checks run on the device)
int raw_shape(const int64_t* off, int64_t T, RawShape* R, int64_t* bad) {
  if (!off || T < 0) return set_error(XM_EINVAL, "xm_simulate_raw: null offsets or negative n_traces");
  if (off[0] != 0) return set_error(XM_EINVAL, "xm_simulate_raw: off[0] != 0");
  int64_t mx = 0;
  for (int64_t t = 0; t < T; ++t) {
    const int64_t n = off[t + 1] - off[t];
    if (n < 0) { if (bad) *bad = t; return set_error(XM_EINVAL, "xm_simulate_raw: offsets not monotone"); }
    if (n > 0x7FFFFFFFll) {
      if (bad) *bad = t;
      return set_error(XM_ERANGE, "xm_simulate_raw: trace longer than 2^31-1 events");
    }
    mx = std::max(mx, n);
  }
  R->T = T;
  R->E = off[T];
  R->max_events = uint32_t(mx);
  // dense ids of the loader: <= max live + 31 (K5), bounded by the trace length
  R->max_ids = uint32_t(std::min<int64_t>(mx + 32, int64_t(1) << 27));
  return XM_OK;
}

// device-usable pointer of page-locked host memory, or null (pageable)
const void* mapped(const void* h) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, h) != cudaSuccess) { cudaGetLastError(); return nullptr; }
  return a.type == cudaMemoryTypeHost ? a.devicePointer : nullptr;
}

// the loader's verdicts: XM_EINVAL naming the first trace that breaks the
// xm_load_traces contract, else XM_OK
int raw_verdicts(const std::vector<xm_lifecycle>& rec, int64_t T, int64_t* bad_trace) {
  for (int64_t t = 0; t < T; ++t) {
    const xm_lifecycle& r = rec[size_t(t)];
    const char* m = r.n_invalid ? "zero-byte or >= 2^40 request (SPEC.md:231)"
                  : r.n_reopened ? "alloc of a live id (SPEC.md:249)"
                  : r.n_orphan ? "free of a non-live id (SPEC.md:258)"
                  : r.n_mismatch ? "free size differs from the alloc's request (SPEC.md:258)"
                  : r.n_ids > (1u << 27) ? "more than 2^27 live blocks" : nullptr;
    if (m) {
      if (bad_trace) *bad_trace = t;
      return set_error(XM_EINVAL, std::string("xm_simulate_raw: trace ") + std::to_string(t) + ": " + m);
    }
  }
  clear_error();
  return XM_OK;
}
}  // namespace

extern "C" size_t xm_raw_ws_bytes(const int64_t* h_off, int64_t n_traces, const xm_config* cfg) {
  RawShape R{};
  if (!cfg || raw_shape(h_off, n_traces, &R, nullptr)) return 0;
  return raw_layout(R, cfg).total;
}

extern "C" int xm_simulate_raw(const int64_t* h_bytes, const uint32_t* h_tag, const int64_t* h_off,
                               int64_t n_traces, const uint64_t* h_capacity, const xm_config* cfg,
                               void* d_ws, size_t ws_bytes, xm_result* h_out, int64_t* bad_trace,
                               void* stream) {
  if (bad_trace) *bad_trace = -1;
  if (!cfg || !h_out) return set_error(XM_EINVAL, "xm_simulate_raw: null argument");
  RawShape R{};
  int rc = raw_shape(h_off, n_traces, &R, bad_trace);
  if (rc) return rc;
  if (R.T == 0) return XM_OK;
  if (R.E > 0 && (!h_bytes || !h_tag)) return set_error(XM_EINVAL, "xm_simulate_raw: null event arrays");
  if (cfg->mode != XM_FULL) return set_error(XM_EINVAL, "xm_simulate_raw: XM_FULL mode only");
  UnitConfig u;
  if ((rc = make_unit_config(cfg, &u))) return rc;
  const RawLayout L = raw_layout(R, cfg);
  if (!d_ws || ws_bytes < L.total) return set_error(XM_ENOMEM, "xm_simulate_raw: workspace too small");
  if (!cuda_usable()) return set_error(XM_ECUDA, "no CUDA device");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char* w = static_cast<char*>(d_ws);
  cudaError_t e = cudaSuccess;
  auto cp = [&](size_t o, const void* src, size_t n) {
    if (e == cudaSuccess && n) e = cudaMemcpyAsync(w + o, src, n, cudaMemcpyHostToDevice, st);
  };
  // events. Page-locked (the usual case): copied by the DMA engine in chunks
  // of whole traces (contiguous in caller order) on the library's copy
  // stream, the chunks holding the longest traces first (a trace's loader and
  // replay time grow with its length, so the last chunks to land should hold
  // short ones); each chunk is followed by a stream-ordered write of its
  // flag, which the loader's warps wait on (trace t's warp starts once its
  // chunk has landed). The transfer thus overlaps the loader (the copy engine
  // moves ~55 GB/s where warps reading host memory in place managed ~36).
  // XM_RAW_INPUT=direct reads in place instead (tooling). Pageable: copied
  // first.
  const int64_t* d_bytes = static_cast<const int64_t*>(mapped(h_bytes));
  const uint32_t* d_tag = static_cast<const uint32_t*>(mapped(h_tag));
  const char* rin = std::getenv("XM_RAW_INPUT");
  const bool direct = rin && !std::strcmp(rin, "direct");
  const bool streamed = d_bytes && d_tag && !direct && R.E > 0;
  cp(L.off, h_off, 8 * size_t(R.T + 1));
  uint32_t* chunk_first = reinterpret_cast<uint32_t*>(w + L.ready);
  uint32_t* chunk_flag = chunk_first + (kRawChunks + 1);
  int n_chunks = 0;
  Pipe* pp = nullptr;
  static thread_local std::vector<uint32_t> firsts;    // outlive the async copies
  static thread_local std::vector<uint32_t> ones;      // chunk ranks (upload)
  static thread_local std::vector<uint32_t> counts;    // landed-count values (fallback copies)
  int n_cs = 1;                                        // copy streams the chunks alternate over
  std::vector<int> corder;
  if (streamed) {
    // chunks: whole traces up to about (c+1)/n of the events (n: XM_RAW_CHUNKS,
    // tooling, at most kRawChunks)
    const char* nc = std::getenv("XM_RAW_CHUNKS");
    const int want = nc ? std::max(1, std::min(kRawChunks, std::atoi(nc))) : kRawDefaultChunks;
    firsts.clear();
    firsts.reserve(size_t(want) + 1);
    std::vector<int64_t> maxlen;
    int64_t t = 0;
    for (int c = 0; c < want && t < R.T; ++c) {
      const int64_t goal = (R.E * (c + 1)) / want;
      const int64_t t0 = t;
      int64_t ml = 0;
      while (t < R.T && (h_off[t + 1] <= goal || c == want - 1)) {
        ml = std::max<int64_t>(ml, h_off[t + 1] - h_off[t]);
        ++t;
      }
      if (t == t0) continue;
      firsts.push_back(uint32_t(t0));
      maxlen.push_back(ml);
    }
    n_chunks = int(firsts.size());
    firsts.push_back(uint32_t(R.T));
    cp(L.ready, firsts.data(), sizeof(uint32_t) * firsts.size());
    if (e == cudaSuccess) e = get_pipe(&pp);
    corder.resize(size_t(n_chunks));
    for (int c = 0; c < n_chunks; ++c) corder[size_t(c)] = c;
    std::stable_sort(corder.begin(), corder.end(),
                     [&](int x, int y) { return maxlen[size_t(x)] > maxlen[size_t(y)]; });
    // chunk_flag[0] / [1]: chunks landed so far on copy stream 0 / 1 (0 now);
    // [2 + c]: chunk c's stream << 31 | rank in that stream's copy order
    // (uploaded from `ones`); the i-th chunk in copy order goes to stream
    // i % n_cs. counts[i] = i: the landed counts' values, for the fallback
    // copy where the driver lacks cuStreamWriteValue32
    const char* ncs = std::getenv("XM_RAW_COPY_STREAMS");                // tooling: 1 or 2
    n_cs = (ncs && ncs[0] == '2') ? 2 : kRawCopyStreams;
    ones.assign(size_t(kRawChunks) + 2, 0u);
    for (int i = 0; i < n_chunks; ++i)
      ones[size_t(2 + corder[size_t(i)])] = (uint32_t(i % n_cs) << 31) | uint32_t(i / n_cs);
    cp(size_t(reinterpret_cast<char*>(chunk_flag) - w), ones.data(), sizeof(uint32_t) * (size_t(n_chunks) + 2));
    counts.resize(size_t(kRawChunks) + 1);
    for (int i = 0; i <= kRawChunks; ++i) counts[size_t(i)] = uint32_t(i);
    d_bytes = reinterpret_cast<const int64_t*>(w + L.bytes);
    d_tag = reinterpret_cast<const uint32_t*>(w + L.tag);
  } else if (!direct || !d_bytes || !d_tag) {
    if (!d_bytes) { cp(L.bytes, h_bytes, 8 * size_t(R.E)); d_bytes = reinterpret_cast<int64_t*>(w + L.bytes); }
    if (!d_tag) { cp(L.tag, h_tag, 4 * size_t(R.E)); d_tag = reinterpret_cast<uint32_t*>(w + L.tag); }
  }
  // the chunk copies and their flags on the copy stream, which starts after
  // everything queued on `stream` so far (earlier users of the workspace, the
  // flag resets); `copied` is recorded after the last one
  // after: an event already recorded on `stream` before any kernel that waits
  // on the chunks (else one is recorded now)
  auto enqueue_chunks = [&](cudaEvent_t after) {
    if (!after) {
      after = pp->start;
      if (e == cudaSuccess) e = cudaEventRecord(after, st);
    }
    if (e == cudaSuccess) e = cudaStreamWaitEvent(pp->cs, after, 0);
    if (e == cudaSuccess && n_cs > 1) e = cudaStreamWaitEvent(pp->cs2, after, 0);
    const WriteValue32Fn wv = write_value32();
    // the landed count is published after every `every`-th chunk (and the
    // last): fewer stream memory operations between the copies (XM_RAW_FLAG_EVERY,
    // tooling)
    const char* fe = std::getenv("XM_RAW_FLAG_EVERY");
    const int every = fe ? std::max(1, std::atoi(fe)) : kRawFlagEvery;
    int landed[2] = {0, 0};
    int pos = 0;
    for (int c : corder) {
      if (e != cudaSuccess) break;
      const int sidx = pos % n_cs;
      ++pos;
      cudaStream_t cst = sidx ? pp->cs2 : pp->cs;
      // the copied range is widened to 32-event boundaries (whole cache lines:
      // a boundary line is written by both neighbours, with the same bytes)
      const int64_t ev0 = h_off[firsts[size_t(c)]] & ~int64_t(31);
      const int64_t ev1 = std::min<int64_t>(R.E, (h_off[firsts[size_t(c) + 1]] + 31) & ~int64_t(31));
      if (ev1 > ev0) {
        e = cudaMemcpyAsync(w + L.bytes + 8 * size_t(ev0), h_bytes + ev0, 8 * size_t(ev1 - ev0),
                            cudaMemcpyHostToDevice, cst);
        if (e == cudaSuccess)
          e = cudaMemcpyAsync(w + L.tag + 4 * size_t(ev0), h_tag + ev0, 4 * size_t(ev1 - ev0),
                              cudaMemcpyHostToDevice, cst);
      }
      if (e != cudaSuccess) break;
      const int lc = ++landed[sidx];
      const int last_here = (n_chunks - 1 - sidx) / n_cs + 1;   // chunks on this stream
      if (lc % every != 0 && lc != last_here) continue;
      if (wv) {
        if (wv(cst, reinterpret_cast<unsigned long long>(chunk_flag + sidx), uint32_t(lc), 0) != 0)
          e = cudaErrorUnknown;
      } else {
        e = cudaMemcpyAsync(chunk_flag + sidx, &counts[size_t(lc)], sizeof(uint32_t), cudaMemcpyHostToDevice,
                            cst);
      }
    }
    if (e == cudaSuccess && n_cs > 1) e = cudaEventRecord(pp->copied2, pp->cs2);
    if (e == cudaSuccess && n_cs > 1) e = cudaStreamWaitEvent(pp->cs, pp->copied2, 0);
    if (e == cudaSuccess) e = cudaEventRecord(pp->copied, pp->cs);
  };
  // processing order of the replay: longest first, ties in caller order (as
  // xm_load_traces)
  std::vector<uint32_t> order(size_t(R.T));
  for (int64_t i = 0; i < R.T; ++i) order[size_t(i)] = uint32_t(i);
  std::stable_sort(order.begin(), order.end(), [&](uint32_t x, uint32_t y) {
    return h_off[x + 1] - h_off[x] > h_off[y + 1] - h_off[y];
  });
  cp(L.order, order.data(), 4 * size_t(R.T));
  if (h_capacity) cp(L.cap, h_capacity, 8 * size_t(R.T));
  // the wire arrays' offsets (stored order: a valid trace keeps all its
  // events) and each caller trace's stored index, so the loader writes the
  // wire in place (no staging / compaction pass)
  static thread_local std::vector<int64_t> woff;      // outlive the async copies
  static thread_local std::vector<uint32_t> pos;
  woff.assign(size_t(R.T) + 1, 0);
  pos.assign(size_t(R.T), 0);
  for (int64_t k = 0; k < R.T; ++k) {
    const uint32_t t = order[size_t(k)];
    pos[t] = uint32_t(k);
    woff[size_t(k) + 1] = woff[size_t(k)] + (h_off[t + 1] - h_off[t]);
  }
  cp(L.woff, woff.data(), 8 * size_t(R.T + 1));
  cp(L.pos, pos.data(), 4 * size_t(R.T));
  if (e != cudaSuccess) return set_error(XM_ECUDA, std::string("xm_simulate_raw H2D: ") + cudaGetErrorString(e));
  int launches = 0;
  xm_lifecycle* d_rec = reinterpret_cast<xm_lifecycle*>(w + L.rec);
  xm_batch b{};
  b.bytes = reinterpret_cast<const int64_t*>(w + L.wbytes);
  b.tag = reinterpret_cast<const uint32_t*>(w + L.wtag);
  b.off = reinterpret_cast<const int64_t*>(w + L.woff);
  b.n_ids = reinterpret_cast<const uint32_t*>(w + L.wnids);
  b.order = reinterpret_cast<const uint32_t*>(w + L.order);
  b.capacity = h_capacity ? reinterpret_cast<const uint64_t*>(w + L.cap) : nullptr;
  b.n_traces = R.T;
  b.n_events = R.E;
  b.max_ids = R.max_ids;
  b.max_events = R.max_events;
  xm_result* d_out = reinterpret_cast<xm_result*>(w + L.out);
  // Overlapped replay (the default for batches that fill the GPU): the loader
  // runs on `loader_sms` SMs (one 32-warp CTA each, on the library's loader
  // stream), longest trace first among those whose chunk has landed, and
  // appends each finished trace to a completion queue; the replay runs on the
  // other SMs from the start, its i-th pull taking the queue's i-th entry, so
  // traces replay while the rest is still crossing PCIe; a second replay
  // launch on the loader's SMs follows the loader and shares the first one's
  // work counter. The two kernels cannot share an SM (registers), so each CTA
  // holds a whole SM. The chunk copies are queued after the launches (the
  // kernels wait on their flags), so the host's API calls overlap the GPU.
  const ReplayPlan plan = plan_replay(&b, cfg);
  int dev_sms = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, dev);
    cudaGetLastError();
  }
  const char* ov = std::getenv("XM_RAW_OVERLAP");                      // tooling: "0" = off
  const char* lsm = std::getenv("XM_RAW_LOADER_SMS");                  // tooling
  // a batch that fills the GPU: the loader on loader_sms SMs, the replay on
  // the rest and then on the loader's; a smaller one (>= kRawOverlapMinTraces
  // traces: below that the streams' synchronisation costs more than the
  // overlap saves -- one 486-event trace: 0.59 vs 0.47 ms): the replay on the
  // SMs it needs (plan.ctas), the loader on all the others, no second launch
  const bool big = plan.ctas >= dev_sms;
  const int loader_sms = big ? (lsm ? std::atoi(lsm) : kRawLoaderSms) : dev_sms - plan.ctas;
  const bool overlap = streamed && !(ov && ov[0] == '0') && loader_sms >= 1 && loader_sms < dev_sms &&
                       R.T >= kRawOverlapMinTraces && L.total - L.scratch >= plan.scratch_bytes;
  if (overlap) {
    uint32_t* loaded = reinterpret_cast<uint32_t*>(w + L.loaded);
    void* k2s = w + L.scratch;
    // both modules loaded before either kernel runs: a lazy module load at a
    // launch may wait for the running kernels, which here wait on the chunk
    // copies queued after the launches
    int pe = preload_loader();
    if (!pe) pe = preload_replay();
    if (pe) return set_error(XM_ECUDA, std::string("xm_simulate_raw: module load: ") +
                                           cudaGetErrorString(cudaError_t(pe)));
    e = cudaMemsetAsync(loaded, 0, 4 * size_t(R.T + 1), st);
    if (e == cudaSuccess) e = cudaMemsetAsync(k2s, 0, 256, st);       // the replay's counters
    if (e == cudaSuccess) e = cudaEventRecord(pp->meta, st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(pp->ls, pp->meta, 0);
    if (e != cudaSuccess) return set_error(XM_ECUDA, std::string("xm_simulate_raw: ") + cudaGetErrorString(e));
    int ek = launch_loader(d_bytes, d_tag, reinterpret_cast<const int64_t*>(w + L.off), R.T, R.E,
                           R.max_events, w + L.k5, d_rec, reinterpret_cast<const uint32_t*>(w + L.order),
                           reinterpret_cast<int64_t*>(w + L.wbytes), reinterpret_cast<uint32_t*>(w + L.wtag),
                           reinterpret_cast<int64_t*>(w + L.woff), reinterpret_cast<uint32_t*>(w + L.wnids),
                           pp->ls, &launches, chunk_first, chunk_flag, n_chunks,
                           reinterpret_cast<const uint32_t*>(w + L.pos), loaded, loader_sms,
                           reinterpret_cast<uint32_t*>(static_cast<char*>(k2s) + 4 * 24));
    if (!ek) ek = launch_replay(&b, cfg, u, plan, k2s, d_out, st, &launches, nullptr, loaded,
                                big ? dev_sms - loader_sms : plan.ctas, false);
    if (!ek && big)
      ek = launch_replay(&b, cfg, u, plan, k2s, d_out, pp->ls, &launches, nullptr, loaded,
                         loader_sms, false);
    enqueue_chunks(pp->meta);    // also when a launch failed: `copied` must exist
    // `stream` resumes after the loader's stream and the copies, also on failure
    const cudaError_t e1 = cudaEventRecord(pp->ldone, pp->ls);
    const cudaError_t e2 = e1 == cudaSuccess ? cudaStreamWaitEvent(st, pp->ldone, 0) : e1;
    const cudaError_t e3 = cudaStreamWaitEvent(st, pp->copied, 0);
    if (ek) return set_error(XM_ECUDA, std::string("xm_simulate_raw launch: ") + cudaGetErrorString(cudaError_t(ek)));
    if (e != cudaSuccess) return set_error(XM_ECUDA, std::string("xm_simulate_raw H2D: ") + cudaGetErrorString(e));
    if (e2 != cudaSuccess || e3 != cudaSuccess)
      return set_error(XM_ECUDA, std::string("stream wait: ") + cudaGetErrorString(e2 != cudaSuccess ? e2 : e3));
    launch_counter() = launches;
    std::vector<xm_lifecycle> rec(size_t(R.T));
    uint32_t stall = 0;
    e = cudaMemcpyAsync(h_out, d_out, sizeof(xm_result) * size_t(R.T), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(rec.data(), d_rec, sizeof(xm_lifecycle) * size_t(R.T), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(&stall, static_cast<char*>(k2s) + 4 * 24, sizeof(uint32_t), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return set_error(XM_ECUDA, std::string("xm_simulate_raw D2H: ") + cudaGetErrorString(e));
    if (stall)
      return set_error(XM_ECUDA, "xm_simulate_raw: the loader made no progress (too few free SMs for "
                                 "the overlapped loader; set XM_RAW_OVERLAP=0)");
    return raw_verdicts(rec, R.T, bad_trace);
  }
  if (streamed) {
    // sequential: every copy and flag write is queued before the loader that
    // waits on them
    enqueue_chunks(nullptr);
    if (e != cudaSuccess) return set_error(XM_ECUDA, std::string("xm_simulate_raw H2D: ") + cudaGetErrorString(e));
  }
  int ek = launch_loader(d_bytes, d_tag, reinterpret_cast<const int64_t*>(w + L.off), R.T, R.E,
                         R.max_events, w + L.k5, d_rec, reinterpret_cast<const uint32_t*>(w + L.order),
                         reinterpret_cast<int64_t*>(w + L.wbytes), reinterpret_cast<uint32_t*>(w + L.wtag),
                         reinterpret_cast<int64_t*>(w + L.woff), reinterpret_cast<uint32_t*>(w + L.wnids),
                         stream, &launches, streamed ? chunk_first : nullptr,
                         streamed ? chunk_flag : nullptr, n_chunks,
                         reinterpret_cast<const uint32_t*>(w + L.pos));
  // `stream` resumes (the replay, result download, later users of the
  // workspace) only after the copies too, also when the launch failed
  if (streamed) {
    const cudaError_t e2 = cudaStreamWaitEvent(st, pp->copied, 0);
    if (!ek && e2 != cudaSuccess)
      return set_error(XM_ECUDA, std::string("stream wait: ") + cudaGetErrorString(e2));
  }
  if (ek) return set_error(XM_ECUDA, std::string("xm_simulate_raw loader: ") + cudaGetErrorString(cudaError_t(ek)));
  rc = simulate(&b, cfg, w + L.scratch, L.total - L.scratch, d_out, stream, nullptr);
  launch_counter() += launches;
  if (rc) return rc;
  // results and the loader's verdicts back (one synchronisation)
  std::vector<xm_lifecycle> rec(size_t(R.T));
  e = cudaMemcpyAsync(h_out, d_out, sizeof(xm_result) * size_t(R.T), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(rec.data(), d_rec, sizeof(xm_lifecycle) * size_t(R.T), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return set_error(XM_ECUDA, std::string("xm_simulate_raw D2H: ") + cudaGetErrorString(e));
  return raw_verdicts(rec, R.T, bad_trace);
}
