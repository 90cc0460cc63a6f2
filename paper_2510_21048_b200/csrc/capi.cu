// capi.cu -- the extern "C" entry points of libxmem.so (include/xmem.h) that
// are not the loader: configuration, scratch sizing, the device and host
// simulate calls, result download and error reporting.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>

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
  if (c->mode != XM_FULL && c->mode != XM_ALLOCATED_ONLY)
    return set_error(XM_EINVAL, "xm_config: unknown mode");
  int sh = 0;
  while ((1ull << sh) < m) ++sh;
  u->unit_shift = uint32_t(sh);
  u->small_u = uint32_t(c->small_size / m);
  u->sbuf_u = uint32_t(c->small_buffer / m);
  u->lbuf_u = uint32_t(c->large_buffer / m);
  u->minlarge_u = uint32_t(c->min_large_alloc / m);
  u->rlarge_u = uint32_t(c->round_large / m);
  u->strict = c->large_split_strict ? 1u : 0u;
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
}

extern "C" const char* xm_last_error(void) { return g_err.c_str(); }

extern "C" int xm_last_launch_count(void) { return launch_counter(); }

static int check_batch(const xm_batch* b) {
  if (!b) return set_error(XM_EINVAL, "null batch");
  if (b->n_traces < 0 || b->n_events < 0) return set_error(XM_EINVAL, "negative sizes");
  if (b->n_traces > 0x7FFFFFFFll) return set_error(XM_ERANGE, "more than 2^31-1 traces");
  if (b->n_traces > 0 && (!b->off || !b->n_ids || !b->order))
    return set_error(XM_EINVAL, "null device array in batch");
  if (b->n_events > 0 && (!b->bytes || !b->tag)) return set_error(XM_EINVAL, "null event arrays");
  return XM_OK;
}

extern "C" size_t xm_scratch_bytes(const xm_batch* b, const xm_config* cfg) {
  if (!b || !cfg) return 0;
  if (cfg->mode == XM_ALLOCATED_ONLY) return scan_scratch_bytes(b);
  return plan_replay(b, cfg).scratch_bytes;
}

extern "C" int xm_simulate_batch(const xm_batch* b, const xm_config* cfg, void* d_scratch,
                                 size_t scratch_bytes, xm_result* d_out, void* stream) {
  launch_counter() = 0;
  if (!cfg) return set_error(XM_EINVAL, "null config");
  int rc = check_batch(b);
  if (rc) return rc;
  UnitConfig u;
  if ((rc = make_unit_config(cfg, &u))) return rc;
  if (b->n_traces == 0) return XM_OK;
  if (!d_out || !d_scratch) return set_error(XM_EINVAL, "null output or scratch");
  if (!cuda_usable()) return set_error(XM_ECUDA, "no CUDA device");
  int e;
  if (cfg->mode == XM_ALLOCATED_ONLY) {
    if (cfg->capacity != XM_UNLIMITED || b->capacity)
      return set_error(XM_EINVAL, "XM_ALLOCATED_ONLY requires unlimited capacity");
    if (b->curve) return set_error(XM_EINVAL, "the memory curve needs XM_FULL");
    if (scratch_bytes < scan_scratch_bytes(b)) return set_error(XM_ENOMEM, "scratch too small");
    e = launch_scan(b, u, d_scratch, scratch_bytes, d_out, stream, &launch_counter());
  } else {
    ReplayPlan plan = plan_replay(b, cfg);
    if (scratch_bytes < plan.scratch_bytes)
      return set_error(XM_ENOMEM, "scratch smaller than xm_scratch_bytes()");
    e = launch_replay(b, cfg, u, plan, d_scratch, d_out, stream, &launch_counter());
  }
  if (e != 0)
    return set_error(XM_ECUDA, std::string("launch failed: ") + cudaGetErrorString(cudaError_t(e)));
  clear_error();
  return XM_OK;
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
  size_t bytes, tag, off, n_ids, order, cap, out, scratch, total;
};
size_t al(size_t x) { return (x + 255) & ~size_t(255); }

HostLayout host_layout(const xm_traces_info& I, const xm_config* cfg, bool with_cap) {
  HostLayout L{};
  size_t p = 0;
  L.bytes = p; p += al(sizeof(int64_t) * I.n_events);
  L.tag = p; p += al(sizeof(uint32_t) * I.n_events);
  L.off = p; p += al(sizeof(int64_t) * (I.n_traces + 1));
  L.n_ids = p; p += al(sizeof(uint32_t) * I.n_traces);
  L.order = p; p += al(sizeof(uint32_t) * I.n_traces);
  L.cap = p; p += with_cap ? al(sizeof(uint64_t) * I.n_traces) : 0;
  L.out = p; p += al(sizeof(xm_result) * I.n_traces);
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
}  // namespace

extern "C" size_t xm_host_ws_bytes(const xm_traces* tr, const xm_config* cfg) {
  if (!tr || !cfg) return 0;
  return host_layout(traces_info(tr), cfg, true).total;
}

extern "C" int xm_simulate_host(const xm_traces* tr, const uint64_t* capacity,
                                const xm_config* cfg, void* d_ws, size_t ws_bytes,
                                xm_result* h_out, void* stream) {
  if (!tr || !cfg || !d_ws || !h_out) return set_error(XM_EINVAL, "xm_simulate_host: null argument");
  const xm_traces_info I = traces_info(tr);
  const HostLayout L = host_layout(I, cfg, true);
  if (ws_bytes < L.total) return set_error(XM_ENOMEM, "xm_simulate_host: workspace too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char* w = static_cast<char*>(d_ws);
  cudaError_t e = cudaSuccess;
  auto cp = [&](size_t o, const void* src, size_t n) {
    if (e == cudaSuccess && n) e = cudaMemcpyAsync(w + o, src, n, cudaMemcpyHostToDevice, st);
  };
  cp(L.bytes, I.bytes, sizeof(int64_t) * I.n_events);
  cp(L.tag, I.tag, sizeof(uint32_t) * I.n_events);
  cp(L.off, I.off, sizeof(int64_t) * (I.n_traces + 1));
  cp(L.n_ids, I.n_ids, sizeof(uint32_t) * I.n_traces);
  cp(L.order, I.order, sizeof(uint32_t) * I.n_traces);
  if (capacity) cp(L.cap, capacity, sizeof(uint64_t) * I.n_traces);
  if (e != cudaSuccess) return set_error(XM_ECUDA, std::string("H2D: ") + cudaGetErrorString(e));
  xm_batch b{};
  b.bytes = reinterpret_cast<const int64_t*>(w + L.bytes);
  b.tag = reinterpret_cast<const uint32_t*>(w + L.tag);
  b.off = reinterpret_cast<const int64_t*>(w + L.off);
  b.n_ids = reinterpret_cast<const uint32_t*>(w + L.n_ids);
  b.order = reinterpret_cast<const uint32_t*>(w + L.order);
  b.capacity = capacity ? reinterpret_cast<const uint64_t*>(w + L.cap) : nullptr;
  b.n_traces = I.n_traces;
  b.n_events = I.n_events;
  b.max_ids = I.max_ids;
  b.max_events = I.max_events;
  xm_result* d_out = reinterpret_cast<xm_result*>(w + L.out);
  int rc = xm_simulate_batch(&b, cfg, w + L.scratch, L.total - L.scratch, d_out, stream);
  if (rc) return rc;
  return xm_peaks(d_out, I.n_traces, h_out, nullptr, XM_UNLIMITED, stream);
}
