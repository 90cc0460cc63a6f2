// metrics.cu -- batched evaluation metrics over many runs (SURVEY.md §8(f)
// NEXT-4): the paper's MRE, PEF and MCP (Eqs.
// relative-error, median-error, 1st/2nd correctness, failed-estimation-
// probability, memory-savings, estimator-memory-average-saving).
//
//   k_metrics_map  one thread per run: C1, C2, M_save, the selected relative
//                  error (as its IEEE-754 bit pattern: errors are >= 0, so the
//                  bits order like the values); CTA-reduced sums -> atomics.
//   k_select_hist  grid-wide: histogram of the next 8-bit digit of the error
//   k_select_pick  keys matching the digits chosen so far; one warp picks the
//                  digit holding each wanted rank (8 passes) -> the k-th and
//                  (k+1)-th smallest keys -> the median (mean of the central
//                  pair for even counts) and the finished record.
// HBM: 40 B/run read, 8 B/run written + 8 passes x 8 B/run re-read (L2).
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>

#include "xm_internal.h"

namespace {

constexpr int kMapThreads = 256;
constexpr int kHistThreads = 512;
constexpr size_t kHdr = 4096;          // Acc, SelState, result record; keys follow

static_assert(sizeof(xm_metrics) <= 128, "scratch layout");

struct Acc {                      // scratch accumulators (zeroed per call)
  unsigned long long c1, c2, n_sel, bad;
  unsigned long long save;        // signed sum, two's complement
  unsigned long long pad[3];
};

__global__ void __launch_bounds__(kMapThreads) k_metrics_map(const xm_run* __restrict__ runs,
                                                             int64_t n, uint64_t* keys, Acc* acc) {
  unsigned long long c1s = 0, c2s = 0, sel = 0, bad = 0, save = 0;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const xm_run r = runs[i];
    const bool oom1 = r.oom1 != 0;
    const bool r2 = r.oom2 != XM_ROUND2_NOT_RUN;
    const bool oom2_0 = r2 && r.oom2 == 0;
    const int c1 = (r.oom_pred != 0) == oom1;                       // Eq. 1st-correctness
    const int c2 = c1 && (oom2_0 || oom1);                          // Eq. 2nd correctness
    bad += (r2 && !(c1 && !oom1)) || (!oom1 && !oom2_0 && r.m_peak_meas1 == 0) ||
           (oom2_0 && r.m_peak_meas2 == 0);
    long long sv;                                                   // Eq. memory-savings
    if (c1 && oom2_0) sv = (long long)r.m_max - (long long)r.m_peak_est;
    else if (c1 && oom1) sv = (long long)r.m_max;
    else sv = -(long long)r.m_max;
    c1s += c1;
    c2s += c2;
    save += (unsigned long long)sv;
    uint64_t key = ~0ull;                                           // not selected
    if (!oom1) {                                                    // OOM_jd1 = 0
      const uint64_t meas = oom2_0 ? r.m_peak_meas2 : r.m_peak_meas1;
      const uint64_t diff = r.m_peak_est > meas ? r.m_peak_est - meas : meas - r.m_peak_est;
      const double e = meas ? __ull2double_rn(diff) / __ull2double_rn(meas) : 0.0;
      key = uint64_t(__double_as_longlong(e));
      ++sel;
    }
    keys[i] = key;
  }
  // CTA reduction, one atomic per field per CTA
  __shared__ unsigned long long red[5][kMapThreads / 32];
  unsigned long long v[5] = {c1s, c2s, sel, bad, save};
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int f = 0; f < 5; ++f) {
    unsigned long long x = v[f];
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xFFFFFFFFu, x, o);
    if (lane == 0) red[f][w] = x;
  }
  __syncthreads();
  if (threadIdx.x < 5) {
    unsigned long long x = 0;
    for (int k = 0; k < kMapThreads / 32; ++k) x += red[threadIdx.x][k];
    unsigned long long* dst[5] = {&acc->c1, &acc->c2, &acc->n_sel, &acc->bad, &acc->save};
    atomicAdd(dst[threadIdx.x], x);
  }
}

// The two central order statistics of the selected keys by 8-bit MSD radix
// select, 8 passes; each pass is a grid-wide histogram of the next digit over
// the keys that match the digits chosen so far (per-CTA shared-memory
// histograms merged with one atomic per bin), then one small kernel picks the
// digit that holds each wanted rank. Both order statistics (the k-th and
// (k+1)-th smallest, for the median of an even count) are selected at once.
struct SelState {                 // scratch, zeroed per call
  uint64_t prefix[2];             // digits chosen so far (the selected keys' high bits)
  uint64_t mask;                  // the bits chosen so far
  unsigned long long rank[2];     // rank still to skip inside the current prefix
  unsigned int hist[2][256];
};

__global__ void __launch_bounds__(kHistThreads) k_select_hist(const uint64_t* __restrict__ keys,
                                                              int64_t n, int shift, SelState* S) {
  __shared__ unsigned int h[2][256];
  for (int b = threadIdx.x; b < 512; b += blockDim.x) (&h[0][0])[b] = 0;
  __syncthreads();
  const uint64_t mask = S->mask, p0 = S->prefix[0], p1 = S->prefix[1];
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t k = __ldg(keys + i);
    const unsigned d = unsigned(k >> shift) & 0xFFu;
    if ((k & mask) == p0) atomicAdd(&h[0][d], 1u);
    if ((k & mask) == p1) atomicAdd(&h[1][d], 1u);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < 512; b += blockDim.x) {
    const unsigned v = (&h[0][0])[b];
    if (v) atomicAdd(&(&S->hist[0][0])[b], v);
  }
}

// one warp: lane j < 2 picks the digit holding rank[j]; the histograms are
// cleared for the next pass; after the last pass, the metrics record
__global__ void k_select_pick(int shift, SelState* S, const Acc* acc, int64_t n, xm_metrics* res) {
  const unsigned long long m = acc->n_sel;
  const int j = threadIdx.x;
  if (j < 2 && m > 0) {
    unsigned long long rank = shift == 56 ? (m - 1) / 2 + (j == 1 && (m % 2 == 0) ? 1 : 0) : S->rank[j];
    unsigned long long c = 0;
    int d = 0;
    for (; d < 255; ++d) {
      if (c + S->hist[j][d] > rank) break;
      c += S->hist[j][d];
    }
    S->prefix[j] |= uint64_t(d) << shift;
    S->rank[j] = rank - c;
  }
  __syncwarp();
  for (int b = threadIdx.x; b < 512; b += blockDim.x) (&S->hist[0][0])[b] = 0;
  if (j == 0) S->mask |= 0xFFull << shift;
  if (shift == 0 && j == 0) {
    const double nn = double(n);
    xm_metrics r;
    r.n = uint64_t(n);
    r.n_mre = m;
    r.sum_c1 = acc->c1;
    r.sum_c2 = acc->c2;
    r.sum_save = (long long)acc->save;
    const double a = __longlong_as_double((long long)S->prefix[0]);
    const double b = __longlong_as_double((long long)S->prefix[1]);
    r.mre = m == 0 ? __longlong_as_double(0x7FF8000000000000ll) : ((m % 2) ? a : (a + b) / 2.0);
    r.pef1 = double(uint64_t(n) - acc->c1) / nn;               // Eq. failed-estimation-probability
    r.pef2 = double(uint64_t(n) - acc->c2) / nn;
    r.mcp = double((long long)acc->save) / nn;                 // Eq. estimator-memory-average-saving
    *res = r;
  }
}

}  // namespace

using namespace xm_internal;

extern "C" size_t xm_metrics_scratch_bytes(int64_t n_runs) {
  return kHdr + size_t(n_runs > 0 ? n_runs : 0) * 8;
}

extern "C" int xm_metrics_batch(const xm_run* d_runs, int64_t n, void* d_scratch,
                                size_t scratch_bytes, xm_metrics* h_out, void* stream) {
  launch_counter() = 0;
  if (!h_out || n < 0) return set_error(XM_EINVAL, "xm_metrics_batch: bad arguments");
  std::memset(h_out, 0, sizeof(*h_out));
  if (n == 0) return set_error(XM_EINVAL, "xm_metrics_batch: no runs (SPEC.md:386 no-data)");
  if (!d_runs || !d_scratch) return set_error(XM_EINVAL, "xm_metrics_batch: null pointer");
  if (scratch_bytes < xm_metrics_scratch_bytes(n)) return set_error(XM_ENOMEM, "scratch too small");
  if (!cuda_usable()) return set_error(XM_ECUDA, "no CUDA device");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char* base = static_cast<char*>(d_scratch);
  Acc* acc = reinterpret_cast<Acc*>(base);
  xm_metrics* d_res = reinterpret_cast<xm_metrics*>(base + 128);
  SelState* sel = reinterpret_cast<SelState*>(base + 256);
  static_assert(256 + sizeof(SelState) <= kHdr, "metrics scratch header");
  uint64_t* keys = reinterpret_cast<uint64_t*>(base + kHdr);
  cudaError_t e = cudaMemsetAsync(d_scratch, 0, kHdr, st);
  if (e != cudaSuccess) return set_error(XM_ECUDA, cudaGetErrorString(e));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (n + kMapThreads - 1) / kMapThreads;
  const int grid = int(want < int64_t(sms) * 8 ? want : int64_t(sms) * 8);
  k_metrics_map<<<grid, kMapThreads, 0, st>>>(d_runs, n, keys, acc);
  const int64_t hwant = (n + kHistThreads * 4 - 1) / (kHistThreads * 4);
  const int hgrid = int(hwant < int64_t(sms) * 2 ? (hwant > 0 ? hwant : 1) : int64_t(sms) * 2);
  for (int shift = 56; shift >= 0; shift -= 8) {
    k_select_hist<<<hgrid, kHistThreads, 0, st>>>(keys, n, shift, sel);
    k_select_pick<<<1, 32, 0, st>>>(shift, sel, acc, n, d_res);
  }
  launch_counter() = 1 + 2 * 8;
  Acc h{};
  if ((e = cudaMemcpyAsync(&h, acc, sizeof(h), cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
      (e = cudaMemcpyAsync(h_out, d_res, sizeof(*h_out), cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
      (e = cudaStreamSynchronize(st)) != cudaSuccess)
    return set_error(XM_ECUDA, std::string("xm_metrics_batch: ") + cudaGetErrorString(e));
  if (h.bad) {
    std::memset(h_out, 0, sizeof(*h_out));
    return set_error(XM_EINVAL, "xm_metrics_batch: invalid run record (round-2 gating "
                                "P:385, or a zero measured peak)");
  }
  return XM_OK;
}
