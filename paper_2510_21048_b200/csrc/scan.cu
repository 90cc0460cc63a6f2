// scan.cu -- K1: allocated-bytes peak as a segmented prefix-scan/max (sm_100a).
//
// For every trace, peak_allocated = max over events i of sum_{k<=i} +-s_k with
// s_k the 512 B round-up of event k's request (PAPER.md:256 (i)
// "allocated_bytes changes by exactly the rounded request"), and its first
// index (reading Q7). Allocator state is not needed for this quantity, so it
// is exact whenever no OOM truncates the trace (unlimited capacity).
//
// v1: one warp per trace, persistent, longest trace first; each lane owns 4
// consecutive events per 128-event round (in-lane scan + one warp scan per
// round). The flat, trace-oblivious tiling is the planned v2 (K1).
#include <cuda_runtime.h>

#include "xm_internal.h"

namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;

struct SParams {
  const int64_t* __restrict__ bytes;
  const int64_t* __restrict__ off;
  const uint32_t* __restrict__ order;
  int64_t n_traces;
  uint32_t unit_shift;
  uint32_t* counter;
  xm_result* out;
};

__device__ __forceinline__ int64_t rounded_delta(int64_t b, uint32_t sh) {
  const uint64_t mag = b > 0 ? uint64_t(b) : uint64_t(-b);
  const int64_t s = int64_t((mag + ((1ull << sh) - 1)) >> sh);
  return b > 0 ? s : -s;
}

__global__ void __launch_bounds__(256) k_scan_warp(SParams P) {
  const uint32_t lane = threadIdx.x & 31;
  const long long* __restrict__ by = reinterpret_cast<const long long*>(P.bytes);
  for (;;) {
    uint32_t k = 0;
    if (lane == 0) k = atomicAdd(P.counter, 1u);
    k = __shfl_sync(kFull, k, 0);
    if (int64_t(k) >= P.n_traces) break;
    const uint32_t t = P.order[k];
    const int64_t e0 = P.off[t];
    const int64_t n = P.off[t + 1] - e0;
    int64_t run = 0, peak = 0;
    int64_t pidx = 0;
    for (int64_t base = 0; base < n; base += 128) {
      int64_t v[4];
      const int64_t i0 = base + 4 * lane;
#pragma unroll
      for (int r = 0; r < 4; ++r)
        v[r] = (i0 + r < n) ? rounded_delta(__ldcs(by + e0 + i0 + r), P.unit_shift) : 0;
      // in-lane inclusive scan
      v[1] += v[0];
      v[2] += v[1];
      v[3] += v[2];
      // warp exclusive offset of lane totals
      int64_t tot = v[3];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(kFull, tot, o);
        if (lane >= uint32_t(o)) tot += y;
      }
      const int64_t excl = run + tot - v[3];
      // lane max with first index
      int64_t lm = INT64_MIN;
      int li = 0;
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int64_t x = (i0 + r < n) ? excl + v[r] : INT64_MIN;
        if (x > lm) { lm = x; li = r; }
      }
      int64_t wm = lm;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const int64_t y = __shfl_xor_sync(kFull, wm, o);
        wm = y > wm ? y : wm;
      }
      if (wm > peak) {
        const unsigned bm = __ballot_sync(kFull, lm == wm);
        const int src = __ffs(bm) - 1;
        const int r = __shfl_sync(kFull, li, src);
        peak = wm;
        pidx = base + 4 * src + r;
      }
      run = __shfl_sync(kFull, excl + v[3], 31);
    }
    if (lane == 0) {
      xm_result R{};
      R.peak_allocated = uint64_t(peak) << P.unit_shift;
      R.peak_allocated_idx = uint32_t(pidx);
      R.events_done = uint32_t(n);
      R.status = XM_T_OK;
      P.out[t] = R;
    }
    __syncwarp();
  }
}

}  // namespace

namespace xm_internal {

size_t scan_scratch_bytes(const xm_batch*) { return 256; }

int launch_scan(const xm_batch* b, const UnitConfig& u, void* d_scratch, size_t,
                xm_result* d_out, void* stream, int* n_launches) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  SParams P{};
  P.bytes = b->bytes;
  P.off = b->off;
  P.order = b->order;
  P.n_traces = b->n_traces;
  P.unit_shift = u.unit_shift;
  P.counter = static_cast<uint32_t*>(d_scratch);
  P.out = d_out;
  cudaError_t e = cudaMemsetAsync(d_scratch, 0, 256, st);
  if (e != cudaSuccess) return int(e);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t ctas = int64_t(sms) * 8;
  const int64_t need = (b->n_traces + 7) / 8;
  if (need < ctas) ctas = need > 0 ? need : 1;
  k_scan_warp<<<int(ctas), 256, 0, st>>>(P);
  *n_launches += 1;
  return int(cudaGetLastError());
}

}  // namespace xm_internal
