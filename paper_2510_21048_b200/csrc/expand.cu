// expand.cu -- K4: on-device expansion of Monte Carlo traces from templates
// (support kernel; not part of the allocator
// model). Input generation only: it writes the wire-format event arrays that
// k_replay then consumes, so that a paper-scale batch (1M traces, ~5.6e9
// events, "Monte Carlo") never crosses PCIe.
//
// The recipe is the counter-based one of workloads/mc5.py (the host side that
// rebuilds any trace for the oracle): event j of a trace with seed sigma and
// template (fixed, per, tag) of length n is template position src(j), where
//   c(j)    = j <= n-2 && splitmix64(sigma + j + 1) < threshold
//   keep(j) = c(j) && !c(j-1) && id(j) != id(j+1)       (id = tag bits 0-27)
//   src(j)  = keep(j) ? j+1 : keep(j-1) ? j-1 : j
// and bytes = fixed[src] + per[src] * b (sign folded into fixed/per), tag = tag[src].
//
// One warp per trace (grid-stride), lanes over consecutive events: coalesced
// 8 B + 4 B stores; template reads hit L2 (the whole pool is ~23 MB). HBM
// traffic: 12 B written per event.
#include <cuda_runtime.h>

#include "xm_internal.h"

namespace {

struct EParams {
  const int64_t* __restrict__ fixed;
  const int64_t* __restrict__ per;
  const uint32_t* __restrict__ ttag;
  const int64_t* __restrict__ tpl_off;
  int64_t n_tpl;
  const uint32_t* __restrict__ tpl;     // [n] template of stored trace k
  const uint32_t* __restrict__ bsz;     // [n] batch size
  const uint64_t* __restrict__ seed;    // [n]
  const int64_t* __restrict__ off;      // [n+1] stored output offsets
  int64_t n;
  uint64_t threshold;
  int64_t* bytes;
  uint32_t* tag;
  uint32_t* bad;                        // set to 1 if a length disagrees with off
};

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void __launch_bounds__(256) k_expand(EParams P) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t k = w0; k < P.n; k += nw) {
    const uint32_t t = P.tpl[k];
    const int64_t s0 = P.tpl_off[t];
    const int64_t n = P.tpl_off[t + 1] - s0;
    const int64_t d0 = P.off[k];
    if (P.off[k + 1] - d0 != n) {            // inconsistent descriptors: flag, write nothing
      if (lane == 0) atomicExch(P.bad, 1u);
      continue;
    }
    const int64_t b = P.bsz[k];
    const uint64_t sg = P.seed[k];
    const int64_t* fx = P.fixed + s0;
    const int64_t* pr = P.per + s0;
    const uint32_t* tg = P.ttag + s0;
    // One splitmix64 per event: c(j-1), c(j-2) and the neighbours' ids come
    // from the adjacent lanes, or from the previous tile's lanes 30-31.
    bool c31 = false, c30 = false;              // c(base-1), c(base-2)
    uint32_t id31 = 0xFFFFFFFFu;                // id(base-1)
    for (int64_t base = 0; base < n; base += 32) {
      const int64_t j = base + lane;
      const bool v = j < n;
      const uint32_t tj = v ? __ldg(tg + j) : 0u;
      const uint32_t id = tj & 0x0FFFFFFFu;
      const bool cj = v && j + 1 < n && splitmix64(sg + uint64_t(j) + 1) < P.threshold;
      bool cm = __shfl_up_sync(0xFFFFFFFFu, cj, 1);
      bool cmm = __shfl_up_sync(0xFFFFFFFFu, cj, 2);
      uint32_t idm = __shfl_up_sync(0xFFFFFFFFu, id, 1);
      uint32_t idp = __shfl_down_sync(0xFFFFFFFFu, id, 1);
      if (lane == 0) { cm = c31; cmm = c30; idm = id31; }
      if (lane == 1) cmm = c31;
      if (lane == 31 && cj) idp = __ldg(tg + j + 1) & 0x0FFFFFFFu;
      const bool keep_j = cj && !cm && id != idp;             // swap (j, j+1)
      const bool keep_m = cm && !cmm && idm != id;            // swap (j-1, j)
      if (v) {
        const int64_t src = keep_j ? j + 1 : (keep_m ? j - 1 : j);
        P.bytes[d0 + j] = __ldg(fx + src) + __ldg(pr + src) * b;
        P.tag[d0 + j] = src == j ? tj : __ldg(tg + src);
      }
      c31 = __shfl_sync(0xFFFFFFFFu, cj, 31);
      c30 = __shfl_sync(0xFFFFFFFFu, cj, 30);
      id31 = __shfl_sync(0xFFFFFFFFu, id, 31);
    }
  }
}

}  // namespace

using namespace xm_internal;

extern "C" int xm_expand_templates(const xm_templates* tp, const uint32_t* d_tpl,
                                   const uint32_t* d_b, const uint64_t* d_seed,
                                   uint64_t swap_threshold, const int64_t* d_off,
                                   int64_t n_traces, int64_t* d_bytes, uint32_t* d_tag,
                                   uint32_t* d_flag, void* stream) {
  launch_counter() = 0;
  if (!tp || n_traces < 0 || tp->n_tpl < 0) return set_error(XM_EINVAL, "xm_expand_templates: bad arguments");
  if (n_traces == 0) return XM_OK;
  if (!tp->fixed || !tp->per || !tp->tag || !tp->tpl_off || !d_tpl || !d_b || !d_seed || !d_off ||
      !d_bytes || !d_tag || !d_flag)
    return set_error(XM_EINVAL, "xm_expand_templates: null pointer");
  if (!cuda_usable()) return set_error(XM_ECUDA, "no CUDA device");
  EParams P{tp->fixed, tp->per, tp->tag, tp->tpl_off, tp->n_tpl, d_tpl, d_b, d_seed, d_off,
            n_traces, swap_threshold, d_bytes, d_tag, d_flag};
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (n_traces + 7) / 8;                 // 8 warps per CTA
  const int grid = int(want < int64_t(sms) * 8 ? want : int64_t(sms) * 8);
  k_expand<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(P);
  launch_counter() = 1;
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(XM_ECUDA, std::string("k_expand: ") + cudaGetErrorString(e));
  return XM_OK;
}
