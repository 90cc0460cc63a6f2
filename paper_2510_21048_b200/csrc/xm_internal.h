// xm_internal.h -- declarations shared by the product's translation units
// (loader.cpp, capi.cu, replay.cu, scan.cu). Not part of the public ABI.
#pragma once
#include <cstddef>
#include <cstdint>
#include <string>

#include "xmem.h"

namespace xm_internal {

int set_error(int code, const std::string& msg);
void clear_error();
bool cuda_usable();

struct xm_traces_info {
  const int64_t* bytes;
  const uint32_t* tag;
  const int64_t* off;
  const uint32_t* n_ids;
  const uint32_t* order;
  int64_t n_traces, n_events;
  uint32_t max_ids, max_events;
  const uint32_t* chunk_end;   // pinned [n_chunks]: stored-trace end of each upload chunk
  int n_chunks;
  const uint64_t* packed;      // compact events (xm_batch.packed) or null
};
// upload chunks of the streamed host entry point (xm_simulate_host)
constexpr int kUploadChunks = 24;
const xm_traces_info traces_info(const xm_traces* tr);

// Allocator constants in units of min_block.
struct UnitConfig {
  uint32_t unit_shift;   // log2(min_block)
  uint32_t small_u;      // small_size / min_block
  uint32_t sbuf_u;       // small_buffer / min_block
  uint32_t lbuf_u;       // large_buffer / min_block
  uint32_t minlarge_u;   // min_large_alloc / min_block
  uint32_t rlarge_u;     // round_large / min_block
  uint32_t strict;       // large split iff rem > small (1) or >= (0)
  uint32_t div_shift;    // log2(roundup_power2_divisions), 0 = off (NEXT-4 variant)
  uint32_t reclaim_d3;   // 1: SPEC D3 largest-first reclamation (NEXT-4 variant)
  uint32_t msplit_u;     // torch max_split_size / min_block; 0xFFFFFFFF = off (Q26)
  uint32_t nsr_u;        // torch max_non_split_rounding / min_block (Q26)
  double gc_threshold;   // torch garbage_collection_threshold; 0 = off (Q27)
};

// Launch geometry + scratch layout of the replay kernel for one batch.
struct ReplayPlan {
  int warps_per_cta;
  int ctas;
  uint32_t heap_pages;      // shared-memory heap pages (512 B) per CTA
  size_t arena_per_warp;    // bytes per global-memory arena slot (overflow path)
  uint32_t n_arena;         // arena slots in scratch
  uint32_t arena_ids, arena_free;
  size_t scratch_bytes;     // header + arenas
};

int make_unit_config(const xm_config* cfg, UnitConfig* u);
int& launch_counter();
ReplayPlan plan_replay(const xm_batch* b, const xm_config* cfg);

// Kernel launchers (replay.cu / scan.cu). Return cudaError_t as int.
int launch_replay(const xm_batch* b, const xm_config* cfg, const UnitConfig& u,
                  const ReplayPlan& plan, void* d_scratch, xm_result* d_out, void* stream,
                  int* n_launches, const uint32_t* ready = nullptr,
                  const uint32_t* loaded = nullptr, int ctas = 0, bool reset = true);
int launch_scan(const xm_batch* b, const UnitConfig& u, void* d_scratch, size_t scratch_bytes,
                xm_result* d_out, void* stream, int* n_launches);
size_t scan_scratch_bytes(const xm_batch* b);

// Force-load a kernel module before kernels that wait on each other run
// concurrently (CUDA lazy loading); return cudaError_t as int.
int preload_replay();
int preload_loader();

// Device loader of xm_simulate_raw (lifecycle.cu): K5 keyed by raw block ids.
size_t loader_scratch_bytes(int64_t T, int64_t E, uint32_t max_events);
int launch_loader(const int64_t* d_bytes, const uint32_t* d_tag, const int64_t* d_off, int64_t T,
                  int64_t E, uint32_t max_events, void* d_scratch, xm_lifecycle* d_rec,
                  const uint32_t* d_order, int64_t* w_bytes, uint32_t* w_tag, int64_t* w_off,
                  uint32_t* w_nids, void* stream, int* n_launches,
                  const uint32_t* chunk_first = nullptr, const uint32_t* chunk_flag = nullptr,
                  int n_chunks = 0, const uint32_t* d_pos = nullptr, uint32_t* loaded = nullptr,
                  int loader_sms = 0, uint32_t* stall = nullptr);

}  // namespace xm_internal
