/*
 * xmem.h -- C ABI of libxmem.so, the B200-native batched caching-allocator
 * trace replayer (the data-parallel hot path of xMem, arXiv 2510.21048).
 *
 * What is computed. xMem's Simulator (§3.4) replays an
 * ordered alloc/free event sequence through a two-level model of PyTorch's
 * CUDA caching allocator -- (i) 512 B round-up, (ii) segments of 2 MiB /
 * 20 MiB / 2 MiB-rounded size, (iii) best-fit-with-coalescing search, split
 * and merge, (iv) caching of freed blocks, (v) OOM only after reclaiming
 * cached segments fails -- and reports the peak of the segment-sum time
 * series ("The Estimated Peak Memory is then identified as the maximum value
 * in this time series"). libxmem does this for a BATCH of
 * independent traces on one GPU, one warp per trace. The exact rules and
 * every reading of the paper are in DESIGN.md §Readings (Q1-Q16).
 *
 * Beyond the replay (the rows around it): xm_expand_templates
 * (config-5 traces generated on the device), xm_reconstruct /
 * xm_reconstruct_wire (lifecycle reconstruction from profiler instants),
 * xm_orchestrate / xm_orchestrate_wire (the Memory Orchestrator), and
 * xm_metrics_batch (the paper's MRE / PEF / MCP).
 *
 * Conventions for every entry point:
 *   - returns int: XM_OK (0) or a negative XM_E* code; never throws, never
 *     aborts. xm_last_error() returns a thread-local message for the last
 *     failing call on this thread.
 *   - "host" pointers are CPU memory, "device" pointers are CUDA device memory
 *     of the current device; the caller owns every pointer it passes in.
 *   - device entry points are asynchronous on the given cudaStream_t (passed
 *     as void* so this header needs no CUDA include) and never allocate
 *     device memory: the caller provides scratch of xm_scratch_bytes().
 *   - all sizes are in bytes unless a name says otherwise.
 */
#ifndef XMEM_H_
#define XMEM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------------------------------------------------------- errors */
#define XM_OK 0
#define XM_EINVAL (-1)  /* malformed argument or trace (contract violation,   */
                        /* SPEC.md:231,249,258,267)                           */
#define XM_ECUDA (-2)   /* a CUDA runtime call failed                         */
#define XM_ENOMEM (-3)  /* host allocation failed, or scratch too small       */
#define XM_ERANGE (-4)  /* a value exceeds a documented limit                 */

/* ------------------------------------------------------- per-trace status */
#define XM_T_OK 0        /* replayed every event                               */
#define XM_T_OOM 1       /* simulated OOM (PAPER.md:260 (v); Eq. 1):  */
                         /* a result, not an error (SPEC.md:284 D4)            */
#define XM_T_OVERFLOW 2  /* state exceeded its arena (defensive; never occurs  */
                         /* when scratch is sized by xm_scratch_bytes)          */
#define XM_T_INVALID 3   /* not replayed: n_ids = 0 for a trace with events    */
                         /* (a batch contract violation; xm_simulate_raw marks  */
                         /* a trace its loader rejected this way and returns    */
                         /* XM_EINVAL naming it)                                */

/* -------------------------------------------------------------- modes */
#define XM_FULL 0            /* full allocator replay (K2)                     */
#define XM_RECLAIM_ALL 0
#define XM_RECLAIM_LARGEST_FIRST 1

/* xm_config.host_input: how xm_simulate_host moves the events (see there) */
#define XM_HOST_INPUT_AUTO 0      /* direct when the packed array is mapped, else stream */
#define XM_HOST_INPUT_DIRECT 1
#define XM_HOST_INPUT_STREAM 2
#define XM_HOST_INPUT_COPY 3
#define XM_ALLOCATED_ONLY 1  /* only peak_allocated / _idx via the segmented   */
                             /* prefix-scan/max (K1). Exact only with unlimited */
                             /* capacity, which it requires (else XM_EINVAL).   */

/* Wire format limits (checked by xm_load_traces).                          */
#define XM_ID_BITS 28          /* tag bits 0-27: block id                     */
#define XM_STREAM_SHIFT 28     /* tag bits 28-31: stream (0..15)              */
#define XM_MAX_REQUEST (1ull << 40)   /* |bytes| must be < 2^40 (1 TiB)       */
#define XM_UNLIMITED UINT64_MAX

/*
 * Allocator constants (SPEC.md:210-213 SimConfig; defaults are the PyTorch
 * CUDACachingAllocator constants the paper defers to, PAPER.md:257 footnote,
 * confirmed in torch/include/c10/core/AllocatorConfig.h:17-25).
 * xm_config_default() fills them. min_block must be a power of two and every
 * other size a multiple of it.
 */
typedef struct {
  uint64_t min_block;       /* 512      round-up granule, PAPER.md:154,256 (i)  */
  uint64_t small_size;      /* 1 MiB    small-pool threshold (s <= small_size)  */
  uint64_t small_buffer;    /* 2 MiB    small segment             */
  uint64_t large_buffer;    /* 20 MiB   segment for small_size < s < min_large, */
                            /*          PAPER.md:654                            */
  uint64_t min_large_alloc; /* 10 MiB   at or above: round to round_large       */
  uint64_t round_large;     /* 2 MiB                                            */
  uint64_t capacity;        /* device capacity; XM_UNLIMITED (default) = none   */
  uint32_t large_split_strict; /* 1 (default): large split iff remainder >     */
                               /* small_size (torch); 0: >=       */
  uint32_t mode;               /* XM_FULL (default) or XM_ALLOCATED_ONLY        */
  uint32_t smem_per_warp;      /* caps the per-CTA shared-memory heap at        */
                               /* smem_per_warp * warps_per_cta bytes (tests);  */
                               /* 0 = the whole 227 KB                          */
  uint32_t warps_per_cta;      /* 0 = default (14)                              */
  /* Allocator variants (readings Q19, Q20):  */
  uint32_t roundup_power2_divisions; /* torch PYTORCH_CUDA_ALLOC_CONF          */
                               /* roundup_power2_divisions:N, one N for all sizes: */
                               /* a request above min_block*N is rounded up to the */
                               /* next of N equal steps between the powers of two  */
                               /* around it. 0 or 1 = off (default); else a power  */
                               /* of two <= 64 (XM_EINVAL otherwise)               */
  uint32_t reclaim_policy;     /* XM_RECLAIM_ALL (default, torch                  */
                               /* release_cached_blocks, reading Q3) or            */
                               /* XM_RECLAIM_LARGEST_FIRST (SPEC.md:283 D3: fully  */
                               /* free segments largest first, ties lowest address,*/
                               /* only until the request fits)                     */
  uint32_t host_input;         /* XM_HOST_INPUT_* (xm_simulate_host only);        */
                               /* default AUTO                                     */
  uint32_t _pad0;
  /* torch PYTORCH_CUDA_ALLOC_CONF knobs (NEXT-4; readings Q26, Q27;    */
  /* PAPER.md:257 defers the allocator rules to PyTorch):                          */
  uint64_t max_split_size;     /* max_split_size_mb:N = N MiB; XM_UNLIMITED (the   */
                               /* default) = off. When set: a free block of at     */
                               /* least this size is not handed to a smaller       */
                               /* request, nor one of >= s + max_non_split_rounding*/
                               /* to a request s >= it; such requests are never   */
                               /* split; and before releasing every cached segment */
                               /* (reading Q3) torch's release_available_cached_   */
                               /* blocks runs. A multiple of min_block, > 0.       */
  uint64_t max_non_split_rounding; /* max_non_split_rounding_mb (default 20 MiB)   */
  double garbage_collection_threshold; /* in (0, 1): every free-block search that  */
                               /* finds nothing first runs torch's garbage_collect_*/
                               /* cached_blocks when reserved > threshold x the    */
                               /* trace's capacity (finite capacities only; torch  */
                               /* needs set_per_process_memory_fraction): whole    */
                               /* large-pool cached segments at least as old as the*/
                               /* mean age are released, pass after pass. 0 = off  */
                               /* (default); XM_EINVAL outside [0, 1).             */
} xm_config;

/*
 * Per-trace result, 64 bytes, written by xm_simulate_batch at index t of the
 * caller's trace order. Field names map to torch.cuda.memory_stats() keys.
 * "idx" fields are the FIRST event index whose post-event value reaches the
 * maximum (reading Q7); events at or after a failing index are not counted.
 */
typedef struct {
  uint64_t peak_allocated;      /* max sum of round_up(request) of live blocks   */
                                /* (the prefix-scan/max quantity)   */
  uint64_t peak_allocated_blk;  /* max sum of allocated block sizes (SPEC.md:219;*/
                                /* torch allocated_bytes.all.peak), reading Q2   */
  uint64_t peak_reserved;       /* max sum of segment sizes = the paper's Mpeak  */
                                /* (torch reserved_bytes.all.peak) */
  uint64_t final_reserved;      /* reserved after the last processed event       */
  uint32_t peak_allocated_idx;
  uint32_t peak_allocated_blk_idx;
  uint32_t peak_reserved_idx;
  uint32_t n_seg_alloc;         /* segments obtained from the device level       */
  uint32_t n_seg_release;       /* segments returned by reclamation (Q3)         */
  uint32_t max_live_segments;
  uint32_t events_done;         /* = n_events if status==XM_T_OK, else the index */
                                /* of the failing event (reading Q9)             */
  uint16_t status;              /* XM_T_*                                        */
  uint16_t n_free_blocks_end;   /* free blocks after the last event, saturated   */
                                /* at 65535 (== live segments for a closed trace)*/
} xm_result;

/* Batch summary computed by xm_peaks. */
typedef struct {
  uint64_t n_traces;
  uint64_t events_done;         /* sum of events_done                            */
  uint64_t n_oom;               /* traces with status XM_T_OOM                   */
  uint64_t n_overflow;          /* traces with status XM_T_OVERFLOW (must be 0)  */
  uint64_t max_peak_reserved;
  uint64_t max_peak_allocated;
  uint64_t sum_peak_reserved;
  uint64_t n_predicted_oom;     /* Eq. 1:    */
                                /* status==OOM or peak_reserved > capacity_for_eq1*/
} xm_summary;

/* Opaque validated + packed batch of traces (host memory, page-locked when   */
/* CUDA is available).                                                        */
typedef struct xm_traces xm_traces;

/* Device view of a batch, as passed to xm_simulate_batch. All pointers are   */
/* DEVICE memory owned by the caller, laid out exactly as xm_traces_views    */
/* returns them (normally copied there by the caller). Traces are STORED in   */
/* processing order: the kernel starts stored trace 0 first, then 1, ...;     */
/* xm_load_traces stores them longest-first (LPT). Results stay in the        */
/* caller's order through `order`.                                            */
typedef struct {
  const int64_t* bytes;     /* [n_events] signed request bytes: +req alloc, -req free */
  const uint32_t* tag;      /* [n_events] dense id (bits 0-26) | stream << 28; a free */
                            /* carries its block's alloc stream (as xm_load_traces   */
                            /* writes it)                                            */
  const int64_t* off;       /* [n_traces+1] stored trace i = events [off[i], off[i+1])*/
  const uint32_t* n_ids;    /* [n_traces] dense id space of stored trace i (max live) */
  const uint32_t* order;    /* [n_traces] caller index of stored trace i (a          */
                            /* permutation): its result goes to d_out[order[i]]      */
  const uint64_t* capacity; /* [n_traces] per-trace capacity in CALLER order, or NULL*/
                            /* (cfg->capacity for all)                               */
  int64_t n_traces;
  int64_t n_events;
  uint32_t max_ids;         /* max over n_ids                                        */
  uint32_t max_events;      /* max trace length                                      */
  uint64_t* curve;          /* optional DEVICE output [n_events][3] or NULL: the     */
                            /* memory-usage curve ("the full series can */
                            /* optionally be output"): after stored     */
                            /* event e, {allocated (sum of rounded requests),        */
                            /* allocated block bytes, reserved bytes}. Rows of events*/
                            /* a trace did not process (after a simulated OOM) are   */
                            /* left untouched. XM_FULL mode only.                    */
  const uint64_t* packed;   /* optional [n_events] compact events (8 B instead of    */
                            /* 12): bits 0-40 |request bytes|, bit 41 = allocation,   */
                            /* bits 42-45 stream, bits 46-63 dense id (< 2^18). When  */
                            /* non-NULL the kernels read it and ignore bytes / tag.   */
} xm_batch;

#define XM_PACKED_ID_BITS 18

/* Fill *cfg with the defaults above. */
void xm_config_default(xm_config* cfg);

/*
 * Validate and pack a batch of host traces (SPEC.md:156-163 ordered sequence;
 * signed-bytes convention SPEC.md:27).
 *   bytes[n_events], tag[n_events], off[n_traces+1]: HOST, caller-owned, read only.
 *   Array order within a trace is replay order (reading Q6). Block ids may be
 *   any 28-bit values; they are renumbered densely (an id is reused after its
 *   free) so each trace's id space is its maximum number of live blocks.
 *   The packed copy stores the traces longest-first (ties in caller order);
 *   see xm_batch for how stored and caller indices relate.
 * Rejects (XM_EINVAL, *bad_trace = first offending trace): off not monotone or
 *   off[0] != 0; a zero-byte event (reading Q8); |bytes| >=
 *   XM_MAX_REQUEST (XM_ERANGE); an alloc of a live id; a free of a
 *   non-live id or with |bytes| != the alloc's request; a trace
 *   with more than 2^27 live blocks or 2^32-1 events (XM_ERANGE).
 * On success *out is owned by the library until xm_free_traces(*out).
 */
int xm_load_traces(const int64_t* bytes, const uint32_t* tag, const int64_t* off,
                   int64_t n_traces, xm_traces** out, int64_t* bad_trace);

/* Borrow host views of a packed batch (valid until xm_free_traces). Any output */
/* pointer may be NULL. The views fill an xm_batch after copying to device.     */
int xm_traces_views(const xm_traces* tr, const int64_t** bytes, const uint32_t** tag,
                    const int64_t** off, const uint32_t** n_ids, const uint32_t** order,
                    int64_t* n_traces, int64_t* n_events, uint32_t* max_ids,
                    uint32_t* max_events);

void xm_free_traces(xm_traces* tr);

/* The compact event array of a packed batch (xm_batch.packed layout), built by */
/* xm_load_traces when every trace's id space is below 2^XM_PACKED_ID_BITS;     */
/* *packed = NULL otherwise. HOST, valid until xm_free_traces.                 */
int xm_traces_packed(const xm_traces* tr, const uint64_t** packed);

/*
 * Device scratch needed by xm_simulate_batch for this batch and config
 * (work counters + per-warp global-memory state arenas for traces whose state
 * does not fit the shared-memory budget). Host-only computation.
 */
size_t xm_scratch_bytes(const xm_batch* batch, const xm_config* cfg);

/*
 * Replay every trace of the batch on the current device,
 * asynchronously on `stream` (a cudaStream_t; NULL = legacy default stream).
 *   batch: host struct holding DEVICE pointers (see xm_batch).
 *   d_scratch[scratch_bytes]: DEVICE scratch, >= xm_scratch_bytes(); contents
 *     on entry are ignored.
 *   d_out[n_traces]: DEVICE output, one xm_result per trace in caller order.
 * Errors: XM_EINVAL (bad config: min_block not a power of two, sizes not
 * multiples of it, XM_ALLOCATED_ONLY with finite capacity), XM_ENOMEM
 * (scratch too small), XM_ECUDA (launch failure). A simulated OOM is a
 * per-trace status, not an error.
 */
int xm_simulate_batch(const xm_batch* batch, const xm_config* cfg, void* d_scratch,
                      size_t scratch_bytes, xm_result* d_out, void* stream);

/*
 * Per-trace results to host and a batch summary. Synchronises `stream`.
 *   d_res[n]: DEVICE results. h_out[n]: HOST destination or NULL.
 *   capacity_for_eq1: M_d^max of Eq. 1 for n_predicted_oom;
 *     XM_UNLIMITED = only simulated OOMs count.
 */
int xm_peaks(const xm_result* d_res, int64_t n, xm_result* h_out, xm_summary* h_sum,
             uint64_t capacity_for_eq1, void* stream);

/*
 * End-to-end entry point with HOST buffers: moves the batch's events from
 * host memory to the replay, replays it using the DEVICE workspace d_ws
 * (>= xm_host_ws_bytes(); the metadata always goes there), copies the
 * results to h_out[n_traces] (HOST, caller order) and synchronises `stream`.
 *   capacity: HOST [n_traces] per-trace capacities (caller order) or NULL.
 * Event input in XM_FULL mode, cfg->host_input (env XM_HOST_INPUT=direct|
 * stream|copy overrides it, for tooling):
 *   direct  (AUTO's choice when the packed array is page-locked and mapped,
 *           i.e. the batch was loaded with CUDA available): each replaying
 *           warp loads its trace's 8-byte events IN PLACE from the host array
 *           over PCIe, two 32-event tiles ahead of the replay; nothing is
 *           staged in HBM. The host array must stay alive and unchanged until
 *           the call returns (it does: the call is synchronous).
 *   stream  (AUTO's fallback; DIRECT's too when the array is not mapped): chunks of whole traces, in stored order, are
 *           copied into d_ws on a library-owned copy stream while the replay
 *           kernel already runs on `stream`, each trace starting once its
 *           chunk is resident.
 *   copy    (also env XM_NO_STREAM=1; always for XM_ALLOCATED_ONLY): everything is
 *           copied before the launch.
 * All three give identical results.
 */
size_t xm_host_ws_bytes(const xm_traces* tr, const xm_config* cfg);
int xm_simulate_host(const xm_traces* tr, const uint64_t* capacity, const xm_config* cfg,
                     void* d_ws, size_t ws_bytes, xm_result* h_out, void* stream);

/*
 * End-to-end from the caller's RAW host arrays, validated on the device: the
 * xm_load_traces contract (same inputs: bytes[n_events], tag[n_events] = any
 * 28-bit block id | stream << 28, off[n_traces+1]; same checks: zero or
 * >= 2^40 request S:231, alloc of a live id S:249, free of a non-live id or
 * with another size S:258; a free replays on its block's alloc stream) and
 * xm_simulate_host's results, without the host loader: the events go to the
 * device as they are (page-locked: DMA-copied into d_ws in chunks of whole
 * traces, longest-traces-first, on a library-owned copy stream; pageable:
 * copied first), the device loader k_load (keyed by the raw block id: one
 * open block per id in a valid trace) validates every trace and renumbers its
 * ids densely while writing the wire arrays longest first, and k_replay
 * replays them. Page-locked batches of >= 16 traces run OVERLAPPED: the
 * replay takes traces as the loader (on SMs of its own, library-owned stream)
 * finishes them -- for a batch that fills the GPU (>= SMs x 14 traces) the
 * loader has 16 SMs and a second replay launch follows it onto them; for a
 * smaller one the replay has the SMs it needs and the loader all the others
 * (env XM_RAW_OVERLAP=0: loader, then replay). The overlapped mode needs those SMs free of other work: a loader
 * that makes no progress for 4 s makes the call fail with XM_ECUDA instead
 * of hanging. Synchronous; h_out[n_traces] HOST, caller order; the results
 * are identical in every mode.
 *   capacity: HOST [n_traces] or NULL (cfg->capacity).  d_ws: DEVICE,
 *   >= xm_raw_ws_bytes(off, n_traces, cfg) (~52 B per event).
 * Errors: XM_EINVAL / XM_ERANGE with *bad_trace = the first invalid caller
 * trace (its results, and those of every other trace, are still written but
 * meaningless for it); XM_ENOMEM; XM_ECUDA (also: the overlapped loader made
 * no progress). XM_FULL mode only. Traces longer than 2^31-1 events:
 * XM_ERANGE.
 */
size_t xm_raw_ws_bytes(const int64_t* off, int64_t n_traces, const xm_config* cfg);
int xm_simulate_raw(const int64_t* bytes, const uint32_t* tag, const int64_t* off, int64_t n_traces,
                    const uint64_t* capacity, const xm_config* cfg, void* d_ws, size_t ws_bytes,
                    xm_result* h_out, int64_t* bad_trace, void* stream);

/*
 * Config-5 support (kernel K4; input generation, not part of
 * the allocator model): expand Monte Carlo traces from templates ON THE DEVICE
 * so that a paper-scale batch (1M traces) never crosses PCIe.
 * The recipe is the counter-based one of workloads/mc5.py (the host side that
 * rebuilds any single trace for the oracle). For stored trace k with template
 * t = d_tpl[k] of length n = tpl_off[t+1] - tpl_off[t], event j is template
 * position src(j):
 *   c(j)    = j <= n-2 && splitmix64(d_seed[k] + j + 1) < swap_threshold
 *   keep(j) = c(j) && !c(j-1) && id(j) != id(j+1)     (id = tag bits 0-27)
 *   src(j)  = keep(j) ? j+1 : keep(j-1) ? j-1 : j   (CPU-timing jitter)
 * bytes = fixed[src] + per[src] * d_b[k], tag = tag[src] (template block ids are
 * already dense, so the output satisfies xm_batch's id contract).
 *   tp: host struct of DEVICE template arrays (caller-owned):
 *     fixed/per [n_tpl_events] signed per-event bytes (+ alloc, - free);
 *     tag [n_tpl_events]; tpl_off [n_tpl+1].
 *   d_tpl, d_b, d_seed [n_traces] (DEVICE, stored order); d_off [n_traces+1]
 *     (DEVICE) output offsets, which must equal the template lengths; a trace
 *     whose length disagrees is skipped and *d_flag (DEVICE u32) is set to 1.
 *   d_bytes [off[n]], d_tag [off[n]]: DEVICE outputs (caller-owned).
 * Asynchronous on `stream`; one kernel launch. Errors: XM_EINVAL (null or
 * negative arguments), XM_ECUDA.
 */
typedef struct {
  const int64_t* fixed;
  const int64_t* per;
  const uint32_t* tag;
  const int64_t* tpl_off;
  int64_t n_tpl;
} xm_templates;
int xm_expand_templates(const xm_templates* tp, const uint32_t* d_tpl, const uint32_t* d_b,
                        const uint64_t* d_seed, uint64_t swap_threshold, const int64_t* d_off,
                        int64_t n_traces, int64_t* d_bytes, uint32_t* d_tag, uint32_t* d_flag,
                        void* stream);

/*
 * Batched evaluation metrics: the paper's MRE, PEF
 * and MCP over N runs (SPEC.md:339-417 metrics module),
 * given the estimates (e.g. xm_result.peak_reserved and Eq. 1's ÔOM from the
 * replay) and user-supplied measurements of real runs (Table 1 notation).
 * One record per run, DEVICE memory, 40 bytes:
 */
#define XM_ROUND2_NOT_RUN 2
typedef struct {
  uint64_t m_peak_est;    /* M̂peak_jde, the estimate                              */
  uint64_t m_peak_meas1;  /* Mpeak_jd1, measured in round 1 (used iff OOM_jd1 = 0)  */
  uint64_t m_peak_meas2;  /* Mpeak_jd2, measured in round 2 (used iff OOM_jde2 = 0) */
  uint64_t m_max;         /* M_d^max                                               */
  uint8_t oom_pred;       /* ÔOM_jde (Eq. 1: M̂peak > M_d^max)          */
  uint8_t oom1;           /* OOM_jd1 (round 1 with full device memory)             */
  uint8_t oom2;           /* OOM_jde2: 0, 1, or XM_ROUND2_NOT_RUN (round 2 runs     */
                          /* only when C1 = 1 and OOM_jd1 = 0)              */
  uint8_t _pad[5];
} xm_run;

typedef struct {
  uint64_t n;             /* N runs                                                */
  uint64_t n_mre;         /* runs with OOM_jd1 = 0 (the MRE selection)       */
  double mre;             /* median of error_jde2 if OOM_jde2 = 0 else error_jde1; */
                          /* even count: mean of the central pair; NaN if none     */
  double pef1, pef2;      /* (N - sum C_1) / N and (N - sum C_2) / N                */
  double mcp;             /* mean of M_save (bytes, signed)                         */
  int64_t sum_save;       /* exact sum of M_save                                    */
  uint64_t sum_c1, sum_c2;
} xm_metrics;

/* Device scratch needed for n runs (host-only computation). */
size_t xm_metrics_scratch_bytes(int64_t n_runs);
/*
 * Evaluate the metrics of d_runs[n] (DEVICE) into *h_out (HOST); synchronises
 * `stream`. Errors: XM_EINVAL for n == 0 (SPEC.md:386 no-data), null
 * pointers, or an invalid record (round-2 fields where P:385's gating excludes
 * round 2; a zero measured peak that the MRE would divide by);
 * XM_ENOMEM (scratch too small); XM_ECUDA. Floating point: fp64, each error
 * computed as double(|est - meas|) / double(meas).
 */
int xm_metrics_batch(const xm_run* d_runs, int64_t n, void* d_scratch, size_t scratch_bytes,
                     xm_metrics* h_out, void* stream);

/*
 * Lifecycle reconstruction (the Analyzer step two
 * before the Simulator): pair the profiler's memory instants (address, signed
 * bytes, in time order) into blocks -- "pairing allocation and deallocation
 * events based on address tracking and timing ... correctly handling address
 * reuse. Blocks lacking a deallocation event are considered persistent"
 * (§3.2). Rules: a free closes the most
 * recently opened still-open block at its address (LIFO, D1); none open ->
 * orphan (tallied, dropped); |bytes| != the block's size -> mismatch
 * (tallied; the block is closed with its own size).
 */
typedef struct {
  const uint64_t* addr;     /* [n_events] DEVICE: the instant's address                   */
  const int64_t* bytes;     /* [n_events] DEVICE: +size allocation, -size deallocation;    */
                            /* 0 or |bytes| >= XM_MAX_REQUEST is invalid (counted in     */
                            /* n_invalid, otherwise ignored: never reaches the replay)    */
  const uint8_t* stream;    /* [n_events] DEVICE stream (0..15) or NULL (all 0)            */
  const int64_t* off;       /* [n_traces+1] DEVICE: trace t = instants [off[t], off[t+1])  */
  int64_t n_traces, n_events;
  uint32_t max_events;      /* longest trace (host value; sizes the scratch)               */
} xm_instants;

typedef struct {            /* per trace, 64 bytes                                         */
  uint64_t n_blocks;        /* allocations                                                 */
  uint64_t n_orphan;        /* frees with no open block at their address                   */
  uint64_t n_mismatch;      /* matched frees whose |bytes| differs from the block's size   */
  uint64_t n_persistent;    /* blocks never closed                                         */
  uint64_t n_kept;          /* allocations + matched frees = replay events of the trace    */
  uint64_t n_invalid;       /* zero-byte or out-of-range (>= XM_MAX_REQUEST) instants       */
  uint32_t max_open;        /* most blocks open at once                                    */
  uint32_t n_ids;           /* dense id space of the wire trace (<= max_open + 31); the    */
                            /* replay needs <= 2^27 (xm_batch tag bits 0-26)               */
  uint64_t n_reopened;      /* allocations at an address whose block is still open (a     */
                            /* lost free in a profile; an invalid trace for the device     */
                            /* loader of xm_simulate_raw)                     */
} xm_lifecycle;

size_t xm_reconstruct_scratch_bytes(const xm_instants* in);
/*
 * Reconstruct every trace (asynchronous on `stream`, one launch). Outputs,
 * DEVICE, caller-owned:
 *   d_partner[n_events] int32, trace-local index: for an allocation the free
 *     that closes it (-1 = persistent), for a free the allocation it closes
 *     (-1 = orphan); d_mismatch[n_events] 1 on a mismatched free;
 *   d_rec[n_traces] per-trace tallies.
 * d_scratch (>= xm_reconstruct_scratch_bytes) also keeps the replay trace each
 * reconstruction defines, for xm_reconstruct_wire. Errors: XM_EINVAL (null /
 * negative), XM_ERANGE (a trace of >= 2^31 instants), XM_ENOMEM (scratch),
 * XM_ECUDA.
 */
int xm_reconstruct(const xm_instants* in, void* d_scratch, size_t scratch_bytes,
                   int32_t* d_partner, uint8_t* d_mismatch, xm_lifecycle* d_rec, void* stream);
/*
 * After xm_reconstruct (same `in`, same scratch, d_rec its output): write the
 * replay input the reconstruction defines -- per trace, its allocations and
 * matched frees in order, a free carrying -(its block's size) and its block's
 * stream, block ids dense (reused only after their block closes) -- as an
 * xm_batch's arrays, traces STORED in the order d_order[n_traces] (stored ->
 * caller index, a permutation; NULL = identity; e.g. longest first by
 * d_rec[].n_kept, as xm_load_traces stores). Outputs, DEVICE, caller-owned:
 * d_wire_bytes / d_wire_tag [sum n_kept], d_wire_off [n_traces+1],
 * d_wire_nids [n_traces] (stored order). Two launches, asynchronous.
 */
int xm_reconstruct_wire(const xm_instants* in, const void* d_scratch, size_t scratch_bytes,
                        const xm_lifecycle* d_rec, const uint32_t* d_order,
                        int64_t* d_wire_bytes, uint32_t* d_wire_tag, int64_t* d_wire_off,
                        uint32_t* d_wire_nids, void* stream);

/*
 * Reconstruction -> orchestrator input: the blocks each reconstruction defines,
 * as the Analyzer hands them on ("size, initial CPU-based
 * allocation and deallocation timestamps"), in allocation order. DEVICE in:
 * the instants `in` (plus their times d_ts[n_events], microseconds), d_partner
 * from xm_reconstruct, d_boff[n_traces+1] = exclusive prefix sum of the
 * reconstruction's n_blocks (trace t's blocks start at d_boff[t]). DEVICE out
 * [sum n_blocks]: allocation time, free time (-1 = persistent), size (the
 * allocation's bytes), stream. One launch, asynchronous. Orphan frees are
 * dropped; a mismatched free still closes its block (reading Q22).
 */
int xm_blocks_from_instants(const xm_instants* in, const int64_t* d_ts, const int32_t* d_partner,
                            const int64_t* d_boff, int64_t* d_alloc_ts, int64_t* d_free_ts,
                            int64_t* d_size, uint8_t* d_stream, void* stream);

/*
 * Memory Orchestrator (§3.3;
 * SPEC.md:151-203), the step directly before the Simulator. Input: the
 * Analyzer's blocks of each trace in allocation order (CPU timestamps in
 * microseconds) and the training loop's annotation windows per
 * iteration. Output: each block's class and, for the analysis
 * iteration (SPEC D1: the second, index 1), the re-timed sequence ordered by
 * (ts, Free before Alloc, block) (D4). Rules (Q22-Q25):
 * classes by priority Parameter (no free, allocated before the first
 * iteration), OptimizerState (allocated in an optimizer.step window with a
 * Parameter's size; two per Parameter of that size, in allocation order,
 * SPEC D3), Gradient (allocated in a backward window, not freed before its
 * end), BatchData (allocated in a data window), Activation (forward or
 * backward window), Other. Re-timing for W = [Ws, We) of the analysis
 * iteration: blocks allocated at/after We or dead at Ws are left out; a
 * BatchData free is clamped to its iteration's end; carried-over blocks are
 * allocated at Ws, Parameter/OptimizerState never freed, a carried-over
 * Gradient freed at the end of W's zero_grad window (We if none, SPEC D5);
 * a Gradient allocated in W is freed at We; other frees are kept if before
 * We, else at We; a free never precedes or ties its allocation (F' >= A'+1).
 */
#define XM_O_OK 0
#define XM_O_FEW_ITERATIONS 1   /* fewer iterations than analysis_iter + 1      */
#define XM_O_TS_RANGE 2         /* a re-timed timestamp >= 2^32 us after Ws, or */
                                /* a block size outside (0, XM_MAX_REQUEST)    */
typedef struct {
  const int64_t* alloc_ts;  /* [n_blocks] DEVICE, allocation time (us)                  */
  const int64_t* free_ts;   /* [n_blocks] DEVICE, deallocation time, -1 = none observed */
  const int64_t* size;      /* [n_blocks] DEVICE, bytes (> 0)                           */
  const uint8_t* stream;    /* [n_blocks] DEVICE stream (0..15) or NULL                 */
  const int64_t* boff;      /* [n_traces+1] DEVICE, blocks of trace t, allocation order */
  const int64_t* win;       /* [n_iters][6][2] DEVICE windows [start, end] per          */
                            /* iteration: iteration, data, forward, backward,          */
                            /* zero_grad (-1,-1 = none), optimizer.step                */
  const int64_t* woff;      /* [n_traces+1] DEVICE, iterations of trace t              */
  int64_t n_traces, n_blocks;
  uint32_t max_blocks;      /* largest trace (host value; sizes the scratch), <= 2^23  */
                            /* (XM_ERANGE otherwise)                                   */
} xm_profiles;

typedef struct {            /* per trace, 56 bytes                                      */
  int64_t ws, we;           /* the analysis window                                      */
  uint64_t n_events;        /* length of the re-timed sequence                          */
  uint32_t n_ids;           /* dense id space of its wire form                          */
  uint32_t status;          /* XM_O_*                                                   */
  uint32_t n_class[6];      /* blocks per class (Parameter, OptimizerState, Gradient,   */
                            /* BatchData, Activation, Other)                            */
} xm_orchestrated;

size_t xm_orchestrate_scratch_bytes(const xm_profiles* in);
/*
 * Orchestrate every trace (asynchronous, one launch). Outputs, DEVICE,
 * caller-owned: d_class[n_blocks] (0-5 as above; undefined for traces whose
 * status is not XM_O_OK); d_seq[2 n_blocks]: trace t's sorted sequence at
 * d_seq[2 boff[t] ...], n_events keys each (ts - ws) << 32 | kind << 31 |
 * block (kind 0 = Free, 1 = Alloc; block = index in the trace's allocation
 * order); d_rec[n_traces]. The scratch keeps the staged wire form for
 * xm_orchestrate_wire. Errors: XM_EINVAL, XM_ERANGE, XM_ENOMEM, XM_ECUDA.
 */
int xm_orchestrate(const xm_profiles* in, uint32_t analysis_iter, void* d_scratch,
                   size_t scratch_bytes, uint8_t* d_class, uint64_t* d_seq,
                   xm_orchestrated* d_rec, void* stream);
/*
 * After xm_orchestrate (same in / scratch): the re-timed sequences as an
 * xm_batch's arrays (allocation +size, free -size, dense ids, the block's
 * stream), traces stored in d_order (stored -> caller; NULL = identity).
 * DEVICE outputs sized sum n_events / n_traces+1 / n_traces. Two launches.
 */
int xm_orchestrate_wire(const xm_profiles* in, const void* d_scratch, size_t scratch_bytes,
                        const xm_orchestrated* d_rec, const uint32_t* d_order,
                        int64_t* d_wire_bytes, uint32_t* d_wire_tag, int64_t* d_wire_off,
                        uint32_t* d_wire_nids, void* stream);

/* Number of device kernel launches the last xm_simulate_batch on this thread */
/* issued (for the bench's gpu_launches claim).                               */
int xm_last_launch_count(void);

/* Thread-local message of the last failing call ("" if none). */
const char* xm_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* XMEM_H_ */
