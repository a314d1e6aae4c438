/* sbs_b200 — B200-native (sm_100a) hot path of the Staggered Batch Scheduling
 * reference simulator (arXiv 2512.16134, "sbsim").
 *
 * C-ABI drop-in boundary.  Plain pointers and sizes only; no torch / C++ types.
 * Each entry point names the reference interface it replaces
 * (paths relative to the reference tree, /root/reference/proj).
 *
 * Return codes mirror the reference's error classes:
 *   SBS_OK             0
 *   SBS_ERR_CONFIG     1  ≙ sbsim::ConfigError          (core.h:34-37)
 *   SBS_ERR_INVARIANT  3  ≙ std::logic_error invariant  (simclock.cpp:25-28,
 *                          engine_model.cpp:129-130, simulation.cpp:516-533)
 *   SBS_ERR_OVERFLOW   4  a fixed-capacity device arena overflowed (the host
 *                          wrappers retry with doubled capacity; never silent)
 *   SBS_ERR_CUDA       5  CUDA runtime error / no device / extension missing
 *   SBS_ERR_ENVELOPE   6  a replica left the GPU path's integer envelope: a
 *                          decode unit with B >= 2^15 or K >= 2^32, or more
 *                          than 2^32 - 2^16 scheduled events (the device seq
 *                          counter is 32-bit; simclock.h:63 uses 64)
 * sbs_last_error() returns a thread-local message for the last failure.
 */
#ifndef SBS_B200_H_
#define SBS_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SBS_OK 0
#define SBS_ERR_CONFIG 1
#define SBS_ERR_INVARIANT 3
#define SBS_ERR_OVERFLOW 4
#define SBS_ERR_CUDA 5
#define SBS_ERR_ENVELOPE 6

/* SchedulerPolicy (config.h:19-24) */
#define SBS_POLICY_SBS 0
#define SBS_POLICY_IMMEDIATE 1
#define SBS_POLICY_ROUND_ROBIN 2
#define SBS_POLICY_LEAST_OUTSTANDING 3
/* DecodePolicy (config.h:26) */
#define SBS_DECODE_IQR 0
#define SBS_DECODE_RANDOM 1
#define SBS_DECODE_ROUND_ROBIN 2
/* AllocMode (prefill_alloc.h:15) */
#define SBS_ALLOC_BASIC 0
#define SBS_ALLOC_CACHE_AWARE 1
/* ArrivalProcess (workload.h:16-20) / LengthDist (workload.h:22) */
#define SBS_ARRIVAL_POISSON 0
#define SBS_ARRIVAL_UNIFORM 1
#define SBS_ARRIVAL_UNIFORM_JITTER 2
#define SBS_LEN_CONSTANT 0
#define SBS_LEN_UNIFORM 1
#define SBS_LEN_LOGNORMAL 2

/* ClusterConfig (core.h:236-260) incl. EngineCoefficients (core.h:222-228). */
typedef struct sbs_cluster {
  int32_t n_instances_prefill;
  int32_t n_instances_decode;
  int32_t dp_degree;
  int32_t dp_degree_decode; /* 0 = same as dp_degree */
  int64_t c_chunk;
  double t_default_s;
  int64_t w_size;
  double l_net_s;
  int32_t n_limit;
  int32_t decode_max_batch_per_dp; /* 0 = unbounded */
  double iqr_k;
  double watchdog_multiplier;
  double prefill_base_s;
  double prefill_per_token_s;
  double decode_base_s;
  double decode_per_request_s;
  double decode_per_kv_token_s;
  int64_t decode_tokens_per_step;
  /* CacheSettings (core.h:230-234): the per-DP PrefixCache stub (core.h:87-123) */
  int32_t cache_enabled;
  int32_t cache_n_probes;
  int64_t cache_budget_tokens;
  const int64_t* cache_probe_lens; /* cache_n_probes entries, each >= 1 */
} sbs_cluster;

/* LengthSpec (workload.h:28-35) */
typedef struct sbs_length_spec {
  int32_t dist;
  int32_t _pad;
  int64_t value, min, max;
  double mu, sigma;
} sbs_length_spec;

/* WorkloadSpec (workload.h:37-50) */
typedef struct sbs_workload {
  int32_t process;
  int32_t initial_burst;
  double rate_qps;
  double duration_s;
  sbs_length_spec prompt;
  sbs_length_spec output;
  double shared_prefix_fraction;
  int32_t prefix_pool;
  int32_t _pad;
  int64_t prefix_len;
} sbs_workload;

/* FaultPlan entries (config.h:35-58) */
typedef struct sbs_drop_fault { int32_t instance; int32_t _pad; double from_s, until_s; } sbs_drop_fault;
typedef struct sbs_dead_fault { int32_t instance; int32_t _pad; double time_s; } sbs_dead_fault;
typedef struct sbs_topology_fault { int32_t instance; int32_t healthy; double time_s; } sbs_topology_fault;

/* ExperimentConfig (config.h:66-75).  One replica = one experiment. */
typedef struct sbs_experiment {
  sbs_cluster cluster;
  sbs_workload workload;
  int32_t policy;
  int32_t prefill_mode;
  int32_t decode_policy;
  int32_t n_drops;
  uint64_t seed;
  double warmup_fraction;
  const sbs_drop_fault* drops;
  const sbs_dead_fault* deads;
  const sbs_topology_fault* topology;
  int32_t n_deads;
  int32_t n_topology;
} sbs_experiment;

/* A request trace in SoA form: the output of generate_workload
 * (workload.cpp:67-142), ids = positions.  16 B per request, plus 8 B when
 * requests carry shared prefixes: Request::prefix_tokens (core.h:57-58) is
 * the first prefix_size tokens of pool prefix_pool_id (workload.cpp:30-37,
 * 129-138); -1 / 0 = no prefix.  Both NULL: no request has a prefix. */
typedef struct sbs_trace {
  const int64_t* arrival_ns;
  const int32_t* prompt_len;
  const int32_t* output_len;
  int64_t n;
  uint64_t digest; /* workload_digest (workload.cpp:144-162) */
  const int32_t* prefix_pool_id;
  const int32_t* prefix_size;
} sbs_trace;

/* Aggregates (metrics.h:67-102), same field meaning, plus the sweep extras. */
typedef struct sbs_aggregates {
  uint64_t generated, completed, throttled, in_flight, window_requests;
  double ttft_mean_s, ttft_p50_s, ttft_p95_s;
  double scheduler_wait_mean_s, device_wait_mean_s, total_wait_mean_s;
  uint64_t passes;
  double chunk_util_mean;
  uint64_t decode_steps, output_tokens;
  double output_tokens_per_s, kv_mean_time_avg, kv_sigma_time_avg;
  double completed_per_s;
  uint64_t watchdog_fires, dropped_end_forwards, rejected_samples, deferrals,
      flow_control_events, mask_events, fallback_events;
  double warmup_cutoff_s, duration_s;
  /* extras (not in the reference) */
  uint64_t alloc_calls;     /* allocate_batch invocations (cluster-windows) */
  uint64_t decode_selects;  /* decode placements */
  uint64_t events;          /* live events processed */
  double tpot_mean_s;       /* mean over completed requests with output_len > 1 of
                               (completion_ns - first_token_ns) / (output_len - 1),
                               one IEEE FP64 division per request, then / 1e9 */
  uint64_t tpot_count;
  int64_t ttft_sum_ns, sched_sum_ns, device_sum_ns; /* exact int64 sums */
  int32_t error;            /* per-replica SBS_* code */
  int32_t _pad;
} sbs_aggregates;

#define SBS_HIST_BINS 64
/* TTFT / TPOT log2-spaced histograms (bin b counts values in [2^b, 2^(b+1)) ns,
 * bin 0 also holds 0) summed over replicas; NCCL-reducible as int64.
 * ttft: first_token - arrival of the window requests (completed, arrival >=
 * warmup: metrics.cpp:122-136); tpot: trunc of the per-request TPOT in ns. */
typedef struct sbs_histograms {
  int64_t ttft[SBS_HIST_BINS];
  int64_t tpot[SBS_HIST_BINS];
} sbs_histograms;

/* ----------------------------------------------------------------------- */
/* Trace generation (host, multi-threaded).  Replaces generate_workload +   */
/* workload_digest (workload.cpp:67-162); bit-identical on the same glibc.  */
/* With arrays NULL only *n_out (and *digest) are produced; the prefix     */
/* arrays may be NULL on their own (then only lengths are written).         */
int sbs_generate_workload(const sbs_workload* spec, uint64_t seed,
                          int64_t* arrival_ns, int32_t* prompt_len,
                          int32_t* output_len, int32_t* prefix_pool_id,
                          int32_t* prefix_size, int64_t cap, int64_t* n_out,
                          uint64_t* digest);

/* ----------------------------------------------------------------------- */
/* Trace generation ON THE DEVICE: generate_workload + workload_digest      */
/* (workload.cpp:67-162), one warp per trace, bit-identical to the host     */
/* run on glibc 2.39 x86-64 (its FMA-path log/cos/exp are restated in       */
/* csrc/glibc_libm.cuh).  Output arrays and `stats` are DEVICE pointers;     */
/* a trace longer than `cap` sets stats->error = SBS_ERR_OVERFLOW (n = 0).   */
typedef struct sbs_gen_stats {
  int64_t n;            /* requests generated */
  uint64_t digest;      /* workload_digest (when requested, else 0) */
  int32_t max_prompt, max_output;
  int32_t n_pools;      /* 1 + largest prefix pool id used (0: none) */
  int32_t max_psize;    /* largest prefix size */
  int32_t error;        /* SBS_OK / SBS_ERR_OVERFLOW / SBS_ERR_CONFIG (length > 2^30) */
  int32_t _pad;
  int64_t draws;        /* mt19937_64 outputs consumed */
} sbs_gen_stats;
typedef struct sbs_gen_job {
  sbs_workload spec;
  uint64_t seed;
  int64_t cap;
  int64_t* arrival_ns;
  int32_t* prompt_len;
  int32_t* output_len;
  int32_t* prefix_pool_id; /* both NULL unless spec.shared_prefix_fraction > 0 */
  int32_t* prefix_size;
  sbs_gen_stats* stats;
} sbs_gen_job;
/* jobs: HOST array (copied); seeds: DEVICE array overriding jobs[i].seed, or
 * NULL.  Enqueued on `stream`. */
int sbs_generate_workload_device(const sbs_gen_job* jobs, int32_t n_jobs, const uint64_t* seeds,
                                 int32_t want_digest, void* stream);
/* An upper bound on the requests generate_workload can produce for `spec`
 * with probability 1 - 1e-12 (Poisson: initial_burst + mean + 8 sd + 64),
 * exact for the uniform processes. */
int64_t sbs_workload_capacity(const sbs_workload* spec);

/* ----------------------------------------------------------------------- */
/* Persistent replica simulator (the DES hot path).                         */
/* Replaces run_experiment (simulation.h:33 / simulation.cpp:537-541) for   */
/* many independent replicas at once: one warp per replica.                 */
typedef struct sbs_sim sbs_sim;

#define SBS_FLAG_PER_REQUEST 1u /* keep per-request timestamps (parity mode) */
#define SBS_FLAG_LOGS 2u        /* keep run records (MetricsCollector, metrics.h:107-152) */
#define SBS_FLAG_KV_LOADS 4u    /* with LOGS: also the per-unit KV loads of every decode step
                                   (record 6), what MetricsCollector::record_kv receives */

/* traces: host arrays (uploaded here).  trace_of_point[i] selects the trace of
 * point i (NULL: point i uses trace i).  Points sharing a trace share HBM. */
int sbs_sim_create(const sbs_experiment* points, int32_t n_points,
                   const sbs_trace* traces, int32_t n_traces,
                   const int32_t* trace_of_point, uint32_t flags,
                   int32_t device, sbs_sim** out);
/* Traces generated ON THE DEVICE (sbs_generate_workload_device): trace t is
 * generate_workload(points[i].workload, points[i].seed) of the first point i
 * with trace_of_point[i] == t (all points sharing a trace must share both;
 * trace_of_point NULL: one trace per point).  Arenas are sized from the
 * workload spec (sbs_workload_capacity, length bounds), so any seed fits.
 * Slot 0 is generated before this returns.  Replaces the reference's
 * generate_workload call inside Runner::run (simulation.cpp:141). */
int sbs_sim_create_generated(const sbs_experiment* points, int32_t n_points,
                             const int32_t* trace_of_point, int32_t n_traces, uint32_t flags,
                             int32_t device, sbs_sim** out);
/* Regenerate every trace of a generated simulator into trace slot `slot` on
 * `stream` with new seeds (HOST array, one per trace; NULL = the current
 * seeds): 8 B per trace host->device, the rest is device work.  The next
 * sbs_sim_launch_slot(slot) on the same stream reads them. */
int sbs_sim_generate_slot(sbs_sim* sim, const uint64_t* seeds, int32_t slot, int32_t want_digest,
                          void* stream);
/* Generation stats of a trace in a slot (synchronises the device). */
int sbs_sim_trace_stats(sbs_sim* sim, int32_t trace, int32_t slot, sbs_gen_stats* out);
/* Copy a trace of a slot back to the host (synchronises); *n_out = length. */
int sbs_sim_trace_arrays(sbs_sim* sim, int32_t trace, int32_t slot, int64_t* arrival_ns,
                         int32_t* prompt_len, int32_t* output_len, int32_t* prefix_pool_id,
                         int32_t* prefix_size, int64_t cap, int64_t* n_out);
/* Re-upload host traces on `stream` (16 B/request).  Each must fit what the
 * simulator was created with — same length, outputs no longer than the
 * create-time maximum (decode completion ring), prefix pools/sizes within the
 * create-time ones — else SBS_ERR_CONFIG (nothing is uploaded).  When every
 * array is pinned host memory the device gathers them in one launch (a copy
 * kernel over the mapped host pages); otherwise one copy per array. */
int sbs_sim_upload_traces(sbs_sim* sim, const sbs_trace* traces, void* stream);
/* Enqueue one full simulation of every point (DES kernel + finalize kernel). */
int sbs_sim_launch(sbs_sim* sim, void* stream);
/* Double-buffered traces: with 2 slots the next step's traces can be uploaded
 * (sbs_sim_upload_traces_slot, e.g. on a copy stream) while a launch reads the
 * other slot (sbs_sim_launch_slot).  The caller orders the streams: a slot is
 * not re-uploaded while a launch that reads it is in flight.  Slot 0 is the
 * one sbs_sim_create / sbs_sim_upload_traces / sbs_sim_launch use. */
int sbs_sim_enable_trace_slots(sbs_sim* sim, int32_t n_slots);
int sbs_sim_upload_traces_slot(sbs_sim* sim, const sbs_trace* traces, int32_t slot, void* stream);
int sbs_sim_launch_slot(sbs_sim* sim, int32_t slot, void* stream);
/* Synchronise `stream`, copy results back, finish the aggregate arithmetic. */
int sbs_sim_results(sbs_sim* sim, sbs_aggregates* out, sbs_histograms* hist,
                    void* stream);
/* Parity mode: per-request timestamps of one point (ns, -1 when unset) and
 * status (RequestStatus, core.h:41-48). */
int sbs_sim_requests(sbs_sim* sim, int32_t point, int64_t* dispatch_ns,
                     int64_t* prefill_start_ns, int64_t* first_token_ns,
                     int64_t* completion_ns, int8_t* status);
/* SBS_FLAG_LOGS: the point's run records as int64 words: header
 * kind | (payload words << 8) then payload; kinds 1 dispatch (time, instance),
 * 2 control (time, i_opt, t_fwd_bar, n_active), 3 pass (time, instance,
 * assigned[dp_degree]), 4 step (time, generated), 5 kv band (time, mean bits,
 * sigma bits, min, max), 6 kv loads (time, K[unit] of the healthy live
 * decode units; SBS_FLAG_KV_LOADS only).  These are the records behind passes.csv,
 * kvband.csv, control.csv and the dispatch log (metrics.cpp:194-273).
 * With words NULL only *n_out is set. */
int sbs_sim_log(sbs_sim* sim, int32_t point, int64_t* words, int64_t cap, int64_t* n_out);
/* Development hook: SBS_PROF_COUNTERS per-region clock64 cycle / spin
 * counters summed over replicas (non-zero only in an SBS_PROF=1 build). */
#define SBS_PROF_COUNTERS 24
int sbs_sim_profile_counters(const sbs_sim* sim, int64_t* out);
/* Device time of the DES kernels of the last sbs_sim_launch (CUDA events on
 * its stream, finalize excluded); waits for them to finish. */
int sbs_sim_des_ms(sbs_sim* sim, double* ms);
/* Number of kernel launches enqueued by one sbs_sim_launch. */
int32_t sbs_sim_launches_per_run(const sbs_sim* sim);
/* Device bytes allocated for this simulator. */
int64_t sbs_sim_device_bytes(const sbs_sim* sim);
void sbs_sim_destroy(sbs_sim* sim);

/* One-shot: generate traces on the host (threads), upload, simulate, return
 * aggregates.  The reference-facing call behind run_experiment. */
int sbs_run_experiments(const sbs_experiment* points, int32_t n_points,
                        sbs_aggregates* out, int32_t device);

/* ----------------------------------------------------------------------- */
/* Batched PBAA window allocation (allocate_batch, prefill_alloc.cpp:61-88, */
/* greedy_dispatch :23-59).  One warp per cluster-window.                   */
/* All pointers are DEVICE pointers; window w owns requests                 */
/* [req_off[w], req_off[w+1]) of which the first n_pending[w] are q_pending */
/* and the rest q_new (each in caller queue order), and DP capacities       */
/* [dp_off[w], dp_off[w+1]) (c_avail snapshots, updated in place).          */
/* Outputs per request: out_dp = DP index placed, -1 deferred, -2 throttled;*/
/* out_rank = position in the placement order (-1 if not placed);           */
/* wait_out = wait_cycles after the cycle.  flow[w] = flow-control flag.    */
/* Cache-aware mode (capacity_after, prefill_alloc.cpp:12-21): hit != NULL  */
/* gives Len_hit(r, d) of every (request, DP) pair of window w, row-major   */
/* from hit[hit_off[w]] (request-major, n_dp per row); NULL = Basic mode.   */
/* max_requests / max_dp: optional bounds over the batch's windows (0 =     */
/* unknown: the 1024 / 1024 envelope).  Windows of <= 32 requests and <= 32 */
/* DP units (Basic mode, ids < 2^27) run on registers only; the bounds size */
/* the shared-memory slice of the rest, so small batches run many warps per */
/* SM.                                                                      */
typedef struct sbs_window_batch {
  int32_t n_windows;
  int32_t max_requests;
  const int64_t* req_off;
  const int32_t* n_pending;
  const int64_t* dp_off;
  const int32_t* n_limit;
  const int64_t* req_id;
  const int64_t* prompt_len;
  const int32_t* wait_in;
  int64_t* caps;
  int32_t* out_dp;
  int32_t* out_rank;
  int32_t* wait_out;
  uint8_t* flow;
  const int64_t* hit_off;
  const int64_t* hit;
  int32_t max_dp;
  int32_t _pad;
} sbs_window_batch;
int sbs_prefill_allocate(const sbs_window_batch* batch, void* stream);
/* One window from HOST arrays, synchronous (the reference's one-call shape,
 * allocate_batch prefill_alloc.h:59-62): rows = (id, prompt_len, wait_cycles)
 * for the n_pending pending then n_new new requests; caps = c_avail per DP
 * (updated in place); hits = Len_hit rows (NULL: Basic mode).  Outputs as in
 * sbs_window_batch.  Small Basic windows need one launch and no copies. */
int sbs_prefill_allocate_one(const int64_t* rows, int32_t n_pending, int32_t n_new,
                             int64_t* caps, int32_t n_dp, int32_t n_limit,
                             const int64_t* hits, int32_t* out_dp, int32_t* out_rank,
                             int32_t* wait_out, uint8_t* flow);
/* Asynchronous form: enqueue only.  `error_out` is a DEVICE int32 the caller
 * zeroes beforehand; the kernel sets it to SBS_ERR_OVERFLOW when a window
 * exceeds the kernel envelope (1024 requests, 1024 DP units). */
int sbs_prefill_allocate_async(const sbs_window_batch* batch, int32_t* error_out, void* stream);

/* Batched IQR-masked lexicographic decode selection (select_decode_unit,    */
/* decode_alloc.cpp:38-81).  Call c considers units [unit_off[c],           */
/* unit_off[c+1]) with (B, K); returns the selected position, the fallback  */
/* flag and the threshold Q3 + k(Q3-Q1).  DEVICE pointers.                  */
typedef struct sbs_decode_batch {
  int32_t n_calls;
  int32_t max_units; /* optional bound over the calls (0 = unknown); calls of */
                     /* <= 512 units are sorted in registers                  */
  const int64_t* unit_off;
  const int32_t* batch;
  const int64_t* kv;
  double k;
  int32_t* pos_out;
  uint8_t* fallback_out;
  double* threshold_out;
} sbs_decode_batch;
int sbs_decode_select(const sbs_decode_batch* batch, void* stream);
/* Asynchronous form (see sbs_prefill_allocate_async); error 3 = empty call,
 * 4 = more units than max_units (2048 when 0; at most 16384). */
int sbs_decode_select_async(const sbs_decode_batch* batch, int32_t* error_out, void* stream);

/* Batched schedule_decode_batch (decode_alloc.cpp:83-106): batch b places
 * candidates [cand_off[b], cand_off[b+1]) onto units [unit_off[b],
 * unit_off[b+1]) in the reference's order (sort_len desc, request_id asc,
 * stable), one select_decode_unit each, adding B += 1, K += kv_len to the
 * chosen unit (batch / kv updated in place).  Outputs per placement j of
 * batch b (at cand_off[b] + j): order_out = input index of the candidate
 * placed j-th, pos_out = the unit position chosen, and (nullable) the
 * fallback flag and threshold the observer would see.  One warp per batch;
 * max_candidates / max_units bound every batch (<= 4096 each).  DEVICE
 * pointers; synchronous (checks the error flag). */
typedef struct sbs_decode_schedule {
  int32_t n_batches;
  int32_t max_candidates;
  int32_t max_units;
  int32_t _pad;
  const int64_t* cand_off;
  const uint64_t* request_id;
  const int64_t* sort_len;
  const int64_t* kv_len;
  const int64_t* unit_off;
  int32_t* batch;
  int64_t* kv;
  double k;
  int32_t* order_out;
  int32_t* pos_out;
  uint8_t* fallback_out;
  double* threshold_out;
} sbs_decode_schedule;
int sbs_decode_schedule_batch(const sbs_decode_schedule* s, void* stream);
/* Asynchronous form; error 3 = a batch with candidates but no units
 * (select_decode_unit's logic_error), 4 = beyond max_candidates/max_units. */
int sbs_decode_schedule_batch_async(const sbs_decode_schedule* s, int32_t* error_out, void* stream);

const char* sbs_last_error(void);
const char* sbs_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SBS_B200_H_ */
