/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference algorithms
 * on the hot path, used as a checker by tests/, smoke() and bench.py's CPU
 * leg.  Never linked into the product.  Pinned against the compiled reference
 * (oracle/_ref) and the reference's own known-answer values (tests/). */
#ifndef SBS_ORACLE_H_
#define SBS_ORACLE_H_
#include <stdint.h>

/* allocate_batch, Basic mode (prefill_alloc.cpp:61-88; greedy_dispatch :23-59).
 * pend/fresh: rows (id, prompt_len, wait_cycles).  caps updated in place.
 * out_map rows (id, dp) in placement order, out_def rows (id, wait) in
 * FCFS order, out_thr ids; counts = {n_map, n_def, n_thr}; returns flow flag. */
int orc_allocate_batch(const int64_t* pend, int64_t n_pend, const int64_t* fresh,
                       int64_t n_fresh, int64_t* caps, int64_t n_dp, int n_limit,
                       int64_t* out_map, int64_t* out_def, int64_t* out_thr,
                       int64_t* counts);

/* allocate_batch in cache-aware mode: hits (nullable) rows of Len_hit(r, d),
 * n_dp per row, rows in pend-then-fresh order (capacity_after,
 * prefill_alloc.cpp:12-21). */
int orc_allocate_batch_hits(const int64_t* pend, int64_t n_pend, const int64_t* fresh,
                            int64_t n_fresh, int64_t* caps, int64_t n_dp, int n_limit,
                            const int64_t* hits, int64_t* out_map, int64_t* out_def,
                            int64_t* out_thr, int64_t* counts);

/* percentile (decode_alloc.cpp:13-23): p clamped to [0,100]; n >= 1. */
double orc_percentile(const double* values, int64_t n, double p);

/* outlier_threshold (decode_alloc.cpp:25-30): Q3 + k (Q3 - Q1). */
double orc_outlier_threshold(const int64_t* kv, int64_t n, double k);

/* select_decode_unit (decode_alloc.cpp:38-81). */
int orc_select_decode_unit(const int64_t* batch, const int64_t* kv, int64_t n, double k,
                           int* fallback, double* threshold);

/* schedule_decode_batch (decode_alloc.cpp:83-106): candidates rows
 * (request_id, sort_len, kv_len); units B/K updated in place; out rows
 * (request_id, unit_index) in placement order. */
void orc_schedule_decode_batch(const int64_t* cand, int64_t n_cand, int64_t* batch,
                               int64_t* kv, int64_t n_units, double k, int64_t* out);

/* Batched allocate_batch over the CSR layout of sbs_window_batch. */
void orc_allocate_many(int64_t n_windows, const int64_t* req_off, const int32_t* n_pending,
                       const int64_t* dp_off, const int32_t* n_limit, const int64_t* req_id,
                       const int64_t* prompt_len, const int32_t* wait_in, int64_t* caps,
                       int32_t* out_dp, int32_t* out_rank, int32_t* wait_out, uint8_t* flow);

/* ---- full simulator restatement (sbs_oracle_des.c) ---- */
typedef struct { int instance; double from_s, until_s; } orc_drop;
typedef struct { int instance; double time_s; } orc_dead;
typedef struct { int instance; int healthy; double time_s; } orc_topo;

/* ExperimentConfig fields on the path (config.h:66-75, core.h:236-260) */
typedef struct {
  int n_instances_prefill, n_instances_decode, dp_degree, dp_degree_decode;
  int64_t c_chunk, w_size, decode_tokens_per_step;
  double t_default_s, l_net_s, iqr_k, watchdog_multiplier;
  int n_limit, decode_max_batch_per_dp;
  double prefill_base_s, prefill_per_token_s, decode_base_s, decode_per_request_s,
      decode_per_kv_token_s;
  int policy;        /* 0 sbs, 1 immediate/round_robin, 3 least_outstanding */
  int decode_policy; /* 0 iqr, 1 random, 2 round_robin */
  uint64_t seed;
  double duration_s, warmup_fraction;
  const orc_drop* drops;
  int n_drops;
  const orc_dead* deads;
  int n_deads;
  const orc_topo* topology;
  int n_topology;
  /* cache-aware PBAA (simulation.cpp:267-268) + CacheSettings (core.h:230-234) */
  int prefill_mode; /* 0 basic, 1 cache_aware */
  int cache_enabled;
  int64_t cache_budget_tokens;
  const int64_t* cache_probe_lens;
  int n_probe_lens;
} orc_config;

/* Aggregates (metrics.h:67-102) + counters */
typedef struct {
  uint64_t generated, completed, throttled, in_flight, window_requests;
  double ttft_mean_s, ttft_p50_s, ttft_p95_s, scheduler_wait_mean_s, device_wait_mean_s,
      total_wait_mean_s;
  uint64_t passes;
  double chunk_util_mean;
  uint64_t decode_steps, output_tokens;
  double output_tokens_per_s, kv_mean_time_avg, kv_sigma_time_avg, completed_per_s;
  uint64_t watchdog_fires, dropped_end_forwards, rejected_samples, deferrals,
      flow_control_events, mask_events, fallback_events;
  double warmup_cutoff_s, duration_s;
  uint64_t alloc_calls, decode_selects;
  int error;
} orc_result;

/* run_experiment (simulation.cpp:136-169) on a given trace.  per_req
 * (nullable): n rows of (status, dispatch, prefill_start, first_token,
 * completion), -1 when unset.  Returns 0 or 3 (invariant). */
int orc_run(const orc_config* cfg, const int64_t* arr, const int32_t* prompt,
            const int32_t* output, int64_t n, orc_result* res, int64_t* per_req);
/* The same with shared prefixes: request r's prefix_tokens are the first
 * pfx_size[r] tokens of pool pfx_pool[r] (workload.cpp:30-37, 129-138);
 * both nullable. */
int orc_run_prefix(const orc_config* cfg, const int64_t* arr, const int32_t* prompt,
                   const int32_t* output, const int32_t* pfx_pool, const int32_t* pfx_size,
                   int64_t n, orc_result* res, int64_t* per_req);

#endif
