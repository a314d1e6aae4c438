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

#endif
