/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference's hot-path
 * algorithms (the checker, never the product).  Each function cites the
 * reference lines it restates; compiled with -ffp-contract=off so the FP64
 * expressions round like the reference's x86-64 build.
 *
 * Pinned by tests/test_oracle.py against (a) the reference's known-answer
 * values (acceptance.cpp:275-295, SPEC.md worked examples), (b) the compiled
 * reference itself (oracle/_ref) on the exhaustive PBAA grid
 * (acceptance.cpp:415-446) and on random cases, and (c) committed golden
 * vectors recorded from the reference simulator (tests/golden/). */
#include "sbs_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------- PBAA (Alg. 2) ---------------- */

typedef struct {
  int64_t id, len, wait;
  int64_t pos;        /* input position */
  const int64_t* hit; /* cache-aware: Len_hit per DP unit, NULL = Basic */
} orc_req;

static int cmp_len_desc_id_asc(const void* a, const void* b) {
  const orc_req* x = (const orc_req*)a;
  const orc_req* y = (const orc_req*)b;
  if (x->len != y->len) return x->len > y->len ? -1 : 1; /* prompt_len desc */
  if (x->id != y->id) return x->id < y->id ? -1 : 1;     /* then id asc */
  return x->pos < y->pos ? -1 : (x->pos > y->pos);        /* stable */
}

/* greedy_dispatch (prefill_alloc.cpp:23-59): longest first; argmax of
 * capacity_after = c_avail - (prompt_len - hit) (strict >, lowest index;
 * prefill_alloc.cpp:12-21, hit = 0 in Basic mode); guard on the chosen unit's
 * pre-assignment c_avail > 0; deferred keep input order. */
static void greedy(orc_req* q, int64_t n, int64_t* caps, int64_t n_dp, int64_t* out_map,
                   int64_t* n_map, orc_req* deferred, int64_t* n_def) {
  orc_req* order = (orc_req*)malloc(sizeof(orc_req) * (size_t)(n > 0 ? n : 1));
  char* placed = (char*)calloc((size_t)(n > 0 ? n : 1), 1);
  memcpy(order, q, sizeof(orc_req) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) order[i].pos = i;
  qsort(order, (size_t)n, sizeof(orc_req), cmp_len_desc_id_asc);
  for (int64_t t = 0; t < n; ++t) {
    const orc_req* r = &order[t];
    int64_t best = -1, best_after = 0;
    for (int64_t d = 0; d < n_dp; ++d) {
      int64_t after = caps[d] - (r->len - (r->hit ? r->hit[d] : 0));
      if (best < 0 || after > best_after) {
        best = d;
        best_after = after;
      }
    }
    if (best < 0 || caps[best] <= 0) continue;
    caps[best] = best_after;
    out_map[2 * *n_map] = r->id;
    out_map[2 * *n_map + 1] = best;
    *n_map += 1;
    placed[r->pos] = 1;
  }
  for (int64_t i = 0; i < n; ++i)
    if (!placed[i]) deferred[(*n_def)++] = q[i];
  free(order);
  free(placed);
}

/* allocate_batch (prefill_alloc.cpp:61-88). */
int orc_allocate_batch(const int64_t* pend, int64_t n_pend, const int64_t* fresh,
                       int64_t n_fresh, int64_t* caps, int64_t n_dp, int n_limit,
                       int64_t* out_map, int64_t* out_def, int64_t* out_thr,
                       int64_t* counts) {
  return orc_allocate_batch_hits(pend, n_pend, fresh, n_fresh, caps, n_dp, n_limit, NULL,
                                 out_map, out_def, out_thr, counts);
}

int orc_allocate_batch_hits(const int64_t* pend, int64_t n_pend, const int64_t* fresh,
                            int64_t n_fresh, int64_t* caps, int64_t n_dp, int n_limit,
                            const int64_t* hits, int64_t* out_map, int64_t* out_def,
                            int64_t* out_thr, int64_t* counts) {
  int64_t n = n_pend + n_fresh;
  orc_req* qp = (orc_req*)malloc(sizeof(orc_req) * (size_t)(n_pend > 0 ? n_pend : 1));
  orc_req* qn = (orc_req*)malloc(sizeof(orc_req) * (size_t)(n_fresh > 0 ? n_fresh : 1));
  orc_req* dp = (orc_req*)malloc(sizeof(orc_req) * (size_t)(n > 0 ? n : 1));
  orc_req* dn = (orc_req*)malloc(sizeof(orc_req) * (size_t)(n > 0 ? n : 1));
  for (int64_t i = 0; i < n_pend; ++i) {
    qp[i].id = pend[3 * i]; qp[i].len = pend[3 * i + 1]; qp[i].wait = pend[3 * i + 2];
    qp[i].hit = hits ? hits + i * n_dp : NULL;
  }
  for (int64_t i = 0; i < n_fresh; ++i) {
    qn[i].id = fresh[3 * i]; qn[i].len = fresh[3 * i + 1]; qn[i].wait = fresh[3 * i + 2];
    qn[i].hit = hits ? hits + (n_pend + i) * n_dp : NULL;
  }
  int64_t n_map = 0, n_dp_def = 0, n_new_def = 0, n_d = 0, n_t = 0;
  greedy(qp, n_pend, caps, n_dp, out_map, &n_map, dp, &n_dp_def);
  greedy(qn, n_fresh, caps, n_dp, out_map, &n_map, dn, &n_new_def);
  /* aging: pending-deferred first, then new-deferred (prefill_alloc.cpp:74-85) */
  for (int phase = 0; phase < 2; ++phase) {
    orc_req* q = phase == 0 ? dp : dn;
    int64_t m = phase == 0 ? n_dp_def : n_new_def;
    for (int64_t i = 0; i < m; ++i) {
      int64_t w = q[i].wait + 1;
      if (w > n_limit) {
        out_thr[n_t++] = q[i].id;
      } else {
        out_def[2 * n_d] = q[i].id;
        out_def[2 * n_d + 1] = w;
        n_d += 1;
      }
    }
  }
  counts[0] = n_map;
  counts[1] = n_d;
  counts[2] = n_t;
  free(qp); free(qn); free(dp); free(dn);
  return n_t > 0;
}

/* ---------------- IQR decode placement (Alg. 3) ---------------- */

static int cmp_double(const void* a, const void* b) {
  double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}

/* percentile (decode_alloc.cpp:13-23). */
double orc_percentile(const double* values, int64_t n, double p) {
  if (n < 1) return NAN;
  if (p < 0.0) p = 0.0;
  if (p > 100.0) p = 100.0;
  double* v = (double*)malloc(sizeof(double) * (size_t)n);
  memcpy(v, values, sizeof(double) * (size_t)n);
  qsort(v, (size_t)n, sizeof(double), cmp_double);
  double rank = ((double)n - 1.0) * p / 100.0;
  size_t lo = (size_t)floor(rank), hi = (size_t)ceil(rank);
  double out;
  if (lo == hi) {
    out = v[lo];
  } else {
    double frac = rank - (double)lo;
    out = v[lo] + frac * (v[hi] - v[lo]);
  }
  free(v);
  return out;
}

/* outlier_threshold (decode_alloc.cpp:25-30). */
double orc_outlier_threshold(const int64_t* kv, int64_t n, double k) {
  double* v = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  for (int64_t i = 0; i < n; ++i) v[i] = (double)kv[i];
  double q1 = orc_percentile(v, n, 25.0);
  double q3 = orc_percentile(v, n, 75.0);
  free(v);
  return q3 + k * (q3 - q1);
}

/* select_decode_unit (decode_alloc.cpp:38-81): mask K <= Th (fallback: all),
 * lex-min (B, K) with strict <, first position on ties (lex_less :32-36). */
int orc_select_decode_unit(const int64_t* batch, const int64_t* kv, int64_t n, double k,
                           int* fallback, double* threshold) {
  if (n < 1) return -1;
  double th = orc_outlier_threshold(kv, n, k);
  int64_t nsafe = 0;
  for (int64_t i = 0; i < n; ++i) nsafe += ((double)kv[i] <= th);
  int fb = nsafe == 0;
  int64_t best = -1;
  for (int64_t i = 0; i < n; ++i) {
    if (!fb && !((double)kv[i] <= th)) continue;
    if (best < 0) { best = i; continue; }
    if (batch[i] < batch[best] || (batch[i] == batch[best] && kv[i] < kv[best])) best = i;
  }
  if (fallback) *fallback = fb;
  if (threshold) *threshold = th;
  return (int)best;
}

typedef struct {
  int64_t id, sort_len, kv_len, pos;
} orc_cand;

static int cmp_cand(const void* a, const void* b) {
  const orc_cand* x = (const orc_cand*)a;
  const orc_cand* y = (const orc_cand*)b;
  if (x->sort_len != y->sort_len) return x->sort_len > y->sort_len ? -1 : 1;
  if (x->id != y->id) return x->id < y->id ? -1 : 1;
  return x->pos < y->pos ? -1 : (x->pos > y->pos);
}

/* schedule_decode_batch (decode_alloc.cpp:83-106). */
void orc_schedule_decode_batch(const int64_t* cand, int64_t n_cand, int64_t* batch,
                               int64_t* kv, int64_t n_units, double k, int64_t* out) {
  orc_cand* c = (orc_cand*)malloc(sizeof(orc_cand) * (size_t)(n_cand > 0 ? n_cand : 1));
  for (int64_t i = 0; i < n_cand; ++i) {
    c[i].id = cand[3 * i]; c[i].sort_len = cand[3 * i + 1]; c[i].kv_len = cand[3 * i + 2];
    c[i].pos = i;
  }
  qsort(c, (size_t)n_cand, sizeof(orc_cand), cmp_cand);
  for (int64_t i = 0; i < n_cand; ++i) {
    int pos = orc_select_decode_unit(batch, kv, n_units, k, 0, 0);
    batch[pos] += 1;
    kv[pos] += c[i].kv_len;
    out[2 * i] = c[i].id;
    out[2 * i + 1] = pos;
  }
  free(c);
}

/* Batch driver over the same CSR window layout as sbs_prefill_allocate
 * (include/sbs_b200.h): out_dp (-1 deferred, -2 throttled), out_rank,
 * wait_out per request, caps updated, flow per window. */
void orc_allocate_many(int64_t n_windows, const int64_t* req_off, const int32_t* n_pending,
                       const int64_t* dp_off, const int32_t* n_limit, const int64_t* req_id,
                       const int64_t* prompt_len, const int32_t* wait_in, int64_t* caps,
                       int32_t* out_dp, int32_t* out_rank, int32_t* wait_out, uint8_t* flow) {
  for (int64_t w = 0; w < n_windows; ++w) {
    int64_t r0 = req_off[w], n = req_off[w + 1] - r0, np_ = n_pending[w];
    int64_t* rows = (int64_t*)malloc(sizeof(int64_t) * 3 * (size_t)(n > 0 ? n : 1));
    int64_t* om = (int64_t*)malloc(sizeof(int64_t) * 2 * (size_t)(n > 0 ? n : 1));
    int64_t* od = (int64_t*)malloc(sizeof(int64_t) * 2 * (size_t)(n > 0 ? n : 1));
    int64_t* ot = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    for (int64_t i = 0; i < n; ++i) {
      rows[3 * i] = req_id[r0 + i];
      rows[3 * i + 1] = prompt_len[r0 + i];
      rows[3 * i + 2] = wait_in[r0 + i];
    }
    int64_t cnt[3];
    flow[w] = (uint8_t)orc_allocate_batch(rows, np_, rows + 3 * np_, n - np_, caps + dp_off[w],
                                          dp_off[w + 1] - dp_off[w], n_limit[w], om, od, ot, cnt);
    /* map ids back to positions (ids are unique within a window) */
    for (int64_t i = 0; i < n; ++i) { out_dp[r0 + i] = -3; out_rank[r0 + i] = -1; }
    for (int64_t k = 0; k < cnt[0]; ++k)
      for (int64_t i = 0; i < n; ++i)
        if (req_id[r0 + i] == om[2 * k]) {
          out_dp[r0 + i] = (int32_t)om[2 * k + 1];
          out_rank[r0 + i] = (int32_t)k;
          wait_out[r0 + i] = wait_in[r0 + i];
          break;
        }
    for (int64_t k = 0; k < cnt[1]; ++k)
      for (int64_t i = 0; i < n; ++i)
        if (req_id[r0 + i] == od[2 * k]) { out_dp[r0 + i] = -1; wait_out[r0 + i] = (int32_t)od[2 * k + 1]; break; }
    for (int64_t k = 0; k < cnt[2]; ++k)
      for (int64_t i = 0; i < n; ++i)
        if (req_id[r0 + i] == ot[k]) { out_dp[r0 + i] = -2; wait_out[r0 + i] = wait_in[r0 + i] + 1; break; }
    free(rows); free(om); free(od); free(ot);
  }
}
