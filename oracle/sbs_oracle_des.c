/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference simulator's
 * hot path (one run_experiment, proj/src/simulation.cpp:136-169) used as a
 * checker: a (time, seq) binary-heap event loop (simclock.cpp:24-45), the
 * Runner handlers (simulation.cpp:171-512), the engine model
 * (engine_model.cpp:12-217), interval control (interval_control.cpp:11-99),
 * PBAA (via orc_allocate_batch), IQR/random/round-robin decode placement and
 * MetricsCollector::finalize (metrics.cpp:103-190).  It follows the
 * reference's straightforward data structures (per-DP FIFO deques, resident
 * lists scanned every step), not the GPU kernel's restructured ones, so a
 * shared bug is unlikely.  Pinned by tests/test_oracle_des.py against the
 * compiled reference and the golden fixtures. */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "sbs_oracle.h"

#define INF64 INT64_MAX
enum { EV_ARR = 0, EV_TICK, EV_EF, EV_WD, EV_TOPO, EV_DS };
enum { ST_PENDING = 0, ST_DISPATCHED, ST_PREFILLING, ST_DECODING, ST_COMPLETED, ST_THROTTLED };

static int64_t s2ns(double s) { return (int64_t)llround(s * 1e9); } /* core.h:26-28 */

/* ---------------- event heap (simclock.h:89-94) ---------------- */
typedef struct { int64_t t; uint64_t seq; int kind; int a; uint64_t b; } ev_t;
typedef struct { ev_t* v; int64_t n, cap; uint64_t next_seq; int64_t now; int bad; } clock_t_;

static int ev_less(const ev_t* x, const ev_t* y) {
  return x->t != y->t ? x->t < y->t : x->seq < y->seq;
}
static void schedule(clock_t_* c, int64_t t, int kind, int a, uint64_t b) {
  if (t < c->now) c->bad = 1; /* simclock.cpp:25-28 logic_error */
  if (c->n == c->cap) {
    c->cap = c->cap ? 2 * c->cap : 1024;
    c->v = (ev_t*)realloc(c->v, sizeof(ev_t) * (size_t)c->cap);
  }
  ev_t e = {t, c->next_seq++, kind, a, b};
  int64_t i = c->n++;
  while (i > 0) {
    int64_t p = (i - 1) / 2;
    if (!ev_less(&e, &c->v[p])) break;
    c->v[i] = c->v[p];
    i = p;
  }
  c->v[i] = e;
}
static ev_t pop(clock_t_* c) {
  ev_t top = c->v[0], last = c->v[--c->n];
  int64_t i = 0;
  for (;;) {
    int64_t l = 2 * i + 1, r = l + 1, m = i;
    const ev_t* best = &last;
    if (l < c->n && ev_less(&c->v[l], best)) { m = l; best = &c->v[l]; }
    if (r < c->n && ev_less(&c->v[r], best)) { m = r; }
    if (m == i) break;
    c->v[i] = c->v[m];
    i = m;
  }
  if (c->n > 0) c->v[i] = last;
  return top;
}

/* ---------------- growable arrays ---------------- */
typedef struct { int64_t* v; int64_t n, cap; } vec_t;
static void vpush(vec_t* a, int64_t x) {
  if (a->n == a->cap) {
    a->cap = a->cap ? 2 * a->cap : 16;
    a->v = (int64_t*)realloc(a->v, sizeof(int64_t) * (size_t)a->cap);
  }
  a->v[a->n++] = x;
}
static void verase(vec_t* a, int64_t i) {
  memmove(a->v + i, a->v + i + 1, sizeof(int64_t) * (size_t)(a->n - i - 1));
  a->n -= 1;
}

/* PendingChunk deque (core.h:126-130): id, tokens, backlog */
typedef struct { int64_t* id; int64_t* tok; char* bl; int64_t head, n, cap; } deq_t;
static void dq_push(deq_t* d, int64_t id, int64_t tok, char bl) {
  if (d->n == d->cap) {
    int64_t nc = d->cap ? 2 * d->cap : 16;
    int64_t* ni = (int64_t*)malloc(sizeof(int64_t) * (size_t)nc);
    int64_t* nt = (int64_t*)malloc(sizeof(int64_t) * (size_t)nc);
    char* nb = (char*)malloc((size_t)nc);
    for (int64_t k = 0; k < d->n; ++k) {
      int64_t j = (d->head + k) % (d->cap ? d->cap : 1);
      ni[k] = d->id[j]; nt[k] = d->tok[j]; nb[k] = d->bl[j];
    }
    free(d->id); free(d->tok); free(d->bl);
    d->id = ni; d->tok = nt; d->bl = nb; d->head = 0; d->cap = nc;
  }
  int64_t j = (d->head + d->n) % d->cap;
  d->id[j] = id; d->tok[j] = tok; d->bl[j] = bl;
  d->n += 1;
}
#define DQ(d, k) (((d)->head + (k)) % (d)->cap)

/* PrefixCache (core.h:87-123, core.cpp:13-75): LRU list of (hash, k), entry 0
 * is the front (most recent); linear lookups (test sizes are small). */
typedef struct {
  uint64_t* key;
  int64_t* k;
  int64_t n, cap, used;
} pcache_t;

typedef struct {
  int64_t u_flight, r_queued;
  deq_t pending;
  pcache_t cache;
  int64_t batch, kv;
  vec_t residents;
  vec_t pass_id, pass_tok; /* pass_content (core.h:178) */
} dp_t;

typedef struct {
  int healthy, dead, busy, stepping, ef_seen, wd_fired, has_deadline;
  int64_t pass_started, deadline, death;
  uint64_t pass_seq, step_seq, wd_gen;
  int task_depth;
  dp_t* dp;
  int n_dp;
} inst_t;

/* ---------------- mt19937_64 (std::mersenne_twister_engine) ---------------- */
typedef struct { uint64_t mt[312]; int idx; } mt64_t;
static void mt_seed(mt64_t* m, uint64_t s) {
  m->mt[0] = s;
  for (int i = 1; i < 312; ++i) m->mt[i] = 6364136223846793005ULL * (m->mt[i - 1] ^ (m->mt[i - 1] >> 62)) + (uint64_t)i;
  m->idx = 312;
}
static uint64_t mt_next(mt64_t* m) {
  if (m->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (m->mt[i] & 0xFFFFFFFF80000000ULL) | (m->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t xa = (x >> 1) ^ ((x & 1) ? 0xB5026F5AA96619E9ULL : 0);
      m->mt[i] = m->mt[(i + 156) % 312] ^ xa;
    }
    m->idx = 0;
  }
  uint64_t y = m->mt[m->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

/* ---------------- prefix cache ---------------- */
static int32_t prefix_token(int pool, int64_t i) { /* workload.cpp:30-37 */
  uint64_t h = 1469598103934665603ull;
  h ^= (uint64_t)pool * 0x9e3779b97f4a7c15ull;
  h ^= (uint64_t)i + 0x632be59bd9b4e019ull;
  h *= 1099511628211ull;
  return (int32_t)(h & 0x7fffffff);
}
static uint64_t hash_prefix(int pool, int64_t k) { /* core.cpp:18-31 */
  uint64_t h = 14695981039346656037ull ^ (uint64_t)k;
  for (int64_t i = 0; i < k; ++i) {
    uint32_t v = (uint32_t)prefix_token(pool, i);
    for (int b = 0; b < 4; ++b) {
      h ^= (v >> (8 * b)) & 0xff;
      h *= 1099511628211ull;
    }
  }
  return h;
}
static int64_t pc_find(const pcache_t* c, uint64_t key) {
  for (int64_t i = 0; i < c->n; ++i)
    if (c->key[i] == key) return i;
  return -1;
}
static void pc_to_front(pcache_t* c, int64_t i) { /* touch: splice to begin */
  uint64_t key = c->key[i];
  int64_t k = c->k[i];
  memmove(c->key + 1, c->key, sizeof(uint64_t) * (size_t)i);
  memmove(c->k + 1, c->k, sizeof(int64_t) * (size_t)i);
  c->key[0] = key;
  c->k[0] = k;
}
/* longest_hit (core.cpp:33-41); probes ascending */
static int64_t pc_longest_hit(const pcache_t* c, const int64_t* probes, int np, int pool,
                              int64_t psize, int64_t prompt) {
  int64_t best = 0;
  for (int j = 0; j < np; ++j) {
    int64_t k = probes[j];
    if (k > prompt || k > psize) break;
    if (pc_find(c, hash_prefix(pool, k)) >= 0) best = k;
  }
  return best;
}
/* insert + evict_to_budget (core.cpp:43-75) */
static void pc_insert(pcache_t* c, const int64_t* probes, int np, int64_t budget, int pool,
                      int64_t psize, int64_t prompt) {
  if (budget <= 0) return;
  for (int j = 0; j < np; ++j) {
    int64_t k = probes[j];
    if (k > prompt || k > psize) break;
    uint64_t key = hash_prefix(pool, k);
    int64_t at = pc_find(c, key);
    if (at >= 0) { pc_to_front(c, at); continue; }
    if (c->n == c->cap) {
      c->cap = c->cap ? 2 * c->cap : 16;
      c->key = (uint64_t*)realloc(c->key, sizeof(uint64_t) * (size_t)c->cap);
      c->k = (int64_t*)realloc(c->k, sizeof(int64_t) * (size_t)c->cap);
    }
    c->key[c->n] = key;
    c->k[c->n] = k;
    c->n += 1;
    pc_to_front(c, c->n - 1);
    c->used += k;
  }
  while (c->used > budget && c->n > 0) { /* pop_back */
    c->n -= 1;
    c->used -= c->k[c->n];
  }
}

/* ---------------- runner ---------------- */
typedef struct {
  const orc_config* cfg;
  int64_t n;
  const int64_t* arr;
  const int32_t* prompt;
  const int32_t* output;
  const int32_t* pfx_pool; /* nullable */
  const int32_t* pfx_size;
  int64_t* probes;         /* cache.probe_lens sorted (core.cpp:15) */
  int n_probes, cache_aware;
  int8_t* status;
  int* wait;
  int64_t *disp, *pstart, *ftok, *comp, *ctot, *cdone, *ddone;
  uint64_t* mark;
  inst_t* inst;
  int P, Dn, n_inst;
  clock_t_ clk;
  /* scheduler (core.h:197-218) */
  int64_t* win;
  int64_t win_n, win_head;
  int64_t t_default, t_bar, l_net, i_opt;
  int n_active, last_inst, has_last;
  int64_t last_dispatch;
  uint64_t tick_gen, rejected;
  vec_t q_pending, q_new, decode_wait;
  /* baselines */
  int rr_next;
  int* rr_dp;
  mt64_t rng;
  uint64_t dec_rr;
  /* metrics */
  orc_result* res;
  int64_t warmup, horizon;
  double util_sum, kv_mean_sum, kv_sig_sum;
  int64_t passes, steps, out_tok, kv_n;
  int error;
} run_t;

static void maybe_die(run_t* R, int i) { /* simulation.cpp:122-126 */
  inst_t* I = &R->inst[i];
  if (!I->dead && R->clk.now >= I->death) I->dead = 1;
}
static int drop_matches(run_t* R, int i) { /* simulation.cpp:128-134 */
  for (int k = 0; k < R->cfg->n_drops; ++k) {
    const orc_drop* d = &R->cfg->drops[k];
    int64_t from = s2ns(d->from_s), until = isfinite(d->until_s) ? s2ns(d->until_s) : INF64;
    if ((d->instance == -1 || d->instance == i) && R->clk.now >= from && R->clk.now < until) return 1;
  }
  return 0;
}

static void recompute_interval(run_t* R) { /* interval_control.cpp:18-24 */
  if (R->win_n == 0) {
    R->t_bar = R->t_default;
  } else {
    int64_t s = 0;
    for (int64_t k = 0; k < R->win_n; ++k) s += R->win[(R->win_head + k) % R->cfg->w_size];
    R->t_bar = s / R->win_n;
  }
  if (R->n_active <= 0) return;
  int64_t v = (R->t_bar + R->l_net) / R->n_active;
  R->i_opt = v > 1 ? v : 1;
}

static void arm_tick(run_t* R, int64_t at) { /* simulation.cpp:234-238 */
  R->tick_gen += 1;
  schedule(&R->clk, at > R->clk.now ? at : R->clk.now, EV_TICK, 0, R->tick_gen);
}

static void dispatch_prefill(run_t* R, int i, int d, int64_t id, int64_t tokens) { /* engine_model.cpp:37-49 */
  dp_t* D = &R->inst[i].dp[d];
  char bl = (char)R->inst[i].busy;
  dq_push(&D->pending, id, tokens, bl);
  if (bl) D->r_queued += tokens; else D->u_flight += tokens;
}

static void try_start_pass(run_t* R, int i) { /* engine_model.cpp:51-116 + record_pass */
  inst_t* I = &R->inst[i];
  if (I->busy || I->dead) return;
  int any = 0;
  for (int d = 0; d < I->n_dp; ++d) any |= I->dp[d].pending.n > 0;
  if (!any) return;
  int64_t now = R->clk.now, maxload = 0;
  I->pass_seq += 1;
  int64_t c = R->cfg->c_chunk;
  double usum = 0.0;
  for (int d = 0; d < I->n_dp; ++d) {
    dp_t* D = &I->dp[d];
    D->pass_id.n = 0;
    D->pass_tok.n = 0;
    int64_t room = c;
    while (room > 0 && D->pending.n > 0) {
      int64_t h = DQ(&D->pending, 0);
      int64_t take = D->pending.tok[h] < room ? D->pending.tok[h] : room;
      int64_t id = D->pending.id[h];
      vpush(&D->pass_id, id);
      vpush(&D->pass_tok, take);
      room -= take;
      if (R->pstart[id] < 0) { R->pstart[id] = now; R->status[id] = ST_PREFILLING; }
      if (D->pending.bl[h]) D->r_queued -= take; else D->u_flight -= take;
      D->pending.tok[h] -= take;
      if (D->pending.tok[h] == 0) { D->pending.head = (D->pending.head + 1) % D->pending.cap; D->pending.n -= 1; }
    }
    for (int64_t k = 0; k < D->pending.n; ++k) {
      int64_t j = DQ(&D->pending, k);
      if (!D->pending.bl[j]) { D->u_flight -= D->pending.tok[j]; D->r_queued += D->pending.tok[j]; D->pending.bl[j] = 1; }
    }
    int64_t assigned = c - room;
    if (assigned > maxload) maxload = assigned;
    usum += (double)(assigned < c ? assigned : c) / (double)c; /* metrics.cpp:193-202 */
  }
  I->busy = 1;
  I->pass_started = now;
  double dur = R->cfg->prefill_base_s + R->cfg->prefill_per_token_s * (double)maxload;
  schedule(&R->clk, now + s2ns(dur), EV_EF, i, I->pass_seq);
  if (now >= R->warmup) { R->passes += 1; R->util_sum += usum / (double)I->n_dp; }
}

static int cmp_u64(const void* a, const void* b) {
  uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return (x > y) - (x < y);
}

static void complete(run_t* R, int64_t id) {
  R->status[id] = ST_COMPLETED;
  R->comp[id] = R->clk.now;
}

static void try_begin_step(run_t* R, int i) { /* engine_model.cpp:153-179 */
  inst_t* I = &R->inst[i];
  if (I->stepping || I->dead) return;
  int any = 0;
  for (int d = 0; d < I->n_dp; ++d) any |= I->dp[d].residents.n > 0;
  if (!any) return;
  I->step_seq += 1;
  double worst = 0.0;
  for (int d = 0; d < I->n_dp; ++d) {
    dp_t* D = &I->dp[d];
    for (int64_t k = 0; k < D->residents.n; ++k) R->mark[D->residents.v[k]] = I->step_seq;
    double t = R->cfg->decode_per_request_s * (double)D->batch + R->cfg->decode_per_kv_token_s * (double)D->kv;
    if (t > worst) worst = t;
  }
  I->stepping = 1;
  schedule(&R->clk, R->clk.now + s2ns(R->cfg->decode_base_s + worst), EV_DS, i, I->step_seq);
}

static void drain_decode(run_t* R) { /* simulation.cpp:413-484 */
  if (R->decode_wait.n == 0) return;
  const int cap = R->cfg->decode_max_batch_per_dp;
  int touched[64], nt = 0;
  int64_t U = 0;
  for (int i = R->P; i < R->n_inst; ++i) U += R->inst[i].n_dp;
  int64_t* ui = (int64_t*)malloc(sizeof(int64_t) * (size_t)(U + 1));
  int64_t* ud = (int64_t*)malloc(sizeof(int64_t) * (size_t)(U + 1));
  int64_t* ub = (int64_t*)malloc(sizeof(int64_t) * (size_t)(U + 1));
  int64_t* uk = (int64_t*)malloc(sizeof(int64_t) * (size_t)(U + 1));
  while (R->decode_wait.n > 0) {
    int64_t nu = 0;
    for (int i = R->P; i < R->n_inst; ++i) {
      maybe_die(R, i);
      inst_t* I = &R->inst[i];
      if (!I->healthy || I->dead) continue;
      for (int d = 0; d < I->n_dp; ++d) {
        if (cap > 0 && I->dp[d].batch >= cap) continue;
        ui[nu] = i; ud[nu] = d; ub[nu] = I->dp[d].batch; uk[nu] = I->dp[d].kv;
        nu += 1;
      }
    }
    if (nu == 0) break;
    int64_t best = 0;
    for (int64_t k = 1; k < R->decode_wait.n; ++k) {
      int64_t a = R->decode_wait.v[k], b = R->decode_wait.v[best];
      int64_t la = (int64_t)R->prompt[a] + R->output[a], lb = (int64_t)R->prompt[b] + R->output[b];
      if (la > lb || (la == lb && a < b)) best = k;
    }
    int64_t id = R->decode_wait.v[best];
    int64_t pos = 0;
    if (R->cfg->decode_policy == 0) {
      int fb = 0;
      double th = 0;
      pos = orc_select_decode_unit(ub, uk, nu, R->cfg->iqr_k, &fb, &th);
      int64_t ns = 0;
      for (int64_t k = 0; k < nu; ++k) ns += ((double)uk[k] <= th);
      if (fb) R->res->fallback_events += 1;
      else if (ns < nu) R->res->mask_events += 1;
    } else if (R->cfg->decode_policy == 1) {
      double u = (double)(mt_next(&R->rng) >> 11) * 0x1.0p-53;
      int64_t q = (int64_t)(u * (double)nu);
      pos = q < nu - 1 ? q : nu - 1;
    } else {
      pos = (int64_t)(R->dec_rr % (uint64_t)nu);
      R->dec_rr += 1;
    }
    R->res->decode_selects += 1;
    inst_t* I = &R->inst[ui[pos]];
    dp_t* D = &I->dp[ud[pos]];
    vpush(&D->residents, id); /* admit_decode (engine_model.cpp:145-151) */
    D->batch += 1;
    D->kv += R->prompt[id];
    R->status[id] = ST_DECODING;
    verase(&R->decode_wait, best);
    int seen = 0;
    for (int k = 0; k < nt; ++k) seen |= touched[k] == (int)ui[pos];
    if (!seen) touched[nt++] = (int)ui[pos];
  }
  free(ui); free(ud); free(ub); free(uk);
  for (int k = 0; k < nt; ++k) try_begin_step(R, touched[k]);
}

static void hand_off(run_t* R, const vec_t* fin) { /* simulation.cpp:397-411 */
  for (int64_t k = 0; k < fin->n; ++k) {
    int64_t id = fin->v[k];
    R->ftok[id] = R->clk.now;
    if (R->output[id] <= 1) { complete(R, id); continue; }
    vpush(&R->decode_wait, id);
  }
  drain_decode(R);
}

static void perform_dispatch(run_t* R, int i) { /* simulation.cpp:265-342 */
  inst_t* I = &R->inst[i];
  int64_t np = R->q_pending.n, nn = R->q_new.n, D = I->n_dp;
  int64_t* rows = (int64_t*)malloc(sizeof(int64_t) * 3 * (size_t)(np + nn + 1));
  for (int64_t k = 0; k < np + nn; ++k) {
    int64_t id = k < np ? R->q_pending.v[k] : R->q_new.v[k - np];
    rows[3 * k] = id; rows[3 * k + 1] = R->prompt[id]; rows[3 * k + 2] = R->wait[id];
  }
  int64_t* caps = (int64_t*)malloc(sizeof(int64_t) * (size_t)D);
  for (int d = 0; d < D; ++d) caps[d] = R->cfg->c_chunk - I->dp[d].u_flight - I->dp[d].r_queued;
  int64_t n = np + nn + 1;
  int64_t *om = (int64_t*)malloc(sizeof(int64_t) * 2 * (size_t)n), *od = (int64_t*)malloc(sizeof(int64_t) * 2 * (size_t)n),
          *ot = (int64_t*)malloc(sizeof(int64_t) * (size_t)n), cnt[3];
  /* cache-aware: Len_hit of every (request, DP) against the pre-dispatch
   * caches, used by the allocation and by the effective lengths below */
  int64_t* hits = NULL;
  if (R->cache_aware) {
    hits = (int64_t*)calloc((size_t)(n * D), sizeof(int64_t));
    for (int64_t k = 0; k < np + nn; ++k) {
      int64_t id = rows[3 * k];
      if (!R->pfx_pool || R->pfx_size[id] <= 0) continue;
      for (int d = 0; d < D; ++d)
        hits[k * D + d] = pc_longest_hit(&I->dp[d].cache, R->probes, R->n_probes, R->pfx_pool[id],
                                         R->pfx_size[id], R->prompt[id]);
    }
  }
  int flow = orc_allocate_batch_hits(rows, np, rows + 3 * np, nn, caps, D, R->cfg->n_limit, hits,
                                     om, od, ot, cnt);
  R->res->alloc_calls += 1;
  R->res->deferrals += (uint64_t)cnt[1];
  if (flow) R->res->flow_control_events += 1;
  for (int64_t k = 0; k < cnt[2]; ++k) R->status[ot[k]] = ST_THROTTLED;
  R->q_pending.n = 0;
  for (int64_t k = 0; k < cnt[1]; ++k) { vpush(&R->q_pending, od[2 * k]); R->wait[od[2 * k]] = (int)od[2 * k + 1]; }
  R->q_new.n = 0;
  if (cnt[0] == 0) {
    if (R->q_pending.n > 0) arm_tick(R, R->clk.now + R->i_opt);
  } else {
    for (int64_t k = 0; k < cnt[0]; ++k) {
      int64_t id = om[2 * k];
      int dsel = (int)om[2 * k + 1];
      int64_t hit = 0;
      if (hits)
        for (int64_t r = 0; r < np + nn; ++r)
          if (rows[3 * r] == id) { hit = hits[r * D + dsel]; break; }
      int64_t eff = R->prompt[id] - hit > 1 ? R->prompt[id] - hit : 1;
      R->status[id] = ST_DISPATCHED;
      R->disp[id] = R->clk.now;
      R->ctot[id] = eff;
      dispatch_prefill(R, i, dsel, id, eff);
      if (R->cache_aware && R->pfx_pool && R->pfx_size[id] > 0)
        pc_insert(&I->dp[dsel].cache, R->probes, R->n_probes, R->cfg->cache_budget_tokens,
                  R->pfx_pool[id], R->pfx_size[id], R->prompt[id]);
    }
    R->has_last = 1;
    R->last_dispatch = R->clk.now;
    R->last_inst = i;
    I->task_depth += 1;
    I->ef_seen = 0;
    I->wd_fired = 0;
    int64_t dl = R->clk.now + (int64_t)llround(R->cfg->watchdog_multiplier * (double)R->t_bar);
    I->wd_gen += 1;
    I->has_deadline = 1;
    I->deadline = dl;
    schedule(&R->clk, dl, EV_WD, i, I->wd_gen);
    maybe_die(R, i);
    try_start_pass(R, i);
    if (R->q_pending.n > 0) arm_tick(R, R->clk.now + R->i_opt);
  }
  free(rows); free(caps); free(om); free(od); free(ot); free(hits);
}

static int ready(run_t* R, int i) { /* interval_control.cpp:43-48 */
  inst_t* I = &R->inst[i];
  if (I->task_depth == 0 && !I->busy) return 1;
  if (I->ef_seen || I->wd_fired) return 1;
  return I->has_deadline && R->clk.now >= I->deadline;
}

static void try_dispatch(run_t* R) { /* simulation.cpp:245-263 */
  if (R->q_pending.n + R->q_new.n == 0) return;
  if (R->n_active <= 0) return;
  int64_t now = R->clk.now;
  if (R->has_last && now < R->last_dispatch + R->i_opt) { arm_tick(R, R->last_dispatch + R->i_opt); return; }
  int target = -1;
  for (int i = 0; i < R->P; ++i) if (R->inst[i].healthy && i > R->last_inst) { target = i; break; }
  if (target < 0) for (int i = 0; i < R->P; ++i) if (R->inst[i].healthy) { target = i; break; }
  if (target < 0 || !ready(R, target)) { arm_tick(R, now + R->i_opt); return; }
  perform_dispatch(R, target);
}

static void baseline_dispatch(run_t* R, int64_t id) { /* simulation.cpp:206-223, baselines.cpp */
  int tp = -1, td = -1;
  if (R->cfg->policy == 3) {
    int64_t bl = 0;
    for (int i = 0; i < R->P; ++i) {
      inst_t* I = &R->inst[i];
      if (!I->healthy || I->dead) continue;
      for (int d = 0; d < I->n_dp; ++d) {
        int64_t l = I->dp[d].u_flight + I->dp[d].r_queued;
        if (tp < 0 || l < bl) { tp = i; td = d; bl = l; }
      }
    }
  } else {
    for (int t = 0; t < R->P; ++t) {
      int pos = R->rr_next % R->P;
      R->rr_next = (pos + 1) % R->P;
      inst_t* I = &R->inst[pos];
      if (!I->healthy || I->dead) continue;
      int dp = R->rr_dp[pos] % I->n_dp;
      R->rr_dp[pos] = (dp + 1) % I->n_dp;
      tp = pos; td = dp;
      break;
    }
  }
  if (tp < 0) return;
  R->status[id] = ST_DISPATCHED;
  R->disp[id] = R->clk.now;
  R->ctot[id] = R->prompt[id];
  dispatch_prefill(R, tp, td, id, R->prompt[id]);
  maybe_die(R, tp);
  try_start_pass(R, tp);
}

static void on_end_forward(run_t* R, int i, uint64_t pseq) { /* simulation.cpp:346-372 */
  inst_t* I = &R->inst[i];
  maybe_die(R, i);
  if (I->dead) return;
  if (!I->busy || pseq != I->pass_seq) return;
  int64_t measured = R->clk.now - I->pass_started;
  vec_t fin = {0, 0, 0};
  for (int d = 0; d < I->n_dp; ++d) { /* finish_prefill_pass (engine_model.cpp:118-141) */
    dp_t* D = &I->dp[d];
    for (int64_t k = 0; k < D->pass_id.n; ++k) {
      int64_t id = D->pass_id.v[k];
      R->cdone[id] += D->pass_tok.v[k];
      if (R->cdone[id] > R->ctot[id]) R->error = 3;
      if (R->cdone[id] == R->ctot[id]) vpush(&fin, id);
    }
    D->pass_id.n = 0;
    D->pass_tok.n = 0;
  }
  I->busy = 0;
  hand_off(R, &fin);
  free(fin.v);
  try_start_pass(R, i);
  if (R->cfg->policy != 0) return;
  if (drop_matches(R, i)) { R->res->dropped_end_forwards += 1; return; }
  if (measured <= 0) { /* on_end_forward_sample (interval_control.cpp:26-36) */
    R->rejected += 1;
  } else {
    if (R->win_n < R->cfg->w_size) {
      R->win[(R->win_head + R->win_n) % R->cfg->w_size] = measured;
      R->win_n += 1;
    } else {
      R->win[R->win_head] = measured;
      R->win_head = (R->win_head + 1) % R->cfg->w_size;
    }
    recompute_interval(R);
  }
  I->task_depth = I->task_depth > 0 ? I->task_depth - 1 : 0;
  I->ef_seen = 1;
  I->wd_gen += 1; /* disarm_watchdog */
  I->has_deadline = 0;
  try_dispatch(R);
}

static void on_decode_step(run_t* R, int i, uint64_t sseq) { /* simulation.cpp:497-512 */
  inst_t* I = &R->inst[i];
  maybe_die(R, i);
  if (I->dead) return;
  if (!I->stepping || sseq != I->step_seq) return;
  int64_t gen = 0, tps = R->cfg->decode_tokens_per_step;
  for (int d = 0; d < I->n_dp; ++d) { /* finish_decode_step (engine_model.cpp:181-217) */
    dp_t* D = &I->dp[d];
    for (int64_t k = 0; k < D->residents.n;) {
      int64_t id = D->residents.v[k];
      if (R->mark[id] != I->step_seq) { ++k; continue; }
      int64_t target = R->output[id] > 0 ? R->output[id] - 1 : 0;
      int64_t pr = target - R->ddone[id] < tps ? target - R->ddone[id] : tps;
      R->ddone[id] += pr;
      D->kv += pr;
      gen += pr;
      if (R->ddone[id] == target) {
        complete(R, id);
        D->batch -= 1;
        D->kv -= R->prompt[id] + R->ddone[id];
        verase(&D->residents, k);
        continue;
      }
      ++k;
    }
  }
  I->stepping = 0;
  if (R->clk.now >= R->warmup) { R->steps += 1; R->out_tok += gen; }
  /* record_kv_snapshot (simulation.cpp:486-495) -> kv_band (metrics.cpp:50-72) */
  int64_t cnt = 0;
  double sum = 0.0;
  for (int j = R->P; j < R->n_inst; ++j) {
    inst_t* J = &R->inst[j];
    if (!J->healthy || J->dead) continue;
    for (int d = 0; d < J->n_dp; ++d) { sum += (double)J->dp[d].kv; cnt += 1; }
  }
  if (cnt > 0 && R->clk.now >= R->warmup) {
    double mean = sum / (double)cnt, var = 0.0;
    for (int j = R->P; j < R->n_inst; ++j) {
      inst_t* J = &R->inst[j];
      if (!J->healthy || J->dead) continue;
      for (int d = 0; d < J->n_dp; ++d) { double dv = (double)J->dp[d].kv - mean; var += dv * dv; }
    }
    R->kv_mean_sum += mean;
    R->kv_sig_sum += sqrt(var / (double)cnt);
    R->kv_n += 1;
  }
  drain_decode(R);
  try_begin_step(R, i);
}

static int cmp_f64(const void* a, const void* b) {
  double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}

static int cmp_i64(const void* a, const void* b) {
  int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return (x > y) - (x < y);
}

int orc_run(const orc_config* cfg, const int64_t* arr, const int32_t* prompt,
            const int32_t* output, int64_t n, orc_result* res, int64_t* per_req) {
  return orc_run_prefix(cfg, arr, prompt, output, NULL, NULL, n, res, per_req);
}

int orc_run_prefix(const orc_config* cfg, const int64_t* arr, const int32_t* prompt,
                   const int32_t* output, const int32_t* pfx_pool, const int32_t* pfx_size,
                   int64_t n, orc_result* res, int64_t* per_req) {
  run_t R;
  memset(&R, 0, sizeof(R));
  memset(res, 0, sizeof(*res));
  R.cfg = cfg; R.n = n; R.arr = arr; R.prompt = prompt; R.output = output; R.res = res;
  R.pfx_pool = pfx_pool;
  R.pfx_size = pfx_size;
  /* simulation.cpp:267-268 */
  R.cache_aware = cfg->prefill_mode == 1 && cfg->cache_enabled;
  if (R.cache_aware) {
    R.n_probes = cfg->n_probe_lens;
    R.probes = (int64_t*)malloc(sizeof(int64_t) * (size_t)(R.n_probes + 1));
    memcpy(R.probes, cfg->cache_probe_lens, sizeof(int64_t) * (size_t)R.n_probes);
    qsort(R.probes, (size_t)R.n_probes, sizeof(int64_t), cmp_i64);
  }
  R.P = cfg->n_instances_prefill;
  R.Dn = cfg->n_instances_decode;
  R.n_inst = R.P + R.Dn;
  int dd = cfg->dp_degree_decode > 0 ? cfg->dp_degree_decode : cfg->dp_degree;
  R.inst = (inst_t*)calloc((size_t)R.n_inst, sizeof(inst_t));
  for (int i = 0; i < R.n_inst; ++i) {
    R.inst[i].healthy = 1;
    R.inst[i].death = INF64;
    R.inst[i].n_dp = i < R.P ? cfg->dp_degree : dd;
    R.inst[i].dp = (dp_t*)calloc((size_t)R.inst[i].n_dp, sizeof(dp_t));
  }
  for (int k = 0; k < cfg->n_deads; ++k) { /* setup_faults (simulation.cpp:93-104) */
    int64_t t = s2ns(cfg->deads[k].time_s);
    inst_t* I = &R.inst[cfg->deads[k].instance];
    if (t < I->death) I->death = t;
  }
  for (int k = 0; k < cfg->n_topology; ++k)
    schedule(&R.clk, s2ns(cfg->topology[k].time_s), EV_TOPO, cfg->topology[k].instance,
             (uint64_t)cfg->topology[k].healthy);
  R.status = (int8_t*)calloc((size_t)n + 1, 1);
  R.wait = (int*)calloc((size_t)n + 1, sizeof(int));
  int64_t** cols[] = {&R.disp, &R.pstart, &R.ftok, &R.comp};
  for (int c = 0; c < 4; ++c) {
    *cols[c] = (int64_t*)malloc(sizeof(int64_t) * ((size_t)n + 1));
    for (int64_t k = 0; k < n; ++k) (*cols[c])[k] = -1;
  }
  R.ctot = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  R.cdone = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  R.ddone = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  R.mark = (uint64_t*)calloc((size_t)n + 1, sizeof(uint64_t));
  R.win = (int64_t*)calloc((size_t)cfg->w_size + 1, sizeof(int64_t));
  R.rr_dp = (int*)calloc((size_t)R.P, sizeof(int));
  R.t_default = s2ns(cfg->t_default_s); /* new_cluster (core.cpp:162-168) */
  R.t_bar = R.t_default;
  R.l_net = s2ns(cfg->l_net_s);
  R.n_active = R.P;
  R.i_opt = (R.t_bar + R.l_net) / R.n_active;
  R.last_inst = -1;
  mt_seed(&R.rng, cfg->seed ^ 0x9E3779B97F4A7C15ULL);
  R.horizon = s2ns(cfg->duration_s);
  R.warmup = s2ns(cfg->duration_s * cfg->warmup_fraction);
  for (int64_t k = 0; k < n; ++k) schedule(&R.clk, arr[k], EV_ARR, 0, (uint64_t)k);
  /* run_until (simclock.cpp:32-45) */
  while (R.clk.n > 0 && R.clk.v[0].t <= R.horizon && !R.error) {
    ev_t e = pop(&R.clk);
    R.clk.now = e.t;
    switch (e.kind) {
      case EV_ARR:
        if (cfg->policy == 0) { vpush(&R.q_new, (int64_t)e.b); try_dispatch(&R); }
        else baseline_dispatch(&R, (int64_t)e.b);
        break;
      case EV_TICK:
        if (e.b == R.tick_gen) try_dispatch(&R);
        break;
      case EV_EF: on_end_forward(&R, e.a, e.b); break;
      case EV_WD: {
        inst_t* I = &R.inst[e.a];
        if (e.b != I->wd_gen) break; /* watchdog_expired (interval_control.cpp:93-99) */
        I->wd_fired = 1;
        I->task_depth = 0;
        I->has_deadline = 0;
        res->watchdog_fires += 1;
        if (cfg->policy == 0) try_dispatch(&R);
        break;
      }
      case EV_TOPO: {
        R.inst[e.a].healthy = (int)e.b;
        int na = 0;
        for (int i = 0; i < R.P; ++i) na += R.inst[i].healthy;
        if (cfg->policy != 0) break;
        R.n_active = na;
        recompute_interval(&R);
        try_dispatch(&R);
        break;
      }
      case EV_DS: on_decode_step(&R, e.a, e.b); break;
    }
  }
  if (R.clk.bad) R.error = 3;
  /* finalize (metrics.cpp:103-190) */
  double* tt = (double*)malloc(sizeof(double) * ((size_t)n + 1));
  int64_t nt = 0, cw = 0;
  double ts = 0, ss = 0, ds = 0;
  for (int64_t k = 0; k < n; ++k) {
    res->generated += 1;
    if (R.status[k] == ST_THROTTLED) continue;
    if (R.status[k] != ST_COMPLETED) { res->in_flight += 1; continue; }
    res->completed += 1;
    if (R.comp[k] >= R.warmup) cw += 1;
    if (arr[k] < R.warmup) continue;
    res->window_requests += 1;
    double t = (double)(R.ftok[k] - arr[k]) / 1e9, s = (double)(R.disp[k] - arr[k]) / 1e9,
           d = (double)(R.pstart[k] - R.disp[k]) / 1e9;
    tt[nt++] = t;
    ts += t; ss += s; ds += d;
  }
  res->throttled = res->generated - res->completed - res->in_flight;
  if (nt > 0) {
    double m = (double)nt;
    res->ttft_mean_s = ts / m;
    res->scheduler_wait_mean_s = ss / m;
    res->device_wait_mean_s = ds / m;
    res->total_wait_mean_s = (ss + ds) / m;
    res->ttft_p50_s = orc_percentile(tt, nt, 50.0);
    res->ttft_p95_s = orc_percentile(tt, nt, 95.0);
  }
  free(tt);
  res->passes = (uint64_t)R.passes;
  if (R.passes > 0) res->chunk_util_mean = R.util_sum / (double)R.passes;
  res->decode_steps = (uint64_t)R.steps;
  res->output_tokens = (uint64_t)R.out_tok;
  double window = (double)(R.horizon - R.warmup) / 1e9;
  if (window > 0) {
    res->output_tokens_per_s = (double)res->output_tokens / window;
    res->completed_per_s = (double)cw / window;
  }
  if (R.kv_n > 0) {
    res->kv_mean_time_avg = R.kv_mean_sum / (double)R.kv_n;
    res->kv_sigma_time_avg = R.kv_sig_sum / (double)R.kv_n;
  }
  res->rejected_samples = R.rejected;
  res->warmup_cutoff_s = (double)R.warmup / 1e9;
  res->duration_s = (double)R.horizon / 1e9;
  res->error = R.error;
  if (per_req)
    for (int64_t k = 0; k < n; ++k) {
      per_req[5 * k] = R.status[k];
      per_req[5 * k + 1] = R.disp[k];
      per_req[5 * k + 2] = R.pstart[k];
      per_req[5 * k + 3] = R.ftok[k];
      per_req[5 * k + 4] = R.comp[k];
    }
  /* free */
  for (int i = 0; i < R.n_inst; ++i) {
    for (int d = 0; d < R.inst[i].n_dp; ++d) {
      dp_t* D = &R.inst[i].dp[d];
      free(D->pending.id); free(D->pending.tok); free(D->pending.bl);
      free(D->residents.v); free(D->pass_id.v); free(D->pass_tok.v);
      free(D->cache.key); free(D->cache.k);
    }
    free(R.inst[i].dp);
  }
  free(R.inst); free(R.status); free(R.wait); free(R.disp); free(R.pstart); free(R.ftok);
  free(R.comp); free(R.ctot); free(R.cdone); free(R.ddone); free(R.mark); free(R.win);
  free(R.probes);
  free(R.rr_dp); free(R.clk.v); free(R.q_pending.v); free(R.q_new.v); free(R.decode_wait.v);
  (void)cmp_u64; (void)cmp_f64;
  return R.error;
}
