/*
 * symoracle.c -- TEST INFRASTRUCTURE ONLY (parity checker / CPU baseline).
 *
 * A plain-C restatement of the reference's sequential event loop: one binary
 * heap ordered by (tick, prio, seq) with stale entries left in place, exactly
 * as batchsym/simulator.py:191-272 does, driving the two scheduler planes of
 * batchsym/scheduler.py.  The three sortedcontainers.SortedList indices of
 * RankPlane (scheduler.py:338-341) are replaced by indexed binary heaps; the
 * reference only ever reads their first/last element and removes/inserts
 * exact tuples, and all keys are unique (ids break ties), so the observable
 * behaviour is identical.
 *
 * Every function cites the reference lines it restates.  Paths are relative
 * to the reference package root pkg/src/batchsym/.
 */
#include "symoracle.h"

#include <stdlib.h>
#include <string.h>

#define NEG_INF (-(INT64_C(1) << 62)) /* units.py:17 */
#define OUTSTANDING (-1)              /* scheduler.py:41 */

enum { EV_COMPLETION = 0, EV_GPU_TIMER = 1, EV_MODEL_TIMER = 2,
       EV_DROP_TIMER = 3, EV_ARRIVAL = 4 }; /* simulator.py:29-33 */
enum { OUT_COMPLETED = 0, OUT_LATE = 1, OUT_DROPPED = 2 }; /* simulator.py:35-37 */
enum { DROP_DEADLINE = 0, DROP_POLICY = 1 };                /* scheduler.py:46-47 */

/* ---------------------------------------------------------------- utils */

#define GROW(ptr, cap, need)                                               \
  do {                                                                     \
    if ((need) > (cap)) {                                                  \
      int64_t nc_ = (cap) ? (cap) * 2 : 64;                                \
      while (nc_ < (need)) nc_ *= 2;                                       \
      void *np_ = realloc((ptr), (size_t)nc_ * sizeof(*(ptr)));            \
      if (!np_) return SYMO_ENOMEM;                                        \
      (ptr) = np_;                                                         \
      (cap) = nc_;                                                         \
    }                                                                      \
  } while (0)

static inline int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }

/* ------------------------------------------ numpy Philox4x64-10 stream -- */
/* numpy.random.Philox with an explicit key: counter starts at 0 and is
 * incremented before each block of 4 words; random() is (u64 >> 11) * 2^-53
 * and choice(vals, p) is vals[searchsorted(cumsum(p)/sum, u, 'right')]
 * (numpy _generator.pyx choice / philox.h; verified against numpy by
 * tests/test_oracle_golden.py::test_philox_stream_matches_numpy). */

typedef struct {
  uint64_t key[2];
  uint64_t ctr;
  uint64_t buf[4];
  int pos;
} philox_t;

static void philox_block(uint64_t ctr, const uint64_t key[2], uint64_t out[4]) {
  uint64_t c0 = ctr, c1 = 0, c2 = 0, c3 = 0, k0 = key[0], k1 = key[1];
  for (int r = 0; r < 10; r++) {
    if (r) {
      k0 += UINT64_C(0x9E3779B97F4A7C15);
      k1 += UINT64_C(0xBB67AE8584CAA73B);
    }
    __uint128_t p0 = (__uint128_t)UINT64_C(0xD2E7470EE14C6C93) * c0;
    __uint128_t p1 = (__uint128_t)UINT64_C(0xCA5A826395121157) * c2;
    uint64_t hi0 = (uint64_t)(p0 >> 64), lo0 = (uint64_t)p0;
    uint64_t hi1 = (uint64_t)(p1 >> 64), lo1 = (uint64_t)p1;
    uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

static double philox_random(philox_t *g) {
  if (g->pos >= 4) {
    g->ctr += 1;
    philox_block(g->ctr, g->key, g->buf);
    g->pos = 0;
  }
  return (double)(g->buf[g->pos++] >> 11) * (1.0 / 9007199254740992.0);
}

static int64_t choice_draw(philox_t *g, int32_t n, const int64_t *vals,
                           const double *cdf) {
  double u = philox_random(g);
  int32_t lo = 0, hi = n; /* number of cdf entries <= u */
  while (lo < hi) {
    int32_t mid = (lo + hi) / 2;
    if (cdf[mid] <= u)
      lo = mid + 1;
    else
      hi = mid;
  }
  return vals[lo < n ? lo : n - 1];
}

/* ------------------------------------------------------ event heap (L3) */

typedef struct {
  int64_t tick;
  int64_t seq;
  int32_t prio;
  int32_t id;   /* mid / gid / order index */
  int32_t size;
  int32_t _pad;
  int64_t gen;
  int64_t exec_at, latest;
} ev_t;

static inline int ev_less(const ev_t *a, const ev_t *b) {
  if (a->tick != b->tick) return a->tick < b->tick;
  if (a->prio != b->prio) return a->prio < b->prio;
  return a->seq < b->seq;
}

typedef struct {
  ev_t *v;
  int64_t n, cap;
} evheap_t;

static int evheap_push(evheap_t *h, ev_t e) {
  GROW(h->v, h->cap, h->n + 1);
  int64_t i = h->n++;
  while (i > 0) {
    int64_t p = (i - 1) >> 1;
    if (!ev_less(&e, &h->v[p])) break;
    h->v[i] = h->v[p];
    i = p;
  }
  h->v[i] = e;
  return SYMO_OK;
}

static ev_t evheap_pop(evheap_t *h) {
  ev_t top = h->v[0];
  ev_t last = h->v[--h->n];
  int64_t i = 0, n = h->n;
  for (;;) {
    int64_t c = 2 * i + 1;
    if (c >= n) break;
    if (c + 1 < n && ev_less(&h->v[c + 1], &h->v[c])) c++;
    if (!ev_less(&h->v[c], &last)) break;
    h->v[i] = h->v[c];
    i = c;
  }
  if (n > 0) h->v[i] = last;
  return top;
}

/* ------------------------- indexed heap standing in for a SortedList ---- */
/* Items are ids 0..cap-1 with key (k, id).  sign=+1: min at top (free_idx,
 * mc_by_latest); sign=-1: max at top (mc_by_bs, whose last element is read). */

typedef struct {
  int32_t *heap; /* heap position -> id */
  int32_t *pos;  /* id -> heap position, -1 if absent */
  int64_t *key;  /* id -> k */
  int32_t n;
  int32_t sign;
} ixheap_t;

static inline int ix_before(const ixheap_t *h, int32_t a, int32_t b) {
  int64_t ka = h->key[a], kb = h->key[b];
  if (h->sign > 0) return ka != kb ? ka < kb : a < b;
  return ka != kb ? ka > kb : a > b;
}

static void ix_up(ixheap_t *h, int32_t i) {
  int32_t id = h->heap[i];
  while (i > 0) {
    int32_t p = (i - 1) >> 1;
    if (!ix_before(h, id, h->heap[p])) break;
    h->heap[i] = h->heap[p];
    h->pos[h->heap[i]] = i;
    i = p;
  }
  h->heap[i] = id;
  h->pos[id] = i;
}

static void ix_down(ixheap_t *h, int32_t i) {
  int32_t id = h->heap[i];
  for (;;) {
    int32_t c = 2 * i + 1;
    if (c >= h->n) break;
    if (c + 1 < h->n && ix_before(h, h->heap[c + 1], h->heap[c])) c++;
    if (!ix_before(h, h->heap[c], id)) break;
    h->heap[i] = h->heap[c];
    h->pos[h->heap[i]] = i;
    i = c;
  }
  h->heap[i] = id;
  h->pos[id] = i;
}

static int ix_init(ixheap_t *h, int32_t cap, int32_t sign) {
  h->heap = malloc(sizeof(int32_t) * (size_t)(cap > 0 ? cap : 1));
  h->pos = malloc(sizeof(int32_t) * (size_t)(cap > 0 ? cap : 1));
  h->key = malloc(sizeof(int64_t) * (size_t)(cap > 0 ? cap : 1));
  if (!h->heap || !h->pos || !h->key) return SYMO_ENOMEM;
  for (int32_t i = 0; i < cap; i++) h->pos[i] = -1;
  h->n = 0;
  h->sign = sign;
  return SYMO_OK;
}

static void ix_free(ixheap_t *h) {
  free(h->heap);
  free(h->pos);
  free(h->key);
}

static void ix_add(ixheap_t *h, int32_t id, int64_t k) {
  h->key[id] = k;
  h->heap[h->n] = id;
  h->pos[id] = h->n;
  h->n++;
  ix_up(h, h->n - 1);
}

static void ix_remove(ixheap_t *h, int32_t id) {
  int32_t i = h->pos[id];
  int32_t last = h->heap[--h->n];
  h->pos[id] = -1;
  if (i == h->n) return;
  h->heap[i] = last;
  h->pos[last] = i;
  ix_up(h, i);
  ix_down(h, h->pos[last]);
}

static inline int32_t ix_top(const ixheap_t *h) { return h->heap[0]; }

/* ------------------------------------------------------------ state ---- */

typedef struct {
  /* ModelPlane fields (scheduler.py:142-164) */
  const int64_t *lat;
  int32_t max_batch, target_batch;
  int64_t slo, timeout_ns;
  int64_t qbase, qh, qt; /* queue = qbuf[qbase+qh .. qbase+qt) */
  int has_cand;
  int32_t c_size;
  int64_t c_exec, c_latest, c_head_deadline, c_head_rid;
  int64_t drop_gen, armed_drop_rid, drops;
} model_t;

typedef struct {
  const symo_config *cfg;
  const int64_t *arr_ticks, *arr_midx;
  int64_t n;
  /* request records (simulator.py:124-131); index = rid - 1 */
  int64_t *arrival, *deadline;
  int32_t *model;
  symo_result *out;
  int64_t *qbuf;
  model_t *m;
  /* RankPlane (scheduler.py:328-347) */
  int64_t *free_at;
  ixheap_t free_idx, mc_by_latest, mc_by_bs;
  int32_t *mc_has, *mc_size;
  int64_t *mc_exec, *mc_latest;
  int64_t *model_gen;
  int64_t gpu_gen;
  int armed_gpu;
  int64_t armed_fire;
  int32_t armed_gid;
  int64_t ops, evictions, registrations;
  /* EmulatedGpu (simulator.py:46-62) */
  int64_t *busy_until;
  /* engine (simulator.py:110-140) */
  int64_t now, seq;
  evheap_t heap;
  int64_t n_arrivals, n_queued, n_inflight, n_completed, n_dropped;
  int64_t handler_ops_max;
  /* orders */
  int64_t ord_cap, ord_mem_cap;
  int64_t *ord_mem_off, *ord_mem; /* member rids per order */
  int64_t tr_cap, tr_rid_cap;
  int err;
  int jitter;
  philox_t net;
} sim_t;

/* ------------------------------------------------- host callbacks ------ */

static int push_ev(sim_t *s, int64_t tick, int32_t prio, int32_t id,
                   int64_t gen, int32_t size, int64_t exec_at,
                   int64_t latest) {
  /* simulator.py:191-193 */
  ev_t e;
  memset(&e, 0, sizeof e);
  s->seq++;
  e.tick = tick;
  e.prio = prio;
  e.seq = s->seq;
  e.id = id;
  e.gen = gen;
  e.size = size;
  e.exec_at = exec_at;
  e.latest = latest;
  s->out->events_pushed++;
  return evheap_push(&s->heap, e);
}

static int trace_add(sim_t *s, int64_t t, int32_t kind, int32_t mid,
                     int32_t gid, int32_t size, int64_t start, int64_t finish,
                     const int64_t *rids, int64_t nrids) {
  symo_result *o = s->out;
  int64_t k = o->n_trace;
  if (k + 1 > s->tr_cap) {
    int64_t nc = s->tr_cap ? s->tr_cap * 2 : 256;
    o->tr_t = realloc(o->tr_t, sizeof(int64_t) * nc);
    o->tr_start = realloc(o->tr_start, sizeof(int64_t) * nc);
    o->tr_finish = realloc(o->tr_finish, sizeof(int64_t) * nc);
    o->tr_kind = realloc(o->tr_kind, sizeof(int32_t) * nc);
    o->tr_model = realloc(o->tr_model, sizeof(int32_t) * nc);
    o->tr_gpu = realloc(o->tr_gpu, sizeof(int32_t) * nc);
    o->tr_size = realloc(o->tr_size, sizeof(int32_t) * nc);
    o->tr_rid_off = realloc(o->tr_rid_off, sizeof(int64_t) * (nc + 1));
    if (!o->tr_t || !o->tr_start || !o->tr_finish || !o->tr_kind ||
        !o->tr_model || !o->tr_gpu || !o->tr_size || !o->tr_rid_off)
      return SYMO_ENOMEM;
    if (k == 0) o->tr_rid_off[0] = 0;
    s->tr_cap = nc;
  }
  int64_t base = o->tr_rid_off[k];
  GROW(o->tr_rids, s->tr_rid_cap, base + nrids);
  memcpy(o->tr_rids + base, rids, sizeof(int64_t) * (size_t)nrids);
  o->tr_t[k] = t;
  o->tr_kind[k] = kind;
  o->tr_model[k] = mid;
  o->tr_gpu[k] = gid;
  o->tr_size[k] = size;
  o->tr_start[k] = start;
  o->tr_finish[k] = finish;
  o->tr_rid_off[k + 1] = base + nrids;
  o->n_trace = k + 1;
  return SYMO_OK;
}

/* simulator.py:175-182 */
static int record_drop(sim_t *s, int64_t rid, int64_t now) {
  int64_t i = rid - 1;
  s->out->req_outcome[i] = OUT_DROPPED;
  s->n_queued -= 1;
  s->n_dropped += 1;
  if (s->cfg->record_trace)
    return trace_add(s, now, SYMO_TR_DROP, s->model[i], -1, 0, -1, -1, &rid,
                     1);
  return SYMO_OK;
}

/* simulator.py:184-187 */
static int record_shrink(sim_t *s, int32_t mid, int32_t gid, int32_t size,
                         int64_t now) {
  if (s->cfg->record_trace)
    return trace_add(s, now, SYMO_TR_SHRINK, mid, gid, size, -1, -1, NULL, 0);
  return SYMO_OK;
}

/* simulator.py:159-173 with EmulatedGpu.execute (simulator.py:54-62) */
static int emit_order(sim_t *s, int32_t gid, int32_t mid, int32_t b,
                      int64_t start, int64_t finish, int64_t emitted,
                      const int64_t *rids) {
  symo_result *o = s->out;
  if (start < s->busy_until[gid]) { /* only under jitter */
    int64_t shift = s->busy_until[gid] - start;
    start += shift;
    finish += shift;
  }
  s->busy_until[gid] = finish;
  int64_t k = o->n_orders;
  if (k + 1 > s->ord_cap) {
    int64_t nc = s->ord_cap ? s->ord_cap * 2 : 256;
    o->ord_gpu = realloc(o->ord_gpu, sizeof(int32_t) * nc);
    o->ord_model = realloc(o->ord_model, sizeof(int32_t) * nc);
    o->ord_size = realloc(o->ord_size, sizeof(int32_t) * nc);
    o->ord_start = realloc(o->ord_start, sizeof(int64_t) * nc);
    o->ord_finish = realloc(o->ord_finish, sizeof(int64_t) * nc);
    o->ord_emitted = realloc(o->ord_emitted, sizeof(int64_t) * nc);
    s->ord_mem_off = realloc(s->ord_mem_off, sizeof(int64_t) * (nc + 1));
    if (!o->ord_gpu || !o->ord_model || !o->ord_size || !o->ord_start ||
        !o->ord_finish || !o->ord_emitted || !s->ord_mem_off)
      return SYMO_ENOMEM;
    if (k == 0) s->ord_mem_off[0] = 0;
    s->ord_cap = nc;
  }
  int64_t base = s->ord_mem_off[k];
  GROW(s->ord_mem, s->ord_mem_cap, base + b);
  memcpy(s->ord_mem + base, rids, sizeof(int64_t) * (size_t)b);
  s->ord_mem_off[k + 1] = base + b;
  o->ord_gpu[k] = gid;
  o->ord_model[k] = mid;
  o->ord_size[k] = b;
  o->ord_start[k] = start;
  o->ord_finish[k] = finish;
  o->ord_emitted[k] = emitted;
  o->n_orders = k + 1;
  s->n_queued -= b;
  s->n_inflight += b;
  for (int32_t j = 0; j < b; j++) {
    int64_t i = rids[j] - 1;
    o->req_dispatch[i] = emitted;
    o->req_start[i] = start;
    o->req_finish[i] = finish;
    o->req_batch[i] = b;
  }
  int rc = push_ev(s, finish, EV_COMPLETION, (int32_t)k, 0, b, 0, 0);
  if (rc) return rc;
  if (s->cfg->record_trace)
    return trace_add(s, emitted, SYMO_TR_DISPATCH, mid, gid, b, start, finish,
                     rids, b);
  return SYMO_OK;
}

/* ------------------------------------------------------- RankPlane ----- */

static int model_granted_gpu(sim_t *s, int32_t mid, int32_t gid,
                             int64_t gpu_free_at, int64_t now);

/* scheduler.py:430-436 */
static void rank_unregister(sim_t *s, int32_t mid) {
  if (s->mc_has[mid]) {
    s->mc_has[mid] = 0;
    ix_remove(&s->mc_by_latest, mid);
    ix_remove(&s->mc_by_bs, mid);
    s->ops += 2;
  }
}

/* scheduler.py:438-457 */
static int rank_set_gpu_timer(sim_t *s, int64_t now) {
  if (s->mc_by_latest.n == 0 || s->free_idx.n == 0) {
    if (s->armed_gpu) {
      s->armed_gpu = 0;
      s->gpu_gen += 1;
    }
    return SYMO_OK;
  }
  int32_t gid = ix_top(&s->free_idx);
  int64_t fa = s->free_at[gid];
  int32_t bm = ix_top(&s->mc_by_bs);
  int64_t size = s->mc_size[bm];
  s->ops += 2;
  int64_t fire = fa - (s->cfg->d_ctrl_ns + s->cfg->d_data_ns * size);
  if (fire < now) fire = now;
  if (s->armed_gpu && s->armed_fire == fire && s->armed_gid == gid)
    return SYMO_OK;
  s->armed_gpu = 1;
  s->armed_fire = fire;
  s->armed_gid = gid;
  s->gpu_gen += 1;
  return push_ev(s, fire, EV_GPU_TIMER, gid, s->gpu_gen, 0, 0, 0);
}

/* scheduler.py:354-365 */
static int rank_inform_candidate(sim_t *s, int32_t mid, int64_t now) {
  if (mid < 0 || mid >= s->cfg->n_models) return SYMO_EPROTO;
  model_t *p = &s->m[mid];
  s->model_gen[mid] += 1;
  rank_unregister(s, mid);
  if (p->has_cand) {
    int64_t fire =
        p->c_exec - (s->cfg->d_ctrl_ns + s->cfg->d_data_ns * p->c_size);
    if (fire < now) fire = now;
    return push_ev(s, fire, EV_MODEL_TIMER, mid, s->model_gen[mid], p->c_size,
                   p->c_exec, p->c_latest);
  }
  return SYMO_OK;
}

/* scheduler.py:367-377 */
static int rank_inform_gpu(sim_t *s, int32_t gid, int64_t free_at,
                           int64_t now) {
  if (gid < 0 || gid >= s->cfg->n_gpus) return SYMO_EPROTO;
  int64_t old = s->free_at[gid];
  if (old != OUTSTANDING) {
    ix_remove(&s->free_idx, gid);
    s->ops += 1;
  }
  s->free_at[gid] = free_at;
  ix_add(&s->free_idx, gid, free_at);
  s->ops += 1;
  return rank_set_gpu_timer(s, now);
}

/* scheduler.py:381-399 */
static int rank_on_model_timer(sim_t *s, const ev_t *e, int64_t now) {
  int32_t mid = e->id;
  if (e->gen != s->model_gen[mid]) return SYMO_OK;
  if (s->free_idx.n > 0) {
    int32_t gid = ix_top(&s->free_idx);
    int64_t fa = s->free_at[gid];
    s->ops += 1;
    if (fa <= e->exec_at) {
      ix_remove(&s->free_idx, gid);
      s->ops += 1;
      s->free_at[gid] = OUTSTANDING;
      return model_granted_gpu(s, mid, gid, fa, now);
    }
  }
  s->mc_has[mid] = 1;
  s->mc_size[mid] = e->size;
  s->mc_exec[mid] = e->exec_at;
  s->mc_latest[mid] = e->latest;
  ix_add(&s->mc_by_latest, mid, e->latest);
  ix_add(&s->mc_by_bs, mid, e->size);
  s->ops += 2;
  s->registrations += 1;
  return rank_set_gpu_timer(s, now);
}

/* scheduler.py:401-426 */
static int rank_on_gpu_timer(sim_t *s, const ev_t *e, int64_t now) {
  if (e->gen != s->gpu_gen) return SYMO_OK;
  s->armed_gpu = 0;
  int32_t gid = e->id;
  int64_t fa = s->free_at[gid];
  if (fa == OUTSTANDING) return rank_set_gpu_timer(s, now);
  while (s->mc_by_latest.n > 0 &&
         s->mc_latest[ix_top(&s->mc_by_latest)] < fa) {
    int32_t m = ix_top(&s->mc_by_latest);
    ix_remove(&s->mc_by_latest, m);
    ix_remove(&s->mc_by_bs, m);
    s->mc_has[m] = 0;
    s->ops += 2;
    s->evictions += 1;
  }
  if (s->mc_by_latest.n > 0) {
    int32_t m = ix_top(&s->mc_by_latest);
    s->ops += 1;
    rank_unregister(s, m);
    ix_remove(&s->free_idx, gid);
    s->ops += 1;
    s->free_at[gid] = OUTSTANDING;
    int rc = model_granted_gpu(s, m, gid, fa, now);
    if (rc) return rc;
  }
  return rank_set_gpu_timer(s, now);
}

/* ------------------------------------------------------ ModelPlane ----- */

static inline int64_t q_len(const model_t *p) { return p->qt - p->qh; }
static inline int64_t q_at(const sim_t *s, const model_t *p, int64_t k) {
  return s->qbuf[p->qbase + p->qh + k];
}

/* scheduler.py:213-216 */
static int model_drop_head(sim_t *s, model_t *p, int64_t now) {
  int64_t rid = q_at(s, p, 0);
  p->qh += 1;
  p->drops += 1;
  return record_drop(s, rid, now);
}

/* scheduler.py:301-315 */
static int model_arm_drop_timer(sim_t *s, int32_t mid, int64_t now) {
  model_t *p = &s->m[mid];
  if (q_len(p) == 0) {
    if (p->armed_drop_rid != -1) {
      p->armed_drop_rid = -1;
      p->drop_gen += 1;
    }
    return SYMO_OK;
  }
  int64_t head = q_at(s, p, 0);
  if (head == p->armed_drop_rid) return SYMO_OK;
  p->armed_drop_rid = head;
  p->drop_gen += 1;
  int64_t fire = s->deadline[head - 1] -
                 (s->cfg->d_ctrl_ns + s->cfg->d_data_ns + p->lat[0]) + 1;
  return push_ev(s, max64(fire, now), EV_DROP_TIMER, mid, p->drop_gen, 0, 0,
                 0);
}

/* scheduler.py:277-299 */
static int32_t model_max_feasible(const sim_t *s, const model_t *p,
                                  int64_t now, int64_t floor, int64_t cap,
                                  int64_t d) {
  const int64_t dc = s->cfg->d_ctrl_ns, dd = s->cfg->d_data_ns;
#define OK_(b) (max64(now + dc + dd * (b), floor) + p->lat[(b)-1] <= d)
  if (!OK_(1)) return 0;
  int64_t lo = 1, hi = cap;
  while (lo < hi) {
    int64_t mid = (lo + hi + 1) / 2;
    if (OK_(mid))
      lo = mid;
    else
      hi = mid - 1;
  }
#undef OK_
  return (int32_t)lo;
}

/* scheduler.py:218-275; *changed receives the return value */
static int model_update_candidate(sim_t *s, int32_t mid, int64_t now,
                                  int64_t gpu_floor, int *changed) {
  model_t *p = &s->m[mid];
  const symo_config *c = s->cfg;
  int rc;
  *changed = 0;
  int64_t base1 = c->d_ctrl_ns + c->d_data_ns + p->lat[0];
  while (q_len(p) > 0 && now + base1 > s->deadline[q_at(s, p, 0) - 1])
    if ((rc = model_drop_head(s, p, now))) return rc;
  if (c->kind == SYMO_TIMEOUT) {
    while (q_len(p) > 0) {
      int64_t h = q_at(s, p, 0) - 1;
      if (!(s->arrival[h] + p->timeout_ns + p->lat[0] > s->deadline[h])) break;
      if ((rc = model_drop_head(s, p, now))) return rc;
    }
  }
  if (c->gather == SYMO_GATHER_DROP_HEAD && q_len(p) > p->target_batch) {
    int64_t tb = p->target_batch;
    int64_t need = now + c->d_ctrl_ns + c->d_data_ns * tb + p->lat[tb - 1];
    while (q_len(p) > tb && need > s->deadline[q_at(s, p, 0) - 1])
      if ((rc = model_drop_head(s, p, now))) return rc;
  }
  if (q_len(p) == 0) {
    if ((rc = model_arm_drop_timer(s, mid, now))) return rc;
    if (p->has_cand) {
      p->has_cand = 0;
      *changed = 1;
    }
    return SYMO_OK;
  }
  int64_t head = q_at(s, p, 0);
  int64_t d = s->deadline[head - 1];
  int64_t cap = q_len(p) < p->max_batch ? q_len(p) : p->max_batch;
  if (c->gather == SYMO_GATHER_DROP_HEAD && p->target_batch < cap)
    cap = p->target_batch;
  int64_t pol_floor =
      c->kind == SYMO_TIMEOUT ? s->arrival[head - 1] + p->timeout_ns : NEG_INF;
  int64_t floor2 = max64(pol_floor, gpu_floor);
  int32_t b = model_max_feasible(s, p, now, floor2, cap, d);
  if (b == 0) {
    if ((rc = model_arm_drop_timer(s, mid, now))) return rc;
    if (p->has_cand) {
      p->has_cand = 0;
      *changed = 1;
    }
    return SYMO_OK;
  }
  int64_t l_next = b < p->max_batch ? p->lat[b] : p->lat[p->max_batch - 1];
  int64_t exec_at = now + c->d_ctrl_ns + c->d_data_ns * b;
  if (c->kind == SYMO_DEFERRED) {
    int64_t fr = d - l_next;
    if (fr > exec_at) exec_at = fr;
  }
  if (floor2 > exec_at) exec_at = floor2;
  int64_t latest = d - p->lat[b - 1];
  if ((rc = model_arm_drop_timer(s, mid, now))) return rc;
  if (p->has_cand && p->c_size == b && p->c_exec == exec_at &&
      p->c_latest == latest && p->c_head_rid == head)
    return SYMO_OK;
  p->has_cand = 1;
  p->c_size = b;
  p->c_exec = exec_at;
  p->c_latest = latest;
  p->c_head_deadline = d;
  p->c_head_rid = head;
  *changed = 1;
  return SYMO_OK;
}

/* scheduler.py:168-171 */
static int model_on_new_request(sim_t *s, int32_t mid, int64_t rid,
                                int64_t now) {
  model_t *p = &s->m[mid];
  s->qbuf[p->qbase + p->qt] = rid;
  p->qt += 1;
  int changed, rc;
  if ((rc = model_update_candidate(s, mid, now, NEG_INF, &changed))) return rc;
  if (changed) return rank_inform_candidate(s, mid, now);
  return SYMO_OK;
}

/* scheduler.py:173-178 */
static int model_on_drop_timer(sim_t *s, const ev_t *e, int64_t now) {
  model_t *p = &s->m[e->id];
  if (e->gen != p->drop_gen) return SYMO_OK;
  p->armed_drop_rid = -1;
  int changed, rc;
  if ((rc = model_update_candidate(s, e->id, now, NEG_INF, &changed)))
    return rc;
  if (changed) return rank_inform_candidate(s, e->id, now);
  return SYMO_OK;
}

/* scheduler.py:180-209 (jitterless: sample_dispatch_delay is None) */
static int model_granted_gpu(sim_t *s, int32_t mid, int32_t gid,
                             int64_t gpu_free_at, int64_t now) {
  model_t *p = &s->m[mid];
  int rc, changed;
  int32_t pre_size = p->has_cand ? p->c_size : 0;
  if ((rc = model_update_candidate(s, mid, now, max64(gpu_free_at, 0),
                                   &changed)))
    return rc;
  if (!p->has_cand) {
    if ((rc = rank_inform_gpu(s, gid, max64(now, gpu_free_at), now)))
      return rc;
    if ((rc = model_update_candidate(s, mid, now, NEG_INF, &changed)))
      return rc;
    return rank_inform_candidate(s, mid, now);
  }
  if (p->c_size < pre_size)
    if ((rc = record_shrink(s, mid, gid, p->c_size, now))) return rc;
  int32_t b = p->c_size;
  const int64_t *members = s->qbuf + p->qbase + p->qh;
  p->qh += b;
  int64_t start = p->c_exec;
  int64_t lat_b = p->lat[b - 1];
  if (s->jitter) { /* sample_dispatch_delay: ctrl() + data() * b */
    const symo_config *c = s->cfg;
    int64_t dctrl = c->net_ctrl_n ? choice_draw(&s->net, c->net_ctrl_n, c->net_ctrl_vals,
                                                c->net_ctrl_cdf)
                                  : c->net_ctrl_const;
    int64_t ddata = c->net_data_n ? choice_draw(&s->net, c->net_data_n, c->net_data_vals,
                                                c->net_data_cdf)
                                  : c->net_data_const;
    int64_t actual = dctrl + ddata * b;
    if (now + actual > start) start = now + actual;
  }
  if ((rc = emit_order(s, gid, mid, b, start, start + lat_b, now, members)))
    return rc;
  int64_t believed_free = p->c_exec + lat_b;
  p->has_cand = 0;
  if ((rc = model_update_candidate(s, mid, now, NEG_INF, &changed))) return rc;
  if ((rc = rank_inform_gpu(s, gid, believed_free, now))) return rc;
  return rank_inform_candidate(s, mid, now);
}

/* ------------------------------------------------------ engine loop ---- */

/* simulator.py:276-305 (the checks that are meaningful in this layout) */
static int verify(sim_t *s) {
  int64_t queued = 0;
  for (int32_t m = 0; m < s->cfg->n_models; m++) queued += q_len(&s->m[m]);
  if (queued != s->n_queued) return SYMO_EINVARIANT;
  if (s->n_arrivals !=
      s->n_completed + s->n_dropped + s->n_queued + s->n_inflight)
    return SYMO_EINVARIANT;
  for (int32_t g = 0; g < s->cfg->n_gpus; g++) {
    int in_idx = s->free_idx.pos[g] >= 0;
    if (s->free_at[g] == OUTSTANDING) return SYMO_EINVARIANT; /* both/outst. */
    if (!in_idx) return SYMO_EINVARIANT;                       /* lost */
  }
  if (s->mc_by_latest.n != s->mc_by_bs.n) return SYMO_EINVARIANT;
  for (int32_t m = 0; m < s->cfg->n_models; m++) {
    model_t *p = &s->m[m];
    if (!p->has_cand) continue;
    if (p->c_exec > p->c_latest) return SYMO_EINVARIANT;
    if (p->c_exec + p->lat[p->c_size - 1] > p->c_head_deadline)
      return SYMO_EINVARIANT;
  }
  return SYMO_OK;
}

/* simulator.py:244-272 */
static int dispatch_event(sim_t *s, const ev_t *e) {
  s->now = e->tick;
  int64_t ops0 = s->ops, ev0 = s->evictions;
  int rc = SYMO_OK;
  s->out->events_popped++;
  switch (e->prio) {
    case EV_COMPLETION: {
      symo_result *o = s->out;
      int64_t k = e->id;
      int32_t b = o->ord_size[k];
      s->n_inflight -= b;
      s->n_completed += b;
      for (int64_t j = s->ord_mem_off[k]; j < s->ord_mem_off[k + 1]; j++) {
        int64_t i = s->ord_mem[j] - 1;
        o->req_outcome[i] =
            o->ord_finish[k] <= s->deadline[i] ? OUT_COMPLETED : OUT_LATE;
      }
      break;
    }
    case EV_GPU_TIMER: rc = rank_on_gpu_timer(s, e, e->tick); break;
    case EV_MODEL_TIMER: rc = rank_on_model_timer(s, e, e->tick); break;
    case EV_DROP_TIMER: rc = model_on_drop_timer(s, e, e->tick); break;
  }
  int64_t ops = (s->ops - ops0) - 2 * (s->evictions - ev0);
  if (ops > s->handler_ops_max) s->handler_ops_max = ops;
  return rc;
}

static int run_stream(sim_t *s) {
  /* simulator.py:201-226 */
  const int64_t n = s->n;
  const int32_t M = s->cfg->n_models;
  int64_t i = 0;
  int rc;
  while (s->heap.n > 0 || i < n) {
    if (i < n) {
      int64_t at = s->arr_ticks[i];
      const ev_t *top = s->heap.n ? &s->heap.v[0] : NULL;
      if (top && (top->tick < at || (top->tick == at && top->prio <= EV_ARRIVAL))) {
        ev_t e = evheap_pop(&s->heap);
        if ((rc = dispatch_event(s, &e))) return rc;
      } else {
        int64_t midx = s->arr_midx[i];
        if (midx < 0 || midx >= M) {
          s->out->err_index = i;
          return SYMO_EPROTO;
        }
        i += 1;
        int64_t rid = s->n_arrivals + 1;
        s->now = at;
        /* _record_arrival (simulator.py:228-242) */
        s->n_arrivals += 1;
        s->n_queued += 1;
        s->model[rid - 1] = (int32_t)midx;
        s->arrival[rid - 1] = at;
        s->deadline[rid - 1] = at + s->m[midx].slo;
        if ((rc = model_on_new_request(s, (int32_t)midx, rid, at))) return rc;
      }
    } else {
      ev_t e = evheap_pop(&s->heap);
      if ((rc = dispatch_event(s, &e))) return rc;
    }
    if (s->cfg->check_invariants && (rc = verify(s))) return rc;
  }
  return SYMO_OK;
}

int32_t symo_run(const symo_config *cfg, const int64_t *arr_ticks,
                 const int64_t *arr_midx, int64_t n, symo_result *out) {
  if (!cfg || !out || n < 0 || cfg->n_gpus < 1 || cfg->n_models < 1)
    return SYMO_EINVAL;
  sim_t S;
  memset(&S, 0, sizeof S);
  sim_t *s = &S;
  int64_t keep_n = out->n;
  int64_t *kd = out->req_dispatch, *ks = out->req_start, *kf = out->req_finish,
          *kb = out->req_batch, *ko = out->req_outcome;
  memset(out, 0, sizeof *out);
  out->n = keep_n;
  out->req_dispatch = kd;
  out->req_start = ks;
  out->req_finish = kf;
  out->req_batch = kb;
  out->req_outcome = ko;
  out->err_index = -1;
  if (out->n != n) return SYMO_EINVAL;
  s->cfg = cfg;
  s->jitter = cfg->net_ctrl_n > 0 || cfg->net_data_n > 0;
  s->net.key[0] = cfg->net_key[0];
  s->net.key[1] = cfg->net_key[1];
  s->net.ctr = 0;
  s->net.pos = 4;
  s->arr_ticks = arr_ticks;
  s->arr_midx = arr_midx;
  s->n = n;
  s->out = out;
  const int32_t M = cfg->n_models, G = cfg->n_gpus;
  int rc = SYMO_ENOMEM;
  size_t nn = (size_t)(n > 0 ? n : 1);
  s->arrival = malloc(sizeof(int64_t) * nn);
  s->deadline = malloc(sizeof(int64_t) * nn);
  s->model = malloc(sizeof(int32_t) * nn);
  s->qbuf = malloc(sizeof(int64_t) * nn);
  s->m = calloc((size_t)M, sizeof(model_t));
  s->free_at = calloc((size_t)G, sizeof(int64_t));
  s->busy_until = calloc((size_t)G, sizeof(int64_t));
  s->mc_has = calloc((size_t)M, sizeof(int32_t));
  s->mc_size = calloc((size_t)M, sizeof(int32_t));
  s->mc_exec = calloc((size_t)M, sizeof(int64_t));
  s->mc_latest = calloc((size_t)M, sizeof(int64_t));
  s->model_gen = calloc((size_t)M, sizeof(int64_t));
  int64_t *cnt = calloc((size_t)M, sizeof(int64_t));
  if (!s->arrival || !s->deadline || !s->model || !s->qbuf || !s->m ||
      !s->free_at || !s->busy_until || !s->mc_has || !s->mc_size ||
      !s->mc_exec || !s->mc_latest || !s->model_gen || !cnt)
    goto done;
  if (ix_init(&s->free_idx, G, +1) || ix_init(&s->mc_by_latest, M, +1) ||
      ix_init(&s->mc_by_bs, M, -1))
    goto done;
  for (int64_t i = 0; i < n; i++) {
    int64_t mi = arr_midx[i];
    if (mi >= 0 && mi < M) cnt[mi]++;
    out->req_dispatch[i] = out->req_start[i] = out->req_finish[i] = -1;
    out->req_batch[i] = out->req_outcome[i] = -1;
  }
  int64_t off = 0;
  for (int32_t m = 0; m < M; m++) {
    model_t *p = &s->m[m];
    p->lat = cfg->lat_ns + (int64_t)m * cfg->lat_stride;
    p->max_batch = cfg->max_batch[m];
    if (p->max_batch < 1 || p->max_batch > cfg->lat_stride) {
      rc = SYMO_EINVAL;
      goto done;
    }
    p->target_batch = cfg->target_batch < p->max_batch ? cfg->target_batch
                                                       : p->max_batch;
    p->slo = cfg->slo_ns[m];
    p->timeout_ns = cfg->timeout_ns ? cfg->timeout_ns[m] : 0;
    p->qbase = off;
    p->armed_drop_rid = -1;
    off += cnt[m];
  }
  /* RankPlane.__init__: every GPU free at 0 (scheduler.py:337-338) */
  for (int32_t g = 0; g < G; g++) ix_add(&s->free_idx, g, 0);
  rc = run_stream(s);
  out->drops = s->n_dropped;
  out->completions = s->n_completed;
  int64_t late = 0;
  for (int64_t i = 0; i < n; i++) late += out->req_outcome[i] == OUT_LATE;
  out->late = late;
  out->ops = s->ops;
  out->evictions = s->evictions;
  out->registrations = s->registrations;
  out->handler_ops_max = s->handler_ops_max;
done:
  free(cnt);
  free(s->arrival);
  free(s->deadline);
  free(s->model);
  free(s->qbuf);
  free(s->m);
  free(s->free_at);
  free(s->busy_until);
  free(s->mc_has);
  free(s->mc_size);
  free(s->mc_exec);
  free(s->mc_latest);
  free(s->model_gen);
  free(s->ord_mem_off);
  free(s->ord_mem);
  free(s->heap.v);
  ix_free(&s->free_idx);
  ix_free(&s->mc_by_latest);
  ix_free(&s->mc_by_bs);
  return rc;
}

void symo_free_result(symo_result *o) {
  if (!o) return;
  free(o->ord_gpu);
  free(o->ord_model);
  free(o->ord_size);
  free(o->ord_start);
  free(o->ord_finish);
  free(o->ord_emitted);
  free(o->tr_t);
  free(o->tr_start);
  free(o->tr_finish);
  free(o->tr_kind);
  free(o->tr_model);
  free(o->tr_gpu);
  free(o->tr_size);
  free(o->tr_rid_off);
  free(o->tr_rids);
  o->ord_gpu = o->ord_model = o->ord_size = NULL;
  o->ord_start = o->ord_finish = o->ord_emitted = NULL;
  o->tr_t = o->tr_start = o->tr_finish = NULL;
  o->tr_kind = o->tr_model = o->tr_gpu = o->tr_size = NULL;
  o->tr_rid_off = o->tr_rids = NULL;
}
