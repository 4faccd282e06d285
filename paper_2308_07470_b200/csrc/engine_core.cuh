// engine_core.cuh -- the per-sub-cluster "live-event chain" of the B200
// scheduler engine.
//
// The reference (batchsym simulator.py:191-272) pushes one heap entry per
// candidate change (~1 per arrival) and discards 92-97 % of them as stale.
// This engine never materialises stale entries.  Each model keeps at most one
// live model timer, one live drop timer and its unabsorbed arrival suffix;
// arrivals of a model that is not registered at the rank plane only touch that
// model, so they are absorbed *locally* (ahead of global time) until the
// model's next event that reads or writes shared state.  Only those "chain
// events" -- live model-timer pops, live drop-timer pops, the live GPU timer,
// and arrivals of registered models -- are ordered globally.
//
// Exact ordering.  The reference orders heap entries by (tick, prio, seq)
// where seq is a global push counter, and merges arrival i when no entry with
// (tick, prio) <= (a_i, 4) remains (simulator.py:210).  We replace seq by an
// order-isomorphic key that can be computed without a global counter:
//   A   = number of arrivals processed before the event.  Processing order is
//         non-decreasing in (tick, A); an event pushed at an earlier tick has
//         A = L(tick) (#arrivals strictly before tick), stored canonically as
//         BASE (-1); an event pushed during a same-tick cascade inherits the
//         explicit A of its pusher (> L(tick)).
//   pusher position (tp, ap, sub): the processing position of the event that
//         pushed it.  Chain events take sub = a chain counter (monotone in
//         processing order); arrival g takes (a_g, A'_g, +inf) because it is
//         processed after every chain event at (a_g, A'_g).
// Two live events compare by (tick, A', prio, tp, ap, sub); DESIGN.md §3
// proves this is the reference's pop order among live events.
//
// Everything here is __host__ __device__ so tools/hostcheck can run the exact
// same chain on the CPU against the oracle while iterating; the product only
// ever runs it inside the CUDA kernels of engine.cu.
#pragma once
#include <stdint.h>

#ifndef SYM_HD
#ifdef __CUDACC__
#define SYM_HD __host__ __device__ __forceinline__
#else
#define SYM_HD inline
#endif
#endif

namespace sym {

// Dev-only cycle attribution of the chain (tools/chain_prof.py builds a
// separate library with -DSYM_CHAIN_PROF): [0..3] handler cycles by event
// type (MT, DT, ARR, GPU), [4..7] their counts, [8] dispatch, [9] refresh,
// [10] pq_update, [11] refreshed models, [12] update_candidate,
// [13] update_candidate calls, [14] scan_model, [15] set_gpu_timer.
#if defined(SYM_CHAIN_PROF) && defined(__CUDACC__)
__device__ unsigned long long g_chain_prof[16];
__device__ int g_chain_prof_on;  // set by k_chain only (other kernels share helpers)
#endif
#if defined(SYM_CHAIN_PROF) && defined(__CUDA_ARCH__)
#define SYM_PROF_T(v) const long long v = clock64()
#define SYM_PROF_ADD(i, x) \
  (g_chain_prof_on ? atomicAdd(&g_chain_prof[i], (unsigned long long)(x)) : 0ull)
#else
#define SYM_PROF_T(v)
#define SYM_PROF_ADD(i, x)
#endif

constexpr int64_t NEG_INF = -(int64_t(1) << 62);  // units.py:17
constexpr int64_t OUTSTANDING = -1;               // scheduler.py:41
constexpr int64_t FREE_SENTINEL = INT64_MAX;      // leaf absent from an index
constexpr int32_t A_BASE = -1;                    // canonical "A = L(tick)"
constexpr int64_t SUB_ARRIVAL = INT64_MAX;        // arrival pusher sub-rank

enum : int32_t { PR_GPU = 1, PR_MODEL = 2, PR_DROP = 3, PR_ARRIVAL = 4 };
enum : int32_t { EV_NONE = 0, EV_MT = 1, EV_DT = 2, EV_ARR = 3 };
enum : int32_t { K_DEFERRED = 0, K_EAGER = 1, K_TIMEOUT = 2 };
enum : int32_t { G_PREFIX = 0, G_DROP_HEAD = 1 };

struct EvKey {
  int64_t t;    // tick
  int64_t tp;   // pusher tick
  int64_t sub;  // pusher sub-rank (chain counter or SUB_ARRIVAL)
  int32_t a;    // canonical A'
  int32_t prio;
  int32_t ap;   // pusher A'
  int32_t _pad;
};

SYM_HD bool key_less(const EvKey& x, const EvKey& y) {
  if (x.t != y.t) return x.t < y.t;
  if (x.a != y.a) return x.a < y.a;
  if (x.prio != y.prio) return x.prio < y.prio;
  if (x.tp != y.tp) return x.tp < y.tp;
  if (x.ap != y.ap) return x.ap < y.ap;
  return x.sub < y.sub;
}

// Processing position of the event currently being handled; every push made
// while handling it is stamped with it.
struct Pusher {
  int64_t t;
  int64_t sub;
  int32_t a_self;   // A' of the pusher itself (ordering)
  int32_t a_after;  // A' inherited by a push at the same tick
};

SYM_HD EvKey push_key(int64_t fire, int32_t prio, const Pusher& P) {
  EvKey k;
  k.t = fire;
  k.a = (fire == P.t) ? P.a_after : A_BASE;
  k.prio = prio;
  k.tp = P.t;
  k.ap = P.a_self;
  k.sub = P.sub;
  k._pad = 0;
  return k;
}

// Static per-model parameters (ModelPlane.__init__, scheduler.py:147-164).
struct ModelParam {
  int64_t slo;
  int64_t timeout_ns;   // resolved (PolicyConfig.resolve_timeout_ns)
  int64_t base1;        // d_ctrl + d_data + l(1)
  int64_t aff_a, aff_b; // l(b) = aff_a * b + aff_b exactly, when affine != 0
  int32_t affine;       // the lat row is exactly affine in b (linear profiles)
  int32_t _pad;
  int32_t off;          // first position of this model in the sorted stream
  int32_t cnt;          // arrivals of this model
  int32_t max_batch;
  int32_t target_batch; // min(policy.target_batch, max_batch)
};

// Mutable per-model state.
struct ModelState {
  int64_t c_exec, c_latest;
  int64_t c_d;        // candidate head deadline
  int64_t c_lb;       // l(c_size)
  int64_t c_lb1;      // l(c_size+1), or l(max_batch) at the cap (l_next)
  EvKey mt_key;       // live model timer (valid iff has_mt)
  EvKey dt_key;       // live drop timer (valid iff dt_head >= 0)
  EvKey nx_key;       // next chain event of this model
  int64_t drops;
  int64_t qbase;      // arrivals compacted out of the layout by earlier steps
  int32_t qh, qt;     // queue = positions [off+qh, off+qt)
  int32_t has_cand, c_size;
  int32_t c_head;     // queue position of the candidate head (head rid)
  int32_t registered; // present in RankPlane.mc
  int32_t has_mt;
  int32_t dt_head;    // armed_drop_rid as a position, -1 = disarmed
  int32_t nx_type;    // EV_*
  int32_t fresh_skip; // performance only: fresh starts to scan before trying
                      // the adoption table again (refresh_model)
};

struct alignas(16) BatchRec {
  // the first 32 bytes are what the per-request results need (k_out reads
  // them as two 16-byte words)
  int64_t emitted, start, finish;
  int32_t size, model;
  int64_t kt, ksub;   // processing position of the granting event (trace)
  int32_t ka;
  int32_t gpu;
  int32_t first;      // sorted-stream position of the first member
  int32_t shrunk_from;// pre-grant candidate size if it shrank, else 0
};

// All arrays of one sub-cluster.  Pointers may target global or shared
// memory; the chain is written against this view only.
struct Shard {
  // configuration
  int32_t M, G, Mp, Gp;  // counts and power-of-two tree widths
  int32_t Mlog, Glog;    // log2(Mp), log2(Gp)
  int32_t kind, gather, record_trace, _pad;
  int64_t d_ctrl, d_data;
  int32_t lat_stride, _pad2;
  const int64_t* lat;          // [M * lat_stride]
  const ModelParam* mp;        // [M]
  // arrivals, sorted by (model, stream order)
  const int64_t* s_tick;       // [n] tick of sorted position p
  const int32_t* s_g;          // [n] shard-stream index of sorted position p
  const int64_t* sh_tick;      // [n] ticks in shard-stream order (for A')
  const int32_t* s_aself;      // [n] A' of sorted position p, precomputed
                               // (stepped runs); nullptr = derive it
  // mutable
  ModelState* ms;              // [M]
  int32_t* pq;                 // [2*Mp] tournament tree of models (next event)
  // the winners' keys held inline beside every tree node (INT64_MAX / -1 =
  // none), so a climb compares its sibling's key without first loading the
  // sibling's id and then its key: one shared-memory round trip per level
  int64_t* pq_t;               // [2*Mp] winner's next-event tick
  int64_t* gt_f;               // [2*Gp] winner's free_at
  int64_t* mlt_v;              // [2*Mp] winner's registered latest
  int64_t* mbt_v;              // [2*Mp] winner's registered size
  int64_t* free_at;            // [G]
  int32_t* gt;                 // [2*Gp] tournament tree, min (free_at, gid)
  int32_t* mc_lat_tree;        // [2*Mp] min (latest, mid) over registered
  int32_t* mc_bs_tree;         // [2*Mp] max (size, mid) over registered
  int32_t* mc_size;            // [M]
  int64_t* mc_latest;          // [M]
  // GPU timer
  int32_t gt_armed, gt_gid;
  int64_t gt_fire;
  EvKey gt_key;
  // outputs
  BatchRec* recs;
  int64_t n_recs, rec_cap;
  int64_t* drop_t;             // [n] by sorted position (trace only)
  int64_t* drop_ksub;          // [n]
  int32_t* drop_ka;            // [n]
  // counters
  int64_t chain_events, absorbed, fresh_adoptions;
  int64_t ops, evictions, registrations, handler_ops_max;
  int32_t error;
  int32_t sh_base;             // first shard-stream index of this shard
  // invariant mode (Engine(check_invariants=True), simulator.py:276-305)
  int64_t served;              // requests dispatched so far (sum of batch sizes)
  int32_t check;               // verify the state after every chain event
  int32_t inject;              // test hook: corrupt the state at chain event `inject` (-1 off)
};

// Canonical A' of the arrival at sorted position pos (engine_core.cuh top):
// its shard-stream index if the previous arrival of the shard has the same
// tick, else BASE.
SYM_HD int32_t aself_at(const Shard& S, int32_t pos) {
  if (S.s_aself) return S.s_aself[pos];
  const int32_t j = S.s_g[pos];
  return (j > S.sh_base && S.sh_tick[j - 1] == S.s_tick[pos]) ? j : A_BASE;
}

enum : int32_t {
  ERR_NONE = 0, ERR_REC_OVERFLOW = 1, ERR_STATE = 2,
  // per-event invariants (simulator.py:276-305), checked with Shard.check
  ERR_INV_CONSERVATION = 3,  // processed arrivals != dispatched + dropped + queued
  ERR_INV_GPU = 4,           // a GPU left OUTSTANDING across an event, or index out of sync
  ERR_INV_INDEX = 5,         // registered-candidate indices out of sync
  ERR_INV_CANDIDATE = 6      // candidate exec_at > latest, or misses its head deadline
};

SYM_HD int64_t imax(int64_t a, int64_t b) { return a > b ? a : b; }
SYM_HD int64_t imin(int64_t a, int64_t b) { return a < b ? a : b; }

// ------------------------------------------------------------ trees -------

// GPU index: min (free_at, gid) (scheduler.py:338, free_idx[0]).
SYM_HD bool gpu_before(const Shard& S, int32_t x, int32_t y) {
  if (y < 0) return x >= 0;
  if (x < 0) return false;
  int64_t fx = S.free_at[x], fy = S.free_at[y];
  if (fx != fy) return fx < fy;
  return x < y;
}

// Leaf-to-root update of a tournament tree along one path: at each level the
// path's winner meets the winner of the sibling subtree (siblings are not
// modified by the climb).  A plain loop over the tree's actual height: the
// trees live in shared memory, and unrolling to a fixed 14 levels with
// runtime guards cost the single chain thread more than the loads
// (tools/chain_prof.py).
SYM_HD void gpu_tree_update(Shard& S, int32_t gid) {
  int32_t node = S.Gp + gid;
  const int64_t f = S.free_at[gid];
  int32_t cur = f == OUTSTANDING ? -1 : gid;
  int64_t ck = f == OUTSTANDING ? INT64_MAX : f;
  S.gt[node] = cur;
  S.gt_f[node] = ck;
  for (; node > 1; node >>= 1) {
    const int32_t o = S.gt[node ^ 1];
    const int64_t ok = S.gt_f[node ^ 1];
    if (o >= 0 && (cur < 0 || ok < ck || (ok == ck && o < cur))) {
      cur = o;
      ck = ok;
    }
    S.gt[node >> 1] = cur;
    S.gt_f[node >> 1] = ck;
  }
}

// registered candidates: min (latest, mid) and max (size, mid)
// (scheduler.py:340-341).
SYM_HD bool lat_before(const Shard& S, int32_t x, int32_t y) {
  if (y < 0) return x >= 0;
  if (x < 0) return false;
  int64_t lx = S.mc_latest[x], ly = S.mc_latest[y];
  if (lx != ly) return lx < ly;
  return x < y;
}
SYM_HD bool bs_before(const Shard& S, int32_t x, int32_t y) {
  if (y < 0) return x >= 0;
  if (x < 0) return false;
  int32_t sx = S.mc_size[x], sy = S.mc_size[y];
  if (sx != sy) return sx > sy;
  return x > y;
}

SYM_HD void mc_tree_update(Shard& S, int32_t mid) {
  int32_t i = S.Mp + mid;
  const bool reg = S.ms[mid].registered;
  int32_t lw = reg ? mid : -1, bw = lw;
  int64_t lv = reg ? S.mc_latest[mid] : INT64_MAX, bv = reg ? S.mc_size[mid] : -1;
  S.mc_lat_tree[i] = lw;
  S.mlt_v[i] = lv;
  S.mc_bs_tree[i] = bw;
  S.mbt_v[i] = bv;
  for (; i > 1; i >>= 1) {
    const int32_t sib = i ^ 1;
    const int32_t lo = S.mc_lat_tree[sib], bo = S.mc_bs_tree[sib];
    const int64_t lov = S.mlt_v[sib], bov = S.mbt_v[sib];
    // min (latest, mid) and max (size, mid): ids break ties (lat_before / bs_before)
    if (lo >= 0 && (lw < 0 || lov < lv || (lov == lv && lo < lw))) {
      lw = lo;
      lv = lov;
    }
    if (bo >= 0 && (bw < 0 || bov > bv || (bov == bv && bo > bw))) {
      bw = bo;
      bv = bov;
    }
    S.mc_lat_tree[i >> 1] = lw;
    S.mlt_v[i >> 1] = lv;
    S.mc_bs_tree[i >> 1] = bw;
    S.mbt_v[i >> 1] = bv;
  }
}

// model priority queue: min next chain-event key.
SYM_HD bool model_before(const Shard& S, int32_t x, int32_t y) {
  if (y < 0) return x >= 0 && S.ms[x].nx_type != EV_NONE;
  if (x < 0 || S.ms[x].nx_type == EV_NONE) return false;
  if (S.ms[y].nx_type == EV_NONE) return true;
  return key_less(S.ms[x].nx_key, S.ms[y].nx_key);
}

SYM_HD void pq_update(Shard& S, int32_t mid) {
  int32_t node = S.Mp + mid;
  int32_t cur = S.ms[mid].nx_type != EV_NONE ? mid : -1;
  int64_t ck = cur >= 0 ? S.ms[mid].nx_key.t : INT64_MAX;
  S.pq[node] = cur;
  S.pq_t[node] = ck;
  for (; node > 1; node >>= 1) {
    const int32_t o = S.pq[node ^ 1];
    const int64_t ot = S.pq_t[node ^ 1];
    // leaves of models without a next event are -1, so o >= 0 has one;
    // equal ticks (rare) fall back to the full key
    if (o >= 0 &&
        (cur < 0 || ot < ck || (ot == ck && key_less(S.ms[o].nx_key, S.ms[cur].nx_key)))) {
      cur = o;
      ck = ot;
    }
    S.pq[node >> 1] = cur;
    S.pq_t[node >> 1] = ck;
  }
}

// (Re)build a tree's internal nodes from its leaves.
SYM_HD void pq_build(Shard& S) {
  for (int32_t i = S.Mp - 1; i >= 1; i--) {
    const int32_t l = S.pq[2 * i], r = S.pq[2 * i + 1];
    const bool right = model_before(S, r, l);
    S.pq[i] = right ? r : l;
    S.pq_t[i] = right ? S.pq_t[2 * i + 1] : S.pq_t[2 * i];
  }
}

// ------------------------------------------------------- ModelPlane -------

// l(b) for 1 <= b <= max_batch.  An exactly affine row (every linear
// profile, detected in sym_create) is computed from two on-chip scalars
// instead of a load from the row, which for a large model set lives in
// global memory: the single chain thread would otherwise pay an L2 round
// trip per probe.
SYM_HD int64_t lat_of(const Shard& S, int32_t m, int32_t b) {
  const ModelParam& P = S.mp[m];
  return P.affine ? P.aff_a * b + P.aff_b : S.lat[(int64_t)m * S.lat_stride + (b - 1)];
}
SYM_HD int64_t deadline_at(const Shard& S, const ModelParam& P, int32_t q) {
  return S.s_tick[P.off + q] + P.slo;
}

// Record one dropped head (scheduler.py:213-216, simulator.py:175-182).
SYM_HD void drop_head(const Shard& S, ModelState& st, const ModelParam& P,
                      int64_t now, const Pusher& who) {
  int32_t pos = P.off + st.qh;
  st.qh += 1;
  st.drops += 1;
  if (S.record_trace) {
    S.drop_t[pos] = now;
    S.drop_ka[pos] = who.a_self;
    S.drop_ksub[pos] = who.sub;
  }
}

// scheduler.py:301-315
SYM_HD void arm_drop_timer(const Shard& S, ModelState& st, const ModelParam& P,
                           int32_t m, int64_t now, const Pusher& who) {
  if (st.qh == st.qt) {
    st.dt_head = -1;
    return;
  }
  if (st.qh == st.dt_head) return;
  st.dt_head = st.qh;
  int64_t fire = deadline_at(S, P, st.qh) - P.base1 + 1;
  st.dt_key = push_key(imax(fire, now), PR_DROP, who);
}

// scheduler.py:277-299.  The predicate ok(b) is monotone in b (both the
// start bound and l(b) are non-decreasing), so the largest feasible b is
// unique and any search finds it.  The search is galloping from a hint (the
// previous candidate's size): as arrivals stream in, the answer moves by a
// step or two, so this costs ~2 probes of the l(b) row instead of ~log2(cap).
SYM_HD int32_t max_feasible(const Shard& S, int32_t m, int64_t now,
                            int64_t floor, int32_t cap, int64_t d,
                            int32_t hint = 0) {
  const int64_t* lat = S.lat + (int64_t)m * S.lat_stride;
  const ModelParam& P = S.mp[m];
  const bool aff = P.affine != 0;
  const int64_t la = P.aff_a, lb0 = P.aff_b;
  const int64_t dc = S.d_ctrl, dd = S.d_data;
  auto ok = [&](int32_t b) {
    return imax(now + dc + dd * b, floor) + (aff ? la * b + lb0 : lat[b - 1]) <= d;
  };
  int32_t lo, hi;  // invariant: ok(lo) (or lo == 0), !ok(hi + 1) (or hi == cap)
  if (hint < 1 || hint > cap) hint = 1;
  if (ok(hint)) {
    lo = hint;
    int32_t step = 1;
    for (;;) {  // gallop up
      const int32_t nb = lo + step;
      if (nb > cap) {
        hi = cap;
        break;
      }
      if (!ok(nb)) {
        hi = nb - 1;
        break;
      }
      lo = nb;
      step <<= 1;
    }
  } else {
    hi = hint - 1;
    int32_t step = 1;
    for (;;) {  // gallop down
      const int32_t nb = hint - step;
      if (nb < 1) {
        lo = 0;
        break;
      }
      if (ok(nb)) {
        lo = nb;
        break;
      }
      hi = nb - 1;
      step <<= 1;
    }
    if (lo == 0) {
      if (hi < 1 || !ok(1)) return 0;
      lo = 1;
    }
  }
  while (lo < hi) {
    const int32_t mid = (lo + hi + 1) >> 1;
    if (ok(mid))
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

// scheduler.py:218-275.  Returns true when the candidate changed.
// The candidate caches its head deadline, l(b) and l(b+1): when the head is
// unchanged, the reference's bisection is replaced by the two probes that
// certify the same answer (the predicate is monotone in b, so b is the
// unique maximum iff ok(b) and not ok(b+1) or b == cap).
SYM_HD bool update_candidate_impl(const Shard& S, int32_t m, ModelState& st,
                                  int64_t now, int64_t gpu_floor,
                                  const Pusher& who) {
  const ModelParam& P = S.mp[m];
  bool hc = st.has_cand && st.c_head == st.qh;  // cache valid for the head
  int64_t dh = 0;
  if (st.qh < st.qt) dh = hc ? st.c_d : deadline_at(S, P, st.qh);
  while (st.qh < st.qt && now + P.base1 > dh) {
    drop_head(S, st, P, now, who);
    hc = false;
    if (st.qh < st.qt) dh = deadline_at(S, P, st.qh);
  }
  if (S.kind == K_TIMEOUT) {
    // arrival + k + l(1) > deadline  <=>  k + l(1) > slo (scheduler.py:229)
    const int64_t l1 = P.base1 - S.d_ctrl - S.d_data;
    while (st.qh < st.qt && P.timeout_ns + l1 > P.slo) {
      drop_head(S, st, P, now, who);
      hc = false;
    }
    if (st.qh < st.qt && !hc) dh = deadline_at(S, P, st.qh);
  }
  if (S.gather == G_DROP_HEAD && st.qt - st.qh > P.target_batch) {
    const int32_t tb = P.target_batch;
    const int64_t need = now + S.d_ctrl + S.d_data * tb + lat_of(S, m, tb);
    while (st.qt - st.qh > tb && need > dh) {
      drop_head(S, st, P, now, who);
      hc = false;
      dh = deadline_at(S, P, st.qh);
    }
  }
  if (st.qh == st.qt) {
    arm_drop_timer(S, st, P, m, now, who);
    if (st.has_cand) {
      st.has_cand = 0;
      return true;
    }
    return false;
  }
  const int64_t d = dh;
  int32_t cap = st.qt - st.qh;
  if (cap > P.max_batch) cap = P.max_batch;
  if (S.gather == G_DROP_HEAD && cap > P.target_batch) cap = P.target_batch;
  // timeout floor = head arrival + k = (deadline - slo) + k
  const int64_t pol_floor = S.kind == K_TIMEOUT ? d - P.slo + P.timeout_ns : NEG_INF;
  const int64_t floor2 = imax(pol_floor, gpu_floor);
  const int64_t dc = S.d_ctrl, dd = S.d_data;
  int32_t b;
  int64_t lb, lnext;
  const int32_t cb = st.c_size;
  if (hc && cb <= cap && imax(now + dc + dd * cb, floor2) + st.c_lb <= d &&
      (cb == cap || imax(now + dc + dd * (cb + 1), floor2) + st.c_lb1 > d)) {
    b = cb;
    lb = st.c_lb;
    lnext = st.c_lb1;
  } else {
    b = max_feasible(S, m, now, floor2, cap, d, st.has_cand ? st.c_size : 1);
    if (b == 0) {
      arm_drop_timer(S, st, P, m, now, who);
      if (st.has_cand) {
        st.has_cand = 0;
        return true;
      }
      return false;
    }
    lb = lat_of(S, m, b);
    lnext = b < P.max_batch ? lat_of(S, m, b + 1) : lat_of(S, m, P.max_batch);
  }
  int64_t exec_at = now + dc + dd * b;
  if (S.kind == K_DEFERRED && d - lnext > exec_at) exec_at = d - lnext;
  if (floor2 > exec_at) exec_at = floor2;
  const int64_t latest = d - lb;
  arm_drop_timer(S, st, P, m, now, who);
  if (st.has_cand && st.c_size == b && st.c_exec == exec_at &&
      st.c_latest == latest && st.c_head == st.qh)
    return false;
  st.has_cand = 1;
  st.c_size = b;
  st.c_exec = exec_at;
  st.c_latest = latest;
  st.c_head = st.qh;
  st.c_d = d;
  st.c_lb = lb;
  st.c_lb1 = lnext;
  return true;
}

SYM_HD bool update_candidate(const Shard& S, int32_t m, ModelState& st, int64_t now,
                             int64_t gpu_floor, const Pusher& who) {
  SYM_PROF_T(u0);
  const bool r = update_candidate_impl(S, m, st, now, gpu_floor, who);
  SYM_PROF_T(u1);
  SYM_PROF_ADD(12, u1 - u0);
  SYM_PROF_ADD(13, 1);
  return r;
}

// ------------------------------------------------------- RankPlane --------

SYM_HD void unregister(Shard& S, int32_t m) {  // scheduler.py:430-436
  if (S.ms[m].registered) {
    S.ms[m].registered = 0;
    mc_tree_update(S, m);
    S.ops += 2;
  }
}

// scheduler.py:438-457
SYM_HD void set_gpu_timer_impl(Shard& S, int64_t now, const Pusher& who) {
  const int32_t gid = S.gt[1];
  const int32_t bm = S.mc_bs_tree[1];
  if (bm < 0 || gid < 0) {
    S.gt_armed = 0;
    return;
  }
  S.ops += 2;
  int64_t fire = S.free_at[gid] - (S.d_ctrl + S.d_data * S.mc_size[bm]);
  if (fire < now) fire = now;
  if (S.gt_armed && S.gt_fire == fire && S.gt_gid == gid) return;
  S.gt_armed = 1;
  S.gt_fire = fire;
  S.gt_gid = gid;
  S.gt_key = push_key(fire, PR_GPU, who);
}

SYM_HD void set_gpu_timer(Shard& S, int64_t now, const Pusher& who) {
  SYM_PROF_T(g0);
  set_gpu_timer_impl(S, now, who);
  SYM_PROF_T(g1);
  SYM_PROF_ADD(15, g1 - g0);
}

// Model-local half of inform_candidate: model_gen[m] += 1 supersedes the
// live timer, and a candidate gets a new one (scheduler.py:358-365).
SYM_HD void renew_model_timer(const Shard& S, ModelState& st, int64_t now,
                              const Pusher& who) {
  st.has_mt = 0;
  if (st.has_cand) {
    int64_t fire = st.c_exec - (S.d_ctrl + S.d_data * st.c_size);
    if (fire < now) fire = now;
    st.mt_key = push_key(fire, PR_MODEL, who);
    st.has_mt = 1;
  }
}

// scheduler.py:354-365
SYM_HD void inform_candidate(Shard& S, int32_t m, int64_t now,
                             const Pusher& who) {
  unregister(S, m);
  renew_model_timer(S, S.ms[m], now, who);
}

// scheduler.py:367-377 (the GPU is always OUTSTANDING here: grants resolve
// inline, so the only caller re-inserts the granted GPU)
SYM_HD void inform_gpu(Shard& S, int32_t gid, int64_t free_at, int64_t now,
                       const Pusher& who) {
  if (S.free_at[gid] != OUTSTANDING) S.ops += 1;
  S.free_at[gid] = free_at;
  gpu_tree_update(S, gid);
  S.ops += 1;
  set_gpu_timer(S, now, who);
}

// scheduler.py:180-209 (jitterless network: start = exec_at)
SYM_HD void granted_gpu(Shard& S, int32_t m, int32_t gid, int64_t gpu_free_at,
                        int64_t now, const Pusher& who) {
  ModelState& st = S.ms[m];
  const int32_t pre_size = st.has_cand ? st.c_size : 0;
  update_candidate(S, m, st, now, imax(gpu_free_at, 0), who);
  if (!st.has_cand) {
    inform_gpu(S, gid, imax(now, gpu_free_at), now, who);
    update_candidate(S, m, st, now, NEG_INF, who);
    inform_candidate(S, m, now, who);
    return;
  }
  const int32_t b = st.c_size;
  const int64_t lat_b = st.c_lb;
  if (S.n_recs < S.rec_cap) {
    BatchRec& r = S.recs[S.n_recs];
    r.emitted = now;
    r.start = st.c_exec;
    r.finish = st.c_exec + lat_b;
    r.kt = who.t;
    r.ka = who.a_self;
    r.ksub = who.sub;
    r.model = m;
    r.gpu = gid;
    r.size = b;
    r.first = S.mp[m].off + st.qh;
    r.shrunk_from = b < pre_size ? pre_size : 0;
  } else {
    S.error = ERR_REC_OVERFLOW;
  }
  S.n_recs += 1;
  S.served += b;
  st.qh += b;
  const int64_t believed_free = st.c_exec + lat_b;
  st.has_cand = 0;
  update_candidate(S, m, st, now, NEG_INF, who);
  inform_gpu(S, gid, believed_free, now, who);
  inform_candidate(S, m, now, who);
}

// scheduler.py:381-399 (always live here: only live timers exist)
SYM_HD void on_model_timer(Shard& S, int32_t m, int64_t now,
                           const Pusher& who) {
  ModelState& st = S.ms[m];
  st.has_mt = 0;
  const int32_t gid = S.gt[1];
  if (gid >= 0) {
    const int64_t fa = S.free_at[gid];
    S.ops += 1;
    if (fa <= st.c_exec) {
      S.ops += 1;
      S.free_at[gid] = OUTSTANDING;  // tree refreshed by inform_gpu
      granted_gpu(S, m, gid, fa, now, who);
      return;
    }
  }
  st.registered = 1;
  S.mc_size[m] = st.c_size;
  S.mc_latest[m] = st.c_latest;
  mc_tree_update(S, m);
  S.ops += 2;
  S.registrations += 1;
  set_gpu_timer(S, now, who);
}

// scheduler.py:173-178
SYM_HD void on_drop_timer(Shard& S, int32_t m, int64_t now,
                          const Pusher& who) {
  ModelState& st = S.ms[m];
  st.dt_head = -1;
  if (update_candidate(S, m, st, now, NEG_INF, who))
    inform_candidate(S, m, now, who);
}

// scheduler.py:168-171 for the arrival at sorted position off+qt of a model
// that is NOT registered (the unregister of inform_candidate is a no-op).
SYM_HD void absorb_arrival(const Shard& S, int32_t m, ModelState& st) {
  const int32_t pos = S.mp[m].off + st.qt;
  const int64_t now = S.s_tick[pos];
  Pusher who;
  who.t = now;
  who.a_self = aself_at(S, pos);
  who.a_after = S.s_g[pos] + 1;
  who.sub = SUB_ARRIVAL;
  st.qt += 1;
  if (update_candidate(S, m, st, now, NEG_INF, who))
    renew_model_timer(S, st, now, who);
}

// The same arrival for a registered model: a chain event, because its
// inform_candidate unregisters it from the rank plane.
SYM_HD void registered_arrival(Shard& S, int32_t m) {
  ModelState& st = S.ms[m];
  const int32_t pos = S.mp[m].off + st.qt;
  const int64_t now = S.s_tick[pos];
  Pusher who;
  who.t = now;
  who.a_self = aself_at(S, pos);
  who.a_after = S.s_g[pos] + 1;
  who.sub = SUB_ARRIVAL;
  st.qt += 1;
  if (update_candidate(S, m, st, now, NEG_INF, who))
    inform_candidate(S, m, now, who);
}

// ----------------------------------------------- local absorption scan ----
// Absorb this model's arrivals until its next chain event, which is stored
// in nx_key/nx_type.  Valid because an unregistered model's arrivals touch
// nothing but the model itself, and no other chain event touches it.
// Returns the number of absorbed arrivals; stops early (returning -1) after
// max_steps absorptions when max_steps >= 0.
SYM_HD int32_t scan_model(const Shard& S, int32_t m, ModelState& st,
                          int32_t max_steps) {
  const ModelParam& P = S.mp[m];
  int32_t steps = 0;
  for (;;) {
    int32_t type = EV_NONE;
    EvKey best;
    if (st.has_mt) {
      best = st.mt_key;
      type = EV_MT;
    }
    if (st.dt_head >= 0 && (type == EV_NONE || key_less(st.dt_key, best))) {
      best = st.dt_key;
      type = EV_DT;
    }
    if (st.qt < P.cnt) {
      const int32_t pos = P.off + st.qt;
      const int64_t ta = S.s_tick[pos];
      const int32_t aa = aself_at(S, pos);
      // an arrival precedes a timer iff (a, A') < (tick, A') (prio 4 > 3)
      const bool first = type == EV_NONE || ta < best.t ||
                         (ta == best.t && aa < best.a);
      if (first) {
        if (st.registered) {
          best.t = ta;
          best.a = aa;
          best.prio = PR_ARRIVAL;
          best.tp = 0;
          best.ap = 0;
          best.sub = 0;
          best._pad = 0;
          type = EV_ARR;
        } else {
          if (max_steps >= 0 && steps >= max_steps) return -1;
          absorb_arrival(S, m, st);
          steps += 1;
          continue;
        }
      }
    }
    st.nx_type = type;
    if (type != EV_NONE) st.nx_key = best;
    return steps;
  }
}

// ------------------------------------------- fresh-start pre-scan (K2) ----
// After a grant empties a model's queue the model is "fresh": no candidate,
// no timers, not registered.  Its evolution from the next arrival on is a
// pure function of its own arrivals, so it is pre-computed for EVERY sorted
// position in parallel and the chain adopts the record in O(1).

struct alignas(128) FreshRec {
  int64_t c_exec, c_latest;
  int64_t c_d, c_lb, c_lb1;
  int64_t mt_t, mt_tp;  // model-timer key (prio 2, sub = arrival)
  int64_t dt_t, dt_tp;  // drop-timer key (prio 3, sub = arrival)
  int32_t qt, qh;       // queue after the scan (model-relative)
  int32_t c_size;       // 0 = no candidate
  int32_t mt_a, mt_ap, dt_a, dt_ap;
  int32_t drops;        // heads dropped during the scan
  int32_t steps;        // arrivals absorbed; -1 = scan too long, not valid
};

SYM_HD void fresh_state(ModelState& st, int32_t q) {
  st.qh = st.qt = q;
  st.has_cand = 0;
  st.c_size = 0;
  st.c_head = -1;
  st.c_exec = st.c_latest = 0;
  st.c_d = st.c_lb = st.c_lb1 = 0;
  st.registered = 0;
  st.has_mt = 0;
  st.dt_head = -1;
  st.nx_type = EV_NONE;
  st.drops = 0;
}

SYM_HD bool is_fresh(const ModelState& st) {
  return st.qh == st.qt && !st.has_cand && !st.has_mt && st.dt_head < 0 &&
         !st.registered;
}

SYM_HD FreshRec fresh_scan(const Shard& S, int32_t m, int32_t q,
                           int32_t max_steps) {
  ModelState st;
  fresh_state(st, q);
  FreshRec r;
  r.steps = scan_model(S, m, st, max_steps);
  r.qt = st.qt;
  r.qh = st.qh;
  r.c_size = st.has_cand ? st.c_size : 0;
  r.c_exec = st.c_exec;
  r.c_latest = st.c_latest;
  r.c_d = st.c_d;
  r.c_lb = st.c_lb;
  r.c_lb1 = st.c_lb1;
  r.mt_t = st.mt_key.t;
  r.mt_tp = st.mt_key.tp;
  r.mt_a = st.mt_key.a;
  r.mt_ap = st.mt_key.ap;
  r.dt_t = st.dt_key.t;
  r.dt_tp = st.dt_key.tp;
  r.dt_a = st.dt_key.a;
  r.dt_ap = st.dt_key.ap;
  r.drops = (int32_t)st.drops;
  return r;
}

// Rebuild the model state a valid fresh scan ended in (inverse of
// fresh_scan: a fresh scan stops at its first chain event, so the model
// timer is live iff there is a candidate and the drop timer is armed for
// the current head iff the queue is non-empty).
SYM_HD void adopt_fresh(ModelState& st, const FreshRec& r) {
  const int64_t drops = st.drops;
  fresh_state(st, r.qt);
  st.drops = drops + r.drops;
  st.qh = r.qh;
  if (r.c_size > 0) {
    st.has_cand = 1;
    st.c_size = r.c_size;
    st.c_exec = r.c_exec;
    st.c_latest = r.c_latest;
    st.c_head = r.qh;
    st.c_d = r.c_d;
    st.c_lb = r.c_lb;
    st.c_lb1 = r.c_lb1;
    st.has_mt = 1;
    st.mt_key.t = r.mt_t;
    st.mt_key.a = r.mt_a;
    st.mt_key.prio = PR_MODEL;
    st.mt_key.tp = r.mt_tp;
    st.mt_key.ap = r.mt_ap;
    st.mt_key.sub = SUB_ARRIVAL;
    st.mt_key._pad = 0;
  }
  if (r.qh < r.qt) {
    st.dt_head = r.qh;
    st.dt_key.t = r.dt_t;
    st.dt_key.a = r.dt_a;
    st.dt_key.prio = PR_DROP;
    st.dt_key.tp = r.dt_tp;
    st.dt_key.ap = r.dt_ap;
    st.dt_key.sub = SUB_ARRIVAL;
    st.dt_key._pad = 0;
  }
  st.nx_type = EV_NONE;
  if (st.has_mt) {
    st.nx_type = EV_MT;
    st.nx_key = st.mt_key;
  }
  if (st.dt_head >= 0 &&
      (st.nx_type == EV_NONE || key_less(st.dt_key, st.nx_key))) {
    st.nx_type = EV_DT;
    st.nx_key = st.dt_key;
  }
}

// ------------------------------------------------------------ chain -------

SYM_HD void on_gpu_timer(Shard& S, const Pusher& who, int32_t* dirty,
                         int32_t& nd) {
  S.gt_armed = 0;
  const int32_t gid = S.gt_gid;
  const int64_t fa = S.free_at[gid];
  const int64_t now = who.t;
  if (fa == OUTSTANDING) {
    set_gpu_timer(S, now, who);
    return;
  }
  for (;;) {
    const int32_t m = S.mc_lat_tree[1];
    if (m < 0 || S.mc_latest[m] >= fa) break;
    S.ms[m].registered = 0;
    mc_tree_update(S, m);
    S.ops += 2;
    S.evictions += 1;
    dirty[nd++] = m;
  }
  const int32_t m = S.mc_lat_tree[1];
  if (m >= 0) {
    S.ops += 1;
    unregister(S, m);
    S.ops += 1;
    S.free_at[gid] = OUTSTANDING;  // tree refreshed by inform_gpu
    granted_gpu(S, m, gid, fa, now, who);
    dirty[nd++] = m;
  }
  set_gpu_timer(S, now, who);
}

// The record this model will most likely adopt next (its queue drains at
// its next grant) is pulled into L2 now, long before that grant.
SYM_HD void prefetch_fresh(const FreshRec* fresh, const ModelParam& P,
                           const ModelState& st) {
#ifdef __CUDA_ARCH__
  if (fresh && st.qt < P.cnt)
    asm volatile("prefetch.global.L1 [%0];" ::"l"(fresh + P.off + st.qt));
#else
  (void)fresh;
  (void)P;
  (void)st;
#endif
}

// Bring a model whose state just changed up to its next chain event, using
// the fresh-start table when the state is fresh.
//
// Adopting a record costs one global load (~600 cycles); scanning costs a
// few hundred cycles per absorbed arrival.  A model whose adopted records
// absorb almost nothing (eager dispatch, overload: one arrival per fresh
// start) therefore scans its next kFreshBackoff fresh starts instead.  Both
// give the identical state, so this only affects speed.
constexpr int32_t kFreshBackoff = 16;

SYM_HD void refresh_model(Shard& S, int32_t m, const FreshRec* fresh) {
  ModelState& st = S.ms[m];
  const ModelParam& P = S.mp[m];
  if (fresh && is_fresh(st) && st.qt < P.cnt) {
    if (st.fresh_skip > 0) {
      st.fresh_skip -= 1;
    } else {
      const FreshRec& r = fresh[P.off + st.qt];
      if (r.steps >= 0) {
        adopt_fresh(st, r);
        st.fresh_skip = r.steps <= 2 ? kFreshBackoff : 0;
        S.absorbed += r.steps;
        S.fresh_adoptions += 1;
        prefetch_fresh(fresh, P, st);
        return;
      }
    }
  }
  SYM_PROF_T(s0);
  S.absorbed += scan_model(S, m, st, -1);
  SYM_PROF_T(s1);
  SYM_PROF_ADD(14, s1 - s0);
  if (st.fresh_skip == 0) prefetch_fresh(fresh, P, st);
}

// The reference's _verify (simulator.py:276-305) on the chain state after an
// event, O(M + G): conservation (every processed arrival is dispatched,
// dropped or queued), the GPU state machine (no grant outstanding across an
// event boundary, the free index equal to min (free_at, gid)), the
// registered-candidate indices in sync with the registered flags, and every
// candidate feasible (exec_at <= latest, exec_at + l(b) <= head deadline).
SYM_HD int32_t verify_state(const Shard& S) {
  int64_t queued_total = 0, processed = 0, dropped = 0;
  int32_t min_lat = -1, max_bs = -1;
  for (int32_t m = 0; m < S.M; m++) {
    const ModelState& st = S.ms[m];
    if (st.qh < 0 || st.qh > st.qt || st.qt > S.mp[m].cnt) return ERR_INV_CONSERVATION;
    queued_total += st.qt - st.qh;
    processed += st.qbase + st.qt;
    dropped += st.drops;
    if (st.has_cand) {
      if (st.c_exec > st.c_latest) return ERR_INV_CANDIDATE;
      if (st.c_exec + lat_of(S, m, st.c_size) > st.c_d) return ERR_INV_CANDIDATE;
    }
    if (st.registered) {
      if (!st.has_cand) return ERR_INV_INDEX;
      if (lat_before(S, m, min_lat)) min_lat = m;
      if (bs_before(S, m, max_bs)) max_bs = m;
    }
  }
  if (processed != S.served + dropped + queued_total) return ERR_INV_CONSERVATION;
  if (S.mc_lat_tree[1] != min_lat || S.mc_bs_tree[1] != max_bs) return ERR_INV_INDEX;
  int32_t best = -1;
  for (int32_t g = 0; g < S.G; g++) {
    if (S.free_at[g] == OUTSTANDING) return ERR_INV_GPU;
    if (gpu_before(S, g, best)) best = g;
  }
  if (S.gt[1] != best) return ERR_INV_GPU;
  return ERR_NONE;
}

// Process one chain event; returns false when the sub-cluster is drained or
// its next event lies after `until` (a stepped run stops there: every event
// with tick <= until is processed, later ones wait for the next step).
// dirty must hold M+1 entries.
SYM_HD bool chain_step(Shard& S, int32_t* dirty, const FreshRec* fresh,
                       int64_t until = INT64_MAX) {
  SYM_PROF_T(t0);
  const int32_t m = S.pq[1];
  const bool have_m = m >= 0;
  if (!have_m && !S.gt_armed) return false;
  int32_t nd = 0;
  const int64_t ops0 = S.ops, ev0 = S.evictions;
  bool timer_event = true;
#ifdef SYM_CHAIN_PROF
  int prof_type = 3;
#endif
  SYM_PROF_T(t1);
  const bool gpu_event = S.gt_armed && (!have_m || key_less(S.gt_key, S.ms[m].nx_key));
  if ((gpu_event ? S.gt_key.t : S.ms[m].nx_key.t) > until) return false;
  if (gpu_event) {
    Pusher who;
    who.t = S.gt_key.t;
    who.a_self = who.a_after = S.gt_key.a;
    who.sub = S.chain_events;
    on_gpu_timer(S, who, dirty, nd);
  } else {
    ModelState& st = S.ms[m];
    Pusher who;
    who.t = st.nx_key.t;
    who.a_self = who.a_after = st.nx_key.a;
    who.sub = S.chain_events;
#ifdef SYM_CHAIN_PROF
    prof_type = st.nx_type - 1;
#endif
    switch (st.nx_type) {
      case EV_MT: on_model_timer(S, m, who.t, who); break;
      case EV_DT: on_drop_timer(S, m, who.t, who); break;
      case EV_ARR:
        registered_arrival(S, m);
        timer_event = false;
        break;
      default: S.error = ERR_STATE; return false;
    }
  }
  SYM_PROF_T(t2);
  S.chain_events += 1;
  if (timer_event) {
    const int64_t ops = (S.ops - ops0) - 2 * (S.evictions - ev0);
    if (ops > S.handler_ops_max) S.handler_ops_max = ops;
  }
  // a model event dirties only its own model (kept in a register); a GPU
  // timer may dirty several (evictions), listed in `dirty`
  const int32_t nref = gpu_event ? nd : 1;
  for (int32_t i = 0; i < nref; i++) {
    const int32_t dm = gpu_event ? dirty[i] : m;
    SYM_PROF_T(r0);
    refresh_model(S, dm, fresh);
    SYM_PROF_T(r1);
    pq_update(S, dm);
    SYM_PROF_T(r2);
    SYM_PROF_ADD(9, r1 - r0);
    SYM_PROF_ADD(10, r2 - r1);
  }
  SYM_PROF_ADD(prof_type, t2 - t1);
  SYM_PROF_ADD(4 + prof_type, 1);
  SYM_PROF_ADD(8, t1 - t0);
  SYM_PROF_ADD(11, nref);
  if (S.check) {
    if (S.inject >= 0 && S.chain_events == S.inject + 1) {
      // test hook: lose the head of the model that just moved without
      // counting a drop, or (empty queue) leave GPU 0 outstanding
      const int32_t cm = gpu_event ? (nd > 0 ? dirty[0] : 0) : m;
      if (S.ms[cm].qh < S.ms[cm].qt) S.ms[cm].qh += 1;
      else S.free_at[0] = OUTSTANDING;
    }
    const int32_t e = verify_state(S);
    if (e) {
      S.error = e;
      return false;
    }
  }
  return true;
}

// Initialise trees and bring every model to its first chain event.
SYM_HD void chain_init(Shard& S, const FreshRec* fresh) {
  for (int32_t g = 0; g < S.G; g++) S.free_at[g] = 0;
  for (int32_t i = 0; i < 2 * S.Gp; i++) {
    S.gt[i] = -1;
    S.gt_f[i] = INT64_MAX;
  }
  for (int32_t g = 0; g < S.G; g++) {
    S.gt[S.Gp + g] = g;
    S.gt_f[S.Gp + g] = 0;
  }
  for (int32_t i = S.Gp - 1; i >= 1; i--) {
    const int32_t l = S.gt[2 * i], r = S.gt[2 * i + 1];
    const bool right = gpu_before(S, r, l);
    S.gt[i] = right ? r : l;
    S.gt_f[i] = right ? S.gt_f[2 * i + 1] : S.gt_f[2 * i];
  }
  for (int32_t i = 0; i < 2 * S.Mp; i++) {
    S.pq[i] = -1;
    S.pq_t[i] = INT64_MAX;
    S.mc_lat_tree[i] = -1;
    S.mc_bs_tree[i] = -1;
    S.mlt_v[i] = INT64_MAX;
    S.mbt_v[i] = -1;
  }
  S.gt_armed = 0;
  S.n_recs = 0;
  S.served = 0;
  S.chain_events = S.absorbed = S.fresh_adoptions = 0;
  S.ops = S.evictions = S.registrations = S.handler_ops_max = 0;
  S.error = ERR_NONE;
  for (int32_t m = 0; m < S.M; m++) {
    fresh_state(S.ms[m], 0);
    S.ms[m].fresh_skip = 0;
    S.ms[m].qbase = 0;
    S.mc_size[m] = 0;
    S.mc_latest[m] = 0;
    refresh_model(S, m, fresh);
    const bool act = S.ms[m].nx_type != EV_NONE;
    S.pq[S.Mp + m] = act ? m : -1;
    S.pq_t[S.Mp + m] = act ? S.ms[m].nx_key.t : INT64_MAX;
  }
  pq_build(S);
}

// Resume a stepped run: the state of every model, the trees and the GPU
// timer are as the previous step left them; the sorted stream now also
// holds this step's arrivals.  Each model is brought to its next event
// again (an unregistered model absorbs new arrivals that precede its
// pending timers; those timers all lie after the previous step's until, and
// the new arrivals at or after it) and the model tree is rebuilt.
SYM_HD void chain_resume(Shard& S) {
  S.n_recs = 0;
  S.error = ERR_NONE;
  for (int32_t m = 0; m < S.M; m++) {
    S.absorbed += scan_model(S, m, S.ms[m], -1);
    const bool act = S.ms[m].nx_type != EV_NONE;
    S.pq[S.Mp + m] = act ? m : -1;
    S.pq_t[S.Mp + m] = act ? S.ms[m].nx_key.t : INT64_MAX;
  }
  pq_build(S);
}

SYM_HD int64_t total_drops(const Shard& S) {
  int64_t d = 0;
  for (int32_t m = 0; m < S.M; m++) d += S.ms[m].drops;
  return d;
}

}  // namespace sym
