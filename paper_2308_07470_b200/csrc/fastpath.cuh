// fastpath.cuh -- the parallel "validated regime" of a sub-cluster.
//
// Observation.  While every live model timer finds the
// earliest-free GPU free by its exec_at (scheduler.py:385-393 never takes
// the registration branch), the rank plane never feeds anything back into a
// model: the revalidation in granted_gpu (scheduler.py:185) reproduces the
// candidate unchanged, and no GPU timer is ever armed (mc stays empty,
// scheduler.py:442).  Each model's batch sequence is then a pure function of
// its own arrivals ("unconstrained evolution", k_evolve), and the whole
// sub-cluster reduces to
//   (1) sort all batches of the sub-cluster by their event key,
//   (2) batch i pops the smallest (free_at, gid) of the GPU index and pushes
//       (exec_i + l(b_i), same gid).  The index is a monotone priority queue
//       (every push exceeds the popped key), so batch i pops the i-th
//       smallest token overall -- initial tokens (0, g) first, in gid
//       order, then the finish times -- provided that token was created
//       before batch i.  A token's gid is its creator batch's gid, resolved
//       by pointer jumping.
// Every assumption is checked (flags below); a sub-cluster that violates any
// of them is re-run by the exact sequential chain (k_chain).
#pragma once
#include "engine_core.cuh"

namespace sym {

// validation failure reasons (bit flags per sub-cluster)
enum : uint32_t {
  FP_DROP_TIMER = 1u,      // a drop timer would pop before the model timer
  FP_SAME_TICK_GRANT = 2u, // a grant pushes a timer firing at its own tick
  FP_REVALIDATE = 4u,      // revalidation at the pop changed the candidate
  FP_KEY_TIE = 8u,         // two batch keys tie up to the chain counter
  FP_NO_GPU = 16u,         // popped token free after exec_at (registration)
  FP_LATE_TOKEN = 32u,     // token created after the batch that pops it
  FP_TOKEN_TIE = 64u,      // equal finish times popped out of gid order
  FP_CAPACITY = 128u,      // scratch exhausted / scan too long
};

// One batch of a model's unconstrained evolution.
struct EvBatch {
  int64_t t;       // model-timer tick (the grant's processing tick)
  int64_t tp;      // pusher tick
  int64_t exec;    // exec_at = start
  int64_t lat;     // l(size)
  int32_t a;       // canonical A' of the timer
  int32_t ap;      // pusher A'
  int32_t size;
  int32_t first;   // sorted-stream position of the first member
  int32_t model;   // shard-local model id
  int32_t chain;   // 1 = pushed by the model's previous grant, 0 = arrival
};

// Strict weak order of two batch events of one sub-cluster, excluding the
// chain-counter tie-break (ties there are rejected with FP_KEY_TIE).
SYM_HD int batch_cmp(const EvBatch& x, const EvBatch& y) {
  if (x.t != y.t) return x.t < y.t ? -1 : 1;
  if (x.a != y.a) return x.a < y.a ? -1 : 1;
  if (x.tp != y.tp) return x.tp < y.tp ? -1 : 1;
  if (x.ap != y.ap) return x.ap < y.ap ? -1 : 1;
  // at an equal pusher position a chain event precedes the arrival
  if (x.chain != y.chain) return x.chain ? -1 : 1;
  return 0;
}

// Unconstrained evolution of model m of shard S: emits its batches in event
// order into out[0..), returns their count (or -1 on a validation failure
// recorded in *fail).  The model-side effect of a grant is exactly
// granted_gpu (scheduler.py:180-209) with the GPU floor elided: the floor is
// <= exec_at in the validated regime and leaves the candidate unchanged,
// which is asserted (FP_REVALIDATE).
SYM_HD int32_t evolve_model(const Shard& S, int32_t m, const FreshRec* fresh,
                            EvBatch* out, int32_t cap, int64_t* drops,
                            uint32_t* fail) {
  const ModelParam& P = S.mp[m];
  ModelState st;
  fresh_state(st, 0);
  int32_t nb = 0;
  bool first_refresh = true;
  for (;;) {
    // bring the model to its next event (fresh-start table when possible)
    if (first_refresh || is_fresh(st)) {
      first_refresh = false;
      if (st.qt < P.cnt && fresh) {
        const FreshRec& r = fresh[P.off + st.qt];
        if (r.steps >= 0) {
          adopt_fresh(st, r);
        } else {
          scan_model(S, m, st, -1);
        }
      } else {
        scan_model(S, m, st, -1);
      }
    } else {
      scan_model(S, m, st, -1);
    }
    if (st.nx_type == EV_NONE) break;
    if (st.nx_type != EV_MT) {
      *fail |= FP_DROP_TIMER;
      return -1;
    }
    if (nb >= cap) {
      *fail |= FP_CAPACITY;
      return -1;
    }
    const EvKey k = st.mt_key;
    const int64_t now = k.t;
    Pusher who;
    who.t = now;
    who.a_self = who.a_after = k.a;
    who.sub = 0;  // placeholder: the chain counter is never compared here
    // granted_gpu: revalidation with a floor <= exec_at
    const int32_t b0 = st.c_size;
    const int64_t e0 = st.c_exec, l0 = st.c_latest;
    update_candidate(S, m, st, now, 0, who);
    if (!st.has_cand || st.c_size != b0 || st.c_exec != e0 || st.c_latest != l0) {
      *fail |= FP_REVALIDATE;
      return -1;
    }
    EvBatch& e = out[nb++];
    e.t = now;
    e.a = k.a;
    e.tp = k.tp;
    e.ap = k.ap;
    e.chain = k.sub != SUB_ARRIVAL;
    e.exec = st.c_exec;
    e.lat = st.c_lb;
    e.size = st.c_size;
    e.first = P.off + st.qh;
    e.model = m;
    st.qh += st.c_size;
    st.has_cand = 0;
    update_candidate(S, m, st, now, NEG_INF, who);
    renew_model_timer(S, st, now, who);
    if (st.has_mt && st.mt_key.t == now) {
      *fail |= FP_SAME_TICK_GRANT;
      return -1;
    }
  }
  *drops = st.drops;
  return nb;
}

}  // namespace sym

namespace sym {

// Batch-chain pointer of a fresh start at position p (fastpath.cuh):
//   >= 0  a batch starts at p and drains the queue; the model is fresh again
//         at that absolute position
//   NX_LAST  a batch starts at p, drains the queue, no arrivals remain
//   NX_NONE  no batch: every queued request was dropped, none remain
//   NX_SPECIAL  anything else (non-draining grant, drop timer first, scan cap)
constexpr int32_t NX_LAST = -1, NX_NONE = -2, NX_SPECIAL = -3;
constexpr int32_t NX_UNSURE = -4;  // ask the general fresh_scan
constexpr int32_t NX_LAST_LEAN = NX_LAST;

SYM_HD int32_t chain_next(const FreshRec& r, const ModelParam& mp) {
  if (r.steps < 0) return NX_SPECIAL;
  if (r.c_size == 0) return r.qh == r.qt && r.qt == mp.cnt ? NX_NONE : NX_SPECIAL;
  if (r.c_size != r.qt - r.qh) return NX_SPECIAL;  // grant would leave a remainder
  // the model timer must be the next event (it precedes the drop timer in a
  // fresh scan, fastpath.cuh FP_DROP_TIMER)
  const bool mt_first = r.mt_t < r.dt_t || (r.mt_t == r.dt_t && r.mt_a <= r.dt_a);
  if (!mt_first) return NX_SPECIAL;
  return r.qt == mp.cnt ? NX_LAST : mp.off + r.qt;
}


// Lean restatement of a fresh start at model position q for the deferred
// policy with prefix gathering, valid while no head is dropped and the
// candidate holds the whole queue (the underload regime).  Returns the
// batch-chain pointer (absolute next fresh position or NX_LAST), or
// NX_UNSURE as soon as the run leaves that regime.  Exact by construction:
//  * drops: none while now + d_ctrl + d_data + l(1) <= head deadline
//    (scheduler.py:223-225); later entries have later deadlines (FIFO, one
//    SLO per model);
//  * candidate: b = max_feasible with cap = min(len, max_batch)
//    (scheduler.py:246-252), exec_at/latest as scheduler.py:262-270; the
//    model timer is re-pushed only when (size, exec_at, latest) changes (the
//    head is fixed, scheduler.py:272-273), at max(exec_at - delay(b), now)
//    (scheduler.py:361-363);
//  * the model timer precedes the drop timer (it fires no later than
//    latest - delay < deadline - l(1) - delay(1) + 1), and precedes an
//    arrival at the same tick, so the batch closes at the
//    first arrival k with fire <= a_{k+1}.
SYM_HD int32_t lean_chain_next(const Shard& S, int32_t m, int32_t q) {
  const ModelParam& P = S.mp[m];
  if (S.kind != K_DEFERRED || S.gather != G_PREFIX) return NX_UNSURE;
  const int64_t* lat_row = S.lat + (int64_t)m * S.lat_stride;
  const bool aff = P.affine != 0;
  const int64_t la = P.aff_a, lb0 = P.aff_b;
  auto lat = [&](int32_t i) { return aff ? la * (i + 1) + lb0 : lat_row[i]; };
  const int64_t* tick = S.s_tick + P.off;
  const int64_t dc = S.d_ctrl, dd = S.d_data;
  const int64_t d = tick[q] + P.slo;
  const int32_t mb = P.max_batch, cnt = P.cnt;
  // While the candidate drains the queue its size is the queue length, so
  // it changes at every arrival and the timer is re-pushed each time: the
  // test at arrival k depends only on (q, k).
  int64_t now = tick[q];
  for (int32_t k = q; k < cnt; k++) {
    const int32_t len = k - q + 1;
    if (len > mb) return NX_UNSURE;  // capped: would not drain
    const int64_t delay = dc + dd * len;
    // b == len  <=>  ok(len) (monotone); also excludes head drops
    if (now + delay + lat(len - 1) > d) return NX_UNSURE;
    const int64_t l_next = len < mb ? lat(len) : lat(mb - 1);
    const int64_t exec = now + delay > d - l_next ? now + delay : d - l_next;
    const int64_t f = exec - delay;
    const int64_t fire = f < now ? now : f;
    if (k + 1 >= cnt) return NX_LAST_LEAN;
    const int64_t next = tick[k + 1];
    if (fire <= next) return P.off + k + 1;
    now = next;
  }
  return NX_UNSURE;
}

// lean_chain_next in 32-bit arithmetic relative to the head's tick, for an
// affine l(b).  Every quantity compared is within [0, slo + l(max_batch) +
// delay(max_batch)] of the head tick as long as the batch is still open
// (now <= deadline - l(1) - delay(1)), so int32 is exact when that bound is
// below 2^31 -- the caller checks it (rel32_ok) and otherwise uses the
// 64-bit form.  The next tick is compared after clamping at the bound.
SYM_HD bool rel32_ok(const Shard& S, const ModelParam& P) {
  const int64_t top = P.slo + P.aff_a * (int64_t)P.max_batch + P.aff_b +
                      S.d_ctrl + S.d_data * (int64_t)P.max_batch;
  return P.affine && S.kind == K_DEFERRED && S.gather == G_PREFIX && top < (int64_t(1) << 30) &&
         P.aff_a >= 0 && P.aff_b >= 0;
}

SYM_HD int32_t lean_chain_next32(const Shard& S, int32_t m, int32_t q) {
  const ModelParam& P = S.mp[m];
  const int64_t* tick = S.s_tick + P.off;
  const int64_t t0 = tick[q];
  const int32_t la = (int32_t)P.aff_a, lb0 = (int32_t)P.aff_b;
  const int32_t dc = (int32_t)S.d_ctrl, dd = (int32_t)S.d_data;
  const int32_t d = (int32_t)P.slo;  // deadline relative to the head
  const int32_t mb = P.max_batch, cnt = P.cnt;
  const int64_t cap = int64_t(1) << 30;
  int32_t now = 0;
  for (int32_t k = q; k < cnt; k++) {
    const int32_t len = k - q + 1;
    if (len > mb) return NX_UNSURE;
    const int32_t delay = dc + dd * len;
    if (now + delay + la * len + lb0 > d) return NX_UNSURE;  // b < len
    const int32_t l_next = la * (len < mb ? len + 1 : mb) + lb0;
    const int32_t exec = now + delay > d - l_next ? now + delay : d - l_next;
    const int32_t f = exec - delay;
    const int32_t fire = f < now ? now : f;
    if (k + 1 >= cnt) return NX_LAST;
    const int64_t nx = tick[k + 1] - t0;
    const int32_t next = (int32_t)(nx < cap ? nx : cap);
    if (fire <= next) return P.off + k + 1;
    now = next;
  }
  return NX_UNSURE;
}

// lean_chain_next for an exactly affine l(b) = a*b + b0, restated on
// u_j = tick_j + c1*j with c1 = a + d_data.  With len = k - q + 1 and
// len < max_batch the closing test  d_q - l(len+1) - delay(len) <= tick_{k+1}
// is  u_{k+1} >= u_q + (slo - a - b0 - d_ctrl),  and ok(len) is
// u_k <= u_q + (slo - d_ctrl - b0 - c1); both sides are exact int64, so the
// scan is one load, one multiply-add and one compare per step instead of the
// full candidate arithmetic.  ok is monotone in k, so it is checked once at
// the closing index.  The len == max_batch step (l_next = l(max_batch)) and
// the last arrival keep the scalar form.  Equals lean_chain_next at every
// position (tools/hostcheck).
SYM_HD int32_t lean_chain_next_affine_tail(const Shard& S, const ModelParam& P, int32_t q);

SYM_HD int32_t lean_chain_next_affine(const Shard& S, const ModelParam& P, int32_t q) {
  const int64_t* tick = S.s_tick + P.off;
  const int64_t a = P.aff_a, b0 = P.aff_b, dc = S.d_ctrl, dd = S.d_data;
  const int64_t c1 = a + dd;
  const int32_t mb = P.max_batch, cnt = P.cnt;
  const int64_t uq = tick[q] + c1 * q;
  const int64_t T = uq + (P.slo - a - b0 - dc);
  const int64_t OK = uq + (P.slo - dc - b0 - c1);
  const int32_t kmax = cnt - 2 < q + mb - 2 ? cnt - 2 : q + mb - 2;  // len < mb, k+1 < cnt
  int32_t k = q;
  while (k <= kmax && tick[k + 1] + c1 * (k + 1) < T) k++;
  if (k <= kmax)  // closes at k
    return tick[k] + c1 * k <= OK ? P.off + k + 1 : NX_UNSURE;
  return lean_chain_next_affine_tail(S, P, q);
}

// The not-closed-below-max_batch tail of lean_chain_next_affine: every k up
// to kmax must be ok, then the step at k1 = min(cnt - 1, q + mb - 1) in the
// scalar form (l_next = l(max_batch) at the cap).
SYM_HD int32_t lean_chain_next_affine_tail(const Shard& S, const ModelParam& P, int32_t q) {
  const int64_t* tick = S.s_tick + P.off;
  const int64_t a = P.aff_a, b0 = P.aff_b, dc = S.d_ctrl, dd = S.d_data;
  const int64_t c1 = a + dd;
  const int32_t mb = P.max_batch, cnt = P.cnt;
  const int64_t OK = tick[q] + c1 * q + (P.slo - dc - b0 - c1);
  const int32_t kmax = cnt - 2 < q + mb - 2 ? cnt - 2 : q + mb - 2;
  const int32_t k1 = kmax + 1;
  if (k1 - q + 1 > mb) return NX_UNSURE;
  const int64_t now = tick[k1];
  if (now + c1 * k1 > OK) return NX_UNSURE;  // ok(len) fails at k1 (or earlier)
  if (k1 + 1 >= cnt) return NX_LAST;
  const int32_t len = k1 - q + 1;  // == mb here
  const int64_t d = tick[q] + P.slo;
  const int64_t delay = dc + dd * len;
  const int64_t l_next = a * mb + b0;
  const int64_t exec = now + delay > d - l_next ? now + delay : d - l_next;
  const int64_t f = exec - delay;
  const int64_t fire = f < now ? now : f;
  return fire <= tick[k1 + 1] ? P.off + k1 + 1 : NX_UNSURE;
}

// Monotone sweep of lean_chain_next over consecutive positions [q0, q1) of
// model m.  For a start q the batch closes at the first k with
//   fire(q, k) = max(a_k, d_q - l(len+1) - delay(len)) <= a_{k+1},
// len = k - q + 1.  Moving the start to q+1 raises d and lowers len, so
// fire(q+1, k) >= fire(q, k): close(q+1, k) implies close(q, k), and the
// regime tests ok(len) / len <= max_batch only get weaker.  Hence the
// closing index never moves backwards and one forward pointer serves the
// whole range (two-pointer sweep, O(q1 - q0 + b) instead of O((q1 - q0) b)).
// The result for each q equals lean_chain_next(S, m, q) (host-verified).
// `tick(k)` returns the k-th (model-relative) arrival tick; the CUDA kernel
// serves it from a shared-memory window.
template <class Emit, class Tick>
SYM_HD void lean_chain_sweep(const Shard& S, int32_t m, int32_t q0, int32_t q1, Emit emit,
                             Tick tick) {
  const ModelParam& P = S.mp[m];
  if (S.kind != K_DEFERRED || S.gather != G_PREFIX) {
    for (int32_t q = q0; q < q1; q++) emit(q, NX_UNSURE, 0);
    return;
  }
  const int64_t* lat_row = S.lat + (int64_t)m * S.lat_stride;
  const bool aff = P.affine != 0;
  const int64_t la = P.aff_a, lb0 = P.aff_b;
  // l(b): exact affine form for linear profiles (no table loads), else the row
  auto lat = [&](int32_t i) { return aff ? la * (i + 1) + lb0 : lat_row[i]; };
  const int64_t dc = S.d_ctrl, dd = S.d_data;
  const int32_t mb = P.max_batch, cnt = P.cnt;
  int32_t k = q0;
  for (int32_t q = q0; q < q1; q++) {
    if (k < q) k = q;
    const int64_t d = tick(q) + P.slo;
    int32_t v = NX_UNSURE;
    for (;; k++) {
      const int32_t len = k - q + 1;
      if (len > mb) break;  // capped: would not drain (UNSURE)
      const int64_t now = tick(k);
      const int64_t delay = dc + dd * len;
      if (now + delay + lat(len - 1) > d) break;  // b < len (UNSURE)
      const int64_t l_next = len < mb ? lat(len) : lat(mb - 1);
      const int64_t exec = now + delay > d - l_next ? now + delay : d - l_next;
      const int64_t f = exec - delay;
      const int64_t fire = f < now ? now : f;
      if (k + 1 >= cnt) {
        v = NX_LAST;
        break;
      }
      if (fire <= tick(k + 1)) {
        v = P.off + k + 1;
        break;
      }
    }
    emit(q, v, k);
  }
}

template <class Emit>
SYM_HD void lean_chain_sweep(const Shard& S, int32_t m, int32_t q0, int32_t q1, Emit emit) {
  const int64_t* t = S.s_tick + S.mp[m].off;
  lean_chain_sweep(S, m, q0, q1, emit, [t](int32_t k) { return t[k]; });
}

// The batch a certified fresh start q produces, from (q, k) alone: the
// candidate (len, exec_at) at the closing arrival k and its model timer,
// pushed by arrival k (the size changes at every arrival in this regime).
SYM_HD void lean_batch(const Shard& S, int32_t m, int32_t q, int32_t k, EvBatch& e) {
  const ModelParam& P = S.mp[m];
  const int64_t* lat = S.lat + (int64_t)m * S.lat_stride;
  const int64_t* tick = S.s_tick + P.off;
  const int32_t len = k - q + 1, mb = P.max_batch;
  const int64_t d = tick[q] + P.slo, now = tick[k];
  const int64_t delay = S.d_ctrl + S.d_data * len;
  // affine rows need no table loads: l(b) = aff_a * b + aff_b
  const int64_t l_next = P.affine ? P.aff_a * (len < mb ? len + 1 : mb) + P.aff_b
                                  : (len < mb ? lat[len] : lat[mb - 1]);
  const int64_t exec = now + delay > d - l_next ? now + delay : d - l_next;
  const int64_t f = exec - delay;
  const int64_t fire = f < now ? now : f;
  const int32_t pos = P.off + k;
  e.t = fire;
  e.a = fire == now ? S.s_g[pos] + 1 : A_BASE;  // push_key with pusher = arrival k
  e.tp = now;
  e.ap = aself_at(S, pos);
  e.chain = 0;
  e.exec = exec;
  e.lat = P.affine ? P.aff_a * len + P.aff_b : lat[len - 1];
  e.size = len;
  e.first = P.off + q;
  e.model = m;
}

}  // namespace sym
