// partition.cu -- sub-cluster partitioning on the GPU (reference
// batchsym/partitioner.py).
//
// Three searches over assignments x: model -> sub-cluster, all scoring with
// the reference's evaluate (partitioner.py:114-145) in the same order of
// double-precision operations (explicit _rn intrinsics: no FMA contraction),
// so objectives and tie-breaks are bit-identical:
//   * brute force (partitioner.py:422-435): every one of l^m assignments, in
//     itertools.product order, one per thread; the lexicographically first
//     minimum of (infeasible, objective) wins.
//   * batch evaluation for the random baseline (partitioner.py:392-419): the
//     host draws rows from the reference's numpy stream, the GPU scores them.
//   * multi-start local search (partitioner.py:247-389): one warp per
//     restart runs greedy construction plus first-improvement moves and
//     swaps on the lexicographic (violation, objective) score.  The reference
//     runs restarts one after another under a wall-clock budget; here a
//     launch runs thousands of independent restarts at once.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <vector>

#include "../../include/symphony_b200.h"

namespace {

constexpr int kMaxL = 64;  // sub-clusters held in registers/local memory

struct Prob {
  int32_t m, l;
  const double *rates, *stat, *dyn;
  double rate_cap, mem_cap, w, r_bar, s_bar;
  const int32_t* current;  // may be null
  const double* cost;      // [m*l], may be null (=> 1.0)
  double budget;
};

__device__ __forceinline__ double cost_of(const Prob& p, int i, int j) {
  return p.cost ? p.cost[(int64_t)i * p.l + j] : 1.0;
}

__device__ __forceinline__ double move_cost(const Prob& p, int i, int jf, int jt) {
  return jf == jt ? 0.0 : __dadd_rn(cost_of(p, i, jf), cost_of(p, i, jt));
}

// evaluate(problem, x) (partitioner.py:114-145): returns the objective and
// whether the assignment is feasible.  `xof(i)` yields x[i].
template <class X>
__device__ __forceinline__ double evaluate(const Prob& p, X xof, bool* feasible) {
  double rate[kMaxL], mem[kMaxL], dyn[kMaxL];
  for (int j = 0; j < p.l; j++) rate[j] = mem[j] = dyn[j] = 0.0;
  for (int i = 0; i < p.m; i++) {
    const int j = xof(i);
    rate[j] = __dadd_rn(rate[j], p.rates[i]);
    mem[j] = __dadd_rn(mem[j], p.stat[i]);
    if (p.dyn[i] > dyn[j]) dyn[j] = p.dyn[i];
  }
  double d_rate = 0.0, d_mem = 0.0;
  bool ok = true;
  for (int j = 0; j < p.l; j++) {
    const double a = fabs(__dadd_rn(rate[j], -p.r_bar));
    const double b = fabs(__dadd_rn(mem[j], -p.s_bar));
    if (j == 0 || a > d_rate) d_rate = a;
    if (j == 0 || b > d_mem) d_mem = b;
    if (rate[j] > p.rate_cap) ok = false;
    if (__dadd_rn(mem[j], dyn[j]) > p.mem_cap) ok = false;
  }
  if (p.current) {
    double cc = 0.0;
    for (int i = 0; i < p.m; i++) cc = __dadd_rn(cc, move_cost(p, i, p.current[i], xof(i)));
    if (cc > p.budget) ok = false;
  }
  *feasible = ok;
  return __dadd_rn(d_rate, __dmul_rn(p.w, d_mem));
}

// (infeasible, objective, index): lexicographic, first index on ties
struct Best {
  double obj;
  int64_t idx;
  int32_t bad;
};

__device__ __forceinline__ bool better(const Best& a, const Best& b) {
  if (a.bad != b.bad) return a.bad < b.bad;
  if (a.obj != b.obj) return a.obj < b.obj;
  return a.idx < b.idx;
}

__device__ Best block_best(Best v) {
  __shared__ Best sh[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int d = 16; d; d >>= 1) {
    Best o;
    o.obj = __shfl_down_sync(0xffffffffu, v.obj, d);
    o.idx = __shfl_down_sync(0xffffffffu, v.idx, d);
    o.bad = __shfl_down_sync(0xffffffffu, v.bad, d);
    if (better(o, v)) v = o;
  }
  if (lane == 0) sh[w] = v;
  __syncthreads();
  if (w == 0) {
    v = lane < (int)(blockDim.x >> 5) ? sh[lane] : Best{INFINITY, INT64_MAX, 2};
    for (int d = 16; d; d >>= 1) {
      Best o;
      o.obj = __shfl_down_sync(0xffffffffu, v.obj, d);
      o.idx = __shfl_down_sync(0xffffffffu, v.idx, d);
      o.bad = __shfl_down_sync(0xffffffffu, v.bad, d);
      if (better(o, v)) v = o;
    }
  }
  return v;
}

// brute force: assignment k in itertools.product(range(l), repeat=m) order,
// x[0] the most significant base-l digit
__global__ void __launch_bounds__(256) k_brute(Prob p, int64_t total, Best* out) {
  Best best{INFINITY, INT64_MAX, 2};
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < total;
       k += (int64_t)gridDim.x * blockDim.x) {
    int32_t x[32];
    int64_t r = k;
    for (int i = p.m - 1; i >= 0; i--) {
      x[i] = (int32_t)(r % p.l);
      r /= p.l;
    }
    bool ok;
    const double obj = evaluate(p, [&](int i) { return x[i]; }, &ok);
    Best c{obj, k, ok ? 0 : 1};
    if (better(c, best)) best = c;
  }
  best = block_best(best);
  if (threadIdx.x == 0) out[blockIdx.x] = best;
}

// score rows of a [count x m] assignment matrix
__global__ void __launch_bounds__(256) k_eval_rows(Prob p, const int32_t* xs, int64_t count,
                                                   double* obj, int32_t* feasible, Best* out) {
  Best best{INFINITY, INT64_MAX, 2};
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t* x = xs + k * p.m;
    bool ok;
    const double o = evaluate(p, [&](int i) { return x[i]; }, &ok);
    obj[k] = o;
    feasible[k] = ok;
    Best c{o, k, ok ? 0 : 1};
    if (better(c, best)) best = c;
  }
  best = block_best(best);
  if (threadIdx.x == 0) out[blockIdx.x] = best;
}

__global__ void k_best(const Best* in, int n, Best* out) {
  Best best{INFINITY, INT64_MAX, 2};
  for (int k = threadIdx.x; k < n; k += blockDim.x)
    if (better(in[k], best)) best = in[k];
  best = block_best(best);
  if (threadIdx.x == 0) *out = best;
}

// ---------------------------------------------------- local search ------

struct Rng {  // splitmix64 stream per restart
  uint64_t s;
  __device__ uint64_t next() {
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  __device__ double uniform() { return (next() >> 11) * (1.0 / 9007199254740992.0); }
  __device__ int below(int n) { return (int)(next() % (uint64_t)n); }
};

__device__ __forceinline__ uint64_t now_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Per-restart search state, one warp per restart, in shared memory:
// per-sub-cluster sums, the dynamic peak as (top value, its multiplicity,
// runner-up) so the peak after removing any one member is O(1), and the
// change cost so far (_State, partitioner.py:166-236).
struct WarpState {
  double rate[kMaxL], mem[kMaxL], top1[kMaxL], top2[kMaxL];
  int32_t cnt1[kMaxL];
  double ccost, viol, obj;  // current score (viol, obj)
};

// Score with up to two sub-clusters replaced (j = -1: none):
// (violation, objective) exactly as _State.score (partitioner.py:199-211).
__device__ __forceinline__ void score_with(const Prob& p, const WarpState& w, int ja,
                                           double ra, double ma, double pa, int jb, double rb,
                                           double mb, double pb, double* viol, double* obj) {
  double v = 0.0, dr = 0.0, dm = 0.0;
  for (int j = 0; j < p.l; j++) {
    double r = w.rate[j], m = w.mem[j], pk = w.top1[j];
    if (j == ja) { r = ra; m = ma; pk = pa; }
    if (j == jb) { r = rb; m = mb; pk = pb; }
    v = __dadd_rn(v, fmax(0.0, __dadd_rn(r, -p.rate_cap)));
    v = __dadd_rn(v, fmax(0.0, __dadd_rn(__dadd_rn(m, pk), -p.mem_cap)));
    const double a = fabs(__dadd_rn(r, -p.r_bar));
    const double b = fabs(__dadd_rn(m, -p.s_bar));
    if (j == 0 || a > dr) dr = a;
    if (j == 0 || b > dm) dm = b;
  }
  *viol = v;
  *obj = __dadd_rn(dr, __dmul_rn(p.w, dm));
}

__device__ __forceinline__ bool lex_less(double v1, double o1, double v2, double o2) {
  return v1 < v2 || (v1 == v2 && o1 < o2);
}

// peak of sub-cluster j once member i (in j) leaves
__device__ __forceinline__ double peak_without(const Prob& p, const WarpState& w, int j, int i) {
  return (p.dyn[i] == w.top1[j] && w.cnt1[j] == 1) ? w.top2[j] : w.top1[j];
}

// Rebuild (top1, cnt1, top2) of sub-cluster j from the members; warp-wide.
__device__ void rebuild_peak(const Prob& p, WarpState& w, const int32_t* x, int j) {
  const int lane = threadIdx.x & 31;
  double t1 = 0.0;
  for (int i = lane; i < p.m; i += 32)
    if (x[i] == j && p.dyn[i] > t1) t1 = p.dyn[i];
  for (int d = 16; d; d >>= 1) t1 = fmax(t1, __shfl_xor_sync(0xffffffffu, t1, d));
  double t2 = 0.0;
  int c = 0;
  for (int i = lane; i < p.m; i += 32)
    if (x[i] == j) {
      if (p.dyn[i] == t1) c++;
      else if (p.dyn[i] > t2) t2 = p.dyn[i];
    }
  for (int d = 16; d; d >>= 1) {
    t2 = fmax(t2, __shfl_xor_sync(0xffffffffu, t2, d));
    c += __shfl_xor_sync(0xffffffffu, c, d);
  }
  __syncwarp();
  if (lane == 0) {
    w.top1[j] = t1;
    w.cnt1[j] = c;
    w.top2[j] = t2;
  }
  __syncwarp();
}

__device__ __forceinline__ double budget_delta(const Prob& p, const int32_t* x, int i, int jt) {
  if (!p.current) return 0.0;
  const int cur = p.current[i];
  return __dadd_rn(move_cost(p, i, cur, jt), -move_cost(p, i, cur, x[i]));
}

// One restart per warp: greedy construction (partitioner.py:247-280) or the
// current assignment for restart 0, then first-improvement single moves and
// pairwise swaps (partitioner.py:283-341) until a local optimum or the time
// budget.  The lanes score 32 candidate moves (or swap partners) at once;
// the first improving one in the reference's scan order is taken.
constexpr int kSolveWarps = 4;

__global__ void __launch_bounds__(32 * kSolveWarps)
k_solve(Prob p, const int32_t* order, uint64_t seed, int64_t r0, int32_t R, int32_t* xs,
        int32_t* perm, double* out_viol, double* out_obj, int64_t* out_steps,
        uint64_t budget_ns) {
  __shared__ WarpState ws[kSolveWarps];
  const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
  const int r = blockIdx.x * kSolveWarps + wi;
  if (r >= R) return;
  const uint64_t t_start = now_ns();
  WarpState& w = ws[wi];
  const int m = p.m, l = p.l;
  int32_t* x = xs + (int64_t)r * m;
  int32_t* pm = perm + (int64_t)r * m;
  Rng rng{seed * 0x100000001B3ull ^ (uint64_t)(r0 + r) * 0xD1B54A32D192ED03ull};
  if (lane == 0) {
    if (r0 + r == 0 && p.current) {
      for (int i = 0; i < m; i++) x[i] = p.current[i];
    } else {  // heaviest first onto the least-loaded feasible sub-cluster
      // The reference's restarts differ only by 1e-9 tie noise
      // (partitioner.py:255); with thousands of parallel restarts, 7 of every
      // 8 also scale the noise up to half the mean load so the local
      // searches start from (and end in) different regions.
      const double amp = 1e-9 + (double)((r0 + r) & 7) / 16.0 *
                                    __dadd_rn(fabs(p.r_bar), fabs(__dmul_rn(p.w, p.s_bar)));
      for (int j = 0; j < l; j++) w.rate[j] = w.mem[j] = w.top1[j] = 0.0;
      for (int k = 0; k < m; k++) {
        const int i = order[k];
        int best_j = 0;
        double bp = 0.0, bk = 0.0;
        for (int j = 0; j < l; j++) {
          const double nr = __dadd_rn(w.rate[j], p.rates[i]);
          const double nm = __dadd_rn(w.mem[j], p.stat[i]);
          const double nd = fmax(w.top1[j], p.dyn[i]);
          const double pen = __dadd_rn(fmax(0.0, __dadd_rn(nr, -p.rate_cap)),
                                       fmax(0.0, __dadd_rn(__dadd_rn(nm, nd), -p.mem_cap)));
          const double key = __dadd_rn(__dadd_rn(__dadd_rn(nr, -p.r_bar), __dmul_rn(p.w, nm)),
                                       rng.uniform() * amp);
          if (j == 0 || pen < bp || (pen == bp && key < bk)) {
            bp = pen;
            bk = key;
            best_j = j;
          }
        }
        x[i] = best_j;
        w.rate[best_j] = __dadd_rn(w.rate[best_j], p.rates[i]);
        w.mem[best_j] = __dadd_rn(w.mem[best_j], p.stat[i]);
        w.top1[best_j] = fmax(w.top1[best_j], p.dyn[i]);
      }
    }
  }
  __syncwarp();
  auto init = [&]() {  // sums, peaks and change cost from x
    if (lane == 0) {
      for (int j = 0; j < l; j++) w.rate[j] = w.mem[j] = 0.0;
      for (int i = 0; i < m; i++) {
        w.rate[x[i]] = __dadd_rn(w.rate[x[i]], p.rates[i]);
        w.mem[x[i]] = __dadd_rn(w.mem[x[i]], p.stat[i]);
      }
      double cc = 0.0;
      if (p.current)
        for (int i = 0; i < m; i++) cc = __dadd_rn(cc, move_cost(p, i, p.current[i], x[i]));
      w.ccost = cc;
    }
    __syncwarp();
    for (int j = 0; j < l; j++) rebuild_peak(p, w, x, j);
  };
  init();
  if (p.current && w.ccost > p.budget) {  // construction overshot the budget
    for (int i = lane; i < m; i += 32) x[i] = p.current[i];
    __syncwarp();
    init();
  }
  if (lane == 0) score_with(p, w, -1, 0, 0, 0, -1, 0, 0, 0, &w.viol, &w.obj);
  __syncwarp();
  int64_t steps = 0;
  bool timed_out = false;
  auto permute = [&]() {
    if (lane == 0) {
      for (int i = 0; i < m; i++) pm[i] = i;
      for (int i = m - 1; i > 0; i--) {
        const int j = rng.below(i + 1);
        const int32_t t = pm[i];
        pm[i] = pm[j];
        pm[j] = t;
      }
    }
    __syncwarp();
  };
  for (bool improved = true; improved && !timed_out;) {
    improved = false;
    permute();
    for (int k = 0; k < m && !timed_out; k++) {  // single-model moves
      const int i = pm[k], jf = x[i];
      const double left = __dadd_rn(p.budget, -w.ccost);
      const double pf = peak_without(p, w, jf, i);
      for (int jt0 = 0; jt0 < l; jt0 += 32) {
        const int jt = jt0 + lane;
        bool ok = false;
        double v = 0.0, o = 0.0;
        if (jt < l && jt != jf && !(budget_delta(p, x, i, jt) > left)) {
          score_with(p, w, jf, __dadd_rn(w.rate[jf], -p.rates[i]),
                     __dadd_rn(w.mem[jf], -p.stat[i]), pf, jt,
                     __dadd_rn(w.rate[jt], p.rates[i]), __dadd_rn(w.mem[jt], p.stat[i]),
                     fmax(w.top1[jt], p.dyn[i]), &v, &o);
          ok = lex_less(v, o, w.viol, w.obj);
        }
        const unsigned hit = __ballot_sync(0xffffffffu, ok);
        if (hit) {
          const int src = __ffs(hit) - 1;
          const int jt_best = jt0 + src;
          v = __shfl_sync(0xffffffffu, v, src);
          o = __shfl_sync(0xffffffffu, o, src);
          if (lane == 0) {
            w.ccost = __dadd_rn(w.ccost, budget_delta(p, x, i, jt_best));
            w.rate[jf] = __dadd_rn(w.rate[jf], -p.rates[i]);
            w.mem[jf] = __dadd_rn(w.mem[jf], -p.stat[i]);
            w.rate[jt_best] = __dadd_rn(w.rate[jt_best], p.rates[i]);
            w.mem[jt_best] = __dadd_rn(w.mem[jt_best], p.stat[i]);
            x[i] = jt_best;
            w.viol = v;
            w.obj = o;
          }
          __syncwarp();
          rebuild_peak(p, w, x, jf);
          rebuild_peak(p, w, x, jt_best);
          improved = true;
          steps++;
          break;
        }
      }
      if ((k & 7) == 7) timed_out = __shfl_sync(0xffffffffu, now_ns() - t_start > budget_ns, 0);
    }
    if (improved || timed_out) continue;
    permute();
    for (int k = 0; k < m && !improved && !timed_out; k++) {  // pairwise swaps
      const int a = pm[k], ja = x[a];
      const double left = __dadd_rn(p.budget, -w.ccost);
      const double pa_wo = peak_without(p, w, ja, a);
      for (int b0 = 0; b0 < m; b0 += 32) {
        const int b = b0 + lane;
        bool ok = false;
        double v = 0.0, o = 0.0;
        int jb = -1;
        if (b < m) {
          jb = x[b];
          if (jb != ja &&
              !(__dadd_rn(budget_delta(p, x, a, jb), budget_delta(p, x, b, ja)) > left)) {
            // a: ja -> jb, b: jb -> ja (apply_move(a) then apply_move(b))
            const double ra = __dadd_rn(__dadd_rn(w.rate[ja], -p.rates[a]), p.rates[b]);
            const double ma = __dadd_rn(__dadd_rn(w.mem[ja], -p.stat[a]), p.stat[b]);
            const double rb = __dadd_rn(__dadd_rn(w.rate[jb], p.rates[a]), -p.rates[b]);
            const double mb = __dadd_rn(__dadd_rn(w.mem[jb], p.stat[a]), -p.stat[b]);
            const double pka = fmax(pa_wo, p.dyn[b]);
            const double pkb = fmax(peak_without(p, w, jb, b), p.dyn[a]);
            score_with(p, w, ja, ra, ma, pka, jb, rb, mb, pkb, &v, &o);
            ok = lex_less(v, o, w.viol, w.obj);
          }
        }
        const unsigned hit = __ballot_sync(0xffffffffu, ok);
        if (hit) {
          const int src = __ffs(hit) - 1;
          const int bb = b0 + src;
          v = __shfl_sync(0xffffffffu, v, src);
          o = __shfl_sync(0xffffffffu, o, src);
          const int jbb = __shfl_sync(0xffffffffu, jb, src);
          if (lane == 0) {
            w.ccost = __dadd_rn(w.ccost, __dadd_rn(budget_delta(p, x, a, jbb),
                                                   budget_delta(p, x, bb, ja)));
            w.rate[ja] = __dadd_rn(__dadd_rn(w.rate[ja], -p.rates[a]), p.rates[bb]);
            w.mem[ja] = __dadd_rn(__dadd_rn(w.mem[ja], -p.stat[a]), p.stat[bb]);
            w.rate[jbb] = __dadd_rn(__dadd_rn(w.rate[jbb], p.rates[a]), -p.rates[bb]);
            w.mem[jbb] = __dadd_rn(__dadd_rn(w.mem[jbb], p.stat[a]), -p.stat[bb]);
            x[a] = jbb;
            x[bb] = ja;
            w.viol = v;
            w.obj = o;
          }
          __syncwarp();
          rebuild_peak(p, w, x, ja);
          rebuild_peak(p, w, x, jbb);
          improved = true;
          steps++;
          break;
        }
      }
      timed_out = __shfl_sync(0xffffffffu, now_ns() - t_start > budget_ns, 0);
    }
  }
  if (lane == 0) {
    // the incremental sums drift from a fresh left-to-right sum; report
    // the score of the final assignment recomputed from scratch
    for (int j = 0; j < l; j++) w.rate[j] = w.mem[j] = 0.0;
    for (int i = 0; i < m; i++) {
      w.rate[x[i]] = __dadd_rn(w.rate[x[i]], p.rates[i]);
      w.mem[x[i]] = __dadd_rn(w.mem[x[i]], p.stat[i]);
    }
  }
  __syncwarp();
  if (lane == 0) {
    score_with(p, w, -1, 0, 0, 0, -1, 0, 0, 0, &w.viol, &w.obj);
    out_viol[r] = w.viol;
    out_obj[r] = w.obj;
    out_steps[r] = steps;
  }
}

Prob to_prob(const sym_part_problem* q, const double* d_rates, const double* d_stat,
             const double* d_dyn, const int32_t* d_cur, const double* d_cost) {
  Prob p;
  p.m = q->m;
  p.l = q->l;
  p.rates = d_rates;
  p.stat = d_stat;
  p.dyn = d_dyn;
  p.rate_cap = q->rate_cap;
  p.mem_cap = q->mem_cap;
  p.w = q->weight;
  p.r_bar = q->mean_rate;
  p.s_bar = q->mean_mem;
  p.current = d_cur;
  p.cost = d_cost;
  p.budget = q->change_budget;
  return p;
}

// Device copy of a problem on a private stream (stream-ordered memory).
struct Dev {
  cudaStream_t st = nullptr;
  char* blob = nullptr;
  Prob p{};
  int prev = 0;
  int32_t init(const sym_part_problem* q, int device, size_t extra) {
    cudaGetDevice(&prev);
    if (cudaSetDevice(device) != cudaSuccess) return SYM_ECUDA;
    if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return SYM_ECUDA;
    const size_t m = (size_t)q->m, l = (size_t)q->l;
    const size_t bytes = 3 * m * 8 + m * 4 + 8 + m * l * 8 + extra + 64;
    if (cudaMallocAsync((void**)&blob, bytes, st) != cudaSuccess) return SYM_ENOMEM;
    double* r = (double*)blob;
    double* s = r + m;
    double* d = s + m;
    double* c = d + m;                           // m*l
    int32_t* cur = (int32_t*)(c + m * l);        // m
    if (cudaMemcpyAsync(r, q->rates, m * 8, cudaMemcpyHostToDevice, st) ||
        cudaMemcpyAsync(s, q->static_mem, m * 8, cudaMemcpyHostToDevice, st) ||
        cudaMemcpyAsync(d, q->dynamic_mem, m * 8, cudaMemcpyHostToDevice, st))
      return SYM_ECUDA;
    if (q->change_cost &&
        cudaMemcpyAsync(c, q->change_cost, m * l * 8, cudaMemcpyHostToDevice, st))
      return SYM_ECUDA;
    if (q->current && cudaMemcpyAsync(cur, q->current, m * 4, cudaMemcpyHostToDevice, st))
      return SYM_ECUDA;
    p = to_prob(q, r, s, d, q->current ? cur : nullptr, q->change_cost ? c : nullptr);
    return SYM_OK;
  }
  char* extra_ptr(const sym_part_problem* q) const {
    const size_t m = (size_t)q->m, l = (size_t)q->l;
    return blob + ((3 * m * 8 + m * l * 8 + m * 4 + 63) & ~size_t(63));
  }
  ~Dev() {
    if (blob) cudaFreeAsync(blob, st);
    if (st) {
      cudaStreamSynchronize(st);
      cudaStreamDestroy(st);
    }
    cudaSetDevice(prev);
  }
};

bool valid(const sym_part_problem* q) {
  return q && q->m >= 1 && q->l >= 1 && q->l <= kMaxL && q->rates && q->static_mem &&
         q->dynamic_mem;
}

}  // namespace

extern "C" {

int32_t sym_part_brute_force(const sym_part_problem* q, int32_t device, int32_t* best_x,
                             double* best_obj, int32_t* best_feasible) {
  if (!valid(q) || q->m > 32) return SYM_EINVAL;
  double total_d = pow((double)q->l, (double)q->m);
  if (total_d > 4.0e6) return SYM_EINVAL;  // partitioner.py:426-427
  int64_t total = 1;
  for (int i = 0; i < q->m; i++) total *= q->l;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 1184);
  Dev D;
  int32_t rc = D.init(q, device, sizeof(Best) * (blocks + 1));
  if (rc) return rc;
  Best* part = (Best*)D.extra_ptr(q);
  k_brute<<<blocks, 256, 0, D.st>>>(D.p, total, part);
  k_best<<<1, 256, 0, D.st>>>(part, blocks, part + blocks);
  Best h;
  if (cudaMemcpyAsync(&h, part + blocks, sizeof h, cudaMemcpyDeviceToHost, D.st) ||
      cudaStreamSynchronize(D.st) || cudaGetLastError())
    return SYM_ECUDA;
  int64_t r = h.idx;
  for (int i = q->m - 1; i >= 0; i--) {
    best_x[i] = (int32_t)(r % q->l);
    r /= q->l;
  }
  *best_obj = h.obj;
  *best_feasible = h.bad == 0;
  return SYM_OK;
}

int32_t sym_part_evaluate(const sym_part_problem* q, int32_t device, const int32_t* xs,
                          int64_t count, double* obj, int32_t* feasible, int64_t* best_index) {
  if (!valid(q) || count < 1) return SYM_EINVAL;
  const int blocks = (int)std::min<int64_t>((count + 255) / 256, 1184);
  const size_t rows = (size_t)count * q->m * 4;
  Dev D;
  int32_t rc = D.init(q, device, rows + count * 12 + sizeof(Best) * (blocks + 1) + 64);
  if (rc) return rc;
  char* e = D.extra_ptr(q);
  Best* part = (Best*)e;
  double* d_obj = (double*)(e + ((sizeof(Best) * (blocks + 1) + 15) & ~size_t(15)));
  int32_t* d_feas = (int32_t*)(d_obj + count);
  int32_t* d_x = d_feas + count;
  for (int64_t k = 0; k < count * q->m; k++)
    if (xs[k] < 0 || xs[k] >= q->l) return SYM_EINVAL;
  if (cudaMemcpyAsync(d_x, xs, rows, cudaMemcpyHostToDevice, D.st)) return SYM_ECUDA;
  k_eval_rows<<<blocks, 256, 0, D.st>>>(D.p, d_x, count, d_obj, d_feas, part);
  k_best<<<1, 256, 0, D.st>>>(part, blocks, part + blocks);
  Best h;
  if (cudaMemcpyAsync(obj, d_obj, count * 8, cudaMemcpyDeviceToHost, D.st) ||
      cudaMemcpyAsync(feasible, d_feas, count * 4, cudaMemcpyDeviceToHost, D.st) ||
      cudaMemcpyAsync(&h, part + blocks, sizeof h, cudaMemcpyDeviceToHost, D.st) ||
      cudaStreamSynchronize(D.st) || cudaGetLastError())
    return SYM_ECUDA;
  *best_index = h.idx;
  return SYM_OK;
}

int32_t sym_part_solve(const sym_part_problem* q, int32_t device, const int32_t* order,
                       uint64_t seed, int64_t first_restart, int32_t restarts,
                       double budget_s, int32_t* xs, double* viol, double* obj,
                       int64_t* steps) {
  if (!valid(q) || restarts < 1 || !order) return SYM_EINVAL;
  const size_t m = (size_t)q->m, R = (size_t)restarts;
  Dev D;
  int32_t rc = D.init(q, device, m * 4 + 2 * R * m * 4 + R * 24 + 64);
  if (rc) return rc;
  char* e = D.extra_ptr(q);
  double* d_viol = (double*)e;
  double* d_obj = d_viol + R;
  int64_t* d_steps = (int64_t*)(d_obj + R);
  int32_t* d_order = (int32_t*)(d_steps + R);
  int32_t* d_x = d_order + m;
  int32_t* d_perm = d_x + R * m;
  if (cudaMemcpyAsync(d_order, order, m * 4, cudaMemcpyHostToDevice, D.st)) return SYM_ECUDA;
  const uint64_t budget_ns = budget_s > 0 ? (uint64_t)(budget_s * 1e9) : UINT64_MAX;
  k_solve<<<(unsigned)((R + kSolveWarps - 1) / kSolveWarps), 32 * kSolveWarps, 0, D.st>>>(
      D.p, d_order, seed, first_restart, restarts, d_x, d_perm, d_viol, d_obj, d_steps,
      budget_ns);
  if (cudaMemcpyAsync(xs, d_x, R * m * 4, cudaMemcpyDeviceToHost, D.st) ||
      cudaMemcpyAsync(viol, d_viol, R * 8, cudaMemcpyDeviceToHost, D.st) ||
      cudaMemcpyAsync(obj, d_obj, R * 8, cudaMemcpyDeviceToHost, D.st) ||
      cudaMemcpyAsync(steps, d_steps, R * 8, cudaMemcpyDeviceToHost, D.st) ||
      cudaStreamSynchronize(D.st) || cudaGetLastError())
    return SYM_ECUDA;
  return SYM_OK;
}

}  // extern "C"
