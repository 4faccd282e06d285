// multi.cu -- one engine call over several B200s (SURVEY §8b "multi-GPU
// handled inside one call", §8e sub-cluster partitioning).
//
// Sub-clusters are independent ("no communications
// between dispatcher threads"), so sub-cluster s runs on device
// devices[s mod D] inside an ordinary single-device engine, and the
// multi-device engine is a composition of those engines through this
// library's own C ABI: the host splits the stream by device (stable, so each
// sub-stream keeps the reference's stream order), the devices run
// concurrently, and per-request results, batch records and window
// reductions are mapped back to global request, model and GPU ids.  Results
// equal the one-device run bit for bit; nothing crosses NVLink because no
// sub-cluster reads another's state.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <thread>
#include <vector>

#include "../../include/symphony_b200.h"
#include "multi.h"

namespace {

struct Child {
  void* h = nullptr;
  int device = 0;
  std::vector<int32_t> global_model;  // local model id -> global
  std::vector<int32_t> global_gpu;    // local GPU id -> global
  std::vector<int32_t> shards;        // global ids of its sub-clusters, in order
  std::vector<int64_t> idx;           // local stream index -> global (last run)
  std::vector<int64_t> ticks;         // staging of the last run's sub-stream
  std::vector<int32_t> model;
  int64_t n = 0;
  sym_result res{};
  std::vector<sym_batch> batches;
  int32_t rc = SYM_OK;
};

struct MultiCtx {
  uint32_t magic = kSymMultiMagic;
  int32_t M = 0, G = 0, P = 0, D = 0;
  std::vector<int32_t> child_of_model, local_of_model, shard_of_model, gpu_base;
  std::vector<int64_t> slo;  // by global model id (req_deadline)
  std::vector<Child> kids;
  std::vector<sym_batch> last_batches;  // merged, global ids
  bool has_run = false;
  std::string err, ktimes;
};

int host_threads() {
  const unsigned t = std::thread::hardware_concurrency();
  return (int)std::max(1u, std::min(16u, t));
}

// run f(lo, hi, t) over [0, n) in T contiguous spans on T threads
template <class F>
void parallel_spans(int64_t n, int T, F f) {
  if (T <= 1 || n < (1 << 16)) {
    f(int64_t(0), n, 0);
    return;
  }
  std::vector<std::thread> th;
  for (int t = 0; t < T; t++) {
    const int64_t lo = n * t / T, hi = n * (t + 1) / T;
    th.emplace_back([=] { f(lo, hi, t); });
  }
  for (auto& x : th) x.join();
}

}  // namespace

bool sym_is_multi(const void* engine) {
  return engine && *static_cast<const uint32_t*>(engine) == kSymMultiMagic;
}

void* sym_multi_create(const sym_config* cfg, int32_t* status) {
  *status = SYM_EINVAL;
  const int M = cfg->n_models, P = cfg->n_shards;
  if (!cfg->devices || cfg->n_devices < 2 || P < 1 || M < 1) return nullptr;
  MultiCtx* mc = new MultiCtx();
  mc->M = M;
  mc->G = cfg->n_gpus;
  mc->P = P;
  mc->D = std::min(cfg->n_devices, P);  // devices beyond P would sit idle
  mc->shard_of_model.assign(M, 0);
  mc->slo.assign(cfg->slo_ns, cfg->slo_ns + M);
  for (int m = 0; m < M; m++) {
    const int s = cfg->shard_of_model ? cfg->shard_of_model[m] : 0;
    if (s < 0 || s >= P) { delete mc; return nullptr; }
    mc->shard_of_model[m] = s;
  }
  mc->gpu_base.assign(P + 1, 0);
  for (int s = 0; s < P; s++) {
    const int g = cfg->gpus_per_shard ? cfg->gpus_per_shard[s] : cfg->n_gpus;
    if (g < 1) { delete mc; return nullptr; }
    mc->gpu_base[s + 1] = mc->gpu_base[s] + g;
  }
  if (mc->gpu_base[P] != cfg->n_gpus) { delete mc; return nullptr; }
  mc->kids.resize(mc->D);
  mc->child_of_model.assign(M, 0);
  mc->local_of_model.assign(M, 0);
  for (int d = 0; d < mc->D; d++) {
    Child& c = mc->kids[d];
    c.device = cfg->devices[d];
    for (int s = d; s < P; s += mc->D) c.shards.push_back(s);
    for (int m = 0; m < M; m++)
      if (mc->shard_of_model[m] % mc->D == d) {
        mc->child_of_model[m] = d;
        mc->local_of_model[m] = (int32_t)c.global_model.size();
        c.global_model.push_back(m);
      }
    for (int s : c.shards)
      for (int g = mc->gpu_base[s]; g < mc->gpu_base[s + 1]; g++) c.global_gpu.push_back(g);
    // the child's configuration: its models in global-id order, its
    // sub-clusters renumbered 0.. in global order
    const int Mc = (int)c.global_model.size();
    std::vector<int64_t> lat((size_t)Mc * cfg->lat_stride), slo(Mc), tmo(Mc);
    std::vector<int32_t> mb(Mc), som(Mc), gps;
    for (int k = 0; k < Mc; k++) {
      const int m = c.global_model[k];
      memcpy(&lat[(size_t)k * cfg->lat_stride], cfg->lat_ns + (size_t)m * cfg->lat_stride,
             sizeof(int64_t) * cfg->lat_stride);
      slo[k] = cfg->slo_ns[m];
      tmo[k] = cfg->timeout_ns ? cfg->timeout_ns[m] : 0;
      mb[k] = cfg->max_batch[m];
      som[k] = mc->shard_of_model[m] / mc->D;
    }
    for (int s : c.shards) gps.push_back(mc->gpu_base[s + 1] - mc->gpu_base[s]);
    sym_config cc = *cfg;
    cc.n_models = Mc;
    cc.n_gpus = (int32_t)c.global_gpu.size();
    cc.lat_ns = lat.data();
    cc.max_batch = mb.data();
    cc.slo_ns = slo.data();
    cc.timeout_ns = tmo.data();
    cc.n_shards = (int32_t)c.shards.size();
    cc.device = c.device;
    cc.shard_of_model = som.data();
    cc.gpus_per_shard = gps.data();
    cc.devices = nullptr;
    cc.n_devices = 0;
    int32_t st = 0;
    c.h = sym_create(&cc, &st);
    if (!c.h) {
      *status = st;
      sym_multi_destroy(mc);
      return nullptr;
    }
  }
  *status = SYM_OK;
  return mc;
}

void sym_multi_destroy(void* engine) {
  MultiCtx* mc = static_cast<MultiCtx*>(engine);
  for (Child& c : mc->kids)
    if (c.h) sym_destroy(c.h);
  delete mc;
}

const char* sym_multi_last_error(void* engine) {
  MultiCtx* mc = static_cast<MultiCtx*>(engine);
  return mc->err.c_str();
}

int32_t sym_multi_run(void* engine, const int64_t* ticks, const void* model_v, int64_t n,
                      uint32_t flags, sym_result* out) {
  MultiCtx* mc = static_cast<MultiCtx*>(engine);
  mc->has_run = false;
  mc->last_batches.clear();
  if (flags & SYM_FLAG_KERNEL_TIMES) flags &= ~SYM_FLAG_KERNEL_TIMES;
  const bool i64 = flags & SYM_FLAG_MODEL_I64;
  auto model_at = [&](int64_t i) -> int64_t {
    return i64 ? static_cast<const int64_t*>(model_v)[i] : static_cast<const int32_t*>(model_v)[i];
  };
  const int D = mc->D, T = host_threads();
  // pass 1: validate (first bad id / first time inversion in stream order)
  // and count each span's arrivals per device
  std::vector<std::vector<int64_t>> cnt(T, std::vector<int64_t>(D, 0));
  std::vector<int64_t> bad_id(T, INT64_MAX), bad_time(T, INT64_MAX);
  parallel_spans(n, T, [&](int64_t lo, int64_t hi, int t) {
    for (int64_t i = lo; i < hi; i++) {
      const int64_t m = model_at(i);
      if (m < 0 || m >= mc->M) {
        bad_id[t] = std::min(bad_id[t], i);
        continue;
      }
      if (i > 0 && ticks[i] < ticks[i - 1]) bad_time[t] = std::min(bad_time[t], i);
      cnt[t][mc->child_of_model[m]]++;
    }
  });
  const int64_t first_bad = *std::min_element(bad_id.begin(), bad_id.end());
  if (first_bad != INT64_MAX) {
    out->err_index = first_bad;
    mc->err = "request for unknown model";
    return SYM_EPROTO;
  }
  const int64_t first_inv = *std::min_element(bad_time.begin(), bad_time.end());
  if (first_inv != INT64_MAX) {
    out->err_index = first_inv;
    mc->err = "arrival ticks must be non-decreasing";
    return SYM_EINVAL;
  }
  // pass 2: stable split into per-device sub-streams with their global index
  std::vector<std::vector<int64_t>> base(T, std::vector<int64_t>(D, 0));
  for (int d = 0; d < D; d++) {
    int64_t run = 0;
    for (int t = 0; t < T; t++) {
      base[t][d] = run;
      run += cnt[t][d];
    }
    Child& c = mc->kids[d];
    c.n = run;
    c.ticks.resize(run);
    c.model.resize(run);
    c.idx.resize(run);
  }
  parallel_spans(n, T, [&](int64_t lo, int64_t hi, int t) {
    std::vector<int64_t> pos = base[t];
    for (int64_t i = lo; i < hi; i++) {
      const int64_t m = model_at(i);
      const int d = mc->child_of_model[m];
      Child& c = mc->kids[d];
      const int64_t j = pos[d]++;
      c.ticks[j] = ticks[i];
      c.model[j] = mc->local_of_model[m];
      c.idx[j] = i;
    }
  });
  // the devices run concurrently, one host thread each; every child writes
  // its per-request results into staging arrays of its own
  const bool want = out->req_dispatch && !(flags & SYM_FLAG_NO_EXPAND);
  const bool trace = (flags & SYM_FLAG_TRACE) && out->drop_t;
  struct Stage {
    std::vector<int64_t> r[5], dt, dks;
    std::vector<int32_t> dka;
  };
  std::vector<Stage> stage(D);
  std::vector<std::thread> th;
  for (int d = 0; d < D; d++) {
    th.emplace_back([&, d] {
      Child& c = mc->kids[d];
      Stage& sg = stage[d];
      sym_result r{};
      r.n = c.n;
      if (want)
        for (int k = 0; k < 5; k++) sg.r[k].resize(c.n);
      if (want) {
        r.req_dispatch = sg.r[0].data();
        r.req_start = sg.r[1].data();
        r.req_finish = sg.r[2].data();
        r.req_batch = sg.r[3].data();
        r.req_outcome = sg.r[4].data();
      }
      if (trace) {
        sg.dt.resize(c.n);
        sg.dks.resize(c.n);
        sg.dka.resize(c.n);
        r.drop_t = sg.dt.data();
        r.drop_key_sub = sg.dks.data();
        r.drop_key_a = sg.dka.data();
      }
      c.batches.resize(c.n + 1);
      r.batches = c.batches.data();
      r.batch_cap = c.n + 1;
      c.rc = sym_run(c.h, c.ticks.data(), c.model.data(), c.n,
                     flags & ~SYM_FLAG_MODEL_I64, &r);
      c.res = r;
      if (c.rc == SYM_OK) c.batches.resize(r.n_batches);
    });
  }
  for (auto& x : th) x.join();
  for (int d = 0; d < D; d++) {
    Child& c = mc->kids[d];
    if (c.rc != SYM_OK) {
      mc->err = std::string("device ") + std::to_string(c.device) + ": " +
                sym_last_error(c.h);
      if (c.rc == SYM_EPROTO && c.res.err_index >= 0 && c.res.err_index < c.n)
        out->err_index = c.idx[c.res.err_index];
      return c.rc;
    }
  }
  // per-request results back to global stream positions (disjoint writes)
  th.clear();
  for (int d = 0; d < D; d++) {
    th.emplace_back([&, d] {
      const Child& c = mc->kids[d];
      const Stage& sg = stage[d];
      int64_t* dst[5] = {out->req_dispatch, out->req_start, out->req_finish, out->req_batch,
                         out->req_outcome};
      for (int64_t j = 0; j < c.n; j++) {
        const int64_t i = c.idx[j];
        if (want)
          for (int k = 0; k < 5; k++) dst[k][i] = sg.r[k][j];
        if (out->req_arrival) out->req_arrival[i] = c.ticks[j];
        if (out->req_model) out->req_model[i] = c.global_model[c.model[j]];
        if (out->req_deadline) out->req_deadline[i] = c.ticks[j] + mc->slo[c.global_model[c.model[j]]];
        if (trace) {
          out->drop_t[i] = sg.dt[j];
          out->drop_key_sub[i] = sg.dks[j];
          out->drop_key_a[i] = sg.dka[j];
        }
      }
    });
  }
  for (auto& x : th) x.join();
  // batch records: sub-cluster s's records (emission order) come from
  // device s mod D, in global sub-cluster order as a one-device run lists
  // them; model, GPU and first-member ids become global
  std::vector<size_t> cur(D, 0);
  for (int s = 0; s < mc->P; s++) {
    const int d = s % D;
    Child& c = mc->kids[d];
    const int32_t g_lo = mc->gpu_base[s], g_hi = mc->gpu_base[s + 1];
    while (cur[d] < c.batches.size()) {
      sym_batch b = c.batches[cur[d]];
      const int32_t gg = c.global_gpu[b.gpu];
      if (gg < g_lo || gg >= g_hi) break;
      b.gpu = gg;
      b.model = c.global_model[b.model];
      b.first_index = (int32_t)c.idx[b.first_index];
      mc->last_batches.push_back(b);
      cur[d]++;
    }
  }
  const int64_t total = (int64_t)mc->last_batches.size();
  out->n = n;
  out->n_batches = total;
  if (out->batches) {
    if (total > out->batch_cap) {
      mc->err = "batch buffer too small";
      return SYM_EINVAL;
    }
    memcpy(out->batches, mc->last_batches.data(), sizeof(sym_batch) * total);
  }
  out->drops = out->completions = out->late = 0;
  out->ops = out->evictions = out->registrations = out->handler_ops_max = 0;
  out->chain_events = out->absorbed_arrivals = out->fresh_adoptions = 0;
  out->launches = out->fast_shards = out->fast_fail_mask = 0;
  out->ms_ingest = out->ms_fresh = out->ms_fast = out->ms_chain = out->ms_expand =
      out->ms_total = 0;
  for (const Child& c : mc->kids) {
    const sym_result& r = c.res;
    out->drops += r.drops;
    out->completions += r.completions;
    out->late += r.late;
    out->ops += r.ops;
    out->evictions += r.evictions;
    out->registrations += r.registrations;
    out->handler_ops_max = std::max(out->handler_ops_max, r.handler_ops_max);
    out->chain_events += r.chain_events;
    out->absorbed_arrivals += r.absorbed_arrivals;
    out->fresh_adoptions += r.fresh_adoptions;
    out->launches += r.launches;
    out->fast_shards += r.fast_shards;
    out->fast_fail_mask |= r.fast_fail_mask;
    // the devices run concurrently: the call's device time is the slowest
    out->ms_ingest = std::max(out->ms_ingest, r.ms_ingest);
    out->ms_fresh = std::max(out->ms_fresh, r.ms_fresh);
    out->ms_fast = std::max(out->ms_fast, r.ms_fast);
    out->ms_chain = std::max(out->ms_chain, r.ms_chain);
    out->ms_expand = std::max(out->ms_expand, r.ms_expand);
    out->ms_total = std::max(out->ms_total, r.ms_total);
  }
  mc->has_run = true;
  return SYM_OK;
}

int64_t sym_multi_last_batches(void* engine, sym_batch* host, int64_t cap) {
  MultiCtx* mc = static_cast<MultiCtx*>(engine);
  if (!mc->has_run) return -SYM_EINVAL;
  const int64_t total = (int64_t)mc->last_batches.size();
  if (total > cap) return -SYM_EINVAL;
  memcpy(host, mc->last_batches.data(), sizeof(sym_batch) * total);
  return total;
}

int32_t sym_multi_window_stats(void* engine, int64_t lo_ns, int64_t hi_ns,
                               int64_t* model_arrivals, int64_t* model_completed,
                               int64_t* model_late, int64_t* model_dropped,
                               int64_t* gpu_busy_ns, int64_t* model_p99_ns,
                               int64_t* model_max_qd_ns, int64_t* model_batch_hist,
                               int32_t hist_stride) {
  MultiCtx* mc = static_cast<MultiCtx*>(engine);
  if (!mc->has_run) {
    mc->err = "no successful run to reduce";
    return SYM_EINVAL;
  }
  const bool full = model_p99_ns != nullptr;
  for (Child& c : mc->kids) {
    const size_t Mc = c.global_model.size(), Gc = c.global_gpu.size();
    std::vector<int64_t> a(Mc), co(Mc), la(Mc), dr(Mc), busy(Gc), p99(Mc), qd(Mc),
        hist(full ? Mc * hist_stride : 1);
    const int32_t rc =
        full ? sym_window_stats(c.h, lo_ns, hi_ns, a.data(), co.data(), la.data(), dr.data(),
                                busy.data(), p99.data(), qd.data(), hist.data(), hist_stride)
             : sym_window_counts(c.h, lo_ns, hi_ns, a.data(), co.data(), la.data(), dr.data(),
                                 busy.data());
    if (rc != SYM_OK) {
      mc->err = sym_last_error(c.h);
      return rc;
    }
    for (size_t k = 0; k < Mc; k++) {
      const int m = c.global_model[k];
      model_arrivals[m] = a[k];
      model_completed[m] = co[k];
      model_late[m] = la[k];
      model_dropped[m] = dr[k];
      if (full) {
        model_p99_ns[m] = p99[k];
        model_max_qd_ns[m] = qd[k];
        memcpy(model_batch_hist + (size_t)m * hist_stride, &hist[k * hist_stride],
               sizeof(int64_t) * hist_stride);
      }
    }
    for (size_t g = 0; g < Gc; g++) gpu_busy_ns[c.global_gpu[g]] = busy[g];
  }
  return SYM_OK;
}
