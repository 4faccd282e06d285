// DEV TOOL ONLY: compiles the chain of csrc/engine_core.cuh for the host so
// the algorithm can be iterated against the oracle without a GPU round trip.
// Not part of the product (the package only ever loads the CUDA library).
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <vector>
#include <algorithm>
#include "../../paper_2308_07470_b200/csrc/engine_core.cuh"
#include "../../paper_2308_07470_b200/csrc/fastpath.cuh"
#include "../../oracle/symoracle.h"

using namespace sym;

extern "C" int32_t hc_run(int32_t use_fresh, const symo_config* cfg, const int64_t* ticks,
                          const int64_t* midx, int64_t n, int64_t* out_req5,
                          int64_t* out_ord7, int64_t* n_ord, int64_t* counters) {
  const int32_t M = cfg->n_models, G = cfg->n_gpus;
  std::vector<int32_t> cnt(M, 0), off(M + 1, 0);
  for (int64_t i = 0; i < n; i++) { if (midx[i] < 0 || midx[i] >= M) return 1; cnt[midx[i]]++; }
  for (int m = 0; m < M; m++) off[m + 1] = off[m] + cnt[m];
  std::vector<int64_t> s_tick(n); std::vector<int32_t> s_g(n), s_as(n);
  std::vector<int32_t> fill(off.begin(), off.end() - 1);
  for (int64_t i = 0; i < n; i++) {
    int p = fill[midx[i]]++;
    s_tick[p] = ticks[i]; s_g[p] = (int32_t)i;
    s_as[p] = (i > 0 && ticks[i - 1] == ticks[i]) ? (int32_t)i : A_BASE;
  }
  std::vector<ModelParam> mp(M);
  for (int m = 0; m < M; m++) {
    mp[m].slo = cfg->slo_ns[m]; mp[m].timeout_ns = cfg->timeout_ns[m];
    mp[m].base1 = cfg->d_ctrl_ns + cfg->d_data_ns + cfg->lat_ns[(int64_t)m * cfg->lat_stride];
    mp[m].off = off[m]; mp[m].cnt = cnt[m]; mp[m].max_batch = cfg->max_batch[m];
    mp[m].target_batch = std::min(cfg->target_batch, cfg->max_batch[m]);
    { const int64_t* row = cfg->lat_ns + (int64_t)m * cfg->lat_stride; int mb = cfg->max_batch[m];
      mp[m].aff_a = mb > 1 ? row[1] - row[0] : 0; mp[m].aff_b = row[0] - mp[m].aff_a; mp[m].affine = 1;
      for (int b = 0; b < mb; b++) if (row[b] != mp[m].aff_a * (b + 1) + mp[m].aff_b) mp[m].affine = 0; }
  }
  int32_t Mp = 1; while (Mp < M) Mp <<= 1;
  int32_t Gp = 1; while (Gp < G) Gp <<= 1;
  std::vector<ModelState> ms(M);
  std::vector<int32_t> pq(2 * Mp), gt(2 * Gp), mlt(2 * Mp), mbt(2 * Mp), mcs(M);
  std::vector<int64_t> fa(G), mcl(M), pqt(2 * Mp), gtf(2 * Gp), mltv(2 * Mp), mbtv(2 * Mp);
  std::vector<BatchRec> recs(n + 1);
  std::vector<int64_t> dt(n, -1), dks(n); std::vector<int32_t> dka(n);
  Shard S; memset(&S, 0, sizeof S);
  S.M = M; S.G = G; S.Mp = Mp; S.Gp = Gp; while ((1 << S.Mlog) < Mp) S.Mlog++; while ((1 << S.Glog) < Gp) S.Glog++; S.kind = cfg->kind; S.gather = cfg->gather;
  S.record_trace = 1; S.d_ctrl = cfg->d_ctrl_ns; S.d_data = cfg->d_data_ns;
  S.lat_stride = cfg->lat_stride; S.lat = cfg->lat_ns; S.mp = mp.data();
  S.s_tick = s_tick.data(); S.s_g = s_g.data(); S.sh_tick = ticks; S.sh_base = 0;
  S.ms = ms.data(); S.pq = pq.data(); S.free_at = fa.data(); S.gt = gt.data();
  S.mc_lat_tree = mlt.data(); S.mc_bs_tree = mbt.data(); S.mc_size = mcs.data(); S.mc_latest = mcl.data();
  S.pq_t = pqt.data(); S.gt_f = gtf.data(); S.mlt_v = mltv.data(); S.mbt_v = mbtv.data();
  S.check = 1; S.inject = -1;  // verify_state after every event
  S.recs = recs.data(); S.rec_cap = n + 1; S.drop_t = dt.data(); S.drop_ksub = dks.data(); S.drop_ka = dka.data();
  S.record_trace = use_fresh ? 0 : 1;
  std::vector<FreshRec> fresh;
  if (use_fresh) {
    fresh.resize(n);
    for (int m = 0; m < M; m++)
      for (int q = 0; q < cnt[m]; q++) fresh[off[m] + q] = fresh_scan(S, m, q, 4096);
  }
  chain_init(S, use_fresh ? fresh.data() : nullptr);
  std::vector<int32_t> dirty(M + 1);
  while (chain_step(S, dirty.data(), use_fresh ? fresh.data() : nullptr)) {}
  if (S.error) return 100 + S.error;
  for (int64_t i = 0; i < n; i++) { for (int k = 0; k < 4; k++) out_req5[k * n + i] = -1; out_req5[4 * n + i] = 2; }
  for (int64_t r = 0; r < S.n_recs; r++) {
    const BatchRec& b = recs[r];
    for (int j = 0; j < b.size; j++) {
      int64_t g = s_g[b.first + j];
      out_req5[0 * n + g] = b.emitted; out_req5[1 * n + g] = b.start; out_req5[2 * n + g] = b.finish;
      out_req5[3 * n + g] = b.size; out_req5[4 * n + g] = (b.finish <= s_tick[b.first + j] + mp[b.model].slo) ? 0 : 1;
    }
    int64_t* o = out_ord7 + 7 * r;
    o[0] = b.gpu; o[1] = b.model; o[2] = b.size; o[3] = b.start; o[4] = b.finish; o[5] = b.emitted; o[6] = b.shrunk_from;
  }
  *n_ord = S.n_recs;
  counters[0] = total_drops(S); counters[1] = S.ops; counters[2] = S.evictions; counters[3] = S.registrations;
  counters[4] = S.handler_ops_max; counters[5] = S.chain_events; counters[6] = S.absorbed; counters[7] = S.fresh_adoptions;
  // lean chain pointer vs the general scan, every position
  int64_t certified = 0, mismatch = 0;
  for (int m = 0; m < M; m++)
    for (int q = 0; q < cnt[m]; q++) {
      int32_t v = lean_chain_next(S, m, q);
      if (rel32_ok(S, mp[m]) && lean_chain_next32(S, m, q) != v) mismatch += 1000000000;
      if (mp[m].affine && S.kind == K_DEFERRED && S.gather == G_PREFIX &&
          lean_chain_next_affine(S, mp[m], q) != v) mismatch += 100000000;
      if (v == NX_UNSURE) continue;
      certified++;
      if (v != chain_next(fresh_scan(S, m, q, 1 << 16), mp[m])) mismatch++;
    }
  // monotone sweep == per-position lean result; lean_batch == general record
  for (int m = 0; m < M; m++) {
    for (int q0 = 0; q0 < cnt[m]; q0 += 7) {
      int q1 = std::min(cnt[m], q0 + 7);
      lean_chain_sweep(S, m, q0, q1, [&](int32_t q, int32_t v, int32_t k) {
        if (v != lean_chain_next(S, m, q)) mismatch += 1000;
        if (v == NX_UNSURE) return;
        FreshRec r = fresh_scan(S, m, q, 1 << 16);
        EvBatch e; lean_batch(S, m, q, k, e);
        if (e.t != r.mt_t || e.a != r.mt_a || e.tp != r.mt_tp || e.ap != r.mt_ap ||
            e.exec != r.c_exec || e.lat != r.c_lb || e.size != r.c_size ||
            e.first != off[m] + r.qh || r.drops != 0) mismatch += 1000000;
      });
    }
  }
  counters[8] = certified; counters[9] = mismatch;
  return 0;
}
