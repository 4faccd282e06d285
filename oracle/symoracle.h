/*
 * symoracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement (plain C) of the reference scheduler hot path
 * (`batchsym` 0.1.0: scheduler.py ModelPlane/RankPlane + simulator.py
 * Engine.run_stream).  It is the parity checker for the CUDA engine and the
 * CPU baseline leg of bench.py; it is never linked into, or called by, the
 * product path (paper_2308_07470_b200/).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.
 *
 * Pinning: validated against the Python reference imported in the build
 * container (tests/golden/make_golden.py writes the fixtures it is checked
 * against by tests/test_oracle_golden.py).
 */
#ifndef SYMORACLE_H
#define SYMORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { SYMO_DEFERRED = 0, SYMO_EAGER = 1, SYMO_TIMEOUT = 2 };
enum { SYMO_GATHER_PREFIX = 0, SYMO_GATHER_DROP_HEAD = 1 };
enum { SYMO_OK = 0, SYMO_EPROTO = 1, SYMO_EINVAL = 2, SYMO_EINVARIANT = 3,
       SYMO_ENOMEM = 5 };
enum { SYMO_TR_DISPATCH = 0, SYMO_TR_DROP = 1, SYMO_TR_SHRINK = 2 };

typedef struct {
  int32_t n_models;
  int32_t n_gpus;
  int32_t kind;          /* SYMO_DEFERRED / EAGER / TIMEOUT */
  int32_t gather;        /* SYMO_GATHER_* */
  int32_t target_batch;  /* policy.target_batch (clipped per model inside) */
  int32_t record_trace;
  int32_t check_invariants;
  int32_t _pad;
  int64_t d_ctrl_ns;
  int64_t d_data_ns;
  const int64_t *lat_ns;      /* [n_models * lat_stride], lat[b-1] */
  int32_t lat_stride;
  int32_t _pad2;
  const int32_t *max_batch;   /* [n_models] */
  const int64_t *slo_ns;      /* [n_models] */
  const int64_t *timeout_ns;  /* [n_models], resolved per model */
  /* jittered network (network.py:69-77): a histogram delay is one
   * Generator(Philox(key)).choice(vals, p) draw; n == 0 means the constant
   * value (no draw).  Both constant => no sampling (simulator.py:116-117). */
  int32_t net_ctrl_n, net_data_n;
  const int64_t *net_ctrl_vals, *net_data_vals;
  const double *net_ctrl_cdf, *net_data_cdf;
  int64_t net_ctrl_const, net_data_const;
  uint64_t net_key[2];
} symo_config;

typedef struct {
  int64_t n;
  /* per-request arrays, caller-allocated length n (index = rid-1) */
  int64_t *req_dispatch, *req_start, *req_finish, *req_batch, *req_outcome;
  /* filled by the library (malloc'd; free with symo_free_result) */
  int64_t n_orders;      /* dispatched batches, in emission order */
  int32_t *ord_gpu, *ord_model, *ord_size;
  int64_t *ord_start, *ord_finish, *ord_emitted;
  int64_t n_trace;
  int64_t *tr_t, *tr_start, *tr_finish;
  int32_t *tr_kind, *tr_model, *tr_gpu, *tr_size;
  int64_t *tr_rid_off;   /* [n_trace + 1] offsets into tr_rids */
  int64_t *tr_rids;
  /* counters */
  int64_t drops, completions, late;
  int64_t ops, evictions, registrations, handler_ops_max;
  int64_t events_popped, events_pushed;
  int64_t err_index;     /* arrival index that raised, or -1 */
} symo_result;

int32_t symo_run(const symo_config *cfg, const int64_t *arr_ticks,
                 const int64_t *arr_midx, int64_t n, symo_result *out);
void symo_free_result(symo_result *out);

#ifdef __cplusplus
}
#endif
#endif
