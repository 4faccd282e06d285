/*
 * symphony_b200.h -- C ABI of the B200-native Symphony scheduler engine.
 *
 * Drop-in boundary for the reference's simulate/step entry points:
 *   Engine(models, gpu_count, policy, network, seed, record_trace,
 *          check_invariants)          batchsym/simulator.py:99-140
 *   Engine.run_stream(arr_ticks, arr_midx, duration_s) -> RunResult
 *                                     batchsym/simulator.py:201-226, 65-87
 *   run_scenario(scenario, ...)       batchsym/scenario.py:264-273
 * The Python package paper_2308_07470_b200 mirrors those names on top of
 * this ABI (ctypes); see INTEGRATION.md for the binding a batchsym maintainer
 * would add.  Plain pointers and sizes only; all times are int64 ns ticks
 * (batchsym/units.py:1-17).
 *
 * A handle owns one CUDA stream and its device scratch on one device; it is
 * not thread-safe.  Every call is blocking (stream-synchronised on return).
 */
#ifndef SYMPHONY_B200_H
#define SYMPHONY_B200_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes: the Python layer maps them to the reference's
 * exception types */
enum {
  SYM_OK = 0,
  SYM_EPROTO = 1,     /* ProtocolError: unknown model id in the stream
                         (simulator.py:213-215) */
  SYM_EINVAL = 2,     /* ValueError: bad configuration (simulator.py:103-104,
                         scheduler.py:70-82) */
  SYM_EINVARIANT = 3, /* InvariantViolation (simulator.py:90-91) */
  SYM_ECUDA = 4,      /* CUDA runtime failure -> RuntimeError */
  SYM_ENOMEM = 5,
  SYM_EGUARD = 6      /* guard mode (SYM_GUARD=1): a device write outside its
                         buffer -> RuntimeError naming the buffer */
};

enum { SYM_KIND_DEFERRED = 0, SYM_KIND_EAGER = 1, SYM_KIND_TIMEOUT = 2 };
enum { SYM_GATHER_PREFIX = 0, SYM_GATHER_DROP_HEAD = 1 };

/* run flags */
enum {
  SYM_FLAG_TRACE = 1u,      /* record_trace=True: per-drop keys for the trace */
  SYM_FLAG_NO_FRESH = 2u,   /* disable the parallel fresh-start pre-scan */
  SYM_FLAG_NO_EXPAND = 4u,  /* leave per-request arrays untouched (bench) */
  SYM_FLAG_NO_FAST = 8u,    /* always run the sequential live-event chain */
  SYM_FLAG_KERNEL_TIMES = 16u, /* CUDA-event time every kernel (profiling) */
  SYM_FLAG_MODEL_I64 = 32u,   /* arr_model holds int64 ids (numpy default) */
  SYM_FLAG_CHECK_INVARIANTS = 64u, /* check_invariants=True: the exact chain
                                 verifies the reference's invariants
                                 (simulator.py:276-305) after every event;
                                 a violation returns SYM_EINVARIANT */
  SYM_FLAG_INJECT_FAULT = 128u /* test hook (with CHECK_INVARIANTS): corrupt
                                 the state at the 10th chain event */
};

/* Engine configuration.  Models are numbered 0..n_models-1 in the order of
 * the reference's `models` list; a sub-cluster (shard) is an independent
 * Engine over its models and its own GPU sub-pool (scalebench.py:98-99,
 * PAPER.md:475-490).  With n_shards == 1 this is exactly the reference
 * Engine.  GPU ids are global: shard s owns the contiguous id range after
 * shards 0..s-1. */
typedef struct {
  int32_t n_models;
  int32_t n_gpus;             /* total = sum(gpus_per_shard) */
  int32_t kind;               /* PolicyConfig.kind (scheduler.py:62) */
  int32_t gather;             /* PolicyConfig.gather (scheduler.py:67) */
  int32_t target_batch;       /* PolicyConfig.target_batch (scheduler.py:68) */
  int32_t lat_stride;         /* row stride of lat_ns (>= max max_batch) */
  int64_t d_ctrl_ns;          /* PolicyConfig.d_ctrl_ns (scheduler.py:65) */
  int64_t d_data_ns;          /* PolicyConfig.d_data_ns (scheduler.py:66) */
  const int64_t *lat_ns;      /* [n_models * lat_stride]; LatencyProfile.lat_ns
                                 (profile.py:40), lat[b-1] = l(b) */
  const int32_t *max_batch;   /* [n_models] LatencyProfile.max_batch */
  const int64_t *slo_ns;      /* [n_models] ModelSpec.slo_ns (profile.py:122) */
  const int64_t *timeout_ns;  /* [n_models] resolve_timeout_ns (scheduler.py:84) */
  int32_t n_shards;           /* >= 1 */
  int32_t device;             /* CUDA device ordinal */
  const int32_t *shard_of_model; /* [n_models], NULL = all in shard 0 */
  const int32_t *gpus_per_shard; /* [n_shards], NULL = n_gpus in shard 0 */
  /* Jittered network (network.py:69-77, scheduler.py:197-200): per dispatch,
   * ctrl() + data() * b where a histogram delay is one numpy
   * Generator(Philox(net_key)).choice(vals, p) draw (vals[searchsorted(cdf,
   * u, 'right')]) and n == 0 means the constant (no draw).  Both n == 0:
   * jitterless.  Every sub-cluster starts its own stream (one Engine each). */
  int32_t net_ctrl_n, net_data_n;
  const int64_t *net_ctrl_vals, *net_data_vals;
  const double *net_ctrl_cdf, *net_data_cdf;
  int64_t net_ctrl_const, net_data_const;
  uint64_t net_key[2];
  /* Several devices in one call: with n_devices >= 2,
   * sub-cluster s runs on devices[s mod n_devices] and every call spans
   * them; results equal the one-device run.  NULL / 0 = `device` alone.
   * The device-pointer, step and kernel-timing entry points take
   * one-device handles only. */
  const int32_t *devices;
  int32_t n_devices;
  int32_t _pad_dev;
} sym_config;

/* Batch record = one ExecutionOrder (scheduler.py:123-135) / one gpu_logs
 * entry (simulator.py:322-323).  Records of one GPU appear in emission
 * order. */
typedef struct {
  int64_t emitted, start, finish;
  int64_t key_t, key_sub;   /* processing position of the granting event */
  int32_t key_a;
  int32_t model, gpu, size;
  int32_t first_index;      /* stream index of the batch's first member */
  int32_t shrunk_from;      /* pre-grant candidate size if it shrank, else 0 */
} sym_batch;

typedef struct {
  int64_t n;                  /* requests in the run */
  /* Per-request outputs, caller-allocated [n], index = stream position
   * (= rid - 1 for a single shard); RunResult fields simulator.py:74-78.
   * May be NULL with SYM_FLAG_NO_EXPAND. */
  int64_t *req_dispatch, *req_start, *req_finish, *req_batch, *req_outcome;
  /* optional (may be NULL): arrival, deadline = arrival + SLO, model id as
   * int64 -- the remaining RunResult arrays (simulator.py:71-73) */
  int64_t *req_arrival, *req_deadline, *req_model;
  /* Trace support (SYM_FLAG_TRACE): per request, tick and processing
   * position of its drop, -1 if not dropped. */
  int64_t *drop_t, *drop_key_sub;
  int32_t *drop_key_a;
  /* batch records, caller-allocated capacity batch_cap (n is always
   * enough); n_batches receives the count */
  sym_batch *batches;
  int64_t batch_cap;
  int64_t n_batches;
  /* counters, summed over shards */
  int64_t drops, completions, late;
  int64_t ops, evictions, registrations, handler_ops_max;
  int64_t chain_events, absorbed_arrivals, fresh_adoptions;
  int64_t launches;           /* kernels this call launched */
  int64_t fast_shards;        /* sub-clusters resolved by the parallel path */
  int64_t fast_fail_mask;     /* OR of the validation failures (fastpath.cuh) */
  /* device timings of the last run (CUDA events on the engine stream) */
  float ms_ingest, ms_fresh, ms_fast, ms_chain, ms_expand, ms_total;
  int64_t err_index;          /* offending stream index for SYM_EPROTO */
} sym_result;

/* Create an engine; returns NULL and sets *status on failure. */
void *sym_create(const sym_config *cfg, int32_t *status);
void sym_destroy(void *engine);

/* Host buffers in, host buffers out (end-to-end API: the H2D and D2H copies
 * are part of the call).  arr_model is int32, or int64 with
 * SYM_FLAG_MODEL_I64.  arr_ticks must be non-decreasing (generate_arrivals /
 * load_replay_trace guarantee it); a violation returns SYM_EINVAL with
 * err_index set. */
int32_t sym_run(void *engine, const int64_t *arr_ticks,
                const void *arr_model, int64_t n, uint32_t flags,
                sym_result *out);

/* Same, but every pointer in the call (arrivals, per-request outputs,
 * drop arrays and batches) is a DEVICE pointer on the engine's device;
 * nothing crosses PCIe except the counters.  Used with inputs already
 * resident in HBM. */
int32_t sym_run_device(void *engine, const int64_t *d_arr_ticks,
                       const void *d_arr_model, int64_t n, uint32_t flags,
                       sym_result *out);

/* ---- stepped runs (the reference's step API: scalebench._shard_loop drives
 * Engine._record_arrival / ModelPlane.on_new_request / _dispatch_event,
 * scalebench.py:67-84, simulator.py:201-242) ---------------------------------
 * sym_step_reset starts a stepped run on the handle (a whole-run call ends
 * it).  Each sym_step appends n arrivals (host buffers, stream order, ticks
 * non-decreasing and within [previous until_tick, until_tick]) and processes
 * every event with tick <= until_tick; the caller promises that later
 * arrivals have tick >= until_tick.  Queues, candidates, timers, the GPU
 * index and the registered sets stay on the device between calls.
 * until_tick = INT64_MAX drains the engine.  After the last step the run
 * equals one sym_run over the concatenated stream, bit for bit.  `out`
 * receives the cumulative counters (n = arrivals so far, n_batches, drops,
 * completions = requests dispatched so far).  Jitterless networks only. */
int32_t sym_step_reset(void *engine);
int32_t sym_step(void *engine, const int64_t *arr_ticks, const void *arr_model, int64_t n,
                 int64_t until_tick, uint32_t flags, sym_result *out);
/* RunResult arrays of every arrival so far (caller buffers of out->n =
 * arrivals-so-far entries; NULL pointers are skipped): outcomes of requests
 * whose completion tick is after the last until_tick are -1 (unresolved),
 * as in the reference mid-run.  Batch records in step order. */
int32_t sym_step_result(void *engine, sym_result *out);

/* Copy the last run's batch records (emission order per GPU) to a host
 * buffer of capacity cap; returns the count (or -status on failure). */
int64_t sym_last_batches(void *engine, sym_batch *host, int64_t cap);

/* Integer reductions of a finished run for compute_stats
 * (metrics.py:71-132): per model counts of completed/late/dropped among
 * arrivals in [lo_ns, hi_ns), per GPU busy ns clipped to the window.
 * Pointers are host arrays sized n_models / n_gpus. */
int32_t sym_window_counts(void *engine, int64_t lo_ns, int64_t hi_ns,
                          int64_t *model_arrivals, int64_t *model_completed,
                          int64_t *model_late, int64_t *model_dropped,
                          int64_t *gpu_busy_ns);

/* Everything else compute_stats (metrics.py:71-132) needs for the window,
 * on the device: the counts and busy time above, plus per model the p99
 * latency by nearest rank with drops as +inf (-1 = inf, 0 = no arrivals),
 * the largest queueing delay of a served request, and the batch-size
 * histogram of the batches starting in the window ([n_models][hist_stride],
 * hist_stride > max batch size).  Needs the last run's per-request outputs
 * on the device (valid until the next run). */
int32_t sym_window_stats(void *engine, int64_t lo_ns, int64_t hi_ns,
                         int64_t *model_arrivals, int64_t *model_completed,
                         int64_t *model_late, int64_t *model_dropped,
                         int64_t *gpu_busy_ns, int64_t *model_p99_ns,
                         int64_t *model_max_qd_ns, int64_t *model_batch_hist,
                         int32_t hist_stride);

const char *sym_last_error(void *engine);

/* JSON object {"kernel": [launches, total_ms], ...} accumulated over runs
 * made with SYM_FLAG_KERNEL_TIMES; reset != 0 clears the table.  The string
 * lives until the next call on the handle. */
const char *sym_kernel_times(void *engine, int32_t reset);
int32_t sym_version(void);

/* ---- result-file text (reference outputs.py:72-121) ----------------------
 * The per-request CSV bodies are formatted on the GPU: one thread per row
 * renders the decimal fields, a block scan places rows, the text stays in
 * HBM until fetched.  Rows only; the caller prepends the header line.
 *   SYM_TEXT_REQUESTS: requests.csv rows (outputs.py:72-88)
 *   SYM_TEXT_LATENCY:  latency.csv rows, served requests only
 *                      (outputs.py:112-121) */
enum { SYM_TEXT_REQUESTS = 0, SYM_TEXT_LATENCY = 1 };

typedef struct {
  int64_t n;                  /* requests; row i is request id i+1 */
  /* per-request int64 columns, host or device pointers (UVA); model ids
   * index `names` */
  const int64_t *req_model, *req_arrival, *req_dispatch, *req_start,
      *req_finish, *req_batch, *req_outcome;
  int32_t n_names, _pad;
  const char *names;          /* concatenated UTF-8 model names */
  const int64_t *name_off;    /* [n_names + 1] byte offsets into names */
} sym_text_columns;

/* Format on `device`; returns a text handle (NULL + *status on failure:
 * SYM_EINVAL for a model id outside names or an outcome outside -1..2) and
 * sets *out_len to the byte length. */
void *sym_text_format(int32_t kind, const sym_text_columns *cols, int32_t device,
                      int64_t *out_len, int32_t *status);
/* Copy the text to a host buffer of len bytes (len == *out_len). */
int32_t sym_text_fetch(void *text, char *dst, int64_t len);
void sym_text_free(void *text);

/* ---- sub-cluster partitioning (reference partitioner.py) ----------------
 * Scores follow evaluate (partitioner.py:114-145) operation for operation in
 * IEEE double, so objectives and tie-breaks match the reference exactly. */
typedef struct {
  int32_t m, l;                 /* models, sub-clusters (l <= 64) */
  const double *rates, *static_mem, *dynamic_mem;  /* [m] */
  double rate_cap, mem_cap;     /* +inf when absent */
  double weight;                /* effective_weight() */
  double mean_rate, mean_mem;   /* sum(x) / l, as the reference computes them */
  const int32_t *current;       /* [m] or NULL */
  const double *change_cost;    /* [m * l] or NULL (every entry 1.0) */
  double change_budget;
} sym_part_problem;

/* brute_force (partitioner.py:422-435): the first (itertools.product order)
 * minimum of (infeasible, objective) over all l^m <= 4e6 assignments. */
int32_t sym_part_brute_force(const sym_part_problem *p, int32_t device, int32_t *best_x,
                             double *best_obj, int32_t *best_feasible);
/* Score `count` assignments (row-major [count][m]); best_index is the first
 * minimum of (infeasible, objective) -- the random baseline's selection
 * (partitioner.py:392-419). */
int32_t sym_part_evaluate(const sym_part_problem *p, int32_t device, const int32_t *xs,
                          int64_t count, double *obj, int32_t *feasible,
                          int64_t *best_index);
/* `restarts` independent greedy + first-improvement local searches
 * (partitioner.py:247-389), restart ids first_restart.. (restart 0 starts
 * from `current` when given); order = models heaviest first.  One warp per
 * restart; a restart stops at its local optimum or after budget_s seconds
 * (<= 0: no limit).  Writes every restart's final assignment
 * [restarts][m], score (violation, objective) and improving steps. */
int32_t sym_part_solve(const sym_part_problem *p, int32_t device, const int32_t *order,
                       uint64_t seed, int64_t first_restart, int32_t restarts,
                       double budget_s, int32_t *xs, double *viol, double *obj,
                       int64_t *steps);

#ifdef __cplusplus
}
#endif
#endif
