// multi.h -- the multi-device engine (multi.cu) behind the same handles:
// every C ABI entry point checks the handle's magic and forwards.
#pragma once
#include <stdint.h>

#include "../../include/symphony_b200.h"

constexpr uint32_t kSymSingleMagic = 0x53594d31u;  // "SYM1": one device (engine.cu)
constexpr uint32_t kSymMultiMagic = 0x53594d4du;   // "SYMM": several devices

bool sym_is_multi(const void* engine);
void* sym_multi_create(const sym_config* cfg, int32_t* status);
void sym_multi_destroy(void* engine);
const char* sym_multi_last_error(void* engine);
int32_t sym_multi_run(void* engine, const int64_t* ticks, const void* model, int64_t n,
                      uint32_t flags, sym_result* out);
int64_t sym_multi_last_batches(void* engine, sym_batch* host, int64_t cap);
// model_p99_ns == nullptr: only the counts (sym_window_counts)
int32_t sym_multi_window_stats(void* engine, int64_t lo_ns, int64_t hi_ns,
                               int64_t* model_arrivals, int64_t* model_completed,
                               int64_t* model_late, int64_t* model_dropped,
                               int64_t* gpu_busy_ns, int64_t* model_p99_ns,
                               int64_t* model_max_qd_ns, int64_t* model_batch_hist,
                               int32_t hist_stride);
