// engine.cu -- B200 (sm_100a) kernels and the C ABI of include/symphony_b200.h.
//
// Pipeline of one run (all on the engine's stream, inputs resident in HBM):
//   K1  k_part_count / flat scan / k_part_binoff / k_part
//                   stable partition to the (shard, model)-sorted layout
//                   (two passes with several sub-clusters: by sub-cluster,
//                   then by model), warp __match_any_sync ranking
//   (A' of an arrival -- same-tick cascades -- is derived on the fly, aself_at)
//   K2  k_nxt_tma   batch-chain pointers (bulk-copied tiles, binary search)
//   K3  k_jump4 / k_walk / k_walk_expand / k_chain_recs / bucket sorts /
//       k_match_coop / k_tie_fix / k_fast_emit   the parallel validated path
//       (fastpath.cuh); k_fresh / k_chain for sub-clusters that fail it
//   K4  k_chain     one CTA per sub-cluster runs the live-event chain
//   K5  k_bid / k_out  per-request RunResult arrays from batch records
// The chain (engine_core.cuh) is the only sequential part; everything else is
// a bandwidth-bound pass over the request stream.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <map>
#include <chrono>
#include <cstdlib>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/symphony_b200.h"
#include "engine_core.cuh"
#include "fastpath.cuh"
#include "multi.h"

using namespace sym;

namespace {

constexpr int kChunkR = 256;      // keys per warp in the radix passes
constexpr int kFreshMaxSteps = 1 << 16;
constexpr int kVersion = 1;

struct Ctx {
  uint32_t magic = kSymSingleMagic;  // first member: multi.h tells the handles apart
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev[6] = {};
  std::string err;
  // configuration
  int32_t M = 0, G = 0, P = 1, kind = 0, gather = 0, lat_stride = 1;
  int64_t d_ctrl = 0, d_data = 0;
  std::vector<int32_t> shard_of_model, slot_of_model, model_of_slot;
  std::vector<int32_t> slot_base;   // [P+1] first slot of each shard
  std::vector<int32_t> gpu_base;    // [P+1]
  std::vector<ModelParam> mp_host;  // by slot
  // static device data
  int64_t* d_lat = nullptr;         // rows in slot order
  ModelParam* d_mp = nullptr;       // [M] by slot
  int32_t* d_slot_of_model = nullptr;
  int32_t* d_shard_of_model = nullptr;
  int32_t* d_slot_base = nullptr;   // [P+1]
  int64_t* d_slo_model = nullptr;   // [M] SLO by global model id
  // jittered network
  bool jitter = false;
  int32_t net_ctrl_n = 0, net_data_n = 0;
  int64_t net_ctrl_const = 0, net_data_const = 0;
  uint64_t net_key[2] = {0, 0};
  int64_t* d_net_vals = nullptr;   // ctrl vals | data vals
  double* d_net_cdf = nullptr;     // ctrl cdf | data cdf
  // chain state (independent of n)
  ModelState* d_ms = nullptr;
  int32_t *d_pq = nullptr, *d_gt = nullptr, *d_mlt = nullptr,
          *d_mbt = nullptr, *d_mcs = nullptr, *d_dirty = nullptr;
  int64_t *d_pqt = nullptr, *d_gtf = nullptr, *d_mltv = nullptr, *d_mbtv = nullptr;
  int64_t *d_free = nullptr, *d_mcl = nullptr;
  Shard* d_shards = nullptr;
  std::vector<Shard> shards;        // host images
  size_t chain_smem = 0;            // dynamic smem of k_chain
  int64_t max_slo = 0, max_lat = 0; // bounds for the sort-key width
  // per-run buffers (grown)
  int64_t cap = 0;
  int64_t *d_ticks = nullptr, *d_s_tick = nullptr, *d_sh_tick = nullptr;
  int32_t *d_bid = nullptr;         // stream index -> batch record (k_bid)
  int32_t *d_model = nullptr, *d_s_g = nullptr, *d_s_i = nullptr;
  int32_t* d_bins = nullptr;        // [B+1] (unused) | shard_off | model_of_slot | gpu_base
  int32_t *d_sh_i = nullptr, *d_sh_slot = nullptr;  // P > 1: level 1
  int32_t* d_hist = nullptr;        // [B][tiles] bin counts -> positions
  int32_t* d_hist_part = nullptr;   // block sums of its scan
  int32_t *d_bkt = nullptr, *d_bkt_part = nullptr;  // bucket sort counts / ends
  int64_t* d_seg = nullptr;         // [4*(P+1)] segmented partition geometry
  int64_t bkt_cap = 0;
  int64_t hist_cap = 0;
  int32_t* d_err = nullptr;
  FreshRec* d_fresh = nullptr;
  BatchRec* d_recs = nullptr;
  // fast path scratch
  EvBatch* d_evb = nullptr;
  uint64_t *d_bkA = nullptr, *d_bkB = nullptr, *d_tkA = nullptr, *d_tkB = nullptr;
  uint32_t *d_bvA = nullptr, *d_bvB = nullptr, *d_tvA = nullptr, *d_tvB = nullptr;
  int32_t *d_ptrA = nullptr, *d_rhist = nullptr;
  int32_t *d_nb = nullptr, *d_bbase = nullptr, *d_changed = nullptr;
  int64_t *d_mdrops = nullptr, *d_sbase = nullptr;
  uint32_t* d_fail = nullptr;
  int32_t* d_skip = nullptr;
  int64_t* d_meta = nullptr;       // [3*(P+1)]: rec_base | rec_count | spare
  int32_t* d_scan_part = nullptr;   // block sums of flat_scan
  // staging for the host-buffer entry point (grown, never freed per call)
  int64_t *d_req = nullptr, *d_drop = nullptr;
  int32_t* d_dka = nullptr;
  sym_batch* d_bat = nullptr;
  int64_t stage_cap = 0, bat_cap = 0;
  int32_t* d_closek = nullptr;      // closing arrival of each batch start (-1: general)
  int32_t* d_special = nullptr;     // [M] models left to the sequential evolution
  int32_t *d_jC = nullptr;          // J_64 kept while J_256 is built
  int32_t *d_unsure = nullptr;      // [n] positions the lean pointer could not certify
  int32_t *d_unsure_n = nullptr;    // [1] their count
  int32_t *d_cpoff = nullptr;       // [M+1] compact checkpoint offsets (k_cp_scan)
  // tie groups (k_match_coop -> k_tie_fix -> k_fast_emit), per sub-cluster
  int32_t *d_tie_cnt = nullptr, *d_tie_list = nullptr;
  int4* d_tie_eff = nullptr;        // effective groups: R, E, pair offset, pair count
  int2* d_tie_sig = nullptr;        // label pairs old -> new
  uint32_t* d_tie_mask = nullptr;   // [P][32] hashed old labels
  int32_t *d_nxt = nullptr, *d_jA = nullptr, *d_jB = nullptr, *d_cp_pos = nullptr,
          *d_cp_model = nullptr;
  int64_t *d_drop_t = nullptr, *d_drop_ks = nullptr;
  int32_t* d_drop_ka = nullptr;
  // last run (for sym_window_counts)
  int64_t last_n = 0;
  const int64_t* last_ticks = nullptr;
  const int32_t* last_model = nullptr;
  std::vector<int64_t> last_nrecs, last_rec_base;
  const int64_t* last_outcome = nullptr;
  const int64_t* last_start = nullptr;   // per-request start / finish of the
  const int64_t* last_finish = nullptr;  // last expanded run (device)
  std::vector<uint32_t> last_fast_fail;
  bool has_run = false;
  std::map<std::string, std::pair<int64_t, double>> ktimes;  // name -> (launches, ms)
  std::string ktimes_json;
  // ---- stepped run (sym_step): the chain's state persists in the chain
  // arrays above (d_ms, d_free, trees) and the device Shard images; the
  // sorted layout holds each model's unresolved arrivals followed by the
  // new ones, double buffered and rebuilt every step
  bool step_active = false, step_first = true;
  int64_t step_n = 0;                 // arrivals so far (stream length)
  int64_t step_until = INT64_MIN;     // until_tick of the previous step
  int64_t step_served = 0, step_drops = 0;
  int64_t g_cap = 0;                  // capacity of the per-request arrays
  int64_t* d_g_ticks = nullptr;       // every arrival so far, stream order
  int32_t* d_g_model = nullptr;
  int64_t* d_g_out = nullptr;         // [5][g_cap] dispatch start finish batch outcome
  int64_t lay_cap = 0, lay_n = 0;
  int cur = 0;
  int64_t* d_lay_tick[2] = {nullptr, nullptr};
  int32_t* d_lay_g[2] = {nullptr, nullptr};
  int32_t* d_lay_i[2] = {nullptr, nullptr};
  int32_t* d_lay_aself[2] = {nullptr, nullptr};
  int32_t* d_lay_flag = nullptr;      // served flag per layout position
  ModelParam* d_mp_chunk = nullptr;   // off/cnt of the chunk's own sorted layout
  int32_t* d_step_slot = nullptr;     // [4*(M+1)]: newcnt | newoff | keep | oldsrc
  int64_t* d_step_shard = nullptr;    // [3*P]: shard base | last tick | has-previous
  int64_t* d_step_cnt = nullptr;      // [2]: served, dropped this step
  std::vector<int64_t> shard_count, shard_last;
  sym_batch* d_gbat = nullptr;
  int64_t gbat_cap = 0, gbat_n = 0;
  // guard mode (SYM_GUARD=1 when the engine is created): every device buffer
  // sits between two redzones, its body filled with a poison byte
  // (SYM_GUARD_POISON), and each run ends by checking every redzone
  bool guard = false;
  bool guard_selftest = false;
  int n_sm = 148;
  unsigned char poison = 0xff;
  std::map<void*, std::pair<size_t, const char*>> guards;  // body -> (bytes, name)
};

#define CK(call)                                                        \
  do {                                                                  \
    cudaError_t e_ = (call);                                            \
    if (e_ != cudaSuccess) {                                            \
      ctx->err = std::string(#call) + ": " + cudaGetErrorString(e_);    \
      return SYM_ECUDA;                                                 \
    }                                                                   \
  } while (0)

// Device memory is stream-ordered (the device's default pool, release
// threshold at max): no allocation or free synchronises the device, so
// several engines (threads, streams) run their kernels concurrently.
//
// Guard mode stands in for compute-sanitizer's memcheck and initcheck (the
// pool's GPUs cannot run it): a write outside any buffer lands in a redzone
// and fails the run; a read of memory the engine never wrote sees the poison
// byte, so two runs with different poison bytes that both equal the oracle
// read nothing uninitialised that matters.
constexpr size_t kRedzone = 4096;
constexpr unsigned char kRedByte = 0xa5;

cudaError_t dmalloc(Ctx* ctx, void** p, size_t bytes, cudaStream_t st, const char* name) {
  if (!ctx->guard) return cudaMallocAsync(p, bytes, st);
  char* base = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&base, bytes + 2 * kRedzone, st);
  if (e != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(base, kRedByte, kRedzone, st)) != cudaSuccess ||
      (e = cudaMemsetAsync(base + kRedzone, ctx->poison, bytes, st)) != cudaSuccess ||
      (e = cudaMemsetAsync(base + kRedzone + bytes, kRedByte, kRedzone, st)) != cudaSuccess)
    return e;
  *p = base + kRedzone;
  ctx->guards[*p] = {bytes, name};
  return cudaSuccess;
}

void dfree(Ctx* ctx, void* p, cudaStream_t st) {
  if (!p) return;
  if (!ctx->guard) {
    cudaFreeAsync(p, st);
    return;
  }
  ctx->guards.erase(p);
  cudaFreeAsync(static_cast<char*>(p) - kRedzone, st);
}

// Synchronises and reads every redzone back: SYM_EGUARD naming the first
// buffer written outside its bounds.
int guard_check(Ctx* ctx) {
  if (!ctx->guard) return SYM_OK;
  CK(cudaStreamSynchronize(ctx->stream));
  if (ctx->guard_selftest && !ctx->guards.empty()) {  // test hook: one byte past a buffer
    auto it = ctx->guards.begin();
    CK(cudaMemset(static_cast<char*>(it->first) + it->second.first, 0, 1));
  }
  std::vector<unsigned char> zone(kRedzone);
  for (auto& g : ctx->guards) {
    char* body = static_cast<char*>(g.first);
    for (int side = 0; side < 2; side++) {
      CK(cudaMemcpy(zone.data(), side ? body + g.second.first : body - kRedzone, kRedzone,
                    cudaMemcpyDeviceToHost));
      for (size_t i = 0; i < kRedzone; i++)
        if (zone[i] != kRedByte) {
          const size_t off = side ? i + 1 : kRedzone - i;
          ctx->err = std::string("guard: byte ") + std::to_string(off) +
                     (side ? " past the end of " : " before the start of ") +
                     g.second.second + " (" + std::to_string(g.second.first) + " bytes)";
          return SYM_EGUARD;
        }
    }
  }
  return SYM_OK;
}

template <class T>
int grow_named(Ctx* ctx, T*& p, int64_t count, const char* name) {
  dfree(ctx, p, ctx->stream);
  p = nullptr;
  CK(dmalloc(ctx, (void**)&p, sizeof(T) * (size_t)(count > 0 ? count : 1), ctx->stream, name));
  return SYM_OK;
}
#define grow(ctx, p, count) grow_named(ctx, p, count, #p)

// --------------------------------------------------------------- K1 -------

// ---- device-wide exclusive scan of an int32 array (reduce, scan the block
// sums, rescan with offsets).  Histograms are stored bin-major (hist[b][w]),
// so this one scan yields every stable scatter base: base(w, b) =
// sum over bins < b + sum over chunks < w of bin b.
constexpr int kScanItems = 4096;  // elements per block (1024 threads x 4)

__device__ __forceinline__ int32_t block_exclusive_scan(int32_t v, int32_t* total) {
  __shared__ int32_t wsum[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int32_t w = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    wsum[lane] = w;  // inclusive warp prefix
  }
  __syncthreads();
  const int32_t before = wid > 0 ? wsum[wid - 1] : 0;
  *total = wsum[(blockDim.x >> 5) - 1];
  __syncthreads();
  return before + x - v;
}

__global__ void __launch_bounds__(1024)
k_scan_up(const int32_t* __restrict__ a, int64_t len, int32_t* __restrict__ part) {
  const int64_t base = (int64_t)blockIdx.x * kScanItems + threadIdx.x * 4;
  int32_t v = 0;
#pragma unroll
  for (int k = 0; k < 4; k++)
    if (base + k < len) v += a[base + k];
  int32_t tot;
  block_exclusive_scan(v, &tot);
  if (threadIdx.x == 0) part[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(1024)
k_scan_mid(int32_t* __restrict__ part, int64_t nparts) {
  __shared__ int32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t b0 = 0; b0 < nparts; b0 += 1024) {
    const int64_t i = b0 + threadIdx.x;
    const int32_t v = i < nparts ? part[i] : 0;
    int32_t tot;
    const int32_t ex = block_exclusive_scan(v, &tot);
    const int32_t c = carry;
    if (i < nparts) part[i] = c + ex;
    __syncthreads();
    if (threadIdx.x == 0) carry = c + tot;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(1024)
k_scan_down(int32_t* __restrict__ a, int64_t len, const int32_t* __restrict__ part) {
  const int64_t base = (int64_t)blockIdx.x * kScanItems + threadIdx.x * 4;
  int32_t loc[4];
  int32_t v = 0;
#pragma unroll
  for (int k = 0; k < 4; k++) {
    loc[k] = base + k < len ? a[base + k] : 0;
    v += loc[k];
  }
  int32_t tot;
  int32_t run = block_exclusive_scan(v, &tot) + part[blockIdx.x];
#pragma unroll
  for (int k = 0; k < 4; k++) {
    if (base + k < len) a[base + k] = run;
    run += loc[k];
  }
}

// ---- K1: stable partition of the stream into the (shard, model) layout ---
// One building block, a stable partition of a time-ordered stream into few
// bins by reduce-then-scan over tiles of kTileI arrivals:
//   k_part_count  one block per tile counts its bins (shared atomics) and
//                 checks the model ids -> hist[bin][tile]
//   flat_scan     one exclusive scan of the bin-major histogram: every
//                 (bin, tile)'s first output position
//   k_part        one block per tile: stable ranks within the tile
//                 (per-warp bin counts + __match_any_sync), the tile staged in
//                 shared memory in bin order, bin runs written out
// One sub-cluster (P = 1): one partition by model id.  Several (P > 1): by
// sub-cluster first (P bins: the sub-cluster streams, whose ticks the chain
// reads for A'), then each sub-cluster stream by model slot -- two
// partitions with few bins each run far faster than one over M + P bins,
// whose per-tile bin bookkeeping and shared memory (1016 bins for C4 on one
// B200) starve the SMs.
//   mode 0 (P = 1):  bin = model          out: s_tick, s_i = i
//   mode 1 (level 1): bin = shard(model)  out: sh_tick, sh_i = i, sh_slot
//   mode 2 (level 2): bin = sh_slot       out: s_tick, s_g = j, s_i = sh_i[j]
// (the inverse maps are optional outputs: the per-request results come from
// k_bid's by-request record index, so the engine passes none)
constexpr int kTileWarps = 8;
constexpr int kTilePerLane = 8;
constexpr int kTileI = kTileWarps * 32 * kTilePerLane;  // 2048 arrivals per tile

// Geometry of tile t.  Modes 0 and 1: tiles of the whole stream, global
// bins, hist[bin][tile].  Mode 2 (segmented): the input is the sub-cluster
// streams back to back, and tiles never straddle two of them: tile t of
// sub-cluster s partitions its arrivals by the sub-cluster's own model slots
// (local bins 0..B_s), and the histogram is stored sub-cluster by
// sub-cluster, [local bin][tile] within each, so one flat scan still yields
// global output positions.  seg: tile_base[P+1] | hist_base[P+1] |
// shard_off[P+1] | slot_base[P+1].
struct TileGeom {
  int64_t lo, hi, hbase, hstride, col;
  int32_t B, bin0;
};

template <int kMode>
__device__ __forceinline__ bool tile_geom(int64_t t, int64_t n, int32_t B, int64_t W,
                                          const int64_t* __restrict__ seg, int32_t P,
                                          TileGeom& g) {
  if (kMode != 2) {
    g.lo = t * kTileI;
    g.hi = g.lo + kTileI < n ? g.lo + kTileI : n;
    g.B = B;
    g.bin0 = 0;
    g.hbase = 0;
    g.hstride = W;
    g.col = t;
    return true;
  }
  const int64_t* tile_base = seg;
  const int64_t* hist_base = seg + (P + 1);
  const int64_t* shard_off = seg + 2 * (P + 1);
  const int64_t* slot_base = seg + 3 * (P + 1);
  if (t >= tile_base[P]) return false;
  // the tile's sub-cluster: every lane tests one boundary (one load latency,
  // not a chain of P); called by whole warps
  int s = 0;
  if (P <= 32) {
    const int lane = threadIdx.x & 31;
    s = __popc(__ballot_sync(0xffffffffu, lane < P && tile_base[lane + 1] <= t));
  } else {
    int lo = 0, hi = P;  // last s with tile_base[s] <= t
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (tile_base[mid] <= t) lo = mid; else hi = mid;
    }
    s = lo;
  }
  const int64_t lt = t - tile_base[s];
  g.lo = shard_off[s] + lt * kTileI;
  g.hi = g.lo + kTileI < shard_off[s + 1] ? g.lo + kTileI : shard_off[s + 1];
  g.B = (int32_t)(slot_base[s + 1] - slot_base[s]);
  g.bin0 = (int32_t)slot_base[s];
  g.hbase = hist_base[s];
  g.hstride = tile_base[s + 1] - tile_base[s];
  g.col = lt;
  return true;
}

// mode 2's geometry from the level-1 sub-cluster offsets (one thread)
__global__ void k_part_seg(const int32_t* __restrict__ shard_off,
                           const int32_t* __restrict__ slot_base, int32_t P,
                           int64_t* __restrict__ seg) {
  if (threadIdx.x != 0) return;
  int64_t tb = 0, hb = 0;
  for (int s = 0; s <= P; s++) {
    seg[s] = tb;
    seg[(P + 1) + s] = hb;
    seg[2 * (P + 1) + s] = shard_off[s];
    seg[3 * (P + 1) + s] = slot_base[s];
    if (s < P) {
      const int64_t tiles = (shard_off[s + 1] - shard_off[s] + kTileI - 1) / kTileI;
      tb += tiles;
      hb += tiles * (slot_base[s + 1] - slot_base[s]);
    }
  }
}

template <int kMode>
__global__ void __launch_bounds__(256)
k_part_count(const int32_t* __restrict__ key, int64_t n, int32_t M,
             const int32_t* __restrict__ shard_of_model, int32_t B,
             int32_t* __restrict__ hist, int64_t W, const int64_t* __restrict__ seg,
             int32_t P, int32_t* __restrict__ err) {
  extern __shared__ int32_t hcnt[];
  TileGeom g;
  if (!tile_geom<kMode>(blockIdx.x, n, B, W, seg, P, g)) return;
  for (int b = threadIdx.x; b < g.B; b += blockDim.x) hcnt[b] = 0;
  __syncthreads();
  // launched with 256 threads: every element's key load issued before any
  // counting (kTileI / 256 per thread)
  constexpr int kPer = kTileI / 256;
  int32_t mk[kPer];
#pragma unroll
  for (int k = 0; k < kPer; k++) {
    const int64_t i = g.lo + threadIdx.x + k * 256;
    mk[k] = i < g.hi ? key[i] : 0;
  }
#pragma unroll
  for (int k = 0; k < kPer; k++) {
    const int64_t i = g.lo + threadIdx.x + k * 256;
    const int32_t m = mk[k];
    if (i >= g.hi) break;
    if (kMode != 2 && (m < 0 || m >= M)) {
      atomicMin(err, (int32_t)(i < INT32_MAX ? i : INT32_MAX));
      mk[k] = -1;
      continue;
    }
    mk[k] = kMode == 1 ? shard_of_model[m] : m - g.bin0;
  }
#pragma unroll
  for (int k = 0; k < kPer; k++) {
    const int64_t i = g.lo + threadIdx.x + k * 256;
    if (i >= g.hi) break;
    if (mk[k] >= 0) atomicAdd(&hcnt[mk[k]], 1);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < g.B; b += blockDim.x)
    hist[g.hbase + (int64_t)b * g.hstride + g.col] = hcnt[b];
}

// ModelParam.off/cnt per slot (mp == null: shard_off instead) from the
// first tile column of the scanned histogram
template <int kMode>
__global__ void k_part_binoff(const int32_t* __restrict__ hist, int64_t W, int32_t B, int64_t n,
                              const int64_t* __restrict__ seg, int32_t P,
                              ModelParam* __restrict__ mp, int32_t* __restrict__ shard_off) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  int32_t o, e;
  if (kMode != 2) {
    o = W > 0 ? hist[(int64_t)b * W] : 0;
    e = b + 1 < B ? (W > 0 ? hist[(int64_t)(b + 1) * W] : 0) : (int32_t)n;
  } else {
    const int64_t* tile_base = seg;
    const int64_t* hist_base = seg + (P + 1);
    const int64_t* soff = seg + 2 * (P + 1);
    const int64_t* slot_base = seg + 3 * (P + 1);
    int s = 0;
    while (slot_base[s + 1] <= b) s++;
    const int64_t lb = b - slot_base[s], tiles = tile_base[s + 1] - tile_base[s];
    if (tiles == 0) {
      o = e = (int32_t)soff[s];
    } else {
      o = hist[hist_base[s] + lb * tiles];
      e = lb + 1 < slot_base[s + 1] - slot_base[s] ? hist[hist_base[s] + (lb + 1) * tiles]
                                                     : (int32_t)soff[s + 1];
    }
  }
  if (mp) {
    mp[b].off = o;
    mp[b].cnt = e - o;
  } else {
    shard_off[b] = o;
    if (b == B - 1) shard_off[B] = (int32_t)n;
  }
}

__host__ __device__ inline size_t part_smem(int B) {
  return (size_t)kTileI * (sizeof(int64_t) + 2 * sizeof(int32_t) + sizeof(int16_t)) +
         sizeof(int32_t) * ((size_t)kTileWarps * B + 2 * (size_t)B + 32);
}

template <int kMode>
__global__ void __launch_bounds__(32 * kTileWarps, 4)
k_part(const int64_t* __restrict__ tick_in, const int32_t* __restrict__ key,
       const int32_t* __restrict__ aux_in, int64_t n, int32_t M,
       const int32_t* __restrict__ shard_of_model, const int32_t* __restrict__ slot_of_model,
       int32_t Bmax, const int32_t* __restrict__ hist, int64_t W,
       const int64_t* __restrict__ seg, int32_t P,
       int64_t* __restrict__ out_tick, int32_t* __restrict__ out_idx,
       int32_t* __restrict__ out_aux, int32_t* __restrict__ inv_out,
       int32_t* __restrict__ err) {
  constexpr bool kAux = kMode != 0;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  TileGeom geo;
  if (!tile_geom<kMode>(blockIdx.x, n, Bmax, W, seg, P, geo)) return;
  const int32_t B = geo.B;
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int64_t* st_t = reinterpret_cast<int64_t*>(smem_raw);
  int32_t* st_i = reinterpret_cast<int32_t*>(st_t + kTileI);
  int32_t* st_a = st_i + kTileI;               // kAux only
  int32_t* wcnt = st_a + kTileI;               // [warp][bin] counts -> offsets
  int32_t* gbase = wcnt + kTileWarps * B;      // global position of the tile's bin run
  int32_t* lstart = gbase + B;                 // local start of a bin's run
  int32_t* scratch = lstart + B;               // [32] block scan
  int16_t* st_b = reinterpret_cast<int16_t*>(scratch + 32);
  int32_t* mine = wcnt + wib * B;
  for (int b = lane; b < B; b += 32) mine[b] = 0;
  const int64_t lo = geo.lo, hi = geo.hi;
  const int64_t wlo = lo + (int64_t)wib * 32 * kTilePerLane;
  __syncwarp();
  // pass 1: load this lane's elements once (every row's loads issued before
  // any is used), count the warp's bins
  int64_t tk[kTilePerLane];
  int32_t bn[kTilePerLane], ax[kTilePerLane];
#pragma unroll
  for (int r = 0; r < kTilePerLane; r++) {
    const int64_t i = wlo + r * 32 + lane;
    tk[r] = 0;
    bn[r] = -1;
    ax[r] = 0;
    if (i < hi) {
      tk[r] = tick_in[i];
      bn[r] = key[i];
      if (kMode == 2) ax[r] = aux_in[i];
    }
  }
  const int64_t before_warp = kMode != 2 && lane == 0 && wlo > 0 && wlo < hi ? tick_in[wlo - 1]
                                                                            : INT64_MIN;
  // the tile's bin bases (read after the counting barrier), loaded while the
  // element loads are in flight
  for (int b = threadIdx.x; b < B; b += blockDim.x)
    gbase[b] = hist[geo.hbase + (int64_t)b * geo.hstride + geo.col];
#pragma unroll
  for (int r = 0; r < kTilePerLane; r++) {
    const int64_t i = wlo + r * 32 + lane;
    const int32_t m = bn[r];
    bn[r] = -1 - lane;
    if (i < hi && (kMode == 2 || (m >= 0 && m < M))) {  // unknown ids: k_part_count
      bn[r] = kMode == 1 ? shard_of_model[m] : m - geo.bin0;
      if (kMode == 1) ax[r] = slot_of_model[m];
    }
  }
  if (kMode != 2) {  // arrivals must be time-ordered: the previous element by shuffle
#pragma unroll
    for (int r = 0; r < kTilePerLane; r++) {
      const int64_t i = wlo + r * 32 + lane;
      int64_t prev = __shfl_up_sync(0xffffffffu, tk[r], 1);
      const int64_t last_row = __shfl_sync(0xffffffffu, r > 0 ? tk[r > 0 ? r - 1 : 0] : 0, 31);
      if (lane == 0) prev = r > 0 ? last_row : before_warp;
      if (i < hi && i > 0 && tk[r] < prev)
        atomicMin(err + 1, (int32_t)(i < INT32_MAX ? i : INT32_MAX));
    }
  }
#pragma unroll
  for (int r = 0; r < kTilePerLane; r++)
    if (bn[r] >= 0) atomicAdd_block(&mine[bn[r]], 1);
  __syncthreads();
  // per bin: warp offsets and the tile's count; local starts by a block scan
  {
    const int per = (B + blockDim.x - 1) / blockDim.x;
    int32_t run = 0;
    for (int k = 0; k < per; k++) {
      const int b = threadIdx.x * per + k;
      if (b >= B) break;
      int32_t acc = 0;
      for (int q = 0; q < kTileWarps; q++) {
        const int32_t c = wcnt[q * B + b];
        wcnt[q * B + b] = acc;
        acc += c;
      }
      lstart[b] = acc;  // the bin's count, for now
      run += acc;
    }
    int32_t x = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) scratch[wib] = x;
    __syncthreads();
    if (wib == 0) {
      int32_t v = lane < kTileWarps ? scratch[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
      }
      if (lane < kTileWarps) scratch[lane] = v;
    }
    __syncthreads();
    int32_t before = (wib ? scratch[wib - 1] : 0) + x - run;
    for (int k = 0; k < per; k++) {
      const int b = threadIdx.x * per + k;
      if (b >= B) break;
      const int32_t c = lstart[b];
      lstart[b] = before;
      before += c;
    }
  }
  __syncthreads();
  // pass 2: stable rank, stage in bin order, inverse map
  const unsigned ltm = (1u << lane) - 1u;
#pragma unroll
  for (int r = 0; r < kTilePerLane; r++) {
    const int64_t i = wlo + r * 32 + lane;
    const bool act = i < hi && bn[r] >= 0;
    const unsigned ps = __match_any_sync(0xffffffffu, bn[r]);
    int32_t e = 0;
    if (act) e = mine[bn[r]] + __popc(ps & ltm);
    __syncwarp();
    if (act) {
      if ((ps >> lane) == 1u) mine[bn[r]] += __popc(ps);  // highest peer advances
      const int32_t le = lstart[bn[r]] + e;
      st_t[le] = tk[r];
      st_i[le] = (int32_t)i;
      st_b[le] = (int16_t)bn[r];
      if (kAux) st_a[le] = ax[r];
      if (inv_out) inv_out[i] = gbase[bn[r]] + e;  // coalesced in i
    }
    __syncwarp();
  }
  __syncthreads();
  const int32_t len = scratch[kTileWarps - 1];  // elements staged (valid ids)
  constexpr int kOutIlp = 4;  // independent shared-memory chains per thread
  for (int32_t e0 = threadIdx.x; e0 < len; e0 += kOutIlp * blockDim.x) {  // bin runs
    int32_t pos[kOutIlp];
#pragma unroll
    for (int k = 0; k < kOutIlp; k++) {
      const int32_t e = e0 + k * blockDim.x;
      const int32_t b = e < len ? st_b[e] : 0;
      pos[k] = gbase[b] + (e - lstart[b]);
    }
#pragma unroll
    for (int k = 0; k < kOutIlp; k++) {
      const int32_t e = e0 + k * blockDim.x;
      if (e < len) {
        out_tick[pos[k]] = st_t[e];
        out_idx[pos[k]] = st_i[e];
        if (kAux) out_aux[pos[k]] = st_a[e];
      }
    }
  }
}

// --------------------------------------------------------------- K2 -------

// K2 (window / candidate per fresh start, fast path): the batch-chain
// pointer of every sorted position q -- where the batch a fresh start at q
// forms closes (fastpath.cuh, lean_chain_next*) -- and its closing arrival
// for k_chain_recs.  For an affine l(b) (deferred, prefix) the closing index
// is the first j > q with u_j >= u_q + (slo - a - b0 - d_ctrl) on the
// non-decreasing u_j = tick_j + (a + d_data) j (lean_chain_next_affine): a
// lower bound in a sorted sequence, found per lane by a fixed binary search
// over shared memory (k_nxt_tma).  Model boundaries come from the per-slot
// offsets (no per-position model array).  Positions the lean test cannot
// certify are listed for the general fresh scan (k_nxt_general); other
// profiles and policies take the scalar lean forms per position
// (also in k_nxt_tma).

// k_nxt_tma: a warp owns kNxtRounds x 32 consecutive positions (lane =
// position), their u plus a look-ahead staged in shared memory.  For the
// affine deferred/prefix form the closing index of a fresh start p is the
// first j in (p, jend] with u_j >= T_p, so a lane finds it by a fixed 5-step
// binary search over the 32 staged u after p -- every lane runs the same
// instructions, no data-dependent loop -- and stores nxt/close_k coalesced.
// Batches longer than 32 arrivals, the last arrivals of a model and the
// max-batch tail take the scalar lean_chain_next_affine.
#ifndef SYM_NXT_ROUNDS
#define SYM_NXT_ROUNDS 16
#endif
#ifndef SYM_NXT_BPS
#define SYM_NXT_BPS 3
#endif
#ifndef SYM_NXT_WARPS
#define SYM_NXT_WARPS 8
#endif
constexpr int kNxtRounds = SYM_NXT_ROUNDS;
constexpr int kNxtTile = 32 * kNxtRounds;  // positions per warp
constexpr int kNxtWin = 32;                // binary-search window after q
constexpr int kNxtStage = kNxtTile + 2 * kNxtWin;

__device__ __forceinline__ bool lean_affine(const Shard& S, const ModelParam& mp) {
  return mp.affine && S.kind == K_DEFERRED && S.gather == G_PREFIX;
}

__device__ __forceinline__ int shard_of_slot_linear(const int32_t* __restrict__ slot_base,
                                                    int32_t k) {
  int sh = 0;
  while (slot_base[sh + 1] <= k) sh++;
  return sh;
}

// ---- TMA-staged K2 (the launch used).  A persistent warp walks tiles
// t = w, w + W, ...; the tile's ticks [t0, t0 + kNxtStage) arrive in shared
// memory by one bulk copy (cp.async.bulk, completion on an mbarrier) issued
// one tile ahead into the warp's other buffer, so the DRAM latency of tile
// t+W hides behind the search of tile t.  The ticks become u in place
// (u_j = tick_j + (a + d_data)(j - off)), one model segment at a time.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "NXT_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra NXT_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Last slot with off <= p (empty slots skipped): a 32-ary search, one load
// per lane per level (two levels up to 1024 slots).
__device__ __forceinline__ int32_t warp_slot_of_position(const ModelParam* __restrict__ mp_all,
                                                         int32_t M, int32_t p, int lane) {
  int32_t lo = 0, hi = M;  // answer in [lo, hi)
  while (hi - lo > 1) {
    const int32_t step = (hi - lo + 31) / 32;
    const int32_t idx = lo + lane * step;
    const bool le = idx < hi && (idx == lo || mp_all[idx].off <= p);
    const unsigned b = __ballot_sync(0xffffffffu, le);
    const int32_t L = 31 - __clz(b);
    lo = lo + L * step;
    hi = min(lo + step, hi);
  }
  while (lo + 1 < M && mp_all[lo].off + mp_all[lo].cnt <= p) lo++;
  return lo;
}

// Last index with a[idx] <= x over a non-decreasing int32 array (a[0] <= x):
// a 32-ary search, one load per lane per level.
__device__ __forceinline__ int32_t warp_last_le(const int32_t* __restrict__ a, int32_t M,
                                                int64_t x, int lane) {
  int32_t lo = 0, hi = M;
  while (hi - lo > 1) {
    const int32_t step = (hi - lo + 31) / 32;
    const int32_t idx = lo + lane * step;
    const bool le = idx < hi && (idx == lo || a[idx] <= x);
    const unsigned b = __ballot_sync(0xffffffffu, le);
    lo = lo + (31 - __clz(b)) * step;
    hi = min(lo + step, hi);
  }
  return lo;
}

constexpr int kNxtTmaWarps = SYM_NXT_WARPS;
constexpr int kNxtTmaBlocksPerSm = SYM_NXT_BPS;
constexpr int kNxtTmaSmemBuf = kNxtTmaWarps * 2 * kNxtStage * 8;
constexpr int kNxtTmaSmem = kNxtTmaSmemBuf + kNxtTmaWarps * 2 * 8;  // + mbarriers

__global__ void __launch_bounds__(32 * kNxtTmaWarps, kNxtTmaBlocksPerSm)
k_nxt_tma(const int64_t* __restrict__ tick, const Shard* __restrict__ shards,
          const int32_t* __restrict__ slot_base, const ModelParam* __restrict__ mp_all,
          int32_t P, int32_t M, int32_t n, int32_t* __restrict__ nxt,
          int32_t* __restrict__ close_k, int32_t* __restrict__ unsure,
          int32_t* __restrict__ unsure_n) {
  extern __shared__ __align__(128) unsigned char nxt_smem[];
  auto sbuf = reinterpret_cast<int64_t(*)[2][kNxtStage]>(nxt_smem);
  auto sbar = reinterpret_cast<uint64_t(*)[2]>(nxt_smem + kNxtTmaSmemBuf);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int32_t ntiles = (n + kNxtTile - 1) / kNxtTile;
  const int32_t W = gridDim.x * kNxtTmaWarps;
  int32_t t = blockIdx.x * kNxtTmaWarps + w;
  if (lane == 0) {
    mbar_init(&sbar[w][0], 1);
    mbar_init(&sbar[w][1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  auto issue = [&](int32_t tt, int b) {
    const int32_t t0 = tt * kNxtTile;
    const int32_t cnt = n - t0 < kNxtStage ? n - t0 : kNxtStage;
    // whole 16-byte units: an odd tail reads one element past n (capacity
    // n + 1024), never used
    bulk_load(sbuf[w][b], tick + t0, (uint32_t)((cnt + 1) & ~1) * 8u, &sbar[w][b]);
  };
  if (lane == 0 && t < ntiles) issue(t, 0);
  uint32_t phase = 0;  // bit b: parity of buffer b's next completion
  for (int b = 0; t < ntiles; t += W, b ^= 1) {
    if (lane == 0 && t + W < ntiles) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(t + W, b ^ 1);
    }
    const int32_t t0 = t * kNxtTile;
    const int32_t send = n - t0 < kNxtStage ? n : t0 + kNxtStage;
    int32_t k = warp_slot_of_position(mp_all, M, t0, lane);
    const int32_t pend = n - t0 < kNxtTile ? n : t0 + kNxtTile;
    int64_t* __restrict__ u = sbuf[w][b];
    mbar_wait(&sbar[w][b], (phase >> b) & 1);
    phase ^= 1u << b;
    // the tile's positions, one model segment at a time (warp-uniform loop;
    // usually one segment)
    for (int32_t a = t0; a < pend;) {
      while (mp_all[k].off + mp_all[k].cnt <= a) k++;
      const ModelParam& mk = mp_all[k];
      const int sh = shard_of_slot_linear(slot_base, k);
      const Shard& S = shards[sh];
      const int32_t off = mk.off, cnt = mk.cnt;
      const int32_t seg_end = off + cnt < pend ? off + cnt : pend;
      if (lean_affine(S, mk)) {
        const int64_t c1 = mk.aff_a + S.d_data;
        const int64_t D1 = mk.slo - mk.aff_a - mk.aff_b - S.d_ctrl;
        const int64_t D2 = mk.slo - S.d_ctrl - mk.aff_b - c1;
        // jend = min(off + cnt - 1, p + mb - 1) >= p + 32  <=>  p <= pfull
        const int32_t pfull = mk.max_batch - 1 >= kNxtWin ? off + cnt - 1 - kNxtWin : INT32_MIN;
        const int32_t ub = off + cnt < send ? off + cnt : send;  // this model's staged part
        for (int32_t e = a - t0 + lane; e < ub - t0; e += 32) u[e] += c1 * (t0 + e - off);
        __syncwarp();
        // two positions per lane per iteration (p and p + 32): their searches
        // interleave, so one's shared-memory latency hides behind the other's
        auto finish = [&](int32_t pp, bool fast, int32_t x, int64_t uq, int64_t ukk) {
          const int32_t v = fast ? (ukk <= uq + D2 ? pp + x + 1 : NX_UNSURE)
                                 : lean_chain_next_affine(S, mk, pp - off);
          nxt[pp] = v;
          close_k[pp] = v >= 0 ? v - 1 - off : (v == NX_LAST ? cnt - 1 : -1);
          if (v == NX_UNSURE) unsure[atomicAdd(unsure_n, 1)] = pp;
        };
#pragma unroll 1
        for (int32_t p = a + lane; p < seg_end; p += 64) {
          const int32_t p2 = p + 32;
          const bool has2 = p2 < seg_end;
          const int e = p - t0, e2 = e + 32;  // e2 + 32 < kNxtStage: always staged
          const int64_t uq = u[e], uq2 = u[e2];
          const int64_t T = uq + D1, T2 = uq2 + D1;
          // the batch closes within 32 arrivals: first j in (p, p+32] with u_j >= T
          const bool f1 = p <= pfull && u[e + kNxtWin] >= T;
          const bool f2 = p2 <= pfull && u[e2 + kNxtWin] >= T2;
          int32_t x = 0, x2 = 0;
#pragma unroll
          for (int st = kNxtWin / 2; st >= 1; st >>= 1) {
            if (u[e + x + st] < T) x += st;
            if (u[e2 + x2 + st] < T2) x2 += st;
          }
          finish(p, f1, x, uq, u[e + x]);
          if (has2) finish(p2, f2, x2, uq2, u[e2 + x2]);
        }
      } else {  // other profiles / policies: the scalar lean forms
        const int32_t m = k - slot_base[sh];
        const bool r32 = rel32_ok(S, mk);
        for (int32_t p = a + lane; p < seg_end; p += 32) {
          const int32_t q = p - off;
          const int32_t v = r32 ? lean_chain_next32(S, m, q) : lean_chain_next(S, m, q);
          nxt[p] = v;
          close_k[p] = v >= 0 ? v - 1 - off : (v == NX_LAST ? cnt - 1 : -1);
          if (v == NX_UNSURE) unsure[atomicAdd(unsure_n, 1)] = p;
        }
      }
      a = seg_end;
    }
    __syncwarp();  // every lane is done with buffer b before it is refilled
  }
}

// Positions the lean loop could not certify: the general fresh_scan.
__device__ __forceinline__ void nxt_general_one(const Shard* __restrict__ shards,
                                                const int32_t* __restrict__ slot_base,
                                                const ModelParam* __restrict__ mp_all, int32_t P,
                                                int64_t p, int32_t* __restrict__ nxt,
                                                int32_t* __restrict__ close_k) {
  int lo = 0, hi = slot_base[P];
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (mp_all[mid].off <= p) lo = mid; else hi = mid;
  }
  while (mp_all[lo].cnt == 0 || mp_all[lo].off + mp_all[lo].cnt <= p) lo++;
  int s = 0;
  while (slot_base[s + 1] <= lo) s++;
  const int32_t q = (int32_t)(p - mp_all[lo].off);
  nxt[p] = chain_next(fresh_scan(shards[s], lo - slot_base[s], q, kFreshMaxSteps), mp_all[lo]);
  close_k[p] = -1;  // not certified by the lean sweep: k_chain_recs rescans
}

__global__ void __launch_bounds__(256)
k_nxt_general(const Shard* __restrict__ shards, const int32_t* __restrict__ slot_base,
              const ModelParam* __restrict__ mp_all, int32_t P,
              const int32_t* __restrict__ unsure, const int32_t* __restrict__ unsure_n,
              int32_t* __restrict__ nxt, int32_t* __restrict__ close_k) {
  const int32_t cnt = *unsure_n;  // listed by k_nxt_tma; usually none
  for (int32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < cnt; u += gridDim.x * blockDim.x)
    nxt_general_one(shards, slot_base, mp_all, P, unsure[u], nxt, close_k);
}


__global__ void __launch_bounds__(256)
k_fresh(const Shard* __restrict__ shards, const int32_t* __restrict__ slot_base,
        const ModelParam* __restrict__ mp_all, int32_t P, int64_t n,
        FreshRec* __restrict__ out, int32_t* __restrict__ nxt) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  // slot of p: last slot with off <= p and cnt > 0
  int lo = 0, hi = slot_base[P];
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (mp_all[mid].off <= p) lo = mid; else hi = mid;
  }
  while (mp_all[lo].cnt == 0 || mp_all[lo].off + mp_all[lo].cnt <= p) lo++;
  int s = 0;
  while (slot_base[s + 1] <= lo) s++;
  const Shard& S = shards[s];
  const int32_t m = lo - slot_base[s];
  const FreshRec r = fresh_scan(S, m, (int32_t)(p - mp_all[lo].off), kFreshMaxSteps);
  out[p] = r;
  if (nxt) nxt[p] = chain_next(r, mp_all[lo]);
}

// --------------------------------------------------------------- K4 -------

// Shared-memory plan of one sub-cluster's chain state.  Arrays are placed in
// smem in order of how often the chain touches them; whatever does not fit
// stays in its global scratch (the chain is agnostic: it only sees pointers).
struct SmemPlan {
  static SYM_HD size_t al(size_t x) { return (x + 15) & ~size_t(15); }
  static SYM_HD size_t need(const Shard& S) {
    return al(sizeof(int32_t) * 2 * S.Gp) + al(sizeof(int64_t) * 2 * S.Gp) +
           al(sizeof(int64_t) * S.G) + al(sizeof(int32_t) * 2 * S.Mp) +
           al(sizeof(int64_t) * 2 * S.Mp) + al(sizeof(ModelState) * S.M) +
           al(sizeof(ModelParam) * S.M) + 2 * al(sizeof(int32_t) * 2 * S.Mp) +
           2 * al(sizeof(int64_t) * 2 * S.Mp) + al(sizeof(int32_t) * S.M) +
           al(sizeof(int64_t) * S.M) + al(sizeof(int64_t) * S.M * S.lat_stride);
  }
};

// mode: 0 = a whole run (init, run to the end; only the model states are
// written back, for the drop counts); 1 = the first step of a stepped run
// (init, run to `until`, write back ALL state); 2 = a later step (load all
// state, resume, run to `until`, write it back).
constexpr int kChainWhole = 0, kChainFirstStep = 1, kChainResume = 2;

__global__ void __launch_bounds__(32)
k_chain(Shard* shards, const FreshRec* __restrict__ fresh,
        int32_t* __restrict__ dirty_all, const int32_t* __restrict__ slot_base,
        size_t smem_bytes, const int32_t* __restrict__ skip, int mode, int64_t until) {
  extern __shared__ __align__(16) unsigned char smem[];
  if (threadIdx.x != 0 || skip[blockIdx.x]) return;
  Shard S = shards[blockIdx.x];  // hot scalars of the sub-cluster in registers
  const Shard orig = S;  // global pointers, restored before the write-back
  const bool load = mode == kChainResume, keep = mode != kChainWhole;
  size_t used = 0;
  auto place = [&](auto*& ptr, size_t exact, bool copy_in) {
    const size_t bytes = SmemPlan::al(exact);
    if (used + bytes > smem_bytes) return false;
    using T = std::remove_pointer_t<std::remove_reference_t<decltype(ptr)>>;
    T* dst = reinterpret_cast<T*>(smem + used);
    if (copy_in) {  // element-wise: sources need not be 16-byte aligned
      const size_t cnt = exact / sizeof(T);
      for (size_t k = 0; k < cnt; k++) dst[k] = ptr[k];
    }
    ptr = dst;
    used += bytes;
    return true;
  };
  // state arrays placed on chip, with their sizes for the write-back
  const bool gt_s = place(S.gt, sizeof(int32_t) * 2 * S.Gp, load);
  const bool gf_s = place(S.gt_f, sizeof(int64_t) * 2 * S.Gp, load);
  const bool fa_s = place(S.free_at, sizeof(int64_t) * S.G, load);
  const bool pq_s = place(S.pq, sizeof(int32_t) * 2 * S.Mp, load);
  const bool pt_s = place(S.pq_t, sizeof(int64_t) * 2 * S.Mp, load);
  const bool ms_in_smem = place(S.ms, sizeof(ModelState) * S.M, load);
  const ModelParam* mp = S.mp;
  ModelParam* mp_s = const_cast<ModelParam*>(mp);
  if (place(mp_s, sizeof(ModelParam) * S.M, true)) S.mp = mp_s;
  const bool ml_s = place(S.mc_lat_tree, sizeof(int32_t) * 2 * S.Mp, load);
  const bool mb_s = place(S.mc_bs_tree, sizeof(int32_t) * 2 * S.Mp, load);
  const bool mlv_s = place(S.mlt_v, sizeof(int64_t) * 2 * S.Mp, load);
  const bool mbv_s = place(S.mbt_v, sizeof(int64_t) * 2 * S.Mp, load);
  const bool mz_s = place(S.mc_size, sizeof(int32_t) * S.M, load);
  const bool mt_s = place(S.mc_latest, sizeof(int64_t) * S.M, load);
  {  // latency rows last: small model sets keep every l(b) probe on chip
    const int64_t* lat_g = S.lat;
    int64_t* lat_s = const_cast<int64_t*>(lat_g);
    if (place(lat_s, sizeof(int64_t) * S.M * S.lat_stride, true)) S.lat = lat_s;
  }
  int32_t* dirty = dirty_all + slot_base[blockIdx.x] + blockIdx.x;
#ifdef SYM_CHAIN_PROF
  sym::g_chain_prof_on = 1;
#endif
  if (load)
    chain_resume(S);
  else
    chain_init(S, fresh);
  while (chain_step(S, dirty, fresh, until)) {
  }
#ifdef SYM_CHAIN_PROF
  sym::g_chain_prof_on = 0;
#endif
  auto back = [](auto* dst, const auto* src, size_t cnt) {
    for (size_t k = 0; k < cnt; k++) dst[k] = src[k];
  };
  if (ms_in_smem) back(orig.ms, S.ms, S.M);
  if (keep) {  // a stepped run carries every structure to the next step
    if (gt_s) back(orig.gt, S.gt, 2 * (size_t)S.Gp);
    if (gf_s) back(orig.gt_f, S.gt_f, 2 * (size_t)S.Gp);
    if (fa_s) back(orig.free_at, S.free_at, S.G);
    if (pq_s) back(orig.pq, S.pq, 2 * (size_t)S.Mp);
    if (pt_s) back(orig.pq_t, S.pq_t, 2 * (size_t)S.Mp);
    if (ml_s) back(orig.mc_lat_tree, S.mc_lat_tree, 2 * (size_t)S.Mp);
    if (mb_s) back(orig.mc_bs_tree, S.mc_bs_tree, 2 * (size_t)S.Mp);
    if (mlv_s) back(orig.mlt_v, S.mlt_v, 2 * (size_t)S.Mp);
    if (mbv_s) back(orig.mbt_v, S.mbt_v, 2 * (size_t)S.Mp);
    if (mz_s) back(orig.mc_size, S.mc_size, S.M);
    if (mt_s) back(orig.mc_latest, S.mc_latest, S.M);
  }
  S.ms = orig.ms;
  S.mp = orig.mp;
  S.lat = orig.lat;
  S.gt = orig.gt;
  S.gt_f = orig.gt_f;
  S.free_at = orig.free_at;
  S.pq = orig.pq;
  S.pq_t = orig.pq_t;
  S.mc_lat_tree = orig.mc_lat_tree;
  S.mc_bs_tree = orig.mc_bs_tree;
  S.mlt_v = orig.mlt_v;
  S.mbt_v = orig.mbt_v;
  S.mc_size = orig.mc_size;
  S.mc_latest = orig.mc_latest;
  shards[blockIdx.x] = S;
}

// --------------------------------------------------------------- K5 -------

__global__ void k_narrow(const int64_t* __restrict__ in, int64_t n, int32_t* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t v = in[i];
  out[i] = (v < 0 || v > INT32_MAX) ? -1 : (int32_t)v;  // out of range -> EPROTO
}


// every batch stamps its record index on its member positions
// Record index of every request, by stream index: bid[s_i[p]] = record for
// each member position p of each batch record.  The records are interleaved
// across sub-clusters (thread w: sub-cluster w mod P, its (w / P)-th record),
// and each sub-cluster's records are in dispatch order, so the requests the
// resident warps stamp at any moment lie in one short stretch of the stream
// and their scattered 4-byte writes complete whole sectors in L2.  A warp
// takes 32 records; each record's members are read (s_i, contiguous) and
// stamped by the whole warp.  k_out then reads bid[i] coalesced instead of
// the gather chain stream -> sub-cluster stream -> layout -> record.
__global__ void k_bid(const BatchRec* __restrict__ recs, const int64_t* __restrict__ rec_base,
                      const int64_t* __restrict__ rec_count, int32_t P, int64_t slots,
                      const int32_t* __restrict__ s_i, int32_t* __restrict__ bid) {
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  int32_t ri = -1, first = 0, size = 0;
  if (w < slots) {
    const int s = (int)(w % P);
    const int64_t k = w / P;
    if (k < rec_count[s]) {
      ri = (int32_t)(rec_base[s] + k);
      const BatchRec& r = recs[ri];
      first = r.first;
      size = r.size;
    }
  }
  // eight records at a time: their member loads are all issued before any
  // store (one latency per eight records); runs beyond 32 members afterwards
  for (int b0 = 0; b0 < 32; b0 += 8) {
    int32_t tgt[8], rbv[8];
#pragma unroll
    for (int q = 0; q < 8; q++) {
      const int32_t fb = __shfl_sync(0xffffffffu, first, b0 + q);
      const int32_t sb = __shfl_sync(0xffffffffu, size, b0 + q);
      rbv[q] = __shfl_sync(0xffffffffu, ri, b0 + q);
      tgt[q] = lane < sb ? s_i[fb + lane] : -1;
    }
#pragma unroll
    for (int q = 0; q < 8; q++)
      if (tgt[q] >= 0) bid[tgt[q]] = rbv[q];
  }
  if (__any_sync(0xffffffffu, size > 32))
    for (int b = 0; b < 32; b++) {
      const int32_t rb = __shfl_sync(0xffffffffu, ri, b);
      const int32_t fb = __shfl_sync(0xffffffffu, first, b);
      const int32_t sb = __shfl_sync(0xffffffffu, size, b);
      for (int32_t j = lane + 32; j < sb; j += 32) bid[s_i[fb + j]] = rb;
    }
}

// RunResult arrays (simulator.py:74-78, 159-173, 249-258) in stream order:
// one thread per request, reads scattered, writes coalesced.  A request no
// batch covers was dropped (every request resolves).
// Two requests per thread: the stream-order loads and the five output
// stores are 16-byte vector accesses (the kernel is bound by the LSU queue
// and by the gather chain inv -> bid -> record, whose loads for the two
// requests are issued together).  Outputs must be 16-byte aligned (torch
// and the pinned host pool allocate 256-byte aligned buffers); an odd n
// leaves the last request to a scalar tail.
struct OutRow {
  int64_t disp, start, fin, bat, outc;
};

__device__ __forceinline__ OutRow out_row(int32_t r, const BatchRec* __restrict__ recs,
                                          int64_t dl) {
  OutRow o;
  if (r < 0) {
    o.disp = o.start = o.fin = o.bat = -1;
    o.outc = 2;  // OUTCOME_DROPPED
    return o;
  }
  // emitted | start, finish | size: two 16-byte gathers instead of four
  const longlong2 w0 = __ldg(reinterpret_cast<const longlong2*>(recs + r));
  const longlong2 w1 = __ldg(reinterpret_cast<const longlong2*>(recs + r) + 1);
  o.disp = w0.x;
  o.start = w0.y;
  o.fin = w1.x;
  o.bat = (int32_t)(w1.y & 0xffffffff);  // size: the low word (little-endian)
  o.outc = w1.x <= dl ? 0 : 1;
  return o;
}

template <bool kVec>
__global__ void __launch_bounds__(256)
k_out(int64_t n, const int32_t* __restrict__ bid, const BatchRec* __restrict__ recs,
      const int64_t* __restrict__ ticks, const int32_t* __restrict__ model,
      const int64_t* __restrict__ slo_by_model,
      int64_t* __restrict__ disp, int64_t* __restrict__ start,
      int64_t* __restrict__ fin, int64_t* __restrict__ bat,
      int64_t* __restrict__ outc, int64_t* __restrict__ o_arr,
      int64_t* __restrict__ o_dl, int64_t* __restrict__ o_model) {
  const int64_t i = 2 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x);
  if (i >= n) return;
  if (!kVec || i + 1 >= n) {  // scalar: unaligned caller buffers, or the tail
    for (int64_t k = i; k < i + 2 && k < n; k++) {
      const int64_t tick = ticks[k];
      const int32_t mi = model[k];
      const int64_t dl = tick + slo_by_model[mi];
      if (o_arr) o_arr[k] = tick;
      if (o_dl) o_dl[k] = dl;
      if (o_model) o_model[k] = mi;
      const OutRow o = out_row(bid[k], recs, dl);
      disp[k] = o.disp;
      start[k] = o.start;
      fin[k] = o.fin;
      bat[k] = o.bat;
      outc[k] = o.outc;
    }
    return;
  }
  const longlong2 t2 = *reinterpret_cast<const longlong2*>(ticks + i);
  const int2 m2 = *reinterpret_cast<const int2*>(model + i);
  const int2 r2 = *reinterpret_cast<const int2*>(bid + i);  // records, by request
  const int32_t r0 = r2.x, r1 = r2.y;
  const int64_t dl0 = t2.x + slo_by_model[m2.x], dl1 = t2.y + slo_by_model[m2.y];
  const OutRow a = out_row(r0, recs, dl0), b = out_row(r1, recs, dl1);
  if (o_arr) *reinterpret_cast<longlong2*>(o_arr + i) = t2;
  if (o_dl) *reinterpret_cast<longlong2*>(o_dl + i) = make_longlong2(dl0, dl1);
  if (o_model) *reinterpret_cast<longlong2*>(o_model + i) = make_longlong2(m2.x, m2.y);
  *reinterpret_cast<longlong2*>(disp + i) = make_longlong2(a.disp, b.disp);
  *reinterpret_cast<longlong2*>(start + i) = make_longlong2(a.start, b.start);
  *reinterpret_cast<longlong2*>(fin + i) = make_longlong2(a.fin, b.fin);
  *reinterpret_cast<longlong2*>(bat + i) = make_longlong2(a.bat, b.bat);
  *reinterpret_cast<longlong2*>(outc + i) = make_longlong2(a.outc, b.outc);
}

__global__ void k_drop_out(int64_t n, const int32_t* __restrict__ s_i,
                           const int64_t* __restrict__ dt,
                           const int64_t* __restrict__ dks,
                           const int32_t* __restrict__ dka,
                           int64_t* __restrict__ o_t, int64_t* __restrict__ o_ks,
                           int32_t* __restrict__ o_ka) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int64_t i = s_i[p];
  o_t[i] = dt[p];
  o_ks[i] = dks[p];
  o_ka[i] = dka[p];
}

__global__ void k_fill64(int64_t* p, int64_t n, int64_t v) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

__global__ void k_copy_batches(const BatchRec* __restrict__ recs,
                               const int64_t* __restrict__ rec_base,
                               const int64_t* __restrict__ rec_count,
                               int32_t P, const int32_t* __restrict__ s_i,
                               const int32_t* __restrict__ model_of_slot,
                               const int32_t* __restrict__ slot_base,
                               const int32_t* __restrict__ gpu_base,
                               int64_t total, sym_batch* __restrict__ out) {
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= total) return;
  int s = 0;
  int64_t k = w;
  while (s < P && k >= rec_count[s]) {
    k -= rec_count[s];
    s++;
  }
  const BatchRec& r = recs[rec_base[s] + k];
  sym_batch b;
  b.emitted = r.emitted;
  b.start = r.start;
  b.finish = r.finish;
  b.key_t = r.kt;
  b.key_sub = r.ksub;
  b.key_a = r.ka;
  b.model = model_of_slot[slot_base[s] + r.model];
  b.gpu = gpu_base[s] + r.gpu;
  b.size = r.size;
  b.first_index = s_i[r.first];
  b.shrunk_from = r.shrunk_from;
  out[w] = b;
}

inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }


// --------------------------------------------------------- K3 fast path ---
// (fastpath.cuh).  All sub-clusters are processed together: sort keys carry
// the shard id above the tick bits (tb = bits needed by the run's ticks).


__device__ __forceinline__ int shard_of_slot(const int32_t* slot_base, int32_t P,
                                             int32_t k) {
  int s = 0;
  while (s + 1 < P && slot_base[s + 1] <= k) s++;
  return s;
}

// K3a: one thread per model: its unconstrained batch sequence
__global__ void __launch_bounds__(64)
k_evolve(const Shard* __restrict__ shards, const int32_t* __restrict__ slot_base,
         int32_t P, int32_t M, const FreshRec* __restrict__ fresh,
         EvBatch* __restrict__ evb, int32_t* __restrict__ nb,
         int64_t* __restrict__ mdrops, uint32_t* __restrict__ fail,
         const int32_t* __restrict__ only) {
  const int32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= M || (only && !only[k])) return;
  const int s = shard_of_slot(slot_base, P, k);
  const Shard& S = shards[s];
  const int32_t m = k - slot_base[s];
  const ModelParam& mp = S.mp[m];
  uint32_t f = 0;
  int64_t dr = 0;
  const int32_t c = evolve_model(S, m, fresh, evb + mp.off, mp.cnt, &dr, &f);
  nb[k] = c < 0 ? 0 : c;
  mdrops[k] = dr;
  if (f) atomicOr(&fail[s], f);
}


// K3a' (parallel unconstrained evolution).  J1 = the chain pointer where it
// continues; J_{2k}[p] = J_k[J_k[p]]: the position 2k batches after p, or -1
// if the chain ends (or needs the sequential path) within 2k batches.
// J_{4k} = (J_k)^4 in one pass: three gathers that stay near p (chains move
// forward by ~a batch per hop), so four doublings' worth of pointer chasing
// costs one read, three L2-local gathers and one write per position.
// first: jin is the raw chain pointer (NX_* sentinels -> -1).
// Each thread follows kJumpIlp independent chains (block-strided, so loads
// and stores stay coalesced) with their gathers interleaved: the pass is
// bound by dependent L2 latency, not bytes.
constexpr int kJumpIlp = 4;
__global__ void __launch_bounds__(256)
k_jump4(const int32_t* __restrict__ jin, int32_t* __restrict__ jout, int64_t n) {
  const int64_t base = (int64_t)blockIdx.x * blockDim.x * kJumpIlp + threadIdx.x;
  int32_t v[kJumpIlp];
#pragma unroll
  for (int k = 0; k < kJumpIlp; k++) {
    const int64_t p = base + (int64_t)k * blockDim.x;
    v[k] = p < n ? jin[p] : -1;
  }
#pragma unroll
  for (int h = 0; h < 3; h++)
#pragma unroll
    for (int k = 0; k < kJumpIlp; k++) v[k] = v[k] >= 0 ? jin[v[k]] : -1;
#pragma unroll
  for (int k = 0; k < kJumpIlp; k++) {
    const int64_t p = base + (int64_t)k * blockDim.x;
    if (p < n) jout[p] = v[k] >= 0 ? v[k] : -1;
  }
}

constexpr int kJump = 64;  // batches per checkpoint (J_64)

// One thread per model: follow J_64 from the model's first position,
// recording a checkpoint every 64 batches; then count the tail with the
// single-step pointers.  Models whose chain meets NX_SPECIAL are left to
// the sequential k_evolve (special[k] = 1).
// One thread per model walks its batch chain: J_256 hops (coarse
// checkpoints, every 4th checkpoint slot), then J_64 hops, then the < 64
// remaining batches one by one (counting them and spotting a special
// model).  The three checkpoints between two coarse ones are filled in
// parallel by k_walk_fill.  A coarse slot that has a successor is marked by
// cp_model = -2 - k until filled.
constexpr int kCoarse = 4;  // checkpoints per J_256 hop
constexpr int kSub = 16;    // batches per k_walk_expand thread (J_16)

__global__ void k_walk(const ModelParam* __restrict__ mp_all, int32_t M,
                       const int32_t* __restrict__ nxt, const int32_t* __restrict__ j16,
                       const int32_t* __restrict__ j64, const int32_t* __restrict__ j256,
                       int32_t* __restrict__ cp_pos, int32_t* __restrict__ cp_model,
                       int32_t* __restrict__ nb, int32_t* __restrict__ special) {
  const int32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= M) return;
  const ModelParam& mp = mp_all[k];
  int32_t count = 0, sp = 0;
  if (mp.cnt > 0) {
    const int64_t cbase = mp.off / kJump + k;  // disjoint per-model slots
    int32_t p = mp.off, c = 0;
    for (int32_t q = j256[p]; q >= 0; q = j256[p]) {
      cp_pos[cbase + c] = p;
      cp_model[cbase + c] = -2 - k;  // k_walk_fill completes slots c+1..c+3
      c += kCoarse;
      p = q;
    }
    while (j64[p] >= 0) {
      cp_pos[cbase + c] = p;
      cp_model[cbase + c] = k;
      c++;
      p = j64[p];
    }
    cp_pos[cbase + c] = p;
    cp_model[cbase + c] = k;
    count = c * kJump;
    for (int32_t q = j16[p]; q >= 0; q = j16[p]) {  // < 64 left: J_16 hops
      count += kSub;
      p = q;
    }
    for (;;) {  // tail: < 16 batches
      const int32_t v = nxt[p];
      if (v == NX_SPECIAL) {
        sp = 1;
        break;
      }
      if (v == NX_NONE) break;
      count++;
      if (v == NX_LAST) break;
      p = v;
    }
  }
  nb[k] = sp ? 0 : count;
  special[k] = sp;
}

__global__ void k_walk_fill(int32_t* __restrict__ cp_pos, int32_t* __restrict__ cp_model,
                            int64_t ncp, const int32_t* __restrict__ j64) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= ncp) return;
  const int32_t tag = cp_model[q];
  if (tag > -2) return;  // not a coarse slot with a successor
  const int32_t k = -2 - tag;
  int32_t p = cp_pos[q];
  cp_model[q] = k;
  for (int h = 1; h < kCoarse; h++) {
    p = j64[p];
    cp_pos[q + h] = p;
    cp_model[q + h] = k;
  }
}

// Compact checkpoint numbering for k_walk_expand: cpoff[k] = first compact
// checkpoint of model k (exclusive scan of max(1, ceil(nb / kJump)) over the
// models k_walk walked; special models have none), cpoff[M] = the total.
// k_walk lays checkpoints out in per-model slot ranges sized by arrivals
// (~10x the batches), so a launch over slots would leave 90 % of its threads
// idle beside the few that walk.
__global__ void __launch_bounds__(1024)
k_cp_scan(const ModelParam* __restrict__ mp_all, int32_t M, const int32_t* __restrict__ nb,
          const int32_t* __restrict__ special, int32_t* __restrict__ cpoff) {
  __shared__ int32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int32_t b0 = 0; b0 < M; b0 += 1024) {
    const int32_t k = b0 + threadIdx.x;
    int32_t v = 0;
    if (k < M && mp_all[k].cnt > 0 && !special[k]) v = max(1, (nb[k] + kJump - 1) / kJump);
    int32_t tot;
    const int32_t ex = block_exclusive_scan(v, &tot);
    const int32_t c = carry;
    if (k < M) cpoff[k] = c + ex;
    __syncthreads();
    if (threadIdx.x == 0) carry = c + tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) cpoff[M] = carry;
}

// One warp per checkpoint (compact numbering), persistent: the checkpoint's
// <= 64 batch starts lie in a short run of its model's positions, so the
// chain pointers (J_1) and the J_16 pointers of kExpandWin positions from the
// checkpoint arrive in shared memory by bulk copies (cp.async.bulk on one
// mbarrier) issued one checkpoint ahead into the warp's other buffer.  Lanes
// 0..3 take J_16 hops to batches 0, 16, 32, 48 and each follows 16 chain
// pointers through shared memory (global loads only past the window); they
// write the starts to bstart[] (k_chain_recs reads them there, not from the
// 56-byte EvBatch records).
constexpr int kExpandWin = 1024;
constexpr int kExpandWarps = 4;
constexpr int kExpandSmem = kExpandWarps * (4 * kExpandWin * 4 + 16);
__device__ __forceinline__ void bulk_load2(void* dst0, const void* src0, void* dst1,
                                           const void* src1, uint32_t bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(2 * bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_u32(dst0)), "l"(src0), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_u32(dst1)), "l"(src1), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__global__ void __launch_bounds__(32 * kExpandWarps)
k_walk_expand(const int32_t* __restrict__ cp_pos, const int32_t* __restrict__ cpoff, int32_t M,
              const ModelParam* __restrict__ mp_all,
              const int32_t* __restrict__ slot_base, int32_t P,
              const int32_t* __restrict__ nxt, const int32_t* __restrict__ j16,
              const Shard* __restrict__ shards,
              int32_t* __restrict__ bstart, unsigned long long* __restrict__ mdrops) {
  extern __shared__ __align__(128) unsigned char ex_smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  // per warp: [buffer][J_1 | J_16][kExpandWin]
  int32_t(*win)[2][kExpandWin] =
      reinterpret_cast<int32_t(*)[2][kExpandWin]>(ex_smem + w * 4 * kExpandWin * 4);
  uint64_t* bar = reinterpret_cast<uint64_t*>(ex_smem + kExpandWarps * 4 * kExpandWin * 4) + w * 2;
  const int32_t total = cpoff[M];
  const int32_t W = gridDim.x * kExpandWarps;
  int32_t c = blockIdx.x * kExpandWarps + w;
  if (lane == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  // checkpoint cc: model k, ordinal, first position, window base (16-byte aligned)
  int32_t k = 0, ord = 0, p0 = 0, base = 0;
  auto locate = [&](int32_t cc) {
    k = warp_last_le(cpoff, M, cc, lane);  // cpoff[k] <= cc < cpoff[k+1]
    ord = cc - cpoff[k];
    p0 = cp_pos[mp_all[k].off / kJump + k + ord];
    base = p0 & ~3;
  };
  // reads up to kExpandWin - 1 past n (capacity n + 1024); never used
  auto issue = [&](int b) {
    bulk_load2(win[b][0], nxt + base, win[b][1], j16 + base, kExpandWin * 4, &bar[b]);
  };
  if (c < total) {
    locate(c);
    if (lane == 0) issue(0);
  }
  uint32_t phase = 0;
  for (int b = 0; c < total; c += W, b ^= 1) {
    const int32_t ck = k, cord = ord, cp0 = p0, cbase = base;
    if (c + W < total) {  // the next checkpoint's windows, one ahead
      locate(c + W);
      if (lane == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(b ^ 1);
      }
    }
    const ModelParam& mp = mp_all[ck];
    mbar_wait(&bar[b], (phase >> b) & 1);
    phase ^= 1u << b;
    if (lane < kJump / kSub) {
      const int32_t* w1 = win[b][0];
      const int32_t* w16 = win[b][1];
      int32_t p = cp0;
      for (int h = 0; h < lane && p >= 0; h++)
        p = p - cbase < kExpandWin ? w16[p - cbase] : j16[p];
      if (p >= 0) {
        int64_t out = mp.off + (int64_t)cord * kJump + lane * kSub;
        for (int j = 0; j < kSub && p >= 0; j++) {
          const int32_t v = p - cbase < kExpandWin ? w1[p - cbase] : nxt[p];
          if (v == NX_NONE) {  // trailing all-dropped scan: count its drops
            const int s = shard_of_slot(slot_base, P, ck);
            const FreshRec r =
                fresh_scan(shards[s], ck - slot_base[s], p - mp.off, kFreshMaxSteps);
            atomicAdd(&mdrops[ck], (unsigned long long)r.drops);
            break;
          }
          if (v == NX_SPECIAL) break;
          bstart[out++] = p;
          if (v == NX_LAST) break;
          p = v;
        }
      }
    }
    __syncwarp();  // every lane is done with buffer b before it is refilled
  }
}

// One thread per batch of the fast path: the full fresh-start record of its
// chain position gives the batch (timer key, exec_at, l(b), size, members)
// and the heads dropped before it.
__global__ void __launch_bounds__(256)
k_chain_recs(const Shard* __restrict__ shards, const int32_t* __restrict__ slot_base,
             int32_t P, int32_t M, const ModelParam* __restrict__ mp_all,
             const int32_t* __restrict__ nb, const int32_t* __restrict__ bbase,
             const int32_t* __restrict__ special, int64_t nt, EvBatch* __restrict__ evb,
             unsigned long long* __restrict__ mdrops, const int32_t* __restrict__ close_k,
             const int32_t* __restrict__ bstart,
             uint64_t* __restrict__ keys, uint32_t* __restrict__ vals,
             uint32_t* __restrict__ fail, int tb) {
  const int64_t d = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  // the warp's first batch locates its model by a 32-ary search (two loads
  // per lane); a warp's 32 batches almost always share it
  const int64_t d0 = __shfl_sync(0xffffffffu, d, 0);
  int lo = warp_last_le(bbase, M, d0 < nt ? d0 : nt - 1, threadIdx.x & 31);
  if (d >= nt) return;
  while (nb[lo] == 0 || bbase[lo] + nb[lo] <= d) lo++;
  const int s = shard_of_slot(slot_base, P, lo);
  const ModelParam& mp = mp_all[lo];
  const int64_t p = mp.off + (d - bbase[lo]);
  EvBatch& e = evb[p];
  if (!special[lo]) {  // special models' records come from k_evolve
    const int32_t m = lo - slot_base[s];
    const int32_t first = bstart[p];  // listed by k_walk_expand
    const int32_t ck = close_k[first];
    if (ck >= 0) {  // certified by the lean sweep: O(1) from (q, k)
      lean_batch(shards[s], m, first - mp.off, ck, e);
    } else {
      const FreshRec r = fresh_scan(shards[s], m, first - mp.off, kFreshMaxSteps);
      e.t = r.mt_t;
      e.a = r.mt_a;
      e.tp = r.mt_tp;
      e.ap = r.mt_ap;
      e.chain = 0;  // fresh scans only hold arrival-pushed timers
      e.exec = r.c_exec;
      e.lat = r.c_lb;
      e.size = r.c_size;
      e.first = mp.off + r.qh;
      e.model = m;
      if (r.drops) atomicAdd(&mdrops[lo], (unsigned long long)r.drops);
    }
  }
  // the batch's merge key, in the per-model run layout
  const int64_t t = e.t;
  if (t < 0 || t >= (int64_t(1) << tb)) atomicOr(&fail[s], FP_CAPACITY);
  keys[d] = ((uint64_t)s << tb) | (uint64_t)(t & ((int64_t(1) << tb) - 1));
  vals[d] = (uint32_t)p;
}

// K3b: dense batch numbering: bbase[k] per model (slot order is
// shard-major), sbase[s] per shard; one block scan
__global__ void __launch_bounds__(1024)
k_nb_scan(const int32_t* __restrict__ nb, int32_t M, int32_t P,
          const int32_t* __restrict__ slot_base, int32_t* __restrict__ bbase,
          int64_t* __restrict__ sbase) {
  __shared__ int32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int32_t b0 = 0; b0 < M; b0 += 1024) {
    const int32_t k = b0 + threadIdx.x;
    int32_t tot;
    const int32_t ex = block_exclusive_scan(k < M ? nb[k] : 0, &tot);
    const int32_t c = carry;
    if (k < M) bbase[k] = c + ex;
    __syncthreads();
    if (threadIdx.x == 0) carry = c + tot;
    __syncthreads();
  }
  const int32_t total = carry;
  for (int32_t sh = threadIdx.x; sh <= P; sh += blockDim.x)
    sbase[sh] = sh < P && slot_base[sh] < M ? bbase[slot_base[sh]] : total;
}

// K3c: (shard|tick) keys of every batch, value = its EvBatch index

// --- LSD radix sort of (u64 key, u32 value) pairs, 8-bit digits, stable ---

constexpr int kDigitBits = 8;
constexpr int kDigits = 1 << kDigitBits;  // radix bins
constexpr int kRadixWarps = 4;            // warps per block (1 KB smem each)

__global__ void __launch_bounds__(32 * kRadixWarps)
k_rhist(const uint64_t* __restrict__ keys, int64_t n, int shift,
        int32_t* __restrict__ hist, int64_t W) {
  __shared__ int32_t cnt[kRadixWarps][kDigits];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t w = (int64_t)blockIdx.x * kRadixWarps + wib;
  for (int b = lane; b < kDigits; b += 32) cnt[wib][b] = 0;
  __syncwarp();
  if (w < W) {  // all of the lane's keys in flight at once, then count
    constexpr int R = kChunkR / 32;
    const int64_t lo = w * kChunkR, hi = (lo + kChunkR < n ? lo + kChunkR : n);
    uint64_t k[R];
#pragma unroll
    for (int r = 0; r < R; r++) {
      const int64_t i = lo + r * 32 + lane;
      k[r] = i < hi ? keys[i] : 0;
    }
#pragma unroll
    for (int r = 0; r < R; r++)
      if (lo + r * 32 + lane < hi) atomicAdd(&cnt[wib][(k[r] >> shift) & (kDigits - 1)], 1);
  }
  __syncwarp();
  if (w < W)
    for (int b = lane; b < kDigits; b += 32) hist[(int64_t)b * W + w] = cnt[wib][b];
}

__global__ void __launch_bounds__(32 * kRadixWarps)
k_rscatter(const uint64_t* __restrict__ kin,
                           const uint32_t* __restrict__ vin, int64_t n, int shift,
                           const int32_t* __restrict__ hist, int64_t W,
                           uint64_t* __restrict__ kout, uint32_t* __restrict__ vout) {
  __shared__ int32_t base_s[kRadixWarps][kDigits];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t w = (int64_t)blockIdx.x * kRadixWarps + wib;
  if (w >= W) return;
  int32_t* base = base_s[wib];
  for (int b = lane; b < kDigits; b += 32) base[b] = hist[(int64_t)b * W + w];
  __syncwarp();
  const unsigned lt = (1u << lane) - 1u;
  const int64_t lo = w * kChunkR, hi = (lo + kChunkR < n ? lo + kChunkR : n);
  // all of the lane's keys and values in flight at once (the pass is
  // latency-bound: few warps per SM for ~10^6 keys), then rank round by round
  constexpr int R = kChunkR / 32;
  uint64_t k[R];
  uint32_t v[R];
#pragma unroll
  for (int r = 0; r < R; r++) {
    const int64_t i = lo + r * 32 + lane;
    k[r] = i < hi ? kin[i] : 0;
    v[r] = i < hi ? vin[i] : 0;
  }
#pragma unroll
  for (int r = 0; r < R; r++) {
    const bool act = lo + r * 32 + lane < hi;
    const int32_t dg = act ? (int32_t)((k[r] >> shift) & (kDigits - 1)) : -1 - lane;
    const unsigned peers = __match_any_sync(0xffffffffu, dg);
    int32_t pos = 0;
    if (act) pos = base[dg] + __popc(peers & lt);
    __syncwarp();
    if (act) {
      if ((peers >> lane) == 1u) base[dg] += __popc(peers);
      kout[pos] = k[r];
      vout[pos] = v[r];
    }
    __syncwarp();
  }
}

// ---- bucket sort of (shard|time key, value) pairs -------------------------
// Batch grant ticks and finish times are spread over the run, ~1 per bucket
// of 2^S ns when there are about as many buckets as keys: count per bucket
// (atomics), one exclusive scan, scatter (atomic slot per bucket, order
// within a bucket arbitrary), then one thread per bucket insertion-sorts its
// few keys by the full order.  Four launches instead of a radix sort's
// five passes of histogram + scan + scatter (or ceil(log2 M) merge rounds),
// and the result is the same total order: ties beyond the key are broken by
// the batch event order (batches, FP_KEY_TIE if that ties too) or the value
// (tokens: the creator's rank, i.e. the stable order).
__global__ void k_bkt_count(const uint64_t* __restrict__ keys, int64_t n, int shift,
                            int32_t* __restrict__ cnt) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) atomicAdd(&cnt[keys[i] >> shift], 1);
}

__global__ void k_bkt_scatter(const uint64_t* __restrict__ kin, const uint32_t* __restrict__ vin,
                              int64_t n, int shift, int32_t* __restrict__ next,
                              uint64_t* __restrict__ kout, uint32_t* __restrict__ vout) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t k = kin[i];
  const int32_t pos = atomicAdd(&next[k >> shift], 1);  // ends up at the bucket's end
  kout[pos] = k;
  vout[pos] = vin[i];
}

template <bool kBatches>
__global__ void k_bkt_sort(const int32_t* __restrict__ end, int64_t nbuckets,
                           uint64_t* __restrict__ keys, uint32_t* __restrict__ vals,
                           const EvBatch* __restrict__ evb) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nbuckets) return;
  const int32_t lo = b ? end[b - 1] : 0, hi = end[b];
  for (int32_t a = lo + 1; a < hi; a++) {
    const uint64_t k = keys[a];
    const uint32_t v = vals[a];
    int32_t c = a;
    for (; c > lo; c--) {
      const uint64_t pk = keys[c - 1];
      const uint32_t pv = vals[c - 1];
      bool before;  // (k, v) strictly before (pk, pv)
      if (k != pk) {
        before = k < pk;
      } else if (kBatches) {
        const int o = batch_cmp(evb[v], evb[pv]);
        before = o != 0 ? o < 0 : v < pv;
      } else {
        before = v < pv;
      }
      if (!before) break;
      keys[c] = pk;
      vals[c] = pv;
    }
    keys[c] = k;
    vals[c] = v;
  }
}

// K3e: finish-time token of every sorted batch: key (shard|finish),
// value = the batch's rank within its shard
__global__ void k_token_keys(const uint32_t* __restrict__ bvals, int64_t nt,
                             const uint64_t* __restrict__ bkeys,
                             const EvBatch* __restrict__ evb,
                             const int64_t* __restrict__ sbase,
                             uint64_t* __restrict__ tkeys, uint32_t* __restrict__ tvals,
                             uint32_t* __restrict__ fail, int tb) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nt) return;
  const int s = (int)(bkeys[i] >> tb);
  const EvBatch& e = evb[bvals[i]];
  // two batches whose keys tie up to the chain counter: order undecidable
  if (i + 1 < nt && bkeys[i + 1] == bkeys[i] && batch_cmp(e, evb[bvals[i + 1]]) == 0)
    atomicOr(&fail[s], FP_KEY_TIE);
  const int64_t fin = e.exec + e.lat;
  if (fin < 0 || fin >= (int64_t(1) << tb)) atomicOr(&fail[s], FP_CAPACITY);
  tkeys[i] = ((uint64_t)s << tb) | (uint64_t)(fin & ((int64_t(1) << tb) - 1));
  tvals[i] = (uint32_t)(i - sbase[s]);
}

constexpr int kTieMax = 256;    // tie groups listed per sub-cluster
constexpr int kTieEff = 64;     // effective (re-sorted) groups per sub-cluster
constexpr int kTieX = 256;      // sigma pairs (= explicit labels) per sub-cluster

// The matching phase in one cooperative launch: match (batch r pops token
// r) -> pointer jumping to convergence -> list the equal-finish token groups
// (k_tie_fix orders them by gid; k_fast_emit applies the relabelling).
// Grid-wide syncs replace host round trips.
__global__ void __launch_bounds__(256)
k_match_coop(const uint64_t* __restrict__ bkeys, const uint32_t* __restrict__ bvals,
             int64_t nt, const int64_t* __restrict__ sbase,
             const Shard* __restrict__ shards, const uint64_t* __restrict__ tkeys,
             uint32_t* __restrict__ tvals, int32_t* __restrict__ ptrA,
             int32_t* __restrict__ flags, int tb, int32_t* __restrict__ tie_cnt,
             int32_t* __restrict__ tie_list) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  (void)flags;
  for (int64_t i = tid0; i < nt; i += stride) {  // match
    const int s = (int)(bkeys[i] >> tb);
    const int64_t r = i - sbase[s];
    const int32_t G = shards[s].G;
    if (r < G) {
      ptrA[i] = -(int32_t)r - 1;
    } else {
      const int64_t c = tvals[sbase[s] + (r - G)];
      ptrA[i] = c < r ? (int32_t)(sbase[s] + c) : -1;
    }
  }
  grid.sync();
  // Resolve gids by pointer jumping IN PLACE and without barriers: every
  // entry always holds an ancestor on its creator chain (or the resolved
  // -gid-1), so reading a neighbour's stale or freshly jumped value is
  // equally valid, and each jump strictly shortens the remaining chain.
  // Loads bypass L1 (other SMs write these entries).  Each thread sweeps
  // its entries until all are resolved: ~log2(depth) sweeps, one grid
  // barrier in total instead of two per doubling round.
  for (bool open = true; open;) {
    open = false;
    for (int64_t i = tid0; i < nt; i += stride) {
      const int32_t v = __ldcg(ptrA + i);
      if (v < 0) continue;
      const int32_t w = __ldcg(ptrA + v);
      __stcg(ptrA + i, w);
      open |= w >= 0;
    }
  }
  // equal-finish token groups: listed per sub-cluster for k_tie_fix (a
  // handful per sub-cluster: C4 has 5-6 in 870k batches)
  for (int64_t i = tid0; i < nt; i += stride) {
    if (i > 0 && tkeys[i - 1] == tkeys[i]) continue;
    if (i + 1 >= nt || tkeys[i + 1] != tkeys[i]) continue;
    const int s = (int)(tkeys[i] >> tb);
    const int32_t slot = atomicAdd(&tie_cnt[s], 1);
    if (slot < kTieMax) tie_list[(int64_t)s * kTieMax + slot] = (int32_t)(i - sbase[s]);
  }
}

// Equal-finish tokens must pop in gid order, but the gids depend on which
// batch pops which token.  k_match_coop resolved the gids with each tie
// group in creator order; here one thread per sub-cluster walks its tie
// groups in rank order.  Re-sorting group g (tokens a..b, popped by the
// batches R = a + G ... R + k - 1) by its creators' labels swaps which chain
// continues through which of those batches: every later batch whose label
// is one of the group's old labels L_j lies on that chain after R + j, so
// its label becomes L'_j (sigma_g), and batch R + j itself gets L'_j.  A
// batch's final label is its pass-one gid with the sigmas of the groups
// below it applied in rank order (a few label pairs in all: C4 has 5-6 tie
// groups per sub-cluster), so k_fast_emit reads every final gid in passing
// instead of the match and the pointer jumping running again.  A creator inside its
// own group, or more groups or pairs than the scratch holds, sends the
// sub-cluster to the exact chain (FP_TOKEN_TIE); k_fast_emit re-checks every
// tie against the final gids.
__device__ __forceinline__ int32_t tie_label(int32_t x, int32_t lab,
                                             const int4* __restrict__ eff, int32_t neff,
                                             const int2* __restrict__ sig) {
  for (int32_t m = 0; m < neff; m++) {
    const int4 e = eff[m];  // R, E, pair offset, pair count (= E - R)
    if (x < e.x) break;
    if (x < e.y) return sig[e.z + (x - e.x)].y;  // a popping batch: explicit
    for (int32_t j = 0; j < e.w; j++)
      if (lab == sig[e.z + j].x) {
        lab = sig[e.z + j].y;
        break;
      }
  }
  return lab;
}

constexpr int kTieGroupS = 8;   // tokens per tie group held for the relabelling
constexpr int kTieThreads = 256;
static_assert(kTieThreads >= kTieMax, "one thread per listed tie group");

// One block per sub-cluster: the groups' tokens, creators and pass-one gids
// are loaded in parallel (one thread per group), thread 0 walks the groups
// in rank order through shared memory, and the block writes the results.
__global__ void __launch_bounds__(kTieThreads)
k_tie_fix(const int64_t* __restrict__ sbase, const Shard* __restrict__ shards,
          int32_t P, const uint64_t* __restrict__ tkeys, uint32_t* __restrict__ tvals,
          const int32_t* __restrict__ ptrA, int32_t* __restrict__ tie_cnt,
          const int32_t* __restrict__ tie_list, int4* __restrict__ tie_eff,
          int2* __restrict__ tie_sig, uint32_t* __restrict__ tie_mask,
          int32_t* __restrict__ overflow) {
  __shared__ int32_t s_list[kTieMax], g_a[kTieMax], g_k[kTieMax];
  __shared__ int32_t g_cr[kTieMax][kTieGroupS], g_g1[kTieMax][kTieGroupS];
  __shared__ int32_t g_ord[kTieMax][kTieGroupS];
  __shared__ int32_t g_moved[kTieMax];
  __shared__ int4 e_sm[kTieEff];
  __shared__ int2 sig_sm[kTieX];
  __shared__ uint32_t mask_sm[32];
  __shared__ int32_t s_cnt, s_bad, s_neff, s_used;
  const int s = blockIdx.x, t = threadIdx.x;
  if (s >= P) return;
  if (t == 0) {
    s_cnt = tie_cnt[s];
    s_bad = s_cnt > kTieMax;
    s_neff = s_used = 0;
  }
  if (t < 32) mask_sm[t] = 0;
  __syncthreads();
  const int32_t cnt = s_cnt;
  if (s_bad) {
    if (t == 0) {
      tie_cnt[s] = 0;
      *overflow = 1;  // k_match_iter redoes the matching
    }
    if (t < 32) tie_mask[(int64_t)s * 32 + t] = 0;
    return;
  }
  const int64_t base = sbase[s];
  const int32_t nb = (int32_t)(sbase[s + 1] - base), G = shards[s].G;
  if (t < cnt) s_list[t] = tie_list[(int64_t)s * kTieMax + t];
  __syncthreads();
  if (t < cnt) {  // rank order of the group starts (distinct)
    const int32_t a = s_list[t];
    int32_t pos = 0;
    for (int32_t u = 0; u < cnt; u++) pos += s_list[u] < a;
    g_a[pos] = a;
  }
  __syncthreads();
  if (t < cnt) {  // this group's tokens: extent, creators, pass-one gids
    const int32_t a = g_a[t];
    int32_t k = 1;
    while (k <= kTieGroupS && a + k < nb && tkeys[base + a + k] == tkeys[base + a]) k++;
    const int32_t R = a + G;
    bool bad = k > kTieGroupS;
    for (int32_t j = 0; j < k && !bad; j++) {
      const int32_t c = (int32_t)tvals[base + a + j];
      g_cr[t][j] = c;
      if (R < nb && c >= R) bad = true;  // a creator inside its own group
      else g_g1[t][j] = -ptrA[base + c] - 1;
    }
    g_k[t] = k;
    if (bad) atomicExch(&s_bad, 1);
  }
  __syncthreads();
  if (s_bad) {
    if (t == 0) {
      tie_cnt[s] = 0;
      *overflow = 1;
    }
    if (t < 32) tie_mask[(int64_t)s * 32 + t] = 0;
    return;
  }
  if (t == 0) {  // the groups in rank order
    int32_t neff = 0, used = 0;
    for (int32_t q = 0; q < cnt && !s_bad; q++) {
      const int32_t a = g_a[q], k = g_k[q], R = a + G;
      const int32_t kp = R < nb ? min(k, nb - R) : 0;  // tokens some batch pops
      int32_t lab[kTieGroupS];
      for (int32_t j = 0; j < k; j++) {
        lab[j] = tie_label(g_cr[q][j], g_g1[q][j], e_sm, neff, sig_sm);
        g_ord[q][j] = j;
      }
      bool moved = false;
      for (int32_t j = 1; j < k; j++) {  // insertion sort by label (distinct GPUs)
        const int32_t v = g_ord[q][j];
        int32_t b = j;
        for (; b > 0 && lab[g_ord[q][b - 1]] > lab[v]; b--) {
          g_ord[q][b] = g_ord[q][b - 1];
          moved = true;
        }
        g_ord[q][b] = v;
      }
      g_moved[q] = moved;
      if (!moved || kp == 0) continue;  // unpopped tokens: order only
      if (neff == kTieEff || used + kp > kTieX) {
        s_bad = 1;
        break;
      }
      for (int32_t j = 0; j < kp; j++) {
        sig_sm[used + j] = make_int2(lab[j], lab[g_ord[q][j]]);
        mask_sm[(lab[j] >> 5) & 31] |= 1u << (lab[j] & 31);
      }
      e_sm[neff] = make_int4(R, R + kp, used, kp);
      neff++;
      used += kp;
    }
    s_neff = neff;
    s_used = used;
  }
  __syncthreads();
  if (s_bad) {
    if (t == 0) {
      tie_cnt[s] = 0;
      *overflow = 1;
    }
    if (t < 32) tie_mask[(int64_t)s * 32 + t] = 0;
    return;
  }
  if (t < cnt && g_moved[t]) {  // re-sorted tokens
    const int32_t a = g_a[t];
    for (int32_t j = 0; j < g_k[t]; j++) tvals[base + a + j] = (uint32_t)g_cr[t][g_ord[t][j]];
  }
  for (int32_t q = t; q < s_neff; q += blockDim.x) tie_eff[(int64_t)s * kTieEff + q] = e_sm[q];
  for (int32_t q = t; q < s_used; q += blockDim.x) tie_sig[(int64_t)s * kTieX + q] = sig_sm[q];
  if (t < 32) tie_mask[(int64_t)s * 32 + t] = mask_sm[t];
  if (t == 0) tie_cnt[s] = s_neff;
}

// Fallback for tie-heavy runs (more tie groups, relabelled labels or
// group tokens than k_tie_fix's scratch holds, or a creator inside its own
// group: e.g. C3's 50 % same-tick arrivals): the whole matching phase again,
// iterated -- match, pointer jumping, re-sort every equal-finish group by
// gid -- until no group moves.  Launched every run; returns at once unless
// k_tie_fix raised the overflow flag.
__global__ void __launch_bounds__(256)
k_match_iter(const uint64_t* __restrict__ bkeys, const uint32_t* __restrict__ bvals,
             int64_t nt, const int64_t* __restrict__ sbase,
             const Shard* __restrict__ shards, const uint64_t* __restrict__ tkeys,
             uint32_t* __restrict__ tvals, int32_t* __restrict__ ptrA,
             int32_t* __restrict__ flags, int tb, int32_t* __restrict__ tie_neff,
             int32_t P) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (flags[0] == 0) return;  // no sub-cluster overflowed k_tie_fix (grid-uniform)
  grid.sync();                 // every thread has read the flag
  if (tid0 == 0) flags[0] = flags[1] = flags[2] = flags[3] = 0;
  if (tid0 < P) tie_neff[tid0] = 0;  // the gids below are final: no relabelling
  grid.sync();
  for (int it = 0; it < 16; it++) {
    for (int64_t i = tid0; i < nt; i += stride) {  // match
      const int s = (int)(bkeys[i] >> tb);
      const int64_t r = i - sbase[s];
      const int32_t G = shards[s].G;
      if (r < G) {
        ptrA[i] = -(int32_t)r - 1;
      } else {
        const int64_t c = tvals[sbase[s] + (r - G)];
        ptrA[i] = c < r ? (int32_t)(sbase[s] + c) : -1;
      }
    }
    grid.sync();
    // Resolve gids by pointer jumping IN PLACE and without barriers: every
    // entry always holds an ancestor on its creator chain (or the resolved
    // -gid-1), so reading a neighbour's stale or freshly jumped value is
    // equally valid, and each jump strictly shortens the remaining chain.
    // Loads bypass L1 (other SMs write these entries).  Each thread sweeps
    // its entries until all are resolved: ~log2(depth) sweeps, one grid
    // barrier in total instead of two per doubling round.
    for (bool open = true; open;) {
      open = false;
      for (int64_t i = tid0; i < nt; i += stride) {
        const int32_t v = __ldcg(ptrA + i);
        if (v < 0) continue;
        const int32_t w = __ldcg(ptrA + v);
        __stcg(ptrA + i, w);
        open |= w >= 0;
      }
    }
    grid.sync();
    if (tid0 == 0) flags[2 + ((it + 1) & 1)] = 0;
    bool moved = false;
    for (int64_t i = tid0; i < nt; i += stride) {  // equal-finish groups by gid
      if (i > 0 && tkeys[i - 1] == tkeys[i]) continue;
      if (i + 1 >= nt || tkeys[i + 1] != tkeys[i]) continue;
      const int64_t base = sbase[tkeys[i] >> tb];
      int64_t e = i + 1;
      while (e < nt && tkeys[e] == tkeys[i]) e++;
      for (int64_t a = i + 1; a < e; a++) {
        const uint32_t v = tvals[a];
        const int32_t gv = -ptrA[base + v] - 1;
        int64_t b = a;
        while (b > i && -ptrA[base + tvals[b - 1]] - 1 > gv) {
          tvals[b] = tvals[b - 1];
          b--;
          moved = true;
        }
        tvals[b] = v;
      }
    }
    if (moved) flags[2 + (it & 1)] = 1;
    grid.sync();
    if (tid0 == 0) flags[1] = it + 1;  // passes run (SYM_DEBUG_TIMING=1 prints it)
    if (flags[2 + (it & 1)] == 0) break;
    grid.sync();
  }
}

// K3g: token ties must pop in gid order; emit the BatchRec of every batch
__global__ void k_fast_emit(const uint64_t* __restrict__ bkeys,
                            const uint32_t* __restrict__ bvals, int64_t nt,
                            const EvBatch* __restrict__ evb,
                            const int64_t* __restrict__ sbase,
                            const uint64_t* __restrict__ tkeys,
                            const uint32_t* __restrict__ tvals,
                            const int32_t* __restrict__ gid,
                            const int32_t* __restrict__ tie_neff,
                            const int4* __restrict__ tie_eff, const int2* __restrict__ tie_sig,
                            const uint32_t* __restrict__ tie_mask,
                            const int64_t* __restrict__ rec_base,
                            const Shard* __restrict__ shards,
                            BatchRec* __restrict__ recs, uint32_t* __restrict__ fail, int tb) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nt) return;
  const int s = (int)(bkeys[i] >> tb);
  const int64_t r = i - sbase[s];
  // final gid of the sub-cluster's batch d: the pass-one gid, relabelled by
  // the tie groups below d (k_tie_fix; usually none below)
  const int32_t neff = tie_neff[s];
  const int4* eff = tie_eff + (int64_t)s * kTieEff;
  const int2* sig = tie_sig + (int64_t)s * kTieX;
  const uint32_t* msk = tie_mask + (int64_t)s * 32;
  auto final_gid = [&](int32_t d) {
    const int32_t g = -gid[sbase[s] + d] - 1;
    // a label no sigma takes as input never changes (and every popping
    // batch of a group carries such an input label)
    return neff > 0 && d >= eff[0].x && (msk[(g >> 5) & 31] >> (g & 31) & 1u)
               ? tie_label(d, g, eff, neff, sig)
               : g;
  };
  // token i (shard order) vs token i+1: equal finish => gid order
  if (i + 1 < nt && tkeys[i + 1] == tkeys[i]) {
    const int32_t g0 = final_gid((int32_t)tvals[i]);
    const int32_t g1 = final_gid((int32_t)tvals[i + 1]);
    if (g0 > g1) atomicOr(&fail[s], FP_TOKEN_TIE);
  }
  const EvBatch& e = evb[bvals[i]];
  const int32_t G = shards[s].G;
  if (r >= G) {  // popped token: free by exec_at, created before this batch
    const int64_t ti = sbase[s] + (r - G);
    const int64_t fa = (int64_t)(tkeys[ti] & ((uint64_t(1) << tb) - 1));
    if (fa > e.exec) atomicOr(&fail[s], FP_NO_GPU);
    if ((int64_t)tvals[ti] >= r) atomicOr(&fail[s], FP_LATE_TOKEN);
  }
  BatchRec o;
  o.emitted = e.t;
  o.start = e.exec;
  o.finish = e.exec + e.lat;
  o.kt = e.t;
  o.ka = e.a;
  o.ksub = r;  // processing order = rank (the chain counter of the chain)
  o.model = e.model;
  o.gpu = final_gid((int32_t)r);
  o.size = e.size;
  o.first = e.first;
  o.shrunk_from = 0;
  // four 16-byte stores instead of eleven field stores (the kernel is bound
  // by the LSU queue)
  static_assert(sizeof(BatchRec) == 64 && offsetof(BatchRec, size) == 24,
                "BatchRec is four 16-byte words, size in the second");
  const int4* src = reinterpret_cast<const int4*>(&o);
  int4* dst = reinterpret_cast<int4*>(recs + rec_base[s] + r);
#pragma unroll
  for (int q = 0; q < 4; q++) dst[q] = src[q];
}


// ------------------------------------------------ window reductions (K5) --
// Integer parts of compute_stats (metrics.py:79-94) over the last run:
// per-model outcome counts of arrivals in [lo, hi) and per-GPU busy time
// clipped to the window.
__global__ void k_window_req(const int64_t* __restrict__ ticks,
                             const int32_t* __restrict__ model,
                             const int64_t* __restrict__ outcome, int64_t n, int64_t lo,
                             int64_t hi, unsigned long long* __restrict__ cnt /*[4][M]*/,
                             int32_t M) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t t = ticks[i];
  if (t < lo || t >= hi) return;
  const int32_t m = model[i];
  atomicAdd(&cnt[m], 1ull);
  const int64_t o = outcome[i];
  if (o >= 0 && o <= 2) atomicAdd(&cnt[(1 + o) * M + m], 1ull);
}

__global__ void k_window_busy(const BatchRec* __restrict__ recs,
                              const int64_t* __restrict__ rec_base,
                              const int64_t* __restrict__ rec_count, int32_t P,
                              const int32_t* __restrict__ gpu_base, int64_t total,
                              int64_t lo, int64_t hi, unsigned long long* __restrict__ busy) {
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= total) return;
  int s = 0;
  int64_t k = w;
  while (s < P && k >= rec_count[s]) {
    k -= rec_count[s];
    s++;
  }
  const BatchRec& r = recs[rec_base[s] + k];
  const int64_t a = r.start > lo ? r.start : lo;
  const int64_t b = r.finish < hi ? r.finish : hi;
  if (b > a) atomicAdd(&busy[gpu_base[s] + r.gpu], (unsigned long long)(b - a));
}

// ---- per-model window statistics (compute_stats, metrics.py:71-132) ------
// Sort key of request i for the per-model p99: (model slot, latency) for
// arrivals in the window, latency = finish - arrival or kStatInf for a drop
// (the reference's +inf); arrivals outside go to a trailing dummy slot M.
constexpr int kStatLatBits = 40;
constexpr uint64_t kStatInf = (uint64_t(1) << kStatLatBits) - 1;

__global__ void k_stat_keys(const int64_t* __restrict__ ticks, const int32_t* __restrict__ model,
                            const int64_t* __restrict__ outcome,
                            const int64_t* __restrict__ start, const int64_t* __restrict__ fin,
                            const int32_t* __restrict__ slot_of_model, int64_t n, int64_t lo,
                            int64_t hi, int32_t M, uint64_t* __restrict__ keys,
                            uint32_t* __restrict__ vals, unsigned long long* __restrict__ qd_max,
                            int32_t* __restrict__ err) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t t = ticks[i];
  uint64_t key = (uint64_t)M << kStatLatBits;
  if (t >= lo && t < hi) {
    const int32_t m = model[i];
    uint64_t lat = kStatInf;
    if (outcome[i] != 2) {  // served: latency and queueing delay
      const int64_t l = fin[i] - t;
      if (l < 0 || (uint64_t)l >= kStatInf) atomicExch(err, 1);
      lat = (uint64_t)l;
      atomicMax(&qd_max[m], (unsigned long long)(start[i] - t));
    }
    key = ((uint64_t)slot_of_model[m] << kStatLatBits) | lat;
  }
  keys[i] = key;
  vals[i] = 0;
}

// Batch-size histogram per model of the batches starting in the window.
__global__ void k_stat_hist(const BatchRec* __restrict__ recs, const int64_t* __restrict__ rec_base,
                            const int64_t* __restrict__ rec_count, int32_t P,
                            const int32_t* __restrict__ slot_base,
                            const int32_t* __restrict__ model_of_slot, int64_t total, int64_t lo,
                            int64_t hi, int32_t stride, unsigned long long* __restrict__ hist) {
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= total) return;
  int s = 0;
  int64_t k = w;
  while (s < P && k >= rec_count[s]) {
    k -= rec_count[s];
    s++;
  }
  const BatchRec& r = recs[rec_base[s] + k];
  if (r.start < lo || r.start >= hi) return;
  const int32_t gm = model_of_slot[slot_base[s] + r.model];
  atomicAdd(&hist[(int64_t)gm * stride + r.size], 1ull);
}

// p99 (nearest rank, drops as +inf: metrics.py:54-61) per model from the
// sorted keys: rank k = max(1, ceil(0.99 * arrivals)) in the model's segment.
// One block; segments in slot order.
__global__ void __launch_bounds__(1024)
k_stat_p99(const uint64_t* __restrict__ keys, const unsigned long long* __restrict__ arrivals,
           const int32_t* __restrict__ model_of_slot, int32_t M,
           long long* __restrict__ p99 /* -1 = inf, by model id */) {
  __shared__ long long carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int32_t b0 = 0; b0 < M; b0 += 1024) {
    const int32_t slot = b0 + threadIdx.x;
    const int32_t gm = slot < M ? model_of_slot[slot] : 0;
    const int32_t cnt = slot < M ? (int32_t)arrivals[gm] : 0;
    int32_t tot;
    const int32_t ex = block_exclusive_scan(cnt, &tot);
    const long long base = carry;
    if (slot < M) {
      if (cnt == 0) {
        p99[gm] = 0;
      } else {
        long long k = (long long)ceil(0.99 * (double)cnt);
        if (k < 1) k = 1;
        const uint64_t lat = keys[base + ex + k - 1] & kStatInf;
        p99[gm] = lat == kStatInf ? -1 : (long long)lat;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) carry = base + tot;
    __syncthreads();
  }
}


// ------------------------------------------- jittered network (K5') ------
// numpy's Philox4x64-10 (philox.h) is counter based: word j of the engine's
// network stream is word j % 4 of the block for counter j / 4 + 1, and
// Generator.random() is (word >> 11) * 2^-53.  The k-th dispatch of a
// sub-cluster draws ctrl then data (each only if it is a histogram), so its
// delay is computable in parallel from k alone (scheduler.py:197-200).

__device__ __forceinline__ uint64_t philox_word(uint64_t j, uint64_t k0, uint64_t k1) {
  uint64_t c0 = j / 4 + 1, c1 = 0, c2 = 0, c3 = 0;
#pragma unroll
  for (int r = 0; r < 10; r++) {
    if (r) {
      k0 += 0x9E3779B97F4A7C15ull;
      k1 += 0xBB67AE8584CAA73Bull;
    }
    const uint64_t a = 0xD2E7470EE14C6C93ull * c0, ah = __umul64hi(0xD2E7470EE14C6C93ull, c0);
    const uint64_t b = 0xCA5A826395121157ull * c2, bh = __umul64hi(0xCA5A826395121157ull, c2);
    const uint64_t n0 = bh ^ c1 ^ k0, n2 = ah ^ c3 ^ k1;
    c0 = n0;
    c1 = b;
    c2 = n2;
    c3 = a;
  }
  const int w = (int)(j & 3);
  return w == 0 ? c0 : w == 1 ? c1 : w == 2 ? c2 : c3;
}

__device__ __forceinline__ int64_t choice_draw(uint64_t j, uint64_t k0, uint64_t k1,
                                               const int64_t* vals, const double* cdf,
                                               int32_t n) {
  const double u = (double)(philox_word(j, k0, k1) >> 11) * (1.0 / 9007199254740992.0);
  int32_t lo = 0, hi = n;  // searchsorted(cdf, u, 'right')
  while (lo < hi) {
    const int32_t mid = (lo + hi) >> 1;
    if (cdf[mid] <= u) lo = mid + 1; else hi = mid;
  }
  return vals[lo < n ? lo : n - 1];
}

// start = max(exec_at, emitted + ctrl() + data() * b); sort key (gpu, record)
__global__ void k_jitter_start(BatchRec* __restrict__ recs, const int64_t* __restrict__ rec_base,
                               const int64_t* __restrict__ rec_count, int32_t P, int64_t total,
                               const int32_t* __restrict__ gpu_base, int32_t nc, int32_t nd,
                               const int64_t* __restrict__ vals, const double* __restrict__ cdf,
                               int64_t cconst, int64_t dconst, uint64_t k0, uint64_t k1,
                               uint64_t* __restrict__ keys, uint32_t* __restrict__ idx) {
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= total) return;
  int s = 0;
  int64_t k = w;
  while (s < P && k >= rec_count[s]) {
    k -= rec_count[s];
    s++;
  }
  const int64_t ri = rec_base[s] + k;
  BatchRec& r = recs[ri];
  const int per = (nc > 0) + (nd > 0);
  const uint64_t j0 = (uint64_t)k * per;  // k-th dispatch of this sub-cluster
  const int64_t dc = nc > 0 ? choice_draw(j0, k0, k1, vals, cdf, nc) : cconst;
  const int64_t dd = nd > 0 ? choice_draw(j0 + (nc > 0), k0, k1, vals + nc, cdf + nc, nd) : dconst;
  const int64_t actual = dc + dd * r.size;
  const int64_t lat = r.finish - r.start;
  if (r.emitted + actual > r.start) r.start = r.emitted + actual;
  r.finish = r.start + lat;
  keys[w] = ((uint64_t)(gpu_base[s] + r.gpu) << 32) | (uint64_t)ri;
  idx[w] = (uint32_t)ri;
}

// EmulatedGpu.execute (simulator.py:54-62): per GPU, in emission order, a
// start before the previous finish is shifted to it
__global__ void k_serialize(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ idx,
                            int64_t total, BatchRec* __restrict__ recs) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  if (i > 0 && (keys[i - 1] >> 32) == (keys[i] >> 32)) return;  // not a GPU's first
  int64_t busy = 0;
  for (int64_t e = i; e < total && (keys[e] >> 32) == (keys[i] >> 32); e++) {
    BatchRec& r = recs[idx[e]];
    if (r.start < busy) {
      const int64_t sh = busy - r.start;
      r.start += sh;
      r.finish += sh;
    }
    busy = r.finish;
  }
}

// ------------------------------------------- stepped runs (sym_step) -----
// A stepped run keeps the chain's state on the device between calls.  Each
// step rebuilds the sorted layout as, per model, its unresolved arrivals
// (queue positions >= qh) followed by the step's new arrivals, so queue
// positions stay model-relative and the chain resumes where it stopped.

// per slot: new count, kept count and the first kept old position
__global__ void k_step_sizes(const ModelParam* __restrict__ mp,
                             const ModelState* __restrict__ ms,
                             const ModelParam* __restrict__ mpc, int32_t M, int first,
                             int have_chunk, int32_t* __restrict__ slot_meta) {
  const int32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= M) return;
  const int32_t qh = first ? 0 : ms[k].qh;
  const int32_t keep = first ? 0 : mp[k].cnt - qh;
  const int32_t add = have_chunk ? mpc[k].cnt : 0;
  slot_meta[k] = keep + add;                      // newcnt
  slot_meta[2 * (M + 1) + k] = keep;              // keep
  slot_meta[3 * (M + 1) + k] = first ? 0 : mp[k].off + qh;  // oldsrc
}

// newoff = exclusive scan of newcnt (one block); newoff[M] = total
__global__ void __launch_bounds__(1024) k_step_offsets(int32_t* __restrict__ slot_meta,
                                                       int32_t M) {
  __shared__ int32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  int32_t* newcnt = slot_meta;
  int32_t* newoff = slot_meta + (M + 1);
  for (int32_t b0 = 0; b0 < M; b0 += 1024) {
    const int32_t k = b0 + threadIdx.x;
    const int32_t v = k < M ? newcnt[k] : 0;
    int32_t tot;
    const int32_t ex = block_exclusive_scan(v, &tot);
    const int32_t c = carry;
    if (k < M) newoff[k] = c + ex;
    __syncthreads();
    if (threadIdx.x == 0) carry = c + tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) newoff[M] = carry;
}

__device__ __forceinline__ int32_t slot_of_pos(const int32_t* __restrict__ newoff, int32_t M,
                                               int64_t p) {
  int32_t lo = 0, hi = M;  // last slot with newoff <= p (empty slots skipped)
  while (hi - lo > 1) {
    const int32_t mid = (lo + hi) >> 1;
    if (newoff[mid] <= p) lo = mid; else hi = mid;
  }
  while (lo + 1 < M && newoff[lo + 1] <= p) lo++;
  return lo;
}

// The new layout: kept positions copied from the old layout, new ones from
// the chunk's sorted layout with their stream index, shard-stream index and
// A' (the shard's previous arrival may sit in an earlier step).
__global__ void k_step_copy(int64_t bound, const int32_t* __restrict__ slot_meta, int32_t M,
                            int32_t P, const int32_t* __restrict__ slot_base,
                            const ModelParam* __restrict__ mpc,
                            const int64_t* __restrict__ o_tick, const int32_t* __restrict__ o_g,
                            const int32_t* __restrict__ o_i, const int32_t* __restrict__ o_as,
                            const int64_t* __restrict__ c_tick, const int32_t* __restrict__ c_g,
                            const int32_t* __restrict__ c_i, const int64_t* __restrict__ c_sh,
                            const int64_t* __restrict__ c_in_ticks,
                            const int32_t* __restrict__ c_shard_off,
                            const int64_t* __restrict__ shard_meta, int64_t stream_base,
                            int64_t* __restrict__ n_tick, int32_t* __restrict__ n_g,
                            int32_t* __restrict__ n_i, int32_t* __restrict__ n_as,
                            int32_t* __restrict__ flag) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int32_t* newoff = slot_meta + (M + 1);
  if (p >= bound || p >= newoff[M]) return;
  const int32_t k = slot_of_pos(newoff, M, p);
  const int32_t local = (int32_t)(p - newoff[k]);
  const int32_t keep = slot_meta[2 * (M + 1) + k];
  flag[p] = 0;
  if (local < keep) {
    const int32_t src = slot_meta[3 * (M + 1) + k] + local;
    n_tick[p] = o_tick[src];
    n_g[p] = o_g[src];
    n_i[p] = o_i[src];
    n_as[p] = o_as[src];
    return;
  }
  const int32_t c = mpc[k].off + (local - keep);
  const int64_t tick = c_tick[c];
  const int32_t il = c_i[c];  // chunk-local stream index
  int s = 0;
  while (s + 1 < P && slot_base[s + 1] <= k) s++;
  int64_t jl, prev_tick;
  if (P == 1) {  // one shard: the shard stream is the stream
    jl = il;
    prev_tick = il > 0 ? c_in_ticks[il - 1] : shard_meta[P + s];
  } else {
    const int32_t j = c_g[c];
    jl = j - c_shard_off[s];
    prev_tick = jl > 0 ? c_sh[j - 1] : shard_meta[P + s];
  }
  const int64_t gsh = shard_meta[s] + jl;  // the shard's own stream index
  const bool has_prev = jl > 0 || shard_meta[2 * P + s] != 0;
  n_tick[p] = tick;
  n_g[p] = (int32_t)gsh;
  n_i[p] = (int32_t)(stream_base + il);
  n_as[p] = has_prev && prev_tick == tick ? (int32_t)gsh : A_BASE;
}

// Queue positions are model-relative: shift them by the dropped prefix.
__global__ void k_step_rebase(ModelParam* __restrict__ mp, ModelState* __restrict__ ms,
                              const int32_t* __restrict__ slot_meta, int32_t M, int first) {
  const int32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= M) return;
  if (!first) {
    ModelState& st = ms[k];
    const int32_t sh = st.qh;
    st.qbase += sh;
    st.qh -= sh;
    st.qt -= sh;
    if (st.c_head >= sh) st.c_head -= sh;
    if (st.dt_head >= 0) st.dt_head -= sh;
  }
  mp[k].off = slot_meta[(M + 1) + k];
  mp[k].cnt = slot_meta[k];
}

// Every record the step's chains emitted: per-request outputs of its
// members (stream index from the layout), its served flags, and the
// sym_batch appended to the run's batch list.
__global__ void k_step_emit(const BatchRec* __restrict__ recs,
                            const int64_t* __restrict__ rec_base,
                            const int64_t* __restrict__ rec_count, int32_t P,
                            const int64_t* __restrict__ total_p,
                            const int32_t* __restrict__ lay_i,
                            const int32_t* __restrict__ model_of_slot,
                            const int32_t* __restrict__ slot_base,
                            const int32_t* __restrict__ gpu_base, int64_t gcap,
                            int64_t* __restrict__ g_out, int32_t* __restrict__ flag,
                            sym_batch* __restrict__ gbat, unsigned long long* __restrict__ cnt) {
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= *total_p) return;
  int s = 0;
  int64_t k = w;
  while (s < P && k >= rec_count[s]) {
    k -= rec_count[s];
    s++;
  }
  const BatchRec& r = recs[rec_base[s] + k];
  for (int32_t j = 0; j < r.size; j++) {
    const int32_t pos = r.first + j;
    const int64_t gi = lay_i[pos];
    g_out[gi] = r.emitted;
    g_out[gcap + gi] = r.start;
    g_out[2 * gcap + gi] = r.finish;
    g_out[3 * gcap + gi] = r.size;
    g_out[4 * gcap + gi] = 0;  // served; the completion tick decides (collect)
    flag[pos] = 1;
  }
  sym_batch b;
  b.emitted = r.emitted;
  b.start = r.start;
  b.finish = r.finish;
  b.key_t = r.kt;
  b.key_sub = r.ksub;
  b.key_a = r.ka;
  b.model = model_of_slot[slot_base[s] + r.model];
  b.gpu = gpu_base[s] + r.gpu;
  b.size = r.size;
  b.first_index = lay_i[r.first];
  b.shrunk_from = r.shrunk_from;
  gbat[w] = b;
  atomicAdd(&cnt[0], (unsigned long long)r.size);
}

// Positions the step resolved (below the model's queue head) that no batch
// took were dropped.
__global__ void k_step_drops(int64_t bound, const int32_t* __restrict__ slot_meta, int32_t M,
                             const ModelState* __restrict__ ms,
                             const int32_t* __restrict__ lay_i,
                             const int32_t* __restrict__ flag, int64_t gcap,
                             int64_t* __restrict__ g_out, unsigned long long* __restrict__ cnt) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int32_t* newoff = slot_meta + (M + 1);
  if (p >= bound || p >= newoff[M]) return;
  const int32_t k = slot_of_pos(newoff, M, p);
  if (p - newoff[k] < ms[k].qh && !flag[p]) {
    g_out[4 * gcap + lay_i[p]] = 2;  // OUTCOME_DROPPED
    atomicAdd(&cnt[1], 1ull);
  }
}

// Per-shard views of the step's layout, patched on the device (the device
// Shard images carry the chain state from the previous step).
__global__ void k_step_views(Shard* __restrict__ shards, int32_t P,
                             const int32_t* __restrict__ slot_meta, int32_t M,
                             const int32_t* __restrict__ slot_base, const int64_t* s_tick,
                             const int32_t* s_g, const int32_t* s_aself, BatchRec* recs,
                             int64_t* __restrict__ meta) {
  const int s = threadIdx.x;
  if (s >= P) return;
  const int32_t* newoff = slot_meta + (M + 1);
  const int64_t lo = newoff[slot_base[s]], hi = newoff[slot_base[s + 1]];
  Shard& S = shards[s];
  S.s_tick = s_tick;
  S.s_g = s_g;
  S.s_aself = s_aself;
  S.sh_tick = nullptr;
  S.sh_base = 0;
  S.record_trace = 0;
  S.drop_t = nullptr;
  S.drop_ksub = nullptr;
  S.drop_ka = nullptr;
  S.recs = recs + lo + s;  // at most one record per layout position
  S.rec_cap = hi - lo + 1;
  meta[s] = lo + s;        // rec_base
}

// rec_count per shard after the chain, and their total
__global__ void k_step_recmeta(const Shard* __restrict__ shards, int32_t P,
                               int64_t* __restrict__ meta) {
  if (threadIdx.x != 0) return;
  int64_t tot = 0;
  for (int s = 0; s < P; s++) {
    meta[P + 1 + s] = shards[s].n_recs;
    tot += shards[s].n_recs;
  }
  meta[2 * (P + 1)] = tot;
}

// Per-shard stream bookkeeping for the next step's A': arrivals so far,
// the last tick, whether the shard has had any arrival.
__global__ void k_step_shard_update(int64_t* __restrict__ shard_meta, int32_t P, int64_t n,
                                    const int32_t* __restrict__ c_shard_off,
                                    const int64_t* __restrict__ c_in_ticks,
                                    const int64_t* __restrict__ c_sh) {
  const int s = threadIdx.x;
  if (s >= P || n == 0) return;
  const int64_t lo = P == 1 ? 0 : c_shard_off[s], hi = P == 1 ? n : c_shard_off[s + 1];
  if (hi <= lo) return;
  shard_meta[s] += hi - lo;
  shard_meta[P + s] = P == 1 ? c_in_ticks[n - 1] : c_sh[hi - 1];
  shard_meta[2 * P + s] = 1;
}

// k_step_emit / k_step_drops launched over a bound: the real extents live
// on the device (newoff[M], meta total)
// ------------------------------------------------------------ driver ------

int ensure_capacity(Ctx* ctx, int64_t n) {
  if (n > ctx->cap) {
    int64_t c = n + n / 8 + 1024;
    int rc;
    if ((rc = grow(ctx, ctx->d_ticks, c)) || (rc = grow(ctx, ctx->d_model, c)) ||
        (rc = grow(ctx, ctx->d_s_tick, c)) || (rc = grow(ctx, ctx->d_sh_tick, c)) ||
        (rc = grow(ctx, ctx->d_s_g, c)) || (rc = grow(ctx, ctx->d_s_i, c)) ||
        (rc = grow(ctx, ctx->d_bid, c)) ||
        (rc = grow(ctx, ctx->d_sh_i, c)) || (rc = grow(ctx, ctx->d_sh_slot, c)) ||
        (rc = grow(ctx, ctx->d_scan_part,
                   ((c + kChunkR - 1) / kChunkR + 1) * kDigits / kScanItems + 2)) ||
        (rc = grow(ctx, ctx->d_fresh, c)) ||
        (rc = grow(ctx, ctx->d_recs, c + ctx->P)) ||
        (rc = grow(ctx, ctx->d_drop_t, c)) || (rc = grow(ctx, ctx->d_drop_ks, c)) ||
        (rc = grow(ctx, ctx->d_drop_ka, c)) || (rc = grow(ctx, ctx->d_evb, c)) ||
        (rc = grow(ctx, ctx->d_bkA, c)) || (rc = grow(ctx, ctx->d_bkB, c)) ||
        (rc = grow(ctx, ctx->d_tkA, c)) || (rc = grow(ctx, ctx->d_tkB, c)) ||
        (rc = grow(ctx, ctx->d_bvA, c)) || (rc = grow(ctx, ctx->d_bvB, c)) ||
        (rc = grow(ctx, ctx->d_tvA, c)) || (rc = grow(ctx, ctx->d_tvB, c)) ||
        (rc = grow(ctx, ctx->d_ptrA, c)) ||
        (rc = grow(ctx, ctx->d_rhist, ((c + kChunkR - 1) / kChunkR + 1) * kDigits)) ||
        (rc = grow(ctx, ctx->d_closek, c)) ||
        (rc = grow(ctx, ctx->d_nxt, c)) || (rc = grow(ctx, ctx->d_jA, c)) ||
        (rc = grow(ctx, ctx->d_jB, c)) || (rc = grow(ctx, ctx->d_jC, c)) ||
        (rc = grow(ctx, ctx->d_unsure, c)) ||
        (rc = grow(ctx, ctx->d_cp_pos, c / kJump + ctx->M + 2)) ||
        (rc = grow(ctx, ctx->d_cp_model, c / kJump + ctx->M + 2)))
      return rc;
    ctx->cap = c;
  }
  return SYM_OK;
}

int ensure_buckets(Ctx* ctx, int64_t nbk) {
  if (nbk + 1 > ctx->bkt_cap) {
    int rc;
    if ((rc = grow(ctx, ctx->d_bkt, nbk + 1)) ||
        (rc = grow(ctx, ctx->d_bkt_part, (nbk + 1) / kScanItems + 2)))
      return rc;
    ctx->bkt_cap = nbk + 1;
  }
  return SYM_OK;
}

// Opt-in host-side phase timing (SYM_DEBUG_TIMING=1): synchronises the
// stream at each mark and prints the wall time since the previous mark.
struct PhaseClock {
  int mode;  // 0 off, 1 host wall time with syncs, 2 device events (no syncs)
  cudaStream_t st;
  std::chrono::steady_clock::time_point t0, h0;
  std::vector<std::pair<const char*, cudaEvent_t>> evs;
  std::vector<double> host_ms;
  explicit PhaseClock(cudaStream_t s) : st(s) {
    const char* e = getenv("SYM_DEBUG_TIMING");
    mode = e ? atoi(e) : 0;
    t0 = h0 = std::chrono::steady_clock::now();
    if (mode == 2) mark("start");
  }
  void mark(const char* what) {
    if (mode == 1) {
      cudaStreamSynchronize(st);
      auto t = std::chrono::steady_clock::now();
      fprintf(stderr, "[sym] %-14s %9.3f ms\n", what,
              std::chrono::duration<double, std::milli>(t - t0).count());
      t0 = t;
    } else if (mode == 2) {
      cudaEvent_t ev;
      cudaEventCreate(&ev);
      cudaEventRecord(ev, st);
      evs.push_back({what, ev});
      host_ms.push_back(std::chrono::duration<double, std::milli>(
                            std::chrono::steady_clock::now() - h0).count());
    }
  }
  ~PhaseClock() {
    if (mode != 2 || evs.empty()) return;
    cudaEventSynchronize(evs.back().second);
    for (size_t i = 1; i < evs.size(); i++) {
      float ms = 0;
      cudaEventElapsedTime(&ms, evs[i - 1].second, evs[i].second);
      fprintf(stderr, "[sym] %-14s gpu %9.3f ms   host-enqueued at %9.3f ms\n",
              evs[i].first, ms, host_ms[i]);
    }
    for (auto& e : evs) cudaEventDestroy(e.second);
  }
};

// Per-kernel device time (SYM_FLAG_KERNEL_TIMES): CUDA events on the engine
// stream bracket every launch; accumulated per kernel name in the context.
struct KernelTimer {
  Ctx* ctx;
  cudaStream_t st;
  bool on;
  std::vector<std::pair<const char*, std::pair<cudaEvent_t, cudaEvent_t>>> marks;
  void begin(const char* name) {
    if (!on) return;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, st);
    marks.push_back({name, {a, b}});
  }
  void end() {
    if (on) cudaEventRecord(marks.back().second.second, st);
  }
  ~KernelTimer() {
    for (auto& m : marks) {
      cudaEventSynchronize(m.second.second);
      float ms = 0;
      cudaEventElapsedTime(&ms, m.second.first, m.second.second);
      std::string key(m.first);
      key = key.substr(0, key.find('<'));  // one entry per kernel template
      auto& acc = ctx->ktimes[key];
      acc.first += 1;
      acc.second += ms;
      cudaEventDestroy(m.second.first);
      cudaEventDestroy(m.second.second);
    }
  }
};

#define KL(name, ...)          \
  do {                         \
    kt.begin(#name);           \
    ++launches;                \
    name<<<__VA_ARGS__;        \
    kt.end();                  \
  } while (0)

// The previous run's device views die when a new run starts: a failed run
// must not leave sym_window_* / sym_last_batches reading buffers the call
// may have regrown, or caller tensors it no longer vouches for.
void forget_last_run(Ctx* ctx) {
  ctx->has_run = false;
  ctx->last_n = 0;
  ctx->last_ticks = nullptr;
  ctx->last_model = nullptr;
  ctx->last_outcome = ctx->last_start = ctx->last_finish = nullptr;
  ctx->last_nrecs.clear();
  ctx->last_rec_base.clear();
}

void flat_scan(Ctx* ctx, int32_t* a, int64_t len, KernelTimer& kt, int64_t& launches,
               int32_t* part = nullptr) {
  cudaStream_t st = ctx->stream;
  if (!part) part = ctx->d_scan_part;
  const int64_t nparts = (len + kScanItems - 1) / kScanItems;
  KL(k_scan_up, nparts, 1024, 0, st>>>(a, len, part));
  KL(k_scan_mid, 1, 1024, 0, st>>>(part, nparts));
  KL(k_scan_down, nparts, 1024, 0, st>>>(a, len, part));
}

// What the ingest reads back for the host (one synchronisation).
struct IngestInfo {
  int64_t last_tick = 0;
  std::vector<int32_t> shard_off;   // [P+1] first shard-stream index per shard
  std::vector<ModelParam> mp;       // per-slot off/cnt of the sorted layout
};

// K1: stable partition of n time-ordered arrivals into the (shard, model)-
// sorted layout (ctx->d_s_tick, d_s_g, d_s_i, d_sh_tick;
// per-slot off/cnt into mp_out).  Validates model ids (EPROTO) and the
// time order (EINVAL) on the device.
// One stable partition (k_part_count, flat_scan, k_part_binoff, k_part).
// Mode 2 partitions each sub-cluster stream by its own slots (tiles within
// one sub-cluster, local bins: Bmax = the largest sub-cluster's model count).
template <int kMode>
int partition(Ctx* ctx, const int64_t* tick_in, const int32_t* key, const int32_t* aux_in,
              int64_t n, int32_t B, ModelParam* mp_out, int32_t* shard_off_out,
              int64_t* out_tick, int32_t* out_idx, int32_t* out_aux, int32_t* inv_out,
              KernelTimer& kt, int64_t& launches) {
  cudaStream_t st = ctx->stream;
  const int32_t P = ctx->P;
  const int64_t W = (n + kTileI - 1) / kTileI;
  int32_t Bmax = B;
  int64_t grid = W, hlen = W * B;
  int64_t* seg = ctx->d_seg;
  if (kMode == 2) {
    Bmax = 1;
    for (int s = 0; s < P; s++) Bmax = std::max(Bmax, ctx->slot_base[s + 1] - ctx->slot_base[s]);
    grid = W + P;              // >= sum over sub-clusters of their tiles
    hlen = (int64_t)Bmax * (W + P);
    KL(k_part_seg, 1, 32, 0, st>>>(ctx->d_bins + (ctx->M + P) + 1, ctx->d_slot_base, P, seg));
  }
  if (hlen + 1 > ctx->hist_cap) {
    int rc;
    if ((rc = grow(ctx, ctx->d_hist, hlen + 1)) ||
        (rc = grow(ctx, ctx->d_hist_part, (hlen + 1) / kScanItems + 2)))
      return rc;
    ctx->hist_cap = hlen + 1;
  }
  if (W > 0) {
    if (kMode == 2) CK(cudaMemsetAsync(ctx->d_hist, 0, sizeof(int32_t) * hlen, st));
    KL(k_part_count<kMode>, grid, 256, sizeof(int32_t) * Bmax, st>>>(
        key, n, ctx->M, ctx->d_shard_of_model, B, ctx->d_hist, W, seg, P, ctx->d_err));
    flat_scan(ctx, ctx->d_hist, hlen, kt, launches, ctx->d_hist_part);
  }
  KL(k_part_binoff<kMode>, nblk(B, 128), 128, 0, st>>>(ctx->d_hist, W, B, n, seg, P, mp_out,
                                                        shard_off_out));
  if (W > 0)
    KL(k_part<kMode>, grid, 32 * kTileWarps, part_smem(Bmax), st>>>(
        tick_in, key, aux_in, n, ctx->M, ctx->d_shard_of_model, ctx->d_slot_of_model, Bmax,
        ctx->d_hist, W, seg, P, out_tick, out_idx, out_aux, inv_out, ctx->d_err));
  CK(cudaGetLastError());
  return SYM_OK;
}

int ingest(Ctx* ctx, const int64_t* d_ticks, const int32_t* d_model, int64_t n,
           ModelParam* mp_out, KernelTimer& kt, int64_t& launches, IngestInfo& info,
           sym_result* out) {
  cudaStream_t st = ctx->stream;
  const int32_t M = ctx->M, P = ctx->P;
  const int32_t big[2] = {INT32_MAX, INT32_MAX};
  CK(cudaMemcpyAsync(ctx->d_err, big, sizeof big, cudaMemcpyHostToDevice, st));
  int32_t* shard_off = ctx->d_bins + (M + P) + 1;
  int rc;
  if (P == 1) {
    const int32_t zn[2] = {0, (int32_t)n};
    CK(cudaMemcpyAsync(shard_off, zn, sizeof zn, cudaMemcpyHostToDevice, st));
    if ((rc = partition<0>(ctx, d_ticks, d_model, nullptr, n, M, mp_out, nullptr,
                           ctx->d_s_tick, ctx->d_s_i, nullptr, nullptr, kt, launches)))
      return rc;
  } else {
    // by sub-cluster (the sub-cluster streams), then each of them by model
    if ((rc = partition<1>(ctx, d_ticks, d_model, nullptr, n, P, nullptr, shard_off,
                           ctx->d_sh_tick, ctx->d_sh_i, ctx->d_sh_slot, nullptr, kt,
                           launches)) ||
        (rc = partition<2>(ctx, ctx->d_sh_tick, ctx->d_sh_slot, ctx->d_sh_i, n, M, mp_out,
                           nullptr, ctx->d_s_tick, ctx->d_s_g, ctx->d_s_i, nullptr, kt,
                           launches)))
      return rc;
  }
  CK(cudaGetLastError());
  int32_t herr2[2] = {INT32_MAX, INT32_MAX};
  info.last_tick = 0;
  info.shard_off.assign(P + 1, 0);
  CK(cudaMemcpyAsync(herr2, ctx->d_err, sizeof herr2, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(info.shard_off.data(), shard_off, sizeof(int32_t) * (P + 1),
                     cudaMemcpyDeviceToHost, st));
  if (n > 0)
    CK(cudaMemcpyAsync(&info.last_tick, d_ticks + (n - 1), sizeof info.last_tick,
                       cudaMemcpyDeviceToHost, st));
  // per-model arrival counts ride on the same readback
  info.mp.resize(M);
  CK(cudaMemcpyAsync(info.mp.data(), mp_out, sizeof(ModelParam) * M,
                     cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (herr2[0] != INT32_MAX) {
    out->err_index = herr2[0];
    ctx->err = "request for unknown model";
    return SYM_EPROTO;
  }
  if (herr2[1] != INT32_MAX) {
    out->err_index = herr2[1];
    ctx->err = "arrival ticks must be non-decreasing";
    return SYM_EINVAL;
  }
  return SYM_OK;
}

int run_device(Ctx* ctx, const int64_t* d_ticks, const int32_t* d_model,
               int64_t n, uint32_t flags, sym_result* out, bool outs_on_device) {
  cudaStream_t st = ctx->stream;
  int64_t launches = 0;
  PhaseClock pc(st);
  KernelTimer kt{ctx, st, (flags & SYM_FLAG_KERNEL_TIMES) != 0, {}};
  auto flat_scan = [&](int32_t* a, int64_t len) { ::flat_scan(ctx, a, len, kt, launches); };
  const int32_t M = ctx->M, P = ctx->P;
  const int B = M + P;
  const bool trace = flags & SYM_FLAG_TRACE;
  const bool check = flags & SYM_FLAG_CHECK_INVARIANTS;
  const bool use_fresh = !trace && !(flags & SYM_FLAG_NO_FRESH);
  forget_last_run(ctx);
  ctx->step_active = false;  // a whole run reuses the chain arrays
  int rc;
  if ((rc = ensure_capacity(ctx, n))) return rc;
  CK(cudaEventRecord(ctx->ev[0], st));
  // ---- K1 ingest
  IngestInfo info;
  if ((rc = ingest(ctx, d_ticks, d_model, n, ctx->d_mp, kt, launches, info, out))) return rc;
  const int64_t last_tick = info.last_tick;
  const std::vector<int32_t>& shard_off = info.shard_off;
  const std::vector<ModelParam>& mp = info.mp;
  // every event tick and finish time of a validated run is below the last
  // arrival + SLO; the bound is generous and checked (FP_CAPACITY)
  int tick_bits = 1;
  {
    const uint64_t bound = (uint64_t)(last_tick > 0 ? last_tick : 0) +
                           2 * (uint64_t)ctx->max_slo + (uint64_t)ctx->max_lat + 1;
    while (tick_bits < 62 && (uint64_t(1) << tick_bits) <= bound) tick_bits++;
  }
  CK(cudaGetLastError());
  pc.mark("ingest");
  CK(cudaEventRecord(ctx->ev[1], st));
  // ---- per-shard views
  for (int s = 0; s < P; s++) {
    Shard& S = ctx->shards[s];
    S.s_tick = ctx->d_s_tick;
    S.s_g = P > 1 ? ctx->d_s_g : ctx->d_s_i;  // one shard: j == i
    S.sh_tick = P > 1 ? ctx->d_sh_tick : d_ticks;
    S.sh_base = shard_off[s];
    S.s_aself = nullptr;
    S.record_trace = trace ? 1 : 0;
    S.check = check ? 1 : 0;
    S.inject = check && (flags & SYM_FLAG_INJECT_FAULT) ? 9 : -1;
    S.drop_t = ctx->d_drop_t;
    S.drop_ksub = ctx->d_drop_ks;
    S.drop_ka = ctx->d_drop_ka;
  }
  // record capacity per shard: its arrival count (+1)
  std::vector<int64_t> rec_base(P + 1, 0);
  for (int s = 0; s < P; s++) {
    int64_t cnt = 0;
    for (int k = ctx->slot_base[s]; k < ctx->slot_base[s + 1]; k++)
      cnt += mp[k].cnt;
    rec_base[s + 1] = rec_base[s] + cnt + 1;
    ctx->shards[s].recs = ctx->d_recs + rec_base[s];
    ctx->shards[s].rec_cap = cnt + 1;
  }
  CK(cudaMemcpyAsync(ctx->d_shards, ctx->shards.data(), sizeof(Shard) * P,
                     cudaMemcpyHostToDevice, st));
  if (trace && n > 0)
    KL(k_fill64, nblk(n, 256), 256, 0, st>>>(ctx->d_drop_t, n, -1));
  // ---- K2 fresh-start pre-scan: chain pointers for the fast path, full
  // records (needed only by the sequential chain) otherwise
  // per-event invariants need the event-by-event chain (no fast path)
  const bool fast = use_fresh && !check && !(flags & SYM_FLAG_NO_FAST) && n > 0;
  bool have_fresh = false;
  if (fast) {
    CK(cudaMemsetAsync(ctx->d_unsure_n, 0, sizeof(int32_t), st));
    const int64_t tiles = (n + kNxtTile - 1) / kNxtTile;
    const int64_t want = (tiles + kNxtTmaWarps - 1) / kNxtTmaWarps;
    KL(k_nxt_tma, (unsigned)std::min<int64_t>(want, (int64_t)ctx->n_sm * kNxtTmaBlocksPerSm),
       32 * kNxtTmaWarps, kNxtTmaSmem, st>>>(
           ctx->d_s_tick, ctx->d_shards, ctx->d_slot_base, ctx->d_mp, P, M, (int32_t)n,
           ctx->d_nxt, ctx->d_closek, ctx->d_unsure, ctx->d_unsure_n));
    KL(k_nxt_general, 148 * 4, 256, 0, st>>>(ctx->d_shards, ctx->d_slot_base, ctx->d_mp, P,
                                             ctx->d_unsure, ctx->d_unsure_n, ctx->d_nxt,
                                             ctx->d_closek));
  } else if (use_fresh && n > 0) {
    KL(k_fresh, nblk(n, 256), 256, 0, st>>>(ctx->d_shards, ctx->d_slot_base,
                                          ctx->d_mp, P, n, ctx->d_fresh, nullptr));
    have_fresh = true;
  }
  CK(cudaGetLastError());
  pc.mark("fresh");
  CK(cudaEventRecord(ctx->ev[2], st));
  // ---- K3 parallel fast path (validated regime), K4 chain for the rest
  std::vector<uint32_t> fail(P, 0);
  std::vector<int64_t> sbase(P + 1, 0);
  std::vector<int64_t> mdrops(M, 0);
  if (fast) {
    CK(cudaMemsetAsync(ctx->d_fail, 0, sizeof(uint32_t) * P, st));
    CK(cudaMemsetAsync(ctx->d_mdrops, 0, sizeof(int64_t) * M, st));
    const int64_t ncp = n / kJump + M + 2;
    CK(cudaMemsetAsync(ctx->d_cp_model, 0xff, sizeof(int32_t) * ncp, st));
    // J_4, J_16, J_64 (kept in jC), J_256 by quadrupling the chain pointer
    KL(k_jump4, nblk(n, 256 * kJumpIlp), 256, 0, st>>>(ctx->d_nxt, ctx->d_jA, n));
    KL(k_jump4, nblk(n, 256 * kJumpIlp), 256, 0, st>>>(ctx->d_jA, ctx->d_jB, n));
    KL(k_jump4, nblk(n, 256 * kJumpIlp), 256, 0, st>>>(ctx->d_jB, ctx->d_jC, n));
    KL(k_jump4, nblk(n, 256 * kJumpIlp), 256, 0, st>>>(ctx->d_jC, ctx->d_jA, n));
    KL(k_walk, nblk(M, 64), 64, 0, st>>>(ctx->d_mp, M, ctx->d_nxt, ctx->d_jB, ctx->d_jC,
                                         ctx->d_jA,
                                         ctx->d_cp_pos, ctx->d_cp_model, ctx->d_nb,
                                         ctx->d_special));
    KL(k_walk_fill, nblk(ncp, 256), 256, 0, st>>>(ctx->d_cp_pos, ctx->d_cp_model, ncp,
                                                 ctx->d_jC));
    KL(k_cp_scan, 1, 1024, 0, st>>>(ctx->d_mp, M, ctx->d_nb, ctx->d_special, ctx->d_cpoff));
    // J_256 (jA) is dead after k_walk / k_walk_fill: it holds the batch starts
    KL(k_walk_expand, (unsigned)std::min<int64_t>(nblk(ncp, kExpandWarps), (int64_t)ctx->n_sm * 3),
       32 * kExpandWarps, kExpandSmem, st>>>(ctx->d_cp_pos, ctx->d_cpoff, M, ctx->d_mp,
                                             ctx->d_slot_base, P, ctx->d_nxt, ctx->d_jB,
                                             ctx->d_shards, ctx->d_jA,
                                             (unsigned long long*)ctx->d_mdrops));
    // models whose chain needs the general (non-draining) evolution
    KL(k_evolve, nblk(M, 64), 64, 0, st>>>(ctx->d_shards, ctx->d_slot_base, P, M,
                                                     nullptr, ctx->d_evb, ctx->d_nb,
                                                     ctx->d_mdrops, ctx->d_fail,
                                                     ctx->d_special));
  pc.mark("evolve");
    KL(k_nb_scan, 1, 1024, 0, st>>>(ctx->d_nb, M, P, ctx->d_slot_base, ctx->d_bbase,
                                            ctx->d_sbase));
    CK(cudaMemcpyAsync(sbase.data(), ctx->d_sbase, sizeof(int64_t) * (P + 1),
                       cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const int64_t nt = sbase[P];
    if (nt > 0) {
      KL(k_chain_recs, nblk(nt, 256), 256, 0, st>>>(
          ctx->d_shards, ctx->d_slot_base, P, M, ctx->d_mp, ctx->d_nb, ctx->d_bbase,
          ctx->d_special, nt, ctx->d_evb, (unsigned long long*)ctx->d_mdrops, ctx->d_closek,
          ctx->d_jA, ctx->d_bkA, ctx->d_bvA, ctx->d_fail, tick_bits));

      // key = (shard << tick_bits) | tick: bits in use
      int bits = tick_bits;
      while ((1 << (bits - tick_bits)) < P) bits++;
  pc.mark("batch_keys");
      // bucket sorts: ~1 key per bucket of 2^shift ns over the (shard|tick) range
      int shift = 0;
      while ((int64_t(1) << (bits - shift)) > 2 * nt && shift < bits) shift++;
      const int64_t nbk = ((int64_t)P << tick_bits) >> shift;
      if ((rc = ensure_buckets(ctx, nbk))) return rc;
      auto bucket_sort = [&](uint64_t*& ka, uint32_t*& va, uint64_t*& kb, uint32_t*& vb,
                             bool batches) {
        CK(cudaMemsetAsync(ctx->d_bkt, 0, sizeof(int32_t) * (nbk + 1), st));
        KL(k_bkt_count, nblk(nt, 256), 256, 0, st>>>(ka, nt, shift, ctx->d_bkt));
        ::flat_scan(ctx, ctx->d_bkt, nbk, kt, launches, ctx->d_bkt_part);
        KL(k_bkt_scatter, nblk(nt, 256), 256, 0, st>>>(ka, va, nt, shift, ctx->d_bkt, kb, vb));
        if (batches)
          KL(k_bkt_sort<true>, nblk(nbk, 256), 256, 0, st>>>(ctx->d_bkt, nbk, kb, vb,
                                                             ctx->d_evb));
        else
          KL(k_bkt_sort<false>, nblk(nbk, 256), 256, 0, st>>>(ctx->d_bkt, nbk, kb, vb,
                                                              ctx->d_evb));
        std::swap(ka, kb);
        std::swap(va, vb);
        return SYM_OK;
      };
      if ((rc = bucket_sort(ctx->d_bkA, ctx->d_bvA, ctx->d_bkB, ctx->d_bvB, true))) return rc;
  pc.mark("sort_batches");
      KL(k_token_keys, nblk(nt, 256), 256, 0, st>>>(
          ctx->d_bvA, nt, ctx->d_bkA, ctx->d_evb, ctx->d_sbase, ctx->d_tkA, ctx->d_tvA,
          ctx->d_fail, tick_bits));
  pc.mark("token_keys");
      if ((rc = bucket_sort(ctx->d_tkA, ctx->d_tvA, ctx->d_tkB, ctx->d_tvB, false))) return rc;
  pc.mark("sort_tokens");
      {
        int bps = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_match_coop, 256, 0);
        int nsm = 0;
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, ctx->device);
        const int64_t want = (nt + 255) / 256;
        dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)bps * nsm)));
        int64_t a_nt = nt;
        int a_tb = tick_bits;
        CK(cudaMemsetAsync(ctx->d_tie_cnt, 0, sizeof(int32_t) * P, st));
        CK(cudaMemsetAsync(ctx->d_changed, 0, sizeof(int32_t) * 4, st));  // [0]: overflow
        void* args[] = {&ctx->d_bkA, &ctx->d_bvA, &a_nt, &ctx->d_sbase, &ctx->d_shards,
                        &ctx->d_tkA, &ctx->d_tvA, &ctx->d_ptrA, &ctx->d_changed, &a_tb,
                        &ctx->d_tie_cnt, &ctx->d_tie_list};
        kt.begin("k_match_coop");
        ++launches;
        CK(cudaLaunchCooperativeKernel((void*)k_match_coop, grid, dim3(256), args, 0, st));
        kt.end();
      }
      KL(k_tie_fix, P, kTieThreads, 0, st>>>(ctx->d_sbase, ctx->d_shards, P, ctx->d_tkA,
                                              ctx->d_tvA, ctx->d_ptrA, ctx->d_tie_cnt,
                                              ctx->d_tie_list, ctx->d_tie_eff, ctx->d_tie_sig,
                                              ctx->d_tie_mask, ctx->d_changed));
      {  // tie-heavy runs only (returns at once otherwise)
        int bps = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_match_iter, 256, 0);
        const int64_t want = (nt + 255) / 256;
        dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)bps * ctx->n_sm)));
        int64_t a_nt = nt;
        int a_tb = tick_bits, a_P = P;
        void* args[] = {&ctx->d_bkA, &ctx->d_bvA, &a_nt, &ctx->d_sbase, &ctx->d_shards,
                        &ctx->d_tkA, &ctx->d_tvA, &ctx->d_ptrA, &ctx->d_changed, &a_tb,
                        &ctx->d_tie_cnt, &a_P};
        kt.begin("k_match_iter");
        ++launches;
        CK(cudaLaunchCooperativeKernel((void*)k_match_iter, grid, dim3(256), args, 0, st));
        kt.end();
      }
  pc.mark("match_loop");
      int64_t* d_rb = ctx->d_meta + 2 * (P + 1);
      CK(cudaMemcpyAsync(d_rb, rec_base.data(), sizeof(int64_t) * (P + 1),
                         cudaMemcpyHostToDevice, st));
      KL(k_fast_emit, nblk(nt, 256), 256, 0, st>>>(
          ctx->d_bkA, ctx->d_bvA, nt, ctx->d_evb, ctx->d_sbase, ctx->d_tkA, ctx->d_tvA,
          ctx->d_ptrA, ctx->d_tie_cnt, ctx->d_tie_eff, ctx->d_tie_sig, ctx->d_tie_mask, d_rb,
          ctx->d_shards,
          ctx->d_recs, ctx->d_fail, tick_bits));
    }
    CK(cudaMemcpyAsync(fail.data(), ctx->d_fail, sizeof(uint32_t) * P,
                       cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(mdrops.data(), ctx->d_mdrops, sizeof(int64_t) * M,
                       cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  }
  pc.mark("fast_tail");
  CK(cudaEventRecord(ctx->ev[5], st));
  std::vector<int32_t> skip(P, 0);
  int32_t n_chain = 0;
  for (int s = 0; s < P; s++) {
    skip[s] = fast && fail[s] == 0;
    n_chain += !skip[s];
    if (skip[s]) {  // counters the chain would have produced
      Shard& S = ctx->shards[s];
      const int64_t nbs = sbase[s + 1] - sbase[s];
      S.n_recs = nbs;
      S.ops = 3 * nbs;
      S.handler_ops_max = nbs > 0 ? 3 : 0;
      S.registrations = S.evictions = 0;
      S.chain_events = nbs;
      S.absorbed = rec_base[s + 1] - rec_base[s] - 1;
      S.fresh_adoptions = 0;
      S.error = ERR_NONE;
    }
  }
  ctx->last_fast_fail = fail;
  if (n_chain > 0) {
    if (use_fresh && !have_fresh && n > 0) {  // adoption records for the chain
      KL(k_fresh, nblk(n, 256), 256, 0, st>>>(ctx->d_shards, ctx->d_slot_base, ctx->d_mp, P,
                                              n, ctx->d_fresh, nullptr));
      have_fresh = true;
    }
    CK(cudaMemcpyAsync(ctx->d_shards, ctx->shards.data(), sizeof(Shard) * P,
                       cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(ctx->d_skip, skip.data(), sizeof(int32_t) * P,
                       cudaMemcpyHostToDevice, st));
    KL(k_chain, P, 32, ctx->chain_smem, st>>>(
        ctx->d_shards, use_fresh ? ctx->d_fresh : nullptr, ctx->d_dirty,
        ctx->d_slot_base, ctx->chain_smem, ctx->d_skip, kChainWhole, INT64_MAX));
  } else {
    CK(cudaMemcpyAsync(ctx->d_shards, ctx->shards.data(), sizeof(Shard) * P,
                       cudaMemcpyHostToDevice, st));
  }
  CK(cudaGetLastError());
  pc.mark("chain");
  CK(cudaEventRecord(ctx->ev[3], st));
  std::vector<ModelState> ms(M);
  if (n_chain > 0) {  // otherwise the host copy is current and ms is unused
    CK(cudaMemcpyAsync(ctx->shards.data(), ctx->d_shards, sizeof(Shard) * P,
                       cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(ms.data(), ctx->d_ms, sizeof(ModelState) * M,
                       cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  }
  int64_t total = 0;
  std::vector<int64_t> rec_count(P);
  for (int s = 0; s < P; s++) {
    const Shard& S = ctx->shards[s];
    if (S.error) {
      static const char* what[] = {"", "record overflow", "bad chain state",
                                   "conservation broken (arrivals != dispatched + dropped + "
                                   "queued)",
                                   "gpu state machine broken (grant outstanding across an "
                                   "event, or free index out of sync)",
                                   "rank candidate indices out of sync",
                                   "candidate infeasible (exec_at > latest or misses its head "
                                   "deadline)"};
      ctx->err = std::string(S.error >= 1 && S.error <= 6 ? what[S.error] : "chain error") +
                 " in sub-cluster " + std::to_string(s) + " after chain event " +
                 std::to_string(S.chain_events);
      return SYM_EINVARIANT;
    }
    rec_count[s] = S.n_recs;
    total += S.n_recs;
  }
  // ---- K5 outputs
  int64_t* d_meta = ctx->d_meta;  // rec_base[P] + rec_count[P]
  CK(cudaMemcpyAsync(d_meta, rec_base.data(), sizeof(int64_t) * P,
                     cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_meta + P + 1, rec_count.data(), sizeof(int64_t) * P,
                     cudaMemcpyHostToDevice, st));
  if (ctx->jitter && total > 0) {
    if (total > ctx->cap) {
      ctx->err = "jitter scratch too small";
      return SYM_EINVAL;
    }
    const int32_t* d_gpu_base = ctx->d_bins + B + P + 2 + M;
    KL(k_jitter_start, nblk(total, 256), 256, 0, st>>>(
        ctx->d_recs, d_meta, d_meta + P + 1, P, total, d_gpu_base, ctx->net_ctrl_n,
        ctx->net_data_n, ctx->d_net_vals, ctx->d_net_cdf, ctx->net_ctrl_const,
        ctx->net_data_const, ctx->net_key[0], ctx->net_key[1], ctx->d_tkA, ctx->d_tvA));
    int bits = 32;
    while ((int64_t(1) << (bits - 32)) < ctx->G) bits++;
    const int64_t Wj = (total + kChunkR - 1) / kChunkR;
    uint64_t* ka = ctx->d_tkA; uint64_t* kb = ctx->d_tkB;
    uint32_t* va = ctx->d_tvA; uint32_t* vb = ctx->d_tvB;
    for (int shift = 32; shift < bits; shift += kDigitBits) {  // records already in order
      KL(k_rhist, nblk(Wj, kRadixWarps), 32 * kRadixWarps, 0, st>>>(ka, total, shift,
                                                                      ctx->d_rhist, Wj));
      flat_scan(ctx->d_rhist, Wj * kDigits);
      KL(k_rscatter, nblk(Wj, kRadixWarps), 32 * kRadixWarps, 0, st>>>(
          ka, va, total, shift, ctx->d_rhist, Wj, kb, vb));
      std::swap(ka, kb);
      std::swap(va, vb);
    }
    KL(k_serialize, nblk(total, 256), 256, 0, st>>>(ka, va, total, ctx->d_recs));
  }
  const bool expand = !(flags & SYM_FLAG_NO_EXPAND) && out->req_dispatch;
  if (expand && n > 0) {
    // every request starts as "no batch" (dropped); k_bid stamps the members
    CK(cudaMemsetAsync(ctx->d_bid, 0xff, sizeof(int32_t) * n, st));
    int64_t most = 0;
    for (int s2 = 0; s2 < P; s2++) most = std::max<int64_t>(most, rec_count[s2]);
    if (total > 0)
      KL(k_bid, nblk(most * P, 256), 256, 0, st>>>(ctx->d_recs, d_meta, d_meta + P + 1, P,
                                                    most * P, ctx->d_s_i, ctx->d_bid));
    auto al16 = [](const void* q) { return ((uintptr_t)q & 15u) == 0; };
    const bool vec = al16(d_ticks) && ((uintptr_t)d_model & 7u) == 0 &&
                     al16(out->req_dispatch) && al16(out->req_start) &&
                     al16(out->req_finish) && al16(out->req_batch) && al16(out->req_outcome) &&
                     al16(out->req_arrival) && al16(out->req_deadline) && al16(out->req_model);
    if (vec)
      KL(k_out<true>, nblk((n + 1) / 2, 256), 256, 0, st>>>(
          n, ctx->d_bid, ctx->d_recs, d_ticks,
          d_model, ctx->d_slo_model, out->req_dispatch, out->req_start, out->req_finish,
          out->req_batch, out->req_outcome, out->req_arrival, out->req_deadline, out->req_model));
    else
      KL(k_out<false>, nblk((n + 1) / 2, 256), 256, 0, st>>>(
          n, ctx->d_bid, ctx->d_recs, d_ticks,
          d_model, ctx->d_slo_model, out->req_dispatch, out->req_start, out->req_finish,
          out->req_batch, out->req_outcome, out->req_arrival, out->req_deadline, out->req_model));
  }
  if (trace && out->drop_t && n > 0)
    KL(k_drop_out, nblk(n, 256), 256, 0, st>>>(
        n, ctx->d_s_i, ctx->d_drop_t, ctx->d_drop_ks, ctx->d_drop_ka,
        out->drop_t, out->drop_key_sub, out->drop_key_a));
  if (out->batches && total > 0) {
    if (total > out->batch_cap) {
      ctx->err = "batch buffer too small";
      return SYM_EINVAL;
    }
    KL(k_copy_batches, nblk(total, 256), 256, 0, st>>>(
        ctx->d_recs, d_meta, d_meta + P + 1, P, ctx->d_s_i,
        ctx->d_bins + B + P + 2, ctx->d_slot_base, ctx->d_bins + B + P + 2 + M,
        total, out->batches));
  }
  CK(cudaGetLastError());
  pc.mark("outputs");
  CK(cudaEventRecord(ctx->ev[4], st));
  CK(cudaStreamSynchronize(st));
  (void)outs_on_device;
  // ---- counters
  out->n_batches = total;
  out->launches = launches;
  out->drops = out->completions = out->late = 0;
  out->ops = out->evictions = out->registrations = out->handler_ops_max = 0;
  out->chain_events = out->absorbed_arrivals = out->fresh_adoptions = 0;
  for (int s = 0; s < P; s++) {
    const Shard& S = ctx->shards[s];
    out->ops += S.ops;
    out->evictions += S.evictions;
    out->registrations += S.registrations;
    if (S.handler_ops_max > out->handler_ops_max)
      out->handler_ops_max = S.handler_ops_max;
    out->chain_events += S.chain_events;
    out->absorbed_arrivals += S.absorbed;
    out->fresh_adoptions += S.fresh_adoptions;
  }
  for (int s = 0; s < P; s++)
    for (int k = ctx->slot_base[s]; k < ctx->slot_base[s + 1]; k++)
      out->drops += skip[s] ? mdrops[k] : ms[k].drops;
  out->fast_shards = P - n_chain;
  out->fast_fail_mask = 0;
  for (int s = 0; s < P; s++) out->fast_fail_mask |= fail[s];
  out->completions = n - out->drops;  // jitterless: nothing is late
  float t;
  cudaEventElapsedTime(&t, ctx->ev[0], ctx->ev[1]);
  out->ms_ingest = t;
  cudaEventElapsedTime(&t, ctx->ev[1], ctx->ev[2]);
  out->ms_fresh = t;
  cudaEventElapsedTime(&t, ctx->ev[2], ctx->ev[5]);
  out->ms_fast = t;
  cudaEventElapsedTime(&t, ctx->ev[5], ctx->ev[3]);
  out->ms_chain = t;
  cudaEventElapsedTime(&t, ctx->ev[3], ctx->ev[4]);
  out->ms_expand = t;
  cudaEventElapsedTime(&t, ctx->ev[0], ctx->ev[4]);
  out->ms_total = t;
  ctx->last_n = n;
  ctx->last_ticks = d_ticks;
  ctx->last_model = d_model;
  ctx->last_outcome = expand ? out->req_outcome : nullptr;
  ctx->last_start = expand ? out->req_start : nullptr;
  ctx->last_finish = expand ? out->req_finish : nullptr;
  ctx->last_nrecs = rec_count;
  ctx->last_rec_base = rec_base;
  ctx->has_run = true;
  return SYM_OK;
}

// Realloc keeping the first `keep` elements (stream-ordered, no sync).
template <class T>
int grow_keep_named(Ctx* ctx, T*& p, int64_t keep, int64_t count, const char* name) {
  T* q = nullptr;
  CK(dmalloc(ctx, (void**)&q, sizeof(T) * (size_t)(count > 0 ? count : 1), ctx->stream, name));
  if (p && keep > 0)
    CK(cudaMemcpyAsync(q, p, sizeof(T) * (size_t)keep, cudaMemcpyDeviceToDevice, ctx->stream));
  dfree(ctx, p, ctx->stream);
  p = q;
  return SYM_OK;
}
#define grow_keep(ctx, p, keep, count) grow_keep_named(ctx, p, keep, count, #p)

void step_reset(Ctx* ctx) {
  forget_last_run(ctx);
  ctx->step_active = true;
  ctx->step_first = true;
  ctx->step_n = 0;
  ctx->step_until = INT64_MIN;
  ctx->step_served = ctx->step_drops = 0;
  ctx->lay_n = 0;
  ctx->gbat_n = 0;
}

// One step of a stepped run: the chunk (device buffers, stream order, ticks
// within [previous until, until]) joins the sorted layout and the chain runs
// every event with tick <= until.  Two synchronisations: the ingest's
// validation readback and the step's counters.
int step_device(Ctx* ctx, const int64_t* d_ticks, const int32_t* d_model, int64_t n,
                int64_t until, uint32_t flags, sym_result* out) {
  cudaStream_t st = ctx->stream;
  int64_t launches = 0;
  KernelTimer kt{ctx, st, (flags & SYM_FLAG_KERNEL_TIMES) != 0, {}};
  const int32_t M = ctx->M, P = ctx->P;
  const int B = M + P;
  const bool first = ctx->step_first;
  int rc;
  CK(cudaEventRecord(ctx->ev[0], st));
  const int64_t bound = ctx->lay_n + n;  // the new layout's size is at most this
  if ((rc = ensure_capacity(ctx, std::max<int64_t>(n, bound)))) return rc;
  if (ctx->step_n + n > ctx->g_cap) {
    const int64_t c = std::max<int64_t>(2 * ctx->g_cap, ctx->step_n + n + 1024);
    int64_t* o = nullptr;
    CK(dmalloc(ctx, (void**)&o, sizeof(int64_t) * 5 * (size_t)c, st, "d_g_out"));
    for (int k = 0; k < 5 && ctx->step_n > 0; k++)
      CK(cudaMemcpyAsync(o + k * c, ctx->d_g_out + k * ctx->g_cap,
                         sizeof(int64_t) * ctx->step_n, cudaMemcpyDeviceToDevice, st));
    dfree(ctx, ctx->d_g_out, st);
    ctx->d_g_out = o;
    if ((rc = grow_keep(ctx, ctx->d_g_ticks, ctx->step_n, c)) ||
        (rc = grow_keep(ctx, ctx->d_g_model, ctx->step_n, c)))
      return rc;
    ctx->g_cap = c;
  }
  if (bound + 1 > ctx->lay_cap) {
    const int64_t c = std::max<int64_t>(2 * ctx->lay_cap, bound + 1024);
    const int64_t k = ctx->lay_n;
    for (int b = 0; b < 2; b++) {
      const int64_t kb = b == ctx->cur ? k : 0;
      if ((rc = grow_keep(ctx, ctx->d_lay_tick[b], kb, c)) ||
          (rc = grow_keep(ctx, ctx->d_lay_g[b], kb, c)) ||
          (rc = grow_keep(ctx, ctx->d_lay_i[b], kb, c)) ||
          (rc = grow_keep(ctx, ctx->d_lay_aself[b], kb, c)))
        return rc;
    }
    if ((rc = grow(ctx, ctx->d_lay_flag, c))) return rc;
    ctx->lay_cap = c;
  }
  if (ctx->gbat_n + bound + P > ctx->gbat_cap) {
    const int64_t c = std::max<int64_t>(2 * ctx->gbat_cap, ctx->gbat_n + bound + P + 1024);
    if ((rc = grow_keep(ctx, ctx->d_gbat, ctx->gbat_n, c))) return rc;
    ctx->gbat_cap = c;
  }
  // ---- the chunk: ingest (validates ids and time order before any state
  // changes), stream copy, outputs unresolved
  IngestInfo info;
  if (n > 0) {
    if ((rc = ingest(ctx, d_ticks, d_model, n, ctx->d_mp_chunk, kt, launches, info, out)))
      return rc;
    CK(cudaMemcpyAsync(ctx->d_g_ticks + ctx->step_n, d_ticks, sizeof(int64_t) * n,
                       cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(ctx->d_g_model + ctx->step_n, d_model, sizeof(int32_t) * n,
                       cudaMemcpyDeviceToDevice, st));
    for (int k = 0; k < 5; k++)
      KL(k_fill64, nblk(n, 256), 256, 0, st>>>(ctx->d_g_out + k * ctx->g_cap + ctx->step_n, n,
                                               -1));
  }
  if (first) {
    for (Shard& S : ctx->shards) {
      S.check = (flags & SYM_FLAG_CHECK_INVARIANTS) ? 1 : 0;
      S.inject = -1;
    }
    CK(cudaMemsetAsync(ctx->d_step_shard, 0, sizeof(int64_t) * 3 * P, st));
    // static configuration and pointers of every shard (the chain state
    // itself is initialised by the first step's chain)
    CK(cudaMemcpyAsync(ctx->d_shards, ctx->shards.data(), sizeof(Shard) * P,
                       cudaMemcpyHostToDevice, st));
  }
  // ---- the new layout
  const int nxt = ctx->cur ^ 1, cur = ctx->cur;
  KL(k_step_sizes, nblk(M, 128), 128, 0, st>>>(ctx->d_mp, ctx->d_ms, ctx->d_mp_chunk, M,
                                               first ? 1 : 0, n > 0 ? 1 : 0, ctx->d_step_slot));
  KL(k_step_offsets, 1, 1024, 0, st>>>(ctx->d_step_slot, M));
  if (bound > 0)
    KL(k_step_copy, nblk(bound, 256), 256, 0, st>>>(
        bound, ctx->d_step_slot, M, P, ctx->d_slot_base, ctx->d_mp_chunk,
        ctx->d_lay_tick[cur], ctx->d_lay_g[cur], ctx->d_lay_i[cur], ctx->d_lay_aself[cur],
        ctx->d_s_tick, P > 1 ? ctx->d_s_g : ctx->d_s_i, ctx->d_s_i,
        P > 1 ? ctx->d_sh_tick : d_ticks, d_ticks, ctx->d_bins + B + 1, ctx->d_step_shard,
        ctx->step_n, ctx->d_lay_tick[nxt], ctx->d_lay_g[nxt], ctx->d_lay_i[nxt],
        ctx->d_lay_aself[nxt], ctx->d_lay_flag));
  KL(k_step_rebase, nblk(M, 128), 128, 0, st>>>(ctx->d_mp, ctx->d_ms, ctx->d_step_slot, M,
                                                first ? 1 : 0));
  KL(k_step_shard_update, 1, 32 * ((P + 31) / 32), 0, st>>>(
      ctx->d_step_shard, P, n, ctx->d_bins + B + 1, d_ticks, ctx->d_sh_tick));
  ctx->cur = nxt;
  int64_t* meta = ctx->d_meta;  // rec_base [P] | rec_count [P] | total
  KL(k_step_views, 1, 32 * ((P + 31) / 32), 0, st>>>(
      ctx->d_shards, P, ctx->d_step_slot, M, ctx->d_slot_base, ctx->d_lay_tick[nxt],
      ctx->d_lay_g[nxt], ctx->d_lay_aself[nxt], ctx->d_recs, meta));
  CK(cudaEventRecord(ctx->ev[1], st));
  // ---- the chain, every sub-cluster, up to `until`
  CK(cudaMemsetAsync(ctx->d_skip, 0, sizeof(int32_t) * P, st));
  KL(k_chain, P, 32, ctx->chain_smem, st>>>(
      ctx->d_shards, nullptr, ctx->d_dirty, ctx->d_slot_base, ctx->chain_smem, ctx->d_skip,
      first ? kChainFirstStep : kChainResume, until));
  CK(cudaEventRecord(ctx->ev[3], st));
  // ---- what the step decided
  KL(k_step_recmeta, 1, 32, 0, st>>>(ctx->d_shards, P, meta));
  CK(cudaMemsetAsync(ctx->d_step_cnt, 0, sizeof(int64_t) * 2, st));
  if (bound + P > 0)
    KL(k_step_emit, nblk(bound + P, 256), 256, 0, st>>>(
        ctx->d_recs, meta, meta + P + 1, P, meta + 2 * (P + 1), ctx->d_lay_i[nxt],
        ctx->d_bins + B + P + 2, ctx->d_slot_base, ctx->d_bins + B + P + 2 + M, ctx->g_cap,
        ctx->d_g_out, ctx->d_lay_flag, ctx->d_gbat + ctx->gbat_n,
        (unsigned long long*)ctx->d_step_cnt));
  if (bound > 0)
    KL(k_step_drops, nblk(bound, 256), 256, 0, st>>>(
        bound, ctx->d_step_slot, M, ctx->d_ms, ctx->d_lay_i[nxt], ctx->d_lay_flag, ctx->g_cap,
        ctx->d_g_out, (unsigned long long*)ctx->d_step_cnt));
  CK(cudaGetLastError());
  CK(cudaEventRecord(ctx->ev[4], st));
  int64_t hc[2] = {0, 0}, htot = 0;
  int32_t lay_total = 0;
  CK(cudaMemcpyAsync(ctx->shards.data(), ctx->d_shards, sizeof(Shard) * P,
                     cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(hc, ctx->d_step_cnt, sizeof hc, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&htot, meta + 2 * (P + 1), sizeof htot, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&lay_total, ctx->d_step_slot + (M + 1) + M, sizeof lay_total,
                     cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  for (int s = 0; s < P; s++) {
    if (ctx->shards[s].error) {
      ctx->step_active = false;
      ctx->err = "chain error " + std::to_string(ctx->shards[s].error) + " in sub-cluster " +
                 std::to_string(s) + " (invariant codes 3-6: see engine_core.cuh)";
      return SYM_EINVARIANT;
    }
  }
  ctx->step_first = false;
  ctx->step_n += n;
  ctx->step_until = until;
  ctx->gbat_n += htot;
  ctx->step_served += hc[0];
  ctx->step_drops += hc[1];
  ctx->lay_n = lay_total;
  out->n = ctx->step_n;
  out->n_batches = ctx->gbat_n;
  out->drops = ctx->step_drops;
  out->completions = ctx->step_served;
  out->late = 0;
  out->launches = launches;
  out->ops = out->evictions = out->registrations = out->handler_ops_max = 0;
  out->chain_events = out->absorbed_arrivals = out->fresh_adoptions = 0;
  for (int s = 0; s < P; s++) {
    const Shard& S = ctx->shards[s];
    out->ops += S.ops;
    out->evictions += S.evictions;
    out->registrations += S.registrations;
    out->handler_ops_max = std::max<int64_t>(out->handler_ops_max, S.handler_ops_max);
    out->chain_events += S.chain_events;
    out->absorbed_arrivals += S.absorbed;
  }
  out->fast_shards = 0;
  out->fast_fail_mask = 0;
  float t;
  cudaEventElapsedTime(&t, ctx->ev[0], ctx->ev[1]);
  out->ms_ingest = t;
  out->ms_fresh = 0;
  out->ms_fast = 0;
  cudaEventElapsedTime(&t, ctx->ev[1], ctx->ev[3]);
  out->ms_chain = t;
  cudaEventElapsedTime(&t, ctx->ev[3], ctx->ev[4]);
  out->ms_expand = t;
  cudaEventElapsedTime(&t, ctx->ev[0], ctx->ev[4]);
  out->ms_total = t;
  return SYM_OK;
}

}  // namespace

// ------------------------------------------------------------- C ABI ------

extern "C" {

int32_t sym_version(void) { return kVersion; }

#ifdef SYM_CHAIN_PROF
// dev build only (tools/chain_prof.py): read and clear the chain counters
int32_t sym_chain_prof(unsigned long long* out) {
  if (cudaMemcpyFromSymbol(out, sym::g_chain_prof, sizeof(unsigned long long) * 16) !=
      cudaSuccess)
    return SYM_ECUDA;
  unsigned long long z[16] = {};
  cudaMemcpyToSymbol(sym::g_chain_prof, z, sizeof z);
  return SYM_OK;
}
#endif

const char* sym_kernel_times(void* engine, int32_t reset) {
  if (sym_is_multi(engine)) return "{}";
  Ctx* ctx = static_cast<Ctx*>(engine);
  if (!ctx) return "{}";
  std::string j = "{";
  bool first = true;
  for (auto& kv : ctx->ktimes) {
    char buf[256];
    snprintf(buf, sizeof buf, "%s\"%s\": [%lld, %.6f]", first ? "" : ", ", kv.first.c_str(),
             (long long)kv.second.first, kv.second.second);
    j += buf;
    first = false;
  }
  j += "}";
  ctx->ktimes_json = j;
  if (reset) ctx->ktimes.clear();
  return ctx->ktimes_json.c_str();
}

const char* sym_last_error(void* engine) {
  if (sym_is_multi(engine)) return sym_multi_last_error(engine);
  return engine ? static_cast<Ctx*>(engine)->err.c_str() : "null engine";
}

void* sym_create(const sym_config* cfg, int32_t* status) {
  int32_t dummy;
  if (!status) status = &dummy;
  *status = SYM_EINVAL;
  if (!cfg || cfg->n_models < 1 || cfg->n_gpus < 1 || cfg->n_shards < 1 ||
      cfg->lat_stride < 1 || !cfg->lat_ns || !cfg->max_batch || !cfg->slo_ns)
    return nullptr;
  if (cfg->kind < 0 || cfg->kind > 2 || cfg->gather < 0 || cfg->gather > 1 ||
      cfg->d_ctrl_ns < 0 || cfg->d_data_ns < 0)
    return nullptr;
  if (cfg->gather == SYM_GATHER_DROP_HEAD && cfg->target_batch < 1)
    return nullptr;
  if (cfg->n_devices > 1 && cfg->devices) return sym_multi_create(cfg, status);
  Ctx* ctx = new Ctx();
  ctx->M = cfg->n_models;
  ctx->G = cfg->n_gpus;
  ctx->P = cfg->n_shards;
  ctx->kind = cfg->kind;
  ctx->gather = cfg->gather;
  ctx->lat_stride = cfg->lat_stride;
  ctx->d_ctrl = cfg->d_ctrl_ns;
  ctx->d_data = cfg->d_data_ns;
  ctx->device = cfg->device;
  if (const char* g = getenv("SYM_GUARD")) {
    ctx->guard = g[0] && g[0] != '0';
    if (const char* v = getenv("SYM_GUARD_POISON")) ctx->poison = (unsigned char)strtol(v, nullptr, 0);
    ctx->guard_selftest = getenv("SYM_GUARD_SELFTEST") != nullptr;
  }
  const int M = ctx->M, P = ctx->P;
  // shard membership and slot order (shard-major, model id within shard)
  ctx->shard_of_model.assign(M, 0);
  for (int m = 0; m < M; m++) {
    const int s = cfg->shard_of_model ? cfg->shard_of_model[m] : 0;
    if (s < 0 || s >= P) { delete ctx; return nullptr; }
    ctx->shard_of_model[m] = s;
  }
  ctx->slot_base.assign(P + 1, 0);
  for (int m = 0; m < M; m++) ctx->slot_base[ctx->shard_of_model[m] + 1]++;
  for (int s = 0; s < P; s++) ctx->slot_base[s + 1] += ctx->slot_base[s];
  ctx->slot_of_model.assign(M, 0);
  ctx->model_of_slot.assign(M, 0);
  {
    std::vector<int32_t> fill(ctx->slot_base.begin(), ctx->slot_base.end() - 1);
    for (int m = 0; m < M; m++) {
      const int k = fill[ctx->shard_of_model[m]]++;
      ctx->slot_of_model[m] = k;
      ctx->model_of_slot[k] = m;
    }
  }
  ctx->gpu_base.assign(P + 1, 0);
  for (int s = 0; s < P; s++) {
    const int g = cfg->gpus_per_shard ? cfg->gpus_per_shard[s] : ctx->G;
    if (g < 1) { delete ctx; return nullptr; }
    ctx->gpu_base[s + 1] = ctx->gpu_base[s] + g;
  }
  if (ctx->gpu_base[P] != ctx->G) { delete ctx; return nullptr; }
  for (int s = 0; s < P; s++)
    if (ctx->slot_base[s + 1] == ctx->slot_base[s]) { delete ctx; return nullptr; }
  // static model parameters by slot
  ctx->mp_host.resize(M);
  std::vector<int64_t> lat((size_t)M * ctx->lat_stride);
  for (int m = 0; m < M; m++) {
    const int k = ctx->slot_of_model[m];
    const int mb = cfg->max_batch[m];
    if (mb < 1 || mb > ctx->lat_stride) { delete ctx; return nullptr; }
    const int64_t* row = cfg->lat_ns + (int64_t)m * ctx->lat_stride;
    for (int b = 0; b < mb; b++) {
      if (row[b] <= 0 || (b > 0 && row[b] < row[b - 1])) { delete ctx; return nullptr; }
    }
    memcpy(&lat[(size_t)k * ctx->lat_stride], row, sizeof(int64_t) * ctx->lat_stride);
    ModelParam& p = ctx->mp_host[k];
    p.slo = cfg->slo_ns[m];
    p.timeout_ns = cfg->timeout_ns ? cfg->timeout_ns[m] : 0;
    p.base1 = cfg->d_ctrl_ns + cfg->d_data_ns + row[0];
    p.off = 0;
    p.cnt = 0;
    p.max_batch = mb;
    p.target_batch = cfg->target_batch < mb ? cfg->target_batch : mb;
    // exact affine detection: l(b) = a*b + c for every b in [1, max_batch]
    p.aff_a = mb > 1 ? row[1] - row[0] : 0;
    p.aff_b = row[0] - p.aff_a;
    p.affine = 1;
    for (int b = 0; b < mb; b++)
      if (row[b] != p.aff_a * (b + 1) + p.aff_b) p.affine = 0;
    p._pad = 0;
    ctx->max_slo = std::max<int64_t>(ctx->max_slo, p.slo);
    ctx->max_lat = std::max<int64_t>(ctx->max_lat, row[mb - 1]);
  }
  *status = SYM_ECUDA;
  auto fail = [&](const char* what, cudaError_t e) -> void* {
    fprintf(stderr, "sym_create: %s: %s\n", what, cudaGetErrorString(e));
    delete ctx;
    return nullptr;
  };
  cudaError_t e;
  if ((e = cudaSetDevice(ctx->device)) != cudaSuccess) return fail("cudaSetDevice", e);
  if ((e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking)) != cudaSuccess)
    return fail("stream", e);
  for (auto& ev : ctx->ev)
    if ((e = cudaEventCreate(&ev)) != cudaSuccess) return fail("event", e);
  if ((e = cudaDeviceGetAttribute(&ctx->n_sm, cudaDevAttrMultiProcessorCount, ctx->device)) !=
          cudaSuccess ||
      (e = cudaFuncSetAttribute(k_nxt_tma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                kNxtTmaSmem)) != cudaSuccess ||
      (e = cudaFuncSetAttribute(k_walk_expand, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                kExpandSmem)) != cudaSuccess)
    return fail("k_nxt_tma attributes", e);
  {  // keep pool memory mapped across synchronisations (no remap stalls)
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, ctx->device) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  // chain state
  ctx->shards.resize(P);
  std::vector<int32_t> mp2(P), gp2(P);
  int64_t tot_m2 = 0, tot_g2 = 0;
  for (int s = 0; s < P; s++) {
    int Ms = ctx->slot_base[s + 1] - ctx->slot_base[s];
    int Gs = ctx->gpu_base[s + 1] - ctx->gpu_base[s];
    int a = 1, b = 1;
    while (a < Ms) a <<= 1;
    while (b < Gs) b <<= 1;
    mp2[s] = a;
    gp2[s] = b;
    tot_m2 += 2 * a;
    tot_g2 += 2 * b;
  }
#define ALLOC(p, cnt)                                                        \
  if ((e = dmalloc(ctx, (void**)&(p), sizeof(*(p)) * (size_t)(cnt),         \
                   ctx->stream, #p)) != cudaSuccess)                          \
    return fail(#p, e);
  ALLOC(ctx->d_lat, (int64_t)M * ctx->lat_stride);
  ALLOC(ctx->d_mp, M);
  ALLOC(ctx->d_slot_of_model, M);
  ALLOC(ctx->d_shard_of_model, M);
  ALLOC(ctx->d_slot_base, P + 1);
  ALLOC(ctx->d_ms, M);
  ALLOC(ctx->d_pq, tot_m2);
  ALLOC(ctx->d_mlt, tot_m2);
  ALLOC(ctx->d_mbt, tot_m2);
  ALLOC(ctx->d_gt, tot_g2);
  ALLOC(ctx->d_pqt, tot_m2);
  ALLOC(ctx->d_gtf, tot_g2);
  ALLOC(ctx->d_mltv, tot_m2);
  ALLOC(ctx->d_mbtv, tot_m2);
  ALLOC(ctx->d_mcs, M);
  ALLOC(ctx->d_mcl, M);
  ALLOC(ctx->d_free, ctx->G);
  ALLOC(ctx->d_dirty, M + P);
  ALLOC(ctx->d_shards, P);
  // bins: [B+1] totals, then shard_off [P+1], model_of_slot [M], gpu_base [P+1]
  ALLOC(ctx->d_bins, (M + P + 1) + (P + 1) + M + (P + 1));
  ALLOC(ctx->d_err, 2);

  ALLOC(ctx->d_nb, M);
  ALLOC(ctx->d_bbase, M);
  ALLOC(ctx->d_mdrops, M);
  ALLOC(ctx->d_sbase, P + 1);
  ALLOC(ctx->d_fail, P);
  ALLOC(ctx->d_skip, P);
  ALLOC(ctx->d_changed, 4);
  ALLOC(ctx->d_unsure_n, 1);
  ALLOC(ctx->d_cpoff, M + 1);
  ALLOC(ctx->d_tie_cnt, P);
  ALLOC(ctx->d_tie_list, (int64_t)P * kTieMax);
  ALLOC(ctx->d_tie_eff, (int64_t)P * kTieEff);
  ALLOC(ctx->d_tie_sig, (int64_t)P * kTieX);
  ALLOC(ctx->d_tie_mask, (int64_t)P * 32);
  ALLOC(ctx->d_seg, 4 * (P + 1));
  ALLOC(ctx->d_special, M);
  ALLOC(ctx->d_slo_model, M);
  ctx->net_ctrl_n = cfg->net_ctrl_n > 0 ? cfg->net_ctrl_n : 0;
  ctx->net_data_n = cfg->net_data_n > 0 ? cfg->net_data_n : 0;
  ctx->jitter = ctx->net_ctrl_n + ctx->net_data_n > 0;
  ctx->net_ctrl_const = cfg->net_ctrl_const;
  ctx->net_data_const = cfg->net_data_const;
  ctx->net_key[0] = cfg->net_key[0];
  ctx->net_key[1] = cfg->net_key[1];
  ALLOC(ctx->d_net_vals, ctx->net_ctrl_n + ctx->net_data_n + 1);
  ALLOC(ctx->d_net_cdf, ctx->net_ctrl_n + ctx->net_data_n + 1);
  if (ctx->net_ctrl_n) {
    cudaMemcpyAsync(ctx->d_net_vals, cfg->net_ctrl_vals, sizeof(int64_t) * ctx->net_ctrl_n, cudaMemcpyHostToDevice, ctx->stream);
    cudaMemcpyAsync(ctx->d_net_cdf, cfg->net_ctrl_cdf, sizeof(double) * ctx->net_ctrl_n, cudaMemcpyHostToDevice, ctx->stream);
  }
  if (ctx->net_data_n) {
    cudaMemcpyAsync(ctx->d_net_vals + ctx->net_ctrl_n, cfg->net_data_vals, sizeof(int64_t) * ctx->net_data_n, cudaMemcpyHostToDevice, ctx->stream);
    cudaMemcpyAsync(ctx->d_net_cdf + ctx->net_ctrl_n, cfg->net_data_cdf, sizeof(double) * ctx->net_data_n, cudaMemcpyHostToDevice, ctx->stream);
  }
  ALLOC(ctx->d_meta, 3 * (P + 1));
  ALLOC(ctx->d_mp_chunk, M);
  ALLOC(ctx->d_step_slot, 4 * (M + 1));
  ALLOC(ctx->d_step_shard, 3 * P);
  ALLOC(ctx->d_step_cnt, 2);
#undef ALLOC
  const int B = M + P;
  cudaMemcpyAsync(ctx->d_lat, lat.data(), sizeof(int64_t) * lat.size(), cudaMemcpyHostToDevice, ctx->stream);
  cudaMemcpyAsync(ctx->d_mp, ctx->mp_host.data(), sizeof(ModelParam) * M, cudaMemcpyHostToDevice, ctx->stream);
  cudaMemcpyAsync(ctx->d_slot_of_model, ctx->slot_of_model.data(), sizeof(int32_t) * M, cudaMemcpyHostToDevice, ctx->stream);
  cudaMemcpyAsync(ctx->d_shard_of_model, ctx->shard_of_model.data(), sizeof(int32_t) * M, cudaMemcpyHostToDevice, ctx->stream);
  cudaMemcpyAsync(ctx->d_slot_base, ctx->slot_base.data(), sizeof(int32_t) * (P + 1), cudaMemcpyHostToDevice, ctx->stream);
  cudaMemcpyAsync(ctx->d_slo_model, cfg->slo_ns, sizeof(int64_t) * M, cudaMemcpyHostToDevice, ctx->stream);
  cudaMemcpyAsync(ctx->d_bins + B + P + 2, ctx->model_of_slot.data(), sizeof(int32_t) * M, cudaMemcpyHostToDevice, ctx->stream);
  cudaMemcpyAsync(ctx->d_bins + B + P + 2 + M, ctx->gpu_base.data(), sizeof(int32_t) * (P + 1), cudaMemcpyHostToDevice, ctx->stream);
  int64_t om = 0, og = 0;
  for (int s = 0; s < P; s++) {
    Shard& S = ctx->shards[s];
    memset(&S, 0, sizeof S);
    S.M = ctx->slot_base[s + 1] - ctx->slot_base[s];
    S.G = ctx->gpu_base[s + 1] - ctx->gpu_base[s];
    S.Mp = mp2[s];
    S.Gp = gp2[s];
    S.Mlog = 0;
    while ((1 << S.Mlog) < S.Mp) S.Mlog++;
    S.Glog = 0;
    while ((1 << S.Glog) < S.Gp) S.Glog++;
    S.kind = ctx->kind;
    S.gather = ctx->gather;
    S.d_ctrl = ctx->d_ctrl;
    S.d_data = ctx->d_data;
    S.lat_stride = ctx->lat_stride;
    S.lat = ctx->d_lat + (int64_t)ctx->slot_base[s] * ctx->lat_stride;
    S.mp = ctx->d_mp + ctx->slot_base[s];
    S.ms = ctx->d_ms + ctx->slot_base[s];
    S.pq = ctx->d_pq + om;
    S.pq_t = ctx->d_pqt + om;
    S.mc_lat_tree = ctx->d_mlt + om;
    S.mc_bs_tree = ctx->d_mbt + om;
    S.mlt_v = ctx->d_mltv + om;
    S.mbt_v = ctx->d_mbtv + om;
    S.gt = ctx->d_gt + og;
    S.gt_f = ctx->d_gtf + og;
    S.mc_size = ctx->d_mcs + ctx->slot_base[s];
    S.mc_latest = ctx->d_mcl + ctx->slot_base[s];
    S.free_at = ctx->d_free + ctx->gpu_base[s];
    om += 2 * S.Mp;
    og += 2 * S.Gp;
  }
  {
    int dev_max = 0;
    cudaDeviceGetAttribute(&dev_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device);
    size_t want = 0;
    for (const Shard& S : ctx->shards) want = std::max(want, SmemPlan::need(S));
    const size_t cap = dev_max > 4096 ? (size_t)dev_max - 2048 : 0;  // room for static S
    ctx->chain_smem = std::min(want, cap);
    if ((e = cudaFuncSetAttribute(k_chain, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)ctx->chain_smem)) != cudaSuccess)
      return fail("smem attribute", e);
    const size_t sc = part_smem(std::max(ctx->M, ctx->P));
    if (sc > (size_t)dev_max || ctx->M + ctx->P >= 32768)
      return fail("too many models for the ingest partition", cudaErrorInvalidValue);
    if ((e = cudaFuncSetAttribute(k_part<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)sc)) != cudaSuccess ||
        (e = cudaFuncSetAttribute(k_part<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)sc)) != cudaSuccess ||
        (e = cudaFuncSetAttribute(k_part<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)sc)) != cudaSuccess)
      return fail("partition smem attribute", e);
  }
  if ((e = cudaStreamSynchronize(ctx->stream)) != cudaSuccess) return fail("init", e);
  *status = SYM_OK;
  return ctx;
}

void sym_destroy(void* engine) {
  if (sym_is_multi(engine)) return sym_multi_destroy(engine);
  Ctx* ctx = static_cast<Ctx*>(engine);
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  void* ptrs[] = {ctx->d_lat,  ctx->d_mp,     ctx->d_slot_of_model,
                  ctx->d_shard_of_model, ctx->d_slot_base, ctx->d_ms,
                  ctx->d_pq,   ctx->d_gt,     ctx->d_mlt,   ctx->d_mbt,
                  ctx->d_mcs,  ctx->d_dirty,  ctx->d_free,  ctx->d_mcl,
                  ctx->d_pqt, ctx->d_gtf, ctx->d_mltv, ctx->d_mbtv,
                  ctx->d_shards, ctx->d_ticks, ctx->d_s_tick, ctx->d_sh_tick,
                  ctx->d_model, ctx->d_s_g,   ctx->d_s_i,
                  ctx->d_bid, ctx->d_scan_part, ctx->d_closek,
                  ctx->d_bins,   ctx->d_err,   ctx->d_fresh, ctx->d_hist, ctx->d_hist_part, ctx->d_bkt, ctx->d_bkt_part, ctx->d_seg, ctx->d_sh_i,
                  ctx->d_sh_slot,
                  ctx->d_recs, ctx->d_drop_t, ctx->d_drop_ks, ctx->d_drop_ka,
                  ctx->d_evb, ctx->d_bkA, ctx->d_bkB, ctx->d_tkA, ctx->d_tkB,
                  ctx->d_bvA, ctx->d_bvB, ctx->d_tvA, ctx->d_tvB, ctx->d_ptrA,
                  ctx->d_rhist, ctx->d_nb, ctx->d_bbase,
                  ctx->d_changed, ctx->d_mdrops, ctx->d_sbase, ctx->d_fail,
                  ctx->d_skip, ctx->d_nxt, ctx->d_jA, ctx->d_jB, ctx->d_jC,
                  ctx->d_unsure, ctx->d_unsure_n, ctx->d_cpoff, ctx->d_tie_cnt, ctx->d_tie_list, ctx->d_tie_eff,
                  ctx->d_tie_sig, ctx->d_tie_mask, ctx->d_cp_pos, ctx->d_cp_model,
                  ctx->d_special, ctx->d_meta, ctx->d_req,
                  ctx->d_drop, ctx->d_dka, ctx->d_bat, ctx->d_slo_model,
                  ctx->d_net_vals, ctx->d_net_cdf, ctx->d_g_ticks, ctx->d_g_model,
                  ctx->d_g_out, ctx->d_lay_tick[0], ctx->d_lay_tick[1], ctx->d_lay_g[0],
                  ctx->d_lay_g[1], ctx->d_lay_i[0], ctx->d_lay_i[1], ctx->d_lay_aself[0],
                  ctx->d_lay_aself[1], ctx->d_lay_flag, ctx->d_mp_chunk, ctx->d_step_slot,
                  ctx->d_step_shard, ctx->d_step_cnt, ctx->d_gbat};
  for (void* p : ptrs) dfree(ctx, p, ctx->stream);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  for (auto& ev : ctx->ev)
    if (ev) cudaEventDestroy(ev);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

int32_t sym_run_device(void* engine, const int64_t* d_arr_ticks,
                       const void* d_arr_model, int64_t n, uint32_t flags,
                       sym_result* out) {
  if (sym_is_multi(engine)) return SYM_EINVAL;  // device pointers live on one device
  Ctx* ctx = static_cast<Ctx*>(engine);
  if (!ctx || !out || n < 0 || n >= INT32_MAX) return SYM_EINVAL;
  if (cudaSetDevice(ctx->device) != cudaSuccess) return SYM_ECUDA;
  forget_last_run(ctx);
  out->n = n;
  out->err_index = -1;
  const int32_t* model = static_cast<const int32_t*>(d_arr_model);
  if (flags & SYM_FLAG_MODEL_I64) {
    int rc;
    if ((rc = ensure_capacity(ctx, n))) return rc;
    if (n > 0)
      k_narrow<<<nblk(n, 256), 256, 0, ctx->stream>>>(static_cast<const int64_t*>(d_arr_model),
                                                        n, ctx->d_model);
    model = ctx->d_model;
  }
  const int rc = run_device(ctx, d_arr_ticks, model, n, flags, out, true);
  return rc == SYM_OK ? guard_check(ctx) : rc;
}

int32_t sym_run(void* engine, const int64_t* arr_ticks, const void* arr_model,
                int64_t n, uint32_t flags, sym_result* out) {
  if (sym_is_multi(engine)) {
    if (!out || n < 0 || n >= INT32_MAX) return SYM_EINVAL;
    out->err_index = -1;
    return sym_multi_run(engine, arr_ticks, arr_model, n, flags, out);
  }
  Ctx* ctx = static_cast<Ctx*>(engine);
  if (!ctx || !out || n < 0 || n >= INT32_MAX) return SYM_EINVAL;
  CK(cudaSetDevice(ctx->device));
  forget_last_run(ctx);
  int rc;
  if ((rc = ensure_capacity(ctx, n))) return rc;
  cudaStream_t st = ctx->stream;
  if (n > 0) {
    CK(cudaMemcpyAsync(ctx->d_ticks, arr_ticks, sizeof(int64_t) * n,
                       cudaMemcpyHostToDevice, st));
    if (flags & SYM_FLAG_MODEL_I64) {  // widen on the device, not the host
      CK(cudaMemcpyAsync(ctx->d_s_tick, arr_model, sizeof(int64_t) * n,
                         cudaMemcpyHostToDevice, st));  // s_tick is free until ingest
      k_narrow<<<nblk(n, 256), 256, 0, st>>>(ctx->d_s_tick, n, ctx->d_model);
    } else {
      CK(cudaMemcpyAsync(ctx->d_model, arr_model, sizeof(int32_t) * n,
                         cudaMemcpyHostToDevice, st));
    }
  }
  // device-side output staging (persistent, grown on demand)
  sym_result dev = *out;
  const bool want_req = out->req_dispatch && !(flags & SYM_FLAG_NO_EXPAND);
  const bool want_drop = (flags & SYM_FLAG_TRACE) && out->drop_t;
  if (n + 1 > ctx->stage_cap) {
    const int64_t c = (n + 32) & ~int64_t(31);  // every staged array 256-byte aligned
    if ((rc = grow(ctx, ctx->d_req, 8 * c)) || (rc = grow(ctx, ctx->d_drop, 2 * c)) ||
        (rc = grow(ctx, ctx->d_dka, c)))
      return rc;
    ctx->stage_cap = c;
  }
  if (out->batches && out->batch_cap + 1 > ctx->bat_cap) {
    if ((rc = grow(ctx, ctx->d_bat, out->batch_cap + 1))) return rc;
    ctx->bat_cap = out->batch_cap + 1;
  }
  const int64_t sc = ctx->stage_cap;
  int64_t* d_req = ctx->d_req;
  int64_t* d_drop = ctx->d_drop;
  int32_t* d_dka = ctx->d_dka;
  sym_batch* d_b = out->batches ? ctx->d_bat : nullptr;
  dev.req_dispatch = want_req ? d_req : nullptr;
  dev.req_start = want_req ? d_req + sc : nullptr;
  dev.req_finish = want_req ? d_req + 2 * sc : nullptr;
  dev.req_batch = want_req ? d_req + 3 * sc : nullptr;
  dev.req_outcome = want_req ? d_req + 4 * sc : nullptr;
  dev.req_arrival = want_req && out->req_arrival ? d_req + 5 * sc : nullptr;
  dev.req_deadline = want_req && out->req_deadline ? d_req + 6 * sc : nullptr;
  dev.req_model = want_req && out->req_model ? d_req + 7 * sc : nullptr;
  dev.drop_t = want_drop ? d_drop : nullptr;
  dev.drop_key_sub = want_drop ? d_drop + sc : nullptr;
  dev.drop_key_a = want_drop ? d_dka : nullptr;
  dev.batches = d_b;
  dev.n = n;
  dev.err_index = -1;
  rc = run_device(ctx, ctx->d_ticks, ctx->d_model, n, flags, &dev, true);
  if (rc == SYM_OK) {
    if (want_req && n > 0) {
      int64_t* dsts[8] = {out->req_dispatch, out->req_start, out->req_finish,
                          out->req_batch, out->req_outcome, out->req_arrival,
                          out->req_deadline, out->req_model};
      for (int k = 0; k < 8; k++)
        if (dsts[k])
          CK(cudaMemcpyAsync(dsts[k], d_req + k * sc, sizeof(int64_t) * n,
                             cudaMemcpyDeviceToHost, st));
    }
    if (want_drop && n > 0) {
      CK(cudaMemcpyAsync(out->drop_t, d_drop, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(out->drop_key_sub, d_drop + sc, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(out->drop_key_a, d_dka, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st));
    }
    if (d_b && dev.n_batches > 0)
      CK(cudaMemcpyAsync(out->batches, d_b, sizeof(sym_batch) * dev.n_batches,
                         cudaMemcpyDeviceToHost, st));
  }
  CK(cudaStreamSynchronize(st));
  // copy back counters / timings
  sym_batch* keep_b = out->batches;
  int64_t keep_cap = out->batch_cap;
  int64_t *k0 = out->req_dispatch, *k1 = out->req_start, *k2 = out->req_finish,
          *k3 = out->req_batch, *k4 = out->req_outcome, *k5 = out->drop_t,
          *k6 = out->drop_key_sub, *k8 = out->req_arrival, *k9 = out->req_deadline,
          *k10 = out->req_model;
  int32_t* k7 = out->drop_key_a;
  *out = dev;
  out->batches = keep_b;
  out->batch_cap = keep_cap;
  out->req_dispatch = k0;
  out->req_start = k1;
  out->req_finish = k2;
  out->req_batch = k3;
  out->req_outcome = k4;
  out->req_arrival = k8;
  out->req_deadline = k9;
  out->req_model = k10;
  out->drop_t = k5;
  out->drop_key_sub = k6;
  out->drop_key_a = k7;
  return rc == SYM_OK ? guard_check(ctx) : rc;
}

int32_t sym_step_reset(void* engine) {
  if (sym_is_multi(engine)) return SYM_EINVAL;
  Ctx* ctx = static_cast<Ctx*>(engine);
  if (!ctx) return SYM_EINVAL;
  if (ctx->jitter) {
    ctx->err = "stepped runs support jitterless networks only";
    return SYM_EINVAL;
  }
  step_reset(ctx);
  return SYM_OK;
}

int32_t sym_step(void* engine, const int64_t* arr_ticks, const void* arr_model, int64_t n,
                 int64_t until_tick, uint32_t flags, sym_result* out) {
  if (sym_is_multi(engine)) return SYM_EINVAL;
  Ctx* ctx = static_cast<Ctx*>(engine);
  if (!ctx || !out || n < 0 || (n > 0 && (!arr_ticks || !arr_model))) return SYM_EINVAL;
  out->err_index = -1;
  if (!ctx->step_active) {
    ctx->err = "no stepped run in progress (sym_step_reset starts one)";
    return SYM_EINVAL;
  }
  if (flags & (SYM_FLAG_TRACE | SYM_FLAG_NO_EXPAND)) {
    ctx->err = "stepped runs take neither TRACE nor NO_EXPAND";
    return SYM_EINVAL;
  }
  if (until_tick < ctx->step_until || (n > 0 && (arr_ticks[0] < ctx->step_until ||
                                                  arr_ticks[n - 1] > until_tick))) {
    ctx->err = "a step's arrivals must lie in [previous until_tick, until_tick]";
    out->err_index = n > 0 && arr_ticks[0] < ctx->step_until ? 0 : n - 1;
    return SYM_EINVAL;
  }
  if (ctx->step_n + n >= INT32_MAX) {
    ctx->err = "stepped run too long (2^31 arrivals)";
    return SYM_EINVAL;
  }
  CK(cudaSetDevice(ctx->device));
  int rc;
  // scratch sized for the chunk and the new layout before the chunk lands
  if ((rc = ensure_capacity(ctx, std::max<int64_t>(n, ctx->lay_n + n)))) return rc;
  cudaStream_t st = ctx->stream;
  if (n > 0) {
    CK(cudaMemcpyAsync(ctx->d_ticks, arr_ticks, sizeof(int64_t) * n, cudaMemcpyHostToDevice,
                       st));
    if (flags & SYM_FLAG_MODEL_I64) {
      CK(cudaMemcpyAsync(ctx->d_s_tick, arr_model, sizeof(int64_t) * n, cudaMemcpyHostToDevice,
                         st));  // s_tick is free until the ingest
      k_narrow<<<nblk(n, 256), 256, 0, st>>>(ctx->d_s_tick, n, ctx->d_model);
    } else {
      CK(cudaMemcpyAsync(ctx->d_model, arr_model, sizeof(int32_t) * n, cudaMemcpyHostToDevice,
                         st));
    }
  }
  const int rc2 = step_device(ctx, ctx->d_ticks, ctx->d_model, n, until_tick, flags, out);
  return rc2 == SYM_OK ? guard_check(ctx) : rc2;
}

int32_t sym_step_result(void* engine, sym_result* out) {
  if (sym_is_multi(engine)) return SYM_EINVAL;
  Ctx* ctx = static_cast<Ctx*>(engine);
  if (!ctx || !out) return SYM_EINVAL;
  if (ctx->step_first && !ctx->step_active) {
    ctx->err = "no stepped run";
    return SYM_EINVAL;
  }
  CK(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  const int64_t n = ctx->step_n, cap = ctx->g_cap;
  if (out->batches && ctx->gbat_n > out->batch_cap) {
    ctx->err = "batch buffer too small";
    return SYM_EINVAL;
  }
  int64_t* dsts[5] = {out->req_dispatch, out->req_start, out->req_finish, out->req_batch,
                      out->req_outcome};
  for (int k = 0; k < 5; k++)
    if (dsts[k] && n > 0)
      CK(cudaMemcpyAsync(dsts[k], ctx->d_g_out + k * cap, sizeof(int64_t) * n,
                         cudaMemcpyDeviceToHost, st));
  std::vector<int32_t> model;
  if ((out->req_model || out->req_deadline) && n > 0) {
    model.resize(n);
    CK(cudaMemcpyAsync(model.data(), ctx->d_g_model, sizeof(int32_t) * n,
                       cudaMemcpyDeviceToHost, st));
  }
  std::vector<int64_t> ticks;
  int64_t* arr = out->req_arrival;
  if (!arr && out->req_deadline && n > 0) {
    ticks.resize(n);
    arr = ticks.data();
  }
  if (arr && n > 0)
    CK(cudaMemcpyAsync(arr, ctx->d_g_ticks, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, st));
  if (out->batches && ctx->gbat_n > 0)
    CK(cudaMemcpyAsync(out->batches, ctx->d_gbat, sizeof(sym_batch) * ctx->gbat_n,
                       cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  // a served request completes at its finish tick (simulator.py:249-258):
  // until then its outcome is unresolved, as in the reference mid-run
  int64_t completions = 0;
  if (out->req_outcome && out->req_finish)
    for (int64_t i = 0; i < n; i++) {
      if (out->req_outcome[i] == 0) {
        if (out->req_finish[i] > ctx->step_until) out->req_outcome[i] = -1;
        else completions++;
      }
    }
  if (out->req_model)
    for (int64_t i = 0; i < n; i++) out->req_model[i] = model[i];
  if (out->req_deadline)
    for (int64_t i = 0; i < n; i++)
      out->req_deadline[i] = arr[i] + ctx->mp_host[ctx->slot_of_model[model[i]]].slo;
  out->n = n;
  out->n_batches = ctx->gbat_n;
  out->drops = ctx->step_drops;
  out->completions = completions;
  out->late = 0;
  out->ops = out->evictions = out->registrations = out->handler_ops_max = 0;
  out->chain_events = out->absorbed_arrivals = out->fresh_adoptions = 0;
  for (const Shard& S : ctx->shards) {
    out->ops += S.ops;
    out->evictions += S.evictions;
    out->registrations += S.registrations;
    out->handler_ops_max = std::max<int64_t>(out->handler_ops_max, S.handler_ops_max);
    out->chain_events += S.chain_events;
    out->absorbed_arrivals += S.absorbed;
  }
  return SYM_OK;
}

int64_t sym_last_batches(void* engine, sym_batch* host, int64_t cap) {
  if (sym_is_multi(engine)) return sym_multi_last_batches(engine, host, cap);
  Ctx* ctx = static_cast<Ctx*>(engine);
  if (!ctx || !ctx->has_run) return -SYM_EINVAL;
  if (cudaSetDevice(ctx->device) != cudaSuccess) return -SYM_ECUDA;
  int64_t total = 0;
  for (int64_t c : ctx->last_nrecs) total += c;
  if (total > cap) return -SYM_EINVAL;
  if (total == 0) return 0;
  cudaStream_t st = ctx->stream;
  const int32_t M = ctx->M, P = ctx->P, B = M + P;
  if (total + 1 > ctx->bat_cap) {
    if (grow(ctx, ctx->d_bat, total + 1)) return -SYM_ECUDA;
    ctx->bat_cap = total + 1;
  }
  int64_t* meta = ctx->d_meta;
  if (cudaMemcpyAsync(meta, ctx->last_rec_base.data(), sizeof(int64_t) * P,
                      cudaMemcpyHostToDevice, st) != cudaSuccess ||
      cudaMemcpyAsync(meta + P + 1, ctx->last_nrecs.data(), sizeof(int64_t) * P,
                      cudaMemcpyHostToDevice, st) != cudaSuccess)
    return -SYM_ECUDA;
  k_copy_batches<<<nblk(total, 256), 256, 0, st>>>(
      ctx->d_recs, meta, meta + P + 1, P, ctx->d_s_i, ctx->d_bins + B + P + 2,
      ctx->d_slot_base, ctx->d_bins + B + P + 2 + M, total, ctx->d_bat);
  if (cudaMemcpyAsync(host, ctx->d_bat, sizeof(sym_batch) * total, cudaMemcpyDeviceToHost,
                      st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return -SYM_ECUDA;
  if (const int g = guard_check(ctx)) return -g;
  return total;
}

int32_t sym_window_counts(void* engine, int64_t lo_ns, int64_t hi_ns,
                          int64_t* model_arrivals, int64_t* model_completed,
                          int64_t* model_late, int64_t* model_dropped,
                          int64_t* gpu_busy_ns) {
  if (sym_is_multi(engine))
    return sym_multi_window_stats(engine, lo_ns, hi_ns, model_arrivals, model_completed,
                                  model_late, model_dropped, gpu_busy_ns, nullptr, nullptr,
                                  nullptr, 0);
  Ctx* ctx = static_cast<Ctx*>(engine);
  if (!ctx) return SYM_EINVAL;
  if (!ctx->has_run || !ctx->last_outcome) {
    ctx->err = "sym_window_counts: no expanded run to reduce";
    return SYM_EINVAL;
  }
  CK(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  const int32_t M = ctx->M, P = ctx->P, G = ctx->G;
  const int64_t n = ctx->last_n;
  unsigned long long* d = nullptr;
  CK(dmalloc(ctx, (void**)&d, sizeof(unsigned long long) * (4 * (size_t)M + G), st,
             "window counts"));
  CK(cudaMemsetAsync(d, 0, sizeof(unsigned long long) * (4 * (size_t)M + G), st));
  if (n > 0)
    k_window_req<<<nblk(n, 256), 256, 0, st>>>(ctx->last_ticks, ctx->last_model,
                                               ctx->last_outcome, n, lo_ns, hi_ns, d, M);
  int64_t total = 0;
  for (int64_t c : ctx->last_nrecs) total += c;
  if (total > 0) {
    int64_t* meta = ctx->d_meta;
    CK(cudaMemcpyAsync(meta, ctx->last_rec_base.data(), sizeof(int64_t) * P,
                       cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(meta + P + 1, ctx->last_nrecs.data(), sizeof(int64_t) * P,
                       cudaMemcpyHostToDevice, st));
    const int32_t B = M + P;
    k_window_busy<<<nblk(total, 256), 256, 0, st>>>(
        ctx->d_recs, meta, meta + P + 1, P, ctx->d_bins + B + P + 2 + M, total, lo_ns, hi_ns,
        d + 4 * (size_t)M);
  }
  std::vector<unsigned long long> h(4 * (size_t)M + G);
  CK(cudaMemcpyAsync(h.data(), d, sizeof(unsigned long long) * h.size(),
                     cudaMemcpyDeviceToHost, st));
  int grc = guard_check(ctx);
  dfree(ctx, d, st);
  CK(cudaStreamSynchronize(st));
  if (grc) return grc;
  for (int32_t m = 0; m < M; m++) {
    model_arrivals[m] = (int64_t)h[m];
    model_completed[m] = (int64_t)h[M + m];
    model_late[m] = (int64_t)h[2 * M + m];
    model_dropped[m] = (int64_t)h[3 * M + m];
  }
  for (int32_t g = 0; g < G; g++) gpu_busy_ns[g] = (int64_t)h[4 * (size_t)M + g];
  return SYM_OK;
}

int32_t sym_window_stats(void* engine, int64_t lo_ns, int64_t hi_ns, int64_t* model_arrivals,
                         int64_t* model_completed, int64_t* model_late, int64_t* model_dropped,
                         int64_t* gpu_busy_ns, int64_t* model_p99_ns, int64_t* model_max_qd_ns,
                         int64_t* model_batch_hist, int32_t hist_stride) {
  if (sym_is_multi(engine))
    return hist_stride < 1 ? SYM_EINVAL
                           : sym_multi_window_stats(engine, lo_ns, hi_ns, model_arrivals,
                                                    model_completed, model_late, model_dropped,
                                                    gpu_busy_ns, model_p99_ns, model_max_qd_ns,
                                                    model_batch_hist, hist_stride);
  Ctx* ctx = static_cast<Ctx*>(engine);
  if (!ctx || hist_stride < 1) return SYM_EINVAL;
  if (!ctx->has_run || !ctx->last_outcome || !ctx->last_start || !ctx->last_finish) {
    ctx->err = "sym_window_stats: no expanded run to reduce";
    return SYM_EINVAL;
  }
  int32_t rc = sym_window_counts(engine, lo_ns, hi_ns, model_arrivals, model_completed,
                                 model_late, model_dropped, gpu_busy_ns);
  if (rc != SYM_OK) return rc;
  cudaStream_t st = ctx->stream;
  const int32_t M = ctx->M, P = ctx->P, B = M + P;
  const int64_t n = ctx->last_n;
  for (int32_t m = 0; m < M; m++) model_max_qd_ns[m] = 0;
  const size_t nh = (size_t)M * hist_stride;
  // scratch: arrivals [M] | qd [M] | p99 [M] | hist [M*stride] | err
  unsigned long long* d = nullptr;
  CK(dmalloc(ctx, (void**)&d, sizeof(unsigned long long) * (3 * (size_t)M + nh + 1), st,
             "window stats"));
  CK(cudaMemsetAsync(d, 0, sizeof(unsigned long long) * (3 * (size_t)M + nh + 1), st));
  std::vector<unsigned long long> arr(model_arrivals, model_arrivals + M);
  CK(cudaMemcpyAsync(d, arr.data(), sizeof(unsigned long long) * M, cudaMemcpyHostToDevice, st));
  unsigned long long* d_qd = d + M;
  long long* d_p99 = reinterpret_cast<long long*>(d + 2 * M);
  unsigned long long* d_hist = d + 3 * (size_t)M;
  int32_t* d_err = reinterpret_cast<int32_t*>(d + 3 * (size_t)M + nh);
  const int32_t* model_of_slot = ctx->d_bins + B + P + 2;
  if (n > 0) {
    k_stat_keys<<<nblk(n, 256), 256, 0, st>>>(ctx->last_ticks, ctx->last_model,
                                              ctx->last_outcome, ctx->last_start,
                                              ctx->last_finish, ctx->d_slot_of_model, n, lo_ns,
                                              hi_ns, M, ctx->d_bkA, ctx->d_bvA, d_qd, d_err);
    int bits = kStatLatBits;
    while ((int64_t(1) << (bits - kStatLatBits)) <= M) bits++;
    const int64_t W = (n + kChunkR - 1) / kChunkR;
    for (int shift = 0; shift < bits; shift += kDigitBits) {
      k_rhist<<<nblk(W, kRadixWarps), 32 * kRadixWarps, 0, st>>>(ctx->d_bkA, n, shift,
                                                                 ctx->d_rhist, W);
      const int64_t len = W * kDigits, nparts = (len + kScanItems - 1) / kScanItems;
      k_scan_up<<<nparts, 1024, 0, st>>>(ctx->d_rhist, len, ctx->d_scan_part);
      k_scan_mid<<<1, 1024, 0, st>>>(ctx->d_scan_part, nparts);
      k_scan_down<<<nparts, 1024, 0, st>>>(ctx->d_rhist, len, ctx->d_scan_part);
      k_rscatter<<<nblk(W, kRadixWarps), 32 * kRadixWarps, 0, st>>>(
          ctx->d_bkA, ctx->d_bvA, n, shift, ctx->d_rhist, W, ctx->d_bkB, ctx->d_bvB);
      std::swap(ctx->d_bkA, ctx->d_bkB);
      std::swap(ctx->d_bvA, ctx->d_bvB);
    }
    k_stat_p99<<<1, 1024, 0, st>>>(ctx->d_bkA, d, model_of_slot, M, d_p99);
  }
  int64_t total = 0;
  for (int64_t c : ctx->last_nrecs) total += c;
  if (total > 0)  // d_meta still holds this run's rec_base / rec_count (sym_window_counts)
    k_stat_hist<<<nblk(total, 256), 256, 0, st>>>(ctx->d_recs, ctx->d_meta,
                                                   ctx->d_meta + P + 1, P, ctx->d_slot_base,
                                                   model_of_slot, total, lo_ns, hi_ns,
                                                   hist_stride, d_hist);
  CK(cudaGetLastError());
  std::vector<unsigned long long> h(3 * (size_t)M + nh + 1);
  CK(cudaMemcpyAsync(h.data(), d, sizeof(unsigned long long) * h.size(),
                     cudaMemcpyDeviceToHost, st));
  int grc = guard_check(ctx);
  dfree(ctx, d, st);
  CK(cudaStreamSynchronize(st));
  if (grc) return grc;
  if (reinterpret_cast<int32_t*>(&h[3 * (size_t)M + nh])[0]) {
    ctx->err = "sym_window_stats: a latency exceeds the 40-bit sort key";
    return SYM_EINVAL;
  }
  for (int32_t m = 0; m < M; m++) {
    model_max_qd_ns[m] = (int64_t)h[M + m];
    model_p99_ns[m] = n > 0 ? (int64_t)(long long)h[2 * M + m] : 0;
  }
  for (size_t k = 0; k < nh; k++) model_batch_hist[k] = (int64_t)h[3 * (size_t)M + k];
  return SYM_OK;
}

}  // extern "C"
