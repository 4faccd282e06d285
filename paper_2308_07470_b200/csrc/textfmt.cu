// textfmt.cu -- result-file text on the GPU (reference outputs.py:72-121).
//
// requests.csv / latency.csv are one line per request: a handful of int64
// columns rendered as decimal.  The reference builds them with a Python loop
// over numpy scalars (outputs.py:76-87, 116-120); at the stream sizes the
// engine handles (10^7..10^8 requests) that loop dominates wall time.  Here
// a block of kRows threads renders kRows consecutive rows: pass 1 sizes every
// row and reduces per block, a single-block scan places the blocks, pass 2
// sizes again, scans within the block, renders the rows into shared memory
// and streams the block's bytes out contiguously.  The text stays in HBM
// until the caller fetches it.  HBM-bound: ~56 B of columns in and ~55 B of
// text out per request.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <new>

#include "../../include/symphony_b200.h"

namespace {

constexpr int kRows = 256;        // rows (threads) per block
constexpr int kRowFixed = 160;    // bytes of a row besides the model name

struct Cols {
  const int64_t *model, *arr, *disp, *start, *fin, *batch, *outc;
  const char* names;
  const int64_t* noff;
  int32_t n_names;
  int64_t n;
};

__device__ __forceinline__ int ulen(uint64_t u) {
  int n = 1;
  uint64_t p = 10;
  while (n < 20 && u >= p) {
    ++n;
    p *= 10;
  }
  return n;
}

__device__ __forceinline__ uint64_t uabs(int64_t v) {
  return v < 0 ? 0ull - (uint64_t)v : (uint64_t)v;
}

// Emitters: the same row program sizes (Len) and renders (Put) a row, so the
// two passes cannot disagree.
struct Len {
  int n = 0;
  __device__ void ch(char) { ++n; }
  __device__ void str(const char*, int k) { n += k; }
  __device__ void num(int64_t v) { n += ulen(uabs(v)) + (v < 0); }
};

struct Put {
  char* p;
  __device__ void ch(char c) { *p++ = c; }
  __device__ void str(const char* s, int k) {
    for (int j = 0; j < k; ++j) p[j] = s[j];
    p += k;
  }
  __device__ void num(int64_t v) {
    uint64_t u = uabs(v);
    if (v < 0) *p++ = '-';
    char* e = p + ulen(u);
    p = e;
    do {  // exact u / 10 for every uint64 (multiply by 2^67/10, shift)
      uint64_t q = __umul64hi(u, 0xCCCCCCCCCCCCCCCDull) >> 3;
      *--e = char('0' + int(u - q * 10));
      u = q;
    } while (u);
  }
};

// One row; returns false for an invalid row (model id or outcome).
template <int KIND, class E>
__device__ __forceinline__ bool row(const Cols& c, int64_t i, E& e) {
  int64_t m = c.model[i], o = c.outc[i];
  if (m < 0 || m >= c.n_names || o < -1 || o > 2) return false;
  const char* name = c.names + c.noff[m];
  int nlen = int(c.noff[m + 1] - c.noff[m]);
  int64_t a = c.arr[i];
  if (KIND == SYM_TEXT_REQUESTS) {  // outputs.py:76-87
    e.num(i + 1); e.ch(','); e.str(name, nlen); e.ch(','); e.num(a);
    if (o == 2) {
      e.str(",,,,,dropped", 12);
    } else {
      e.ch(','); e.num(c.disp[i]); e.ch(','); e.num(c.start[i]); e.ch(',');
      e.num(c.fin[i]); e.ch(','); e.num(c.batch[i]); e.ch(',');
      if (o == 0) e.str("completed", 9);
      else if (o == 1) e.str("late", 4);
    }
    e.ch('\n');
  } else if (o == 0 || o == 1) {    // outputs.py:116-120
    e.str(name, nlen); e.ch(','); e.num(i + 1); e.ch(',');
    e.num(c.start[i] - a); e.ch(','); e.num(c.fin[i] - a); e.ch('\n');
  }
  return true;
}

template <int KIND>
__device__ __forceinline__ int row_len(const Cols& c, int64_t i, int* err) {
  if (i >= c.n) return 0;
  Len e;
  if (!row<KIND>(c, i, e)) {
    atomicExch(err, 1);
    return 0;
  }
  return e.n;
}

// Block-wide exclusive scan of one int per thread (kRows threads).
__device__ __forceinline__ int block_excl_scan(int v, int* total) {
  __shared__ int warp_sum[kRows / 32];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += y;
  }
  if (lane == 31) warp_sum[w] = x;
  __syncthreads();
  if (w == 0) {
    int s = lane < kRows / 32 ? warp_sum[lane] : 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, s, d);
      if (lane >= d) s += y;
    }
    if (lane < kRows / 32) warp_sum[lane] = s;
  }
  __syncthreads();
  int base = w ? warp_sum[w - 1] : 0;
  *total = warp_sum[kRows / 32 - 1];
  return base + x - v;
}

template <int KIND>
__global__ void __launch_bounds__(kRows) k_text_len(Cols c, int64_t* chunk, int* err) {
  int64_t i = int64_t(blockIdx.x) * kRows + threadIdx.x;
  int total;
  block_excl_scan(row_len<KIND>(c, i, err), &total);
  if (threadIdx.x == 0) chunk[blockIdx.x] = total;
}

// Exclusive scan of nb chunk sizes in place, total into chunk[nb]; one block.
__global__ void __launch_bounds__(1024) k_text_scan(int64_t* chunk, int64_t nb) {
  __shared__ int64_t part[1024];
  int64_t per = (nb + 1023) / 1024;
  int64_t lo = threadIdx.x * per, hi = lo + per < nb ? lo + per : nb;
  int64_t s = 0;
  for (int64_t k = lo; k < hi; ++k) s += chunk[k];
  part[threadIdx.x] = s;
  __syncthreads();
  for (int d = 1; d < 1024; d <<= 1) {  // Hillis-Steele on 1024 partials
    int64_t y = threadIdx.x >= d ? part[threadIdx.x - d] : 0;
    __syncthreads();
    part[threadIdx.x] += y;
    __syncthreads();
  }
  int64_t run = part[threadIdx.x] - s;
  for (int64_t k = lo; k < hi; ++k) {
    int64_t v = chunk[k];
    chunk[k] = run;
    run += v;
  }
  if (threadIdx.x == 1023) chunk[nb] = part[1023];
}

template <int KIND>
__global__ void __launch_bounds__(kRows) k_text_write(Cols c, const int64_t* chunk, char* text,
                                                      int* err) {
  extern __shared__ char stage[];
  int64_t i = int64_t(blockIdx.x) * kRows + threadIdx.x;
  int total;
  int off = block_excl_scan(row_len<KIND>(c, i, err), &total);
  if (i < c.n) {
    Put e{stage + off};
    row<KIND>(c, i, e);
  }
  __syncthreads();
  char* dst = text + chunk[blockIdx.x];
  for (int k = threadIdx.x; k < total; k += kRows) dst[k] = stage[k];
}

struct Text {
  int device;
  char* d;
  int64_t len;
  cudaStream_t st;  // stream-ordered memory: nothing here syncs the device
};

#define CK(x)                              \
  do {                                     \
    if ((x) != cudaSuccess) goto cuda_fail; \
  } while (0)

template <int KIND>
int32_t format(const Cols& c, int64_t nb, size_t smem, cudaStream_t st, int64_t* d_chunk,
               int* d_err, Text* t) {
  int h_err = 0;
  if (nb) {
    k_text_len<KIND><<<(unsigned)nb, kRows, 0, st>>>(c, d_chunk, d_err);
    k_text_scan<<<1, 1024, 0, st>>>(d_chunk, nb);
  } else if (cudaMemsetAsync(d_chunk, 0, 8, st) != cudaSuccess) {
    return SYM_ECUDA;
  }
  if (cudaMemcpyAsync(&t->len, d_chunk + nb, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaMemcpyAsync(&h_err, d_err, 4, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return SYM_ECUDA;
  if (h_err) return SYM_EINVAL;
  if (cudaMallocAsync((void**)&t->d, t->len ? t->len : 1, st) != cudaSuccess) return SYM_ENOMEM;
  if (nb) {
    if (cudaFuncSetAttribute(k_text_write<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
      return SYM_ECUDA;
    k_text_write<KIND><<<(unsigned)nb, kRows, smem, st>>>(c, d_chunk, t->d, d_err);
  }
  if (cudaStreamSynchronize(st) != cudaSuccess || cudaGetLastError() != cudaSuccess)
    return SYM_ECUDA;
  return SYM_OK;
}

}  // namespace

extern "C" {

void* sym_text_format(int32_t kind, const sym_text_columns* cols, int32_t device,
                      int64_t* out_len, int32_t* status) {
  *status = SYM_EINVAL;
  if (!cols || cols->n < 0 || cols->n_names < 0 ||
      (kind != SYM_TEXT_REQUESTS && kind != SYM_TEXT_LATENCY))
    return nullptr;
  int64_t n = cols->n, N = cols->n_names;
  int64_t maxname = 0;
  for (int64_t m = 0; m < N; ++m) {
    int64_t l = cols->name_off[m + 1] - cols->name_off[m];
    if (l < 0) return nullptr;
    maxname = l > maxname ? l : maxname;
  }
  size_t smem = size_t(kRows) * size_t(kRowFixed + maxname);
  if (smem > 200 * 1024) return nullptr;  // model names > ~640 bytes
  int64_t nb = (n + kRows - 1) / kRows;

  *status = SYM_ECUDA;
  int prev = 0;
  cudaGetDevice(&prev);
  if (cudaSetDevice(device) != cudaSuccess) return nullptr;
  Text* t = new (std::nothrow) Text{device, nullptr, 0, nullptr};
  cudaStream_t st = nullptr;
  char* blob = nullptr;  // columns | chunk sizes | names | offsets | err
  int32_t rc = SYM_ECUDA;
  if (!t) {
    *status = SYM_ENOMEM;
    cudaSetDevice(prev);
    return nullptr;
  }
  {
    const int64_t* src[7] = {cols->req_model, cols->req_arrival, cols->req_dispatch,
                             cols->req_start, cols->req_finish, cols->req_batch,
                             cols->req_outcome};
    int64_t names_len = N ? cols->name_off[N] : 0;
    size_t col_bytes = size_t(n) * 8;
    size_t o_chunk = 7 * col_bytes, o_names = o_chunk + size_t(nb + 1) * 8;
    size_t o_noff = (o_names + names_len + 15) & ~size_t(15);
    size_t o_err = o_noff + size_t(N + 1) * 8, bytes = o_err + 16;
    Cols c{};
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    if (cudaMallocAsync((void**)&blob, bytes, st) != cudaSuccess) {
      rc = SYM_ENOMEM;
      goto done;
    }
    for (int k = 0; k < 7; ++k)
      if (n) CK(cudaMemcpyAsync(blob + k * col_bytes, src[k], col_bytes, cudaMemcpyDefault, st));
    if (names_len)
      CK(cudaMemcpyAsync(blob + o_names, cols->names, names_len, cudaMemcpyDefault, st));
    CK(cudaMemcpyAsync(blob + o_noff, cols->name_off, (N + 1) * 8, cudaMemcpyDefault, st));
    CK(cudaMemsetAsync(blob + o_err, 0, 16, st));
    c.model = (const int64_t*)(blob);
    c.arr = (const int64_t*)(blob + col_bytes);
    c.disp = (const int64_t*)(blob + 2 * col_bytes);
    c.start = (const int64_t*)(blob + 3 * col_bytes);
    c.fin = (const int64_t*)(blob + 4 * col_bytes);
    c.batch = (const int64_t*)(blob + 5 * col_bytes);
    c.outc = (const int64_t*)(blob + 6 * col_bytes);
    c.names = blob + o_names;
    c.noff = (const int64_t*)(blob + o_noff);
    c.n_names = (int32_t)N;
    c.n = n;
    rc = kind == SYM_TEXT_REQUESTS
             ? format<SYM_TEXT_REQUESTS>(c, nb, smem, st, (int64_t*)(blob + o_chunk),
                                         (int*)(blob + o_err), t)
             : format<SYM_TEXT_LATENCY>(c, nb, smem, st, (int64_t*)(blob + o_chunk),
                                        (int*)(blob + o_err), t);
    goto done;
  }
cuda_fail:
  rc = SYM_ECUDA;
done:
  if (blob) cudaFreeAsync(blob, st);
  if (rc != SYM_OK) {
    if (t->d) cudaFreeAsync(t->d, st);
    if (st) {
      cudaStreamSynchronize(st);
      cudaStreamDestroy(st);
    }
    cudaSetDevice(prev);
    *status = rc;
    delete t;
    return nullptr;
  }
  t->st = st;
  cudaSetDevice(prev);
  *status = rc;
  *out_len = t->len;
  return t;
}

int32_t sym_text_fetch(void* text, char* dst, int64_t len) {
  Text* t = (Text*)text;
  if (!t || len != t->len) return SYM_EINVAL;
  if (!len) return SYM_OK;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(t->device);
  cudaError_t e = cudaMemcpyAsync(dst, t->d, size_t(len), cudaMemcpyDeviceToHost, t->st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(t->st);
  cudaSetDevice(prev);
  return e == cudaSuccess ? SYM_OK : SYM_ECUDA;
}

void sym_text_free(void* text) {
  Text* t = (Text*)text;
  if (!t) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(t->device);
  if (t->d) cudaFreeAsync(t->d, t->st);
  cudaStreamSynchronize(t->st);
  cudaStreamDestroy(t->st);
  cudaSetDevice(prev);
  delete t;
}

}  // extern "C"
