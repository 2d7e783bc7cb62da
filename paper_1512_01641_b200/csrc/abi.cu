// abi.cu -- the extern "C" boundary (include/bimine_b200.h) and launchers.
//
// Single translation unit: the kernels live in the included headers.
// Built by paper_1512_01641_b200/build.py with
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false
// (-fmad=false: no contraction anywhere; the glibc exp restatement uses
// explicit __fma_rn where the host libm fuses).
#include <cuda_runtime.h>

#include <cub/device/device_scan.cuh>
#include <thrust/iterator/transform_iterator.h>

#include <algorithm>
#include <chrono>
#include <emmintrin.h>
#include <array>
#include <cstdlib>
#include <cstdio>
#include <map>
#include <memory>
#include <cstring>
#include <condition_variable>
#include <functional>
#include <future>
#include <mutex>
#include <numeric>
#include <string>
#include <unordered_map>
#include <thread>
#include <vector>

#include "../../include/bimine_b200.h"
#include "common.cuh"
#include "lexicon_em.cuh"
#include "nw_kernel.cuh"
#include "pair_kernel.cuh"
#include "score_kernel.cuh"
#include "terms.cuh"

using namespace bimine;

namespace {

thread_local std::string g_error;

int fail(int code, const std::string &msg) {
  g_error = msg;
  return code;
}

#define BIMINE_CUDA(expr)                                                                  \
  do {                                                                                     \
    cudaError_t _e = (expr);                                                               \
    if (_e != cudaSuccess)                                                                 \
      return fail(BIMINE_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));      \
  } while (0)

cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

// a non-blocking upload stream per device (host -> device copies that
// overlap the mining of the previous chunk)
std::mutex g_cs_mu;
std::map<int, cudaStream_t> g_copy_streams;
cudaStream_t copy_stream() {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_cs_mu);
  auto it = g_copy_streams.find(dev);
  if (it != g_copy_streams.end()) return it->second;
  cudaStream_t s = nullptr;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  g_copy_streams[dev] = s;
  return s;
}

// sentence offsets rebuilt on the device: exclusive sum of the lengths,
// accumulated in int64
struct LenToI64 {
  __host__ __device__ int64_t operator()(int32_t x) const { return (int64_t)x; }
};
cudaError_t offsets_from_lengths(const int32_t *len, int64_t *off, int64_t n, void *tmp, size_t *tmp_bytes,
                                 cudaStream_t st) {
  return cub::DeviceScan::ExclusiveSum(tmp, *tmp_bytes, thrust::make_transform_iterator(len, LenToI64()), off, n,
                                       st);
}

// pinned host scratch per thread, grown on demand (upload staging)
struct PinnedScratch {
  void *p = nullptr;
  size_t n = 0;
  ~PinnedScratch() {
    if (p) cudaFreeHost(p);
  }
};
thread_local PinnedScratch tl_pinned;
void *pinned_grow(PinnedScratch &b, size_t bytes) {
  if (b.n < bytes) {
    if (b.p) cudaFreeHost(b.p);
    b.p = nullptr;
    b.n = 0;
    if (cudaMallocHost(&b.p, bytes) != cudaSuccess) return nullptr;
    b.n = bytes;
  }
  return b.p;
}
void *pinned_scratch(size_t bytes) { return pinned_grow(tl_pinned, bytes); }
// a small batch's whole upload, laid out like the device arena's front
thread_local PinnedScratch tl_mirror;

// Upload gate of bimine_mine_host: the score kernel waits per chunk; the
// launches that read everything (long-sentence kernel, NW) wait for `all`.
struct UploadGate {
  const int32_t *ready;  // grows as pieces land
  cudaEvent_t all;
  std::function<void()> before_all;  // host side: `all` is recorded once this returns
  bool pair_launched = false;        // the pair kernel already runs (bimine_mine_host launches it early)
  int64_t n_sentences = 0, n_tokens = 0;
  int32_t n_pieces = 0;
  const int64_t *piece_start = nullptr;
};
thread_local const UploadGate *tl_gate = nullptr;
cudaError_t gate_wait_all(cudaStream_t st) {
  if (!tl_gate) return cudaSuccess;
  if (tl_gate->before_all) tl_gate->before_all();
  return cudaStreamWaitEvent(st, tl_gate->all, 0);
}

// ---- pageable host input staged through page-locked memory ----------------
// A cudaMemcpyAsync from pageable memory is synchronous and goes through the
// driver's own small staging buffer.  Pageable arrays are instead copied by
// a few host threads into a ring of page-locked slots, each slot's H2D
// issued as soon as it is full and the slot reused once that copy is done.
bool is_pageable(const void *p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

const char *const kNarrowOnlyHost =
    "uint16 sentence arrays (bimine_batch.sent_bytes = 2) are accepted by bimine_mine_host only";

// memcpy into page-locked staging with streaming (non-temporal) stores: the
// destination is only read again by the DMA engine, so its lines need not
// be fetched first (a cached store reads each line before writing it; glibc
// switches to streaming stores only above a size tied to the L3)
void stream_copy(char *dst, const char *src, size_t n) {
  size_t head = (64 - ((uintptr_t)dst & 63)) & 63;
  if (head > n) head = n;
  memcpy(dst, src, head);
  dst += head;
  src += head;
  n -= head;
  const size_t body = n & ~(size_t)63;
  for (size_t i = 0; i < body; i += 64) {
    const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i *>(src + i));
    const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i *>(src + i + 16));
    const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i *>(src + i + 32));
    const __m128i d = _mm_loadu_si128(reinterpret_cast<const __m128i *>(src + i + 48));
    _mm_stream_si128(reinterpret_cast<__m128i *>(dst + i), a);
    _mm_stream_si128(reinterpret_cast<__m128i *>(dst + i + 16), b);
    _mm_stream_si128(reinterpret_cast<__m128i *>(dst + i + 32), c);
    _mm_stream_si128(reinterpret_cast<__m128i *>(dst + i + 48), d);
  }
  _mm_sfence();  // the streamed lines are globally visible before the H2D is issued
  memcpy(dst + body, src + body, n - body);
}

class MemcpyPool {  // fork-join memcpy over a few persistent threads
 public:
  static MemcpyPool &get() {
    static MemcpyPool pool;
    return pool;
  }
  void copy(void *dst, const void *src, size_t bytes) {
    if (bytes < ((size_t)1 << 20) || n_ == 0) {
      stream_copy((char *)dst, (const char *)src, bytes);
      return;
    }
    std::lock_guard<std::mutex> op(op_mu_);  // one copy at a time (several host threads may stage)
    std::unique_lock<std::mutex> lk(mu_);
    dst_ = (char *)dst;
    src_ = (const char *)src;
    bytes_ = bytes;
    pending_ = n_;
    ++gen_;
    cv_.notify_all();
    // this thread takes the last part
    const size_t part = (bytes + n_) / (n_ + 1), lo = std::min(bytes, part * n_);
    lk.unlock();
    stream_copy((char *)dst + lo, (const char *)src + lo, bytes - lo);
    lk.lock();
    done_.wait(lk, [&] { return pending_ == 0; });
  }

 private:
  MemcpyPool() {
    const unsigned hc = std::max(1u, std::thread::hardware_concurrency());
    const char *v = getenv("BIMINE_STAGE_THREADS");  // helper threads (the caller copies too)
    // default: 7 helpers from 16 hardware threads up (C2 pageable e2e on the
    // 16-thread B200 host: 3 -> 4.3 ms, 7 -> 3.2, 11 -> 3.3, 15 -> 3.2)
    n_ = v ? std::max(0, std::min(63, atoi(v))) : (int)std::min(7u, std::max(1u, hc / 2));
    for (int k = 0; k < n_; ++k) threads_.emplace_back([this, k] { run(k); });
  }
  ~MemcpyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto &t : threads_) t.join();
  }
  void run(int k) {
    uint64_t seen = 0;
    std::unique_lock<std::mutex> lk(mu_);
    while (true) {
      cv_.wait(lk, [&] { return gen_ != seen; });
      seen = gen_;
      if (stop_) return;
      char *dst = dst_;
      const char *src = src_;
      const size_t bytes = bytes_, part = (bytes + n_) / (n_ + 1);
      lk.unlock();
      const size_t lo = std::min(bytes, part * k), hi = std::min(bytes, part * (k + 1));
      if (hi > lo) stream_copy(dst + lo, src + lo, hi - lo);
      lk.lock();
      if (--pending_ == 0) done_.notify_all();
    }
  }
  std::mutex op_mu_, mu_;
  std::condition_variable cv_, done_;
  std::vector<std::thread> threads_;
  int n_ = 0, pending_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
  char *dst_ = nullptr;
  const char *src_ = nullptr;
  size_t bytes_ = 0;
};

class Stager {  // H2D on `st`: pinned sources directly, pageable ones through the ring
 public:
  static constexpr int kSlots = 4;
  static constexpr size_t kSlotBytes = (size_t)32 << 20;
  Stager(cudaStream_t st, int device) : st_(st), dev_(device) {}
  ~Stager() {
    for (auto &e : ev_)
      if (e) cudaEventDestroy(e);
    if (lease_) lease_->mu.unlock();
  }
  cudaError_t copy(void *dst, const void *src, size_t bytes, bool pageable) {
    if (!bytes) return cudaSuccess;
    if (!pageable) return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st_);
    cudaError_t e = ensure();
    for (size_t off = 0; off < bytes && e == cudaSuccess; off += kSlotBytes) {
      const size_t n = std::min(kSlotBytes, bytes - off);
      const int k = next_++ % kSlots;
      if (used_[k]) e = cudaEventSynchronize(ev_[k]);  // the slot's previous copy is done
      if (e != cudaSuccess) break;
      char *slot = lease_->p + (size_t)k * kSlotBytes;
      MemcpyPool::get().copy(slot, (const char *)src + off, n);
      e = cudaMemcpyAsync((char *)dst + off, slot, n, cudaMemcpyHostToDevice, st_);
      if (e == cudaSuccess) e = cudaEventRecord(ev_[k], st_);
      used_[k] = true;
    }
    return e;
  }

 private:
  // one page-locked ring per device, leased for a whole upload (calls on
  // one device stage one after the other)
  struct Ring {
    std::mutex mu;
    char *p = nullptr;
  };
  static Ring &ring_of(int dev) {
    static std::mutex mu;
    static std::map<int, Ring *> rings;
    std::lock_guard<std::mutex> lk(mu);
    Ring *&r = rings[dev];
    if (!r) r = new Ring();  // process lifetime
    return *r;
  }
  cudaError_t ensure() {
    if (!lease_) {
      Ring &r = ring_of(dev_);
      r.mu.lock();
      lease_ = &r;
      // events are recorded on st_ and never outlive it; the ring's last
      // copies completed before the previous lease ended (see ~Stager use)
      if (!r.p && cudaMallocHost((void **)&r.p, kSlots * kSlotBytes) != cudaSuccess) {
        r.p = nullptr;
        return cudaErrorMemoryAllocation;
      }
    }
    for (auto &e : ev_)
      if (!e) {
        const cudaError_t r = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
        if (r != cudaSuccess) return r;
      }
    return cudaSuccess;
  }

 public:
  // the ring may be reused by the next lease only once its copies are done
  cudaError_t drain() {
    cudaError_t e = cudaSuccess;
    for (int k = 0; k < kSlots; ++k)
      if (used_[k] && e == cudaSuccess) e = cudaEventSynchronize(ev_[k]);
    return e;
  }

 private:
  cudaStream_t st_;
  int dev_;
  Ring *lease_ = nullptr;
  cudaEvent_t ev_[kSlots] = {};
  bool used_[kSlots] = {};
  int next_ = 0;
};

// a device word the long-sentence kernel reports overflows in (one per
// device: one process may drive several GPUs, one host thread each)
int *device_status_word() {
  static std::mutex mu;
  static std::map<int, int *> words;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  int *&w = words[dev];
  if (!w && cudaMalloc(&w, sizeof(int)) != cudaSuccess) w = nullptr;
  return w;
}

// the current device's default pool keeps freed blocks cached (once per
// device: one process may drive several GPUs, one host thread each)
void pool_setup() {
  static std::mutex mu;
  static uint64_t done = 0;  // bit per device id < 64
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return;
  std::lock_guard<std::mutex> lk(mu);
  if (done >> dev & 1) return;
  done |= 1ull << dev;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t threshold = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold);
  }
}

int next_pow2(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

int ilog2(int x) {
  int b = 0;
  while ((1 << b) < x) ++b;
  return b;
}

constexpr int kMaxCapU = 4096;
constexpr int kMaxCapT = 16384;
constexpr int kNwWarpsPerBlock = 4;
constexpr size_t kNwSmemPerBlockMax = 200 * 1024;

}  // namespace

struct bimine_dict {
  int device = 0;
  int64_t n_rows = 0;
  int64_t n_entries = 0;
  int64_t *row_ptr = nullptr;
  int32_t *tgt = nullptr;
  double *prob = nullptr;
  uint64_t *rowdesc = nullptr;  // score kernel's copy: start << 24 | length per row
  DictEntry *ent = nullptr;     //                      {p, t} per entry
};

// bimine_plan_batch over sentence arrays of either width (T = int32_t, or
// uint16_t for bimine_mine_host's narrow form)
template <class T>
int plan_batch_t(const bimine_batch *b, const T *sent_len, const T *sent_uniq, int64_t *work, int64_t work_cap,
                 bimine_plan *plan) {
  bimine_plan P;
  memset(&P, 0, sizeof(P));
  // maxima over the sentences the pairs reference (a view of a larger batch
  // plans in time proportional to its own pairs)
  std::vector<int64_t> longs, larges;
  int64_t t = 0;
  for (int64_t p = 0; p < b->n_pairs; ++p)
    P.n_cells = std::max(P.n_cells, b->pair_sim_off[p] + (int64_t)b->pair_n[p] * b->pair_m[p]);
  for (int64_t p = 0; p < b->n_pairs; ++p) {
    const int32_t n = b->pair_n[p], m = b->pair_m[p];
    if (n < 1 || m < 1) return fail(BIMINE_E_ARG, "bimine_plan_batch: empty document");
    P.max_n = std::max(P.max_n, n);
    P.max_m = std::max(P.max_m, m);
    int32_t ml = 0, mu = 0;
    for (int32_t i = 0; i < n; ++i) {
      ml = std::max(ml, (int32_t)sent_len[b->pair_src[p] + i]);
      mu = std::max(mu, (int32_t)sent_uniq[b->pair_src[p] + i]);
    }
    for (int32_t j = 0; j < m; ++j) {
      ml = std::max(ml, (int32_t)sent_len[b->pair_tgt[p] + j]);
      mu = std::max(mu, (int32_t)sent_uniq[b->pair_tgt[p] + j]);
    }
    P.max_len = std::max(P.max_len, ml);
    P.max_uniq = std::max(P.max_uniq, mu);
    if (n > kPairMax || m > kPairMax) larges.push_back(p);  // NW: cluster kernel
    if (ml > kPairMaxLen) {
      longs.push_back(p);
      P.long_max_n = std::max(P.long_max_n, n);
      P.long_max_m = std::max(P.long_max_m, m);
    } else if (n > kPairMax || m > kPairMax) {
      for (int32_t i0 = 0; i0 < n; i0 += kPairMax)
        for (int32_t j0 = 0; j0 < m; j0 += kPairMax) {
          if (3 * t + 3 <= work_cap) {
            work[3 * t] = p;
            work[3 * t + 1] = i0;
            work[3 * t + 2] = j0;
          }
          ++t;
        }
    }
  }
  P.n_tiles = t;
  P.n_long = (int64_t)longs.size();
  P.n_large = (int64_t)larges.size();
  P.work_len = 3 * P.n_tiles + P.n_long + 3 * P.n_large;
  *plan = P;
  if (P.work_len > work_cap) return fail(BIMINE_E_ARG, "bimine_plan_batch: work_cap < plan->work_len");
  for (int64_t k = 0; k < P.n_long; ++k) work[3 * P.n_tiles + k] = longs[k];
  int64_t *lw = work + 3 * P.n_tiles + P.n_long;
  for (int64_t k = 0; k < P.n_large; ++k) {
    lw[k] = larges[k];
    lw[P.n_large + 2 * k] = b->pair_n[larges[k]];
    lw[P.n_large + 2 * k + 1] = b->pair_m[larges[k]];
  }
  return BIMINE_OK;
}


extern "C" {

const char *bimine_last_error(void) { return g_error.c_str(); }

const char *bimine_version(void) { return "bimine_b200 0.1.0 (sm_100a)"; }

// ------------------------------------------------------------------------
// dictionary
// ------------------------------------------------------------------------

int bimine_dict_create(const int32_t *src, const int32_t *tgt, const double *prob, int64_t n_entries,
                       bimine_dict **out) {
  if (!out || n_entries < 0 || (n_entries > 0 && (!src || !tgt || !prob)))
    return fail(BIMINE_E_ARG, "bimine_dict_create: bad arguments");
  // last value per (src, tgt) wins (lexicon.py:177); drop !(p > 0)
  std::vector<int64_t> order(n_entries);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int64_t x, int64_t y) {
    if (src[x] != src[y]) return src[x] < src[y];
    return tgt[x] < tgt[y];
  });
  std::vector<int32_t> ks, kt;
  std::vector<double> kp;
  ks.reserve(n_entries);
  kt.reserve(n_entries);
  kp.reserve(n_entries);
  for (int64_t k = 0; k < n_entries; ++k) {
    const int64_t e = order[k];
    const bool last_of_key =
        k + 1 == n_entries || src[order[k + 1]] != src[e] || tgt[order[k + 1]] != tgt[e];
    if (!last_of_key) continue;  // stable sort: the later duplicate comes last
    if (src[e] < 0 || tgt[e] < 0) return fail(BIMINE_E_ARG, "bimine_dict_create: negative token id");
    if (!(prob[e] > 0.0)) continue;
    ks.push_back(src[e]);
    kt.push_back(tgt[e]);
    kp.push_back(prob[e]);
  }
  auto *d = new bimine_dict();
  cudaGetDevice(&d->device);
  d->n_entries = (int64_t)ks.size();
  d->n_rows = ks.empty() ? 0 : (int64_t)ks.back() + 1;
  std::vector<int64_t> row_ptr(d->n_rows + 1, 0);
  for (int32_t s : ks) row_ptr[s + 1]++;
  for (int64_t r = 0; r < d->n_rows; ++r) row_ptr[r + 1] += row_ptr[r];
  if (d->n_entries >= ((int64_t)1 << 40)) {
    delete d;
    return fail(BIMINE_E_LIMIT, "bimine_dict_create: more than 2^40 entries");
  }
  // the score kernel's layout: one 8-byte descriptor per row, one 16-byte
  // {p, t} record per entry
  std::vector<uint64_t> rowdesc(std::max<int64_t>(1, d->n_rows));
  for (int64_t r = 0; r < d->n_rows; ++r) {
    const int64_t len = row_ptr[r + 1] - row_ptr[r];
    if (len >= (1 << 24)) {
      delete d;
      return fail(BIMINE_E_LIMIT, "bimine_dict_create: a source word has 2^24 or more translations");
    }
    rowdesc[r] = ((uint64_t)row_ptr[r] << 24) | (uint64_t)len;
  }
  std::vector<DictEntry> ent(std::max<int64_t>(1, d->n_entries));
  for (int64_t k = 0; k < d->n_entries; ++k) ent[k] = DictEntry{kp[k], kt[k], 0};
  auto cleanup = [&](const char *what) {
    cudaFree(d->row_ptr);
    cudaFree(d->tgt);
    cudaFree(d->prob);
    cudaFree(d->rowdesc);
    cudaFree(d->ent);
    delete d;
    return fail(BIMINE_E_CUDA, std::string("bimine_dict_create: ") + what);
  };
  if (cudaMalloc(&d->row_ptr, sizeof(int64_t) * (d->n_rows + 1)) != cudaSuccess) return cleanup("cudaMalloc");
  if (cudaMalloc(&d->tgt, sizeof(int32_t) * std::max<int64_t>(1, d->n_entries)) != cudaSuccess) return cleanup("cudaMalloc");
  if (cudaMalloc(&d->prob, sizeof(double) * std::max<int64_t>(1, d->n_entries)) != cudaSuccess) return cleanup("cudaMalloc");
  if (cudaMalloc(&d->rowdesc, sizeof(uint64_t) * rowdesc.size()) != cudaSuccess) return cleanup("cudaMalloc");
  if (cudaMalloc(&d->ent, sizeof(DictEntry) * ent.size()) != cudaSuccess) return cleanup("cudaMalloc");
  if (cudaMemcpy(d->row_ptr, row_ptr.data(), sizeof(int64_t) * (d->n_rows + 1), cudaMemcpyHostToDevice) != cudaSuccess ||
      (d->n_entries &&
       (cudaMemcpy(d->tgt, kt.data(), sizeof(int32_t) * d->n_entries, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(d->prob, kp.data(), sizeof(double) * d->n_entries, cudaMemcpyHostToDevice) != cudaSuccess)) ||
      cudaMemcpy(d->rowdesc, rowdesc.data(), sizeof(uint64_t) * rowdesc.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(d->ent, ent.data(), sizeof(DictEntry) * ent.size(), cudaMemcpyHostToDevice) != cudaSuccess)
    return cleanup("cudaMemcpy");
  *out = d;
  return BIMINE_OK;
}

int bimine_dict_destroy(bimine_dict *d) {
  if (!d) return BIMINE_OK;
  cudaFree(d->row_ptr);
  cudaFree(d->tgt);
  cudaFree(d->prob);
  cudaFree(d->rowdesc);
  cudaFree(d->ent);
  delete d;
  return BIMINE_OK;
}

int bimine_dict_view_get(const bimine_dict *d, bimine_dict_view *v) {
  if (!d || !v) return fail(BIMINE_E_ARG, "bimine_dict_view_get: null");
  v->n_rows = d->n_rows;
  v->n_entries = d->n_entries;
  v->row_ptr = d->row_ptr;
  v->tgt = d->tgt;
  v->prob = d->prob;
  return BIMINE_OK;
}

int64_t bimine_dict_entries(const bimine_dict *d) { return d ? d->n_entries : -1; }

// ------------------------------------------------------------------------
// score matrix
// ------------------------------------------------------------------------

int bimine_plan_batch(const bimine_batch *b, int64_t *work, int64_t work_cap, bimine_plan *plan) {
  if (!b || !plan || (work_cap > 0 && !work)) return fail(BIMINE_E_ARG, "bimine_plan_batch: null argument");
  if (b->sent_bytes == 2) return fail(BIMINE_E_ARG, kNarrowOnlyHost);
  return plan_batch_t<int32_t>(b, b->sent_len, b->sent_uniq, work, work_cap, plan);
}

}  // extern "C"

namespace {

// Term tables (terms.cuh) per (device, model), built once on the device.
struct TermCacheEntry {
  double *base = nullptr;
  TermTables T;
};

std::mutex g_term_mu;
std::map<std::pair<int, std::array<double, 21>>, TermCacheEntry> g_terms;

int term_tables(const double *model, cudaStream_t st, TermTables *out) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::array<double, 21> key;
  memcpy(key.data(), model, sizeof(double) * 21);
  std::lock_guard<std::mutex> lock(g_term_mu);
  auto it = g_terms.find({dev, key});
  if (it != g_terms.end()) {
    *out = it->second.T;
    return BIMINE_OK;
  }
  const size_t D2 = (size_t)kTermDim * kTermDim, C2 = (size_t)kCharDim * kCharDim;
  const size_t total = 4 * D2 + C2 + kRecipDim + 2;
  TermCacheEntry e;
  BIMINE_CUDA(cudaMalloc(&e.base, total * sizeof(double)));
  double *q = e.base;
  double *t0 = q, *t1 = q + D2, *t2 = q + 2 * D2, *t5 = q + 3 * D2, *t4 = q + 4 * D2;
  double *rc = t4 + C2, *misc = rc + kRecipDim;
  const int64_t n = (int64_t)std::max(C2, D2);
  build_term_tables<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(to_model(model), t0, t1, t2, t5, t4, rc, misc);
  BIMINE_CUDA(cudaGetLastError());
  BIMINE_CUDA(cudaStreamSynchronize(st));
  e.T = TermTables{t0, t1, t2, t5, t4, rc, misc};
  g_terms[{dev, key}] = e;
  *out = e.T;
  return BIMINE_OK;
}

}  // namespace

extern "C" {

}  // extern "C"

namespace {

// uint16 sentence arrays (bimine_mine_host's narrow upload) -> the int32
// arrays every kernel reads: src holds len | uniq | chars, n each
__global__ void widen_u16_kernel(const uint16_t *__restrict__ src, int64_t n, int32_t *__restrict__ len,
                                 int32_t *__restrict__ uniq, int32_t *__restrict__ chars) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < 3 * n; k += (int64_t)gridDim.x * blockDim.x) {
    int32_t *dst = k < n ? len : k < 2 * n ? uniq : chars;
    dst[k - (k < n ? 0 : k < 2 * n ? n : 2 * n)] = (int32_t)src[k];
  }
}

// One launch of the pair kernel: the tiles of pairs larger than 64x64, then
// one item per pair, over persistent CTAs.  gate: the upload gate of
// bimine_mine_host (null: the data are in place).
int launch_pair_kernel(const bimine_dict *dict, const double *model, const bimine_batch *b, const int64_t *tiles,
                       int64_t n_tiles, int64_t n_cells, double *sim_dev, cudaStream_t st, double *features,
                       const UploadGate *gate) {
  if (b->n_pairs > 0x7fffffffLL) return fail(BIMINE_E_LIMIT, "bimine_score_batch: more than 2^31-1 pairs per call");
  PairArgs A;
  memset(&A, 0, sizeof(A));
  A.b = to_dev(*b);
  A.d = DictDev{dict->n_rows, dict->row_ptr, dict->tgt, dict->prob, dict->rowdesc, dict->ent};
  A.md = to_model(model);
  int rc = term_tables(model, st, &A.T);
  if (rc != BIMINE_OK) return rc;
  A.sim = sim_dev;
  // per-cell counters (L2 resident while a CTA works on them), then the
  // persistent CTAs' work counter
  const size_t aux_bytes = (sizeof(uint16_t) * std::max<int64_t>(n_cells, 1) + 15) & ~(size_t)15;
  BIMINE_CUDA(cudaMallocAsync((void **)&A.aux, aux_bytes + 16, st));
  A.next_item = (unsigned long long *)((char *)A.aux + aux_bytes);
  BIMINE_CUDA(cudaMemsetAsync(A.next_item, 0, 8, st));
  const size_t smem = kPairSmemBytes;
  const bool packed = b->token_bytes == 3;
  auto kern = features ? (packed ? pair_kernel<true, true> : pair_kernel<true, false>)
                       : (packed ? pair_kernel<false, true> : pair_kernel<false, false>);
  BIMINE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  BIMINE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  A.tiles = n_tiles ? tiles : nullptr;
  A.n_tiles = n_tiles;
  A.features = features;
  if (gate) {
    A.ready = gate->ready;
    A.n_sentences = gate->n_sentences;
    A.n_tokens = gate->n_tokens;
    A.n_pieces = gate->n_pieces;
    A.piece_start = gate->piece_start;
  }
  const int64_t items = n_tiles + b->n_pairs;
  static thread_local std::map<std::pair<int, const void *>, int> resident;  // (device, kernel) -> CTAs per SM
  int dev = 0;
  cudaGetDevice(&dev);
  int &per_sm = resident[{dev, (const void *)kern}];
  if (per_sm == 0) {
    BIMINE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kPairThreads, smem));
    per_sm = std::max(per_sm, 1);
  }
  const int64_t grid = std::min<int64_t>(items, (int64_t)num_sms() * per_sm);
  kern<<<(unsigned)grid, kPairThreads, smem, st>>>(A);
  const cudaError_t le = cudaGetLastError();
  cudaFreeAsync(A.aux, st);
  if (le != cudaSuccess) return fail(BIMINE_E_CUDA, std::string("pair_kernel: ") + cudaGetErrorString(le));
  return BIMINE_OK;
}

int launch_scores(const bimine_dict *dict, const double *model, const bimine_batch *b, const bimine_plan *plan,
                  double *sim_dev, cudaStream_t st, double *features = nullptr) {
  if (!dict || !model || !b || !plan || !sim_dev) return fail(BIMINE_E_ARG, "bimine_score_batch: null argument");
  if (b->sent_bytes == 2) return fail(BIMINE_E_ARG, kNarrowOnlyHost);
  if (b->n_pairs == 0) return BIMINE_OK;
  if (plan->max_n < 1 || plan->max_m < 1 || plan->max_uniq < 1 || plan->max_len < 1)
    return fail(BIMINE_E_ARG, "bimine_score_batch: empty document or sentence");
  if (plan->max_uniq > kMaxCapU || plan->max_len > kMaxCapT)
    return fail(BIMINE_E_LIMIT, "bimine_score_batch: a sentence has more than 4096 distinct or 16384 total tokens");
  if (b->n_pairs > 0x7fffffffLL) return fail(BIMINE_E_LIMIT, "bimine_score_batch: more than 2^31-1 pairs per call");
  if (plan->work_len > 0 && !plan->work) return fail(BIMINE_E_ARG, "bimine_score_batch: plan.work not set");
  pool_setup();  // stream-ordered scratch stays cached (no remapping per call)
  const BatchDev bd = to_dev(*b);
  const DictDev dd = DictDev{dict->n_rows, dict->row_ptr, dict->tgt, dict->prob, dict->rowdesc, dict->ent};
  const Model md = to_model(model);
  if (!(tl_gate && tl_gate->pair_launched)) {
    const int rc = launch_pair_kernel(dict, model, b, plan->n_tiles ? plan->work : nullptr, plan->n_tiles,
                                      plan->n_cells, sim_dev, st, features, tl_gate);
    if (rc != BIMINE_OK) return rc;
  }
  if (plan->n_long > 0) {
    BIMINE_CUDA(gate_wait_all(st));
    ScoreArgs A;
    A.b = bd;
    A.d = dd;
    A.md = md;
    A.sim = sim_dev;
    A.pair_ids = plan->work + 3 * plan->n_tiles;
    A.cap_u = std::min(kMaxCapU, std::max(1024, next_pow2(plan->max_uniq)));
    A.cap_t = std::min(kMaxCapT, std::max(4096, next_pow2(plan->max_len)));
    A.hash_bits = ilog2(2 * A.cap_u);
    int *status = device_status_word();
    if (!status) return fail(BIMINE_E_CUDA, "score_kernel: status word allocation failed");
    A.status = status;
    const size_t smem = score_smem_layout(nullptr, A.cap_u, A.cap_t, nullptr);
    BIMINE_CUDA(cudaFuncSetAttribute(score_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    dim3 grid((unsigned)plan->n_long, (unsigned)((plan->long_max_n + kScoreTile - 1) / kScoreTile),
              (unsigned)((plan->long_max_m + kScoreTile - 1) / kScoreTile));
    if (grid.y > 65535 || grid.z > 65535) return fail(BIMINE_E_LIMIT, "bimine_score_batch: document too long");
    score_kernel<<<grid, kScoreThreads, smem, st>>>(A);
    BIMINE_CUDA(cudaGetLastError());
  }
  return BIMINE_OK;
}

}  // namespace

extern "C" {

int bimine_score_batch(const bimine_dict *dict, const double *model, const bimine_batch *b, const bimine_plan *plan,
                       double *sim_dev, void *stream) {
  return launch_scores(dict, model, b, plan, sim_dev, as_stream(stream));
}

}  // extern "C"

// ------------------------------------------------------------------------
// NW launch helper
// ------------------------------------------------------------------------
namespace {

// host_ids / host_dims (optional, host memory): the problems' pair ids and
// (N, M), so that the large-problem path sizes its scratch without a device
// round trip (one setting per problem)
template <int MODE>
int launch_nw(NwArgs A, int32_t max_n, int32_t max_m, cudaStream_t st, const int64_t *host_ids = nullptr,
              const int64_t *host_dims = nullptr) {
  if (A.n_problems == 0) return BIMINE_OK;
  pool_setup();
  const int row_d = ((max_m + 1) + 1) & ~1;  // doubles, even
  const int64_t dir_w = (MODE == kNwTable) ? 0 : (lean_dir_words16(max_n, max_m) + 1) / 2;  // u32 words
  const size_t per_warp = (size_t)row_d * 8 + (size_t)dir_w * 4;
  A.row_doubles_per_warp = row_d;
  if (MODE == kNwTable) A.dir_words_per_warp = 0;
  const size_t per_block = per_warp * kNwWarpsPerBlock;
  // one warp per problem for small problems; problems taller than 64 rows
  // go to the band pipeline (one CTA each)
  if (MODE != kNwTable && max_n <= 64 && dir_w < (1LL << 31) && per_block <= kNwSmemPerBlockMax) {
    A.dir_words_per_warp = (int)dir_w;
    A.g_dirs = nullptr;
    A.g_rows = nullptr;
    BIMINE_CUDA(cudaFuncSetAttribute(nw_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)per_block));
    int blocks_per_sm = 0;
    BIMINE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, nw_kernel<MODE>,
                                                              kNwWarpsPerBlock * 32, per_block));
    if (blocks_per_sm < 1) blocks_per_sm = 1;
    const int64_t want = (A.n_problems + kNwWarpsPerBlock - 1) / kNwWarpsPerBlock;
    const int64_t grid = std::min<int64_t>(want, (int64_t)num_sms() * blocks_per_sm);
    nw_kernel<MODE><<<(unsigned)grid, kNwWarpsPerBlock * 32, per_block, st>>>(A);
    BIMINE_CUDA(cudaGetLastError());
    return BIMINE_OK;
  }
  if (MODE != kNwTable) {
    // large problems: K CTAs each (16 warps pipelined over row bands per CTA);
    // K > 1 only while every CTA of the launch can be resident at once
    const int64_t nprob = A.n_problems;
    if (nprob > 0x7fffffffLL) return fail(BIMINE_E_LIMIT, "nw: too many large problems");
    const int gmax = (max_n + 31) / 32;
    int kc = std::max(1, std::min(16, (gmax + kBigW - 1) / kBigW));  // CTAs per cluster (= per problem)
#ifdef BIMINE_PROFILE_SKIP_TRACEBACK  // profiling builds only: time the sweep alone
    constexpr bool skip_tb = true;
#else
    constexpr bool skip_tb = false;
#endif
    constexpr size_t smem = big_smem_bytes<kBigW>();
    auto kern = nw_big_kernel<MODE, kBigW>;
    BIMINE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    BIMINE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    cfg.blockDim = dim3(kBigW * 32, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    {  // the largest cluster the device schedules for this kernel (queried once per device and size)
      static std::mutex mu;
      static std::map<std::pair<int, int>, int> best;
      int dev = 0;
      cudaGetDevice(&dev);
      std::lock_guard<std::mutex> lk(mu);
      auto it = best.find({dev, kc});
      if (it != best.end()) {
        kc = it->second;
      } else {
        const int want = kc;
        while (kc > 1) {
          attr[0].val.clusterDim.x = (unsigned)kc;
          attr[0].val.clusterDim.y = 1;
          attr[0].val.clusterDim.z = 1;
          cfg.gridDim = dim3((unsigned)kc, 1, 1);
          int ok = 0;
          if (cudaOccupancyMaxActiveClusters(&ok, kern, &cfg) == cudaSuccess && ok > 0) break;
          cudaGetLastError();
          --kc;
        }
        best[{dev, want}] = kc;
      }
    }
    attr[0].val.clusterDim.x = (unsigned)kc;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    if (nprob * kc > 0x7fffffffLL) return fail(BIMINE_E_LIMIT, "nw: too many large problems");
    cfg.gridDim = dim3((unsigned)(nprob * kc), 1, 1);
    // per-problem scratch: exact offsets from the caller's host plan (ids and
    // (N, M) of every problem; a pair's operand layout shared by its
    // problems), else uniform strides from max_n / max_m computed on the
    // device -- no host round trip either way
    const bool exact = host_dims && host_ids && A.n_settings == 1;
    int64_t nd = 0, dtotal = 0, dirtotal = 0, rowtotal = 0;
    int gmax_d = 1, mmax = 1;
    std::vector<int64_t> offs;
    int64_t dir_stride = 0, rows_stride = 0, diag_stride = 0;
    if (exact) {
      std::vector<int64_t> dpairs, dslot(nprob);
      {
        std::unordered_map<int64_t, int64_t> seen;
        for (int64_t k = 0; k < nprob; ++k) {
          const int64_t pr = host_ids[k];
          auto it = seen.find(pr);
          if (it == seen.end()) it = seen.emplace(pr, (int64_t)dpairs.size()).first, dpairs.push_back(pr);
          dslot[k] = it->second;
        }
      }
      // [distinct pairs] | pair diag offsets | per problem: diag, dirs, rows
      nd = (int64_t)dpairs.size();
      offs.resize(2 * nd + 3 * nprob);
      int64_t *h_pairs = offs.data(), *h_pdoff = h_pairs + nd, *h_doff = h_pdoff + nd, *h_dir = h_doff + nprob,
              *h_rows = h_dir + nprob;
      std::vector<int64_t> first_prob(nd, -1);
      for (int64_t k = 0; k < nprob; ++k)
        if (first_prob[dslot[k]] < 0) first_prob[dslot[k]] = k;
      for (int64_t q = 0; q < nd; ++q) {
        const int n = (int)host_dims[2 * first_prob[q]], m = (int)host_dims[2 * first_prob[q] + 1];
        h_pairs[q] = dpairs[q];
        h_pdoff[q] = dtotal;
        gmax_d = std::max(gmax_d, (n + 31) / 32);
        mmax = std::max(mmax, m);
        dtotal += (int64_t)((n + 31) / 32) * nw_diag_steps(m) * 32;
      }
      for (int64_t k = 0; k < nprob; ++k) {
        const int n = (int)host_dims[2 * k], m = (int)host_dims[2 * k + 1];
        h_doff[k] = h_pdoff[dslot[k]];
        h_dir[k] = dirtotal;
        dirtotal += (lean_dir_words16(n, m) + 1) / 2;
        h_rows[k] = rowtotal;
        rowtotal += 2 * ((int64_t)m + 1);
      }
    } else {
      gmax_d = (max_n + 31) / 32;
      mmax = max_m;
      nd = A.problem_ids ? nprob : nprob / A.n_settings;  // listed problems: a layout each
      dir_stride = (lean_dir_words16(max_n, max_m) + 1) / 2;
      rows_stride = 2 * ((int64_t)max_m + 1);
      diag_stride = (int64_t)gmax_d * nw_diag_steps(max_m) * 32;
      dtotal = nd * diag_stride;
      dirtotal = nprob * dir_stride;
      rowtotal = nprob * rows_stride;
    }
    double *diag = nullptr, *lastv = nullptr;
    int64_t *d_offs = nullptr;
    uint32_t *dirs = nullptr;
    double2 *rows = nullptr;
    BIMINE_CUDA(cudaMallocAsync((void **)&diag, sizeof(double) * std::max<int64_t>(dtotal, 1), st));
    BIMINE_CUDA(cudaMallocAsync((void **)&d_offs, sizeof(int64_t) * (2 * nd + 3 * nprob), st));
    BIMINE_CUDA(cudaMallocAsync((void **)&dirs, sizeof(uint32_t) * std::max<int64_t>(dirtotal, 1), st));
    BIMINE_CUDA(cudaMallocAsync((void **)&lastv, sizeof(double) * nprob, st));
    BIMINE_CUDA(cudaMallocAsync((void **)&rows, sizeof(double2) * std::max<int64_t>(rowtotal, 1), st));
    if (exact) {  // (pageable: the call returns once `offs` is copied)
      BIMINE_CUDA(cudaMemcpyAsync(d_offs, offs.data(), sizeof(int64_t) * offs.size(), cudaMemcpyHostToDevice, st));
    } else {
      uniform_offsets_kernel<<<(unsigned)std::min<int64_t>((nprob + 255) / 256, 4096), 256, 0, st>>>(
          A.problem_ids, nprob, A.n_settings, nd, dir_stride, rows_stride, diag_stride, d_offs);
      BIMINE_CUDA(cudaGetLastError());
    }
    BIMINE_CUDA(cudaMemsetAsync(rows, 0xff, sizeof(double2) * std::max<int64_t>(rowtotal, 1), st));
    const int64_t *dd_pairs = d_offs, *dd_pdoff = d_offs + nd, *dd_doff = dd_pdoff + nd, *dd_dir = dd_doff + nprob,
                  *dd_rows = dd_dir + nprob;
    {
      const int64_t per_band = nw_diag_steps(mmax) * 32;
      const dim3 grid((unsigned)std::min<int64_t>((per_band + 255) / 256, 64), (unsigned)std::min(gmax_d, 65535),
                      (unsigned)std::min<int64_t>(nd, 65535));
      nw_diag_kernel<<<grid, 256, 0, st>>>(A.sim, A.sim_off, A.pair_n, A.pair_m, dd_pairs, dd_pdoff, nd, A.mismatch,
                                           A.bonus - A.mismatch, diag);  // one IEEE subtraction, as fsub
      BIMINE_CUDA(cudaGetLastError());
    }
    BIMINE_CUDA(cudaLaunchKernelEx(&cfg, kern, A, dirs, dd_dir, rows, dd_rows, lastv, (const double *)diag, dd_doff));
    if (MODE != kNwTable && !skip_tb)
      nw_big_traceback_kernel<MODE><<<(unsigned)std::min<int64_t>(nprob, 1 << 20), 32, 0, st>>>(A, dirs, dd_dir,
                                                                                                    lastv, nprob);
    const cudaError_t e = cudaGetLastError();
    cudaFreeAsync(dirs, st);
    cudaFreeAsync(rows, st);
    cudaFreeAsync(lastv, st);
    cudaFreeAsync(diag, st);
    cudaFreeAsync(d_offs, st);
    if (e != cudaSuccess) return fail(BIMINE_E_CUDA, std::string("nw_big_kernel: ") + cudaGetErrorString(e));
    return BIMINE_OK;
  }
  // table mode (B1 shim): global scratch, one slot per launched warp, bounded to ~2 GiB
  if (dir_w >= (1LL << 31)) return fail(BIMINE_E_LIMIT, "nw: alignment table too large");
  int64_t warps = std::min<int64_t>(A.n_problems, (int64_t)num_sms() * 16);
  warps = std::max<int64_t>(1, std::min<int64_t>(warps, (int64_t)((size_t)2 << 30) / (int64_t)per_warp));
  const int64_t blocks = (warps + kNwWarpsPerBlock - 1) / kNwWarpsPerBlock;
  const int64_t slots = blocks * kNwWarpsPerBlock;  // every launched warp owns a slot
  A.dir_words_per_warp = (MODE == kNwTable) ? 0 : (int)dir_w;
  void *scratch = nullptr;
  BIMINE_CUDA(cudaMallocAsync(&scratch, per_warp * slots, st));
  A.g_rows = (double *)scratch;  // [slots][row_d] then [slots][dir_w]
  A.g_dirs = (uint32_t *)((char *)scratch + (size_t)row_d * 8 * slots);
  if (MODE == kNwTable) A.g_dirs = (uint32_t *)A.g_rows;  // never dereferenced; marks "global"
  nw_kernel<MODE><<<(unsigned)blocks, kNwWarpsPerBlock * 32, 0, st>>>(A);
  cudaError_t e = cudaGetLastError();
  cudaFreeAsync(scratch, st);
  if (e != cudaSuccess) return fail(BIMINE_E_CUDA, std::string("nw_kernel: ") + cudaGetErrorString(e));
  return BIMINE_OK;
}

NwArgs nw_args_base(const double *sim, const int64_t *sim_off, const int32_t *pn, const int32_t *pm,
                    int64_t n_problems, int32_t n_settings, const double *gap, double mismatch, double bonus) {
  NwArgs A;
  memset(&A, 0, sizeof(A));
  A.sim = sim;
  A.sim_off = sim_off;
  A.pair_n = pn;
  A.pair_m = pm;
  A.problem_ids = nullptr;
  A.n_problems = n_problems;
  A.n_settings = n_settings;
  A.gap = gap;
  A.mismatch = mismatch;
  A.bonus = bonus;
  return A;
}

}  // namespace

extern "C" {

int bimine_nw_mine_batch(const double *sim_dev, const int64_t *pair_sim_off, const int32_t *pair_n,
                         const int32_t *pair_m, int64_t n_pairs, int32_t max_n, int32_t max_m, int32_t n_settings,
                         const double *gap_dev, const double *threshold_dev, double mismatch, double bonus,
                         const int64_t *out_off_dev, bimine_match *matches_dev, int32_t *counts_dev,
                         double *score_dev, void *stream) {
  if (!sim_dev || !pair_sim_off || !pair_n || !pair_m || !gap_dev || !threshold_dev || !out_off_dev ||
      !matches_dev || !counts_dev || n_settings < 1)
    return fail(BIMINE_E_ARG, "bimine_nw_mine_batch: bad arguments");
  if (n_pairs == 0) return BIMINE_OK;
  if (max_n < 1 || max_m < 1) return fail(BIMINE_E_ARG, "bimine_nw_mine_batch: empty matrix");
  NwArgs A = nw_args_base(sim_dev, pair_sim_off, pair_n, pair_m, n_pairs * n_settings, n_settings, gap_dev,
                          mismatch, bonus);
  A.threshold = threshold_dev;
  A.out_off = out_off_dev;
  A.matches = matches_dev;
  A.counts = counts_dev;
  A.score = score_dev;
  return launch_nw<kNwMine>(A, max_n, max_m, as_stream(stream));
}

int bimine_mine_batch(const bimine_dict *dict, const double *model, const bimine_batch *b, const bimine_plan *plan,
                      double gap, double threshold, double mismatch, double bonus, double *sim_dev,
                      const int64_t *out_off_dev, bimine_match *matches_dev, int32_t *counts_dev, double *score_dev,
                      void *stream) {
  if (!out_off_dev || !matches_dev || !counts_dev) return fail(BIMINE_E_ARG, "bimine_mine_batch: null output");
  if (!b || b->n_pairs == 0) return BIMINE_OK;
  cudaStream_t st = as_stream(stream);
  pool_setup();
  int rc = launch_scores(dict, model, b, plan, sim_dev, st);
  if (rc != BIMINE_OK) return rc;
  BIMINE_CUDA(gate_wait_all(st));
  // NW + traceback + filter: pairs of at most 64 x 64 sentences one warp
  // each; the plan's larger pairs on the cluster kernel (one setting,
  // gap and threshold by value)
  NwArgs A = nw_args_base(sim_dev, b->pair_sim_off, b->pair_n, b->pair_m, b->n_pairs, 1, nullptr, mismatch, bonus);
  A.gap1 = gap;
  A.threshold1 = threshold;
  A.out_off = out_off_dev;
  A.matches = matches_dev;
  A.counts = counts_dev;
  A.score = score_dev;
  if (plan->n_large < b->n_pairs) {
    NwArgs As = A;
    As.small_only = plan->n_large > 0;
    rc = launch_nw<kNwMine>(As, std::min(plan->max_n, kPairMax), std::min(plan->max_m, kPairMax), st);
    if (rc != BIMINE_OK) return rc;
  }
  if (plan->n_large > 0) {
    NwArgs Al = A;
    const int64_t at = 3 * plan->n_tiles + plan->n_long;
    Al.problem_ids = plan->work + at;
    Al.n_problems = plan->n_large;
    const int64_t *hw = plan->work_host;
    rc = launch_nw<kNwMine>(Al, plan->max_n, plan->max_m, st, hw ? hw + at : nullptr,
                            hw ? hw + at + plan->n_large : nullptr);
  }
  return rc;
}

int bimine_nw_steps_batch(const double *sim_dev, const int64_t *pair_sim_off, const int32_t *pair_n,
                          const int32_t *pair_m, int64_t n_pairs, int32_t max_n, int32_t max_m,
                          const double *gap_dev, double mismatch, double bonus, const int64_t *step_off_dev,
                          uint8_t *steps_dev, int32_t *n_steps_dev, double *score_dev, void *stream) {
  if (!sim_dev || !pair_sim_off || !pair_n || !pair_m || !gap_dev || !step_off_dev || !steps_dev || !n_steps_dev)
    return fail(BIMINE_E_ARG, "bimine_nw_steps_batch: bad arguments");
  if (n_pairs == 0) return BIMINE_OK;
  if (max_n < 1 || max_m < 1) return fail(BIMINE_E_ARG, "bimine_nw_steps_batch: empty matrix");
  // one setting per pair: problem q == pair q, gap_dev[q]
  NwArgs A = nw_args_base(sim_dev, pair_sim_off, pair_n, pair_m, n_pairs, 1, gap_dev, mismatch, bonus);
  A.gap_per_problem = 1;
  A.step_off = step_off_dev;
  A.steps = steps_dev;
  A.n_steps = n_steps_dev;
  A.score = score_dev;
  return launch_nw<kNwSteps>(A, max_n, max_m, as_stream(stream));
}

int bimine_compact_matches(const bimine_match *matches_dev, const int64_t *out_off_dev, const int32_t *counts_dev,
                           int64_t n_problems, int64_t *match_base_dev, bimine_match *compact_dev,
                           int64_t *total_dev, void *stream) {
  if (n_problems == 0) {
    BIMINE_CUDA(cudaMemsetAsync(total_dev, 0, sizeof(int64_t), as_stream(stream)));
    return BIMINE_OK;
  }
  scan_counts_kernel<<<1, 1024, 0, as_stream(stream)>>>(counts_dev, n_problems, match_base_dev, total_dev);
  BIMINE_CUDA(cudaGetLastError());
  const int64_t threads = n_problems * 32;
  gather_matches_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, as_stream(stream)>>>(
      matches_dev, out_off_dev, counts_dev, match_base_dev, n_problems, compact_dev);
  BIMINE_CUDA(cudaGetLastError());
  return BIMINE_OK;
}

int bimine_agreement_batch(const bimine_match *matches_dev, const int64_t *out_off_dev, const int32_t *counts_dev,
                           int64_t n_pairs, int32_t n_settings, const int32_t *ref_ij_dev, const int64_t *ref_off_dev,
                           const int32_t *ref_len_dev, int32_t max_k, int32_t max_r, int32_t *matched_dev,
                           void *stream) {
  if (!matches_dev || !out_off_dev || !counts_dev || !ref_ij_dev || !ref_off_dev || !ref_len_dev || !matched_dev ||
      n_settings < 1)
    return fail(BIMINE_E_ARG, "bimine_agreement_batch: bad arguments");
  const int64_t n = n_pairs * n_settings;
  if (n == 0) return BIMINE_OK;
  pool_setup();
  AgreeArgs A;
  A.matches = matches_dev;
  A.out_off = out_off_dev;
  A.counts = counts_dev;
  A.n_problems = n;
  A.n_settings = n_settings;
  A.ref_ij = ref_ij_dev;
  A.ref_off = ref_off_dev;
  A.ref_len = ref_len_dev;
  A.matched = matched_dev;
  const int mk = std::max(1, max_k), mr = std::max(1, max_r);
  A.row_doubles_per_warp = ((mr + 1) + 1) & ~1;
  const int64_t dw = (int64_t)(mk + 1) * ((mr >> 4) + 1);
  A.dir_words_per_warp = dw;
  A.g_rows = nullptr;
  A.g_dirs = nullptr;
  cudaStream_t st = as_stream(stream);
  const size_t per_warp = (size_t)A.row_doubles_per_warp * 8 + (size_t)dw * 4;
  const size_t per_block = (size_t)kNwWarpsPerBlock * per_warp;
  if (per_block <= kNwSmemPerBlockMax) {
    BIMINE_CUDA(cudaFuncSetAttribute(agree_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)per_block));
    agree_kernel<<<(unsigned)((n + kNwWarpsPerBlock - 1) / kNwWarpsPerBlock), kNwWarpsPerBlock * 32, per_block,
                   st>>>(A);
    BIMINE_CUDA(cudaGetLastError());
    return BIMINE_OK;
  }
  // long lists: each launched warp gets a global scratch slot (<= ~2 GiB in all)
  int64_t warps = std::min<int64_t>(n, (int64_t)num_sms() * 16);
  warps = std::max<int64_t>(1, std::min<int64_t>(warps, (int64_t)(((size_t)2 << 30) / per_warp)));
  const int64_t blocks = (warps + kNwWarpsPerBlock - 1) / kNwWarpsPerBlock;
  const int64_t slots = blocks * kNwWarpsPerBlock;
  char *scratch = nullptr;
  BIMINE_CUDA(cudaMallocAsync((void **)&scratch, per_warp * slots + 16, st));
  A.g_rows = (double *)scratch;
  A.g_dirs = (uint32_t *)(scratch + (size_t)A.row_doubles_per_warp * 8 * slots);
  agree_kernel<<<(unsigned)blocks, kNwWarpsPerBlock * 32, 0, st>>>(A);
  const cudaError_t e = cudaGetLastError();
  cudaFreeAsync(scratch, st);
  if (e != cudaSuccess) return fail(BIMINE_E_CUDA, std::string("agree_kernel: ") + cudaGetErrorString(e));
  return BIMINE_OK;
}

// ------------------------------------------------------------------------
// B1 shim: the reference's _nwcore.nw_fill / nw_fill_wavefront
// ------------------------------------------------------------------------

int bimine_nw_fill(double *dp, const double *sim, int64_t n, int64_t m, double mismatch, double bonus, double gap,
                   void *stream) {
  if (!dp || !sim || n < 1 || m < 1) return fail(BIMINE_E_ARG, "bimine_nw_fill: bad arguments");
  if (n > 0x7fffffff || m > 0x7fffffff) return fail(BIMINE_E_LIMIT, "bimine_nw_fill: too large");
  pool_setup();
  cudaStream_t st = as_stream(stream);
  const size_t sim_b = sizeof(double) * n * m, dp_b = sizeof(double) * (n + 1) * (m + 1);
  const size_t small_b = 64;
  char *buf = nullptr;
  BIMINE_CUDA(cudaMallocAsync((void **)&buf, sim_b + dp_b + small_b, st));
  double *d_sim = (double *)buf, *d_dp = (double *)(buf + sim_b);
  char *sm = buf + sim_b + dp_b;
  int64_t h_off = 0;
  int32_t h_n = (int32_t)n, h_m = (int32_t)m;
  // small parameter block: sim_off | n | m | gap
  char host_small[64];
  memcpy(host_small, &h_off, 8);
  memcpy(host_small + 8, &h_n, 4);
  memcpy(host_small + 12, &h_m, 4);
  memcpy(host_small + 16, &gap, 8);
  BIMINE_CUDA(cudaMemcpyAsync(sm, host_small, 24, cudaMemcpyHostToDevice, st));
  BIMINE_CUDA(cudaMemcpyAsync(d_sim, sim, sim_b, cudaMemcpyHostToDevice, st));
  BIMINE_CUDA(cudaMemcpyAsync(d_dp, dp, dp_b, cudaMemcpyHostToDevice, st));
  NwArgs A = nw_args_base(d_sim, (const int64_t *)sm, (const int32_t *)(sm + 8), (const int32_t *)(sm + 12), 1, 1,
                          (const double *)(sm + 16), mismatch, bonus);
  A.table = d_dp;
  int rc = launch_nw<kNwTable>(A, (int32_t)n, (int32_t)m, st);
  if (rc != BIMINE_OK) {
    cudaFreeAsync(buf, st);
    return rc;
  }
  BIMINE_CUDA(cudaMemcpyAsync(dp, d_dp, dp_b, cudaMemcpyDeviceToHost, st));
  BIMINE_CUDA(cudaFreeAsync(buf, st));
  BIMINE_CUDA(cudaStreamSynchronize(st));
  return BIMINE_OK;
}

int bimine_nw_fill_wavefront(double *dp, const double *sim, int64_t n, int64_t m, double mismatch, double bonus,
                             double gap, int workers, void *stream) {
  if (workers < 1) return fail(BIMINE_E_ARG, "workers must be >= 1");
  return bimine_nw_fill(dp, sim, n, m, mismatch, bonus, gap, stream);
}

// ------------------------------------------------------------------------
// end to end from host buffers
// ------------------------------------------------------------------------

std::mutex &mine_host_mutex() {
  static std::mutex mu;
  static std::map<int, std::unique_ptr<std::mutex>> per_dev;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  std::unique_ptr<std::mutex> &m = per_dev[dev];
  if (!m) m.reset(new std::mutex());
  return *m;
}

// Under lazy module loading (CUDA_MODULE_LOADING=LAZY, the CUDA 12 default)
// a kernel is loaded at its first launch, and that load can wait for the
// device to go idle.  bimine_mine_host's score kernel waits on copies still
// in flight, so a first launch of another kernel while it waits (NW,
// compaction, the offsets scan) risks a deadlock -- seen on B200 with an
// earlier-launched score kernel.  Every kernel the path can launch is loaded
// here first, once per device.
cudaError_t preload_kernels(cudaStream_t st) {
  static std::mutex mu;
  static std::map<int, bool> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  if (done[dev]) return cudaSuccess;
  const void *fns[] = {
      (const void *)pair_kernel<false, false>, (const void *)pair_kernel<false, true>,
      (const void *)pair_kernel<true, false>, (const void *)pair_kernel<true, true>,
      (const void *)score_kernel, (const void *)build_term_tables,
      (const void *)nw_kernel<kNwMine>, (const void *)nw_kernel<kNwSteps>, (const void *)nw_kernel<kNwTable>,
      (const void *)nw_big_kernel<kNwMine, kBigW>, (const void *)nw_big_kernel<kNwSteps, kBigW>,
      (const void *)nw_big_kernel<kNwTable, kBigW>, (const void *)nw_big_traceback_kernel<kNwMine>,
      (const void *)nw_big_traceback_kernel<kNwSteps>, (const void *)nw_big_traceback_kernel<kNwTable>,
      (const void *)nw_diag_kernel, (const void *)uniform_offsets_kernel, (const void *)scan_counts_kernel,
      (const void *)gather_matches_kernel, (const void *)agree_kernel, (const void *)widen_u16_kernel};
  cudaFuncAttributes fa;
  for (const void *f : fns) {
    const cudaError_t e = cudaFuncGetAttributes(&fa, f);  // loads the kernel
    if (e != cudaSuccess) return e;
  }
  // CUB's scan kernels are not nameable here: one scan of one length loads them
  size_t bytes = 0;
  cudaError_t e = offsets_from_lengths(nullptr, nullptr, 1, nullptr, &bytes, st);
  char *buf = nullptr;
  e = e ? e : cudaMallocAsync((void **)&buf, 64 + bytes, st);
  e = e ? e : cudaMemsetAsync(buf, 0, 64, st);
  e = e ? e : offsets_from_lengths((const int32_t *)buf, (int64_t *)(buf + 8), 1, buf + 64, &bytes, st);
  if (buf) cudaFreeAsync(buf, st);
  e = e ? e : cudaStreamSynchronize(st);
  if (e == cudaSuccess) done[dev] = true;
  return e;
}

int bimine_mine_host(const bimine_dict *dict, const double *model, const bimine_batch *h, double gap,
                     double threshold, double mismatch, double bonus, int32_t *counts_host,
                     bimine_match *matches_host, int64_t capacity, int64_t *total_host, double *sim_host,
                     void *stream) {
  if (!dict || !model || !h || !counts_host || !total_host) return fail(BIMINE_E_ARG, "bimine_mine_host: null");
  const int64_t P = h->n_pairs, S = h->n_sentences, T = h->n_tokens;
  *total_host = 0;
  if (P == 0) return BIMINE_OK;
  if (h->sent_bytes != 0 && h->sent_bytes != 2 && h->sent_bytes != 4)
    return fail(BIMINE_E_ARG, "bimine_mine_host: sent_bytes must be 2 or 4");
  const bool narrow = h->sent_bytes == 2;  // uint16 sentence arrays: half the upload, widened on the device
  pool_setup();
  cudaStream_t st = as_stream(stream);
  BIMINE_CUDA(preload_kernels(st));
  // One call per device at a time: the calls share the device's copy
  // stream, and a call's score CTAs (persistent, possibly on every SM) wait
  // for uploads that must not queue behind another call's scan kernel.
  std::unique_lock<std::mutex> call_lock(mine_host_mutex());
  // Uploads start at once on a copy stream: pair and sentence arrays, then
  // the tokens in `nt` equal pieces, a device counter bumped after each
  // (1 = pairs + sentences, 1 + j = token pieces 0..j-1).  The score kernel
  // is launched right behind them; each of its CTAs derives the counter
  // value its pair needs (pair_kernel.cuh, self gate).  Meanwhile host
  // threads check and plan the batch in chunks of pairs; the rest of the
  // path follows the plan.
  static const int max_chunks = [] {
    const char *v = getenv("BIMINE_E2E_CHUNKS");
    return v ? std::max(1, atoi(v)) : 16;
  }();
  static const int64_t min_tokens = [] {
    const char *v = getenv("BIMINE_E2E_MIN_TOKENS");
    return v ? std::max<int64_t>(1, atoll(v)) : (int64_t)1 << 20;
  }();
  const int nt = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)max_chunks, T / min_tokens));
  static const int max_analysis = [] {
    const char *v = getenv("BIMINE_E2E_ANALYSIS_THREADS");
    return v ? std::max(1, atoi(v)) : 8;
  }();
  const int nc = (int)std::max<int64_t>(1, std::min<int64_t>(max_analysis, P));  // analysis threads
  std::vector<int64_t> cut(nc + 1), tcut(nt + 1);
  for (int k = 0; k <= nc; ++k) cut[k] = P * k / nc;
  for (int j = 0; j <= nt; ++j) tcut[j] = T * j / nt;
  // pinned staging: slot offsets [P] | counter values [nt + 1] (int32) | merged work | tiles | piece
  // boundaries
  int64_t work_bound = 0, n_tiles_pre = 0;  // (tiles: the 64x64 blocks of pairs larger than 64x64)
  for (int64_t p = 0; p < P; ++p) {
    const int32_t n = h->pair_n[p], m = h->pair_m[p];
    const int64_t tl = (int64_t)((n + kPairMax - 1) / kPairMax) * ((m + kPairMax - 1) / kPairMax);
    work_bound += 3 + 3 * tl;
    if (n > kPairMax || m > kPairMax) n_tiles_pre += tl;
  }
  const int64_t n_stage = P + (nt + 2) / 2 + 1 + std::max<int64_t>(work_bound, 1) +
                          3 * std::max<int64_t>(n_tiles_pre, 0) + (nt + 1);
  int64_t *staging = (int64_t *)pinned_scratch(sizeof(int64_t) * n_stage);
  if (!staging) return fail(BIMINE_E_CUDA, "bimine_mine_host: pinned staging allocation failed");
  int64_t *out_off = staging;
  int32_t *ready_vals = (int32_t *)(staging + P);
  int64_t *work = staging + P + (nt + 2) / 2 + 1;
  int64_t *tiles_pre = work + std::max<int64_t>(work_bound, 1);
  int64_t *tcut_pinned = tiles_pre + 3 * n_tiles_pre;  // the piece boundaries, uploaded with the pair arrays
  for (int j = 0; j <= nt; ++j) tcut_pinned[j] = tcut[j];
  for (int j = 0; j <= nt; ++j) ready_vals[j] = j + 1;
  // per pair (O(P)): match slots, cells
  int64_t cap = 0, cells = 0;
  for (int64_t p = 0; p < P; ++p) {
    const int32_t n = h->pair_n[p], m = h->pair_m[p];
    if (n < 1 || m < 1) return fail(BIMINE_E_ARG, "bimine_plan_batch: empty document");
    if (h->pair_sim_off[p] < 0) return fail(BIMINE_E_ARG, "bimine_mine_host: negative pair_sim_off");
    out_off[p] = cap;
    cap += std::min(n, m);
    cells = std::max(cells, h->pair_sim_off[p] + (int64_t)n * m);
  }
  if (capacity < cap) return fail(BIMINE_E_ARG, "bimine_mine_host: capacity < sum of min(N, M)");
  // per chunk, on host threads: validity, the sentence / token prefix it
  // reads, its plan (a view: pair arrays from p0, sentence arrays whole)
#ifdef BIMINE_E2E_PROFILE
  auto hclock = [] { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
  const double h0 = hclock();
  double h_an = 0, h_enq = 0, h_mine = 0;
  cudaEvent_t pe[5];
  for (auto &x : pe) cudaEventCreate(&x);
#endif
  // one device arena, carved in 256-byte aligned pieces
  size_t off = 0;
  auto carve = [&](size_t bytes) {
    size_t o = (off + 255) & ~(size_t)255;
    off = o + bytes;
    return o;
  };
  if (h->token_bytes != 0 && h->token_bytes != 3 && h->token_bytes != 4)
    return fail(BIMINE_E_ARG, "bimine_mine_host: token_bytes must be 3 or 4");
  const int tb = h->token_bytes == 3 ? 3 : 4;  // bytes per token id on the wire and on the device
  // the uploaded arrays first (one contiguous front, so a small batch goes
  // up in one transfer), then the device-only buffers
  const size_t o_tok = carve((size_t)tb * T + 4), o_slen = carve(4 * S), o_suniq = carve(4 * S),
               o_schar = carve(4 * S), o_s16 = carve(narrow ? 6 * (size_t)S : 1), o_psrc = carve(8 * P),
               o_pn = carve(4 * P), o_ptgt = carve(8 * P), o_pm = carve(4 * P), o_psim = carve(8 * P),
               o_outoff = carve(8 * P), o_tcut = carve(8 * (size_t)(nt + 1));
  const size_t up_end = off;  // end of the uploaded front
  const size_t o_soff = carve(8 * S), o_sim = carve(8 * cells), o_slots = carve(sizeof(bimine_match) * cap),
               o_counts = carve(4 * P), o_base = carve(8 * P), o_comp = carve(sizeof(bimine_match) * cap),
               o_total = carve(8), o_work = carve(8 * std::max<int64_t>(work_bound, 1)),
               o_tiles = carve(8 * std::max<int64_t>(3 * n_tiles_pre, 1)), o_ready = carve(4);
  // sent_tok_off is not uploaded: the copy stream rebuilds it from sent_len
  // (the usual packed layout); the analysis threads check that the caller's
  // offsets are exactly that, else they are uploaded on `st` before scoring
  size_t scan_bytes = 0;
  BIMINE_CUDA(offsets_from_lengths(nullptr, nullptr, S, nullptr, &scan_bytes, st));
  const size_t o_scan = carve(std::max<size_t>(scan_bytes, 1));
  char *arena = nullptr;
  BIMINE_CUDA(cudaMallocAsync((void **)&arena, off, st));
  cudaStream_t cs = copy_stream();
  cudaEvent_t ev_start = nullptr, ev_all = nullptr, ev_scan = nullptr;
  BIMINE_CUDA(cudaEventCreateWithFlags(&ev_start, cudaEventDisableTiming));
  BIMINE_CUDA(cudaEventCreateWithFlags(&ev_all, cudaEventDisableTiming));
  BIMINE_CUDA(cudaEventCreateWithFlags(&ev_scan, cudaEventDisableTiming));
  auto cleanup = [&]() {
    cudaEventDestroy(ev_start);
    cudaEventDestroy(ev_all);
    cudaEventDestroy(ev_scan);
  };
#ifdef BIMINE_E2E_PROFILE
  cudaEventRecord(pe[0], st);
#endif
  // ---- uploads, issued before any host-side analysis.  Pinned inputs are
  //      enqueued at once; pageable ones are staged through page-locked
  //      memory by an uploader thread (bumping the same device counter), so
  //      that the analysis below and the gated score launch run meanwhile.
  cudaError_t e = cudaMemsetAsync(arena + o_ready, 0, 4, st);
  e = e ? e : cudaEventRecord(ev_start, st);  // arena + ready counter exist
  e = e ? e : cudaStreamWaitEvent(cs, ev_start, 0);
  const bool pg_pairs = is_pageable(h->pair_src) || is_pageable(h->pair_n) || is_pageable(h->pair_tgt) ||
                        is_pageable(h->pair_m) || is_pageable(h->pair_sim_off);
  const bool pg_sent = is_pageable(h->sent_len) || is_pageable(h->sent_uniq) || is_pageable(h->sent_chars);
  const bool pg_tok = is_pageable(h->tokens);
  const bool staged = pg_pairs || pg_sent || pg_tok;
  int dev_id = 0;
  cudaGetDevice(&dev_id);
  std::promise<cudaError_t> phase1;  // sentence arrays, offsets scan and ev_scan enqueued
  std::future<cudaError_t> phase1_done = phase1.get_future();
  cudaError_t up_err = cudaSuccess;
  // A small batch goes up in ONE transfer: its arrays are copied on the
  // host into a page-locked mirror of the arena's front (each transfer of
  // the general path costs ~5-10 us of setup: a one-pair call waited ~70
  // us for a dozen of them before the score kernel could start)
  constexpr size_t kSmallUpload = 512 << 10;
  char *mirror = up_end <= kSmallUpload ? (char *)pinned_grow(tl_mirror, up_end) : nullptr;
  auto upload = [&, dev_id, e0 = e]() {
    cudaSetDevice(dev_id);
    Stager sg(cs, dev_id);
    cudaError_t ue = e0;
    auto H2D = [&](size_t o, const void *src, size_t bytes, bool pg) {
      if (ue == cudaSuccess && bytes) ue = sg.copy(arena + o, src, bytes, pg);
    };
    if (mirror) {
      auto put = [&](size_t o, const void *src, size_t bytes) {
        if (bytes) memcpy(mirror + o, src, bytes);
      };
      put(o_tok, h->tokens, (size_t)tb * T);
      if (narrow) {
        put(o_s16, h->sent_len, 2 * S);
        put(o_s16 + 2 * S, h->sent_uniq, 2 * S);
        put(o_s16 + 4 * S, h->sent_chars, 2 * S);
      } else {
        put(o_slen, h->sent_len, 4 * S);
        put(o_suniq, h->sent_uniq, 4 * S);
        put(o_schar, h->sent_chars, 4 * S);
      }
      put(o_psrc, h->pair_src, 8 * P);
      put(o_pn, h->pair_n, 4 * P);
      put(o_ptgt, h->pair_tgt, 8 * P);
      put(o_pm, h->pair_m, 4 * P);
      put(o_psim, h->pair_sim_off, 8 * P);
      put(o_outoff, out_off, 8 * P);
      put(o_tcut, tcut_pinned, 8 * (size_t)(nt + 1));
      if (ue == cudaSuccess) ue = cudaMemcpyAsync(arena, mirror, up_end, cudaMemcpyHostToDevice, cs);
      if (narrow && ue == cudaSuccess && S > 0) {
        widen_u16_kernel<<<(unsigned)std::min<int64_t>((3 * S + 255) / 256, 4096), 256, 0, cs>>>(
            (const uint16_t *)(arena + o_s16), S, (int32_t *)(arena + o_slen), (int32_t *)(arena + o_suniq),
            (int32_t *)(arena + o_schar));
        ue = cudaGetLastError();
      }
      if (ue == cudaSuccess)
        ue = offsets_from_lengths((const int32_t *)(arena + o_slen), (int64_t *)(arena + o_soff), S,
                                  arena + o_scan, &scan_bytes, cs);
      ue = ue ? ue : cudaEventRecord(ev_scan, cs);
      H2D(o_ready, &ready_vals[nt], 4, false);  // nt + 1: everything is in place
      phase1.set_value(ue);
      ue = ue ? ue : cudaEventRecord(ev_all, cs);
      up_err = ue;
      return;
    }
    H2D(o_psrc, h->pair_src, 8 * P, pg_pairs);
    H2D(o_pn, h->pair_n, 4 * P, pg_pairs);
    H2D(o_ptgt, h->pair_tgt, 8 * P, pg_pairs);
    H2D(o_pm, h->pair_m, 4 * P, pg_pairs);
    H2D(o_psim, h->pair_sim_off, 8 * P, pg_pairs);
    H2D(o_outoff, out_off, 8 * P, false);
    if (narrow) {
      H2D(o_s16, h->sent_len, 2 * S, pg_sent);
      H2D(o_s16 + 2 * S, h->sent_uniq, 2 * S, pg_sent);
      H2D(o_s16 + 4 * S, h->sent_chars, 2 * S, pg_sent);
      if (ue == cudaSuccess && S > 0) {
        widen_u16_kernel<<<(unsigned)std::min<int64_t>((3 * S + 255) / 256, 4096), 256, 0, cs>>>(
            (const uint16_t *)(arena + o_s16), S, (int32_t *)(arena + o_slen), (int32_t *)(arena + o_suniq),
            (int32_t *)(arena + o_schar));
        ue = cudaGetLastError();
      }
    } else {
      H2D(o_slen, h->sent_len, 4 * S, pg_sent);
      H2D(o_suniq, h->sent_uniq, 4 * S, pg_sent);
      H2D(o_schar, h->sent_chars, 4 * S, pg_sent);
    }
    H2D(o_tcut, tcut_pinned, 8 * (size_t)(nt + 1), false);
    if (ue == cudaSuccess)
      ue = offsets_from_lengths((const int32_t *)(arena + o_slen), (int64_t *)(arena + o_soff), S, arena + o_scan,
                                &scan_bytes, cs);
    ue = ue ? ue : cudaEventRecord(ev_scan, cs);
    H2D(o_ready, &ready_vals[0], 4, false);  // 1: pairs and sentences are in place
    phase1.set_value(ue);
    for (int j = 0; j < nt; ++j) {
      H2D(o_tok + (size_t)tb * tcut[j], (const char *)h->tokens + (size_t)tb * tcut[j],
          (size_t)tb * (tcut[j + 1] - tcut[j]), pg_tok);
      H2D(o_ready, &ready_vals[j + 1], 4, false);  // j + 2: token pieces 0..j
    }
    ue = ue ? ue : cudaEventRecord(ev_all, cs);
    const cudaError_t de = sg.drain();  // the ring is free for the next upload
    up_err = ue ? ue : de;
  };
  std::thread uploader;
  if (staged && !mirror) {
    uploader = std::thread(upload);
  } else {
    upload();
  }
  auto join_uploader = [&]() {
    if (uploader.joinable()) uploader.join();
  };
#ifdef BIMINE_E2E_PROFILE
  cudaEventRecord(pe[1], cs);
  h_enq = hclock() - h0;
#endif
  auto abort_with = [&](int code, const std::string &msg) {
    join_uploader();
    cudaStreamSynchronize(cs);
    cudaFreeAsync(arena, st);
    cudaStreamSynchronize(st);
    cleanup();
    return fail(code, msg);
  };
  if (e != cudaSuccess) return abort_with(BIMINE_E_CUDA, std::string("bimine_mine_host H2D: ") + cudaGetErrorString(e));
  // ---- the score kernel goes now, before the host has looked at the
  //      batch: its CTAs bounds-check their pairs and derive their upload
  //      gates themselves (pair_kernel.cuh, self gate), and the analysis
  //      below runs beside it.  The tiles of pairs larger than 64x64 come
  //      from the shapes alone.  The launch follows the offsets scan on the
  //      copy stream: waiting CTAs may fill every SM.
  bimine_batch d;
  d.n_pairs = P;
  d.n_sentences = S;
  d.n_tokens = T;
  d.tokens = (const int32_t *)(arena + o_tok);
  d.token_bytes = tb;
  d.sent_tok_off = (const int64_t *)(arena + o_soff);
  d.sent_len = (const int32_t *)(arena + o_slen);
  d.sent_uniq = (const int32_t *)(arena + o_suniq);
  d.sent_chars = (const int32_t *)(arena + o_schar);
  d.pair_src = (const int64_t *)(arena + o_psrc);
  d.pair_n = (const int32_t *)(arena + o_pn);
  d.pair_tgt = (const int64_t *)(arena + o_ptgt);
  d.pair_m = (const int32_t *)(arena + o_pm);
  d.pair_sim_off = (const int64_t *)(arena + o_psim);
  d.sent_bytes = 4;  // (widened on the device)
  UploadGate gate{(const int32_t *)(arena + o_ready), ev_all, join_uploader};
  gate.n_sentences = S;
  gate.n_tokens = T;
  gate.n_pieces = nt;
  gate.piece_start = (const int64_t *)(arena + o_tcut);
  {
    int64_t t = 0;
    for (int64_t p = 0; p < P; ++p) {
      const int32_t n = h->pair_n[p], m = h->pair_m[p];
      if (n > kPairMax || m > kPairMax)
        for (int32_t i0 = 0; i0 < n; i0 += kPairMax)
          for (int32_t j0 = 0; j0 < m; j0 += kPairMax) {
            tiles_pre[3 * t] = p;
            tiles_pre[3 * t + 1] = i0;
            tiles_pre[3 * t + 2] = j0;
            ++t;
          }
    }
    if (n_tiles_pre) e = cudaMemcpyAsync(arena + o_tiles, tiles_pre, 8 * 3 * n_tiles_pre, cudaMemcpyHostToDevice, st);
    const cudaError_t e1 = phase1_done.get();  // the uploader has enqueued the offsets scan
    e = e ? e : e1;
    e = e ? e : cudaStreamWaitEvent(st, ev_scan, 0);
    if (e != cudaSuccess) return abort_with(BIMINE_E_CUDA, std::string("bimine_mine_host: ") + cudaGetErrorString(e));
    const int rc0 = launch_pair_kernel(dict, model, &d, (const int64_t *)(arena + o_tiles), n_tiles_pre, cells,
                                       (double *)(arena + o_sim), st, nullptr, &gate);
    if (rc0 != BIMINE_OK) {
      const std::string msg = g_error;
      return abort_with(rc0, msg);
    }
    gate.pair_launched = true;
  }
  // ---- per chunk of pairs, on host threads: validity, each pair's counter
  //      value, the chunk's plan (a view: pair arrays from p0, sentence arrays whole)
  struct ChunkInfo {
    int rc = BIMINE_OK;
    std::string err;
    bimine_plan plan;
    std::vector<int64_t> work;
    bool packed = true;  // sentences [S k / nc, S (k+1) / nc) are at the rebuilt offsets
  };
  std::vector<ChunkInfo> ci(nc);
  // the host's own reads of the sentence arrays, in whichever width they are
  const uint16_t *const n_len = (const uint16_t *)h->sent_len, *const n_uniq = (const uint16_t *)h->sent_uniq;
  auto sent_len_at = [&](int64_t x) -> int32_t { return narrow ? (int32_t)n_len[x] : h->sent_len[x]; };
  auto analyse = [&](int k) {
    ChunkInfo &c = ci[k];
    {
      const int64_t s0 = S * k / nc, s1 = S * (k + 1) / nc;
      const int64_t *so = h->sent_tok_off;
      bool ok = s0 > 0 || S == 0 || so[0] == 0;
      for (int64_t x = s0; ok && x + 1 < s1 + (s1 < S ? 1 : 0); ++x) ok = so[x + 1] == so[x] + sent_len_at(x);
      c.packed = ok;
    }
    const int64_t p0 = cut[k], p1 = cut[k + 1];
    int64_t wcap = 3 * (p1 - p0);
    for (int64_t p = p0; p < p1; ++p) {
      const int32_t n = h->pair_n[p], m = h->pair_m[p];
      wcap += 3 * (int64_t)((n + kPairMax - 1) / kPairMax) * ((m + kPairMax - 1) / kPairMax);
      int64_t te = 0;
      for (int pass = 0; pass < 2; ++pass) {
        const int64_t s0 = pass ? h->pair_tgt[p] : h->pair_src[p];
        const int32_t cnt = pass ? m : n;
        if (s0 < 0 || s0 + cnt > S) {
          c.rc = BIMINE_E_ARG;
          c.err = "bimine_mine_host: sentence index out of range";
          return;
        }
        for (int32_t q = 0; q < cnt; ++q) {
          const int32_t len = sent_len_at(s0 + q);
          if (len < 1) {
            c.rc = BIMINE_E_ARG;
            c.err = "bimine_mine_host: empty sentence";
            return;
          }
          te = std::max(te, h->sent_tok_off[s0 + q] + len);
        }
      }
      if (te > T) {
        c.rc = BIMINE_E_ARG;
        c.err = "bimine_mine_host: token range out of bounds";
        return;
      }
    }
    bimine_batch hv = *h;
    hv.n_pairs = p1 - p0;
    hv.pair_src = h->pair_src + p0;
    hv.pair_n = h->pair_n + p0;
    hv.pair_tgt = h->pair_tgt + p0;
    hv.pair_m = h->pair_m + p0;
    hv.pair_sim_off = h->pair_sim_off + p0;
    c.work.resize(std::max<int64_t>(wcap, 1));
    c.rc = narrow ? plan_batch_t<uint16_t>(&hv, n_len, n_uniq, c.work.data(), wcap, &c.plan)
                  : plan_batch_t<int32_t>(&hv, h->sent_len, h->sent_uniq, c.work.data(), wcap, &c.plan);
    if (c.rc != BIMINE_OK) c.err = g_error;  // this thread's message
  };
  {
    std::vector<std::thread> th;
    for (int k = 1; k < nc; ++k) th.emplace_back(analyse, k);
    analyse(0);
    for (auto &t : th) t.join();
  }
  for (int k = 0; k < nc; ++k)
    if (ci[k].rc != BIMINE_OK) return abort_with(ci[k].rc, ci[k].err);
  bool packed = true;
  for (int k = 0; k < nc; ++k) packed = packed && ci[k].packed;
  if (!packed) {  // the caller's own layout: overwrite the rebuilt offsets and score again
    e = cudaMemcpyAsync(arena + o_soff, h->sent_tok_off, 8 * S, cudaMemcpyHostToDevice, st);
    gate.pair_launched = false;
  }
  if (e != cudaSuccess) return abort_with(BIMINE_E_CUDA, std::string("bimine_mine_host: ") + cudaGetErrorString(e));
#ifdef BIMINE_E2E_PROFILE
  h_an = hclock() - h0;
#endif
  // merged plan: tiles, then long pairs, then large pairs (chunk order, global pair ids)
  bimine_plan plan;
  memset(&plan, 0, sizeof(plan));
  for (int k = 0; k < nc; ++k) {
    const bimine_plan &q = ci[k].plan;
    plan.max_n = std::max(plan.max_n, q.max_n);
    plan.max_m = std::max(plan.max_m, q.max_m);
    plan.max_uniq = std::max(plan.max_uniq, q.max_uniq);
    plan.max_len = std::max(plan.max_len, q.max_len);
    plan.long_max_n = std::max(plan.long_max_n, q.long_max_n);
    plan.long_max_m = std::max(plan.long_max_m, q.long_max_m);
    plan.n_tiles += q.n_tiles;
    plan.n_long += q.n_long;
    plan.n_large += q.n_large;
    plan.n_cells = std::max(plan.n_cells, q.n_cells);
  }
  plan.work_len = 3 * plan.n_tiles + plan.n_long + 3 * plan.n_large;
  {
    int64_t t = 0, l = 3 * plan.n_tiles, g = l + plan.n_long, gd = g + plan.n_large;
    for (int k = 0; k < nc; ++k) {
      const bimine_plan &q = ci[k].plan;
      const int64_t *w = ci[k].work.data(), p0 = cut[k];
      for (int64_t x = 0; x < q.n_tiles; ++x, ++t) {
        work[3 * t] = w[3 * x] + p0;
        work[3 * t + 1] = w[3 * x + 1];
        work[3 * t + 2] = w[3 * x + 2];
      }
      for (int64_t x = 0; x < q.n_long; ++x) work[l++] = w[3 * q.n_tiles + x] + p0;
      const int64_t *lw = w + 3 * q.n_tiles + q.n_long;
      for (int64_t x = 0; x < q.n_large; ++x) {
        work[g++] = lw[x] + p0;
        work[gd++] = lw[q.n_large + 2 * x];
        work[gd++] = lw[q.n_large + 2 * x + 1];
      }
    }
  }
  e = cudaMemcpyAsync(arena + o_work, work, 8 * plan.work_len, cudaMemcpyHostToDevice, st);
  int rc = BIMINE_OK;
  if (e == cudaSuccess) {
    plan.work = (const int64_t *)(arena + o_work);
    plan.work_host = work;
    tl_gate = &gate;
    rc = bimine_mine_batch(dict, model, &d, &plan, gap, threshold, mismatch, bonus, (double *)(arena + o_sim),
                           (const int64_t *)(arena + o_outoff), (bimine_match *)(arena + o_slots),
                           (int32_t *)(arena + o_counts), nullptr, stream);
    tl_gate = nullptr;
    join_uploader();
    if (rc == BIMINE_OK && up_err != cudaSuccess)
      rc = fail(BIMINE_E_CUDA, std::string("bimine_mine_host H2D: ") + cudaGetErrorString(up_err));
    // (every later launch on st follows NW, which waited for all uploads)
#ifdef BIMINE_E2E_PROFILE
    cudaEventRecord(pe[2], st);
    h_mine = hclock() - h0;
#endif
  } else {
    join_uploader();
    rc = fail(BIMINE_E_CUDA, std::string("bimine_mine_host H2D: ") + cudaGetErrorString(e));
  }
  if (rc == BIMINE_OK)
    rc = bimine_compact_matches((const bimine_match *)(arena + o_slots), (const int64_t *)(arena + o_outoff),
                                (const int32_t *)(arena + o_counts), P, (int64_t *)(arena + o_base),
                                (bimine_match *)(arena + o_comp), (int64_t *)(arena + o_total), stream);
  if (rc != BIMINE_OK) {
    cudaStreamSynchronize(cs);
    cudaStreamSynchronize(st);
    cudaFreeAsync(arena, st);
    cudaStreamSynchronize(st);
    cleanup();
    return rc;
  }
#ifdef BIMINE_E2E_PROFILE
  cudaEventRecord(pe[3], st);
#endif
  e = cudaMemcpyAsync(counts_host, arena + o_counts, 4 * P, cudaMemcpyDeviceToHost, st);
  e = e ? e : cudaMemcpyAsync(total_host, arena + o_total, 8, cudaMemcpyDeviceToHost, st);
  if (sim_host && !e) e = cudaMemcpyAsync(sim_host, arena + o_sim, 8 * cells, cudaMemcpyDeviceToHost, st);
  e = e ? e : cudaStreamSynchronize(st);
  if (!e && *total_host > 0 && matches_host)
    e = cudaMemcpyAsync(matches_host, arena + o_comp, sizeof(bimine_match) * (*total_host), cudaMemcpyDeviceToHost,
                        st);
  cudaFreeAsync(arena, st);
#ifdef BIMINE_E2E_PROFILE
  cudaEventRecord(pe[4], st);
#endif
  e = e ? e : cudaStreamSynchronize(st);
  cleanup();
#ifdef BIMINE_E2E_PROFILE
  {
    float t[5];
    for (int k = 1; k < 5; ++k) cudaEventElapsedTime(&t[k], pe[0], pe[k]);
    fprintf(stderr, "e2e host: analysed %.3f enqueued copies %.3f enqueued mine %.3f done %.3f | device from first op: copies done %.3f, mine+nw done %.3f, compaction done %.3f, d2h done %.3f\n",
            h_an, h_enq, h_mine, hclock() - h0, t[1], t[2], t[3], t[4]);
    for (auto &x : pe) cudaEventDestroy(x);
  }
#endif
  if (e != cudaSuccess) return fail(BIMINE_E_CUDA, std::string("bimine_mine_host: ") + cudaGetErrorString(e));
  return BIMINE_OK;
}

#ifdef BIMINE_PROF_GLOBAL
// profiling builds only: the band end times of the last nw_big_kernel launch
extern "C" int bimine_debug_band_times(uint64_t *out, int n) {
  return cudaMemcpyFromSymbol(out, g_prof_band, sizeof(uint64_t) * std::min(n, 4096)) == cudaSuccess ? 0 : -2;
}
#endif

int bimine_host_copy(void *dst, const void *src, int64_t bytes) {
  if (bytes < 0 || (bytes > 0 && (!dst || !src))) return fail(BIMINE_E_ARG, "bimine_host_copy: bad arguments");
  if (bytes) MemcpyPool::get().copy(dst, src, (size_t)bytes);
  return BIMINE_OK;
}

// ------------------------------------------------------------------------
// test hook: the device exp
// ------------------------------------------------------------------------

__global__ void exp_kernel(const double *x, double *y, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = glibc_exp(x[i], kExpTableDev);
}

int bimine_features_batch(const bimine_dict *dict, const double *model, const bimine_batch *b,
                          const bimine_plan *plan, double *sim_dev, double *features_dev, void *stream) {
  if (!features_dev) return fail(BIMINE_E_ARG, "bimine_features_batch: null features buffer");
  if (plan && plan->n_long > 0)
    return fail(BIMINE_E_LIMIT, "bimine_features_batch: sentences longer than 255 tokens are not supported");
  pool_setup();
  return launch_scores(dict, model, b, plan, sim_dev, as_stream(stream), features_dev);
}

int bimine_lexicon_em(const int32_t *tgt_off, const int32_t *tgt_tok, int64_t n_pairs, int32_t n_src,
                      const int64_t *row_ptr, const int32_t *row_tgt, int64_t n_entries, double *prob,
                      uint8_t *alive, const int64_t *occ_ptr, const int32_t *occ_pair, int32_t iterations,
                      void *stream) {
  if (iterations < 1) return fail(BIMINE_E_ARG, "iterations must be >= 1");
  if (n_src <= 0 || n_entries <= 0 || n_pairs <= 0) return BIMINE_OK;
  if (!tgt_off || !tgt_tok || !row_ptr || !row_tgt || !prob || !alive || !occ_ptr || !occ_pair)
    return fail(BIMINE_E_ARG, "bimine_lexicon_em: null argument");
  pool_setup();
  cudaStream_t st = as_stream(stream);
  EmArgs A;
  A.tgt_off = tgt_off;
  A.tgt_tok = tgt_tok;
  A.n_src = n_src;
  A.row_ptr = row_ptr;
  A.row_tgt = row_tgt;
  A.prob = prob;
  A.alive = alive;
  A.occ_ptr = occ_ptr;
  A.occ_pair = occ_pair;
  char *scratch = nullptr;
  const size_t b_cnt = sizeof(double) * n_entries, b_first = sizeof(int32_t) * n_entries;
  BIMINE_CUDA(cudaMallocAsync((void **)&scratch, b_cnt + 2 * b_first + 16, st));
  A.cnt = (double *)scratch;
  A.first = (int32_t *)(scratch + b_cnt);
  A.order = (int32_t *)(scratch + b_cnt + b_first);
  A.status = (int32_t *)(scratch + b_cnt + 2 * b_first);
  BIMINE_CUDA(cudaMemsetAsync(A.status, 0, sizeof(int32_t), st));
  const int grid = (int)std::min<int64_t>((n_src + kEmWarps - 1) / kEmWarps, (int64_t)num_sms() * 8);
  for (int it = 0; it < iterations; ++it) {
    BIMINE_CUDA(cudaMemsetAsync(A.cnt, 0, b_cnt, st));
    BIMINE_CUDA(cudaMemsetAsync(A.first, 0xff, b_first, st));
    lexicon_em_round<<<grid, kEmWarps * 32, 0, st>>>(A);
    BIMINE_CUDA(cudaGetLastError());
  }
  int32_t status = 0;
  BIMINE_CUDA(cudaMemcpyAsync(&status, A.status, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  BIMINE_CUDA(cudaStreamSynchronize(st));
  cudaFreeAsync(scratch, st);
  if (status) return fail(BIMINE_E_ARG, "bimine_lexicon_em: a target left its row and was looked up again");
  return BIMINE_OK;
}

int bimine_exp_device(const double *x_host, double *y_host, int64_t n) {
  if (n <= 0) return BIMINE_OK;
  double *d = nullptr;
  BIMINE_CUDA(cudaMalloc(&d, 16 * n));
  cudaError_t e = cudaMemcpy(d, x_host, 8 * n, cudaMemcpyHostToDevice);
  if (!e) {
    exp_kernel<<<(unsigned)((n + 255) / 256), 256>>>(d, d + n, n);
    e = cudaGetLastError();
  }
  if (!e) e = cudaMemcpy(y_host, d + n, 8 * n, cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e) return fail(BIMINE_E_CUDA, std::string("bimine_exp_device: ") + cudaGetErrorString(e));
  return BIMINE_OK;
}

}  // extern "C"
