// Device buffers (grow-only, so repeated setups reuse their arenas without
// cudaMalloc/cudaFree inside timed steps) and an opt-in stage profiler
// (BDDC_B200_PROFILE=1 prints CUDA-event stage times to stderr).
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

namespace b200 {

void cuda_check(cudaError_t e, const char* file, int line);
#define CK(x) ::b200::cuda_check((x), __FILE__, __LINE__)

template <class T>
struct DBuf {
  T* p = nullptr;
  std::size_t n = 0, cap = 0;
  bool owned = true;  // false: a view into another allocation (a stage arena region)
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { release(); }
  void release() {
    if (p && owned) cudaFree(p);
    p = nullptr;
    n = cap = 0;
    owned = true;
  }
  void alloc(std::size_t k) {
    if (k > cap) {
      release();
      CK(cudaMalloc(&p, k * sizeof(T)));
      cap = k;
    }
    n = k;
  }
  /// Use [ptr, ptr + k) of an allocation owned elsewhere.
  void view(T* ptr, std::size_t k) {
    release();
    p = ptr;
    n = cap = k;
    owned = false;
  }
  void upload(const std::vector<T>& v, cudaStream_t s) {
    alloc(v.empty() ? 1 : v.size());
    if (!v.empty()) CK(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s));
  }
  void zero(cudaStream_t s) {
    if (n) CK(cudaMemsetAsync(p, 0, n * sizeof(T), s));
  }
};

/// Grow-only device arena shared by the two scratch-heavy stages of a setup:
/// the pair stage (face eigenproblems) and the preconditioner (transform
/// scratch, transformed leaf fronts, primal tree, root).  The preconditioner
/// region starts at 0; the pair region follows it when the device holds both,
/// else it overlays it (the pair stage then clobbers the preconditioner, which
/// the next set_constraints rebuilds).  No cudaMalloc/cudaFree in steady state.
class StageArena {
 public:
  /// Base of a region of n doubles.  *clobbers_prec: the region overlays the
  /// preconditioner's (or the arena moved), so its contents are lost.
  double* region(bool pair, std::size_t n, bool* clobbers_prec) {
    *clobbers_prec = false;
    std::size_t& mine = pair ? pair_ : prec_;
    if (n > mine) mine = n;
    bool split = prec_ + pair_ <= buf_.cap;  // both fit already: no query
    const bool fits_overlaid = (prec_ > pair_ ? prec_ : pair_) <= buf_.cap;
    if (!split && !fits_overlaid) {  // the arena must grow: side by side if the device holds both
      std::size_t fr = 0, tot = 0;
      if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) fr = 0;
      const double room = double(buf_.cap) * sizeof(double) + double(fr) - 1.5e9;
      split = double(prec_ + pair_) * sizeof(double) <= room;
    }
    const std::size_t total = split ? prec_ + pair_ : (prec_ > pair_ ? prec_ : pair_);
    if (total > buf_.cap) {
      buf_.release();
      buf_.alloc(total);
      *clobbers_prec = true;
    }
    if (pair && !split) *clobbers_prec = true;
    return buf_.p + (pair && split ? prec_ : 0);
  }
  std::size_t capacity() const { return buf_.cap; }

 private:
  DBuf<double> buf_;
  std::size_t prec_ = 0, pair_ = 0;  // largest request of each region so far
};

/// Consecutive views into one region (256-byte aligned parts).
struct RegionPlan {
  std::vector<std::pair<DBuf<double>*, std::size_t>> parts;
  void add(DBuf<double>& b, std::size_t n) { parts.emplace_back(&b, n < 1 ? 1 : n); }
  std::size_t total() const {
    std::size_t t = 0;
    for (const auto& q : parts) t += (q.second + 31) / 32 * 32;
    return t;
  }
  void place(double* base) const {
    std::size_t off = 0;
    for (const auto& q : parts) {
      q.first->view(base + off, q.second);
      off += (q.second + 31) / 32 * 32;
    }
  }
};

/// Many small host->device uploads as one copy: the arrays are packed into a
/// pinned host blob and copied with one cudaMemcpyAsync into a grow-only device
/// blob; every target DBuf becomes a view into it.  Add every array of a setup
/// to the same batch (a grown blob invalidates the previous views), then
/// flush() before the first kernel that reads them.
class UploadBatch {
 public:
  UploadBatch() = default;
  UploadBatch(const UploadBatch&) = delete;
  UploadBatch& operator=(const UploadBatch&) = delete;
  ~UploadBatch() {
    if (host_) cudaFreeHost(host_);
    if (ev_) cudaEventDestroy(ev_);
  }
  template <class T>
  void add(DBuf<T>& target, const std::vector<T>& v) {
    if (items_.empty() && ev_) CK(cudaEventSynchronize(ev_));  // the previous copy out of the host blob is done
    const std::size_t n = v.empty() ? 1 : v.size();
    const std::size_t bytes = n * sizeof(T), span = (bytes + 255) / 256 * 256;
    reserve(used_ + span);
    if (v.empty())
      std::memset(host_ + used_, 0, bytes);
    else
      copy(host_ + used_, v.data(), bytes);
    items_.push_back(Item{reinterpret_cast<void*>(&target), used_, n, &UploadBatch::bind<T>});
    used_ += span;
  }
  /// An array of n elements that `fill` writes straight into the page-locked
  /// blob (no staging vector, no second copy): for the large ones.
  template <class T, class Fill>
  void add_fill(DBuf<T>& target, std::size_t n_in, Fill fill) {
    if (items_.empty() && ev_) CK(cudaEventSynchronize(ev_));
    const std::size_t n = n_in ? n_in : 1;
    const std::size_t bytes = n * sizeof(T), span = (bytes + 255) / 256 * 256;
    reserve(used_ + span);
    if (n_in)
      fill(reinterpret_cast<T*>(host_ + used_));
    else
      std::memset(host_ + used_, 0, bytes);
    items_.push_back(Item{reinterpret_cast<void*>(&target), used_, n, &UploadBatch::bind<T>});
    used_ += span;
  }
  void flush(cudaStream_t st) {
    if (items_.empty()) return;
    dev_.alloc(used_);
    CK(cudaMemcpyAsync(dev_.p, host_, used_, cudaMemcpyHostToDevice, st));
    if (!ev_) CK(cudaEventCreateWithFlags(&ev_, cudaEventDisableTiming));
    CK(cudaEventRecord(ev_, st));
    for (const Item& it : items_) it.bind_fn(it.target, dev_.p + it.off, it.count);
    items_.clear();
    used_ = 0;
  }

 private:
  void reserve(std::size_t need) {
    if (need <= host_cap_) return;
    const std::size_t cap = need + need / 2;
    char* h = nullptr;
    CK(cudaHostAlloc(reinterpret_cast<void**>(&h), cap, cudaHostAllocDefault));
    if (host_) {
      std::memcpy(h, host_, used_);
      CK(cudaFreeHost(host_));
    }
    host_ = h;
    host_cap_ = cap;
  }
  // large arrays are copied by several threads (page-locked destination)
  static void copy(char* dst, const void* src, std::size_t bytes) {
    const std::size_t chunk = std::size_t(1) << 18;  // arrays of 1 MB and more are split
    if (bytes < 4 * chunk) {
      std::memcpy(dst, src, bytes);
      return;
    }
    const long nch = static_cast<long>((bytes + chunk - 1) / chunk);
#pragma omp parallel for schedule(static)
    for (long c = 0; c < nch; ++c) {
      const std::size_t o = c * chunk, len = std::min(chunk, bytes - o);
      std::memcpy(dst + o, static_cast<const char*>(src) + o, len);
    }
  }
  template <class T>
  static void bind(void* target, char* p, std::size_t n) {
    static_cast<DBuf<T>*>(target)->view(reinterpret_cast<T*>(p), n);
  }
  struct Item {
    void* target;
    std::size_t off, count;
    void (*bind_fn)(void*, char*, std::size_t);
  };
  std::vector<Item> items_;
  std::size_t used_ = 0, host_cap_ = 0;
  char* host_ = nullptr;
  cudaEvent_t ev_ = nullptr;
  DBuf<char> dev_;
};

/// Grow-only page-locked host buffer (device-to-host result copies).
template <class T>
struct HBuf {
  T* p = nullptr;
  std::size_t cap = 0;
  T* reserve(std::size_t n) {
    if (n > cap) {
      if (p) CK(cudaFreeHost(p));
      p = nullptr;
      CK(cudaHostAlloc(reinterpret_cast<void**>(&p), std::max<std::size_t>(n, 1) * sizeof(T), cudaHostAllocDefault));
      cap = n;
    }
    return p;
  }
  HBuf() = default;
  HBuf(const HBuf&) = delete;
  HBuf& operator=(const HBuf&) = delete;
  ~HBuf() {
    if (p) cudaFreeHost(p);
  }
};

/// NVTX range over a phase of the hot path (header-only NVTX 3: a no-op unless a
/// profiler is attached).  ncu / nsys can filter on these names:
/// "bddc:analysis", "bddc:eigen", "bddc:set_constraints", "bddc:pcg",
/// "bddc:schur_apply", "bddc:precond_apply", "bddc:step".
class NvtxRange {
 public:
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

/// Host-side stage timer (printed with BDDC_B200_PROFILE=1).
class HostTimer {
 public:
  explicit HostTimer(const char* what) : what_(what), t0_(std::chrono::steady_clock::now()), last_(t0_) {
    const char* e = std::getenv("BDDC_B200_PROFILE");
    on_ = e && *e && *e != '0';
  }
  void mark(const char* name) {
    if (!on_) return;
    const auto now = std::chrono::steady_clock::now();
    char buf[96];
    std::snprintf(buf, sizeof(buf), " %s=%.3fms", name,
                  std::chrono::duration<double, std::milli>(now - last_).count());
    line_ += buf;
    last_ = now;
  }
  ~HostTimer() {
    if (on_) std::fprintf(stderr, "[profile] %s host:%s\n", what_, line_.c_str());
  }

 private:
  const char* what_;
  std::chrono::steady_clock::time_point t0_, last_;
  bool on_ = false;
  std::string line_;
};

class StageProfiler {
 public:
  StageProfiler(const char* what, cudaStream_t st) : what_(what), st_(st) {
    const char* e = std::getenv("BDDC_B200_PROFILE");
    on_ = e && *e && *e != '0';
    if (on_) mark("start");
  }
  /// Collecting mode: stage seconds are added to `sink` (name -> seconds)
  /// instead of printed (Engine::time_operators).
  StageProfiler(const char* what, cudaStream_t st, std::vector<std::pair<std::string, double>>* sink)
      : what_(what), st_(st), on_(true), sink_(sink) {
    mark("start");
  }
  bool on() const { return on_; }
  void mark(const char* name) {
    if (!on_) return;
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    CK(cudaEventRecord(e, st_));
    ev_.push_back(e);
    names_.push_back(name);
  }
  ~StageProfiler() {
    if (!on_) return;
    cudaEventSynchronize(ev_.back());
    if (sink_) {
      for (std::size_t i = 1; i < ev_.size(); ++i) {
        float ms = 0;
        cudaEventElapsedTime(&ms, ev_[i - 1], ev_[i]);
        sink_->emplace_back(names_[i], ms * 1e-3);
      }
      for (auto e : ev_) cudaEventDestroy(e);
      return;
    }
    std::string line = std::string("[profile] ") + what_;
    for (std::size_t i = 1; i < ev_.size(); ++i) {
      float ms = 0;
      cudaEventElapsedTime(&ms, ev_[i - 1], ev_[i]);
      char buf[96];
      std::snprintf(buf, sizeof(buf), " %s=%.3fms", names_[i].c_str(), ms);
      line += buf;
    }
    std::fprintf(stderr, "%s\n", line.c_str());
    for (auto e : ev_) cudaEventDestroy(e);
  }

 private:
  const char* what_;
  cudaStream_t st_;
  bool on_ = false;
  std::vector<cudaEvent_t> ev_;
  std::vector<std::string> names_;
  std::vector<std::pair<std::string, double>>* sink_ = nullptr;
};

}  // namespace b200
