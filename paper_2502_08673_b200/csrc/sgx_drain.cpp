#include "sgx_drain.hpp"

#include <sys/mman.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <vector>

namespace sgx {

namespace {

struct Done {};  // a job finished early (direct copy)
constexpr size_t kHuge = size_t{2} << 20;

size_t round_huge(size_t b) { return (b + kHuge - 1) / kHuge * kHuge; }

void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// memcpy on up to drain_threads() threads (the destination's first touch --
// page faults, huge-page zeroing -- happens inside, in parallel).
// Copy-out threads (SGX_DRAIN_THREADS, default 2).  Measured on C2 (10
// restarts, 400 MB of keys): 8 threads slowed the device loop by ~7 % (host
// memory bandwidth / cycles taken from the launching thread), 1-2 threads by
// nothing, and 2 keep the final copy-out after the run at ~1 ms.
int drain_threads() {
  static const int t = [] {
    const char* e = std::getenv("SGX_DRAIN_THREADS");
    const int v = e ? std::atoi(e) : 2;
    return v >= 1 && v <= 32 ? v : 2;
  }();
  return t;
}

void par_copy(char* dst, const char* src, size_t n) {
  if (n == 0) return;
  const int T = static_cast<int>(std::min<size_t>(drain_threads(), std::max<size_t>(1, n / (4u << 20))));
  auto work = [dst, src, n, T](int t) {
    const size_t lo = n / T * t, hi = t + 1 == T ? n : n / T * (t + 1);
    std::memcpy(dst + lo, src + lo, hi - lo);
  };
  if (T == 1) {
    work(0);
    return;
  }
  std::vector<std::thread> th;
  for (int t = 1; t < T; ++t) th.emplace_back(work, t);
  work(0);
  for (auto& x : th) x.join();
}

// Process-wide pinned staging per device: two 32 MB buffers, allocated once
// (cudaHostAlloc is ~0.5 ms/MB; a per-run allocation would cost more than
// the copies).  The D2H copies are then real DMA that return at once,
// instead of pageable copies that hold the driver while they run.
constexpr size_t kStage = size_t{32} << 20;
struct Staging {
  char* buf[2] = {nullptr, nullptr};
  cudaEvent_t done[2] = {nullptr, nullptr};
  std::mutex mu;  // one drain at a time per device
};
Staging& staging(int device) {
  static std::mutex mu;
  static std::vector<std::unique_ptr<Staging>> all;
  std::lock_guard<std::mutex> lk(mu);
  if (static_cast<int>(all.size()) <= device) all.resize(device + 1);
  if (!all[device]) {
    auto st = std::make_unique<Staging>();
    for (int k = 0; k < 2; ++k) {
      check(cudaHostAlloc(reinterpret_cast<void**>(&st->buf[k]), kStage, cudaHostAllocPortable), "drain staging");
      check(cudaEventCreateWithFlags(&st->done[k], cudaEventDisableTiming), "drain staging event");
    }
    all[device] = std::move(st);
  }
  return *all[device];
}

}  // namespace

// Released result mappings are parked (up to two; cache_bytes() in all) and handed
// to the next run: their pages are already faulted in, so a run does not pay
// the first touch -- or the kernel's huge-page compaction -- again.  A parked
// mapping is also page-locked (cudaHostRegister, once, when it is parked), so
// the next run's drain DMAs straight into it at PCIe speed instead of through
// the staging buffers and a host memcpy (C4: 1.3 GB of keys per restart;
// staged, the copy-out bounded the end-to-end rate).  SGX_PIN_PARKED=0 turns
// the locking off.
namespace {
std::mutex g_cache_mu;
std::vector<std::pair<void*, size_t>> g_cache;
std::vector<std::pair<void*, size_t>> g_pinned;  // page-locked mappings (base, bytes)
constexpr size_t kCacheEntries = 2;
// Parked bytes in all: a quarter of physical memory, 16-96 GB (a 10-restart
// C4 run returns 13 GB of keys in a mapping grown to ~20 GB).
size_t cache_bytes() {
  static const size_t lim = [] {
    const long pages = sysconf(_SC_PHYS_PAGES), psz = sysconf(_SC_PAGESIZE);
    const size_t phys = pages > 0 && psz > 0 ? static_cast<size_t>(pages) * static_cast<size_t>(psz) : 0;
    return std::clamp<size_t>(phys / 4, size_t{16} << 30, size_t{96} << 30);
  }();
  return lim;
}

bool trace_on() {
  static const bool on = std::getenv("SGX_TRACE") != nullptr;
  return on;
}
double now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

bool pin_parked() {
  static const bool on = [] {
    const char* e = std::getenv("SGX_PIN_PARKED");
    return !(e && e[0] == '0');
  }();
  return on;
}

// (g_cache_mu held)
size_t pinned_bytes(const void* p) {
  for (auto& e : g_pinned)
    if (e.first == p) return e.second;
  return 0;
}
void unpin(void* p) {
  for (size_t i = 0; i < g_pinned.size(); ++i)
    if (g_pinned[i].first == p) {
      cudaHostUnregister(p);
      g_pinned.erase(g_pinned.begin() + static_cast<long>(i));
      return;
    }
}
}  // namespace

// [dst, dst + n) lies inside one page-locked mapping.
bool host_range_pinned(const void* dst, size_t n) {
  std::lock_guard<std::mutex> lk(g_cache_mu);
  const char* d = static_cast<const char*>(dst);
  for (auto& e : g_pinned) {
    const char* b = static_cast<const char*>(e.first);
    if (d >= b && d + n <= b + e.second) return true;
  }
  return false;
}

// Before a mapping moves or shrinks (mremap / munmap): drop its page lock.
void host_unpin(void* p) {
  std::lock_guard<std::mutex> lk(g_cache_mu);
  unpin(p);
}

void* host_map(size_t bytes, size_t* actual) {
  const size_t b = round_huge(std::max<size_t>(bytes, 1));
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    size_t best = g_cache.size();
    for (size_t i = 0; i < g_cache.size(); ++i)  // the largest parked mapping
      if (best == g_cache.size() || g_cache[i].second > g_cache[best].second) best = i;
    if (best < g_cache.size()) {
      auto [p, n] = g_cache[best];
      g_cache.erase(g_cache.begin() + static_cast<long>(best));
      if (n < b) {
        unpin(p);
        void* q = mremap(p, n, b, MREMAP_MAYMOVE);
        if (q == MAP_FAILED) {
          munmap(p, n);
        } else {
          madvise(q, b, MADV_HUGEPAGE);
          *actual = b;
          return q;
        }
      } else {
        *actual = n;
        return p;
      }
    }
  }
  void* p = mmap(nullptr, b, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  if (p == MAP_FAILED) throw std::runtime_error("host result mapping failed");
  madvise(p, b, MADV_HUGEPAGE);
  *actual = b;
  return p;
}

void host_free(void* p, size_t bytes) {
  if (!p) return;
  const size_t b = round_huge(std::max<size_t>(bytes, 1));
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    size_t held = 0;
    for (auto& e : g_cache) held += e.second;
    // A larger mapping displaces smaller parked ones (the next run of the
    // same size can then take it without growing).
    while (!g_cache.empty() && (g_cache.size() >= kCacheEntries || held + b > cache_bytes())) {
      size_t s = 0;
      for (size_t i = 1; i < g_cache.size(); ++i)
        if (g_cache[i].second < g_cache[s].second) s = i;
      if (g_cache[s].second >= b || b > cache_bytes()) break;
      auto [q, n] = g_cache[s];
      g_cache.erase(g_cache.begin() + static_cast<long>(s));
      held -= n;
      unpin(q);
      munmap(q, n);
    }
    if (g_cache.size() < kCacheEntries && held + b <= cache_bytes()) {
      g_cache.emplace_back(p, b);
      if (pin_parked() && pinned_bytes(p) != b) {
        unpin(p);
        const double t0 = now_ms();
        const cudaError_t rc = cudaHostRegister(p, b, cudaHostRegisterPortable);
        if (rc == cudaSuccess)
          g_pinned.emplace_back(p, b);
        else
          cudaGetLastError();  // (e.g. a locked-memory limit): the staged path stays correct
        if (trace_on())
          fprintf(stderr, "[sgx] drain: parked %.2f GB, page-lock %s in %.1f ms\n", b / 1e9,
                  rc == cudaSuccess ? "ok" : cudaGetErrorString(rc), now_ms() - t0);
      }
      return;
    }
    unpin(p);
  }
  if (trace_on()) fprintf(stderr, "[sgx] drain: released %.2f GB (not parked)\n", b / 1e9);
  munmap(p, b);
}

HostDrain::HostDrain(int device, int key_words)
    : device_(device), row_bytes_(static_cast<size_t>(key_words) * sizeof(uint64_t)) {
  check(cudaSetDevice(device_), "cudaSetDevice");
  check(cudaStreamCreateWithFlags(&cst_, cudaStreamNonBlocking), "copy stream");
  th_ = std::thread([this] { loop(); });
}

HostDrain::~HostDrain() {
  {
    std::lock_guard<std::mutex> lk(mu_);
    stop_ = true;
  }
  cv_.notify_all();
  if (th_.joinable()) th_.join();
  for (auto& j : q_) cudaEventDestroy(j.ev);
  if (cst_) cudaStreamDestroy(cst_);
  host_free(buf_, cap_bytes_);
}

void HostDrain::push(const uint64_t* dstore, int64_t first, int64_t count, cudaStream_t st) {
  if (count <= 0) return;
  if (first != queued_) throw std::logic_error("host drain: rows out of order");
  cudaEvent_t ev;
  check(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "drain event");
  check(cudaEventRecord(ev, st), "drain event record");
  {
    std::lock_guard<std::mutex> lk(mu_);
    q_.push_back(Job{dstore, first, count, ev});
  }
  queued_ = first + count;
  cv_.notify_one();
}

void HostDrain::wait_idle() {
  hurry_ = true;
  std::unique_lock<std::mutex> lk(mu_);
  idle_cv_.wait(lk, [this] { return (q_.empty() && !busy_) || !err_.empty(); });
  hurry_ = false;
  if (!err_.empty()) throw std::runtime_error("host drain: " + err_);
}

void HostDrain::reset() {
  wait_idle();
  host_free(buf_, cap_bytes_);
  buf_ = nullptr;
  cap_bytes_ = 0;
  landed_ = queued_ = 0;
}

uint64_t* HostDrain::take(int64_t* rows, size_t* bytes) {
  wait_idle();
  uint64_t* p = reinterpret_cast<uint64_t*>(buf_);
  *rows = landed_;
  *bytes = cap_bytes_;
  buf_ = nullptr;
  cap_bytes_ = 0;
  landed_ = queued_ = 0;
  return p;
}

void HostDrain::ensure(int64_t rows) {
  const size_t need = static_cast<size_t>(rows) * row_bytes_;
  if (need > cap_bytes_) {
    const size_t ncap = round_huge(std::max<size_t>({need + need / 2, 2 * cap_bytes_, size_t{64} << 20}));
    if (!buf_) {
      size_t got = 0;
      buf_ = static_cast<char*>(host_map(ncap, &got));
      cap_bytes_ = got;
      return;
    } else {
      host_unpin(buf_);
      void* p = mremap(buf_, cap_bytes_, ncap, MREMAP_MAYMOVE);
      if (p == MAP_FAILED) throw std::runtime_error("host result mapping could not grow");
      buf_ = static_cast<char*>(p);
      madvise(buf_, ncap, MADV_HUGEPAGE);
    }
    cap_bytes_ = ncap;
  }
}

void HostDrain::loop() {
  cudaSetDevice(device_);
  for (;;) {
    Job j;
    {
      std::unique_lock<std::mutex> lk(mu_);
      cv_.wait(lk, [this] { return stop_ || !q_.empty(); });
      if (q_.empty()) return;  // stop_ and nothing left
      j = q_.front();
      q_.pop_front();
      busy_ = true;
    }
    std::string e;
    try {
      if (err_.empty()) {
        ensure(j.first + j.count);
        check(cudaStreamWaitEvent(cst_, j.ev, 0), "drain wait");
        const char* src = reinterpret_cast<const char*>(j.src + static_cast<size_t>(j.first) * (row_bytes_ / sizeof(uint64_t)));
        char* dst = buf_ + static_cast<size_t>(j.first) * row_bytes_;
        const size_t total = static_cast<size_t>(j.count) * row_bytes_;
        if (trace_on() && (j.first == 0 || !host_range_pinned(dst, total)))
          fprintf(stderr, "[sgx] drain: rows %lld+%lld into a %.2f GB mapping, %s\n", (long long)j.first,
                  (long long)j.count, cap_bytes_ / 1e9, host_range_pinned(dst, total) ? "page-locked: direct DMA" : "staged");
        if (host_range_pinned(dst, total)) {  // a page-locked (parked) mapping: DMA straight in
          // In chunks, each waited for: one big D2H copy beside the soft
          // passes slows them (C4: ~9 ms of device time per GB copied in
          // 220 MB copies, ~1 ms per GB in 4 MB copies, e2e).
          // Once the host waits for the drain (the run is over), the rest
          // goes in one copy.
          static const size_t chunk = [] {
            const char* e = std::getenv("SGX_DRAIN_CHUNK");  // MB; 0 = one copy
            const long v = e ? std::atol(e) : 8;
            return v > 0 ? static_cast<size_t>(v) << 20 : ~size_t{0};
          }();
          for (size_t off = 0, n = 0; off < total; off += n) {
            n = hurry_ ? total - off : std::min(chunk, total - off);
            check(cudaMemcpyAsync(dst + off, src + off, n, cudaMemcpyDeviceToHost, cst_), "drain copy");
            check(cudaStreamSynchronize(cst_), "drain copy wait");  // the gap is the point: chunks
          }                                                           // queued back to back cost as one copy
          landed_ = j.first + j.count;
          throw Done{};
        }
        // D2H through the pinned double buffer: chunk c lands in buf[c % 2]
        // while chunk c - 1 is copied out of the other one.
        Staging& sg = staging(device_);
        std::lock_guard<std::mutex> lk(sg.mu);
        const size_t nchunk = (total + kStage - 1) / kStage;
        for (size_t c = 0; c <= nchunk; ++c) {
          if (c < nchunk) {
            const size_t n = std::min(kStage, total - c * kStage);
            check(cudaMemcpyAsync(sg.buf[c & 1], src + c * kStage, n, cudaMemcpyDeviceToHost, cst_), "drain copy");
            check(cudaEventRecord(sg.done[c & 1], cst_), "drain copy event");
          }
          if (c > 0) {
            const size_t p = c - 1;
            check(cudaEventSynchronize(sg.done[p & 1]), "drain copy wait");
            par_copy(dst + p * kStage, sg.buf[p & 1], std::min(kStage, total - p * kStage));
          }
        }
        landed_ = j.first + j.count;
      }
    } catch (const Done&) {
    } catch (const std::exception& x) {
      e = x.what();
    }
    cudaEventDestroy(j.ev);
    {
      std::lock_guard<std::mutex> lk(mu_);
      if (!e.empty() && err_.empty()) err_ = e;
      busy_ = false;
    }
    idle_cv_.notify_all();
  }
}

}  // namespace sgx
