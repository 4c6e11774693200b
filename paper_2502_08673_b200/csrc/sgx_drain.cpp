#include "sgx_drain.hpp"

#include <sys/mman.h>

#include <algorithm>
#include <cstring>
#include <stdexcept>
#include <vector>

namespace sgx {

namespace {

constexpr size_t kHuge = size_t{2} << 20;

size_t round_huge(size_t b) { return (b + kHuge - 1) / kHuge * kHuge; }

void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// First touch of [p, p + n) on up to 8 threads, one write per 4 KB page (a
// huge page is zeroed once, by the first write into it).
void touch(char* p, size_t n) {
  if (n == 0) return;
  const int T = static_cast<int>(std::min<size_t>(8, std::max<size_t>(1, n / (8u << 20))));
  auto work = [p, n, T](int t) {
    const size_t lo = n / T * t, hi = t + 1 == T ? n : n / T * (t + 1);
    for (size_t o = lo; o < hi; o += 4096) p[o] = 0;
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

}  // namespace

void* host_map(size_t bytes) {
  const size_t b = round_huge(std::max<size_t>(bytes, 1));
  void* p = mmap(nullptr, b, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  if (p == MAP_FAILED) throw std::runtime_error("host result mapping failed");
  madvise(p, b, MADV_HUGEPAGE);
  return p;
}

void host_free(void* p, size_t bytes) {
  if (p) munmap(p, round_huge(std::max<size_t>(bytes, 1)));
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
  std::unique_lock<std::mutex> lk(mu_);
  idle_cv_.wait(lk, [this] { return (q_.empty() && !busy_) || !err_.empty(); });
  if (!err_.empty()) throw std::runtime_error("host drain: " + err_);
}

void HostDrain::reset() {
  wait_idle();
  host_free(buf_, cap_bytes_);
  buf_ = nullptr;
  cap_bytes_ = touched_bytes_ = 0;
  landed_ = queued_ = 0;
}

uint64_t* HostDrain::take(int64_t* rows, size_t* bytes) {
  wait_idle();
  uint64_t* p = reinterpret_cast<uint64_t*>(buf_);
  *rows = landed_;
  *bytes = cap_bytes_;
  buf_ = nullptr;
  cap_bytes_ = touched_bytes_ = 0;
  landed_ = queued_ = 0;
  return p;
}

void HostDrain::ensure(int64_t rows) {
  const size_t need = static_cast<size_t>(rows) * row_bytes_;
  if (need > cap_bytes_) {
    const size_t ncap = round_huge(std::max<size_t>({need + need / 2, 2 * cap_bytes_, size_t{64} << 20}));
    if (!buf_) {
      buf_ = static_cast<char*>(host_map(ncap));
    } else {
      void* p = mremap(buf_, cap_bytes_, ncap, MREMAP_MAYMOVE);
      if (p == MAP_FAILED) throw std::runtime_error("host result mapping could not grow");
      buf_ = static_cast<char*>(p);
      madvise(buf_, ncap, MADV_HUGEPAGE);
    }
    cap_bytes_ = ncap;
  }
  if (need > touched_bytes_) {
    touch(buf_ + touched_bytes_, need - touched_bytes_);
    touched_bytes_ = need;
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
        check(cudaMemcpyAsync(buf_ + static_cast<size_t>(j.first) * row_bytes_,
                              j.src + static_cast<size_t>(j.first) * (row_bytes_ / sizeof(uint64_t)),
                              static_cast<size_t>(j.count) * row_bytes_, cudaMemcpyDeviceToHost, cst_),
              "drain copy");
        check(cudaStreamSynchronize(cst_), "drain sync");
        landed_ = j.first + j.count;
      }
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
