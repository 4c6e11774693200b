// Host drain of the solution store: while the sampler keeps running, each
// harvest's newly appended solution keys are copied to host memory by a
// worker thread on its own copy stream, so that handing the result to the
// caller (satgrad::run's RunResult, include/satgrad/sampler.hpp:79-81) costs
// no copy at the end of the run.
//
// Host memory is one anonymous mapping with transparent huge pages, grown by
// mremap.  Keys arrive by DMA into a process-wide pinned double buffer (2 x
// 32 MB, allocated once) and are copied out on drain_threads() threads (2), which also
// spreads the first touch (measured on the B200 host: a 400 MB first touch
// costs ~200 ms on one thread with 4 KB pages, ~16 ms on 8 threads with huge
// pages; pinning 400 MB with cudaHostAlloc costs ~220 ms, more than the copy
// it would speed up; pageable copies hold the driver while they run).
// Ownership of the mapping moves to the caller with take(); host_free()
// unmaps it.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <deque>
#include <mutex>
#include <string>
#include <thread>

namespace sgx {

class HostDrain {
 public:
  HostDrain(int device, int key_words);
  ~HostDrain();
  HostDrain(const HostDrain&) = delete;
  HostDrain& operator=(const HostDrain&) = delete;

  // Queue rows [first, first + count) of the device store for copy once the
  // work queued on `st` so far (the append) has finished.  Rows must arrive
  // in order (first == rows queued so far).
  void push(const uint64_t* dstore, int64_t first, int64_t count, cudaStream_t st);
  // Block until every queued copy has landed; rethrows a worker error.
  void wait_idle();
  // Drop the current buffer and counters (a new run starts at row 0).
  void reset();
  // Rows queued so far.
  int64_t queued() const { return queued_; }
  // After wait_idle(): hand the mapping to the caller (nullptr if no rows).
  uint64_t* take(int64_t* rows, size_t* bytes);

 private:
  struct Job {
    const uint64_t* src;
    int64_t first, count;
    cudaEvent_t ev;
  };
  void loop();
  void ensure(int64_t rows);  // capacity up to `rows` (first touch happens in the copy)

  int device_;
  size_t row_bytes_;
  cudaStream_t cst_ = nullptr;
  std::thread th_;
  std::mutex mu_;
  std::condition_variable cv_, idle_cv_;
  std::deque<Job> q_;
  bool stop_ = false, busy_ = false;
  std::atomic<bool> hurry_{false};  // someone waits for the drain: copy what is left in one go
  std::string err_;
  // worker-owned while busy
  char* buf_ = nullptr;
  size_t cap_bytes_ = 0;
  int64_t landed_ = 0;
  int64_t queued_ = 0;  // main thread
};

// Allocate / release host result memory of the drain's kind (a released
// mapping is parked for reuse; *actual = the mapping's size).
void* host_map(size_t bytes, size_t* actual);
void host_free(void* p, size_t bytes);

}  // namespace sgx
