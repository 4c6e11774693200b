// Device-side solution emission: the reference's format_solutions
// (sampler.cpp:66-85) -- "v1 -v2 ... vn 0\n" per solution in insertion order,
// a literal v when the variable is true, -v when false -- rendered on the GPU
// from the packed keys of the solution store (dedupe_key layout,
// sampler.cpp:18-26).  At C2 scale the text is ~60 KB per solution (19 GB for
// a 310k-solution run), which a host loop formats at ~100 MB/s.
//
// Layout of a line: variable v starts at S(v) + neg(v), where S(v) is the
// width of the literals 1..v-1 written positive (closed form over decimal
// digit counts) and neg(v) the number of false variables before v (a
// popcount prefix over the key words).  A line is num_vars + 2 + sum of
// digit widths + (false variables) bytes long, so per-solution lengths come
// from one popcount per key word, an exclusive scan gives the offsets, and
// every thread writes its variables independently.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cub/cub.cuh>

#include "sgx_launch.hpp"

namespace sgx {

namespace {

__host__ __device__ inline long long digits_sum_below(long long v) {
  // sum of decimal widths of 1..v-1
  long long s = 0, lo = 1, w = 1;
  while (lo < v) {
    const long long hi = lo * 10;  // [lo, hi) has width w
    const long long top = hi < v ? hi : v;
    s += (top - lo) * w;
    lo = hi;
    ++w;
  }
  return s;
}

__device__ __forceinline__ int width(int v) {
  int w = 1;
  for (int t = 10; t <= v; t *= 10) ++w;
  return w;
}

__global__ void k_fmt_len(const uint64_t* __restrict__ store, long long first, long long n, int words, int num_vars,
                          long long base_len, long long* __restrict__ len) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const uint64_t* k = store + (first + i) * words;
    long long ones = 0;
    for (int w = 0; w < words; ++w) {
      uint64_t x = __ldg(k + w);
      const int rem = num_vars - 64 * w;
      if (rem < 64) x &= (1ull << rem) - 1ull;
      ones += __popcll(x);
    }
    len[i] = base_len + (num_vars - ones);
  }
}

// One CTA per solution: popcount prefix of the key words in shared memory,
// then every thread writes the literals of its variables.
__global__ void __launch_bounds__(256)
k_fmt_write(const uint64_t* __restrict__ store, long long first, long long n, int words, int num_vars,
            const long long* __restrict__ off, long long out_base, char* __restrict__ out) {
  extern __shared__ int pref[];  // [words + 1]: true variables before word w
  for (long long i = blockIdx.x; i < n; i += gridDim.x) {
    const uint64_t* k = store + (first + i) * words;
    __syncthreads();
    if (threadIdx.x == 0) {
      int acc = 0;
      for (int w = 0; w < words; ++w) {
        pref[w] = acc;
        uint64_t x = __ldg(k + w);
        const int rem = num_vars - 64 * w;
        if (rem < 64) x &= (1ull << rem) - 1ull;
        acc += __popcll(x);
      }
      pref[words] = acc;
    }
    __syncthreads();
    char* line = out + (off[i] - out_base);
    for (int v = 1 + threadIdx.x; v <= num_vars; v += blockDim.x) {
      const int w = (v - 1) >> 6, b = (v - 1) & 63;
      const uint64_t x = __ldg(k + w);
      const bool bit = (x >> b) & 1ull;
      const int ones_before = pref[w] + __popcll(b ? (x & ((1ull << b) - 1ull)) : 0ull);
      const long long pos = (v - 1) + digits_sum_below(v) + ((v - 1) - ones_before);
      char* p = line + pos;
      if (!bit) *p++ = '-';
      const int wd = width(v);
      int t = v;
      for (int d = wd - 1; d >= 0; --d) {
        p[d] = static_cast<char>('0' + t % 10);
        t /= 10;
      }
      p[wd] = ' ';
    }
    if (threadIdx.x == 0) {
      const long long end = (num_vars + digits_sum_below(num_vars + 1)) + (num_vars - pref[words]);
      line[end] = '0';
      line[end + 1] = '\n';
    }
  }
}

}  // namespace

long long fmt_base_len(int num_vars) { return num_vars + digits_sum_below(num_vars + 1) + 2; }

void launch_fmt_lengths(cudaStream_t st, const uint64_t* store, long long first, long long n, int words,
                        int num_vars, long long* len_off, void* scratch, size_t* scratch_bytes) {
  // len_off holds n + 1 entries: lengths, then (in place) exclusive offsets
  if (scratch == nullptr) {
    cub::DeviceScan::ExclusiveSum(nullptr, *scratch_bytes, len_off, len_off, static_cast<int>(n + 1), st);
    return;
  }
  if (n > 0) {
    const int grid = static_cast<int>(std::min<long long>((n + 255) / 256, 148 * 16));
    k_fmt_len<<<grid, 256, 0, st>>>(store, first, n, words, num_vars, fmt_base_len(num_vars), len_off);
  }
  cudaMemsetAsync(len_off + n, 0, sizeof(long long), st);
  cub::DeviceScan::ExclusiveSum(scratch, *scratch_bytes, len_off, len_off, static_cast<int>(n + 1), st);
}

void launch_fmt_write(cudaStream_t st, const uint64_t* store, long long first, long long n, int words,
                      int num_vars, const long long* off, long long out_base, char* out) {
  if (n <= 0) return;
  const int grid = static_cast<int>(std::min<long long>(n, 148 * 8));
  k_fmt_write<<<grid, 256, (words + 1) * sizeof(int), st>>>(store, first, n, words, num_vars, off, out_base, out);
}

}  // namespace sgx
