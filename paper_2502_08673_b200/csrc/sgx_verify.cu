// Solution verification: the reference's `satgrad verify` (cmd_verify,
// tools/satgrad_main.cpp:242-302) over a solution text of "v1 -v2 ... 0"
// lines, with its error cases and line numbers:
//   * host threads parse the text into packed keys (dedupe_key layout,
//     sampler.cpp:18-26), split at line boundaries;
//   * the GPU checks every assignment against the CNF bit-sliced, 32
//     solutions per word: keys are transposed into [var][word] rows by warp
//     ballots, then each thread ANDs the clause ORs of one word (eval_cnf,
//     cnf.cpp:129-147), clause data read as broadcasts;
//   * the GPU fingerprints every key and radix-sorts (fingerprint, row); the
//     host walks runs of equal fingerprints with an exact key compare to find
//     duplicates (SolutionSet::insert, sampler.cpp:28-44).
// The first error in line order wins, as in the reference's single pass.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include <cub/cub.cuh>

#include "sgx_kernels.cuh"
#include "sgx_launch.hpp"

namespace sgx {

namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// BT[v][w] bit i = variable v+1 of solution 32w+i (one warp per (word, key word)).
__global__ void k_keys_to_bt(const uint64_t* __restrict__ keys, int64_t n, int kw, int num_vars, int W,
                             uint32_t* __restrict__ BT) {
  const int lane = threadIdx.x & 31;
  const long long gw = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5;
  if (gw >= static_cast<long long>(W) * kw) return;
  const int w = static_cast<int>(gw / kw), q = static_cast<int>(gw % kw);
  const int64_t r = static_cast<int64_t>(w) * 32 + lane;
  const uint64_t x = r < n ? __ldg(keys + r * kw + q) : 0ull;
  for (int b = 0; b < 64; ++b) {
    const int v = q * 64 + b;
    const uint32_t word = __ballot_sync(0xffffffffu, (x >> b) & 1ull);
    if (lane == 0 && v < num_vars) BT[static_cast<size_t>(v) * W + w] = word;
  }
}

// ok[w] bit i: solution 32w+i satisfies every clause (enc = var << 1 | neg).
// Clauses are split over blockIdx.y chunks (a thread per (word, chunk)),
// folded by atomicAnd into ok_out, which starts all-ones.
constexpr int kVerifyClauseChunk = 256;
__global__ void k_cnf_words(const uint32_t* __restrict__ BT, int W, int64_t n, const int* __restrict__ cptr,
                            const int* __restrict__ enc, int n_clauses, uint32_t* __restrict__ ok_out) {
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= W) return;
  const int64_t r0 = static_cast<int64_t>(w) * 32;
  uint32_t ok = blockIdx.y > 0 ? 0xffffffffu : (r0 + 32 <= n ? 0xffffffffu : (r0 >= n ? 0u : ((1u << (n - r0)) - 1u)));
  const int c0 = blockIdx.y * kVerifyClauseChunk;
  const int c1 = min(n_clauses, c0 + kVerifyClauseChunk);
  for (int c = c0; c < c1 && ok; ++c) {
    uint32_t any = 0u;
    const int e = __ldg(cptr + c + 1);
    for (int k = __ldg(cptr + c); k < e; ++k) {
      const int x = __ldg(enc + k);
      any |= __ldg(BT + static_cast<size_t>(x >> 1) * W + w) ^ (0u - static_cast<uint32_t>(x & 1));
    }
    ok &= any;
  }
  if (ok != 0xffffffffu) atomicAnd(ok_out + w, ok);
}

__global__ void k_iota(int64_t* __restrict__ v, int64_t n) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) v[i] = i;
}

__global__ void k_key_fp(const uint64_t* __restrict__ keys, int64_t n, int kw, uint64_t* __restrict__ fp) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (r >= n) return;
  uint64_t h = 0x9E3779B97F4A7C15ull;
  for (int q = 0; q < kw; ++q) h = fold(h, __ldg(keys + r * kw + q));
  fp[r] = h;
}

// One line of cmd_verify's loop (satgrad_main.cpp:250-289).  Returns 0 for a
// parsed assignment (written to key), -1 for a blank line, else an error kind.
int parse_line(const char* p, const char* e, int num_vars, int kw, uint64_t* key, uint64_t* seen, int64_t* var) {
  std::memset(key, 0, kw * sizeof(uint64_t));
  std::memset(seen, 0, kw * sizeof(uint64_t));
  bool terminated = false, any = false;
  for (;;) {
    while (p < e && (*p == ' ' || *p == '\t' || *p == '\r' || *p == '\v' || *p == '\f')) ++p;
    // istream >> long long: optional sign, then digits; anything else ends the line
    const char* q = p;
    bool neg = false;
    if (q < e && (*q == '-' || *q == '+')) neg = *q++ == '-';
    if (q >= e || *q < '0' || *q > '9') break;
    long long v = 0;
    bool overflow = false;
    while (q < e && *q >= '0' && *q <= '9') {
      overflow |= __builtin_mul_overflow(v, 10LL, &v) || __builtin_add_overflow(v, static_cast<long long>(*q - '0'), &v);
      ++q;
    }
    if (overflow) break;  // the stream fails: the line ends here, as on any non-number
    p = q;
    any = true;
    if (v == 0) {
      terminated = true;
      break;
    }
    if (v > num_vars) {
      *var = v;
      return 1;
    }
    const int i = static_cast<int>(v - 1), w = i >> 6;
    const uint64_t m = 1ull << (i & 63);
    const bool bit = !neg;
    if (seen[w] & m) {
      if (((key[w] & m) != 0) != bit) {
        *var = v;
        return 2;
      }
    }
    seen[w] |= m;
    if (bit) key[w] |= m;
  }
  if (!any) return -1;
  if (!terminated) return 3;
  for (int w = 0; w < kw; ++w) {
    const int rem = num_vars - 64 * w;
    const uint64_t full = rem >= 64 ? ~0ull : ((1ull << rem) - 1ull);
    if ((seen[w] & full) != full) {
      const uint64_t miss = ~seen[w] & full;
      *var = 64 * w + __builtin_ctzll(miss) + 1;
      return 4;
    }
  }
  return 0;
}

struct Chunk {
  std::vector<uint64_t> keys;
  std::vector<int64_t> line;  // local line index of each row
  int64_t lines = 0;          // lines in the chunk (up to the error, if any)
  int64_t err_line = -1;      // local line of the first error
  int err_kind = 0;
  int64_t err_var = 0;
};

}  // namespace

// The device half of a check: ok[w] bit i = row 32w+i satisfies every clause;
// sfp / srow = fingerprints of all rows radix-sorted, with their rows.
void check_keys_device(int device, const std::vector<int64_t>& cptr, const std::vector<int32_t>& clit, int num_vars,
                       int kw, const uint64_t* keys, int64_t n, std::vector<uint32_t>& ok,
                       std::vector<uint64_t>& sfp, std::vector<int64_t>& srow, int64_t* launches) {
  VerifyResult launch_count;
  VerifyResult* out = &launch_count;
  // ---- device: CNF check (bit-sliced) + fingerprints, in row chunks
  ok.assign((n + 31) / 32, 0u);
  sfp.resize(n);  // fingerprints, sorted
  srow.resize(n);  // their rows (stable: ascending within a run)
  if (n > 0) {
    if (n > (int64_t{1} << 31) - 1) throw std::invalid_argument("too many solutions for one verify call");
    ck(cudaSetDevice(device), "cudaSetDevice");
    cudaStream_t st;
    ck(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "verify stream");
    const int nc = static_cast<int>(cptr.size()) - 1;
    std::vector<int> p32(cptr.begin(), cptr.end()), enc(clit.size());
    for (size_t k = 0; k < clit.size(); ++k) enc[k] = ((std::abs(clit[k]) - 1) << 1) | (clit[k] < 0 ? 1 : 0);
    const int64_t R = std::min<int64_t>(n, int64_t{1} << 16);  // rows per chunk
    const int Wc = static_cast<int>((R + 31) / 32);
    int *dptr = nullptr, *denc = nullptr;
    uint64_t *dkeys = nullptr, *dfp = nullptr, *dfp2 = nullptr;
    int64_t *drow = nullptr, *drow2 = nullptr;
    uint32_t *dbt = nullptr, *dok = nullptr;
    ck(cudaMallocAsync(&dptr, p32.size() * sizeof(int), st), "verify alloc");
    ck(cudaMallocAsync(&denc, std::max<size_t>(1, enc.size()) * sizeof(int), st), "verify alloc");
    ck(cudaMallocAsync(&dkeys, static_cast<size_t>(R) * kw * sizeof(uint64_t), st), "verify alloc");
    ck(cudaMallocAsync(&dfp, static_cast<size_t>(n) * sizeof(uint64_t), st), "verify alloc");
    ck(cudaMallocAsync(&dfp2, static_cast<size_t>(n) * sizeof(uint64_t), st), "verify alloc");
    ck(cudaMallocAsync(&drow, static_cast<size_t>(n) * sizeof(int64_t), st), "verify alloc");
    ck(cudaMallocAsync(&drow2, static_cast<size_t>(n) * sizeof(int64_t), st), "verify alloc");
    ck(cudaMallocAsync(&dbt, static_cast<size_t>(std::max(1, num_vars)) * Wc * sizeof(uint32_t), st), "verify alloc");
    ck(cudaMallocAsync(&dok, static_cast<size_t>(Wc) * sizeof(uint32_t), st), "verify alloc");
    ck(cudaMemcpyAsync(dptr, p32.data(), p32.size() * sizeof(int), cudaMemcpyHostToDevice, st), "verify h2d");
    if (!enc.empty())
      ck(cudaMemcpyAsync(denc, enc.data(), enc.size() * sizeof(int), cudaMemcpyHostToDevice, st), "verify h2d");
    for (int64_t r0 = 0; r0 < n; r0 += R) {
      const int64_t m = std::min(R, n - r0);
      const int W = static_cast<int>((m + 31) / 32);
      ck(cudaMemcpyAsync(dkeys, keys + r0 * kw, static_cast<size_t>(m) * kw * sizeof(uint64_t),
                         cudaMemcpyHostToDevice, st), "verify h2d");
      const long long warps = static_cast<long long>(W) * kw;
      k_keys_to_bt<<<static_cast<unsigned>((warps * 32 + 255) / 256), 256, 0, st>>>(dkeys, m, kw, num_vars, W, dbt);
      ck(cudaMemsetAsync(dok, 0xff, W * sizeof(uint32_t), st), "verify memset");
      k_cnf_words<<<dim3((W + 127) / 128, std::max(1, (nc + kVerifyClauseChunk - 1) / kVerifyClauseChunk)), 128, 0, st>>>(
          dbt, W, m, dptr, denc, nc, dok);
      k_key_fp<<<static_cast<unsigned>((m + 255) / 256), 256, 0, st>>>(dkeys, m, kw, dfp + r0);
      ck(cudaMemcpyAsync(ok.data() + r0 / 32, dok, W * sizeof(uint32_t), cudaMemcpyDeviceToHost, st), "verify d2h");
      ck(cudaStreamSynchronize(st), "verify sync");  // the key chunk buffer is reused
      out->launches += 3;
    }
    k_iota<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(drow, n);
    size_t tmp_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, dfp, dfp2, drow, drow2, static_cast<int>(n), 0, 64, st);
    void* tmp = nullptr;
    ck(cudaMallocAsync(&tmp, std::max<size_t>(1, tmp_bytes), st), "verify alloc");
    cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, dfp, dfp2, drow, drow2, static_cast<int>(n), 0, 64, st);
    ck(cudaMemcpyAsync(sfp.data(), dfp2, n * sizeof(uint64_t), cudaMemcpyDeviceToHost, st), "verify d2h");
    ck(cudaMemcpyAsync(srow.data(), drow2, n * sizeof(int64_t), cudaMemcpyDeviceToHost, st), "verify d2h");
    out->launches += 3;
    ck(cudaGetLastError(), "verify kernels");
    for (void* p : {static_cast<void*>(dptr), static_cast<void*>(denc), static_cast<void*>(dkeys),
                    static_cast<void*>(dfp), static_cast<void*>(dbt), static_cast<void*>(dok),
                    static_cast<void*>(dfp2), static_cast<void*>(drow), static_cast<void*>(drow2), tmp})
      cudaFreeAsync(p, st);
    ck(cudaStreamSynchronize(st), "verify free");
    cudaStreamDestroy(st);
  }
  *launches += out->launches;
}

void verify_solutions(int device, const std::vector<int64_t>& cptr, const std::vector<int32_t>& clit, int num_vars,
                      const char* text, int64_t len, VerifyResult* out) {
  *out = VerifyResult{};
  const int kw = std::max(1, (num_vars + 63) / 64);
  // ---- parse, one chunk per host thread, split after a newline
  const int T = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(16, len / (1 << 20))));
  std::vector<int64_t> cut(T + 1, len);
  cut[0] = 0;
  for (int t = 1; t < T; ++t) {
    int64_t c = std::max(cut[t - 1], len / T * t);
    const void* nl = c < len ? std::memchr(text + c, '\n', len - c) : nullptr;
    cut[t] = nl ? static_cast<const char*>(nl) - text + 1 : len;
  }
  std::vector<Chunk> ch(T);
  auto work = [&](int t) {
    Chunk& C = ch[t];
    std::vector<uint64_t> key(kw), seen(kw);
    const char* p = text + cut[t];
    const char* end = text + cut[t + 1];
    while (p < end) {
      const char* nl = static_cast<const char*>(std::memchr(p, '\n', end - p));
      const char* le = nl ? nl : end;
      int64_t var = 0;
      const int k = parse_line(p, le, num_vars, kw, key.data(), seen.data(), &var);
      if (k > 0) {
        C.err_line = C.lines;
        C.err_kind = k;
        C.err_var = var;
        return;
      }
      if (k == 0) {
        C.keys.insert(C.keys.end(), key.begin(), key.end());
        C.line.push_back(C.lines);
      }
      ++C.lines;
      p = nl ? nl + 1 : end;
    }
  };
  {
    std::vector<std::thread> th;
    for (int t = 1; t < T; ++t) th.emplace_back(work, t);
    work(0);
    for (auto& x : th) x.join();
  }
  // rows in order up to the first parse error; global 1-based line numbers
  std::vector<uint64_t> keys;
  std::vector<int64_t> line_of;
  int64_t base = 0, parse_err_line = -1;
  for (int t = 0; t < T; ++t) {
    const Chunk& C = ch[t];
    keys.insert(keys.end(), C.keys.begin(), C.keys.end());
    for (int64_t l : C.line) line_of.push_back(base + l + 1);
    if (C.err_line >= 0) {
      parse_err_line = base + C.err_line + 1;
      out->err_kind = C.err_kind;
      out->err_var = C.err_var;
      break;
    }
    // a chunk's line count: its newlines (every chunk but the last ends in one)
    base += C.lines;
  }
  const int64_t n = static_cast<int64_t>(line_of.size());
  std::vector<uint32_t> ok;
  std::vector<uint64_t> sfp;
  std::vector<int64_t> srow;
  check_keys_device(device, cptr, clit, num_vars, kw, keys.data(), n, ok, sfp, srow, &out->launches);
  // ---- first unsatisfied row, first duplicate row (of an earlier, valid row)
  int64_t bad = n;
  int bad_kind = 0;
  for (int64_t r = 0; r < n; ++r)
    if (!((ok[r >> 5] >> (r & 31)) & 1u)) {
      bad = r;
      bad_kind = 5;
      break;
    }
  // a row duplicates an earlier one iff an earlier member of its fingerprint
  // run has the same key; only rows before the first error matter
  for (int64_t a = 0; a < n;) {
    int64_t b = a + 1;
    while (b < n && sfp[b] == sfp[a]) ++b;
    for (int64_t j = a + 1; j < b && srow[j] < bad; ++j) {
      const uint64_t* kj = keys.data() + srow[j] * kw;
      for (int64_t i = a; i < j; ++i)
        if (std::memcmp(keys.data() + srow[i] * kw, kj, kw * sizeof(uint64_t)) == 0) {
          bad = srow[j];
          bad_kind = 6;
          break;
        }
    }
    a = b;
  }
  if (bad < n) {  // a row error precedes any parse error (rows stop before it)
    out->checked = bad;
    out->err_line = line_of[bad];
    out->err_kind = bad_kind;
    out->err_var = 0;
  } else {
    out->checked = n;
    out->err_line = parse_err_line > 0 ? parse_err_line : 0;
    if (parse_err_line <= 0) {
      out->err_kind = 0;
      out->err_var = 0;
    }
  }
}

void verify_keys(int device, const std::vector<int64_t>& cptr, const std::vector<int32_t>& clit, int num_vars,
                 const uint64_t* keys, int64_t n, KeyCheck* out) {
  *out = KeyCheck{};
  const int kw = std::max(1, (num_vars + 63) / 64);
  std::vector<uint32_t> ok;
  std::vector<uint64_t> sfp;
  std::vector<int64_t> srow;
  check_keys_device(device, cptr, clit, num_vars, kw, keys, n, ok, sfp, srow, &out->launches);
  out->checked = n;
  for (int64_t r = 0; r < n; ++r)
    if (!((ok[r >> 5] >> (r & 31)) & 1u)) ++out->unsat;
  // bits above num_vars must be zero in a packed key (dedupe_key, sampler.cpp:18-26)
  if (num_vars % 64) {
    const uint64_t hi = ~uint64_t{0} << (num_vars % 64);
    for (int64_t r = 0; r < n; ++r)
      if (keys[r * kw + kw - 1] & hi) ++out->malformed;
  }
  for (int64_t a = 0; a < n;) {
    int64_t b = a + 1;
    while (b < n && sfp[b] == sfp[a]) ++b;
    for (int64_t j = a + 1; j < b; ++j) {
      const uint64_t* kj = keys + srow[j] * kw;
      for (int64_t i = a; i < j; ++i)
        if (std::memcmp(keys + srow[i] * kw, kj, kw * sizeof(uint64_t)) == 0) {
          ++out->duplicate;
          break;
        }
    }
    a = b;
  }
}

}  // namespace sgx
