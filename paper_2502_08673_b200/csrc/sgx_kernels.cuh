// sm_100a kernels of the sampling loop.  See DESIGN.md for the data layout
// and the roofline each kernel is held to.
//
//   k_init_v      init_soft_inputs + cast (sampler.cpp:54-64, 156-159)
//   k_forward     embed + forward (autodiff.cpp:57-152)         [soft program]
//   k_backward    loss + backward + gd_step (autodiff.cpp:154-290), pull-CSR
//   k_harden      harden (autodiff.cpp:292-297) + free bits (sampler.cpp:132-137),
//                 warp ballot -> 32 samples per word
//   k_bit_eval    eval_discrete (circuit.cpp:124-152) bit-sliced, PO check
//                 (sampler.cpp:140-146), eval_cnf (cnf.cpp:129-147)
//   k_keys        dedupe_key (sampler.cpp:18-26) via 32x32 bit transposes,
//                 64-bit fingerprint, device hash-table insert
//   k_new_rows / k_scan_blocks / k_append
//                 SolutionSet::insert order + quota (sampler.cpp:38-44, :129)
//
// Every floating-point operation is written with an explicit _rn intrinsic in
// the reference's evaluation order (no FMA contraction), and the sigmoid uses
// a restatement of glibc's expf, so the device reproduces the reference's
// float instantiation bit for bit.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "sgx_layout.hpp"

namespace sgx {

constexpr int kThreads = 256;
constexpr uint32_t kFull = 0xffffffffu;
constexpr uint64_t kPi = 0x243f6a8885a308d3ull;   // rng.hpp:22
constexpr uint64_t kInitTag = 0x696e6974ull;      // sampler.cpp:12
constexpr uint64_t kFreeTag = 0x66726565ull;      // sampler.cpp:13

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {  // rng.hpp:14-19
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

// One hash_stream fold step (rng.hpp:23).
__host__ __device__ __forceinline__ uint64_t fold(uint64_t h, uint64_t x) { return mix64(h ^ mix64(x)); }

// Fingerprint of a dedupe key: mix64(sum over key words q of
// mix64(word_q ^ (q+1)*pi)) mod 2^64.  The sum is order-independent, so the
// key words of one row can be folded by different warps.  Identity of a
// solution is its full key; the fingerprint only indexes the dedup table
// (a collision can drop a solution, never emit a wrong or duplicate one).
__host__ __device__ __forceinline__ uint64_t key_term(uint64_t kw, int q) {
  return mix64(kw ^ (kPi * static_cast<uint64_t>(q + 1)));
}

#if defined(__CUDACC__)
// glibc 2.39 expf (sysdeps/ieee754/flt-32/e_expf.c, FMA ifunc variant) for
// |x| < 88: 2^(k/32) table + cubic in double.  Constants are glibc's
// __exp2f_data; tests/test_expf.py checks every float in [-40, 40].
__device__ __forceinline__ float expf_glibc(float x, const uint64_t* __restrict__ tab) {
  const double kInvLn2N = 0x1.71547652b82fep+5, kShift = 0x1.8p+52;
  const double c0 = 0x1.c6af84b912394p-20, c1 = 0x1.ebfce50fac4f3p-13, c2 = 0x1.62e42ff0c52d6p-6;
  double xd = static_cast<double>(x);
  double kd = __fma_rn(kInvLn2N, xd, kShift);
  uint64_t ki = static_cast<uint64_t>(__double_as_longlong(kd));
  kd = __dsub_rn(kd, kShift);
  double r = __fma_rn(kInvLn2N, xd, -kd);
  uint64_t t = __ldg(reinterpret_cast<const unsigned long long*>(tab) + (ki & 31)) + (ki << 47);
  double s = __longlong_as_double(static_cast<long long>(t));
  double z = __fma_rn(c0, r, c1);
  double r2 = __dmul_rn(r, r);
  double y = __fma_rn(c2, r, 1.0);
  y = __fma_rn(z, r2, y);
  y = __dmul_rn(y, s);
  return __double2float_rn(y);
}

// sigmoid_clamped<float> (autodiff.cpp:12-16).
__device__ __forceinline__ float sigmoid_ref(float v, const uint64_t* __restrict__ tab) {
  float x = v < -40.0f ? -40.0f : (40.0f < v ? 40.0f : v);
  return __fdiv_rn(1.0f, __fadd_rn(1.0f, expf_glibc(-x, tab)));
}

#endif  // __CUDACC__

struct HarvestOut {
  double loss_total;     // last step's loss (sum over rows)
  long long new_rows;    // rows new to the table this harvest (before quota)
  long long accepted;    // rows appended to the solution store
  long long last_row;    // row of the last accepted solution (quota cut)
  long long overflow;    // solution store too small: grow and re-append
  unsigned long long fresh;  // multi-GPU merge: remote fingerprints new to the table
};

}  // namespace sgx
