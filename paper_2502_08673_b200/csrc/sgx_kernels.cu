#include <cuda_runtime.h>

#include <algorithm>

#include <map>
#include <mutex>
#include <utility>

#include "sgx_kernels.cuh"
#include "sgx_launch.hpp"

namespace sgx {

// Dynamic shared-memory opt-in, recorded per (kernel, device): the attribute
// belongs to one device, and samplers on several devices (or host threads)
// share these launchers.
static void opt_in_smem(const void* kernel, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  size_t& have = done[{kernel, dev}];
  if (bytes > have) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
    have = bytes;
  }
}


// ---------------------------------------------------------------------------
// K1: V0 = (float)(2 * u01(hash{seed, 'init', restart, row, col}) - 1)
// Layout [col][Bp]; consecutive threads take consecutive rows of one column.
// ---------------------------------------------------------------------------
// V is tile-major like the tape: [tile][col][tile_rows]; i walks it in
// memory order.
// The harvest's hardened input words hb[word][col] (bit = V >= 0,
// autodiff.cpp:292-297) come out of the same pass: a warp covers 32
// consecutive rows of one column (ncols * Bp and the stride are multiples of
// 32, so every warp stays converged).
__global__ void __launch_bounds__(kThreads)
k_init_v(float* __restrict__ V, int ncols, int Bp, int tile_rows, uint64_t prefix, long long row_offset,
         uint32_t* __restrict__ hb) {
  const long long total = static_cast<long long>(ncols) * Bp;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long tile = i / (static_cast<long long>(ncols) * tile_rows);
    const int within = static_cast<int>(i - tile * ncols * tile_rows);
    const int c = within / tile_rows;
    const int r = static_cast<int>(tile * tile_rows) + within % tile_rows;
    uint64_t h = fold(fold(prefix, static_cast<uint64_t>(row_offset + r)), static_cast<uint64_t>(c));
    double u = static_cast<double>(h >> 11) * 0x1.0p-53;  // u01, rng.hpp:28-30
    const float v = __double2float_rn(__dsub_rn(__dmul_rn(2.0, u), 1.0));
    V[i] = v;
    const uint32_t word = __ballot_sync(kFull, v >= 0.0f);
    if ((threadIdx.x & 31) == 0) hb[static_cast<size_t>(r >> 5) * ncols + c] = word;
  }
}

// Per-row restart (an extension: the reference restarts
// the whole batch, sampler.cpp:178-185).  Rows whose hardened assignment was
// valid but not new at the last harvest have converged onto a known
// solution; their logits are redrawn (u01 keyed by a per-iteration prefix,
// row and column, like init_soft_inputs), the others keep theirs.  The next
// step's backward epilogue re-hardens every row, so hb is not touched here.
__global__ void __launch_bounds__(kThreads)
k_reinit_rows(float* __restrict__ V, int ncols, int Bp, int tile_rows, uint64_t prefix, long long row_offset,
              const uint32_t* __restrict__ valid, const uint32_t* __restrict__ newmask) {
  const long long total = static_cast<long long>(ncols) * Bp;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long tile = i / (static_cast<long long>(ncols) * tile_rows);
    const int within = static_cast<int>(i - tile * ncols * tile_rows);
    const int c = within / tile_rows;
    const int r = static_cast<int>(tile * tile_rows) + within % tile_rows;
    const uint32_t stuck =
        newmask ? __ldg(valid + (r >> 5)) & ~__ldg(newmask + (r >> 5)) : __ldg(valid + (r >> 5));  // or a redraw mask
    if (!((stuck >> (r & 31)) & 1u)) continue;
    const uint64_t h = fold(fold(prefix, static_cast<uint64_t>(row_offset + r)), static_cast<uint64_t>(c));
    const double u = static_cast<double>(h >> 11) * 0x1.0p-53;
    V[i] = __double2float_rn(__dsub_rn(__dmul_rn(2.0, u), 1.0));
  }
}

// SGX_RESTART_REINIT_INVALID: the rows the next k_reinit_rows redraws --
// valid but not new, or invalid `min_age` or more GD steps after their last
// draw -- one thread per row, a warp per 32-row word.  age counts the steps
// since a row's draw (zeroed by every init); a redrawn row restarts at 0,
// every other row ages by the step that follows.
__global__ void __launch_bounds__(kThreads)
k_reinit_mask(const uint32_t* __restrict__ valid, const uint32_t* __restrict__ newmask, uint8_t* __restrict__ age,
              int W, int min_age, uint32_t* __restrict__ redraw) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;  // W * 32 threads exactly (kThreads divides 32)
  if (r >= W * 32) return;
  const int w = r >> 5, b = r & 31;
  const uint32_t v = (__ldg(valid + w) >> b) & 1u, n = (__ldg(newmask + w) >> b) & 1u;
  const int a = age[r];
  const bool go = (v && !n) || (!v && a >= min_age);
  age[r] = go ? 0 : static_cast<uint8_t>(a < 255 ? a + 1 : 255);
  const uint32_t m = __ballot_sync(kFull, go);
  if (b == 0) redraw[w] = m;
}

// Vector access of V consecutive samples of one tape row.
template <int V>
__device__ __forceinline__ void vload(const float* p, float (&o)[V]) {
  if constexpr (V == 1) {
    o[0] = *p;
  } else if constexpr (V == 2) {
    const float2 t = *reinterpret_cast<const float2*>(p);
    o[0] = t.x;
    o[1] = t.y;
  } else {
    const float4 t = *reinterpret_cast<const float4*>(p);
    o[0] = t.x;
    o[1] = t.y;
    o[2] = t.z;
    o[3] = t.w;
  }
}

template <int V>
__device__ __forceinline__ void vstore(float* p, const float (&o)[V]) {
  if constexpr (V == 1) {
    *p = o[0];
  } else if constexpr (V == 2) {
    *reinterpret_cast<float2*>(p) = make_float2(o[0], o[1]);
  } else {
    *reinterpret_cast<float4*>(p) = make_float4(o[0], o[1], o[2], o[3]);
  }
}

// autodiff.cpp:99-141, one node value.
__device__ __forceinline__ float gate_value(int code, float a, float b) {
  switch (code) {
    case SGX_CONST0: return 0.0f;
    case SGX_CONST1: return 1.0f;
    case SGX_BUF: return a;
    case SGX_NOT: return __fsub_rn(1.0f, a);
    case SGX_AND2: return __fmul_rn(a, b);
    case SGX_OR2: return __fsub_rn(1.0f, __fmul_rn(__fsub_rn(1.0f, a), __fsub_rn(1.0f, b)));
    case SGX_XOR2: return __fadd_rn(__fmul_rn(__fsub_rn(1.0f, a), b), __fmul_rn(a, __fsub_rn(1.0f, b)));
    case SGX_XNOR2: return __fadd_rn(__fmul_rn(a, b), __fmul_rn(__fsub_rn(1.0f, a), __fsub_rn(1.0f, b)));
    default: return 0.0f;
  }
}

// autodiff.cpp:225-277, one fan-out contribution pulled into acc.
__device__ __forceinline__ float pull(int ck, float acc, float g, float vo) {
  switch (ck) {
    case SGX_BUF: return __fadd_rn(acc, g);
    case SGX_NOT: return __fsub_rn(acc, g);
    case SGX_AND2: return __fadd_rn(acc, __fmul_rn(g, vo));
    case SGX_OR2: return __fadd_rn(acc, __fmul_rn(g, __fsub_rn(1.0f, vo)));
    case SGX_XOR2: return __fadd_rn(acc, __fmul_rn(g, __fsub_rn(1.0f, __fmul_rn(2.0f, vo))));
    case SGX_XNOR2: return __fadd_rn(acc, __fmul_rn(g, __fsub_rn(__fmul_rn(2.0f, vo), 1.0f)));
    default: return acc;
  }
}

// Folded-operand read: row << 1 | negate (a folded NOT reads 1 - x, exactly
// the reference's NOT, autodiff.cpp:112).
template <int V>
__device__ __forceinline__ void load_operand(const float* T, int enc, float (&o)[V]) {
  vload<V>(T + static_cast<size_t>(enc >> 1) * (32 * V), o);
  if (enc & 1) {
#pragma unroll
    for (int v = 0; v < V; ++v) o[v] = __fsub_rn(1.0f, o[v]);
  }
}

// Backward pull coefficients per consumer kind: contribution = g * (c0 + c1*v)
// with c1*v exact, so one fma reproduces the reference's (1 - v), (1 - 2v),
// (2v - 1), v, +1, -1 factors bit for bit (autodiff.cpp:225-277).
__constant__ float kPullC0[9] = {0.f, 0.f, 0.f, 1.f, -1.f, 0.f, 1.f, 1.f, -1.f};
__constant__ float kPullC1[9] = {0.f, 0.f, 0.f, 0.f, 0.f, 1.f, -1.f, -2.f, 2.f};

// ---------------------------------------------------------------------------
// K2: forward over the soft program (NOT/BUF folded into operand reads).  A
// CTA owns a tile of 32*V samples; its tape slice is [row][32*V] contiguous
// (tile-major), so one warp access is 128*V contiguous bytes and an address
// is one multiply-add.  kWarps warps split each level; __syncthreads()
// separates levels.  Work arrives as kind-homogeneous groups of <= kGroup
// ops: one uniform dispatch per group, then straight-line code that issues
// every operand load of the group before computing.
// ---------------------------------------------------------------------------
template <int V>
__global__ void __launch_bounds__(32 * kWarps)
k_forward(const int4* __restrict__ grp, const int2* __restrict__ lvl, int n_levels,
          const float* __restrict__ src, int ncols, float* tape, int n_rows, int src_is_prob,
          const uint64_t* __restrict__ exp_tab) {
  constexpr int TILE = 32 * V;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* T = tape + static_cast<size_t>(blockIdx.x) * n_rows * TILE + lane * V;
  const float* S = src + static_cast<size_t>(blockIdx.x) * ncols * TILE + lane * V;
  for (int l = 0; l < n_levels; ++l) {
    const int2 L = __ldg(lvl + l * kWarps + warp);
    for (int g = 0; g < L.y; ++g) {
      const int4* rec = grp + static_cast<size_t>(L.x + g) * kGroupRecs;
      const int4 h = __ldg(rec);
      int opd[2 * kGroup];
#pragma unroll
      for (int q = 0; q < kGroup / 2; ++q) {
        const int4 t = __ldg(rec + 1 + q);
        opd[4 * q] = t.x;
        opd[4 * q + 1] = t.y;
        opd[4 * q + 2] = t.z;
        opd[4 * q + 3] = t.w;
      }
      const int kind = h.x, n = h.y;
      float* out = T + static_cast<size_t>(h.z) * TILE;
      float x[kGroup][V], y[kGroup][V];
      if (kind >= SGX_AND2) {
#pragma unroll
        for (int k = 0; k < kGroup; ++k)
          if (k < n) {
            load_operand<V>(T, opd[2 * k], x[k]);
            load_operand<V>(T, opd[2 * k + 1], y[k]);
          }
#pragma unroll
        for (int k = 0; k < kGroup; ++k)
          if (k < n) {
            float r[V];
#pragma unroll
            for (int v = 0; v < V; ++v) r[v] = gate_value(kind, x[k][v], y[k][v]);
            vstore<V>(out + k * TILE, r);
          }
      } else if (kind == SGX_NOT || kind == SGX_BUF) {
#pragma unroll
        for (int k = 0; k < kGroup; ++k)
          if (k < n) load_operand<V>(T, opd[2 * k], x[k]);
#pragma unroll
        for (int k = 0; k < kGroup; ++k)
          if (k < n) {
            float r[V];
#pragma unroll
            for (int v = 0; v < V; ++v) r[v] = kind == SGX_NOT ? __fsub_rn(1.0f, x[k][v]) : x[k][v];
            vstore<V>(out + k * TILE, r);
          }
      } else if (kind == SGX_INPUT) {
#pragma unroll
        for (int k = 0; k < kGroup; ++k)
          if (k < n && opd[2 * k] >= 0) vload<V>(S + static_cast<size_t>(opd[2 * k]) * TILE, x[k]);
#pragma unroll
        for (int k = 0; k < kGroup; ++k)
          if (k < n) {
            float r[V];
#pragma unroll
            for (int v = 0; v < V; ++v)
              r[v] = opd[2 * k] < 0 ? 0.5f : (src_is_prob ? x[k][v] : sigmoid_ref(x[k][v], exp_tab));
            vstore<V>(out + k * TILE, r);
          }
      } else {  // CONST0 / CONST1
        float r[V];
#pragma unroll
        for (int v = 0; v < V; ++v) r[v] = kind == SGX_CONST1 ? 1.0f : 0.0f;
#pragma unroll
        for (int k = 0; k < kGroup; ++k)
          if (k < n) vstore<V>(out + k * TILE, r);
      }
    }
    __syncthreads();
  }
}

// END of a V column: dV = g p (1 - p) with p recomputed from V
// (autodiff.cpp:212-221), then V -= lr dV (gd_step, :285-290) -- or, for the
// parity tap, dV and dP out.  (Measured: an out-of-line version forces the
// ABI to keep the caller's live state in local memory and ran the C2
// backward 2.6x slower, so it stays inline.)
template <int V>
__device__ __forceinline__ void input_end(const float (&x)[V], const float (&acc)[V], float lr,
                                          const uint64_t* __restrict__ exp_tab, size_t at, float* Vp,
                                          float* dv_out, float* dp_out, float (&nv)[V]) {
  float dv[V];
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const float p = sigmoid_ref(x[v], exp_tab);
    dv[v] = __fmul_rn(__fmul_rn(acc[v], p), __fsub_rn(1.0f, p));
    nv[v] = __fsub_rn(x[v], __fmul_rn(lr, dv[v]));
  }
  if (dv_out) {
    vstore<V>(dv_out + at, dv);
    vstore<V>(dp_out + at, acc);
  } else {
    vstore<V>(Vp + at, nv);
  }
}

// Hardened input words from a tile's ballots: b[v] bit l = sample V*l + v of
// the tile; word k of the tile (rows 32k .. 32k+31) interleaves the k-th
// 32/V-bit slice of every b[v] with stride V.
__device__ __forceinline__ uint32_t spread4(uint32_t x) {  // bit m -> bit 4m (8 bits)
  x = (x | (x << 12)) & 0x000F000Fu;
  x = (x | (x << 6)) & 0x03030303u;
  return (x | (x << 3)) & 0x11111111u;
}
__device__ __forceinline__ uint32_t spread2(uint32_t x) {  // bit m -> bit 2m (16 bits)
  x = (x | (x << 8)) & 0x00FF00FFu;
  x = (x | (x << 4)) & 0x0F0F0F0Fu;
  x = (x | (x << 2)) & 0x33333333u;
  return (x | (x << 1)) & 0x55555555u;
}
template <int V>
__device__ __forceinline__ uint32_t pack_word(const uint32_t (&b)[V], int k) {
  if constexpr (V == 1) {
    return b[0];
  } else if constexpr (V == 2) {
    return spread2((b[0] >> (16 * k)) & 0xffffu) | (spread2((b[1] >> (16 * k)) & 0xffffu) << 1);
  } else {
    uint32_t w = 0u;
#pragma unroll
    for (int v = 0; v < 4; ++v) w |= spread4((b[v] >> (8 * k)) & 0xffu) << v;
    return w;
  }
}

// Edge-record decode tables (sgx_layout.hpp kR* flags).  kRecC[ck | in_sub<<4]
// = {c0a, c1a, c0b, c1b}: the pull factor c0 + c1*vo routed to acc (a) or to
// the SUB accumulator acc2 (b), zero on the other side.  kRecS[neg_other |
// first<<1 | sub_first<<2] = {ns, no, k, k2}: vo = ns*y + no, acc keeps factor
// k, acc2 keeps k2.  kRecE[sub_last | sub_not<<1]: acc += e * acc2.
__constant__ float4 kRecC[32] = {
    {0.0f, 0.0f, 0.0f, 0.0f}, {0.0f, 0.0f, 0.0f, 0.0f},  {0.0f, 0.0f, 0.0f, 0.0f},  {1.0f, 0.0f, 0.0f, 0.0f},
    {-1.0f, 0.0f, 0.0f, 0.0f}, {0.0f, 1.0f, 0.0f, 0.0f}, {1.0f, -1.0f, 0.0f, 0.0f}, {1.0f, -2.0f, 0.0f, 0.0f},
    {-1.0f, 2.0f, 0.0f, 0.0f}, {0.0f, 0.0f, 0.0f, 0.0f}, {0.0f, 0.0f, 0.0f, 0.0f},  {0.0f, 0.0f, 0.0f, 0.0f},
    {0.0f, 0.0f, 0.0f, 0.0f},  {0.0f, 0.0f, 0.0f, 0.0f}, {0.0f, 0.0f, 0.0f, 0.0f},  {0.0f, 0.0f, 0.0f, 0.0f},
    {0.0f, 0.0f, 0.0f, 0.0f},  {0.0f, 0.0f, 0.0f, 0.0f}, {0.0f, 0.0f, 0.0f, 0.0f},  {0.0f, 0.0f, 1.0f, 0.0f},
    {0.0f, 0.0f, -1.0f, 0.0f}, {0.0f, 0.0f, 0.0f, 1.0f}, {0.0f, 0.0f, 1.0f, -1.0f}, {0.0f, 0.0f, 1.0f, -2.0f},
    {0.0f, 0.0f, -1.0f, 2.0f}, {0.0f, 0.0f, 0.0f, 0.0f}, {0.0f, 0.0f, 0.0f, 0.0f},  {0.0f, 0.0f, 0.0f, 0.0f},
    {0.0f, 0.0f, 0.0f, 0.0f},  {0.0f, 0.0f, 0.0f, 0.0f}, {0.0f, 0.0f, 0.0f, 0.0f},  {0.0f, 0.0f, 0.0f, 0.0f}};
__constant__ float4 kRecS[8] = {{1.0f, 0.0f, 1.0f, 1.0f},  {-1.0f, 1.0f, 1.0f, 1.0f}, {1.0f, 0.0f, 0.0f, 1.0f},
                                {-1.0f, 1.0f, 0.0f, 1.0f}, {1.0f, 0.0f, 1.0f, 0.0f},  {-1.0f, 1.0f, 1.0f, 0.0f},
                                {1.0f, 0.0f, 0.0f, 0.0f},  {-1.0f, 1.0f, 0.0f, 0.0f}};
__constant__ float kRecE[4] = {0.0f, 1.0f, 0.0f, -1.0f};
// Pull factor and operand sign in one entry, indexed by consumer kind |
// kRNegOther >> 1: {c0, c1, ns, no} with vo = ns*y + no (y or 1 - y) and
// factor c0 + c1*vo (autodiff.cpp:225-277).
#define SGX_PULL4(c0, c1) {c0, c1, 1.0f, 0.0f}
#define SGX_PULL4N(c0, c1) {c0, c1, -1.0f, 1.0f}
__constant__ float4 kPull4[32] = {
    SGX_PULL4(0.f, 0.f),  SGX_PULL4(0.f, 0.f),  SGX_PULL4(0.f, 0.f),   SGX_PULL4(1.f, 0.f),
    SGX_PULL4(-1.f, 0.f), SGX_PULL4(0.f, 1.f),  SGX_PULL4(1.f, -1.f),  SGX_PULL4(1.f, -2.f),
    SGX_PULL4(-1.f, 2.f), SGX_PULL4(0.f, 0.f),  SGX_PULL4(0.f, 0.f),   SGX_PULL4(0.f, 0.f),
    SGX_PULL4(0.f, 0.f),  SGX_PULL4(0.f, 0.f),  SGX_PULL4(0.f, 0.f),   SGX_PULL4(0.f, 0.f),
    SGX_PULL4N(0.f, 0.f), SGX_PULL4N(0.f, 0.f), SGX_PULL4N(0.f, 0.f),  SGX_PULL4N(1.f, 0.f),
    SGX_PULL4N(-1.f, 0.f), SGX_PULL4N(0.f, 1.f), SGX_PULL4N(1.f, -1.f), SGX_PULL4N(1.f, -2.f),
    SGX_PULL4N(-1.f, 2.f), SGX_PULL4N(0.f, 0.f), SGX_PULL4N(0.f, 0.f),  SGX_PULL4N(0.f, 0.f),
    SGX_PULL4N(0.f, 0.f), SGX_PULL4N(0.f, 0.f), SGX_PULL4N(0.f, 0.f),  SGX_PULL4N(0.f, 0.f)};
#undef SGX_PULL4
#undef SGX_PULL4N

template <int V>
__device__ __forceinline__ void vload_nc(const float* p, float (&o)[V]) {
  if constexpr (V == 4) {
    const float4 t = __ldg(reinterpret_cast<const float4*>(p));
    o[0] = t.x;
    o[1] = t.y;
    o[2] = t.z;
    o[3] = t.w;
  } else {
    vload<V>(p, o);
  }
}

// Column epilogue of the backward, shared by the register and the staged
// kernels: dV = g p (1 - p) (autodiff.cpp:212-221), V -= lr dV (gd_step,
// :285-290), and the hardened new V into hb[word][col].
template <int V, int UC>
__device__ __forceinline__ void backward_columns(int warp, int lane, int tile, const float* A, float* Vp, size_t vbase,
                                                 int ncols, const int* __restrict__ col_row, float* dv_out,
                                                 float* dp_out, float lr, const uint64_t* __restrict__ exp_tab,
                                                 uint32_t* __restrict__ hb) {
  constexpr int TILE = 32 * V;
  for (int j0 = warp * UC; j0 < ncols; j0 += kWarps * UC) {
    int rw[UC];
    float x[UC][V], gg[UC][V];
#pragma unroll
    for (int q = 0; q < UC; ++q) {
      rw[q] = j0 + q < ncols ? __ldg(col_row + j0 + q) : -1;
      if (rw[q] >= 0) {
        vload<V>(A + static_cast<size_t>(rw[q]) * TILE, gg[q]);
        vload<V>(Vp + vbase + static_cast<size_t>(j0 + q) * TILE, x[q]);
      }
    }
#pragma unroll
    for (int q = 0; q < UC; ++q)
      if (rw[q] >= 0) {  // warp-uniform
        float nv[V];
        input_end<V>(x[q], gg[q], lr, exp_tab, vbase + static_cast<size_t>(j0 + q) * TILE, Vp, dv_out, dp_out, nv);
        if (hb) {  // harden (autodiff.cpp:292-297): bit = V >= 0, NaN -> 0
          uint32_t b[V];
#pragma unroll
          for (int v = 0; v < V; ++v) b[v] = __ballot_sync(kFull, nv[v] >= 0.0f);
          if (lane < V) hb[(static_cast<size_t>(tile) * V + lane) * ncols + j0 + q] = pack_word<V>(b, lane);
        }
      }
  }
}

// ---------------------------------------------------------------------------
// K3+K4+K5a: per-row loss, pull-CSR backward, fused GD step and harden.
// Same tile and level split as the forward, levels high to low; no atomics:
// every adjoint is produced once, by the warp that owns the node, summing
// its fan-out in the reference's order (seed, then consumers in descending
// id, a-slot first, a folded NOT/BUF consumer's own sum nested as a SUB
// run).  The micro-op control (BEGIN / SUB_BEGIN / SUB_END / END) rides as
// flag bits on the edge records, so every record runs the same branch-free
// arithmetic:
//   acc  = acc  * k  + seed        (k = 0 on a node's first record)
//   acc2 = acc2 * k2 + seed2       (k2 = 0 on a SUB run's first record)
//   vo = ns * T[other] + no;  acc += g * (c0a + c1a vo);  acc2 += g * (c0b + c1b vo)
//   acc += e * acc2                (e = -1 / +1 on a SUB run's last record)
// Bit-exactness: the c's, k's, ns/no and e are in {0, +-1, +-2}, so every
// product with them is exact and each fma rounds once, exactly like the
// reference's add / sub; adding a (signed) zero is the identity because an
// accumulator is never -0 (it starts at +0 and RN sums only give -0 from
// -0 + -0).  Seeds (output nodes, autodiff.cpp:206) take a rare uniform
// branch.  Column-input adjoints are stored like any other and the V update
// (dV = g p (1 - p), V -= lr dV) runs as an epilogue over the tile's columns,
// which also hardens the new V into the harvest's input words (hb).
// ---------------------------------------------------------------------------
#ifndef SGX_REC_UC
#define SGX_REC_UC 2
#endif
#ifndef SGX_REC_U
#define SGX_REC_U 4  // records per chunk at 4 samples per lane (C2 backward: 4 -> 40.7, 6 -> 41.9, 8 -> 46.2 ms per 5 restarts)
#endif
template <int V, int U>
__global__ void __launch_bounds__(32 * kWarps, (64 / (V * kWarps)) > 0 ? 64 / (V * kWarps) : 1)
k_backward_rec(const int4* __restrict__ rec, const int2* __restrict__ lvl, int n_levels,
               const float* __restrict__ tape, float* adj, float* Vp, int ncols, int n_rows,
               const int* __restrict__ col_row, float* dv_out, float* dp_out, float lr,
               const int* __restrict__ out_enc, const uint8_t* __restrict__ out_tgt, int n_out,
               float* __restrict__ row_loss, const uint64_t* __restrict__ exp_tab, uint32_t* __restrict__ hb,
               int n_tiles) {
  constexpr int TILE = 32 * V;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const size_t tbase = static_cast<size_t>(tile) * n_rows * TILE + lane * V;
    const float* T = tape + tbase;
    float* A = adj + tbase;
    const size_t vbase = static_cast<size_t>(tile) * ncols * TILE + lane * V;
    if (row_loss && warp == 0) {  // loss (autodiff.cpp:160-166): outputs in order
      float l[V];
#pragma unroll
      for (int v = 0; v < V; ++v) l[v] = 0.0f;
      for (int m = 0; m < n_out; ++m) {
        float yv[V];
        load_operand<V>(T, __ldg(out_enc + m), yv);
        const float t = __ldg(out_tgt + m) ? 1.0f : 0.0f;
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const float d = __fsub_rn(yv[v], t);
          l[v] = __fadd_rn(l[v], __fmul_rn(d, d));
        }
      }
      vstore<V>(row_loss + static_cast<size_t>(tile) * TILE + lane * V, l);
    }
    float acc[V], acc2[V];
#pragma unroll
    for (int v = 0; v < V; ++v) acc[v] = acc2[v] = 0.0f;
    for (int li = 0; li < n_levels; ++li) {
      const int2 L = __ldg(lvl + li * kWarps + warp);
      for (int c = 0; c < L.y; c += U) {
        int4 r[U];
#pragma unroll
        for (int k = 0; k < U; ++k) r[k] = c + k < L.y ? __ldg(rec + L.x + c + k) : make_int4(0, -1, -1, 0);
        float g[U][V], y[U][V];
#pragma unroll
        for (int k = 0; k < U; ++k) {
#pragma unroll
          for (int v = 0; v < V; ++v) g[k][v] = y[k][v] = 0.0f;
          if (r[k].y >= 0) vload<V>(A + static_cast<size_t>(r[k].y) * TILE, g[k]);
          if (r[k].z >= 0) vload_nc<V>(T + static_cast<size_t>(r[k].z) * TILE, y[k]);
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
          const int f = r[k].x;
          const float4 C = kRecC[f & 0x1f];
          const float4 S = kRecS[(f >> 5) & 0x7];
          const float e = kRecE[(f >> 8) & 0x3];
          float sd[V], sd2[V];
#pragma unroll
          for (int v = 0; v < V; ++v) sd[v] = sd2[v] = 0.0f;
          if (f & (kRSeed | kRSubSeed)) {  // adj[out] += 2 (y - t) on a zero adjoint (autodiff.cpp:206)
            float yw[V];
            vload_nc<V>(T + static_cast<size_t>(r[k].w) * TILE, yw);
            const float t = (f & kRTarget) ? 1.0f : 0.0f, t2 = (f & kRSubTarget) ? 1.0f : 0.0f;
#pragma unroll
            for (int v = 0; v < V; ++v) {
              if (f & kRSeed) sd[v] = __fadd_rn(0.0f, __fmul_rn(2.0f, __fsub_rn(yw[v], t)));
              if (f & kRSubSeed) {
                const float ys = (f & kRNegSelf) ? __fsub_rn(1.0f, yw[v]) : yw[v];
                sd2[v] = __fadd_rn(0.0f, __fmul_rn(2.0f, __fsub_rn(ys, t2)));
              }
            }
          }
#pragma unroll
          for (int v = 0; v < V; ++v) {
            acc[v] = __fmaf_rn(acc[v], S.z, sd[v]);
            acc2[v] = __fmaf_rn(acc2[v], S.w, sd2[v]);
            const float vo = __fmaf_rn(S.x, y[k][v], S.y);
            const float fa = __fmaf_rn(C.y, vo, C.x), fb = __fmaf_rn(C.w, vo, C.z);
            acc[v] = __fadd_rn(acc[v], __fmul_rn(g[k][v], fa));
            acc2[v] = __fadd_rn(acc2[v], __fmul_rn(g[k][v], fb));
            acc[v] = __fmaf_rn(e, acc2[v], acc[v]);
          }
          if (f & kRLast) vstore<V>(A + static_cast<size_t>(r[k].w) * TILE, acc);
        }
      }
      __syncthreads();
    }
    // V columns: dV = g p (1 - p) (autodiff.cpp:212-221), V -= lr dV (gd_step, :285-290).
    constexpr int UC = V == 4 ? SGX_REC_UC : 1;  // narrower tiles run at 16/V CTAs per SM: no room
    backward_columns<V, UC>(warp, lane, tile, A, Vp, vbase, ncols, col_row, dv_out, dp_out, lr, exp_tab, hb);
    if (n_tiles > static_cast<int>(gridDim.x)) __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// The forward with every operand row staged through shared memory by cp.async
// (LDGSTS, 16 B per lane = the lane's 4 samples).  Each warp keeps kStages
// groups in flight without spending registers on them, so the loads of the
// next groups overlap the arithmetic of the current one.  Lanes only ever
// read their own staged bytes, so per-thread cp.async.wait_group is the only
// synchronisation inside a level.
// ---------------------------------------------------------------------------
#ifndef SGX_STAGES
#define SGX_STAGES 3
#endif
constexpr int kStages = SGX_STAGES;      // groups in flight per warp
constexpr int kSlots = 2 * kGroup;       // staged rows per stage
constexpr int kAsyncSmem = kWarps * kStages * kSlots * 32 * 16;  // bytes per CTA

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
// L2 eviction-priority policies (createpolicy): tape rows the backward
// streams are read evict_first, adjoint rows it will re-read soon are stored
// evict_last, so the L2 keeps adjoints rather than tape.
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ void cp_async16_hint(void* smem, const void* gmem, uint64_t pol) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void st_hint(float* p, const float (&o)[4], uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;\n" ::"l"(p), "f"(o[0]), "f"(o[1]),
               "f"(o[2]), "f"(o[3]), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void discard_l2(const void* p) {
  asm volatile("discard.global.L2 [%0], 128;\n" ::"l"(p) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

__device__ __forceinline__ void f4(const float4& t, float (&o)[4]) {
  o[0] = t.x;
  o[1] = t.y;
  o[2] = t.z;
  o[3] = t.w;
}

// Folded NOT on read without a branch: fma(-1, x, 1) rounds 1 - x exactly as
// __fsub_rn(1, x) does; fma(1, x, 0) = x.
__device__ __forceinline__ float fold_read(float x, int enc) {
  const bool neg = enc & 1;
  return __fmaf_rn(neg ? -1.0f : 1.0f, x, neg ? 1.0f : 0.0f);
}

template <int KIND>
__device__ __forceinline__ void group_binary(const float4* base, const int (&opd)[8], int n, float* out) {
#pragma unroll
  for (int k = 0; k < kGroup; ++k) {
    if (k >= n) break;
    float a[4], b[4], r[4];
    f4(base[(2 * k) * 32], a);
    f4(base[(2 * k + 1) * 32], b);
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const float x = fold_read(a[v], opd[2 * k]), y = fold_read(b[v], opd[2 * k + 1]);
      if constexpr (KIND == SGX_AND2) r[v] = __fmul_rn(x, y);
      if constexpr (KIND == SGX_OR2) r[v] = __fsub_rn(1.0f, __fmul_rn(__fsub_rn(1.0f, x), __fsub_rn(1.0f, y)));
      if constexpr (KIND == SGX_XOR2)
        r[v] = __fadd_rn(__fmul_rn(__fsub_rn(1.0f, x), y), __fmul_rn(x, __fsub_rn(1.0f, y)));
      if constexpr (KIND == SGX_XNOR2)
        r[v] = __fadd_rn(__fmul_rn(x, y), __fmul_rn(__fsub_rn(1.0f, x), __fsub_rn(1.0f, y)));
    }
    vstore<4>(out + k * 128, r);
  }
}

template <bool NOT>
__device__ __forceinline__ void group_unary(const float4* base, const int (&opd)[8], int n, float* out) {
#pragma unroll
  for (int k = 0; k < kGroup; ++k) {
    if (k >= n) break;
    float a[4], r[4];
    f4(base[(2 * k) * 32], a);
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const float x = fold_read(a[v], opd[2 * k]);
      r[v] = NOT ? __fsub_rn(1.0f, x) : x;
    }
    vstore<4>(out + k * 128, r);
  }
}

__global__ void __launch_bounds__(32 * kWarps)
k_forward_async(const int4* __restrict__ grp, const int2* __restrict__ lvl, int n_levels,
                const float* __restrict__ src, int ncols, float* tape, int n_rows, int src_is_prob,
                const uint64_t* __restrict__ exp_tab, int n_tiles) {
  constexpr int TILE = 128;
  extern __shared__ float4 stage_mem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* T = nullptr;        // this tile's tape slice (set per tile below)
  const float* S = nullptr;  // this tile's V slice
  float4* my = stage_mem + warp * kStages * kSlots * 32 + lane;  // slot (d, j): my[(d*kSlots + j) * 32]
  auto issue = [&](int g, int d) {
    const int4* rec = grp + static_cast<size_t>(g) * kGroupRecs;
    const int4 h = __ldg(rec), o0 = __ldg(rec + 1), o1 = __ldg(rec + 2);
    const int opd[8] = {o0.x, o0.y, o0.z, o0.w, o1.x, o1.y, o1.z, o1.w};
    const int kind = h.x, n = h.y;
    float4* base = my + d * kSlots * 32;
#pragma unroll
    for (int k = 0; k < kGroup; ++k) {
      if (k >= n) break;
      if (kind >= SGX_AND2) {
        cp_async16(base + (2 * k) * 32, T + static_cast<size_t>(opd[2 * k] >> 1) * TILE);
        cp_async16(base + (2 * k + 1) * 32, T + static_cast<size_t>(opd[2 * k + 1] >> 1) * TILE);
      } else if (kind == SGX_NOT || kind == SGX_BUF) {
        cp_async16(base + (2 * k) * 32, T + static_cast<size_t>(opd[2 * k] >> 1) * TILE);
      } else if (kind == SGX_INPUT && opd[2 * k] >= 0) {
        cp_async16(base + (2 * k) * 32, S + static_cast<size_t>(opd[2 * k]) * TILE);
      }
    }
    cp_async_commit();
  };
  // Persistent over tiles when the grid is smaller than the tile count.
  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
  T = tape + static_cast<size_t>(tile) * n_rows * TILE + lane * 4;
  S = src + static_cast<size_t>(tile) * ncols * TILE + lane * 4;
  for (int l = 0; l < n_levels; ++l) {
    const int2 L = __ldg(lvl + l * kWarps + warp);
#pragma unroll
    for (int i = 0; i < kStages - 1; ++i) {
      if (i < L.y)
        issue(L.x + i, i);
      else
        cp_async_commit();
    }
    for (int i = 0; i < L.y; ++i) {
      const int nxt = i + kStages - 1;
      if (nxt < L.y)
        issue(L.x + nxt, nxt % kStages);
      else
        cp_async_commit();
      cp_async_wait<kStages - 1>();
      const int4* rec = grp + static_cast<size_t>(L.x + i) * kGroupRecs;
      const int4 h = __ldg(rec), o0 = __ldg(rec + 1), o1 = __ldg(rec + 2);
      const int opd[8] = {o0.x, o0.y, o0.z, o0.w, o1.x, o1.y, o1.z, o1.w};
      const int kind = h.x, n = h.y;
      const float4* base = my + (i % kStages) * kSlots * 32;
      float* out = T + static_cast<size_t>(h.z) * TILE;
      // One dispatch per group; the per-sample loops below are branch-free.
      switch (kind) {
        case SGX_AND2: group_binary<SGX_AND2>(base, opd, n, out); break;
        case SGX_OR2: group_binary<SGX_OR2>(base, opd, n, out); break;
        case SGX_XOR2: group_binary<SGX_XOR2>(base, opd, n, out); break;
        case SGX_XNOR2: group_binary<SGX_XNOR2>(base, opd, n, out); break;
        case SGX_NOT: group_unary<true>(base, opd, n, out); break;
        case SGX_BUF: group_unary<false>(base, opd, n, out); break;
        case SGX_INPUT:
#pragma unroll
          for (int k = 0; k < kGroup; ++k) {
            if (k >= n) break;
            float a[4] = {0.0f, 0.0f, 0.0f, 0.0f}, r[4];
            if (opd[2 * k] >= 0) f4(base[(2 * k) * 32], a);
#pragma unroll
            for (int v = 0; v < 4; ++v)
              r[v] = opd[2 * k] < 0 ? 0.5f : (src_is_prob ? a[v] : sigmoid_ref(a[v], exp_tab));
            vstore<4>(out + k * TILE, r);
          }
          break;
        default: {
          const float c = kind == SGX_CONST1 ? 1.0f : 0.0f;
          const float r[4] = {c, c, c, c};
#pragma unroll
          for (int k = 0; k < kGroup; ++k) {
            if (k >= n) break;
            vstore<4>(out + k * TILE, r);
          }
        }
      }
    }
    __syncthreads();
  }
  }  // tile loop
}

// ---------------------------------------------------------------------------
// The backward with its edge operands staged through shared memory by
// cp.async.  Same records, order and arithmetic as k_backward_rec (so the
// same bits); what changes is the memory pipeline.  Per warp, a ring of BS
// stages of BU records each: the adjoint row of the consumer (g) and the
// value row of the other operand (y) of every record land in the lane's own
// 16-byte slots while the warp computes BS-1 chunks behind, so a level's
// loads are all in flight instead of one chunk's.  The records of the chunk
// after the next issue are prefetched into registers, so issuing never waits
// on a record load either.  Only the level barrier drains the ring: the next
// level's adjoint reads depend on this level's stores.
// ---------------------------------------------------------------------------
#ifndef SGX_BU
#define SGX_BU 4
#endif
#ifndef SGX_BS
#define SGX_BS 3
#endif
#ifndef SGX_HINT_Y
#define SGX_HINT_Y 1
#endif
#ifndef SGX_FWD_HINT
#define SGX_FWD_HINT 1  // forward: last reads of a row evict_first
#endif
#ifndef SGX_HINT_ADJ
#define SGX_HINT_ADJ 1
#endif
constexpr int kBU = SGX_BU, kBS = SGX_BS;
constexpr int kBwdSmem = kWarps * kBS * kBU * 2 * 32 * 16;  // bytes per CTA

// One backward edge record (sgx_layout.hpp kR* flags) on a lane's 4 samples,
// g = adjoint row of the consumer, y = value row of the other operand (both
// staged on chip).  Plain edges take a 4-op path; seeds, SUB runs and
// edge-less records branch (warp-uniform) and follow the reference's
// operations exactly.
__device__ __forceinline__ void backward_record(const int4 r, const float4 gs, const float4 ys, float (&acc)[4],
                                                float (&acc2)[4], const float* T, float* A, uint64_t pol_last) {
  constexpr int V = 4, TILE = 128;
  const int f = r.x;
  float g[V], y[V];
  f4(gs, g);
  f4(ys, y);
          // Pull factor c0 + c1*vo of the consumer kind, vo = y or 1 - y
          // (other operand read through a folded NOT): both fmas round
          // exactly as the reference's (1 - v), (1 - 2v), ... (c1*vo exact).
          const float4 C = kPull4[(f & 0xf) | ((f >> 1) & 0x10)];  // {c0, c1, ns, no}
          const float ns = C.z, no = C.w;
          if (!(f & kRSlow)) {  // plain edge into this node's adjoint (most records; the
                                // accumulator is already +0 at a node's first record)
#pragma unroll
            for (int v = 0; v < V; ++v) {
              const float fa = __fmaf_rn(C.y, __fmaf_rn(ns, y[v], no), C.x);
              acc[v] = __fadd_rn(acc[v], __fmul_rn(g[v], fa));
            }
          } else if (f & kRSubOne) {  // a one-edge, unseeded SUB run: adj[j] = +0 + g*fa (the reference's
                                      // fresh zero adjoint, autodiff.cpp:191), then acc -/+= adj[j] (:225-233)
#pragma unroll
            for (int v = 0; v < V; ++v) {
              const float fa = __fmaf_rn(C.y, __fmaf_rn(ns, y[v], no), C.x);
              const float sj = __fadd_rn(0.0f, __fmul_rn(g[v], fa));
              acc[v] = (f & kRSubNot) ? __fsub_rn(acc[v], sj) : __fadd_rn(acc[v], sj);
            }
          } else {  // seeds, longer SUB runs (folded NOT/BUF consumers), empty nodes
            if (f & (kRFirst | kRSubFirst)) {
              float sd[V] = {0.0f, 0.0f, 0.0f, 0.0f}, sd2[V] = {0.0f, 0.0f, 0.0f, 0.0f};
              if (f & (kRSeed | kRSubSeed)) {  // adj[out] += 2 (y - t) on a zero adjoint (autodiff.cpp:206)
                float yw[V];
                vload_nc<V>(T + static_cast<size_t>(r.w) * TILE, yw);
                const float t = (f & kRTarget) ? 1.0f : 0.0f, t2 = (f & kRSubTarget) ? 1.0f : 0.0f;
#pragma unroll
                for (int v = 0; v < V; ++v) {
                  if (f & kRSeed) sd[v] = __fadd_rn(0.0f, __fmul_rn(2.0f, __fsub_rn(yw[v], t)));
                  if (f & kRSubSeed) {
                    const float ys = (f & kRNegSelf) ? __fsub_rn(1.0f, yw[v]) : yw[v];
                    sd2[v] = __fadd_rn(0.0f, __fmul_rn(2.0f, __fsub_rn(ys, t2)));
                  }
                }
              }
#pragma unroll
              for (int v = 0; v < V; ++v) {
                if (f & kRFirst) acc[v] = sd[v];
                if (f & kRSubFirst) acc2[v] = sd2[v];
              }
            }
            if (r.y >= 0) {
#pragma unroll
              for (int v = 0; v < V; ++v) {
                const float t = __fmul_rn(g[v], __fmaf_rn(C.y, __fmaf_rn(ns, y[v], no), C.x));
                if (f & kRInSub)
                  acc2[v] = __fadd_rn(acc2[v], t);
                else
                  acc[v] = __fadd_rn(acc[v], t);
              }
            }
            if (f & kRSubLast) {  // adj[i] += -adj[j] (NOT) / +adj[j] (BUF), autodiff.cpp:225-233
#pragma unroll
              for (int v = 0; v < V; ++v)
                acc[v] = (f & kRSubNot) ? __fsub_rn(acc[v], acc2[v]) : __fadd_rn(acc[v], acc2[v]);
            }
          }
          if (f & kRLast) {
            if (SGX_HINT_ADJ)
              st_hint(A + static_cast<size_t>(r.w) * TILE, acc, pol_last);
            else
              vstore<V>(A + static_cast<size_t>(r.w) * TILE, acc);
            // the next node starts from +0: every emitted node run ends with
            // kRLast, and a seed 0 + x is never -0, so this equals the
            // reference's fresh zero adjoint (autodiff.cpp:191).  Chunk
            // padding records are kRSlow without an edge, so they never
            // touch the accumulator (a stale slot times zero could be NaN).
#pragma unroll
            for (int v = 0; v < V; ++v) acc[v] = 0.0f;
          }
}

__global__ void __launch_bounds__(32 * kWarps)
k_backward_async(const int4* __restrict__ rec, const int2* __restrict__ lvl, int n_levels,
                 const float* __restrict__ tape, float* adj, float* Vp, int ncols, int n_rows,
                 const int* __restrict__ col_row, float* dv_out, float* dp_out, float lr,
                 const int* __restrict__ out_enc, const uint8_t* __restrict__ out_tgt, int n_out,
                 float* __restrict__ row_loss, const uint64_t* __restrict__ exp_tab, uint32_t* __restrict__ hb,
                 int n_tiles, const int* __restrict__ dead, const int2* __restrict__ dead_lvl) {
  constexpr int V = 4, TILE = 128;
  extern __shared__ float4 bstage[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float4* my = bstage + warp * kBS * kBU * 2 * 32 + lane;  // slot (d, k, j): my[((d * kBU + k) * 2 + j) * 32]
  const uint64_t pol_first = policy_evict_first(), pol_last = policy_evict_last();
  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const size_t tbase = static_cast<size_t>(tile) * n_rows * TILE + lane * V;
    const float* T = tape + tbase;
    float* A = adj + tbase;
    float* Abase = adj + static_cast<size_t>(tile) * n_rows * TILE;
    const size_t vbase = static_cast<size_t>(tile) * ncols * TILE + lane * V;
    if (row_loss && warp == 0) {  // loss (autodiff.cpp:160-166): outputs in order
      float l[V] = {0.0f, 0.0f, 0.0f, 0.0f};
      for (int m = 0; m < n_out; ++m) {
        float yv[V];
        load_operand<V>(T, __ldg(out_enc + m), yv);
        const float t = __ldg(out_tgt + m) ? 1.0f : 0.0f;
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const float d = __fsub_rn(yv[v], t);
          l[v] = __fadd_rn(l[v], __fmul_rn(d, d));
        }
      }
      vstore<V>(row_loss + static_cast<size_t>(tile) * TILE + lane * V, l);
    }
    float acc[V], acc2[V];
#pragma unroll
    for (int v = 0; v < V; ++v) acc[v] = acc2[v] = 0.0f;
    for (int li = 0; li < n_levels; ++li) {
      const int2 L = __ldg(lvl + li * kWarps + warp);
      const int nch = (L.y + kBU - 1) / kBU;
      const int4* R = rec + L.x;
      int4 pre[kBU];  // records of the next chunk to issue
      auto fetch = [&](int ch) {
#pragma unroll
        for (int k = 0; k < kBU; ++k)
          pre[k] = ch * kBU + k < L.y ? __ldg(R + ch * kBU + k) : make_int4(0, -1, -1, 0);
      };
      auto issue = [&](int d) {
        float4* base = my + d * kBU * 2 * 32;
#pragma unroll
        for (int k = 0; k < kBU; ++k) {
          if (pre[k].y >= 0) cp_async16(base + (2 * k) * 32, A + static_cast<size_t>(pre[k].y) * TILE);
          if (pre[k].z >= 0) {
            if (SGX_HINT_Y)
              cp_async16_hint(base + (2 * k + 1) * 32, T + static_cast<size_t>(pre[k].z) * TILE, pol_first);
            else
              cp_async16(base + (2 * k + 1) * 32, T + static_cast<size_t>(pre[k].z) * TILE);
          } else {
            base[(2 * k + 1) * 32] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);  // unary consumer: c1 * 0
          }
        }
        cp_async_commit();
      };
      fetch(0);
#pragma unroll
      for (int i = 0; i < kBS - 1; ++i) {
        if (i < nch) {
          issue(i);
          fetch(i + 1);
        } else {
          cp_async_commit();
        }
      }
      for (int ch = 0; ch < nch; ++ch) {
        const int nxt = ch + kBS - 1;
        if (nxt < nch) {
          issue(nxt % kBS);
          fetch(nxt + 1);
        } else {
          cp_async_commit();
        }
        cp_async_wait<kBS - 1>();
        const float4* base = my + (ch % kBS) * kBU * 2 * 32;
#pragma unroll
        for (int k = 0; k < kBU; ++k) {
          const int4 r = ch * kBU + k < L.y ? __ldg(R + ch * kBU + k) : make_int4(kRSlow, -1, -1, 0);  // inert pad
          backward_record(r, base[(2 * k) * 32], base[(2 * k + 1) * 32], acc, acc2, T, A, pol_last);
        }
      }
      __syncthreads();
      if (dead) {  // adjoints whose last reader ran in this pass: drop from L2, no write-back
        const int2 D = __ldg(dead_lvl + li);
        for (int i = threadIdx.x; i < 4 * D.y; i += 32 * kWarps)
          discard_l2(Abase + static_cast<size_t>(__ldg(dead + D.x + (i >> 2))) * TILE + (i & 3) * 32);
      }
    }
    backward_columns<V, SGX_REC_UC>(warp, lane, tile, A, Vp, vbase, ncols, col_row, dv_out, dp_out, lr, exp_tab, hb);
    __syncthreads();
    if (dead) {
      for (int i = threadIdx.x; i < 4 * ncols; i += 32 * kWarps) {
        const int rw = __ldg(col_row + (i >> 2));
        if (rw >= 0) discard_l2(Abase + static_cast<size_t>(rw) * TILE + (i & 3) * 32);
      }
    }
  }
}


// ---------------------------------------------------------------------------
// TMA-fed backward.  Like k_backward_async, but the control stream is on
// chip too: each pass's block (sgx_layout.hpp sblk: header, per-warp record
// ranges, records, the previous pass's dead adjoint rows) arrives by one
// cp.async.bulk into a double buffer, completion on an mbarrier, issued one
// pass ahead by thread 0.  Record reads (issue side and compute side) and
// the dead-row list are shared-memory broadcasts, so no load in the loop
// waits on L2 except the staged data rows themselves.
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* m, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(m)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* m, unsigned phase) {
  unsigned done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(m)), "r"(phase)
        : "memory");
  } while (!done);
}
// Thread-0 only: bring n4 int4s at src into dst, completing on m.
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned n4, uint64_t* m) {
  const unsigned bytes = n4 * 16u;
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(m)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(m))
               : "memory");
}

template <int BS>
__global__ void __launch_bounds__(32 * kWarps, 16 / kWarps)
k_backward_tma(const int4* __restrict__ sblk, int blk0_n4, int blk_max, int n_levels, const float* __restrict__ tape,
               float* adj, float* Vp, int ncols, int n_rows, const int* __restrict__ col_row, float* dv_out,
               float* dp_out, float lr, const int* __restrict__ out_enc, const uint8_t* __restrict__ out_tgt,
               int n_out, float* __restrict__ row_loss, const uint64_t* __restrict__ exp_tab,
               uint32_t* __restrict__ hb, int n_tiles, const int* __restrict__ tail_dead, int n_tail_dead,
               int discard) {
  constexpr int V = 4, TILE = 128;
  extern __shared__ __align__(128) float4 tstage[];
  __shared__ __align__(8) uint64_t mbar[2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float4* my = tstage + warp * BS * kBU * 2 * 32 + lane;  // slot (d, k, j): my[((d * kBU + k) * 2 + j) * 32]
  int4* const blk0 = reinterpret_cast<int4*>(tstage + kWarps * BS * kBU * 2 * 32);  // buffer b: blk0 + b * blk_max
  const uint64_t pol_first = policy_evict_first(), pol_last = policy_evict_last();
  if (threadIdx.x == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  unsigned phase = 0u;  // bit b: parity of buffer b's next completion
  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    if (threadIdx.x == 0) bulk_load(blk0, sblk, blk0_n4, &mbar[0]);
    const size_t tbase = static_cast<size_t>(tile) * n_rows * TILE + lane * V;
    const float* T = tape + tbase;
    float* A = adj + tbase;
    float* Abase = adj + static_cast<size_t>(tile) * n_rows * TILE;
    const size_t vbase = static_cast<size_t>(tile) * ncols * TILE + lane * V;
    if (row_loss && warp == 0) {  // loss (autodiff.cpp:160-166): outputs in order
      float l[V] = {0.0f, 0.0f, 0.0f, 0.0f};
      for (int m = 0; m < n_out; ++m) {
        float yv[V];
        load_operand<V>(T, __ldg(out_enc + m), yv);
        const float t = __ldg(out_tgt + m) ? 1.0f : 0.0f;
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const float d = __fsub_rn(yv[v], t);
          l[v] = __fadd_rn(l[v], __fmul_rn(d, d));
        }
      }
      vstore<V>(row_loss + static_cast<size_t>(tile) * TILE + lane * V, l);
    }
    float acc[V], acc2[V];
#pragma unroll
    for (int v = 0; v < V; ++v) acc[v] = acc2[v] = 0.0f;
    for (int li = 0; li < n_levels; ++li) {
      const int b = li & 1;
      mbar_wait(mbar + b, (phase >> b) & 1u);
      phase ^= 1u << b;
      const int4* B = blk0 + b * blk_max;
      const int4 H = B[0];  // {dead_rel, n_dead, next_start, next_n4}
      if (threadIdx.x == 0 && li + 1 < n_levels) bulk_load(blk0 + (b ^ 1) * blk_max, sblk + H.z, H.w, mbar + (b ^ 1));
      if (discard) {  // rows whose last reader ran in the previous pass (barrier passed): no write-back
        const int* D = reinterpret_cast<const int*>(B + H.x);
        for (int i = threadIdx.x; i < 4 * H.y; i += 32 * kWarps)
          discard_l2(Abase + static_cast<size_t>(D[i >> 2]) * TILE + (i & 3) * 32);
      }
      const int2 W = reinterpret_cast<const int2*>(B + 1)[warp];  // {first_rel, count}
      const int4* R = B + W.x;
      const int nch = (W.y + kBU - 1) / kBU;
      auto issue = [&](int ch, int d) {
        float4* base = my + d * kBU * 2 * 32;
#pragma unroll
        for (int k = 0; k < kBU; ++k) {
          const int4 q = ch * kBU + k < W.y ? R[ch * kBU + k] : make_int4(0, -1, -1, 0);
          if (q.y >= 0) cp_async16(base + (2 * k) * 32, A + static_cast<size_t>(q.y) * TILE);
          if (q.z >= 0 && SGX_HINT_Y && !(q.x & kRYKeep))
            cp_async16_hint(base + (2 * k + 1) * 32, T + static_cast<size_t>(q.z) * TILE, pol_first);
          else if (q.z >= 0)
            cp_async16(base + (2 * k + 1) * 32, T + static_cast<size_t>(q.z) * TILE);
          else
            base[(2 * k + 1) * 32] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);  // unary consumer: c1 * 0
        }
        cp_async_commit();
      };
#pragma unroll
      for (int i = 0; i < BS - 1; ++i) {
        if (i < nch)
          issue(i, i);
        else
          cp_async_commit();
      }
      for (int ch = 0; ch < nch; ++ch) {
        const int nxt = ch + BS - 1;
        if (nxt < nch)
          issue(nxt, nxt % BS);
        else
          cp_async_commit();
        cp_async_wait<BS - 1>();
        const float4* base = my + (ch % BS) * kBU * 2 * 32;
#pragma unroll
        for (int k = 0; k < kBU; ++k) {
          const int4 r = ch * kBU + k < W.y ? R[ch * kBU + k] : make_int4(kRSlow, -1, -1, 0);  // inert pad
          backward_record(r, base[(2 * k) * 32], base[(2 * k + 1) * 32], acc, acc2, T, A, pol_last);
        }
      }
      __syncthreads();
    }
    backward_columns<V, SGX_REC_UC>(warp, lane, tile, A, Vp, vbase, ncols, col_row, dv_out, dp_out, lr, exp_tab, hb);
    __syncthreads();
    if (discard) {  // the last pass's dead rows and the column inputs (read by the epilogue)
      for (int i = threadIdx.x; i < 4 * n_tail_dead; i += 32 * kWarps)
        discard_l2(Abase + static_cast<size_t>(__ldg(tail_dead + (i >> 2))) * TILE + (i & 3) * 32);
      for (int i = threadIdx.x; i < 4 * ncols; i += 32 * kWarps) {
        const int rw = __ldg(col_row + (i >> 2));
        if (rw >= 0) discard_l2(Abase + static_cast<size_t>(rw) * TILE + (i & 3) * 32);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// TMA-fed forward: k_forward_async's staged operand pipeline with the group
// records on chip -- each level's block (sgx_layout.hpp fblk: header, warp
// ranges, groups) arrives by cp.async.bulk one level ahead, so neither the
// issue side nor the compute side waits on a record load.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(32 * kWarps)
k_forward_tma(const int4* __restrict__ fblk, int blk0_n4, int blk_max, int n_levels, const float* __restrict__ src,
              int ncols, float* tape, int n_rows, int src_is_prob, const uint64_t* __restrict__ exp_tab,
              int n_tiles) {
  constexpr int TILE = 128;
  extern __shared__ __align__(128) float4 fstage[];
  __shared__ __align__(8) uint64_t mbar[2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float4* my = fstage + warp * kStages * kSlots * 32 + lane;  // slot (d, j): my[(d*kSlots + j) * 32]
  int4* const blk0 = reinterpret_cast<int4*>(fstage + kWarps * kStages * kSlots * 32);
  const uint64_t pol = policy_evict_first();
  auto load_row = [](float4* dst, const float* src, int last, uint64_t p) {
    if (SGX_FWD_HINT && last)
      cp_async16_hint(dst, src, p);
    else
      cp_async16(dst, src);
  };
  if (threadIdx.x == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  unsigned phase = 0u;
  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    if (threadIdx.x == 0) bulk_load(blk0, fblk, blk0_n4, &mbar[0]);
    float* T = tape + static_cast<size_t>(tile) * n_rows * TILE + lane * 4;
    const float* S = src + static_cast<size_t>(tile) * ncols * TILE + lane * 4;
    for (int l = 0; l < n_levels; ++l) {
      const int b = l & 1;
      mbar_wait(mbar + b, (phase >> b) & 1u);
      phase ^= 1u << b;
      const int4* B = blk0 + b * blk_max;
      const int4 H = B[0];  // {next_start, next_n4}
      if (threadIdx.x == 0 && l + 1 < n_levels) bulk_load(blk0 + (b ^ 1) * blk_max, fblk + H.x, H.y, mbar + (b ^ 1));
      const int2 Wr = reinterpret_cast<const int2*>(B + 1)[warp];  // {first_rel, groups}
      const int4* G = B + Wr.x;
      auto issue = [&](int g, int d) {
        const int4* rec = G + g * kGroupRecs;
        const int4 h = rec[0], o0 = rec[1], o1 = rec[2];
        const int opd[8] = {o0.x, o0.y, o0.z, o0.w, o1.x, o1.y, o1.z, o1.w};
        const int kind = h.x, n = h.y;
        float4* base = my + d * kSlots * 32;
#pragma unroll
        for (int k = 0; k < kGroup; ++k) {
          if (k >= n) break;
          // a row's last forward read (header mask) and the V columns (read
          // once) leave L2 first
          if (kind >= SGX_AND2) {
            load_row(base + (2 * k) * 32, T + static_cast<size_t>(opd[2 * k] >> 1) * TILE, (h.w >> (2 * k)) & 1, pol);
            load_row(base + (2 * k + 1) * 32, T + static_cast<size_t>(opd[2 * k + 1] >> 1) * TILE,
                     (h.w >> (2 * k + 1)) & 1, pol);
          } else if (kind == SGX_NOT || kind == SGX_BUF) {
            load_row(base + (2 * k) * 32, T + static_cast<size_t>(opd[2 * k] >> 1) * TILE, (h.w >> (2 * k)) & 1, pol);
          } else if (kind == SGX_INPUT && opd[2 * k] >= 0) {
            load_row(base + (2 * k) * 32, S + static_cast<size_t>(opd[2 * k]) * TILE, 1, pol);
          }
        }
        cp_async_commit();
      };
#pragma unroll
      for (int i = 0; i < kStages - 1; ++i) {
        if (i < Wr.y)
          issue(i, i);
        else
          cp_async_commit();
      }
      for (int i = 0; i < Wr.y; ++i) {
        const int nxt = i + kStages - 1;
        if (nxt < Wr.y)
          issue(nxt, nxt % kStages);
        else
          cp_async_commit();
        cp_async_wait<kStages - 1>();
        const int4* rec = G + i * kGroupRecs;
        const int4 h = rec[0], o0 = rec[1], o1 = rec[2];
        const int opd[8] = {o0.x, o0.y, o0.z, o0.w, o1.x, o1.y, o1.z, o1.w};
        const int kind = h.x, n = h.y;
        const float4* base = my + (i % kStages) * kSlots * 32;
        float* out = T + static_cast<size_t>(h.z) * TILE;
        switch (kind) {
          case SGX_AND2: group_binary<SGX_AND2>(base, opd, n, out); break;
          case SGX_OR2: group_binary<SGX_OR2>(base, opd, n, out); break;
          case SGX_XOR2: group_binary<SGX_XOR2>(base, opd, n, out); break;
          case SGX_XNOR2: group_binary<SGX_XNOR2>(base, opd, n, out); break;
          case SGX_NOT: group_unary<true>(base, opd, n, out); break;
          case SGX_BUF: group_unary<false>(base, opd, n, out); break;
          case SGX_INPUT:
#pragma unroll
            for (int k = 0; k < kGroup; ++k) {
              if (k >= n) break;
              float a[4] = {0.0f, 0.0f, 0.0f, 0.0f}, r[4];
              if (opd[2 * k] >= 0) f4(base[(2 * k) * 32], a);
#pragma unroll
              for (int v = 0; v < 4; ++v)
                r[v] = opd[2 * k] < 0 ? 0.5f : (src_is_prob ? a[v] : sigmoid_ref(a[v], exp_tab));
              vstore<4>(out + k * TILE, r);
            }
            break;
          default: {
            const float c = kind == SGX_CONST1 ? 1.0f : 0.0f;
            const float r[4] = {c, c, c, c};
#pragma unroll
            for (int k = 0; k < kGroup; ++k) {
              if (k >= n) break;
              vstore<4>(out + k * TILE, r);
            }
          }
        }
      }
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------------------
// On-chip soft pass (small circuits): embed + forward + loss + backward + GD
// + harden for a 32-sample tile in ONE warp, with the tape [row][32] and the
// adjoint slots [slot][32] in that warp's shared memory and the program
// (copied once per persistent CTA) read as shared-memory broadcasts.  Each
// lane owns one sample and touches only its own column, so no barrier or
// fence is needed anywhere: program order of one thread orders every
// dependency.  Loads are hoisted only within a level, where records are
// independent.  Arithmetic and order are those of the HBM kernels (so the
// same bits); the only HBM traffic left is V and the harvest's input words.
// ---------------------------------------------------------------------------
constexpr int kOcMaxWarps = 8;

__device__ __forceinline__ void onchip_record(const int4 r, float g, float y, float& acc, float& acc2, const float* T,
                                              float* A, int lane) {
  const int f = r.x;
  const float4 C = kRecC[f & 0xf];
  const float ns = (f & kRNegOther) ? -1.0f : 1.0f, no = (f & kRNegOther) ? 1.0f : 0.0f;
  if (!(f & kRSlow)) {
    if (f & kRFirst) acc = 0.0f;
    acc = __fadd_rn(acc, __fmul_rn(g, __fmaf_rn(C.y, __fmaf_rn(ns, y, no), C.x)));
  } else {
    if (f & (kRFirst | kRSubFirst)) {
      float sd = 0.0f, sd2 = 0.0f;
      if (f & (kRSeed | kRSubSeed)) {  // adj[out] += 2 (y - t) on a zero adjoint (autodiff.cpp:206)
        const float yw = T[r.w * 32 + lane];
        const float t = (f & kRTarget) ? 1.0f : 0.0f, t2 = (f & kRSubTarget) ? 1.0f : 0.0f;
        if (f & kRSeed) sd = __fadd_rn(0.0f, __fmul_rn(2.0f, __fsub_rn(yw, t)));
        if (f & kRSubSeed) {
          const float ys = (f & kRNegSelf) ? __fsub_rn(1.0f, yw) : yw;
          sd2 = __fadd_rn(0.0f, __fmul_rn(2.0f, __fsub_rn(ys, t2)));
        }
      }
      if (f & kRFirst) acc = sd;
      if (f & kRSubFirst) acc2 = sd2;
    }
    if (r.y >= 0) {
      const float t = __fmul_rn(g, __fmaf_rn(C.y, __fmaf_rn(ns, y, no), C.x));
      if (f & kRInSub)
        acc2 = __fadd_rn(acc2, t);
      else
        acc = __fadd_rn(acc, t);
    }
    if (f & kRSubLast) acc = (f & kRSubNot) ? __fsub_rn(acc, acc2) : __fadd_rn(acc, acc2);
  }
  if (f & kRLast) A[(f >> kOcSlotShift) * 32 + lane] = acc;
}

__global__ void __launch_bounds__(32 * kOcMaxWarps)
k_soft_onchip(const OnchipArgs a) {
  extern __shared__ int4 osm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  for (int i = threadIdx.x; i < a.prog_n4; i += blockDim.x) osm[i] = __ldg(a.prog + i);
  __syncthreads();
  const int4* G = osm;                      // groups
  const int4* R = osm + a.off_rec;          // records
  const int4* LV = osm + a.off_lvl;         // per level / pass ranges
  const int* COL = reinterpret_cast<const int*>(osm + a.off_col);
  const int* OUT = reinterpret_cast<const int*>(osm + a.off_out);
  float* T = reinterpret_cast<float*>(osm + a.prog_n4) + static_cast<size_t>(warp) * (a.n_rows + a.n_slots) * 32;
  float* A = T + static_cast<size_t>(a.n_rows) * 32;
  for (int tile = blockIdx.x * nw + warp; tile < a.n_tiles; tile += gridDim.x * nw) {
    float* Vt = a.V + static_cast<size_t>(tile) * a.ncols * 32 + lane;
    // forward (autodiff.cpp:64-152), NOT/BUF folded into operand reads
    for (int l = 0; l < a.n_levels; ++l) {
      const int4 L = LV[l];
      for (int gi = L.x; gi < L.x + L.y; ++gi) {
        const int4* rec = G + gi * kGroupRecs;
        const int4 h = rec[0], o0 = rec[1], o1 = rec[2];
        const int opd[8] = {o0.x, o0.y, o0.z, o0.w, o1.x, o1.y, o1.z, o1.w};
        const int kind = h.x, n = h.y;
        float* out = T + h.z * 32 + lane;
        float xa[kGroup], xb[kGroup];
#pragma unroll
        for (int k = 0; k < kGroup; ++k) {
          xa[k] = xb[k] = 0.0f;
          if (k < n) {
            if (kind >= SGX_AND2) {
              xa[k] = fold_read(T[(opd[2 * k] >> 1) * 32 + lane], opd[2 * k]);
              xb[k] = fold_read(T[(opd[2 * k + 1] >> 1) * 32 + lane], opd[2 * k + 1]);
            } else if (kind == SGX_NOT || kind == SGX_BUF) {
              xa[k] = fold_read(T[(opd[2 * k] >> 1) * 32 + lane], opd[2 * k]);
            } else if (kind == SGX_INPUT && opd[2 * k] >= 0) {
              xa[k] = Vt[opd[2 * k] * 32];
            }
          }
        }
#pragma unroll
        for (int k = 0; k < kGroup; ++k) {
          if (k >= n) break;
          float r;
          if (kind == SGX_INPUT)
            r = opd[2 * k] < 0 ? 0.5f : sigmoid_ref(xa[k], a.exp_tab);
          else if (kind == SGX_CONST0 || kind == SGX_CONST1)
            r = kind == SGX_CONST1 ? 1.0f : 0.0f;
          else
            r = gate_value(kind, xa[k], xb[k]);
          out[k * 32] = r;
        }
      }
    }
    // loss (autodiff.cpp:160-166): outputs in order
    if (a.row_loss) {
      float l = 0.0f;
      for (int m = 0; m < a.n_out; ++m) {
        const int e = OUT[m];
        const float yv = fold_read(T[(e >> 1) * 32 + lane], e);
        const float t = __ldg(a.out_tgt + m) ? 1.0f : 0.0f;
        const float d = __fsub_rn(yv, t);
        l = __fadd_rn(l, __fmul_rn(d, d));
      }
      a.row_loss[static_cast<size_t>(tile) * 32 + lane] = l;
    }
    // backward (autodiff.cpp:172-283), pull records in the reference's order
    float acc = 0.0f, acc2 = 0.0f;
    for (int li = 0; li < a.n_levels; ++li) {
      const int4 L = LV[li];
      for (int k0 = L.z; k0 < L.z + L.w; k0 += 4) {
        int4 r[4];
        float g[4], y[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          r[k] = k0 + k < L.z + L.w ? R[k0 + k] : make_int4(0, -1, -1, 0);
          g[k] = r[k].y >= 0 ? A[r[k].y * 32 + lane] : 0.0f;
          y[k] = r[k].z >= 0 ? T[r[k].z * 32 + lane] : 0.0f;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (k0 + k < L.z + L.w) onchip_record(r[k], g[k], y[k], acc, acc2, T, A, lane);
      }
    }
    // V columns: dV = g p (1 - p) (autodiff.cpp:212-221), V -= lr dV
    // (gd_step, :285-290), harden (:292-297) into the harvest's words
    for (int j = 0; j < a.ncols; ++j) {
      const int sl = COL[j];
      if (sl < 0) continue;  // warp-uniform
      const float x = Vt[j * 32], gg = A[sl * 32 + lane];
      const float p = sigmoid_ref(x, a.exp_tab);
      const float dv = __fmul_rn(__fmul_rn(gg, p), __fsub_rn(1.0f, p));
      const float nv = __fsub_rn(x, __fmul_rn(a.lr, dv));
      Vt[j * 32] = nv;
      const uint32_t b = __ballot_sync(kFull, nv >= 0.0f);
      if (lane == 0) a.hb[static_cast<size_t>(tile) * a.ncols + j] = b;
    }
  }
}

int onchip_warps(int n_rows, int n_slots, int prog_n4) {
  const size_t per_warp = static_cast<size_t>(n_rows + n_slots) * 32 * sizeof(float);
  const size_t prog = static_cast<size_t>(prog_n4) * 16;
  const size_t budget = 200 * 1024;
  if (prog + 2 * per_warp > budget) return 0;  // at least two warps per SM
  return static_cast<int>(std::min<size_t>(kOcMaxWarps, (budget - prog) / per_warp));
}

bool launch_soft_onchip(cudaStream_t st, const OnchipArgs& a) {
  const int nw = onchip_warps(a.n_rows, a.n_slots, a.prog_n4);
  if (nw == 0) return false;
  const size_t smem = static_cast<size_t>(a.prog_n4) * 16 +
                      static_cast<size_t>(nw) * (a.n_rows + a.n_slots) * 32 * sizeof(float);
  opt_in_smem(reinterpret_cast<const void*>(k_soft_onchip), smem);
  int ctas = (a.n_tiles + nw - 1) / nw;
  if (ctas > 148) ctas = 148;  // persistent: one CTA per SM (the program is copied once)
  k_soft_onchip<<<ctas, 32 * nw, smem, st>>>(a);
  return true;
}

// Opt-in Adam update (sgx_optimizer SGX_OPT_ADAM; no reference counterpart,
// SPEC.md:418): the backward stored dV (same tile-major layout as V); per
// logit m, v moments, bias-corrected step, then the harvest's hardened words
// of the new V (harden, autodiff.cpp:292-297).  One thread per logit, in
// layout order, so a warp's 32 logits are 32 consecutive samples of one
// column of one tile (tile_rows >= 32).
__global__ void __launch_bounds__(kThreads)
k_adam(float* __restrict__ Vp, const float* __restrict__ dV, float* __restrict__ m, float* __restrict__ v, int ncols,
       int Bp, int tile_rows, float lr, float b1, float b2, float c1, float c2, float eps, uint32_t* __restrict__ hb) {
  const long long n = static_cast<long long>(ncols) * Bp;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const float g = dV[i];
    const float mi = b1 * m[i] + (1.0f - b1) * g;
    const float vi = b2 * v[i] + (1.0f - b2) * g * g;
    m[i] = mi;
    v[i] = vi;
    const float nv = Vp[i] - lr * (mi / c1) / (sqrtf(vi / c2) + eps);
    Vp[i] = nv;
    const uint32_t word = __ballot_sync(kFull, nv >= 0.0f);
    if ((threadIdx.x & 31) == 0) {
      const long long per_tile = static_cast<long long>(ncols) * tile_rows;
      const long long tile = i / per_tile, rem = i - tile * per_tile;
      const int col = static_cast<int>(rem / tile_rows), pos = static_cast<int>(rem - static_cast<long long>(col) * tile_rows);
      hb[static_cast<size_t>((tile * tile_rows + pos) >> 5) * ncols + col] = word;
    }
  }
}

static int grid_for(long long n, int per_block, int cap);

void launch_adam(cudaStream_t st, float* V, const float* dV, float* m, float* v, int ncols, int Bp, int tile_rows,
                 float lr, float b1, float b2, int t, float eps, uint32_t* hb) {
  const long long n = static_cast<long long>(ncols) * Bp;
  if (n == 0) return;
  const float c1 = 1.0f - powf(b1, static_cast<float>(t)), c2 = 1.0f - powf(b2, static_cast<float>(t));
  k_adam<<<grid_for(n, kThreads, 148 * 16), kThreads, 0, st>>>(V, dV, m, v, ncols, Bp, tile_rows, lr, b1, b2, c1, c2,
                                                              eps, hb);
}

// Deterministic loss total: fixed per-block partial sums in double, then one
// block folds the partials in block order.
__global__ void __launch_bounds__(kThreads)
k_loss_partial(const float* __restrict__ row_loss, int batch, double* __restrict__ partial) {
  __shared__ double sh[kThreads];
  double acc = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < batch; i += gridDim.x * blockDim.x)
    acc += static_cast<double>(row_loss[i]);
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = sh[0];
}

__global__ void k_loss_final(const double* __restrict__ partial, int n, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < n; ++i) t += partial[i];
    *out = t;
  }
}

// ---------------------------------------------------------------------------
// K5a: harden + free bits.  One warp per (input, 32-row word): lane = row.
// Constrained column c: ballot(V >= 0) (ties -> 1, NaN -> 0).  Free input k:
// ballot(hash{seed, 'free', restart, iter, row, k} & 1).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads)
k_harden(const float* __restrict__ V, int ncpi, int nucpi, const int* __restrict__ cpi_row,
         const int* __restrict__ ucpi_row, uint32_t* __restrict__ BT, int W, int tile_rows,
         uint64_t free_prefix, long long row_offset) {
  const int lane = threadIdx.x & 31;
  const long long total = static_cast<long long>(ncpi + nucpi) * W;
  for (long long gw = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5; gw < total;
       gw += (static_cast<long long>(gridDim.x) * blockDim.x) >> 5) {
    const int input = static_cast<int>(gw / W);
    const int w = static_cast<int>(gw - static_cast<long long>(input) * W);
    const int r = w * 32 + lane;
    bool bit;
    int row;
    if (input < ncpi) {
      const size_t tile = static_cast<size_t>(r / tile_rows);
      bit = V[(tile * ncpi + input) * tile_rows + r % tile_rows] >= 0.0f;
      row = __ldg(cpi_row + input);
    } else {
      const int k = input - ncpi;
      bit = fold(fold(free_prefix, static_cast<uint64_t>(row_offset + r)), static_cast<uint64_t>(k)) & 1;
      row = __ldg(ucpi_row + k);
    }
    const uint32_t word = __ballot_sync(kFull, bit);
    if (lane == 0) BT[static_cast<size_t>(row) * W + w] = word;
  }
}

__device__ __forceinline__ uint32_t bit_gate(int kind, uint32_t a, uint32_t b) {
  switch (kind) {  // circuit.cpp:137-144 on 32 rows at once
    case SGX_CONST0: return 0u;
    case SGX_CONST1: return kFull;
    case SGX_BUF: return a;
    case SGX_NOT: return ~a;
    case SGX_AND2: return a & b;
    case SGX_OR2: return a | b;
    case SGX_XOR2: return a ^ b;
    case SGX_XNOR2: return ~(a ^ b);
    default: return 0u;
  }
}

// ---------------------------------------------------------------------------
// K5b+K6: bit-sliced eval of every node, then PO check and CNF check.  A CTA
// owns WPC consecutive words (32*WPC rows); its threads are (slot, word)
// pairs, slots split each level's nodes, __syncthreads between levels.
// Output valid[w]: bit r set iff row 32w+r hits every output target and
// satisfies every clause.
// ---------------------------------------------------------------------------
template <int WPC>
__global__ void __launch_bounds__(kThreads)
k_bit_eval(const int4* __restrict__ ops, const int* __restrict__ lvl_ptr, int n_levels,
           uint32_t* BT, int W, const int* __restrict__ out_row, const uint8_t* __restrict__ out_tgt,
           int n_out, const int* __restrict__ clause_ptr, const int* __restrict__ clause_enc,
           int n_clauses, uint32_t* __restrict__ valid, int batch) {
  constexpr int S = kThreads / WPC;
  const int lw = threadIdx.x % WPC, slot = threadIdx.x / WPC;
  const int w = blockIdx.x * WPC + lw;
  const size_t Wz = static_cast<size_t>(W);
  for (int l = 0; l < n_levels; ++l) {
    const int e = __ldg(lvl_ptr + l + 1);
    for (int i = __ldg(lvl_ptr + l) + slot; i < e; i += 4 * S) {
      int4 op[4];
      uint32_t xa[4], xb[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int ii = i + u * S;
        op[u] = ii < e ? __ldg(ops + ii) : make_int4(SGX_CONST0, -1, 0, 0);
        xa[u] = op[u].y >= 0 ? BT[op[u].z * Wz + w] : 0u;
        xb[u] = op[u].y >= 0 ? BT[op[u].w * Wz + w] : 0u;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (op[u].y >= 0) BT[op[u].y * Wz + w] = bit_gate(op[u].x, xa[u], xb[u]);
    }
    __syncthreads();
  }
  uint32_t ok = kFull;
  for (int m = slot; m < n_out; m += S) {  // sampler.cpp:140-146
    const uint32_t x = BT[static_cast<size_t>(__ldg(out_row + m)) * Wz + w];
    ok &= __ldg(out_tgt + m) ? x : ~x;
  }
  // eval_cnf (cnf.cpp:136-145): this slot's contiguous clause range, as a
  // flat literal stream so the loads pipeline.
  const int c0 = static_cast<int>(static_cast<long long>(n_clauses) * slot / S);
  const int c1 = static_cast<int>(static_cast<long long>(n_clauses) * (slot + 1) / S);
  const int l1 = __ldg(clause_ptr + c1);
  uint32_t any = 0u;
#pragma unroll 8
  for (int l = __ldg(clause_ptr + c0); l < l1; ++l) {
    const int e = __ldg(clause_enc + l);
    const uint32_t x = BT[static_cast<size_t>(e >> 2) * Wz + w];
    any |= (e & 1) ? ~x : x;
    if (e & 2) {
      ok &= any;
      any = 0u;
    }
  }
  __shared__ uint32_t red[kThreads];
  red[threadIdx.x] = ok;
  __syncthreads();
  if (slot == 0) {
#pragma unroll
    for (int j = 1; j < S; ++j) ok &= red[j * WPC + lw];
    const int r0 = w * 32;
    uint32_t mask = r0 + 32 <= batch ? kFull : (r0 >= batch ? 0u : ((1u << (batch - r0)) - 1u));
    valid[w] = ok & mask;
  }
}

// 32x32 bit transpose across a warp: lane i holds row i on entry, column i on
// exit (bit k of lane i <-> bit i of lane k).
__device__ __forceinline__ uint32_t transpose32(uint32_t x, int lane) {
  const uint32_t masks[5] = {0x0000ffffu, 0x00ff00ffu, 0x0f0f0f0fu, 0x33333333u, 0x55555555u};
#pragma unroll
  for (int t = 0; t < 5; ++t) {
    const int j = 16 >> t;
    const uint32_t m = masks[t];
    const uint32_t o = __shfl_xor_sync(kFull, x, j);
    x = (lane & j) ? ((x & ~m) | ((o >> j) & m)) : ((x & m) | ((o & m) << j));
  }
  return x;
}

// ---------------------------------------------------------------------------
// K7: dedupe keys + fingerprints + table insert.  A warp owns 8 consecutive
// words (256 rows).  For each group of 32 variables, lane k loads the 8 words
// of variable 32g+k (one 32-byte sector) and 8 warp transposes turn them into
// per-row variable bits.  Key word q packs vars 64q+1..64q+64 LSB first
// (dedupe_key, sampler.cpp:18-26).  Valid rows: K[q][row] = key word,
// fp = splitmix chain over the key words, then the first-row-wins insert:
// meta = min over rows of (epoch << 32 | row) for fingerprints first seen in
// this epoch; older fingerprints keep a smaller meta, so they never win.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads)
k_keys(const uint32_t* __restrict__ BT, int W, const int* __restrict__ key_row, int key_words,
       const uint32_t* __restrict__ valid, int Bp, uint64_t* __restrict__ K, int* __restrict__ slot_of_row,
       unsigned long long* tkeys, unsigned long long* tmeta, uint64_t tmask, uint64_t epoch) {
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int w0 = warp * 8;
  if (w0 >= W) return;
  uint32_t vm[8];
  uint32_t anyv = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    vm[j] = __ldg(valid + w0 + j);
    anyv |= vm[j];
  }
  if (anyv == 0) return;  // warp-uniform
  uint64_t h[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) h[j] = 0ull;
  const size_t Wz = static_cast<size_t>(W);
  for (int q = 0; q < key_words; ++q) {
    uint32_t half[2][8];
#pragma unroll
    for (int hf = 0; hf < 2; ++hf) {
      const int row = __ldg(key_row + (2 * q + hf) * 32 + lane);
      uint4 A = make_uint4(0, 0, 0, 0), Bv = make_uint4(0, 0, 0, 0);
      if (row >= 0) {
        const uint4* p = reinterpret_cast<const uint4*>(BT + row * Wz + w0);
        A = __ldg(p);
        Bv = __ldg(p + 1);
      }
      uint32_t x[8] = {A.x, A.y, A.z, A.w, Bv.x, Bv.y, Bv.z, Bv.w};
#pragma unroll
      for (int j = 0; j < 8; ++j) half[hf][j] = transpose32(x[j], lane);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint64_t kw = static_cast<uint64_t>(half[0][j]) | (static_cast<uint64_t>(half[1][j]) << 32);
      h[j] += key_term(kw, q);
      if ((vm[j] >> lane) & 1u) K[static_cast<size_t>(q) * Bp + (w0 + j) * 32 + lane] = kw;
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    if (!((vm[j] >> lane) & 1u)) continue;
    const int r = (w0 + j) * 32 + lane;
    const uint64_t hf = mix64(h[j]);
    const unsigned long long fp = hf ? hf : 1ull;  // 0 marks an empty slot
    uint64_t idx = (fp ^ (fp >> 29)) & tmask;
    for (;;) {
      unsigned long long cur = tkeys[idx];
      if (cur == fp) break;
      if (cur == 0ull) {
        cur = atomicCAS(tkeys + idx, 0ull, fp);
        if (cur == 0ull || cur == fp) break;
      }
      idx = (idx + 1) & tmask;
    }
    atomicMin(tmeta + idx, static_cast<unsigned long long>((epoch << 32) | static_cast<uint32_t>(r)));
    slot_of_row[r] = static_cast<int>(idx);
  }
}

// ---------------------------------------------------------------------------
// K5+K6+K7 fused, shared-memory resident: one CTA owns WPC words (32*WPC
// rows) and keeps its whole folded bit tape [row][WPC] in shared memory, so
// harden -> every level of eval_discrete -> PO + CNF check -> dedupe keys +
// fingerprint + table insert run without touching HBM except for V, the
// key words of valid rows and the table.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t neg_mask(int enc) { return (enc & 1) ? kFull : 0u; }

template <int WPC>
__global__ void __launch_bounds__(kThreads)
k_harvest_smem(int n_rows, const uint32_t* __restrict__ hb, int ncpi, int nucpi, const int* __restrict__ cpi_row,
               const int* __restrict__ ucpi_row, uint64_t free_prefix, long long row_offset,
               const int4* __restrict__ ops, const int* __restrict__ lvl_ptr, int n_levels,
               const int* __restrict__ out_enc, const uint8_t* __restrict__ out_tgt, int n_out,
               const int4* __restrict__ cnf4, int cnf_steps,
               const int* __restrict__ key_enc, int key_words, int batch, int Bp,
               uint32_t* __restrict__ valid_out, uint64_t* __restrict__ K, int* __restrict__ slot_of_row,
               unsigned long long* tkeys, unsigned long long* tmeta, uint64_t tmask, uint64_t epoch) {
  extern __shared__ uint32_t bits[];  // [row][WPC], row n_rows = 0 (CNF padding)
  __shared__ uint32_t red[kThreads];
  __shared__ uint32_t vw[WPC];
  constexpr int NW = kThreads / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int w0 = blockIdx.x * WPC;
  if (threadIdx.x < WPC) bits[n_rows * WPC + threadIdx.x] = 0u;
  // hardened inputs (autodiff.cpp:292-297), produced by k_init_v / the
  // backward epilogue as hb[word][col]: consecutive threads, consecutive
  // columns of one word
  for (int item = threadIdx.x; item < ncpi * WPC; item += kThreads) {
    const int wl = item / ncpi, input = item - wl * ncpi;
    bits[__ldg(cpi_row + input) * WPC + wl] = __ldg(hb + static_cast<size_t>(w0 + wl) * ncpi + input);
  }
  // free bits (sampler.cpp:132-137)
  for (int item = warp; item < nucpi * WPC; item += NW) {
    const int k = item / WPC, wl = item - k * WPC;
    const int r = (w0 + wl) * 32 + lane;
    const bool bit = fold(fold(free_prefix, static_cast<uint64_t>(row_offset + r)), static_cast<uint64_t>(k)) & 1;
    const uint32_t word = __ballot_sync(kFull, bit);
    if (lane == 0) bits[__ldg(ucpi_row + k) * WPC + wl] = word;
  }
  __syncthreads();
  // eval_discrete (circuit.cpp:126-146), level by level.  The op record of a
  // thread's first item of level l+1 is fetched before level l's barrier, so
  // the L2 round trip overlaps the level instead of following it.
  {
    int b = __ldg(lvl_ptr), e = n_levels > 0 ? __ldg(lvl_ptr + 1) : b;
    int4 nxt = threadIdx.x < (e - b) * WPC ? __ldg(ops + b + threadIdx.x / WPC) : make_int4(0, 0, 0, 0);
    for (int l = 0; l < n_levels; ++l) {
      const int4 cur = nxt;
      const int nb = e, ne = l + 2 <= n_levels ? __ldg(lvl_ptr + l + 2) : e;
      if (threadIdx.x < (ne - nb) * WPC) nxt = __ldg(ops + nb + threadIdx.x / WPC);
      for (int item = threadIdx.x; item < (e - b) * WPC; item += kThreads) {
        const int wl = item % WPC;
        const int4 op = item == static_cast<int>(threadIdx.x) ? cur : __ldg(ops + b + item / WPC);
        const uint32_t a = bits[(op.z >> 1) * WPC + wl] ^ neg_mask(op.z);
        const uint32_t c = bits[(op.w >> 1) * WPC + wl] ^ neg_mask(op.w);
        bits[op.y * WPC + wl] = bit_gate(op.x, a, c);
      }
      b = nb;
      e = ne;
      __syncthreads();
    }
  }
  // PO check (sampler.cpp:140-146) + eval_cnf (cnf.cpp:136-145).  Each
  // thread owns whole clauses as int4 literal records stored transposed, so a
  // step's reads are coalesced; every record serves all WPC words.
  {
    uint32_t ok[WPC], any[WPC];
#pragma unroll
    for (int wl = 0; wl < WPC; ++wl) {
      ok[wl] = kFull;
      any[wl] = 0u;
    }
    for (int m = threadIdx.x; m < n_out; m += kThreads) {
      const int e = __ldg(out_enc + m);
      const uint32_t t = __ldg(out_tgt + m) ? 0u : kFull;
#pragma unroll
      for (int wl = 0; wl < WPC; ++wl) ok[wl] &= bits[(e >> 1) * WPC + wl] ^ neg_mask(e) ^ t;
    }
    // Branch-free: a literal is row or ~row (negated), s = e >> 31 recovers
    // both the row (e ^ s) and the word mask (x ^ s); padding reads the zero
    // row; a record closes its clause unless .w is kCnfOpen.
    int4 nrec = cnf_steps > 0 ? __ldg(cnf4 + threadIdx.x) : make_int4(0, 0, 0, kCnfOpen);
    for (int j = 0; j < cnf_steps; ++j) {
      const int4 rec = nrec;  // next step's record is in flight while this one runs
      if (j + 1 < cnf_steps) nrec = __ldg(cnf4 + static_cast<size_t>(j + 1) * kThreads + threadIdx.x);
      const bool open = rec.w == kCnfOpen;
      const uint32_t keep = open ? kFull : 0u;
      const int lit[4] = {rec.x, rec.y, rec.z, open ? n_rows : rec.w};
#pragma unroll
      for (int wl = 0; wl < WPC; ++wl) {
        uint32_t a = 0u;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int sgn = lit[u] >> 31;
          a |= bits[(lit[u] ^ sgn) * WPC + wl] ^ static_cast<uint32_t>(sgn);
        }
        any[wl] |= a;
        ok[wl] &= any[wl] | keep;
        any[wl] &= keep;
      }
    }
#pragma unroll
    for (int wl = 0; wl < WPC; ++wl) {
      const uint32_t v = __reduce_and_sync(kFull, ok[wl]);
      if (lane == 0) red[warp * WPC + wl] = v;
    }
    __syncthreads();
    if (threadIdx.x < WPC) {
      const int wl = threadIdx.x;
      uint32_t v = kFull;
#pragma unroll
      for (int j = 0; j < NW; ++j) v &= red[j * WPC + wl];
      const int r0 = (w0 + wl) * 32;
      const uint32_t mask = r0 + 32 <= batch ? kFull : (r0 >= batch ? 0u : ((1u << (batch - r0)) - 1u));
      vw[wl] = v & mask;
      valid_out[w0 + wl] = v & mask;
    }
    __syncthreads();
  }
  // dedupe keys (sampler.cpp:18-26) by warp transposes; all warps share the
  // (word, key word) items and fold their fingerprint terms with shared atomics
  __shared__ unsigned long long hsum[WPC * 32];
  for (int t = threadIdx.x; t < WPC * 32; t += kThreads) hsum[t] = 0ull;
  __syncthreads();
  for (int item = warp; item < WPC * key_words; item += NW) {
    const int q = item / WPC, wl = item - q * WPC;
    const uint32_t vm = vw[wl];
    if (vm == 0) continue;  // warp-uniform
    uint32_t half[2];
#pragma unroll
    for (int hf = 0; hf < 2; ++hf) {
      const int e = __ldg(key_enc + (2 * q + hf) * 32 + lane);
      const uint32_t x = e >= 0 ? (bits[(e >> 1) * WPC + wl] ^ neg_mask(e)) : 0u;
      half[hf] = transpose32(x, lane);
    }
    const uint64_t kw = static_cast<uint64_t>(half[0]) | (static_cast<uint64_t>(half[1]) << 32);
    atomicAdd(hsum + wl * 32 + lane, static_cast<unsigned long long>(key_term(kw, q)));
    if ((vm >> lane) & 1u) K[static_cast<size_t>(q) * Bp + (w0 + wl) * 32 + lane] = kw;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < WPC * 32; t += kThreads) {
    const int wl = t >> 5, ln = t & 31;
    if (!((vw[wl] >> ln) & 1u)) continue;
    const int r = (w0 + wl) * 32 + ln;
    const uint64_t h = mix64(hsum[t]);
    const unsigned long long fp = h ? h : 1ull;
    uint64_t idx = (fp ^ (fp >> 29)) & tmask;
    for (;;) {
      unsigned long long cur = tkeys[idx];
      if (cur == fp) break;
      if (cur == 0ull) {
        cur = atomicCAS(tkeys + idx, 0ull, fp);
        if (cur == 0ull || cur == fp) break;
      }
      idx = (idx + 1) & tmask;
    }
    atomicMin(tmeta + idx, static_cast<unsigned long long>((epoch << 32) | static_cast<uint32_t>(r)));
    slot_of_row[r] = static_cast<int>(idx);
  }
}

// ---------------------------------------------------------------------------
// K5+K6+K7 fused with a liveness-allocated bit tape: a CTA owns WPC words
// (32*WPC rows); its shared memory holds only the LIVE rows of the folded
// bit program, in host-assigned slots (sgx_layout.cpp build_live_bits), so
// deep and wide circuits (C4: 8,072 slots instead of 54,234 rows) stay on chip
// and shallow ones fit several CTAs per SM.  Per phase: that level's gate ops
// (eval_discrete, circuit.cpp:126-146), then the output checks and CNF
// clauses whose latest literal was defined one phase earlier (sampler.cpp:
// 140-147, cnf.cpp:136-145); one barrier.  Rows of CNF variables are also
// written to a global spill tape, which the key phase (dedupe_key,
// sampler.cpp:18-26) reads back after the last phase.
// ---------------------------------------------------------------------------
template <int WPC>
__device__ __forceinline__ void load_words(const uint32_t* p, uint32_t (&x)[WPC]) {
  if constexpr (WPC == 4) {
    const uint4 t = *reinterpret_cast<const uint4*>(p);
    x[0] = t.x; x[1] = t.y; x[2] = t.z; x[3] = t.w;
  } else if constexpr (WPC == 8) {
    const uint4 t = reinterpret_cast<const uint4*>(p)[0], u = reinterpret_cast<const uint4*>(p)[1];
    x[0] = t.x; x[1] = t.y; x[2] = t.z; x[3] = t.w; x[4] = u.x; x[5] = u.y; x[6] = u.z; x[7] = u.w;
  } else if constexpr (WPC == 2) {
    const uint2 t = *reinterpret_cast<const uint2*>(p);
    x[0] = t.x; x[1] = t.y;
  } else {
    x[0] = *p;
  }
}

// WPC consecutive words of one shared-memory slot as one vector access.
template <int WPC>
__device__ __forceinline__ void lds_words(const uint32_t* p, uint32_t (&x)[WPC]) {
  load_words<WPC>(p, x);
}
template <int WPC>
__device__ __forceinline__ void sts_words(uint32_t* p, const uint32_t (&x)[WPC]) {
  if constexpr (WPC == 4) {
    *reinterpret_cast<uint4*>(p) = make_uint4(x[0], x[1], x[2], x[3]);
  } else if constexpr (WPC == 8) {
    reinterpret_cast<uint4*>(p)[0] = make_uint4(x[0], x[1], x[2], x[3]);
    reinterpret_cast<uint4*>(p)[1] = make_uint4(x[4], x[5], x[6], x[7]);
  } else if constexpr (WPC == 2) {
    *reinterpret_cast<uint2*>(p) = make_uint2(x[0], x[1]);
  } else {
    *p = x[0];
  }
}

template <int WPC>
__global__ void __launch_bounds__(kThreads)
k_harvest_live(const HarvestLiveArgs a) {
  extern __shared__ uint32_t bits[];  // [slot][WPC]; slot 0 = 0
  __shared__ uint32_t red[kThreads];
  __shared__ uint32_t vw[WPC];
  __shared__ unsigned long long hsum[WPC * 32];
  constexpr int NW = kThreads / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int w0 = blockIdx.x * WPC;
  const size_t Wz = static_cast<size_t>(a.W);
  if (threadIdx.x < WPC) bits[threadIdx.x] = 0u;
  for (int t = threadIdx.x; t < WPC * 32; t += kThreads) hsum[t] = 0ull;
  // phase 0 inputs: hardened V (autodiff.cpp:292-297) and free bits (sampler.cpp:132-137)
  for (int item = threadIdx.x; item < a.ncpi * WPC; item += kThreads) {
    const int wl = item / a.ncpi, j = item - wl * a.ncpi;
    const int2 cs = __ldg(a.cpi + j);
    const uint32_t word = __ldg(a.hb + static_cast<size_t>(w0 + wl) * a.ncpi + j);
    bits[cs.x * WPC + wl] = word;
    if (cs.y >= 0) a.spill[cs.y * Wz + w0 + wl] = word;
  }
  for (int item = warp; item < a.nucpi * WPC; item += NW) {
    const int k = item / WPC, wl = item - k * WPC;
    const int r = (w0 + wl) * 32 + lane;
    const bool bit = fold(fold(a.free_prefix, static_cast<uint64_t>(a.row_offset + r)), static_cast<uint64_t>(k)) & 1;
    const uint32_t word = __ballot_sync(kFull, bit);
    if (lane == 0) {
      const int2 cs = __ldg(a.ucpi + k);
      bits[cs.x * WPC + wl] = word;
      if (cs.y >= 0) a.spill[cs.y * Wz + w0 + wl] = word;
    }
  }
  __syncthreads();
  uint32_t ok[WPC];
#pragma unroll
  for (int wl = 0; wl < WPC; ++wl) ok[wl] = kFull;
  // Each thread's first op and first check of the next phase are loaded
  // before this phase's barrier (and the phase bounds one phase further
  // ahead), so a phase starts on records already in registers instead of an
  // L2 round trip (C4: 635 phases).
  int ob = __ldg(a.op_ptr), oe = __ldg(a.op_ptr + 1), cb = __ldg(a.chk_ptr), ce = __ldg(a.chk_ptr + 1);
  // Narrow CTAs (WPC <= 2) spread a phase's ops over (op, word) items for
  // more threads per phase; wider ones process an op's WPC words as vectors.
  constexpr int OW = WPC <= 2 ? WPC : 1;  // items per op
  int4 nop = threadIdx.x < (oe - ob) * OW ? __ldg(a.ops + ob + threadIdx.x / OW) : make_int4(0, 0, 0, -1);
  int4 nchk = threadIdx.x < ce - cb ? __ldg(a.chk + cb + threadIdx.x) : make_int4(0, 0, 0, 0);
  int oe2 = a.n_phases > 1 ? __ldg(a.op_ptr + 2) : oe, ce2 = a.n_phases > 1 ? __ldg(a.chk_ptr + 2) : ce;
  for (int ph = 0; ph < a.n_phases; ++ph) {
    const int4 cop = nop, cchk = nchk;
    const int nob = oe, noe = oe2, ncb = ce, nce = ce2;  // phase ph + 1
    if (ph + 1 < a.n_phases) {
      nop = threadIdx.x < (noe - nob) * OW ? __ldg(a.ops + nob + threadIdx.x / OW) : make_int4(0, 0, 0, -1);
      nchk = threadIdx.x < nce - ncb ? __ldg(a.chk + ncb + threadIdx.x) : make_int4(0, 0, 0, 0);
      oe2 = ph + 3 <= a.n_phases ? __ldg(a.op_ptr + ph + 3) : noe;
      ce2 = ph + 3 <= a.n_phases ? __ldg(a.chk_ptr + ph + 3) : nce;
    }
    if constexpr (OW > 1) {
      for (int item = threadIdx.x; item < (oe - ob) * OW; item += kThreads) {  // (op, word)
        const int wl = item % OW;
        const int4 op = item == static_cast<int>(threadIdx.x) ? cop : __ldg(a.ops + ob + item / OW);
        const uint32_t x = bits[(op.y >> 1) * WPC + wl] ^ neg_mask(op.y);
        const uint32_t y = bits[(op.z >> 1) * WPC + wl] ^ neg_mask(op.z);
        const uint32_t v = bit_gate(op.x & 0xf, x, y);
        bits[(op.x >> 4) * WPC + wl] = v;
        if (op.w >= 0) a.spill[op.w * Wz + w0 + wl] = v;
      }
    } else {
      for (int item = threadIdx.x; item < oe - ob; item += kThreads) {  // one op, all WPC words
        const int4 op = item == static_cast<int>(threadIdx.x) ? cop : __ldg(a.ops + ob + item);
        uint32_t x[WPC], y[WPC], v[WPC];
        lds_words<WPC>(bits + (op.y >> 1) * WPC, x);
        lds_words<WPC>(bits + (op.z >> 1) * WPC, y);
        const uint32_t mx = neg_mask(op.y), my = neg_mask(op.z);
#pragma unroll
        for (int wl = 0; wl < WPC; ++wl) v[wl] = bit_gate(op.x & 0xf, x[wl] ^ mx, y[wl] ^ my);
        sts_words<WPC>(bits + (op.x >> 4) * WPC, v);
        if (op.w >= 0) sts_words<WPC>(a.spill + op.w * Wz + w0, v);
      }
    }
    for (int i = cb + threadIdx.x; i < ce; i += kThreads) {
      const int4 rec = i == cb + static_cast<int>(threadIdx.x) ? cchk : __ldg(a.chk + i);
      if (rec.w == kLbBig) {  // a long clause, literal by literal
        uint32_t any[WPC];
#pragma unroll
        for (int wl = 0; wl < WPC; ++wl) any[wl] = 0u;
        for (int l = rec.x; l < rec.x + rec.y; ++l) {
          const int lit = __ldg(a.big_lits + l), sgn = lit >> 31;
#pragma unroll
          for (int wl = 0; wl < WPC; ++wl) any[wl] |= bits[(lit ^ sgn) * WPC + wl] ^ static_cast<uint32_t>(sgn);
        }
#pragma unroll
        for (int wl = 0; wl < WPC; ++wl) ok[wl] &= any[wl];
      } else {
        const int lit[4] = {rec.x, rec.y, rec.z, rec.w};
        uint32_t any[WPC];
#pragma unroll
        for (int wl = 0; wl < WPC; ++wl) any[wl] = 0u;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int sgn = lit[u] >> 31;
          uint32_t x[WPC];
          lds_words<WPC>(bits + (lit[u] ^ sgn) * WPC, x);
#pragma unroll
          for (int wl = 0; wl < WPC; ++wl) any[wl] |= x[wl] ^ static_cast<uint32_t>(sgn);
        }
#pragma unroll
        for (int wl = 0; wl < WPC; ++wl) ok[wl] &= any[wl];
      }
    }
    ob = nob;
    oe = noe;
    cb = ncb;
    ce = nce;
    __syncthreads();
  }
#pragma unroll
  for (int wl = 0; wl < WPC; ++wl) {
    const uint32_t v = __reduce_and_sync(kFull, ok[wl]);
    if (lane == 0) red[warp * WPC + wl] = v;
  }
  __syncthreads();
  if (threadIdx.x < WPC) {
    const int wl = threadIdx.x;
    uint32_t v = kFull;
#pragma unroll
    for (int j = 0; j < NW; ++j) v &= red[j * WPC + wl];
    const int r0 = (w0 + wl) * 32;
    const uint32_t mask = r0 + 32 <= a.batch ? kFull : (r0 >= a.batch ? 0u : ((1u << (a.batch - r0)) - 1u));
    vw[wl] = v & mask;
    a.valid[w0 + wl] = v & mask;
  }
  __syncthreads();
  // dedupe keys (sampler.cpp:18-26) from the spill tape: one warp per key
  // word, all WPC words of a variable row in one vector load
  uint32_t anyv = 0u;
#pragma unroll
  for (int wl = 0; wl < WPC; ++wl) anyv |= vw[wl];
  if (anyv) {
    for (int q = warp; q < a.key_words; q += NW) {
      uint32_t half[2][WPC];
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        const int e = __ldg(a.key_enc + (2 * q + hf) * 32 + lane);
        uint32_t x[WPC];
        if (e >= 0) {
          load_words<WPC>(a.spill + (e >> 1) * Wz + w0, x);
#pragma unroll
          for (int wl = 0; wl < WPC; ++wl) x[wl] ^= neg_mask(e);
        } else {
#pragma unroll
          for (int wl = 0; wl < WPC; ++wl) x[wl] = 0u;
        }
#pragma unroll
        for (int wl = 0; wl < WPC; ++wl) half[hf][wl] = transpose32(x[wl], lane);
      }
#pragma unroll
      for (int wl = 0; wl < WPC; ++wl) {
        if (!vw[wl]) continue;  // block-uniform
        const uint64_t kw = static_cast<uint64_t>(half[0][wl]) | (static_cast<uint64_t>(half[1][wl]) << 32);
        atomicAdd(hsum + wl * 32 + lane, static_cast<unsigned long long>(key_term(kw, q)));
        if ((vw[wl] >> lane) & 1u) a.K[static_cast<size_t>(q) * a.Bp + (w0 + wl) * 32 + lane] = kw;
      }
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < WPC * 32; t += kThreads) {
    const int wl = t >> 5, ln = t & 31;
    if (!((vw[wl] >> ln) & 1u)) continue;
    const int r = (w0 + wl) * 32 + ln;
    const uint64_t h = mix64(hsum[t]);
    const unsigned long long fp = h ? h : 1ull;
    uint64_t idx = (fp ^ (fp >> 29)) & a.tmask;
    for (;;) {
      unsigned long long cur = a.tkeys[idx];
      if (cur == fp) break;
      if (cur == 0ull) {
        cur = atomicCAS(a.tkeys + idx, 0ull, fp);
        if (cur == 0ull || cur == fp) break;
      }
      idx = (idx + 1) & a.tmask;
    }
    atomicMin(a.tmeta + idx, static_cast<unsigned long long>((a.epoch << 32) | static_cast<uint32_t>(r)));
    a.slot_of_row[r] = static_cast<int>(idx);
  }
}

// ---------------------------------------------------------------------------
// Warp-synchronous live harvest (default for deep circuits): ONE WARP owns one
// 32-row word and walks the whole folded bit program alone, so a phase ends
// with __syncwarp instead of a CTA barrier and no warp idles through another
// warp's phase.  The program is the live program above (same slots, spill
// rows and checks) re-cut into 32-record iterations (sgx_layout.cpp lw_ops):
// lane l runs record l of each iteration; the last iteration of a phase
// carries kLwEnd (and kLwChk when the phase has checks).  Every warp of a CTA
// reads the same record stream, so it is staged once per CTA: a ring of
// kLwBuf chunks of kLwChunk iterations, each brought in by one cp.async.bulk
// (TMA) completing on its `full` mbarrier; warps release a chunk on its
// `empty` mbarrier and warp 0 refills it once all have.  Gates are evaluated
// branch-free from their ANF (mixed kinds in a warp do not diverge).  Keys,
// fingerprints and the table insert follow in k_keys_spill, which reads the
// spill tape in whole sectors.  eval_discrete (circuit.cpp:124-152), output
// check (sampler.cpp:140-145), eval_cnf (cnf.cpp:129-147).
// ---------------------------------------------------------------------------
// f = c0 ^ c1 X ^ c2 Y ^ c3 XY, coefficient k = bit k of f (sgx_layout.cpp anf_of)
__device__ __forceinline__ uint32_t anf_gate(uint32_t f, uint32_t X, uint32_t Y) {
  const uint32_t c0 = 0u - (f & 1u), c1 = 0u - ((f >> 1) & 1u), c2 = 0u - ((f >> 2) & 1u), c3 = 0u - ((f >> 3) & 1u);
  return c0 ^ (X & c1) ^ (Y & c2) ^ (X & Y & c3);
}
__device__ __forceinline__ void mbar_arrive(uint64_t* m) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(m)) : "memory");
}

__global__ void __launch_bounds__(256)
k_harvest_lw(const HarvestLiveArgs a, const int4* __restrict__ lw, int n_iters) {
  extern __shared__ __align__(128) int4 lwsm[];  // ring [kLwBuf][kLwChunk][32], then [warp][slots + 1] words
  __shared__ __align__(8) uint64_t full[kLwBuf], empty[kLwBuf];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  const int w0 = blockIdx.x * nw;
  const int active = min(nw, a.W - w0);  // warps with a word (the rest return at once)
  const int n_chunks = n_iters / kLwChunk;  // lw_ops is padded to whole chunks
  constexpr unsigned kChunkBytes = kLwChunk * 32 * sizeof(int4);
  if (threadIdx.x == 0) {
    for (int b = 0; b < kLwBuf; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&empty[b], static_cast<unsigned>(active));
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (warp >= active) return;
  if (threadIdx.x == 0)
    for (int b = 0; b < kLwBuf && b < n_chunks; ++b) bulk_load(lwsm + b * kLwChunk * 32, lw + static_cast<size_t>(b) * kLwChunk * 32, kChunkBytes / 16, &full[b]);
  const int w = w0 + warp;
  uint32_t* bits = reinterpret_cast<uint32_t*>(lwsm + kLwBuf * kLwChunk * 32) + static_cast<size_t>(warp) * (a.slots + 1);
  const size_t Wz = static_cast<size_t>(a.W);
  if (lane == 0) bits[0] = 0u;
  // phase 0 inputs: hardened V (autodiff.cpp:292-297) and free bits (sampler.cpp:132-137)
  for (int j = lane; j < a.ncpi; j += 32) {
    const int2 cs = __ldg(a.cpi + j);
    const uint32_t word = __ldg(a.hb + static_cast<size_t>(w) * a.ncpi + j);
    bits[cs.x] = word;
    if (cs.y >= 0) a.spill[cs.y * Wz + w] = word;
  }
  const int r = w * 32 + lane;
  for (int k = 0; k < a.nucpi; ++k) {
    const bool bit = fold(fold(a.free_prefix, static_cast<uint64_t>(a.row_offset + r)), static_cast<uint64_t>(k)) & 1;
    const uint32_t word = __ballot_sync(kFull, bit);
    if (lane == 0) {
      const int2 cs = __ldg(a.ucpi + k);
      bits[cs.x] = word;
      if (cs.y >= 0) a.spill[cs.y * Wz + w] = word;
    }
  }
  __syncwarp();
  uint32_t ok = kFull;
  int ph = 0;
  for (int c = 0; c < n_chunks; ++c) {
    const int b = c % kLwBuf;
    const unsigned par = static_cast<unsigned>(c / kLwBuf) & 1u;
    mbar_wait(&full[b], par);
    const int4* R = lwsm + b * kLwChunk * 32 + lane;
    // output checks and clauses of phase ph (read-only), at its last iteration
    auto phase_end = [&](const int4 op) {
      if (op.x & kLwChk) {
        const int cb = __ldg(a.chk_ptr + ph), ce = __ldg(a.chk_ptr + ph + 1);
        for (int i = cb + lane; i < ce; i += 32) {
          const int4 rec = __ldg(a.chk + i);
          uint32_t any = 0u;
          if (rec.w == kLbBig) {  // a long clause, literal by literal
            for (int l = rec.x; l < rec.x + rec.y; ++l) {
              const int lit = __ldg(a.big_lits + l), sgn = lit >> 31;
              any |= bits[lit ^ sgn] ^ static_cast<uint32_t>(sgn);
            }
          } else {
            const int lit[4] = {rec.x, rec.y, rec.z, rec.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int sgn = lit[u] >> 31;
              any |= bits[lit[u] ^ sgn] ^ static_cast<uint32_t>(sgn);
            }
          }
          ok &= any;
        }
      }
      ++ph;
      __syncwarp();
    };
    // Iterations in pairs: when the first of a pair does not end its phase,
    // both read only slots of earlier phases (and write slots no op of this
    // phase reads), so the second's operand loads go out before the first's
    // store -- two independent chains per lane.
#pragma unroll 2
    for (int it = 0; it < kLwChunk; it += 2) {
      const int4 o0 = R[it * 32], o1 = R[(it + 1) * 32];
      const uint32_t X0 = bits[o0.y], Y0 = bits[o0.z];
      const bool same = !(o0.x & kLwEnd);  // warp-uniform
      uint32_t X1 = 0u, Y1 = 0u;
      if (same) {
        X1 = bits[o1.y];
        Y1 = bits[o1.z];
      }
      const uint32_t v0 = anf_gate(o0.x, X0, Y0);
      bits[(o0.x >> 4) & 0xffffff] = v0;
      if (o0.w >= 0) a.spill[o0.w * Wz + w] = v0;
      if (!same) {
        phase_end(o0);
        X1 = bits[o1.y];
        Y1 = bits[o1.z];
      }
      const uint32_t v1 = anf_gate(o1.x, X1, Y1);
      bits[(o1.x >> 4) & 0xffffff] = v1;
      if (o1.w >= 0) a.spill[o1.w * Wz + w] = v1;
      if (o1.x & kLwEnd) phase_end(o1);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[b]);
    if (threadIdx.x == 0 && c + kLwBuf < n_chunks) {  // refill once every warp has released the chunk
      mbar_wait(&empty[b], par);
      bulk_load(lwsm + b * kLwChunk * 32, lw + static_cast<size_t>(c + kLwBuf) * kLwChunk * 32, kChunkBytes / 16, &full[b]);
    }
  }
  const uint32_t v = __reduce_and_sync(kFull, ok);
  const int r0 = w * 32;
  const uint32_t mask = r0 + 32 <= a.batch ? kFull : (r0 >= a.batch ? 0u : ((1u << (a.batch - r0)) - 1u));
  if (lane == 0) a.valid[w] = v & mask;
}

// Keys from the spill tape (dedupe_key, sampler.cpp:18-26): a CTA owns 8
// consecutive words (256 rows) and its 8 warps split the key words; lane k of
// a warp loads the 8 words of variable 32g+k as one 32-byte sector, 8 warp
// transposes give per-row key bits.  Fingerprint = mix64 of the sum of
// key_term over the key words (the same as every other harvest path), then
// the first-row-wins table insert.
__global__ void __launch_bounds__(256)
k_keys_spill(const HarvestLiveArgs a) {
  __shared__ unsigned long long hsum[256];
  __shared__ uint32_t vw[8];
  __shared__ unsigned long long kt[2][256 * 9];  // a round's 8 key words of the CTA's 256 rows, [row][8 (+1 pad)], double-buffered
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int w0 = blockIdx.x * 8;
  hsum[threadIdx.x] = 0ull;
  if (threadIdx.x < 8) vw[threadIdx.x] = w0 + threadIdx.x < a.W ? a.valid[w0 + threadIdx.x] : 0u;
  __syncthreads();
  uint32_t vm[8], anyv = 0u;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    vm[j] = vw[j];
    anyv |= vm[j];
  }
  if (anyv == 0u) return;  // block-uniform
  const size_t Wz = static_cast<size_t>(a.W);
  uint64_t h[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) h[j] = 0ull;
  // Software-pipelined over this warp's key words: the spill rows of key word
  // q + 8 are in flight while q is transposed and hashed.
  uint4 nx[2][2];
  uint32_t nm[2];
  auto fetch = [&](int q) {
#pragma unroll
    for (int hf = 0; hf < 2; ++hf) {
      const int e = q < a.key_words ? __ldg(a.key_enc + (2 * q + hf) * 32 + lane) : -1;
      nx[hf][0] = nx[hf][1] = make_uint4(0, 0, 0, 0);
      nm[hf] = e >= 0 ? neg_mask(e) : 0u;
      if (e >= 0) {
        const uint4* p = reinterpret_cast<const uint4*>(a.spill + (e >> 1) * Wz + w0);
        nx[hf][0] = __ldg(p);
        nx[hf][1] = __ldg(p + 1);
      }
    }
  };
  fetch(warp);
  // Rounds of 8 key words (warp w takes key word q0 + w), then the round's
  // words of every valid row go out row-major -- K as [row][key_words], 64
  // contiguous bytes per row per round -- so k_append_rows copies whole rows.
  const int kwn = a.key_words;
  for (int q0 = 0; q0 < kwn; q0 += 8) {
    const int q = q0 + warp;
    unsigned long long* const kb = kt[(q0 >> 3) & 1];  // written this round, stored after the barrier
    if (q < kwn) {
      uint4 cx[2][2] = {{nx[0][0], nx[0][1]}, {nx[1][0], nx[1][1]}};
      const uint32_t cm[2] = {nm[0], nm[1]};
      fetch(q + 8);
      uint32_t half[2][8];
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        const uint4 A = cx[hf][0], Bv = cx[hf][1];
        const uint32_t m = cm[hf];
        const uint32_t x[8] = {A.x ^ m, A.y ^ m, A.z ^ m, A.w ^ m, Bv.x ^ m, Bv.y ^ m, Bv.z ^ m, Bv.w ^ m};
#pragma unroll
        for (int j = 0; j < 8; ++j) half[hf][j] = transpose32(x[j], lane);
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (!vm[j]) continue;  // block-uniform
        const uint64_t kw = static_cast<uint64_t>(half[0][j]) | (static_cast<uint64_t>(half[1][j]) << 32);
        h[j] += key_term(kw, q);
        kb[(j * 32 + lane) * 9 + warp] = kw;
      }
    }
    __syncthreads();
    {  // 4 threads per row, 16 bytes each: a warp stores 8 rows x 64 B
      const int nq = min(8, kwn - q0);
      for (int t = threadIdx.x; t < 256 * 4; t += blockDim.x) {
        const int row = t >> 2, sub = t & 3, jj = row >> 5;
        if (!((vm[jj] >> (row & 31)) & 1u) || 2 * sub >= nq) continue;
        uint64_t* dst = a.K + static_cast<size_t>(w0 * 32 + row) * kwn + q0 + 2 * sub;
        if (2 * sub + 1 < nq)
          *reinterpret_cast<ulonglong2*>(dst) = make_ulonglong2(kb[row * 9 + 2 * sub], kb[row * 9 + 2 * sub + 1]);
        else
          *dst = kb[row * 9 + 2 * sub];
      }
    }
    // (no second barrier: the next round writes the other buffer, and this
    // one is rewritten only after the next round's barrier)
  }
#pragma unroll
  for (int j = 0; j < 8; ++j)
    if (vm[j]) atomicAdd(hsum + j * 32 + lane, static_cast<unsigned long long>(h[j]));
  __syncthreads();
  const int j = threadIdx.x >> 5;
  if (!((vm[j] >> lane) & 1u)) return;
  const int rr = (w0 + j) * 32 + lane;
  const uint64_t hf = mix64(hsum[threadIdx.x]);
  const unsigned long long fp = hf ? hf : 1ull;  // 0 marks an empty slot
  uint64_t idx = (fp ^ (fp >> 29)) & a.tmask;
  for (;;) {
    unsigned long long cur = a.tkeys[idx];
    if (cur == fp) break;
    if (cur == 0ull) {
      cur = atomicCAS(a.tkeys + idx, 0ull, fp);
      if (cur == 0ull || cur == fp) break;
    }
    idx = (idx + 1) & a.tmask;
  }
  atomicMin(a.tmeta + idx, static_cast<unsigned long long>((a.epoch << 32) | static_cast<uint32_t>(rr)));
  a.slot_of_row[rr] = static_cast<int>(idx);
}

bool launch_harvest_lw(cudaStream_t st, int warps_per_cta, const HarvestLiveArgs& a, const int4* lw, int n_iters) {
  const size_t smem = static_cast<size_t>(a.slots + 1) * sizeof(uint32_t) * warps_per_cta + kLwRingBytes;
  if (smem > 226 * 1024 || n_iters % kLwChunk) return false;
  opt_in_smem(reinterpret_cast<const void*>(k_harvest_lw), smem);
  k_harvest_lw<<<(a.W + warps_per_cta - 1) / warps_per_cta, 32 * warps_per_cta, smem, st>>>(a, lw, n_iters);
  k_keys_spill<<<(a.W + 7) / 8, 256, 0, st>>>(a);
  return true;
}

template <int WPC>
static bool harvest_live_t(cudaStream_t st, const HarvestLiveArgs& a) {
  const size_t smem = static_cast<size_t>(a.slots) * WPC * sizeof(uint32_t);
  if (smem > 200 * 1024) return false;
  opt_in_smem(reinterpret_cast<const void*>(k_harvest_live<WPC>), smem);
  k_harvest_live<WPC><<<a.W / WPC, kThreads, smem, st>>>(a);
  return true;
}

bool launch_harvest_live(cudaStream_t st, int wpc, const HarvestLiveArgs& a) {
  switch (wpc) {
    case 8: return harvest_live_t<8>(st, a);
    case 4: return harvest_live_t<4>(st, a);
    case 2: return harvest_live_t<2>(st, a);
    default: return harvest_live_t<1>(st, a);
  }
}

// new[w] bit r: valid row whose fingerprint this epoch first saw at this row.
// Per-block counts for the row-order scan.
__global__ void __launch_bounds__(kThreads)
k_new_rows(const uint32_t* __restrict__ valid, const int* __restrict__ slot_of_row,
           const unsigned long long* __restrict__ tmeta, uint64_t epoch, int Bp,
           uint32_t* __restrict__ newmask, int* __restrict__ block_count) {
  __shared__ int warp_cnt[kThreads / 32];
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  bool is_new = false;
  if (r < Bp && ((__ldg(valid + (r >> 5)) >> lane) & 1u)) {
    const int idx = slot_of_row[r];
    is_new = tmeta[idx] == ((epoch << 32) | static_cast<uint32_t>(r));
  }
  const uint32_t m = __ballot_sync(kFull, is_new);
  if (lane == 0) {
    if (r < Bp) newmask[r >> 5] = m;
    warp_cnt[wid] = __popc(m);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int i = 0; i < kThreads / 32; ++i) t += warp_cnt[i];
    block_count[blockIdx.x] = t;
  }
}

// Exclusive scan of the block counts (single CTA, sequential chunks), then
// the quota cut: accepted = min(new_rows, quota_left) (quota_left < 0 = none).
__global__ void __launch_bounds__(1024)
k_scan_blocks(int* __restrict__ block_count, int n_blocks, long long quota_left, HarvestOut* out) {
  __shared__ int sh[1024];
  __shared__ long long carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < n_blocks; base += 1024) {
    const int i = base + threadIdx.x;
    const int v = i < n_blocks ? block_count[i] : 0;
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {
      const int t = threadIdx.x >= off ? sh[threadIdx.x - off] : 0;
      __syncthreads();
      sh[threadIdx.x] += t;
      __syncthreads();
    }
    if (i < n_blocks) block_count[i] = static_cast<int>(carry) + sh[threadIdx.x] - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry += sh[1023];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out->new_rows = carry;
    out->accepted = quota_left < 0 ? carry : (carry < quota_left ? carry : quota_left);
    out->last_row = -1;
    out->overflow = 0;
  }
}

// Append accepted new rows, in row order, to the row-major solution store.
__global__ void __launch_bounds__(kThreads)
k_append(const uint32_t* __restrict__ newmask, const int* __restrict__ block_off, const uint64_t* __restrict__ K,
         int key_words, int Bp, uint64_t* __restrict__ store, long long store_base, long long store_cap,
         HarvestOut* out) {
  __shared__ int warp_off[kThreads / 32];
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t m = r < Bp ? __ldg(newmask + (r >> 5)) : 0u;
  if (lane == 0) warp_off[wid] = __popc(m);
  __syncthreads();
  if (!((m >> lane) & 1u)) return;
  int pos = __ldg(block_off + blockIdx.x);
  for (int i = 0; i < wid; ++i) pos += warp_off[i];
  pos += __popc(m & ((1u << lane) - 1u));
  const long long accepted = out->accepted;
  if (pos >= accepted) return;
  if (pos == accepted - 1) out->last_row = r;
  const long long dst = store_base + pos;
  if (dst >= store_cap) {
    out->overflow = 1;
    return;
  }
  for (int q = 0; q < key_words; ++q)
    store[static_cast<size_t>(dst) * key_words + q] = K[static_cast<size_t>(q) * Bp + r];
}

// ---------------------------------------------------------------------------
// Multi-GPU exchange (sample sharding): rank g owns global rows
// [g*B, (g+1)*B).  After the local insert, each rank publishes its new
// fingerprints in row order; a fingerprint new on several ranks counts for the
// lowest rank, which is exactly the reference's row order over the union of
// the shards.
// ---------------------------------------------------------------------------

// Row-order list of this harvest's locally-new fingerprints.
__global__ void __launch_bounds__(kThreads)
k_compact_new(const uint32_t* __restrict__ newmask, const int* __restrict__ block_off,
              const int* __restrict__ slot_of_row, const unsigned long long* __restrict__ tkeys, int Bp,
              unsigned long long* __restrict__ out) {
  __shared__ int warp_off[kThreads / 32];
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t m = r < Bp ? __ldg(newmask + (r >> 5)) : 0u;
  if (lane == 0) warp_off[wid] = __popc(m);
  __syncthreads();
  if (!((m >> lane) & 1u)) return;
  int pos = __ldg(block_off + blockIdx.x);
  for (int i = 0; i < wid; ++i) pos += warp_off[i];
  pos += __popc(m & ((1u << lane) - 1u));
  out[pos] = tkeys[slot_of_row[r]];
}

// Remote fingerprints: ones from lower ranks that this epoch first saw at a
// local row take that row out of the new set; every remote fingerprint not
// yet in the table is inserted with an unmatchable row tag so later epochs
// see it as old.  all_fps is [nranks][stride], counts on the host side are
// folded into n_of[rank].
__global__ void __launch_bounds__(kThreads)
k_merge_remote(const unsigned long long* __restrict__ all_fps, const long long* __restrict__ n_of,
               int nranks, int me, long long stride, unsigned long long* tkeys, unsigned long long* tmeta,
               uint64_t tmask, uint64_t epoch, uint32_t* newmask, unsigned long long* fresh) {
  const long long total = static_cast<long long>(nranks) * stride;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int rank = static_cast<int>(i / stride);
    const long long j = i - static_cast<long long>(rank) * stride;
    if (rank == me || j >= n_of[rank]) continue;
    const unsigned long long fp = all_fps[i];
    uint64_t idx = (fp ^ (fp >> 29)) & tmask;
    for (;;) {
      unsigned long long cur = tkeys[idx];
      if (cur == fp) break;
      if (cur == 0ull) {
        cur = atomicCAS(tkeys + idx, 0ull, fp);
        if (cur == 0ull) {
          atomicMin(tmeta + idx, static_cast<unsigned long long>((epoch << 32) | 0xffffffffull));
          atomicAdd(fresh, 1ull);  // |union| = local new + fresh, the same on every rank
          cur = fp;
          idx = ~0ull;  // freshly inserted: nothing local to revoke
          break;
        }
        if (cur == fp) break;
      }
      idx = (idx + 1) & tmask;
    }
    if (idx == ~0ull || rank > me) continue;
    const unsigned long long meta = tmeta[idx];
    if ((meta >> 32) == epoch && (meta & 0xffffffffull) != 0xffffffffull) {
      const uint32_t row = static_cast<uint32_t>(meta & 0xffffffffull);
      atomicAnd(newmask + (row >> 5), ~(1u << (row & 31)));
    }
  }
}

// Block counts of the (possibly revoked) new mask, for the row-order scan.
__global__ void __launch_bounds__(kThreads)
k_count_new(const uint32_t* __restrict__ newmask, int Bp, int* __restrict__ block_count) {
  __shared__ int warp_cnt[kThreads / 32];
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) warp_cnt[wid] = r < Bp ? __popc(newmask[r >> 5]) : 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int i = 0; i < kThreads / 32; ++i) t += warp_cnt[i];
    block_count[blockIdx.x] = t;
  }
}

// Move every occupied slot of the old table into the new one.
__global__ void __launch_bounds__(kThreads)
k_rehash(const unsigned long long* __restrict__ okeys, const unsigned long long* __restrict__ ometa,
         uint64_t ocap, unsigned long long* nkeys, unsigned long long* nmeta, uint64_t nmask) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < ocap;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const unsigned long long fp = okeys[i];
    if (fp == 0ull) continue;
    uint64_t idx = (fp ^ (fp >> 29)) & nmask;
    for (;;) {
      const unsigned long long cur = atomicCAS(nkeys + idx, 0ull, fp);
      if (cur == 0ull) break;
      idx = (idx + 1) & nmask;
    }
    nmeta[idx] = ometa[i];
  }
}

__global__ void k_expf(const float* __restrict__ x, long long n, float* __restrict__ out,
                       const uint64_t* __restrict__ tab, int sigmoid) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    out[i] = sigmoid ? sigmoid_ref(x[i], tab) : expf_glibc(x[i], tab);
}

// ---------------------------------------------------------------------------
// Host launch wrappers.
// ---------------------------------------------------------------------------
static int grid_for(long long n, int per_block, int cap) {
  long long g = (n + per_block - 1) / per_block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return static_cast<int>(g);
}

void launch_init_v(cudaStream_t st, float* V, int ncols, int Bp, int tile_rows, uint64_t prefix,
                   long long row_offset, uint32_t* hb) {
  if (ncols == 0) return;
  k_init_v<<<grid_for(static_cast<long long>(ncols) * Bp, kThreads, 148 * 64), kThreads, 0, st>>>(
      V, ncols, Bp, tile_rows, prefix, row_offset, hb);
}

void launch_reinit_rows(cudaStream_t st, float* V, int ncols, int Bp, int tile_rows, uint64_t prefix,
                        long long row_offset, const uint32_t* valid, const uint32_t* newmask) {
  if (ncols == 0) return;
  k_reinit_rows<<<grid_for(static_cast<long long>(ncols) * Bp, kThreads, 148 * 64), kThreads, 0, st>>>(
      V, ncols, Bp, tile_rows, prefix, row_offset, valid, newmask);
}

void launch_reinit_mask(cudaStream_t st, const uint32_t* valid, const uint32_t* newmask, uint8_t* age, int W,
                        int min_age, uint32_t* redraw) {
  k_reinit_mask<<<(W * 32 + kThreads - 1) / kThreads, kThreads, 0, st>>>(valid, newmask, age, W, min_age, redraw);
}

// Forward variant (measured on B200, c2_iscas @ 64k rows): the
// cp.async-staged forward beats the register one (1.41 vs 1.78 ms);
// SGX_SOFT=3 forces the register kernel.
static bool async_enabled_fwd() {
  static const bool on = [] {
    const char* e = std::getenv("SGX_SOFT");
    return !(e && e[0] == '3');
  }();
  return on;
}

// Grid for the tile-looped soft kernels: default one CTA per tile; SGX_GRID_FWD /
// SGX_GRID_BWD cap it (a persistent grid walks tiles with a stride).
static int tile_grid(const char* env, int tiles) {
  const char* e = getenv(env);
  int g = e ? atoi(e) : 0;
  return (g > 0 && g < tiles) ? g : tiles;
}

void launch_forward(cudaStream_t st, int vec, const int4* grp, const int2* lvl, int n_levels,
                    const float* src, int ncols, float* tape, int n_rows, int Bp, int src_is_prob,
                    const uint64_t* exp_tab, const FwdBlocks* fb) {
  const int tiles = Bp / (32 * vec);
  static const bool tma = [] {  // SGX_FWD=async: staged operands, records from L2
    const char* e = std::getenv("SGX_FWD");
    return !(e && e[0] == 'a');
  }();
  if (vec == 4 && async_enabled_fwd() && tma && fb && fb->fblk) {
    const size_t smem = static_cast<size_t>(kAsyncSmem) + 2 * static_cast<size_t>(fb->blk_max) * 16;
    if (smem <= 200 * 1024) {
      opt_in_smem(reinterpret_cast<const void*>(k_forward_tma), smem);
      static const int gcap = tile_grid("SGX_GRID_FWD", 1 << 30);
      const int grid = gcap < tiles ? gcap : tiles;
      k_forward_tma<<<grid, 32 * kWarps, smem, st>>>(fb->fblk, fb->blk0_n4, fb->blk_max, n_levels, src, ncols, tape,
                                                    n_rows, src_is_prob, exp_tab, tiles);
      return;
    }
  }
  if (vec == 4 && async_enabled_fwd()) {
    opt_in_smem(reinterpret_cast<const void*>(k_forward_async), kAsyncSmem);
    static const int gcap = tile_grid("SGX_GRID_FWD", 1 << 30);
    const int grid = gcap < tiles ? gcap : tiles;
    k_forward_async<<<grid, 32 * kWarps, kAsyncSmem, st>>>(grp, lvl, n_levels, src, ncols, tape, n_rows,
                                                          src_is_prob, exp_tab, tiles);
    return;
  }
  switch (vec) {
    case 4:
      k_forward<4><<<tiles, 32 * kWarps, 0, st>>>(grp, lvl, n_levels, src, ncols, tape, n_rows, src_is_prob, exp_tab);
      break;
    case 2:
      k_forward<2><<<tiles, 32 * kWarps, 0, st>>>(grp, lvl, n_levels, src, ncols, tape, n_rows, src_is_prob, exp_tab);
      break;
    default:
      k_forward<1><<<tiles, 32 * kWarps, 0, st>>>(grp, lvl, n_levels, src, ncols, tape, n_rows, src_is_prob, exp_tab);
  }
}


// SGX_DISCARD=0 keeps dead adjoints in L2 (A/B of the discard lists).
static bool discard_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("SGX_DISCARD");
    return !(e && e[0] == '0');
  }();
  return on;
}

void launch_backward_rec(cudaStream_t st, int vec, const int4* rec, const int2* lvl, int n_levels,
                         const float* tape, float* adj, float* V, int ncols, int n_rows, const int* col_row,
                         float* dv_out, float* dp_out, int Bp, float lr, const int* out_enc,
                         const uint8_t* out_tgt, int n_out, float* row_loss, const uint64_t* exp_tab,
                         uint32_t* hb, const int* dead, const int2* dead_lvl, const BwdBlocks* bb) {
  const int tiles = Bp / (32 * vec);
  static const int gcap = tile_grid("SGX_GRID_BWD", 1 << 30);
  const int grid = gcap < tiles ? gcap : tiles;
  static const bool staged = [] {  // SGX_BWD=reg forces the register-pipelined kernel
    const char* e = std::getenv("SGX_BWD");
    return !(e && e[0] == 'r');
  }();
  static const bool tma = [] {  // SGX_BWD=async: staged data, records from L2 (no TMA control stream)
    const char* e = std::getenv("SGX_BWD");
    return !(e && e[0] == 'a');
  }();
  if (!tma) bb = nullptr;
  if (vec == 4 && staged && bb && bb->sblk) {
    // TMA-fed kernel: 3-stage data ring when 4 CTAs still fit per SM, else 2.
    const size_t blk = 2 * static_cast<size_t>(bb->blk_max) * 16;
    const size_t s3 = static_cast<size_t>(kWarps) * 3 * kBU * 2 * 32 * 16 + blk;
    const size_t s2 = static_cast<size_t>(kWarps) * 2 * kBU * 2 * 32 * 16 + blk;
    const int disc = discard_enabled() ? 1 : 0;
    static const int force_bs = [] {  // SGX_BWD_BS=2|3 (A/B): stages regardless of occupancy
      const char* e = std::getenv("SGX_BWD_BS");
      return e ? std::atoi(e) : 0;
    }();
    if ((force_bs == 3 || (force_bs != 2 && s3 <= 54 * 1024)) && s3 <= 200 * 1024) {
      opt_in_smem(reinterpret_cast<const void*>(k_backward_tma<3>), s3);
      k_backward_tma<3><<<grid, 32 * kWarps, s3, st>>>(bb->sblk, bb->blk0_n4, bb->blk_max, n_levels, tape, adj, V,
                                                     ncols, n_rows, col_row, dv_out, dp_out, lr, out_enc, out_tgt,
                                                     n_out, row_loss, exp_tab, hb, tiles, bb->tail_dead,
                                                     bb->n_tail_dead, disc);
      return;
    }
    if (s2 <= 200 * 1024) {
      opt_in_smem(reinterpret_cast<const void*>(k_backward_tma<2>), s2);
      k_backward_tma<2><<<grid, 32 * kWarps, s2, st>>>(bb->sblk, bb->blk0_n4, bb->blk_max, n_levels, tape, adj, V,
                                                     ncols, n_rows, col_row, dv_out, dp_out, lr, out_enc, out_tgt,
                                                     n_out, row_loss, exp_tab, hb, tiles, bb->tail_dead,
                                                     bb->n_tail_dead, disc);
      return;
    }
  }
  if (vec == 4 && staged) {
    opt_in_smem(reinterpret_cast<const void*>(k_backward_async), kBwdSmem);
    k_backward_async<<<grid, 32 * kWarps, kBwdSmem, st>>>(rec, lvl, n_levels, tape, adj, V, ncols, n_rows, col_row,
                                                          dv_out, dp_out, lr, out_enc, out_tgt, n_out, row_loss,
                                                          exp_tab, hb, tiles, discard_enabled() ? dead : nullptr,
                                                          dead_lvl);
    return;
  }
  switch (vec) {
    case 4:
      k_backward_rec<4, SGX_REC_U><<<grid, 32 * kWarps, 0, st>>>(rec, lvl, n_levels, tape, adj, V, ncols, n_rows,
                                                                 col_row, dv_out, dp_out, lr, out_enc, out_tgt,
                                                                 n_out, row_loss, exp_tab, hb, tiles);
      break;
    case 2:
      k_backward_rec<2, 4><<<grid, 32 * kWarps, 0, st>>>(rec, lvl, n_levels, tape, adj, V, ncols, n_rows, col_row,
                                                         dv_out, dp_out, lr, out_enc, out_tgt, n_out, row_loss,
                                                         exp_tab, hb, tiles);
      break;
    default:
      k_backward_rec<1, 4><<<grid, 32 * kWarps, 0, st>>>(rec, lvl, n_levels, tape, adj, V, ncols, n_rows, col_row,
                                                         dv_out, dp_out, lr, out_enc, out_tgt, n_out, row_loss,
                                                         exp_tab, hb, tiles);
  }
}

void launch_loss(cudaStream_t st, const float* row_loss, int batch, double* partial, int n_partial,
                 double* out) {
  k_loss_partial<<<n_partial, kThreads, 0, st>>>(row_loss, batch, partial);
  k_loss_final<<<1, 32, 0, st>>>(partial, n_partial, out);
}

void launch_harden(cudaStream_t st, const float* V, int ncpi, int nucpi, const int* cpi_row,
                   const int* ucpi_row, uint32_t* BT, int W, int tile_rows, uint64_t free_prefix,
                   long long row_offset) {
  const long long warps = static_cast<long long>(ncpi + nucpi) * W;
  if (warps == 0) return;
  k_harden<<<grid_for(warps * 32, kThreads, 148 * 64), kThreads, 0, st>>>(
      V, ncpi, nucpi, cpi_row, ucpi_row, BT, W, tile_rows, free_prefix, row_offset);
}

void launch_bit_eval(cudaStream_t st, int wpc, const int4* ops, const int* lvl_ptr, int n_levels,
                     uint32_t* BT, int W, const int* out_row, const uint8_t* out_tgt, int n_out,
                     const int* clause_ptr, const int* clause_enc, int n_clauses, uint32_t* valid,
                     int batch) {
  switch (wpc) {
    case 8:
      k_bit_eval<8><<<W / 8, kThreads, 0, st>>>(ops, lvl_ptr, n_levels, BT, W, out_row, out_tgt, n_out,
                                                clause_ptr, clause_enc, n_clauses, valid, batch);
      break;
    case 16:
      k_bit_eval<16><<<W / 16, kThreads, 0, st>>>(ops, lvl_ptr, n_levels, BT, W, out_row, out_tgt, n_out,
                                                  clause_ptr, clause_enc, n_clauses, valid, batch);
      break;
    default:
      k_bit_eval<32><<<W / 32, kThreads, 0, st>>>(ops, lvl_ptr, n_levels, BT, W, out_row, out_tgt, n_out,
                                                  clause_ptr, clause_enc, n_clauses, valid, batch);
      break;
  }
}

void launch_keys(cudaStream_t st, const uint32_t* BT, int W, const int* key_row, int key_words,
                 const uint32_t* valid, int Bp, uint64_t* K, int* slot_of_row, unsigned long long* tkeys,
                 unsigned long long* tmeta, uint64_t tmask, uint64_t epoch) {
  const int warps = W / 8;
  k_keys<<<grid_for(static_cast<long long>(warps) * 32, kThreads, 1 << 30), kThreads, 0, st>>>(
      BT, W, key_row, key_words, valid, Bp, K, slot_of_row, tkeys, tmeta, tmask, epoch);
}

void launch_commit(cudaStream_t st, const uint32_t* valid, const int* slot_of_row,
                   const unsigned long long* tmeta, uint64_t epoch, int Bp, uint32_t* newmask,
                   int* block_count, long long quota_left, HarvestOut* out) {
  const int nb = Bp / kThreads;
  k_new_rows<<<nb, kThreads, 0, st>>>(valid, slot_of_row, tmeta, epoch, Bp, newmask, block_count);
  k_scan_blocks<<<1, 1024, 0, st>>>(block_count, nb, quota_left, out);
}

// k_append for keys staged row-major (k_keys_spill: K as [row][key_words]):
// warp j of the CTA takes the new rows of word j in row order and copies each
// whole row -- key_words contiguous u64 -- with coalesced loads and stores.
// Store position, quota cut, last row and overflow as in k_append.
__global__ void __launch_bounds__(kThreads)
k_append_rows(const uint32_t* __restrict__ newmask, const int* __restrict__ block_off, const uint64_t* __restrict__ Kr,
              int key_words, int Bp, uint64_t* __restrict__ store, long long store_base, long long store_cap,
              HarvestOut* out) {
  __shared__ int warp_off[kThreads / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int w = (blockIdx.x * kThreads >> 5) + wid;
  const uint32_t m = w * 32 < Bp ? __ldg(newmask + w) : 0u;
  if (lane == 0) warp_off[wid] = __popc(m);
  __syncthreads();
  if (!m) return;  // warp-uniform
  int pos = __ldg(block_off + blockIdx.x);
  for (int i = 0; i < wid; ++i) pos += warp_off[i];
  const long long accepted = out->accepted;
  for (uint32_t left = m; left; left &= left - 1, ++pos) {
    const int r = w * 32 + __ffs(left) - 1;
    if (pos >= accepted) return;  // (positions rise with the row)
    const long long dst = store_base + pos;
    if (dst >= store_cap) {
      if (lane == 0) out->overflow = 1;
      return;
    }
    if (pos == accepted - 1 && lane == 0) out->last_row = r;
    const uint64_t* src = Kr + static_cast<size_t>(r) * key_words;
    uint64_t* d = store + static_cast<size_t>(dst) * key_words;
    for (int i = lane; i < key_words; i += 32) d[i] = __ldg(src + i);
  }
}

void launch_append(cudaStream_t st, const uint32_t* newmask, const int* block_off, const uint64_t* K,
                   int key_words, int Bp, uint64_t* store, long long base, long long cap,
                   HarvestOut* out, bool row_major) {
  if (row_major)
    k_append_rows<<<Bp / kThreads, kThreads, 0, st>>>(newmask, block_off, K, key_words, Bp, store, base, cap, out);
  else
    k_append<<<Bp / kThreads, kThreads, 0, st>>>(newmask, block_off, K, key_words, Bp, store, base, cap, out);
}

template <int WPC>
static void harvest_smem_t(cudaStream_t st, int grid, int n_rows, size_t smem, const HarvestSmemArgs& a) {
  // Opt in whenever static (~10 KB) + dynamic could pass the 48 KB default.
  opt_in_smem(reinterpret_cast<const void*>(k_harvest_smem<WPC>), smem);
  k_harvest_smem<WPC><<<grid, kThreads, smem, st>>>(
      n_rows, a.hb, a.ncpi, a.nucpi, a.cpi_row, a.ucpi_row, a.free_prefix, a.row_offset, a.ops, a.lvl_ptr,
      a.n_levels, a.out_enc, a.out_tgt, a.n_out, a.cnf4, a.cnf_steps, a.key_enc, a.key_words,
      a.batch, a.Bp, a.valid, a.K, a.slot_of_row, a.tkeys, a.tmeta, a.tmask, a.epoch);
}

void launch_harvest_smem(cudaStream_t st, int wpc, int n_rows, int W, const HarvestSmemArgs& a) {
  const size_t smem = static_cast<size_t>(n_rows + 1) * wpc * sizeof(uint32_t);  // + the zero row
  const int grid = W / wpc;
  switch (wpc) {
    case 32: harvest_smem_t<32>(st, grid, n_rows, smem, a); break;
    case 16: harvest_smem_t<16>(st, grid, n_rows, smem, a); break;
    case 8: harvest_smem_t<8>(st, grid, n_rows, smem, a); break;
    case 4: harvest_smem_t<4>(st, grid, n_rows, smem, a); break;
    case 2: harvest_smem_t<2>(st, grid, n_rows, smem, a); break;
    default: harvest_smem_t<1>(st, grid, n_rows, smem, a); break;
  }
}

void launch_compact_new(cudaStream_t st, const uint32_t* newmask, const int* block_off, const int* slot_of_row,
                        const unsigned long long* tkeys, int Bp, unsigned long long* out) {
  k_compact_new<<<Bp / kThreads, kThreads, 0, st>>>(newmask, block_off, slot_of_row, tkeys, Bp, out);
}

void launch_merge_remote(cudaStream_t st, const unsigned long long* all_fps, const long long* n_of, int nranks,
                         int me, long long stride, unsigned long long* tkeys, unsigned long long* tmeta,
                         uint64_t tmask, uint64_t epoch, uint32_t* newmask, int Bp, int* block_count,
                         HarvestOut* out) {
  const long long total = static_cast<long long>(nranks) * stride;
  cudaMemsetAsync(&out->fresh, 0, sizeof(unsigned long long), st);
  if (total > 0)
    k_merge_remote<<<grid_for(total, kThreads, 148 * 32), kThreads, 0, st>>>(all_fps, n_of, nranks, me, stride,
                                                                          tkeys, tmeta, tmask, epoch, newmask,
                                                                          &out->fresh);
  const int nb = Bp / kThreads;
  k_count_new<<<nb, kThreads, 0, st>>>(newmask, Bp, block_count);
  k_scan_blocks<<<1, 1024, 0, st>>>(block_count, nb, -1, out);
}

void launch_rehash(cudaStream_t st, const unsigned long long* okeys, const unsigned long long* ometa,
                   uint64_t ocap, unsigned long long* nkeys, unsigned long long* nmeta, uint64_t nmask) {
  k_rehash<<<grid_for(static_cast<long long>(ocap), kThreads, 148 * 32), kThreads, 0, st>>>(
      okeys, ometa, ocap, nkeys, nmeta, nmask);
}

void launch_expf(cudaStream_t st, const float* x, long long n, float* out, const uint64_t* tab, int sigmoid) {
  k_expf<<<grid_for(n, kThreads, 148 * 32), kThreads, 0, st>>>(x, n, out, tab, sigmoid);
}

}  // namespace sgx
