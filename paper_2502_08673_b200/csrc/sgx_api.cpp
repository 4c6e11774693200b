// C-ABI implementation: device context, circuit upload, the sampler and its
// run loop (a restatement of run_impl, sampler.cpp:89-194, driving the
// kernels in sgx_kernels.cu), and the parity taps.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/satgrad_b200.h"
#include "sgx_drain.hpp"
#include "sgx_extract.hpp"
#include "sgx_jit.hpp"
#include "sgx_kernels.cuh"
#include "sgx_launch.hpp"
#include "sgx_layout.hpp"

namespace {

thread_local std::string g_err;

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NoMem : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct StateError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      throw CudaError(std::string(#call) + ": " + cudaGetErrorString(e_));                \
  } while (0)

// glibc __exp2f_data.tab (see sgx_kernels.cuh expf_glibc).
const uint64_t kExpTab[32] = {
    0x3ff0000000000000ull, 0x3fefd9b0d3158574ull, 0x3fefb5586cf9890full, 0x3fef9301d0125b51ull,
    0x3fef72b83c7d517bull, 0x3fef54873168b9aaull, 0x3fef387a6e756238ull, 0x3fef1e9df51fdee1ull,
    0x3fef06fe0a31b715ull, 0x3feef1a7373aa9cbull, 0x3feedea64c123422ull, 0x3feece086061892dull,
    0x3feebfdad5362a27ull, 0x3feeb42b569d4f82ull, 0x3feeab07dd485429ull, 0x3feea47eb03a5585ull,
    0x3feea09e667f3bcdull, 0x3fee9f75e8ec5f74ull, 0x3feea11473eb0187ull, 0x3feea589994cce13ull,
    0x3feeace5422aa0dbull, 0x3feeb737b0cdc5e5ull, 0x3feec49182a3f090ull, 0x3feed503b23e255dull,
    0x3feee89f995ad3adull, 0x3feeff76f2fb5e47ull, 0x3fef199bdd85529cull, 0x3fef3720dcef9069ull,
    0x3fef5818dcfba487ull, 0x3fef7c97337b9b5full, 0x3fefa4afa2a490daull, 0x3fefd0765b6e4540ull};

// Quiescent big device blocks kept for the next sampler of the same shape
// (exact byte size, per device): a run after a run of the same circuit and
// batch allocates its tape / adjoint / store / key buffers without asking the
// stream-ordered pool, which after a run with store growth can need new
// physical mappings for them (10-175 ms of sampler creation measured on C4).
// Capped at 40 % of device memory; flushed when an allocation fails.
namespace blockcache {
constexpr size_t kMin = size_t{64} << 20;
std::mutex mu;
std::map<std::pair<int, size_t>, std::vector<void*>> held;
std::map<int, size_t> held_bytes;
size_t cap(int dev) {
  static std::map<int, size_t> caps;
  auto it = caps.find(dev);
  if (it == caps.end()) {
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) {
      cudaGetLastError();
      tot = 0;
    }
    it = caps.emplace(dev, tot / 10 * 4).first;
  }
  return it->second;
}
void* take(size_t bytes) {
  if (bytes < kMin) return nullptr;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  auto it = held.find({dev, bytes});
  if (std::getenv("SGX_TRACE"))
    std::fprintf(stderr, "[sgx] block cache %s %.3f GB (held %.2f GB)\n",
                 (it == held.end() || it->second.empty()) ? "miss" : "hit", bytes / 1e9, held_bytes[dev] / 1e9);
  if (it == held.end() || it->second.empty()) return nullptr;
  void* p = it->second.back();
  it->second.pop_back();
  held_bytes[dev] -= bytes;
  return p;
}
bool give(void* p, size_t bytes) {
  if (bytes < kMin || std::getenv("SGX_NO_BLOCK_CACHE")) return false;
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  std::lock_guard<std::mutex> lk(mu);
  if (held_bytes[at.device] + bytes > cap(at.device)) return false;
  held[{at.device, bytes}].push_back(p);
  held_bytes[at.device] += bytes;
  return true;
}
void flush() {  // back to the pool (current device's blocks)
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  for (auto& [k, v] : held)
    if (k.first == dev) {
      for (void* p : v) cudaFreeAsync(p, 0);
      v.clear();
    }
  held_bytes[dev] = 0;
  cudaStreamSynchronize(0);
}
}  // namespace blockcache

// Owning device buffer.
template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  bool pooled = false;  // from the stream-ordered pool (freed without a device sync)
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { reset(); }
  // Owners free quiescent buffers only (samplers sync their streams first; a
  // circuit outlives its samplers), so a pooled buffer goes back to the pool
  // in the legacy stream's order instead of through cudaFree's device sync.
  void reset() {
    if (p) {
      if (pooled) {
        if (!blockcache::give(p, std::max<size_t>(n, 1) * sizeof(T))) cudaFreeAsync(p, 0);
      } else {
        cudaFree(p);
      }
    }
    p = nullptr;
    n = 0;
    pooled = false;
  }
  void alloc(size_t count) {
    reset();
    size_t bytes = std::max<size_t>(count, 1) * sizeof(T);
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) {
      cudaGetLastError();
      p = nullptr;
      throw NoMem("cudaMalloc(" + std::to_string(bytes) + " bytes): " + cudaGetErrorString(e));
    }
    n = count;
  }
  // Stream-ordered (pool) allocation: no device-wide synchronisation, so the
  // sampler can grow its table / solution store between kernels.
  void alloc_async(size_t count, cudaStream_t st) {
    reset_async(st);
    size_t bytes = std::max<size_t>(count, 1) * sizeof(T);
    if (void* q = blockcache::take(bytes)) {  // quiescent: usable on any stream
      p = static_cast<T*>(q);
      n = count;
      pooled = true;
      return;
    }
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&p), bytes, st);
    if (e != cudaSuccess) {  // the cached blocks may be what is missing
      cudaGetLastError();
      blockcache::flush();
      e = cudaMallocAsync(reinterpret_cast<void**>(&p), bytes, st);
    }
    if (e != cudaSuccess) {
      cudaGetLastError();
      p = nullptr;
      throw NoMem("cudaMallocAsync(" + std::to_string(bytes) + " bytes): " + cudaGetErrorString(e));
    }
    n = count;
    pooled = true;
  }
  void reset_async(cudaStream_t st) {
    if (p) cudaFreeAsync(p, st);
    p = nullptr;
    n = 0;
    pooled = false;
  }
  // Stream-ordered upload (pool memory; the caller syncs `st` before use
  // elsewhere).
  void upload(const std::vector<T>& v, cudaStream_t st) {
    alloc_async(v.size(), st);
    if (!v.empty()) CK(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st));
  }
  void swap(DBuf& o) {
    std::swap(p, o.p);
    std::swap(n, o.n);
    std::swap(pooled, o.pooled);
  }
};

int round_up(long long x, int m) { return static_cast<int>((x + m - 1) / m * m); }

// Small pinned host slots (a sampler's harvest counters and loss copies) from
// one process-wide pinned slab: cudaMallocHost / cudaFreeHost per sampler cost
// milliseconds (and the free synchronises), more than a quota run itself.
constexpr size_t kPinSlot = 64;
std::mutex g_pin_mu;
std::vector<void*> g_pin_free;
void* pin_slot() {
  std::lock_guard<std::mutex> lk(g_pin_mu);
  if (g_pin_free.empty()) {
    constexpr size_t kSlab = 64 * 1024;
    char* slab = nullptr;
    CK(cudaHostAlloc(reinterpret_cast<void**>(&slab), kSlab, cudaHostAllocPortable));
    for (size_t o = 0; o < kSlab; o += kPinSlot) g_pin_free.push_back(slab + o);
  }
  void* p = g_pin_free.back();
  g_pin_free.pop_back();
  std::memset(p, 0, kPinSlot);
  return p;
}
void pin_release(void* p) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_pin_mu);
  g_pin_free.push_back(p);
}

// Parity taps run the sampler's kernels with 128-sample tiles (4 per lane).
constexpr int kTapVec = 4, kTapTile = 32 * kTapVec;

// Tile-major index: sample r, row j of a [tile][rows][kTapTile] array.
size_t tile_index(int r, size_t j, size_t rows) {
  return (static_cast<size_t>(r / kTapTile) * rows + j) * kTapTile + static_cast<size_t>(r % kTapTile);
}

uint64_t next_pow2(uint64_t x) {
  uint64_t p = 1;
  while (p < x) p <<= 1;
  return p;
}

std::vector<int4> to_int4(const std::vector<sgx::I4>& v) {
  std::vector<int4> out(v.size());
  for (size_t i = 0; i < v.size(); ++i) out[i] = make_int4(v[i].x, v[i].y, v[i].z, v[i].w);
  return out;
}

std::vector<int2> to_int2(const std::vector<int32_t>& v) {
  std::vector<int2> out(v.size() / 2);
  for (size_t i = 0; i < out.size(); ++i) out[i] = make_int2(v[2 * i], v[2 * i + 1]);
  return out;
}

struct DevSoft {
  DBuf<int4> fwd, rec;
  DBuf<int2> fwd_lvl, rec_lvl, dead_lvl;
  DBuf<int> out_enc, col_row, dead, tail_dead;
  DBuf<int4> sblk, fblk;
  sgx::BwdBlocks bb;
  sgx::FwdBlocks fb;
  DBuf<int4> oc;  // on-chip program (sgx_launch.hpp OnchipArgs layout)
  int oc_n4 = 0, oc_rec = 0, oc_lvl = 0, oc_col = 0, oc_out = 0, oc_slots = 0;
  int n_fwd_levels = 0, n_bwd_levels = 0, n_rows = 0;
  void upload(const sgx::SoftProgram& P, cudaStream_t st) {
    fwd.upload(to_int4(P.fwd), st);
    rec.upload(to_int4(P.rec), st);
    fwd_lvl.upload(to_int2(P.fwd_lvl), st);
    rec_lvl.upload(to_int2(P.rec_lvl), st);
    out_enc.upload(P.out_enc, st);
    col_row.upload(P.col_row, st);
    dead.upload(P.dead.empty() ? std::vector<int32_t>{-1} : P.dead, st);
    dead_lvl.upload(to_int2(P.dead_lvl), st);
    sblk.upload(to_int4(P.sblk), st);
    tail_dead.upload(P.tail_dead.empty() ? std::vector<int32_t>{-1} : P.tail_dead, st);
    fblk.upload(to_int4(P.fblk), st);
    oc_n4 = 0;
    if (!P.oc_fwd_lvl.empty()) {  // [groups][records][per level: fwd first, count, rec first, count][col slots][out enc]
      std::vector<int4> pg;
      for (const auto& g : P.oc_fwd) pg.push_back(make_int4(g.x, g.y, g.z, g.w));
      oc_rec = static_cast<int>(pg.size());
      for (const auto& r : P.oc_rec) pg.push_back(make_int4(r.x, r.y, r.z, r.w));
      oc_lvl = static_cast<int>(pg.size());
      for (int l = 0; l < P.n_levels; ++l)
        pg.push_back(make_int4(P.oc_fwd_lvl[2 * l], P.oc_fwd_lvl[2 * l + 1], P.oc_rec_lvl[2 * l], P.oc_rec_lvl[2 * l + 1]));
      auto pack = [&](const std::vector<int32_t>& v) {
        const int at = static_cast<int>(pg.size());
        for (size_t i = 0; i < v.size(); i += 4) {
          int q[4] = {-1, -1, -1, -1};
          for (size_t j = 0; j < 4 && i + j < v.size(); ++j) q[j] = v[i + j];
          pg.push_back(make_int4(q[0], q[1], q[2], q[3]));
        }
        return at;
      };
      oc_col = pack(P.oc_col_slot);
      oc_out = pack(P.out_enc);
      oc_n4 = static_cast<int>(pg.size());
      oc_slots = P.oc_adj_slots;
      oc.upload(pg, st);
    }
    fb = sgx::FwdBlocks{};
    if (!P.fblk.empty()) {
      fb.fblk = fblk.p;
      fb.blk0_n4 = P.fblk_lvl[1];
      fb.blk_max = P.fblk_max;
    }
    bb = sgx::BwdBlocks{};
    if (!P.sblk.empty()) {
      bb.sblk = sblk.p;
      bb.blk0_n4 = P.sblk_lvl[1];
      bb.blk_max = P.sblk_max;
      bb.tail_dead = tail_dead.p;
      bb.n_tail_dead = static_cast<int>(P.tail_dead.size());
    }
    n_fwd_levels = static_cast<int>(P.fwd_lvl.size() / (2 * sgx::kWarps));
    n_bwd_levels = static_cast<int>(P.rec_lvl.size() / (2 * sgx::kWarps));
    n_rows = P.n_rows;
  }
};

void backward(cudaStream_t st, int vec, const DevSoft& P, const float* tape, float* adj, float* V, int ncols,
              float* dv_out, float* dp_out, int Bp, float lr, const uint8_t* out_tgt, int n_out, float* row_loss,
              const uint64_t* tab, uint32_t* hb) {
  sgx::launch_backward_rec(st, vec, P.rec.p, P.rec_lvl.p, P.n_bwd_levels, tape, adj, V, ncols, P.n_rows,
                           P.col_row.p, dv_out, dp_out, Bp, lr, P.out_enc.p, out_tgt, n_out, row_loss, tab, hb,
                           P.dead.p, P.dead_lvl.p, &P.bb);
}

}  // namespace

struct sgx_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  DBuf<uint64_t> exp_tab;
};

struct sgx_circuit {
  sgx_ctx* ctx = nullptr;
  sgx::Layout L;
  bool layout_ok = false;
  DevSoft cone, full;
  DBuf<int4> bit_ops;
  DBuf<int> bit_lvl_ptr, cpi_bit_row, ucpi_bit_row, out_bit_row, clause_ptr, clause_enc, key_bit_row;
  DBuf<uint8_t> out_tgt;
  int n_bit_levels = 0;
  // folded bit program (shared-memory harvest)
  DBuf<int4> fb_ops;
  DBuf<int> fb_lvl_ptr, fb_cpi_row, fb_ucpi_row, fb_out_enc, fb_key_enc;
  DBuf<int4> fb_cnf4;
  int fb_levels = 0;
  // liveness-allocated harvest (Layout::lb_*)
  DBuf<int4> lb_ops, lb_chk, lw_ops;
  DBuf<int> lb_op_ptr, lb_chk_ptr, lb_big, lb_key_enc;
  DBuf<int2> lb_cpi, lb_ucpi;
  // circuit-specialised soft pass (sgx_jit.hpp), shared by its samplers
  std::shared_ptr<sgx::JitKernel> jit;
};

// Streams and events of a sampler, pooled per (device, priority): creating
// and destroying 2 streams and 23 events per sampler costs a few hundred
// microseconds, a third of a quota-1000 run end to end.  A kit is returned
// only after both streams were synchronised, so every event in it has
// completed and a wait on one is a no-op for the next owner.
struct StreamKit {
  int device = -1;
  bool prio = false;
  cudaStream_t st = nullptr, sh = nullptr;
  cudaEvent_t ev[8] = {}, sev[2][4] = {}, soft = nullptr, front = nullptr, join = nullptr, run[4] = {};
};
std::mutex g_kit_mu;
std::vector<StreamKit> g_kits;

StreamKit kit_take(int device, bool prio, int prio_lo, int prio_hi) {
  {
    std::lock_guard<std::mutex> lk(g_kit_mu);
    for (size_t i = 0; i < g_kits.size(); ++i)
      if (g_kits[i].device == device && g_kits[i].prio == prio) {
        StreamKit k = g_kits[i];
        g_kits.erase(g_kits.begin() + static_cast<long>(i));
        return k;
      }
  }
  StreamKit k;
  k.device = device;
  k.prio = prio;
  CK(cudaStreamCreateWithPriority(&k.st, cudaStreamNonBlocking, prio ? prio_hi : prio_lo));
  CK(cudaStreamCreateWithPriority(&k.sh, cudaStreamNonBlocking, prio_lo));
  for (auto& e : k.ev) CK(cudaEventCreate(&e));
  for (auto& row : k.sev)
    for (auto& e : row) CK(cudaEventCreate(&e));
  for (auto& e : k.run) CK(cudaEventCreate(&e));
  for (auto* e : {&k.soft, &k.front, &k.join}) CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  return k;
}

void kit_destroy(StreamKit& k) {
  for (auto& e : k.ev)
    if (e) cudaEventDestroy(e);
  for (auto& row : k.sev)
    for (auto& e : row)
      if (e) cudaEventDestroy(e);
  for (auto& e : k.run)
    if (e) cudaEventDestroy(e);
  for (auto e : {k.soft, k.front, k.join})
    if (e) cudaEventDestroy(e);
  if (k.st) cudaStreamDestroy(k.st);
  if (k.sh) cudaStreamDestroy(k.sh);
}

// Return a kit whose streams are idle; at most 4 are kept per process.
void kit_give(StreamKit k) {
  {
    std::lock_guard<std::mutex> lk(g_kit_mu);
    if (g_kits.size() < 4) {
      g_kits.push_back(k);
      return;
    }
  }
  kit_destroy(k);
}

struct sgx_sampler {
  sgx_circuit* c = nullptr;
  sgx_sampler_cfg cfg{};
  cudaStream_t st = nullptr;
  int Bp = 0, W = 0, wpc = 8, vec = 2, n_partial = 148;
  int hwpc = 0;  // words per CTA of the shared-memory harvest (0: global-memory path)
  int hlive = 0;  // words per CTA of the liveness-allocated harvest (0: not used)
  int hlw = 0;    // > 0: the live program runs warp-synchronously (k_harvest_lw), warps per CTA
  bool onchip = false;  // small circuit: fused on-chip soft pass (k_soft_onchip)
  sgx::JitKernel* jit = nullptr;  // circuit-specialised soft pass (c->jit), once compiled
  bool have_tape = false;         // tape / adjoint buffers allocated (HBM soft kernels usable)
  int last_soft = 0;              // kernels of the last step: 0 HBM tape, 1 JIT, 2 on-chip
  long long jit_steps = 0;        // steps run by the JIT kernel
  int hb_cur = 0;       // HB holds two buffers; the last init / step wrote this one
  DBuf<uint32_t> SP;  // its spill tape of CNF-variable rows [n_spill][W]
  DBuf<float> V, tape, adj, row_loss;
  DBuf<float> adam_dv, adam_dp, adam_m, adam_v;  // SGX_OPT_ADAM: dV (and dP) of the step, moments
  int adam_t = 0;                                // steps since the last init
  DBuf<double> partial;
  DBuf<uint32_t> BT, valid, newmask;
  DBuf<uint8_t> row_age;    // per-row restarts: GD steps since each row's last draw
  DBuf<uint32_t> redraw;    // ... and the rows to redraw, [harvest parity][W]
  DBuf<uint32_t> HB;  // hardened V columns [word][ncpi] (shared-memory harvest input)
  DBuf<int> slot_of_row, block_count;
  DBuf<uint64_t> K, store;
  DBuf<unsigned long long> fps_local;  // multi-GPU: this harvest's new fingerprints
  DBuf<long long> n_of;                // multi-GPU: per-rank counts of the gathered lists
  DBuf<unsigned long long> fps_all;    // multi-GPU: the gathered lists [nranks][Bp + 1] (sgx_run_sharded)
  int dist_stage = 0;                  // 0 idle, 1 after local, 2 after merge
  DBuf<unsigned long long> tkeys, tmeta;
  uint64_t tcap = 0;
  long long table_count = 0;
  long long store_cap = 0, n_solutions = 0;
  std::unique_ptr<sgx::HostDrain> drain;  // host streaming of new solutions (sgx_set_host_stream)
  // The harvest runs on its own stream, overlapping the next step's forward:
  // ev_soft (st: init / step done) orders a harvest after the soft pass that
  // produced its inputs; ev_front (sh: the harvest's reads of V / HB done)
  // orders the next backward / init, which rewrite them, after it.
  cudaStream_t sh = nullptr;
  cudaEvent_t ev_soft = nullptr, ev_front = nullptr, ev_join = nullptr;
  cudaEvent_t sev[2][4] = {};  // per step parity: fwd begin / end, bwd begin / end
  cudaEvent_t rev[4] = {};     // sampler_run's init / run brackets
  bool kit_prio = false;
  DBuf<double> dloss;          // per step parity: loss total (sum over rows)
  double* hloss = nullptr;     // pinned copies of dloss (sgx_step_async / sgx_step_loss)
  long long steps = 0;         // steps launched (parity of the next)
  bool slot_pending[2] = {false, false};  // step slot launched, loss not read yet (sgx_step_loss)
  uint64_t epoch = 0;
  long long launches = 0;
  DBuf<sgx::HarvestOut> hout;
  sgx::HarvestOut* hpin = nullptr;
  // last run
  std::vector<double> loss_trace;
  std::vector<int64_t> new_unique;
  std::vector<int64_t> local_added;  // sgx_run_sharded: this rank's share of each harvest
  sgx_run_stats stats{};
  double phase_ms[8] = {0};
  double host_ms[8] = {0};  // harvest wall, table growth, store growth, (spare)
  cudaEvent_t ev[8] = {nullptr};
};

namespace {

template <typename F>
int guard(F&& f) {
  try {
    f();
    return SGX_OK;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return SGX_E_INVALID;
  } catch (const NoMem& e) {
    g_err = e.what();
    return SGX_E_NOMEM;
  } catch (const CudaError& e) {
    g_err = e.what();
    return SGX_E_CUDA;
  } catch (const StateError& e) {
    g_err = e.what();
    return SGX_E_STATE;
  } catch (const std::exception& e) {
    g_err = e.what();
    return SGX_E_INVALID;
  }
}

void need(const void* p, const char* what) {
  if (!p) throw std::invalid_argument(std::string(what) + " is null");
}

// The harvest's input words (hardened V) are double-buffered: an init or a
// step writes the buffer the running harvest is not reading.
uint32_t* hb_write(sgx_sampler* s) {
  s->hb_cur ^= 1;
  return s->HB.p + static_cast<size_t>(s->hb_cur) * s->c->L.cpi.size() * s->W;
}
uint32_t* hb_read(sgx_sampler* s) {
  return s->HB.p + static_cast<size_t>(s->hb_cur) * s->c->L.cpi.size() * s->W;
}
// Only the global-memory harvest reads V itself.
bool harvest_reads_v(const sgx_sampler* s) { return s->hwpc == 0 && s->hlive == 0; }

float elapsed(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.0f;
  CK(cudaEventElapsedTime(&ms, a, b));
  return ms;
}

// ---------------------------------------------------------------- sampler ops
void sampler_init(sgx_sampler* s, int restart) {
  const auto& L = s->c->L;
  CK(cudaStreamWaitEvent(s->st, s->ev_front, 0));  // the last harvest is done reading V
  uint64_t prefix = sgx::fold(sgx::fold(sgx::fold(sgx::kPi, s->cfg.seed), sgx::kInitTag),
                              static_cast<uint64_t>(static_cast<int64_t>(restart)));
  sgx::launch_init_v(s->st, s->V.p, static_cast<int>(L.cpi.size()), s->Bp, 32 * s->vec, prefix,
                     s->cfg.row_offset, hb_write(s));
  s->launches += L.cpi.empty() ? 0 : 1;
  if (s->row_age.p) CK(cudaMemsetAsync(s->row_age.p, 0, s->row_age.n, s->st));
  if (s->cfg.optimizer == SGX_OPT_ADAM) {
    CK(cudaMemsetAsync(s->adam_m.p, 0, s->adam_m.n * sizeof(float), s->st));
    CK(cudaMemsetAsync(s->adam_v.p, 0, s->adam_v.n * sizeof(float), s->st));
    s->adam_t = 0;
  }
  CK(cudaEventRecord(s->ev_soft, s->st));
  CK(cudaGetLastError());
}

// Per-row restarts.  SGX_RESTART_REINIT_ROWS redraws the logits of the rows a
// harvest found valid but not new; SGX_RESTART_REINIT_INVALID also those
// still invalid `reinit_age` steps after their last draw.  k_reinit_mask turns
// a harvest's valid / new masks (and the per-row ages) into a redraw mask,
// k_reinit_rows applies it.  Two schedules:
//  * at once (default): the mask of harvest it - 1 is applied before step
//    it, which then waits for that harvest;
//  * lagged (SGX_REINIT_LAG=1, no quota): the mask of harvest h is built on the harvest stream
//    right after it and applied before step h + 2, so step h + 1 still
//    overlaps harvest h.  A flagged row takes one more step (and harvest) on
//    its old draw; its age restarts at the flag, so it counts the new draw's
//    steps from the harvest after it.
int reinit_min_age(const sgx_sampler* s) {
  if (s->cfg.restart_policy != SGX_RESTART_REINIT_INVALID) return 1 << 30;  // duplicates only
  return s->cfg.reinit_age > 0 ? s->cfg.reinit_age : 2;
}

void reinit_mask(sgx_sampler* s, cudaStream_t stream, int h) {
  if (s->c->L.cpi.empty()) return;
  sgx::launch_reinit_mask(stream, s->valid.p, s->newmask.p, s->row_age.p, s->W, reinit_min_age(s),
                          s->redraw.p + static_cast<size_t>(h & 1) * s->W);
  s->launches += 1;
  CK(cudaGetLastError());
}

void reinit_apply(sgx_sampler* s, int restart, int it, int h) {
  const auto& L = s->c->L;
  if (L.cpi.empty()) return;
  const uint64_t prefix =
      sgx::fold(sgx::fold(sgx::fold(sgx::fold(sgx::kPi, s->cfg.seed), sgx::kInitTag),
                          static_cast<uint64_t>(static_cast<int64_t>(restart))),
                0x726f7773ull + static_cast<uint64_t>(it));  // "rows" + iteration
  const uint32_t* mask = s->redraw.p + static_cast<size_t>(h & 1) * s->W;
  if (std::getenv("SGX_REINIT_DEBUG")) {
    std::vector<uint32_t> m(s->W);
    CK(cudaStreamSynchronize(s->st));
    CK(cudaMemcpy(m.data(), mask, s->W * 4, cudaMemcpyDeviceToHost));
    long long nf = 0;
    for (int w = 0; w < s->W; ++w) nf += __builtin_popcount(m[w]);
    std::fprintf(stderr, "[sgx] reinit restart %d before step %d (harvest %d): %lld rows redrawn (W %d)\n", restart,
                 it, h, nf, s->W);
  }
  sgx::launch_reinit_rows(s->st, s->V.p, static_cast<int>(L.cpi.size()), s->Bp, 32 * s->vec, prefix,
                          s->cfg.row_offset, mask, nullptr);
  s->launches += 1;
  CK(cudaGetLastError());
}

// At once: the harvest before step `it` has finished (finish() waited on it).
void reinit_rows(sgx_sampler* s, int restart, int it) {
  CK(cudaEventRecord(s->ev_join, s->sh));  // valid / newmask of that harvest
  CK(cudaStreamWaitEvent(s->st, s->ev_join, 0));
  reinit_mask(s, s->st, it - 1);
  reinit_apply(s, restart, it, it - 1);
}

// How the harvest of iteration i overlaps the step of iteration i + 1
// (SGX_OVERLAP): 0 = not at all (the step waits for the harvest), 1 = the
// whole step, 2 = the forward only (the backward waits for the harvest; the
// default).  Measured on B200 (bench.py, 3 alternations): C4 4.87 M/s (1),
// 4.91-4.97 (0), 5.01-5.03 (2); C2 5.21-5.27 (1), 5.07 (0), 5.24-5.30 (2).
// The backward is the pass most hurt by a harvest beside it (C4 163 ms per
// run with it, 141 without), the forward hides it.  Letting only the harvest's
// commit / append run beside the backward (waiting on ev_front instead) was
// even on C4 (4.99-5.01 vs 4.96-4.98 M/s) with a slower backward; not kept.
int overlap_mode() {
  static const int m = [] {
    const char* e = std::getenv("SGX_OVERLAP");
    if (!e) return 2;
    if (e[0] == 'f') return 2;
    return e[0] == '0' ? 0 : 1;
  }();
  return m;
}

// One GD step; returns its parity slot (loss total in dloss[slot], timing in sev[slot]).
int sampler_step(sgx_sampler* s) {
  sgx_circuit* c = s->c;
  const uint64_t* tab = c->ctx->exp_tab.p;
  const int slot = static_cast<int>(s->steps++ & 1);
  s->slot_pending[slot] = true;
  cudaEvent_t* ev = s->sev[slot];
  CK(cudaEventRecord(ev[0], s->st));
  const int ncpi = static_cast<int>(c->L.cpi.size());
  uint32_t* hb = hb_write(s);
  if (s->jit && sgx::jit_ready(s->jit)) {
    // circuit-specialised kernel: the whole soft pass in registers
    if (harvest_reads_v(s)) CK(cudaStreamWaitEvent(s->st, s->ev_front, 0));
    CK(cudaEventRecord(ev[1], s->st));
    CK(cudaEventRecord(ev[2], s->st));
    sgx::jit_launch(s->jit, s->st, s->V.p, 32 * s->vec, hb, s->row_loss.p, tab,
                    static_cast<float>(s->cfg.learning_rate), s->Bp);
    s->last_soft = 1;
    ++s->jit_steps;
  } else if (!s->have_tape && !s->onchip) {
    throw StateError("soft pass: no kernel available (JIT not ready, no tape allocated)");
  } else if (s->onchip) {
    s->last_soft = 2;
    // forward + loss rows + backward + GD + harden in one kernel
    if (harvest_reads_v(s)) CK(cudaStreamWaitEvent(s->st, s->ev_front, 0));
    CK(cudaEventRecord(ev[1], s->st));
    CK(cudaEventRecord(ev[2], s->st));
    const DevSoft& P = c->cone;
    sgx::OnchipArgs a{};
    a.prog = P.oc.p;
    a.prog_n4 = P.oc_n4;
    a.off_rec = P.oc_rec;
    a.off_lvl = P.oc_lvl;
    a.off_col = P.oc_col;
    a.off_out = P.oc_out;
    a.n_levels = P.n_fwd_levels;
    a.n_rows = P.n_rows;
    a.n_slots = P.oc_slots;
    a.ncols = ncpi;
    a.n_out = static_cast<int>(c->L.out_node.size());
    a.V = s->V.p;
    a.hb = hb;
    a.row_loss = s->row_loss.p;
    a.out_tgt = c->out_tgt.p;
    a.exp_tab = tab;
    a.lr = static_cast<float>(s->cfg.learning_rate);
    a.n_tiles = s->Bp / 32;
    if (!sgx::launch_soft_onchip(s->st, a)) throw CudaError("on-chip soft pass does not fit");
  } else {
    s->last_soft = 0;
    sgx::launch_forward(s->st, s->vec, c->cone.fwd.p, c->cone.fwd_lvl.p, c->cone.n_fwd_levels, s->V.p, ncpi,
                        s->tape.p, c->cone.n_rows, s->Bp, 0, tab, &c->cone.fb);
    CK(cudaEventRecord(ev[1], s->st));
    if (harvest_reads_v(s)) CK(cudaStreamWaitEvent(s->st, s->ev_front, 0));  // the running harvest reads V
    if (overlap_mode() == 2) CK(cudaStreamWaitEvent(s->st, s->ev[6], 0));   // ... or all of it
    CK(cudaEventRecord(ev[2], s->st));
    if (s->cfg.optimizer == SGX_OPT_ADAM) {
      // dV out of the backward (its V update and hardening skipped), then Adam
      backward(s->st, s->vec, c->cone, s->tape.p, s->adj.p, s->V.p, ncpi, s->adam_dv.p, s->adam_dp.p, s->Bp,
               static_cast<float>(s->cfg.learning_rate), c->out_tgt.p, static_cast<int>(c->L.out_node.size()),
               s->row_loss.p, tab, nullptr);
      const auto& cf = s->cfg;
      sgx::launch_adam(s->st, s->V.p, s->adam_dv.p, s->adam_m.p, s->adam_v.p, ncpi, s->Bp, 32 * s->vec,
                       static_cast<float>(cf.learning_rate), static_cast<float>(cf.adam_beta1 > 0 ? cf.adam_beta1 : 0.9),
                       static_cast<float>(cf.adam_beta2 > 0 ? cf.adam_beta2 : 0.999), ++s->adam_t,
                       static_cast<float>(cf.adam_eps > 0 ? cf.adam_eps : 1e-8), hb);
      s->launches += 1;
    } else {
      backward(s->st, s->vec, c->cone, s->tape.p, s->adj.p, s->V.p, ncpi, nullptr, nullptr, s->Bp,
               static_cast<float>(s->cfg.learning_rate), c->out_tgt.p, static_cast<int>(c->L.out_node.size()),
               s->row_loss.p, tab, hb);
    }
  }
  sgx::launch_loss(s->st, s->row_loss.p, s->cfg.batch, s->partial.p, s->n_partial, s->dloss.p + slot);
  s->launches += s->last_soft == 0 ? 4 : 3;
  if (s->hloss)
    CK(cudaMemcpyAsync(s->hloss + slot, s->dloss.p + slot, sizeof(double), cudaMemcpyDeviceToHost, s->st));
  CK(cudaEventRecord(ev[3], s->st));
  CK(cudaEventRecord(s->ev_soft, s->st));
  CK(cudaGetLastError());
  return slot;
}

void ensure_table(sgx_sampler* s) {
  // Keep the load factor under 1/2 even if every row of this harvest is new.
  uint64_t want = static_cast<uint64_t>(s->table_count + s->Bp) * 2;
  if (want <= s->tcap) return;
  // Geometric growth with a first size covering several restarts.
  // quota runs stay small; a declared solution capacity presizes the table
  uint64_t first = s->cfg.max_solutions > 0 ? 0 : 32ull * s->Bp;
  if (s->cfg.solution_capacity > 0) first = std::max<uint64_t>(first, 2ull * s->cfg.solution_capacity);
  uint64_t ncap = next_pow2(std::max<uint64_t>(std::max<uint64_t>(want * 2, first), 1u << 16));
  DBuf<unsigned long long> nk, nm;
  nk.alloc_async(ncap, s->sh);
  nm.alloc_async(ncap, s->sh);
  CK(cudaMemsetAsync(nk.p, 0, ncap * sizeof(unsigned long long), s->sh));
  CK(cudaMemsetAsync(nm.p, 0xff, ncap * sizeof(unsigned long long), s->sh));
  if (s->tcap) {
    sgx::launch_rehash(s->sh, s->tkeys.p, s->tmeta.p, s->tcap, nk.p, nm.p, ncap - 1);
    s->launches += 1;
  }
  CK(cudaGetLastError());
  s->tkeys.swap(nk);
  s->tmeta.swap(nm);
  nk.reset_async(s->sh);  // the old table, after the rehash in stream order
  nm.reset_async(s->sh);
  s->tcap = ncap;
}

// Stream-ordered growth of the row-major solution store (no host sync).
void grow_store(sgx_sampler* s, long long need_rows) {
  long long ncap = std::max<long long>(need_rows, s->store_cap * 2);
  const size_t kw = static_cast<size_t>(s->c->L.key_words);
  if (s->drain) s->drain->wait_idle();  // no host copy may still read the old store
  DBuf<uint64_t> ns;
  ns.alloc_async(static_cast<size_t>(ncap) * kw, s->sh);
  if (s->n_solutions)
    CK(cudaMemcpyAsync(ns.p, s->store.p, static_cast<size_t>(s->n_solutions) * kw * sizeof(uint64_t),
                       cudaMemcpyDeviceToDevice, s->sh));
  s->store.swap(ns);
  ns.reset_async(s->sh);
  s->store_cap = ncap;
}

// The harvest lambda of sampler.cpp:124-153 for one (restart, iter).
// quota_left < 0 means no quota.  Returns rows attempted and solutions added.
// Front half: harden, bit-sliced eval + PO/CNF check, keys + local insert, the
// row-order scan of the new rows (quota applied when quota_left >= 0).
void harvest_front(sgx_sampler* s, int restart, int iter, long long quota_left) {
  sgx_circuit* c = s->c;
  const auto& L = c->L;
  {
    const auto t0 = std::chrono::steady_clock::now();
    ensure_table(s);
    s->host_ms[1] += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }
  CK(cudaStreamWaitEvent(s->sh, s->ev_soft, 0));  // the soft pass that produced V / HB
  CK(cudaEventRecord(s->ev[3], s->sh));
  uint64_t fprefix = sgx::fold(
      sgx::fold(sgx::fold(sgx::fold(sgx::kPi, s->cfg.seed), sgx::kFreeTag), static_cast<uint64_t>(static_cast<int64_t>(restart))),
      static_cast<uint64_t>(static_cast<int64_t>(iter)));
  s->epoch += 1;
  if (s->hlive > 0) {
    sgx::HarvestLiveArgs a{};
    a.hb = hb_read(s);
    a.ncpi = static_cast<int>(L.cpi.size());
    a.nucpi = static_cast<int>(L.ucpi.size());
    a.cpi = c->lb_cpi.p;
    a.ucpi = c->lb_ucpi.p;
    a.free_prefix = fprefix;
    a.row_offset = s->cfg.row_offset;
    a.ops = c->lb_ops.p;
    a.op_ptr = c->lb_op_ptr.p;
    a.chk = c->lb_chk.p;
    a.chk_ptr = c->lb_chk_ptr.p;
    a.big_lits = c->lb_big.p;
    a.n_phases = L.lb_levels;
    a.slots = L.lb_slots;
    a.spill = s->SP.p;
    a.W = s->W;
    a.n_spill = std::max(L.lb_n_spill, 1);
    a.key_enc = c->lb_key_enc.p;
    a.key_words = L.key_words;
    a.batch = s->cfg.batch;
    a.Bp = s->Bp;
    a.valid = s->valid.p;
    a.K = s->K.p;
    a.slot_of_row = s->slot_of_row.p;
    a.tkeys = s->tkeys.p;
    a.tmeta = s->tmeta.p;
    a.tmask = s->tcap - 1;
    a.epoch = s->epoch;
    if (s->hlw > 0) {
      if (!sgx::launch_harvest_lw(s->sh, s->hlw, a, c->lw_ops.p, L.lw_iters))
        throw CudaError("live harvest does not fit shared memory");
      s->launches += 1;
    } else if (!sgx::launch_harvest_live(s->sh, s->hlive, a)) {
      throw CudaError("live harvest does not fit shared memory");
    }
    CK(cudaEventRecord(s->ev[4], s->sh));
    CK(cudaEventRecord(s->ev[5], s->sh));
    s->launches += 1;
  } else if (s->hwpc > 0) {
    sgx::HarvestSmemArgs a{};
    a.hb = hb_read(s);
    a.ncpi = static_cast<int>(L.cpi.size());
    a.nucpi = static_cast<int>(L.ucpi.size());
    a.cpi_row = c->fb_cpi_row.p;
    a.ucpi_row = c->fb_ucpi_row.p;
    a.free_prefix = fprefix;
    a.row_offset = s->cfg.row_offset;
    a.ops = c->fb_ops.p;
    a.lvl_ptr = c->fb_lvl_ptr.p;
    a.n_levels = c->fb_levels;
    a.out_enc = c->fb_out_enc.p;
    a.out_tgt = c->out_tgt.p;
    a.n_out = static_cast<int>(L.out_node.size());
    a.cnf4 = c->fb_cnf4.p;
    a.cnf_steps = L.fb_cnf_steps;
    a.key_enc = c->fb_key_enc.p;
    a.key_words = L.key_words;
    a.batch = s->cfg.batch;
    a.Bp = s->Bp;
    a.valid = s->valid.p;
    a.K = s->K.p;
    a.slot_of_row = s->slot_of_row.p;
    a.tkeys = s->tkeys.p;
    a.tmeta = s->tmeta.p;
    a.tmask = s->tcap - 1;
    a.epoch = s->epoch;
    sgx::launch_harvest_smem(s->sh, s->hwpc, L.fb_rows, s->W, a);
    CK(cudaEventRecord(s->ev[4], s->sh));
    CK(cudaEventRecord(s->ev[5], s->sh));
    s->launches += 1;
  } else {
    sgx::launch_harden(s->sh, s->V.p, static_cast<int>(L.cpi.size()), static_cast<int>(L.ucpi.size()),
                       c->cpi_bit_row.p, c->ucpi_bit_row.p, s->BT.p, s->W, 32 * s->vec, fprefix,
                       s->cfg.row_offset);
    sgx::launch_bit_eval(s->sh, s->wpc, c->bit_ops.p, c->bit_lvl_ptr.p, c->n_bit_levels, s->BT.p, s->W,
                         c->out_bit_row.p, c->out_tgt.p, static_cast<int>(L.out_node.size()), c->clause_ptr.p,
                         c->clause_enc.p, static_cast<int>(L.hclause_ptr.size()) - 1, s->valid.p, s->cfg.batch);
    CK(cudaEventRecord(s->ev[4], s->sh));
    sgx::launch_keys(s->sh, s->BT.p, s->W, c->key_bit_row.p, L.key_words, s->valid.p, s->Bp, s->K.p,
                     s->slot_of_row.p, s->tkeys.p, s->tmeta.p, s->tcap - 1, s->epoch);
    CK(cudaEventRecord(s->ev[5], s->sh));
    s->launches += (L.cpi.size() + L.ucpi.size() ? 1 : 0) + 2;
  }
  CK(cudaEventRecord(s->ev_front, s->sh));
  sgx::launch_commit(s->sh, s->valid.p, s->slot_of_row.p, s->tmeta.p, s->epoch, s->Bp, s->newmask.p,
                     s->block_count.p, quota_left, s->hout.p);
  s->launches += 2;
}

// Back half, launch: append the accepted rows (hout->accepted) in row order
// and queue the counters (and the loss of step `loss_slot`, if any) for the
// host; no sync.
void harvest_back_launch(sgx_sampler* s, int loss_slot) {
  const auto& L = s->c->L;
  sgx::launch_append(s->sh, s->newmask.p, s->block_count.p, s->K.p, L.key_words, s->Bp, s->store.p,
                     s->n_solutions, s->store_cap, s->hout.p, s->hlw > 0);
  s->launches += 1;
  CK(cudaEventRecord(s->ev[6], s->sh));
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(s->hpin, s->hout.p, sizeof(sgx::HarvestOut), cudaMemcpyDeviceToHost, s->sh));
  if (loss_slot >= 0)
    CK(cudaMemcpyAsync(&s->hpin->loss_total, s->dloss.p + loss_slot, sizeof(double), cudaMemcpyDeviceToHost,
                       s->sh));
}

// Back half, finish: the one host sync of the harvest, store overflow
// handling, counters.  Device time of the harvest (and of the step it
// followed, slot `step_slot`) is accumulated here, once its events are done.
void harvest_back_finish(sgx_sampler* s, long long quota_left, long long* attempts, long long* added,
                         int step_slot) {
  const auto& L = s->c->L;
  static const bool trace2 = std::getenv("SGX_TRACE2") != nullptr;
  const auto tw = std::chrono::steady_clock::now();
  CK(cudaStreamSynchronize(s->sh));
  if (trace2) {
    const double w = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tw).count();
    std::fprintf(stderr, "[sgx] harvest sync wait %.3f ms, harvest gpu %.3f ms, step gpu %.3f ms\n", w,
                 elapsed(s->ev[3], s->ev[6]), step_slot >= 0 ? elapsed(s->sev[step_slot][0], s->sev[step_slot][3]) : 0.0);
  }
  if (s->hpin->overflow) {
    const double loss = s->hpin->loss_total;
    const auto t0 = std::chrono::steady_clock::now();
    grow_store(s, s->n_solutions + s->hpin->accepted);
    s->host_ms[2] += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    CK(cudaMemsetAsync(&s->hout.p->overflow, 0, sizeof(long long), s->sh));
    sgx::launch_append(s->sh, s->newmask.p, s->block_count.p, s->K.p, L.key_words, s->Bp, s->store.p,
                       s->n_solutions, s->store_cap, s->hout.p, s->hlw > 0);
    s->launches += 1;
    CK(cudaMemcpyAsync(s->hpin, s->hout.p, sizeof(sgx::HarvestOut), cudaMemcpyDeviceToHost, s->sh));
    CK(cudaStreamSynchronize(s->sh));
    s->hpin->loss_total = loss;
    if (s->hpin->overflow) throw CudaError("solution store overflow after growth");
  }
  const sgx::HarvestOut& h = *s->hpin;
  s->table_count += h.new_rows;
  if (s->drain && h.accepted > 0) s->drain->push(s->store.p, s->n_solutions, h.accepted, s->sh);
  s->n_solutions += h.accepted;
  *added = h.accepted;
  // Grow ahead of need, in stream order, so the next harvest never overflows.
  if (s->store_cap - s->n_solutions < s->Bp) {
    const auto t0 = std::chrono::steady_clock::now();
    grow_store(s, s->n_solutions + 2LL * s->Bp);
    s->host_ms[2] += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }
  // Quota met inside this harvest: the reference stops at the row after the
  // one that filled it (sampler.cpp:129).
  if (quota_left >= 0 && h.accepted == quota_left && h.accepted > 0)
    *attempts = h.last_row + 1;
  else
    *attempts = s->cfg.batch;
  s->phase_ms[2] += elapsed(s->ev[3], s->ev[6]);
  s->phase_ms[5] += elapsed(s->ev[3], s->ev[4]);
  s->phase_ms[6] += elapsed(s->ev[4], s->ev[5]);
  s->phase_ms[7] += elapsed(s->ev[5], s->ev[6]);
  if (step_slot >= 0) {
    cudaEvent_t* ev = s->sev[step_slot];
    s->phase_ms[1] += elapsed(ev[0], ev[3]);
    s->phase_ms[3] += elapsed(ev[0], ev[1]);
    s->phase_ms[4] += elapsed(ev[2], ev[3]);
  }
}

// The harvest lambda of sampler.cpp:124-153 for one (restart, iter), single
// device: quota applied in the scan, one host sync.  `step_slot` = parity
// slot of the step this harvest follows (-1 after init).
void sampler_harvest(sgx_sampler* s, int restart, int iter, long long quota_left, long long* attempts,
                     long long* added, int step_slot) {
  harvest_front(s, restart, iter, quota_left);
  harvest_back_launch(s, step_slot);
  harvest_back_finish(s, quota_left, attempts, added, step_slot);
}

// run_impl<float> (sampler.cpp:89-194).
void sampler_run(sgx_sampler* s) {
  using clock = std::chrono::steady_clock;
  const auto t0 = clock::now();
  auto now_s = [&] { return std::chrono::duration<double>(clock::now() - t0).count(); };
  const sgx_sampler_cfg& cfg = s->cfg;
  s->loss_trace.clear();
  s->new_unique.clear();
  s->stats = sgx_run_stats{};
  std::fill(s->phase_ms, s->phase_ms + 8, 0.0);
  std::fill(s->host_ms, s->host_ms + 8, 0.0);
  s->launches = 0;
  if (s->c->L.unsat) {
    s->stats.unsat = 1;
    s->stats.wall_time_s = now_s();
    return;
  }
  const bool quota = cfg.max_solutions > 0;
  auto quota_met = [&] { return quota && s->n_solutions >= cfg.max_solutions; };
  auto out_of_time = [&] { return cfg.timeout_s > 0.0 && now_s() >= cfg.timeout_s; };
  // Harvest `iter` finishes on the host; its counters feed the reference's
  // bookkeeping (attempts, per-harvest new-unique, loss trace).
  auto finish = [&](int iter, long long quota_left, int step_slot) {
    long long att = 0, add = 0;
    const auto h0 = clock::now();
    harvest_back_finish(s, quota_left, &att, &add, step_slot);
    s->host_ms[0] += std::chrono::duration<double, std::milli>(clock::now() - h0).count();
    s->stats.attempts += att;
    s->new_unique.push_back(add);
    if (iter > 0) s->loss_trace.push_back(s->hpin->loss_total / cfg.batch);
  };
  auto quota_left = [&] { return quota ? cfg.max_solutions - s->n_solutions : -1LL; };
  const bool overlap = overlap_mode() != 0;  // SGX_OVERLAP=0: the next step waits for the harvest
  const int max_restarts = cfg.max_restarts > 0 ? cfg.max_restarts : 1000;
  const bool per_row =
      cfg.restart_policy == SGX_RESTART_REINIT_ROWS || cfg.restart_policy == SGX_RESTART_REINIT_INVALID;
  // SGX_REINIT_LAG=1: per-row redraws one harvest late, keeping the overlap
  // (reinit_rows above).  Opt-in: a row flagged at harvest h may turn valid
  // at h + 1 and is redrawn anyway (C4 age 1: 1.13x against 1.20x at once;
  // C2 loses solutions, tools/reinit_invalid_ab.py).
  const char* lag_env = std::getenv("SGX_REINIT_LAG");
  const bool lag = per_row && overlap && !quota && lag_env && lag_env[0] == '1';
  auto lag_apply = [&](int restart, int it) {     // mask of harvest it - 2 (finished: finish() synced it)
    if (it < 2) return;
    if (harvest_reads_v(s)) CK(cudaStreamWaitEvent(s->st, s->ev_front, 0));  // harvest it - 1 reads V
    reinit_apply(s, restart, it, it - 2);
  };
  bool timed_out = false;
  cudaEvent_t e0 = s->rev[0], e1 = s->rev[1], r0 = s->rev[2], r1 = s->rev[3];
  CK(cudaEventRecord(r0, s->st));
  for (int restart = 0;; ++restart) {
    CK(cudaEventRecord(e0, s->st));
    sampler_init(s, restart);
    CK(cudaEventRecord(e1, s->st));
    const long long before = s->n_solutions;
    // Harvest `h_iter` (stream sh) runs while the step of iteration h_iter + 1
    // (stream st) already samples: the step needs only V, the harvest only
    // the hardened words, and the backward waits for the harvest's reads
    // (ev_front) before rewriting them.  Without a quota the next step is
    // launched before the host waits on the harvest (it is discarded if the
    // run stops there); with a quota it follows the harvest, as the reference
    // decides per row whether to continue (sampler.cpp:129, :163).
    long long h_quota = quota_left();
    auto hclk = clock::now();
    auto hlap = [&](int k) {
      const auto n = clock::now();
      s->host_ms[k] += std::chrono::duration<double, std::milli>(n - hclk).count();
      hclk = n;
    };
    harvest_front(s, restart, 0, h_quota);
    harvest_back_launch(s, -1);
    if (lag) reinit_mask(s, s->sh, 0);
    hlap(3);
    int h_iter = 0, h_slot = -1;
    for (;;) {
      const int it = h_iter + 1;
      int slot = -1;
      if (overlap && (!per_row || lag) && !quota && it <= cfg.iterations && !out_of_time()) {
        if (lag) lag_apply(restart, it);
        slot = sampler_step(s);
      }
      hlap(4);
      finish(h_iter, h_quota, h_slot);
      if (h_iter == 0) s->phase_ms[0] += elapsed(e0, e1);
      hlap(5);
      if (it > cfg.iterations || quota_met()) break;
      if (out_of_time()) {  // sampler.cpp:164: checked before every step
        timed_out = true;
        break;
      }
      if (per_row && !lag && slot < 0) reinit_rows(s, restart, it);
      if (slot < 0) {
        if (lag) lag_apply(restart, it);
        slot = sampler_step(s);
      }
      h_quota = quota_left();
      hlap(4);
      harvest_front(s, restart, it, h_quota);
      harvest_back_launch(s, slot);
      if (lag) reinit_mask(s, s->sh, it);
      hlap(3);
      h_iter = it;
      h_slot = slot;
    }
    if (quota_met() || timed_out) break;
    if (cfg.restart_policy == SGX_RESTART_NONE) break;
    if (s->n_solutions == before) break;
    if (restart >= max_restarts) break;
    if (out_of_time()) {
      timed_out = true;
      break;
    }
    s->stats.restarts = restart + 1;
  }
  CK(cudaEventRecord(s->ev_join, s->sh));
  CK(cudaStreamWaitEvent(s->st, s->ev_join, 0));
  CK(cudaEventRecord(r1, s->st));
  CK(cudaEventSynchronize(r1));
  s->stats.device_ms = elapsed(r0, r1);
  s->stats.launches = s->launches;
  if (std::getenv("SGX_TRACE"))
    std::fprintf(stderr, "[sgx] device %.2f ms; harvest wall %.2f ms (table growth %.2f, store growth %.2f); "
                 "phases init %.2f step %.2f harvest %.2f; host: harvest launch %.2f step launch %.2f finish %.2f, "
                 "run wall %.2f ms\n", s->stats.device_ms, s->host_ms[0], s->host_ms[1],
                 s->host_ms[2], s->phase_ms[0], s->phase_ms[1], s->phase_ms[2], s->host_ms[3], s->host_ms[4],
                 s->host_ms[5], 1000.0 * now_s());
  s->stats.timed_out = timed_out ? 1 : 0;
  s->stats.unique_count = s->n_solutions;
  s->stats.wall_time_s = now_s();
  s->stats.throughput = s->stats.wall_time_s > 0.0 ? s->n_solutions / s->stats.wall_time_s : 0.0;
  s->stats.n_loss = static_cast<int32_t>(s->loss_trace.size());
  s->stats.n_harvest = static_cast<int32_t>(s->new_unique.size());
}

// ------------------------------------------------------------ multi-GPU
// The split harvest (sample sharding): the local front half
// publishes this harvest's new fingerprints in row order (count at [Bp]),
// the caller's all-gather exchanges them, the merge revokes rows a lower rank
// also found (lowest rank wins = the reference's row order over the union)
// and inserts every remote fingerprint, the commit appends the winners.
long long dist_local(sgx_sampler* s, int restart, int iter) {
  if (s->dist_stage != 0) throw StateError("sgx_harvest_local: previous harvest not committed");
  if (!s->fps_local.p) s->fps_local.alloc_async(static_cast<size_t>(s->Bp) + 1, s->sh);
  harvest_front(s, restart, iter, -1);
  sgx::launch_compact_new(s->sh, s->newmask.p, s->block_count.p, s->slot_of_row.p, s->tkeys.p, s->Bp,
                          s->fps_local.p);
  s->launches += 1;
  CK(cudaGetLastError());
  // the count rides at [stride] so one all-gather carries fingerprints and counts
  CK(cudaMemcpyAsync(s->fps_local.p + s->Bp, &s->hout.p->new_rows, sizeof(long long), cudaMemcpyDeviceToDevice,
                     s->sh));
  CK(cudaMemcpyAsync(s->hpin, s->hout.p, sizeof(sgx::HarvestOut), cudaMemcpyDeviceToHost, s->sh));
  CK(cudaStreamSynchronize(s->sh));
  s->dist_stage = 1;
  return s->hpin->new_rows;
}

// Returns the rows still new here; *fresh = remote fingerprints new to the
// table, so |union of this harvest| = local new + *fresh on every rank.
long long dist_merge(sgx_sampler* s, const uint64_t* all_fps, const std::vector<long long>& cnt, int rank,
                     long long stride, long long* fresh) {
  if (s->dist_stage != 1) throw StateError("sgx_harvest_merge: call sgx_harvest_local first");
  const int nranks = static_cast<int>(cnt.size());
  const long long n_local = s->hpin->new_rows;
  long long remote = 0;
  for (int r = 0; r < nranks; ++r) {
    if (cnt[r] < 0 || cnt[r] > stride) throw std::invalid_argument("fingerprint count out of range");
    if (r != rank) remote += cnt[r];
  }
  // Room for every remote fingerprint at load factor <= 1/2.
  s->table_count += remote;
  ensure_table(s);
  if (!s->n_of.p || static_cast<int>(s->n_of.n) < nranks) s->n_of.alloc_async(std::max(nranks, 64), s->sh);
  CK(cudaMemcpyAsync(s->n_of.p, cnt.data(), nranks * sizeof(long long), cudaMemcpyHostToDevice, s->sh));
  sgx::launch_merge_remote(s->sh, reinterpret_cast<const unsigned long long*>(all_fps), s->n_of.p,
                           nranks > 1 ? nranks : 0, rank, stride, s->tkeys.p, s->tmeta.p, s->tcap - 1, s->epoch,
                           s->newmask.p, s->Bp, s->block_count.p, s->hout.p);
  s->launches += nranks > 1 ? 3 : 2;
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(s->hpin, s->hout.p, sizeof(sgx::HarvestOut), cudaMemcpyDeviceToHost, s->sh));
  CK(cudaStreamSynchronize(s->sh));
  // Locally-new rows another rank claimed still occupy table slots; so do
  // the remote fingerprints (counted above), minus those already present.
  s->table_count += n_local - s->hpin->new_rows;
  s->table_count -= remote - static_cast<long long>(s->hpin->fresh);
  *fresh = static_cast<long long>(s->hpin->fresh);
  s->dist_stage = 2;
  return s->hpin->new_rows;
}

void dist_commit(sgx_sampler* s, long long quota_left, long long* attempts, long long* added) {
  if (s->dist_stage != 2) throw StateError("sgx_harvest_commit: call sgx_harvest_merge first");
  sgx::HarvestOut h = *s->hpin;
  h.accepted = quota_left < 0 ? h.new_rows : std::min<long long>(h.new_rows, quota_left);
  h.last_row = -1;
  h.overflow = 0;
  *s->hpin = h;
  CK(cudaMemcpyAsync(s->hout.p, s->hpin, sizeof(sgx::HarvestOut), cudaMemcpyHostToDevice, s->sh));
  harvest_back_launch(s, -1);
  harvest_back_finish(s, quota_left, attempts, added, -1);  // counts the winners into table_count
  s->dist_stage = 0;
}

void check_ex(int rc, const char* what) {
  if (rc != 0) throw CudaError(std::string("exchange ") + what + " failed (" + std::to_string(rc) + ")");
}

// run_impl<float> (sampler.cpp:89-194) over the union of nranks sample
// shards, one sampler per rank (rank g owns global rows [g*B, (g+1)*B) via
// cfg.row_offset).  One device all-gather per harvest carries every rank's
// new fingerprints and their counts; the union's size is derived locally
// (local new + fresh remote inserts).  Under a quota the winners' counts are
// all-gathered too (the cut goes in rank order), and with a timeout a late
// flag, so every rank takes the same branch.  The next step is launched as
// soon as the local harvest kernels are done, so the exchange overlaps it.
void sampler_run_sharded(sgx_sampler* s, const sgx_exchange* ex) {
  using clock = std::chrono::steady_clock;
  const auto t0 = clock::now();
  auto now_s = [&] { return std::chrono::duration<double>(clock::now() - t0).count(); };
  const sgx_sampler_cfg& cfg = s->cfg;
  const int R = ex->nranks, me = ex->rank;
  s->loss_trace.clear();
  s->new_unique.clear();
  s->local_added.clear();
  s->stats = sgx_run_stats{};
  std::fill(s->phase_ms, s->phase_ms + 8, 0.0);
  std::fill(s->host_ms, s->host_ms + 8, 0.0);
  s->launches = 0;
  if (s->c->L.unsat) {
    s->stats.unsat = 1;
    s->stats.wall_time_s = now_s();
    return;
  }
  const long long stride = static_cast<long long>(s->Bp) + 1;
  if (!s->fps_local.p) s->fps_local.alloc_async(static_cast<size_t>(stride), s->sh);
  if (s->fps_all.n < static_cast<size_t>(R * stride)) s->fps_all.alloc_async(static_cast<size_t>(R * stride), s->sh);
  std::vector<long long> counts(R);
  std::vector<int64_t> hv(R);
  const bool quota = cfg.max_solutions > 0;
  long long unique = 0;  // global
  auto quota_met = [&] { return quota && unique >= cfg.max_solutions; };
  auto gather1 = [&](int64_t x) {
    check_ex(ex->allgather_host(ex->user, &x, hv.data(), 1), "allgather_host");
    return hv;
  };
  auto out_of_time = [&] {  // any rank over time stops every rank
    if (cfg.timeout_s <= 0.0) return false;
    const auto all = gather1(now_s() >= cfg.timeout_s ? 1 : 0);
    return std::any_of(all.begin(), all.end(), [](int64_t v) { return v != 0; });
  };
  const bool overlap = overlap_mode() != 0;
  auto harvest = [&](int restart, int it, bool launch_next) {
    const auto h0 = clock::now();
    dist_local(s, restart, it);
    const int slot = launch_next ? sampler_step(s) : -1;
    check_ex(ex->allgather_device(ex->user, s->fps_local.p, s->fps_all.p, stride * 8, s->sh), "allgather_device");
    CK(cudaMemcpy2DAsync(counts.data(), sizeof(long long), s->fps_all.p + s->Bp, stride * sizeof(long long),
                         sizeof(long long), R, cudaMemcpyDeviceToHost, s->sh));
    CK(cudaStreamSynchronize(s->sh));
    long long fresh = 0;
    const long long n_local = s->hpin->new_rows;
    const long long won = dist_merge(s, reinterpret_cast<const uint64_t*>(s->fps_all.p), counts, me, stride, &fresh);
    long long att = 0, add = 0, acc = 0;
    if (!quota) {
      dist_commit(s, -1, &att, &add);
      acc = n_local + fresh;
      s->stats.attempts += static_cast<long long>(cfg.batch) * R;
    } else {
      const long long left = cfg.max_solutions - unique;
      const auto wons = gather1(won);
      long long before = 0;
      for (int q = 0; q < me; ++q) before += wons[q];
      const long long my_left = std::max(0LL, left - before);
      dist_commit(s, my_left, &att, &add);
      if (my_left == 0) att = 0;  // a lower rank filled the quota: these rows come after the cut
      for (int q = 0; q < R; ++q) acc += std::max(0LL, std::min<long long>(wons[q], left - acc));
      const auto atts = gather1(att);
      for (int q = 0; q < R; ++q) s->stats.attempts += atts[q];
    }
    unique += acc;
    s->new_unique.push_back(acc);
    s->local_added.push_back(add);
    s->host_ms[0] += std::chrono::duration<double, std::milli>(clock::now() - h0).count();
    return slot;
  };
  auto speculate = [&](int it) { return overlap && !quota && cfg.timeout_s <= 0.0 && it <= cfg.iterations; };
  auto step_loss = [&](int slot) {
    CK(cudaEventSynchronize(s->sev[slot][3]));
    s->slot_pending[slot] = false;
    cudaEvent_t* ev = s->sev[slot];
    s->phase_ms[1] += elapsed(ev[0], ev[3]);
    s->phase_ms[3] += elapsed(ev[0], ev[1]);
    s->phase_ms[4] += elapsed(ev[2], ev[3]);
    return s->hloss[slot];
  };
  const int max_restarts = cfg.max_restarts > 0 ? cfg.max_restarts : 1000;
  bool timed_out = false;
  cudaEvent_t r0 = s->rev[2], r1 = s->rev[3];
  CK(cudaEventRecord(r0, s->st));
  for (int restart = 0;; ++restart) {
    sampler_init(s, restart);
    const long long before = unique;
    int slot = harvest(restart, 0, speculate(1));
    for (int it = 1; it <= cfg.iterations; ++it) {
      if (quota_met()) break;
      if (out_of_time()) {
        timed_out = true;
        break;
      }
      if (slot < 0) slot = sampler_step(s);
      s->loss_trace.push_back(step_loss(slot) / cfg.batch);
      slot = harvest(restart, it, speculate(it + 1));
    }
    if (slot >= 0) step_loss(slot);  // a speculative step nobody harvests: let it finish
    if (quota_met() || timed_out) break;
    if (cfg.restart_policy == SGX_RESTART_NONE) break;
    if (unique == before) break;
    if (restart >= max_restarts) break;
    if (out_of_time()) {
      timed_out = true;
      break;
    }
    s->stats.restarts = restart + 1;
  }
  CK(cudaEventRecord(s->ev_join, s->sh));
  CK(cudaStreamWaitEvent(s->st, s->ev_join, 0));
  CK(cudaEventRecord(r1, s->st));
  CK(cudaEventSynchronize(r1));
  s->stats.device_ms = elapsed(r0, r1);
  s->stats.launches = s->launches;
  s->stats.timed_out = timed_out ? 1 : 0;
  s->stats.unique_count = unique;
  s->stats.wall_time_s = now_s();
  s->stats.throughput = s->stats.wall_time_s > 0.0 ? unique / s->stats.wall_time_s : 0.0;
  s->stats.n_loss = static_cast<int32_t>(s->loss_trace.size());
  s->stats.n_harvest = static_cast<int32_t>(s->new_unique.size());
}

void reset_solutions(sgx_sampler* s) {
  s->n_solutions = 0;
  if (s->drain) s->drain->reset();
  s->table_count = 0;
  s->epoch = 0;
  if (s->tcap) {
    CK(cudaMemsetAsync(s->tkeys.p, 0, s->tcap * sizeof(unsigned long long), s->sh));
    CK(cudaMemsetAsync(s->tmeta.p, 0xff, s->tcap * sizeof(unsigned long long), s->sh));
  }
}

}  // namespace

namespace sgx {
void set_last_error(const std::string& msg) { g_err = msg; }
}  // namespace sgx

extern "C" {

const char* sgx_last_error(void) { return g_err.c_str(); }
const char* sgx_version(void) { return "satgrad_b200 0.1 (sm_100a)"; }

int sgx_open(int device, sgx_ctx** out) {
  return guard([&] {
    need(out, "out");
    auto ctx = std::make_unique<sgx_ctx>();
    ctx->device = device;
    CK(cudaSetDevice(device));
    CK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    std::vector<uint64_t> tab(kExpTab, kExpTab + 32);
    ctx->exp_tab.upload(tab, ctx->stream);
    // Keep freed stream-ordered allocations in the pool (table / store growth).
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    CK(cudaStreamSynchronize(ctx->stream));
    *out = ctx.release();
  });
}

int sgx_close(sgx_ctx* ctx) {
  return guard([&] {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    ctx->exp_tab.reset();
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
    blockcache::flush();  // the device's cached sampler blocks back to the pool
  });
}

int sgx_layout_stats(const sgx_circuit_desc* desc, int64_t* info16) {
  return guard([&] {
    need(desc, "desc");
    need(info16, "info16");
    sgx::Layout L = sgx::build_layout(*desc);
    sgx::layout_info(L, info16);
  });
}

int sgx_harvest_clause_mask(const sgx_circuit_desc* desc, uint8_t* implied) {
  return guard([&] {
    need(desc, "desc");
    sgx::Layout L = sgx::build_layout(*desc);
    if (!L.clause_implied.empty()) {
      need(implied, "implied");
      std::copy(L.clause_implied.begin(), L.clause_implied.end(), implied);
    }
  });
}

int sgx_jit_source(const sgx_circuit_desc* desc, char* out, int64_t cap, int64_t* len) {
  return guard([&] {
    need(desc, "desc");
    need(len, "len");
    sgx::Layout L = sgx::build_layout(*desc);
    if (!sgx::jit_eligible(L)) throw std::invalid_argument("circuit is not eligible for the specialised soft pass");
    const std::string src = sgx::jit_source(L, sgx::jit_min_blocks(L));
    *len = static_cast<int64_t>(src.size()) + 1;
    if (out) {
      if (cap < *len) throw std::invalid_argument("buffer too small");
      std::memcpy(out, src.c_str(), src.size() + 1);
    }
  });
}

int sgx_sampler_soft_info(const sgx_sampler* s, int64_t* info8) {
  return guard([&] {
    need(s, "sampler");
    need(info8, "info8");
    int64_t* info4 = info8;
    const sgx::JitKernel* k = s->c->jit.get();
    info4[0] = s->last_soft;
    info4[1] = s->jit_steps;
    info4[2] = !k ? -1 : (sgx::jit_ready(k) ? 1 : (sgx::jit_failed(k) ? 2 : 0));
    info4[3] = k ? static_cast<int64_t>(sgx::jit_compile_ms(k) * 1000.0) : 0;
    info8[4] = s->hlw ? 3 : (s->hlive ? 2 : (s->hwpc ? 1 : 0));  // harvest: warp-sync live / live / full-tape smem / global
    info8[5] = s->hlw ? s->hlw : (s->hlive ? s->hlive : s->hwpc);  // its words per CTA
    info8[6] = s->vec;                            // samples per lane of the HBM soft kernels
    info8[7] = s->Bp;
  });
}

// In-process layout cache: the levelized programs of the last few circuits,
// keyed by a hash of the whole descriptor (and the environment knobs the
// layout compiler reads), so a run() on a circuit this process has already
// compiled copies its layout instead of rebuilding it (C4: ~30 ms of the
// end-to-end call on the GPU host).  SGX_NO_LAYOUT_CACHE=1 turns it off.
extern "C++" {
namespace layoutcache {
uint64_t mix(uint64_t h, uint64_t x) {
  h ^= x + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
  return h * 0xff51afd7ed558ccdull;
}
template <typename T>
uint64_t add(uint64_t h, const T* p, int64_t n) {
  h = mix(h, static_cast<uint64_t>(n));
  if (!p || n <= 0) return h;
  const size_t bytes = static_cast<size_t>(n) * sizeof(T);
  const unsigned char* c = reinterpret_cast<const unsigned char*>(p);
  size_t i = 0;
  for (; i + 8 <= bytes; i += 8) {
    uint64_t w;
    std::memcpy(&w, c + i, 8);
    h = mix(h, w);
  }
  uint64_t t = 0;
  std::memcpy(&t, c + i, bytes - i);
  return mix(h, t);
}
uint64_t key(const sgx_circuit_desc& d) {
  uint64_t h = 0x5367785f6c61796full;
  h = add(h, d.kind, d.n_nodes);
  h = add(h, d.a, d.n_nodes);
  h = add(h, d.b, d.n_nodes);
  h = add(h, d.var, d.n_nodes);
  h = mix(h, static_cast<uint64_t>(d.num_vars));
  h = add(h, d.out_var, d.n_outputs);
  h = add(h, d.out_target, d.n_outputs);
  h = add(h, d.cpi, d.n_cpi);
  h = add(h, d.ucpi, d.n_ucpi);
  h = add(h, d.clause_ptr, d.n_clauses + 1);
  h = add(h, d.clause_lit, d.clause_ptr && d.n_clauses >= 0 ? d.clause_ptr[d.n_clauses] : 0);
  for (const char* k : {"SGX_ALL_CLAUSES", "SGX_SCHED", "SGX_FWD_FAR", "SGX_BWD_KEEP", "SGX_BWD_SPLIT"}) {
    const char* v = std::getenv(k);
    h = add(h, v, v ? static_cast<int64_t>(std::strlen(v)) : 0);
  }
  return h;
}
std::mutex mu;
std::vector<std::pair<uint64_t, std::shared_ptr<const sgx::Layout>>> lru;  // most recent last
std::string dir;  // on-disk cache directory (sgx_set_layout_cache_dir / SGX_LAYOUT_CACHE_DIR), "" = none
bool on() { return !std::getenv("SGX_NO_LAYOUT_CACHE"); }
std::string disk_dir() {
  std::lock_guard<std::mutex> lk(mu);
  if (!dir.empty()) return dir;
  const char* e = std::getenv("SGX_LAYOUT_CACHE_DIR");
  return e ? std::string(e) : std::string();
}
// memory (last 4 circuits) -> disk (<dir>/<key>.sgxlayout) -> build (and save);
// *source = 0 built, 1 memory, 2 disk
sgx::Layout get(const sgx_circuit_desc& d, int* source = nullptr) {
  if (source) *source = 0;
  const std::string dd = disk_dir();
  if (!on() && dd.empty()) return sgx::build_layout(d);
  const uint64_t k = key(d);
  if (on()) {
    std::lock_guard<std::mutex> lk(mu);
    for (size_t i = 0; i < lru.size(); ++i)
      if (lru[i].first == k) {
        auto e = lru[i];
        lru.erase(lru.begin() + static_cast<long>(i));
        lru.push_back(e);
        if (source) *source = 1;
        return *e.second;
      }
  }
  std::shared_ptr<const sgx::Layout> L;
  char name[32];
  std::snprintf(name, sizeof(name), "/%016llx.sgxlayout", static_cast<unsigned long long>(k));
  if (!dd.empty()) {
    sgx::Layout x;
    if (sgx::load_layout(&x, dd + name, k)) {
      L = std::make_shared<const sgx::Layout>(std::move(x));
      if (source) *source = 2;
      if (std::getenv("SGX_TRACE")) std::fprintf(stderr, "[sgx] layout loaded from %s%s\n", dd.c_str(), name);
    }
  }
  if (!L) {
    L = std::make_shared<const sgx::Layout>(sgx::build_layout(d));
    if (!dd.empty() && !sgx::save_layout(*L, dd + name, k) && std::getenv("SGX_TRACE"))
      std::fprintf(stderr, "[sgx] layout not saved to %s%s\n", dd.c_str(), name);
  }
  if (on()) {
    std::lock_guard<std::mutex> lk(mu);
    lru.emplace_back(k, L);
    if (lru.size() > 4) lru.erase(lru.begin());
  }
  return *L;
}
}  // namespace layoutcache
}  // extern "C++"

int sgx_layout_digest(const sgx_circuit_desc* desc, uint64_t* digest, int32_t* source) {
  return guard([&] {
    need(desc, "desc");
    need(digest, "digest");
    int src = 0;
    const sgx::Layout L = layoutcache::get(*desc, &src);
    *digest = sgx::layout_digest(L);
    if (source) *source = src;
  });
}

int sgx_jit_quiesce(void) {
  return guard([&] { sgx::jit_quiesce(); });
}

int sgx_set_layout_cache_dir(const char* dir) {
  return guard([&] {
    std::lock_guard<std::mutex> lk(layoutcache::mu);
    layoutcache::dir = dir ? std::string(dir) : std::string();
  });
}

int sgx_circuit_upload(sgx_ctx* ctx, const sgx_circuit_desc* d, sgx_circuit** out) {
  return guard([&] {
    need(ctx, "ctx");
    need(d, "desc");
    need(out, "out");
    CK(cudaSetDevice(ctx->device));
    auto c = std::make_unique<sgx_circuit>();
    c->ctx = ctx;
    if (d->unsat) {
      // run() returns before touching the circuit (sampler.cpp:105-110).
      try {
        c->L = sgx::build_layout(*d);
        c->layout_ok = true;
      } catch (const std::invalid_argument&) {
        c->L = sgx::Layout{};
        c->L.unsat = true;
        c->L.num_vars = d->num_vars;
        c->L.key_words = (d->num_vars + 63) / 64;
      }
    } else {
      c->L = layoutcache::get(*d);
      c->layout_ok = true;
    }
    if (c->layout_ok) {
      cudaStream_t st = ctx->stream;
      const auto& L = c->L;
      c->cone.upload(L.cone, st);
      c->bit_ops.upload(to_int4(L.bit_ops), st);
      c->bit_lvl_ptr.upload(L.bit_lvl_ptr, st);
      c->n_bit_levels = static_cast<int>(L.bit_lvl_ptr.size()) - 1;
      c->cpi_bit_row.upload(L.cpi_bit_row, st);
      c->ucpi_bit_row.upload(L.ucpi_bit_row, st);
      c->out_bit_row.upload(L.out_bit_row, st);
      c->out_tgt.upload(L.out_tgt, st);
      c->clause_ptr.upload(L.clause_ptr32, st);
      c->clause_enc.upload(L.clause_enc, st);
      c->key_bit_row.upload(L.key_bit_row, st);
      c->fb_ops.upload(to_int4(L.fb_ops), st);
      c->fb_lvl_ptr.upload(L.fb_lvl_ptr, st);
      c->fb_levels = static_cast<int>(L.fb_lvl_ptr.size()) - 1;
      c->fb_cpi_row.upload(L.fb_cpi_row, st);
      c->fb_ucpi_row.upload(L.fb_ucpi_row, st);
      c->fb_out_enc.upload(L.fb_out_enc, st);
      c->fb_key_enc.upload(L.fb_key_enc, st);
      c->fb_cnf4.upload(to_int4(L.fb_cnf4), st);
      c->lb_ops.upload(to_int4(L.lb_ops), st);
      c->lw_ops.upload(to_int4(L.lw_ops), st);
      c->lb_chk.upload(to_int4(L.lb_chk), st);
      c->lb_op_ptr.upload(L.lb_op_ptr, st);
      c->lb_chk_ptr.upload(L.lb_chk_ptr, st);
      c->lb_big.upload(L.lb_big_lits.empty() ? std::vector<int32_t>{0} : L.lb_big_lits, st);
      c->lb_key_enc.upload(L.lb_key_enc, st);
      c->lb_cpi.upload(to_int2(L.lb_cpi), st);
      c->lb_ucpi.upload(to_int2(L.lb_ucpi), st);
      CK(cudaStreamSynchronize(st));
    }
    *out = c.release();
  });
}

int sgx_circuit_info(const sgx_circuit* c, int64_t* info16) {
  return guard([&] {
    need(c, "circuit");
    need(info16, "info16");
    sgx::layout_info(c->L, info16);
  });
}

int sgx_circuit_free(sgx_circuit* c) {
  return guard([&] {
    if (!c) return;
    cudaSetDevice(c->ctx->device);
    delete c;
  });
}

int sgx_sampler_create(sgx_circuit* c, const sgx_sampler_cfg* cfg, sgx_sampler** out) {
  const auto t_create = std::chrono::steady_clock::now();
  return guard([&] {
    need(c, "circuit");
    need(cfg, "cfg");
    need(out, "out");
    if (cfg->batch < 1) throw std::invalid_argument("batch must be positive");  // sampler.cpp:93
    if (cfg->iterations < 0) throw std::invalid_argument("iterations must be non-negative");
    if (cfg->restart_policy < SGX_RESTART_NONE || cfg->restart_policy > SGX_RESTART_REINIT_INVALID)
      throw std::invalid_argument("unknown restart policy");
    if (cfg->reinit_age < 0 || cfg->reinit_age > 255) throw std::invalid_argument("reinit_age must be in [0, 255]");
    if (cfg->optimizer != SGX_OPT_GD && cfg->optimizer != SGX_OPT_ADAM) throw std::invalid_argument("unknown optimizer");
    if (cfg->optimizer == SGX_OPT_ADAM &&
        (cfg->adam_beta1 < 0 || cfg->adam_beta1 >= 1 || cfg->adam_beta2 < 0 || cfg->adam_beta2 >= 1 || cfg->adam_eps < 0))
      throw std::invalid_argument("Adam needs 0 <= beta1, beta2 < 1 and eps >= 0");
    CK(cudaSetDevice(c->ctx->device));
    auto s = std::make_unique<sgx_sampler>();
    s->c = c;
    s->cfg = *cfg;
    // The soft passes (st) outrank the harvest (sh) at the block scheduler:
    // the harvest has a whole iteration of slack (double-buffered input).
    // Measured with the warp-synchronous harvest: C4 +2-3 %, C2 even.  Not
    // for circuits the specialised soft pass runs (its step fills every SM,
    // so a lower-priority harvest waits for it: C3a -3 %, C3b -1 %).
    // SGX_PRIO=0 / 1: equal / prioritised always.
    int prio_lo = 0, prio_hi = 0;
    CK(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    const char* pe = std::getenv("SGX_PRIO");
    const char* je = std::getenv("SGX_JIT");
    const bool jit_circuit = c->layout_ok && !c->L.unsat && cfg->soft_kernel != SGX_SOFT_HBM &&
                             !(je && je[0] == '0') && sgx::jit_eligible(c->L);
    const bool prio = pe ? pe[0] == '1' : !jit_circuit;
    {
      StreamKit k = kit_take(c->ctx->device, prio, prio_lo, prio_hi);
      s->kit_prio = prio;
      s->st = k.st;
      s->sh = k.sh;
      std::copy(k.ev, k.ev + 8, s->ev);
      for (int p = 0; p < 2; ++p) std::copy(k.sev[p], k.sev[p] + 4, s->sev[p]);
      std::copy(k.run, k.run + 4, s->rev);
      s->ev_soft = k.soft;
      s->ev_front = k.front;
      s->ev_join = k.join;
    }
    // From here on a failure (e.g. out of memory for the tape) must hand the
    // stream kit, the pinned slots and every buffer back: sgx_sampler_free
    // does exactly that on the half-built sampler.
    try {
      // The kit's events may carry its previous owner's completed records: a
      // wait on them is a no-op, and sgx_step_loss only reads the slots this
      // sampler launched (slot_pending).
      s->dloss.alloc_async(2, s->st);  // pool memory: freed without cudaFree's device sync
      static_assert(sizeof(sgx::HarvestOut) <= kPinSlot, "pinned slot too small");
      s->hloss = static_cast<double*>(pin_slot());
      s->hpin = static_cast<sgx::HarvestOut*>(pin_slot());
      std::memset(s->hpin, 0, sizeof(sgx::HarvestOut));
      s->hout.alloc_async(1, s->st);
      CK(cudaStreamSynchronize(s->st));
      const auto t_head = std::chrono::steady_clock::now();
      if (c->layout_ok && !c->L.unsat) {
        const auto& L = c->L;
        s->Bp = round_up(cfg->batch, 1024);
        s->W = s->Bp / 32;
        s->wpc = s->W / 32 >= 2 * 148 ? 32 : (s->W / 16 >= 2 * 148 ? 16 : 8);
        // Widest samples-per-thread that still leaves >= 3 tiles per SM
        // (SGX_VEC overrides, for tuning).
        s->vec = s->Bp / 128 >= 3 * 148 ? 4 : (s->Bp / 64 >= 3 * 148 ? 2 : 1);
        if (const char* e = std::getenv("SGX_VEC")) {
          int v = std::atoi(e);
          if (v == 1 || v == 2 || v == 4) s->vec = v;
        }
        // SGX_ONCHIP=1: small circuits (>= 2 tiles of tape + adjoint slots per
        // SM) run the fused on-chip soft pass on 32-sample tiles.  Opt-in:
        // measured on C3a it is 2.3x SLOWER than the HBM-tape kernels (one
        // sample per lane spends ~23k warp instructions per 32-sample tile on
        // record control, at 8 warps per SM).
        {
          const char* e = std::getenv("SGX_ONCHIP");
          s->onchip = e && e[0] == '1' && cfg->optimizer == SGX_OPT_GD && c->cone.oc_n4 > 0 &&
                      sgx::onchip_warps(c->cone.n_rows, c->cone.oc_slots, c->cone.oc_n4) >= 2;
          if (s->onchip) s->vec = 1;
        }
        // Circuit-specialised soft pass (sgx_jit.hpp) for small cones.
        {
          int mode = cfg->soft_kernel;
          if (const char* e = std::getenv("SGX_JIT")) {
            if (e[0] == '0') mode = SGX_SOFT_HBM;
            else if (e[0] == 's') mode = SGX_SOFT_JIT;
          }
          if (cfg->optimizer == SGX_OPT_ADAM) mode = SGX_SOFT_HBM;  // Adam runs the HBM kernels' dV tap
        if (mode != SGX_SOFT_HBM && !s->onchip && sgx::jit_eligible(L)) {
            if (!c->jit) c->jit = sgx::jit_get(L, mode != SGX_SOFT_JIT);
            if (mode == SGX_SOFT_JIT) sgx::jit_wait(c->jit.get());
            if (!sgx::jit_failed(c->jit.get())) s->jit = c->jit.get();
          }
        }
        // Shared-memory harvest: the widest word block whose folded bit tape
        // fits ~100 KB (two CTAs per SM) while leaving >= 2 CTAs per SM of work;
        // one word (up to 200 KB) for deep circuits; else the global path.
        const size_t row_bytes = static_cast<size_t>(L.fb_rows + 1) * sizeof(uint32_t);
        s->hwpc = 0;
        // (<= 8 words: the CNF check keeps one accumulator pair per word in
        // registers)
        for (int w = 8; w >= 1; w /= 2)
          if (row_bytes * w <= 100 * 1024 && s->W / w >= 2 * 148) {
            s->hwpc = w;
            break;
          }
        if (!s->hwpc && row_bytes <= 200 * 1024) s->hwpc = 1;
        if (const char* e = std::getenv("SGX_HARVEST")) {
          if (e[0] == 'g') s->hwpc = 0;  // force the global-memory harvest
        }
        if (const char* e = std::getenv("SGX_HWPC")) {  // A/B: words per harvest CTA
          const int w = std::atoi(e);
          if ((w == 1 || w == 2 || w == 4 || w == 8) && row_bytes * w <= 220 * 1024) s->hwpc = w;
        }
        // Liveness-allocated harvest (default): the words per CTA that keep the
        // most words resident per SM (8 CTAs of 256 threads at most, ~227 KB of
        // shared memory) with at least one CTA per SM; ties go to more words per
        // CTA (per-level overhead amortised).  SGX_HARVEST=smem / g force the
        // full-tape shared-memory / global-memory harvests.
        s->hlive = 0;
        {
          const char* e = std::getenv("SGX_HARVEST");
          const bool live_ok = !(e && (e[0] == 'g' || e[0] == 's'));
          // words resident per SM for a tape of `rows` rows per word
          auto best = [&](long long rows, int* wpc) {
            int words = 0;
            for (int w = 1; w <= 8; w *= 2) {
              const size_t smem = static_cast<size_t>(rows) * w * sizeof(uint32_t) + 3 * 1024;
              if (smem > 200 * 1024 || s->W / w < 148) continue;
              const int ctas = std::min<int>(8, static_cast<int>((227 * 1024) / (smem + 1024)));
              if (ctas * w >= words) {
                words = ctas * w;
                *wpc = w;
              }
            }
            return words;
          };
          int wl = 0, wf = 0;
          const int live_words = live_ok ? best(L.lb_slots, &wl) : 0;
          const int full_words = best(L.fb_rows + 1, &wf);
          // The full tape needs no spill round trip for the keys: it wins ties.
          if (live_words > full_words) s->hlive = wl;
          if (const char* v = std::getenv("SGX_LWPC")) {  // A/B: words per live-harvest CTA
            const int w = std::atoi(v);
            if ((w == 1 || w == 2 || w == 4 || w == 8) && live_ok &&
                static_cast<size_t>(L.lb_slots) * w * 4 <= 200 * 1024)
              s->hlive = w;
          }
          if (s->hlive) s->hwpc = 0;
          // Warp-synchronous cut of the live program: one warp per word, as
          // many words per CTA as fit ~227 KB (<= 8).  SGX_HARVEST=live keeps
          // the CTA-synchronous kernel; SGX_HARVEST=lw selects this one even
          // where the full tape would win.
          s->hlw = 0;
          const size_t per_warp = static_cast<size_t>(L.lb_slots + 1) * sizeof(uint32_t);
          const int lw_fit = static_cast<int>(std::min<size_t>(8, (226 * 1024 - sgx::kLwRingBytes) / per_warp));
          const bool want_lw = e && std::string(e) == "lw";
          const bool cta_live = (e && std::string(e) == "live") || std::getenv("SGX_LWPC");
          if (lw_fit >= 1 && (s->hlive || want_lw) && !cta_live) {
            s->hlw = lw_fit;
            if (!s->hlive) s->hlive = 1;
            s->hwpc = 0;
          }
          if (const char* v = std::getenv("SGX_LWW")) {  // A/B: warps (words) per warp-synchronous CTA
            const int k = std::atoi(v);
            if (s->hlw && k >= 1 && k <= lw_fit) s->hlw = k;
          }
        }
        // Stream-ordered pool allocations: a sampler created after another one
        // reuses its memory without cudaMalloc / cudaFree round trips.
        const size_t Bp = static_cast<size_t>(s->Bp);
        cudaStream_t st = s->st;
        s->V.alloc_async(L.cpi.size() * Bp, st);
        s->HB.alloc_async(2 * L.cpi.size() * s->W, st);
        // The on-chip and the (compiled) JIT passes keep tape and adjoints on chip.
        if (!s->onchip && !(s->jit && sgx::jit_ready(s->jit))) {
          s->tape.alloc_async(static_cast<size_t>(L.cone.n_rows) * Bp, st);
          s->adj.alloc_async(static_cast<size_t>(L.cone.n_rows) * Bp, st);
          s->have_tape = true;
        }
        if (cfg->optimizer == SGX_OPT_ADAM) {
          for (auto* b : {&s->adam_dv, &s->adam_dp, &s->adam_m, &s->adam_v}) b->alloc_async(L.cpi.size() * Bp, st);
          CK(cudaMemsetAsync(s->adam_m.p, 0, s->adam_m.n * sizeof(float), st));
          CK(cudaMemsetAsync(s->adam_v.p, 0, s->adam_v.n * sizeof(float), st));
        }
        s->row_loss.alloc_async(Bp, st);
        s->partial.alloc_async(s->n_partial, st);
        if (!s->hwpc && !s->hlive) s->BT.alloc_async(static_cast<size_t>(L.n_bit_rows) * s->W, st);
        if (s->hlive) s->SP.alloc_async(static_cast<size_t>(std::max(L.lb_n_spill, 1)) * s->W, st);
        s->valid.alloc_async(s->W, st);
        s->newmask.alloc_async(s->W, st);
        if (cfg->restart_policy == SGX_RESTART_REINIT_ROWS || cfg->restart_policy == SGX_RESTART_REINIT_INVALID) {
          s->row_age.alloc_async(Bp, st);
          s->redraw.alloc_async(2 * static_cast<size_t>(s->W), st);  // one per harvest parity (lagged schedule)
        }
        s->slot_of_row.alloc_async(Bp, st);
        s->block_count.alloc_async(Bp / sgx::kThreads, st);
        s->K.alloc_async(static_cast<size_t>(L.key_words) * Bp, st);
        // Room for every row the run can harvest (restarts x (iterations + 1)
        // batches, + 2 for the growth trigger) when that fits 48 GB and a
        // third of the free device memory, else the old floor (16 harvests,
        // at most 4 GB): a growth waits for the host drain, copies the store
        // and allocates from the pool mid-run (C4: up to 1.7 s of fresh
        // mappings on a first run).  A quota caps it.
        const long long key_bytes = static_cast<long long>(L.key_words) * 8;
        long long want_rows = 16 * static_cast<long long>(Bp);
        const long long cap_4g = (4ll << 30) / key_bytes;
        want_rows = std::max<long long>(std::min(want_rows, cap_4g), 2 * static_cast<long long>(Bp));
        {
          const bool restarts = cfg->restart_policy != SGX_RESTART_NONE;
          const long long n_restarts = restarts ? (cfg->max_restarts > 0 ? cfg->max_restarts : 1000) + 1 : 1;
          const long long bound = (n_restarts * (static_cast<long long>(cfg->iterations) + 1) + 2) * Bp;
          size_t fr = 0, tot = 0;
          if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) {
            cudaGetLastError();
            fr = 0;
          }
          {  // blocks the cache holds are as good as free
            int dev = 0;
            cudaGetDevice(&dev);
            std::lock_guard<std::mutex> lk(blockcache::mu);
            fr += blockcache::held_bytes[dev];
          }
          const long long roomy = std::min<long long>((48ll << 30), static_cast<long long>(fr / 3)) / key_bytes;
          if (bound <= roomy) want_rows = std::max(want_rows, bound);
        }
        if (cfg->max_solutions > 0) want_rows = std::min<long long>(want_rows, cfg->max_solutions + Bp);
        s->store_cap = cfg->solution_capacity > 0 ? cfg->solution_capacity : want_rows;
        s->store.alloc_async(static_cast<size_t>(s->store_cap) * L.key_words, st);
        CK(cudaMemsetAsync(s->V.p, 0, s->V.n * sizeof(float), s->st));
        CK(cudaMemsetAsync(s->HB.p, 0xff, s->HB.n * sizeof(uint32_t), s->st));  // harden(0) = 1
        const auto ta = std::chrono::steady_clock::now();
        const double t_alloc = std::chrono::duration<double, std::milli>(ta - t_head).count();
        const double t_front = std::chrono::duration<double, std::milli>(t_head - t_create).count();
        ensure_table(s.get());
        const auto tb = std::chrono::steady_clock::now();
        CK(cudaStreamSynchronize(s->st));
        CK(cudaStreamSynchronize(s->sh));
        if (std::getenv("SGX_TRACE")) {
          const auto tc = std::chrono::steady_clock::now();
          std::fprintf(stderr, "[sgx] sampler create: %.2f ms (streams + first sync %.2f, buffers %.2f, table %.2f ms, allocation / memset sync %.2f ms, store %.2f GB)\n",
                       std::chrono::duration<double, std::milli>(tc - t_create).count(), t_front, t_alloc,
                       std::chrono::duration<double, std::milli>(tb - ta).count(),
                       std::chrono::duration<double, std::milli>(tc - tb).count(),
                       s->store_cap * L.key_words * 8.0 / 1e9);
        }
      }
    } catch (...) {
      sgx_sampler_free(s.release());
      throw;
    }
    *out = s.release();
  });
}

int sgx_sampler_free(sgx_sampler* s) {
  return guard([&] {
    if (!s) return;
    const auto t0 = std::chrono::steady_clock::now();
    auto ms = [&] { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(); };
    cudaSetDevice(s->c->ctx->device);
    cudaStream_t st = s->st;
    if (s->sh) cudaStreamSynchronize(s->sh);  // no harvest work left
    const double t_sync = ms();
    s->drain.reset();                          // no host copy left reading the store
    const double t_drain = ms();
    if (st) cudaStreamSynchronize(st);
    const double t_sync2 = ms();
    if (st) {  // quiescent: big buffers go to the block cache, the rest back to the pool
      for (auto* b : {&s->V, &s->tape, &s->adj, &s->row_loss, &s->adam_dv, &s->adam_dp, &s->adam_m, &s->adam_v})
        b->reset();
      s->partial.reset();
      for (auto* b : {&s->BT, &s->valid, &s->newmask, &s->HB, &s->SP}) b->reset();
      s->fps_local.reset();
      s->fps_all.reset();
      s->n_of.reset();
      s->slot_of_row.reset();
      s->block_count.reset();
      s->K.reset();
      s->store.reset();
      s->tkeys.reset();
      s->tmeta.reset();
    }
    const double t_reset = ms();
    StreamKit k;
    k.device = s->c->ctx->device;
    k.prio = s->kit_prio;
    k.st = s->st;
    k.sh = s->sh;
    std::copy(s->ev, s->ev + 8, k.ev);
    for (int p = 0; p < 2; ++p) std::copy(s->sev[p], s->sev[p] + 4, k.sev[p]);
    std::copy(s->rev, s->rev + 4, k.run);
    k.soft = s->ev_soft;
    k.front = s->ev_front;
    k.join = s->ev_join;
    pin_release(s->hpin);  // (the streams were synchronised above)
    pin_release(s->hloss);
    delete s;
    if (k.st && k.sh) kit_give(k);  // both streams idle: every event has completed
    else kit_destroy(k);
    if (std::getenv("SGX_TRACE"))
      std::fprintf(stderr, "[sgx] sampler free: harvest sync %.2f, drain %.2f, frees %.2f, stream sync %.2f, total %.2f ms\n",
                   t_sync, t_drain, t_reset, t_sync2, ms());
  });
}

static void need_ready(sgx_sampler* s) {
  need(s, "sampler");
  if (!s->c->layout_ok || s->c->L.unsat) throw StateError("instance is unsatisfiable by construction");
}

int sgx_init(sgx_sampler* s, int32_t restart) {
  return guard([&] {
    need_ready(s);
    CK(cudaSetDevice(s->c->ctx->device));
    sampler_init(s, restart);
    CK(cudaStreamSynchronize(s->st));
  });
}

int sgx_step(sgx_sampler* s, double* loss_total) {
  return guard([&] {
    need_ready(s);
    CK(cudaSetDevice(s->c->ctx->device));
    const int slot = sampler_step(s);
    double loss = 0.0;
    CK(cudaMemcpyAsync(&loss, s->dloss.p + slot, sizeof(double), cudaMemcpyDeviceToHost, s->st));
    CK(cudaStreamSynchronize(s->st));
    if (loss_total) *loss_total = loss;
  });
}

int sgx_step_async(sgx_sampler* s, int32_t* slot) {
  return guard([&] {
    need_ready(s);
    need(slot, "slot");
    CK(cudaSetDevice(s->c->ctx->device));
    *slot = sampler_step(s);
  });
}

int sgx_step_loss(sgx_sampler* s, int32_t slot, double* loss_total) {
  return guard([&] {
    need_ready(s);
    if (slot != 0 && slot != 1) throw std::invalid_argument("step slot must be 0 or 1");
    // Pooled stream kits hand over events the previous owner recorded: only a
    // slot this sampler launched (and has not read yet) carries its step.
    if (!s->slot_pending[slot]) throw StateError("sgx_step_loss: no step pending in this slot");
    s->slot_pending[slot] = false;
    CK(cudaSetDevice(s->c->ctx->device));
    CK(cudaEventSynchronize(s->sev[slot][3]));
    if (loss_total) *loss_total = s->hloss[slot];
    cudaEvent_t* ev = s->sev[slot];  // device time of the step (sgx_phase_times)
    s->phase_ms[1] += elapsed(ev[0], ev[3]);
    s->phase_ms[3] += elapsed(ev[0], ev[1]);
    s->phase_ms[4] += elapsed(ev[2], ev[3]);
  });
}

int64_t sgx_launch_count(const sgx_sampler* s) { return s ? s->launches : -1; }

int sgx_harvest(sgx_sampler* s, int32_t restart, int32_t iter, int64_t* attempts, int64_t* added) {
  return guard([&] {
    need_ready(s);
    CK(cudaSetDevice(s->c->ctx->device));
    long long quota_left = s->cfg.max_solutions > 0 ? s->cfg.max_solutions - s->n_solutions : -1;
    if (quota_left == 0) {
      if (attempts) *attempts = 0;
      if (added) *added = 0;
      return;
    }
    long long att = 0, add = 0;
    sampler_harvest(s, restart, iter, quota_left, &att, &add, -1);
    if (attempts) *attempts = att;
    if (added) *added = add;
  });
}

int sgx_run(sgx_sampler* s, sgx_run_stats* stats) {
  return guard([&] {
    need(s, "sampler");
    CK(cudaSetDevice(s->c->ctx->device));
    if (s->c->layout_ok && !s->c->L.unsat) {
      reset_solutions(s);
    } else {
      s->n_solutions = 0;
      if (s->drain) s->drain->reset();
    }
    sampler_run(s);
    if (stats) *stats = s->stats;
  });
}

int sgx_run_traces(sgx_sampler* s, double* loss_trace, int64_t* new_unique) {
  return guard([&] {
    need(s, "sampler");
    if (loss_trace && !s->loss_trace.empty())
      std::memcpy(loss_trace, s->loss_trace.data(), s->loss_trace.size() * sizeof(double));
    if (new_unique && !s->new_unique.empty())
      std::memcpy(new_unique, s->new_unique.data(), s->new_unique.size() * sizeof(int64_t));
  });
}

int64_t sgx_solution_count(const sgx_sampler* s) { return s ? s->n_solutions : -1; }

int32_t sgx_key_words(const sgx_sampler* s) { return s ? s->c->L.key_words : -1; }

int sgx_fetch_solutions(sgx_sampler* s, int64_t first, int64_t count, uint64_t* keys) {
  return guard([&] {
    need(s, "sampler");
    if (first < 0 || count < 0 || first + count > s->n_solutions)
      throw std::invalid_argument("solution range out of bounds");
    if (count == 0) return;
    need(keys, "keys");
    CK(cudaSetDevice(s->c->ctx->device));
    const size_t kw = static_cast<size_t>(s->c->L.key_words);
    CK(cudaMemcpyAsync(keys, s->store.p + static_cast<size_t>(first) * kw,
                       static_cast<size_t>(count) * kw * sizeof(uint64_t), cudaMemcpyDeviceToHost, s->sh));
    CK(cudaStreamSynchronize(s->sh));
  });
}

int sgx_set_host_stream(sgx_sampler* s, int32_t on) {
  return guard([&] {
    need(s, "sampler");
    CK(cudaSetDevice(s->c->ctx->device));
    if (!on) {
      s->drain.reset();
    } else if (!s->drain) {
      if (s->n_solutions) throw StateError("sgx_set_host_stream: enable before the run");
      s->drain = std::make_unique<sgx::HostDrain>(s->c->ctx->device, s->c->L.key_words);
    }
  });
}

int sgx_solutions_take(sgx_sampler* s, uint64_t** keys, int64_t* rows, int64_t* map_bytes) {
  return guard([&] {
    need(s, "sampler");
    need(keys, "keys");
    CK(cudaSetDevice(s->c->ctx->device));
    const size_t kw = static_cast<size_t>(s->c->L.key_words);
    *keys = nullptr;
    *rows = 0;
    *map_bytes = 0;
    if (s->n_solutions == 0) return;
    if (s->drain && s->drain->queued() == s->n_solutions) {
      int64_t r = 0;
      size_t b = 0;
      uint64_t* p = s->drain->take(&r, &b);
      if (r != s->n_solutions) {
        sgx::host_free(p, b);
        throw CudaError("host drain lost rows");
      }
      *keys = p;
      *rows = r;
      *map_bytes = static_cast<int64_t>(b);
      return;
    }
    const size_t need_bytes = static_cast<size_t>(s->n_solutions) * kw * sizeof(uint64_t);
    size_t bytes = 0;
    void* p = sgx::host_map(need_bytes, &bytes);
    const cudaError_t e = cudaMemcpyAsync(p, s->store.p, need_bytes, cudaMemcpyDeviceToHost, s->sh);
    const cudaError_t e2 = e == cudaSuccess ? cudaStreamSynchronize(s->sh) : e;
    if (e2 != cudaSuccess) {
      sgx::host_free(p, bytes);
      CK(e2);
    }
    *keys = static_cast<uint64_t*>(p);
    *rows = s->n_solutions;
    *map_bytes = static_cast<int64_t>(bytes);
  });
}

int sgx_host_free(uint64_t* keys, int64_t map_bytes) {
  return guard([&] { sgx::host_free(keys, static_cast<size_t>(map_bytes)); });
}

int sgx_verify_solutions(sgx_circuit* c, const char* text, int64_t len, int64_t* out) {
  return guard([&] {
    need(c, "circuit");
    need(out, "out");
    if (len < 0) throw std::invalid_argument("negative text length");
    if (len > 0) need(text, "text");
    sgx::VerifyResult r;
    sgx::verify_solutions(c->ctx->device, c->L.clause_ptr, c->L.clause_lit, c->L.num_vars, text, len, &r);
    out[0] = r.checked;
    out[1] = r.err_line;
    out[2] = r.err_var;
    out[3] = r.err_kind;
    out[4] = r.launches;
  });
}

int sgx_verify_keys(sgx_circuit* c, const uint64_t* keys, int64_t n, int64_t* out) {
  return guard([&] {
    need(c, "circuit");
    need(out, "out");
    if (n < 0) throw std::invalid_argument("negative key count");
    if (n > 0) need(keys, "keys");
    sgx::KeyCheck r;
    sgx::verify_keys(c->ctx->device, c->L.clause_ptr, c->L.clause_lit, c->L.num_vars, keys, n, &r);
    out[0] = r.checked;
    out[1] = r.unsat;
    out[2] = r.malformed;
    out[3] = r.duplicate;
    out[4] = r.launches;
  });
}

int sgx_verify_cnf(sgx_ctx* ctx, int32_t num_vars, const int64_t* clause_ptr, const int32_t* clause_lit,
                   int64_t n_clauses, const char* text, int64_t len, int64_t* out) {
  return guard([&] {
    need(ctx, "context");
    need(out, "out");
    if (num_vars < 0 || n_clauses < 0 || len < 0) throw std::invalid_argument("negative size");
    if (len > 0) need(text, "text");
    std::vector<int64_t> ptr{0};
    std::vector<int32_t> lit;
    if (n_clauses > 0) {
      need(clause_ptr, "clause_ptr");
      need(clause_lit, "clause_lit");
      ptr.assign(clause_ptr, clause_ptr + n_clauses + 1);
      if (ptr[0] != 0) throw std::invalid_argument("clause_ptr[0] must be 0");
      for (int64_t c = 0; c < n_clauses; ++c)
        if (ptr[c + 1] < ptr[c]) throw std::invalid_argument("clause_ptr not monotone");
      lit.assign(clause_lit, clause_lit + ptr[n_clauses]);
      for (int32_t l : lit)
        if (l == 0 || l > num_vars || -l > num_vars) throw std::invalid_argument("literal out of range");
    }
    sgx::VerifyResult r;
    sgx::verify_solutions(ctx->device, ptr, lit, num_vars, text, len, &r);
    out[0] = r.checked;
    out[1] = r.err_line;
    out[2] = r.err_var;
    out[3] = r.err_kind;
    out[4] = r.launches;
  });
}

int sgx_format_solutions(sgx_sampler* s, int64_t first, int64_t count, char* out, int64_t cap, int64_t* len) {
  return guard([&] {
    need(s, "sampler");
    need(len, "len");
    if (first < 0 || count < 0 || first + count > s->n_solutions)
      throw std::invalid_argument("solution range out of bounds");
    *len = 0;
    if (count == 0) return;
    CK(cudaSetDevice(s->c->ctx->device));
    const int kw = s->c->L.key_words, nv = s->c->L.num_vars;
    cudaStream_t st = s->sh;  // the store belongs to the harvest stream
    DBuf<long long> lo;
    lo.alloc_async(static_cast<size_t>(count) + 1, st);
    size_t scratch_bytes = 0;
    sgx::launch_fmt_lengths(st, s->store.p, first, count, kw, nv, lo.p, nullptr, &scratch_bytes);
    DBuf<unsigned char> scratch;
    scratch.alloc_async(std::max<size_t>(scratch_bytes, 1), st);
    sgx::launch_fmt_lengths(st, s->store.p, first, count, kw, nv, lo.p, scratch.p, &scratch_bytes);
    std::vector<long long> off(static_cast<size_t>(count) + 1);
    CK(cudaMemcpyAsync(off.data(), lo.p, off.size() * sizeof(long long), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    *len = off[count];
    if (!out) {
      scratch.reset_async(st);
      lo.reset_async(st);
      return;
    }
    if (cap < off[count]) throw std::invalid_argument("format_solutions: output buffer too small");
    // Render in chunks of at most 256 MB of text (a single longer line gets its own chunk).
    const long long chunk = 256ll << 20;
    long long longest = 0;
    for (long long i = 0; i < count; ++i) longest = std::max(longest, off[i + 1] - off[i]);
    DBuf<char> buf;
    buf.alloc_async(static_cast<size_t>(std::max(std::min(chunk, off[count]), longest)), st);
    for (long long i = 0; i < count;) {
      long long j = i + 1;
      while (j < count && off[j + 1] - off[i] <= static_cast<long long>(buf.n)) ++j;
      sgx::launch_fmt_write(st, s->store.p, first + i, j - i, kw, nv, lo.p + i, off[i], buf.p);
      CK(cudaGetLastError());
      CK(cudaMemcpyAsync(out + off[i], buf.p, static_cast<size_t>(off[j] - off[i]), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      i = j;
    }
    buf.reset_async(st);
    scratch.reset_async(st);
    lo.reset_async(st);
  });
}

int sgx_phase_times(const sgx_sampler* s, double* ms8) {
  return guard([&] {
    need(s, "sampler");
    need(ms8, "ms8");
    std::memcpy(ms8, s->phase_ms, sizeof(s->phase_ms));
  });
}

int sgx_read_logits(sgx_sampler* s, float* v) {
  return guard([&] {
    need_ready(s);
    const size_t ncpi = s->c->L.cpi.size();
    if (!ncpi) return;
    need(v, "v");
    CK(cudaSetDevice(s->c->ctx->device));
    std::vector<float> h(ncpi * s->Bp);
    CK(cudaMemcpyAsync(h.data(), s->V.p, h.size() * sizeof(float), cudaMemcpyDeviceToHost, s->st));
    CK(cudaStreamSynchronize(s->st));
    const int tile = 32 * s->vec;
    for (int r = 0; r < s->cfg.batch; ++r)
      for (size_t j = 0; j < ncpi; ++j)
        v[static_cast<size_t>(r) * ncpi + j] = h[(static_cast<size_t>(r / tile) * ncpi + j) * tile + r % tile];
  });
}

// ------------------------------------------------------- multi-GPU harvest
int sgx_fingerprint_stride(const sgx_sampler* s) { return s ? s->Bp : -1; }

int sgx_harvest_local(sgx_sampler* s, int32_t restart, int32_t iter, int64_t* n_new, uint64_t** fps) {
  return guard([&] {
    need_ready(s);
    CK(cudaSetDevice(s->c->ctx->device));
    const long long n = dist_local(s, restart, iter);
    if (n_new) *n_new = n;
    if (fps) *fps = reinterpret_cast<uint64_t*>(s->fps_local.p);
  });
}

int sgx_harvest_merge(sgx_sampler* s, const uint64_t* all_fps, const int64_t* counts, int32_t nranks,
                      int32_t rank, int64_t stride, int64_t* n_won) {
  return guard([&] {
    need_ready(s);
    if (nranks < 1 || rank < 0 || rank >= nranks) throw std::invalid_argument("bad rank / nranks");
    if (nranks > 1) {
      need(all_fps, "all_fps");
      need(counts, "counts");
    }
    CK(cudaSetDevice(s->c->ctx->device));
    std::vector<long long> cnt(nranks, 0);
    for (int r = 0; r < nranks; ++r) cnt[r] = counts ? counts[r] : (r == rank ? s->hpin->new_rows : 0);
    long long fresh = 0;
    const long long won = dist_merge(s, all_fps, cnt, rank, stride, &fresh);
    if (n_won) *n_won = won;
  });
}

int sgx_harvest_commit(sgx_sampler* s, int64_t quota_left, int64_t* attempts, int64_t* added) {
  return guard([&] {
    need_ready(s);
    CK(cudaSetDevice(s->c->ctx->device));
    long long att = 0, add = 0;
    dist_commit(s, quota_left, &att, &add);
    if (attempts) *attempts = att;
    if (added) *added = add;
  });
}

int sgx_run_local_added(const sgx_sampler* s, int64_t* added) {
  return guard([&] {
    need(s, "sampler");
    need(added, "added");
    std::copy(s->local_added.begin(), s->local_added.end(), added);
  });
}

int sgx_run_sharded(sgx_sampler* s, const sgx_exchange* ex, sgx_run_stats* stats) {
  return guard([&] {
    need(s, "sampler");
    need(ex, "exchange");
    if (ex->nranks < 1 || ex->rank < 0 || ex->rank >= ex->nranks) throw std::invalid_argument("bad rank / nranks");
    if (!ex->allgather_device || !ex->allgather_host) throw std::invalid_argument("exchange without collectives");
    if (s->cfg.restart_policy == SGX_RESTART_REINIT_ROWS || s->cfg.restart_policy == SGX_RESTART_REINIT_INVALID)
      throw std::invalid_argument("SGX_RESTART_REINIT_ROWS / REINIT_INVALID are single-device only (sgx_run)");
    CK(cudaSetDevice(s->c->ctx->device));
    if (s->c->layout_ok && !s->c->L.unsat) {
      reset_solutions(s);
    } else {
      s->n_solutions = 0;
      if (s->drain) s->drain->reset();
    }
    sampler_run_sharded(s, ex);
    if (stats) *stats = s->stats;
  });
}

// ------------------------------------------------------------------ taps
// The parity taps run the all-node program, compiled and uploaded on first use.
static void ensure_full(sgx_circuit* c) {
  if (c->full.fwd.p) return;
  sgx::build_full_program(c->L);
  c->full.upload(c->L.full, c->ctx->stream);
  CK(cudaStreamSynchronize(c->ctx->stream));
}

int sgx_forward(sgx_circuit* c, const float* p, int32_t batch, float* tape, float* y) {
  return guard([&] {
    need(c, "circuit");
    if (!c->layout_ok) throw StateError("circuit has no device layout");
    CK(cudaSetDevice(c->ctx->device));
    ensure_full(c);
    if (batch < 0) throw std::invalid_argument("batch must be non-negative");
    const auto& L = c->L;
    const size_t ncpi = L.cpi.size();
    if (batch * ncpi) need(p, "p");
    for (size_t i = 0; i < batch * ncpi; ++i)  // autodiff.cpp:71-73
      if (!(p[i] >= 0.0f && p[i] <= 1.0f)) throw std::invalid_argument("probabilities must lie in [0, 1]");
    if (batch == 0) return;
    CK(cudaSetDevice(c->ctx->device));
    cudaStream_t st = c->ctx->stream;
    const int Bp = round_up(batch, sgx::kThreads);
    const size_t nr = static_cast<size_t>(L.full.n_rows);
    std::vector<float> src(std::max<size_t>(ncpi * Bp, 1), 0.5f);
    for (int r = 0; r < batch; ++r)
      for (size_t j = 0; j < ncpi; ++j) src[tile_index(r, j, ncpi)] = p[r * ncpi + j];
    DBuf<float> dsrc, dtape;
    dsrc.upload(src, st);
    dtape.alloc(nr * Bp);
    sgx::launch_forward(st, kTapVec, c->full.fwd.p, c->full.fwd_lvl.p, c->full.n_fwd_levels, dsrc.p,
                        static_cast<int>(ncpi), dtape.p, L.full.n_rows, Bp, 1, c->ctx->exp_tab.p, &c->full.fb);
    CK(cudaGetLastError());
    std::vector<float> h(nr * Bp);
    CK(cudaMemcpyAsync(h.data(), dtape.p, h.size() * sizeof(float), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    // Reference node order; a folded node is recomputed from its operand with
    // the same float operation the device applies on read.
    auto value = [&](int node, int r) {
      int row = L.full.row_of_node[node];
      bool neg = false;
      if (row < 0) {
        row = L.full.virt_base[node];
        neg = L.full.virt_neg[node] != 0;
      }
      float x = h[tile_index(r, row, nr)];
      return neg ? 1.0f - x : x;
    };
    if (tape)
      for (int i = 0; i < L.n_nodes; ++i)
        for (int r = 0; r < batch; ++r) tape[static_cast<size_t>(i) * batch + r] = value(i, r);
    if (y) {
      const size_t m = L.out_node.size();
      for (size_t o = 0; o < m; ++o)
        for (int r = 0; r < batch; ++r) y[r * m + o] = value(L.out_node[o], r);
    }
  });
}

int sgx_backward(sgx_circuit* c, const float* tape, int32_t batch, const float* v, float* dv, float* dp) {
  return guard([&] {
    need(c, "circuit");
    if (!c->layout_ok) throw StateError("circuit has no device layout");
    CK(cudaSetDevice(c->ctx->device));
    ensure_full(c);
    if (batch < 0) throw std::invalid_argument("batch must be non-negative");
    if (batch == 0) return;
    need(tape, "tape");
    const auto& L = c->L;
    const size_t ncpi = L.cpi.size();
    if (ncpi) need(v, "v");
    CK(cudaSetDevice(c->ctx->device));
    cudaStream_t st = c->ctx->stream;
    const int Bp = round_up(batch, sgx::kThreads);
    const size_t nr = static_cast<size_t>(L.full.n_rows);
    // Only materialized rows are uploaded: folded nodes are re-derived from
    // their operand on read, exactly as the reference computes them.
    std::vector<float> ht(nr * Bp, 0.5f);
    for (int i = 0; i < L.n_nodes; ++i) {
      const int row = L.full.row_of_node[i];
      if (row < 0) continue;
      for (int r = 0; r < batch; ++r) ht[tile_index(r, row, nr)] = tape[static_cast<size_t>(i) * batch + r];
    }
    std::vector<float> hv(std::max<size_t>(ncpi * Bp, 1), 0.0f);
    for (int r = 0; r < batch; ++r)
      for (size_t j = 0; j < ncpi; ++j) hv[tile_index(r, j, ncpi)] = v[r * ncpi + j];
    DBuf<float> dt, dadj, dV, ddv, ddp;
    dt.upload(ht, st);
    dV.upload(hv, st);
    dadj.alloc(nr * Bp);
    ddv.alloc(std::max<size_t>(ncpi * Bp, 1));
    ddp.alloc(std::max<size_t>(ncpi * Bp, 1));
    CK(cudaMemsetAsync(ddv.p, 0, ddv.n * sizeof(float), st));
    CK(cudaMemsetAsync(ddp.p, 0, ddp.n * sizeof(float), st));
    backward(st, kTapVec, c->full, dt.p, dadj.p, dV.p, static_cast<int>(ncpi), ddv.p, ddp.p, Bp, 0.0f,
             c->out_tgt.p, static_cast<int>(L.out_node.size()), nullptr, c->ctx->exp_tab.p, nullptr);
    CK(cudaGetLastError());
    std::vector<float> hdv(ddv.n), hdp(ddp.n);
    CK(cudaMemcpyAsync(hdv.data(), ddv.p, hdv.size() * sizeof(float), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hdp.data(), ddp.p, hdp.size() * sizeof(float), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int r = 0; r < batch; ++r)
      for (size_t j = 0; j < ncpi; ++j) {
        if (dv) dv[r * ncpi + j] = hdv[tile_index(r, j, ncpi)];
        if (dp) dp[r * ncpi + j] = hdp[tile_index(r, j, ncpi)];
      }
  });
}

static int device_unary(sgx_ctx* ctx, const float* x, int64_t n, float* out, int sigmoid) {
  return guard([&] {
    need(ctx, "ctx");
    if (n < 0) throw std::invalid_argument("n must be non-negative");
    if (n == 0) return;
    need(x, "x");
    need(out, "out");
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    DBuf<float> dx, dy;
    dx.alloc(n);
    dy.alloc(n);
    CK(cudaMemcpyAsync(dx.p, x, n * sizeof(float), cudaMemcpyHostToDevice, st));
    sgx::launch_expf(st, dx.p, n, dy.p, ctx->exp_tab.p, sigmoid);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, dy.p, n * sizeof(float), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  });
}

int sgx_embed(sgx_ctx* ctx, const float* v, int64_t n, float* p) { return device_unary(ctx, v, n, p, 1); }

int sgx_expf(sgx_ctx* ctx, const float* x, int64_t n, float* out) { return device_unary(ctx, x, n, out, 0); }

struct sgx_extraction {
  sgx::ext::Result r;
};

int sgx_extract(int32_t num_vars, const int32_t* clause_ptr, const int32_t* clause_lit, int64_t n_clauses,
                int32_t complement_cap, int32_t minimize_cap, sgx_extraction** out) {
  return guard([&] {
    need(out, "out");
    *out = nullptr;
    if (num_vars < 0 || n_clauses < 0) throw std::invalid_argument("negative CNF size");
    if (n_clauses > 0) {
      need(clause_ptr, "clause_ptr");
      need(clause_lit, "clause_lit");
      if (clause_ptr[0] != 0) throw std::invalid_argument("clause_ptr[0] must be 0");
      for (int64_t c = 0; c < n_clauses; ++c)
        if (clause_ptr[c + 1] < clause_ptr[c]) throw std::invalid_argument("clause_ptr not monotone");
    }
    if (complement_cap < 0 || minimize_cap < 0 || minimize_cap > 16)
      throw std::invalid_argument("caps must be >= 0 (minimize_cap <= 16, the truth-table limit)");
    auto h = std::make_unique<sgx_extraction>();
    sgx::ext::extract_build(num_vars, clause_ptr, clause_lit, n_clauses, complement_cap, minimize_cap, h->r);
    *out = h.release();
  });
}

int sgx_extraction_sizes(const sgx_extraction* x, int64_t* out) {
  return guard([&] {
    need(x, "extraction");
    need(out, "out");
    const auto& r = x->r;
    out[0] = static_cast<int64_t>(r.kind.size());
    out[1] = static_cast<int64_t>(r.pi.size());
    out[2] = static_cast<int64_t>(r.po.size());
    out[3] = static_cast<int64_t>(r.iv.size());
    out[4] = static_cast<int64_t>(r.aux.size());
    out[5] = r.n_defs;
    out[6] = r.unsat ? 1 : 0;
  });
}

int sgx_extraction_export(const sgx_extraction* x, int32_t* kind, int32_t* a, int32_t* b, int32_t* var,
                          int32_t* inputs, int32_t* out_var, uint8_t* out_tgt, int32_t* iv, int32_t* aux) {
  return guard([&] {
    need(x, "extraction");
    const auto& r = x->r;
    auto put = [](int32_t* dst, const std::vector<int>& src) {
      if (dst) std::copy(src.begin(), src.end(), dst);
    };
    put(kind, r.kind);
    put(a, r.a);
    put(b, r.b);
    put(var, r.var);
    put(inputs, r.pi);
    put(iv, r.iv);
    put(aux, r.aux);
    for (size_t i = 0; i < r.po.size(); ++i) {
      if (out_var) out_var[i] = r.po[i].first;
      if (out_tgt) out_tgt[i] = r.po[i].second ? 1 : 0;
    }
  });
}

const char* sgx_extraction_note(const sgx_extraction* x) { return x ? x->r.unsat_note.c_str() : ""; }

void sgx_extraction_free(sgx_extraction* x) { delete x; }

}  // extern "C"
