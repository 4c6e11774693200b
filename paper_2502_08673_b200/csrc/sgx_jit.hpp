// Circuit-specialised soft pass (small circuits): the cone's soft program is
// compiled at run time (NVRTC, sm_100a) into ONE straight-line kernel per
// circuit -- embed, forward, per-row loss, backward, the V update and the
// hardening of the new V, one sample per thread, with every tape value and
// adjoint a register (or a spill slot the compiler chooses).  The tape never
// touches HBM: the only traffic is V (read, written), the row loss and the
// harvest's input words.
//
// The generated code is a literal transcription of the records the HBM
// kernels interpret (sgx_layout.hpp SoftProgram::fwd / ::rec, in the same
// order, with the same _rn intrinsics), so it reproduces their bits -- and
// thereby the reference's (autodiff.cpp:57-297) -- exactly.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <string>

#include "sgx_layout.hpp"

namespace sgx {

// Largest program the generator takes on (tape rows / records): beyond this
// the live set no longer fits registers + L1 and the HBM kernels win.
constexpr int kJitMaxRows = 1536;
constexpr int64_t kJitMaxRecs = 6144;

struct JitKernel;  // compiled kernel, shared by every sampler of the circuit

bool jit_eligible(const Layout& L);
// Waits for every background compile (sgx_jit_quiesce; also run at exit).
void jit_quiesce();
// CUDA C++ source of the kernel `sgx_jit_step` for L.cone (deterministic);
// min_blocks = __launch_bounds__ minimum CTAs per SM (register budget).
std::string jit_source(const Layout& L, int min_blocks);
// The min_blocks the sampler uses for L (SGX_JIT_MINB overrides).
int jit_min_blocks(const Layout& L);

// Compile (or find in the process cache) the kernel for L.  async: compile on
// a worker thread and return at once; the handle becomes ready() later.
std::shared_ptr<JitKernel> jit_get(const Layout& L, bool async);
bool jit_ready(const JitKernel* k);   // compiled and loadable
bool jit_failed(const JitKernel* k);  // compile error (log in jit_log)
void jit_wait(const JitKernel* k);
std::string jit_log(const JitKernel* k);
double jit_compile_ms(const JitKernel* k);

// One GD step on a [tile][col][TR] V block of n_samples rows (multiple of
// 128): V updated in place, hb[word][ncols] hardened words, row_loss[row].
void jit_launch(JitKernel* k, cudaStream_t st, float* V, int TR, uint32_t* hb, float* row_loss,
                const uint64_t* exp_tab, float lr, int n_samples);

}  // namespace sgx
