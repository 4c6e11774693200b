// Host-callable launch wrappers for the kernels in sgx_kernels.cu.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

namespace sgx {

struct HarvestOut;

void launch_reinit_rows(cudaStream_t st, float* V, int ncols, int Bp, int tile_rows, uint64_t prefix,
                        long long row_offset, const uint32_t* valid, const uint32_t* newmask);
void launch_reinit_mask(cudaStream_t st, const uint32_t* valid, const uint32_t* newmask, uint8_t* age, int W,
                        int min_age, uint32_t* redraw);
void launch_init_v(cudaStream_t st, float* V, int ncols, int Bp, int tile_rows, uint64_t prefix,
                   long long row_offset, uint32_t* hb);
// The TMA-fed forward's control stream (sgx_layout.hpp SoftProgram::fblk).
struct FwdBlocks {
  const int4* fblk = nullptr;
  int blk0_n4 = 0, blk_max = 0;
};
void launch_forward(cudaStream_t st, int vec, const int4* grp, const int2* lvl, int n_levels,
                    const float* src, int ncols, float* tape, int n_rows, int Bp, int src_is_prob,
                    const uint64_t* exp_tab, const FwdBlocks* fb);
// Edge-record backward (sgx_layout.hpp kR* records); col_row[ncols] = tape row
// of each V column's INPUT node (-1: outside the program).  With hb, the new V
// is also hardened into hb[word][col] for the shared-memory harvest.
// The TMA-fed backward's control stream (sgx_layout.hpp SoftProgram::sblk).
struct BwdBlocks {
  const int4* sblk = nullptr;
  int blk0_n4 = 0, blk_max = 0;
  const int* tail_dead = nullptr;
  int n_tail_dead = 0;
};
void launch_backward_rec(cudaStream_t st, int vec, const int4* rec, const int2* lvl, int n_levels,
                         const float* tape, float* adj, float* V, int ncols, int n_rows, const int* col_row,
                         float* dv_out, float* dp_out, int Bp, float lr, const int* out_enc,
                         const uint8_t* out_tgt, int n_out, float* row_loss, const uint64_t* exp_tab,
                         uint32_t* hb, const int* dead, const int2* dead_lvl, const BwdBlocks* bb);
// Opt-in Adam logit update from a stored dV (step t >= 1 since the last init).
void launch_adam(cudaStream_t st, float* V, const float* dV, float* m, float* v, int ncols, int Bp, int tile_rows,
                 float lr, float b1, float b2, int t, float eps, uint32_t* hb);
void launch_loss(cudaStream_t st, const float* row_loss, int batch, double* partial, int n_partial,
                 double* out);
void launch_harden(cudaStream_t st, const float* V, int ncpi, int nucpi, const int* cpi_row,
                   const int* ucpi_row, uint32_t* BT, int W, int tile_rows, uint64_t free_prefix,
                   long long row_offset);
void launch_bit_eval(cudaStream_t st, int wpc, const int4* ops, const int* lvl_ptr, int n_levels,
                     uint32_t* BT, int W, const int* out_row, const uint8_t* out_tgt, int n_out,
                     const int* clause_ptr, const int* clause_enc, int n_clauses, uint32_t* valid,
                     int batch);
void launch_keys(cudaStream_t st, const uint32_t* BT, int W, const int* key_row, int key_words,
                 const uint32_t* valid, int Bp, uint64_t* K, int* slot_of_row, unsigned long long* tkeys,
                 unsigned long long* tmeta, uint64_t tmask, uint64_t epoch);
void launch_commit(cudaStream_t st, const uint32_t* valid, const int* slot_of_row,
                   const unsigned long long* tmeta, uint64_t epoch, int Bp, uint32_t* newmask,
                   int* block_count, long long quota_left, HarvestOut* out);
void launch_append(cudaStream_t st, const uint32_t* newmask, const int* block_off, const uint64_t* K,
                   int key_words, int Bp, uint64_t* store, long long base, long long cap,
                   HarvestOut* out,
                   bool row_major = false);
struct HarvestSmemArgs {
  const uint32_t* hb;  // hardened V columns [word][ncpi]
  int ncpi, nucpi;
  const int *cpi_row, *ucpi_row;
  uint64_t free_prefix;
  long long row_offset;
  const int4* ops;
  const int* lvl_ptr;
  int n_levels;
  const int* out_enc;
  const uint8_t* out_tgt;
  int n_out;
  const int4* cnf4;
  int cnf_steps;
  const int* key_enc;
  int key_words, batch, Bp;
  uint32_t* valid;
  uint64_t* K;
  int* slot_of_row;
  unsigned long long *tkeys, *tmeta;
  uint64_t tmask, epoch;
};
// Fused shared-memory harvest (harden + eval + PO/CNF + keys + insert); the
// folded bit tape of wpc words must fit in shared memory.
void launch_harvest_smem(cudaStream_t st, int wpc, int n_rows, int W, const HarvestSmemArgs& a);
// Device-side format_solutions (sgx_format.cu).  len_off: n + 1 int64,
// lengths then in-place exclusive offsets; call once with scratch = nullptr
// to size the scan's scratch.
long long fmt_base_len(int num_vars);
void launch_fmt_lengths(cudaStream_t st, const uint64_t* store, long long first, long long n, int words,
                        int num_vars, long long* len_off, void* scratch, size_t* scratch_bytes);
void launch_fmt_write(cudaStream_t st, const uint64_t* store, long long first, long long n, int words,
                      int num_vars, const long long* off, long long out_base, char* out);

// On-chip soft pass for small circuits (sgx_layout.hpp SoftProgram::oc_*):
// one warp per 32-sample tile runs forward, loss, backward, the V update and
// the hardening with its tape and adjoints in shared memory.  prog is one
// int4 buffer: [groups (kGroupRecs each)][records][per level / pass: fwd
// first, fwd count, rec first, rec count][column adjoint slots, 4 per int4]
// [output encodings, 4 per int4].
struct OnchipArgs {
  const int4* prog;
  int prog_n4, off_rec, off_lvl, off_col, off_out;
  int n_levels, n_rows, n_slots, ncols, n_out;
  float* V;             // [tile][col][32]
  uint32_t* hb;         // [word][col]
  float* row_loss;      // [B]
  const uint8_t* out_tgt;
  const uint64_t* exp_tab;
  float lr;
  int n_tiles;
};
// Returns false when the tile does not fit (the caller keeps the HBM kernels).
bool launch_soft_onchip(cudaStream_t st, const OnchipArgs& a);
int onchip_warps(int n_rows, int n_slots, int prog_n4);  // 0 = not eligible

// Liveness-allocated harvest (sgx_layout.hpp Layout::lb_*): bit tape in
// `slots` shared-memory rows per word, CNF-variable rows spilled to a global
// tape [n_spill][W] for the key phase.
struct HarvestLiveArgs {
  const uint32_t* hb;  // hardened V columns [word][ncpi]
  int ncpi, nucpi;
  const int2 *cpi, *ucpi;  // {slot, spill}
  uint64_t free_prefix;
  long long row_offset;
  const int4* ops;
  const int* op_ptr;
  const int4* chk;
  const int* chk_ptr;
  const int* big_lits;
  int n_phases, slots;
  uint32_t* spill;  // [n_spill][W]
  int W, n_spill;
  const int* key_enc;
  int key_words, batch, Bp;
  uint32_t* valid;
  uint64_t* K;
  int* slot_of_row;
  unsigned long long *tkeys, *tmeta;
  uint64_t tmask, epoch;
};
// wpc words per CTA; returns false if the slots do not fit shared memory.
bool launch_harvest_live(cudaStream_t st, int wpc, const HarvestLiveArgs& a);
// Warp-synchronous live harvest (one warp per word, k_harvest_lw) + spill
// keys (k_keys_spill); false if a CTA's slots do not fit shared memory.
bool launch_harvest_lw(cudaStream_t st, int warps_per_cta, const HarvestLiveArgs& a, const int4* lw, int n_iters);
void launch_compact_new(cudaStream_t st, const uint32_t* newmask, const int* block_off, const int* slot_of_row,
                        const unsigned long long* tkeys, int Bp, unsigned long long* out);
void launch_merge_remote(cudaStream_t st, const unsigned long long* all_fps, const long long* n_of, int nranks,
                         int me, long long stride, unsigned long long* tkeys, unsigned long long* tmeta,
                         uint64_t tmask, uint64_t epoch, uint32_t* newmask, int Bp, int* block_count,
                         HarvestOut* out);
void launch_rehash(cudaStream_t st, const unsigned long long* okeys, const unsigned long long* ometa,
                   uint64_t ocap, unsigned long long* nkeys, unsigned long long* nmeta, uint64_t nmask);
void launch_expf(cudaStream_t st, const float* x, long long n, float* out, const uint64_t* tab, int sigmoid);


// cmd_verify (tools/satgrad_main.cpp:242-302) on the device (sgx_verify.cu).
// err_kind: 0 ok, 1 exceeds the variable count, 2 assigned both ways,
// 3 missing 0 terminator, 4 unassigned, 5 does not satisfy, 6 duplicate.
struct VerifyResult {
  int64_t checked = 0, err_line = 0, err_var = 0;
  int32_t err_kind = 0;
  int64_t launches = 0;
};
// The same checks on packed keys (no text): rows that do not satisfy the CNF,
// rows with bits set above num_vars, rows that repeat an earlier row.
struct KeyCheck {
  int64_t checked = 0, unsat = 0, malformed = 0, duplicate = 0, launches = 0;
};
void verify_keys(int device, const std::vector<int64_t>& clause_ptr, const std::vector<int32_t>& clause_lit,
                 int num_vars, const uint64_t* keys, int64_t n, KeyCheck* out);
void verify_solutions(int device, const std::vector<int64_t>& clause_ptr, const std::vector<int32_t>& clause_lit,
                      int num_vars, const char* text, int64_t len, VerifyResult* out);
}  // namespace sgx
