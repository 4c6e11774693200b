// Host-side levelizer and device-layout compiler.
//
// The reference evaluates its circuit in plain node-id order
// (autodiff.cpp:87-143, circuit.cpp:126-146); it has no levelization.  This
// pass turns the reference's topological node array (circuit.hpp:20-40) into
// the programs the sm_100a kernels execute:
//
//  * a SOFT program over the primary-output cone (or every node, for the
//    parity taps): tape rows sorted by (ASAP level, node id); a forward op
//    stream and a pull-style backward micro-op stream, both cut into chunks of
//    kU ops that never cross a level boundary, so every op in a chunk is
//    independent of the others and all of a chunk's loads can be in flight
//    at once;
//  * a BIT program over every node for the bit-sliced harvest (32 samples per
//    word): level pointers for a level-synchronous sweep, the CNF as bit-row
//    literals, the output checks and the dedupe-key variable map.
//
// Summation order is the reference's by construction: an adjoint is seeded
// first (autodiff.cpp:201-207) and then pulls its fan-out in descending
// consumer id, a-slot before b-slot (the push order of :208-280).  Consumers
// outside the cone carry an exactly-zero adjoint, so pruning them changes no
// bits.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/satgrad_b200.h"

namespace sgx {

constexpr int kU = 8;      // ops per chunk (loads in flight per thread)
#ifndef SGX_WARPS
#define SGX_WARPS 4
#endif
constexpr int kWarps = SGX_WARPS;  // warps per CTA sharing one sample tile (node split)

// Forward group: kGroupRecs int4 records.  Header {kind, n, first_out_row, 0},
// then kGroup operand pairs (a, b) packed two per int4; an operand is
// row << 1 | negate (negate = read through a folded NOT).  INPUT: a = V
// column or -1 (= 0.5).  The group's outputs are rows first_out_row + [0, n).
// Backward micro-op (int4, host-side intermediate of the edge records), opcode
// in the low byte:
//   BEGIN     {kBegin | seed | target, row, 0, 0}
//   EDGE      {kEdge | consumer_kind << 12 | neg_other | in_sub,
//              adj_row_of_consumer, other_row (-1), 0}
//   SUB_BEGIN {kSubBegin | seed | target | neg_self, row of the folded node's
//              operand, 0, 0}      -- opens adj[j] of a folded NOT/BUF j
//   SUB_END   {kSubEnd | kind(j) << 12}   -- acc -= adj[j] (NOT) / += (BUF)
//   END       {kEnd, adj_row_to_store (-1), V column (-1), 0}
// Bit op (int4): {kind, out_row, a_row, b_row}.
// Clause literal (int32): bit_row << 2 | last_in_clause << 1 | negated.
enum OpCode : int32_t { kNop = 15, kBegin = 16, kEdge = 17, kEnd = 18, kSubBegin = 19, kSubEnd = 20 };
constexpr int32_t kSeedBit = 1 << 8, kTargetBit = 1 << 9, kNegOtherBit = 1 << 10,
                  kNegSelfBit = 1 << 11, kKindShift = 12, kInSubBit = 1 << 16;
// Backward edge record (int4) {flags, adj_row_of_consumer (-1), other_row (-1),
// own_row}: one record per fan-out edge, with the micro-ops' control folded
// into flag bits so the kernel runs every record through the same
// straight-line arithmetic (acc = acc*k + seed; acc += g*fa; acc2 += g*fb;
// acc += s*acc2; see k_backward_rec).  A record without an edge (y = -1)
// carries an empty node / empty SUB run.  Flags:
//   bits 0-3 consumer kind, kRInSub (edge of a SUB run: feeds acc2),
//   kRNegOther (other operand read through a folded NOT),
//   kRFirst / kRSubFirst (reset acc / acc2 to the seed or +0 first),
//   kRSubLast (+ kRSubNot: then acc -= acc2, else acc += acc2),
//   kRSeed|kRTarget, kRSubSeed|kRSubTarget|kRNegSelf (output seeds from T[own_row]),
//   kRLast (store acc to adj[own_row]).
constexpr int32_t kRInSub = 1 << 4, kRNegOther = 1 << 5, kRFirst = 1 << 6, kRSubFirst = 1 << 7,
                  kRSubLast = 1 << 8, kRSubNot = 1 << 9, kRSeed = 1 << 10, kRTarget = 1 << 11,
                  kRSubSeed = 1 << 12, kRSubTarget = 1 << 13, kRNegSelf = 1 << 14, kRLast = 1 << 15;
// kRSlow: anything but a plain edge into the node's own accumulator (seeds,
// SUB-run records, records without an edge) -- the staged kernel's fast path
// is taken only without it.
constexpr int32_t kRSlow = 1 << 16;
// kRSubOne (with kRSlow, staged records only): a SUB run of ONE edge and no
// seed -- adj[j] = +0 + g*fa, then acc -= / += adj[j] -- which the staged
// kernel runs on a short branch of its own (79 % of the SUB-run records on
// C4 and C2).  Cleared in oc_rec, whose bits 17+ hold slots.
constexpr int32_t kRSubOne = 1 << 29;
// kRYKeep (staged records only): the other operand's tape row is read again
// within SGX_BWD_KEEP passes, so this read keeps it in L2 (no evict_first).
// Cleared in oc_rec.
constexpr int32_t kRYKeep = 1 << 28;
constexpr int kOcSlotShift = 17;  // oc_rec: adjoint store slot in the flag word
constexpr int kCnfThreads = 256;               // threads of the shared-memory harvest CTA
constexpr int32_t kCnfOpen = INT32_MIN;        // CNF record continues (see fb_cnf4)
constexpr int32_t kLwEnd = 1 << 30, kLwChk = 1 << 29;
// k_harvest_lw record ring: kLwBuf chunks of kLwChunk iterations (32 int4 each); lw_ops is padded to whole chunks
constexpr int kLwChunk = 8, kLwBuf = 4, kLwRingBytes = kLwChunk * kLwBuf * 32 * 16;
static_assert(kLwChunk % 2 == 0, "k_harvest_lw runs iterations in pairs inside a chunk");  // lw_ops .x flags (op kind | out_slot << 4 below)
constexpr int32_t kLbBig = INT32_MIN;          // lb_chk: long clause, literals in lb_big_lits
constexpr int kGroup = 4;                      // ops per forward group
constexpr int kGroupRecs = 1 + kGroup / 2;     // int4 records per group

struct I4 {
  int32_t x, y, z, w;
};

struct SoftProgram {
  int32_t n_rows = 0;                // tape rows (materialized nodes)
  int32_t n_set = 0;                 // nodes in the program's set (cone)
  int32_t n_levels = 0;
  int64_t n_edges = 0;               // operand edges inside the program
  std::vector<int32_t> row_of_node;  // -1 if the node is not in the program
  std::vector<int32_t> node_of_row;
  std::vector<I4> fwd;               // groups, kGroupRecs records each
  std::vector<int32_t> fwd_lvl;      // per (level, warp): first group, group count
  std::vector<I4> rec;               // backward edge records
  std::vector<int32_t> rec_lvl;      // per (level high to low, warp): first record, count
  // Adjoint rows whose last reader runs in backward pass li (levels high to
  // low): after that pass's barrier the rows are dead and are discarded from
  // L2 without write-back (discard.global.L2).  Column-input rows are read by
  // the V epilogue and discarded after it.
  std::vector<int32_t> dead;         // rows, grouped by pass
  std::vector<int32_t> dead_lvl;     // per pass: first index into dead, count
  // Staged blocks for the TMA-fed backward: per pass li one contiguous block
  // of int4s = a header {dead_rel, n_dead, next_start, next_n4}, per warp
  // {first_rel, count} (two warps per int4), the pass's records (all warps,
  // warp order), then the rows that died in pass li-1, packed four per int4
  // (-1 padding).  One bulk copy brings a pass's whole control stream on
  // chip, and the header says where the next one is.
  std::vector<I4> sblk;
  std::vector<int32_t> sblk_lvl;     // per pass: start, n_int4, dead start (relative), n_dead
  std::vector<int32_t> srec_lvl;     // per (pass, warp): first record (relative to the block), count
  std::vector<int32_t> tail_dead;    // rows that died in the last pass (+ none) -> discarded after it
  // Staged forward blocks: per level a header {next_start, next_n4, 0, 0},
  // per warp {first_rel, groups} (two warps per int4), then the level's
  // groups (kGroupRecs int4s each, warp order).
  std::vector<I4> fblk;
  std::vector<int32_t> fblk_lvl;     // per level: start, n_int4
  int32_t fblk_max = 0;
  // On-chip program (k_soft_onchip, small circuits): one warp owns 32
  // samples and runs the whole program alone, so levels need no barrier and
  // the streams are linear: oc_fwd = the forward groups in level order,
  // oc_rec = the backward records (levels high to low) with the adjoint
  // rows renamed to live-range slots: .y = slot of the consumer's adjoint,
  // flags bits 17+ = slot the node's adjoint is stored to (kRLast); .z / .w
  // stay tape rows.  oc_col_slot = adjoint slot of each V column's input
  // (live until the V epilogue).
  std::vector<I4> oc_fwd;
  std::vector<I4> oc_rec;
  std::vector<int32_t> oc_fwd_lvl;   // per level: first group, count (records hoist loads only within a level)
  std::vector<int32_t> oc_rec_lvl;   // per pass (high to low): first record, count
  std::vector<int32_t> oc_col_slot;
  int32_t oc_adj_slots = 0;
  int32_t sblk_max = 0;              // largest block, int4s
  std::vector<int32_t> out_enc;      // each output as row << 1 | negate (-1: not in set)
  std::vector<int32_t> col_row;      // tape row of each V column's INPUT node
  std::vector<int32_t> virt_base;    // folded node -> row of its operand (-1 otherwise)
  std::vector<uint8_t> virt_neg;     // folded node is a NOT
};

struct Layout {
  // Reference inputs (validated copies).
  int32_t n_nodes = 0, num_vars = 0, max_var = 0;
  std::vector<int32_t> kind, a, b, var;
  std::vector<int32_t> node_of_var;  // max_var + 1, -1 = no node
  std::vector<int32_t> out_var, out_node;
  std::vector<uint8_t> out_tgt;
  std::vector<int32_t> cpi, ucpi;
  std::vector<int64_t> clause_ptr;
  std::vector<int32_t> clause_lit;
  // The clauses the harvest checks (sgx_layout.cpp harvest_clauses): the CNF
  // minus those implied by gate definitions or output targets.
  std::vector<int64_t> hclause_ptr;
  std::vector<int32_t> hclause_lit;
  int64_t n_implied = 0;
  std::vector<uint8_t> clause_implied;  // per CNF clause: 1 = not checked by the harvest
  bool unsat = false;
  std::vector<int32_t> level;        // ASAP level per node

  SoftProgram cone;                  // sampling
  SoftProgram full;                  // parity taps (every node)

  // Bit-sliced harvest program over every node.
  int32_t n_bit_rows = 0;
  std::vector<int32_t> bit_row_of_node;
  std::vector<I4> bit_ops;           // non-INPUT nodes, level-sorted
  std::vector<int32_t> bit_lvl_ptr;  // into bit_ops
  std::vector<int32_t> cpi_bit_row, ucpi_bit_row;
  std::vector<int32_t> out_bit_row;
  std::vector<int32_t> clause_ptr32; // n_clauses + 1
  std::vector<int32_t> clause_enc;   // bit_row << 1 | negated
  int32_t key_words = 0;             // (num_vars + 63) / 64
  std::vector<int32_t> key_bit_row;  // key_words * 64, -1 = padding

  // Folded bit program for the shared-memory harvest: NOT/BUF nodes whose
  // operand is materialized own no row (read as row ^ mask); every reference
  // is row << 1 | negate.
  int32_t fb_rows = 0;
  std::vector<I4> fb_ops;            // {kind, out_row, a_enc, b_enc}, level-sorted
  std::vector<int32_t> fb_lvl_ptr;
  std::vector<int32_t> fb_cpi_row, fb_ucpi_row;
  std::vector<int32_t> fb_out_enc;
  std::vector<int32_t> fb_key_enc;   // key_words * 64, -1 = padding
  // CNF as int4 records of up to 4 literals (row, or ~row when negated;
  // padding = the zero row fb_rows; .w == kCnfOpen: the clause continues in
  // the thread's next record), clauses kept whole per thread and stored
  // transposed [step][kCnfThreads] so that at every step the CTA's threads
  // read consecutive records.  Shared-memory tapes hold fb_rows + 1 rows.
  int32_t fb_cnf_steps = 0;
  std::vector<I4> fb_cnf4;

  // Liveness-allocated harvest (k_harvest_live): the folded bit program with
  // rows mapped to shared-memory SLOTS by a linear scan over the levels (a
  // slot is reused once its row's last reader -- gate operand, clause or
  // output check -- has run), so only the live set is on chip.  Every check
  // runs one level after its latest literal is defined (one barrier per
  // level).  Rows whose node carries a CNF variable are also written to a
  // global spill tape [lb_n_spill][words], read back by the key phase.
  //   op record:      {kind | out_slot << 4, a_enc, b_enc, spill (-1)}, enc = slot << 1 | negate
  //   check record:   up to 4 literals, slot or ~slot (negated), padding = slot 0
  //                   (always zero); a longer clause is {lit offset, count, 0, kLbBig}
  //                   with its literals in lb_big_lits
  //   input:          {slot, spill} per constrained / free input (int2)
  int32_t lb_slots = 0;              // slots incl. the zero slot 0
  int32_t lb_levels = 0;             // phases (levels + one trailing check phase)
  int32_t lb_n_spill = 0;
  std::vector<I4> lb_ops;
  std::vector<int32_t> lb_op_ptr;    // per phase
  std::vector<I4> lb_chk;
  std::vector<int32_t> lb_chk_ptr;   // per phase
  std::vector<int32_t> lb_big_lits;
  std::vector<int32_t> lb_cpi, lb_ucpi;  // {slot, spill} pairs
  std::vector<int32_t> lb_key_enc;   // key_words * 64: spill << 1 | negate (-1 padding)
  // The same program for the warp-synchronous harvest (k_harvest_lw): each
  // phase's ops cut into iterations of 32 records (one per lane), padded with
  // records writing the sink slot lb_slots; the last iteration of a phase has
  // kLwEnd (+ kLwChk when the phase has checks) in .x.  Record:
  // {anf | out_slot << 4 | flags, a_slot, b_slot, spill}: the gate and its
  // operand negations as f = c0 ^ c1 X ^ c2 Y ^ c3 XY (coefficient k = bit k).
  std::vector<I4> lw_ops;            // n_iters * 32
  int32_t lw_iters = 0;

  int64_t n_lits() const { return static_cast<int64_t>(clause_lit.size()); }
};

// Throws std::invalid_argument with the reference's wording where one exists.
Layout build_layout(const sgx_circuit_desc& d);

void layout_info(const Layout& L, int64_t* info16);

// On-disk layout (sgx_layout_io.cpp): false on any I/O failure or mismatch
// (magic, version, key, truncation); the caller then rebuilds.
bool save_layout(const Layout& L, const std::string& path, uint64_t key);
bool load_layout(Layout* L, const std::string& path, uint64_t key);
// FNV-1a over every persisted field (tests: a loaded layout equals a built one).
uint64_t layout_digest(const Layout& L);

// The all-node soft program of the parity taps (sgx_forward / sgx_backward),
// built on first use.
void build_full_program(Layout& L);

}  // namespace sgx
