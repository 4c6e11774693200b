/*
 * satgrad_b200 -- C-ABI of the B200-native (sm_100a) sampling loop.
 *
 * This is the drop-in boundary for the reference's data-parallel sampling
 * path (satgrad, arXiv 2502.08673).  The sampling loop below this header runs
 * on the GPU; CNF parsing and path classification stay in the caller, and
 * circuit extraction may (the reference's) or may not (sgx_extract, host
 * C++ in this library, node-for-node equal).  Plain C types only: no C++ or torch
 * types cross the boundary, arrays are host pointers with explicit sizes, and
 * every function returns 0 on success or a negative SGX_E* code, with a
 * thread-local message in sgx_last_error().
 *
 * Which reference interface each entry point replaces (paths relative to
 * /root/reference/proj):
 *
 *   sgx_circuit_upload   Circuit + CnfFormula + PathClassification as consumed
 *                        by run() (include/satgrad/circuit.hpp:20-40,
 *                        include/satgrad/cnf.hpp:27-38,
 *                        include/satgrad/extract.hpp:58-63); adds the
 *                        levelization / device-layout pass the reference lacks.
 *   sgx_sampler_create   SamplerConfig (include/satgrad/sampler.hpp:23-33).
 *   sgx_run              satgrad::run (include/satgrad/sampler.hpp:79-81,
 *                        src/sampler.cpp:89-203), f32 instantiation.
 *   sgx_init             init_soft_inputs (sampler.hpp:76-77, sampler.cpp:54-64)
 *                        + the double->S cast at sampler.cpp:156-159.
 *   sgx_step             embed + forward + loss + backward + gd_step
 *                        (autodiff.hpp:31-82, autodiff.cpp:57-290) fused.
 *   sgx_harvest          the harvest lambda (sampler.cpp:124-153): harden,
 *                        free bits, eval_discrete (circuit.cpp:124-152), PO
 *                        check, eval_cnf (cnf.cpp:129-147), dedupe_key +
 *                        SolutionSet::insert (sampler.cpp:18-44).
 *   sgx_fetch_solutions  SolutionSet keys in insertion order
 *                        (sampler.hpp:37-55), packed like dedupe_key.
 *   sgx_forward /        forward<float> / backward<float> (autodiff.hpp:52-78)
 *   sgx_backward         as parity taps, in the reference's layouts.
 *   sgx_verify_solutions cmd_verify (tools/satgrad_main.cpp:242-302).
 *   sgx_extract          extract + build (extract.hpp:53, circuit.hpp:42;
 *                        src/extract.cpp:43-172, src/circuit.cpp:60-122).
 */
#ifndef SATGRAD_B200_H
#define SATGRAD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SGX_OK 0
#define SGX_E_INVALID (-1)  /* std::invalid_argument in the reference */
#define SGX_E_CUDA (-2)     /* CUDA runtime / device failure          */
#define SGX_E_NOMEM (-3)    /* device allocation failed               */
#define SGX_E_STATE (-4)    /* call out of order                      */

/* GateKind order of circuit.hpp:20-22. */
enum sgx_gate_kind {
  SGX_INPUT = 0, SGX_CONST0, SGX_CONST1, SGX_BUF, SGX_NOT,
  SGX_AND2, SGX_OR2, SGX_XOR2, SGX_XNOR2
};

/* RestartPolicy, sampler.hpp:21.  SGX_RESTART_REINIT_ROWS and
 * SGX_RESTART_REINIT_INVALID are extensions (SPEC.md:473
 * "finer policies are future work"; no reference counterpart, so no count
 * parity), both on top of REINIT_ON_EXHAUST:
 *   REINIT_ROWS: after every harvest the rows that are valid but not new
 *     redraw their logits;
 *   REINIT_INVALID: as REINIT_ROWS, plus rows that are still invalid after
 *     `reinit_age` GD steps since their last draw redraw theirs.
 * The redraw decided at harvest h is applied before step h + 1, which then
 * waits for harvest h (SGX_REINIT_LAG=1: before step h + 2, keeping the
 * harvest/step overlap; slower to find solutions, measured in DESIGN.md). */
enum sgx_restart_policy {
  SGX_RESTART_NONE = 0, SGX_RESTART_REINIT_ON_EXHAUST = 1, SGX_RESTART_REINIT_ROWS = 2,
  SGX_RESTART_REINIT_INVALID = 3
};

typedef struct sgx_ctx sgx_ctx;
typedef struct sgx_circuit sgx_circuit;
typedef struct sgx_sampler sgx_sampler;

/* The reference's hot-path inputs, host-owned, copied by sgx_circuit_upload. */
typedef struct {
  /* Circuit::nodes in topological order: operands always at lower ids. */
  int32_t n_nodes;
  const int32_t* kind; /* sgx_gate_kind                                  */
  const int32_t* a;    /* operand node ids, -1 if unused                  */
  const int32_t* b;
  const int32_t* var;  /* variable owned by the node, 0 = internal        */
  int32_t num_vars;    /* CnfFormula::num_vars (aux vars are above it)    */
  /* Circuit::outputs (PoEntry list, incl. aux outputs), in order. */
  int32_t n_outputs;
  const int32_t* out_var;
  const uint8_t* out_target;
  /* PathClassification: V column order and free-bit order. */
  int32_t n_cpi;
  const int32_t* cpi;
  int32_t n_ucpi;
  const int32_t* ucpi;
  /* CnfFormula::clauses as CSR of DIMACS literals (+v / -v). */
  int64_t n_clauses;
  const int64_t* clause_ptr; /* n_clauses + 1 */
  const int32_t* clause_lit;
  /* ExtractionResult::unsat: run() returns immediately with a note. */
  int32_t unsat;
} sgx_circuit_desc;

/* SamplerConfig plus the sharding fields the multi-GPU path needs. */
typedef struct {
  int32_t batch;           /* rows on this device                        */
  int32_t iterations;
  double learning_rate;
  uint64_t seed;
  int64_t max_solutions;   /* 0 = no quota                               */
  double timeout_s;        /* 0 = none; checked between iterations       */
  int32_t restart_policy;  /* sgx_restart_policy                         */
  int64_t row_offset;      /* global row of local row 0 (RNG coordinates)*/
  int64_t solution_capacity; /* initial device solution store, 0 = auto  */
  int32_t max_restarts;    /* safety valve, reference uses 1000          */
  int32_t soft_kernel;     /* sgx_soft_kernel: which soft-pass kernels    */
  int32_t optimizer;       /* sgx_optimizer; 0 = the reference's GD       */
  double adam_beta1;       /* SGX_OPT_ADAM only; 0 = 0.9                  */
  double adam_beta2;       /* 0 = 0.999                                   */
  double adam_eps;         /* 0 = 1e-8                                    */
  int32_t reinit_age;      /* SGX_RESTART_REINIT_INVALID: GD steps an invalid
                              row keeps its draw; 0 = 2                   */
} sgx_sampler_cfg;

/* Logit update.  GD is the reference's gd_step (V -= lr dV, autodiff.cpp:
 * 285-290) and the default.  ADAM is an extension the reference lacks
 * (SPEC.md:418 lists adaptive optimizers as a non-goal, so it has no parity
 * anchor): per logit m = b1 m + (1 - b1) dV, v = b2 v + (1 - b2) dV^2,
 * V -= lr (m / (1 - b1^t)) / (sqrt(v / (1 - b2^t)) + eps), with m, v, t reset
 * by every init (restart).  It runs the HBM soft kernels. */
enum sgx_optimizer { SGX_OPT_GD = 0, SGX_OPT_ADAM = 1 };

/* Soft pass (embed + forward + loss + backward + GD + harden) kernels.  All
 * are bit-identical; they differ only in speed.
 *   AUTO: small circuits (cone tape <= 1,536 rows) get a circuit-specialised
 *         kernel compiled at run time (NVRTC, sm_100a) on a worker thread;
 *         steps run the HBM-tape kernels until it is ready.  Env SGX_JIT=0
 *         disables it, SGX_JIT=sync waits for the compile.
 *   HBM:  the level-synchronous tape kernels only.
 *   JIT:  compile at sampler creation and wait (HBM kernels if ineligible). */
enum sgx_soft_kernel { SGX_SOFT_AUTO = 0, SGX_SOFT_HBM = 1, SGX_SOFT_JIT = 2 };

typedef struct {
  int64_t unique_count;
  int64_t attempts;
  double wall_time_s;
  double throughput;
  int32_t restarts;
  int32_t timed_out;
  int32_t n_loss;     /* entries in the loss trace                       */
  int32_t n_harvest;  /* entries in the new-unique trace                 */
  int32_t unsat;      /* run skipped: instance unsatisfiable             */
  int32_t reserved;
  double device_ms;   /* CUDA-event time of the whole run on its stream  */
  int64_t launches;   /* kernels launched by the run                      */
} sgx_run_stats;

const char* sgx_last_error(void);
const char* sgx_version(void);

int sgx_open(int device, sgx_ctx** out);
int sgx_close(sgx_ctx* ctx);

int sgx_circuit_upload(sgx_ctx* ctx, const sgx_circuit_desc* desc, sgx_circuit** out);

/* Layout caches of sgx_circuit_upload.  In process: the compiled programs of
 * the last 4 circuits, keyed by a hash of the whole descriptor
 * (SGX_NO_LAYOUT_CACHE=1 turns it off).  On disk: with a directory set here
 * (or SGX_LAYOUT_CACHE_DIR), an upload reads <dir>/<key>.sgxlayout if present
 * and valid, else compiles and writes it -- the counterpart of the reference
 * CLI's circuit-JSON cache (tools/satgrad_main.cpp:137-184) one stage later.
 * NULL or "" disables the disk cache. */
int sgx_set_layout_cache_dir(const char* dir);

/* Waits for every background compile of the circuit-specialised soft pass
 * (SGX_SOFT_AUTO compiles it with NVRTC on a worker thread).  Also run
 * automatically at exit; a host that tears the process down some other way
 * (e.g. _exit, or unloading this library) calls it first. */
int sgx_jit_quiesce(void);
/* Host only: the layout sgx_circuit_upload would use (through both caches),
 * as a digest of every persisted field; *source = 0 compiled, 1 from the
 * in-process cache, 2 from the disk cache. */
int sgx_layout_digest(const sgx_circuit_desc* desc, uint64_t* digest, int32_t* source);
/* info[0..15]: nodes, cone nodes, cone edges, soft levels, bit levels,
 * fwd ops, bwd ops, bit ops, clauses, literals, key words, cpi, ucpi,
 * outputs, num_vars, unsat */
int sgx_circuit_info(const sgx_circuit* c, int64_t* info16);
int sgx_circuit_free(sgx_circuit* c);

/* Host-only layout compiler (no device calls): the same levelization and
 * device program construction sgx_circuit_upload performs.  For CPU tests. */
int sgx_layout_stats(const sgx_circuit_desc* desc, int64_t* info16);

/* Host only: implied[c] = 1 for every CNF clause the harvest does not check
 * because the gate definitions or the output targets imply it (every row
 * that passes eval_discrete + the output check satisfies it; replaces part
 * of eval_cnf, src/cnf.cpp:129-147, without changing any row's verdict).
 * implied holds n_clauses bytes.  SGX_ALL_CLAUSES=1 in the environment
 * disables the pruning (all zeros). */
int sgx_harvest_clause_mask(const sgx_circuit_desc* desc, uint8_t* implied);

/* Source of the circuit-specialised soft-pass kernel (host only, no device
 * calls; SGX_E_INVALID if the circuit is not eligible).  *len = bytes incl.
 * the NUL; out = NULL only sizes. */
int sgx_jit_source(const sgx_circuit_desc* desc, char* out, int64_t cap, int64_t* len);

int sgx_sampler_create(sgx_circuit* c, const sgx_sampler_cfg* cfg, sgx_sampler** out);
int sgx_sampler_free(sgx_sampler* s);
/* info[0] soft kernel of the last step (0 HBM tape, 1 JIT, 2 on-chip),
 * info[1] steps run by the JIT kernel, info[2] JIT state (-1 none,
 * 0 compiling, 1 ready, 2 failed), info[3] its compile time in us,
 * info[4] harvest kernel (0 global-memory, 1 full-tape shared-memory,
 * 2 live-slot), info[5] its words per CTA, info[6] samples per lane of the
 * HBM soft kernels, info[7] padded batch. */
int sgx_sampler_soft_info(const sgx_sampler* s, int64_t* info8);

/* One restart's building blocks (what sgx_run loops over). */
int sgx_init(sgx_sampler* s, int32_t restart);
int sgx_step(sgx_sampler* s, double* loss_total);
int sgx_harvest(sgx_sampler* s, int32_t restart, int32_t iter, int64_t* attempts,
                int64_t* added);

/* Multi-GPU harvest (sample sharding: rank g owns global rows [g*B, (g+1)*B)
 * via cfg.row_offset).  sgx_harvest is split around the caller's all-gather:
 *   sgx_harvest_local   harden, eval, CNF check, keys, local table insert;
 *                       *n_new = locally-new rows, *fps = DEVICE pointer to
 *                       their 64-bit fingerprints in row order (stride =
 *                       sgx_fingerprint_stride entries; valid until commit).
 *   sgx_harvest_merge   all_fps = DEVICE array [nranks][stride] gathered
 *                       from every rank, counts = HOST array of each rank's
 *                       n_new.  A fingerprint found by several ranks stays
 *                       new only on the lowest one (the reference's row
 *                       order over the union of the shards); every remote
 *                       fingerprint joins the local table.  *n_won = rows
 *                       still new here.
 *   sgx_harvest_commit  append the first min(n_won, quota_left) of them
 *                       (quota_left < 0: no quota); attempts as sgx_harvest. */
int sgx_fingerprint_stride(const sgx_sampler* s);
/* The fingerprint buffer of sgx_harvest_local holds stride + 1 int64: the
 * harvest's new fingerprints in row order, then their count at [stride], so
 * one all-gather of stride + 1 values per rank carries both. */
/* A GD step launched without waiting (the multi-GPU loop runs the next step
 * while the harvest's exchange is in flight); *slot names it for
 * sgx_step_loss, which waits for that step and returns its loss total. */
int sgx_step_async(sgx_sampler* s, int32_t* slot);
int sgx_step_loss(sgx_sampler* s, int32_t slot, double* loss_total);
/* Kernels this sampler launched (since its last sgx_run, or since creation). */
int64_t sgx_launch_count(const sgx_sampler* s);
int sgx_harvest_local(sgx_sampler* s, int32_t restart, int32_t iter, int64_t* n_new, uint64_t** fps);
int sgx_harvest_merge(sgx_sampler* s, const uint64_t* all_fps, const int64_t* counts, int32_t nranks,
                      int32_t rank, int64_t stride, int64_t* n_won);
int sgx_harvest_commit(sgx_sampler* s, int64_t quota_left, int64_t* attempts, int64_t* added);

/* ---- Multi-GPU run through the C-ABI ----------------
 * Sample sharding: rank g of nranks runs its own sampler with
 * cfg.row_offset = g * cfg.batch (global rows [g*B, (g+1)*B); every random
 * draw is keyed by global row, so the union of the shards IS a one-device run
 * at batch nranks * B).  sgx_run_sharded is satgrad::run over that union:
 * per harvest ONE all-gather of the new 64-bit fingerprints (+ their count);
 * a fingerprint found by several ranks counts once, for the lowest rank (the
 * reference's row order); quota / restart / timeout decisions are taken on
 * gathered values, so every rank takes the same branch.  stats.unique_count
 * is the global count; each rank stores the solutions it won
 * (sgx_fetch_solutions), their union is the global solution set.
 *
 * The collective comes from the caller as an sgx_exchange, or from the
 * library: sgx_exchange_nccl_create (one process per GPU; NCCL over
 * NVLink / NVSwitch, libnccl.so.2 resolved at run time -- the copy already
 * loaded in the process if any) or sgx_exchange_local_create (one process,
 * one host thread per rank, device-to-device copies; ranks may share a GPU). */
typedef struct sgx_exchange {
  void* user;
  int32_t rank;
  int32_t nranks;
  /* All-gather `bytes` of DEVICE memory `send` from every rank into DEVICE
   * memory `recv` (nranks * bytes, rank-major), ordered on `stream` (a
   * cudaStream_t): producers of `send` precede it there, and consumers of
   * `recv` follow it there.  0 on success. */
  int (*allgather_device)(void* user, const void* send, void* recv, int64_t bytes, void* stream);
  /* All-gather n int64 host values per rank into recv[nranks * n]; blocking. */
  int (*allgather_host)(void* user, const int64_t* send, int64_t* recv, int32_t n);
} sgx_exchange;

int sgx_run_sharded(sgx_sampler* s, const sgx_exchange* ex, sgx_run_stats* stats);
/* After sgx_run_sharded: how many of each harvest's new solutions this rank
 * stored (stats.n_harvest entries).  Rank order within a harvest is the
 * reference's insertion order over the union. */
int sgx_run_local_added(const sgx_sampler* s, int64_t* added);

/* NCCL: rank 0 makes the id, the caller distributes it (MPI, torch.distributed,
 * a file), every rank creates its exchange on its device. */
int sgx_nccl_unique_id(uint8_t id[128]);
int sgx_exchange_nccl_create(int32_t nranks, const uint8_t id[128], int32_t rank, int32_t device,
                             sgx_exchange* out);
int sgx_exchange_nccl_destroy(sgx_exchange* ex);
/* In-process group of nranks: fills out[0..nranks-1], one per rank / thread.
 * Destroy once, with any of them, after every rank has finished. */
int sgx_exchange_local_create(int32_t nranks, sgx_exchange* out);
int sgx_exchange_local_destroy(sgx_exchange* ex);

/* satgrad::run: the whole restart x iteration loop with quota, timeout and
 * restart policy; solutions stay on the device until fetched. */
int sgx_run(sgx_sampler* s, sgx_run_stats* stats);
int sgx_run_traces(sgx_sampler* s, double* loss_trace, int64_t* new_unique);
int64_t sgx_solution_count(const sgx_sampler* s);
int32_t sgx_key_words(const sgx_sampler* s);
int sgx_fetch_solutions(sgx_sampler* s, int64_t first, int64_t count, uint64_t* keys);
/* Host streaming of the result (satgrad::run returns every solution,
 * sampler.hpp:79-81): with it on, each harvest's new keys are copied to host
 * memory by a worker thread while sampling continues.  Enable before sgx_run. */
int sgx_set_host_stream(sgx_sampler* s, int32_t on);
/* Move all solution keys ([rows][key_words], insertion order) to the caller
 * without a copy when host streaming had them already, else copy them now.
 * The memory belongs to the caller: release it with sgx_host_free(keys,
 * map_bytes).  keys = NULL when there are no solutions. */
int sgx_solutions_take(sgx_sampler* s, uint64_t** keys, int64_t* rows, int64_t* map_bytes);
int sgx_host_free(uint64_t* keys, int64_t map_bytes);
/* format_solutions (include/satgrad/sampler.hpp:86, sampler.cpp:78-85) of
 * solutions [first, first + count), rendered on the device: "v1 -v2 ... vn 0\n"
 * per solution.  *len = text bytes; with out = NULL only the length is
 * computed, else out must hold cap >= *len bytes (SGX_E_INVALID otherwise). */
int sgx_format_solutions(sgx_sampler* s, int64_t first, int64_t count, char* out, int64_t cap, int64_t* len);
/* The sampler's current logits V as [batch][n_cpi] row-major (the reference's
 * Mat<float> v of run_impl, sampler.cpp:157-173): trajectory parity tap. */
int sgx_read_logits(sgx_sampler* s, float* v);
/* Device time of the last sgx_run by phase, milliseconds:
 * [init, step(fwd+bwd), harvest, fwd, bwd, eval, keys, commit] */
int sgx_phase_times(const sgx_sampler* s, double* ms8);

/* Parity taps over ALL nodes, reference layouts: p / v / dv / dp are [batch][n_cpi]
 * row-major, tape is [n_nodes][batch] in reference node order, y is
 * [batch][n_outputs]. */
int sgx_forward(sgx_circuit* c, const float* p, int32_t batch, float* tape, float* y);
int sgx_backward(sgx_circuit* c, const float* tape, int32_t batch, const float* v,
                 float* dv, float* dp);
/* embed (autodiff.cpp:57-62): clamped sigmoid of a host array, on device. */
int sgx_embed(sgx_ctx* ctx, const float* v, int64_t n, float* p);

/* Bit-exact device sigmoid / expf over a host array (parity of the glibc
 * expf restatement used by embed/backward). */
int sgx_expf(sgx_ctx* ctx, const float* x, int64_t n, float* out);

/* cmd_verify (tools/satgrad_main.cpp:242-302): check a solution text of
 * "v1 -v2 ... 0" lines against the circuit's CNF -- every line a complete,
 * consistent assignment that satisfies the formula, all pairwise distinct --
 * parsed on host threads, CNF-checked on the GPU.  out[5] = {checked,
 * err_line (1-based, 0 = none), err_var, err_kind, kernel launches}; err_kind
 * 0 ok, 1 variable exceeds the count, 2 assigned both ways, 3 missing 0
 * terminator, 4 unassigned (err_var = first), 5 does not satisfy the formula,
 * 6 duplicate assignment.  checked = solutions verified before the error. */
int sgx_verify_solutions(sgx_circuit* c, const char* text, int64_t len, int64_t* out);
/* The same checks on packed keys ([n][key_words], dedupe_key layout, host
 * memory), counting instead of stopping at the first error: out[0] checked,
 * out[1] keys that do not satisfy the CNF, out[2] keys with bits above
 * num_vars, out[3] keys equal to an earlier key, out[4] kernels launched. */
int sgx_verify_keys(sgx_circuit* c, const uint64_t* keys, int64_t n, int64_t* out);
/* The same from the CNF alone (what cmd_verify has): CSR clause_ptr[n_clauses
 * + 1] over DIMACS literals. */
int sgx_verify_cnf(sgx_ctx* ctx, int32_t num_vars, const int64_t* clause_ptr, const int32_t* clause_lit,
                   int64_t n_clauses, const char* text, int64_t len, int64_t* out);

/* ---- Circuit extraction (host) -------------------------
 * extract + build (src/extract.cpp:43-172, src/boolexpr.cpp, src/circuit.cpp:
 * 60-122; include/satgrad/extract.hpp:53, circuit.hpp:42): the CNF (CSR
 * clause_ptr[n_clauses + 1] over DIMACS literals) to the reference's
 * ExtractionResult and gate-level Circuit, node for node.  Caps are
 * ExtractorConfig (extract.hpp:14-17: complement_cap 16, minimize_cap 12). */
typedef struct sgx_extraction sgx_extraction;
int sgx_extract(int32_t num_vars, const int32_t* clause_ptr, const int32_t* clause_lit, int64_t n_clauses,
                int32_t complement_cap, int32_t minimize_cap, sgx_extraction** out);
/* out[7] = {n_nodes, |pi|, |po|, |iv|, |aux|, |be|, unsat} */
int sgx_extraction_sizes(const sgx_extraction* x, int64_t* out);
/* Node arrays [n_nodes] (GateKind codes, operand ids or -1, var or 0), pi,
 * po (var, target), iv, aux in the reference's orders; any pointer may be NULL. */
int sgx_extraction_export(const sgx_extraction* x, int32_t* kind, int32_t* a, int32_t* b, int32_t* var,
                          int32_t* inputs, int32_t* out_var, uint8_t* out_tgt, int32_t* iv, int32_t* aux);
/* ExtractionResult::unsat_note ("" when satisfiable so far). */
const char* sgx_extraction_note(const sgx_extraction* x);
void sgx_extraction_free(sgx_extraction* x);

#ifdef __cplusplus
}
#endif
#endif /* SATGRAD_B200_H */
