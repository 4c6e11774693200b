/*
 * TEST INFRASTRUCTURE ONLY -- the parity oracle, never the product.
 *
 * A plain-C restatement of the reference's data-parallel sampling loop
 * (satgrad, /root/reference/proj), single precision (the reference's
 * `use_f32` instantiation, the one the GPU path matches).  It is pinned
 * bit-for-bit against the reference library itself (oracle/_ref, built from
 * the reference sources by oracle/Makefile) by tests/test_oracle.py, and
 * against the committed golden vectors in tests/golden/.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library.
 *
 * Node arrays are in the reference's topological node order
 * (circuit.hpp:20-40): kind follows GateKind {Input, Const0, Const1, Buf, Not,
 * And2, Or2, Xor2, Xnor2}.  Matrices are row-major [row][col] like Mat<S>
 * (autodiff.hpp:20-29); the tape is node-major [node][batch]
 * (autodiff.hpp:36-44).
 */
#define _POSIX_C_SOURCE 199309L
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

enum { K_INPUT, K_CONST0, K_CONST1, K_BUF, K_NOT, K_AND, K_OR, K_XOR, K_XNOR };

/* rng.hpp:14-19 */
uint64_t so_mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

/* rng.hpp:21-25 */
uint64_t so_hash_stream(const uint64_t* xs, int n) {
  uint64_t h = 0x243f6a8885a308d3ull;
  for (int i = 0; i < n; ++i) h = so_mix64(h ^ so_mix64(xs[i]));
  return h;
}

/* rng.hpp:28-30 */
static double u01(uint64_t bits) { return (double)(bits >> 11) * 0x1.0p-53; }

#define INIT_TAG 0x696e6974ull /* sampler.cpp:12 */
#define FREE_TAG 0x66726565ull /* sampler.cpp:13 */

/* sampler.cpp:54-64 */
void so_init_soft_inputs(int batch, int cols, uint64_t seed, int restart, double* out) {
  for (int r = 0; r < batch; ++r)
    for (int c = 0; c < cols; ++c) {
      uint64_t xs[5] = {seed, INIT_TAG, (uint64_t)restart, (uint64_t)r, (uint64_t)c};
      out[(size_t)r * cols + c] = 2.0 * u01(so_hash_stream(xs, 5)) - 1.0;
    }
}

/* autodiff.cpp:12-16: clamp to +-40, then 1 / (1 + exp(-x)) in float. */
float so_sigmoid(float v) {
  float x = v < -40.0f ? -40.0f : (v > 40.0f ? 40.0f : v);
  return 1.0f / (1.0f + expf(-x));
}

/* autodiff.cpp:57-62 */
void so_embed(const float* v, int64_t n, float* p) {
  for (int64_t i = 0; i < n; ++i) p[i] = so_sigmoid(v[i]);
}

/* autodiff.cpp:64-152.  col_of_node[i] = P column of INPUT node i or -1
 * (map_input_columns, autodiff.cpp:38-53). */
void so_forward(int n_nodes, const int32_t* kind, const int32_t* a, const int32_t* b,
                const int32_t* col_of_node, int ncols, const float* p, int batch,
                int n_out, const int32_t* out_node, float* tape, float* y) {
  for (int i = 0; i < n_nodes; ++i) {
    float* o = tape + (size_t)i * batch;
    const float* va = a[i] >= 0 ? tape + (size_t)a[i] * batch : NULL;
    const float* vb = b[i] >= 0 ? tape + (size_t)b[i] * batch : NULL;
    switch (kind[i]) {
      case K_INPUT:
        for (int r = 0; r < batch; ++r)
          o[r] = col_of_node[i] < 0 ? 0.5f : p[(size_t)r * ncols + col_of_node[i]];
        break;
      case K_CONST0: for (int r = 0; r < batch; ++r) o[r] = 0.0f; break;
      case K_CONST1: for (int r = 0; r < batch; ++r) o[r] = 1.0f; break;
      case K_BUF: for (int r = 0; r < batch; ++r) o[r] = va[r]; break;
      case K_NOT: for (int r = 0; r < batch; ++r) o[r] = 1.0f - va[r]; break;
      case K_AND: for (int r = 0; r < batch; ++r) o[r] = va[r] * vb[r]; break;
      case K_OR:
        for (int r = 0; r < batch; ++r) o[r] = 1.0f - (1.0f - va[r]) * (1.0f - vb[r]);
        break;
      case K_XOR:
        for (int r = 0; r < batch; ++r) o[r] = (1.0f - va[r]) * vb[r] + va[r] * (1.0f - vb[r]);
        break;
      case K_XNOR:
        for (int r = 0; r < batch; ++r) o[r] = va[r] * vb[r] + (1.0f - va[r]) * (1.0f - vb[r]);
        break;
    }
  }
  if (y)
    for (int m = 0; m < n_out; ++m)
      for (int r = 0; r < batch; ++r) y[(size_t)r * n_out + m] = tape[(size_t)out_node[m] * batch + r];
}

/* autodiff.cpp:154-170 */
float so_loss(const float* y, int rows, int cols, const uint8_t* targets, float* per_row) {
  float total = 0.0f;
  for (int r = 0; r < rows; ++r) {
    float s = 0.0f;
    for (int m = 0; m < cols; ++m) {
      float d = y[(size_t)r * cols + m] - (float)targets[m];
      s += d * d;
    }
    if (per_row) per_row[r] = s;
    total += s; /* row-order sum, :168 */
  }
  return total;
}

/* autodiff.cpp:172-283 (push-style reverse sweep over node ids).  adj is
 * caller scratch of n_nodes * batch floats. */
void so_backward(int n_nodes, const int32_t* kind, const int32_t* a, const int32_t* b,
                 const int32_t* col_of_node, int ncols, const float* tape, int batch,
                 int n_out, const int32_t* out_node, const uint8_t* targets, const float* v,
                 float* dv, float* dp, float* adj) {
  memset(adj, 0, sizeof(float) * (size_t)n_nodes * batch);
  for (int m = 0; m < n_out; ++m) { /* seeds, :201-207 */
    const float* yy = tape + (size_t)out_node[m] * batch;
    float* g = adj + (size_t)out_node[m] * batch;
    float t = targets[m] ? 1.0f : 0.0f;
    for (int r = 0; r < batch; ++r) g[r] += 2.0f * (yy[r] - t);
  }
  for (int i = n_nodes - 1; i >= 0; --i) {
    const float* g = adj + (size_t)i * batch;
    float* ga = a[i] >= 0 ? adj + (size_t)a[i] * batch : NULL;
    float* gb = b[i] >= 0 ? adj + (size_t)b[i] * batch : NULL;
    const float* va = a[i] >= 0 ? tape + (size_t)a[i] * batch : NULL;
    const float* vb = b[i] >= 0 ? tape + (size_t)b[i] * batch : NULL;
    switch (kind[i]) {
      case K_INPUT: {
        int col = col_of_node[i];
        if (col < 0) break;
        for (int r = 0; r < batch; ++r) {
          float p = so_sigmoid(v[(size_t)r * ncols + col]);
          if (dp) dp[(size_t)r * ncols + col] = g[r];
          dv[(size_t)r * ncols + col] = g[r] * p * (1.0f - p);
        }
        break;
      }
      case K_CONST0:
      case K_CONST1: break;
      case K_BUF: for (int r = 0; r < batch; ++r) ga[r] += g[r]; break;
      case K_NOT: for (int r = 0; r < batch; ++r) ga[r] -= g[r]; break;
      case K_AND:
        for (int r = 0; r < batch; ++r) {
          ga[r] += g[r] * vb[r];
          gb[r] += g[r] * va[r];
        }
        break;
      case K_OR:
        for (int r = 0; r < batch; ++r) {
          ga[r] += g[r] * (1.0f - vb[r]);
          gb[r] += g[r] * (1.0f - va[r]);
        }
        break;
      case K_XOR:
        for (int r = 0; r < batch; ++r) {
          ga[r] += g[r] * (1.0f - 2.0f * vb[r]);
          gb[r] += g[r] * (1.0f - 2.0f * va[r]);
        }
        break;
      case K_XNOR:
        for (int r = 0; r < batch; ++r) {
          ga[r] += g[r] * (2.0f * vb[r] - 1.0f);
          gb[r] += g[r] * (2.0f * va[r] - 1.0f);
        }
        break;
    }
  }
}

/* autodiff.cpp:285-290 */
void so_gd_step(float* v, const float* g, int64_t n, float lr) {
  for (int64_t i = 0; i < n; ++i) v[i] -= lr * g[i];
}

/* autodiff.cpp:292-297 */
void so_harden(const float* v, int64_t n, uint8_t* bits) {
  for (int64_t i = 0; i < n; ++i) bits[i] = v[i] >= 0.0f ? 1 : 0;
}

/* circuit.cpp:124-146 for one row: node values from per-var PI values. */
static void eval_discrete(int n_nodes, const int32_t* kind, const int32_t* a, const int32_t* b,
                          const int32_t* var, const uint8_t* pi_vals, uint8_t* val) {
  for (int i = 0; i < n_nodes; ++i) {
    switch (kind[i]) {
      case K_INPUT: val[i] = pi_vals[var[i]]; break;
      case K_CONST0: val[i] = 0; break;
      case K_CONST1: val[i] = 1; break;
      case K_BUF: val[i] = val[a[i]]; break;
      case K_NOT: val[i] = !val[a[i]]; break;
      case K_AND: val[i] = val[a[i]] & val[b[i]]; break;
      case K_OR: val[i] = val[a[i]] | val[b[i]]; break;
      case K_XOR: val[i] = val[a[i]] ^ val[b[i]]; break;
      case K_XNOR: val[i] = !(val[a[i]] ^ val[b[i]]); break;
    }
  }
}

/* ---- SolutionSet (sampler.cpp:18-52): insertion-ordered full-key set ---- */
typedef struct {
  int words;
  int64_t size, cap;
  uint64_t* keys;  /* size * words, insertion order */
  int64_t* slots;  /* open addressing over key index, -1 empty */
  int64_t nslots;
} KeySet;

static uint64_t fnv(const uint64_t* k, int words) { /* sampler.cpp:28-36 */
  uint64_t h = 1469598103934665603ull;
  for (int i = 0; i < words; ++i) {
    h ^= k[i];
    h *= 1099511628211ull;
  }
  return h;
}

static void ks_rehash(KeySet* s, int64_t nslots) {
  free(s->slots);
  s->nslots = nslots;
  s->slots = (int64_t*)malloc(sizeof(int64_t) * nslots);
  for (int64_t i = 0; i < nslots; ++i) s->slots[i] = -1;
  for (int64_t k = 0; k < s->size; ++k) {
    uint64_t h = fnv(s->keys + k * s->words, s->words) & (uint64_t)(nslots - 1);
    while (s->slots[h] >= 0) h = (h + 1) & (uint64_t)(nslots - 1);
    s->slots[h] = k;
  }
}

static int ks_insert(KeySet* s, const uint64_t* key) {
  if ((s->size + 1) * 2 > s->nslots) ks_rehash(s, s->nslots ? s->nslots * 2 : 1024);
  uint64_t h = fnv(key, s->words) & (uint64_t)(s->nslots - 1);
  while (s->slots[h] >= 0) {
    if (memcmp(s->keys + s->slots[h] * s->words, key, sizeof(uint64_t) * s->words) == 0) return 0;
    h = (h + 1) & (uint64_t)(s->nslots - 1);
  }
  if (s->size == s->cap) {
    s->cap = s->cap ? s->cap * 2 : 1024;
    s->keys = (uint64_t*)realloc(s->keys, sizeof(uint64_t) * s->words * s->cap);
  }
  memcpy(s->keys + s->size * s->words, key, sizeof(uint64_t) * s->words);
  s->slots[h] = s->size++;
  return 1;
}

/* ---- run_impl<float> (sampler.cpp:89-194) ---- */
typedef struct {
  /* inputs (borrowed) */
  int n_nodes;
  const int32_t *kind, *a, *b, *var;
  int num_vars, max_var;
  const int32_t* node_of_var; /* max_var + 1 */
  int n_out;
  const int32_t* out_var;
  const uint8_t* out_tgt;
  int ncpi, nucpi;
  const int32_t *cpi, *ucpi;
  int64_t n_clauses;
  const int64_t* clause_ptr;
  const int32_t* clause_lit;
  /* results */
  KeySet sols;
  int64_t attempts;
  int restarts, timed_out;
  double wall;
  double* loss_trace;
  int64_t n_loss, cap_loss;
  int64_t* new_unique;
  int64_t n_nu, cap_nu;
} SoRun;

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

static void push_loss(SoRun* r, double x) {
  if (r->n_loss == r->cap_loss) {
    r->cap_loss = r->cap_loss ? 2 * r->cap_loss : 64;
    r->loss_trace = (double*)realloc(r->loss_trace, sizeof(double) * r->cap_loss);
  }
  r->loss_trace[r->n_loss++] = x;
}

static void push_nu(SoRun* r, int64_t x) {
  if (r->n_nu == r->cap_nu) {
    r->cap_nu = r->cap_nu ? 2 * r->cap_nu : 64;
    r->new_unique = (int64_t*)realloc(r->new_unique, sizeof(int64_t) * r->cap_nu);
  }
  r->new_unique[r->n_nu++] = x;
}

/* unsat != 0 reproduces the early return at sampler.cpp:105-110. */
void* so_run(int n_nodes, const int32_t* kind, const int32_t* a, const int32_t* b,
             const int32_t* var, int num_vars, int max_var, const int32_t* node_of_var, int n_out,
             const int32_t* out_var, const uint8_t* out_tgt, int ncpi, const int32_t* cpi,
             int nucpi, const int32_t* ucpi, int64_t n_clauses, const int64_t* clause_ptr,
             const int32_t* clause_lit, int unsat, int batch, int iterations, double lr,
             uint64_t seed, int64_t max_solutions, double timeout_s, int restart_policy) {
  SoRun* R = (SoRun*)calloc(1, sizeof(SoRun));
  R->n_nodes = n_nodes; R->kind = kind; R->a = a; R->b = b; R->var = var;
  R->num_vars = num_vars; R->max_var = max_var; R->node_of_var = node_of_var;
  R->n_out = n_out; R->out_var = out_var; R->out_tgt = out_tgt;
  R->ncpi = ncpi; R->nucpi = nucpi; R->cpi = cpi; R->ucpi = ucpi;
  R->n_clauses = n_clauses; R->clause_ptr = clause_ptr; R->clause_lit = clause_lit;
  R->sols.words = (num_vars + 63) / 64;
  double t0 = now_s();
  if (unsat) {
    R->wall = now_s() - t0;
    return R;
  }

  int32_t* col_of_node = (int32_t*)malloc(sizeof(int32_t) * n_nodes);
  for (int i = 0; i < n_nodes; ++i) col_of_node[i] = -1;
  for (int j = 0; j < ncpi; ++j) col_of_node[node_of_var[cpi[j]]] = j;
  int32_t* out_node = (int32_t*)malloc(sizeof(int32_t) * (n_out ? n_out : 1));
  for (int m = 0; m < n_out; ++m) out_node[m] = node_of_var[out_var[m]];

  size_t nv = (size_t)batch * ncpi;
  double* v0 = (double*)malloc(sizeof(double) * (nv ? nv : 1));
  float* v = (float*)malloc(sizeof(float) * (nv ? nv : 1));
  float* p = (float*)malloc(sizeof(float) * (nv ? nv : 1));
  float* dv = (float*)malloc(sizeof(float) * (nv ? nv : 1));
  uint8_t* bits = (uint8_t*)malloc(nv ? nv : 1);
  float* tape = (float*)malloc(sizeof(float) * (size_t)n_nodes * batch);
  float* adj = (float*)malloc(sizeof(float) * (size_t)n_nodes * batch);
  float* y = (float*)malloc(sizeof(float) * (size_t)batch * (n_out ? n_out : 1));
  uint8_t* pi_vals = (uint8_t*)malloc(max_var + 1);
  uint8_t* val = (uint8_t*)malloc(n_nodes ? n_nodes : 1);
  uint64_t* key = (uint64_t*)malloc(sizeof(uint64_t) * (R->sols.words ? R->sols.words : 1));
  memset(pi_vals, 0xFF, max_var + 1);

#define QUOTA_MET() (max_solutions > 0 && R->sols.size >= max_solutions)
#define OUT_OF_TIME() (timeout_s > 0.0 && now_s() - t0 >= timeout_s)

  for (int restart = 0;; ++restart) {
    so_init_soft_inputs(batch, ncpi, seed, restart, v0);
    for (size_t i = 0; i < nv; ++i) v[i] = (float)v0[i];
    int64_t before = R->sols.size;
    for (int iter = 0; iter <= iterations; ++iter) {
      if (iter > 0) {
        if (QUOTA_MET()) break;
        if (OUT_OF_TIME()) {
          R->timed_out = 1;
          break;
        }
        so_embed(v, (int64_t)nv, p);
        so_forward(n_nodes, kind, a, b, col_of_node, ncpi, p, batch, n_out, out_node, tape, y);
        float total = so_loss(y, batch, n_out, out_tgt, NULL);
        push_loss(R, (double)total / batch);
        so_backward(n_nodes, kind, a, b, col_of_node, ncpi, tape, batch, n_out, out_node, out_tgt,
                    v, dv, NULL, adj);
        so_gd_step(v, dv, (int64_t)nv, (float)lr);
      }
      /* harvest (sampler.cpp:124-153) */
      so_harden(v, (int64_t)nv, bits);
      int64_t added = 0;
      for (int r = 0; r < batch; ++r) {
        if (QUOTA_MET()) break;
        for (int j = 0; j < ncpi; ++j) pi_vals[cpi[j]] = bits[(size_t)r * ncpi + j];
        for (int k = 0; k < nucpi; ++k) {
          uint64_t xs[6] = {seed, FREE_TAG, (uint64_t)restart, (uint64_t)iter, (uint64_t)r,
                            (uint64_t)k};
          pi_vals[ucpi[k]] = (uint8_t)(so_hash_stream(xs, 6) & 1);
        }
        eval_discrete(n_nodes, kind, a, b, var, pi_vals, val);
        R->attempts++;
        int hit = 1;
        for (int m = 0; m < n_out && hit; ++m)
          if (val[out_node[m]] != (out_tgt[m] ? 1 : 0)) hit = 0;
        if (!hit) continue;
        int sat = 1; /* eval_cnf, cnf.cpp:129-147 */
        for (int64_t c = 0; c < n_clauses && sat; ++c) {
          int any = 0;
          for (int64_t l = clause_ptr[c]; l < clause_ptr[c + 1] && !any; ++l) {
            int lit = clause_lit[l];
            int vv = lit < 0 ? -lit : lit;
            int x = val[node_of_var[vv]];
            any = lit < 0 ? !x : x;
          }
          sat = any;
        }
        if (!sat) continue;
        memset(key, 0, sizeof(uint64_t) * R->sols.words); /* dedupe_key, :18-26 */
        for (int vv = 1; vv <= num_vars; ++vv)
          if (val[node_of_var[vv]]) key[(vv - 1) / 64] |= 1ull << ((vv - 1) % 64);
        if (ks_insert(&R->sols, key)) ++added;
      }
      push_nu(R, added);
    }
    if (QUOTA_MET() || R->timed_out) break;
    if (restart_policy != 1) break;
    if (R->sols.size == before) break;
    if (restart >= 1000) break;
    if (OUT_OF_TIME()) {
      R->timed_out = 1;
      break;
    }
    R->restarts = restart + 1;
  }
  R->wall = now_s() - t0;
  free(col_of_node); free(out_node); free(v0); free(v); free(p); free(dv); free(bits);
  free(tape); free(adj); free(y); free(pi_vals); free(val); free(key);
  return R;
}

/* out: unique, attempts, restarts, timed_out, n_loss, n_new_unique, words */
void so_run_stats(void* h, int64_t* out, double* wall) {
  SoRun* R = (SoRun*)h;
  out[0] = R->sols.size;
  out[1] = R->attempts;
  out[2] = R->restarts;
  out[3] = R->timed_out;
  out[4] = R->n_loss;
  out[5] = R->n_nu;
  out[6] = R->sols.words;
  *wall = R->wall;
}

void so_run_traces(void* h, double* loss, int64_t* nu) {
  SoRun* R = (SoRun*)h;
  if (R->n_loss) memcpy(loss, R->loss_trace, sizeof(double) * R->n_loss);
  if (R->n_nu) memcpy(nu, R->new_unique, sizeof(int64_t) * R->n_nu);
}

void so_run_keys(void* h, uint64_t* keys) {
  SoRun* R = (SoRun*)h;
  if (R->sols.size) memcpy(keys, R->sols.keys, sizeof(uint64_t) * R->sols.words * R->sols.size);
}

void so_run_free(void* h) {
  SoRun* R = (SoRun*)h;
  free(R->sols.keys); free(R->sols.slots); free(R->loss_trace); free(R->new_unique);
  free(R);
}

/* eval_cnf on a packed key (vars 1..num_vars, dedupe_key layout): the host
 * re-verifier used by tests. */
int so_check_key(int64_t n_clauses, const int64_t* clause_ptr, const int32_t* clause_lit,
                 const uint64_t* key) {
  for (int64_t c = 0; c < n_clauses; ++c) {
    int any = 0;
    for (int64_t l = clause_ptr[c]; l < clause_ptr[c + 1] && !any; ++l) {
      int lit = clause_lit[l];
      int vv = lit < 0 ? -lit : lit;
      int x = (int)((key[(vv - 1) / 64] >> ((vv - 1) % 64)) & 1);
      any = lit < 0 ? !x : x;
    }
    if (!any) return 0;
  }
  return 1;
}

/* glibc expf over a range of floats: used by the device-sigmoid parity test. */
void so_expf_range(const float* x, int64_t n, float* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = expf(x[i]);
}
