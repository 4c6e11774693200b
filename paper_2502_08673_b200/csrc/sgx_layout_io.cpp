// On-disk levelized layout: the compiled programs of a
// circuit (sgx_layout.hpp Layout, minus the on-demand parity-tap program)
// written once and read back by later processes instead of being rebuilt --
// the B200 counterpart of the reference CLI's circuit-JSON cache
// (tools/satgrad_main.cpp:137-184), one level further down: the JSON cache
// saves extraction, this saves extraction's consumer, the layout compiler.
//
// Format: "SGXLAYT" + version byte, the descriptor key (sgx_api.cpp
// layoutcache::key: a hash of every descriptor array and the layout's
// environment knobs), then every field in layout_fields() order -- scalars
// raw, vectors as a u64 count + raw elements -- then the key again.  Readers
// reject any mismatch (magic, version, key, truncation) and rebuild.
#include <cstdio>
#include <cstring>
#include <string>
#include <type_traits>
#include <vector>

#include "sgx_layout.hpp"

namespace sgx {

namespace {

constexpr char kMagic[8] = {'S', 'G', 'X', 'L', 'A', 'Y', 'T', 5};  // 3: forward read hints for far next reads; 4: backward kRYKeep; 5: split backward passes

// Every persisted field, in file order.  Adding a field to SoftProgram or
// Layout changes their size and trips the static_asserts below, so this list
// cannot silently fall behind the structs.
template <class P, class F>
void program_fields(P& p, F&& f) {
  f(p.n_rows); f(p.n_set); f(p.n_levels); f(p.n_edges);
  f(p.row_of_node); f(p.node_of_row); f(p.fwd); f(p.fwd_lvl); f(p.rec); f(p.rec_lvl);
  f(p.dead); f(p.dead_lvl); f(p.sblk); f(p.sblk_lvl); f(p.srec_lvl); f(p.tail_dead);
  f(p.fblk); f(p.fblk_lvl); f(p.fblk_max); f(p.oc_fwd); f(p.oc_rec); f(p.oc_fwd_lvl);
  f(p.oc_rec_lvl); f(p.oc_col_slot); f(p.oc_adj_slots); f(p.sblk_max); f(p.out_enc);
  f(p.col_row); f(p.virt_base); f(p.virt_neg);
}
template <class L, class F>
void layout_fields(L& x, F&& f) {
  f(x.n_nodes); f(x.num_vars); f(x.max_var);
  f(x.kind); f(x.a); f(x.b); f(x.var); f(x.node_of_var); f(x.out_var); f(x.out_node); f(x.out_tgt);
  f(x.cpi); f(x.ucpi); f(x.clause_ptr); f(x.clause_lit); f(x.hclause_ptr); f(x.hclause_lit);
  f(x.n_implied); f(x.clause_implied); f(x.unsat); f(x.level);
  program_fields(x.cone, f);  // (x.full: the parity-tap program, built on demand, is not persisted)
  f(x.n_bit_rows); f(x.bit_row_of_node); f(x.bit_ops); f(x.bit_lvl_ptr); f(x.cpi_bit_row);
  f(x.ucpi_bit_row); f(x.out_bit_row); f(x.clause_ptr32); f(x.clause_enc); f(x.key_words);
  f(x.key_bit_row); f(x.fb_rows); f(x.fb_ops); f(x.fb_lvl_ptr); f(x.fb_cpi_row); f(x.fb_ucpi_row);
  f(x.fb_out_enc); f(x.fb_key_enc); f(x.fb_cnf_steps); f(x.fb_cnf4); f(x.lb_slots); f(x.lb_levels);
  f(x.lb_n_spill); f(x.lb_ops); f(x.lb_op_ptr); f(x.lb_chk); f(x.lb_chk_ptr); f(x.lb_big_lits);
  f(x.lb_cpi); f(x.lb_ucpi); f(x.lb_key_enc); f(x.lw_ops); f(x.lw_iters);
}
static_assert(sizeof(SoftProgram) == 592, "SoftProgram changed: update program_fields");
static_assert(sizeof(Layout) == 2256, "Layout changed: update layout_fields");

struct Writer {
  FILE* fp;
  bool ok = true;
  void raw(const void* p, size_t n) {
    if (ok && n && std::fwrite(p, 1, n, fp) != n) ok = false;
  }
  template <class T>
  void operator()(const T& v) {
    if constexpr (std::is_arithmetic_v<T>) {
      raw(&v, sizeof(T));
    } else {
      const uint64_t n = v.size();
      raw(&n, sizeof(n));
      raw(v.data(), n * sizeof(typename T::value_type));
    }
  }
};
struct Reader {
  FILE* fp;
  bool ok = true;
  void raw(void* p, size_t n) {
    if (ok && n && std::fread(p, 1, n, fp) != n) ok = false;
  }
  template <class T>
  void operator()(T& v) {
    if constexpr (std::is_arithmetic_v<T>) {
      raw(&v, sizeof(T));
    } else {
      uint64_t n = 0;
      raw(&n, sizeof(n));
      if (!ok || n > (uint64_t{1} << 34) / sizeof(typename T::value_type)) {
        ok = false;
        return;
      }
      v.resize(n);
      raw(v.data(), n * sizeof(typename T::value_type));
    }
  }
};

struct Hasher {
  uint64_t h = 0x6c61796f75742121ull;
  void raw(const void* p, size_t n) {
    const unsigned char* c = static_cast<const unsigned char*>(p);
    for (size_t i = 0; i < n; ++i) h = (h ^ c[i]) * 0x100000001b3ull;
  }
  template <class T>
  void operator()(const T& v) {
    if constexpr (std::is_arithmetic_v<T>) {
      raw(&v, sizeof(T));
    } else {
      const uint64_t n = v.size();
      raw(&n, sizeof(n));
      raw(v.data(), n * sizeof(typename T::value_type));
    }
  }
};

}  // namespace

uint64_t layout_digest(const Layout& L) {
  Hasher h;
  layout_fields(L, h);
  return h.h;
}

bool save_layout(const Layout& L, const std::string& path, uint64_t key) {
  const std::string tmp = path + ".tmp" + std::to_string(reinterpret_cast<uintptr_t>(&L));
  FILE* fp = std::fopen(tmp.c_str(), "wb");
  if (!fp) return false;
  Writer w{fp};
  w.raw(kMagic, sizeof(kMagic));
  w(key);
  layout_fields(L, w);
  w(key);
  const bool ok = w.ok && std::fclose(fp) == 0;
  if (!ok || std::rename(tmp.c_str(), path.c_str()) != 0) {  // atomic publish
    std::remove(tmp.c_str());
    return false;
  }
  return true;
}

bool load_layout(Layout* L, const std::string& path, uint64_t key) {
  FILE* fp = std::fopen(path.c_str(), "rb");
  if (!fp) return false;
  Reader r{fp};
  char magic[sizeof(kMagic)];
  r.raw(magic, sizeof(magic));
  uint64_t k0 = 0, k1 = 0;
  r(k0);
  Layout x;
  if (r.ok && std::memcmp(magic, kMagic, sizeof(kMagic)) == 0 && k0 == key) {
    layout_fields(x, r);
    r(k1);
  }
  const bool at_end = r.ok && std::fgetc(fp) == EOF;
  std::fclose(fp);
  if (!r.ok || !at_end || k0 != key || k1 != key) return false;
  *L = std::move(x);
  return true;
}

}  // namespace sgx
