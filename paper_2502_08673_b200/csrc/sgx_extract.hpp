// Native circuit extraction + build (see sgx_extract.cpp).
#pragma once

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

namespace sgx::ext {

// ExtractionResult (extract.hpp:31-41) + the built Circuit's node arrays
// (circuit.hpp:24-40, GateKind codes of sgx_gate_kind).
struct Result {
  int num_vars = 0;
  std::vector<int> pi, iv, aux;
  std::vector<std::pair<int, bool>> po;
  bool unsat = false;
  std::string unsat_note;
  int64_t n_defs = 0;
  std::vector<int> kind, a, b, var;
};

// CNF as CSR (clause_ptr[n_clauses + 1], DIMACS literals).  Throws
// std::invalid_argument like the reference.
void extract_build(int num_vars, const int32_t* clause_ptr, const int32_t* clause_lit, int64_t n_clauses,
                   int complement_cap, int minimize_cap, Result& out);

}  // namespace sgx::ext
