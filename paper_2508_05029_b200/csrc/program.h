// program.h — the register-machine form of Expr executed by
// the warp-tile interpreter in pipeline.cu, and the host-side compiler that
// lowers tq_expr trees (prefix order) into it.
//
// Values are per-row lanes of a warp; a "slot" is per-warp shared memory:
//   value slots  (I: int128, F: double)  16 B x rows-per-warp
//   bool slots   two 32-bit masks (value, validity) per 32 rows
// Operands name a staged column, a slot, or a literal.  Typing and promotion
// follow DESIGN.md §3 (shared decisions with the oracle).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/tq_types.h"

#include "program_types.h"

namespace tq {

struct ColumnDesc {
  uint8_t kind, precision, scale;
  bool has_validity;
};

struct CompileError {
  int status;
  std::string msg;
};

class ProgramBuilder {
 public:
  explicit ProgramBuilder(std::vector<ColumnDesc> schema) : schema_(std::move(schema)) {}
  // Register an expression root; returns a handle resolved after finish().
  int add_root(const tq_expr& e);
  // Register a plain column reference (staged, no instruction).
  int add_column(uint32_t col);
  // Roots registered so far belong to the predicate prefix.
  void end_predicate() { pred_roots_ = (int)roots_.size(); }
  void finish();

  const Operand& root(int h) const { return root_ops_[h]; }
  const std::vector<DInstr>& code() const { return code_; }
  const std::vector<DLit>& lits() const { return lits_; }
  const std::vector<uint32_t>& staged() const { return staged_; }  // staged slot -> input column
  int n_pred_instr() const { return n_pred_instr_; }
  int value_slots() const { return max_v_; }
  int bool_slots() const { return max_b_; }
  int staged_index(uint32_t col);  // stage a column, return staged slot
  // Bitmask of staged columns that the given root handles depend on.
  uint32_t column_deps(const std::vector<int>& roots) const;

 private:
  struct Node {
    int tag, op;
    int a = -1, b = -1;
    uint32_t col = 0;
    uint8_t cls = C_I, scale = 0;
    bool lit_null = false;
    uint64_t lo = 0, hi = 0;  // literal bits
    double f = 0;
    bool maybe_null = false;
    int uses = 0;
    Operand res;
    bool done = false;
  };
  int parse(const tq_expr& e, uint32_t& pos);
  int intern(Node n);
  Operand gen(int id);
  void release(const Operand& o);
  uint16_t lit_index(const DLit& l);
  uint8_t factor_lit(int k);

  std::vector<ColumnDesc> schema_;
  std::vector<Node> nodes_;
  std::vector<int> roots_;  // node ids (or -1-col for plain columns)
  std::vector<Operand> root_ops_;
  int pred_roots_ = 0;
  std::vector<DInstr> code_;
  std::vector<DLit> lits_;
  std::vector<uint32_t> staged_;
  int n_pred_instr_ = 0;
  bool free_v_[kMaxValueSlots] = {};
  bool free_b_[kMaxBoolSlots] = {};
  int max_v_ = 0, max_b_ = 0;
};

}  // namespace tq
