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

namespace tq {

enum OpndKind : uint8_t {
  K_NONE = 0,
  K_COL_I64,
  K_COL_DEC,
  K_COL_F64,
  K_COL_BOOL,
  K_TMP_I,
  K_TMP_F,
  K_TMP_B,
  K_LIT_I,
  K_LIT_F,
  K_LIT_B,
};

enum OpCode : uint8_t {
  OP_ADD_I = 0,
  OP_SUB_I,
  OP_MUL_I,
  OP_ADD_F,
  OP_SUB_F,
  OP_MUL_F,
  OP_CMP_I,
  OP_CMP_F,
  OP_CMP_B,
  OP_AND,
  OP_OR,
  OP_NOT,
};

// 16-byte instruction.  For I ops fa/fb are literal indices of 10^k rescale
// factors (0xff = none) and `wrap` truncates to int64.  For F ops fa/fb carry
// the decimal scale used to convert an I operand to double.
struct DInstr {
  uint8_t op, sub, dst, ak, bk, fa, fb, wrap;
  uint16_t a, b;
  uint16_t _pad[2];
};
static_assert(sizeof(DInstr) == 16, "instr size");

struct DLit {
  uint64_t lo, hi;  // int128 (I) or bool (lo)
  double f;
  uint32_t valid;
  uint32_t _pad;
};
static_assert(sizeof(DLit) == 32, "lit size");

// Result class of a compiled expression.
enum Cls : uint8_t { C_I = 0, C_D = 1, C_F = 2, C_B = 3, C_S = 4 };

struct Operand {
  uint8_t kind = K_NONE;
  uint16_t idx = 0;
  uint8_t cls = C_I;  // value class
  uint8_t scale = 0;  // decimal scale (C_D)
  bool maybe_null = false;
};

constexpr int kMaxValueSlots = 16;
constexpr int kMaxBoolSlots = 16;
constexpr int kMaxStaged = 24;
constexpr int kMaxInstr = 128;
constexpr int kMaxLits = 64;

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
