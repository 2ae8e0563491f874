// program.cpp — lowers Expr trees (prefix-serialized
// tq_expr_node[]) into the warp-tile register machine of program.h.
//
// Typing (same decisions as the CPU oracle, implemented
// independently):
//   Arith: Float64 if either side is Float64; else Decimal if either side is
//          Decimal (+,- : scale max(sa,sb) with 10^k rescale; * : scale sa+sb);
//          else Int64 (two's-complement wrap).
//   Compare: numeric vs numeric (rescaled int128 or double), Bool vs Bool.
//   And / Or / Not on Bool.  Any null operand -> null.
// Common subexpressions are shared (hash-consing), temp slots are recycled
// once their last consumer has been emitted, and predicate roots are emitted
// first so the interpreter can skip the rest of a warp-tile whose rows all
// failed the predicate.
#include "program.h"

#include <algorithm>
#include <cstring>
#include <map>
#include <tuple>

namespace tq {

namespace {
[[noreturn]] void bad(const std::string& m) { throw CompileError{TQ_INVALID_PLAN, m}; }
uint8_t cls_of_kind(uint8_t kind) {
  switch (kind) {
    case TQ_INT64: return C_I;
    case TQ_DECIMAL: return C_D;
    case TQ_FLOAT64: return C_F;
    case TQ_BOOL: return C_B;
    case TQ_UTF8: return C_S;
  }
  bad("bad type kind");
}
bool numeric(uint8_t c) { return c == C_I || c == C_D || c == C_F; }
}  // namespace

int ProgramBuilder::staged_index(uint32_t col) {
  for (size_t i = 0; i < staged_.size(); ++i)
    if (staged_[i] == col) return (int)i;
  if (staged_.size() >= (size_t)kMaxStaged) bad("too many referenced columns");
  staged_.push_back(col);
  return (int)staged_.size() - 1;
}

int ProgramBuilder::intern(Node n) {
  // structural key for common-subexpression sharing
  static_assert(sizeof(double) == 8, "");
  for (size_t i = 0; i < nodes_.size(); ++i) {
    const Node& m = nodes_[i];
    if (m.tag == n.tag && m.op == n.op && m.a == n.a && m.b == n.b && m.col == n.col && m.cls == n.cls &&
        m.scale == n.scale && m.lit_null == n.lit_null && m.lo == n.lo && m.hi == n.hi &&
        std::memcmp(&m.f, &n.f, 8) == 0)
      return (int)i;
  }
  nodes_.push_back(n);
  return (int)nodes_.size() - 1;
}

int ProgramBuilder::parse(const tq_expr& e, uint32_t& pos) {
  if (pos >= e.len) bad("truncated expression");
  const tq_expr_node& x = e.nodes[pos++];
  Node n;
  n.tag = x.tag;
  n.op = x.op;
  switch (x.tag) {
    case TQ_EX_COL: {
      if (x.column >= schema_.size()) bad("column out of range");
      const ColumnDesc& c = schema_[x.column];
      n.col = x.column;
      n.cls = cls_of_kind(c.kind);
      if (n.cls == C_S) bad("utf8 expressions are not supported on the GPU path");
      n.scale = c.kind == TQ_DECIMAL ? c.scale : 0;
      n.maybe_null = c.has_validity;
      break;
    }
    case TQ_EX_LIT:
      n.cls = cls_of_kind(x.kind);
      if (n.cls == C_S) bad("utf8 literals unsupported");
      n.scale = x.kind == TQ_DECIMAL ? x.scale : 0;
      n.lit_null = x.is_null != 0;
      n.maybe_null = n.lit_null;
      if (!n.lit_null) {
        if (n.cls == C_F) std::memcpy(&n.f, &x.lo, 8);
        else if (n.cls == C_B) n.lo = x.lo != 0;
        else if (n.cls == C_D) { n.lo = x.lo; n.hi = x.hi; }
        else { n.lo = x.lo; n.hi = (int64_t)x.lo < 0 ? ~0ull : 0; }
      }
      break;
    case TQ_EX_ARITH: case TQ_EX_CMP: case TQ_EX_AND: case TQ_EX_OR: {
      n.a = parse(e, pos);
      n.b = parse(e, pos);
      const Node &A = nodes_[n.a], &B = nodes_[n.b];
      n.maybe_null = A.maybe_null || B.maybe_null;
      if (x.tag == TQ_EX_ARITH) {
        if (x.op > TQ_MUL) bad("bad arith op");
        if (!numeric(A.cls) || !numeric(B.cls)) bad("arith on non-numeric");
        if (A.cls == C_F || B.cls == C_F) n.cls = C_F;
        else if (A.cls == C_D || B.cls == C_D) {
          n.cls = C_D;
          int s = x.op == TQ_MUL ? A.scale + B.scale : std::max(A.scale, B.scale);
          if (s > 38) bad("decimal scale overflow");
          n.scale = (uint8_t)s;
        } else n.cls = C_I;
      } else if (x.tag == TQ_EX_CMP) {
        if (x.op > TQ_GT) bad("bad compare op");
        bool ok = (numeric(A.cls) && numeric(B.cls)) || (A.cls == C_B && B.cls == C_B);
        if (!ok) bad("compare of incompatible types");
        n.cls = C_B;
      } else {
        if (A.cls != C_B || B.cls != C_B) bad("logic on non-bool");
        n.cls = C_B;
      }
      break;
    }
    case TQ_EX_NOT:
      n.a = parse(e, pos);
      if (nodes_[n.a].cls != C_B) bad("not on non-bool");
      n.maybe_null = nodes_[n.a].maybe_null;
      n.cls = C_B;
      break;
    default:
      bad("unknown expression tag");
  }
  return intern(n);
}

int ProgramBuilder::add_root(const tq_expr& e) {
  uint32_t pos = 0;
  int id = parse(e, pos);
  if (pos != e.len) bad("trailing expression nodes");
  roots_.push_back(id);
  return (int)roots_.size() - 1;
}

int ProgramBuilder::add_column(uint32_t col) {
  if (col >= schema_.size()) bad("column out of range");
  tq_expr_node x{};
  x.tag = TQ_EX_COL;
  x.column = col;
  tq_expr e{&x, 1, 0};
  const ColumnDesc& c = schema_[col];
  if (c.kind == TQ_UTF8) bad("utf8 columns are not supported on the GPU path");
  return add_root(e);
}

uint16_t ProgramBuilder::lit_index(const DLit& l) {
  for (size_t i = 0; i < lits_.size(); ++i)
    if (std::memcmp(&lits_[i], &l, sizeof(DLit)) == 0) return (uint16_t)i;
  if (lits_.size() >= (size_t)kMaxLits) bad("too many literals");
  lits_.push_back(l);
  return (uint16_t)(lits_.size() - 1);
}

uint8_t ProgramBuilder::factor_lit(int k) {
  if (k <= 0) return 0xff;
  unsigned __int128 v = 1;
  for (int i = 0; i < k; ++i) v *= 10u;
  DLit l{};
  l.lo = (uint64_t)v;
  l.hi = (uint64_t)(v >> 64);
  l.valid = 1;
  return (uint8_t)lit_index(l);
}

void ProgramBuilder::release(const Operand& o) {
  if (o.kind == K_TMP_I || o.kind == K_TMP_F) free_v_[o.idx] = true;
  if (o.kind == K_TMP_B) free_b_[o.idx] = true;
}

Operand ProgramBuilder::gen(int id) {
  Node& n = nodes_[id];
  if (n.done) return n.res;
  Operand r;
  r.cls = n.cls;
  r.scale = n.scale;
  r.maybe_null = n.maybe_null;
  if (n.tag == TQ_EX_COL) {
    const ColumnDesc& c = schema_[n.col];
    r.kind = c.kind == TQ_INT64 ? K_COL_I64 : c.kind == TQ_DECIMAL ? K_COL_DEC : c.kind == TQ_FLOAT64 ? K_COL_F64
                                                                                                     : K_COL_BOOL;
    r.idx = (uint16_t)staged_index(n.col);
  } else if (n.tag == TQ_EX_LIT) {
    DLit l{};
    l.valid = n.lit_null ? 0 : 1;
    if (n.cls == C_F) { l.f = n.f; r.kind = K_LIT_F; }
    else if (n.cls == C_B) { l.lo = n.lo; r.kind = K_LIT_B; }
    else { l.lo = n.lo; l.hi = n.hi; r.kind = K_LIT_I; }
    r.idx = lit_index(l);
  } else {
    Operand a = gen(n.a);
    Operand b = n.b >= 0 ? gen(n.b) : Operand{};
    // children consumed: release temps whose last consumer this is
    Node& A = nodes_[n.a];
    if (--A.uses == 0) release(a);
    if (n.b >= 0) {
      Node& B = nodes_[n.b];
      if (--B.uses == 0) release(b);
    }
    DInstr in{};
    in.ak = a.kind; in.a = a.idx;
    in.bk = b.kind; in.b = b.idx;
    in.fa = in.fb = 0xff;
    if (n.tag == TQ_EX_ARITH) {
      if (n.cls == C_F) {
        in.op = (uint8_t)(OP_ADD_F + n.op);
        in.fa = a.cls == C_F ? 0 : a.scale;
        in.fb = b.cls == C_F ? 0 : b.scale;
      } else {
        in.op = (uint8_t)(OP_ADD_I + n.op);
        if (n.cls == C_D && n.op != TQ_MUL) {
          in.fa = factor_lit(n.scale - a.scale);
          in.fb = factor_lit(n.scale - b.scale);
        }
        in.wrap = n.cls == C_I;
      }
    } else if (n.tag == TQ_EX_CMP) {
      in.sub = (uint8_t)n.op;
      if (a.cls == C_F || b.cls == C_F) {
        in.op = OP_CMP_F;
        in.fa = a.cls == C_F ? 0 : a.scale;
        in.fb = b.cls == C_F ? 0 : b.scale;
      } else if (a.cls == C_B) {
        in.op = OP_CMP_B;
      } else {
        in.op = OP_CMP_I;
        int s = std::max(a.scale, b.scale);
        in.fa = factor_lit(s - a.scale);
        in.fb = factor_lit(s - b.scale);
      }
    } else if (n.tag == TQ_EX_AND) in.op = OP_AND;
    else if (n.tag == TQ_EX_OR) in.op = OP_OR;
    else in.op = OP_NOT;
    // destination slot
    if (n.cls == C_B) {
      int s = -1;
      for (int i = 0; i < max_b_; ++i) if (free_b_[i]) { s = i; break; }
      if (s < 0) { if (max_b_ >= kMaxBoolSlots) bad("expression too complex (bool slots)"); s = max_b_++; }
      free_b_[s] = false;
      r.kind = K_TMP_B;
      r.idx = (uint16_t)s;
    } else {
      int s = -1;
      for (int i = 0; i < max_v_; ++i) if (free_v_[i]) { s = i; break; }
      if (s < 0) { if (max_v_ >= kMaxValueSlots) bad("expression too complex (value slots)"); s = max_v_++; }
      free_v_[s] = false;
      r.kind = n.cls == C_F ? K_TMP_F : K_TMP_I;
      r.idx = (uint16_t)s;
    }
    in.dst = (uint8_t)r.idx;
    if (code_.size() >= (size_t)kMaxInstr) bad("expression too long");
    code_.push_back(in);
  }
  n.res = r;
  n.done = true;
  return r;
}

uint32_t ProgramBuilder::column_deps(const std::vector<int>& roots) const {
  uint32_t vdep[kMaxValueSlots] = {}, bdep[kMaxBoolSlots] = {};
  auto opnd = [&](uint8_t k, uint16_t idx) -> uint32_t {
    switch (k) {
      case K_COL_I64: case K_COL_DEC: case K_COL_F64: case K_COL_BOOL: return 1u << idx;
      case K_TMP_I: case K_TMP_F: return vdep[idx];
      case K_TMP_B: return bdep[idx];
      default: return 0;
    }
  };
  for (const DInstr& in : code_) {
    uint32_t m = opnd(in.ak, in.a) | (in.op == OP_NOT ? 0u : opnd(in.bk, in.b));
    bool b = in.op >= OP_CMP_I;
    if (b) bdep[in.dst] = m;
    else vdep[in.dst] = m;
  }
  uint32_t out = 0;
  for (int h : roots) out |= opnd(root_ops_[h].kind, root_ops_[h].idx);
  return out;
}

void ProgramBuilder::finish() {
  for (auto& n : nodes_) n.uses = 0;
  for (auto& n : nodes_) {
    if (n.a >= 0) nodes_[n.a].uses++;
    if (n.b >= 0) nodes_[n.b].uses++;
  }
  for (int id : roots_) nodes_[id].uses += 1 << 20;  // pinned until the sink reads them
  root_ops_.resize(roots_.size());
  for (int i = 0; i < (int)roots_.size(); ++i) {
    root_ops_[i] = gen(roots_[i]);
    if (i + 1 == pred_roots_) n_pred_instr_ = (int)code_.size();
  }
  if (pred_roots_ == 0) n_pred_instr_ = 0;
}

}  // namespace tq
