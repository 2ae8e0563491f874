// jit.cu — specialises a pipeline launch: the typed register-machine program
// (program.h) that the interpreter would run is lowered to straight-line CUDA
// C++ (one SSA value per instruction, staged-column offsets, literals, key and
// accumulator layouts baked in) and compiled by NVRTC for sm_100a into the
// same kernel skeleton (kernel_common.cuh) the interpreter uses.  Kernels are
// cached per generated source for the life of the process; any failure falls
// back to the ahead-of-time interpreter kernel (pipeline.cu) — both run on the
// GPU, there is no CPU path.
#include <dlfcn.h>

#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <cstring>
#include <map>
#include <mutex>
#include <sstream>
#include <string>
#include <vector>

#include "ctx.h"
#include "device.cuh"
#include "pipeline.h"

namespace tq {

cudaError_t launch_interp(int sink, const PipeParams& p, u32 smem_bytes, u32 grid, cudaStream_t st);

// ------------------------------------------------------------------ NVRTC (dlopen'd)
namespace {

typedef int nvrtcResult_t;
typedef struct _nvrtcProgram* nvrtcProgram_t;
struct Nvrtc {
  bool ok = false;
  nvrtcResult_t (*create)(nvrtcProgram_t*, const char*, const char*, int, const char* const*, const char* const*);
  nvrtcResult_t (*compile)(nvrtcProgram_t, int, const char* const*);
  nvrtcResult_t (*log_size)(nvrtcProgram_t, size_t*);
  nvrtcResult_t (*log)(nvrtcProgram_t, char*);
  nvrtcResult_t (*cubin_size)(nvrtcProgram_t, size_t*);
  nvrtcResult_t (*cubin)(nvrtcProgram_t, char*);
  nvrtcResult_t (*destroy)(nvrtcProgram_t*);
};

Nvrtc& nvrtc() {
  static Nvrtc n;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12",
                           "/usr/local/cuda/lib64/libnvrtc.so"};
    void* h = nullptr;
    for (const char* nm : names)
      if ((h = dlopen(nm, RTLD_NOW | RTLD_LOCAL))) break;
    if (!h) return;
    n.create = (decltype(n.create))dlsym(h, "nvrtcCreateProgram");
    n.compile = (decltype(n.compile))dlsym(h, "nvrtcCompileProgram");
    n.log_size = (decltype(n.log_size))dlsym(h, "nvrtcGetProgramLogSize");
    n.log = (decltype(n.log))dlsym(h, "nvrtcGetProgramLog");
    n.cubin_size = (decltype(n.cubin_size))dlsym(h, "nvrtcGetCUBINSize");
    n.cubin = (decltype(n.cubin))dlsym(h, "nvrtcGetCUBIN");
    n.destroy = (decltype(n.destroy))dlsym(h, "nvrtcDestroyProgram");
    n.ok = n.create && n.compile && n.log_size && n.log && n.cubin_size && n.cubin && n.destroy;
  });
  return n;
}

std::string csrc_dir() {
  Dl_info info;
  if (dladdr((void*)&csrc_dir, &info) && info.dli_fname) {
    std::string so(info.dli_fname);
    auto pos = so.rfind('/');
    std::string dir = pos == std::string::npos ? "." : so.substr(0, pos);
    return dir + "/csrc";
  }
  return "csrc";
}

struct Entry {
  cudaLibrary_t lib = nullptr;
  cudaKernel_t kern = nullptr;
  bool ok = false;
};
std::mutex g_mu;
std::map<std::string, Entry> g_cache;
struct Stats {
  uint64_t compiled = 0, hits = 0, failed = 0;
  double compile_ms = 0;
  std::string last_error;
} g_stats;

bool jit_env_enabled() {
  const char* e = getenv("TQ_JIT");
  return !(e && e[0] == '0');
}

// ------------------------------------------------------------------ code generation
std::string hex64(uint64_t v) {
  char b[32];
  snprintf(b, sizeof b, "0x%016llxull", (unsigned long long)v);
  return b;
}

struct Gen {
  const PipeParams& p;
  const std::vector<DInstr>& code;
  const std::vector<DLit>& lits;
  std::ostringstream os;
  // current SSA names per slot
  std::string vv[kMaxValueSlots], vn[kMaxValueSlots], bv[kMaxBoolSlots], bn[kMaxBoolSlots];
  bool v64[kMaxValueSlots] = {};  // slot value known to fit int64

  int min_blocks = 1;  // resident CTAs per SM the launch plans for (__launch_bounds__)

  Gen(const PipeParams& p_, const std::vector<DInstr>& c_, const std::vector<DLit>& l_) : p(p_), code(c_), lits(l_) {}

  // staged column c of the current row, already in registers (struct Raw)
  std::string col_val(int c) { return "R.c" + std::to_string(c); }
  std::string col_valid(int c) {
    if (!p.cols[c].validity) return "true";
    return "R.v" + std::to_string(c);
  }
  static const char* raw_type(uint8_t kind) {
    switch (kind) {
      case TQ_FLOAT64: return "double";
      case TQ_BOOL: return "uint8_t";
      case TQ_DECIMAL: return "i128";
      default: return "long long";
    }
  }
  std::string lit_i(int i) { return "mk128(" + hex64(lits[i].lo) + ", " + hex64(lits[i].hi) + ")"; }
  bool lit_fits64(int i) {
    uint64_t lo = lits[i].lo, hi = lits[i].hi;
    return hi == ((int64_t)lo < 0 ? ~0ull : 0ull);
  }

  // int128-class operand; sets valid expr and whether it fits int64 statically
  std::string opnd_i(uint8_t k, uint16_t idx, std::string& valid, bool& is64) {
    is64 = false;
    switch (k) {
      case K_COL_I64: valid = col_valid(idx); is64 = true;
        return col_val(idx);
      case K_COL_DEC: valid = col_valid(idx);
        return col_val(idx);
      case K_COL_BOOL: valid = col_valid(idx); is64 = true;
        return "(long long)(" + col_val(idx) + " != 0)";
      case K_TMP_I: valid = vn[idx]; is64 = v64[idx]; return vv[idx];
      case K_TMP_B: valid = bn[idx]; is64 = true; return "(long long)" + bv[idx];
      case K_LIT_I: case K_LIT_B:
        valid = lits[idx].valid ? "true" : "false";
        if (lit_fits64(idx)) { is64 = true; return "(long long)" + hex64(lits[idx].lo); }
        return lit_i(idx);
    }
    fail(TQ_INTERNAL, "jit: bad int operand");
  }
  std::string as128(const std::string& e, bool is64) { return is64 ? "((i128)(" + e + "))" : e; }
  std::string opnd_f(uint8_t k, uint16_t idx, uint8_t scale, std::string& valid) {
    switch (k) {
      case K_COL_F64: valid = col_valid(idx); return col_val(idx);
      case K_TMP_F: valid = vn[idx]; return vv[idx];
      case K_LIT_F: {
        valid = lits[idx].valid ? "true" : "false";
        uint64_t bits;
        std::memcpy(&bits, &lits[idx].f, 8);
        return "__longlong_as_double((long long)" + hex64(bits) + ")";
      }
      default: {
        bool is64;
        std::string x = opnd_i(k, idx, valid, is64);
        std::string d = is64 ? "((double)(" + x + "))" : "i128_to_f64(" + x + ")";
        if (scale) d = "(" + d + " / 1e" + std::to_string(scale) + ")";
        return d;
      }
    }
  }
  std::string opnd_b(uint8_t k, uint16_t idx, std::string& valid) {
    if (k == K_TMP_B) { valid = bn[idx]; return bv[idx]; }
    bool is64;
    std::string x = opnd_i(k, idx, valid, is64);
    return "((" + x + ") != 0)";
  }

  static const char* cmp_op(uint8_t sub) {
    switch (sub) {
      case TQ_LT: return "<";
      case TQ_LE: return "<=";
      case TQ_EQ: return "==";
      case TQ_NE: return "!=";
      case TQ_GE: return ">=";
      default: return ">";
    }
  }

  void body(int upto) {
    for (int pc = 0; pc < upto; ++pc) {
      const DInstr& in = code[pc];
      std::string r = "r" + std::to_string(pc), n = "n" + std::to_string(pc);
      std::string va, vb;
      switch (in.op) {
        case OP_ADD_I: case OP_SUB_I: case OP_MUL_I: {
          bool xa, xb;
          std::string x = opnd_i(in.ak, in.a, va, xa), y = opnd_i(in.bk, in.b, vb, xb);
          std::string X = as128(x, xa), Y = as128(y, xb);
          if (in.fa != 0xff) { X = "mul128(" + X + ", " + lit_i(in.fa) + ")"; xa = false; }
          if (in.fb != 0xff) { Y = "mul128(" + Y + ", " + lit_i(in.fb) + ")"; xb = false; }
          std::string e;
          if (in.op == OP_MUL_I && xa && xb)
            e = "mul64x64(" + x + ", " + y + ")";
          else
            e = std::string(in.op == OP_ADD_I ? "add128(" : in.op == OP_SUB_I ? "sub128(" : "mul128(") + X + ", " + Y + ")";
          if (in.wrap) {
            if (xa && xb && in.op != OP_MUL_I)
              e = "((i128)(long long)((unsigned long long)(" + x + ") " + (in.op == OP_ADD_I ? "+" : "-") +
                  " (unsigned long long)(" + y + ")))";
            else
              e = "wrap64(" + e + ")";
          }
          os << "    const i128 " << r << " = " << e << "; const bool " << n << " = " << va << " && " << vb << ";\n";
          vv[in.dst] = r; vn[in.dst] = n; v64[in.dst] = in.wrap != 0;
          break;
        }
        case OP_ADD_F: case OP_SUB_F: case OP_MUL_F: {
          std::string x = opnd_f(in.ak, in.a, in.fa, va), y = opnd_f(in.bk, in.b, in.fb, vb);
          const char* o = in.op == OP_ADD_F ? "+" : in.op == OP_SUB_F ? "-" : "*";
          os << "    const double " << r << " = (" << x << ") " << o << " (" << y << "); const bool " << n << " = " << va
             << " && " << vb << ";\n";
          vv[in.dst] = r; vn[in.dst] = n; v64[in.dst] = false;
          break;
        }
        case OP_CMP_I: {
          bool xa, xb;
          std::string x = opnd_i(in.ak, in.a, va, xa), y = opnd_i(in.bk, in.b, vb, xb);
          std::string e;
          if (xa && xb && in.fa == 0xff && in.fb == 0xff) {
            e = "(" + x + ") " + cmp_op(in.sub) + " (" + y + ")";
          } else {
            std::string X = as128(x, xa), Y = as128(y, xb);
            if (in.fa != 0xff) X = "mul128(" + X + ", " + lit_i(in.fa) + ")";
            if (in.fb != 0xff) Y = "mul128(" + Y + ", " + lit_i(in.fb) + ")";
            e = "(" + X + ") " + cmp_op(in.sub) + " (" + Y + ")";
          }
          os << "    const bool " << r << " = " << e << "; const bool " << n << " = " << va << " && " << vb << ";\n";
          bv[in.dst] = r; bn[in.dst] = n;
          break;
        }
        case OP_CMP_F: {
          std::string x = opnd_f(in.ak, in.a, in.fa, va), y = opnd_f(in.bk, in.b, in.fb, vb);
          os << "    const bool " << r << " = (" << x << ") " << cmp_op(in.sub) << " (" << y << "); const bool " << n
             << " = " << va << " && " << vb << ";\n";
          bv[in.dst] = r; bn[in.dst] = n;
          break;
        }
        case OP_CMP_B: {
          std::string x = opnd_b(in.ak, in.a, va), y = opnd_b(in.bk, in.b, vb);
          os << "    const bool " << r << " = ((int)(" << x << ")) " << cmp_op(in.sub) << " ((int)(" << y
             << ")); const bool " << n << " = " << va << " && " << vb << ";\n";
          bv[in.dst] = r; bn[in.dst] = n;
          break;
        }
        case OP_AND: case OP_OR: {
          std::string x = opnd_b(in.ak, in.a, va), y = opnd_b(in.bk, in.b, vb);
          os << "    const bool " << r << " = (" << x << ") " << (in.op == OP_AND ? "&&" : "||") << " (" << y
             << "); const bool " << n << " = " << va << " && " << vb << ";\n";
          bv[in.dst] = r; bn[in.dst] = n;
          break;
        }
        case OP_NOT: {
          std::string x = opnd_b(in.ak, in.a, va);
          os << "    const bool " << r << " = !(" << x << "); const bool " << n << " = " << va << ";\n";
          bv[in.dst] = r; bn[in.dst] = n;
          break;
        }
        default:
          fail(TQ_INTERNAL, "jit: bad opcode");
      }
    }
  }

  // value of a root operand as the given class
  std::string root_i(uint8_t k, uint16_t idx, std::string& valid) {
    bool is64;
    std::string x = opnd_i(k, idx, valid, is64);
    return as128(x, is64);
  }
  bool is_f(uint8_t k) { return k == K_COL_F64 || k == K_TMP_F || k == K_LIT_F; }
  bool is_b(uint8_t k) { return k == K_TMP_B || k == K_COL_BOOL || k == K_LIT_B; }

  std::string source(int sink) {
    const int nacc = (int)p.nacc;
    const int kw = (int)p.key_words;
    os << "// generated by libtq_gpu.so jit.cu — do not edit\n";
    os << "#include \"kernel_common.cuh\"\nnamespace tq {\n";
    os << "__device__ __forceinline__ i128 ld_dec(const uint8_t* b, u32 r) { const ulonglong2 q = "
          "((const ulonglong2*)b)[r]; return mk128(q.x, q.y); }\n";
    os << "__device__ __forceinline__ i128 mul64x64(long long x, long long y) { return mk128((u64)x * (u64)y, "
          "(u64)__mul64hi(x, y)); }\n";
    os << "struct Gen {\n  static constexpr bool kInterp = false;\n";
    os << "  static constexpr int kKwa = " << (kw + 1) << ", kKw = " << kw << ", kNacc = " << nacc << ";\n";
    os << "  static constexpr bool kKey1x8 = " << ((p.nkeys == 1 && p.keys[0].bytes == 8 && p.keys[0].words == 1) ? "true" : "false")
       << ";\n";
    os << "  __device__ __forceinline__ static u32 nacc(const PipeParams&) { return " << nacc << "; }\n";
    os << "  __device__ __forceinline__ static u32 nplanes(const PipeParams&) { return " << p.nplanes << "; }\n";
    os << "  __device__ __forceinline__ static uint8_t acc_op(const PipeParams&, u32 a) {\n    switch (a) {";
    for (int a = 0; a < nacc; ++a) os << " case " << a << ": return " << (int)p.acc[a].op << ";";
    os << " default: return 0; }\n  }\n";
    os << "  __device__ __forceinline__ static uint8_t acc_kind(const PipeParams&, u32 a) {\n    switch (a) {";
    for (int a = 0; a < nacc; ++a) os << " case " << a << ": return " << (int)p.acc[a].kind << ";";
    os << " default: return 0; }\n  }\n";
    os << "  __device__ __forceinline__ static u32 acc_plane(const PipeParams&, u32 a) {\n    switch (a) {";
    for (int a = 0; a < nacc; ++a) os << " case " << a << ": return " << (int)p.acc_plane[a] << ";";
    os << " default: return 0; }\n  }\n";
    // ---- predicate
    // ---- the row's staged columns, copied out of the stage into registers
    os << "  struct Raw {";
    for (u32 c = 0; c < p.nstaged; ++c) {
      os << " " << raw_type(p.cols[c].kind) << " c" << c << ";";
      if (p.cols[c].validity) os << " bool v" << c << ";";
    }
    os << " };\n";
    os << "  __device__ __forceinline__ static void load(const WCtx& w, int v, Raw& R) {\n"
          "    const u32 r = trow(w, v);\n    (void)r;\n";
    for (u32 c = 0; c < p.nstaged; ++c) {
      const std::string base = "(w.stage + " + std::to_string(p.cols[c].off) + "u)";
      const std::string f = "R.c" + std::to_string(c);
      if (!((p.load_mask >> c) & 1)) {  // not loaded by this launch: dead in the generated code
        os << "    " << f << " = 0;\n";
        if (p.cols[c].validity) os << "    R.v" << c << " = false;\n";
        continue;
      }
      if (p.cols[c].kind == TQ_DECIMAL) os << "    " << f << " = ld_dec(" << base << ", r);\n";
      else
        os << "    " << f << " = ((const " << raw_type(p.cols[c].kind) << "*)" << base << ")[r];\n";
      if (p.cols[c].validity)
        os << "    R.v" << c << " = (((const u32*)(w.stage + " << p.cols[c].voff
           << "u))[(w.row0 >> 5) + v] >> w.lane) & 1u;\n";
    }
    os << "  }\n";
    // the same columns straight from global memory (count_direct_body)
    os << "  __device__ __forceinline__ static void load_g(const WCtx& w, u64 row, Raw& R) {\n"
          "    const PipeParams& p = *w.p;\n    (void)p;\n";
    for (u32 c = 0; c < p.nstaged; ++c) {
      const std::string f = "R.c" + std::to_string(c);
      const std::string col = "p.cols[" + std::to_string(c) + "]";
      if (!((p.load_mask >> c) & 1)) {
        os << "    " << f << " = 0;\n";
        if (p.cols[c].validity) os << "    R.v" << c << " = false;\n";
        continue;
      }
      if (p.cols[c].kind == TQ_DECIMAL)
        os << "    { const ulonglong2 q = __ldg((const ulonglong2*)" << col << ".values + row); " << f
           << " = mk128(q.x, q.y); }\n";
      else
        os << "    " << f << " = __ldg((const " << raw_type(p.cols[c].kind) << "*)" << col << ".values + row);\n";
      if (p.cols[c].validity)
        os << "    R.v" << c << " = (__ldg(" << col << ".validity + (row >> 3)) >> (row & 7)) & 1u;\n";
    }
    os << "  }\n";
    os << "  __device__ __forceinline__ static u32 tile_begin(WCtx& w, const DInstr*, u32* pm, const Raw* Rs) {\n"
          "    u32 any = 0;\n#pragma unroll\n    for (int v = 0; v < kV; ++v) {\n      const u32 r = trow(w, v);\n"
          "      const Raw& R = Rs[v];\n      (void)R;\n      bool pass = r < w.nrows;\n";
    if (p.pred_kind != K_NONE) {
      os << "      if (pass) {\n";
      Gen g(p, code, lits);
      g.body(p.npred);
      os << g.os.str();
      std::string pv;
      std::string pe = g.opnd_b(p.pred_kind, p.pred_idx, pv);
      os << "      pass = (" << pv << ") && (" << pe << ");\n      }\n";
    }
    os << "      pm[v] = __ballot_sync(kFull, pass);\n      any |= pm[v];\n    }\n    return any;\n  }\n";
    // ---- keys
    os << "  __device__ __forceinline__ static bool keys(const WCtx& w, int v, u64* kw, const Raw& R) {\n"
          "    const u32 r = trow(w, v);\n    (void)r; (void)R;\n";
    if (p.nkeys) {
      Gen g(p, code, lits);
      g.body((int)code.size());
      os << g.os.str();
      os << "    u64 nm = 0;\n";
      int pos = 0;
      for (u32 k = 0; k < p.nkeys; ++k) {
        const KeyOpnd& ko = p.keys[k];
        std::string valid;
        if (is_f(ko.kind)) {
          std::string x = g.opnd_f(ko.kind, ko.idx, 0, valid);
          os << "    { const bool kv = " << valid << "; kw[" << pos << "] = kv ? (u64)__double_as_longlong(" << x
             << ") : 0ull; if (!kv) nm |= " << (1ull << k) << "ull; }\n";
        } else {
          std::string x = g.root_i(ko.kind, ko.idx, valid);
          os << "    { const bool kv = " << valid << "; const i128 kx = " << x << "; kw[" << pos
             << "] = kv ? lo64(kx) : 0ull;";
          if (ko.words == 2) os << " kw[" << pos + 1 << "] = kv ? hi64(kx) : 0ull;";
          os << " if (!kv) nm |= " << (1ull << k) << "ull; }\n";
        }
        pos += ko.words;
      }
      os << "    kw[" << pos << "] = nm;\n    return nm != 0;\n  }\n";
    } else {
      os << "    (void)r; kw[0] = 0; return false;\n  }\n";
    }
    // ---- aggregate inputs
    os << "  __device__ __forceinline__ static void accs(const WCtx& w, int v, RowVals& x, const Raw& R) {\n"
          "    const u32 r = trow(w, v);\n    (void)R;\n";
    if (sink == SINK_AGG && nacc) {
      Gen g(p, code, lits);
      g.body((int)code.size());
      os << g.os.str();
      for (int a = 0; a < nacc; ++a) {
        const AccSpec& as = p.acc[a];
        std::string valid;
        if (as.op == ACC_CNT) {
          if (as.kind == K_NONE) os << "    x.av[" << a << "] = true;\n";
          else {
            if (is_f(as.kind)) (void)g.opnd_f(as.kind, as.idx, 0, valid);
            else (void)g.root_i(as.kind, as.idx, valid);
            os << "    x.av[" << a << "] = " << valid << ";\n";
          }
        } else if (as.op == ACC_SUM_I || as.op == ACC_MIN_I || as.op == ACC_MAX_I) {
          std::string e = g.root_i(as.kind, as.idx, valid);
          os << "    x.ai[" << a << "] = " << e << "; x.av[" << a << "] = " << valid << ";\n";
        } else {
          std::string e = g.opnd_f(as.kind, as.idx, as.scale, valid);
          os << "    x.af[" << a << "] = " << e << "; x.av[" << a << "] = " << valid << ";\n";
        }
      }
    } else {
      os << "    (void)r; (void)x;\n";
    }
    os << "  }\n";
    // ---- materialised outputs
    os << "  __device__ __forceinline__ static void store(const WCtx& w, int v, u64 pos, long long brow, const Raw& R) "
          "{\n    const u32 r = trow(w, v);\n    const PipeParams& p = *w.p;\n    (void)R;\n";
    if (sink == SINK_EMIT && p.nout) {
      Gen g(p, code, lits);
      g.body((int)code.size());
      os << g.os.str();
      for (u32 c = 0; c < p.nout; ++c) {
        const OutCol& o = p.out[c];
        std::string oc = "p.out[" + std::to_string(c) + "]";
        if (o.src == OUT_BUILD) {
          os << "    store_build(" << oc << ", pos, brow, w.out_delta);\n";
          continue;
        }
        std::string valid;
        switch (o.kind) {
          case K_COL_I64:
            valid = g.col_valid(o.idx);
            os << "    *(u64*)(" << oc << ".values + w.out_delta + pos * 8) = (u64)" << g.col_val(o.idx) << ";\n";
            break;
          case K_COL_F64:
            valid = g.col_valid(o.idx);
            os << "    *(u64*)(" << oc << ".values + w.out_delta + pos * 8) = (u64)__double_as_longlong(" << g.col_val(o.idx)
               << ");\n";
            break;
          case K_COL_DEC:
            valid = g.col_valid(o.idx);
            os << "    *(ulonglong2*)(" << oc << ".values + w.out_delta + pos * 16) = make_ulonglong2(lo64(" << g.col_val(o.idx)
               << "), hi64(" << g.col_val(o.idx) << "));\n";
            break;
          case K_COL_BOOL:
            valid = g.col_valid(o.idx);
            os << "    (" << oc << ".values + w.out_delta)[pos] = " << g.col_val(o.idx) << ";\n";
            break;
          case K_TMP_F: case K_LIT_F: {
            std::string e = g.opnd_f(o.kind, o.idx, 0, valid);
            os << "    *(double*)(" << oc << ".values + w.out_delta + pos * 8) = " << e << ";\n";
            break;
          }
          case K_TMP_B: case K_LIT_B: {
            std::string e = g.opnd_b(o.kind, o.idx, valid);
            os << "    (" << oc << ".values + w.out_delta)[pos] = (" << e << ") ? 1 : 0;\n";
            break;
          }
          default: {
            std::string e = g.root_i(o.kind, o.idx, valid);
            if (o.width == 16)
              os << "    { const i128 ox = " << e << "; *(ulonglong2*)(" << oc
                 << ".values + w.out_delta + pos * 16) = make_ulonglong2(lo64(ox), hi64(ox)); }\n";
            else
              os << "    *(u64*)(" << oc << ".values + w.out_delta + pos * 8) = lo64(" << e << ");\n";
          }
        }
        if (o.validity)
          os << "    if ((w.vmask >> " << c << ") & 1u) set_valid(" << oc << ", pos, " << valid << ", w.out_delta);\n";
      }
    } else {
      os << "    (void)r; (void)p; (void)pos; (void)brow;\n";
    }
    os << "  }\n};\n}  // namespace tq\n";
    if (sink >= SINK_COUNT_DIRECT) {
      os << "extern \"C\" __global__ void __launch_bounds__(256) tq_jit_main(const __grid_constant__ "
            "tq::PipeParams p) {\n  tq::count_direct_loop<tq::Gen, "
         << (sink - SINK_COUNT_DIRECT) << ">(p);\n}\n";
      return os.str();
    }
    os << "extern \"C\" __global__ void __launch_bounds__(tq::kBlock, " << min_blocks
       << ") tq_jit_main(const __grid_constant__ "
          "tq::PipeParams p) {\n  tq::pipe_body<"
       << sink << ", tq::Gen>(p);\n}\n";
    return os.str();
  }
};

void dump(const std::string& src, const std::string& log) {
  const char* d = getenv("TQ_JIT_DUMP");
  if (!d) return;
  static int seq = 0;
  std::string path = std::string(d) + "/tq_jit_" + std::to_string(seq++) + ".cu";
  if (FILE* f = fopen(path.c_str(), "w")) {
    fwrite(src.data(), 1, src.size(), f);
    if (!log.empty()) fprintf(f, "\n/* NVRTC LOG:\n%s\n*/\n", log.c_str());
    fclose(f);
  }
}

Entry compile(const std::string& src) {
  Entry e;
  Nvrtc& n = nvrtc();
  if (!n.ok) {
    g_stats.last_error = "libnvrtc not found";
    return e;
  }
  auto t0 = std::chrono::steady_clock::now();
  nvrtcProgram_t prog;
  if (n.create(&prog, src.c_str(), "tq_jit.cu", 0, nullptr, nullptr) != 0) {
    g_stats.last_error = "nvrtcCreateProgram failed";
    return e;
  }
  std::string dir = csrc_dir();
  std::string inc1 = "-I" + dir, inc2 = "-I" + dir + "/../../include";
  // the tile geometry this library was built with (pipeline.h)
  std::string dw = "-DTQ_KWARPS=" + std::to_string(kWarps), dv = "-DTQ_KV=" + std::to_string(kV);
  // TQ_JIT_DEFS: one extra -D for experiments (e.g. TQ_PB=4)
  static const std::string xdef = [] {
    const char* e = getenv("TQ_JIT_DEFS");
    return e && *e ? std::string("-D") + e : std::string("-DTQ_JIT_NOEXTRA=1");
  }();
  const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "-lineinfo", "-DTQ_JIT=1", "--device-int128",
                        inc1.c_str(), inc2.c_str(), dw.c_str(), dv.c_str(), xdef.c_str()};
  int rc = n.compile(prog, 10, opts);
  if (rc != 0) {
    size_t ls = 0;
    n.log_size(prog, &ls);
    std::string log(ls, '\0');
    if (ls) n.log(prog, &log[0]);
    g_stats.last_error = "nvrtc compile failed: " + log.substr(0, 2000);
    dump(src, log);
    n.destroy(&prog);
    return e;
  }
  size_t cs = 0;
  n.cubin_size(prog, &cs);
  std::vector<char> cubin(cs);
  n.cubin(prog, cubin.data());
  n.destroy(&prog);
  if (cudaLibraryLoadData(&e.lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0) != cudaSuccess ||
      cudaLibraryGetKernel(&e.kern, e.lib, "tq_jit_main") != cudaSuccess) {
    cudaGetLastError();
    g_stats.last_error = "cudaLibraryLoadData failed";
    return e;
  }
  e.ok = true;
  dump(src, "");
  g_stats.compile_ms +=
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return e;
}

}  // namespace

// Launch a pipeline kernel: NVRTC-specialised when possible, else interpreted.
cudaError_t launch_pipeline_prog(tq_ctx* c, int sink, const PipeParams& p, u32 smem, u32 grid, cudaStream_t st,
                                 const std::vector<DInstr>& code, const std::vector<DLit>& lits) {
  if (c->jit && jit_env_enabled()) {
    TQ_HT("jit key+lookup+launch");
    // cache key: every launch parameter the generator bakes into the source
    std::string key;
    key.reserve(1024);
    auto put = [&](const void* d, size_t n) { key.append((const char*)d, n); };
    put(&sink, sizeof sink);
    put(code.data(), code.size() * sizeof(DInstr));
    put(lits.data(), lits.size() * sizeof(DLit));
    put(&p.npred, sizeof p.npred);
    put(&p.pred_kind, 1);
    put(&p.pred_idx, 2);
    for (u32 c2 = 0; c2 < p.nstaged; ++c2) {
      const StagedCol& sc = p.cols[c2];
      uint32_t f[5] = {sc.off, sc.voff, sc.width, (uint32_t)(sc.validity != nullptr), sc.kind};
      put(f, sizeof f);
    }
    put(&p.load_mask, 4);
    const int min_blocks = grid > (u32)c->sms ? 2 : 1;
    put(&min_blocks, 4);
    put(&p.nkeys, 4);
    put(&p.key_words, 4);
    put(p.keys, sizeof(KeyOpnd) * p.nkeys);
    put(&p.nacc, 4);
    put(&p.nplanes, 4);
    put(p.acc, sizeof(AccSpec) * p.nacc);
    put(p.acc_plane, p.nacc);
    put(&p.nout, 4);
    for (u32 o = 0; o < p.nout; ++o) {
      const OutCol& oc = p.out[o];
      uint32_t f[6] = {oc.src, oc.kind, oc.width, oc.out_kind, oc.idx, (uint32_t)(oc.validity != nullptr)};
      put(f, sizeof f);
    }
    Entry e;
    bool have = false;
    {
      std::lock_guard<std::mutex> lk(g_mu);
      auto it = g_cache.find(key);
      if (it != g_cache.end()) {
        e = it->second;
        g_stats.hits++;
        have = true;
      }
    }
    if (!have) {
      std::string src;
      try {
        Gen g(p, code, lits);
        g.min_blocks = min_blocks;
        src = g.source(sink);
      } catch (const Fail&) {
        src.clear();
      }
      std::lock_guard<std::mutex> lk(g_mu);
      auto it = g_cache.find(key);
      if (it != g_cache.end()) {
        e = it->second;
      } else {
        e = src.empty() ? Entry{} : compile(src);
        g_cache[key] = e;
        if (e.ok) g_stats.compiled++;
        else g_stats.failed++;
      }
    }
    {
      if (e.ok) {
        cudaError_t err = cudaSuccess;
        if (sink < SINK_COUNT_DIRECT)
          err = cudaFuncSetAttribute((const void*)e.kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (err != cudaSuccess) return err;
        PipeParams pp = p;
        void* args[] = {&pp};
        err = cudaLaunchKernel((const void*)e.kern, dim3(grid), dim3(sink >= SINK_COUNT_DIRECT ? 256 : kBlock), args,
                               sink >= SINK_COUNT_DIRECT ? 0 : smem, st);
        if (err == cudaSuccess) c->jit_launches.fetch_add(1);
        return err;
      }
    }
  }
  if (sink >= SINK_COUNT_DIRECT) return cudaErrorNotSupported;  // generated code only: the caller uses SINK_COUNT
  return launch_interp(sink, p, smem, grid, st);
}

}  // namespace tq

extern "C" {

void tq_ctx_set_jit(tq_ctx* c, int on) { c->jit = on != 0; }

uint64_t tq_jit_report(tq_ctx* c, char* buf, uint64_t cap) {
  std::lock_guard<std::mutex> lk(tq::g_mu);
  std::string s = "compiled " + std::to_string(tq::g_stats.compiled) + "\nhits " + std::to_string(tq::g_stats.hits) +
                  "\nfailed " + std::to_string(tq::g_stats.failed) + "\ncompile_ms " +
                  std::to_string(tq::g_stats.compile_ms) + "\njit_launches " +
                  std::to_string(c ? c->jit_launches.load() : 0) + "\nlast_error " +
                  tq::g_stats.last_error.substr(0, 1500) + "\n";
  uint64_t n = std::min<uint64_t>(s.size(), cap ? cap - 1 : 0);
  if (cap) {
    std::memcpy(buf, s.data(), n);
    buf[n] = 0;
  }
  return n;
}

}  // extern "C"
