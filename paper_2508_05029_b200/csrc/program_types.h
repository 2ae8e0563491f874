// program_types.h — POD types of the Expr register machine (program.h),
// shared by the host compiler, the AOT interpreter and NVRTC-compiled
// specialised kernels (RTC-safe: no host headers).
#pragma once
#ifdef __CUDACC_RTC__
typedef unsigned char uint8_t;
typedef unsigned short uint16_t;
typedef unsigned int uint32_t;
typedef unsigned long long uint64_t;
typedef long long int64_t;
typedef int int32_t;
typedef unsigned long long uintptr_t;
#else
#include <cstdint>
#endif

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

}  // namespace tq
