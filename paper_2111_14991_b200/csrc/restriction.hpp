// Restriction language of the search space (host side): lexer, parser and
// static type checker with the reference's grammar, precedence, typing and
// error messages (restriction.hpp:1-521, errors.hpp:17-26), compiled to a
// postfix program that the device enumeration kernel (gtc_kernels.cu
// k_enum_mask) evaluates for every point of the Cartesian grid.
//
// Device semantics are the reference's: numbers are IEEE doubles (+ - * /
// without contraction, `%` is fmod, comparisons against NaN are false),
// booleans compare with == / != only, and string comparisons (std::string
// ordering) are decided here on the host: every string comparison becomes a
// table of booleans indexed by the value ranks of the categorical parameters
// it reads, so the device never touches string data.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace gtc {

enum class ParamKind : int32_t { numeric = 0, categorical = 1, boolean = 2 };

// One tuning parameter (parameter.hpp:62-125): a name and its ordered values.
struct ParamDef {
  std::string name;
  ParamKind kind = ParamKind::numeric;
  std::vector<double> numbers;       // numeric
  std::vector<std::string> strings;  // categorical
  std::vector<bool> booleans;        // boolean
  size_t size() const {
    return kind == ParamKind::numeric ? numbers.size()
           : kind == ParamKind::categorical ? strings.size() : booleans.size();
  }
};

// ParseError (errors.hpp:17-26): message already suffixed with the position.
struct RestrictionError {
  std::string message;
  size_t position;
  bool parse;  // true: ParseError; false: gridtune::Error (limits)
};

// Device instruction of the postfix program (16 bytes).
enum EnumOp : uint8_t {
  kOpConst = 0,   // push k
  kOpParam,       // push value table entry of param a at its current rank
  kOpStrTable,    // push table[c + rank(a) * kb + rank(b)] (a/b = 255: absent)
  kOpNeg,
  kOpAdd,
  kOpSub,
  kOpMul,
  kOpDiv,
  kOpMod,
  kOpEq,
  kOpNe,
  kOpLt,
  kOpLe,
  kOpGt,
  kOpGe,
  kOpNot,
  kOpAnd,
  kOpOr,
  kOpEnd,         // end of one restriction: pop, the point is invalid if false
};

struct EnumInstr {
  uint8_t op;
  uint8_t a;
  uint8_t b;
  uint8_t pad;
  int32_t c;
  double k;
};

constexpr int kEnumMaxParams = 64;
constexpr int kEnumMaxStack = 32;
constexpr int kEnumMaxInstr = 2048;

// All restrictions of a space, compiled.
struct EnumProgram {
  std::vector<EnumInstr> code;     // restrictions back to back, each ended by kOpEnd
  std::vector<uint8_t> str_tables; // boolean tables of the string comparisons
  int max_stack = 0;
};

// Parses and type-checks `text` against `params` and appends its postfix
// code to `prog`.  Returns false and fills `err` on a ParseError.
bool compile_restriction(const std::string& text, const std::vector<ParamDef>& params, EnumProgram* prog,
                         RestrictionError* err);

// Validates parameter definitions like ParameterDef::validate
// (parameter.hpp:84-125); returns false and fills `err` (not a ParseError).
bool validate_params(const std::vector<ParamDef>& params, RestrictionError* err);

}  // namespace gtc
