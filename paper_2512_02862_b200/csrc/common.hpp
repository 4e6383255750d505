// Shared host-side types: errors (1:1 with the reference's exception classes), schema, CUDA/NCCL
// checks. Reference: /root/reference/proj/include/pystachio/errors.hpp:21-87, types.hpp:29-57.
#pragma once

#include <cstdint>
#include <cstring>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "psg.h"

namespace psg {

/// Engine error carrying the psg_status code of the reference class it mirrors.
class Error : public std::runtime_error {
 public:
  Error(int code, const std::string& msg) : std::runtime_error(msg), code_(code) {}
  int code() const { return code_; }

 private:
  int code_;
};

inline Error UnknownColumn(const std::string& n) { return Error(PSG_ERR_UNKNOWN_COLUMN, "unknown column: " + n); }
inline Error IoFailure(const std::string& m) { return Error(PSG_ERR_IO_FAILURE, "io failure: " + m); }
inline Error CorruptFooter(const std::string& m) { return Error(PSG_ERR_CORRUPT_FOOTER, "corrupt footer: " + m); }
inline Error InvalidInput(const std::string& m) { return Error(PSG_ERR_INVALID_INPUT, "invalid input: " + m); }
inline Error InfeasibleBudget(const std::string& m) { return Error(PSG_ERR_INFEASIBLE_BUDGET, "infeasible budget: " + m); }
inline Error MemoryExceeded(uint64_t req, uint64_t used, uint64_t cap) {
  return Error(PSG_ERR_MEMORY_EXCEEDED, "memory budget exceeded: requested " + std::to_string(req) +
                                            " bytes with " + std::to_string(used) + "/" +
                                            std::to_string(cap) + " in use");
}

enum class LType : uint8_t { Int64 = 0, Float64 = 1 };
constexpr size_t kValueBytes = 8;

struct Field {
  std::string name;
  LType type = LType::Int64;
  bool operator==(const Field&) const = default;
};

struct Schema {
  std::vector<Field> fields;
  size_t size() const { return fields.size(); }
  std::optional<size_t> index_of(const std::string& name) const {
    for (size_t i = 0; i < fields.size(); ++i)
      if (fields[i].name == name) return i;
    return std::nullopt;
  }
  size_t require(const std::string& name) const {
    auto i = index_of(name);
    if (!i) throw UnknownColumn(name);
    return *i;
  }
  bool operator==(const Schema&) const = default;
};

enum class CmpOp : uint8_t { Lt = 0, Le, Eq, Ne, Ge, Gt };
CmpOp cmp_op_from_string(const std::string& s);

/// Conjunction atom: single column vs literal (predicate.hpp:30-41).
struct Atom {
  std::string column;
  CmpOp op = CmpOp::Lt;
  bool lit_is_float = false;
  int64_t lit_i = 0;
  double lit_f = 0;
  /// literal_as<int64_t> / literal_as<double> (predicate.cpp:69-74).
  int64_t as_int() const { return lit_is_float ? static_cast<int64_t>(lit_f) : lit_i; }
  double as_float() const { return lit_is_float ? lit_f : static_cast<double>(lit_i); }
};
using Predicate = std::vector<Atom>;

}  // namespace psg

#define PSG_CUDA(call)                                                                  \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      throw ::psg::Error(PSG_ERR_CUDA, std::string("cuda: ") + cudaGetErrorString(e_) + \
                                           " at " + __FILE__ + ":" + std::to_string(__LINE__)); \
  } while (0)
