// hps/error.hpp — error vocabulary of the B200 sparse-embedding path.
//
// Declaration-compatible with the CPU reference (proj/include/hps/error.hpp:24-56):
// the same ErrorCode enumerators with the same integer values, the same Error
// exception type and the same raise() helper. On top of that this header defines
// how the GPU C-ABI's integer status (include/hps_gpu.h) maps back onto the
// enum, so a host caller that throws on failure sees exactly the reference's
// codes: statuses 1..17 are ErrorCode values verbatim; device failures (>= 256:
// CUDA, NCCL, out-of-memory) are folded into ErrorCode::Io, and capacity
// exhaustion into ErrorCode::Infeasible (SURVEY.md §8(b) "Errors").
#pragma once

#include <stdexcept>
#include <string>

namespace hps {

// Integer values are part of the ABI (hps_gpu.h status codes 1..17).
enum class ErrorCode : int {
  InvalidArgument = 1,
  BadMagic = 2,
  BadFormatVersion = 3,
  Truncated = 4,
  TrailingBytes = 5,
  DuplicateKey = 6,
  DimMismatch = 7,
  DtypeMismatch = 8,
  F16Range = 9,
  NonFinite = 10,
  UnknownTable = 11,
  TableExists = 12,
  BadShard = 13,
  Io = 14,
  Corruption = 15,
  Infeasible = 16,
  Protocol = 17,
};

/// Enumerator name ("InvalidArgument", ...); "Unknown" for values outside 1..17.
const char* error_code_name(ErrorCode code);

/// The one exception type of the API. what() carries the message, code() the class.
class Error : public std::runtime_error {
 public:
  Error(ErrorCode code, const std::string& what) : std::runtime_error(what), code_(code) {}
  ErrorCode code() const noexcept { return code_; }

 private:
  ErrorCode code_;
};

[[noreturn]] inline void raise(ErrorCode code, const std::string& what) { throw Error(code, what); }

/// Map a C-ABI status (0 = OK) onto the reference enum. Only meaningful for status != 0.
inline ErrorCode error_code_from_status(int status) {
  if (status >= 1 && status <= 17) return static_cast<ErrorCode>(status);
  if (status == 257 /* HPS_GPU_E_OUT_OF_MEMORY */) return ErrorCode::Infeasible;
  return ErrorCode::Io;
}

}  // namespace hps
