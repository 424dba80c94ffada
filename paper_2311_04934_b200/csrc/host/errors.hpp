// Error taxonomy of the Prompt Cache hot path.  Codes and their ordinal order
// mirror the reference's pc::ErrorCode (reference proj/core/include/promptcache/
// errors.hpp:8-30) so the C ABI status (ordinal + 1, 0 = OK) maps 1:1 onto the
// exception a reference caller would have caught.
#pragma once

#include <stdexcept>
#include <string>

namespace pcb {

enum class ErrorCode : int {
  SyntaxError,
  MissingSchemaAttr,
  UnknownRole,
  TokenizerFailure,
  FreeTextOverflow,
  ArgTooLong,
  InvalidConfig,
  PositionOutOfRange,
  ShapeMismatch,
  UnknownModule,
  CapacityExceeded,
  IoError,
  VersionMismatch,
  ConfigHashMismatch,
  ValidationFailed,
  PositionOverlap,
  UnknownCall,
  RecursionDetected,
  DuplicateName,
  InvalidProgram,
  Internal,
  CudaError,  // new: device failures (reference has no device); reported as Internal + detail
};

const char* error_code_name(ErrorCode c);

class Error : public std::runtime_error {
 public:
  Error(ErrorCode code, const std::string& message, int line = 0, int col = 0)
      : std::runtime_error(std::string(error_code_name(code)) + ": " + message),
        code_(code), line_(line), col_(col) {}
  ErrorCode code() const { return code_; }
  int line() const { return line_; }
  int col() const { return col_; }

 private:
  ErrorCode code_;
  int line_, col_;
};

}  // namespace pcb
