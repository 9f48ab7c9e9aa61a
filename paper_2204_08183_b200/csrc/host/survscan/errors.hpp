// survscan/errors.hpp — the reference's exception hierarchy
// (/root/reference/proj/include/survscan/errors.hpp:9-65), raised from the C-ABI
// status codes of include/gss.h (one code per class).
#pragma once

#include <stdexcept>
#include <string>

namespace survscan {

struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ParseError : Error { using Error::Error; };
struct SchemaError : Error { using Error::Error; };
struct DomainError : Error { using Error::Error; };
struct IndexError : Error { using Error::Error; };
struct DuplicateEntryError : Error { using Error::Error; };
struct InvalidColumnError : Error { using Error::Error; };
struct NonPositiveDenominatorError : Error { using Error::Error; };
struct OverflowError : Error { using Error::Error; };
struct DegenerateCurveError : Error { using Error::Error; };
struct EmptyFoldError : Error { using Error::Error; };
// device / runtime failures that have no reference counterpart
struct DeviceError : Error { using Error::Error; };

// Throw the class matching a gss_status code with the C ABI's last message.
[[noreturn]] void throw_status(int code);
inline void check(int rc) {
  if (rc != 0) throw_status(rc);
}

}  // namespace survscan
