// errors.hpp -- internal error type; kinds map 1:1 onto the reference's
// ErrorKind (errors.hpp:11-21) and onto fsvd_status at the C ABI.
#pragma once

#include <stdexcept>
#include <string>

namespace fsvd {

enum class Kind : int {
  Shape = 1,
  Rank = 2,
  Config = 3,
  Budget = 4,
  Accounting = 5,
  Format = 6,
  Numeric = 7,
  Infeasible = 8,
  Io = 9,
  Cuda = 10
};

struct Error : std::runtime_error {
  Kind kind;
  Error(Kind k, const std::string& w) : std::runtime_error(w), kind(k) {}
};

[[noreturn]] inline void fail(Kind k, const std::string& w) { throw Error(k, w); }

}  // namespace fsvd
