// dbsp error classes — the drop-in counterpart of the reference's
// proj/include/dbsp/error.hpp:10-44 (same class names and hierarchy, so code
// written against the reference catches the same types).  The C ABI reports
// failures as status codes (include/dbsp_b200.h); throw_status() turns a code
// back into the matching exception class.
#pragma once

#include <stdexcept>
#include <string>

#include "../dbsp_b200.h"

namespace dbsp {

class error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class config_error : public error {  // bad degrees, densities, thresholds, ...
 public:
  using error::error;
};
class io_error : public error {  // filesystem failures
 public:
  using error::error;
};
class parse_error : public io_error {  // malformed file contents
 public:
  using io_error::io_error;
};
class contract_error : public error {  // values that should already agree do not
 public:
  using error::error;
};
class search_space_error : public config_error {  // brute-force guard
 public:
  using config_error::config_error;
};
// No reference counterpart: a CUDA runtime/driver failure in the GPU path.
class cuda_error : public error {
 public:
  using error::error;
};

namespace detail {

[[noreturn]] inline void throw_status(int code) {
  const std::string msg = dbsp_last_error();
  switch (code) {
    case DBSP_ERR_CONFIG: throw config_error(msg);
    case DBSP_ERR_SEARCH_SPACE: throw search_space_error(msg);
    case DBSP_ERR_IO: throw io_error(msg);
    case DBSP_ERR_PARSE: throw parse_error(msg);
    case DBSP_ERR_CONTRACT: throw contract_error(msg);
    case DBSP_ERR_CUDA: throw cuda_error(msg);
    default: throw error(msg);
  }
}

inline void check(int code) {
  if (code != DBSP_OK) throw_status(code);
}

}  // namespace detail
}  // namespace dbsp
