// gridtune_b200 — C++ host API mirroring the reference `gridtune` library
// (/root/reference/proj/include/gridtune) for the BO surrogate path, layered on
// the C ABI in gridtune_cuda.h.  Exception hierarchy: errors.hpp:55-108.
#pragma once

#include <cstddef>
#include <stdexcept>
#include <string>

#include "gridtune_cuda.h"

namespace gridtune_b200 {

class Error : public std::runtime_error {
 public:
  explicit Error(const std::string& what) : std::runtime_error(what) {}
};
class ModelConditioningError : public Error {
 public:
  using Error::Error;
};
class SamplingError : public Error {
 public:
  using Error::Error;
};
class ConfigError : public Error {
 public:
  using Error::Error;
};
/// CUDA failure (no device, launch error, out of memory).  No CPU fallback.
class DeviceError : public Error {
 public:
  using Error::Error;
};

/// Maps a C-ABI status onto the reference's exception types.
inline void check(int rc) {
  if (rc == GTC_OK) return;
  const std::string msg = gtc_last_error();
  switch (rc) {
    case GTC_ERR_CONDITIONING: throw ModelConditioningError(msg);
    case GTC_ERR_CONFIG: throw ConfigError(msg);
    case GTC_ERR_CUDA:
    case GTC_ERR_OOM: throw DeviceError(msg);
    default: throw Error(msg);
  }
}

}  // namespace gridtune_b200
