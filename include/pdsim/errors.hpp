// pdsim/errors.hpp — drop-in exception taxonomy of the reference
// (proj/include/pdsim/errors.hpp:25-46). The C-ABI status codes
// PDSIM_ERR_CONFIG / _DOMAIN / _PARSE map back onto these types.
#pragma once

#include <stdexcept>
#include <string>

namespace pdsim {

class ConfigError : public std::runtime_error {
 public:
  explicit ConfigError(const std::string& msg) : std::runtime_error(msg) {}
};

class DomainError : public std::invalid_argument {
 public:
  explicit DomainError(const std::string& msg) : std::invalid_argument(msg) {}
};

class ParseError : public std::runtime_error {
 public:
  ParseError(const std::string& where, const std::string& msg) : std::runtime_error(where + ": " + msg), where_(where) {}
  const std::string& where() const { return where_; }

 private:
  std::string where_;
};

// Raised for PDSIM_ERR_CUDA / PDSIM_ERR_INTERNAL: no usable B200, or an
// engine invariant failure. There is no CPU fallback.
class DeviceError : public std::runtime_error {
 public:
  explicit DeviceError(const std::string& msg) : std::runtime_error(msg) {}
};

}  // namespace pdsim
