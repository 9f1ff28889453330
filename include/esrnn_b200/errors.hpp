// esrnn::Error hierarchy of the drop-in API (mirrors the reference's errors.hpp:9-67) plus
// the device-side failures the B200 engine can report.  Every C-ABI status maps to one
// class (include/esrnn_b200.h: esrnn_status).
#pragma once
#include <stdexcept>
#include <string>

#include "../esrnn_b200.h"

namespace esrnn {

struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ParseError : Error { using Error::Error; };
struct ValidationError : Error { using Error::Error; };
struct ShapeError : Error { using Error::Error; };
struct InsufficientLengthError : Error { using Error::Error; };
struct NumericDomainError : Error { using Error::Error; };
struct ConfigError : Error { using Error::Error; };
struct ContractError : Error { using Error::Error; };
struct EquivalenceError : Error { using Error::Error; };
struct CheckpointError : Error { using Error::Error; };
}  // namespace esrnn

#include "status.hpp"
