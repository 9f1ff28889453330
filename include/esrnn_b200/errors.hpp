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
struct CudaError : Error { using Error::Error; };   // no reference analogue
struct NcclError : Error { using Error::Error; };   // no reference analogue

namespace detail {
[[noreturn]] inline void throw_status(esrnn_status st, const std::string& msg) {
    switch (st) {
        case ESRNN_PARSE_ERROR: throw ParseError(msg);
        case ESRNN_VALIDATION_ERROR: throw ValidationError(msg);
        case ESRNN_SHAPE_ERROR: throw ShapeError(msg);
        case ESRNN_INSUFFICIENT_LENGTH: throw InsufficientLengthError(msg);
        case ESRNN_NUMERIC_DOMAIN_ERROR: throw NumericDomainError(msg);
        case ESRNN_CONFIG_ERROR: throw ConfigError(msg);
        case ESRNN_CONTRACT_ERROR: throw ContractError(msg);
        case ESRNN_EQUIVALENCE_ERROR: throw EquivalenceError(msg);
        case ESRNN_CHECKPOINT_ERROR: throw CheckpointError(msg);
        case ESRNN_CUDA_ERROR: throw CudaError(msg);
        case ESRNN_NCCL_ERROR: throw NcclError(msg);
        default: throw Error(msg);
    }
}
inline void check(esrnn_status st, const esrnn_trainer* h) {
    if (st != ESRNN_OK) throw_status(st, esrnn_last_error(h));
}
}  // namespace detail

}  // namespace esrnn
