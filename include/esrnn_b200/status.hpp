// C-ABI status -> exception mapping of the drop-in API, plus the two device-side failure
// classes the reference has no analogue for.  Needs the esrnn::Error hierarchy declared
// first: the drop-in's errors.hpp, or the reference's own esrnn/errors.hpp when only
// trainer.hpp is swapped (ESRNN_B200_HOST_TYPES, see trainer.hpp).
#pragma once
#include <string>

#include "../esrnn_b200.h"

namespace esrnn {

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
