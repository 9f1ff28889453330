// Include overlay: the ONE header a reference maintainer swaps to move the hot path onto
// the B200 engine.  Everything else in the caller's tree (esrnn/data.hpp, network.hpp,
// holt_winters.hpp, matrix.hpp, errors.hpp, checkpoint.hpp, commands.hpp, ...) stays the
// reference's own; the drop-in Trainer is declared over those types.
#pragma once
#define ESRNN_B200_HOST_TYPES 1
#include <esrnn_b200/trainer.hpp>
