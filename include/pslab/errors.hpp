// pslab error classes for the B200 façade (drop-in for errors.hpp:11-69 of the
// reference). Every C-ABI status maps to exactly one of these
// (pslab_b200::throw_status), so code written against the reference catches
// the same types.
#pragma once

#include <stdexcept>
#include <string>

namespace pslab {

struct Error : std::runtime_error {
    explicit Error(const std::string& what) : std::runtime_error(what) {}
};

#define PSLAB_B200_ERROR(Name)                                   \
    struct Name : Error {                                        \
        explicit Name(const std::string& what) : Error(what) {} \
    }

PSLAB_B200_ERROR(PartitionError);
PSLAB_B200_ERROR(ShapeError);
PSLAB_B200_ERROR(LayerError);
PSLAB_B200_ERROR(ParseError);
PSLAB_B200_ERROR(ConfigError);
PSLAB_B200_ERROR(FormatError);
PSLAB_B200_ERROR(ProtocolError);
PSLAB_B200_ERROR(SimulatorBug);
PSLAB_B200_ERROR(LoggingError);
PSLAB_B200_ERROR(NumericError);
PSLAB_B200_ERROR(IoError);
// Device/runtime failure of the B200 path (no reference analogue).
PSLAB_B200_ERROR(DeviceError);

#undef PSLAB_B200_ERROR

}  // namespace pslab
