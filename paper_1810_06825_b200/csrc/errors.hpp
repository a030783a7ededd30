// Exceptions carried to the C-ABI boundary and mapped to FRPCA_ERR_* codes
// (abi.cu guarded): the reference's std::invalid_argument / NumericalError /
// IoError (types.hpp:19-30), plus CUDA failures.
#pragma once

#include <stdexcept>
#include <string>

namespace fb {

struct InvalidArgument : std::runtime_error {
    explicit InvalidArgument(const std::string& w) : std::runtime_error(w) {}
};
struct NumericalError : std::runtime_error {
    explicit NumericalError(const std::string& w) : std::runtime_error(w) {}
};
struct CudaError : std::runtime_error {
    explicit CudaError(const std::string& w) : std::runtime_error(w) {}
};
struct IoError : std::runtime_error {
    explicit IoError(const std::string& w) : std::runtime_error(w) {}
};

}  // namespace fb
