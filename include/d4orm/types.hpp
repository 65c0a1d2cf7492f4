#pragma once
// Drop-in for proj/include/d4orm/types.hpp:7-8 (Eigen::MatrixXd / VectorXd),
// Eigen-free: column-major double storage, see dense.hpp.
#include "d4orm/dense.hpp"

namespace d4orm {

using Matrix = dense::Matrix<double, dense::Dynamic, dense::Dynamic>;
using Vector = dense::Matrix<double, dense::Dynamic, 1>;
using Index = dense::Index;

}  // namespace d4orm
