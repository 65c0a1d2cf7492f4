#pragma once
// Drop-in for proj/include/d4orm/types.hpp:7-8 (Eigen::MatrixXd / VectorXd),
// Eigen-free: column-major double storage, see dense.hpp.
#include "d4orm/dense.hpp"

namespace d4orm {

using Matrix = dense::Matrix<double, dense::Dynamic, dense::Dynamic>;
using Vector = dense::Matrix<double, dense::Dynamic, 1>;
using Index = dense::Index;

}  // namespace d4orm

// The reference's callers name Eigen::Index directly (proj/src/bench.cpp:167-182,
// proj/tools/main.cpp:477).  Eigen declares it as std::ptrdiff_t, so this alias
// also coexists with a real Eigen included in the same translation unit.
namespace Eigen {
using Index = std::ptrdiff_t;
}  // namespace Eigen
