// ORACLE — TEST INFRASTRUCTURE ONLY (oracle/_ref). The reference's MLP (proj/src/mlp.cpp) is not on the
// voxel search path this build checks; its symbols, referenced by the MLP overloads in skinning.cpp and
// deformer.cpp, are defined here to throw if ever called.
#include <stdexcept>

#include "fskin/mlp.hpp"

namespace fskin {
namespace {
[[noreturn]] void no_mlp() { throw std::logic_error("oracle/_ref: the reference's Mlp is not built (voxel path only)"); }
}  // namespace
Mlp::Mlp(std::vector<int>, std::uint64_t) { no_mlp(); }
MatrixXd Mlp::forward(const MatrixXd&, MlpTape*) const { no_mlp(); }
MatrixXd Mlp::input_tangent(const MlpTape&, const MatrixXd&) const { no_mlp(); }
const VectorXd& Mlp::forward_single(Eigen::Ref<const VectorXd>, Scratch&) const { no_mlp(); }
void Mlp::scale_output_layer(double) { no_mlp(); }
void Mlp::condition_input(const VectorXd&, const VectorXd&) { no_mlp(); }
void softmax_inplace(MatrixXd&) { no_mlp(); }
void softmax_inplace(VectorXd&) { no_mlp(); }
VectorXd softmax(const VectorXd&) { no_mlp(); }
}  // namespace fskin
