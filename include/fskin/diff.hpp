#pragma once
// fskin-b200 — reference-facing implicit-differentiation API (drop-in for the grid-routed part of
// proj/include/fskin/diff.hpp:16-40). The reference differentiates through its skinning MLP
// (MlpGrad); this build's skinning field is the voxel grid, so the same two linear maps —
// exact (∂d/∂x*)⁻¹ and the Broyden estimate J~ — carry the root cotangent to the grid:
//   u = −(∂d/∂x*)⁻ᵀ v  (implicit_grad_exact, diff.cpp:31-41)   or   u = −J~ᵀ v  (approx, :43-51)
//   dL/dT_c += φ_c(x*) · u (x*, 1)ᵀ,   dL/dw_{c,i} = <dL/dT_c, B_i>_F.
// Runs on the GPU through include/fsk.h.

#include <span>
#include <stdexcept>
#include <vector>

#include "fskin/correspondence.hpp"
#include "fskin/geometry.hpp"
#include "fskin/skinning.hpp"

namespace fskin {

/// Raised when the exact implicit gradient is requested at a root whose deformation Jacobian is
/// numerically singular (|det| < 1e-10); callers skip the sample (diff.hpp:20-22, diff.cpp:10-12).
struct SingularRootError : std::runtime_error {
    explicit SingularRootError(double det);
};

/// u = −(∂d/∂x*)⁻ᵀ·v with ∂d/∂x* = deform_jacobian(x*, grid, bones) (float64, LU as diff.cpp:36).
/// Throws SingularRootError.
Vec3 implicit_cotangent_exact(const Vec3& x_star, const SkinningVoxelGrid& grid, std::span<const RigidTransform> bones,
                              const Vec3& cotangent);

/// u = −J~ᵀ·v (diff.cpp:46). Never throws.
Vec3 implicit_cotangent_approx(const Mat3& inv_jacobian, const Vec3& cotangent);

/// Gradient of Σ_q v_q·x*_q with respect to the skinning grid for one root per query (the training
/// block, diff.cpp:336-359): root_of_query[q] indexes sets[q].roots (or -1: no root), cotangents[q]
/// = dL/dx*_q. exact = false uses each root's J~ (implicit_grad_approx); exact = true the exact
/// Jacobian (singular roots are skipped, as the reference's callers do; `skipped` counts them).
struct GridGradient {
    std::vector<double> d_tgrid;    ///< [V][12] dL/dT
    std::vector<double> d_weights;  ///< [V][n_b] dL/dw
    int skipped = 0;
};
GridGradient implicit_grad_grid(std::span<const CorrespondenceSet> sets, std::span<const int> root_of_query,
                                std::span<const Vec3> cotangents, const SkinningVoxelGrid& grid,
                                std::span<const RigidTransform> bones, bool exact);

}  // namespace fskin
