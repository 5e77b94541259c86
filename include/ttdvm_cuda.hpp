// ttdvm_cuda.hpp -- header-only C++ host layer over the C ABI (ttdvm_cuda.h).
//
// The reference is a C++20 library (proj/include/ttdvm/*.hpp) whose errors
// are std::invalid_argument / std::runtime_error; this RAII wrapper gives
// the B200 step the same contract for a C++ caller: one Solver per GPU
// (context), every call synchronous, status codes mapped back to the
// reference's exception types.  TT tensors cross as the reference's Eigen
// column-major cores packed back to back (see PackedTt), so a caller holding
// std::vector<ttdvm::TtTensor> packs with one memcpy per core matrix
// (INTEGRATION.md shows that adapter; it is the only Eigen-dependent part).
#ifndef TTDVM_CUDA_HPP_
#define TTDVM_CUDA_HPP_

#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "ttdvm_cuda.h"

namespace ttdvm {
namespace cuda {

// std::invalid_argument for TTDVM_EINVAL (argument / shape / eps errors),
// std::runtime_error for everything else (nonpositive density / temperature
// with the cell id, wall-ghost degeneracy with the face id, CUDA / NCCL).
inline void check(const ttdvm_ctx* c, int rc) {
  if (rc == TTDVM_OK) return;
  const std::string msg = c ? ttdvm_cuda_last_error(c) : "ttdvm_cuda: no context";
  if (rc == TTDVM_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

// A batch of order-3 TT tensors in the C ABI packing (ttdvm_tt_batch).
struct PackedTt {
  int n1 = 0, n2 = 0, n3 = 0;
  std::vector<int32_t> ranks;    // 2 per tensor
  std::vector<int64_t> offsets;  // count + 1
  std::vector<double> cores;

  int count() const { return static_cast<int>(offsets.empty() ? 0 : offsets.size() - 1); }
  ttdvm_tt_batch view() const {
    return ttdvm_tt_batch{count(), n1, n2, n3, ranks.data(), offsets.data(), cores.data()};
  }
  // A(i,j,k) = first.row(i) * middle[j] * last.col(k) (TtTensor::value,
  // proj/src/tt_tensor.cpp:89-91)
  double value(int t, int i, int j, int k) const {
    const int r1 = ranks[2 * t], r2 = ranks[2 * t + 1];
    const double* f = cores.data() + offsets[t];
    const double* m = f + static_cast<int64_t>(n1) * r1 + static_cast<int64_t>(j) * r1 * r2;
    const double* l = f + static_cast<int64_t>(n1) * r1 + static_cast<int64_t>(n2) * r1 * r2;
    double s = 0.0;
    for (int b = 0; b < r2; ++b) {
      double x = 0.0;
      for (int a = 0; a < r1; ++a) x += f[i + n1 * a] * m[a + r1 * b];
      s += x * l[b + r2 * k];
    }
    return s;
  }
};

// Mesh arrays the step consumes (UnstructuredMesh, proj/include/ttdvm/mesh.hpp:15-41).
struct MeshArrays {
  std::vector<int32_t> left, right, group;      // per face; right = -1 on boundary
  std::vector<double> area, normal;             // normal: 3 per face, out of left
  std::vector<double> volume;                   // per cell
  std::vector<int64_t> cell_face_off;           // ncell + 1
  std::vector<int32_t> cell_face_id;
  std::vector<int8_t> cell_face_sign;           // +1 iff the normal points out of the cell
};

class Solver {
 public:
  explicit Solver(int device = 0) { check(nullptr, ttdvm_cuda_create(device, &c_)); }
  ~Solver() {
    if (c_) ttdvm_cuda_destroy(c_);
  }
  Solver(const Solver&) = delete;
  Solver& operator=(const Solver&) = delete;

  // VelocityGrid(n, bound) (proj/src/velocity_grid.cpp:11-19)
  void set_grid(int n, double bound) { check(c_, ttdvm_cuda_set_grid(c_, n, bound)); }
  // GasParameters {m, R, Pr, mu_ref, T_ref, omega} (proj/include/ttdvm/physics.hpp:11-18)
  void set_gas(const std::array<double, 6>& g) { check(c_, ttdvm_cuda_set_gas(c_, g.data())); }
  void set_mesh(const MeshArrays& m) {
    check(c_, ttdvm_cuda_set_mesh(c_, static_cast<int32_t>(m.volume.size()),
                                  static_cast<int32_t>(m.left.size()), m.left.data(),
                                  m.right.data(), m.group.data(), m.area.data(), m.normal.data(),
                                  m.volume.data(), m.cell_face_off.data(), m.cell_face_id.data(),
                                  m.cell_face_sign.data()));
  }
  // BoundaryCondition per group (proj/src/boundary.cpp:45-82)
  void set_bcs(const std::vector<ttdvm_bc>& b) {
    check(c_, ttdvm_cuda_set_bcs(c_, static_cast<int32_t>(b.size()), b.data()));
  }
  void upload_state(const PackedTt& f) {
    const ttdvm_tt_batch v = f.view();
    check(c_, ttdvm_cuda_upload_state(c_, &v));
  }
  PackedTt download_state(int ncell, int n) const {
    PackedTt p;
    p.n1 = p.n2 = p.n3 = n;
    p.ranks.resize(2 * static_cast<size_t>(ncell));
    p.offsets.resize(static_cast<size_t>(ncell) + 1);
    check(c_, ttdvm_cuda_state_layout(c_, p.ranks.data(), p.offsets.data()));
    p.cores.resize(static_cast<size_t>(p.offsets.back()));
    check(c_, ttdvm_cuda_download_state(c_, p.cores.data(), p.offsets.back()));
    return p;
  }
  // SPEC.md:391 explicit_step, nsteps times, state resident on the device
  void explicit_step(double dt, double eps, int cap = 0, int nsteps = 1) {
    check(c_, ttdvm_cuda_step(c_, dt, eps, cap, nsteps));
  }
  // Macroparameters of the state the last step started from (11 per cell)
  std::vector<double> macros(int ncell) const {
    std::vector<double> out(11 * static_cast<size_t>(ncell));
    check(c_, ttdvm_cuda_macros(c_, out.data()));
    return out;
  }
  ttdvm_ctx* handle() const { return c_; }

 private:
  ttdvm_ctx* c_ = nullptr;
};

}  // namespace cuda
}  // namespace ttdvm

#endif  // TTDVM_CUDA_HPP_
