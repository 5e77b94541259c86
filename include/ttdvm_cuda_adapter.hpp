// ttdvm_cuda_adapter.hpp -- the drop-in on the REFERENCE'S OWN TYPES.
//
// A maintainer of the reference adds this header next to
// proj/include/ttdvm/*.hpp and links libttdvm_cuda.so: the explicit step
// then runs on the B200 behind the signature the reference's solver module
// specifies (SPEC.md:391 `explicit_step(state, mesh, grid, gas, problem,
// config) -> state`), taking and returning std::vector<ttdvm::TtTensor>
// (proj/include/ttdvm/tt_tensor.hpp:19-77), ttdvm::UnstructuredMesh
// (mesh.hpp:15-41), ttdvm::VelocityGrid, ttdvm::GasParameters
// (physics.hpp:11-18) and ttdvm::BoundaryCondition (boundary.hpp:13-41).
// Nothing here is elided: mesh flattening, packing of the Eigen column-major
// cores, boundary conditions, unpacking and the macroparameters are all
// below.  It is the only Eigen-dependent part of the repo's boundary; the
// C ABI under it (ttdvm_cuda.h) has plain pointers and sizes only.
//
// Compiled and run against the reference's headers by
// oracle/build_ref.py -> oracle/_ref/dropin_step (tests/test_dropin.py).
#ifndef TTDVM_CUDA_ADAPTER_HPP_
#define TTDVM_CUDA_ADAPTER_HPP_

#include <cmath>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "ttdvm/boundary.hpp"
#include "ttdvm/mesh.hpp"
#include "ttdvm/physics.hpp"
#include "ttdvm/tt_tensor.hpp"
#include "ttdvm/velocity_grid.hpp"
#include "ttdvm_cuda.hpp"

namespace ttdvm {
namespace cuda {

// UnstructuredMesh -> the flat arrays of ttdvm_cuda_set_mesh.  Faces keep
// their indices; each cell keeps its (face, sign) list in the reference's
// order (mesh.hpp:33-35), so the residual sums add the same summands in the
// same order as a loop over mesh.cell_faces.
inline MeshArrays flatten_mesh(const UnstructuredMesh& mesh) {
  MeshArrays m;
  const int nf = mesh.face_count(), nc = mesh.cell_count();
  m.left.resize(nf);
  m.right.resize(nf);
  m.group.resize(nf);
  m.area.resize(nf);
  m.normal.resize(3 * static_cast<size_t>(nf));
  for (int j = 0; j < nf; ++j) {
    const MeshFace& f = mesh.faces[j];
    m.left[j] = f.left;
    m.right[j] = f.right;
    m.group[j] = f.group;
    m.area[j] = f.area;
    for (int a = 0; a < 3; ++a) m.normal[3 * static_cast<size_t>(j) + a] = f.normal(a);
  }
  m.volume.assign(mesh.volumes.begin(), mesh.volumes.end());
  m.cell_face_off.resize(static_cast<size_t>(nc) + 1);
  m.cell_face_off[0] = 0;
  for (int i = 0; i < nc; ++i) {
    for (const auto& fs : mesh.cell_faces[i]) {
      m.cell_face_id.push_back(fs.first);
      m.cell_face_sign.push_back(static_cast<int8_t>(fs.second));
    }
    m.cell_face_off[i + 1] = static_cast<int64_t>(m.cell_face_id.size());
  }
  return m;
}

// BoundaryCondition per mesh group -> ttdvm_bc.  BcKind's enumerator order
// (boundary.hpp:13) is the C ABI's kind code.
inline std::vector<ttdvm_bc> flatten_bcs(const std::vector<BoundaryCondition>& bcs) {
  std::vector<ttdvm_bc> out(bcs.size());
  for (size_t g = 0; g < bcs.size(); ++g) {
    ttdvm_bc& b = out[g];
    std::memset(&b, 0, sizeof(b));
    switch (bcs[g].kind) {
      case BcKind::Wall: b.kind = 0; break;
      case BcKind::SymmetryX: b.kind = 1; break;
      case BcKind::SymmetryY: b.kind = 2; break;
      case BcKind::SymmetryZ: b.kind = 3; break;
      case BcKind::Inflow: b.kind = 4; break;
      case BcKind::Outflow: b.kind = 5; break;
    }
    b.wall_temperature = bcs[g].wall_temperature;
    b.free_n = bcs[g].free_n;
    b.free_t = bcs[g].free_t;
    for (int a = 0; a < 3; ++a) b.free_u[a] = bcs[g].free_u(a);
  }
  return out;
}

// std::vector<TtTensor> -> packed batch: the Eigen column-major cores back
// to back (first, middle slices in order, last), one memcpy per core matrix.
inline PackedTt pack(const std::vector<TtTensor>& f) {
  PackedTt p;
  p.offsets.push_back(0);
  size_t total = 0;
  for (const TtTensor& t : f) total += static_cast<size_t>(t.storage_count());
  p.cores.resize(total);
  double* dst = p.cores.data();
  for (const TtTensor& t : f) {
    if (t.empty()) throw std::invalid_argument("explicit_step: empty tensor in the state");
    const auto n = t.mode_sizes();
    const auto r = t.ranks();
    if (p.n1 == 0) {
      p.n1 = n[0];
      p.n2 = n[1];
      p.n3 = n[2];
    } else if (p.n1 != n[0] || p.n2 != n[1] || p.n3 != n[2]) {
      throw std::invalid_argument("explicit_step: mode sizes differ between cells");
    }
    p.ranks.push_back(r[1]);
    p.ranks.push_back(r[2]);
    auto put = [&](const Eigen::MatrixXd& m) {
      std::memcpy(dst, m.data(), sizeof(double) * static_cast<size_t>(m.size()));
      dst += m.size();
    };
    put(t.first_core());
    for (const Eigen::MatrixXd& g : t.middle_core()) put(g);
    put(t.last_core());
    p.offsets.push_back(static_cast<int64_t>(dst - p.cores.data()));
  }
  return p;
}

inline std::vector<TtTensor> unpack(const PackedTt& p) {
  std::vector<TtTensor> out;
  out.reserve(static_cast<size_t>(p.count()));
  for (int t = 0; t < p.count(); ++t) {
    const int r1 = p.ranks[2 * t], r2 = p.ranks[2 * t + 1];
    const double* src = p.cores.data() + p.offsets[t];
    Eigen::MatrixXd first(p.n1, r1), last(r2, p.n3);
    std::memcpy(first.data(), src, sizeof(double) * static_cast<size_t>(p.n1) * r1);
    src += static_cast<size_t>(p.n1) * r1;
    std::vector<Eigen::MatrixXd> middle(static_cast<size_t>(p.n2));
    for (int j = 0; j < p.n2; ++j) {
      middle[j].resize(r1, r2);
      std::memcpy(middle[j].data(), src, sizeof(double) * static_cast<size_t>(r1) * r2);
      src += static_cast<size_t>(r1) * r2;
    }
    std::memcpy(last.data(), src, sizeof(double) * static_cast<size_t>(r2) * p.n3);
    out.emplace_back(std::move(first), std::move(middle), std::move(last));
  }
  return out;
}

// The 11 doubles per cell of ttdvm_cuda_macros -> Macroparameters
// (physics.hpp:23-31); heat_flux as compute_macro derives it
// (proj/src/physics.cpp:62-65): q = 0.5 m (2RT)^{3/2} n S.
inline std::vector<Macroparameters> to_macros(const std::vector<double>& m, int ncell,
                                              const GasParameters& gas) {
  std::vector<Macroparameters> out(static_cast<size_t>(ncell));
  for (int i = 0; i < ncell; ++i) {
    const double* o = &m[11 * static_cast<size_t>(i)];
    Macroparameters& q = out[i];
    q.number_density = o[0];
    for (int a = 0; a < 3; ++a) q.velocity(a) = o[1 + a];
    q.temperature = o[4];
    q.mass_density = o[5];
    q.pressure = o[6];
    for (int a = 0; a < 3; ++a) q.shakhov_s(a) = o[7 + a];
    const double s = std::sqrt(2.0 * gas.gas_constant * q.temperature);
    const double s3 = std::pow(s, 3);
    for (int a = 0; a < 3; ++a)
      q.heat_flux(a) = 0.5 * gas.molecule_mass * s3 * q.number_density * q.shakhov_s(a);
  }
  return out;
}

// Bind a Solver (one per GPU) to a problem: grid, gas, mesh, BCs.  Call once;
// the one-time face-factor set-up happens at the first step.
inline void bind(Solver& s, const UnstructuredMesh& mesh, const VelocityGrid& grid,
                 const GasParameters& gas, const std::vector<BoundaryCondition>& bcs) {
  s.set_grid(grid.n(), grid.xi_max());
  s.set_gas({gas.molecule_mass, gas.gas_constant, gas.prandtl, gas.mu_ref, gas.t_ref, gas.omega});
  s.set_mesh(flatten_mesh(mesh));
  s.set_bcs(flatten_bcs(bcs));
}

// SPEC.md:391 explicit_step on the reference's types, on the GPU: `nsteps`
// explicit steps S1 of `state` (one TtTensor per mesh cell), the rounding
// tolerance `eps_round` and rank cap `max_rank` (0 = none) as
// TtTensor::rounded takes them.  macro_out, when given, receives the
// macroparameters of the state the LAST step started from (the moment pass
// compute_collision reports, physics.hpp:62-65).  Errors follow the
// reference: std::invalid_argument for argument/shape errors,
// std::runtime_error (with the cell or face id) for nonpositive density /
// temperature and wall-ghost failures.
inline std::vector<TtTensor> explicit_step(Solver& s, const std::vector<TtTensor>& state,
                                           const UnstructuredMesh& mesh,
                                           const VelocityGrid& grid, const GasParameters& gas,
                                           const std::vector<BoundaryCondition>& bcs, double dt,
                                           double eps_round, int max_rank = 0, int nsteps = 1,
                                           std::vector<Macroparameters>* macro_out = nullptr) {
  if (static_cast<int>(state.size()) != mesh.cell_count())
    throw std::invalid_argument("explicit_step: one tensor per mesh cell expected");
  bind(s, mesh, grid, gas, bcs);
  s.upload_state(pack(state));
  s.explicit_step(dt, eps_round, max_rank, nsteps);
  if (macro_out) *macro_out = to_macros(s.macros(mesh.cell_count()), mesh.cell_count(), gas);
  return unpack(s.download_state(mesh.cell_count(), grid.n()));
}

}  // namespace cuda
}  // namespace ttdvm

#endif  // TTDVM_CUDA_ADAPTER_HPP_
