// dropin_step.cpp -- the drop-in boundary exercised on the REFERENCE'S OWN
// TYPES (TEST INFRASTRUCTURE; built by oracle/build_ref.py into
// oracle/_ref/dropin_step, run by tests/test_dropin.py on the GPU box).
//
// One program links both sides:
//   * the unmodified reference (proj/src/*.cpp against oracle/shim) -- it
//     builds the UnstructuredMesh (build_mesh), the VelocityGrid, the
//     boundary conditions and the initial TtTensor state, and steps them
//     with the S1 composition written below from reference API calls only;
//   * the product: include/ttdvm_cuda_adapter.hpp's
//     ttdvm::cuda::explicit_step(std::vector<TtTensor>, UnstructuredMesh,
//     VelocityGrid, GasParameters, std::vector<BoundaryCondition>, ...) over
//     libttdvm_cuda.so.
// Lock-step for a few steps on an 8x2x1 box (SPEC.md explicit_step example:
// "8-cell mesh, 16^3 grid") with an inflow, a diffuse wall and symmetry
// planes: per-cell dense difference <= 10 eps, identical ranks,
// macroparameters to 1e-8.  Exit code 0 = parity.
#include <cmath>
#include <cstdio>
#include <map>
#include <string>
#include <vector>

#include "ttdvm/boundary.hpp"
#include "ttdvm/mesh.hpp"
#include "ttdvm/physics.hpp"
#include "ttdvm/tt_tensor.hpp"
#include "ttdvm/velocity_grid.hpp"
#include "ttdvm_cuda_adapter.hpp"

using Eigen::Vector3d;
using namespace ttdvm;

namespace {

// nx x ny x nz unit hexes, VTK vertex order; boundary quads tagged by side
UnstructuredMesh box(int nx, int ny, int nz) {
  auto vid = [&](int i, int j, int k) { return (k * (ny + 1) + j) * (nx + 1) + i; };
  std::vector<Vector3d> v;
  for (int k = 0; k <= nz; ++k)
    for (int j = 0; j <= ny; ++j)
      for (int i = 0; i <= nx; ++i) v.emplace_back(i, j, k);
  std::vector<std::array<int, 8>> cells;
  std::vector<BoundaryQuad> bnd;
  for (int k = 0; k < nz; ++k)
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) {
        cells.push_back({vid(i, j, k), vid(i + 1, j, k), vid(i + 1, j + 1, k), vid(i, j + 1, k),
                         vid(i, j, k + 1), vid(i + 1, j, k + 1), vid(i + 1, j + 1, k + 1),
                         vid(i, j + 1, k + 1)});
        auto quad = [&](std::array<int, 4> q, const char* g) { bnd.push_back({q, g}); };
        if (i == 0) quad({vid(0, j, k), vid(0, j + 1, k), vid(0, j + 1, k + 1), vid(0, j, k + 1)}, "in");
        if (i == nx - 1)
          quad({vid(nx, j, k), vid(nx, j + 1, k), vid(nx, j + 1, k + 1), vid(nx, j, k + 1)}, "wall");
        if (j == 0) quad({vid(i, 0, k), vid(i + 1, 0, k), vid(i + 1, 0, k + 1), vid(i, 0, k + 1)}, "sym-y");
        if (j == ny - 1)
          quad({vid(i, ny, k), vid(i + 1, ny, k), vid(i + 1, ny, k + 1), vid(i, ny, k + 1)}, "sym-y");
        if (k == 0) quad({vid(i, j, 0), vid(i + 1, j, 0), vid(i + 1, j + 1, 0), vid(i, j + 1, 0)}, "sym-z");
        if (k == nz - 1)
          quad({vid(i, j, nz), vid(i + 1, j, nz), vid(i + 1, j + 1, nz), vid(i, j + 1, nz)}, "sym-z");
      }
  return build_mesh(std::move(v), std::move(cells), bnd);
}

// S1 from reference calls only (Alg. 1 with
// upwind signs; SPEC.md:391-398 cadence).
std::vector<TtTensor> reference_step(const std::vector<TtTensor>& f, const UnstructuredMesh& mesh,
                                     const VelocityGrid& grid, const GasParameters& gas,
                                     const std::vector<BoundaryCondition>& bcs, double dt,
                                     double eps, int cap, std::vector<Macroparameters>& macros) {
  std::vector<TtTensor> phi(mesh.face_count());
  for (int j = 0; j < mesh.face_count(); ++j) {
    const MeshFace& fc = mesh.faces[j];
    const TtTensor& fl = f[fc.left];
    TtTensor fr;
    if (fc.right >= 0) {
      fr = f[fc.right];
    } else {
      const BoundaryCondition& bc = bcs[fc.group];
      if (is_symmetry(bc.kind)) fr = symmetry_ghost(fl, symmetry_axis(bc.kind));
      else if (bc.kind == BcKind::Wall) fr = wall_ghost(fl, bc.wall_temperature, grid, gas, fc.normal, 4);
      else fr = freestream_ghost(bc);
    }
    const TtTensor xn = grid.xi_normal(fc.normal), e = grid.abs_xi_estimate(fc.normal, 4);
    const TtTensor xp = (xn + e).scaled(0.5).rounded(1e-14), xm = (xn - e).scaled(0.5).rounded(1e-14);
    phi[j] = (xp.hadamard(fl) + xm.hadamard(fr)).rounded(eps, cap);
  }
  std::vector<TtTensor> out(f.size());
  macros.resize(f.size());
  for (int i = 0; i < mesh.cell_count(); ++i) {
    TtTensor acc = compute_collision(f[i], grid, gas, eps, macros[i]);
    for (const auto& [fid, sign] : mesh.cell_faces[i])
      acc = acc + phi[fid].scaled(-sign * mesh.faces[fid].area / mesh.volumes[i]);
    const TtTensor r = acc.rounded(eps, cap);
    out[i] = (f[i] + r.scaled(dt)).rounded(eps, cap);
  }
  return out;
}

double rel_diff(const TtTensor& a, const TtTensor& b) {
  const Dense3 x = a.to_full(), y = b.to_full();
  double num = 0.0, den = 0.0;
  const auto n = a.mode_sizes();
  for (int i = 0; i < n[0]; ++i)
    for (int j = 0; j < n[1]; ++j)
      for (int k = 0; k < n[2]; ++k) {
        const double d = x(i, j, k) - y(i, j, k);
        num += d * d;
        den += y(i, j, k) * y(i, j, k);
      }
  return std::sqrt(num / den);
}

}  // namespace

int main(int argc, char** argv) {
  const int steps = argc > 1 ? std::atoi(argv[1]) : 3;
  const UnstructuredMesh mesh = box(8, 2, 1);
  const VelocityGrid grid(16, 5.0);
  GasParameters gas;
  gas.molecule_mass = 1.0;
  gas.gas_constant = 0.5;
  gas.prandtl = 2.0 / 3.0;
  gas.mu_ref = 0.4;
  gas.t_ref = 1.0;
  gas.omega = 0.5;
  const Vector3d u0(0.4, 0.0, 0.0);
  std::map<std::string, BoundaryCondition> by_name = {
      {"in", BoundaryCondition::freestream_in(1.0, 1.0, u0, grid, gas)},
      {"wall", BoundaryCondition::wall(1.2)},
      {"sym-y", BoundaryCondition::symmetry(2)},
      {"sym-z", BoundaryCondition::symmetry(3)}};
  std::vector<BoundaryCondition> bcs;
  for (const std::string& g : mesh.group_names) bcs.push_back(by_name.at(g));
  std::vector<TtTensor> f;
  for (int i = 0; i < mesh.cell_count(); ++i) {
    const double x = mesh.centroids[i](0), y = mesh.centroids[i](1);
    f.push_back(maxwell_tt(1.0 + 0.1 * std::sin(x), 1.0 + 0.05 * std::cos(x + y),
                           Vector3d(0.4 - 0.03 * x, 0.02 * y, 0.0), grid, gas));
  }
  const double dt = 0.9 / (3.0 * grid.xi_max()), eps = 1e-6;
  cuda::Solver solver(0);
  double worst = 0.0, worst_macro = 0.0;
  int rank_mismatch = 0;
  for (int it = 0; it < steps; ++it) {
    std::vector<Macroparameters> mref, mgpu;
    const std::vector<TtTensor> want = reference_step(f, mesh, grid, gas, bcs, dt, eps, 0, mref);
    const std::vector<TtTensor> got =
        cuda::explicit_step(solver, f, mesh, grid, gas, bcs, dt, eps, 0, 1, &mgpu);
    for (int i = 0; i < mesh.cell_count(); ++i) {
      worst = std::max(worst, rel_diff(got[i], want[i]));
      if (got[i].ranks() != want[i].ranks()) ++rank_mismatch;
      auto rel = [](double a, double b) { return std::fabs(a - b) / std::max(std::fabs(b), 1.0); };
      worst_macro = std::max({worst_macro, rel(mgpu[i].number_density, mref[i].number_density),
                              rel(mgpu[i].temperature, mref[i].temperature),
                              rel(mgpu[i].pressure, mref[i].pressure)});
      for (int a = 0; a < 3; ++a)
        worst_macro = std::max({worst_macro, rel(mgpu[i].velocity(a), mref[i].velocity(a)),
                                rel(mgpu[i].shakhov_s(a), mref[i].shakhov_s(a)),
                                rel(mgpu[i].heat_flux(a), mref[i].heat_flux(a))});
    }
    f = want;  // lock-step: both sides start every step from the reference's state
  }
  std::printf("dropin_step: %d cells, %d steps, max rel err %.3e (bar %.1e), macro %.3e (bar 1e-8), "
              "rank mismatches %d\n",
              mesh.cell_count(), steps, worst, 10 * eps, worst_macro, rank_mismatch);
  const bool ok = worst <= 10 * eps && worst_macro <= 1e-8 && rank_mismatch == 0;
  std::printf(ok ? "dropin ok\n" : "dropin FAILED\n");
  return ok ? 0 : 1;
}
