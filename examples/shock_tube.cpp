// C++ host driver of the B200 step (north_star: "host code is C++ calling
// CUDA through a thin C-ABI layer"): BASELINE.json config 1 -- 64 x 1 x 1
// unit hexes, specular (sym-x) x-walls, y/z periodic (single-cell periodic
// axes cancel and are omitted, as in paper_1912_04582_b200/mesh.py),
// VelocityGrid(16, 5), Maxwellians (n, T) = (1, 1) | (0.125, 0.8) split at
// x = 32, u = 0, Pr = 2/3, omega = 0.5, Kn = 0.1, eps 1e-6.
//
//   shock_tube [steps] [out.bin]
//
// Writes the final state (ranks, offsets, cores) and the last macros to
// out.bin for the parity test (tests/test_cpp_host.py).  Exit code 3 means
// no usable CUDA device (the library has no CPU fallback).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <stdexcept>
#include <vector>

#include "ttdvm_cuda.hpp"

int main(int argc, char** argv) {
  const int steps = argc > 1 ? std::atoi(argv[1]) : 100;
  const char* out = argc > 2 ? argv[2] : nullptr;
  const int nx = 64, n = 16;
  const double bound = 5.0, kn = 0.1, eps = 1e-6;
  const double m = 1.0, R = 0.5, pr = 2.0 / 3.0, omega = 0.5;
  // mu_ref from Kn via the hard-sphere mean free path, L_ref = nx (problems.py)
  const double p0 = 1.0 * m * R * 1.0;
  const double mu_ref = kn * nx * p0 / std::sqrt(M_PI * R * 1.0 / 2.0);
  const double dt = 0.9 * 1.0 / (3.0 * bound);
  try {
    ttdvm::cuda::Solver s(0);
    s.set_grid(n, bound);
    s.set_gas({m, R, pr, mu_ref, 1.0, omega});
    // faces along x: interior i|i+1, then the two walls (normals out of the domain)
    ttdvm::cuda::MeshArrays mesh;
    for (int i = 0; i + 1 < nx; ++i) {
      mesh.left.push_back(i);
      mesh.right.push_back(i + 1);
      mesh.group.push_back(-1);
    }
    mesh.left.push_back(nx - 1), mesh.right.push_back(-1), mesh.group.push_back(1);  // xmax
    mesh.left.push_back(0), mesh.right.push_back(-1), mesh.group.push_back(0);       // xmin
    const int nface = static_cast<int>(mesh.left.size());
    mesh.area.assign(nface, 1.0);
    for (int f = 0; f < nface; ++f) {
      const double sx = f == nface - 1 ? -1.0 : 1.0;
      mesh.normal.insert(mesh.normal.end(), {sx, 0.0, 0.0});
    }
    mesh.volume.assign(nx, 1.0);
    mesh.cell_face_off.push_back(0);
    for (int c = 0; c < nx; ++c) {  // per-cell (face, sign), ascending face id
      std::vector<std::pair<int, int>> fs;
      for (int f = 0; f < nface; ++f) {
        if (mesh.left[f] == c) fs.push_back({f, +1});
        if (mesh.right[f] == c) fs.push_back({f, -1});
      }
      for (auto [f, sg] : fs) {
        mesh.cell_face_id.push_back(f);
        mesh.cell_face_sign.push_back(static_cast<int8_t>(sg));
      }
      mesh.cell_face_off.push_back(static_cast<int64_t>(mesh.cell_face_id.size()));
    }
    s.set_mesh(mesh);
    std::vector<ttdvm_bc> bcs(2);
    for (auto& b : bcs) b = ttdvm_bc{1, 0.0, 0.0, 0.0, {0.0, 0.0, 0.0}};  // sym-x
    s.set_bcs(bcs);
    // maxwell_tt(n, T, 0) per cell (proj/src/physics.cpp:69-87), rank 1
    ttdvm::cuda::PackedTt f;
    f.n1 = f.n2 = f.n3 = n;
    f.offsets.push_back(0);
    const double dxi = 2.0 * bound / (n - 1);
    for (int c = 0; c < nx; ++c) {
      const double nd = c < nx / 2 ? 1.0 : 0.125, t = c < nx / 2 ? 1.0 : 0.8;
      const double two_rt = 2.0 * R * t, norm1d = 1.0 / std::sqrt(M_PI * two_rt);
      for (int a = 0; a < 3; ++a)
        for (int i = 0; i < n; ++i) {
          const double v = -bound + i * dxi;
          double val = norm1d * std::exp(-v * v / two_rt);
          if (a == 0) val *= nd;
          f.cores.push_back(val);
        }
      f.ranks.push_back(1);
      f.ranks.push_back(1);
      f.offsets.push_back(static_cast<int64_t>(f.cores.size()));
    }
    s.upload_state(f);
    s.explicit_step(dt, eps, 0, steps);
    const ttdvm::cuda::PackedTt g = s.download_state(nx, n);
    const std::vector<double> mac = s.macros(nx);
    int rmax = 0;
    for (int r : g.ranks) rmax = r > rmax ? r : rmax;
    std::printf("shock_tube: %d steps, %d cells, max rank %d, n[0] %.6f n[%d] %.6f T[32] %.6f\n",
                steps, nx, rmax, mac[0], nx - 1, mac[11 * (nx - 1)], mac[11 * 32 + 4]);
    if (out) {
      std::ofstream o(out, std::ios::binary);
      const int32_t hdr[3] = {nx, n, steps};
      o.write(reinterpret_cast<const char*>(hdr), sizeof(hdr));
      o.write(reinterpret_cast<const char*>(g.ranks.data()), g.ranks.size() * 4);
      o.write(reinterpret_cast<const char*>(g.offsets.data()), g.offsets.size() * 8);
      o.write(reinterpret_cast<const char*>(g.cores.data()), g.cores.size() * 8);
      o.write(reinterpret_cast<const char*>(mac.data()), mac.size() * 8);
    }
  } catch (const std::invalid_argument& e) {
    std::fprintf(stderr, "invalid_argument: %s\n", e.what());
    return 2;
  } catch (const std::runtime_error& e) {
    std::fprintf(stderr, "runtime_error: %s\n", e.what());
    return 3;
  }
  return 0;
}
