// ref_step.cpp -- the explicit step S1 composed ONLY of calls into the
// unmodified reference library (proj/src/*.cpp, compiled by
// oracle/build_ref.py against the oracle/shim subsets), behind a small C ABI
// for ctypes.  TEST INFRASTRUCTURE: the parity checker and the CPU baseline;
// the product never links it.
//
// The step is not in the reference code.  This is the
// canonical composition of SURVEY.md §8(a) S1 -- PAPER.md:165-182 (Alg. 1,
// upwind signs) with SPEC.md:391-398's cadence:
//
//   xp = ((xi_normal(n) + abs_xi_estimate(n,4)).scaled(0.5)).rounded(1e-14)
//   xm = ((xi_normal(n) - abs_xi_estimate(n,4)).scaled(0.5)).rounded(1e-14)
//   Phi_j = (hadamard(xp, f_L) + hadamard(xm, f_R)).rounded(eps, cap)
//   J_i   = compute_collision(f_i, grid, gas, eps, macro_i)     physics.cpp:112-119
//   R_i   = (J_i + sum_j Phi_j.scaled(-s_ij A_j / V_i)).rounded(eps, cap)
//   f_i'  = (f_i + R_i.scaled(dt)).rounded(eps, cap)
//
// f_R: neighbour | symmetry_ghost (boundary.cpp:103-107) | freestream_ghost
// (boundary.hpp:51-53) | wall_ghost (boundary.cpp:84-101).  TtTensor ops
// are pure (tt_tensor.hpp:16-18), so faces and cells run under OpenMP; the
// face factors of distinct normals are computed in parallel on per-thread
// VelocityGrid instances (the reference's grid cache serialises misses under
// one mutex, velocity_grid.cpp:70) and reused from a solver-level cache.
#include <omp.h>

#include <array>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "ttdvm/boundary.hpp"
#include "ttdvm/physics.hpp"
#include "ttdvm/tt_tensor.hpp"
#include "ttdvm/velocity_grid.hpp"

using Eigen::MatrixXd;
using Eigen::Vector3d;
using ttdvm::TtTensor;

extern "C" {
typedef struct {
  int32_t count, n1, n2, n3;
  const int32_t* ranks;
  const int64_t* offsets;
  const double* cores;
} ttref_batch;  // same packing as ttdvm_tt_batch (include/ttdvm_cuda.h)

typedef struct {
  int32_t kind;  // 0 wall, 1 sym-x, 2 sym-y, 3 sym-z, 4 in, 5 out
  double wall_temperature;
  double free_n, free_t, free_u[3];
} ttref_bc;
}

namespace {

TtTensor unpack(const ttref_batch& b, int t) {
  const int r1 = b.ranks[2 * t], r2 = b.ranks[2 * t + 1];
  const double* p = b.cores + b.offsets[t];
  MatrixXd first(b.n1, r1), last(r2, b.n3);
  std::memcpy(first.data(), p, sizeof(double) * b.n1 * r1);
  p += (long)b.n1 * r1;
  std::vector<MatrixXd> middle(b.n2);
  for (int j = 0; j < b.n2; ++j) {
    middle[j].resize(r1, r2);
    std::memcpy(middle[j].data(), p, sizeof(double) * r1 * r2);
    p += (long)r1 * r2;
  }
  std::memcpy(last.data(), p, sizeof(double) * r2 * b.n3);
  return TtTensor(std::move(first), std::move(middle), std::move(last));
}

long packed_size(const TtTensor& t) { return t.empty() ? 0 : t.storage_count(); }

void pack_layout(const std::vector<TtTensor>& v, int32_t* ranks, int64_t* offsets) {
  int64_t o = 0;
  for (size_t i = 0; i < v.size(); ++i) {
    const auto r = v[i].empty() ? std::array<int, 4>{1, 0, 0, 1} : v[i].ranks();
    if (ranks) {
      ranks[2 * i] = r[1];
      ranks[2 * i + 1] = r[2];
    }
    if (offsets) offsets[i] = o;
    o += packed_size(v[i]);
  }
  if (offsets) offsets[v.size()] = o;
}

void pack_cores(const std::vector<TtTensor>& v, double* out) {
  for (const TtTensor& t : v) {
    if (t.empty()) continue;
    std::memcpy(out, t.first_core().data(), sizeof(double) * t.first_core().size());
    out += t.first_core().size();
    for (const MatrixXd& g : t.middle_core()) {
      std::memcpy(out, g.data(), sizeof(double) * g.size());
      out += g.size();
    }
    std::memcpy(out, t.last_core().data(), sizeof(double) * t.last_core().size());
    out += t.last_core().size();
  }
}

std::array<long long, 3> normal_key(const Vector3d& n) {
  return {std::llround(n(0) / 1e-12), std::llround(n(1) / 1e-12), std::llround(n(2) / 1e-12)};
}

struct Factors {
  TtTensor xp, xm;
  int grid = 0;  // per-thread grid holding this normal's cache entry
};

}  // namespace

struct ttref_solver {
  int nv = 0;
  double bound = 0.0;
  ttdvm::GasParameters gas{};
  std::vector<std::unique_ptr<ttdvm::VelocityGrid>> grids;  // [0] main + one per thread
  int nthreads = 1;
  // mesh
  int ncell = 0, nface = 0;
  std::vector<int> left, right, group;
  std::vector<double> area, volume;
  std::vector<Vector3d> normal;
  std::vector<long long> cfo;
  std::vector<int> cfid;
  std::vector<signed char> cfs;
  std::vector<ttdvm::BoundaryCondition> bcs;
  // state and outputs of the last step
  std::vector<TtTensor> f;
  std::map<std::array<long long, 3>, Factors> factors;
  std::vector<TtTensor> phi, jr, res, result;
  std::vector<int> last_cells;
  std::vector<double> macros;  // 11 per selected cell
  double step_s = 0.0, factor_s = 0.0;
  std::string err;
};

namespace {

template <class F>
int guard(ttref_solver* s, F&& fn) {
  if (!s) return 1;
  try {
    fn();
    s->err.clear();
    return 0;
  } catch (const std::invalid_argument& e) {
    s->err = e.what();
    return 1;
  } catch (const std::exception& e) {
    s->err = e.what();
    return 2;
  }
}

const ttdvm::VelocityGrid& main_grid(ttref_solver* s) { return *s->grids[0]; }

void ensure_grids(ttref_solver* s) {
  while ((int)s->grids.size() < s->nthreads + 1)
    s->grids.emplace_back(new ttdvm::VelocityGrid(s->nv, s->bound));
}

// xp / xm of every distinct normal among `faces` not yet cached (SURVEY.md
// §8(a) T13), computed in parallel, one VelocityGrid per thread.
void warm_factors(ttref_solver* s, const std::vector<int>& faces) {
  ensure_grids(s);
  std::vector<std::array<long long, 3>> keys;
  std::vector<Vector3d> todo;
  std::map<std::array<long long, 3>, int> seen;
  for (int j : faces) {
    const auto k = normal_key(s->normal[j]);
    if (s->factors.count(k) || seen.count(k)) continue;
    seen.emplace(k, (int)keys.size());
    keys.push_back(k);
    todo.push_back(s->normal[j]);
  }
  std::vector<Factors> out(todo.size());
  const auto t0 = std::chrono::steady_clock::now();
  std::string fail;
#pragma omp parallel for schedule(dynamic, 1) num_threads(s->nthreads)
  for (long i = 0; i < (long)todo.size(); ++i) {
    const int g = 1 + omp_get_thread_num();
    try {
      const ttdvm::VelocityGrid& grid = *s->grids[g];
      TtTensor xn = grid.xi_normal(todo[i]);
      const TtTensor& e = grid.abs_xi_estimate(todo[i], 4);
      out[i].xp = (xn + e).scaled(0.5).rounded(1e-14);
      out[i].xm = (xn - e).scaled(0.5).rounded(1e-14);
      out[i].grid = g;
    } catch (const std::exception& ex) {
#pragma omp critical
      fail = ex.what();
    }
  }
  if (!fail.empty()) throw std::runtime_error(fail);
  for (size_t i = 0; i < todo.size(); ++i) s->factors.emplace(keys[i], std::move(out[i]));
  s->factor_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

TtTensor ghost(ttref_solver* s, int face, const TtTensor& fl) {
  const int g = s->group[face];
  if (g < 0 || g >= (int)s->bcs.size()) throw std::invalid_argument("boundary face without a condition");
  const ttdvm::BoundaryCondition& bc = s->bcs[g];
  if (ttdvm::is_symmetry(bc.kind)) return ttdvm::symmetry_ghost(fl, ttdvm::symmetry_axis(bc.kind));
  if (bc.kind == ttdvm::BcKind::Inflow || bc.kind == ttdvm::BcKind::Outflow)
    return ttdvm::freestream_ghost(bc);
  const Factors& fa = s->factors.at(normal_key(s->normal[face]));
  return ttdvm::wall_ghost(fl, bc.wall_temperature, *s->grids[fa.grid], s->gas, s->normal[face], 4);
}

TtTensor face_flux(ttref_solver* s, int j, double eps, int cap) {
  const TtTensor& fl = s->f[s->left[j]];
  const int r = s->right[j];
  TtTensor fr_ghost;
  const TtTensor& fr = r >= 0 ? s->f[r] : (fr_ghost = ghost(s, j, fl));
  const Factors& fa = s->factors.at(normal_key(s->normal[j]));
  return (ttdvm::hadamard(fa.xp, fl) + ttdvm::hadamard(fa.xm, fr)).rounded(eps, cap);
}

void step(ttref_solver* s, double dt, double eps, int cap, const std::vector<int>& cells) {
  if ((int)s->f.size() != s->ncell) throw std::invalid_argument("state count must equal the cell count");
  std::vector<char> need(s->nface, 0);
  for (int c : cells)
    for (long long e = s->cfo[c]; e < s->cfo[c + 1]; ++e) need[s->cfid[e]] = 1;
  std::vector<int> faces;
  for (int j = 0; j < s->nface; ++j)
    if (need[j]) faces.push_back(j);
  warm_factors(s, faces);
  const auto t0 = std::chrono::steady_clock::now();
  s->phi.assign(s->nface, TtTensor());
  std::string fail;
#pragma omp parallel for schedule(dynamic, 8) num_threads(s->nthreads)
  for (long q = 0; q < (long)faces.size(); ++q) {
    try {
      s->phi[faces[q]] = face_flux(s, faces[q], eps, cap);
    } catch (const std::exception& ex) {
#pragma omp critical
      fail = ex.what();
    }
  }
  if (!fail.empty()) throw std::runtime_error(fail);
  const int nc = (int)cells.size();
  std::vector<TtTensor> fnew(nc);
  s->jr.assign(nc, TtTensor());
  s->res.assign(nc, TtTensor());
  s->macros.assign(11 * (size_t)nc, 0.0);
#pragma omp parallel for schedule(dynamic, 4) num_threads(s->nthreads)
  for (int q = 0; q < nc; ++q) {
    try {
      const int i = cells[q];
      ttdvm::Macroparameters m;
      TtTensor acc = ttdvm::compute_collision(s->f[i], main_grid(s), s->gas, eps, m);
      s->jr[q] = acc;
      for (long long e = s->cfo[i]; e < s->cfo[i + 1]; ++e) {
        const int fid = s->cfid[e];
        acc = acc + s->phi[fid].scaled(-s->cfs[e] * s->area[fid] / s->volume[i]);
      }
      TtTensor r = acc.rounded(eps, cap);
      fnew[q] = (s->f[i] + r.scaled(dt)).rounded(eps, cap);
      s->res[q] = std::move(r);
      double* o = &s->macros[11 * (size_t)q];
      o[0] = m.number_density;
      for (int a = 0; a < 3; ++a) o[1 + a] = m.velocity(a);
      o[4] = m.temperature;
      o[5] = m.mass_density;
      o[6] = m.pressure;
      for (int a = 0; a < 3; ++a) o[7 + a] = m.shakhov_s(a);
      o[10] = m.pressure / ttdvm::viscosity(m.temperature, s->gas);
    } catch (const std::exception& ex) {
#pragma omp critical
      fail = ex.what() + std::string(" (cell ") + std::to_string(cells[q]) + ")";
    }
  }
  if (!fail.empty()) throw std::runtime_error(fail);
  for (int q = 0; q < nc; ++q) s->f[cells[q]] = std::move(fnew[q]);
  s->last_cells = cells;
  s->step_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// One LU-SGS iteration from reference API calls only:
// the composition of SPEC.md:399-407 that oracle/step.py lusgs_step documents
// -- the explicit residual of S1, forward and backward Gauss-Seidel sweeps in
// cell index order with the first-order upwind Jacobian splitting, the
// diagonal replaced by the constant rank-1 over-estimate and divided out by
// TtTensor::divided_by_rank_one (tt_tensor.cpp:247-261).  Sequential sweeps
// (SPEC.md "Concurrency Model"); fluxes and residuals in parallel.
void lusgs(ttref_solver* s, double dt, double eps, int cap) {
  if ((int)s->f.size() != s->ncell) throw std::invalid_argument("state count must equal the cell count");
  std::vector<int> faces(s->nface);
  for (int j = 0; j < s->nface; ++j) faces[j] = j;
  warm_factors(s, faces);
  const int nc = s->ncell, n = s->nv;
  s->phi.assign(s->nface, TtTensor());
#pragma omp parallel for schedule(dynamic, 8) num_threads(s->nthreads)
  for (int j = 0; j < s->nface; ++j) s->phi[j] = face_flux(s, j, eps, cap);
  std::vector<TtTensor> res(nc);
  std::vector<double> diag(nc);
  s->macros.assign(11 * (size_t)nc, 0.0);
  const double xi_abs_max = std::sqrt(3.0) * s->bound;
#pragma omp parallel for schedule(dynamic, 4) num_threads(s->nthreads)
  for (int i = 0; i < nc; ++i) {
    ttdvm::Macroparameters m;
    TtTensor acc = ttdvm::compute_collision(s->f[i], main_grid(s), s->gas, eps, m);
    double sa = 0.0;
    for (long long e = s->cfo[i]; e < s->cfo[i + 1]; ++e) {
      const int fid = s->cfid[e];
      acc = acc + s->phi[fid].scaled(-s->cfs[e] * s->area[fid] / s->volume[i]);
      sa += s->area[fid];
    }
    res[i] = acc.rounded(eps, cap);
    const double nu = m.pressure / ttdvm::viscosity(m.temperature, s->gas);
    diag[i] = 1.0 / dt + nu + 0.5 * sa * xi_abs_max / s->volume[i];
    double* o = &s->macros[11 * (size_t)i];
    o[0] = m.number_density;
    for (int a = 0; a < 3; ++a) o[1 + a] = m.velocity(a);
    o[4] = m.temperature;
    o[5] = m.mass_density;
    o[6] = m.pressure;
    for (int a = 0; a < 3; ++a) o[7 + a] = m.shakhov_s(a);
    o[10] = nu;
  }
  const Eigen::VectorXd ones = Eigen::VectorXd::Ones(n);
  auto bracket = [&](int i, TtTensor acc, bool lower, const std::vector<TtTensor>& d) {
    for (long long e = s->cfo[i]; e < s->cfo[i + 1]; ++e) {
      const int fid = s->cfid[e];
      const int l = s->left[fid], r = s->right[fid];
      if (r < 0) continue;
      const int k = l == i ? r : l;
      if (lower ? !(k < i) : !(k > i)) continue;
      const Factors& fa = s->factors.at(normal_key(s->normal[fid]));
      const double w = s->area[fid] / s->volume[i];
      acc = acc + (l == i ? ttdvm::hadamard(fa.xm, d[k]).scaled(-w) : ttdvm::hadamard(fa.xp, d[k]).scaled(w));
    }
    return acc.rounded(eps, cap);
  };
  std::vector<TtTensor> bstar(nc), dstar(nc), delta(nc);
  for (int i = 0; i < nc; ++i) {
    bstar[i] = bracket(i, res[i], true, dstar);
    dstar[i] = bstar[i].divided_by_rank_one(diag[i] * ones, ones, ones);
  }
  for (int i = nc - 1; i >= 0; --i)
    delta[i] = bracket(i, bstar[i], false, delta).divided_by_rank_one(diag[i] * ones, ones, ones);
  std::vector<TtTensor> fnew(nc);
#pragma omp parallel for schedule(dynamic, 4) num_threads(s->nthreads)
  for (int i = 0; i < nc; ++i) fnew[i] = (s->f[i] + delta[i]).rounded(eps, cap);
  s->f = std::move(fnew);
  s->res = std::move(res);
  s->last_cells.resize(nc);
  for (int i = 0; i < nc; ++i) s->last_cells[i] = i;
}

std::vector<TtTensor> unpack_all(const ttref_batch* b) {
  if (!b || b->count < 0) throw std::invalid_argument("null batch");
  std::vector<TtTensor> v(b->count);
  for (int t = 0; t < b->count; ++t) v[t] = unpack(*b, t);
  return v;
}

}  // namespace

extern "C" {

ttref_solver* ttref_create(int nv, double bound, const double gas[6]) {
  auto* s = new ttref_solver;
  try {
    s->nv = nv;
    s->bound = bound;
    s->gas.molecule_mass = gas[0];
    s->gas.gas_constant = gas[1];
    s->gas.prandtl = gas[2];
    s->gas.mu_ref = gas[3];
    s->gas.t_ref = gas[4];
    s->gas.omega = gas[5];
    s->nthreads = omp_get_max_threads();
    s->grids.emplace_back(new ttdvm::VelocityGrid(nv, bound));
  } catch (const std::exception& e) {
    s->err = e.what();
  }
  return s;
}

void ttref_destroy(ttref_solver* s) { delete s; }
const char* ttref_last_error(ttref_solver* s) { return s ? s->err.c_str() : "null solver"; }

int ttref_set_threads(ttref_solver* s, int n) {
  return guard(s, [&] {
    s->nthreads = n > 0 ? n : omp_get_max_threads();
    ensure_grids(s);
  });
}

int ttref_set_mesh(ttref_solver* s, int32_t ncell, int32_t nface, const int32_t* left,
                   const int32_t* right, const int32_t* group, const double* area,
                   const double* normal, const double* volume, const int64_t* cfo,
                   const int32_t* cfid, const int8_t* cfs) {
  return guard(s, [&] {
    s->ncell = ncell;
    s->nface = nface;
    s->left.assign(left, left + nface);
    s->right.assign(right, right + nface);
    s->group.assign(group, group + nface);
    s->area.assign(area, area + nface);
    s->volume.assign(volume, volume + ncell);
    s->normal.resize(nface);
    for (int j = 0; j < nface; ++j)
      s->normal[j] = Vector3d(normal[3 * j], normal[3 * j + 1], normal[3 * j + 2]);
    s->cfo.assign(cfo, cfo + ncell + 1);
    s->cfid.assign(cfid, cfid + cfo[ncell]);
    s->cfs.assign(cfs, cfs + cfo[ncell]);
  });
}

int ttref_set_bcs(ttref_solver* s, int32_t ngroup, const ttref_bc* bcs) {
  return guard(s, [&] {
    s->bcs.clear();
    for (int g = 0; g < ngroup; ++g) {
      const ttref_bc& b = bcs[g];
      const Vector3d u(b.free_u[0], b.free_u[1], b.free_u[2]);
      switch (b.kind) {
        case 0: s->bcs.push_back(ttdvm::BoundaryCondition::wall(b.wall_temperature)); break;
        case 1: case 2: case 3: s->bcs.push_back(ttdvm::BoundaryCondition::symmetry(b.kind)); break;
        case 4:
          s->bcs.push_back(ttdvm::BoundaryCondition::freestream_in(b.free_n, b.free_t, u, main_grid(s), s->gas));
          break;
        case 5:
          s->bcs.push_back(ttdvm::BoundaryCondition::freestream_out(b.free_n, b.free_t, u, main_grid(s), s->gas));
          break;
        default: throw std::invalid_argument("unknown boundary condition kind");
      }
    }
  });
}

int ttref_set_state(ttref_solver* s, const ttref_batch* f) {
  return guard(s, [&] { s->f = unpack_all(f); });
}

// One explicit step of `ncells` selected cells (cells == NULL: all cells);
// the selected cells' states are replaced by their new states.
int ttref_step(ttref_solver* s, double dt, double eps, int32_t cap, int32_t ncells, const int32_t* cells) {
  return guard(s, [&] {
    if (!(eps > 0.0)) throw std::invalid_argument("rounded: eps must be > 0");
    std::vector<int> sel;
    if (cells) sel.assign(cells, cells + ncells);
    else
      for (int i = 0; i < s->ncell; ++i) sel.push_back(i);
    step(s, dt, eps, cap, sel);
  });
}

int ttref_lusgs_step(ttref_solver* s, double dt, double eps, int32_t cap) {
  return guard(s, [&] { lusgs(s, dt, eps, cap); });
}

int ttref_times(ttref_solver* s, double* step_s_and_factor_s) {
  return guard(s, [&] {
    step_s_and_factor_s[0] = s->step_s;
    step_s_and_factor_s[1] = s->factor_s;
  });
}

// Tensor sets for download: 0 state (all cells), 1 Phi (per face; faces the
// last step did not need have ranks 0), 2 J (per selected cell, with the nu
// scale), 3 R (per selected cell), 4 result of the last primitive call.
static std::vector<TtTensor>& tset(ttref_solver* s, int which) {
  switch (which) {
    case 0: return s->f;
    case 1: return s->phi;
    case 2: return s->jr;
    case 3: return s->res;
    case 4: return s->result;
    default: throw std::invalid_argument("unknown tensor set");
  }
}

int ttref_layout(ttref_solver* s, int32_t which, int32_t* count, int32_t* ranks, int64_t* offsets) {
  return guard(s, [&] {
    auto& v = tset(s, which);
    if (count) *count = (int32_t)v.size();
    if (ranks || offsets) pack_layout(v, ranks, offsets);
  });
}

int ttref_download(ttref_solver* s, int32_t which, double* cores) {
  return guard(s, [&] { pack_cores(tset(s, which), cores); });
}

int ttref_macros(ttref_solver* s, double* out) {
  return guard(s, [&] { std::memcpy(out, s->macros.data(), sizeof(double) * s->macros.size()); });
}

// Primitives (golden fixtures): results land in set 4.
// round(sum_{t in group} scale[t] * in[t], eps, cap) -- TtTensor::operator+,
// scaled and rounded (tt_tensor.cpp:139-193, 206-210, 290-312).
int ttref_round_sums(ttref_solver* s, const ttref_batch* in, int32_t nout, const int64_t* group_off,
                     const double* scale, double eps, int32_t cap) {
  return guard(s, [&] {
    std::vector<TtTensor> v = unpack_all(in);
    s->result.assign(nout, TtTensor());
    std::string fail;
#pragma omp parallel for schedule(dynamic, 1) num_threads(s->nthreads)
    for (int o = 0; o < nout; ++o) {
      try {
        const long g0 = group_off ? group_off[o] : o, g1 = group_off ? group_off[o + 1] : o + 1;
        TtTensor acc = v[g0].scaled(scale ? scale[g0] : 1.0);
        for (long t = g0 + 1; t < g1; ++t) acc = acc + v[t].scaled(scale ? scale[t] : 1.0);
        s->result[o] = acc.rounded(eps, cap);
      } catch (const std::exception& ex) {
#pragma omp critical
        fail = ex.what();
      }
    }
    if (!fail.empty()) throw std::invalid_argument(fail);
  });
}

// compute_macro per tensor (physics.cpp:17-67): 11 doubles as ttref_macros.
int ttref_compute_macro(ttref_solver* s, const ttref_batch* in, double* out) {
  return guard(s, [&] {
    std::vector<TtTensor> v = unpack_all(in);
    for (size_t t = 0; t < v.size(); ++t) {
      ttdvm::Macroparameters m = ttdvm::compute_macro(v[t], main_grid(s), s->gas);
      double* o = out + 11 * t;
      o[0] = m.number_density;
      for (int a = 0; a < 3; ++a) o[1 + a] = m.velocity(a);
      o[4] = m.temperature;
      o[5] = m.mass_density;
      o[6] = m.pressure;
      for (int a = 0; a < 3; ++a) o[7 + a] = m.shakhov_s(a);
      o[10] = m.pressure / ttdvm::viscosity(m.temperature, s->gas);
    }
  });
}

// compute_collision per tensor (physics.cpp:112-119): J (nu applied) in set 4.
int ttref_collision(ttref_solver* s, const ttref_batch* in, double eps) {
  return guard(s, [&] {
    std::vector<TtTensor> v = unpack_all(in);
    s->result.assign(v.size(), TtTensor());
    for (size_t t = 0; t < v.size(); ++t) s->result[t] = ttdvm::compute_collision(v[t], main_grid(s), s->gas, eps);
  });
}

// Face tensors per normal (velocity_grid.cpp:61-146): mode 0 abs_xi_estimate,
// 1 xi_normal_positive, 2 xi_normal_negative, 3 xp, 4 xm.
int ttref_face_factors(ttref_solver* s, int32_t count, const double* normals, int32_t cap, int32_t mode) {
  return guard(s, [&] {
    ensure_grids(s);
    s->result.assign(count, TtTensor());
    std::string fail;
#pragma omp parallel for schedule(dynamic, 1) num_threads(s->nthreads)
    for (int i = 0; i < count; ++i) {
      try {
        const ttdvm::VelocityGrid& g = *s->grids[1 + omp_get_thread_num()];
        const Vector3d n(normals[3 * i], normals[3 * i + 1], normals[3 * i + 2]);
        if (mode == 0) s->result[i] = g.abs_xi_estimate(n, cap);
        else if (mode == 1) s->result[i] = g.xi_normal_positive(n, cap);
        else if (mode == 2) s->result[i] = g.xi_normal_negative(n, cap);
        else {
          TtTensor xn = g.xi_normal(n);
          const TtTensor& e = g.abs_xi_estimate(n, cap);
          s->result[i] = (mode == 3 ? xn + e : xn - e).scaled(0.5).rounded(1e-14);
        }
      } catch (const std::exception& ex) {
#pragma omp critical
        fail = ex.what();
      }
    }
    if (!fail.empty()) throw std::invalid_argument(fail);
  });
}

}  // extern "C"
