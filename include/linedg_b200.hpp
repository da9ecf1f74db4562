// linedg_b200.hpp -- header-only C++ adapter: the reference's own setup
// objects in, the reconstructed hot-path API out, over the C-ABI of
// liblinedg_b200.so.  A reference-side caller includes this next to the
// reference headers (proj/include/linedg/*.hpp) and links liblinedg_b200.so.
//
//   linedg::b200::Context ctx(basis, mesh, mappings, &switches,
//                             linedg::b200::euler(gas, LDG_ROE));
//   linedg::GridFunction dUdt = ctx.residual_first_order(U, t);
//   ctx.assemble_jacobians(U, t);
//   std::vector<double> y = ctx.split_matvec(alpha_dt, v);
//
// Errors are rethrown as the reference's exception types (errors.hpp:10-28).
// Physics crosses as a descriptor (ldg_physics), not a PhysicsModel&:
// virtual per-point callbacks cannot run on the device.  Boundary data: the
// constant ldg_bc values per tag, or a BoundaryCondition-style
// std::function(x, t, out) per tag (set_boundary_function), evaluated on the
// host at the boundary end nodes.
#pragma once

#include <functional>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "linedg/basis.hpp"
#include "linedg/errors.hpp"
#include "linedg/field.hpp"
#include "linedg/mapping.hpp"
#include "linedg/mesh.hpp"
#include "linedg_b200.h"

namespace linedg {
namespace b200 {

inline ldg_physics euler(double gamma, int riemann = LDG_ROE) {
  ldg_physics p{};
  p.kind = LDG_EULER;
  p.riemann = riemann;
  p.gamma = gamma;
  p.prandtl = 0.72;
  return p;
}
inline ldg_physics navier_stokes(double gamma, double mu, double prandtl, int riemann = LDG_ROE) {
  ldg_physics p = euler(gamma, riemann);
  p.kind = LDG_NAVIER_STOKES;
  p.mu = mu;
  p.prandtl = prandtl;
  return p;
}
inline ldg_physics poisson(double c11_bd = 1.0) {
  ldg_physics p{};
  p.kind = LDG_POISSON;
  p.c11_bd = c11_bd;
  return p;
}

class Context {
 public:
  // NodalBasis1D (basis.hpp:17), QuadMesh (mesh.hpp:28), ElementMapping
  // (mapping.hpp:19), SwitchAssignment (mesh.hpp:74; may be null for
  // first-order physics).  The tables are copied; the inputs may go away.
  Context(const NodalBasis1D& b, const QuadMesh& mesh, const std::vector<ElementMapping>& maps,
          const SwitchAssignment* sw, const ldg_physics& physics, void* cuda_stream = nullptr) {
    const int np = b.p + 1, nq = b.n_quad(), E = mesh.num_elems(), npe = np * np;
    npe_ = npe;
    E_ = E;
    nodes_.assign(b.nodes.data(), b.nodes.data() + np);
    qp_.assign(b.quad_points.data(), b.quad_points.data() + nq);
    qw_.assign(b.quad_weights.data(), b.quad_weights.data() + nq);
    phi_.resize(np * nq);
    dphi_.resize(np * nq);
    for (int i = 0; i < np; ++i)
      for (int q = 0; q < nq; ++q) {
        phi_[i * nq + q] = b.phi_at_quad(i, q);
        dphi_[i * nq + q] = b.dphi_at_quad(i, q);
      }
    mass_.resize(np * np);
    for (int i = 0; i < np; ++i)
      for (int j = 0; j < np; ++j) mass_[i * np + j] = b.mass(i, j);
    for (const Face& f : mesh.faces) {
      fel_.push_back(f.elem_l);
      ffl_.push_back(f.face_l);
      fer_.push_back(f.elem_r);
      ffr_.push_back(f.face_r);
      fo_.push_back(f.reversed ? 1 : 0);
      ftag_.push_back(f.tag);
    }
    for (const auto& ef : mesh.elem_face) ef_.insert(ef_.end(), ef.begin(), ef.end());
    if (sw)
      for (const auto& s : sw->plus_sign) sw_.insert(sw_.end(), s.begin(), s.end());
    for (const ElementMapping& em : maps) {
      for (int n = 0; n < npe; ++n) {
        jac_.push_back(em.jac_at_nodes[n]);
        xy_.push_back(em.nodes_xy(0, n));
        xy_.push_back(em.nodes_xy(1, n));
      }
      for (int dir = 0; dir < 2; ++dir)
        for (int col = 0; col < np * nq; ++col)
          for (int d = 0; d < 2; ++d) nvec_.push_back(em.nvec_quad[dir](d, col));
      for (int dir = 0; dir < 2; ++dir)
        for (int side = 0; side < 2; ++side)
          for (int line = 0; line < np; ++line)
            for (int d = 0; d < 2; ++d) nend_.push_back(em.normal_end[dir][side](d, line));
    }
    ldg_setup s{};
    s.dim = 2;
    s.p = b.p;
    s.n_quad = nq;
    s.n_elems = E;
    s.n_faces = mesh.num_faces();
    s.nodes = nodes_.data();
    s.quad_points = qp_.data();
    s.quad_weights = qw_.data();
    s.phi_at_quad = phi_.data();
    s.dphi_at_quad = dphi_.data();
    s.mass = mass_.data();
    s.face_elem_l = fel_.data();
    s.face_face_l = ffl_.data();
    s.face_elem_r = fer_.data();
    s.face_face_r = ffr_.data();
    s.face_orient = fo_.data();
    s.face_tag = ftag_.data();
    s.elem_face = ef_.data();
    s.switch_plus = sw ? sw_.data() : nullptr;
    s.jac_at_nodes = jac_.data();
    s.nvec_quad = nvec_.data();
    s.normal_end = nend_.data();
    s.node_coords = xy_.data();
    check(ldg_create(&s, &physics, cuda_stream, &ctx_), nullptr);
    m_ = ldg_components(ctx_);
  }
  ~Context() { ldg_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;

  ldg_ctx* raw() const { return ctx_; }

  // residual_first_order / residual_primal, host buffers.
  GridFunction residual_first_order(const GridFunction& U, double t) {
    GridFunction R(U.n_elems, U.nodes_per_elem, U.comps);
    check(ldg_residual_host(ctx_, U.data.data(), t, R.data.data(), nullptr), ctx_);
    return R;
  }
  GridFunction residual_primal(const GridFunction& U, double t) { return residual_first_order(U, t); }

  // gradient_residual: Q = (1/J) sum_dir d, an AuxGradient with
  // component index c*2 + d (field.hpp:38-40).  Second-order physics.
  AuxGradient gradient_residual(const GridFunction& U, double t) {
    AuxGradient Q(U.n_elems, U.nodes_per_elem, U.comps * 2);
    check(ldg_gradient_host(ctx_, U.data.data(), t, Q.data.data()), ctx_);
    return Q;
  }
  // residual_second_order: R(U, Q) for a given Q.
  GridFunction residual_second_order(const GridFunction& U, const AuxGradient& Q, double t) {
    GridFunction R(U.n_elems, U.nodes_per_elem, U.comps);
    check(ldg_residual_uq_host(ctx_, U.data.data(), Q.data.data(), t, R.data.data()), ctx_);
    return R;
  }
  int components() const { return m_; }

  // assemble_jacobians(ctx, U, t, Analytic); the blocks stay on
  // the device for split_matvec / SpMV.
  void assemble_jacobians(const GridFunction& U, double t) {
    check(ldg_jacobian_assemble_host(ctx_, U.data.data(), t), ctx_);
  }

  // split_matvec: y = v - alpha_dt (K11 v + K12 (K21 v)).
  std::vector<double> split_matvec(double alpha_dt, const std::vector<double>& v) {
    std::vector<double> y(v.size());
    check(ldg_split_matvec_host(ctx_, alpha_dt, v.data(), y.data()), ctx_);
    return y;
  }

  // build_preconditioner(blocks, alpha_dt): block-Jacobi factors
  // of I - alpha_dt A~ on the device (after assemble_jacobians).
  void build_preconditioner(double alpha_dt) { check(ldg_precond_build(ctx_, alpha_dt), ctx_); }

  // Position/time-dependent boundary data for the condition on `tag`, with the
  // signature of BoundaryCondition::dirichlet / ::neumann (physics.hpp:22-23).
  using BoundaryFn = std::function<void(const Eigen::Vector2d&, double, double*)>;
  void set_boundary_function(int tag, BoundaryFn g) {
    if (!g) {
      check(ldg_set_boundary_function(ctx_, tag, nullptr, nullptr), ctx_);
      bfns_.erase(tag);
      return;
    }
    auto holder = std::make_unique<BoundaryFn>(std::move(g));
    check(ldg_set_boundary_function(ctx_, tag, &Context::boundary_trampoline, holder.get()), ctx_);
    bfns_[tag] = std::move(holder);
  }

  // gmres(split_matvec, precond, b, rtol, maxit, restart):
  // right-preconditioned GMRES on (I - alpha_dt (K11 + K12 K21)) x = b, x0 = 0.
  struct GmresResult {
    std::vector<double> x;
    int iterations = 0;
    bool converged = false;
    double residual_norm = 0.0;
  };
  GmresResult gmres(double alpha_dt, const std::vector<double>& b, double rtol, int maxit, int restart,
                    bool precond = true) {
    GmresResult out;
    out.x.assign(b.size(), 0.0);
    int32_t it = 0, conv = 0;
    check(ldg_gmres_host(ctx_, alpha_dt, b.data(), out.x.data(), rtol, maxit, restart, precond ? 1 : 0, &it, &conv,
                         &out.residual_norm),
          ctx_);
    out.iterations = it;
    out.converged = conv != 0;
    return out;
  }

  // Triplet export `i j value` of one matrix, scalar indices.
  struct Triplets {
    std::vector<long long> i, j;
    std::vector<double> v;
  };
  Triplets triplets(int which) {
    ldg_pattern_info info{};
    check(ldg_pattern_info_get(ctx_, which, &info), ctx_);
    std::vector<int64_t> rows(info.nnzb), cols(info.nnzb);
    std::vector<double> vals(info.nnzb * info.block_rows * info.block_cols);
    check(ldg_export_blocks(ctx_, which, rows.data(), cols.data(), vals.data()), ctx_);
    Triplets out;
    for (int64_t k = 0; k < info.nnzb; ++k)
      for (int a = 0; a < info.block_rows; ++a)
        for (int c = 0; c < info.block_cols; ++c) {
          out.i.push_back(rows[k] * info.block_rows + a);
          out.j.push_back(cols[k] * info.block_cols + c);
          out.v.push_back(vals[(k * info.block_rows + a) * info.block_cols + c]);
        }
    return out;
  }
  // Text wire formats: `i j value` triplet file and the
  // `p,avg_cols_per_block_row,nnz` sparsity summary.
  void write_triplets(int which, const std::string& path) {
    check(ldg_write_triplets(ctx_, which, path.c_str()), ctx_);
  }
  void write_sparsity_csv(int which, const std::string& path, bool append = false) {
    check(ldg_write_sparsity_csv(ctx_, which, path.c_str(), append ? 1 : 0), ctx_);
  }

 private:
  static void boundary_trampoline(void* user, const double* x, double t, double* out) {
    (*static_cast<BoundaryFn*>(user))(Eigen::Vector2d(x[0], x[1]), t, out);
  }
  std::map<int, std::unique_ptr<BoundaryFn>> bfns_;
  static void check(int status, const ldg_ctx* c) {
    if (status == LDG_OK) return;
    const std::string msg = ldg_last_error(c);
    if (status == LDG_ERR_PHYSICAL_STATE) {
      std::vector<double> st(8, 0.0);
      ldg_last_error_state(c, nullptr, nullptr, st.data());
      throw physical_state_error(msg, st);
    }
    if (status == LDG_ERR_CONFIG) throw config_error(msg);
    if (status == LDG_ERR_SOLVER) throw solver_error(msg);
    throw std::runtime_error(msg);
  }

  ldg_ctx* ctx_ = nullptr;
  int m_ = 1, npe_ = 1, E_ = 0;
  std::vector<double> nodes_, qp_, qw_, phi_, dphi_, mass_, jac_, nvec_, nend_, xy_;
  std::vector<int32_t> fel_, ffl_, fer_, ffr_, fo_, ftag_, ef_;
  std::vector<int8_t> sw_;
};

}  // namespace b200
}  // namespace linedg
