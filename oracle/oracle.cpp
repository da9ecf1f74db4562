// oracle.cpp -- TEST INFRASTRUCTURE ONLY: the CPU parity oracle and the CPU
// baseline of the Line-DG hot path.  Never linked or loaded by the product.
//
// A from-scratch CPU restatement of the reference operations whose sources
// are absent from the reference tree (proj/src/CMakeLists.txt:5-8):
//   line_divergence / residual_first_order
//   gradient_residual
//   residual_second_order / residual_primal
//   assemble_jacobians (Analytic + FD)
//   CscMatrix, split_matvec
//   build_preconditioner, gmres
//   rk4_step, dirk3_step (Newton, reuse)
// It follows the reference's numerics literally where they are specified:
// r = M^-1 b through the Cholesky factor of M column by column
// (basis.cpp:81-88, 185-189), fluxes at the quadrature points of the
// interpolated state, point-wise endpoint fluxes with the
// precomputed non-normalised normals, dU/dt =
// S - (1/J)(r^1 + ... + r^D), exact Jacobians through Dual<N>
// (dual.hpp:8-10).  Inputs are the flattened reference setup objects
// (include/linedg_b200.h: ldg_setup), read verbatim.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "linedg_b200.h"
#include "oracle_physics.hpp"

#ifdef _OPENMP
#include <omp.h>
#endif

namespace ora {

namespace {
constexpr int MAXNP = 8, MAXNQ = 12, MAXM = 5, MAXD = 3;
}

// Node-level block matrix (compressed rows) with dense br x bc blocks.
struct BlockMat {
  int br = 0, bc = 0;
  int64_t nrows = 0;
  std::vector<int64_t> rowptr;  // nrows+1
  std::vector<int64_t> col;     // node columns, ascending per row
  std::vector<double> val;      // nnzb * br * bc
  bool built = false;
  bool subset = false;
  int64_t find(int64_t row, int64_t c) const {
    const int64_t* b = col.data() + rowptr[row];
    const int64_t* e = col.data() + rowptr[row + 1];
    const int64_t* it = std::lower_bound(b, e, c);
    return (it != e && *it == c) ? (it - col.data()) : -1;
  }
};

struct Ctx {
  int D = 2, p = 1, np = 2, nq = 2, npe = 4, NL = 2, m = 1, E = 0;
  int kind = LDG_EULER, riemann = LDG_ROE;
  bool second = false, has_inv = false, vis_u = false;
  Gas gas;
  double c11 = 0.0, c11_bd = 0.0;
  std::vector<double> qw, phi, dphi, L;  // L: Cholesky factor of M (lower, row-major)
  std::vector<int8_t> sw;
  std::vector<double> jac, invJ, nvec, nend, source;
  // Endpoint table [E][D][2][NL]: neighbour element / node, or boundary.
  std::vector<int32_t> ep_elem, ep_node, ep_bc;  // ep_bc: -1 interior, else index in bcv
  std::vector<std::vector<double>> bcv;          // boundary data (g_D / g_N / far-field state)
  std::vector<int> bck;                          // boundary kind per bcv entry (ldg_bc_kind)
  std::vector<int> bctag;                        // mesh tag per bcv entry
  // boundary functions: end-node coordinates per line end [E][D][2][NL][D],
  // per-line-end data ep_g [E][D][2][NL][m] when any function is registered
  std::vector<double> ep_x, ep_g;
  std::map<int, std::pair<ldg_bc_fn, void*>> bfun;
  double bfun_t = 0.0;
  bool bfun_dirty = false;
  BlockMat K[3];
  // block-Jacobi preconditioner: per element LU (partial pivoting) of
  // I - alpha_dt A~ restricted to the element (dense n_e x n_e, row-major)
  std::vector<double> pcLU;
  std::vector<int32_t> pcPiv;
  bool pc_built = false;
  int pc_inverse = 0;  // 0 LU solves, 1 explicit block inverse (ldg_set_precond_mode)
  int pc_mode = 0;     // ldg_set_precond_mode: 0 auto, 1 element inverse, 2 line-ADI
  bool pc_adi = false; // the built preconditioner is the line-ADI one
  double pc_adt = 0.0;
  std::string err;
  std::vector<double> err_state;
  int err_elem = -1, err_node = -1;

  int node_on_line(int dir, int line, int t) const {
    if (D == 2) return dir == 0 ? t + np * line : line + np * t;
    const int l1 = line % np, l2 = line / np;
    const int st[3] = {1, np, np * np};
    const int a1 = dir == 0 ? 1 : 0, a2 = dir == 2 ? 1 : 2;
    return t * st[dir] + l1 * st[a1] + l2 * st[a2];
  }
  size_t epi(int e, int dir, int side, int line) const {
    return ((static_cast<size_t>(e) * D + dir) * 2 + side) * NL + line;
  }
  const double* nv(int e, int dir, int line, int q) const {
    return &nvec[((((static_cast<size_t>(e) * D + dir) * NL + line) * nq) + q) * D];
  }
  const double* ne(int e, int dir, int side, int line) const {
    return &nend[epi(e, dir, side, line) * D];
  }
  int sign(int e, int dir, int side) const {
    const int s = sw.empty() ? 1 : sw[static_cast<size_t>(e) * D + dir];
    return side ? s : -s;
  }
  // Cholesky solve of one column in place (basis.cpp:81-88).
  template <class T>
  void mass_solve(T* x, int stride) const {
    T y[MAXNP];
    for (int i = 0; i < np; ++i) {
      T s = x[i * stride];
      for (int j = 0; j < i; ++j) s -= L[i * np + j] * y[j];
      y[i] = s / L[i * np + i];
    }
    for (int i = np - 1; i >= 0; --i) {
      T s = y[i];
      for (int j = i + 1; j < np; ++j) s -= L[j * np + i] * x[j * stride];
      x[i * stride] = s / L[i * np + i];
    }
  }
};

namespace {

// Face node of local face lf at face parameter(s): 2-D follows
// face_node_indices (mesh.cpp:51-65); 3-D: node with index side*p along the
// face direction and (a,b) along the two transverse axes in increasing order.
int face_node(const Ctx& c, int lf, int a, int b) {
  const int p = c.p, np = c.np;
  if (c.D == 2) {
    switch (lf) {
      case 0: return a;
      case 1: return p + np * a;
      case 2: return (p - a) + np * p;
      default: return np * (p - a);
    }
  }
  const int dir = lf / 2, side = lf % 2;
  const int st[3] = {1, np, np * np};
  const int a1 = dir == 0 ? 1 : 0, a2 = dir == 2 ? 1 : 2;
  return side * p * st[dir] + a * st[a1] + b * st[a2];
}

int lface_of(int D, int dir, int side) {
  if (D == 2) return dir == 0 ? (side ? 1 : 3) : (side ? 2 : 0);
  return 2 * dir + side;
}

void dihedral(int o, int a, int b, int p, int& ao, int& bo) {
  int x = a, y = b;
  if (o & 1) std::swap(x, y);
  ao = (o & 2) ? p - x : x;
  bo = (o & 4) ? p - y : y;
}

void build_endpoints(Ctx& c, const ldg_setup& s, const ldg_physics& ph) {
  const size_t n = static_cast<size_t>(c.E) * c.D * 2 * c.NL;
  c.ep_elem.assign(n, -1);
  c.ep_node.assign(n, -1);
  c.ep_bc.assign(n, -1);
  std::map<int, int> tag2bc;
  for (int i = 0; i < ph.n_bc; ++i) {
    const int kind = ph.bcs[i].kind;
    if (kind < LDG_BC_DIRICHLET || kind > LDG_BC_NO_SLIP_ADIABATIC)
      throw std::runtime_error("oracle: unsupported boundary-condition kind");
    if ((kind == LDG_BC_SLIP_WALL || kind == LDG_BC_NO_SLIP_ADIABATIC) && !c.has_inv)
      throw std::runtime_error("oracle: slip-wall boundaries need Euler or Navier-Stokes physics");
    tag2bc[ph.bcs[i].tag] = static_cast<int>(c.bcv.size());
    c.bcv.emplace_back(ph.bcs[i].value, ph.bcs[i].value + c.m);
    c.bck.push_back(kind);
    c.bctag.push_back(ph.bcs[i].tag);
  }
  const int F = 2 * c.D;
  for (int e = 0; e < c.E; ++e)
    for (int dir = 0; dir < c.D; ++dir)
      for (int side = 0; side < 2; ++side) {
        const int lf = lface_of(c.D, dir, side);
        const int fid = s.elem_face[static_cast<size_t>(e) * F + lf];
        if (fid < 0 || fid >= s.n_faces) throw std::runtime_error("oracle: bad elem_face entry");
        const bool bdry = s.face_elem_r[fid] < 0;
        int bci = -1;
        if (bdry) {
          auto it = tag2bc.find(s.face_tag[fid]);
          if (it == tag2bc.end())
            throw std::runtime_error("oracle: no boundary condition for tag " +
                                     std::to_string(s.face_tag[fid]));
          bci = it->second;
        }
        const bool is_left = s.face_elem_l[fid] == e && s.face_face_l[fid] == lf;
        const int oe = is_left ? s.face_elem_r[fid] : s.face_elem_l[fid];
        const int olf = is_left ? s.face_face_r[fid] : s.face_face_l[fid];
        const int code = s.face_orient[fid];
        for (int line = 0; line < c.NL; ++line) {
          const size_t k = c.epi(e, dir, side, line);
          if (bdry) {
            c.ep_bc[k] = bci;
            continue;
          }
          const int own = c.node_on_line(dir, line, side ? c.p : 0);
          int na = -1, nb = 0;
          if (c.D == 2) {
            int kk = -1;
            for (int t = 0; t <= c.p; ++t)
              if (face_node(c, lf, t, 0) == own) kk = t;
            na = code ? c.p - kk : kk;  // Face::reversed (mesh.hpp:18-22)
          } else {
            const int a = line % c.np, b = line / c.np;
            if (is_left) {
              dihedral(code, a, b, c.p, na, nb);
            } else {  // inverse transform
              for (int x = 0; x <= c.p && na < 0; ++x)
                for (int y = 0; y <= c.p; ++y) {
                  int ra, rb;
                  dihedral(code, x, y, c.p, ra, rb);
                  if (ra == a && rb == b) {
                    na = x;
                    nb = y;
                    break;
                  }
                }
            }
          }
          c.ep_elem[k] = oe;
          c.ep_node[k] = face_node(c, olf, na, nb);
        }
      }
}

// ----------------------------------------------------------- point fluxes

// Physical flux dotted with n: inviscid + viscous parts.
template <class T>
void flux_dot(const Ctx& c, const T* u, const T* q, const double* n, T* out) {
  const int D = c.D, m = c.m;
  T F[MAXM * MAXD], G[MAXM * MAXD];
  for (int i = 0; i < m * D; ++i) F[i] = 0.0;
  if (c.has_inv) euler_flux(D, u, c.gas, F);
  if (c.second) {
    if (c.kind == LDG_POISSON) {
      for (int d = 0; d < D; ++d) G[d] = -q[d];
    } else {
      ns_viscous_flux(D, u, q, c.gas, G);
    }
    for (int i = 0; i < m * D; ++i) F[i] = F[i] + G[i];
  }
  for (int cc = 0; cc < m; ++cc) {
    T s = 0.0;
    for (int d = 0; d < D; ++d) s = s + F[cc * D + d] * n[d];
    out[cc] = s;
  }
}

// Viscous flux only, dotted with n.
template <class T>
void vflux_dot(const Ctx& c, const T* u, const T* q, const double* n, T* out) {
  const int D = c.D, m = c.m;
  T G[MAXM * MAXD];
  if (c.kind == LDG_POISSON) {
    for (int d = 0; d < D; ++d) G[d] = -q[d];
  } else {
    ns_viscous_flux(D, u, q, c.gas, G);
  }
  for (int cc = 0; cc < m; ++cc) {
    T s = 0.0;
    for (int d = 0; d < D; ++d) s = s + G[cc * D + d] * n[d];
    out[cc] = s;
  }
}

double norm_of(const double* n, int D) {
  double s = 0.0;
  for (int d = 0; d < D; ++d) s += n[d] * n[d];
  return std::sqrt(s);
}

// u_hat of a boundary end is the interior trace (Neumann-type with C22 = 0,
// PAPER.md:580; slip wall), else the prescribed state.
inline bool uhat_inner(int bkind) {
  return bkind == LDG_BC_NEUMANN || bkind == LDG_BC_SLIP_WALL || bkind == LDG_BC_NO_SLIP_ADIABATIC;
}
// per component: the no-slip adiabatic wall is mixed -- Dirichlet
// zero momentum (u_hat = 0), Neumann density and energy (u_hat = u_in)
inline bool uhat_inner_c(int bkind, int comp, int m) {
  if (bkind == LDG_BC_NO_SLIP_ADIABATIC) return comp == 0 || comp == m - 1;
  return uhat_inner(bkind);
}

// Endpoint numerical flux F_hat . n (inviscid Riemann + LDG viscous switch
// flux; boundaries PAPER.md:566-582).
//   interior: uo/qo are the neighbour's node values; bc == nullptr
//   boundary: bc = the boundary data, bkind its ldg_bc_kind, uo/qo ignored:
//     Dirichlet / characteristic: Riemann vs g, + F(u,q).n + C11_bd|n|(u - g)
//     slip wall: Riemann vs the interior state with mirrored normal momentum
//                (a function of u_in, so Dual seeds carry through), + F(u,q).n
//     Neumann:   the prescribed normal flux g_N |n|
template <class T>
void endpoint_flux(const Ctx& c, const T* ui, const T* qi, const T* uo, const T* qo,
                   const double* bc, int bkind, const double* n, int S, T* out) {
  const int m = c.m, D = c.D;
  for (int k = 0; k < m; ++k) out[k] = 0.0;
  const double nn = norm_of(n, D);
  if (bc && bkind == LDG_BC_NEUMANN) {
    for (int k = 0; k < m; ++k) out[k] = bc[k] * nn;
    return;
  }
  if (c.has_inv) {
    T g[MAXM];
    const T* other = uo;
    if (bc && bkind == LDG_BC_NO_SLIP_ADIABATIC) {
      // no-slip wall: the interior state with its full momentum reversed
      g[0] = ui[0];
      for (int d = 0; d < D; ++d) g[1 + d] = -ui[1 + d];
      g[m - 1] = ui[m - 1];
      other = g;
    } else if (bc && bkind == LDG_BC_SLIP_WALL) {
      double n2 = 0.0;
      for (int d = 0; d < D; ++d) n2 += n[d] * n[d];
      T mn = ui[1] * n[0];
      for (int d = 1; d < D; ++d) mn = mn + ui[1 + d] * n[d];
      const T f = mn * (2.0 / n2);
      g[0] = ui[0];
      for (int d = 0; d < D; ++d) g[1 + d] = ui[1 + d] - f * n[d];
      g[m - 1] = ui[m - 1];
      other = g;
    } else if (bc) {
      for (int k = 0; k < m; ++k) g[k] = bc[k];
      other = g;
    }
    if (c.riemann == LDG_ROE) roe_flux(D, other, ui, n, c.gas, out);
    else llf_flux(D, other, ui, n, c.gas, out);
  }
  if (c.second) {
    T fv[MAXM];
    if (bc) {
      vflux_dot(c, ui, qi, n, fv);
      if (bkind == LDG_BC_SLIP_WALL) {
        for (int k = 0; k < m; ++k) out[k] = out[k] + fv[k];
      } else if (bkind == LDG_BC_NO_SLIP_ADIABATIC) {
        // momentum: Dirichlet zero velocity, F(u,q).n + C11_bd |n| (m - 0);
        // density: F(u,q).n (zero row); energy: zero normal flux (adiabatic, no wall work)
        const double c11 = c.c11_bd * c.p * c.p / std::pow(nn, 1.0 / (D - 1));
        out[0] = out[0] + fv[0];
        for (int k = 1; k < m - 1; ++k) out[k] = out[k] + fv[k] + c11 * nn * ui[k];
      } else {
        const double c11 = c.c11_bd * c.p * c.p / std::pow(nn, 1.0 / (D - 1));
        for (int k = 0; k < m; ++k) out[k] = out[k] + fv[k] + c11 * nn * (ui[k] - bc[k]);
      }
    } else {
      if (S > 0) vflux_dot(c, uo, qo, n, fv);
      else vflux_dot(c, ui, qi, n, fv);
      for (int k = 0; k < m; ++k) out[k] = out[k] + fv[k];
      if (c.c11 != 0.0)
        for (int k = 0; k < m; ++k) out[k] = out[k] + c.c11 * nn * (ui[k] - uo[k]);
    }
  }
}

// ----------------------------------------------------------------- gather

template <class T = double>
struct LineData {
  T u[MAXNP][MAXM];
  T q[MAXNP][MAXM * MAXD];
  T uo[2][MAXM], qo[2][MAXM * MAXD];
  const double* bc[2];
  int bk[2];  // boundary kind of each end (-1 interior)
};

template <class T>
void gather_line(const Ctx& c, int e, int dir, int line, const double* U, const T* Q,
                 LineData<T>& L) {
  const int m = c.m, mD = c.m * c.D;
  for (int t = 0; t < c.np; ++t) {
    const size_t nd = static_cast<size_t>(e) * c.npe + c.node_on_line(dir, line, t);
    for (int k = 0; k < m; ++k) L.u[t][k] = U[nd * m + k];
    if (Q)
      for (int k = 0; k < mD; ++k) L.q[t][k] = Q[nd * mD + k];
  }
  for (int side = 0; side < 2; ++side) {
    const size_t k = c.epi(e, dir, side, line);
    L.bc[side] = nullptr;
    L.bk[side] = -1;
    if (c.ep_bc[k] >= 0) {
      L.bc[side] = c.ep_g.empty() ? c.bcv[c.ep_bc[k]].data() : &c.ep_g[k * c.m];
      L.bk[side] = c.bck[c.ep_bc[k]];
      continue;
    }
    const size_t nd = static_cast<size_t>(c.ep_elem[k]) * c.npe + c.ep_node[k];
    for (int q = 0; q < m; ++q) L.uo[side][q] = U[nd * m + q];
    if (Q)
      for (int q = 0; q < mD; ++q) L.qo[side][q] = Q[nd * mD + q];
  }
}

// --------------------------------------------------------------- residual

// r^(dir) of one line (before the 1/J scaling), b = M^-1(...).
template <class T>
void line_residual(const Ctx& c, int e, int dir, int line, const LineData<T>& L, T r[][MAXM]) {
  const int m = c.m, np = c.np, nq = c.nq, D = c.D, mD = m * D;
  for (int i = 0; i < np; ++i)
    for (int k = 0; k < m; ++k) r[i][k] = 0.0;
  for (int q = 0; q < nq; ++q) {
    T uq[MAXM] = {0}, qq[MAXM * MAXD] = {0};
    for (int t = 0; t < np; ++t) {
      const double ph = c.phi[t * nq + q];
      for (int k = 0; k < m; ++k) uq[k] += ph * L.u[t][k];
      if (c.second)
        for (int k = 0; k < mD; ++k) qq[k] += ph * L.q[t][k];
    }
    T ft[MAXM];
    flux_dot(c, uq, qq, c.nv(e, dir, line, q), ft);
    for (int i = 0; i < np; ++i) {
      const double w = c.qw[q] * c.dphi[i * nq + q];
      for (int k = 0; k < m; ++k) r[i][k] -= w * ft[k];
    }
  }
  for (int side = 0; side < 2; ++side) {
    const int ie = side ? c.p : 0;
    T fh[MAXM];
    endpoint_flux<T>(c, L.u[ie], L.q[ie], L.uo[side], L.qo[side], L.bc[side], L.bk[side],
                          c.ne(e, dir, side, line), c.sign(e, dir, side), fh);
    for (int k = 0; k < m; ++k) r[ie][k] += fh[k];
  }
  for (int k = 0; k < m; ++k) c.mass_solve(&r[0][k], MAXM);
}

template <class T>
void elem_residual(const Ctx& c, int e, const double* U, const T* Q, double* R) {
  const int m = c.m, npe = c.npe;
  std::vector<T> acc(static_cast<size_t>(npe) * m, T(0.0));
  LineData<T> L;
  T r[MAXNP][MAXM];
  for (int dir = 0; dir < c.D; ++dir)
    for (int line = 0; line < c.NL; ++line) {
      gather_line(c, e, dir, line, U, Q, L);
      line_residual(c, e, dir, line, L, r);
      for (int t = 0; t < c.np; ++t) {
        const int nd = c.node_on_line(dir, line, t);
        for (int k = 0; k < m; ++k) acc[nd * m + k] += r[t][k];
      }
    }
  for (int nd = 0; nd < npe; ++nd) {
    const size_t g = static_cast<size_t>(e) * npe + nd;
    for (int k = 0; k < m; ++k) {
      const double s = c.source.empty() ? 0.0 : c.source[g * m + k];
      R[g * m + k] = static_cast<double>(s - c.invJ[g] * acc[nd * m + k]);
    }
  }
}

// d^(dir) of one line: M^-1 [u_hat (x) n at the ends - sum_q w phi' u_q (x) nvec_q].
template <class T>
void line_gradient(const Ctx& c, int e, int dir, int line, const LineData<T>& L,
                   T d[][MAXM * MAXD]) {
  const int m = c.m, np = c.np, nq = c.nq, D = c.D, mD = m * D;
  for (int i = 0; i < np; ++i)
    for (int k = 0; k < mD; ++k) d[i][k] = 0.0;
  for (int q = 0; q < nq; ++q) {
    T uq[MAXM] = {0};
    for (int t = 0; t < np; ++t)
      for (int k = 0; k < m; ++k) uq[k] += c.phi[t * nq + q] * L.u[t][k];
    const double* nvq = c.nv(e, dir, line, q);
    for (int i = 0; i < np; ++i) {
      const double w = c.qw[q] * c.dphi[i * nq + q];
      for (int k = 0; k < m; ++k)
        for (int dd = 0; dd < D; ++dd) d[i][k * D + dd] -= w * (uq[k] * nvq[dd]);
    }
  }
  for (int side = 0; side < 2; ++side) {
    const int ie = side ? c.p : 0;
    const double* n = c.ne(e, dir, side, line);
    const T* uh;
    T uhw[MAXM];
    if (L.bc[side] && L.bk[side] == LDG_BC_NO_SLIP_ADIABATIC) {  // mixed: momentum 0, rho and E interior
      for (int k = 0; k < m; ++k) uhw[k] = uhat_inner_c(L.bk[side], k, m) ? L.u[ie][k] : 0.0;
      uh = uhw;
    } else if (L.bc[side] && !uhat_inner(L.bk[side])) {
      for (int k = 0; k < m; ++k) uhw[k] = L.bc[side][k];  // u_hat = g_D
      uh = uhw;
    } else if (L.bc[side]) {
      uh = L.u[ie];  // Neumann-type / slip wall
    }
    else uh = c.sign(e, dir, side) > 0 ? L.u[ie] : L.uo[side];
    for (int k = 0; k < m; ++k)
      for (int dd = 0; dd < D; ++dd) d[ie][k * D + dd] += uh[k] * n[dd];
  }
  for (int k = 0; k < mD; ++k) c.mass_solve(&d[0][k], MAXM * MAXD);
}

template <class T>
void elem_gradient(const Ctx& c, int e, const double* U, T* Q) {
  const int mD = c.m * c.D, npe = c.npe;
  std::vector<T> acc(static_cast<size_t>(npe) * mD, T(0.0));
  LineData<T> L;
  T d[MAXNP][MAXM * MAXD];
  for (int dir = 0; dir < c.D; ++dir)
    for (int line = 0; line < c.NL; ++line) {
      gather_line<T>(c, e, dir, line, U, nullptr, L);
      line_gradient(c, e, dir, line, L, d);
      for (int t = 0; t < c.np; ++t) {
        const int nd = c.node_on_line(dir, line, t);
        for (int k = 0; k < mD; ++k) acc[nd * mD + k] += d[t][k];
      }
    }
  for (int nd = 0; nd < npe; ++nd) {
    const size_t g = static_cast<size_t>(e) * npe + nd;
    for (int k = 0; k < mD; ++k) Q[g * mD + k] = c.invJ[g] * acc[nd * mD + k];
  }
}

template <class F>
void for_elems(const Ctx& c, const std::vector<int>* subset, F&& f) {
  const int n = subset ? static_cast<int>(subset->size()) : c.E;
  std::atomic<bool> failed{false};
  std::string msg;
  std::vector<double> st;
  int se = -1;
  std::mutex mu;
#pragma omp parallel for schedule(dynamic, 16)
  for (int i = 0; i < n; ++i) {
    if (failed.load(std::memory_order_relaxed)) continue;
    const int e = subset ? (*subset)[i] : i;
    try {
      f(e);
    } catch (const physical_state_error& ex) {
      std::lock_guard<std::mutex> g(mu);
      if (!failed.exchange(true)) {
        msg = ex.what();
        st = ex.state;
        se = e;
      }
    }
  }
  if (failed) {
    physical_state_error ex(msg + " (element " + std::to_string(se) + ")", st);
    throw ex;
  }
}

// --------------------------------------------------------------- Jacobians

// Structural rules (shared definition of the pattern):
//   K11 volume blocks exist iff the flux depends on u at quadrature points;
//   endpoint blocks exist for every u the endpoint flux depends on.
struct Contrib {
  int64_t row, col;
};

void pattern_line(const Ctx& c, int e, int dir, int line, int which, std::vector<Contrib>& out) {
  const int64_t base = static_cast<int64_t>(e) * c.npe;
  auto own = [&](int t) { return base + c.node_on_line(dir, line, t); };
  const bool vol = which == LDG_K11 ? (c.has_inv || (c.second && c.vis_u)) : c.second;
  if (which != LDG_K11 && !c.second) return;
  for (int i = 0; i < c.np; ++i) {
    if (vol)
      for (int t = 0; t < c.np; ++t) out.push_back({own(i), own(t)});
    for (int side = 0; side < 2; ++side) {
      const size_t k = c.epi(e, dir, side, line);
      const int ie = side ? c.p : 0;
      const bool bd = c.ep_bc[k] >= 0;
      const int bkind = bd ? c.bck[c.ep_bc[k]] : -1;
      const bool neu = bkind == LDG_BC_NEUMANN;  // prescribed flux: no u or q dependence
      const int64_t nbr = bd ? -1 : static_cast<int64_t>(c.ep_elem[k]) * c.npe + c.ep_node[k];
      const int S = c.sign(e, dir, side);
      if (which == LDG_K11) {
        bool in = false, outn = false;
        if (c.has_inv) {
          in = !neu;
          outn = !bd;
        }
        if (c.second) {
          if (bd) {
            in = in || (!neu && (c.vis_u || (bkind != LDG_BC_SLIP_WALL && c.c11_bd != 0.0)));
          } else {
            if (c.vis_u) {
              if (S > 0) outn = true;
              else in = true;
            }
            if (c.c11 != 0.0) in = outn = true;
          }
        }
        if (in) out.push_back({own(i), own(ie)});
        if (outn) out.push_back({own(i), nbr});
      } else if (which == LDG_K12) {
        if (bd) {
          if (!neu) out.push_back({own(i), own(ie)});
        } else if (S <= 0) out.push_back({own(i), own(ie)});
        else out.push_back({own(i), nbr});
      } else {  // K21: u_hat
        if (bd) {
          if (uhat_inner(bkind)) out.push_back({own(i), own(ie)});
          continue;
        }
        if (S > 0) out.push_back({own(i), own(ie)});
        else out.push_back({own(i), nbr});
      }
    }
  }
}

void build_pattern(Ctx& c, int which, const std::vector<int>* subset) {
  BlockMat& K = c.K[which];
  K.nrows = static_cast<int64_t>(c.E) * c.npe;
  K.br = which == LDG_K21 ? c.m * c.D : c.m;
  K.bc = which == LDG_K12 ? c.m * c.D : c.m;
  std::vector<std::vector<int64_t>> rows_of(c.E);
  const int n = subset ? static_cast<int>(subset->size()) : c.E;
  std::vector<char> active(c.E, subset ? 0 : 1);
  if (subset)
    for (int e : *subset) active[e] = 1;
#pragma omp parallel for schedule(dynamic, 64)
  for (int i = 0; i < n; ++i) {
    const int e = subset ? (*subset)[i] : i;
    std::vector<Contrib> v;
    for (int dir = 0; dir < c.D; ++dir)
      for (int line = 0; line < c.NL; ++line) pattern_line(c, e, dir, line, which, v);
    std::sort(v.begin(), v.end(), [](const Contrib& a, const Contrib& b) {
      return a.row != b.row ? a.row < b.row : a.col < b.col;
    });
    v.erase(std::unique(v.begin(), v.end(),
                        [](const Contrib& a, const Contrib& b) { return a.row == b.row && a.col == b.col; }),
            v.end());
    std::vector<int64_t> flat;
    flat.reserve(2 * v.size());
    for (const auto& x : v) {
      flat.push_back(x.row);
      flat.push_back(x.col);
    }
    rows_of[e].swap(flat);
  }
  K.rowptr.assign(K.nrows + 1, 0);
  for (int e = 0; e < c.E; ++e)
    for (size_t k = 0; k < rows_of[e].size(); k += 2) K.rowptr[rows_of[e][k] + 1]++;
  for (int64_t r = 0; r < K.nrows; ++r) K.rowptr[r + 1] += K.rowptr[r];
  K.col.assign(K.rowptr[K.nrows], 0);
  for (int e = 0; e < c.E; ++e) {
    int64_t last = -1, pos = 0;
    for (size_t k = 0; k < rows_of[e].size(); k += 2) {
      const int64_t r = rows_of[e][k];
      if (r != last) {
        pos = K.rowptr[r];
        last = r;
      }
      K.col[pos++] = rows_of[e][k + 1];
    }
  }
  K.val.assign(K.col.size() * K.br * K.bc, 0.0);
  K.built = true;
}

// Analytic Jacobian of one element's rows.  NU = m (u-derivative slots),
// NQ = m*D (q-derivative slots).
template <int NU, int NQ>
void elem_jacobian(Ctx& c, int e, const double* U, const double* Q) {
  const int m = c.m, np = c.np, nq = c.nq, D = c.D, mD = m * D;
  const int64_t base = static_cast<int64_t>(e) * c.npe;
  LineData<> L;
  using DU = Dual<NU>;
  using DQ = Dual<NQ>;
  auto addblk = [&](int which, int64_t row, int64_t col, const double* blk, double scale) {
    BlockMat& K = c.K[which];
    const int64_t pos = K.find(row, col);
    if (pos < 0) throw std::logic_error("oracle: contribution outside the pattern");
    double* v = &K.val[pos * K.br * K.bc];
    for (int i = 0; i < K.br * K.bc; ++i) v[i] += scale * blk[i];
  };
  for (int dir = 0; dir < D; ++dir)
    for (int line = 0; line < c.NL; ++line) {
      gather_line(c, e, dir, line, U, Q, L);
      auto own = [&](int t) { return base + c.node_on_line(dir, line, t); };
      // ---------------- K11 / K12 volume: dB[i][t] = -sum_q w dphi_i phi_t dft/du
      const bool vol11 = c.has_inv || (c.second && c.vis_u);
      // v11[t][i][a][b] (a: residual comp, b: u comp); v12[t][i][a][b] (b: q comp)
      std::vector<double> v11(static_cast<size_t>(np) * np * m * m, 0.0);
      std::vector<double> v12(c.second ? static_cast<size_t>(np) * np * m * mD : 0, 0.0);
      for (int q = 0; q < nq; ++q) {
        double uq[MAXM] = {0}, qq[MAXM * MAXD] = {0};
        for (int t = 0; t < np; ++t) {
          const double ph = c.phi[t * nq + q];
          for (int k = 0; k < m; ++k) uq[k] += ph * L.u[t][k];
          if (c.second)
            for (int k = 0; k < mD; ++k) qq[k] += ph * L.q[t][k];
        }
        const double* nvq = c.nv(e, dir, line, q);
        double A[MAXM][MAXM * MAXD];
        if (vol11) {
          DU du[MAXM], dq[MAXM * MAXD], f[MAXM];
          for (int k = 0; k < m; ++k) {
            du[k] = DU(uq[k]);
            du[k].d[k] = 1.0;
          }
          for (int k = 0; k < mD; ++k) dq[k] = DU(qq[k]);
          flux_dot(c, du, dq, nvq, f);
          for (int a = 0; a < m; ++a)
            for (int b = 0; b < m; ++b) A[a][b] = f[a].d[b];
          for (int i = 0; i < np; ++i) {
            const double w = c.qw[q] * c.dphi[i * nq + q];
            for (int t = 0; t < np; ++t) {
              const double wt = w * c.phi[t * nq + q];
              double* dst = &v11[((static_cast<size_t>(t) * np + i) * m) * m];
              for (int a = 0; a < m; ++a)
                for (int b = 0; b < m; ++b) dst[a * m + b] -= wt * A[a][b];
            }
          }
        }
        if (c.second) {
          DQ du[MAXM], dq[MAXM * MAXD], f[MAXM];
          for (int k = 0; k < m; ++k) du[k] = DQ(uq[k]);
          for (int k = 0; k < mD; ++k) {
            dq[k] = DQ(qq[k]);
            dq[k].d[k] = 1.0;
          }
          vflux_dot(c, du, dq, nvq, f);
          for (int i = 0; i < np; ++i) {
            const double w = c.qw[q] * c.dphi[i * nq + q];
            for (int t = 0; t < np; ++t) {
              const double wt = w * c.phi[t * nq + q];
              double* dst = &v12[((static_cast<size_t>(t) * np + i) * m) * mD];
              for (int a = 0; a < m; ++a)
                for (int b = 0; b < mD; ++b) dst[a * mD + b] -= wt * f[a].d[b];
            }
          }
        }
      }
      // ---------------- endpoints
      // e11[side][which-col 0=own end,1=nbr][a][b], e12 likewise
      double e11[2][2][MAXM * MAXM] = {}, e12[2][2][MAXM * MAXM * MAXD] = {};
      bool has11[2][2] = {}, has12[2][2] = {};
      for (int side = 0; side < 2; ++side) {
        const int ie = side ? c.p : 0;
        const double* n = c.ne(e, dir, side, line);
        const int S = c.sign(e, dir, side);
        const bool bd = L.bc[side] != nullptr;
        // d/du_in and d/du_out with q fixed
        for (int pass = 0; pass < (bd ? 1 : 2); ++pass) {
          DU ui[MAXM], uo[MAXM], qi[MAXM * MAXD], qo[MAXM * MAXD], f[MAXM];
          for (int k = 0; k < m; ++k) {
            ui[k] = DU(L.u[ie][k]);
            uo[k] = DU(bd ? 0.0 : L.uo[side][k]);
            if (pass == 0) ui[k].d[k] = 1.0;
            else uo[k].d[k] = 1.0;
          }
          for (int k = 0; k < mD; ++k) {
            qi[k] = DU(c.second ? L.q[ie][k] : 0.0);
            qo[k] = DU(c.second && !bd ? L.qo[side][k] : 0.0);
          }
          endpoint_flux<DU>(c, ui, qi, uo, qo, L.bc[side], L.bk[side], n, S, f);
          for (int a = 0; a < m; ++a)
            for (int b = 0; b < m; ++b) e11[side][pass][a * m + b] = f[a].d[b];
          has11[side][pass] = true;
        }
        if (c.second) {
          const int pass = (bd || S <= 0) ? 0 : 1;
          DQ ui[MAXM], uo[MAXM], qi[MAXM * MAXD], qo[MAXM * MAXD], f[MAXM];
          for (int k = 0; k < m; ++k) {
            ui[k] = DQ(L.u[ie][k]);
            uo[k] = DQ(bd ? 0.0 : L.uo[side][k]);
          }
          for (int k = 0; k < mD; ++k) {
            qi[k] = DQ(L.q[ie][k]);
            qo[k] = DQ(bd ? 0.0 : L.qo[side][k]);
            if (pass == 0) qi[k].d[k] = 1.0;
            else qo[k].d[k] = 1.0;
          }
          endpoint_flux<DQ>(c, ui, qi, uo, qo, L.bc[side], L.bk[side], n, S, f);
          for (int a = 0; a < m; ++a)
            for (int b = 0; b < mD; ++b) e12[side][pass][a * mD + b] = f[a].d[b];
          has12[side][pass] = true;
        }
      }
      // ---------------- apply M^-1 along i and scatter into rows
      // K11: columns own(t) (volume + own-end terms) and nbr(side)
      std::vector<Contrib> pat;
      pattern_line(c, e, dir, line, LDG_K11, pat);
      auto has_pat = [&](const std::vector<Contrib>& pv, int64_t row, int64_t col) {
        for (const auto& x : pv)
          if (x.row == row && x.col == col) return true;
        return false;
      };
      {
        // columns: t in [0,np) own nodes, then side 0/1 neighbours
        for (int cidx = 0; cidx < np + 2; ++cidx) {
          double col[MAXNP][MAXM * MAXM];
          for (int i = 0; i < np; ++i)
            for (int k = 0; k < m * m; ++k) col[i][k] = 0.0;
          int64_t gcol;
          if (cidx < np) {
            gcol = own(cidx);
            for (int i = 0; i < np; ++i)
              for (int k = 0; k < m * m; ++k)
                col[i][k] = v11[((static_cast<size_t>(cidx) * np + i) * m) * m + k];
            for (int side = 0; side < 2; ++side) {
              const int ie = side ? c.p : 0;
              if (ie == cidx && has11[side][0])
                for (int k = 0; k < m * m; ++k) col[ie][k] += e11[side][0][k];
            }
          } else {
            const int side = cidx - np;
            if (L.bc[side] || !has11[side][1]) continue;
            const size_t k = c.epi(e, dir, side, line);
            gcol = static_cast<int64_t>(c.ep_elem[k]) * c.npe + c.ep_node[k];
            const int ie = side ? c.p : 0;
            for (int kk = 0; kk < m * m; ++kk) col[ie][kk] = e11[side][1][kk];
          }
          for (int k = 0; k < m * m; ++k) c.mass_solve(&col[0][k], MAXM * MAXM);
          for (int i = 0; i < np; ++i) {
            if (!has_pat(pat, own(i), gcol)) continue;
            addblk(LDG_K11, own(i), gcol, col[i], -c.invJ[own(i)]);
          }
        }
      }
      if (c.second) {
        std::vector<Contrib> p12;
        pattern_line(c, e, dir, line, LDG_K12, p12);
        for (int cidx = 0; cidx < np + 2; ++cidx) {
          std::vector<double> col(static_cast<size_t>(np) * m * mD, 0.0);
          int64_t gcol;
          if (cidx < np) {
            gcol = own(cidx);
            for (int i = 0; i < np; ++i)
              for (int k = 0; k < m * mD; ++k)
                col[i * m * mD + k] = v12[((static_cast<size_t>(cidx) * np + i) * m) * mD + k];
            for (int side = 0; side < 2; ++side) {
              const int ie = side ? c.p : 0;
              if (ie == cidx && has12[side][0])
                for (int k = 0; k < m * mD; ++k) col[ie * m * mD + k] += e12[side][0][k];
            }
          } else {
            const int side = cidx - np;
            if (L.bc[side] || !has12[side][1]) continue;
            const size_t k = c.epi(e, dir, side, line);
            gcol = static_cast<int64_t>(c.ep_elem[k]) * c.npe + c.ep_node[k];
            const int ie = side ? c.p : 0;
            for (int kk = 0; kk < m * mD; ++kk) col[ie * m * mD + kk] = e12[side][1][kk];
          }
          for (int k = 0; k < m * mD; ++k) c.mass_solve(&col[k], m * mD);
          for (int i = 0; i < np; ++i) {
            if (!has_pat(p12, own(i), gcol)) continue;
            addblk(LDG_K12, own(i), gcol, &col[i * m * mD], -c.invJ[own(i)]);
          }
        }
        // K21 (U-independent): D scalars per node pair, expanded to the
        // component-diagonal mD x m block on storage.
        std::vector<Contrib> p21;
        pattern_line(c, e, dir, line, LDG_K21, p21);
        for (int cidx = 0; cidx < np + 2; ++cidx) {
          double col[MAXNP][MAXD] = {}, colw[MAXNP][MAXD] = {};  // colw: no-slip ends (rho, E only)
          int64_t gcol;
          if (cidx < np) {
            gcol = own(cidx);
            for (int q = 0; q < nq; ++q) {
              const double* nvq = c.nv(e, dir, line, q);
              const double ph = c.phi[cidx * nq + q];
              for (int i = 0; i < np; ++i) {
                const double w = c.qw[q] * c.dphi[i * nq + q];
                for (int dd = 0; dd < D; ++dd) col[i][dd] -= w * (ph * nvq[dd]);
              }
            }
            for (int side = 0; side < 2; ++side) {
              const int ie = side ? c.p : 0;
              if (ie == cidx && L.bc[side] && L.bk[side] == LDG_BC_NO_SLIP_ADIABATIC) {
                const double* n = c.ne(e, dir, side, line);
                for (int dd = 0; dd < D; ++dd) colw[ie][dd] += n[dd];
              } else if (ie == cidx && ((!L.bc[side] && c.sign(e, dir, side) > 0) ||
                                        (L.bc[side] && uhat_inner(L.bk[side])))) {
                const double* n = c.ne(e, dir, side, line);
                for (int dd = 0; dd < D; ++dd) col[ie][dd] += n[dd];
              }
            }
          } else {
            const int side = cidx - np;
            if (L.bc[side] || c.sign(e, dir, side) > 0) continue;
            const size_t k = c.epi(e, dir, side, line);
            gcol = static_cast<int64_t>(c.ep_elem[k]) * c.npe + c.ep_node[k];
            const int ie = side ? c.p : 0;
            const double* n = c.ne(e, dir, side, line);
            for (int dd = 0; dd < D; ++dd) col[ie][dd] = n[dd];
          }
          for (int dd = 0; dd < D; ++dd) c.mass_solve(&col[0][dd], MAXD);
          for (int dd = 0; dd < D; ++dd) c.mass_solve(&colw[0][dd], MAXD);
          for (int i = 0; i < np; ++i) {
            if (!has_pat(p21, own(i), gcol)) continue;
            double blk[MAXM * MAXD * MAXM] = {};
            for (int k = 0; k < m; ++k)
              for (int dd = 0; dd < D; ++dd)
                blk[(k * D + dd) * m + k] = col[i][dd] + ((k == 0 || k == m - 1) ? colw[i][dd] : 0.0);
            addblk(LDG_K21, own(i), gcol, blk, c.invJ[own(i)]);
          }
        }
      }
    }
}

using JacFn = void (*)(Ctx&, int, const double*, const double*);
JacFn pick_jac(int m, int D) {
  if (m == 1 && D == 2) return elem_jacobian<1, 2>;
  if (m == 1 && D == 3) return elem_jacobian<1, 3>;
  if (m == 4 && D == 2) return elem_jacobian<4, 8>;
  if (m == 5 && D == 3) return elem_jacobian<5, 15>;
  throw std::runtime_error("oracle: unsupported (m, D) for the Jacobian");
}

}  // namespace

// -------------------------------------------------------------- public ops

template <class T>
void residual(const Ctx& c, const double* U, const T* Q, double* R,
              const std::vector<int>* subset = nullptr) {
  for_elems(c, subset, [&](int e) { elem_residual<T>(c, e, U, Q, R); });
}
template <class T>
void gradient(const Ctx& c, const double* U, T* Q, const std::vector<int>* subset = nullptr) {
  for_elems(c, subset, [&](int e) { elem_gradient<T>(c, e, U, Q); });
}

// ------------------------------------------------------------ flop counting
// Algorithmic FP64 operation counts: the oracle's own
// templated flux functions run on a counting scalar; +, -, *, /, sqrt count 1
// each (negation, |.|, max and comparisons 0).  Forward-mode Jacobians are
// costed from the primal counts: with N seeds an add costs 1+N, a multiply
// 1+3N, a divide 2+2N, a sqrt 2+N.
struct FlCount {
  double add = 0, mul = 0, div = 0, sqrt = 0;
  double total() const { return add + mul + div + sqrt; }
  double dual(int N) const { return add * (1 + N) + mul * (1 + 3 * N) + div * (2 + 2 * N) + sqrt * (2 + N); }
};
inline thread_local FlCount g_fl;
struct Fl {
  double v = 0.0;
  Fl() = default;
  Fl(double x) : v(x) {}  // NOLINT: constants promote implicitly
};
inline Fl operator+(Fl a, Fl b) { g_fl.add += 1; return Fl(a.v + b.v); }
inline Fl operator-(Fl a, Fl b) { g_fl.add += 1; return Fl(a.v - b.v); }
inline Fl operator*(Fl a, Fl b) { g_fl.mul += 1; return Fl(a.v * b.v); }
inline Fl operator/(Fl a, Fl b) { g_fl.div += 1; return Fl(a.v / b.v); }
inline Fl operator+(Fl a, double b) { return a + Fl(b); }
inline Fl operator+(double a, Fl b) { return Fl(a) + b; }
inline Fl operator-(Fl a, double b) { return a - Fl(b); }
inline Fl operator-(double a, Fl b) { return Fl(a) - b; }
inline Fl operator*(Fl a, double b) { return a * Fl(b); }
inline Fl operator*(double a, Fl b) { return Fl(a) * b; }
inline Fl operator/(Fl a, double b) { return a / Fl(b); }
inline Fl operator/(double a, Fl b) { return Fl(a) / b; }
inline Fl operator-(Fl a) { return Fl(-a.v); }
inline bool operator<(Fl a, Fl b) { return a.v < b.v; }
inline bool operator<(Fl a, double b) { return a.v < b; }
inline bool operator<=(Fl a, double b) { return a.v <= b; }
inline Fl sqrt(Fl a) { g_fl.sqrt += 1; return Fl(std::sqrt(a.v)); }
inline Fl abs(Fl a) { return Fl(a.v >= 0.0 ? a.v : -a.v); }
inline Fl max(Fl a, Fl b) { return a.v >= b.v ? a : b; }
inline double value_of(Fl x) { return x.v; }

template <class F>
FlCount count_ops(F&& f) {
  g_fl = FlCount{};
  f();
  return g_fl;
}

}  // namespace ora

// ===================================================================== C-ABI
using namespace ora;

struct lo_ctx {
  Ctx c;
};

namespace {
thread_local std::string g_err;
thread_local std::vector<double> g_state;
thread_local int g_elem = -1;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return LDG_OK;
  } catch (const physical_state_error& ex) {
    g_err = ex.what();
    g_state = ex.state;
    return LDG_ERR_PHYSICAL_STATE;
  } catch (const std::invalid_argument& ex) {
    g_err = ex.what();
    return LDG_ERR_INVALID_ARGUMENT;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return LDG_ERR_CONFIG;
  }
}

std::vector<int> subset_of(const int32_t* elems, int32_t n) {
  return std::vector<int>(elems, elems + n);
}
}  // namespace

extern "C" {

const char* lo_last_error(void) { return g_err.c_str(); }
int lo_last_error_state(double* state, int32_t* n) {
  *n = static_cast<int32_t>(g_state.size());
  if (state) std::copy(g_state.begin(), g_state.end(), state);
  return LDG_OK;
}
void lo_set_threads(int32_t n) {
#ifdef _OPENMP
  omp_set_num_threads(n);
#else
  (void)n;
#endif
}
int32_t lo_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

int lo_create(const ldg_setup* s, const ldg_physics* ph, lo_ctx** out) {
  return guarded([&] {
    auto x = std::make_unique<lo_ctx>();
    Ctx& c = x->c;
    c.D = s->dim;
    c.p = s->p;
    c.np = c.p + 1;
    c.nq = s->n_quad;
    c.npe = c.D == 2 ? c.np * c.np : c.np * c.np * c.np;
    c.NL = c.D == 2 ? c.np : c.np * c.np;
    c.E = s->n_elems;
    if (c.E < 1) throw std::runtime_error("oracle: mesh has no elements");
    if (c.np > MAXNP || c.nq > MAXNQ) throw std::invalid_argument("oracle: p too large");
    c.kind = ph->kind;
    c.riemann = ph->riemann;
    c.gas.gamma = ph->gamma;
    c.gas.mu = ph->mu;
    c.gas.prandtl = ph->prandtl;
    c.c11 = ph->c11;
    c.c11_bd = ph->c11_bd;
    if (ph->c22 != 0.0) throw std::runtime_error("residual_primal requires C22 = 0 (SPEC.md:250-252)");
    c.m = c.kind == LDG_POISSON ? 1 : c.D + 2;
    c.has_inv = c.kind != LDG_POISSON;
    c.second = c.kind == LDG_POISSON || (c.kind == LDG_NAVIER_STOKES && c.gas.mu != 0.0);
    c.vis_u = c.kind == LDG_NAVIER_STOKES;
    const int np = c.np, nq = c.nq;
    c.qw.assign(s->quad_weights, s->quad_weights + nq);
    c.phi.assign(s->phi_at_quad, s->phi_at_quad + np * nq);
    c.dphi.assign(s->dphi_at_quad, s->dphi_at_quad + np * nq);
    c.L.assign(s->mass, s->mass + np * np);
    for (int k = 0; k < np; ++k) {  // lower Cholesky, in place
      double d = c.L[k * np + k];
      for (int j = 0; j < k; ++j) d -= c.L[k * np + j] * c.L[k * np + j];
      if (!(d > 0.0)) throw std::runtime_error("oracle: mass matrix not SPD");
      d = std::sqrt(d);
      c.L[k * np + k] = d;
      for (int i = k + 1; i < np; ++i) {
        double v = c.L[i * np + k];
        for (int j = 0; j < k; ++j) v -= c.L[i * np + j] * c.L[k * np + j];
        c.L[i * np + k] = v / d;
      }
      for (int j = k + 1; j < np; ++j) c.L[k * np + j] = 0.0;
    }
    const size_t nn = static_cast<size_t>(c.E) * c.npe;
    c.jac.assign(s->jac_at_nodes, s->jac_at_nodes + nn);
    c.invJ.resize(nn);
    for (size_t i = 0; i < nn; ++i) c.invJ[i] = 1.0 / c.jac[i];
    c.nvec.assign(s->nvec_quad, s->nvec_quad + static_cast<size_t>(c.E) * c.D * c.NL * nq * c.D);
    c.nend.assign(s->normal_end, s->normal_end + static_cast<size_t>(c.E) * c.D * 2 * c.NL * c.D);
    if (c.second) {
      if (!s->switch_plus) throw std::runtime_error("second-order physics needs switches");
      c.sw.assign(s->switch_plus, s->switch_plus + static_cast<size_t>(c.E) * c.D);
    }
    build_endpoints(c, *s, *ph);
    if (s->node_coords) {  // own end-node coordinates of every line end (boundary functions)
      c.ep_x.assign(c.ep_bc.size() * c.D, 0.0);
      for (int e = 0; e < c.E; ++e)
        for (int dir = 0; dir < c.D; ++dir)
          for (int side = 0; side < 2; ++side)
            for (int line = 0; line < c.NL; ++line) {
              const int nd = c.node_on_line(dir, line, side ? c.p : 0);
              const size_t k = c.epi(e, dir, side, line);
              for (int d = 0; d < c.D; ++d)
                c.ep_x[k * c.D + d] = s->node_coords[(static_cast<size_t>(e) * c.npe + nd) * c.D + d];
            }
    }
    *out = x.release();
  });
}

void lo_destroy(lo_ctx* x) { delete x; }
int32_t lo_components(const lo_ctx* x) { return x->c.m; }

int lo_set_source(lo_ctx* x, const double* S) {
  return guarded([&] {
    const size_t n = static_cast<size_t>(x->c.E) * x->c.npe * x->c.m;
    if (S) x->c.source.assign(S, S + n);
    else x->c.source.clear();
  });
}

}  // extern "C"
namespace {
// boundary functions: evaluate at every boundary line end's own end node
void refresh_boundary(Ctx& c, double t) {
  if (c.bfun.empty()) {
    c.ep_g.clear();
    return;
  }
  if (!c.bfun_dirty && t == c.bfun_t && !c.ep_g.empty()) return;
  const size_t n = c.ep_bc.size();
  c.ep_g.assign(n * c.m, 0.0);
  for (size_t k = 0; k < n; ++k) {
    const int bc = c.ep_bc[k];
    if (bc < 0) continue;
    auto it = c.bfun.find(c.bctag[bc]);
    if (it == c.bfun.end()) std::copy(c.bcv[bc].begin(), c.bcv[bc].end(), c.ep_g.begin() + k * c.m);
    else it->second.first(it->second.second, &c.ep_x[k * c.D], t, &c.ep_g[k * c.m]);
  }
  c.bfun_t = t;
  c.bfun_dirty = false;
}
}  // namespace
extern "C" {

int lo_set_boundary_function(lo_ctx* x, int32_t tag, ldg_bc_fn fn, void* user) {
  return guarded([&] {
    Ctx& c = x->c;
    if (std::find(c.bctag.begin(), c.bctag.end(), tag) == c.bctag.end())
      throw std::runtime_error("oracle: no boundary condition with tag " + std::to_string(tag));
    if (fn && c.ep_x.empty()) throw std::runtime_error("oracle: boundary functions need node coordinates");
    if (fn) c.bfun[tag] = {fn, user};
    else c.bfun.erase(tag);
    c.bfun_dirty = true;
  });
}

int lo_gradient(lo_ctx* x, const double* U, double t, double* Q) {
  return guarded([&] {
    refresh_boundary(x->c, t);
    gradient(x->c, U, Q);
  });
}

int lo_residual_uq(lo_ctx* x, const double* U, const double* Q, double t, double* R) {
  return guarded([&] {
    refresh_boundary(x->c, t);
    residual(x->c, U, Q, R);
  });
}

// Residual, optionally restricted to a subset of elements (rows of other
// elements are left untouched).  Second-order physics computes Q = D(U)
// first (on the needed elements plus their neighbours: here, all).
int lo_residual(lo_ctx* x, const double* U, double t, double* R, double* Qout,
                const int32_t* elems, int32_t n_sub) {
  return guarded([&] {
    Ctx& c = x->c;
    refresh_boundary(c, t);
    std::vector<int> sub;
    const std::vector<int>* sp = nullptr;
    if (elems) {
      sub = subset_of(elems, n_sub);
      sp = &sub;
    }
    if (c.second) {
      std::vector<double> Qv;
      double* Q = Qout;
      if (!Q) {
        Qv.assign(static_cast<size_t>(c.E) * c.npe * c.m * c.D, 0.0);
        Q = Qv.data();
      }
      gradient(c, U, Q);
      residual(c, U, Q, R, sp);
    } else {
      residual<double>(c, U, nullptr, R, sp);
    }
  });
}

// Extended-precision residual (x87 80-bit long double, 64-bit significand):
// the same restatement evaluated with every intermediate -- interpolated
// states, fluxes, line projections, the mass solve, the direction sum and, for
// second-order physics, Q -- carried in long double and rounded to double once
// at the end.  Inputs (U, metric, basis tables) are the same doubles.  Used by
// the parity tests as the accuracy yardstick on near-steady states where the
// residual is a large cancellation.
int lo_residual_ext(lo_ctx* x, const double* U, double t, double* R, const int32_t* elems,
                    int32_t n_sub) {
  return guarded([&] {
    Ctx& c = x->c;
    refresh_boundary(c, t);
    std::vector<int> sub;
    const std::vector<int>* sp = nullptr;
    if (elems) {
      sub = subset_of(elems, n_sub);
      sp = &sub;
    }
    if (c.second) {
      std::vector<long double> Q(static_cast<size_t>(c.E) * c.npe * c.m * c.D, 0.0L);
      gradient<long double>(c, U, Q.data());
      residual<long double>(c, U, Q.data(), R, sp);
    } else {
      residual<long double>(c, U, nullptr, R, sp);
    }
  });
}

// Analytic assembly (mode 0) of K11 (+K12, K21 for second-order physics),
// optionally only for the rows of a subset of elements.
int lo_assemble(lo_ctx* x, const double* U, double t, const int32_t* elems, int32_t n_sub) {
  return guarded([&] {
    Ctx& c = x->c;
    refresh_boundary(c, t);
    std::vector<int> sub;
    const std::vector<int>* sp = nullptr;
    if (elems) {
      sub = subset_of(elems, n_sub);
      sp = &sub;
    }
    const int nm = c.second ? 3 : 1;
    // The pattern depends only on the mesh: build it once for full assemblies
    // (values are re-zeroed), rebuild for element subsets.
    for (int w = 0; w < nm; ++w) {
      if (sp || !c.K[w].built || c.K[w].subset) {
        build_pattern(c, w, sp);
        c.K[w].subset = sp != nullptr;
      } else {
        std::fill(c.K[w].val.begin(), c.K[w].val.end(), 0.0);
      }
    }
    std::vector<double> Qv;
    const double* Q = nullptr;
    if (c.second) {
      Qv.assign(static_cast<size_t>(c.E) * c.npe * c.m * c.D, 0.0);
      gradient(c, U, Qv.data());
      Q = Qv.data();
    }
    JacFn f = pick_jac(c.m, c.D);
    for_elems(c, sp, [&](int e) { f(c, e, U, Q); });
    c.pc_built = false;  // factors of the old Jacobian are stale
  });
}

// Assembly from an explicit Q (K11 and K12 at (U,Q)); for FD comparisons.
int lo_assemble_uq(lo_ctx* x, const double* U, const double* Q) {
  return guarded([&] {
    Ctx& c = x->c;
    const int nm = c.second ? 3 : 1;
    for (int w = 0; w < nm; ++w) {
      build_pattern(c, w, nullptr);
      c.K[w].subset = false;
    }
    JacFn f = pick_jac(c.m, c.D);
    for_elems(c, nullptr, [&](int e) { f(c, e, U, Q); });
  });
}

int lo_pattern_info(const lo_ctx* x, int32_t which, int64_t* nnzb, int32_t* br, int32_t* bc) {
  return guarded([&] {
    const BlockMat& K = x->c.K[which];
    if (!K.built) throw std::runtime_error("oracle: matrix not assembled");
    *nnzb = static_cast<int64_t>(K.col.size());
    *br = K.br;
    *bc = K.bc;
  });
}

int lo_export_blocks(const lo_ctx* x, int32_t which, int64_t* rows, int64_t* cols, double* vals) {
  return guarded([&] {
    const BlockMat& K = x->c.K[which];
    if (!K.built) throw std::runtime_error("oracle: matrix not assembled");
    for (int64_t r = 0; r < K.nrows; ++r)
      for (int64_t k = K.rowptr[r]; k < K.rowptr[r + 1]; ++k) {
        if (rows) rows[k] = r;
        if (cols) cols[k] = K.col[k];
      }
    if (vals) std::copy(K.val.begin(), K.val.end(), vals);
  });
}

// Scalar compressed-column export: colptr (ncols+1),
// rowidx/vals (nnz).  Component-diagonal structure of K21 is kept dense per
// block (zeros included), as for all blocks.
int lo_export_csc(const lo_ctx* x, int32_t which, int64_t* colptr, int64_t* rowidx, double* vals,
                  int64_t* nnz_out) {
  return guarded([&] {
    const Ctx& c = x->c;
    const BlockMat& K = c.K[which];
    if (!K.built) throw std::runtime_error("oracle: matrix not assembled");
    const int64_t ncols = K.nrows * K.bc;
    const int64_t nnz = static_cast<int64_t>(K.col.size()) * K.br * K.bc;
    if (nnz_out) *nnz_out = nnz;
    if (!colptr) return;
    std::fill(colptr, colptr + ncols + 1, 0);
    for (size_t k = 0; k < K.col.size(); ++k)
      for (int b = 0; b < K.bc; ++b) colptr[K.col[k] * K.bc + b + 1] += K.br;
    for (int64_t j = 0; j < ncols; ++j) colptr[j + 1] += colptr[j];
    std::vector<int64_t> fill(colptr, colptr + ncols);
    for (int64_t r = 0; r < K.nrows; ++r)  // rows ascending -> sorted within columns
      for (int a = 0; a < K.br; ++a)
        for (int64_t k = K.rowptr[r]; k < K.rowptr[r + 1]; ++k)
          for (int b = 0; b < K.bc; ++b) {
            const int64_t j = K.col[k] * K.bc + b;
            const int64_t pos = fill[j]++;
            rowidx[pos] = r * K.br + a;
            vals[pos] = K.val[(k * K.br + a) * K.bc + b];
          }
  });
}

int lo_spmv(const lo_ctx* x, int32_t which, const double* v, double* y) {
  return guarded([&] {
    const BlockMat& K = x->c.K[which];
    if (!K.built) throw std::runtime_error("oracle: matrix not assembled");
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < K.nrows; ++r) {
      double acc[MAXM * MAXD] = {0};
      for (int64_t k = K.rowptr[r]; k < K.rowptr[r + 1]; ++k) {
        const double* blk = &K.val[k * K.br * K.bc];
        const double* xv = v + K.col[k] * K.bc;
        for (int a = 0; a < K.br; ++a)
          for (int b = 0; b < K.bc; ++b) acc[a] += blk[a * K.bc + b] * xv[b];
      }
      for (int a = 0; a < K.br; ++a) y[r * K.br + a] = acc[a];
    }
  });
}

// CPU baseline sample (bench.py's cpu_baseline leg and --impl reference):
// one bounded, cost-proportional sample of the bench step on the elements
// `elems` with `threads` OpenMP threads -- gradient (second order), residual,
// analytic Jacobian values (the pattern of the subset is built once, untimed,
// like the device store layout at context creation) and `nmv` matvecs over the
// subset's rows (K21 rows then v - adt (K11 v + K12 w), or K11 v for first-order
// physics).  Each phase is timed with steady_clock; secs[0..3] = gradient,
// residual, Jacobian, all matvecs, each the median over `reps` repetitions.
// Per element this is exactly the work of the full step, so the full-mesh time
// extrapolates linearly (t_full = t_sample E / n).
int lo_time_sample(lo_ctx* x, const double* U, const double* v, double adt, int32_t nmv, const int32_t* elems,
                   int32_t n_sub, int32_t threads, int32_t reps, double* secs) {
  return guarded([&] {
    Ctx& c = x->c;
#ifdef _OPENMP
    const int old = omp_get_max_threads();
    omp_set_num_threads(threads > 0 ? threads : old);
#endif
    refresh_boundary(c, 0.0);
    std::vector<int> sub = subset_of(elems, n_sub);
    const int nm = c.second ? 3 : 1;
    for (int w = 0; w < nm; ++w) {
      build_pattern(c, w, &sub);
      c.K[w].subset = true;
    }
    const size_t nU = static_cast<size_t>(c.E) * c.npe * c.m;
    std::vector<double> Q(c.second ? nU * c.D : 0, 0.0), R(nU, 0.0), y(nU, 0.0), wv(c.second ? nU * c.D : 0, 0.0);
    JacFn jf = pick_jac(c.m, c.D);
    using clk = std::chrono::steady_clock;
    auto since = [](clk::time_point t0) { return std::chrono::duration<double>(clk::now() - t0).count(); };
    std::vector<double> tg, tr, tj, tm;
    const int ns = static_cast<int>(sub.size());
    auto rows_mv = [&](const BlockMat& K, const double* xv, double* out, int64_t row0) {
      double acc[MAXM * MAXD] = {0};
      for (int64_t k = K.rowptr[row0]; k < K.rowptr[row0 + 1]; ++k) {
        const double* blk = &K.val[k * K.br * K.bc];
        const double* xx = xv + K.col[k] * K.bc;
        for (int a = 0; a < K.br; ++a)
          for (int b = 0; b < K.bc; ++b) acc[a] += blk[a * K.bc + b] * xx[b];
      }
      for (int a = 0; a < K.br; ++a) out[a] += acc[a];
    };
    for (int rep = 0; rep < (reps > 0 ? reps : 1); ++rep) {
      auto t0 = clk::now();
      if (c.second) gradient<double>(c, U, Q.data(), &sub);
      tg.push_back(since(t0));
      t0 = clk::now();
      residual<double>(c, U, c.second ? Q.data() : nullptr, R.data(), &sub);
      tr.push_back(since(t0));
      for (int w = 0; w < nm; ++w) std::fill(c.K[w].val.begin(), c.K[w].val.end(), 0.0);
      t0 = clk::now();
      for_elems(c, &sub, [&](int e) { jf(c, e, U, c.second ? Q.data() : nullptr); });
      tj.push_back(since(t0));
      t0 = clk::now();
      for (int k = 0; k < nmv; ++k) {
        if (c.second) {
#pragma omp parallel for schedule(static)
          for (int i = 0; i < ns; ++i)
            for (int nd = 0; nd < c.npe; ++nd) {
              const int64_t r = static_cast<int64_t>(sub[i]) * c.npe + nd;
              double* o = &wv[r * c.m * c.D];
              for (int a = 0; a < c.m * c.D; ++a) o[a] = 0.0;
              rows_mv(c.K[LDG_K21], v, o, r);
            }
        }
#pragma omp parallel for schedule(static)
        for (int i = 0; i < ns; ++i)
          for (int nd = 0; nd < c.npe; ++nd) {
            const int64_t r = static_cast<int64_t>(sub[i]) * c.npe + nd;
            double a[MAXM] = {0};
            rows_mv(c.K[LDG_K11], v, a, r);
            if (c.second) rows_mv(c.K[LDG_K12], wv.data(), a, r);
            for (int q = 0; q < c.m; ++q) y[r * c.m + q] = v[r * c.m + q] - adt * a[q];
          }
      }
      tm.push_back(since(t0));
    }
    auto med = [](std::vector<double> t) {
      std::sort(t.begin(), t.end());
      return t[t.size() / 2];
    };
    secs[0] = med(tg);
    secs[1] = med(tr);
    secs[2] = med(tj);
    secs[3] = med(tm);
#ifdef _OPENMP
    omp_set_num_threads(old);
#endif
  });
}

// y = v - alpha_dt (K11 v + K12 (K21 v))
int lo_split_matvec(const lo_ctx* x, double adt, const double* v, double* y) {
  return guarded([&] {
    const Ctx& c = x->c;
    const size_t n = static_cast<size_t>(c.E) * c.npe * c.m;
    std::vector<double> a(n), w, b;
    if (lo_spmv(x, LDG_K11, v, a.data()) != LDG_OK) throw std::runtime_error(g_err);
    if (c.second) {
      w.assign(n * c.D, 0.0);
      b.assign(n, 0.0);
      if (lo_spmv(x, LDG_K21, v, w.data()) != LDG_OK) throw std::runtime_error(g_err);
      if (lo_spmv(x, LDG_K12, w.data(), b.data()) != LDG_OK) throw std::runtime_error(g_err);
      for (size_t i = 0; i < n; ++i) a[i] = a[i] + b[i];
    }
    for (size_t i = 0; i < n; ++i) y[i] = v[i] - adt * a[i];
  });
}

// ---- block-Jacobi preconditioner
// A~ equals A = K11 + K12 K21 on the block-diagonal Line-DG pattern -- row
// and column node in the same element and on a common coordinate line -- and
// is zero elsewhere: fill of the product and inter-element couplings are
// dropped, while the product's entries that land on the pattern are exact
// (summed over every middle node, neighbour elements included).  Each element
// block of I - alpha_dt A~ is LU-factorised with partial pivoting.
namespace {
bool on_line_pattern(const Ctx& c, int r, int col) {
  int same = 0;
  int a = r, b = col;
  for (int d = 0; d < c.D; ++d) {
    same += (a % c.np) == (b % c.np);
    a /= c.np;
    b /= c.np;
  }
  return same >= c.D - 1;
}
}  // namespace

namespace {
// Element block of A~ (without the I - adt scaling): K11 on the in-element
// Line-DG pattern plus the K12 K21 products landing on it.
void element_block(const Ctx& c, int e, double* Me) {
  const BlockMat& K11 = c.K[LDG_K11];
  const int m = c.m, npe = c.npe, ne = npe * m;
  std::fill(Me, Me + static_cast<size_t>(ne) * ne, 0.0);
  const int64_t base = static_cast<int64_t>(e) * npe;
  for (int r = 0; r < npe; ++r) {
    const int64_t R = base + r;
    for (int64_t k = K11.rowptr[R]; k < K11.rowptr[R + 1]; ++k) {
      const int64_t cn = K11.col[k];
      if (cn < base || cn >= base + npe || !on_line_pattern(c, r, static_cast<int>(cn - base))) continue;
      const int cl = static_cast<int>(cn - base);
      for (int a = 0; a < m; ++a)
        for (int b = 0; b < m; ++b) Me[(r * m + a) * ne + cl * m + b] += K11.val[(k * m + a) * m + b];
    }
    if (c.second) {
      const BlockMat& K12 = c.K[LDG_K12];
      const BlockMat& K21 = c.K[LDG_K21];
      const int mD = m * c.D;
      for (int64_t k = K12.rowptr[R]; k < K12.rowptr[R + 1]; ++k) {
        const int64_t mid = K12.col[k];
        const double* b12 = &K12.val[k * m * mD];  // m x mD
        for (int64_t j = K21.rowptr[mid]; j < K21.rowptr[mid + 1]; ++j) {
          const int64_t cn = K21.col[j];
          if (cn < base || cn >= base + npe || !on_line_pattern(c, r, static_cast<int>(cn - base))) continue;
          const int cl = static_cast<int>(cn - base);
          const double* b21 = &K21.val[j * mD * m];  // mD x m
          for (int a = 0; a < m; ++a)
            for (int b = 0; b < m; ++b) {
              double s = 0.0;
              for (int q = 0; q < mD; ++q) s += b12[a * mD + q] * b21[q * m + b];
              Me[(r * m + a) * ne + cl * m + b] += s;
            }
        }
      }
    }
  }
}

// Dense LU with partial pivoting of an n x n row-major block; false if singular.
bool lu_pp(double* A, int32_t* piv, int n) {
  for (int kk = 0; kk < n; ++kk) {
    int pr = kk;
    double best = std::fabs(A[kk * n + kk]);
    for (int i = kk + 1; i < n; ++i)
      if (std::fabs(A[i * n + kk]) > best) {
        best = std::fabs(A[i * n + kk]);
        pr = i;
      }
    piv[kk] = pr;
    if (!(best > 0.0)) return false;
    if (pr != kk)
      for (int j = 0; j < n; ++j) std::swap(A[kk * n + j], A[pr * n + j]);
    const double ip = 1.0 / A[kk * n + kk];
    for (int i = kk + 1; i < n; ++i) {
      const double l = A[i * n + kk] * ip;
      A[i * n + kk] = l;
      for (int j = kk + 1; j < n; ++j) A[i * n + j] -= l * A[kk * n + j];
    }
  }
  return true;
}

// x <- (LU)^-1 P x for one factored block
void lu_solve(const double* LU, const int32_t* piv, int n, double* x) {
  for (int i = 0; i < n; ++i) std::swap(x[i], x[piv[i]]);
  for (int i = 0; i < n; ++i) {
    double s = x[i];
    for (int j = 0; j < i; ++j) s -= LU[i * n + j] * x[j];
    x[i] = s;
  }
  for (int i = n - 1; i >= 0; --i) {
    double s = x[i];
    for (int j = i + 1; j < n; ++j) s -= LU[i * n + j] * x[j];
    x[i] = s / LU[i * n + i];
  }
}

// Element-block LU is stored dense (n_e^2 per element); above 128 unknowns per
// element (3-D p >= 2) the preconditioner keeps the line-based sparsity the
// paper calls for in 3-D ("low-order approximations, ADI
// iterations"): the line-ADI factorisation
//   I - adt A~  ~  prod_d (I - adt A~_d),
// A~_d = the couplings of A~ along direction-d coordinate lines with the
// node-diagonal blocks split evenly over the D directions; each factor is
// block diagonal over the d-lines, one dense (p+1)m block per line (LU with
// partial pivoting), applied as z = (I - adt A~_{D-1})^-1 ... (I - adt A~_0)^-1 r.
bool use_line_adi(const Ctx& c) {
  return c.pc_mode == 2 || (c.pc_mode == 0 && c.npe * c.m > 128);
}
}  // namespace

int lo_precond_build(lo_ctx* x, double adt) {
  return guarded([&] {
    Ctx& c = x->c;
    const BlockMat& K11 = c.K[LDG_K11];
    if (!K11.built) throw std::runtime_error("oracle: Jacobian not assembled");
    const int m = c.m, npe = c.npe, ne = npe * m;
    std::atomic<int> bad{-1};
    if (use_line_adi(c)) {
      const int nb = c.np * m, D = c.D, NL = c.NL;
      c.pcLU.assign(static_cast<size_t>(c.E) * D * NL * nb * nb, 0.0);
      c.pcPiv.assign(static_cast<size_t>(c.E) * D * NL * nb, 0);
#pragma omp parallel for schedule(dynamic, 16)
      for (int e = 0; e < c.E; ++e) {
        std::vector<double> Me(static_cast<size_t>(ne) * ne);
        element_block(c, e, Me.data());
        for (int d = 0; d < D; ++d)
          for (int l = 0; l < NL; ++l) {
            const size_t blk = (static_cast<size_t>(e) * D + d) * NL + l;
            double* B = &c.pcLU[blk * nb * nb];
            for (int t = 0; t < c.np; ++t)
              for (int a = 0; a < m; ++a)
                for (int t2 = 0; t2 < c.np; ++t2)
                  for (int b = 0; b < m; ++b) {
                    const int r = c.node_on_line(d, l, t), cl = c.node_on_line(d, l, t2);
                    double v = Me[(r * m + a) * ne + cl * m + b];
                    if (t == t2) v = v / D;  // node-diagonal block shared by the D directions
                    B[(t * m + a) * nb + t2 * m + b] = (t == t2 && a == b ? 1.0 : 0.0) - adt * v;
                  }
            if (!lu_pp(B, &c.pcPiv[blk * nb], nb)) {
              int expect = -1;
              bad.compare_exchange_strong(expect, e);
            }
          }
      }
      if (bad.load() >= 0)
        throw std::runtime_error("oracle: singular preconditioner block at element " + std::to_string(bad.load()));
      c.pc_adi = true;
      c.pc_built = true;
      c.pc_adt = adt;
      return;
    }
    c.pc_adi = false;
    c.pcLU.assign(static_cast<size_t>(c.E) * ne * ne, 0.0);
    c.pcPiv.assign(static_cast<size_t>(c.E) * ne, 0);
#pragma omp parallel for schedule(dynamic, 16)
    for (int e = 0; e < c.E; ++e) {
      double* Me = &c.pcLU[static_cast<size_t>(e) * ne * ne];
      element_block(c, e, Me);
      for (int i = 0; i < ne * ne; ++i) Me[i] *= -adt;
      for (int i = 0; i < ne; ++i) Me[i * ne + i] += 1.0;
      // LU with partial pivoting (row interchanges recorded in piv)
      int32_t* piv = &c.pcPiv[static_cast<size_t>(e) * ne];
      if (!lu_pp(Me, piv, ne)) {
        int expect = -1;
        bad.compare_exchange_strong(expect, e);
        continue;
      }
      if (!c.pc_inverse) continue;
      // explicit block inverse X = U^-1 L^-1 P (as the device build: per
      // column the operation order of a forward / back substitution of P e_j);
      // the apply is then a dense block matvec
      std::vector<int> perm(ne);
      for (int i = 0; i < ne; ++i) perm[i] = i;
      for (int kk = 0; kk < ne; ++kk) std::swap(perm[kk], perm[piv[kk]]);
      std::vector<double> X(static_cast<size_t>(ne) * ne);
      for (int i = 0; i < ne; ++i)
        for (int j = 0; j < ne; ++j) X[i * ne + j] = perm[i] == j ? 1.0 : 0.0;
      for (int kk = 0; kk < ne - 1; ++kk)
        for (int i = kk + 1; i < ne; ++i)
          for (int j = 0; j < ne; ++j) X[i * ne + j] -= Me[i * ne + kk] * X[kk * ne + j];
      for (int kk = ne - 1; kk >= 0; --kk) {
        for (int j = 0; j < ne; ++j) X[kk * ne + j] = X[kk * ne + j] / Me[kk * ne + kk];
        for (int i = 0; i < kk; ++i)
          for (int j = 0; j < ne; ++j) X[i * ne + j] -= Me[i * ne + kk] * X[kk * ne + j];
      }
      std::copy(X.begin(), X.end(), Me);
    }
    if (bad.load() >= 0)
      throw std::runtime_error("oracle: singular preconditioner block at element " + std::to_string(bad.load()));
    c.pc_built = true;
    c.pc_adt = adt;
  });
}

namespace {
void pc_apply(const Ctx& c, const double* r, double* z) {
  const int ne = c.npe * c.m;
  if (c.pc_adi) {
    const int nb = c.np * c.m, m = c.m;
#pragma omp parallel for schedule(static)
    for (int e = 0; e < c.E; ++e) {
      double* ze = z + static_cast<size_t>(e) * ne;
      const double* re = r + static_cast<size_t>(e) * ne;
      for (int i = 0; i < ne; ++i) ze[i] = re[i];
      double xl[MAXNP * MAXM];
      for (int d = 0; d < c.D; ++d)
        for (int l = 0; l < c.NL; ++l) {
          const size_t blk = (static_cast<size_t>(e) * c.D + d) * c.NL + l;
          for (int t = 0; t < c.np; ++t)
            for (int a = 0; a < m; ++a) xl[t * m + a] = ze[c.node_on_line(d, l, t) * m + a];
          lu_solve(&c.pcLU[blk * nb * nb], &c.pcPiv[blk * nb], nb, xl);
          for (int t = 0; t < c.np; ++t)
            for (int a = 0; a < m; ++a) ze[c.node_on_line(d, l, t) * m + a] = xl[t * m + a];
        }
    }
    return;
  }
#pragma omp parallel for schedule(static)
  for (int e = 0; e < c.E; ++e) {
    const double* LU = &c.pcLU[static_cast<size_t>(e) * ne * ne];
    const int32_t* piv = &c.pcPiv[static_cast<size_t>(e) * ne];
    double* ze = z + static_cast<size_t>(e) * ne;
    const double* re = r + static_cast<size_t>(e) * ne;
    if (c.pc_inverse) {
      for (int i = 0; i < ne; ++i) {  // explicit inverse (lo_precond_build)
        double s = 0.0;
        for (int j = 0; j < ne; ++j) s += LU[i * ne + j] * re[j];
        ze[i] = s;
      }
      continue;
    }
    for (int i = 0; i < ne; ++i) ze[i] = re[i];
    for (int i = 0; i < ne; ++i) std::swap(ze[i], ze[piv[i]]);
    for (int i = 0; i < ne; ++i) {
      double s = ze[i];
      for (int j = 0; j < i; ++j) s -= LU[i * ne + j] * ze[j];
      ze[i] = s;
    }
    for (int i = ne - 1; i >= 0; --i) {
      double s = ze[i];
      for (int j = i + 1; j < ne; ++j) s -= LU[i * ne + j] * ze[j];
      ze[i] = s / LU[i * ne + i];
    }
  }
}
// Deterministic for any thread count: fixed chunk partial sums, summed in order.
double dotv(const double* a, const double* b, size_t n) {
  constexpr int NB = 64;
  double part[NB];
#pragma omp parallel for schedule(static)
  for (int j = 0; j < NB; ++j) {
    const size_t lo = n * j / NB, hi = n * (j + 1) / NB;
    double s = 0.0;
    for (size_t i = lo; i < hi; ++i) s += a[i] * b[i];
    part[j] = s;
  }
  double s = 0.0;
  for (int j = 0; j < NB; ++j) s += part[j];
  return s;
}
}  // namespace

int lo_set_precond_mode(lo_ctx* x, int32_t mode) {
  return guarded([&] {
    if (mode < 0 || mode > 2) throw std::invalid_argument("oracle: precond mode");
    x->c.pc_mode = mode;
    x->c.pc_inverse = mode == 1;
    x->c.pc_built = false;
  });
}

int lo_precond_apply(const lo_ctx* x, const double* r, double* z) {
  return guarded([&] {
    if (!x->c.pc_built) throw std::runtime_error("oracle: preconditioner not built");
    pc_apply(x->c, r, z);
  });
}

// Right-preconditioned restarted GMRES with modified Gram-Schmidt and Givens
// rotations, operator = split_matvec(alpha_dt), preconditioner
// = block-Jacobi (use_pc) or identity; x0 = 0.  Stops when the true residual
// ||b - A x|| <= rtol ||b|| (checked at every restart and at the end) or the
// Givens estimate says so, or after maxit iterations.
int lo_gmres(const lo_ctx* x, double adt, const double* b, double rtol, int32_t maxit, int32_t restart,
             int32_t use_pc, double* xout, int32_t* iters, int32_t* converged, double* resnorm) {
  return guarded([&] {
    const Ctx& c = x->c;
    if (!(rtol > 0.0) || maxit < 1 || restart < 1) throw std::invalid_argument("oracle: gmres arguments");
    if (use_pc && !c.pc_built) throw std::runtime_error("oracle: preconditioner not built");
    const size_t n = static_cast<size_t>(c.E) * c.npe * c.m;
    auto op = [&](const double* v, double* y) {
      if (lo_split_matvec(x, adt, v, y) != LDG_OK) throw std::runtime_error(g_err);
    };
    std::fill(xout, xout + n, 0.0);
    const double bn = std::sqrt(dotv(b, b, n));
    *iters = 0;
    *converged = 0;
    *resnorm = bn;
    if (bn == 0.0) {
      *converged = 1;
      return;
    }
    std::vector<double> r(b, b + n), w(n), t(n);
    const int mr = restart;
    std::vector<std::vector<double>> V(mr + 1, std::vector<double>(n)), Z(mr, std::vector<double>(n));
    std::vector<double> H((mr + 1) * mr), cs(mr), sn(mr), g(mr + 1);
    double beta = bn;
    int it = 0;
    while (true) {
      for (size_t i = 0; i < n; ++i) V[0][i] = r[i] / beta;
      std::fill(g.begin(), g.end(), 0.0);
      g[0] = beta;
      int j = 0;
      for (; j < mr && it < maxit; ++j) {
        if (use_pc) pc_apply(c, V[j].data(), Z[j].data());
        else std::copy(V[j].begin(), V[j].end(), Z[j].begin());
        op(Z[j].data(), w.data());
        for (int i = 0; i <= j; ++i) {
          const double h = dotv(w.data(), V[i].data(), n);
          H[i * mr + j] = h;
          for (size_t q = 0; q < n; ++q) w[q] -= h * V[i][q];
        }
        const double hn = std::sqrt(dotv(w.data(), w.data(), n));
        if (!std::isfinite(hn)) throw std::runtime_error("oracle: gmres numerical breakdown");
        H[(j + 1) * mr + j] = hn;
        if (hn > 0.0)
          for (size_t q = 0; q < n; ++q) V[j + 1][q] = w[q] / hn;
        for (int i = 0; i < j; ++i) {
          const double a0 = H[i * mr + j], a1 = H[(i + 1) * mr + j];
          H[i * mr + j] = cs[i] * a0 + sn[i] * a1;
          H[(i + 1) * mr + j] = -sn[i] * a0 + cs[i] * a1;
        }
        const double a0 = H[j * mr + j], a1 = H[(j + 1) * mr + j];
        const double den = std::hypot(a0, a1);
        cs[j] = den > 0.0 ? a0 / den : 1.0;
        sn[j] = den > 0.0 ? a1 / den : 0.0;
        H[j * mr + j] = den;
        H[(j + 1) * mr + j] = 0.0;
        g[j + 1] = -sn[j] * g[j];
        g[j] = cs[j] * g[j];
        ++it;
        if (std::fabs(g[j + 1]) <= rtol * bn || hn == 0.0) {
          ++j;
          break;
        }
      }
      // x += Z y,  H(0:j,0:j) y = g(0:j)
      std::vector<double> y(j, 0.0);
      for (int i = j - 1; i >= 0; --i) {
        double s = g[i];
        for (int q = i + 1; q < j; ++q) s -= H[i * mr + q] * y[q];
        y[i] = s / H[i * mr + i];
      }
      for (int i = 0; i < j; ++i)
        for (size_t q = 0; q < n; ++q) xout[q] += y[i] * Z[i][q];
      op(xout, t.data());
      for (size_t q = 0; q < n; ++q) r[q] = b[q] - t[q];
      beta = std::sqrt(dotv(r.data(), r.data(), n));
      *resnorm = beta;
      if (beta <= rtol * bn) {
        *converged = 1;
        break;
      }
      if (it >= maxit) break;
    }
    *iters = it;
  });
}

// ---- time integration
namespace {
double inf_norm(const double* a, size_t n) {
  double m = 0.0;
  for (size_t i = 0; i < n; ++i) m = std::max(m, std::fabs(a[i]));
  return m;
}
}  // namespace

int lo_rk4_step(lo_ctx* x, double* U, double t, double dt) {
  return guarded([&] {
    const Ctx& c = x->c;
    const size_t n = static_cast<size_t>(c.E) * c.npe * c.m;
    std::vector<double> k1(n), k2(n), k3(n), k4(n), us(n);
    // stage times t, t + dt/2, t + dt/2, t + dt
    auto F = [&](const double* u, double* k, int stage) {
      const double ts = t + (stage == 1 ? 0.0 : stage == 4 ? dt : 0.5 * dt);
      if (lo_residual(x, u, ts, k, nullptr, nullptr, 0) != LDG_OK) throw std::runtime_error(g_err);
      for (size_t i = 0; i < n; ++i)
        if (!std::isfinite(k[i])) throw std::runtime_error("oracle: rk4 blow-up at stage " + std::to_string(stage));
    };
    F(U, k1.data(), 1);
    for (size_t i = 0; i < n; ++i) us[i] = U[i] + 0.5 * dt * k1[i];
    F(us.data(), k2.data(), 2);
    for (size_t i = 0; i < n; ++i) us[i] = U[i] + 0.5 * dt * k2[i];
    F(us.data(), k3.data(), 3);
    for (size_t i = 0; i < n; ++i) us[i] = U[i] + dt * k3[i];
    F(us.data(), k4.data(), 4);
    for (size_t i = 0; i < n; ++i) U[i] += dt / 6.0 * (k1[i] + 2.0 * k2[i] + 2.0 * k3[i] + k4[i]);
  });
}

// DIRK3: a = [[al,0,0],[tau2-al,al,0],[b1,b2,al]], b = (b1, b2, al).
int lo_dirk3_step(lo_ctx* x, double* U, double t, double dt, const ldg_newton_cfg* cfg, ldg_solver_stats* st) {
  return guarded([&] {
    Ctx& c = x->c;
    if (!(dt > 0.0) || !cfg || cfg->gmres_iters < 1 || cfg->recompute_threshold < 1 || cfg->max_newton < 1)
      throw std::invalid_argument("oracle: dirk3 arguments");
    const double al = 0.435866521508459, tau2 = (1.0 + al) / 2.0;
    const double b1 = -(6.0 * al * al - 16.0 * al + 1.0) / 4.0, b2 = (6.0 * al * al - 20.0 * al + 5.0) / 4.0;
    const double A[3][3] = {{al, 0.0, 0.0}, {tau2 - al, al, 0.0}, {b1, b2, al}};
    const double B[3] = {b1, b2, al};
    const size_t n = static_cast<size_t>(c.E) * c.npe * c.m;
    const double adt = al * dt;
    ldg_solver_stats s{};
    // stage times t + c_i dt, c = (alpha, tau2, 1)
    const double cst[3] = {al, tau2, 1.0};
    auto assemble = [&](const double* u, double ta) {
      if (lo_assemble(x, u, ta, nullptr, 0) != LDG_OK) throw std::runtime_error(g_err);
      ++s.jacobian_assemblies;
      c.pc_built = false;
    };
    auto ensure_pc = [&]() {
      if (cfg->use_precond && (!c.pc_built || c.pc_adt != adt))
        if (lo_precond_build(x, adt) != LDG_OK) throw std::runtime_error(g_err);
    };
    auto F = [&](const double* u, double* k, double ta) {
      if (lo_residual(x, u, ta, k, nullptr, nullptr, 0) != LDG_OK) throw std::runtime_error(g_err);
      ++s.residual_evals;
    };
    if (!c.K[LDG_K11].built) assemble(U, t);
    ensure_pc();
    std::vector<std::vector<double>> K(3, std::vector<double>(n));
    std::vector<double> Kc(n), us(n), Fv(n), G(n), dK(n);
    F(U, Kc.data(), t);  // initial slope guess of stage 1: R(U_n)
    for (int i = 0; i < 3; ++i) {
      int it = 0;
      while (true) {
        for (size_t q = 0; q < n; ++q) {
          double sacc = 0.0;
          for (int j = 0; j < i; ++j) sacc += A[i][j] * K[j][q];
          us[q] = U[q] + dt * (sacc + al * Kc[q]);
        }
        F(us.data(), Fv.data(), t + cst[i] * dt);
        for (size_t q = 0; q < n; ++q) G[q] = Kc[q] - Fv[q];
        const double gn = inf_norm(G.data(), n);
        if (!std::isfinite(gn)) throw std::runtime_error("oracle: dirk3 non-finite stage");
        s.residual_norm = gn;
        if (gn <= cfg->newton_tol) break;
        if (it >= cfg->max_newton) throw std::runtime_error("oracle: dirk3 step failure (Newton did not converge)");
        if (it > 0 && it % cfg->recompute_threshold == 0) {
          assemble(us.data(), t + cst[i] * dt);
          ensure_pc();
        }
        for (size_t q = 0; q < n; ++q) G[q] = -G[q];
        int32_t gi = 0, gc = 0;
        double gr = 0.0;
        if (lo_gmres(x, adt, G.data(), 1e-300, cfg->gmres_iters, cfg->gmres_iters, cfg->use_precond, dK.data(), &gi,
                     &gc, &gr) != LDG_OK)
          throw std::runtime_error(g_err);
        s.gmres_iters += gi;
        for (size_t q = 0; q < n; ++q) Kc[q] += dK[q];
        ++it;
        ++s.newton_iters;
      }
      K[i] = Kc;
    }
    for (size_t q = 0; q < n; ++q) U[q] += dt * (B[0] * K[0][q] + B[1] * K[1][q] + B[2] * K[2][q]);
    if (st) *st = s;
  });
}

// Pseudo-transient continuation: the
// restatement the device driver ldg_steady_solve mirrors operation by
// operation (see include/linedg_b200.h for the contract).
int lo_steady_solve(lo_ctx* x, double* U, double t, const ldg_steady_cfg* cfg, ldg_solver_stats* st) {
  return guarded([&] {
    Ctx& c = x->c;
    if (!cfg || !(cfg->dt0 > 0.0) || !(cfg->growth >= 1.0) || cfg->n_steps < 0 || cfg->gmres_iters < 1 ||
        cfg->recompute_threshold < 1 || cfg->max_newton < 1)
      throw std::invalid_argument("oracle: steady_solve arguments");
    const size_t n = static_cast<size_t>(c.E) * c.npe * c.m;
    const double dt_final = cfg->dt_final > 0.0 ? cfg->dt_final : 1e12;
    const double rtol = cfg->gmres_rtol > 0.0 ? cfg->gmres_rtol : 1e-300;
    ldg_solver_stats s{};
    std::vector<double> R(n), b(n), dU(n), Us(n), Rs(n);
    // residual at U into R; false on a non-physical state (the update is rejected)
    auto F = [&](double& rn) {
      const int code = lo_residual(x, U, t, R.data(), nullptr, nullptr, 0);
      ++s.residual_evals;
      if (code == LDG_ERR_PHYSICAL_STATE) return false;
      if (code != LDG_OK) throw std::runtime_error(g_err);
      rn = inf_norm(R.data(), n);
      return true;
    };
    double rn = 0.0;
    if (!F(rn)) throw std::runtime_error("oracle: steady_solve: non-physical initial state");
    if (!std::isfinite(rn)) throw std::runtime_error("oracle: steady_solve non-finite residual");
    s.residual_norm = rn;
    const double rn0 = rn;
    bool done = rn <= cfg->newton_tol;
    int since = 0, rejects = 0;
    bool fresh = true;  // (re)assemble before the next update
    double dt = cfg->dt0, pc_dt = -1.0;
    // continuation updates left before the final (Newton) phase; a rejected
    // final-phase update returns to continuation for 5 more updates
    int cont_left = cfg->n_steps, newton_left = cfg->max_newton;
    for (int k = 0; !done && (cont_left > 0 || newton_left > 0); ++k) {
      const bool fin = cont_left == 0;
      const double h = fin ? dt_final : dt;
      if (fresh || since >= cfg->recompute_threshold) {
        if (lo_assemble(x, U, t, nullptr, 0) != LDG_OK) throw std::runtime_error(g_err);
        ++s.jacobian_assemblies;
        since = 0;
        fresh = false;
        c.pc_built = false;
      }
      if (cfg->use_precond && (!c.pc_built || pc_dt != h)) {
        if (lo_precond_build(x, h) != LDG_OK) throw std::runtime_error(g_err);
        pc_dt = h;
      }
      for (size_t q = 0; q < n; ++q) b[q] = h * R[q];
      int32_t gi = 0, gc = 0;
      double gr = 0.0;
      if (lo_gmres(x, h, b.data(), rtol, cfg->gmres_iters, cfg->gmres_iters, cfg->use_precond, dU.data(), &gi, &gc,
                   &gr) != LDG_OK)
        throw std::runtime_error(g_err);
      s.gmres_iters += gi;
      std::copy(U, U + n, Us.begin());
      std::copy(R.begin(), R.end(), Rs.begin());
      for (size_t q = 0; q < n; ++q) U[q] += dU[q];
      ++since;
      ++s.newton_iters;
      double rn1 = 0.0;
      const bool phys = F(rn1);
      if (!phys || !(rn1 <= 1e4 * rn0)) {
        // rejected update: restore, halve the pseudo-time step, fresh Jacobian
        // (SPEC.md:535 step-failure policy); the final phase cannot back off
        if (++rejects > 10) throw std::runtime_error("oracle: steady_solve diverged");
        std::copy(Us.begin(), Us.end(), U);
        std::copy(Rs.begin(), Rs.end(), R.begin());
        if (fin) {
          cont_left = 5;  // back to continuation at the last pseudo-time step
          --newton_left;
        } else {
          dt *= 0.5;
        }
        fresh = true;
        continue;
      }
      rn = rn1;
      s.residual_norm = rn;
      done = rn <= cfg->newton_tol;
      if (fin) {
        --newton_left;
      } else {
        --cont_left;
        dt *= cfg->growth;
      }
    }
    if (st) *st = s;
    if (!done) throw std::runtime_error("oracle: steady_solve did not converge");
  });
}

// Algorithmic FP64 flops per ELEMENT of the hot-path kernels,
// from the oracle's templated flux functions on a counting scalar plus the
// line algebra of the algorithm (interpolation, projection, lifting,
// block expansion, 1/J scaling):
//   out[0] residual (first order) or gradient + residual (second order)
//   out[1] Jacobian assembly (K11, + K12 for second order; K21 is U-independent)
//   out[2] K11 SpMV (2 flops per stored value)
//   out[3..6] per evaluation: inviscid normal flux, Riemann flux, viscous
//             normal flux, and (dual-cost) Riemann Jacobian with m seeds
// The Riemann flux is counted once per line end (residual) and its Jacobian
// once per face side pair (face-shared, as the assembly computes it).
int lo_flop_model(const lo_ctx* x, double* out) {
  return guarded([&] {
    const Ctx& c = x->c;
    const int D = c.D, m = c.m, NP = c.np, NQ = c.nq, NL = c.NL, NPE = c.npe, MD = m * D;
    // a physical sample state (free stream + gradient) for the counting runs
    Fl u[MAXM], uo[MAXM], q[MAXM * MAXD], f[MAXM];
    if (c.kind == LDG_POISSON) {
      u[0] = 0.3;
      uo[0] = 0.2;
    } else {
      u[0] = 1.0;
      uo[0] = 1.05;
      for (int d = 0; d < D; ++d) {
        u[1 + d] = 0.3 - 0.1 * d;
        uo[1 + d] = 0.25 + 0.05 * d;
      }
      u[m - 1] = 2.5;
      uo[m - 1] = 2.6;
    }
    for (int k = 0; k < MD; ++k) q[k] = 0.01 * (k + 1);
    const double n[3] = {0.6, 0.8, 0.1};
    const FlCount fn = c.has_inv ? count_ops([&] {
      Ctx cc = c;
      cc.second = false;
      flux_dot(cc, u, q, n, f);
    }) : FlCount{};
    const FlCount fv = c.second ? count_ops([&] { vflux_dot(c, u, q, n, f); }) : FlCount{};
    const FlCount fr = c.has_inv ? count_ops([&] {
      if (c.riemann == LDG_ROE) roe_flux(D, uo, u, n, c.gas, f);
      else llf_flux(D, uo, u, n, c.gas, f);
    }) : FlCount{};
    const double L = D * NL;
    const double interp = 2.0 * NP * m, proj = 2.0 * NP * m, lift = 2.0 * NP * m;
    double res = 0.0, jac = 0.0;
    if (!c.second) {
      res = L * (NQ * (interp + fn.total() + proj) + 2 * (fr.total() + lift)) + NPE * m * (D + 1.0);
    } else {
      // gradient pass: per (line, component): interpolation, u_q nvec_q, projection, lifting
      const double grad = L * m * (NQ * (2.0 * NP + D + 2.0 * NP * D) + 2 * (D + 2.0 * NP * D)) + NPE * MD * D;
      const double resid = L * (NQ * (interp + 2.0 * NP * MD + fn.total() + fv.total() + m + proj) +
                                2 * (fr.total() + fv.total() + m + lift)) + NPE * m * (D + 1.0);
      res = grad + resid;
    }
    const double ns11 = D * c.p + 1 + 2 * D, ns12 = D * c.p + 1 + D;
    // K11: quadrature-point flux Jacobians (forward mode, m seeds), the line
    // block expansion sum_q cc[i][t][q] A_q, endpoint lifting, 1/J scaling
    const double Aq = (c.has_inv ? fn.dual(m) : 0.0) + (c.second && c.vis_u ? fv.dual(m) : 0.0);
    jac = L * (NQ * (interp + Aq) + 2.0 * NP * NP * NQ * m * m + 2 * (fr.dual(m) + 2.0 * NP * m * m)) +
          NPE * ns11 * m * m;
    if (c.second) {
      // K12: dF_vis/dq at the quadrature points (m*D seeds) and its expansion; endpoint viscous Jacobians
      jac += L * (NQ * (2.0 * NP * MD + fv.dual(MD)) + 2.0 * NP * NP * NQ * m * MD + 2 * (fv.dual(MD) + 2.0 * NP * m * MD)) +
             NPE * ns12 * m * MD;
    }
    out[0] = res;
    out[1] = jac;
    out[2] = 2.0 * NPE * ns11 * m * m;
    out[3] = fn.total();
    out[4] = fr.total();
    out[5] = fv.total();
    out[6] = fr.dual(m);
  });
}

// Central-difference Jacobian of one matrix, dense (for <= a few hundred
// unknowns): K11 via R(U +- h e_j, Q), K12 via R(U, Q +- h e_j), K21 via
// D(U +- h e_j); step h = 1e-7 (1 + |x_j|).  Output row-major
// dense nrows x ncols scalars.
int lo_fd_dense(lo_ctx* x, int32_t which, const double* U, const double* Q, double* out) {
  return guarded([&] {
    Ctx& c = x->c;
    const size_t nu = static_cast<size_t>(c.E) * c.npe * c.m;
    const size_t nqd = nu * c.D;
    const size_t ncols = which == LDG_K12 ? nqd : nu;
    const size_t nrows = which == LDG_K21 ? nqd : nu;
    std::vector<double> Up(U, U + nu), Qp;
    if (Q) Qp.assign(Q, Q + nqd);
    std::vector<double> rp(nrows), rm(nrows);
    auto eval = [&](double* r) {
      if (which == LDG_K21) gradient(c, Up.data(), r);
      else residual(c, Up.data(), c.second ? Qp.data() : nullptr, r);
    };
    for (size_t j = 0; j < ncols; ++j) {
      double* xj = which == LDG_K12 ? &Qp[j] : &Up[j];
      const double x0 = *xj, h = 1e-7 * (1.0 + std::abs(x0));
      *xj = x0 + h;
      eval(rp.data());
      *xj = x0 - h;
      eval(rm.data());
      *xj = x0;
      for (size_t i = 0; i < nrows; ++i) out[i * ncols + j] = (rp[i] - rm[i]) / (2.0 * h);
    }
  });
}

}  // extern "C"

// ------------------------------------------------------------------------
// Point physics for the SPEC.md known-answer tests (physics module,
// SPEC.md:309-364).  Return 0 or 1 (physical-state error).
extern "C" {

int lo_euler_flux(int32_t D, const double* u, double gamma, double* F) {
  return guarded([&] {
    Gas g;
    g.gamma = gamma;
    euler_flux(D, u, g, F);
  });
}

int lo_riemann(int32_t kind, int32_t D, const double* uo, const double* ui, const double* n, double gamma,
               double* fh) {
  return guarded([&] {
    Gas g;
    g.gamma = gamma;
    if (kind == LDG_ROE) roe_flux(D, uo, ui, n, g, fh);
    else llf_flux(D, uo, ui, n, g, fh);
  });
}

int lo_ns_viscous_flux(int32_t D, const double* u, const double* q, double gamma, double mu, double pr,
                       double* F) {
  return guarded([&] {
    Gas g;
    g.gamma = gamma;
    g.mu = mu;
    g.prandtl = pr;
    ns_viscous_flux(D, u, q, g, F);
  });
}

}  // extern "C"
