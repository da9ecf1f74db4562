// oracle_physics.hpp -- TEST INFRASTRUCTURE ONLY (the parity checker).
//
// CPU restatement of the reference's per-point physics plug-in
// (physics.hpp:37-93; its implementation physics.cpp is absent from the
// reference tree, proj/src/CMakeLists.txt:5) and of the forward-mode AD
// scalar Dual<N> (dual.hpp:11-118) that turns the templated flux kernels
// into exact Jacobian columns.  Only tests/, __graft_entry__.smoke() and
// bench.py's CPU-baseline leg may load this code; the product never does.
//
// Flux layout F[c*D+d] (physics.hpp:38 generalised from D=2), viscous
// gradient layout q[c*D+d] (field.hpp:38-40).
#pragma once

#include <array>
#include <cmath>
#include <stdexcept>
#include <string>
#include <vector>

namespace ora {

// ------------------------------------------------------------------ Dual<N>
// Same value/derivative rules and branch conventions as dual.hpp:26-103:
// abs() picks a.v >= 0, max()/min() pick the first argument on ties.
template <int N>
struct Dual {
  double v = 0.0;
  std::array<double, N> d{};
  Dual() = default;
  Dual(double x) : v(x) {}  // NOLINT: constants promote implicitly
};
template <int N> inline Dual<N> operator+(const Dual<N>& a, const Dual<N>& b) {
  Dual<N> r(a.v + b.v);
  for (int i = 0; i < N; ++i) r.d[i] = a.d[i] + b.d[i];
  return r;
}
template <int N> inline Dual<N> operator-(const Dual<N>& a, const Dual<N>& b) {
  Dual<N> r(a.v - b.v);
  for (int i = 0; i < N; ++i) r.d[i] = a.d[i] - b.d[i];
  return r;
}
template <int N> inline Dual<N> operator-(const Dual<N>& a) {
  Dual<N> r(-a.v);
  for (int i = 0; i < N; ++i) r.d[i] = -a.d[i];
  return r;
}
template <int N> inline Dual<N> operator*(const Dual<N>& a, const Dual<N>& b) {
  Dual<N> r(a.v * b.v);
  for (int i = 0; i < N; ++i) r.d[i] = a.d[i] * b.v + a.v * b.d[i];
  return r;
}
template <int N> inline Dual<N> operator/(const Dual<N>& a, const Dual<N>& b) {
  Dual<N> r(a.v / b.v);
  const double ib2 = 1.0 / (b.v * b.v);
  for (int i = 0; i < N; ++i) r.d[i] = (a.d[i] * b.v - a.v * b.d[i]) * ib2;
  return r;
}
template <int N> inline Dual<N> operator+(const Dual<N>& a, double b) { return a + Dual<N>(b); }
template <int N> inline Dual<N> operator+(double a, const Dual<N>& b) { return Dual<N>(a) + b; }
template <int N> inline Dual<N> operator-(const Dual<N>& a, double b) { return a - Dual<N>(b); }
template <int N> inline Dual<N> operator-(double a, const Dual<N>& b) { return Dual<N>(a) - b; }
template <int N> inline Dual<N> operator*(const Dual<N>& a, double b) { return a * Dual<N>(b); }
template <int N> inline Dual<N> operator*(double a, const Dual<N>& b) { return Dual<N>(a) * b; }
template <int N> inline Dual<N> operator/(const Dual<N>& a, double b) { return a / Dual<N>(b); }
template <int N> inline Dual<N> operator/(double a, const Dual<N>& b) { return Dual<N>(a) / b; }
template <int N> inline bool operator<(const Dual<N>& a, const Dual<N>& b) { return a.v < b.v; }
template <int N> inline bool operator<(const Dual<N>& a, double b) { return a.v < b; }
template <int N> inline bool operator<=(const Dual<N>& a, double b) { return a.v <= b; }
template <int N> inline Dual<N> sqrt(const Dual<N>& a) {
  Dual<N> r(std::sqrt(a.v));
  const double s = 0.5 / r.v;
  for (int i = 0; i < N; ++i) r.d[i] = s * a.d[i];
  return r;
}
template <int N> inline Dual<N> abs(const Dual<N>& a) { return a.v >= 0.0 ? a : -a; }
template <int N> inline Dual<N> max(const Dual<N>& a, const Dual<N>& b) { return a.v >= b.v ? a : b; }
inline double value_of(double x) { return x; }
inline double value_of(long double x) { return static_cast<double>(x); }
template <int N> inline double value_of(const Dual<N>& x) { return x.v; }
using std::abs;
using std::sqrt;
inline double max(double a, double b) { return a >= b ? a : b; }
inline long double max(long double a, long double b) { return a >= b ? a : b; }

// Raised on rho <= 0 or p <= 0 (errors.hpp:10-18; physics.hpp:192).
struct physical_state_error : std::runtime_error {
  std::vector<double> state;
  physical_state_error(const std::string& w, std::vector<double> s)
      : std::runtime_error(w), state(std::move(s)) {}
};

struct Gas {
  double gamma = 1.4, mu = 0.0, prandtl = 0.72;
};

template <class T>
[[noreturn]] void bad_state(const char* what, const T* u, int m) {
  std::vector<double> s(m);
  for (int c = 0; c < m; ++c) s[c] = value_of(u[c]);
  throw physical_state_error(what, s);
}

// Euler flux tensor F[c*D+d] and pressure.
template <class T>
void euler_flux(int D, const T* u, const Gas& g, T* F, T* p_out = nullptr) {
  const int m = D + 2;
  const T rho = u[0];
  if (!(value_of(rho) > 0.0)) bad_state("euler_flux: non-positive density", u, m);
  T vel[3];
  T mom2 = 0.0;
  for (int d = 0; d < D; ++d) {
    vel[d] = u[1 + d] / rho;
    mom2 = mom2 + u[1 + d] * vel[d];
  }
  const T p = (g.gamma - 1.0) * (u[D + 1] - 0.5 * mom2);
  if (!(value_of(p) > 0.0)) bad_state("euler_flux: non-positive pressure", u, m);
  for (int d = 0; d < D; ++d) {
    F[0 * D + d] = u[1 + d];
    for (int i = 0; i < D; ++i) F[(1 + i) * D + d] = u[1 + i] * vel[d] + (i == d ? p : T(0.0));
    F[(D + 1) * D + d] = vel[d] * (u[D + 1] + p);
  }
  if (p_out) *p_out = p;
}

// Roe flux with the Harten entropy fix on the acoustic waves, delta =
// 0.05(|u.n|+a), evaluated on the unit normal and scaled by |n|
// (physics.hpp:194-198).
// Argument order follows PhysicsModel::riemann(u_out, u_in, n) with the
// outward, non-normalised normal n (physics.hpp:54-58).
template <class T>
void roe_flux(int D, const T* uo, const T* ui, const double* n, const Gas& g, T* fh) {
  const int m = D + 2;
  double nn = 0.0;
  for (int d = 0; d < D; ++d) nn += n[d] * n[d];
  nn = std::sqrt(nn);
  double nb[3];
  for (int d = 0; d < D; ++d) nb[d] = n[d] / nn;
  T FL[15], FR[15], pL, pR;
  euler_flux(D, ui, g, FL, &pL);
  euler_flux(D, uo, g, FR, &pR);
  const T rL = ui[0], rR = uo[0];
  T vL[3], vR[3];
  for (int d = 0; d < D; ++d) {
    vL[d] = ui[1 + d] / rL;
    vR[d] = uo[1 + d] / rR;
  }
  const T HL = (ui[D + 1] + pL) / rL, HR = (uo[D + 1] + pR) / rR;
  const T sL = sqrt(rL), sR = sqrt(rR);
  const T sw = sL + sR;
  T vt[3], q2 = 0.0, unt = 0.0;
  for (int d = 0; d < D; ++d) {
    vt[d] = (sL * vL[d] + sR * vR[d]) / sw;
    q2 = q2 + vt[d] * vt[d];
    unt = unt + vt[d] * nb[d];
  }
  const T Ht = (sL * HL + sR * HR) / sw;
  const T a2 = (g.gamma - 1.0) * (Ht - 0.5 * q2);
  if (!(value_of(a2) > 0.0)) bad_state("roe_flux: non-positive Roe sound speed", ui, m);
  const T a = sqrt(a2);
  const T rt = sL * sR;
  const T drho = rR - rL, dp = pR - pL;
  T dv[3], dun = 0.0, vtdv = 0.0;
  for (int d = 0; d < D; ++d) {
    dv[d] = vR[d] - vL[d];
    dun = dun + dv[d] * nb[d];
    vtdv = vtdv + vt[d] * dv[d];
  }
  T l1 = abs(unt - a), l2 = abs(unt), l3 = abs(unt + a);
  const T del = 0.05 * (abs(unt) + a);
  if (l1 < del) l1 = (l1 * l1 + del * del) / (2.0 * del);
  if (l3 < del) l3 = (l3 * l3 + del * del) / (2.0 * del);
  const T al1 = (dp - rt * a * dun) / (2.0 * a2);
  const T al3 = (dp + rt * a * dun) / (2.0 * a2);
  const T al2 = drho - dp / a2;
  T dis[5];
  dis[0] = l1 * al1 + l2 * al2 + l3 * al3;
  for (int i = 0; i < D; ++i)
    dis[1 + i] = l1 * al1 * (vt[i] - a * nb[i]) + l2 * (al2 * vt[i] + rt * (dv[i] - dun * nb[i])) +
                 l3 * al3 * (vt[i] + a * nb[i]);
  dis[D + 1] = l1 * al1 * (Ht - unt * a) + l2 * (al2 * (0.5 * q2) + rt * (vtdv - unt * dun)) +
               l3 * al3 * (Ht + unt * a);
  for (int c = 0; c < m; ++c) {
    T fl = 0.0, fr = 0.0;
    for (int d = 0; d < D; ++d) {
      fl = fl + FL[c * D + d] * nb[d];
      fr = fr + FR[c * D + d] * nb[d];
    }
    fh[c] = nn * (0.5 * (fl + fr) - 0.5 * dis[c]);
  }
}

// Local Lax-Friedrichs: 1/2 (F(u_in)+F(u_out)).n + 1/2 lambda |n| (u_in - u_out),
// lambda = max over both states of |u.n_unit| + c.  (Extension: config 4.)
template <class T>
void llf_flux(int D, const T* uo, const T* ui, const double* n, const Gas& g, T* fh) {
  const int m = D + 2;
  double nn = 0.0;
  for (int d = 0; d < D; ++d) nn += n[d] * n[d];
  nn = std::sqrt(nn);
  T FL[15], FR[15], pL, pR;
  euler_flux(D, ui, g, FL, &pL);
  euler_flux(D, uo, g, FR, &pR);
  T unL = 0.0, unR = 0.0;
  for (int d = 0; d < D; ++d) {
    unL = unL + ui[1 + d] * (n[d] / nn);
    unR = unR + uo[1 + d] * (n[d] / nn);
  }
  unL = unL / ui[0];
  unR = unR / uo[0];
  const T cL = sqrt(g.gamma * pL / ui[0]), cR = sqrt(g.gamma * pR / uo[0]);
  const T lam = max(abs(unL) + cL, abs(unR) + cR);
  for (int c = 0; c < m; ++c) {
    T fl = 0.0, fr = 0.0;
    for (int d = 0; d < D; ++d) {
      fl = fl + FL[c * D + d] * n[d];
      fr = fr + FR[c * D + d] * n[d];
    }
    fh[c] = 0.5 * (fl + fr) + 0.5 * lam * nn * (ui[c] - uo[c]);
  }
}

// Navier-Stokes viscous stress in the +tau convention (physics.hpp:200-205;
// SPEC.md:340-348): row 0 zero, momentum rows tau_ij, energy row
// u_i tau_ij - heat_j with heat_j = -(mu/Pr) d/dx_j (E + p/rho - |u|^2/2).
// Dilatation uses the divergence du_k/dx_k.  The model
// viscous flux is -T.
template <class T>
void ns_viscous_flux(int D, const T* u, const T* q, const Gas& g, T* F) {
  const int m = D + 2;
  const T rho = u[0];
  if (!(value_of(rho) > 0.0)) bad_state("ns_viscous_flux: non-positive density", u, m);
  T vel[3], gv[3][3], gE[3];
  const T E = u[D + 1] / rho;
  for (int i = 0; i < D; ++i) vel[i] = u[1 + i] / rho;
  for (int d = 0; d < D; ++d) {
    for (int i = 0; i < D; ++i) gv[i][d] = (q[(1 + i) * D + d] - vel[i] * q[d]) / rho;
    gE[d] = (q[(D + 1) * D + d] - E * q[d]) / rho;
  }
  T div = 0.0;
  for (int k = 0; k < D; ++k) div = div + gv[k][k];
  const double mu = g.mu, kap = g.mu / g.prandtl * g.gamma;
  for (int d = 0; d < D; ++d) F[d] = 0.0;
  for (int i = 0; i < D; ++i)
    for (int j = 0; j < D; ++j) {
      T tau = mu * (gv[i][j] + gv[j][i]);
      if (i == j) tau = tau - (2.0 / 3.0) * mu * div;
      F[(1 + i) * D + j] = -tau;
    }
  for (int j = 0; j < D; ++j) {
    T work = 0.0, ugv = 0.0;
    for (int i = 0; i < D; ++i) {
      work = work + vel[i] * (-F[(1 + i) * D + j]);
      ugv = ugv + vel[i] * gv[i][j];
    }
    F[(D + 1) * D + j] = -(work + kap * (gE[j] - ugv));
  }
}

}  // namespace ora
