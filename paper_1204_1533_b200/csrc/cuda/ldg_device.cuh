// ldg_device.cuh -- compile-time configuration, device forward-mode scalar
// and point physics for the sm_100a Line-DG kernels.
//
// Physics follows the reference plug-in semantics (physics.hpp:37-93):
// riemann(u_out, u_in, n) with the outward non-normalised normal, F_hat.n =
// |n| F_hat.n_unit; Roe with the Harten fix on the
// acoustic waves (physics.hpp:194-198); Navier-Stokes stress and
// heat flux from conservative gradients.  The device code
// works directly with normal fluxes F.n (never forms the D x m tensor).
#pragma once

#include <cstdint>

#include "linedg_b200.h"

namespace ldg {

enum { PH_POISSON = 0, PH_EULER = 1, PH_NS = 2 };

template <int D_, int P_, int PH_, int RI_>
struct Cfg {
  static constexpr int D = D_, P = P_, PH = PH_, RI = RI_;
  static constexpr int NP = P + 1;
  static constexpr int NQ = (3 * P + 2) / 2;              // basis.cpp:176
  static constexpr int NPE = D == 2 ? NP * NP : NP * NP * NP;
  static constexpr int NL = D == 2 ? NP : NP * NP;        // lines per direction
  static constexpr int LPE = D * NL;                      // lines per element
  static constexpr int M = PH == PH_POISSON ? 1 : D + 2;  // components
  static constexpr int MD = M * D;
  static constexpr bool HAS_INV = PH != PH_POISSON;
  static constexpr bool SECOND = PH != PH_EULER;          // LDG auxiliary gradient present
  static constexpr bool VIS_U = PH == PH_NS;              // viscous flux depends on u
  // Metric tables per element (processing order), padded to 16 bytes.
  static constexpr int MET_NV = D * NL * NQ * D;
  static constexpr int MET_NE = D * 2 * NL * D;
  static constexpr int MET = MET_NV + MET_NE + NPE;
  static constexpr int METP = (MET + 1) / 2 * 2;
  // Line-structured Jacobian store: rows tiled by NT rows.  2-D: one
  // element (NP^2 rows); 3-D: one slab x2 = const (NP^2 rows), or, for the
  // 3-D p >= 4 Navier-Stokes operator whose slab tile does not fit shared
  // memory, one dir-0 coordinate line (NP rows).  Node = tile*NT + row.
  static constexpr int TD = (D == 3 && PH == PH_NS && P >= 4) ? 1 : 2;
  static constexpr int NT = TD == 1 ? NP : NP * NP;
  static constexpr int TPE = NPE / NT;                    // tiles per element
  // Assembly work unit of one CTA (independent of the store tile): the whole
  // element when its flux-Jacobian working set fits shared memory, else one
  // slab (x2 = const) or one dir-0 line of rows (3-D only).
  static constexpr long long wu_bytes(int nlt) {
    return 8LL * (NPE * M + (PH != PH_EULER ? NPE * M * D : 0) + nlt * NQ * M * M * ((PH == PH_NS) ? 2 : 1) +
                  (PH != PH_EULER ? nlt * NQ * M * M * D : 0) +
                  nlt * 2 * (2 * M * M + (PH != PH_EULER ? M * M * D : 0)));
  }
  static constexpr int WU = D == 2 ? 0
                            : (wu_bytes(D * NL) <= 100 * 1024 ? 0
                                                              : (wu_bytes(2 * NP + NP * NP) <= 200 * 1024 ? 1 : 2));
  static constexpr int UPE = WU == 0 ? 1 : (WU == 1 ? NP : NP * NP);  // work units per element
  static constexpr int NS11 = D * P + 1 + 2 * D;          // K11 node-columns per row
  static constexpr int NS12 = D * P + 1 + D;              // K12 / K21 node-columns per row
  static constexpr int B11 = M * M;
  static constexpr int R12 = PH == PH_NS ? M - 1 : M;     // K12 rows stored (density row dropped)
  static constexpr int B12 = R12 * MD;
  static constexpr int B21 = D;                           // component-diagonal scalars
};

// Basis tables folded for the line operators (host-built once):
//   dq[i][q] = -(M^-1 Phi' W)[i][q]   volume operator,
//   mi[i][s] = M^-1[i][s ? p : 0]     endpoint lifting,
//   cc[i][t][q] = dq[i][q] phi[t][q]  Jacobian line blocks.
template <int NP, int NQ>
struct BasisTab {
  double phi[NP][NQ];
  double dq[NP][NQ];
  double mi[NP][2];
  double cc[NP][NP][NQ];
};

struct DevError {
  int flag;       // 0 ok, 1 physical state
  int elem;
  int node;
  int pad;
  double state[8];
};

struct PhysParams {
  double gamma, mu, kap;  // kap = mu * gamma / Pr
  double c11, c11bd;      // interior C11; boundary coefficient c11_bd * p^2
};

// Boundary condition kinds (reference BcKind, physics.hpp:16; the values of
// ldg_bc_kind in include/linedg_b200.h).
enum BcKindDev : int { BC_DIRICHLET = 0, BC_NEUMANN = 1, BC_CHARACTERISTIC = 2, BC_SLIP_WALL = 3, BC_NO_SLIP = 4 };

// ------------------------------------------------------------ Dual<N>
template <int N>
struct Dual {
  double v;
  double d[N];
  __device__ __forceinline__ Dual() {}
  __device__ __forceinline__ Dual(double x) : v(x) {
#pragma unroll
    for (int i = 0; i < N; ++i) d[i] = 0.0;
  }
};
template <int N> __device__ __forceinline__ Dual<N> operator+(const Dual<N>& a, const Dual<N>& b) {
  Dual<N> r; r.v = a.v + b.v;
#pragma unroll
  for (int i = 0; i < N; ++i) r.d[i] = a.d[i] + b.d[i];
  return r;
}
template <int N> __device__ __forceinline__ Dual<N> operator-(const Dual<N>& a, const Dual<N>& b) {
  Dual<N> r; r.v = a.v - b.v;
#pragma unroll
  for (int i = 0; i < N; ++i) r.d[i] = a.d[i] - b.d[i];
  return r;
}
template <int N> __device__ __forceinline__ Dual<N> operator-(const Dual<N>& a) {
  Dual<N> r; r.v = -a.v;
#pragma unroll
  for (int i = 0; i < N; ++i) r.d[i] = -a.d[i];
  return r;
}
template <int N> __device__ __forceinline__ Dual<N> operator*(const Dual<N>& a, const Dual<N>& b) {
  Dual<N> r; r.v = a.v * b.v;
#pragma unroll
  for (int i = 0; i < N; ++i) r.d[i] = a.d[i] * b.v + a.v * b.d[i];
  return r;
}
template <int N> __device__ __forceinline__ Dual<N> operator/(const Dual<N>& a, const Dual<N>& b) {
  Dual<N> r; r.v = a.v / b.v;
  const double ib = 1.0 / b.v;
#pragma unroll
  for (int i = 0; i < N; ++i) r.d[i] = (a.d[i] - r.v * b.d[i]) * ib;
  return r;
}
template <int N> __device__ __forceinline__ Dual<N> operator+(const Dual<N>& a, double b) {
  Dual<N> r = a; r.v += b; return r;
}
template <int N> __device__ __forceinline__ Dual<N> operator+(double a, const Dual<N>& b) { return b + a; }
template <int N> __device__ __forceinline__ Dual<N> operator-(const Dual<N>& a, double b) {
  Dual<N> r = a; r.v -= b; return r;
}
template <int N> __device__ __forceinline__ Dual<N> operator-(double a, const Dual<N>& b) {
  Dual<N> r; r.v = a - b.v;
#pragma unroll
  for (int i = 0; i < N; ++i) r.d[i] = -b.d[i];
  return r;
}
template <int N> __device__ __forceinline__ Dual<N> operator*(const Dual<N>& a, double b) {
  Dual<N> r; r.v = a.v * b;
#pragma unroll
  for (int i = 0; i < N; ++i) r.d[i] = a.d[i] * b;
  return r;
}
template <int N> __device__ __forceinline__ Dual<N> operator*(double a, const Dual<N>& b) { return b * a; }
template <int N> __device__ __forceinline__ Dual<N> operator/(const Dual<N>& a, double b) {
  const double ib = 1.0 / b;
  Dual<N> r; r.v = a.v / b;
#pragma unroll
  for (int i = 0; i < N; ++i) r.d[i] = a.d[i] * ib;
  return r;
}
template <int N> __device__ __forceinline__ Dual<N> operator/(double a, const Dual<N>& b) {
  return Dual<N>(a) / b;
}
template <int N> __device__ __forceinline__ Dual<N> dsqrt(const Dual<N>& a) {
  Dual<N> r; r.v = sqrt(a.v);
  const double s = 0.5 / r.v;
#pragma unroll
  for (int i = 0; i < N; ++i) r.d[i] = s * a.d[i];
  return r;
}
template <int N> __device__ __forceinline__ Dual<N> dabs(const Dual<N>& a) { return a.v >= 0.0 ? a : -a; }
template <int N> __device__ __forceinline__ Dual<N> dmax(const Dual<N>& a, const Dual<N>& b) {
  return a.v >= b.v ? a : b;
}
__device__ __forceinline__ double dsqrt(double a) { return sqrt(a); }
__device__ __forceinline__ double dabs(double a) { return a >= 0.0 ? a : -a; }
__device__ __forceinline__ double dmax(double a, double b) { return a >= b ? a : b; }
__device__ __forceinline__ double val(double a) { return a; }
template <int N> __device__ __forceinline__ double val(const Dual<N>& a) { return a.v; }

// Records the first physical-state failure (errors.hpp:10-18).
template <class T, int M>
__device__ __noinline__ void report_bad_state(DevError* err, int elem, int node, const T* u) {
  if (atomicCAS(&err->flag, 0, 1) == 0) {
    err->elem = elem;
    err->node = node;
    for (int c = 0; c < M && c < 8; ++c) err->state[c] = val(u[c]);
  }
}

// ------------------------------------------------------------- physics
// Normal Euler flux F(u).n for a (non-normalised) vector n; returns p.
// ok = false on rho <= 0 or p <= 0.
template <int D, class T>
__device__ __forceinline__ T euler_fn(const T* u, const double* n, double gamma, T* fn, bool& ok) {
  const T rho = u[0];
  const T irho = 1.0 / rho;
  T mom2 = u[1] * u[1];
  T mn = u[1] * n[0];
#pragma unroll
  for (int d = 1; d < D; ++d) {
    mom2 = mom2 + u[1 + d] * u[1 + d];
    mn = mn + u[1 + d] * n[d];
  }
  const T p = (gamma - 1.0) * (u[D + 1] - 0.5 * mom2 * irho);
  ok = ok && (val(rho) > 0.0) && (val(p) > 0.0);
  const T un = mn * irho;
  fn[0] = mn;
#pragma unroll
  for (int i = 0; i < D; ++i) fn[1 + i] = u[1 + i] * un + p * n[i];
  fn[D + 1] = un * (u[D + 1] + p);
  return p;
}

// Closed-form d(F(u).n)/du (row-major M x M) for the Euler flux.
template <int D>
__device__ __forceinline__ void euler_jac_n(const double* u, const double* n, double gamma, double* A,
                                            bool& ok) {
  constexpr int M = D + 2;
  const double g1 = gamma - 1.0;
  const double rho = u[0], irho = 1.0 / rho;
  double v[D], un = 0.0, q2 = 0.0;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    v[d] = u[1 + d] * irho;
    un += v[d] * n[d];
    q2 += v[d] * v[d];
  }
  const double p = g1 * (u[D + 1] - 0.5 * rho * q2);
  ok = ok && (rho > 0.0) && (p > 0.0);
  const double H = (u[D + 1] + p) * irho;
  const double hq = 0.5 * g1 * q2;
  A[0] = 0.0;
#pragma unroll
  for (int j = 0; j < D; ++j) A[1 + j] = n[j];
  A[D + 1] = 0.0;
#pragma unroll
  for (int i = 0; i < D; ++i) {
    double* r = A + (1 + i) * M;
    r[0] = hq * n[i] - v[i] * un;
#pragma unroll
    for (int j = 0; j < D; ++j) r[1 + j] = v[i] * n[j] - g1 * v[j] * n[i] + (i == j ? un : 0.0);
    r[D + 1] = g1 * n[i];
  }
  double* r = A + (D + 1) * M;
  r[0] = un * (hq - H);
#pragma unroll
  for (int j = 0; j < D; ++j) r[1 + j] = H * n[j] - g1 * un * v[j];
  r[D + 1] = gamma * un;
}

// Exterior state of a boundary line end for the Riemann flux
// (SPEC.md:266, 366-368): Dirichlet / characteristic far field -> g (the
// prescribed / free-stream state); slip wall -> the interior state with its
// normal momentum mirrored, m - 2 (m.n) n / |n|^2.  T = double or Dual<N>
// (the ghost is a function of u_in, so its derivative carries through).
template <int D, int M, class T>
__device__ __forceinline__ void bc_ghost(int kind, const double* g, const T* ui, const double* n, T* uo) {
  if (M == D + 2 && kind == BC_NO_SLIP) {
    // no-slip wall: the interior state with its full momentum reversed
    uo[0] = ui[0];
#pragma unroll
    for (int d = 0; d < D; ++d) uo[1 + d] = -ui[1 + d];
    uo[M - 1] = ui[M - 1];
  } else if (M == D + 2 && kind == BC_SLIP_WALL) {
    double n2 = n[0] * n[0];
#pragma unroll
    for (int d = 1; d < D; ++d) n2 += n[d] * n[d];
    T mn = ui[1] * n[0];
#pragma unroll
    for (int d = 1; d < D; ++d) mn = mn + ui[1 + d] * n[d];
    const T f = mn * (2.0 / n2);
    uo[0] = ui[0];
#pragma unroll
    for (int d = 0; d < D; ++d) uo[1 + d] = ui[1 + d] - f * n[d];
    uo[M - 1] = ui[M - 1];
  } else {
#pragma unroll
    for (int c = 0; c < M; ++c) uo[c] = T(__ldg(g + c));
  }
}

// Roe flux (u_out = R, u_in = L), outward normal n.
template <int D, class T>
__device__ __forceinline__ void roe_fn(const T* uo, const T* ui, const double* n, double gamma,
                                       T* fh, bool& ok) {
  double nn = n[0] * n[0];
#pragma unroll
  for (int d = 1; d < D; ++d) nn += n[d] * n[d];
  nn = sqrt(nn);
  const double inn = 1.0 / nn;
  double nb[D];
#pragma unroll
  for (int d = 0; d < D; ++d) nb[d] = n[d] * inn;
  T fl[D + 2], fr[D + 2];
  const T pL = euler_fn<D>(ui, nb, gamma, fl, ok);
  const T pR = euler_fn<D>(uo, nb, gamma, fr, ok);
  const T irL = 1.0 / ui[0], irR = 1.0 / uo[0];
  const T sL = dsqrt(ui[0]), sR = dsqrt(uo[0]);
  const T isw = 1.0 / (sL + sR);
  const T wL = sL * isw, wR = sR * isw;
  T vL[D], vR[D], vt[D];
  T q2 = 0.0, unt = 0.0, dun = 0.0, vtdv = 0.0;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    vL[d] = ui[1 + d] * irL;
    vR[d] = uo[1 + d] * irR;
    vt[d] = wL * vL[d] + wR * vR[d];
    q2 = q2 + vt[d] * vt[d];
    unt = unt + vt[d] * nb[d];
  }
  const T HL = (ui[D + 1] + pL) * irL, HR = (uo[D + 1] + pR) * irR;
  const T Ht = wL * HL + wR * HR;
  const T a2 = (gamma - 1.0) * (Ht - 0.5 * q2);
  ok = ok && (val(a2) > 0.0);
  const T a = dsqrt(a2);
  const T ia2 = 1.0 / a2;
  const T rt = sL * sR;
  const T drho = uo[0] - ui[0], dp = pR - pL;
  T dv[D];
#pragma unroll
  for (int d = 0; d < D; ++d) {
    dv[d] = vR[d] - vL[d];
    dun = dun + dv[d] * nb[d];
    vtdv = vtdv + vt[d] * dv[d];
  }
  T l1 = dabs(unt - a), l2 = dabs(unt), l3 = dabs(unt + a);
  const T del = 0.05 * (l2 + a);
  if (val(l1) < val(del)) l1 = (l1 * l1 + del * del) / (2.0 * del);
  if (val(l3) < val(del)) l3 = (l3 * l3 + del * del) / (2.0 * del);
  const T ra = rt * a * dun;
  const T al1 = 0.5 * (dp - ra) * ia2;
  const T al3 = 0.5 * (dp + ra) * ia2;
  const T al2 = drho - dp * ia2;
  const T w1 = l1 * al1, w3 = l3 * al3;
  const T hn = 0.5 * nn;
  fh[0] = hn * (fl[0] + fr[0] - (w1 + l2 * al2 + w3));
#pragma unroll
  for (int i = 0; i < D; ++i) {
    const T dis = w1 * (vt[i] - a * nb[i]) + l2 * (al2 * vt[i] + rt * (dv[i] - dun * nb[i])) +
                  w3 * (vt[i] + a * nb[i]);
    fh[1 + i] = hn * (fl[1 + i] + fr[1 + i] - dis);
  }
  const T dise = w1 * (Ht - unt * a) + l2 * (al2 * (0.5 * q2) + rt * (vtdv - unt * dun)) +
                 w3 * (Ht + unt * a);
  fh[D + 1] = hn * (fl[D + 1] + fr[D + 1] - dise);
}

// Local Lax-Friedrichs (extension, config 4).
template <int D, class T>
__device__ __forceinline__ void llf_fn(const T* uo, const T* ui, const double* n, double gamma,
                                       T* fh, bool& ok) {
  double nn = n[0] * n[0];
#pragma unroll
  for (int d = 1; d < D; ++d) nn += n[d] * n[d];
  nn = sqrt(nn);
  const double inn = 1.0 / nn;
  double nb[D];
#pragma unroll
  for (int d = 0; d < D; ++d) nb[d] = n[d] * inn;
  T fl[D + 2], fr[D + 2];
  const T pL = euler_fn<D>(ui, n, gamma, fl, ok);
  const T pR = euler_fn<D>(uo, n, gamma, fr, ok);
  T mL = ui[1] * nb[0], mR = uo[1] * nb[0];
#pragma unroll
  for (int d = 1; d < D; ++d) {
    mL = mL + ui[1 + d] * nb[d];
    mR = mR + uo[1 + d] * nb[d];
  }
  const T irL = 1.0 / ui[0], irR = 1.0 / uo[0];
  const T lam = dmax(dabs(mL * irL) + dsqrt(gamma * pL * irL), dabs(mR * irR) + dsqrt(gamma * pR * irR));
  const T hl = 0.5 * nn * lam;
#pragma unroll
  for (int c = 0; c < D + 2; ++c) fh[c] = 0.5 * (fl[c] + fr[c]) + hl * (ui[c] - uo[c]);
}

// Closed-form Jacobian of llf_fn: pass 0 -> dFh/du_in, pass 1 -> dFh/du_out
// (row-major M x M).  The primal expressions (p, m.nb, lambda) are written
// exactly as in llf_fn so the |.| and max branch choices are the same as the
// dual-number evaluation's:
//   dFh/du_X = 1/2 A(u_X, n) +- 1/2 |n| lam I + 1/2 |n| (u_in - u_out) (x) dlam/du_X,
// dlam/du_X nonzero only for the side max() selected.
template <int D>
__device__ __forceinline__ void llf_jac(const double* uo, const double* ui, const double* n, double gamma,
                                        const int pass, double* J, bool& ok) {
  constexpr int M = D + 2;
  double nn = n[0] * n[0];
#pragma unroll
  for (int d = 1; d < D; ++d) nn += n[d] * n[d];
  nn = sqrt(nn);
  const double inn = 1.0 / nn;
  double nb[D];
#pragma unroll
  for (int d = 0; d < D; ++d) nb[d] = n[d] * inn;
  double fl[M], fr[M];
  const double pL = euler_fn<D>(ui, n, gamma, fl, ok);
  const double pR = euler_fn<D>(uo, n, gamma, fr, ok);
  double mL = ui[1] * nb[0], mR = uo[1] * nb[0];
#pragma unroll
  for (int d = 1; d < D; ++d) {
    mL = mL + ui[1 + d] * nb[d];
    mR = mR + uo[1 + d] * nb[d];
  }
  const double irL = 1.0 / ui[0], irR = 1.0 / uo[0];
  const double unL = mL * irL, unR = mR * irR;
  const double cL = sqrt(gamma * pL * irL), cR = sqrt(gamma * pR * irR);
  const double lamL = dabs(unL) + cL, lamR = dabs(unR) + cR;
  const bool pickL = lamL >= lamR;
  const double lam = pickL ? lamL : lamR;
  const double* u = pass == 0 ? ui : uo;
  euler_jac_n<D>(u, n, gamma, J, ok);
  const double hn = 0.5 * nn, dg = pass == 0 ? hn * lam : -hn * lam;
#pragma unroll
  for (int c = 0; c < M * M; ++c) J[c] *= 0.5;
#pragma unroll
  for (int c = 0; c < M; ++c) J[c * M + c] += dg;
  if (pickL == (pass == 0)) {
    // dlam/du of the selected side: s dun/du + dc/du
    const double ir = pass == 0 ? irL : irR, un = pass == 0 ? unL : unR, c = pass == 0 ? cL : cR;
    const double p = pass == 0 ? pL : pR;
    const double s = un >= 0.0 ? 1.0 : -1.0;
    double mom2 = 0.0;
#pragma unroll
    for (int d = 0; d < D; ++d) mom2 += u[1 + d] * u[1 + d];
    const double g1 = gamma - 1.0, k = 0.5 * gamma * ir / c;
    double dl[M];
    dl[0] = -s * un * ir + k * (0.5 * g1 * mom2 * ir * ir - p * ir);
#pragma unroll
    for (int d = 0; d < D; ++d) dl[1 + d] = s * nb[d] * ir - k * g1 * u[1 + d] * ir;
    dl[D + 1] = k * g1;
#pragma unroll
    for (int c = 0; c < M; ++c) {
      const double w = hn * (ui[c] - uo[c]);
#pragma unroll
      for (int b = 0; b < M; ++b) J[c * M + b] += w * dl[b];
    }
  }
}

// Viscous normal flux F_vis(u, q).n.  Poisson: -q.n.  Navier-Stokes: minus
// the +tau stress tensor dotted with n.  q layout q[c*D+d].
template <int D, int PH, class T, class TQ, class TR>
__device__ __forceinline__ void visc_fn(const T* u, const TQ* q, const double* n, const PhysParams& pp,
                                        TR* fv, bool& ok) {
  if (PH == PH_POISSON) {
    TR s = -(q[0] * n[0]);
#pragma unroll
    for (int d = 1; d < D; ++d) s = s - q[d] * n[d];
    fv[0] = s;
  } else {
    const T rho = u[0];
    ok = ok && (val(rho) > 0.0);
    const T irho = 1.0 / rho;
    T vel[D];
#pragma unroll
    for (int i = 0; i < D; ++i) vel[i] = u[1 + i] * irho;
    const T E = u[D + 1] * irho;
    TR gv[D][D], gE[D];
#pragma unroll
    for (int d = 0; d < D; ++d) {
#pragma unroll
      for (int i = 0; i < D; ++i) gv[i][d] = (q[(1 + i) * D + d] - vel[i] * q[d]) * irho;
      gE[d] = (q[(D + 1) * D + d] - E * q[d]) * irho;
    }
    TR div = gv[0][0];
#pragma unroll
    for (int k = 1; k < D; ++k) div = div + gv[k][k];
    const double mu = pp.mu;
    // tau . n and the heat term
    TR tn[D];
#pragma unroll
    for (int i = 0; i < D; ++i) {
      TR s = (mu * (gv[i][0] + gv[0][i])) * n[0];
#pragma unroll
      for (int j = 1; j < D; ++j) s = s + (mu * (gv[i][j] + gv[j][i])) * n[j];
      tn[i] = s - ((2.0 / 3.0) * mu) * div * n[i];
    }
    fv[0] = TR(0.0);
    TR en = TR(0.0);
#pragma unroll
    for (int i = 0; i < D; ++i) {
      fv[1 + i] = -tn[i];
      en = en + vel[i] * tn[i];
    }
    TR hn = TR(0.0);
#pragma unroll
    for (int j = 0; j < D; ++j) {
      TR ugv = vel[0] * gv[0][j];
#pragma unroll
      for (int i = 1; i < D; ++i) ugv = ugv + vel[i] * gv[i][j];
      hn = hn + (gE[j] - ugv) * n[j];
    }
    fv[D + 1] = -(en + pp.kap * hn);
  }
}

// Closed-form d(F_vis.n)/dq (row-major M x MD, column c'*D + d).  The viscous
// flux of visc_fn is linear in q, F_vis = L(u) q; L's columns follow from
// the responses of the flux to unit velocity-gradient and energy-gradient
// entries (gv = (q_m - v q_rho)/rho, gE = (q_E - E q_rho)/rho):
//   q_{1+k,d}: (1/rho) R(gv[k][d]),   q_{D+1,d}: (1/rho) R(gE[d]),
//   q_{0,d}:   -(sum_k v_k col(q_{1+k,d}) + E col(q_{D+1,d})).
template <int D, int PH>
__device__ __forceinline__ void visc_dq(const double* u, const double* n, const PhysParams& pp, double* L,
                                        bool& ok) {
  constexpr int M = PH == PH_POISSON ? 1 : D + 2, MD = M * D;
#pragma unroll
  for (int i = 0; i < M * MD; ++i) L[i] = 0.0;
  if (PH == PH_POISSON) {
#pragma unroll
    for (int d = 0; d < D; ++d) L[d] = -n[d];
    return;
  }
  const double rho = u[0];
  ok = ok && (rho > 0.0);
  const double irho = 1.0 / rho;
  double v[D], vn = 0.0;
#pragma unroll
  for (int i = 0; i < D; ++i) {
    v[i] = u[1 + i] * irho;
    vn += v[i] * n[i];
  }
  const double E = u[D + 1] * irho;
  const double mu = pp.mu, kap = pp.kap, c23 = 2.0 / 3.0;
#pragma unroll
  for (int k = 0; k < D; ++k)
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const int col = (1 + k) * D + d;
#pragma unroll
      for (int i = 0; i < D; ++i) {
        const double t = (i == k ? n[d] : 0.0) + (i == d ? n[k] : 0.0) - (k == d ? c23 * n[i] : 0.0);
        L[(1 + i) * MD + col] = -irho * (mu * t);
      }
      const double en = mu * (v[k] * n[d] + v[d] * n[k]) - (k == d ? c23 * mu * vn : 0.0);
      L[(D + 1) * MD + col] = irho * (kap * v[k] * n[d] - en);
    }
#pragma unroll
  for (int d = 0; d < D; ++d) L[(D + 1) * MD + (D + 1) * D + d] = -irho * kap * n[d];
#pragma unroll
  for (int c = 1; c < M; ++c)
#pragma unroll
    for (int d = 0; d < D; ++d) {
      double s = E * L[c * MD + (D + 1) * D + d];
#pragma unroll
      for (int k = 0; k < D; ++k) s += v[k] * L[c * MD + (1 + k) * D + d];
      L[c * MD + d] = -s;
    }
}

// Closed-form d(F_vis.n)/du at fixed q (row-major M x M), Navier-Stokes.
// visc_fn is linear in the velocity / energy gradients
//   gv[i][d] = (q_{1+i,d} - v_i q_{0,d}) / rho,  gE[d] = (q_{D+1,d} - E q_{0,d}) / rho,
// with T_i(G) = mu sum_j (G_ij + G_ji) n_j - 2/3 mu tr(G) n_i:
//   F[1+i] = -T_i(gv),  F[D+1] = -(sum_i v_i T_i(gv) + kap sum_j (gE_j - sum_i v_i gv_ij) n_j),
// so column c follows from (dv, dG, dgE) = d(v, gv, gE)/du_c:
//   rho:  dv_i = -v_i/rho, dG_ij = (v_i q_0j/rho - gv_ij)/rho, dgE_j = (E q_0j/rho - gE_j)/rho
//   m_k:  dv_i = delta_ik/rho, dG_ij = -delta_ik q_0j/rho^2, dgE = 0
//   e:    dv = 0, dG = 0, dgE_j = -q_0j/rho^2.
// Poisson: F_vis does not depend on u (zero).
template <int D, int PH>
__device__ __forceinline__ void visc_du(const double* u, const double* q, const double* n, const PhysParams& pp,
                                        double* J, bool& ok) {
  constexpr int M = PH == PH_POISSON ? 1 : D + 2;
#pragma unroll
  for (int i = 0; i < M * M; ++i) J[i] = 0.0;
  if (PH == PH_POISSON) return;
  const double rho = u[0];
  ok = ok && (rho > 0.0);
  const double irho = 1.0 / rho;
  double v[D];
#pragma unroll
  for (int i = 0; i < D; ++i) v[i] = u[1 + i] * irho;
  const double E = u[D + 1] * irho;
  double gv[D][D], gE[D];
#pragma unroll
  for (int d = 0; d < D; ++d) {
#pragma unroll
    for (int i = 0; i < D; ++i) gv[i][d] = (q[(1 + i) * D + d] - v[i] * q[d]) * irho;
    gE[d] = (q[(D + 1) * D + d] - E * q[d]) * irho;
  }
  const double mu = pp.mu, kap = pp.kap, c23 = 2.0 / 3.0;
  auto T = [&](const double (&G)[D][D], double* t) {
    double tr = G[0][0];
#pragma unroll
    for (int k = 1; k < D; ++k) tr += G[k][k];
#pragma unroll
    for (int i = 0; i < D; ++i) {
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < D; ++j) s += mu * (G[i][j] + G[j][i]) * n[j];
      t[i] = s - c23 * mu * tr * n[i];
    }
  };
  double tn[D];
  T(gv, tn);
  const double ir2 = irho * irho;
#pragma unroll
  for (int c = 0; c < M; ++c) {
    double dv[D], dG[D][D], dgE[D];
#pragma unroll
    for (int i = 0; i < D; ++i) {
      dv[i] = c == 0 ? -v[i] * irho : (c == 1 + i ? irho : 0.0);
#pragma unroll
      for (int j = 0; j < D; ++j)
        dG[i][j] = c == 0 ? (v[i] * q[j] * irho - gv[i][j]) * irho : (c == 1 + i ? -q[j] * ir2 : 0.0);
    }
#pragma unroll
    for (int j = 0; j < D; ++j) dgE[j] = c == 0 ? (E * q[j] * irho - gE[j]) * irho : (c == D + 1 ? -q[j] * ir2 : 0.0);
    double dtn[D];
    T(dG, dtn);
    double den = 0.0, dhn = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) {
      J[(1 + i) * M + c] = -dtn[i];
      den += dv[i] * tn[i] + v[i] * dtn[i];
    }
#pragma unroll
    for (int j = 0; j < D; ++j) {
      double s = dgE[j];
#pragma unroll
      for (int i = 0; i < D; ++i) s -= dv[i] * gv[i][j] + v[i] * dG[i][j];
      dhn += s * n[j];
    }
    J[(D + 1) * M + c] = -(den + kap * dhn);
  }
}

}  // namespace ldg
