// linedg_host.cpp -- setup restatement (see linedg_host.hpp for the map to
// the reference sources).  No Eigen: small dense operations are written out.
#include <fstream>
#include <istream>
#include <ostream>

#include "linedg_host.hpp"

#include <algorithm>
#include <map>
#include <cmath>
#include <numeric>
#include <unordered_map>

namespace ldgh {

// =================================================================== basis

namespace {

// P_n(x) and P_n'(x) by the three-term recurrence (basis.cpp:11-25).
void legendre_pair(int n, double x, double& pn, double& dpn) {
  if (n == 0) {
    pn = 1.0;
    dpn = 0.0;
    return;
  }
  double prev = 1.0, cur = x;
  for (int k = 2; k <= n; ++k) {
    const double nxt = ((2 * k - 1) * x * cur - (k - 1) * prev) / k;
    prev = cur;
    cur = nxt;
  }
  pn = cur;
  dpn = n * (x * cur - prev) / (x * x - 1.0);
}

// Interior GLL node: Newton on P_p' with P_p'' from the Legendre ODE
// (basis.cpp:27-40).
double gll_root(int p, double x) {
  for (int it = 0; it < 100; ++it) {
    double pn, dpn;
    legendre_pair(p, x, pn, dpn);
    const double d2 = (2.0 * x * dpn - p * (p + 1) * pn) / (1.0 - x * x);
    const double step = dpn / d2;
    x -= step;
    if (std::abs(step) < 1e-15) break;
  }
  return x;
}

// Mirror symmetry about 1/2, bitwise (basis.cpp:42-52).
void symmetrize_unit(std::vector<double>& v) {
  const int n = static_cast<int>(v.size());
  for (int lo = 0, hi = n - 1; lo < hi; ++lo, --hi) {
    const double a = 0.5 * (v[lo] + (1.0 - v[hi]));
    v[lo] = a;
    v[hi] = 1.0 - a;
  }
  if (n % 2 == 1) v[n / 2] = 0.5;
}

// In-place lower Cholesky of an SPD n x n matrix; false if not SPD.
bool cholesky_lower(std::vector<double>& a, int n) {
  for (int k = 0; k < n; ++k) {
    double d = a[k * n + k];
    for (int j = 0; j < k; ++j) d -= a[k * n + j] * a[k * n + j];
    if (!(d > 0.0)) return false;
    d = std::sqrt(d);
    a[k * n + k] = d;
    for (int i = k + 1; i < n; ++i) {
      double s = a[i * n + k];
      for (int j = 0; j < k; ++j) s -= a[i * n + j] * a[k * n + j];
      a[i * n + k] = s / d;
    }
  }
  return true;
}

}  // namespace

void gauss_legendre(int n, std::vector<double>& x, std::vector<double>& w) {
  if (n < 1) throw std::invalid_argument("gauss_legendre: need n >= 1");
  x.assign(n, 0.0);
  w.assign(n, 0.0);
  for (int k = 0; k < (n + 1) / 2; ++k) {
    double z = std::cos(M_PI * (k + 0.75) / (n + 0.5));  // Chebyshev-type guess
    double pn = 0.0, dpn = 1.0;
    for (int it = 0; it < 100; ++it) {
      legendre_pair(n, z, pn, dpn);
      const double dz = pn / dpn;
      z -= dz;
      if (std::abs(dz) < 1e-15) break;
    }
    legendre_pair(n, z, pn, dpn);
    x[n - 1 - k] = 0.5 * (1.0 + z);  // roots come largest-first
    x[k] = 0.5 * (1.0 - z);
    const double wk = 1.0 / ((1.0 - z * z) * dpn * dpn);  // weights on [0,1]
    w[k] = wk;
    w[n - 1 - k] = wk;
  }
  symmetrize_unit(x);
}

std::vector<double> Basis1D::eval_phi(const std::vector<double>& pts) const {
  const int n = np(), k = static_cast<int>(pts.size());
  std::vector<double> out(static_cast<size_t>(n) * k, 0.0);
  for (int c = 0; c < k; ++c) {
    const double x = pts[c];
    int hit = -1;
    for (int i = 0; i < n; ++i)
      if (std::abs(x - nodes[i]) < 1e-14) hit = i;
    if (hit >= 0) {
      out[hit * k + c] = 1.0;
      continue;
    }
    double den = 0.0;
    for (int i = 0; i < n; ++i) den += bary[i] / (x - nodes[i]);
    for (int i = 0; i < n; ++i) out[i * k + c] = (bary[i] / (x - nodes[i])) / den;
  }
  return out;
}

std::vector<double> Basis1D::eval_dphi(const std::vector<double>& pts) const {
  const int n = np(), k = static_cast<int>(pts.size());
  const std::vector<double> ph = eval_phi(pts);
  std::vector<double> out(static_cast<size_t>(n) * k, 0.0);
  for (int c = 0; c < k; ++c) {
    const double x = pts[c];
    int hit = -1;
    for (int i = 0; i < n; ++i)
      if (std::abs(x - nodes[i]) < 1e-14) hit = i;
    if (hit >= 0) {  // differentiation-matrix row at node s_hit
      double acc = 0.0;
      for (int i = 0; i < n; ++i) {
        if (i == hit) continue;
        const double v = (bary[i] / bary[hit]) / (nodes[hit] - nodes[i]);
        out[i * k + c] = v;
        acc += v;
      }
      out[hit * k + c] = -acc;
      continue;
    }
    for (int i = 0; i < n; ++i) {
      double s = 0.0;
      for (int j = 0; j < n; ++j)
        if (j != i) s += 1.0 / (x - nodes[j]);
      out[i * k + c] = ph[i * k + c] * s;
    }
  }
  return out;
}

Basis1D make_basis(int p, bool gll) {
  if (p < 1) throw std::invalid_argument("make_basis: need p >= 1");
  Basis1D b;
  b.p = p;
  b.gll = gll;
  const int n = p + 1;
  b.nodes.assign(n, 0.0);
  if (!gll) {
    for (int i = 0; i <= p; ++i) b.nodes[i] = static_cast<double>(i) / p;
  } else {
    b.nodes[0] = 0.0;
    b.nodes[p] = 1.0;
    for (int k = 1; k < p; ++k) {
      const double z = gll_root(p, std::cos(M_PI * k / p));
      b.nodes[p - k] = 0.5 * (1.0 + z);
    }
  }
  symmetrize_unit(b.nodes);
  for (int i = 0; i < p; ++i)
    if (!(b.nodes[i + 1] > b.nodes[i]))
      throw std::runtime_error("make_basis: nodes not strictly increasing");

  b.bary.assign(n, 0.0);
  for (int i = 0; i < n; ++i) {
    double w = 1.0;
    for (int j = 0; j < n; ++j)
      if (j != i) w /= (b.nodes[i] - b.nodes[j]);
    b.bary[i] = w;
  }

  gauss_legendre((3 * p + 2) / 2, b.qp, b.qw);  // ceil((3p+1)/2) points (basis.cpp:176)
  const int nq = b.nq();
  b.phi = b.eval_phi(b.qp);
  b.dphi = b.eval_dphi(b.qp);
  const std::vector<double> dn = b.eval_dphi(b.nodes);  // [i][j] = phi_i'(s_j)
  b.diff.assign(static_cast<size_t>(n) * n, 0.0);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) b.diff[j * n + i] = dn[i * n + j];

  std::vector<double> m(static_cast<size_t>(n) * n, 0.0);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double s = 0.0;
      for (int q = 0; q < nq; ++q) s += (b.phi[i * nq + q] * b.qw[q]) * b.phi[j * nq + q];
      m[i * n + j] = s;
    }
  b.mass.assign(static_cast<size_t>(n) * n, 0.0);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) b.mass[i * n + j] = 0.5 * (m[i * n + j] + m[j * n + i]);
  std::vector<double> l = b.mass;
  if (!cholesky_lower(l, n)) throw std::runtime_error("make_basis: mass matrix not SPD");

  b.node_w.assign(n, 0.0);
  for (int i = 0; i < n; ++i) {
    double s = 0.0;
    for (int q = 0; q < nq; ++q) s += b.phi[i * nq + q] * b.qw[q];
    b.node_w[i] = s;
  }
  return b;
}

// ==================================================================== mesh

int face_direction(int dim, int lf) { return dim == 2 ? ((lf % 2 == 1) ? 0 : 1) : lf / 2; }
int face_is_plus(int dim, int lf) { return dim == 2 ? ((lf == 1 || lf == 2) ? 1 : 0) : lf % 2; }
int face_of(int dim, int dir, int side) {
  if (dim == 2) return dir == 0 ? (side ? 1 : 3) : (side ? 2 : 0);
  return 2 * dir + side;
}

namespace {

// 3-D: local vertex (bits a,b,c) of the corner (ca,cb) of face lf, where the
// face parameters run along the two transverse axes in increasing order.
int hex_face_corner(int lf, int ca, int cb) {
  const int dir = lf / 2, side = lf % 2;
  const int ax1 = dir == 0 ? 1 : 0, ax2 = dir == 2 ? 1 : 2;
  return (side << dir) | (ca << ax1) | (cb << ax2);
}

// Dihedral code o applied to corner parameters in {0,1}.
void dihedral_apply(int o, int a, int b, int pmax, int& ao, int& bo) {
  int x = a, y = b;
  if (o & 1) std::swap(x, y);
  ao = (o & 2) ? pmax - x : x;
  bo = (o & 4) ? pmax - y : y;
}

void check_quad_ccw(const Mesh& m, int e) {
  const int* q = &m.elems[4 * e];
  for (int c = 0; c < 4; ++c) {
    const double* v0 = &m.verts[2 * q[c]];
    const double* v1 = &m.verts[2 * q[(c + 1) % 4]];
    const double* v3 = &m.verts[2 * q[(c + 3) % 4]];
    const double ax = v1[0] - v0[0], ay = v1[1] - v0[1];
    const double bx = v3[0] - v0[0], by = v3[1] - v0[1];
    if (ax * by - ay * bx <= 0.0)
      throw config_error("mesh: element " + std::to_string(e) +
                         " is not counter-clockwise (corner " + std::to_string(c) + ")");
  }
}

void check_hex_positive(const Mesh& m, int e) {
  const int* h = &m.elems[8 * e];
  for (int c = 0; c < 8; ++c) {
    double ed[3][3];
    for (int d = 0; d < 3; ++d) {
      const int nb = c ^ (1 << d);
      const double sgn = (c >> d) & 1 ? -1.0 : 1.0;
      for (int k = 0; k < 3; ++k) ed[d][k] = sgn * (m.verts[3 * h[nb] + k] - m.verts[3 * h[c] + k]);
    }
    const double det = ed[0][0] * (ed[1][1] * ed[2][2] - ed[1][2] * ed[2][1]) -
                       ed[0][1] * (ed[1][0] * ed[2][2] - ed[1][2] * ed[2][0]) +
                       ed[0][2] * (ed[1][0] * ed[2][1] - ed[1][1] * ed[2][0]);
    if (!(det > 0.0))
      throw config_error("mesh: hexahedron " + std::to_string(e) + " is inverted at corner " +
                         std::to_string(c));
  }
}

void rebuild_elem_face(Mesh& m) {
  m.elem_face.assign(static_cast<size_t>(m.ne()) * m.fpe(), -1);
  for (int i = 0; i < m.nf(); ++i) {
    const Face& f = m.faces[i];
    m.elem_face[f.elem_l * m.fpe() + f.face_l] = i;
    if (!f.boundary()) m.elem_face[f.elem_r * m.fpe() + f.face_r] = i;
  }
}

// Global vertex of a 3-D face corner.
int hex_corner_vertex(const Mesh& m, int e, int lf, int ca, int cb) {
  return m.elems[8 * e + hex_face_corner(lf, ca, cb)];
}

}  // namespace

void build_faces(Mesh& m) {
  m.faces.clear();
  const int ne = m.ne();
  if (m.dim == 2) {
    for (int e = 0; e < ne; ++e) check_quad_ccw(m, e);
    // (sorted edge key, element, local face, first vertex), grouped by key in
    // key order and in (element, face) order within a key -- the iteration
    // order of the reference's std::map of vectors (mesh.cpp:76-85).
    struct Occ {
      int lo, hi, elem, lf, va;
    };
    std::vector<Occ> occ;
    occ.reserve(4 * static_cast<size_t>(ne));
    for (int e = 0; e < ne; ++e)
      for (int f = 0; f < 4; ++f) {
        const int va = m.elems[4 * e + f], vb = m.elems[4 * e + (f + 1) % 4];
        occ.push_back({std::min(va, vb), std::max(va, vb), e, f, va});
      }
    std::stable_sort(occ.begin(), occ.end(), [](const Occ& a, const Occ& b) {
      return a.lo != b.lo ? a.lo < b.lo : a.hi < b.hi;
    });
    for (size_t i = 0; i < occ.size();) {
      size_t j = i;
      while (j < occ.size() && occ[j].lo == occ[i].lo && occ[j].hi == occ[i].hi) ++j;
      const size_t cnt = j - i;
      if (cnt > 2)
        throw config_error("mesh: edge (" + std::to_string(occ[i].lo) + "," +
                           std::to_string(occ[i].hi) + ") shared by " + std::to_string(cnt) +
                           " elements (non-conforming)");
      Face face;
      if (cnt == 1) {
        face.elem_l = occ[i].elem;
        face.face_l = occ[i].lf;
        face.tag = 0;
        face.orient = 1;
      } else {
        const Occ& a = occ[i].elem <= occ[i + 1].elem ? occ[i] : occ[i + 1];
        const Occ& b = occ[i].elem <= occ[i + 1].elem ? occ[i + 1] : occ[i];
        if (a.va == b.va)
          throw config_error("mesh: elements " + std::to_string(a.elem) + " and " +
                             std::to_string(b.elem) +
                             " traverse a shared edge in the same direction");
        face.elem_l = a.elem;
        face.face_l = a.lf;
        face.elem_r = b.elem;
        face.face_r = b.lf;
        face.orient = 1;
      }
      m.faces.push_back(face);
      i = j;
    }
  } else {
    for (int e = 0; e < ne; ++e) check_hex_positive(m, e);
    struct Occ {
      std::array<int, 4> key;
      int elem, lf;
    };
    std::vector<Occ> occ;
    occ.reserve(6 * static_cast<size_t>(ne));
    for (int e = 0; e < ne; ++e)
      for (int f = 0; f < 6; ++f) {
        Occ o;
        o.elem = e;
        o.lf = f;
        for (int c = 0; c < 4; ++c) o.key[c] = hex_corner_vertex(m, e, f, c & 1, c >> 1);
        std::sort(o.key.begin(), o.key.end());
        occ.push_back(o);
      }
    std::stable_sort(occ.begin(), occ.end(),
                     [](const Occ& a, const Occ& b) { return a.key < b.key; });
    for (size_t i = 0; i < occ.size();) {
      size_t j = i;
      while (j < occ.size() && occ[j].key == occ[i].key) ++j;
      const size_t cnt = j - i;
      if (cnt > 2)
        throw config_error("mesh: face shared by " + std::to_string(cnt) +
                           " hexahedra (non-conforming)");
      Face face;
      if (cnt == 1) {
        face.elem_l = occ[i].elem;
        face.face_l = occ[i].lf;
        face.tag = 0;
        face.orient = 0;
      } else {
        const Occ& a = occ[i].elem <= occ[i + 1].elem ? occ[i] : occ[i + 1];
        const Occ& b = occ[i].elem <= occ[i + 1].elem ? occ[i + 1] : occ[i];
        int code = -1;
        for (int o = 0; o < 8 && code < 0; ++o) {
          bool ok = true;
          for (int c = 0; c < 4 && ok; ++c) {
            int ra, rb;
            dihedral_apply(o, c & 1, c >> 1, 1, ra, rb);
            ok = hex_corner_vertex(m, a.elem, a.lf, c & 1, c >> 1) ==
                 hex_corner_vertex(m, b.elem, b.lf, ra, rb);
          }
          if (ok) code = o;
        }
        if (code < 0) throw config_error("mesh: inconsistent shared hexahedron face");
        face.elem_l = a.elem;
        face.face_l = a.lf;
        face.elem_r = b.elem;
        face.face_r = b.lf;
        face.orient = code;
      }
      m.faces.push_back(face);
      i = j;
    }
  }
  rebuild_elem_face(m);
}

void make_periodic(Mesh& m, int tag_a, int tag_b, const double* tr) {
  const int D = m.dim;
  std::vector<int> fa, fb;
  for (int i = 0; i < m.nf(); ++i) {
    if (!m.faces[i].boundary()) continue;
    if (m.faces[i].tag == tag_a) fa.push_back(i);
    if (m.faces[i].tag == tag_b) fb.push_back(i);
  }
  if (fa.size() != fb.size())
    throw config_error("make_periodic: tag " + std::to_string(tag_a) + " has " +
                       std::to_string(fa.size()) + " faces but tag " + std::to_string(tag_b) +
                       " has " + std::to_string(fb.size()));
  auto vx = [&](int v, int k) { return m.verts[D * v + k]; };
  double tnorm = 0.0;
  for (int k = 0; k < D; ++k) tnorm += tr[k] * tr[k];
  tnorm = std::sqrt(tnorm);

  std::vector<Face> merged;
  merged.reserve(fa.size());
  if (D == 2) {
    // Direct restatement of mesh.cpp:228-277 (O(n_a n_b) pairing).
    auto ends = [&](int fid, int& va, int& vb) {
      const Face& f = m.faces[fid];
      va = m.elems[4 * f.elem_l + f.face_l];
      vb = m.elems[4 * f.elem_l + (f.face_l + 1) % 4];
    };
    double h = 0.0;
    for (int fid : fa) {
      int a0, a1;
      ends(fid, a0, a1);
      const double dx = vx(a1, 0) - vx(a0, 0), dy = vx(a1, 1) - vx(a0, 1);
      h = std::max(h, std::sqrt(dx * dx + dy * dy));
    }
    const double tol = 1e-8 * std::max(h, tnorm);
    auto close = [&](double x0, double y0, int v) {
      const double dx = x0 - vx(v, 0), dy = y0 - vx(v, 1);
      return std::sqrt(dx * dx + dy * dy) < tol;
    };
    std::vector<char> used(fb.size(), 0);
    for (size_t ia = 0; ia < fa.size(); ++ia) {
      int a0, a1;
      ends(fa[ia], a0, a1);
      const double t0x = vx(a0, 0) + tr[0], t0y = vx(a0, 1) + tr[1];
      const double t1x = vx(a1, 0) + tr[0], t1y = vx(a1, 1) + tr[1];
      int match = -1, rev = 1;
      for (size_t ib = 0; ib < fb.size(); ++ib) {
        if (used[ib]) continue;
        int b0, b1;
        ends(fb[ib], b0, b1);
        if (close(t0x, t0y, b1) && close(t1x, t1y, b0)) {
          match = static_cast<int>(ib);
          rev = 1;
          break;
        }
        if (close(t0x, t0y, b0) && close(t1x, t1y, b1)) {
          match = static_cast<int>(ib);
          rev = 0;
          break;
        }
      }
      if (match < 0) throw config_error("make_periodic: no partner for face " + std::to_string(fa[ia]));
      used[match] = 1;
      const Face& A = m.faces[fa[ia]];
      const Face& B = m.faces[fb[match]];
      Face f;
      f.elem_l = A.elem_l;
      f.face_l = A.face_l;
      f.elem_r = B.elem_l;
      f.face_r = B.face_l;
      f.orient = rev;
      f.tag = -1;
      merged.push_back(f);
    }
  } else {
    // 3-D: same pairing semantics (first unused partner in index order, same
    // tolerance rule), accelerated with a centroid grid hash.
    auto corner_xyz = [&](int fid, int c, double* out) {
      const Face& f = m.faces[fid];
      const int v = hex_corner_vertex(m, f.elem_l, f.face_l, c & 1, c >> 1);
      for (int k = 0; k < 3; ++k) out[k] = vx(v, k);
    };
    double h = 0.0;
    for (int fid : fa) {
      double c0[3], c3[3];
      corner_xyz(fid, 0, c0);
      corner_xyz(fid, 3, c3);
      double d2 = 0.0;
      for (int k = 0; k < 3; ++k) d2 += (c3[k] - c0[k]) * (c3[k] - c0[k]);
      h = std::max(h, std::sqrt(d2));
    }
    const double tol = 1e-8 * std::max(h, tnorm);
    const double cell = std::max(h, 1e-300);
    auto cell_key = [&](const double* c) {
      const int64_t ix = static_cast<int64_t>(std::floor(c[0] / cell));
      const int64_t iy = static_cast<int64_t>(std::floor(c[1] / cell));
      const int64_t iz = static_cast<int64_t>(std::floor(c[2] / cell));
      return (ix * 73856093) ^ (iy * 19349663) ^ (iz * 83492791);
    };
    auto centroid = [&](int fid, const double* shift, double* c) {
      c[0] = c[1] = c[2] = 0.0;
      for (int q = 0; q < 4; ++q) {
        double x[3];
        corner_xyz(fid, q, x);
        for (int k = 0; k < 3; ++k) c[k] += 0.25 * (x[k] + (shift ? shift[k] : 0.0));
      }
    };
    std::unordered_multimap<int64_t, int> grid;
    for (size_t ib = 0; ib < fb.size(); ++ib) {
      double c[3];
      centroid(fb[ib], nullptr, c);
      grid.emplace(cell_key(c), static_cast<int>(ib));
    }
    std::vector<char> used(fb.size(), 0);
    for (size_t ia = 0; ia < fa.size(); ++ia) {
      double ca[3];
      centroid(fa[ia], tr, ca);
      std::vector<int> cand;
      for (int dz = -1; dz <= 1; ++dz)
        for (int dy = -1; dy <= 1; ++dy)
          for (int dx = -1; dx <= 1; ++dx) {
            const double probe[3] = {ca[0] + dx * cell, ca[1] + dy * cell, ca[2] + dz * cell};
            auto rng = grid.equal_range(cell_key(probe));
            for (auto it = rng.first; it != rng.second; ++it) cand.push_back(it->second);
          }
      std::sort(cand.begin(), cand.end());
      cand.erase(std::unique(cand.begin(), cand.end()), cand.end());
      int match = -1, code = -1;
      for (int ib : cand) {
        if (used[ib]) continue;
        for (int o = 0; o < 8 && code < 0; ++o) {
          bool ok = true;
          for (int c = 0; c < 4 && ok; ++c) {
            int ra, rb;
            dihedral_apply(o, c & 1, c >> 1, 1, ra, rb);
            double xa[3], xb[3];
            corner_xyz(fa[ia], c, xa);
            corner_xyz(fb[ib], ra | (rb << 1), xb);
            double d2 = 0.0;
            for (int k = 0; k < 3; ++k) d2 += (xa[k] + tr[k] - xb[k]) * (xa[k] + tr[k] - xb[k]);
            ok = std::sqrt(d2) < tol;
          }
          if (ok) code = o;
        }
        if (code >= 0) {
          match = ib;
          break;
        }
      }
      if (match < 0) throw config_error("make_periodic: no partner for face " + std::to_string(fa[ia]));
      used[match] = 1;
      const Face& A = m.faces[fa[ia]];
      const Face& B = m.faces[fb[match]];
      Face f;
      f.elem_l = A.elem_l;
      f.face_l = A.face_l;
      f.elem_r = B.elem_l;
      f.face_r = B.face_l;
      f.orient = code;
      f.tag = -1;
      merged.push_back(f);
    }
  }
  // Survivors keep their order; the merged faces are appended (mesh.cpp:279-293).
  std::vector<char> drop(m.nf(), 0);
  for (int fid : fa) drop[fid] = 1;
  for (int fid : fb) drop[fid] = 1;
  std::vector<Face> faces;
  faces.reserve(m.faces.size());
  for (int i = 0; i < m.nf(); ++i)
    if (!drop[i]) faces.push_back(m.faces[i]);
  faces.insert(faces.end(), merged.begin(), merged.end());
  m.faces.swap(faces);
  rebuild_elem_face(m);
}

std::vector<int8_t> assign_switches(const Mesh& m) {
  const int D = m.dim, F = m.fpe();
  std::vector<int8_t> plus(static_cast<size_t>(m.ne()) * D, 0);
  // Walk a global line entering `elem` through `lf`, carrying the sign this
  // element holds on its entry face (mesh.cpp:296-344).  The sign is
  // invariant along the walk: the far face holds -sign on this element and
  // the neighbour holds the opposite of that.
  auto walk = [&](int elem, int lf, int sign) {
    while (elem >= 0) {
      const int dir = face_direction(D, lf);
      const int pl = face_is_plus(D, lf) ? sign : -sign;
      int8_t& slot = plus[static_cast<size_t>(elem) * D + dir];
      if (slot != 0) {
        if (slot != pl) throw std::logic_error("assign_switches: inconsistent line traversal");
        return;  // cycle closed
      }
      slot = static_cast<int8_t>(pl);
      const int far_lf = face_of(D, dir, face_is_plus(D, lf) ? 0 : 1);
      const int fid = m.elem_face[static_cast<size_t>(elem) * F + far_lf];
      if (fid < 0) return;
      const Face& nf = m.faces[fid];
      if (nf.boundary()) return;
      if (nf.elem_l == elem && nf.face_l == far_lf) {
        elem = nf.elem_r;
        lf = nf.face_r;
      } else {
        elem = nf.elem_l;
        lf = nf.face_l;
      }
    }
  };
  for (int fid = 0; fid < m.nf(); ++fid) {
    const Face& f = m.faces[fid];
    if (plus[static_cast<size_t>(f.elem_l) * D + face_direction(D, f.face_l)] != 0) continue;
    walk(f.elem_l, f.face_l, 1);
    if (!f.boundary()) walk(f.elem_r, f.face_r, -1);
  }
  for (auto& s : plus)
    if (s == 0) s = 1;  // directions no face sweep reached (mesh.cpp:346-350)
  return plus;
}

int count_switch_violations(const Mesh& m, const std::vector<int8_t>& sw) {
  const int D = m.dim;
  auto sign = [&](int e, int dir, int side) {
    const int s = sw[static_cast<size_t>(e) * D + dir];
    return side ? s : -s;
  };
  int bad = 0;
  for (int e = 0; e < m.ne(); ++e)
    for (int d = 0; d < D; ++d)
      if (sign(e, d, 0) != -sign(e, d, 1)) ++bad;
  for (const Face& f : m.faces) {
    if (f.boundary()) continue;
    const int sl = sign(f.elem_l, face_direction(D, f.face_l), face_is_plus(D, f.face_l));
    const int sr = sign(f.elem_r, face_direction(D, f.face_r), face_is_plus(D, f.face_r));
    if (sl != -sr) ++bad;
  }
  return bad;
}

// ================================================================= mapping

Mapping compute_mapping(const Mesh& m, const Basis1D& b, const CurveProjector* curve) {
  const int D = m.dim, p = b.p, n = p + 1, nq = b.nq(), ne = m.ne();
  const int npe = D == 2 ? n * n : n * n * n;
  const int NL = D == 2 ? n : n * n;
  Mapping mp;
  mp.dim = D;
  mp.p = p;
  mp.nq = nq;
  mp.ne = ne;
  mp.coords.assign(static_cast<size_t>(ne) * npe * D, 0.0);
  mp.jac.assign(static_cast<size_t>(ne) * npe, 0.0);
  mp.nvec.assign(static_cast<size_t>(ne) * D * NL * nq * D, 0.0);
  mp.nend.assign(static_cast<size_t>(ne) * D * 2 * NL * D, 0.0);
  const std::vector<double>& Dm = b.diff;  // Dm[j*n+i] = phi_i'(s_j)
  const int stride[3] = {1, n, n * n};

  std::vector<double> dx(static_cast<size_t>(D) * npe * D);  // [axis][node][k]
  for (int e = 0; e < ne; ++e) {
    double* X = &mp.coords[static_cast<size_t>(e) * npe * D];
    const int* ev = &m.elems[static_cast<size_t>(e) * m.vpe()];
    // Isoparametric placement (mapping.cpp:12-29, bilinear; trilinear in 3-D).
    if (D == 2) {
      const double* v0 = &m.verts[2 * ev[0]];
      const double* v1 = &m.verts[2 * ev[1]];
      const double* v2 = &m.verts[2 * ev[2]];
      const double* v3 = &m.verts[2 * ev[3]];
      for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) {
          const double si = b.nodes[i], sj = b.nodes[j];
          const double w0 = (1 - si) * (1 - sj), w1 = si * (1 - sj), w2 = si * sj, w3 = (1 - si) * sj;
          for (int k = 0; k < 2; ++k)
            X[(i + n * j) * 2 + k] = w0 * v0[k] + w1 * v1[k] + w2 * v2[k] + w3 * v3[k];
        }
      // Curved boundary (mapping.cpp:30-65): project the nodes of every
      // boundary face, in local-face order, and blend each face's
      // displacement linearly into the interior (weight 1 on the face, 0 on
      // the opposite one).  Faces are processed in sequence on the updated
      // positions, so a corner moved by face lf is re-projected by face lf+1.
      if (curve && curve->fn) {
        for (int lf = 0; lf < 4; ++lf) {
          const Face& f = m.faces[m.elem_face[4 * e + lf]];
          if (!f.boundary()) continue;
          std::vector<double> delta(2 * n);
          bool moved = false;
          for (int k = 0; k < n; ++k) {
            int i = 0, j = 0;  // face node k in face-parameter order (mesh.cpp:51-63)
            switch (lf) {
              case 0: i = k; j = 0; break;
              case 1: i = p; j = k; break;
              case 2: i = p - k; j = p; break;
              default: i = 0; j = p - k; break;
            }
            const double* x0 = &X[(i + n * j) * 2];
            double xp[2];
            curve->fn(curve->user, x0, f.tag, xp);
            delta[2 * k] = xp[0] - x0[0];
            delta[2 * k + 1] = xp[1] - x0[1];
            if (std::sqrt(delta[2 * k] * delta[2 * k] + delta[2 * k + 1] * delta[2 * k + 1]) > 0.0) moved = true;
          }
          if (!moved) continue;
          for (int j = 0; j < n; ++j)
            for (int i = 0; i < n; ++i) {
              const double si = b.nodes[i], sj = b.nodes[j];
              double blend;
              int k;
              switch (lf) {
                case 0: blend = 1 - sj; k = i; break;
                case 1: blend = si; k = j; break;
                case 2: blend = sj; k = p - i; break;
                default: blend = 1 - si; k = p - j; break;
              }
              X[(i + n * j) * 2] += blend * delta[2 * k];
              X[(i + n * j) * 2 + 1] += blend * delta[2 * k + 1];
            }
        }
      }
    } else {
      for (int kk = 0; kk < n; ++kk)
        for (int j = 0; j < n; ++j)
          for (int i = 0; i < n; ++i) {
            const double s[3] = {b.nodes[i], b.nodes[j], b.nodes[kk]};
            double acc[3] = {0, 0, 0};
            for (int c = 0; c < 8; ++c) {
              double w = 1.0;
              for (int a = 0; a < 3; ++a) w *= ((c >> a) & 1) ? s[a] : (1 - s[a]);
              for (int k = 0; k < 3; ++k) acc[k] += w * m.verts[3 * ev[c] + k];
            }
            for (int k = 0; k < 3; ++k) X[(i + n * j + n * n * kk) * 3 + k] = acc[k];
          }
    }
    // Nodal derivatives along every reference axis (mapping.cpp:82-93).
    for (int node = 0; node < npe; ++node) {
      int idx[3] = {node % n, (node / n) % n, node / (n * n)};
      for (int ax = 0; ax < D; ++ax) {
        double g[3] = {0, 0, 0};
        const int base = node - idx[ax] * stride[ax];
        for (int k = 0; k < n; ++k) {
          const double c = Dm[idx[ax] * n + k];
          for (int q = 0; q < D; ++q) g[q] += c * X[(base + k * stride[ax]) * D + q];
        }
        for (int q = 0; q < D; ++q) dx[(static_cast<size_t>(ax) * npe + node) * D + q] = g[q];
      }
    }
    auto dxv = [&](int ax, int node) { return &dx[(static_cast<size_t>(ax) * npe + node) * D]; };
    // Jacobian determinant at nodes (mapping.cpp:95-102).
    for (int node = 0; node < npe; ++node) {
      double jac;
      if (D == 2) {
        const double* a = dxv(0, node);
        const double* c = dxv(1, node);
        jac = a[0] * c[1] - c[0] * a[1];
      } else {
        const double* g0 = dxv(0, node);
        const double* g1 = dxv(1, node);
        const double* g2 = dxv(2, node);
        jac = g0[0] * (g1[1] * g2[2] - g1[2] * g2[1]) - g0[1] * (g1[0] * g2[2] - g1[2] * g2[0]) +
              g0[2] * (g1[0] * g2[1] - g1[1] * g2[0]);
      }
      if (!(jac > 0.0))
        throw config_error("mapping: element " + std::to_string(e) + " is inverted (J <= 0 at node " +
                           std::to_string(node) + ")");
      mp.jac[static_cast<size_t>(e) * npe + node] = jac;
    }
    // Line tables (mapping.cpp:104-149): adjugate row `dir` at every line
    // quadrature point and the non-normalised endpoint normals.
    for (int dir = 0; dir < D; ++dir) {
      const int ta = (dir + 1) % D, tb = (dir + 2) % D;  // 3-D cyclic transverse axes
      const int t1 = dir == 0 ? 1 : 0, t2 = dir == 2 ? 1 : 2;  // 3-D line-index axes
      for (int line = 0; line < NL; ++line) {
        int base;
        if (D == 2) base = dir == 0 ? n * line : line;
        else base = (line % n) * stride[t1] + (line / n) * stride[t2];
        auto node_t = [&](int t) { return base + t * stride[dir]; };
        double* nv_out = &mp.nvec[((((static_cast<size_t>(e) * D + dir) * NL + line) * nq)) * D];
        for (int q = 0; q < nq; ++q) {
          double along[3] = {0, 0, 0}, tra[3] = {0, 0, 0}, trb[3] = {0, 0, 0};
          for (int t = 0; t < n; ++t) {
            const int nd = node_t(t);
            const double dph = b.dphi[t * nq + q], ph = b.phi[t * nq + q];
            for (int k = 0; k < D; ++k) along[k] += dph * X[nd * D + k];
            if (D == 2) {
              const double* bt = dxv(dir == 0 ? 1 : 0, nd);
              for (int k = 0; k < 2; ++k) tra[k] += ph * bt[k];
            } else {
              const double* ba = dxv(ta, nd);
              const double* bb = dxv(tb, nd);
              for (int k = 0; k < 3; ++k) {
                tra[k] += ph * ba[k];
                trb[k] += ph * bb[k];
              }
            }
          }
          double nv[3], jac;
          if (D == 2) {
            if (dir == 0) {
              nv[0] = tra[1];
              nv[1] = -tra[0];
              jac = along[0] * tra[1] - tra[0] * along[1];
            } else {
              nv[0] = -tra[1];
              nv[1] = tra[0];
              jac = tra[0] * along[1] - along[0] * tra[1];
            }
          } else {
            nv[0] = tra[1] * trb[2] - tra[2] * trb[1];
            nv[1] = tra[2] * trb[0] - tra[0] * trb[2];
            nv[2] = tra[0] * trb[1] - tra[1] * trb[0];
            jac = along[0] * nv[0] + along[1] * nv[1] + along[2] * nv[2];
          }
          if (!(jac > 0.0))
            throw config_error("mapping: element " + std::to_string(e) +
                               " is inverted (J <= 0 at a quadrature point)");
          for (int k = 0; k < D; ++k) nv_out[q * D + k] = nv[k];
        }
        for (int side = 0; side < 2; ++side) {
          const int nd = node_t(side ? p : 0);
          double* ne_out =
              &mp.nend[((((static_cast<size_t>(e) * D + dir) * 2 + side) * NL + line)) * D];
          if (D == 2) {
            const double* bt = dxv(dir == 0 ? 1 : 0, nd);
            const double sx = bt[0], sy = bt[1];
            if (dir == 0) {
              ne_out[0] = side ? sy : -sy;
              ne_out[1] = side ? -sx : sx;
            } else {
              ne_out[0] = side ? -sy : sy;
              ne_out[1] = side ? sx : -sx;
            }
          } else {
            const double* ba = dxv(ta, nd);
            const double* bb = dxv(tb, nd);
            const double c[3] = {ba[1] * bb[2] - ba[2] * bb[1], ba[2] * bb[0] - ba[0] * bb[2],
                                 ba[0] * bb[1] - ba[1] * bb[0]};
            for (int k = 0; k < 3; ++k) ne_out[k] = side ? c[k] : -c[k];
          }
        }
      }
    }
  }
  return mp;
}

// ===================================================================== RNG

uint64_t Rng::next() {
  uint64_t z = (s += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
double Rng::uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
double Rng::uniform(double a, double b) { return a + (b - a) * uniform(); }
double Rng::normal() {
  double u1 = uniform();
  while (u1 <= 0.0) u1 = uniform();
  const double u2 = uniform();
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
}

// ============================================================== generators

namespace {

// The 24 proper rotations of the reference cube as vertex permutations:
// new local vertex c takes the old vertex perm[c].
std::vector<std::array<int, 8>> cube_rotations() {
  std::vector<std::array<int, 8>> out;
  int ax[3] = {0, 1, 2};
  do {
    for (int sg = 0; sg < 8; ++sg) {
      // signed permutation matrix R: (R x)_i = s_i x_{ax[i]}
      int par = 0;  // permutation parity
      for (int i = 0; i < 3; ++i)
        for (int j = i + 1; j < 3; ++j)
          if (ax[i] > ax[j]) ++par;
      int neg = ((sg & 1) + ((sg >> 1) & 1) + ((sg >> 2) & 1));
      if ((par + neg) % 2 != 0) continue;  // det = -1
      std::array<int, 8> perm{};
      for (int c = 0; c < 8; ++c) {
        int bits[3] = {c & 1, (c >> 1) & 1, (c >> 2) & 1};
        int nb[3];
        for (int i = 0; i < 3; ++i) {
          const int b = bits[ax[i]];
          nb[i] = ((sg >> i) & 1) ? 1 - b : b;
        }
        perm[c] = nb[0] | (nb[1] << 1) | (nb[2] << 2);
      }
      out.push_back(perm);
    }
  } while (std::next_permutation(ax, ax + 3));
  return out;
}

}  // namespace

Mesh make_lattice_mesh(const LatticeSpec& s, std::vector<int>* tag_lines) {
  const int D = s.dim, n = s.n, nv1 = n + 1;
  if (D != 2 && D != 3) throw config_error("lattice: dim must be 2 or 3");
  if (n < 1) throw config_error("lattice: n must be >= 1");
  if (s.periodic && n < 2) throw config_error("lattice: periodic meshes need n >= 2");
  Mesh m;
  m.dim = D;
  const int nverts = D == 2 ? nv1 * nv1 : nv1 * nv1 * nv1;
  m.verts.assign(static_cast<size_t>(nverts) * D, 0.0);
  std::vector<std::array<int, 3>> lat(nverts);
  // Jitter draws: D uniforms per lattice vertex in index order (x fastest).
  std::vector<double> draw(static_cast<size_t>(nverts) * D);
  {
    Rng rng(s.seed_jitter);
    for (auto& d : draw) d = rng.uniform(-1.0, 1.0);
  }
  auto vid = [&](int i, int j, int k) { return D == 2 ? i + nv1 * j : i + nv1 * (j + nv1 * k); };
  const int kmax = D == 2 ? 1 : nv1;
  for (int k = 0; k < kmax; ++k)
    for (int j = 0; j < nv1; ++j)
      for (int i = 0; i < nv1; ++i) {
        const int v = vid(i, j, k);
        lat[v] = {i, j, k};
        const int idx[3] = {i, j, k};
        bool bdry = false;
        for (int a = 0; a < D; ++a) bdry = bdry || idx[a] == 0 || idx[a] == n;
        int src = v;
        if (s.periodic) src = vid(i % n, j % n, D == 2 ? 0 : k % n);
        const bool move = s.jitter != 0.0 && (s.periodic || s.jitter_boundary || !bdry);
        for (int a = 0; a < D; ++a) {
          const double h = s.length[a] / n;
          double x = idx[a] * h;
          if (move) x += s.jitter * h * draw[static_cast<size_t>(src) * D + a];
          m.verts[static_cast<size_t>(v) * D + a] = x;
        }
      }
  // Elements in lattice order, CCW (2-D) / v(a,b,c)=a+2b+4c (3-D).
  const int ne = D == 2 ? n * n : n * n * n;
  const int vpe = 1 << D;
  std::vector<int> el(static_cast<size_t>(ne) * vpe);
  {
    int e = 0;
    for (int k = 0; k < (D == 2 ? 1 : n); ++k)
      for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i, ++e) {
          int* q = &el[static_cast<size_t>(e) * vpe];
          if (D == 2) {
            q[0] = vid(i, j, 0);
            q[1] = vid(i + 1, j, 0);
            q[2] = vid(i + 1, j + 1, 0);
            q[3] = vid(i, j + 1, 0);
          } else {
            for (int c = 0; c < 8; ++c) q[c] = vid(i + (c & 1), j + ((c >> 1) & 1), k + ((c >> 2) & 1));
          }
        }
  }
  std::vector<int> order(ne);
  std::iota(order.begin(), order.end(), 0);
  if (s.permute) {
    Rng rng(s.seed_perm);
    for (int i = ne - 1; i > 0; --i) {
      const int j = static_cast<int>(rng.next() % static_cast<uint64_t>(i + 1));
      std::swap(order[i], order[j]);
    }
  }
  m.elems.assign(static_cast<size_t>(ne) * vpe, 0);
  {
    Rng rng(s.seed_rot);
    const auto rots = cube_rotations();
    for (int e = 0; e < ne; ++e) {
      const int* src = &el[static_cast<size_t>(order[e]) * vpe];
      int* dst = &m.elems[static_cast<size_t>(e) * vpe];
      if (!s.rotate) {
        std::copy(src, src + vpe, dst);
      } else if (D == 2) {
        const int r = static_cast<int>(rng.next() % 4);
        for (int c = 0; c < 4; ++c) dst[c] = src[(c + r) % 4];
      } else {
        const auto& R = rots[rng.next() % rots.size()];
        for (int c = 0; c < 8; ++c) dst[c] = src[R[c]];
      }
    }
  }
  build_faces(m);
  // Boundary tags from lattice position (emulates the tag lines of load_mesh).
  for (Face& f : m.faces) {
    if (!f.boundary()) continue;
    std::vector<int> fv;
    if (D == 2) {
      fv = {m.elems[4 * f.elem_l + f.face_l], m.elems[4 * f.elem_l + (f.face_l + 1) % 4]};
    } else {
      for (int c = 0; c < 4; ++c) fv.push_back(hex_corner_vertex(m, f.elem_l, f.face_l, c & 1, c >> 1));
    }
    int tag = 0;
    for (int a = 0; a < D && tag == 0; ++a) {
      bool lo = true, hi = true;
      for (int v : fv) {
        lo = lo && lat[v][a] == 0;
        hi = hi && lat[v][a] == n;
      }
      if (D == 2) {
        if (a == 0 && lo) tag = 4;
        if (a == 0 && hi) tag = 2;
        if (a == 1 && lo) tag = 1;
        if (a == 1 && hi) tag = 3;
      } else {
        if (lo) tag = 2 * a + 1;
        if (hi) tag = 2 * a + 2;
      }
    }
    f.tag = tag;
    if (tag_lines) {
      tag_lines->push_back(f.elem_l);
      tag_lines->push_back(f.face_l);
      tag_lines->push_back(tag);
    }
  }
  if (s.periodic) {
    if (D == 2) {
      const double tx[2] = {s.length[0], 0.0}, ty[2] = {0.0, s.length[1]};
      make_periodic(m, 4, 2, tx);
      make_periodic(m, 1, 3, ty);
    } else {
      for (int a = 0; a < 3; ++a) {
        double t[3] = {0, 0, 0};
        t[a] = s.length[a];
        make_periodic(m, 2 * a + 1, 2 * a + 2, t);
      }
    }
  }
  return m;
}

// ------------------------------------------------------------ refinement
// refine_uniform (mesh.cpp:168-213): every quad split into four at its edge
// midpoints and centroid; boundary-edge midpoints are created first (face
// order), then per element m01, m12, m23, m30 (shared through an edge map) and
// the centroid; children keep their parent edge's boundary tag.  2-D.
Mesh refine_uniform(const Mesh& mesh) {
  if (mesh.dim != 2) throw config_error("mesh: uniform refinement is 2-D only");
  Mesh out;
  out.dim = 2;
  out.verts = mesh.verts;
  std::map<std::pair<int, int>, int> edge_mid;
  auto midpoint = [&](int a, int b) {
    const auto key = std::make_pair(std::min(a, b), std::max(a, b));
    auto it = edge_mid.find(key);
    if (it != edge_mid.end()) return it->second;
    const int id = out.nv();
    for (int k = 0; k < 2; ++k) out.verts.push_back(0.5 * (mesh.verts[2 * a + k] + mesh.verts[2 * b + k]));
    edge_mid.emplace(key, id);
    return id;
  };
  std::map<std::pair<int, int>, int> child_edge_tag;
  for (const Face& f : mesh.faces) {
    if (!f.boundary()) continue;
    const int va = mesh.elems[4 * f.elem_l + f.face_l];
    const int vb = mesh.elems[4 * f.elem_l + (f.face_l + 1) % 4];
    const int m = midpoint(va, vb);
    child_edge_tag[{std::min(va, m), std::max(va, m)}] = f.tag;
    child_edge_tag[{std::min(m, vb), std::max(m, vb)}] = f.tag;
  }
  for (int e = 0; e < mesh.ne(); ++e) {
    const int* q = &mesh.elems[4 * e];
    const int m01 = midpoint(q[0], q[1]);
    const int m12 = midpoint(q[1], q[2]);
    const int m23 = midpoint(q[2], q[3]);
    const int m30 = midpoint(q[3], q[0]);
    const int c = out.nv();
    for (int k = 0; k < 2; ++k)
      out.verts.push_back(0.25 * (mesh.verts[2 * q[0] + k] + mesh.verts[2 * q[1] + k] + mesh.verts[2 * q[2] + k] +
                                  mesh.verts[2 * q[3] + k]));
    const int kids[4][4] = {{q[0], m01, c, m30}, {m01, q[1], m12, c}, {c, m12, q[2], m23}, {m30, c, m23, q[3]}};
    for (const auto& kq : kids) out.elems.insert(out.elems.end(), kq, kq + 4);
  }
  build_faces(out);
  for (Face& f : out.faces) {
    if (!f.boundary()) continue;
    const int va = out.elems[4 * f.elem_l + f.face_l];
    const int vb = out.elems[4 * f.elem_l + (f.face_l + 1) % 4];
    auto it = child_edge_tag.find({std::min(va, vb), std::max(va, vb)});
    if (it != child_edge_tag.end()) f.tag = it->second;
  }
  return out;
}

// ------------------------------------------------------------- mesh text I/O
// The reference mesh file (SPEC.md "External Interfaces"; mesh.cpp:115-166):
// `nv ne nb`, nv lines `x y`, ne lines `v0 v1 v2 v3` (0-based, CCW), nb lines
// `elem local_face tag`.  Same parse order, checks and config_error messages
// as load_mesh (mesh.cpp:115-146); faces are built before the tag lines are
// applied, every untagged boundary face keeps tag 0 (mesh.cpp:94).  2-D only,
// like the format.
Mesh load_mesh(std::istream& in) {
  Mesh mesh;
  mesh.dim = 2;
  int nv = 0, ne = 0, nb = 0;
  if (!(in >> nv >> ne >> nb)) throw config_error("mesh: failed to read header `nv ne nb`");
  if (nv < 0 || ne < 0 || nb < 0) throw config_error("mesh: failed to read header `nv ne nb`");
  mesh.verts.resize(static_cast<size_t>(nv) * 2);
  for (int i = 0; i < nv; ++i)
    if (!(in >> mesh.verts[2 * i] >> mesh.verts[2 * i + 1]))
      throw config_error("mesh: failed to read vertex " + std::to_string(i));
  mesh.elems.resize(static_cast<size_t>(ne) * 4);
  for (int e = 0; e < ne; ++e)
    for (int c = 0; c < 4; ++c) {
      int& v = mesh.elems[4 * e + c];
      if (!(in >> v)) throw config_error("mesh: failed to read element " + std::to_string(e));
      if (v < 0 || v >= nv)
        throw config_error("mesh: element " + std::to_string(e) + " has vertex index out of range");
    }
  build_faces(mesh);
  for (int b = 0; b < nb; ++b) {
    int e = 0, lf = 0, tag = 0;
    if (!(in >> e >> lf >> tag)) throw config_error("mesh: failed to read boundary tag line " + std::to_string(b));
    if (e < 0 || e >= ne || lf < 0 || lf > 3)
      throw config_error("mesh: boundary tag line " + std::to_string(b) + " out of range");
    Face& f = mesh.faces[mesh.elem_face[4 * e + lf]];
    if (!f.boundary())
      throw config_error("mesh: tagged face (" + std::to_string(e) + "," + std::to_string(lf) +
                         ") is not a boundary face");
    f.tag = tag;
  }
  return mesh;
}

Mesh load_mesh(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw config_error("mesh: cannot open '" + path + "'");
  return load_mesh(in);
}

// save_mesh (mesh.cpp:148-160): 17 significant digits, the faces still on the
// boundary (after any periodic pairing) in face order as `elem_l face_l tag`.
void save_mesh(const Mesh& mesh, std::ostream& out) {
  if (mesh.dim != 2) throw config_error("mesh: the text format is 2-D only");
  out.precision(17);
  std::vector<const Face*> bf;
  for (const Face& f : mesh.faces)
    if (f.boundary()) bf.push_back(&f);
  out << mesh.nv() << " " << mesh.ne() << " " << bf.size() << "\n";
  for (int i = 0; i < mesh.nv(); ++i) out << mesh.verts[2 * i] << " " << mesh.verts[2 * i + 1] << "\n";
  for (int e = 0; e < mesh.ne(); ++e)
    out << mesh.elems[4 * e] << " " << mesh.elems[4 * e + 1] << " " << mesh.elems[4 * e + 2] << " "
        << mesh.elems[4 * e + 3] << "\n";
  for (const Face* f : bf) out << f->elem_l << " " << f->face_l << " " << f->tag << "\n";
}

void save_mesh(const Mesh& mesh, const std::string& path) {
  std::ofstream out(path);
  if (!out) throw config_error("mesh: cannot write '" + path + "'");
  save_mesh(mesh, out);
}

}  // namespace ldgh
