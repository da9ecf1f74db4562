// linedg_host.hpp -- host-side setup for the Line-DG hot path.
//
// The reference builds its setup objects with basis.cpp, mesh.cpp and
// mapping.cpp (present in the reference tree but unbuildable here: they need
// Eigen3, proj/CMakeLists.txt:12).  This library restates their behaviour
// without Eigen so the hot path has inputs to consume, and extends them to
// 3-D hexahedra (the paper's formulation):
//   * NodalBasis1D / make_basis / gauss_legendre   basis.cpp:11-193
//   * build_faces / make_periodic / assign_switches mesh.cpp:51-364
//   * compute_mapping (+ curved boundary projection) mapping.cpp:12-153
//   * lattice mesh generators + seeded states for the BASELINE.json configs
// Everything here is setup, run once per case; the hot path lives in the
// CUDA library (csrc/cuda) behind include/linedg_b200.h.
#pragma once

#include <array>
#include <cstdint>
#include <iosfwd>
#include <stdexcept>
#include <string>
#include <vector>

#include "linedg_b200.h"

namespace ldgh {

struct config_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// ------------------------------------------------------------------ basis
struct Basis1D {
  int p = 0;
  bool gll = true;
  std::vector<double> nodes;      // np
  std::vector<double> qp, qw;     // nq
  std::vector<double> phi, dphi;  // [i][q] row-major, np x nq
  std::vector<double> mass;       // np x np
  std::vector<double> diff;       // np x np, diff[j*np+i] = phi_i'(s_j)
  std::vector<double> node_w;     // integral of phi_i
  std::vector<double> bary;       // barycentric weights
  int np() const { return p + 1; }
  int nq() const { return static_cast<int>(qp.size()); }
  // Lagrange basis values / derivatives at arbitrary points, row-major [i][k].
  std::vector<double> eval_phi(const std::vector<double>& pts) const;
  std::vector<double> eval_dphi(const std::vector<double>& pts) const;
};

void gauss_legendre(int n, std::vector<double>& x, std::vector<double>& w);
Basis1D make_basis(int p, bool gll = true);

// ------------------------------------------------------------------- mesh
struct Face {
  int elem_l = -1, face_l = -1, elem_r = -1, face_r = -1;
  int orient = 1;   // 2-D: reversed flag; 3-D: dihedral code
  int tag = -1;
  bool boundary() const { return elem_r < 0; }
};

struct Mesh {
  int dim = 2;
  std::vector<double> verts;   // dim per vertex
  std::vector<int> elems;      // 2^dim per element (2-D: CCW; 3-D: v(a,b,c) = a+2b+4c)
  std::vector<Face> faces;
  std::vector<int> elem_face;  // 2*dim per element
  int nv() const { return static_cast<int>(verts.size()) / dim; }
  int ne() const { return static_cast<int>(elems.size()) / (1 << dim); }
  int nf() const { return static_cast<int>(faces.size()); }
  int vpe() const { return 1 << dim; }
  int fpe() const { return 2 * dim; }
};

// Local-face conventions.  2-D follows the reference (mesh.hpp:12-14, 41-48):
// face 0 at X2=0, 1 at X1=1, 2 at X2=1, 3 at X1=0.  3-D: face = 2*dir+side.
int face_direction(int dim, int lf);
int face_is_plus(int dim, int lf);
int face_of(int dim, int dir, int side);

void build_faces(Mesh& m);  // sets every boundary tag to 0 (mesh.cpp:94)
void make_periodic(Mesh& m, int tag_a, int tag_b, const double* translation);
std::vector<int8_t> assign_switches(const Mesh& m);  // [E][dim]
int count_switch_violations(const Mesh& m, const std::vector<int8_t>& sw);

// ---------------------------------------------------------------- mapping
struct Mapping {
  int dim = 2, p = 0, nq = 0, ne = 0;
  std::vector<double> coords;  // [E][npe][D]
  std::vector<double> jac;     // [E][npe]
  std::vector<double> nvec;    // [E][D][NL][nq][D]
  std::vector<double> nend;    // [E][D][2][NL][D]
};
// Boundary projection of high-order nodes (the reference CurveProjector,
// mapping.hpp:13-15): out = projection of the straight-sided position x of a
// node on a boundary face with the given tag.
struct CurveProjector {
  void (*fn)(void* user, const double* x, int tag, double* out) = nullptr;
  void* user = nullptr;
};
// curve (optional, 2-D): boundary projection + transfinite blend (mapping.cpp:30-65).
Mapping compute_mapping(const Mesh& m, const Basis1D& b, const CurveProjector* curve = nullptr);

// ---------------------------------------------------------------- RNG
// splitmix64; uniform from the top 53 bits; normal by Box-Muller.
struct Rng {
  uint64_t s;
  explicit Rng(uint64_t seed) : s(seed) {}
  uint64_t next();
  double uniform();                    // [0,1)
  double uniform(double a, double b);  // [a,b)
  double normal();
};

// ------------------------------------------------------------- generators
struct LatticeSpec {
  int dim = 2;
  int n = 4;                 // elements per direction
  double length[3] = {1, 1, 1};
  double jitter = 0.0;       // fraction of h
  bool periodic = false;     // all directions
  bool jitter_boundary = false;  // non-periodic: move boundary vertices too
  bool permute = false;
  bool rotate = false;       // random local orientation
  uint64_t seed_jitter = 1, seed_perm = 2, seed_rot = 3;
};
// Boundary tags before pairing: 2-D 1=bottom 2=right 3=top 4=left;
// 3-D 1=x- 2=x+ 3=y- 4=y+ 5=z- 6=z+.
// tag_lines (optional): the boundary tag lines (elem, local_face, tag) as a
// reference mesh file would carry them, recorded before periodic pairing.
Mesh make_lattice_mesh(const LatticeSpec& s, std::vector<int>* tag_lines = nullptr);

// refine_uniform (mesh.cpp:168-213), 2-D.
Mesh refine_uniform(const Mesh& mesh);

// Reference mesh text format (mesh.cpp:115-166), 2-D.
Mesh load_mesh(std::istream& in);
Mesh load_mesh(const std::string& path);
void save_mesh(const Mesh& mesh, std::ostream& out);
void save_mesh(const Mesh& mesh, const std::string& path);

}  // namespace ldgh
