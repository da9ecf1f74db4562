// ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
// C wrapper around the reference's own present setup sources (basis.cpp,
// mesh.cpp, mapping.cpp, compiled unmodified from /root/reference against the
// Eigen shim) so tests can compare the setup restatement with them.
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "linedg/basis.hpp"
#include "linedg/mapping.hpp"
#include "linedg/mesh.hpp"

using namespace linedg;

namespace {
std::string g_err;
struct RefCase {
  NodalBasis1D b;
  QuadMesh m;
  SwitchAssignment sw;
  std::vector<ElementMapping> maps;
};
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_basis(int p, int gll, double* nodes, double* qp, double* qw, double* phi, double* dphi,
              double* mass) {
  try {
    NodalBasis1D b = make_basis(p, gll ? NodeRule::GaussLobatto : NodeRule::Uniform);
    const int np = p + 1, nq = b.n_quad();
    for (int i = 0; i < np; ++i) nodes[i] = b.nodes[i];
    for (int q = 0; q < nq; ++q) {
      qp[q] = b.quad_points[q];
      qw[q] = b.quad_weights[q];
    }
    for (int i = 0; i < np; ++i)
      for (int q = 0; q < nq; ++q) {
        phi[i * nq + q] = b.phi_at_quad(i, q);
        dphi[i * nq + q] = b.dphi_at_quad(i, q);
      }
    for (int i = 0; i < np; ++i)
      for (int j = 0; j < np; ++j) mass[i * np + j] = b.mass(i, j);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

void* ref_case_create(int p, int nv, const double* verts, int ne, const int* elems, int nb,
                      const int* btags, int nper, const int* ptags, const double* ptr) {
  try {
    auto* c = new RefCase;
    c->b = make_basis(p);
    c->m.vertices.resize(nv);
    for (int i = 0; i < nv; ++i) c->m.vertices[i] = Eigen::Vector2d(verts[2 * i], verts[2 * i + 1]);
    c->m.elems.resize(ne);
    for (int e = 0; e < ne; ++e)
      for (int k = 0; k < 4; ++k) c->m.elems[e][k] = elems[4 * e + k];
    build_faces(c->m);
    for (int i = 0; i < nb; ++i) {
      const int fid = c->m.elem_face[btags[3 * i]][btags[3 * i + 1]];
      c->m.faces[fid].tag = btags[3 * i + 2];
    }
    for (int k = 0; k < nper; ++k)
      make_periodic(c->m, ptags[2 * k], ptags[2 * k + 1], Eigen::Vector2d(ptr[3 * k], ptr[3 * k + 1]));
    c->sw = assign_switches(c->m);
    c->maps = compute_mapping(c->m, c->b);
    return c;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

// The reference's own load_mesh (mesh.cpp:115-146) + optional periodic pairs.
void* ref_case_load(int p, const char* path, int nper, const int* ptags, const double* ptr) {
  try {
    auto* c = new RefCase;
    c->b = make_basis(p);
    c->m = load_mesh(std::string(path));
    for (int k = 0; k < nper; ++k)
      make_periodic(c->m, ptags[2 * k], ptags[2 * k + 1], Eigen::Vector2d(ptr[3 * k], ptr[3 * k + 1]));
    c->sw = assign_switches(c->m);
    c->maps = compute_mapping(c->m, c->b);
    return c;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

// The reference's own save_mesh (mesh.cpp:148-160).
int ref_case_save(void* h, const char* path) {
  try {
    save_mesh(static_cast<RefCase*>(h)->m, std::string(path));
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// The reference's compute_mapping with a CurveProjector (mapping.cpp:30-65).
int ref_case_remap(void* h, void (*fn)(void*, const double*, int, double*), void* user) {
  try {
    auto* c = static_cast<RefCase*>(h);
    CurveProjector cp = [fn, user](const Eigen::Vector2d& x, int tag) {
      const double xin[2] = {x.x(), x.y()};
      double out[2];
      fn(user, xin, tag, out);
      return Eigen::Vector2d(out[0], out[1]);
    };
    c->maps = compute_mapping(c->m, c->b, &cp);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// The reference's own refine_uniform (mesh.cpp:168-213) of a case's mesh.
void* ref_case_refine(void* h) {
  try {
    auto* src = static_cast<RefCase*>(h);
    auto* c = new RefCase;
    c->b = src->b;
    c->m = refine_uniform(src->m);
    c->sw = assign_switches(c->m);
    c->maps = compute_mapping(c->m, c->b);
    return c;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}
int ref_case_num_vertices(void* h) { return static_cast<int>(static_cast<RefCase*>(h)->m.vertices.size()); }
void ref_case_vertices(void* h, double* out) {
  const auto& v = static_cast<RefCase*>(h)->m.vertices;
  for (size_t i = 0; i < v.size(); ++i) {
    out[2 * i] = v[i].x();
    out[2 * i + 1] = v[i].y();
  }
}
void ref_case_elements(void* h, int* out) {
  const auto& q = static_cast<RefCase*>(h)->m.elems;
  for (size_t e = 0; e < q.size(); ++e)
    for (int k = 0; k < 4; ++k) out[4 * e + k] = q[e][k];
}

void ref_case_free(void* h) { delete static_cast<RefCase*>(h); }
int ref_case_num_faces(void* h) { return static_cast<RefCase*>(h)->m.num_faces(); }

void ref_case_faces(void* h, int* out) {  // elem_l, face_l, elem_r, face_r, reversed, tag
  const auto& f = static_cast<RefCase*>(h)->m.faces;
  for (size_t i = 0; i < f.size(); ++i) {
    out[6 * i + 0] = f[i].elem_l;
    out[6 * i + 1] = f[i].face_l;
    out[6 * i + 2] = f[i].elem_r;
    out[6 * i + 3] = f[i].face_r;
    out[6 * i + 4] = f[i].reversed ? 1 : 0;
    out[6 * i + 5] = f[i].tag;
  }
}

void ref_case_elem_face(void* h, int* out) {
  const auto& ef = static_cast<RefCase*>(h)->m.elem_face;
  for (size_t e = 0; e < ef.size(); ++e)
    for (int k = 0; k < 4; ++k) out[4 * e + k] = ef[e][k];
}

void ref_case_switches(void* h, signed char* out) {
  const auto& s = static_cast<RefCase*>(h)->sw.plus_sign;
  for (size_t e = 0; e < s.size(); ++e) {
    out[2 * e] = s[e][0];
    out[2 * e + 1] = s[e][1];
  }
}

// coords [E][npe][2], jac [E][npe], nvec [E][2][np][nq][2], nend [E][2][2][np][2]
void ref_case_mapping(void* h, double* coords, double* jac, double* nvec, double* nend) {
  auto* c = static_cast<RefCase*>(h);
  const int np = c->b.p + 1, nq = c->b.n_quad(), npe = np * np;
  for (size_t e = 0; e < c->maps.size(); ++e) {
    const ElementMapping& em = c->maps[e];
    for (int n = 0; n < npe; ++n) {
      coords[(e * npe + n) * 2 + 0] = em.nodes_xy(0, n);
      coords[(e * npe + n) * 2 + 1] = em.nodes_xy(1, n);
      jac[e * npe + n] = em.jac_at_nodes[n];
    }
    for (int dir = 0; dir < 2; ++dir) {
      for (int col = 0; col < np * nq; ++col)
        for (int d = 0; d < 2; ++d)
          nvec[(((e * 2 + dir) * np * nq) + col) * 2 + d] = em.nvec_quad[dir](d, col);
      for (int side = 0; side < 2; ++side)
        for (int line = 0; line < np; ++line)
          for (int d = 0; d < 2; ++d)
            nend[((((e * 2 + dir) * 2 + side) * np) + line) * 2 + d] = em.normal_end[dir][side](d, line);
    }
  }
}

}  // extern "C"
