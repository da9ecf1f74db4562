// lh_capi.cpp -- C-ABI of the setup library (liblinedg_host.so).
//
// Builds a "case": basis, mesh, switches and mapping for the BASELINE.json
// configurations (or a custom vertex/element list), exposes them as the
// flattened ldg_setup the hot path consumes, and fills seeded states.
#include <cmath>
#include <cstring>
#include <memory>
#include <string>

#include "linedg_host.hpp"

using namespace ldgh;

namespace {
thread_local std::string g_err;

int fail(const std::exception& ex) {
  g_err = ex.what();
  if (dynamic_cast<const config_error*>(&ex)) return LDG_ERR_CONFIG;
  if (dynamic_cast<const std::invalid_argument*>(&ex)) return LDG_ERR_INVALID_ARGUMENT;
  return LDG_ERR_SOLVER;
}
}  // namespace

struct lh_case {
  Basis1D basis;
  Mesh mesh;
  std::vector<int8_t> sw;
  Mapping map;
  std::vector<int32_t> fel, ffl, fer, ffr, for_, ftag, ef;
  std::vector<int> tag_lines;
  ldg_setup setup{};
  void flatten() {
    const int nf = mesh.nf();
    fel.resize(nf);
    ffl.resize(nf);
    fer.resize(nf);
    ffr.resize(nf);
    for_.resize(nf);
    ftag.resize(nf);
    for (int i = 0; i < nf; ++i) {
      const Face& f = mesh.faces[i];
      fel[i] = f.elem_l;
      ffl[i] = f.face_l;
      fer[i] = f.elem_r;
      ffr[i] = f.face_r;
      for_[i] = f.orient;
      ftag[i] = f.tag;
    }
    ef.assign(mesh.elem_face.begin(), mesh.elem_face.end());
    setup.dim = mesh.dim;
    setup.p = basis.p;
    setup.n_quad = basis.nq();
    setup.n_elems = mesh.ne();
    setup.n_faces = nf;
    setup.nodes = basis.nodes.data();
    setup.quad_points = basis.qp.data();
    setup.quad_weights = basis.qw.data();
    setup.phi_at_quad = basis.phi.data();
    setup.dphi_at_quad = basis.dphi.data();
    setup.mass = basis.mass.data();
    setup.face_elem_l = fel.data();
    setup.face_face_l = ffl.data();
    setup.face_elem_r = fer.data();
    setup.face_face_r = ffr.data();
    setup.face_orient = for_.data();
    setup.face_tag = ftag.data();
    setup.elem_face = ef.data();
    setup.switch_plus = sw.data();
    setup.jac_at_nodes = map.jac.data();
    setup.nvec_quad = map.nvec.data();
    setup.normal_end = map.nend.data();
    setup.node_coords = map.coords.data();
  }
};

extern "C" {

typedef struct lh_lattice_params {
  int32_t dim, n, p, gll;
  double length[3];
  double jitter;
  int32_t periodic, jitter_boundary, permute, rotate;
  uint64_t seed_jitter, seed_perm, seed_rot;
} lh_lattice_params;

const char* lh_last_error(void) { return g_err.c_str(); }

static void finish_case(lh_case* c) {
  c->sw = assign_switches(c->mesh);
  c->map = compute_mapping(c->mesh, c->basis);
  c->flatten();
}

int lh_case_lattice(const lh_lattice_params* prm, lh_case** out) {
  try {
    auto c = std::make_unique<lh_case>();
    LatticeSpec s;
    s.dim = prm->dim;
    s.n = prm->n;
    for (int a = 0; a < 3; ++a) s.length[a] = prm->length[a];
    s.jitter = prm->jitter;
    s.periodic = prm->periodic != 0;
    s.jitter_boundary = prm->jitter_boundary != 0;
    s.permute = prm->permute != 0;
    s.rotate = prm->rotate != 0;
    s.seed_jitter = prm->seed_jitter;
    s.seed_perm = prm->seed_perm;
    s.seed_rot = prm->seed_rot;
    c->basis = make_basis(prm->p, prm->gll != 0);
    c->mesh = make_lattice_mesh(s, &c->tag_lines);
    finish_case(c.get());
    *out = c.release();
    return LDG_OK;
  } catch (const std::exception& ex) {
    return fail(ex);
  }
}

// Custom mesh: vertices (nv*dim), elements (ne*2^dim), optional boundary tag
// lines (elem, local_face, tag) as in the reference text format
// (mesh.cpp:115-146), optional periodic pairs (tag_a, tag_b, translation).
int lh_case_custom(int32_t dim, int32_t p, int32_t gll, int32_t nv, const double* verts,
                   int32_t ne, const int32_t* elems, int32_t nb, const int32_t* btags,
                   int32_t nper, const int32_t* per_tags, const double* per_tr, lh_case** out) {
  try {
    auto c = std::make_unique<lh_case>();
    c->basis = make_basis(p, gll != 0);
    c->mesh.dim = dim;
    c->mesh.verts.assign(verts, verts + static_cast<size_t>(nv) * dim);
    c->mesh.elems.assign(elems, elems + static_cast<size_t>(ne) * (1 << dim));
    for (int v : c->mesh.elems)
      if (v < 0 || v >= nv) throw config_error("mesh: element has vertex index out of range");
    build_faces(c->mesh);
    for (int b = 0; b < nb; ++b) {
      const int e = btags[3 * b], lf = btags[3 * b + 1], tag = btags[3 * b + 2];
      if (e < 0 || e >= ne || lf < 0 || lf >= 2 * dim)
        throw config_error("mesh: boundary tag line " + std::to_string(b) + " out of range");
      const int fid = c->mesh.elem_face[e * 2 * dim + lf];
      if (!c->mesh.faces[fid].boundary())
        throw config_error("mesh: tagged face is not a boundary face");
      c->mesh.faces[fid].tag = tag;
    }
    for (int k = 0; k < nper; ++k)
      make_periodic(c->mesh, per_tags[2 * k], per_tags[2 * k + 1], per_tr + 3 * k);
    finish_case(c.get());
    *out = c.release();
    return LDG_OK;
  } catch (const std::exception& ex) {
    return fail(ex);
  }
}

// Reference mesh file (mesh.cpp:115-146) + optional periodic pairs, then the
// same switch / mapping setup as every case.  tag_lines records the boundary
// faces as loaded (before pairing).
int lh_case_load_mesh(const char* path, int32_t p, int32_t gll, int32_t nper, const int32_t* per_tags,
                      const double* per_tr, lh_case** out) {
  try {
    if (!path) throw std::invalid_argument("path is NULL");
    auto c = std::make_unique<lh_case>();
    c->basis = make_basis(p, gll != 0);
    c->mesh = load_mesh(std::string(path));
    for (const Face& f : c->mesh.faces)
      if (f.boundary()) c->tag_lines.insert(c->tag_lines.end(), {f.elem_l, f.face_l, f.tag});
    for (int k = 0; k < nper; ++k)
      make_periodic(c->mesh, per_tags[2 * k], per_tags[2 * k + 1], per_tr + 3 * k);
    finish_case(c.get());
    *out = c.release();
    return LDG_OK;
  } catch (const std::exception& ex) {
    return fail(ex);
  }
}

// save_mesh (mesh.cpp:148-160) of a case's mesh (2-D).
int lh_case_save_mesh(const lh_case* c, const char* path) {
  try {
    if (!path) throw std::invalid_argument("path is NULL");
    save_mesh(c->mesh, std::string(path));
    return LDG_OK;
  } catch (const std::exception& ex) {
    return fail(ex);
  }
}

// Curved boundaries: recompute the mapping with a boundary projection
// (CurveProjector, mapping.hpp:13-15; mapping.cpp:30-65).  fn(user, x, tag,
// out) returns the projected position of a straight-sided boundary node.
int lh_case_remap(lh_case* c, void (*fn)(void*, const double*, int, double*), void* user) {
  try {
    if (c->mesh.dim != 2) throw config_error("mapping: curved boundaries are 2-D only (reference mapping.cpp)");
    CurveProjector cp;
    cp.fn = fn;
    cp.user = user;
    c->map = compute_mapping(c->mesh, c->basis, fn ? &cp : nullptr);
    c->flatten();
    return LDG_OK;
  } catch (const std::exception& ex) {
    return fail(ex);
  }
}

namespace {
struct Circles {
  std::vector<int> tags;
  std::vector<double> cx, cy, r;
};
// radial projection onto the circle of the face's tag (identity for other tags)
void circle_proj(void* user, const double* x, int tag, double* out) {
  const Circles& cs = *static_cast<const Circles*>(user);
  out[0] = x[0];
  out[1] = x[1];
  for (size_t i = 0; i < cs.tags.size(); ++i)
    if (cs.tags[i] == tag) {
      const double dx = x[0] - cs.cx[i], dy = x[1] - cs.cy[i];
      const double s = cs.r[i] / std::sqrt(dx * dx + dy * dy);
      out[0] = cs.cx[i] + s * dx;
      out[1] = cs.cy[i] + s * dy;
      return;
    }
}
}  // namespace

// Built-in projector: boundary faces tagged tags[k] lie on the circle of
// centre (cx[k], cy[k]) and radius r[k] (the paper's cylinder geometry).
int lh_case_remap_circles(lh_case* c, int32_t n, const int32_t* tags, const double* cx, const double* cy,
                          const double* r) {
  Circles cs;
  cs.tags.assign(tags, tags + n);
  cs.cx.assign(cx, cx + n);
  cs.cy.assign(cy, cy + n);
  cs.r.assign(r, r + n);
  return lh_case_remap(c, circle_proj, &cs);
}

// Uniformly refined copy of a case's mesh (refine_uniform, mesh.cpp:168-213),
// same basis, then optional periodic pairs.  tag_lines: the refined boundary.
int lh_case_refine(const lh_case* src, int32_t nper, const int32_t* per_tags, const double* per_tr,
                   lh_case** out) {
  try {
    auto c = std::make_unique<lh_case>();
    c->basis = src->basis;
    c->mesh = refine_uniform(src->mesh);
    for (const Face& f : c->mesh.faces)
      if (f.boundary()) c->tag_lines.insert(c->tag_lines.end(), {f.elem_l, f.face_l, f.tag});
    for (int k = 0; k < nper; ++k)
      make_periodic(c->mesh, per_tags[2 * k], per_tags[2 * k + 1], per_tr + 3 * k);
    finish_case(c.get());
    *out = c.release();
    return LDG_OK;
  } catch (const std::exception& ex) {
    return fail(ex);
  }
}

void lh_case_free(lh_case* c) { delete c; }
int32_t lh_case_num_tag_lines(const lh_case* c) { return static_cast<int32_t>(c->tag_lines.size() / 3); }
void lh_case_tag_lines(const lh_case* c, int32_t* out) {
  for (size_t i = 0; i < c->tag_lines.size(); ++i) out[i] = c->tag_lines[i];
}
const ldg_setup* lh_case_setup(const lh_case* c) { return &c->setup; }
int32_t lh_case_num_vertices(const lh_case* c) { return c->mesh.nv(); }
const double* lh_case_vertices(const lh_case* c) { return c->mesh.verts.data(); }
const int32_t* lh_case_elements(const lh_case* c) { return c->mesh.elems.data(); }
int32_t lh_case_switch_violations(const lh_case* c) { return count_switch_violations(c->mesh, c->sw); }
int32_t lh_case_num_boundary_faces(const lh_case* c) {
  int n = 0;
  for (const Face& f : c->mesh.faces) n += f.boundary() ? 1 : 0;
  return n;
}

// Basis tables for KATs: every output is optional.
int lh_basis(int32_t p, int32_t gll, double* nodes, double* qp, double* qw, double* phi,
             double* dphi, double* mass, double* diff, double* node_w) {
  try {
    const Basis1D b = make_basis(p, gll != 0);
    auto cp = [](const std::vector<double>& v, double* o) {
      if (o) std::memcpy(o, v.data(), v.size() * sizeof(double));
    };
    cp(b.nodes, nodes);
    cp(b.qp, qp);
    cp(b.qw, qw);
    cp(b.phi, phi);
    cp(b.dphi, dphi);
    cp(b.mass, mass);
    cp(b.diff, diff);
    cp(b.node_w, node_w);
    return LDG_OK;
  } catch (const std::exception& ex) {
    return fail(ex);
  }
}

int lh_gauss_legendre(int32_t n, double* x, double* w) {
  try {
    std::vector<double> xs, ws;
    gauss_legendre(n, xs, ws);
    std::memcpy(x, xs.data(), n * sizeof(double));
    std::memcpy(w, ws.data(), n * sizeof(double));
    return LDG_OK;
  } catch (const std::exception& ex) {
    return fail(ex);
  }
}

// ------------------------------------------------------------------ states
// kind 1: scalar sin(pi x) sin(pi y) (C1)            prm: [noise]
// kind 2: isentropic vortex (physics.hpp:207-222)    prm: [eps, r_c, mach, theta, x0, y0, rho_inf,
//                                                          u_inf, p_inf, gamma, t, noise]
// kind 3: uniform flow + Fourier perturbation (C3)   prm: [rho, u, v, p, gamma, amp, modes, noise]
// kind 4: Taylor-Green vortex (C4/C5, 3-D)           prm: [V0, rho0, p0, gamma, k, noise]
// kind 5: N(0,1) per entry                           prm: []
// noise: U(-noise, noise) added to every conserved variable.
int lh_fill_state(const lh_case* c, int32_t kind, int32_t m, const double* prm, uint64_t seed,
                  double* out) {
  try {
    const int D = c->mesh.dim;
    const size_t nn = c->map.jac.size();  // E * npe
    const double* X = c->map.coords.data();
    Rng rng(seed);
    auto noise = [&](double amp) { return amp == 0.0 ? 0.0 : rng.uniform(-amp, amp); };
    if (kind == 1) {
      for (size_t i = 0; i < nn; ++i) {
        const double x = X[i * D], y = X[i * D + 1];
        out[i * m] = std::sin(M_PI * x) * std::sin(M_PI * y) + noise(prm[0]);
      }
    } else if (kind == 2) {
      if (D != 2 || m != 4) throw config_error("vortex state needs D=2, m=4");
      const double eps = prm[0], rc = prm[1], mach = prm[2], th = prm[3], x0 = prm[4], y0 = prm[5];
      const double rinf = prm[6], uinf = prm[7], pinf = prm[8], g = prm[9], t = prm[10];
      const double ub = uinf * std::cos(th), vb = uinf * std::sin(th);
      for (size_t i = 0; i < nn; ++i) {
        const double dx = (X[i * 2] - x0) - ub * t, dy = (X[i * 2 + 1] - y0) - vb * t;
        const double f = (1.0 - dx * dx - dy * dy) / (rc * rc);
        const double u = uinf * (std::cos(th) - eps * dy / (2.0 * M_PI * rc) * std::exp(f / 2.0));
        const double v = uinf * (std::sin(th) + eps * dx / (2.0 * M_PI * rc) * std::exp(f / 2.0));
        const double base = 1.0 - eps * eps * (g - 1.0) * mach * mach / (8.0 * M_PI * M_PI) * std::exp(f);
        const double rho = rinf * std::pow(base, 1.0 / (g - 1.0));
        const double pr = pinf * std::pow(base, g / (g - 1.0));
        double* o = out + i * 4;
        o[0] = rho;
        o[1] = rho * u;
        o[2] = rho * v;
        o[3] = pr / (g - 1.0) + 0.5 * rho * (u * u + v * v);
        for (int k = 0; k < 4; ++k) o[k] += noise(prm[11]);
      }
    } else if (kind == 3) {
      if (D != 2 || m != 4) throw config_error("Fourier state needs D=2, m=4");
      const double r0 = prm[0], u0 = prm[1], v0 = prm[2], p0 = prm[3], g = prm[4], amp = prm[5];
      const int modes = static_cast<int>(prm[6]);
      // Coefficients c[var][a][b] ~ U(-1,1)/modes^2 and phases U(0,2pi), drawn first.
      std::vector<double> coef(static_cast<size_t>(4) * modes * modes), ph(coef.size());
      for (size_t k = 0; k < coef.size(); ++k) {
        coef[k] = rng.uniform(-1.0, 1.0) / (modes * modes);
        ph[k] = rng.uniform(0.0, 2.0 * M_PI);
      }
      for (size_t i = 0; i < nn; ++i) {
        const double x = X[i * 2], y = X[i * 2 + 1];
        double d[4] = {0, 0, 0, 0};
        for (int var = 0; var < 4; ++var)
          for (int a = 1; a <= modes; ++a)
            for (int b = 1; b <= modes; ++b) {
              const size_t k = (static_cast<size_t>(var) * modes + (a - 1)) * modes + (b - 1);
              d[var] += coef[k] * std::sin(2.0 * M_PI * (a * x + b * y) + ph[k]);
            }
        const double rho = r0 + amp * d[0], u = u0 + amp * d[1], v = v0 + amp * d[2];
        const double pr = p0 + amp * d[3];
        double* o = out + i * 4;
        o[0] = rho;
        o[1] = rho * u;
        o[2] = rho * v;
        o[3] = pr / (g - 1.0) + 0.5 * rho * (u * u + v * v);
      }
      for (size_t i = 0; i < nn * 4; ++i) out[i] += noise(prm[7]);
    } else if (kind == 4) {
      if (D != 3 || m != 5) throw config_error("Taylor-Green state needs D=3, m=5");
      const double V0 = prm[0], r0 = prm[1], p0 = prm[2], g = prm[3], k = prm[4];
      for (size_t i = 0; i < nn; ++i) {
        const double x = X[i * 3], y = X[i * 3 + 1], z = X[i * 3 + 2];
        const double u = V0 * std::sin(k * x) * std::cos(k * y) * std::cos(k * z);
        const double v = -V0 * std::cos(k * x) * std::sin(k * y) * std::cos(k * z);
        const double w = 0.0;
        const double pr = p0 + r0 * V0 * V0 / 16.0 * (std::cos(2 * k * x) + std::cos(2 * k * y)) *
                                   (std::cos(2 * k * z) + 2.0);
        const double rho = r0 * pr / p0;  // isothermal initial density
        double* o = out + i * 5;
        o[0] = rho;
        o[1] = rho * u;
        o[2] = rho * v;
        o[3] = rho * w;
        o[4] = pr / (g - 1.0) + 0.5 * rho * (u * u + v * v + w * w);
        for (int q = 0; q < 5; ++q) o[q] += noise(prm[5]);
      }
    } else if (kind == 5) {
      for (size_t i = 0; i < nn * static_cast<size_t>(m); ++i) out[i] = rng.normal();
    } else {
      throw std::invalid_argument("lh_fill_state: unknown kind");
    }
    return LDG_OK;
  } catch (const std::exception& ex) {
    return fail(ex);
  }
}

}  // extern "C"
