// ldg_capi.cu -- context, host-side table preparation and the C-ABI of the
// B200 Line-DG hot path (include/linedg_b200.h).
//
// Host work done once per context (setup, never on the hot path):
//   * fold the basis: M^-1 from the Cholesky factor of M (basis.cpp:185-189),
//     dq = -M^-1 Phi' W, lifting columns M^-1[:,0], M^-1[:,p], line-block
//     coefficients cc[i][t][q] = dq[i][q] phi[t][q];
//   * derive, from the reference Face / elem_face / reversed tables
//     (mesh.hpp:15-32), for every element line end the neighbour element and
//     the affine map line -> neighbour node (c0 + c1 l1 + c2 l2), plus the
//     LDG switch sign at that end (mesh.hpp:74-89);
//   * re-lay the ElementMapping tables (mapping.hpp:19-33) per element in
//     processing order, with 1/J precomputed, and upload.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "ldg_ops.cuh"
#include "linedg_b200.h"

// ---------------------------------------------------------------- dispatch
#define LDG_FOR_PH(X, D, P) X(D, P, 0, 0) X(D, P, 1, 0) X(D, P, 1, 1) X(D, P, 2, 0) X(D, P, 2, 1)
#define LDG_FOR_ALL(X)                                                                    \
  LDG_FOR_PH(X, 2, 1) LDG_FOR_PH(X, 2, 2) LDG_FOR_PH(X, 2, 3) LDG_FOR_PH(X, 2, 4)        \
  LDG_FOR_PH(X, 3, 1) LDG_FOR_PH(X, 3, 2) LDG_FOR_PH(X, 3, 3) LDG_FOR_PH(X, 3, 4)
LDG_FOR_ALL(LDG_DECLARE_OPS)

namespace {

const ldg::Ops* find_ops(int D, int P, int PH, int RI) {
#define LDG_MATCH(d, p, ph, ri) \
  if (D == d && P == p && PH == ph && RI == ri) return LDG_OPS_NAME(d, p, ph, ri)();
  LDG_FOR_ALL(LDG_MATCH)
#undef LDG_MATCH
  return nullptr;
}

struct ldg_error : std::runtime_error {
  int status;
  ldg_error(int s, const std::string& w) : std::runtime_error(w), status(s) {}
};

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw ldg_error(LDG_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

thread_local std::string g_create_err;

}  // namespace

struct ldg_ctx {
  const ldg::Ops* ops = nullptr;
  ldg::DevCtx dc;
  int D = 2, p = 1, np = 2, nq = 2, npe = 4, NL = 2, m = 1, E = 0;
  int kind = 0, riemann = 0, ph = 0;
  bool second = false, has_inv = false, vis_u = false;
  double c11 = 0.0, c11bd = 0.0;
  std::vector<double> phi, dq, mi, cc;
  std::vector<int32_t> order, inv_order;
  std::vector<int2> conn;
  std::vector<int2> fpart;       // [k][2D] face partner {k', 2 dir' + side'} or {-1, 0}
  std::vector<int64_t> owned_off;  // per Jacobian chunk, into d_owned
  std::vector<int64_t> bspec_off;  // per Jacobian chunk, into d_bspec (slip-wall / Neumann ends)
  // device
  int2* d_fpart = nullptr;
  int32_t* d_owned = nullptr;
  int32_t* d_bspec = nullptr;
  int32_t* d_inv_order = nullptr;
  // block-Jacobi preconditioner (per element LU, column-major) and GMRES workspace
  double* d_pcLU = nullptr;
  int32_t* d_pcPiv = nullptr;
  int* d_pcbad = nullptr;
  bool pc_valid = false;
  double pc_adt = 0.0;
  int pc_mode = 0;       // ldg_set_precond_mode
  bool pc_adi = false;   // the built preconditioner is line-ADI
  size_t pc_nlu = 0, pc_npiv = 0;  // allocated factor / pivot entries
  double* d_ti = nullptr;  // time-integration workspace (8 vectors)
  double* d_kv = nullptr;  // Krylov vectors V[0..restart] then Z[0..restart-1]
  int kv_restart = 0;
  double* d_kw = nullptr;  // w, t, r
  double* d_kred = nullptr;  // reduction partials + Hessenberg (column-major) + scalars
  double* h_gst = nullptr;            // pinned ring of GMRES cycle states
  cudaEvent_t ev_gw[4] = {nullptr, nullptr, nullptr, nullptr};
  int32_t* d_order = nullptr;
  double* d_metric = nullptr;
  int2* d_conn = nullptr;
  double* d_bcv = nullptr;
  int32_t* d_bck = nullptr;     // boundary kind per boundary index
  std::vector<int32_t> bck;
  // boundary functions (ldg_set_boundary_function): boundary faces (k, ds) in
  // processing order, their tags, end-node coordinates [face][NL][D]
  std::vector<int32_t> bface_of, bface_tag, bc_tag;
  std::vector<double> bface_x, bcv_host;
  std::map<int, std::pair<ldg_bc_fn, void*>> bfun;
  double bfun_t = 0.0;
  bool bfun_dirty = false, has_coords = false;
  int32_t* d_bface = nullptr;
  double* d_bvals = nullptr;
  double* d_source = nullptr;
  ldg::DevError* h_err = nullptr;
  ldg::DevError* d_err = nullptr;
  double* d_Q = nullptr;  // workspace Q = D(U)
  double* d_w = nullptr;  // workspace w = K21 v
  double* d_K11 = nullptr;
  double* d_K12 = nullptr;
  double* d_K21 = nullptr;
  double* d_SE = nullptr;  // endpoint flux-Jacobian scratch
  size_t n11 = 0, n12 = 0, n21 = 0;
  bool jac_valid = false, k21_valid = false;
  double* d_hu = nullptr;  // staging for host variants
  double* d_hu2 = nullptr;  // (assembly input: a separate buffer so its upload overlaps the residual)
  double* d_hr = nullptr;
  // asynchronous host variants (sync_errors off): uploads on cs_in, downloads
  // on cs_out, kernels on `stream`; events order buffer reuse
  cudaStream_t cs_in = nullptr, cs_out = nullptr;
  cudaEvent_t ev_in = nullptr, ev_k = nullptr, ev_free_hu = nullptr, ev_free_hu2 = nullptr, ev_free_hx = nullptr,
              ev_out_r = nullptr, ev_out_y = nullptr, ev_join = nullptr;
  double* d_hx = nullptr;
  double* d_hy = nullptr;
  // split_matvec_host staging ring (asynchronous mode)
  double* d_mv_in[2] = {nullptr, nullptr};
  double* d_mv_out[2] = {nullptr, nullptr};
  cudaEvent_t ev_mv_free[2] = {nullptr, nullptr}, ev_mv_out[2] = {nullptr, nullptr};
  int mv_slot = 0;
  cudaStream_t stream = nullptr;
  long long launches = 0;
  bool sync_errors = true;
  bool zero_copy = true;  // LDG_OPT_ZERO_COPY
  int device = -1;       // CUDA device of the context (current at ldg_create)
  std::string err;
  int err_elem = -1, err_node = -1;
  double err_state[8] = {0};

  size_t nU() const { return static_cast<size_t>(E) * npe * m; }
  size_t nQ() const { return nU() * D; }

  ~ldg_ctx() {
    cudaFree(d_order);
    cudaFree(d_metric);
    cudaFree(d_conn);
    cudaFree(d_fpart);
    cudaFree(d_owned);
    cudaFree(d_bspec);
    cudaFree(d_inv_order);
    cudaFree(d_pcLU);
    cudaFree(d_pcPiv);
    cudaFree(d_pcbad);
    cudaFree(d_kv);
    cudaFree(d_kw);
    cudaFree(d_kred);
    cudaFree(d_ti);
    cudaFree(d_bcv);
    cudaFree(d_bck);
    cudaFree(d_bface);
    cudaFree(d_bvals);
    cudaFree(d_source);
    cudaFree(d_Q);
    cudaFree(d_w);
    cudaFree(d_K11);
    cudaFree(d_K12);
    cudaFree(d_K21);
    cudaFree(d_SE);
    cudaFree(d_hu);
    cudaFree(d_hu2);
    cudaFree(d_hr);
    for (cudaEvent_t ev : {ev_in, ev_k, ev_free_hu, ev_free_hu2, ev_free_hx, ev_out_r, ev_out_y, ev_join})
      if (ev) cudaEventDestroy(ev);
    if (cs_in) cudaStreamDestroy(cs_in);
    if (cs_out) cudaStreamDestroy(cs_out);
    cudaFree(d_hx);
    cudaFree(d_hy);
    for (int k = 0; k < 2; ++k) {
      cudaFree(d_mv_in[k]);
      cudaFree(d_mv_out[k]);
      if (ev_mv_free[k]) cudaEventDestroy(ev_mv_free[k]);
      if (ev_mv_out[k]) cudaEventDestroy(ev_mv_out[k]);
    }
    if (h_err) cudaFreeHost(h_err);
    if (h_gst) cudaFreeHost(h_gst);
    for (cudaEvent_t ev : ev_gw)
      if (ev) cudaEventDestroy(ev);
  }

  int node_on_line(int dir, int line, int t) const {
    if (D == 2) return dir == 0 ? t + np * line : line + np * t;
    const int l1 = line % np, l2 = line / np;
    if (dir == 0) return t + np * l1 + np * np * l2;
    if (dir == 1) return l1 + np * t + np * np * l2;
    return l1 + np * l2 + np * np * t;
  }
  void line_of(int dir, int nd, int& line, int& pos) const {
    const int x0 = nd % np, x1 = (nd / np) % np, x2 = nd / (np * np);
    if (D == 2) {
      line = dir == 0 ? x1 : x0;
      pos = dir == 0 ? x0 : x1;
    } else if (dir == 0) {
      line = x1 + np * x2;
      pos = x0;
    } else if (dir == 1) {
      line = x0 + np * x2;
      pos = x1;
    } else {
      line = x0 + np * x1;
      pos = x2;
    }
  }
  const int2& cn(int k, int dir, int side) const {
    return conn[(static_cast<size_t>(k) * D + dir) * 2 + side];
  }
  static int csign(const int2& c) { return (c.y >> 24) & 1 ? 1 : -1; }
  int cnode(const int2& c, int line) const {
    const int c0 = c.y & 0xff;
    const int c1 = static_cast<int8_t>((c.y >> 8) & 0xff);
    const int c2 = static_cast<int8_t>((c.y >> 16) & 0xff);
    return c0 + c1 * (line % np) + c2 * (line / np);
  }

  // ---- structural pattern: which slots of a row exist
  bool in_dep(int k, int dir, int side) const {
    const int2& c = cn(k, dir, side);
    const bool bd = c.x < 0;
    const int bkind = bd ? bck[-1 - c.x] : -1;
    if (bkind == LDG_BC_NEUMANN) return false;  // prescribed flux: no u dependence
    if (has_inv) return true;
    if (!second) return false;
    if (bd) return vis_u || (bkind != LDG_BC_SLIP_WALL && c11bd != 0.0);
    return (vis_u && csign(c) <= 0) || c11 != 0.0;
  }
  bool out_dep(int k, int dir, int side) const {
    const int2& c = cn(k, dir, side);
    if (c.x < 0) return false;
    if (has_inv) return true;
    if (!second) return false;
    return (vis_u && csign(c) > 0) || c11 != 0.0;
  }
  int nslots(int which) const { return which == LDG_K11 ? D * p + 1 + 2 * D : D * p + 1 + D; }
  // Column node (reference numbering) of `slot` for row (k, nd); -1 if none;
  // `present` = structural presence.
  int64_t slot_col(int which, int k, int nd, int slot, bool& present) const {
    const int64_t e = order[k];
    const int x[3] = {nd % np, (nd / np) % np, nd / (np * np)};
    const int st[3] = {1, np, np * np};
    const int nin = D * p + 1;
    present = false;
    if (slot < nin) {
      int dir, t;
      if (slot < np) {
        dir = 0;
        t = slot;
      } else {
        const int z = slot - np;
        dir = 1 + z / p;
        t = z % p;
        if (t >= x[dir]) ++t;
      }
      auto dep = [&](int d, int tt) {
        if (which != LDG_K11) return second;  // K12, K21: volume terms always
        const bool vol = has_inv || (second && vis_u);
        return vol || (tt == 0 && in_dep(k, d, 0)) || (tt == p && in_dep(k, d, 1));
      };
      if (dir == 0 && t == x[0]) {  // self column: any direction
        for (int d = 0; d < D; ++d) present = present || dep(d, x[d]);
      } else {
        present = dep(dir, t);
      }
      return e * npe + nd + static_cast<int64_t>(t - x[dir]) * st[dir];
    }
    int dir, side;
    const int z = slot - nin;
    if (which == LDG_K11) {
      dir = z >> 1;
      side = z & 1;
    } else {
      dir = z;
      const bool plus1 = csign(cn(k, dir, 1)) > 0;
      side = which == LDG_K12 ? (plus1 ? 1 : 0) : (plus1 ? 0 : 1);
    }
    const int2& c = cn(k, dir, side);
    if (c.x < 0) return -1;
    if (which == LDG_K11) present = out_dep(k, dir, side);
    else present = second;
    int line, pos;
    line_of(dir, nd, line, pos);
    return static_cast<int64_t>(c.x) * npe + cnode(c, line);
  }
};

namespace {

int face_of(int D, int dir, int side) {
  if (D == 2) return dir == 0 ? (side ? 1 : 3) : (side ? 2 : 0);
  return 2 * dir + side;
}

// Inverse of face_of: reference local face -> 2 dir + side.
int local_face_ds(int D, int lf) {
  for (int ds = 0; ds < 2 * D; ++ds)
    if (face_of(D, ds >> 1, ds & 1) == lf) return ds;
  return -1;
}

// Face sharing of the endpoint flux Jacobians: keep a partner link only where
// it is mutual and (second-order physics) the LDG switch flips across the
// face; then list, chunk by chunk, the faces whose Jacobians the chunk
// computes: every face whose partner lies outside the chunk, and of an
// in-chunk pair the one with the lower (k, ds).
// Boundary ends with a slip-wall or Neumann condition are listed apart
// (bspec): k_endjac<..., BND = true> handles them, so the main instantiation
// keeps a seed-independent exterior state.
void build_face_sharing(ldg_ctx& c, int chunk, bool share) {
  const int F = 2 * c.D;
  if (!share) std::fill(c.fpart.begin(), c.fpart.end(), int2{-1, 0});
  for (int k = 0; k < c.E; ++k)
    for (int ds = 0; ds < F; ++ds) {
      int2& p = c.fpart[static_cast<size_t>(k) * F + ds];
      if (p.x < 0) continue;
      const int2 q = c.fpart[static_cast<size_t>(p.x) * F + p.y];
      const int s0 = (c.conn[static_cast<size_t>(k) * F + ds].y >> 24) & 1;
      const int s1 = (c.conn[static_cast<size_t>(p.x) * F + p.y].y >> 24) & 1;
      if (p.y < 0 || q.x != k || q.y != ds || (c.second && s0 == s1)) p = int2{-1, 0};
    }
  std::vector<int32_t> owned, bspec;
  c.owned_off.assign(1, 0);
  c.bspec_off.assign(1, 0);
  for (int kb = 0; kb < c.E; kb += chunk) {
    const int ke = std::min(c.E, kb + chunk);
    for (int k = kb; k < ke; ++k)
      for (int ds = 0; ds < F; ++ds) {
        const int2 cx = c.conn[static_cast<size_t>(k) * F + ds];
        if (cx.x < 0) {
          const int kind = c.bck[-1 - cx.x];
          if (kind == LDG_BC_SLIP_WALL || kind == LDG_BC_NEUMANN || kind == LDG_BC_NO_SLIP_ADIABATIC) {
            bspec.push_back(k * F + ds);
            continue;
          }
        }
        const int2 p = c.fpart[static_cast<size_t>(k) * F + ds];
        const bool mine = p.x < kb || p.x >= ke || static_cast<int64_t>(k) * F + ds < static_cast<int64_t>(p.x) * F + p.y;
        if (mine) owned.push_back(k * F + ds);
      }
    c.owned_off.push_back(static_cast<int64_t>(owned.size()));
    c.bspec_off.push_back(static_cast<int64_t>(bspec.size()));
  }
  ck(cudaMalloc(&c.d_bspec, std::max<size_t>(1, bspec.size()) * sizeof(int32_t)), "cudaMalloc bspec");
  ck(cudaMemcpy(c.d_bspec, bspec.data(), bspec.size() * sizeof(int32_t), cudaMemcpyHostToDevice), "upload bspec");
  ck(cudaMalloc(&c.d_fpart, c.fpart.size() * sizeof(int2)), "cudaMalloc fpart");
  ck(cudaMemcpy(c.d_fpart, c.fpart.data(), c.fpart.size() * sizeof(int2), cudaMemcpyHostToDevice), "upload fpart");
  ck(cudaMalloc(&c.d_owned, std::max<size_t>(1, owned.size()) * sizeof(int32_t)), "cudaMalloc owned");
  ck(cudaMemcpy(c.d_owned, owned.data(), owned.size() * sizeof(int32_t), cudaMemcpyHostToDevice), "upload owned");
}

// 2-D reference face parameterisation (mesh.cpp:51-65).
int face_param_2d(int p, int lf, int nd) {
  const int np = p + 1, i = nd % np, j = nd / np;
  switch (lf) {
    case 0: return i;
    case 1: return j;
    case 2: return p - i;
    default: return p - j;
  }
}
int face_node_2d(int p, int lf, int k) {
  const int np = p + 1;
  switch (lf) {
    case 0: return k;
    case 1: return p + np * k;
    case 2: return (p - k) + np * p;
    default: return np * (p - k);
  }
}
// 3-D: face (dir, side), parameters along the transverse axes in increasing order.
int face_node_3d(int p, int lf, int a, int b) {
  const int np = p + 1, dir = lf / 2, side = lf % 2;
  const int st[3] = {1, np, np * np};
  const int a1 = dir == 0 ? 1 : 0, a2 = dir == 2 ? 1 : 2;
  return side * p * st[dir] + a * st[a1] + b * st[a2];
}
void dihedral(int o, int a, int b, int p, int& ao, int& bo) {
  int x = a, y = b;
  if (o & 1) std::swap(x, y);
  ao = (o & 2) ? p - x : x;
  bo = (o & 4) ? p - y : y;
}

// Cholesky-based inverse of the SPD mass matrix.
std::vector<double> spd_inverse(const double* A, int n) {
  std::vector<double> L(A, A + n * n);
  for (int k = 0; k < n; ++k) {
    double d = L[k * n + k];
    for (int j = 0; j < k; ++j) d -= L[k * n + j] * L[k * n + j];
    if (!(d > 0.0)) throw ldg_error(LDG_ERR_CONFIG, "mass matrix is not SPD");
    d = std::sqrt(d);
    L[k * n + k] = d;
    for (int i = k + 1; i < n; ++i) {
      double s = L[i * n + k];
      for (int j = 0; j < k; ++j) s -= L[i * n + j] * L[k * n + j];
      L[i * n + k] = s / d;
    }
  }
  std::vector<double> inv(n * n, 0.0);
  for (int c = 0; c < n; ++c) {
    std::vector<double> y(n, 0.0), x(n, 0.0);
    for (int i = 0; i < n; ++i) {
      double s = i == c ? 1.0 : 0.0;
      for (int j = 0; j < i; ++j) s -= L[i * n + j] * y[j];
      y[i] = s / L[i * n + i];
    }
    for (int i = n - 1; i >= 0; --i) {
      double s = y[i];
      for (int j = i + 1; j < n; ++j) s -= L[j * n + i] * x[j];
      x[i] = s / L[i * n + i];
    }
    for (int i = 0; i < n; ++i) inv[i * n + c] = x[i];
  }
  return inv;
}

// Element processing order.  Kernels walk elements in this order and gather
// face neighbours by reference id, so an order in which face neighbours are
// processed close together in time turns the neighbour-trace gathers of the
// residual, the endpoint Jacobians and the SpMV into L2 hits (a renumbered
// mesh in storage order has none).  Default: Morton (Z-order) of the element
// centroids on a 2^(60/D)-per-axis grid over the bounding box, ties by id;
// without node coordinates a breadth-first order over the face graph.
std::vector<int32_t> processing_order(const ldg_setup& s, int D, int npe) {
  const int E = s.n_elems;
  std::vector<int32_t> ord(E);
  for (int e = 0; e < E; ++e) ord[e] = e;
  if (s.node_coords) {
    std::vector<double> cen(static_cast<size_t>(E) * D, 0.0);
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    for (int e = 0; e < E; ++e)
      for (int d = 0; d < D; ++d) {
        double a = 0.0;
        for (int n = 0; n < npe; ++n) a += s.node_coords[(static_cast<size_t>(e) * npe + n) * D + d];
        a /= npe;
        cen[static_cast<size_t>(e) * D + d] = a;
        lo[d] = std::min(lo[d], a);
        hi[d] = std::max(hi[d], a);
      }
    const int bits = D == 2 ? 30 : 20;
    const double cells = static_cast<double>((1u << bits) - 1);
    std::vector<std::pair<uint64_t, int32_t>> key(E);
    for (int e = 0; e < E; ++e) {
      uint64_t code = 0;
      uint32_t q[3] = {0, 0, 0};
      for (int d = 0; d < D; ++d) {
        const double w = hi[d] > lo[d] ? (cen[static_cast<size_t>(e) * D + d] - lo[d]) / (hi[d] - lo[d]) : 0.0;
        q[d] = static_cast<uint32_t>(std::min(cells, std::max(0.0, w * cells)));
      }
      for (int b = bits - 1; b >= 0; --b)
        for (int d = D - 1; d >= 0; --d) code = (code << 1) | ((q[d] >> b) & 1u);
      key[e] = {code, e};
    }
    std::sort(key.begin(), key.end());
    for (int e = 0; e < E; ++e) ord[e] = key[e].second;
    return ord;
  }
  // breadth-first over face neighbours, restarting at the lowest unvisited id
  const int F = 2 * D;
  std::vector<char> seen(E, 0);
  int head = 0, tail = 0;
  for (int root = 0; root < E; ++root) {
    if (seen[root]) continue;
    seen[root] = 1;
    ord[tail++] = root;
    while (head < tail) {
      const int e = ord[head++];
      for (int lf = 0; lf < F; ++lf) {
        const int fid = s.elem_face[static_cast<size_t>(e) * F + lf];
        if (fid < 0 || fid >= s.n_faces || s.face_elem_r[fid] < 0) continue;
        const int oe = s.face_elem_l[fid] == e && s.face_face_l[fid] == lf ? s.face_elem_r[fid] : s.face_elem_l[fid];
        if (oe >= 0 && oe < E && !seen[oe]) {
          seen[oe] = 1;
          ord[tail++] = oe;
        }
      }
    }
  }
  return ord;
}

void build_connectivity(ldg_ctx& c, const ldg_setup& s, const ldg_physics& ph) {
  std::map<int, int> tag2bc;
  std::vector<double> bcv;
  c.bck.clear();
  for (int i = 0; i < ph.n_bc; ++i) {
    const int kind = ph.bcs[i].kind;
    if (kind < LDG_BC_DIRICHLET || kind > LDG_BC_NO_SLIP_ADIABATIC)
      throw ldg_error(LDG_ERR_CONFIG, "unsupported boundary-condition kind");
    if ((kind == LDG_BC_SLIP_WALL || kind == LDG_BC_NO_SLIP_ADIABATIC) && !c.has_inv)
      throw ldg_error(LDG_ERR_CONFIG, "slip-wall and no-slip-wall boundaries need Euler or Navier-Stokes physics");
    if (kind == LDG_BC_NO_SLIP_ADIABATIC) ++c.dc.noslip;
    tag2bc[ph.bcs[i].tag] = i;
    c.bck.push_back(kind);
    for (int k = 0; k < c.m; ++k) bcv.push_back(ph.bcs[i].value[k]);
  }
  if (bcv.empty()) bcv.push_back(0.0);
  if (c.bck.empty()) c.bck.push_back(0);
  const int F = 2 * c.D, P = c.p;
  c.conn.assign(static_cast<size_t>(c.E) * c.D * 2, int2{0, 0});
  c.fpart.assign(static_cast<size_t>(c.E) * c.D * 2, int2{-1, 0});
  for (int k = 0; k < c.E; ++k) {
    const int e = c.order[k];
    for (int dir = 0; dir < c.D; ++dir) {
      int splus = 1;
      if (c.second) splus = s.switch_plus[static_cast<size_t>(e) * c.D + dir] >= 0 ? 1 : -1;
      for (int side = 0; side < 2; ++side) {
        const int S = side ? splus : -splus;
        const int flag = S > 0 ? (1 << 24) : 0;
        const int lf = face_of(c.D, dir, side);
        const int fid = s.elem_face[static_cast<size_t>(e) * F + lf];
        if (fid < 0 || fid >= s.n_faces)
          throw ldg_error(LDG_ERR_CONFIG, "elem_face entry out of range for element " + std::to_string(e));
        int2& out = c.conn[(static_cast<size_t>(k) * c.D + dir) * 2 + side];
        if (s.face_elem_r[fid] < 0) {
          auto it = tag2bc.find(s.face_tag[fid]);
          if (it == tag2bc.end())
            throw ldg_error(LDG_ERR_CONFIG, "no boundary condition for boundary tag " +
                                                std::to_string(s.face_tag[fid]));
          out.x = -1 - it->second;
          out.y = flag;
          continue;
        }
        const bool is_left = s.face_elem_l[fid] == e && s.face_face_l[fid] == lf;
        const int oe = is_left ? s.face_elem_r[fid] : s.face_elem_l[fid];
        const int olf = is_left ? s.face_face_r[fid] : s.face_face_l[fid];
        const int code = s.face_orient[fid];
        auto nbr_node = [&](int line) {
          const int own = c.node_on_line(dir, line, side ? P : 0);
          if (c.D == 2) {
            const int kk = face_param_2d(P, lf, own);
            return face_node_2d(P, olf, code ? P - kk : kk);
          }
          const int a = line % c.np, b = line / c.np;
          int na = -1, nb = -1;
          if (is_left) {
            dihedral(code, a, b, P, na, nb);
          } else {
            for (int xx = 0; xx <= P && na < 0; ++xx)
              for (int yy = 0; yy <= P; ++yy) {
                int ra, rb;
                dihedral(code, xx, yy, P, ra, rb);
                if (ra == a && rb == b) {
                  na = xx;
                  nb = yy;
                  break;
                }
              }
          }
          return face_node_3d(P, olf, na, nb);
        };
        const int f00 = nbr_node(0);
        const int c1 = c.np > 1 ? nbr_node(1) - f00 : 0;
        const int c2 = c.D == 3 ? nbr_node(c.np) - f00 : 0;
        for (int line = 0; line < c.NL; ++line) {
          const int pred = f00 + c1 * (line % c.np) + c2 * (line / c.np);
          if (pred != nbr_node(line)) throw ldg_error(LDG_ERR_CONFIG, "non-affine face node map");
        }
        if (f00 < 0 || f00 > 255 || c1 < -128 || c1 > 127 || c2 < -128 || c2 > 127)
          throw ldg_error(LDG_ERR_CONFIG, "face node map out of packing range");
        out.x = oe;
        out.y = (f00 & 0xff) | ((c1 & 0xff) << 8) | ((c2 & 0xff) << 16) | flag;
        c.fpart[(static_cast<size_t>(k) * c.D + dir) * 2 + side] = int2{c.inv_order[oe], local_face_ds(c.D, olf)};
      }
    }
  }
  ck(cudaMalloc(&c.d_bcv, bcv.size() * sizeof(double)), "cudaMalloc bcv");
  ck(cudaMemcpy(c.d_bcv, bcv.data(), bcv.size() * sizeof(double), cudaMemcpyHostToDevice), "upload bcv");
  ck(cudaMalloc(&c.d_bck, c.bck.size() * sizeof(int32_t)), "cudaMalloc bck");
  ck(cudaMemcpy(c.d_bck, c.bck.data(), c.bck.size() * sizeof(int32_t), cudaMemcpyHostToDevice), "upload bck");
  ck(cudaMalloc(&c.d_conn, c.conn.size() * sizeof(int2)), "cudaMalloc conn");
  ck(cudaMemcpy(c.d_conn, c.conn.data(), c.conn.size() * sizeof(int2), cudaMemcpyHostToDevice),
     "upload conn");
}

// Makes the context's device current for the duration of an entry point
// (launch configuration, allocations and streams all belong to it) and
// restores the caller's device afterwards.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(const ldg_ctx* c) {
    if (!c || c->device < 0) return;
    int cur = 0;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != c->device && cudaSetDevice(c->device) == cudaSuccess) prev = cur;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

template <class F>
int guarded(ldg_ctx* c, F&& f) {
  DeviceGuard dg(c);
  try {
    return f();
  } catch (const ldg_error& ex) {
    if (c) c->err = ex.what();
    else g_create_err = ex.what();
    return ex.status;
  } catch (const std::exception& ex) {
    if (c) c->err = ex.what();
    else g_create_err = ex.what();
    return LDG_ERR_INVALID_ARGUMENT;
  }
}

// Completes a stream-ordered operation: surfaces launch errors and, when
// error synchronisation is on, waits and reports a physical-state failure
// recorded by any kernel (errors.hpp:10-18).
int finish(ldg_ctx* c, cudaError_t launch) {
  ck(launch, "kernel launch");
  if (!c->sync_errors) return LDG_OK;
  ck(cudaStreamSynchronize(c->stream), "stream synchronize");
  if (c->h_err->flag) {
    c->err_elem = c->h_err->elem;
    c->err_node = c->h_err->node;
    std::memcpy(c->err_state, c->h_err->state, sizeof(c->err_state));
    c->err = "physical state error: non-positive density or pressure (element " +
             std::to_string(c->err_elem) + ", node " + std::to_string(c->err_node) + ")";
    c->h_err->flag = 0;
    return LDG_ERR_PHYSICAL_STATE;
  }
  return LDG_OK;
}

// Device vectors are read with 16-byte vector / bulk-async loads: reject a
// misaligned pointer (e.g. a view at an odd element offset) instead of letting
// it fault the context.
void check_aligned(const void* p, const char* what) {
  if (reinterpret_cast<uintptr_t>(p) & 15u)
    throw ldg_error(LDG_ERR_INVALID_ARGUMENT, std::string(what) + " must be 16-byte aligned");
}

double* ensure(double*& p, size_t n) {
  if (!p) ck(cudaMalloc(&p, n * sizeof(double)), "cudaMalloc workspace");
  return p;
}

// ---- Krylov vector kernels.  Reductions are deterministic: fixed-grid block
// partial sums, then one block sums the partials in a fixed tree order.
constexpr int KR_THREADS = 256, KR_BLOCKS = 592;

__global__ void __launch_bounds__(KR_THREADS) k_dot_part(const double* __restrict__ a, const double* __restrict__ b,
                                                         size_t n, double* __restrict__ part) {
  __shared__ double sh[KR_THREADS];
  double s = 0.0;
  for (size_t i = static_cast<size_t>(blockIdx.x) * KR_THREADS + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * KR_THREADS)
    s += a[i] * b[i];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = KR_THREADS / 2; o > 0; o >>= 1) {
    if (static_cast<int>(threadIdx.x) < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}
__global__ void __launch_bounds__(KR_THREADS) k_dot_fin(const double* __restrict__ part, int np, double* out,
                                                        int root) {
  __shared__ double sh[KR_THREADS];
  double s = 0.0;
  for (int i = threadIdx.x; i < np; i += KR_THREADS) s += part[i];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = KR_THREADS / 2; o > 0; o >>= 1) {
    if (static_cast<int>(threadIdx.x) < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = root ? sqrt(sh[0]) : sh[0];
}
// y -= (*coef) x
__global__ void k_axpy_dev(double* __restrict__ y, const double* __restrict__ x, size_t n,
                           const double* __restrict__ coef) {
  const double a = *coef;
  for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    y[i] -= a * x[i];
}
// y += a x
__global__ void k_axpy(double* __restrict__ y, const double* __restrict__ x, size_t n, double a) {
  for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    y[i] += a * x[i];
}
// y = x / (*den)  (den > 0), or y = x / den_h when den == nullptr
__global__ void k_div(double* __restrict__ y, const double* __restrict__ x, size_t n, const double* den,
                      double den_h) {
  const double d = den ? *den : den_h;
  if (!(d > 0.0)) return;
  for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    y[i] = x[i] / d;
}
// GMRES: Givens update of Hessenberg column j on the device (one thread), so
// the host never waits for it.  st[0] = done (converged / lucky breakdown /
// non-finite), st[1] = iterations of the cycle, st[2] = non-finite flag; once
// done, the cycle's remaining (launched-ahead) iterations are ignored.
__global__ void k_gmres_givens(double* __restrict__ H, int mr, int j, double* __restrict__ cs,
                               double* __restrict__ sn, double* __restrict__ g, double tol, double* __restrict__ st) {
  if (st[0] != 0.0) return;
  double* col = H + static_cast<size_t>(j) * (mr + 1);
  const double hn = col[j + 1];
  if (!isfinite(hn)) {
    st[2] = 1.0;
    st[0] = 1.0;
    return;
  }
  for (int i = 0; i < j; ++i) {
    const double a0 = col[i], a1 = col[i + 1];
    col[i] = cs[i] * a0 + sn[i] * a1;
    col[i + 1] = -sn[i] * a0 + cs[i] * a1;
  }
  const double a0 = col[j], a1 = col[j + 1];
  const double den = hypot(a0, a1);
  cs[j] = den > 0.0 ? a0 / den : 1.0;
  sn[j] = den > 0.0 ? a1 / den : 0.0;
  col[j] = den;
  col[j + 1] = 0.0;
  g[j + 1] = -sn[j] * g[j];
  g[j] = cs[j] * g[j];
  st[1] = j + 1;
  if (fabs(g[j + 1]) <= tol || hn == 0.0) st[0] = 1.0;
}
__global__ void k_gmres_cycle_init(double* __restrict__ g, int mr, double beta, double* __restrict__ st) {
  for (int i = threadIdx.x; i <= mr; i += blockDim.x) g[i] = i == 0 ? beta : 0.0;
  if (threadIdx.x == 0) st[0] = st[1] = st[2] = 0.0;
}
// max |a_i|: block partials, then one block (deterministic)
__global__ void __launch_bounds__(KR_THREADS) k_amax_part(const double* __restrict__ a, size_t n,
                                                          double* __restrict__ part) {
  __shared__ double sh[KR_THREADS];
  double s = 0.0;
  for (size_t i = static_cast<size_t>(blockIdx.x) * KR_THREADS + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * KR_THREADS) {
    const double v = fabs(a[i]);
    s = (v > s || v != v) ? v : s;  // NaN propagates
  }
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = KR_THREADS / 2; o > 0; o >>= 1) {
    if (static_cast<int>(threadIdx.x) < o) {
      const double v = sh[threadIdx.x + o];
      if (v > sh[threadIdx.x] || v != v) sh[threadIdx.x] = v;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}
__global__ void __launch_bounds__(KR_THREADS) k_amax_fin(const double* __restrict__ part, int np, double* out) {
  __shared__ double sh[KR_THREADS];
  double s = 0.0;
  for (int i = threadIdx.x; i < np; i += KR_THREADS) s = (part[i] > s || part[i] != part[i]) ? part[i] : s;
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = KR_THREADS / 2; o > 0; o >>= 1) {
    if (static_cast<int>(threadIdx.x) < o) {
      const double v = sh[threadIdx.x + o];
      if (v > sh[threadIdx.x] || v != v) sh[threadIdx.x] = v;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0];
}
// us = U + dt (a0 K0 + a1 K1 + al Kc)   (stage state; nprev previous slopes)
__global__ void k_stage_state(double* __restrict__ us, const double* __restrict__ U, const double* __restrict__ K0,
                              const double* __restrict__ K1, const double* __restrict__ Kc, size_t n, double dt,
                              double a0, double a1, double al, int nprev) {
  for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    double sacc = 0.0;
    if (nprev > 0) sacc += a0 * K0[i];
    if (nprev > 1) sacc += a1 * K1[i];
    us[i] = U[i] + dt * (sacc + al * Kc[i]);
  }
}
// G = Fv - Kc (the Newton right-hand side -(K - F))
__global__ void k_rhs(double* __restrict__ g, const double* __restrict__ Kc, const double* __restrict__ Fv, size_t n) {
  for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    g[i] = -(Kc[i] - Fv[i]);
}
// U += dt (b0 K0 + b1 K1 + b2 K2)
__global__ void k_dirk_update(double* __restrict__ U, const double* __restrict__ K0, const double* __restrict__ K1,
                              const double* __restrict__ K2, size_t n, double dt, double b0, double b1, double b2) {
  for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    U[i] += dt * (b0 * K0[i] + b1 * K1[i] + b2 * K2[i]);
}
// RK4: us = U + f k ; final U += dt/6 (k1 + 2 k2 + 2 k3 + k4)
__global__ void k_rk_state(double* __restrict__ us, const double* __restrict__ U, const double* __restrict__ k,
                           size_t n, double f) {
  for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    us[i] = U[i] + f * k[i];
}
__global__ void k_rk4_update(double* __restrict__ U, const double* __restrict__ k1, const double* __restrict__ k2,
                             const double* __restrict__ k3, const double* __restrict__ k4, size_t n, double dt) {
  for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    U[i] += dt / 6.0 * (k1[i] + 2.0 * k2[i] + 2.0 * k3[i] + k4[i]);
}
__global__ void k_sub(double* __restrict__ r, const double* __restrict__ b, const double* __restrict__ t, size_t n) {
  for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    r[i] = b[i] - t[i];
}

}  // namespace

extern "C" {

const char* ldg_last_error(const ldg_ctx* c) { return c ? c->err.c_str() : g_create_err.c_str(); }

int ldg_create(const ldg_setup* s, const ldg_physics* ph, void* stream, ldg_ctx** out) {
  return guarded(nullptr, [&]() -> int {
    if (!s || !ph || !out) throw ldg_error(LDG_ERR_INVALID_ARGUMENT, "null argument");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
      throw ldg_error(LDG_ERR_CUDA, "no CUDA device: the B200 hot path has no CPU fallback");
    auto c = std::make_unique<ldg_ctx>();
    ck(cudaGetDevice(&c->device), "cudaGetDevice");
    c->D = s->dim;
    c->p = s->p;
    c->np = c->p + 1;
    c->nq = s->n_quad;
    c->E = s->n_elems;
    if (c->D != 2 && c->D != 3) throw ldg_error(LDG_ERR_CONFIG, "dim must be 2 or 3");
    if (c->E < 1) throw ldg_error(LDG_ERR_CONFIG, "mesh has no elements");
    if (c->nq != (3 * c->p + 2) / 2) throw ldg_error(LDG_ERR_CONFIG, "n_quad must be (3p+2)/2");
    if (ph->c22 != 0.0)
      throw ldg_error(LDG_ERR_CONFIG, "residual_primal requires C22 = 0 (SPEC.md:250-252)");
    c->npe = c->D == 2 ? c->np * c->np : c->np * c->np * c->np;
    c->NL = c->D == 2 ? c->np : c->np * c->np;
    c->kind = ph->kind;
    c->riemann = ph->riemann;
    c->m = ph->kind == LDG_POISSON ? 1 : c->D + 2;
    c->has_inv = ph->kind != LDG_POISSON;
    c->second = ph->kind == LDG_POISSON || (ph->kind == LDG_NAVIER_STOKES && ph->mu != 0.0);
    c->vis_u = c->second && ph->kind == LDG_NAVIER_STOKES;
    // Navier-Stokes with mu = 0 is the first-order Euler operator.
    c->ph = ph->kind == LDG_POISSON ? ldg::PH_POISSON : (c->second ? ldg::PH_NS : ldg::PH_EULER);
    const int ri = c->ph == ldg::PH_POISSON ? 0 : ph->riemann;
    c->ops = find_ops(c->D, c->p, c->ph, ri);
    if (!c->ops)
      throw ldg_error(LDG_ERR_CONFIG, "no sm_100a kernel instantiation for dim=" + std::to_string(c->D) +
                                          " p=" + std::to_string(c->p));
    if (c->second && !s->switch_plus)
      throw ldg_error(LDG_ERR_CONFIG, "second-order physics needs the LDG switch table");
    c->c11 = ph->c11;
    c->c11bd = ph->c11_bd;
    c->stream = static_cast<cudaStream_t>(stream);

    // Basis folding.
    const int np = c->np, nq = c->nq;
    const std::vector<double> minv = spd_inverse(s->mass, np);
    c->phi.assign(s->phi_at_quad, s->phi_at_quad + np * nq);
    c->dq.assign(np * nq, 0.0);
    for (int i = 0; i < np; ++i)
      for (int q = 0; q < nq; ++q) {
        double acc = 0.0;
        for (int kk = 0; kk < np; ++kk) acc += minv[i * np + kk] * s->dphi_at_quad[kk * nq + q];
        c->dq[i * nq + q] = -acc * s->quad_weights[q];
      }
    c->mi.assign(np * 2, 0.0);
    for (int i = 0; i < np; ++i) {
      c->mi[i * 2 + 0] = minv[i * np + 0];
      c->mi[i * 2 + 1] = minv[i * np + c->p];
    }
    c->cc.assign(np * np * nq, 0.0);
    for (int i = 0; i < np; ++i)
      for (int t = 0; t < np; ++t)
        for (int q = 0; q < nq; ++q) c->cc[(i * np + t) * nq + q] = c->dq[i * nq + q] * c->phi[t * nq + q];

    // Processing order (the Jacobian store and the metric are laid out in it).
    c->order = processing_order(*s, c->D, c->npe);
    c->inv_order.resize(c->E);
    for (int k = 0; k < c->E; ++k) c->inv_order[c->order[k]] = k;
    ck(cudaMalloc(&c->d_order, c->E * sizeof(int32_t)), "cudaMalloc order");
    ck(cudaMemcpy(c->d_order, c->order.data(), c->E * sizeof(int32_t), cudaMemcpyHostToDevice), "upload order");
    ck(cudaMalloc(&c->d_inv_order, c->E * sizeof(int32_t)), "cudaMalloc inv_order");
    ck(cudaMemcpy(c->d_inv_order, c->inv_order.data(), c->E * sizeof(int32_t), cudaMemcpyHostToDevice),
       "upload inv_order");

    build_connectivity(*c, *s, *ph);
    // boundary faces (processing order) for boundary functions
    {
      const int F = 2 * c->D;
      c->bface_of.assign(static_cast<size_t>(c->E) * F, -1);
      c->has_coords = s->node_coords != nullptr;
      for (int i = 0; i < ph->n_bc; ++i) c->bc_tag.push_back(ph->bcs[i].tag);
      for (int i = 0; i < ph->n_bc; ++i)
        for (int k2 = 0; k2 < c->m; ++k2) c->bcv_host.push_back(ph->bcs[i].value[k2]);
      for (int k = 0; k < c->E; ++k)
        for (int ds = 0; ds < F; ++ds) {
          const int2 cx = c->conn[static_cast<size_t>(k) * F + ds];
          if (cx.x >= 0) continue;
          c->bface_of[static_cast<size_t>(k) * F + ds] = static_cast<int32_t>(c->bface_tag.size());
          c->bface_tag.push_back(-1 - cx.x);  // boundary index
          const int dir = ds >> 1, side = ds & 1, e = c->order[k];
          for (int line = 0; line < c->NL; ++line) {
            // own end node of the line (node_on_line): position 0 or p along dir
            int base;
            if (c->D == 2) base = dir == 0 ? c->np * line : line;
            else {
              const int t1 = dir == 0 ? 1 : 0, t2 = dir == 2 ? 1 : 2;
              const int st[3] = {1, c->np, c->np * c->np};
              base = (line % c->np) * st[t1] + (line / c->np) * st[t2];
            }
            const int stride = dir == 0 ? 1 : (dir == 1 ? c->np : c->np * c->np);
            const int nd = base + (side ? c->p : 0) * stride;
            for (int d = 0; d < c->D; ++d)
              c->bface_x.push_back(c->has_coords ? s->node_coords[(static_cast<size_t>(e) * c->npe + nd) * c->D + d]
                                                 : 0.0);
          }
        }
    }

    // Metric in processing order, 1/J precomputed.
    const ldg::Ops& o = *c->ops;
    std::vector<double> met(static_cast<size_t>(c->E) * o.METP, 0.0);
    for (int k = 0; k < c->E; ++k) {
      const size_t e = c->order[k];
      double* dst = &met[static_cast<size_t>(k) * o.METP];
      std::memcpy(dst, s->nvec_quad + e * o.MET_NV, o.MET_NV * sizeof(double));
      std::memcpy(dst + o.MET_NV, s->normal_end + e * o.MET_NE, o.MET_NE * sizeof(double));
      for (int n = 0; n < c->npe; ++n) {
        const double J = s->jac_at_nodes[e * c->npe + n];
        if (!(J > 0.0)) throw ldg_error(LDG_ERR_CONFIG, "non-positive mapping Jacobian");
        dst[o.MET_NV + o.MET_NE + n] = 1.0 / J;
      }
    }
    ck(cudaMalloc(&c->d_metric, met.size() * sizeof(double)), "cudaMalloc metric");
    ck(cudaMemcpy(c->d_metric, met.data(), met.size() * sizeof(double), cudaMemcpyHostToDevice),
       "upload metric");
    ck(cudaHostAlloc(&c->h_err, sizeof(ldg::DevError), cudaHostAllocMapped), "cudaHostAlloc error word");
    std::memset(c->h_err, 0, sizeof(ldg::DevError));
    ck(cudaHostGetDevicePointer(&c->d_err, c->h_err, 0), "map error word");

    ldg::DevCtx& d = c->dc;
    d.stream = c->stream;
    ck(cudaStreamCreateWithFlags(&c->cs_in, cudaStreamNonBlocking), "create upload stream");
    ck(cudaStreamCreateWithFlags(&c->cs_out, cudaStreamNonBlocking), "create download stream");
    for (cudaEvent_t* ev : {&c->ev_in, &c->ev_k, &c->ev_free_hu, &c->ev_free_hu2, &c->ev_free_hx, &c->ev_out_r,
                            &c->ev_out_y, &c->ev_join, &c->ev_mv_free[0], &c->ev_mv_free[1], &c->ev_mv_out[0],
                            &c->ev_mv_out[1]}) {
      ck(cudaEventCreateWithFlags(ev, cudaEventDisableTiming), "create event");
      ck(cudaEventRecord(*ev, c->stream), "record event");  // completed: nothing to wait for yet
    }
    d.phi = c->phi.data();
    d.dq = c->dq.data();
    d.mi = c->mi.data();
    d.cc = c->cc.data();
    d.pp.gamma = ph->gamma;
    d.pp.mu = ph->mu;
    d.pp.kap = ph->prandtl > 0.0 ? ph->mu * ph->gamma / ph->prandtl : 0.0;
    d.pp.c11 = ph->c11;
    d.pp.c11bd = ph->c11_bd * c->p * c->p;
    d.order = c->d_order;
    d.metric = c->d_metric;
    d.conn = c->d_conn;
    d.bcv = c->d_bcv;
    d.bck = c->d_bck;
    d.source = nullptr;
    d.err = c->d_err;
    d.E = c->E;
    d.inv_order = c->d_inv_order;
    {
      build_face_sharing(*c, o.chunk_elems(c->E), true);
      d.fpart = c->d_fpart;
      d.owned = c->d_owned;
      d.owned_off = c->owned_off.data();
      d.bspec = c->d_bspec;
      d.bspec_off = c->bspec_off.data();
    }

    d.launches = &c->launches;
    *out = c.release();
    return LDG_OK;
  });
}

void ldg_destroy(ldg_ctx* c) {
  DeviceGuard dg(c);  // frees on the context's device
  delete c;
}

int ldg_last_error_state(const ldg_ctx* c, int32_t* elem, int32_t* node, double* state) {
  if (!c) return LDG_ERR_INVALID_ARGUMENT;
  if (elem) *elem = c->err_elem;
  if (node) *node = c->err_node;
  if (state) std::memcpy(state, c->err_state, sizeof(double) * c->m);
  return LDG_OK;
}
int ldg_components(const ldg_ctx* c) { return c->m; }
int64_t ldg_num_dofs(const ldg_ctx* c) { return static_cast<int64_t>(c->nU()); }
int64_t ldg_kernel_launches(const ldg_ctx* c) { return c->launches; }
int64_t ldg_jacobian_bytes(const ldg_ctx* c) {
  return static_cast<int64_t>((c->n11 + c->n12 + c->n21) * sizeof(double));
}
int ldg_set_option(ldg_ctx* c, int option, int64_t value) {
  return guarded(c, [&]() -> int {
    if (option == LDG_OPT_SPMV_ROW_ORDER) {
      if (value < 0 || value > 2) throw ldg_error(LDG_ERR_INVALID_ARGUMENT, "row order must be 0, 1 or 2");
      c->dc.spmv_order = static_cast<int>(value);
    } else if (option == LDG_OPT_ZERO_COPY) {
      if (value != 0 && value != 1) throw ldg_error(LDG_ERR_INVALID_ARGUMENT, "zero copy must be 0 or 1");
      c->zero_copy = value != 0;
    } else {
      throw ldg_error(LDG_ERR_INVALID_ARGUMENT, "unknown option " + std::to_string(option));
    }
    return LDG_OK;
  });
}
int ldg_set_sync_errors(ldg_ctx* c, int on) {
  c->sync_errors = on != 0;
  return LDG_OK;
}
int ldg_synchronize(ldg_ctx* c) {
  return guarded(c, [&]() -> int {
    // join the asynchronous host variants' copy streams into the context stream
    ck(cudaEventRecord(c->ev_join, c->cs_in), "record join");
    ck(cudaStreamWaitEvent(c->stream, c->ev_join, 0), "join uploads");
    ck(cudaEventRecord(c->ev_join, c->cs_out), "record join");
    ck(cudaStreamWaitEvent(c->stream, c->ev_join, 0), "join downloads");
    const bool was = c->sync_errors;
    c->sync_errors = true;
    const int st = finish(c, cudaSuccess);
    c->sync_errors = was;
    return st;
  });
}

int ldg_set_source(ldg_ctx* c, const double* S) {
  return guarded(c, [&]() -> int {
    if (!S) {
      cudaFree(c->d_source);
      c->d_source = nullptr;
    } else {
      ensure(c->d_source, c->nU());
      ck(cudaMemcpy(c->d_source, S, c->nU() * sizeof(double), cudaMemcpyHostToDevice), "upload source");
    }
    c->dc.source = c->d_source;
    return LDG_OK;
  });
}

namespace {
// Boundary functions: (re)evaluate at the boundary end nodes when registered
// data changed or t differs from the last evaluation, upload, point the
// kernels at it (DevCtx::bface / bvals); none registered -> constant data.
void refresh_boundary(ldg_ctx* c, double t) {
  if (c->bfun.empty()) {
    c->dc.bface = nullptr;
    c->dc.bvals = nullptr;
    return;
  }
  if (!c->bfun_dirty && t == c->bfun_t && c->dc.bface) return;
  const size_t nf = c->bface_tag.size();
  const int NL = c->NL, m = c->m, D = c->D;
  std::vector<double> h(std::max<size_t>(1, nf * NL * m));
  for (size_t f = 0; f < nf; ++f) {
    const int bc = c->bface_tag[f];
    auto it = c->bfun.find(c->bc_tag[bc]);
    for (int line = 0; line < NL; ++line) {
      double* out = &h[(f * NL + line) * m];
      if (it == c->bfun.end()) {
        for (int k = 0; k < m; ++k) out[k] = c->bcv_host[static_cast<size_t>(bc) * m + k];
      } else {
        it->second.first(it->second.second, &c->bface_x[(f * NL + line) * D], t, out);
      }
    }
  }
  if (!c->d_bface) {
    ck(cudaMalloc(&c->d_bface, c->bface_of.size() * sizeof(int32_t)), "cudaMalloc bface");
    ck(cudaMemcpy(c->d_bface, c->bface_of.data(), c->bface_of.size() * sizeof(int32_t), cudaMemcpyHostToDevice),
       "upload bface");
    ck(cudaMalloc(&c->d_bvals, h.size() * sizeof(double)), "cudaMalloc bvals");
  }
  // (stream-ordered: kernels already queued read the previous values first)
  ck(cudaMemcpyAsync(c->d_bvals, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream),
     "upload boundary data");
  ck(cudaStreamSynchronize(c->stream), "stream synchronize");  // h is a local buffer
  c->dc.bface = c->d_bface;
  c->dc.bvals = c->d_bvals;
  c->bfun_t = t;
  c->bfun_dirty = false;
}
}  // namespace

int ldg_set_boundary_function(ldg_ctx* c, int32_t tag, ldg_bc_fn fn, void* user) {
  return guarded(c, [&]() -> int {
    if (std::find(c->bc_tag.begin(), c->bc_tag.end(), tag) == c->bc_tag.end())
      throw ldg_error(LDG_ERR_CONFIG, "no boundary condition with tag " + std::to_string(tag));
    if (fn && !c->has_coords)
      throw ldg_error(LDG_ERR_CONFIG, "boundary functions need ldg_setup.node_coords");
    if (fn) c->bfun[tag] = {fn, user};
    else c->bfun.erase(tag);
    c->bfun_dirty = true;
    return LDG_OK;
  });
}

int ldg_gradient(ldg_ctx* c, const double* U, double t, double* Q) {
  return guarded(c, [&]() -> int {
    check_aligned(U, "U");
    check_aligned(Q, "Q");
    refresh_boundary(c, t);
    if (!c->second) throw ldg_error(LDG_ERR_CONFIG, "gradient_residual needs second-order physics");
    return finish(c, c->ops->gradient(c->dc, U, Q));
  });
}

int ldg_residual_uq(ldg_ctx* c, const double* U, const double* Q, double t, double* R) {
  return guarded(c, [&]() -> int {
    check_aligned(U, "U");
    check_aligned(R, "R");
    if (c->second) check_aligned(Q, "Q");
    refresh_boundary(c, t);
    if (!c->second) return finish(c, c->ops->residual(c->dc, U, nullptr, R));
    return finish(c, c->ops->residual(c->dc, U, Q, R));
  });
}

int ldg_residual(ldg_ctx* c, const double* U, double t, double* R, double* Q) {
  return guarded(c, [&]() -> int {
    check_aligned(U, "U");
    check_aligned(R, "R");
    if (Q) check_aligned(Q, "Q");
    refresh_boundary(c, t);
    if (!c->second) return finish(c, c->ops->residual(c->dc, U, nullptr, R));
    double* q = Q ? Q : ensure(c->d_Q, c->nQ());
    ck(c->ops->gradient(c->dc, U, q), "gradient launch");
    return finish(c, c->ops->residual(c->dc, U, q, R));
  });
}

namespace {
// Assembly at (U, Q): Q = D(U) already on the device (second-order physics),
// or computed here when q_given is null.
int assemble_at(ldg_ctx* c, const double* U, const double* q_given, double t) {
  refresh_boundary(c, t);
  const ldg::Ops& o = *c->ops;
  if (o.jac_smem > 227 * 1024)
    throw ldg_error(LDG_ERR_CONFIG, "Jacobian tile of this configuration exceeds shared memory (" +
                                        std::to_string(o.jac_smem) + " B)");
  const size_t rows = static_cast<size_t>(c->E) * c->npe;
  if (!c->d_K11) {
    c->n11 = rows * o.NS11 * o.B11;
    ck(cudaMalloc(&c->d_K11, c->n11 * sizeof(double) + 64), "cudaMalloc K11");  // +64: tile loads round to 16 B
    if (c->second) {
      c->n12 = rows * o.NS12 * o.B12;
      c->n21 = rows * o.NS12 * c->D;
      ck(cudaMalloc(&c->d_K12, c->n12 * sizeof(double) + 64), "cudaMalloc K12");  // +64: tile loads round to 16 B
      ck(cudaMalloc(&c->d_K21, c->n21 * sizeof(double) + 64), "cudaMalloc K21");  // +64: tile loads round to 16 B
    }
  }
  const double* q = nullptr;
  if (c->second) {
    if (q_given) {
      q = q_given;
    } else {
      q = ensure(c->d_Q, c->nQ());
      ck(o.gradient(c->dc, U, c->d_Q), "gradient launch");
    }
    // K21 is U- and t-independent: assembled once.
    if (!c->k21_valid) {
      ck(o.k21(c->dc, c->d_K21), "K21 launch");
      c->k21_valid = true;
    }
  }
  ensure(c->d_SE, o.scratch_elems(c->E));
  // a new Jacobian invalidates the block-Jacobi factors built from the old one
  c->pc_valid = false;
  const int st = finish(c, o.jacobian(c->dc, U, q, c->d_SE, c->d_K11, c->d_K12));
  c->jac_valid = st == LDG_OK;
  return st;
}
}  // namespace

int ldg_jacobian_assemble(ldg_ctx* c, const double* U, double t) {
  return guarded(c, [&]() -> int {
    check_aligned(U, "U");
    return assemble_at(c, U, nullptr, t);
  });
}

int ldg_jacobian_assemble_q(ldg_ctx* c, const double* U, const double* Q, double t) {
  return guarded(c, [&]() -> int {
    if (c->second && !Q) throw ldg_error(LDG_ERR_INVALID_ARGUMENT, "Q required for second-order physics");
    check_aligned(U, "U");
    if (Q) check_aligned(Q, "Q");
    return assemble_at(c, U, c->second ? Q : nullptr, t);
  });
}

int ldg_pattern_info_get(const ldg_ctx* cc, int which, ldg_pattern_info* info) {
  ldg_ctx* c = const_cast<ldg_ctx*>(cc);
  return guarded(c, [&]() -> int {
    if (which < 0 || which > 2 || (which != LDG_K11 && !c->second))
      throw ldg_error(LDG_ERR_INVALID_ARGUMENT, "matrix not available for this physics");
    int64_t nnzb = 0;
    std::vector<int64_t> cols;
    for (int k = 0; k < c->E; ++k)
      for (int nd = 0; nd < c->npe; ++nd) {
        cols.clear();
        for (int sl = 0; sl < c->nslots(which); ++sl) {
          bool pres;
          const int64_t col = c->slot_col(which, k, nd, sl, pres);
          if (pres && col >= 0) cols.push_back(col);
        }
        std::sort(cols.begin(), cols.end());
        nnzb += std::unique(cols.begin(), cols.end()) - cols.begin();
      }
    info->n_rows = static_cast<int64_t>(c->E) * c->npe;
    info->nnzb = nnzb;
    info->block_rows = which == LDG_K21 ? c->m * c->D : c->m;
    info->block_cols = which == LDG_K12 ? c->m * c->D : c->m;
    return LDG_OK;
  });
}

// Export of rows of the given reference elements (all if elems == NULL).
int ldg_export_blocks_subset(ldg_ctx* c, int which, const int32_t* elems, int32_t n_elems,
                             int64_t* rows, int64_t* cols, double* vals, int64_t* nnzb_out) {
  return guarded(c, [&]() -> int {
    if (!c->jac_valid) throw ldg_error(LDG_ERR_SOLVER, "Jacobian not assembled");
    if (which < 0 || which > 2 || (which != LDG_K11 && !c->second))
      throw ldg_error(LDG_ERR_INVALID_ARGUMENT, "matrix not available for this physics");
    const ldg::Ops& o = *c->ops;
    const int NT = o.NT, NS = c->nslots(which);
    const int bsz = which == LDG_K11 ? o.B11 : (which == LDG_K12 ? o.B12 : c->D);
    const double* dsrc = which == LDG_K11 ? c->d_K11 : (which == LDG_K12 ? c->d_K12 : c->d_K21);
    const int br = which == LDG_K21 ? c->m * c->D : c->m;
    const int bc = which == LDG_K12 ? c->m * c->D : c->m;
    const size_t per_elem = static_cast<size_t>(c->npe) * NS * bsz;
    std::vector<int32_t> list;
    if (elems) list.assign(elems, elems + n_elems);
    else {
      list.resize(c->E);
      for (int e = 0; e < c->E; ++e) list[e] = e;
    }
    std::vector<double> chunk(per_elem), metk(o.METP);
    int64_t pos = 0;
    std::vector<std::pair<int64_t, int>> cl;
    for (const int32_t e : list) {
      if (e < 0 || e >= c->E) throw ldg_error(LDG_ERR_INVALID_ARGUMENT, "element out of range");
      const int k = c->inv_order[e];
      if (vals)
        ck(cudaMemcpy(chunk.data(), dsrc + static_cast<size_t>(k) * per_elem, per_elem * sizeof(double),
                      cudaMemcpyDeviceToHost),
           "download Jacobian");
      if (vals && which == LDG_K21 && c->dc.noslip)
        ck(cudaMemcpy(metk.data(), c->d_metric + static_cast<size_t>(k) * o.METP, o.METP * sizeof(double),
                      cudaMemcpyDeviceToHost),
           "download metric");
      for (int nd = 0; nd < c->npe; ++nd) {
        const int tile = nd / NT, r = nd % NT;
        cl.clear();
        for (int sl = 0; sl < NS; ++sl) {
          bool pres;
          const int64_t col = c->slot_col(which, k, nd, sl, pres);
          if (pres && col >= 0) cl.emplace_back(col, sl);
        }
        std::sort(cl.begin(), cl.end());
        for (size_t a = 0; a < cl.size();) {
          size_t b = a;
          while (b < cl.size() && cl[b].first == cl[a].first) ++b;
          if (rows) rows[pos] = static_cast<int64_t>(e) * c->npe + nd;
          if (cols) cols[pos] = cl[a].first;
          if (vals) {
            double* blk = vals + pos * br * bc;
            std::fill(blk, blk + br * bc, 0.0);
            for (size_t z = a; z < b; ++z) {
              const int sl = cl[z].second;
              // store: per (tile, slot) a bsz*NT run laid out [block row][row r][column]
              const int scol = which == LDG_K11 ? c->m : (which == LDG_K12 ? o.MD : c->D);
              auto at = [&](int ab) {
                const int aa = ab / scol, bb = ab % scol;
                return chunk[(static_cast<size_t>(tile) * NS + sl) * bsz * NT + (static_cast<size_t>(aa) * NT + r) * scol + bb];
              };
              if (which == LDG_K11) {
                for (int ab = 0; ab < bsz; ++ab) blk[ab] += at(ab);
              } else if (which == LDG_K12) {
                const int a0 = c->ph == ldg::PH_NS ? 1 : 0;
                for (int aa = 0; aa < o.R12; ++aa)
                  for (int bb = 0; bb < o.MD; ++bb) blk[(aa + a0) * bc + bb] += at(aa * o.MD + bb);
              } else {
                for (int cc2 = 0; cc2 < c->m; ++cc2)
                  for (int d = 0; d < c->D; ++d) blk[(cc2 * c->D + d) * bc + cc2] += at(d);
              }
            }
            if (which == LDG_K21 && c->dc.noslip) {
              // wall terms (k21_wall_terms): density and energy rows of no-slip ends
              for (int dir = 0; dir < c->D; ++dir)
                for (int side = 0; side < 2; ++side) {
                  const int2& cx = c->cn(k, dir, side);
                  if (cx.x >= 0 || c->bck[-1 - cx.x] != LDG_BC_NO_SLIP_ADIABATIC) continue;
                  int line, lp;
                  c->line_of(dir, nd, line, lp);
                  const int xs[3] = {nd % c->np, (nd / c->np) % c->np, nd / (c->np * c->np)};
                  const int st[3] = {1, c->np, c->np * c->np};
                  const int endn = nd + ((side ? c->p : 0) - xs[dir]) * st[dir];
                  if (static_cast<int64_t>(e) * c->npe + endn != cl[a].first) continue;
                  const double invJ = metk[o.MET_NV + o.MET_NE + nd];
                  const double mi = c->mi[lp * 2 + side];
                  for (int d = 0; d < c->D; ++d) {
                    const double cf = invJ * (mi * metk[o.MET_NV + ((dir * 2 + side) * c->NL + line) * c->D + d]);
                    blk[(0 * c->D + d) * bc + 0] += cf;
                    blk[((c->m - 1) * c->D + d) * bc + c->m - 1] += cf;
                  }
                }
            }
          }
          ++pos;
          a = b;
        }
      }
    }
    if (nnzb_out) *nnzb_out = pos;
    return LDG_OK;
  });
}

int ldg_export_blocks(ldg_ctx* c, int which, int64_t* rows, int64_t* cols, double* vals) {
  return ldg_export_blocks_subset(c, which, nullptr, 0, rows, cols, vals, nullptr);
}

// Structural scalar entries of a node block (a, b): K11 all m x m; K12 all
// but the Navier-Stokes density row (its flux has no viscous part); K21 the
// component diagonal (c, d) <- c.  Shared by the triplet and CSV writers.
static bool scalar_structural(const ldg_ctx* c, int which, int a, int b) {
  if (which == LDG_K12) return !(c->ph == ldg::PH_NS && a == 0);
  if (which == LDG_K21) return a / c->D == b;
  return true;
}

// Matrix export as text triplets `i j value`, one structural
// scalar entry per line, 0-based indices in the reference numbering (rows:
// DOF (e*npe+node)*m+c, or the Q index for K21; columns likewise), rows in
// ascending order, values printed with 17 significant digits.  Streams the
// store element by element (no full host copy).
int ldg_write_triplets(ldg_ctx* c, int which, const char* path) {
  return guarded(c, [&]() -> int {
    if (!path) throw ldg_error(LDG_ERR_INVALID_ARGUMENT, "path is NULL");
    if (!c->jac_valid) throw ldg_error(LDG_ERR_SOLVER, "Jacobian not assembled");
    if (which < 0 || which > 2 || (which != LDG_K11 && !c->second))
      throw ldg_error(LDG_ERR_INVALID_ARGUMENT, "matrix not available for this physics");
    FILE* f = std::fopen(path, "w");
    if (!f) throw ldg_error(LDG_ERR_CONFIG, std::string("cannot write '") + path + "'");
    const int br = which == LDG_K21 ? c->m * c->D : c->m;
    const int bc = which == LDG_K12 ? c->m * c->D : c->m;
    const size_t cap = static_cast<size_t>(c->npe) * c->nslots(which);
    std::vector<int64_t> rows(cap), cols(cap);
    std::vector<double> vals(cap * br * bc);
    std::vector<char> buf(1 << 20);
    std::setvbuf(f, buf.data(), _IOFBF, buf.size());
    int st = LDG_OK;
    for (int32_t e = 0; e < c->E && st == LDG_OK; ++e) {
      int64_t nb = 0;
      st = ldg_export_blocks_subset(c, which, &e, 1, rows.data(), cols.data(), vals.data(), &nb);
      if (st != LDG_OK) break;
      // the export is sorted by (row node, col node); emit scalar rows in order
      for (int64_t z0 = 0; z0 < nb;) {
        int64_t z1 = z0;
        while (z1 < nb && rows[z1] == rows[z0]) ++z1;
        for (int a = 0; a < br; ++a)
          for (int64_t z = z0; z < z1; ++z)
            for (int b = 0; b < bc; ++b)
              if (scalar_structural(c, which, a, b))
                std::fprintf(f, "%lld %lld %.17g\n", static_cast<long long>(rows[z] * br + a),
                             static_cast<long long>(cols[z] * bc + b), vals[(z * br + a) * bc + b]);
        z0 = z1;
      }
    }
    if (std::fclose(f) != 0 && st == LDG_OK) throw ldg_error(LDG_ERR_CONFIG, std::string("write failed: ") + path);
    return st;
  });
}

// Sparsity summary CSV `p,avg_cols_per_block_row,nnz` (the
// `linedg sparsity` Table-1 oracle): node-columns per node row
// (the Table-1 quantity) and structural scalar nonzeros.
// append != 0 adds a row to an existing file (header only when it is empty).
int ldg_write_sparsity_csv(ldg_ctx* c, int which, const char* path, int append) {
  return guarded(c, [&]() -> int {
    if (!path) throw ldg_error(LDG_ERR_INVALID_ARGUMENT, "path is NULL");
    ldg_pattern_info info;
    int st = ldg_pattern_info_get(c, which, &info);
    if (st != LDG_OK) return st;
    int per = 0;
    for (int a = 0; a < info.block_rows; ++a)
      for (int b = 0; b < info.block_cols; ++b) per += scalar_structural(c, which, a, b);
    FILE* f = std::fopen(path, append ? "a" : "w");
    if (!f) throw ldg_error(LDG_ERR_CONFIG, std::string("cannot write '") + path + "'");
    if (std::ftell(f) == 0) std::fprintf(f, "p,avg_cols_per_block_row,nnz\n");
    std::fprintf(f, "%d,%.6f,%lld\n", c->p, static_cast<double>(info.nnzb) / static_cast<double>(info.n_rows),
                 static_cast<long long>(info.nnzb * per));
    if (std::fclose(f) != 0) throw ldg_error(LDG_ERR_CONFIG, std::string("write failed: ") + path);
    return LDG_OK;
  });
}

int ldg_bsr_spmv(ldg_ctx* c, int which, const double* x, double* y) {
  return guarded(c, [&]() -> int {
    check_aligned(x, "x");
    check_aligned(y, "y");
    if (!c->jac_valid) throw ldg_error(LDG_ERR_SOLVER, "Jacobian not assembled");
    const ldg::Ops& o = *c->ops;
    if (which == LDG_K11) return finish(c, o.spmv11(c->dc, c->d_K11, x, y));
    if (!c->second) throw ldg_error(LDG_ERR_INVALID_ARGUMENT, "matrix not available for this physics");
    if (which == LDG_K12) return finish(c, o.spmv12(c->dc, c->d_K12, x, y));
    if (which == LDG_K21) return finish(c, o.spmv21(c->dc, c->d_K21, x, y));
    throw ldg_error(LDG_ERR_INVALID_ARGUMENT, "unknown matrix");
  });
}

int ldg_split_matvec(ldg_ctx* c, double adt, const double* v, double* y) {
  return guarded(c, [&]() -> int {
    check_aligned(v, "v");
    check_aligned(y, "y");
    if (!c->jac_valid) throw ldg_error(LDG_ERR_SOLVER, "Jacobian not assembled");
    const ldg::Ops& o = *c->ops;
    const double* w = nullptr;
    if (c->second) {
      ensure(c->d_w, c->nQ());
      ck(o.spmv21(c->dc, c->d_K21, v, c->d_w), "K21 launch");
      w = c->d_w;
    }
    return finish(c, o.split(c->dc, c->d_K11, c->d_K12, v, w, adt, y));
  });
}

// ----------------------------------------- block-Jacobi preconditioner + GMRES
//
namespace {
// preconditioner application of the built kind (element-block LU / inverse or line-ADI)
cudaError_t pc_apply_any(ldg_ctx* c, const double* r, double* z) {
  const ldg::Ops& o = *c->ops;
  return c->pc_adi ? o.pc_line_apply(c->dc, c->d_pcLU, c->d_pcPiv, r, z)
                   : o.pc_apply(c->dc, c->d_pcLU, c->d_pcPiv, r, z);
}
}  // namespace

int ldg_precond_build(ldg_ctx* c, double alpha_dt) {
  return guarded(c, [&]() -> int {
    if (!c->jac_valid) throw ldg_error(LDG_ERR_SOLVER, "Jacobian not assembled");
    const ldg::Ops& o = *c->ops;
    // mode 0: element-block LU up to 128 unknowns per element, line-ADI above
    // (3-D p >= 2); 1: explicit element-block inverses; 2: line-ADI
    const bool adi = c->pc_mode == 2 || (c->pc_mode == 0 && o.pc_ne <= 0);
    if (!adi && o.pc_ne <= 0)
      throw ldg_error(LDG_ERR_CONFIG, "element-block preconditioner: element blocks above 128 unknowns "
                                      "(3-D p >= 2) use the line-ADI mode");
    if (adi && o.pc_line_nb <= 0)
      throw ldg_error(LDG_ERR_CONFIG, "line-ADI preconditioner not available for this configuration");
    size_t nlu, npiv;
    if (adi) {
      const size_t nb = static_cast<size_t>(o.pc_line_nb), blocks = static_cast<size_t>(c->E) * c->D * c->NL;
      nlu = blocks * nb * nb;
      npiv = blocks * nb;
    } else {
      const size_t ne = static_cast<size_t>(o.pc_ne);
      nlu = static_cast<size_t>(c->E) * ne * ne;
      npiv = static_cast<size_t>(c->E) * ne;
    }
    if (nlu != c->pc_nlu || npiv != c->pc_npiv) {
      cudaFree(c->d_pcLU);
      cudaFree(c->d_pcPiv);
      c->d_pcLU = nullptr;
      c->d_pcPiv = nullptr;
      c->pc_nlu = c->pc_npiv = 0;
      size_t fr = 0, tot = 0;
      ck(cudaMemGetInfo(&fr, &tot), "cudaMemGetInfo");
      const size_t need = nlu * sizeof(double) + npiv * sizeof(int32_t);
      if (need + (64u << 20) > fr)
        throw ldg_error(LDG_ERR_CONFIG, std::string(adi ? "line-ADI" : "element-block") + " preconditioner needs " +
                                            std::to_string(need >> 20) + " MiB of factors, " +
                                            std::to_string(fr >> 20) + " MiB of device memory free");
      ck(cudaMalloc(&c->d_pcLU, nlu * sizeof(double)), "cudaMalloc LU");
      ck(cudaMalloc(&c->d_pcPiv, npiv * sizeof(int32_t)), "cudaMalloc piv");
      c->pc_nlu = nlu;
      c->pc_npiv = npiv;
    }
    if (!c->d_pcbad) ck(cudaMalloc(&c->d_pcbad, sizeof(int)), "cudaMalloc flag");
    ck(cudaMemsetAsync(c->d_pcbad, 0xff, sizeof(int), c->stream), "reset flag");
    c->pc_valid = false;
    if (adi)
      ck(o.pc_line_build(c->dc, c->d_K11, c->d_K12, c->d_K21, alpha_dt, c->d_pcLU, c->d_pcPiv, c->d_pcbad),
         "pc build");
    else
      ck(o.pc_build(c->dc, c->d_K11, c->d_K12, c->d_K21, alpha_dt, c->d_pcLU, c->d_pcPiv, c->d_pcbad), "pc build");
    int bad = -1;
    ck(cudaMemcpyAsync(&bad, c->d_pcbad, sizeof(int), cudaMemcpyDeviceToHost, c->stream), "read flag");
    ck(cudaStreamSynchronize(c->stream), "stream synchronize");
    if (bad >= 0)
      throw ldg_error(LDG_ERR_SOLVER, "singular block-Jacobi block at element " + std::to_string(bad));
    c->pc_adi = adi;
    c->pc_valid = true;
    c->pc_adt = alpha_dt;
    return LDG_OK;
  });
}

int ldg_set_precond_mode(ldg_ctx* c, int mode) {
  return guarded(c, [&]() -> int {
    if (mode < 0 || mode > 2)
      throw ldg_error(LDG_ERR_INVALID_ARGUMENT, "precond mode must be 0 (auto), 1 (element inverse) or 2 (line-ADI)");
    c->pc_mode = mode;
    c->dc.pc_inverse = mode == 1;
    c->pc_valid = false;
    return LDG_OK;
  });
}

int ldg_precond_apply(ldg_ctx* c, const double* r, double* z) {
  return guarded(c, [&]() -> int {
    check_aligned(r, "r");
    check_aligned(z, "z");
    if (!c->pc_valid) throw ldg_error(LDG_ERR_SOLVER, "preconditioner not built");
    return finish(c, pc_apply_any(c, r, z));
  });
}

int ldg_gmres(ldg_ctx* c, double alpha_dt, const double* b, double* x, double rtol, int32_t maxit, int32_t restart,
              int32_t use_precond, int32_t* iters, int32_t* converged, double* resnorm) {
  return guarded(c, [&]() -> int {
    if (!c->jac_valid) throw ldg_error(LDG_ERR_SOLVER, "Jacobian not assembled");
    if (!(rtol > 0.0) || maxit < 1 || restart < 1 || !b || !x)
      throw ldg_error(LDG_ERR_INVALID_ARGUMENT, "gmres: rtol > 0, maxit >= 1, restart >= 1 and vectors required");
    check_aligned(b, "b");
    check_aligned(x, "x");
    if (use_precond && !c->pc_valid) throw ldg_error(LDG_ERR_SOLVER, "preconditioner not built");
    const ldg::Ops& o = *c->ops;
    const size_t n = c->nU();
    const int mr = restart;
    if (c->kv_restart < mr) {
      cudaFree(c->d_kv);
      c->d_kv = nullptr;
      ck(cudaMalloc(&c->d_kv, (2 * static_cast<size_t>(mr) + 1) * n * sizeof(double)), "cudaMalloc Krylov");
      cudaFree(c->d_kred);
      c->d_kred = nullptr;
      c->kv_restart = mr;
    }
    ensure(c->d_kw, 3 * n);
    ensure(c->d_kred, KR_BLOCKS + (static_cast<size_t>(mr) + 1) * mr + 8 + 3 * static_cast<size_t>(mr) + 4);
    double* V = c->d_kv;                 // (mr+1) x n
    double* Zs = c->d_kv + (mr + 1) * n;  // mr x n
    double* w = c->d_kw;
    double* t = w + n;
    double* r = t + n;
    double* part = c->d_kred;
    double* Hd = part + KR_BLOCKS;       // column-major (mr+1) x mr
    double* sc = Hd + (mr + 1) * mr;     // scalars
    cudaStream_t st = c->stream;
    const int vb = 592, vt = 256;
    auto dot = [&](const double* a, const double* bb, double* out, int root) {
      c->launches += 2;
      k_dot_part<<<KR_BLOCKS, KR_THREADS, 0, st>>>(a, bb, n, part);
      k_dot_fin<<<1, KR_THREADS, 0, st>>>(part, KR_BLOCKS, out, root);
    };
    auto op = [&](const double* v, double* y) {
      const double* ww = nullptr;
      if (c->second) {
        ensure(c->d_w, c->nQ());
        ck(o.spmv21(c->dc, c->d_K21, v, c->d_w), "K21 launch");
        ww = c->d_w;
      }
      ck(o.split(c->dc, c->d_K11, c->d_K12, v, ww, alpha_dt, y), "split launch");
    };
    auto host_scalar = [&](const double* dptr_) {
      double h = 0.0;
      ck(cudaMemcpyAsync(&h, dptr_, sizeof(double), cudaMemcpyDeviceToHost, st), "D2H scalar");
      ck(cudaStreamSynchronize(st), "stream synchronize");
      return h;
    };
    ck(cudaMemsetAsync(x, 0, n * sizeof(double), st), "zero x");
    dot(b, b, sc, 1);
    const double bn = host_scalar(sc);
    *iters = 0;
    *converged = 0;
    *resnorm = bn;
    if (bn == 0.0) {
      *converged = 1;
      return LDG_OK;
    }
    ck(cudaMemcpyAsync(r, b, n * sizeof(double), cudaMemcpyDeviceToDevice, st), "copy b");
    // Hessenberg / Givens state on the device; the host keeps up to GW
    // iterations in flight and learns a cycle's end from a pinned copy of the
    // state, polled GW iterations behind (no per-iteration stall)
    constexpr int GW = 4;
    double* gcs = sc + 8;       // cs[mr], sn[mr], g[mr+1], state[3]
    double* gsn = gcs + mr;
    double* gg = gsn + mr;
    double* gst = gg + mr + 1;
    if (!c->h_gst) ck(cudaHostAlloc(reinterpret_cast<void**>(&c->h_gst), GW * 4 * sizeof(double), 0), "pinned");
    if (!c->ev_gw[0])
      for (int q = 0; q < GW; ++q) ck(cudaEventCreateWithFlags(&c->ev_gw[q], cudaEventDisableTiming), "event");
    std::vector<double> H(static_cast<size_t>(mr + 1) * mr), g(mr + 1);
    double beta = bn;
    int it = 0;
    while (true) {
      k_div<<<vb, vt, 0, st>>>(V, r, n, nullptr, beta);
      k_gmres_cycle_init<<<1, 64, 0, st>>>(gg, mr, beta, gst);
      c->launches += 2;
      int j = 0, launched = 0;
      bool done = false;
      for (; j < mr && it + j < maxit && !done; ++j) {
        double* Vj = V + static_cast<size_t>(j) * n;
        double* Zj = use_precond ? Zs + static_cast<size_t>(j) * n : Vj;
        if (use_precond) ck(pc_apply_any(c, Vj, Zj), "pc apply");
        op(Zj, w);
        for (int i = 0; i <= j; ++i) {  // modified Gram-Schmidt
          double* hij = Hd + static_cast<size_t>(j) * (mr + 1) + i;
          dot(w, V + static_cast<size_t>(i) * n, hij, 0);
          k_axpy_dev<<<vb, vt, 0, st>>>(w, V + static_cast<size_t>(i) * n, n, hij);
          ++c->launches;
        }
        double* hn_d = Hd + static_cast<size_t>(j) * (mr + 1) + j + 1;
        dot(w, w, hn_d, 1);
        k_div<<<vb, vt, 0, st>>>(V + static_cast<size_t>(j + 1) * n, w, n, hn_d, 0.0);
        k_gmres_givens<<<1, 1, 0, st>>>(Hd, mr, j, gcs, gsn, gg, rtol * bn, gst);
        c->launches += 2;
        ck(cudaMemcpyAsync(c->h_gst + (j % GW) * 4, gst, 3 * sizeof(double), cudaMemcpyDeviceToHost, st), "D2H st");
        ck(cudaEventRecord(c->ev_gw[j % GW], st), "record");
        ++launched;
        if (j >= GW - 1) {  // poll the state of iteration j - GW + 1
          ck(cudaEventSynchronize(c->ev_gw[(j - GW + 1) % GW]), "event synchronize");
          done = c->h_gst[((j - GW + 1) % GW) * 4] != 0.0;
        }
      }
      (void)launched;
      ck(cudaStreamSynchronize(st), "stream synchronize");
      double stt[3];
      ck(cudaMemcpy(stt, gst, 3 * sizeof(double), cudaMemcpyDeviceToHost), "D2H state");
      if (stt[2] != 0.0) throw ldg_error(LDG_ERR_SOLVER, "gmres: numerical breakdown (non-finite Krylov vector)");
      j = static_cast<int>(stt[1]);
      it += j;
      ck(cudaMemcpy(g.data(), gg, (j + 1) * sizeof(double), cudaMemcpyDeviceToHost), "D2H g");
      std::vector<double> Rc(static_cast<size_t>(mr + 1) * (j > 0 ? j : 1));
      if (j > 0)
        ck(cudaMemcpy(Rc.data(), Hd, static_cast<size_t>(mr + 1) * j * sizeof(double), cudaMemcpyDeviceToHost),
           "D2H R");
      for (int q = 0; q < j; ++q)
        for (int i = 0; i <= q; ++i) H[i * mr + q] = Rc[static_cast<size_t>(q) * (mr + 1) + i];
      std::vector<double> y(j, 0.0);
      for (int i = j - 1; i >= 0; --i) {
        double s_ = g[i];
        for (int q = i + 1; q < j; ++q) s_ -= H[i * mr + q] * y[q];
        y[i] = s_ / H[i * mr + i];
      }
      for (int i = 0; i < j; ++i)
      {
        k_axpy<<<vb, vt, 0, st>>>(x, use_precond ? Zs + static_cast<size_t>(i) * n : V + static_cast<size_t>(i) * n,
                                  n, y[i]);
        ++c->launches;
      }
      op(x, t);
      k_sub<<<vb, vt, 0, st>>>(r, b, t, n);
      ++c->launches;
      dot(r, r, sc, 1);
      beta = host_scalar(sc);
      *resnorm = beta;
      if (beta <= rtol * bn) {
        *converged = 1;
        break;
      }
      if (it >= maxit) break;
    }
    *iters = it;
    return finish(c, cudaGetLastError());
  });
}

int ldg_gmres_host(ldg_ctx* c, double alpha_dt, const double* b, double* x, double rtol, int32_t maxit,
                   int32_t restart, int32_t use_precond, int32_t* iters, int32_t* converged, double* resnorm) {
  return guarded(c, [&]() -> int {
    ensure(c->d_hx, c->nQ());  // (shared with ldg_bsr_spmv_host: sized for K12 / K21 vectors)
    ensure(c->d_hy, c->nQ());
    ck(cudaMemcpyAsync(c->d_hx, b, c->nU() * sizeof(double), cudaMemcpyHostToDevice, c->stream), "H2D b");
    const int st = ldg_gmres(c, alpha_dt, c->d_hx, c->d_hy, rtol, maxit, restart, use_precond, iters, converged,
                             resnorm);
    if (st != LDG_OK) return st;
    ck(cudaMemcpyAsync(x, c->d_hy, c->nU() * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "D2H x");
    return finish(c, cudaSuccess) == LDG_OK && cudaStreamSynchronize(c->stream) == cudaSuccess ? LDG_OK
                                                                                               : LDG_ERR_CUDA;
  });
}

int ldg_precond_apply_host(ldg_ctx* c, const double* r, double* z) {
  return guarded(c, [&]() -> int {
    ensure(c->d_hx, c->nQ());
    ensure(c->d_hy, c->nQ());
    ck(cudaMemcpyAsync(c->d_hx, r, c->nU() * sizeof(double), cudaMemcpyHostToDevice, c->stream), "H2D r");
    const int st = ldg_precond_apply(c, c->d_hx, c->d_hy);
    if (st != LDG_OK) return st;
    ck(cudaMemcpyAsync(z, c->d_hy, c->nU() * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "D2H z");
    ck(cudaStreamSynchronize(c->stream), "stream synchronize");
    return LDG_OK;
  });
}

// ---------------------------------------------------------- time integration
// (PAPER.md:641-685, 755-775), mirroring the oracle's
// lo_rk4_step / lo_dirk3_step operation by operation.
int ldg_rk4_step(ldg_ctx* c, double* U, double t, double dt) {
  return guarded(c, [&]() -> int {
    if (!(dt > 0.0) || !U) throw ldg_error(LDG_ERR_INVALID_ARGUMENT, "rk4_step: dt > 0 and U required");
    const size_t n = c->nU();
    double* w = ensure(c->d_ti, 8 * n);
    double *k1 = w, *k2 = w + n, *k3 = w + 2 * n, *k4 = w + 3 * n, *us = w + 4 * n;
    double* red = ensure(c->d_kred, KR_BLOCKS + 8);
    cudaStream_t st = c->stream;
    const bool was = c->sync_errors;
    c->sync_errors = true;
    // classical RK4 stage times t, t + dt/2, t + dt/2, t + dt (time-dependent
    // boundary data is evaluated at each stage's own time)
    auto F = [&](const double* u, double* k, int stage) {
      const double ts = t + (stage == 1 ? 0.0 : stage == 4 ? dt : 0.5 * dt);
      int s_ = ldg_residual(c, u, ts, k, nullptr);
      if (s_ != LDG_OK) {
        c->sync_errors = was;
        throw ldg_error(s_, c->err);
      }
      k_amax_part<<<KR_BLOCKS, KR_THREADS, 0, st>>>(k, n, red);
      k_amax_fin<<<1, KR_THREADS, 0, st>>>(red, KR_BLOCKS, red + KR_BLOCKS);
      c->launches += 2;
      double m = 0.0;
      ck(cudaMemcpyAsync(&m, red + KR_BLOCKS, sizeof(double), cudaMemcpyDeviceToHost, st), "D2H");
      ck(cudaStreamSynchronize(st), "stream synchronize");
      if (!std::isfinite(m)) {
        c->sync_errors = was;
        throw ldg_error(LDG_ERR_SOLVER, "rk4 blow-up at stage " + std::to_string(stage));
      }
    };
    const int vb = 592, vt = 256;
    F(U, k1, 1);
    k_rk_state<<<vb, vt, 0, st>>>(us, U, k1, n, 0.5 * dt);
    F(us, k2, 2);
    k_rk_state<<<vb, vt, 0, st>>>(us, U, k2, n, 0.5 * dt);
    F(us, k3, 3);
    k_rk_state<<<vb, vt, 0, st>>>(us, U, k3, n, dt);
    F(us, k4, 4);
    k_rk4_update<<<vb, vt, 0, st>>>(U, k1, k2, k3, k4, n, dt);
    c->launches += 4;
    c->sync_errors = was;
    return finish(c, cudaGetLastError());
  });
}

int ldg_dirk3_step(ldg_ctx* c, double* U, double t, double dt, const ldg_newton_cfg* cfg, ldg_solver_stats* stats) {
  return guarded(c, [&]() -> int {
    if (!(dt > 0.0) || !U || !cfg || cfg->gmres_iters < 1 || cfg->recompute_threshold < 1 || cfg->max_newton < 1)
      throw ldg_error(LDG_ERR_INVALID_ARGUMENT, "dirk3_step: dt > 0, U and a valid ldg_newton_cfg required");
    const double al = 0.435866521508459, tau2 = (1.0 + al) / 2.0;
    const double b1 = -(6.0 * al * al - 16.0 * al + 1.0) / 4.0, b2 = (6.0 * al * al - 20.0 * al + 5.0) / 4.0;
    const double A[3][3] = {{al, 0.0, 0.0}, {tau2 - al, al, 0.0}, {b1, b2, al}};
    const double B[3] = {b1, b2, al};
    const size_t n = c->nU();
    const double adt = al * dt;
    double* w = ensure(c->d_ti, 8 * n);
    double* K[3] = {w, w + n, w + 2 * n};
    double *Kc = w + 3 * n, *us = w + 4 * n, *Fv = w + 5 * n, *G = w + 6 * n, *dK = w + 7 * n;
    cudaStream_t st = c->stream;
    const int vb = 592, vt = 256;
    ldg_solver_stats s{};
    const bool was = c->sync_errors;
    c->sync_errors = true;
    auto chk = [&](int code) {
      if (code != LDG_OK) {
        c->sync_errors = was;
        throw ldg_error(code, c->err);
      }
    };
    // stage times t + c_i dt, c = (alpha, tau2, 1) (row sums of the tableau)
    const double cst[3] = {al, tau2, 1.0};
    auto assemble = [&](const double* u, double ta) {
      chk(ldg_jacobian_assemble(c, u, ta));
      ++s.jacobian_assemblies;
      c->pc_valid = false;
    };
    auto ensure_pc = [&]() {
      if (cfg->use_precond && (!c->pc_valid || c->pc_adt != adt)) chk(ldg_precond_build(c, adt));
    };
    auto F = [&](const double* u, double* k, double ta) {
      chk(ldg_residual(c, u, ta, k, nullptr));
      ++s.residual_evals;
    };
    if (!c->jac_valid) assemble(U, t);
    ensure_pc();
    F(U, Kc, t);
    for (int i = 0; i < 3; ++i) {
      int it = 0;
      while (true) {
        k_stage_state<<<vb, vt, 0, st>>>(us, U, K[0], K[1], Kc, n, dt, A[i][0], A[i][1], al, i);
        ++c->launches;
        F(us, Fv, t + cst[i] * dt);
        k_rhs<<<vb, vt, 0, st>>>(G, Kc, Fv, n);
        // (re-fetched each time: ldg_gmres reallocates d_kred when its restart grows)
        double* red = ensure(c->d_kred, KR_BLOCKS + 8);
        k_amax_part<<<KR_BLOCKS, KR_THREADS, 0, st>>>(G, n, red);
        k_amax_fin<<<1, KR_THREADS, 0, st>>>(red, KR_BLOCKS, red + KR_BLOCKS);
        c->launches += 3;
        double gn = 0.0;
        ck(cudaMemcpyAsync(&gn, red + KR_BLOCKS, sizeof(double), cudaMemcpyDeviceToHost, st), "D2H");
        ck(cudaStreamSynchronize(st), "stream synchronize");
        if (!std::isfinite(gn)) {
          c->sync_errors = was;
          throw ldg_error(LDG_ERR_SOLVER, "dirk3: non-finite stage");
        }
        s.residual_norm = gn;
        if (gn <= cfg->newton_tol) break;
        if (it >= cfg->max_newton) {
          c->sync_errors = was;
          throw ldg_error(LDG_ERR_SOLVER, "dirk3: step failure (Newton did not converge)");
        }
        if (it > 0 && it % cfg->recompute_threshold == 0) {
          assemble(us, t + cst[i] * dt);
          ensure_pc();
        }
        int32_t gi = 0, gc = 0;
        double gr = 0.0;
        chk(ldg_gmres(c, adt, G, dK, 1e-300, cfg->gmres_iters, cfg->gmres_iters, cfg->use_precond, &gi, &gc, &gr));
        s.gmres_iters += gi;
        k_axpy<<<vb, vt, 0, st>>>(Kc, dK, n, 1.0);
        ++c->launches;
        ++it;
        ++s.newton_iters;
      }
      ck(cudaMemcpyAsync(K[i], Kc, n * sizeof(double), cudaMemcpyDeviceToDevice, st), "copy stage slope");
    }
    k_dirk_update<<<vb, vt, 0, st>>>(U, K[0], K[1], K[2], n, dt, B[0], B[1], B[2]);
    ++c->launches;
    c->sync_errors = was;
    if (stats) *stats = s;
    return finish(c, cudaGetLastError());
  });
}

// Pseudo-transient continuation to a steady state (PAPER.md:
// 641-652); mirrors the oracle's lo_steady_solve operation by operation.
int ldg_steady_solve(ldg_ctx* c, double* U, double t, const ldg_steady_cfg* cfg, ldg_solver_stats* stats) {
  return guarded(c, [&]() -> int {
    if (!U || !cfg || !(cfg->dt0 > 0.0) || !(cfg->growth >= 1.0) || cfg->n_steps < 0 || cfg->gmres_iters < 1 ||
        cfg->recompute_threshold < 1 || cfg->max_newton < 1)
      throw ldg_error(LDG_ERR_INVALID_ARGUMENT, "steady_solve: U and a valid ldg_steady_cfg required");
    const size_t n = c->nU();
    const double dt_final = cfg->dt_final > 0.0 ? cfg->dt_final : 1e12;
    const double rtol = cfg->gmres_rtol > 0.0 ? cfg->gmres_rtol : 1e-300;
    double* w = ensure(c->d_ti, 8 * n);  // (the DIRK3 workspace: 8 vectors)
    double *R = w, *b = w + n, *dU = w + 2 * n, *Us = w + 3 * n, *Rs = w + 4 * n;
    cudaStream_t st = c->stream;
    const int vb = 592, vt = 256;
    ldg_solver_stats s{};
    const bool was = c->sync_errors;
    c->sync_errors = true;
    FILE* log = nullptr;
    if (cfg->log_csv) {
      log = std::fopen(cfg->log_csv, "w");
      if (!log) {
        c->sync_errors = was;
        throw ldg_error(LDG_ERR_CONFIG, std::string("cannot write '") + cfg->log_csv + "'");
      }
      std::fprintf(log, "step,stage,newton_iters,gmres_iters,jacobian_refreshed,residual_norm\n");
    }
    auto fail = [&](int code, const std::string& msg) {
      c->sync_errors = was;
      if (log) std::fclose(log);
      if (stats) *stats = s;
      throw ldg_error(code, msg);
    };
    auto chk = [&](int code) {
      if (code != LDG_OK) fail(code, c->err);
    };
    // residual at U into R (and its inf-norm); false on a non-physical state
    auto F = [&](double& rn) {
      const int code = ldg_residual(c, U, t, R, nullptr);
      ++s.residual_evals;
      if (code == LDG_ERR_PHYSICAL_STATE) return false;
      chk(code);
      // (re-fetched each time: ldg_gmres reallocates d_kred when its restart grows)
      double* red = ensure(c->d_kred, KR_BLOCKS + 8);
      k_amax_part<<<KR_BLOCKS, KR_THREADS, 0, st>>>(R, n, red);
      k_amax_fin<<<1, KR_THREADS, 0, st>>>(red, KR_BLOCKS, red + KR_BLOCKS);
      c->launches += 2;
      ck(cudaMemcpyAsync(&rn, red + KR_BLOCKS, sizeof(double), cudaMemcpyDeviceToHost, st), "D2H");
      ck(cudaStreamSynchronize(st), "stream synchronize");
      return true;
    };
    double rn = 0.0;
    if (!F(rn)) fail(LDG_ERR_PHYSICAL_STATE, c->err);
    if (!std::isfinite(rn)) fail(LDG_ERR_SOLVER, "steady_solve: non-finite residual");
    s.residual_norm = rn;
    const double rn0 = rn;
    bool done = rn <= cfg->newton_tol;
    int since = 0, rejects = 0;
    bool fresh = true;
    double dt = cfg->dt0;
    // continuation updates left before the final (Newton) phase; a rejected
    // final-phase update returns to continuation for 5 more updates
    int cont_left = cfg->n_steps, newton_left = cfg->max_newton;
    for (int k = 0; !done && (cont_left > 0 || newton_left > 0); ++k) {
      const bool fin = cont_left == 0;
      const double h = fin ? dt_final : dt;
      bool refreshed = false;
      if (fresh || since >= cfg->recompute_threshold) {
        chk(ldg_jacobian_assemble(c, U, t));
        ++s.jacobian_assemblies;
        since = 0;
        fresh = false;
        c->pc_valid = false;
        refreshed = true;
      }
      if (cfg->use_precond && (!c->pc_valid || c->pc_adt != h)) chk(ldg_precond_build(c, h));
      ck(cudaMemsetAsync(b, 0, n * sizeof(double), st), "memset");
      k_axpy<<<vb, vt, 0, st>>>(b, R, n, h);  // b = h R
      ++c->launches;
      int32_t gi = 0, gc = 0;
      double gr = 0.0;
      chk(ldg_gmres(c, h, b, dU, rtol, cfg->gmres_iters, cfg->gmres_iters, cfg->use_precond, &gi, &gc, &gr));
      s.gmres_iters += gi;
      ck(cudaMemcpyAsync(Us, U, n * sizeof(double), cudaMemcpyDeviceToDevice, st), "save U");
      ck(cudaMemcpyAsync(Rs, R, n * sizeof(double), cudaMemcpyDeviceToDevice, st), "save R");
      k_axpy<<<vb, vt, 0, st>>>(U, dU, n, 1.0);
      ++c->launches;
      ++since;
      ++s.newton_iters;
      double rn1 = 0.0;
      const bool phys = F(rn1);
      if (!phys || !(rn1 <= 1e4 * rn0)) {
        // rejected update: restore, halve the pseudo-time step, fresh Jacobian
        // (SPEC.md:535 step-failure policy); the final phase cannot back off
        if (log) std::fprintf(log, "%d,2,%d,%d,%d,%.17g\n", k, s.newton_iters, gi, refreshed ? 1 : 0, phys ? rn1 : -1.0);
        if (++rejects > 10) fail(LDG_ERR_SOLVER, "steady_solve: diverged");
        ck(cudaMemcpyAsync(U, Us, n * sizeof(double), cudaMemcpyDeviceToDevice, st), "restore U");
        ck(cudaMemcpyAsync(R, Rs, n * sizeof(double), cudaMemcpyDeviceToDevice, st), "restore R");
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
      if (log)
        std::fprintf(log, "%d,%d,%d,%d,%d,%.17g\n", k, fin ? 1 : 0, s.newton_iters, gi, refreshed ? 1 : 0, rn);
      done = rn <= cfg->newton_tol;
      if (fin) {
        --newton_left;
      } else {
        --cont_left;
        dt *= cfg->growth;
      }
    }
    if (!done) fail(LDG_ERR_SOLVER, "steady_solve: no convergence within n_steps + max_newton updates");
    c->sync_errors = was;
    if (log) std::fclose(log);
    if (stats) *stats = s;
    return finish(c, cudaGetLastError());
  });
}

// ------------------------------------------------------------ host variants
// Host-buffer variants.  With error synchronisation on (the default) each
// call uploads on the context stream, runs, downloads and synchronises.  With
// it off (ldg_set_sync_errors(ctx, 0)) the calls are asynchronous like the
// device entry points: uploads run on a copy stream (cs_in) and downloads on
// another (cs_out), ordered against the kernels by events, so the transfers
// of consecutive calls overlap each other and the kernels in both PCIe
// directions; host buffers must stay valid (pinned for true overlap) and
// results are ready after ldg_synchronize().
namespace {
// device address of a mapped pinned host buffer (cudaHostAlloc / registered
// memory under unified addressing), else nullptr
double* mapped_host(const ldg_ctx* c, double* h) {
  if (!c->zero_copy) return nullptr;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, h) != cudaSuccess) {
    (void)cudaGetLastError();
    return nullptr;
  }
  if (a.type != cudaMemoryTypeHost || !a.devicePointer) return nullptr;
  if (reinterpret_cast<uintptr_t>(a.devicePointer) & 15u) return nullptr;  // staged copy instead
  return static_cast<double*>(a.devicePointer);
}
// upload n doubles to dbuf once `free_ev` (the last reader of dbuf) completed;
// the context stream then waits for the upload
void upload_async(ldg_ctx* c, double* dbuf, const double* h, size_t n, cudaEvent_t free_ev) {
  ck(cudaStreamWaitEvent(c->cs_in, free_ev, 0), "wait buffer");
  ck(cudaMemcpyAsync(dbuf, h, n * sizeof(double), cudaMemcpyHostToDevice, c->cs_in), "H2D");
  ck(cudaEventRecord(c->ev_in, c->cs_in), "record upload");
  ck(cudaStreamWaitEvent(c->stream, c->ev_in, 0), "wait upload");
}
// download n doubles from dbuf after the context stream's work so far
void download_async(ldg_ctx* c, double* h, const double* dbuf, size_t n, cudaEvent_t done_ev) {
  ck(cudaEventRecord(c->ev_k, c->stream), "record kernels");
  ck(cudaStreamWaitEvent(c->cs_out, c->ev_k, 0), "wait kernels");
  ck(cudaMemcpyAsync(h, dbuf, n * sizeof(double), cudaMemcpyDeviceToHost, c->cs_out), "D2H");
  ck(cudaEventRecord(done_ev, c->cs_out), "record download");
}
}  // namespace

int ldg_residual_host(ldg_ctx* c, const double* U, double t, double* R, double* Q) {
  return guarded(c, [&]() -> int {
    ensure(c->d_hu, c->nU());
    ensure(c->d_hr, c->nU());
    double* dq = c->second ? ensure(c->d_Q, c->nQ()) : nullptr;
    if (!c->sync_errors) {
      upload_async(c, c->d_hu, U, c->nU(), c->ev_free_hu);
      ck(cudaStreamWaitEvent(c->stream, c->ev_out_r, 0), "wait R/Q download");  // d_hr, d_Q reuse
      int st = ldg_residual(c, c->d_hu, t, c->d_hr, dq);
      if (st != LDG_OK) return st;
      ck(cudaEventRecord(c->ev_free_hu, c->stream), "record");
      ck(cudaEventRecord(c->ev_k, c->stream), "record kernels");
      ck(cudaStreamWaitEvent(c->cs_out, c->ev_k, 0), "wait kernels");
      ck(cudaMemcpyAsync(R, c->d_hr, c->nU() * sizeof(double), cudaMemcpyDeviceToHost, c->cs_out), "D2H R");
      if (Q && dq)
        ck(cudaMemcpyAsync(Q, dq, c->nQ() * sizeof(double), cudaMemcpyDeviceToHost, c->cs_out), "D2H Q");
      ck(cudaEventRecord(c->ev_out_r, c->cs_out), "record download");
      return LDG_OK;
    }
    ck(cudaMemcpyAsync(c->d_hu, U, c->nU() * sizeof(double), cudaMemcpyHostToDevice, c->stream), "H2D U");
    const bool was = c->sync_errors;
    c->sync_errors = false;
    int st = ldg_residual(c, c->d_hu, t, c->d_hr, dq);
    c->sync_errors = was;
    if (st != LDG_OK) return st;
    ck(cudaMemcpyAsync(R, c->d_hr, c->nU() * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "D2H R");
    if (Q && dq)
      ck(cudaMemcpyAsync(Q, dq, c->nQ() * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "D2H Q");
    const bool w2 = c->sync_errors;
    c->sync_errors = true;
    st = finish(c, cudaSuccess);
    c->sync_errors = w2;
    return st;
  });
}

// Residual and Jacobian at one state from ONE upload of U (a Newton step's
// R(U) and J(U)): second-order physics computes Q = D(U) once for both.
int ldg_residual_assemble_host(ldg_ctx* c, const double* U, double t, double* R, double* Q) {
  return guarded(c, [&]() -> int {
    ensure(c->d_hu, c->nU());
    ensure(c->d_hr, c->nU());
    double* dq = c->second ? ensure(c->d_Q, c->nQ()) : nullptr;
    const size_t nb = c->nU() * sizeof(double);
    if (!c->sync_errors) {
      upload_async(c, c->d_hu, U, c->nU(), c->ev_free_hu);
      ck(cudaStreamWaitEvent(c->stream, c->ev_out_r, 0), "wait R/Q download");  // d_hr, d_Q reuse
      int st = ldg_residual(c, c->d_hu, t, c->d_hr, dq);
      if (st != LDG_OK) return st;
      ck(cudaEventRecord(c->ev_k, c->stream), "record kernels");
      ck(cudaStreamWaitEvent(c->cs_out, c->ev_k, 0), "wait kernels");
      ck(cudaMemcpyAsync(R, c->d_hr, nb, cudaMemcpyDeviceToHost, c->cs_out), "D2H R");
      if (Q && dq) ck(cudaMemcpyAsync(Q, dq, nb * c->D, cudaMemcpyDeviceToHost, c->cs_out), "D2H Q");
      ck(cudaEventRecord(c->ev_out_r, c->cs_out), "record download");
      st = assemble_at(c, c->d_hu, dq, t);  // the download overlaps the assembly
      if (st != LDG_OK) return st;
      ck(cudaEventRecord(c->ev_free_hu, c->stream), "record");
      return LDG_OK;
    }
    ck(cudaMemcpyAsync(c->d_hu, U, nb, cudaMemcpyHostToDevice, c->stream), "H2D U");
    c->sync_errors = false;
    int st = ldg_residual(c, c->d_hu, t, c->d_hr, dq);
    if (st == LDG_OK) {
      ck(cudaMemcpyAsync(R, c->d_hr, nb, cudaMemcpyDeviceToHost, c->stream), "D2H R");
      if (Q && dq) ck(cudaMemcpyAsync(Q, dq, nb * c->D, cudaMemcpyDeviceToHost, c->stream), "D2H Q");
      st = assemble_at(c, c->d_hu, dq, t);
    }
    c->sync_errors = true;
    return st == LDG_OK ? finish(c, cudaSuccess) : st;
  });
}

// gradient_residual / residual_second_order with host buffers (synchronous)
int ldg_gradient_host(ldg_ctx* c, const double* U, double t, double* Q) {
  return guarded(c, [&]() -> int {
    if (!c->second) throw ldg_error(LDG_ERR_CONFIG, "gradient_residual needs second-order physics");
    double* du = ensure(c->d_hu, c->nU());
    double* dq = ensure(c->d_Q, c->nQ());
    ck(cudaMemcpyAsync(du, U, c->nU() * sizeof(double), cudaMemcpyHostToDevice, c->stream), "H2D U");
    c->sync_errors = false;
    int st = ldg_gradient(c, du, t, dq);
    c->sync_errors = true;
    if (st != LDG_OK) return st;
    ck(cudaMemcpyAsync(Q, dq, c->nQ() * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "D2H Q");
    return finish(c, cudaSuccess);
  });
}

int ldg_residual_uq_host(ldg_ctx* c, const double* U, const double* Q, double t, double* R) {
  return guarded(c, [&]() -> int {
    double* du = ensure(c->d_hu, c->nU());
    double* dr = ensure(c->d_hr, c->nU());
    double* dq = c->second ? ensure(c->d_Q, c->nQ()) : nullptr;
    ck(cudaMemcpyAsync(du, U, c->nU() * sizeof(double), cudaMemcpyHostToDevice, c->stream), "H2D U");
    if (dq) ck(cudaMemcpyAsync(dq, Q, c->nQ() * sizeof(double), cudaMemcpyHostToDevice, c->stream), "H2D Q");
    c->sync_errors = false;
    int st = ldg_residual_uq(c, du, dq, t, dr);
    c->sync_errors = true;
    if (st != LDG_OK) return st;
    ck(cudaMemcpyAsync(R, dr, c->nU() * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "D2H R");
    return finish(c, cudaSuccess);
  });
}

int ldg_jacobian_assemble_host(ldg_ctx* c, const double* U, double t) {
  return guarded(c, [&]() -> int {
    ensure(c->d_hu2, c->nU());
    if (!c->sync_errors) {
      upload_async(c, c->d_hu2, U, c->nU(), c->ev_free_hu2);
      if (c->second) ck(cudaStreamWaitEvent(c->stream, c->ev_out_r, 0), "wait Q download");  // d_Q reuse
      const int st = ldg_jacobian_assemble(c, c->d_hu2, t);
      if (st != LDG_OK) return st;
      ck(cudaEventRecord(c->ev_free_hu2, c->stream), "record");
      return LDG_OK;
    }
    ck(cudaMemcpyAsync(c->d_hu2, U, c->nU() * sizeof(double), cudaMemcpyHostToDevice, c->stream), "H2D U");
    const bool was = c->sync_errors;
    c->sync_errors = true;
    const int st = ldg_jacobian_assemble(c, c->d_hu2, t);
    c->sync_errors = was;
    return st;
  });
}

int ldg_bsr_spmv_host(ldg_ctx* c, int which, const double* x, double* y) {
  return guarded(c, [&]() -> int {
    const size_t nx = which == LDG_K12 ? c->nQ() : c->nU();
    const size_t ny = which == LDG_K21 ? c->nQ() : c->nU();
    double* dx = ensure(c->d_hx, c->nQ());
    double* dy = ensure(c->d_hy, c->nQ());
    // zero-copy output: a K11 product into mapped pinned host memory is
    // written by the kernel itself (whole node rows per warp store, see
    // k_spmv11), so the PCIe transfer of y overlaps the product instead of
    // following it; pageable buffers take the staged copy
    double* yz = which == LDG_K11 && c->ops->M == 4 ? mapped_host(c, y) : nullptr;
    auto product = [&](double* dst) -> int {
      if (!yz) return ldg_bsr_spmv(c, which, dx, dst);
      if (!c->jac_valid) throw ldg_error(LDG_ERR_SOLVER, "Jacobian not assembled");
      return finish(c, c->ops->spmv11_zc(c->dc, c->d_K11, dx, dst));
    };
    if (!c->sync_errors) {
      upload_async(c, dx, x, nx, c->ev_free_hx);
      ck(cudaStreamWaitEvent(c->stream, c->ev_out_y, 0), "wait y download");
      const int st = product(yz ? yz : dy);
      if (st != LDG_OK) return st;
      ck(cudaEventRecord(c->ev_free_hx, c->stream), "record");
      if (yz) ck(cudaEventRecord(c->ev_out_y, c->stream), "record product");
      else download_async(c, y, dy, ny, c->ev_out_y);
      return LDG_OK;
    }
    if (yz) {
      ck(cudaMemcpyAsync(dx, x, nx * sizeof(double), cudaMemcpyHostToDevice, c->stream), "H2D x");
      const bool was = c->sync_errors;
      c->sync_errors = true;
      const int st = product(yz);
      c->sync_errors = was;
      return st;
    }
    ck(cudaMemcpyAsync(dx, x, nx * sizeof(double), cudaMemcpyHostToDevice, c->stream), "H2D x");
    const bool was = c->sync_errors;
    c->sync_errors = false;
    int st = ldg_bsr_spmv(c, which, dx, dy);
    c->sync_errors = was;
    if (st != LDG_OK) return st;
    ck(cudaMemcpyAsync(y, dy, ny * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "D2H y");
    const bool w2 = c->sync_errors;
    c->sync_errors = true;
    st = finish(c, cudaSuccess);
    c->sync_errors = w2;
    return st;
  });
}

int ldg_split_matvec_host(ldg_ctx* c, double adt, const double* v, double* y) {
  return guarded(c, [&]() -> int {
    const size_t n = c->nU();
    if (!c->sync_errors) {
      // two staging slots: the upload of the next v and the download of the
      // previous y overlap this product (GMRES-style back-to-back calls)
      const int s = c->mv_slot;
      c->mv_slot ^= 1;
      double* dv = ensure(c->d_mv_in[s], n);
      double* dy = ensure(c->d_mv_out[s], n);
      upload_async(c, dv, v, n, c->ev_mv_free[s]);
      ck(cudaStreamWaitEvent(c->stream, c->ev_mv_out[s], 0), "wait y download");
      const int st = ldg_split_matvec(c, adt, dv, dy);
      if (st != LDG_OK) return st;
      ck(cudaEventRecord(c->ev_mv_free[s], c->stream), "record");
      download_async(c, y, dy, n, c->ev_mv_out[s]);
      return LDG_OK;
    }
    ensure(c->d_hu, n);
    ensure(c->d_hr, n);
    ck(cudaMemcpyAsync(c->d_hu, v, n * sizeof(double), cudaMemcpyHostToDevice, c->stream), "H2D v");
    c->sync_errors = false;
    int st = ldg_split_matvec(c, adt, c->d_hu, c->d_hr);
    c->sync_errors = true;
    if (st != LDG_OK) return st;
    ck(cudaMemcpyAsync(y, c->d_hr, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "D2H y");
    return finish(c, cudaSuccess);
  });
}

}  // extern "C"
