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
    return (mx < 1e-11 && sol.converged) ? 0 : 3;
  } catch (const std::exception& e) {
    std::printf("threw: %s\n", e.what());
    return 2;
  }
}
'''


def test_cpp_adapter_compiles_and_fails_loudly_without_gpu(tmp_path):
    if not os.path.isdir(REF):
        pytest.skip("reference tree not present")
    src = tmp_path / "adapter.cpp"
    src.write_text(PROG)
    exe = tmp_path / "adapter"
    cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
    lib = os.path.join(ROOT, "paper_1204_1533_b200")
    cmd = [cxx, "-std=c++20", "-O1", "-I", os.path.join(ROOT, "oracle", "ref_build", "eigen_shim"),
           "-I", os.path.join(REF, "include"), "-I", os.path.join(ROOT, "include"), str(src),
           os.path.join(REF, "src", "basis.cpp"), os.path.join(REF, "src", "mesh.cpp"),
           os.path.join(REF, "src", "mapping.cpp"), "-L", lib, "-llinedg_b200", f"-Wl,-rpath,{lib}",
           "-o", str(exe)]
    subprocess.check_call(cmd)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    import torch

    if torch.cuda.is_available():
        assert r.returncode == 0, r.stdout + r.stderr
    else:
        assert r.returncode == 2 and "no CUDA device" in r.stdout, r.stdout + r.stderr
