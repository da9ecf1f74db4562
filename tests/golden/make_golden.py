"""Generates tests/golden/*.npz: small seeded cases with the CPU oracle's
residual, gradient, Jacobian blocks and products.  The reference's own
hot-path sources do not exist, so these fixtures are oracle
outputs frozen as regression vectors; the oracle itself is pinned by
tests/test_oracle_kats.py (SPEC.md KATs, Table-1 goldens) and
tests/test_setup_vs_reference.py (the reference's basis/mesh/mapping code).

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.pyoracle import Oracle  # noqa: E402
from paper_1204_1533_b200 import CONFIGS  # noqa: E402

# (config index, n, p) -- the configs' own meshes/states, scaled down (3-D at p=2 keeps files small)
CASES = [(0, 3, None), (1, 3, None), (2, 3, None), (3, 2, 2), (4, 2, 2)]


def make(ci, n, p):
    cfg = CONFIGS[ci]
    case, U = cfg.build(n=n, p=p)
    o = Oracle(case, cfg.physics)
    src = cfg.source_for(case)
    if src is not None:
        o.set_source(src)
    x = case.normal_vector(o.m, cfg.vector_seed)
    out = {"U": U, "x": x, "R": o.residual(U)}
    o.assemble(U)
    r, c, v = o.export_blocks(0)
    out.update(K11_rows=r, K11_cols=c, K11_vals=v, y11=o.spmv(0, x))
    if cfg.physics.second_order():
        out["Q"] = o.gradient(U)
        for w, mat in ((1, "K12"), (2, "K21")):
            r, c, v = o.export_blocks(w)
            out.update({f"{mat}_rows": r, f"{mat}_cols": c, f"{mat}_vals": v})
        out["split"] = o.split_matvec(0.37, x)
    np.savez_compressed(os.path.join(HERE, name(ci, n, p)), **out)


def name(ci, n, p):
    return f"golden_c{ci + 1}_n{n}" + (f"_p{p}" if p else "") + ".npz"


if __name__ == "__main__":
    for ci, n, p in CASES:
        make(ci, n, p)
        print("wrote", name(ci, n, p))
