"""Full-size parity probe (diagnostic): GPU vs oracle residual and Jacobian
rows of 32 random elements on a config's own (unperturbed) state."""
import sys, time, json
import numpy as np
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import torch
from paper_1204_1533_b200 import CONFIGS, LDG_K11, LDG_K12, LDG_K21, LineDG
from oracle.pyoracle import Oracle


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


for ci in [int(a) for a in sys.argv[1:]]:
    cfg = CONFIGS[ci]
    case, U = cfg.build()
    gpu = LineDG(case, cfg.physics)
    ora = Oracle(case, cfg.physics)
    rng = np.random.default_rng(11)
    elems = np.sort(rng.choice(case.E, 32, replace=False)).astype(np.int32)
    m = gpu.m
    dofs = (elems[:, None] * case.npe * m + np.arange(case.npe * m)[None, :]).ravel()
    R = gpu.residual(torch.from_numpy(U).cuda()).cpu().numpy()
    R0 = ora.residual(U, elems=elems)
    out = {"config": ci + 1, "residual": rel(R[dofs], R0[dofs]), "maxR": float(np.abs(R0[dofs]).max())}
    gpu.assemble_jacobians(torch.from_numpy(U).cuda())
    ora.assemble(U, elems=elems)
    ws = [LDG_K11] + ([LDG_K12, LDG_K21] if cfg.physics.second_order() else [])
    for w in ws:
        r0, c0, v0 = ora.export_blocks(w)
        keep = np.isin(r0 // case.npe, elems)
        r1, c1, v1 = gpu.export_blocks(w, elems=elems)
        out[f"K{w}_pattern"] = bool(np.array_equal(r0[keep], r1) and np.array_equal(c0[keep], c1))
        out[f"K{w}"] = rel(v1, v0[keep])
    print(json.dumps(out), flush=True)
    gpu.close()
