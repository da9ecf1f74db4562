"""B200-native (sm_100a) hot path of the line-based DG scheme of arXiv 1204.1533.

Product: the CUDA library ``liblinedg_b200.so`` (residual, LDG gradient,
analytic Jacobian assembly into a line-structured block store, block SpMV and
split matvec) behind the C-ABI ``include/linedg_b200.h``; the setup library
``liblinedg_host.so`` (basis / mesh / mapping / generators); and this Python
mirror of the reference API.
"""
from . import _abi
from ._abi import LDG_EULER, LDG_K11, LDG_K12, LDG_K21, LDG_LLF, LDG_NAVIER_STOKES, LDG_POISSON, LDG_ROE
from .cases import CONFIGS, Case, Config, Physics
from .linedg import ConfigError, LineDG, PhysicalStateError, SolverError

__all__ = [
    "LineDG", "Case", "Config", "Physics", "CONFIGS", "ConfigError", "PhysicalStateError",
    "SolverError", "LDG_POISSON", "LDG_EULER", "LDG_NAVIER_STOKES", "LDG_ROE", "LDG_LLF", "LDG_K11",
    "LDG_K12", "LDG_K21",
]
