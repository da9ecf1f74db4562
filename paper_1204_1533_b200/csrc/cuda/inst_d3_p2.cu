// Explicit instantiation of the sm_100a kernels for dim=3, p=2:
// Poisson, Euler (Roe, LLF), Navier-Stokes (Roe, LLF).
#include "ldg_ops.cuh"
LDG_DEFINE_OPS(3, 2, 0, 0)
LDG_DEFINE_OPS(3, 2, 1, 0)
LDG_DEFINE_OPS(3, 2, 1, 1)
LDG_DEFINE_OPS(3, 2, 2, 0)
LDG_DEFINE_OPS(3, 2, 2, 1)
