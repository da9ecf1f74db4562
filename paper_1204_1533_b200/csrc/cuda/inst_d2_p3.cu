// Explicit instantiation of the sm_100a kernels for dim=2, p=3:
// Poisson, Euler (Roe, LLF), Navier-Stokes (Roe, LLF).
#include "ldg_ops.cuh"
LDG_DEFINE_OPS(2, 3, 0, 0)
LDG_DEFINE_OPS(2, 3, 1, 0)
LDG_DEFINE_OPS(2, 3, 1, 1)
LDG_DEFINE_OPS(2, 3, 2, 0)
LDG_DEFINE_OPS(2, 3, 2, 1)
