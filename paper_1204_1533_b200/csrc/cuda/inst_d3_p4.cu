// Explicit instantiation of the sm_100a kernels for dim=3, p=4:
// Poisson, Euler (Roe, LLF), Navier-Stokes (Roe, LLF).
#include "ldg_ops.cuh"
LDG_DEFINE_OPS(3, 4, 0, 0)
LDG_DEFINE_OPS(3, 4, 1, 0)
LDG_DEFINE_OPS(3, 4, 1, 1)
LDG_DEFINE_OPS(3, 4, 2, 0)
LDG_DEFINE_OPS(3, 4, 2, 1)
