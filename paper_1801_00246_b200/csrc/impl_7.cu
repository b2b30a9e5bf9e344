// Degree-7 instantiation of the kernels and their host dispatch (impl.cuh).
#include "impl.cuh"
IPDG_DEFINE_OPS(7)
