// instantiation of the NTD kernels for K=11 cells per lane (see ntd.cu)
#include "ntd_kernels.cuh"
NTD_INSTANTIATE(11)
