// instantiation of the NTD kernels for K=1 cells per lane (see ntd.cu)
#include "ntd_kernels.cuh"
#include "ntd_apply_ts.cuh"
NTD_INSTANTIATE(1)
NTD_INSTANTIATE_TS(1)
