// The 6-planes-per-thread instantiations of the tensor-ring kernel (see spmv_pattern_tma.cu), built as their own
// translation unit so that the two halves compile in parallel.
#define SPMVB_RING_TU_Q6 1
#include "spmv_pattern_tma.cu"
