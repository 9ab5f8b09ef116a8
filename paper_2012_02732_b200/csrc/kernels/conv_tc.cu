// tcgen05 / TMEM implicit-GEMM convolution (placeholder until the tensor-core
// path lands; the planner never selects K_CONV_TC before then).
#include "common.cuh"

namespace sw {
int launch_conv_tc(const sw_op_desc&, void*) { return (int)cudaErrorNotSupported; }
}  // namespace sw
