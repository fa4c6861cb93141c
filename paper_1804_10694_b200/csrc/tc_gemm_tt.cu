// tc_gemm_tt.cu -- instantiates the 3xTF32 tensor-core GEMM for op(A) = A^T, op(B) = B^T.
#include "tc_gemm.cuh"

namespace tmk {
template tm_status launch_tc_op<true, true>(const GemmArgs&, const TcChoice&, int, cudaStream_t);
}  // namespace tmk
