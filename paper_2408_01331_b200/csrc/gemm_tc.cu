// tcgen05 3xTF32 grouped GEMM — placeholder until the tensor-core path lands.
#include "common.cuh"

namespace hnn {

int gemm_tc_tile_shape(int op, int32_t* tm, int32_t* tn) {
  set_error("hnn_gemm_tile_shape", "3xTF32 tensor-core path not built");
  return HNN_ERR_UNSUPPORTED;
}

int grouped_gemm_tc(int op, const hnn_gemm_problem* probs, int nprob, int total_tiles, const hnn_step_row* cur,
                    const hnn_model_status* status, cudaStream_t s) {
  set_error("hnn_grouped_gemm", "3xTF32 tensor-core path not built");
  return HNN_ERR_UNSUPPORTED;
}

}  // namespace hnn
