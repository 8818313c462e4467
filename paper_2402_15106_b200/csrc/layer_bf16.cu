// layer_bf16.cu - BF16 mode (tcgen05) of the layer.  (stub: filled in next)
#include "layer_bf16.cuh"

namespace dsmpnn {

dsmpnn_status bf16_check_desc(const dsmpnn_layer_desc &d) {
  DS_CHECK_ARG(false, DSMPNN_ERR_UNSUPPORTED, "layer: BF16 mode not built yet");
  return DSMPNN_OK;
}
size_t bf16_packed_bytes(const dsmpnn_layer_desc &) { return 0; }
dsmpnn_status bf16_pack(const dsmpnn_layer_desc &, const dsmpnn_weights &, void *, cudaStream_t) {
  return DSMPNN_ERR_UNSUPPORTED;
}
size_t bf16_fwd_ws_bytes(const dsmpnn_layer_desc &, int64_t, int64_t) { return 0; }
size_t bf16_bwd_ws_bytes(const dsmpnn_layer_desc &, int64_t, int64_t, int64_t) { return 0; }
dsmpnn_status bf16_fwd(const dsmpnn_layer_desc &, const dsmpnn_weights &, const __nv_bfloat16 *,
                       const __nv_bfloat16 *, const int64_t *, const int32_t *, int64_t, int64_t, int64_t, int64_t,
                       int64_t, int64_t, float *, __nv_bfloat16 *, void *, size_t, cudaStream_t) {
  return DSMPNN_ERR_UNSUPPORTED;
}
dsmpnn_status bf16_bwd(const dsmpnn_layer_desc &, const dsmpnn_weights &, const __nv_bfloat16 *,
                       const __nv_bfloat16 *, const int64_t *, const int32_t *, const int32_t *, const int64_t *,
                       int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, const float *, float *, float *,
                       const dsmpnn_grads &, const void *, void *, size_t, cudaStream_t) {
  return DSMPNN_ERR_UNSUPPORTED;
}

}  // namespace dsmpnn
