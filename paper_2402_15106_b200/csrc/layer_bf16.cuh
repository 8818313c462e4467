// layer_bf16.cuh - BF16 mode of the layer: tcgen05 (sm_100a) kernels.
#pragma once
#include "common.cuh"

namespace dsmpnn {

dsmpnn_status bf16_check_desc(const dsmpnn_layer_desc &d);
size_t bf16_packed_bytes(const dsmpnn_layer_desc &d);
dsmpnn_status bf16_pack(const dsmpnn_layer_desc &d, const dsmpnn_weights &w, void *packed, cudaStream_t s);
size_t bf16_fwd_ws_bytes(const dsmpnn_layer_desc &d, int64_t n_dst, int64_t E);
size_t bf16_bwd_ws_bytes(const dsmpnn_layer_desc &d, int64_t n_dst, int64_t n_loc, int64_t E);
dsmpnn_status bf16_fwd(const dsmpnn_layer_desc &d, const dsmpnn_weights &w, const __nv_bfloat16 *v,
                       const __nv_bfloat16 *e, const int64_t *row_ptr, const int32_t *col, int64_t n_dst, int64_t E,
                       int64_t rb, int64_t re, int64_t eb, int64_t ee, float *out, __nv_bfloat16 *out_lowp, void *ws,
                       size_t ws_bytes, cudaStream_t s);
dsmpnn_status bf16_bwd(const dsmpnn_layer_desc &d, const dsmpnn_weights &w, const __nv_bfloat16 *v,
                       const __nv_bfloat16 *e, const int64_t *row_ptr, const int32_t *col, const int32_t *perm,
                       const int64_t *cptr, int64_t n_dst, int64_t n_loc, int64_t E, int64_t rb, int64_t re,
                       int64_t eb, int64_t ee, const float *G, float *dv, float *de, const dsmpnn_grads &gr,
                       const void *ws, void *bws, size_t bws_bytes, cudaStream_t s);

}  // namespace dsmpnn
