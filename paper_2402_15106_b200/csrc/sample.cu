// sample.cu - a1 Nystrom node sampling (Alg. 1 :391; reading R9).
// keys k_g = key_node(seed, g) for g in [0,N); stable radix sort of (k_g, g)
// (stability gives the g tie-break); flag the first min(s,N); compact the
// flags in id order, which yields the ids ascending.
#include <cub/cub.cuh>

#include "common.cuh"
#include "hash.cuh"

namespace dsmpnn {

__global__ void sample_keys_kernel(uint64_t s0, int64_t n, uint64_t *keys, int32_t *ids) {
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < n; g += (int64_t)gridDim.x * blockDim.x) {
    keys[g] = key_node(s0, (uint64_t)g);
    ids[g] = (int32_t)g;
  }
}

__global__ void sample_flag_kernel(const int32_t *sorted_ids, int64_t n, int64_t s, int32_t *flags) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    flags[sorted_ids[t]] = t < s ? 1 : 0;
}

__global__ void sample_compact_kernel(const int32_t *flags, const int32_t *pos, int64_t n, int32_t *out) {
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < n; g += (int64_t)gridDim.x * blockDim.x)
    if (flags[g]) out[pos[g]] = (int32_t)g;
}

static size_t sample_ws(int64_t n, size_t *sort_tmp, size_t *scan_tmp) {
  cub::DeviceRadixSort::SortPairs(nullptr, *sort_tmp, (const uint64_t *)nullptr, (uint64_t *)nullptr,
                                  (const int32_t *)nullptr, (int32_t *)nullptr, (int)n);
  cub::DeviceScan::ExclusiveSum(nullptr, *scan_tmp, (const int32_t *)nullptr, (int32_t *)nullptr, (int)n);
  Carver c(nullptr, 0);
  c.take<uint64_t>(n); c.take<uint64_t>(n); c.take<int32_t>(n); c.take<int32_t>(n);
  c.take<int32_t>(n); c.take<int32_t>(n);
  c.take<char>(*sort_tmp); c.take<char>(*scan_tmp);
  return c.used();
}

}  // namespace dsmpnn

using namespace dsmpnn;

extern "C" {

dsmpnn_status dsmpnn_sample_workspace_size(int64_t n_points, size_t *bytes) {
  DS_CHECK_ARG(n_points >= 0 && n_points < (1ll << 31), DSMPNN_ERR_INVALID_ARG, "sample: N out of range");
  size_t a, b;
  *bytes = sample_ws(n_points, &a, &b);
  return DSMPNN_OK;
}

dsmpnn_status dsmpnn_sample(int64_t n_points, int64_t s, uint64_t seed, int32_t *ids, void *ws, size_t ws_bytes,
                            void *stream) {
  DS_CHECK_ARG(s >= 1 && n_points >= 0 && n_points < (1ll << 31), DSMPNN_ERR_INVALID_ARG,
               "sample: need s >= 1 and 0 <= N < 2^31 (s=%lld N=%lld)", (long long)s, (long long)n_points);
  if (n_points == 0) return DSMPNN_OK;
  cudaStream_t st = as_stream(stream);
  size_t sort_tmp, scan_tmp;
  size_t need = sample_ws(n_points, &sort_tmp, &scan_tmp);
  DS_CHECK_ARG(ws_bytes >= need, DSMPNN_ERR_CAPACITY, "sample: workspace %zu < %zu", ws_bytes, need);
  Carver c(ws, ws_bytes);
  int64_t n = n_points;
  uint64_t *keys = c.take<uint64_t>(n), *keys2 = c.take<uint64_t>(n);
  int32_t *idv = c.take<int32_t>(n), *idv2 = c.take<int32_t>(n);
  int32_t *flags = c.take<int32_t>(n), *pos = c.take<int32_t>(n);
  void *t1 = c.take<char>(sort_tmp), *t2 = c.take<char>(scan_tmp);
  int grid = (int)std::min<int64_t>(ceil_div(n, 256), 148 * 8);
  sample_keys_kernel<<<grid, 256, 0, st>>>(smx(seed), n, keys, idv);
  DS_LAUNCH_CHECK();
  DS_CUDA(cub::DeviceRadixSort::SortPairs(t1, sort_tmp, keys, keys2, idv, idv2, (int)n, 0, 64, st));
  sample_flag_kernel<<<grid, 256, 0, st>>>(idv2, n, s, flags);
  DS_CUDA(cub::DeviceScan::ExclusiveSum(t2, scan_tmp, flags, pos, (int)n, st));
  sample_compact_kernel<<<grid, 256, 0, st>>>(flags, pos, n, ids);
  DS_LAUNCH_CHECK();
  return DSMPNN_OK;
}

}  // extern "C"
