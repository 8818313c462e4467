// halo.cuh - the halo row copies shared by the loopback exchange (misc.cu)
// and the NCCL exchange (comm.cu): "the overlap area of a given
// domain is updated from the neighboring domains' interiors"; Alg. 1 :411.
#pragma once
#include "common.cuh"

namespace dsmpnn {

// all same-device halo copies of one refresh in one launch: job j = blockIdx.y
// copies rows src[rows[r]] -> dst[r] of `row16` 16-byte chunks each
struct HaloJobs {
  static constexpr int kMax = 64;
  const uint4 *src[kMax];
  const int32_t *rows[kMax];
  uint4 *dst[kMax];
  int64_t n_rows[kMax];
};
static __global__ void halo_gather_jobs_kernel(const __grid_constant__ HaloJobs jobs, int row16) {
  const int j = blockIdx.y;
  const int64_t total = jobs.n_rows[j] * row16;
  const uint4 *__restrict__ src = jobs.src[j];
  const int32_t *__restrict__ rows = jobs.rows[j];
  uint4 *__restrict__ dst = jobs.dst[j];
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / row16, c = t - r * row16;
    dst[t] = src[(int64_t)rows[r] * row16 + c];
  }
}

}  // namespace dsmpnn
