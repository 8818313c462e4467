// simt.cu - fp32 SIMT GEMM / column sums for the F32 mode.
#include "simt.cuh"

namespace dsmpnn {

constexpr int TM = 64, TN = 64, TK = 16;

__global__ void __launch_bounds__(256) sgemm_kernel(SgemmArgs a, int splits, int64_t k_chunk, float *partial,
                                                    int a_kfast, int b_nfast) {
  __shared__ float As[TK][TM + 4];
  __shared__ float Bs[TK][TN + 4];
  int tid = threadIdx.x;
  int tx = tid & 15, ty = tid >> 4;
  int64_t m0 = (int64_t)blockIdx.y * TM, n0 = (int64_t)blockIdx.x * TN;
  int64_t kb = (int64_t)blockIdx.z * k_chunk;
  int64_t ke = kb + k_chunk < a.K ? kb + k_chunk : a.K;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  for (int64_t k0 = kb; k0 < ke; k0 += TK) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      int e = tid + 256 * r;
      int mm, kk;
      if (a_kfast) { kk = e & 15; mm = e >> 4; } else { mm = e & 63; kk = e >> 6; }
      int64_t gm = m0 + mm, gk = k0 + kk;
      As[kk][mm] = (gm < a.M && gk < ke) ? a.A[gm * a.sam + gk * a.sak] : 0.f;
      int nn;
      if (b_nfast) { nn = e & 63; kk = e >> 6; } else { kk = e & 15; nn = e >> 4; }
      int64_t gn = n0 + nn;
      gk = k0 + kk;
      Bs[kk][nn] = (gn < a.N && gk < ke) ? a.B[gk * a.sbk + gn * a.sbn] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
      float av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int64_t gm = m0 + ty + 16 * i;
    if (gm >= a.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int64_t gn = n0 + tx + 16 * j;
      if (gn >= a.N) continue;
      if (splits > 1) {
        partial[((int64_t)blockIdx.z * a.M + gm) * a.N + gn] = acc[i][j];
      } else {
        float v = a.alpha * acc[i][j];
        if (a.bias) v += a.bias[gn];
        if (a.relu) v = fmaxf(v, 0.f);
        float *c = a.C + gm * a.ldc + gn;
        *c = a.beta ? *c + v : v;
      }
    }
  }
}

__global__ void splitk_reduce_kernel(SgemmArgs a, int splits, const float *__restrict__ partial) {
  int64_t total = a.M * a.N;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int z = 0; z < splits; ++z) s += partial[z * total + t];
    int64_t m = t / a.N, n = t - m * a.N;
    float v = a.alpha * s;
    if (a.bias) v += a.bias[n];
    if (a.relu) v = fmaxf(v, 0.f);
    float *c = a.C + m * a.ldc + n;
    *c = a.beta ? *c + v : v;
  }
}

dsmpnn_status sgemm(const SgemmArgs &a, int splits, float *partial, cudaStream_t s) {
  if (a.M <= 0 || a.N <= 0) return DSMPNN_OK;
  if (splits < 1) splits = 1;
  if (a.K <= 0) splits = 1;
  int64_t k_chunk = splits > 1 ? ceil_div(ceil_div(a.K, splits), TK) * TK : (a.K > 0 ? a.K : 1);
  if (splits > 1) splits = (int)ceil_div(a.K, k_chunk);
  dim3 grid((unsigned)ceil_div(a.N, TN), (unsigned)ceil_div(a.M, TM), (unsigned)splits);
  DS_CHECK_ARG(grid.y < 65536, DSMPNN_ERR_UNSUPPORTED, "sgemm: M too large for grid.y");
  int a_kfast = a.sak == 1 ? 1 : 0;
  int b_nfast = a.sbn == 1 ? 1 : 0;
  sgemm_kernel<<<grid, 256, 0, s>>>(a, splits, k_chunk, partial, a_kfast, b_nfast);
  DS_LAUNCH_CHECK();
  if (splits > 1) {
    int g = (int)std::min<int64_t>(ceil_div(a.M * a.N, 256), 148 * 8);
    splitk_reduce_kernel<<<g, 256, 0, s>>>(a, splits, partial);
    DS_LAUNCH_CHECK();
  }
  return DSMPNN_OK;
}

// one block per 32 columns; 32 row lanes per column, fixed reduction order
__global__ void __launch_bounds__(1024) colsum_kernel(const float *__restrict__ A, int64_t M, int64_t N, int64_t lda,
                                                      float *__restrict__ out, int accumulate) {
  pdl_wait();
  pdl_trigger();
  __shared__ float red[32][33];
  int c = threadIdx.x & 31, r = threadIdx.x >> 5;
  int64_t n = (int64_t)blockIdx.x * 32 + c;
  // 8 independent accumulators (loads in flight), combined in a fixed order
  float p[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (n < N) {
    int64_t m = r;
    for (; m + 7 * 32 < M; m += 8 * 32) {
#pragma unroll
      for (int u = 0; u < 8; ++u) p[u] += A[(m + u * 32) * lda + n];
    }
    for (; m < M; m += 32) p[0] += A[m * lda + n];
  }
  const float s = ((p[0] + p[1]) + (p[2] + p[3])) + ((p[4] + p[5]) + (p[6] + p[7]));
  red[r][c] = s;
  __syncthreads();
  if (r == 0 && n < N) {
    float t = 0.f;
    for (int k = 0; k < 32; ++k) t += red[k][c];
    out[n] = accumulate ? out[n] + t : t;
  }
}

__global__ void __launch_bounds__(1024) colsum_chunk_kernel(const float *__restrict__ A, int64_t M, int64_t N,
                                                            int64_t lda, int64_t chunk, float *__restrict__ ws) {
  __shared__ float red[32][33];
  const int c = threadIdx.x & 31, r = threadIdx.x >> 5;
  const int64_t n = (int64_t)blockIdx.x * 32 + c;
  const int64_t m0 = (int64_t)blockIdx.y * chunk, m1 = m0 + chunk < M ? m0 + chunk : M;
  float s = 0.f;
  if (n < N)
    for (int64_t m = m0 + r; m < m1; m += 32) s += A[m * lda + n];
  red[r][c] = s;
  __syncthreads();
  if (r == 0 && n < N) {
    float t = 0.f;
    for (int k = 0; k < 32; ++k) t += red[k][c];
    ws[(int64_t)blockIdx.y * N + n] = t;
  }
}

dsmpnn_status colsum(const float *A, int64_t M, int64_t N, int64_t lda, float *out, int accumulate, cudaStream_t s) {
  if (N <= 0 || !out) return DSMPNN_OK;
  DS_CUDA(launch_pdl(colsum_kernel, (unsigned)ceil_div(N, 32), 1024, 0, s, A, M, N, lda, out, accumulate));
  DS_LAUNCH_CHECK();
  return DSMPNN_OK;
}

dsmpnn_status colsum_ws(const float *A, int64_t M, int64_t N, int64_t lda, float *out, int accumulate, float *ws,
                        cudaStream_t s) {
  if (N <= 0 || !out) return DSMPNN_OK;
  if (!ws || M <= 2048) return colsum(A, M, N, lda, out, accumulate, s);
  const int64_t chunk = ceil_div(M, (int64_t)kColsumChunks);
  const int R = (int)ceil_div(M, chunk);
  // level 1: chunk r of rows -> ws[r, :]   (grid.y = chunk)
  colsum_chunk_kernel<<<dim3((unsigned)ceil_div(N, 32), R), 1024, 0, s>>>(A, M, N, lda, chunk, ws);
  DS_LAUNCH_CHECK();
  return colsum(ws, R, N, N, out, accumulate, s);
}

}  // namespace dsmpnn
