// dz1w1.cuh - fused B5 + B6 of the BF16 layer backward (Alg. 1 :417, the
// first kappa_phi layer's gradients), tcgen05 (sm_100a).
//
// Per 128-edge tile (rows of dZ2 / e, in edge order), transposed so that
// kappa' runs over TMEM lanes and edges over TMEM columns:
//   z1^T  = W1 e^T                       (recomputed; a1 > 0 <=> bf16(relu(z1 + b1)) > 0
//                                         <=> z1 + b1 > 2^-134 in fp32)
//   dz1^T = (W2^T dz2^T) * [a1 > 0]      (bf16, never written to HBM)
//   dW1  += dz1^T e                      (tcgen05, accumulated in TMEM across tiles)
//   db1  += row sums of dz1^T            (per-thread registers: thread = kappa')
// This replaces B5 -> B6's dz1 round trip (write + read of 2k bytes per edge)
// and B5's read of A1 (2k bytes per edge): the kernel reads dz2 (2k B) and e
// (32 B) per edge.
//
// Work split: CTA pairs (2q, 2q+1) walk the same tiles; CTA h of a pair owns
// kappa' in [128h, 128h + 128) (the M = 128 lanes of its products), so its
// W2 half (64 KB) stays in SMEM.  Both CTAs of a pair read the same dz2 tile;
// the second read is an L2 hit.
//
// Warps: 0 TMA producer, 1 MMA issuer for z1 / dz1, 2..9 epilogue (TMEM lane
// group g = warp & 3 = 32 kappa', edge-column half cq = (warp - 2) >> 2),
// 10 MMA issuer for dW1 (separate, so the staging buffer is released as soon
// as the epilogue fills it, whatever the dz1 issuer is waiting on).
// TMEM (512 columns): Z [0,128) z1^T of the current tile; D0/D1 [128,384)
// dz1^T (double buffered); ACC [384,400) dW1.
// SMEM: W2^T half (4 K blocks x 2 x [64 kappa][64 kappa'] SW128, MN-major A),
// dz2 ring (S x [128 edges][64 kappa] SW128, K-major B), W1 half ([128][16]
// SW32, K-major A), e ring (4 x [128 edges][16] SW32: K-major B of z1,
// MN-major B of dW1), dz1^T staging ([2 edge blocks][128 kappa'][64 edges]
// SW128, K-major A of dW1).
#pragma once
#include "layer_bf16_common.cuh"
#include "tc.cuh"

namespace dsmpnn {

struct DZ1C {
  static constexpr int STAGES = 6;
  static constexpr int E_STAGES = 4;                // e tiles run ahead of the dz2 ring
  static constexpr int W2_BYTES = 4 * 16384;   // 4 K blocks of [64][128] bf16
  static constexpr int DZ_BYTES = 16384;       // [128 edges][64 kappa] bf16
  static constexpr int STG_BYTES = 32768;      // [128 kappa'][128 edges] bf16
  static constexpr int E_BYTES = 4096;         // [128 edges][16] bf16
  static constexpr int OFF_W2 = 0;
  static constexpr int OFF_DZ = OFF_W2 + W2_BYTES;
  static constexpr int OFF_STG = OFF_DZ + STAGES * DZ_BYTES;
  static constexpr int OFF_W1 = OFF_STG + STG_BYTES;
  static constexpr int OFF_E = OFF_W1 + 4096;
  static constexpr int OFF_BAR = OFF_E + E_STAGES * E_BYTES;
  static constexpr int SMEM = 1024 + OFF_BAR + 256;
  static constexpr uint32_t COL_Z = 0, COL_D = 128, COL_W = 384;
  static constexpr int THREADS = 352;
};

struct DZ1Bars {
  uint64_t wres;
  uint64_t dz_full[DZ1C::STAGES], dz_empty[DZ1C::STAGES];
  uint64_t e_full[DZ1C::E_STAGES], e_empty[DZ1C::E_STAGES];
  uint64_t z_full, z_free;
  uint64_t d_full[2], d_free[2];
  uint64_t s_ready, s_free;
  uint64_t acc_full;
  uint32_t tmem_slot;
};

// tW2: W2 [256 x 256] box {64, 64}; tW1: W1 [256 x 16] box {16, 128};
// tDZ: dz2 rows [eb, ee) box {64, 128}; tE: e rows [eb, ee) box {16, 128}.
// part_w [pairs][256][16]: this pair's dW1 sums; part_b [pairs][2][256]: db1
// sums of each edge-column half.
__global__ void __launch_bounds__(DZ1C::THREADS, 1)
    dz1w1_kernel(const __grid_constant__ CUtensorMap tW2, const __grid_constant__ CUtensorMap tW1,
                 const __grid_constant__ CUtensorMap tDZ, const __grid_constant__ CUtensorMap tE, int64_t nE,
                 const float *__restrict__ b1, float *__restrict__ part_w, float *__restrict__ part_b) {
  using C = DZ1C;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *sm = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  DZ1Bars *m = reinterpret_cast<DZ1Bars *>(sm + C::OFF_BAR);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int half = blockIdx.x & 1;
  const int64_t pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int64_t ntiles = (nE + 127) / 128;
  const int64_t nmine = pair < ntiles ? (ntiles - pair + npairs - 1) / npairs : 0;

  if (warp == 0 && lane == 0) {
    tc::mbar_init(&m->wres, 1);
    for (int s = 0; s < C::STAGES; ++s) {
      tc::mbar_init(&m->dz_full[s], 1);
      tc::mbar_init(&m->dz_empty[s], 1);
    }
    for (int b = 0; b < C::E_STAGES; ++b) {
      tc::mbar_init(&m->e_full[b], 1);
      tc::mbar_init(&m->e_empty[b], 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&m->d_full[b], 1);
      tc::mbar_init(&m->d_free[b], 8);
    }
    tc::mbar_init(&m->s_ready, 8);
    tc::mbar_init(&m->s_free, 1);
    tc::mbar_init(&m->z_full, 1);
    tc::mbar_init(&m->z_free, 8);
    tc::mbar_init(&m->acc_full, 1);
    tc::fence_mbar_init();
    tc::tma_prefetch(&tDZ);
    tc::tma_prefetch(&tE);
  }
  if (warp == 1) tc::tmem_alloc<512>(&m->tmem_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = m->tmem_slot;
  pdl_wait();  // dz2 / e of other kernels from here on
  pdl_trigger();

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (tc::elect_one()) {
      tc::mbar_expect_tx(&m->wres, C::W2_BYTES + 4096);
      for (int kb = 0; kb < 4; ++kb)
        for (int j = 0; j < 2; ++j)
          tc::tma_load_2d(sm + C::OFF_W2 + kb * 16384 + j * 8192, &tW2, &m->wres, half * 128 + j * 64, kb * 64);
      tc::tma_load_2d(sm + C::OFF_W1, &tW1, &m->wres, 0, half * 128);
      uint32_t it = 0;
      for (int64_t li = 0; li < nmine; ++li) {
        const int32_t e0 = (int32_t)((pair + li * npairs) * 128);
        const uint32_t se = (uint32_t)(li % C::E_STAGES);
        if (li >= C::E_STAGES) tc::mbar_wait(&m->e_empty[se], (uint32_t)(((li / C::E_STAGES) - 1) & 1));
        tc::mbar_expect_tx(&m->e_full[se], C::E_BYTES);
        tc::tma_load_2d(sm + C::OFF_E + se * C::E_BYTES, &tE, &m->e_full[se], 0, e0);
        for (int kb = 0; kb < 4; ++kb, ++it) {
          const uint32_t s = it % C::STAGES, r = it / C::STAGES;
          if (r > 0) tc::mbar_wait(&m->dz_empty[s], (r - 1) & 1);
          tc::mbar_expect_tx(&m->dz_full[s], C::DZ_BYTES);
          tc::tma_load_2d(sm + C::OFF_DZ + s * C::DZ_BYTES, &tDZ, &m->dz_full[s], kb * 64, e0);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------- MMA issuer: z1, dz1
    constexpr uint32_t ID1 = tc::idesc_bf16(128, 128, false, false);  // z1^T  = W1 E^T
    constexpr uint32_t ID2 = tc::idesc_bf16(128, 128, true, false);   // dz1^T = W2^T dZ2^T
    if (tc::elect_one()) {
      tc::mbar_wait(&m->wres, 0);
      const uint32_t aW2 = tc::smem_u32(sm + C::OFF_W2), aW1 = tc::smem_u32(sm + C::OFF_W1),
                     aDZ = tc::smem_u32(sm + C::OFF_DZ), aE = tc::smem_u32(sm + C::OFF_E);
      uint32_t it = 0;
      for (int64_t li = 0; li < nmine; ++li) {
        const uint32_t b = (uint32_t)(li & 1);
        // z1^T (Z is single-buffered: the epilogue drains it first)
        if (li >= 1) tc::mbar_wait(&m->z_free, (uint32_t)((li - 1) & 1));
        const uint32_t se = (uint32_t)(li % C::E_STAGES);
        tc::mbar_wait(&m->e_full[se], (uint32_t)((li / C::E_STAGES) & 1));
        tc::tc_fence_after();
        tc::mma_bf16_ss(tmem + C::COL_Z, tc::sdesc(aW1, 16, 256, tc::kSw32),
                        tc::sdesc(aE + se * C::E_BYTES, 16, 256, tc::kSw32), ID1, 0u);
        tc::mma_commit(&m->z_full);
        // dz1^T pre-mask into D[b]
        if (li >= 2) tc::mbar_wait(&m->d_free[b], (uint32_t)(((li >> 1) - 1) & 1));
        tc::tc_fence_after();
        const uint32_t dcol = tmem + C::COL_D + b * 128;
        for (int kb = 0; kb < 4; ++kb, ++it) {
          const uint32_t s = it % C::STAGES;
          tc::mbar_wait(&m->dz_full[s], (it / C::STAGES) & 1);
          tc::tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t ad = tc::sdesc(aW2 + kb * 16384 + kk * 2048, 8192, 1024, tc::kSw128);
            const uint64_t bd = tc::sdesc(aDZ + s * C::DZ_BYTES + kk * 32, 16, 1024, tc::kSw128);
            tc::mma_bf16_ss(dcol, ad, bd, ID2, (kb > 0 || kk > 0) ? 1u : 0u);
          }
          tc::mma_commit(&m->dz_empty[s]);
        }
        tc::mma_commit(&m->d_full[b]);
      }
    }
    __syncwarp();
  } else if (warp == 10) {
    // ------------------------------------------------- MMA issuer: dW1
    constexpr uint32_t ID3 = tc::idesc_bf16(128, 16, false, true);  // dW1 = dz1^T E
    if (tc::elect_one()) {
      const uint32_t aS = tc::smem_u32(sm + C::OFF_STG), aE = tc::smem_u32(sm + C::OFF_E);
      for (int64_t li = 0; li < nmine; ++li) {
        const uint32_t se = (uint32_t)(li % C::E_STAGES);
        tc::mbar_wait(&m->s_ready, (uint32_t)(li & 1));
        tc::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {  // 16 edges per step
          const uint64_t ad = tc::sdesc(aS + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024, tc::kSw128);
          const uint64_t bd = tc::sdesc(aE + se * C::E_BYTES + kk * 512, 2048, 256, tc::kSw32);
          tc::mma_bf16_ss(tmem + C::COL_W, ad, bd, ID3, (li > 0 || kk > 0) ? 1u : 0u);
        }
        tc::mma_commit(&m->s_free);
        tc::mma_commit(&m->e_empty[se]);
      }
      tc::mma_commit(&m->acc_full);
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ epilogue
    const int g = warp & 3, cq = (warp - 2) >> 2;
    const int krow = g * 32 + lane;  // kappa' - 128 * half = TMEM lane
    const uint32_t lane_off = (uint32_t)(g * 32) << 16;
    const float bias = b1[half * 128 + krow];
    float db = 0.f;
    for (int64_t li = 0; li < nmine; ++li) {
      const uint32_t b = (uint32_t)(li & 1);
      // a = z1 + b1 for this thread's kappa' and 64 edges
      tc::mbar_wait(&m->z_full, (uint32_t)(li & 1));
      tc::tc_fence_after();
      uint32_t x[64], y[64];
      tc::tmem_ld32(tmem + lane_off + C::COL_Z + cq * 64, *reinterpret_cast<uint32_t (*)[32]>(&x[0]));
      tc::tmem_ld32(tmem + lane_off + C::COL_Z + cq * 64 + 32, *reinterpret_cast<uint32_t (*)[32]>(&x[32]));
      tc::tmem_ld_wait();
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&m->z_free);
      // dz1 = D[b] * [bf16(relu(z1 + b1)) > 0]
      tc::mbar_wait(&m->d_full[b], (uint32_t)((li >> 1) & 1));
      tc::tc_fence_after();
      tc::tmem_ld32(tmem + lane_off + C::COL_D + b * 128 + cq * 64, *reinterpret_cast<uint32_t (*)[32]>(&y[0]));
      tc::tmem_ld32(tmem + lane_off + C::COL_D + b * 128 + cq * 64 + 32,
                    *reinterpret_cast<uint32_t (*)[32]>(&y[32]));
      tc::tmem_ld_wait();
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&m->d_free[b]);
      uint32_t pk[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float g0 = __uint_as_float(x[2 * j]) + bias > 0x1p-134f ? __uint_as_float(y[2 * j]) : 0.f;
        const float g1 = __uint_as_float(x[2 * j + 1]) + bias > 0x1p-134f ? __uint_as_float(y[2 * j + 1]) : 0.f;
        db += g0 + g1;
        pk[j] = tc::pack_bf16(g0, g1);
      }
      if (li >= 1) tc::mbar_wait(&m->s_free, (uint32_t)((li - 1) & 1));
      uint8_t *row = sm + C::OFF_STG + cq * 16384;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        *reinterpret_cast<uint4 *>(row + tc::sw128_off((uint32_t)krow, (uint32_t)u)) =
            make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
      tc::fence_async_shared();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&m->s_ready);
    }
    // per-pair partial sums: warps cq = 0 drain dW1; every warp writes its db1 half
    const int64_t kap = half * 128 + krow;
    part_b[(pair * 2 + cq) * 256 + kap] = db;
    if (cq == 0) {
      float4 *dst = reinterpret_cast<float4 *>(part_w + (pair * 256 + kap) * 16);
      if (nmine > 0) {
        tc::mbar_wait(&m->acc_full, 0);
        tc::tc_fence_after();
        uint32_t v[16];
        tc::tmem_ld16(tmem + lane_off + C::COL_W, v);
        tc::tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 4; ++j)
          dst[j] = make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                               __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3]));
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) dst[j] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc<512>(tmem);
}

// gW1[r, c] += sum_q part_w[q][r][c] (c < d_e), gb1[r] += sum_q sum_h part_b[q][h][r].
// One warp per output: lane l sums q = l, l + 32, ... then a butterfly; the
// order is fixed, so the result is run-to-run identical.
__global__ void dz1w1_reduce_kernel(const float *__restrict__ part_w, const float *__restrict__ part_b, int npairs,
                                    int d_e, float *__restrict__ gW1, float *__restrict__ gb1) {
  pdl_wait();
  pdl_trigger();
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int r = w / (d_e + 1), c = w - r * (d_e + 1);
  if (r >= KH) return;
  float *dst = c < d_e ? (gW1 ? gW1 + r * d_e + c : nullptr) : gb1 ? gb1 + r : nullptr;
  if (!dst) return;
  float s = 0.f;
  for (int q = lane; q < npairs; q += 32)
    s += c < d_e ? part_w[((int64_t)q * KH + r) * 16 + c]
                 : part_b[(int64_t)(2 * q) * KH + r] + part_b[(int64_t)(2 * q + 1) * KH + r];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) *dst += s;
}

}  // namespace dsmpnn
