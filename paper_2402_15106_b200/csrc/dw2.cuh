// dw2.cuh - B4 of the BF16 layer backward without the A1 round trip
// (Alg. 1 :417, the second kappa_phi layer's weight gradient), tcgen05 (sm_100a).
//
//   dW2[kappa, kappa'] += sum_p dz2[p, kappa] a1[p, kappa'],
//   a1 = bf16(relu(e W1^T + b1))  recomputed per 128-edge tile on tcgen05,
// so the edge kernel does not write A1 (2k bytes per edge) and this kernel
// reads dz2 (2k B) and e (32 B) per edge instead of dz2 + A1 (4k B).
//
// Work split: CTA pairs (2q, 2q+1) walk the same tiles; CTA h owns kappa' in
// [128h, 128h + 128): its z1^T half (M = 128 kappa' lanes, N = 128 edges,
// K = 16) and its dW2 column half, accumulated in TMEM across all its tiles
// (two M = 128 kappa halves x N = 128).  Both CTAs of a pair read the same
// dz2 tile; the second read is an L2 hit.
//
// Warps: 0 TMA producer, 1 MMA issuer, 2..9 epilogue (TMEM lane group
// g = warp & 3, edge half cq = (warp - 2) >> 2): a1 = bf16(relu(z1 + b1)) in
// registers -> staging row (K-major B of the dW2 product).
// TMEM (512 columns): Z0/Z1 [0,256) z1^T (double buffered); ACC [256,512)
// dW2 (kappa half m at 256 + 128m).
// SMEM: dz2 ring (8 x [128 edges][64 kappa] SW128; the 4 blocks of a tile are
// the MN-major A = dz2^T, 64-kappa chunks 16 KB apart), a1 staging (2 x [2
// edge blocks][128 kappa'][64 edges] SW128), W1 half ([128][16] SW32), e ring
// (4 x [128 edges][16] SW32).
#pragma once
#include "layer_bf16_common.cuh"
#include "tc.cuh"

namespace dsmpnn {

struct DW2C {
  static constexpr int STAGES = 8;               // two tiles of dz2 (even: a tile's 64-kappa block pairs never wrap)
  static constexpr int E_STAGES = 4;
  static constexpr int DZ_BYTES = 16384;         // [128 edges][64 kappa] bf16
  static constexpr int STG_BYTES = 32768;        // [128 kappa'][128 edges] bf16
  static constexpr int E_BYTES = 4096;
  static constexpr int OFF_DZ = 0;
  static constexpr int OFF_STG = OFF_DZ + STAGES * DZ_BYTES;
  static constexpr int OFF_W1 = OFF_STG + 2 * STG_BYTES;
  static constexpr int OFF_E = OFF_W1 + 4096;
  static constexpr int OFF_BAR = OFF_E + E_STAGES * E_BYTES;
  static constexpr int SMEM = 1024 + OFF_BAR + 256;
  static constexpr uint32_t COL_Z = 0, COL_ACC = 256;
  static constexpr int THREADS = 320;
};

struct DW2Bars {
  uint64_t wres;
  uint64_t dz_full[DW2C::STAGES], dz_empty[DW2C::STAGES];
  uint64_t e_full[DW2C::E_STAGES], e_empty[DW2C::E_STAGES];
  uint64_t z_full[2], z_free[2];
  uint64_t s_ready[2], s_free[2];
  uint64_t acc_full;
  uint32_t tmem_slot;
};

// tW1: W1 [256 x 16] box {16, 128}; tDZ: dz2 rows [eb, ee) box {64, 128};
// tE: e rows [eb, ee) box {16, 128}.  part [pairs][256 kappa][256 kappa']:
// this pair's dW2 sums.
__global__ void __launch_bounds__(DW2C::THREADS, 1)
    dw2_kernel(const __grid_constant__ CUtensorMap tW1, const __grid_constant__ CUtensorMap tDZ,
               const __grid_constant__ CUtensorMap tE, int64_t nE, const float *__restrict__ b1,
               float *__restrict__ part) {
  using C = DW2C;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *sm = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  DW2Bars *m = reinterpret_cast<DW2Bars *>(sm + C::OFF_BAR);
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
    for (int s = 0; s < C::E_STAGES; ++s) {
      tc::mbar_init(&m->e_full[s], 1);
      tc::mbar_init(&m->e_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&m->z_full[b], 1);
      tc::mbar_init(&m->z_free[b], 8);
      tc::mbar_init(&m->s_ready[b], 8);
      tc::mbar_init(&m->s_free[b], 1);
    }
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
      tc::mbar_expect_tx(&m->wres, 4096);
      tc::tma_load_2d(sm + C::OFF_W1, &tW1, &m->wres, 0, half * 128);
      // e runs up to E_STAGES tiles ahead; dz2 tile li waits for MMA4(li - 2)
      int64_t le = 0;
      auto issue_e = [&](int64_t upto) {
        for (; le < nmine && le <= upto; ++le) {
          const uint32_t se = (uint32_t)(le % C::E_STAGES);
          if (le >= C::E_STAGES) tc::mbar_wait(&m->e_empty[se], (uint32_t)(((le / C::E_STAGES) - 1) & 1));
          tc::mbar_expect_tx(&m->e_full[se], C::E_BYTES);
          tc::tma_load_2d(sm + C::OFF_E + se * C::E_BYTES, &tE, &m->e_full[se], 0,
                          (int32_t)((pair + le * npairs) * 128));
        }
      };
      issue_e(1);
      uint32_t it = 0;
      for (int64_t li = 0; li < nmine; ++li) {
        const int32_t e0 = (int32_t)((pair + li * npairs) * 128);
        for (int kb = 0; kb < 4; ++kb, ++it) {
          const uint32_t s = it % C::STAGES, r = it / C::STAGES;
          if (r > 0) tc::mbar_wait(&m->dz_empty[s], (r - 1) & 1);
          tc::mbar_expect_tx(&m->dz_full[s], C::DZ_BYTES);
          tc::tma_load_2d(sm + C::OFF_DZ + s * C::DZ_BYTES, &tDZ, &m->dz_full[s], kb * 64, e0);
        }
        issue_e(li + 2);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer
    constexpr uint32_t ID1 = tc::idesc_bf16(128, 128, false, false);  // z1^T = W1 E^T
    constexpr uint32_t ID4 = tc::idesc_bf16(128, 128, true, false);   // dW2  = dZ2^T A1
    if (tc::elect_one()) {
      tc::mbar_wait(&m->wres, 0);
      const uint32_t aW1 = tc::smem_u32(sm + C::OFF_W1), aDZ = tc::smem_u32(sm + C::OFF_DZ),
                     aS = tc::smem_u32(sm + C::OFF_STG), aE = tc::smem_u32(sm + C::OFF_E);
      auto mma1 = [&](int64_t l) {
        const uint32_t b = (uint32_t)(l & 1), se = (uint32_t)(l % C::E_STAGES);
        if (l >= 2) tc::mbar_wait(&m->z_free[b], (uint32_t)(((l >> 1) - 1) & 1));
        tc::mbar_wait(&m->e_full[se], (uint32_t)((l / C::E_STAGES) & 1));
        tc::tc_fence_after();
        tc::mma_bf16_ss(tmem + C::COL_Z + b * 128, tc::sdesc(aW1, 16, 256, tc::kSw32),
                        tc::sdesc(aE + se * C::E_BYTES, 16, 256, tc::kSw32), ID1, 0u);
        tc::mma_commit(&m->z_full[b]);
        tc::mma_commit(&m->e_empty[se]);
      };
      if (nmine > 0) mma1(0);
      for (int64_t li = 0; li < nmine; ++li) {
        const uint32_t b = (uint32_t)(li & 1);
        if (li + 1 < nmine) mma1(li + 1);
        // dW2 += dZ2^T A1 over this tile's 128 edges
        tc::mbar_wait(&m->s_ready[b], (uint32_t)((li >> 1) & 1));
        const uint32_t s0 = (uint32_t)((li * 4) % C::STAGES);
        for (int kb = 0; kb < 4; ++kb) {
          const uint32_t it = (uint32_t)(li * 4 + kb);
          tc::mbar_wait(&m->dz_full[it % C::STAGES], (it / C::STAGES) & 1);
        }
        tc::tc_fence_after();
#pragma unroll
        for (int mh = 0; mh < 2; ++mh) {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {  // 16 edges per step
            const uint64_t ad = tc::sdesc(aDZ + ((s0 + 2 * mh) % C::STAGES) * C::DZ_BYTES + kk * 2048,
                                          C::DZ_BYTES, 1024, tc::kSw128);
            const uint64_t bd =
                tc::sdesc(aS + b * C::STG_BYTES + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024, tc::kSw128);
            tc::mma_bf16_ss(tmem + C::COL_ACC + mh * 128, ad, bd, ID4, (li > 0 || kk > 0) ? 1u : 0u);
          }
        }
        for (int kb = 0; kb < 4; ++kb) tc::mma_commit(&m->dz_empty[(s0 + kb) % C::STAGES]);
        tc::mma_commit(&m->s_free[b]);
      }
      tc::mma_commit(&m->acc_full);
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ epilogue
    const int g = warp & 3, cq = (warp - 2) >> 2;
    const int krow = g * 32 + lane;  // kappa' - 128 * half = TMEM lane of Z
    const uint32_t lane_off = (uint32_t)(g * 32) << 16;
    const float bias = b1[half * 128 + krow];
    for (int64_t li = 0; li < nmine; ++li) {
      const uint32_t b = (uint32_t)(li & 1);
      tc::mbar_wait(&m->z_full[b], (uint32_t)((li >> 1) & 1));
      tc::tc_fence_after();
      uint32_t x[64];
      tc::tmem_ld32(tmem + lane_off + C::COL_Z + b * 128 + cq * 64, *reinterpret_cast<uint32_t (*)[32]>(&x[0]));
      tc::tmem_ld32(tmem + lane_off + C::COL_Z + b * 128 + cq * 64 + 32,
                    *reinterpret_cast<uint32_t (*)[32]>(&x[32]));
      tc::tmem_ld_wait();
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&m->z_free[b]);
      uint32_t pk[32];
#pragma unroll
      for (int j = 0; j < 32; ++j)
        pk[j] = tc::pack_bf16(fmaxf(__uint_as_float(x[2 * j]) + bias, 0.f),
                              fmaxf(__uint_as_float(x[2 * j + 1]) + bias, 0.f));
      if (li >= 2) tc::mbar_wait(&m->s_free[b], (uint32_t)(((li >> 1) - 1) & 1));
      uint8_t *row = sm + C::OFF_STG + b * C::STG_BYTES + cq * 16384;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        *reinterpret_cast<uint4 *>(row + tc::sw128_off((uint32_t)krow, (uint32_t)u)) =
            make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
      tc::fence_async_shared();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&m->s_ready[b]);
    }
    // this pair's dW2 block [256 kappa][128 kappa'] -> SMEM (rows padded to
    // 528 B: conflict-free 16-byte stores) -> coalesced rows of part.  Warp
    // (g, cq) drains kappa half cq (TMEM lanes = kappa rows 32g ..).
    float *stage = reinterpret_cast<float *>(sm + C::OFF_DZ);  // ring idle after acc_full
    constexpr int LDS = 132;
    if (nmine > 0) {
      tc::mbar_wait(&m->acc_full, 0);
      tc::tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < 128; c += 32) {
        uint32_t v[32];
        tc::tmem_ld32(tmem + lane_off + C::COL_ACC + cq * 128 + c, v);
        tc::tmem_ld_wait();
        float4 *srow = reinterpret_cast<float4 *>(stage + (cq * 128 + krow) * LDS + c);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          srow[j] = make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                                __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3]));
      }
    }
    tc::named_sync(1, 256);
    const int t = threadIdx.x - 64;  // 0..255
    for (int i = t; i < 256 * 32; i += 256) {  // 32 float4 per kappa row
      const int r = i >> 5, q = i & 31;
      const float4 val = nmine > 0 ? *reinterpret_cast<const float4 *>(stage + r * LDS + 4 * q)
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
      reinterpret_cast<float4 *>(part + (pair * 256 + r) * 256 + half * 128)[q] = val;
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc<512>(tmem);
}

// dW2 partials -> gW2 in two fixed-order passes: pass 1 sums pair groups
// (blockIdx.y = group of ceil(npairs / kDw2Groups) pairs) into tmp[group];
// pass 2 adds the groups in order.  Deterministic run to run.
constexpr int kDw2Groups = 8;
__global__ void dw2_reduce1_kernel(const float4 *__restrict__ part, int npairs, float4 *__restrict__ tmp) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= KH * KH / 4) return;
  const int per = (npairs + kDw2Groups - 1) / kDw2Groups;
  const int p0 = blockIdx.y * per, p1 = min(npairs, p0 + per);
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int p = p0; p < p1; ++p) {
    const float4 v = part[(int64_t)p * (KH * KH / 4) + i];
    s.x += v.x;
    s.y += v.y;
    s.z += v.z;
    s.w += v.w;
  }
  tmp[(int64_t)blockIdx.y * (KH * KH / 4) + i] = s;
}
__global__ void dw2_reduce2_kernel(const float4 *__restrict__ tmp, float4 *__restrict__ gW2) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= KH * KH / 4) return;
  float4 s = gW2[i];
#pragma unroll
  for (int g = 0; g < kDw2Groups; ++g) {
    const float4 v = tmp[(int64_t)g * (KH * KH / 4) + i];
    s.x += v.x;
    s.y += v.y;
    s.z += v.z;
    s.w += v.w;
  }
  gW2[i] = s;
}

}  // namespace dsmpnn
