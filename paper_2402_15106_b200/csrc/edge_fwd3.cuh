// edge_fwd3.cuh - fused edge kernel (forward), transposed second layer:
// kappa_phi MLP on tcgen05 + per-row S_i = H_i^T V_i with H^T read from TMEM,
// K_p never formed (layer_bf16.cu step 2).
//
// Per tile of whole rows (edge_fwd2.cuh tiling: each row padded to a multiple
// of 16 slots, at most NMAX rows / 128 slots):
//   MMA1  z1   = E W1^T                 TMEM Z, lane = slot, column = kappa
//   epi1  a1   = relu(z1 + b1)          -> SMEM AH [slot][kappa] (bf16)
//   MMA2  z2^T = W2 a1^T                TMEM Z, lane = kappa', column = slot
//                                       (A = resident W2, B = AH, two M halves)
//   epi2  h^T  = relu(z2^T + b2)        -> bf16 pairs back into TMEM Z in place
//                                       (lane kappa', column slot / 2): the A
//                                       operand layout of tcgen05.mma [a_tmem]
//   S     S_i[kappa'][c] = sum_p h^T[kappa'][p] v_j(p)[c]   (A = H^T in TMEM,
//                                       B = gathered V rows; TMEM S region)
//   epiB  S~_aug[i][c*k + kappa'] = bf16(S_i / deg_i)   (global)
// Compared with edge_fwd2 (z2 = a1 W2^T with h written back to SMEM): AH is
// free as soon as MMA2 has read it, so the next tile's a1 epilogue no longer
// waits for this tile's S products, and the h epilogue has a per-thread bias
// (thread = kappa') and no SMEM stores.
//
// Roles (16 warps): loader 0,2,3 (walker, e / v gathers), MMA 1, EPI_A 4-11
// (epi1: slot rows, two column groups; epi2: group cg drains M half cg),
// EPI_B 12-15.  TMEM: Z = columns 0..255 (z1, then z2^T half mh at 128*mh,
// h^T half mh packed at 128*mh .. 128*mh + 63), S = 256..511 (row g, half mh
// at 256 + 128*mh + g*D).
#pragma once
#include "edge_fwd2.cuh"

namespace dsmpnn {

// clock64 timeline of CTA 0 (development builds only: -DDSMPNN_TIMELINE;
// tools/timeline.py).  Slot s of tile t (< 32) at g_tl3[t * 32 + s].
#ifdef DSMPNN_TIMELINE
__device__ unsigned long long *g_tl3;
#define TL3(t, s) do { if (g_tl3 && blockIdx.x == 0 && (t) < 32) g_tl3[(t) * 32 + (s)] = clock64(); } while (0)
#else
#define TL3(t, s) do { } while (0)
#endif

struct Misc3 {
  TileDesc2 desc[2];
  uint64_t e_full[2], e_empty, desc_free[2];
  uint64_t v_full, v_empty, d1_full, a1_ready, d2_full[2], h_ready[2], s_full, s_free;
  uint64_t w2_full;  // resident W2 loaded (TMA)
  int64_t cur_row, row_end;
  uint32_t tmem;
  alignas(16) float b1[KH];  // read as float4
  alignas(16) float b2[KH];
};

template <int D>
struct EF3 {
  static constexpr int NMAX = D == 64 ? 2 : 4;
  static constexpr int W2_BYTES = KH * KH * 2;   // 131072
  static constexpr int AH_BYTES = 128 * KH * 2;  // 65536
  static constexpr int V_BYTES = 128 * D * 2;
  static constexpr int W1_BYTES = KH * 32;
  static constexpr int E_BYTES = 128 * 32;
  static constexpr int OFF_W2 = 0;
  static constexpr int OFF_AH = OFF_W2 + W2_BYTES;
  static constexpr int OFF_V = OFF_AH + AH_BYTES;
  static constexpr int OFF_W1 = OFF_V + V_BYTES;
  static constexpr int OFF_E = OFF_W1 + W1_BYTES;
  static constexpr int OFF_MISC = OFF_E + E_BYTES;
  static constexpr int SMEM = OFF_MISC + (int)sizeof(Misc3) + 1024;
  static_assert(SMEM <= 232448, "edge_fwd3: shared memory budget");
};

template <int D>
__global__ void __launch_bounds__(512, 1)
    edge_fwd3_kernel(const __grid_constant__ CUtensorMap tW2, const __nv_bfloat16 *__restrict__ e16,
                     const __nv_bfloat16 *__restrict__ v, const int64_t *__restrict__ row_ptr, int64_t rb, int64_t re,
                     int64_t eb, int64_t ee, Packed pw, const float *__restrict__ b1, const float *__restrict__ b2,
                     __nv_bfloat16 *__restrict__ S, int64_t kp, const int32_t *__restrict__ col) {
  using C = EF3<D>;
  constexpr int NMAX = C::NMAX;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *sm = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t *sW2 = sm + C::OFF_W2, *sAH = sm + C::OFF_AH, *sV = sm + C::OFF_V, *sW1 = sm + C::OFF_W1,
          *sE = sm + C::OFF_E;
  Misc3 *m = reinterpret_cast<Misc3 *>(sm + C::OFF_MISC);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // ---------------------------------------------------------------- setup
  if (tid == 0) {
    int64_t E = ee - eb;
    int64_t t0 = eb + E * (int64_t)blockIdx.x / gridDim.x;
    int64_t t1 = eb + E * (int64_t)(blockIdx.x + 1) / gridDim.x;
    auto lb = [&](int64_t t) {
      int64_t lo = rb, hi = re;
      while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (row_ptr[mid] < t) lo = mid + 1; else hi = mid;
      }
      return lo;
    };
    m->cur_row = blockIdx.x == 0 ? rb : lb(t0);
    m->row_end = blockIdx.x + 1 == gridDim.x ? re : lb(t1);
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&m->e_full[b], 96);
      tc::mbar_init(&m->desc_free[b], 1 + 8 + 4);  // MMA + every epilogue warp
      tc::mbar_init(&m->d2_full[b], 1);
      tc::mbar_init(&m->h_ready[b], 128);
    }
    tc::mbar_init(&m->e_empty, 1);
    tc::mbar_init(&m->v_full, 96);
    tc::mbar_init(&m->v_empty, 1);
    tc::mbar_init(&m->d1_full, 1);
    tc::mbar_init(&m->a1_ready, 256);
    tc::mbar_init(&m->s_full, 1);
    tc::mbar_init(&m->s_free, 4);
    tc::mbar_init(&m->w2_full, 1);
    tc::fence_mbar_init();
    tc::mbar_expect_tx(&m->w2_full, C::W2_BYTES);
    for (int j = 0; j < 4; ++j) tc::tma_load_2d(sW2 + j * (KH * 128), &tW2, &m->w2_full, j * 64, 0);
  }
  if (warp == 1) tc::tmem_alloc<512>(&m->tmem);
  {
    const uint4 *g1 = reinterpret_cast<const uint4 *>(pw.W1);
    for (int q = tid; q < KH * 2; q += 512) {
      int r = q / 2, u = q % 2;
      *reinterpret_cast<uint4 *>(sW1 + il_off(r, u)) = g1[q];
    }
    for (int q = tid; q < KH; q += 512) {
      m->b1[q] = b1[q];
      m->b2[q] = b2[q];
    }
  }
  tc::fence_async_shared();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = m->tmem;
  pdl_wait();  // v, e and S of other kernels from here on
  pdl_trigger();

  if (warp == 0 || warp == 2 || warp == 3) {
    // ============================================================ loader
    const int li = warp == 0 ? lane : (warp - 1) * 32 + lane;  // 0..95
    for (uint32_t t = 0;; ++t) {
      const int b = t & 1;
      TileDesc2 *dsc = &m->desc[b];
      if (t >= 2) tc::mbar_wait(&m->desc_free[b], ((t >> 1) - 1) & 1);
      if (warp == 0) walk_tile<NMAX>(m, dsc, row_ptr, lane);
      tc::named_sync(1, 96);
      if (warp == 0 && lane == 0) TL3(t, 0);
      if (!dsc->more) {
        tc::mbar_arrive(&m->e_full[b]);
        break;
      }
      constexpr int CH = D / 8;
      TileRegs<NMAX> tr;
      tr.load(dsc);
      int32_t pe[2], cj[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) pe[u] = (li + 96 * u < 128) ? tr.edge(li + 96 * u) : -1;
#pragma unroll
      for (int u = 0; u < 2; ++u) cj[u] = pe[u] >= 0 ? __ldg(col + pe[u]) : -1;
      uint4 ev[2][2], vv[2][CH];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
#pragma unroll
        for (int c = 0; c < 2; ++c)
          ev[u][c] = pe[u] >= 0 ? __ldg(reinterpret_cast<const uint4 *>(e16 + (int64_t)pe[u] * 16) + c)
                                : make_uint4(0, 0, 0, 0);
        if (pe[u] >= 0) {  // bias columns 13..15 = 1 (bf16 0x3F80): z1 = E W1^T includes + b1
          ev[u][1].z |= 0x3F800000u;
          ev[u][1].w = 0x3F803F80u;
        }
#pragma unroll
        for (int c = 0; c < CH; ++c)
          vv[u][c] = cj[u] >= 0 ? __ldg(reinterpret_cast<const uint4 *>(v + (int64_t)cj[u] * D) + c)
                                : make_uint4(0, 0, 0, 0);
      }
      if (t >= 1) tc::mbar_wait(&m->e_empty, (t - 1) & 1);
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        if (li + 96 * u >= 128) continue;
#pragma unroll
        for (int c = 0; c < 2; ++c) *reinterpret_cast<uint4 *>(sE + il_off(li + 96 * u, c)) = ev[u][c];
      }
      tc::fence_async_shared();
      tc::mbar_arrive(&m->e_full[b]);
      if (warp == 0 && lane == 0) TL3(t, 1);
      if (t >= 1) tc::mbar_wait(&m->v_empty, (t - 1) & 1);
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        if (li + 96 * u >= 128) continue;
#pragma unroll
        for (int c = 0; c < CH; ++c) *reinterpret_cast<uint4 *>(sV + v_off<D>(li + 96 * u, c)) = vv[u][c];
      }
      tc::fence_async_shared();
      tc::mbar_arrive(&m->v_full);
      if (warp == 0 && lane == 0) TL3(t, 2);
    }
  } else if (warp == 1) {
    // =============================================================== MMA
    if (lane == 0) {
      const uint32_t aW2 = tc::smem_u32(sW2), aAH = tc::smem_u32(sAH), aV = tc::smem_u32(sV),
                     aW1 = tc::smem_u32(sW1), aE = tc::smem_u32(sE);
      constexpr uint32_t IDESC1 = tc::idesc_bf16(128, KH, false, false);
      constexpr uint32_t IDESC2 = tc::idesc_bf16(128, 128, false, false);
      constexpr uint32_t IDESC_S = tc::idesc_bf16(128, D, false, true);
      const uint32_t tZ = tmem, tS = tmem + 256;
      // MMA1 of tile t: z1 = E W1^T (one K=16 step) into Z.  Issued after the
      // previous tile's S products, which read h^T from Z (tcgen05.mma of one
      // thread execute in issue order)
      auto mma1 = [&](uint32_t t) -> bool {
        const int b = t & 1;
        tc::mbar_wait(&m->e_full[b], (t >> 1) & 1);
        if (!m->desc[b].more) return false;
        tc::tc_fence_after();
        tc::mma_bf16_ss(tZ, tc::sdesc(aE, 128, 256, tc::kSwNone), tc::sdesc(aW1, 128, 256, tc::kSwNone), IDESC1, 0u);
        tc::mma_commit(&m->d1_full);
        tc::mma_commit(&m->e_empty);
        return true;
      };
      bool more = mma1(0);
      tc::mbar_wait(&m->w2_full, 0);
      for (uint32_t t = 0; more; ++t) {
        const int b = t & 1;
        const uint32_t p1 = t & 1;
        TileRegs<NMAX> tr;
        tr.load(&m->desc[b]);
        tc::mbar_arrive(&m->desc_free[b]);
        // MMA2: z2^T = W2 a1^T, M half mh (kappa' 128 mh ..) into Z columns 128 mh ..
        TL3(t, 3);
        tc::mbar_wait(&m->a1_ready, p1);
        TL3(t, 4);
        tc::tc_fence_after();
#pragma unroll 1
        for (int mh = 0; mh < 2; ++mh) {
#pragma unroll
          for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              uint64_t ad = tc::sdesc(aW2 + j * (KH * 128) + mh * (128 * 128) + kk * 32, 16, 1024, tc::kSw128);
              uint64_t bd = tc::sdesc(aAH + j * (128 * 128) + kk * 32, 16, 1024, tc::kSw128);
              tc::mma_bf16_ss(tZ + mh * 128, ad, bd, IDESC2, (j > 0 || kk > 0) ? 1u : 0u);
            }
          tc::mma_commit(&m->d2_full[mh]);
        }
        // S_i = H_i^T V_i per row and kappa' half; A = h^T from TMEM
        TL3(t, 5);
        tc::mbar_wait(&m->v_full, p1);
        TL3(t, 6);
        if (t >= 1) tc::mbar_wait(&m->s_free, (t - 1) & 1);
        TL3(t, 7);
#pragma unroll 1
        for (int mh = 0; mh < 2; ++mh) {
          tc::mbar_wait(&m->h_ready[mh], p1);
          TL3(t, 8 + mh);
          tc::tc_fence_after();
          // K steps of the tile's rows interleaved (q outer): consecutive
          // products go to different accumulators
          int nkmax = 0;
#pragma unroll
          for (int g = 0; g < NMAX; ++g)
            if (g < tr.nn) nkmax = max(nkmax, (tr.deg[g] + 15) >> 4);
          for (int q = 0; q < nkmax; ++q) {
#pragma unroll
            for (int g = 0; g < NMAX; ++g) {
              if (g >= tr.nn || q >= ((tr.deg[g] + 15) >> 4)) continue;
              const int s = tr.s0[g] + 16 * q;
              uint64_t bd = D == 64 ? tc::sdesc(aV + (s / 8) * 1024, 8192, 1024, tc::kSw128)
                                    : tc::sdesc(aV + (s / 8) * 512, 4096, 512, tc::kSw64);
              tc::mma_bf16_ts(tS + mh * 128 + g * D, tZ + mh * 128 + (uint32_t)(s >> 1), bd, IDESC_S,
                              q > 0 ? 1u : 0u);
            }
          }
        }
        tc::mma_commit(&m->s_full);
        tc::mma_commit(&m->v_empty);
        TL3(t, 10);
        more = mma1(t + 1);
        TL3(t, 11);
      }
    }
    __syncwarp();
  } else if (warp < 12) {
    // ============================================================= EPI_A
    const int grp = warp & 3, cg = (warp - 4) >> 2;
    const int erow = grp * 32 + lane;  // epi1: slot row == TMEM lane
    const uint32_t lane_off = (uint32_t)(grp * 32) << 16;
    const uint32_t rz = tmem + lane_off;
    // epi2 of M half cg: thread = kappa' = 128 cg + 32 grp + lane, bias constant
    const float bias2 = m->b2[cg * 128 + grp * 32 + lane];
    for (uint32_t t = 0;; ++t) {
      const int b = t & 1;
      const uint32_t ph = (t >> 1) & 1, p1 = t & 1;
      tc::mbar_wait(&m->e_full[b], ph);
      if (!m->desc[b].more) break;
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&m->desc_free[b]);
      // a1 = relu(z1 + b1) -> AH, columns 128 cg .. 128 cg + 127 (AH is free:
      // d1_full of this tile implies MMA2 of the previous tile completed)
      tc::mbar_wait(&m->d1_full, p1);
      if (lane == 0 && (warp == 4 || warp == 8)) TL3(t, 12 + (warp == 8));
      tc::tc_fence_after();
#pragma unroll 1
      for (int cc = 0; cc < 2; ++cc) {
        const int j = cg * 2 + cc;  // AH block (64 kappa)
        uint32_t x[64], pk[32];
        tc::tmem_ld32(rz + j * 64, *reinterpret_cast<uint32_t (*)[32]>(&x[0]));
        tc::tmem_ld32(rz + j * 64 + 32, *reinterpret_cast<uint32_t (*)[32]>(&x[32]));
        tc::tmem_ld_wait();
#pragma unroll
        for (int q = 0; q < 32; ++q)  // z1 holds + b1 (bias columns of E and W1)
          pk[q] = tc::pack_bf16_relu(__uint_as_float(x[2 * q]), __uint_as_float(x[2 * q + 1]));
        uint8_t *blk = sAH + j * (128 * 128);
#pragma unroll
        for (int c = 0; c < 8; ++c)
          *reinterpret_cast<uint4 *>(blk + tc::sw128_off(erow, c)) =
              make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
      }
      tc::fence_async_shared();
      tc::tc_fence_before();
      tc::mbar_arrive(&m->a1_ready);
      if (lane == 0 && (warp == 4 || warp == 8)) TL3(t, 14 + (warp == 8));
      // h^T = relu(z2^T + b2) for M half cg, packed in place: columns
      // [64 cc, 64 cc + 64) are read before the packed pairs of the same
      // slots are written to [32 cc, 32 cc + 32)
      tc::mbar_wait(&m->d2_full[cg], p1);
      if (lane == 0 && (warp == 4 || warp == 8)) TL3(t, 16 + (warp == 8));
      tc::tc_fence_after();
      const uint32_t rh = rz + cg * 128;
#pragma unroll 1
      for (int cc = 0; cc < 2; ++cc) {
        uint32_t x[64], pk[32];
        tc::tmem_ld32(rh + cc * 64, *reinterpret_cast<uint32_t (*)[32]>(&x[0]));
        tc::tmem_ld32(rh + cc * 64 + 32, *reinterpret_cast<uint32_t (*)[32]>(&x[32]));
        tc::tmem_ld_wait();
#pragma unroll
        for (int q = 0; q < 32; ++q)
          pk[q] = tc::pack_bf16_relu(__uint_as_float(x[2 * q]) + bias2, __uint_as_float(x[2 * q + 1]) + bias2);
        tc::tmem_st32(rh + cc * 32, pk);
      }
      tc::tmem_st_wait();
      tc::tc_fence_before();
      tc::mbar_arrive(&m->h_ready[cg]);
      if (lane == 0 && (warp == 4 || warp == 8)) TL3(t, 18 + (warp == 8));
    }
  } else {
    // ============================================================= EPI_B
    const int grp = warp & 3;
    const uint32_t lane_off = (uint32_t)(grp * 32) << 16;
    for (uint32_t t = 0;; ++t) {
      const int b = t & 1;
      const uint32_t ph = (t >> 1) & 1, p1 = t & 1;
      const TileDesc2 *dsc = &m->desc[b];
      tc::mbar_wait(&m->e_full[b], ph);
      if (!dsc->more) break;
      TileRegs<NMAX> tr;
      tr.load(dsc);
      int64_t node[NMAX];
#pragma unroll
      for (int g = 0; g < NMAX; ++g) node[g] = g < tr.nn ? dsc->node[g] : 0;
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&m->desc_free[b]);
      tc::mbar_wait(&m->s_full, p1);
      if (warp == 12 && lane == 0) TL3(t, 20);
      tc::tc_fence_after();
      const uint32_t r = tmem + 256 + lane_off;
      // S~_i layout [c][kappa] (kappa contiguous): lane pairs (kappa, kappa+1)
      // swap packed bf16 pairs so every 4-byte store of the warp covers 64
      // contiguous bytes of two S~ rows (columns c and c+1)
      const bool odd = lane & 1;
      const uint32_t sel = odd ? 0x3276u : 0x5410u;
#pragma unroll
      for (int g = 0; g < NMAX; ++g) {
        if (g >= tr.nn) break;
        const float inv = 1.0f / (float)tr.deg[g];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int kap = 128 * h + grp * 32 + lane;
          __nv_bfloat16 *dst = S + node[g] * kp + (odd ? 1 : 0) * KH + (kap & ~1);
          uint32_t x[D];
#pragma unroll
          for (int c0 = 0; c0 < D; c0 += 32)
            tc::tmem_ld32(r + h * 128 + g * D + c0, *reinterpret_cast<uint32_t (*)[32]>(&x[c0]));
          tc::tmem_ld_wait();
#pragma unroll
          for (int q = 0; q < D / 2; ++q) {
            const uint32_t own = tc::pack_bf16(__uint_as_float(x[2 * q]) * inv, __uint_as_float(x[2 * q + 1]) * inv);
            const uint32_t oth = __shfl_xor_sync(0xffffffffu, own, 1);
            const uint32_t pr = __byte_perm(own, oth, sel);
            asm volatile("st.global.L1::no_allocate.b32 [%0], %1;" ::"l"(dst + (int64_t)(2 * q) * KH), "r"(pr)
                         : "memory");
          }
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&m->s_free);
      if (warp == 12 && lane == 0) TL3(t, 21);
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc<512>(tmem);
}

}  // namespace dsmpnn
