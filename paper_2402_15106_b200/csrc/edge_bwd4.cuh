// edge_bwd4.cuh - fused edge kernel (backward, step B3 of layer_bf16_bwd.cu):
// edge_bwd3's TMEM design (a1 / h as tcgen05 A operands, W2 resident, kappa
// bias through the MMA) with the dz2 tile leaving through the TMA engine.
// Per tile of whole rows (edge_fwd2.cuh tiling), recompute a1, h and form
//   U    = H dS_i         (M = 128 slots, N = NMAX * D, K = kappa)
//   dH^T = dS_i V_seg^T   (M = kappa halves, N = the row's slots, K = c)
// then dz2 = dH * [h > 0] -> dZ2 (global, bf16), u_p = U + dS_i[k] -> U
// (global, bf16; row upos[p] when upos is given) and per-CTA db2 partial sums.
//
// What changed against edge_bwd3 (whose per-tile chain ended with the dz2
// epilogue storing 64 KB to HBM at the write ceiling while the tensor cores
// waited for the z columns):
//  * the dz2 epilogue writes the tile's dz2 rows into the dS buffer (free once
//    U and dH have read it: 128 slots x 512 B = the 64 KB of dS) and the TMA
//    warp copies each tile row to dZ2 with one cp.async.bulk; the z columns
//    are released after the TMEM reads, so the next tile's MLP overlaps the
//    HBM write-back, and the dS of the next tile is loaded after the bulk
//    copies have read the buffer;
//  * [h > 0] bits: each thread packs its 32 slots' bits (vcmpne2 on the bf16
//    pairs), one 32 x 32 warp bit transpose gives every lane its kappa' word
//    (instead of 32 ballots and select chains per 32 kappa');
//  * per-tile dS buffer (rows at slots 0 .. nn-1) instead of a ring.
//
// Roles (16 warps): loader 0 (walker, e rows, dS_i[k] rows), loader 2 (v
// rows), warp 3 lane 16 (dS loads, dz2 bulk stores), MMA 1, EPI_A 4-11 (h,
// bits; then the dz2 epilogue of kappa half cg), EPI_B 12-15 (a1 epilogue,
// then the U epilogue).
// TMEM: Z = 0..255 (z2, then dH^T half h at 128 h + slot), A = 256..383 (z1
// kappa 0..127, then a1 packed, then h), U = 384..511 (z1 kappa 128..255,
// then U row g at 384 + g D).  z1 of tile t+1 goes to A and U as soon as U
// of tile t is drained, so the next tile's MLP starts while tile t's dz2
// drain still reads Z; MMA2 of tile t+1 waits for that drain (dh_free).
#pragma once
#include "edge_bwd3.cuh"

namespace dsmpnn {

#ifdef DSMPNN_TIMELINE
__device__ unsigned long long *g_tlb4;
#define TLB4(t, s) do { if (g_tlb4 && blockIdx.x == 0 && (t) < 32) g_tlb4[(t) * 32 + (s)] = clock64(); } while (0)
#else
#define TLB4(t, s) do { } while (0)
#endif

// dz2 for NS consecutive slots of one row (one TMEM wait) into the SMEM
// staging rows [slot][kappa] (512 B per slot): lane pairs (kappa, kappa+1)
// swap packed pairs so each 4-byte store holds two kappa of one slot.
// Returns the sum of the lane's fp32 dz2 values (db2 partial).
template <int NS>
__device__ __forceinline__ float dz2_stage(uint32_t taddr, uint64_t bits, int kap, int s_abs, uint32_t stage) {
  uint32_t x[NS];
  if constexpr (NS == 16) {
    tc::tmem_ld16(taddr, *reinterpret_cast<uint32_t (*)[16]>(&x[0]));
  } else {
#pragma unroll
    for (int u = 0; u < NS / 32; ++u) tc::tmem_ld32(taddr + 32 * u, *reinterpret_cast<uint32_t (*)[32]>(&x[32 * u]));
  }
  tc::tmem_ld_wait();
  const bool odd = kap & 1;
  const uint32_t sel = odd ? 0x3276u : 0x5410u;
  const uint32_t base = stage + (uint32_t)(s_abs + (odd ? 1 : 0)) * 512u + (uint32_t)(kap & ~1) * 2u;
  float acc = 0.f;
#pragma unroll
  for (int q = 0; q < NS / 2; ++q) {
    const uint32_t m0 = 0u - (uint32_t)((bits >> (2 * q)) & 1u), m1 = 0u - (uint32_t)((bits >> (2 * q + 1)) & 1u);
    const float d0 = __uint_as_float(x[2 * q] & m0), d1 = __uint_as_float(x[2 * q + 1] & m1);
    acc += d0 + d1;
    const uint32_t own = tc::pack_bf16(d0, d1);
    const uint32_t oth = __shfl_xor_sync(0xffffffffu, own, 1);
    const uint32_t pr = __byte_perm(own, oth, sel);
    asm volatile("st.shared.b32 [%0], %1;" ::"r"(base + (uint32_t)(2 * q) * 512u), "r"(pr) : "memory");
  }
  return acc;
}

template <int D>
struct EB4 {
  static constexpr int NMAX = D == 64 ? 2 : 4;
  static constexpr int W2_BYTES = KH * KH * 2;  // 128 KB, resident
  static constexpr int DS_BYTES = KH * D * 2;   // 32 / 16 KB per row
  static constexpr int STAGE_BYTES = 128 * KH * 2;
  static_assert(NMAX * DS_BYTES == STAGE_BYTES, "the dS buffer doubles as the dz2 staging tile");
  static constexpr int V_BYTES = 128 * D * 2;
  static constexpr int W1_BYTES = KH * 32;
  static constexpr int E_BYTES = 128 * 32;
  static constexpr int MASK_BYTES = 4 * KH * 4;
  static constexpr int OFF_W2 = 0;
  static constexpr int OFF_DS = OFF_W2 + W2_BYTES;
  static constexpr int OFF_V = OFF_DS + STAGE_BYTES;
  static constexpr int OFF_W1 = OFF_V + V_BYTES;
  static constexpr int OFF_E = OFF_W1 + W1_BYTES;
  static constexpr int OFF_MASK = OFF_E + E_BYTES;
  static constexpr int OFF_B2 = OFF_MASK + MASK_BYTES;
  static constexpr int OFF_MISC = OFF_B2 + KH * 4;
  struct Misc {
    TileDescB desc[2];
    __nv_bfloat16 brow[2][NMAX][D];
    uint64_t e_full[2], desc_free[2];
    uint64_t ds_full, e_empty, v_full, v_empty, d1_full, a1_ready, d2_full, h_ready, a_free;
    uint64_t u_full, u_free, dh_full, dh_free, staged, w2_full, z_free;
    int64_t cur_row, row_end;
    uint32_t tmem;
  };
  static constexpr int SMEM = OFF_MISC + (int)sizeof(Misc);
  static_assert(SMEM <= 232448, "edge_bwd4: shared memory budget");
  static constexpr uint32_t ROWB = D * 2;
  static constexpr uint32_t SWZ = D == 64 ? tc::kSw128 : tc::kSw64;
};

template <int D>
__global__ void __launch_bounds__(512, 1)
    edge_bwd4_kernel(const __grid_constant__ CUtensorMap tW2, const __grid_constant__ CUtensorMap tDS,
                     const __nv_bfloat16 *__restrict__ e16, const __nv_bfloat16 *__restrict__ v,
                     const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col, int64_t rb, int64_t re,
                     int64_t eb, int64_t ee, Packed pw, const float *__restrict__ b2,
                     const __nv_bfloat16 *__restrict__ dS, __nv_bfloat16 *__restrict__ dZ2g,
                     __nv_bfloat16 *__restrict__ Ug, const int32_t *__restrict__ upos,
                     float *__restrict__ db2_part) {
  using C = EB4<D>;
  using Misc = typename C::Misc;
  constexpr int NMAX = C::NMAX;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *sm = smem_raw;
  uint8_t *sW2 = sm + C::OFF_W2, *sDS = sm + C::OFF_DS, *sV = sm + C::OFF_V, *sW1 = sm + C::OFF_W1,
          *sE = sm + C::OFF_E;
  uint32_t *sMask = reinterpret_cast<uint32_t *>(sm + C::OFF_MASK);
  float *sB2 = reinterpret_cast<float *>(sm + C::OFF_B2);
  Misc *m = reinterpret_cast<Misc *>(sm + C::OFF_MISC);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // ---------------------------------------------------------------- setup
  if (tid == 0) {
    if (tc::smem_u32(smem_raw) & 1023u) __trap();
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
      tc::mbar_init(&m->e_full[b], 32);
      tc::mbar_init(&m->desc_free[b], 1 + 8 + 4 + 1 + 1);  // MMA, epilogue warps, TMA warp, v loader
    }
    tc::mbar_init(&m->ds_full, 1);
    tc::mbar_init(&m->e_empty, 1);
    tc::mbar_init(&m->v_full, 32);
    tc::mbar_init(&m->v_empty, 1);
    tc::mbar_init(&m->d1_full, 1);
    tc::mbar_init(&m->a1_ready, 128);  // EPI_B (the a1 epilogue)
    tc::mbar_init(&m->d2_full, 1);
    tc::mbar_init(&m->h_ready, 256);
    tc::mbar_init(&m->a_free, 1);
    tc::mbar_init(&m->u_full, 1);
    tc::mbar_init(&m->u_free, 128);
    tc::mbar_init(&m->dh_full, 1);
    tc::mbar_init(&m->dh_free, 256);
    tc::mbar_init(&m->staged, 256);
    tc::mbar_init(&m->z_free, 256);
    tc::mbar_init(&m->w2_full, 1);
    tc::fence_mbar_init();
    tc::tma_prefetch(&tDS);
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
    for (int q = tid; q < KH; q += 512) sB2[q] = b2[q];
  }
  tc::fence_async_shared();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = m->tmem;
  const uint32_t tZ = tmem, tA = tmem + 256, tU = tmem + 384;
  pdl_wait();  // dS, v, e and the outputs of other kernels from here on
  pdl_trigger();

  if (warp == 0 || warp == 2) {
    // ============================================================ loaders
    constexpr int CH = D / 8;
    for (uint32_t t = 0;; ++t) {
      const int b = t & 1;
      TileDescB *dsc = &m->desc[b];
      if (warp == 0) {
        if (t >= 2) tc::mbar_wait(&m->desc_free[b], ((t >> 1) - 1) & 1);
        walk_tile<NMAX>(m, dsc, row_ptr, lane);
        if (!dsc->more) {
          tc::mbar_arrive(&m->e_full[b]);
          break;
        }
        TileRegs<NMAX> tr;
        tr.load(dsc);
        int32_t pe[4];
        uint4 ev[4][2];
#pragma unroll
        for (int u = 0; u < 4; ++u) pe[u] = tr.edge(lane + 32 * u);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
#pragma unroll
          for (int c = 0; c < 2; ++c)
            ev[u][c] = pe[u] >= 0 ? __ldg(reinterpret_cast<const uint4 *>(e16 + (int64_t)pe[u] * 16) + c)
                                  : make_uint4(0, 0, 0, 0);
          if (pe[u] >= 0) {  // bias columns 13..15 = 1 (bf16 0x3F80): z1 = E W1^T includes + b1
            ev[u][1].z |= 0x3F800000u;
            ev[u][1].w = 0x3F803F80u;
          }
        }
        for (int q = lane; q < tr.nn * CH; q += 32) {
          const int g = q / CH, c = q % CH;
          reinterpret_cast<uint4 *>(&m->brow[b][g][0])[c] =
              __ldg(reinterpret_cast<const uint4 *>(dS + (dsc->node[g] * (KH + 1) + KH) * D) + c);
        }
        if (t >= 1) tc::mbar_wait(&m->e_empty, (t - 1) & 1);
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int c = 0; c < 2; ++c) *reinterpret_cast<uint4 *>(sE + il_off(lane + 32 * u, c)) = ev[u][c];
        tc::fence_async_shared();
        tc::mbar_arrive(&m->e_full[b]);
      } else {
        tc::mbar_wait(&m->e_full[b], (t >> 1) & 1);
        if (!dsc->more) break;
        TileRegs<NMAX> tr;
        tr.load(dsc);
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&m->desc_free[b]);
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
          int32_t cj[2];
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int32_t pe = tr.edge(lane + 32 * (2 * h + u));
            cj[u] = pe >= 0 ? __ldg(col + pe) : -1;
          }
          uint4 vv[2][CH];
#pragma unroll
          for (int u = 0; u < 2; ++u)
#pragma unroll
            for (int c = 0; c < CH; ++c)
              vv[u][c] = cj[u] >= 0 ? __ldg(reinterpret_cast<const uint4 *>(v + (int64_t)cj[u] * D) + c)
                                    : make_uint4(0, 0, 0, 0);
          if (h == 0 && t >= 1) tc::mbar_wait(&m->v_empty, (t - 1) & 1);
#pragma unroll
          for (int u = 0; u < 2; ++u)
#pragma unroll
            for (int c = 0; c < CH; ++c)
              *reinterpret_cast<uint4 *>(sV + v_off<D>(lane + 32 * (2 * h + u), c)) = vv[u][c];
        }
        tc::fence_async_shared();
        tc::mbar_arrive(&m->v_full);
      }
    }
  } else if (warp == 3) {
    // ================================= dz2 bulk stores of tile t-1, dS loads of tile t
    if (lane == 16) {
      int np = 0;                // rows of the previous tile
      int64_t peb[NMAX];         // their first edge
      int32_t ps0[NMAX], pdeg[NMAX];
#pragma unroll
      for (int g = 0; g < NMAX; ++g) peb[g] = 0, ps0[g] = 0, pdeg[g] = 0;
      for (uint32_t t = 0;; ++t) {
        const int b = t & 1;
        const TileDescB *dsc = &m->desc[b];
        tc::mbar_wait(&m->e_full[b], (t >> 1) & 1);
        const bool more = dsc->more;
        const int nn = more ? dsc->nnodes : 0;
        int64_t node[NMAX], ebn[NMAX];
        int32_t s0n[NMAX], degn[NMAX];
#pragma unroll
        for (int g = 0; g < NMAX; ++g) {
          const bool ok = g < nn;
          node[g] = ok ? dsc->node[g] : 0;
          ebn[g] = ok ? dsc->ebase[g] : 0;
          s0n[g] = ok ? dsc->slot0[g] : 0;
          degn[g] = ok ? dsc->deg[g] : 0;
        }
        if (more) tc::mbar_arrive(&m->desc_free[b]);
        if (t >= 1) {  // tile t-1's dz2 rows are staged in the dS buffer
          tc::mbar_wait(&m->staged, (t - 1) & 1);
#pragma unroll
          for (int g = 0; g < NMAX; ++g)
            if (g < np && pdeg[g] > 0)
              tc::bulk_store_1d(dZ2g + peb[g] * KH, sDS + ps0[g] * (KH * 2), (uint32_t)pdeg[g] * (KH * 2));
          tc::bulk_commit();
          tc::bulk_wait_read<0>();  // the buffer may take the next dS
        }
        if (!more) break;
        tc::mbar_expect_tx(&m->ds_full, (uint32_t)nn * C::DS_BYTES);
#pragma unroll
        for (int g = 0; g < NMAX; ++g)
          if (g < nn) tc::tma_load_2d(sDS + g * C::DS_BYTES, &tDS, &m->ds_full, 0, (int32_t)(node[g] * (KH + 1)));
        np = nn;
#pragma unroll
        for (int g = 0; g < NMAX; ++g) peb[g] = ebn[g], ps0[g] = s0n[g], pdeg[g] = degn[g];
      }
      tc::bulk_wait<0>();  // every dz2 row written before the kernel ends
    }
    __syncwarp();
  } else if (warp == 1) {
    // =============================================================== MMA
    if (lane == 0) {
      const uint32_t aW2 = tc::smem_u32(sW2), aDS = tc::smem_u32(sDS), aV = tc::smem_u32(sV),
                     aW1 = tc::smem_u32(sW1), aE = tc::smem_u32(sE);
      constexpr uint32_t IDESC_MLP = tc::idesc_bf16(128, KH, false, false);
      constexpr uint32_t IDESC_MLP_H = tc::idesc_bf16(128, KH / 2, false, false);
      constexpr uint32_t IDESC_U = tc::idesc_bf16(128, NMAX * D, false, true);
      auto mma1 = [&](uint32_t t) -> bool {
        const int b = t & 1;
        tc::mbar_wait(&m->e_full[b], (t >> 1) & 1);
        if (!m->desc[b].more) return false;
        tc::tc_fence_after();
        // z1 in two kappa halves: 0..127 into A, 128..255 into U (both free once
        // U of the previous tile is drained), so the a1 epilogue of this tile
        // runs while the previous tile's dz2 drain still reads Z
        tc::mma_bf16_ss(tA, tc::sdesc(aE, 128, 256, tc::kSwNone), tc::sdesc(aW1, 128, 256, tc::kSwNone),
                        IDESC_MLP_H, 0u);
        tc::mma_bf16_ss(tU, tc::sdesc(aE, 128, 256, tc::kSwNone),
                        tc::sdesc(aW1 + (KH / 2 / 8) * 256, 128, 256, tc::kSwNone), IDESC_MLP_H, 0u);
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
        // MMA2: z2 = a1 W2^T (A = a1 in TMEM, W2 resident)
        TLB4(t, 0);
        tc::mbar_wait(&m->a1_ready, p1);
        if (t >= 1) tc::mbar_wait(&m->dh_free, (t - 1) & 1);  // the previous tile's dz2 drain has read Z
        TLB4(t, 1);
        tc::tc_fence_after();
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t bd = tc::sdesc(aW2 + j * (KH * 128) + kk * 32, 16, 1024, tc::kSw128);
            tc::mma_bf16_ts(tZ, tA + (uint32_t)(j * 32 + kk * 8), bd, IDESC_MLP, (j > 0 || kk > 0) ? 1u : 0u);
          }
        tc::mma_commit(&m->d2_full);
        // dH^T halves into Z as soon as the h epilogue has read z2 out of it
        // (dH needs neither h nor the bits), then U = H [dS_0 | dS_1 | ..]
        // with A = h in TMEM once h is written
        tc::mbar_wait(&m->ds_full, p1);
        tc::mbar_wait(&m->v_full, p1);
        tc::mbar_wait(&m->z_free, p1);
        TLB4(t, 2);
        tc::tc_fence_after();
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
#pragma unroll
          for (int g = 0; g < NMAX; ++g) {
            if (g >= tr.nn) break;
            const uint32_t ds = aDS + g * C::DS_BYTES;
            const int s0 = tr.s0[g];
            const uint32_t idesc_h = tc::idesc_bf16(128, (tr.deg[g] + 15) & ~15, false, false);
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
              uint64_t ad = tc::sdesc(ds + h * 128 * C::ROWB + kk * 32, 16, 8 * C::ROWB, C::SWZ);
              uint64_t bd = tc::sdesc(aV + (s0 / 8) * 8 * C::ROWB + kk * 32, 16, 8 * C::ROWB, C::SWZ);
              tc::mma_bf16_ss(tZ + h * 128 + s0, ad, bd, idesc_h, kk > 0 ? 1u : 0u);
            }
          }
        }
        tc::mma_commit(&m->v_empty);
        tc::mbar_wait(&m->h_ready, p1);
        TLB4(t, 3);
        TLB4(t, 4);  // U's region: freed before this tile's MMA1 (u_free of the previous tile)
        tc::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < KH / 16; ++kk) {
          uint64_t bd = tc::sdesc(aDS + kk * 16 * C::ROWB, C::DS_BYTES, 8 * C::ROWB, C::SWZ);
          tc::mma_bf16_ts(tU, tA + (uint32_t)(kk * 8), bd, IDESC_U, kk > 0 ? 1u : 0u);
        }
        tc::mma_commit(&m->u_full);
        tc::mma_commit(&m->a_free);
        tc::mma_commit(&m->dh_full);  // dH and U done: Z holds dH^T, the dS buffer is free
        TLB4(t, 5);
        // the next tile's MMA1 into A and U once this tile's U is drained
        tc::mbar_wait(&m->u_free, p1);
        TLB4(t, 6);
        tc::tc_fence_after();
        more = mma1(t + 1);
        TLB4(t, 7);
      }
    }
    __syncwarp();
  } else if (warp < 12) {
    // ============================================================= EPI_A
    const int grp = warp & 3, cg = (warp - 4) >> 2;
    const uint32_t lane_off = (uint32_t)(grp * 32) << 16;
    const uint32_t rz = tZ + lane_off, ra = tA + lane_off;
    const int kap = 128 * cg + grp * 32 + lane;  // dz2 epilogue
    const uint32_t stage = tc::smem_u32(sDS);
    // column of the transposed bit word held by this lane (see the h epilogue)
    const int tcol = lane < 16 ? 2 * lane : 2 * (lane - 16) + 1;
    float db2_acc = 0.f;
    for (uint32_t t = 0;; ++t) {
      const int b = t & 1;
      const uint32_t p1 = t & 1;
      const TileDescB *dsc = &m->desc[b];
      tc::mbar_wait(&m->e_full[b], (t >> 1) & 1);
      if (!dsc->more) break;
      TileRegs<NMAX> tr;
      tr.load(dsc);
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&m->desc_free[b]);
      // (a1 is formed by the EPI_B warps, below)
      // h = relu(z2 + b2) -> A, and the [h > 0] bits: the lane's 32 slot...
      // rather its own slot's 32 kappa' bits (bit q = kappa' c0 + 2q, bit
      // 16 + q = kappa' c0 + 2q + 1, from the bf16 pairs), transposed across
      // the warp so lane j holds the slot word of kappa' c0 + tcol(j)
      tc::mbar_wait(&m->d2_full, p1);
      if (warp == 4 && lane == 0) TLB4(t, 10);
      tc::tc_fence_after();
#pragma unroll 1
      for (int cc = 0; cc < 4; cc += 2) {
        const int cb = cg * 128 + cc * 32;  // 64 kappa' columns
        uint32_t xx[64], pk[32];
        tc::tmem_ld32(rz + cb, *reinterpret_cast<uint32_t (*)[32]>(&xx[0]));
        tc::tmem_ld32(rz + cb + 32, *reinterpret_cast<uint32_t (*)[32]>(&xx[32]));
        tc::tmem_ld_wait();
        if (cc == 2) {  // z2 fully read: dH may overwrite Z
          tc::tc_fence_before();
          tc::mbar_arrive(&m->z_free);
        }
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          const int c0 = cb + 32 * half;
          const uint32_t *x = &xx[32 * half];
          uint32_t row = 0;
#pragma unroll
          for (int q4 = 0; q4 < 8; ++q4) {
            const float4 bb = *reinterpret_cast<const float4 *>(sB2 + c0 + 4 * q4);
            const uint32_t p0 = tc::pack_bf16_relu(__uint_as_float(x[4 * q4]) + bb.x, __uint_as_float(x[4 * q4 + 1]) + bb.y);
            const uint32_t p2 =
                tc::pack_bf16_relu(__uint_as_float(x[4 * q4 + 2]) + bb.z, __uint_as_float(x[4 * q4 + 3]) + bb.w);
            pk[16 * half + 2 * q4] = p0;
            pk[16 * half + 2 * q4 + 1] = p2;
            // [h > 0] = nonzero bf16 (relu'd, sign bit cleared): pair q -> bits q, 16 + q
            row |= (__vcmpne2(p0 & 0x7FFF7FFFu, 0u) & 0x00010001u) << (2 * q4);
            row |= (__vcmpne2(p2 & 0x7FFF7FFFu, 0u) & 0x00010001u) << (2 * q4 + 1);
          }
          sMask[grp * KH + c0 + tcol] = tc::warp_transpose32(row, lane);
        }
        tc::tmem_st32(ra + cb / 2, pk);
      }
      tc::tmem_st_wait();
      tc::tc_fence_before();
      tc::mbar_arrive(&m->h_ready);
      if (warp == 4 && lane == 0) TLB4(t, 11);
      // dz2 = dH * [h > 0] for kappa half cg into the staging rows
      tc::mbar_wait(&m->h_ready, p1);  // every warp's bits are in sMask
      uint32_t mw[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) mw[u] = sMask[u * KH + kap];
      tc::mbar_wait(&m->dh_full, p1);  // dH and U done: the dS buffer is free
      if (warp == 4 && lane == 0) TLB4(t, 12);
      tc::tc_fence_after();
      {
        float acc = 0.f;
#pragma unroll 1
        for (int g = 0; g < NMAX; ++g) {
          if (g >= tr.nn) break;
          int s0 = tr.s0[0], deg = tr.deg[0];
#pragma unroll
          for (int i = 1; i < NMAX; ++i)
            if (g == i) {
              s0 = tr.s0[i];
              deg = tr.deg[i];
            }
          const int ns = (deg + 15) & ~15;
          const uint32_t ta = tZ + lane_off + cg * 128 + s0;
          if ((warp == 4 || warp == 8) && lane == 0 && g < 2) TLB4(t, 16 + 2 * g + (warp == 8 ? 4 : 0));
          int c0 = 0;
          for (; c0 + 64 <= ns; c0 += 64) acc += dz2_stage<64>(ta + c0, slot_bits(mw, s0 + c0), kap, s0 + c0, stage);
          if (c0 + 32 <= ns) {
            acc += dz2_stage<32>(ta + c0, slot_bits(mw, s0 + c0), kap, s0 + c0, stage);
            c0 += 32;
          }
          if (c0 < ns) acc += dz2_stage<16>(ta + c0, slot_bits(mw, s0 + c0), kap, s0 + c0, stage);
          if ((warp == 4 || warp == 8) && lane == 0 && g < 2) TLB4(t, 17 + 2 * g + (warp == 8 ? 4 : 0));
        }
        db2_acc += acc;
      }
      tc::tc_fence_before();
      tc::mbar_arrive(&m->dh_free);
      tc::fence_async_shared();  // staging writes -> the bulk copies (async proxy)
      tc::mbar_arrive(&m->staged);
      if (warp == 4 && lane == 0) TLB4(t, 13);
    }
    db2_part[(int64_t)blockIdx.x * KH + kap] = db2_acc;
  } else {
    // ============================================================= EPI_B
    // U epilogue (thread <-> slot row): u_p = U[slot] + dS_i[k]
    const int grp = warp & 3;
    const uint32_t lane_off = (uint32_t)(grp * 32) << 16;
    for (uint32_t t = 0;; ++t) {
      const int b = t & 1;
      const uint32_t p1 = t & 1;
      const TileDescB *dsc = &m->desc[b];
      tc::mbar_wait(&m->e_full[b], (t >> 1) & 1);
      if (!dsc->more) break;
      TileRegs<NMAX> tr;
      tr.load(dsc);
      const int nn = tr.nn;
      {
        // a1 = relu(z1) (z1 holds + b1): kappa 0..127 from A, 128..255 from U,
        // packed bf16 pairs to A columns 0..127 (lane = slot).  Each thread
        // reads its lane's A columns before it overwrites them; the U
        // columns are free for this tile's U product afterwards.
        tc::mbar_wait(&m->d1_full, p1);
        if (warp == 12 && lane == 0) TLB4(t, 8);
        tc::tc_fence_after();
        const uint32_t ra = tA + lane_off, ru = tU + lane_off;
        auto chunk = [&](uint32_t addr, uint32_t (&pk)[32]) {
          uint32_t x[64];
          tc::tmem_ld32(addr, *reinterpret_cast<uint32_t (*)[32]>(&x[0]));
          tc::tmem_ld32(addr + 32, *reinterpret_cast<uint32_t (*)[32]>(&x[32]));
          tc::tmem_ld_wait();
#pragma unroll
          for (int q = 0; q < 32; ++q)
            pk[q] = tc::pack_bf16_relu(__uint_as_float(x[2 * q]), __uint_as_float(x[2 * q + 1]));
        };
        uint32_t pk0[32], pk1[32];
        chunk(ra, pk0);       // kappa 0..63
        chunk(ra + 64, pk1);  // kappa 64..127
        tc::tmem_st32(ra, pk0);
        tc::tmem_st32(ra + 32, pk1);
        chunk(ru, pk0);       // kappa 128..191
        tc::tmem_st32(ra + 64, pk0);
        chunk(ru + 64, pk1);  // kappa 192..255
        tc::tmem_st32(ra + 96, pk1);
        tc::tmem_st_wait();
        tc::tc_fence_before();
        tc::mbar_arrive(&m->a1_ready);
        if (warp == 12 && lane == 0) TLB4(t, 9);
      }
      tc::mbar_wait(&m->u_full, p1);
      if (warp == 12 && lane == 0) TLB4(t, 14);
      tc::tc_fence_after();
      {
        const int s = grp * 32 + lane;
        const int p = tr.edge(s);
#pragma unroll
        for (int g = 0; g < NMAX; ++g) {
          if (g >= nn) break;
          const int g0 = tr.s0[g], gd = tr.deg[g];
          if (g0 >= grp * 32 + 32 || g0 + gd <= grp * 32) continue;  // row not in this warp's slots
          const bool mine = p >= 0 && s >= g0 && s < g0 + gd;
          const __nv_bfloat16 *brow = &m->brow[b][g][0];
          uint32_t xx[D];
#pragma unroll
          for (int c0 = 0; c0 < D; c0 += 32)
            tc::tmem_ld32(tU + lane_off + g * D + c0, *reinterpret_cast<uint32_t (*)[32]>(&xx[c0]));
          tc::tmem_ld_wait();
#pragma unroll
          for (int c0 = 0; c0 < D; c0 += 32) {
            const uint32_t *x = &xx[c0];
            if (mine) {
              // u_p goes to row upos[p] (its CSC position: the scatter then streams
              // each source's rows contiguously) or to row p
              const int64_t urow = upos ? (int64_t)__ldg(upos + p) : (int64_t)p;
              uint4 *dst = reinterpret_cast<uint4 *>(Ug + urow * D + c0);
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const uint4 bb = *reinterpret_cast<const uint4 *>(brow + c0 + 8 * u);
                const __nv_bfloat162 *bv = reinterpret_cast<const __nv_bfloat162 *>(&bb);
                uint32_t pk[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                  const float2 bf = __bfloat1622float2(bv[q]);
                  pk[q] = tc::pack_bf16(__uint_as_float(x[8 * u + 2 * q]) + bf.x,
                                        __uint_as_float(x[8 * u + 2 * q + 1]) + bf.y);
                }
                dst[u] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
              }
            }
          }
        }
      }
      tc::tc_fence_before();
      tc::mbar_arrive(&m->u_free);
      if (warp == 12 && lane == 0) TLB4(t, 15);
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&m->desc_free[b]);  // brow[b] read
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc<512>(tmem);
}

}  // namespace dsmpnn
