// edge_bwd2.cuh - pipelined, warp-specialised fused edge kernel (backward,
// step B3 of layer_bf16_bwd.cu).  Per tile of whole rows (edge_fwd2.cuh
// tiling): recompute a1, h on tcgen05; per row i of the tile
//   dH^T = dS_i V_seg^T   (M = kappa halves, N = the row's slots, K = c)
//   U    = H dS_i         (M = 128 slots, N = D, K = kappa)
// then  dz2 = dH * [h > 0]  -> dZ2 (global, bf16),  u_p = U + dS_i[k] -> U
// (global, bf16), a1 -> A1 (global, bf16; skipped when A1 is null: the
// unfused B4/B5 read it, dw2.cuh / dz1w1.cuh recompute a1) and per-CTA db2
// partial sums.
//
// Roles (16 warps):
//   loader (warps 0,2)  : tile walker, e / v row gathers (register staged),
//                         dS_i[k] bias rows
//   TMA    (warp 3)     : lane 0 streams W2 K-blocks (2-slot ring), lane 16
//                         streams dS_i tiles (2-slot ring)
//   MMA    (warp 1)     : tcgen05 issue
//   EPI_A  (warps 4-11) : a1 epilogue + coalesced a1 copy-out (overlaps MMA2),
//                         h epilogue + [h > 0] bitmask
//   EPI_B  (warps 12-15): U and dz2 epilogues
// TMEM: columns 0..255 z1 / z2; 256..383 U (row g at 256 + slot(g)*D), then,
// once EPI_B has drained U, dH^T kappa half 1 (slot s at 256 + s); 384..511
// dH^T kappa half 0.  z is free once the h epilogue has drained it, so MMA1 of
// the next tile is issued before this tile's U / dH products.
#pragma once
#include "edge_fwd2.cuh"

namespace dsmpnn {

struct TileDescB {
  int64_t node[4];
  int64_t ebase[4];  // row_ptr[node]
  int32_t slot0[4], deg[4];
  int32_t nnodes, more;
};

// edge held by tile slot s, or -1 for a padding slot
__device__ __forceinline__ int32_t slot_edge_of(const TileDescB *d, int nn, int s) {
  int32_t pe = -1;
  for (int g = 0; g < nn; ++g) {
    const int o = s - d->slot0[g];
    if (o >= 0 && o < d->deg[g]) pe = (int32_t)(d->ebase[g] + o);
  }
  return pe;
}

// [h > 0] bits of slots s .. s+63 (bit j = slot s + j) from the 128 slot bits
// w[0..3]; shifts and selects only (no register-array indexing)
__device__ __forceinline__ uint64_t slot_bits(const uint32_t (&w)[4], int s) {
  const uint64_t q0 = (uint64_t)w[0] | ((uint64_t)w[1] << 32), q1 = (uint64_t)w[2] | ((uint64_t)w[3] << 32);
  if (s == 0) return q0;
  if (s < 64) return (q0 >> s) | (q1 << (64 - s));
  return s == 64 ? q1 : q1 >> (s - 64);
}

// dz2 for NS consecutive slots of one row (one wait): dz2 = dH * [h > 0].
// Lane pairs (kappa, kappa+1) swap packed bf16 pairs so every 4-byte store
// of the warp covers 64 contiguous bytes of two dZ2 rows.  Returns the sum
// of the lane's fp32 dz2 values (db2 partial).
template <int NS>
__device__ __forceinline__ float dz2_chunk(uint32_t taddr, uint64_t bits, int kap, int c0, int deg,
                                           __nv_bfloat16 *__restrict__ dz2_row0) {
  uint32_t x[NS];
  if constexpr (NS == 16) {
    uint32_t (&y)[16] = *reinterpret_cast<uint32_t (*)[16]>(&x[0]);
    tc::tmem_ld16(taddr, y);
  } else {
#pragma unroll
    for (int u = 0; u < NS / 32; ++u) tc::tmem_ld32(taddr + 32 * u, *reinterpret_cast<uint32_t (*)[32]>(&x[32 * u]));
  }
  tc::tmem_ld_wait();
  const bool odd = kap & 1;
  const uint32_t sel = odd ? 0x3276u : 0x5410u;  // odd: (partner.hi, own.hi); even: (own.lo, partner.lo)
  __nv_bfloat16 *dst = dz2_row0 + (int64_t)(c0 + (odd ? 1 : 0)) * KH + (kap & ~1);
  float acc = 0.f;
#pragma unroll
  for (int q = 0; q < NS / 2; ++q) {
    const uint32_t m0 = 0u - (uint32_t)((bits >> (2 * q)) & 1u), m1 = 0u - (uint32_t)((bits >> (2 * q + 1)) & 1u);
    const float d0 = __uint_as_float(x[2 * q] & m0), d1 = __uint_as_float(x[2 * q + 1] & m1);
    acc += d0 + d1;  // padding slots hold dH = 0 (zero V rows)
    const uint32_t own = tc::pack_bf16(d0, d1);  // (slot 2q, slot 2q+1) of this kappa
    const uint32_t oth = __shfl_xor_sync(0xffffffffu, own, 1);
    const uint32_t pr = __byte_perm(own, oth, sel);
    if (c0 + 2 * q + (odd ? 1 : 0) < deg)
      asm volatile("st.global.L1::no_allocate.b32 [%0], %1;" ::"l"(dst + (int64_t)(2 * q) * KH), "r"(pr) : "memory");
  }
  return acc;
}

template <int D>
struct EB2 {
  static constexpr int NMAX = D == 64 ? 2 : 4;
  static constexpr int W2BLK = KH * 64 * 2;        // 32 KB
  static constexpr int AH_BYTES = 128 * KH * 2;    // 64 KB
  static constexpr int DS_BYTES = KH * D * 2;      // 32 / 16 KB
  static constexpr int V_BYTES = 128 * D * 2;
  static constexpr int W1_BYTES = KH * 32;
  static constexpr int E_BYTES = 128 * 32;
  static constexpr int MASK_BYTES = 4 * KH * 4;  // [slot/32][kappa] words, bit = slot % 32
  static constexpr int OFF_W2 = 0;
  static constexpr int OFF_AH = OFF_W2 + 2 * W2BLK;
  static constexpr int OFF_DS = OFF_AH + AH_BYTES;
  static constexpr int NDS = NMAX;                 // dS ring slots: every row of a tile resident
  static constexpr int OFF_V = OFF_DS + NDS * DS_BYTES;
  static constexpr int OFF_W1 = OFF_V + V_BYTES;
  static constexpr int OFF_E = OFF_W1 + W1_BYTES;
  static constexpr int OFF_MASK = OFF_E + E_BYTES;
  static constexpr int OFF_BIAS = OFF_MASK + MASK_BYTES;   // b1[KH], b2[KH] (fp32)
  static constexpr int OFF_MISC = OFF_BIAS + 2 * KH * 4;
  struct Misc {
    TileDescB desc[2];
    __nv_bfloat16 brow[2][NMAX][D];  // dS_i[k] of the rows of desc[b]
    uint64_t e_full[2], desc_free[2], w2_full[2], w2_empty[2], ds_full[NMAX], ds_empty[NMAX];
    uint64_t e_empty, v_full, v_empty, d1_full, a1_ready, d2_full, h_ready, ah_free, mask_read;
    uint64_t u_full, u_free, dh0_full, dh0_free, dh1_full, dh_free;
    int64_t cur_row, row_end;
    uint32_t tmem;
  };
  static constexpr int SMEM = OFF_MISC + (int)sizeof(Misc);
  static_assert(SMEM <= 232448, "edge_bwd2: shared memory budget");
  static constexpr uint32_t ROWB = D * 2;
  static constexpr uint32_t SWZ = D == 64 ? tc::kSw128 : tc::kSw64;
};

template <int D>
__global__ void __launch_bounds__(512, 1)
    edge_bwd2_kernel(const __grid_constant__ CUtensorMap tW2, const __grid_constant__ CUtensorMap tDS,
                     const __nv_bfloat16 *__restrict__ e16, const __nv_bfloat16 *__restrict__ v,
                     const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col, int64_t rb, int64_t re,
                     int64_t eb, int64_t ee, Packed pw, const float *__restrict__ b1, const float *__restrict__ b2,
                     const __nv_bfloat16 *__restrict__ dS, __nv_bfloat16 *__restrict__ A1g,
                     __nv_bfloat16 *__restrict__ dZ2g, __nv_bfloat16 *__restrict__ Ug, float *__restrict__ db2_part) {
  using C = EB2<D>;
  using Misc = typename C::Misc;
  constexpr int NMAX = C::NMAX;
  // 1024-byte aligned (SW128 operands); no slack is reserved, so check it
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *sm = smem_raw;
  uint8_t *sW2 = sm + C::OFF_W2, *sAH = sm + C::OFF_AH, *sDS = sm + C::OFF_DS, *sV = sm + C::OFF_V,
          *sW1 = sm + C::OFF_W1, *sE = sm + C::OFF_E;
  uint32_t *sMask = reinterpret_cast<uint32_t *>(sm + C::OFF_MASK);
  float *sB1 = reinterpret_cast<float *>(sm + C::OFF_BIAS), *sB2 = sB1 + KH;
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
      tc::mbar_init(&m->desc_free[b], 1 + 8 + 4 + 2 + 1);  // MMA, epilogue warps, TMA-W2, TMA-dS, v loader
      tc::mbar_init(&m->w2_full[b], 1);
      tc::mbar_init(&m->w2_empty[b], 1);
    }
    for (int b = 0; b < NMAX; ++b) {
      tc::mbar_init(&m->ds_full[b], 1);
      tc::mbar_init(&m->ds_empty[b], 1);
    }
    tc::mbar_init(&m->e_empty, 1);
    tc::mbar_init(&m->v_full, 32);
    tc::mbar_init(&m->v_empty, 1);
    tc::mbar_init(&m->d1_full, 1);
    tc::mbar_init(&m->a1_ready, 256);
    tc::mbar_init(&m->d2_full, 1);
    tc::mbar_init(&m->h_ready, 256);
    tc::mbar_init(&m->mask_read, 128);
    tc::mbar_init(&m->u_full, 1);
    tc::mbar_init(&m->u_free, 128);
    tc::mbar_init(&m->dh0_full, 1);
    tc::mbar_init(&m->dh0_free, 128);
    tc::mbar_init(&m->dh1_full, 1);
    tc::mbar_init(&m->dh_free, 128);
    tc::mbar_init(&m->ah_free, 1);
    tc::fence_mbar_init();
    tc::tma_prefetch(&tW2);
    tc::tma_prefetch(&tDS);
  }
  if (warp == 1) tc::tmem_alloc<512>(&m->tmem);
  {
    const uint4 *g1 = reinterpret_cast<const uint4 *>(pw.W1);
    for (int q = tid; q < KH * 2; q += 512) {
      int r = q / 2, u = q % 2;
      *reinterpret_cast<uint4 *>(sW1 + il_off(r, u)) = g1[q];
    }
    for (int q = tid; q < KH; q += 512) {
      sB1[q] = b1[q];
      sB2[q] = b2[q];
    }
  }
  tc::fence_async_shared();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = m->tmem;

  if (warp == 0 || warp == 2) {
    // ============================================================ loaders
    // warp 0: tile walker + e rows + dS_i[k] rows; warp 2: v_j rows.  The two
    // progress independently, so e (and MMA1) of the next tile never wait
    // for the v buffer, which is released only after the second dH half.
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
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int c = 0; c < 2; ++c)
            ev[u][c] = pe[u] >= 0 ? __ldg(reinterpret_cast<const uint4 *>(e16 + (int64_t)pe[u] * 16) + c)
                                  : make_uint4(0, 0, 0, 0);
        // dS_i[k] rows (the constant term of u_p) for EPI_B
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
        // two rows per lane per batch: index loads, then every row load in flight
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
    // ============================================================ TMA producers
    if (lane == 0) {  // W2 K-blocks in a 2-slot ring, K-block k in slot k & 1
      // Tile 0 loads all four; afterwards each tile first consumes the two
      // blocks the previous tile left in the ring (odd tiles: 2, 3; even
      // tiles: 0, 1) and loads only the other two, so one load per slot per
      // tile, each after the slot's first consumption of that tile
      uint32_t nload[2] = {0, 0};
      for (uint32_t t = 0;; ++t) {
        const int b = t & 1;
        tc::mbar_wait(&m->e_full[b], (t >> 1) & 1);
        if (!m->desc[b].more) break;
        tc::mbar_arrive(&m->desc_free[b]);
        const int k0 = t == 0 ? 0 : ((t & 1) ? 0 : 2), nk = t == 0 ? 4 : 2;
        for (int k = k0; k < k0 + nk; ++k) {
          const uint32_t sl = (uint32_t)(k & 1), i = ++nload[sl];  // i-th load into slot sl
          if (i >= 2) tc::mbar_wait(&m->w2_empty[sl], (i - 2) & 1);
          tc::mbar_expect_tx(&m->w2_full[sl], C::W2BLK);
          tc::tma_load_2d(sW2 + sl * C::W2BLK, &tW2, &m->w2_full[sl], k * 64, 0);
        }
      }
    } else if (lane == 16) {  // dS_i tiles, one per row, NMAX-slot ring
      uint32_t q = 0;
      for (uint32_t t = 0;; ++t) {
        const int b = t & 1;
        const TileDescB *dsc = &m->desc[b];
        tc::mbar_wait(&m->e_full[b], (t >> 1) & 1);
        if (!dsc->more) break;
        const int nn = dsc->nnodes;
        int64_t node[NMAX];
#pragma unroll
        for (int g = 0; g < NMAX; ++g) node[g] = g < nn ? dsc->node[g] : 0;
        tc::mbar_arrive(&m->desc_free[b]);
#pragma unroll
        for (int g = 0; g < NMAX; ++g) {
          if (g >= nn) break;
          const uint32_t s = q % C::NDS, r = q / C::NDS;
          if (r > 0) tc::mbar_wait(&m->ds_empty[s], (r - 1) & 1);
          tc::mbar_expect_tx(&m->ds_full[s], C::DS_BYTES);
          tc::tma_load_2d(sDS + s * C::DS_BYTES, &tDS, &m->ds_full[s], 0, (int32_t)(node[g] * (KH + 1)));
          ++q;
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // =============================================================== MMA
    if (lane == 0) {
      const uint32_t aW2 = tc::smem_u32(sW2), aAH = tc::smem_u32(sAH), aDS = tc::smem_u32(sDS),
                     aV = tc::smem_u32(sV), aW1 = tc::smem_u32(sW1), aE = tc::smem_u32(sE);
      constexpr uint32_t IDESC_MLP = tc::idesc_bf16(128, KH, false, false);
      constexpr uint32_t IDESC_U = tc::idesc_bf16(128, C::NDS * D, false, true);
      uint32_t w2l[2] = {0, 0}, dsq = 0;  // W2 loads consumed per slot
      auto mma1 = [&]() {  // z1 = E W1^T into columns 0..255
        tc::mma_bf16_ss(tmem, tc::sdesc(aE, 128, 256, tc::kSwNone), tc::sdesc(aW1, 128, 256, tc::kSwNone),
                        IDESC_MLP, 0u);
        tc::mma_commit(&m->d1_full);
        tc::mma_commit(&m->e_empty);
      };
      auto mma2 = [&](uint32_t t) {  // z2 = a1 W2^T (W2 K blocks through the 2-slot ring)
        tc::mbar_wait(&m->a1_ready, t & 1);
        tc::tc_fence_after();
#pragma unroll 1
        for (int jj = 0; jj < 4; ++jj) {
          // odd tiles start with blocks 2, 3 (left in the ring by the previous
          // tile), even tiles with 0, 1; tile 0 has all four loaded
          const int j = (t & 1) ? (jj + 2) & 3 : jj;
          const uint32_t s = (uint32_t)(j & 1);
          if (t == 0 || jj >= 2) {  // a freshly loaded block
            tc::mbar_wait(&m->w2_full[s], w2l[s] & 1);
            ++w2l[s];
          }
          tc::tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            uint64_t ad = tc::sdesc(aAH + j * (128 * 128) + kk * 32, 16, 1024, tc::kSw128);
            uint64_t bd = tc::sdesc(aW2 + s * C::W2BLK + kk * 32, 16, 1024, tc::kSw128);
            tc::mma_bf16_ss(tmem, ad, bd, IDESC_MLP, (jj > 0 || kk > 0) ? 1u : 0u);
          }
          if (jj < 2) tc::mma_commit(&m->w2_empty[s]);  // the slot's reload for this tile may start
        }
        tc::mma_commit(&m->d2_full);
      };
      tc::mbar_wait(&m->e_full[0], 0);
      bool more = m->desc[0].more;
      if (more) {
        tc::tc_fence_after();
        mma1();
        mma2(0);
      }
      for (uint32_t t = 0; more; ++t) {
        const int b = t & 1, nb = (t + 1) & 1;
        const uint32_t p1 = t & 1;
        TileRegs<NMAX> tr;
        tr.load(&m->desc[b]);
        tc::mbar_arrive(&m->desc_free[b]);
        tc::mbar_wait(&m->v_full, p1);
        tc::mbar_wait(&m->h_ready, p1);  // z2 drained: z is free for the next tile
        tc::tc_fence_after();
        // next tile's MMA1 now if its edge tile is already loaded (never blocks here)
        bool next_known = false, next_more = false;
        if (tc::mbar_test(&m->e_full[nb], ((t + 1) >> 1) & 1)) {
          next_known = true;
          next_more = m->desc[nb].more;
          if (next_more) {
            tc::tc_fence_after();
            mma1();
          }
        }
        // U = H [dS_slot0 | dS_slot1 | ..] in one product (N = NDS * D): row g's
        // block sits at columns 256 + slot(g) * D (slots not holding a row of
        // this tile give unused columns)
        if (t >= 1) tc::mbar_wait(&m->dh_free, (t - 1) & 1);  // U region: dz2 half 1 of t-1 drained
#pragma unroll
        for (int g = 0; g < NMAX; ++g) {
          if (g >= tr.nn) break;
          const uint32_t q = dsq + g;
          tc::mbar_wait(&m->ds_full[q % C::NDS], (q / C::NDS) & 1);
        }
        tc::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < KH / 16; ++kk) {
          uint64_t ad = tc::sdesc(aAH + (kk / 4) * (128 * 128) + (kk % 4) * 32, 16, 1024, tc::kSw128);
          uint64_t bd = tc::sdesc(aDS + kk * 16 * C::ROWB, C::DS_BYTES, 8 * C::ROWB, C::SWZ);
          tc::mma_bf16_ss(tmem + 256, ad, bd, IDESC_U, kk > 0 ? 1u : 0u);
        }
        tc::mma_commit(&m->u_full);
        tc::mma_commit(&m->ah_free);
        // dH^T = dS_i V_seg^T, kappa half h (columns 384 + slot)
        auto dh_half = [&](int h) {  // half 0 -> columns 384.., half 1 -> 256..
#pragma unroll
          for (int g = 0; g < NMAX; ++g) {
            if (g >= tr.nn) break;
            const uint32_t ds = aDS + ((dsq + g) % C::NDS) * C::DS_BYTES;
            const int s0 = tr.s0[g];
            const uint32_t idesc_h = tc::idesc_bf16(128, (tr.deg[g] + 15) & ~15, false, false);
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
              uint64_t ad = tc::sdesc(ds + h * 128 * C::ROWB + kk * 32, 16, 8 * C::ROWB, C::SWZ);
              uint64_t bd = tc::sdesc(aV + (s0 / 8) * 8 * C::ROWB + kk * 32, 16, 8 * C::ROWB, C::SWZ);
              tc::mma_bf16_ss(tmem + (h == 0 ? 384 : 256) + s0, ad, bd, idesc_h, kk > 0 ? 1u : 0u);
            }
          }
        };
        if (t >= 1) tc::mbar_wait(&m->dh0_free, (t - 1) & 1);  // dH region: dz2 half 0 of t-1 drained
        tc::tc_fence_after();
        dh_half(0);
        tc::mma_commit(&m->dh0_full);
        if (!next_known) {  // the next tile's MMA1 before waiting on the dz2 epilogue
          tc::mbar_wait(&m->e_full[nb], ((t + 1) >> 1) & 1);
          next_more = m->desc[nb].more;
          if (next_more) {
            tc::tc_fence_after();
            mma1();
          }
        }
        tc::mbar_wait(&m->u_free, p1);  // U drained: dH half 1 goes to the U columns
        tc::tc_fence_after();
        dh_half(1);
        tc::mma_commit(&m->dh1_full);
        tc::mma_commit(&m->v_empty);
#pragma unroll
        for (int g = 0; g < NMAX; ++g) {
          if (g >= tr.nn) break;
          tc::mma_commit(&m->ds_empty[(dsq + g) % C::NDS]);
        }
        // the next tile's MMA2 while the dz2 epilogue drains both dH halves
        if (next_more) mma2(t + 1);
        dsq += tr.nn;
        more = next_more;
      }
    }
    __syncwarp();
  } else if (warp < 12) {
    // ============================================================= EPI_A
    const int grp = warp & 3, cg = (warp - 4) >> 2, wi = warp - 4;
    const int erow = grp * 32 + lane;
    const uint32_t r = tmem + ((uint32_t)(grp * 32) << 16);
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
      tc::mbar_wait(&m->d1_full, p1);
      tc::tc_fence_after();
      // a1 = relu(z1 + b1) -> AH  (group cg: columns 128*cg .., 64 at a time).
      // The first 64 are computed while the previous tile's U product still
      // reads h from AH.
#pragma unroll 1
      for (int cc = 0; cc < 2; ++cc) {
        const int c0 = cg * 128 + cc * 64;
        uint32_t x[64], pk[32];
        tc::tmem_ld32(r + c0, *reinterpret_cast<uint32_t (*)[32]>(&x[0]));
        tc::tmem_ld32(r + c0 + 32, *reinterpret_cast<uint32_t (*)[32]>(&x[32]));
        tc::tmem_ld_wait();
#pragma unroll
        for (int q4 = 0; q4 < 16; ++q4) {  // biases as float4 broadcasts
          const float4 bb = *reinterpret_cast<const float4 *>(sB1 + c0 + 4 * q4);
          pk[2 * q4] = tc::pack_bf16(fmaxf(__uint_as_float(x[4 * q4]) + bb.x, 0.f),
                                     fmaxf(__uint_as_float(x[4 * q4 + 1]) + bb.y, 0.f));
          pk[2 * q4 + 1] = tc::pack_bf16(fmaxf(__uint_as_float(x[4 * q4 + 2]) + bb.z, 0.f),
                                         fmaxf(__uint_as_float(x[4 * q4 + 3]) + bb.w, 0.f));
        }
        if (cc == 0 && t >= 1) tc::mbar_wait(&m->ah_free, (t - 1) & 1);
        uint8_t *blk = sAH + (c0 / 64) * (128 * 128);
#pragma unroll
        for (int u = 0; u < 8; ++u)
          *reinterpret_cast<uint4 *>(blk + tc::sw128_off(erow, u)) =
              make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
      }
      tc::fence_async_shared();
      tc::tc_fence_before();
      tc::mbar_arrive(&m->a1_ready);
      // a1 rows -> A1 (one 512-byte row per warp instruction), overlapping MMA2;
      // only when A1 is requested (the unfused B4 / B5)
      if (A1g) {
        tc::named_sync(2, 256);
        const int j = lane >> 3, c = lane & 7;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint4 xs[8];
          int32_t ps[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int s = wi + 8 * (8 * h + k);
            ps[k] = tr.edge(s);
            xs[k] = *reinterpret_cast<const uint4 *>(sAH + j * (128 * 128) + tc::sw128_off(s, c));
          }
#pragma unroll
          for (int k = 0; k < 8; ++k)
            if (ps[k] >= 0) reinterpret_cast<uint4 *>(A1g + (int64_t)ps[k] * KH)[lane] = xs[k];
        }
      }
      // h = relu(z2 + b2) -> AH (after MMA2 and the a1 copy-out), + [h > 0] bits
      tc::mbar_wait(&m->d2_full, p1);
      if (t >= 1) tc::mbar_wait(&m->mask_read, (t - 1) & 1);
      tc::named_sync(2, 256);
      tc::tc_fence_after();
#pragma unroll 1
      for (int cc = 0; cc < 4; cc += 2) {
        uint32_t xx[64];
        tc::tmem_ld32(r + cg * 128 + cc * 32, *reinterpret_cast<uint32_t (*)[32]>(&xx[0]));
        tc::tmem_ld32(r + cg * 128 + cc * 32 + 32, *reinterpret_cast<uint32_t (*)[32]>(&xx[32]));
        tc::tmem_ld_wait();
#pragma unroll
        for (int half = 0; half < 2; ++half) {
        const int c0 = cg * 128 + (cc + half) * 32;
        const uint32_t *x = &xx[32 * half];
        uint32_t pk[16], bits = 0;
        float bq[32];
#pragma unroll
        for (int q4 = 0; q4 < 8; ++q4) {  // biases as float4 broadcasts
          const float4 bb = *reinterpret_cast<const float4 *>(sB2 + c0 + 4 * q4);
          bq[4 * q4] = bb.x;
          bq[4 * q4 + 1] = bb.y;
          bq[4 * q4 + 2] = bb.z;
          bq[4 * q4 + 3] = bb.w;
        }
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const float h0 = fmaxf(__uint_as_float(x[2 * q]) + bq[2 * q], 0.f);
          const float h1 = fmaxf(__uint_as_float(x[2 * q + 1]) + bq[2 * q + 1], 0.f);
          pk[q] = tc::pack_bf16(h0, h1);
          // word for kappa = c0 + j over this warp's 32 slots; lane j keeps it
          const uint32_t w0 = __ballot_sync(0xffffffffu, h0 > 0.f);
          const uint32_t w1 = __ballot_sync(0xffffffffu, h1 > 0.f);
          if (lane == 2 * q) bits = w0;
          if (lane == 2 * q + 1) bits = w1;
        }
        uint8_t *blk = sAH + (c0 / 64) * (128 * 128);
        const int ch = (c0 % 64) / 8;
#pragma unroll
        for (int u = 0; u < 4; ++u)
          *reinterpret_cast<uint4 *>(blk + tc::sw128_off(erow, ch + u)) =
              make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
        sMask[grp * KH + c0 + lane] = bits;
        }
      }
      tc::fence_async_shared();
      tc::tc_fence_before();
      tc::mbar_arrive(&m->h_ready);
    }
  } else {
    // ============================================================= EPI_B
    const int grp = warp & 3;
    const uint32_t lane_off = (uint32_t)(grp * 32) << 16;
    float db2_lo = 0.f, db2_hi = 0.f;  // kappa = 32*grp + lane, and + 128
    uint32_t dsq = 0;                  // running row count = dS ring position of this tile's row 0
    for (uint32_t t = 0;; ++t) {
      const int b = t & 1;
      const uint32_t p1 = t & 1;
      const TileDescB *dsc = &m->desc[b];
      tc::mbar_wait(&m->e_full[b], (t >> 1) & 1);
      if (!dsc->more) break;
      // dH / U ready (h_ready: the [h > 0] bits written by EPI_A are visible)
      tc::mbar_wait(&m->h_ready, p1);
      uint32_t mw0[4], mw1[4];  // [h > 0] over the 128 slots for kappa and kappa + 128
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        mw0[u] = sMask[u * KH + grp * 32 + lane];
        mw1[u] = sMask[u * KH + 128 + grp * 32 + lane];
      }
      tc::mbar_arrive(&m->mask_read);
      TileRegs<NMAX> tr;
      tr.load(dsc);
      const int nn = tr.nn;
      tc::mbar_wait(&m->u_full, p1);
      tc::tc_fence_after();
      // U part (thread <-> slot row): u_p = U[slot] + dS_i[k]
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
            tc::tmem_ld32(tmem + lane_off + 256 + ((dsq + g) % C::NDS) * D + c0,
                          *reinterpret_cast<uint32_t (*)[32]>(&xx[c0]));
          tc::tmem_ld_wait();
#pragma unroll
          for (int c0 = 0; c0 < D; c0 += 32) {
            const uint32_t *x = &xx[c0];
            if (mine) {
              uint4 *dst = reinterpret_cast<uint4 *>(Ug + (int64_t)p * D + c0);
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
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&m->desc_free[b]);  // brow[b] read
      // dz2 part (thread <-> kappa), one kappa half per dH product
#pragma unroll 1
      for (int h = 0; h < 2; ++h) {
        tc::mbar_wait(h == 0 ? &m->dh0_full : &m->dh1_full, p1);
        tc::tc_fence_after();
        const int kap = 128 * h + grp * 32 + lane;
        uint32_t mwh[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) mwh[u] = h ? mw1[u] : mw0[u];
        float acc = 0.f;
        // rows not unrolled: one copy of the chunk code keeps this loop's
        // footprint in the instruction cache (the kernel is ~100 KB of SASS)
#pragma unroll 1
        for (int g = 0; g < NMAX; ++g) {
          if (g >= nn) break;
          // register selects, not a dynamically indexed (local-memory) array
          int s0 = tr.s0[0], deg = tr.deg[0];
          int64_t ebg = tr.eb[0];
#pragma unroll
          for (int i = 1; i < NMAX; ++i)
            if (g == i) {
              s0 = tr.s0[i];
              deg = tr.deg[i];
              ebg = tr.eb[i];
            }
          const int ns = (deg + 15) & ~15;
          __nv_bfloat16 *row0 = dZ2g + ebg * KH;
          const uint32_t ta = tmem + lane_off + (h == 0 ? 384 : 256) + s0;
          int c0 = 0;
          for (; c0 + 64 <= ns; c0 += 64) acc += dz2_chunk<64>(ta + c0, slot_bits(mwh, s0 + c0), kap, c0, deg, row0);
          if (c0 + 32 <= ns) {
            acc += dz2_chunk<32>(ta + c0, slot_bits(mwh, s0 + c0), kap, c0, deg, row0);
            c0 += 32;
          }
          if (c0 < ns) acc += dz2_chunk<16>(ta + c0, slot_bits(mwh, s0 + c0), kap, c0, deg, row0);
        }
        if (h == 0) db2_lo += acc; else db2_hi += acc;
        tc::tc_fence_before();
        tc::mbar_arrive(h == 0 ? &m->dh0_free : &m->dh_free);
      }
      dsq += nn;
    }
    db2_part[(int64_t)blockIdx.x * KH + grp * 32 + lane] = db2_lo;
    db2_part[(int64_t)blockIdx.x * KH + 128 + grp * 32 + lane] = db2_hi;
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc<512>(tmem);
}

}  // namespace dsmpnn
