// layer_bf16_bwd.cu - BF16 backward of the edge-conditioned convolution
// (Alg. 1 :417 "Backprop", reading R16 detach), tcgen05 (sm_100a).
//
// With ghat = G * sigma'(pre), S~_aug and the packed Theta~_aug of the forward:
//   B0  ghat (fp32 + bf16 copy), db += colsum(ghat), root term of dv
//   B1  dTheta~_aug = S~_aug^T ghat              (tgemm, M-major A, N-major B)
//       -> dW3, db3, dW_root
//   B2  dS_i = (ghat_i Theta~^T) / deg_i          (tgemm, bf16 epilogue, row scale)
//   B3  edge kernel per 128-slot tile: recompute a1, h (W1 resident, W2
//       streamed by TMA), then per row  dH^T = dS_i V^T  and  U = H dS_i
//       (tcgen05), dz2 = dH * [h > 0] -> global, u_p = U + dS_i[k] -> global,
//       a1 -> global, per-CTA db2 partial sums.
//   B4  dW2 += dz2^T a1                           (tgemm, split-K over edges)
//   B5  dz1 = (dz2 W2) * [a1 > 0]                  (tgemm, bf16 + mask epilogue,
//                                                   column sums -> db1)
//   B6  dW1 += dz1^T e ; de = dz1 W1              (tgemm)
//   B7  dv[j] += sum_{p: col(p)=j} u_p            (deterministic CSC scatter)
#include <cuda.h>

#include "layer_bf16.cuh"
#include "layer_bf16_common.cuh"
#include "simt.cuh"
#include "tc.cuh"
#include "tgemm.cuh"

namespace dsmpnn {

// ------------------------------------------------------------- B0 kernels
__global__ void ghat_bf16_kernel(const float *__restrict__ G, const float *__restrict__ pre,
                                 const int64_t *__restrict__ row_ptr, int64_t rb, int64_t re, int D, int act,
                                 float *__restrict__ gh, __nv_bfloat16 *__restrict__ gh16, float *__restrict__ inv_deg) {
  int64_t total = (re - rb) * D;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t idx = rb * D + t;
    float g = G[idx];
    if (act == DSMPNN_ACT_RELU && !(pre[idx] > 0.f)) g = 0.f;
    gh[idx] = g;
    gh16[idx] = __float2bfloat16_rn(g);
    if (t % D == 0) {
      int64_t i = rb + t / D;
      int64_t deg = row_ptr[i + 1] - row_ptr[i];
      inv_deg[i] = deg > 0 ? 1.0f / (float)deg : 0.f;
    }
  }
}

// dW3[c*D+o, kap] += dT[kap*D+c, o]; db3[c*D+o] += dT[k*D+c, o]; dW_root[o, c] += dT[(k+1)*D+c, o]
__global__ void unpack_dtheta_aug_kernel(const float *__restrict__ dT, int k, int D, float *__restrict__ dW3,
                                         float *__restrict__ db3, float *__restrict__ dWr) {
  int64_t total = (int64_t)(k + 2) * D * D;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t row = t / D;  // K index of the forward S~_aug layout
    int o = (int)(t - row * D);
    int kap, c;
    if (row < (int64_t)k * D) {  // [c][kappa] block
      c = (int)(row / k);
      kap = (int)(row - (int64_t)c * k);
    } else {
      kap = (int)(row / D);
      c = (int)(row - (int64_t)kap * D);
    }
    float x = dT[t];
    if (kap < k) { if (dW3) dW3[((int64_t)c * D + o) * k + kap] += x; }
    else if (kap == k) { if (db3) db3[(int64_t)c * D + o] += x; }
    else if (dWr) dWr[(int64_t)o * D + c] += x;
  }
}

// dW1[r, c] += full[r, c] for c < d_e (full is [k x 16]); same for de rows
__global__ void add_cols_kernel(const float *__restrict__ full, int64_t rows, int ld_full, int ncols,
                                float *__restrict__ dst, int accumulate) {
  int64_t total = rows * ncols;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = t / ncols;
    int c = (int)(t - r * ncols);
    float x = full[r * ld_full + c];
    dst[t] = accumulate ? dst[t] + x : x;
  }
}

// ---------------------------------------------------------- B3 edge kernel
template <int D>
struct EB {
  static constexpr int W2BLK = KH * 64 * 2;       // one 64-wide K block of W2: 32 KB
  static constexpr int AH_BYTES = 128 * KH * 2;   // 64 KB
  static constexpr int V_BYTES = 128 * D * 2;
  static constexpr int DS_BYTES = KH * D * 2;     // 32 KB / 16 KB
  static constexpr int W1_BYTES = KH * 32;
  static constexpr int E_BYTES = 128 * 32;
  static constexpr int OFF_W2 = 0;                // 2-slot ring
  static constexpr int OFF_AH = OFF_W2 + 2 * W2BLK;
  static constexpr int OFF_DS = OFF_AH + AH_BYTES;
  static constexpr int OFF_V = OFF_DS + DS_BYTES;
  static constexpr int OFF_W1 = OFF_V + V_BYTES;
  static constexpr int OFF_E = OFF_W1 + W1_BYTES;
  static constexpr int OFF_MISC = OFF_E + E_BYTES;
  static constexpr int SMEM = OFF_MISC + 2048 + 1024;
  static constexpr uint32_t ROWB = D * 2;          // bytes per dS / V smem row
  static constexpr uint32_t SWZ = D == 64 ? tc::kSw128 : tc::kSw64;
};

struct BwdMisc {
  uint64_t w2_full[2], w2_empty[2], ds_full;
  uint32_t w2_issued, w2_used;  // W2 block loads issued / consumed (thread 0 only)
};

template <int D>
__global__ void __launch_bounds__(256, 1)
    edge_bwd_kernel(const __grid_constant__ CUtensorMap tW2, const __grid_constant__ CUtensorMap tDS,
                    const __nv_bfloat16 *__restrict__ e16, const __nv_bfloat16 *__restrict__ v,
                    const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col, int64_t rb, int64_t re,
                    int64_t eb, int64_t ee, Packed pw, const float *__restrict__ b1, const float *__restrict__ b2,
                    const __nv_bfloat16 *__restrict__ dS, __nv_bfloat16 *__restrict__ A1g,
                    __nv_bfloat16 *__restrict__ dZ2g, float *__restrict__ Ug, float *__restrict__ db2_part) {
  using C = EB<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *sm = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);  // keeps the shared address space (LDS/STS)
  uint8_t *sW2 = sm + C::OFF_W2, *sAH = sm + C::OFF_AH, *sDS = sm + C::OFF_DS, *sV = sm + C::OFF_V,
          *sW1 = sm + C::OFF_W1, *sE = sm + C::OFF_E;
  EdgeMisc *m = reinterpret_cast<EdgeMisc *>(sm + C::OFF_MISC);
  BwdMisc *bm = reinterpret_cast<BwdMisc *>(sm + C::OFF_MISC + 1536);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

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
    m->cur_off = 0;
    m->node_ctr = 0;
    tc::mbar_init(&m->bar, 1);
    for (int s = 0; s < 2; ++s) {
      tc::mbar_init(&bm->w2_full[s], 1);
      tc::mbar_init(&bm->w2_empty[s], 1);
    }
    tc::mbar_init(&bm->ds_full, 1);
    bm->w2_issued = 0;
    bm->w2_used = 0;
    tc::fence_mbar_init();
    tc::tma_prefetch(&tW2);
    tc::tma_prefetch(&tDS);
  }
  if (warp == 0) tc::tmem_alloc<512>(&m->tmem);
  {
    const uint4 *g1 = reinterpret_cast<const uint4 *>(pw.W1);
    for (int q = tid; q < KH * 2; q += 256) {
      int r = q / 2, u = q % 2;
      *reinterpret_cast<uint4 *>(sW1 + il_off(r, u)) = g1[q];
    }
  }
  tc::fence_async_shared();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = m->tmem;
  uint32_t phase = 0, ds_phase = 0;

  const uint32_t aW2 = tc::smem_u32(sW2), aAH = tc::smem_u32(sAH), aDS = tc::smem_u32(sDS), aV = tc::smem_u32(sV),
                 aW1 = tc::smem_u32(sW1), aE = tc::smem_u32(sE);
  constexpr uint32_t IDESC_MLP = tc::idesc_bf16(128, KH, false, false);
  constexpr uint32_t IDESC_U = tc::idesc_bf16(128, D, false, true);
  const bool epi = warp >= 4;
  const int erow = tid - 128;
  const uint32_t lane_base = epi ? ((uint32_t)(32 * (warp - 4)) << 16) : 0u;
  float db2_acc0 = 0.f, db2_acc1 = 0.f;  // kappa = erow, 128 + erow

  auto wait_mma = [&]() {
    tc::mbar_wait(&m->bar, phase & 1);
    phase++;
    tc::tc_fence_after();
  };
  // thread 0: issue the TMA of the next W2 K-block into the ring
  auto w2_issue = [&]() {
    uint32_t q = bm->w2_issued;
    uint32_t s = q & 1, r = q >> 1;
    if (r > 0) tc::mbar_wait(&bm->w2_empty[s], (r - 1) & 1);
    tc::mbar_expect_tx(&bm->w2_full[s], C::W2BLK);
    tc::tma_load_2d(sW2 + s * C::W2BLK, &tW2, &bm->w2_full[s], (int32_t)((q & 3) * 64), 0);
    bm->w2_issued = q + 1;
  };

  for (;;) {
    if (tid == 0) {
      build_tile(m, row_ptr);
      if (m->more) {  // prefetch W2 blocks 0 and 1 of this tile
        w2_issue();
        w2_issue();
      }
    }
    __syncthreads();
    if (!m->more) break;

    {  // gather E and V rows of the slots
      int s = tid >> 1, u = tid & 1;
      int p = m->slot_edge[s];
      uint4 val = make_uint4(0, 0, 0, 0);
      if (p >= 0) val = reinterpret_cast<const uint4 *>(e16 + (int64_t)p * 16)[u];
      *reinterpret_cast<uint4 *>(sE + il_off(s, u)) = val;
      constexpr int CH = D / 8;
      for (int q = tid; q < 128 * CH; q += 256) {
        int sl = q / CH, c = q % CH;
        int pe = m->slot_edge[sl];
        uint4 x = make_uint4(0, 0, 0, 0);
        if (pe >= 0) x = reinterpret_cast<const uint4 *>(v + (int64_t)col[pe] * D)[c];
        *reinterpret_cast<uint4 *>(sV + v_off<D>(sl, c)) = x;
      }
    }
    tc::fence_async_shared();
    tc::tc_fence_before();
    __syncthreads();

    // ---- MMA1 + epilogue 1: a1 -> AH and -> A1 (global, for the dW2 / dz1 GEMMs)
    if (tid == 0) {
      tc::tc_fence_after();
      tc::mma_bf16_ss(tmem, tc::sdesc(aE, 128, 256, tc::kSwNone), tc::sdesc(aW1, 128, 256, tc::kSwNone), IDESC_MLP,
                      0u);
      tc::mma_commit(&m->bar);
    }
    wait_mma();
    if (epi) {
      const int p = m->slot_edge[erow];
#pragma unroll 1
      for (int c0 = 0; c0 < KH; c0 += 16) {
        uint32_t r[16];
        tc::tmem_ld16(tmem + lane_base + c0, r);
        tc::tmem_ld_wait();
        uint32_t pk[8];
#pragma unroll
        for (int j = 0; j < 8; ++j)
          pk[j] = tc::pack_bf16(fmaxf(__uint_as_float(r[2 * j]) + __ldg(b1 + c0 + 2 * j), 0.f),
                                fmaxf(__uint_as_float(r[2 * j + 1]) + __ldg(b1 + c0 + 2 * j + 1), 0.f));
        uint8_t *blk = sAH + (c0 / 64) * (128 * 128);
        int ch = (c0 % 64) / 8;
        uint4 x0 = make_uint4(pk[0], pk[1], pk[2], pk[3]), x1 = make_uint4(pk[4], pk[5], pk[6], pk[7]);
        *reinterpret_cast<uint4 *>(blk + tc::sw128_off(erow, ch)) = x0;
        *reinterpret_cast<uint4 *>(blk + tc::sw128_off(erow, ch + 1)) = x1;
        if (p >= 0) {
          uint4 *g = reinterpret_cast<uint4 *>(A1g + (int64_t)p * KH + c0);
          g[0] = x0;
          g[1] = x1;
        }
      }
    }
    tc::fence_async_shared();
    tc::tc_fence_before();
    __syncthreads();

    // ---- MMA2 with W2 streamed through the 2-slot ring
    if (tid == 0) {
      tc::tc_fence_after();
      for (int j = 0; j < 4; ++j) {
        uint32_t q = bm->w2_used;
        uint32_t s = q & 1;
        tc::mbar_wait(&bm->w2_full[s], (q >> 1) & 1);
        tc::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          uint64_t ad = tc::sdesc(aAH + j * (128 * 128) + kk * 32, 16, 1024, tc::kSw128);
          uint64_t bd = tc::sdesc(aW2 + s * C::W2BLK + kk * 32, 16, 1024, tc::kSw128);
          tc::mma_bf16_ss(tmem, ad, bd, IDESC_MLP, (j > 0 || kk > 0) ? 1u : 0u);
        }
        tc::mma_commit(&bm->w2_empty[s]);
        bm->w2_used = q + 1;
        // blocks 2, 3 reuse the slots of 0, 1; issued one block late so the
        // tensor pipe still holds queued MMAs while we wait for the slot
        if (j == 1 || j == 2) w2_issue();
      }
      tc::mma_commit(&m->bar);
    }
    wait_mma();
    if (epi) {  // h = relu(z2 + b2) -> AH
#pragma unroll 1
      for (int c0 = 0; c0 < KH; c0 += 16) {
        uint32_t r[16];
        tc::tmem_ld16(tmem + lane_base + c0, r);
        tc::tmem_ld_wait();
        uint32_t pk[8];
#pragma unroll
        for (int j = 0; j < 8; ++j)
          pk[j] = tc::pack_bf16(fmaxf(__uint_as_float(r[2 * j]) + __ldg(b2 + c0 + 2 * j), 0.f),
                                fmaxf(__uint_as_float(r[2 * j + 1]) + __ldg(b2 + c0 + 2 * j + 1), 0.f));
        uint8_t *blk = sAH + (c0 / 64) * (128 * 128);
        int ch = (c0 % 64) / 8;
        *reinterpret_cast<uint4 *>(blk + tc::sw128_off(erow, ch)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        *reinterpret_cast<uint4 *>(blk + tc::sw128_off(erow, ch + 1)) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
      }
    }
    tc::fence_async_shared();
    tc::tc_fence_before();
    __syncthreads();

    // ---- per row segment: dH^T = dS_i V_seg^T and U = H dS_i
    const int nseg = m->nseg;
    for (int g = 0; g < nseg; ++g) {
      const Seg sg = m->seg[g];
      if (tid == 0) {
        tc::mbar_expect_tx(&bm->ds_full, C::DS_BYTES);
        tc::tma_load_2d(sDS, &tDS, &bm->ds_full, 0, (int32_t)(sg.node * (KH + 1)));
        tc::mbar_wait(&bm->ds_full, ds_phase & 1);
        tc::tc_fence_after();
        const uint32_t idesc_h = tc::idesc_bf16(128, sg.nslots, false, false);
        for (int h = 0; h < 2; ++h) {
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            uint64_t ad = tc::sdesc(aDS + h * 128 * C::ROWB + kk * 32, 16, 8 * C::ROWB, C::SWZ);
            uint64_t bd = tc::sdesc(aV + (sg.slot0 / 8) * 8 * C::ROWB + kk * 32, 16, 8 * C::ROWB, C::SWZ);
            tc::mma_bf16_ss(tmem + h * 128, ad, bd, idesc_h, kk > 0 ? 1u : 0u);
          }
        }
#pragma unroll
        for (int kk = 0; kk < KH / 16; ++kk) {
          uint64_t ad = tc::sdesc(aAH + (kk / 4) * (128 * 128) + (kk % 4) * 32, 16, 1024, tc::kSw128);
          uint64_t bd = tc::sdesc(aDS + kk * 16 * C::ROWB, 64 * C::ROWB, 8 * C::ROWB, C::SWZ);
          tc::mma_bf16_ss(tmem + KH, ad, bd, IDESC_U, kk > 0 ? 1u : 0u);
        }
        tc::mma_commit(&m->bar);
      }
      ds_phase++;
      wait_mma();
      if (epi) {
        // dz2[slot][kap] = dH^T[kap][slot] * [h[slot][kap] > 0]  (thread <-> kap)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int kap = 128 * h + erow;
          const uint8_t *hblk = sAH + (kap / 64) * (128 * 128);
          const int hch = (kap % 64) / 8, hel = kap % 8;
          float acc = 0.f;
#pragma unroll 1
          for (int c0 = 0; c0 < sg.nslots; c0 += 16) {
            uint32_t r[16];
            tc::tmem_ld16(tmem + lane_base + h * 128 + c0, r);
            tc::tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const int s = sg.slot0 + c0 + j;
              const int p = m->slot_edge[s];
              const __nv_bfloat16 hv =
                  *reinterpret_cast<const __nv_bfloat16 *>(hblk + tc::sw128_off(s, hch) + hel * 2);
              float dz = __bfloat162float(hv) > 0.f ? __uint_as_float(r[j]) : 0.f;
              __nv_bfloat16 dzb = __float2bfloat16_rn(dz);
              if (p >= 0) {
                dZ2g[(int64_t)p * KH + kap] = dzb;
                acc += __bfloat162float(dzb);
              }
            }
          }
          if (h == 0) db2_acc0 += acc; else db2_acc1 += acc;
        }
        // u_p[c] = U[slot][c] + dS_i[k][c]  (thread <-> slot)
        const int s = erow;
        const int p = m->slot_edge[s];
        const bool mine = s >= sg.slot0 && s < sg.slot0 + sg.nslots && p >= 0;
        const __nv_bfloat16 *brow = dS + (sg.node * (KH + 1) + KH) * D;
#pragma unroll
        for (int c0 = 0; c0 < D; c0 += 16) {
          uint32_t r[16];
          tc::tmem_ld16(tmem + lane_base + KH + c0, r);  // warp-collective: executed by all lanes
          tc::tmem_ld_wait();
          if (mine) {
            float4 *dst = reinterpret_cast<float4 *>(Ug + (int64_t)p * D + c0);
#pragma unroll
            for (int j = 0; j < 4; ++j)
              dst[j] = make_float4(__uint_as_float(r[4 * j]) + __bfloat162float(brow[c0 + 4 * j]),
                                   __uint_as_float(r[4 * j + 1]) + __bfloat162float(brow[c0 + 4 * j + 1]),
                                   __uint_as_float(r[4 * j + 2]) + __bfloat162float(brow[c0 + 4 * j + 2]),
                                   __uint_as_float(r[4 * j + 3]) + __bfloat162float(brow[c0 + 4 * j + 3]));
          }
        }
      }
      tc::tc_fence_before();
      __syncthreads();
    }
  }
  if (epi) {
    db2_part[(int64_t)blockIdx.x * KH + erow] = db2_acc0;
    db2_part[(int64_t)blockIdx.x * KH + 128 + erow] = db2_acc1;
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}

// ------------------------------------------------------------ workspace
struct BBwd {
  float *gh;               // [n_dst x D]
  __nv_bfloat16 *gh16;     // [n_dst x D]
  float *inv_deg;          // [n_dst]
  float *dT;               // [kp x D]
  __nv_bfloat16 *dS;       // [n_dst x (k+1) x D]
  __nv_bfloat16 *A1;       // [E x k]
  __nv_bfloat16 *dZ2;      // [E x k]
  __nv_bfloat16 *dZ1;      // [E x k]
  float *U;                // [E x D]
  float *part;             // split-K partials (max over users)
  float *db2_part;         // [kNumSMs x k]
  float *db1_part;         // [ceil(E/128)*4 x k]
  float *dW1f;             // [k x 16]
  float *de16;             // [E x 16]
};
constexpr int kSplitsW = 64;
static BBwd carve_bf16_bwd(Carver &c, const dsmpnn_layer_desc &d, int64_t n_dst, int64_t E) {
  BBwd b;
  const int D = d.d_in;
  int64_t kp = (int64_t)(d.k + 2) * D;
  kp = (kp + 63) / 64 * 64;
  b.gh = c.take<float>(n_dst * D);
  b.gh16 = c.take<__nv_bfloat16>(n_dst * D);
  b.inv_deg = c.take<float>(n_dst);
  b.dT = c.take<float>(kp * D);
  b.dS = c.take<__nv_bfloat16>(n_dst * (int64_t)(d.k + 1) * D);
  b.A1 = c.take<__nv_bfloat16>(E * d.k);
  b.dZ2 = c.take<__nv_bfloat16>(E * d.k);
  b.dZ1 = c.take<__nv_bfloat16>(E * d.k);
  b.U = c.take<float>(E * D);
  b.part = c.take<float>((int64_t)kSplitsW * d.k * d.k);
  b.db2_part = c.take<float>((int64_t)kNumSMs * d.k);
  b.db1_part = c.take<float>((int64_t)kColsumRows * d.k);
  b.dW1f = c.take<float>((int64_t)d.k * 16);
  b.de16 = c.take<float>(E * 16);
  return b;
}

size_t bf16_bwd_ws_bytes(const dsmpnn_layer_desc &d, int64_t n_dst, int64_t n_loc, int64_t E) {
  Carver c(nullptr, 0);
  carve_bf16_bwd(c, d, n_dst, E);
  return c.used();
}

static int grid_of(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), 148 * 8)); }

// forward workspace layout (must match layer_bf16.cu)
struct BFwdView {
  const __nv_bfloat16 *S;
  const float *pre;
};
static BFwdView view_fwd(const dsmpnn_layer_desc &d, const void *ws, int64_t n_dst) {
  Carver c(const_cast<void *>(ws), SIZE_MAX);
  BFwdView f;
  f.S = c.take<__nv_bfloat16>(n_dst * kpad_of(d));
  f.pre = c.take<float>(n_dst * d.d_out);
  return f;
}

__global__ void scatter_csc_f32_kernel(const float *__restrict__ U, const int32_t *__restrict__ perm,
                                       const int64_t *__restrict__ cptr, int64_t n_loc, int di, int64_t eb,
                                       int64_t ee, float *__restrict__ dv) {
  int64_t total = n_loc * di;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t j = t / di;
    int c = (int)(t - j * di);
    float s = 0.f;
    bool any = false;
    for (int64_t q = cptr[j]; q < cptr[j + 1]; ++q) {
      int64_t p = perm[q];
      if (p >= eb && p < ee) { s += U[p * di + c]; any = true; }
    }
    if (any) dv[t] += s;
  }
}

__global__ void add_rows_f32_kernel(const float *__restrict__ src, int64_t rb, int64_t re, int w,
                                    float *__restrict__ dst) {
  int64_t total = (re - rb) * w;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x)
    dst[rb * w + t] += src[rb * w + t];
}

template <int D>
static dsmpnn_status launch_edge_bwd(const dsmpnn_layer_desc &d, const Packed &pw, const __nv_bfloat16 *e,
                                     const __nv_bfloat16 *v, const int64_t *row_ptr, const int32_t *col, int64_t n_dst,
                                     int64_t rb, int64_t re, int64_t eb, int64_t ee, const float *b1, const float *b2,
                                     const BBwd &b, int *grid_out, cudaStream_t s) {
  using C = EB<D>;
  CUtensorMap tW2, tDS;
  DS_TRY(make_tmap_bf16(&tW2, pw.W2, KH, KH, KH, 64, KH));
  DS_TRY(make_tmap_bf16(&tDS, b.dS, D, n_dst * (int64_t)(KH + 1), D, D, KH));
  auto kern = edge_bwd_kernel<D>;
  DS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
  int64_t tiles = (ee - eb + 127) / 128 + 1;
  int grid = (int)std::max<int64_t>(1, std::min<int64_t>(kNumSMs, tiles));
  *grid_out = grid;
  ProbeScope probe(DSMPNN_PROBE_BF16_EDGE_BWD, s);
  kern<<<grid, 256, C::SMEM, s>>>(tW2, tDS, e, v, row_ptr, col, rb, re, eb, ee, pw, b1, b2, b.dS, b.A1, b.dZ2, b.U,
                                  b.db2_part);
  DS_LAUNCH_CHECK();
  return DSMPNN_OK;
}

dsmpnn_status bf16_bwd(const dsmpnn_layer_desc &d, const dsmpnn_weights &w, const __nv_bfloat16 *v,
                       const __nv_bfloat16 *e, const int64_t *row_ptr, const int32_t *col, const int32_t *perm,
                       const int64_t *cptr, int64_t n_dst, int64_t n_loc, int64_t E, int64_t rb, int64_t re,
                       int64_t eb, int64_t ee, const float *G, float *dv, float *de, const dsmpnn_grads &gr,
                       const void *ws, void *bws, size_t bws_bytes, cudaStream_t s) {
  Carver c(bws, bws_bytes);
  BBwd b = carve_bf16_bwd(c, d, n_dst, E);
  DS_CHECK_ARG(c.ok(), DSMPNN_ERR_CAPACITY, "layer_bwd: bwd workspace too small");
  BFwdView f = view_fwd(d, ws, n_dst);
  Packed pw = carve_packed(d, const_cast<void *>(w.packed));
  const int D = d.d_in, k = d.k;
  const int64_t kp = kpad_of(d);
  const int64_t nR = re - rb, nE = ee - eb;
  if (nR <= 0) return DSMPNN_OK;

  // B0
  ghat_bf16_kernel<<<grid_of(nR * D), 256, 0, s>>>(G, f.pre, row_ptr, rb, re, D, d.act, b.gh, b.gh16, b.inv_deg);
  DS_LAUNCH_CHECK();
  DS_TRY(colsum(b.gh + rb * D, nR, D, D, gr.b, 1, s));
  if (d.root == DSMPNN_ROOT_DENSE && dv) {
    SgemmArgs g{nR, D, D, b.gh + rb * D, D, 1, w.W_root, D, 1, dv + rb * D, D, nullptr, 0, 1, 1.f};
    DS_TRY(sgemm(g, 1, nullptr, s));
  } else if (d.root == DSMPNN_ROOT_IDENTITY && dv) {
    add_rows_f32_kernel<<<grid_of(nR * D), 256, 0, s>>>(b.gh, rb, re, D, dv);
    DS_LAUNCH_CHECK();
  }
  // B1: dTheta~_aug [kp x D] = S~_aug^T ghat  (K = rows)
  if (gr.W3 || gr.b3 || gr.W_root) {
    TgemmArgs a{kp, D, nR, f.S + rb * kp, kp, true, b.gh16 + rb * D, D, true, b.dT, D, 1, 0, 0};
    DS_TRY(tgemm(a, s));
    unpack_dtheta_aug_kernel<<<grid_of((int64_t)(k + 2) * D * D), 256, 0, s>>>(
        b.dT, k, D, gr.W3, gr.b3, d.root == DSMPNN_ROOT_DENSE ? gr.W_root : nullptr);
    DS_LAUNCH_CHECK();
  }
  if (nE <= 0) return DSMPNN_OK;
  // B2: dS_i = (ghat_i Theta~^T) / deg_i   -> bf16 [n_dst x (k+1)*D]
  {
    TgemmArgs a{nR, (int64_t)(k + 1) * D, D, b.gh16 + rb * D, D, false, pw.Th, D, false, nullptr, 0, 1, 0, 0};
    a.out16 = b.dS + rb * (int64_t)(k + 1) * D;
    a.ld16 = (int64_t)(k + 1) * D;
    a.row_scale = b.inv_deg + rb;
    DS_TRY(tgemm(a, s));
  }
  // B3: edge kernel
  int grid = 1;
  if (D == 64) DS_TRY(launch_edge_bwd<64>(d, pw, e, v, row_ptr, col, n_dst, rb, re, eb, ee, w.b1, w.b2, b, &grid, s));
  else DS_TRY(launch_edge_bwd<32>(d, pw, e, v, row_ptr, col, n_dst, rb, re, eb, ee, w.b1, w.b2, b, &grid, s));
  DS_TRY(colsum(b.db2_part, grid, k, k, gr.b2, 1, s));
  // B4: dW2 += dz2^T a1   (M = k, N = k, K = edges)
  if (gr.W2) {
    int splits = (int)std::max<int64_t>(1, std::min<int64_t>(kSplitsW, nE / 512));
    TgemmArgs a{k, k, nE, b.dZ2 + eb * k, k, true, b.A1 + eb * k, k, true, b.part, k, splits, (int64_t)k * k, 0};
    DS_TRY(tgemm(a, s));
    int64_t nkb = (nE + 63) / 64;
    int kbps = (int)std::max<int64_t>(1, ceil_div(nkb, splits));
    int real = (int)std::max<int64_t>(1, ceil_div(nkb, kbps));
    DS_TRY(splitk_sum(b.part, real, (int64_t)k * k, k, k, k, gr.W2, k, 1, s));
  }
  // B5: dz1 = (dz2 W2) * [a1 > 0]  (bf16), column sums -> db1
  {
    TgemmArgs a{nE, k, k, b.dZ2 + eb * k, k, false, pw.W2, k, true, nullptr, 0, 1, 0, 0};
    a.out16 = b.dZ1 + eb * k;
    a.ld16 = k;
    a.mask16 = b.A1 + eb * k;
    a.ldmask = k;
    a.colsum_part = b.db1_part;
    DS_CUDA(cudaMemsetAsync(b.db1_part, 0, (size_t)kColsumRows * k * sizeof(float), s));
    DS_TRY(tgemm(a, s));
    DS_TRY(colsum(b.db1_part, kColsumRows, k, k, gr.b1, 1, s));
  }
  // B6: dW1 += dz1^T e ;  de = dz1 W1
  if (gr.W1) {
    int splits = (int)std::max<int64_t>(1, std::min<int64_t>(kSplitsW, nE / 512));
    TgemmArgs a{k, 16, nE, b.dZ1 + eb * k, k, true, e + eb * 16, 16, true, b.part, 16, splits, (int64_t)k * 16, 0};
    DS_TRY(tgemm(a, s));
    int64_t nkb = (nE + 63) / 64;
    int kbps = (int)std::max<int64_t>(1, ceil_div(nkb, splits));
    int real = (int)std::max<int64_t>(1, ceil_div(nkb, kbps));
    DS_TRY(splitk_sum(b.part, real, (int64_t)k * 16, k, 16, 16, b.dW1f, 16, 0, s));
    add_cols_kernel<<<grid_of((int64_t)k * d.d_e), 256, 0, s>>>(b.dW1f, k, 16, d.d_e, gr.W1, 1);
    DS_LAUNCH_CHECK();
  }
  if (de) {
    TgemmArgs a{nE, 16, k, b.dZ1 + eb * k, k, false, pw.W1, 16, true, b.de16, 16, 1, 0, 0};
    DS_TRY(tgemm(a, s));
    add_cols_kernel<<<grid_of(nE * d.d_e), 256, 0, s>>>(b.de16, nE, 16, d.d_e, de + eb * d.d_e, 0);
    DS_LAUNCH_CHECK();
  }
  // B7: dv[j] += sum of u_p over edges with source j (CSC order)
  if (dv) {
    scatter_csc_f32_kernel<<<grid_of(n_loc * D), 256, 0, s>>>(b.U, perm, cptr, n_loc, D, eb, ee, dv);
    DS_LAUNCH_CHECK();
  }
  return DSMPNN_OK;
}

}  // namespace dsmpnn
