// tgemm.cu - bf16 GEMM on the 5th-generation tensor cores (sm_100a).
//
// One CTA per 128 x BN output tile (and per split-K slice).  Warp 0 (one
// elected lane) streams 128x64 A and BNx64 B tiles with TMA into a 4-stage
// shared-memory ring (128-byte swizzle); warp 1 (one elected lane) issues
// tcgen05.mma (M=128, N=BN, K=16) accumulating in TMEM and releases ring
// slots with tcgen05.commit; then all 4 warps drain TMEM (tcgen05.ld
// 32x32b, one thread per output row) to fp32 global memory.  TMA zero-fills
// out-of-range boxes, so ragged M/N/K tails need no special path.
#include <cuda.h>
#include <string.h>

#include "tc.cuh"
#include "tgemm.cuh"

namespace dsmpnn {

namespace {

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void *p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

}  // namespace

// 2-D bf16 tensor map: inner dimension `inner` (contiguous), `outer` rows of
// `ld` elements; box {box_inner, box_outer}; swizzle from the box row bytes.
dsmpnn_status make_tmap_bf16(CUtensorMap *m, const void *base, int64_t inner, int64_t outer, int64_t ld,
                             int box_inner, int box_outer) {
  EncodeTiledFn fn = encode_fn();
  DS_CHECK_ARG(fn != nullptr, DSMPNN_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  DS_CHECK_ARG(((uintptr_t)base & 15) == 0 && ((ld * 2) & 15) == 0, DSMPNN_ERR_SHAPE,
               "TMA operand needs 16-byte aligned base and row stride (ld=%lld)", (long long)ld);
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer};
  cuuint32_t es[2] = {1, 1};
  int row_bytes = box_inner * 2;
  CUtensorMapSwizzle sw = row_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                          : row_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                          : row_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                            : CU_TENSOR_MAP_SWIZZLE_NONE;
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  DS_CHECK_ARG(r == CUDA_SUCCESS, DSMPNN_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return DSMPNN_OK;
}

template <int BN, bool A_MN, bool B_MN, bool E16 = false, bool BRES = false>
struct TG {
  static constexpr int BM = 128, BK = 64;
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  // BRES: the whole B (N <= BN, K <= NKB_RES * BK) stays in SMEM for every
  // tile; only A streams through the stages
  static constexpr int NKB_RES = 4;
  // epilogue warps: 4 (one per TMEM lane quarter); the streaming bf16
  // epilogue (E16 without a resident B) uses 8 -- two per lane quarter taking
  // alternate 64-column chunks -- as one warp per scheduler cannot hide the
  // latency of its TMEM-load / convert / store chain (the B2 GEMM of the
  // backward is bound by that chain, not by HBM or the tensor pipe)
  static constexpr int EPI = (E16 && !BRES) ? 8 : 4;
  static constexpr int THREADS = 64 + 32 * EPI;
  static constexpr int STAGES = BRES ? 2 : (BN >= 256 ? (E16 ? 2 : 4) : (BN >= 128 ? (E16 ? 3 : 5) : (E16 ? 4 : 6)));
  static constexpr int B_STAGE_BYTES = BRES ? 0 : B_BYTES;
  static constexpr int B_RES_BYTES = BRES ? NKB_RES * B_BYTES : 0;
  // bf16 epilogue staging per epilogue warp: 2 output buffers + 2 mask buffers (32 rows x 128 B each)
  static constexpr int STG_BYTES = E16 ? EPI * 4 * 4096 : 0;
  static constexpr int B_INNER = B_MN ? (BN < 64 ? BN : 64) : 64;  // box inner elements for B
  static constexpr int B_ROW = B_INNER * 2;                          // bytes per smem row of B (MN-major)
  static constexpr uint32_t ACC_COLS = BN <= 32 ? 32 : (BN <= 64 ? 64 : (BN <= 128 ? 128 : 256));
  static constexpr uint32_t TMEM_COLS = 2 * ACC_COLS;                 // double-buffered accumulator
  static constexpr int SMEM = 1024 + STAGES * (A_BYTES + B_STAGE_BYTES) + B_RES_BYTES + STG_BYTES + 512;
};

// Persistent: CTA c handles tiles c, c + G, ...  (tile = (m-block, n-block,
// k-slice), m fastest).  Warp 0 = TMA producer, warp 1 = MMA issuer, warps
// 2..5 = epilogue; the accumulator is double-buffered in TMEM so the epilogue
// of tile i overlaps the mainloop of tile i+1.
template <int BN, bool A_MN, bool B_MN, bool E16, bool BRES>
__global__ void __launch_bounds__(TG<BN, A_MN, B_MN, E16, BRES>::THREADS, 1)
    tgemm_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                 const __grid_constant__ CUtensorMap tout, const __grid_constant__ CUtensorMap tmask, int64_t M,
                 int64_t N, int64_t K, int kb_per_split, const TgemmArgs ep, int splits) {
  using T = TG<BN, A_MN, B_MN, E16, BRES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);  // keeps the shared address space
  uint8_t *sA = smem;
  uint8_t *sB = smem + T::STAGES * T::A_BYTES;
  uint8_t *sStg = sB + T::STAGES * T::B_STAGE_BYTES + T::B_RES_BYTES;  // E16 staging (1024-aligned)
  uint64_t *full = reinterpret_cast<uint64_t *>(sStg + T::STG_BYTES);
  uint64_t *empty = full + T::STAGES;
  uint64_t *tfull = empty + T::STAGES;   // [2]
  uint64_t *tempty = tfull + 2;          // [2]
  uint64_t *mbar = tempty + 2;           // [EPI][2] mask loads, two buffers per epilogue warp
  uint64_t *bres = mbar + 2 * T::EPI;    // resident B loaded (BRES)
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bres + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nm = (M + T::BM - 1) / T::BM, nn = (N + BN - 1) / BN;
  const int64_t ntiles = nm * nn * splits;
  const int64_t nkb_total = (K + T::BK - 1) / T::BK;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < T::STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(&tfull[a], 1);
      tc::mbar_init(&tempty[a], T::EPI);
    }
    for (int a = 0; a < 2 * T::EPI; ++a) tc::mbar_init(&mbar[a], 1);
    tc::mbar_init(bres, 1);
    tc::fence_mbar_init();
    tc::tma_prefetch(&ta);
    tc::tma_prefetch(&tb);
  }
  if (warp == 1) tc::tmem_alloc<T::TMEM_COLS>(tmem_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // operands and outputs of other kernels from here on
  pdl_trigger();

  auto tile_coords = [&](int64_t t, int64_t &m0, int64_t &n0, int64_t &kb0, int &nkb, int &z) {
    z = (int)(t / (nm * nn));
    int64_t rem = t - (int64_t)z * nm * nn;
    m0 = (rem % nm) * T::BM;
    n0 = (rem / nm) * BN;
    kb0 = (int64_t)z * kb_per_split;
    int64_t kb1 = kb0 + kb_per_split < nkb_total ? kb0 + kb_per_split : nkb_total;
    nkb = (int)(kb1 > kb0 ? kb1 - kb0 : 0);
  };

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (tc::elect_one()) {
      if (BRES) {  // the whole B once (single N block, no split-K)
        tc::mbar_expect_tx(bres, (uint32_t)(nkb_total * T::B_BYTES));
        for (int i = 0; i < nkb_total; ++i) {
          uint8_t *b = sB + i * T::B_BYTES;
          const int32_t kc = (int32_t)(i * T::BK);
          if (!B_MN) {
            tc::tma_load_2d(b, &tb, bres, kc, 0);
          } else {
#pragma unroll
            for (int j = 0; j < BN / T::B_INNER; ++j)
              tc::tma_load_2d(b + j * (T::B_ROW * T::BK), &tb, bres, j * T::B_INNER, kc);
          }
        }
      }
      uint32_t it = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        int64_t m0, n0, kb0;
        int nkb, z;
        tile_coords(t, m0, n0, kb0, nkb, z);
        for (int i = 0; i < nkb; ++i, ++it) {
          const uint32_t s = it % T::STAGES, r = it / T::STAGES;
          if (r > 0) tc::mbar_wait(&empty[s], (r - 1) & 1);
          tc::mbar_expect_tx(&full[s], T::A_BYTES + T::B_STAGE_BYTES);
          const int32_t kc = (int32_t)((kb0 + i) * T::BK);
          uint8_t *a = sA + s * T::A_BYTES;
          uint8_t *b = sB + s * T::B_STAGE_BYTES;
          if (!A_MN) {
            tc::tma_load_2d(a, &ta, &full[s], kc, (int32_t)m0);
          } else {
            tc::tma_load_2d(a, &ta, &full[s], (int32_t)m0, kc);
            tc::tma_load_2d(a + 8192, &ta, &full[s], (int32_t)(m0 + 64), kc);
          }
          if (BRES) {
          } else if (!B_MN) {
            tc::tma_load_2d(b, &tb, &full[s], kc, (int32_t)n0);
          } else {
#pragma unroll
            for (int j = 0; j < BN / T::B_INNER; ++j)
              tc::tma_load_2d(b + j * (T::B_ROW * T::BK), &tb, &full[s], (int32_t)(n0 + j * T::B_INNER), kc);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc = tc::idesc_bf16(T::BM, BN, A_MN, B_MN);
    if (tc::elect_one()) {
      if (BRES) tc::mbar_wait(bres, 0);
      uint32_t it = 0, li = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++li) {
        int64_t m0, n0, kb0;
        int nkb, z;
        tile_coords(t, m0, n0, kb0, nkb, z);
        const uint32_t acc = li & 1;
        if (li >= 2) tc::mbar_wait(&tempty[acc], ((li >> 1) - 1) & 1);
        tc::tc_fence_after();
        const uint32_t d = tmem + acc * T::ACC_COLS;
        for (int i = 0; i < nkb; ++i, ++it) {
          const uint32_t s = it % T::STAGES;
          tc::mbar_wait(&full[s], (it / T::STAGES) & 1);
          tc::tc_fence_after();
          const uint32_t a = tc::smem_u32(sA + s * T::A_BYTES);
          const uint32_t b = tc::smem_u32(BRES ? sB + (kb0 + i) * T::B_BYTES : sB + s * T::B_BYTES);
#pragma unroll
          for (int kk = 0; kk < T::BK / 16; ++kk) {
            uint64_t ad = A_MN ? tc::sdesc(a + kk * 2048, 8192, 1024, tc::kSw128)
                               : tc::sdesc(a + kk * 32, 16, 1024, tc::kSw128);
            uint64_t bd;
            if (!B_MN) {
              bd = tc::sdesc(b + kk * 32, 16, 1024, tc::kSw128);
            } else {
              constexpr uint32_t swz = T::B_ROW == 128 ? tc::kSw128 : (T::B_ROW == 64 ? tc::kSw64 : tc::kSw32);
              bd = tc::sdesc(b + kk * 16 * T::B_ROW, T::B_ROW * T::BK, 8 * T::B_ROW, swz);
            }
            tc::mma_bf16_ss(d, ad, bd, idesc, (i > 0 || kk > 0) ? 1u : 0u);
          }
          tc::mma_commit(&empty[s]);
        }
        tc::mma_commit(&tfull[acc]);
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ epilogue
    const int g = warp & 3;  // TMEM lane group accessible to this warp
    const int ew = warp - 2;                    // epilogue warp index: staging buffers, mask barriers
    constexpr int CSTEP = T::EPI / 4;           // 64-column chunks: this warp takes h, h + CSTEP, ...
    const int h = ew / 4;
    uint32_t li = 0, ocount = 0;
    float csum[BN / 64 > 0 ? BN / 64 : 1][2] = {};
    // mask tiles are prefetched one 64-column chunk ahead (two buffers)
    auto mask_load = [&](int64_t t, int c64, uint32_t q) {
      if (!E16 || !ep.mask16 || lane != 0 || t >= ntiles) return;
      int64_t m0, n0, kb0;
      int nkb_, z_;
      tile_coords(t, m0, n0, kb0, nkb_, z_);
      if (n0 + c64 * 64 >= N) return;
      tc::mbar_expect_tx(&mbar[ew * 2 + (q & 1)], 4096);
      tc::tma_load_2d(sStg + (ew * 4 + 2 + (q & 1)) * 4096, &tmask, &mbar[ew * 2 + (q & 1)],
                      (int32_t)(n0 + c64 * 64), (int32_t)(m0 + g * 32));
    };
    mask_load(blockIdx.x, h, 0);
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++li) {
      int64_t m0, n0, kb0;
      int nkb, z;
      tile_coords(t, m0, n0, kb0, nkb, z);
      const uint32_t acc = li & 1;
      tc::mbar_wait(&tfull[acc], (li >> 1) & 1);
      tc::tc_fence_after();
      const uint32_t dcol = tmem + acc * T::ACC_COLS + ((uint32_t)(g * 32) << 16);
      const int64_t row = m0 + g * 32 + lane;
      if (ep.out16 == nullptr) {
        float *out = ep.C + (splits > 1 ? (int64_t)z * ep.split_stride : 0);
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 16) {
          uint32_t v[16];
          tc::tmem_ld16(dcol + (uint32_t)c0, v);
          tc::tmem_ld_wait();
          if (row < M) {
            float *dst = out + row * ep.ldc + n0 + c0;
            if (n0 + c0 + 16 <= N && !(ep.accumulate && splits == 1) &&
                ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
#pragma unroll
              for (int j = 0; j < 4; ++j)
                reinterpret_cast<float4 *>(dst)[j] =
                    nkb > 0 ? make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                                          __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3]))
                            : make_float4(0.f, 0.f, 0.f, 0.f);
            } else {
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                if (n0 + c0 + j < N) {
                  float x = nkb > 0 ? __uint_as_float(v[j]) : 0.f;
                  dst[j] = (ep.accumulate && splits == 1) ? dst[j] + x : x;
                }
              }
            }
          }
        }
      } else if constexpr (E16) {
        // bf16 epilogue, 64 columns at a time: TMEM -> registers (scale,
        // mask from a TMA-loaded tile) -> swizzled SMEM staging -> TMA store
        const float sc = (ep.row_scale && row < M) ? ep.row_scale[row] : 1.f;
        const int nch = (int)((N - n0 + 63) / 64) < BN / 64 ? (int)((N - n0 + 63) / 64) : BN / 64;
#pragma unroll 1
        for (int c64 = h; c64 < nch; c64 += CSTEP) {
          const int64_t ncol = n0 + c64 * 64;
          uint8_t *ost = sStg + (ew * 4 + (ocount & 1)) * 4096;
          uint8_t *mst = sStg + (ew * 4 + 2 + (ocount & 1)) * 4096;
          // prefetch this warp's next chunk's mask (this tile's, else the next tile's first)
          if (c64 + CSTEP < nch) mask_load(t, c64 + CSTEP, ocount + 1);
          else mask_load(t + gridDim.x, h, ocount + 1);
          uint32_t v[64];
          tc::tmem_ld32(dcol + (uint32_t)(c64 * 64), *reinterpret_cast<uint32_t (*)[32]>(&v[0]));
          tc::tmem_ld32(dcol + (uint32_t)(c64 * 64 + 32), *reinterpret_cast<uint32_t (*)[32]>(&v[32]));
          tc::tmem_ld_wait();
          float x[64];
#pragma unroll
          for (int j = 0; j < 64; ++j) x[j] = (nkb > 0 && row < M) ? __uint_as_float(v[j]) * sc : 0.f;
          if (ep.mask16) {
            tc::mbar_wait(&mbar[ew * 2 + (ocount & 1)], (ocount >> 1) & 1);
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              const uint4 mv = *reinterpret_cast<const uint4 *>(mst + tc::sw128_off(lane, c));
              const __nv_bfloat16 *mb = reinterpret_cast<const __nv_bfloat16 *>(&mv);
#pragma unroll
              for (int j = 0; j < 8; ++j)
                if (!(__bfloat162float(mb[j]) > 0.f)) x[c * 8 + j] = 0.f;
            }
          }
          if (lane == 0) tc::bulk_wait_read<1>();  // this staging buffer's previous store has read it
          __syncwarp();
#pragma unroll
          for (int c = 0; c < 8; ++c)
            *reinterpret_cast<uint4 *>(ost + tc::sw128_off(lane, c)) =
                make_uint4(tc::pack_bf16(x[c * 8 + 0], x[c * 8 + 1]), tc::pack_bf16(x[c * 8 + 2], x[c * 8 + 3]),
                           tc::pack_bf16(x[c * 8 + 4], x[c * 8 + 5]), tc::pack_bf16(x[c * 8 + 6], x[c * 8 + 7]));
          tc::fence_async_shared();
          __syncwarp();
          if (lane == 0) {
            tc::tma_store_2d(&tout, ost, (int32_t)ncol, (int32_t)(m0 + g * 32));
            tc::bulk_commit();
          }
          if (ep.colsum_part) {
            // lane j sums columns 2j, 2j+1 of the written (bf16) tile over the 32 rows
            float y0 = 0.f, y1 = 0.f;
            const int c = (2 * lane) >> 3, e = (2 * lane) & 7;
#pragma unroll 8
            for (int r = 0; r < 32; ++r) {
              const __nv_bfloat162 p = *reinterpret_cast<const __nv_bfloat162 *>(ost + tc::sw128_off(r, c) + e * 2);
              y0 += __bfloat162float(p.x);
              y1 += __bfloat162float(p.y);
            }
            csum[c64][0] += y0;  // accumulated over this CTA's tiles (single N block)
            csum[c64][1] += y1;
          }
          ++ocount;
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&tempty[acc]);
    }
    if (E16 && ep.colsum_part) {
#pragma unroll
      for (int c64 = 0; c64 < BN / 64; ++c64)
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int col = c64 * 64 + 2 * lane + u;
          if (col < N) ep.colsum_part[((int64_t)blockIdx.x * 4 + g) * N + col] = csum[c64][u];
        }
    }
  }
  if (E16 && warp >= 2 && lane == 0) tc::bulk_wait<0>();  // TMA stores drained before exit
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc<T::TMEM_COLS>(tmem);
}

template <int BN, bool A_MN, bool B_MN, bool E16, bool BRES = false>
static dsmpnn_status launch_tgemm(const TgemmArgs &a, cudaStream_t s) {
  using T = TG<BN, A_MN, B_MN, E16, BRES>;
  CUtensorMap ta, tb, tout, tmask;
  memset(&tout, 0, sizeof(tout));
  memset(&tmask, 0, sizeof(tmask));
  if (E16) {
    DS_TRY(make_tmap_bf16(&tout, a.out16, a.N, a.M, a.ld16, 64, 32));
    if (a.mask16) DS_TRY(make_tmap_bf16(&tmask, a.mask16, a.N, a.M, a.ldmask, 64, 32));
  }
  if (!A_MN) DS_TRY(make_tmap_bf16(&ta, a.A, a.K, a.M, a.lda, 64, 128));
  else DS_TRY(make_tmap_bf16(&ta, a.A, a.M, a.K, a.lda, 64, 64));
  if (!B_MN) DS_TRY(make_tmap_bf16(&tb, a.B, a.K, a.N, a.ldb, 64, BN));
  else DS_TRY(make_tmap_bf16(&tb, a.B, a.N, a.K, a.ldb, T::B_INNER, 64));
  auto kern = tgemm_kernel<BN, A_MN, B_MN, E16, BRES>;
  // set on every launch: the attribute belongs to the current device's context
  DS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, T::SMEM));
  int64_t nkb = (a.K + 63) / 64;
  int splits = a.splits < 1 ? 1 : a.splits;
  int kbps = (int)ceil_div(nkb, splits);
  if (kbps < 1) kbps = 1;
  splits = (int)std::max<int64_t>(1, ceil_div(nkb, kbps));
  int64_t ntiles = ceil_div(a.M, T::BM) * ceil_div(a.N, BN) * splits;
  int per_sm = (227 * 1024) / T::SMEM;
  if (per_sm < 1) per_sm = 1;
  if (per_sm > 2) per_sm = 2;
  if (per_sm * T::TMEM_COLS > 512) per_sm = 512 / T::TMEM_COLS;
  int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)kNumSMs * per_sm));
  DS_CHECK_ARG(T::EPI == 4 || a.colsum_part == nullptr, DSMPNN_ERR_UNSUPPORTED,
               "tgemm: column sums need the resident-B bf16 epilogue");
  DS_CUDA(launch_pdl(kern, grid, T::THREADS, T::SMEM, s, ta, tb, tout, tmask, a.M, a.N, a.K, kbps, a, splits));
  DS_LAUNCH_CHECK();
  return DSMPNN_OK;
}

template <bool A_MN, bool B_MN>
static dsmpnn_status dispatch_bn(const TgemmArgs &a, cudaStream_t s) {
  if (a.out16) {
    DS_CHECK_ARG(a.N >= 64, DSMPNN_ERR_UNSUPPORTED, "tgemm: bf16 epilogue needs N >= 64");
    DS_CHECK_ARG(!a.colsum_part || a.N <= 256, DSMPNN_ERR_UNSUPPORTED, "tgemm: column sums need N <= 256");
    if (a.N <= 64) return launch_tgemm<64, A_MN, B_MN, true>(a, s);
    if (a.N <= 128) return launch_tgemm<128, A_MN, B_MN, true>(a, s);
    if (a.b_resident && a.N <= 256 && a.K <= 4 * 64 && a.splits <= 1)
      return launch_tgemm<256, A_MN, B_MN, true, true>(a, s);
    return launch_tgemm<256, A_MN, B_MN, true>(a, s);
  }
  if (a.N <= 16) return launch_tgemm<16, A_MN, B_MN, false>(a, s);
  if (a.N <= 32) return launch_tgemm<32, A_MN, B_MN, false>(a, s);
  if (a.N <= 64) return launch_tgemm<64, A_MN, B_MN, false>(a, s);
  if (a.N <= 128) return launch_tgemm<128, A_MN, B_MN, false>(a, s);
  return launch_tgemm<256, A_MN, B_MN, false>(a, s);
}

dsmpnn_status tgemm(const TgemmArgs &a, cudaStream_t s) {
  if (a.M <= 0 || a.N <= 0) return DSMPNN_OK;
  DS_CHECK_ARG(a.out16 == nullptr || a.splits <= 1, DSMPNN_ERR_INVALID_ARG, "tgemm: bf16 epilogue needs splits == 1");
  DS_CHECK_ARG(!(a.N > 64 && a.N % 64 != 0 && a.b_mn_major), DSMPNN_ERR_UNSUPPORTED,
               "tgemm: N-major B with N > 64 needs N %% 64 == 0");
  if (!a.a_mn_major && !a.b_mn_major) return dispatch_bn<false, false>(a, s);
  if (!a.a_mn_major && a.b_mn_major) return dispatch_bn<false, true>(a, s);
  if (a.a_mn_major && !a.b_mn_major) return dispatch_bn<true, false>(a, s);
  return dispatch_bn<true, true>(a, s);
}

__global__ void splitk_sum_kernel(const float *__restrict__ p, int splits, int64_t stride, int64_t M, int64_t N,
                                  int64_t ld, float *__restrict__ C, int64_t ldc, int accumulate) {
  int64_t total = M * N;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t m = t / N, n = t - m * N;
    float q[4] = {0.f, 0.f, 0.f, 0.f};  // 4 loads in flight, fixed combination order
    const float *src = p + m * ld + n;
    int z = 0;
    for (; z + 4 <= splits; z += 4) {
#pragma unroll
      for (int u = 0; u < 4; ++u) q[u] += src[(int64_t)(z + u) * stride];
    }
    for (; z < splits; ++z) q[0] += src[(int64_t)z * stride];
    const float s = (q[0] + q[1]) + (q[2] + q[3]);
    float *c = C + m * ldc + n;
    *c = accumulate ? *c + s : s;
  }
}

dsmpnn_status splitk_sum(const float *partial, int splits, int64_t split_stride, int64_t M, int64_t N, int64_t ld,
                         float *C, int64_t ldc, int accumulate, cudaStream_t s) {
  if (M <= 0 || N <= 0) return DSMPNN_OK;
  int g = (int)std::min<int64_t>(ceil_div(M * N, 256), 148 * 8);
  splitk_sum_kernel<<<g, 256, 0, s>>>(partial, splits, split_stride, M, N, ld, C, ldc, accumulate);
  DS_LAUNCH_CHECK();
  return DSMPNN_OK;
}

}  // namespace dsmpnn

using namespace dsmpnn;

extern "C" dsmpnn_status dsmpnn_gemm_bf16(int64_t M, int64_t N, int64_t K, const void *A, int64_t lda,
                                          int32_t a_mn_major, const void *B, int64_t ldb, int32_t b_mn_major,
                                          float *C, int64_t ldc, int32_t splits, float *partial, int32_t accumulate,
                                          void *stream) {
  DS_CHECK_ARG(M >= 0 && N >= 0 && K >= 0, DSMPNN_ERR_INVALID_ARG, "gemm_bf16: negative size");
  cudaStream_t s = as_stream(stream);
  if (splits > 1) {
    DS_CHECK_ARG(partial != nullptr, DSMPNN_ERR_INVALID_ARG, "gemm_bf16: split-K needs a partial buffer");
    TgemmArgs a{M, N, K, A, lda, a_mn_major != 0, B, ldb, b_mn_major != 0, partial, N, splits, M * N, 0};
    DS_TRY(tgemm(a, s));
    int64_t nkb = (K + 63) / 64;
    int kbps = (int)std::max<int64_t>(1, ceil_div(nkb, splits));
    int real = (int)std::max<int64_t>(1, ceil_div(nkb, kbps));
    return splitk_sum(partial, real, M * N, M, N, N, C, ldc, accumulate, s);
  }
  TgemmArgs a{M, N, K, A, lda, a_mn_major != 0, B, ldb, b_mn_major != 0, C, ldc, 1, 0, accumulate};
  return tgemm(a, s);
}
