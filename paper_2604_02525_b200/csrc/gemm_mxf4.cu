// gemm_mxf4.cu — block-scaled MXFP4 GEMM on the 5th-gen tensor cores (sm_100a).
//
// C[M x N] = deq(A_store) · deq(B_store)^T, both operands K-major E2M1 (two codes per
// byte, element 2j in the low nibble) with one UE8M0 scale per 32 elements along K
// (the "MXFP4 matmul" of eq:inner_hadamard P:95 / eq:oe_left P:273 / eq:oe_right P:280).
//
// Design (persistent, warp-specialised, one CTA per SM):
//   warp 0      TMA producer: A/B tiles (128 B x rows, 128B swizzle) + scale-factor
//               chunks (1D bulk copies) into a kStages-deep smem ring (mbarrier full/empty)
//   warp 1      MMA issuer (one thread): tcgen05.cp of the stage's scale factors into TMEM,
//               then 4 x tcgen05.mma.kind::mxf4.block_scale.block32 (128 x BN x 64) per
//               stage; tcgen05.commit frees the smem slot / publishes the accumulator
//   warp 2      TMEM allocator (512 columns: 2 accumulator buffers + scale factors)
//   warps 4..7  epilogue: tcgen05.ld 32x32b -> registers -> global (fp32 or bf16), while
//               the MMA warp already accumulates the next tile into the other buffer.
#include "common.cuh"
#include "kernels.h"
#include "epilogue.cuh"
#include "ptx.cuh"

namespace adahop {
namespace mxf4 {

constexpr int BM = 128;
constexpr int BN = 128;
constexpr int BK = 256;                 // fp4 elements per stage (= 128 bytes per row)
constexpr int kStages = 6;
constexpr int kABytes = BM * BK / 2;    // 16 KB
constexpr int kBBytes = BN * BK / 2;    // 16 KB
constexpr int kSfaBytes = (BM / 128) * 2 * 512;  // 2 K-chunks of 128 rows
constexpr int kSfbBytes = (BN / 128) * 2 * 512;
constexpr int kStageBytes = kABytes + kBBytes + kSfaBytes + kSfbBytes;
constexpr int kTmemCols = 512;
constexpr int kAccCols = BN;            // per accumulator buffer
constexpr int kSfCol = 2 * kAccCols;    // first TMEM column of the scale factors
constexpr int kSfbColOff = 8;           // SFB after the 8 SFA columns
constexpr int kThreads = 256;
constexpr int kEpiBytes = 4 * kEpiStageBytes;   // one staging block per epilogue warp
constexpr size_t kSmemBytes = size_t(kStages) * kStageBytes + kEpiBytes + 1024 /*align*/ + 256 /*barriers*/;

// Instruction descriptor, kind::mxf4 block-scaled (E2M1 x E2M1, UE8M0, fp32 accumulate).
__host__ __device__ constexpr uint32_t make_idesc(int m, int n) {
  return (1u << 7)             // a_format = E2M1
         | (1u << 10)          // b_format = E2M1
         | (uint32_t(n >> 3) << 17)
         | (1u << 23)          // scale format UE8M0
         | (uint32_t(m >> 4) << 24);
}

// Grouped rasterisation: tiles are walked in groups of kGroupM m-blocks with n fastest
// inside a group, so the ~148 tiles in flight share a few A panels and the B panels stay
// L2-resident (plain m-fastest order streams all of A once per n-block).
constexpr int64_t kGroupM = 8;
__device__ __forceinline__ void tile_coords(int64_t t, int64_t mblocks, int64_t nblocks, int64_t& mb,
                                            int64_t& nb) {
  const int64_t per_group = kGroupM * nblocks;
  const int64_t g = t / per_group;
  const int64_t first_m = g * kGroupM;
  const int64_t gm = mblocks - first_m < kGroupM ? mblocks - first_m : kGroupM;
  const int64_t local = t - g * per_group;
  mb = first_m + local % gm;
  nb = local / gm;
}

__global__ void __launch_bounds__(kThreads, 1)
    k_gemm_mxf4(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                const uint8_t* __restrict__ sfa, const uint8_t* __restrict__ sfb, void* C,
                int out_f32, int64_t ldc, int64_t M, int64_t N, int64_t K, const OePatch oe) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);  // stays in the shared window
  uint8_t* epi_smem = smem + size_t(kStages) * kStageBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(epi_smem + kEpiBytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + kStages;
  uint64_t* tfull = bars + 2 * kStages;
  uint64_t* tempty = bars + 2 * kStages + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 4);

  const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
  const int64_t mblocks = (M + BM - 1) / BM;
  const int64_t nblocks = (N + BN - 1) / BN;
  const int64_t ntiles = mblocks * nblocks;
  const int nks = int((K + BK - 1) / BK);
  const int64_t kchunks = sf_kchunks(K);

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tm_a);
    ptx::prefetch_tmap(&tm_b);
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&tfull[b], 1);
      ptx::mbar_init(&tempty[b], 4);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc<kTmemCols>(tmem_slot);
  ptx::griddep_launch();
  ptx::griddep_wait();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // ------------------------------------------------------------ TMA producer
    int stage = 0;
    uint32_t phase = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      int64_t mb, nb;
      tile_coords(tile, mblocks, nblocks, mb, nb);
      for (int ks = 0; ks < nks; ++ks) {
        ptx::mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* sa = smem + size_t(stage) * kStageBytes;
        uint8_t* sb = sa + kABytes;
        uint8_t* ssfa = sb + kBBytes;
        uint8_t* ssfb = ssfa + kSfaBytes;
        ptx::mbar_arrive_expect_tx(&full[stage], kStageBytes);
        ptx::tma_load_2d(sa, &tm_a, &full[stage], ks * (BK / 2), int32_t(mb * BM));
        ptx::tma_load_2d(sb, &tm_b, &full[stage], ks * (BK / 2), int32_t(nb * BN));
        ptx::bulk_load(ssfa, sfa + (mb * kchunks + 2 * ks) * 512, kSfaBytes, &full[stage]);
        ptx::bulk_load(ssfb, sfb + (nb * kchunks + 2 * ks) * 512, kSfbBytes, &full[stage]);
        if (++stage == kStages) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = make_idesc(BM, BN);
    int stage = 0;
    uint32_t phase = 0;
    int64_t lt = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++lt) {
      const uint32_t buf = uint32_t(lt & 1);
      const uint32_t use = uint32_t(lt >> 1);
      ptx::mbar_wait(&tempty[buf], (use & 1) ^ 1);
      ptx::tc_fence_after();
      const uint32_t d_tmem = tmem_base + buf * kAccCols;
      for (int ks = 0; ks < nks; ++ks) {
        ptx::mbar_wait(&full[stage], phase);
        ptx::tc_fence_after();
        uint8_t* sa = smem + size_t(stage) * kStageBytes;
        uint8_t* sb = sa + kABytes;
        uint8_t* ssfa = sb + kBBytes;
        uint8_t* ssfb = ssfa + kSfaBytes;
        // scale factors -> TMEM (executes in order with the MMAs below)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          ptx::tmem_cp_32x128b_warpx4(tmem_base + kSfCol + 4 * c,
                                      ptx::make_sdesc(ptx::smem_u32(ssfa + c * 512), 0, 128, 0));
          ptx::tmem_cp_32x128b_warpx4(tmem_base + kSfCol + kSfbColOff + 4 * c,
                                      ptx::make_sdesc(ptx::smem_u32(ssfb + c * 512), 0, 128, 0));
        }
        const uint32_t a_addr = ptx::smem_u32(sa), b_addr = ptx::smem_u32(sb);
#pragma unroll
        for (int j = 0; j < BK / 64; ++j) {
          const uint32_t sf_id = uint32_t(j & 1) * 2;
          const uint32_t sfa_t = (tmem_base + kSfCol + 4 * (j >> 1)) | (sf_id << 30);
          const uint32_t sfb_t = (tmem_base + kSfCol + kSfbColOff + 4 * (j >> 1)) | (sf_id << 30);
          const uint32_t id = idesc | (sf_id << 4) | (sf_id << 29);
          const uint64_t adesc = ptx::make_sdesc(a_addr + j * 32, 16, 1024, 2);
          const uint64_t bdesc = ptx::make_sdesc(b_addr + j * 32, 16, 1024, 2);
          ptx::mma_mxf4(d_tmem, adesc, bdesc, id, sfa_t, sfb_t, (ks > 0 || j > 0) ? 1u : 0u);
        }
        ptx::tc_commit(&empty[stage]);
        if (++stage == kStages) { stage = 0; phase ^= 1; }
      }
      ptx::tc_commit(&tfull[buf]);
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    const uint32_t q = warp & 3;  // TMEM lane quadrant of this warp
    // fused outlier product: fold this CTA's share of Dt while the first main loop runs
    oe_prefold(oe, int(threadIdx.x) - 128, 128, 1);
    oe_prefold_wait(oe);
    int64_t lt = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++lt) {
      int64_t mb, nb;
      tile_coords(tile, mblocks, nblocks, mb, nb);
      const uint32_t buf = uint32_t(lt & 1);
      const uint32_t use = uint32_t(lt >> 1);
      ptx::mbar_wait(&tfull[buf], use & 1);
      ptx::tc_fence_after();
      // coalesced store through the per-warp smem stage: 128 bytes of each row at a time
      uint8_t* stg = epi_smem + q * kEpiStageBytes;
      const int64_t m0 = mb * BM + q * 32;
      const int rows_valid = int(M - m0 < 32 ? (M - m0 > 0 ? M - m0 : 0) : 32);
      const int elt = out_f32 ? 4 : 2;
      const int cols_per_grp = 128 / elt;            // 32 fp32 or 64 bf16 columns
      const bool vec_ok = ((reinterpret_cast<uintptr_t>(C) | uintptr_t(ldc * elt)) & 15) == 0;
#pragma unroll 1
      for (int g = 0; g < BN / cols_per_grp; ++g) {
        const int64_t n0 = nb * BN + g * cols_per_grp;
        const uint32_t tbase = tmem_base + ((q * 32) << 16) + buf * kAccCols + g * cols_per_grp;
        uint32_t w[32];
        if (out_f32) {
          ptx::tmem_ld_32x32b_x32(tbase, w);
          ptx::tmem_ld_wait();
        } else {
          uint32_t r0[32], r1[32];
          ptx::tmem_ld_32x32b_x32(tbase, r0);
          ptx::tmem_ld_32x32b_x32(tbase + 32, r1);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            w[i] = pack_bf16x2(r0[2 * i], r0[2 * i + 1]);
            w[16 + i] = pack_bf16x2(r1[2 * i], r1[2 * i + 1]);
          }
        }
        const int64_t nrem = N - n0;
        const int bytes_valid = int(nrem >= cols_per_grp ? 128 : (nrem > 0 ? nrem * elt : 0));
        if (rows_valid > 0 && bytes_valid > 0) {
          epi_stage_only128(stg, w);
          epi_patch_outliers(stg, oe, m0, n0, cols_per_grp, elt, M, N);
          epi_flush128(stg, static_cast<char*>(C) + (m0 * ldc + n0) * elt, ldc * elt, rows_valid, bytes_valid, elt,
                       vec_ok);
          __syncwarp();
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&tempty[buf]);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<kTmemCols>(tmem_base);
  }
}

}  // namespace mxf4

cudaError_t launch_gemm_mxf4(const Mxf4GemmArgs& a, int num_sms, cudaStream_t st) {
  using namespace mxf4;
  CUtensorMap tma, tmb;
  // FP4 codes as bytes: [rows][K/2], box 128 bytes x 128 rows, 128B swizzle.
  if (!make_tmap_2d(&tma, CU_TENSOR_MAP_DATA_TYPE_UINT8, a.a_codes, uint64_t(a.K / 2), uint64_t(a.M),
                    uint64_t(a.K / 2), 128, BM, CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;
  if (!make_tmap_2d(&tmb, CU_TENSOR_MAP_DATA_TYPE_UINT8, a.b_codes, uint64_t(a.K / 2), uint64_t(a.N),
                    uint64_t(a.K / 2), 128, BN, CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;
  static std::atomic<uint64_t> attr{0};
  cudaError_t ae = once_per_device(attr, [] {
    return cudaFuncSetAttribute(k_gemm_mxf4, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmemBytes));
  });
  if (ae != cudaSuccess) return ae;
  const int64_t tiles = ((a.M + BM - 1) / BM) * ((a.N + BN - 1) / BN);
  const int grid = int(tiles < num_sms ? tiles : num_sms);
  return launch_k(k_gemm_mxf4, dim3(grid), dim3(kThreads), kSmemBytes, st, 1, tma, tmb, a.a_sf, a.b_sf, a.C,
                  a.out_f32 ? 1 : 0, a.ldc, a.M, a.N, a.K, a.oe);
}

}  // namespace adahop
