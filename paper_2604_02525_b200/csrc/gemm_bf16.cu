// gemm_bf16.cu — BF16 GEMM on the 5th-gen tensor cores (tcgen05.mma.kind::f16, sm_100a).
//
// Serves two roles on the AdaHOP path:
//   * the BF16 outlier GEMM of OE (A_out·B, eq:oe_left P:273; A·B_out, eq:oe_right P:280),
//     computed as D[Mb x k] = Big[Mb x K] · Slice[k x K]^T with split-K fp32 partials that
//     launch_outlier_reduce folds and scatters into C ("Fused Scatter-Add");
//   * the full BF16 product of AdaHOP-Lv2 CC pairs, written directly to C.
// Operands may be K-major or MN-major (the wgrad / dgrad operands are K-strided in memory);
// TMA loads 128B-swizzled tiles of either kind and the UMMA descriptors describe both.
//
// One output tile (128 x BN) per CTA over a K range; warp 0 = TMA producer, warp 1 = MMA
// issuer, warp 2 = TMEM allocator, all 4 warps run the epilogue.
#include "common.cuh"
#include "kernels.h"
#include "epilogue.cuh"
#include "ptx.cuh"

namespace adahop {
namespace bf16g {

constexpr int BM = 128;
constexpr int BK = 64;  // bf16 elements per stage (128 bytes along K)
constexpr int kStagesMax = 4;
constexpr int kThreads = 128;

__host__ __device__ constexpr uint32_t make_idesc(int m, int n, int a_mn, int b_mn) {
  return (1u << 4)                 // D format F32
         | (1u << 7)               // A = BF16
         | (1u << 10)              // B = BF16
         | (uint32_t(a_mn) << 15)  // A major (0 = K, 1 = MN)
         | (uint32_t(b_mn) << 16)  // B major
         | (uint32_t(n >> 3) << 17)
         | (uint32_t(m >> 4) << 24);
}

template <int BN, bool kDeep = false>
struct Cfg {
  static constexpr int kABytes = BM * BK * 2;  // 16 KB
  static constexpr int kBBytes = BN * BK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kTmemCols = BN < 32 ? 32 : BN;
  // skinny outlier tiles (BN <= 64): 3 stages so that two CTAs share an SM (the split-K grid is
  // sized for two per SM); wider tiles: 4 stages, one CTA per SM
  // kDeep (one short K range per CTA, the direct-Dt outlier product): every k-step in flight at once
  static constexpr int kStages = kDeep ? 8 : (BN <= 64 ? 3 : kStagesMax);
  static constexpr size_t kSmem = size_t(kStages) * kStageBytes + 4 * kEpiStageBytes + 1024 + 256;
};

// Load one operand tile of `rows` x 64(K) into smem (128B swizzle).
//  K-major: one box {64 k, rows}            -> rows x 128 B
//  MN-major: rows/64 boxes {64 mn, 64 k}    -> each 64 k-rows x 128 B, stacked every 8 KB
template <int ROWS>
__device__ __forceinline__ void load_operand(uint8_t* dst, const CUtensorMap* tm, int mn,
                                             uint64_t* bar, int32_t k0, int32_t r0) {
  if (!mn) {
    ptx::tma_load_2d(dst, tm, bar, k0, r0);
  } else {
#pragma unroll
    for (int b = 0; b < ROWS / 64; ++b) ptx::tma_load_2d(dst + b * 8192, tm, bar, r0 + b * 64, k0);
  }
}

__device__ __forceinline__ uint64_t operand_desc(uint32_t base, int mn, int j) {
  // j-th K=16 slice of the stage
  return mn ? ptx::make_sdesc(base + j * 2048, 8192, 1024, 2)   // MN-major: 16 k-rows x 128 B
            : ptx::make_sdesc(base + j * 32, 16, 1024, 2);      // K-major: 32 bytes along K
}

template <int BN, bool kDeep = false>
__global__ void __launch_bounds__(kThreads)
    k_gemm_bf16(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                int a_mn, int b_mn, int64_t Mb, int64_t Nb, int64_t K, int mode, void* C,
                int out_f32, int64_t ldc, float* part, int64_t npad, float* Dt) {
  using G = Cfg<BN, kDeep>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);  // stays in the shared window
  constexpr int kStages = G::kStages;
  uint8_t* epi_smem = smem + size_t(kStages) * G::kStageBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(epi_smem + 4 * kEpiStageBytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + kStages;
  uint64_t* done = bars + 2 * kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 1);

  const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
  const int64_t m0 = int64_t(blockIdx.x) * BM;
  const int64_t n0 = int64_t(blockIdx.y) * BN;
  const int split = blockIdx.z, splits = gridDim.z;
  const int nks = int((K + BK - 1) / BK);
  const int per = (nks + splits - 1) / splits;
  const int ks0 = split * per;
  const int ks1 = min(nks, ks0 + per);

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tm_a);
    ptx::prefetch_tmap(&tm_b);
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    ptx::mbar_init(done, 1);
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc<G::kTmemCols>(tmem_slot);
  ptx::griddep_launch();
  ptx::griddep_wait();   // the prologue above overlapped the previous kernel's tail
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0 && lane == 0) {
    int stage = 0;
    uint32_t phase = 0;
    for (int ks = ks0; ks < ks1; ++ks) {
      ptx::mbar_wait(&empty[stage], phase ^ 1);
      uint8_t* sa = smem + size_t(stage) * G::kStageBytes;
      uint8_t* sb = sa + G::kABytes;
      ptx::mbar_arrive_expect_tx(&full[stage], G::kStageBytes);
      load_operand<BM>(sa, &tm_a, a_mn, &full[stage], ks * BK, int32_t(m0));
      load_operand<BN>(sb, &tm_b, b_mn, &full[stage], ks * BK, int32_t(n0));
      if (++stage == kStages) { stage = 0; phase ^= 1; }
    }
  } else if (warp == 1 && lane == 0) {
    const uint32_t idesc = make_idesc(BM, BN, a_mn, b_mn);
    int stage = 0;
    uint32_t phase = 0;
    for (int ks = ks0; ks < ks1; ++ks) {
      ptx::mbar_wait(&full[stage], phase);
      ptx::tc_fence_after();
      const uint32_t a_addr = ptx::smem_u32(smem + size_t(stage) * G::kStageBytes);
      const uint32_t b_addr = a_addr + G::kABytes;
#pragma unroll
      for (int j = 0; j < BK / 16; ++j)
        ptx::mma_bf16(tmem_base, operand_desc(a_addr, a_mn, j), operand_desc(b_addr, b_mn, j), idesc,
                      (ks > ks0 || j > 0) ? 1u : 0u);
      ptx::tc_commit(&empty[stage]);
      if (++stage == kStages) { stage = 0; phase ^= 1; }
    }
    ptx::tc_commit(done);
  }
  // ---------------------------------------------------------------- epilogue (4 warps)
  const bool has_k = ks1 > ks0;
  if (has_k) {
    ptx::mbar_wait(done, 0);
    ptx::tc_fence_after();
  }
  __syncwarp();
  // coalesced store through the per-warp smem stage (epilogue.cuh)
  uint8_t* stg = epi_smem + warp * kEpiStageBytes;
  const int64_t mw = m0 + warp * 32;
  const int rows_valid = int(Mb - mw < 32 ? (Mb - mw > 0 ? Mb - mw : 0) : 32);
  char* cbase;
  int64_t ldb_bytes, ncols;
  int elt;
  if (mode == 1) {
    elt = 4;
    cbase = reinterpret_cast<char*>(part + (int64_t(split) * Mb + mw) * npad);
    ldb_bytes = npad * 4;
    ncols = npad;
  } else {
    elt = out_f32 ? 4 : 2;
    cbase = static_cast<char*>(C) + mw * ldc * elt;
    ldb_bytes = ldc * elt;
    ncols = Nb;
  }
  const bool vec_ok = ((reinterpret_cast<uintptr_t>(cbase) | uintptr_t(ldb_bytes)) & 15) == 0;
  const int cols_per_grp = 128 / elt;
#pragma unroll 1
  for (int g = 0; g < (BN + cols_per_grp - 1) / cols_per_grp; ++g) {
    const int64_t nc = n0 + g * cols_per_grp;
    uint32_t w[32];
    uint32_t r0[32], r1[32];
    const uint32_t tb = tmem_base + ((warp * 32) << 16) + g * cols_per_grp;
    if (has_k) {
      ptx::tmem_ld_32x32b_x32(tb, r0);
      if (elt == 2) ptx::tmem_ld_32x32b_x32(tb + 32, r1);
      ptx::tmem_ld_wait();
    } else {
#pragma unroll
      for (int v = 0; v < 32; ++v) { r0[v] = 0u; r1[v] = 0u; }
    }
    if (elt == 4) {
#pragma unroll
      for (int v = 0; v < 32; ++v) w[v] = r0[v];
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        w[i] = pack_bf16x2(r0[2 * i], r0[2 * i + 1]);
        w[16 + i] = pack_bf16x2(r1[2 * i], r1[2 * i + 1]);
      }
    }
    if (mode == 1 && Dt != nullptr) {
      // one K range (no split): lane = row m, register v = column j -> Dt[j][m], 128-byte runs
      const int64_t m = mw + lane;
#pragma unroll
      for (int v = 0; v < 32; ++v)
        if (m < Mb && nc + v < Nb) Dt[(nc + v) * Mb + m] = __uint_as_float(r0[v]);
      continue;
    }
    const int64_t nrem = ncols - nc;
    const int bytes_valid = int(nrem >= cols_per_grp ? 128 : (nrem > 0 ? nrem * elt : 0));
    if (rows_valid > 0 && bytes_valid > 0)
      epi_store_rows128(stg, w, cbase + nc * elt, ldb_bytes, rows_valid, bytes_valid,
                        elt, vec_ok);
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<G::kTmemCols>(tmem_base);
  }
}

// Deterministic split-K fold into the transposed outlier product Dt[j][m] = sum_s part[s][m][j]
// (fixed order s = 0, 1, ...), through a 32 x 32 smem tile so that both the partial reads
// (along j) and the Dt writes (along m) are coalesced. The MXFP4 GEMM epilogue then reads Dt
// with lanes along m (OE-Right) or along n (OE-Left): coalesced in both cases.
__global__ void __launch_bounds__(1024) k_outlier_fold(const float* __restrict__ part, int splits, int64_t Mb,
                                                      int64_t npad, int k, float* __restrict__ Dt) {
  ptx::griddep_launch();
  ptx::griddep_wait();
  __shared__ float tile[32][33];
  const int64_t m0 = int64_t(blockIdx.x) * 32;
  const int j0 = blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;
  {
    const int64_t m = m0 + ty;
    const int j = j0 + tx;
    float v = 0.f;
    if (m < Mb && j < k) {
      const float* pp = part + m * npad + j;
      const int64_t stride = Mb * npad;
      int s = 0;
      for (; s + 8 <= splits; s += 8) {
        float t[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) t[u] = pp[(s + u) * stride];
#pragma unroll
        for (int u = 0; u < 8; ++u) v += t[u];
      }
      for (; s < splits; ++s) v += pp[s * stride];
    }
    tile[ty][tx] = v;
  }
  __syncthreads();
  const int j = j0 + ty;
  const int64_t m = m0 + tx;
  if (m < Mb && j < k) Dt[int64_t(j) * Mb + m] = tile[tx][ty];
}

}  // namespace bf16g

int64_t bf16_gemm_npad(int64_t Nb) {
  if (Nb <= 32) return 32;
  if (Nb <= 64) return 64;
  if (Nb <= 128) return 128;
  return ((Nb + 255) / 256) * 256;
}

int bf16_gemm_splits(int64_t Mb, int64_t K, int num_sms) {
  const int64_t mt = (Mb + bf16g::BM - 1) / bf16g::BM;
  const int64_t nks = (K + bf16g::BK - 1) / bf16g::BK;
  // short K (the dgrad OE-Left product over d_out, e.g. 64 x 512 x 2048): one K range per CTA,
  // whose epilogue writes Dt itself — split-K would add the partial round trip and a fold launch
  if (nks <= 16) return 1;
  int64_t s = (2 * num_sms) / mt;            // one full wave of ~2 CTAs per SM
  if (s > nks) s = nks;
  if (s > 32) s = 32;
  if (s < 1) s = 1;
  return int(s);
}

template <int BN, bool kDeep = false>
static cudaError_t launch_bn(const Bf16GemmArgs& a, cudaStream_t st) {
  using G = bf16g::Cfg<BN, kDeep>;
  CUtensorMap tma, tmb;
  // A: K-major [Mb][K] (box {64, 128}) or MN-major [K][Mb] (box {64, 64})
  if (!a.a_mn) {
    if (!make_tmap_2d(&tma, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, a.A, uint64_t(a.K), uint64_t(a.Mb),
                      uint64_t(a.lda) * 2, 64, bf16g::BM, CU_TENSOR_MAP_SWIZZLE_128B))
      return cudaErrorInvalidValue;
  } else {
    if (!make_tmap_2d(&tma, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, a.A, uint64_t(a.Mb), uint64_t(a.K),
                      uint64_t(a.lda) * 2, 64, 64, CU_TENSOR_MAP_SWIZZLE_128B))
      return cudaErrorInvalidValue;
  }
  if (!a.b_mn) {
    if (!make_tmap_2d(&tmb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, a.B, uint64_t(a.K), uint64_t(a.Nb),
                      uint64_t(a.ldb) * 2, 64, BN, CU_TENSOR_MAP_SWIZZLE_128B))
      return cudaErrorInvalidValue;
  } else {
    if (BN < 64) return cudaErrorInvalidValue;
    if (!make_tmap_2d(&tmb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, a.B, uint64_t(a.Nb), uint64_t(a.K),
                      uint64_t(a.ldb) * 2, 64, 64, CU_TENSOR_MAP_SWIZZLE_128B))
      return cudaErrorInvalidValue;
  }
  static std::atomic<uint64_t> attr{0};
  cudaError_t ae = once_per_device(attr, [] {
    return cudaFuncSetAttribute(bf16g::k_gemm_bf16<BN, kDeep>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(G::kSmem));
  });
  if (ae != cudaSuccess) return ae;
  const int splits = a.mode == 1 ? a.splits : 1;
  dim3 grid(unsigned((a.Mb + bf16g::BM - 1) / bf16g::BM),
            unsigned(a.mode == 1 ? 1 : (a.Nb + BN - 1) / BN), unsigned(splits));
  return launch_k(bf16g::k_gemm_bf16<BN, kDeep>, grid, dim3(bf16g::kThreads), G::kSmem, st, 1, tma, tmb, a.a_mn, a.b_mn,
                  a.Mb, a.Nb, a.K, a.mode, a.C, a.out_f32 ? 1 : 0, a.ldc, a.part, a.npad,
                  a.mode == 1 && splits == 1 ? a.Dt : nullptr);
}

cudaError_t launch_gemm_bf16(const Bf16GemmArgs& a, cudaStream_t st) {
  if (a.mode == 0) return launch_bn<128>(a, st);
  if (a.splits == 1 && a.Dt != nullptr && (a.K + bf16g::BK - 1) / bf16g::BK <= 8) {
    switch (a.npad) {   // direct Dt, short K: the CTA's whole K range in flight
      case 32: return launch_bn<32, true>(a, st);
      case 64: return launch_bn<64, true>(a, st);   // 8 x 24 KB stages
      default: break;
    }
  }
  switch (a.npad) {
    case 32: return launch_bn<32>(a, st);
    case 64: return launch_bn<64>(a, st);
    case 128: return launch_bn<128>(a, st);
    case 256: return launch_bn<256>(a, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_outlier_fold(const float* part, int splits, int64_t Mb, int64_t npad, int k, float* Dt,
                                cudaStream_t st) {
  dim3 grid(unsigned((Mb + 31) / 32), unsigned((k + 31) / 32));
  return launch_k(bf16g::k_outlier_fold, grid, dim3(32, 32), 0, st, 1, part, splits, Mb, npad, k, Dt);
}

}  // namespace adahop
