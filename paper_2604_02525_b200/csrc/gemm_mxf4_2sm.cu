// gemm_mxf4_2sm.cu — block-scaled MXFP4 GEMM on CTA pairs (tcgen05 cta_group::2, sm_100a).
//
// Same operation as gemm_mxf4.cu (C = deq(A_store) · deq(B_store)^T, E2M1 with UE8M0 per 32
// along K — the MXFP4 matmul of eq:inner_hadamard P:95 / eq:oe_left P:273 / eq:oe_right
// P:280) but each output tile is 256 x BN and is computed by a 2-CTA cluster: CTA r holds
// rows [128 r, 128 r + 128) of the A tile and rows [BN/2 r, BN/2 (r+1)) of the B tile, the
// leader CTA issues tcgen05.mma.cta_group::2 (M = 256) and each CTA's TMEM receives its own
// 128 x BN accumulator half. Per SM this halves the operand bytes per flop of the 1-CTA
// 128 x 128 kernel, which was bound by the latency of refilling its smem ring from L2.
//
// Roles (384 threads per CTA): warp 0 TMA producer (both CTAs; completion is signalled on
// the leader's barrier), warp 1 MMA issuer (leader only), warp 2 TMEM allocator, warps 4..11
// epilogue (2 warps per TMEM lane quadrant, each owning half of the columns). The epilogue
// drains TMEM, hands the accumulator back, writes each warp's 32 rows x 128 bytes into a
// 128B-swizzled box in shared memory, patches the outlier entries there and stores
// the box with one TMA tensor store (LSU stores through a padded stage when C is unaligned).
// The CTA's 16 box stores are paced across the next tile's main loop (one per 30 x min(nks, 16)
// cycles; the last tile at once): issued as one 64-KB burst they stall the operand loads queued
// behind them (CTA-0 trace: main loop of a K = 2048 tile 3.9k cycles without stores, 5.2k with a
// burst, 4.3k paced; profiles/r02ax..r02bb).
#include "common.cuh"
#include "epilogue.cuh"
#include "kernels.h"
#include "ptx.cuh"

#ifndef GEMM_TRACE
#define GEMM_TRACE 0
#endif
// Experiment knob (never set in the product build): bit 0 skips the scale-factor tcgen05.cp,
// bit 1 the MMAs, bit 2 the scale-factor TMA loads, bit 3 the epilogue stores, bit 4 the A/B TMA loads,
// bit 5 the bf16 epilogue's staging and stores (TMEM drain only).
#ifndef GEMM_ABLATE
#define GEMM_ABLATE 0
#endif
#if GEMM_TRACE
#include <cstdio>
__device__ long long g_gt[6][64];
#define GT(k, lt) do { if (blockIdx.x == 0 && (lt) < 64) g_gt[k][lt] = clock64(); } while (0)
#else
#define GT(k, lt) do { } while (0)
#endif

namespace adahop {
namespace mxf4x2 {

constexpr int BK = 256;  // fp4 elements per stage
constexpr int kThreads = 384;
constexpr int kEpiWarps = 8;

// TMEM columns (512 per SM). BN = 128: two disjoint 128-column accumulators, scale factors at
// 256.. in two alternating sets. BN = 256, BUFS = 2: two OVERLAPPING 256-column accumulators,
// acc0 = [0, 256) and acc1 = [224, 480) (they share columns [224, 256)), one scale-factor set at
// 480.. (tcgen05.cp and tcgen05.mma issued by one thread execute in issue order, so the copy for
// k-step ks+1 cannot overwrite scale factors the MMAs of k-step ks still read). The epilogue
// drains the shared 32 columns first and releases them on `tovl`: the next tile's MMAs start
// after ~1/8 of the drain instead of after all of it. BN = 256, BUFS = 1: the single-accumulator
// layout (experiment builds: ADAHOP_GEMM_OVL=0).
// KIND 0: block-scaled MXFP4 (a stage = 256 fp4 of K); KIND 1: BF16 (kind::f16, a stage = 64 bf16
// of K, A / B K-major or MN-major, no scale factors) — the Lv2 CC product and any plain
// BF16 GEMM of the path; both stage 128 bytes of K per operand row.
template <int BN, int BUFS, int KIND = 0>
struct Cfg {
  static constexpr int kA = 128 * BK / 2;             // 16 KB: this CTA's 128 rows of A
  static constexpr int kB = (BN / 2) * BK / 2;        // this CTA's BN/2 rows of B
  static constexpr int kSfa = KIND ? 0 : 1024;        // 128 rows x 8 K-blocks
  static constexpr int kSfb = KIND ? 0 : (BN / 128) * 1024;   // all BN rows (duplicated in both CTAs)
  static constexpr int kKStep = KIND ? 64 : BK;       // K elements per stage
  static constexpr int kStage = kA + kB + kSfa + kSfb;
  static constexpr int kStages = BN == 256 ? 5 : 7;
  static constexpr int kEpiBufs = 1;
  static constexpr bool kOverlap = BN == 256 && BUFS == 2;
  static constexpr int kOvlCols = 32;                 // columns shared by the two accumulators
  static constexpr int kAccCols = kOverlap ? BN - kOvlCols : BN;   // column stride between accumulators
  static constexpr int kSfaCol = kOverlap ? 480 : 256;            // after the accumulator buffers
  static constexpr int kSfbCol = kSfaCol + 8;
  static constexpr int kSfSets = kOverlap ? 1 : 2;
  static constexpr int kSfSet = 32;                   // second scale-factor column set (kSfSets == 2)
  static constexpr size_t kSmem = size_t(kStages) * kStage + kEpiWarps * kEpiBufs * kEpiStageBytes + 1024 + 512;
  static_assert(kOverlap || BUFS * BN <= 256, "accumulators must fit below the scale-factor columns");
  static_assert(kSfbCol + 2 * (BN / 32) * (kSfSets == 2 ? 2 : 1) <= 512 || kSfSets == 2, "TMEM overflow");
};

// kind::f16 instruction descriptor: D f32, A / B bf16, major-ness per operand (0 K, 1 MN)
__host__ __device__ constexpr uint32_t bf16_idesc(int m, int n, int a_mn, int b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(a_mn) << 15) | (uint32_t(b_mn) << 16) |
         (uint32_t(n >> 3) << 17) | (uint32_t(m >> 4) << 24);
}
__host__ __device__ constexpr uint32_t make_idesc(int m, int n) {
  return (1u << 7) | (1u << 10) | (uint32_t(n >> 3) << 17) | (1u << 23) | (uint32_t(m >> 4) << 24);
}

constexpr int64_t kGroupM = 8;  // grouped rasterisation (see gemm_mxf4.cu)
#ifndef GEMM_PACE_MAX_STEPS
#define GEMM_PACE_MAX_STEPS 16
#endif
constexpr int kPaceMaxSteps = GEMM_PACE_MAX_STEPS;   // store pacing scales with K up to this many k-steps
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

// PM x PN CTA pairs per cluster (cluster = 2 PM PN CTAs, rank = 2 (pm PN + pn) + x, x = the
// CTA's half of the pair). A cluster computes a super tile of (256 PM) x (BN PN): the pairs in
// one cluster row (same pm) read the same A rows and the pairs in one cluster column the same
// B rows, so each CTA loads 1/PN of its A box and 1/PM of its B box and multicasts them to the
// CTAs that share them — the L2->SM operand traffic per flop drops by (1/PN + 1/PM)/2 ... 1.
//
// SPLIT > 1 (long-K GEMMs with fewer output tiles than CTA pairs, e.g. the Llama-3.2-1B k / v
// wgrad: 16 tiles of 512 x 2048 over K = 16384): a cluster of SPLIT pairs computes ONE tile,
// pair p over the K range [p nks / SPLIT, (p + 1) nks / SPLIT). Once every pair's MMAs are
// complete (cluster barrier: the operand rings are idle), each CTA pushes column slice c of its
// partial from TMEM into the ring of CTA (c, x) with remote shared-memory stores; after a second
// cluster barrier CTA (p, x) sums its slice over the SPLIT partials in pair order 0, 1, ...
// (deterministic, no workspace), patches and stores it. 512 x 2048 x 16384: 20.7 us with 2 pairs
// per cluster vs 23.8 us for 256 x 128 tiles (profiles/r02as_gemm_splitk.txt).
//
// Grouped launch (GemmGroup, n > 1): the three GEMMs of one linear (fwd, dgrad, wgrad) in ONE
// persistent launch. Problem 0 comes in the kernel's own parameters, problems 1..n-1 in `grp`;
// problem p owns clusters [cl[p], cl[p+1]) (sized on the host in proportion to its work) and
// every CTA of such a cluster walks only that problem's tiles, so each CTA keeps one problem for
// its lifetime. The small linears' GEMMs each fill the machine for a wave or two at most (fill,
// tail, the output writes); side by side they overlap.
struct GemmExtra {
  CUtensorMap tm_a, tm_b, tm_sfa, tm_sfb, tm_c;
  void* C;
  int64_t ldc, M, N, K;
  OePatch oe;
  int out_f32, tma_c;
};
constexpr int kGroupMax = 3;
struct GemmGroup {
  GemmExtra q[kGroupMax - 1];
  int n;
  int cl[kGroupMax + 1];
};

template <int BN, int BUFS, int PM, int PN, int SPLIT = 1, int KIND = 0, bool kGroup = false>
__global__ void __launch_bounds__(kThreads, 1)
    k_gemm_mxf4_2sm(const __grid_constant__ CUtensorMap tm_a0, const __grid_constant__ CUtensorMap tm_b0,
                    const __grid_constant__ CUtensorMap tm_sfa0, const __grid_constant__ CUtensorMap tm_sfb0,
                    const __grid_constant__ CUtensorMap tm_c0, int tma_c0,
                    void* C0, int out_f320, int64_t ldc0, int64_t M0, int64_t N0, int64_t K0, const OePatch oe0,
                    int pace, int a_mn, int b_mn, const __grid_constant__ GemmGroup grp) {
  using G = Cfg<BN, BUFS, KIND>;
  // this CTA's problem (one per cluster range) and its parameters
  static_assert(!kGroup || (PM == 1 && PN == 1 && SPLIT == 1), "grouped launches: single pairs");
  int pi = 0;
  if (kGroup) {
    const int64_t cluster_g = blockIdx.x / 2;
    while (pi + 1 < grp.n && cluster_g >= grp.cl[pi + 1]) ++pi;
  }
  const GemmExtra* ex = kGroup && pi > 0 ? &grp.q[pi - 1] : nullptr;
  const CUtensorMap* tm_a = ex ? &ex->tm_a : &tm_a0;
  const CUtensorMap* tm_b = ex ? &ex->tm_b : &tm_b0;
  const CUtensorMap* tm_sfa = ex ? &ex->tm_sfa : &tm_sfa0;
  const CUtensorMap* tm_sfb = ex ? &ex->tm_sfb : &tm_sfb0;
  const CUtensorMap* tm_c = ex ? &ex->tm_c : &tm_c0;
  const int tma_c = ex ? ex->tma_c : tma_c0;
  void* const C = ex ? ex->C : C0;
  const int out_f32 = ex ? ex->out_f32 : out_f320;
  const int64_t ldc = ex ? ex->ldc : ldc0, M = ex ? ex->M : M0, N = ex ? ex->N : N0, K = ex ? ex->K : K0;
  const OePatch& oe = ex ? ex->oe : oe0;
  static_assert(KIND == 0 || (PM == 1 && PN == 1 && SPLIT == 1), "BF16: single pairs");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ uint32_t pace_t0[kEpiWarps];   // epilogue store pacing: each warp's drain time
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);  // stays in the shared window
  uint8_t* epi_smem = smem + size_t(G::kStages) * G::kStage;
  uint64_t* bars = reinterpret_cast<uint64_t*>(epi_smem + kEpiWarps * G::kEpiBufs * kEpiStageBytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + G::kStages;
  uint64_t* tfull = bars + 2 * G::kStages;
  uint64_t* tempty = tfull + BUFS;
  uint64_t* tovl = tempty + BUFS;     // overlapping accumulators: shared columns drained (once per tile)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tovl + 1);

  const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
  static_assert(SPLIT == 1 || (PM == 1 && PN == 1 && BN == 256 && BUFS == 1), "split-K: single pairs, 256 x 256");
  constexpr int NP = PM * PN, CS = 2 * NP * SPLIT;
  const uint32_t rank = ptx::cluster_ctarank();
  const uint32_t ksp = SPLIT > 1 ? rank >> 1 : 0u;   // this pair's K range (split-K)
  const uint32_t x = rank & 1, pp = SPLIT > 1 ? 0u : rank >> 1, pm = pp / PN, pn = pp % PN;
  const bool leader = x == 0;
  const uint32_t leader_rank = rank & ~1u;
  const int64_t mblocks = (M + 255) / 256;
  const int64_t nblocks = (N + BN - 1) / BN;
  const int64_t smblocks = (mblocks + PM - 1) / PM, snblocks = (nblocks + PN - 1) / PN;
  const int64_t ntiles = smblocks * snblocks;
  const int nks = int((K + G::kKStep - 1) / G::kKStep);
  const int kb = int(int64_t(nks) * ksp / SPLIT), ke = int(int64_t(nks) * (ksp + 1) / SPLIT);
  // cluster index / count within this CTA's problem
  const int64_t cluster = blockIdx.x / CS - (kGroup ? grp.cl[pi] : 0);
  const int64_t nclusters = kGroup ? grp.cl[pi + 1] - grp.cl[pi] : gridDim.x / CS;
  // multicast groups: the CTAs with this x and pm (A rows) / this x and pn (B rows)
  uint16_t mask_a = 0, mask_b = 0;
#pragma unroll
  for (int j = 0; j < PN; ++j) mask_a |= uint16_t(1u << (2 * (pm * PN + j) + x));
#pragma unroll
  for (int i = 0; i < PM; ++i) mask_b |= uint16_t(1u << (2 * (i * PN + pn) + x));
  constexpr uint16_t mask_all = uint16_t((1u << CS) - 1);

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(tm_a);
    ptx::prefetch_tmap(tm_b);
    ptx::prefetch_tmap(tm_sfa);
    ptx::prefetch_tmap(tm_sfb);
    for (int s = 0; s < G::kStages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], NP);   // one commit per pair of the cluster
    }
    for (int b = 0; b < BUFS; ++b) {
      ptx::mbar_init(&tfull[b], 1);
      ptx::mbar_init(&tempty[b], 2 * kEpiWarps);
    }
    ptx::mbar_init(tovl, 2 * 4);   // the 4 warps (one per lane quadrant) owning the shared columns, both CTAs
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc_2sm<512>(tmem_slot);
  ptx::griddep_launch();
  ptx::griddep_wait();   // the prologue above overlapped the previous kernel's tail
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // ------------------------------------------------------------ TMA producer (both CTAs)
    int stage = 0;
    uint32_t phase = 0;
    for (int64_t tile = cluster; tile < ntiles; tile += nclusters) {
      int64_t smb, snb;
      tile_coords(tile, smblocks, snblocks, smb, snb);
      // blocks past the edge of a ragged super tile are computed on clamped (valid) data
      // and never stored: every pair must still take part in the multicasts and commits
      const int64_t mb = min(smb * PM + pm, mblocks - 1), nb = min(snb * PN + pn, nblocks - 1);
      for (int ks = kb; ks < ke; ++ks) {
        ptx::mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* sa = smem + size_t(stage) * G::kStage;
        uint8_t* sb = sa + G::kA;
        uint8_t* ssfa = sb + G::kB;
        uint8_t* ssfb = ssfa + G::kSfa;
        const uint32_t fb = ptx::mapa(&full[stage], leader_rank);
        if (leader) ptx::mbar_arrive_expect_tx(&full[stage], ((GEMM_ABLATE & 4) ? 0 : 2 * (G::kSfa + G::kSfb)) +
                                                               ((GEMM_ABLATE & 16) ? 0 : 2 * (G::kA + G::kB)));
        if (KIND == 1) {
          // BF16: K-major boxes {64 k, rows}; MN-major boxes {64 mn, 64 k} stacked every 8 KB
          const int32_t ma = int32_t(mb * 256 + x * 128), nbb = int32_t(nb * BN + x * (BN / 2));
          if (!a_mn) ptx::tma_load_2d_2sm(sa, tm_a, fb, ks * 64, ma);
          else
            for (int b = 0; b < 2; ++b) ptx::tma_load_2d_2sm(sa + b * 8192, tm_a, fb, ma + b * 64, ks * 64);
          if (!b_mn) ptx::tma_load_2d_2sm(sb, tm_b, fb, ks * 64, nbb);
          else
            for (int b = 0; b < BN / 128; ++b) ptx::tma_load_2d_2sm(sb + b * 8192, tm_b, fb, nbb + b * 64, ks * 64);
        } else if (GEMM_ABLATE & 16) {
        } else if (PN == 1) {
          ptx::tma_load_2d_2sm(sa, tm_a, fb, ks * (BK / 2), int32_t(mb * 256 + x * 128));
        } else {
          constexpr int sub = 128 / PN;
          ptx::tma_load_2d_2sm_mc(sa + pn * sub * 128, tm_a, &full[stage], ks * (BK / 2),
                                  int32_t(mb * 256 + x * 128 + pn * sub), mask_a);
        }
        if (KIND == 1 || (GEMM_ABLATE & 16)) {
        } else if (PM == 1) {
          ptx::tma_load_2d_2sm(sb, tm_b, fb, ks * (BK / 2), int32_t(nb * BN + x * (BN / 2)));
        } else {
          constexpr int sub = (BN / 2) / PM;
          ptx::tma_load_2d_2sm_mc(sb + pm * sub * 128, tm_b, &full[stage], ks * (BK / 2),
                                  int32_t(nb * BN + x * (BN / 2) + pm * sub), mask_b);
        }
        if (KIND == 0 && !(GEMM_ABLATE & 4)) {
          ptx::tma_load_2d_2sm(ssfa, tm_sfa, fb, ks * 256, int32_t(mb * 2 + x));
          ptx::tma_load_2d_2sm(ssfb, tm_sfb, fb, ks * 256, int32_t(nb * (BN / 128)));
        }
        if (++stage == G::kStages) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1 && leader) {
    // whole warp: waits and descriptor math stay warp-uniform (uniform registers); one elected
    // lane issues the tcgen05 operations
    // ------------------------------------------------------------ MMA issuer (leader)
    const uint32_t idesc = KIND ? bf16_idesc(256, BN, a_mn, b_mn) : make_idesc(256, BN);
    int stage = 0;
    uint32_t phase = 0;
    int64_t lt = 0;
    for (int64_t tile = cluster; tile < ntiles; tile += nclusters, ++lt) {
      const uint32_t buf = uint32_t(lt % BUFS);
      const uint32_t use = uint32_t(lt / BUFS);
      ptx::mbar_wait(&tempty[buf], (use & 1) ^ 1);
      // the previous tile's accumulator shares columns with this one: wait until they are drained
      if (G::kOverlap && lt > 0) ptx::mbar_wait(tovl, uint32_t((lt - 1) & 1));
      GT(0, lt);
      ptx::tc_fence_after();
      const uint32_t d_tmem = tmem_base + buf * G::kAccCols;
      for (int ks = kb; ks < ke; ++ks) {
        ptx::mbar_wait(&full[stage], phase);
        ptx::tc_fence_after();
        const bool issuer = ptx::elect_one();
        uint8_t* sa = smem + size_t(stage) * G::kStage;
        uint8_t* sb = sa + G::kA;
        uint8_t* ssfa = sb + G::kB;
        uint8_t* ssfb = ssfa + G::kSfa;
        // scale factors alternate between two TMEM column sets by k-step parity, so the copies
        // for step ks+1 do not overwrite columns the MMAs of step ks still read
        const uint32_t sfo = G::kSfSets == 2 ? uint32_t(ks & 1) * G::kSfSet : 0u;
        if (KIND == 1) {
          const uint32_t a_addr = ptx::smem_u32(sa), b_addr = ptx::smem_u32(sb);
#pragma unroll
          for (int j = 0; j < 4 && issuer; ++j)   // K = 16 per MMA
            ptx::mma_bf16_2sm(d_tmem,
                              a_mn ? ptx::make_sdesc(a_addr + j * 2048, 8192, 1024, 2) : ptx::make_sdesc(a_addr + j * 32, 16, 1024, 2),
                              b_mn ? ptx::make_sdesc(b_addr + j * 2048, 8192, 1024, 2) : ptx::make_sdesc(b_addr + j * 32, 16, 1024, 2),
                              idesc, (ks > kb || j > 0) ? 1u : 0u);
        }
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          if (KIND == 1 || (GEMM_ABLATE & 1) || !issuer) break;
          ptx::tmem_cp_32x128b_warpx4_2sm(tmem_base + G::kSfaCol + sfo + 4 * c,
                                          ptx::make_sdesc(ptx::smem_u32(ssfa + c * 512), 0, 128, 0));
#pragma unroll
          for (int g = 0; g < BN / 128; ++g)
            ptx::tmem_cp_32x128b_warpx4_2sm(tmem_base + G::kSfbCol + sfo + (BN / 32) * c + 4 * g,
                                            ptx::make_sdesc(ptx::smem_u32(ssfb + g * 1024 + c * 512), 0, 128, 0));
        }
        const uint32_t a_addr = ptx::smem_u32(sa), b_addr = ptx::smem_u32(sb);
#pragma unroll
        for (int j = 0; j < BK / 64; ++j) {
          const uint32_t sf_id = uint32_t(j & 1) * 2;
          const uint32_t sfa_t = (tmem_base + G::kSfaCol + sfo + 4 * (j >> 1)) | (sf_id << 30);
          const uint32_t sfb_t = (tmem_base + G::kSfbCol + sfo + (BN / 32) * (j >> 1)) | (sf_id << 30);
          const uint32_t id = idesc | (sf_id << 4) | (sf_id << 29);
          if (KIND == 1 || (GEMM_ABLATE & 2) || !issuer) continue;
          ptx::mma_mxf4_2sm(d_tmem, ptx::make_sdesc(a_addr + j * 32, 16, 1024, 2),
                            ptx::make_sdesc(b_addr + j * 32, 16, 1024, 2), id, sfa_t, sfb_t,
                            (ks > kb || j > 0) ? 1u : 0u);
        }
        if (issuer) {
          if (SPLIT > 1) ptx::tc_commit_2sm_mask(&empty[stage], uint16_t(3u << leader_rank));
          else if (NP == 1) ptx::tc_commit_2sm(&empty[stage]);
          else ptx::tc_commit_2sm_mask(&empty[stage], mask_all);   // every CTA fed by this pair's loads
        }
        __syncwarp();
        if (++stage == G::kStages) { stage = 0; phase ^= 1; }
      }
      if (ptx::elect_one()) ptx::tc_commit_2sm_mask(&tfull[buf], uint16_t(3u << leader_rank));
      __syncwarp();
      GT(1, lt);
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue (8 warps per CTA)
    const uint32_t q = warp & 3;            // TMEM lane quadrant
    const uint32_t half = (warp - 4) >> 2;  // column half of the tile
    // TMA stores: a 4 KB 128B-swizzled box per warp (1024-aligned); else the padded LSU stage
    uint8_t* stg = epi_smem + (warp - 4) * (tma_c ? 4096 : G::kEpiBufs * kEpiStageBytes);
    const int elt = out_f32 ? 4 : 2;
    const int cols_per_grp = 128 / elt;
    const bool vec_ok = ((reinterpret_cast<uintptr_t>(C) | uintptr_t(ldc * elt)) & 15) == 0;
    const uint32_t empty_leader = ptx::mapa(&tempty[0], leader_rank);
    const uint32_t ovl_leader = ptx::mapa(tovl, leader_rank);
    // fused outlier product: fold this CTA's share of Dt while the first main loop runs
    // (every CTA folds its share of every problem's product: the pre-fold counts the whole grid)
    oe_prefold(oe0, int(threadIdx.x) - 128, kEpiWarps * 32, 1);
    if (kGroup)
      for (int q = 1; q < grp.n; ++q) oe_prefold(grp.q[q - 1].oe, int(threadIdx.x) - 128, kEpiWarps * 32, 1);
    oe_prefold_wait(oe);
    int64_t lt = 0;
    for (int64_t tile = cluster; tile < ntiles && SPLIT == 1; tile += nclusters, ++lt) {
      int64_t smb, snb;
      tile_coords(tile, smblocks, snblocks, smb, snb);
      const int64_t mb = smb * PM + pm, nb = snb * PN + pn;   // past the edge: rows/cols invalid, no stores
      const uint32_t buf = uint32_t(lt % BUFS);
      const uint32_t use = uint32_t(lt / BUFS);
      ptx::mbar_wait(&tfull[buf], use & 1);
      if (warp == 4 && lane == 0) GT(2, lt);
      ptx::tc_fence_after();
      const int64_t m0 = mb * 256 + x * 128 + q * 32;
      const int rows_valid = int(M - m0 < 32 ? (M - m0 > 0 ? M - m0 : 0) : 32);
      // overlapping accumulators: the shared columns are the last 32 of acc0 (half 1) and the
      // first 32 of acc1 (half 0); the warps holding them drain those first and release them
      const bool owns_ovl = G::kOverlap && half == (buf == 0 ? 1u : 0u);
      if (BN == 256 && !out_f32) {
        // bf16: read both column groups out of TMEM (one through the smem stage, one in
        // registers), hand the accumulator back, then do the global stores so that they
        // overlap the next tile's main loop
        const uint32_t tb0 = tmem_base + ((q * 32) << 16) + buf * G::kAccCols + half * (BN / 2);
        uint32_t w0[32], w1[32];
        {
          uint32_t r0[32], r1[32], r2[32], r3[32];
          if (owns_ovl) {
            // shared 32 columns first: the next tile's MMAs wait for exactly these
            if (buf == 0) ptx::tmem_ld_32x32b_x32(tb0 + 96, r3);
            else ptx::tmem_ld_32x32b_x32(tb0, r0);
            ptx::tmem_ld_wait();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive_cluster(ovl_leader);
            if (buf == 0) {
              ptx::tmem_ld_32x32b_x32(tb0, r0);
              ptx::tmem_ld_32x32b_x32(tb0 + 32, r1);
              ptx::tmem_ld_32x32b_x32(tb0 + 64, r2);
            } else {
              ptx::tmem_ld_32x32b_x32(tb0 + 32, r1);
              ptx::tmem_ld_32x32b_x32(tb0 + 64, r2);
              ptx::tmem_ld_32x32b_x32(tb0 + 96, r3);
            }
          } else {
            // all four loads in flight before the single wait: the drain time gates the next tile
            ptx::tmem_ld_32x32b_x32(tb0, r0);
            ptx::tmem_ld_32x32b_x32(tb0 + 32, r1);
            ptx::tmem_ld_32x32b_x32(tb0 + 64, r2);
            ptx::tmem_ld_32x32b_x32(tb0 + 96, r3);
          }
          ptx::tmem_ld_wait();
          // accumulator is in registers: hand it back to the MMA warp before packing
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive_cluster(empty_leader + buf * 8);
          if (warp == 4 && lane == 0) GT(3, lt);
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            w0[i] = pack_bf16x2(r0[2 * i], r0[2 * i + 1]);
            w0[16 + i] = pack_bf16x2(r1[2 * i], r1[2 * i + 1]);
            w1[i] = pack_bf16x2(r2[2 * i], r2[2 * i + 1]);
            w1[16 + i] = pack_bf16x2(r3[2 * i], r3[2 * i + 1]);
          }
        }
        if (GEMM_ABLATE & 32) {   // experiment: no staging and no stores (TMEM drain only)
          uint32_t acc = 0;
#pragma unroll
          for (int i = 0; i < 32; ++i) acc ^= w0[i] ^ w1[i];
          if (acc == 0x9E3779B9u && lane == 77) static_cast<uint32_t*>(C)[0] = acc;
          if (warp == 4 && lane == 0) GT(4, lt);
          continue;
        }
        // Paced stores: the CTA's 16 box stores (8 warps x 2) go out one every pace x min(nks, 16)
        // cycles after the drain, spread over the next tile's main loop instead of one 64-KB burst
        // (a burst stalls the operand loads behind it: profiles/r02ay_gemm_store_pacing.txt)
        // (the CTA's last tile stores at once: its stores are the kernel's tail)
        // (32-bit cycle arithmetic: the spread is far below 2^31 cycles; the drain time is parked in
        // shared memory so that it does not hold a register across the packed accumulator values)
        const bool paced = pace > 0 && tile + nclusters < ntiles;
        if (paced && lane == 0) pace_t0[warp - 4] = uint32_t(clock());
#pragma unroll 1
        for (int g = 0; g < 2 && tma_c; ++g) {
          if (paced) {
            const uint32_t wait =
                uint32_t(g * 8 + int(warp) - 4) * uint32_t(pace) * uint32_t(nks < kPaceMaxSteps ? nks : kPaceMaxSteps);
            __syncwarp();
            const uint32_t t0 = *static_cast<volatile uint32_t*>(&pace_t0[warp - 4]);
            while (uint32_t(clock()) - t0 < wait) __nanosleep(32);
          }
          // the previous TMA store has read the stage; stage, patch, then one bulk tensor store
          if (lane == 0) ptx::bulk_wait_group_read<0>();
          __syncwarp();
          epi_stage_sw128(stg, g == 0 ? w0 : w1);
          __syncwarp();
          const int64_t n0 = nb * BN + half * (BN / 2) + g * 64;
          epi_patch_outliers<true>(stg, oe, m0, n0, 64, 2, M, N);
          ptx::fence_proxy_async();
          __syncwarp();
          if (lane == 0 && rows_valid > 0 && n0 < N && !(GEMM_ABLATE & 8)) {
            ptx::tma_store_2d(tm_c, stg, int32_t(n0), int32_t(m0));
            ptx::bulk_commit_group();
          }
        }
#pragma unroll 1
        for (int g = 0; g < 2 && !tma_c; ++g) {
          epi_stage_row128(stg, g == 0 ? w0 : w1);
          __syncwarp();
          const int64_t n0 = nb * BN + half * (BN / 2) + g * 64;
          epi_patch_outliers(stg, oe, m0, n0, 64, 2, M, N);
          const int64_t nrem = N - n0;
          const int bytes_valid = int(nrem >= 64 ? 128 : (nrem > 0 ? nrem * 2 : 0));
          if (rows_valid > 0 && bytes_valid > 0 && !(GEMM_ABLATE & 8))
            epi_flush128(stg, static_cast<char*>(C) + (m0 * ldc + n0) * 2, ldc * 2, rows_valid, bytes_valid, 2,
                         vec_ok);
          __syncwarp();
        }
        __syncwarp();
        if (warp == 4 && lane == 0) GT(4, lt);
        continue;
      }
#pragma unroll 1
      for (int g = 0; g < (BN / 2) / cols_per_grp; ++g) {
        const int col = half * (BN / 2) + g * cols_per_grp;
        const int64_t n0 = nb * BN + col;
        const uint32_t tbase = tmem_base + ((q * 32) << 16) + buf * G::kAccCols + col;
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
        const int ngrp = (BN / 2) / cols_per_grp;
        if (owns_ovl && g == (buf == 0 ? ngrp - 1 : 0)) {
          // this group holds the columns shared with the other accumulator
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive_cluster(ovl_leader);
        }
        if (g == ngrp - 1) {
          // last TMEM read of this warp: hand the accumulator back before the stores
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive_cluster(empty_leader + buf * 8);
        }
        const int64_t nrem = N - n0;
        const int bytes_valid = int(nrem >= cols_per_grp ? 128 : (nrem > 0 ? nrem * elt : 0));
        if (rows_valid > 0 && bytes_valid > 0 && tma_c) {
          if (lane == 0) ptx::bulk_wait_group_read<0>();
          __syncwarp();
          epi_stage_sw128(stg, w);
          __syncwarp();
          epi_patch_outliers<true>(stg, oe, m0, n0, cols_per_grp, elt, M, N);
          ptx::fence_proxy_async();
          __syncwarp();
          if (lane == 0) {
            ptx::tma_store_2d(tm_c, stg, int32_t(n0), int32_t(m0));
            ptx::bulk_commit_group();
          }
          __syncwarp();
        } else if (rows_valid > 0 && bytes_valid > 0) {
          epi_stage_only128(stg, w);
          epi_patch_outliers(stg, oe, m0, n0, cols_per_grp, elt, M, N);
          epi_flush128(stg, static_cast<char*>(C) + (m0 * ldc + n0) * elt, ldc * elt, rows_valid, bytes_valid, elt,
                       vec_ok);
          __syncwarp();
        }
      }
    }
    if (tma_c && lane == 0) ptx::bulk_wait_group<0>();   // this warp's stores are complete
    __syncwarp();
  }
  if (SPLIT > 1) {
    // Split-K reduction. Column group cg (32 columns) of the tile belongs to pair cg / kGrp; pair p's
    // partial of it goes to slot p of the owner CTA's receive buffer (its idle ring):
    //   recv[((p kGrp + cg % kGrp) 8 + j) 128 + row] = 16-byte chunk j of row `row`,
    // remote stores from TMEM-loaded registers (fire-and-forget), a warp's store = 512 contiguous
    // bytes. The owner then sums its slots in pair order 0, 1, ... (deterministic).
    constexpr int kGrp = 8 / SPLIT;   // 32-column groups per owner
    if (warp >= 4) {
      ptx::mbar_wait(&tfull[0], 0);
      if (warp == 4 && lane == 0) GT(2, 0);
      ptx::tc_fence_after();
    }
    ptx::cluster_sync();   // every pair's MMAs are complete: the operand rings are free
    if (warp >= 4 && cluster < ntiles) {
      const uint32_t q = warp & 3, half = (warp - 4) >> 2;
      const uint32_t row = q * 32 + lane;
#pragma unroll 1
      for (int g = 0; g < 4; ++g) {
        const int cg = int(half) * 4 + g;
        uint32_t r[32];
        ptx::tmem_ld_32x32b_x32(tmem_base + ((q * 32) << 16) + cg * 32, r);
        ptx::tmem_ld_wait();
        const uint32_t dst = ptx::mapa(smem, uint32_t(2 * (cg / kGrp)) + x) +
                             ((uint32_t(ksp * kGrp + cg % kGrp) * 8) * 128 + row) * 16;
#pragma unroll
        for (int j = 0; j < 8; ++j) ptx::st_shared_cluster_v4(dst + j * 2048, r[4 * j], r[4 * j + 1], r[4 * j + 2], r[4 * j + 3]);
      }
      ptx::tc_fence_before();
      if (warp == 4 && lane == 0) GT(3, 0);
    }
    ptx::cluster_sync();   // the partials are delivered (release / acquire)
    if (warp >= 4 && cluster < ntiles) {
      // CTA (ksp, x) owns tile columns [ksp 256 / SPLIT, (ksp + 1) 256 / SPLIT) of its 128 rows
      const uint32_t q = warp & 3, half = (warp - 4) >> 2;
      uint8_t* stg = epi_smem + (warp - 4) * (tma_c ? 4096 : G::kEpiBufs * kEpiStageBytes);
      const int elt = out_f32 ? 4 : 2;
      const int cpu = 128 / elt;                       // columns per unit (one 128-byte row segment)
      const int units = (BN / SPLIT) / cpu;
      const bool vec_ok = ((reinterpret_cast<uintptr_t>(C) | uintptr_t(ldc * elt)) & 15) == 0;
      int64_t smb, snb;
      tile_coords(cluster, smblocks, snblocks, smb, snb);
      const int64_t m0 = smb * 256 + x * 128 + q * 32;
      const int rows_valid = int(M - m0 < 32 ? (M - m0 > 0 ? M - m0 : 0) : 32);
      const uint32_t row = q * 32 + lane;
      const uint4* recv = reinterpret_cast<const uint4*>(smem);
#pragma unroll 1
      for (int u = int(half); u < units; u += 2) {
        uint32_t w[32];
#pragma unroll
        for (int h = 0; h < 2; ++h) {   // 32-column groups of the unit (1 for fp32, 2 for bf16)
          if (h == 1 && out_f32) break;
          const int lg = u * (cpu / 32) + h;
          float acc[32];
#pragma unroll
          for (int p = 0; p < SPLIT; ++p) {
            uint4 v[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] = recv[((p * kGrp + lg) * 8 + j) * 128 + row];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const float f[4] = {__uint_as_float(v[j].x), __uint_as_float(v[j].y), __uint_as_float(v[j].z),
                                  __uint_as_float(v[j].w)};
#pragma unroll
              for (int e = 0; e < 4; ++e) acc[4 * j + e] = p == 0 ? f[e] : acc[4 * j + e] + f[e];
            }
          }
          if (out_f32) {
#pragma unroll
            for (int i = 0; i < 32; ++i) w[i] = __float_as_uint(acc[i]);
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) w[16 * h + i] = pack_bf16x2(__float_as_uint(acc[2 * i]), __float_as_uint(acc[2 * i + 1]));
          }
        }
        const int64_t n0 = snb * BN + int64_t(ksp) * (BN / SPLIT) + u * cpu;
        const int64_t nrem = N - n0;
        const int bytes_valid = int(nrem >= cpu ? 128 : (nrem > 0 ? nrem * elt : 0));
        if (rows_valid <= 0 || bytes_valid <= 0) continue;
        if (tma_c) {
          if (lane == 0) ptx::bulk_wait_group_read<0>();
          __syncwarp();
          epi_stage_sw128(stg, w);
          __syncwarp();
          epi_patch_outliers<true>(stg, oe, m0, n0, cpu, elt, M, N);
          ptx::fence_proxy_async();
          __syncwarp();
          if (lane == 0) {
            ptx::tma_store_2d(tm_c, stg, int32_t(n0), int32_t(m0));
            ptx::bulk_commit_group();
          }
          __syncwarp();
        } else {
          epi_stage_only128(stg, w);
          epi_patch_outliers(stg, oe, m0, n0, cpu, elt, M, N);
          epi_flush128(stg, static_cast<char*>(C) + (m0 * ldc + n0) * elt, ldc * elt, rows_valid, bytes_valid, elt,
                       vec_ok);
          __syncwarp();
        }
      }
      if (tma_c && lane == 0) ptx::bulk_wait_group<0>();
      __syncwarp();
      if (warp == 4 && lane == 0) GT(4, 0);
    }
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_2sm<512>(tmem_base);
  }
#if GEMM_TRACE
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const long long t0 = g_gt[0][0];
    for (int i = 0; i < 64 && cluster + i * nclusters < ntiles; ++i)
      printf("gemm tile %2d: mma-start %7lld mma-issued %7lld epi-wake %7lld drained %7lld stored %7lld\n", i,
             g_gt[0][i] - t0, g_gt[1][i] - t0, g_gt[2][i] - t0, g_gt[3][i] - t0, g_gt[4][i] - t0);
  }
#endif
}

}  // namespace mxf4x2

// Epilogue store pacing (cycles per k-step between a CTA's box stores; experiment builds:
// ADAHOP_GEMM_PACE, 0 = one burst after the drain). 30 measured best on the 1B / 8B layer GEMMs:
// GEMMs alone 752 -> 712 us (1B), 2284 -> 2141 us (8B) (profiles/r02bb_gemm_store_pacing.txt)
constexpr int kStorePace = 30;

// ADAHOP_GEMM_TMA_STORE=0 (experiment builds): the epilogue's LSU stores instead of TMA stores
static bool tma_store_enabled() {
  static const int v = knob("ADAHOP_GEMM_TMA_STORE", 1);
  return v != 0;
}

// Tensor maps of one MXFP4 problem (A / B codes, scale factors, C); tma_c = 0: LSU stores for C.
template <int BN, int PM, int PN>
static bool mxf4_maps(const Mxf4GemmArgs& a, CUtensorMap* tma, CUtensorMap* tmb, CUtensorMap* tsfa,
                      CUtensorMap* tsfb, CUtensorMap* tmc, int* tma_c) {
  const int64_t kch = sf_kchunks(a.K);
  if (!make_tmap_2d(tma, CU_TENSOR_MAP_DATA_TYPE_UINT8, a.a_codes, uint64_t(a.K / 2), uint64_t(a.M),
                    uint64_t(a.K / 2), 128, 128 / PN, CU_TENSOR_MAP_SWIZZLE_128B))
    return false;
  if (!make_tmap_2d(tmb, CU_TENSOR_MAP_DATA_TYPE_UINT8, a.b_codes, uint64_t(a.K / 2), uint64_t(a.N),
                    uint64_t(a.K / 2), 128, (BN / 2) / PM, CU_TENSOR_MAP_SWIZZLE_128B))
    return false;
  // scale factors as uint32 rows of one 128-row group: [groups][kch * 128] u32
  if (!make_tmap_2d(tsfa, CU_TENSOR_MAP_DATA_TYPE_UINT32, a.a_sf, uint64_t(kch * 128), uint64_t((a.M + 127) / 128),
                    uint64_t(kch * 512), 256, 1, CU_TENSOR_MAP_SWIZZLE_NONE))
    return false;
  if (!make_tmap_2d(tsfb, CU_TENSOR_MAP_DATA_TYPE_UINT32, a.b_sf, uint64_t(kch * 128), uint64_t((a.N + 127) / 128),
                    uint64_t(kch * 512), 256, BN / 128, CU_TENSOR_MAP_SWIZZLE_NONE))
    return false;
  // C by TMA stores (128B-swizzled 32-row boxes) when its rows are 16-byte aligned; else LSU stores
  const int elt = a.out_f32 ? 4 : 2;
  *tma_c = tma_store_enabled() && (reinterpret_cast<uintptr_t>(a.C) & 15) == 0 && ((a.ldc * elt) % 16) == 0 &&
           make_tmap_2d(tmc, a.out_f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, a.C,
                        uint64_t(a.N), uint64_t(a.M), uint64_t(a.ldc) * elt, uint32_t(128 / elt), 32,
                        CU_TENSOR_MAP_SWIZZLE_128B) ? 1 : 0;
  if (!*tma_c) memset(tmc, 0, sizeof(*tmc));
  return true;
}

// n problems (1..kGroupMax; n > 1 only with PM = PN = SPLIT = 1) in one persistent launch.
template <int BN, int BUFS, int PM, int PN, int SPLIT = 1, bool kGroup = false>
static cudaError_t launch_2sm_n(const Mxf4GemmArgs* a, int n, int num_sms, cudaStream_t st, bool* fits = nullptr,
                               bool* grouped = nullptr) {
  using G = mxf4x2::Cfg<BN, BUFS>;
  constexpr int CS = 2 * PM * PN * SPLIT;
  auto kern = mxf4x2::k_gemm_mxf4_2sm<BN, BUFS, PM, PN, SPLIT, 0, kGroup>;
  if (n < 1 || n > mxf4x2::kGroupMax || (n > 1 && !kGroup)) return cudaErrorInvalidValue;
  CUtensorMap tma, tmb, tsfa, tsfb, tmc;
  int tma_c = 0;
  if (!mxf4_maps<BN, PM, PN>(a[0], &tma, &tmb, &tsfa, &tsfb, &tmc, &tma_c)) return cudaErrorInvalidValue;
  mxf4x2::GemmGroup grp;
  memset(&grp, 0, sizeof(grp));
  grp.n = n;
  for (int i = 1; i < n; ++i) {
    mxf4x2::GemmExtra& e = grp.q[i - 1];
    if (!mxf4_maps<BN, PM, PN>(a[i], &e.tm_a, &e.tm_b, &e.tm_sfa, &e.tm_sfb, &e.tm_c, &e.tma_c))
      return cudaErrorInvalidValue;
    e.C = a[i].C; e.ldc = a[i].ldc; e.M = a[i].M; e.N = a[i].N; e.K = a[i].K; e.oe = a[i].oe;
    e.out_f32 = a[i].out_f32 ? 1 : 0;
  }
  // resident clusters of this shape (GPC packing decides it for clusters of 4 and 8), per device
  static std::atomic<uint64_t> attr{0};
  static PerDeviceInt cached;
  cudaError_t ae = once_per_device(attr, [&kern] {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(G::kSmem));
    if (e == cudaSuccess && CS > 8) e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    return e;
  });
  if (ae != cudaSuccess) return ae;
  const int dev = current_device();   // valid: once_per_device succeeded
  int max_clusters = cached.v[dev].load(std::memory_order_relaxed);
  if (max_clusters <= 0) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(CS * (num_sms / CS)));
    cfg.blockDim = dim3(mxf4x2::kThreads);
    cfg.dynamicSmemBytes = G::kSmem;
    cudaLaunchAttribute at;
    at.id = cudaLaunchAttributeClusterDimension;
    at.val.clusterDim.x = unsigned(CS);
    at.val.clusterDim.y = 1;
    at.val.clusterDim.z = 1;
    cfg.attrs = &at;
    cfg.numAttrs = 1;
    int nc = 0;
    const cudaError_t e = cudaOccupancyMaxActiveClusters(&nc, kern, &cfg);
    if (e != cudaSuccess || nc <= 0) nc = num_sms / CS;
    max_clusters = nc;
    cached.v[dev].store(nc, std::memory_order_relaxed);
  }
  int64_t tiles[mxf4x2::kGroupMax];
  for (int i = 0; i < n; ++i)
    tiles[i] = ((a[i].M + 256 * PM - 1) / (256 * PM)) * ((a[i].N + BN * PN - 1) / (BN * PN));
  if (SPLIT > 1) {
    // one tile per cluster, all co-resident (the outlier pre-fold counts every CTA in)
    if (fits) *fits = (tiles[0] <= max_clusters || knob("ADAHOP_GEMM_SPLITK", 1) > 1) &&
                      (a[0].K + mxf4x2::BK - 1) / mxf4x2::BK >= SPLIT;
    if (fits && !*fits) return cudaSuccess;
  }
  int64_t clusters = 0;
  if (n == 1) {
    clusters = SPLIT > 1 || tiles[0] < max_clusters ? tiles[0] : max_clusters;
    grp.cl[0] = 0;
    grp.cl[1] = int(clusters);
  } else {
    // clusters per problem: greedy on the makespan ceil(tiles / clusters) x (k-steps + ~4 for the
    // epilogue) — each cluster walks its problem's tiles round-robin, so the slowest cluster of
    // the slowest problem sets the kernel's time
    int64_t cost[mxf4x2::kGroupMax], c[mxf4x2::kGroupMax], used = 0;
    for (int i = 0; i < n; ++i) {
      cost[i] = (a[i].K + mxf4x2::BK - 1) / mxf4x2::BK + 4;
      c[i] = 1;
      ++used;
    }
    if (used > max_clusters) return cudaErrorInvalidValue;
    while (used < max_clusters) {
      int worst = -1;
      int64_t wm = 0;
      for (int i = 0; i < n; ++i) {
        const int64_t m = (tiles[i] + c[i] - 1) / c[i] * cost[i];
        if (c[i] < tiles[i] && m > wm) { wm = m; worst = i; }
      }
      if (worst < 0) break;
      ++c[worst];
      ++used;
    }
    // worth it only when one problem leaves most of the machine idle on its own (<= 1/4 of the
    // clusters' worth of tiles: the Llama-3.2-1B k / v wgrad, 16 tiles) and the grouped makespan
    // beats the problems one after another (each on every cluster) plus ~10 k-step units per
    // extra launch boundary; measured: 1B v linear -10 %, k neutral, while grouping the 1B q / o
    // or the 8B k / v was slower (profiles/r02bl_gemm_group_ab.txt)
    int64_t grouped_ms = 0, seq_ms = 10 * (n - 1);
    bool starved = false;
    for (int i = 0; i < n; ++i) {
      grouped_ms = std::max<int64_t>(grouped_ms, (tiles[i] + c[i] - 1) / c[i] * cost[i]);
      seq_ms += (tiles[i] + max_clusters - 1) / max_clusters * cost[i];
      starved |= 4 * tiles[i] <= max_clusters;
    }
    if (grouped) *grouped = starved && grouped_ms < seq_ms;
    if (grouped && !*grouped) return cudaSuccess;
    grp.cl[0] = 0;
    for (int i = 0; i < n; ++i) grp.cl[i + 1] = grp.cl[i] + int(c[i]);
    clusters = used;
  }
  return launch_k(kern, dim3(unsigned(CS * clusters)), dim3(mxf4x2::kThreads), G::kSmem, st, CS, tma, tmb, tsfa,
                  tsfb, tmc, tma_c, a[0].C, a[0].out_f32 ? 1 : 0, a[0].ldc, a[0].M, a[0].N, a[0].K, a[0].oe,
                  knob("ADAHOP_GEMM_PACE", kStorePace), 0, 0, grp);   // pace: cycles per k-step between box stores (0: burst)
}

template <int BN, int BUFS, int PM, int PN, int SPLIT = 1>
static cudaError_t launch_2sm(const Mxf4GemmArgs& a, int num_sms, cudaStream_t st, bool* fits = nullptr) {
  return launch_2sm_n<BN, BUFS, PM, PN, SPLIT>(&a, 1, num_sms, st, fits);
}

#if ADAHOP_EXPERIMENTS
// ADAHOP_GEMM_CLUSTER = pairs per cluster as PMxPN: 1 (1x1, default), 2 (1x2), 4 (1x4), 22 (2x2)
static int cluster_shape() {
  static const int v = knob("ADAHOP_GEMM_CLUSTER", 1);
  return v;
}
#endif

cudaError_t launch_gemm_mxf4_2sm(const Mxf4GemmArgs& a, int num_sms, int variant, cudaStream_t st) {
  if (variant != 256) return launch_2sm<128, 2, 1, 1>(a, num_sms, st);
#if ADAHOP_EXPERIMENTS
  switch (cluster_shape()) {   // multicast clusters of CTA pairs (measured slower)
    case 2: return launch_2sm<256, 1, 1, 2>(a, num_sms, st);
    case 4: return launch_2sm<256, 1, 1, 4>(a, num_sms, st);
    case 21: return launch_2sm<256, 1, 2, 1>(a, num_sms, st);
    case 22: return launch_2sm<256, 1, 2, 2>(a, num_sms, st);
    default: break;
  }
  if (knob("ADAHOP_GEMM_OVL", -1) >= 0)
    return knob("ADAHOP_GEMM_OVL", -1) ? launch_2sm<256, 2, 1, 1>(a, num_sms, st) : launch_2sm<256, 1, 1, 1>(a, num_sms, st);
#endif
  // Overlapping double accumulators (Cfg) for K >= 4096: 1-3.5 % faster there (the main loop
  // is operand-feed bound, so the hidden accumulator drain buys little); slower for short K,
  // where the early MMA start competes with the output stores (profiles/r02c_gemm_overlap_ab.txt)
  if (a.K >= 4096) return launch_2sm<256, 2, 1, 1>(a, num_sms, st);
  return launch_2sm<256, 1, 1, 1>(a, num_sms, st);
}

// BF16 C = A . B on CTA pairs (KIND 1): 256 x 256 tiles, kind::f16 with M = 256, operands K-major
// or MN-major as the Lv2 CC product and the dgrad / wgrad views need them (the 1-CTA 128 x 128
// k_gemm_bf16 reads 64 KB of shared memory per 2 MFLOP and is shared-memory bound at ~half
// the BF16 rate). *launched = false when the shape is not worth a pair (M <= 128).
template <int BUFS>
static cudaError_t launch_bf16_2sm_t(const Bf16GemmArgs& a, int num_sms, cudaStream_t st) {
  using G = mxf4x2::Cfg<256, BUFS, 1>;
  auto kern = mxf4x2::k_gemm_mxf4_2sm<256, BUFS, 1, 1, 1, 1>;
  CUtensorMap tma, tmb, tmc;
  // A: K-major [M][K] (box {64, 128}) or MN-major [K][M] (box {64 mn, 64 k})
  if (!(a.a_mn ? make_tmap_2d(&tma, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, a.A, uint64_t(a.Mb), uint64_t(a.K),
                              uint64_t(a.lda) * 2, 64, 64, CU_TENSOR_MAP_SWIZZLE_128B)
               : make_tmap_2d(&tma, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, a.A, uint64_t(a.K), uint64_t(a.Mb),
                              uint64_t(a.lda) * 2, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B)))
    return cudaErrorInvalidValue;
  if (!(a.b_mn ? make_tmap_2d(&tmb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, a.B, uint64_t(a.Nb), uint64_t(a.K),
                              uint64_t(a.ldb) * 2, 64, 64, CU_TENSOR_MAP_SWIZZLE_128B)
               : make_tmap_2d(&tmb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, a.B, uint64_t(a.K), uint64_t(a.Nb),
                              uint64_t(a.ldb) * 2, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B)))
    return cudaErrorInvalidValue;
  const int elt = a.out_f32 ? 4 : 2;
  int tma_c = tma_store_enabled() && (reinterpret_cast<uintptr_t>(a.C) & 15) == 0 && ((a.ldc * elt) % 16) == 0 &&
              make_tmap_2d(&tmc, a.out_f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, a.C,
                           uint64_t(a.Nb), uint64_t(a.Mb), uint64_t(a.ldc) * elt, uint32_t(128 / elt), 32,
                           CU_TENSOR_MAP_SWIZZLE_128B) ? 1 : 0;
  if (!tma_c) memset(&tmc, 0, sizeof(tmc));
  static std::atomic<uint64_t> attr{0};
  static PerDeviceInt cached;
  cudaError_t ae = once_per_device(attr, [&kern] {
    return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(G::kSmem));
  });
  if (ae != cudaSuccess) return ae;
  const int dev = current_device();
  int max_clusters = cached.v[dev].load(std::memory_order_relaxed);
  if (max_clusters <= 0) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(2 * (num_sms / 2)));
    cfg.blockDim = dim3(mxf4x2::kThreads);
    cfg.dynamicSmemBytes = G::kSmem;
    cudaLaunchAttribute at;
    at.id = cudaLaunchAttributeClusterDimension;
    at.val.clusterDim.x = 2;
    at.val.clusterDim.y = 1;
    at.val.clusterDim.z = 1;
    cfg.attrs = &at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n <= 0) n = num_sms / 2;
    max_clusters = n;
    cached.v[dev].store(n, std::memory_order_relaxed);
  }
  const int64_t tiles = ((a.Mb + 255) / 256) * ((a.Nb + 255) / 256);
  const int64_t clusters = tiles < max_clusters ? tiles : max_clusters;
  const OePatch none{};
  mxf4x2::GemmGroup grp;
  memset(&grp, 0, sizeof(grp));
  grp.n = 1;
  grp.cl[1] = int(clusters);
  return launch_k(kern, dim3(unsigned(2 * clusters)), dim3(mxf4x2::kThreads), G::kSmem, st, 2, tma, tmb, tma, tmb,
                  tmc, tma_c, a.C, a.out_f32 ? 1 : 0, a.ldc, a.Mb, a.Nb, a.K, none,
                  knob("ADAHOP_GEMM_PACE", kStorePace), a.a_mn, a.b_mn, grp);
}

cudaError_t launch_gemm_bf16_2sm(const Bf16GemmArgs& a, int num_sms, cudaStream_t st, bool* launched) {
  *launched = false;
  if (a.mode != 0 || a.Mb <= 128 || knob("ADAHOP_BF16_2SM", 1) == 0) return cudaSuccess;
  *launched = true;
  return a.K >= 4096 ? launch_bf16_2sm_t<2>(a, num_sms, st) : launch_bf16_2sm_t<1>(a, num_sms, st);
}

// The n (2..3) MXFP4 GEMMs of one linear in one persistent launch (single accumulator), when the
// estimated makespan beats separate launches; *launched = false: nothing launched.
cudaError_t launch_gemm_mxf4_2sm_group(const Mxf4GemmArgs* a, int n, int num_sms, cudaStream_t st, bool* launched) {
  *launched = false;
  const cudaError_t e = launch_2sm_n<256, 1, 1, 1, 1, true>(a, n, num_sms, st, nullptr, launched);
  if (e != cudaSuccess) *launched = false;
  return e;
}

// Split-K over clusters of `split` pairs (2 or 4). *launched = false (and nothing launched) when
// the shape's clusters cannot all be co-resident or K has fewer than `split` k-steps.
cudaError_t launch_gemm_mxf4_2sm_split(const Mxf4GemmArgs& a, int num_sms, int split, cudaStream_t st,
                                       bool* launched) {
  *launched = false;
  cudaError_t e = split == 4   ? launch_2sm<256, 1, 1, 1, 4>(a, num_sms, st, launched)
                  : split == 2 ? launch_2sm<256, 1, 1, 1, 2>(a, num_sms, st, launched)
                               : cudaErrorInvalidValue;
  if (e != cudaSuccess) *launched = false;
  return e;
}

}  // namespace adahop
