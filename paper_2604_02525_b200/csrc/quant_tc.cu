// quant_tc.cu — IHT + MXFP4 quantisation with the Hadamard contraction on the tensor cores.
//
// The inner Hadamard transform is the dense contraction A·H_k of eq:inner_hadamard,
// blockwise with H_32. The scalar butterfly version spends ~12 instructions per
// element and is issue-bound well below HBM bandwidth; here each 32-block is multiplied by
// the +-1 Sylvester matrix with tcgen05.mma.kind::f16 (bf16 inputs are exact, the +-x
// products are exact, the 32-term sums accumulate in fp32), and the epilogue warps only
// scale by RN32(1/sqrt 32), take the block amax, and convert to E2M1/E8M0.
// Bit-exactness contract: codes and scales equal the OCP quantiser applied to the fp32
// Hadamard output this kernel produces (SURVEY c19 protocol (a)); that output is within
// 1e-6 relative of the exact transform (R2).
//
// One pass over a bf16 tensor T [R x C] can emit
//   the row quantisation    (stored rows = the R rows,    K = C)  — kRow,
//   the column quantisation (stored rows = the C columns, K = R)  — kCol,
// each with its own OE mask (extracted rows / columns become zero blocks: codes 0, scale
// 0x7F) and raw bf16 slice. Tiles of 128 x 128 arrive by TMA (two 128B-swizzled 64-column
// boxes, issued by two producer lanes) in a 4-stage ring. Per tile the MMA warp issues, per
// 32-block, M=128 x N=32 x K=32:
//   row blocks: A = the tile's 32-column slice, K-major;
//   column blocks: A = the transposed 32-row slice, MN-major (the same smem bytes);
// B = H_32 (K-major, in smem). Accumulators (double-buffered, 2 x 256 TMEM columns) are
// drained by 16 epilogue warps: 8 for row blocks (TMEM lane = tile row), 8 for column blocks
// (TMEM lane = tile column). With the fused wgrad outlier product (kOr, see "Fused outlier
// product" below) the ring is 3 stages deep, the Hadamard accumulator single-buffered and the
// product accumulators occupy TMEM columns [256 + 64 i, 256 + 64 i + npad) (up to two products
// per launch: the wgrad's on G_Y's or X's tiles, the dgrad OE-Left's on W's).
#include "common.cuh"
#include "kernels.h"
#include "ptx.cuh"

// Experiment knob (never set in the product build): bit 0 skips the MMAs, bit 1 the
// epilogue TMEM loads + quantisation, bit 2 the code TMA stores, bit 3 the scale stores.
#ifndef QTC_ABLATE
#define QTC_ABLATE 0
#endif

// The tile's two TMA boxes are issued from two lanes of the producer warp: one issuing thread caps
// a CTA's L2/HBM -> SM delivery near 27 B/clk, two lanes reach 34 (profiles/r02aa_tma_lanes.txt);
// the layer step is ~1 % faster. QTC_PROD_LANES=1 restores the single issuing thread.
#ifndef QTC_PROD_LANES
#define QTC_PROD_LANES 2
#endif

// Experiment knob: QTC_TRACE=1 records per-tile timestamps of CTA 0 and prints them.
#ifndef QTC_TRACE
#define QTC_TRACE 0
#endif
#if QTC_TRACE
#include <cstdio>
__device__ long long g_qtc_trace[6][64];
#define QTC_T(k, lt) do { if (blockIdx.x == 0 && (lt) < 64) g_qtc_trace[k][lt] = clock64(); } while (0)
#else
#define QTC_T(k, lt) do { } while (0)
#endif

namespace adahop {
namespace qtc {

constexpr int kBox = 16384;           // 128 rows x 128 bytes (64 bf16 columns)
constexpr int kTile = 2 * kBox;       // 128 x 128 bf16
// Ring depth and stage size: the fused outlier product (kOr) adds the tile's slice rows (two
// boxes of 64 rows x npad <= 64 slice rows) to every stage and runs 3 stages deep.
constexpr int kOrMaxN = 64;
constexpr int kOrBytes = 2 * kOrMaxN * 128;
template <bool kOr> struct Ring {
  static constexpr int kStages = kOr ? 3 : 4;
  static constexpr int kStage = kTile + (kOr ? kOrBytes : 0);
};
constexpr int kEpiGroups = 4;         // epilogue groups of 4 warps (one warp per TMEM lane quarter)
constexpr int kThreads = 128 + kEpiGroups * 128;   // warps 0..3 control, 4..19 epilogue
constexpr int kHBytes = 32 * 32 * 2;  // H_32 in the canonical no-swizzle K-major layout
constexpr int kStg = 128 * 64;        // one tile's codes of one orientation: 128 stored rows x 64 bytes

// The OE rows / columns of one (job, orientation): the sorted index list (k <= 256) and a
// membership bitmap over the operand's stored rows, both staged in shared memory (the bitmap is
// sized per launch: ceil(rows / 32) words; a per-row binary search instead made the quant stage
// 9 % slower, profiles/r02k_mask_ab.txt).
constexpr int64_t kMaskMaxRows = kFoidMaxRows;   // the OE index sets come from FOID
struct Mask {
  int32_t idx[256];
};
__device__ __forceinline__ void mask_build(Mask* m, uint32_t* bits, const int32_t* __restrict__ idx, int n,
                                           int64_t rows) {
  const int words = int((rows + 31) / 32);
  for (int i = threadIdx.x; i < words; i += blockDim.x) bits[i] = 0u;
  for (int i = threadIdx.x; i < n; i += blockDim.x) m->idx[i] = idx[i];
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) atomicOr(&bits[idx[i] >> 5], 1u << (idx[i] & 31));
  __syncthreads();
}
// first position in the sorted list idx[0, n) whose value is >= v
__device__ __forceinline__ int lower_bound_idx(const int32_t* idx, int n, int v) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (idx[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}
__device__ __forceinline__ int mask_slot(const Mask* m, int n, int64_t r) {
  int lo = 0, hi = n - 1;
  while (lo <= hi) {
    const int mid = (lo + hi) >> 1;
    const int x = m->idx[mid];
    if (x == r) return mid;
    if (x < r) lo = mid + 1; else hi = mid - 1;
  }
  return -1;
}

struct Out {
  uint8_t* q; uint8_t* sf; const int32_t* zero; int nzero; __nv_bfloat16* slice; float* had;
  int bits_off;   // first word of this mask's bitmap in the shared bitmap region
};

// kind::f16 instruction descriptor: D f32, A/B bf16, M = 128, N = 32, A major selectable.
__host__ __device__ constexpr uint32_t idesc_h(int a_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(a_mn) << 15) | (uint32_t(32 >> 3) << 17) |
         (uint32_t(128 >> 4) << 24);
}

__device__ __forceinline__ float inv_sqrt32() { return __uint_as_float(0x3E3504F3u); }

__device__ __forceinline__ uint32_t e2m1x8(const float* v) {
  uint32_t out;
  asm("{\n\t.reg .b8 b0, b1, b2, b3;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b0, %2, %1;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b1, %4, %3;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b2, %6, %5;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b3, %8, %7;\n\t"
      "mov.b32 %0, {b0, b1, b2, b3};\n\t}"
      : "=r"(out)
      : "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]));
  return out;
}

// Quantise one 32-block from its unnormalised Hadamard sums d[32] (fp32 accumulator).
// y = RN(d c); e = floor(log2 max|y|) - 2 (clamped, 0 for a zero block); codes = E2M1(y 2^-e).
template <bool kHad>
__device__ __forceinline__ void quant_block(const uint32_t (&d)[32], uint4& codes, uint32_t& sbyte, float* y_out) {
  const float c = inv_sqrt32();
  // max |d| as a depth-4 tree of 3-input maxima (FMNMX3) instead of a 32-long chain
  float m[11];
#pragma unroll
  for (int i = 0; i < 10; ++i)
    m[i] = fmaxf(fmaxf(fabsf(__uint_as_float(d[3 * i])), fabsf(__uint_as_float(d[3 * i + 1]))),
                 fabsf(__uint_as_float(d[3 * i + 2])));
  m[10] = fmaxf(fabsf(__uint_as_float(d[30])), fabsf(__uint_as_float(d[31])));
  const float amax = fmaxf(fmaxf(fmaxf(fmaxf(m[0], m[1]), m[2]), fmaxf(fmaxf(m[3], m[4]), m[5])),
                           fmaxf(fmaxf(fmaxf(m[6], m[7]), m[8]), fmaxf(m[9], m[10])));
  const float amax_y = __fmul_rn(amax, c);
  const uint32_t bits = __float_as_uint(amax_y);
  int e;
  if (amax_y == 0.f) e = 0;
  else if ((bits >> 23) != 0) e = int(bits >> 23) - 127 - 2;
  else e = (31 - __clz(int(bits))) - 149 - 2;
  e = max(-127, min(127, e));
  sbyte = uint32_t(e + 127);
  float v[32];
  if (kHad || e > 120 || e < -100) {
    const float s = __uint_as_float(uint32_t(127 - e) << 23);
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const float y = __fmul_rn(__uint_as_float(d[i]), c);
      if (kHad) y_out[i] = y;
      v[i] = __fmul_rn(y, s);
    }
  } else {
    // fused c * 2^-e (exact: no subnormal / overflow in this exponent range), packed FMUL2
    const uint32_t cs = __float_as_uint(__fmul_rn(c, __uint_as_float(uint32_t(127 - e) << 23)));
    const uint64_t cs2 = (uint64_t(cs) << 32) | cs;
#pragma unroll
    for (int i = 0; i < 32; i += 2) {
      uint64_t p;
      asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(p) : "l"((uint64_t(d[i + 1]) << 32) | d[i]), "l"(cs2));
      v[i] = __uint_as_float(uint32_t(p));
      v[i + 1] = __uint_as_float(uint32_t(p >> 32));
    }
  }
  codes = make_uint4(e2m1x8(v), e2m1x8(v + 8), e2m1x8(v + 16), e2m1x8(v + 24));
}

// Several tensors in one persistent launch. The "plain" jobs' tiles form one global index (job 0's
// tiles, then job 1's, ...) that CTA b visits with stride gridDim.x, row bands first (ct fastest):
// concurrent CTAs stream whole row bands, so the bf16 reads are long contiguous runs.
//
// Fused outlier product of the wgrad (eq:oe_right P:280 with A = G_Y^T, B_out = X[:, S]: T = G_Y,
// S = X's column slice; eq:oe_left P:273 with A_out = G_Y[:, S]^T, B = X: T = X, S = G_Y's):
//   P[c][j] = sum_r T[r][c] * S[j][r]     (T = the streamed tensor [R x C], S = the slice [kk][R])
// The last job of the launch may carry it (Jobs::orr). Its tiles are visited after the plain ones,
// column band by column band (rt fastest), in contiguous chunks: OR-chunk b (of min(n, SMs)) goes
// to CTA b, so a CTA accumulates a band's product across consecutive token tiles in TMEM (one
// tcgen05.mma kind::f16 per 16 rows, A = the staged tile read MN-major, B = the TMA-loaded slice
// rows) and writes one partial per (band, CTA) segment; k_or_fold sums a band's partials in CTA
// order (deterministic) into Dt[j][c] for the MXFP4 GEMM epilogue (eq:oe_right's "+ A B_out").
constexpr int kMaxJobs = 3;
struct Job {
  int64_t R, C;
  int ctiles, tile0;
  int64_t kch_row, kch_col;
  Out orow, ocol;
};
struct OrSpec {
  int on;          // 1: the last job carries the outlier product
  int npad, kk;    // MMA N (kk rounded up to 16, <= kOrMaxN) and slice rows
  int n, rtiles;   // OR tiles (= rtiles x ctiles of the job) and row tiles per column band
  int chunks;      // min(n, SMs): OR-chunk b = tiles [b n / chunks, (b + 1) n / chunks)
  int spb;         // partial slots per band
  float* part;     // [ctiles][spb][npad][128] fp32
  unsigned* ticket;   // zeroed here; the MXFP4 GEMM's pre-fold counts its CTAs on it
  int dry;            // experiment builds (ADAHOP_OR_FUSED=3): the OR tile order without the product
};
constexpr int kMaxOr = 2;   // fused products per launch (the wgrad's and the dgrad OE-Left's)
struct Jobs {
  CUtensorMap tm[kMaxJobs], tqr[kMaxJobs], tqc[kMaxJobs], tor[kMaxOr];
  Job j[kMaxJobs];
  int n, ntiles;   // jobs; plain tiles (every job but the OR jobs)
  int nor;         // OR jobs: the last nor jobs of the launch, job n - nor + i carries orr[i]
  OrSpec orr[kMaxOr];
};
struct TileRef {
  int jb, rt, ct;
  bool orr, first, last;   // an OR tile; first / last tile of its (band, CTA) segment
  int oi;                  // its product (Jobs::orr index)
};
__device__ __forceinline__ int or_chunk_lo(const OrSpec& o, int b) { return int((int64_t(b) * o.n) / o.chunks); }
// This CTA's tile sequence (the same in every role): plain tiles b, b + G, ... then its OR chunk.
struct TileCursor {
  int g, u, uend;   // next plain tile; next / end OR tile of product oi
  int lo;           // first OR tile of the chunk
  int oi;           // product whose chunk is being walked
  __device__ __forceinline__ void start(const Jobs& J) {
    u = uend = lo = 0;
    if (oi < J.nor && J.orr[oi].on && int(blockIdx.x) < J.orr[oi].chunks) {
      lo = u = or_chunk_lo(J.orr[oi], int(blockIdx.x));
      uend = or_chunk_lo(J.orr[oi], int(blockIdx.x) + 1);
    }
  }
  __device__ __forceinline__ explicit TileCursor(const Jobs& J) {
    g = int(blockIdx.x);
    oi = 0;
    start(J);
  }
  __device__ __forceinline__ bool next(const Jobs& J, TileRef& t) {
    if (g < J.ntiles) {
      const int nplain = J.n - J.nor;
      int jb = 0;
      while (jb + 1 < nplain && g >= J.j[jb + 1].tile0) ++jb;
      const int lt0 = g - J.j[jb].tile0, ctiles = J.j[jb].ctiles;
      t = TileRef{jb, lt0 / ctiles, lt0 % ctiles, false, false, false, 0};
      g += int(gridDim.x);
      return true;
    }
    while (u >= uend) {   // this product's chunk is done: the next product's
      if (++oi >= J.nor) return false;
      start(J);
    }
    const OrSpec& o = J.orr[oi];
    const int rt = u % o.rtiles;
    t = TileRef{J.n - J.nor + oi, rt, u / o.rtiles, true, u == lo || rt == 0, u + 1 == uend || rt == o.rtiles - 1, oi};
    ++u;
    return true;
  }
};
// OR-chunk holding OR tile u: the largest b with lo(b) <= u
__device__ __forceinline__ int or_chunk_of(const OrSpec& o, int u) {
  return int(((int64_t(u) + 1) * o.chunks - 1) / o.n);
}

// kind::f16 instruction descriptor of the outlier product: M = 128 (tile columns, A MN-major),
// N = npad (slice rows, B K-major), D f32.
__host__ __device__ constexpr uint32_t idesc_or(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (uint32_t(n >> 3) << 17) | (uint32_t(128 >> 4) << 24);
}

template <bool kRow, bool kCol, bool kHad, bool kOr>
__global__ void __launch_bounds__(kThreads, 1) k_quant_tc(const __grid_constant__ Jobs J) {
  using RG = Ring<kOr>;
  constexpr int kStages = RG::kStages;
  // TMEM: the Hadamard accumulators double-buffered (2 x 256 columns); with the fused outlier
  // product single-buffered at [0, 256) and the product's accumulator at [256, 256 + npad)
  constexpr int kTBufs = kOr ? 1 : 2;
  constexpr uint32_t kOrCol = 256;
  extern __shared__ __align__(1024) uint8_t smem_q[];
  uint8_t* ring = smem_q + ((1024u - (ptx::smem_u32(smem_q) & 1023u)) & 1023u);
  uint8_t* stg = ring + kStages * RG::kStage;   // codes [orientation][buffer][128 rows x 64 B], 64B-swizzled
  uint8_t* sfstg = stg + 4 * kStg;         // scales [orientation][buffer][512 B] = one SF chunk each
  uint8_t* hmat = sfstg + 4 * 512;
  uint64_t* full = reinterpret_cast<uint64_t*>(hmat + kHBytes);
  uint64_t* empty = full + 4;
  uint64_t* tfull = empty + 4;         // [2]
  uint64_t* tempty = tfull + 2;        // [2]
  uint64_t* staged = tempty + 2;       // [2] epilogue warps -> store warp
  uint64_t* stgfree = staged + 2;      // [2] store warp -> epilogue warps
  uint64_t* orfull = stgfree + 2;      // [kMaxOr] MMA -> flush warps: a segment's product is complete
  uint64_t* orempty = orfull + kMaxOr; // [kMaxOr] flush warps -> MMA: the product accumulator is drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(orempty + kMaxOr);
  Mask* masks = reinterpret_cast<Mask*>(reinterpret_cast<uint8_t*>(tmem_slot) + 16);   // [job][row, col]
  uint32_t* mbits = reinterpret_cast<uint32_t*>(masks + 2 * kMaxJobs);               // bitmaps (Out::bits_off)
  const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
  constexpr int kEpiWarps = kEpiGroups * 4;

  // ---- setup: barriers, H_32, TMEM, OE masks
  if (warp == 0 && lane == 0) {
    for (int jb = 0; jb < J.n; ++jb) {
      ptx::prefetch_tmap(&J.tm[jb]);
      if (kRow) ptx::prefetch_tmap(&J.tqr[jb]);
      if (kCol) ptx::prefetch_tmap(&J.tqc[jb]);
    }
    if (kOr)
      for (int o = 0; o < J.nor; ++o) ptx::prefetch_tmap(&J.tor[o]);
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 2);   // MMA commit + OE-slice gather warp
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&tfull[b], 1);
      ptx::mbar_init(&tempty[b], kEpiWarps);
      ptx::mbar_init(&staged[b], kEpiWarps);
      ptx::mbar_init(&stgfree[b], 1);
    }
    for (int o = 0; o < kMaxOr; ++o) {
      ptx::mbar_init(&orfull[o], 1);
      ptx::mbar_init(&orempty[o], 4);   // the four warps of epilogue group 0
    }
    ptx::fence_barrier_init();
  }
  // H (n = j rows, k = i): core matrices of 8 rows x 16 bytes, (n/8, k/8) -> ((n/8)*4 + k/8)*128
  for (int e = threadIdx.x; e < 32 * 32; e += blockDim.x) {
    const int n = e >> 5, k = e & 31;
    const bool neg = __popc(n & k) & 1;
    *reinterpret_cast<__nv_bfloat16*>(hmat + ((n >> 3) * 4 + (k >> 3)) * 128 + (n & 7) * 16 + (k & 7) * 2) =
        __float2bfloat16_rn(neg ? -1.f : 1.f);
  }
  if (warp == 2) ptx::tmem_alloc<512>(tmem_slot);
  ptx::griddep_launch();
  ptx::griddep_wait();   // the prologue above overlapped the previous kernel's tail
  for (int jb = 0; jb < J.n; ++jb) {
    if (kRow && J.j[jb].orow.nzero > 0)
      mask_build(&masks[2 * jb], mbits + J.j[jb].orow.bits_off, J.j[jb].orow.zero, J.j[jb].orow.nzero, J.j[jb].R);
    if (kCol && J.j[jb].ocol.nzero > 0)
      mask_build(&masks[2 * jb + 1], mbits + J.j[jb].ocol.bits_off, J.j[jb].ocol.zero, J.j[jb].ocol.nzero, J.j[jb].C);
  }
  // the previous user of the ticket (an earlier GEMM) has completed: griddep_wait above
  if (kOr && blockIdx.x == 0 && threadIdx.x == 0)
    for (int o = 0; o < J.nor; ++o)
      if (J.orr[o].on) *J.orr[o].ticket = 0u;
  ptx::fence_proxy_async();  // H written by threads, read by the tensor core
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0 && lane < uint32_t(QTC_PROD_LANES)) {
    // ------------------------------------------------------------ TMA producer
    int stage = 0;
    uint32_t phase = 0;
    TileRef t;
    TileCursor cur(J);
    for (int i = 0; cur.next(J, t); ++i) {
      ptx::mbar_wait(&empty[stage], phase ^ 1);
      QTC_T(0, i);
      uint8_t* dst = ring + stage * RG::kStage;
      const bool o = kOr && t.orr && !J.orr[t.oi].dry;
      const int npad = o ? J.orr[t.oi].npad : 0;
      if (lane == 0) ptx::mbar_arrive_expect_tx(&full[stage], kTile + (o ? 2 * npad * 128 : 0));
      if (QTC_PROD_LANES == 1 || lane == 0)
        ptx::tma_load_2d(dst, &J.tm[t.jb], &full[stage], int32_t(t.ct * 128), int32_t(t.rt * 128));
      if (QTC_PROD_LANES == 1 || lane == 1)
        ptx::tma_load_2d(dst + kBox, &J.tm[t.jb], &full[stage], int32_t(t.ct * 128 + 64), int32_t(t.rt * 128));
      if (o && lane == 0) {
        // the slice rows S[0, npad) x tile rows [128 rt, +128) as two 64-row K boxes (rows >= kk: zeros)
        ptx::tma_load_2d(dst + kTile, &J.tor[t.oi], &full[stage], int32_t(t.rt * 128), 0);
        ptx::tma_load_2d(dst + kTile + npad * 128, &J.tor[t.oi], &full[stage], int32_t(t.rt * 128 + 64), 0);
      }
      if (++stage == kStages) { stage = 0; phase ^= 1; }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (whole warp, one elected lane
    // issues; descriptors stay warp-uniform so they live in uniform registers)
    const uint64_t bdesc = ptx::make_sdesc(ptx::smem_u32(hmat), 128, 512, 0);
    int stage = 0;
    uint32_t phase = 0;
    int segs[kMaxOr] = {0, 0};   // completed outlier-product segments per product
    TileRef t;
    TileCursor cur(J);
    for (int lt = 0; cur.next(J, t); ++lt) {
      const uint32_t buf = kTBufs == 2 ? uint32_t(lt & 1) : 0u;
      const uint32_t use = kTBufs == 2 ? uint32_t(lt >> 1) : uint32_t(lt);
      ptx::mbar_wait(&tempty[buf], (use & 1) ^ 1);
      QTC_T(1, lt);
      ptx::mbar_wait(&full[stage], phase);
      QTC_T(2, lt);
      const bool o = kOr && t.orr && !J.orr[t.oi].dry;
      const int npad = o ? J.orr[t.oi].npad : 0;
      const int sg = o ? segs[t.oi] : 0;
      // a new segment reuses its product's accumulator once the previous segment is flushed
      if (o && t.first && sg > 0) ptx::mbar_wait(&orempty[t.oi], uint32_t((sg - 1) & 1));
      ptx::tc_fence_after();
      const uint32_t base = ptx::smem_u32(ring + stage * RG::kStage);
      const uint32_t d0 = tmem_base + buf * 256;
      // start-address field = bits [0,14) of the descriptor in 16-byte units: offsets add directly
      const uint64_t arow = ptx::make_sdesc(base, 16, 1024, 2);     // K-major (row blocks)
      const uint64_t acol = ptx::make_sdesc(base, kBox, 1024, 2);   // MN-major (column blocks)
      if (ptx::elect_one()) {
        if (!(QTC_ABLATE & 1)) {
#pragma unroll
          for (int b = 0; b < 4; ++b) {
#pragma unroll
            for (int s = 0; s < 2; ++s) {   // K = 32 as two K = 16 steps
              // row blocks: rows of the tile x columns [32 b + 16 s, +16): box b/2, byte 64 (b%2) + 32 s
              if (kRow)
                ptx::mma_bf16(d0 + b * 32, arow + uint64_t(((b >> 1) * kBox + (b & 1) * 64 + s * 32) >> 4),
                              bdesc + uint64_t(s * 16), idesc_h(0), s);
              // column blocks: columns of the tile x rows [32 b + 16 s, +16): MN-major, two 64-column atoms
              if (kCol)
                ptx::mma_bf16(d0 + 128 + b * 32, acol + uint64_t(((b * 32 + s * 16) * 128) >> 4),
                              bdesc + uint64_t(s * 16), idesc_h(1), s);
            }
          }
        }
        // the epilogue waits only for the Hadamard MMAs; the stage waits for the product's too
        ptx::tc_commit(&tfull[buf]);
        if (o) {
          // P[c][j] += sum over the tile's 128 rows r of T[r][c] S[j][r]: eight K = 16 steps; A = the
          // tile MN-major (as the column blocks), B = the slice boxes K-major (128B swizzle)
          const uint64_t bor = ptx::make_sdesc(base + kTile, 16, 1024, 2);
#pragma unroll
          for (int k = 0; k < 8; ++k)
            ptx::mma_bf16(tmem_base + kOrCol + kOrMaxN * t.oi, acol + uint64_t((k * 16 * 128) >> 4),
                          bor + uint64_t(((k >> 2) * npad * 128 + (k & 3) * 32) >> 4), idesc_or(npad),
                          (t.first && k == 0) ? 0u : 1u);
        }
        ptx::tc_commit(&empty[stage]);
        if (o && t.last) ptx::tc_commit(&orfull[t.oi]);
      }
      __syncwarp();
      if (o && t.last) ++segs[t.oi];
      if (++stage == kStages) { stage = 0; phase ^= 1; }
    }
  } else if (warp == 3) {
    // ------------------------------------------------------------ OE-slice gather warp
    // Copies the extracted rows / columns of T that fall in this tile from the staged tile
    // (128B-swizzled boxes) into the raw bf16 slices, then releases the stage together with
    // the MMA commit. out_row[s][c] = T[idx[s], c], out_col[s][r] = T[r, idx[s]].
    int stage = 0;
    uint32_t phase = 0;
    TileRef t;
    TileCursor cur(J);
    for (int i = 0; cur.next(J, t); ++i) {
      const Job& jj = J.j[t.jb];
      const int rt = t.rt, ct = t.ct;
      ptx::mbar_wait(&full[stage], phase);
      const uint8_t* base = ring + stage * RG::kStage;
      if (kCol && jj.ocol.slice != nullptr && jj.ocol.nzero > 0) {
        const Mask* m = &masks[2 * t.jb + 1];
        const int n = jj.ocol.nzero;
        int j = lower_bound_idx(m->idx, n, ct * 128);
        const int j1 = lower_bound_idx(m->idx, n, ct * 128 + 128);
        for (; j < j1; ++j) {
          const int c = m->idx[j] - ct * 128, box = c >> 6, cc = c & 63;
          for (int r = int(lane); r < 128; r += 32) {
            const int64_t row = int64_t(rt) * 128 + r;
            if (row >= jj.R) break;
            const int off = box * kBox + r * 128 + ((((cc >> 3) ^ (r & 7)) << 4) | ((cc & 7) << 1));
            jj.ocol.slice[int64_t(j) * jj.R + row] = *reinterpret_cast<const __nv_bfloat16*>(base + off);
          }
        }
      }
      if (kRow && jj.orow.slice != nullptr && jj.orow.nzero > 0) {
        const Mask* m = &masks[2 * t.jb];
        const int n = jj.orow.nzero;
        int j = lower_bound_idx(m->idx, n, rt * 128);
        const int j1 = lower_bound_idx(m->idx, n, rt * 128 + 128);
        for (; j < j1; ++j) {
          const int r = m->idx[j] - rt * 128;
          const int c = int(lane) * 4;   // 4 columns (8 bytes, inside one 16-byte chunk) per lane
          if (int64_t(ct) * 128 + c < jj.C) {
            const int box = c >> 6, cc = c & 63;
            const int off = box * kBox + r * 128 + ((((cc >> 3) ^ (r & 7)) << 4) | ((cc & 7) << 1));
            *reinterpret_cast<uint2*>(jj.orow.slice + int64_t(j) * jj.C + int64_t(ct) * 128 + c) =
                *reinterpret_cast<const uint2*>(base + off);
          }
        }
      }
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&empty[stage]);
      if (++stage == kStages) { stage = 0; phase ^= 1; }
    }
  } else if (warp == 2) {
    // ------------------------------------------------------------ store warp
    // One TMA store of the 128 x 64-byte code box and one 512-byte bulk copy of the scale chunk
    // per orientation and tile, so the epilogue warps never stall on global-store issue.
    TileRef t;
    TileCursor cur(J);
    for (int lt = 0; cur.next(J, t); ++lt) {
      const Job jj = J.j[t.jb];   // by value: one param-space read per tile
      const int rt = t.rt, ct = t.ct;
      const uint32_t buf = uint32_t(lt & 1), use = uint32_t(lt >> 1);
      ptx::mbar_wait(&staged[buf], use & 1);
      if (ptx::elect_one()) {
        ptx::fence_proxy_async();
#pragma unroll
        for (int o = 0; o < 2; ++o) {
          if ((o == 0 && !kRow) || (o == 1 && !kCol)) continue;
          const bool cs = o == 1;
          const int oi = kRow ? o : 0;   // staging slot of this orientation
          const int64_t srow0 = cs ? int64_t(ct) * 128 : int64_t(rt) * 128;
          const int kt = cs ? rt : ct;   // K-tile index: K-blocks [4 kt, 4 kt + 4)
          if (!(QTC_ABLATE & 4))
            ptx::tma_store_2d(cs ? &J.tqc[t.jb] : &J.tqr[t.jb], stg + (oi * 2 + buf) * kStg, kt * 64, int32_t(srow0));
          if (!(QTC_ABLATE & 8)) {
            uint8_t* gsf = (cs ? jj.ocol.sf : jj.orow.sf) + ((srow0 >> 7) * (cs ? jj.kch_col : jj.kch_row) + kt) * 512;
            ptx::bulk_store(gsf, sfstg + (oi * 2 + buf) * 512, 512);
          }
        }
        ptx::bulk_commit_group();
        ptx::bulk_wait_group_read<0>();
        QTC_T(5, lt);
        ptx::mbar_arrive(&stgfree[buf]);
      }
      __syncwarp();
    }
    if (ptx::elect_one()) ptx::bulk_wait_group<0>();
    __syncwarp();
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    // Dual launch: groups 0,1 -> row blocks {0,1},{2,3}; groups 2,3 -> column blocks {0,1},{2,3}.
    // Single orientation: group g -> block g. Four warps per SM sub-partition hide the
    // TMEM-load -> amax -> convert latency chain of each block. Group 0 also flushes the outlier
    // product of a finished segment (TMEM lane = tile column).
    constexpr int kOrients = (kRow ? 1 : 0) + (kCol ? 1 : 0);
    constexpr int kBlocksPerGroup = 4 * kOrients / kEpiGroups;
    constexpr int kGroupsPerOrient = kEpiGroups / kOrients;
    const uint32_t group = (warp - 4) >> 2;
    const uint32_t orient = group / kGroupsPerOrient;          // 0: first enabled orientation
    const uint32_t sub = group % kGroupsPerOrient;
    const bool col_side = kRow ? (orient == 1) : true;
    const uint32_t q = warp & 3;
    const uint32_t row = q * 32 + lane;        // stored row within the tile = TMEM lane
    const uint32_t blk0 = sub * kBlocksPerGroup;
    const uint32_t oi = kRow ? orient : 0;     // staging slot of this orientation
    const uint32_t sw = (row >> 1) & 3;        // 64B swizzle of the staging row
    int segs[kMaxOr] = {0, 0};
    TileRef t;
    TileCursor cur(J);
    for (int lt = 0; cur.next(J, t); ++lt) {
      const Job jj = J.j[t.jb];   // by value: one param-space read per tile
      const int rt = t.rt, ct = t.ct;
      const Out& o = col_side ? jj.ocol : jj.orow;
      const uint32_t* bits = mbits + o.bits_off;
      const int64_t K = col_side ? jj.R : jj.C;
      const int64_t rows_total = col_side ? jj.C : jj.R;
      const uint32_t sbuf = uint32_t(lt & 1), suse = uint32_t(lt >> 1);   // staging buffers
      const uint32_t buf = kTBufs == 2 ? sbuf : 0u;                         // TMEM buffer
      const uint32_t use = kTBufs == 2 ? suse : uint32_t(lt);
      uint8_t* st = stg + (oi * 2 + sbuf) * kStg;
      uint8_t* sst = sfstg + (oi * 2 + sbuf) * 512;
      const int64_t srow = (col_side ? int64_t(ct) * 128 : int64_t(rt) * 128) + row;
      const int64_t kb0 = (col_side ? int64_t(rt) * 4 : int64_t(ct) * 4) + blk0;   // first K-block of this group
      const bool extracted = srow < rows_total && o.nzero > 0 && ((bits[srow >> 5] >> (srow & 31)) & 1u);
      ptx::mbar_wait(&stgfree[sbuf], (suse & 1) ^ 1);   // the store warp has read this staging buffer
      ptx::mbar_wait(&tfull[buf], use & 1);
      if (warp == 4 && lane == 0) QTC_T(3, lt);
      ptx::tc_fence_after();
#pragma unroll
      for (int b = 0; b < kBlocksPerGroup; ++b) {
        uint32_t d[32];
        if (QTC_ABLATE & 2) {
#pragma unroll
          for (int i = 0; i < 32; ++i) d[i] = 0;
        } else {
          ptx::tmem_ld_32x32b_x32(tmem_base + ((q * 32) << 16) + buf * 256 + (col_side ? 128 : 0) + (blk0 + b) * 32, d);
          ptx::tmem_ld_wait();
        }
        if (b == kBlocksPerGroup - 1) {   // accumulators drained: the MMA warp may reuse this buffer
          if (warp == 4 && lane == 0) QTC_T(4, lt);
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&tempty[buf]);
        }
        float ysink[kHad ? 32 : 1];
        uint4 c;
        uint32_t sbyte;
        if (QTC_ABLATE & 2) { c = make_uint4(d[0], d[1], d[2], d[3]); sbyte = 127; }
        else quant_block<kHad>(d, c, sbyte, ysink);
        if (extracted) { c = make_uint4(0, 0, 0, 0); sbyte = 127u; }
        *reinterpret_cast<uint4*>(st + row * 64 + (((blk0 + b) ^ sw) << 4)) = c;
        // SF chunk byte of (row, K-block) = (row % 32) * 16 + (row / 32) * 4 + kb % 4
        sst[lane * 16 + q * 4 + blk0 + b] = uint8_t(sbyte);
        if (kHad && srow < rows_total && (kb0 + b) * kBlk < K) {
          float* dst = o.had + srow * K + (kb0 + b) * kBlk;
#pragma unroll
          for (int i = 0; i < 32; ++i) dst[i] = extracted ? 0.f : ysink[i];
        }
      }
      ptx::fence_proxy_async();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&staged[sbuf]);
      if (kOr && t.orr && t.last && !J.orr[t.oi].dry) {
        if (group == 0) {
          // flush the finished segment: P[c = 128 ct + row][j] -> its (band, CTA) partial slot
          const OrSpec& os = J.orr[t.oi];
          const int npad = os.npad;
          const uint32_t pcol = kOrCol + kOrMaxN * t.oi;
          ptx::mbar_wait(&orfull[t.oi], uint32_t(segs[t.oi] & 1));
          ptx::tc_fence_after();
          uint32_t p0[32], p1[32];
          ptx::tmem_ld_32x32b_x32(tmem_base + ((q * 32) << 16) + pcol, p0);
          if (npad > 32) ptx::tmem_ld_32x32b_x32(tmem_base + ((q * 32) << 16) + pcol + 32, p1);
          ptx::tmem_ld_wait();
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&orempty[t.oi]);
          const int u0 = ct * os.rtiles;
          const int slot = int(blockIdx.x) - or_chunk_of(os, u0);
          float* dst = os.part + (int64_t(ct) * os.spb + slot) * npad * 128 + row;
          // lanes = consecutive columns: one 128-byte store per (warp, j)
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (j < npad) dst[int64_t(j) * 128] = __uint_as_float(p0[j]);
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (32 + j < npad) dst[int64_t(32 + j) * 128] = __uint_as_float(p1[j]);
        }
        ++segs[t.oi];
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem_base);
  }
#if QTC_TRACE
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const long long t0 = g_qtc_trace[0][0];
    TileRef t;
    TileCursor cur(J);
    for (int i = 0; i < 64 && cur.next(J, t); ++i)
      printf("qtc tile %2d: tma %7lld tempty %7lld full %7lld epi %7lld drained %7lld stored %7lld\n", i,
             g_qtc_trace[0][i] - t0, g_qtc_trace[1][i] - t0, g_qtc_trace[2][i] - t0, g_qtc_trace[3][i] - t0,
             g_qtc_trace[4][i] - t0, g_qtc_trace[5][i] - t0);
  }
#endif
}

}  // namespace qtc

// bitmap_words: the total size of the launch's OE membership bitmaps (0 without masks)
static size_t quant_tc_smem(bool masks, int64_t bitmap_words, bool orr) {
  const size_t ring = orr ? size_t(qtc::Ring<true>::kStages) * qtc::Ring<true>::kStage
                          : size_t(qtc::Ring<false>::kStages) * qtc::Ring<false>::kStage;
  return ring + 4 * qtc::kStg + 4 * 512 + qtc::kHBytes + 1024 + 176 +
         (masks ? 2 * qtc::kMaxJobs * sizeof(qtc::Mask) + size_t(bitmap_words) * 4 : 0);
}
constexpr size_t kSmemLimit = 232448;   // 227 KB per CTA on sm_100
// every (job, orientation) of a launch may carry a mask over up to kMaskMaxRows stored rows
static size_t quant_tc_smem_max(bool orr) {
  const size_t m = quant_tc_smem(true, 2 * qtc::kMaxJobs * (qtc::kMaskMaxRows / 32), orr);
  return m < kSmemLimit ? m : kSmemLimit;
}

bool quant_tc_supported(int64_t R, int64_t C, int64_t ld, const void* in, bool row_mask, bool col_mask) {
  return (ld * 2) % 16 == 0 && (reinterpret_cast<uintptr_t>(in) & 15) == 0 &&
         (!row_mask || R <= qtc::kMaskMaxRows) && (!col_mask || C <= qtc::kMaskMaxRows);
}

// Partial slots per column band of the fused outlier product over T [R x C] when the OR tiles
// are cut into chunks = min(tiles, num_sms) contiguous chunks (host copy of the device rule).
static int or_slots_per_band(const qtc::OrSpec& o) {
  int spb = 0;
  for (int ct = 0; ct * o.rtiles < o.n; ++ct) {
    const int64_t u0 = int64_t(ct) * o.rtiles, u1 = std::min<int64_t>(o.n, int64_t(ct + 1) * o.rtiles) - 1;
    const int64_t b0 = ((u0 + 1) * o.chunks - 1) / o.n, b1 = ((u1 + 1) * o.chunks - 1) / o.n;
    spb = std::max(spb, int(b1 - b0 + 1));
  }
  return spb;
}
static qtc::OrSpec or_spec(int64_t R, int64_t C, int kk, int num_sms) {
  qtc::OrSpec o{};
  o.on = 1;
  o.kk = kk;
  o.npad = int((kk + 15) / 16 * 16);
  o.rtiles = int((R + 127) / 128);
  o.n = o.rtiles * int((C + 127) / 128);
  o.chunks = std::min(o.n, num_sms);
  o.spb = or_slots_per_band(o);
  return o;
}
OePatch quant_tc_or_patch(int64_t R, int64_t C, int kk, int num_sms, const float* part, unsigned* ticket, float* Dt,
                          const int32_t* idx, int mode) {
  const qtc::OrSpec o = or_spec(R, C, kk, num_sms);
  OePatch p{Dt, idx, C, kk, mode};
  p.part = part;
  p.ticket = ticket;
  p.spb = o.spb;
  p.npad = o.npad;
  p.or_n = o.n;
  p.or_rtiles = o.rtiles;
  p.or_chunks = o.chunks;
  return p;
}
size_t quant_tc_or_part_bytes(int64_t R, int64_t C, int kk, int num_sms) {
  if (kk <= 0 || kk > qtc::kOrMaxN || R <= 0 || C <= 0) return 0;
  const qtc::OrSpec o = or_spec(R, C, kk, num_sms);
  return size_t((C + 127) / 128) * size_t(o.spb) * size_t(o.npad) * 128 * 4;
}

template <bool kRow, bool kCol, bool kHad, bool kOr>
static cudaError_t launch_tc(const qtc::Jobs& J, bool masks, int64_t bitmap_words, int num_sms, cudaStream_t st) {
  const size_t smem = quant_tc_smem(masks, bitmap_words, kOr);
  if (smem > kSmemLimit) return cudaErrorInvalidValue;
  static std::atomic<uint64_t> attr{0};
  cudaError_t ae = once_per_device(attr, [] {
    return cudaFuncSetAttribute(qtc::k_quant_tc<kRow, kCol, kHad, kOr>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                int(quant_tc_smem_max(kOr)));
  });
  if (ae != cudaSuccess) return ae;
  int tiles = J.ntiles;
  if (kOr)
    for (int o = 0; o < J.nor; ++o) tiles += J.orr[o].n;
  const unsigned grid = unsigned(tiles < num_sms ? tiles : num_sms);
  return launch_k(qtc::k_quant_tc<kRow, kCol, kHad, kOr>, dim3(grid), dim3(qtc::kThreads), smem, st, 1, J);
}

// Each job: T [R x C] bf16 (pitch ld). Row outputs (stored rows = R, K = C) and / or column
// outputs (stored rows = C, K = R); all jobs of one launch produce the same orientations.
// had_* (debug, nullable) receive the fp32 Hadamard output of the respective orientation.
// OE slices (the extracted rows / columns, raw bf16) for the BF16 outlier GEMM:
//   orient 0: out[s][c] = T[idx[s], c]  (c < C)      orient 1: out[s][r] = T[r, idx[s]]  (r < R)
// Column gathers: a block covers 32 rows; lane = row (coalesced 64-byte writes per slice row).
__global__ void __launch_bounds__(256) k_oe_gather(const __nv_bfloat16* __restrict__ T, int64_t R, int64_t C,
                                                   int64_t ld, int orient, const int32_t* __restrict__ idx, int n,
                                                   __nv_bfloat16* __restrict__ out) {
  ptx::griddep_launch();
  ptx::griddep_wait();
  if (orient == 0) {
    // block (s, chunk): 256 threads x 8 elements
    const int s = blockIdx.y;
    const int64_t c = (int64_t(blockIdx.x) * 256 + threadIdx.x) * 8;
    if (s >= n || c >= C) return;
    const __nv_bfloat16* src = T + int64_t(idx[s]) * ld + c;
    __nv_bfloat16* dst = out + int64_t(s) * C + c;
    if (c + 8 <= C && ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {
      *reinterpret_cast<uint4*>(dst) = __ldg(reinterpret_cast<const uint4*>(src));
    } else {
      for (int i = 0; i < 8 && c + i < C; ++i) dst[i] = src[i];
    }
  } else {
    const int lane = threadIdx.x & 31, wy = threadIdx.x >> 5;   // 8 warps: slots wy, wy + 8, ...
    const int64_t r = int64_t(blockIdx.x) * 32 + lane;
    if (r >= R) return;
    const __nv_bfloat16* row = T + r * ld;
    // eight independent loads in flight per thread before the stores
    for (int s0 = wy; s0 < n; s0 += 64) {
      __nv_bfloat16 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int s = s0 + 8 * u;
        v[u] = s < n ? row[__ldg(idx + s)] : __nv_bfloat16();
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int s = s0 + 8 * u;
        if (s < n) out[int64_t(s) * R + r] = v[u];
      }
    }
  }
}

static cudaError_t launch_oe_gather(const __nv_bfloat16* T, int64_t R, int64_t C, int64_t ld, int orient,
                                    const int32_t* idx, int n, __nv_bfloat16* out, cudaStream_t st) {
  if (n <= 0 || out == nullptr) return cudaSuccess;
  if (orient == 0) {
    const dim3 grid(unsigned((C + 2047) / 2048), unsigned(n));
    return launch_k(k_oe_gather, grid, dim3(256), 0, st, 1, T, R, C, ld, 0, idx, n, out);
  }
  return launch_k(k_oe_gather, dim3(unsigned((R + 31) / 32)), dim3(256), 0, st, 1, T, R, C, ld, 1, idx, n, out);
}

// ADAHOP_GATHER_AFTER=1: gathers after the quant pass, the gathered tensor's tiles last (so the
// gather reads L2) — measured slower (quant stage 0.65 vs 0.53 ms per Llama-3.2-1B layer step)
// ADAHOP_GATHER_FUSED=1: OE slices copied by the quant kernel's gather warp (warp 3) from the
// staged tiles instead of the separate k_oe_gather launches — measured slower (quant stage 0.59
// vs 0.54 ms per Llama-3.2-1B layer step: the stage release waits for the copies)
static bool gather_fused() {
  static const int v = knob("ADAHOP_GATHER_FUSED", 0);
  return v != 0;
}
// ADAHOP_OR_FUSED=2 (experiment builds): every dual launch runs the fused-product kernel variant
// (single TMEM buffer, 3-stage ring) without a product, to separate its costs
static bool or_variant_without_product() {
  static const int v = knob("ADAHOP_OR_FUSED", 1);
  return v == 2;
}
static bool gather_after_quant() {
  static const int v = knob("ADAHOP_GATHER_AFTER", 0);
  return v != 0;
}

cudaError_t launch_quant_tc_multi(const QuantTcJob* jobs_in, int n, int num_sms, cudaStream_t st, int* launches,
                                  bool* or_fused) {
  if (or_fused)
    for (int i = 0; i < n; ++i) or_fused[i] = false;
  if (n <= 0) return cudaSuccess;
  if (n > qtc::kMaxJobs) return cudaErrorInvalidValue;
  // The OE slices come from a separate gather (copying them inside the quant pipeline stalls
  // it), launched before the quant pass (see gather_after_quant for the measured alternative).
  const bool after = gather_after_quant();
  const bool fused = gather_fused() && !after;
  // The fused outlier products (up to kMaxOr jobs; their slices must exist before the launch, so
  // not with the in-kernel gathers) run on the dual-orientation kernel; their jobs go last.
  int or_in[qtc::kMaxOr], nor = 0;
  bool orr = !after && !fused;
  for (int i = 0; i < n; ++i) {
    if (!jobs_in[i].or_slice) continue;
    if (nor == qtc::kMaxOr) return cudaErrorInvalidValue;
    or_in[nor++] = i;
    const QuantTcJob& q = jobs_in[i];
    orr &= q.q_row && q.q_col && !q.had_row && !q.had_col && q.or_kk > 0 && q.or_kk <= qtc::kOrMaxN && q.or_ticket &&
           q.or_part_bytes >= quant_tc_or_part_bytes(q.R, q.C, q.or_kk, num_sms);
  }
  orr &= nor > 0;
  auto is_or = [&](int i) {
    for (int o = 0; o < nor; ++o)
      if (or_in[o] == i) return true;
    return false;
  };
  QuantTcJob jobs[qtc::kMaxJobs];
  int src[qtc::kMaxJobs];   // jobs_in index of jobs[m]
  int m = 0;
  for (int pass = 0; pass < (after ? 2 : 1); ++pass)
    for (int i = 0; i < n; ++i) {
      const bool colg = jobs_in[i].q_col && jobs_in[i].ncol_zero > 0 && jobs_in[i].slice_col;
      if (orr ? !is_or(i) : (!after || colg == (pass == 1))) { src[m] = i; jobs[m++] = jobs_in[i]; }
    }
  if (orr)
    for (int o = 0; o < nor; ++o) { src[m] = or_in[o]; jobs[m++] = jobs_in[or_in[o]]; }
  const int nor_l = orr ? nor : 0;   // OR jobs of this launch (the last nor_l)
  auto gathers = [&]() -> cudaError_t {
    for (int i = 0; i < n; ++i) {
      const QuantTcJob& q = jobs[i];
      if (q.q_row && q.nrow_zero > 0 && q.slice_row) {
        cudaError_t e = launch_oe_gather(q.in, q.R, q.C, q.ld, 0, q.row_zero, q.nrow_zero, q.slice_row, st);
        if (e != cudaSuccess) return e;
        if (launches) ++*launches;
      }
      if (q.q_col && q.ncol_zero > 0 && q.slice_col) {
        cudaError_t e = launch_oe_gather(q.in, q.R, q.C, q.ld, 1, q.col_zero, q.ncol_zero, q.slice_col, st);
        if (e != cudaSuccess) return e;
        if (launches) ++*launches;
      }
    }
    return cudaSuccess;
  };
  qtc::Jobs J;
  memset(&J, 0, sizeof(J));
  J.n = n;
  const bool row = jobs[0].q_row != nullptr, col = jobs[0].q_col != nullptr;
  const bool had = jobs[0].had_row != nullptr || jobs[0].had_col != nullptr;
  bool masks = false;
  int64_t words = 0;   // bitmap words of the launch's masks
  int tiles = 0;
  for (int i = 0; i < n; ++i) {
    const QuantTcJob& q = jobs[i];
    if ((q.q_row != nullptr) != row || (q.q_col != nullptr) != col ||
        (q.had_row != nullptr || q.had_col != nullptr) != had)
      return cudaErrorInvalidValue;
    if (!make_tmap_2d(&J.tm[i], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, q.in, uint64_t(q.C), uint64_t(q.R),
                      uint64_t(q.ld) * 2, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B))
      return cudaErrorInvalidValue;
    // code outputs, stored by TMA: [stored rows][K/2] bytes, 128 x 64-byte boxes, 64B swizzle
    J.tqr[i] = J.tqc[i] = J.tm[i];
    if (row && !make_tmap_2d(&J.tqr[i], CU_TENSOR_MAP_DATA_TYPE_UINT8, q.q_row, uint64_t(q.C / 2), uint64_t(q.R),
                             uint64_t(q.C / 2), 64, 128, CU_TENSOR_MAP_SWIZZLE_64B))
      return cudaErrorInvalidValue;
    if (col && !make_tmap_2d(&J.tqc[i], CU_TENSOR_MAP_DATA_TYPE_UINT8, q.q_col, uint64_t(q.R / 2), uint64_t(q.C),
                             uint64_t(q.R / 2), 64, 128, CU_TENSOR_MAP_SWIZZLE_64B))
      return cudaErrorInvalidValue;
    qtc::Job& jj = J.j[i];
    jj.R = q.R; jj.C = q.C;
    jj.ctiles = int((q.C + 127) / 128);
    jj.tile0 = tiles;
    if (i < n - nor_l) tiles += jj.ctiles * int((q.R + 127) / 128);
    jj.kch_row = sf_kchunks(q.C);
    jj.kch_col = sf_kchunks(q.R);
    jj.orow = qtc::Out{q.q_row, q.sf_row, q.row_zero, row ? q.nrow_zero : 0, fused ? q.slice_row : nullptr, q.had_row, 0};
    jj.ocol = qtc::Out{q.q_col, q.sf_col, q.col_zero, col ? q.ncol_zero : 0, fused ? q.slice_col : nullptr, q.had_col, 0};
    if (jj.orow.nzero > 0) {
      if (q.R > qtc::kMaskMaxRows) return cudaErrorInvalidValue;
      jj.orow.bits_off = int(words);
      words += (q.R + 31) / 32;
    }
    if (jj.ocol.nzero > 0) {
      if (q.C > qtc::kMaskMaxRows) return cudaErrorInvalidValue;
      jj.ocol.bits_off = int(words);
      words += (q.C + 31) / 32;
    }
    masks |= jj.orow.nzero > 0 || jj.ocol.nzero > 0;
  }
  J.ntiles = tiles;
  J.nor = nor_l;
  bool fits = quant_tc_smem(masks, words, true) <= kSmemLimit;
  for (int o = 0; o < nor_l && fits; ++o) {
    const QuantTcJob& q = jobs[n - nor_l + o];
    J.orr[o] = or_spec(q.R, q.C, q.or_kk, num_sms);
    J.orr[o].part = q.or_part;
    J.orr[o].ticket = q.or_ticket;
    J.orr[o].dry = knob("ADAHOP_OR_FUSED", 1) == 3 ? 1 : 0;
    // the slice S [kk][R] (R contiguous): boxes of 64 rows of T (128 B) x npad slice rows, OOB -> 0
    fits = make_tmap_2d(&J.tor[o], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, q.or_slice, uint64_t(q.R), uint64_t(q.or_kk),
                        uint64_t(q.R) * 2, 64, uint32_t(J.orr[o].npad), CU_TENSOR_MAP_SWIZZLE_128B);
  }
  if (orr && !fits) {
    // does not fit: the caller runs the BF16 outlier GEMMs; the jobs become plain ones again
    orr = false;
    J.nor = 0;
    for (int o = 0; o < qtc::kMaxOr; ++o) J.orr[o] = qtc::OrSpec{};
    for (int o = 0; o < nor_l; ++o) {
      const qtc::Job& jj = J.j[n - nor_l + o];
      J.ntiles += jj.ctiles * int((jj.R + 127) / 128);
    }
  }
  if (!after && !fused) {
    cudaError_t e = gathers();
    if (e != cudaSuccess) return e;
  }
  if (launches) ++*launches;
  cudaError_t e = cudaSuccess;
  if (orr || (row && col && !had && or_variant_without_product()))
    e = launch_tc<true, true, false, true>(J, masks, words, num_sms, st);
  else if (row && col) e = had ? launch_tc<true, true, true, false>(J, masks, words, num_sms, st)
                               : launch_tc<true, true, false, false>(J, masks, words, num_sms, st);
  else if (row) e = had ? launch_tc<true, false, true, false>(J, masks, words, num_sms, st)
                        : launch_tc<true, false, false, false>(J, masks, words, num_sms, st);
  else if (col) e = had ? launch_tc<false, true, true, false>(J, masks, words, num_sms, st)
                        : launch_tc<false, true, false, false>(J, masks, words, num_sms, st);
  if (e != cudaSuccess) return e;
  if (orr && or_fused)
    for (int o = 0; o < nor_l; ++o) or_fused[src[n - nor_l + o]] = true;
  return after ? gathers() : cudaSuccess;
}

cudaError_t launch_quant_tc(const __nv_bfloat16* in, int64_t R, int64_t C, int64_t ld, const int32_t* row_zero,
                            int nrow_zero, __nv_bfloat16* slice_row, uint8_t* q_row, uint8_t* sf_row, float* had_row,
                            const int32_t* col_zero, int ncol_zero, __nv_bfloat16* slice_col, uint8_t* q_col,
                            uint8_t* sf_col, float* had_col, int num_sms, cudaStream_t st) {
  const QuantTcJob q{in, R, C, ld, row_zero, nrow_zero, slice_row, q_row, sf_row, had_row,
                     col_zero, ncol_zero, slice_col, q_col, sf_col, had_col};
  return launch_quant_tc_multi(&q, 1, num_sms, st, nullptr, nullptr);
}

}  // namespace adahop
