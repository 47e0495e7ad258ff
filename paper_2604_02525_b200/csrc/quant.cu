// quant.cu — HBM-bound kernels of the AdaHOP hot path (sm_100a):
//   * fused residual mask + blockwise FWHT (b = 32) + MXFP4 quantisation, in a row
//     (K-contiguous) and a transposing column (K-strided) variant   [P:350, P:761]
//   * FOID: fp64 probe variance, deterministic top-k, outlier-slice gather  [P:760]
//   * pattern statistics for calibration (per-row / per-column moments)    [P:523-541]
//   * layout converters used only by the debug / parity entry points
#include <cstdio>
#include "common.cuh"
#include "kernels.h"
#include "ptx.cuh"
#include <algorithm>
#include <cstdlib>

namespace adahop {

// RN32(1/sqrt(32)) — 1/sqrt(2) (0x3F3504F3) scaled by 2^-2, exact.
#define ADAHOP_INV_SQRT32 __uint_as_float(0x3E3504F3u)

// Pack 8 fp32 values (already divided by the block scale) into 8 E2M1 nibbles,
// element 0 in the low nibble. Hardware RNE + saturation to +-6.
__device__ __forceinline__ uint32_t e2m1x8_hw(const float* v) {
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

// Software reference of the same rounding: nearest of {0,.5,1,1.5,2,3,4,6}, ties to
// the even-mantissa code, saturating, sign bit = signbit(v).
__device__ __forceinline__ uint32_t e2m1_sw(float v) {
  const float a = fabsf(v);
  uint32_t c = (a > 0.25f) + (a >= 0.75f) + (a > 1.25f) + (a >= 1.75f) + (a > 2.5f) +
               (a >= 3.5f) + (a > 5.0f);
  return c | ((__float_as_uint(v) >> 28) & 8u);
}
__device__ __forceinline__ uint32_t e2m1x8_sw(const float* v) {
  uint32_t out = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) out |= e2m1_sw(v[i]) << (4 * i);
  return out;
}

// ------------------------------------------------------------------------------------
// Packed fp32x2 arithmetic (sm_100 FADD2 / FMUL2): two independent IEEE round-to-nearest
// operations per instruction, bit-identical to the scalar ones. A thread quantises TWO
// 32-element blocks at once (two stored rows in the column variant, two adjacent K-blocks
// of one row in the row variant) with lane 0 / lane 1 of every pair holding block 0 / 1.
// ------------------------------------------------------------------------------------
__device__ __forceinline__ uint64_t f2_add(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t f2_sub(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t f2_mul(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t f2_pack(float lo, float hi) {
  // plain integer composition: the register allocator places lo/hi in the pair directly
  return (uint64_t(__float_as_uint(hi)) << 32) | uint64_t(__float_as_uint(lo));
}
__device__ __forceinline__ float f2_lo(uint64_t v) { return __uint_as_float(uint32_t(v)); }
__device__ __forceinline__ float f2_hi(uint64_t v) { return __uint_as_float(uint32_t(v >> 32)); }

// E8M0 exponent of a block from max|fwht| (before the 1/sqrt(32) scaling):
// e = floor(log2 RN(amax c)) - 2, clamped; zero block -> 0.
__device__ __forceinline__ int mx_exponent(float amax_raw) {
  const float amax_y = __fmul_rn(amax_raw, ADAHOP_INV_SQRT32);  // == max|RN(x c)| (RN monotone)
  const uint32_t bits = __float_as_uint(amax_y);
  int e;
  if (amax_y == 0.f) e = 0;
  else if ((bits >> 23) != 0) e = int(bits >> 23) - 127 - 2;
  else e = (31 - __clz(int(bits))) - 149 - 2;  // subnormal amax
  return max(-127, min(127, e));
}
__device__ __forceinline__ float pow2f(int e) { return __uint_as_float(uint32_t(127 + e) << 23); }

template <bool kSwCvt>
__device__ __forceinline__ uint32_t cvt8(const float* v) {
  return kSwCvt ? e2m1x8_sw(v) : e2m1x8_hw(v);
}

// IHT + MX quantisation of two blocks packed in P[i] = (block0[i], block1[i]).
// Radix-2 butterflies with strides 1,2,4,8,16 (natural-order Walsh–Hadamard) in fp32 RN,
// then y = RN(x c) with c = RN32(1/sqrt 32), then v = y 2^-e (exact), E2M1 RNE satfinite.
template <bool kHad, bool kSwCvt>
__device__ __forceinline__ void iht_quant_pair(uint64_t (&P)[32], uint4& codes0, uint4& codes1,
                                               uint32_t& s0, uint32_t& s1, float* y0, float* y1) {
#pragma unroll
  for (int h = 1; h < 32; h <<= 1) {
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      if ((i & h) == 0) {
        const uint64_t a = P[i], b = P[i + h];
        P[i] = f2_add(a, b);
        P[i + h] = f2_sub(a, b);
      }
    }
  }
  // block amax as a depth-5 tree (a serial max chain would stall the warp ~128 cycles)
  float t0[16], t1[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    t0[i] = fmaxf(fabsf(f2_lo(P[i])), fabsf(f2_lo(P[i + 16])));
    t1[i] = fmaxf(fabsf(f2_hi(P[i])), fabsf(f2_hi(P[i + 16])));
  }
#pragma unroll
  for (int wdt = 8; wdt >= 1; wdt >>= 1) {
#pragma unroll
    for (int i = 0; i < wdt; ++i) {
      t0[i] = fmaxf(t0[i], t0[i + wdt]);
      t1[i] = fmaxf(t1[i], t1[i + wdt]);
    }
  }
  const float m0 = t0[0], m1 = t1[0];
  const int e0 = mx_exponent(m0), e1 = mx_exponent(m1);
  s0 = uint32_t(e0 + 127);
  s1 = uint32_t(e1 + 127);
  const float c = ADAHOP_INV_SQRT32;
  if (kHad || e0 > 120 || e0 < -100 || e1 > 120 || e1 < -100) {
    // exact two-step path: y = RN(x c); v = y * 2^-e (power-of-two scaling, exact)
    float v0[32], v1[32];
    const uint64_t cc = f2_pack(c, c);
    const uint64_t ss = f2_pack(pow2f(-e0), pow2f(-e1));
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const uint64_t y = f2_mul(P[i], cc);
      if (kHad) {
        y0[i] = f2_lo(y);
        y1[i] = f2_hi(y);
      }
      const uint64_t v = f2_mul(y, ss);
      v0[i] = f2_lo(v);
      v1[i] = f2_hi(v);
    }
    codes0 = make_uint4(cvt8<kSwCvt>(v0), cvt8<kSwCvt>(v0 + 8), cvt8<kSwCvt>(v0 + 16), cvt8<kSwCvt>(v0 + 24));
    codes1 = make_uint4(cvt8<kSwCvt>(v1), cvt8<kSwCvt>(v1 + 8), cvt8<kSwCvt>(v1 + 16), cvt8<kSwCvt>(v1 + 24));
  } else {
    // fused: RN(x (c 2^-e)) == RN(x c) 2^-e for every value that can reach a nonzero code;
    // converted 8 at a time to keep register pressure low
    const uint64_t cs = f2_pack(__fmul_rn(c, pow2f(-e0)), __fmul_rn(c, pow2f(-e1)));
    uint32_t w0[4], w1[4];
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      float a[8], b[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint64_t v = f2_mul(P[8 * g + i], cs);
        a[i] = f2_lo(v);
        b[i] = f2_hi(v);
      }
      w0[g] = cvt8<kSwCvt>(a);
      w1[g] = cvt8<kSwCvt>(b);
    }
    codes0 = make_uint4(w0[0], w0[1], w0[2], w0[3]);
    codes1 = make_uint4(w1[0], w1[1], w1[2], w1[3]);
  }
}

__device__ __forceinline__ void store_f32x32(float* dst, const float* y) {
#pragma unroll
  for (int i = 0; i < 32; ++i) dst[i] = y[i];
}

// bf16 / fp32 element -> fp32 (exact)
__device__ __forceinline__ float bf16lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

// 32 raw values -> 64 contiguous bytes of the bf16 outlier slice (RN for fp32 inputs).
__device__ __forceinline__ void store_slice32(__nv_bfloat16* dst, const float* x) {
  uint4* d = reinterpret_cast<uint4*>(dst);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    uint32_t w[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      __nv_bfloat162 h = __floats2bfloat162_rn(x[8 * j + 2 * t], x[8 * j + 2 * t + 1]);
      w[t] = *reinterpret_cast<uint32_t*>(&h);
    }
    d[j] = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// Raw 64 contiguous elements (two K-blocks) of one row, as 16-byte vectors.
template <typename T> struct RowRaw;
template <> struct RowRaw<__nv_bfloat16> {
  uint4 v[8];
  __device__ __forceinline__ void load(const __nv_bfloat16* p, bool two) {
    const uint4* q = reinterpret_cast<const uint4*>(p);
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = __ldg(q + j);
#pragma unroll
    for (int j = 4; j < 8; ++j) v[j] = two ? __ldg(q + j) : make_uint4(0, 0, 0, 0);
  }
  __device__ __forceinline__ float get(int b, int i) const {  // block b, element i
    const uint4& u = v[b * 4 + (i >> 3)];
    const uint32_t w = ((i >> 1) & 3) == 0 ? u.x : ((i >> 1) & 3) == 1 ? u.y : ((i >> 1) & 3) == 2 ? u.z : u.w;
    return (i & 1) ? bf16hi(w) : bf16lo(w);
  }
};
template <> struct RowRaw<float> {
  float4 v[16];
  __device__ __forceinline__ void load(const float* p, bool two) {
    const float4* q = reinterpret_cast<const float4*>(p);
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = __ldg(q + j);
#pragma unroll
    for (int j = 8; j < 16; ++j) v[j] = two ? __ldg(q + j) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  __device__ __forceinline__ float get(int b, int i) const {
    const float4& u = v[b * 8 + (i >> 2)];
    return (i & 3) == 0 ? u.x : (i & 3) == 1 ? u.y : (i & 3) == 2 ? u.z : u.w;
  }
};

// Row variant: stored row r is in[r*ld + 0..K). One thread per (row, pair of K-blocks),
// persistent grid-stride loop with the next pair's 128 B prefetched into registers.
template <typename T, bool kHad, bool kSwCvt>
__global__ void __launch_bounds__(256) k_iht_quant_row(const T* __restrict__ in, int64_t R,
                                                       int64_t K, int64_t ld,
                                                       const int32_t* __restrict__ zero_rows,
                                                       int nzero, uint8_t* __restrict__ codes,
                                                       uint8_t* __restrict__ sf, int64_t kchunks,
                                                       float* __restrict__ had_out,
                                                       __nv_bfloat16* __restrict__ slice) {
  const int64_t nkb = K / kBlk;
  const int64_t npair = (nkb + 1) / 2;
  const int64_t total = R * npair;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= total) return;
  // 32-bit index math (the host guarantees total < 2^31)
  const uint32_t np32 = uint32_t(npair);
  RowRaw<T> cur, nxt;
  {
    const int64_t r = uint32_t(t) / np32, q = t - r * npair;
    cur.load(in + r * ld + q * 2 * kBlk, 2 * q + 1 < nkb);
  }
  for (; t < total; t += stride) {
    const int64_t r = uint32_t(t) / np32, q = t - r * npair;
    const int64_t kb0 = 2 * q;
    const bool two = kb0 + 1 < nkb;
    const int64_t tn = t + stride;
    if (tn < total) {
      const int64_t rn = uint32_t(tn) / np32, qn = tn - rn * npair;
      nxt.load(in + rn * ld + qn * 2 * kBlk, 2 * qn + 1 < nkb);
    }
    uint64_t P[32];
    const int slot = nzero > 0 ? find_sorted(zero_rows, nzero, r) : -1;
    if (slot >= 0) {
      // OE row: raw values -> BF16 outlier slice, residual row = +0
      if (slice) {
        float x[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) x[i] = cur.get(0, i);
        store_slice32(slice + int64_t(slot) * K + kb0 * kBlk, x);
        if (two) {
#pragma unroll
          for (int i = 0; i < 32; ++i) x[i] = cur.get(1, i);
          store_slice32(slice + int64_t(slot) * K + (kb0 + 1) * kBlk, x);
        }
      }
#pragma unroll
      for (int i = 0; i < 32; ++i) P[i] = 0ull;
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) P[i] = f2_pack(cur.get(0, i), cur.get(1, i));
    }
    uint4 c0, c1;
    uint32_t s0, s1;
    float ya[kHad ? 32 : 1], yb[kHad ? 32 : 1];
    iht_quant_pair<kHad, kSwCvt>(P, c0, c1, s0, s1, ya, yb);
    if (kHad) {
      store_f32x32(had_out + r * K + kb0 * kBlk, ya);
      if (two) store_f32x32(had_out + r * K + (kb0 + 1) * kBlk, yb);
    }
    uint8_t* cdst = codes + r * (K / 2) + kb0 * 16;
    if (two) {
      reinterpret_cast<uint4*>(cdst)[0] = c0;
      reinterpret_cast<uint4*>(cdst)[1] = c1;
    } else {
      reinterpret_cast<uint4*>(cdst)[0] = c0;
    }
    sf[sf_offset(r, kb0, kchunks)] = uint8_t(s0);
    if (two) sf[sf_offset(r, kb0 + 1, kchunks)] = uint8_t(s1);
    cur = nxt;
  }
}

// ------------------------------------------------------------------------------------
// OE masks in shared memory: a bitmap over the stored rows for the O(1) "is this row
// extracted" test every thread makes per tile, plus a copy of the sorted index list for
// the (rare) slot lookup of an extracted row. Built once per CTA.
// ------------------------------------------------------------------------------------
constexpr int kMaskMaxRows = 32768;                 // bitmap capacity per mask
constexpr int kMaskWords = kMaskMaxRows / 32;
constexpr int kMaskMaxK = 256;

struct SmemMask {
  uint32_t bits[kMaskWords];
  int32_t idx[kMaskMaxK];
};

__device__ __forceinline__ void mask_build(SmemMask* m, const int32_t* __restrict__ idx, int n, int64_t rows) {
  const int words = int((rows + 31) / 32);
  for (int i = threadIdx.x; i < words; i += blockDim.x) m->bits[i] = 0u;
  for (int i = threadIdx.x; i < n; i += blockDim.x) m->idx[i] = idx[i];
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int r = idx[i];
    atomicOr(&m->bits[r >> 5], 1u << (r & 31));
  }
  __syncthreads();
}
__device__ __forceinline__ int mask_slot(const SmemMask* m, int n, int64_t r) {
  if (!((m->bits[r >> 5] >> (r & 31)) & 1u)) return -1;
  int lo = 0, hi = n - 1;
  while (lo <= hi) {
    const int mid = (lo + hi) >> 1;
    const int x = m->idx[mid];
    if (x == r) return mid;
    if (x < r) lo = mid + 1; else hi = mid - 1;
  }
  return -1;
}


// TMA-ring variant for bf16 sources with 16-byte aligned pitch (the production path).
// Persistent CTAs (one per SM, 256 threads) walk 32-KB tiles that a kStages-deep TMA ring
// keeps in flight; each thread quantises two 32-blocks per tile with fp32x2 arithmetic.
//  row (K-contiguous): tile = 256 stored rows x 64 K, 128B-swizzled, thread = one row's
//       pair of blocks; the swizzle makes the per-row 128-byte reads bank-conflict free.
//  col (K-strided, transposing): tile = 128 K x 128 stored rows, thread = (row pair, block),
//       reading both rows of a pair from one 4-byte word.
constexpr int kQStages = 3;
constexpr int kQTileBytes = 32768;

template <bool kCol, bool kHad, bool kSwCvt>
__global__ void __launch_bounds__(256, 2) k_iht_quant_tma(const __grid_constant__ CUtensorMap tm, int64_t R,
                                                          int64_t K, const int32_t* __restrict__ zero_rows,
                                                          int nzero, uint8_t* __restrict__ codes,
                                                          uint8_t* __restrict__ sf, int64_t kchunks,
                                                          float* __restrict__ had_out,
                                                          __nv_bfloat16* __restrict__ slice) {
  // row: TR = 256 rows, TK = 64; col: TR = 128 rows, TK = 128
  constexpr int TR = kCol ? 128 : 256, TK = kCol ? 128 : 64;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* ring = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + kQStages * kQTileBytes);
  SmemMask* mask = reinterpret_cast<SmemMask*>(full + kQStages);
  const int64_t rtiles = (R + TR - 1) / TR, ktiles = (K + TK - 1) / TK;
  const int64_t ntiles = rtiles * ktiles;
  const int tid = threadIdx.x;
  if (tid == 0) {
    ptx::prefetch_tmap(&tm);
    for (int i = 0; i < kQStages; ++i) ptx::mbar_init(&full[i], 1);
    ptx::fence_barrier_init();
  }
  if (nzero > 0) mask_build(mask, zero_rows, nzero, R);
  __syncthreads();
  const int64_t first = blockIdx.x, stride = gridDim.x;
  auto issue = [&](int64_t tile, int st) {
    const int64_t rt = tile % rtiles, kt = tile / rtiles;
    ptx::mbar_arrive_expect_tx(&full[st], kQTileBytes);
    if (kCol) ptx::tma_load_2d(ring + st * kQTileBytes, &tm, &full[st], int32_t(rt * TR), int32_t(kt * TK));
    else ptx::tma_load_2d(ring + st * kQTileBytes, &tm, &full[st], int32_t(kt * TK), int32_t(rt * TR));
  };
  if (tid == 0)
    for (int i = 0; i < kQStages; ++i)
      if (first + i * stride < ntiles) issue(first + i * stride, i);
  int it = 0;
  for (int64_t tile = first; tile < ntiles; tile += stride, ++it) {
    const int st = it % kQStages;
    ptx::mbar_wait(&full[st], uint32_t((it / kQStages) & 1));
    const int64_t rt = tile % rtiles, kt = tile / rtiles;
    const uint8_t* tb = ring + st * kQTileBytes;
    uint64_t P[32];            // P[i] = (block a element i, block b element i), raw values
    int64_t ra, rb, kba, kbb;  // (stored row, K-block) of the two blocks
    if (kCol) {
      const int p = tid % (TR / 2), kbl = tid / (TR / 2);
      ra = rt * TR + 2 * p;
      rb = ra + 1;
      kba = kbb = kt * (TK / kBlk) + kbl;
      const uint32_t* src = reinterpret_cast<const uint32_t*>(tb) + (kbl * 32) * (TR / 2) + p;
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const uint32_t w = src[i * (TR / 2)];
        P[i] = f2_pack(bf16lo(w), bf16hi(w));
      }
    } else {
      ra = rb = rt * TR + tid;
      kba = kt * 2;
      kbb = kba + 1;
      const uint8_t* row = tb + tid * 128;
      const int sw = tid & 7;   // 128B swizzle: 16-byte chunk j lives at j ^ (row % 8)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint4 ua = *reinterpret_cast<const uint4*>(row + ((j ^ sw) << 4));
        const uint4 ub = *reinterpret_cast<const uint4*>(row + (((j + 4) ^ sw) << 4));
        const uint32_t wa[4] = {ua.x, ua.y, ua.z, ua.w};
        const uint32_t wb[4] = {ub.x, ub.y, ub.z, ub.w};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          P[8 * j + 2 * t] = f2_pack(bf16lo(wa[t]), bf16lo(wb[t]));
          P[8 * j + 2 * t + 1] = f2_pack(bf16hi(wa[t]), bf16hi(wb[t]));
        }
      }
    }
    __syncthreads();                                   // stage consumed by every thread
    if (tid == 0 && tile + kQStages * stride < ntiles) issue(tile + kQStages * stride, st);
    const bool va = ra < R && kba * kBlk < K;
    const bool vb = rb < R && kbb * kBlk < K;
    if (nzero > 0) {
      const int sa = va ? mask_slot(mask, nzero, ra) : -1;
      const int sb = vb ? (kCol ? mask_slot(mask, nzero, rb) : sa) : -1;
      if (sa >= 0 || sb >= 0) {
        float x[32];
        if (sa >= 0 && slice) {
#pragma unroll
          for (int i = 0; i < 32; ++i) x[i] = f2_lo(P[i]);
          store_slice32(slice + int64_t(sa) * K + kba * kBlk, x);
        }
        if (sb >= 0 && slice) {
#pragma unroll
          for (int i = 0; i < 32; ++i) x[i] = f2_hi(P[i]);
          store_slice32(slice + int64_t(sb) * K + kbb * kBlk, x);
        }
#pragma unroll
        for (int i = 0; i < 32; ++i) P[i] = f2_pack(sa >= 0 ? 0.f : f2_lo(P[i]), sb >= 0 ? 0.f : f2_hi(P[i]));
      }
    }
    uint4 c0, c1;
    uint32_t s0, s1;
    float ya[kHad ? 32 : 1], yb[kHad ? 32 : 1];   // debug: the fp32 Hadamard output
    iht_quant_pair<kHad, kSwCvt>(P, c0, c1, s0, s1, ya, yb);
    if (kHad) {
      if (va) store_f32x32(had_out + ra * K + kba * kBlk, ya);
      if (vb) store_f32x32(had_out + rb * K + kbb * kBlk, yb);
    }
    if (va) {
      *reinterpret_cast<uint4*>(codes + ra * (K / 2) + kba * 16) = c0;
      sf[sf_offset(ra, kba, kchunks)] = uint8_t(s0);
    }
    if (vb) {
      *reinterpret_cast<uint4*>(codes + rb * (K / 2) + kbb * 16) = c1;
      sf[sf_offset(rb, kbb, kchunks)] = uint8_t(s1);
    }
  }
}


// ------------------------------------------------------------------------------------
// Dual-orientation IHT + MXFP4 quantisation: ONE pass over a bf16 tensor T [R x C] emits
//   the row quantisation   (stored rows = the R rows,    K = C) -> q_row, sf_row
//   the column quantisation (stored rows = the C columns, K = R) -> q_col, sf_col
// with independent OE masks for each orientation (row_zero: rows of T extracted from the
// row quantisation, gathered raw into slice_row [k x C]; col_zero: columns of T extracted
// from the column quantisation, gathered into slice_col [k x R]). This is how X, W and G_Y
// feed both of their matmuls (X: fwd + wgrad, W: fwd + dgrad, G_Y: dgrad + wgrad) from a
// single HBM read — the quantised copies are what the paper saves for backward.
// Tiles: 128 rows x 128 cols, loaded by TMA as two 128B-swizzled 64-column boxes into a
// 3-stage ring; thread t quantises one row pair-of-blocks and one column pair per tile.
// ------------------------------------------------------------------------------------
struct DualOut {
  uint8_t* q_row; uint8_t* sf_row; const int32_t* row_zero; int nrow_zero; __nv_bfloat16* slice_row;
  uint8_t* q_col; uint8_t* sf_col; const int32_t* col_zero; int ncol_zero; __nv_bfloat16* slice_col;
};

template <bool kSwCvt, int kMinBlocks>
__global__ void __launch_bounds__(256, kMinBlocks) k_iht_quant_dual(const __grid_constant__ CUtensorMap tm, int64_t R,
                                                           int64_t C, const DualOut o) {
  constexpr int TR = 128, TC = 128, kBox = 16384;
  extern __shared__ __align__(1024) uint8_t smem_dual[];
  uint8_t* ring = smem_dual + ((1024u - (ptx::smem_u32(smem_dual) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + kQStages * kQTileBytes);
  const int64_t rtiles = (R + TR - 1) / TR, ctiles = (C + TC - 1) / TC;
  const int64_t ntiles = rtiles * ctiles;
  const int64_t kch_row = sf_kchunks(C), kch_col = sf_kchunks(R);
  SmemMask* mrow = reinterpret_cast<SmemMask*>(full + kQStages);
  SmemMask* mcol = mrow + 1;
  const int tid = threadIdx.x;
  if (tid == 0) {
    ptx::prefetch_tmap(&tm);
    for (int i = 0; i < kQStages; ++i) ptx::mbar_init(&full[i], 1);
    ptx::fence_barrier_init();
  }
  if (o.nrow_zero > 0) mask_build(mrow, o.row_zero, o.nrow_zero, R);
  if (o.ncol_zero > 0) mask_build(mcol, o.col_zero, o.ncol_zero, C);
  __syncthreads();
  const int64_t first = blockIdx.x, stride = gridDim.x;
  auto issue = [&](int64_t tile, int st) {
    // row-tile fastest: consecutive CTAs share the same column strip of the output
    const int64_t rt = tile % rtiles, ct = tile / rtiles;
    ptx::mbar_arrive_expect_tx(&full[st], 2 * kBox);
    uint8_t* dst = ring + st * kQTileBytes;
    ptx::tma_load_2d(dst, &tm, &full[st], int32_t(ct * TC), int32_t(rt * TR));
    ptx::tma_load_2d(dst + kBox, &tm, &full[st], int32_t(ct * TC + 64), int32_t(rt * TR));
  };
  if (tid == 0)
    for (int i = 0; i < kQStages; ++i)
      if (first + i * stride < ntiles) issue(first + i * stride, i);
  int it = 0;
  for (int64_t tile = first; tile < ntiles; tile += stride, ++it) {
    const int st = it % kQStages;
    ptx::mbar_wait(&full[st], uint32_t((it / kQStages) & 1));
    const int64_t rt = tile % rtiles, ct = tile / rtiles;
    const uint8_t* tb = ring + st * kQTileBytes;
    // row part: row rr, the 64 columns of box bx; column part: columns 2cp, 2cp+1, rows
    // rb*32 .. +32. Values are read straight from the swizzled stage into the fp32x2 pairs;
    // the (rare) OE rows/columns copy their raw values to the slice from the stage as well,
    // so no raw copy stays live in registers.
    const int rr = tid & 127, bx = tid >> 7;
    const int cp = tid & 63, rb = tid >> 6;
    const uint8_t* rowp = tb + bx * kBox + rr * 128;
    const int sw = rr & 7;
    uint64_t P[32];
    // ---- row quantisation: stored row r0 + rr, K-blocks kb0, kb0 + 1 along C
    {
      const int64_t r = rt * TR + rr;
      const int64_t kb0 = (ct * TC + bx * 64) / kBlk;
      const bool va = r < R && kb0 * kBlk < C, vb = r < R && (kb0 + 1) * kBlk < C;
      const int s = (o.nrow_zero > 0 && va) ? mask_slot(mrow, o.nrow_zero, r) : -1;
      if (s >= 0) {
        if (o.slice_row) {
          // raw bf16 row segment -> slice (two 64-byte halves, un-swizzled)
          __nv_bfloat16* dst = o.slice_row + int64_t(s) * C + kb0 * kBlk;
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (j < 4 || vb)
              reinterpret_cast<uint4*>(dst)[j] = *reinterpret_cast<const uint4*>(rowp + ((j ^ sw) << 4));
        }
#pragma unroll
        for (int i = 0; i < 32; ++i) P[i] = 0ull;
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint4 ua = *reinterpret_cast<const uint4*>(rowp + ((j ^ sw) << 4));
          const uint4 ub = *reinterpret_cast<const uint4*>(rowp + (((j + 4) ^ sw) << 4));
          P[8 * j + 0] = f2_pack(bf16lo(ua.x), bf16lo(ub.x));
          P[8 * j + 1] = f2_pack(bf16hi(ua.x), bf16hi(ub.x));
          P[8 * j + 2] = f2_pack(bf16lo(ua.y), bf16lo(ub.y));
          P[8 * j + 3] = f2_pack(bf16hi(ua.y), bf16hi(ub.y));
          P[8 * j + 4] = f2_pack(bf16lo(ua.z), bf16lo(ub.z));
          P[8 * j + 5] = f2_pack(bf16hi(ua.z), bf16hi(ub.z));
          P[8 * j + 6] = f2_pack(bf16lo(ua.w), bf16lo(ub.w));
          P[8 * j + 7] = f2_pack(bf16hi(ua.w), bf16hi(ub.w));
        }
      }
      uint4 c0, c1;
      uint32_t s0, s1;
      float ydummy[1];
      iht_quant_pair<false, kSwCvt>(P, c0, c1, s0, s1, ydummy, ydummy);
      if (va) {
        *reinterpret_cast<uint4*>(o.q_row + r * (C / 2) + kb0 * 16) = c0;
        o.sf_row[sf_offset(r, kb0, kch_row)] = uint8_t(s0);
      }
      if (vb) {
        *reinterpret_cast<uint4*>(o.q_row + r * (C / 2) + (kb0 + 1) * 16) = c1;
        o.sf_row[sf_offset(r, kb0 + 1, kch_row)] = uint8_t(s1);
      }
    }
    // ---- column quantisation: stored rows c0 + 2cp, +1; K-block rb along R
    const int64_t ca = ct * TC + 2 * cp, cb2 = ca + 1;
    const int64_t kbc = (rt * TR) / kBlk + rb;
    const bool cva = ca < C && kbc * kBlk < R, cvb = cb2 < C && kbc * kBlk < R;
    {
      const int ccol = (2 * cp) & 63;
      const uint8_t* box = tb + ((2 * cp) >> 6) * kBox + rb * 32 * 128 + ((ccol * 2) & 15);
      const int chunk = (ccol * 2) >> 4;
      const int sa = (o.ncol_zero > 0 && cva) ? mask_slot(mcol, o.ncol_zero, ca) : -1;
      const int sb = (o.ncol_zero > 0 && cvb) ? mask_slot(mcol, o.ncol_zero, cb2) : -1;
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const uint32_t w = *reinterpret_cast<const uint32_t*>(box + i * 128 + ((chunk ^ (i & 7)) << 4));
        P[i] = f2_pack(bf16lo(w), bf16hi(w));
      }
      if (sa >= 0 || sb >= 0) {
        float x[32];
        if (sa >= 0) {
#pragma unroll
          for (int i = 0; i < 32; ++i) x[i] = f2_lo(P[i]);
          if (o.slice_col) store_slice32(o.slice_col + int64_t(sa) * R + kbc * kBlk, x);
        }
        if (sb >= 0) {
#pragma unroll
          for (int i = 0; i < 32; ++i) x[i] = f2_hi(P[i]);
          if (o.slice_col) store_slice32(o.slice_col + int64_t(sb) * R + kbc * kBlk, x);
        }
#pragma unroll
        for (int i = 0; i < 32; ++i) P[i] = f2_pack(sa >= 0 ? 0.f : f2_lo(P[i]), sb >= 0 ? 0.f : f2_hi(P[i]));
      }
    }
    __syncthreads();                                   // stage consumed by every thread
    if (tid == 0 && tile + kQStages * stride < ntiles) issue(tile + kQStages * stride, st);
    {
      uint4 c0, c1;
      uint32_t s0, s1;
      float ydummy[1];
      iht_quant_pair<false, kSwCvt>(P, c0, c1, s0, s1, ydummy, ydummy);
      if (cva) {
        *reinterpret_cast<uint4*>(o.q_col + ca * (R / 2) + kbc * 16) = c0;
        o.sf_col[sf_offset(ca, kbc, kch_col)] = uint8_t(s0);
      }
      if (cvb) {
        *reinterpret_cast<uint4*>(o.q_col + cb2 * (R / 2) + kbc * 16) = c1;
        o.sf_col[sf_offset(cb2, kbc, kch_col)] = uint8_t(s1);
      }
    }
  }
}

thread_local int g_quant_launches = 0;
int quant_last_launches() { return g_quant_launches; }

cudaError_t launch_iht_quant_dual(const __nv_bfloat16* in, int64_t R, int64_t C, int64_t ld,
                                  const int32_t* row_zero, int nrow_zero, __nv_bfloat16* slice_row,
                                  uint8_t* q_row, uint8_t* sf_row, const int32_t* col_zero, int ncol_zero,
                                  __nv_bfloat16* slice_col, uint8_t* q_col, uint8_t* sf_col, int num_sms,
                                  cudaStream_t st) {
  g_quant_launches = 1;
  if (quant_use_tc() && quant_tc_supported(R, C, ld, in, nrow_zero > 0, ncol_zero > 0)) {
    const QuantTcJob q{in, R, C, ld, row_zero, nrow_zero, slice_row, q_row, sf_row, nullptr,
                       col_zero, ncol_zero, slice_col, q_col, sf_col, nullptr};
    g_quant_launches = 0;
    return launch_quant_tc_multi(&q, 1, num_sms, st, &g_quant_launches, nullptr);
  }
  if ((ld * 2) % 16 != 0 || (reinterpret_cast<uintptr_t>(in) & 15) != 0) return cudaErrorInvalidValue;
  CUtensorMap tm;
  if (!make_tmap_2d(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, in, uint64_t(C), uint64_t(R), uint64_t(ld) * 2, 64,
                    128, CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;
  DualOut o{q_row, sf_row, row_zero, nrow_zero, slice_row, q_col, sf_col, col_zero, ncol_zero, slice_col};
  const size_t smem = size_t(kQStages) * kQTileBytes + 1024 + 64 +
                      ((nrow_zero > 0 || ncol_zero > 0) ? 2 * sizeof(SmemMask) : 0);
  if ((nrow_zero > 0 && R > kMaskMaxRows) || (ncol_zero > 0 && C > kMaskMaxRows)) return cudaErrorInvalidValue;
  static const int occ = knob("ADAHOP_DUAL_OCC", 2);
  static std::atomic<uint64_t> attr{0};
  cudaError_t ae = once_per_device(attr, [] {
    const int mx = int(size_t(kQStages) * kQTileBytes + 1024 + 64 + 2 * sizeof(SmemMask));
    cudaError_t e = cudaFuncSetAttribute(k_iht_quant_dual<false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_iht_quant_dual<false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    return e;
  });
  if (ae != cudaSuccess) return ae;
  const int64_t ntiles = ((R + 127) / 128) * ((C + 127) / 128);
  const int64_t cap = int64_t(num_sms) * occ;
  const unsigned grid = unsigned(ntiles < cap ? ntiles : cap);
  if (occ == 1) k_iht_quant_dual<false, 1><<<grid, 256, smem, st>>>(tm, R, C, o);
  else k_iht_quant_dual<false, 2><<<grid, 256, smem, st>>>(tm, R, C, o);
  return cudaGetLastError();
}

// Generic transposing variant for sources whose row pitch is not 16-byte aligned (TMA
// cannot address them): one 64(k) x 256(r) tile per CTA through dynamic shared memory.
template <typename T, bool kHad, bool kSwCvt>
__global__ void __launch_bounds__(256) k_iht_quant_col_generic(const T* __restrict__ in, int64_t R,
                                                               int64_t K, int64_t ld,
                                                               const int32_t* __restrict__ zero_rows,
                                                               int nzero, uint8_t* __restrict__ codes,
                                                               uint8_t* __restrict__ sf, int64_t kchunks,
                                                               float* __restrict__ had_out,
                                                               __nv_bfloat16* __restrict__ slice) {
  constexpr int TK = 64, TR = 256;
  extern __shared__ __align__(1024) uint8_t smem_gen[];
  T* tile = reinterpret_cast<T*>(smem_gen);
  const int64_t r0 = int64_t(blockIdx.x) * TR, k0 = int64_t(blockIdx.y) * TK;
  for (int v = threadIdx.x; v < TK * TR; v += blockDim.x) {
    const int kr = v / TR, c = v % TR;
    const bool ok = (k0 + kr < K) && (r0 + c < R);
    tile[kr * TR + c] = ok ? in[(k0 + kr) * ld + r0 + c] : T(0.f);
  }
  __syncthreads();
  const int p = threadIdx.x % (TR / 2), kbl = threadIdx.x / (TR / 2);
  const int64_t r = r0 + 2 * p, kb = k0 / kBlk + kbl;
  const bool va = r < R && kb * kBlk < K, vb = r + 1 < R && kb * kBlk < K;
  if (!va && !vb) return;
  float xa[32], xb[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    xa[i] = float(tile[(kbl * 32 + i) * TR + 2 * p]);
    xb[i] = float(tile[(kbl * 32 + i) * TR + 2 * p + 1]);
  }
  if (nzero > 0) {
    const int sa = va ? find_sorted(zero_rows, nzero, r) : -1;
    const int sb = vb ? find_sorted(zero_rows, nzero, r + 1) : -1;
    if (sa >= 0) {
      if (slice) store_slice32(slice + int64_t(sa) * K + kb * kBlk, xa);
#pragma unroll
      for (int i = 0; i < 32; ++i) xa[i] = 0.f;
    }
    if (sb >= 0) {
      if (slice) store_slice32(slice + int64_t(sb) * K + kb * kBlk, xb);
#pragma unroll
      for (int i = 0; i < 32; ++i) xb[i] = 0.f;
    }
  }
  uint64_t P[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) P[i] = f2_pack(xa[i], xb[i]);
  uint4 c0, c1;
  uint32_t s0, s1;
  float ya[kHad ? 32 : 1], yb[kHad ? 32 : 1];
  iht_quant_pair<kHad, kSwCvt>(P, c0, c1, s0, s1, ya, yb);
  if (kHad) {
    if (va) store_f32x32(had_out + r * K + kb * kBlk, ya);
    if (vb) store_f32x32(had_out + (r + 1) * K + kb * kBlk, yb);
  }
  if (va) {
    *reinterpret_cast<uint4*>(codes + r * (K / 2) + kb * 16) = c0;
    sf[sf_offset(r, kb, kchunks)] = uint8_t(s0);
  }
  if (vb) {
    *reinterpret_cast<uint4*>(codes + (r + 1) * (K / 2) + kb * 16) = c1;
    sf[sf_offset(r + 1, kb, kchunks)] = uint8_t(s1);
  }
}

// ------------------------------------------------------------------------ launchers
template <typename T, bool kHad, bool kSw>
static cudaError_t launch_quant_t(const T* in, int64_t R, int64_t K, int64_t ld, int kstrided,
                                  const int32_t* zero_rows, int nzero, uint8_t* codes, uint8_t* sf,
                                  float* had_out, __nv_bfloat16* slice, int num_sms, cudaStream_t st) {
  const int64_t kch = sf_kchunks(K);
  const bool tma_ok = sizeof(T) == 2 && (ld * 2) % 16 == 0 && (reinterpret_cast<uintptr_t>(in) & 15) == 0 &&
                      (nzero == 0 || R <= kMaskMaxRows);
  if (tma_ok) {
    CUtensorMap tm;
    bool ok;
    int64_t ntiles;
    if (kstrided) {   // [K][R] source, box 128 rows(r) x 128 k
      ok = make_tmap_2d(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, in, uint64_t(R), uint64_t(K), uint64_t(ld) * 2,
                        128, 128, CU_TENSOR_MAP_SWIZZLE_NONE);
      ntiles = ((R + 127) / 128) * ((K + 127) / 128);
    } else {          // [R][K] source, box 64 k x 256 rows, 128B swizzle
      ok = make_tmap_2d(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, in, uint64_t(K), uint64_t(R), uint64_t(ld) * 2,
                        64, 256, CU_TENSOR_MAP_SWIZZLE_128B);
      ntiles = ((R + 255) / 256) * ((K + 63) / 64);
    }
    if (!ok || R > kMaskMaxRows) return cudaErrorInvalidValue;
    const size_t smem = size_t(kQStages) * kQTileBytes + 1024 + 64 + (nzero > 0 ? sizeof(SmemMask) : 0);
    static std::atomic<uint64_t> attr{0};
    cudaError_t ae = once_per_device(attr, [] {
      const int mx = int(size_t(kQStages) * kQTileBytes + 1024 + 64 + sizeof(SmemMask));
      cudaError_t e = cudaFuncSetAttribute(k_iht_quant_tma<true, kHad, kSw>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_iht_quant_tma<false, kHad, kSw>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
      return e;
    });
    if (ae != cudaSuccess) return ae;
    const int64_t cap = int64_t(num_sms) * 2;   // two persistent CTAs per SM
    const unsigned grid = unsigned(ntiles < cap ? ntiles : cap);
    if (kstrided)
      k_iht_quant_tma<true, kHad, kSw><<<grid, 256, smem, st>>>(tm, R, K, zero_rows, nzero, codes, sf, kch,
                                                                 had_out, slice);
    else
      k_iht_quant_tma<false, kHad, kSw><<<grid, 256, smem, st>>>(tm, R, K, zero_rows, nzero, codes, sf, kch,
                                                                  had_out, slice);
  } else if (!kstrided) {
    const int64_t total = R * ((K / kBlk + 1) / 2);
    const int64_t want = (total + 255) / 256;
    const int64_t cap = int64_t(num_sms) * 8;   // grid-stride
    k_iht_quant_row<T, kHad, kSw><<<unsigned(want < cap ? want : cap), 256, 0, st>>>(
        in, R, K, ld, zero_rows, nzero, codes, sf, kch, had_out, slice);
  } else {
    const size_t smem = size_t(64) * 256 * sizeof(T);
    static std::atomic<uint64_t> attr_g{0};
    cudaError_t ae = once_per_device(attr_g, [smem] {
      return cudaFuncSetAttribute(k_iht_quant_col_generic<T, kHad, kSw>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(smem));
    });
    if (ae != cudaSuccess) return ae;
    dim3 grid(unsigned((R + 255) / 256), unsigned((K + 63) / 64));
    k_iht_quant_col_generic<T, kHad, kSw><<<grid, 256, smem, st>>>(in, R, K, ld, zero_rows, nzero, codes,
                                                                    sf, kch, had_out, slice);
  }
  return cudaGetLastError();
}

bool quant_use_tc() {
  static const bool tc = knob("ADAHOP_QUANT_SCALAR", 0) == 0;   // experiment builds: 1 selects the butterfly kernels
  return tc;
}

cudaError_t launch_iht_quant(const void* in, bool in_f32, int64_t R, int64_t K, int64_t ld,
                             int kstrided, const int32_t* zero_rows, int nzero, uint8_t* codes,
                             uint8_t* sf, float* had_out, __nv_bfloat16* slice, bool sw_cvt,
                             int num_sms, cudaStream_t st) {
  g_quant_launches = 1;
  if (!in_f32 && !sw_cvt && quant_use_tc()) {
    const __nv_bfloat16* src = static_cast<const __nv_bfloat16*>(in);
    if (!kstrided && quant_tc_supported(R, K, ld, in, nzero > 0, false)) {   // T = [R][K], row orientation
      const QuantTcJob q{src, R, K, ld, zero_rows, nzero, slice, codes, sf, had_out,
                         nullptr, 0, nullptr, nullptr, nullptr, nullptr};
      g_quant_launches = 0;
      return launch_quant_tc_multi(&q, 1, num_sms, st, &g_quant_launches, nullptr);
    }
    if (kstrided && quant_tc_supported(K, R, ld, in, false, nzero > 0)) {   // T = [K][R], column orientation
      const QuantTcJob q{src, K, R, ld, nullptr, 0, nullptr, nullptr, nullptr, nullptr,
                         zero_rows, nzero, slice, codes, sf, had_out};
      g_quant_launches = 0;
      return launch_quant_tc_multi(&q, 1, num_sms, st, &g_quant_launches, nullptr);
    }
  }
#define ADAHOP_Q(T, H, S)                                                                   \
  return launch_quant_t<T, H, S>(static_cast<const T*>(in), R, K, ld, kstrided, zero_rows, \
                                 nzero, codes, sf, had_out, slice, num_sms, st)
  const bool had = had_out != nullptr;
  if (in_f32) {
    if (had) { if (sw_cvt) ADAHOP_Q(float, true, true); else ADAHOP_Q(float, true, false); }
    else { if (sw_cvt) ADAHOP_Q(float, false, true); else ADAHOP_Q(float, false, false); }
  } else {
    if (had) { if (sw_cvt) ADAHOP_Q(__nv_bfloat16, true, true); else ADAHOP_Q(__nv_bfloat16, true, false); }
    else { if (sw_cvt) ADAHOP_Q(__nv_bfloat16, false, true); else ADAHOP_Q(__nv_bfloat16, false, false); }
  }
#undef ADAHOP_Q
}

// ================================================================== layout converters
__global__ void k_sf_to_canonical(const uint8_t* __restrict__ sf, int64_t R, int64_t K,
                                  uint8_t* __restrict__ canon) {
  const int64_t nkb = K / kBlk;
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= R * nkb) return;
  const int64_t r = t / nkb, kb = t - r * nkb;
  canon[t] = sf[sf_offset(r, kb, sf_kchunks(K))];
}
__global__ void k_sf_from_canonical(const uint8_t* __restrict__ canon, int64_t R, int64_t K,
                                    uint8_t* __restrict__ sf) {
  const int64_t nkb = K / kBlk;
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= R * nkb) return;
  const int64_t r = t / nkb, kb = t - r * nkb;
  sf[sf_offset(r, kb, sf_kchunks(K))] = canon[t];
}
cudaError_t launch_sf_convert(const uint8_t* src, int64_t R, int64_t K, uint8_t* dst,
                              bool to_canonical, cudaStream_t st) {
  const int64_t n = R * (K / kBlk);
  const unsigned blocks = unsigned((n + 255) / 256);
  if (to_canonical) k_sf_to_canonical<<<blocks, 256, 0, st>>>(src, R, K, dst);
  else k_sf_from_canonical<<<blocks, 256, 0, st>>>(src, R, K, dst);
  return cudaGetLastError();
}

// ================================================================== FOID
// Key of stored row r: population variance of its first p K-elements, fp64, summed
// sequentially with separate multiply and add (no FMA), matching the oracle bitwise.
__device__ __forceinline__ double foid_key_seq(const float* x, int p) {
  double s = 0.0;
  for (int j = 0; j < p; ++j) s = __dadd_rn(s, double(x[j]));
  const double mu = s / double(p);
  double v = 0.0;
  for (int j = 0; j < p; ++j) {
    const double d = __dsub_rn(double(x[j]), mu);
    v = __dadd_rn(v, __dmul_rn(d, d));
  }
  return v / double(p);
}

constexpr int kProbeMax = 64;  // probe lengths above this take the generic path

// K-strided operand (stored row r = column r of a [K][R] array): the probe is the first p
// rows of the source, read coalesced (thread per r).
// K-contiguous operand: a warp stages the probes of its 32 rows into shared memory with
// 16-byte loads, then each lane folds its own row.
template <typename T>
__device__ __forceinline__ void foid_keys_block(const T* __restrict__ in, int64_t R, int64_t ld, int kstrided, int p,
                                                double* __restrict__ keys, int bid) {
  __shared__ __align__(16) float stage[4][32][kProbeMax + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r = int64_t(bid) * blockDim.x + threadIdx.x;
  if (p > kProbeMax) {  // generic (slow) path
    if (r >= R) return;
    double s = 0.0;
    for (int j = 0; j < p; ++j)
      s = __dadd_rn(s, double(load_as_float(in, kstrided ? int64_t(j) * ld + r : r * ld + j)));
    const double mu = s / double(p);
    double v = 0.0;
    for (int j = 0; j < p; ++j) {
      const double d = __dsub_rn(double(load_as_float(in, kstrided ? int64_t(j) * ld + r : r * ld + j)), mu);
      v = __dadd_rn(v, __dmul_rn(d, d));
    }
    keys[r] = v / double(p);
    return;
  }
  float* mine = stage[warp][lane];
  if (kstrided) {
    if (r < R) {
      if (p == kProbeMax) {
        float x[kProbeMax];  // all loads issued before the first use (no serialised latency)
#pragma unroll
        for (int j = 0; j < kProbeMax; ++j) x[j] = load_as_float(in, int64_t(j) * ld + r);
        keys[r] = foid_key_seq(x, kProbeMax);
        return;
      }
#pragma unroll 16
      for (int j = 0; j < p; ++j) mine[j] = load_as_float(in, int64_t(j) * ld + r);
    }
  } else {
    const int64_t rw = int64_t(bid) * blockDim.x + warp * 32;  // first row of this warp
    if (sizeof(T) == 2 && p == 64 && ((ld * 2) % 16) == 0 && ((reinterpret_cast<uintptr_t>(in) & 15) == 0)) {
      // 32 rows x 128 B: 256 16-byte chunks, 8 per lane, 8 lanes per row -> full lines
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int c = lane + 32 * i, rr = c >> 3, c8 = (c & 7) * 8;
        if (rw + rr < R) {
          const uint4 u = __ldg(reinterpret_cast<const uint4*>(in + (rw + rr) * ld + c8));
          const uint32_t wv[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            stage[warp][rr][c8 + 2 * t] = __uint_as_float(wv[t] << 16);
            stage[warp][rr][c8 + 2 * t + 1] = __uint_as_float(wv[t] & 0xFFFF0000u);
          }
        }
      }
    } else {
      // cooperative: lane handles element (row = rw + e / p, col = e % p), e strided by 32
      for (int e = lane; e < 32 * p; e += 32) {
        const int rr = e / p, c = e % p;
        if (rw + rr < R) stage[warp][rr][c] = load_as_float(in, (rw + rr) * ld + c);
      }
    }
    __syncwarp();
  }
  if (r < R) keys[r] = foid_key_seq(mine, p);
}

template <typename T>
__global__ void __launch_bounds__(128) k_foid_keys(const T* __restrict__ in, int64_t R, int64_t ld, int kstrided,
                                                   int p, double* __restrict__ keys) {
  foid_keys_block(in, R, ld, kstrided, p, keys, blockIdx.x);
}

// A batch of FOID jobs (the OE operands of one linear): one keys launch and one select launch
// for all of them. Job j owns key blocks [kb_off[j], kb_off[j+1]) and select blocks
// [sb_off[j], sb_off[j+1]).
struct FoidJobDev {
  const void* in; int64_t R, ld; int kstrided, p, k; double* scratch; int32_t* idx;
};
struct FoidBatchDev {
  FoidJobDev j[kFoidMaxJobs];
  int n;
  int rows_per_block;   // select: rows ranked per CTA (1024 .. 4096)
  int kb_off[kFoidMaxJobs + 1], sb_off[kFoidMaxJobs + 1];
};
__device__ __forceinline__ int foid_job_of(const int* off, int n, int b) {
  int j = 0;
  while (j + 1 < n && b >= off[j + 1]) ++j;
  return j;
}
__device__ __forceinline__ unsigned* foid_counter(const FoidJobDev& J) {
  const int64_t nb = (J.R + 1023) / 1024;
  return reinterpret_cast<unsigned*>(reinterpret_cast<uint8_t*>(J.scratch) + J.R * 8 + nb * 256 * 12);
}

template <typename T>
__global__ void __launch_bounds__(128) k_foid_keys_batch(const __grid_constant__ FoidBatchDev B) {
  ptx::griddep_launch();
  ptx::griddep_wait();
  const int jb = foid_job_of(B.kb_off, B.n, blockIdx.x);
  const FoidJobDev& J = B.j[jb];
  const int bid = blockIdx.x - B.kb_off[jb];
  if (bid == 0 && threadIdx.x == 0) *foid_counter(J) = 0u;   // for k_foid_select
  foid_keys_block(static_cast<const T*>(J.in), J.R, J.ld, J.kstrided, J.p, J.scratch, bid);
}

// Top-k by (key desc, index asc), written as ascending indices. Keys come from k_foid_keys.
// The selection never sorts all R keys. topk_core selects the kk best of n <= 4096 pairs in
// one CTA of 1024 threads:
//  1. thread t holds entries t, t + 1024, ... (E <= 4); the 8 threads 8g..8g+7 form group g
//     (128 groups) and find the group maximum in the total order (key desc, index asc);
//  2. L = the kk-th largest group maximum (each maximum ranked by its 8 threads against all
//     maxima). At least kk entries (those maxima) are >= L, so every top-kk entry is >= L; an
//     entry >= L lies in a group whose maximum is >= L, so at most kk * 8E entries are >= L;
//  3. the entries >= L are compacted into shared memory and ranked exactly among themselves.
// k_foid_select runs it per block of up to 4096 rows (rows -> the block's kk best), and the last block
// to finish runs it again over the blocks' nb * kk survivors. Keys are fp64 >= 0, so their
// bit patterns order like the values; the index breaks ties, so the selected set is unique.
constexpr int kTopkThreads = 1024;
// rows per select block (<= 4 per thread, topk_core's bound): 4096 — most OE operands (d_in or
// d_out = 2048 stored rows) then need one block and no merge (FOID stage 0.133 -> 0.118 ms per
// Llama-3.2-1B layer step). ADAHOP_FOID_BLOCK_ROWS = 1024 / 2048 for comparison.
static int foid_block_rows() {
  static const int v = [] {
    const int r = knob("ADAHOP_FOID_BLOCK_ROWS", 4096);
    return r == 1024 || r == 2048 ? r : 4096;
  }();
  return v;
}
constexpr int kTopkGroupLanes = 8;
constexpr int kTopkGroups = kTopkThreads / kTopkGroupLanes;
constexpr int kTopkMaxPer = 4;                                   // n <= 4096
constexpr int kTopkMaxCand = 256 * kTopkGroupLanes * kTopkMaxPer; // kk * 8E bound

__device__ __forceinline__ bool foid_before(unsigned long long ka, int ia, unsigned long long kb, int ib) {
  return ka > kb || (ka == kb && ia < ib);
}

struct TopkSmem {
  unsigned long long gmk[kTopkGroups];
  int gmi[kTopkGroups];
  unsigned long long lk;
  int li, nc, last;
};

// Entries come from (src_key[e], src_idx ? src_idx[e] : idx0 + e), e < n. Writes the kk best
// in rank order to sel_key / sel_idx (shared or global) — rank r at position r.
__device__ void topk_core(const unsigned long long* __restrict__ src_key, const int* __restrict__ src_idx, int idx0,
                          int n, int kk, TopkSmem& sm, unsigned long long* ckey, int* cidx,
                          unsigned long long* sel_key, int* sel_idx) {
  const int tid = threadIdx.x;
  const int E = (n + kTopkThreads - 1) / kTopkThreads;
  const int NG = min(kTopkGroups, (n + kTopkGroupLanes - 1) / kTopkGroupLanes);   // groups with entries
  const int g = tid / kTopkGroupLanes, qq = tid % kTopkGroupLanes;
  unsigned long long k[kTopkMaxPer];
  int x[kTopkMaxPer];
#pragma unroll
  for (int j = 0; j < kTopkMaxPer; ++j) {
    const int e = j * kTopkThreads + tid;
    const bool ok = j < E && e < n;
    k[j] = ok ? src_key[e] : 0ull;
    x[j] = ok ? (src_idx ? src_idx[e] : idx0 + e) : 0x7FFFFFFF;
  }
  unsigned long long mk = 0;
  int mi = 0x7FFFFFFF;
#pragma unroll
  for (int j = 0; j < kTopkMaxPer; ++j)
    if (foid_before(k[j], x[j], mk, mi)) { mk = k[j]; mi = x[j]; }
#pragma unroll
  for (int o = 1; o < kTopkGroupLanes; o <<= 1) {
    const unsigned long long ok = __shfl_xor_sync(0xffffffffu, mk, o);
    const int oi = __shfl_xor_sync(0xffffffffu, mi, o);
    if (foid_before(ok, oi, mk, mi)) { mk = ok; mi = oi; }
  }
  if (qq == 0) { sm.gmk[g] = mk; sm.gmi[g] = mi; }
  if (tid == 0) sm.nc = 0;
  __syncthreads();
  if (kk <= NG) {
    int rank = 0;
    if (g < NG)
      for (int u = qq; u < NG; u += kTopkGroupLanes) rank += foid_before(sm.gmk[u], sm.gmi[u], mk, mi);
#pragma unroll
    for (int o = 1; o < kTopkGroupLanes; o <<= 1) rank += __shfl_xor_sync(0xffffffffu, rank, o);
    if (qq == 0 && g < NG && rank == kk - 1) { sm.lk = mk; sm.li = mi; }
  } else if (tid == 0) {
    sm.lk = 0; sm.li = 0x7FFFFFFF;   // fewer groups than kk: every entry is a candidate
  }
  __syncthreads();
  const unsigned long long lk = sm.lk;
  const int li = sm.li;
#pragma unroll
  for (int j = 0; j < kTopkMaxPer; ++j) {
    if (j >= E) break;
    const bool c = j * kTopkThreads + tid < n && !foid_before(lk, li, k[j], x[j]);   // >= L
    const unsigned m = __ballot_sync(0xffffffffu, c);
    if (m) {
      int wbase = 0;
      if ((tid & 31) == 0) wbase = atomicAdd(&sm.nc, __popc(m));
      wbase = __shfl_sync(0xffffffffu, wbase, 0);
      if (c) {
        const int pos = wbase + __popc(m & ((1u << (tid & 31)) - 1u));
        ckey[pos] = k[j];
        cidx[pos] = x[j];
      }
    }
  }
  __syncthreads();
  const int nc = sm.nc;
  // rank of candidate c: a team of 8 lanes (the group lanes) splits the comparisons
  const int ncr = (nc + kTopkGroups - 1) / kTopkGroups * kTopkGroups;   // uniform trip count per warp
  for (int c = g; c < ncr; c += kTopkGroups) {
    const bool live = c < nc;
    const unsigned long long a = live ? ckey[c] : 0ull;
    const int ai = live ? cidx[c] : 0;
    int rank = 0;
    if (live)
      for (int u = qq; u < nc; u += kTopkGroupLanes) rank += foid_before(ckey[u], cidx[u], a, ai);
#pragma unroll
    for (int o = 1; o < kTopkGroupLanes; o <<= 1) rank += __shfl_xor_sync(0xffffffffu, rank, o);
    if (live && qq == 0 && rank < kk) { sel_key[rank] = a; sel_idx[rank] = ai; }
  }
  __syncthreads();
}

#ifndef FOID_TRACE
#define FOID_TRACE 0
#endif
#if FOID_TRACE
__device__ __forceinline__ long long gtime() { long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
#endif
__global__ void __launch_bounds__(kTopkThreads) k_foid_select(const __grid_constant__ FoidBatchDev B) {
  ptx::griddep_launch();
  ptx::griddep_wait();
#if FOID_TRACE
  const long long t0 = gtime();
#endif
  extern __shared__ __align__(16) unsigned long long ckey[];   // [kTopkMaxCand] keys, then indices
  int* cidx = reinterpret_cast<int*>(ckey + kTopkMaxCand);
  __shared__ TopkSmem sm;
  __shared__ int fidx[256];
  const int jb = foid_job_of(B.sb_off, B.n, blockIdx.x);
  const FoidJobDev& J = B.j[jb];
  const int R = int(J.R), kk = J.k;
  const int nb = B.sb_off[jb + 1] - B.sb_off[jb], b = blockIdx.x - B.sb_off[jb], tid = threadIdx.x;
  unsigned long long* part_key = reinterpret_cast<unsigned long long*>(J.scratch + R);
  int* part_idx = reinterpret_cast<int*>(part_key + size_t(nb) * 256);
  unsigned* counter = foid_counter(J);
  const int rows_per = B.rows_per_block;
  const int n_b = min(rows_per, R - b * rows_per);
  const int kb = min(kk, n_b);
  const unsigned long long* keys = reinterpret_cast<const unsigned long long*>(J.scratch);
  // this block's kb best rows (padding up to kk with entries that rank after every row)
  topk_core(keys + int64_t(b) * rows_per, nullptr, b * rows_per, n_b, kb, sm, ckey, cidx,
            part_key + int64_t(b) * kk, part_idx + int64_t(b) * kk);
  for (int t = kb + tid; t < kk; t += kTopkThreads) { part_key[int64_t(b) * kk + t] = 0ull; part_idx[int64_t(b) * kk + t] = 0x7FFFFFFF; }
#if FOID_TRACE
  const long long t1 = gtime();
  const int nc1 = sm.nc;
#endif
  if (nb == 1) {
    if (tid < kk) fidx[tid] = part_idx[tid];
  } else {
    __threadfence();
    __syncthreads();
    if (tid == 0) sm.last = atomicAdd(counter, 1u) == unsigned(nb - 1);
    __syncthreads();
    if (!sm.last) return;
    __threadfence();
#if FOID_TRACE
    const long long t2 = gtime();
#endif
    // merge: the nb lists are each sorted; merge them pairwise (log2 nb levels), keeping the
    // first kk of every merge. An entry at position p of one list lands at p + (entries of the
    // partner list before it), found by binary search.
    unsigned long long* ka = ckey;
    int* xa = cidx;
    unsigned long long* kb2 = ckey + 4096;
    int* xb = cidx + 4096;
    for (int e = tid; e < nb * kk; e += kTopkThreads) { ka[e] = __ldcg(part_key + e); xa[e] = __ldcg(part_idx + e); }
    __syncthreads();
    for (int m = nb; m > 1; m = (m + 1) >> 1) {
      for (int e = tid; e < m * kk; e += kTopkThreads) {
        const int l = e / kk, pe = e - l * kk;
        const int q = l >> 1;
        if (l == m - 1 && (m & 1)) {   // odd list out: carried over unchanged
          kb2[q * kk + pe] = ka[e]; xb[q * kk + pe] = xa[e];
          continue;
        }
        const int other = (l ^ 1) * kk;
        const unsigned long long a = ka[e];
        const int ai = xa[e];
        int lo = 0, hi = kk;   // entries of the partner list before (a, ai)
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (foid_before(ka[other + mid], xa[other + mid], a, ai)) lo = mid + 1; else hi = mid;
        }
        const int pos = pe + lo;
        if (pos < kk) { kb2[q * kk + pos] = a; xb[q * kk + pos] = ai; }
      }
      __syncthreads();
      unsigned long long* tk = ka; ka = kb2; kb2 = tk;
      int* tx = xa; xa = xb; xb = tx;
    }
    for (int t = tid; t < kk; t += kTopkThreads) fidx[t] = xa[t];
#if FOID_TRACE
    if (tid == 0) printf("select b=%d: start %lld phaseL %lld (nc %d) merge-start %lld end %lld\n", b, t0 % 100000000, t1 - t0, nc1, t2 - t0, gtime() - t0);
#endif
  }
  __syncthreads();
  const int kkr = min(kk, R);
  if (tid < kkr) {   // ascending index order
    const int v = fidx[tid];
    int pos = 0;
    for (int u = 0; u < kkr; ++u) pos += fidx[u] < v;
    J.idx[pos] = v;
  }
}

// scratch: keys [R] f64 | survivors [nb * 256] (u64 key, i32 index) | counter
size_t foid_ws_bytes(int64_t R) {
  const int64_t nb = (R + kTopkThreads - 1) / kTopkThreads;
  return size_t(R) * 8 + size_t(nb) * 256 * 12 + 64;
}

cudaError_t launch_foid_batch(const FoidJob* jobs, int n, bool in_f32, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  if (n > kFoidMaxJobs) return cudaErrorInvalidValue;
  FoidBatchDev B{};
  B.n = n;
  B.rows_per_block = foid_block_rows();
  B.kb_off[0] = B.sb_off[0] = 0;
  for (int i = 0; i < n; ++i) {
    const FoidJob& J = jobs[i];
    if (J.R > kFoidMaxRows || J.R <= 0 || J.k <= 0 || J.k > 256) return cudaErrorInvalidValue;
    // the merge keeps every block's k survivors in 4096 shared-memory slots
    if ((J.R + B.rows_per_block - 1) / B.rows_per_block * J.k > 4096 && J.R > B.rows_per_block)
      return cudaErrorInvalidValue;
    B.j[i] = FoidJobDev{J.in, J.R, J.ld, J.kstrided, int(std::min<int64_t>(J.probe, J.K)), J.k, J.scratch, J.idx};
    B.kb_off[i + 1] = B.kb_off[i] + int((J.R + 127) / 128);
    B.sb_off[i + 1] = B.sb_off[i] + int((J.R + B.rows_per_block - 1) / B.rows_per_block);
  }
  // ADAHOP_FOID_PDL (experiment builds): 1 = the keys launch with programmatic dependent launch,
  // 2 = both launches; default 0 (early-resident select CTAs measured slower in round 1)
  static const int pdl = knob("ADAHOP_FOID_PDL", 0);
  if (pdl >= 1) {
    cudaError_t e = in_f32 ? launch_k(k_foid_keys_batch<float>, dim3(B.kb_off[n]), dim3(128), 0, st, 1, B)
                           : launch_k(k_foid_keys_batch<__nv_bfloat16>, dim3(B.kb_off[n]), dim3(128), 0, st, 1, B);
    if (e != cudaSuccess) return e;
  } else if (in_f32) {
    k_foid_keys_batch<float><<<B.kb_off[n], 128, 0, st>>>(B);
  } else {
    k_foid_keys_batch<__nv_bfloat16><<<B.kb_off[n], 128, 0, st>>>(B);
  }
  static std::atomic<uint64_t> attr{0};
  cudaError_t ae = once_per_device(attr, [] {
    return cudaFuncSetAttribute(k_foid_select, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kTopkMaxCand * 12));
  });
  if (ae != cudaSuccess) return ae;
  if (pdl >= 2)
    return launch_k(k_foid_select, dim3(B.sb_off[n]), dim3(kTopkThreads), size_t(kTopkMaxCand) * 12, st, 1, B);
  k_foid_select<<<B.sb_off[n], kTopkThreads, size_t(kTopkMaxCand) * 12, st>>>(B);
  return cudaGetLastError();
}

cudaError_t launch_foid(const void* in, bool in_f32, int64_t R, int64_t K, int64_t ld,
                        int kstrided, int k, int probe, double* keys, int32_t* idx_sorted,
                        cudaStream_t st) {
  const FoidJob J{in, R, K, ld, kstrided, k, probe, keys, idx_sorted};
  return launch_foid_batch(&J, 1, in_f32, st);
}

cudaError_t launch_foid_keys_only(const void* in, bool in_f32, int64_t R, int64_t K, int64_t ld, int kstrided,
                                  int probe, double* keys, cudaStream_t st) {
  const int p = int(std::min<int64_t>(probe, K));
  const unsigned kb = unsigned((R + 127) / 128);
  if (in_f32) k_foid_keys<float><<<kb, 128, 0, st>>>(static_cast<const float*>(in), R, ld, kstrided, p, keys);
  else k_foid_keys<__nv_bfloat16><<<kb, 128, 0, st>>>(static_cast<const __nv_bfloat16*>(in), R, ld, kstrided, p, keys);
  return cudaGetLastError();
}

bool dual_quant_supported(int64_t R, int64_t C, bool row_mask, bool col_mask) {
  return (!row_mask || R <= kMaskMaxRows) && (!col_mask || C <= kMaskMaxRows);
}

int foid_launches(int64_t, int64_t, int) { return 2; }

// ================================================================== calibration stats
// One pass over T [R x C] for both statistics (App. A: per-row and per-column
// sum x, sum x^2, sum |x|, max |x|). Block (cb, chunk) covers columns [256 cb, +256) and rows
// [rb chunk, +rb) (rb = stats_rb: 64..512, two waves of blocks) in tiles of 64 rows staged in shared memory by coalesced 16-byte
// loads; then thread t accumulates column t down the tile, and 4 threads per row accumulate 64
// columns each (combined by two xor shuffles). Sums are fp64 (max is exact in fp32); every
// reduction runs in a fixed order, so the result is deterministic.
//   row partial  rpart[cb][r]      col partial  cpart[chunk][c]
// k_stats_reduce folds them (cb, then chunk, ascending) into rs[R][4] and cs[C][4].
constexpr int kStatsRBMax = 512;
// rows per block: enough blocks for two waves of 148 SMs, 64..512 rows (a multiple of 64)
__host__ __device__ inline int64_t stats_rb(int64_t R, int64_t C) {
  const int64_t ncb = (C + 255) / 256;
  int64_t rb = (R * ncb / 296 + 63) / 64 * 64;
  return rb < 64 ? 64 : (rb > kStatsRBMax ? kStatsRBMax : rb);
}
constexpr int kStatsThreads = 256;
constexpr int kStatsTileRows = 64;
constexpr int kStatsPitch = 256 * 2 + 16;   // padded row pitch (bytes): conflict-free row reads

struct StatAcc {
  double s = 0, s2 = 0, sa = 0;
  float mx = 0.f;
  __device__ __forceinline__ void add(float v) {
    const double x = double(v);
    s = __dadd_rn(s, x);
    s2 = __fma_rn(x, x, s2);
    sa = __dadd_rn(sa, fabs(x));
    mx = fmaxf(mx, fabsf(v));
  }
  __device__ __forceinline__ void merge(const StatAcc& o) {
    s = __dadd_rn(s, o.s);
    s2 = __dadd_rn(s2, o.s2);
    sa = __dadd_rn(sa, o.sa);
    mx = fmaxf(mx, o.mx);
  }
};

template <typename T>
__device__ __forceinline__ void stats_tile_block(const T* __restrict__ in, int64_t R, int64_t C, int64_t ld,
                                                 int64_t rb_rows, double* __restrict__ rpart,
                                                 double* __restrict__ cpart, int cb, int chunk, uint8_t* tile) {
  const int tid = threadIdx.x;
  const int64_t c0 = int64_t(cb) * 256;
  const int64_t r_end = min(R, int64_t(chunk) * rb_rows + rb_rows);
  const bool vec = sizeof(T) == 2 && c0 + 256 <= C && ((ld * 2) % 16) == 0 && (reinterpret_cast<uintptr_t>(in) & 15) == 0;
  StatAcc col;
  const int rr = tid >> 2, q = tid & 3;   // row stats: row rr of the tile, columns [64 q, 64 q + 64)
  for (int64_t r0 = int64_t(chunk) * rb_rows; r0 < r_end; r0 += kStatsTileRows) {
    const int nrows = int(min(int64_t(kStatsTileRows), r_end - r0));
    // ---- stage 64 x 256 values as bf16 bit patterns (fp32 inputs: generic path below)
    if (vec) {
      uint4 u[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int e = tid + i * kStatsThreads, row = e >> 5, c16 = e & 31;
        u[i] = row < nrows ? __ldg(reinterpret_cast<const uint4*>(in + (r0 + row) * ld + c0 + c16 * 8))
                           : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int e = tid + i * kStatsThreads, row = e >> 5, c16 = e & 31;
        *reinterpret_cast<uint4*>(tile + row * kStatsPitch + c16 * 16) = u[i];
      }
    } else if (sizeof(T) == 2) {   // ragged / unaligned bf16: element loads (exact bit copies)
      for (int e = tid; e < kStatsTileRows * 256; e += kStatsThreads) {
        const int row = e >> 8, c = e & 255;
        float v = 0.f;
        if (row < nrows && c0 + c < C) v = load_as_float(in, (r0 + row) * ld + c0 + c);
        reinterpret_cast<uint16_t*>(tile + row * kStatsPitch)[c] = uint16_t(__float_as_uint(v) >> 16);
      }
    }
    __syncthreads();
    if (sizeof(T) == 2) {
      // column tid down the tile
      const uint16_t* cp = reinterpret_cast<const uint16_t*>(tile) + tid;
#pragma unroll 8
      for (int row = 0; row < nrows; ++row) col.add(__uint_as_float(uint32_t(cp[row * (kStatsPitch / 2)]) << 16));
      // row rr, 64 columns
      StatAcc racc;
      if (rr < nrows) {
        const uint4* rp = reinterpret_cast<const uint4*>(tile + rr * kStatsPitch + q * 128);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const uint4 u = rp[i];
          const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            racc.add(__uint_as_float(w[t] << 16));
            racc.add(__uint_as_float(w[t] & 0xFFFF0000u));
          }
        }
      }
#pragma unroll
      for (int o = 1; o < 4; o <<= 1) {
        racc.s = __dadd_rn(racc.s, __shfl_xor_sync(0xffffffffu, racc.s, o));
        racc.s2 = __dadd_rn(racc.s2, __shfl_xor_sync(0xffffffffu, racc.s2, o));
        racc.sa = __dadd_rn(racc.sa, __shfl_xor_sync(0xffffffffu, racc.sa, o));
        racc.mx = fmaxf(racc.mx, __shfl_xor_sync(0xffffffffu, racc.mx, o));
      }
      if (q == 0 && rr < nrows) {
        double* p = rpart + (int64_t(cb) * R + r0 + rr) * 4;
        p[0] = racc.s; p[1] = racc.s2; p[2] = racc.sa; p[3] = double(racc.mx);
      }
    }
    __syncthreads();
    if (sizeof(T) != 2) {
      // fp32 inputs (tests only): direct global reads, thread per column / 4 threads per row
      for (int row = 0; row < nrows; ++row)
        if (c0 + tid < C) col.add(load_as_float(in, (r0 + row) * ld + c0 + tid));
      StatAcc racc;
      if (rr < nrows)
        for (int c = q * 64; c < q * 64 + 64; ++c)
          if (c0 + c < C) racc.add(load_as_float(in, (r0 + rr) * ld + c0 + c));
#pragma unroll
      for (int o = 1; o < 4; o <<= 1) {
        racc.s = __dadd_rn(racc.s, __shfl_xor_sync(0xffffffffu, racc.s, o));
        racc.s2 = __dadd_rn(racc.s2, __shfl_xor_sync(0xffffffffu, racc.s2, o));
        racc.sa = __dadd_rn(racc.sa, __shfl_xor_sync(0xffffffffu, racc.sa, o));
        racc.mx = fmaxf(racc.mx, __shfl_xor_sync(0xffffffffu, racc.mx, o));
      }
      if (q == 0 && rr < nrows) {
        double* p = rpart + (int64_t(cb) * R + r0 + rr) * 4;
        p[0] = racc.s; p[1] = racc.s2; p[2] = racc.sa; p[3] = double(racc.mx);
      }
    }
  }
  if (c0 + tid < C) {
    double* p = cpart + (int64_t(chunk) * C + c0 + tid) * 4;
    p[0] = col.s; p[1] = col.s2; p[2] = col.sa; p[3] = double(col.mx);
  }
}
template <typename T>
__global__ void __launch_bounds__(kStatsThreads) k_stats_tile(const T* __restrict__ in, int64_t R, int64_t C,
                                                              int64_t ld, int64_t rb_rows, double* __restrict__ rpart,
                                                              double* __restrict__ cpart) {
  __shared__ __align__(16) uint8_t tile[kStatsTileRows * kStatsPitch];   // bf16 inputs only
  stats_tile_block(in, R, C, ld, rb_rows, rpart, cpart, int(blockIdx.x), int(blockIdx.y), tile);
}

// cvpart (nullable): per-block partial sums of the CV terms std/(mean|x| + eps) of the rows
// (cvpart[2 b]) and columns (cvpart[2 b + 1]) this block finalised (App. A), for
// k_classify_partials. Fixed-order tree sums: deterministic.
constexpr int kReduceThreads = 256;
__device__ __forceinline__ double cv_term(double s, double s2, double sa, double n, double eps) {
  const double mu = s / n;
  const double var = fmax(s2 / n - mu * mu, 0.0);
  return sqrt(var) / (sa / n + eps);
}
// Threads: one per row (the row section padded to whole warps), then `lanes` per column (8 for
// narrow tensors, whose few columns each have many row-chunk partials; 1 for wide ones); the
// lanes of a column sum the partials q = lane, lane + lanes, ... in order and combine by xor
// shuffles (a fixed pattern: deterministic).
__host__ __device__ inline int stats_col_lanes(int64_t C) { return C <= 2048 ? 8 : (C <= 4096 ? 4 : 1); }
__host__ __device__ inline int64_t stats_reduce_threads(int64_t R, int64_t C) {
  return (R + 31) / 32 * 32 + C * stats_col_lanes(C);
}
__device__ __forceinline__ void stats_reduce_block(const double* __restrict__ rpart, int64_t ncb, int64_t R,
                                                   const double* __restrict__ cpart, int64_t nch, int64_t C,
                                                   double* __restrict__ rs, double* __restrict__ cs,
                                                   double* __restrict__ cvpart, double eps, int blk,
                                                   double (*red)[kReduceThreads]) {
  const int64_t i = int64_t(blk) * blockDim.x + threadIdx.x;
  const int64_t rpad = (R + 31) / 32 * 32;
  const int lanes = stats_col_lanes(C);
  const bool is_row = i < rpad;                                   // warp-uniform
  const int sub = is_row ? 0 : int((i - rpad) % lanes);
  const int64_t j = is_row ? i : (i - rpad) / lanes;
  const bool live = is_row ? i < R : j < C;
  double a = 0, b = 0, d = 0, m = 0;
  {
    const double* src = is_row ? rpart : cpart;
    const int64_t n = is_row ? ncb : nch, stride = is_row ? R : C;
    const int step = is_row ? 1 : lanes;
    int64_t q = sub;
    if (live) {
      for (; q + 3 * step < n; q += 4 * step) {   // four loads in flight, summed in order
        double4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = *reinterpret_cast<const double4*>(src + ((q + u * step) * stride + j) * 4);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          a = __dadd_rn(a, v[u].x); b = __dadd_rn(b, v[u].y); d = __dadd_rn(d, v[u].z); m = fmax(m, v[u].w);
        }
      }
      for (; q < n; q += step) {
        const double4 v = *reinterpret_cast<const double4*>(src + (q * stride + j) * 4);
        a = __dadd_rn(a, v.x); b = __dadd_rn(b, v.y); d = __dadd_rn(d, v.z); m = fmax(m, v.w);
      }
    }
    if (!is_row) {
      for (int o = 1; o < lanes; o <<= 1) {
        a = __dadd_rn(a, __shfl_xor_sync(0xffffffffu, a, o));
        b = __dadd_rn(b, __shfl_xor_sync(0xffffffffu, b, o));
        d = __dadd_rn(d, __shfl_xor_sync(0xffffffffu, d, o));
        m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
      }
    }
    if (live && sub == 0) {
      double* dst = (is_row ? rs : cs) + j * 4;
      dst[0] = a; dst[1] = b; dst[2] = d; dst[3] = m;
    }
  }
  if (cvpart == nullptr) return;   // block-uniform
  const bool owner = live && sub == 0;
  const double t = owner ? cv_term(a, b, d, double(is_row ? C : R), eps) : 0.0;
  red[0][threadIdx.x] = owner && is_row ? t : 0.0;
  red[1][threadIdx.x] = owner && !is_row ? t : 0.0;
  __syncthreads();
  for (int h = kReduceThreads / 2; h > 0; h >>= 1) {
    if (int(threadIdx.x) < h) {
      red[0][threadIdx.x] += red[0][threadIdx.x + h];
      red[1][threadIdx.x] += red[1][threadIdx.x + h];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    cvpart[2 * blk] = red[0][0];
    cvpart[2 * blk + 1] = red[1][0];
  }
}
__global__ void __launch_bounds__(kReduceThreads) k_stats_reduce(const double* __restrict__ rpart, int64_t ncb,
                                                                 int64_t R, const double* __restrict__ cpart,
                                                                 int64_t nch, int64_t C, double* __restrict__ rs,
                                                                 double* __restrict__ cs, double* __restrict__ cvpart,
                                                                 double eps) {
  __shared__ double red[2][kReduceThreads];
  stats_reduce_block(rpart, ncb, R, cpart, nch, C, rs, cs, cvpart, eps, int(blockIdx.x), red);
}

// App. A decision (DESIGN R7) from the two CV sums: d_cv[0..1] = the sums,
// d_cv[2..3] = CV_row = sum_row / rows, CV_col = sum_col / cols; Row if CV_col > tau, Column if
// CV_row > tau, the larger when both, an exact tie -> Row.
__device__ __forceinline__ void classify_store(double sum_row, double sum_col, int64_t rows, int64_t cols, double tau,
                                               double* d_cv, uint8_t* pattern) {
  const double cv_row = sum_row / double(rows), cv_col = sum_col / double(cols);
  d_cv[0] = sum_row;
  d_cv[1] = sum_col;
  d_cv[2] = cv_row;
  d_cv[3] = cv_col;
  const bool row_hit = cv_col > tau, col_hit = cv_row > tau;
  uint8_t p = 0;
  if (row_hit && (!col_hit || cv_col >= cv_row)) p = 1;
  else if (col_hit) p = 2;
  pattern[0] = p;
}

// Sum of the blocks' CV partials (fixed order) and the single-rank classification.
__device__ __forceinline__ void classify_partials_block(const double* __restrict__ cvpart, int nb, int64_t rows,
                                                        int64_t cols, double tau, double* __restrict__ d_cv,
                                                        uint8_t* __restrict__ pattern, double (*red)[256]) {
  double a = 0, b = 0;
  for (int k = threadIdx.x; k < nb; k += 256) { a += cvpart[2 * k]; b += cvpart[2 * k + 1]; }
  red[0][threadIdx.x] = a;
  red[1][threadIdx.x] = b;
  __syncthreads();
  for (int h = 128; h > 0; h >>= 1) {
    if (int(threadIdx.x) < h) {
      red[0][threadIdx.x] += red[0][threadIdx.x + h];
      red[1][threadIdx.x] += red[1][threadIdx.x + h];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) classify_store(red[0][0], red[1][0], rows, cols, tau, d_cv, pattern);
}
__global__ void __launch_bounds__(256) k_classify_partials(const double* __restrict__ cvpart, int nb, int64_t rows,
                                                          int64_t cols, double tau, double* __restrict__ d_cv,
                                                          uint8_t* __restrict__ pattern) {
  __shared__ double red[2][256];
  classify_partials_block(cvpart, nb, rows, cols, tau, d_cv, pattern, red);
}

// Batched calibration: up to kCalibMaxJobs tensors per launch triple, every job's blocks exactly
// as in the single-tensor launches (same partition, same reduction order: bitwise the same).
struct CalibJobDev {
  const void* in; int64_t R, C, ld, rb, ncb, nch;
  double *rpart, *cpart, *rs, *cs, *cvpart, *d_cv;
  uint8_t* pattern;
  int nbr;   // reduce blocks
};
struct CalibBatchDev {
  CalibJobDev j[kCalibMaxJobs];
  int n, f32;
  int tile_off[kCalibMaxJobs + 1], red_off[kCalibMaxJobs + 1];
  double eps, tau;
};
__device__ __forceinline__ int calib_job_of(const int* off, int n, int b) {
  int j = 0;
  while (j + 1 < n && b >= off[j + 1]) ++j;
  return j;
}
__global__ void __launch_bounds__(kStatsThreads) k_stats_tile_batch(const __grid_constant__ CalibBatchDev B) {
  __shared__ __align__(16) uint8_t tile[kStatsTileRows * kStatsPitch];
  const int jb = calib_job_of(B.tile_off, B.n, blockIdx.x);
  const CalibJobDev& J = B.j[jb];
  const int lid = int(blockIdx.x) - B.tile_off[jb];
  const int cb = int(lid % J.ncb), chunk = int(lid / J.ncb);
  if (B.f32) stats_tile_block(static_cast<const float*>(J.in), J.R, J.C, J.ld, J.rb, J.rpart, J.cpart, cb, chunk, tile);
  else stats_tile_block(static_cast<const __nv_bfloat16*>(J.in), J.R, J.C, J.ld, J.rb, J.rpart, J.cpart, cb, chunk, tile);
}
__global__ void __launch_bounds__(kReduceThreads) k_stats_reduce_batch(const __grid_constant__ CalibBatchDev B) {
  __shared__ double red[2][kReduceThreads];
  const int jb = calib_job_of(B.red_off, B.n, blockIdx.x);
  const CalibJobDev& J = B.j[jb];
  stats_reduce_block(J.rpart, J.ncb, J.R, J.cpart, J.nch, J.C, J.rs, J.cs, J.cvpart, B.eps,
                     int(blockIdx.x) - B.red_off[jb], red);
}
__global__ void __launch_bounds__(256) k_classify_partials_batch(const __grid_constant__ CalibBatchDev B) {
  __shared__ double red[2][256];
  const CalibJobDev& J = B.j[blockIdx.x];
  classify_partials_block(J.cvpart, J.nbr, J.R, J.C, B.tau, J.d_cv, J.pattern, red);
}

size_t calib_cvpart_bytes(int64_t R, int64_t C) {
  return size_t((stats_reduce_threads(R, C) + kReduceThreads - 1) / kReduceThreads) * 16;
}

size_t stats_ws_bytes(int64_t R, int64_t C) {
  const int64_t ncb = (C + 255) / 256, rb = stats_rb(R, C), nch = (R + rb - 1) / rb;
  return size_t(ncb * R + nch * C) * 32 + 256;
}

cudaError_t launch_stats(const void* in, bool in_f32, int64_t R, int64_t C, int64_t ld,
                         double* rs, double* cs, double* part, cudaStream_t st) {
  const int64_t ncb = (C + 255) / 256, rb = stats_rb(R, C), nch = (R + rb - 1) / rb;
  double* rpart = part;
  double* cpart = part + ncb * R * 4;
  const dim3 grid{unsigned(ncb), unsigned(nch)};
  if (in_f32) k_stats_tile<float><<<grid, kStatsThreads, 0, st>>>(static_cast<const float*>(in), R, C, ld, rb, rpart, cpart);
  else k_stats_tile<__nv_bfloat16><<<grid, kStatsThreads, 0, st>>>(static_cast<const __nv_bfloat16*>(in), R, C, ld,
                                                                   rb, rpart, cpart);
  k_stats_reduce<<<unsigned((stats_reduce_threads(R, C) + kReduceThreads - 1) / kReduceThreads), kReduceThreads, 0, st>>>(
      rpart, ncb, R, cpart, nch, C, rs, cs, nullptr, 0.0);
  return cudaGetLastError();
}

cudaError_t launch_calibrate(const void* in, bool in_f32, int64_t R, int64_t C, int64_t ld, double* rs, double* cs,
                             double* part, double* cvpart, double eps, double tau, double* d_cv, uint8_t* pattern,
                             cudaStream_t st) {
  const int64_t ncb = (C + 255) / 256, rb = stats_rb(R, C), nch = (R + rb - 1) / rb;
  double* rpart = part;
  double* cpart = part + ncb * R * 4;
  const dim3 grid{unsigned(ncb), unsigned(nch)};
  if (in_f32) k_stats_tile<float><<<grid, kStatsThreads, 0, st>>>(static_cast<const float*>(in), R, C, ld, rb, rpart, cpart);
  else k_stats_tile<__nv_bfloat16><<<grid, kStatsThreads, 0, st>>>(static_cast<const __nv_bfloat16*>(in), R, C, ld,
                                                                   rb, rpart, cpart);
  const int nb = int((stats_reduce_threads(R, C) + kReduceThreads - 1) / kReduceThreads);
  k_stats_reduce<<<unsigned(nb), kReduceThreads, 0, st>>>(rpart, ncb, R, cpart, nch, C, rs, cs, cvpart, eps);
  k_classify_partials<<<1, 256, 0, st>>>(cvpart, nb, R, C, tau, d_cv, pattern);
  return cudaGetLastError();
}

cudaError_t launch_calibrate_batch(const CalibJob* jobs, int n, bool in_f32, double eps, double tau, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  if (n > kCalibMaxJobs) return cudaErrorInvalidValue;
  CalibBatchDev B{};
  B.n = n;
  B.f32 = in_f32 ? 1 : 0;
  B.eps = eps;
  B.tau = tau;
  B.tile_off[0] = B.red_off[0] = 0;
  for (int i = 0; i < n; ++i) {
    const CalibJob& q = jobs[i];
    CalibJobDev& J = B.j[i];
    J.in = q.in; J.R = q.R; J.C = q.C; J.ld = q.ld;
    J.ncb = (q.C + 255) / 256;
    J.rb = stats_rb(q.R, q.C);
    J.nch = (q.R + J.rb - 1) / J.rb;
    J.rpart = q.part;
    J.cpart = q.part + J.ncb * q.R * 4;
    J.rs = q.rs; J.cs = q.cs; J.cvpart = q.cvpart; J.d_cv = q.d_cv; J.pattern = q.pattern;
    J.nbr = int((stats_reduce_threads(q.R, q.C) + kReduceThreads - 1) / kReduceThreads);
    B.tile_off[i + 1] = B.tile_off[i] + int(J.ncb * J.nch);
    B.red_off[i + 1] = B.red_off[i] + J.nbr;
  }
  k_stats_tile_batch<<<unsigned(B.tile_off[n]), kStatsThreads, 0, st>>>(B);
  k_stats_reduce_batch<<<unsigned(B.red_off[n]), kReduceThreads, 0, st>>>(B);
  k_classify_partials_batch<<<unsigned(n), 256, 0, st>>>(B);
  return cudaGetLastError();
}

// Outlier rows / columns of each calibrated tensor (App. D, DESIGN R16): from the
// statistics the batch left in its workspace — sum |x| of every row (fixed order over the rows)
// gives mean |x|; rows / columns whose max |x| exceeds kappa * mean |x| are counted.
__global__ void __launch_bounds__(256) k_outlier_counts_batch(const __grid_constant__ CalibBatchDev B, double kappa,
                                                             int32_t* __restrict__ counts) {
  __shared__ double red[256];
  __shared__ int cnt[2];
  const CalibJobDev& J = B.j[blockIdx.x];
  double a = 0;
  for (int64_t i = threadIdx.x; i < J.R; i += 256) a += J.rs[i * 4 + 2];
  red[threadIdx.x] = a;
  if (threadIdx.x < 2) cnt[threadIdx.x] = 0;
  __syncthreads();
  for (int h = 128; h > 0; h >>= 1) {
    if (int(threadIdx.x) < h) red[threadIdx.x] += red[threadIdx.x + h];
    __syncthreads();
  }
  const double thr = kappa * (red[0] / (double(J.R) * double(J.C)));
  int nr = 0, nc = 0;
  for (int64_t i = threadIdx.x; i < J.R; i += 256) nr += J.rs[i * 4 + 3] > thr;
  for (int64_t j = threadIdx.x; j < J.C; j += 256) nc += J.cs[j * 4 + 3] > thr;
  atomicAdd(&cnt[0], nr);
  atomicAdd(&cnt[1], nc);
  __syncthreads();
  if (threadIdx.x == 0) {
    counts[2 * blockIdx.x] = cnt[0];
    counts[2 * blockIdx.x + 1] = cnt[1];
  }
}

cudaError_t launch_outlier_counts_batch(const CalibJob* jobs, int n, double kappa, int32_t* counts, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  if (n > kCalibMaxJobs) return cudaErrorInvalidValue;
  CalibBatchDev B{};
  B.n = n;
  for (int i = 0; i < n; ++i) {
    B.j[i].R = jobs[i].R;
    B.j[i].C = jobs[i].C;
    B.j[i].rs = jobs[i].rs;
    B.j[i].cs = jobs[i].cs;
  }
  k_outlier_counts_batch<<<unsigned(n), 256, 0, st>>>(B, kappa, counts);
  return cudaGetLastError();
}

// CV sums (App. A) and the single-rank classification (DESIGN R7).
__global__ void __launch_bounds__(1024) k_classify(const double* __restrict__ rs, int64_t rows,
                                                   int64_t row_len, const double* __restrict__ cs,
                                                   int64_t cols, int64_t col_len, double eps,
                                                   double tau, double* __restrict__ d_cv,
                                                   uint8_t* __restrict__ pattern) {
  __shared__ double red[2][1024];
  double a = 0, b = 0;
  for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) {
    const double n = double(row_len);
    const double mu = rs[i * 4] / n;
    const double var = fmax(rs[i * 4 + 1] / n - mu * mu, 0.0);
    a += sqrt(var) / (rs[i * 4 + 2] / n + eps);
  }
  for (int64_t j = threadIdx.x; j < cols; j += blockDim.x) {
    const double n = double(col_len);
    const double mu = cs[j * 4] / n;
    const double var = fmax(cs[j * 4 + 1] / n - mu * mu, 0.0);
    b += sqrt(var) / (cs[j * 4 + 2] / n + eps);
  }
  red[0][threadIdx.x] = a;
  red[1][threadIdx.x] = b;
  __syncthreads();
  for (int s = 512; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      red[0][threadIdx.x] += red[0][threadIdx.x + s];
      red[1][threadIdx.x] += red[1][threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) classify_store(red[0][0], red[1][0], rows, cols, tau, d_cv, pattern);
}
// Multi-rank decision: d_cv[0] = the row-CV sum over ALL ranks' rows (all-reduced by the caller),
// d_cv[1] = the column-CV sum from the merged column statistics; rows = the global row count.
__global__ void k_classify_sums(double* d_cv, int64_t rows, int64_t cols, double tau, uint8_t* pattern) {
  if (threadIdx.x == 0) classify_store(d_cv[0], d_cv[1], rows, cols, tau, d_cv, pattern);
}
cudaError_t launch_classify_sums(double* d_cv, int64_t rows, int64_t cols, double tau, uint8_t* pattern,
                                 cudaStream_t st) {
  k_classify_sums<<<1, 32, 0, st>>>(d_cv, rows, cols, tau, pattern);
  return cudaGetLastError();
}
cudaError_t launch_classify(const double* rs, int64_t rows, int64_t row_len, const double* cs,
                            int64_t cols, int64_t col_len, double eps, double tau, double* d_cv,
                            uint8_t* pattern, cudaStream_t st) {
  k_classify<<<1, 1024, 0, st>>>(rs, rows, row_len, cs, cols, col_len, eps, tau, d_cv, pattern);
  return cudaGetLastError();
}

}  // namespace adahop

namespace adahop {
// ================================================================== E2M1 conversion checks
// Codes of arbitrary fp32 values through the production conversion (hardware cvt) and the
// software rounding rule, for the parity tests.
__global__ void k_e2m1_codes(const float* __restrict__ v, int64_t n, uint8_t* __restrict__ hw,
                             uint8_t* __restrict__ sw) {
  const int64_t i = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 8;
  if (i >= n) return;
  float x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = i + j < n ? v[i + j] : 0.f;
  const uint32_t h = e2m1x8_hw(x), s = e2m1x8_sw(x);
  for (int j = 0; j < 8 && i + j < n; ++j) {
    hw[i + j] = uint8_t((h >> (4 * j)) & 0xF);
    sw[i + j] = uint8_t((s >> (4 * j)) & 0xF);
  }
}
// Exhaustive: every fp32 bit pattern in [lo, hi) that is finite, compare hw vs sw.
__global__ void k_e2m1_exhaustive(uint64_t lo, uint64_t hi, unsigned long long* mismatches,
                                  unsigned int* first_bad) {
  unsigned long long bad = 0;
  for (uint64_t b = lo + (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 8; b < hi;
       b += uint64_t(gridDim.x) * blockDim.x * 8) {
    float x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t u = uint32_t(b + j);
      const bool fin = ((u >> 23) & 0xFF) != 0xFF;
      x[j] = fin ? __uint_as_float(u) : 0.f;
    }
    const uint32_t h = e2m1x8_hw(x), s = e2m1x8_sw(x);
    if (h != s) {
      for (int j = 0; j < 8; ++j)
        if (((h >> (4 * j)) & 0xF) != ((s >> (4 * j)) & 0xF)) {
          ++bad;
          atomicMin(first_bad, uint32_t(b + j));
        }
    }
  }
  if (bad) atomicAdd(mismatches, bad);
}
cudaError_t launch_e2m1_codes(const float* v, int64_t n, uint8_t* hw, uint8_t* sw, cudaStream_t st) {
  const int64_t threads = (n + 7) / 8;
  k_e2m1_codes<<<unsigned((threads + 255) / 256), 256, 0, st>>>(v, n, hw, sw);
  return cudaGetLastError();
}
cudaError_t launch_e2m1_exhaustive(uint64_t lo, uint64_t hi, unsigned long long* mism,
                                   unsigned int* first_bad, cudaStream_t st) {
  k_e2m1_exhaustive<<<148 * 8, 256, 0, st>>>(lo, hi, mism, first_bad);
  return cudaGetLastError();
}
}  // namespace adahop
