// quant.cu — HBM-bound kernels of the AdaHOP hot path (sm_100a):
//   * fused residual mask + blockwise FWHT (b = 32) + MXFP4 quantisation, in a row
//     (K-contiguous) and a transposing column (K-strided) variant   [P:350, P:761]
//   * FOID: fp64 probe variance, deterministic top-k, outlier-slice gather  [P:760]
//   * pattern statistics for calibration (per-row / per-column moments)    [P:523-541]
//   * layout converters used only by the debug / parity entry points
#include "common.cuh"
#include "kernels.h"
#include <algorithm>

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

// In-register IHT + MX quantisation of one 32-element block.
// x: raw values (residual mask already applied). On return: codes (16 bytes, element
// 2j in the low nibble), the biased E8M0 scale byte, and (kHad) y = the fp32 Hadamard
// output that enters the quantiser.
template <bool kHad, bool kSwCvt>
__device__ __forceinline__ void iht_quant32(float (&x)[32], uint4& codes, uint32_t& sbyte,
                                            float* y_out) {
  // Radix-2 butterflies, strides 1,2,4,8,16 (natural-order Walsh–Hadamard), fp32 RN.
#pragma unroll
  for (int h = 1; h < 32; h <<= 1) {
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      if ((i & h) == 0) {
        const float a = x[i], b = x[i + h];
        x[i] = __fadd_rn(a, b);
        x[i + h] = __fsub_rn(a, b);
      }
    }
  }
  float amax = 0.f;
#pragma unroll
  for (int i = 0; i < 32; ++i) amax = fmaxf(amax, fabsf(x[i]));
  const float c = ADAHOP_INV_SQRT32;
  // max |RN(x_i c)| == RN(max|x_i| c) since RN is monotone.
  const float amax_y = __fmul_rn(amax, c);
  const uint32_t bits = __float_as_uint(amax_y);
  int e;
  if (amax_y == 0.f) {
    e = 0;
  } else if ((bits >> 23) != 0) {
    e = int(bits >> 23) - 127 - 2;            // floor(log2 amax) - emax(E2M1)
  } else {
    e = (31 - __clz(int(bits))) - 149 - 2;    // subnormal amax
  }
  e = max(-127, min(127, e));
  sbyte = uint32_t(e + 127);
  float v[32];
  if (kHad || e > 120 || e < -100) {
    // exact two-step path: y = RN(x c); v = y * 2^-e (exact power-of-two scaling)
    const float s = __uint_as_float(uint32_t(127 - e) << 23);
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const float y = __fmul_rn(x[i], c);
      if (kHad) y_out[i] = y;
      v[i] = __fmul_rn(y, s);
    }
  } else {
    // fused: RN(x (c 2^-e)) == RN(x c) 2^-e for every value that can reach a nonzero code
    const float cs = __fmul_rn(c, __uint_as_float(uint32_t(127 - e) << 23));
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __fmul_rn(x[i], cs);
  }
  if (kSwCvt) {
    codes.x = e2m1x8_sw(v + 0);
    codes.y = e2m1x8_sw(v + 8);
    codes.z = e2m1x8_sw(v + 16);
    codes.w = e2m1x8_sw(v + 24);
  } else {
    codes.x = e2m1x8_hw(v + 0);
    codes.y = e2m1x8_hw(v + 8);
    codes.z = e2m1x8_hw(v + 16);
    codes.w = e2m1x8_hw(v + 24);
  }
}

__device__ __forceinline__ void load32(const __nv_bfloat16* p, float (&x)[32]) {
  const uint4* q = reinterpret_cast<const uint4*>(p);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint4 u = __ldg(q + j);
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      x[j * 8 + 2 * t] = __uint_as_float(w[t] << 16);
      x[j * 8 + 2 * t + 1] = __uint_as_float(w[t] & 0xFFFF0000u);
    }
  }
}
__device__ __forceinline__ void load32(const float* p, float (&x)[32]) {
  const float4* q = reinterpret_cast<const float4*>(p);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float4 u = __ldg(q + j);
    x[4 * j] = u.x; x[4 * j + 1] = u.y; x[4 * j + 2] = u.z; x[4 * j + 3] = u.w;
  }
}

// Row variant: stored row r is in[r*ld + 0..K). One thread per (row, 32-block).
template <typename T, bool kHad, bool kSwCvt>
__global__ void __launch_bounds__(256) k_iht_quant_row(const T* __restrict__ in, int64_t R,
                                                       int64_t K, int64_t ld,
                                                       const int32_t* __restrict__ zero_rows,
                                                       int nzero, uint8_t* __restrict__ codes,
                                                       uint8_t* __restrict__ sf, int64_t kchunks,
                                                       float* __restrict__ had_out) {
  const int64_t nkb = K / kBlk;
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= R * nkb) return;
  const int64_t r = t / nkb;
  const int64_t kb = t - r * nkb;
  float x[32];
  if (nzero > 0 && in_sorted(zero_rows, nzero, r)) {
#pragma unroll
    for (int i = 0; i < 32; ++i) x[i] = 0.f;
  } else {
    load32(in + r * ld + kb * kBlk, x);
  }
  uint4 c;
  uint32_t s;
  iht_quant32<kHad, kSwCvt>(x, c, s, kHad ? had_out + r * K + kb * kBlk : nullptr);
  *reinterpret_cast<uint4*>(codes + r * (K / 2) + kb * 16) = c;
  sf[sf_offset(r, kb, kchunks)] = uint8_t(s);
}

// Column (transposing) variant: stored row r is in[k*ld + r], k = 0..K. A CTA transposes
// a 64(k) x 128(r) tile through shared memory; thread (r, kb) then owns one 32-block.
template <typename T, bool kHad, bool kSwCvt>
__global__ void __launch_bounds__(256) k_iht_quant_col(const T* __restrict__ in, int64_t R,
                                                       int64_t K, int64_t ld,
                                                       const int32_t* __restrict__ zero_rows,
                                                       int nzero, uint8_t* __restrict__ codes,
                                                       uint8_t* __restrict__ sf, int64_t kchunks,
                                                       float* __restrict__ had_out) {
  constexpr int TK = 64, TR = 128;
  __shared__ __align__(16) T tile[TK][TR];
  const int64_t r0 = int64_t(blockIdx.x) * TR;
  const int64_t k0 = int64_t(blockIdx.y) * TK;
  constexpr int kVec = 16 / sizeof(T);  // elements per 16-byte vector
  constexpr int kVecPerRow = TR / kVec;
  const bool full = (r0 + TR <= R) && (k0 + TK <= K) && ((ld * sizeof(T)) % 16 == 0) &&
                    ((reinterpret_cast<uintptr_t>(in) & 15) == 0);
  if (full) {
    for (int v = threadIdx.x; v < TK * kVecPerRow; v += blockDim.x) {
      const int kr = v / kVecPerRow, c = (v % kVecPerRow) * kVec;
      *reinterpret_cast<uint4*>(&tile[kr][c]) =
          __ldg(reinterpret_cast<const uint4*>(in + (k0 + kr) * ld + r0 + c));
    }
  } else {
    for (int v = threadIdx.x; v < TK * TR; v += blockDim.x) {
      const int kr = v / TR, c = v % TR;
      const bool ok = (k0 + kr < K) && (r0 + c < R);
      tile[kr][c] = ok ? in[(k0 + kr) * ld + r0 + c] : T(0.f);
    }
  }
  __syncthreads();
  const int rr = threadIdx.x % TR;
  const int kbl = threadIdx.x / TR;  // 0 or 1
  const int64_t r = r0 + rr;
  const int64_t kb = k0 / kBlk + kbl;
  if (r >= R || kb * kBlk >= K) return;
  float x[32];
  if (nzero > 0 && in_sorted(zero_rows, nzero, r)) {
#pragma unroll
    for (int i = 0; i < 32; ++i) x[i] = 0.f;
  } else {
#pragma unroll
    for (int i = 0; i < 32; ++i) x[i] = float(tile[kbl * 32 + i][rr]);
  }
  uint4 c;
  uint32_t s;
  iht_quant32<kHad, kSwCvt>(x, c, s, kHad ? had_out + r * K + kb * kBlk : nullptr);
  *reinterpret_cast<uint4*>(codes + r * (K / 2) + kb * 16) = c;
  sf[sf_offset(r, kb, kchunks)] = uint8_t(s);
}

// ------------------------------------------------------------------------ launchers
template <typename T, bool kHad, bool kSw>
static cudaError_t launch_quant_t(const T* in, int64_t R, int64_t K, int64_t ld, int kstrided,
                                  const int32_t* zero_rows, int nzero, uint8_t* codes, uint8_t* sf,
                                  float* had_out, cudaStream_t st) {
  const int64_t kch = sf_kchunks(K);
  if (!kstrided) {
    const int64_t n = R * (K / kBlk);
    const int64_t blocks = (n + 255) / 256;
    k_iht_quant_row<T, kHad, kSw><<<dim3(unsigned(blocks)), 256, 0, st>>>(
        in, R, K, ld, zero_rows, nzero, codes, sf, kch, had_out);
  } else {
    dim3 grid(unsigned((R + 127) / 128), unsigned((K + 63) / 64));
    k_iht_quant_col<T, kHad, kSw><<<grid, 256, 0, st>>>(in, R, K, ld, zero_rows, nzero, codes,
                                                         sf, kch, had_out);
  }
  return cudaGetLastError();
}

cudaError_t launch_iht_quant(const void* in, bool in_f32, int64_t R, int64_t K, int64_t ld,
                             int kstrided, const int32_t* zero_rows, int nzero, uint8_t* codes,
                             uint8_t* sf, float* had_out, bool sw_cvt, cudaStream_t st) {
#define ADAHOP_Q(T, H, S)                                                                   \
  return launch_quant_t<T, H, S>(static_cast<const T*>(in), R, K, ld, kstrided, zero_rows, \
                                 nzero, codes, sf, had_out, st)
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
template <typename T>
__global__ void k_foid_keys(const T* __restrict__ in, int64_t R, int64_t ld, int kstrided, int p,
                            double* __restrict__ keys) {
  const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= R) return;
  double s = 0.0;
  for (int j = 0; j < p; ++j) {
    const double x = double(load_as_float(in, kstrided ? int64_t(j) * ld + r : r * ld + j));
    s = __dadd_rn(s, x);
  }
  const double mu = s / double(p);
  double v = 0.0;
  for (int j = 0; j < p; ++j) {
    const double x = double(load_as_float(in, kstrided ? int64_t(j) * ld + r : r * ld + j));
    const double d = __dsub_rn(x, mu);
    v = __dadd_rn(v, __dmul_rn(d, d));
  }
  keys[r] = v / double(p);
}

// (key, index) order: larger key first, equal keys -> lower index first.
__device__ __forceinline__ bool foid_before(double ka, int32_t ia, double kb, int32_t ib) {
  return ka > kb || (ka == kb && ia < ib);
}

// Bitonic sort of n (power of two) (key, idx) pairs in shared memory, "before" order.
__device__ void bitonic_sort_pairs(double* key, int32_t* idx, int n) {
  for (int size = 2; size <= n; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int j = i ^ stride;
        if (j > i) {
          const bool up = (i & size) == 0;
          const bool sw = up ? foid_before(key[j], idx[j], key[i], idx[i])
                             : foid_before(key[i], idx[i], key[j], idx[j]);
          if (sw) {
            const double tk = key[i]; key[i] = key[j]; key[j] = tk;
            const int32_t ti = idx[i]; idx[i] = idx[j]; idx[j] = ti;
          }
        }
      }
      __syncthreads();
    }
  }
}

constexpr int kFoidChunk = 2048;

// Top-k of each chunk of kFoidChunk rows.
__global__ void __launch_bounds__(1024) k_foid_chunk_topk(const double* __restrict__ keys, int64_t R,
                                                          int k, double* __restrict__ cand_key,
                                                          int32_t* __restrict__ cand_idx) {
  __shared__ double skey[kFoidChunk];
  __shared__ int32_t sidx[kFoidChunk];
  const int64_t base = int64_t(blockIdx.x) * kFoidChunk;
  for (int i = threadIdx.x; i < kFoidChunk; i += blockDim.x) {
    const int64_t r = base + i;
    skey[i] = r < R ? keys[r] : -1.0;
    sidx[i] = r < R ? int32_t(r) : INT32_MAX;
  }
  __syncthreads();
  bitonic_sort_pairs(skey, sidx, kFoidChunk);
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    cand_key[int64_t(blockIdx.x) * k + i] = skey[i];
    cand_idx[int64_t(blockIdx.x) * k + i] = sidx[i];
  }
}

// Merge the candidates (ncand <= 8192), keep the global top-k, write indices ascending.
__global__ void __launch_bounds__(1024) k_foid_merge(const double* __restrict__ cand_key,
                                                     const int32_t* __restrict__ cand_idx,
                                                     int ncand, int npow2, int k, int64_t R,
                                                     int32_t* __restrict__ idx_sorted) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* skey = reinterpret_cast<double*>(smem_raw);
  int32_t* sidx = reinterpret_cast<int32_t*>(skey + npow2);
  for (int i = threadIdx.x; i < npow2; i += blockDim.x) {
    skey[i] = i < ncand ? cand_key[i] : -1.0;
    sidx[i] = i < ncand ? cand_idx[i] : INT32_MAX;
  }
  __syncthreads();
  bitonic_sort_pairs(skey, sidx, npow2);
  // rank-sort the first kk indices ascending
  const int kk = int(int64_t(k) < R ? int64_t(k) : R);
  __shared__ int32_t top[256];
  for (int i = threadIdx.x; i < kk; i += blockDim.x) top[i] = sidx[i];
  __syncthreads();
  for (int i = threadIdx.x; i < kk; i += blockDim.x) {
    int rank = 0;
    for (int j = 0; j < kk; ++j) rank += top[j] < top[i];
    idx_sorted[rank] = top[i];
  }
}

cudaError_t launch_foid(const void* in, bool in_f32, int64_t R, int64_t K, int64_t ld,
                        int kstrided, int k, int probe, double* keys, double* cand_key,
                        int32_t* cand_idx, int32_t* idx_sorted, cudaStream_t st) {
  const int p = int(std::min<int64_t>(probe, K));
  const unsigned kb = unsigned((R + 255) / 256);
  if (in_f32) k_foid_keys<float><<<kb, 256, 0, st>>>(static_cast<const float*>(in), R, ld, kstrided, p, keys);
  else k_foid_keys<__nv_bfloat16><<<kb, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(in), R, ld, kstrided, p, keys);
  const int kk = int(std::min<int64_t>(k, R));
  const int nchunks = int((R + kFoidChunk - 1) / kFoidChunk);
  k_foid_chunk_topk<<<nchunks, 1024, 0, st>>>(keys, R, kk, cand_key, cand_idx);
  const int ncand = nchunks * kk;
  int npow2 = 1;
  while (npow2 < ncand) npow2 <<= 1;
  const size_t smem = size_t(npow2) * (sizeof(double) + sizeof(int32_t));
  if (smem > 48 * 1024) {
    cudaFuncSetAttribute(k_foid_merge, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  }
  k_foid_merge<<<1, 1024, smem, st>>>(cand_key, cand_idx, ncand, npow2, kk, R, idx_sorted);
  return cudaGetLastError();
}

// Outlier slice (bf16, k x K, K contiguous): out[s][j] = store(idx[s], j).
__global__ void k_gather_rows_kc(const __nv_bfloat16* __restrict__ in, int64_t K, int64_t ld,
                                 const int32_t* __restrict__ idx, __nv_bfloat16* __restrict__ out) {
  const int s = blockIdx.y;
  const int64_t r = idx[s];
  const uint4* src = reinterpret_cast<const uint4*>(in + r * ld);
  uint4* dst = reinterpret_cast<uint4*>(out + int64_t(s) * K);
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < K / 8;
       v += int64_t(gridDim.x) * blockDim.x)
    dst[v] = __ldg(src + v);
}
__global__ void k_gather_rows_ks(const __nv_bfloat16* __restrict__ in, int64_t K, int64_t ld,
                                 const int32_t* __restrict__ idx, int k,
                                 __nv_bfloat16* __restrict__ out) {
  // warp w of the CTA handles slot s = blockIdx.y*8 + w, 32 consecutive k-positions per lane-loop
  const int s = blockIdx.y * 8 + (threadIdx.x >> 5);
  if (s >= k) return;
  const int64_t r = idx[s];
  for (int64_t t = int64_t(blockIdx.x) * 32 + (threadIdx.x & 31); t < K; t += int64_t(gridDim.x) * 32)
    out[int64_t(s) * K + t] = in[t * ld + r];
}
cudaError_t launch_gather(const void* in, int64_t K, int64_t ld, int kstrided,
                          const int32_t* idx, int k, __nv_bfloat16* out, cudaStream_t st) {
  const __nv_bfloat16* src = static_cast<const __nv_bfloat16*>(in);
  if (!kstrided) {
    const unsigned gx = unsigned(std::min<int64_t>((K / 8 + 255) / 256, int64_t(64)));
    k_gather_rows_kc<<<dim3(gx, unsigned(k)), 256, 0, st>>>(src, K, ld, idx, out);
  } else {
    const unsigned gx = unsigned(std::min<int64_t>((K + 31) / 32, int64_t(512)));
    k_gather_rows_ks<<<dim3(gx, unsigned((k + 7) / 8)), 256, 0, st>>>(src, K, ld, idx, k, out);
  }
  return cudaGetLastError();
}

// ================================================================== calibration stats
// Row statistics: one warp per row, fp64 accumulation, fixed-order shuffle reduction.
template <typename T>
__global__ void k_stats_rows(const T* __restrict__ in, int64_t R, int64_t C, int64_t ld,
                             double* __restrict__ rs) {
  const int64_t r = int64_t(blockIdx.x) * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= R) return;
  double s = 0, s2 = 0, sa = 0, mx = 0;
  for (int64_t j = lane; j < C; j += 32) {
    const double x = double(load_as_float(in, r * ld + j));
    s += x; s2 += x * x; sa += fabs(x); mx = fmax(mx, fabs(x));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    sa += __shfl_xor_sync(0xffffffffu, sa, o);
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if (lane == 0) {
    rs[r * 4 + 0] = s; rs[r * 4 + 1] = s2; rs[r * 4 + 2] = sa; rs[r * 4 + 3] = mx;
  }
}
// Column statistics, pass 1: thread per column over a chunk of rows.
template <typename T>
__global__ void k_stats_cols_part(const T* __restrict__ in, int64_t R, int64_t C, int64_t ld,
                                  int64_t rows_per_chunk, double* __restrict__ part) {
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= C) return;
  const int64_t r0 = int64_t(blockIdx.y) * rows_per_chunk;
  const int64_t r1 = min(R, r0 + rows_per_chunk);
  double s = 0, s2 = 0, sa = 0, mx = 0;
  for (int64_t r = r0; r < r1; ++r) {
    const double x = double(load_as_float(in, r * ld + j));
    s += x; s2 += x * x; sa += fabs(x); mx = fmax(mx, fabs(x));
  }
  double* p = part + (int64_t(blockIdx.y) * C + j) * 4;
  p[0] = s; p[1] = s2; p[2] = sa; p[3] = mx;
}
__global__ void k_stats_cols_reduce(const double* __restrict__ part, int64_t nch, int64_t C,
                                    double* __restrict__ cs) {
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= C) return;
  double s = 0, s2 = 0, sa = 0, mx = 0;
  for (int64_t c = 0; c < nch; ++c) {
    const double* p = part + (c * C + j) * 4;
    s += p[0]; s2 += p[1]; sa += p[2]; mx = fmax(mx, p[3]);
  }
  cs[j * 4 + 0] = s; cs[j * 4 + 1] = s2; cs[j * 4 + 2] = sa; cs[j * 4 + 3] = mx;
}

int64_t stats_chunks(int64_t R) { return (R + 511) / 512; }

cudaError_t launch_stats(const void* in, bool in_f32, int64_t R, int64_t C, int64_t ld,
                         double* rs, double* cs, double* part, cudaStream_t st) {
  const unsigned rb = unsigned((R + 7) / 8);
  const int64_t nch = stats_chunks(R);
  dim3 cg(unsigned((C + 255) / 256), unsigned(nch));
  if (in_f32) {
    const float* p = static_cast<const float*>(in);
    k_stats_rows<float><<<rb, 256, 0, st>>>(p, R, C, ld, rs);
    k_stats_cols_part<float><<<cg, 256, 0, st>>>(p, R, C, ld, 512, part);
  } else {
    const __nv_bfloat16* p = static_cast<const __nv_bfloat16*>(in);
    k_stats_rows<__nv_bfloat16><<<rb, 256, 0, st>>>(p, R, C, ld, rs);
    k_stats_cols_part<__nv_bfloat16><<<cg, 256, 0, st>>>(p, R, C, ld, 512, part);
  }
  k_stats_cols_reduce<<<unsigned((C + 255) / 256), 256, 0, st>>>(part, nch, C, cs);
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
  if (threadIdx.x == 0) {
    d_cv[0] = red[0][0];
    d_cv[1] = red[1][0];
    const double cv_row = red[0][0] / double(rows), cv_col = red[1][0] / double(cols);
    const bool row_hit = cv_col > tau, col_hit = cv_row > tau;
    uint8_t p = 0;
    if (row_hit && (!col_hit || cv_col >= cv_row)) p = 1;
    else if (col_hit) p = 2;
    pattern[0] = p;
  }
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
