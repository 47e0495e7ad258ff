// epilogue.cuh — GEMM epilogue stores through a per-warp shared-memory stage, and the OE patch.
//
// After tcgen05.ld (32x32b) lane i of an epilogue warp holds one accumulator ROW. Storing
// that directly makes every warp store touch 32 rows (32 L1 wavefronts per instruction);
// instead each lane writes its 128-byte row segment into a stage: a 128B-swizzled box that one
// TMA tensor store writes out (the pair GEMM), or a padded stage that the warp re-reads so
// that 8 consecutive lanes write one full 128-byte line of C (the LSU path).
#pragma once
#include <cstdint>
#include <cuda_bf16.h>

namespace adahop {

constexpr int kEpiPitch = 144;                // 128 B row + 16 B pad (bank spread, 16B aligned)
constexpr int kEpiStageBytes = 32 * kEpiPitch;  // per warp

__device__ __forceinline__ uint32_t pack_bf16x2(uint32_t lo, uint32_t hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(lo), __uint_as_float(hi));
  return *reinterpret_cast<uint32_t*>(&h);
}

// w[32]: this lane's 128-byte row segment. cbase: address of (row 0, first byte) of the
// 32-row block in global memory; ldc_bytes: row pitch; rows_valid / bytes_valid clip the
// M / N tails; elt: element size (2 or 4) for the tail path; vec_ok: 16-byte aligned rows.
// write this lane's 128-byte row segment into the warp's stage
__device__ __forceinline__ void epi_stage_row128(uint8_t* stg, const uint32_t (&w)[32]) {
  const int lane = threadIdx.x & 31;
  uint4* srow = reinterpret_cast<uint4*>(stg + lane * kEpiPitch);
#pragma unroll
  for (int j = 0; j < 8; ++j) srow[j] = make_uint4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
}

// coalesced copy of a staged 32-row x 128-byte block to global memory
__device__ __forceinline__ void epi_flush128(const uint8_t* stg, char* cbase, int64_t ldc_bytes, int rows_valid,
                                             int bytes_valid, int elt, bool vec_ok) {
  const int lane = threadIdx.x & 31;
  const int c = lane & 7;
#pragma unroll
  for (int it = 0; it < 8; ++it) {
    const int row = it * 4 + (lane >> 3);
    if (row < rows_valid) {
      const int b0 = c * 16;
      const uint8_t* src = stg + row * kEpiPitch + b0;
      char* dst = cbase + int64_t(row) * ldc_bytes + b0;
      if (vec_ok && b0 + 16 <= bytes_valid) {
        *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(src);
      } else if (b0 < bytes_valid) {
        const int end = min(b0 + 16, bytes_valid);
        if (elt == 4) {
          for (int b = b0; b < end; b += 4)
            *reinterpret_cast<uint32_t*>(dst + (b - b0)) = *reinterpret_cast<const uint32_t*>(src + (b - b0));
        } else {
          for (int b = b0; b < end; b += 2)
            *reinterpret_cast<uint16_t*>(dst + (b - b0)) = *reinterpret_cast<const uint16_t*>(src + (b - b0));
        }
      }
    }
  }
}

__device__ __forceinline__ void epi_store_rows128(uint8_t* stg, const uint32_t (&w)[32], char* cbase,
                                                  int64_t ldc_bytes, int rows_valid, int bytes_valid,
                                                  int elt, bool vec_ok) {
  const int lane = threadIdx.x & 31;
  uint4* srow = reinterpret_cast<uint4*>(stg + lane * kEpiPitch);
#pragma unroll
  for (int j = 0; j < 8; ++j) srow[j] = make_uint4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
  __syncwarp();
  const int c = lane & 7;
#pragma unroll
  for (int it = 0; it < 8; ++it) {
    const int row = it * 4 + (lane >> 3);
    if (row < rows_valid) {
      const int b0 = c * 16;
      const uint8_t* src = stg + row * kEpiPitch + b0;
      char* dst = cbase + int64_t(row) * ldc_bytes + b0;
      if (vec_ok && b0 + 16 <= bytes_valid) {
        *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(src);
      } else if (b0 < bytes_valid) {
        const int end = min(b0 + 16, bytes_valid);
        if (elt == 4) {
          for (int b = b0; b < end; b += 4)
            *reinterpret_cast<uint32_t*>(dst + (b - b0)) = *reinterpret_cast<const uint32_t*>(src + (b - b0));
        } else {
          for (int b = b0; b < end; b += 2)
            *reinterpret_cast<uint16_t*>(dst + (b - b0)) = *reinterpret_cast<const uint16_t*>(src + (b - b0));
        }
      }
    }
  }
  __syncwarp();
}

// OE outlier values written into C by the MXFP4 GEMM epilogue ("Fused Scatter-Add"):
// the residual operand has the OE rows (OE-Left) / columns (OE-Right) zeroed, so the main
// product is exactly 0 there and those entries of C are the BF16 outlier product alone:
//   OE-Right (mode 1): C[m][idx[j]] = Dt[j][m]       OE-Left (mode 2): C[idx[j]][n] = Dt[j][n]
// with Dt the split-K-folded, transposed outlier product (launch_outlier_fold). With `ticket`
// (the wgrad product fused into the quant pass, quant_tc.cu) Dt is first folded by the GEMM's own
// epilogue threads from the quant pass's per-(band, CTA) partials, in CTA order:
//   Dt[j][m] = sum_s part[m / 128][s][j][m % 128],  s < the band's slot count,
// each CTA a disjoint share while its first main loop runs; every CTA then counts itself in on
// `ticket` (zeroed by the quant pass) and the first patch waits for all of them (the persistent
// grid is co-resident).
struct OePatch {
  const float* Dt;         // [k][Mb]
  const int32_t* idx;      // sorted, k entries
  int64_t Mb;
  int k, mode;             // mode 0: none
  const float* part = nullptr;   // [Mb / 128 bands][spb][npad][128]
  unsigned* ticket = nullptr;
  int spb = 0, npad = 0;
  int or_n = 0, or_rtiles = 0, or_chunks = 0;   // the quant pass's chunking (see qtc::OrSpec)
};
__device__ __forceinline__ float oe_fold_value(const OePatch& op, int j, int64_t m) {
  const int ct = int(m >> 7);
  const int64_t u0 = int64_t(ct) * op.or_rtiles;
  const int64_t u1 = min(int64_t(op.or_n), u0 + op.or_rtiles) - 1;
  const int nslots = int(((u1 + 1) * op.or_chunks - 1) / op.or_n - ((u0 + 1) * op.or_chunks - 1) / op.or_n) + 1;
  const float* p = op.part + (int64_t(ct) * op.spb * op.npad + j) * 128 + (m & 127);
  const int64_t stride = int64_t(op.npad) * 128;
  float v = 0.f;
  int s = 0;
  for (; s + 4 <= nslots; s += 4) {   // independent loads, summed in slot order
    const float a = __ldg(p + s * stride), b = __ldg(p + (s + 1) * stride);
    const float c = __ldg(p + (s + 2) * stride), d = __ldg(p + (s + 3) * stride);
    v = (((v + a) + b) + c) + d;
  }
  for (; s < nslots; ++s) v += __ldg(p + s * stride);
  return v;
}
// All epilogue threads of the CTA (tid < nthreads, named barrier `bar`): fold this CTA's share.
__device__ __forceinline__ void oe_prefold(const OePatch& op, int tid, int nthreads, uint32_t bar) {
  if (op.ticket == nullptr) return;
  const int64_t total = int64_t(op.k) * op.Mb;
  const int64_t per = (total + gridDim.x - 1) / gridDim.x;
  const int64_t lo = per * blockIdx.x, hi = min(total, lo + per);
  float* dt = const_cast<float*>(op.Dt);
  for (int64_t e = lo + tid; e < hi; e += nthreads) {
    const int j = int(e / op.Mb);
    dt[e] = oe_fold_value(op, j, e - int64_t(j) * op.Mb);
  }
  __threadfence();
  asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(nthreads) : "memory");
  if (tid == 0) atomicAdd(op.ticket, 1u);
}
// Whole warp, before its first patch: every CTA has folded its share.
__device__ __forceinline__ void oe_prefold_wait(const OePatch& op) {
  if (op.ticket == nullptr) return;
  if ((threadIdx.x & 31) == 0) {
    uint32_t v;
    for (;;) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(op.ticket) : "memory");
      if (v >= gridDim.x) break;
      __nanosleep(100);
    }
  }
  __syncwarp();
}
// Dt[j][m] (m: the row of C for OE-Right, its column for OE-Left); values written in this kernel
// (pre-fold) are read through L2, never the non-coherent path
__device__ __forceinline__ float oe_patch_value(const OePatch& op, int j, int64_t m) {
  return op.ticket ? __ldcg(op.Dt + int64_t(j) * op.Mb + m) : __ldg(op.Dt + int64_t(j) * op.Mb + m);
}

// [j0, j1) = the entries of sorted idx in [lo, hi): one pass of the warp over idx (k <= 256)
__device__ __forceinline__ void idx_range(const int32_t* __restrict__ idx, int k, int64_t lo, int64_t hi, int& j0,
                                          int& j1) {
  const int lane = threadIdx.x & 31;
  int below = 0, inside = 0;
  for (int b = 0; b < k; b += 32) {
    const int64_t v = b + lane < k ? int64_t(__ldg(idx + b + lane)) : hi;
    below += __popc(__ballot_sync(~0u, v < lo));
    inside += __popc(__ballot_sync(~0u, v >= lo && v < hi));
  }
  j0 = below;
  j1 = below + inside;
}

// Byte offset of (row, byte) in a warp's 32 x 128-byte stage: padded rows (LSU flush) or the
// 128B-swizzled box a TMA store reads (16-byte chunk j of row r at chunk j ^ (r % 8)).
template <bool kSw128>
__device__ __forceinline__ int epi_stage_off(int row, int byte) {
  return kSw128 ? row * 128 + ((((byte >> 4) ^ (row & 7)) << 4) | (byte & 15)) : row * kEpiPitch + byte;
}

// Patch the staged 32-row block (rows m0 .. m0+31, columns n0 .. n0+ncols-1) of C in the warp's
// smem stage; call between staging and flushing (whole warp).
template <bool kSw128 = false>
__device__ __forceinline__ void epi_patch_outliers(uint8_t* stg, const OePatch& op, int64_t m0, int64_t n0,
                                                   int ncols, int elt, int64_t M, int64_t N) {
  if (op.mode == 0) return;
  const int lane = threadIdx.x & 31;
  int j0, j1;
  if (op.mode == 1) idx_range(op.idx, op.k, n0, n0 + ncols, j0, j1);
  else idx_range(op.idx, op.k, m0, m0 + 32, j0, j1);
  if (j0 == j1) return;
  __syncwarp();
  if (op.mode == 1) {   // columns idx[j] in [n0, n0 + ncols): lane = row
    const int64_t m = m0 + lane;
    if (m < M)
      for (int j = j0; j < j1; ++j) {
        const int cl = int(__ldg(op.idx + j) - n0);
        const float v = oe_patch_value(op, j, m);
        uint8_t* dst = stg + epi_stage_off<kSw128>(lane, cl * elt);
        if (elt == 4) *reinterpret_cast<float*>(dst) = v;
        else *reinterpret_cast<__nv_bfloat16*>(dst) = __float2bfloat16_rn(v);
      }
  } else {              // rows idx[j] in [m0, m0 + 32): lane = column
    for (int j = j0; j < j1; ++j) {
      const int rl = int(__ldg(op.idx + j) - m0);
      for (int c = lane; c < ncols; c += 32) {
        const int64_t n = n0 + c;
        if (n >= N) continue;
        const float v = oe_patch_value(op, j, n);
        uint8_t* dst = stg + epi_stage_off<kSw128>(rl, c * elt);
        if (elt == 4) *reinterpret_cast<float*>(dst) = v;
        else *reinterpret_cast<__nv_bfloat16*>(dst) = __float2bfloat16_rn(v);
      }
    }
  }
  __syncwarp();
}

// this lane's 128-byte row segment into a 128B-swizzled 32 x 128-byte stage (a TMA store box)
__device__ __forceinline__ void epi_stage_sw128(uint8_t* stg, const uint32_t (&w)[32]) {
  const int lane = threadIdx.x & 31;
  uint8_t* srow = stg + lane * 128;
#pragma unroll
  for (int j = 0; j < 8; ++j)
    *reinterpret_cast<uint4*>(srow + ((j ^ (lane & 7)) << 4)) = make_uint4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
}

__device__ __forceinline__ void epi_stage_only128(uint8_t* stg, const uint32_t (&w)[32]) {
  const int lane = threadIdx.x & 31;
  uint4* srow = reinterpret_cast<uint4*>(stg + lane * kEpiPitch);
#pragma unroll
  for (int j = 0; j < 8; ++j) srow[j] = make_uint4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
  __syncwarp();
}

}  // namespace adahop
