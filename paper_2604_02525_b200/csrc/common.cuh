// common.cuh — shared definitions for the AdaHOP sm_100a kernels (not shared with oracle/).
#pragma once
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace adahop {

constexpr int kBlk = 32;  // MX block and Hadamard block along K

// ------------------------------------------------------------------------------------
// Scale-factor layout consumed by tcgen05 block-scaled MMA (one byte per 32-block).
// A "chunk" holds 128 rows x 4 K-blocks in 512 bytes:
//   byte = (r % 32) * 16 + ((r % 128) / 32) * 4 + (kb % 4)
// Chunks are tiled K-first: chunk index = (r / 128) * kchunks + kb / 4, where kchunks is
// the number of 4-block chunks per 128-row group, padded to a multiple of 2 (one GEMM
// stage = 256 K = 2 chunks). Copied to TMEM with tcgen05.cp 32x128b.warpx4 this puts the
// scale of row r, block kb at lane r, column word r/32, byte kb%4.
// ------------------------------------------------------------------------------------
__host__ __device__ inline int64_t sf_kchunks(int64_t K) { return ((K + 255) / 256) * 2; }
__host__ __device__ inline int64_t sf_bytes(int64_t R, int64_t K) {
  return ((R + 127) / 128) * sf_kchunks(K) * 512;
}
__host__ __device__ inline int64_t sf_offset(int64_t r, int64_t kb, int64_t kchunks) {
  return ((r >> 7) * kchunks + (kb >> 2)) * 512 + (r & 31) * 16 + ((r >> 5) & 3) * 4 + (kb & 3);
}

__device__ __forceinline__ float load_as_float(const __nv_bfloat16* p, int64_t i) {
  return __bfloat162float(p[i]);
}
__device__ __forceinline__ float load_as_float(const float* p, int64_t i) { return p[i]; }

// Position of v in a sorted device list of at most a few hundred indices, or -1.
__device__ __forceinline__ int find_sorted(const int32_t* idx, int n, int64_t v) {
  int lo = 0, hi = n - 1;
  while (lo <= hi) {
    const int mid = (lo + hi) >> 1;
    const int64_t x = __ldg(idx + mid);
    if (x == v) return mid;
    if (x < v) lo = mid + 1; else hi = mid - 1;
  }
  return -1;
}

}  // namespace adahop
