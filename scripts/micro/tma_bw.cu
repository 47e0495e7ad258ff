// Microbenchmark: TMA L2->smem delivery rate for (a) distinct tiles per CTA, (b) the same tile
// loaded by every CTA of a cluster (unicast), (c) the same tile multicast to the cluster.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tma_bw.cu -lcuda -o tma_bw
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

constexpr int kStages = 4;
constexpr int kBox = 16384;   // 128 rows x 128 B

template <int kMode>   // 0 distinct, 1 same-unicast, 2 multicast
__global__ void __cluster_dims__(1, 1, 1) dummy() {}

template <int kMode>
__global__ void k(const __grid_constant__ CUtensorMap tm, int iters, int rows_total, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  __shared__ __align__(8) uint64_t full[kStages];
  uint32_t csize, crank;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(csize));
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("barrier.cluster.arrive.release;\n\tbarrier.cluster.wait.acquire;");
  const long long t0 = clock64();
  if (threadIdx.x == 0) {
    const int cluster_id = blockIdx.x / csize;
    const int nclusters = gridDim.x / csize;
    for (int i = 0; i < iters; ++i) {
      const int s = i % kStages;
      const uint32_t ph = (i / kStages) & 1;
      if (i >= kStages) {
        asm volatile("{\n\t.reg .pred P;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W;\n\t}"
                     ::"r"(su32(&full[s])), "r"(ph ^ 1));
        asm volatile("barrier.cluster.arrive.release;" ::: "memory");   // (no-op sync pattern below)
        asm volatile("barrier.cluster.wait.acquire;" ::: "memory");
      }
      // tile index: distinct per CTA (mode 0) or per cluster (modes 1,2)
      const int tile = kMode == 0 ? (i * gridDim.x + blockIdx.x) : (i * nclusters + cluster_id);
      const int row = (tile * 128) % rows_total;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(kBox * 2));
      uint8_t* dst = base + s * 2 * kBox;
      if (kMode != 2) {
        for (int h = 0; h < 2; ++h)
          asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                       ::"r"(su32(dst + h * kBox)), "l"(&tm), "r"(su32(&full[s])), "r"(h * 128), "r"(row) : "memory");
      } else {
        // each rank loads 1/csize of the 256 rows... here: rank r loads row-slab r of the tile, multicast to all
        const uint16_t mask = uint16_t((1u << csize) - 1);
        const int slab = 128 / csize;
        for (int h = 0; h < 2; ++h)
          asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%3, %4}], [%2], %5;"
                       ::"r"(su32(dst + h * kBox + crank * slab * 128)), "l"(&tm), "r"(su32(&full[s])), "r"(h * 128),
                       "r"(row + int(crank) * slab), "h"(mask) : "memory");
      }
    }
    for (int i = iters; i < iters + kStages; ++i) {
      const int s = i % kStages;
      const uint32_t ph = (i / kStages) & 1;
      asm volatile("{\n\t.reg .pred P;\n\tW2: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W2;\n\t}"
                   ::"r"(su32(&full[s])), "r"(ph ^ 1));
    }
  } else {
    for (int i = kStages; i < iters; ++i) {
      asm volatile("barrier.cluster.arrive.release;" ::: "memory");
      asm volatile("barrier.cluster.wait.acquire;" ::: "memory");
    }
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int rows = 1 << 17;   // 131072 rows x 256 B = 32 MB (L2-resident after first touch)
  uint8_t* buf;
  cudaMalloc(&buf, size_t(rows) * 256);
  cudaMemset(buf, 1, size_t(rows) * 256);
  unsigned long long* out;
  cudaMalloc(&out, 1024 * 8);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap tm;
  cuuint64_t dims[2] = {256, cuuint64_t(rows)}, strides[1] = {256};
  cuuint32_t box[2] = {128, 128}, es[2] = {1, 1};
  reinterpret_cast<EncodeFn>(fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, buf, dims, strides, box, es,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int iters = 2000;
  const size_t smem = kStages * 2 * kBox + 1024;
  for (int mode = 0; mode < 3; ++mode) {
    for (int cs : {1, 2, 4, 8}) {
      if (mode == 2 && cs == 1) continue;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(144);   // multiple of 8 clusters
      cfg.blockDim = dim3(32);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
      cudaError_t e;
      void (*kf)(const CUtensorMap, int, int, unsigned long long*) =
          mode == 0 ? k<0> : (mode == 1 ? k<1> : k<2>);
      cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      cudaFuncSetAttribute(kf, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      for (int r = 0; r < 2; ++r) e = cudaLaunchKernelEx(&cfg, kf, tm, iters, rows, out);
      cudaError_t e2 = cudaDeviceSynchronize();
      unsigned long long c[144];
      cudaMemcpy(c, out, sizeof(c), cudaMemcpyDeviceToHost);
      unsigned long long mx = 0;
      for (int i = 0; i < 144; ++i) mx = c[i] > mx ? c[i] : mx;
      const double delivered = double(iters) * 2 * kBox * 144;   // bytes landed in smem
      printf("mode %d (%s) cluster %d: delivered %.0f B/cyc chip-wide (%s/%s)\n", mode,
             mode == 0 ? "distinct" : mode == 1 ? "same-unicast" : "multicast", cs, delivered / mx,
             cudaGetErrorString(e), cudaGetErrorString(e2));
    }
  }
  return 0;
}
