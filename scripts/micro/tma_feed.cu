// Microbenchmark: chip-wide L2 -> SM delivery rate of TMA tile loads (the MXFP4 GEMM's operand
// feed). Every CTA streams 128-row x 128-byte boxes (16 KB, 128B swizzle, as the GEMM's A/B
// loads) from an L2-resident buffer through an S-stage ring, one thread re-issuing each stage as
// soon as it lands (no consumer work). Reports bytes per SM clock and TB/s (globaltimer).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tma_feed.cu -o tma_feed
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void k_feed(const __grid_constant__ CUtensorMap tm, int stages, int boxes_per_stage, int iters, int rows_total,
                       unsigned long long* cyc, unsigned long long* ns) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  __shared__ __align__(8) uint64_t full[16];
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  unsigned long long t0, g0, t1, g1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  t0 = clock64();
  if (threadIdx.x == 0) {
    const uint32_t stage_bytes = uint32_t(boxes_per_stage) * 16384u;
    for (int i = 0; i < iters + stages; ++i) {
      const int s = i % stages;
      if (i >= stages) {
        const uint32_t ph = uint32_t((i / stages - 1) & 1);
        asm volatile("{\n\t.reg .pred P;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W;\n\t}"
                     ::"r"(su32(&full[s])), "r"(ph) : "memory");
      }
      if (i >= iters) continue;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(stage_bytes)
                   : "memory");
      for (int b = 0; b < boxes_per_stage; ++b) {
        const int row = int((((long long)i * gridDim.x + blockIdx.x) * boxes_per_stage + b) * 128 % rows_total);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
            ::"r"(su32(base + (s * boxes_per_stage + b) * 16384)), "l"(&tm), "r"(su32(&full[s])), "r"(0), "r"(row)
            : "memory");
      }
    }
  }
  __syncthreads();
  t1 = clock64();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  if (threadIdx.x == 0) {
    cyc[blockIdx.x] = t1 - t0;
    ns[blockIdx.x] = g1 - g0;
  }
}

// Multicast variant: clusters of cs CTAs; CTA r loads row slab r of every box and multicasts it to
// all cs CTAs (each CTA receives whole boxes, L2 serves each byte once per cluster). A stage is
// re-armed only after every CTA of the cluster has seen it land (remote arrives on `empty`).
__global__ void k_feed_mc(const __grid_constant__ CUtensorMap tm, int stages, int boxes_per_stage, int iters,
                          int rows_total, unsigned long long* cyc, unsigned long long* ns) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  __shared__ __align__(8) uint64_t full[16];
  __shared__ __align__(8) uint64_t empty[16];
  uint32_t cs, cr;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(cs));
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(cr));
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[s])), "r"(cs));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  unsigned long long t0, g0, t1, g1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  t0 = clock64();
  if (threadIdx.x == 0) {
    const uint32_t stage_bytes = uint32_t(boxes_per_stage) * 16384u;
    const int slab = 128 / int(cs);
    const uint16_t mask = uint16_t((1u << cs) - 1);
    const int cluster = blockIdx.x / int(cs), nclusters = gridDim.x / int(cs);
    for (int i = 0; i < iters + stages; ++i) {
      const int s = i % stages;
      if (i >= stages) {
        const uint32_t ph = uint32_t((i / stages - 1) & 1);
        asm volatile("{\n\t.reg .pred P;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W;\n\t}"
                     ::"r"(su32(&full[s])), "r"(ph) : "memory");
        // tell every CTA of the cluster that this CTA's copy of stage s has landed
        for (uint32_t c = 0; c < cs; ++c) {
          uint32_t remote;
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(su32(&empty[s])), "r"(c));
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
        }
        // every CTA has it: the stage may be re-filled
        asm volatile("{\n\t.reg .pred P;\n\tW2: mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%0], %1;\n\t@!P bra W2;\n\t}"
                     ::"r"(su32(&empty[s])), "r"(ph) : "memory");
      }
      if (i >= iters) continue;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(stage_bytes)
                   : "memory");
      for (int b = 0; b < boxes_per_stage; ++b) {
        const int row = int((((long long)i * nclusters + cluster) * boxes_per_stage + b) * 128 % rows_total);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster "
            "[%0], [%1, {%3, %4}], [%2], %5;"
            ::"r"(su32(base + (s * boxes_per_stage + b) * 16384 + int(cr) * slab * 128)), "l"(&tm),
            "r"(su32(&full[s])), "r"(0), "r"(row + int(cr) * slab), "h"(mask)
            : "memory");
      }
    }
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  t1 = clock64();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  if (threadIdx.x == 0) {
    cyc[blockIdx.x] = t1 - t0;
    ns[blockIdx.x] = g1 - g0;
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int rows = 1 << 18;   // 262144 rows x 128 B = 32 MB: L2-resident after the first pass
  uint8_t* buf;
  cudaMalloc(&buf, size_t(rows) * 128);
  cudaMemset(buf, 1, size_t(rows) * 128);
  unsigned long long *cyc, *ns;
  cudaMalloc(&cyc, 4096 * 8);
  cudaMalloc(&ns, 4096 * 8);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap tm;
  cuuint64_t dims[2] = {128, cuuint64_t(rows)}, strides[1] = {128};
  cuuint32_t box[2] = {128, 128}, es[2] = {1, 1};
  reinterpret_cast<EncodeFn>(fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, buf, dims, strides, box, es,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUtensorMap tms[3];   // slab boxes for cluster sizes 2, 4, 8
  for (int k = 0; k < 3; ++k) {
    cuuint32_t bx[2] = {128, cuuint32_t(128 >> (k + 1))};
    reinterpret_cast<EncodeFn>(fn)(&tms[k], CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, buf, dims, strides, bx, es,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 4000;
  struct Cfg { int ctas_per_sm, stages, boxes; };
  for (Cfg c : {Cfg{1, 4, 2}, Cfg{1, 6, 2}, Cfg{1, 10, 2}, Cfg{1, 6, 4}, Cfg{2, 3, 2}, Cfg{2, 6, 1}}) {
    const size_t smem = size_t(c.stages) * c.boxes * 16384 + 1024;
    cudaFuncSetAttribute(k_feed, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    const int grid = nsm * c.ctas_per_sm;
    for (int r = 0; r < 2; ++r) k_feed<<<grid, 32, smem>>>(tm, c.stages, c.boxes, iters, rows, cyc, ns);
    cudaError_t e = cudaDeviceSynchronize();
    static unsigned long long hc[4096], hn[4096];
    cudaMemcpy(hc, cyc, grid * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(hn, ns, grid * 8, cudaMemcpyDeviceToHost);
    unsigned long long mc = 0, mn = 0;
    for (int i = 0; i < grid; ++i) { mc = hc[i] > mc ? hc[i] : mc; mn = hn[i] > mn ? hn[i] : mn; }
    const double bytes = double(iters) * c.boxes * 16384 * grid;
    printf("ctas/SM %d stages %d boxes/stage %d (%3d KB in flight per SM): %6.0f B/clk chip, %5.1f B/clk/SM, %5.2f TB/s (%s)\n",
           c.ctas_per_sm, c.stages, c.boxes, c.ctas_per_sm * c.stages * c.boxes * 16, bytes / mc, bytes / mc / nsm,
           bytes / mn / 1e3, cudaGetErrorString(e));
  }
  for (int k = 0; k < 3; ++k) {
    const int csz = 2 << k;
    const int stages = 6, boxes = 2;
    const size_t smem = size_t(stages) * boxes * 16384 + 1024;
    cudaFuncSetAttribute(k_feed_mc, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    const int grid = (nsm / csz) * csz;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(32);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = csz; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaError_t e = cudaSuccess;
    for (int r = 0; r < 2; ++r) e = cudaLaunchKernelEx(&cfg, k_feed_mc, tms[k], stages, boxes, iters, rows, cyc, ns);
    cudaError_t e2 = cudaDeviceSynchronize();
    static unsigned long long hc[4096], hn[4096];
    cudaMemcpy(hc, cyc, grid * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(hn, ns, grid * 8, cudaMemcpyDeviceToHost);
    unsigned long long mc = 0, mn = 0;
    for (int i = 0; i < grid; ++i) { mc = hc[i] > mc ? hc[i] : mc; mn = hn[i] > mn ? hn[i] : mn; }
    const double bytes = double(iters) * boxes * 16384 * grid;   // delivered into smem
    printf("multicast cluster %d, stages %d boxes %d: delivered %6.0f B/clk chip (%5.1f B/clk/SM, %5.2f TB/s), "
           "L2 reads %5.2f TB/s (%s/%s)\n", csz, stages, boxes, bytes / mc, bytes / mc / grid, bytes / mn / 1e3,
           bytes / csz / mn / 1e3, cudaGetErrorString(e), cudaGetErrorString(e2));
  }
  return 0;
}
