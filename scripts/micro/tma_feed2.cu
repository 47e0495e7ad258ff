// Microbenchmark (round 2, second pass): what limits the L2 -> SM delivery rate of TMA tile
// loads for ONE CTA per SM (profiles/r02d_tma_feed.txt: 1 CTA/SM ~31 B/clk/SM whatever the
// bytes in flight, 2 CTAs/SM ~62). Varies, one at a time: producer warps per CTA (each with its
// own ring), box rows (8/16/32 KB per instruction), CTAs per SM, L2 footprint, and the 2-CTA
// pattern of the GEMM (both CTAs' loads complete on the leader's barrier).
// Launch failures are detected (cudaGetLastError) and printed as SKIP.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tma_feed2.cu -o tma_feed2 -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void wait_parity(uint32_t bar, uint32_t ph) {
  asm volatile("{\n\t.reg .pred P;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W;\n\t}"
               ::"r"(bar), "r"(ph) : "memory");
}

struct P {
  int stages, boxes, rows_per_box, nprod, iters, rows_total, pair, lanes;   // lanes: issuing lanes of each producer warp
};

// nprod producer warps (lane 0 of warps 0..nprod-1), each owning `stages` stages of `boxes`
// boxes of rows_per_box x 128 B. pair=1: cluster of 2; every load signals the leader CTA's
// barrier for that (producer, stage) (as the 2-SM GEMM does), and both CTAs' producers wait on it.
template <bool kPair>
__global__ void k_feed(const __grid_constant__ CUtensorMap tm, P p, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  __shared__ __align__(8) uint64_t full[64];
  __shared__ __align__(8) uint64_t rel[64];   // pair: follower's "leader saw stage complete"
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  uint32_t rank = 0;
  if (kPair) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages * p.nprod; ++s)
    {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[s])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&rel[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (kPair) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  else __syncthreads();
  const unsigned long long t0 = clock64();
  if (warp < p.nprod && lane < p.lanes) {
    const uint32_t box_bytes = uint32_t(p.rows_per_box) * 128u;
    const uint32_t stage_bytes = uint32_t(p.boxes) * box_bytes;
    const int gid = kPair ? int(blockIdx.x / 2) : int(blockIdx.x);
    const int ng = kPair ? int(gridDim.x / 2) : int(gridDim.x);
    for (int i = 0; i < p.iters + p.stages; ++i) {
      const int s = i % p.stages;
      const int bi = warp * p.stages + s;
      const uint32_t bar_local = su32(&full[bi]);
      if (i >= p.stages) {
        const uint32_t ph = uint32_t((i / p.stages - 1) & 1);
        if (kPair && rank == 1) {
          wait_parity(su32(&rel[bi]), ph);
        } else {
          wait_parity(bar_local, ph);
          if (kPair) {
            uint32_t r;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(su32(&rel[bi])), "r"(1));
            asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(r) : "memory");
          }
        }
      }
      if (i >= p.iters) continue;
      uint32_t bar = bar_local;
      if (kPair) {
        // completion lands on the leader's barrier; the leader's barrier expects both CTAs' bytes
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(bar) : "r"(bar_local), "r"(0));
      }
      // the leader arms its own barrier for both CTAs' bytes (as the 2-SM GEMM does)
      if (rank == 0 && lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_local),
                     "r"(stage_bytes * (kPair ? 2u : 1u)) : "memory");
      for (int b = lane; b < p.boxes; b += p.lanes) {
        const long long unit = ((long long)i * ng + gid) * p.nprod * p.boxes * 2 + (warp * p.boxes + b) * 2 + rank;
        const int row = int(unit * p.rows_per_box % p.rows_total);
        const uint32_t dst = su32(base + size_t(bi * p.boxes + b) * box_bytes);
        if (kPair)
          asm volatile(
              "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
              ::"r"(dst), "l"(&tm), "r"(bar), "r"(0), "r"(row) : "memory");
        else
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
              ::"r"(dst), "l"(&tm), "r"(bar), "r"(0), "r"(row) : "memory");
      }
    }
  }
  if (kPair) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  else __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int rows = 1 << 18;  // 32 MB
  uint8_t* buf;
  cudaMalloc(&buf, size_t(rows) * 128);
  cudaMemset(buf, 1, size_t(rows) * 128);
  unsigned long long* cyc;
  cudaMalloc(&cyc, 8192 * 8);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap tms[3];
  const int box_rows[3] = {64, 128, 256};
  for (int k = 0; k < 3; ++k) {
    cuuint64_t dims[2] = {128, cuuint64_t(rows)}, strides[1] = {128};
    cuuint32_t box[2] = {128, cuuint32_t(box_rows[k])}, es[2] = {1, 1};
    reinterpret_cast<EncodeFn>(fn)(&tms[k], CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, buf, dims, strides, box, es,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  struct C { const char* what; int ctas_per_sm, stages, boxes, rows_per_box, nprod, rows_total, pair, lanes = 1; };
  const C cfgs[] = {
      {"baseline 1 CTA 1 prod 4x2 16KB", 1, 4, 2, 128, 1, rows, 0},
      {"1 CTA 1 prod 12x1 16KB", 1, 12, 1, 128, 1, rows, 0},
      {"1 CTA 1 prod 3x4 16KB", 1, 3, 4, 128, 1, rows, 0},
      {"1 CTA 1 prod 6x4 8KB boxes", 1, 6, 4, 64, 1, rows, 0},
      {"1 CTA 1 prod 3x2 32KB boxes", 1, 3, 2, 256, 1, rows, 0},
      {"1 CTA 2 prod warps 3x2 16KB each", 1, 3, 2, 128, 2, rows, 0},
      {"1 CTA 4 prod warps 3x1 16KB each", 1, 3, 1, 128, 4, rows, 0},
      {"1 CTA 2 prod warps 2x2 32KB each", 1, 2, 2, 256, 2, rows, 0},
      {"2 CTA/SM 1 prod 3x2 16KB", 2, 3, 2, 128, 1, rows, 0},
      {"1 CTA 1 prod 4x2 16KB, 2 MB footprint", 1, 4, 2, 128, 1, 1 << 14, 0},
      {"1 CTA 2 prod 3x2 16KB, 2 MB footprint", 1, 3, 2, 128, 2, 1 << 14, 0},
      {"1 CTA 1 prod 6x2 16KB", 1, 6, 2, 128, 1, rows, 0},
      {"1 CTA 1 prod warp, 2 issuing lanes, 4x2 16KB", 1, 4, 2, 128, 1, rows, 0, 2},
      {"1 CTA 1 prod warp, 4 issuing lanes, 3x4 16KB", 1, 3, 4, 128, 1, rows, 0, 4},
      {"1 CTA 3 prod warps 2x2 16KB each", 1, 2, 2, 128, 3, rows, 0},
      {"1 CTA 6 prod warps 2x1 16KB each", 1, 2, 1, 128, 6, rows, 0},
      {"1 CTA 8 prod warps 1x1 16KB each", 1, 1, 1, 128, 8, rows, 0},
      {"pair (cluster 2) 1 prod 4x2 16KB, leader barrier", 1, 4, 2, 128, 1, rows, 1},
      {"pair (cluster 2) 1 prod 6x2 16KB, leader barrier", 1, 6, 2, 128, 1, rows, 1},
      {"pair (cluster 2) 3 prod 2x2 16KB, leader barrier", 1, 2, 2, 128, 3, rows, 1},
      {"pair (cluster 2) 4 prod 3x1 16KB, leader barrier", 1, 3, 1, 128, 4, rows, 1},
      {"pair (cluster 2) 2 prod 3x2 16KB, leader barrier", 1, 3, 2, 128, 2, rows, 1},
  };
  for (const C& c : cfgs) {
    P p;
    p.stages = c.stages; p.boxes = c.boxes; p.rows_per_box = c.rows_per_box; p.nprod = c.nprod;
    p.iters = 3000; p.rows_total = c.rows_total; p.pair = c.pair; p.lanes = c.lanes;
    const int k = c.rows_per_box == 64 ? 0 : c.rows_per_box == 128 ? 1 : 2;
    const size_t smem = size_t(c.nprod) * c.stages * c.boxes * c.rows_per_box * 128 + 1024;
    auto kern = c.pair ? k_feed<true> : k_feed<false>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    int grid = nsm * c.ctas_per_sm;
    if (c.pair) grid &= ~1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = c.pair ? 2 : 1; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = c.pair ? 1 : 0;
    cudaError_t e = cudaSuccess;
    cudaMemset(cyc, 0, 8192 * 8);
    for (int r = 0; r < 2 && e == cudaSuccess; ++r) {
      e = cudaLaunchKernelEx(&cfg, kern, tms[k], p, cyc);
      if (e == cudaSuccess) e = cudaGetLastError();
    }
    cudaError_t e2 = cudaDeviceSynchronize();
    if (e != cudaSuccess || e2 != cudaSuccess) {
      printf("%-52s SKIP (%s / %s)\n", c.what, cudaGetErrorString(e), cudaGetErrorString(e2));
      cudaGetLastError();
      continue;
    }
    static unsigned long long hc[8192];
    cudaMemcpy(hc, cyc, grid * 8, cudaMemcpyDeviceToHost);
    unsigned long long mc = 0;
    for (int i = 0; i < grid; ++i) mc = hc[i] > mc ? hc[i] : mc;
    const double bytes = double(p.iters) * c.nprod * c.boxes * c.rows_per_box * 128.0 * grid;
    printf("%-52s %6.0f B/clk chip, %5.1f B/clk/SM, %5.2f TB/s at %d MHz (%3zu KB smem/CTA)\n", c.what, bytes / mc,
           bytes / mc / nsm, bytes / mc * clk_khz * 1e3 / 1e12, clk_khz / 1000, smem / 1024);
  }
  return 0;
}
