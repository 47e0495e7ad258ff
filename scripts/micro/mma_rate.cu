// Microbenchmark: tcgen05.mma.kind::f16 (bf16 -> f32) issue-to-completion cost per instruction
// for M = 128 and several N / operand layouts. One CTA per SM, one elected thread issues.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t sdesc(uint32_t a, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return uint64_t((a >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) | (uint64_t((sbo >> 4) & 0x3FFF) << 32) |
         (1ull << 46) | (uint64_t(layout & 7) << 61);
}
__host__ __device__ constexpr uint32_t idesc(int n, int a_mn, int b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(a_mn) << 15) | (uint32_t(b_mn) << 16) | (uint32_t(n >> 3) << 17) |
         (uint32_t(128 >> 4) << 24);
}

// kNoise: 0 none, 1 = warps 1..15 stream tcgen05.ld from TMEM cols [256,512), 2 = warps 1..15 hammer smem
template <int N, int kBLayout, int kAmn, int kNoise>
__global__ void k(int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0x3f803f80u * (i & 1);
  if (threadIdx.x == 0) *reinterpret_cast<uint32_t*>(base + 65536) = 0;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (threadIdx.x == 0) {
    const uint32_t a = su32(base), b = su32(base + 32768);
    const uint64_t ad = kAmn ? sdesc(a, 16384, 1024, 2) : sdesc(a, 16, 1024, 2);
    const uint64_t bd = kBLayout == 0 ? sdesc(b, 128, 512, 0) : sdesc(b, 16, 1024, 2);
    const uint32_t id = idesc(N, kAmn, 0);
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t d = slot + (N <= 64 ? (i & 3) * 64 : 0);
      const uint64_t aoff = kAmn ? uint64_t(((i & 7) * 16 * 128) >> 4) : uint64_t(((i & 3) * 32) >> 4);
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                   ::"r"(d), "l"(ad + aoff), "l"(bd), "r"(id), "r"(i & 1));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
    asm volatile("{\n\t.reg .pred P;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n\t@!P bra W;\n\t}" ::"r"(su32(&bar)));
    const long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
    *reinterpret_cast<volatile uint32_t*>(&slot + 0) = slot;   // keep
    asm volatile("st.shared.u32 [%0], 1;" ::"r"(su32(base + 65536)));
  } else if (kNoise && threadIdx.x >= 32) {
    volatile uint32_t* flag = reinterpret_cast<volatile uint32_t*>(base + 65536);
    uint32_t acc = 0;
    const int w = threadIdx.x >> 5;
    while (*flag == 0) {
      if (kNoise == 1) {
        uint32_t r[32];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
            "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
              "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
              "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
              "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
              "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
            : "r"(slot + (((w & 3) * 32) << 16) + 256 + (w >> 2) * 32));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int j = 0; j < 32; ++j) acc += r[j];
      } else {
        uint32_t x0, x1, x2, x3;
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(x0), "=r"(x1), "=r"(x2), "=r"(x3)
                     : "r"(su32(base + 70000 + (threadIdx.x & 255) * 16)));
        asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(su32(base + 70000 + ((threadIdx.x + 7) & 255) * 16)),
                     "r"(x0 + 1), "r"(x1), "r"(x2), "r"(x3));
        acc += x0;
      }
    }
    if (acc == 12345) out[1] = acc;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

template <int N, int BL, int AMN, int NOISE = 0>
void run(const char* name, long long* d) {
  const int iters = 4096;
  cudaFuncSetAttribute(k<N, BL, AMN, NOISE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  for (int r = 0; r < 2; ++r) k<N, BL, AMN, NOISE><<<148, NOISE ? 512 : 128, 100000>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long c;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  printf("%-28s noise=%d N=%3d: %6.1f cycles/MMA  (ideal 128*N/256 = %d)  %s\n", name, NOISE, N, double(c) / iters, 128 * N / 256,
         cudaGetErrorString(e));
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  run<32, 0, 0>("A K-major SW128, B none", d);
  run<64, 0, 0>("A K-major SW128, B none", d);
  run<128, 0, 0>("A K-major SW128, B none", d);
  run<256, 0, 0>("A K-major SW128, B none", d);
  run<32, 1, 0>("A K-major SW128, B SW128", d);
  run<64, 1, 0>("A K-major SW128, B SW128", d);
  run<128, 1, 0>("A K-major SW128, B SW128", d);
  run<32, 0, 1>("A MN-major SW128, B none", d);
  run<128, 0, 1>("A MN-major SW128, B none", d);
  run<32, 1, 1>("A MN-major SW128, B SW128", d);
  run<32, 0, 0, 1>("A K-major SW128, B none", d);
  run<32, 0, 1, 1>("A MN-major SW128, B none", d);
  run<128, 0, 0, 1>("A K-major SW128, B none", d);
  run<32, 0, 0, 2>("A K-major SW128, B none", d);
  run<32, 0, 1, 2>("A MN-major SW128, B none", d);
  return 0;
}
