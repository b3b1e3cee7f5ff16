// Diagnostics: cost of one SS tcgen05.mma (M = 128, K = 16, N = 96, bf16, no swizzle) as a function
// of how many DISTINCT A and B operand addresses a stream cycles through.  exp/mma_replay.cu shows
// the CNN chunk's own stream at ~73 cycles per N = 96 MMA vs 56 in exp/mma_swz.cu (2 B blocks, 3 A
// shifts); this isolates A-address and B-address diversity.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o exp/mma_div exp/mma_div.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__host__ __device__ inline uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
__host__ __device__ constexpr uint32_t make_idesc(int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t ad, uint64_t bd, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
               ::"r"(d), "l"(ad), "l"(bd), "r"(id), "r"(acc));
}
constexpr int GS = 2080;                       // A: [4 groups][130 positions][16 B] per row buffer (8,320 B)
constexpr int ABUF = 4 * GS, BBLK = 96 * 2 * 16;   // B block: [2 halves][96 rows][16 B] = 3 KB
constexpr int NA = 12, NB = 18;
constexpr uint32_t A0 = 0, B0 = NA * ABUF, TOTAL = B0 + NB * BBLK;

// stream of 36 MMAs per iteration; MMA i uses A address index (i % na) (+ dx shift i % 3 when na > 1)
// and B block (i % nb)
template <int NAU, int NBU, int ASH>
__global__ void __launch_bounds__(128, 1) kern(int iters, long long *cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (uint32_t e = threadIdx.x; e < TOTAL / 16; e += blockDim.x)
    reinterpret_cast<uint4 *>(smem)[e] = make_uint4(0x3c003c00u, 0, 0x3c00u, 0);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = tslot, sb = smem_u32(smem);
  if (threadIdx.x == 0) {
    const uint32_t id = make_idesc(96);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 36; ++i) {
        const uint32_t aa = sb + A0 + (uint32_t)((i % NAU) * ABUF) + (ASH ? (uint32_t)((i % 3) * 16) : 0u) +
                            (uint32_t)(((i / 3) & 1) * 2 * GS);
        const uint32_t ba = sb + B0 + (uint32_t)((i % NBU) * BBLK);
        mma(tb + 32u * (uint32_t)((i / 6) & 3), make_desc(aa, GS, 128), make_desc(ba, 96 * 16, 128), id, 1);
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(&bar)));
    cyc[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
}

template <int NAU, int NBU, int ASH>
void run() {
  long long *dC;
  cudaMalloc(&dC, 148 * 8);
  cudaFuncSetAttribute(kern<NAU, NBU, ASH>, cudaFuncAttributeMaxDynamicSharedMemorySize, TOTAL);
  kern<NAU, NBU, ASH><<<148, 128, TOTAL>>>(20, dC);
  cudaDeviceSynchronize();
  const int iters = 500;
  kern<NAU, NBU, ASH><<<148, 128, TOTAL>>>(iters, dC);
  cudaDeviceSynchronize();
  long long h[148]; cudaMemcpy(h, dC, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
  printf("A buffers %2d (dx shifts %d)  B blocks %2d : %6.1f cycles / N=96 MMA  %s\n", NAU, ASH, NBU, avg / (iters * 36.0),
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(dC);
}

int main() {
  printf("smem %u B\n", TOTAL);
  run<1, 1, 0>(); run<1, 2, 0>(); run<1, 6, 0>(); run<1, 18, 0>();
  run<1, 1, 1>(); run<3, 1, 1>(); run<12, 1, 1>();
  run<1, 6, 1>(); run<3, 6, 1>(); run<12, 6, 1>(); run<12, 18, 1>(); run<4, 18, 1>();
  return 0;
}
