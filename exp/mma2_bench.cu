// Microbenchmark (diagnostics): tcgen05.mma kind::f16 with cta_group::2 (CTA pair, M = 256)
// vs cta_group::1 (M = 128), K-major no-swizzle SMEM operands in the CNN kernel's geometry.
// One cluster of 2 CTAs per TPC (74 clusters); the leader CTA issues `iters` MMAs into one
// accumulator and commits to both CTAs' barriers.  Reports cycles per MMA and per-SM TFLOP/s.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
__host__ __device__ constexpr uint32_t make_idesc(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

template <int N, int PAIR>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) bench2(int iters, long long *out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tbase = tslot;
  long long t0 = clock64();
  const bool issuer = threadIdx.x == 0 && (!PAIR || rank == 0);
  if (issuer) {
    const uint32_t s0 = smem_u32(smem);
    const uint64_t ad = make_desc(s0, 2080, 128);                              // A: 128 rows per CTA
    const uint64_t bd = make_desc(s0 + 32768, (PAIR ? N / 2 : N) * 16, 128);   // B: N (or N/2 per CTA) rows
    const uint32_t id = make_idesc(PAIR ? 256 : 128, N);
    for (int i = 0; i < iters; ++i) {
      if (PAIR)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\t"
                     "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %4, p;\n\t}" ::"r"(tbase),
                     "l"(ad + (uint64_t)((i & 3) * 1)), "l"(bd), "r"(1), "r"(id));
      else
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %4, p;\n\t}" ::"r"(tbase),
                     "l"(ad + (uint64_t)((i & 3) * 1)), "l"(bd), "r"(1), "r"(id));
    }
    if (PAIR)
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                       smem_u32(&bar)), "h"((uint16_t)3));
    else
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
  }
  if (threadIdx.x == 0 && (issuer || PAIR)) {
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(&bar)));
    out[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) {
    if (PAIR) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tbase));
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
  }
}

template <int N, int PAIR>
void run() {
  const int ctas = 148;
  long long *d, h[148];
  cudaMalloc(&d, ctas * sizeof(long long));
  cudaMemset(d, 0, ctas * sizeof(long long));
  auto k = bench2<N, PAIR>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const int iters = 4096;
  k<<<ctas, 128, 64 * 1024>>>(64, d);
  cudaDeviceSynchronize();
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k<<<ctas, 128, 64 * 1024>>>(iters, d);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  int n = 0;
  for (int i = 0; i < ctas; ++i)
    if (h[i]) { avg += h[i]; ++n; }
  avg /= n > 0 ? n : 1;
  const int issuers = PAIR ? ctas / 2 : ctas;
  const double flops = 2.0 * (PAIR ? 256 : 128) * N * 16 * (double)iters * issuers;
  printf("%s N=%3d: %7.1f cyc/MMA instr  (per SM: 128x%dx16 in %5.1f cyc, ideal %5.1f)  %7.1f TFLOP/s  err=%s\n",
         PAIR ? "cta_group::2 M=256" : "cta_group::1 M=128", N, avg / iters, N, avg / iters, N / 2.0,
         flops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<96, 0>();
  run<96, 1>();
  run<64, 0>();
  run<64, 1>();
  run<32, 0>();
  run<32, 1>();
  run<128, 0>();
  run<128, 1>();
  run<256, 1>();
  return 0;
}
