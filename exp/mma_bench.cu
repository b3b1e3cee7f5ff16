// Microbenchmark (diagnostics): tcgen05.mma kind::f16 M=128 throughput vs N, K-major
// no-swizzle SMEM operands (SS) and A-from-TMEM (TS).  One CTA per SM, one thread issues
// `iters` MMAs into one accumulator, then waits on a commit barrier; clock64 per CTA.
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
__host__ __device__ constexpr uint32_t make_idesc(int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

template <int N, bool TS, int NACC = 1, int ISS = 1>
__global__ void __launch_bounds__(128, 1) bench(int iters, long long *out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(ISS));
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
  const uint32_t tbase = tslot;
  long long t0 = 0, t1 = 0;
  if ((threadIdx.x & 31) == 0 && warp < ISS) {
    const uint32_t s0 = smem_u32(smem);
    const uint64_t ad = make_desc(s0, 2080, 128);             // A: 128 rows, activation-ring geometry
    const uint64_t bd = make_desc(s0 + 32768, N * 16, 128);   // B: N rows
    const uint32_t id = make_idesc(N);
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (TS) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %4, p;\n\t}" ::"r"(tbase),
            "r"(tbase + 256), "l"(bd), "r"(1), "r"(id));
      } else {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %4, p;\n\t}" ::"r"(tbase + (uint32_t)(((i % NACC) + warp * NACC) * N)),
            "l"(ad + (uint64_t)((i & 3) * 1)), "l"(bd), "r"(1), "r"(id));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    uint32_t ok = 0;
    while (!ok) {
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(&bar)));
    }
    t1 = clock64();
    if (warp == 0) out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

template <int N, bool TS, int NACC = 1, int ISS = 1>
void run(int sms) {
  long long *d;
  cudaMalloc(&d, sms * sizeof(long long));
  auto k = bench<N, TS, NACC, ISS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const int iters = 4096;
  k<<<sms, 128, 64 * 1024>>>(64, d);
  cudaDeviceSynchronize();
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k<<<sms, 128, 64 * 1024>>>(iters, d);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  long long h[256];
  cudaMemcpy(h, d, sms * sizeof(long long), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += h[i];
  avg /= sms;
  const double flops = 2.0 * 128 * N * 16 * (double)iters * sms * ISS;
  printf("N=%3d %s acc=%d issuers=%d: %7.1f cyc/MMA (ideal %5.1f)  %7.1f TFLOP/s  err=%s\n", N, TS ? "TS" : "SS", NACC, ISS, avg / iters / ISS,
         128.0 * N / 256.0, flops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  int sms = 148;
  run<32, false>(sms);
  run<64, false>(sms);
  run<96, false>(sms);
  run<128, false>(sms);
  run<192, false>(sms);
  run<256, false>(sms);
  run<32, true>(sms);
  run<96, true>(sms);
  run<256, true>(sms);
  run<32, false, 4>(sms);
  run<64, false, 4>(sms);
  run<96, false, 4>(sms);
  run<32, false, 1, 2>(sms);
  run<64, false, 1, 2>(sms);
  run<96, false, 1, 2>(sms);
  run<32, false, 2, 2>(sms);
  run<96, false, 2, 2>(sms);
  run<32, true, 4>(sms);
  run<64, true, 4>(sms);
  return 0;
}
