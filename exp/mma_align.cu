// Microbenchmark (diagnostics): does the TMEM column offset of an N = 96 accumulator window, or
// concurrent tcgen05.ld / tcgen05.st traffic from other warps, slow tcgen05.mma kind::f16
// (M = 128, K = 16, SS operands in the CNN kernel's activation-ring geometry)?  One CTA per SM;
// warp 0 lane 0 issues `iters` MMAs into D = base + off (+ an alternate window), warps 4-7 (one
// per TMEM lane quarter) optionally hammer other TMEM columns with ld/st while it runs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o exp/mma_align exp/mma_align.cu
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

// off1 / off2: TMEM column offsets of two accumulator windows used alternately (off2 < 0: one)
// noise: 0 none, 1 tcgen05.ld x16 loop, 2 ld + st loop on columns [400, 512)
__global__ void __launch_bounds__(256, 1) bench(int iters, int off1, int off2, int noise, int shift, long long *out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  __shared__ volatile int done;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
    done = 0;
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
  if (warp == 0) {
    long long t0 = 0, t1 = 0;
    if ((threadIdx.x & 31) == 0) {
      const uint32_t s0 = smem_u32(smem);
      const uint64_t ad = make_desc(s0, 2080, 128);
      const uint64_t bd = make_desc(s0 + 32768, 96 * 16, 128);
      const uint32_t id = make_idesc(96);
      t0 = clock64();
      for (int i = 0; i < iters; ++i) {
        const int off = (off2 >= 0 && (i & 1)) ? off2 : off1;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %4, p;\n\t}" ::"r"(tbase + (uint32_t)off),
            "l"(ad + (uint64_t)(shift == 0 ? 0 : shift == 4 ? (i & 3) : (i % 3))), "l"(bd), "r"(1), "r"(id));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
      uint32_t ok = 0;
      while (!ok) {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n\t}"
                     : "=r"(ok) : "r"(smem_u32(&bar)));
      }
      t1 = clock64();
      out[blockIdx.x] = t1 - t0;
      done = 1;
    }
  } else if (warp >= 4 && noise) {
    const uint32_t ta = tbase + ((uint32_t)((warp & 3) * 32) << 16) + 400;
    while (!done) {
      uint32_t r[16];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
            "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
          : "r"(ta) : "memory");
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (noise == 2) {
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(ta + 32),
            "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
            "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]) : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

void run(const char *name, int off1, int off2, int noise, int shift = 3) {
  const int sms = 148, iters = 4096;
  long long *d;
  cudaMalloc(&d, sms * sizeof(long long));
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  bench<<<sms, 256, 64 * 1024>>>(64, off1, off2, noise, shift, d);
  cudaDeviceSynchronize();
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  bench<<<sms, 256, 64 * 1024>>>(iters, off1, off2, noise, shift, d);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  long long h[148];
  cudaMemcpy(h, d, sms * sizeof(long long), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += h[i];
  avg /= sms;
  const double tf = 2.0 * 128 * 96 * 16 * (double)iters * sms / (ms * 1e-3) / 1e12;
  printf("%-34s %6.1f cycles/MMA  %7.1f TFLOP/s (%.3f ms)  err=%s\n", name, avg / iters, tf, ms, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run("N=96 A aligned (no shift)", 0, -1, 0, 0);
  run("N=96 A shift (i&3) x16B (r01 bench)", 0, -1, 0, 4);
  run("N=96 A shift (i%3) x16B", 0, -1, 0, 3);
  run("N=96 D@0", 0, -1, 0);
  run("N=96 D@32", 32, -1, 0);
  run("N=96 D@64 (crosses 128)", 64, -1, 0);
  run("N=96 D@96 (crosses 128)", 96, -1, 0);
  run("N=96 D@160 (crosses 256)", 160, -1, 0);
  run("N=96 D@128", 128, -1, 0);
  run("N=96 alternating D@0 / D@128", 0, 128, 0);
  run("N=96 alternating D@64 / D@224", 64, 224, 0);
  run("N=96 D@0 + TMEM ld noise", 0, -1, 1);
  run("N=96 D@0 + TMEM ld/st noise", 0, -1, 2);
  run("N=96 D@64 + TMEM ld/st noise", 64, -1, 2);
  return 0;
}
