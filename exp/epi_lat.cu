// Diagnostics: latency of the CNN epilogue's steps, on an idle tensor pipe and while warp 0 issues
// the chunk-1 MMA stream (exp/mma_noise.cu).  Warp 1 (TMEM lane quarter 1) loops over:
//   A  tcgen05.ld 32x32b.x16 x2 + tcgen05.wait::ld
//   B  tcgen05.st 32x32b.x16 x2 (zeros) + tcgen05.wait::st
//   C  4 x STS.128 + fence.proxy.async.shared::cta + __syncwarp
//   D  mbarrier arrive (lane 0) + try_wait on a barrier of count 1 (round trip)
// and reports the mean cycles per step (clock64 around each).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o exp/epi_lat exp/epi_lat.cu
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
__device__ __forceinline__ bool elect_one() {
  uint32_t pred;
  asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t ad, uint64_t bd, uint32_t id) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
               ::"r"(d), "l"(ad), "l"(bd), "r"(id));
}
constexpr int P = 32, GS = 130 * 16;
constexpr uint32_t TOTAL = 200 * 1024, SCR = 176 * 1024;

template <int S>
__device__ __forceinline__ void fill(uint32_t acc0, uint32_t a0, uint32_t b0) {
  constexpr int n1 = (4 - S < 3 ? 4 - S : 3);
  constexpr int n2 = 3 - n1;
#pragma unroll
  for (int dx = 0; dx < 3; ++dx)
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      const uint64_t ad = make_desc(a0 + 2 * ks * GS + dx * 16, GS, 128);
      const uint32_t bb = b0 + (dx * 2 + ks) * 96 * 32;
      mma(acc0 + S * P, ad, make_desc(bb, 96 * 16, 128), make_idesc(n1 * P));
      if (n2 > 0) mma(acc0, ad, make_desc(bb + n1 * P * 16, 96 * 16, 128), make_idesc(n2 * P));
    }
}

template <int BUSY>
__global__ void __launch_bounds__(128, 1) kern(int iters, long long *out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar, mb;
  __shared__ volatile int stop;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (uint32_t e = threadIdx.x; e < TOTAL / 16; e += blockDim.x)
    reinterpret_cast<uint4 *>(smem)[e] = make_uint4(0x3c003c00u, 0, 0x3c00u, 0);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mb)));
    asm volatile("fence.mbarrier_init.release.cluster;");
    stop = 0;
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
  if (warp == 0) {
    if (BUSY) {
      while (!stop) {
        if (elect_one()) {
#define G(S, R)                                                                                              \
  mma(tb + (R) * P, make_desc(sb + (R) * 4096, 2048, 128), make_desc(sb + 116224, P * 16, 128), make_idesc(32)); \
  fill<S>(tb + 128, sb + 16384 + (R) * 4 * GS, sb + 117248);                                                  \
  fill<S>(tb + 256, sb + 49664 + (R) * 4 * GS, sb + 135680);                                                  \
  fill<S>(tb + 384, sb + 82944 + (R) * 4 * GS, sb + 154112);
          G(0, 0) G(1, 1) G(2, 2) G(3, 3)
#undef G
        }
        __syncwarp();
      }
      if (elect_one())
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
      __syncwarp();
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n\t}"
                     : "=r"(ok) : "r"(smem_u32(&bar)));
    }
  } else if (warp == 1) {
    const uint32_t lb = 32u << 16;     // lane quarter 1
    const uint32_t ta = tb + lb + 200; // columns the MMAs also use (layer 1's ring): realistic contention
    uint32_t v[32];
    long long tA = 0, tB = 0, tC = 0, tD = 0;
    uint32_t ph = 0;
    uint8_t *scr = smem + SCR;
    for (int it = 0; it < iters; ++it) {
      long long t0 = clock64();
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                     "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                   : "r"(ta) : "memory");
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                   : "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                     "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                   : "r"(ta + 16) : "memory");
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      long long t1 = clock64();
      uint32_t z = 0;
      asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(ta + 32 * 4), "r"(z) : "memory");
      asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(ta + 32 * 4 + 16), "r"(z) : "memory");
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      long long t2 = clock64();
      uint32_t acc = 0;
      for (int c = 0; c < 32; ++c) acc += v[c];
#pragma unroll
      for (int g = 0; g < 4; ++g)
        *reinterpret_cast<uint4 *>(scr + g * 2080 + lane * 16) = make_uint4(acc, acc + 1, acc + 2, acc + 3);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      long long t3 = clock64();
      if (lane == 0) asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&mb)) : "memory");
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                     : "=r"(ok) : "r"(smem_u32(&mb)), "r"(ph) : "memory");
      ph ^= 1;
      long long t4 = clock64();
      if (it >= 8) { tA += t1 - t0; tB += t2 - t1; tC += t3 - t2; tD += t4 - t3; }
    }
    if (lane == 0 && blockIdx.x == 0) {
      const int n = iters - 8;
      out[0] = tA / n; out[1] = tB / n; out[2] = tC / n; out[3] = tD / n;
    }
    stop = 1;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
}

template <int BUSY>
void run(const char *name) {
  long long *d, h[4];
  cudaMalloc(&d, 4 * sizeof(long long));
  cudaFuncSetAttribute(kern<BUSY>, cudaFuncAttributeMaxDynamicSharedMemorySize, TOTAL);
  kern<BUSY><<<148, 128, TOTAL>>>(2000, d);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("%-26s tcgen05.ld x2+wait %5lld | tcgen05.st x2+wait %5lld | 4 STS+fence.proxy.async %5lld | mbarrier round trip %5lld  %s\n",
         name, h[0], h[1], h[2], h[3], cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<0>("idle tensor pipe");
  run<1>("busy (chunk-1 MMA stream)");
  return 0;
}
