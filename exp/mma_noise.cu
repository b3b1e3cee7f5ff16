// Diagnostics: does any of the CNN kernel's non-MMA activity slow its MMA stream?  Warp 0 issues
// the c5 chunk-1 MMA stream (exp/mma_split.cu PAT 9: im2col + 3 windowed layers, the kernel's
// shared-memory layout, descriptors precomputed; 1,340 cycles per row step alone) while warps 1-7
// run one kind of full-rate "noise" modelled on the kernel's producers / epilogues:
//   0 none; 1 STS.128 + fence.proxy.async; 2 fence.proxy.async alone; 3 mbarrier arrive + try_wait
//   ping-pong; 4 tcgen05.ld x16 + wait + tcgen05.st x16 + wait + tcgen05.fence::before_thread_sync;
//   5 cp.async.bulk global -> shared (4 KB per copy, mbarrier complete_tx); 6 all of 1, 3, 4, 5
// (one kind per warp, round-robin).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o exp/mma_noise exp/mma_noise.cu
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
constexpr uint32_t TOTAL = 200 * 1024, NOISE = 176 * 1024;   // noise scratch: 176 KB .. 200 KB

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

template <int NZ>
__global__ void __launch_bounds__(256, 1) kern(int iters, const float4 *gsrc, long long *cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar, nb[8];
  __shared__ volatile int stop;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (uint32_t e = threadIdx.x; e < TOTAL / 16; e += blockDim.x)
    reinterpret_cast<uint4 *>(smem)[e] = make_uint4(0x3c003c00u, 0, 0x3c00u, 0);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&nb[i])));
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
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
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
    if (lane == 0) { cyc[blockIdx.x] = clock64() - t0; stop = 1; }
  } else if (NZ != 0) {
    const int kind = NZ == 6 ? ((warp & 3) == 0 ? 1 : (warp & 3) == 1 ? 3 : (warp & 3) == 2 ? 4 : 5) : NZ;
    uint8_t *scr = smem + NOISE + (warp - 1) * 3072;   // 3 KB per noise warp
    const uint32_t mb = smem_u32(&nb[warp]);
    uint32_t ph = 0;
    uint32_t v[16];
    for (int c = 0; c < 16; ++c) v[c] = c + lane;
    const uint32_t lb = (uint32_t)((warp & 3) * 32) << 16;   // the warp's TMEM lane quarter
    while (!stop) {
      if (kind == 1) {
#pragma unroll
        for (int r = 0; r < 4; ++r)
          *reinterpret_cast<uint4 *>(scr + r * 512 + lane * 16) = make_uint4(v[0], v[1], v[2], v[3]);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
      } else if (kind == 2) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      } else if (kind == 3) {
        if (lane == 0) asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(mb) : "memory");
        uint32_t ok = 0;
        while (!ok)
          asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                       : "=r"(ok) : "r"(mb), "r"(ph) : "memory");
        ph ^= 1;
      } else if (kind == 4) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                       "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                     : "r"(tb + lb + 64) : "memory");
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                     ::"r"(tb + lb + 96), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]),
                     "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
                     : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
      } else if (kind == 5) {
        if (lane == 0) {
          asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(3072u) : "memory");
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                           smem_u32(scr)), "l"(gsrc + (blockIdx.x * 8 + warp) * 192), "r"(3072u), "r"(mb)
                       : "memory");
        }
        __syncwarp();
        uint32_t ok = 0;
        while (!ok)
          asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                       : "=r"(ok) : "r"(mb), "r"(ph) : "memory");
        ph ^= 1;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
}

template <int NZ>
void run(const char *name, const float4 *gsrc) {
  long long *dC;
  cudaMalloc(&dC, 148 * 8);
  cudaFuncSetAttribute(kern<NZ>, cudaFuncAttributeMaxDynamicSharedMemorySize, TOTAL);
  kern<NZ><<<148, 256, TOTAL>>>(20, gsrc, dC);
  cudaDeviceSynchronize();
  const int iters = 1000;
  kern<NZ><<<148, 256, TOTAL>>>(iters, gsrc, dC);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148]; cudaMemcpy(h, dC, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
  printf("%-58s %7.1f cycles per row step  %s\n", name, avg / (iters * 4.0), cudaGetErrorString(e));
  cudaFree(dC);
}

int main() {
  float4 *g;
  cudaMalloc(&g, 148 * 8 * 192 * sizeof(float4));
  cudaMemset(g, 0, 148 * 8 * 192 * sizeof(float4));
  run<0>("chunk-1 MMA stream alone", g);
  run<1>("+ 7 warps STS.128 x4 + fence.proxy.async", g);
  run<2>("+ 7 warps fence.proxy.async", g);
  run<3>("+ 7 warps mbarrier arrive / try_wait", g);
  run<4>("+ 7 warps tcgen05.ld/st x16 + waits + tcgen05.fence", g);
  run<5>("+ 7 warps cp.async.bulk 3 KB global->smem", g);
  run<6>("+ 7 warps mixed (STS+fence, mbarrier, tcgen05 ld/st, bulk)", g);
  return 0;
}
