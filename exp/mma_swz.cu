// Microbenchmark + correctness probe (diagnostics): tcgen05.mma kind::f16, M = 128, K = 16, N = 96,
// A in shared memory as 64-B rows (32 bf16 channels per pixel) with the 64-B swizzle, B K-major no
// swizzle.  Question: can the A start be shifted by whole rows (one pixel = 64 B, the CNN's dx
// taps) and stay exact and fast?  Checks D against a host reference for row shifts 0..2, both K
// steps and two base-offset conventions, then times N = 96 streams.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o exp/mma_swz exp/mma_swz.cu
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
// layout: 0 none, 4 = SWIZZLE_64B; base: 3-bit base offset
__host__ __device__ inline uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout, uint32_t base) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)(base & 7) << 49;
  d |= (uint64_t)(layout & 7) << 61;
  return d;
}
__host__ __device__ constexpr uint32_t make_idesc(int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
constexpr int ROWS = 130, NB = 96;
// A: ROWS x 32 bf16, row r at 1024-aligned base + r*64, 16-B chunk c stored at chunk c ^ ((r >> 1) & 3)
// B: [2 K-halves][96 rows][8] bf16 (no swizzle), K step ks uses channels 16 ks .. 16 ks + 15

// mode 0: check -- one MMA (shift s, K step ks, base convention bc), D -> out (128 x 96 floats)
// mode 1: time  -- iters MMAs cycling shifts 0,1,2 and both K steps
__global__ void __launch_bounds__(128, 1) kern(const uint16_t *gA, const uint16_t *gB, int mode, int s, int ks, int bc,
                                              int swz, int iters, float *out, long long *cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t *A = smem, *B = smem + 16384;
  // stage A (swizzled or plain rows of 64 B) and B
  for (int e = threadIdx.x; e < ROWS * 4; e += blockDim.x) {
    const int r = e >> 2, c = e & 3;
    if (swz) {
      const int cs = c ^ ((r >> 1) & 3);
      *reinterpret_cast<uint4 *>(A + r * 64 + cs * 16) = *reinterpret_cast<const uint4 *>(gA + r * 32 + c * 8);
    } else {   // the CNN kernel's r01 ring layout: [8-channel group][130 positions][16 B], group stride 2080 B
      *reinterpret_cast<uint4 *>(A + c * 2080 + r * 16) = *reinterpret_cast<const uint4 *>(gA + r * 32 + c * 8);
    }
  }
  for (int e = threadIdx.x; e < 2 * 2 * NB; e += blockDim.x)   // 2 K steps x 2 halves x 96 rows of 16 B
    *reinterpret_cast<uint4 *>(B + e * 16) = *reinterpret_cast<const uint4 *>(gB + e * 8);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = tslot;
  const uint32_t a0 = smem_u32(A), b0 = smem_u32(B);
  auto adesc = [&](int sh, int k) -> uint64_t {
    if (!swz) return make_desc(a0 + sh * 16 + k * 2 * 2080, 2080, 128, 0, 0);   // r01 ring layout
    const uint32_t addr = a0 + sh * 64 + k * 32;
    const uint32_t base = bc == 0 ? 0u : ((addr >> 7) & 7u);
    return make_desc(addr, 16, 512, 4, base);
  };
  const uint32_t id = make_idesc(NB);
  if (threadIdx.x == 0) {
    if (mode == 0) {
      const uint64_t bd = make_desc(b0 + ks * (2 * NB * 16), NB * 16, 128, 0, 0);
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %4, p;\n\t}"
                   ::"r"(tb), "l"(adesc(s, ks)), "l"(bd), "r"(0), "r"(id));
    } else {
      uint64_t ad[3][2], bd[2];
      for (int k = 0; k < 2; ++k) {
        bd[k] = make_desc(b0 + k * (2 * NB * 16), NB * 16, 128, 0, 0);
        for (int sh = 0; sh < 3; ++sh) ad[sh][k] = adesc(sh, k);
      }
      const long long t0 = clock64();
      for (int i = 0; i < iters; i += 6) {
#pragma unroll
        for (int sh = 0; sh < 3; ++sh)
#pragma unroll
          for (int k = 0; k < 2; ++k)
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %4, p;\n\t}"
                         ::"r"(tb), "l"(ad[sh][k]), "l"(bd[k]), "r"(1), "r"(id));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n\t}"
                     : "=r"(ok) : "r"(smem_u32(&bar)));
      cyc[blockIdx.x] = clock64() - t0;
    }
    if (mode == 0) {
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n\t}"
                     : "=r"(ok) : "r"(smem_u32(&bar)));
    }
  }
  __syncwarp();
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (mode == 0 && blockIdx.x == 0) {
    const uint32_t ta = tb + ((uint32_t)(warp * 32) << 16);
    for (int c = 0; c < NB; ++c) {
      uint32_t r;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(ta + c) : "memory");
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      out[(warp * 32 + lane) * NB + c] = __uint_as_float(r);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tb));
}

static uint16_t f2bf(float f) { uint32_t u; memcpy(&u, &f, 4); return (uint16_t)((u + 0x7fffu + ((u >> 16) & 1u)) >> 16); }
static float bf2f(uint16_t h) { uint32_t u = (uint32_t)h << 16; float f; memcpy(&f, &u, 4); return f; }

int main() {
  uint16_t hA[ROWS * 32], hB[2 * 2 * NB * 8];
  for (int i = 0; i < ROWS * 32; ++i) hA[i] = f2bf((float)((i * 37 % 17) - 8) / 8.0f);
  for (int i = 0; i < 2 * 2 * NB * 8; ++i) hB[i] = f2bf((float)((i * 11 % 13) - 6) / 4.0f);
  uint16_t *dA, *dB; float *dO; long long *dC;
  cudaMalloc(&dA, sizeof(hA)); cudaMalloc(&dB, sizeof(hB)); cudaMalloc(&dO, 128 * NB * 4); cudaMalloc(&dC, 148 * 8);
  cudaMemcpy(dA, hA, sizeof(hA), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof(hB), cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  static float out[128 * NB];
  for (int cfg = 0; cfg < 3; ++cfg)   // 0: no swizzle (r01 layout), 1: swz64 base 0, 2: swz64 base (addr>>7)&7
    for (int s = 0; s < 3; ++s)
      for (int ks = 0; ks < 2; ++ks) {
        const int bc = cfg == 2, swz = cfg > 0;
        kern<<<1, 128, 64 * 1024>>>(dA, dB, 0, s, ks, bc, swz, 0, dO, dC);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(out, dO, sizeof(out), cudaMemcpyDeviceToHost);
        double maxerr = 0;
        for (int m = 0; m < 128; ++m)
          for (int n = 0; n < NB; ++n) {
            double ref = 0;
            for (int k = 0; k < 16; ++k) {
              const int kk = ks * 16 + k;   // channel
              const float a = bf2f(hA[(m + s) * 32 + kk]);
              const float b = bf2f(hB[((ks * 2 + k / 8) * NB + n) * 8 + (k % 8)]);
              ref += (double)a * b;
            }
            maxerr = fmax(maxerr, fabs(ref - out[m * NB + n]));
          }
        printf("check cfg=%d shift=%d ks=%d: max |err| = %.3g  %s\n", cfg, s, ks, maxerr, cudaGetErrorString(e));
      }
  for (int cfg = 0; cfg < 3; ++cfg) {
    const int bc = cfg == 2, swz = cfg > 0;
    const int iters = 6 * 1000;
    kern<<<148, 128, 64 * 1024>>>(dA, dB, 1, 0, 0, bc, swz, 60, dO, dC);
    cudaDeviceSynchronize();
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    kern<<<148, 128, 64 * 1024>>>(dA, dB, 1, 0, 0, bc, swz, iters, dO, dC);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    long long h[148]; cudaMemcpy(h, dC, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
    printf("time cfg=%d: %.1f cycles/MMA (N=96, shifts 0..2 x 2 K steps), %.1f TFLOP/s  %s\n", cfg, avg / iters,
           2.0 * 128 * 96 * 16 * iters * 148 / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
