// Microbenchmark + correctness probe (diagnostics): tcgen05.mma kind::f16, M = 128, K = 16, with
// the A operand in TENSOR MEMORY ("TS": [a_tmem]) instead of shared memory ("SS").  Question for
// the CNN kernel (profiles/r02_cnn_schemes.md: SS N = 96 MMAs stream at 56 cycles = 7 KB of
// shared-memory operand fetch at 128 B/clk): does an A-in-TMEM MMA run at the tensor floor
// (128 N / 256 = 48 cycles for N = 96), and do the ring-wrap split pairs (N = 64 + 32) cost no more
// than one N = 96?  Also: cost of concurrent tcgen05.st traffic (the epilogue writing A copies).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o exp/mma_ts exp/mma_ts.cu
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
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
constexpr int NB = 96;

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t bd, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
               ::"r"(d), "r"(a), "l"(bd), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t ad, uint64_t bd, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
               ::"r"(d), "l"(ad), "l"(bd), "r"(id), "r"(acc));
}
__device__ __forceinline__ bool elect_one_() {
  uint32_t pred;
  asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void commit_wait(uint64_t *bar, uint32_t ph) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)));
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                 : "=r"(ok) : "r"(smem_u32(bar)), "r"(ph));
}

// TMEM map (512 columns): D at 0..95 (acc ring 0..127), A copies at 256 + 8 j (j = 0..11).
// mode 0: check  (one TS MMA, A copy 0, K step ks) -> out
// mode 1: time   TS N=96, 6 MMAs per group over 6 A addresses x 2 B K-steps
// mode 2: time   SS N=96 (A in smem, canonical no-swizzle layout)
// mode 3: time   TS split pairs N=64 + N=32 (ring wrap)
// mode 4: time   TS N=96 with warps 1-3 doing tcgen05.st of 48 columns per 6 MMAs (epilogue A writes)
// mode 5: time   TS N=32 stream
// mode 6: time   TS N=96 with warps 1-3 doing tcgen05.ld 32 cols + st 32 cols per 6 MMAs (epilogue drain)
template <int mode, int dp>
__global__ void __launch_bounds__(128, 1) kern(const uint16_t *gA, const uint16_t *gB, int ks, int iters,
                                              float *out, long long *cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  __shared__ volatile int stop;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t *A = smem, *B = smem + 16384;
  // A: 128 rows x 32 channels (bf16) into smem ([group of 8][128 rows][16 B]) for SS
  for (int e = threadIdx.x; e < 128 * 4; e += blockDim.x) {
    const int r = e >> 2, c = e & 3;
    *reinterpret_cast<uint4 *>(A + c * 2048 + r * 16) = *reinterpret_cast<const uint4 *>(gA + r * 32 + c * 8);
  }
  for (int e = threadIdx.x; e < 2 * 2 * NB; e += blockDim.x)
    *reinterpret_cast<uint4 *>(B + e * 16) = *reinterpret_cast<const uint4 *>(gB + e * 8);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
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
  const uint32_t tb = tslot;
  // A copies into TMEM: row m = lane (warp quarter), 16 channels of K step k in 8 columns,
  // channel pair (2c, 2c+1) in column c (low half = even channel); 12 copies (6 addresses x 2 k)
  {
    const int m = warp * 32 + lane;
    const uint32_t lb = (uint32_t)(warp * 32) << 16;
    for (int j = 0; j < 12; ++j) {
      const int k = j & 1;
      uint32_t v[8];
      for (int c = 0; c < 8; ++c)
        v[c] = (uint32_t)gA[m * 32 + k * 16 + 2 * c] | ((uint32_t)gA[m * 32 + k * 16 + 2 * c + 1] << 16);
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(tb + lb + 256 + 8 * j),
                   "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]) : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t b0 = smem_u32(B), a0 = smem_u32(A);
  uint64_t bd[2];
  for (int k = 0; k < 2; ++k) bd[k] = make_desc(b0 + k * (2 * NB * 16), NB * 16, 128);
  if constexpr (mode >= 12) {
    __shared__ __align__(8) uint64_t junk[4], fin[4];
    const int nw = mode == 13 ? 1 : mode == 15 ? 2 : 4;
    if (threadIdx.x == 0)
      for (int w = 0; w < 4; ++w) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&junk[w])), "r"(1 << 20));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&fin[w])));
      }
    asm volatile("fence.mbarrier_init.release.cluster;");
    __syncthreads();
    if (warp < nw) {
      const uint32_t i96 = make_idesc(96);
      uint64_t ad[2];
      for (int k = 0; k < 2; ++k) ad[k] = make_desc(a0 + k * 2 * 2048, 2048, 128);
      const long long t0 = clock64();
      for (int i = 0; i < iters / nw; i += 24) {
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          if (elect_one_()) {
#pragma unroll
            for (int j = 0; j < 6; ++j) {
              const uint32_t dd = tb + (uint32_t)warp * 112u + 16u * (g & 1);
              if constexpr (mode == 14) mma_ts(dd, tb + 448 + 8 * (j & 1), bd[j & 1], i96, 1);
              else mma_ss(dd, ad[j & 1], bd[j & 1], i96, 1);
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&junk[warp])));
          }
          __syncwarp();
        }
      }
      if (elect_one_()) commit_wait(&fin[warp], 0);
      __syncwarp();
      if (lane == 0 && warp == 0) cyc[blockIdx.x] = clock64() - t0;
    }
  } else
  if (warp == 0) {
    if (threadIdx.x == 0) {
      if (mode == 0) {
        mma_ts(tb, tb + 256 + 8 * ks, bd[ks], make_idesc(NB), 0);
        commit_wait(&bar, 0);
      } else {
        const uint32_t i96 = make_idesc(96), i64 = make_idesc(64), i32 = make_idesc(32);
        uint64_t ad[2];
        for (int k = 0; k < 2; ++k) ad[k] = make_desc(a0 + k * 2 * 2048, 2048, 128);
        // D pattern dp (24 MMAs per iteration = 4 groups of 6): 0 all at D = 0; 1 per-MMA rotation
        // 0/32/64/96 (overlapping); 2 per-group rotation 0/32/64/96 (the CNN ring: 6 MMAs per input
        // row on one D, next row's D 32 columns on); 3 per-group 0/128 (disjoint); 4 per-MMA 0/128
        const long long t0 = clock64();
        for (int i = 0; i < iters; i += 24) {
#pragma unroll
          for (int g = 0; g < 4; ++g)
#pragma unroll
          for (int j = 0; j < 6; ++j) {
            const uint32_t at = tb + 256 + 8 * (2 * (j >> 1) + (j & 1));
            const int q = 6 * g + j;
            const uint32_t off = dp == 0 ? 0u : dp == 1 ? 32u * (q % 4) : dp == 2 ? 32u * g : dp == 3 ? 128u * (g & 1) : 128u * (q & 1);
            const uint32_t dd = tb + off;
            if constexpr (mode == 1 || mode == 4 || mode == 6) mma_ts(dd, at, bd[j & 1], i96, 1);
            else if constexpr (mode == 2) mma_ss(dd, ad[j & 1], bd[j & 1], i96, 1);
            else if constexpr (mode == 3) { mma_ts(tb + off + 64, at, bd[j & 1], i64, 1); mma_ts(tb + off, at, bd[j & 1] + 64 * 2, i32, 1); }
            else if constexpr (mode == 5) mma_ts(dd, at, bd[j & 1], i32, 1);
            else if constexpr (mode == 7) { mma_ss(tb + off + 64, ad[j & 1], bd[j & 1], i64, 1); mma_ss(tb + off, ad[j & 1], bd[j & 1] + 64 * 2, i32, 1); }
            else if constexpr (mode == 8 || mode == 10) mma_ss(dd, ad[j & 1], bd[j & 1], i96, 1);
            else if constexpr (mode == 9 || mode == 11) mma_ts(dd, at, bd[j & 1], i96, 1);
          }
        }
        commit_wait(&bar, 0);
        cyc[blockIdx.x] = clock64() - t0;
        stop = 1;
      }
    }
    __syncwarp();
  } else if (mode >= 8 && mode <= 11) {
    // shared-memory store noise (STS.128, conflict-free) into a region the MMAs do not read
    uint4 *dst = reinterpret_cast<uint4 *>(smem + 32768 + (warp - 1) * 4096);
    const uint4 v = make_uint4(lane, lane + 1, lane + 2, lane + 3);
    while (!stop) {
#pragma unroll
      for (int r = 0; r < 8; ++r) dst[r * 32 + lane] = v;
      if (mode >= 10) { const long long t = clock64(); while (clock64() - t < 200) { } }
    }
  } else if (mode == 4 || mode == 6) {
    // noise: epilogue-like TMEM traffic on columns 384.. (not used by the MMAs)
    const uint32_t lb = (uint32_t)(warp * 32) << 16;
    uint32_t v[16];
    for (int c = 0; c < 16; ++c) v[c] = c * 3 + lane;
    while (!stop) {
      if (mode == 4) {
        for (int r = 0; r < 3; ++r)
          asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                       ::"r"(tb + lb + 384 + 16 * r), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]),
                       "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
                       "r"(v[15]) : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      } else {
        for (int r = 0; r < 2; ++r) {
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                       : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                         "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                       : "r"(tb + lb + 384 + 16 * r) : "memory");
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                       ::"r"(tb + lb + 448 + 16 * r), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]),
                       "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
                       "r"(v[15]) : "memory");
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
      }
    }
  }
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
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
}

static uint16_t f2bf(float f) { uint32_t u; memcpy(&u, &f, 4); return (uint16_t)((u + 0x7fffu + ((u >> 16) & 1u)) >> 16); }
static float bf2f(uint16_t h) { uint32_t u = (uint32_t)h << 16; float f; memcpy(&f, &u, 4); return f; }

int main() {
  static uint16_t hA[128 * 32], hB[2 * 2 * NB * 8];
  for (int i = 0; i < 128 * 32; ++i) hA[i] = f2bf((float)((i * 37 % 17) - 8) / 8.0f);
  for (int i = 0; i < 2 * 2 * NB * 8; ++i) hB[i] = f2bf((float)((i * 11 % 13) - 6) / 4.0f);
  uint16_t *dA, *dB; float *dO; long long *dC;
  cudaMalloc(&dA, sizeof(hA)); cudaMalloc(&dB, sizeof(hB)); cudaMalloc(&dO, 128 * NB * 4); cudaMalloc(&dC, 148 * 8);
  cudaMemcpy(dA, hA, sizeof(hA), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof(hB), cudaMemcpyHostToDevice);
  
  cudaFuncSetAttribute(kern<0, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  static float out[128 * NB];
  for (int ks = 0; ks < 2; ++ks) {
    kern<0, 0><<<1, 128, 64 * 1024>>>(dA, dB, ks, 0, dO, dC);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(out, dO, sizeof(out), cudaMemcpyDeviceToHost);
    double maxerr = 0, maxref = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < NB; ++n) {
        double ref = 0;
        for (int k = 0; k < 16; ++k) {
          const float a = bf2f(hA[m * 32 + ks * 16 + k]);
          const float b = bf2f(hB[((ks * 2 + k / 8) * NB + n) * 8 + (k % 8)]);
          ref += (double)a * b;
        }
        maxerr = fmax(maxerr, fabs(ref - out[m * NB + n]));
        maxref = fmax(maxref, fabs(ref));
      }
    printf("check TS ks=%d: max |err| = %.3g (max |ref| %.3g)  %s\n", ks, maxerr, maxref, cudaGetErrorString(e));
  }
  const char *names[] = {"", "TS N=96", "SS N=96", "TS split N=64+N=32 (per pair)", "TS N=96 + tcgen05.st noise (3 warps)",
                         "TS N=32", "TS N=96 + tcgen05.ld/st noise (3 warps)", "SS split N=64+N=32 (per pair)", "SS N=96 + STS noise full", "TS N=96 + STS noise full", "SS N=96 + STS noise 8/200cyc", "TS N=96 + STS noise 8/200cyc", "SS N=96 4 warps + commit/6", "SS N=96 1 warp + commit/6", "TS N=96 4 warps + commit/6", "SS N=96 2 warps + commit/6"};
  const char *dpn[] = {"D fixed", "D per-MMA +32 (overlap)", "D per-6 +32 (CNN ring)", "D per-6 0/128", "D per-MMA 0/128"};
  for (int mode = 1; mode <= 15; ++mode)
    for (int dp = 0; dp < 5; ++dp) {
      if (mode != 1 && mode != 2 && dp != 2) continue;
      const int iters = 24 * 500;
      auto launch = [&](int it) {
#define L_(M, D) if (mode == M && dp == D) { cudaFuncSetAttribute(kern<M, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024); kern<M, D><<<148, 128, 48 * 1024>>>(dA, dB, 0, it, dO, dC); }
#define LM_(M) L_(M, 0) L_(M, 1) L_(M, 2) L_(M, 3) L_(M, 4)
        LM_(1) LM_(2) LM_(3) LM_(4) LM_(5) LM_(6) LM_(7) LM_(8) LM_(9) LM_(10) LM_(11) LM_(12) LM_(13) LM_(14) LM_(15)
      };
      launch(48);
      cudaDeviceSynchronize();
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      launch(iters);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      long long h[148]; cudaMemcpy(h, dC, sizeof(h), cudaMemcpyDeviceToHost);
      double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
      const int nn = mode == 5 ? 32 : 96;
      printf("%-40s %-26s %6.1f cycles/MMA  %7.1f TFLOP/s  %s\n", names[mode], dpn[dp], avg / iters,
             2.0 * 128 * nn * 16 * iters * 148 / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
