// Diagnostics: cost of the ring-4 accumulator fill patterns of one windowed CNN layer (P = 32,
// N = 96 = rows f-2, f-1, f at slots (f-2) mod 4 ..; a window that wraps the 4-slot ring is issued
// as two MMAs).  Descriptors precomputed in uniform registers, fully unrolled (no issue overhead).
// exp/mma_replay.cu: the chunk's stream costs ~2,100 cycles per row step with the splits vs ~1,130
// without -- far more than 6 extra MMAs x 44 cycles.  Each pattern: 6 (dx, ks) MMA positions per
// fill, fills cycling through the listed ring phases s = (f-2) mod 4.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o exp/mma_split exp/mma_split.cu
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
constexpr uint32_t AOFF = 0, BOFF = 4 * 4 * GS, TOTAL0 = BOFF + 6 * 96 * 32;
// chunk layout: 3 windowed layers, each 4 ring rows (4 x 8,320 B) + 18 KB weights; im2col ring 4 x 4 KB + 1 KB
constexpr uint32_t LSTRIDE = 4 * 4 * GS + 6 * 96 * 32, IMOFF = 3 * LSTRIDE, TOTAL = 190 * 1024;

// one fill at ring phase S: rows at slots S, S+1, S+2 (mod 4); SPLITMODE 0 ring-4 split, 1 always
// N = 32 x 3 (three MMAs), 2 never split (D window at S even past slot 3: TMEM 0..191)
template <int S, int SPLITMODE>
__device__ __forceinline__ void fill(uint32_t acc0, uint32_t a0, uint32_t b0) {
  constexpr int n1 = SPLITMODE == 2 ? 3 : (4 - S < 3 ? 4 - S : 3);
  constexpr int n2 = 3 - n1;
#pragma unroll
  for (int dx = 0; dx < 3; ++dx)
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      const uint64_t ad = make_desc(a0 + 2 * ks * GS + dx * 16, GS, 128);
      const uint32_t bb = b0 + (dx * 2 + ks) * 96 * 32;
      if (SPLITMODE == 1) {
#pragma unroll
        for (int q = 0; q < 3; ++q) mma(acc0 + ((S + q) & 3) * P, ad, make_desc(bb + q * P * 16, 96 * 16, 128), make_idesc(32));
      } else {
        mma(acc0 + S * P, ad, make_desc(bb, 96 * 16, 128), make_idesc(n1 * P));
        if (n2 > 0) mma(acc0, ad, make_desc(bb + n1 * P * 16, 96 * 16, 128), make_idesc(n2 * P));
      }
    }
}

template <int PAT>
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
  if constexpr (PAT == 8 || PAT == 11 || PAT == 12 || PAT == 13) {
    __shared__ __align__(8) uint64_t junk2[4][2];
    if (threadIdx.x == 0)
      for (int w = 0; w < 4; ++w)
        for (int j = 0; j < 2; ++j) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&junk2[w][j])), "r"(1 << 20));
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (elect_one()) {
        if (warp == 3) {
#pragma unroll
          for (int R = 0; R < 4; ++R)
            mma(tb + R * P, make_desc(sb + IMOFF + R * 4096, 2048, 128), make_desc(sb + IMOFF + 4 * 4096, P * 16, 128), make_idesc(32));
        } else {
          const uint32_t L0 = sb + (uint32_t)warp * LSTRIDE, acc = tb + 128u * (uint32_t)(warp + 1);
#define FF(S) \
          if (PAT == 11 || PAT == 13) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); \
          fill<S, 0>(acc, L0 + S * 4 * GS, L0 + 4 * 4 * GS); \
          if (PAT == 11 || PAT == 12) { \
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&junk2[warp][0]))); \
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&junk2[warp][1]))); }
          FF(0) FF(1) FF(2) FF(3)
#undef FF
        }
      }
      __syncwarp();
    }
    __shared__ __align__(8) uint64_t fin[4];
    if (threadIdx.x == 0) for (int w = 0; w < 4; ++w) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&fin[w])));
    __syncthreads();
    if (elect_one())
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&fin[warp])));
    __syncwarp();
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(&fin[warp])));
    __syncthreads();
    if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
  } else
  if (warp == 0) {
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (elect_one()) {
        const uint32_t b0 = sb + BOFF;
#define F(S, M, R) fill<S, M>(tb, sb + AOFF + (R) * 4 * GS, b0)
        if constexpr (PAT == 0) { F(0, 0, 0); F(1, 0, 1); F(2, 0, 2); F(3, 0, 3); }        // ring-4 cycle
        if constexpr (PAT == 1) { F(0, 0, 0); F(1, 0, 1); F(0, 0, 2); F(1, 0, 3); }        // unsplit phases only
        if constexpr (PAT == 2) { F(2, 0, 0); F(3, 0, 1); F(2, 0, 2); F(3, 0, 3); }        // split phases only
        if constexpr (PAT == 3) { F(2, 0, 0); F(2, 0, 1); F(2, 0, 2); F(2, 0, 3); }        // phase 2 (64 | 32)
        if constexpr (PAT == 4) { F(3, 0, 0); F(3, 0, 1); F(3, 0, 2); F(3, 0, 3); }        // phase 3 (32 | 64)
        if constexpr (PAT == 5) { F(0, 1, 0); F(1, 1, 1); F(2, 1, 2); F(3, 1, 3); }        // three N = 32 per position
        if constexpr (PAT == 6) { F(0, 2, 0); F(1, 2, 1); F(2, 2, 2); F(3, 2, 3); }        // never split (D up to 191)
        if constexpr (PAT == 9) {   // chunk 1 with cnn_kernels.cu make_layout(32, 4, 1, 0, 1) offsets
          // rings: im2col 4 x 4,096 at 0; layers 1-3: 4 x 8,320 at 16,384 / 49,664 / 82,944;
          // weights: im2col 1,024 at 116,224; layers 1-3 18,432 at 117,248 / 135,680 / 154,112
#define G(S, R)                                                                                              \
  mma(tb + (R) * P, make_desc(sb + (R) * 4096, 2048, 128), make_desc(sb + 116224, P * 16, 128), make_idesc(32)); \
  fill<S, 0>(tb + 128, sb + 16384 + (R) * 4 * GS, sb + 117248);                                               \
  fill<S, 0>(tb + 256, sb + 49664 + (R) * 4 * GS, sb + 135680);                                               \
  fill<S, 0>(tb + 384, sb + 82944 + (R) * 4 * GS, sb + 154112);
          G(0, 0) G(1, 1) G(2, 2) G(3, 3)
#undef G
        }
        if constexpr (PAT == 10) {  // chunk 2 with make_layout(32, 4, 0, 1, 1): rings 4 x 8,320 at 0 / 33,280 /
          // 66,560 / 99,840; weights 18,432 at 133,120 / 151,552 / 169,984, folded 1,024 at 188,416
#define G(S, R)                                                                                              \
  fill<S, 0>(tb + 0, sb + 0 + (R) * 4 * GS, sb + 133120);                                                     \
  fill<S, 0>(tb + 128, sb + 33280 + (R) * 4 * GS, sb + 151552);                                               \
  fill<S, 0>(tb + 256, sb + 66560 + (R) * 4 * GS, sb + 169984);                                               \
  mma(tb + 384 + ((R) & 1) * 16, make_desc(sb + 99840 + (R) * 4 * GS + 16, GS, 128), make_desc(sb + 188416, 256, 128), make_idesc(16)); \
  mma(tb + 384 + ((R) & 1) * 16, make_desc(sb + 99840 + (R) * 4 * GS + 16 + 2 * GS, GS, 128), make_desc(sb + 188416 + 512, 256, 128), make_idesc(16));
          G(0, 0) G(1, 1) G(2, 2) G(3, 3)
#undef G
        }
        if constexpr (PAT == 7) {   // chunk stream from one warp: per row step im2col + 3 layers
#define G(S, R)                                                                                              \
  mma(tb + (R) * P, make_desc(sb + IMOFF + (R) * 4096, 2048, 128), make_desc(sb + IMOFF + 4 * 4096, P * 16, 128), \
      make_idesc(32));                                                                                       \
  fill<S, 0>(tb + 128, sb + 0 * LSTRIDE + (R) * 4 * GS, sb + 0 * LSTRIDE + 4 * 4 * GS);                       \
  fill<S, 0>(tb + 256, sb + 1 * LSTRIDE + (R) * 4 * GS, sb + 1 * LSTRIDE + 4 * 4 * GS);                       \
  fill<S, 0>(tb + 384, sb + 2 * LSTRIDE + (R) * 4 * GS, sb + 2 * LSTRIDE + 4 * 4 * GS);
          G(0, 0) G(1, 1) G(2, 2) G(3, 3)
#undef G
        }
#undef F
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
    if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
}

template <int PAT>
void run(const char *name) {
  long long *dC;
  cudaMalloc(&dC, 148 * 8);
  cudaFuncSetAttribute(kern<PAT>, cudaFuncAttributeMaxDynamicSharedMemorySize, TOTAL);
  kern<PAT><<<148, 128, TOTAL>>>(20, dC);
  cudaDeviceSynchronize();
  const int iters = 1000;
  kern<PAT><<<148, 128, TOTAL>>>(iters, dC);
  cudaDeviceSynchronize();
  long long h[148]; cudaMemcpy(h, dC, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
  printf("%-46s %7.1f cycles per fill (6 MMA positions)  %s\n", name, avg / (iters * 4.0), cudaGetErrorString(cudaGetLastError()));
  cudaFree(dC);
}

int main() {
  run<0>("ring-4 cycle (phases 0,1,2,3)");
  run<1>("unsplit phases only (0,1,0,1)");
  run<2>("split phases only (2,3,2,3)");
  run<3>("phase 2 only (N=64 @2 | N=32 @0)");
  run<4>("phase 3 only (N=32 @3 | N=64 @0)");
  run<5>("three N=32 MMAs per position");
  run<6>("never split (D window from slot S, up to col 191)");
  run<7>("chunk stream, 1 warp (per ROW STEP = 4 fills... /4)");
  run<8>("chunk stream, 4 warps (1 per layer)");
  run<9>("chunk 1 stream, kernel smem layout, 1 warp");
  run<10>("chunk 2 stream, kernel smem layout, 1 warp");
  run<11>("4 warps + tcgen05.fence::after_thread_sync + 2 commits per fill");
  run<12>("4 warps + 2 commits per fill");
  run<13>("4 warps + tcgen05.fence::after_thread_sync per fill");
  return 0;
}
