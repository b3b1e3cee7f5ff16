// Diagnostics: replay the CNN kernel's tcgen05.mma issue pattern (P=32, 4-layer chunk,
// first layer im2col) with no pipeline waits, to separate tensor-pipe throughput from
// dependency stalls.  One CTA per SM; MODE 0: 4 issuer warps (one per layer, as the
// kernel), MODE 1: one warp issues all layers in step order; SPLIT 0: never split at the
// accumulator-ring wrap (one N=96 MMA per (dx,ks)).  Prints cycles per schedule step.
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
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

constexpr int P = 32, NL = 4, KS = 2;
constexpr uint32_t GS = 130 * 16;
constexpr uint32_t SLOT = 4 * GS;   // 8320 B

// NOISE (extra warps 4..15 run alongside the issuers until they finish):
//  0 none, 1 TMEM ld 32 cols + st 32 cols (epilogue-like), 2 st.shared.v4 stream,
//  3 mbarrier try_wait polling, 4 = 1 + 2
template <int MODE, int SPLIT, int NOISE = 0, int RND = 0>
__global__ void __launch_bounds__(512, 1) replay(int S, long long *out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bars[8];
  const int warp = threadIdx.x >> 5;
  // layout: rings (layer 0: 4 x 4 KB; layers 1-3: 4 x SLOT), weights
  const uint32_t ring0 = 0, ringl = 16384, wl0 = ringl + 3 * 4 * SLOT, wl = wl0 + 1024;
  for (int i = threadIdx.x; i < (int)(wl + 3 * 9 * P * P * 2) / 4; i += blockDim.x)
    reinterpret_cast<uint32_t *>(smem)[i] = RND ? ((i * 2654435761u) ^ (i >> 3)) & 0xbfffbfffu : 0x3c003c00u;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[i])));
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
  const uint32_t tbase = tslot, sb = smem_u32(smem);
  __shared__ volatile int done_flag;
  if (threadIdx.x == 0) done_flag = 0;
  __syncthreads();
  long long t0 = clock64();
  if (warp >= 4) {
    if (NOISE == 0) return;
    const uint32_t lb = (uint32_t)((warp & 3) * 32) << 16;
    const int lane = threadIdx.x & 31;
    uint8_t *scratch = smem + ringl + (warp - 4) * 512;   // overwrite ring data (values irrelevant)
    int it = 0;
    while (!done_flag) {
      if (NOISE == 1 || NOISE == 4) {
        uint32_t r[16];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                       "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                     : "r"(tbase + lb + (it & 15) * 32) : "memory");
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(
                         tbase + lb + 480), "r"(r[0] & 0) : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      }
      if (NOISE == 2 || NOISE == 4) {
        *reinterpret_cast<uint4 *>(scratch + lane * 16) = make_uint4(it, it, it, it);
        __syncwarp();
      }
      if (NOISE == 5 || NOISE == 6) {   // sleep-wait on the issuers' commit barriers, phase by phase
        uint32_t ok = 0;
        const uint32_t b = smem_u32(&bars[NOISE == 5 ? (warp & 3) : 4 + (warp & 3)]);
        while (!ok && !done_flag)
          asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\tselp.u32 %0,1,0,p;\n\t}"
                       : "=r"(ok) : "r"(b), "r"((uint32_t)(it & 1)), "r"(500000u) : "memory");
      }
      if (NOISE == 3) {
        uint32_t ok;
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 1;\n\tselp.u32 %0,1,0,p;\n\t}"
                     : "=r"(ok) : "r"(smem_u32(&bars[7])));
      }
      ++it;
    }
    return;
  }
  if (MODE == 2) {
    for (int s = 0; s < S; ++s) {
      const int l = warp;
      const int f = s - 3 * l;
      if (f < 0) continue;
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t acc0 = tbase + l * 4 * P;
      uint32_t pred;
      asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(pred));
      if (pred) {
        if (l == 0) {
          mma(acc0 + (f & 3) * P, make_desc(sb + ring0 + (f & 3) * 4096, 2048, 128), make_desc(sb + wl0, P * 16, 128),
              make_idesc(P), 0);
        } else {
          const uint32_t slot = sb + ringl + ((l - 1) * 4 + (f & 3)) * SLOT;
          const uint32_t wb = sb + wl + (l - 1) * 9 * P * P * 2;
          const int Ilo = f - 2;
          const uint64_t ad0 = make_desc(slot, GS, 128), bd0 = make_desc(wb, 3u * P * 16u, 128);
          if (SPLIT >= 2) {
            // SPLIT 2: wrap steps as one N=128 MMA per (dx,ks) (zero block for the draining slot);
            // SPLIT 3: same + one N=32 accumulate=0 MMA zeroing the fresh row's slot per step
            const bool wrap = (Ilo & 3) >= 2;
            if (SPLIT == 3) mma(acc0 + (f & 3) * P, ad0, bd0, make_idesc(P), 0);
            const uint32_t d1 = wrap ? acc0 : acc0 + (Ilo & 3) * P, id1 = make_idesc(wrap ? 4 * P : 3 * P);
#pragma unroll
            for (int dx = 0; dx < 3; ++dx)
#pragma unroll
              for (int ks = 0; ks < KS; ++ks) {
                const uint64_t ad = ad0 + (uint64_t)((2 * ks * GS + dx * 16) >> 4);
                const uint64_t bd = bd0 + (uint64_t)((dx * KS + ks) * 3u * P * 2u);
                mma(d1, ad, bd, id1, 1);
              }
          } else {
          const int n1 = SPLIT ? (4 - (Ilo & 3) < 3 ? 4 - (Ilo & 3) : 3) : 3;
          const int n2 = 3 - n1;
          const uint32_t d1 = acc0 + (SPLIT ? (Ilo & 3) * P : 0), id1 = make_idesc(n1 * P), id2 = make_idesc((n2 ? n2 : 1) * P);
#pragma unroll
          for (int dx = 0; dx < 3; ++dx)
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) {
              const uint64_t ad = ad0 + (uint64_t)((2 * ks * GS + dx * 16) >> 4);
              const uint64_t bd = bd0 + (uint64_t)((dx * KS + ks) * 3u * P * 2u);
              mma(d1, ad, bd, id1, 1);
              if (n2 > 0) mma(acc0, ad, bd + (uint64_t)(n1 * P), id2, 1);
            }
          }
        }
      }
      __syncwarp();
      asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(pred));
      if (pred) { commit(smem_u32(&bars[l])); commit(smem_u32(&bars[l])); }
      __syncwarp();
    }
    if ((threadIdx.x & 31) == 0) {
      commit(smem_u32(&bars[4 + warp]));
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n\t}"
                     : "=r"(ok) : "r"(smem_u32(&bars[4 + warp])));
    }
    __syncwarp();
  } else if ((threadIdx.x & 31) == 0 && (MODE == 0 || warp == 0)) {
    for (int s = 0; s < S; ++s) {
      for (int l = 0; l < NL; ++l) {
        if (MODE == 0 && l != warp) continue;
        const int f = s - 3 * l;
        if (f < 0) continue;
        const uint32_t acc0 = tbase + l * 4 * P;
        if (l == 0) {
          mma(acc0 + (f & 3) * P, make_desc(sb + ring0 + (f & 3) * 4096, 2048, 128), make_desc(sb + wl0, P * 16, 128),
              make_idesc(P), 0);
        } else {
          const uint32_t slot = sb + ringl + ((l - 1) * 4 + (f & 3)) * SLOT;
          const uint32_t wb = sb + wl + (l - 1) * 9 * P * P * 2;
          const int Ilo = f - 2;   // steady state: 3 rows
          const int n1 = SPLIT ? (4 - (Ilo & 3) < 3 ? 4 - (Ilo & 3) : 3) : 3;
          const int n2 = 3 - n1;
          const uint64_t ad0 = make_desc(slot, GS, 128), bd0 = make_desc(wb, 3u * P * 16u, 128);
          const uint32_t d1 = acc0 + (SPLIT ? (Ilo & 3) * P : 0), id1 = make_idesc(n1 * P), id2 = make_idesc((n2 ? n2 : 1) * P);
          for (int dx = 0; dx < 3; ++dx)
            for (int ks = 0; ks < KS; ++ks) {
              const uint64_t ad = ad0 + (uint64_t)((2 * ks * GS + dx * 16) >> 4);
              const uint64_t bd = bd0 + (uint64_t)((dx * KS + ks) * 3u * P * 2u);
              mma(d1, ad, bd, id1, 1);
              if (n2 > 0) mma(acc0, ad, bd + (uint64_t)(n1 * P), id2, 1);
            }
        }
        commit(smem_u32(&bars[l]));
      }
    }
    commit(smem_u32(&bars[4 + warp]));
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(&bars[4 + warp])));
  }
  __syncwarp();
  if (MODE != 1) asm volatile("bar.sync 1, 128;");
  if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
  if (threadIdx.x == 0) done_flag = 1;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

template <int MODE, int SPLIT, int NOISE = 0, int RND = 0>
void run(const char *name) {
  long long *d, h[148];
  cudaMalloc(&d, 148 * sizeof(long long));
  auto k = replay<MODE, SPLIT, NOISE, RND>;
  const int smem = 16384 + 12 * SLOT + 1024 + 3 * 9 * P * P * 2 + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int S = 2000;
  k<<<148, 512, smem>>>(20, d);
  k<<<148, 512, smem>>>(S, d);
  cudaDeviceSynchronize();
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  printf("%-28s %8.1f cycles/step  err=%s\n", name, avg / S, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<0, 1>("4 issuers, split at wrap");
  run<0, 0>("4 issuers, no split");
  run<1, 1>("1 issuer, split at wrap");
  run<1, 0>("1 issuer, no split");
  run<2, 1>("4 warps elect+sync, split");
  run<2, 2>("... wrap as N=128");
  run<2, 3>("... wrap as N=128 + zero MMA");
  run<2, 1, 0, 1>("... random bf16 data");
  run<2, 1, 5>("... + sleeping waiters on commits");
  run<2, 1, 6>("... + sleeping waiters elsewhere");
  run<2, 1, 4, 1>("... random + TMEM + st.sh");
  run<2, 0>("4 warps elect+sync, no split");
  run<0, 1, 1>("4 iss, split + TMEM ld/st");
  run<0, 1, 2>("4 iss, split + st.shared");
  run<0, 1, 3>("4 iss, split + mbar poll");
  run<0, 1, 4>("4 iss, split + TMEM + st.sh");
  return 0;
}
