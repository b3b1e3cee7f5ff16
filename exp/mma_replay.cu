// Diagnostics: replay the c5 CNN chunk's exact tcgen05.mma stream (operand addresses, shapes, split
// pairs, D columns) from ONE thread with no pipeline around it, on all 148 SMs, to separate the
// tensor core's own rate on these operands from pipeline / power effects.  The c5 chunk kernel
// (P = 32, layers 1-4 of a K = 8 DnCNN, ring-4) spends ~58 cycles per MMA in the kernel (ncu) vs
// 44-56 in exp/mma_ts.cu.  Layout = make_layout(32, 4, first = 1, last = 0, 1) of cnn_kernels.cu:
// ring 0 = im2col rows (4 x 4 KB), rings 1-3 = activation rows (4 x 8,320 B), then the weights.
//   mode 0: steady state, short (~1 ms); mode 1: the same for ~1 s (power / clock under load);
//   mode 2: windowed layers only, no splits (every fill N = 96); mode 3: B of all layers at layer 1's.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o exp/mma_replay exp/mma_replay.cu
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
__device__ __forceinline__ void mma(uint32_t d, uint64_t ad, uint64_t bd, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
               ::"r"(d), "l"(ad), "l"(bd), "r"(id), "r"(acc));
}
constexpr int P = 32, GS = 130 * 16, SLOT_ACT = 4 * GS, SLOT_IM = 2 * 128 * 16;
constexpr uint32_t align128(uint32_t v) { return (v + 127) / 128 * 128; }
constexpr uint32_t RING0 = 0, RING1 = align128(RING0 + 4 * SLOT_IM), RING2 = align128(RING1 + 4 * SLOT_ACT),
                   RING3 = align128(RING2 + 4 * SLOT_ACT), W0 = align128(RING3 + 4 * SLOT_ACT),
                   W1 = align128(W0 + 16 * 32 * 2), W2 = align128(W1 + 9 * 32 * 32 * 2), W3 = align128(W2 + 9 * 32 * 32 * 2),
                   TOTAL = align128(W3 + 9 * 32 * 32 * 2);

template <int mode>
__global__ void __launch_bounds__(128, 1) kern(int rows, long long *cyc) {
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
  if (mode == 4) {   // warp w issues layer w only (run-time descriptors, as the kernel's MMA warps)
    const uint32_t ring[4] = {RING0, RING1, RING2, RING3};
    const uint32_t wo[4] = {W0, W1, W2, W3};
    __shared__ __align__(8) uint64_t fin[4];
    if (threadIdx.x == 0) for (int w = 0; w < 4; ++w) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&fin[w])));
    __syncthreads();
    const long long t0 = clock64();
    const int l = warp;
    for (int r = 0; r < rows; ++r) {
      if (l == 0) {
        const uint64_t ad = make_desc(sb + RING0 + (r & 3) * SLOT_IM, 2048, 128);
        const uint64_t bd = make_desc(sb + W0, P * 16, 128);
        if (elect_one()) mma(tb + (r & 3) * P, ad, bd, make_idesc(P), 0);
        __syncwarp();
      } else {
        const uint32_t acc0 = tb + l * 4 * P;
        const uint32_t slot = sb + ring[l] + (r & 3) * SLOT_ACT;
        const uint32_t wb = sb + wo[l];
        const uint32_t Ilo = (uint32_t)(r + 2);
        const int n1 = (int)min(3u, 4u - (Ilo & 3));
        const int n2 = 3 - n1;
        const uint64_t ad0 = make_desc(slot, GS, 128), bd0 = make_desc(wb, 3 * P * 16, 128);
        const uint32_t d1 = acc0 + (Ilo & 3) * P, d2 = acc0;
        const uint32_t id1 = make_idesc(n1 * P), id2 = make_idesc(n2 > 0 ? n2 * P : P);
        if (elect_one()) {
#pragma unroll
          for (int dx = 0; dx < 3; ++dx)
#pragma unroll
            for (int ks = 0; ks < 2; ++ks) {
              const uint64_t ad = ad0 + (uint64_t)((2 * ks * GS + dx * 16) >> 4);
              const uint64_t bd = bd0 + (uint64_t)((dx * 2 + ks) * 3 * P * 2);
              mma(d1, ad, bd, id1, 1);
              if (n2 > 0) mma(d2, ad, bd + (uint64_t)(n1 * P), id2, 1);
            }
        }
        __syncwarp();
      }
    }
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
  if (warp == 0) {   // the whole warp walks the stream (warp-uniform descriptors), one elected lane issues
    const uint32_t ring[4] = {RING0, RING1, RING2, RING3};
    const uint32_t wo[4] = {W0, W1, W2, W3};
    const long long t0 = clock64();
    for (int r = 0; r < rows; ++r) {
      // layer 0: im2col, one N = 32 K = 16 MMA into slot r & 3
      if (mode != 2) {
        const uint64_t ad = make_desc(sb + RING0 + (r & 3) * SLOT_IM, 2048, 128);
        const uint64_t bd = make_desc(sb + W0, P * 16, 128);
        if (elect_one()) mma(tb + (r & 3) * P, ad, bd, make_idesc(P), 0);
        __syncwarp();
      }
      // layers 1-3: windowed, fill r (rows r-2 .. r at slots (r-2)&3 ..), ring-4 splits
#pragma unroll 1
      for (int l = 1; l < 4; ++l) {
        const uint32_t acc0 = tb + l * 4 * P;
        const uint32_t slot = sb + ring[l] + (r & 3) * SLOT_ACT;
        const uint32_t wb = sb + (mode == 3 ? W1 : wo[l]);
        const uint32_t Ilo = (uint32_t)(r + 2);   // (r - 2) & 3 without the sign
        const int n1 = mode == 2 ? 3 : (int)min(3u, 4u - (Ilo & 3));
        const int n2 = 3 - n1;
        const uint64_t ad0 = make_desc(slot, GS, 128), bd0 = make_desc(wb, 3 * P * 16, 128);
        const uint32_t d1 = acc0 + (mode == 2 ? 0u : (Ilo & 3) * P), d2 = acc0;
        const uint32_t id1 = make_idesc(n1 * P), id2 = make_idesc(n2 > 0 ? n2 * P : P);
        if (elect_one()) {
#pragma unroll
        for (int dx = 0; dx < 3; ++dx)
#pragma unroll
          for (int ks = 0; ks < 2; ++ks) {
            const uint64_t ad = ad0 + (uint64_t)((2 * ks * GS + dx * 16) >> 4);
            const uint64_t bd = bd0 + (uint64_t)((dx * 2 + ks) * 3 * P * 2);
            mma(d1, ad, bd, id1, 1);
            if (n2 > 0) mma(d2, ad, bd + (uint64_t)(n1 * P), id2, 1);
          }
        }
        __syncwarp();
      }
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

template <int mode>
void run(const char *name, int rows) {
  long long *dC;
  cudaMalloc(&dC, 148 * 8);
  cudaFuncSetAttribute(kern<mode>, cudaFuncAttributeMaxDynamicSharedMemorySize, TOTAL);
  kern<mode><<<148, 128, TOTAL>>>(64, dC);
  cudaDeviceSynchronize();
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  kern<mode><<<148, 128, TOTAL>>>(rows, dC);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  long long h[148]; cudaMemcpy(h, dC, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
  const double macs = (double)rows * 148 * (mode == 2 ? 3 * 6 * 128.0 * 96 * 16 : (128.0 * 32 * 16 + 3 * 6 * 128.0 * 96 * 16));
  printf("%-44s rows %7d: %7.1f cycles/row step (%.3f ms, %.0f MHz effective), %6.1f TFLOP/s  %s\n", name, rows, avg / rows, ms,
         avg / (ms * 1e3), 2 * macs / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  printf("smem %u B\n", TOTAL);
  run<0>("kernel chunk-1 MMA stream (ring-4 splits)", 2000);
  run<2>("windowed layers, no splits (N = 96 only)", 2000);
  run<3>("as mode 0, one weight block for all layers", 2000);
  run<4>("chunk-1 stream, 4 warps (one layer each), run-time descriptors", 2000);
  return 0;
}
