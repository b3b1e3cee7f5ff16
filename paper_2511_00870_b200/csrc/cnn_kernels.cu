// cnn_kernels.cu -- the DnCNN-style prior G_eps on 5th-generation tensor
// cores (tcgen05 + TMEM), sm_100a.  One launch evaluates a chain of NL consecutive
// 3x3 conv layers (eq:cnn:convolution P:358-363) of the net on a tile region.
//
// Design:
//  * implicit GEMM, M = 128 consecutive pixels of one image row, K = 16 input channels
//    per MMA.  A = one input row (bf16, shared memory) shifted by dx in {-1,0,1} -- the
//    shift is a change of the UMMA descriptor start address;
//  * the three vertical taps are folded into N: B(dx, k) stacks the weights of
//    dy = +1, 0, -1, so one MMA with N = 3 Cb (Cb = P, or 16 for the 1-channel last
//    layer) adds input row r's contribution to output rows r-1, r, r+1 at once.
//    Output rows accumulate in a 4-slot TMEM ring (one Cb-column slot per row): an
//    output row is complete after the MMAs of input row r+1; the epilogue reads it and
//    re-zeroes its slot.  Each input row is consumed by exactly one MMA group;
//  * activations live in shared memory in "channel-group planar" rows
//    [group of 8 ch][130 positions][8 x bf16] -- the canonical K-major, no-swizzle
//    UMMA layout (core matrix = 8 positions x 16 B); a CTA owns a 130-column strip and
//    streams down its rows, every layer of the chain lagging the previous one by 3 rows;
//  * warp roles: 4 producer warps load input rows (x -> bf16 im2col rows for the first
//    layer, or one TMA bulk copy per 8-channel group for activation rows from HBM),
//    up to 4 MMA warps (one per layer) issue tcgen05.mma / tcgen05.commit (warp-uniform
//    operands, one elected lane issues), the remaining warps are the epilogue in up to 4
//    groups of 4 warps (one per TMEM lane quarter), group g owning layers l % G == g:
//    tcgen05.ld -> +bias, ReLU, zero outside the image -> bf16 -> next layer's ring,
//    or HBM / the fp32 residual G for the chain's last layer;
//  * each role runs one compact code path with a run-time layer index (a warp that owns a
//    single layer walks its fills / output rows directly; the layer-unrolled form lost
//    ~20% of its warp time to instruction-fetch stalls, profiles/r01_cnn_icache.md);
//    the pipeline trace is compiled only with -DPNPULA_TRACE=1;
//  * fp32 accumulation in TMEM.
// Every output pixel's arithmetic (K order, rounding points) is independent of the
// strip/tile it falls in, so results are bitwise identical for every tile grid.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <type_traits>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "internal.h"
#include "update_math.cuh"

namespace pnpula {

namespace {

#ifndef PNPULA_EPI_GROUPS
#define PNPULA_EPI_GROUPS 4
#endif
constexpr int kRowPos = 130;                    // positions per ring row (128 MMA rows + 1 each side)
// Shared-memory alignment of the activation rings (r02, exp/mma_align.cu): a tcgen05 operand whose
// core matrices (8 rows x 16 B) do not start on a 128-B boundary costs about 1.3x the fetch of an
// aligned one (N = 96: ~90 vs ~69 cycles).  The dx taps shift A by 16 B, so at most one of the
// three can be aligned: the channel-group stride is padded to 136 positions (2,176 B = 17 x 128)
// and each ring starts 16 B before a 128-B boundary, so position 1 -- the centre tap of a windowed
// layer and the unshifted A of the folded last layer -- is aligned in every channel group.
#ifndef PNPULA_RING_ALIGN
#define PNPULA_RING_ALIGN 0   // measured neutral on c5 (profiles/r02_cnn_schemes.md): off, 6 KB less smem
#endif
constexpr int kRowStride = PNPULA_RING_ALIGN ? 136 : kRowPos;   // positions between channel groups
constexpr uint32_t kRingPad = PNPULA_RING_ALIGN ? 112u : 0u;      // ring base = 128 k + 112
constexpr int kEpiGroups = PNPULA_EPI_GROUPS;   // max epilogue groups (each: 4 warps = 4 TMEM lane quarters)
#ifndef PNPULA_MMA_WARPS
#define PNPULA_MMA_WARPS 4
#endif
constexpr int kMmaWarps = PNPULA_MMA_WARPS;     // max MMA issuers: MMA warp w owns layers l % MW == w
#ifndef PNPULA_PROD_WARPS
#define PNPULA_PROD_WARPS 4
#endif
constexpr int kProdWarps = PNPULA_PROD_WARPS;   // producers: warp w fills ring-0 rows f % kProdWarps == w
constexpr int kMma0 = kProdWarps;               // first MMA warp (also allocates TMEM)
// Per chain length NL: MMA warps MW and epilogue groups EG (at most one per layer), first
// epilogue warp, block size -- producer warps, MMA warps, epilogue warps.
__host__ __device__ constexpr int mma_warps(int nl) { return nl < kMmaWarps ? nl : kMmaWarps; }
// two-layer chains (DDFB operator pairs; P = 64 DnCNN chunks) give layer 0 two epilogue groups
// (even / odd output rows): its P-channel epilogue, not the MMAs, bounds those launches
__host__ __device__ constexpr int epi_groups(int nl) { return nl == 2 ? 3 : nl < kEpiGroups ? nl : kEpiGroups; }
__host__ __device__ constexpr int epi0(int nl) { return kMma0 + mma_warps(nl); }
__host__ __device__ constexpr int block_threads(int nl) { return 32 * (epi0(nl) + 4 * epi_groups(nl)); }
constexpr int kRing = 4;                        // input-row ring slots of layer 0 (one per producer warp)
#ifndef PNPULA_RING_ACT
#define PNPULA_RING_ACT 4
#endif
constexpr int kRingAct = PNPULA_RING_ACT;       // ring slots of the epilogue-fed layers l >= 1
static_assert(kRingAct >= 3 && kRingAct <= 8, "input ring slots");
__host__ __device__ constexpr uint32_t ring_slots(int l) { return l == 0 ? (uint32_t)kRing : (uint32_t)kRingAct; }
constexpr int kAcc = 4;                         // accumulator-row slots per layer (TMEM)
constexpr int kXS = 136;                        // staged floats per x row (130 ring positions + alignment)
#ifndef PNPULA_LAG
#define PNPULA_LAG 3
#endif
constexpr int kLag = PNPULA_LAG;                // schedule steps between consecutive layers
static_assert(kLag >= 3 && kLag <= 5, "layer l+1 needs rows completed 2 fills later; ring holds 4");

struct SmemLayout {
  uint32_t ring_off[kMaxChunk];
  uint32_t slot_bytes[kMaxChunk];
  uint32_t w_off[kMaxChunk];
  uint32_t xs_off;      // first-layer x staging: [producer warp][3 C rows][kXS] fp32, then one mbarrier per warp
  uint32_t bar_off;
  uint32_t misc_off;
  uint32_t fu_off;      // fused update (last chunk): x rows [2][144], T1 ring [16][136], Rs rows [2][136],
                        // T2 ring [16][128], G ring [8][128]; then mbarriers gfull[8], gempty[8], sync[2]
  uint32_t total;
};
// fused-update buffers (floats): strip columns <= 126 valid + 2 R (R <= 4); T1 / T2 rings of 16 rows
// (2 R + 1 <= 9 live), G ring of 8 rows handed from the folded layer's epilogue to the producers
constexpr int kFuXS = 144, kFuT1 = 136, kFuT2 = 128, kFuRing = 16, kFuG = 8;
constexpr uint32_t kFuFloats = 2 * kFuXS + kFuRing * kFuT1 + 2 * kFuT1 + kFuRing * kFuT2 + kFuG * 128;

__host__ __device__ inline uint32_t align_up(uint32_t v, uint32_t a) { return (v + a - 1) / a * a; }

// Image channels C (1 grayscale, 3 colour; reading R43) only touch the first layer (im2col:
// 9C taps, K padded to 16 or 32) and the folded last layer (N = 16 per output channel).
__host__ __device__ constexpr int im2col_k(int nc) { return 9 * nc <= 16 ? 16 : 32; }

__host__ __device__ inline uint32_t packed_layer_elems(int cout, int cin) {
  if (cin <= 3) return (uint32_t)im2col_k(cin) * (uint32_t)cout;   // im2col layer: [K/8][N][8]
  if (cout <= 3) return 16u * (uint32_t)cout * (uint32_t)cin;      // folded P -> C: [K step][2][16 C][8]
  return 9u * (uint32_t)cin * (uint32_t)cout;
}

__host__ __device__ inline SmemLayout make_layout(int P, int nl, int first, int last, int nc, int fuse = 0) {
  SmemLayout L{};
  uint32_t off = 0;
  const uint32_t act_slot = (uint32_t)(P / 8) * kRowStride * 16u;
  for (int l = 0; l < nl; ++l) {
    const bool im = l == 0 && first;
    L.slot_bytes[l] = im ? (uint32_t)(im2col_k(nc) / 8) * 128u * 16u : act_slot;
    if (!im) off += kRingPad;   // position 1 of every activation row on a 128-B boundary
    L.ring_off[l] = off;
    off = align_up(off + ring_slots(l) * L.slot_bytes[l], 128);
  }
  for (int l = 0; l < nl; ++l) {
    const int cin = (l == 0 && first) ? nc : P;
    const int cout = (l == nl - 1 && last) ? nc : P;
    L.w_off[l] = off;
    off = align_up(off + packed_layer_elems(cout, cin) * 2u, 128);
  }
  if (first) {       // x rows of the im2col producer (TMA bulk copies), + one mbarrier per producer warp
    L.xs_off = off;
    off = align_up(off + (uint32_t)(kProdWarps * 3 * nc * kXS) * 4u + (uint32_t)kProdWarps * 8u, 128);
  }
  L.bar_off = off;   // per layer: full[8], empty[8], tfull[4], tempty[4]
  off = align_up(off + (uint32_t)nl * 24u * 8u, 128);
  L.misc_off = off;  // tmem address, abort flag, drain barrier, per-layer table {ring, slot, w, 0},
                     // folded last layer's warp-edge exchange [2][C][4 warps][6] floats
  off += 16 + 16u * (uint32_t)nl + 192u * (uint32_t)nc;
  if (fuse) {
    off = align_up(off, 16);
    L.fu_off = off;
    off += kFuFloats * 4u + (2u * kFuG + 2u) * 8u;   // + the producers' row barriers sync[2]
  }
  L.total = align_up(off, 128);
  return L;
}

// ---------------------------------------------------------------- PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ bool mbar_test(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
// try_wait with a suspend-time hint: the warp sleeps in hardware until the phase completes
// (or ~0.5 ms pass) instead of spinning.
__device__ __forceinline__ bool mbar_test_sleep(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity), "r"(500000u)
      : "memory");
  return ok != 0;
}
// Bounded wait: gives up (sets the CTA abort flag and the device error flag) after
// ~4e9 cycles so a pipeline bug cannot hang the GPU.
#ifndef PNPULA_ONE_COMMIT
#define PNPULA_ONE_COMMIT 1   // one tcgen05.commit per fill (see epi_step)
#endif
#ifndef PNPULA_POLL_BATCH
#define PNPULA_POLL_BATCH 32   // tries between two watchdog checks (profiles/r02_cnn_schemes.md)
#endif
__device__ __noinline__ bool mbar_wait_slow(uint32_t bar, uint32_t parity, volatile int *abort, int *err, int code) {
  const long long t0 = clock64();
  while (true) {
#pragma unroll 1
    for (int i = 0; i < PNPULA_POLL_BATCH; ++i)
      if (mbar_test_sleep(bar, parity)) return true;
    if (*abort) return false;
    if (clock64() - t0 > (1ll << 32)) {
      *abort = 1;
      atomicExch(err, code);
      return false;
    }
  }
}
__device__ __forceinline__ bool mbar_wait(uint32_t bar, uint32_t parity, volatile int *abort, int *err, int code) {
  if (mbar_test(bar, parity)) return true;
  return mbar_wait_slow(bar, parity, abort, err, code);
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// UMMA shared-memory descriptor, K-major, no swizzle (canonical layout
// ((8,m),(8,2)) : ((16B, SBO), (2B, LBO)) -- core matrix = 8 rows x 16 bytes).
// Adding k to the descriptor moves its start address by 16k bytes.
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;   // descriptor version (sm_100)
  // base offset 0, lbo mode 0, layout type 0 (SWIZZLE_NONE)
  return d;
}

// Instruction descriptor, kind::f16: D = F32, A = B = BF16, both K-major, M = 128.
__host__ __device__ constexpr uint32_t make_idesc(int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// A-operand collector reuse (kernel experiment PNPULA_COLLECTOR_A): the first MMA of a ring-wrap
// split pair keeps its A tile in the tensor core's operand collector, the second reuses it.
__device__ __forceinline__ void mma_bf16_afill(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc) {
  asm volatile("tcgen05.mma.cta_group::1.kind::f16.collector::a::fill [%0], %1, %2, %3, 1;" ::"r"(d_tmem), "l"(adesc),
               "l"(bdesc), "r"(idesc)
               : "memory");
}
__device__ __forceinline__ void mma_bf16_alast(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc) {
  asm volatile("tcgen05.mma.cta_group::1.kind::f16.collector::a::lastuse [%0], %1, %2, %3, 1;" ::"r"(d_tmem), "l"(adesc),
               "l"(bdesc), "r"(idesc)
               : "memory");
}
#ifndef PNPULA_COLLECTOR_A
#define PNPULA_COLLECTOR_A 0
#endif

__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}

template <int N>
__device__ __forceinline__ void tmem_load(uint32_t taddr, float *v);

template <>
__device__ __forceinline__ void tmem_load<1>(uint32_t taddr, float *v) {
  uint32_t r;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(taddr) : "memory");
  v[0] = __uint_as_float(r);
}
template <>
__device__ __forceinline__ void tmem_load<16>(uint32_t taddr, float *v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
template <>
__device__ __forceinline__ void tmem_load<32>(uint32_t taddr, float *v) {
  tmem_load<16>(taddr, v);
  tmem_load<16>(taddr + 16, v + 16);
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// zero n consecutive TMEM columns of this warp's 32 lanes
template <int N>
__device__ __forceinline__ void tmem_zero(uint32_t taddr);
template <>
__device__ __forceinline__ void tmem_zero<1>(uint32_t taddr) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(taddr), "r"(0u) : "memory");
}
template <>
__device__ __forceinline__ void tmem_zero<16>(uint32_t taddr) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr),
      "r"(0u)
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// ReLU + round-to-nearest bf16 of a pair, packed (lo in the low half): one instruction
__device__ __forceinline__ uint32_t relu_pack_bf16(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.relu.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
#ifndef PNPULA_EPI_CVT
#define PNPULA_EPI_CVT 1   // 1: bias add + cvt.rn.relu.bf16x2 per pair, outside-image zeroing behind a vote
#endif

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t *>(&v);
}

// Pipeline trace (diagnostics only; p.trace == nullptr in production): one 64-bit record
// per event = clock64 << 20 | code << 16 | step << 4 | layer.  Each tracing thread owns a
// private region (code 1-2: producer, 3-5 and 14: MMA, 6-11: epilogue), plain stores only.
#ifndef PNPULA_TRACE
#define PNPULA_TRACE 0   // 1: compile the pipeline trace (diagnostics builds only)
#endif
__device__ __forceinline__ void trace_ev(unsigned long long *tr, bool on, int code, int s, int l) {
  if (!PNPULA_TRACE || !on) return;
  const unsigned long long t = (unsigned long long)clock64();
  const int region = code <= 2 ? 0 : (code <= 5 || code == 14) ? 1 : 2;
  const unsigned idx = (unsigned)(s * 8 + l) * 8 + (unsigned)(code & 7);
  if (idx < (1u << 18))
    tr[1 + (region << 18) + idx] =
        (t << 20) | ((unsigned long long)code << 16) | ((unsigned long long)(s & 0xfff) << 4) | (unsigned)l;
}

// ---------------------------------------------------------------- the kernel
template <int P, int NL, int NC, bool FU>
__global__ void __launch_bounds__(block_threads(NL), 1) cnn_chunk_kernel(const __grid_constant__ CnnChunkParams p) {
  constexpr int kMmaWarps = mma_warps(NL), kEpiGroups = epi_groups(NL), kEpi0 = epi0(NL);
  constexpr int kThreads = block_threads(NL);
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int G = P / 8;              // channel groups of 8
  constexpr int KS = P / 16;            // K steps per tap
  constexpr uint32_t GS = kRowStride * 16; // bytes between channel groups in a ring row
  const bool first = p.first_is_input != 0;
  const bool last = p.last_is_output != 0;
  // fused x / z / moment update (chains whose layer 0 is fed by TMA: the producers have the time)
  const bool fuse = FU && last && !first && p.fuse != 0;
  const SmemLayout L = make_layout(P, NL, first, last, NC, fuse ? 1 : 0);
  constexpr int K0 = im2col_k(NC);      // im2col K (9 NC taps, zero padded)
  constexpr bool kDdfb = NL <= 2;   // DDFB operator modes compiled in (R39-R42; C = 1 or 3)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar0 = sbase + L.bar_off;
  // per layer: full[8], empty[8] (input ring), tfull[4], tempty[4] (accumulator ring)
  auto bar_full = [&](int l, uint32_t s) { return bar0 + (uint32_t)(l * 24 + s) * 8u; };
  auto bar_empty = [&](int l, uint32_t s) { return bar0 + (uint32_t)(l * 24 + 8 + s) * 8u; };
  auto bar_tfull = [&](int l, uint32_t s) { return bar0 + (uint32_t)(l * 24 + 16 + s) * 8u; };
  auto bar_tempty = [&](int l, uint32_t s) { return bar0 + (uint32_t)(l * 24 + 20 + s) * 8u; };
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + L.misc_off);
  volatile int *abort_flag = reinterpret_cast<volatile int *>(smem + L.misc_off + 4);
  const uint32_t bar_done = sbase + L.misc_off + 8;
  // TMEM: layer l owns columns [l*4P, l*4P + 4*Cb): accumulator-row slot q at l*4P + q*Cb
  constexpr uint32_t tmem_need = (uint32_t)NL * kAcc * P;
  static_assert(tmem_need <= 512, "TMEM columns");
  constexpr uint32_t tmem_cols = tmem_need <= 32 ? 32 : tmem_need <= 64 ? 64 : tmem_need <= 128 ? 128
                                 : tmem_need <= 256 ? 256 : 512;

  pdl_trigger();   // the next kernel's CTAs may start their own prologue as SMs free up
  // ---- one-time setup: weights, biases, zero rings, barriers, TMEM (nothing the previous kernel wrote)
#pragma unroll
  for (int l = 0; l < NL; ++l) {
    const int cin = (l == 0 && first) ? NC : P;
    const int cout = (l == NL - 1 && last) ? NC : P;
    const uint32_t n16 = packed_layer_elems(cout, cin) / 8;   // 16-byte chunks
    const uint4 *src = reinterpret_cast<const uint4 *>(p.w[l]);
    uint4 *dst = reinterpret_cast<uint4 *>(smem + L.w_off[l]);
    for (uint32_t e = threadIdx.x; e < n16; e += kThreads) dst[e] = src[e];
    uint4 *r = reinterpret_cast<uint4 *>(smem + L.ring_off[l]);
    const uint32_t nr = ring_slots(l) * L.slot_bytes[l] / 16;
    for (uint32_t e = threadIdx.x; e < nr; e += kThreads) r[e] = make_uint4(0, 0, 0, 0);
  }
  if (threadIdx.x == 0) {
    for (int l = 0; l < NL; ++l) {
      for (int s = 0; s < (int)ring_slots(l); ++s) {
        mbar_init(bar_full(l, s), (l == 0) ? 1 : 4);   // producer lane, or the 4 warps of one group
        mbar_init(bar_empty(l, s), 1);
      }
      for (int s = 0; s < kAcc; ++s) {
        mbar_init(bar_tfull(l, s), 1);
        mbar_init(bar_tempty(l, s), 4);
      }
    }
    mbar_init(bar_done, kMmaWarps);
    if (FU && fuse)
      for (int g2 = 0; g2 < kFuG; ++g2) {
        mbar_init(sbase + L.fu_off + kFuFloats * 4u + (uint32_t)g2 * 8u, 4);            // G row full: 4 epilogue warps
        mbar_init(sbase + L.fu_off + kFuFloats * 4u + (uint32_t)(kFuG + g2) * 8u, 4);   // G row read: 4 producer warps
        if (g2 < 2) mbar_init(sbase + L.fu_off + kFuFloats * 4u + (uint32_t)(2 * kFuG + g2) * 8u, 4);   // stencil rows
      }
    if (first)
      for (int w = 0; w < kProdWarps; ++w) mbar_init(sbase + L.xs_off + (uint32_t)(kProdWarps * 3 * NC * kXS) * 4u + w * 8u, 1);
    *abort_flag = 0;
    uint4 *tab = reinterpret_cast<uint4 *>(smem + L.misc_off + 16);
    for (int l = 0; l < NL; ++l) tab[l] = make_uint4(L.ring_off[l], L.slot_bytes[l], L.w_off[l], 0u);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kMma0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // accumulators start at zero (every slot is re-zeroed by the epilogue after it is read)
  if (warp >= kEpi0 && warp < kEpi0 + 4) {
    const uint32_t lb = (uint32_t)((warp & 3) * 32) << 16;
    for (uint32_t c = 0; c < tmem_need; c += 16) tmem_zero<16>(tmem_base + lb + c);
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_wait();      // programmatic dependent launch: the previous kernel's writes are visible from here
  // fused update: iteration scalars (by value, or the device IterState of a graph replay), and the
  // next iteration's scalars written once (as the first update launch of an unfused step does)
  uint32_t fu_t1 = 0;
  int fu_acc = 0;
  float fu_invn = 0.f;
  if (FU && fuse) {
    const UpdateParams &U = p.up;
    if (U.it) { fu_t1 = (uint32_t)U.it->t1; fu_acc = U.it->accumulate; fu_invn = U.it->inv_n; }
    else { fu_t1 = U.t1; fu_acc = U.accumulate; fu_invn = U.inv_n; }
    if (U.it_next && blockIdx.x == 0 && threadIdx.x == 0) {
      const long long t1n = U.it->t1 + 1, b = U.it->burn_in;
      const bool acc = t1n > b;
      U.it_next->t1 = t1n;
      U.it_next->burn_in = b;
      U.it_next->accumulate = acc;
      U.it_next->inv_n = (float)(1.0 / (acc ? (double)(t1n - b) : 1.0));
    }
  }

  // valid output columns per strip: each fused layer costs one column per side; the folded
  // P -> 1 layer needs its MMA rows m +- 1, so a 1-layer chunk ending the net counts as 2
  constexpr int NLg0 = NL < 2 ? 2 : NL;
  const int NLg = last ? NLg0 : NL;
  const int Wv = kRowPos - 2 * NLg;
  const int strips = p.strips;
  const int R = p.rows_per_unit;
  const int units = p.units;
  // The role loops below index layers at run time (no unrolling over layers): every warp
  // executes one compact code path, which keeps the hot code inside the instruction cache
  // (the layer-unrolled form spent ~20% of its warp time in instruction-fetch stalls).
  // Per-layer shared-memory offsets come from the table written at setup.
  const uint4 *ltab = reinterpret_cast<const uint4 *>(smem + L.misc_off + 16);   // {ring, slot, w, -}
  auto is_im2col = [&](int l) { return l == 0 && first; };
  // running counters before the current unit (k = units this CTA finished, sumRn = their rows):
  // fills of layer l: sumRn + k (2 (NL-1-l) + 2 [l not im2col]); output rows: sumRn + k 2 (NL-1-l)
  uint32_t sumRn = 0, kdone = 0;
  auto Fcnt = [&](int l) { return sumRn + kdone * (uint32_t)(2 * (NL - 1 - l) + (is_im2col(l) ? 0 : 2)); };
  auto Ocnt = [&](int l) { return sumRn + kdone * (uint32_t)(2 * (NL - 1 - l)); };

  uint32_t xphase = 0;   // im2col producers: phase of this warp's x-staging mbarrier
  // fused update: stencil row barriers this producer warp has passed -- across units, as the
  // mbarrier phases persist (all 4 producer warps pass the same sequence)
  [[maybe_unused]] uint32_t fu_nsync = 0;
  // Work units.  Row blocks (rows_per_cta == 0): unit u = (row block u / strips, strip u % strips),
  // CTAs take units round-robin.  Contiguous (rows_per_cta = T > 0): CTA b owns the strip-major
  // output rows [b T, (b+1) T) of the strips x oh grid, one unit per strip it touches -- every unit
  // pays the pipeline's fill once, so a CTA pays it once or twice instead of once per row block.
  // (2-layer chains -- DDFB operator pairs -- always use row blocks: their kernel keeps the plain
  // round-robin loop, whose code generation the ranges' bookkeeping measurably perturbed)
  const int Tc = NL <= 2 ? 0 : p.rows_per_cta;
  int64_t cpos = (int64_t)blockIdx.x * Tc;
  const int64_t cend = Tc > 0 ? min((int64_t)(blockIdx.x + 1) * Tc, (int64_t)strips * p.oh) : 0;
  bool first_unit = true;
  for (int u = blockIdx.x;;) {
    int strip, r_lo, r_hi;
    if (Tc > 0) {
      if (cpos >= cend) break;
      strip = (int)(cpos / p.oh);
      const int64_t segend = min(cend, (int64_t)(strip + 1) * p.oh);
      r_lo = p.oi0 + (int)(cpos - (int64_t)strip * p.oh);
      r_hi = r_lo + (int)(segend - cpos);
      cpos = segend;
    } else {
      if (u >= units) break;
      const int rb = u / strips;
      strip = u - rb * strips;
      r_lo = p.oi0 + rb * R;
      r_hi = min(r_lo + R, p.oi0 + p.oh);
      u += gridDim.x;
    }
    if (*abort_flag) break;
    const int Rn = r_hi - r_lo;
    const int c_strip0 = p.oj0 + strip * Wv;         // first valid output column of the strip
    const int col0 = c_strip0 - NLg + 1;             // column of MMA row 0 (ring position 1)
    const bool tr_on = p.trace != nullptr && blockIdx.x == 0 && first_unit;
    // layer l: nout(l) = Rn + 2 (NL-1-l) output rows starting at global row r_lo-(NL-1-l);
    // its input fills are rows r0(l)-1 .. (nout+2 fills), or nout im2col rows for an im2col layer.
    auto nout = [&](int l) { return Rn + 2 * (NL - 1 - l); };
    auto nfill = [&](int l) { return is_im2col(l) ? nout(0) : nout(l) + 2; };
    const int S = kLag * (NL - 1) + nfill(NL - 1) > nfill(0) ? kLag * (NL - 1) + nfill(NL - 1) : nfill(0);

    if (warp < kProdWarps) {
      // ================= producers: ring 0.  Warp w owns ring slot w for the whole kernel (fills
      // with (Fcnt + f) & 3 == w): a slot's fills are then issued in order by one warp, which can
      // never run two mbarrier phases ahead of the slot (a parity wait would pass spuriously).
      static_assert(kProdWarps == kRing || kProdWarps == 1, "one producer per ring slot");
      const int nf = nfill(0);
      const uint32_t F0 = Fcnt(0);
      const uint32_t ring0 = ltab[0].x, slot0 = ltab[0].y;
      const int f0 = (kProdWarps == 1) ? 0 : (int)(((uint32_t)warp - F0) & 3u);
      // ---- fused update (FU && fuse): the 4 producer warps (one pixel per lane: m = 32 w + lane,
      // the folded layer's lane mapping) also run the x / z / moment update of every completed
      // output row.  g = H^T(eta H x - y) is streamed row by row in the order of update_sep_kernel:
      //   T1(r, c) = sum_q kx[q+R] x(r, c - q)                 (columns c = fcT + k, k < fKW)
      //   Rs(r, c) = eta sum_q ky[q+R] T1(r - q, c) - y(r, c)  (0 outside the image)
      //   T2(r, c) = sum_q kx[q+R] Rs(r, c + q)                (the strip's valid columns)
      //   g(o, c)  = sum_q ky[q+R] T2(o + q, c)                (q = -R .. R, fma chains from 0)
      // (T1 / Rs columns k = m, m + 128 and the T2 column of a lane's pixel are its own: the rings
      // need no barrier; the x and Rs rows read across lanes are double-buffered behind one named
      // barrier of the 128 producer threads per row.)  G arrives through the G ring.  A warp
      // finishes output row ic only after issuing its layer-0 fills up to ic + 2 + kLag (NL-1) + 4,
      // so a row it waits for never depends on a fill it has not issued (no deadlock).
      [[maybe_unused]] int fu_done = 0;
      // the next row's global operands, loaded one row ahead (valid when fu_pf == fu_done)
      [[maybe_unused]] int fu_pf = -1;
      [[maybe_unused]] float pf_x = 0.f, pf_z = 0.f, pf_m = 0.f, pf_s = 0.f, pf_y = 0.f;
      [[maybe_unused]] float pf_xa = 0.f, pf_xb = 0.f, pf_ya = 0.f, pf_yb = 0.f;
      [[maybe_unused]] uint8_t pf_mk = 0;
      [[maybe_unused]] const int fu_lag = 2 + kLag * (NL - 1) + 4;
      [[maybe_unused]] bool fu_warm = false;
      // rows [fu_done, icmax] of this unit, for a compile-time stencil radius R (0: mask, no stencil)
      auto fu_rows_R = [&](auto Rc, int icmax) -> bool {
        constexpr int R = decltype(Rc)::value;
        const UpdateParams &U = p.up;
        const int l = NL - 1;
        const int no = nout(l);
        constexpr int KX = 2 * R;
        const int fKW = Wv + KX;            // T1 / Rs columns c = fcT + k
        const int fcT = c_strip0 - R;
        const int m = warp * 32 + lane;
        const int cm = col0 + m;
        const bool fu_lane = cm >= c_strip0 && cm < c_strip0 + Wv;
        const bool cvalid = fu_lane && cm < p.oj0 + p.ow;
        const bool k2 = m + 128 < fKW;      // this lane also owns T1 / Rs column m + 128
        const bool x2 = m + 128 < fKW + KX; // ... and x staging column m + 128
        float *const fxs = reinterpret_cast<float *>(smem + L.fu_off);
        float *const fT1 = fxs + 2 * kFuXS;
        float *const fRS = fT1 + kFuRing * kFuT1;
        float *const fT2 = fRS + 2 * kFuT1;
        float *const fG = fT2 + kFuRing * kFuT2;
        const uint32_t gb = sbase + L.fu_off + kFuFloats * 4u;
        const TileGeom &g = U.g;
        auto ldpad = [&](const float *b, int row, int col) -> float {   // 0 outside the buffer (TMA)
          const int pr = row - (g.i0 - g.h), pc = col - (g.j0 - g.hx);
          return (pr >= 0 && pr < g.ph && pc >= 0 && pc < g.pitch) ? b[(int64_t)pr * g.pitch + pc] : 0.f;
        };
        // barrier of the 4 producer warps (two mbarriers used alternately, one arrival per warp; the
        // bounded wait keeps an aborted CTA from hanging, unlike a named barrier)
        auto pbar = [&]() -> bool {
          const uint32_t b = gb + (2u * kFuG + (fu_nsync & 1u)) * 8u;
          const uint32_t ph = (fu_nsync >> 1) & 1u;
          ++fu_nsync;
          __syncwarp();
          if (lane == 0) mbar_arrive(b);
          return mbar_wait(b, ph, abort_flag, p.err, 11);
        };
        auto stage_x = [&](int row, float a0, float a1) {   // x row `row`, columns fcT - R + u
          float *const xs = fxs + (row & 1) * kFuXS;
          xs[m] = a0;
          if (x2) xs[m + 128] = a1;
        };
        auto t1_at = [&](int row, int k) {                   // T1(row, fcT + k) = sum_q kx[q+R] x(row, c - q)
          const float *const xs = fxs + (row & 1) * kFuXS;
          float sa = 0.f;
#pragma unroll
          for (int q = -R; q <= R; ++q) sa = fmaf(U.kx[q + R], xs[k + R - q], sa);
          fT1[(row & (kFuRing - 1)) * kFuT1 + k] = sa;
        };
        auto rs_at = [&](int row, int k, float yv) {         // Rs(row, c) = eta sum_q ky[q+R] T1(row - q, c) - y
          float sa = 0.f;
#pragma unroll
          for (int q = -R; q <= R; ++q) sa = fmaf(U.ky[q + R], fT1[((row - q) & (kFuRing - 1)) * kFuT1 + k], sa);
          const int c = fcT + k;
          fRS[(row & 1) * kFuT1 + k] = (row >= 0 && row < p.ny && c >= 0 && c < p.nx) ? U.eta * sa - yv : 0.f;
        };
        auto t2_own = [&](int row) {                         // T2(row, cm) = sum_q kx[q+R] Rs(row, cm + q)
          if (!fu_lane) return;
          const float *const rs = fRS + (row & 1) * kFuT1 + (cm - fcT);
          float sa = 0.f;
#pragma unroll
          for (int q = -R; q <= R; ++q) sa = fmaf(U.kx[q + R], rs[q], sa);
          fT2[(row & (kFuRing - 1)) * kFuT2 + m] = sa;
        };
        if constexpr (R > 0) {
          if (!fu_warm) {   // unit start: T1 rows r_lo-2R .. r_lo+2R-1, Rs / T2 rows r_lo-R .. r_lo+R-1
            for (int t = r_lo - 2 * R; t < r_lo + 2 * R; ++t) {
              stage_x(t, ldpad(U.x, t, fcT - R + m), x2 ? ldpad(U.x, t, fcT - R + m + 128) : 0.f);
              if (!pbar()) return false;
              t1_at(t, m);
              if (k2) t1_at(t, m + 128);
            }
            for (int t = r_lo - R; t < r_lo + R; ++t) {
              rs_at(t, m, ldpad(U.y, t, fcT + m));
              if (k2) rs_at(t, m + 128, ldpad(U.y, t, fcT + m + 128));
              if (!pbar()) return false;
              t2_own(t);
            }
            const int t = r_lo + 2 * R;
            stage_x(t, ldpad(U.x, t, fcT - R + m), x2 ? ldpad(U.x, t, fcT - R + m + 128) : 0.f);
            if (!pbar()) return false;
          }
        }
        fu_warm = true;
        const int last_ic = icmax < no - 1 ? icmax : no - 1;
        // global operands of row ic (pixel: x, z, mean, M2 [, mask, y]; stencil: x row o + 2R + 1 and
        // y row o + R at this lane's staging / Rs columns) into the pf_ registers
        auto prefetch = [&](int ic) {
          const int o = r_lo + ic;
          if (cvalid) {
            const int64_t idx = (int64_t)(o - (g.i0 - g.h)) * g.pitch + (cm - (g.j0 - g.hx));
            pf_x = U.x[idx];
            if (U.has_z) pf_z = U.z[idx];
            if (fu_acc) { pf_m = U.mean[idx]; pf_s = U.m2[idx]; }
            if (R == 0) { pf_mk = U.mask[idx]; pf_y = U.y[idx]; }
          }
          if constexpr (R > 0) {
            const int tx = o + 2 * R + 1, ty = o + R;
            pf_xa = ldpad(U.x, tx, fcT - R + m);
            pf_xb = x2 ? ldpad(U.x, tx, fcT - R + m + 128) : 0.f;
            pf_ya = ldpad(U.y, ty, fcT + m);
            pf_yb = k2 ? ldpad(U.y, ty, fcT + m + 128) : 0.f;
          }
          fu_pf = ic;
        };
        for (; fu_done <= last_ic; ++fu_done) {
          const int ic = fu_done;
          const int o = r_lo + ic;
          // A. this row's operands (loaded one row ahead), then the next row's requested
          if (fu_pf != ic) prefetch(ic);
          const float fx = pf_x, fz = pf_z, fm0 = pf_m, fs0 = pf_s, fy = pf_y;
          const uint8_t fmk = pf_mk;
          const float xa = pf_xa, xb = pf_xb, ya = pf_ya, yb = pf_yb;
          const int64_t idx = (int64_t)(o - (g.i0 - g.h)) * g.pitch + (cm - (g.j0 - g.hx));
          if (ic + 1 < no) prefetch(ic + 1);
          // the noise does not depend on the stencil or G: computed while the loads are in flight
          float xi = 0.f, ze = 0.f;
          if (cvalid) {
            xi = upd::normal1(U.seed_lo, U.seed_hi, (uint32_t)cm >> 2, (uint32_t)o, fu_t1, U.sb + 0u, cm & 3);
            if (U.has_z) ze = upd::normal1(U.seed_lo, U.seed_hi, (uint32_t)cm >> 2, (uint32_t)o, fu_t1, U.sb + 1u, cm & 3);
          }
          float fm = fm0, fs = fs0;
          float gr = 0.f;
          if constexpr (R > 0) {
            const int tx = o + 2 * R + 1, ty = o + R;
            // B. T1(o + 2R) (x row staged last iteration); C. Rs(o + R); D. stage x(o + 2R + 1)
            t1_at(o + 2 * R, m);
            if (k2) t1_at(o + 2 * R, m + 128);
            rs_at(ty, m, ya);
            if (k2) rs_at(ty, m + 128, yb);
            stage_x(tx, xa, xb);
            if (!pbar()) return false;   // E. one barrier per row
            t2_own(ty);                  // F. T2(o + R)
            if (fu_lane) {               // G. g(o) = sum_q ky[q+R] T2(o + q, cm)
#pragma unroll
              for (int q = -R; q <= R; ++q) gr = fmaf(U.ky[q + R], fT2[((o + q) & (kFuRing - 1)) * kFuT2 + m], gr);
            }
          } else if (cvalid) {
            const float mk = fmk ? 1.f : 0.f;
            gr = mk * (mk * fx - fy);
          }
          // H. G from the ring, then the K7 tail (update_math.cuh)
          const uint32_t Ig = Ocnt(l) + (uint32_t)ic;
          const uint32_t gs = Ig & (kFuG - 1);
          if (!mbar_wait(gb + gs * 8u, (Ig / kFuG) & 1, abort_flag, p.err, 10)) return false;
          const float Gv = fG[gs * 128 + m];
          __syncwarp();
          if (lane == 0) mbar_arrive(gb + (kFuG + gs) * 8u);
          if (cvalid) {
            const float xn = upd::x_step<0>(U, false, fx, gr, Gv, fz, 0.f, xi);
            U.xn[idx] = xn;
            if (U.has_z) U.z[idx] = upd::z_step(U, fz, xn, ze);
            if (fu_acc) {
              upd::welford(xn, fu_invn, fm, fs);
              U.mean[idx] = fm;
              U.m2[idx] = fs;
            }
          }
        }
        return true;
      };
      auto fu_rows_upto = [&](int icmax) -> bool {
        if constexpr (FU) {
          if (!fuse) return true;
          const int fR = p.up.op != 1 ? p.up.ry : 0;
          if (fR == 4) return fu_rows_R(std::integral_constant<int, 4>{}, icmax);
          if (fR == 2) return fu_rows_R(std::integral_constant<int, 2>{}, icmax);
          return fu_rows_R(std::integral_constant<int, 0>{}, icmax);
        }
        return true;
      };
      for (int f = f0; f < nf; f += kProdWarps) {
        const uint32_t Fg = F0 + f;
        if (Fg >= 4 && !mbar_wait(bar_empty(0, Fg & 3), ((Fg >> 2) - 1) & 1, abort_flag, p.err, 1)) break;
        trace_ev(p.trace, tr_on && lane == 0, 1, f, 0);
        uint8_t *slot = smem + ring0 + (Fg & 3) * slot0;
        if (first) {
          // im2col row for layer-1 output row o: 9 taps per image channel of x (bf16), tap
          // k = ch * 9 + (dy+1) * 3 + (dx+1), K padded to 16 (C = 1) or 32 (C = 3).  The 3 C x
          // rows (positions col0-1 .. col0+128) are first staged in shared memory by TMA bulk
          // copies (one round trip per fill instead of one per 32 pixels), then read from there.
          const int o = r_lo - NL + f + 1;
          const TileGeom &g = p.xg;
          float *xs = reinterpret_cast<float *>(smem + L.xs_off) + warp * 3 * NC * kXS;
          const uint32_t xbar = sbase + L.xs_off + (uint32_t)(kProdWarps * 3 * NC * kXS) * 4u + warp * 8u;
          const int pc0 = col0 - 1 - (g.j0 - g.hx);   // padded column of ring position 0 (>= 0: h >= K)
          const int a0 = pc0 & ~3;                     // 16-byte aligned copy start
          uint32_t total = 0;
#pragma unroll
          for (int r = 0; r < 3 * NC; ++r) {
            const int pr = o + (r % 3) - 1 - (g.i0 - g.h);
            const int nv = (pr >= 0 && pr < g.ph) ? min(kXS, g.pitch - a0) : 0;   // multiple of 4
            for (int e = nv + lane; e < kXS; e += 32) xs[r * kXS + e] = 0.f;    // outside the buffer
            total += (uint32_t)nv * 4u;
          }
          fence_proxy_async();   // earlier generic reads / the zero fill before the async-proxy writes
          __syncwarp();
          if (lane == 0) {
            asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(xbar), "r"(total)
                         : "memory");
#pragma unroll
            for (int r = 0; r < 3 * NC; ++r) {
              const int pr = o + (r % 3) - 1 - (g.i0 - g.h);
              const int nv = (pr >= 0 && pr < g.ph) ? min(kXS, g.pitch - a0) : 0;
              if (nv > 0)
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        smem_u32(xs + r * kXS)),
                    "l"(p.x + (int64_t)(r / 3) * p.xcs + (int64_t)pr * g.pitch + a0), "r"(nv * 4), "r"(xbar)
                    : "memory");
            }
          }
          if (!mbar_wait(xbar, xphase, abort_flag, p.err, 7)) break;
          xphase ^= 1u;
          for (int m = lane; m < 128; m += 32) {
            float t[K0];
#pragma unroll
            for (int k = 9 * NC; k < K0; ++k) t[k] = 0.f;
            const float *xm = xs + (pc0 - a0) + m;   // position m (= column cm - 1) of row 0
#pragma unroll
            for (int ch = 0; ch < NC; ++ch)
#pragma unroll
              for (int u2 = 0; u2 < 3; ++u2)
#pragma unroll
                for (int v2 = 0; v2 < 3; ++v2) t[ch * 9 + u2 * 3 + v2] = xm[(ch * 3 + u2) * kXS + v2];
#pragma unroll
            for (int kg = 0; kg < K0 / 8; ++kg)
              *reinterpret_cast<uint4 *>(slot + kg * 2048 + m * 16) =
                  make_uint4(pack_bf16(t[kg * 8], t[kg * 8 + 1]), pack_bf16(t[kg * 8 + 2], t[kg * 8 + 3]),
                             pack_bf16(t[kg * 8 + 4], t[kg * 8 + 5]), pack_bf16(t[kg * 8 + 6], t[kg * 8 + 7]));
          }
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) mbar_arrive(bar_full(0, Fg & 3));
        } else {
          // activation row from HBM: one TMA bulk copy per 8-channel group (16 B per position,
          // contiguous in the [group][row][col][8] layout); positions outside the stored region
          // are zero-filled with plain stores (only at region edges).
          const int row = r_lo - NL + f;
          const int c0 = col0 - 1;
          const bool row_ok = row >= p.a_i0 && row < p.a_i0 + p.a_rows;
          const int qlo = row_ok ? max(0, p.a_j0 - c0) : kRowPos;
          const int qhi = row_ok ? min(kRowPos, p.a_j0 + p.a_cols - c0) : kRowPos;
          const uint32_t nbytes = qhi > qlo ? (uint32_t)(qhi - qlo) * 16u : 0u;
          if (qlo > 0 || qhi < kRowPos) {
            for (int e = lane; e < G * kRowPos; e += 32) {
              const int gq = e / kRowPos, q = e - gq * kRowPos;
              if (q < qlo || q >= qhi) *reinterpret_cast<uint4 *>(slot + gq * GS + q * 16) = make_uint4(0, 0, 0, 0);
            }
            fence_proxy_async();
          }
          __syncwarp();
          if (lane == 0) {
            const uint32_t fb = bar_full(0, Fg & 3);
            asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(fb),
                         "r"(nbytes * G)
                         : "memory");
            if (nbytes) {
              const uint16_t *src = p.ain + ((int64_t)(row - p.a_i0) * p.a_cols + (c0 + qlo - p.a_j0)) * 8;
              for (int gq = 0; gq < G; ++gq)
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        smem_u32(slot + gq * GS + qlo * 16)),
                    "l"(src + (int64_t)gq * p.a_rows * p.a_cols * 8), "r"(nbytes), "r"(fb)
                    : "memory");
            }
          }
        }
        trace_ev(p.trace, tr_on && lane == 0, 2, f, 0);
        if (FU && fuse && !fu_rows_upto(f - fu_lag)) break;
      }
      if (FU && fuse && !*abort_flag) fu_rows_upto(nout(NL - 1) - 1);
    } else if (warp < kEpi0) {
      // ================= MMA issuers (whole warp walks the schedule; one elected lane issues).
      // MMA warp w owns the layers l % kMmaWarps == w, so one warp's barrier waits overlap the
      // others' MMA issue; layers use disjoint TMEM columns and shared-memory operands.
      const int mw = warp - kMma0;
      // one schedule step of layer l: input fill f (step s = f + kLag l); false on abort
      auto mma_step = [&](const int l, const int f) -> bool {
          const int s = f + kLag * l;
          const int no = nout(l);
          bool ok;
          const bool im2col = is_im2col(l);
          const bool netlast = (l == NL - 1) && last && !im2col;
          const uint32_t Fg = Fcnt(l) + (uint32_t)f;
          trace_ev(p.trace, tr_on && lane == 0, 3, s, l);
          // ring slot and phase of this input row: compile-time divisors on both branches (a ring
          // size selected at run time would put an integer division on the issue path)
          const uint32_t rs = l == 0 ? Fg % (uint32_t)kRing : Fg % (uint32_t)kRingAct;
          const uint32_t rph = l == 0 ? (Fg / (uint32_t)kRing) & 1u : (Fg / (uint32_t)kRingAct) & 1u;
          ok = mbar_wait(bar_full(l, rs), rph, abort_flag, p.err, 2);
          trace_ev(p.trace, tr_on && lane == 0, 14, s, l);
          // output row that receives its first contribution (im2col: the only one)
          const uint32_t O0 = Ocnt(l);
          const uint32_t Ig = O0 + (uint32_t)f;
          if (netlast) {   // 2-slot ring of per-fill accumulators: fill Fg-2 must have been read
            if (ok && Fg >= 2u) ok = mbar_wait(bar_tempty(l, Fg & 1), ((Fg >> 1) - 1) & 1, abort_flag, p.err, 3);
          } else if (ok && f < no && Ig >= (uint32_t)kAcc)
            ok = mbar_wait(bar_tempty(l, Ig & 3), ((Ig >> 2) - 1) & 1, abort_flag, p.err, 3);
          ok = __shfl_sync(0xffffffffu, ok ? 1 : 0, 0) != 0;
          trace_ev(p.trace, tr_on && lane == 0, 4, s, l);
          if (!ok) return false;
          tc_fence_after();
          const uint4 lt = ltab[l];
          const uint32_t acc0 = tmem_base + (uint32_t)(l * kAcc * P);
          const uint32_t wbase = sbase + lt.z;
          const uint32_t slot = sbase + lt.x + rs * lt.y;
          if (im2col) {
            const uint64_t ad = make_desc(slot, 2048, 128);
            const uint64_t bd = make_desc(wbase, (uint32_t)P * 16, 128);
            if (elect_one()) {
#pragma unroll
              for (int ks = 0; ks < K0 / 16; ++ks)   // K step = 2 core-matrix groups of A and B
                mma_bf16(acc0 + (Ig & 3) * P, ad + (uint64_t)(ks * 256), bd + (uint64_t)(ks * 2 * P),
                         make_idesc(P), ks > 0 ? 1u : 0u);
            }
          } else if (netlast) {
            // P -> 1 layer: all nine taps folded into N = 16 (column n = q*3 + dxi, q = 1 - dy),
            // A unshifted (MMA row m = pixel col0 + m); the epilogue adds the dx-shifted columns
            // of neighbouring lanes and the dy rows of consecutive fills.  Fresh 16-column slot
            // per fill (accumulate = 0 on the first K step): no zeroing, no ring wrap.
            // C output channels: 16 columns each (N = 16 C).
            const uint64_t ad0 = make_desc(slot + 16, GS, 128);
            const uint64_t bd0 = make_desc(wbase, 16u * 16u * NC, 128);
            if (elect_one()) {
#pragma unroll
              for (int ks = 0; ks < KS; ++ks)
                mma_bf16(acc0 + (Fg & 1) * 16u * NC, ad0 + (uint64_t)((2 * ks * GS) >> 4),
                         bd0 + (uint64_t)(ks * 32 * NC), make_idesc(16 * NC), ks > 0 ? 1u : 0u);
            }
          } else {
            // input row f contributes to output rows f-2 (dy=+1), f-1 (dy=0), f (dy=-1): B block q=0,1,2.
            // Only rows in [0, no) are accumulated; slots wrap, so the row range splits into <= 2 runs.
            const uint32_t Cb = (uint32_t)P;
            const int ilo = f - 2 > 0 ? f - 2 : 0;
            const int ihi = f < no - 1 ? f : no - 1;
            const uint32_t Ilo = O0 + (uint32_t)ilo;
            const int n1 = (int)min((uint32_t)(ihi - ilo + 1), kAcc - (Ilo & 3));   // rows before the wrap
            const int n2 = (ihi - ilo + 1) - n1;
            const uint64_t ad0 = make_desc(slot, GS, 128);
            const uint64_t bd0 = make_desc(wbase, 3u * Cb * 16u, 128);
            const uint32_t bstep = 3u * Cb * 2u;      // (16 * 3Cb * 2 bytes) >> 4 per (dx, ks) block
            const uint32_t q0 = (uint32_t)(ilo - (f - 2));
            const uint32_t d1 = acc0 + (Ilo & 3) * Cb;
            const uint32_t id1 = make_idesc((int)(n1 * Cb)), id2 = make_idesc((int)((n2 > 0 ? n2 : 1) * Cb));
            const uint32_t d2 = acc0;
            if (elect_one()) {
#pragma unroll
              for (int dx = 0; dx < 3; ++dx) {
#pragma unroll
                for (int ks = 0; ks < KS; ++ks) {
                  const uint64_t ad = ad0 + (uint64_t)((2 * ks * GS + dx * 16) >> 4);
                  const uint64_t bd = bd0 + (uint64_t)((dx * KS + ks) * bstep);
                  if (PNPULA_COLLECTOR_A && n2 > 0) {
                    mma_bf16_afill(d1, ad, bd + (uint64_t)(q0 * Cb), id1);
                    mma_bf16_alast(d2, ad, bd + (uint64_t)((q0 + n1) * Cb), id2);
                  } else {
                    mma_bf16(d1, ad, bd + (uint64_t)(q0 * Cb), id1, 1);
                    if (n2 > 0) mma_bf16(d2, ad, bd + (uint64_t)((q0 + n1) * Cb), id2, 1);
                  }
                }
              }
            }
          }
          __syncwarp();
          if (elect_one()) {
            mma_commit(bar_empty(l, rs));                // input row consumed
            if (netlast) {
              if (!PNPULA_ONE_COMMIT) mma_commit(bar_tfull(l, Fg & 1));   // this fill's tap sums
            } else {
              const int ic = im2col ? f : f - 2;         // output row completed by this group
              // (PNPULA_ONE_COMMIT: the epilogue waits on the input ring's empty barrier of this fill
              // instead -- the same completion, one commit fewer per fill)
              if (!PNPULA_ONE_COMMIT && ic >= 0 && ic < no) mma_commit(bar_tfull(l, (O0 + (uint32_t)ic) & 3));
            }
          }
          __syncwarp();
          trace_ev(p.trace, tr_on && lane == 0, 5, s, l);
          return true;
      };
      if constexpr (NL <= kMmaWarps) {
        // one layer per MMA warp: walk its fills directly
        const int nf = nfill(mw);
        for (int f = 0; f < nf; ++f)
          if (!mma_step(mw, f)) break;
      } else {
        bool ok = true;
        for (int s = 0; s < S && ok; ++s) {
#pragma unroll 1
          for (int l = mw; l < NL && ok; l += kMmaWarps) {
            const int f = s - kLag * l;                  // input fill processed by layer l at step s
            if (f >= 0 && f < nfill(l)) ok = mma_step(l, f);
          }
        }
      }
    } else {
      // ================= epilogue: group g (warps kEpi0+4g ..) owns layers l % kEpiGroups == g
      const int quarter = warp & 3;
      const int grp = (warp - kEpi0) >> 2;
      const int m = quarter * 32 + lane;
      const int cm = col0 + m;
      const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
      const bool col_valid = cm >= c_strip0 && cm < c_strip0 + Wv && cm < p.oj0 + p.ow;
      const bool col_in = cm >= 0 && cm < p.nx;
      const bool trw = tr_on && lane == 0 && quarter == 2;
      // Folded P -> 1 output layer, one input fill f at a time: tap sums d[q*3 + dxi] of this
      // lane's pixel; pixel m's contribution to output row (f - 2 + q) is
      // d_{m-1}[q*3] + d_m[q*3+1] + d_{m+1}[q*3+2] (lanes m +- 1: shuffles, warp edges through
      // shared memory); a row is complete after its third fill.  Lanes 0 / 127 of the strip
      // are never valid output columns.
      float nacc0[NC], nacc1[NC];   // per output channel: running sums of output rows f-2 and f-1
#pragma unroll
      for (int co = 0; co < NC; ++co) { nacc0[co] = 0.f; nacc1[co] = 0.f; }
      float *const xch = reinterpret_cast<float *>(smem + L.misc_off + 16 + 16 * NL);
      auto netlast_fill = [&](const int l, const int f) -> bool {
          const int s = f + kLag * l;
          const uint32_t Fg = Fcnt(l) + (uint32_t)f;
          float fu_g = 0.f;   // fused update: this lane's G value of the completed row
          if (PNPULA_ONE_COMMIT) {
            // this fill's tap sums are complete with its MMAs: its input-ring empty barrier (the slot is
            // re-used by fill Fg + ring size, whose MMAs need fill Fg + 2's accumulators read first)
            const uint32_t rsc = l == 0 ? Fg % (uint32_t)kRing : Fg % (uint32_t)kRingAct;
            const uint32_t phc = l == 0 ? (Fg / (uint32_t)kRing) & 1u : (Fg / (uint32_t)kRingAct) & 1u;
            if (!mbar_wait(bar_empty(l, rsc), phc, abort_flag, p.err, 4)) return false;
          } else if (!mbar_wait(bar_tfull(l, Fg & 1), (Fg >> 1) & 1, abort_flag, p.err, 4)) return false;
          trace_ev(p.trace, trw, 6, s, l);
          tc_fence_after();
          float d[NC][16];
#pragma unroll
          for (int co = 0; co < NC; ++co)
            tmem_load<16>(tmem_base + lane_base + (uint32_t)(l * kAcc * P) + (Fg & 1) * 16u * NC + co * 16u, d[co]);
          tmem_wait_ld();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(bar_tempty(l, Fg & 1));
          float lft[NC][3], rgt[NC][3];
#pragma unroll
          for (int co = 0; co < NC; ++co) {
#pragma unroll
            for (int q = 0; q < 3; ++q) {
              lft[co][q] = __shfl_up_sync(0xffffffffu, d[co][q * 3], 1);
              rgt[co][q] = __shfl_down_sync(0xffffffffu, d[co][q * 3 + 2], 1);
            }
            // [parity][channel][quarter][0-2: lane 31's left taps, 3-5: lane 0's right taps]
            float *xb = xch + ((f & 1) * NC + co) * 24;
            if (lane == 31) {
#pragma unroll
              for (int q = 0; q < 3; ++q) xb[quarter * 6 + q] = d[co][q * 3];
            }
            if (lane == 0) {
#pragma unroll
              for (int q = 0; q < 3; ++q) xb[quarter * 6 + 3 + q] = d[co][q * 3 + 2];
            }
          }
          asm volatile("bar.sync %0, 128;" ::"r"(1 + grp) : "memory");   // the group's 4 warps
          const int ic = f - 2;
          const int o = r_lo - (NL - 1 - l) + ic;
          const TileGeom &g = p.gg;
          const int64_t gidx = (int64_t)(o - (g.i0 - g.h)) * g.pitch + (cm - (g.j0 - g.hx));
          const bool store = ic >= 0 && ic < nout(l) && col_valid;
#pragma unroll
          for (int co = 0; co < NC; ++co) {
            const float *xb = xch + ((f & 1) * NC + co) * 24;
            if (lane == 0 && quarter > 0) {
#pragma unroll
              for (int q = 0; q < 3; ++q) lft[co][q] = xb[(quarter - 1) * 6 + q];
            }
            if (lane == 31 && quarter < 3) {
#pragma unroll
              for (int q = 0; q < 3; ++q) rgt[co][q] = xb[(quarter + 1) * 6 + 3 + q];
            }
            float c[3];
#pragma unroll
            for (int q = 0; q < 3; ++q) c[q] = (lft[co][q] + d[co][q * 3 + 1]) + rgt[co][q];
            const float row_done = nacc0[co] + c[0];   // output row f-2 (dy = +1 is its last fill)
            nacc0[co] = nacc1[co] + c[1];
            nacc1[co] = c[2];
            if (store) {
              if (FU && fuse) {
                fu_g = row_done + p.bias[l][co];   // handed to the producers below (no G store)
              } else if (!kDdfb || p.mode < 2) {   // DDFB modes exist for 1- and 2-operator launches only
                p.G[(int64_t)co * p.gcs + gidx] = row_done + p.bias[l][co];
              } else if (o >= 0 && o < p.ny && cm >= 0 && cm < p.nx) {
                // DDFB adjoint step (R39): q = proj_[0,1](v - W_k^* u); final: G = v - q (channel co)
                const TileGeom &xg = p.xg;
                const float v = p.xv[(int64_t)co * p.xcs + (int64_t)(o - (xg.i0 - xg.h)) * xg.pitch + (cm - (xg.j0 - xg.hx))];
                const float q = fminf(fmaxf(v - row_done, 0.f), 1.f);
                p.G[(int64_t)co * p.gcs + gidx] = p.mode == 4 ? v - q : q;
              }
            }
          }
          if constexpr (FU) {
            // fused update: the completed G row goes to the G ring the producer warps read
            // (slot = running output-row count mod 8; a slot is re-filled once the 4 producer
            // warps have read it)
            if (fuse && ic >= 0 && ic < nout(l)) {
              const uint32_t Ig = Ocnt(l) + (uint32_t)ic;
              const uint32_t gs = Ig & (kFuG - 1);
              const uint32_t gb = sbase + L.fu_off + kFuFloats * 4u;
              if (Ig >= (uint32_t)kFuG &&
                  !mbar_wait(gb + (kFuG + gs) * 8u, ((Ig / kFuG) - 1) & 1, abort_flag, p.err, 9))
                return false;
              float *const fG = reinterpret_cast<float *>(smem + L.fu_off) + (kFuFloats - kFuG * 128);
              fG[gs * 128 + m] = fu_g;
              __syncwarp();
              if (lane == 0) mbar_arrive(gb + gs * 8u);
            }
          }
          trace_ev(p.trace, trw, 8, s, l);
          return true;
      };
      auto is_netlast = [&](int l) { return l == NL - 1 && last && !is_im2col(l); };
      // output row ic of layer l (completed at step s = f + kLag l, f = ic, or ic + 2 with the
      // dy fold); false on abort
      // DDFB mode 3: u at the pixel of the next output row, loaded while this row is processed
      // (the epilogue of a single im2col layer is otherwise latency-bound on these loads)
      uint32_t upre[kDdfb ? P / 2 : 1];
      int upre_ic = -1;
      auto load_u = [&](int o2, uint32_t *dst) {
        const bool in_a = col_in && o2 >= 0 && o2 < p.ny && o2 >= p.a_i0 && o2 < p.a_i0 + p.a_rows &&
                          cm >= p.a_j0 && cm < p.a_j0 + p.a_cols;
        const int64_t ab = ((int64_t)(o2 - p.a_i0) * p.a_cols + (cm - p.a_j0)) * 8;
#pragma unroll
        for (int gq = 0; gq < G; ++gq) {
          const uint4 t = in_a ? *reinterpret_cast<const uint4 *>(p.ain + (int64_t)gq * p.a_rows * p.a_cols * 8 + ab)
                               : make_uint4(0, 0, 0, 0);
          dst[4 * gq] = t.x; dst[4 * gq + 1] = t.y; dst[4 * gq + 2] = t.z; dst[4 * gq + 3] = t.w;
        }
      };
      auto epi_step = [&](const int l, const int ic) -> bool {
          const bool im2col = is_im2col(l);
          const int s = (im2col ? ic : ic + 2) + kLag * l;
          const uint32_t Ig = Ocnt(l) + (uint32_t)ic;
          if (PNPULA_ONE_COMMIT) {
            // row ic is complete when the MMAs of the fill that finishes it (im2col: fill ic; windowed:
            // fill ic + 2) have completed -- the commit to that fill's input-ring empty barrier.  The
            // slot is re-used (and its barrier completes again) only by fill + ring size, whose MMAs
            // need this row's accumulator slot drained first: the parity cannot alias.
            const uint32_t Fgc = Fcnt(l) + (uint32_t)(im2col ? ic : ic + 2);
            const uint32_t rsc = l == 0 ? Fgc % (uint32_t)kRing : Fgc % (uint32_t)kRingAct;
            const uint32_t phc = l == 0 ? (Fgc / (uint32_t)kRing) & 1u : (Fgc / (uint32_t)kRingAct) & 1u;
            if (!mbar_wait(bar_empty(l, rsc), phc, abort_flag, p.err, 4)) return false;
          } else if (!mbar_wait(bar_tfull(l, Ig & 3), (Ig >> 2) & 1, abort_flag, p.err, 4)) return false;
          trace_ev(p.trace, trw, 6, s, l);
          tc_fence_after();
          const uint32_t taddr = tmem_base + lane_base + (uint32_t)(l * kAcc * P);
          const int o = r_lo - (NL - 1 - l) + ic;      // global output row
          const bool inside = col_in && o >= 0 && o < p.ny;
          if ((l == NL - 1) && last) {
            // network output G (no ReLU), column 0 of the 16-column slot
            float v[1];
            const uint32_t ta = taddr + (Ig & 3) * 16u;
            tmem_load<1>(ta, v);
            tmem_wait_ld();
            tmem_zero<1>(ta);
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(bar_tempty(l, Ig & 3));
            if (col_valid) {
              const TileGeom &g = p.gg;
              p.G[(int64_t)(o - (g.i0 - g.h)) * g.pitch + (cm - (g.j0 - g.hx))] = v[0] + p.bias[l][0];
            }
            return true;
          }
          const uint32_t ta = taddr + (Ig & 3) * (uint32_t)P;
          uint32_t w[P / 2];
          const int m0 = NL == 1 ? p.mode : p.mode0;   // DDFB mode of the im2col layer
          if (kDdfb && is_im2col(l) && (m0 == 1 || m0 == 3)) {
            // DDFB im2col layers (R39, R40): mode 1 u0 = W_K v (no bias, no activation);
            // mode 3 u' = HT(u + gamma_k W_k p) with u read (bf16) at the same pixel
            uint32_t *uin = upre;
            if (m0 == 3 && upre_ic != ic) load_u(o, upre);   // not prefetched (first row of a unit)
            const float ht = p.ht_eps;
#pragma unroll
            for (int h = 0; h < P; h += 16) {
              float v[16];
              tmem_load<16>(ta + h, v);
              tmem_wait_ld();
#pragma unroll
              for (int c = 0; c < 16; c += 2) {
                float a0 = v[c], a1 = v[c + 1];
                if (m0 == 3) {
                  const uint32_t pr = uin[(h + c) / 2];
                  a0 = fminf(fmaxf(__uint_as_float(pr << 16) + a0, -ht), ht);
                  a1 = fminf(fmaxf(__uint_as_float(pr & 0xffff0000u) + a1, -ht), ht);
                }
                w[(h + c) / 2] = pack_bf16(inside ? a0 : 0.f, inside ? a1 : 0.f);
              }
            }
            if (m0 == 3) {
              constexpr int kStep = NL == 2 ? 2 : 1;   // next row this thread's group handles
              if (ic + kStep < nout(l)) { load_u(o + kStep, upre); upre_ic = ic + kStep; }
              else upre_ic = -1;
            }
          } else {
          // 16 channels at a time (tcgen05.ld -> +bias, ReLU -> bf16 pairs): keeps at most 16
          // accumulator values live next to the bias registers
#pragma unroll
          for (int h = 0; h < P; h += 16) {
            float v[16];
            tmem_load<16>(ta + h, v);
            tmem_wait_ld();
#pragma unroll
            for (int c = 0; c < 16; c += 4) {
              const float4 b4 = *reinterpret_cast<const float4 *>(&p.bias[l][h + c]);   // constant cache
              if (PNPULA_EPI_CVT) {
                w[(h + c) / 2] = relu_pack_bf16(v[c] + b4.x, v[c + 1] + b4.y);
                w[(h + c) / 2 + 1] = relu_pack_bf16(v[c + 2] + b4.z, v[c + 3] + b4.w);
              } else {
                w[(h + c) / 2] = pack_bf16(inside ? fmaxf(v[c] + b4.x, 0.f) : 0.f, inside ? fmaxf(v[c + 1] + b4.y, 0.f) : 0.f);
                w[(h + c) / 2 + 1] = pack_bf16(inside ? fmaxf(v[c + 2] + b4.z, 0.f) : 0.f, inside ? fmaxf(v[c + 3] + b4.w, 0.f) : 0.f);
              }
            }
          }
          if (PNPULA_EPI_CVT && __any_sync(0xffffffffu, !inside)) {
#pragma unroll
            for (int k = 0; k < P / 2; ++k) w[k] = inside ? w[k] : 0u;
          }
          }
          if (!im2col) {       // im2col MMAs overwrite (accumulate = 0): no re-zeroing needed
#pragma unroll
            for (int c = 0; c < P; c += 16) tmem_zero<16>(ta + c);
            tmem_wait_st();
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(bar_tempty(l, Ig & 3));
          trace_ev(p.trace, trw, 7, s, l);
          if (l < NL - 1) {
            // next layer's input fill = this layer's output row index ic
            const uint32_t Fg = Fcnt(l + 1) + (uint32_t)ic;
            if (Fg >= kRingAct && !mbar_wait(bar_empty(l + 1, Fg % kRingAct), ((Fg / kRingAct) - 1) & 1, abort_flag, p.err, 5))
              return false;
            trace_ev(p.trace, trw, 9, s, l);
            const uint4 lt = ltab[l + 1];
            uint8_t *slot = smem + lt.x + (Fg % kRingAct) * lt.y + (m + 1) * 16;
#pragma unroll
            for (int gq = 0; gq < G; ++gq)
              *reinterpret_cast<uint4 *>(slot + gq * GS) = make_uint4(w[4 * gq], w[4 * gq + 1], w[4 * gq + 2], w[4 * gq + 3]);
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) mbar_arrive(bar_full(l + 1, Fg % kRingAct));
            if (kDdfb && NL == 2 && p.mode0 != 0 && o >= p.o_i0 && o < p.o_i0 + p.o_rows && cm >= p.o_j0 &&
                cm < p.o_j0 + p.o_cols) {
              // fused DDFB launch: u' also goes to HBM (the next launch's residual); positions two
              // strips share are written twice with identical values
#pragma unroll
              for (int gq = 0; gq < G; ++gq) {
                const int64_t idx = (((int64_t)gq * p.o_rows + (o - p.o_i0)) * p.o_cols + (cm - p.o_j0)) * 8;
                *reinterpret_cast<uint4 *>(p.aout + idx) = make_uint4(w[4 * gq], w[4 * gq + 1], w[4 * gq + 2], w[4 * gq + 3]);
              }
            }
          } else if (col_valid) {
            // chunk output (activations for the next launch), valid columns only
#pragma unroll
            for (int gq = 0; gq < G; ++gq) {
              const int64_t idx = (((int64_t)gq * p.o_rows + (o - p.o_i0)) * p.o_cols + (cm - p.o_j0)) * 8;
              *reinterpret_cast<uint4 *>(p.aout + idx) = make_uint4(w[4 * gq], w[4 * gq + 1], w[4 * gq + 2], w[4 * gq + 3]);
            }
          }
          trace_ev(p.trace, trw, 8, s, l);
          return true;
      };
      if constexpr (NL == 2) {
        // groups 0 / 1: layer 0, rows of their parity; group 2: layer 1
        if (grp < 2) {
          const int no = nout(0);
          for (int ic = grp; ic < no; ic += 2)
            if (!epi_step(0, ic)) break;
        } else if (is_netlast(1)) {
          const int nf = nfill(1);
          for (int f = 0; f < nf; ++f)
            if (!netlast_fill(1, f)) break;
        } else {
          const int no = nout(1);
          for (int ic = 0; ic < no; ++ic)
            if (!epi_step(1, ic)) break;
        }
      } else if constexpr (NL <= kEpiGroups) {
        // one layer per group: walk its output rows (or, folded last layer, its fills) directly
        if (is_netlast(grp)) {
          const int nf = nfill(grp);
          for (int f = 0; f < nf; ++f)
            if (!netlast_fill(grp, f)) break;
        } else {
          const int no = nout(grp);
          for (int ic = 0; ic < no; ++ic)
            if (!epi_step(grp, ic)) break;
        }
      } else {
        bool ok = true;
        for (int s = 0; s < S && ok; ++s) {
#pragma unroll 1
          for (int l = grp; l < NL && ok; l += kEpiGroups) {
            const int f = s - kLag * l;
            if (f < 0 || f >= nfill(l)) continue;
            if (is_netlast(l)) {
              ok = netlast_fill(l, f);
            } else {
              const int ic = is_im2col(l) ? f : f - 2;   // output row completed at this step
              if (ic >= 0 && ic < nout(l)) ok = epi_step(l, ic);
            }
          }
        }
      }
    }
    sumRn += (uint32_t)Rn;
    ++kdone;
    first_unit = false;
  }

  // ---- teardown: make sure every tcgen05 op (and its mbarrier arrivals) has retired
  if (warp >= kMma0 && warp < kEpi0) {
    if (elect_one()) mma_commit(bar_done);       // one arrival per MMA warp
    __syncwarp();
    mbar_wait(bar_done, 0, abort_flag, p.err, 6);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == kMma0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(tmem_cols)
                 : "memory");
  }
}

template <int P, int NL, int NC, bool FU>
cudaError_t launch_pn(const CnnChunkParams &p0, int num_sms, cudaStream_t s) {
  CnnChunkParams p = p0;
  const SmemLayout L = make_layout(P, NL, p.first_is_input, p.last_is_output, NC, FU && p.last_is_output && p.fuse);
  const int Wv = kRowPos - 2 * ((p.last_is_output && NL < 2) ? 2 : NL);   // as in the kernel
  const int strips = (p.ow + Wv - 1) / Wv;
  // rows per unit: minimise (waves) x (rows per unit + pipeline fill) over row-block counts
  int R = p.oh;
  {
    double best = 1e300;
    for (int rb = 1; rb <= (p.oh + 7) / 8; ++rb) {
      const int r = (p.oh + rb - 1) / rb;
      const int nrb = (p.oh + r - 1) / r;
      const int waves = (strips * nrb + num_sms - 1) / num_sms;
      const double cost = (double)waves * (r + 3.0 * NL);
      if (cost < best) { best = cost; R = r; }
    }
  }
  p.strips = strips;
  p.rows_per_unit = R;
  p.units = strips * ((p.oh + R - 1) / R);
  p.rows_per_cta = 0;
  int grid = p.units < num_sms ? p.units : num_sms;
  if (p.contig && NL > 2) {
    // contiguous strip-major ranges of T rows per CTA: a CTA touches <= ceil(T / oh) + 1 strips, each
    // a unit with one pipeline fill; use them when that model beats the row blocks' waves x (R + fill)
    const int64_t total = (int64_t)strips * p.oh;
    const int g2 = (int)std::min<int64_t>(num_sms, total);
    const int64_t T = (total + g2 - 1) / g2;
    const double cost_c = (double)T + 3.0 * NL * (double)((T + p.oh - 1) / p.oh + 1);
    const int nrb = (p.oh + R - 1) / R;
    const double cost_b = (double)((strips * nrb + num_sms - 1) / num_sms) * (R + 3.0 * NL);
    if (cost_c < cost_b || p.contig == 2) {   // 2: forced (tests)
      p.rows_per_cta = (int)T;
      grid = (int)((total + T - 1) / T);
    }
  }
  auto kfn = cnn_chunk_kernel<P, NL, NC, FU>;
  cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block_threads(NL));
  cfg.dynamicSmemBytes = L.total;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = p.pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kfn, p);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// compile-time chain lengths: TMEM (NL * 4 * P <= 512 columns) and 227 KB of shared memory
constexpr int max_nl(int P) { return P == 16 ? 8 : P == 32 ? 4 : 2; }

template <int P, int NL, int NC, bool FU = false>
cudaError_t dispatch_nl(const CnnChunkParams &p, int num_sms, cudaStream_t s) {
  if constexpr (NL > max_nl(P)) {
    return cudaErrorInvalidValue;
  } else {
    if (p.nl == NL) return launch_pn<P, NL, NC, FU>(p, num_sms, s);
    if constexpr (NL < kMaxChunk) return dispatch_nl<P, NL + 1, NC, FU>(p, num_sms, s);
    return cudaErrorInvalidValue;
  }
}

}  // namespace

size_t cnn_chunk_smem_bytes(int P, int nl, int first, int last, int nc, int fuse) {
  // (TMEM: nl * 4 P <= 512 columns holds for every chain max_nl admits)
  if (nl < 1 || nl > kMaxChunk) return SIZE_MAX;
  if (nl > max_nl(P)) return SIZE_MAX;
  if (nc != 1 && (nc != 3 || P < 32)) return SIZE_MAX;   // C = 3: N = 48 columns of the folded last layer
  return make_layout(P, nl, first, last, nc, fuse && last).total;
}

bool cnn_fused_update_supported(int P, int nc, const UpdateParams &u) {
  if (P != 32 || nc != 1 || u.has_tv) return false;
  if (u.op == 1) return true;                                         // mask: no stencil
  return u.op == 0 && u.separable && u.ry == u.rx && (u.ry == 2 || u.ry == 4);   // update_sep_kernel's cases
}

size_t cnn_packed_layer_elems(int cout, int cin) { return packed_layer_elems(cout, cin); }

static uint16_t f32_to_bf16_rne(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) return (uint16_t)(u >> 16);
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

// B-operand image of one layer.  cin = C <= 3 (image): K = 16 or 32 whose k index is the tap
// ci*9 + (u+1)*3+(v+1).  cin == P: per (horizontal tap dx, K step ks) one block
// [2 halves][N3 = 3 Cb rows][8 cin] bf16 whose row n = q*Cb + co holds the weight of
// vertical tap dy = 1 - q (q = 0, 1, 2 <-> dy = +1, 0, -1); Cb = cout.  cout = C <= 3: the
// folded layer (all nine taps of output channel co in rows co*16 + q*3 + dxi).
void cnn_pack_layer(const float *w, int cout, int cin, uint16_t *out) {
  const size_t n = packed_layer_elems(cout, cin);
  memset(out, 0, n * sizeof(uint16_t));
  if (cin <= 3) {
    // im2col layer: K index t = ci * 9 + tap (matching the producer's row), [K/8][N][8]
    const int N = cout;
    for (int co = 0; co < cout; ++co)
      for (int t = 0; t < 9 * cin; ++t) {
        const int g2 = t / 8, k8 = t % 8;
        out[((size_t)g2 * N + co) * 8 + k8] = f32_to_bf16_rne(w[(size_t)co * cin * 9 + t]);
      }
    return;
  }
  const int KS = cin / 16;
  if (cout <= 3) {
    // folded P -> C layer: per K step one block [2 halves][16 C taps][8 cin]; tap row
    // n = co*16 + q*3 + dxi holds W_co(dy = 1 - q, dx = dxi - 1); rows co*16 + 9..15 zero
    const size_t N = 16u * (size_t)cout;
    for (int ks = 0; ks < KS; ++ks)
      for (int co = 0; co < cout; ++co)
        for (int q = 0; q < 3; ++q)
          for (int dxi = 0; dxi < 3; ++dxi)
            for (int c = 0; c < 16; ++c) {
              const int ci = ks * 16 + c, dyi = 2 - q;
              out[(size_t)ks * 16 * N + ((size_t)(c / 8) * N + (size_t)(co * 16 + q * 3 + dxi)) * 8 + (c % 8)] =
                  f32_to_bf16_rne(w[((size_t)co * cin + ci) * 9 + dyi * 3 + dxi]);
            }
    return;
  }
  const int Cb = cout;
  const int N3 = 3 * Cb;
  for (int dxi = 0; dxi < 3; ++dxi)
    for (int ks = 0; ks < KS; ++ks) {
      uint16_t *blk = out + (size_t)(dxi * KS + ks) * 16 * N3;
      for (int q = 0; q < 3; ++q) {
        const int dyi = 2 - q;     // dy = 1 - q  ->  row index dy + 1
        for (int co = 0; co < cout; ++co)
          for (int c = 0; c < 16; ++c) {
            const int ci = ks * 16 + c;
            const int g2 = c / 8, k8 = c % 8;
            const int nrow = q * Cb + co;
            blk[((size_t)g2 * N3 + nrow) * 8 + k8] = f32_to_bf16_rne(w[((size_t)co * cin + ci) * 9 + dyi * 3 + dxi]);
          }
      }
    }
}

cudaError_t launch_cnn_chunk(const CnnChunkParams &p, int num_sms, cudaStream_t s) {
  // image channels matter only to chunks holding the first or the last layer
  const int nc = (p.first_is_input || p.last_is_output) && p.nc > 1 ? p.nc : 1;
  if (nc == 3) {
    switch (p.P) {
      case 32: return dispatch_nl<32, 1, 3>(p, num_sms, s);
      case 64: return dispatch_nl<64, 1, 3>(p, num_sms, s);
      default: return cudaErrorInvalidValue;
    }
  }
  if (nc != 1) return cudaErrorInvalidValue;
  if (p.fuse && p.last_is_output) {   // fused update: compiled for P = 32 (cnn_fused_update_supported)
    if (p.P != 32) return cudaErrorInvalidValue;
    return dispatch_nl<32, 1, 1, true>(p, num_sms, s);
  }
  switch (p.P) {
    case 16: return dispatch_nl<16, 1, 1>(p, num_sms, s);
    case 32: return dispatch_nl<32, 1, 1>(p, num_sms, s);
    case 64: return dispatch_nl<64, 1, 1>(p, num_sms, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace pnpula
