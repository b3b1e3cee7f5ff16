// update_kernels.cu -- K7: the fused, memory-bound part of one PnP-ULA iteration
// (Algorithm 1 lines 6-13) for one tile, plus halo copy / fill /
// moment-finalisation helpers.  sm_100a.
//
// Per owned pixel (i, j) the kernel computes, in this fixed order (fp32):
//   r   = (H1 x - y) on tile (+) r_H (zero outside the image)   P:612 (true conv, zero BC)
//   g   = H1^T r                                                 P:612, P:619 (owner computes its
//                                                                 whole adjoint: no overlap-add)
//   x+  = x - a_g g - a_rho (x - z) - a_d G + a_lam (clamp(x) - x) + a_xi xi
//   z+  = clamp(z - b_rho (z - x+) + b_zeta zeta, z_lo, z_hi)
//   Welford(mean, M2; x+) if t+1 > burn_in
// with a_g = gamma/sigma2, a_rho = gamma/rho, a_d = alpha gamma/eps^2, a_lam = gamma/lambda,
// a_xi = sqrt(2 gamma), b_rho = kappa/rho, b_zeta = sqrt(2 kappa).
// xi, zeta: Philox4x32-10 (key = seed, counter = (j>>2, i, t+1, stream)) + Box-Muller.
//
// The stencil is staged through shared memory: a block owns a 32 x 64 output
// block, loads x on the block (+) 2 r_H once, and runs the separable (4 passes of
// L taps) or general 2-D (2 passes of L^2 taps) forward/adjoint stencil there.
// Every pixel's arithmetic is independent of the block / tile it lands in, so the
// chain is bitwise identical for any tile grid.
#include <cstdint>
#include <cuda.h>   // CUtensorMap (encoded through the runtime's driver entry point: no -lcuda)
#include <cuda_runtime.h>

#include "internal.h"
#include "update_math.cuh"

namespace pnpula {

namespace {

constexpr int TY = 32;            // output rows per block
constexpr int TX = 64;            // output columns per block (16 quads)
constexpr int NTHREADS = 256;

// Philox4x32-10 + Box-Muller noise and the per-pixel tail: update_math.cuh (shared with the update
// fused into the last CNN chunk)
using namespace upd;

// Iteration scalars: by value (direct launches) or from the device IterState (CUDA-graph
// replays; see IterState), read once per thread at kernel entry.
struct IterScalars {
  uint32_t t1;
  int acc;
  float inv_n;
};
template <class P> __device__ __forceinline__ uint32_t iter_t1(const P &p) {
  return p.it ? (uint32_t)p.it->t1 : p.t1;
}
__device__ __forceinline__ IterScalars iter_scalars(const UpdateParams &p) {
  if (p.it) return IterScalars{(uint32_t)p.it->t1, p.it->accumulate, p.it->inv_n};
  return IterScalars{p.t1, p.accumulate, p.inv_n};
}
// next iteration's scalars (same fp64 -> fp32 rounding of 1 / (t+2 - burn_in) as the host's)
__device__ __forceinline__ void it_advance(const UpdateParams &p) {
  if (p.it_next && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
    const long long t1 = p.it->t1 + 1, b = p.it->burn_in;
    const bool acc = t1 > b;
    p.it_next->t1 = t1;
    p.it_next->burn_in = b;
    p.it_next->accumulate = acc;
    p.it_next->inv_n = (float)(1.0 / (acc ? (double)(t1 - b) : 1.0));
  }
}

__device__ __forceinline__ int64_t pidx(const TileGeom &g, int gi, int gj) {
  return (int64_t)(gi - (g.i0 - g.h)) * g.pitch + (gj - (g.j0 - g.hx));
}

// Elementwise tail of K7 for one quad of 4 horizontally adjacent pixels starting at
// global column gj4 (multiple of 4) in row gi; gr[] = H1^T(H1 x - y) (unscaled).
// Per-quad inputs of the elementwise tail (loaded early so their latency overlaps the
// stencil arithmetic and the Philox / Box-Muller work).
struct QuadIn {
  float x[4], G[4], z[4], m[4], s[4];
};

// TVM (as for ula_finish): 2 = a TV launch, whose posterior has no denoiser G, no H2 = I z block
// and no box term (create rejects those with the TV prior): their loads and terms compile out.
// TVM = 2 is instantiated separately so the generic loader's code is unchanged.
template <int TVM>
__device__ __forceinline__ void ula_load_t(const UpdateParams &p, const IterScalars &is, int gi, int gj4, QuadIn &q) {
  const TileGeom &g = p.g;
  const int64_t base = pidx(g, gi, gj4);
  const bool full = gj4 >= g.j0 && gj4 + 4 <= g.j0 + g.tw;
#pragma unroll
  for (int l = 0; l < 4; ++l) { q.G[l] = 0.f; q.z[l] = 0.f; q.m[l] = 0.f; q.s[l] = 0.f; }
  if (full) {
    const float4 a = __ldg(reinterpret_cast<const float4 *>(p.x + base));
    q.x[0] = a.x; q.x[1] = a.y; q.x[2] = a.z; q.x[3] = a.w;
    if (TVM != 2 && p.has_G) {
      const float4 b = __ldg(reinterpret_cast<const float4 *>(p.G + base));
      q.G[0] = b.x; q.G[1] = b.y; q.G[2] = b.z; q.G[3] = b.w;
    }
    if (TVM != 2 && p.has_z) {
      const float4 b = *reinterpret_cast<const float4 *>(p.z + base);
      q.z[0] = b.x; q.z[1] = b.y; q.z[2] = b.z; q.z[3] = b.w;
    }
    if (is.acc) {
      const float4 a2 = *reinterpret_cast<const float4 *>(p.mean + base);
      const float4 b2 = *reinterpret_cast<const float4 *>(p.m2 + base);
      q.m[0] = a2.x; q.m[1] = a2.y; q.m[2] = a2.z; q.m[3] = a2.w;
      q.s[0] = b2.x; q.s[1] = b2.y; q.s[2] = b2.z; q.s[3] = b2.w;
    }
  } else {
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      q.x[l] = p.x[base + l];
      if (TVM != 2 && p.has_G) q.G[l] = p.G[base + l];
      if (TVM != 2 && p.has_z) q.z[l] = p.z[base + l];
      if (is.acc) { q.m[l] = p.mean[base + l]; q.s[l] = p.m2[base + l]; }
    }
  }
}

__device__ __forceinline__ void ula_load(const UpdateParams &p, const IterScalars &is, int gi, int gj4, QuadIn &q) {
  if (p.has_tv) ula_load_t<2>(p, is, gi, gj4, q);
  else ula_load_t<1>(p, is, gi, gj4, q);
}

// D^T (D x - z) at the 4 pixels of a quad (R35, R37):
//   g_v[i-1,j] [i >= 1] - g_v[i,j] [i < ny-1] + g_h[i,j-1] [j >= 1] - g_h[i,j] [j < nx-1],
//   g_v = (x[i+1,j] - x[i,j]) - z_v, g_h = (x[i,j+1] - x[i,j]) - z_h.  Neighbours come from the
// padded x (halo >= 2) and z (valid on tile (+) 1), through L1.
__device__ __forceinline__ void tv_term(const UpdateParams &p, int gi, int gj4, const float *xc, float out[4]) {
  const TileGeom &g = p.g;
  const int64_t base = pidx(g, gi, gj4);   // 16-byte aligned (padded column of gj4 is a multiple of 4)
  const int64_t pitch = g.pitch;
  // the quad's neighbourhood as 6 float4 + 2 scalar loads (x above / below, z_v above / here,
  // z_h here, x left / right and z_h left); out-of-image terms are masked below
  const float4 xu = __ldg(reinterpret_cast<const float4 *>(p.x + base - pitch));
  const float4 xd = __ldg(reinterpret_cast<const float4 *>(p.x + base + pitch));
  const float4 vu = __ldg(reinterpret_cast<const float4 *>(p.zv + base - pitch));
  const float4 vc = __ldg(reinterpret_cast<const float4 *>(p.zv + base));
  const float4 hc = __ldg(reinterpret_cast<const float4 *>(p.zh + base));
  const float xl = __ldg(p.x + base - 1), xr = __ldg(p.x + base + 4), hl = __ldg(p.zh + base - 1);
  const float xup[4] = {xu.x, xu.y, xu.z, xu.w}, xdn[4] = {xd.x, xd.y, xd.z, xd.w};
  const float zvu[4] = {vu.x, vu.y, vu.z, vu.w}, zvc[4] = {vc.x, vc.y, vc.z, vc.w};
  const float zhc[4] = {hc.x, hc.y, hc.z, hc.w};
#pragma unroll
  for (int l = 0; l < 4; ++l) {
    const int gj = gj4 + l;
    if (gj >= p.nx) { out[l] = 0.f; continue; }
    const float xlf = l > 0 ? xc[l - 1] : xl, xrt = l < 3 ? xc[l + 1] : xr, zhl = l > 0 ? zhc[l - 1] : hl;
    float s = 0.f;
    if (gi >= 1) s += (xc[l] - xup[l]) - zvu[l];
    if (gi < p.ny - 1) s -= (xdn[l] - xc[l]) - zvc[l];
    if (gj >= 1) s += (xc[l] - xlf) - zhl;
    if (gj < p.nx - 1) s -= (xrt - xc[l]) - zhc[l];
    out[l] = s;
  }
}

// TVM: 0 = the TV term is compiled out (non-TV launches of the separable kernel), 1 = p.has_tv at run time
template <int TVM = 1>
__device__ __forceinline__ void ula_finish(const UpdateParams &p, const IterScalars &is, int gi, int gj4, const float gr[4],
                                           QuadIn &q, const float *xi_pre = nullptr) {
  const bool has_tv = TVM != 0 && p.has_tv;
  const TileGeom &g = p.g;
  const int64_t base = pidx(g, gi, gj4);
  const bool full = gj4 >= g.j0 && gj4 + 4 <= g.j0 + g.tw;
  const float *xv = q.x, *Gv = q.G, *zv = q.z;
  float *mv = q.m, *sv = q.s;
  float xi[4];
  if (xi_pre) {
#pragma unroll
    for (int l = 0; l < 4; ++l) xi[l] = xi_pre[l];
  } else {
    normals4(p.seed_lo, p.seed_hi, (uint32_t)gj4 >> 2, (uint32_t)gi, is.t1, p.sb + 0u, xi);
  }
  float dtv[4] = {0.f, 0.f, 0.f, 0.f};
  if (has_tv) tv_term(p, gi, gj4, xv, dtv);
  float xn[4];
#pragma unroll
  for (int l = 0; l < 4; ++l) xn[l] = x_step<TVM>(p, has_tv, xv[l], gr[l], Gv[l], zv[l], dtv[l], xi[l]);
  float zn[4];
  if (TVM != 2 && p.has_z) {
    float ze[4];
    normals4(p.seed_lo, p.seed_hi, (uint32_t)gj4 >> 2, (uint32_t)gi, is.t1, p.sb + 1u, ze);
#pragma unroll
    for (int l = 0; l < 4; ++l) zn[l] = z_step(p, zv[l], xn[l], ze[l]);
  }
  if (is.acc) {
#pragma unroll
    for (int l = 0; l < 4; ++l) welford(xn[l], is.inv_n, mv[l], sv[l]);
  }
  if (full) {
    *reinterpret_cast<float4 *>(p.xn + base) = make_float4(xn[0], xn[1], xn[2], xn[3]);
    if (TVM != 2 && p.has_z) *reinterpret_cast<float4 *>(p.z + base) = make_float4(zn[0], zn[1], zn[2], zn[3]);
    if (is.acc) {
      *reinterpret_cast<float4 *>(p.mean + base) = make_float4(mv[0], mv[1], mv[2], mv[3]);
      *reinterpret_cast<float4 *>(p.m2 + base) = make_float4(sv[0], sv[1], sv[2], sv[3]);
    }
  } else {
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      const int gj = gj4 + l;
      if (gj < g.j0 || gj >= g.j0 + g.tw) continue;
      p.xn[base + l] = xn[l];
      if (TVM != 2 && p.has_z) p.z[base + l] = zn[l];
      if (is.acc) { p.mean[base + l] = mv[l]; p.m2[base + l] = sv[l]; }
    }
  }
}

__device__ __forceinline__ void ula_quad(const UpdateParams &p, const IterScalars &is, int gi, int gj4,
                                         const float gr[4]) {
  QuadIn q;
  ula_load(p, is, gi, gj4, q);
  ula_finish(p, is, gi, gj4, gr, q);
}

// ---------------------------------------------------------------- conv K7
// RY/RX >= 0: compile-time radii; -1: runtime (p.ry, p.rx).
template <int RY_, int RX_, bool SEP>
__global__ void __launch_bounds__(NTHREADS)
update_conv_kernel(const __grid_constant__ UpdateParams p) {
  pdl_trigger();
  extern __shared__ float smem[];
  it_advance(p);
  const IterScalars is = iter_scalars(p);
  const int RY = RY_ >= 0 ? RY_ : p.ry;
  const int RX = RX_ >= 0 ? RX_ : p.rx;
  const TileGeom &g = p.g;
  const int bi0 = g.i0 + blockIdx.y * TY;
  const int bj0 = (g.j0 & ~3) + blockIdx.x * TX;
  const int XR = TY + 4 * RY, XC = TX + 4 * RX;     // x region
  const int RR = TY + 2 * RY, RC = TX + 2 * RX;     // residual region
  float *X = smem;                                   // XR x XC
  float *T1 = X + XR * XC;                           // XR x RC   (separable only)
  float *Rr = SEP ? T1 + XR * RC : T1;               // RR x RC
  float *T2 = X;                                     // RR x TX   (reuses X, separable only)
  const int tid = threadIdx.x;

  // phase 0: x on block (+) 2 r_H, zero outside the padded buffer
  for (int e = tid; e < XR * XC; e += NTHREADS) {
    const int a = e / XC, b = e - a * XC;
    const int pr = bi0 - 2 * RY + a - (g.i0 - g.h);
    const int pc = bj0 - 2 * RX + b - (g.j0 - g.hx);
    float v = 0.f;
    if (pr >= 0 && pr < g.ph && pc >= 0 && pc < g.pitch) v = p.x[(int64_t)pr * g.pitch + pc];
    X[e] = v;
  }
  __syncthreads();

  if (SEP) {
    // phase 1: horizontal forward pass  T1[a][b] = sum_q kx[q] X[a][b + RX - q]
    for (int e = tid; e < XR * RC; e += NTHREADS) {
      const int a = e / RC, b = e - a * RC;
      const float *xr = X + a * XC + b + RX;
      float s = 0.f;
#pragma unroll
      for (int q = -RX; q <= RX; ++q) s = fmaf(p.kx[q + RX], xr[-q], s);
      T1[e] = s;
    }
    __syncthreads();
    // phase 2: vertical forward pass minus y -> residual (zero outside the image)
    for (int e = tid; e < RR * RC; e += NTHREADS) {
      const int a = e / RC, b = e - a * RC;
      const int gi = bi0 - RY + a, gj = bj0 - RX + b;
      float s = 0.f;
#pragma unroll
      for (int q = -RY; q <= RY; ++q) s = fmaf(p.ky[q + RY], T1[(a + RY - q) * RC + b], s);
      float r = 0.f;
      if (gi >= 0 && gi < p.ny && gj >= 0 && gj < p.nx) {
        const int pr = gi - (g.i0 - g.h), pc = gj - (g.j0 - g.hx);
        const float yv = (pr >= 0 && pr < g.ph && pc >= 0 && pc < g.pitch) ? p.y[(int64_t)pr * g.pitch + pc] : 0.f;
        r = p.eta * s - yv;
      }
      Rr[e] = r;
    }
    __syncthreads();
    // phase 3: horizontal adjoint pass  T2[a][b] = sum_q kx[q] Rr[a][b + RX + q]
    for (int e = tid; e < RR * TX; e += NTHREADS) {
      const int a = e / TX, b = e - a * TX;
      const float *rr = Rr + a * RC + b + RX;
      float s = 0.f;
#pragma unroll
      for (int q = -RX; q <= RX; ++q) s = fmaf(p.kx[q + RX], rr[q], s);
      T2[e] = s;
    }
    __syncthreads();
  } else {
    // phase 2': residual with the 2-D kernel
    for (int e = tid; e < RR * RC; e += NTHREADS) {
      const int a = e / RC, b = e - a * RC;
      const int gi = bi0 - RY + a, gj = bj0 - RX + b;
      float r = 0.f;
      if (gi >= 0 && gi < p.ny && gj >= 0 && gj < p.nx) {
        float s = 0.f;
        for (int q1 = -RY; q1 <= RY; ++q1) {
          const float *xr = X + (a + RY - q1) * XC + b + RX;
          const float *kr = p.k2d + (q1 + RY) * (2 * RX + 1) + RX;
#pragma unroll 5
          for (int q2 = -RX; q2 <= RX; ++q2) s = fmaf(kr[q2], xr[-q2], s);
        }
        const int pr = gi - (g.i0 - g.h), pc = gj - (g.j0 - g.hx);
        const float yv = (pr >= 0 && pr < g.ph && pc >= 0 && pc < g.pitch) ? p.y[(int64_t)pr * g.pitch + pc] : 0.f;
        r = p.eta * s - yv;
      }
      Rr[e] = r;
    }
    __syncthreads();
  }

  // phase 4: vertical adjoint pass (or 2-D adjoint) + elementwise update, one quad per thread-row
  const int qx = tid & 15;
  for (int rr = tid >> 4; rr < TY; rr += NTHREADS / 16) {
    const int gi = bi0 + rr;
    const int gj4 = bj0 + 4 * qx;
    if (gi >= g.i0 + g.th || gj4 >= g.j0 + g.tw || gj4 + 4 <= g.j0) continue;
    float gr[4];
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      const int b = 4 * qx + l;
      float s = 0.f;
      if (SEP) {
#pragma unroll
        for (int q = -RY; q <= RY; ++q) s = fmaf(p.ky[q + RY], T2[(rr + RY + q) * TX + b], s);
      } else {
        for (int q1 = -RY; q1 <= RY; ++q1) {
          const float *rw = Rr + (rr + RY + q1) * RC + b + RX;
          const float *kr = p.k2d + (q1 + RY) * (2 * RX + 1) + RX;
#pragma unroll 5
          for (int q2 = -RX; q2 <= RX; ++q2) s = fmaf(kr[q2], rw[q2], s);
        }
      }
      gr[l] = s;
    }
    ula_quad(p, is, gi, gj4, gr);
  }
}

// ---------------------------------------------------------------- separable conv K7 (v3)
// Same arithmetic contract as update_conv_kernel<R, R, true>, restructured for throughput:
//  * persistent CTAs (2 per SM) walk the 32 x 64 output blocks of the tile; the x region
//    (block (+) 2R) and the y region (block (+) R rows) of the NEXT block are staged into a
//    second shared-memory buffer by two 2-D TMA tile loads (zero fill outside the padded
//    buffer = the kernel's boundary rule) while the current block computes, so the HBM stream
//    never waits for a stencil pass and no thread spends instructions on staging;
//  * every stencil pass is register-blocked on 4-wide (horizontal) or 4x4 / 2x4 (vertical)
//    output blocks read with 128-bit shared-memory loads.
__device__ __forceinline__ void mbar_init1(uint32_t bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint32_t bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
}
// 2-D TMA tile load (zero fill outside the tensor), completion counted on an mbarrier
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap *map, int c0, int r0, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(r0), "r"(bar)
      : "memory");
}

// PNPULA_UPD_CTAS (kernel experiment): CTAs per SM of update_sep_kernel.  3 keeps the residual
// H x - y in place of the staged y it is formed from (each phase-2 item reads its own 4 y values
// and writes its 4 residuals at the same addresses), so a CTA needs ~70 KB of shared memory.
#ifndef PNPULA_UPD_CTAS
#define PNPULA_UPD_CTAS 2
#endif
constexpr int kUpdCtas = PNPULA_UPD_CTAS;
template <int R>
struct SepGeom {
  static constexpr int XR = TY + 4 * R, XC = TX + 4 * R;   // x region
  static constexpr int RR = TY + 2 * R, RC = TX + 2 * R;   // residual region (y staged RR x XC)
  static constexpr int NW = 2 * R + 4;                     // inputs of a 4-wide output block
  static constexpr bool kRsInY = kUpdCtas >= 3 && R % 4 == 0;   // float4-aligned in-place residual
  static constexpr size_t floats = 2 * (size_t)XR * XC + 2 * (size_t)RR * XC + (size_t)XR * RC +
                                   (kRsInY ? 0 : (size_t)RR * RC);
  static_assert((XR * XC * 4) % 128 == 0 && (RR * XC * 4) % 128 == 0, "TMA destinations 128-B aligned");
  static constexpr size_t bytes = floats * sizeof(float) + 16;   // + 2 mbarriers
};

template <int R, int TVM>
__global__ void __launch_bounds__(NTHREADS, kUpdCtas)
update_sep_kernel(const __grid_constant__ UpdateParams p, const __grid_constant__ CUtensorMap tmx,
                  const __grid_constant__ CUtensorMap tmy, int nbx, int nblk) {
  pdl_trigger();
  using Gm = SepGeom<R>;
  constexpr int XR = Gm::XR, XC = Gm::XC, RR = Gm::RR, RC = Gm::RC, NW = Gm::NW;
  static_assert(RC % 4 == 0 && XC % 4 == 0 && NW % 4 == 0, "R must be even");
  static_assert(RR * TX <= XR * XC, "T2 reuses the x buffer");
  extern __shared__ __align__(128) float sm[];
  it_advance(p);
  const IterScalars is = iter_scalars(p);
  // TMA completion barrier per staging buffer, after the float regions (no static shared
  // memory: the dynamic region then starts 1024-B aligned, as the TMA destinations need)
  uint64_t *const full_bar = reinterpret_cast<uint64_t *>(sm + Gm::floats);
  float *const T1 = sm + 2 * XR * XC + 2 * RR * XC;   // horizontal forward pass, XR x RC
  // residual H x - y, RR x RC (Gm::kRsInY: in place of the staged y of this block, row pitch XC)
  float *const Rs0 = T1 + XR * RC;
  constexpr int RP = Gm::kRsInY ? XC : RC;
  const TileGeom &g = p.g;
  const int tid = threadIdx.x;
  const float *ky = p.ky, *kx = p.kx;   // parameter space: FFMA constant-bank operands
  const int q4 = tid & 15, a2 = tid >> 4;   // phase 4: 16 quads x 16 row pairs

  // stage block blk's x and y regions into buffer buf: one thread, two TMA tile loads
  auto stage = [&](int blk, int buf) {
    const int bi0 = g.i0 + (blk / nbx) * TY;
    const int bj0 = (g.j0 & ~3) + (blk - (blk / nbx) * nbx) * TX;
    const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&full_bar[buf]);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // buffer was read by generic loads
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                 "r"((uint32_t)((XR + RR) * XC * 4))
                 : "memory");
    const int c0 = bj0 - 2 * R - (g.j0 - g.hx);
    tma_load_2d((uint32_t)__cvta_generic_to_shared(sm + buf * XR * XC), &tmx, c0, bi0 - 2 * R - (g.i0 - g.h), bar);
    tma_load_2d((uint32_t)__cvta_generic_to_shared(sm + 2 * XR * XC + buf * RR * XC), &tmy, c0, bi0 - R - (g.i0 - g.h), bar);
  };

  if (tid == 0) {
    mbar_init1((uint32_t)__cvta_generic_to_shared(&full_bar[0]));
    mbar_init1((uint32_t)__cvta_generic_to_shared(&full_bar[1]));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  int blk = blockIdx.x;
  if (tid == 0 && blk < nblk) stage(blk, 0);
  // block coordinates advanced incrementally (one run-time division at entry, not one per block)
  const int gq = (int)gridDim.x / nbx, gr_ = (int)gridDim.x - gq * nbx;
  int bby = blk / nbx, bbx = blk - bby * nbx;
  for (int k = 0; blk < nblk; blk += gridDim.x, ++k) {
    const int buf = k & 1;
    const int nxt = blk + gridDim.x;
    const int bi0 = g.i0 + bby * TY;
    const int bj0 = (g.j0 & ~3) + bbx * TX;
    bbx += gr_;
    bby += gq;
    if (bbx >= nbx) { bbx -= nbx; ++bby; }
    float *const X = sm + buf * XR * XC;
    float *const Yw = sm + 2 * XR * XC + buf * RR * XC;
    const float *const Y = Yw;
    float *const Rs = Gm::kRsInY ? Yw + R : Rs0;
    float *const T2 = X;

    // the update's own operands (x, G, z, mean, M2 of this thread's 2 rows x 1 quad) are
    // requested before the stencil so their latency overlaps it
    const int gj4 = bj0 + 4 * q4;
    bool act[2];
    QuadIn qin[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int gi = bi0 + 2 * a2 + r;
      act[r] = !(gi >= g.i0 + g.th || gj4 >= g.j0 + g.tw || gj4 + 4 <= g.j0);
      if (act[r]) ula_load_t<TVM == 2 ? 2 : 1>(p, is, gi, gj4, qin[r]);
    }
    mbar_wait_parity((uint32_t)__cvta_generic_to_shared(&full_bar[buf]), (uint32_t)(k >> 1) & 1u);

    // phase 1: T1[a][b] = sum_q kx[q+R] X[a][b+R-q]   (4 outputs per item)
    for (int e = tid; e < XR * (RC / 4); e += NTHREADS) {
      const int a = e / (RC / 4), k4 = e - a * (RC / 4);
      float xs[NW];
#pragma unroll
      for (int i = 0; i < NW; i += 4) {
        const float4 t = *reinterpret_cast<const float4 *>(X + a * XC + 4 * k4 + i);
        xs[i] = t.x; xs[i + 1] = t.y; xs[i + 2] = t.z; xs[i + 3] = t.w;
      }
      float o[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float s = 0.f;
#pragma unroll
        for (int q = -R; q <= R; ++q) s = fmaf(kx[q + R], xs[j + R - q], s);
        o[j] = s;
      }
      *reinterpret_cast<float4 *>(T1 + a * RC + 4 * k4) = make_float4(o[0], o[1], o[2], o[3]);
    }
    __syncthreads();
    // buffer buf ^ 1 (x / T2 and y of the previous block) is free once every thread has passed
    // this barrier, so the next block's prefetch is issued here (no end-of-block barrier)
    if (tid == 0 && nxt < nblk) stage(nxt, buf ^ 1);
    // phase 2: Rs[a][b] = sum_p ky[p+R] T1[a+R-p][b] - y, zero outside the image (4x4 per item)
    const bool rs_inside = bi0 - R >= 0 && bi0 - R + RR <= p.ny && bj0 - R >= 0 && bj0 - R + RC <= p.nx;
    for (int e = tid; e < (RR / 4) * (RC / 4); e += NTHREADS) {
      const int a4 = e / (RC / 4), k4 = e - a4 * (RC / 4);
      float col[NW][4];
#pragma unroll
      for (int i = 0; i < NW; ++i) {
        const float4 t = *reinterpret_cast<const float4 *>(T1 + (4 * a4 + i) * RC + 4 * k4);
        col[i][0] = t.x; col[i][1] = t.y; col[i][2] = t.z; col[i][3] = t.w;
      }
      const int gj = bj0 - R + 4 * k4;
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int a = 4 * a4 + r;
        const int gi = bi0 - R + a;
        float o[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float s = 0.f;
#pragma unroll
          for (int q = -R; q <= R; ++q) s = fmaf(ky[q + R], col[r + R - q][j], s);
          o[j] = s;
        }
        float yv[4];
        const float *yr = Y + a * XC + R + 4 * k4;   // y column gj + j  <->  staged column R + 4 k4 + j
        if (R % 4 == 0) {
          const float4 t = *reinterpret_cast<const float4 *>(yr);
          yv[0] = t.x; yv[1] = t.y; yv[2] = t.z; yv[3] = t.w;
        } else {
          const float2 t0 = *reinterpret_cast<const float2 *>(yr), t1 = *reinterpret_cast<const float2 *>(yr + 2);
          yv[0] = t0.x; yv[1] = t0.y; yv[2] = t1.x; yv[3] = t1.y;
        }
        if (rs_inside) {   // the block's whole residual region lies in the image: no per-element test
#pragma unroll
          for (int j = 0; j < 4; ++j) o[j] = p.eta * o[j] - yv[j];
        } else {
          const bool rin = gi >= 0 && gi < p.ny;
#pragma unroll
          for (int j = 0; j < 4; ++j) o[j] = (rin && gj + j >= 0 && gj + j < p.nx) ? p.eta * o[j] - yv[j] : 0.f;
        }
        *reinterpret_cast<float4 *>(Rs + a * RP + 4 * k4) = make_float4(o[0], o[1], o[2], o[3]);
      }
    }
    __syncthreads();
    // phase 3: T2[a][b] = sum_q kx[q+R] Rs[a][b+R+q]   (4 outputs per item)
    for (int e = tid; e < RR * (TX / 4); e += NTHREADS) {
      const int a = e / (TX / 4), k4 = e - a * (TX / 4);
      float rs[NW];
#pragma unroll
      for (int i = 0; i < NW; i += 4) {
        const float4 t = *reinterpret_cast<const float4 *>(Rs + a * RP + 4 * k4 + i);
        rs[i] = t.x; rs[i + 1] = t.y; rs[i + 2] = t.z; rs[i + 3] = t.w;
      }
      float o[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float s = 0.f;
#pragma unroll
        for (int q = -R; q <= R; ++q) s = fmaf(kx[q + R], rs[j + R + q], s);
        o[j] = s;
      }
      *reinterpret_cast<float4 *>(T2 + a * TX + 4 * k4) = make_float4(o[0], o[1], o[2], o[3]);
    }
    __syncthreads();
    // phase 4: g = sum_p ky[p+R] T2[a+R+p][b] for 2 rows x 1 quad per thread, then the update
    {
      float col[2 * R + 2][4];
#pragma unroll
      for (int i = 0; i < 2 * R + 2; ++i) {
        const float4 t = *reinterpret_cast<const float4 *>(T2 + (2 * a2 + i) * TX + 4 * q4);
        col[i][0] = t.x; col[i][1] = t.y; col[i][2] = t.z; col[i][3] = t.w;
      }
      float xi2[2][4];   // xi of both rows (rows outside the tile: computed, unused)
      normals4x2(p.seed_lo, p.seed_hi, (uint32_t)gj4 >> 2, (uint32_t)(bi0 + 2 * a2), is.t1, p.sb + 0u, xi2);
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        if (!act[r]) continue;
        float gr[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float s = 0.f;
#pragma unroll
          for (int pp = -R; pp <= R; ++pp) s = fmaf(ky[pp + R], col[r + R + pp][j], s);
          gr[j] = s;
        }
        ula_finish<TVM>(p, is, bi0 + 2 * a2 + r, gj4, gr, qin[r], xi2[r]);
      }
    }
  }
}

// ---------------------------------------------------------------- Poisson z1 block
// One thread per column quad of tile (+) r_H (quads aligned to global column multiples of 4,
// so the Philox call is shared exactly as in the x-update), 2-D stencil of x+ read through L1.
// Pixels outside tile (+) r_H or the image are skipped (z1 stays 0 outside the image).
__global__ void __launch_bounds__(NTHREADS) z1_update_kernel(const __grid_constant__ Z1Params p) {
  pdl_trigger();
  const uint32_t t1 = iter_t1(p);
  const TileGeom &g = p.g;
  const int ry = p.ry, rx = p.rx, kw = 2 * rx + 1;
  const int r0 = max(g.i0 - ry, 0), r1 = min(g.i0 + g.th + ry, p.ny);
  const int c0 = max(g.j0 - rx, 0), c1 = min(g.j0 + g.tw + rx, p.nx);
  const int q0 = c0 >> 2, nq = ((c1 + 3) >> 2) - q0;
  const uint32_t total = (uint32_t)nq * (uint32_t)(r1 - r0);   // < 2^31 quads per tile
  for (uint32_t e = blockIdx.x * NTHREADS + threadIdx.x; e < total; e += gridDim.x * NTHREADS) {
    const uint32_t qr = e / (uint32_t)nq;
    const int gi = r0 + (int)qr;
    const int gj4 = 4 * (q0 + (int)(e - qr * (uint32_t)nq));
    float ze[4];
    normals4(p.seed_lo, p.seed_hi, (uint32_t)gj4 >> 2, (uint32_t)gi, t1, p.sb + 2u, ze);
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      const int gj = gj4 + l;
      if (gj < c0 || gj >= c1) continue;
      float s = 0.f;   // (H x+)[gi][gj] = sum_{a,b} k[a][b] x+[gi - (a - ry)][gj - (b - rx)]
      for (int a = 0; a < 2 * ry + 1; ++a) {
        const float *xr = p.x + pidx(g, gi - (a - ry), gj + rx);
        const float *kr = p.k2d + a * kw;
        for (int b = 0; b < kw; ++b) s = fmaf(kr[b], __ldg(xr - b), s);
      }
      const int64_t n = pidx(g, gi, gj);
      const float z = p.z1[n];
      const float v = z - p.b1 * (z - p.eta * s) + p.s1 * ze[l];
      // prox of kappa1 KL(y || .): the non-negative root of u^2 - (v - kappa1) u - kappa1 y = 0 (R31)
      const float a = v - p.kappa1;
      p.z1[n] = 0.5f * (a + sqrtf(fmaf(a, a, 4.0f * p.kappa1 * __ldg(p.y + n))));
    }
  }
}

// Separable fast path of the z1 block: a CTA owns a 32 x 64 block of tile (+) r_H (columns
// quad-aligned), stages x+ on block (+) R with one 2-D TMA tile load (zero fill outside the
// padded buffer), runs the horizontal then the vertical pass of H = ky (x) kx in shared memory,
// and updates 2 rows x 1 quad per thread (one Philox call per quad, stream 2).
template <int R>
__global__ void __launch_bounds__(NTHREADS) z1_sep_kernel(const __grid_constant__ Z1Params p,
                                                        const __grid_constant__ CUtensorMap tmx, int r0, int q0,
                                                        int nbx) {
  pdl_trigger();
  const uint32_t t1 = iter_t1(p);
  // the staged columns start 16-B aligned (XL = R rounded up to 4): TMA tile loads need a
  // 16-B aligned inner start coordinate
  constexpr int XL = (R + 3) / 4 * 4;
  constexpr int XR = TY + 2 * R, XC = TX + 2 * XL;
  static_assert((XC * 4) % 16 == 0, "TMA row bytes");
  __shared__ __align__(128) float X[XR * XC];
  __shared__ __align__(16) float T[XR * TX];
  __shared__ __align__(8) uint64_t bar;
  const float *kys = p.ky, *kxs = p.kx;   // parameter space
  const TileGeom &g = p.g;
  const int tid = threadIdx.x;
  const int bi0 = r0 + (int)(blockIdx.x / nbx) * TY;
  const int bj0 = 4 * q0 + (int)(blockIdx.x % nbx) * TX;
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
  if (tid == 0) {
    mbar_init1(b);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(b),
                 "r"((uint32_t)(XR * XC * 4))
                 : "memory");
    tma_load_2d((uint32_t)__cvta_generic_to_shared(X), &tmx, bj0 - XL - (g.j0 - g.hx), bi0 - R - (g.i0 - g.h), b);
  }
  // this thread's outputs: 2 rows x 1 quad; z1 and y are requested now so their latency overlaps
  // the TMA wait and the horizontal pass (float4 when the quad lies inside tile (+) r_H)
  const int q = tid & 15, a2 = tid >> 4;
  const int gj4 = bj0 + 4 * q;
  const int rlo = g.i0 - p.ry < 0 ? 0 : g.i0 - p.ry, rhi = g.i0 + g.th + p.ry > p.ny ? p.ny : g.i0 + g.th + p.ry;
  const int clo = g.j0 - p.rx < 0 ? 0 : g.j0 - p.rx, chi = g.j0 + g.tw + p.rx > p.nx ? p.nx : g.j0 + g.tw + p.rx;
  bool act[2], full[2];
  float zr[2][4], yr[2][4];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int gi = bi0 + 2 * a2 + r;
    act[r] = !(gi < rlo || gi >= rhi || gj4 >= chi || gj4 + 4 <= clo);
    full[r] = act[r] && gj4 >= clo && gj4 + 4 <= chi;
    const int64_t n0 = pidx(g, gi, gj4);   // 16-byte aligned
    if (full[r]) {
      const float4 zv = *reinterpret_cast<const float4 *>(p.z1 + n0);
      const float4 yv = __ldg(reinterpret_cast<const float4 *>(p.y + n0));
      zr[r][0] = zv.x; zr[r][1] = zv.y; zr[r][2] = zv.z; zr[r][3] = zv.w;
      yr[r][0] = yv.x; yr[r][1] = yv.y; yr[r][2] = yv.z; yr[r][3] = yv.w;
    } else {
#pragma unroll
      for (int l = 0; l < 4; ++l) {
        const bool in = act[r] && gj4 + l >= clo && gj4 + l < chi;
        zr[r][l] = in ? p.z1[n0 + l] : 0.f;
        yr[r][l] = in ? __ldg(p.y + n0 + l) : 0.f;
      }
    }
  }
  __syncthreads();
  mbar_wait_parity(b, 0);
  // horizontal: T[a][c] = sum_q kx[q+R] X[a][c + XL - q]   (x+ column bj0 + c - q)
  for (int e = tid; e < XR * (TX / 4); e += NTHREADS) {
    const int a = e / (TX / 4), c4 = 4 * (e - a * (TX / 4));
    float o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float s = 0.f;
#pragma unroll
      for (int q2 = -R; q2 <= R; ++q2) s = fmaf(kxs[q2 + R], X[a * XC + c4 + j + XL - q2], s);
      o[j] = s;
    }
    *reinterpret_cast<float4 *>(T + a * TX + 4 * (e - a * (TX / 4))) = make_float4(o[0], o[1], o[2], o[3]);
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    if (!act[r]) continue;
    const int a = 2 * a2 + r, gi = bi0 + a;
    float ze[4];
    normals4(p.seed_lo, p.seed_hi, (uint32_t)gj4 >> 2, (uint32_t)gi, t1, p.sb + 2u, ze);
    float out[4];
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      float s = 0.f;   // vertical: sum_p ky[p+R] T[a + R - p][c]
#pragma unroll
      for (int pp = -R; pp <= R; ++pp) s = fmaf(kys[pp + R], T[(a + R - pp) * TX + 4 * q + l], s);
      const float z = zr[r][l];
      const float v = z - p.b1 * (z - p.eta * s) + p.s1 * ze[l];
      const float av = v - p.kappa1;
      const float r2 = fmaf(av, av, 4.0f * p.kappa1 * yr[r][l]);   // KL prox (R31): (av + sqrt(r2)) / 2
      out[l] = 0.5f * (av + (r2 > 0.f ? r2 * rsqrtf(r2) : 0.f));
    }
    const int64_t n0 = pidx(g, gi, gj4);
    if (full[r]) {
      *reinterpret_cast<float4 *>(p.z1 + n0) = make_float4(out[0], out[1], out[2], out[3]);
    } else {
#pragma unroll
      for (int l = 0; l < 4; ++l)
        if (gj4 + l >= clo && gj4 + l < chi) p.z1[n0 + l] = out[l];
    }
  }
}

// ---------------------------------------------------------------- TV z block (R37, R38)
// One thread per column quad of tile (+) 1 (global quads: the Philox calls match the oracle's
// (stream, pixel) counters); D x+ from the padded x+ (halo >= 2), block soft threshold per pixel.
__global__ void __launch_bounds__(NTHREADS) tv_z_kernel(const __grid_constant__ TvZParams p) {
  pdl_trigger();
  const uint32_t t1 = iter_t1(p);
  const TileGeom &g = p.g;
  const int r0 = max(g.i0 - 1, 0), r1 = min(g.i0 + g.th + 1, p.ny);
  const int c0 = max(g.j0 - 1, 0), c1 = min(g.j0 + g.tw + 1, p.nx);
  const int q0 = c0 >> 2, nq = ((c1 + 3) >> 2) - q0;
  const uint32_t total = (uint32_t)nq * (uint32_t)(r1 - r0);   // < 2^31 quads per tile
  for (uint32_t e = blockIdx.x * NTHREADS + threadIdx.x; e < total; e += gridDim.x * NTHREADS) {
    const uint32_t qr = e / (uint32_t)nq;
    const int gi = r0 + (int)qr;
    const int gj4 = 4 * (q0 + (int)(e - qr * (uint32_t)nq));
    float zev[4], zeh[4];
    normals4(p.seed_lo, p.seed_hi, (uint32_t)gj4 >> 2, (uint32_t)gi, t1, p.sb + 1u, zev);
    normals4(p.seed_lo, p.seed_hi, (uint32_t)gj4 >> 2, (uint32_t)gi, t1, p.sb + 3u, zeh);
    const int64_t n0 = pidx(g, gi, gj4);   // 16-byte aligned
    if (gj4 >= c0 && gj4 + 4 <= c1) {
      // whole quad inside: 4 float4 loads + 1 scalar (x right of the quad), 2 float4 stores
      const float4 x4 = __ldg(reinterpret_cast<const float4 *>(p.x + n0));
      const float4 d4 = __ldg(reinterpret_cast<const float4 *>(p.x + n0 + g.pitch));
      const float xr = __ldg(p.x + n0 + 4);
      const float4 v4 = *reinterpret_cast<const float4 *>(p.zv + n0);
      const float4 h4 = *reinterpret_cast<const float4 *>(p.zh + n0);
      const float xc[5] = {x4.x, x4.y, x4.z, x4.w, xr}, xd[4] = {d4.x, d4.y, d4.z, d4.w};
      const float zv[4] = {v4.x, v4.y, v4.z, v4.w}, zh[4] = {h4.x, h4.y, h4.z, h4.w};
      float ov[4], oh[4];
#pragma unroll
      for (int l = 0; l < 4; ++l) {
        const float dv = gi < p.ny - 1 ? xd[l] - xc[l] : 0.f;
        const float dh = gj4 + l < p.nx - 1 ? xc[l + 1] - xc[l] : 0.f;
        const float vv = zv[l] - p.b * (zv[l] - dv) + p.s * zev[l];
        const float vh = zh[l] - p.b * (zh[l] - dh) + p.s * zeh[l];
        const float n2 = fmaf(vv, vv, vh * vh);   // shrink: 1 - tau / ||(vv, vh)|| if the norm exceeds tau
        const float sc = n2 > p.tau * p.tau ? 1.f - p.tau * rsqrtf(n2) : 0.f;
        ov[l] = vv * sc;
        oh[l] = vh * sc;
      }
      *reinterpret_cast<float4 *>(p.zv + n0) = make_float4(ov[0], ov[1], ov[2], ov[3]);
      *reinterpret_cast<float4 *>(p.zh + n0) = make_float4(oh[0], oh[1], oh[2], oh[3]);
      continue;
    }
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      const int gj = gj4 + l;
      if (gj < c0 || gj >= c1) continue;
      const int64_t n = n0 + l;
      const float xc = __ldg(p.x + n);
      const float dv = gi < p.ny - 1 ? __ldg(p.x + n + g.pitch) - xc : 0.f;
      const float dh = gj < p.nx - 1 ? __ldg(p.x + n + 1) - xc : 0.f;
      const float zv = p.zv[n], zh = p.zh[n];
      const float vv = zv - p.b * (zv - dv) + p.s * zev[l];
      const float vh = zh - p.b * (zh - dh) + p.s * zeh[l];
      const float n2 = fmaf(vv, vv, vh * vh);
      const float sc = n2 > p.tau * p.tau ? 1.f - p.tau * rsqrtf(n2) : 0.f;
      p.zv[n] = vv * sc;
      p.zh[n] = vh * sc;
    }
  }
}

// ---------------------------------------------------------------- power iteration for ||H||^2
// (step sizes of P:774 / P:782 need ||H||^2).  v: padded with a valid halo
// (>= 2 r_H).  Pass 1: w = H v on tile (+) r_H, zero outside the image.  Pass 2: u = H^T w on the
// tile, written in place of v's interior is NOT allowed (v is read by neighbours' pass 1), so into
// the padded u buffer; per-block partial sums of u^2 and u.v go to acc[0], acc[1] (fp64 atomics).
__global__ void __launch_bounds__(NTHREADS) opnorm_fwd_kernel(const __grid_constant__ OpNormParams p) {
  const TileGeom &g = p.g;
  const int ry = p.ry, rx = p.rx, kw = 2 * rx + 1;
  const int r0 = max(g.i0 - ry, 0), r1 = min(g.i0 + g.th + ry, p.ny);
  const int c0 = max(g.j0 - rx, 0), c1 = min(g.j0 + g.tw + rx, p.nx);
  const int w = c1 - c0;
  const int64_t total = (int64_t)w * (r1 - r0);
  for (int64_t e = (int64_t)blockIdx.x * NTHREADS + threadIdx.x; e < total; e += (int64_t)gridDim.x * NTHREADS) {
    const int gi = r0 + (int)(e / w), gj = c0 + (int)(e % w);
    float s = 0.f;
    for (int a = 0; a < 2 * ry + 1; ++a) {
      const float *vr = p.v + pidx(g, gi - (a - ry), gj + rx);
      const float *kr = p.k2d + a * kw;
      for (int b = 0; b < kw; ++b) s = fmaf(kr[b], __ldg(vr - b), s);
    }
    p.w[pidx(g, gi, gj)] = s;
  }
}

__global__ void __launch_bounds__(NTHREADS) opnorm_adj_kernel(const __grid_constant__ OpNormParams p) {
  const TileGeom &g = p.g;
  const int ry = p.ry, rx = p.rx, kw = 2 * rx + 1;
  const int64_t total = (int64_t)g.th * g.tw;
  double su = 0.0, suv = 0.0;
  for (int64_t e = (int64_t)blockIdx.x * NTHREADS + threadIdx.x; e < total; e += (int64_t)gridDim.x * NTHREADS) {
    const int gi = g.i0 + (int)(e / g.tw), gj = g.j0 + (int)(e % g.tw);
    float s = 0.f;   // (H^T w)[i][j] = sum_{a,b} k[a][b] w[i + (a - ry)][j + (b - rx)], w = 0 outside the image
    for (int a = 0; a < 2 * ry + 1; ++a) {
      const int ii = gi + (a - ry);
      if (ii < 0 || ii >= p.ny) continue;
      for (int b = 0; b < kw; ++b) {
        const int jj = gj + (b - rx);
        if (jj < 0 || jj >= p.nx) continue;
        s = fmaf(p.k2d[a * kw + b], p.w[pidx(g, ii, jj)], s);
      }
    }
    const int64_t n = pidx(g, gi, gj);
    p.u[n] = s;
    su += (double)s * s;
    suv += (double)s * p.v[n];
  }
  // block reduction then one fp64 atomic per block and quantity
  __shared__ double red[2][NTHREADS / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    su += __shfl_down_sync(0xffffffffu, su, o);
    suv += __shfl_down_sync(0xffffffffu, suv, o);
  }
  if ((threadIdx.x & 31) == 0) { red[0][threadIdx.x >> 5] = su; red[1][threadIdx.x >> 5] = suv; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int i = 0; i < NTHREADS / 32; ++i) { a += red[0][i]; b += red[1][i]; }
    atomicAdd(p.acc, a);
    atomicAdd(p.acc + 1, b);
  }
}

// v <- u * scale on the tile interior (the halo is refreshed by the exchange)
__global__ void opnorm_scale_kernel(const __grid_constant__ OpNormParams p, const double *scale) {
  const TileGeom &g = p.g;
  const float sc = (float)*scale;
  const int64_t total = (int64_t)g.th * g.tw;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int gi = g.i0 + (int)(e / g.tw), gj = g.j0 + (int)(e % g.tw);
    const int64_t n = pidx(g, gi, gj);
    p.v[n] = p.u[n] * sc;
  }
}

// deterministic start vector: Philox normals (stream 7, iteration 0) on the interior
__global__ void opnorm_init_kernel(const __grid_constant__ OpNormParams p) {
  const TileGeom &g = p.g;
  const int64_t total = (int64_t)g.th * g.tw;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int gi = g.i0 + (int)(e / g.tw), gj = g.j0 + (int)(e % g.tw);
    float z[4];
    normals4(0x2511u, 0x870u, (uint32_t)gj >> 2, (uint32_t)gi, 0u, 7u, z);
    p.v[pidx(g, gi, gj)] = z[gj & 3];
  }
}

// ---------------------------------------------------------------- mask K7 (no stencil)
__global__ void __launch_bounds__(NTHREADS) update_mask_kernel(const __grid_constant__ UpdateParams p) {
  pdl_trigger();
  it_advance(p);
  const IterScalars is = iter_scalars(p);
  const TileGeom &g = p.g;
  const int nq = ((g.j0 + g.tw + 3) >> 2) - (g.j0 >> 2);
  const uint32_t total = (uint32_t)nq * (uint32_t)g.th;   // < 2^31 quads per tile
  for (uint32_t e = blockIdx.x * NTHREADS + threadIdx.x; e < total; e += gridDim.x * NTHREADS) {
    const int rr = (int)(e / (uint32_t)nq), q = (int)(e - (uint32_t)rr * (uint32_t)nq);
    const int gi = g.i0 + rr, gj4 = (g.j0 & ~3) + 4 * q;
    const int64_t base = pidx(g, gi, gj4);
    float gr[4];
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      const float m = p.mask[base + l] ? 1.f : 0.f;
      gr[l] = m * (m * p.x[base + l] - p.y[base + l]);
    }
    ula_quad(p, is, gi, gj4, gr);
  }
}

__global__ void copy_jobs_kernel(const CopyJob *__restrict__ jobs) {
  pdl_trigger();
  const CopyJob j = jobs[blockIdx.y];
  const int64_t n = (int64_t)j.rows * j.cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e / j.cols), c = (int)(e - (int64_t)r * j.cols);
    j.dst[(int64_t)r * j.dst_pitch + c] = j.src[(int64_t)r * j.src_pitch + c];
  }
}

__global__ void fill_kernel(float *p, float v, size_t n) {
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x) p[e] = v;
}

__global__ void finalize_kernel(const FinalizeParams p) {
  const TileGeom &g = p.g;
  const int64_t n = (int64_t)g.th * g.tw;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e / g.tw), c = (int)(e - (int64_t)r * g.tw);
    const int64_t s = (int64_t)(r + g.h) * g.pitch + (c + g.hx);
    if (p.out_mean) p.out_mean[e] = p.mean[s];
    if (p.out_var) p.out_var[e] = p.m2[s] * p.inv_nm1;
  }
}

template <int RY, int RX, bool SEP>
cudaError_t launch_conv(const UpdateParams &p, cudaStream_t s) {
  const int ry = RY >= 0 ? RY : p.ry, rx = RX >= 0 ? RX : p.rx;
  const int XR = TY + 4 * ry, XC = TX + 4 * rx, RR = TY + 2 * ry, RC = TX + 2 * rx;
  size_t smem = (size_t)XR * XC + (SEP ? (size_t)XR * RC : 0) + (size_t)RR * RC;
  if (SEP && (size_t)RR * TX > (size_t)XR * XC) return cudaErrorInvalidValue;
  smem *= sizeof(float);
  auto kfn = update_conv_kernel<RY, RX, SEP>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const int cols = p.g.j0 + p.g.tw - (p.g.j0 & ~3);
  dim3 grid((cols + TX - 1) / TX, (p.g.th + TY - 1) / TY);
  kfn<<<grid, NTHREADS, smem, s>>>(p);
  return cudaGetLastError();
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (the library links cudart only)
using EncodeTiledFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                   const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_tiled_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void *f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(f);
  }
  return fn;
}

// 2-D fp32 map over a padded tile buffer (ph rows x pitch floats), box = box_c x box_r,
// out-of-bounds elements read as zero
bool encode_padded_2d(CUtensorMap *m, const float *base, const TileGeom &g, int box_c, int box_r) {
  EncodeTiledFn fn = encode_tiled_fn();
  if (!fn) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)g.pitch, (cuuint64_t)g.ph};
  const cuuint64_t strides[1] = {(cuuint64_t)g.pitch * sizeof(float)};
  const cuuint32_t box[2] = {(cuuint32_t)box_c, (cuuint32_t)box_r};
  const cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

cudaError_t launch_update(const UpdateParams &p, cudaStream_t s) {
  if (p.op == 1) {
    const int nq = ((p.g.j0 + p.g.tw + 3) >> 2) - (p.g.j0 >> 2);
    const int64_t total = (int64_t)nq * p.g.th;
    int blocks = (int)((total + NTHREADS - 1) / NTHREADS);
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (blocks < 1) blocks = 1;
    update_mask_kernel<<<blocks, NTHREADS, 0, s>>>(p);
    return cudaGetLastError();
  }
  if (p.separable) {
    if (p.ry == p.rx && (p.ry == 4 || p.ry == 2)) {
      const int cols = p.g.j0 + p.g.tw - (p.g.j0 & ~3);
      const int nbx = (cols + TX - 1) / TX, nby = (p.g.th + TY - 1) / TY;
      const int nblk = nbx * nby;
      // opt in to > 48 KB of shared memory (a per-device attribute: set on every launch)
      int dev = 0, num_sms = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
      const int R = p.ry;
      const size_t smem = R == 4 ? SepGeom<4>::bytes : SepGeom<2>::bytes;
      auto kfn = R == 4 ? (p.has_tv ? update_sep_kernel<4, 2> : update_sep_kernel<4, 0>)
                        : (p.has_tv ? update_sep_kernel<2, 2> : update_sep_kernel<2, 0>);
      cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      // TMA maps of the padded x and y buffers (ph x pitch fp32), boxes = the staged regions
      CUtensorMap tmx, tmy;
      const int XC = TX + 4 * R;
      if (!encode_padded_2d(&tmx, p.x, p.g, XC, TY + 4 * R) || !encode_padded_2d(&tmy, p.y, p.g, XC, TY + 2 * R))
        return cudaErrorInvalidValue;
      const int grid = nblk < kUpdCtas * num_sms ? nblk : kUpdCtas * num_sms;
      kfn<<<grid, NTHREADS, smem, s>>>(p, tmx, tmy, nbx, nblk);
      return cudaGetLastError();
    }
    return launch_conv<-1, -1, true>(p, s);
  }
  if (p.ry == 2 && p.rx == 2) return launch_conv<2, 2, false>(p, s);
  if (p.ry == 4 && p.rx == 4) return launch_conv<4, 4, false>(p, s);
  return launch_conv<-1, -1, false>(p, s);
}

cudaError_t launch_z1_update(const Z1Params &p, cudaStream_t s) {
  const int r0 = p.g.i0 - p.ry < 0 ? 0 : p.g.i0 - p.ry;
  const int r1 = p.g.i0 + p.g.th + p.ry > p.ny ? p.ny : p.g.i0 + p.g.th + p.ry;
  const int c0 = p.g.j0 - p.rx < 0 ? 0 : p.g.j0 - p.rx;
  const int c1 = p.g.j0 + p.g.tw + p.rx > p.nx ? p.nx : p.g.j0 + p.g.tw + p.rx;
  if (p.separable && p.ry == p.rx && (p.ry == 4 || p.ry == 2)) {
    const int R = p.ry, q0 = c0 >> 2;
    const int nbx = (((c1 + 3) >> 2) - q0 + 15) / 16, nby = (r1 - r0 + TY - 1) / TY;
    CUtensorMap tmx;
    if (!encode_padded_2d(&tmx, p.x, p.g, TX + 2 * ((R + 3) / 4 * 4), TY + 2 * R)) return cudaErrorInvalidValue;
    if (R == 4) z1_sep_kernel<4><<<nbx * nby, NTHREADS, 0, s>>>(p, tmx, r0, q0, nbx);
    else z1_sep_kernel<2><<<nbx * nby, NTHREADS, 0, s>>>(p, tmx, r0, q0, nbx);
    return cudaGetLastError();
  }
  const int64_t total = (int64_t)(((c1 + 3) >> 2) - (c0 >> 2)) * (r1 - r0);
  int64_t blocks = (total + NTHREADS - 1) / NTHREADS;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  z1_update_kernel<<<(unsigned)blocks, NTHREADS, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_tv_z_update(const TvZParams &p, cudaStream_t s) {
  const int r0 = p.g.i0 - 1 < 0 ? 0 : p.g.i0 - 1;
  const int r1 = p.g.i0 + p.g.th + 1 > p.ny ? p.ny : p.g.i0 + p.g.th + 1;
  const int c0 = p.g.j0 - 1 < 0 ? 0 : p.g.j0 - 1;
  const int c1 = p.g.j0 + p.g.tw + 1 > p.nx ? p.nx : p.g.j0 + p.g.tw + 1;
  const int64_t total = (int64_t)(((c1 + 3) >> 2) - (c0 >> 2)) * (r1 - r0);
  int64_t blocks = (total + NTHREADS - 1) / NTHREADS;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  tv_z_kernel<<<(unsigned)blocks, NTHREADS, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_opnorm(int which, const OpNormParams &p, const double *scale, cudaStream_t s) {
  const int blocks = 148 * 4;
  switch (which) {
    case 0: opnorm_init_kernel<<<blocks, NTHREADS, 0, s>>>(p); break;
    case 1: opnorm_fwd_kernel<<<blocks, NTHREADS, 0, s>>>(p); break;
    case 2: opnorm_adj_kernel<<<blocks, NTHREADS, 0, s>>>(p); break;
    default: opnorm_scale_kernel<<<blocks, NTHREADS, 0, s>>>(p, scale); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_copy_jobs(const CopyJob *d_jobs, int njobs, int max_elems, cudaStream_t s) {
  if (njobs == 0) return cudaSuccess;
  int bx = (max_elems + 255) / 256;
  if (bx > 64) bx = 64;
  if (bx < 1) bx = 1;
  copy_jobs_kernel<<<dim3(bx, njobs), 256, 0, s>>>(d_jobs);
  return cudaGetLastError();
}

// Test hook (pnpula_debug_philox): the raw Philox4x32-10 words and the four Box-Muller normals of
// counters ctr[i] = (column quad, row, t+1, stream) under key `seed`, computed by the very device
// functions the update kernels call (normals4 / normals4x2); bad[0] counts counters whose
// normals4 and normals4x2 results differ in any bit (they must not).
__global__ void debug_philox_kernel(uint32_t seed_lo, uint32_t seed_hi, const uint4 *ctr, int64_t n, uint4 *words,
                                    float4 *normals, int *bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 c = ctr[i];
    words[i] = philox4x32_10(c, seed_lo, seed_hi);
    float a[4], b[2][4];
    normals4(seed_lo, seed_hi, c.x, c.y, c.z, c.w, a);
    normals4x2(seed_lo, seed_hi, c.x, c.y, c.z, c.w, b);
    normals[i] = make_float4(a[0], a[1], a[2], a[3]);
    bool same = true;
#pragma unroll
    for (int l = 0; l < 4; ++l) same = same && __float_as_uint(a[l]) == __float_as_uint(b[0][l]);
    if (!same) atomicAdd(bad, 1);
  }
}

cudaError_t launch_debug_philox(uint64_t seed, const uint32_t *d_ctr, int64_t n, uint32_t *d_words, float *d_normals,
                                int *d_bad, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  debug_philox_kernel<<<(unsigned)blocks, 256, 0, s>>>((uint32_t)seed, (uint32_t)(seed >> 32),
                                                       reinterpret_cast<const uint4 *>(d_ctr), n,
                                                       reinterpret_cast<uint4 *>(d_words),
                                                       reinterpret_cast<float4 *>(d_normals), d_bad);
  return cudaGetLastError();
}

cudaError_t launch_fill(float *ptr, float v, size_t n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  size_t blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  fill_kernel<<<(unsigned)blocks, 256, 0, s>>>(ptr, v, n);
  return cudaGetLastError();
}

cudaError_t launch_finalize(const FinalizeParams &p, cudaStream_t s) {
  const int64_t n = (int64_t)p.g.th * p.g.tw;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
  finalize_kernel<<<(unsigned)blocks, 256, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace pnpula
