// update_math.cuh -- device arithmetic of the K7 x / z / moment update (Algorithm 1 lines 6-13,
// P:612-645) shared by the stand-alone update kernels (update_kernels.cu) and the update fused
// into the last CNN chunk (cnn_kernels.cu): Philox4x32-10 + Box-Muller noise and the per-pixel
// elementwise tail.  Both paths inline these same expressions, so a fused and a stand-alone
// update of the same pixel compute the same bits.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "internal.h"

namespace pnpula {
namespace upd {

// ---------------------------------------------------------------- Philox4x32-10 (Random123)
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = 0xD2511F53u * c.x;
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

// ln(u), u = (U + 0.5) 2^-32, accurate for u near 0 and near 1, without a data-dependent branch
// (both halves are evaluated and selected, so a warp never runs two paths):
//  * u <= 1/2: the hardware log2 (abs. error ~2^-22 on |log2 u| >= 1, i.e. relative 2^-22);
//  * u > 1/2: ln(1 - v) = -2 atanh(z), z = v / (2 - v) in (0, 1/3], with v = 1 - u formed
//    exactly from the integer; atanh(z) = z (1 + w/3 + w^2/5 + ... + w^7/15), w = z^2 <= 1/9
//    (truncation < w^8/17 ~ 1e-9 relative; a few ulp of rounding).
__device__ __forceinline__ float log_unit(uint32_t U) {
  const float lo = __log2f(fmaf((float)U, 0x1p-32f, 0x1p-33f)) * 0.69314718055994531f;
  const float v = fmaf((float)(~U), 0x1p-32f, 0x1p-33f);   // 1 - u
  const float z = __fdividef(v, 2.0f - v);
  const float w = z * z;
  float a = 1.0f / 15.0f;
  a = fmaf(a, w, 1.0f / 13.0f);
  a = fmaf(a, w, 1.0f / 11.0f);
  a = fmaf(a, w, 1.0f / 9.0f);
  a = fmaf(a, w, 1.0f / 7.0f);
  a = fmaf(a, w, 1.0f / 5.0f);
  a = fmaf(a, w, 1.0f / 3.0f);
  a = fmaf(a, w, 1.0f);
  const float hi = -2.0f * z * a;
  return U < 0x80000000u ? lo : hi;
}

// Box-Muller pair from (Ua, Ub): (rho cos theta, rho sin theta), theta = 2 pi (Ub+0.5) 2^-32,
// evaluated as pi * x with x = ((int)Ub + 0.5) 2^-31 in (-1, 1) (same angle mod 2 pi) with
// the hardware sin/cos (abs. error ~2^-21 on [-pi, pi]).
__device__ __forceinline__ float2 box_muller(uint32_t Ua, uint32_t Ub) {
  const float rho = sqrtf(-2.0f * log_unit(Ua));
  const float xs = fmaf((float)(int32_t)Ub, 0x1p-31f, 0x1p-32f);
  float s, c;
  __sincosf(3.14159265358979323846f * xs, &s, &c);
  return make_float2(rho * c, rho * s);
}

__device__ __forceinline__ void normals4(uint32_t seed_lo, uint32_t seed_hi, uint32_t quad,
                                         uint32_t row, uint32_t t1, uint32_t stream, float out[4]) {
  const uint4 w = philox4x32_10(make_uint4(quad, row, t1, stream), seed_lo, seed_hi);
  const float2 a = box_muller(w.x, w.y);
  const float2 b = box_muller(w.z, w.w);
  out[0] = a.x; out[1] = a.y; out[2] = b.x; out[3] = b.y;
}

// the normal of one pixel of a quad (element l = column & 3 of normals4): one Philox call and
// the one Box-Muller pair the element belongs to -- the same bits as normals4(...)[l]
__device__ __forceinline__ float normal1(uint32_t seed_lo, uint32_t seed_hi, uint32_t quad, uint32_t row,
                                         uint32_t t1, uint32_t stream, int l) {
  const uint4 w = philox4x32_10(make_uint4(quad, row, t1, stream), seed_lo, seed_hi);
  const float2 a = (l & 2) ? box_muller(w.z, w.w) : box_muller(w.x, w.y);
  return (l & 1) ? a.y : a.x;
}

// normals4 for rows `row` and `row + 1` of the same quad, the two Philox chains advanced in one
// loop (independent chains interleave: twice the instruction-level parallelism of two calls)
__device__ __forceinline__ void normals4x2(uint32_t seed_lo, uint32_t seed_hi, uint32_t quad, uint32_t row,
                                           uint32_t t1, uint32_t stream, float out[2][4]) {
  uint4 c0 = make_uint4(quad, row, t1, stream), c1 = make_uint4(quad, row + 1u, t1, stream);
  uint32_t k0 = seed_lo, k1 = seed_hi;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = 0xD2511F53u * c0.x, hi0 = __umulhi(0xD2511F53u, c0.x);
    const uint32_t lo1 = 0xCD9E8D57u * c0.z, hi1 = __umulhi(0xCD9E8D57u, c0.z);
    const uint32_t lo2 = 0xD2511F53u * c1.x, hi2 = __umulhi(0xD2511F53u, c1.x);
    const uint32_t lo3 = 0xCD9E8D57u * c1.z, hi3 = __umulhi(0xCD9E8D57u, c1.z);
    c0 = make_uint4(hi1 ^ c0.y ^ k0, lo1, hi0 ^ c0.w ^ k1, lo0);
    c1 = make_uint4(hi3 ^ c1.y ^ k0, lo3, hi2 ^ c1.w ^ k1, lo2);
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  const float2 a0 = box_muller(c0.x, c0.y), b0 = box_muller(c0.z, c0.w);
  const float2 a1 = box_muller(c1.x, c1.y), b1 = box_muller(c1.z, c1.w);
  out[0][0] = a0.x; out[0][1] = a0.y; out[0][2] = b0.x; out[0][3] = b0.y;
  out[1][0] = a1.x; out[1][1] = a1.y; out[1][2] = b1.x; out[1][3] = b1.y;
}

// ---------------------------------------------------------------- per-pixel elementwise tail
// x+ = x - a_g g - a_rho (x - z) - a_d G + a_lam (clamp(x) - x) - a_tv dtv + a_xi xi
// TVM: 0 TV compiled out, 1 TV at run time, 2 a TV launch (no z / G / box terms; x+ = max(., 0), R37)
template <int TVM>
__device__ __forceinline__ float x_step(const UpdateParams &p, bool has_tv, float x, float gr, float G, float z,
                                        float dtv, float xi) {
  float v = x - p.a_g * gr;
  if (TVM != 2 && p.has_z) v -= p.a_rho * (x - z);
  if (TVM != 2 && p.has_G) v += p.a_d * (-G);
  if (TVM != 2 && p.has_box) v += p.a_lam * (fminf(fmaxf(x, p.c_lo), p.c_hi) - x);
  if (has_tv) v -= p.a_tv * dtv;
  v += p.a_xi * xi;
  return has_tv ? fmaxf(v, 0.f) : v;   // TV: PSGLA projection onto R+ after the step (R37)
}
// z+ = clamp(z - b_rho (z - x+) + b_zeta zeta, z_lo, z_hi)
__device__ __forceinline__ float z_step(const UpdateParams &p, float z, float xn, float ze) {
  const float v = z - p.b_rho * (z - xn) + p.b_zeta * ze;
  return fminf(fmaxf(v, p.z_lo), p.z_hi);
}
// Welford running mean / M2
__device__ __forceinline__ void welford(float xn, float inv_n, float &m, float &s) {
  const float d = xn - m;
  m = m + d * inv_n;
  s = s + d * (xn - m);
}

}  // namespace upd
}  // namespace pnpula
