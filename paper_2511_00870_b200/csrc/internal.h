// internal.h -- device-side parameter blocks shared by the host runtime
// (pnpula_host.cpp) and the sm_100a kernels (*.cu).  Not part of the C ABI.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace pnpula {

constexpr int kMaxTaps = 15;      // max kernel extent (odd), radius <= 7
constexpr int kMaxChunk = 8;      // max CNN layers fused in one launch

// Padded per-tile geometry: padded(r, c) holds global (i0 - h + r, j0 - hx + c).
struct TileGeom {
  int i0, j0, th, tw;   // interior rectangle (global)
  int h;                // halo width (rows and columns)
  int hx;               // padded column of interior column 0; (hx - j0) % 4 == 0 (mod 4 alignment)
  int ph;               // padded rows = th + 2h
  int pitch;            // floats per padded row (multiple of 32)
};

// Iteration state on the device for CUDA-graph replays (the graph of one iteration is replayed
// with unchanged parameters).  Two slots: the graph for x-buffer parity b reads slot b (this
// iteration's scalars) and its first update kernel writes slot b^1 (the next iteration's).
struct IterState {
  long long t1;           // iteration index t+1
  long long burn_in;
  int accumulate;         // t1 > burn_in
  float inv_n;            // 1 / (t1 - burn_in)
};

// K7: fused data-fidelity stencil + Moreau box + AXDA coupling + ULA update +
// Philox/Box-Muller noise + z PSGLA step + Welford moments, one tile.
struct UpdateParams {
  const float *x;       // padded x^t (halo filled)
  float *xn;            // padded x^{t+1} (interior written)
  const float *y;       // padded y (valid on tile (+) r_H, zero outside the image)
  const uint8_t *mask;  // padded mask (OP_MASK)
  const float *G;       // padded CNN residual (interior), or nullptr
  float *z;             // padded z (interior), in place, or nullptr
  float *mean, *m2;     // padded moments (interior), in place
  TileGeom g;
  int ny, nx;
  int op;               // 0 conv, 1 mask
  int ry, rx;           // kernel radii
  int separable;
  float k2d[kMaxTaps * kMaxTaps];
  float ky[kMaxTaps], kx[kMaxTaps];
  // coefficients (fp64 on host, rounded once)
  float a_g, a_rho, a_d, a_lam, a_xi;
  float c_lo, c_hi;
  float b_rho, b_zeta, z_lo, z_hi;
  int has_z, has_G, has_box;
  uint32_t seed_lo, seed_hi, t1;   // Philox key and iteration index t+1
  int accumulate;                  // t+1 > burn_in
  float inv_n;                     // 1 / (t+1 - burn_in)
  float eta;                       // residual r = eta (H x) - y: 1 for the Gaussian likelihood;
                                   // Poisson (reading R32): eta, with y -> z1 (AXDA block eta H x)
  int has_tv;                      // TV prior (R37): - a_tv D^T (D x - z) and x+ = max(., 0)
  float a_tv;                      // gamma / rho
  const float *zv, *zh;            // padded z = (z_v, z_h) ~ D x, valid on tile (+) 1
  const IterState *it;             // non-null: t1 / accumulate / inv_n from here (graph replay)
  IterState *it_next;              // non-null: block 0 writes the next iteration's scalars here
  uint32_t sb;                     // Philox stream base of this image channel (4 c, reading R43)
};

// TV z block (R37, R38): on tile (+) 1 inside the image
//   z <- prox_{kappa beta ||.||_{2,1}}( z - (kappa/rho)(z - D x+) + sqrt(2 kappa) zeta ),
// zeta_v = Philox stream 1, zeta_h = stream 3.
struct TvZParams {
  const float *x;       // padded x^{t+1} (halo >= 2 valid)
  float *zv, *zh;       // padded, in place on tile (+) 1
  TileGeom g;
  int ny, nx;
  float b, s, tau;      // kappa/rho, sqrt(2 kappa), kappa beta
  uint32_t seed_lo, seed_hi, t1;
  const IterState *it;  // non-null: t1 from here (graph replay)
  uint32_t sb;          // Philox stream base of this image channel (4 c, reading R43): zeta_v sb+1, zeta_h sb+3
};

// z1 block of the Poisson posterior (readings R32-R34): on tile (+) r_H (inside the image)
//   z1 <- prox_{kappa1 KL(y || .)}( z1 - (kappa1/rho1)(z1 - eta H x+) + sqrt(2 kappa1) zeta1 )
// with zeta1 = Philox stream 2 at the global pixel; x+ padded (halo >= 2 r_H valid).
struct Z1Params {
  const float *x;       // padded x^{t+1}
  const float *y;       // padded counts (valid on tile (+) r_H)
  float *z1;            // padded z1, in place on tile (+) r_H
  TileGeom g;
  int ny, nx;
  int ry, rx;
  float k2d[kMaxTaps * kMaxTaps];   // 2-D taps (separable factors multiplied out on the host)
  int separable;                    // ky / kx valid: separable fast path (R = 2, 4)
  float ky[kMaxTaps], kx[kMaxTaps];
  float eta, b1, s1, kappa1;        // eta, kappa1/rho1, sqrt(2 kappa1), kappa1
  uint32_t seed_lo, seed_hi, t1;
  const IterState *it;              // non-null: t1 from here (graph replay)
  uint32_t sb;                      // Philox stream base of this image channel (4 c)
};

// One rectangular copy between pitched fp32 buffers (halo exchange, pack/unpack).
struct CopyJob {
  const float *src;
  float *dst;
  int src_pitch, dst_pitch;   // floats
  int rows, cols;
};

// Moments finalisation: var = M2 / (n - 1), packed interior -> contiguous.
struct FinalizeParams {
  const float *mean, *m2;
  float *out_mean, *out_var;   // contiguous th x tw (either may be nullptr)
  TileGeom g;
  float inv_nm1;
};

// CNN chain: layers [l0, l0+nl) of the DnCNN-style net in one launch (see cnn_kernels.cu).
struct CnnChunkParams {
  int P;                 // features
  int nl;                // layers in this launch
  int first_is_input;    // layer l0 == 1: input is x (fp32, 1 channel)
  int last_is_output;    // layer l0+nl-1 == K: output is G (fp32, 1 channel, no ReLU)
  const uint16_t *w[kMaxChunk];   // packed bf16 B-operand images, one per layer
  float bias[kMaxChunk][64];      // fp32 biases per layer (zero padded): kernel parameter space,
                                  // read through the constant cache (no shared-memory traffic)
  // input: x (padded fp32) or activation buffer
  const float *x; TileGeom xg;
  const uint16_t *ain; int a_i0, a_j0, a_rows, a_cols;   // activation region (global origin, extent)
  // output region (global) for the chunk's last layer
  int oi0, oj0, oh, ow;
  uint16_t *aout; int o_i0, o_j0, o_rows, o_cols;        // activation output buffer region
  float *G; TileGeom gg;                                  // G output (padded geometry)
  int ny, nx;
  int strips;            // column strips
  int rows_per_unit;     // output rows per work unit
  int units;             // strips * row blocks
  int rows_per_cta;      // > 0: CTA b owns strip-major output rows [b T, (b+1) T) instead (set by the launcher)
  int contig;            // 1: contiguous decomposition when the launcher's cost model prefers it; 2: always
  int *err;              // device error flag (watchdog)
  unsigned long long *trace;   // optional pipeline trace (CTA 0, first unit): [0] = count, then records
  int mode;              // 0 DnCNN; DDFB (R39-R42): 1 u0 = W_K v, 2 p = proj(v - W^* u), 3 u = HT(u + gamma W p),
                         // 4 G = v - proj(v - gamma_K W_K^* u)
  float ht_eps;          // DDFB hard-tanh level
  int mode0;             // DDFB two-operator launch (NL = 2): mode of the im2col layer (1 or 3); the folded
                         // layer uses `mode` (2 or 4); u' of layer 0 is also stored to aout
  const float *xv;       // DDFB: v (padded, geometry xg) for modes 2 / 4
  int nc;                // image channels C (1, or 3 with P >= 32; reading R43): planes of x / G
  int64_t xcs, gcs;      // floats between the channel planes of x and of G
  int pdl;               // launch as a programmatic dependent of the previous kernel (see pdl_wait)
  // Fused x / z / moment update (the chain's last layer, C = 1, P = 32): instead of storing G, the
  // folded layer's epilogue evaluates H^T(eta H x - y) in a streaming separable stencil (or the mask
  // term) and the K7 tail of `up` for every tile pixel it completes -- the same per-pixel
  // arithmetic as update_sep_kernel / update_mask_kernel (update_math.cuh), so results are bitwise
  // those of the unfused iteration.  up.G is unused.
  int fuse;
  UpdateParams up;
};

// Programmatic dependent launch (PDL): the CNN chain kernels are launched as dependents of the
// kernel before them, so their prologue (weights to shared memory, barriers, TMEM) runs on the SMs
// the previous kernel's CTAs have left while its last CTAs finish; they execute griddepcontrol.wait
// before touching anything the previous kernel wrote.  Every kernel that can precede a CNN launch
// signals griddepcontrol.launch_dependents at its start.  Env PNPULA_PDL=0 at create: plain launches.
#if defined(__CUDACC__)
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
#endif

// Launchers (return cudaGetLastError()).
cudaError_t launch_update(const UpdateParams &p, cudaStream_t s);
cudaError_t launch_z1_update(const Z1Params &p, cudaStream_t s);

// power iteration for ||H||^2 (pnpula_opnorm2)
struct OpNormParams {
  float *v;          // padded iterate (halo exchanged)
  float *w;          // padded H v on tile (+) r_H
  float *u;          // padded H^T H v on the tile
  double *acc;       // [0] sum u^2, [1] sum u.v (device, accumulated over tiles)
  TileGeom g;
  int ny, nx, ry, rx;
  float k2d[kMaxTaps * kMaxTaps];
};
// which: 0 init v, 1 w = H v, 2 u = H^T w (+ sums), 3 v = u * (*scale)
cudaError_t launch_opnorm(int which, const OpNormParams &p, const double *scale, cudaStream_t s);
cudaError_t launch_tv_z_update(const TvZParams &p, cudaStream_t s);
cudaError_t launch_copy_jobs(const CopyJob *d_jobs, int njobs, int max_rows, cudaStream_t s);
cudaError_t launch_fill(float *p, float v, size_t n, cudaStream_t s);
cudaError_t launch_finalize(const FinalizeParams &p, cudaStream_t s);
// test hook: raw Philox words + normals of n counters (device arrays, n x 4 each)
cudaError_t launch_debug_philox(uint64_t seed, const uint32_t *d_ctr, int64_t n, uint32_t *d_words, float *d_normals,
                                int *d_bad, cudaStream_t s);
cudaError_t launch_cnn_chunk(const CnnChunkParams &p, int num_sms, cudaStream_t s);
// shared-memory bytes of a chain, or SIZE_MAX if it does not fit
size_t cnn_chunk_smem_bytes(int P, int nl, int first_is_input, int last_is_output, int nc, int fuse = 0);
// the fused update is compiled for P = 32, C = 1 chains; conv: separable with ry = rx in {2, 4}, or mask
bool cnn_fused_update_supported(int P, int nc, const UpdateParams &u);
// Pack host fp32 OIHW weights of one layer into the device B-operand image (host side).
void cnn_pack_layer(const float *w, int cout, int cin, uint16_t *out);
size_t cnn_packed_layer_elems(int cout, int cin);

}  // namespace pnpula
