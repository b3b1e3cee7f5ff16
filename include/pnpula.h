/*
 * pnpula.h -- C ABI of the B200-native data-parallel hot path of the distributed
 * Plug-and-Play ULA sampler of arXiv 2511.00870 ("A Distributed Plug-and-Play MCMC
 * Algorithm for High-Dimensional Inverse Problems").  PAPER.md line n is cited "P:n".
 *
 * One chain, one image of ny x nx grayscale pixels (C = 1), split into a
 * tiles_y x tiles_x grid of tiles (eq:subsets_cartesian_partition P:473-482 applied
 * to both axes, "A 2D tessellation can be obtained ...").  Every rank owns
 * n_tiles/world_size consecutive tiles (row-major tile order) on one CUDA device.
 * Each iteration t -> t+1 computes, for every owned pixel (Algorithm 1):
 *
 *   x+ = x - (gamma/sigma2) H1^T (H1 x - y)                      lines 6-7
 *          - (gamma/rho) (x - z)                                   line 6b, P:615  (H2 = I)
 *          - (alpha gamma/eps^2) G_eps(x)                          line 8,  P:623  (D = Id - G)
 *          + (gamma/lambda) (proj_[c_lo,c_hi](x) - x)
 *          + sqrt(2 gamma) xi^{t+1}                                line 9,
 *   z+ = proj_[z_lo,z_hi]( z - (kappa/rho)(z - x+) + sqrt(2 kappa) zeta^{t+1} )   lines 12-13
 *   if t+1 > burn_in: Welford update of the per-pixel mean / M2 with x+           P:839
 *
 * H1 is either a same-size true convolution with zero boundary (odd kh x kw kernel,
 * P:716-724) or a 0/1 mask.  G_eps is a DnCNN-style CNN:
 * 1 -> P, (K-2) x (P -> P), P -> 1 channels, 3x3 cross-correlation with zero
 * padding, bias on every layer, ReLU on all but the last layer.
 * Noise: Philox4x32-10 with key = seed and counter = (j >> 2, i, t+1, stream),
 * lane j & 3, Box-Muller -- a function of (seed, t, global pixel), so the chain is
 * bitwise independent of the tile grid and of world_size (strengthening P:1063-1064).
 *
 * The only per-iteration communication is one grouped halo exchange of x
 * (Alg. 1 line 5, grouped as in the remark P:674), of width
 * h = max(2 r_H, K) where r_H = max(kh, kw)/2 (0 for a mask) and K = n_layers
 * (0 without a prior): the receptive-field strategy of P:529-531 replaces the
 * per-layer exchanges of P:526 and the overlap-add of line 7 by redundant
 * computation on the halo.  Neighbours on other ranks are reached with NCCL
 * point-to-point calls; tiles on the same rank with device copies.
 *
 * Conventions (all functions):
 *  - return pnpula_status; PNPULA_OK = 0.  A thread-local message describing the
 *    last failure (or a step-size warning) is available from pnpula_last_error().
 *  - host pointers are only read during the call and are never retained; the
 *    caller keeps ownership.  Device memory is owned by the context.
 *  - a CUDA or NCCL failure poisons the context: every later call except
 *    pnpula_destroy returns PNPULA_E_STATE.
 *  - collective calls (marked [collective]) must be made by every rank in the
 *    same order.
 *  - a context is not thread-safe.
 *  - there is no CPU fallback: creation fails with PNPULA_E_CUDA when no sm_100
 *    device is available.
 */
#ifndef PNPULA_H
#define PNPULA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  PNPULA_OK = 0,
  PNPULA_E_INVALID_ARG = 1,        /* null pointer, non-positive step, even kernel, kappa not in (0, rho) */
  PNPULA_E_SHAPE = 2,              /* in_rect does not cover the rank's tiles (+) r_H, bad sizes */
  PNPULA_E_PARTITION_TOO_FINE = 3, /* a tile extent < halo width h along an axis with >= 2 tiles (Def. 1 (i)) */
  PNPULA_E_STEPSIZE = 4,           /* reserved: eq:stepsize_cond violations are warnings only */
  PNPULA_E_STATS_EMPTY = 5,        /* fewer than 1 (mean) / 2 (variance) post-burn-in samples */
  PNPULA_E_STATE = 6,              /* context poisoned by an earlier CUDA/NCCL error, or wrong call order */
  PNPULA_E_CUDA = 7,
  PNPULA_E_NCCL = 8,
  PNPULA_E_OOM = 9,
  PNPULA_E_UNSUPPORTED = 10        /* e.g. channels not in {16, 32, 64} */
} pnpula_status;

enum { PNPULA_OP_CONV = 0, PNPULA_OP_MASK = 1, PNPULA_OP_POISSON = 2 };
enum { PNPULA_SCOPE_LOCAL = 0, PNPULA_SCOPE_GLOBAL_ON_ROOT = 1 };

/* flags */
#define PNPULA_FLAG_HALO_VIA_NCCL 0x1  /* route same-rank halos through NCCL self send/recv (tests) */
#define PNPULA_FLAG_CNN_LAYERWISE 0x2  /* one CNN layer per launch instead of fused layer chains */
#define PNPULA_FLAG_NO_GRAPH      0x4  /* launch every kernel directly (default: after the first iteration, each
                                         untimed iteration replays a captured CUDA graph, the NCCL halo group
                                         included; env PNPULA_GRAPHS=0 does the same) */

typedef struct {
  int32_t i0, j0, h, w; /* rectangle of global pixel coordinates: rows [i0, i0+h), cols [j0, j0+w) */
} pnpula_rect;

enum { PNPULA_DEN_DNCNN = 0, PNPULA_DEN_DDFB = 1 };

/* Denoiser weights, fp32, copied at create and stored as bf16.
 * PNPULA_DEN_DNCNN: DnCNN-style, D = Id - G.
 * PNPULA_DEN_DDFB (Example sec:denoiser:cnn:ddfb P:378-395; R39-R42): unrolled dual
 *   forward-backward, D(v) = proj_[0,1](v - gamma_K W_K^* T_{K-1}(...T_1(W_K v))), T_k(u) =
 *   HT(u + gamma_k W_k proj_[0,1](v - W_k^* u)), HT = clamp to [-ht_eps, ht_eps]. */
typedef struct {
  int32_t n_layers;      /* K >= 2 (DnCNN), >= 1 (DDFB) */
  int32_t channels;      /* P, one of 16, 32, 64 */
  const float *weights;  /* host; DnCNN: OIHW per layer, layers concatenated:
                            [P][1][3][3], (K-2) x [P][P][3][3], [1][P][3][3];
                            DDFB: K x [P][C][3][3] (W_k : C -> P, PyTorch conv2d convention;
                            C = img_channels) */
  const float *biases;   /* host; DnCNN: P per layer for layers 1..K-1, then 1; DDFB: unused */
  int32_t kind;          /* PNPULA_DEN_DNCNN (0) or PNPULA_DEN_DDFB */
  const float *ddfb_gammas;  /* DDFB: K steps gamma_k in (0, 2/||W_k||^2) */
  double ht_eps;         /* DDFB: hard-tanh level > 0 */
} pnpula_denoiser;

typedef struct {
  /* geometry and SPMD identity */
  int32_t ny, nx;                /* global image (channels: img_channels below) */
  int32_t tiles_y, tiles_x;      /* tile grid; tiles_y*tiles_x must be a multiple of world_size */
  int32_t rank, world_size;      /* this process; world_size >= 1 */
  int32_t device;                /* CUDA device ordinal used by this rank */
  const uint8_t *nccl_uid;       /* 128 bytes from pnpula_get_unique_id on rank 0; required if world_size > 1 */
  uint64_t stream;               /* cudaStream_t to launch on, or 0 for a context-owned stream */

  /* likelihood f1(H1 x) = ||y - H1 x||^2 / (2 sigma2)  (eq:potential_gaussian_likelihood P:708-711),
   * or (PNPULA_OP_POISSON) y ~ Poisson(eta H x) handled through AXDA (eq:poisson:f2 P:737-741):
   * f1 = 0, block z1 ~ eta H x with f2,1 = KL(y || .) (eta, rho1, kappa1 below), block z2 ~ x
   * with f2,2 = indicator of [z_lo, z_hi] (rho, kappa; the paper's R+ is z_lo = 0, z_hi = inf) */
  int32_t op;                    /* PNPULA_OP_CONV, PNPULA_OP_MASK or PNPULA_OP_POISSON */
  const float *kernel;           /* host kh x kw row-major true-convolution kernel; may be NULL if separable factors given */
  const float *kernel_y;         /* optional separable factors: kernel[p][q] = kernel_y[p] * kernel_x[q] exactly */
  const float *kernel_x;
  int32_t kh, kw;                /* odd sizes, <= 15 */
  const uint8_t *mask;           /* host, covers in_rect, OP_MASK only (nonzero = observed) */
  const float *y;                /* host observations covering in_rect (OP_POISSON: counts >= 0) */
  const float *x0;               /* host initial state covering in_rect, or NULL for zeros */
  pnpula_rect in_rect;           /* the rectangle y / mask / x0 cover (row-major h x w); must contain
                                    every owned tile (+) r_H clipped to the image.  Use the whole image
                                    {0, 0, ny, nx} when passing global arrays. */
  double sigma2;                 /* noise variance > 0 (ignored by OP_POISSON) */

  /* prior */
  const pnpula_denoiser *den;    /* NULL or alpha == 0: no CNN term */
  double alpha, eps;             /* prior strength and denoiser noise level */
  double lambda, c_lo, c_hi;     /* Moreau/box term (gamma/lambda)(proj_C(x) - x); lambda <= 0 disables */

  /* AXDA z-block with H2 = I, f2 = indicator of [z_lo, z_hi]; rho <= 0 disables */
  double rho, kappa, z_lo, z_hi;

  double gamma;                  /* ULA step > 0 */

  /* optional constants for the eq:stepsize_cond check (warning only; 0 = unknown) */
  double lipschitz_L, lipschitz_LD;

  int32_t flags;                 /* PNPULA_FLAG_* */

  /* OP_POISSON only (sec:poisson_deconvolution P:727-744; R31-R34):
   * eta > 0 Poisson scale, rho1 > 0 coupling of z1 ~ eta H x, kappa1 in (0, rho1) its PSGLA step.
   * Per iteration: x+ = x - (gamma/rho1)(eta H)^T(eta H x - z1) - (gamma/rho)(x - z2) + prior and
   * box terms + sqrt(2 gamma) xi;  z2+ as for OP_CONV;  z1+ = prox_{kappa1 KL(y||.)}(z1 -
   * (kappa1/rho1)(z1 - eta H x+) + sqrt(2 kappa1) zeta1), zeta1 = Philox stream 2. */
  double eta, rho1, kappa1;

  /* TV prior instead of the denoiser (item:prior_choice:tv P:786-809; R35-R38):
   * tv_beta > 0 turns the z block into z = (z_v, z_h) ~ D x (2-D forward differences) with
   * f2 = tv_beta ||.||_{2,1} (coupling rho, step kappa), and x moves by PSGLA with p = 1_{R+}:
   * x+ = max(x - gamma grad f1 - (gamma/rho) D^T (D x - z) + sqrt(2 gamma) xi, 0).
   * Requires rho > 0, no denoiser, lambda <= 0; with OP_POISSON the z1 block is kept
   * and f1 = 0.  pnpula_get_state returns z_v, pnpula_get_tv_zh z_h. */
  double tv_beta;

  /* Image channels C (colour images; R43): 0 or 1 = grayscale, 3 = RGB.
   * y, x0 and every per-pixel output (x, z, z1, mean, var, G) are C planes [C][h][w] (planar);
   * the mask is one plane shared by the channels.  H, the box and the z blocks act on each
   * channel; the DnCNN's first layer is C -> P and its last P -> C (weights OIHW as for C = 1,
   * with I = C / O = C; needs channels P >= 32).  Channel c draws Philox streams 4c + s.
   * DDFB: W_k : C -> P and W_k^* : P -> C (P = 32 or 64).  TV: channel-wise isotropic
   * ||.||_{2,1} (D acts on every plane), z_v / z_h have C planes. */
  int32_t img_channels;
} pnpula_config;

typedef struct pnpula_ctx pnpula_ctx;

/* Library version string. */
const char *pnpula_version(void);

/* Thread-local description of the last error or warning ("" if none). */
const char *pnpula_last_error(void);

/* 128-byte NCCL unique id; call on rank 0 and broadcast it (e.g. torch.distributed). */
pnpula_status pnpula_get_unique_id(uint8_t out[128]);

/* [collective] Validate cfg, partition the image, initialise NCCL (world_size > 1),
 * allocate device buffers, copy y / mask / x0 / kernel / weights (bf16) to the device.
 * On success *out receives a new context.  Step-size condition violations
 * (eq:stepsize_cond P:581-587, read with ||H2||^2/rho, R11) are reported
 * through pnpula_last_error() but do not fail. */
pnpula_status pnpula_create(const pnpula_config *cfg, pnpula_ctx **out);

/* [collective] Reset the chain: x = x0 (halos exchanged), z = 0, moments = 0, t = 0,
 * and set burn_in and seed for the following pnpula_advance calls. */
pnpula_status pnpula_reset(pnpula_ctx *ctx, int64_t burn_in, uint64_t seed);

/* [collective] Run n_iter further iterations (asynchronous on the context stream).
 * Execution (results are bitwise the same either way): after the first iteration, untimed
 * iterations replay a captured CUDA graph per x-buffer parity, with the NCCL halo group of a
 * multi-rank run captured inside it (PNPULA_FLAG_NO_GRAPH / env PNPULA_GRAPHS=0: direct
 * launches); with NCCL halo messages on a row-strip grid the update runs the h boundary rows of
 * each tile first and the exchange, on a second stream (a fork/join inside the graph), overlaps
 * the interior rows (env PNPULA_OVERLAP=0 at create: serial).  Every rank must use the same
 * graph setting (the captured NCCL calls are matched across ranks). */
pnpula_status pnpula_advance(pnpula_ctx *ctx, int64_t n_iter);

/* [collective] pnpula_reset(burn_in, seed) then pnpula_advance(n_iter), then
 * synchronise.  Deterministic in (cfg, n_iter, burn_in, seed) and bitwise independent
 * of the tile grid and of world_size. */
pnpula_status pnpula_run(pnpula_ctx *ctx, int64_t n_iter, int64_t burn_in, uint64_t seed);

/* Block until all work queued on the context stream has finished. */
pnpula_status pnpula_synchronize(pnpula_ctx *ctx);

/* Rectangle covered by LOCAL-scope outputs: the bounding box of this rank's tiles. */
pnpula_status pnpula_local_bbox(pnpula_ctx *ctx, pnpula_rect *out);

/* [collective for GLOBAL scope] Posterior mean (MMSE) and per-pixel variance
 * M2/(n-1) of x^{(t)}, t = burn_in+1 .. current t.  mean / var (either may be
 * NULL) are host buffers of the LOCAL bbox size, or ny*nx on rank 0 for
 * PNPULA_SCOPE_GLOBAL_ON_ROOT (other ranks may pass NULL); times C planes for C > 1.  Returns
 * PNPULA_E_STATS_EMPTY if n < 1 (mean) or n < 2 (var requested); GLOBAL_ON_ROOT with
 * world_size > 1 returns it on every rank when n < 2, whatever pointers a rank passes (the
 * outcome of a collective call must not differ between ranks). */
pnpula_status pnpula_get_moments(pnpula_ctx *ctx, float *mean, float *var, int64_t *n_samples,
                                 int32_t scope);

/* [collective for GLOBAL scope] Current state x^t, z^t (either may be NULL) and t. */
pnpula_status pnpula_get_state(pnpula_ctx *ctx, float *x, float *z, int64_t *t, int32_t scope);

/* [collective for GLOBAL scope] OP_POISSON: current z1 block (the AXDA variable ~ eta H x), on
 * the LOCAL bbox or, on root, the whole image. */
pnpula_status pnpula_get_z1(pnpula_ctx *ctx, float *z1, int32_t scope);

/* [collective for GLOBAL scope] TV prior: the horizontal component z_h of z ~ D x (z_v is the z of
 * pnpula_get_state); C planes for colour images, like every per-pixel output. */
pnpula_status pnpula_get_tv_zh(pnpula_ctx *ctx, float *zh, int32_t scope);

/* Checkpoint / resume.  The blob holds this rank's complete chain state:
 * t, burn-in, seed and, per owned tile, the padded buffers (interior + ghost frame) of x^t,
 * the z blocks (z; z1 for OP_POISSON / z_h for TV) and the Welford mean / M2, so that
 * load + advance(n) is bitwise identical to never having stopped.  Host memory, caller-owned.
 * pnpula_checkpoint_bytes: size of the blob.  pnpula_save_checkpoint: writes it (bytes must be
 * >= the size, else E_INVALID_ARG).  pnpula_load_checkpoint: restores a blob saved by a context
 * created with the same configuration, tile grid and rank (E_SHAPE if the header differs); it
 * replaces pnpula_reset. */
pnpula_status pnpula_checkpoint_bytes(pnpula_ctx *ctx, uint64_t *bytes);
pnpula_status pnpula_save_checkpoint(pnpula_ctx *ctx, void *buf, uint64_t bytes);
pnpula_status pnpula_load_checkpoint(pnpula_ctx *ctx, const void *buf, uint64_t bytes);

/* Number of tiles owned by this rank; halo width h; the i-th owned tile's rectangle. */
pnpula_status pnpula_tile_info(pnpula_ctx *ctx, int32_t local_index, pnpula_rect *rect,
                               int32_t *n_local_tiles, int32_t *halo);

/* Diagnostic: padded buffer (tile (+) h ghost frame, row-major (th+2h) x (tw+2h)) of the
 * current x of owned tile local_index, as the next iteration will read it. */
pnpula_status pnpula_get_padded_x(pnpula_ctx *ctx, int32_t local_index, float *out);

/* [collective] Diagnostic: evaluate the CNN residual G_eps on the current x^t and
 * return it for the LOCAL bbox (host buffer, owned tiles written). */
pnpula_status pnpula_get_denoiser_residual(pnpula_ctx *ctx, float *G);

/* Per-kernel-class device time accumulated since the last call with reset != 0,
 * measured with CUDA events on the launching stream while timing is enabled.
 * name: "cnn", "update", "halo" (launches = timed launch groups), or "all": the number
 * of kernels this library launched (counted even with timing off; ms = 0). */
pnpula_status pnpula_set_timing(pnpula_ctx *ctx, int32_t enable);
pnpula_status pnpula_kernel_time(pnpula_ctx *ctx, const char *name, double *ms, int64_t *launches,
                                 int32_t reset);

/* [collective] Free everything.  The per-tile state buffers (x, y, z blocks, moments, CNN
 * activations) come from a per-process, per-device stream-ordered memory pool that keeps freed
 * memory for the next context (env PNPULA_POOL=0 at create: plain cudaMalloc / cudaFree). */
pnpula_status pnpula_destroy(pnpula_ctx *ctx);

/* Return the pool's unused device memory of `device` to the driver (cudaMemPoolTrimTo 0).
 * E_INVALID_ARG if the device has no pool. */
pnpula_status pnpula_release_memory(int32_t device);

/* Test hook for the noise of a6 (reading R9): the generator the update kernels use,
 * evaluated on the device for n caller-chosen counters.  counters: host, n x 4 uint32
 * (column quad j>>2, row i, iteration index t+1, stream) -- the Philox4x32-10 counter of R9 --
 * under key (seed lo, seed hi).  words: host, n x 4, the raw Philox4x32-10 output words;
 * normals: host, n x 4 fp32, the four Box-Muller normals of the quad (lanes j&3 = 0..3) exactly
 * as the x / z updates draw them (the same device functions; reading R45 bounds their error
 * against the fp64 definition).  Synchronous; allocates and frees its own device memory.
 * PNPULA_E_STATE if the kernels' two normal paths (one and two Philox chains per thread)
 * disagree in any bit. */
pnpula_status pnpula_debug_philox(int32_t device, uint64_t seed, const uint32_t *counters, int64_t n,
                                  uint32_t *words, float *normals);

/* ---------------- host-only planning helpers (no GPU needed) ---------------- */

/* Balanced 0-based partition of n items into parts: [lo, hi) of part p (R4). */
void pnpula_partition(int64_t n, int64_t parts, int64_t p, int64_t *lo, int64_t *hi);

/* Halo width h = max(2 r_H, K) (receptive-field strategy, R5). */
int32_t pnpula_halo_width(int32_t op, int32_t kh, int32_t kw, int32_t n_layers);

/* [collective] ||H||_2^2 of this context's forward operator (the same-size, zero-boundary
 * convolution over the whole image, every tile and rank) by `iters` >= 2 power iterations on the
 * GPU (v <- H^T H v / ||.||, Rayleigh quotient of the last unit iterate; start vector = fixed
 * Philox normals).  OP_MASK returns 1.  Uses the idle x buffer as scratch: call between
 * iterations only (the chain state is untouched).  SURVEY 8(f) rank 4 (step sizes P:774/P:782). */
pnpula_status pnpula_opnorm2(pnpula_ctx *ctx, int32_t iters, double *out);

/* Host helper for the step sizes: upper bound of ||H||_2^2 for the same-size,
 * zero-boundary convolution with the kh x kw kernel k (host, row-major): max over a grid x grid
 * DFT of |K(w)|^2 (the zero-boundary operator is a restriction of the full convolution, whose
 * norm is sup |K(w)|; grid >= max(kh, kw), e.g. 256).  Returns PNPULA_E_INVALID_ARG on bad sizes. */
pnpula_status pnpula_conv_norm2_bound(const float *k, int32_t kh, int32_t kw, int32_t grid, double *out);

/* One ghost-region message: the global rectangle `rect` of tile src's interior
 * that tile dst stores in its ghost frame (Fig. 2(b)). */
typedef struct {
  int32_t src_tile, dst_tile; /* row-major tile indices */
  pnpula_rect rect;
} pnpula_halo_msg;

/* All messages of one exchange for a tiles_y x tiles_x grid and halo h, in the
 * canonical (src_tile, dst_tile) order used to post NCCL sends/receives.
 * Writes at most cap messages to out (out may be NULL) and returns the total count,
 * or -1 if a tile extent is smaller than h along an axis split into >= 2 tiles. */
int32_t pnpula_plan_halo(int32_t ny, int32_t nx, int32_t tiles_y, int32_t tiles_x, int32_t h,
                         pnpula_halo_msg *out, int32_t cap);

/* eq:stepsize_cond with ||H2||^2 read as h2_over_rho = ||H2||^2/rho
 * (R11).  Returns 0 if both hold, bit 0 / bit 1 for the failing inequality. */
int32_t pnpula_check_stepsizes(double L, double h2_over_rho, double alpha, double eps,
                               double L_D, double lambda, double gamma);

#ifdef __cplusplus
}
#endif
#endif /* PNPULA_H */
