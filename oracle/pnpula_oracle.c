/*
 * pnpula_oracle.c -- plain, slow, obviously-correct CPU oracle for the
 * distributed PnP-ULA sampler of arXiv 2511.00870 (PAPER.md, "P:n" = line n).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * (paper_2511_00870_b200/csrc); neither includes the other.
 *
 * Arithmetic: IEEE binary64 throughout; plain nested loops in the paper's
 * order; no blocking, fusion or reordering.  Optional "bf16 emulation" rounds
 * CNN weights / the CNN input / inter-layer activations to bfloat16 (RNE) at the
 * points where the GPU path stores bf16 (reading R26), still
 * accumulating in fp64.
 *
 * What each function follows:
 *   or_partition        eq:subsets_cartesian_partition P:473-482 (0-based, reading R4)
 *   or_philox4x32_10    Philox4x32-10 (Salmon et al. 2011, Random123 constants) -- reading R9
 *   or_normal           Box-Muller of Philox words, counter keyed on (seed, t+1, i, j, stream) R9/R10
 *   or_conv_fwd/adj     H1 = same-size true convolution with zero boundary and its adjoint
 *                       (readings R1/R2/R7); mask operator P:697-713
 *   or_dncnn_residual   G_eps = T_K o ... o T_1 (eq:feedforward_cnn P:346-351,
 *                       eq:cnn:convolution P:358-363, DnCNN example P:366-375)
 *   or_run              Algorithm 1: x-update eq:sgs_pnp_ula_psgla:pnp_ula,
 *                       z-update eq:sgs_pnp_ula_psgla:psgla, online moments
 *   or_run (tiles>1)    same chain, every tile computed from its own padded copy S_b x
 *                       (Def. prop:localselection P:135-152, ghost regions P:494-498)
 *   or_ddfb_residual_c  DDFB denoiser G = v - D(v) (Example sec:denoiser:cnn:ddfb, eq:ddfb_operator
 *                       P:382-385, eq:dfb_operator:T P:390-393) for C image channels: W_k : C -> P,
 *                       W_k^* : P -> C (readings R39-R42, R43)
 *   or_run (C = 3)      colour images (reading R43): planes; H / mask / box / z blocks / TV per
 *                       channel (TV: channel-wise isotropic ||.||_{2,1}, D acting per plane)
 *   or_check_stepsizes  eq:stepsize_cond P:581-587 (reading R11: ||H2||^2 -> ||H2||^2/rho)
 *   or_prox_kl          prox of kappa KL(y || .) for the Poisson likelihood (eq:poisson:f2 P:737-741;
 *                       closed form = the positive root of u^2 - (v - kappa) u - kappa y = 0, reading R31)
 *   or_grad2d / adj     D = 2-D discrete gradient (item:prior_choice:tv P:786-806): forward
 *                       differences, zero at the last row / column; D^T its exact transpose (R35)
 *   or_prox_l21         prox of tau ||.||_{2,1}: per-pixel block soft threshold (R36)
 *   or_run (tv_beta>0)  TV prior with Gaussian noise: x by PSGLA with p = 1_{R+},
 *                       z ~ D x with f2 = beta ||.||_{2,1} (rho, kappa) (readings R35-R38)
 *   or_run (op = 2)     Poisson deconvolution (sec:poisson_deconvolution P:727-744):
 *                       f1 = 0, z = (z1, z2), z1 ~ eta H x with f2,1 = KL(y || .) (rho1, kappa1),
 *                       z2 ~ x with f2,2 = indicator of [z_lo, z_hi] (rho, kappa); Algorithm 1 lines
 *                       6-13 with H2 = [eta H; I] (readings R32-R34)
 *
 * Parity pins for each function live in tests/test_oracle_*.py (see DESIGN.md
 * section "Oracle pins").
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_E_INVALID 1
#define OR_E_STATS_EMPTY 5

/* ------------------------------------------------------------------ */
/* Partition: 0-based form of eq:subsets_cartesian_partition:
 * block p of n items split in `parts` covers [floor(p n/parts), floor((p+1) n/parts)). */
void or_partition(int64_t n, int64_t parts, int64_t p, int64_t *lo, int64_t *hi) {
  *lo = (p * n) / parts;
  *hi = ((p + 1) * n) / parts;
}

/* OpenMP over output rows (the oracle is timed single-thread and on all cores).
 * Every parallelised loop writes disjoint outputs, each computed exactly as in the serial loop
 * (same operands, same order), so results do not depend on the thread count; built without
 * -fopenmp the pragmas vanish. */
#ifdef _OPENMP
#define OR_PARALLEL_ROWS _Pragma("omp parallel for schedule(static)")
#define OR_PARALLEL_ROWS2 _Pragma("omp parallel for collapse(2) schedule(static)")
#else
#define OR_PARALLEL_ROWS
#define OR_PARALLEL_ROWS2
#endif

/* ------------------------------------------------------------------ */
/* Philox4x32-10 (Random123).  10 rounds; key schedule bumped between rounds. */
static void or_mulhilo(uint32_t a, uint32_t b, uint32_t *hi, uint32_t *lo) {
  uint64_t p = (uint64_t)a * (uint64_t)b;
  *hi = (uint32_t)(p >> 32);
  *lo = (uint32_t)p;
}

void or_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int r = 0; r < 10; r++) {
    if (r > 0) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    uint32_t hi0, lo0, hi1, lo1;
    or_mulhilo(0xD2511F53u, c0, &hi0, &lo0);
    or_mulhilo(0xCD9E8D57u, c2, &hi1, &lo1);
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Standard normal at global pixel (i, j), iteration index t1 = t+1, stream s
 * (0 = xi for x, 1 = zeta for z).  Reading R9: counter = (j>>2, i, t1, s),
 * key = (seed lo, seed hi); lane = j & 3.  Box-Muller in fp64:
 *   u_k = (U_k + 0.5) 2^-32,  rho = sqrt(-2 ln u_0),  theta = 2 pi u_1,
 *   lanes 0,1 = rho cos(theta), rho sin(theta); lanes 2,3 likewise from (U_2, U_3). */
double or_normal(uint64_t seed, uint32_t t1, int64_t i, int64_t j, uint32_t stream) {
  uint32_t ctr[4] = {(uint32_t)((uint64_t)j >> 2), (uint32_t)i, t1, stream};
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t w[4];
  or_philox4x32_10(ctr, key, w);
  int lane = (int)(j & 3);
  int pair = lane >> 1;
  double u0 = ((double)w[2 * pair] + 0.5) * 0x1p-32;
  double u1 = ((double)w[2 * pair + 1] + 0.5) * 0x1p-32;
  double rho = sqrt(-2.0 * log(u0));
  double theta = 2.0 * M_PI * u1;
  return (lane & 1) ? rho * sin(theta) : rho * cos(theta);
}

void or_normal_field(uint64_t seed, uint32_t t1, int32_t ny, int32_t nx, uint32_t stream, double *out) {
  for (int64_t i = 0; i < ny; i++)
    for (int64_t j = 0; j < nx; j++) out[i * nx + j] = or_normal(seed, t1, i, j, stream);
}

/* ------------------------------------------------------------------ */
/* H1 = same-size true convolution, zero boundary (readings R1, R2):
 *   (Hx)[i,j] = sum_{p=-ry..ry} sum_{q=-rx..rx} k[p+ry][q+rx] x[i-p][j-q]      */
void or_conv_fwd(const double *x, int32_t ny, int32_t nx, const double *k, int32_t kh, int32_t kw,
                 double *out) {
  int ry = kh / 2, rx = kw / 2;
  OR_PARALLEL_ROWS
  for (int i = 0; i < ny; i++)
    for (int j = 0; j < nx; j++) {
      double s = 0.0;
      for (int p = -ry; p <= ry; p++)
        for (int q = -rx; q <= rx; q++) {
          int ii = i - p, jj = j - q;
          if (ii < 0 || ii >= ny || jj < 0 || jj >= nx) continue;
          s += k[(p + ry) * kw + (q + rx)] * x[(int64_t)ii * nx + jj];
        }
      out[(int64_t)i * nx + j] = s;
    }
}

/* Adjoint H1^T: correlation with the same kernel, zero boundary:
 *   (H^T r)[i,j] = sum_{p,q} k[p+ry][q+rx] r[i+p][j+q]                            */
void or_conv_adj(const double *r, int32_t ny, int32_t nx, const double *k, int32_t kh, int32_t kw,
                 double *out) {
  int ry = kh / 2, rx = kw / 2;
  OR_PARALLEL_ROWS
  for (int i = 0; i < ny; i++)
    for (int j = 0; j < nx; j++) {
      double s = 0.0;
      for (int p = -ry; p <= ry; p++)
        for (int q = -rx; q <= rx; q++) {
          int ii = i + p, jj = j + q;
          if (ii < 0 || ii >= ny || jj < 0 || jj >= nx) continue;
          s += k[(p + ry) * kw + (q + rx)] * r[(int64_t)ii * nx + jj];
        }
      out[(int64_t)i * nx + j] = s;
    }
}

/* ------------------------------------------------------------------ */
/* bfloat16 round-to-nearest-even of a double, via fp32 (the GPU stores fp32
 * values converted with __float2bfloat16_rn). */
static double or_bf16(double v) {
  float f = (float)v;
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) return (double)f; /* inf/nan passthrough */
  uint32_t lsb = (u >> 16) & 1u;
  u += 0x7fffu + lsb;
  u &= 0xffff0000u;
  memcpy(&f, &u, 4);
  return (double)f;
}

/* Number of weights / biases of a DnCNN-style net with n_layers 3x3 layers,
 * C image channels and P features: C->P, (K-2) x P->P, P->C. */
int64_t or_dncnn_param_count(int32_t n_layers, int32_t P, int32_t C) {
  int64_t w = (int64_t)C * P * 9 + (int64_t)(n_layers - 2) * P * P * 9 + (int64_t)P * C * 9;
  int64_t b = (int64_t)P * (n_layers - 1) + C;
  return w + b;
}

/* CNN residual G_eps(x) for C image channels (D_eps = Id - G_eps; C = 3 for the
 * colour DnCNN of P:843, reading R43): layer 1 is C -> P, layer K is P -> C; x and G are C planes.
 * Layer k: a^k_{c'}[i,j] = eta_k( b_k[c'] + sum_c sum_{u,v=-1..1} W_k[c'][c][u+1][v+1] a^{k-1}_c[i+u][j+v] )
 * (PyTorch conv2d cross-correlation, half padding, reading R2/R8: zero outside
 * the image at every layer input); eta = ReLU for k < K, identity for k = K.
 * weights: fp32 OIHW, layers concatenated; biases: per layer, concatenated.     */
int or_dncnn_residual_c(const double *x, int32_t ny, int32_t nx, int32_t C, int32_t n_layers, int32_t P,
                        const float *weights, const float *biases, int32_t bf16_emulate, double *G) {
  if (n_layers < 2 || P < 1 || C < 1) return OR_E_INVALID;
  int64_t npx = (int64_t)ny * nx;
  int64_t wide = P > C ? P : C;
  double *a = (double *)calloc((size_t)(npx * wide), sizeof(double));
  double *b = (double *)calloc((size_t)(npx * wide), sizeof(double));
  if (!a || !b) { free(a); free(b); return OR_E_INVALID; }
  /* a^0 = x (C channels) */
  for (int64_t n = 0; n < npx * C; n++) a[n] = bf16_emulate ? or_bf16(x[n]) : x[n];
  int cin = C;
  const float *w = weights;
  const float *bb = biases;
  for (int k = 1; k <= n_layers; k++) {
    int cout = (k == n_layers) ? C : P;
    OR_PARALLEL_ROWS2
    for (int co = 0; co < cout; co++)
      for (int i = 0; i < ny; i++)
        for (int j = 0; j < nx; j++) {
          double s = 0.0;
          for (int ci = 0; ci < cin; ci++)
            for (int u = -1; u <= 1; u++)
              for (int v = -1; v <= 1; v++) {
                int ii = i + u, jj = j + v;
                if (ii < 0 || ii >= ny || jj < 0 || jj >= nx) continue;
                double wt = (double)w[((co * cin + ci) * 3 + (u + 1)) * 3 + (v + 1)];
                if (bf16_emulate) wt = or_bf16(wt);
                s += wt * a[(int64_t)ci * npx + (int64_t)ii * nx + jj];
              }
          s += (double)bb[co];
          if (k < n_layers) {
            if (s < 0.0) s = 0.0;                 /* ReLU */
            if (bf16_emulate) s = or_bf16(s);     /* GPU stores activations as bf16 */
          }
          b[(int64_t)co * npx + (int64_t)i * nx + j] = s;
        }
    w += (int64_t)cout * cin * 9;
    bb += cout;
    double *t = a; a = b; b = t;
    cin = cout;
  }
  for (int64_t n = 0; n < npx * C; n++) G[n] = a[n];
  free(a);
  free(b);
  return OR_OK;
}

int or_dncnn_residual(const double *x, int32_t ny, int32_t nx, int32_t n_layers, int32_t P,
                      const float *weights, const float *biases, int32_t bf16_emulate, double *G) {
  return or_dncnn_residual_c(x, ny, nx, 1, n_layers, P, weights, biases, bf16_emulate, G);
}

/* ------------------------------------------------------------------ */
/* DDFB (eq:ddfb_operator P:382-385, eq:dfb_operator:T P:390-393), C = 1 image channel, P features:
 *   W_k : R^N -> R^{P x N},  (W_k v)_c[i,j] = sum_{u,v=-1..1} w_k[c][u+1][v+1] v[i+u][j+v]
 *         (PyTorch conv2d cross-correlation, zero boundary; weights [P][1][3][3], reading R39)
 *   W_k^*: its adjoint,     (W_k^* a)[i,j] = sum_c sum_{u,v} w_k[c][u+1][v+1] a_c[i-u][j-v]
 *   T_k(u) = HT( u + gamma_k W_k proj_[0,1](v - W_k^* u) ),  HT = clamp to [-ht_eps, ht_eps] (R40)
 *   D(v)   = proj_[0,1]( v - gamma_K W_K^* T_{K-1}( ... T_1( W_K v ) ) )
 * Output G = v - D(v), so that the x-update's -G term is D(v) - v.
 * bf16_emulate rounds at the GPU's points (R41): the conv weights as bf16(w_K) in u0 = W_K v,
 * bf16(gamma_k w_k) in T_k, bf16(w_k) in W_k^* (k < K), bf16(gamma_K w_K) in the final adjoint;
 * v and p at every W_k input; u after u0 and after every T_k.  Accumulation stays fp64. */
static void or_ddfb_w(const double *v, int ny, int nx, int C, int P, const float *w, double scale, int emul,
                      double *out) {
  /* (W v)_p[i,j] = sum_c sum_{u,q=-1..1} w[p][c][u+1][q+1] v_c[i+u][j+q]   (C -> P) */
  int64_t npx = (int64_t)ny * nx;
  OR_PARALLEL_ROWS2
  for (int c = 0; c < P; c++)
    for (int i = 0; i < ny; i++)
      for (int j = 0; j < nx; j++) {
        double s = 0.0;
        for (int ci = 0; ci < C; ci++)
          for (int u = -1; u <= 1; u++)
            for (int q = -1; q <= 1; q++) {
              int ii = i + u, jj = j + q;
              if (ii < 0 || ii >= ny || jj < 0 || jj >= nx) continue;
              double wt = scale * (double)w[((c * C + ci) * 3 + (u + 1)) * 3 + (q + 1)];
              if (emul) wt = or_bf16(wt);
              double a = v[(int64_t)ci * npx + (int64_t)ii * nx + jj];
              if (emul) a = or_bf16(a);
              s += wt * a;
            }
        out[(int64_t)c * npx + (int64_t)i * nx + j] = s;
      }
}

static void or_ddfb_wadj(const double *a, int ny, int nx, int C, int P, const float *w, double scale, int emul,
                         double *out) {
  /* (W^* a)_c[i,j] = sum_p sum_{u,q} w[p][c][u+1][q+1] a_p[i-u][j-q]   (P -> C, the adjoint) */
  int64_t npx = (int64_t)ny * nx;
  OR_PARALLEL_ROWS2
  for (int ci = 0; ci < C; ci++)
    for (int i = 0; i < ny; i++)
      for (int j = 0; j < nx; j++) {
        double s = 0.0;
        for (int c = 0; c < P; c++)
          for (int u = -1; u <= 1; u++)
            for (int q = -1; q <= 1; q++) {
              int ii = i - u, jj = j - q;
              if (ii < 0 || ii >= ny || jj < 0 || jj >= nx) continue;
              double wt = scale * (double)w[((c * C + ci) * 3 + (u + 1)) * 3 + (q + 1)];
              if (emul) wt = or_bf16(wt);
              s += wt * a[(int64_t)c * npx + (int64_t)ii * nx + jj];
            }
        out[(int64_t)ci * npx + (int64_t)i * nx + j] = s;
      }
}

int64_t or_ddfb_param_count(int32_t K, int32_t P, int32_t C) { return (int64_t)K * P * C * 9; }

/* C image channels (the colour DDFB of P:387: W_k : C -> P, W_k^* : P -> C; weights per layer
 * [P][C][3][3], layers concatenated).  in != NULL: only pixels with in[n] != 0 belong to the
 * image (a worker's padded crop, reading R8): u and p are zero elsewhere, exactly as the global
 * image's zero boundary. */
static int or_ddfb_masked(const double *v, int32_t ny, int32_t nx, int32_t C, int32_t K, int32_t P,
                          const float *weights, const float *gammas, double ht_eps, int32_t emul, const uint8_t *in,
                          double *G) {
  if (K < 1 || P < 1 || C < 1) return OR_E_INVALID;
  int64_t npx = (int64_t)ny * nx;
  int64_t lw = (int64_t)P * C * 9;   /* weights per layer */
  double *u = (double *)calloc((size_t)(npx * P), sizeof(double));
  double *t = (double *)calloc((size_t)(npx * P), sizeof(double));
  double *a = (double *)calloc((size_t)(npx * C), sizeof(double));
  double *pp = (double *)calloc((size_t)(npx * C), sizeof(double));
  if (!u || !t || !a || !pp) { free(u); free(t); free(a); free(pp); return OR_E_INVALID; }
  const float *wK = weights + (int64_t)(K - 1) * lw;
  or_ddfb_w(v, ny, nx, C, P, wK, 1.0, emul, u);                   /* u0 = W_K v */
  for (int64_t n = 0; n < npx * P; n++) {
    if (emul) u[n] = or_bf16(u[n]);
    if (in && !in[n % npx]) u[n] = 0.0;
  }
  for (int k = 1; k <= K - 1; k++) {                               /* u <- T_k(u) */
    const float *wk = weights + (int64_t)(k - 1) * lw;
    or_ddfb_wadj(u, ny, nx, C, P, wk, 1.0, emul, a);
    for (int64_t n = 0; n < npx * C; n++) {
      double q = v[n] - a[n];
      pp[n] = q < 0.0 ? 0.0 : (q > 1.0 ? 1.0 : q);                 /* proj_[0,1] */
      if (in && !in[n % npx]) pp[n] = 0.0;
    }
    or_ddfb_w(pp, ny, nx, C, P, wk, (double)gammas[k - 1], emul, t);
    for (int64_t n = 0; n < npx * P; n++) {
      double q = u[n] + t[n];
      q = q < -ht_eps ? -ht_eps : (q > ht_eps ? ht_eps : q);      /* HT_eps */
      u[n] = emul ? or_bf16(q) : q;
      if (in && !in[n % npx]) u[n] = 0.0;
    }
  }
  or_ddfb_wadj(u, ny, nx, C, P, wK, (double)gammas[K - 1], emul, a);  /* gamma_K W_K^* u */
  for (int64_t n = 0; n < npx * C; n++) {
    double q = v[n] - a[n];
    double d = q < 0.0 ? 0.0 : (q > 1.0 ? 1.0 : q);
    G[n] = v[n] - d;
  }
  free(u); free(t); free(a); free(pp);
  return OR_OK;
}

int or_ddfb_residual_c(const double *v, int32_t ny, int32_t nx, int32_t C, int32_t K, int32_t P,
                       const float *weights, const float *gammas, double ht_eps, int32_t emul, double *G) {
  return or_ddfb_masked(v, ny, nx, C, K, P, weights, gammas, ht_eps, emul, NULL, G);
}

int or_ddfb_residual(const double *v, int32_t ny, int32_t nx, int32_t K, int32_t P, const float *weights,
                     const float *gammas, double ht_eps, int32_t emul, double *G) {
  return or_ddfb_masked(v, ny, nx, 1, K, P, weights, gammas, ht_eps, emul, NULL, G);
}

/* ------------------------------------------------------------------ */
/* Step-size conditions eq:stepsize_cond, with ||H2||^2 read as
 * ||H2||^2/rho (reading R11).  Returns bit 0 set if the first inequality fails,
 * bit 1 if the second fails.  h2_over_rho = ||H2||^2/rho (0 when AXDA is off). */
int or_check_stepsizes(double L, double h2_over_rho, double alpha, double eps, double L_D,
                       double lambda, double gamma) {
  int bad = 0;
  double prior = (alpha > 0.0 && L_D > 0.0) ? alpha * L_D / (eps * eps) : 0.0;
  double lhs1 = 2.0 * (L + h2_over_rho) + prior;
  if (!(lhs1 <= 1.0 / (2.0 * lambda))) bad |= 1;
  double lhs2 = 3.0 * gamma * (L + h2_over_rho + 1.0 / lambda + prior);
  if (!(lhs2 < 1.0)) bad |= 2;
  return bad;
}

/* ------------------------------------------------------------------ */
/* prox_{kappa KL(y || .)}(v) = argmin_{u > 0} kappa (u - y log u) + (u - v)^2 / 2 (the Poisson
 * negative log-likelihood of eq:likelihood:poisson_deconvolution up to constants).
 * Stationarity: kappa (1 - y/u) + u - v = 0  <=>  u^2 - (v - kappa) u - kappa y = 0; the prox
 * is the non-negative root  u = ((v - kappa) + sqrt((v - kappa)^2 + 4 kappa y)) / 2
 * (y = 0: max(v - kappa, 0)).  Reading R31.                                                   */
double or_prox_kl(double v, double y, double kappa) {
  double a = v - kappa;
  return 0.5 * (a + sqrt(a * a + 4.0 * kappa * y));
}

/* ------------------------------------------------------------------ */
/* 2-D discrete gradient D, reading R35:
 *   (Dx)_v[i,j] = x[i+1,j] - x[i,j] for i < ny-1, 0 on the last row;
 *   (Dx)_h[i,j] = x[i,j+1] - x[i,j] for j < nx-1, 0 on the last column.                       */
void or_grad2d(const double *x, int32_t ny, int32_t nx, double *gv, double *gh) {
  for (int64_t i = 0; i < ny; i++)
    for (int64_t j = 0; j < nx; j++) {
      int64_t n = i * nx + j;
      gv[n] = (i < ny - 1) ? x[n + nx] - x[n] : 0.0;
      gh[n] = (j < nx - 1) ? x[n + 1] - x[n] : 0.0;
    }
}

/* D^T: (D^T g)[i,j] = g_v[i-1,j] [i >= 1] - g_v[i,j] [i < ny-1] + g_h[i,j-1] [j >= 1] - g_h[i,j] [j < nx-1]. */
void or_grad2d_adj(const double *gv, const double *gh, int32_t ny, int32_t nx, double *out) {
  for (int64_t i = 0; i < ny; i++)
    for (int64_t j = 0; j < nx; j++) {
      int64_t n = i * nx + j;
      double s = 0.0;
      if (i >= 1) s += gv[n - nx];
      if (i < ny - 1) s -= gv[n];
      if (j >= 1) s += gh[n - 1];
      if (j < nx - 1) s -= gh[n];
      out[n] = s;
    }
}

/* prox of tau ||.||_{2,1} on one pixel's 2-vector, reading R36:
 * g -> g max(0, 1 - tau / ||g||_2), 0 -> 0. */
void or_prox_l21(double gv, double gh, double tau, double *ov, double *oh) {
  double nrm = sqrt(gv * gv + gh * gh);
  double sc = (nrm > tau) ? 1.0 - tau / nrm : 0.0;
  *ov = gv * sc;
  *oh = gh * sc;
}

/* ------------------------------------------------------------------ */
typedef struct {
  int32_t ny, nx;
  int32_t op;                    /* 0 = convolution H1, 1 = mask H1 = diag(m),
                                    2 = Poisson deconvolution (f1 = 0; z1 ~ eta H x, KL prox) */
  const float *kernel;           /* kh x kw true-convolution kernel, or NULL when separable given */
  const float *ksep_y;           /* optional separable factors: k[p][q] = ksep_y[p] * ksep_x[q] */
  const float *ksep_x;
  int32_t kh, kw;
  const uint8_t *mask;           /* ny*nx, op = 1 */
  const float *y;                /* ny*nx observations */
  double sigma2;
  int32_t n_layers, channels;    /* 0 layers = no CNN prior */
  const float *weights, *biases;
  double alpha, eps;
  int32_t bf16_emulate;
  double lambda, c_lo, c_hi;     /* Moreau box term, lambda <= 0 = off */
  double rho, kappa, z_lo, z_hi; /* AXDA z-block (H2 = I, f2 = indicator of [z_lo,z_hi]); rho <= 0 = off */
  double gamma;
  const float *x0;               /* NULL = zeros */
  int64_t n_iter, burn_in;
  uint64_t seed;
  int32_t tiles_y, tiles_x;      /* <= 1 means untiled */
  int64_t i_off, j_off;          /* global coordinates of pixel (0,0) of this (cropped) image:
                                    the noise is indexed by global pixel (reading R9), so a crop
                                    of a larger image draws the same xi/zeta at the same pixel */
  double eta, rho1, kappa1;      /* op = 2: Poisson scale and the z1 block's coupling / step */
  int32_t den_kind;              /* 0 = DnCNN (weights/biases), 1 = DDFB (weights [K][P][1][3][3],
                                    ddfb_gammas[K], ht_eps; biases unused) */
  const float *ddfb_gammas;
  double ht_eps;
  double tv_beta;                /* > 0: TV prior: the z block is z ~ D x (two
                                    components) with f2 = tv_beta ||.||_{2,1} and x moves by PSGLA
                                    with p = 1_{R+}; requires rho > 0, no CNN, no box term */
  int32_t n_chan;                /* image channels C (0 or 1 = grayscale; 3 = RGB, reading R43): y, x0
                                    and every state array are C planes [C][ny][nx]; H acts on each
                                    plane, the mask is shared, channel c draws Philox streams 4c + s;
                                    C > 1: untiled, DnCNN or no prior, no TV */
} or_config;

static int or_nchan(const or_config *c) { return c->n_chan > 1 ? c->n_chan : 1; }

static void or_kernel2d(const or_config *c, double *k) {
  for (int p = 0; p < c->kh; p++)
    for (int q = 0; q < c->kw; q++)
      k[p * c->kw + q] = c->ksep_y ? (double)c->ksep_y[p] * (double)c->ksep_x[q]
                                   : (double)c->kernel[p * c->kw + q];
}

/* One untiled iteration of Algorithm 1 (lines 5-13) for one image channel (plane) on global
 * arrays, given the channel's CNN residual G; the channel draws Philox streams sb + s (R43). */
static int or_step_plane(const or_config *c, const double *k, const double *yd, uint64_t t,
                         const double *x, const double *z, const double *z1, const double *zh, double *xn,
                         double *zn, double *z1n, double *zhn, double *r, double *g, const double *G,
                         uint32_t sb) {
  int ny = c->ny, nx = c->nx;
  int64_t npx = (int64_t)ny * nx;
  /* line 6: u1 = H1^T grad f1(H1 x),  f1(v) = ||y - v||^2/(2 sigma^2) (eq:potential_gaussian_likelihood) */
  if (c->op == 0) {
    or_conv_fwd(x, ny, nx, k, c->kh, c->kw, r);
    for (int64_t n = 0; n < npx; n++) r[n] -= yd[n];
    or_conv_adj(r, ny, nx, k, c->kh, c->kw, g);
    for (int64_t n = 0; n < npx; n++) g[n] /= c->sigma2;
  } else if (c->op == 1) {
    for (int64_t n = 0; n < npx; n++) {
      double m = c->mask[n] ? 1.0 : 0.0;
      g[n] = m * (m * x[n] - yd[n]);
    }
    for (int64_t n = 0; n < npx; n++) g[n] /= c->sigma2;
  } else {
    /* op 2: f1 = 0; line 7 for the z1 block: (1/rho1) (eta H)^T (eta H x - z1) */
    or_conv_fwd(x, ny, nx, k, c->kh, c->kw, r);
    for (int64_t n = 0; n < npx; n++) r[n] = c->eta * r[n] - z1[n];
    or_conv_adj(r, ny, nx, k, c->kh, c->kw, g);
    for (int64_t n = 0; n < npx; n++) g[n] = c->eta * g[n] / c->rho1;
  }
  /* line 8: D_eps(x) - x = -G_eps(x), G given */
  int use_cnn = c->n_layers > 0 && c->alpha != 0.0;
  double sq2g = sqrt(2.0 * c->gamma);
  if (c->tv_beta > 0.0) {
    /* TV prior: x^{t+1} = proj_{R+}( x - gamma grad f1(H1 x) - (gamma/rho) D^T (D x - z)
     * + sqrt(2 gamma) xi )  (PSGLA with p = 1_{R+});  z = (z_v, z_h) = (z, z1) arrays here.      */
    double *dv = (double *)malloc(sizeof(double) * (size_t)npx);
    double *dh = (double *)malloc(sizeof(double) * (size_t)npx);
    double *dt = (double *)malloc(sizeof(double) * (size_t)npx);
    if (!dv || !dh || !dt) { free(dv); free(dh); free(dt); return OR_E_INVALID; }
    or_grad2d(x, ny, nx, dv, dh);
    for (int64_t n = 0; n < npx; n++) { dv[n] -= z[n]; dh[n] -= zh[n]; }
    or_grad2d_adj(dv, dh, ny, nx, dt);
    for (int64_t i = 0; i < ny; i++)
      for (int64_t j = 0; j < nx; j++) {
        int64_t n = i * nx + j;
        double v = x[n] - c->gamma * g[n] - (c->gamma / c->rho) * dt[n] +
                   sq2g * or_normal(c->seed, (uint32_t)(t + 1), i + c->i_off, j + c->j_off, sb + 0);
        xn[n] = v < 0.0 ? 0.0 : v;
      }
    /* lines 11-13: z^{t+1} = prox_{kappa beta ||.||_{2,1}}( z - (kappa/rho)(z - D x^{t+1}) + sqrt(2 kappa) zeta ),
     * zeta_v = stream 1, zeta_h = stream 3 (reading R37) */
    or_grad2d(xn, ny, nx, dv, dh);
    double sq2k = sqrt(2.0 * c->kappa);
    for (int64_t i = 0; i < ny; i++)
      for (int64_t j = 0; j < nx; j++) {
        int64_t n = i * nx + j;
        double vv = z[n] - (c->kappa / c->rho) * (z[n] - dv[n]) +
                    sq2k * or_normal(c->seed, (uint32_t)(t + 1), i + c->i_off, j + c->j_off, sb + 1);
        double vh = zh[n] - (c->kappa / c->rho) * (zh[n] - dh[n]) +
                    sq2k * or_normal(c->seed, (uint32_t)(t + 1), i + c->i_off, j + c->j_off, sb + 3);
        or_prox_l21(vv, vh, c->kappa * c->tv_beta, &zn[n], &zhn[n]);
      }
    free(dv); free(dh); free(dt);
  } else {
  OR_PARALLEL_ROWS
  for (int64_t i = 0; i < ny; i++)
    for (int64_t j = 0; j < nx; j++) {
      int64_t n = i * nx + j;
      /* line 10 / eq:sgs_pnp_ula_psgla:pnp_ula */
      double v = x[n] - c->gamma * g[n];
      if (c->rho > 0.0) v -= (c->gamma / c->rho) * (x[n] - z[n]);
      if (use_cnn) v += (c->alpha * c->gamma / (c->eps * c->eps)) * (-G[n]);
      if (c->lambda > 0.0) {
        double pc = x[n] < c->c_lo ? c->c_lo : (x[n] > c->c_hi ? c->c_hi : x[n]);
        v += (c->gamma / c->lambda) * (pc - x[n]);
      }
      v += sq2g * or_normal(c->seed, (uint32_t)(t + 1), i + c->i_off, j + c->j_off, sb + 0);
      xn[n] = v;
    }
  if (c->rho > 0.0) {
    double sq2k = sqrt(2.0 * c->kappa);
    for (int64_t i = 0; i < ny; i++)
      for (int64_t j = 0; j < nx; j++) {
        int64_t n = i * nx + j;
        /* lines 12-13 / eq:sgs_pnp_ula_psgla:psgla with H2 = I, prox = projection onto [z_lo,z_hi] */
        double v = z[n] - (c->kappa / c->rho) * (z[n] - xn[n]) +
                   sq2k * or_normal(c->seed, (uint32_t)(t + 1), i + c->i_off, j + c->j_off, sb + 1);
        zn[n] = v < c->z_lo ? c->z_lo : (v > c->z_hi ? c->z_hi : v);
      }
  }
  }   /* end of the non-TV x / z updates */
  if (c->op == 2) {
    /* lines 11-13 for the z1 block: H2,1 = eta H, prox of kappa1 KL(y || .), stream 2 */
    or_conv_fwd(xn, ny, nx, k, c->kh, c->kw, r);
    double sq2k1 = sqrt(2.0 * c->kappa1);
    for (int64_t i = 0; i < ny; i++)
      for (int64_t j = 0; j < nx; j++) {
        int64_t n = i * nx + j;
        double v = z1[n] - (c->kappa1 / c->rho1) * (z1[n] - c->eta * r[n]) +
                   sq2k1 * or_normal(c->seed, (uint32_t)(t + 1), i + c->i_off, j + c->j_off, sb + 2);
        z1n[n] = or_prox_kl(v, yd[n], c->kappa1);
      }
  }
  return OR_OK;
}

/* One untiled iteration on C channel planes: line 8 (the CNN couples the channels) once, then
 * lines 5-13 per channel (H, the mask, the box and the z blocks act channel by channel). */
static int or_step_global(const or_config *c, const double *k, const double *yd, uint64_t t,
                          const double *x, const double *z, const double *z1, const double *zh, double *xn,
                          double *zn, double *z1n, double *zhn, double *r, double *g, double *G) {
  const int nc = or_nchan(c);
  const int64_t npx = (int64_t)c->ny * c->nx;
  if (c->n_layers > 0 && c->alpha != 0.0) {
    int e = c->den_kind == 1
                ? or_ddfb_residual_c(x, c->ny, c->nx, nc, c->n_layers, c->channels, c->weights, c->ddfb_gammas,
                                     c->ht_eps, c->bf16_emulate, G)
                : or_dncnn_residual_c(x, c->ny, c->nx, nc, c->n_layers, c->channels, c->weights, c->biases,
                                      c->bf16_emulate, G);
    if (e) return e;
  }
  for (int ch = 0; ch < nc; ch++) {
    const int64_t o = (int64_t)ch * npx;
    int e = or_step_plane(c, k, yd + o, t, x + o, z + o, z1 + o, zh + o, xn + o, zn + o, z1n + o, zhn + o, r, g,
                          G + o, 4u * (uint32_t)ch);
    if (e) return e;
  }
  return OR_OK;
}

/* One tiled iteration: every tile b computes its block of x^{t+1}, z^{t+1}
 * from S_b x only (the tile plus a ghost frame of width h, zero outside the
 * image), exactly as worker b of Algorithm 1 would after line 5. */
static int or_step_tiled(const or_config *c, const double *k, const double *yd, uint64_t t,
                         const double *x, const double *z, const double *z1, const double *zh, double *xn,
                         double *zn, double *z1n, double *zhn) {
  int ny = c->ny, nx = c->nx;
  int ry = c->kh / 2, rx = c->kw / 2;
  int use_cnn = c->n_layers > 0 && c->alpha != 0.0;
  int hr = (c->op != 1) ? 2 * (ry > rx ? ry : rx) : 0;
  int rf = use_cnn ? (c->den_kind == 1 ? 2 * c->n_layers : c->n_layers) : 0;   /* DDFB: 2 convs per layer */
  int h = rf > hr ? rf : hr;
  if (c->tv_beta > 0.0 && h < 2) h = 2;   /* D^T D x needs x at distance 1; z on tile (+) 1 needs 2 */
  for (int ty = 0; ty < c->tiles_y; ty++)
    for (int tx = 0; tx < c->tiles_x; tx++) {
      int64_t i0, i1, j0, j1;
      or_partition(ny, c->tiles_y, ty, &i0, &i1);
      or_partition(nx, c->tiles_x, tx, &j0, &j1);
      int th = (int)(i1 - i0), tw = (int)(j1 - j0);
      if (th < h || tw < h) return OR_E_INVALID;
      int ph = th + 2 * h, pw = tw + 2 * h;
      /* S_b x: padded local copy (ghost frame from neighbours, zero outside the image) */
      double *xp = (double *)calloc((size_t)ph * pw, sizeof(double));
      double *rp = (double *)calloc((size_t)ph * pw, sizeof(double));
      double *gl = (double *)calloc((size_t)th * tw, sizeof(double));
      double *Gl = (double *)calloc((size_t)th * tw, sizeof(double));
      if (!xp || !rp || !gl || !Gl) { free(xp); free(rp); free(gl); free(Gl); return OR_E_INVALID; }
      for (int a = 0; a < ph; a++)
        for (int b = 0; b < pw; b++) {
          int64_t gi = i0 - h + a, gj = j0 - h + b;
          if (gi >= 0 && gi < ny && gj >= 0 && gj < nx) xp[(int64_t)a * pw + b] = x[gi * nx + gj];
        }
      if (c->op != 1) {
        /* residual on tile (+) r, zero outside the image (reading R7); op 2: eta H x - z1, where
         * z1 on the ring is worker b's own copy (identical values: it is computed redundantly on
         * tile (+) r_H, reading R33) */
        for (int a = h - ry; a < h + th + ry; a++)
          for (int b = h - rx; b < h + tw + rx; b++) {
            int64_t gi = i0 - h + a, gj = j0 - h + b;
            if (gi < 0 || gi >= ny || gj < 0 || gj >= nx) continue;
            double s = 0.0;
            for (int p = -ry; p <= ry; p++)
              for (int q = -rx; q <= rx; q++) {
                int64_t ii = gi - p, jj = gj - q;
                if (ii < 0 || ii >= ny || jj < 0 || jj >= nx) continue;
                s += k[(p + ry) * c->kw + (q + rx)] * xp[(a - p) * (int64_t)pw + (b - q)];
              }
            rp[(int64_t)a * pw + b] = c->op == 2 ? c->eta * s - z1[gi * nx + gj] : s - yd[gi * nx + gj];
          }
        for (int a = 0; a < th; a++)
          for (int b = 0; b < tw; b++) {
            int64_t gi = i0 + a, gj = j0 + b;
            double s = 0.0;
            for (int p = -ry; p <= ry; p++)
              for (int q = -rx; q <= rx; q++) {
                int64_t ii = gi + p, jj = gj + q;
                if (ii < 0 || ii >= ny || jj < 0 || jj >= nx) continue;
                s += k[(p + ry) * c->kw + (q + rx)] * rp[(a + h + p) * (int64_t)pw + (b + h + q)];
              }
            gl[(int64_t)a * tw + b] = s;
          }
      } else {
        for (int a = 0; a < th; a++)
          for (int b = 0; b < tw; b++) {
            int64_t n = (i0 + a) * nx + (j0 + b);
            double m = c->mask[n] ? 1.0 : 0.0;
            gl[(int64_t)a * tw + b] = m * (m * xp[(int64_t)(a + h) * pw + (b + h)] - yd[n]);
          }
      }
      for (int64_t n = 0; n < (int64_t)th * tw; n++)
        gl[n] = c->op == 2 ? c->eta * gl[n] / c->rho1 : gl[n] / c->sigma2;
      if (use_cnn && c->den_kind == 1) {
        /* DDFB on the worker's padded crop with the image mask; tile pixels are >= 2K from the
         * crop edge, so they see exactly the global computation */
        uint8_t *inm = (uint8_t *)calloc((size_t)ph * pw, 1);
        double *Gp = (double *)calloc((size_t)ph * pw, sizeof(double));
        if (!inm || !Gp) { free(inm); free(Gp); free(xp); free(rp); free(gl); free(Gl); return OR_E_INVALID; }
        for (int a = 0; a < ph; a++)
          for (int b = 0; b < pw; b++) {
            int64_t gi = i0 - h + a, gj = j0 - h + b;
            inm[(int64_t)a * pw + b] = (gi >= 0 && gi < ny && gj >= 0 && gj < nx) ? 1 : 0;
          }
        int e = or_ddfb_masked(xp, ph, pw, 1, c->n_layers, c->channels, c->weights, c->ddfb_gammas, c->ht_eps,
                               c->bf16_emulate, inm, Gp);
        for (int a = 0; a < th; a++)
          for (int b = 0; b < tw; b++) Gl[(int64_t)a * tw + b] = Gp[(int64_t)(a + h) * pw + (b + h)];
        free(inm); free(Gp);
        if (e) { free(xp); free(rp); free(gl); free(Gl); return e; }
      } else if (use_cnn) {
        /* receptive-field strategy: layer k is evaluated on tile (+) (K-k),
         * activations outside the image are zero at every layer input (reading R8). */
        int K = c->n_layers, P = c->channels;
        double *A = (double *)calloc((size_t)ph * pw * P, sizeof(double));
        double *B = (double *)calloc((size_t)ph * pw * P, sizeof(double));
        if (!A || !B) { free(A); free(B); free(xp); free(rp); free(gl); free(Gl); return OR_E_INVALID; }
        int64_t plane = (int64_t)ph * pw;
        for (int64_t n = 0; n < plane; n++) A[n] = c->bf16_emulate ? or_bf16(xp[n]) : xp[n];
        const float *w = c->weights;
        const float *bb = c->biases;
        int cin = 1;
        for (int kk = 1; kk <= K; kk++) {
          int cout = (kk == K) ? 1 : P;
          int ext = K - kk;
          memset(B, 0, sizeof(double) * (size_t)plane * P);
          OR_PARALLEL_ROWS2
          for (int co = 0; co < cout; co++)
            for (int a = h - ext; a < h + th + ext; a++)
              for (int b = h - ext; b < h + tw + ext; b++) {
                int64_t gi = i0 - h + a, gj = j0 - h + b;
                if (gi < 0 || gi >= ny || gj < 0 || gj >= nx) continue; /* stays 0 */
                double s = 0.0;
                for (int ci = 0; ci < cin; ci++)
                  for (int u = -1; u <= 1; u++)
                    for (int v = -1; v <= 1; v++) {
                      int64_t ii = gi + u, jj = gj + v;
                      if (ii < 0 || ii >= ny || jj < 0 || jj >= nx) continue;
                      double wt = (double)w[((co * cin + ci) * 3 + (u + 1)) * 3 + (v + 1)];
                      if (c->bf16_emulate) wt = or_bf16(wt);
                      s += wt * A[(int64_t)ci * plane + (int64_t)(a + u) * pw + (b + v)];
                    }
                s += (double)bb[co];
                if (kk < K) {
                  if (s < 0.0) s = 0.0;
                  if (c->bf16_emulate) s = or_bf16(s);
                }
                B[(int64_t)co * plane + (int64_t)a * pw + b] = s;
              }
          w += (int64_t)cout * cin * 9;
          bb += cout;
          double *tt = A; A = B; B = tt;
          cin = cout;
        }
        for (int a = 0; a < th; a++)
          for (int b = 0; b < tw; b++) Gl[(int64_t)a * tw + b] = A[(int64_t)(a + h) * pw + (b + h)];
        free(A);
        free(B);
      }
      double sq2g = sqrt(2.0 * c->gamma);
      if (c->tv_beta > 0.0) {
        /* TV: worker b evaluates D^T (D x - z) on its tile from S_b x and the ring of z (R38) */
        for (int a = 0; a < th; a++)
          for (int b = 0; b < tw; b++) {
            int64_t gi = i0 + a, gj = j0 + b, n = gi * nx + gj;
            const double *xc = xp + (int64_t)(a + h) * pw + (b + h);
            double s = 0.0;
            if (gi >= 1) s += (xc[0] - xc[-pw]) - z[n - nx];          /* g_v[i-1,j] */
            if (gi < ny - 1) s -= (xc[pw] - xc[0]) - z[n];            /* g_v[i,j]   */
            if (gj >= 1) s += (xc[0] - xc[-1]) - zh[n - 1];           /* g_h[i,j-1] */
            if (gj < nx - 1) s -= (xc[1] - xc[0]) - zh[n];            /* g_h[i,j]   */
            double v = xc[0] - c->gamma * gl[(int64_t)a * tw + b] - (c->gamma / c->rho) * s +
                       sq2g * or_normal(c->seed, (uint32_t)(t + 1), gi + c->i_off, gj + c->j_off, 0);
            xn[n] = v < 0.0 ? 0.0 : v;
          }
        free(xp); free(rp); free(gl); free(Gl);
        continue;
      }
      for (int a = 0; a < th; a++)
        for (int b = 0; b < tw; b++) {
          int64_t gi = i0 + a, gj = j0 + b, n = gi * nx + gj;
          double xv = xp[(int64_t)(a + h) * pw + (b + h)];
          double v = xv - c->gamma * gl[(int64_t)a * tw + b];
          if (c->rho > 0.0) v -= (c->gamma / c->rho) * (xv - z[n]);
          if (use_cnn) v += (c->alpha * c->gamma / (c->eps * c->eps)) * (-Gl[(int64_t)a * tw + b]);
          if (c->lambda > 0.0) {
            double pc = xv < c->c_lo ? c->c_lo : (xv > c->c_hi ? c->c_hi : xv);
            v += (c->gamma / c->lambda) * (pc - xv);
          }
          v += sq2g * or_normal(c->seed, (uint32_t)(t + 1), gi + c->i_off, gj + c->j_off, 0);
          xn[n] = v;
          if (c->rho > 0.0) {
            double zv = z[n] - (c->kappa / c->rho) * (z[n] - v) +
                        sqrt(2.0 * c->kappa) * or_normal(c->seed, (uint32_t)(t + 1), gi + c->i_off, gj + c->j_off, 1);
            zn[n] = zv < c->z_lo ? c->z_lo : (zv > c->z_hi ? c->z_hi : zv);
          }
        }
      free(xp);
      free(rp);
      free(gl);
      free(Gl);
    }
  if (c->tv_beta > 0.0) {
    /* line 11: S_{2,b} x^{t+1} (ghost width 1); lines 12-13 for the worker's block of z = D x */
    double sq2k = sqrt(2.0 * c->kappa);
    for (int ty = 0; ty < c->tiles_y; ty++)
      for (int tx = 0; tx < c->tiles_x; tx++) {
        int64_t i0, i1, j0, j1;
        or_partition(ny, c->tiles_y, ty, &i0, &i1);
        or_partition(nx, c->tiles_x, tx, &j0, &j1);
        for (int64_t gi = i0; gi < i1; gi++)
          for (int64_t gj = j0; gj < j1; gj++) {
            int64_t n = gi * nx + gj;
            double dv = (gi < ny - 1) ? xn[n + nx] - xn[n] : 0.0;
            double dh = (gj < nx - 1) ? xn[n + 1] - xn[n] : 0.0;
            double vv = z[n] - (c->kappa / c->rho) * (z[n] - dv) +
                        sq2k * or_normal(c->seed, (uint32_t)(t + 1), gi + c->i_off, gj + c->j_off, 1);
            double vh = zh[n] - (c->kappa / c->rho) * (zh[n] - dh) +
                        sq2k * or_normal(c->seed, (uint32_t)(t + 1), gi + c->i_off, gj + c->j_off, 3);
            or_prox_l21(vv, vh, c->kappa * c->tv_beta, &zn[n], &zhn[n]);
          }
      }
  }
  if (c->op == 2) {
    /* line 11: every worker retrieves S_{2,b} x^{t+1} (its tile plus a ghost frame of width
     * r_H) once all blocks of x^{t+1} exist; lines 12-13 for its block of z1 */
    double sq2k1 = sqrt(2.0 * c->kappa1);
    for (int ty = 0; ty < c->tiles_y; ty++)
      for (int tx = 0; tx < c->tiles_x; tx++) {
        int64_t i0, i1, j0, j1;
        or_partition(ny, c->tiles_y, ty, &i0, &i1);
        or_partition(nx, c->tiles_x, tx, &j0, &j1);
        int th = (int)(i1 - i0), tw = (int)(j1 - j0);
        int ph = th + 2 * ry, pw = tw + 2 * rx;
        double *xp = (double *)calloc((size_t)ph * pw, sizeof(double));
        if (!xp) return OR_E_INVALID;
        for (int a = 0; a < ph; a++)
          for (int b = 0; b < pw; b++) {
            int64_t gi = i0 - ry + a, gj = j0 - rx + b;
            if (gi >= 0 && gi < ny && gj >= 0 && gj < nx) xp[(int64_t)a * pw + b] = xn[gi * nx + gj];
          }
        for (int a = 0; a < th; a++)
          for (int b = 0; b < tw; b++) {
            int64_t gi = i0 + a, gj = j0 + b, n = gi * nx + gj;
            double s = 0.0;
            for (int p = -ry; p <= ry; p++)
              for (int q = -rx; q <= rx; q++)
                s += k[(p + ry) * c->kw + (q + rx)] * xp[(int64_t)(a + ry - p) * pw + (b + rx - q)];
            double v = z1[n] - (c->kappa1 / c->rho1) * (z1[n] - c->eta * s) +
                       sq2k1 * or_normal(c->seed, (uint32_t)(t + 1), gi + c->i_off, gj + c->j_off, 2);
            z1n[n] = or_prox_kl(v, yd[n], c->kappa1);
          }
        free(xp);
      }
  }
  return OR_OK;
}

/* Full chain.  Outputs (each ny*nx, any may be NULL): final x, final z (the H2 = I block, or
 * the vertical component of z ~ D x for TV), final z1 (op = 2), final z_h (TV horizontal), MMSE mean and variance (M2/(n-1), reading R15) of x^{(t)},
 * t = burn_in+1..n_iter (reading R14), accumulated with Welford's update (P:839 footnote). */
int or_run_ex(const or_config *c, double *x_out, double *z_out, double *z1_out, double *zh_out,
              double *mean_out, double *var_out, int64_t *n_samples) {
  if (c->ny <= 0 || c->nx <= 0 || c->gamma <= 0.0) return OR_E_INVALID;
  if (c->op != 2 && c->sigma2 <= 0.0) return OR_E_INVALID;
  if (c->op != 1 && (c->kh % 2 == 0 || c->kw % 2 == 0)) return OR_E_INVALID;
  if (c->rho > 0.0 && !(c->kappa > 0.0 && c->kappa < c->rho)) return OR_E_INVALID;
  if (c->op == 2 && !(c->eta > 0.0 && c->rho1 > 0.0 && c->kappa1 > 0.0 && c->kappa1 < c->rho1))
    return OR_E_INVALID;
  if (c->tv_beta > 0.0 && (!(c->rho > 0.0) || (c->n_layers > 0 && c->alpha != 0.0) || c->lambda > 0.0))
    return OR_E_INVALID;   /* TV: z block on (the TV block), no CNN, no box term; any likelihood */
  const int nc = or_nchan(c);
  if (nc > 1 && (c->tiles_y > 1 || c->tiles_x > 1)) return OR_E_INVALID;   /* tiled mode: C = 1 */
  int64_t npx = (int64_t)c->ny * c->nx * nc;   /* all C planes */
  double *k = (double *)calloc((size_t)(c->kh > 0 ? c->kh * c->kw : 1), sizeof(double));
  double *yd = (double *)malloc(sizeof(double) * (size_t)npx);
  double *x = (double *)calloc((size_t)npx, sizeof(double));
  double *xn = (double *)calloc((size_t)npx, sizeof(double));
  double *z = (double *)calloc((size_t)npx, sizeof(double));
  double *zn = (double *)calloc((size_t)npx, sizeof(double));
  double *z1 = (double *)calloc((size_t)npx, sizeof(double));
  double *z1n = (double *)calloc((size_t)npx, sizeof(double));
  double *zh = (double *)calloc((size_t)npx, sizeof(double));
  double *zhn = (double *)calloc((size_t)npx, sizeof(double));
  double *r = (double *)calloc((size_t)npx, sizeof(double));
  double *g = (double *)calloc((size_t)npx, sizeof(double));
  double *G = (double *)calloc((size_t)npx, sizeof(double));
  double *mu = (double *)calloc((size_t)npx, sizeof(double));
  double *m2 = (double *)calloc((size_t)npx, sizeof(double));
  int err = OR_OK;
  if (!k || !yd || !x || !xn || !z || !zn || !z1 || !z1n || !zh || !zhn || !r || !g || !G || !mu || !m2) {
    err = OR_E_INVALID;
    goto done;
  }
  if (c->op != 1) or_kernel2d(c, k);
  for (int64_t n = 0; n < npx; n++) {
    yd[n] = (double)c->y[n];
    x[n] = c->x0 ? (double)c->x0[n] : 0.0;   /* x^0 */
  }                                           /* z^0 = 0 */
  int64_t cnt = 0;
  for (int64_t t = 0; t < c->n_iter; t++) {
    if (c->tiles_y > 1 || c->tiles_x > 1)
      err = or_step_tiled(c, k, yd, (uint64_t)t, x, z, z1, zh, xn, zn, z1n, zhn);
    else
      err = or_step_global(c, k, yd, (uint64_t)t, x, z, z1, zh, xn, zn, z1n, zhn, r, g, G);
    if (err) goto done;
    if (t + 1 > c->burn_in) {
      cnt++;
      for (int64_t n = 0; n < npx; n++) {
        double d = xn[n] - mu[n];
        mu[n] += d / (double)cnt;
        m2[n] += d * (xn[n] - mu[n]);
      }
    }
    double *tt = x; x = xn; xn = tt;
    if (c->rho > 0.0) { tt = z; z = zn; zn = tt; }
    if (c->op == 2) { tt = z1; z1 = z1n; z1n = tt; }
    if (c->tv_beta > 0.0) { tt = zh; zh = zhn; zhn = tt; }
  }
  if (x_out) memcpy(x_out, x, sizeof(double) * (size_t)npx);
  if (z_out) memcpy(z_out, z, sizeof(double) * (size_t)npx);
  if (z1_out) memcpy(z1_out, z1, sizeof(double) * (size_t)npx);
  if (zh_out) memcpy(zh_out, zh, sizeof(double) * (size_t)npx);
  if (n_samples) *n_samples = cnt;
  if (mean_out) {
    if (cnt < 1) { err = OR_E_STATS_EMPTY; goto done; }
    memcpy(mean_out, mu, sizeof(double) * (size_t)npx);
  }
  if (var_out) {
    if (cnt < 2) { err = OR_E_STATS_EMPTY; goto done; }
    for (int64_t n = 0; n < npx; n++) var_out[n] = m2[n] / (double)(cnt - 1);
  }
done:
  free(k); free(yd); free(x); free(xn); free(z); free(zn); free(z1); free(z1n); free(zh); free(zhn);
  free(r); free(g); free(G); free(mu); free(m2);
  return err;
}

int or_run(const or_config *c, double *x_out, double *z_out, double *mean_out, double *var_out,
           int64_t *n_samples) {
  return or_run_ex(c, x_out, z_out, NULL, NULL, mean_out, var_out, n_samples);
}
