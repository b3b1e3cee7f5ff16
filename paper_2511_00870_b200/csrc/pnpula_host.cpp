// pnpula_host.cpp -- host runtime of libpnpula: validation, Cartesian tiling with
// ghost frames (Def. 1), device buffer ownership, NCCL halo
// exchange (Alg. 1 line 5, grouped as in P:674), the iteration loop of
// Algorithm 1 and moment gathering.  Implements include/pnpula.h.
#include "pnpula.h"

#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <mutex>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "internal.h"

using namespace pnpula;

namespace {

thread_local std::string g_last_error;

void set_error(const char *fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
}

int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

struct TileDev {
  int index;               // global row-major tile index
  TileGeom g;
  float *x[2] = {nullptr, nullptr};
  float *x0 = nullptr;     // padded x0 (interior), ghost frame zero
  float *y = nullptr;
  uint8_t *mask = nullptr;
  float *z = nullptr, *mean = nullptr, *m2 = nullptr, *G = nullptr;
  float *z1 = nullptr;     // OP_POISSON: z1 block, valid on tile (+) r_H (reading R33)
  float *zh = nullptr;     // TV prior: horizontal component z_h of z ~ D x (z_v lives in z)
  float *pbuf = nullptr;   // DDFB: p = proj(v - W_k^* u), fp32 padded geometry, zero outside the image
  float *pbuf2 = nullptr;  // DDFB fused launches: p alternates between pbuf and pbuf2
  uint16_t *act[2] = {nullptr, nullptr};   // inter-chunk activations
};

struct CnnChunk {
  int l0, nl;               // first layer (1-based), number of layers
  int ext;                  // output region = tile (+) ext
};

struct Timer {
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
  size_t used = 0;
  double ms = 0.0;
  int64_t launches = 0;
};

}  // namespace

struct pnpula_ctx {
  // configuration (host copies of scalars)
  int ny = 0, nx = 0, tiles_y = 1, tiles_x = 1, rank = 0, world = 1, device = 0;
  int op = 0, kh = 0, kw = 0, ry = 0, rx = 0, separable = 0;
  std::vector<float> k2d, ky, kx;
  double sigma2 = 1, alpha = 0, eps = 1, lambda = 0, c_lo = 0, c_hi = 1, rho = 0, kappa = 0,
         z_lo = 0, z_hi = 0, gamma = 0;
  double eta = 1, rho1 = 0, kappa1 = 0;   // OP_POISSON
  double tv_beta = 0;                     // > 0: TV prior (z = (z_v, z_h) ~ D x in td.z, td.z1)
  int flags = 0;
  int n_layers = 0, channels = 0;   // 0 layers = no CNN
  int den_kind = 0;                 // PNPULA_DEN_DNCNN / PNPULA_DEN_DDFB
  int nc = 1;                       // image channels (R43): state buffers hold nc planes
  double ht_eps = 0;
  // DDFB operator images (R39-R42): W_K (im2col) for u0, gamma_k W_k (im2col) for T_k,
  // flipped W_k (folded P -> 1) for W_k^*, flipped gamma_K W_K for the final adjoint
  uint16_t *ddfb_u0 = nullptr, *ddfb_fin = nullptr;
  std::vector<uint16_t *> ddfb_t, ddfb_adj;
  int h = 0;

  cudaStream_t stream = nullptr;
  bool own_stream = false;
  ncclComm_t comm = nullptr;
  int num_sms = 148;
  int *d_err = nullptr;

  int ntiles = 0, n_local = 0, first_tile = 0;
  std::vector<TileDev> tiles;
  pnpula_rect bbox{};

  // CNN
  std::vector<CnnChunk> chunks;
  std::vector<uint16_t *> d_w;      // per layer packed weights
  std::vector<float *> d_b;         // per layer biases
  std::vector<std::vector<float>> h_b;   // host copies (passed to the CNN kernel as parameters)

  // halo plan
  std::vector<pnpula_halo_msg> msgs;
  CopyJob *d_local_jobs[2] = {nullptr, nullptr};
  int n_local_jobs = 0, max_local = 0;
  CopyJob *d_pack_jobs[2] = {nullptr, nullptr}, *d_unpack_jobs[2] = {nullptr, nullptr};
  int n_pack = 0, n_unpack = 0, max_pack = 0, max_unpack = 0;
  float *d_sendbuf = nullptr, *d_recvbuf = nullptr;
  struct PeerMsg { int peer; size_t off, count; };
  std::vector<PeerMsg> sends, recvs;

  // chain state
  int cur = 0;
  int64_t t = 0, burn_in = 0;
  uint64_t seed = 0;
  bool have_reset = false;
  bool poisoned = false;

  // device scratch reused by the result gathers (no cudaMalloc/cudaFree per call)
  void *scratch = nullptr;
  size_t scratch_bytes = 0;
  void *gather_buf = nullptr;   // root: remote tiles of a GLOBAL_ON_ROOT gather (grown on demand)
  size_t gather_bytes = 0;

  // timing
  bool timing = false;
  Timer tm_cnn, tm_update, tm_halo;
  int64_t n_launches = 0;   // kernels of this library launched (all classes)
  bool traced = false;      // PNPULA_CNN_TRACE written

  // CUDA graphs of one iteration, one per x-buffer parity (see step())
  IterState *d_iter = nullptr;     // [2], see IterState
  cudaGraphExec_t gexec[2] = {nullptr, nullptr};
  int64_t glaunches[2] = {0, 0};   // kernels per replay
  int64_t dev_t = -1;              // iteration count held by d_iter (-1: unknown)
  bool graphs_off = false;         // PNPULA_FLAG_NO_GRAPH or PNPULA_GRAPHS=0
  bool warm = false;               // one direct iteration done (modules loaded, attributes set)

  // halo-exchange overlap (row-strip tiles with NCCL messages): boundary bands first, then the
  // exchange on comm_stream concurrently with the interior update
  bool overlap = false;
  // x / z / moment update fused into the last CNN chunk (cnn_kernels.cu, FU): DnCNN, C = 1,
  // P = 32, separable 5x5 / 9x9 conv (or Poisson's x step) or mask, nets of more than one chunk
  // (the last chunk's producer warps run the update).  Env PNPULA_FUSE=1 at create.
  bool fuse = false;
  int cnn_contig = 1;              // contiguous CNN work ranges where the cost model prefers them (PNPULA_CNN_CONTIG=0: off)
  int pdl = 1;                     // CNN launches as programmatic dependents (internal.h pdl_wait)
  cudaMemPool_t pool = nullptr;    // stream-ordered pool of the per-tile buffers (see dmalloc)
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_bands = nullptr, ev_halo = nullptr;
};

namespace {

pnpula_status fail_cuda(pnpula_ctx *c, cudaError_t e, const char *what, int line) {
  set_error("CUDA error %s (%d) in %s (pnpula_host.cpp:%d)", cudaGetErrorString(e), (int)e, what, line);
  if (c) c->poisoned = true;
  return PNPULA_E_CUDA;
}
pnpula_status fail_nccl(pnpula_ctx *c, ncclResult_t e, const char *what, int line) {
  set_error("NCCL error %s (%d) in %s (pnpula_host.cpp:%d)", ncclGetErrorString(e), (int)e, what, line);
  if (c) c->poisoned = true;
  return PNPULA_E_NCCL;
}

#define CU(c, expr)                                                       \
  do {                                                                    \
    cudaError_t _e = (expr);                                              \
    if (_e != cudaSuccess) return fail_cuda((c), _e, #expr, __LINE__);   \
  } while (0)
#define NC(c, expr)                                                       \
  do {                                                                    \
    ncclResult_t _e = (expr);                                             \
    if (_e != ncclSuccess) return fail_nccl((c), _e, #expr, __LINE__);    \
  } while (0)

void timer_begin(pnpula_ctx *c, Timer &t, cudaEvent_t *end_out, cudaStream_t st = nullptr) {
  *end_out = nullptr;
  if (!c->timing) return;
  if (t.used == t.ev.size()) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    t.ev.push_back({a, b});
  }
  cudaEventRecord(t.ev[t.used].first, st ? st : c->stream);
  *end_out = t.ev[t.used].second;
  t.used++;
}
void timer_end(pnpula_ctx *c, cudaEvent_t end, cudaStream_t st = nullptr) {
  if (end) cudaEventRecord(end, st ? st : c->stream);
}
void timer_collect(Timer &t) {
  for (size_t i = 0; i < t.used; ++i) {
    float ms = 0.f;
    cudaEventSynchronize(t.ev[i].second);
    cudaEventElapsedTime(&ms, t.ev[i].first, t.ev[i].second);
    t.ms += ms;
    t.launches++;
  }
  t.used = 0;
}

TileGeom make_geom(int i0, int j0, int th, int tw, int h) {
  TileGeom g;
  g.i0 = i0; g.j0 = j0; g.th = th; g.tw = tw; g.h = h;
  g.hx = (int)round_up(std::max(h, 1), 4) + (j0 & 3);
  g.ph = th + 2 * h;
  g.pitch = (int)round_up(g.hx + tw + std::max(h, 4), 32);
  return g;
}

size_t geom_elems(const TileGeom &g) { return (size_t)g.ph * g.pitch; }

// Per-tile state buffers come from a process-wide stream-ordered pool per device that keeps
// freed memory (release threshold = max): a context created after another was destroyed reuses
// its memory without driver calls (fresh cudaMalloc of GBs stalls for 20-160 ms, measured).
// Allocation and first use are ordered on the context stream.  PNPULA_POOL=0: plain cudaMalloc.
cudaMemPool_t device_pool(int dev) {
  static cudaMemPool_t pools[64] = {};
  static std::mutex mu;
  if (dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  if (!pools[dev]) {
    cudaMemPoolProps pr{};
    pr.allocType = cudaMemAllocationTypePinned;
    pr.location.type = cudaMemLocationTypeDevice;
    pr.location.id = dev;
    if (cudaMemPoolCreate(&pools[dev], &pr) != cudaSuccess) { pools[dev] = nullptr; return nullptr; }
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &thr);
  }
  return pools[dev];
}
template <typename T>
cudaError_t dmalloc(pnpula_ctx *c, T **p, size_t bytes) {
  if (c->pool) return cudaMallocFromPoolAsync(reinterpret_cast<void **>(p), bytes, c->pool, c->stream);
  return cudaMalloc(reinterpret_cast<void **>(p), bytes);
}
void dfree(pnpula_ctx *c, void *p) {
  if (!p) return;
  if (c->pool) cudaFreeAsync(p, c->stream);
  else cudaFree(p);
}

void tile_rect(int ny, int nx, int ty_n, int tx_n, int tile, pnpula_rect *r) {
  int64_t a, b, c, d;
  pnpula_partition(ny, ty_n, tile / tx_n, &a, &b);
  pnpula_partition(nx, tx_n, tile % tx_n, &c, &d);
  r->i0 = (int)a; r->h = (int)(b - a); r->j0 = (int)c; r->w = (int)(d - c);
}

pnpula_status check_ctx(pnpula_ctx *c) {
  if (!c) { set_error("null context"); return PNPULA_E_INVALID_ARG; }
  if (c->poisoned) { set_error("context poisoned by an earlier CUDA/NCCL error"); return PNPULA_E_STATE; }
  return PNPULA_OK;
}

// copy a host rectangle (row-major, rect r of in_rect) into padded device buffer rows
template <typename T>
pnpula_status upload_padded(pnpula_ctx *c, T *dst, const TileGeom &g, const T *host,
                            const pnpula_rect &in, int i0, int j0, int hgt, int wid) {
  // region [i0, i0+hgt) x [j0, j0+wid) (global), clipped to the image and to in_rect
  int a0 = std::max({i0, 0, in.i0}), a1 = std::min({i0 + hgt, c->ny, in.i0 + in.h});
  int b0 = std::max({j0, 0, in.j0}), b1 = std::min({j0 + wid, c->nx, in.j0 + in.w});
  if (a0 >= a1 || b0 >= b1) return PNPULA_OK;
  const T *src = host + (size_t)(a0 - in.i0) * in.w + (b0 - in.j0);
  T *d = dst + (size_t)(a0 - (g.i0 - g.h)) * g.pitch + (b0 - (g.j0 - g.hx));
  CU(c, cudaMemcpy2DAsync(d, (size_t)g.pitch * sizeof(T), src, (size_t)in.w * sizeof(T),
                          (size_t)(b1 - b0) * sizeof(T), (size_t)(a1 - a0), cudaMemcpyHostToDevice, c->stream));
  return PNPULA_OK;
}

// DDFB (R39-R42): K two-operator launches per tile (cnn_chunk_kernel<P, 2>: an im2col 1 -> P
// layer feeding a folded P -> 1 layer through shared memory), on shrinking regions tile (+) e:
//   j = 0:      u0 = W_K v (e = 2K-1, also stored)          -> p1 = proj(v - W_1^* u0) (e = 2K-2)
//   0 < j < K:  u_j = HT(u_{j-1} + gamma_j W_j p_j) (stored) -> p_{j+1} = proj(v - W_{j+1}^* u_j)
//   j = K-1:    the folded layer is G = v - proj(v - gamma_K W_K^* u_{K-1}) (e = 0)
// (output extents e = 2K-2-2j; u_j on e+1).  p alternates between pbuf / pbuf2 and u between the
// two activation buffers, so no launch reads what it writes.
pnpula_status run_ddfb(pnpula_ctx *c, int buf) {
  const int K = c->n_layers, P = c->channels;
  for (auto &td : c->tiles) {
    const TileGeom &g = td.g;
    int cur = 0;              // act buffer receiving u_j
    float *pin = nullptr;     // p_j (im2col input of launch j > 0)
    for (int j = 0; j < K; ++j) {
      const int e = 2 * K - 2 - 2 * j;   // output extent; u_j on e + 1
      CnnChunkParams p{};
      p.P = P;
      p.nl = 2;
      p.nc = c->nc;                                        // colour: W_k C -> P, W_k^* P -> C
      p.xcs = p.gcs = (int64_t)geom_elems(g);
      p.first_is_input = 1;
      p.last_is_output = 1;
      p.mode0 = j == 0 ? 1 : 3;
      p.mode = j == K - 1 ? 4 : 2;
      p.ht_eps = (float)c->ht_eps;
      p.w[0] = j == 0 ? c->ddfb_u0 : c->ddfb_t[j - 1];
      p.w[1] = j == K - 1 ? c->ddfb_fin : c->ddfb_adj[j];
      p.x = j == 0 ? td.x[buf] : pin;   // im2col input: v, then p_j
      p.xv = td.x[buf];
      p.xg = g;
      p.oi0 = g.i0 - e; p.oj0 = g.j0 - e;
      p.oh = g.th + 2 * e; p.ow = g.tw + 2 * e;
      if (j > 0) {             // u_{j-1} on tile (+) e + 3 (read at the pixel by mode 3)
        p.ain = td.act[cur ^ 1];
        p.a_i0 = g.i0 - (e + 3); p.a_j0 = g.j0 - (e + 3);
        p.a_rows = g.th + 2 * (e + 3); p.a_cols = g.tw + 2 * (e + 3);
      }
      p.aout = td.act[cur];     // u_j on tile (+) e + 1
      p.o_i0 = g.i0 - (e + 1); p.o_j0 = g.j0 - (e + 1);
      p.o_rows = g.th + 2 * (e + 1); p.o_cols = g.tw + 2 * (e + 1);
      float *pout = (j % 2 == 0) ? td.pbuf : td.pbuf2;
      p.G = j == K - 1 ? td.G : pout;
      p.gg = g;
      p.ny = c->ny; p.nx = c->nx;
      p.err = c->d_err;
      p.pdl = c->pdl;   // (row-block units: the contiguous ranges measured 1 % slower for DDFB, d5)
      cudaEvent_t end;
      timer_begin(c, c->tm_cnn, &end);
      CU(c, launch_cnn_chunk(p, c->num_sms, c->stream));
      c->n_launches++;
      timer_end(c, end);
      pin = pout;
      cur ^= 1;
    }
  }
  return PNPULA_OK;
}

UpdateParams make_update_params(pnpula_ctx *c, TileDev &td, int buf);

// fused: the last chunk also performs the x / z / moment update of the step reading x[buf]
// (FU, c->fuse; iteration scalars as enqueue_step's update_rows: t1 by value or `it`), and G is
// not stored.  Not fused: G for the update kernels (or pnpula_get_denoiser_residual).
pnpula_status run_cnn(pnpula_ctx *c, int buf, bool fused = false, const IterState *it = nullptr) {
  if (c->den_kind == PNPULA_DEN_DDFB) return run_ddfb(c, buf);
  for (auto &td : c->tiles) {
    for (size_t ci = 0; ci < c->chunks.size(); ++ci) {
      const CnnChunk &ch = c->chunks[ci];
      CnnChunkParams p{};
      p.P = c->channels;
      p.nl = ch.nl;
      p.first_is_input = ch.l0 == 1;
      p.last_is_output = ch.l0 + ch.nl - 1 == c->n_layers;
      for (int l = 0; l < ch.nl; ++l) {
        p.w[l] = c->d_w[ch.l0 - 1 + l];
        const std::vector<float> &hb = c->h_b[ch.l0 - 1 + l];
        for (size_t k = 0; k < hb.size() && k < 64; ++k) p.bias[l][k] = hb[k];
      }
      const TileGeom &g = td.g;
      p.x = td.x[buf];
      p.xg = g;
      const int ein = ch.ext + ch.nl;
      if (!p.first_is_input) {
        p.ain = td.act[(ci + 1) & 1];
        p.a_i0 = g.i0 - ein; p.a_j0 = g.j0 - ein;
        p.a_rows = g.th + 2 * ein; p.a_cols = g.tw + 2 * ein;
      }
      p.oi0 = g.i0 - ch.ext; p.oj0 = g.j0 - ch.ext;
      p.oh = g.th + 2 * ch.ext; p.ow = g.tw + 2 * ch.ext;
      if (!p.last_is_output) {
        p.aout = td.act[ci & 1];
        p.o_i0 = p.oi0; p.o_j0 = p.oj0; p.o_rows = p.oh; p.o_cols = p.ow;
      } else {
        p.G = td.G;
        p.gg = g;
        if (fused) {
          const uint64_t t1 = (uint64_t)c->t + 1;
          const bool acc = (int64_t)t1 > c->burn_in;
          const double k = acc ? (double)((int64_t)t1 - c->burn_in) : 1.0;
          p.fuse = 1;
          p.up = make_update_params(c, td, buf);
          p.up.t1 = (uint32_t)t1;
          p.up.accumulate = acc;
          p.up.inv_n = (float)(1.0 / k);
          p.up.it = it;
          p.up.it_next = (it && &td == &c->tiles[0]) ? c->d_iter + (buf ^ 1) : nullptr;
        }
      }
      p.ny = c->ny; p.nx = c->nx;
      p.nc = c->nc;
      p.xcs = p.gcs = (int64_t)geom_elems(g);
      p.err = c->d_err;
      p.pdl = c->pdl;
      p.contig = c->cnn_contig;
      // optional pipeline trace of the first evaluation (diagnostics; env PNPULA_CNN_TRACE=<path prefix>)
      const char *trace_path = getenv("PNPULA_CNN_TRACE");
      unsigned long long *d_trace = nullptr;
      if (trace_path && !c->traced) {
        CU(c, cudaMalloc(&d_trace, sizeof(unsigned long long) << 21));
        CU(c, cudaMemsetAsync(d_trace, 0, sizeof(unsigned long long) << 21, c->stream));
        p.trace = d_trace;
      }
      cudaEvent_t end;
      timer_begin(c, c->tm_cnn, &end);
      CU(c, launch_cnn_chunk(p, c->num_sms, c->stream));
      c->n_launches++;
      timer_end(c, end);
      if (d_trace) {
        std::vector<unsigned long long> h((size_t)1 << 21);
        CU(c, cudaMemcpyAsync(h.data(), d_trace, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                              c->stream));
        CU(c, cudaStreamSynchronize(c->stream));
        cudaFree(d_trace);
        char fn[1024];
        snprintf(fn, sizeof(fn), "%s.chunk%zu.bin", trace_path, ci);
        if (FILE *fp = fopen(fn, "wb")) {
          std::vector<unsigned long long> recs(1, 0);
          for (size_t i = 1; i < h.size(); ++i)
            if (h[i]) recs.push_back(h[i]);
          recs[0] = recs.size() - 1;
          fwrite(recs.data(), sizeof(unsigned long long), recs.size(), fp);
          fclose(fp);
        }
        if (ci + 1 == c->chunks.size()) c->traced = true;
      }
    }
  }
  return PNPULA_OK;
}

pnpula_status exchange(pnpula_ctx *c, int buf, cudaStream_t st = nullptr) {
  if (!st) st = c->stream;
  cudaEvent_t end;
  timer_begin(c, c->tm_halo, &end, st);
  if (c->n_local_jobs) { CU(c, launch_copy_jobs(c->d_local_jobs[buf], c->n_local_jobs, c->max_local, st)); c->n_launches++; }
  if (!c->sends.empty() || !c->recvs.empty()) {
    if (c->n_pack) { CU(c, launch_copy_jobs(c->d_pack_jobs[buf], c->n_pack, c->max_pack, st)); c->n_launches++; }
    NC(c, ncclGroupStart());
    for (auto &m : c->sends) NC(c, ncclSend(c->d_sendbuf + m.off, m.count, ncclFloat32, m.peer, c->comm, st));
    for (auto &m : c->recvs) NC(c, ncclRecv(c->d_recvbuf + m.off, m.count, ncclFloat32, m.peer, c->comm, st));
    NC(c, ncclGroupEnd());
    if (c->n_unpack) { CU(c, launch_copy_jobs(c->d_unpack_jobs[buf], c->n_unpack, c->max_unpack, st)); c->n_launches++; }
  }
  timer_end(c, end, st);
  return PNPULA_OK;
}

// Rows [r0, r1) (tile-relative) of a tile as a geometry of its own: i0/th move, h grows by r0
// so that i0 - h (the padded-buffer origin) and every padded index stay the same.
TileGeom row_range(const TileGeom &g, int r0, int r1) {
  TileGeom b = g;
  b.i0 = g.i0 + r0;
  b.th = r1 - r0;
  b.h = g.h + r0;
  return b;
}

UpdateParams make_update_params(pnpula_ctx *c, TileDev &td, int buf) {
  UpdateParams p{};
  p.x = td.x[buf];
  p.xn = td.x[buf ^ 1];
  p.y = td.y;
  p.mask = td.mask;
  p.G = (c->n_layers > 0) ? td.G : nullptr;
  p.z = td.z;
  p.mean = td.mean;
  p.m2 = td.m2;
  p.g = td.g;
  p.ny = c->ny; p.nx = c->nx;
  const bool poisson = c->op == PNPULA_OP_POISSON;
  p.op = poisson ? PNPULA_OP_CONV : c->op;   // the x-update runs the conv path with y -> z1 (R32)
  p.ry = c->ry; p.rx = c->rx;
  p.separable = c->separable;
  p.eta = 1.0f;
  if (poisson) { p.y = td.z1; p.eta = (float)c->eta; }
  if (c->op != PNPULA_OP_MASK) {
    for (size_t i = 0; i < c->k2d.size(); ++i) p.k2d[i] = c->k2d[i];
    for (size_t i = 0; i < c->ky.size(); ++i) p.ky[i] = c->ky[i];
    for (size_t i = 0; i < c->kx.size(); ++i) p.kx[i] = c->kx[i];
  }
  p.a_g = poisson ? (float)(c->gamma * c->eta / c->rho1) : (float)(c->gamma / c->sigma2);
  p.has_tv = c->tv_beta > 0;
  p.has_z = c->rho > 0 && !p.has_tv;   // TV: z ~ D x is updated by its own kernel after the exchange
  if (p.has_tv) { p.a_tv = (float)(c->gamma / c->rho); p.zv = td.z; p.zh = td.zh; }
  p.a_rho = p.has_z ? (float)(c->gamma / c->rho) : 0.f;   // (TV: a_tv)
  p.has_G = c->n_layers > 0;
  p.a_d = p.has_G ? (float)(c->alpha * c->gamma / (c->eps * c->eps)) : 0.f;
  p.has_box = c->lambda > 0;
  p.a_lam = p.has_box ? (float)(c->gamma / c->lambda) : 0.f;
  p.c_lo = (float)c->c_lo; p.c_hi = (float)c->c_hi;
  p.a_xi = (float)std::sqrt(2.0 * c->gamma);
  p.b_rho = p.has_z ? (float)(c->kappa / c->rho) : 0.f;
  p.b_zeta = p.has_z ? (float)std::sqrt(2.0 * c->kappa) : 0.f;
  p.z_lo = (float)c->z_lo; p.z_hi = (float)c->z_hi;
  p.seed_lo = (uint32_t)c->seed;
  p.seed_hi = (uint32_t)(c->seed >> 32);
  return p;
}

// Enqueue one iteration reading x[buf]. it == nullptr: the iteration scalars go by value
// (t1 = c->t + 1); otherwise every kernel reads them from it = d_iter[buf] and the first
// update launch writes the next iteration's into d_iter[buf ^ 1] (graph capture).
pnpula_status enqueue_step(pnpula_ctx *c, int buf, const IterState *it) {
  const bool fused = c->fuse && c->n_layers > 0;
  if (c->n_layers > 0) {
    pnpula_status s = run_cnn(c, buf, fused, it);
    if (s) return s;
  }
  const uint64_t t1 = (uint64_t)c->t + 1;
  const bool acc = (int64_t)t1 > c->burn_in;
  const double k = acc ? (double)((int64_t)t1 - c->burn_in) : 1.0;
  // the x / z / moment update of rows [r0, r1) of every tile and channel
  auto update_rows = [&](bool all, bool top_band, bool interior) -> pnpula_status {
    for (auto &td : c->tiles)
    for (int ch = 0; ch < c->nc; ++ch) {
      UpdateParams p = make_update_params(c, td, buf);
      p.t1 = (uint32_t)t1;
      p.accumulate = acc;
      p.inv_n = (float)(1.0 / k);
      p.it = it;
      p.it_next = (it && &td == &c->tiles[0] && ch == 0) ? c->d_iter + (buf ^ 1) : nullptr;
      if (ch > 0) {   // channel plane ch (R43): same geometry, its own Philox streams 4 ch + s
        const size_t o = (size_t)ch * geom_elems(td.g);
        p.x += o; p.xn += o; p.y += o; p.mean += o; p.m2 += o;
        if (p.G) p.G += o;
        if (p.z) p.z += o;
        if (p.zv) p.zv += o;   // TV (colour: channel-wise)
        if (p.zh) p.zh += o;
        p.sb = 4u * (uint32_t)ch;
      }
      const int h = td.g.h, th = td.g.th;
      if (!all) p.g = interior ? row_range(td.g, h, th - h) : top_band ? row_range(td.g, 0, h) : row_range(td.g, th - h, th);
      cudaEvent_t end;
      timer_begin(c, c->tm_update, &end);
      CU(c, launch_update(p, c->stream));
      c->n_launches++;
      timer_end(c, end);
    }
    return PNPULA_OK;
  };
  pnpula_status s;
  if (fused) {
    if ((s = exchange(c, buf ^ 1))) return s;   // x^{t+1} was written by the fused last CNN chunk
  } else if (c->overlap) {
    // boundary bands (the rows neighbours receive) first, then the exchange on the comm stream
    // while the interior rows update (SURVEY 8(e) overlap); the next kernels wait for both
    if ((s = update_rows(false, true, false)) || (s = update_rows(false, false, false))) return s;
    CU(c, cudaEventRecord(c->ev_bands, c->stream));
    CU(c, cudaStreamWaitEvent(c->comm_stream, c->ev_bands, 0));
    if ((s = exchange(c, buf ^ 1, c->comm_stream))) return s;
    CU(c, cudaEventRecord(c->ev_halo, c->comm_stream));
    if ((s = update_rows(false, false, true))) return s;
    CU(c, cudaStreamWaitEvent(c->stream, c->ev_halo, 0));
  } else {
    if ((s = update_rows(true, false, false))) return s;
    if ((s = exchange(c, buf ^ 1))) return s;
  }
  if (c->tv_beta > 0) {
    // TV z block (R37, R38): x^{t+1} (halo now valid) -> z = (z_v, z_h) on tile (+) 1, per
    // channel plane for colour images (channel-wise isotropic TV; streams 4 c + 1 / 3)
    for (auto &td : c->tiles)
    for (int ch = 0; ch < c->nc; ++ch) {
      const size_t o = (size_t)ch * geom_elems(td.g);
      TvZParams q{};
      q.x = td.x[buf ^ 1] + o;
      q.zv = td.z + o;
      q.zh = td.zh + o;
      q.sb = 4u * (uint32_t)ch;
      q.g = td.g;
      q.ny = c->ny; q.nx = c->nx;
      q.b = (float)(c->kappa / c->rho);
      q.s = (float)std::sqrt(2.0 * c->kappa);
      q.tau = (float)(c->kappa * c->tv_beta);
      q.seed_lo = (uint32_t)c->seed;
      q.seed_hi = (uint32_t)(c->seed >> 32);
      q.t1 = (uint32_t)t1;
      q.it = it;
      cudaEvent_t end;
      timer_begin(c, c->tm_update, &end);
      CU(c, launch_tv_z_update(q, c->stream));
      c->n_launches++;
      timer_end(c, end);
    }
  }
  if (c->op == PNPULA_OP_POISSON) {
    // line 11-13 for the z1 block: x^{t+1} (halo now valid) -> z1 on tile (+) r_H (R33, R34)
    for (auto &td : c->tiles)
    for (int ch = 0; ch < c->nc; ++ch) {
      const size_t o = (size_t)ch * geom_elems(td.g);
      Z1Params q{};
      q.x = td.x[buf ^ 1] + o;
      q.y = td.y + o;
      q.z1 = td.z1 + o;
      q.sb = 4u * (uint32_t)ch;
      q.g = td.g;
      q.ny = c->ny; q.nx = c->nx;
      q.ry = c->ry; q.rx = c->rx;
      const int kh = 2 * c->ry + 1, kw = 2 * c->rx + 1;
      for (int a = 0; a < kh; ++a)
        for (int b = 0; b < kw; ++b)
          q.k2d[a * kw + b] = c->separable ? c->ky[a] * c->kx[b] : c->k2d[a * kw + b];
      q.separable = c->separable;
      if (c->separable) {
        for (int a = 0; a < kh; ++a) q.ky[a] = c->ky[a];
        for (int b = 0; b < kw; ++b) q.kx[b] = c->kx[b];
      }
      q.eta = (float)c->eta;
      q.b1 = (float)(c->kappa1 / c->rho1);
      q.s1 = (float)std::sqrt(2.0 * c->kappa1);
      q.kappa1 = (float)c->kappa1;
      q.seed_lo = (uint32_t)c->seed;
      q.seed_hi = (uint32_t)(c->seed >> 32);
      q.t1 = (uint32_t)t1;
      q.it = it;
      cudaEvent_t end;
      timer_begin(c, c->tm_update, &end);
      CU(c, launch_z1_update(q, c->stream));
      c->n_launches++;
      timer_end(c, end);
    }
  }
  return PNPULA_OK;
}

void drop_graphs(pnpula_ctx *c) {
  for (int b = 0; b < 2; ++b) {
    if (c->gexec[b]) cudaGraphExecDestroy(c->gexec[b]);
    c->gexec[b] = nullptr;
  }
  c->dev_t = -1;
}

// Replays are used when nothing in the iteration needs the host between kernels: no per-kernel
// timing events and no pipeline trace.  The NCCL halo group (multi-rank, or FLAG_HALO_VIA_NCCL)
// is captured into the graph like the kernels around it (NCCL supports stream capture); with the
// overlap the comm stream forks from / joins the capturing stream through ev_bands / ev_halo, so
// the replayed graph keeps the exchange concurrent with the interior update.  Every rank
// captures the same sequence of NCCL calls per parity, so the replays stay matched across ranks.
bool graph_eligible(const pnpula_ctx *c) {
  return c->warm && !c->graphs_off && !c->timing && !getenv("PNPULA_CNN_TRACE");
}

pnpula_status step(pnpula_ctx *c) {
  const int buf = c->cur;
  if (graph_eligible(c)) {
    if (!c->gexec[buf]) {
      // capture: every scalar of the iteration read from d_iter[buf]
      const int64_t n0 = c->n_launches;
      cudaGraph_t g = nullptr;
      CU(c, cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeRelaxed));
      pnpula_status s = enqueue_step(c, buf, c->d_iter + buf);
      const cudaError_t e2 = cudaStreamEndCapture(c->stream, &g);
      if (s) { if (g) cudaGraphDestroy(g); return s; }
      CU(c, e2);
      const cudaError_t e3 = cudaGraphInstantiate(&c->gexec[buf], g, 0);
      cudaGraphDestroy(g);
      CU(c, e3);
      c->glaunches[buf] = c->n_launches - n0;
      c->n_launches = n0;
    }
    if (c->dev_t != c->t) {   // d_iter[buf] does not hold iteration t+1 (reset, load, direct steps)
      const int64_t t1 = c->t + 1;
      const bool acc = t1 > c->burn_in;
      IterState h{};
      h.t1 = t1;
      h.burn_in = c->burn_in;
      h.accumulate = acc;
      h.inv_n = (float)(1.0 / (acc ? (double)(t1 - c->burn_in) : 1.0));
      CU(c, cudaMemcpyAsync(c->d_iter + buf, &h, sizeof(h), cudaMemcpyHostToDevice, c->stream));
      CU(c, cudaStreamSynchronize(c->stream));   // h is a stack (pageable) buffer
    }
    CU(c, cudaGraphLaunch(c->gexec[buf], c->stream));
    c->n_launches += c->glaunches[buf];
    c->dev_t = c->t + 1;   // d_iter[buf ^ 1] now holds iteration t+2
  } else {
    pnpula_status s = enqueue_step(c, buf, nullptr);
    if (s) return s;
    c->warm = true;
  }
  c->cur ^= 1;
  c->t += 1;
  return PNPULA_OK;
}

pnpula_status build_halo_plan(pnpula_ctx *c) {
  int n = pnpula_plan_halo(c->ny, c->nx, c->tiles_y, c->tiles_x, c->h, nullptr, 0);
  if (n < 0) { set_error("tile extent smaller than halo width %d", c->h); return PNPULA_E_PARTITION_TOO_FINE; }
  c->msgs.resize(n);
  pnpula_plan_halo(c->ny, c->nx, c->tiles_y, c->tiles_x, c->h, c->msgs.data(), n);
  const int per_rank = c->ntiles / c->world;
  auto owner = [&](int tile) { return tile / per_rank; };
  auto local = [&](int tile) -> TileDev * {
    int li = tile - c->first_tile;
    return (li >= 0 && li < c->n_local) ? &c->tiles[li] : nullptr;
  };
  const bool force_nccl = (c->flags & PNPULA_FLAG_HALO_VIA_NCCL) != 0;
  std::vector<CopyJob> lj[2], pj[2], uj[2];
  size_t soff = 0, roff = 0;
  for (auto &m : c->msgs) {
    TileDev *src = local(m.src_tile), *dst = local(m.dst_tile);
    if (!src && !dst) continue;
    const pnpula_rect &r = m.rect;
    const size_t cnt = (size_t)r.h * r.w;
    auto off = [](const TileGeom &g, int gi, int gj) {
      return (size_t)(gi - (g.i0 - g.h)) * g.pitch + (gj - (g.j0 - g.hx));
    };
    // one job / message per image channel plane (R43)
    for (int ch = 0; ch < c->nc; ++ch) {
      const size_t so = src ? (size_t)ch * geom_elems(src->g) : 0, dso = dst ? (size_t)ch * geom_elems(dst->g) : 0;
      if (src && dst && !force_nccl) {
        for (int b = 0; b < 2; ++b)
          lj[b].push_back({src->x[b] + so + off(src->g, r.i0, r.j0), dst->x[b] + dso + off(dst->g, r.i0, r.j0),
                           src->g.pitch, dst->g.pitch, r.h, r.w});
        c->max_local = std::max(c->max_local, (int)cnt);
        continue;
      }
      if (src) {
        for (int b = 0; b < 2; ++b)
          pj[b].push_back({src->x[b] + so + off(src->g, r.i0, r.j0), nullptr, src->g.pitch, r.w, r.h, r.w});
        c->sends.push_back({owner(m.dst_tile), soff, cnt});
        soff += cnt;
        c->max_pack = std::max(c->max_pack, (int)cnt);
      }
      if (dst) {
        for (int b = 0; b < 2; ++b)
          uj[b].push_back({nullptr, dst->x[b] + dso + off(dst->g, r.i0, r.j0), r.w, dst->g.pitch, r.h, r.w});
        c->recvs.push_back({owner(m.src_tile), roff, cnt});
        roff += cnt;
        c->max_unpack = std::max(c->max_unpack, (int)cnt);
      }
    }
  }
  if (soff) CU(c, cudaMalloc(&c->d_sendbuf, soff * sizeof(float)));
  if (roff) CU(c, cudaMalloc(&c->d_recvbuf, roff * sizeof(float)));
  for (int b = 0; b < 2; ++b) {
    size_t so = 0, ro = 0;
    for (size_t i = 0; i < pj[b].size(); ++i) { pj[b][i].dst = c->d_sendbuf + so; so += (size_t)pj[b][i].rows * pj[b][i].cols; }
    for (size_t i = 0; i < uj[b].size(); ++i) { uj[b][i].src = c->d_recvbuf + ro; ro += (size_t)uj[b][i].rows * uj[b][i].cols; }
  }
  c->n_local_jobs = (int)lj[0].size();
  c->n_pack = (int)pj[0].size();
  c->n_unpack = (int)uj[0].size();
  for (int b = 0; b < 2; ++b) {
    if (c->n_local_jobs) {
      CU(c, cudaMalloc(&c->d_local_jobs[b], lj[b].size() * sizeof(CopyJob)));
      CU(c, cudaMemcpy(c->d_local_jobs[b], lj[b].data(), lj[b].size() * sizeof(CopyJob), cudaMemcpyHostToDevice));
    }
    if (c->n_pack) {
      CU(c, cudaMalloc(&c->d_pack_jobs[b], pj[b].size() * sizeof(CopyJob)));
      CU(c, cudaMemcpy(c->d_pack_jobs[b], pj[b].data(), pj[b].size() * sizeof(CopyJob), cudaMemcpyHostToDevice));
    }
    if (c->n_unpack) {
      CU(c, cudaMalloc(&c->d_unpack_jobs[b], uj[b].size() * sizeof(CopyJob)));
      CU(c, cudaMemcpy(c->d_unpack_jobs[b], uj[b].data(), uj[b].size() * sizeof(CopyJob), cudaMemcpyHostToDevice));
    }
  }
  return PNPULA_OK;
}

// CNN chunking: greedy, as many consecutive layers per launch as shared memory allows.
void plan_cnn_chunks(pnpula_ctx *c) {
  c->chunks.clear();
  const int K = c->n_layers;
  const size_t budget = 227 * 1024;
  int l = 1;
  while (l <= K) {
    int best = 1;
    const char *mnl = getenv("PNPULA_MAX_NL");   // experiment: cap the layers per launch
    const int maxnl = (c->flags & PNPULA_FLAG_CNN_LAYERWISE) ? 1 : (mnl && atoi(mnl) > 0) ? std::min(atoi(mnl), kMaxChunk) : kMaxChunk;
    for (int nl = 1; nl <= std::min(maxnl, K - l + 1); ++nl) {
      if (cnn_chunk_smem_bytes(c->channels, nl, l == 1, l + nl - 1 == K, c->nc, c->fuse) <= budget) best = nl;
    }
    c->chunks.push_back({l, best, K - (l + best - 1)});
    l += best;
  }
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

const char *pnpula_version(void) { return "pnpula-b200 0.1 (sm_100a)"; }

const char *pnpula_last_error(void) { return g_last_error.c_str(); }

void pnpula_partition(int64_t n, int64_t parts, int64_t p, int64_t *lo, int64_t *hi) {
  *lo = (p * n) / parts;
  *hi = ((p + 1) * n) / parts;
}

int32_t pnpula_halo_width(int32_t op, int32_t kh, int32_t kw, int32_t n_layers) {
  int r = (op == PNPULA_OP_CONV || op == PNPULA_OP_POISSON) ? std::max(kh, kw) / 2 : 0;
  return std::max(2 * r, std::max(n_layers, 0));
}

int32_t pnpula_plan_halo(int32_t ny, int32_t nx, int32_t tiles_y, int32_t tiles_x, int32_t h,
                         pnpula_halo_msg *out, int32_t cap) {
  const int nt = tiles_y * tiles_x;
  std::vector<pnpula_rect> rects(nt);
  for (int t = 0; t < nt; ++t) {
    tile_rect(ny, nx, tiles_y, tiles_x, t, &rects[t]);
    // a tile narrower than h would need ghost rows from beyond its neighbour; along an axis with
    // a single tile there is no neighbour, so any extent works there
    if ((tiles_y > 1 && rects[t].h < h) || (tiles_x > 1 && rects[t].w < h)) return -1;
  }
  if (h == 0) return 0;
  int count = 0;
  for (int s = 0; s < nt; ++s) {
    for (int d = 0; d < nt; ++d) {
      if (s == d) continue;
      const pnpula_rect &rs = rects[s], &rd = rects[d];
      // ghost frame of d = (rd (+) h) \ rd, clipped to the image; intersect with interior of s
      int a0 = std::max(rs.i0, std::max(rd.i0 - h, 0));
      int a1 = std::min(rs.i0 + rs.h, std::min(rd.i0 + rd.h + h, ny));
      int b0 = std::max(rs.j0, std::max(rd.j0 - h, 0));
      int b1 = std::min(rs.j0 + rs.w, std::min(rd.j0 + rd.w + h, nx));
      if (a0 >= a1 || b0 >= b1) continue;
      if (out && count < cap) out[count] = {s, d, {a0, b0, a1 - a0, b1 - b0}};
      count++;
    }
  }
  return count;
}

int32_t pnpula_check_stepsizes(double L, double h2_over_rho, double alpha, double eps, double L_D,
                               double lambda, double gamma) {
  int32_t bad = 0;
  const double prior = (alpha > 0 && L_D > 0) ? alpha * L_D / (eps * eps) : 0.0;
  if (!(2.0 * (L + h2_over_rho) + prior <= 0.5 / lambda)) bad |= 1;
  if (!(3.0 * gamma * (L + h2_over_rho + 1.0 / lambda + prior) < 1.0)) bad |= 2;
  return bad;
}

pnpula_status pnpula_get_unique_id(uint8_t out[128]) {
  if (!out) { set_error("null output"); return PNPULA_E_INVALID_ARG; }
  ncclUniqueId id;
  ncclResult_t e = ncclGetUniqueId(&id);
  if (e != ncclSuccess) return fail_nccl(nullptr, e, "ncclGetUniqueId", __LINE__);
  static_assert(sizeof(id) == 128, "nccl id size");
  memcpy(out, &id, 128);
  return PNPULA_OK;
}

pnpula_status pnpula_destroy(pnpula_ctx *c);

pnpula_status pnpula_create(const pnpula_config *cfg, pnpula_ctx **out) {
  // PNPULA_TIME_CREATE=1: per-phase wall times of create on stderr (diagnostics)
  const bool tcre = getenv("PNPULA_TIME_CREATE") != nullptr;
  auto tc0 = std::chrono::steady_clock::now();
  auto phase = [&](const char *what) {
    if (!tcre) return;
    auto t = std::chrono::steady_clock::now();
    fprintf(stderr, "[pnpula_create] %-28s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(t - tc0).count());
    tc0 = t;
  };
  g_last_error.clear();
  if (!cfg || !out) { set_error("null argument"); return PNPULA_E_INVALID_ARG; }
  *out = nullptr;
  const pnpula_config &f = *cfg;
  if (f.ny <= 0 || f.nx <= 0) { set_error("image size must be positive"); return PNPULA_E_SHAPE; }
  if (f.tiles_y <= 0 || f.tiles_x <= 0 || f.tiles_y > f.ny || f.tiles_x > f.nx) {
    set_error("invalid tile grid %dx%d", f.tiles_y, f.tiles_x); return PNPULA_E_PARTITION_TOO_FINE;
  }
  const int ntiles = f.tiles_y * f.tiles_x;
  if (f.world_size <= 0 || ntiles % f.world_size != 0 || f.rank < 0 || f.rank >= f.world_size) {
    set_error("world_size must divide the tile count and rank be in range"); return PNPULA_E_INVALID_ARG;
  }
  if (f.op != PNPULA_OP_CONV && f.op != PNPULA_OP_MASK && f.op != PNPULA_OP_POISSON) {
    set_error("unknown op"); return PNPULA_E_INVALID_ARG;
  }
  const bool poisson = f.op == PNPULA_OP_POISSON;
  if (!(f.gamma > 0) || (!poisson && !(f.sigma2 > 0))) { set_error("gamma and sigma2 must be > 0"); return PNPULA_E_INVALID_ARG; }
  if (!f.y) { set_error("y is required"); return PNPULA_E_INVALID_ARG; }
  if (poisson && !(f.eta > 0 && f.rho1 > 0 && f.kappa1 > 0 && f.kappa1 < f.rho1)) {
    set_error("OP_POISSON needs eta > 0, rho1 > 0 and kappa1 in (0, rho1)"); return PNPULA_E_INVALID_ARG;
  }
  if (f.op != PNPULA_OP_MASK) {
    if (f.kh <= 0 || f.kw <= 0 || f.kh % 2 == 0 || f.kw % 2 == 0 || f.kh > kMaxTaps || f.kw > kMaxTaps) {
      set_error("kernel sizes must be odd and <= %d", kMaxTaps); return PNPULA_E_INVALID_ARG;
    }
    if (!f.kernel && !(f.kernel_y && f.kernel_x)) { set_error("kernel required"); return PNPULA_E_INVALID_ARG; }
  } else if (!f.mask) {
    set_error("mask required for OP_MASK"); return PNPULA_E_INVALID_ARG;
  }
  if (f.rho > 0 && !(f.kappa > 0 && f.kappa < f.rho)) { set_error("kappa must lie in (0, rho)"); return PNPULA_E_INVALID_ARG; }
  const bool use_cnn = f.den && f.alpha != 0.0;
  const bool tv = f.tv_beta > 0;
  if (tv && (!(f.rho > 0) || use_cnn || f.lambda > 0)) {
    set_error("TV prior needs rho > 0 (its z block), no denoiser and lambda <= 0"); return PNPULA_E_INVALID_ARG;
  }
  const bool ddfb = use_cnn && f.den->kind == PNPULA_DEN_DDFB;
  if (use_cnn && f.den->kind != PNPULA_DEN_DNCNN && !ddfb) { set_error("unknown denoiser kind"); return PNPULA_E_INVALID_ARG; }
  if (ddfb && (f.den->n_layers < 1 || !f.den->weights || !f.den->ddfb_gammas || !(f.den->ht_eps > 0))) {
    set_error("DDFB needs >= 1 layer, weights, gammas and ht_eps > 0"); return PNPULA_E_INVALID_ARG;
  }
  if (use_cnn && !ddfb) {
    if (f.den->n_layers < 2 || !f.den->weights || !f.den->biases) { set_error("denoiser needs >= 2 layers and weights"); return PNPULA_E_INVALID_ARG; }
    if (f.den->channels != 16 && f.den->channels != 32 && f.den->channels != 64) {
      set_error("denoiser channels must be 16, 32 or 64"); return PNPULA_E_UNSUPPORTED;
    }
    if (!(f.eps > 0)) { set_error("eps must be > 0"); return PNPULA_E_INVALID_ARG; }
  }
  const int nc = f.img_channels > 1 ? f.img_channels : 1;
  if (nc != 1 && nc != 3) { set_error("img_channels must be 1 or 3"); return PNPULA_E_UNSUPPORTED; }
  if (nc > 1 && ddfb && f.den->channels != 32 && f.den->channels != 64) {
    set_error("colour DDFB needs P = 32 or 64 (N = 48 folded adjoint columns)"); return PNPULA_E_UNSUPPORTED;
  }
  if (nc > 1 && use_cnn && f.den->channels < 32) {
    set_error("colour DnCNN needs channels >= 32 (N = 48 folded output columns)"); return PNPULA_E_UNSUPPORTED;
  }
  const pnpula_rect in = f.in_rect;

  pnpula_ctx *c = new pnpula_ctx();
  c->nc = nc;
  c->ny = f.ny; c->nx = f.nx; c->tiles_y = f.tiles_y; c->tiles_x = f.tiles_x;
  c->rank = f.rank; c->world = f.world_size; c->device = f.device;
  c->op = f.op; c->flags = f.flags;
  c->sigma2 = f.sigma2; c->alpha = f.alpha; c->eps = f.eps; c->lambda = f.lambda;
  c->c_lo = f.c_lo; c->c_hi = f.c_hi; c->rho = f.rho; c->kappa = f.kappa;
  c->z_lo = f.z_lo; c->z_hi = f.z_hi; c->gamma = f.gamma;
  if (poisson) { c->eta = f.eta; c->rho1 = f.rho1; c->kappa1 = f.kappa1; }
  if (tv) c->tv_beta = f.tv_beta;
  if (f.op != PNPULA_OP_MASK) {
    c->kh = f.kh; c->kw = f.kw; c->ry = f.kh / 2; c->rx = f.kw / 2;
    c->separable = (f.kernel_y && f.kernel_x) ? 1 : 0;
    if (c->separable) {
      c->ky.assign(f.kernel_y, f.kernel_y + f.kh);
      c->kx.assign(f.kernel_x, f.kernel_x + f.kw);
    } else {
      c->k2d.assign(f.kernel, f.kernel + f.kh * f.kw);
    }
  }
  if (use_cnn) { c->n_layers = f.den->n_layers; c->channels = f.den->channels; }
  if (ddfb) { c->den_kind = PNPULA_DEN_DDFB; c->ht_eps = f.den->ht_eps; }
  // receptive field of the prior: K 3x3 layers (DnCNN), or two 3x3 operators per DDFB layer
  c->h = pnpula_halo_width(f.op, f.kh, f.kw, ddfb ? 2 * c->n_layers : c->n_layers);
  if (tv) c->h = std::max(c->h, 2);   // D^T D x needs x at distance 1, z on tile (+) 1 needs 2 (R38)
  c->ntiles = ntiles;
  c->n_local = ntiles / f.world_size;
  c->first_tile = f.rank * c->n_local;

  // step-size check (warning only)
  {
    double L = f.lipschitz_L;
    double L_h2 = 0;
    if (L <= 0) {
      double s = 0;
      if (f.op != PNPULA_OP_MASK) {
        if (c->separable) {
          double a = 0, b = 0;
          for (float v : c->ky) a += std::fabs(v);
          for (float v : c->kx) b += std::fabs(v);
          s = a * b;
        } else {
          for (float v : c->k2d) s += std::fabs(v);
        }
      } else {
        s = 1;
      }
      L = s * s / f.sigma2;   // ||H||^2 <= ||k||_1^2 (Young)
      // OP_POISSON: f1 = 0 and the z1 block contributes ||eta H||^2 / rho1 to ||H2||^2/rho
      if (poisson) L = 0;
      if (poisson) s = s * f.eta;
      if (poisson) L_h2 = s * s / f.rho1;
    }
    const double lam = f.lambda > 0 ? f.lambda : 1e300;
    // ||H2||^2 / rho: H2 = I (1/rho), TV H2 = D (||D||^2 <= 8, R35), plus the Poisson z1 block
    const double h2 = f.rho > 0 ? (tv ? 8.0 : 1.0) / f.rho : 0.0;
    int32_t bad = pnpula_check_stepsizes(L, h2 + L_h2, use_cnn ? f.alpha : 0.0,
                                         use_cnn ? f.eps : 1.0, f.lipschitz_LD, lam, f.gamma);
    if (bad) set_error("warning: eq:stepsize_cond violated (mask %d) -- continuing", bad);
  }

  // tiles and validation of in_rect coverage
  const int rH = std::max(c->ry, c->rx);
  pnpula_rect bb{INT32_MAX, INT32_MAX, 0, 0};
  int bi1 = INT32_MIN, bj1 = INT32_MIN;
  for (int li = 0; li < c->n_local; ++li) {
    pnpula_rect r;
    tile_rect(f.ny, f.nx, f.tiles_y, f.tiles_x, c->first_tile + li, &r);
    if ((f.tiles_y > 1 && r.h < c->h) || (f.tiles_x > 1 && r.w < c->h)) {
      set_error("tile %dx%d smaller than halo width %d", r.h, r.w, c->h);
      delete c;
      return PNPULA_E_PARTITION_TOO_FINE;
    }
    int need_i0 = std::max(r.i0 - rH, 0), need_i1 = std::min(r.i0 + r.h + rH, f.ny);
    int need_j0 = std::max(r.j0 - rH, 0), need_j1 = std::min(r.j0 + r.w + rH, f.nx);
    if (need_i0 < in.i0 || need_j0 < in.j0 || need_i1 > in.i0 + in.h || need_j1 > in.j0 + in.w) {
      set_error("in_rect {%d,%d,%d,%d} does not cover tile (+) r_H", in.i0, in.j0, in.h, in.w);
      delete c;
      return PNPULA_E_SHAPE;
    }
    TileDev td;
    td.index = c->first_tile + li;
    td.g = make_geom(r.i0, r.j0, r.h, r.w, c->h);
    c->tiles.push_back(td);
    bb.i0 = std::min(bb.i0, r.i0); bb.j0 = std::min(bb.j0, r.j0);
    bi1 = std::max(bi1, r.i0 + r.h); bj1 = std::max(bj1, r.j0 + r.w);
  }
  bb.h = bi1 - bb.i0; bb.w = bj1 - bb.j0;
  c->bbox = bb;

  std::string warn = g_last_error;
  auto bail = [&](pnpula_status s) { pnpula_destroy(c); return s; };
  cudaError_t e = cudaSetDevice(f.device);
  if (e != cudaSuccess) { fail_cuda(nullptr, e, "cudaSetDevice", __LINE__); return bail(PNPULA_E_CUDA); }
  // three attribute queries (cudaGetDeviceProperties fills every field: ~10 ms)
  int cc_major = 0, cc_minor = 0, n_sms = 0;
  e = cudaDeviceGetAttribute(&cc_major, cudaDevAttrComputeCapabilityMajor, f.device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&cc_minor, cudaDevAttrComputeCapabilityMinor, f.device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&n_sms, cudaDevAttrMultiProcessorCount, f.device);
  if (e != cudaSuccess) { fail_cuda(nullptr, e, "cudaDeviceGetAttribute", __LINE__); return bail(PNPULA_E_CUDA); }
  if (cc_major != 10 || cc_minor != 0) {
    set_error("device %d is sm_%d%d; this library is built for sm_100a only", f.device, cc_major, cc_minor);
    return bail(PNPULA_E_CUDA);
  }
  c->num_sms = n_sms;
  {
    // test hook: cap the CNN grid (persistent CTAs) so that small images give every CTA several
    // work units -- exercises the cross-unit barrier-phase bookkeeping of the tcgen05 pipeline
    const char *mc = getenv("PNPULA_MAX_CTAS");
    if (mc && atoi(mc) > 0) c->num_sms = std::min(n_sms, atoi(mc));
  }
  if (f.stream) {
    c->stream = (cudaStream_t)(uintptr_t)f.stream;
  } else {
    e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) { fail_cuda(nullptr, e, "cudaStreamCreate", __LINE__); return bail(PNPULA_E_CUDA); }
    c->own_stream = true;
  }
#define CUB(expr)                                                              \
  do {                                                                         \
    cudaError_t _e = (expr);                                                   \
    if (_e != cudaSuccess) { fail_cuda(nullptr, _e, #expr, __LINE__);          \
      return bail(_e == cudaErrorMemoryAllocation ? PNPULA_E_OOM : PNPULA_E_CUDA); } \
  } while (0)
  phase("validation + stream");
  CUB(cudaMalloc(&c->d_err, sizeof(int)));
  CUB(cudaMemsetAsync(c->d_err, 0, sizeof(int), c->stream));
  CUB(cudaMalloc(&c->d_iter, 2 * sizeof(IterState)));
  {
    const char *pe = getenv("PNPULA_POOL");
    if (!(pe && atoi(pe) == 0)) c->pool = device_pool(f.device);
  }
  {
    const char *pe2 = getenv("PNPULA_PDL");
    c->pdl = (pe2 && atoi(pe2) == 0) ? 0 : 1;
    const char *pe3 = getenv("PNPULA_CNN_CONTIG");
    c->cnn_contig = (pe3 && atoi(pe3) == 0) ? 0 : (pe3 && atoi(pe3) == 2) ? 2 : 1;   // 2: always (tests)
  }
  {
    const char *ge = getenv("PNPULA_GRAPHS");
    c->graphs_off = (f.flags & PNPULA_FLAG_NO_GRAPH) != 0 || (ge && atoi(ge) == 0);
  }

  if (f.world_size > 1) {
    if (!f.nccl_uid) { set_error("nccl_uid required when world_size > 1"); return bail(PNPULA_E_INVALID_ARG); }
    ncclUniqueId id;
    memcpy(&id, f.nccl_uid, 128);
    ncclResult_t r = ncclCommInitRank(&c->comm, f.world_size, id, f.rank);
    if (r != ncclSuccess) { fail_nccl(nullptr, r, "ncclCommInitRank", __LINE__); return bail(PNPULA_E_NCCL); }
  } else if (c->flags & PNPULA_FLAG_HALO_VIA_NCCL) {
    int dev = f.device;
    ncclResult_t r = ncclCommInitAll(&c->comm, 1, &dev);
    if (r != ncclSuccess) { fail_nccl(nullptr, r, "ncclCommInitAll", __LINE__); return bail(PNPULA_E_NCCL); }
  }

  phase("nccl / small buffers");
  // device buffers
  for (auto &td : c->tiles) {
    const size_t n1 = geom_elems(td.g);   // one plane
    const size_t n = n1 * (size_t)nc;      // state fields: nc planes
    for (int b = 0; b < 2; ++b) {
      CUB(dmalloc(c, &td.x[b], n * sizeof(float)));
      CUB(cudaMemsetAsync(td.x[b], 0, n * sizeof(float), c->stream));
    }
    CUB(dmalloc(c, &td.x0, n * sizeof(float)));
    CUB(cudaMemsetAsync(td.x0, 0, n * sizeof(float), c->stream));
    CUB(dmalloc(c, &td.y, n * sizeof(float)));
    CUB(cudaMemsetAsync(td.y, 0, n * sizeof(float), c->stream));
    CUB(dmalloc(c, &td.mean, n * sizeof(float)));
    CUB(dmalloc(c, &td.m2, n * sizeof(float)));
    if (c->rho > 0) CUB(dmalloc(c, &td.z, n * sizeof(float)));
    if (tv) {
      CUB(dmalloc(c, &td.zh, n * sizeof(float)));
      CUB(cudaMemsetAsync(td.zh, 0, n * sizeof(float), c->stream));
    }
    if (poisson) {   // Poisson z1 block
      CUB(dmalloc(c, &td.z1, n * sizeof(float)));
      CUB(cudaMemsetAsync(td.z1, 0, n * sizeof(float), c->stream));
    }
    if (c->op == PNPULA_OP_MASK) {   // one plane, shared by the channels
      CUB(dmalloc(c, &td.mask, n1));
      CUB(cudaMemsetAsync(td.mask, 0, n1, c->stream));
    }
    if (c->n_layers > 0) {
      CUB(dmalloc(c, &td.G, n * sizeof(float)));
      CUB(cudaMemsetAsync(td.G, 0, n * sizeof(float), c->stream));
    }
    const TileGeom &g = td.g;
    pnpula_status s;
    phase("  tile malloc + memset");
    const size_t in_plane = (size_t)in.h * in.w;
    for (int ch = 0; ch < nc; ++ch) {
      s = upload_padded<float>(c, td.y + ch * n1, g, f.y + ch * in_plane, in, g.i0 - rH, g.j0 - rH, g.th + 2 * rH,
                               g.tw + 2 * rH);
      if (s) return bail(s);
      if (f.x0) {
        s = upload_padded<float>(c, td.x0 + ch * n1, g, f.x0 + ch * in_plane, in, g.i0, g.j0, g.th, g.tw);
        if (s) return bail(s);
      }
    }
    if (c->op == PNPULA_OP_MASK) {
      s = upload_padded<uint8_t>(c, td.mask, g, f.mask, in, g.i0, g.j0, g.th, g.tw);
      if (s) return bail(s);
    }
  }
  phase("tile buffers + uploads");
  // DDFB operator images and buffers
  if (ddfb) {
    const int K = c->n_layers, P = c->channels;
    auto upload = [&](const std::vector<float> &wt, int cout, int cin, uint16_t **dst) -> pnpula_status {
      std::vector<uint16_t> packed(cnn_packed_layer_elems(cout, cin));
      cnn_pack_layer(wt.data(), cout, cin, packed.data());
      cudaError_t e2 = cudaMalloc(dst, packed.size() * sizeof(uint16_t));
      if (e2 == cudaSuccess) e2 = cudaMemcpy(*dst, packed.data(), packed.size() * sizeof(uint16_t), cudaMemcpyHostToDevice);
      if (e2 != cudaSuccess) { fail_cuda(nullptr, e2, "DDFB weights", __LINE__); return PNPULA_E_CUDA; }
      return PNPULA_OK;
    };
    // W_k as a C -> P conv [P][C][3][3] (scaled), and W_k^* as a P -> C conv [C][P][3][3]:
    // w'[c][p][a][b] = s * w_k[p][c][2-a][2-b] (the adjoint of a cross-correlation; C = 1 or 3)
    const size_t lw = (size_t)P * nc * 9;   // weights per DDFB layer
    auto wk = [&](int k, double sc) {
      std::vector<float> o(lw);
      for (size_t i = 0; i < o.size(); ++i) o[i] = (float)(sc * f.den->weights[(size_t)(k - 1) * lw + i]);
      return o;
    };
    auto wadj = [&](int k, double sc) {
      std::vector<float> o(lw);
      for (int ci = 0; ci < nc; ++ci)
        for (int ch = 0; ch < P; ++ch)
          for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b)
              o[(((size_t)ci * P + ch) * 3 + a) * 3 + b] =
                  (float)(sc * f.den->weights[(size_t)(k - 1) * lw + (((size_t)ch * nc + ci) * 3 + (2 - a)) * 3 + (2 - b)]);
      return o;
    };
    pnpula_status s = upload(wk(K, 1.0), P, nc, &c->ddfb_u0);
    if (s) return bail(s);
    for (int k = 1; k < K; ++k) {
      uint16_t *t = nullptr, *a = nullptr;
      s = upload(wk(k, f.den->ddfb_gammas[k - 1]), P, nc, &t);
      if (!s) s = upload(wadj(k, 1.0), nc, P, &a);
      c->ddfb_t.push_back(t);
      c->ddfb_adj.push_back(a);
      if (s) return bail(s);
    }
    s = upload(wadj(K, f.den->ddfb_gammas[K - 1]), nc, P, &c->ddfb_fin);
    if (s) return bail(s);
    for (auto &td : c->tiles) {
      const size_t n = geom_elems(td.g) * (size_t)nc;   // p = proj(v - W^* u): C planes
      CUB(dmalloc(c, &td.pbuf, n * sizeof(float)));
      CUB(cudaMemsetAsync(td.pbuf, 0, n * sizeof(float), c->stream));
      CUB(dmalloc(c, &td.pbuf2, n * sizeof(float)));
      CUB(cudaMemsetAsync(td.pbuf2, 0, n * sizeof(float), c->stream));
      const size_t act = (size_t)(td.g.th + 2 * (2 * K - 1)) * (td.g.tw + 2 * (2 * K - 1)) * P;
      for (int b2 = 0; b2 < 2; ++b2) {
        CUB(dmalloc(c, &td.act[b2], act * sizeof(uint16_t)));
        CUB(cudaMemsetAsync(td.act[b2], 0, act * sizeof(uint16_t), c->stream));
      }
    }
  }
  // CNN weights
  phase("ddfb");
  if (c->n_layers > 0 && !ddfb) {
    {
      const char *fe = getenv("PNPULA_FUSE");
      UpdateParams u{};
      u.op = c->op == PNPULA_OP_MASK ? 1 : 0;   // Poisson's x step runs the conv path (R32)
      u.separable = c->separable;
      u.ry = c->ry; u.rx = c->rx;
      u.has_tv = c->tv_beta > 0;
      c->fuse = (fe && atoi(fe) == 1) && cnn_fused_update_supported(c->channels, nc, u);
    }
    plan_cnn_chunks(c);
    if (c->fuse && c->chunks.back().l0 == 1) {   // one chunk: its producers build im2col rows (no time to spare)
      c->fuse = false;
      plan_cnn_chunks(c);
    }
    const int K = c->n_layers, P = c->channels;
    const float *w = f.den->weights;
    const float *b = f.den->biases;
    int cin = nc;   // layer 1: C -> P, layer K: P -> C (R43)
    for (int l = 1; l <= K; ++l) {
      const int cout = (l == K) ? nc : P;
      std::vector<uint16_t> packed(cnn_packed_layer_elems(cout, cin));
      cnn_pack_layer(w, cout, cin, packed.data());
      uint16_t *dw = nullptr;
      float *db = nullptr;
      CUB(cudaMalloc(&dw, packed.size() * sizeof(uint16_t)));
      CUB(cudaMemcpy(dw, packed.data(), packed.size() * sizeof(uint16_t), cudaMemcpyHostToDevice));
      CUB(cudaMalloc(&db, cout * sizeof(float)));
      CUB(cudaMemcpy(db, b, cout * sizeof(float), cudaMemcpyHostToDevice));
      c->d_w.push_back(dw);
      c->d_b.push_back(db);
      c->h_b.emplace_back(b, b + cout);
      w += (size_t)cout * cin * 9;
      b += cout;
      cin = cout;
    }
    size_t maxact = 0;
    for (auto &ch : c->chunks) {
      if (ch.l0 + ch.nl - 1 == K) continue;
      for (auto &td : c->tiles)
        maxact = std::max(maxact, (size_t)(td.g.th + 2 * ch.ext) * (td.g.tw + 2 * ch.ext) * P);
    }
    if (maxact) {
      // chunk ci writes act[ci & 1] and reads act[(ci + 1) & 1]: two chunks need one buffer
      const int nact = c->chunks.size() > 2 ? 2 : 1;
      for (auto &td : c->tiles)
        for (int b2 = 0; b2 < nact; ++b2) {
          CUB(dmalloc(c, &td.act[b2], maxact * sizeof(uint16_t)));
          // no memset: every activation a chunk reads was written by the previous chunk of the same
          // evaluation (positions outside the stored region are zero-filled by the producer)
        }
    }
  }
  {
    phase("cnn weights + act buffers");
    pnpula_status s = build_halo_plan(c);
    if (s) return bail(s);
  }
  // overlap the NCCL halo exchange with the interior update: row-strip grids (the messages are
  // the h top / bottom rows of a tile) whose tiles have interior rows (env PNPULA_OVERLAP=0: off)
  {
    const char *oe = getenv("PNPULA_OVERLAP");
    bool ok = !(oe && atoi(oe) == 0) && (!c->sends.empty() || !c->recvs.empty()) && c->tiles_x == 1 && c->h > 0 &&
              !c->fuse;   // fused: the update runs inside the CNN, the exchange follows it
    for (auto &td : c->tiles) ok = ok && td.g.th > 2 * td.g.h;
    if (ok) {
      CUB(cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking));
      CUB(cudaEventCreateWithFlags(&c->ev_bands, cudaEventDisableTiming));
      CUB(cudaEventCreateWithFlags(&c->ev_halo, cudaEventDisableTiming));
      c->overlap = true;
    }
  }
  phase("halo plan + overlap");
  CUB(cudaStreamSynchronize(c->stream));
  phase("final sync");
  g_last_error = warn;
  *out = c;
  return PNPULA_OK;
#undef CUB
}

pnpula_status pnpula_reset(pnpula_ctx *c, int64_t burn_in, uint64_t seed) {
  pnpula_status s = check_ctx(c);
  if (s) return s;
  if (burn_in < 0) { set_error("burn_in must be >= 0"); return PNPULA_E_INVALID_ARG; }
  CU(c, cudaSetDevice(c->device));
  for (auto &td : c->tiles) {
    const size_t n = geom_elems(td.g) * sizeof(float) * c->nc;
    CU(c, cudaMemcpyAsync(td.x[0], td.x0, n, cudaMemcpyDeviceToDevice, c->stream));
    CU(c, cudaMemcpyAsync(td.x[1], td.x0, n, cudaMemcpyDeviceToDevice, c->stream));
    if (td.z) CU(c, cudaMemsetAsync(td.z, 0, n, c->stream));
    if (td.z1) CU(c, cudaMemsetAsync(td.z1, 0, n, c->stream));
    if (td.zh) CU(c, cudaMemsetAsync(td.zh, 0, n, c->stream));
    CU(c, cudaMemsetAsync(td.mean, 0, n, c->stream));
    CU(c, cudaMemsetAsync(td.m2, 0, n, c->stream));
  }
  drop_graphs(c);
  c->cur = 0;
  c->t = 0;
  c->burn_in = burn_in;
  c->seed = seed;
  c->have_reset = true;
  return exchange(c, 0);
}

pnpula_status pnpula_advance(pnpula_ctx *c, int64_t n_iter) {
  pnpula_status s = check_ctx(c);
  if (s) return s;
  if (!c->have_reset) { set_error("pnpula_reset must precede pnpula_advance"); return PNPULA_E_STATE; }
  if (n_iter < 0) { set_error("n_iter must be >= 0"); return PNPULA_E_INVALID_ARG; }
  CU(c, cudaSetDevice(c->device));
  for (int64_t i = 0; i < n_iter; ++i) {
    s = step(c);
    if (s) return s;
  }
  CU(c, cudaGetLastError());
  return PNPULA_OK;
}

pnpula_status pnpula_synchronize(pnpula_ctx *c) {
  pnpula_status s = check_ctx(c);
  if (s) return s;
  CU(c, cudaStreamSynchronize(c->stream));
  int err = 0;
  CU(c, cudaMemcpy(&err, c->d_err, sizeof(int), cudaMemcpyDeviceToHost));
  if (err) {
    set_error("device watchdog fired (code %d): a CNN pipeline barrier timed out", err);
    c->poisoned = true;
    return PNPULA_E_CUDA;
  }
  if (c->comm) {
    ncclResult_t ae;
    NC(c, ncclCommGetAsyncError(c->comm, &ae));
    if (ae != ncclSuccess) return fail_nccl(c, ae, "async", __LINE__);
  }
  return PNPULA_OK;
}

pnpula_status pnpula_run(pnpula_ctx *c, int64_t n_iter, int64_t burn_in, uint64_t seed) {
  pnpula_status s = pnpula_reset(c, burn_in, seed);
  if (s) return s;
  s = pnpula_advance(c, n_iter);
  if (s) return s;
  return pnpula_synchronize(c);
}

pnpula_status pnpula_local_bbox(pnpula_ctx *c, pnpula_rect *out) {
  pnpula_status s = check_ctx(c);
  if (s) return s;
  if (!out) { set_error("null output"); return PNPULA_E_INVALID_ARG; }
  *out = c->bbox;
  return PNPULA_OK;
}

pnpula_status pnpula_tile_info(pnpula_ctx *c, int32_t li, pnpula_rect *rect, int32_t *n_local, int32_t *halo) {
  pnpula_status s = check_ctx(c);
  if (s) return s;
  if (n_local) *n_local = c->n_local;
  if (halo) *halo = c->h;
  if (rect) {
    if (li < 0 || li >= c->n_local) { set_error("tile index out of range"); return PNPULA_E_INVALID_ARG; }
    const TileGeom &g = c->tiles[li].g;
    *rect = {g.i0, g.j0, g.th, g.tw};
  }
  return PNPULA_OK;
}

}  // extern "C"

namespace {

// Gather per-tile contiguous fields (count per tile = th*tw*nf floats) into host
// buffers covering `dst_rect`; remote tiles travel to root over NCCL.
pnpula_status gather_fields(pnpula_ctx *c, const std::vector<float *> &d_tile_bufs, int nf,
                            const std::vector<float *> &host_out, const pnpula_rect &dst_rect, bool global) {
  const int per_rank = c->ntiles / c->world;
  // own tiles: one strided device -> host copy per field straight into the caller's buffer
  // (full-rate DMA when the buffer is pinned; no staging vector, no per-row memcpy)
  for (int li = 0; li < c->n_local; ++li) {
    const TileGeom &g = c->tiles[li].g;
    if (global && c->rank != 0) break;
    for (int f = 0; f < nf; ++f) {
      float *o = host_out[f];
      if (!o) continue;
      CU(c, cudaMemcpy2DAsync(o + (size_t)(g.i0 - dst_rect.i0) * dst_rect.w + (g.j0 - dst_rect.j0),
                              (size_t)dst_rect.w * sizeof(float), d_tile_bufs[li] + (size_t)f * g.th * g.tw,
                              (size_t)g.tw * sizeof(float), (size_t)g.tw * sizeof(float), g.th,
                              cudaMemcpyDeviceToHost, c->stream));
    }
  }
  if (!global || c->world == 1) {
    CU(c, cudaStreamSynchronize(c->stream));
    return PNPULA_OK;
  }
  // remote tiles -> rank 0: one NCCL group of receives into a device buffer that lives in the
  // context's gather area (grown once, reused by later calls), then one strided D2H copy per
  // tile and field straight into the caller's buffer (DMA at full rate when it is pinned), one
  // synchronisation at the end.  Senders group their tiles the same way.
  if (c->rank == 0) {
    size_t total = 0;
    for (int t = per_rank; t < c->ntiles; ++t) {
      pnpula_rect r;
      tile_rect(c->ny, c->nx, c->tiles_y, c->tiles_x, t, &r);
      total += (size_t)r.h * r.w * nf;
    }
    if (total * sizeof(float) > c->gather_bytes) {
      dfree(c, c->gather_buf);
      c->gather_buf = nullptr;
      c->gather_bytes = 0;
      CU(c, dmalloc(c, &c->gather_buf, total * sizeof(float)));
      c->gather_bytes = total * sizeof(float);
    }
    float *d = static_cast<float *>(c->gather_buf);
    NC(c, ncclGroupStart());
    size_t off = 0;
    for (int t = per_rank; t < c->ntiles; ++t) {
      pnpula_rect r;
      tile_rect(c->ny, c->nx, c->tiles_y, c->tiles_x, t, &r);
      const size_t cnt = (size_t)r.h * r.w * nf;
      NC(c, ncclRecv(d + off, cnt, ncclFloat32, t / per_rank, c->comm, c->stream));
      off += cnt;
    }
    NC(c, ncclGroupEnd());
    off = 0;
    for (int t = per_rank; t < c->ntiles; ++t) {
      pnpula_rect r;
      tile_rect(c->ny, c->nx, c->tiles_y, c->tiles_x, t, &r);
      for (int f = 0; f < nf; ++f) {
        float *o = host_out[f];
        if (!o) continue;
        CU(c, cudaMemcpy2DAsync(o + (size_t)(r.i0 - dst_rect.i0) * dst_rect.w + (r.j0 - dst_rect.j0),
                                (size_t)dst_rect.w * sizeof(float), d + off + (size_t)f * r.h * r.w,
                                (size_t)r.w * sizeof(float), (size_t)r.w * sizeof(float), r.h,
                                cudaMemcpyDeviceToHost, c->stream));
      }
      off += (size_t)r.h * r.w * nf;
    }
  } else {
    NC(c, ncclGroupStart());
    for (int li = 0; li < c->n_local; ++li) {
      const TileGeom &g = c->tiles[li].g;
      NC(c, ncclSend(d_tile_bufs[li], (size_t)g.th * g.tw * nf, ncclFloat32, 0, c->comm, c->stream));
    }
    NC(c, ncclGroupEnd());
  }
  CU(c, cudaStreamSynchronize(c->stream));
  return PNPULA_OK;
}

// per-tile contiguous staging in the context's reusable device scratch (grown on demand)
pnpula_status tile_staging(pnpula_ctx *c, int nf, std::vector<float *> &bufs) {
  size_t total = 0;
  for (auto &td : c->tiles) total += (size_t)td.g.th * td.g.tw * nf;
  if (total * sizeof(float) > c->scratch_bytes) {
    dfree(c, c->scratch);
    c->scratch = nullptr;
    c->scratch_bytes = 0;
    CU(c, dmalloc(c, &c->scratch, total * sizeof(float)));
    c->scratch_bytes = total * sizeof(float);
  }
  float *d = static_cast<float *>(c->scratch);
  bufs.clear();
  for (auto &td : c->tiles) {
    bufs.push_back(d);
    d += (size_t)td.g.th * td.g.tw * nf;
  }
  return PNPULA_OK;
}

pnpula_status gather_padded_interiors1(pnpula_ctx *c, const std::vector<const float *> &src, float *host,
                                       bool global) {
  // pack interiors to contiguous, then gather
  std::vector<float *> bufs;
  pnpula_status s = tile_staging(c, 1, bufs);
  if (s) return s;
  for (int li = 0; li < c->n_local; ++li) {
    const TileGeom &g = c->tiles[li].g;
    CU(c, cudaMemcpy2DAsync(bufs[li], (size_t)g.tw * sizeof(float), src[li] + (size_t)g.h * g.pitch + g.hx,
                            (size_t)g.pitch * sizeof(float), (size_t)g.tw * sizeof(float), g.th,
                            cudaMemcpyDeviceToDevice, c->stream));
  }
  pnpula_rect dst = global ? pnpula_rect{0, 0, c->ny, c->nx} : c->bbox;
  return gather_fields(c, bufs, 1, {host}, dst, global);
}

// all channel planes of a per-tile padded field -> host [C][h][w]
pnpula_status gather_padded_interiors(pnpula_ctx *c, const std::vector<const float *> &src, float *host,
                                      bool global, int planes = -1) {
  if (planes < 0) planes = c->nc;
  const pnpula_rect dst = global ? pnpula_rect{0, 0, c->ny, c->nx} : c->bbox;
  for (int ch = 0; ch < planes; ++ch) {
    std::vector<const float *> s2;
    for (size_t li = 0; li < src.size(); ++li) s2.push_back(src[li] + (size_t)ch * geom_elems(c->tiles[li].g));
    float *h = (host && (!global || c->rank == 0)) ? host + (size_t)ch * dst.h * dst.w : host;
    pnpula_status s = gather_padded_interiors1(c, s2, h, global);
    if (s) return s;
  }
  return PNPULA_OK;
}

}  // namespace

extern "C" {

pnpula_status pnpula_get_moments(pnpula_ctx *c, float *mean, float *var, int64_t *n_samples, int32_t scope) {
  pnpula_status s = check_ctx(c);
  if (s) return s;
  if (!c->have_reset) { set_error("no chain has been run"); return PNPULA_E_STATE; }
  const bool global = scope == PNPULA_SCOPE_GLOBAL_ON_ROOT;
  CU(c, cudaSetDevice(c->device));
  const int64_t n = std::max<int64_t>(0, c->t - c->burn_in);
  if (n_samples) *n_samples = n;
  // GLOBAL scope with several ranks is collective: every rank gathers both fields, and its
  // outcome must not depend on which pointers a rank passes (non-root ranks pass NULL), or the
  // root would return while the other ranks block in ncclSend.  n is identical on every rank.
  const bool collective = global && c->world > 1;
  if ((collective && n < 2) || (mean && n < 1) || (var && n < 2)) {
    set_error("not enough post-burn-in samples (%lld)%s", (long long)n,
              collective ? "; GLOBAL_ON_ROOT with several ranks needs n >= 2 on every rank" : "");
    return PNPULA_E_STATS_EMPTY;
  }
  std::vector<float *> bufs;
  s = tile_staging(c, 2, bufs);
  if (s) return s;
  pnpula_rect dst = global ? pnpula_rect{0, 0, c->ny, c->nx} : c->bbox;
  const size_t dplane = (size_t)dst.h * dst.w;
  for (int ch = 0; ch < c->nc; ++ch) {   // one channel plane at a time (R43)
    for (size_t li = 0; li < c->tiles.size(); ++li) {
      auto &td = c->tiles[li];
      const TileGeom &g = td.g;
      const size_t o = (size_t)ch * geom_elems(g);
      float *d = bufs[li];
      FinalizeParams p{};
      p.mean = td.mean + o; p.m2 = td.m2 + o; p.g = g;
      p.out_mean = d; p.out_var = d + (size_t)g.th * g.tw;
      p.inv_nm1 = n >= 2 ? (float)(1.0 / (double)(n - 1)) : 0.f;
      CU(c, launch_finalize(p, c->stream));
    }
    const bool here = !global || c->rank == 0;
    s = gather_fields(c, bufs, 2, {mean && here ? mean + ch * dplane : mean, var && here ? var + ch * dplane : var},
                      dst, global);
    if (s) return s;
  }
  return PNPULA_OK;
}

pnpula_status pnpula_get_state(pnpula_ctx *c, float *x, float *z, int64_t *t, int32_t scope) {
  pnpula_status s = check_ctx(c);
  if (s) return s;
  CU(c, cudaSetDevice(c->device));
  const bool global = scope == PNPULA_SCOPE_GLOBAL_ON_ROOT;
  if (t) *t = c->t;
  std::vector<const float *> xs;
  for (auto &td : c->tiles) xs.push_back(td.x[c->cur]);
  s = gather_padded_interiors(c, xs, x, global);
  if (s) return s;
  if (c->rho > 0) {
    std::vector<const float *> zs;
    for (auto &td : c->tiles) zs.push_back(td.z);
    s = gather_padded_interiors(c, zs, z, global);
  } else if (z && (!global || c->rank == 0)) {
    pnpula_rect d = global ? pnpula_rect{0, 0, c->ny, c->nx} : c->bbox;
    memset(z, 0, (size_t)d.h * d.w * c->nc * sizeof(float));
  }
  return s;
}

pnpula_status pnpula_get_z1(pnpula_ctx *c, float *z1, int32_t scope) {
  pnpula_status s = check_ctx(c);
  if (s) return s;
  if (c->op != PNPULA_OP_POISSON) { set_error("z1 exists only for OP_POISSON"); return PNPULA_E_STATE; }
  CU(c, cudaSetDevice(c->device));
  std::vector<const float *> zs;
  for (auto &td : c->tiles) zs.push_back(td.z1);
  return gather_padded_interiors(c, zs, z1, scope == PNPULA_SCOPE_GLOBAL_ON_ROOT);
}

namespace {
constexpr uint64_t kCkptMagic = 0x31544b504c554e50ull;   // "PNULPKT1"
struct CkptHeader {
  uint64_t magic;
  int64_t t, burn_in;
  uint64_t seed;
  int32_t ny, nx, tiles_y, tiles_x, rank, world, n_local, nfields;
  uint64_t elems_total;   // floats after the header
};
// the fields of one tile, in blob order (x^t first)
std::vector<float *> ckpt_fields(pnpula_ctx *c, TileDev &td) {
  std::vector<float *> f{td.x[c->cur], td.mean, td.m2};
  if (td.z) f.push_back(td.z);
  if (td.z1) f.push_back(td.z1);
  if (td.zh) f.push_back(td.zh);
  return f;
}
uint64_t ckpt_bytes(pnpula_ctx *c) {
  uint64_t n = 0;
  for (auto &td : c->tiles) n += (uint64_t)geom_elems(td.g) * c->nc * ckpt_fields(c, td).size();
  return sizeof(CkptHeader) + n * sizeof(float);
}
}  // namespace

pnpula_status pnpula_checkpoint_bytes(pnpula_ctx *c, uint64_t *bytes) {
  pnpula_status s = check_ctx(c);
  if (s) return s;
  if (!bytes) { set_error("null output"); return PNPULA_E_INVALID_ARG; }
  *bytes = ckpt_bytes(c);
  return PNPULA_OK;
}

pnpula_status pnpula_save_checkpoint(pnpula_ctx *c, void *buf, uint64_t bytes) {
  pnpula_status s = check_ctx(c);
  if (s) return s;
  if (!c->have_reset) { set_error("no chain to checkpoint (pnpula_reset first)"); return PNPULA_E_STATE; }
  if (!buf || bytes < ckpt_bytes(c)) { set_error("checkpoint buffer too small"); return PNPULA_E_INVALID_ARG; }
  CU(c, cudaSetDevice(c->device));
  CkptHeader h{kCkptMagic, c->t, c->burn_in, c->seed, c->ny, c->nx, c->tiles_y, c->tiles_x, c->rank, c->world,
               c->n_local, (int32_t)(c->tiles.empty() ? 0 : ckpt_fields(c, c->tiles[0]).size()),
               (ckpt_bytes(c) - sizeof(CkptHeader)) / sizeof(float)};
  memcpy(buf, &h, sizeof(h));
  float *dst = reinterpret_cast<float *>(static_cast<char *>(buf) + sizeof(h));
  for (auto &td : c->tiles) {
    const size_t n = geom_elems(td.g) * c->nc;
    for (float *f : ckpt_fields(c, td)) {
      CU(c, cudaMemcpyAsync(dst, f, n * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
      dst += n;
    }
  }
  CU(c, cudaStreamSynchronize(c->stream));
  return PNPULA_OK;
}

pnpula_status pnpula_load_checkpoint(pnpula_ctx *c, const void *buf, uint64_t bytes) {
  pnpula_status s = check_ctx(c);
  if (s) return s;
  if (!buf || bytes < sizeof(CkptHeader)) { set_error("checkpoint buffer too small"); return PNPULA_E_INVALID_ARG; }
  CkptHeader h;
  memcpy(&h, buf, sizeof(h));
  const uint64_t need = ckpt_bytes(c);   // independent of c->cur
  if (h.magic != kCkptMagic || h.ny != c->ny || h.nx != c->nx || h.tiles_y != c->tiles_y || h.tiles_x != c->tiles_x ||
      h.rank != c->rank || h.world != c->world || h.n_local != c->n_local ||
      h.elems_total != (need - sizeof(CkptHeader)) / sizeof(float) ||
      h.nfields != (int32_t)(c->tiles.empty() ? 0 : ckpt_fields(c, c->tiles[0]).size())) {
    set_error("checkpoint does not match this context (geometry, rank or state fields)");
    return PNPULA_E_SHAPE;
  }
  if (bytes < need) { set_error("checkpoint truncated"); return PNPULA_E_INVALID_ARG; }
  CU(c, cudaSetDevice(c->device));
  // every check passed: only now switch the live context (the restored x^t goes to buffer 0);
  // a rejected blob leaves the chain exactly as it was
  drop_graphs(c);
  c->cur = 0;
  const float *src = reinterpret_cast<const float *>(static_cast<const char *>(buf) + sizeof(h));
  for (auto &td : c->tiles) {
    const size_t n = geom_elems(td.g) * c->nc;
    for (float *f : ckpt_fields(c, td)) {
      CU(c, cudaMemcpyAsync(f, src, n * sizeof(float), cudaMemcpyHostToDevice, c->stream));
      src += n;
    }
  }
  CU(c, cudaStreamSynchronize(c->stream));
  c->t = h.t;
  c->burn_in = h.burn_in;
  c->seed = h.seed;
  c->have_reset = true;
  return PNPULA_OK;
}

pnpula_status pnpula_opnorm2(pnpula_ctx *c, int32_t iters, double *out) {
  pnpula_status s = check_ctx(c);
  if (s) return s;
  if (!out || iters < 2) { set_error("need an output and iters >= 2"); return PNPULA_E_INVALID_ARG; }
  if (c->op == PNPULA_OP_MASK) { *out = 1.0; return PNPULA_OK; }   // diag(m), m in {0, 1}
  CU(c, cudaSetDevice(c->device));
  const int vb = c->cur ^ 1;   // the iterate lives in the idle x buffer (rewritten by the next step)
  std::vector<float *> tmp;
  double *d_acc = nullptr;
  auto cleanup = [&]() {
    for (float *t : tmp) cudaFree(t);
    if (d_acc) cudaFree(d_acc);
  };
  auto params = [&](TileDev &td, int li) {
    OpNormParams q{};
    q.v = td.x[vb];
    q.w = tmp[2 * li];
    q.u = tmp[2 * li + 1];
    q.acc = d_acc;
    q.g = td.g;
    q.ny = c->ny; q.nx = c->nx; q.ry = c->ry; q.rx = c->rx;
    const int kh = 2 * c->ry + 1, kw = 2 * c->rx + 1;
    for (int a = 0; a < kh; ++a)
      for (int b = 0; b < kw; ++b) q.k2d[a * kw + b] = c->separable ? c->ky[a] * c->kx[b] : c->k2d[a * kw + b];
    return q;
  };
  for (auto &td : c->tiles) {
    const size_t n = geom_elems(td.g) * sizeof(float);
    for (int i = 0; i < 2; ++i) {
      float *t = nullptr;
      cudaError_t e = cudaMalloc(&t, n);
      if (e == cudaSuccess) e = cudaMemsetAsync(t, 0, n, c->stream);
      if (e != cudaSuccess) { cleanup(); return fail_cuda(c, e, "opnorm buffers", __LINE__); }
      tmp.push_back(t);
    }
  }
  cudaError_t e = cudaMalloc(&d_acc, 3 * sizeof(double));
  if (e != cudaSuccess) { cleanup(); return fail_cuda(c, e, "opnorm acc", __LINE__); }
  double lam = 0.0;
  for (int li = 0; li < c->n_local; ++li) {
    e = launch_opnorm(0, params(c->tiles[li], li), nullptr, c->stream);
    if (e != cudaSuccess) { cleanup(); return fail_cuda(c, e, "opnorm init", __LINE__); }
  }
  s = exchange(c, vb);
  for (int it = 0; it < iters && !s; ++it) {
    e = cudaMemsetAsync(d_acc, 0, 2 * sizeof(double), c->stream);
    for (int li = 0; li < c->n_local && e == cudaSuccess; ++li) e = launch_opnorm(1, params(c->tiles[li], li), nullptr, c->stream);
    for (int li = 0; li < c->n_local && e == cudaSuccess; ++li) e = launch_opnorm(2, params(c->tiles[li], li), nullptr, c->stream);
    if (e != cudaSuccess) { cleanup(); return fail_cuda(c, e, "opnorm iteration", __LINE__); }
    if (c->world > 1) {
      ncclResult_t r = ncclAllReduce(d_acc, d_acc, 2, ncclFloat64, ncclSum, c->comm, c->stream);
      if (r != ncclSuccess) { cleanup(); return fail_nccl(c, r, "ncclAllReduce", __LINE__); }
    }
    double h[2];
    e = cudaMemcpyAsync(h, d_acc, 2 * sizeof(double), cudaMemcpyDeviceToHost, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) { cleanup(); return fail_cuda(c, e, "opnorm sums", __LINE__); }
    // v has unit norm from the second iteration on: Rayleigh quotient u.v = v^T H^T H v
    if (it > 0) lam = h[1];
    const double sc = h[0] > 0 ? 1.0 / std::sqrt(h[0]) : 0.0;
    e = cudaMemcpyAsync(d_acc + 2, &sc, sizeof(double), cudaMemcpyHostToDevice, c->stream);
    for (int li = 0; li < c->n_local && e == cudaSuccess; ++li) e = launch_opnorm(3, params(c->tiles[li], li), d_acc + 2, c->stream);
    if (e != cudaSuccess) { cleanup(); return fail_cuda(c, e, "opnorm scale", __LINE__); }
    s = exchange(c, vb);
    if (!s) { e = cudaStreamSynchronize(c->stream); if (e != cudaSuccess) { cleanup(); return fail_cuda(c, e, "opnorm sync", __LINE__); } }
  }
  cleanup();
  if (s) return s;
  *out = lam;
  return PNPULA_OK;
}

pnpula_status pnpula_conv_norm2_bound(const float *k, int32_t kh, int32_t kw, int32_t grid, double *out) {
  if (!k || !out || kh <= 0 || kw <= 0 || grid < std::max(kh, kw)) {
    set_error("bad kernel / grid"); return PNPULA_E_INVALID_ARG;
  }
  double best = 0;
  const double w0 = 2.0 * M_PI / grid;
  for (int u = 0; u < grid; ++u)
    for (int v = 0; v < grid; ++v) {
      double re = 0, im = 0;
      for (int p = 0; p < kh; ++p)
        for (int q = 0; q < kw; ++q) {
          const double ph = w0 * ((double)u * p + (double)v * q);
          re += k[p * kw + q] * std::cos(ph);
          im -= k[p * kw + q] * std::sin(ph);
        }
      best = std::max(best, re * re + im * im);
    }
  *out = best;
  return PNPULA_OK;
}

pnpula_status pnpula_get_tv_zh(pnpula_ctx *c, float *zh, int32_t scope) {
  pnpula_status s = check_ctx(c);
  if (s) return s;
  if (!(c->tv_beta > 0)) { set_error("z_h exists only with the TV prior"); return PNPULA_E_STATE; }
  CU(c, cudaSetDevice(c->device));
  std::vector<const float *> zs;
  for (auto &td : c->tiles) zs.push_back(td.zh);
  return gather_padded_interiors(c, zs, zh, scope == PNPULA_SCOPE_GLOBAL_ON_ROOT);
}

pnpula_status pnpula_get_padded_x(pnpula_ctx *c, int32_t li, float *out) {
  pnpula_status s = check_ctx(c);
  if (s) return s;
  if (li < 0 || li >= c->n_local || !out) { set_error("bad tile index / null output"); return PNPULA_E_INVALID_ARG; }
  CU(c, cudaSetDevice(c->device));
  const TileGeom &g = c->tiles[li].g;
  const int w = g.tw + 2 * g.h;
  CU(c, cudaMemcpy2DAsync(out, (size_t)w * sizeof(float), c->tiles[li].x[c->cur] + (g.hx - g.h),
                          (size_t)g.pitch * sizeof(float), (size_t)w * sizeof(float), g.ph,
                          cudaMemcpyDeviceToHost, c->stream));
  CU(c, cudaStreamSynchronize(c->stream));
  return PNPULA_OK;
}

pnpula_status pnpula_get_denoiser_residual(pnpula_ctx *c, float *G) {
  pnpula_status s = check_ctx(c);
  if (s) return s;
  if (c->n_layers == 0) { set_error("no denoiser configured"); return PNPULA_E_STATE; }
  if (!c->have_reset) { set_error("pnpula_reset must precede this call"); return PNPULA_E_STATE; }
  CU(c, cudaSetDevice(c->device));
  s = run_cnn(c, c->cur);
  if (s) return s;
  s = pnpula_synchronize(c);
  if (s) return s;
  std::vector<const float *> gs;
  for (auto &td : c->tiles) gs.push_back(td.G);
  return gather_padded_interiors(c, gs, G, false);
}

pnpula_status pnpula_set_timing(pnpula_ctx *c, int32_t enable) {
  pnpula_status s = check_ctx(c);
  if (s) return s;
  c->timing = enable != 0;
  return PNPULA_OK;
}

pnpula_status pnpula_kernel_time(pnpula_ctx *c, const char *name, double *ms, int64_t *launches, int32_t reset) {
  pnpula_status s = check_ctx(c);
  if (s) return s;
  Timer *t = nullptr;
  if (!name) { set_error("null name"); return PNPULA_E_INVALID_ARG; }
  if (!strcmp(name, "all")) {   // every kernel this library launched (timing not needed)
    if (ms) *ms = 0.0;
    if (launches) *launches = c->n_launches;
    if (reset) c->n_launches = 0;
    return PNPULA_OK;
  }
  if (!strcmp(name, "cnn")) t = &c->tm_cnn;
  else if (!strcmp(name, "update")) t = &c->tm_update;
  else if (!strcmp(name, "halo")) t = &c->tm_halo;
  else { set_error("unknown timer '%s'", name); return PNPULA_E_INVALID_ARG; }
  timer_collect(*t);
  if (ms) *ms = t->ms;
  if (launches) *launches = t->launches;
  if (reset) { t->ms = 0; t->launches = 0; }
  return PNPULA_OK;
}

pnpula_status pnpula_debug_philox(int32_t device, uint64_t seed, const uint32_t *counters, int64_t n,
                                  uint32_t *words, float *normals) {
  if (!counters || !words || !normals || n < 0) { set_error("null argument / negative n"); return PNPULA_E_INVALID_ARG; }
  if (n == 0) return PNPULA_OK;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return fail_cuda(nullptr, e, "cudaSetDevice", __LINE__);
  uint32_t *dc = nullptr, *dw = nullptr;
  float *dn = nullptr;
  int *dbad = nullptr;
  const size_t b4 = (size_t)n * 4 * sizeof(uint32_t);
  int bad = 0;
  e = cudaMalloc(&dc, b4);
  if (e == cudaSuccess) e = cudaMalloc(&dw, b4);
  if (e == cudaSuccess) e = cudaMalloc(&dn, b4);
  if (e == cudaSuccess) e = cudaMalloc(&dbad, sizeof(int));
  if (e == cudaSuccess) e = cudaMemset(dbad, 0, sizeof(int));
  if (e == cudaSuccess) e = cudaMemcpy(dc, counters, b4, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = launch_debug_philox(seed, dc, n, dw, dn, dbad, nullptr);
  if (e == cudaSuccess) e = cudaMemcpy(words, dw, b4, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(normals, dn, b4, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(&bad, dbad, sizeof(int), cudaMemcpyDeviceToHost);
  cudaFree(dc); cudaFree(dw); cudaFree(dn); cudaFree(dbad);
  if (e != cudaSuccess) return fail_cuda(nullptr, e, "pnpula_debug_philox", __LINE__);
  if (bad) { set_error("normals4 and normals4x2 differ on %d counters", bad); return PNPULA_E_STATE; }
  return PNPULA_OK;
}

pnpula_status pnpula_release_memory(int32_t device) {
  cudaMemPool_t p = device_pool(device);
  if (!p) { set_error("no memory pool for device %d", device); return PNPULA_E_INVALID_ARG; }
  cudaError_t e = cudaMemPoolTrimTo(p, 0);
  if (e != cudaSuccess) { set_error("cudaMemPoolTrimTo: %s", cudaGetErrorString(e)); return PNPULA_E_CUDA; }
  return PNPULA_OK;
}

pnpula_status pnpula_destroy(pnpula_ctx *c) {
  if (!c) return PNPULA_OK;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (auto &td : c->tiles) {
    for (void *q : {(void *)td.x[0], (void *)td.x[1], (void *)td.x0, (void *)td.y, (void *)td.mask, (void *)td.z,
                    (void *)td.z1, (void *)td.zh, (void *)td.mean, (void *)td.m2, (void *)td.G, (void *)td.pbuf, (void *)td.pbuf2,
                    (void *)td.act[0], (void *)td.act[1]})
      dfree(c, q);
  }
  for (auto p : c->d_w) cudaFree(p);
  for (auto p : c->d_b) cudaFree(p);
  dfree(c, c->scratch);
  dfree(c, c->gather_buf);
  if (c->pool && c->stream) cudaStreamSynchronize(c->stream);
  cudaFree(c->ddfb_u0); cudaFree(c->ddfb_fin);
  for (auto p : c->ddfb_t) cudaFree(p);
  for (auto p : c->ddfb_adj) cudaFree(p);
  for (int b = 0; b < 2; ++b) {
    cudaFree(c->d_local_jobs[b]); cudaFree(c->d_pack_jobs[b]); cudaFree(c->d_unpack_jobs[b]);
  }
  cudaFree(c->d_sendbuf); cudaFree(c->d_recvbuf); cudaFree(c->d_err);
  drop_graphs(c);
  cudaFree(c->d_iter);
  if (c->comm_stream) { cudaStreamSynchronize(c->comm_stream); cudaStreamDestroy(c->comm_stream); }
  if (c->ev_bands) cudaEventDestroy(c->ev_bands);
  if (c->ev_halo) cudaEventDestroy(c->ev_halo);
  for (Timer *t : {&c->tm_cnn, &c->tm_update, &c->tm_halo})
    for (auto &e : t->ev) { cudaEventDestroy(e.first); cudaEventDestroy(e.second); }
  if (c->comm) ncclCommDestroy(c->comm);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  delete c;
  return PNPULA_OK;
}

}  // extern "C"
