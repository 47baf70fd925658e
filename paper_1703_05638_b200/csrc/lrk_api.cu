// lrk_api.cu — C ABI (include/lrk.h): context, workspace, and the host-side
// orchestration of each reference entry point over the device kernels.
// No host<->device synchronisation happens inside an apply except where the
// ABI returns host values (ranks, traces, inner products) at the very end.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "../../include/lrk.h"
#include "lrk_device.cuh"
#include "lrk_kernels.h"
#include "lrk_sflush.h"
#include "lrk_misc.h"

using namespace lrk;

namespace {
struct Buf {
  void* p = nullptr;
  size_t bytes = 0;
  bool ext = false;  // lives in the peer-shared arena: never freed or regrown here
};
// n_x sharding across processes (one per GPU): this rank's shard index, the
// peer-mapped arenas (exchange buffer + the two sweep panes) of all ranks.
struct Dist {
  int rank = 0, world = 1;
  char* arena = nullptr;
  size_t bytes = 0, off_f = 0, off_b = 0;
  int64_t pane_doubles = 0;
  char* peer[SF_XMAXR] = {};
  bool connected = false;
};
}  // namespace

struct lrk_ctx {
  int device = 0;
  int num_sms = 148;
  int smem_optin = 227 * 1024;
  std::string err;
  int64_t launches = 0;
  // operator
  bool has_op = false;
  lrk_operator_desc op{};
  int64_t n_x = 0;
  int64_t ldp = 0;            // padded leading dimension of n_x-row workspace (see padld)
  int n = 0;
  double* dS = nullptr;       // n x n DST-I (symmetric, orthogonal)
  double* dSsq = nullptr;     // n x n elementwise square of the DST-I (operator diagonals)
  double* dTheta = nullptr;   // n_x: eigenvalues of S^{-1} M  = 1/(1+tau*lambda)
  double* dThetaM = nullptr;  // n_x: theta / m_scale (eigenvalues of S^{-1})
  double* dE0 = nullptr;      // n_t: e_0
  double* dInvLam = nullptr;  // n_x: 1/lambda (steady Poisson solve)
  double* dLam = nullptr;     // n_x: lambda (config prior (delta + gamma lambda)^{-1})
  int emu_shards = 1;         // sweeps as G emulated n_x shards (one launch, tests)
  Dist dist;                  // n_x sharding across processes (lrk_shard_setup)
  unsigned long long xseq = 0;  // exchange sequence number of the sharded streaming sweep
  int rich_it = 0;            // physical step solves: Richardson sweeps (0 unknown, -1 GMRES)
  double rich_q = 1.0;        // measured contraction of I - P^{-1} S
  // observation
  bool has_obs = false;
  int obs_kind = LRK_OBS_FULL;
  int n_obs = 0, s1 = 0, s2 = 0;
  int32_t* dList = nullptr;
  double *dS1T = nullptr, *dS2 = nullptr, *dS1 = nullptr, *dS2T = nullptr;
  std::map<std::string, Buf> ws;
  // instrumentation
  bool prof = false;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  lrk::SFAux aux{};           // second stream of the streaming-flush sweep
  double prof_ms = 0.0, prof_bytes = 0.0;
  int64_t prof_n = 0;
  std::vector<int> last_fwd, last_bwd;
  int last_obs = 0;
  ~lrk_ctx() {
    for (auto& e : ev) if (e) cudaEventDestroy(e);
    if (aux.ready) cudaEventDestroy(aux.ready);
    if (aux.done) cudaEventDestroy(aux.done);
    if (aux.stream) cudaStreamDestroy(aux.stream);
    for (auto& kv : ws) if (!kv.second.ext) cudaFree(kv.second.p);
    for (int q = 0; q < SF_XMAXR; ++q)
      if (dist.peer[q] && q != dist.rank) cudaIpcCloseMemHandle(dist.peer[q]);
    cudaFree(dist.arena);
    cudaFree(dS); cudaFree(dTheta); cudaFree(dThetaM); cudaFree(dE0); cudaFree(dInvLam);
    cudaFree(dLam); cudaFree(dSsq);
    cudaFree(dList); cudaFree(dS1T); cudaFree(dS2); cudaFree(dS1); cudaFree(dS2T);
  }
};

namespace {

int fail(lrk_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  return code;
}

#define CK(expr)                                                                   \
  do {                                                                             \
    cudaError_t e_ = (expr);                                                       \
    if (e_ != cudaSuccess)                                                         \
      return fail(c, LRK_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

#define CKL()                                                                      \
  do {                                                                             \
    ++c->launches;                                                                 \
    cudaError_t e_ = cudaGetLastError();                                           \
    if (e_ != cudaSuccess)                                                         \
      return fail(c, LRK_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e_)); \
  } while (0)

#define TRY(expr)                 \
  do {                            \
    int st_ = (expr);             \
    if (st_ != LRK_OK) return st_; \
  } while (0)

template <typename T>
T* wsp(lrk_ctx* c, const std::string& name, size_t count, bool zero = false) {
  Buf& b = c->ws[name];
  const size_t need = count * sizeof(T) + 256;
  if (b.bytes < need) {
    if (b.ext) {
      c->err = "peer-shared workspace " + name + " is too small for this call";
      return nullptr;
    }
    if (b.p) {
      cudaDeviceSynchronize();
      cudaFree(b.p);
      b.p = nullptr;
      b.bytes = 0;
    }
    if (cudaMalloc(&b.p, need) != cudaSuccess) {
      cudaGetLastError();
      c->err = "cudaMalloc failed for workspace " + name;
      return nullptr;
    }
    b.bytes = need;
    cudaMemset(b.p, 0, need);
  } else if (zero) {
    cudaMemset(b.p, 0, need);
  }
  return static_cast<T*>(b.p);
}

#define WS(T, var, name, count)                                                      \
  T* var = wsp<T>(c, name, (size_t)(count));                                         \
  if (!var) return LRK_ERR_CUDA;

inline int grid1(int64_t n, int per = 256, int cap = 4096) {
  int64_t g = (n + per - 1) / per;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

// Leading dimension for n_x-row, multi-column workspace: column starts are
// staggered (+2.25 KB) so that the columns of a large power-of-two n_x do not
// all map onto the same DRAM channels (C4: n_x = 2^21, a 16 MiB column stride).
int64_t padld(int64_t n) {
  static const int64_t extra = std::getenv("LRK_LDPAD") ? std::atoll(std::getenv("LRK_LDPAD")) : 288;
  if (n < 4096) return n;
  return ((n + 31) / 32) * 32 + extra;
}

int pick_ncta(lrk_ctx* c, int64_t rows) {
  int64_t k = rows / 384;
  if (k < 1) k = 1;
  if (k > c->num_sms) k = c->num_sms;
  return (int)k;
}

// --------------------------------------------------------------- GEMMs
int gemm(lrk_ctx* c, int M, int N, int K, const double* A, int64_t lda, int64_t sA,
         const double* B, int64_t ldb, int64_t sB, double* C, int64_t ldc, int64_t sC,
         double alpha, int batch, const int* batch_dev, cudaStream_t s, int batch_mult = 1,
         const double* emul = nullptr, int64_t lde = 0, double beta = 0.0) {
  GemmArgs g{};
  g.M = M; g.N = N; g.K = K;
  g.A = A; g.lda = lda; g.sA = sA;
  g.B = B; g.ldb = ldb; g.sB = sB;
  g.C = C; g.ldc = ldc; g.sC = sC;
  g.alpha = alpha; g.beta = beta;
  g.emul = emul; g.lde = lde;
  g.batch = batch; g.batch_dev = batch_dev; g.batch_mult = batch_mult;
  g.m_dev = nullptr; g.m_mult = 1;
  CK(launch_gemm(g, s));
  ++c->launches;
  return LRK_OK;
}

// Y[:, j] = alpha * (S (x) S [(x) S]) X[:, j]: 2-D or 3-D DST-I of each column
// (x1 fastest), one DMMA GEMM pass per axis.
// Optional epilogue on the last pass: Y = alpha * DST(X) .* emul + beta * Y
// (emul: an n_x array in the x1-fastest layout, shared by all columns).
int dst2(lrk_ctx* c, const double* X, int64_t ldx, double* Y, int64_t ldy, int ncols,
         const int* ncols_dev, double alpha, cudaStream_t s, const double* emul = nullptr,
         double beta = 0.0, const double* Smat = nullptr) {
  if (ncols <= 0) return LRK_OK;
  const int n = c->n;
  const int64_t nx = c->n_x;
  const double* dS = Smat ? Smat : c->dS;  // per-axis transform (DST-I, or S∘S for diagonals)
  WS(double, T, "dst_T", nx * (int64_t)ncols);
  if (c->op.dim == 2) {
    // T_j = X_j S      (X_j: n x n row-major view of column j)
    TRY(gemm(c, n, n, n, X, n, ldx, dS, n, 0, T, n, nx, 1.0, ncols, ncols_dev, s));
    // Y_j = alpha S T_j
    TRY(gemm(c, n, n, n, dS, n, 0, T, n, nx, Y, n, ldy, alpha, ncols, ncols_dev, s, 1, emul,
             n, beta));
    return LRK_OK;
  }
  const int64_t pl = (int64_t)n * n;
  WS(double, T2, "dst_T2", nx * (int64_t)ncols);
  // x1: T_j = X_j S, X_j viewed as (n^2) x n row-major
  TRY(gemm(c, (int)pl, n, n, X, n, ldx, dS, n, 0, T, n, nx, 1.0, ncols, ncols_dev, s));
  // x2: per (column, x3-plane) slice: T2 = S T_slice  (batch ncols * n, stride n^2)
  TRY(gemm(c, n, n, n, dS, n, 0, T, n, pl, T2, n, pl, 1.0, ncols * n, ncols_dev, s, n));
  // x3: Y_j = alpha S T2_j, T2_j viewed as n x (n^2) row-major
  TRY(gemm(c, n, (int)pl, n, dS, n, 0, T2, pl, nx, Y, pl, ldy, alpha, ncols, ncols_dev, s, 1,
           emul, pl, beta));
  return LRK_OK;
}

// Uobs_j = S[i2,:] Xhat_j S[:,i1]   (sensor-subgrid values of a spectral column)
int subgrid_gather(lrk_ctx* c, const double* X, int64_t ldx, double* Y, int64_t ldy, int ncols,
                   const int* ncols_dev, cudaStream_t s) {
  const int n = c->n, s1 = c->s1, s2 = c->s2;
  WS(double, T, "sg_T", (int64_t)n * s1 * ncols);
  TRY(gemm(c, n, s1, n, X, n, ldx, c->dS1T, s1, 0, T, s1, (int64_t)n * s1, 1.0, ncols, ncols_dev, s));
  TRY(gemm(c, s2, s1, n, c->dS2, n, 0, T, s1, (int64_t)n * s1, Y, s1, ldy, 1.0, ncols, ncols_dev, s));
  return LRK_OK;
}

// Zhat_j = S[:,i2] Z_j S[i1,:]   (spectral image of a sensor-subgrid field)
int subgrid_scatter(lrk_ctx* c, const double* Z, int64_t ldz, double* Y, int64_t ldy, int ncols,
                    const int* ncols_dev, cudaStream_t s) {
  const int n = c->n, s1 = c->s1, s2 = c->s2;
  WS(double, T, "ss_T", (int64_t)s2 * n * ncols);
  TRY(gemm(c, s2, n, s1, Z, s1, ldz, c->dS1, n, 0, T, n, (int64_t)s2 * n, 1.0, ncols, ncols_dev, s));
  TRY(gemm(c, n, n, s2, c->dS2T, s2, 0, T, n, (int64_t)s2 * n, Y, n, ldy, 1.0, ncols, ncols_dev, s));
  return LRK_OK;
}

// Box-stencil coefficients of S = m (I + tau L) for the installed operator
// (discretize.py:90-127 and the config extensions), mirrored for S^T.
StencilArgs make_stencil(const lrk_operator_desc& op, bool adjoint) {
  StencilArgs a{};
  const double h = op.h, ih2 = 1.0 / (h * h);
  auto cf = [&](int d1, int d2, int d3) -> double& { return a.coef[(d3 + 1) * 9 + (d2 + 1) * 3 + (d1 + 1)]; };
  const double sc = op.kind == LRK_OP_HEAT ? 1.0 : op.nu;
  if (op.stencil == LRK_STENCIL_Q1) {
    // K_Q1 / h^2 with lumped mass: centre 8/3, all eight neighbours -1/3
    for (int d2 = -1; d2 <= 1; ++d2)
      for (int d1 = -1; d1 <= 1; ++d1) cf(d1, d2, 0) = -sc * ih2 / 3.0;
    cf(0, 0, 0) = 8.0 * sc * ih2 / 3.0;
  } else {
    cf(0, 0, 0) = 2.0 * op.dim * sc * ih2;
    cf(-1, 0, 0) = cf(1, 0, 0) = cf(0, -1, 0) = cf(0, 1, 0) = -sc * ih2;
    if (op.dim == 3) cf(0, 0, -1) = cf(0, 0, 1) = -sc * ih2;
    if (op.kind != LRK_OP_HEAT && op.wind_field == LRK_WIND_CONST) {
      // first-order upwind per axis by the sign of the wind (discretize.py:96-104)
      for (int ax = 0; ax < op.dim; ++ax) {
        const double w = op.wind[ax];
        int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
        lo[ax] = -1; hi[ax] = 1;
        if (w > 0) { cf(0, 0, 0) += w / h; cf(lo[0], lo[1], lo[2]) -= w / h; }
        else if (w < 0) { cf(0, 0, 0) -= w / h; cf(hi[0], hi[1], hi[2]) += w / h; }
      }
    }
  }
  if (adjoint)
    for (int k = 0; k < 13; ++k) std::swap(a.coef[k], a.coef[26 - k]);
  a.n = op.n_side; a.dim = op.dim; a.m_scale = op.m_scale; a.tau = op.tau;
  const bool galerkin = op.kind != LRK_OP_HEAT && op.stencil == LRK_STENCIL_Q1;
  a.wind_field = (op.kind != LRK_OP_HEAT && !galerkin) ? op.wind_field : 0;
  a.galerkin = galerkin ? 1 : 0;     // Galerkin Q1 convection, wind at the element centres
  a.rotating = galerkin && op.wind_field == LRK_WIND_ROTATING ? 1 : 0;
  a.adjoint = adjoint ? 1 : 0;
  a.w0[0] = op.wind[0]; a.w0[1] = op.wind[1]; a.w0[2] = op.wind[2];
  a.h = h;
  return a;
}

// ---------------------------------------------------------------- sweep
struct SweepOut {
  double* U = nullptr;  // n_x x ucap (slot 0)
  double* V = nullptr;  // n_t x ucap
  double* sigma = nullptr;
  int* info = nullptr;  // device [rank, which, err, pad]
  int* trace = nullptr; // device nflush+1
  int ucap = 0;
  int nflush = 0;
  int64_t ldu = 0, ldv = 0;
  long long* dbg = nullptr;
};

int run_sweep_phys(lrk_ctx* c, const std::string& tag, const double* B, int64_t ldb, int rb,
                   const int* rb_dev, const double* W2, int64_t ldw2, int adjoint, int p,
                   double eps0, int r_max, SweepOut& o, cudaStream_t s);

int run_sweep(lrk_ctx* c, const std::string& tag, const double* B, int64_t ldb, int rb,
              const int* rb_dev, const double* W2, int64_t ldw2, int adjoint, int p, double eps0,
              int r_max, SweepOut& o, cudaStream_t s) {
  if (p < 1 || p > PMAX)
    return fail(c, LRK_ERR_UNSUPPORTED, "compress_every must lie in [1, 16] on the device path");
  if (c->op.kind != LRK_OP_HEAT)
    return run_sweep_phys(c, tag, B, ldb, rb, rb_dev, W2, ldw2, adjoint, p, eps0, r_max, o, s);
  const int64_t nx = c->n_x;
  const int nt = c->op.n_t;
  const int ucap = (r_max >= 0 && r_max < NMAX) ? std::max(r_max, 1) : NMAX;
  const int ncta = pick_ncta(c, nx);
  const int nflush = (nt + p - 1) / p;
  const int64_t ld = padld(nx);
  WS(double, U0, tag + "U0", ld * (int64_t)ucap);
  WS(double, U1, tag + "U1", ld * (int64_t)ucap);
  WS(double, V0, tag + "V0", (int64_t)nt * ucap);
  WS(double, V1, tag + "V1", (int64_t)nt * ucap);
  WS(double, sig, tag + "sig", NMAX);
  WS(int, info, tag + "info", 8);
  WS(int, trace, tag + "trace", nflush + 1);
  WS(double, ybuf, "sw_ybuf", ld * (int64_t)p);
  WS(double, qbuf, "sw_qbuf", ld * (int64_t)p);
  WS(double, yprev, "sw_yprev", nx);
  // emulated n_x shards (lrk_set_emulated_shards): G groups of one launch
  // acting as G GPUs of a sharded sweep, ncta/G CTAs each
  int G = std::max(1, std::min(c->emu_shards, SHARD_MAX));
  if (ncta % G != 0 || ncta / G < 1) G = 1;
  const int ncg = ncta / G;
  const int64_t pst = sweep_part_stride();
  WS(double, part, "sw_part", 3 * (int64_t)ncta * pst);
  const int64_t sst = sweep_scratch_stride(ncta);
  WS(double, scratch, "sw_scratch", (int64_t)ncta * sst);
  WS(unsigned, bar, "sw_bar", 4);
  SweepBatch batch{};
  batch.ngroups = 1;
  SweepArgs& a = batch.g[0];
  a.nshard = 1; a.shard = 0; a.sys_fence = 0;
  a.spart[0] = part; a.gbar = bar;
  a.n_x = nx; a.n_t = nt; a.adjoint = adjoint; a.p = p; a.r_max = r_max; a.eps0 = eps0;
  a.theta = c->dTheta; a.rowscale = c->dThetaM;
  a.B = B; a.ldb = ldb; a.rb = rb; a.rb_dev = rb_dev;
  a.W2 = W2; a.ldw2 = ldw2;
  a.U0 = U0; a.U1 = U1; a.ldu = ld; a.V0 = V0; a.V1 = V1; a.ldv = nt; a.ucap = ucap;
  a.sigma = sig; a.info = info; a.trace = trace;
  a.ybuf = ybuf; a.ldy = ld; a.qbuf = qbuf; a.ldq = ld; a.yprev = yprev;
  a.part = part; a.pstride = pst; a.scratch = scratch; a.scratch_stride = sst;
  a.bar = bar; a.ncta = ncta;
  a.yext = nullptr; a.ldyext = 0;
  a.flush0 = 0; a.flush1 = nflush; a.r_init = 0;
  sweep_plan(a, nx, ncta, ucap, p, (size_t)c->smem_optin);
  a.ftz = std::getenv("LRK_FTZ") ? std::atof(std::getenv("LRK_FTZ")) : 0.0;
  WS(long long, dbg, tag + "dbg", 20);
  a.dbg = std::getenv("LRK_DEBUG") ? dbg : nullptr;
  a.nopipe = std::getenv("LRK_NOPIPE") ? 1 : 0;
  o.dbg = dbg;
  CK(cudaMemsetAsync(info, 0, 8 * sizeof(int), s));
  if (G > 1) {
    // shard g: its own replicated time factor, sigma/info/trace and scratch;
    // the n_x-row arrays are shared (disjoint rows), partials in one table
    WS(double, Vg, tag + "Vsh", 2 * (int64_t)G * nt * ucap);
    WS(double, sg, tag + "sigsh", (int64_t)G * NMAX);
    WS(int, ig, tag + "infosh", 8 * G);
    WS(int, tg, tag + "tracesh", (int64_t)G * (nflush + 1));
    CK(cudaMemsetAsync(ig, 0, 8 * G * sizeof(int), s));
    a.ncta = ncg;
    a.nshard = G;
    a.scratch_stride = sst;
    sweep_plan(a, nx, ncg, ucap, p, (size_t)c->smem_optin, G);
    a.ftz = std::getenv("LRK_FTZ") ? std::atof(std::getenv("LRK_FTZ")) : 0.0;
    for (int g = 0; g < G; ++g) a.spart[g] = part + (int64_t)g * 3 * ncg * pst;
    for (int g = 1; g < G; ++g) {
      SweepArgs& b = batch.g[g];
      b = a;
      b.shard = g;
      b.V0 = Vg + (int64_t)(2 * g) * nt * ucap;
      b.V1 = Vg + (int64_t)(2 * g + 1) * nt * ucap;
      b.sigma = sg + (int64_t)g * NMAX;
      b.info = ig + 8 * g;
      b.trace = tg + (int64_t)g * (nflush + 1);
      b.scratch = scratch + (int64_t)g * ncg * sst;
      b.dbg = nullptr;
    }
    batch.ngroups = G;
  }
  const int slot = adjoint ? 1 : 0;
  // Large n_x (rows not resident in shared memory): the streaming-flush form
  // (lrk_sflush.cu) — one kernel per row pass instead of the persistent
  // kernel's global-row phases.  LRK_SFLUSH=0 forces the persistent kernel,
  // LRK_SFLUSH=1 forces the streaming form (tests).  n_x shards (one per
  // process after lrk_shard_setup, or emulated on this device) always take
  // the streaming form.
  {
    const char* sfe = std::getenv("LRK_SFLUSH");
    const int force = sfe ? std::atoi(sfe) : -1;
    const bool dist = c->dist.world > 1;
    const int S = dist ? c->dist.world : std::max(1, std::min(c->emu_shards, (int)SF_XMAXR));
    const bool fits = p <= SF_P && ucap <= SF_CAP && rb <= SF_CAP && (nx % 2) == 0 &&
                      !std::getenv("LRK_DUMP_CORES") && !std::getenv("LRK_DEBUG");
    const bool want = dist || force == 1 || (force != 0 && !a.resident);
    if (dist && !fits)
      return fail(c, LRK_ERR_UNSUPPORTED,
                  "sharded sweeps need compress_every <= 4, r_max <= 64 and an even n_x");
    if (dist && !c->dist.connected)
      return fail(c, LRK_ERR_CONFIG, "lrk_shard_setup without lrk_shard_connect");
    if (fits && want) {
      const int nlocal = dist ? 1 : S;
      // contiguous row slabs in multiples of 8 rows
      const int64_t per = ((nx / 8 + S - 1) / S) * 8 + (nx < 8 ? 8 : 0);
      if (S > 1 && per * (int64_t)(S - 1) >= nx)
        return fail(c, LRK_ERR_UNSUPPORTED, "too few rows for this many n_x shards");
      WS(SFState, sfst, tag + "sfst", nlocal);
      WS(unsigned, tick, "sf_tick", 8 * nlocal);
      const int Gs = c->num_sms;
      WS(double, sfpart, "sf_part", (int64_t)nlocal * (8 * Gs) * sf_part_stride());
      WS(double, ybuf3, "sw_ybuf3", ld * (int64_t)p);
      WS(double, Vg, tag + "sfVsh", (int64_t)std::max(nlocal - 1, 1) * nt * ucap);
      WS(double, sg, tag + "sfsigsh", (int64_t)nlocal * NMAX);
      WS(int, ig, tag + "sfinfosh", 8 * nlocal);
      WS(int, tg, tag + "sftracesh", (int64_t)nlocal * (nflush + 1));
      SFXBuf* xb = nullptr;
      if (S > 1 && !dist) {
        WS(SFXBuf, xbe, "sf_xbuf", S);
        xb = xbe;
      }
      CK(cudaMemsetAsync(sfst, 0, sizeof(SFState) * nlocal, s));
      CK(cudaMemsetAsync(yprev, 0, nx * sizeof(double), s));
      if (nlocal > 1) CK(cudaMemsetAsync(ig, 0, 8 * nlocal * sizeof(int), s));
      if (!c->aux.stream) {
        CK(cudaStreamCreateWithFlags(&c->aux.stream, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&c->aux.ready, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->aux.done, cudaEventDisableTiming));
      }
      long long* sfdbg = nullptr;
      if (std::getenv("LRK_SF_TIMING")) {
        WS(long long, d, "sf_dbg", 32);
        CK(cudaMemsetAsync(d, 0, 32 * sizeof(long long), s));
        sfdbg = d;
      }
      std::vector<SFArgs> sh(nlocal);
      int64_t my_x0 = 0, my_rows = nx;
      for (int l = 0; l < nlocal; ++l) {
        const int g = dist ? c->dist.rank : l;
        const int64_t x0 = S > 1 ? std::min(nx, (int64_t)g * per) : 0;
        const int64_t x1 = S > 1 ? std::min(nx, x0 + per) : nx;
        if (l == 0) { my_x0 = x0; my_rows = x1 - x0; }
        SFArgs& sa = sh[l];
        sa = SFArgs{};
        sa.n_x = x1 - x0; sa.n_x_glob = nx; sa.nshard = S; sa.shard = g;
        for (int q = 0; q < S && S > 1; ++q)
          sa.xpeer[q] = dist ? reinterpret_cast<SFXBuf*>(c->dist.peer[q]) : xb + q;
        sa.n_t = nt; sa.p = p; sa.cap = ucap; sa.adjoint = adjoint; sa.r_max = r_max;
        sa.nflush = nflush; sa.eps0 = eps0; sa.ftz = a.ftz;
        sa.U = U0 + x0; sa.ldu = ld;
        sa.V = l == 0 ? V0 : Vg + (int64_t)(l - 1) * nt * ucap; sa.ldv = nt;
        sa.Yg[0] = ybuf + x0; sa.Yg[1] = qbuf + x0; sa.Yg[2] = ybuf3 + x0; sa.ldy = ld;
        sa.yprev = yprev + x0; sa.theta = c->dTheta + x0;
        sa.rowscale = c->dThetaM ? c->dThetaM + x0 : nullptr;
        sa.B = B + x0; sa.ldb = ldb; sa.rb = rb; sa.rb_dev = rb_dev; sa.W2 = W2; sa.ldw2 = ldw2;
        sa.part = sfpart + (int64_t)l * (8 * Gs) * sf_part_stride();
        sa.ticket = tick + 8 * l; sa.st = sfst + l;
        sa.trace = l == 0 ? trace : tg + (int64_t)l * (nflush + 1);
        sa.info = l == 0 ? info : ig + 8 * l;
        sa.sigma = l == 0 ? sig : sg + (int64_t)l * NMAX;
        sa.G = Gs; sa.Ggen = 8 * c->num_sms;
        sa.dbg_print = std::getenv("LRK_SF_DEBUG") ? std::atoi(std::getenv("LRK_SF_DEBUG")) : 0;
        sa.smem_pass = (int)sf_smem_pass();
        sa.dbg = sfdbg;
      }
      if (c->prof) CK(cudaEventRecord(c->ev[2 * slot], s));
      CK(launch_sweep_stream(sh.data(), nlocal, nflush, s, c->aux, &c->xseq, &c->launches));
      if (c->prof) CK(cudaEventRecord(c->ev[2 * slot + 1], s));
      if (dist) {
        // every rank needs the whole pane basis for the replicated stages
        double* panes[SF_XMAXR] = {};
        const size_t off = tag == "f_" ? c->dist.off_f : c->dist.off_b;
        if (reinterpret_cast<char*>(U0) != c->dist.arena + off)
          return fail(c, LRK_ERR_CONFIG, "sharded sweep pane is not in the peer-shared arena");
        for (int q = 0; q < S; ++q) panes[q] = reinterpret_cast<double*>(c->dist.peer[q] + off);
        CK(sf_allgather_pane(sh[0], panes, ld, my_x0, my_rows, ucap, s, &c->xseq, &c->launches));
      }
      o.U = U0; o.V = V0; o.sigma = sig; o.info = info; o.trace = trace;
      o.ucap = ucap; o.nflush = nflush; o.ldu = ld; o.ldv = nt;
      return LRK_OK;
    }
  }
  const char* dump = std::getenv("LRK_DUMP_CORES");  // diagnostics (tools/jacobi_bench)
  const int64_t dsz = (int64_t)nflush * (1 + 32 * 33);
  WS(double, cd, tag + "cdump", dump ? dsz : 1);
  if (dump) {
    CK(cudaMemsetAsync(cd, 0, dsz * sizeof(double), s));
    for (int g = 0; g < batch.ngroups; ++g) batch.g[g].cdump = g == 0 ? cd : nullptr;
  }
  if (c->prof) CK(cudaEventRecord(c->ev[2 * slot], s));
  CK(launch_sweep(batch, s));
  if (c->prof) CK(cudaEventRecord(c->ev[2 * slot + 1], s));
  ++c->launches;
  if (dump) {
    std::vector<double> h(dsz);
    CK(cudaMemcpyAsync(h.data(), cd, dsz * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const std::string path = std::string(dump) + (adjoint ? ".bwd" : ".fwd");
    if (FILE* fp = std::fopen(path.c_str(), "wb")) {
      std::fwrite(h.data(), sizeof(double), h.size(), fp);
      std::fclose(fp);
    }
  }
  o.U = U0; o.V = V0; o.sigma = sig; o.info = info; o.trace = trace;
  o.ucap = ucap; o.nflush = nflush; o.ldu = ld; o.ldv = nt;
  return LRK_OK;
}


// ------------------------------------------------- physical-space sweeps
// Convection-diffusion (and any operator the DST does not diagonalise): the
// sweep runs in physical coordinates.  The dense recurrence
//   y_k = S^{-1}(M y_{k-1}) + B~ w2_k,   B~ = S^{-1} B      (forward.py:175-183)
// is advanced with one preconditioned GMRES solve per step and the
// trajectory is materialised in HBM (chunks of whole flushes); the same
// persistent kernel then flushes it (external-trajectory mode).
bool phys_basis(const lrk_ctx* c) { return c->op.kind != LRK_OP_HEAT; }

// x = P^{-1} b, P = m (I + tau nu L_D): the diffusion part of the step
// matrix, diagonal in the DST-I basis (dThetaM holds its inverse symbol).
// (beta = 1: x += P^{-1} b; the spectral scaling and the accumulation ride in
// the DST GEMM epilogues.)
int precond_apply(lrk_ctx* c, const double* b, double* x, cudaStream_t s, double beta = 0.0) {
  const int64_t nx = c->n_x;
  WS(double, T, "pc_T", nx);
  TRY(dst2(c, b, nx, T, nx, 1, nullptr, 1.0, s, c->dThetaM, 0.0));
  TRY(dst2(c, T, nx, x, nx, 1, nullptr, 1.0, s, nullptr, beta));
  return LRK_OK;
}

int step_apply(lrk_ctx* c, const double* x, double* y, bool adjoint, cudaStream_t s) {
  StencilArgs a = make_stencil(c->op, adjoint);
  a.X = x; a.ldx = c->n_x; a.Y = y; a.ldy = c->n_x; a.ncols = 1;
  launch_stencil(a, s);
  CKL();
  ++c->launches;
  return LRK_OK;
}

int axpby(lrk_ctx* c, const double* x, double a, const double* y, double b, double* out,
          cudaStream_t s) {
  axpby_kernel<<<grid1(c->n_x, 256, 2048), 256, 0, s>>>(x, a, y, b, out, c->n_x);
  CKL();
  ++c->launches;
  return LRK_OK;
}

// GMRES(40) with right preconditioning P^{-1} for S x = b (S^T x = b for the
// adjoint); CGS2 Arnoldi on the device (lrk_cgs2), Givens least squares on
// the host; restarts until the TRUE relative residual is <= rtol.
int gmres_solve(lrk_ctx* c, const double* b, double* x, bool adjoint, double rtol, int* iters,
                cudaStream_t s) {
  const int64_t nx = c->n_x;
  const int n = (int)nx;
  constexpr int M = 40;
  WS(double, Qb, "gm_Q", nx * (M + 1));
  WS(double, z, "gm_z", nx);
  WS(double, w, "gm_w", nx);
  double bnorm = 0.0;
  TRY(lrk_cgs2(c, nullptr, nx, 0, const_cast<double*>(b), n, nullptr, &bnorm, s));
  int total = 0;
  if (bnorm == 0.0) {
    CK(cudaMemsetAsync(x, 0, nx * sizeof(double), s));
    if (iters) *iters = 0;
    return LRK_OK;
  }
  TRY(precond_apply(c, b, x, s));  // x0 = P^{-1} b
  double beta_prev = 0.0;
  for (int restart = 0;; ++restart) {
    TRY(step_apply(c, x, w, adjoint, s));
    TRY(axpby(c, b, 1.0, w, -1.0, Qb, s));  // r = b - S x
    double beta = 0.0;
    TRY(lrk_cgs2(c, nullptr, nx, 0, Qb, n, nullptr, &beta, s));
    if (beta <= rtol * bnorm) break;
    // attainable accuracy: for large tau the step matrix is ill conditioned and the
    // true residual stalls at ~eps cond(S) ||b|| (what a direct solve delivers too);
    // a restart that no longer halves a residual already below 1e-10 ||b|| is accepted
    if (restart >= 2 && beta > 0.5 * beta_prev && beta <= 1e-10 * bnorm) break;
    beta_prev = beta;
    if (restart >= 25)
      return fail(c, LRK_ERR_CONVERGENCE, "GMRES step solve did not reach its tolerance");
    TRY(axpby(c, Qb, 1.0 / beta, nullptr, 0.0, Qb, s));
    double R[M][M] = {};
    double cs[M], sn[M], g[M + 1] = {};
    g[0] = beta;
    int jend = 0;
    for (int j = 0; j < M; ++j) {
      double* qn = Qb + (int64_t)(j + 1) * nx;
      TRY(precond_apply(c, Qb + (int64_t)j * nx, z, s));
      TRY(step_apply(c, z, qn, adjoint, s));
      double h[M + 1], hn = 0.0;
      TRY(lrk_cgs2(c, Qb, nx, j + 1, qn, n, h, &hn, s));
      for (int i = 0; i < j; ++i) {
        const double t = cs[i] * h[i] + sn[i] * h[i + 1];
        h[i + 1] = -sn[i] * h[i] + cs[i] * h[i + 1];
        h[i] = t;
      }
      const double d = std::hypot(h[j], hn);
      cs[j] = d > 0.0 ? h[j] / d : 1.0;
      sn[j] = d > 0.0 ? hn / d : 0.0;
      h[j] = d;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      for (int i = 0; i <= j; ++i) R[i][j] = h[i];
      jend = j + 1;
      ++total;
      if (hn == 0.0 || std::fabs(g[j + 1]) <= 0.5 * rtol * bnorm) break;
      TRY(axpby(c, qn, 1.0 / hn, nullptr, 0.0, qn, s));
    }
    double y[M];
    for (int i = jend - 1; i >= 0; --i) {
      double acc = g[i];
      for (int k = i + 1; k < jend; ++k) acc -= R[i][k] * y[k];
      y[i] = R[i][i] != 0.0 ? acc / R[i][i] : 0.0;
    }
    TRY(lrk_combine(c, Qb, nx, jend, y, n, z, s));
    TRY(precond_apply(c, z, w, s));
    TRY(axpby(c, x, 1.0, w, 1.0, x, s));
  }
  if (iters) *iters = total;
  return LRK_OK;
}

constexpr double STEP_RTOL = 1e-13;

// Sync-free preconditioned Richardson for S x = b:  x <- x + P^{-1}(b - S x),
// a fixed number of sweeps c->rich_it chosen from the contraction factor
// measured once per operator (rich_setup); the true residual is checked on
// the device and any miss raises *flag (the caller redoes the work with GMRES).
int rich_solve(lrk_ctx* c, const double* b, double* x, bool adjoint, int* flag, cudaStream_t s) {
  const int64_t nx = c->n_x;
  WS(double, r, "rs_r", nx);
  WS(double, part, "rs_part", RICH_PART_LEN);
  WS(unsigned, cnt, "rs_cnt", 1);
  StencilArgs a = make_stencil(c->op, adjoint);
  // one persistent kernel per solve where it applies (2-D, even n): every phase of
  // the iteration in one cooperative launch instead of ~70 dependent launches
  if (flag && !std::getenv("LRK_RICH_MULTI")) {
    WS(double, T1, "rs_T1", nx);
    WS(double, T2, "rs_T2", nx);
    WS(unsigned, rbar, "rs_bar", 4);
    const cudaError_t e = launch_rich(a, c->n, c->rich_it, c->dS, c->dThetaM, b, x, r, T1, T2, rbar,
                                      part, flag, STEP_RTOL * STEP_RTOL, c->num_sms, s);
    if (e == cudaSuccess) {
      ++c->launches;
      static const bool dbg = std::getenv("LRK_RICH_DEBUG") != nullptr;
      if (dbg) {   // diagnostics: the relative residual the fixed sweep count reached
        static int shown = 0;
        if (shown < 40 || shown % 200 == 0) {
          double hp[3];
          CK(cudaStreamSynchronize(s));
          CK(cudaMemcpy(hp, part + RICH_PART_DIAG, sizeof(hp), cudaMemcpyDeviceToHost));
          std::fprintf(stderr, "[rich] solve %d: %d of at most %d sweeps, ||r||/||b|| = %.3e\n", shown,
                       (int)hp[0], c->rich_it, hp[2] > 0 ? std::sqrt(hp[1] / hp[2]) : 0.0);
        }
        ++shown;
      }
      return LRK_OK;
    }
    // outside the kernel's scope, or the grid cannot be co-resident here (another context on
    // the device): take the multi-launch path; anything else is an error
    if (e != cudaErrorNotSupported && e != cudaErrorCooperativeLaunchTooLarge &&
        e != cudaErrorLaunchOutOfResources)
      CK(e);
    cudaGetLastError();
  }
  TRY(precond_apply(c, b, x, s));
  a.X = x; a.ldx = nx; a.Y = r; a.ldy = nx; a.ncols = 1; a.Bres = b; a.ldbres = nx;
  for (int it = 0; it < c->rich_it; ++it) {
    launch_stencil(a, s);
    CKL();
    ++c->launches;
    TRY(precond_apply(c, r, x, s, 1.0));
  }
  if (flag) {
    launch_stencil(a, s);
    CKL();
    resid_flag_kernel<<<296, 256, 0, s>>>(r, b, nx, STEP_RTOL * STEP_RTOL, part, cnt, flag);
    CKL();
    c->launches += 2;
  }
  return LRK_OK;
}

// Measure q = ||I - P^{-1} S|| on a fixed pseudo-random vector and choose the
// Richardson sweep count (rich_it = -1: contraction too weak, use GMRES).
int rich_setup(lrk_ctx* c, cudaStream_t s) {
  if (c->rich_it != 0) return LRK_OK;
  const int64_t nx = c->n_x;
  WS(double, b, "rq_b", nx);
  WS(double, x, "rq_x", nx);
  WS(double, r, "rq_r", nx);
  WS(unsigned, cnt, "rs_cnt", 1);
  CK(cudaMemsetAsync(cnt, 0, sizeof(unsigned), s));
  std::vector<double> hb(nx);
  uint64_t st = 0x9e3779b97f4a7c15ull;
  for (int64_t i = 0; i < nx; ++i) {
    st ^= st << 13; st ^= st >> 7; st ^= st << 17;
    hb[i] = (double)(st >> 11) * (1.0 / 9007199254740992.0) - 0.5;
  }
  CK(cudaMemcpyAsync(b, hb.data(), nx * sizeof(double), cudaMemcpyHostToDevice, s));
  TRY(precond_apply(c, b, x, s));
  StencilArgs a = make_stencil(c->op, false);
  a.X = x; a.ldx = nx; a.Y = r; a.ldy = nx; a.ncols = 1; a.Bres = b; a.ldbres = nx;
  std::vector<double> res;
  for (int it = 0; it < 10; ++it) {
    launch_stencil(a, s);
    CKL();
    double nr = 0.0;
    TRY(lrk_cgs2(c, nullptr, nx, 0, r, (int)nx, nullptr, &nr, s));
    res.push_back(nr);
    TRY(precond_apply(c, r, x, s, 1.0));
  }
  double q = 1.0;
  if (res[2] > 0.0 && res[9] > 0.0) q = std::pow(res[9] / res[2], 1.0 / 7.0);
  else if (res[2] == 0.0 || res[9] == 0.0) q = 0.0;
  if (!(q < 0.6)) {
    c->rich_it = -1;
  } else {
    // residual after x0 = P^{-1} b is ~ q ||b||; reach 1e-3 * STEP_RTOL with margin
    const double need = std::log(0.1 * STEP_RTOL) / std::log(std::max(q, 1e-6));
    c->rich_it = std::max(2, std::min(60, (int)std::ceil(need) + 1));
    if (const char* e = std::getenv("LRK_RICH_IT")) c->rich_it = std::max(1, std::atoi(e));  // diagnostics
  }
  c->rich_q = q;
  if (std::getenv("LRK_DEBUG")) {
    std::fprintf(stderr, "[lrk] step-solve contraction q = %.3e -> %s %d; residuals:", q,
                 c->rich_it > 0 ? "Richardson sweeps" : "GMRES", c->rich_it);
    for (double v : res) std::fprintf(stderr, " %.2e", v);
    std::fprintf(stderr, "\n");
  }
  return LRK_OK;
}

int run_sweep_phys(lrk_ctx* c, const std::string& tag, const double* B, int64_t ldb, int rb,
                   const int* rb_dev, const double* W2, int64_t ldw2, int adjoint, int p,
                   double eps0, int r_max, SweepOut& o, cudaStream_t s) {
  if (p < 1 || p > PMAX)
    return fail(c, LRK_ERR_UNSUPPORTED, "compress_every must lie in [1, 16] on the device path");
  const int64_t nx = c->n_x;
  const int nt = c->op.n_t;
  int rbh = rb;
  if (rb_dev) {
    int v = 0;
    CK(cudaMemcpyAsync(&v, rb_dev, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    rbh = std::min(rb, v);
  }
  const int slot = adjoint ? 1 : 0;
  TRY(rich_setup(c, s));
  const bool rich = c->rich_it > 0;
  WS(int, flag, "ph_flag", 1);
  CK(cudaMemsetAsync(flag, 0, sizeof(int), s));
  int it = 0;
  auto solve = [&](const double* b, double* x, bool force_gmres) -> int {
    if (rich && !force_gmres) return rich_solve(c, b, x, adjoint != 0, flag, s);
    return gmres_solve(c, b, x, adjoint != 0, STEP_RTOL, &it, s);
  };
  auto flag_raised = [&](bool& raised) -> int {
    raised = false;
    if (!rich) return LRK_OK;
    int hf = 0;
    CK(cudaMemcpyAsync(&hf, flag, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (hf) CK(cudaMemsetAsync(flag, 0, sizeof(int), s));
    raised = hf != 0;
    return LRK_OK;
  };
  if (c->prof) CK(cudaEventRecord(c->ev[2 * slot], s));
  // B~ = S^{-1} B (S^{-T} B for the adjoint), one solve per column
  WS(double, Bs, tag + "Bs", nx * (int64_t)std::max(rbh, 1));
  for (int pass = 0; pass < 2; ++pass) {
    for (int j = 0; j < rbh; ++j)
      TRY(solve(B + (int64_t)j * ldb, Bs + (int64_t)j * nx, pass == 1));
    bool raised = false;
    TRY(flag_raised(raised));
    if (!raised) break;
  }
  const int ucap = (r_max >= 0 && r_max < NMAX) ? std::max(r_max, 1) : NMAX;
  const int ncta = pick_ncta(c, nx);
  const int nflush = (nt + p - 1) / p;
  // trajectory chunk: whole flushes, at most 2^31 doubles (16 GiB)
  const int64_t budget = (int64_t)1 << 31;
  int Tc = nt;
  if (nx * (int64_t)nt > budget) Tc = std::max<int>(p, (int)(budget / nx) / p * p);
  WS(double, Yx, "ph_Y", nx * (int64_t)Tc);
  WS(double, U0, tag + "U0", nx * (int64_t)ucap);
  WS(double, U1, tag + "U1", nx * (int64_t)ucap);
  WS(double, V0, tag + "V0", (int64_t)nt * ucap);
  WS(double, V1, tag + "V1", (int64_t)nt * ucap);
  WS(double, sig, tag + "sig", NMAX);
  WS(int, info, tag + "info", 8);
  WS(int, trace, tag + "trace", nflush + 1);
  WS(double, ybuf, "sw_ybuf", nx * (int64_t)p);
  WS(double, qbuf, "sw_qbuf", nx * (int64_t)p);
  WS(double, yprev, "sw_yprev", nx);
  WS(double, tmp, "ph_tmp", nx);
  const int64_t pst = sweep_part_stride();
  WS(double, part, "sw_part", 3 * (int64_t)ncta * pst);
  const int64_t sst = sweep_scratch_stride(ncta);
  WS(double, scratch, "sw_scratch", (int64_t)ncta * sst);
  WS(unsigned, bar, "sw_bar", 4);
  SweepBatch batch{};
  batch.ngroups = 1;
  SweepArgs& a = batch.g[0];
  a.n_x = nx; a.n_t = nt; a.adjoint = adjoint; a.p = p; a.r_max = r_max; a.eps0 = eps0;
  a.theta = nullptr; a.rowscale = nullptr;
  a.B = nullptr; a.ldb = nx; a.rb = 0; a.rb_dev = nullptr;
  a.W2 = W2; a.ldw2 = ldw2;
  a.U0 = U0; a.U1 = U1; a.ldu = nx; a.V0 = V0; a.V1 = V1; a.ldv = nt; a.ucap = ucap;
  a.sigma = sig; a.info = info; a.trace = trace;
  a.ybuf = ybuf; a.ldy = nx; a.qbuf = qbuf; a.ldq = nx; a.yprev = yprev;
  a.part = part; a.pstride = pst; a.scratch = scratch; a.scratch_stride = sst;
  a.bar = bar; a.ncta = ncta;
  a.yext = Yx; a.ldyext = nx;
  a.nshard = 1; a.shard = 0; a.sys_fence = 0;
  a.spart[0] = part; a.gbar = bar;
  sweep_plan(a, nx, ncta, ucap, p, (size_t)c->smem_optin);
  a.ftz = 0.0;
  WS(long long, dbg, tag + "dbg", 20);
  a.dbg = std::getenv("LRK_DEBUG") ? dbg : nullptr;
  a.nopipe = std::getenv("LRK_NOPIPE") ? 1 : 0;
  o.dbg = dbg;
  CK(cudaMemsetAsync(info, 0, 8 * sizeof(int), s));
  const double m = c->op.m_scale;
  const double* yp = nullptr;
  // LRK_DEBUG: device time of the step solves vs the flush launches
  const bool tdbg = std::getenv("LRK_DEBUG") != nullptr;
  cudaEvent_t te[3];
  float t_steps = 0.f, t_flush = 0.f;
  if (tdbg)
    for (auto& e : te) CK(cudaEventCreate(&e));
  for (int cs0 = 0; cs0 < nt; cs0 += Tc) {
    const int ce = std::min(nt, cs0 + Tc);
    if (tdbg) CK(cudaEventRecord(te[0], s));
    const double* yp0 = yp;  // y before this chunk (yprev or null), for a GMRES redo
    for (int pass = 0; pass < 2; ++pass) {
      yp = yp0;
      for (int j = cs0; j < ce; ++j) {
        const int k = adjoint ? nt - 1 - j : j;  // time step advanced by processing index j
        double* yk = Yx + (int64_t)(j - cs0) * nx;
        if (yp) {
          TRY(axpby(c, yp, m, nullptr, 0.0, tmp, s));
          TRY(solve(tmp, yk, pass == 1));
        } else {
          CK(cudaMemsetAsync(yk, 0, nx * sizeof(double), s));
        }
        if (rbh > 0) {
          rank_axpy_kernel<<<grid1(nx, 256, 2048), 256, 0, s>>>(Bs, nx, rbh, W2 + k, ldw2, yk, nx);
          CKL();
          ++c->launches;
        }
        yp = yk;
      }
      bool raised = false;
      TRY(flag_raised(raised));
      if (!raised) break;
    }
    // the chunk buffer is rewritten next: carry y_{last} in yprev
    CK(cudaMemcpyAsync(yprev, yp, nx * sizeof(double), cudaMemcpyDeviceToDevice, s));
    yp = yprev;
    a.flush0 = cs0 / p;
    a.flush1 = std::min(nflush, (ce + p - 1) / p);
    a.r_init = cs0 == 0 ? 0 : -1;
    if (tdbg) CK(cudaEventRecord(te[1], s));
    CK(launch_sweep(batch, s));
    ++c->launches;
    if (tdbg) {
      CK(cudaEventRecord(te[2], s));
      CK(cudaEventSynchronize(te[2]));
      float a01 = 0.f, a12 = 0.f;
      CK(cudaEventElapsedTime(&a01, te[0], te[1]));
      CK(cudaEventElapsedTime(&a12, te[1], te[2]));
      t_steps += a01;
      t_flush += a12;
    }
  }
  if (tdbg) {
    std::fprintf(stderr, "[lrk] physical sweep (%s): step solves %.1f ms, flush kernels %.1f ms\n",
                 adjoint ? "adjoint" : "forward", t_steps, t_flush);
    for (auto& e : te) cudaEventDestroy(e);
  }
  if (c->prof) CK(cudaEventRecord(c->ev[2 * slot + 1], s));
  o.U = U0; o.V = V0; o.sigma = sig; o.info = info; o.trace = trace;
  o.ucap = ucap; o.nflush = nflush; o.ldu = nx; o.ldv = nt;
  return LRK_OK;
}

// Change of basis between physical coordinates and the sweep basis (DST-I,
// an involution, for DST-diagonal operators; identity otherwise), scaled.
int basis_xform(lrk_ctx* c, const double* X, int64_t ldx, double* Y, int64_t ldy, int ncols,
                const int* ncols_dev, double alpha, cudaStream_t s) {
  if (ncols <= 0) return LRK_OK;
  if (!phys_basis(c)) return dst2(c, X, ldx, Y, ldy, ncols, ncols_dev, alpha, s);
  scale_cols_kernel<<<dim3(grid1(c->n_x, 256, 1024), ncols), 256, 0, s>>>(
      X, ldx, c->n_x, nullptr, ncols_dev, ncols, alpha, Y, ldy);
  CKL();
  ++c->launches;
  return LRK_OK;
}

// -------------------------------------------------------------- truncate
struct TruncOut {
  int* info = nullptr;
};

int run_truncate(lrk_ctx* c, const std::string& tag, int64_t n_x, int n_t, const double* W1,
                 int64_t ld1, const double* W2, int64_t ld2, int R, const int* R_dev, int flags,
                 double eps0, int r_max, double* out1, int64_t ldo1, double* out2, int64_t ldo2,
                 int cap, double* sigma, double* sv_all, int no_flip, TruncOut& o, cudaStream_t s) {
  if (R > NMAX)
    return fail(c, LRK_ERR_UNSUPPORTED,
                "lr_truncate on the device supports at most 160 concatenated columns");
  // small factors (e.g. the sensor rows of the obs truncation): more CTAs than
  // the 384-rows rule (1024 rows: 2 -> 16 CTAs, 556 -> 470 us measured)
  const int64_t rows = std::max<int64_t>(n_x, n_t);
  const int ncta = std::max(pick_ncta(c, rows), (int)std::min<int64_t>(16, std::max<int64_t>(1, rows / 64)));
  const int Rw = std::max(R, 1);
  WS(double, Q1, "tr_Q1", n_x * (int64_t)Rw);
  WS(double, Q2, "tr_Q2", (int64_t)n_t * Rw);
  const int64_t ldt = std::max<int64_t>(n_x, n_t);
  WS(double, tmpw, "tr_tmp", ldt * PMAX);
  const int64_t pst = trunc_part_stride();
  WS(double, part, "tr_part", 3 * (int64_t)ncta * pst);
  const int64_t sst = trunc_scratch_stride(ncta);
  WS(double, scratch, "tr_scratch", (int64_t)ncta * sst);
  WS(unsigned, bar, "tr_bar", 4);
  WS(int, info, tag + "info", 8);
  TruncArgs a{};
  a.n_x = n_x; a.n_t = n_t; a.R = R; a.R_dev = R_dev; a.flags = flags; a.r_max = r_max; a.eps0 = eps0;
  a.W1 = W1; a.ld1 = ld1; a.W2 = W2; a.ld2 = ld2;
  a.Q1 = Q1; a.ldq1 = n_x; a.Q2 = Q2; a.ldq2 = n_t;
  a.tmpw = tmpw; a.ldtmp = ldt;
  a.out1 = out1; a.ldo1 = ldo1; a.out2 = out2; a.ldo2 = ldo2; a.cap = cap;
  a.sigma = sigma; a.sv_all = sv_all; a.info = info;
  a.part = part; a.pstride = pst; a.scratch = scratch; a.scratch_stride = sst;
  a.bar = bar; a.ncta = ncta; a.no_flip = no_flip;
  CK(cudaMemsetAsync(info, 0, 8 * sizeof(int), s));
  CK(launch_truncate(a, s));
  ++c->launches;
  o.info = info;
  return LRK_OK;
}

// _svd_flip on device factors (rank on device)
int flip(lrk_ctx* c, double* U, int64_t ldu, int64_t n_x, double* V, int64_t ldv, int n_t,
         const int* r_dev, int rcap, cudaStream_t s) {
  if (rcap <= 0) return LRK_OK;
  const int nparts = grid1(n_x, 4096, 64);
  WS(double, part, "flip_part", (int64_t)rcap * nparts * 3);
  flip_partial_kernel<<<dim3(nparts, rcap), 256, 0, s>>>(U, ldu, n_x, r_dev, rcap, part);
  CKL();
  flip_apply_kernel<<<dim3(grid1(std::max<int64_t>(n_x, n_t), 256, 256), rcap), 256, 0, s>>>(
      U, ldu, n_x, V, ldv, n_t, r_dev, rcap, part, nparts);
  CKL();
  return LRK_OK;
}

int check_op(lrk_ctx* c) {
  if (!c->has_op) return fail(c, LRK_ERR_CONFIG, "no operator installed (lrk_set_operator)");
  return LRK_OK;
}

// Observation + weight + truncation of the forward pane (apply_obs_weight,
// hessian.py:138-156).  Output: spectral Zhat (n_x x cap), Z2 (n_t x cap), zinfo.
int obs_weight(lrk_ctx* c, const SweepOut& y, double w, int every, double eps0, int r_max,
               double** Zhat, int64_t* ldz_out, double** Z2, int** zinfo, int* zcap, cudaStream_t s) {
  const int64_t nx = c->n_x;
  const int nt = c->op.n_t;
  const int cap = y.ucap;
  WS(double, W2s, "ob_W2s", (int64_t)nt * cap);
  // W2s = V diag(w * sigma)
  scale_cols_kernel<<<dim3(grid1(nt, 256, 64), cap), 256, 0, s>>>(y.V, y.ldv, nt, y.sigma,
                                                                   y.info, cap, w, W2s, nt);
  CKL();
  if (every > 1) {  // time-subsampled sensors
    mask_time_rows_kernel<<<dim3(grid1(nt, 256, 64), cap), 256, 0, s>>>(W2s, nt, nt, cap, every);
    CKL();
  }
  // a time mask breaks the orthonormality of the time factor
  const int w2flag = every > 1 ? 0 : LRK_TRUNC_W2_ORTHOSCALED;
  const int64_t ldz = padld(nx);
  WS(double, Zh, "ob_Zhat", ldz * (int64_t)cap);
  WS(double, Zt, "ob_Z2", (int64_t)nt * cap);
  TruncOut to;
  if (c->obs_kind == LRK_OBS_FULL) {
    TRY(run_truncate(c, "ob_", nx, nt, y.U, y.ldu, W2s, nt, cap, y.info,
                     LRK_TRUNC_W1_ORTHO | w2flag, eps0, r_max, Zh, ldz, Zt, nt,
                     cap, nullptr, nullptr, 1, to, s));
  } else {
    const int no = c->n_obs;
    WS(double, Uo, "ob_Uobs", (int64_t)no * cap);
    WS(double, Zo, "ob_Zobs", (int64_t)no * cap);
    if (phys_basis(c)) {
      gather_rows_kernel<<<dim3(grid1(no, 256, 256), cap), 256, 0, s>>>(y.U, y.ldu, c->dList, no,
                                                                         y.info, cap, Uo, no);
      CKL();
    } else if (c->obs_kind == LRK_OBS_SUBGRID) {
      TRY(subgrid_gather(c, y.U, y.ldu, Uo, no, cap, y.info, s));
    } else {
      WS(double, Up, "ob_Uphys", nx * (int64_t)cap);
      TRY(dst2(c, y.U, y.ldu, Up, nx, cap, y.info, 1.0, s));
      gather_rows_kernel<<<dim3(grid1(no, 256, 256), cap), 256, 0, s>>>(Up, nx, c->dList, no,
                                                                         y.info, cap, Uo, no);
      CKL();
    }
    TRY(run_truncate(c, "ob_", no, nt, Uo, no, W2s, nt, cap, y.info, w2flag,
                     eps0, r_max, Zo, no, Zt, nt, cap, nullptr, nullptr, 1, to, s));
    if (phys_basis(c)) {
      fill_kernel<<<dim3(grid1(nx, 256, 1024), cap), 256, 0, s>>>(Zh, ldz, nx, cap, 0.0);
      CKL();
      scatter_rows_kernel<<<dim3(grid1(no, 256, 256), cap), 256, 0, s>>>(Zo, no, c->dList, no,
                                                                          to.info, cap, Zh, ldz);
      CKL();
    } else if (c->obs_kind == LRK_OBS_SUBGRID) {
      TRY(subgrid_scatter(c, Zo, no, Zh, ldz, cap, to.info, s));
    } else {
      WS(double, Zp, "ob_Zphys", nx * (int64_t)cap);
      fill_kernel<<<dim3(grid1(nx, 256, 1024), cap), 256, 0, s>>>(Zp, nx, nx, cap, 0.0);
      CKL();
      scatter_rows_kernel<<<dim3(grid1(no, 256, 256), cap), 256, 0, s>>>(Zo, no, c->dList, no,
                                                                          to.info, cap, Zp, nx);
      CKL();
      TRY(dst2(c, Zp, nx, Zh, ldz, cap, to.info, 1.0, s));
    }
  }
  *Zhat = Zh;
  *ldz_out = ldz;
  *Z2 = Zt;
  *zinfo = to.info;
  *zcap = cap;
  return LRK_OK;
}

int hd_check(lrk_ctx* c, const lrk_hessian_desc* hd) {
  if (!hd) return fail(c, LRK_ERR_CONFIG, "null Hessian descriptor");
  if (!(hd->eps0 > 0.0 && hd->eps0 < 1.0))
    return fail(c, LRK_ERR_SHAPE, "eps0 must lie in (0, 1)");
  if (!c->has_obs) return fail(c, LRK_ERR_CONFIG, "no observation layout installed");
  if (!(hd->gamma_prior > 0.0)) return fail(c, LRK_ERR_CONFIG, "gamma_prior must be positive");
  if (hd->prior_gamma < 0.0 || (hd->prior_gamma > 0.0 && !(hd->prior_delta > 0.0)))
    return fail(c, LRK_ERR_CONFIG, "operator prior needs prior_delta > 0 and prior_gamma >= 0");
  if (hd->obs_every < 0) return fail(c, LRK_ERR_CONFIG, "obs_every must be >= 0");
  if (hd->compress_every < 1 || hd->compress_every > PMAX)
    return fail(c, LRK_ERR_UNSUPPORTED, "compress_every must lie in [1, 16] on the device path");
  if (hd->r_max > NMAX - hd->compress_every)
    return fail(c, LRK_ERR_UNSUPPORTED,
                "r_max must be <= 160 - compress_every (the sweep core is r + compress_every wide)");
  return LRK_OK;
}

// In-place spectral prior factor (prior_delta + prior_gamma lambda)^{-1} on the
// rows of X (no-op for the reference's scalar prior).
int apply_prior(lrk_ctx* c, const lrk_hessian_desc* hd, double* X, int64_t ldx, int ncols,
                const int* ncols_dev, cudaStream_t s) {
  if (!(hd->prior_gamma > 0.0) || ncols <= 0) return LRK_OK;
  if (phys_basis(c)) {  // physical rows: through the DST and back
    WS(double, T, "pr_T", c->n_x * (int64_t)ncols);
    TRY(dst2(c, X, ldx, T, c->n_x, ncols, ncols_dev, 1.0, s));
    prior_scale_kernel<<<dim3(grid1(c->n_x, 256, 1024), ncols), 256, 0, s>>>(
        T, c->n_x, c->dLam, c->n_x, ncols, ncols_dev, 1.0, hd->prior_delta, hd->prior_gamma, T,
        c->n_x);
    CKL();
    return dst2(c, T, c->n_x, X, ldx, ncols, ncols_dev, 1.0, s);
  }
  prior_scale_kernel<<<dim3(grid1(c->n_x, 256, 1024), ncols), 256, 0, s>>>(
      X, ldx, c->dLam, c->n_x, ncols, ncols_dev, 1.0, hd->prior_delta, hd->prior_gamma, X, ldx);
  CKL();
  return LRK_OK;
}

// Algorithmic (compulsory) bytes of one sweep, from its rank trace (DESIGN.md
// §Roofline): per step 16 n_x for the recurrence + 16 n_x for
// one ideal pass of the spatial solve + 8 n_x r_B where the rhs time factor
// is nonzero; per flush 8 n_x R (Gram) + 8 n_x R + 8 n_x r' (basis update),
// R = r_prev + pc.
double sweep_alg_bytes(int64_t n_x, int n_t, int p, const std::vector<int>& tr, int rb,
                       int nnz_steps) {
  double b = 32.0 * n_x * n_t + 8.0 * n_x * rb * nnz_steps;
  const int nflush = (n_t + p - 1) / p;
  for (int f = 0; f < nflush && f < (int)tr.size(); ++f) {
    const int rprev = f ? tr[f - 1] : 0;
    const int pc = std::min(p, n_t - f * p);
    const int R = rprev + pc;
    b += 8.0 * n_x * (2.0 * R + tr[f]);
  }
  return b;
}

// Reads back the ranks of one apply (the only sync of an apply), derives
// max_rank (hessian.py:225) and, when profiling, the sweep timings/bytes.
int host_max_rank(lrk_ctx* c, const SweepOut& f, const int* zinfo, const SweepOut& g,
                  const int* extra_info, int* out, int p, int rb_f, int nnz_f, cudaStream_t s) {
  std::vector<int> t1(f.nflush + 1), t2(g.nflush + 1);
  int zr[8] = {0}, er[8] = {0}, fi[8] = {0}, gi[8] = {0};
  CK(cudaMemcpyAsync(t1.data(), f.trace, t1.size() * sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(t2.data(), g.trace, t2.size() * sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(zr, zinfo, 8 * sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(fi, f.info, 8 * sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(gi, g.info, 8 * sizeof(int), cudaMemcpyDeviceToHost, s));
  if (extra_info) CK(cudaMemcpyAsync(er, extra_info, 8 * sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  // a sweep whose core outgrew the device limit stops early with info[2] set:
  // never return its (incomplete) pane as a result
  if (fi[2] != 0 || gi[2] != 0)
    return fail(c, LRK_ERR_UNSUPPORTED,
                "sweep core exceeded the 160-column device limit (set r_max <= 160 - compress_every)");
  if (fi[5] != 0 || gi[5] != 0)
    return fail(c, LRK_ERR_CUDA, "n_x-sharded sweep: a peer never reached an exchange (timed out)");
  if (zr[2] != 0) return fail(c, LRK_ERR_SHAPE, "observation truncation exceeded its capacity");
  int m = zr[0];
  for (int v : t1) m = std::max(m, v);
  for (int v : t2) m = std::max(m, v);
  if (extra_info) m = std::max(m, er[0]);
  *out = m;
  c->last_fwd = t1;
  c->last_bwd = t2;
  c->last_obs = zr[0];
  if (std::getenv("LRK_DEBUG")) {
    int fi[8], gi[8];
    CK(cudaMemcpy(fi, f.info, sizeof(fi), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(gi, g.info, sizeof(gi), cudaMemcpyDeviceToHost));
    std::fprintf(stderr, "[lrk] apply: ranks fwd %d obs %d bwd %d; jacobi sweeps fwd %d bwd %d over %d+%d flushes\n",
                 fi[0], zr[0], gi[0], fi[3], gi[3], f.nflush, g.nflush);
    long long fd[20], gd[20];
    CK(cudaMemcpy(fd, f.dbg, sizeof(fd), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(gd, g.dbg, sizeof(gd), cudaMemcpyDeviceToHost));
    const char* names[20] = {"gen+proj1", "barrier1", "reduce2+sub2", "hh_local", "barrier3",
                             "stack_tail", "apply_q", "core+jacobi", "update", "reduce1",
                             "sub1+tn2", "barrier2", "rankcut", "stack_copy", "stack_qr",
                             "stack_q", "upd_U", "upd_V", "x18", "x19"};
    std::fprintf(stderr, "[lrk] cycles/flush (fwd | bwd):");
    for (int k = 0; k < 20; ++k)
      std::fprintf(stderr, " %s %lld|%lld", names[k], fd[k] / std::max(1, f.nflush),
                   gd[k] / std::max(1, g.nflush));
    std::fprintf(stderr, "\n");
  }
  if (c->prof) {
    float ms0 = 0.f, ms1 = 0.f;
    CK(cudaEventElapsedTime(&ms0, c->ev[0], c->ev[1]));
    CK(cudaEventElapsedTime(&ms1, c->ev[2], c->ev[3]));
    c->prof_ms += (double)ms0 + (double)ms1;
    c->prof_n += 2;
    const int nt = c->op.n_t;
    c->prof_bytes += sweep_alg_bytes(c->n_x, nt, p, t1, rb_f, nnz_f) +
                     sweep_alg_bytes(c->n_x, nt, p, t2, zr[0], nt);
  }
  return LRK_OK;
}

}  // namespace

// ======================================================================== ABI
extern "C" {

const char* lrk_version(void) { return "lrk-b200 0.1.0 (sm_100a, fp64)"; }

int lrk_ctx_create(int device, lrk_ctx** out) {
  if (!out) return LRK_ERR_CONFIG;
  *out = nullptr;
  if (cudaSetDevice(device) != cudaSuccess) { cudaGetLastError(); return LRK_ERR_CUDA; }
  lrk_ctx* c = new lrk_ctx();
  c->device = device;
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  cudaDeviceGetAttribute(&c->smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  *out = c;
  return LRK_OK;
}

void lrk_ctx_destroy(lrk_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  delete c;
}

const char* lrk_last_error(const lrk_ctx* c) { return c ? c->err.c_str() : "null context"; }

int64_t lrk_launch_count(const lrk_ctx* c) { return c ? c->launches : 0; }

// Config prior: Y = (delta I + gamma L)^{-power} X
// through the DST-I (physical rows in and out).
int lrk_prior_apply(lrk_ctx* c, double delta, double gamma, int power, const double* X,
                    int64_t ldx, int ncols, double* Y, int64_t ldy, void* stream) {
  if (!c) return LRK_ERR_CONFIG;
  CK(cudaSetDevice(c->device));
  if (!c->has_op) return fail(c, LRK_ERR_CONFIG, "no operator installed");
  if (!(delta > 0.0) || gamma < 0.0 || power < 1 || power > 2)
    return fail(c, LRK_ERR_CONFIG, "prior needs delta > 0, gamma >= 0, power 1 or 2");
  cudaStream_t s = (cudaStream_t)stream;
  if (ncols <= 0) return LRK_OK;
  const int64_t nx = c->n_x;
  WS(double, T, "pa_T", nx * (int64_t)ncols);
  TRY(dst2(c, X, ldx, T, nx, ncols, nullptr, 1.0, s));
  for (int k = 0; k < power; ++k) {
    prior_scale_kernel<<<dim3(grid1(nx, 256, 1024), ncols), 256, 0, s>>>(
        T, nx, c->dLam, nx, ncols, nullptr, 1.0, delta, gamma, T, nx);
    CKL();
  }
  TRY(dst2(c, T, nx, Y, ldy, ncols, nullptr, 1.0, s));
  return LRK_OK;
}

// diag((delta I + gamma L)^{-power}) = (Phi∘Phi) d, d_k = (delta + gamma lambda_k)^{-power}:
// the DST passes with S∘S in place of S (separable, one GEMM per axis).
int lrk_prior_diag(lrk_ctx* c, double delta, double gamma, int power, double* out, void* stream) {
  if (!c) return LRK_ERR_CONFIG;
  CK(cudaSetDevice(c->device));
  if (!c->has_op) return fail(c, LRK_ERR_CONFIG, "no operator installed");
  if (!(delta > 0.0) || gamma < 0.0 || power < 1 || power > 2)
    return fail(c, LRK_ERR_CONFIG, "prior needs delta > 0, gamma >= 0, power 1 or 2");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t nx = c->n_x;
  WS(double, d, "pd_d", nx);
  fill_kernel<<<dim3(grid1(nx, 256, 1024), 1), 256, 0, s>>>(d, nx, nx, 1, 1.0);
  CKL();
  for (int k = 0; k < power; ++k) {
    prior_scale_kernel<<<dim3(grid1(nx, 256, 1024), 1), 256, 0, s>>>(
        d, nx, c->dLam, nx, 1, nullptr, 1.0, delta, gamma, d, nx);
    CKL();
  }
  TRY(dst2(c, d, nx, out, nx, 1, nullptr, 1.0, s, nullptr, 0.0, c->dSsq));
  return LRK_OK;
}

int lrk_set_emulated_shards(lrk_ctx* c, int nshard) {
  if (!c) return LRK_ERR_CONFIG;
  if (nshard < 1 || nshard > SHARD_MAX) return fail(c, LRK_ERR_CONFIG, "nshard must lie in [1, 8]");
  c->emu_shards = nshard;
  return LRK_OK;
}

// n_x sharding across processes: one process per GPU, each with
// its own context holding the whole operator; the sweeps run on this rank's
// row slab and exchange their small rank totals through peer memory.
int lrk_shard_setup(lrk_ctx* c, int rank, int world, void* handle_out) {
  if (!c || !handle_out) return LRK_ERR_CONFIG;
  CK(cudaSetDevice(c->device));
  TRY(check_op(c));
  if (world < 1 || world > SF_XMAXR || rank < 0 || rank >= world)
    return fail(c, LRK_ERR_CONFIG, "shard rank/world out of range (world <= 8)");
  if (c->dist.arena) return fail(c, LRK_ERR_CONFIG, "context is already sharded");
  const int64_t ld = padld(c->n_x);
  const size_t xb = (sizeof(SFXBuf) + 4095) / 4096 * 4096;
  const size_t pane = ((size_t)ld * SF_CAP * sizeof(double) + 256 + 4095) / 4096 * 4096;
  c->dist.bytes = xb + 2 * pane;
  c->dist.off_f = xb;
  c->dist.off_b = xb + pane;
  void* p = nullptr;
  if (cudaMalloc(&p, c->dist.bytes) != cudaSuccess) {
    cudaGetLastError();
    return fail(c, LRK_ERR_CUDA, "cudaMalloc failed for the peer-shared arena");
  }
  CK(cudaMemset(p, 0, xb));
  c->dist.arena = static_cast<char*>(p);
  c->dist.rank = rank;
  c->dist.world = world;
  c->dist.peer[rank] = c->dist.arena;
  for (const char* tag : {"f_U0", "b_U0"}) {
    Buf& b = c->ws[tag];
    if (b.p && !b.ext) cudaFree(b.p);
    b.p = c->dist.arena + (std::string(tag) == "f_U0" ? c->dist.off_f : c->dist.off_b);
    b.bytes = pane;
    b.ext = true;
  }
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, p));
  static_assert(sizeof(h) == 64, "IPC handle size");
  std::memcpy(handle_out, &h, sizeof(h));
  c->dist.connected = world == 1;
  return LRK_OK;
}

// handles: world x 64 bytes, the lrk_shard_setup outputs of all ranks in rank order.
int lrk_shard_connect(lrk_ctx* c, const void* handles) {
  if (!c || !handles) return LRK_ERR_CONFIG;
  CK(cudaSetDevice(c->device));
  if (!c->dist.arena) return fail(c, LRK_ERR_CONFIG, "lrk_shard_connect before lrk_shard_setup");
  for (int q = 0; q < c->dist.world; ++q) {
    if (q == c->dist.rank || c->dist.peer[q]) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, static_cast<const char*>(handles) + (size_t)q * sizeof(h), sizeof(h));
    void* p = nullptr;
    const cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(c, LRK_ERR_CUDA, std::string("cudaIpcOpenMemHandle failed for a peer arena: ") +
                                       cudaGetErrorString(e));
    }
    c->dist.peer[q] = static_cast<char*>(p);
  }
  c->dist.connected = true;
  return LRK_OK;
}

int lrk_profile_enable(lrk_ctx* c, int enable) {
  if (!c) return LRK_ERR_CONFIG;
  CK(cudaSetDevice(c->device));
  if (enable && !c->ev[0])
    for (auto& e : c->ev) CK(cudaEventCreate(&e));
  c->prof = enable != 0;
  return LRK_OK;
}

int lrk_profile_read(lrk_ctx* c, double* sweep_ms, int64_t* sweep_launches,
                     double* sweep_alg_bytes_out, int reset) {
  if (!c) return LRK_ERR_CONFIG;
  if (sweep_ms) *sweep_ms = c->prof_ms;
  if (sweep_launches) *sweep_launches = c->prof_n;
  if (sweep_alg_bytes_out) *sweep_alg_bytes_out = c->prof_bytes;
  if (reset) { c->prof_ms = 0.0; c->prof_n = 0; c->prof_bytes = 0.0; }
  return LRK_OK;
}

int lrk_last_traces(lrk_ctx* c, int* fwd, int* bwd, int cap, int* n_fwd, int* n_bwd,
                    int* obs_rank) {
  if (!c) return LRK_ERR_CONFIG;
  const int nf = std::min<int>(cap, (int)c->last_fwd.size());
  const int nb = std::min<int>(cap, (int)c->last_bwd.size());
  for (int i = 0; i < nf; ++i) fwd[i] = c->last_fwd[i];
  for (int i = 0; i < nb; ++i) bwd[i] = c->last_bwd[i];
  if (n_fwd) *n_fwd = nf;
  if (n_bwd) *n_bwd = nb;
  if (obs_rank) *obs_rank = c->last_obs;
  return LRK_OK;
}

int lrk_set_operator(lrk_ctx* c, const lrk_operator_desc* op) {
  if (!c || !op) return LRK_ERR_CONFIG;
  CK(cudaSetDevice(c->device));
  if (op->dim != 2 && op->dim != 3)
    return fail(c, LRK_ERR_UNSUPPORTED, "dim must be 2 or 3");
  if (op->stencil != LRK_STENCIL_FD && op->stencil != LRK_STENCIL_Q1)
    return fail(c, LRK_ERR_CONFIG, "unknown stencil");
  if (op->wind_field != LRK_WIND_CONST && op->wind_field != LRK_WIND_ROTATING)
    return fail(c, LRK_ERR_CONFIG, "unknown wind field");
  if (op->stencil == LRK_STENCIL_Q1 && op->dim != 2)
    return fail(c, LRK_ERR_UNSUPPORTED, "the Q1 stencils are implemented in 2-D");
  if (op->n_side < 2 || op->n_t < 1 || !(op->tau > 0) || !(op->h > 0) || !(op->m_scale > 0))
    return fail(c, LRK_ERR_CONFIG, "invalid operator descriptor");
  const int n = op->n_side;
  const int64_t nx = op->dim == 3 ? (int64_t)n * n * n : (int64_t)n * n;
  std::vector<double> S((size_t)n * n), th(nx), thm(nx), il(nx), lm(nx), l1(n), m1(n),
      e0(op->n_t, 0.0);
  const double f = std::sqrt(2.0 / (n + 1));
  for (int j = 0; j < n; ++j)
    for (int k = 0; k < n; ++k)
      S[(size_t)j * n + k] = f * std::sin(M_PI * (double)(j + 1) * (double)(k + 1) / (n + 1));
  const double h = op->h;
  // per-axis symbols of the DST-I eigenvectors
  for (int m = 0; m < n; ++m) {
    const double sv = std::sin((m + 1) * M_PI * h / 2.0);
    if (op->stencil == LRK_STENCIL_FD) {
      l1[m] = (4.0 / (h * h)) * sv * sv;  // discretize.py:137-144 (per axis)
    } else {
      // Q1: K1 = (1/h)[-1 2 -1] -> (2/h)(1 - cos), M1 = (h/6)[1 4 1] -> (h/3)(2 + cos);
      // L = (K1 (x) M1 + M1 (x) K1) / h^2
      const double cs = std::cos((m + 1) * M_PI * h);
      l1[m] = (2.0 / h) * (1.0 - cs);
      m1[m] = (h / 3.0) * (2.0 + cs);
    }
  }
  for (int64_t i = 0; i < nx; ++i) {
    const int i1 = (int)(i % n), i2 = (int)((i / n) % n), i3 = (int)(i / ((int64_t)n * n));
    double lam;
    if (op->stencil == LRK_STENCIL_Q1) lam = (l1[i1] * m1[i2] + m1[i1] * l1[i2]) / (h * h);
    else lam = l1[i1] + l1[i2] + (op->dim == 3 ? l1[i3] : 0.0);
    // convdiff: the DST-diagonal part m (I + tau nu L_D) is the GMRES preconditioner
    const double lsym = op->kind == LRK_OP_HEAT ? lam : op->nu * lam;
    const double t = 1.0 / (1.0 + op->tau * lsym);
    th[i] = t;
    thm[i] = t / op->m_scale;
    il[i] = 1.0 / lam;
    lm[i] = lam;
  }
  e0[0] = 1.0;
  cudaFree(c->dS); cudaFree(c->dTheta); cudaFree(c->dThetaM); cudaFree(c->dE0);
  cudaFree(c->dInvLam); cudaFree(c->dLam);
  c->dS = c->dTheta = c->dThetaM = c->dE0 = c->dInvLam = c->dLam = nullptr;
  CK(cudaMalloc(&c->dInvLam, nx * sizeof(double)));
  CK(cudaMemcpy(c->dInvLam, il.data(), nx * sizeof(double), cudaMemcpyHostToDevice));
  CK(cudaMalloc(&c->dLam, nx * sizeof(double)));
  CK(cudaMemcpy(c->dLam, lm.data(), nx * sizeof(double), cudaMemcpyHostToDevice));
  CK(cudaMalloc(&c->dS, S.size() * sizeof(double)));
  {
    std::vector<double> S2(S.size());
    for (size_t k = 0; k < S.size(); ++k) S2[k] = S[k] * S[k];
    cudaFree(c->dSsq);
    CK(cudaMalloc(&c->dSsq, S2.size() * sizeof(double)));
    CK(cudaMemcpy(c->dSsq, S2.data(), S2.size() * sizeof(double), cudaMemcpyHostToDevice));
  }
  CK(cudaMalloc(&c->dTheta, nx * sizeof(double)));
  CK(cudaMalloc(&c->dThetaM, nx * sizeof(double)));
  CK(cudaMalloc(&c->dE0, e0.size() * sizeof(double)));
  CK(cudaMemcpy(c->dS, S.data(), S.size() * sizeof(double), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(c->dTheta, th.data(), nx * sizeof(double), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(c->dThetaM, thm.data(), nx * sizeof(double), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(c->dE0, e0.data(), e0.size() * sizeof(double), cudaMemcpyHostToDevice));
  c->op = *op;
  c->n = n;
  c->n_x = nx;
  c->rich_it = 0;
  c->has_op = true;
  c->has_obs = false;
  return LRK_OK;
}

int lrk_set_observation(lrk_ctx* c, const lrk_obs_desc* obs) {
  if (!c || !obs) return LRK_ERR_CONFIG;
  if (!c->has_op) return fail(c, LRK_ERR_CONFIG, "install the operator first");
  CK(cudaSetDevice(c->device));
  const int n = c->n;
  cudaFree(c->dList); cudaFree(c->dS1T); cudaFree(c->dS2); cudaFree(c->dS1); cudaFree(c->dS2T);
  c->dList = nullptr; c->dS1T = c->dS2 = c->dS1 = c->dS2T = nullptr;
  c->obs_kind = obs->kind;
  if (obs->kind == LRK_OBS_FULL) {
    c->n_obs = (int)c->n_x;
  } else if (obs->kind == LRK_OBS_SUBGRID) {
    if (c->op.dim != 2)
      return fail(c, LRK_ERR_UNSUPPORTED, "separable subgrids are 2-D; pass a dof list in 3-D");
    const int s1 = obs->n1, s2 = obs->n2;
    if (s1 < 1 || s2 < 1) return fail(c, LRK_ERR_CONFIG, "empty sensor subgrid");
    std::vector<double> S1T((size_t)n * s1), S2((size_t)s2 * n), S1((size_t)s1 * n),
        S2T((size_t)n * s2);
    const double f = std::sqrt(2.0 / (n + 1));
    auto Sv = [&](int j, int k) { return f * std::sin(M_PI * (double)(j + 1) * (double)(k + 1) / (n + 1)); };
    for (int a = 0; a < s1; ++a) {
      const int i1 = obs->idx1[a];
      if (i1 < 0 || i1 >= n) return fail(c, LRK_ERR_CONFIG, "sensor index out of range");
      for (int k = 0; k < n; ++k) { S1T[(size_t)k * s1 + a] = Sv(k, i1); S1[(size_t)a * n + k] = Sv(i1, k); }
    }
    for (int b = 0; b < s2; ++b) {
      const int i2 = obs->idx2[b];
      if (i2 < 0 || i2 >= n) return fail(c, LRK_ERR_CONFIG, "sensor index out of range");
      for (int k = 0; k < n; ++k) { S2[(size_t)b * n + k] = Sv(i2, k); S2T[(size_t)k * s2 + b] = Sv(k, i2); }
    }
    CK(cudaMalloc(&c->dS1T, S1T.size() * 8)); CK(cudaMalloc(&c->dS2, S2.size() * 8));
    CK(cudaMalloc(&c->dS1, S1.size() * 8)); CK(cudaMalloc(&c->dS2T, S2T.size() * 8));
    CK(cudaMemcpy(c->dS1T, S1T.data(), S1T.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->dS2, S2.data(), S2.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->dS1, S1.data(), S1.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->dS2T, S2T.data(), S2T.size() * 8, cudaMemcpyHostToDevice));
    c->s1 = s1; c->s2 = s2;
    c->n_obs = s1 * s2;
    // physical dof list of the subgrid (x1 fastest), used by physical-space sweeps
    std::vector<int32_t> lst((size_t)s1 * s2);
    for (int b = 0; b < s2; ++b)
      for (int a2 = 0; a2 < s1; ++a2) lst[(size_t)b * s1 + a2] = obs->idx2[b] * n + obs->idx1[a2];
    CK(cudaMalloc(&c->dList, lst.size() * sizeof(int32_t)));
    CK(cudaMemcpy(c->dList, lst.data(), lst.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
  } else if (obs->kind == LRK_OBS_LIST) {
    if (obs->n_list < 0) return fail(c, LRK_ERR_CONFIG, "negative sensor count");
    c->n_obs = obs->n_list;
    if (obs->n_list > 0) {
      for (int k = 0; k < obs->n_list; ++k)
        if (obs->list[k] < 0 || obs->list[k] >= c->n_x)
          return fail(c, LRK_ERR_CONFIG, "sensor dof out of range");
      CK(cudaMalloc(&c->dList, obs->n_list * sizeof(int32_t)));
      CK(cudaMemcpy(c->dList, obs->list, obs->n_list * sizeof(int32_t), cudaMemcpyHostToDevice));
    }
  } else {
    return fail(c, LRK_ERR_CONFIG, "unknown observation kind");
  }
  c->has_obs = true;
  return LRK_OK;
}

int lrk_truncate(lrk_ctx* c, const lrk_lr* in, lrk_lr* out, double eps0, int r_max, int flags,
                 int* r_out, void* stream) {
  if (!c || !in || !out) return LRK_ERR_CONFIG;
  CK(cudaSetDevice(c->device));
  cudaStream_t s = (cudaStream_t)stream;
  if (!(eps0 > 0.0 && eps0 < 1.0)) return fail(c, LRK_ERR_SHAPE, "eps0 must lie in (0, 1)");
  if (in->n_x != out->n_x || in->n_t != out->n_t) return fail(c, LRK_ERR_SHAPE, "shape mismatch");
  if (in->r == 0) { out->r = 0; if (r_out) *r_out = 0; return LRK_OK; }
  TruncOut to;
  TRY(run_truncate(c, "tu_", in->n_x, in->n_t, in->W1, in->ld1, in->W2, in->ld2, in->r, nullptr,
                   flags, eps0, r_max, out->W1, out->ld1, out->W2, out->ld2, out->cap, nullptr,
                   nullptr, 0, to, s));
  int info[8];
  CK(cudaMemcpyAsync(info, to.info, sizeof(info), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (info[2] != 0) return fail(c, LRK_ERR_SHAPE, "output capacity too small for the truncated rank");
  out->r = info[0];
  if (r_out) *r_out = info[0];
  return LRK_OK;
}

int lrk_singular_values(lrk_ctx* c, const lrk_lr* a, double* s_host, int cap, int* n_out,
                        void* stream) {
  if (!c || !a) return LRK_ERR_CONFIG;
  CK(cudaSetDevice(c->device));
  cudaStream_t s = (cudaStream_t)stream;
  if (a->r == 0) { if (n_out) *n_out = 0; return LRK_OK; }
  const int R = a->r;
  WS(double, o1, "sv_o1", a->n_x * (int64_t)R);
  WS(double, o2, "sv_o2", (int64_t)a->n_t * R);
  WS(double, sv, "sv_all", NMAX);
  TruncOut to;
  TRY(run_truncate(c, "sv_", a->n_x, a->n_t, a->W1, a->ld1, a->W2, a->ld2, R, nullptr, 0, 1e-300,
                   -1, o1, a->n_x, o2, a->n_t, R, nullptr, sv, 1, to, s));
  std::vector<double> h(R);
  CK(cudaMemcpyAsync(h.data(), sv, R * sizeof(double), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  const int n = std::min(R, cap);
  for (int i = 0; i < n; ++i) s_host[i] = h[i];
  if (n_out) *n_out = n;
  return LRK_OK;
}

int lrk_dot(lrk_ctx* c, const lrk_lr* A, const lrk_lr* B, double* out, void* stream) {
  if (!c || !A || !B || !out) return LRK_ERR_CONFIG;
  CK(cudaSetDevice(c->device));
  cudaStream_t s = (cudaStream_t)stream;
  if (A->n_x != B->n_x || A->n_t != B->n_t) return fail(c, LRK_ERR_SHAPE, "shape mismatch");
  if (A->r == 0 || B->r == 0) { *out = 0.0; return LRK_OK; }
  const int na = A->r, nb = B->r, nout = na * nb;
  // Gram blocks A1^T B1 (n_x rows) and A2^T B2 (n_t rows) on the FP64 tensor
  // pipe, per-CTA partials reduced in parallel over the outputs, then the
  // Hadamard sum (lowrank.py:163-168)
  const int g1 = grid1(A->n_x, 4096, c->num_sms), g2 = grid1(A->n_t, 64, c->num_sms / 4);
  const int gd = (nout + 255) / 256;
  WS(double, p1, "dot_p1", (int64_t)g1 * nout);
  WS(double, p2, "dot_p2", (int64_t)g2 * nout);
  WS(double, pd, "dot_pd", gd);
  WS(double, res, "dot_res", 1);
  launch_gram(A->W1, A->ld1, na, B->W1, B->ld1, nb, A->n_x, p1, g1, s);
  CKL();
  launch_gram(A->W2, A->ld2, na, B->W2, B->ld2, nb, A->n_t, p2, g2, s);
  CKL();
  dot_parts_kernel<<<gd, 256, 0, s>>>(p1, g1, p2, g2, nout, pd);
  CKL();
  dot_sum_kernel<<<1, 32, 0, s>>>(pd, gd, res);
  CKL();
  c->launches += 4;
  CK(cudaMemcpyAsync(out, res, sizeof(double), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return LRK_OK;
}

int lrk_step_solve(lrk_ctx* c, const double* B, int64_t ldb, int ncols, int adjoint, double* X,
                   int64_t ldx, void* stream) {
  if (!c) return LRK_ERR_CONFIG;
  CK(cudaSetDevice(c->device));
  TRY(check_op(c));
  cudaStream_t s = (cudaStream_t)stream;
  if (ncols <= 0) return LRK_OK;
  const int64_t nx = c->n_x;
  if (phys_basis(c)) {  // convection-diffusion: preconditioned GMRES per column
    WS(double, xc, "ss_x", nx);
    WS(double, bc, "ss_b", nx);
    for (int j = 0; j < ncols; ++j) {
      CK(cudaMemcpyAsync(bc, B + (int64_t)j * ldb, nx * sizeof(double), cudaMemcpyDeviceToDevice, s));
      TRY(gmres_solve(c, bc, xc, adjoint != 0, STEP_RTOL, nullptr, s));
      CK(cudaMemcpyAsync(X + (int64_t)j * ldx, xc, nx * sizeof(double), cudaMemcpyDeviceToDevice, s));
    }
    return LRK_OK;
  }
  // heat: S is symmetric, S^{-T} = S^{-1}
  WS(double, T2, "ss_T2", nx * (int64_t)ncols);
  TRY(dst2(c, B, ldb, T2, nx, ncols, nullptr, 1.0, s));
  scale_rows_kernel<<<dim3(grid1(nx, 256, 1024), ncols), 256, 0, s>>>(T2, nx, c->dThetaM, nx,
                                                                       ncols, nullptr, 1.0, T2, nx);
  CKL();
  TRY(dst2(c, T2, nx, X, ldx, ncols, nullptr, 1.0, s));
  return LRK_OK;
}

int lrk_poisson_solve(lrk_ctx* c, const double* B, int64_t ldb, int ncols, double* X,
                      int64_t ldx, void* stream) {
  if (!c) return LRK_ERR_CONFIG;
  CK(cudaSetDevice(c->device));
  TRY(check_op(c));
  if (phys_basis(c)) return fail(c, LRK_ERR_UNSUPPORTED, "the steady Poisson solve is heat-only");
  cudaStream_t s = (cudaStream_t)stream;
  if (ncols <= 0) return LRK_OK;
  const int64_t nx = c->n_x;
  WS(double, T2, "ps_T2", nx * (int64_t)ncols);
  TRY(dst2(c, B, ldb, T2, nx, ncols, nullptr, 1.0, s));
  scale_rows_kernel<<<dim3(grid1(nx, 256, 1024), ncols), 256, 0, s>>>(T2, nx, c->dInvLam, nx,
                                                                       ncols, nullptr, 1.0, T2, nx);
  CKL();
  TRY(dst2(c, T2, nx, X, ldx, ncols, nullptr, 1.0, s));
  return LRK_OK;
}

int lrk_operator_apply(lrk_ctx* c, const lrk_lr* Y, int adjoint, lrk_lr* out, void* stream) {
  if (!c || !Y || !out) return LRK_ERR_CONFIG;
  CK(cudaSetDevice(c->device));
  if (!c->has_op) return fail(c, LRK_ERR_CONFIG, "no operator installed");
  cudaStream_t s = (cudaStream_t)stream;
  const int r = Y->r;
  if (out->cap < 2 * r) return fail(c, LRK_ERR_SHAPE, "output capacity must be >= 2r");
  if (r == 0) { out->r = 0; return LRK_OK; }
  const lrk_operator_desc& op = c->op;
  StencilArgs a = make_stencil(op, adjoint != 0);
  a.X = Y->W1; a.ldx = Y->ld1; a.Y = out->W1; a.ldy = out->ld1; a.ncols = r;
  // (-M W1) into the second r columns in the same pass over W1
  a.Ycopy = out->W1 + (int64_t)r * out->ld1; a.ldycopy = out->ld1; a.copy_scale = -op.m_scale;
  launch_stencil(a, s);
  CKL();
  // W2 copy into the first r columns; shifted W2 into the second r
  scale_cols_kernel<<<dim3(grid1(Y->n_t, 256, 64), r), 256, 0, s>>>(Y->W2, Y->ld2, Y->n_t, nullptr,
                                                                     nullptr, r, 1.0, out->W2, out->ld2);
  CKL();
  shift_kernel<<<dim3(grid1(Y->n_t, 256, 1 << 30), r), 256, 0, s>>>(
      Y->W2, Y->ld2, Y->n_t, r, adjoint, out->W2 + (int64_t)r * out->ld2, out->ld2, Y->W1, Y->ld1,
      0, -op.m_scale, out->W1 + (int64_t)r * out->ld1, out->ld1);
  CKL();
  out->r = 2 * r;
  return LRK_OK;
}

int lrk_st_solve_sweep(lrk_ctx* c, const lrk_lr* rhs, int adjoint, int compress_every,
                       double eps0, int r_max, lrk_lr* out, int* trace, int trace_cap,
                       int* trace_len, void* stream) {
  if (!c || !rhs || !out) return LRK_ERR_CONFIG;
  CK(cudaSetDevice(c->device));
  TRY(check_op(c));
  cudaStream_t s = (cudaStream_t)stream;
  if (rhs->n_x != c->n_x || rhs->n_t != c->op.n_t)
    return fail(c, LRK_ERR_SHAPE, "rhs shape does not match the operator");
  if (trace_len) *trace_len = 0;
  if (rhs->r == 0) { out->r = 0; return LRK_OK; }
  const int64_t nx = c->n_x;
  const int nt = c->op.n_t;
  WS(double, Bh, "api_B", nx * (int64_t)rhs->r);
  TRY(basis_xform(c, rhs->W1, rhs->ld1, Bh, nx, rhs->r, nullptr, 1.0, s));
  SweepOut o;
  TRY(run_sweep(c, "s0_", Bh, nx, rhs->r, nullptr, rhs->W2, rhs->ld2, adjoint, compress_every, eps0,
                r_max, o, s));
  int info[8];
  CK(cudaMemcpyAsync(info, o.info, sizeof(info), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (info[2] != 0) return fail(c, LRK_ERR_NUMERICAL, "sweep rank exceeded the device core limit");
  const int r = info[0];
  if (r > out->cap) return fail(c, LRK_ERR_SHAPE, "output capacity too small for the pane rank");
  if (r > 0) {
    TRY(basis_xform(c, o.U, o.ldu, out->W1, out->ld1, r, nullptr, 1.0, s));
    scale_cols_kernel<<<dim3(grid1(nt, 256, 64), r), 256, 0, s>>>(o.V, o.ldv, nt, o.sigma, nullptr,
                                                                   r, 1.0, out->W2, out->ld2);
    CKL();
    TRY(flip(c, out->W1, out->ld1, nx, out->W2, out->ld2, nt, nullptr, r, s));
  }
  out->r = r;
  if (trace) {
    const int n = std::min(trace_cap, o.nflush + 1);
    CK(cudaMemcpyAsync(trace, o.trace, n * sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (trace_len) *trace_len = n;
  }
  return LRK_OK;
}

int lrk_hessian_apply_ic(lrk_ctx* c, const lrk_hessian_desc* hd, int nbatch, const double* V,
                         int64_t ldv, double* OUT, int64_t ldo, int* max_rank, void* stream) {
  if (!c) return LRK_ERR_CONFIG;
  CK(cudaSetDevice(c->device));
  TRY(check_op(c));
  TRY(hd_check(c, hd));
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t nx = c->n_x;
  const int nt = c->op.n_t;
  const double M = c->op.m_scale, sg = std::sqrt(hd->gamma_prior);
  WS(double, Bv, "ic_B", nx);
  WS(double, q, "ic_q", nx);
  for (int b = 0; b < nbatch; ++b) {
    const double* v = V + (int64_t)b * ldv;
    double* out = OUT + (int64_t)b * ldo;
    // inject: rhs = (M sqrt(g) v) e_0^T, spectral  (forward.py:108-109)
    TRY(basis_xform(c, v, nx, Bv, nx, 1, nullptr, sg * M, s));
    TRY(apply_prior(c, hd, Bv, nx, 1, nullptr, s));
    SweepOut fw, bw;
    TRY(run_sweep(c, "f_", Bv, nx, 1, nullptr, c->dE0, nt, 0, hd->compress_every, hd->eps0,
                  hd->r_max, fw, s));
    double *Zh, *Z2;
    int64_t ldz = nx;
    int* zinfo;
    int zcap;
    TRY(obs_weight(c, fw, hd->obs_weight, hd->obs_every, hd->eps0, hd->r_max, &Zh, &ldz, &Z2, &zinfo,
                   &zcap, s));
    TRY(run_sweep(c, "b_", Zh, ldz, zcap, zinfo, Z2, nt, 1, hd->compress_every, hd->eps0, hd->r_max,
                  bw, s));
    // extract: sqrt(g) M Q.column(0)  (forward.py:111-112)
    column_eval_kernel<<<grid1(nx, 256, 1024), 256, 0, s>>>(bw.U, bw.ldu, nx, bw.sigma, bw.V,
                                                              bw.ldv, 0, bw.info, q);
    CKL();
    TRY(apply_prior(c, hd, q, nx, 1, nullptr, s));
    TRY(basis_xform(c, q, nx, out, nx, 1, nullptr, sg * M, s));
    int mr = 0;
    TRY(host_max_rank(c, fw, zinfo, bw, nullptr, &mr, hd->compress_every, 1, 1, s));
    if (max_rank) max_rank[b] = mr;
  }
  return LRK_OK;
}

int lrk_hessian_apply_st(lrk_ctx* c, const lrk_hessian_desc* hd, const lrk_lr* v, lrk_lr* out,
                         int* max_rank, void* stream) {
  if (!c || !v || !out) return LRK_ERR_CONFIG;
  CK(cudaSetDevice(c->device));
  TRY(check_op(c));
  TRY(hd_check(c, hd));
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t nx = c->n_x;
  const int nt = c->op.n_t;
  if (v->n_x != nx || v->n_t != nt) return fail(c, LRK_ERR_SHAPE, "field shape mismatch");
  if (v->r == 0) { out->r = 0; if (max_rank) *max_rank = 0; return LRK_OK; }
  const double M = c->op.m_scale, tau = c->op.tau, sg = std::sqrt(hd->gamma_prior);
  WS(double, Bh, "st_B", nx * (int64_t)v->r);
  // rhs = tau M sqrt(g) v  (forward.py:121-122, hessian.py:236)
  TRY(basis_xform(c, v->W1, v->ld1, Bh, nx, v->r, nullptr, tau * M * sg, s));
  TRY(apply_prior(c, hd, Bh, nx, v->r, nullptr, s));
  SweepOut fw, bw;
  TRY(run_sweep(c, "f_", Bh, nx, v->r, nullptr, v->W2, v->ld2, 0, hd->compress_every, hd->eps0,
                hd->r_max, fw, s));
  double *Zh, *Z2;
  int64_t ldz = nx;
  int* zinfo;
  int zcap;
  TRY(obs_weight(c, fw, hd->obs_weight, hd->obs_every, hd->eps0, hd->r_max, &Zh, &ldz, &Z2, &zinfo,
                 &zcap, s));
  TRY(run_sweep(c, "b_", Zh, ldz, zcap, zinfo, Z2, nt, 1, hd->compress_every, hd->eps0, hd->r_max,
                bw, s));
  // out = truncate(sqrt(g) tau M Q)  (hessian.py:242)
  const int cap = bw.ucap;
  WS(double, Up, "st_Uphys", nx * (int64_t)cap);
  WS(double, W2o, "st_W2o", (int64_t)nt * cap);
  if (hd->prior_gamma > 0.0 && !phys_basis(c)) {
    // spectral rows: prior factor, then one DST to physical rows
    WS(double, Tp, "st_Tprior", nx * (int64_t)cap);
    prior_scale_kernel<<<dim3(grid1(nx, 256, 1024), cap), 256, 0, s>>>(
        bw.U, bw.ldu, c->dLam, nx, cap, bw.info, 1.0, hd->prior_delta, hd->prior_gamma, Tp, nx);
    CKL();
    TRY(dst2(c, Tp, nx, Up, nx, cap, bw.info, 1.0, s));
  } else {
    TRY(basis_xform(c, bw.U, bw.ldu, Up, nx, cap, bw.info, 1.0, s));
  }
  if (hd->prior_gamma > 0.0 && phys_basis(c)) {
    // prior on the output's spatial factor (physical rows)
    WS(double, Tp, "st_Tprior", nx * (int64_t)cap);
    TRY(dst2(c, Up, nx, Tp, nx, cap, bw.info, 1.0, s));
    prior_scale_kernel<<<dim3(grid1(nx, 256, 1024), cap), 256, 0, s>>>(
        Tp, nx, c->dLam, nx, cap, bw.info, 1.0, hd->prior_delta, hd->prior_gamma, Tp, nx);
    CKL();
    TRY(dst2(c, Tp, nx, Up, nx, cap, bw.info, 1.0, s));
  }
  scale_cols_kernel<<<dim3(grid1(nt, 256, 64), cap), 256, 0, s>>>(bw.V, bw.ldv, nt, bw.sigma,
                                                                   bw.info, cap, sg * tau * M, W2o, nt);
  CKL();
  TruncOut to;
  TRY(run_truncate(c, "so_", nx, nt, Up, nx, W2o, nt, cap, bw.info,
                   (hd->prior_gamma > 0.0 ? 0 : LRK_TRUNC_W1_ORTHO) | LRK_TRUNC_W2_ORTHOSCALED, hd->eps0, hd->r_max, out->W1,
                   out->ld1, out->W2, out->ld2, out->cap, nullptr, nullptr, 0, to, s));
  int info[8];
  CK(cudaMemcpyAsync(info, to.info, sizeof(info), cudaMemcpyDeviceToHost, s));
  int mr = 0;
  TRY(host_max_rank(c, fw, zinfo, bw, to.info, &mr, hd->compress_every, v->r, nt, s));
  if (info[2] != 0) return fail(c, LRK_ERR_SHAPE, "output capacity too small");
  out->r = info[0];
  if (max_rank) *max_rank = mr;
  return LRK_OK;
}

int lrk_cgs2(lrk_ctx* c, const double* Q, int64_t ldq, int k, double* w, int n, double* h_host,
             double* norm_out, void* stream) {
  if (!c) return LRK_ERR_CONFIG;
  CK(cudaSetDevice(c->device));
  cudaStream_t s = (cudaStream_t)stream;
  const int g = grid1(n, 4096, 2 * c->num_sms);
  const int kk = std::max(k, 1);
  // the basis grows by one column per Arnoldi step: size the workspace in
  // powers of two so that it is reallocated O(log k) times, not every call
  int kcap = 64;
  while (kcap < kk) kcap *= 2;
  WS(double, part, "cg_part", (int64_t)g * kcap);
  WS(double, hp, "cg_h", kcap);
  WS(double, hacc, "cg_hacc", kcap + 1);
  CK(cudaMemsetAsync(hacc, 0, (kk + 1) * sizeof(double), s));
  for (int pass = 0; pass < 2 && k > 0; ++pass) {
    launch_gram(Q, ldq, k, w, n, 1, n, part, g, s);
    CKL();
    reduce_parts_kernel<<<grid1(k, 256, 64), 256, 0, s>>>(part, g, k, hp, hacc);
    CKL();
    sub_qh_kernel<<<grid1(n, 256, 2048), 256, 0, s>>>(Q, ldq, k, hp, w, n);
    CKL();
  }
  launch_gram(w, n, 1, w, n, 1, n, part, g, s);
  CKL();
  reduce_parts_kernel<<<1, 256, 0, s>>>(part, g, 1, hacc + kk, nullptr);
  CKL();
  std::vector<double> hh(kk + 1);
  CK(cudaMemcpyAsync(hh.data(), hacc, (kk + 1) * sizeof(double), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  for (int i = 0; i < k; ++i) h_host[i] = hh[i];
  if (norm_out) *norm_out = std::sqrt(std::max(hh[kk], 0.0));
  return LRK_OK;
}

int lrk_combine(lrk_ctx* c, const double* Q, int64_t ldq, int k, const double* c_host, int n,
                double* y, void* stream) {
  if (!c) return LRK_ERR_CONFIG;
  CK(cudaSetDevice(c->device));
  cudaStream_t s = (cudaStream_t)stream;
  WS(double, cf, "cb_cf", std::max(k, 1));
  CK(cudaMemcpyAsync(cf, c_host, k * sizeof(double), cudaMemcpyHostToDevice, s));
  combine_kernel<<<grid1(n, 256, 2048), 256, 0, s>>>(Q, ldq, k, cf, y, n);
  CKL();
  CK(cudaStreamSynchronize(s));
  return LRK_OK;
}

}  // extern "C"

// device-resident Krylov layer (fused add-truncate, batched dots, GMRES)
#include "lrk_krylov.inc"
