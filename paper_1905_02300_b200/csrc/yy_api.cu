// yy_api.cu — the C ABI of include/yy.h: context, host-side geometry tables,
// Yin<->Yang stencil construction, and the per-step launch sequence
// (SURVEY.md §3 (ii)).  Device work is entirely in yy_kernels.cu.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cmath>
#include <cstdio>
#include <algorithm>
#include <cstring>
#include <cstdlib>
#include <functional>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/yy.h"
#include "../../include/yy_test.h"
#include "yy_dev.cuh"
#include "yy_internal.h"

using namespace yy;

namespace {

// field slots (both patches contiguous per array)
enum { FT = 0, FP1, FP2, FUR1, FUT1, FUP1, FUR2, FUT2, FUP2, NF };
constexpr int FKIND[NF] = {KC, KC, KC, KR, KT, KP, KR, KT, KP};
// wall fields
enum { WT = 0, WUR, WUT, WUP, NW };
constexpr int WKIND[NW] = {KC, KR, KT, KP};

double tf_value(int tf, double t) {
  switch (tf) {
    case YY_TF_ONE: return 1.0;
    case YY_TF_COS: return std::cos(t);
    case YY_TF_SIN: return std::sin(t);
    case YY_TF_COS2: return std::cos(t) * std::cos(t);
  }
  return 0.0;
}

}  // namespace

struct yy_ctx {
  Geo g{};
  double R1 = 1, R2 = 2, Pr = 1, Ra = 0, dt = 1e-3, chi = 1.0;
  int max_iters = 100, fixed_iters = 0;
  bool fuse = false;           // residual fused into the first sweep (YY_FUSE=1; measured slower on C3 so far)
  // 2: the whole Schwarz loop as one CUDA graph with a device-side WHILE node (one
  // host sync per step); 1: each iteration as a graph, host-side loop; 0: streams
  int use_graph = 2;           // YY_GRAPH=0/1/2
  // alternate the block order of consecutive residual / sweep / pressure kernels
  // (YY_ALT_ORDER=0: off); rev_next = the order of the next one
  bool alt_order = true;
  int rev_next = 0;
  // distribution: npatch = g.npatch local patches, global id of
  // local patch 0 = patch0.  mode 0: both patches here; 1: loopback pair (two
  // contexts in one process sharing a stream, test path); 2: NCCL, one rank per patch.
  int patch0 = 0;
  int nslab = 1, slab = 0, roff = 0, nr_glob = 0;   // radial slab of the patch (nslab > 1)
  int schwarz = 0;             // 0 additive (RD26), 1 multiplicative (Algorithm 1 as printed),
                               // 2 none (single domains, Theorem 1)
  double* energy_buf = nullptr;   // yy_energy: zero wall + block partials + result
  bool imex = false;           // YY_ADVECTION = 1: transport terms explicit only
  // instantiated device-loop graphs (one step's Schwarz loop, YY_GRAPH=2), keyed by
  // everything the captured launches bake in: the level pointers rotate through a
  // short cycle (3 for T/u, 2 for p), so a run replays a handful of executables
  // instead of capturing and instantiating one per step; cleared by set_param /
  // set_stream
  struct LoopGraph {
    std::vector<const void*> key;
    double tol;
    int rev_in, rev_out;
    long long per_iter;
    cudaGraphExec_t exec;
  };
  std::vector<LoopGraph> loop_graphs;
  double* zero = nullptr;      // IMEX: zero a* / row-weight / reaction arrays of the split rows
  bool heat_only = false;      // eq:HeatDouglas alone (u = 0, no momentum / pressure)
  double flux_eps = 0.0;       // > 0: Algorithm 1 step 4 with this penalty eps
  double* bsplit[4][3] = {};   // split-row tables (Geo::bsplit)
  double* tsplit[4][3] = {};   // factor-row tables (Geo::tsplit)
  double* adv[4][3] = {};      // per-step transport-velocity row weights (Geo::adv)
  const double* line_a[3] = {};   // a* of the last yy_line_prepare
  double* react_t = nullptr;   // Astar::rt, Astar::rp (per step)
  double* react_p = nullptr;
  double flux_a2 = 0.0, flux_area = 0.0;   // |a|^2 and |dOmega| of one patch (host geometry)
  int mode = 0;
  int world = 1, rank = 0;
  void* nccl = nullptr;        // ncclComm_t
  double* fr_send = nullptr;   // fringe values this patch donates to the partner
  double* fr_recv = nullptr;   // fringe values received for this patch
  long long fr_n = 0;
  // radial slabs: partitioned r-sweep buffers and the gathered norm sums
  double* Vq[4] = {};          // per quantity: the r-lines' responses to the lower / upper
  double* Wq[4] = {};          // neighbour slab's boundary unknown (per step)
  bool vw_fresh = true;        // this iteration writes Vq / Wq (the step's first)
  double* IFq[4] = {};         // per quantity: [nlines][6] this slab's boundary rows (x0 each
                               // iteration; xlo, xhi columns per step, like Vq / Wq)
  double* IFall = nullptr;     // [nslab][nlines][6] every slab of the patch
  double* LH = nullptr;        // [nlines][2]
  double* gath = nullptr;      // [world][2 + 2 NSLOT] every context's sums
  int nblk[NSLOT] = {};
  std::vector<yy_ctx*> group;  // loopback: every context of the shell, index = rank
  double t = 0.0;
  cudaStream_t st = nullptr;
  std::string err;
  bool dead = false;
  double* tab1d = nullptr;
  double* n[NF] = {};
  double* m[NF] = {};
  double* it[NF] = {};
  double* astar[3] = {};
  double* G[NF] = {};
  double* R = nullptr;
  double* part = nullptr;
  int maxb = 0;
  double* red = nullptr;
  double* red_host = nullptr;   // pinned
  double* ctl = nullptr;        // device-side Schwarz loop: iterations, rho, NaN flag
  double* dp1 = nullptr;        // p1^(k) - p1^n, both patches (two-patch contexts; NULL otherwise)
  // two-patch contexts: the three fringe interpolation classes run concurrently
  // (fork / join on st; YY_PAR_INTERP=0: one after the other)
  cudaStream_t aux[2] = {};
  cudaEvent_t fork[3] = {};
  // YY_DEFER_INTERP=1 (default 0: measured +-0 on B200): only T's fringe ahead of the
  // T solve, the p / u fringes beside it, joined before the first momentum residual
  bool defer_interp = false;
  bool interp_pending = false;
  double* wterm[2][MAXSRC][NW] = {};
  int nw[2] = {0, 0};
  int wtf[2][MAXSRC] = {};
  double* wl[3][NW] = {};       // wall data at t_{n-1}, t_n, t_{n+1}
  double* sterm[2][MAXSRC][4] = {};
  double* wterm_buf[2][MAXSRC][NW] = {};   // owned buffers behind wterm / sterm (reused by re-sets)
  double* sterm_buf[2][MAXSRC][4] = {};
  int ns[2] = {0, 0};
  int stf[2][MAXSRC] = {};
  // interpolation tables (device)
  std::vector<void*> allocs;
  // device memory hook (yy_set_allocator; copied from the process default at create)
  void* (*alloc_fn)(size_t, void*) = nullptr;
  void (*free_fn)(void*, void*) = nullptr;
  void* alloc_user = nullptr;
  CCTab tcc{};
  VecTab tth{}, tph{};
  std::vector<int> st_iters;
  std::vector<double> st_rho;
  // instrumentation: kernel launch counter (always on) and an optional
  // CUDA-event profiler per kernel class (YY_PROFILE)
  long long launches = 0;
  bool prof_on = false;
  struct Rec { const char* name; cudaEvent_t a, b; };
  std::vector<Rec> pending;
  std::vector<cudaEvent_t> pool;
  std::map<std::string, std::pair<long long, double>> prof;
};

namespace {

yy_status fail(yy_ctx* c, yy_status s, const std::string& msg) {
  if (c) c->err = msg;
  if (c && s == YY_ECUDA) c->dead = true;
  return s;
}

#define CK(call)                                                                   \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess) return fail(ctx, YY_ECUDA, std::string(#call ": ") + cudaGetErrorString(e_)); \
  } while (0)

template <class T>
yy_status dalloc(yy_ctx* ctx, T** p, size_t count) {
  void* q = nullptr;
  const size_t bytes = count * sizeof(T) + 16;
  if (ctx->alloc_fn) {                       // injected allocator (yy_set_allocator)
    q = ctx->alloc_fn(bytes, ctx->alloc_user);
    if (!q) return fail(ctx, YY_ENOMEM, "injected allocator returned NULL");
  } else {
    cudaError_t e = cudaMalloc(&q, bytes);
    if (e != cudaSuccess) return fail(ctx, YY_ENOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  }
  ctx->allocs.push_back(q);
  *p = static_cast<T*>(q);
  return YY_OK;
}

#define TRY(x)                      \
  do {                              \
    yy_status s_ = (x);             \
    if (s_ != YY_OK) return s_;     \
  } while (0)

void clear_loop_graphs(yy_ctx* ctx) {
  for (auto& lg : ctx->loop_graphs) cudaGraphExecDestroy(lg.exec);
  ctx->loop_graphs.clear();
}

// ---- instrumentation ----------------------------------------------------------------
cudaEvent_t ev_get(yy_ctx* ctx) {
  if (!ctx->pool.empty()) {
    cudaEvent_t e = ctx->pool.back();
    ctx->pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

const char* kname(const std::string& s);

struct ProfScope {   // brackets one or more launches of one kernel class
  yy_ctx* ctx;
  yy_ctx::Rec r{};
  // the class name is interned only when the per-class profile is on
  ProfScope(yy_ctx* c, const std::string& name, int nlaunch) : ctx(c) {
    ctx->launches += nlaunch;
    if (ctx->prof_on) {
      r.name = kname(name);
      r.a = ev_get(ctx);
      r.b = ev_get(ctx);
      cudaEventRecord(r.a, ctx->st);
    }
  }
  ~ProfScope() {
    if (ctx->prof_on) {
      cudaEventRecord(r.b, ctx->st);
      ctx->pending.push_back(r);
    }
  }
};

void prof_collect(yy_ctx* ctx) {   // call after a stream synchronisation
  for (auto& r : ctx->pending) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    auto& e = ctx->prof[r.name];
    e.first += 1;
    e.second += ms;
    ctx->pool.push_back(r.a);
    ctx->pool.push_back(r.b);
  }
  ctx->pending.clear();
}

const char* QNAME[4] = {"T", "ur", "ut", "up"};
const char* AXNAME[3] = {"r", "th", "ph"};
std::string g_names_store[512];
std::mutex g_names_mu;
const char* kname(const std::string& s) {   // interned kernel-class names (process-wide, locked)
  std::lock_guard<std::mutex> lk(g_names_mu);
  for (auto& x : g_names_store) {
    if (x == s) return x.c_str();
    if (x.empty()) { x = s; return x.c_str(); }
  }
  return "other";
}

// ---- geometry (reading RD1/RD2; §2) --------------------------------------
struct HostGeo {
  int nr, nt, np;
  double dr, dth, dph, th0, ph0, R1;
};

HostGeo host_geo(const yy_grid* gr, double R1, double R2) {
  HostGeo h;
  h.nr = gr->nr;
  h.nt = gr->ntheta;
  h.np = gr->nphi;
  h.dr = (R2 - R1) / h.nr;
  h.dth = M_PI / (2.0 * (h.nt - 4));
  const double delta = 2.0 * h.dth;
  h.dph = (1.5 * M_PI + 2.0 * delta) / h.np;
  h.th0 = M_PI / 4 - delta;
  h.ph0 = -0.75 * M_PI - delta;
  h.R1 = R1;
  return h;
}

// Yin (th, ph) -> the other chart's (th~, ph~); the map is an involution
// (PAPER.md L143-144), so the same function serves Yang -> Yin.
void map_other(double th, double ph, double* tt, double* pp) {
  const double x = std::sin(th) * std::cos(ph), y = std::sin(th) * std::sin(ph), z = std::cos(th);
  *tt = std::acos(std::fmax(-1.0, std::fmin(1.0, y)));
  *pp = std::atan2(z, -x);
}

// M_ab = e_a(target chart) . e_b(donor chart) for a,b in (theta, phi) (RD5)
void rot(double th, double ph, double M[2][2]) {
  double tt, pp;
  map_other(th, ph, &tt, &pp);
  const double et[3] = {std::cos(th) * std::cos(ph), std::cos(th) * std::sin(ph), -std::sin(th)};
  const double ep[3] = {-std::sin(ph), std::cos(ph), 0.0};
  const double dt_[3] = {-std::cos(tt) * std::cos(pp), -std::sin(tt), std::cos(tt) * std::sin(pp)};
  const double dp_[3] = {std::sin(pp), 0.0, std::cos(pp)};
  auto dot = [](const double* a, const double* b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; };
  M[0][0] = dot(et, dt_);
  M[0][1] = dot(et, dp_);
  M[1][0] = dot(ep, dt_);
  M[1][1] = dot(ep, dp_);
}

// 4-point Lagrange on a uniform lattice x_m = x0 + m h; base = ceil(s) - 2 (RD42)
void lagr(double x, double x0, double h, int* base, double w[4]) {
  const double s = (x - x0) / h;
  const int b = (int)std::ceil(s) - 2;
  const double u = s - b;
  for (int a = 0; a < 4; ++a) {
    double v = 1.0;
    for (int q = 0; q < 4; ++q)
      if (q != a) v *= (u - q) / (double)(a - q);
    w[a] = v;
  }
  *base = b;
}

struct Lattice {   // (theta, phi) lattice of a kind
  double t0, p0;
  int nt, np;      // node counts
};

Lattice lattice(const HostGeo& h, int K) {
  Lattice L;
  L.t0 = (K == KT) ? h.th0 : h.th0 + 0.5 * h.dth;
  L.p0 = (K == KP) ? h.ph0 : h.ph0 + 0.5 * h.dph;
  L.nt = h.nt + (K == KT);
  L.np = h.np + (K == KP);
  return L;
}

bool stencil(const HostGeo& h, double th, double ph, int donorK, int* jb, int* kb, double* w8) {
  double tt, pp;
  map_other(th, ph, &tt, &pp);
  Lattice L = lattice(h, donorK);
  lagr(tt, L.t0, h.dth, jb, w8);
  lagr(pp, L.p0, h.dph, kb, w8 + 4);
  // donor stencil must use donor solved nodes only (never the donor fringe)
  return *jb >= 1 && *jb + 3 <= L.nt - 2 && *kb >= 1 && *kb + 3 <= L.np - 2;
}

template <class T>
yy_status upload(yy_ctx* ctx, const std::vector<T>& v, const T** out) {
  T* d = nullptr;
  TRY(dalloc(ctx, &d, v.size() ? v.size() : 1));
  if (!v.empty()) CK(cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  *out = d;
  return YY_OK;
}

yy_status build_tables(yy_ctx* ctx, const HostGeo& h) {
  // C / R fringe on the (theta_c, phi_c) lattice
  {
    Lattice L = lattice(h, KC);
    std::vector<int> tj, tk, jb, kb;
    std::vector<double> w;
    for (int j = 0; j < L.nt; ++j)
      for (int k = 0; k < L.np; ++k) {
        if (!(j == 0 || j == L.nt - 1 || k == 0 || k == L.np - 1)) continue;
        int b1, b2;
        double w8[8];
        if (!stencil(h, L.t0 + j * h.dth, L.p0 + k * h.dph, KC, &b1, &b2, w8))
          return fail(ctx, YY_EINVAL, "overlap too small: fringe stencil reaches the donor fringe");
        tj.push_back(j); tk.push_back(k); jb.push_back(b1); kb.push_back(b2);
        w.insert(w.end(), w8, w8 + 8);
      }
    ctx->tcc.n = (int)tj.size();
    TRY(upload(ctx, tj, &ctx->tcc.tj)); TRY(upload(ctx, tk, &ctx->tcc.tk));
    TRY(upload(ctx, jb, &ctx->tcc.jb)); TRY(upload(ctx, kb, &ctx->tcc.kb));
    TRY(upload(ctx, w, &ctx->tcc.w));
  }
  for (int which = 0; which < 2; ++which) {
    const int K = which == 0 ? KT : KP;
    VecTab& T = which == 0 ? ctx->tth : ctx->tph;
    Lattice L = lattice(h, K);
    std::vector<int> tj, tk, jbt, kbt, jbp, kbp;
    std::vector<double> wt, wp, m0, m1;
    for (int j = 0; j < L.nt; ++j)
      for (int k = 0; k < L.np; ++k) {
        if (!(j == 0 || j == L.nt - 1 || k == 0 || k == L.np - 1)) continue;
        const double th = L.t0 + j * h.dth, ph = L.p0 + k * h.dph;
        int b1, b2, b3, b4;
        double w1[8], w2[8], M[2][2];
        if (!stencil(h, th, ph, KT, &b1, &b2, w1) || !stencil(h, th, ph, KP, &b3, &b4, w2))
          return fail(ctx, YY_EINVAL, "overlap too small: fringe stencil reaches the donor fringe");
        rot(th, ph, M);
        tj.push_back(j); tk.push_back(k);
        jbt.push_back(b1); kbt.push_back(b2); jbp.push_back(b3); kbp.push_back(b4);
        wt.insert(wt.end(), w1, w1 + 8);
        wp.insert(wp.end(), w2, w2 + 8);
        m0.push_back(M[which][0]);
        m1.push_back(M[which][1]);
      }
    T.n = (int)tj.size();
    TRY(upload(ctx, tj, &T.tj)); TRY(upload(ctx, tk, &T.tk));
    TRY(upload(ctx, jbt, &T.jb_t)); TRY(upload(ctx, kbt, &T.kb_t));
    TRY(upload(ctx, jbp, &T.jb_p)); TRY(upload(ctx, kbp, &T.kb_p));
    TRY(upload(ctx, wt, &T.w_t)); TRY(upload(ctx, wp, &T.w_p));
    TRY(upload(ctx, m0, &T.m0)); TRY(upload(ctx, m1, &T.m1));
  }
  return YY_OK;
}

long long fsize(const yy_ctx* ctx, int f) { return psize(ctx->g, FKIND[f]); }

// A context's rows of a field of kind K inside the full-patch host array
// (global rows = local rows + roff): host rows [g0, g1] <-> local rows [g0 - roff, ..].
// own_only: the rows this context owns (solved rows plus the wall faces it holds).
void row_window(const yy_ctx* ctx, int K, bool own_only, int* g0, int* g1) {
  const Geo& g = ctx->g;
  const int nrg = ctx->nr_glob + (K == KR);
  if (own_only && ctx->nslab > 1) {
    if (K == KR) { *g0 = (g.wall_lo ? g.ilo_f - 1 : g.ilo_f) + ctx->roff; *g1 = (g.wall_hi ? g.ihi_f + 1 : g.ihi_f) + ctx->roff; }
    else { *g0 = g.ilo_c + ctx->roff; *g1 = g.ihi_c + ctx->roff; }
    return;
  }
  *g0 = std::max(0, ctx->roff);
  *g1 = std::min(nrg - 1, ctx->roff + NRk(g, K) - 1);
}

// copy the window of one patch's field between a full-patch host array and the context
yy_status copy_window(yy_ctx* ctx, int K, double* dev_patch, double* host, bool to_device, bool own_only) {
  const Geo& g = ctx->g;
  int g0, g1;
  row_window(ctx, K, own_only, &g0, &g1);
  const long long plane = (long long)NTk(g, K) * NPk(g, K);
  const size_t bytes = (size_t)(g1 - g0 + 1) * plane * sizeof(double);
  double* d = dev_patch + (long long)(g0 - ctx->roff) * plane;
  double* hh = host + (long long)g0 * plane;
  // on the context's stream, then synchronised: every upload / download is ordered
  // with the step's kernels and with the device-to-device copies of yy_set_fields
  // (system 0), whatever stream the caller uses; pageable host memory is safe too
  CK(cudaMemcpyAsync(to_device ? (void*)d : (void*)hh, to_device ? (const void*)hh : (const void*)d, bytes,
                     to_device ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost, ctx->st));
  CK(cudaStreamSynchronize(ctx->st));
  return YY_OK;
}

yy_status check_args(yy_ctx* ctx, int32_t patch, int32_t level, int32_t system) {
  if (!ctx) return YY_EINVAL;
  if (ctx->dead) return fail(ctx, YY_ESTATE, "context unusable after a CUDA error");
  if (patch < 0 || patch > 1) return fail(ctx, YY_EINVAL, "patch must be 0 (Yin) or 1 (Yang)");
  if (patch < ctx->patch0 || patch >= ctx->patch0 + ctx->g.npatch)
    return fail(ctx, YY_EINVAL, "this context does not hold that patch");
  if (level < 0 || level > 1) return fail(ctx, YY_EINVAL, "level must be 0 (t^n) or 1 (t^{n-1})");
  if (system < 0 || system > 2) return fail(ctx, YY_EINVAL, "system must be 0, 1 or 2");
  return YY_OK;
}

// ---- one time step ------------------------------------------------
// the wall data of time level L (0: t_{n-1}, 1: t_n, 2: t_{n+1}) of every field and
// patch, appended to one batch of linear combinations of the time-basis terms
yy_status eval_walls(yy_ctx* ctx, int L, double t, LinBatch& b) {
  const Geo& g = ctx->g;
  for (int f = 0; f < NW; ++f) {
    const long long ws = 2 * wsize(g, WKIND[f]);   // inner + outer wall of one patch
    for (int p = 0; p < g.npatch; ++p) {
      if (b.njobs >= MAXLIN) return fail(ctx, YY_ESTATE, "internal: wall batch overflow");
      const int q = b.njobs++;
      int nin = 0;
      for (int m = 0; m < ctx->nw[p]; ++m)
        if (ctx->wterm[p][m][f]) {
          b.p[q][nin] = ctx->wterm[p][m][f];
          b.c[q][nin] = tf_value(ctx->wtf[p][m], t);
          ++nin;
        }
      b.out[q] = ctx->wl[L][f] + p * ws;
      b.n[q] = ws;
      b.nin[q] = nin;
    }
  }
  return YY_OK;
}

StaticArgs static_args(yy_ctx* ctx, int q, double tsrc) {
  StaticArgs a{};
  a.imex = ctx->imex;
  a.ar = ctx->astar[0]; a.at = ctx->astar[1]; a.ap = ctx->astar[2];
  a.rt = ctx->react_t; a.rp = ctx->react_p;
  const int f1 = (q == QT) ? FT : (q == QUR ? FUR1 : q == QUT ? FUT1 : FUP1);
  const int f2 = (q == QT) ? FT : f1 + 3;
  a.fn[0] = ctx->n[f1]; a.fn[1] = ctx->n[f2];
  a.fm[0] = ctx->m[f1]; a.fm[1] = ctx->m[f2];
  const int wf = (q == QT) ? WT : (q == QUR ? -1 : q == QUT ? WUT : WUP);
  a.wn = wf >= 0 ? ctx->wl[1][wf] : nullptr;
  a.wm = wf >= 0 ? ctx->wl[0][wf] : nullptr;
  a.p[0] = ctx->n[FP1]; a.p[1] = ctx->n[FP2];
  a.utn[0] = ctx->n[FUT1]; a.utn[1] = ctx->n[FUT2];
  a.utm[0] = ctx->m[FUT1]; a.utm[1] = ctx->m[FUT2];
  a.upn[0] = ctx->n[FUP1]; a.upn[1] = ctx->n[FUP2];
  a.upm[0] = ctx->m[FUP1]; a.upm[1] = ctx->m[FUP2];
  const int sf = (q == QT) ? 0 : q;    // source field index: T, ur, ut, up
  for (int p = 0; p < ctx->g.npatch; ++p) {
    int k = 0;
    for (int m = 0; m < ctx->ns[p]; ++m)
      if (ctx->sterm[p][m][sf]) {
        a.src[p][k] = ctx->sterm[p][m][sf];
        a.gsrc[p][k] = tf_value(ctx->stf[p][m], tsrc);
        ++k;
      }
    a.nsrc[p] = k;
  }
  a.G[0] = ctx->G[f1];
  a.G[1] = ctx->G[f2];
  return a;
}

// factor orders as printed (RD28): first factor solved first
constexpr int ORDER[4][3] = {{0, 1, 2}, {1, 2, 0}, {2, 0, 1}, {0, 1, 2}};

// ---- transports between the contexts of a group --------------
struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

// NCCL is resolved at run time (the process's already-loaded libnccl, e.g.
// torch's, else libnccl.so.2), so libyy.so itself does not depend on it.
NcclApi& nccl_api() {
  static NcclApi a;
  static bool tried = false;
  if (tried) return a;
  tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return a;
#define YY_SYM(f, n) a.f = reinterpret_cast<decltype(a.f)>(dlsym(h, n))
  YY_SYM(GetUniqueId, "ncclGetUniqueId");
  YY_SYM(CommInitRank, "ncclCommInitRank");
  YY_SYM(CommDestroy, "ncclCommDestroy");
  YY_SYM(Send, "ncclSend");
  YY_SYM(Recv, "ncclRecv");
  YY_SYM(GroupStart, "ncclGroupStart");
  YY_SYM(GroupEnd, "ncclGroupEnd");
  YY_SYM(GetErrorString, "ncclGetErrorString");
#undef YY_SYM
  a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.Send && a.Recv && a.GroupStart && a.GroupEnd &&
         a.GetErrorString;
  return a;
}

#define NK(call)                                                                            \
  do {                                                                                      \
    ncclResult_t r_ = (call);                                                               \
    if (r_ != ncclSuccess) return fail(ctx, YY_ENCCL, std::string(#call ": ") + nccl_api().GetErrorString(r_)); \
  } while (0)

// ---- transfers between the contexts of a group ----------------
// A group is every context of one shell: one context (both patches, or one NCCL
// rank), or a loopback set in this process.  rank = patch * nslab + slab.
struct Xfer {
  int src, dst;                                   // ranks
  std::function<const double*(yy_ctx*)> sp;       // source buffer on the src context
  std::function<double*(yy_ctx*)> dp;             // destination buffer on the dst context
  long long count;
};

yy_ctx* ctx_of(std::vector<yy_ctx*>& cs, int rank) {
  for (yy_ctx* c : cs) if (c->rank == rank) return c;
  return nullptr;
}

yy_status run_xfers(std::vector<yy_ctx*>& cs, const std::vector<Xfer>& ops) {
  if (cs.empty() || ops.empty()) return YY_OK;
  yy_ctx* ctx = cs[0];
  if (ctx->mode == 2) {                           // NCCL: this rank's sends and receives, one group call
    NcclApi& N = nccl_api();
    ncclComm_t comm = static_cast<ncclComm_t>(ctx->nccl);
    NK(N.GroupStart());
    for (const Xfer& x : ops) {
      if (x.src == ctx->rank && x.dst == ctx->rank) continue;
      if (x.src == ctx->rank) NK(N.Send(x.sp(ctx), (size_t)x.count, ncclFloat64, x.dst, comm, ctx->st));
      if (x.dst == ctx->rank) NK(N.Recv(x.dp(ctx), (size_t)x.count, ncclFloat64, x.src, comm, ctx->st));
    }
    NK(N.GroupEnd());
    for (const Xfer& x : ops)
      if (x.src == ctx->rank && x.dst == ctx->rank)
        CK(cudaMemcpyAsync(x.dp(ctx), x.sp(ctx), x.count * sizeof(double), cudaMemcpyDeviceToDevice, ctx->st));
    return YY_OK;
  }
  for (const Xfer& x : ops) {                     // loopback: one shared stream, plain copies
    yy_ctx* a = ctx_of(cs, x.src);
    yy_ctx* b = ctx_of(cs, x.dst);
    if (!a || !b) return fail(ctx, YY_ESTATE, "internal: transfer to a context outside the group");
    CK(cudaMemcpyAsync(x.dp(b), x.sp(a), x.count * sizeof(double), cudaMemcpyDeviceToDevice, ctx->st));
  }
  return YY_OK;
}

bool distributed(const std::vector<yy_ctx*>& cs) { return !(cs.size() == 1 && cs[0]->mode == 0); }
bool has_patch(const std::vector<yy_ctx*>& cs, int p) {
  for (const yy_ctx* c : cs) if (c->patch0 == p) return true;
  return false;
}
std::vector<yy_ctx*> of_patch(const std::vector<yy_ctx*>& cs, int p) {
  std::vector<yy_ctx*> out;
  for (yy_ctx* c : cs) if (c->patch0 == p) out.push_back(c);
  return out;
}
int world_of(const yy_ctx* c) { return 2 * c->nslab; }

// N1: r-halo rows of one iterate field with the slab neighbours of the same patch
yy_status exchange_halos(std::vector<yy_ctx*>& cs, int f) {
  yy_ctx* c0 = cs[0];
  if (c0->nslab == 1) return YY_OK;
  const Geo& g = c0->g;
  const int K = FKIND[f], S = c0->nslab, nl = g.ihi_c - g.ilo_c + 1;
  const long long plane = (long long)NTk(g, K) * NPk(g, K);
  // owned boundary rows and the neighbour's halo rows (local indices)
  const int own_lo = (K == KR) ? 2 : 1, own_hi = (K == KR) ? nl + 1 : nl;
  const int halo_lo = (K == KR) ? 1 : 0, halo_hi = (K == KR) ? nl + 2 : nl + 1;
  std::vector<Xfer> ops;
  for (int p = 0; p < 2; ++p)
    for (int sl = 1; sl < S && (c0->mode == 2 || has_patch(cs, p)); ++sl) {
      const int up = p * S + sl, dn = up - 1;      // slab sl and the one below it
      ops.push_back({up, dn, [=](yy_ctx* c) -> const double* { return c->it[f] + own_lo * plane; },
                     [=](yy_ctx* c) { return c->it[f] + halo_hi * plane; }, plane});
      ops.push_back({dn, up, [=](yy_ctx* c) -> const double* { return c->it[f] + own_hi * plane; },
                     [=](yy_ctx* c) { return c->it[f] + halo_lo * plane; }, plane});
    }
  return run_xfers(cs, ops);
}

// the quantity's iterate field
int qfield(int q, int s) { return (q == QT) ? FT : (q == QUR ? FUR1 : q == QUT ? FUT1 : FUP1) + (s == 2 ? 3 : 0); }

ResidArgs resid_args(yy_ctx* ctx, int q, int s) {
  const int f = qfield(q, s);
  ResidArgs r{};
  r.it = ctx->it[f];
  r.n = ctx->n[f];
  const int wf = (q == QT) ? WT : (q == QUR ? -1 : q == QUT ? WUT : WUP);
  r.wnew = wf >= 0 ? ctx->wl[2][wf] : nullptr;
  r.wn = wf >= 0 ? ctx->wl[1][wf] : nullptr;
  r.ar = ctx->astar[0]; r.at = ctx->astar[1]; r.ap = ctx->astar[2];
  r.rt = ctx->react_t; r.rp = ctx->react_p;
  if (ctx->imex) {   // split rows without transport terms
    r.ar = r.at = r.ap = r.rt = r.rp = ctx->zero;
    r.noadv = 1;
  }
  r.G = ctx->G[f];
  r.R = ctx->R;
  r.Tit = ctx->it[FT]; r.Tn = ctx->n[FT];
  const int o = (s == 2) ? 3 : 0;
  r.urit = ctx->it[FUR1 + o]; r.urn = ctx->n[FUR1 + o];
  r.utit = ctx->it[FUT1 + o]; r.utn = ctx->n[FUT1 + o];
  r.p1it = ctx->it[FP1]; r.p1n = ctx->n[FP1];
  r.dp1 = (s == 2) ? ctx->dp1 : nullptr;
  return r;
}

SweepArgs sweep_args(yy_ctx* ctx, int q, int s, int slot) {
  SweepArgs w{};
  w.ar = ctx->astar[0]; w.at = ctx->astar[1]; w.ap = ctx->astar[2];
  w.rt = ctx->react_t; w.rp = ctx->react_p;
  if (ctx->imex) {
    w.ar = w.at = w.ap = w.rt = w.rp = ctx->zero;
    w.noadv = 1;
  }
  w.R = ctx->R; w.psi = ctx->it[qfield(q, s)];
  w.part = ctx->part + (long long)slot * 2 * ctx->maxb;
  w.maxb = ctx->maxb;
  // radial slabs: V, W of quantity q's r-factor (one matrix per step, shared by
  // both systems) are written by the first iteration of the step only
  w.V = ctx->Vq[q]; w.W = ctx->Wq[q]; w.IF = ctx->IFq[q];
  w.vw = ctx->vw_fresh && (q == QT || s == 1);
  return w;
}

int next_order(yy_ctx* ctx) {
  if (!ctx->alt_order) return 0;
  const int r = ctx->rev_next;
  ctx->rev_next ^= 1;
  return r;
}

// O6/O7/O9 for one quantity on every context of the group: residual, the three
// factor sweeps in the printed order (RD28) — the r-factor of radial slabs as the
// partitioned solve across slabs — and the r-halos of the updated iterate
yy_status solve_quantity(std::vector<yy_ctx*>& cs, int q, int s, int slot) {
  const std::string rname = std::string("resid_") + QNAME[q] + (q ? (s == 1 ? "1" : "2") : "");
  for (yy_ctx* ctx : cs) {
    if (ctx->fuse) continue;
    ResidArgs r = resid_args(ctx, q, s);
    r.rev = next_order(ctx);
    ProfScope ps(ctx, rname, 1);
    launch_resid(ctx->g, q, s, r, ctx->st);
  }
  const int S = cs[0]->nslab;
  for (int a = 0; a < 3; ++a) {
    const int ax = ORDER[q][a];
    const bool fin = (a == 2), first = (a == 0) && cs[0]->fuse;
    const std::string cls = std::string("sweep_") + QNAME[q] + "_" + AXNAME[ax] + (fin ? "_fin" : "") +
                            (first ? "+" + rname : "");
    if (ax == 0 && S > 1) {
      const Geo& g = cs[0]->g;
      const int K = kind_of(q), nlines = (NTk(g, K) - 2) * (NPk(g, K) - 2);
      for (yy_ctx* ctx : cs) {
        SweepArgs w = sweep_args(ctx, q, s, slot);
        ProfScope ps(ctx, cls + "_slab", 1);
        const int nb = launch_sweep(ctx->g, q, ax, s, false, false, true, w, nullptr, 1, ctx->st);
        if (nb < 0) return fail(ctx, YY_ESTATE, "radial slab lines must fill the line chunks (nr / nslab)");
      }
      std::vector<Xfer> ops;                      // N2: boundary rows of every slab to its patch group
      for (int p = 0; p < 2; ++p)
        for (int a1 = 0; a1 < S && (cs[0]->mode == 2 || has_patch(cs, p)); ++a1)
          for (int b1 = 0; b1 < S; ++b1)
            ops.push_back({p * S + a1, p * S + b1, [q](yy_ctx* c) -> const double* { return c->IFq[q]; },
                           [=](yy_ctx* c) { return c->IFall + (long long)a1 * nlines * 6; }, 6LL * nlines});
      TRY(run_xfers(cs, ops));
      for (yy_ctx* ctx : cs) {
        SweepArgs w = sweep_args(ctx, q, s, slot);
        SlabArgs sa{ctx->IFall, ctx->LH, S, ctx->slab, nlines};
        ProfScope ps(ctx, cls + "_couple", 2);
        launch_slab_solve(sa, ctx->st);
        const int nb = launch_slab_correct(ctx->g, K, fin, w, ctx->LH, ctx->st);
        if (fin) ctx->nblk[slot] = nb;
      }
      continue;
    }
    for (yy_ctx* ctx : cs) {
      ResidArgs r = resid_args(ctx, q, s);
      SweepArgs w = sweep_args(ctx, q, s, slot);
      w.rev = next_order(ctx);
      ProfScope ps(ctx, cls, 1);
      const int nb = launch_sweep(ctx->g, q, ax, s, first, fin, false, w, first ? &r : nullptr, ctx->g.npatch,
                                  ctx->st);
      if (nb < 0) return fail(ctx, YY_ESTATE, "internal: no sweep kernel for this factor");
      if (fin) ctx->nblk[slot] = nb;
    }
  }
  return exchange_halos(cs, qfield(q, s));
}

// O2-O4 and the walls of one step (per context)
yy_status step_begin(yy_ctx* ctx) {
  const Geo& g = ctx->g;
  const double tau = ctx->dt, t = ctx->t;
  cudaStream_t st = ctx->st;
  const int NPT = g.npatch;
  // wall data at t_{n-1}, t_n, t_{n+1}
  {
    LinBatch b{};
    for (int L = 0; L < 3; ++L) TRY(eval_walls(ctx, L, t + (L - 1) * tau, b));
    ProfScope ps(ctx, "walls", 1);
    launch_lincomb_batch(b, st);
  }
  // O2: a* = 1.5 u2^n - 0.5 u2^{n-1}
  {
    LinBatch b{};
    for (int c = 0; c < 3; ++c) {
      b.out[c] = ctx->astar[c];
      b.p[c][0] = ctx->n[FUR2 + c]; b.c[c][0] = 1.5;
      b.p[c][1] = ctx->m[FUR2 + c]; b.c[c][1] = -0.5;
      b.n[c] = NPT * fsize(ctx, FUR2 + c);
      b.nin[c] = 2;
    }
    b.njobs = 3;
    ProfScope ps(ctx, "astar", 1);
    launch_lincomb_batch(b, st);
  }
  if (!ctx->imex) {   // IMEX: the split rows take no transport terms (Geo::adv -> zero)
    ProfScope ps(ctx, "react", 1);
    launch_react(g, ctx->astar[0], ctx->astar[1], ctx->react_t, ctx->react_p, st);
    launch_adv(g, ctx->astar[0], ctx->astar[1], ctx->astar[2], ctx->adv, NPT, st);
  }
  // O3: static right-hand sides
  for (int q = 0; q < (ctx->heat_only ? 1 : 4); ++q) {
    StaticArgs a = static_args(ctx, q, t + 0.5 * tau);
    ProfScope ps(ctx, std::string("static_") + QNAME[q], 1);
    launch_static(g, q, a, st);
  }
  // O4: psi^(0) = psi^n; u_r walls at t_{n+1}
  // (two batched copy launches: the iterates, then the wall planes they contain)
  {
    LinBatch b{};
    for (int f = 0; f < NF; ++f) {
      b.out[b.njobs] = ctx->it[f];
      b.p[b.njobs][0] = ctx->n[f];
      b.n[b.njobs] = NPT * fsize(ctx, f);
      b.nin[b.njobs++] = -1;
    }
    ProfScope ps(ctx, "copy_iterate", 1);
    launch_lincomb_batch(b, st);
  }
  {
    const long long plane = (long long)g.nt * g.np;
    LinBatch b{};
    for (int f : {FUR1, FUR2})
      for (int p = 0; p < NPT; ++p)
        for (int w = 0; w < 2; ++w)
          if (w ? g.wall_hi : g.wall_lo) {   // wall faces ilo_f - 1 (r = R1), ihi_f + 1 (r = R2)
            b.out[b.njobs] = ctx->it[f] + p * fsize(ctx, f) + (long long)(w ? g.ihi_f + 1 : g.ilo_f - 1) * plane;
            b.p[b.njobs][0] = ctx->wl[2][WUR] + (p * 2 + w) * plane;
            b.n[b.njobs] = plane;
            b.nin[b.njobs++] = -1;
          }
    ProfScope ps(ctx, "copy_iterate", 1);
    launch_lincomb_batch(b, st);
  }
  CK(cudaGetLastError());
  return YY_OK;
}

InterpArgs interp_args(yy_ctx* ctx) {
  InterpArgs ia{};
  ia.cc[0] = ctx->it[FT]; ia.cc[1] = ctx->it[FP1]; ia.cc[2] = ctx->it[FP2];
  ia.cc[3] = ctx->it[FUR1]; ia.cc[4] = ctx->it[FUR2];
  ia.ut[0] = ctx->it[FUT1]; ia.ut[1] = ctx->it[FUT2];
  ia.up[0] = ctx->it[FUP1]; ia.up[1] = ctx->it[FUP2];
  ia.tab_cc = ctx->tcc; ia.tab_th = ctx->tth; ia.tab_ph = ctx->tph;
  ia.dp1 = ctx->dp1; ia.p1n = ctx->n[FP1];
  return ia;
}

// O6-O9 of one Schwarz iteration on every context of the group and each
// context's per-(slot, patch) norm sums
yy_status iter_solve(std::vector<yy_ctx*>& cs) {
  TRY(solve_quantity(cs, QT, 1, 0));                     // O6
  for (yy_ctx* ctx : cs)
    if (ctx->interp_pending) {                           // the p / u fringes (beside the T solve)
      join_interp(ctx->st, ctx->fork);
      ctx->interp_pending = false;
    }
  for (yy_ctx* ctx : cs)
    if (ctx->heat_only)
      for (int q = 1; q < NSLOT; ++q) ctx->nblk[q] = 0;  // no momentum / pressure slots
  for (int s = 1; s <= 2 && !cs[0]->heat_only; ++s) {    // O7 / O9
    const int base = (s == 1) ? 1 : 5;
    TRY(solve_quantity(cs, QUR, s, base + 0));
    TRY(solve_quantity(cs, QUT, s, base + 1));
    TRY(solve_quantity(cs, QUP, s, base + 2));
    for (yy_ctx* ctx : cs) {
      PresArgs pa{};
      const int o = (s == 2) ? 3 : 0;
      pa.urit = ctx->it[FUR1 + o]; pa.urn = ctx->n[FUR1 + o];
      pa.utit = ctx->it[FUT1 + o]; pa.utn = ctx->n[FUT1 + o];
      pa.upit = ctx->it[FUP1 + o]; pa.upn = ctx->n[FUP1 + o];
      pa.pn = ctx->n[s == 1 ? FP1 : FP2];
      pa.p1it = ctx->it[FP1]; pa.p1n = ctx->n[FP1];
      pa.pit = ctx->it[s == 1 ? FP1 : FP2];
      pa.part = ctx->part + (long long)(base + 3) * 2 * ctx->maxb;
      pa.maxb = ctx->maxb;
      pa.dp1 = ctx->dp1;
      pa.rev = next_order(ctx);
      ProfScope ps(ctx, s == 1 ? "pres_1" : "pres_2", 1);
      ctx->nblk[base + 3] = launch_pres(ctx->g, s, pa, ctx->st);
    }
    TRY(exchange_halos(cs, s == 1 ? FP1 : FP2));
  }
  for (yy_ctx* ctx : cs) {
    ReduceArgs ra{};
    for (int q = 0; q < NSLOT; ++q) ra.nblk[q] = ctx->nblk[q];
    ra.maxb = ctx->maxb;
    ra.npatch = ctx->g.npatch;
    ra.patch0 = ctx->patch0;
    ProfScope ps(ctx, "reduce", 1);
    launch_reduce_slots(ctx->part, ra, ctx->red, ctx->st);   // O10, local patches
  }
  return YY_OK;
}

// O5 for target patch p only (multiplicative Schwarz): the other patch's contexts
// evaluate p's fringe from their current iterate, p's contexts write it
yy_status exchange_fringe_to(std::vector<yy_ctx*>& cs, int p) {
  if (cs[0]->schwarz == 2) return YY_OK;                 // single domains: no exchange
  const int S = cs[0]->nslab;
  for (yy_ctx* ctx : cs) {
    if (ctx->patch0 != 1 - p) continue;
    ProfScope ps(ctx, "fringe_pack", 3);
    launch_fringe_pack(ctx->g, interp_args(ctx), ctx->fr_send, ctx->st);
  }
  const long long n = cs[0]->fr_n;
  std::vector<Xfer> ops;
  for (int sl = 0; sl < S; ++sl)
    ops.push_back({(1 - p) * S + sl, p * S + sl, [](yy_ctx* c) -> const double* { return c->fr_send; },
                   [](yy_ctx* c) { return c->fr_recv; }, n});
  TRY(run_xfers(cs, ops));
  for (yy_ctx* ctx : cs) {
    if (ctx->patch0 != p) continue;
    ProfScope ps(ctx, "fringe_unpack", 3);
    launch_fringe_unpack(ctx->g, interp_args(ctx), ctx->fr_recv, ctx->st);
  }
  return YY_OK;
}

// O5 (N3): fringe of every patch from the other patch's iterate k-1
yy_status exchange_fringe(std::vector<yy_ctx*>& cs) {
  // YY_SCHWARZ = 2: every patch a single domain whose fringe keeps its Dirichlet
  // values (Theorem 1's setting)
  if (cs[0]->schwarz == 2) return YY_OK;
  if (!distributed(cs)) {
    yy_ctx* ctx = cs[0];
    // deferred join: not with the flux correction (it reads the u fringes next)
    // or the heat-only step (no momentum solve to overlap); the per-class timing
    // pass (prof_on) keeps the classes apart
    const bool defer = ctx->aux[0] && ctx->defer_interp && !(ctx->flux_eps > 0) && !ctx->heat_only && !ctx->prof_on;
    ProfScope ps(ctx, "interp", defer ? 4 : 3);
    if (ctx->aux[0]) launch_interp(ctx->g, interp_args(ctx), ctx->st, ctx->aux[0], ctx->aux[1], ctx->fork, defer);
    else launch_interp(ctx->g, interp_args(ctx), ctx->st);
    ctx->interp_pending = defer;
    return YY_OK;
  }
  for (yy_ctx* ctx : cs) {                                // donor side: the partner's fringe
    ProfScope ps(ctx, "fringe_pack", 3);
    launch_fringe_pack(ctx->g, interp_args(ctx), ctx->fr_send, ctx->st);
  }
  const int S = cs[0]->nslab;
  const long long n = cs[0]->fr_n;
  std::vector<Xfer> ops;
  for (int r = 0; r < 2 * S; ++r)
    ops.push_back({r, (r + S) % (2 * S), [](yy_ctx* c) -> const double* { return c->fr_send; },
                   [](yy_ctx* c) { return c->fr_recv; }, n});
  TRY(run_xfers(cs, ops));
  for (yy_ctx* ctx : cs) {
    ProfScope ps(ctx, "fringe_unpack", 3);
    launch_fringe_unpack(ctx->g, interp_args(ctx), ctx->fr_recv, ctx->st);
  }
  return YY_OK;
}

// O10 (N4): rho_k from the sums of all patches and slabs, in fixed order, so that
// every context computes the same value and takes the same iteration count
yy_status reduce_group(std::vector<yy_ctx*>& cs) {
  if (distributed(cs)) {
    const int W = world_of(cs[0]);
    const long long m = 2 + 2 * NSLOT;
    std::vector<Xfer> ops;
    for (int a = 0; a < W; ++a)
      for (int b = 0; b < W; ++b)
        ops.push_back({a, b, [](yy_ctx* c) -> const double* { return c->red; },
                       [=](yy_ctx* c) { return c->gath + a * m; }, m});
    TRY(run_xfers(cs, ops));
    for (yy_ctx* ctx : cs) launch_merge_all(ctx->red, ctx->gath, ctx->nslab, ctx->st);
  }
  for (yy_ctx* ctx : cs) {
    ProfScope ps(ctx, "reduce", 1);
    launch_reduce_final(ctx->red, ctx->st);
  }
  return YY_OK;
}

// Algorithm 1 step 4 on every context of the group (after its fringe exchange)
void flux_fix(std::vector<yy_ctx*>& cs, double tol) {
  for (yy_ctx* ctx : cs) {
    if (!(ctx->flux_eps > 0)) continue;
    FluxArgs fa{};
    fa.ur[0] = ctx->it[FUR1]; fa.ur[1] = ctx->it[FUR2];
    fa.ut[0] = ctx->it[FUT1]; fa.ut[1] = ctx->it[FUT2];
    fa.up[0] = ctx->it[FUP1]; fa.up[1] = ctx->it[FUP2];
    fa.a2 = ctx->flux_a2;
    fa.area = ctx->flux_area;
    fa.eps = ctx->flux_eps;
    fa.tol = tol;
    ProfScope ps(ctx, "flux_fix", 1);
    launch_flux_fix(ctx->g, fa, ctx->st);
  }
}

// O11: rotate levels, advance t (per context)
void step_end(yy_ctx* ctx) {
  for (int f = 0; f < NF; ++f) {
    if (f == FP1 || f == FP2) {
      std::swap(ctx->n[f], ctx->it[f]);
    } else {
      double* tmp = ctx->m[f];
      ctx->m[f] = ctx->n[f];
      ctx->n[f] = ctx->it[f];
      ctx->it[f] = tmp;
    }
  }
  ctx->t += ctx->dt;
}

// One time step of a group of contexts that together hold both patches: one
// context (both patches, or one NCCL rank), or a loopback pair.  Every stage
// runs on every context before the next (the exchange needs all donors done).
yy_status step_group(std::vector<yy_ctx*>& cs, double tol, int* iters, double* rho_out) {
  yy_ctx* ctx = cs[0];
  for (yy_ctx* c : cs) TRY(step_begin(c));
  const int kmax = ctx->fixed_iters > 0 ? ctx->fixed_iters : ctx->max_iters;
  int k = 0;
  double rho = INFINITY;
  // One Schwarz iteration is the same launch sequence every time within a step
  // (a*, G and the level pointers are fixed for the step): capture it once per
  // step as a CUDA graph (single context on a user stream, not profiling) and
  // replay it — the ~35 kernels then follow each other without per-launch gaps.
  // graphs: one context (mode 0) or a loopback group on one shared stream
  // (mode 1, additive Schwarz); NCCL ranks (mode 2) launch stream by stream
  // NCCL ranks (mode 2): the iteration with its grouped ncclSend / ncclRecv captured
  // into one graph per iteration kind when YY_DIST_GRAPH=1 (NCCL >= 2.9 supports
  // stream capture of point-to-point calls; off by default: this round's boxes
  // have one GPU, so the captured NCCL path has not run)
  static const bool dist_graph = [] {
    const char* e = std::getenv("YY_DIST_GRAPH");
    return e && e[0] == '1';
  }();
  const bool graph = ctx->use_graph && ctx->st != nullptr && !ctx->prof_on &&
                     ((cs.size() == 1 && ctx->mode == 0) || (ctx->mode == 1 && ctx->schwarz == 0) ||
                      (dist_graph && ctx->mode == 2 && ctx->schwarz == 0));
  cudaGraphExec_t gexec = nullptr;
  std::vector<long long> glaunches(cs.size(), 0);
  if (graph && ctx->use_graph == 2 && cs.size() == 1 && ctx->mode == 0) {
    // the whole loop on the device: a WHILE node whose body is one iteration
    // (O5-O10) followed by k_schwarz_cond; one launch and one host sync per step
    std::vector<const void*> key;
    for (int f = 0; f < NF; ++f) { key.push_back(ctx->it[f]); key.push_back(ctx->n[f]); }
    key.push_back((const void*)(intptr_t)kmax);
    key.push_back((const void*)(intptr_t)(ctx->fixed_iters > 0));
    cudaGraphExec_t ge = nullptr;
    long long per_iter = 0;
    for (auto& lg : ctx->loop_graphs)
      if (lg.key == key && lg.tol == tol && lg.rev_in == ctx->rev_next) {
        ge = lg.exec;
        per_iter = lg.per_iter;
        ctx->rev_next = lg.rev_out;
        break;
      }
    if (!ge) {
    const int rev_in = ctx->rev_next;
    const long long l0 = ctx->launches;
    cudaGraph_t gr = nullptr;
    CK(cudaGraphCreate(&gr, 0));
    cudaGraphConditionalHandle h;
    cudaError_t e = cudaGraphConditionalHandleCreate(&h, gr, 1, cudaGraphCondAssignDefault);
    cudaGraphNodeParams np = {};
    cudaGraphNode_t node;
    if (e == cudaSuccess) {
      np.type = cudaGraphNodeTypeConditional;
      np.conditional.handle = h;
      np.conditional.type = cudaGraphCondTypeWhile;
      np.conditional.size = 1;
      e = cudaGraphAddNode(&node, gr, nullptr, 0, &np);
    }
    if (e == cudaSuccess) e = cudaStreamBeginCaptureToGraph(ctx->st, np.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                                            cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) { cudaGraphDestroy(gr); CK(e); }
    yy_status sc = exchange_fringe(cs);
    if (sc == YY_OK) { flux_fix(cs, tol); sc = iter_solve(cs); }
    if (sc == YY_OK) sc = reduce_group(cs);
    if (sc == YY_OK) {
      launch_schwarz_cond(h, ctx->red, ctx->ctl, tol, kmax, ctx->fixed_iters > 0, ctx->st);
      ctx->launches += 1;
    }
    cudaGraph_t body = nullptr;
    const cudaError_t ec = cudaStreamEndCapture(ctx->st, &body);
    if (sc != YY_OK) { cudaGraphDestroy(gr); return sc; }
    if (ec != cudaSuccess) { cudaGraphDestroy(gr); CK(ec); }
    per_iter = ctx->launches - l0;   // (incl. k_schwarz_cond)
    ctx->launches = l0;
    const cudaError_t ei = cudaGraphInstantiate(&ge, gr, 0);
    cudaGraphDestroy(gr);
    CK(ei);
    if (ctx->loop_graphs.size() >= 16) clear_loop_graphs(ctx);
    ctx->loop_graphs.push_back({key, tol, rev_in, ctx->rev_next, per_iter, ge});
    }
    CK(cudaMemsetAsync(ctx->ctl, 0, 3 * sizeof(double), ctx->st));
    CK(cudaGraphLaunch(ge, ctx->st));
    CK(cudaMemcpyAsync(ctx->red_host, ctx->ctl, 3 * sizeof(double), cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    k = (int)ctx->red_host[0];
    rho = ctx->red_host[1];
    ctx->launches += per_iter * k;
    if (ctx->red_host[2] != 0.0) {
      fail(ctx, YY_ESOLVER, "NaN/Inf in the Schwarz residual");
      return YY_ESOLVER;
    }
    step_end(ctx);
    *iters = k;
    *rho_out = rho;
    return YY_OK;
  }
  // radial slabs: the step's first iteration also computes the slab coupling
  // responses V / W; later ones solve for x0 alone — two graphs
  cudaGraphExec_t gexec2 = nullptr;
  const bool two = graph && cs[0]->nslab > 1;
  auto capture = [&](bool fresh, cudaGraphExec_t* out) -> yy_status {
    cudaGraph_t gr = nullptr;
    std::vector<long long> l0(cs.size());
    for (size_t q = 0; q < cs.size(); ++q) {
      l0[q] = cs[q]->launches;
      cs[q]->vw_fresh = fresh;
    }
    CK(cudaStreamBeginCapture(ctx->st, cudaStreamCaptureModeThreadLocal));
    yy_status sc = exchange_fringe(cs);
    if (sc == YY_OK) { flux_fix(cs, tol); sc = iter_solve(cs); }
    if (sc == YY_OK) sc = reduce_group(cs);
    if (sc == YY_OK)
      sc = cudaMemcpyAsync(ctx->red_host, ctx->red, 2 * sizeof(double), cudaMemcpyDeviceToHost, ctx->st) == cudaSuccess
               ? YY_OK : YY_ECUDA;
    const cudaError_t ec = cudaStreamEndCapture(ctx->st, &gr);
    if (sc != YY_OK) return sc;
    CK(ec);
    const cudaError_t ei = cudaGraphInstantiate(out, gr, 0);
    cudaGraphDestroy(gr);
    CK(ei);
    for (size_t q = 0; q < cs.size(); ++q) {
      glaunches[q] = cs[q]->launches - l0[q];
      cs[q]->launches = l0[q];
    }
    return YY_OK;
  };
  if (graph) {
    TRY(capture(true, &gexec));
    if (two) {
      const yy_status s2 = capture(false, &gexec2);
      if (s2 != YY_OK) { cudaGraphExecDestroy(gexec); return s2; }
    }
  }
  while (k < kmax) {
    ++k;
    if (!graph)
      for (yy_ctx* c : cs) c->vw_fresh = (k == 1);   // slab V / W: once per step (the step's matrices)
    if (graph) {
      const cudaError_t el = cudaGraphLaunch((k == 1 || !two) ? gexec : gexec2, ctx->st);
      if (el != cudaSuccess) {
        cudaGraphExecDestroy(gexec);
        if (gexec2) cudaGraphExecDestroy(gexec2);
        CK(el);
      }
      for (size_t q = 0; q < cs.size(); ++q) cs[q]->launches += glaunches[q];
    } else if (ctx->schwarz == 1) {                        // multiplicative: Yin, then Yang with Yin's k
      for (int p = 0; p < 2; ++p) {
        TRY(exchange_fringe_to(cs, p));                    // O5 for patch p
        std::vector<yy_ctx*> cp = of_patch(cs, p);
        flux_fix(cp, tol);                                 // Alg. 1 step 4 (optional)
        if (!cp.empty()) TRY(iter_solve(cp));              // O6-O9 on patch p
      }
    } else {
      TRY(exchange_fringe(cs));                            // O5
      flux_fix(cs, tol);                                   // Alg. 1 step 4 (optional)
      TRY(iter_solve(cs));                                 // O6-O9, local norms
    }
    if (!graph) {
      TRY(reduce_group(cs));                               // O10
      for (yy_ctx* c : cs) {
        yy_ctx* ctx = c;
        CK(cudaGetLastError());
      }
      CK(cudaMemcpyAsync(ctx->red_host, ctx->red, 2 * sizeof(double), cudaMemcpyDeviceToHost, ctx->st));
    }
    for (yy_ctx* c : cs) {
      yy_ctx* ctx = c;
      CK(cudaStreamSynchronize(c->st));
      if (c->prof_on) prof_collect(c);
    }
    rho = ctx->red_host[0];
    if (ctx->red_host[1] != 0.0) {
      if (gexec) cudaGraphExecDestroy(gexec);
      if (gexec2) cudaGraphExecDestroy(gexec2);
      for (yy_ctx* c : cs) fail(c, YY_ESOLVER, "NaN/Inf in the Schwarz residual");
      return YY_ESOLVER;
    }
    if (ctx->fixed_iters <= 0 && rho < tol) break;
  }
  if (gexec) cudaGraphExecDestroy(gexec);
  if (gexec2) cudaGraphExecDestroy(gexec2);
  for (yy_ctx* c : cs) step_end(c);
  *iters = k;
  *rho_out = rho;
  return YY_OK;
}

}  // namespace

// =====================================================================================
// C ABI
// =====================================================================================
namespace {
// npatch local patches starting at global patch0; nslab > 1: radial slab `slab`
// of nslab equal slabs (nr / nslab rows, plus one halo row on each side)
// process-wide allocator for contexts created from now on (yy_set_allocator(NULL, ...))
struct AllocHook {
  void* (*alloc)(size_t, void*) = nullptr;
  void (*free_)(void*, void*) = nullptr;
  void* user = nullptr;
} g_alloc;

yy_status create_ctx(const yy_grid* gr, double R1, double R2, double Pr, double Ra, double dt, int npatch,
                     int patch0, yy_ctx** out, int nslab = 1, int slab = 0) {
  if (!out) return YY_EINVAL;
  *out = nullptr;
  if (nslab < 1 || slab < 0 || slab >= nslab || (nslab > 1 && (npatch != 1 || !gr || gr->nr % nslab ||
                                                               gr->nr / nslab < 4)))
    return YY_EINVAL;
  if (!gr || gr->nr < 2 || gr->ntheta < 8 || gr->nphi < 8) return YY_EINVAL;
  // longest lines the register-chunked line solver takes (yy_line.cu)
  if (gr->nr > max_line_len(0) || gr->ntheta - 1 > max_line_len(1) || gr->nphi - 1 > max_line_len(2)) return YY_EINVAL;
  // per-patch offsets are 32-bit in the kernels
  if ((double)(gr->nr + 1) * (gr->ntheta + 1) * (gr->nphi + 1) >= 2147483647.0) return YY_EINVAL;
  if (!(R1 > 0 && R2 > R1) || !(dt > 0) || !(Pr > 0) || !std::isfinite(Ra)) return YY_EINVAL;
  yy_ctx* ctx = new yy_ctx();
  ctx->alloc_fn = g_alloc.alloc;
  ctx->free_fn = g_alloc.free_;
  ctx->alloc_user = g_alloc.user;
  if (const char* e = std::getenv("YY_FUSE")) ctx->fuse = (e[0] && e[0] != '0');
  if (const char* e = std::getenv("YY_ALT_ORDER")) ctx->alt_order = !(e[0] == '0');
  if (const char* e = std::getenv("YY_GRAPH")) ctx->use_graph = (e[0] >= '0' && e[0] <= '2') ? e[0] - '0' : 2;
  ctx->R1 = R1; ctx->R2 = R2; ctx->Pr = Pr; ctx->Ra = Ra; ctx->dt = dt;
  HostGeo h = host_geo(gr, R1, R2);
  Geo& g = ctx->g;
  g.nr = h.nr; g.nt = h.nt; g.np = h.np;
  g.npatch = npatch;
  ctx->patch0 = patch0;
  ctx->nslab = nslab;
  ctx->slab = slab;
  ctx->nr_glob = h.nr;
  g.ilo_c = 0; g.ihi_c = h.nr - 1; g.ilo_f = 1; g.ihi_f = h.nr - 1;
  g.wall_lo = g.wall_hi = 1;
  g.ifr_c0 = 0; g.ifr_c1 = h.nr - 1; g.ifr_f0 = 1; g.ifr_f1 = h.nr - 1;
  if (nslab > 1) {
    // local row i = global row i + roff, roff = slab nl - 1: rows 1..nl owned,
    // rows 0 and nl+1 halos; local face f = global face f + roff
    const int nl = h.nr / nslab;
    ctx->roff = slab * nl - 1;
    g.nr = nl + 2;
    g.wall_lo = slab == 0;
    g.wall_hi = slab == nslab - 1;
    g.ilo_c = 1; g.ihi_c = nl;
    g.ilo_f = 2; g.ihi_f = g.wall_hi ? nl : nl + 1;
    g.ifr_c0 = 0; g.ifr_c1 = nl + 1;
    g.ifr_f0 = g.wall_lo ? 2 : 1; g.ifr_f1 = g.wall_hi ? nl : nl + 2;
  }
  g.dr = h.dr; g.dth = h.dth; g.dph = h.dph; g.R1 = R1;
  g.tau = dt; g.nu = Pr; g.kap = 1.0;
  g.cchi = 1.0 / (2.0 * ctx->chi); g.inv_chi = 1.0 / ctx->chi; g.PrRa = Pr * Ra;
  const double th1 = M_PI / 4 - 2.0 * h.dth;   // RD31
  g.hatph = 1.0 / (R1 * R1 * std::sin(th1) * std::sin(th1) * h.dph * h.dph);
  // 1-D coordinate and factor tables (SURVEY Appendix A rows as products of
  // 1-D factors; computed once here in fp64, so no kernel divides)
  const int nr = g.nr, nt = h.nt;   // local rows (a slab's include its halos)
  const double dr = h.dr, dth = h.dth;
  std::vector<double> rc(nr), rf(nr + 1), sc(nt), sf(nt + 1), cc(nt), cf(nt + 1);
  for (int i = 0; i < nr; ++i) rc[i] = R1 + (i + ctx->roff + 0.5) * dr;
  for (int i = 0; i <= nr; ++i) rf[i] = R1 + (i + ctx->roff) * dr;
  for (int j = 0; j < nt; ++j) { sc[j] = std::sin(h.th0 + (j + 0.5) * dth); cc[j] = std::cos(h.th0 + (j + 0.5) * dth); }
  for (int j = 0; j <= nt; ++j) { sf[j] = std::sin(h.th0 + j * dth); cf[j] = std::cos(h.th0 + j * dth); }
  std::vector<double> tab;
  std::vector<std::pair<const double**, size_t>> slots;   // (Geo member, offset)
  auto put = [&](const double** member, const std::vector<double>& v) {
    slots.push_back({member, tab.size()});
    tab.insert(tab.end(), v.begin(), v.end());
  };
  auto vec = [](int n, auto f) { std::vector<double> v(n); for (int q = 0; q < n; ++q) v[q] = f(q); return v; };
  const double dr2 = dr * dr, dt2 = dth * dth;
  put(&g.rc, rc); put(&g.rf, rf); put(&g.sc, sc); put(&g.sf, sf); put(&g.cc, cc); put(&g.cf, cf);
  {   // Algorithm 1 step 4 constants of one patch (theta sides, phi sides, walls; reading RD-E5)
    double a2 = 0.0, area = 0.0;
    for (int i = 0; i < nr; ++i) {
      for (int side = 0; side < 2; ++side) {
        const double at = rc[i] * sf[side ? nt : 0] * dr * h.dph, ap = rc[i] * dr * dth;
        a2 += h.np * at * at + nt * ap * ap;
        area += h.np * at + nt * ap;
      }
    }
    for (int j = 0; j < nt; ++j) area += (rf[0] * rf[0] + rf[nr] * rf[nr]) * sc[j] * dth * h.dph * h.np;
    ctx->flux_a2 = a2;
    ctx->flux_area = area;
  }
  // r at centres
  put(&g.ir_c, vec(nr, [&](int i) { return 1.0 / rc[i]; }));
  put(&g.ir2_c, vec(nr, [&](int i) { return 1.0 / (rc[i] * rc[i]); }));
  put(&g.lr_cm, vec(nr, [&](int i) { return rf[i] * rf[i] / (rc[i] * rc[i] * dr2); }));
  put(&g.lr_cp, vec(nr, [&](int i) { return rf[i + 1] * rf[i + 1] / (rc[i] * rc[i] * dr2); }));
  put(&g.idv1_c, vec(nr, [&](int i) { return 1.0 / (rc[i] * rc[i] * dr); }));
  // r on faces (entries at the walls i = 0, nr are never used by solved rows)
  auto rcs = [&](int i) { return rc[std::min(std::max(i, 0), nr - 1)]; };
  auto rfs = [&](int i) { return rf[std::min(std::max(i, 0), nr)]; };
  put(&g.ir_f, vec(nr + 1, [&](int i) { return 1.0 / rf[i]; }));
  put(&g.ir2_f, vec(nr + 1, [&](int i) { return 1.0 / (rf[i] * rf[i]); }));
  put(&g.lr_fm, vec(nr + 1, [&](int i) { return rcs(i - 1) * rcs(i - 1) / (rf[i] * rf[i] * dr2); }));
  put(&g.lr_fp, vec(nr + 1, [&](int i) { return rcs(i) * rcs(i) / (rf[i] * rf[i] * dr2); }));
  put(&g.mr_m, vec(nr + 1, [&](int i) { return rfs(i - 1) * rfs(i - 1) / (rf[i] * rf[i] * rf[i] * dr); }));
  put(&g.mr_p, vec(nr + 1, [&](int i) { return rfs(i + 1) * rfs(i + 1) / (rf[i] * rf[i] * rf[i] * dr); }));
  put(&g.d11_m, vec(nr + 1, [&](int i) { return rfs(i - 1) * rfs(i - 1) / (rcs(i - 1) * rcs(i - 1) * dr2); }));
  put(&g.d11_p, vec(nr + 1, [&](int i) { return rfs(i + 1) * rfs(i + 1) / (rcs(i) * rcs(i) * dr2); }));
  put(&g.d11_0, vec(nr + 1, [&](int i) {
    return rf[i] * rf[i] * (1.0 / (rcs(i) * rcs(i)) + 1.0 / (rcs(i - 1) * rcs(i - 1))) / dr2; }));
  put(&g.rf2, vec(nr + 1, [&](int i) { return rf[i] * rf[i]; }));
  // theta at centres
  put(&g.is_c, vec(nt, [&](int j) { return 1.0 / sc[j]; }));
  put(&g.is2_c, vec(nt, [&](int j) { return 1.0 / (sc[j] * sc[j]); }));
  put(&g.cot_c, vec(nt, [&](int j) { return cc[j] / sc[j]; }));
  put(&g.lt_cm, vec(nt, [&](int j) { return sf[j] / (sc[j] * dt2); }));
  put(&g.lt_cp, vec(nt, [&](int j) { return sf[j + 1] / (sc[j] * dt2); }));
  // theta on faces (entries j = 0, nt unused by solved rows)
  auto scs = [&](int j) { return sc[std::min(std::max(j, 0), nt - 1)]; };
  auto sfs = [&](int j) { return sf[std::min(std::max(j, 0), nt)]; };
  put(&g.is_f, vec(nt + 1, [&](int j) { return 1.0 / sf[j]; }));
  put(&g.is2_f, vec(nt + 1, [&](int j) { return 1.0 / (sf[j] * sf[j]); }));
  put(&g.cot_f, vec(nt + 1, [&](int j) { return cf[j] / sf[j]; }));
  put(&g.lt_fm, vec(nt + 1, [&](int j) { return scs(j - 1) / (sf[j] * dt2); }));
  put(&g.lt_fp, vec(nt + 1, [&](int j) { return scs(j) / (sf[j] * dt2); }));
  put(&g.mt_m, vec(nt + 1, [&](int j) { return cf[j] * sfs(j - 1) / (sf[j] * sf[j] * dth); }));
  put(&g.mt_p, vec(nt + 1, [&](int j) { return cf[j] * sfs(j + 1) / (sf[j] * sf[j] * dth); }));
  put(&g.d22_m, vec(nt + 1, [&](int j) { return sfs(j - 1) / (scs(j - 1) * dt2); }));
  put(&g.d22_p, vec(nt + 1, [&](int j) { return sfs(j + 1) / (scs(j) * dt2); }));
  put(&g.d22_0, vec(nt + 1, [&](int j) { return sf[j] * (1.0 / scs(j) + 1.0 / scs(j - 1)) / dt2; }));
  g.idr = 1.0 / dr; g.idth = 1.0 / dth; g.idph = 1.0 / h.dph; g.idph2 = g.idph * g.idph;
  g.iR1sq = 1.0 / (R1 * R1);
  yy_status s;
  const double* dtab = nullptr;
  if ((s = upload(ctx, tab, &dtab)) != YY_OK) { yy_destroy(ctx); return s; }
  for (auto& sl : slots) *sl.first = dtab + sl.second;
  if ((s = build_tables(ctx, h)) != YY_OK) { std::fprintf(stderr, "yy_create: %s\n", ctx->err.c_str()); yy_destroy(ctx); return s; }
  // fields
  long long maxk = 0;
  for (int K = 0; K < 4; ++K) maxk = std::max(maxk, psize(g, K));
  for (int f = 0; f < NF; ++f) {
    const size_t sz = (size_t)npatch * psize(g, FKIND[f]);
    if ((s = dalloc(ctx, &ctx->n[f], sz)) != YY_OK || (s = dalloc(ctx, &ctx->it[f], sz)) != YY_OK) { yy_destroy(ctx); return s; }
    if (f != FP1 && f != FP2) {
      if ((s = dalloc(ctx, &ctx->m[f], sz)) != YY_OK || (s = dalloc(ctx, &ctx->G[f], sz)) != YY_OK) { yy_destroy(ctx); return s; }
    }
    cudaMemset(ctx->n[f], 0, sz * sizeof(double));
    cudaMemset(ctx->it[f], 0, sz * sizeof(double));
    if (ctx->m[f]) cudaMemset(ctx->m[f], 0, sz * sizeof(double));
    if (ctx->G[f]) cudaMemset(ctx->G[f], 0, sz * sizeof(double));
  }
  for (int c = 0; c < 3; ++c)
    if ((s = dalloc(ctx, &ctx->astar[c], npatch * psize(g, KR + c))) != YY_OK) { yy_destroy(ctx); return s; }
  if ((s = dalloc(ctx, &ctx->react_t, npatch * psize(g, KT))) != YY_OK ||
      (s = dalloc(ctx, &ctx->react_p, npatch * psize(g, KP))) != YY_OK) { yy_destroy(ctx); return s; }
  cudaMemset(ctx->react_t, 0, npatch * psize(g, KT) * sizeof(double));
  cudaMemset(ctx->react_p, 0, npatch * psize(g, KP) * sizeof(double));
  if ((s = dalloc(ctx, &ctx->R, npatch * maxk)) != YY_OK) { yy_destroy(ctx); return s; }
  cudaMemset(ctx->R, 0, npatch * maxk * sizeof(double));
  // norm partials: max blocks per (slot, patch)
  long long mb = 0;
  for (int K = 0; K < 4; ++K) {
    mb = std::max(mb, (long long)((NPk(g, K) + 127) / 128) * NTk(g, K) * NRk(g, K));
    mb = std::max(mb, (long long)((NTk(g, K) + 127) / 128) * NRk(g, K));
    mb = std::max(mb, (long long)((NPk(g, K) + 3) / 4) * std::max(NTk(g, K), NRk(g, K)));   // r/theta line tiles
    mb = std::max(mb, (long long)NRk(g, K) * NTk(g, K));                                     // phi line tiles
  }
  ctx->maxb = (int)mb;
  if ((s = dalloc(ctx, &ctx->part, (size_t)NSLOT * 2 * mb)) != YY_OK || (s = dalloc(ctx, &ctx->red, 2 + 2 * NSLOT)) != YY_OK) { yy_destroy(ctx); return s; }
  cudaMemset(ctx->part, 0, (size_t)NSLOT * 2 * mb * sizeof(double));
  if (cudaMallocHost(&ctx->red_host, 64 * sizeof(double)) != cudaSuccess) { yy_destroy(ctx); return YY_ENOMEM; }
  if ((s = dalloc(ctx, &ctx->ctl, 4)) != YY_OK) { yy_destroy(ctx); return s; }
  // both patches in this context (the interpolation kernels write every fringe):
  // system 2 reads p1^(k) - p1^n from one array (YY_DP1=0: off)
  const char* epi = std::getenv("YY_PAR_INTERP");
  const char* edi = std::getenv("YY_DEFER_INTERP");
  ctx->defer_interp = edi && edi[0] == '1';
  if (npatch == 2 && nslab == 1 && !(epi && epi[0] == '0')) {
    for (int q = 0; q < 2; ++q)
      if (cudaStreamCreateWithFlags(&ctx->aux[q], cudaStreamNonBlocking) != cudaSuccess) { yy_destroy(ctx); return YY_ECUDA; }
    for (int q = 0; q < 3; ++q)
      if (cudaEventCreateWithFlags(&ctx->fork[q], cudaEventDisableTiming) != cudaSuccess) { yy_destroy(ctx); return YY_ECUDA; }
  }
  const char* edp = std::getenv("YY_DP1");
  if (npatch == 2 && nslab == 1 && !(edp && edp[0] == '0')) {
    if ((s = dalloc(ctx, &ctx->dp1, npatch * psize(g, KC))) != YY_OK) { yy_destroy(ctx); return s; }
    cudaMemset(ctx->dp1, 0, npatch * psize(g, KC) * sizeof(double));
  }
  for (int L = 0; L < 3; ++L)
    for (int f = 0; f < NW; ++f)
      if ((s = dalloc(ctx, &ctx->wl[L][f], 2 * npatch * wsize(g, WKIND[f]))) != YY_OK) { yy_destroy(ctx); return s; }
  if (npatch == 1) {   // transfer buffers of a one-patch context
    InterpArgs ia{};
    ia.tab_cc = ctx->tcc; ia.tab_th = ctx->tth; ia.tab_ph = ctx->tph;
    ctx->fr_n = fringe_count(g, ia);
    if ((s = dalloc(ctx, &ctx->fr_send, ctx->fr_n)) != YY_OK || (s = dalloc(ctx, &ctx->fr_recv, ctx->fr_n)) != YY_OK ||
        (s = dalloc(ctx, &ctx->gath, (size_t)2 * nslab * (2 + 2 * NSLOT))) != YY_OK) { yy_destroy(ctx); return s; }
  }
  if (nslab > 1) {     // partitioned r-sweep buffers
    long long nlmax = 0;
    for (int K = 0; K < 4; ++K) nlmax = std::max(nlmax, (long long)(NTk(g, K) - 2) * (NPk(g, K) - 2));
    for (int q = 0; q < 4; ++q)
      if ((s = dalloc(ctx, &ctx->Vq[q], psize(g, q))) != YY_OK || (s = dalloc(ctx, &ctx->Wq[q], psize(g, q))) != YY_OK) {
        yy_destroy(ctx);
        return s;
      }
    if (
        (s = dalloc(ctx, &ctx->IFq[0], 6 * nlmax)) != YY_OK || (s = dalloc(ctx, &ctx->IFq[1], 6 * nlmax)) != YY_OK ||
        (s = dalloc(ctx, &ctx->IFq[2], 6 * nlmax)) != YY_OK || (s = dalloc(ctx, &ctx->IFq[3], 6 * nlmax)) != YY_OK ||
        (s = dalloc(ctx, &ctx->IFall, 6 * nslab * nlmax)) != YY_OK ||
        (s = dalloc(ctx, &ctx->LH, 2 * nlmax)) != YY_OK) { yy_destroy(ctx); return s; }
  }
  ctx->rank = patch0 * nslab + slab;
  for (int q = 0; q < 4; ++q)
    for (int ax = 0; ax < 3; ++ax) {
      if ((s = dalloc(ctx, &ctx->bsplit[q][ax], (size_t)3 * NRk(g, q) * NTk(g, q))) != YY_OK ||
          (s = dalloc(ctx, &ctx->tsplit[q][ax], (size_t)3 * NRk(g, q) * NTk(g, q))) != YY_OK) { yy_destroy(ctx); return s; }
      g.bsplit[q][ax] = ctx->bsplit[q][ax];
      g.tsplit[q][ax] = ctx->tsplit[q][ax];
    }
  launch_build_split(g, ctx->bsplit, ctx->tsplit, ctx->st);
  for (int K = 0; K < 4; ++K)
    for (int ax = 0; ax < 3; ++ax) {
      if ((s = dalloc(ctx, &ctx->adv[K][ax], npatch * psize(g, K))) != YY_OK) { yy_destroy(ctx); return s; }
      cudaMemset(ctx->adv[K][ax], 0, npatch * psize(g, K) * sizeof(double));
      g.adv[K][ax] = ctx->adv[K][ax];
    }
  if (cudaDeviceSynchronize() != cudaSuccess) { yy_destroy(ctx); return YY_ECUDA; }
  *out = ctx;
  return YY_OK;
}
}  // namespace

extern "C" {

yy_status yy_create(const yy_grid* gr, double R1, double R2, double Pr, double Ra, double dt, yy_ctx** out) {
  return create_ctx(gr, R1, R2, Pr, Ra, dt, 2, 0, out);
}

yy_status yy_nccl_unique_id(void* out128) {
  if (!out128) return YY_EINVAL;
  NcclApi& N = nccl_api();
  if (!N.ok) return YY_ENCCL;
  ncclUniqueId id;
  if (N.GetUniqueId(&id) != ncclSuccess) return YY_ENCCL;
  static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(out128, &id, sizeof(id));
  return YY_OK;
}

yy_status yy_create_dist(const yy_grid* gr, double R1, double R2, double Pr, double Ra, double dt, int32_t world,
                         int32_t rank, const void* nccl_id, int32_t device, yy_ctx** out) {
  if (!out) return YY_EINVAL;
  *out = nullptr;
  if (world == 1 && rank == 0) {
    if (cudaSetDevice(device) != cudaSuccess) return YY_ECUDA;
    return yy_create(gr, R1, R2, Pr, Ra, dt, out);
  }
  // world = 2 nslab: rank = patch nslab + slab (Yin on ranks 0..nslab-1, Yang on the rest)
  if (world < 2 || world % 2 || world > 16 || rank < 0 || rank >= world || !nccl_id) return YY_EINVAL;
  const int nslab = world / 2;
  NcclApi& N = nccl_api();
  if (!N.ok) return YY_ENCCL;
  if (cudaSetDevice(device) != cudaSuccess) return YY_ECUDA;
  yy_ctx* ctx = nullptr;
  yy_status s = create_ctx(gr, R1, R2, Pr, Ra, dt, 1, rank / nslab, &ctx, nslab, rank % nslab);
  if (s != YY_OK) return s;
  ncclUniqueId id;
  std::memcpy(&id, nccl_id, sizeof(id));
  ncclComm_t comm = nullptr;
  if (N.CommInitRank(&comm, world, id, rank) != ncclSuccess) {
    yy_destroy(ctx);
    return YY_ENCCL;
  }
  ctx->nccl = comm;
  ctx->mode = 2;
  ctx->world = world;
  ctx->rank = rank;
  *out = ctx;
  return YY_OK;
}

yy_status yy_create_pair(const yy_grid* gr, double R1, double R2, double Pr, double Ra, double dt, yy_ctx** out2) {
  if (!out2) return YY_EINVAL;
  out2[0] = out2[1] = nullptr;
  yy_status s = create_ctx(gr, R1, R2, Pr, Ra, dt, 1, 0, &out2[0]);
  if (s != YY_OK) return s;
  s = create_ctx(gr, R1, R2, Pr, Ra, dt, 1, 1, &out2[1]);
  if (s != YY_OK) { yy_destroy(out2[0]); out2[0] = nullptr; return s; }
  out2[0]->mode = out2[1]->mode = 1;
  out2[0]->group = out2[1]->group = {out2[0], out2[1]};
  out2[1]->st = out2[0]->st;
  return YY_OK;
}

yy_status yy_create_slabs(const yy_grid* gr, double R1, double R2, double Pr, double Ra, double dt, int32_t nslab,
                          yy_ctx** out) {
  if (!out || nslab < 1 || nslab > 8) return YY_EINVAL;
  std::vector<yy_ctx*> cs(2 * nslab, nullptr);
  for (int r = 0; r < 2 * nslab; ++r) {
    out[r] = nullptr;
    yy_status s = create_ctx(gr, R1, R2, Pr, Ra, dt, 1, r / nslab, &cs[r], nslab, r % nslab);
    if (s != YY_OK) {
      for (yy_ctx* c : cs) if (c) { c->group.clear(); yy_destroy(c); }
      return s;
    }
  }
  for (int r = 0; r < 2 * nslab; ++r) {
    cs[r]->mode = 1;
    cs[r]->group = cs;
    cs[r]->st = cs[0]->st;
    out[r] = cs[r];
  }
  return YY_OK;
}

yy_status yy_set_fields(yy_ctx* ctx, int32_t patch, int32_t level, int32_t system, const yy_fields* f) {
  TRY(check_args(ctx, patch, level, system));
  if (!f) return fail(ctx, YY_EINVAL, "NULL fields");
  const int sys_lo = system == 0 ? 1 : system, sys_hi = system == 0 ? 2 : system;
  double** L = level == 0 ? ctx->n : ctx->m;
  auto put = [&](int fidx, const double* src) -> yy_status {
    if (!src) return YY_OK;
    const long long sz = fsize(ctx, fidx);
    return copy_window(ctx, FKIND[fidx], L[fidx] + (patch - ctx->patch0) * sz, const_cast<double*>(src), true, false);
  };
  for (int s = sys_lo; s <= sys_hi; ++s) {
    const int o = (s == 2) ? 3 : 0;
    if (s == 2 && system == 0) {
      // both systems from one host copy: system 2's arrays are device copies of
      // system 1's (the same patch window)
      auto dup = [&](int f1, int f2, const double* src) -> yy_status {
        if (!src) return YY_OK;
        const long long sz = fsize(ctx, f1);
        CK(cudaMemcpyAsync(L[f2] + (patch - ctx->patch0) * sz, L[f1] + (patch - ctx->patch0) * sz,
                           sz * sizeof(double), cudaMemcpyDeviceToDevice, ctx->st));
        return YY_OK;
      };
      TRY(dup(FUR1, FUR2, f->ur));
      TRY(dup(FUT1, FUT2, f->ut));
      TRY(dup(FUP1, FUP2, f->up));
      if (level == 0) TRY(dup(FP1, FP2, f->p));
      CK(cudaStreamSynchronize(ctx->st));
      continue;
    }
    TRY(put(FUR1 + o, f->ur));
    TRY(put(FUT1 + o, f->ut));
    TRY(put(FUP1 + o, f->up));
    if (level == 0) TRY(put(s == 1 ? FP1 : FP2, f->p));
  }
  TRY(put(FT, f->T));
  return YY_OK;
}

yy_status yy_get_fields(yy_ctx* ctx, int32_t patch, int32_t level, int32_t system, yy_fields* f) {
  TRY(check_args(ctx, patch, level, system));
  if (!f || system == 0) return fail(ctx, YY_EINVAL, "get_fields needs system 1 or 2");
  double** L = level == 0 ? ctx->n : ctx->m;
  auto get = [&](int fidx, double* dst) -> yy_status {
    if (!dst) return YY_OK;
    const long long sz = fsize(ctx, fidx);
    return copy_window(ctx, FKIND[fidx], L[fidx] + (patch - ctx->patch0) * sz, dst, false, true);
  };
  const int o = (system == 2) ? 3 : 0;
  TRY(get(FUR1 + o, f->ur));
  TRY(get(FUT1 + o, f->ut));
  TRY(get(FUP1 + o, f->up));
  if (level == 0) TRY(get(system == 1 ? FP1 : FP2, f->p));
  TRY(get(FT, f->T));
  return YY_OK;
}

static yy_status set_terms(yy_ctx* ctx, int32_t patch, int32_t nterms, const int32_t* timefn,
                           const yy_fields* terms, bool wall) {
  if (!ctx) return YY_EINVAL;
  if (ctx->dead) return fail(ctx, YY_ESTATE, "context unusable after a CUDA error");
  if (patch < 0 || patch > 1 || nterms < 0 || nterms > MAXSRC || (nterms > 0 && (!timefn || !terms)))
    return fail(ctx, YY_EINVAL, "bad wall/source terms");
  if (patch < ctx->patch0 || patch >= ctx->patch0 + ctx->g.npatch)
    return fail(ctx, YY_EINVAL, "this context does not hold that patch");
  patch -= ctx->patch0;   // local index
  const Geo& g = ctx->g;
  for (int m = 0; m < nterms; ++m)
    if (timefn[m] < YY_TF_ONE || timefn[m] > YY_TF_COS2) return fail(ctx, YY_EINVAL, "bad time function");
  for (int m = 0; m < nterms; ++m) {
    const double* src[4] = {terms[m].T, terms[m].ur, terms[m].ut, terms[m].up};
    for (int f = 0; f < 4; ++f) {
      double*& slot = wall ? ctx->wterm[patch][m][f] : ctx->sterm[patch][m][f];
      if (!src[f]) { slot = nullptr; continue; }
      const long long sz = wall ? 2 * wsize(g, WKIND[f]) : psize(g, WKIND[f]);
      // a slot's size depends only on (wall|source, field): re-setting terms reuses
      // the buffer allocated by the first call instead of allocating again
      double*& keep = wall ? ctx->wterm_buf[patch][m][f] : ctx->sterm_buf[patch][m][f];
      if (!keep) TRY(dalloc(ctx, &keep, sz));
      double* d = keep;
      CK(cudaMemsetAsync(d, 0, sz * sizeof(double), ctx->st));
      if (wall) {
        CK(cudaMemcpyAsync(d, src[f], sz * sizeof(double), cudaMemcpyHostToDevice, ctx->st));
        CK(cudaStreamSynchronize(ctx->st));
      }
      else TRY(copy_window(ctx, WKIND[f], d, const_cast<double*>(src[f]), true, false));
      slot = d;
    }
    (wall ? ctx->wtf : ctx->stf)[patch][m] = timefn[m];
  }
  (wall ? ctx->nw : ctx->ns)[patch] = nterms;
  return YY_OK;
}

yy_status yy_set_wall(yy_ctx* ctx, int32_t patch, int32_t nterms, const int32_t* timefn, const yy_fields* terms) {
  return set_terms(ctx, patch, nterms, timefn, terms, true);
}

yy_status yy_set_source(yy_ctx* ctx, int32_t patch, int32_t nterms, const int32_t* timefn, const yy_fields* terms) {
  return set_terms(ctx, patch, nterms, timefn, terms, false);
}

yy_status yy_energy(yy_ctx* ctx, double* out3) {
  if (!ctx || !out3) return YY_EINVAL;
  if (ctx->dead) return fail(ctx, YY_ESTATE, "context unusable after a CUDA error");
  if (ctx->nslab > 1) return fail(ctx, YY_EINVAL, "yy_energy needs whole patches (no radial slabs)");
  const Geo& g = ctx->g;
  const long long zw = 2 * wsize(g, KC) * g.npatch, nb = energy_blocks(g);
  if (!ctx->energy_buf) {
    TRY(dalloc(ctx, &ctx->energy_buf, zw + 3 * nb + 3));
    CK(cudaMemsetAsync(ctx->energy_buf, 0, zw * sizeof(double), ctx->st));
  }
  launch_energy(g, ctx->n[FT], ctx->m[FT], ctx->energy_buf, ctx->energy_buf + zw, ctx->energy_buf + zw + 3 * nb,
                ctx->st);
  ctx->launches += 2;
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out3, ctx->energy_buf + zw + 3 * nb, 3 * sizeof(double), cudaMemcpyDeviceToHost, ctx->st));
  CK(cudaStreamSynchronize(ctx->st));
  return YY_OK;
}

yy_status yy_set_param(yy_ctx* ctx, int32_t key, double v) {
  if (!ctx) return YY_EINVAL;
  clear_loop_graphs(ctx);
  if (ctx->mode == 1)
    for (yy_ctx* c : ctx->group) if (c && c != ctx) clear_loop_graphs(c);
  switch (key) {
    case YY_CHI:
      if (!(v > 0)) return fail(ctx, YY_EINVAL, "chi must be > 0");
      ctx->chi = v;
      ctx->g.cchi = 1.0 / (2.0 * v);
      ctx->g.inv_chi = 1.0 / v;
      launch_build_split(ctx->g, ctx->bsplit, ctx->tsplit, ctx->st);   // the D_ii rows carry c_chi
      CK(cudaStreamSynchronize(ctx->st));
      return YY_OK;
    case YY_MAX_ITERS:
      if (v < 1) return fail(ctx, YY_EINVAL, "max_iters must be >= 1");
      ctx->max_iters = (int)v;
      return YY_OK;
    case YY_FIXED_ITERS:
      if (v < 0) return fail(ctx, YY_EINVAL, "fixed_iters must be >= 0");
      ctx->fixed_iters = (int)v;
      return YY_OK;
    case YY_SCHWARZ:
      if (v != 0 && v != 1 && v != 2)
        return fail(ctx, YY_EINVAL, "schwarz must be 0 (additive), 1 (multiplicative) or 2 (none: single domains)");
      if (v == 1 && ctx->g.npatch == 2)
        return fail(ctx, YY_EINVAL, "multiplicative Schwarz needs one patch per context (yy_create_pair/_slabs/_dist)");
      ctx->schwarz = (int)v;
      if (ctx->mode == 1)
        for (yy_ctx* c : ctx->group) if (c) c->schwarz = (int)v;
      return YY_OK;
    case YY_FLUX_FIX:
      if (v < 0) return fail(ctx, YY_EINVAL, "flux-fix eps must be >= 0 (0 = off)");
      if (v > 0 && ctx->nslab > 1) return fail(ctx, YY_EINVAL, "flux fix needs whole patches (no radial slabs)");
      ctx->flux_eps = v;
      if (ctx->mode == 1)
        for (yy_ctx* c : ctx->group) if (c) c->flux_eps = v;
      return YY_OK;
    case YY_HEAT_ONLY:
      ctx->heat_only = v != 0;
      if (ctx->mode == 1)
        for (yy_ctx* c : ctx->group) if (c) c->heat_only = ctx->heat_only;
      return YY_OK;
    case YY_ADVECTION: {
      if (v != 0 && v != 1) return fail(ctx, YY_EINVAL, "advection must be 0 (in the split factors) or 1 (IMEX)");
      auto set = [&](yy_ctx* c) -> yy_status {
        c->imex = v != 0;
        if (c->imex && !c->zero) {
          long long mx = 0;
          for (int K = 0; K < 4; ++K) mx = std::max(mx, c->g.npatch * psize(c->g, K));
          TRY(dalloc(c, &c->zero, mx));
          CK(cudaMemset(c->zero, 0, mx * sizeof(double)));
        }
        for (int K = 0; K < 4; ++K)
          for (int ax = 0; ax < 3; ++ax) c->g.adv[K][ax] = c->imex ? c->zero : c->adv[K][ax];
        return YY_OK;
      };
      TRY(set(ctx));
      if (ctx->mode == 1)
        for (yy_ctx* c : ctx->group) if (c && c != ctx) TRY(set(c));
      return YY_OK;
    }
    case YY_INTERP_ORDER:
      if (v != 4) return fail(ctx, YY_EINVAL, "interpolation order: only 4 (4x4 Lagrange, RD4) is built");
      return YY_OK;
    case YY_PROFILE:
      cudaStreamSynchronize(ctx->st);
      prof_collect(ctx);
      ctx->prof.clear();
      ctx->prof_on = v != 0;
      return YY_OK;
  }
  return fail(ctx, YY_EINVAL, "unknown parameter key");
}

yy_status yy_set_allocator(yy_ctx* ctx, void* (*alloc)(size_t, void*), void (*free_)(void*, void*), void* user) {
  if ((alloc == nullptr) != (free_ == nullptr)) return ctx ? fail(ctx, YY_EINVAL, "alloc and free go together") : YY_EINVAL;
  if (ctx) return fail(ctx, YY_ESTATE, "a context allocates at yy_create: set the allocator with ctx = NULL first");
  g_alloc.alloc = alloc;
  g_alloc.free_ = free_;
  g_alloc.user = user;
  return YY_OK;
}

yy_status yy_set_stream(yy_ctx* ctx, void* stream) {
  if (!ctx) return YY_EINVAL;
  clear_loop_graphs(ctx);
  ctx->st = static_cast<cudaStream_t>(stream);
  if (ctx->mode == 1)   // a loopback group shares one stream
    for (yy_ctx* c : ctx->group) if (c) c->st = ctx->st;
  return YY_OK;
}

yy_status yy_step(yy_ctx* ctx, int32_t nsteps, double tol) {
  if (!ctx) return YY_EINVAL;
  if (ctx->dead) return fail(ctx, YY_ESTATE, "context unusable after a CUDA error");
  if (nsteps < 0 || !(tol > 0)) return fail(ctx, YY_EINVAL, "nsteps >= 0 and tol > 0 required");
  // the group that holds both patches: this context, or a loopback pair (Yin first)
  std::vector<yy_ctx*> cs{ctx};
  if (ctx->mode == 1) {
    cs = ctx->group;
    for (yy_ctx* c : cs) {
      if (!c) return fail(ctx, YY_ESTATE, "loopback group member destroyed");
      if (c->dead) return fail(ctx, YY_ESTATE, "loopback group member unusable");
    }
  }
  yy_status res = YY_OK;
  for (int s = 0; s < nsteps; ++s) {
    int it = 0;
    double rho = 0;
    yy_status r = step_group(cs, tol, &it, &rho);
    if (r != YY_OK) {
      if (ctx->err.empty()) for (yy_ctx* c : cs) if (!c->err.empty()) ctx->err = c->err;
      return r;
    }
    for (yy_ctx* c : cs) {
      c->st_iters.push_back(it);
      c->st_rho.push_back(rho);
    }
    if (ctx->fixed_iters <= 0 && !(rho < tol)) res = YY_ENOCONV;
  }
  return res;
}

yy_status yy_get_stats(const yy_ctx* ctx, int32_t cap, int32_t* iters, double* resid, int32_t* n_out) {
  if (!ctx || cap < 0) return YY_EINVAL;
  const int n = (int)ctx->st_iters.size();
  const int cnt = n < cap ? n : cap;
  for (int q = 0; q < cnt; ++q) {
    if (iters) iters[q] = ctx->st_iters[n - cnt + q];
    if (resid) resid[q] = ctx->st_rho[n - cnt + q];
  }
  if (n_out) *n_out = cnt;
  return YY_OK;
}

double yy_time(const yy_ctx* ctx) { return ctx ? ctx->t : 0.0; }

int64_t yy_launch_count(const yy_ctx* ctx) { return ctx ? ctx->launches : -1; }

yy_status yy_profile_report(yy_ctx* ctx, char* buf, int32_t len) {
  if (!ctx || !buf || len <= 0) return YY_EINVAL;
  cudaStreamSynchronize(ctx->st);
  prof_collect(ctx);
  std::string out;
  for (auto& kv : ctx->prof) {
    char line[160];
    std::snprintf(line, sizeof line, "%s %lld %.6f\n", kv.first.c_str(), kv.second.first, kv.second.second);
    out += line;
  }
  std::snprintf(buf, (size_t)len, "%s", out.c_str());
  return (int32_t)out.size() < len ? YY_OK : YY_EINVAL;
}

const char* yy_last_error(const yy_ctx* ctx) { return ctx ? ctx->err.c_str() : "NULL context"; }

void yy_destroy(yy_ctx* ctx) {
  if (!ctx) return;
  if (ctx->mode == 1)
    for (yy_ctx* c : ctx->group)
      if (c && c != ctx)
        for (auto& m : c->group) if (m == ctx) m = nullptr;
  if (ctx->mode == 2 && ctx->nccl) nccl_api().CommDestroy(static_cast<ncclComm_t>(ctx->nccl));
  if (ctx->alloc_fn) cudaStreamSynchronize(ctx->st);   // (a caching allocator may hand the memory on)
  for (void* p : ctx->allocs) {
    if (ctx->alloc_fn) ctx->free_fn(p, ctx->alloc_user);
    else cudaFree(p);
  }
  for (auto& lg : ctx->loop_graphs) cudaGraphExecDestroy(lg.exec);
  if (ctx->red_host) cudaFreeHost(ctx->red_host);
  for (cudaStream_t a : ctx->aux) if (a) cudaStreamDestroy(a);
  for (cudaEvent_t e : ctx->fork) if (e) cudaEventDestroy(e);
  delete ctx;
}

// ---- test / kernel-only entry points (include/yy_test.h) ---------------------------
yy_status yy_debug_get(yy_ctx* ctx, const char* name, int32_t patch, double* host) {
  if (!ctx || !name || !host || patch < ctx->patch0 || patch >= ctx->patch0 + ctx->g.npatch) return YY_EINVAL;
  patch -= ctx->patch0;
  const Geo& g = ctx->g;
  const double* src = nullptr;
  long long sz = 0;
  static const char* gnames[NF] = {"G_T", "", "", "G_ur1", "G_ut1", "G_up1", "G_ur2", "G_ut2", "G_up2"};
  for (int f = 0; f < NF; ++f)
    if (gnames[f][0] && !std::strcmp(name, gnames[f])) { src = ctx->G[f]; sz = psize(g, FKIND[f]); }
  static const char* anames[3] = {"astar_r", "astar_t", "astar_p"};
  for (int c = 0; c < 3; ++c)
    if (!std::strcmp(name, anames[c])) { src = ctx->astar[c]; sz = psize(g, KR + c); }
  if (!src) return fail(ctx, YY_EINVAL, std::string("unknown debug array ") + name);
  CK(cudaMemcpy(host, src + patch * sz, sz * sizeof(double), cudaMemcpyDeviceToHost));
  return YY_OK;
}

}  // extern "C"

extern "C" yy_status yy_line_prepare(yy_ctx* ctx, const double* d_ar, const double* d_at, const double* d_ap) {
  if (!ctx || !d_ar || !d_at || !d_ap) return YY_EINVAL;
  if (ctx->dead) return fail(ctx, YY_ESTATE, "context unusable after a CUDA error");
  // the temperature rows' transport-velocity weights of these a* (patch 0; overwrites
  // the context's per-step ones: the next yy_step recomputes them from its own a*)
  launch_adv(ctx->g, d_ar, d_at, d_ap, ctx->adv, 1, ctx->st, 1 << KC);
  ctx->line_a[0] = d_ar; ctx->line_a[1] = d_at; ctx->line_a[2] = d_ap;
  CK(cudaGetLastError());
  return YY_OK;
}

extern "C" yy_status yy_line_solve(yy_ctx* ctx, int32_t axis, const double* d_ar, const double* d_at,
                                   const double* d_ap, double* d_x) {
  if (!ctx || axis < 0 || axis > 2 || !d_x) return YY_EINVAL;
  const bool given = d_ar || d_at || d_ap;
  if (given && !(d_ar && d_at && d_ap)) return YY_EINVAL;
  if (ctx->dead) return fail(ctx, YY_ESTATE, "context unusable after a CUDA error");
  if (given) {
    yy_status s = yy_line_prepare(ctx, d_ar, d_at, d_ap);
    if (s != YY_OK) return s;
  } else if (!ctx->line_a[0]) {
    return fail(ctx, YY_ESTATE, "yy_line_solve without a*: no yy_line_prepare before");
  }
  d_ar = ctx->line_a[0]; d_at = ctx->line_a[1]; d_ap = ctx->line_a[2];   // (rows that average a* in place)
  SweepArgs w{};
  w.ar = d_ar; w.at = d_at; w.ap = d_ap;
  w.R = d_x; w.psi = nullptr; w.part = nullptr; w.maxb = 0;
  launch_sweep(ctx->g, QT, axis, 1, false, false, false, w, nullptr, 1, ctx->st);
  CK(cudaGetLastError());
  return YY_OK;
}
