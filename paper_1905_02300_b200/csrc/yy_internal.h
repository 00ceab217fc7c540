// yy_internal.h — kernel argument blocks shared by yy_kernels.cu and yy_api.cu.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace yy {

struct Geo;

constexpr int NSLOT = 9;     // T, u1r, u1t, u1p, p1, u2r, u2t, u2p, p2 (convergence slots)
constexpr int MAXSRC = 4;    // time-basis terms per patch

struct LinIn {               // out = sum_m c[m] * p[m]
  const double* p[8];
  double c[8];
};

// a batch of small linear combinations in one launch (the wall data of every
// (time level, field, patch) of a step: 24 launches -> 1)
constexpr int MAXLIN = 32;
struct LinBatch {
  double* out[MAXLIN];
  long long n[MAXLIN];
  int nin[MAXLIN];              // terms; -1: a plain copy of p[.][0]
  const double* p[MAXLIN][4];
  double c[MAXLIN][4];
  int njobs;
};

struct StaticArgs {
  const double* fn[2];       // psi^n   (system 1, 2; T uses [0])
  const double* fm[2];       // psi^{n-1}
  const double* wn;          // wall data at t_n (2 patches x 2 walls x plane), NULL for u_r
  const double* wm;          // wall data at t_{n-1}
  const double *ar, *at, *ap;  // a*
  const double *rt, *rp;     // a*-reaction coefficients (Astar)
  const double* p[2];        // p1^n, p2^n
  const double* utn[2];      // u_th^n, u_th^{n-1} per system (for u_th^*)
  const double* utm[2];
  const double* upn[2];
  const double* upm[2];
  const double* src[2][MAXSRC];   // [patch][term] source arrays of this quantity
  double gsrc[2][MAXSRC];
  int nsrc[2];
  double* G[2];
  int imex;                  // the -1/2 L_split term without transport terms (YY_ADVECTION = 1)
};

struct ResidArgs {
  const double* it;          // psi~ (iterate with fresh fringe / walls)
  const double* n;           // psi^n
  const double* wnew;        // wall data t_{n+1}
  const double* wn;          // wall data t_n
  const double *ar, *at, *ap;
  const double *rt, *rp;
  const double* G;
  double* R;
  const double *Tit, *Tn;    // for u_r buoyancy
  const double *urit, *urn;  // this system's u_r (iterate, level n)
  const double *utit, *utn;
  const double *p1it, *p1n;
  const double* dp1;         // p1^(k) - p1^n (both patches, fringe incl.) or NULL: from p1it, p1n
  int rev;                   // reverse block order (bidx)
  int noadv;                 // IMEX: L_split without transport terms (no a* / row-weight reads)
};

struct SweepArgs {
  const double *ar, *at, *ap;
  const double *rt, *rp;
  double* R;                 // in: rhs, out: solution (non-final); slab r-sweep: x0
  double* psi;               // FINAL: psi += x
  double* part;              // FINAL: norm partials of this slot (2 * maxb)
  int maxb;
  // radial slab r-sweep (partitioned across slabs): responses of the
  // line to the lower / upper neighbour slab's boundary unknowns, and the per-line
  // boundary values (x0, xlo, xhi at the first row, then at the last row)
  double* V;
  double* W;
  double* IF;                // [line][6], line = (j-1)(np_k-2) + (k-1)
  int vw;                    // write V, W (they depend on the step's matrix only: the first
                             // iteration of a step writes them, later ones reuse them)
  int rev;                   // run the grid's blocks in reverse linear order (bidx)
  int noadv;                 // IMEX (YY_ADVECTION = 1): rows without transport terms — the
                             // per-step row weights are not read (16 B per element, 24 final)
  int flat;                  // k_line_th: r boxes over the (theta, phi) plane (odd phi pitch; set by its launcher)
};

// one r-line's slab-coupling solution (yy_slab.cu)
struct SlabArgs {
  const double* IFall;       // [nslab][nlines][6] boundary values of every slab of the patch
  double* LH;                // [nlines][2]: this slab's lower / upper neighbour unknowns
  int nslab, slab, nlines;
};

struct PresArgs {
  const double *urit, *urn, *utit, *utn, *upit, *upn;
  const double* pn;          // this system's p^n
  const double *p1it, *p1n;  // system 2 only
  double* pit;               // this system's p iterate (updated in place)
  double* part;
  int maxb;
  double* dp1;               // system 1 writes p1^(k) - p1^n at the solved cells, system 2 reads it (or NULL)
  int rev;                   // reverse block order (bidx)
};

// Algorithm 1 step 4 (mass-flux correction)
struct FluxArgs {
  double *ur[2], *ut[2], *up[2];   // iterates of systems 1, 2 (all local patches)
  double a2;                       // |a|^2: sum of the squared side-face areas (one patch)
  double area;                     // |dOmega|: total closed-surface area (one patch)
  double eps, tol;
};

struct ReduceArgs {
  int nblk[NSLOT];
  int maxb;
  int npatch;                // local patches
  int patch0;                // global id of local patch 0 (sums land at out[2 + 2 slot + patch])
};

struct CCTab {               // fringe of kinds C / R on the (theta_c, phi_c) lattice
  int n;
  const int *tj, *tk, *jb, *kb;
  const double* w;           // [n][8]: wt[4], wp[4]
};

struct VecTab {              // fringe of kind TH or PH
  int n;
  const int *tj, *tk;
  const int *jb_t, *kb_t, *jb_p, *kb_p;
  const double *w_t, *w_p;   // [n][8]
  const double *m0, *m1;     // rotation row
};

struct InterpArgs {
  double* cc[5];             // T, p1, p2, u1r, u2r iterates (both patches)
  double* ut[2];
  double* up[2];
  CCTab tab_cc;
  VecTab tab_th, tab_ph;
  double* dp1;               // with p1n: also write p1^(k) - p1^n at the p1 fringe (or NULL)
  const double* p1n;
  int cc_q0, cc_nq;          // k_interp_cc: quantities cc_q0 .. cc_q0 + cc_nq - 1 (0 quantities: all 5)
};

void launch_lincomb(double* out, long long n, const LinIn& in, int nin, cudaStream_t st);
void launch_lincomb_batch(const LinBatch& b, cudaStream_t st);
// per step, after a*: the reaction coefficients rt (TH nodes), rp (PH nodes) of Astar
void launch_react(const Geo& g, const double* ar, const double* at, double* rt, double* rp, cudaStream_t st);
// per step, after a*: the transport-velocity row weights Astar::av of the kinds in
// the bit mask `kinds` and every axis (dst[K][d], at the solved nodes; Geo::adv
// points at them)
void launch_adv(const Geo& g, const double* ar, const double* at, const double* ap, double* const (&dst)[4][3],
                int npatch, cudaStream_t st, int kinds = 0xf);
void launch_static(const Geo& g, int q, const StaticArgs& a, cudaStream_t st);
void launch_resid(const Geo& g, int q, int s, const ResidArgs& a, cudaStream_t st);
inline int max_line_len(int ax) { return ax == 2 ? 32 * 36 : 32 * 16; }   // unknowns per line (yy_line.cu)
// line sweeps (yy_line.cu): factor `ax` of quantity Q, system s; first = fused
// eq:er residual from *ra (the quantity's first factor), fin = psi += x and the
// norm partial (its last factor); neither = plain.  Returns blocks launched
// (norm partial count) or -1 if (ax, first, fin) is not a factor position of Q.
// slab = the r-factor of a radial slab (partitioned across slabs: writes x0, V, W,
// IF; finished by launch_slab_solve / launch_slab_correct).
template <int Q>
int launch_sweep_q(const Geo& g, int ax, int s, bool first, bool fin, bool slab, const SweepArgs& a,
                   const ResidArgs* ra, int npatch, cudaStream_t st);
#ifndef YY_LINE_Q   // (the per-quantity line TUs instantiate only their own Q)
inline int launch_sweep(const Geo& g, int q, int ax, int s, bool first, bool fin, bool slab, const SweepArgs& a,
                        const ResidArgs* ra, int npatch, cudaStream_t st) {
  switch (q) {
    case 0: return launch_sweep_q<0>(g, ax, s, first, fin, slab, a, ra, npatch, st);
    case 1: return launch_sweep_q<1>(g, ax, s, first, fin, slab, a, ra, npatch, st);
    case 2: return launch_sweep_q<2>(g, ax, s, first, fin, slab, a, ra, npatch, st);
    default: return launch_sweep_q<3>(g, ax, s, first, fin, slab, a, ra, npatch, st);
  }
}
#endif
int launch_pres(const Geo& g, int s, const PresArgs& a, cudaStream_t st);
// per-(slot, local patch) sums of the norm partials -> out[2 + 2 slot + patch]
void launch_reduce_slots(const double* part, const ReduceArgs& a, double* out, cudaStream_t st);
// rho = max over the 2 NSLOT sums -> out[0], NaN flag -> out[1]
void launch_reduce_final(double* out, cudaStream_t st);
// Theorem 1 diagnostic (yy_energy): out[3] = (1/2 (-L T, T)_w, 1/4 ||dT||^2_D, ||dT||^2_w)
int energy_blocks(const Geo& g);
void launch_energy(const Geo& g, const double* Tn, const double* Tm, const double* zw, double* part, double* out,
                   cudaStream_t st);
// device-side Schwarz loop: ctl = {iterations, rho, NaN flag}; sets the WHILE
// node's condition h (continue: no NaN, k < kmax, fixed or rho >= tol)
void launch_schwarz_cond(cudaGraphConditionalHandle h, const double* red, double* ctl, double tol, int kmax,
                         bool fixed, cudaStream_t st);
// the three fringe classes (cell/r-face lattice, theta faces, phi faces); with s2,
// s3 and ev[3] given they run concurrently (fork / join on st through the events)
// defer: only T's fringe on st; the other four cell-lattice quantities (on s2, ahead
// of the theta faces) and the phi faces are left running — the caller joins them
// with join_interp before anything reads the p / u fringes (they overlap the T solve)
void launch_interp(const Geo& g, const InterpArgs& a, cudaStream_t st, cudaStream_t s2 = nullptr,
                   cudaStream_t s3 = nullptr, cudaEvent_t* ev = nullptr, bool defer = false);
void join_interp(cudaStream_t st, cudaEvent_t* ev);
// one patch per context: the donor evaluates the partner's fringe values from its
// own patch into buf (pack), the target writes a received buf into its fringe
// (unpack).  Layout: [cc: 5 x (nr+1) x n_cc][th: 2 x nr x n_th][ph: 2 x nr x n_ph].
long long fringe_count(const Geo& g, const InterpArgs& a);
void launch_fringe_pack(const Geo& g, const InterpArgs& a, double* buf, cudaStream_t st);
void launch_fringe_unpack(const Geo& g, const InterpArgs& a, const double* buf, cudaStream_t st);
// out[2 + 2 slot + p] <- sum over slabs s (fixed order) of gath[p * nslab + s][2 + 2 slot + p]
// (gath: every context's sums, world = 2 nslab contexts ordered rank = patch nslab + slab)
void launch_flux_fix(const Geo& g, const FluxArgs& a, cudaStream_t st);
// fill the split-row tables dst[Q][AX] (Geo::bsplit; 3 NRk NTk doubles each) and
// the factor-row tables tdst[Q][AX] (Geo::tsplit, the same size)
void launch_build_split(const Geo& g, double* const (&dst)[4][3], double* const (&tdst)[4][3], cudaStream_t st);
void launch_merge_all(double* out, const double* gath, int nslab, cudaStream_t st);
// slab r-sweeps: solve the 2 nslab boundary system of every line, then x = x0 + xlo X_LO + xhi X_HI
void launch_slab_solve(const SlabArgs& a, cudaStream_t st);
int launch_slab_correct(const Geo& g, int kind, bool fin, const SweepArgs& w, const double* LH, cudaStream_t st);

}  // namespace yy
