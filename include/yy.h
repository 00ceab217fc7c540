/*
 * yy.h — C ABI of the B200-native Yin-Yang AC direction-splitting time step
 * (Takhirov, Frolov & Minev, arXiv 1905.02300).
 *
 * One context = one spherical shell R1 <= r <= R2 covered by the two Yin-Yang
 * patches (§2), each a MAC grid of nr x ntheta x nphi cells
 * (PAPER.md L473-475).  yy_step advances the Navier-Stokes-Boussinesq system
 * (eq:eq_ns, eq:eq_heat_convec) by the second-order
 * artificial-compressibility direction-splitting scheme (§3, eq:Convect_Douglas,
 * eq:r_comp, eq:theta_comp, eq:phi_comp, eq:nst_Mass1, eq:ac2) with additive
 * Schwarz iteration between the patches and the splitting-error reduction of
 * eq:er (§4), iterated until the successive-iterate l2 difference
 * is below the tolerance (§5.1).  Readings of garbled passages:
 * DESIGN.md (RD1-RD42 of SURVEY.md §8(c)).
 *
 * Geometry (reading RD1/RD2): per patch theta in [pi/4 - d, 3pi/4 + d],
 * phi in [-3pi/4 - d, 3pi/4 + d], d = 2 theta-cells, dtheta = pi/(2(ntheta-4)),
 * dphi = (3pi/2 + 2d)/nphi, dr = (R2-R1)/nr.  Patch 0 = Yin, 1 = Yang.
 *
 * Array layout (host and device): C order, fp64, phi fastest.  Spherical
 * vector components are in the patch's own chart basis.
 *     u_r   (nr+1, ntheta,   nphi)      r-faces
 *     u_th  (nr,   ntheta+1, nphi)      theta-faces
 *     u_ph  (nr,   ntheta,   nphi+1)    phi-faces
 *     p, T  (nr,   ntheta,   nphi)      cell centres
 * The outermost theta/phi node layer of every array is the Schwarz fringe
 * (reading RD3): values there are Dirichlet data overwritten by interpolation
 * from the other patch every iteration; u_r planes 0 and nr are the walls.
 *
 * Ownership: host pointers are borrowed for the duration of a call; set/get
 * are synchronous with respect to the host.  The context owns every device
 * buffer.  Errors: negative status = failure (see yy_last_error); YY_ENOCONV
 * is a positive warning (state advanced, some step hit max_iters).  After
 * YY_ECUDA the only valid call is yy_destroy.  One context per host thread.
 */
#ifndef YY_H
#define YY_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  YY_OK = 0,
  YY_ENOCONV = 4,   /* warning: a step stopped at max_iters (SPEC exit 4)       */
  YY_EINVAL = -2,   /* argument validation (SPEC exit 2)                          */
  YY_ESOLVER = -3,  /* NaN/Inf residual (SPEC exit 3)                             */
  YY_ECUDA = -10,
  YY_ENCCL = -11,
  YY_ENOMEM = -12,
  YY_ESTATE = -13
} yy_status;

/* time basis of wall data / sources: value(t) = sum_m g_m(t) * term_m */
enum { YY_TF_ONE = 0, YY_TF_COS = 1, YY_TF_SIN = 2, YY_TF_COS2 = 3 };

/* yy_set_param keys */
enum {
  YY_CHI = 1,          /* artificial-compressibility chi (eq:ac1); default 1 (RD19) */
  YY_MAX_ITERS = 2,    /* Schwarz K_max (RD25); default 100                                  */
  YY_FIXED_ITERS = 3,  /* >0: run exactly this many iterations per step, ignore tol          */
  YY_PROFILE = 4,      /* !=0: time every kernel class with CUDA events (resets the table)   */
  YY_SCHWARZ = 5,      /* 0: additive (RD26, default); 1: multiplicative, Algorithm 1 as printed
                          (Yin with Yang's iterate k-1, then Yang with Yin's k).
                          Needs one patch per context (yy_create_dist, or the test-only
                          yy_create_pair / yy_create_slabs); set on every rank.
                          2: none — every patch is a single domain whose fringe keeps the
                          Dirichlet values set by yy_set_fields (Theorem 1's setting,
                          P:L250-260; with YY_HEAT_ONLY and YY_FIXED_ITERS = 1 a step is
                          exactly eq:HeatDouglas)                                          */
  YY_HEAT_ONLY = 6,    /* !=0: the heat Douglas scheme eq:HeatDouglas alone: only
                          T is solved (u, p stay as set, normally 0 so a* = 0), the
                          momentum and pressure kernels are skipped, rho_k is T's norm      */
  YY_ADVECTION = 9,    /* where the linearised advection goes: 0 = inside the
                          direction-wise factors (the paper's scheme, default); 1 = IMEX (SURVEY
                          NEXT-3): the factors and L_split are the a* = 0 rows (diffusion,
                          metric, grad-div), the transport terms (advection, the a*-reaction
                          terms of RD14 / P:L444) stay only in the explicit L_full psi^* of G */
  YY_INTERP_ORDER = 8, /* fringe interpolation order: 4 (4x4 Lagrange in (theta, phi), RD4) is the
                          only one built; any other value is YY_EINVAL                       */
  YY_FLUX_FIX = 7      /* eps > 0: Algorithm 1 step 4 every
                          iteration after the fringe exchange — if |net boundary flux| >= tol
                          the fringe normal velocities become the minimiser of J with penalty
                          eps (1e-6); 0 = off (default, as in the paper's runs).
                          Whole patches only (not with radial slabs)                        */
};

typedef struct {
  int32_t nr, ntheta, nphi;   /* cells per patch; 2 <= nr <= 512, 8 <= ntheta <= 513, 8 <= nphi <= 1153
                                 (longest lines of the chunked line solver; larger -> YY_EINVAL) */
} yy_grid;

typedef struct yy_ctx yy_ctx;

/* Host pointers to one patch's fields (shapes above).  A NULL member means
 * "leave unchanged" (set) or "do not copy" (get). */
typedef struct {
  double *ur, *ut, *up, *p, *T;
} yy_fields;

/* Create a context on the current CUDA device.  R1 < R2 radii, Pr Prandtl
 * number (momentum viscosity nu = Pr, RD33), Ra Rayleigh number (buoyancy
 * +Pr*Ra*T e_r, RD20), dt > 0 time step.  All state starts at zero, t = 0. */
yy_status yy_create(const yy_grid* g, double R1, double R2, double Pr, double Ra, double dt,
                    yy_ctx** out);

/* Multi-GPU: one process per GPU, one context per process.
 * world = 2 nslab (2, 4, 8, 16): rank r holds radial slab r % nslab (nr / nslab
 * rows, nr divisible by nslab) of patch r / nslab (Yin on ranks 0..nslab-1, Yang
 * on the others) on CUDA device `device`.  Every Schwarz iteration the donor rank
 * evaluates the partner's fringe (same slab, other patch) from its own data
 * (Alg. 1 steps 1/3/7) and they swap it; slab neighbours swap r-halo
 * rows after every update; the r-factor sweeps are the partitioned
 * (Schur-complement) solve of P:L477-480 across the slabs of a patch (boundary
 * rows gathered per patch); the per-(quantity, patch, slab) norms (RD24) are
 * gathered and summed in fixed order — all over NCCL point-to-point on the
 * context's stream.  world = 1, rank 0 is yy_create on `device`.  nccl_id: 128 bytes from
 * yy_nccl_unique_id on rank 0, broadcast by the caller (e.g. torch.distributed).
 * Collective semantics: every rank calls the same sequence of yy_step.  NCCL is
 * resolved at run time (libnccl.so.2); missing -> YY_ENCCL.  set/get/wall/source
 * calls accept only the rank's own patch, as full-patch arrays (a slab reads its
 * rows and halos, get writes back the rows it owns). */
yy_status yy_create_dist(const yy_grid* g, double R1, double R2, double Pr, double Ra, double dt,
                         int32_t world, int32_t rank, const void* nccl_id, int32_t device, yy_ctx** out);
yy_status yy_nccl_unique_id(void* out128);

/* Set one patch's state.  level 0 = t^n, 1 = t^{n-1} (p ignored).  system
 * 0 = both bootstrapped systems (u1 = u2, p1 = p2; eq:ac1/eq:ac2; one host copy,
 * system 2 filled by device copies), 1 or 2 = that system only.  T is shared
 * by both systems.  NULL members are left unchanged. */
yy_status yy_set_fields(yy_ctx* ctx, int32_t patch, int32_t level, int32_t system,
                        const yy_fields* f);

/* Copy one patch's state to the host (system 1 or 2; 2 is the second-order answer). */
yy_status yy_get_fields(yy_ctx* ctx, int32_t patch, int32_t level, int32_t system,
                        yy_fields* out);

/* Wall (r = R1, R2) Dirichlet data of one patch as nterms <= 4 time-basis
 * terms.  terms[m].T / .ur are (2, ntheta, nphi), .ut (2, ntheta+1, nphi),
 * .up (2, ntheta, nphi+1) — index 0 = inner wall; NULL member = zero; .p unused.
 * Default: homogeneous walls (eq:eq_ns, eq:eq_heat_convec). */
yy_status yy_set_wall(yy_ctx* ctx, int32_t patch, int32_t nterms, const int32_t* timefn,
                      const yy_fields* terms);

/* Volume sources (manufactured forcing, reading RD32) as nterms <= 4 terms,
 * full 3-D staggered arrays; evaluated at t_{n+1/2}; .p unused. */
yy_status yy_set_source(yy_ctx* ctx, int32_t patch, int32_t nterms, const int32_t* timefn,
                        const yy_fields* terms);

yy_status yy_set_param(yy_ctx* ctx, int32_t key, double value);

/* Device-memory hook (e.g. PyTorch's caching allocator): contexts created after
 * yy_set_allocator(NULL, alloc, free_, user) obtain every device buffer as
 * alloc(bytes, user) and return it with free_(ptr, user) at yy_destroy (after a
 * stream synchronize); alloc = free_ = NULL restores cudaMalloc / cudaFree.
 * A context allocates everything at yy_create, so ctx != NULL is YY_ESTATE.
 * alloc returning NULL fails the create with YY_ENOMEM.  Not thread-safe
 * against concurrent yy_create calls. */
yy_status yy_set_allocator(yy_ctx* ctx, void* (*alloc)(size_t bytes, void* user), void (*free_)(void* ptr, void* user),
                           void* user);

/* Launch every kernel on this stream (a cudaStream_t, e.g.
 * torch.cuda.current_stream().cuda_stream).  Default: the legacy stream. */
yy_status yy_set_stream(yy_ctx* ctx, void* cuda_stream);

/* Advance nsteps time steps; each step iterates Schwarz until
 * rho_k < schwarz_tol (or max_iters / fixed_iters). */
yy_status yy_step(yy_ctx* ctx, int32_t nsteps, double schwarz_tol);

/* Per-step Schwarz iteration counts and final rho of every step taken so far
 * (up to cap entries, most recent last); *n_out = number written. */
yy_status yy_get_stats(const yy_ctx* ctx, int32_t cap, int32_t* iters_per_step,
                       double* resid_per_step, int32_t* n_out);

double yy_time(const yy_ctx* ctx);

/* Theorem 1 diagnostic (eq:Stability; DESIGN.md §8 NEXT-2): for the
 * current levels T^n, T^{n-1} of every patch the context holds, with u = 0 rows
 * (pure diffusion) and HOMOGENEOUS wall / fringe data (the theorem's setting;
 * the stored fringe values must be 0 for the identity to hold), out3 (host, 3
 * doubles) = { 1/2 (-L T^n, T^n)_w,  1/4 (-(Lh - L) dT, dT)_w,  (dT, dT)_w },
 * dT = T^n - T^{n-1}, L the full and Lh the hat (theta, phi) operators of
 * P:L208, (.,.)_w the midpoint omega inner product over solved cell centres
 * (RD24).  The left side of eq:Stability after step N is
 * sum_{n<=N} out3[2]/tau + out3[0] + out3[1]: non-increasing in N for the
 * heat-only single-domain Douglas scheme.  Whole patches only (no radial slabs:
 * YY_EINVAL).  Synchronous with respect to the host. */
yy_status yy_energy(yy_ctx* ctx, double* out3);

/* Number of CUDA kernels this context has launched since creation. */
int64_t yy_launch_count(const yy_ctx* ctx);

/* Per-kernel-class device time since YY_PROFILE was set: one line per class,
 * "name launches total_ms\n", written to buf (len bytes, NUL-terminated). */
yy_status yy_profile_report(yy_ctx* ctx, char* buf, int32_t len);
const char* yy_last_error(const yy_ctx* ctx);
void yy_destroy(yy_ctx* ctx);   /* NULL is a no-op */

#ifdef __cplusplus
}
#endif
#endif /* YY_H */
