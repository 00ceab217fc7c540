/*
 * yy_test.h — test and kernel-only entry points of the Yin-Yang step library.
 * Not part of the user API; used by tests/ (unit parity of internal stages)
 * and by bench.py's C4 kernel-only workload.
 */
#ifndef YY_TEST_H
#define YY_TEST_H
#include "yy.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Copy an internal per-step array of one patch to the host.  Names:
 * "astar_r" | "astar_t" | "astar_p"  (a* = u2^{*,n+1/2}) and
 * "G_T" | "G_ur1" | "G_ut1" | "G_up1" | "G_ur2" | "G_ut2" | "G_up2"
 * (static right-hand sides G_q of the LAST step taken).
 * host must hold the kind's full staggered array. */
yy_status yy_debug_get(yy_ctx* ctx, const char* name, int32_t patch, double* host);

/* C4 kernel-only operator: for ONE patch of ctx's grid solve
 * (I - dt/2 A_axis) x = b on every line of `axis` (0 r, 1 theta, 2 phi) of the
 * temperature operator (eq:Convect_Douglas factors, hat operators, transport
 * velocity a* given by d_ar (nr+1,nt,np), d_at (nr,nt+1,np), d_ap (nr,nt,np+1)).
 * d_x (nr,nt,np) holds b on entry and x on exit at the solved nodes (fringe
 * layer untouched; homogeneous end conditions, wall ghost rule RD23).
 * All pointers are DEVICE pointers; asynchronous on ctx's stream.
 * The rows' transport-velocity weights are first evaluated from a* (as
 * yy_line_prepare); with d_ar = d_at = d_ap = NULL the a* and weights of the
 * last yy_line_prepare are used instead (its a* arrays must still be valid; the
 * per-step precompute of yy_step: a* fixed, many sweeps).  YY_EINVAL if only
 * some of the three are NULL, YY_ESTATE if nothing was prepared. */
yy_status yy_line_solve(yy_ctx* ctx, int32_t axis, const double* d_ar, const double* d_at,
                        const double* d_ap, double* d_x);

/* Evaluate the temperature rows' transport-velocity weights of a* (device
 * pointers, shapes as above) for later yy_line_solve calls with NULL a*.
 * Overwrites the context's per-step weights (the next yy_step recomputes its
 * own).  Asynchronous on ctx's stream. */
yy_status yy_line_prepare(yy_ctx* ctx, const double* d_ar, const double* d_at, const double* d_ap);

/* Two one-patch contexts in this process on the current device (out2[0] holds
 * Yin, out2[1] Yang) that exchange fringe values and norms by device copies on
 * one shared stream: the data path of yy_create_dist (donor-side evaluation,
 * transfer, target write, fixed-order norm merge) without NCCL, so one GPU can
 * check it against the oracle.  yy_step on either context advances both. */
yy_status yy_create_pair(const yy_grid* g, double R1, double R2, double Pr, double Ra, double dt,
                         yy_ctx** out2);

/* 2 nslab one-patch radial-slab contexts in this process on the current device
 * (out[r], r = patch * nslab + slab; nr divisible by nslab, nr / nslab >= 4):
 * the yy_create_dist layout of 2 nslab GPUs — r-halo rows, the partitioned
 * r-sweep across slabs, the fringe swap between (patch, slab)
 * and (other patch, slab), the fixed-order norm merge — exchanging by device
 * copies on one shared stream.  set/get_fields take full-patch arrays (each
 * slab reads its rows and halos, writes back the rows it owns).  yy_step on
 * any member advances all. */
yy_status yy_create_slabs(const yy_grid* g, double R1, double R2, double Pr, double Ra, double dt,
                          int32_t nslab, yy_ctx** out);

#ifdef __cplusplus
}
#endif
#endif
