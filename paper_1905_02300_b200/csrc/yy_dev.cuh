// yy_dev.cuh — device-side layout and the directional operator rows of the
// Yin-Yang AC direction-splitting step (arXiv 1905.02300), sm_100a, fp64.
//
// Every kernel of the step derives its tridiagonal rows from coef<Q,AX,HAT>()
// below, so the residual (which applies L_split) and the line sweeps (which
// invert the factors I - tau/2 A_d) see bit-identical rows.  The rows are the
// operators of PAPER.md §3 (eq:Convect_Douglas L318-325, eq:r_comp L393-396,
// eq:theta_comp L415-419, eq:phi_comp L441-444) with the readings RD6-RD17 of
// DESIGN.md, discretised per SURVEY.md Appendix A (flux-form Laplacians,
// centred first differences, arithmetic averages of the transport velocity).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace yy {

enum Kind { KC = 0, KR = 1, KT = 2, KP = 3 };        // centres, r-, theta-, phi-faces
enum Quant { QT = 0, QUR = 1, QUT = 2, QUP = 3 };    // T, u_r, u_theta, u_phi

__host__ __device__ constexpr int kind_of(int q) { return q; }   // Quant -> Kind (same order)

// Geometry + physics, passed by value to every kernel.
struct Geo {
  int nr, nt, np;                 // cells per patch
  int npatch;                     // patches held by this context: 2 (both), 1 (one rank per patch)
  // local r-rows of this context (a radial slab keeps one halo row on each side;
  // the whole shell: ilo_c = 0, ihi_c = nr-1, ilo_f = 1, ihi_f = nr-1, walls both)
  int ilo_c, ihi_c;               // solved rows of r-centred kinds (C, TH, PH)
  int ilo_f, ihi_f;               // solved r-faces (u_r)
  int wall_lo, wall_hi;           // this context's rows touch r = R1 / r = R2
  int ifr_c0, ifr_c1, ifr_f0, ifr_f1;   // rows whose fringe nodes are interpolated
  double dr, dth, dph, R1;
  double tau, nu, kap, cchi, inv_chi, PrRa;
  double hatph;                   // 1/(R1^2 sin^2(theta_1) dph^2), theta_1 = pi/4 - delta (RD31)
  const double* rc;               // r centres  [nr]
  const double* rf;               // r faces    [nr+1]
  const double* sc;               // sin(theta centres) [nt]
  const double* sf;               // sin(theta faces)   [nt+1]
  const double* cc;               // cos(theta centres) [nt]
  const double* cf;               // cos(theta faces)   [nt+1]
  // reciprocals of the uniform spacings and the hat constant 1/R1^2
  double idr, idth, idph, idph2, iR1sq;
  // 1-D factor tables (host fp64): every row weight is a product of these,
  // so no kernel divides.  _c: nodes at cell centres, _f: nodes on faces.
  const double *ir_c, *ir2_c, *lr_cm, *lr_cp, *idv1_c;                  // [nr]
  const double *ir_f, *ir2_f, *lr_fm, *lr_fp, *mr_m, *mr_p, *d11_m, *d11_p, *d11_0, *rf2;   // [nr+1]
  const double *is_c, *is2_c, *cot_c, *lt_cm, *lt_cp;                    // [nt]
  const double *is_f, *is2_f, *cot_f, *lt_fm, *lt_fp, *mt_m, *mt_p, *d22_m, *d22_p, *d22_0;  // [nt+1]
  // a*-independent part of the split (hat) rows of every (quantity, axis):
  // [i][j][am, a0, ap] over the kind's (r, theta) nodes (k-independent), built once
  // on the device from coef<Q, AX, true, false> (yy_kernels.cu: k_build_split)
  const double* bsplit[4][3];
  // the same rows as the factor rows of I - tau/2 A without the transport /
  // reaction terms, [i][j][lo0, b0, up0] = (-tau/2 am, 1 - tau/2 a0, -tau/2 ap) of
  // coef<Q, AX, true, false> (the one-line-per-thread r / theta sweeps: a row is
  // lo0 - tau/2 adv, b0 + tau/2 rx, up0 + tau/2 adv)
  const double* tsplit[4][3];
  // per-step transport-velocity row weights by node kind and axis (k_adv; Astar::av)
  const double* adv[4][3];
};

// 1/x to full fp64 precision (<= 1 ulp): hardware approximation refined by two
// Newton steps.  Used for the Thomas / PCR pivots.
__device__ __forceinline__ double frcp(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}

__host__ __device__ __forceinline__ int NRk(const Geo& g, int K) { return g.nr + (K == KR); }
__host__ __device__ __forceinline__ int NTk(const Geo& g, int K) { return g.nt + (K == KT); }
__host__ __device__ __forceinline__ int NPk(const Geo& g, int K) { return g.np + (K == KP); }
__host__ __device__ __forceinline__ long long psize(const Geo& g, int K) {
  return (long long)NRk(g, K) * NTk(g, K) * NPk(g, K);
}
__host__ __device__ __forceinline__ long long wsize(const Geo& g, int K) {   // one wall (theta x phi)
  return (long long)NTk(g, K) * NPk(g, K);
}
// Offset of node (i,j,k) inside ONE patch's array of kind K.  32-bit: the
// largest per-patch array (C4, 257x385x1153) has 1.1e8 < 2^31 elements.
// All kinds are written through the cell-centre index c = (i nt + j) np + k so
// that the indices of one node in arrays of different kinds share it (CSE):
//   IX<KT> = (i (nt+1) + j) np + k = c + i np,  IX<KP> = (i nt + j)(np+1) + k = c + i nt + j.
template <int K>
__device__ __forceinline__ int IX(const Geo& g, int i, int j, int k) {
  const int c = (i * g.nt + j) * g.np + k;
  if (K == KT) return c + i * g.np;
  if (K == KP) return c + i * g.nt + j;
  return c;
}
// index strides of kind K along r (SR) and theta (ST); phi stride is 1
template <int K> __host__ __device__ __forceinline__ int SR(const Geo& g) { return NTk(g, K) * NPk(g, K); }
template <int K> __host__ __device__ __forceinline__ int ST(const Geo& g) { return NPk(g, K); }

// Block index of a kernel whose blocks may run in reverse linear order: the
// iteration alternates the order of consecutive kernels so that each starts on
// the tiles the previous one touched last (still in L2).  Every block computes
// the same tile either way (results are unchanged, bit for bit).
__device__ __forceinline__ uint3 bidx(int rev) {
  return rev ? make_uint3(gridDim.x - 1 - blockIdx.x, gridDim.y - 1 - blockIdx.y, gridDim.z - 1 - blockIdx.z)
             : blockIdx;
}

// Transport velocity a* = u2^{*,n+1/2} (RD8), one patch.
struct Astar {
  const double* __restrict__ ar;   // kind R
  const double* __restrict__ at;   // kind TH
  const double* __restrict__ ap;   // kind PH
  // the a*-reaction coefficients of the own-direction rows, evaluated once per step
  // (k_react): rt = abar_r<TH> / r at u_theta nodes (RD14), rp = (abar_r<PH> +
  // abar_t<PH> cot(theta)) / r at u_phi nodes
  const double* __restrict__ rt;
  const double* __restrict__ rp;
  // the transport-velocity row weights of the nodes of one kind, one per axis,
  // evaluated once per step (k_adv; Geo::adv): av[d] = abar_d<K> (0.5 / h_d) times
  // the axis' metric factor, i.e. the `adv` of coef<Q, d> (bind_adv)
  const double* __restrict__ av[3] = {};
};

// Astar::av of kind K for patch `patch` (the RX paths of coef / coef_split read them)
template <int K>
__device__ __forceinline__ void bind_adv(const Geo& g, Astar& A, int patch) {
  const long long o = patch * psize(g, K);
  A.av[0] = g.adv[K][0] + o;
  A.av[1] = g.adv[K][1] + o;
  A.av[2] = g.adv[K][2] + o;
}

// a*_r averaged to the nodes of kind K (average along every axis where the
// staggerings differ; SURVEY Appendix A "Advection").
template <int K>
__device__ __forceinline__ double abar_r(const Geo& g, const Astar& A, int i, int j, int k) {
  const double* a = A.ar + IX<KR>(g, i, j, k);
  const int sr = SR<KR>(g), st = ST<KR>(g);
  if (K == KR) return __ldg(a);
  if (K == KC) return 0.5 * (__ldg(a) + __ldg(a + sr));
  if (K == KT) return 0.25 * (__ldg(a - st) + __ldg(a + sr - st) + __ldg(a) + __ldg(a + sr));
  return 0.25 * (__ldg(a - 1) + __ldg(a + sr - 1) + __ldg(a) + __ldg(a + sr));
}
template <int K>
__device__ __forceinline__ double abar_t(const Geo& g, const Astar& A, int i, int j, int k) {
  const double* a = A.at + IX<KT>(g, i, j, k);
  const int sr = SR<KT>(g), st = ST<KT>(g);
  if (K == KT) return __ldg(a);
  if (K == KC) return 0.5 * (__ldg(a) + __ldg(a + st));
  if (K == KR) return 0.25 * (__ldg(a - sr) + __ldg(a - sr + st) + __ldg(a) + __ldg(a + st));
  return 0.25 * (__ldg(a - 1) + __ldg(a + st - 1) + __ldg(a) + __ldg(a + st));
}
template <int K>
__device__ __forceinline__ double abar_p(const Geo& g, const Astar& A, int i, int j, int k) {
  const double* a = A.ap + IX<KP>(g, i, j, k);
  const int sr = SR<KP>(g), st = ST<KP>(g);
  if (K == KP) return __ldg(a);
  if (K == KC) return 0.5 * (__ldg(a) + __ldg(a + 1));
  if (K == KR) return 0.25 * (__ldg(a - sr) + __ldg(a - sr + 1) + __ldg(a) + __ldg(a + 1));
  return 0.25 * (__ldg(a - st) + __ldg(a - st + 1) + __ldg(a) + __ldg(a + 1));
}

// Node coordinates and 1-D factors at the nodes of kind K.
template <int K> __device__ __forceinline__ double rnode(const Geo& g, int i) {
  return K == KR ? __ldg(g.rf + i) : __ldg(g.rc + i);
}
template <int K> __device__ __forceinline__ double snode(const Geo& g, int j) {
  return K == KT ? __ldg(g.sf + j) : __ldg(g.sc + j);
}
template <int K> __device__ __forceinline__ double irn(const Geo& g, int i) {    // 1/r
  return K == KR ? __ldg(g.ir_f + i) : __ldg(g.ir_c + i);
}
template <int K> __device__ __forceinline__ double ir2n(const Geo& g, int i) {   // 1/r^2
  return K == KR ? __ldg(g.ir2_f + i) : __ldg(g.ir2_c + i);
}
template <int K> __device__ __forceinline__ double isn(const Geo& g, int j) {    // 1/sin(theta)
  return K == KT ? __ldg(g.is_f + j) : __ldg(g.is_c + j);
}
template <int K> __device__ __forceinline__ double is2n(const Geo& g, int j) {   // 1/sin^2(theta)
  return K == KT ? __ldg(g.is2_f + j) : __ldg(g.is2_c + j);
}
template <int K> __device__ __forceinline__ double cotn(const Geo& g, int j) {   // cot(theta)
  return K == KT ? __ldg(g.cot_f + j) : __ldg(g.cot_c + j);
}

// Where the rows take the transport-velocity weight from the per-step arrays
// Astar::av (RX = RX_SWEEP: line sweeps, RX_RESID: residuals; bit 3 Q + AX of the
// masks) instead of averaging a* in place.  RX = 0 (static kernels): a* always.
// Defaults measured on B200 (C3): every residual / sweep except the T residual
// and the phi sweep of T, whose in-place average is as cheap.
enum { RX_NONE = 0, RX_SWEEP = 1, RX_RESID = 2, RX_GIVEN = 3 };   // GIVEN: adv / reaction passed in
#ifndef YY_AV_SWEEP
#define YY_AV_SWEEP 0xffb
#endif
#ifndef YY_AV_RESID
#define YY_AV_RESID 0xff8
#endif
__host__ __device__ constexpr bool use_av(int Q, int AX, int RX) {
  return RX == RX_SWEEP ? ((YY_AV_SWEEP >> (3 * Q + AX)) & 1) : RX == RX_RESID ? ((YY_AV_RESID >> (3 * Q + AX)) & 1) : false;
}

// Row weights (am, a0, ap) of the directional operator L_{Q,AX} at node (i,j,k):
//   (L X)_n = am X_{n-e} + a0 X_n + ap X_{n+e}.
// HAT selects the implicit (split) operator with Delta^_thth, Delta^_phph
// versus the full Delta_thth, Delta_phph of the explicit L psi^*.
// Weights are products of the 1-D tables of Geo (see yy_api.cu: host_tables).
// ADV = false: the transport-velocity terms left out (a* = 0), for the tables.
// RX: the reaction terms from the per-step arrays Astar::rt/rp (the sweeps) instead
// of from the a* averages (the residual and static kernels, which load those a*
// values for the other terms anyway).
template <int Q, int AX, bool HAT, bool ADV = true, int RX = 0>
__device__ __forceinline__ void coef(const Geo& g, const Astar& A, int i, int j, int k,
                                     double& am, double& a0, double& ap, double advin = 0.0) {
  constexpr int K = kind_of(Q);
  const double D = (Q == QT) ? g.kap : g.nu;
  if (AX == 0) {
    // Delta_rr = (1/r^2) d_r(r^2 d_r), flux form; - a_r d_r
    const double dm = D * (K == KR ? __ldg(g.lr_fm + i) : __ldg(g.lr_cm + i));
    const double dp = D * (K == KR ? __ldg(g.lr_fp + i) : __ldg(g.lr_cp + i));
    const double adv = !ADV ? 0.0 : RX == RX_GIVEN ? advin : use_av(Q, 0, RX) ? __ldg(A.av[0] + IX<K>(g, i, j, k)) : abar_r<K>(g, A, i, j, k) * (0.5 * g.idr);
    am = dm + adv;
    ap = dp - adv;
    a0 = -(dm + dp);
    if (Q == QUR) {
      // nu(-2u/r^2 + (2/r^3) d_r(r^2 u)) (eq:r_comp L393) + c_chi D11 (RD11)
      a0 -= 2.0 * g.nu * __ldg(g.ir2_f + i);
      ap += g.nu * __ldg(g.mr_p + i);
      am -= g.nu * __ldg(g.mr_m + i);
      ap += g.cchi * __ldg(g.d11_p + i);
      am += g.cchi * __ldg(g.d11_m + i);
      a0 -= g.cchi * __ldg(g.d11_0 + i);
    }
  } else if (AX == 1) {
    // Delta_thth = (1/(rho^2 sin th)) d_th(sin th d_th), rho = R1 (hat) or r; - (a_th/r) d_th
    const double rho = HAT ? g.iR1sq : ir2n<K>(g, i);
    const double dm = D * rho * (K == KT ? __ldg(g.lt_fm + j) : __ldg(g.lt_cm + j));
    const double dp = D * rho * (K == KT ? __ldg(g.lt_fp + j) : __ldg(g.lt_cp + j));
    const double adv = !ADV ? 0.0
                       : RX == RX_GIVEN ? advin
                       : use_av(Q, 1, RX) ? __ldg(A.av[1] + IX<K>(g, i, j, k))
                            : abar_t<K>(g, A, i, j, k) * (0.5 * g.idth) * irn<K>(g, i);
    am = dm + adv;
    ap = dp - adv;
    a0 = -(dm + dp);
    if (Q == QUT) {
      // nu(-u/(r^2 sin^2) + (2cos/(r^2 sin^2)) d_th(u sin)) (RD13) + c_chi D22 (RD11)
      // - (a_r/r) u (RD14)
      const double ir2 = __ldg(g.ir2_c + i);
      a0 -= g.nu * ir2 * __ldg(g.is2_f + j);
      ap += g.nu * ir2 * __ldg(g.mt_p + j);
      am -= g.nu * ir2 * __ldg(g.mt_m + j);
      ap += g.cchi * ir2 * __ldg(g.d22_p + j);
      am += g.cchi * ir2 * __ldg(g.d22_m + j);
      a0 -= g.cchi * ir2 * __ldg(g.d22_0 + j);
      if (ADV) a0 -= RX ? __ldg(A.rt + IX<KT>(g, i, j, k)) : abar_r<K>(g, A, i, j, k) * __ldg(g.ir_c + i);
    }
  } else {
    // Delta_phph = d_phph/(r^2 sin^2 th); hat: 1/(R1^2 sin^2 th_1); - (a_ph/(r sin th)) d_ph
    const double ir = irn<K>(g, i), is = isn<K>(g, j);
    const double c = HAT ? D * g.hatph : D * ir2n<K>(g, i) * is2n<K>(g, j) * g.idph2;
    const double adv = !ADV ? 0.0 : RX == RX_GIVEN ? advin : use_av(Q, 2, RX) ? __ldg(A.av[2] + IX<K>(g, i, j, k)) : abar_p<K>(g, A, i, j, k) * (0.5 * g.idph) * ir * is;
    am = c + adv;
    ap = c - adv;
    a0 = -2.0 * c;
    if (Q == QUP) {
      // nu(-u/(r^2 sin^2)) + c_chi D33 (RD12) - ((a_r + a_th cot)/r) u
      const double r2s2 = __ldg(g.ir2_c + i) * __ldg(g.is2_c + j);
      a0 -= g.nu * r2s2;
      const double c2 = g.cchi * r2s2 * g.idph2;
      am += c2;
      ap += c2;
      a0 -= 2.0 * c2;
      if (ADV)
        a0 -= RX ? __ldg(A.rp + IX<KP>(g, i, j, k))
                 : (abar_r<K>(g, A, i, j, k) + abar_t<K>(g, A, i, j, k) * __ldg(g.cot_c + j)) * __ldg(g.ir_c + i);
    }
  }
}

// The split (hat) rows of L_{Q,AX} at node (i,j,k) = the tabulated a*-independent
// part (Geo::bsplit) + the transport-velocity terms: the same rows as
// coef<Q,AX,true> up to the order of the additions, with 3 table loads instead of
// the 1-D factor products.
template <int Q, int AX, int RX = 0>
__device__ __forceinline__ void coef_split(const Geo& g, const Astar& A, int i, int j, int k,
                                           double& am, double& a0, double& ap, double advin = 0.0,
                                           double rxin = 0.0) {
  constexpr int K = kind_of(Q);
  // tabulated only where the own-direction row carries the metric / grad-div
  // terms (u_r in r, u_th in theta, u_ph in phi); measured on B200 (C3), the
  // plain Laplacian rows are cheaper from the 1-D factors
  if constexpr (!((Q == QUR && AX == 0) || (Q == QUT && AX == 1) || (Q == QUP && AX == 2))) {
    coef<Q, AX, true, true, RX>(g, A, i, j, k, am, a0, ap, advin);
    return;
  }
  const double* b = g.bsplit[Q][AX] + 3 * (i * NTk(g, K) + j);
  am = __ldg(b);
  a0 = __ldg(b + 1);
  ap = __ldg(b + 2);
  double adv;
  if (RX == RX_GIVEN) {
    adv = advin;
    if ((AX == 1 && Q == QUT) || (AX == 2 && Q == QUP)) a0 -= rxin;
  } else if (use_av(Q, AX, RX)) {
    adv = __ldg(A.av[AX] + IX<K>(g, i, j, k));
    if (AX == 1 && Q == QUT) a0 -= __ldg(A.rt + IX<KT>(g, i, j, k));
    if (AX == 2 && Q == QUP) a0 -= __ldg(A.rp + IX<KP>(g, i, j, k));
  } else if (AX == 0) {
    adv = abar_r<K>(g, A, i, j, k) * (0.5 * g.idr);
  } else if (AX == 1) {
    adv = abar_t<K>(g, A, i, j, k) * (0.5 * g.idth) * irn<K>(g, i);
    if (Q == QUT) a0 -= RX ? __ldg(A.rt + IX<KT>(g, i, j, k)) : abar_r<K>(g, A, i, j, k) * __ldg(g.ir_c + i);
  } else {
    adv = abar_p<K>(g, A, i, j, k) * (0.5 * g.idph) * irn<K>(g, i) * isn<K>(g, j);
    if (Q == QUP)
      a0 -= RX ? __ldg(A.rp + IX<KP>(g, i, j, k))
               : (abar_r<K>(g, A, i, j, k) + abar_t<K>(g, A, i, j, k) * __ldg(g.cot_c + j)) * __ldg(g.ir_c + i);
  }
  am += adv;
  ap -= adv;
}

// Solved-node ranges of a kind (reading RD3): fringe = outermost theta/phi
// layer; u_r wall faces excluded.
template <int K> __host__ __device__ __forceinline__ int i_lo(const Geo& g) { return K == KR ? g.ilo_f : g.ilo_c; }
template <int K> __host__ __device__ __forceinline__ int i_hi(const Geo& g) { return K == KR ? g.ihi_f : g.ihi_c; }

}  // namespace yy
