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
  double dr, dth, dph, R1;
  double tau, nu, kap, cchi, inv_chi, PrRa;
  double hatph;                   // 1/(R1^2 sin^2(theta_1) dph^2), theta_1 = pi/4 - delta (RD31)
  const double* rc;               // r centres  [nr]
  const double* rf;               // r faces    [nr+1]
  const double* sc;               // sin(theta centres) [nt]
  const double* sf;               // sin(theta faces)   [nt+1]
  const double* cc;               // cos(theta centres) [nt]
  const double* cf;               // cos(theta faces)   [nt+1]
};

__host__ __device__ __forceinline__ int NRk(const Geo& g, int K) { return g.nr + (K == KR); }
__host__ __device__ __forceinline__ int NTk(const Geo& g, int K) { return g.nt + (K == KT); }
__host__ __device__ __forceinline__ int NPk(const Geo& g, int K) { return g.np + (K == KP); }
__host__ __device__ __forceinline__ long long psize(const Geo& g, int K) {
  return (long long)NRk(g, K) * NTk(g, K) * NPk(g, K);
}
__host__ __device__ __forceinline__ long long wsize(const Geo& g, int K) {   // one wall (theta x phi)
  return (long long)NTk(g, K) * NPk(g, K);
}
template <int K>
__device__ __forceinline__ long long IX(const Geo& g, int i, int j, int k) {
  return ((long long)i * NTk(g, K) + j) * NPk(g, K) + k;
}

// Transport velocity a* = u2^{*,n+1/2} (RD8), one patch.
struct Astar {
  const double* __restrict__ ar;   // kind R
  const double* __restrict__ at;   // kind TH
  const double* __restrict__ ap;   // kind PH
};

// a*_r averaged to the nodes of kind K (average along every axis where the
// staggerings differ; SURVEY Appendix A "Advection").
template <int K>
__device__ __forceinline__ double abar_r(const Geo& g, const Astar& A, int i, int j, int k) {
  const double* a = A.ar;
  if (K == KR) return __ldg(a + IX<KR>(g, i, j, k));
  if (K == KC) return 0.5 * (__ldg(a + IX<KR>(g, i, j, k)) + __ldg(a + IX<KR>(g, i + 1, j, k)));
  if (K == KT)
    return 0.25 * (__ldg(a + IX<KR>(g, i, j - 1, k)) + __ldg(a + IX<KR>(g, i + 1, j - 1, k)) +
                   __ldg(a + IX<KR>(g, i, j, k)) + __ldg(a + IX<KR>(g, i + 1, j, k)));
  return 0.25 * (__ldg(a + IX<KR>(g, i, j, k - 1)) + __ldg(a + IX<KR>(g, i + 1, j, k - 1)) +
                 __ldg(a + IX<KR>(g, i, j, k)) + __ldg(a + IX<KR>(g, i + 1, j, k)));
}
template <int K>
__device__ __forceinline__ double abar_t(const Geo& g, const Astar& A, int i, int j, int k) {
  const double* a = A.at;
  if (K == KT) return __ldg(a + IX<KT>(g, i, j, k));
  if (K == KC) return 0.5 * (__ldg(a + IX<KT>(g, i, j, k)) + __ldg(a + IX<KT>(g, i, j + 1, k)));
  if (K == KR)
    return 0.25 * (__ldg(a + IX<KT>(g, i - 1, j, k)) + __ldg(a + IX<KT>(g, i - 1, j + 1, k)) +
                   __ldg(a + IX<KT>(g, i, j, k)) + __ldg(a + IX<KT>(g, i, j + 1, k)));
  return 0.25 * (__ldg(a + IX<KT>(g, i, j, k - 1)) + __ldg(a + IX<KT>(g, i, j + 1, k - 1)) +
                 __ldg(a + IX<KT>(g, i, j, k)) + __ldg(a + IX<KT>(g, i, j + 1, k)));
}
template <int K>
__device__ __forceinline__ double abar_p(const Geo& g, const Astar& A, int i, int j, int k) {
  const double* a = A.ap;
  if (K == KP) return __ldg(a + IX<KP>(g, i, j, k));
  if (K == KC) return 0.5 * (__ldg(a + IX<KP>(g, i, j, k)) + __ldg(a + IX<KP>(g, i, j, k + 1)));
  if (K == KR)
    return 0.25 * (__ldg(a + IX<KP>(g, i - 1, j, k)) + __ldg(a + IX<KP>(g, i - 1, j, k + 1)) +
                   __ldg(a + IX<KP>(g, i, j, k)) + __ldg(a + IX<KP>(g, i, j, k + 1)));
  return 0.25 * (__ldg(a + IX<KP>(g, i, j - 1, k)) + __ldg(a + IX<KP>(g, i, j - 1, k + 1)) +
                 __ldg(a + IX<KP>(g, i, j, k)) + __ldg(a + IX<KP>(g, i, j, k + 1)));
}

// Node coordinates of kind K.
template <int K> __device__ __forceinline__ double rnode(const Geo& g, int i) {
  return K == KR ? __ldg(g.rf + i) : __ldg(g.rc + i);
}
template <int K> __device__ __forceinline__ double snode(const Geo& g, int j) {
  return K == KT ? __ldg(g.sf + j) : __ldg(g.sc + j);
}
template <int K> __device__ __forceinline__ double cnode(const Geo& g, int j) {
  return K == KT ? __ldg(g.cf + j) : __ldg(g.cc + j);
}

// Row weights (am, a0, ap) of the directional operator L_{Q,AX} at node (i,j,k):
//   (L X)_n = am X_{n-e} + a0 X_n + ap X_{n+e}.
// HAT selects the implicit (split) operator with Delta^_thth, Delta^_phph
// versus the full Delta_thth, Delta_phph of the explicit L psi^*.
template <int Q, int AX, bool HAT>
__device__ __forceinline__ void coef(const Geo& g, const Astar& A, int i, int j, int k,
                                     double& am, double& a0, double& ap) {
  constexpr int K = kind_of(Q);
  const double D = (Q == QT) ? g.kap : g.nu;
  const double rn = rnode<K>(g, i);
  if (AX == 0) {
    // Delta_rr = (1/r^2) d_r(r^2 d_r), flux form; - a_r d_r
    double rm, rp;
    if (K == KR) { rm = __ldg(g.rc + i - 1); rp = __ldg(g.rc + i); }
    else { rm = __ldg(g.rf + i); rp = __ldg(g.rf + i + 1); }
    const double inv = 1.0 / (rn * rn * g.dr * g.dr);
    const double dm = D * rm * rm * inv, dp = D * rp * rp * inv;
    const double adv = abar_r<K>(g, A, i, j, k) * (0.5 / g.dr);
    am = dm + adv;
    ap = dp - adv;
    a0 = -(dm + dp);
    if (Q == QUR) {
      // nu(-2u/r^2 + (2/r^3) d_r(r^2 u)) (eq:r_comp L393) + c_chi D11 (RD11)
      const double fm = __ldg(g.rf + i - 1), fp = __ldg(g.rf + i + 1);
      const double cm = __ldg(g.rc + i - 1), cp = __ldg(g.rc + i);
      const double r3 = rn * rn * rn;
      a0 -= 2.0 * g.nu / (rn * rn);
      ap += g.nu * fp * fp / (r3 * g.dr);
      am -= g.nu * fm * fm / (r3 * g.dr);
      const double idr2 = 1.0 / (g.dr * g.dr);
      ap += g.cchi * fp * fp / (cp * cp) * idr2;
      am += g.cchi * fm * fm / (cm * cm) * idr2;
      a0 -= g.cchi * rn * rn * (1.0 / (cp * cp) + 1.0 / (cm * cm)) * idr2;
    }
  } else if (AX == 1) {
    // Delta_thth = (1/(rho^2 sin th)) d_th(sin th d_th), rho = R1 (hat) or r; - (a_th/r) d_th
    const double sn = snode<K>(g, j);
    double sm, sp;
    if (K == KT) { sm = __ldg(g.sc + j - 1); sp = __ldg(g.sc + j); }
    else { sm = __ldg(g.sf + j); sp = __ldg(g.sf + j + 1); }
    const double rho2 = HAT ? g.R1 * g.R1 : rn * rn;
    const double inv = D / (rho2 * sn * g.dth * g.dth);
    const double dm = sm * inv, dp = sp * inv;
    const double adv = abar_t<K>(g, A, i, j, k) * (0.5 / (rn * g.dth));
    am = dm + adv;
    ap = dp - adv;
    a0 = -(dm + dp);
    if (Q == QUT) {
      // nu(-u/(r^2 sin^2) + (2cos/(r^2 sin^2)) d_th(u sin)) (RD13) + c_chi D22 (RD11)
      // - (a_r/r) u (RD14)
      const double cn = cnode<K>(g, j);
      const double r2 = rn * rn;
      const double sfm = __ldg(g.sf + j - 1), sfp = __ldg(g.sf + j + 1);
      const double scm = __ldg(g.sc + j - 1), scp = __ldg(g.sc + j);
      a0 -= g.nu / (r2 * sn * sn);
      const double kk = g.nu * cn / (r2 * sn * sn * g.dth);
      ap += kk * sfp;
      am -= kk * sfm;
      const double idt2 = 1.0 / (r2 * g.dth * g.dth);
      ap += g.cchi * sfp / scp * idt2;
      am += g.cchi * sfm / scm * idt2;
      a0 -= g.cchi * sn * (1.0 / scp + 1.0 / scm) * idt2;
      a0 -= abar_r<K>(g, A, i, j, k) / rn;
    }
  } else {
    // Delta_phph = d_phph/(r^2 sin^2 th); hat: 1/(R1^2 sin^2 th_1); - (a_ph/(r sin th)) d_ph
    const double sn = snode<K>(g, j);
    const double c = HAT ? D * g.hatph : D / (rn * rn * sn * sn * g.dph * g.dph);
    const double adv = abar_p<K>(g, A, i, j, k) * (0.5 / (rn * sn * g.dph));
    am = c + adv;
    ap = c - adv;
    a0 = -2.0 * c;
    if (Q == QUP) {
      // nu(-u/(r^2 sin^2)) + c_chi D33 (RD12) - ((a_r + a_th cot)/r) u
      const double cn = cnode<K>(g, j);
      const double r2s2 = rn * rn * sn * sn;
      a0 -= g.nu / r2s2;
      const double c2 = g.cchi / (r2s2 * g.dph * g.dph);
      am += c2;
      ap += c2;
      a0 -= 2.0 * c2;
      a0 -= (abar_r<K>(g, A, i, j, k) + abar_t<K>(g, A, i, j, k) * cn / sn) / rn;
    }
  }
}

// Solved-node ranges of a kind (reading RD3): fringe = outermost theta/phi
// layer; u_r wall faces excluded.
template <int K> __device__ __forceinline__ int i_lo() { return K == KR ? 1 : 0; }
template <int K> __device__ __forceinline__ int i_hi(const Geo& g) { return K == KR ? g.nr - 1 : g.nr - 1; }

}  // namespace yy
