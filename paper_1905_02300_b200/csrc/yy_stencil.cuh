// yy_stencil.cuh — MAC stencils shared by the per-step kernels (yy_kernels.cu)
// and the fused residual of the first line sweep (yy_line.cu): 7-point stars
// with the wall ghost (RD22), sum_d L_{Q,d} (rows of coef<>), divergence pieces
// and the eq:er residual of one node (sign RD9).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "yy_dev.cuh"
#include "yy_internal.h"

namespace yy {

// ---------------------------------------------------------------------------------
// small helpers
// ---------------------------------------------------------------------------------
struct Star {   // 7-point star of a field at a node; x = r, y = theta, z = phi
  double c, xm, xp, ym, yp, zm, zp;
};

__device__ __forceinline__ Star star_lin(const Star& a, double fa, const Star& b, double fb) {
  Star s;
  s.c = fa * a.c + fb * b.c;
  s.xm = fa * a.xm + fb * b.xm;
  s.xp = fa * a.xp + fb * b.xp;
  s.ym = fa * a.ym + fb * b.ym;
  s.yp = fa * a.yp + fb * b.yp;
  s.zm = fa * a.zm + fb * b.zm;
  s.zp = fa * a.zp + fb * b.zp;
  return s;
}

// Star of field F (one patch) at (i,j,k).  For r-centred kinds the r
// neighbours beyond the walls are the ghosts 2 w - psi_0 (reading RD22),
// W = the field's wall data (2, NT, NP) at the matching time level.
// WALL = false: the caller knows (i,j,k) is no wall-adjacent node (no ghost code).
template <int K, bool WALL = true>
__device__ __forceinline__ Star load_star(const Geo& g, const double* __restrict__ F,
                                          const double* __restrict__ W, int i, int j, int k) {
  // read-only (non-coherent) loads: no kernel that calls this writes F or W
  // one base pointer per node, neighbours at +-1 (immediate), +-st, +-sr
  Star s;
  const double* p = F + IX<K>(g, i, j, k);
  const int sr = SR<K>(g), st = ST<K>(g);
  s.c = __ldg(p);
  if (WALL && K != KR && g.wall_lo && i == g.ilo_c) s.xm = 2.0 * __ldg(W + j * NPk(g, K) + k) - s.c;
  else s.xm = __ldg(p - sr);
  if (WALL && K != KR && g.wall_hi && i == g.ihi_c) s.xp = 2.0 * __ldg(W + wsize(g, K) + j * NPk(g, K) + k) - s.c;
  else s.xp = __ldg(p + sr);
  s.ym = __ldg(p - st);
  s.yp = __ldg(p + st);
  s.zm = __ldg(p - 1);
  s.zp = __ldg(p + 1);
  return s;
}

// sum_d L_{Q,d} applied to a star.  RX: transport-velocity and reaction weights
// from the per-step arrays (Astar::av / rt / rp, bound by the caller).
template <int Q, bool HAT, int RX = RX_NONE>
__device__ __forceinline__ double applyL(const Geo& g, const Astar& A, int i, int j, int k, const Star& s) {
  double am, a0, ap, acc;
  if (HAT) coef_split<Q, 0, RX>(g, A, i, j, k, am, a0, ap);
  else coef<Q, 0, false, true, RX>(g, A, i, j, k, am, a0, ap);
  acc = am * s.xm + a0 * s.c + ap * s.xp;
  if (HAT) coef_split<Q, 1, RX>(g, A, i, j, k, am, a0, ap);
  else coef<Q, 1, false, true, RX>(g, A, i, j, k, am, a0, ap);
  acc += am * s.ym + a0 * s.c + ap * s.yp;
  if (HAT) coef_split<Q, 2, RX>(g, A, i, j, k, am, a0, ap);
  else coef<Q, 2, false, true, RX>(g, A, i, j, k, am, a0, ap);
  acc += am * s.zm + a0 * s.c + ap * s.zp;
  return acc;
}

template <int K>
__device__ __forceinline__ bool solved(const Geo& g, int i, int j, int k) {
  return i >= i_lo<K>(g) && i <= i_hi<K>(g) && j >= 1 && j <= NTk(g, K) - 2 && k >= 1 && k <= NPk(g, K) - 2;
}

// divergence contributions at cell centre (i,j,k) of one patch
__device__ __forceinline__ double div1(const Geo& g, const double* ur, int i, int j, int k) {
  return (__ldg(g.rf2 + i + 1) * ur[IX<KR>(g, i + 1, j, k)] - __ldg(g.rf2 + i) * ur[IX<KR>(g, i, j, k)]) *
         __ldg(g.idv1_c + i);
}
__device__ __forceinline__ double div2(const Geo& g, const double* ut, int i, int j, int k) {
  return (__ldg(g.sf + j + 1) * ut[IX<KT>(g, i, j + 1, k)] - __ldg(g.sf + j) * ut[IX<KT>(g, i, j, k)]) *
         (__ldg(g.ir_c + i) * __ldg(g.is_c + j) * g.idth);
}
__device__ __forceinline__ double div3(const Geo& g, const double* up, int i, int j, int k) {
  return (up[IX<KP>(g, i, j, k + 1)] - up[IX<KP>(g, i, j, k)]) * (__ldg(g.ir_c + i) * __ldg(g.is_c + j) * g.idph);
}

// eq:er residual (sign RD9) at solved node (i,j,k) of patch `patch`:
//   R = G + tau E_dyn - (I - tau/2 L_split)(psi~ - psi^n)
// with the Gauss-Seidel dynamic terms E_dyn of SURVEY §8(c) O7/O9 (RD20, RD21,
// RD18, RD-E1).
template <int Q, int S, bool WALL = true, bool NOADV = false>
__device__ __forceinline__ double resid_at(const Geo& g, const ResidArgs& a, int patch, int i, int j, int k) {
  constexpr int K = kind_of(Q);
  const long long po = patch * psize(g, K);
  const long long pc = patch * psize(g, KC);
  const int node = IX<K>(g, i, j, k);
  Astar A{a.ar + patch * psize(g, KR), a.at + patch * psize(g, KT), a.ap + patch * psize(g, KP),
          a.rt + patch * psize(g, KT), a.rp + patch * psize(g, KP)};
  bind_adv<K>(g, A, patch);
  const double* Wnew = a.wnew ? a.wnew + patch * 2 * wsize(g, K) : nullptr;
  const double* Wn = a.wn ? a.wn + patch * 2 * wsize(g, K) : nullptr;
  Star x1 = load_star<K, WALL>(g, a.it + po, Wnew, i, j, k);
  Star x0 = load_star<K, WALL>(g, a.n + po, Wn, i, j, k);
  Star X = star_lin(x1, 1.0, x0, -1.0);
  double E = 0.0;
  if (Q == QUR) {
    // buoyancy +Pr Ra T^{n+1/2,(k)} e_r (RD20, RD21)
    const int c0 = IX<KC>(g, i, j, k), src = SR<KC>(g);
    const double* Ti = a.Tit + pc + c0;
    const double* Tn = a.Tn + pc + c0;
    const double tb0 = 0.5 * (__ldg(Ti - src) + __ldg(Tn - src));
    const double tb1 = 0.5 * (__ldg(Ti) + __ldg(Tn));
    E = g.PrRa * 0.5 * (tb0 + tb1);
  } else if (Q == QUT) {
    // c_chi D21 ub_r + nu((2/r^2) d_th ub_r + (2 cos/(r^3 sin)) d_r(r^2 ub_r))  (eq:theta_comp)
    const long long orr = patch * psize(g, KR);
    const int q0 = IX<KR>(g, i, j, k), srr = SR<KR>(g), str = ST<KR>(g);
    const double *uri = a.urit + orr + q0, *urn = a.urn + orr + q0;
    auto ub = [&](int ii, int jj) {     // (ii, jj) in {i, i+1} x {j-1, j}
      const int q = (ii - i) * srr + (jj - j) * str;
      return 0.5 * (__ldg(uri + q) + __ldg(urn + q));
    };
    const double f0 = __ldg(g.rf2 + i), f1 = __ldg(g.rf2 + i + 1), iv = __ldg(g.idv1_c + i);
    auto d1 = [&](int jj) { return (f1 * ub(i + 1, jj) - f0 * ub(i, jj)) * iv; };
    const double ir = __ldg(g.ir_c + i);
    const double d1a = d1(j - 1), d1b = d1(j);
    E = g.cchi * (d1b - d1a) * (ir * g.idth);
    E += g.nu * (2.0 * ir * ir) * 0.5 * ((ub(i, j) - ub(i, j - 1)) + (ub(i + 1, j) - ub(i + 1, j - 1))) * g.idth;
    E += g.nu * (2.0 * __ldg(g.cot_f + j) * ir) * 0.5 * (d1a + d1b);
  } else if (Q == QUP) {
    // c_chi (D31 ub_r + D32 ub_th) + nu((2/(r^2 sin)) d_ph ub_r + (2cos/(r^2 sin^2)) d_ph ub_th)
    const long long orr = patch * psize(g, KR), ot = patch * psize(g, KT);
    const int qr = IX<KR>(g, i, j, k), qt = IX<KT>(g, i, j, k), srr = SR<KR>(g), stt = ST<KT>(g);
    const double *uri = a.urit + orr + qr, *urn = a.urn + orr + qr, *uti = a.utit + ot + qt, *utn = a.utn + ot + qt;
    auto ubr = [&](int ii, int kk) {    // (ii, kk) in {i, i+1} x {k-1, k}
      const int q = (ii - i) * srr + (kk - k);
      return 0.5 * (__ldg(uri + q) + __ldg(urn + q));
    };
    auto ubt = [&](int jj, int kk) {    // (jj, kk) in {j, j+1} x {k-1, k}
      const int q = (jj - j) * stt + (kk - k);
      return 0.5 * (__ldg(uti + q) + __ldg(utn + q));
    };
    const double ir = __ldg(g.ir_c + i), is = __ldg(g.is_c + j), ct = __ldg(g.cot_c + j);
    const double f0 = __ldg(g.rf2 + i), f1 = __ldg(g.rf2 + i + 1), iv = __ldg(g.idv1_c + i);
    const double s0 = __ldg(g.sf + j), s1 = __ldg(g.sf + j + 1);
    const double rsdt = ir * is * g.idth;
    auto e = [&](int kk) {
      const double dd1 = (f1 * ubr(i + 1, kk) - f0 * ubr(i, kk)) * iv;
      const double dd2 = (s1 * ubt(j + 1, kk) - s0 * ubt(j, kk)) * rsdt;
      return dd1 + dd2;
    };
    const double rsdp = ir * is * g.idph;
    E = g.cchi * (e(k) - e(k - 1)) * rsdp;
    E += g.nu * (2.0 * ir * rsdp) * 0.5 * ((ubr(i, k) - ubr(i, k - 1)) + (ubr(i + 1, k) - ubr(i + 1, k - 1)));
    E += g.nu * (2.0 * ct * ir * rsdp) * 0.5 * ((ubt(j, k) - ubt(j, k - 1)) + (ubt(j + 1, k) - ubt(j + 1, k - 1)));
  }
  if (S == 2 && Q != QT) {
    // -1/2 grad(p1^(k) - p1^n)   (RD18)
    const int c0 = IX<KC>(g, i, j, k);
    const double *pi_ = a.p1it + pc + c0, *pn = a.p1n + pc + c0;
    const double* d1 = a.dp1 ? a.dp1 + pc + c0 : nullptr;
    auto dp = [&](int ii, int jj, int kk) {     // p1^(k) - p1^n (stored once by k_pres<1>, or formed here)
      const int q = (ii - i) * SR<KC>(g) + (jj - j) * ST<KC>(g) + (kk - k);
      return d1 ? __ldg(d1 + q) : __ldg(pi_ + q) - __ldg(pn + q);
    };
    if (Q == QUR) E -= 0.5 * (dp(i, j, k) - dp(i - 1, j, k)) * g.idr;
    if (Q == QUT) E -= 0.5 * (dp(i, j, k) - dp(i, j - 1, k)) * (__ldg(g.ir_c + i) * g.idth);
    if (Q == QUP) E -= 0.5 * (dp(i, j, k) - dp(i, j, k - 1)) * (__ldg(g.ir_c + i) * __ldg(g.is_c + j) * g.idph);
  }
  // IMEX (NOADV): the split rows without transport terms, no per-step weight read
  const double LX = NOADV ? applyL<Q, true, RX_GIVEN>(g, A, i, j, k, X) : applyL<Q, true, RX_RESID>(g, A, i, j, k, X);
  return __ldg(a.G + po + node) + g.tau * E - (X.c - 0.5 * g.tau * LX);
}

}  // namespace yy
