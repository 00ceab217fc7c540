// yy_kernels.cu — sm_100a fp64 kernels of one Yin-Yang AC direction-splitting
// time step (arXiv 1905.02300).  Launch wrappers at the bottom are called by
// yy_api.cu.  Every step of the hot path runs here; the host only sequences
// launches.
//
// Kernels (SURVEY.md §2.2 naming):
//   K0  k_static<Q>      per-step static RHS G_q (O3), both systems fused
//   K1  k_resid<Q,S>     eq:er residual R = G + tau E_dyn - (I - tau/2 L_split)(psi~ - psi^n)
//   K2/K3 k_sweep<Q,AX,F> batched Thomas along AX, rows from coef<> (one line per thread)
//   K5  k_interp_*       Yin<->Yang fringe interpolation (4x4 Lagrange, rotation)
//   K6  k_reduce         deterministic Schwarz residual reduction
//   K7  k_pres<S>        pressure updates eq:nst_Mass1 / eq:ac2 (RD18)
#include <cuda_runtime.h>
#include <stdint.h>

#include "yy_dev.cuh"
#include "yy_internal.h"

#ifndef YY_BWD_PREFETCH
#define YY_BWD_PREFETCH 1
#endif

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
template <int K>
__device__ __forceinline__ Star load_star(const Geo& g, const double* __restrict__ F,
                                          const double* __restrict__ W, int i, int j, int k) {
  Star s;
  s.c = F[IX<K>(g, i, j, k)];
  if (K != KR && i == 0) s.xm = 2.0 * W[(long long)j * NPk(g, K) + k] - s.c;
  else s.xm = F[IX<K>(g, i - 1, j, k)];
  if (K != KR && i == g.nr - 1) s.xp = 2.0 * W[wsize(g, K) + (long long)j * NPk(g, K) + k] - s.c;
  else s.xp = F[IX<K>(g, i + 1, j, k)];
  s.ym = F[IX<K>(g, i, j - 1, k)];
  s.yp = F[IX<K>(g, i, j + 1, k)];
  s.zm = F[IX<K>(g, i, j, k - 1)];
  s.zp = F[IX<K>(g, i, j, k + 1)];
  return s;
}

// sum_d L_{Q,d} applied to a star.
template <int Q, bool HAT>
__device__ __forceinline__ double applyL(const Geo& g, const Astar& A, int i, int j, int k, const Star& s) {
  double am, a0, ap, acc;
  coef<Q, 0, HAT>(g, A, i, j, k, am, a0, ap);
  acc = am * s.xm + a0 * s.c + ap * s.xp;
  coef<Q, 1, HAT>(g, A, i, j, k, am, a0, ap);
  acc += am * s.ym + a0 * s.c + ap * s.yp;
  coef<Q, 2, HAT>(g, A, i, j, k, am, a0, ap);
  acc += am * s.zm + a0 * s.c + ap * s.zp;
  return acc;
}

template <int K>
__device__ __forceinline__ bool solved(const Geo& g, int i, int j, int k) {
  return i >= i_lo<K>() && i <= i_hi<K>(g) && j >= 1 && j <= NTk(g, K) - 2 && k >= 1 && k <= NPk(g, K) - 2;
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

__device__ __forceinline__ void pf_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

__device__ __forceinline__ double omega(const Geo& g, double r, double s) {
  return r * r * s * g.dr * g.dth * g.dph;
}

// deterministic block sum (fixed thread -> data assignment, fixed tree);
// blockDim.x <= NT_, multiple of 32
template <int NT_>
__device__ __forceinline__ double block_sum(double v) {
  __shared__ double sh[NT_ / 32];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  if (l == 0) sh[w] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int q = 0; q < (int)(blockDim.x / 32); ++q) t += sh[q];
  return t;   // valid in thread 0
}

// ---------------------------------------------------------------------------------
// elementwise
// ---------------------------------------------------------------------------------
// out = sum_m c[m] * in[m]   (a* extrapolation O2, wall/time-basis evaluation)
__global__ void k_lincomb(double* __restrict__ out, long long n, int nin, LinIn in) {
  long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (; idx < n; idx += stride) {
    double v = 0.0;
    for (int m = 0; m < nin; ++m) v += in.c[m] * in.p[m][idx];
    out[idx] = v;
  }
}

// ---------------------------------------------------------------------------------
// K0: static right-hand side G (O3):  G = tau [L_full psi^* - 1/2 L_split (psi^n - psi^{n-1}) + E_static]
// grid: x -> k, y -> j, z -> patch * NR + i
// ---------------------------------------------------------------------------------
template <int Q>
__global__ void __launch_bounds__(128) k_static(Geo g, StaticArgs a) {
  constexpr int K = kind_of(Q);
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y;
  const int patch = blockIdx.z / NRk(g, K);
  const int i = blockIdx.z % NRk(g, K);
  if (k >= NPk(g, K) || !solved<K>(g, i, j, k)) return;
  const long long po = patch * psize(g, K);
  const long long pc = patch * psize(g, KC);
  const int node = IX<K>(g, i, j, k);
  Astar A{a.ar + patch * psize(g, KR), a.at + patch * psize(g, KT), a.ap + patch * psize(g, KP)};
  const double* Wn = a.wn ? a.wn + patch * 2 * wsize(g, K) : nullptr;
  const double* Wm = a.wm ? a.wm + patch * 2 * wsize(g, K) : nullptr;
  double src = 0.0;
  for (int m = 0; m < a.nsrc[patch]; ++m) src += a.gsrc[patch][m] * a.src[patch][m][node];

  const double rn = rnode<K>(g, i);
  const int nsys = (Q == QT) ? 1 : 2;
  for (int s = 0; s < nsys; ++s) {
    Star n = load_star<K>(g, a.fn[s] + po, Wn, i, j, k);
    Star m = load_star<K>(g, a.fm[s] + po, Wm, i, j, k);
    Star S = star_lin(n, 1.5, m, -0.5);
    Star D = star_lin(n, 1.0, m, -1.0);
    double E = src;
    if (Q != QT) {
      const double* p = a.p[s] + pc;
      const double* uts = nullptr;
      if (Q == QUR) {
        // -d_r p^n + c_chi d_r(div2 u_th^* + div3 u_ph^*) + (a_th^2 + a_ph^2)/r   (eq:r_comp, RD17)
        const long long ot = patch * psize(g, KT), op = patch * psize(g, KP);
        const double *utn = a.utn[s] + ot, *utm = a.utm[s] + ot, *upn = a.upn[s] + op, *upm = a.upm[s] + op;
        auto dd = [&](int ii) {
          const double d2 = 1.5 * div2(g, utn, ii, j, k) - 0.5 * div2(g, utm, ii, j, k);
          const double d3 = 1.5 * div3(g, upn, ii, j, k) - 0.5 * div3(g, upm, ii, j, k);
          return d2 + d3;
        };
        E += -(p[IX<KC>(g, i, j, k)] - p[IX<KC>(g, i - 1, j, k)]) * g.idr;
        E += g.cchi * (dd(i) - dd(i - 1)) * g.idr;
        const double at_ = abar_t<KR>(g, A, i, j, k), ap_ = abar_p<KR>(g, A, i, j, k);
        E += (at_ * at_ + ap_ * ap_) * __ldg(g.ir_f + i);
        (void)uts;
      } else if (Q == QUT) {
        // -(1/r) d_th p^n + c_chi (1/r) d_th(div3 u_ph^*) + a_ph^2 cot(th)/r   (eq:theta_comp, RD14)
        const long long op = patch * psize(g, KP);
        const double *upn = a.upn[s] + op, *upm = a.upm[s] + op;
        const double d3 = 1.5 * div3(g, upn, i, j, k) - 0.5 * div3(g, upm, i, j, k);
        const double d3m = 1.5 * div3(g, upn, i, j - 1, k) - 0.5 * div3(g, upm, i, j - 1, k);
        const double irdt = __ldg(g.ir_c + i) * g.idth;
        E += -(p[IX<KC>(g, i, j, k)] - p[IX<KC>(g, i, j - 1, k)]) * irdt;
        E += g.cchi * (d3 - d3m) * irdt;
        const double ap_ = abar_p<KT>(g, A, i, j, k);
        E += ap_ * ap_ * __ldg(g.cot_f + j) * __ldg(g.ir_c + i);
      } else {
        // -(1/(r sin th)) d_ph p^n   (eq:phi_comp)
        E += -(p[IX<KC>(g, i, j, k)] - p[IX<KC>(g, i, j, k - 1)]) * (__ldg(g.ir_c + i) * __ldg(g.is_c + j) * g.idph);
      }
    }
    const double Lf = applyL<Q, false>(g, A, i, j, k, S);
    const double Ls = applyL<Q, true>(g, A, i, j, k, D);
    a.G[s][po + node] = g.tau * (Lf - 0.5 * Ls + E);
  }
}

// ---------------------------------------------------------------------------------
// K1: residual of eq:er (sign RD9) with the Gauss-Seidel dynamic terms
// ---------------------------------------------------------------------------------
template <int Q, int S>
__global__ void __launch_bounds__(128) k_resid(Geo g, ResidArgs a) {
  constexpr int K = kind_of(Q);
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y;
  const int patch = blockIdx.z / NRk(g, K);
  const int i = blockIdx.z % NRk(g, K);
  if (k >= NPk(g, K) || !solved<K>(g, i, j, k)) return;
  const long long po = patch * psize(g, K);
  const long long pc = patch * psize(g, KC);
  const int node = IX<K>(g, i, j, k);
  Astar A{a.ar + patch * psize(g, KR), a.at + patch * psize(g, KT), a.ap + patch * psize(g, KP)};
  const double* Wnew = a.wnew ? a.wnew + patch * 2 * wsize(g, K) : nullptr;
  const double* Wn = a.wn ? a.wn + patch * 2 * wsize(g, K) : nullptr;
  Star x1 = load_star<K>(g, a.it + po, Wnew, i, j, k);
  Star x0 = load_star<K>(g, a.n + po, Wn, i, j, k);
  Star X = star_lin(x1, 1.0, x0, -1.0);
  const double rn = rnode<K>(g, i);
  double E = 0.0;
  if (Q == QUR) {
    // buoyancy +Pr Ra T^{n+1/2,(k)} e_r (RD20, RD21)
    const double* Ti = a.Tit + pc;
    const double* Tn = a.Tn + pc;
    const double tb0 = 0.5 * (Ti[IX<KC>(g, i - 1, j, k)] + Tn[IX<KC>(g, i - 1, j, k)]);
    const double tb1 = 0.5 * (Ti[IX<KC>(g, i, j, k)] + Tn[IX<KC>(g, i, j, k)]);
    E = g.PrRa * 0.5 * (tb0 + tb1);
  } else if (Q == QUT) {
    // c_chi D21 ub_r + nu((2/r^2) d_th ub_r + (2 cos/(r^3 sin)) d_r(r^2 ub_r))  (eq:theta_comp)
    const long long orr = patch * psize(g, KR);
    const double *uri = a.urit + orr, *urn = a.urn + orr;
    auto ub = [&](int ii, int jj) {
      const long long q = IX<KR>(g, ii, jj, k);
      return 0.5 * (uri[q] + urn[q]);
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
    const double *uri = a.urit + orr, *urn = a.urn + orr, *uti = a.utit + ot, *utn = a.utn + ot;
    auto ubr = [&](int ii, int kk) {
      const long long q = IX<KR>(g, ii, j, kk);
      return 0.5 * (uri[q] + urn[q]);
    };
    auto ubt = [&](int jj, int kk) {
      const long long q = IX<KT>(g, i, jj, kk);
      return 0.5 * (uti[q] + utn[q]);
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
    const double *pi_ = a.p1it + pc, *pn = a.p1n + pc;
    auto dp = [&](int ii, int jj, int kk) {
      const long long q = IX<KC>(g, ii, jj, kk);
      return pi_[q] - pn[q];
    };
    if (Q == QUR) E -= 0.5 * (dp(i, j, k) - dp(i - 1, j, k)) * g.idr;
    if (Q == QUT) E -= 0.5 * (dp(i, j, k) - dp(i, j - 1, k)) * (__ldg(g.ir_c + i) * g.idth);
    if (Q == QUP) E -= 0.5 * (dp(i, j, k) - dp(i, j, k - 1)) * (__ldg(g.ir_c + i) * __ldg(g.is_c + j) * g.idph);
  }
  const double LX = applyL<Q, true>(g, A, i, j, k, X);
  a.R[po + node] = a.G[po + node] + g.tau * E - (X.c - 0.5 * g.tau * LX);
}

// ---------------------------------------------------------------------------------
// K2/K3: Thomas along AX for every line (one line per thread).  Rows
// (I - tau/2 A_{Q,AX}) from coef<Q,AX,true>; homogeneous Dirichlet increments at
// fringe / u_r wall faces; antisymmetric wall ghost for r-centred kinds (RD23).
// In place on R (d' then x); c' in scratch C.  FINAL: psi += x and norm partial.
// Line grid: AX=0: x -> k, y -> j;  AX=1: x -> k, y -> i;  AX=2: x -> j, y -> i.  z -> patch.
// ---------------------------------------------------------------------------------

template <int Q, int AX, bool FINAL, bool SMC>
__global__ void __launch_bounds__(128, (AX == 1) ? 4 : 7) k_sweep(Geo g, SweepArgs a) {
  // rows per load round (measured on B200, C3: 4 best for r-lines, 8 for theta-lines)
  constexpr int SB = (AX == 0) ? 4 : 8;
  extern __shared__ double csm[];   // SMC: c' column of this thread at csm[m * blockDim.x + threadIdx.x]
  constexpr int K = kind_of(Q);
  const int patch = blockIdx.z;
  int i = 0, j = 0, k = 0, n = 0;
  long long stride = 0;
  const int tx = blockIdx.x * blockDim.x + threadIdx.x;
  bool valid;
  if (AX == 0) {
    k = tx + 1; j = blockIdx.y + 1; i = i_lo<K>();
    valid = k <= NPk(g, K) - 2;
    n = i_hi<K>(g) - i_lo<K>() + 1;
    stride = (long long)NTk(g, K) * NPk(g, K);
  } else if (AX == 1) {
    k = tx + 1; i = blockIdx.y + i_lo<K>(); j = 1;
    valid = k <= NPk(g, K) - 2;
    n = NTk(g, K) - 2;
    stride = NPk(g, K);
  } else {
    j = tx + 1; i = blockIdx.y + i_lo<K>(); k = 1;
    valid = j <= NTk(g, K) - 2;
    n = NPk(g, K) - 2;
    stride = 1;
  }
  double wsum = 0.0;
  if (valid) {
    const long long po = patch * psize(g, K);
    Astar A{a.ar + patch * psize(g, KR), a.at + patch * psize(g, KT), a.ap + patch * psize(g, KP)};
    double* __restrict__ R = a.R + po;
    double* __restrict__ C = a.C + po;
    const long long base = IX<K>(g, i, j, k);
    auto cidx = [&](int m) -> long long {
      return SMC ? (long long)m * blockDim.x + threadIdx.x : base + m * stride;
    };
    double* __restrict__ Cs = SMC ? csm : C;
    const double th = 0.5 * g.tau;
    double cprev = 0.0, dprev = 0.0;
    // forward elimination, 4 rows per round: the round's loads (rhs and the
    // read-only a* / table loads inside coef) are all issued before use
    // L2 prefetch distance (rows) for the inputs of the next rounds
    const double* pfa = (AX == 0) ? A.ar : A.at;
    const int pko = (AX == 0) ? IX<KR>(g, i, j, k) : IX<KT>(g, i, j, k);
    const long long pst = (AX == 0) ? (long long)g.nt * g.np : (long long)g.np;
    for (int m0 = 0; m0 < n; m0 += SB) {
#pragma unroll
      for (int u = 0; u < SB; ++u) {
        const int mp = m0 + 2 * SB + u;
        if (mp < n) {
          pf_l2(R + base + mp * stride);
          pf_l2(pfa + pko + mp * pst);
        }
      }
      double rv[SB], am[SB], a0[SB], ap[SB];
#pragma unroll
      for (int u = 0; u < SB; ++u) rv[u] = (m0 + u < n) ? R[base + (m0 + u) * stride] : 0.0;
#pragma unroll
      for (int u = 0; u < SB; ++u) {
        const int m = m0 + u;
        if (m < n) {
          const int ii = (AX == 0) ? i + m : i, jj = (AX == 1) ? j + m : j, kk = (AX == 2) ? k + m : k;
          coef<Q, AX, true>(g, A, ii, jj, kk, am[u], a0[u], ap[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < SB; ++u) {
        const int m = m0 + u;
        if (m < n) {
          double di = 1.0 - th * a0[u];
          if (AX == 0 && K != KR) {
            if (m == 0) di = 1.0 - th * (a0[u] - am[u]);
            if (m == n - 1) di = 1.0 - th * (a0[u] - ap[u]);
          }
          const double lo = (m == 0) ? 0.0 : -th * am[u];
          const double up = -th * ap[u];
          const double inv = frcp(di - lo * cprev);
          const long long q = base + m * stride;
          const double cp = up * inv;
          const double dp = (rv[u] - lo * dprev) * inv;
          Cs[cidx(m)] = cp;
          R[q] = dp;
          cprev = cp;
          dprev = dp;
        }
      }
    }
    double x = 0.0;
    double* __restrict__ psi = FINAL ? a.psi + po : nullptr;
    for (int m0 = n - 1; m0 >= 0; m0 -= SB) {
#if YY_BWD_PREFETCH
#pragma unroll
      for (int u = 0; u < SB; ++u) {
        const int mp = m0 - 2 * SB - u;
        if (mp >= 0) {
          pf_l2(Cs + cidx(mp));
          pf_l2(R + base + mp * stride);
          if (FINAL) pf_l2(a.psi + po + base + mp * stride);
        }
      }
#endif
      double cv[SB], dv[SB], pv[SB];
#pragma unroll
      for (int u = 0; u < SB; ++u) {
        const int m = m0 - u;
        if (m >= 0) {
          const long long q = base + m * stride;
          cv[u] = Cs[cidx(m)];
          dv[u] = R[q];
          if (FINAL) pv[u] = psi[q];
        }
      }
#pragma unroll
      for (int u = 0; u < SB; ++u) {
        const int m = m0 - u;
        if (m >= 0) {
          const long long q = base + m * stride;
          x = (m == n - 1) ? dv[u] : dv[u] - cv[u] * x;
          if (FINAL) {
            psi[q] = pv[u] + x;
            const int ii = (AX == 0) ? i + m : i, jj = (AX == 1) ? j + m : j;
            wsum += omega(g, rnode<K>(g, ii), snode<K>(g, jj)) * x * x;
          } else {
            R[q] = x;
          }
        }
      }
    }
  }
  if (FINAL) {
    const double t = block_sum<128>(wsum);
    if (threadIdx.x == 0)
      a.part[(long long)patch * a.maxb + blockIdx.y * gridDim.x + blockIdx.x] = t;
  }
}

// ---------------------------------------------------------------------------------
// K3: phi-line sweep (the contiguous axis), one warp per line, partitioned
// (Schur-complement) Thomas — the same algebra as the distributed solve of
// P:L477-480, here across the 32 lanes of a warp:
//  1. rows built with coalesced loads (lane = consecutive k), stored in shared
//     memory in chunk layout (lane l owns rows s_l..e_l; element t of every
//     chunk at smem[t*32 + l]: conflict-free);
//  2. each lane eliminates its chunk interior s_l..e_l-1 with the chunk ends
//     as unknowns: x = y + v g_{l-1} + w g_l (g_l = x_{e_l}); one reciprocal per row;
//  3. row e_l of every chunk gives a tridiagonal system in g_0..g_31, solved by
//     5 steps of parallel cyclic reduction over warp shuffles;
//  4. back-fill x, coalesced write-back.
// Same rows and end conditions as the serial Thomas of k_sweep (x 1e-16 rounding).
// ---------------------------------------------------------------------------------
constexpr int PB = 8;   // elements per lane per load round in the phi sweep

template <int Q, bool FINAL>
__global__ void __launch_bounds__(128) k_sweep_phi(Geo g, SweepArgs a, int nwarps) {
  constexpr int K = kind_of(Q);
  extern __shared__ double sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int patch = blockIdx.y;
  const int n = NPk(g, K) - 2;                       // unknowns k = 1..NP-2
  const int nj = NTk(g, K) - 2;
  const int ni = (K == KR) ? g.nr - 1 : g.nr;
  const int M = (n + 31) >> 5;                       // chunk length: lane l owns rows l*M .. l*M+M-1
  const int Mp = M | 1;                              // odd pitch: conflict-free chunk-major layout
  const int nact = (n + M - 1) / M;                  // lanes owning a (possibly shorter last) chunk
  const float iM = 1.0f / (float)M;
  const long long L = (long long)blockIdx.x * nwarps + warp;
  double wsum = 0.0;
  if (warp < nwarps && L < (long long)ni * nj) {
    const int i = i_lo<K>() + (int)(L / nj), j = 1 + (int)(L % nj);
    // normalised rows x_{e-1} a + x_e + x_{e+1} c = d (b = 1)
    double* LO = sm + (size_t)warp * 3 * 32 * Mp;
    double* UP = LO + 32 * Mp;
    double* RH = UP + 32 * Mp;
    const long long po = patch * psize(g, K);
    Astar As{a.ar + patch * psize(g, KR), a.at + patch * psize(g, KT), a.ap + patch * psize(g, KP)};
    double* __restrict__ R = a.R + po;
    const long long base = IX<K>(g, i, j, 1);
    const double th = 0.5 * g.tau;
    auto slot = [&](int e) {                         // element -> chunk-major index
      const int l = (int)(((float)e + 0.5f) * iM);
      return l * Mp + (e - l * M);
    };
    // 1. rows (I - tau/2 A_ph) of this line; 4 elements per lane per round so
    //    that all of a round's loads are in flight before any is consumed
    for (int e0 = lane; e0 < n; e0 += 32 * PB) {
      double rv[PB], am[PB], a0[PB], ap[PB];
#pragma unroll
      for (int u = 0; u < PB; ++u) {
        const int e = e0 + 32 * u;
        rv[u] = (e < n) ? R[base + e] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < PB; ++u) {
        const int e = e0 + 32 * u;
        if (e < n) coef<Q, 2, true>(g, As, i, j, 1 + e, am[u], a0[u], ap[u]);
      }
#pragma unroll
      for (int u = 0; u < PB; ++u) {
        const int e = e0 + 32 * u;
        if (e < n) {
          const int q = slot(e);
          const double inv = frcp(1.0 - th * a0[u]);
          LO[q] = (e == 0) ? 0.0 : -th * am[u] * inv;
          UP[q] = (e == n - 1) ? 0.0 : -th * ap[u] * inv;
          RH[q] = rv[u] * inv;
        }
      }
    }
    __syncwarp();
    // 2. chunk interior elimination (rows t = 0..m-2 of this lane's chunk) with
    //    x = y + v g_{l-1} + w g_l,  g_l = x at the chunk's last row
    const int m = (lane < nact) ? min(M, n - lane * M) : 0;
    const int o = lane * Mp;
    double cprev = 0.0, yprev = 0.0, vprev = 0.0;
    for (int t = 0; t + 1 < m; ++t) {
      const double lo = LO[o + t];
      const double inv = frcp(1.0 - lo * cprev);
      const double cp = UP[o + t] * inv;
      const double yp = (RH[o + t] - lo * yprev) * inv;
      const double vp = (t ? -lo * vprev : -lo) * inv;
      UP[o + t] = cp;
      RH[o + t] = yp;
      LO[o + t] = vp;
      cprev = cp; yprev = yp; vprev = vp;
    }
    // backward: y, v in place; w (nonzero from the last interior row, w' = -c') kept in UP
    double Y0 = 0.0, V0 = 0.0, W0 = 1.0;             // x_s as y + v g_{l-1} + w g_l (m = 1: g_l)
    double Yl = 0.0, Vl = 1.0, Wl = 0.0;             // x_{e-1} (m = 1: g_{l-1})
    if (m >= 2) {
      double y = RH[o + m - 2], v = LO[o + m - 2], w = -UP[o + m - 2];
      UP[o + m - 2] = w;
      Yl = y; Vl = v; Wl = w;
      for (int t = m - 3; t >= 0; --t) {
        const double cp = UP[o + t];
        y = RH[o + t] - cp * y;
        v = LO[o + t] - cp * v;
        w = -cp * w;
        RH[o + t] = y;
        LO[o + t] = v;
        UP[o + t] = w;
      }
      Y0 = y; V0 = v; W0 = w;
    }
    // 3. reduced tridiagonal system in g (row e_l of every chunk), PCR over shuffles
    double A = 0.0, B = 1.0, C = 0.0, D = 0.0;
    {
      const double Y0n = __shfl_down_sync(0xffffffffu, Y0, 1);
      const double V0n = __shfl_down_sync(0xffffffffu, V0, 1);
      const double W0n = __shfl_down_sync(0xffffffffu, W0, 1);
      if (lane < nact) {
        const double ae = LO[o + m - 1], ce = UP[o + m - 1];   // row e_l (untouched above)
        const bool lastl = (lane == nact - 1);
        A = ae * Vl;
        B = ae * Wl + 1.0 + (lastl ? 0.0 : ce * V0n);
        C = lastl ? 0.0 : ce * W0n;
        D = RH[o + m - 1] - ae * Yl - (lastl ? 0.0 : ce * Y0n);
      }
    }
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
      const double Am = __shfl_up_sync(0xffffffffu, A, s), Bm = __shfl_up_sync(0xffffffffu, B, s);
      const double Cm = __shfl_up_sync(0xffffffffu, C, s), Dm = __shfl_up_sync(0xffffffffu, D, s);
      const double Ap = __shfl_down_sync(0xffffffffu, A, s), Bp = __shfl_down_sync(0xffffffffu, B, s);
      const double Cp = __shfl_down_sync(0xffffffffu, C, s), Dp = __shfl_down_sync(0xffffffffu, D, s);
      const bool hm = lane >= s, hp = lane + s < 32;
      const double al = hm ? -A * frcp(Bm) : 0.0;
      const double ga = hp ? -C * frcp(Bp) : 0.0;
      const double nA = hm ? al * Am : 0.0;
      const double nC = hp ? ga * Cp : 0.0;
      B = B + (hm ? al * Cm : 0.0) + (hp ? ga * Ap : 0.0);
      D = D + (hm ? al * Dm : 0.0) + (hp ? ga * Dp : 0.0);
      A = nA;
      C = nC;
    }
    const double gl = D * frcp(B);
    const double glm = __shfl_up_sync(0xffffffffu, gl, 1);
    // 4. back-fill
    if (lane < nact) {
      const double gprev = lane ? glm : 0.0;
      for (int t = 0; t + 1 < m; ++t) RH[o + t] = RH[o + t] + LO[o + t] * gprev + UP[o + t] * gl;
      RH[o + m - 1] = gl;
    }
    __syncwarp();
    if (FINAL) {
      double* __restrict__ psi = a.psi + po;
      const double w0 = omega(g, rnode<K>(g, i), snode<K>(g, j));
      for (int e = lane; e < n; e += 32) {
        const double v = RH[slot(e)];
        psi[base + e] += v;
        wsum += w0 * v * v;
      }
    } else {
      for (int e = lane; e < n; e += 32) R[base + e] = RH[slot(e)];
    }
  }
  if (FINAL) {
    const double t = block_sum<128>(wsum);
    if (threadIdx.x == 0) a.part[(long long)patch * a.maxb + blockIdx.x] = t;
  }
}

// ---------------------------------------------------------------------------------
// K7: pressure updates (eq:nst_Mass1 P:L457; system 2 per RD18)
// ---------------------------------------------------------------------------------
template <int S>
__global__ void __launch_bounds__(128) k_pres(Geo g, PresArgs a) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y;
  const int nz = (g.nr + 3) / 4;
  const int patch = blockIdx.z / nz, i0 = 4 * (blockIdx.z % nz);
  double w = 0.0;
  if (k >= 1 && k <= g.np - 2 && j >= 1 && j <= g.nt - 2) {
    const long long pc = patch * psize(g, KC);
    const long long orr = patch * psize(g, KR), ot = patch * psize(g, KT), op = patch * psize(g, KP);
    const double *uri = a.urit + orr, *urn = a.urn + orr;
    const double *uti = a.utit + ot, *utn = a.utn + ot;
    const double *upi = a.upit + op, *upn = a.upn + op;
    const double s0 = __ldg(g.sf + j), s1 = __ldg(g.sf + j + 1), sn = __ldg(g.sc + j), is = __ldg(g.is_c + j);
    for (int i = i0; i < i0 + 4 && i < g.nr; ++i) {
      const double ir = __ldg(g.ir_c + i);
      const double f0 = __ldg(g.rf2 + i), f1 = __ldg(g.rf2 + i + 1);
      const double ur0 = 0.5 * (uri[IX<KR>(g, i, j, k)] + urn[IX<KR>(g, i, j, k)]);
      const double ur1 = 0.5 * (uri[IX<KR>(g, i + 1, j, k)] + urn[IX<KR>(g, i + 1, j, k)]);
      const double ut0 = 0.5 * (uti[IX<KT>(g, i, j, k)] + utn[IX<KT>(g, i, j, k)]);
      const double ut1 = 0.5 * (uti[IX<KT>(g, i, j + 1, k)] + utn[IX<KT>(g, i, j + 1, k)]);
      const double up0 = 0.5 * (upi[IX<KP>(g, i, j, k)] + upn[IX<KP>(g, i, j, k)]);
      const double up1 = 0.5 * (upi[IX<KP>(g, i, j, k + 1)] + upn[IX<KP>(g, i, j, k + 1)]);
      const double dv = (f1 * ur1 - f0 * ur0) * __ldg(g.idv1_c + i) + (s1 * ut1 - s0 * ut0) * (ir * is * g.idth) +
                        (up1 - up0) * (ir * is * g.idph);
      const long long q = pc + IX<KC>(g, i, j, k);
      double nv;
      if (S == 1) nv = a.pn[q] - g.inv_chi * dv;
      else nv = a.pn[q] + (a.p1it[q] - a.p1n[q]) - g.inv_chi * dv;
      const double d = nv - a.pit[q];
      a.pit[q] = nv;
      w += omega(g, __ldg(g.rc + i), sn) * d * d;
    }
  }
  const double t = block_sum<128>(w);
  if (threadIdx.x == 0)
    a.part[(long long)patch * a.maxb + ((blockIdx.z % nz) * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = t;
}

// ---------------------------------------------------------------------------------
// K6: deterministic final reduction: 18 (quantity, patch) sums in fixed order,
// rho = max sqrt; NaN/Inf -> flag.
// ---------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_reduce_slots(const double* __restrict__ part, ReduceArgs a,
                                                      double* __restrict__ out) {
  const int slot = blockIdx.x / 2, patch = blockIdx.x % 2;   // one block per (slot, patch)
  const double* p = part + ((long long)slot * 2 + patch) * a.maxb;
  const int nb = a.nblk[slot];
  double v = 0.0;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) v += p[b];
  const double t = block_sum<256>(v);
  if (threadIdx.x == 0) out[2 + blockIdx.x] = t;
}

__global__ void k_reduce_final(double* __restrict__ out) {
  if (threadIdx.x == 0) {
    double rho = 0.0;
    int bad = 0;
    for (int q = 0; q < 2 * NSLOT; ++q) {
      const double s = out[2 + q];
      if (!(s == s) || s > 1e300) bad = 1;
      out[2 + q] = sqrt(s);
      rho = fmax(rho, sqrt(s));
    }
    out[0] = bad ? __longlong_as_double(0x7ff8000000000000LL) : rho;
    out[1] = bad;
  }
}

// ---------------------------------------------------------------------------------
// K5: Yin<->Yang fringe interpolation (Alg.1 steps 1,3,7; RD3-RD5).
// Reads donor solved nodes, writes target fringe nodes: race-free in place.
// ---------------------------------------------------------------------------------
__device__ __forceinline__ double interp16(const Geo& g, int K, const double* __restrict__ X, int i, int jb,
                                           int kb, const double* __restrict__ w) {
  const int NT = NTk(g, K), NP = NPk(g, K);
  const double* base = X + ((long long)i * NT + jb) * NP + kb;
  double v = 0.0;
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const double* row = base + (long long)a * NP;
    const double s = w[4] * row[0] + w[5] * row[1] + w[6] * row[2] + w[7] * row[3];
    v += w[a] * s;
  }
  return v;
}

// scalar-like quantities on the (theta_c, phi_c) lattice: T, p1, p2, u_r1, u_r2
// grid: x -> entry, y -> i (0..nr), z -> patch*5 + quantity
__global__ void k_interp_cc(Geo g, InterpArgs a) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  const int patch = blockIdx.z / 5, q = blockIdx.z % 5;
  if (e >= a.tab_cc.n) return;
  const int K = (q < 3) ? KC : KR;
  if (K == KC && i >= g.nr) return;
  if (K == KR && (i < 1 || i > g.nr - 1)) return;
  const long long ps = psize(g, K);
  double* X = a.cc[q];
  const double* donor = X + (1 - patch) * ps;
  double* tgt = X + patch * ps;
  const int jb = a.tab_cc.jb[e], kb = a.tab_cc.kb[e];
  const double v = interp16(g, K, donor, i, jb, kb, a.tab_cc.w + 8LL * e);
  tgt[((long long)i * NTk(g, K) + a.tab_cc.tj[e]) * NPk(g, K) + a.tab_cc.tk[e]] = v;
}

// tangential vector components: target kind KT (u_th) or KP (u_ph) of both
// systems; both donor components interpolated on their own lattices, rotated.
// grid: x -> entry, y -> i, z -> patch*2 + system
template <int KTGT>
__global__ void k_interp_vec(Geo g, InterpArgs a) {
  const VecTab& t = (KTGT == KT) ? a.tab_th : a.tab_ph;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  const int patch = blockIdx.z / 2, s = blockIdx.z % 2;
  if (e >= t.n) return;
  const double* ut = a.ut[s];
  const double* up = a.up[s];
  const double* dut = ut + (1 - patch) * psize(g, KT);
  const double* dup = up + (1 - patch) * psize(g, KP);
  const double vt = interp16(g, KT, dut, i, t.jb_t[e], t.kb_t[e], t.w_t + 8LL * e);
  const double vp = interp16(g, KP, dup, i, t.jb_p[e], t.kb_p[e], t.w_p + 8LL * e);
  const double v = t.m0[e] * vt + t.m1[e] * vp;
  double* tgt = (KTGT == KT ? a.ut[s] : a.up[s]) + patch * psize(g, KTGT);
  tgt[((long long)i * NTk(g, KTGT) + t.tj[e]) * NPk(g, KTGT) + t.tk[e]] = v;
}

// ---------------------------------------------------------------------------------
// C4 kernel-only operator: one patch, T rows (hats), all lines of one axis.
// ---------------------------------------------------------------------------------

// ---------------------------------------------------------------------------------
// launch wrappers
// ---------------------------------------------------------------------------------
static inline dim3 pgrid(const Geo& g, int K, int npatch) {
  return dim3((NPk(g, K) + 127) / 128, NTk(g, K), NRk(g, K) * npatch);
}

void launch_lincomb(double* out, long long n, const LinIn& in, int nin, cudaStream_t st) {
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  k_lincomb<<<blocks, 256, 0, st>>>(out, n, nin, in);
}

void launch_static(const Geo& g, int q, const StaticArgs& a, cudaStream_t st) {
  switch (q) {
    case QT: k_static<QT><<<pgrid(g, KC, 2), 128, 0, st>>>(g, a); break;
    case QUR: k_static<QUR><<<pgrid(g, KR, 2), 128, 0, st>>>(g, a); break;
    case QUT: k_static<QUT><<<pgrid(g, KT, 2), 128, 0, st>>>(g, a); break;
    case QUP: k_static<QUP><<<pgrid(g, KP, 2), 128, 0, st>>>(g, a); break;
  }
}

void launch_resid(const Geo& g, int q, int s, const ResidArgs& a, cudaStream_t st) {
  if (q == QT) k_resid<QT, 1><<<pgrid(g, KC, 2), 128, 0, st>>>(g, a);
  else if (q == QUR) { if (s == 1) k_resid<QUR, 1><<<pgrid(g, KR, 2), 128, 0, st>>>(g, a); else k_resid<QUR, 2><<<pgrid(g, KR, 2), 128, 0, st>>>(g, a); }
  else if (q == QUT) { if (s == 1) k_resid<QUT, 1><<<pgrid(g, KT, 2), 128, 0, st>>>(g, a); else k_resid<QUT, 2><<<pgrid(g, KT, 2), 128, 0, st>>>(g, a); }
  else { if (s == 1) k_resid<QUP, 1><<<pgrid(g, KP, 2), 128, 0, st>>>(g, a); else k_resid<QUP, 2><<<pgrid(g, KP, 2), 128, 0, st>>>(g, a); }
}

template <int Q, bool F>
static int sweep_phi(const Geo& g, const SweepArgs& a, int npatch, cudaStream_t st) {
  constexpr int K = kind_of(Q);
  const int n = NPk(g, K) - 2;
  const int Mp = ((n + 31) / 32) | 1;
  const size_t per_warp = (size_t)3 * 32 * Mp * sizeof(double);
  int nw = (int)((200 * 1024) / per_warp);   // <= 227 KB opt-in per block on sm_100
  nw = nw < 1 ? 1 : (nw > 4 ? 4 : nw);
  const long long lines = (long long)((K == KR) ? g.nr - 1 : g.nr) * (NTk(g, K) - 2);
  const int blocks = (int)((lines + nw - 1) / nw);
  const size_t smem = per_warp * nw;
  static size_t attr_set = 0;
  if (smem > 48 * 1024 && smem > attr_set) {
    cudaFuncSetAttribute(k_sweep_phi<Q, F>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr_set = smem;
  }
  k_sweep_phi<Q, F><<<dim3(blocks, npatch), 128, smem, st>>>(g, a, nw);
  return blocks;
}

template <int Q, int AX, bool F>
static int sweep_one(const Geo& g, const SweepArgs& a, int npatch, cudaStream_t st) {
  constexpr int K = kind_of(Q);
  if constexpr (AX == 2) {
    return sweep_phi<Q, F>(g, a, npatch, st);
  } else {
  // line length; c' lives in shared memory (64 lines per block) when it fits
  const int n = (AX == 0) ? ((K == KR) ? g.nr - 1 : g.nr) : NTk(g, K) - 2;
  const int tpb = 64;
  const size_t smem = (size_t)n * tpb * sizeof(double);
  // measured on B200 (C3): shared-memory c' halves occupancy and is ~2x slower
  // than the high-occupancy version with c' in L2/global scratch; kept off
  const bool smc = false && smem <= 100 * 1024;
  const int bx = smc ? tpb : 128;
  dim3 grid;
  if (AX == 0) grid = dim3((NPk(g, K) - 2 + bx - 1) / bx, NTk(g, K) - 2, npatch);
  else grid = dim3((NPk(g, K) - 2 + bx - 1) / bx, (K == KR ? g.nr - 1 : g.nr), npatch);
  if (smc) {
    static size_t attr = 0;
    if (smem > 48 * 1024 && smem > attr) {
      cudaFuncSetAttribute(k_sweep<Q, AX, F, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr = smem;
    }
    k_sweep<Q, AX, F, true><<<grid, tpb, smem, st>>>(g, a);
  } else {
    k_sweep<Q, AX, F, false><<<grid, 128, 0, st>>>(g, a);
  }
  return (int)(grid.x * grid.y);
  }
}

template <int Q>
static int sweep_axis(const Geo& g, int ax, bool fin, const SweepArgs& a, int npatch, cudaStream_t st) {
  if (ax == 0) return fin ? sweep_one<Q, 0, true>(g, a, npatch, st) : sweep_one<Q, 0, false>(g, a, npatch, st);
  if (ax == 1) return fin ? sweep_one<Q, 1, true>(g, a, npatch, st) : sweep_one<Q, 1, false>(g, a, npatch, st);
  return fin ? sweep_one<Q, 2, true>(g, a, npatch, st) : sweep_one<Q, 2, false>(g, a, npatch, st);
}

int launch_sweep(const Geo& g, int q, int ax, bool fin, const SweepArgs& a, int npatch, cudaStream_t st) {
  switch (q) {
    case QT: return sweep_axis<QT>(g, ax, fin, a, npatch, st);
    case QUR: return sweep_axis<QUR>(g, ax, fin, a, npatch, st);
    case QUT: return sweep_axis<QUT>(g, ax, fin, a, npatch, st);
    default: return sweep_axis<QUP>(g, ax, fin, a, npatch, st);
  }
}

int launch_pres(const Geo& g, int s, const PresArgs& a, cudaStream_t st) {
  const int nz = (g.nr + 3) / 4;
  dim3 grid((g.np + 127) / 128, g.nt, 2 * nz);
  if (s == 1) k_pres<1><<<grid, 128, 0, st>>>(g, a);
  else k_pres<2><<<grid, 128, 0, st>>>(g, a);
  return (int)(grid.x * grid.y * nz);
}

void launch_reduce(const double* part, const ReduceArgs& a, double* out, cudaStream_t st) {
  k_reduce_slots<<<2 * NSLOT, 256, 0, st>>>(part, a, out);
  k_reduce_final<<<1, 32, 0, st>>>(out);
}

void launch_interp(const Geo& g, const InterpArgs& a, cudaStream_t st) {
  if (a.tab_cc.n) k_interp_cc<<<dim3((a.tab_cc.n + 127) / 128, g.nr + 1, 10), 128, 0, st>>>(g, a);
  if (a.tab_th.n) k_interp_vec<KT><<<dim3((a.tab_th.n + 127) / 128, g.nr, 4), 128, 0, st>>>(g, a);
  if (a.tab_ph.n) k_interp_vec<KP><<<dim3((a.tab_ph.n + 127) / 128, g.nr, 4), 128, 0, st>>>(g, a);
}

}  // namespace yy
