// yy_kernels.cu — sm_100a fp64 kernels of one Yin-Yang AC direction-splitting
// time step (arXiv 1905.02300).  Launch wrappers at the bottom are called by
// yy_api.cu.  Every step of the hot path runs here; the host only sequences
// launches.
//
// Kernels (SURVEY.md §2.2 naming):
//   K0  k_static<Q>      per-step static RHS G_q (O3), both systems fused
//   K1  k_resid<Q,S>     eq:er residual R = G + tau E_dyn - (I - tau/2 L_split)(psi~ - psi^n)
//   K2/K3 line sweeps: yy_line.cu
//   K5  k_interp_*       Yin<->Yang fringe interpolation (4x4 Lagrange, rotation)
//   K6  k_reduce         deterministic Schwarz residual reduction
//   K7  k_pres<S>        pressure updates eq:nst_Mass1 / eq:ac2 (RD18)
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "yy_dev.cuh"
#include "yy_internal.h"
#include "yy_stencil.cuh"

namespace yy {

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

// one job per blockIdx.y, grid-stride in x (same summation order as k_lincomb)
__global__ void k_lincomb_batch(LinBatch b) {
  const int jb = blockIdx.y;
  const long long n = b.n[jb];
  double* __restrict__ out = b.out[jb];
  const int nin = b.nin[jb];
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < n;
       idx += (long long)gridDim.x * blockDim.x) {
    if (nin < 0) {                         // plain copy (bit for bit, signed zeros too)
      out[idx] = b.p[jb][0][idx];
      continue;
    }
    double v = 0.0;
    for (int m = 0; m < nin; ++m) v += b.c[jb][m] * b.p[jb][m][idx];
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
  Astar A{a.ar + patch * psize(g, KR), a.at + patch * psize(g, KT), a.ap + patch * psize(g, KP),
          a.rt + patch * psize(g, KT), a.rp + patch * psize(g, KP)};
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
    // IMEX: the split operator without its transport terms (a* = 0)
    const double Ls = a.imex ? applyL<Q, true, RX_GIVEN>(g, A, i, j, k, D) : applyL<Q, true>(g, A, i, j, k, D);
    a.G[s][po + node] = g.tau * (Lf - 0.5 * Ls + E);
  }
}

// ---------------------------------------------------------------------------------
// K1: residual of eq:er (sign RD9) with the Gauss-Seidel dynamic terms, one node
// per thread (resid_at of yy_stencil.cuh).  The step normally fuses it into the
// first sweep of each quantity (yy_line.cu) when YY_FUSE=1.
// ---------------------------------------------------------------------------------
// residual blocks: BK consecutive k x 128/BK consecutive j (the theta neighbours of
// a column partly in the same block's L1); measured on B200 (C3): 64 for u_r,
// 128 (one theta row) for the others
#ifndef YY_RESID_BK
#define YY_RESID_BK (Q == QUR ? 64 : 128)
#endif
#ifndef YY_RESID_MINB
#define YY_RESID_MINB 8
#endif
template <int Q, int S, int IB, bool NOADV = false>
__global__ void __launch_bounds__(128, YY_RESID_MINB) k_resid(Geo g, ResidArgs a) {
  const uint3 B = bidx(a.rev);
  // thread = one (j, k) column, IB consecutive r-nodes (setup amortised, r-neighbours
  // of consecutive nodes shared through L1)
  constexpr int K = kind_of(Q);
  constexpr int BK = YY_RESID_BK, BJ = 128 / BK;   // block = BK k x BJ j columns
  const int k = B.x * BK + threadIdx.x % BK + 1;
  const int j = B.y * BJ + threadIdx.x / BK + 1;
  const int nch = (i_hi<K>(g) - i_lo<K>(g) + IB) / IB;
  const int patch = B.z / nch;
  const int i0 = i_lo<K>(g) + (B.z % nch) * IB;
  if (k > NPk(g, K) - 2 || j > NTk(g, K) - 2) return;
  double* __restrict__ R = a.R + patch * psize(g, K);
  // blocks away from the walls (all but the first / last chunk of r-nodes) take
  // no wall-ghost code (a block-uniform branch)
  const bool edge = K != KR && ((g.wall_lo && i0 == g.ilo_c) || (g.wall_hi && i0 + IB - 1 >= g.ihi_c));
  if constexpr (NOADV) {   // IMEX: split rows without transport terms (separate instantiation)
#pragma unroll
    for (int u = 0; u < IB; ++u) {
      const int i = i0 + u;
      if (i <= i_hi<K>(g)) R[IX<K>(g, i, j, k)] = resid_at<Q, S, true, true>(g, a, patch, i, j, k);
    }
  } else {
    if (edge) {
#pragma unroll
      for (int u = 0; u < IB; ++u) {
        const int i = i0 + u;
        if (i <= i_hi<K>(g)) R[IX<K>(g, i, j, k)] = resid_at<Q, S, true>(g, a, patch, i, j, k);
      }
    } else {
#pragma unroll
      for (int u = 0; u < IB; ++u) {
        const int i = i0 + u;
        if (i <= i_hi<K>(g)) R[IX<K>(g, i, j, k)] = resid_at<Q, S, false>(g, a, patch, i, j, k);
      }
    }
  }
}

// ---------------------------------------------------------------------------------
// K7: pressure updates (eq:nst_Mass1 P:L457; system 2 per RD18)
// ---------------------------------------------------------------------------------
template <int S>
__global__ void __launch_bounds__(128) k_pres(Geo g, PresArgs a) {
  const uint3 B = bidx(a.rev);
  const int k = B.x * blockDim.x + threadIdx.x;
  const int j = B.y;
  const int nz = (g.ihi_c - g.ilo_c + 4) / 4;
  const int patch = B.z / nz, i0 = g.ilo_c + 4 * (B.z % nz);
  double w = 0.0;
  if (k >= 1 && k <= g.np - 2 && j >= 1 && j <= g.nt - 2) {
    const long long pc = patch * psize(g, KC);
    const long long orr = patch * psize(g, KR), ot = patch * psize(g, KT), op = patch * psize(g, KP);
    const double *uri = a.urit + orr, *urn = a.urn + orr;
    const double *uti = a.utit + ot, *utn = a.utn + ot;
    const double *upi = a.upit + op, *upn = a.upn + op;
    const double s0 = __ldg(g.sf + j), s1 = __ldg(g.sf + j + 1), sn = __ldg(g.sc + j), is = __ldg(g.is_c + j);
    // the new pressure at cell (i, j, k) (loads only)
    auto update = [&](int i, long long& q, double& pn) {
      const double ir = __ldg(g.ir_c + i);
      const double f0 = __ldg(g.rf2 + i), f1 = __ldg(g.rf2 + i + 1);
      const double ur0 = 0.5 * (__ldg(uri + IX<KR>(g, i, j, k)) + __ldg(urn + IX<KR>(g, i, j, k)));
      const double ur1 = 0.5 * (__ldg(uri + IX<KR>(g, i + 1, j, k)) + __ldg(urn + IX<KR>(g, i + 1, j, k)));
      const double ut0 = 0.5 * (__ldg(uti + IX<KT>(g, i, j, k)) + __ldg(utn + IX<KT>(g, i, j, k)));
      const double ut1 = 0.5 * (__ldg(uti + IX<KT>(g, i, j + 1, k)) + __ldg(utn + IX<KT>(g, i, j + 1, k)));
      const double up0 = 0.5 * (__ldg(upi + IX<KP>(g, i, j, k)) + __ldg(upn + IX<KP>(g, i, j, k)));
      const double up1 = 0.5 * (__ldg(upi + IX<KP>(g, i, j, k + 1)) + __ldg(upn + IX<KP>(g, i, j, k + 1)));
      const double dv = (f1 * ur1 - f0 * ur0) * __ldg(g.idv1_c + i) + (s1 * ut1 - s0 * ut0) * (ir * is * g.idth) +
                        (up1 - up0) * (ir * is * g.idph);
      q = pc + IX<KC>(g, i, j, k);
      pn = __ldg(a.pn + q);
      if (S == 1) return pn - g.inv_chi * dv;
      return pn + (a.dp1 ? __ldg(a.dp1 + q) : __ldg(a.p1it + q) - __ldg(a.p1n + q)) - g.inv_chi * dv;
    };
    // 4 r-nodes per thread.  System 1: the four nodes' loads first (all in flight
    // together), then the stores (p1, p1^(k) - p1^n); system 2 (more arrays per
    // node, enough loads in flight already) node by node at 32 registers —
    // measured on B200 (C3)
    if constexpr (S == 1) {
      double dv1[4];
      long long qv[4];
      int nu = 0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (i0 + u > g.ihi_c) break;
        double pn;
        const double nv = update(i0 + u, qv[u], pn);
        const double d = nv - a.pit[qv[u]];
        a.pit[qv[u]] = nv;
        w += omega(g, __ldg(g.rc + i0 + u), sn) * d * d;
        dv1[u] = nv - pn;
        nu = u + 1;
      }
      if (a.dp1) {   // p1^(k) - p1^n for system 2
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (u < nu) a.dp1[qv[u]] = dv1[u];
      }
    } else {
#pragma unroll 1
      for (int i = i0; i < i0 + 4 && i <= g.ihi_c; ++i) {
        long long q;
        double pn;
        const double nv = update(i, q, pn);
        const double d = nv - a.pit[q];
        a.pit[q] = nv;
        w += omega(g, __ldg(g.rc + i), sn) * d * d;
      }
    }
  }
  const double t = block_sum<128>(w);
  if (threadIdx.x == 0)
    a.part[(long long)patch * a.maxb + ((B.z % nz) * gridDim.y + B.y) * gridDim.x + B.x] = t;
}

// ---------------------------------------------------------------------------------
// Theorem 1 diagnostic (eq:Stability; oracle/energy.py): per block the
// omega-weighted sums of  (-L T^n) T^n,  (-(Lh - L)_{th+ph} d) d  and  d d,
// d = T^n - T^{n-1}, over the solved cell centres, with the T rows of coef<>
// (u = 0: pure diffusion) and homogeneous wall data (the theorem's setting).
// One thread per (j, k) column walking r; block = 128 k.
// ---------------------------------------------------------------------------------
__global__ void __launch_bounds__(128) k_energy(Geo g, const double* __restrict__ Tn, const double* __restrict__ Tm,
                                                const double* __restrict__ zw, double* __restrict__ part) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x + 1, j = blockIdx.y + 1, patch = blockIdx.z;
  const Astar A{};
  double e0 = 0.0, e1 = 0.0, e2 = 0.0;
  if (k <= g.np - 2 && j <= g.nt - 2) {
    const double* tn = Tn + patch * psize(g, KC);
    const double* tm = Tm + patch * psize(g, KC);
    for (int i = g.ilo_c; i <= g.ihi_c; ++i) {
      const Star a = load_star<KC>(g, tn, zw, i, j, k);
      const Star b = load_star<KC>(g, tm, zw, i, j, k);
      const Star d = star_lin(a, 1.0, b, -1.0);
      double am, a0, ap, hm, h0, hp;
      coef<QT, 0, false, false>(g, A, i, j, k, am, a0, ap);
      double LT = am * a.xm + a0 * a.c + ap * a.xp;
      coef<QT, 1, false, false>(g, A, i, j, k, am, a0, ap);
      coef<QT, 1, true, false>(g, A, i, j, k, hm, h0, hp);
      LT += am * a.ym + a0 * a.c + ap * a.yp;
      double DL = (hm - am) * d.ym + (h0 - a0) * d.c + (hp - ap) * d.yp;
      coef<QT, 2, false, false>(g, A, i, j, k, am, a0, ap);
      coef<QT, 2, true, false>(g, A, i, j, k, hm, h0, hp);
      LT += am * a.zm + a0 * a.c + ap * a.zp;
      DL += (hm - am) * d.zm + (h0 - a0) * d.c + (hp - ap) * d.zp;
      const double w = omega(g, __ldg(g.rc + i), __ldg(g.sc + j));
      e0 += w * (-LT) * a.c;
      e1 += w * (-DL) * d.c;
      e2 += w * d.c * d.c;
    }
  }
  // block_sum's shared scratch is reused: a barrier between the three sums
  const double s0 = block_sum<128>(e0);
  __syncthreads();
  const double s1 = block_sum<128>(e1);
  __syncthreads();
  const double s2 = block_sum<128>(e2);
  if (threadIdx.x == 0) {
    double* o = part + 3LL * ((blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x);
    o[0] = s0;
    o[1] = s1;
    o[2] = s2;
  }
}

// fixed-order sum of the k_energy partials: out = (1/2 e0, 1/4 e1, e2)
__global__ void __launch_bounds__(128) k_energy_final(const double* __restrict__ part, int nb, double* __restrict__ out) {
  double v[3] = {0.0, 0.0, 0.0};
  for (int b = threadIdx.x; b < nb; b += 128)
    for (int c = 0; c < 3; ++c) v[c] += part[3LL * b + c];
  const double s0 = block_sum<128>(v[0]);
  __syncthreads();
  const double s1 = block_sum<128>(v[1]);
  __syncthreads();
  const double s2 = block_sum<128>(v[2]);
  if (threadIdx.x == 0) {
    out[0] = 0.5 * s0;
    out[1] = 0.25 * s1;
    out[2] = s2;
  }
}

// ---------------------------------------------------------------------------------
// K6: deterministic final reduction: 18 (quantity, patch) sums in fixed order,
// rho = max sqrt; NaN/Inf -> flag.
// ---------------------------------------------------------------------------------
__global__ void __launch_bounds__(512) k_reduce_slots(const double* __restrict__ part, ReduceArgs a,
                                                      double* __restrict__ out) {
  const int slot = blockIdx.x / a.npatch, lp = blockIdx.x % a.npatch;   // one block per (slot, local patch)
  const double* p = part + ((long long)slot * 2 + lp) * a.maxb;
  const int nb = a.nblk[slot];
  // four independent accumulators per thread (fixed assignment: loads in flight
  // together), then a fixed tree
  double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
  constexpr int NT = 512;
  int b = threadIdx.x;
  for (; b + 3 * NT < nb; b += 4 * NT) {
    v0 += __ldg(p + b);
    v1 += __ldg(p + b + NT);
    v2 += __ldg(p + b + 2 * NT);
    v3 += __ldg(p + b + 3 * NT);
  }
  for (; b < nb; b += NT) v0 += __ldg(p + b);
  const double t = block_sum<NT>((v0 + v1) + (v2 + v3));
  if (threadIdx.x == 0) out[2 + 2 * slot + lp + a.patch0] = t;
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
// 4x4 Lagrange stencil at base (rows NP apart) with the entry's 8 weights
// (w[0..3] across rows, w[4..7] along a row) in registers; read-only donor loads
__device__ __forceinline__ double interp16r(const double* __restrict__ base, int NP, const double (&w)[8]) {
  double v = 0.0;
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const double* row = base + a * NP;
    const double s = w[4] * __ldg(row) + w[5] * __ldg(row + 1) + w[6] * __ldg(row + 2) + w[7] * __ldg(row + 3);
    v += w[a] * s;
  }
  return v;
}

// r-levels per thread of the interpolation kernels: the entry's stencil (base
// indices, weights, rotation) is read once and reused for IL levels
constexpr int IL = 4;

// scalar-like quantities on the (theta_c, phi_c) lattice: T, p1, p2, u_r1, u_r2
// grid: x -> entry, y -> group of IL r-levels (0..nr), z -> patch*5 + quantity
__global__ void k_interp_cc(Geo g, InterpArgs a) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  const int nq = a.cc_nq ? a.cc_nq : 5;
  const int patch = blockIdx.z / nq, q = a.cc_q0 + blockIdx.z % nq;
  if (e >= a.tab_cc.n) return;
  const int K = (q < 3) ? KC : KR;
  const int lo = K == KC ? g.ifr_c0 : g.ifr_f0, hi = K == KC ? g.ifr_c1 : g.ifr_f1;
  const int i0 = max(lo, (int)blockIdx.y * IL);
  const int i1 = min(hi, (int)blockIdx.y * IL + IL - 1);
  if (i0 > i1) return;
  const long long ps = psize(g, K);
  double* X = a.cc[q];
  const int NT = NTk(g, K), NP = NPk(g, K);
  const int jb = a.tab_cc.jb[e], kb = a.tab_cc.kb[e];
  double w[8];
#pragma unroll
  for (int m = 0; m < 8; ++m) w[m] = __ldg(a.tab_cc.w + 8LL * e + m);
  const double* donor = X + (1 - patch) * ps + (jb * NP + kb);
  double* tgt = X + patch * ps + (a.tab_cc.tj[e] * NP + a.tab_cc.tk[e]);
  const int sr = NT * NP;
  double v[IL];
#pragma unroll
  for (int u = 0; u < IL; ++u)
    if (i0 + u <= i1) v[u] = interp16r(donor + (long long)(i0 + u) * sr, NP, w);
#pragma unroll
  for (int u = 0; u < IL; ++u)
    if (i0 + u <= i1) tgt[(long long)(i0 + u) * sr] = v[u];
  if (q == 1 && a.dp1) {   // p1 fringe: also p1^(k) - p1^n (read by the system-2 residuals)
    const long long o = patch * ps + (a.tab_cc.tj[e] * NP + a.tab_cc.tk[e]);
#pragma unroll
    for (int u = 0; u < IL; ++u)
      if (i0 + u <= i1) a.dp1[o + (long long)(i0 + u) * sr] = v[u] - __ldg(a.p1n + o + (long long)(i0 + u) * sr);
  }
}

// tangential vector components: target kind KT (u_th) or KP (u_ph) of both
// systems; both donor components interpolated on their own lattices, rotated.
// grid: x -> entry, y -> group of IL r-levels, z -> patch*2 + system
template <int KTGT>
__global__ void k_interp_vec(Geo g, InterpArgs a) {
  const VecTab& t = (KTGT == KT) ? a.tab_th : a.tab_ph;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  const int patch = blockIdx.z / 2, s = blockIdx.z % 2;
  const int i0 = max(g.ifr_c0, (int)blockIdx.y * IL);
  const int i1 = min(g.ifr_c1, (int)blockIdx.y * IL + IL - 1);
  if (e >= t.n || i0 > i1) return;
  const int NPT = NPk(g, KT), NPP = NPk(g, KP);
  const long long srt = (long long)NTk(g, KT) * NPT, srp = (long long)NTk(g, KP) * NPP;
  const double* dut = a.ut[s] + (1 - patch) * psize(g, KT) + (t.jb_t[e] * NPT + t.kb_t[e]);
  const double* dup = a.up[s] + (1 - patch) * psize(g, KP) + (t.jb_p[e] * NPP + t.kb_p[e]);
  double wt[8], wp[8];
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    wt[m] = __ldg(t.w_t + 8LL * e + m);
    wp[m] = __ldg(t.w_p + 8LL * e + m);
  }
  const double m0 = t.m0[e], m1 = t.m1[e];
  const int NPG = NPk(g, KTGT);
  const long long srg = (long long)NTk(g, KTGT) * NPG;
  double* tgt = (KTGT == KT ? a.ut[s] : a.up[s]) + patch * psize(g, KTGT) + (t.tj[e] * NPG + t.tk[e]);
  double v[IL];
#pragma unroll
  for (int u = 0; u < IL; ++u)
    if (i0 + u <= i1)
      v[u] = m0 * interp16r(dut + (i0 + u) * srt, NPT, wt) + m1 * interp16r(dup + (i0 + u) * srp, NPP, wp);
#pragma unroll
  for (int u = 0; u < IL; ++u)
    if (i0 + u <= i1) tgt[(i0 + u) * srg] = v[u];
}

// ---- one patch per context: donor-side evaluation + transfer + target write ----
// The fringe tables are the same in both directions (the patches are congruent
// and the chart map is an involution), so the donor evaluates the
// partner's fringe with the partner's own entries, from its local patch.
// grid: x -> entry, y -> i, z -> quantity
__global__ void k_pack_cc(Geo g, InterpArgs a, double* __restrict__ buf) {
  // grid y: groups of IL r-levels (the entry's stencil read once, as k_interp_cc)
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  const int q = blockIdx.z;
  if (e >= a.tab_cc.n) return;
  const int K = (q < 3) ? KC : KR;
  const int lo = K == KC ? g.ifr_c0 : g.ifr_f0, hi = K == KC ? g.ifr_c1 : g.ifr_f1;
  const int i0 = max(lo, (int)blockIdx.y * IL);
  const int i1 = min(hi, (int)blockIdx.y * IL + IL - 1);
  if (i0 > i1) return;
  const int NT = NTk(g, K), NP = NPk(g, K);
  double w[8];
#pragma unroll
  for (int m = 0; m < 8; ++m) w[m] = __ldg(a.tab_cc.w + 8LL * e + m);
  const double* donor = a.cc[q] + (a.tab_cc.jb[e] * NP + a.tab_cc.kb[e]);
  const long long sr = (long long)NT * NP;
  double v[IL];
#pragma unroll
  for (int u = 0; u < IL; ++u)
    if (i0 + u <= i1) v[u] = interp16r(donor + (i0 + u) * sr, NP, w);
#pragma unroll
  for (int u = 0; u < IL; ++u)
    if (i0 + u <= i1) buf[((long long)q * (g.nr + 1) + i0 + u) * a.tab_cc.n + e] = v[u];
}
__global__ void k_unpack_cc(Geo g, InterpArgs a, const double* __restrict__ buf) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y, q = blockIdx.z;
  if (e >= a.tab_cc.n) return;
  const int K = (q < 3) ? KC : KR;
  if (K == KC && (i < g.ifr_c0 || i > g.ifr_c1)) return;
  if (K == KR && (i < g.ifr_f0 || i > g.ifr_f1)) return;
  a.cc[q][((long long)i * NTk(g, K) + a.tab_cc.tj[e]) * NPk(g, K) + a.tab_cc.tk[e]] =
      buf[((long long)q * (g.nr + 1) + i) * a.tab_cc.n + e];
}
// grid: x -> entry, y -> i, z -> system
template <int KTGT>
__global__ void k_pack_vec(Geo g, InterpArgs a, double* __restrict__ buf) {
  const VecTab& t = (KTGT == KT) ? a.tab_th : a.tab_ph;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  const int s = blockIdx.z;
  const int i0 = max(g.ifr_c0, (int)blockIdx.y * IL);
  const int i1 = min(g.ifr_c1, (int)blockIdx.y * IL + IL - 1);
  if (e >= t.n || i0 > i1) return;
  const int NPT = NPk(g, KT), NPP = NPk(g, KP);
  const long long srt = (long long)NTk(g, KT) * NPT, srp = (long long)NTk(g, KP) * NPP;
  const double* dut = a.ut[s] + (t.jb_t[e] * NPT + t.kb_t[e]);
  const double* dup = a.up[s] + (t.jb_p[e] * NPP + t.kb_p[e]);
  double wt[8], wp[8];
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    wt[m] = __ldg(t.w_t + 8LL * e + m);
    wp[m] = __ldg(t.w_p + 8LL * e + m);
  }
  const double m0 = t.m0[e], m1 = t.m1[e];
  double v[IL];
#pragma unroll
  for (int u = 0; u < IL; ++u)
    if (i0 + u <= i1)
      v[u] = m0 * interp16r(dut + (i0 + u) * srt, NPT, wt) + m1 * interp16r(dup + (i0 + u) * srp, NPP, wp);
#pragma unroll
  for (int u = 0; u < IL; ++u)
    if (i0 + u <= i1) buf[((long long)s * g.nr + i0 + u) * t.n + e] = v[u];
}
template <int KTGT>
__global__ void k_unpack_vec(Geo g, InterpArgs a, const double* __restrict__ buf) {
  const VecTab& t = (KTGT == KT) ? a.tab_th : a.tab_ph;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y, s = blockIdx.z;
  if (e >= t.n || i < g.ifr_c0 || i > g.ifr_c1) return;
  double* tgt = (KTGT == KT) ? a.ut[s] : a.up[s];
  tgt[((long long)i * NTk(g, KTGT) + t.tj[e]) * NPk(g, KTGT) + t.tk[e]] = buf[((long long)s * g.nr + i) * t.n + e];
}

// ---------------------------------------------------------------------------------
// Algorithm 1 step 4: if |oint u_bd . n| >= tol over the
// patch's cell-box surface (the fringe normal velocities u_theta(j = 0, nt),
// u_phi(k = 0, np) and the walls u_r(i = 0, nr); reading RD-E5), replace the side
// values by the minimiser of J:  v = u - mu a, mu = (a.u + b) / (eps |dOmega|^2 + |a|^2)
// (a = signed side-face areas, b = wall flux; the paper reaches it by CG, J is
// quadratic with a rank-one penalty).  One block per (local patch, system); the
// flux is a fixed-order sum (deterministic).
// ---------------------------------------------------------------------------------
__global__ void __launch_bounds__(512) k_flux_fix(Geo g, FluxArgs a) {
  const int p = blockIdx.x / 2, s = blockIdx.x % 2;
  double* ur = a.ur[s] + p * psize(g, KR);
  double* ut = a.ut[s] + p * psize(g, KT);
  double* up = a.up[s] + p * psize(g, KP);
  const int nr = g.nr, nt = g.nt, np = g.np;
  const double s0 = __ldg(g.sf), s1 = __ldg(g.sf + nt);
  double f = 0.0;
  // theta sides: (side, i, k), area -/+ r_c sin(theta_f) dr dphi
  for (int q = threadIdx.x; q < 2 * nr * np; q += blockDim.x) {
    const int side = q / (nr * np), i = (q / np) % nr, k = q % np;
    const double ar = __ldg(g.rc + i) * (side ? s1 : -s0) * g.dr * g.dph;
    f += ar * ut[IX<KT>(g, i, side ? nt : 0, k)];
  }
  // phi sides: (side, i, j), area -/+ r_c dr dtheta
  for (int q = threadIdx.x; q < 2 * nr * nt; q += blockDim.x) {
    const int side = q / (nr * nt), i = (q / nt) % nr, j = q % nt;
    const double ar = __ldg(g.rc + i) * (side ? 1.0 : -1.0) * g.dr * g.dth;
    f += ar * up[IX<KP>(g, i, j, side ? np : 0)];
  }
  // walls: (wall, j, k), area -/+ r_f^2 sin(theta_c) dtheta dphi
  for (int q = threadIdx.x; q < 2 * nt * np; q += blockDim.x) {
    const int w = q / (nt * np), j = (q / np) % nt, k = q % np;
    const double rf = __ldg(g.rf + (w ? nr : 0));
    const double ar = (w ? 1.0 : -1.0) * rf * rf * __ldg(g.sc + j) * g.dth * g.dph;
    f += ar * ur[IX<KR>(g, w ? nr : 0, j, k)];
  }
  __shared__ double sh[16];
  __shared__ double s_mu;
  for (int o = 16; o > 0; o >>= 1) f += __shfl_down_sync(0xffffffffu, f, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = f;
  __syncthreads();
  if (threadIdx.x == 0) {
    double F = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) F += sh[w];
    s_mu = (fabs(F) >= a.tol) ? F / (a.eps * a.area * a.area + a.a2) : 0.0;
  }
  __syncthreads();
  const double mu = s_mu;
  if (mu == 0.0) return;
  for (int q = threadIdx.x; q < 2 * nr * np; q += blockDim.x) {
    const int side = q / (nr * np), i = (q / np) % nr, k = q % np;
    const double ar = __ldg(g.rc + i) * (side ? s1 : -s0) * g.dr * g.dph;
    ut[IX<KT>(g, i, side ? nt : 0, k)] -= mu * ar;
  }
  for (int q = threadIdx.x; q < 2 * nr * nt; q += blockDim.x) {
    const int side = q / (nr * nt), i = (q / nt) % nr, j = q % nt;
    const double ar = __ldg(g.rc + i) * (side ? 1.0 : -1.0) * g.dr * g.dth;
    up[IX<KP>(g, i, j, side ? np : 0)] -= mu * ar;
  }
}

// ---------------------------------------------------------------------------------
// Setup: the a*-independent split rows of (Q, AX) at every (i, j) of Q's kind,
// from the same coef<> the full rows use (Geo::bsplit; rebuilt when chi changes)
// ---------------------------------------------------------------------------------
template <int Q, int AX>
__global__ void k_build_split(Geo g, double* __restrict__ out, double* __restrict__ tout) {
  constexpr int K = kind_of(Q);
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= NRk(g, K) * NTk(g, K)) return;
  const int i = q / NTk(g, K), j = q % NTk(g, K);
  const Astar none{nullptr, nullptr, nullptr, nullptr, nullptr};
  double am, a0, ap;
  coef<Q, AX, true, false>(g, none, i, j, 1, am, a0, ap);
  out[3 * q] = am;
  out[3 * q + 1] = a0;
  out[3 * q + 2] = ap;
  const double th = 0.5 * g.tau;     // Geo::tsplit: the factor rows of I - tau/2 A
  tout[3 * q] = -th * am;
  tout[3 * q + 1] = 1.0 - th * a0;
  tout[3 * q + 2] = -th * ap;
}

// ---------------------------------------------------------------------------------
// per step (a* is fixed for the step, RD8): the a*-reaction coefficients of the
// u_theta theta-rows (RD14) and u_phi phi-rows, read by every
// residual, static RHS and own-direction sweep of both systems instead of their
// 4-point a* averages.  grid: x -> k, y -> j, z -> patch * nr + i
// ---------------------------------------------------------------------------------
__global__ void __launch_bounds__(128) k_react(Geo g, const double* __restrict__ ar, const double* __restrict__ at,
                                               double* __restrict__ rt, double* __restrict__ rp) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y;
  const int patch = blockIdx.z / g.nr, i = blockIdx.z % g.nr;
  const Astar A{ar + patch * psize(g, KR), at + patch * psize(g, KT), nullptr, nullptr, nullptr};
  // u_theta nodes (i, j in 1..nt-1, k) and u_phi nodes (i, j, k in 1..np-1): interior of the averages
  if (j >= 1 && j <= NTk(g, KT) - 2 && k >= 1 && k <= NPk(g, KT) - 2 && i >= 0 && i < g.nr)
    rt[patch * psize(g, KT) + IX<KT>(g, i, j, k)] = abar_r<KT>(g, A, i, j, k) * __ldg(g.ir_c + i);
  if (j >= 1 && j <= NTk(g, KP) - 2 && k >= 1 && k <= NPk(g, KP) - 2)
    rp[patch * psize(g, KP) + IX<KP>(g, i, j, k)] =
        (abar_r<KP>(g, A, i, j, k) + abar_t<KP>(g, A, i, j, k) * __ldg(g.cot_c + j)) * __ldg(g.ir_c + i);
}

// per-step transport-velocity row weights (Astar::av) at the solved nodes of kind
// K: the `adv` term of coef<Q, d> for d = r, theta, phi, the same expressions
// (the sweeps and residuals then read one value per row instead of the a* averages)
template <int K>
__global__ void __launch_bounds__(128) k_adv(Geo g, const double* __restrict__ ar, const double* __restrict__ at,
                                             const double* __restrict__ ap, double* __restrict__ d0,
                                             double* __restrict__ d1, double* __restrict__ d2) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y;
  const int patch = blockIdx.z / NRk(g, K);
  const int i = blockIdx.z % NRk(g, K);
  if (k >= NPk(g, K) || !solved<K>(g, i, j, k)) return;
  const Astar A{ar + patch * psize(g, KR), at + patch * psize(g, KT), ap + patch * psize(g, KP), nullptr, nullptr};
  const long long o = patch * psize(g, K) + IX<K>(g, i, j, k);
  d0[o] = abar_r<K>(g, A, i, j, k) * (0.5 * g.idr);
  d1[o] = abar_t<K>(g, A, i, j, k) * (0.5 * g.idth) * irn<K>(g, i);
  d2[o] = abar_p<K>(g, A, i, j, k) * (0.5 * g.idph) * irn<K>(g, i) * isn<K>(g, j);
}

// ---------------------------------------------------------------------------------
// launch wrappers
// ---------------------------------------------------------------------------------
static inline dim3 pgrid(const Geo& g, int K, int npatch) {
  return dim3((NPk(g, K) + 127) / 128, NTk(g, K), NRk(g, K) * npatch);
}

void launch_lincomb_batch(const LinBatch& b, cudaStream_t st) {
  if (b.njobs <= 0) return;
  long long mx = 0;
  for (int q = 0; q < b.njobs; ++q) mx = b.n[q] > mx ? b.n[q] : mx;
  const long long nb = (mx + 255) / 256;
  const int bx = (int)(nb < 148 ? nb : 148);
  k_lincomb_batch<<<dim3(bx > 0 ? bx : 1, b.njobs), 256, 0, st>>>(b);
}

void launch_lincomb(double* out, long long n, const LinIn& in, int nin, cudaStream_t st) {
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  k_lincomb<<<blocks, 256, 0, st>>>(out, n, nin, in);
}

void launch_static(const Geo& g, int q, const StaticArgs& a, cudaStream_t st) {
  switch (q) {
    case QT: k_static<QT><<<pgrid(g, KC, g.npatch), 128, 0, st>>>(g, a); break;
    case QUR: k_static<QUR><<<pgrid(g, KR, g.npatch), 128, 0, st>>>(g, a); break;
    case QUT: k_static<QUT><<<pgrid(g, KT, g.npatch), 128, 0, st>>>(g, a); break;
    case QUP: k_static<QUP><<<pgrid(g, KP, g.npatch), 128, 0, st>>>(g, a); break;
  }
}

template <int Q, int S, int IB>
void resid_qb(const Geo& g, const ResidArgs& a, cudaStream_t st) {
  constexpr int K = kind_of(Q);
  const int nch = (i_hi<K>(g) - i_lo<K>(g) + IB) / IB;
  constexpr int BK = YY_RESID_BK, BJ = 128 / BK;
  const dim3 grid((NPk(g, K) - 2 + BK - 1) / BK, (NTk(g, K) - 2 + BJ - 1) / BJ, g.npatch * nch);
  if (a.noadv) k_resid<Q, S, IB, true><<<grid, 128, 0, st>>>(g, a);
  else k_resid<Q, S, IB><<<grid, 128, 0, st>>>(g, a);
}
// r-nodes per thread of the residual per (quantity, system), measured on B200
// (C3): T 2, u_r 2 / 1, u_th 2 / 2, u_ph 4 / 4.  YY_RESID_IB=<T>,<ur1>,<ur2>,<ut1>,
// <ut2>,<up1>,<up2> overrides (tuning)
template <int Q, int S>
void resid_q(const Geo& g, const ResidArgs& a, cudaStream_t st) {
  static int ib[7] = {-1, -1, -1, -1, -1, -1, -1};
  if (ib[0] < 0) {
    const int def[7] = {2, 2, 1, 2, 2, 4, 4};
    for (int q = 0; q < 7; ++q) ib[q] = def[q];
    if (const char* e = getenv("YY_RESID_IB"))
      sscanf(e, "%d,%d,%d,%d,%d,%d,%d", &ib[0], &ib[1], &ib[2], &ib[3], &ib[4], &ib[5], &ib[6]);
  }
  const int b = ib[Q == QT ? 0 : 2 * Q - 2 + S];
  if (b == 1) resid_qb<Q, S, 1>(g, a, st);
  else if (b == 2) resid_qb<Q, S, 2>(g, a, st);
  else resid_qb<Q, S, 4>(g, a, st);
}

void launch_resid(const Geo& g, int q, int s, const ResidArgs& a, cudaStream_t st) {
  if (q == QT) resid_q<QT, 1>(g, a, st);
  else if (q == QUR) { if (s == 1) resid_q<QUR, 1>(g, a, st); else resid_q<QUR, 2>(g, a, st); }
  else if (q == QUT) { if (s == 1) resid_q<QUT, 1>(g, a, st); else resid_q<QUT, 2>(g, a, st); }
  else { if (s == 1) resid_q<QUP, 1>(g, a, st); else resid_q<QUP, 2>(g, a, st); }
}

int launch_pres(const Geo& g, int s, const PresArgs& a, cudaStream_t st) {
  const int nz = (g.ihi_c - g.ilo_c + 4) / 4;
  dim3 grid((g.np + 127) / 128, g.nt, g.npatch * nz);
  if (s == 1) k_pres<1><<<grid, 128, 0, st>>>(g, a);
  else k_pres<2><<<grid, 128, 0, st>>>(g, a);
  return (int)(grid.x * grid.y * nz);
}

void launch_reduce_slots(const double* part, const ReduceArgs& a, double* out, cudaStream_t st) {
  k_reduce_slots<<<a.npatch * NSLOT, 512, 0, st>>>(part, a, out);
}

void launch_reduce_final(double* out, cudaStream_t st) { k_reduce_final<<<1, 32, 0, st>>>(out); }

int energy_blocks(const Geo& g) { return ((g.np - 2 + 127) / 128) * (g.nt - 2) * g.npatch; }
void launch_energy(const Geo& g, const double* Tn, const double* Tm, const double* zw, double* part, double* out,
                   cudaStream_t st) {
  const dim3 grid((g.np - 2 + 127) / 128, g.nt - 2, g.npatch);
  k_energy<<<grid, 128, 0, st>>>(g, Tn, Tm, zw, part);
  k_energy_final<<<1, 128, 0, st>>>(part, energy_blocks(g), out);
}

// Device-side Schwarz loop control (the body's last node when the loop runs as a
// conditional WHILE graph node): count the iteration, record rho and the NaN flag
// (ctl[0..2]) and continue while no NaN, k < kmax and (fixed count or rho >= tol)
// — the host loop's test (O10).
__global__ void k_schwarz_cond(cudaGraphConditionalHandle h, const double* __restrict__ red,
                               double* __restrict__ ctl, double tol, int kmax, int fixed) {
  if (threadIdx.x == 0) {
    const double k = ctl[0] + 1.0;
    ctl[0] = k;
    ctl[1] = red[0];
    ctl[2] = red[1];
    const bool more = red[1] == 0.0 && k < (double)kmax && (fixed || !(red[0] < tol));
    cudaGraphSetConditional(h, more ? 1u : 0u);
  }
}

void launch_schwarz_cond(cudaGraphConditionalHandle h, const double* red, double* ctl, double tol, int kmax,
                         bool fixed, cudaStream_t st) {
  k_schwarz_cond<<<1, 32, 0, st>>>(h, red, ctl, tol, kmax, fixed ? 1 : 0);
}

void launch_interp(const Geo& g, const InterpArgs& a, cudaStream_t st, cudaStream_t s2, cudaStream_t s3,
                   cudaEvent_t* ev, bool defer) {
  const int ngc = (g.nr + 1 + IL - 1) / IL, ngv = (g.nr + IL - 1) / IL;
  const bool par = s2 && s3 && ev;
  defer = defer && par;
  if (par) {
    cudaEventRecord(ev[0], st);
    cudaStreamWaitEvent(s2, ev[0], 0);
    cudaStreamWaitEvent(s3, ev[0], 0);
  }
  if (a.tab_cc.n) {
    if (defer) {   // T alone ahead of the T solve; p1, p2, u_r1, u_r2 beside it
      InterpArgs t = a, r = a;
      t.cc_q0 = 0; t.cc_nq = 1;
      r.cc_q0 = 1; r.cc_nq = 4;
      k_interp_cc<<<dim3((a.tab_cc.n + 127) / 128, ngc, 2), 128, 0, st>>>(g, t);
      k_interp_cc<<<dim3((a.tab_cc.n + 127) / 128, ngc, 8), 128, 0, s2>>>(g, r);
    } else {
      k_interp_cc<<<dim3((a.tab_cc.n + 127) / 128, ngc, 10), 128, 0, st>>>(g, a);
    }
  }
  if (a.tab_th.n) k_interp_vec<KT><<<dim3((a.tab_th.n + 127) / 128, ngv, 4), 128, 0, par ? s2 : st>>>(g, a);
  if (a.tab_ph.n) k_interp_vec<KP><<<dim3((a.tab_ph.n + 127) / 128, ngv, 4), 128, 0, par ? s3 : st>>>(g, a);
  if (par) {
    cudaEventRecord(ev[1], s2);
    cudaEventRecord(ev[2], s3);
    if (!defer) join_interp(st, ev);
  }
}

void join_interp(cudaStream_t st, cudaEvent_t* ev) {
  cudaStreamWaitEvent(st, ev[1], 0);
  cudaStreamWaitEvent(st, ev[2], 0);
}

long long fringe_count(const Geo& g, const InterpArgs& a) {
  return 5LL * (g.nr + 1) * a.tab_cc.n + 2LL * g.nr * a.tab_th.n + 2LL * g.nr * a.tab_ph.n;
}

void launch_fringe_pack(const Geo& g, const InterpArgs& a, double* buf, cudaStream_t st) {
  double* bth = buf + 5LL * (g.nr + 1) * a.tab_cc.n;
  double* bph = bth + 2LL * g.nr * a.tab_th.n;
  const int ngc = (g.nr + 1 + IL - 1) / IL, ngv = (g.nr + IL - 1) / IL;
  if (a.tab_cc.n) k_pack_cc<<<dim3((a.tab_cc.n + 127) / 128, ngc, 5), 128, 0, st>>>(g, a, buf);
  if (a.tab_th.n) k_pack_vec<KT><<<dim3((a.tab_th.n + 127) / 128, ngv, 2), 128, 0, st>>>(g, a, bth);
  if (a.tab_ph.n) k_pack_vec<KP><<<dim3((a.tab_ph.n + 127) / 128, ngv, 2), 128, 0, st>>>(g, a, bph);
}

void launch_fringe_unpack(const Geo& g, const InterpArgs& a, const double* buf, cudaStream_t st) {
  const double* bth = buf + 5LL * (g.nr + 1) * a.tab_cc.n;
  const double* bph = bth + 2LL * g.nr * a.tab_th.n;
  if (a.tab_cc.n) k_unpack_cc<<<dim3((a.tab_cc.n + 127) / 128, g.nr + 1, 5), 128, 0, st>>>(g, a, buf);
  if (a.tab_th.n) k_unpack_vec<KT><<<dim3((a.tab_th.n + 127) / 128, g.nr, 2), 128, 0, st>>>(g, a, bth);
  if (a.tab_ph.n) k_unpack_vec<KP><<<dim3((a.tab_ph.n + 127) / 128, g.nr, 2), 128, 0, st>>>(g, a, bph);
}


void launch_flux_fix(const Geo& g, const FluxArgs& a, cudaStream_t st) {
  k_flux_fix<<<2 * g.npatch, 512, 0, st>>>(g, a);
}

template <int Q>
static void build_split_q(const Geo& g, double* const (&dst)[3], double* const (&tdst)[3], cudaStream_t st) {
  constexpr int K = kind_of(Q);
  const int n = NRk(g, K) * NTk(g, K), b = (n + 127) / 128;
  k_build_split<Q, 0><<<b, 128, 0, st>>>(g, dst[0], tdst[0]);
  k_build_split<Q, 1><<<b, 128, 0, st>>>(g, dst[1], tdst[1]);
  k_build_split<Q, 2><<<b, 128, 0, st>>>(g, dst[2], tdst[2]);
}

void launch_build_split(const Geo& g, double* const (&dst)[4][3], double* const (&tdst)[4][3], cudaStream_t st) {
  build_split_q<QT>(g, dst[0], tdst[0], st);
  build_split_q<QUR>(g, dst[1], tdst[1], st);
  build_split_q<QUT>(g, dst[2], tdst[2], st);
  build_split_q<QUP>(g, dst[3], tdst[3], st);
}

void launch_adv(const Geo& g, const double* ar, const double* at, const double* ap, double* const (&dst)[4][3],
                int npatch, cudaStream_t st, int kinds) {
  if (kinds & (1 << KC))
    k_adv<KC><<<pgrid(g, KC, npatch), 128, 0, st>>>(g, ar, at, ap, dst[KC][0], dst[KC][1], dst[KC][2]);
  if (kinds & (1 << KR))
    k_adv<KR><<<pgrid(g, KR, npatch), 128, 0, st>>>(g, ar, at, ap, dst[KR][0], dst[KR][1], dst[KR][2]);
  if (kinds & (1 << KT))
    k_adv<KT><<<pgrid(g, KT, npatch), 128, 0, st>>>(g, ar, at, ap, dst[KT][0], dst[KT][1], dst[KT][2]);
  if (kinds & (1 << KP))
    k_adv<KP><<<pgrid(g, KP, npatch), 128, 0, st>>>(g, ar, at, ap, dst[KP][0], dst[KP][1], dst[KP][2]);
}

void launch_react(const Geo& g, const double* ar, const double* at, double* rt, double* rp, cudaStream_t st) {
  const dim3 grid((g.np + 1 + 127) / 128, g.nt + 1, g.npatch * g.nr);
  k_react<<<grid, 128, 0, st>>>(g, ar, at, rt, rp);
}

}  // namespace yy
