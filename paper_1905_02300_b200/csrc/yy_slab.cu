// yy_slab.cu — radial slabs of a patch on several GPUs: the
// r-lines cross slab boundaries, so the r-factor sweep is the partitioned
// (Schur-complement) tridiagonal solve of P:L477-480 across ranks:
//   1. every slab solves its part of every line with the two couplings to the
//      neighbour slabs kept symbolic (k_line MODE_SLAB):
//        x = x0 + xlo * X_LO + xhi * X_HI,
//      X_LO = last row of the slab below, X_HI = first row of the slab above;
//   2. the first and last rows of (x0, xlo, xhi) of every slab of the patch are
//      gathered (6 values per line per slab);
//   3. k_slab_solve: per line, the 2 nslab boundary unknowns (a_s = first row,
//      b_s = last row of slab s) satisfy
//        a_s = x0_f + xlo_f b_{s-1} + xhi_f a_{s+1},  b_s = x0_l + xlo_l b_{s-1} + xhi_l a_{s+1};
//      every slab solves this small system (redundantly) and keeps its X_LO, X_HI;
//   4. k_slab_correct: x = x0 + xlo X_LO + xhi X_HI, then the sweep's own ending
//      (next factor's right-hand side, or psi += x and the norm partial).
// Also the fixed-order merge of every context's convergence sums.
#include <cuda_runtime.h>
#include <stdint.h>

#include "yy_dev.cuh"
#include "yy_internal.h"

namespace yy {

namespace {

constexpr int MAXS = 8;   // slabs per patch

__global__ void k_slab_solve(SlabArgs a) {
  const int line = blockIdx.x * blockDim.x + threadIdx.x;
  if (line >= a.nlines) return;
  const int S = a.nslab;
  // The 2S boundary unknowns in the order (.., b_{s-1}, a_s, b_s, a_{s+1}, ..) form a
  // banded system (row a_s: b_{s-1}, a_s, a_{s+1}; row b_s: b_{s-1}, b_s, a_{s+1}):
  // one forward sweep keeps b_{s-1} = be + ga a_s and gives a_s = p_s + q_s a_{s+1},
  // the backward sweep from a_S = 0 recovers every a_s (O(S) work, no pivoting: the
  // couplings are responses of diagonally dominant lines, |.| < 1; the same
  // elimination as the boundary system of the multi-warp phi lines, yy_line.cu)
  double p[MAXS], q[MAXS], bb[MAXS], gg[MAXS];
  double be = 0.0, ga = 0.0;                 // b_{-1} = 0: no slab below the first
  for (int s = 0; s < S; ++s) {
    const double* f = a.IFall + ((long long)s * a.nlines + line) * 6;
    const double d = 1.0 / (1.0 - f[1] * ga);
    p[s] = (f[0] + f[1] * be) * d;
    q[s] = f[2] * d;
    bb[s] = be;
    gg[s] = ga;
    be = f[3] + f[4] * (be + ga * p[s]);
    ga = f[4] * ga * q[s] + f[5];
  }
  const int me = a.slab;
  double an = 0.0;                           // a_{s+1}; a_S = 0: no slab above the last
  double xlo = 0.0, xhi = 0.0;
  for (int s = S - 1; s >= 0; --s) {
    const double as = p[s] + q[s] * an;
    if (s == me) {
      xlo = s > 0 ? bb[s] + gg[s] * as : 0.0;   // b_{s-1}
      xhi = s < S - 1 ? an : 0.0;               // a_{s+1}
    }
    an = as;
  }
  a.LH[2LL * line + 0] = xlo;
  a.LH[2LL * line + 1] = xhi;
}

// grid: x -> k (128 per block), y -> j, z -> owned row
template <int K, bool FINAL>
__global__ void __launch_bounds__(128) k_slab_correct(Geo g, SweepArgs w, const double* __restrict__ LH) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x + 1;
  const int j = blockIdx.y + 1;
  const int i = blockIdx.z + i_lo<K>(g);
  double wsum = 0.0;
  if (k <= NPk(g, K) - 2) {
    const int nd = IX<K>(g, i, j, k);
    const int line = (j - 1) * (NPk(g, K) - 2) + (k - 1);
    const double x = w.R[nd] + w.V[nd] * LH[2 * line] + w.W[nd] * LH[2 * line + 1];
    if (FINAL) {
      w.psi[nd] += x;
      const double r = rnode<K>(g, i), s = snode<K>(g, j);
      wsum = r * r * s * x * x;
    } else {
      w.R[nd] = x;
    }
  }
  if (FINAL) {
    __shared__ double sh[4];
    for (int o = 16; o > 0; o >>= 1) wsum += __shfl_down_sync(0xffffffffu, wsum, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = wsum;
    __syncthreads();
    if (threadIdx.x == 0)
      w.part[((long long)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] =
          ((sh[0] + sh[1]) + (sh[2] + sh[3])) * (g.dr * g.dth * g.dph);
  }
}

__global__ void k_merge_all(double* __restrict__ out, const double* __restrict__ gath, int nslab) {
  const int q = threadIdx.x;                  // (slot, patch) = (q / 2, q % 2)
  if (q >= 2 * NSLOT) return;
  const int p = q % 2;
  double v = 0.0;
  for (int s = 0; s < nslab; ++s) v += gath[(long long)(p * nslab + s) * (2 + 2 * NSLOT) + 2 + q];
  out[2 + q] = v;
}

template <int K>
int correct_k(const Geo& g, bool fin, const SweepArgs& w, const double* LH, cudaStream_t st) {
  const dim3 grid((NPk(g, K) - 2 + 127) / 128, NTk(g, K) - 2, i_hi<K>(g) - i_lo<K>(g) + 1);
  if (fin) k_slab_correct<K, true><<<grid, 128, 0, st>>>(g, w, LH);
  else k_slab_correct<K, false><<<grid, 128, 0, st>>>(g, w, LH);
  return (int)(grid.x * grid.y * grid.z);
}

}  // namespace

void launch_slab_solve(const SlabArgs& a, cudaStream_t st) {
  k_slab_solve<<<(a.nlines + 127) / 128, 128, 0, st>>>(a);
}

int launch_slab_correct(const Geo& g, int kind, bool fin, const SweepArgs& w, const double* LH, cudaStream_t st) {
  switch (kind) {
    case KC: return correct_k<KC>(g, fin, w, LH, st);
    case KR: return correct_k<KR>(g, fin, w, LH, st);
    case KT: return correct_k<KT>(g, fin, w, LH, st);
    default: return correct_k<KP>(g, fin, w, LH, st);
  }
}

void launch_merge_all(double* out, const double* gath, int nslab, cudaStream_t st) {
  k_merge_all<<<1, 32, 0, st>>>(out, gath, nslab);
}

}  // namespace yy
