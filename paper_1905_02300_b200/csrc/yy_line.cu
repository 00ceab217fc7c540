// yy_line.cu — the implicit factor sweeps of the Yin-Yang AC direction-splitting
// step (arXiv 1905.02300): on every line of one axis solve
//     (I - tau/2 A_{Q,AX}) x = b
// (the factors of eq:Convect_Douglas L318-325, eq:r_comp L398-401, eq:theta_comp
// L423-425, eq:phi_comp L447-449; homogeneous increments, wall ghost RD23).
//
// One design for the three axes: a line of n rows is split into P contiguous
// chunks of M rows (P*M >= n; rows past n are identity rows), one chunk per
// thread, the P threads of a line forming an aligned segment of a warp.  A block
// (128 threads) owns 128/P lines:
//   1. build: every row of the tile (normalised by its diagonal) from b and the
//      per-step row weights (coef_split / coef of yy_dev.cuh, the rows the
//      residual applies), written coalesced into a chunk-major shared-memory
//      tile (odd line pitch);
//   2. each thread loads its chunk into REGISTERS and eliminates the chunk
//      interior with the chunk's last unknown g_c and the previous chunk's
//      g_{c-1} kept symbolic: x_t = y_t + v_t g_{c-1} + w_t g_c (one reciprocal
//      per row) — the Schur-complement partition of the distributed tridiagonal
//      solve of P:L477-480, here across warp lanes;
//   3. the P-unknown interface system by log2(P) steps of parallel cyclic
//      reduction over segment shuffles (select-free);
//   4. back-fill, x back to the tile, then written coalesced (or psi += x and the
//      convergence norm partial, FINAL).
// No c'/d' scratch in HBM: a sweep moves its algorithmic bytes (read b and the
// row weight, write x; FINAL also psi).
//
// r and theta lines (strided): consecutive threads take consecutive phi-lines
// (128/P per block) in the build, each walking rows of its chunk; the loads of b
// are batched in registers, the row weights L1-prefetched first.
// phi lines (contiguous): one warp (P = 32 threads) per line, the tile's b, row
// weights and reaction values staged in shared memory with cp.async; lines
// longer than 384 rows take four warps (segments with symbolic couplings, then
// the line's 8-unknown boundary system, as for radial slabs).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <atomic>
#include <mutex>
#include <type_traits>

#include "yy_dev.cuh"
#include "yy_internal.h"
#include "yy_stencil.cuh"

#ifndef YY_LINE_MINB
#define YY_LINE_MINB 0   // >0: force this __launch_bounds__ min blocks per SM (tuning)
#endif
#ifndef YY_IMEX_FAST
#define YY_IMEX_FAST 1   // IMEX rows without the per-step weight reads (0: IMEX reads the zero arrays)
#endif
#ifndef YY_PH384
#define YY_PH384 0       // phi lines of 257-384 rows: 0 (32, 12); 1 (64, 6); 2 (128, 3) (tuning)
#endif
#ifndef YY_RT_MENU
#define YY_RT_MENU 0     // r / theta chunkings for n <= 128: 0 r (16,6)/(16,8), theta (8,12)/(8,16); 1 (8,12)/(8,16); 2 (32,3)/(32,4); 3 (16,6)/(16,8)
#endif

namespace yy {

namespace {

constexpr unsigned FULL = 0xffffffffu;

// Opt kernel `kern` into `smem` bytes of dynamic shared memory.  The opted-in
// size of one kernel only grows and is set under a lock, so contexts on several
// host threads (yy.h) never lower it under each other's launches.
// (one instantiation, hence one pair of statics, per kernel: the kernel is the
// template argument, not a function-pointer type that instantiations share)
template <auto kern>
inline void opt_in_smem(size_t smem) {
  static std::atomic<size_t> cur{48 * 1024};
  static std::mutex mu;
  if (smem <= cur.load(std::memory_order_acquire)) return;
  std::lock_guard<std::mutex> lk(mu);
  if (smem > cur.load(std::memory_order_relaxed)) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cur.store(smem, std::memory_order_release);
  }
}

// Steps 2-4 on registers: rows lo_t x_{t-1} + x_t + up_t x_{t+1} = rh_t of this
// thread's chunk c (0..P-1) of its line.  On exit rh[t] = x_t.
template <int P, int M>
__device__ __forceinline__ void part_solve(double (&lo)[M], double (&up)[M], double (&rh)[M], int c) {
  (void)c;
  static_assert(M >= 2, "chunk of at least two rows");
  // forward over the interior rows 0..M-2:  x_t + c'_t x_{t+1} = y'_t + v'_t g_{c-1}
  double cp = 0.0, yp = 0.0, vp = 0.0;
#pragma unroll
  for (int t = 0; t < M - 1; ++t) {
    const double l = lo[t];
    if (t == 0) {
      cp = up[0];
      yp = rh[0];
      vp = -l;
    } else {
      const double inv = frcp(1.0 - l * cp);
      cp = up[t] * inv;
      yp = (rh[t] - l * yp) * inv;
      vp = -l * vp * inv;
    }
    up[t] = cp;
    rh[t] = yp;
    lo[t] = vp;
  }
  // backward: x_t = y_t + v_t g_{c-1} + w_t g_c  (y -> rh, v -> lo, w -> up)
  {
    double y = rh[M - 2], v = lo[M - 2], w = -up[M - 2];
    up[M - 2] = w;
#pragma unroll
    for (int t = M - 3; t >= 0; --t) {
      const double ct = up[t];
      y = rh[t] - ct * y;
      v = lo[t] - ct * v;
      w = -ct * w;
      rh[t] = y;
      lo[t] = v;
      up[t] = w;
    }
  }
  // interface row M-1 of every chunk: A g_{c-1} + B g_c + C g_{c+1} = D,
  // x_M (first row of chunk c+1) = Y0n + V0n g_c + W0n g_{c+1}
  const double Y0n = __shfl_down_sync(FULL, rh[0], 1, P);
  const double V0n = __shfl_down_sync(FULL, lo[0], 1, P);
  const double W0n = __shfl_down_sync(FULL, up[0], 1, P);
  const double ae = lo[M - 1], ce = up[M - 1];     // ce = 0 on a line's last row (and identity rows)
  double A = ae * lo[M - 2];
  double B = ae * up[M - 2] + 1.0 + ce * V0n;
  double C = ce * W0n;
  double D = rh[M - 1] - ae * rh[M - 2] - ce * Y0n;
  // PCR: equation c reads A g_{c-s} + B g_c + C g_{c+s} = D.  A = 0 for c < s and
  // C = 0 for c + s >= P hold at every step (A_0 = 0: chunk 0 starts the line;
  // C_{P-1} = 0: the line ends in chunk P-1), so the out-of-segment partners a
  // width-P shuffle returns (the lane itself) are multiplied by zero: no selects.
  // The partners' reciprocal pivots are shuffled instead of their B.
#pragma unroll
  for (int s = 1; s < P; s <<= 1) {
    const double iB = frcp(B);
    const double Am = __shfl_up_sync(FULL, A, s, P), iBm = __shfl_up_sync(FULL, iB, s, P);
    const double Cm = __shfl_up_sync(FULL, C, s, P), Dm = __shfl_up_sync(FULL, D, s, P);
    const double Ap = __shfl_down_sync(FULL, A, s, P), iBp = __shfl_down_sync(FULL, iB, s, P);
    const double Cp = __shfl_down_sync(FULL, C, s, P), Dp = __shfl_down_sync(FULL, D, s, P);
    const double al = -A * iBm;
    const double ga = -C * iBp;
    B = B + al * Cm + ga * Ap;
    D = D + al * Dm + ga * Dp;
    A = al * Am;
    C = ga * Cp;
  }
  const double gc = D * frcp(B);
  const double gp = __shfl_up_sync(FULL, gc, 1, P);
  const double gm = c ? gp : 0.0;
#pragma unroll
  for (int t = 0; t < M - 1; ++t) rh[t] = rh[t] + lo[t] * gm + up[t] * gc;
  rh[M - 1] = gc;
}

__device__ __forceinline__ void pf_l1(const double* p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }
// 8-byte global -> shared copy that holds no register until it is waited for
__device__ __forceinline__ void cp_async8(double* sdst, const double* gsrc) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
// axes (bit AX) whose build phase stages its inputs with cp.async; measured on
// B200 (C3): faster for the phi tiles (one warp per line), slower for r / theta
#ifndef YY_PSI_EARLY
#define YY_PSI_EARLY 1
#endif
#ifndef YY_LINE_STAGE
#define YY_LINE_STAGE 4
#endif

// L1 prefetch of the per-step row weights coef<Q,AX,true> reads at node (i,j,k)
// of kind K (Astar::av, and the reaction array of an own-direction row)
template <int Q, int AX>
__device__ __forceinline__ void prefetch_rows(const Geo& g, const Astar& A, int i, int j, int k) {
  constexpr int K = kind_of(Q);
  if (use_av(Q, AX, RX_SWEEP)) {
    pf_l1(A.av[AX] + IX<K>(g, i, j, k));
  } else if (AX == 0) {
    pf_l1(A.ar + IX<KR>(g, i, j, k));
    if (K == KT) pf_l1(A.ar + IX<KR>(g, i, j - 1, k));
  } else if (AX == 1) {
    pf_l1(A.at + IX<KT>(g, i, j, k));
    if (K == KR) pf_l1(A.at + IX<KT>(g, i - 1, j, k));
  } else {
    pf_l1(A.ap + IX<KP>(g, i, j, k));
    if (K == KR) pf_l1(A.ap + IX<KP>(g, i - 1, j, k));
    if (K == KT) pf_l1(A.ap + IX<KP>(g, i, j - 1, k));
  }
  if (Q == QUT && AX == 1) pf_l1(A.rt + IX<KT>(g, i, j, k));
  if (Q == QUP && AX == 2) pf_l1(A.rp + IX<KP>(g, i, j, k));
}

// part_solve for a line that is one radial slab of a longer r-line (SURVEY
// §8(e)): row 0 couples (lo_0) to the unknown last row x_lo of the slab below and
// row n-1 = P M - 1 couples (up_{n-1}) to the unknown first row x_hi of the slab
// above.  Returns, per row, x = x0 + xl x_lo + xh x_hi (x0 in rh, xl in lo, xh in
// up): the same elimination, two more right-hand-side columns in the interface
// PCR (the external couplings moved to the right-hand side).  keep_hi requires
// the line to fill the chunks exactly (no identity rows).
template <int P, int M>
__device__ __forceinline__ void part_solve3(double (&lo)[M], double (&up)[M], double (&rh)[M], int c) {
  double cp = 0.0, yp = 0.0, vp = 0.0;
#pragma unroll
  for (int t = 0; t < M - 1; ++t) {
    const double l = lo[t];
    if (t == 0) {
      cp = up[0];
      yp = rh[0];
      vp = -l;
    } else {
      const double inv = frcp(1.0 - l * cp);
      cp = up[t] * inv;
      yp = (rh[t] - l * yp) * inv;
      vp = -l * vp * inv;
    }
    up[t] = cp;
    rh[t] = yp;
    lo[t] = vp;
  }
  {
    double y = rh[M - 2], v = lo[M - 2], w = -up[M - 2];
    up[M - 2] = w;
#pragma unroll
    for (int t = M - 3; t >= 0; --t) {
      const double ct = up[t];
      y = rh[t] - ct * y;
      v = lo[t] - ct * v;
      w = -ct * w;
      rh[t] = y;
      lo[t] = v;
      up[t] = w;
    }
  }
  const double Y0n = __shfl_down_sync(FULL, rh[0], 1, P);
  const double V0n = __shfl_down_sync(FULL, lo[0], 1, P);
  const double W0n = __shfl_down_sync(FULL, up[0], 1, P);
  const double ae = lo[M - 1], ce = up[M - 1];
  const bool last = (c == P - 1);
  double A = ae * lo[M - 2];
  double B = ae * up[M - 2] + 1.0 + (last ? 0.0 : ce * V0n);
  double C = last ? 0.0 : ce * W0n;
  double D = rh[M - 1] - ae * rh[M - 2] - (last ? 0.0 : ce * Y0n);
  double Dl = 0.0, Dh = last ? -ce : 0.0;     // x_hi enters the last row through ce
  if (c == 0) {                               // x_lo enters chunk 0 through v (g_{-1})
    Dl = -A;
    A = 0.0;
  }
#pragma unroll
  for (int s = 1; s < P; s <<= 1) {
    const double iB = frcp(B);
    const double Am = __shfl_up_sync(FULL, A, s, P), iBm = __shfl_up_sync(FULL, iB, s, P);
    const double Cm = __shfl_up_sync(FULL, C, s, P), Dm = __shfl_up_sync(FULL, D, s, P);
    const double Dlm = __shfl_up_sync(FULL, Dl, s, P), Dhm = __shfl_up_sync(FULL, Dh, s, P);
    const double Ap = __shfl_down_sync(FULL, A, s, P), iBp = __shfl_down_sync(FULL, iB, s, P);
    const double Cp = __shfl_down_sync(FULL, C, s, P), Dp = __shfl_down_sync(FULL, D, s, P);
    const double Dlp = __shfl_down_sync(FULL, Dl, s, P), Dhp = __shfl_down_sync(FULL, Dh, s, P);
    const double al = -A * iBm;
    const double ga = -C * iBp;
    B = B + al * Cm + ga * Ap;
    D = D + al * Dm + ga * Dp;
    Dl = Dl + al * Dlm + ga * Dlp;
    Dh = Dh + al * Dhm + ga * Dhp;
    A = al * Am;
    C = ga * Cp;
  }
  const double iB = frcp(B);
  const double g0 = D * iB, gl = Dl * iB, gh = Dh * iB;
  const double g0p = __shfl_up_sync(FULL, g0, 1, P), glp = __shfl_up_sync(FULL, gl, 1, P);
  const double ghp = __shfl_up_sync(FULL, gh, 1, P);
  const double g0m = c ? g0p : 0.0, glm = c ? glp : 1.0, ghm = c ? ghp : 0.0;   // g_{-1} = x_lo
#pragma unroll
  for (int t = 0; t < M - 1; ++t) {
    const double v = lo[t], w = up[t];
    rh[t] = rh[t] + v * g0m + w * g0;
    lo[t] = v * glm + w * gl;
    up[t] = v * ghm + w * gh;
  }
  rh[M - 1] = g0;
  lo[M - 1] = gl;
  up[M - 1] = gh;
}

// normalised row m (0..n-1) of the factor at node (i,j,k); rv = right-hand side
template <int Q, int AX, int RX = RX_SWEEP>
__device__ __forceinline__ void make_row(const Geo& g, const Astar& A, int i, int j, int k, int m, int n,
                                         double rv, double& lo, double& up, double& rh, bool keep_ends = false,
                                         double advin = 0.0, double rxin = 0.0) {
  constexpr int K = kind_of(Q);
  const double th = 0.5 * g.tau;
  double am, a0, ap;
  coef_split<Q, AX, RX>(g, A, i, j, k, am, a0, ap, advin, rxin);
  double di = 1.0 - th * a0;
  if (AX == 0 && K != KR) {          // antisymmetric wall ghost of the increment (RD23)
    if (m == 0 && g.wall_lo) di = 1.0 - th * (a0 - am);
    if (m == n - 1 && g.wall_hi) di = 1.0 - th * (a0 - ap);
  }
  const double inv = frcp(di);
  // line ends: homogeneous Dirichlet increment (fringe, u_r walls) — except the
  // ends of a radial slab that continue in the neighbour slab (keep_ends)
  const bool klo = keep_ends && AX == 0 && !g.wall_lo, khi = keep_ends && AX == 0 && !g.wall_hi;
  lo = (m == 0 && !klo) ? 0.0 : -th * am * inv;
  up = (m == n - 1 && !khi) ? 0.0 : -th * ap * inv;
  rh = rv * inv;
}

// odd line pitch (>= P*MP) of the chunk-major shared-memory tile: rows of 128/P
// consecutive lines are stored conflict-free in the build phase of r/theta tiles
// (lane = line), and chunk reads of the solve phase are <= 2-way conflicted.
template <int P, int MP>
__host__ __device__ constexpr int line_pitch() {
  int best = P * MP + 1, bdeg = 99;
  for (int LP = P * MP + 1; LP < P * MP + 64; LP += 2) {
    int deg = 1;
    for (int h = 0; h < 32; h += 16) {
      int cnt[16] = {};
      for (int t = h; t < h + 16; ++t) {
        const int a = ((t / P) * LP + (t % P) * MP) % 16;
        if (++cnt[a] > deg) deg = cnt[a];
      }
    }
    if (deg < bdeg) { bdeg = deg; best = LP; }
  }
  return best;
}

// ---------------------------------------------------------------------------------
// One kernel for the three axes.  A block (128 threads) owns NL = 128/P lines:
//   AX=0 (r) / AX=1 (theta): NL consecutive k at fixed j / i   (grid x: k tile, y: j / i)
//   AX=2 (phi): NL consecutive lines (i, j), j fastest          (grid x: line tile)
// grid z / y: patch.
// 1. build: M elements per thread (mapping below), coalesced; every thread
//    issues all its M loads before using any;
// 2.-3. thread (line q / P, chunk q % P) solves its chunk in registers;
// 4. write back with the build mapping (FINAL: psi += x and the norm partial).
// ---------------------------------------------------------------------------------
enum { MODE_PLAIN = 0, MODE_FIRST = 1, MODE_FINAL = 2, MODE_SLAB = 3 };

// resident 128-thread blocks per SM the register allocation must allow (the
// chunk arrays are 6 M registers): measured on B200 (C3), 96 registers for
// chunks of <= 12 rows beat the unconstrained ~130 (occupancy over ILP)
#ifndef YY_MINB_3212
#define YY_MINB_3212 4      // phi lines of <= 384 rows: 128 registers, no spills (measured)
#endif
#ifndef YY_MINB_MW
#define YY_MINB_MW 5
#endif
#ifndef YY_MINB_16
#define YY_MINB_16 5        // r/theta (16, 6) / (16, 8) tiles
#endif
#ifndef YY_MINB_M16
#define YY_MINB_M16 3       // chunks of 13-16 rows (C5 theta (16,16)): 168 registers, no spill (measured
                            // faster than 4 blocks at 128 registers with a 76 B spill: C5 100 -> 96 ms/step)
#endif
constexpr int line_minb(int P, int M) {
  return YY_LINE_MINB > 0 ? YY_LINE_MINB
         : P > 32 ? (M <= 6 ? YY_MINB_MW : 4)   // multi-warp phi lines (part_solve3: 3 live arrays)
         : (P == 32 && M == 12) ? YY_MINB_3212
         : (P == 16 && M <= 8) ? YY_MINB_16
         : (P == 8 && M == 12) ? 4          // theta (8, 12): 128 registers, no spills
         : (P == 16 && M == 12) ? 4
                  : (M <= 12 ? 5 : M <= 16 ? YY_MINB_M16 : M <= 24 ? 2 : 1);
}

template <int Q, int AX, int MODE, int S, int P, int M>
__global__ void __launch_bounds__(128, line_minb(P, M)) k_line(Geo g, SweepArgs a, ResidArgs ra) {
  const uint3 B = bidx(a.rev);
  constexpr bool FINAL = (MODE == MODE_FINAL);
  constexpr int K = kind_of(Q);
  constexpr int NL = 128 / P;
  constexpr int MP = M | 1;
  constexpr int LP = line_pitch<P, MP>();
  extern __shared__ double sm[];
  double* LO = sm;
  double* UP = LO + NL * LP;
  double* RH = UP + NL * LP;
  const int patch = (AX == 2) ? B.y : B.z;
  const int n = (AX == 0) ? i_hi<K>(g) - i_lo<K>(g) + 1 : (AX == 1) ? NTk(g, K) - 2 : NPk(g, K) - 2;
  const long long po = patch * psize(g, K);
  Astar A{a.ar + patch * psize(g, KR), a.at + patch * psize(g, KT), a.ap + patch * psize(g, KP),
          a.rt + patch * psize(g, KT), a.rp + patch * psize(g, KP)};
  bind_adv<K>(g, A, patch);
  double* __restrict__ R = a.R + po;
  // Element u (< M) of this thread in the build / write-back phases:
  //  r/theta: line l = t % NL (consecutive threads = consecutive k, coalesced),
  //           rows e = c M + u of chunk c = t / NL (a thread walks its chunk);
  //  phi:     line l = t / P (P threads per line), row e = t % P + P u (coalesced
  //           along the line).
  // Out-of-range elements (ragged tile / padded rows) re-read a valid node and
  // become identity rows: no load sits behind a branch.
  static_assert(AX != 2 || P % 32 == 0, "phi tiles: whole warps per line");
  static_assert(AX == 2 || P <= 32, "r/theta tiles: a line's chunks within one warp");
  static_assert(P <= 32 || MODE != MODE_SLAB, "slab r-lines: one warp per line");
  int lt, c1, nlines, L0, stride, i0 = 0, j0 = 0, k0 = 0, nd0 = 0;
  // phi: the line of this thread (P threads per line) and its (i, j) and node at k = 1
  int li = 0, lj = 0, lnd = 0;
  auto line_of = [&](int t) {
    const int nj = NTk(g, K) - 2;
    const int L = min(L0 + t / P, nlines - 1);   // clamped: a ragged tile reads valid nodes
    li = i_lo<K>(g) + L / nj;
    lj = 1 + L % nj;
    lnd = IX<K>(g, li, lj, 1);
  };
  if (AX == 2) {
    nlines = (i_hi<K>(g) - i_lo<K>(g) + 1) * (NTk(g, K) - 2);
    L0 = B.x * NL;
    line_of(threadIdx.x);
    lt = 0;
    c1 = 0;
    stride = 1;
  } else {
    lt = threadIdx.x % NL;
    c1 = threadIdx.x / NL;
    L0 = B.x * NL + 1;             // first k of the tile
    nlines = NPk(g, K) - 2 - L0 + 1;      // lines of this tile that exist (may exceed NL)
    k0 = L0 + min(lt, nlines - 1);
    if (AX == 0) { i0 = i_lo<K>(g); j0 = B.y + 1; stride = NTk(g, K) * NPk(g, K); }
    else { i0 = B.y + i_lo<K>(g); j0 = 1; stride = NPk(g, K); }
    nd0 = IX<K>(g, i0, j0, k0);
  }
  const bool lvalid = (AX == 2) || lt < nlines;
  auto elem = [&](int u, int& l, int& e) {
    if (AX == 2) { l = threadIdx.x / P; e = threadIdx.x % P + P * u; }
    else { l = lt; e = c1 * M + u; }
  };
  auto exists = [&](int l, int e) { return e < n && (AX == 2 ? L0 + l < nlines : lvalid); };
  auto node = [&](int l, int e, int& i, int& j, int& k) {   // l, e clamped by the caller
    if (AX == 0) { i = i0 + e; j = j0; k = k0; return nd0 + e * stride; }
    if (AX == 1) { i = i0; j = j0 + e; k = k0; return nd0 + e * stride; }
    i = li; j = lj; k = 1 + e;
    return lnd + e;
  };
  // chunk-major slot of row e of line l.  r/theta elements come from elem(), so
  // e = c1 M + u and the slot is lt LP + c1 MP + u: one base per thread, the row
  // an immediate (no division by M per element)
  const int sbase = lt * LP + c1 * MP;
  auto slot = [&](int l, int e) {
    if constexpr (AX != 2) return sbase + (e - c1 * M);
    else return l * LP + (e / M) * MP + (e % M);
  };
  // the same for element u of elem(): phi rows e = lane + P u, so e / M and e % M
  // follow from lane / M, lane % M (once) and the compile-time (P u) / M, (P u) % M
  const int lane_ = (AX == 2) ? (int)(threadIdx.x % P) : 0;
  const int q0 = lane_ / M, r0 = lane_ % M, lb = (AX == 2) ? (int)(threadIdx.x / P) * LP : 0;
  auto slot_u = [&](int u) {
    if constexpr (AX != 2) {
      return sbase + u;
    } else {
      int r = r0 + (P * u) % M, q = q0 + (P * u) / M;
      if (r >= M) { r -= M; ++q; }
      return lb + q * MP + r;
    }
  };
  // 1. build
  if (MODE == MODE_FIRST) {
    // fused eq:er residual: one element at a time (its stencil loads are many and
    // mostly L1 hits of neighbouring threads); occupancy hides the latency
#pragma unroll 2
    for (int u = 0; u < M; ++u) {
      int l, e, i, j, k;
      elem(u, l, e);
      const int ec = min(e, n - 1);
      node(l, ec, i, j, k);
      const double rv = resid_at<Q, S>(g, ra, patch, i, j, k);
      double lo, up, rh;
      make_row<Q, AX>(g, A, i, j, k, ec, n, rv, lo, up, rh);
      const double mk = exists(l, e) ? 1.0 : 0.0;     // identity row outside the tile
      const int s = slot_u(u);
      LO[s] = lo * mk;
      UP[s] = up * mk;
      RH[s] = rh * mk;
    }
  } else if ((YY_LINE_STAGE >> AX) & 1) {
    // every input value of the tile goes to shared memory with cp.async (no
    // registers held, so all of a thread's loads are in flight at once): the
    // right-hand side into the RH slot, the per-step row weight (Astar::av) into
    // LO and the own-direction reaction into UP; the rows are then built in place
    constexpr bool AVG = use_av(Q, AX, RX_SWEEP);
    constexpr bool RXR = (Q == QUT && AX == 1) || (Q == QUP && AX == 2);
    // phi: per-thread line base pointers and 32-bit row offsets (immediates for
    // the unrolled elements); rows past the line end are zero-filled, not loaded
    const double* __restrict__ Rb = R + lnd;
    const double* __restrict__ Vb = A.av[AX] + lnd;
    const double* __restrict__ Xb = (Q == QUT ? A.rt : A.rp) + lnd;
#pragma unroll
    for (int u = 0; u < M; ++u) {
      int l, e, i, j, k;
      elem(u, l, e);
      const int s = slot_u(u);
      if (AX == 2 && AVG) {
        if (e < n && a.noadv) {           // IMEX: no transport terms in the rows
          cp_async8(RH + s, Rb + e);
          LO[s] = 0.0;
          UP[s] = 0.0;
        } else if (e < n) {
          cp_async8(RH + s, Rb + e);
          cp_async8(LO + s, Vb + e);
          if (RXR) cp_async8(UP + s, Xb + e);
        } else {
          RH[s] = 0.0;
          LO[s] = 0.0;
          UP[s] = 0.0;
        }
      } else {
        const int nd = node(l, min(e, n - 1), i, j, k);
        cp_async8(RH + s, R + nd);
        if (AVG) cp_async8(LO + s, A.av[AX] + nd);
        else prefetch_rows<Q, AX>(g, A, i, j, k);
        if (AVG && RXR) cp_async8(UP + s, (Q == QUT ? A.rt : A.rp) + nd);
      }
    }
    cp_async_wait_all();
#pragma unroll
    for (int u = 0; u < M; ++u) {
      int l, e, i, j, k;
      elem(u, l, e);
      const int ec = min(e, n - 1);
      node(l, ec, i, j, k);
      const int s = slot_u(u);
      double lo, up, rh;
      make_row<Q, AX, AVG ? RX_GIVEN : RX_SWEEP>(g, A, i, j, k, ec, n, RH[s], lo, up, rh, MODE == MODE_SLAB,
                                                 AVG ? LO[s] : 0.0, (AVG && RXR) ? UP[s] : 0.0);
      const double mk = exists(l, e) ? 1.0 : 0.0;     // identity row outside the tile
      LO[s] = lo * mk;
      UP[s] = up * mk;
      RH[s] = rh * mk;
    }
  } else {
    // the transport-velocity rows coef<> reads for these elements go to L1 first
    // (no registers held), so make_row below finds them there instead of paying a
    // DRAM round trip per element
    if (!a.noadv) {
#pragma unroll
      for (int u = 0; u < M; ++u) {
        int l, e, i, j, k;
        elem(u, l, e);
        node(l, min(e, n - 1), i, j, k);
        prefetch_rows<Q, AX>(g, A, i, j, k);
      }
    }
    double rv[M];
#pragma unroll
    for (int u = 0; u < M; ++u) {
      int l, e, i, j, k;
      elem(u, l, e);
      rv[u] = R[node(l, min(e, n - 1), i, j, k)];
    }
    // (the IMEX branch is taken once per block, outside the unrolled rows, so the
    // default path keeps its load batching)
    auto build = [&](auto noadv) {
#pragma unroll
      for (int u = 0; u < M; ++u) {
        int l, e, i, j, k;
        elem(u, l, e);
        const int ec = min(e, n - 1);
        node(l, ec, i, j, k);
        double lo, up, rh;
        if constexpr (decltype(noadv)::value)   // IMEX: the a* = 0 rows, no per-step weight read
          make_row<Q, AX, RX_GIVEN>(g, A, i, j, k, ec, n, rv[u], lo, up, rh, MODE == MODE_SLAB, 0.0, 0.0);
        else
          make_row<Q, AX>(g, A, i, j, k, ec, n, rv[u], lo, up, rh, MODE == MODE_SLAB);
        const double mk = exists(l, e) ? 1.0 : 0.0;     // identity row outside the tile
        const int s = slot_u(u);
        LO[s] = lo * mk;
        UP[s] = up * mk;
        RH[s] = rh * mk;
      }
    };
#if YY_IMEX_FAST
    if (a.noadv) build(std::true_type{});
    else
#endif
      build(std::false_type{});
  }
  // r/theta final sweeps (YY_PSI_EARLY): psi of the tile is loaded into registers
  // before the solve, so its DRAM latency overlaps the solve
  double pv[M];
  // (chunks of more than 8 rows keep psi out of the solve's registers: the
  // u_theta (16,16) final sweep of C5 spilled 144 B with it)
  constexpr bool PSE = FINAL && AX != 2 && YY_PSI_EARLY && M <= 8;
  if (PSE) {
#pragma unroll
    for (int u = 0; u < M; ++u) {
      int l, e, i, j, k;
      elem(u, l, e);
      pv[u] = a.psi[po + node(l, min(e, n - 1), i, j, k)];
    }
  }
  __syncthreads();
  // 2.-3. solve chunk c of line l
  {
    const int l = threadIdx.x / P, c = threadIdx.x % P;
    const int o = l * LP + c * MP;
    double lo[M], up[M], rh[M];
#pragma unroll
    for (int u = 0; u < M; ++u) {
      lo[u] = LO[o + u];
      up[u] = UP[o + u];
      rh[u] = RH[o + u];
    }
    if constexpr (P > 32) {
      // long phi lines: W = P/32 warps per line.  Each warp solves its segment
      // with the couplings to the neighbour segments kept symbolic (part_solve3,
      // as for radial slabs), x = x0 + xlo X_LO + xhi X_HI; the 2W boundary
      // unknowns of the line (first / last row of every segment) are then
      // eliminated by one thread, and every thread finishes its chunk.
      constexpr int W = P / 32;
      __shared__ double s_if[NL * W][6], s_lh[NL * W][2];
      const int lane = threadIdx.x & 31, sg = threadIdx.x >> 5;   // segment (line sg / W)
      part_solve3<32, M>(lo, up, rh, lane);
      if (lane == 0) { s_if[sg][0] = rh[0]; s_if[sg][1] = lo[0]; s_if[sg][2] = up[0]; }
      if (lane == 31) { s_if[sg][3] = rh[M - 1]; s_if[sg][4] = lo[M - 1]; s_if[sg][5] = up[M - 1]; }
      __syncthreads();
      if (threadIdx.x < NL) {
        // a_s = first row, b_s = last row of segment s:
        //   a_s = x0_f + xlo_f b_{s-1} + xhi_f a_{s+1},  b_s = x0_l + xlo_l b_{s-1} + xhi_l a_{s+1}
        // forward: b_{s-1} = be + ga a_s  ->  a_s = p_s + q_s a_{s+1}; back: a_W = 0
        const double(*f)[6] = s_if + threadIdx.x * W;
        double p[W], q[W], bb[W], gg[W];
        double be = 0.0, ga = 0.0;
#pragma unroll
        for (int s2 = 0; s2 < W; ++s2) {
          const double d = 1.0 / (1.0 - f[s2][1] * ga);
          p[s2] = (f[s2][0] + f[s2][1] * be) * d;
          q[s2] = f[s2][2] * d;
          bb[s2] = be;
          gg[s2] = ga;
          be = f[s2][3] + f[s2][4] * (be + ga * p[s2]);
          ga = f[s2][4] * ga * q[s2] + f[s2][5];
        }
        double an = 0.0;                         // a_{s+1}
#pragma unroll
        for (int s2 = W - 1; s2 >= 0; --s2) {
          const double as = p[s2] + q[s2] * an;
          s_lh[threadIdx.x * W + s2][0] = bb[s2] + gg[s2] * as;   // b_{s-1} (0 for s = 0)
          s_lh[threadIdx.x * W + s2][1] = an;
          an = as;
        }
      }
      __syncthreads();
      const double XL = s_lh[sg][0], XH = s_lh[sg][1];
#pragma unroll
      for (int u = 0; u < M; ++u) RH[o + u] = rh[u] + lo[u] * XL + up[u] * XH;
    } else if constexpr (MODE == MODE_SLAB) {
      if (a.vw) {
        // the step's first iteration: x0 and the responses xlo, xhi to the
        // neighbour slabs' boundary unknowns (per step: they depend on the matrix only)
        part_solve3<P, M>(lo, up, rh, c);
#pragma unroll
        for (int u = 0; u < M; ++u) {
          RH[o + u] = rh[u];
          LO[o + u] = lo[u];
          UP[o + u] = up[u];
        }
      } else {
        // later iterations: x0 alone (the couplings to the neighbour slabs zero)
        if (c == 0) lo[0] = 0.0;
        if (c == P - 1) up[M - 1] = 0.0;
        part_solve<P, M>(lo, up, rh, c);
#pragma unroll
        for (int u = 0; u < M; ++u) RH[o + u] = rh[u];
      }
    } else {
      part_solve<P, M>(lo, up, rh, c);
#pragma unroll
      for (int u = 0; u < M; ++u) RH[o + u] = rh[u];
    }
  }
  __syncthreads();
  // 4. write back
  if (AX == 2) {
    // recomputed (not kept live in registers across the solve)
    int t = threadIdx.x;
    asm volatile("" : "+r"(t));
    line_of(t);
  }
  double wsum = 0.0;
  if constexpr (AX == 2 && MODE != MODE_SLAB) {
    // phi: line base pointers, 32-bit row offsets, predicated (not clamped) rows
    double* __restrict__ Pw = a.psi + po + lnd;
    double* __restrict__ Rw = R + lnd;
    const bool lv = L0 + (int)threadIdx.x / P < nlines;
    if (FINAL) {
#pragma unroll
      for (int u = 0; u < M; ++u) {
        int l, e;
        elem(u, l, e);
        pv[u] = (e < n) ? Pw[e] : 0.0;
      }
    }
    const double rs = FINAL ? rnode<K>(g, li) * rnode<K>(g, li) * snode<K>(g, lj) : 0.0;
#pragma unroll
    for (int u = 0; u < M; ++u) {
      int l, e;
      elem(u, l, e);
      if (lv && e < n) {
        const double x = RH[slot_u(u)];
        if (FINAL) {
          Pw[e] = pv[u] + x;
          wsum += rs * x * x;
        } else {
          Rw[e] = x;
        }
      }
    }
  } else {
  if (FINAL && !PSE) {
#pragma unroll
    for (int u = 0; u < M; ++u) {
      int l, e, i, j, k;
      elem(u, l, e);
      pv[u] = a.psi[po + node(l, min(e, n - 1), i, j, k)];
    }
  }
#pragma unroll
  for (int u = 0; u < M; ++u) {
    int l, e, i, j, k;
    elem(u, l, e);
    if (exists(l, e)) {
      const int nd = node(l, e, i, j, k);
      const double x = RH[slot_u(u)];
      if (FINAL) {
        a.psi[po + nd] = pv[u] + x;
        const double r = rnode<K>(g, i), s = snode<K>(g, j);
        wsum += r * r * s * x * x;
      } else if (MODE == MODE_SLAB) {
        R[nd] = x;
        double* f = (e == 0 || e == n - 1)    // this slab's boundary rows of the line
                        ? a.IF + 6LL * ((j - 1) * (NPk(g, K) - 2) + (k - 1)) + (e == 0 ? 0 : 3) : nullptr;
        if (a.vw) {                           // (per step: the line's responses to its couplings)
          const double xl = LO[slot_u(u)], xh = UP[slot_u(u)];
          a.V[po + nd] = xl;
          a.W[po + nd] = xh;
          if (f) { f[1] = xl; f[2] = xh; }
        }
        if (f) f[0] = x;
      } else {
        R[nd] = x;
      }
    }
  }
  }
  if (FINAL) {
    wsum *= g.dr * g.dth * g.dph;
    __shared__ double sh[4];
    for (int o = 16; o > 0; o >>= 1) wsum += __shfl_down_sync(FULL, wsum, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = wsum;
    __syncthreads();
    if (threadIdx.x == 0) {
      const int b = (AX == 2) ? B.x : B.y * gridDim.x + B.x;
      a.part[(long long)patch * a.maxb + b] = (sh[0] + sh[1]) + (sh[2] + sh[3]);
    }
  }
}

// ---------------------------------------------------------------------------------
// theta sweeps with TMA-staged tiles (plain and final factors).
// The same tile (NL = 128/P consecutive k-lines of one (j | i, patch)) and the same
// chunk algebra as k_line, but the tile's inputs (right-hand side, row weight
// Astar::av, the u_theta reaction, FINAL psi) arrive by cp.async.bulk.tensor
// (one elected thread, one mbarrier) as [row][line] boxes in shared memory, and
// the result leaves by a bulk tensor store: the global traffic bypasses the LSU /
// L1 data pipe, which ncu shows at ~73 % of its wavefront peak in k_line
// (profiles/r02_ncu.md).  The build reads four consecutive rows of eight lines per
// warp instruction (256 contiguous bytes: conflict-free), so its 1-D table reads
// are one wavefront.  Eligible kinds: row pitch a multiple of 16 B (nphi even;
// the u_phi kind's nphi + 1 is not — it keeps k_line).
// ---------------------------------------------------------------------------------
struct TmaMaps {
  CUtensorMap m[4];          // rhs (R), Astar::av, reaction rt (u_theta theta), psi (FINAL)
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
      ::"r"(smem_u32(dst)), "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2) : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4}], [%1];"
               ::"l"(map), "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2) : "memory");
}

template <int Q, int AX, bool FINAL>
__host__ __device__ constexpr int tma_narr() { return 2 + ((Q == QUT && AX == 1) ? 1 : 0) + (FINAL ? 1 : 0); }

template <int Q, int AX, int MODE, int P, int M>
__global__ void __launch_bounds__(128, line_minb(P, M)) k_line_tma(Geo g, SweepArgs a, const __grid_constant__ TmaMaps maps) {
  static_assert(AX != 2 && (MODE == MODE_PLAIN || MODE == MODE_FINAL), "r / theta plain or final sweeps");
  static_assert(use_av(Q, AX, RX_SWEEP), "the staged rows take the per-step weights Astar::av");
  const uint3 B = bidx(a.rev);
  constexpr bool FINAL = (MODE == MODE_FINAL);
  constexpr bool RXR = (Q == QUT && AX == 1);
  constexpr int K = kind_of(Q);
  constexpr int NL = 128 / P;
  constexpr int MP = M | 1;
  constexpr int LP = line_pitch<P, MP>();
  constexpr int NPAD = P * M;
  constexpr int SA = (NPAD * NL + 15) / 16 * 16;      // one staged array (128-B multiple)
  constexpr int NA = tma_narr<Q, AX, FINAL>();
  // the staged inputs (FINAL: rhs; av; reaction) and the chunk-major solve tile
  // share the front of shared memory (the inputs are read into registers first);
  // the box that is written back follows — FINAL psi, PLAIN the rhs itself — so
  // that the phi-fringe columns of the tile (k = 0, nphi - 1) go back unchanged
  constexpr int NIN = NA - 1;
  constexpr int FRONT = NIN * SA > 3 * NL * LP ? NIN * SA : 3 * NL * LP;
  extern __shared__ __align__(128) double sm[];
  double* Sps = sm + (FRONT + 15) / 16 * 16;          // [row][line] boxes: psi (FINAL) / rhs (PLAIN)
  double* Srh = FINAL ? sm : Sps;
  double* Sav = sm + (FINAL ? SA : 0);
  double* Srx = Sav + SA;
  double* LO = sm;                                    // chunk-major solve tile (as k_line)
  double* UP = LO + NL * LP;
  double* RH = UP + NL * LP;
  __shared__ __align__(8) uint64_t bar;
  const int patch = B.z;
  const int n = (AX == 0) ? i_hi<K>(g) - i_lo<K>(g) + 1 : NTk(g, K) - 2;
  // tiles start at k = 0 (the phi-fringe column, an identity line): a bulk tensor
  // box must start on a 16-B boundary, i.e. at an even k for fp64 (measured: an odd
  // start is an illegal instruction, tools/tma_align_probe.cu)
  const int k0 = B.x * NL;
  auto lvalid = [&](int l) { return k0 + l >= 1 && k0 + l <= NPk(g, K) - 2; };
  int i0, j0;
  if (AX == 0) { i0 = i_lo<K>(g); j0 = B.y + 1; }
  else { i0 = B.y + i_lo<K>(g); j0 = 1; }
  // box origin (k, j, patch-folded r row)
  const int c0 = k0, c1 = j0, c2 = patch * NRk(g, K) + i0;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const uint32_t bytes = (uint32_t)(NA * n * NL * sizeof(double));
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(bytes) : "memory");
    tma_load_3d(Srh, &maps.m[0], &bar, c0, c1, c2);
    tma_load_3d(Sav, &maps.m[1], &bar, c0, c1, c2);
    if (RXR) tma_load_3d(Srx, &maps.m[2], &bar, c0, c1, c2);
    if (FINAL) tma_load_3d(Sps, &maps.m[3], &bar, c0, c1, c2);
  }
  (void)NIN;
  // the factor-row table of the tile's rows (Geo::tsplit: lo0, b0, up0 per row) and,
  // FINAL, the norm weights r^2 sin(theta) into shared memory while the boxes are in
  // flight: the row build reads no global tables (their L2 latency was the largest
  // stall of this kernel, profiles/r02_ncu.md)
  double* St = Sps + SA;
  double* Sw = St + 3 * NPAD;
  {
    const double* __restrict__ T3 = g.tsplit[Q][AX] + 3 * (i0 * NTk(g, K) + j0);
    const int tstride = (AX == 0) ? 3 * NTk(g, K) : 3;
    for (int e = threadIdx.x; e < 3 * n; e += 128) St[e] = __ldg(T3 + (e / 3) * tstride + e % 3);
    if (FINAL)
      for (int m = threadIdx.x; m < n; m += 128) {
        const int i = (AX == 0) ? i0 + m : i0, j = (AX == 0) ? j0 : j0 + m;
        const double r = rnode<K>(g, i);
        Sw[m] = r * r * snode<K>(g, j);
      }
  }
  __syncthreads();                                    // the barrier is initialised
  const double th = 0.5 * g.tau;
  const int lt = threadIdx.x % NL, rg = threadIdx.x / NL;   // build / write-back: line, row group
  auto slot = [&](int l, int e) { return l * LP + (e / M) * MP + (e % M); };
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra WAIT_%=;\n}\n"
      ::"r"(smem_u32(&bar)) : "memory");
  // 1. build: element u of this thread is row e = u P + rg of line lt; the staged
  //    values go to registers first (their space is the solve tile's)
  double vr[M], va[M], vx[M];
#pragma unroll
  for (int u = 0; u < M; ++u) {
    const int q = min(u * P + rg, n - 1) * NL + lt;
    vr[u] = Srh[q];
    va[u] = a.noadv ? 0.0 : Sav[q];
    vx[u] = (RXR && !a.noadv) ? Srx[q] : 0.0;
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < M; ++u) {
    const int e = u * P + rg;
    const int ec = min(e, n - 1);
    // the row of make_row from the folded table: raw weights, then normalised by
    // the diagonal (line ends: homogeneous Dirichlet increments)
    const double lr = fma(-th, va[u], St[3 * ec]), ur = fma(th, va[u], St[3 * ec + 2]);
    double bm = fma(th, vx[u], St[3 * ec + 1]);
    if (AX == 0 && K != KR) {            // antisymmetric wall ghost of the increment (RD23)
      if (ec == 0 && g.wall_lo) bm -= lr;
      if (ec == n - 1 && g.wall_hi) bm -= ur;
    }
    const double inv = frcp(bm);
    const double lo = (ec == 0) ? 0.0 : lr * inv, up = (ec == n - 1) ? 0.0 : ur * inv, rh = vr[u] * inv;
    const double mk = (e < n && lvalid(lt)) ? 1.0 : 0.0;
    const int s = slot(lt, e);
    LO[s] = lo * mk;
    UP[s] = up * mk;
    RH[s] = rh * mk;
  }
  __syncthreads();
  // 2.-3. solve chunk c of line l (as k_line)
  {
    const int l = threadIdx.x / P, c = threadIdx.x % P;
    const int o = l * LP + c * MP;
    double lo[M], up[M], rh[M];
#pragma unroll
    for (int u = 0; u < M; ++u) {
      lo[u] = LO[o + u];
      up[u] = UP[o + u];
      rh[u] = RH[o + u];
    }
    part_solve<P, M>(lo, up, rh, c);
#pragma unroll
    for (int u = 0; u < M; ++u) RH[o + u] = rh[u];
  }
  __syncthreads();
  // 4. the result into the [row][line] box (FINAL: psi + x and the norm), then one
  //    bulk tensor store (rows past n lie outside the box; the fringe columns
  //    k = 0, nphi - 1 carry x = 0, i.e. they write back their own values)
  double wsum = 0.0;
  double* out = Sps;
#pragma unroll
  for (int u = 0; u < M; ++u) {
    const int e = u * P + rg;
    if (e < n && lvalid(lt)) {
      const int q = e * NL + lt;
      const double x = RH[slot(lt, e)];
      if (FINAL) {
        out[q] = Sps[q] + x;
        wsum += Sw[e] * x * x;
      } else {
        out[q] = x;
      }
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    tma_store_3d(FINAL ? &maps.m[3] : &maps.m[0], out, c0, c1, c2);
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  if (FINAL) {
    wsum *= g.dr * g.dth * g.dph;
    __shared__ double sh[4];
    for (int o = 16; o > 0; o >>= 1) wsum += __shfl_down_sync(FULL, wsum, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = wsum;
    __syncthreads();
    if (threadIdx.x == 0)
      a.part[(long long)patch * a.maxb + B.y * gridDim.x + B.x] = (sh[0] + sh[1]) + (sh[2] + sh[3]);
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

// ---------------------------------------------------------------------------------
// r and theta sweeps, one line per thread (Thomas), in place in shared memory.
// A block is ONE warp (TWO: two warps, one per end of the lines, see the kernel)
// and owns 32 consecutive k-lines of one (j | i, patch): the
// tile's inputs arrive by cp.async.bulk.tensor as [row][line] boxes (256-B rows)
// in TH_RC-row chunks (one mbarrier each, so the elimination starts on the first
// chunk while the others are in flight); lane k eliminates its line top-down,
// overwriting the right-hand side with d' and the row weight with c', then
// back-substitutes bottom-up; x leaves by one bulk tensor store (r) or straight
// to global memory in coalesced 256-B rows (theta; FINAL: psi + x, psi read two
// row groups ahead from L2, where a bulk tensor prefetch put the box at the start).  Per element one reciprocal, no shuffles, no chunk algebra: the
// instruction count of the partitioned k_line (~135 per element, profiles/
// r02_ncu.md) drops to the row build (one folded table row, Geo::tsplit) +
// Thomas.  The phi-fringe lanes (k = 0, nphi - 1) and lanes past the array
// compute but never store (their rhs goes back unchanged).  Eligible: kinds with
// an even phi pitch (16-B box origins), n <= 256.
// ---------------------------------------------------------------------------------
constexpr int TH_RC = 32;         // rows per load chunk (box rows)

// r / theta sweeps that run one line per thread: measured on B200 (C3) every
// eligible one except the u_theta theta final factor (three staged arrays: two
// blocks per SM), which keeps k_line_tma
__host__ __device__ constexpr bool th_route(int Q, int AX, int MODE) {
  return AX != 2 && (MODE == 0 || MODE == 2);
}
// the u_theta theta final factor (three staged arrays) on k_line_th: env YY_TH_UTF
// (default 0: k_line_tma)
inline bool use_th_utf() {
  static const bool v = [] {
    const char* e = getenv("YY_TH_UTF");
    return e && e[0] == '1';
  }();
  return v;
}
#ifndef YY_TH_G
#define YY_TH_G 16
#endif
// rows per elimination group (ILP across the group; measured on B200: 16 beats 8
// by 3-5 %, 4 loses 8 %, 32 spills)
constexpr int TH_G = YY_TH_G;

__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* map, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];"
               ::"l"(map), "r"(c0), "r"(c1), "r"(c2) : "memory");
}

// PAIR (theta lines of a kind whose phi pitch is odd, plain factor, no reaction
// array): the tensor maps see the (theta, phi) plane as rows of theta PAIRS
// (pitch 2 NP, a multiple of 16 B); a 32-row chunk arrives as two boxes, the 16
// odd-theta rows (inner origin NP + k0 - 1: 34 wide, the lane's value at +1) and
// the 16 even-theta rows (origin k0, 32 wide), PAIR_CH doubles per chunk
constexpr int PAIR_ODD = 16 * 34, PAIR_CH = PAIR_ODD + 16 * 32;

// TWO (two-way elimination, "burn at both ends"): the block is two warps on the
// same 32 lines; warp 0 eliminates rows 0 .. H0-1 top-down, warp 1 rows NPAD-1 ..
// H0 bottom-up (the mirrored recurrence: lower and upper weights swapped), they
// meet at the 2x2 system of rows H0-1 / H0 and back-substitute outwards.  Same
// shared-memory footprint, twice the warps per SM, half the serial chain.
template <int Q, int AX, int MODE, bool PAIR = false, bool TWO = false>
__global__ void __launch_bounds__(TWO ? 64 : 32) k_line_th(Geo g, SweepArgs a, const __grid_constant__ TmaMaps maps) {
  static_assert(AX != 2 && (MODE == MODE_PLAIN || MODE == MODE_FINAL), "r / theta plain or final sweeps");
  static_assert(!PAIR || (AX == 1 && MODE == MODE_PLAIN && !(Q == QUT && AX == 1)), "pair tiles: theta, plain, no reaction");
  const uint3 B = bidx(a.rev);
  constexpr bool FINAL = (MODE == MODE_FINAL);
  constexpr bool RXR = (Q == QUT && AX == 1);
  constexpr int K = kind_of(Q);
  // rows per elimination group: 16 on one warp; 8 for the two-way form (measured on
  // B200: theta plain +5-7 %, u_r r final +4.5 %, profiles/r02_th2_g8_ab.txt — half
  // the unrolled code per direction in the instruction cache)
  constexpr int G = TWO ? 8 : TH_G;
  constexpr int NT = TWO ? 64 : 32;
  static_assert(!PAIR || G % 2 == 0, "pair tiles: row parity from the group offset");
  static_assert(16 % G == 0, "the halves of a two-way tile (NPAD / 2 rows) and the 32-row chunks in whole groups");
  const int patch = B.z;
  const int n = (AX == 0) ? i_hi<K>(g) - i_lo<K>(g) + 1 : NTk(g, K) - 2;
  const int nch = (n + TH_RC - 1) / TH_RC;
  const int NPAD = nch * TH_RC;
  const int H0 = TWO ? NPAD / 2 : NPAD;               // rows [0, H0): top-down; [H0, NPAD): bottom-up
  const int SA = nch * (PAIR ? PAIR_CH : TH_RC * 32);  // one staged array (doubles)
  extern __shared__ __align__(128) double sm[];
  double* Sd = sm;                                    // rhs -> d' -> x
  double* Sc = Sd + SA;                               // Astar::av -> c'
  double* Sx = Sc + SA;                               // u_theta reaction (RXR)
  __shared__ __align__(8) uint64_t bar[8];            // <= 8 chunks
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int wid = TWO ? tid >> 5 : 0;
  auto sync_block = [&]() {
    if constexpr (TWO) __syncthreads();
    else __syncwarp();
  };
  int i0, j0;
  if (AX == 0) { i0 = i_lo<K>(g); j0 = B.y + 1; }
  else { i0 = B.y + i_lo<K>(g); j0 = 1; }
  // box origin (phi, theta, patch-folded r).  FLAT (r lines of a kind whose phi
  // pitch is odd): the map's inner dimension is the whole (theta, phi) plane, the
  // tile starts at an odd k on odd-parity rows so that the box origin stays on a
  // 16-B boundary
  const int k0 = B.x * 32 + (a.flat ? (j0 * NPk(g, K)) & 1 : 0);
  const int k = k0 + lane;
  const bool valid = k >= 1 && k <= NPk(g, K) - 2;
  const int kk = min(max(k, 1), NPk(g, K) - 2);
  const int c0 = a.flat ? j0 * NPk(g, K) + k0 : k0, c1 = a.flat ? 0 : j0, c2 = patch * NRk(g, K) + i0;
  // rows of this lane's line: element m at Rl + m rs (Rl clamped to a valid node)
  const int rs = (AX == 0) ? SR<K>(g) : ST<K>(g);
  const long long lofs = patch * psize(g, K) + IX<K>(g, i0, j0, kk);
  if (tid == 0) {
    for (int c = 0; c < nch; ++c)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[c])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // IMEX (noadv): the rows carry no transport terms, only the rhs is staged
    const int NIN = a.noadv ? 1 : 2 + (RXR ? 1 : 0);
    const uint32_t cb = (uint32_t)((PAIR ? PAIR_CH : TH_RC * 32) * sizeof(double));
    for (int cc = 0; cc < nch; ++cc) {
      // TWO: the chunks from both ends inwards (each warp starts on its own end)
      const int c = TWO ? ((cc & 1) ? nch - 1 - (cc >> 1) : (cc >> 1)) : cc;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[c])), "r"(NIN * cb)
                   : "memory");
      if constexpr (PAIR) {
        // rows j0 + 32 c + u: u even -> theta pair (j0 - 1) / 2 + 16 c + u / 2 at
        // inner NP + k; u odd -> pair (j0 + 1) / 2 + 16 c + (u - 1) / 2 at inner k
        const int o = c * PAIR_CH, t0 = (j0 - 1) / 2 + 16 * c;
        tma_load_3d(Sd + o, &maps.m[0], &bar[c], NPk(g, K) + k0 - 1, t0, c2);
        tma_load_3d(Sd + o + PAIR_ODD, &maps.m[2], &bar[c], k0, t0 + 1, c2);
        if (!a.noadv) {
          tma_load_3d(Sc + o, &maps.m[1], &bar[c], NPk(g, K) + k0 - 1, t0, c2);
          tma_load_3d(Sc + o + PAIR_ODD, &maps.m[3], &bar[c], k0, t0 + 1, c2);
        }
        continue;
      }
      const int o = c * TH_RC * 32;
      const int r1 = AX == 1 ? c1 + c * TH_RC : c1, r2 = AX == 0 ? c2 + c * TH_RC : c2;
      tma_load_3d(Sd + o, &maps.m[0], &bar[c], c0, r1, r2);
      if (!a.noadv) {
        tma_load_3d(Sc + o, &maps.m[1], &bar[c], c0, r1, r2);
        if (RXR) tma_load_3d(Sx + o, &maps.m[2], &bar[c], c0, r1, r2);
      }
    }
    if (FINAL) tma_prefetch_3d(&maps.m[3], c0, c1, c2);
  }
  sync_block();
  const double th = 0.5 * g.tau;
  auto wait = [&](int c) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra WAIT_%=;\n}\n"
        ::"r"(smem_u32(&bar[c])) : "memory");
  };
  // staged index of row m0 + u of this lane's line (m0 a multiple of 16, u < 16:
  // the parity of the row is u's)
  auto qidx = [&](int m0, int u) {
    if constexpr (PAIR) {
      const int base = (m0 >> 5) * PAIR_CH, h = (m0 & 31) >> 1;
      return (u & 1) ? base + PAIR_ODD + (h + (u >> 1)) * 32 + lane : base + (h + (u >> 1)) * 34 + 1 + lane;
    } else {
      return (m0 + u) * 32 + lane;
    }
  };
  // Forward elimination of the raw rows  a_m x_{m-1} + b_m x_m + c_m x_{m+1} = d_m
  // through the continuants (leading principal minors)
  //     q_m = b_m q_{m-1} - a_m c_{m-1} q_{m-2},   q_{-1} = 1, q_{-2} = 0,
  // whose ratios are the Thomas pivots (b_m - a_m c'_{m-1} = q_m / q_{m-1}): the
  // serial chain is one fma per row, the reciprocals of the pivots are independent
  // of each other (ILP across the G rows of a group), and so is the d' recurrence
  // d'_m = d_m/piv_m - (a_m/piv_m) d'_{m-1} (one fma per row).  The continuants are
  // rescaled by a power of two after every group (exact; no overflow for any tau).
  // Row 0's lower weight meets c_{-1} = q_{-2} = d'_{-1} = 0 and needs no mask;
  // the group holding row n-1 (line end: c = 0, wall ghost) and the padding rows
  // past n (identity rows) takes the masked build (EDGE), like the first group of a
  // wall line.  A bottom-up warp (DIR) runs the same recurrences on the mirrored
  // rows (group offset u -> physical row m0 + G-1-u, lower and upper weights
  // swapped); its first rows are the padding / line-end rows.
  double qm1 = 1.0, qm2 = 0.0, cprev = 0.0, dp = 0.0;
  // the factor-row table of this tile's lines (Geo::tsplit rows i0.., j0..) into
  // shared memory (measured on B200: on a par with coef_split's 1-D factor loads
  // for the plain r-rows, 3-5 % faster for the rest)
  double* St = Sx + (RXR ? SA : 0);
  {
    // (all of a thread's loads in flight at once: <= 3 * 256 / 32 = 24 per lane; the
    // latency overlaps the first chunk's)
    const double* __restrict__ T3 = g.tsplit[Q][AX] + 3 * (i0 * NTk(g, K) + j0);
    const int tstride = (AX == 0) ? 3 * NTk(g, K) : 3;
    constexpr int NLD = 768 / NT;
    double tv[NLD];
#pragma unroll
    for (int t = 0; t < NLD; ++t) {
      const int e = min(tid + NT * t, 3 * n - 1);
      tv[t] = __ldg(T3 + (e / 3) * tstride + e % 3);
    }
#pragma unroll
    for (int t = 0; t < NLD; ++t)
      if (tid + NT * t < 3 * n) St[tid + NT * t] = tv[t];
  }
  // FINAL: the norm weights r^2 sin(theta) of the tile's rows
  double* Sw = St + 3 * n;
  if (FINAL) {
    for (int m = tid; m < n; m += NT) {
      const int i = (AX == 0) ? i0 + m : i0, j = (AX == 0) ? j0 : j0 + m;
      const double r = rnode<K>(g, i);
      Sw[m] = r * r * snode<K>(g, j);
    }
  }
  sync_block();
  // m0: the group's lowest physical row (a multiple of G)
  auto group = [&](int m0, auto edge, auto noadv, auto dir) {
    constexpr bool EDGE = decltype(edge)::value, NOADV = decltype(noadv)::value, DIR = decltype(dir)::value;
    double ra[G], rb[G], rc[G], rd[G];   // physical lower / diagonal / upper weights, rhs of the u-th row in solve order
#pragma unroll
    for (int u = 0; u < G; ++u) {
      const int up_ = DIR ? G - 1 - u : u;
      const int m = m0 + up_, mm = EDGE ? min(m, n - 1) : m;
      const int q = qidx(m0, up_);
      // the row's a*-independent part from Geo::tsplit (staged: a broadcast read),
      // the transport weight Astar::av and the u_theta reaction from the tile
      double lo = St[3 * mm], bm = St[3 * mm + 1], up = St[3 * mm + 2];
      if (!NOADV) {
        const double adv = Sc[q];
        lo = fma(-th, adv, lo);
        up = fma(th, adv, up);
        if (RXR) bm = fma(th, Sx[q], bm);
      }
      ra[u] = lo; rb[u] = bm; rc[u] = up; rd[u] = Sd[q];
    }
    if (EDGE) {
      // the line's first row: antisymmetric wall ghost of the increment (RD23);
      // its last row ul: wall ghost and c = 0 (homogeneous Dirichlet increment);
      // rows past it (padding): identity rows with d = 0
      if (AX == 0 && K != KR && m0 == 0 && g.wall_lo) rb[DIR ? G - 1 : 0] -= ra[DIR ? G - 1 : 0];
      const int ul = n - 1 - m0;
      const bool gh = AX == 0 && K != KR && g.wall_hi;
#pragma unroll
      for (int u = 0; u < G; ++u) {
        const int up_ = DIR ? G - 1 - u : u;
        if (up_ == ul) {
          if (gh) rb[u] -= rc[u];
          rc[u] = 0.0;
        }
        if (up_ > ul) { ra[u] = 0.0; rb[u] = 1.0; rc[u] = 0.0; rd[u] = 0.0; }
      }
    }
    // in solve order: L couples row u to the row solved before it, U to the next
    double (&L)[G] = DIR ? rc : ra;
    double (&U)[G] = DIR ? ra : rc;
    double qv[G];
    const double q0 = qm1;
#pragma unroll
    for (int u = 0; u < G; ++u) {
      const double e = L[u] * (u ? U[u - 1] : cprev);
      const double qn = fma(rb[u], qm1, -(e * qm2));
      qv[u] = qn;
      qm2 = qm1;
      qm1 = qn;
    }
#pragma unroll
    for (int u = 0; u < G; ++u) {
      const int q = qidx(m0, DIR ? G - 1 - u : u);
      const double inv = (u ? qv[u - 1] : q0) * frcp(qv[u]);
      dp = fma(-(L[u] * inv), dp, rd[u] * inv);
      if (valid) {
        Sc[q] = U[u] * inv;
        Sd[q] = dp;
      }
    }
    cprev = U[G - 1];
    // 2^-e of q_{m0+G-1} (exact rescaling of the two carried continuants)
    const long long eb = (__double_as_longlong(qm1) >> 52) & 0x7ff;
    const double sc = __longlong_as_double((2046LL - eb) << 52);
    qm1 *= sc;
    qm2 *= sc;
  };
  // (IMEX, noadv: a block-uniform branch outside the unrolled rows)
  auto forward = [&](auto noadv, auto dir) {
    constexpr bool DIR = decltype(dir)::value;
    const int HL = DIR ? NPAD - H0 : H0;
    for (int ml = 0; ml < HL; ml += G) {
      const int m0 = DIR ? NPAD - G - ml : ml;
      if (m0 % TH_RC == (DIR ? TH_RC - G : 0)) wait(m0 / TH_RC);
      const bool edge = m0 + G > n - 1 || (AX == 0 && K != KR && m0 == 0 && g.wall_lo);
      if (edge) group(m0, std::true_type{}, noadv, dir);
      else group(m0, std::false_type{}, noadv, dir);
    }
  };
  auto forward_dir = [&](auto dir) {
    if (a.noadv) forward(std::true_type{}, dir);
    else forward(std::false_type{}, dir);
  };
  // x: the unknown next to this warp's last eliminated row (the start of its back
  // substitution): 0 past the padded end, or from the 2x2 system at the meeting rows
  //   x_{H0-1} + c' x_{H0} = d'   (top-down),   a'' x_{H0-1} + x_{H0} = d''   (bottom-up)
  double x = 0.0;
  if constexpr (TWO) {
    if (wid) forward_dir(std::true_type{});
    else forward_dir(std::false_type{});
    __syncthreads();
    const int mo = wid ? H0 : H0 - 1, mt = wid ? H0 - 1 : H0;
    const int qo = qidx(mo & ~15, mo & 15), qt = qidx(mt & ~15, mt & 15);
    const double co = Sc[qo], dwn = Sd[qo], ct = Sc[qt], dt = Sd[qt];
    x = (dt - ct * dwn) / (1.0 - ct * co);
    __syncthreads();
  } else {
    forward_dir(std::false_type{});
  }
  // back substitution x_m = d'_m - c'_m x_{m+1} from the padded top (x = 0 there:
  // the padding rows are identity rows with d = 0) or outwards from the meeting
  // rows (TWO).  PLAIN: x over d', then one
  // bulk tensor store.  FINAL: psi + x straight to global (coalesced 256-B rows),
  // psi loaded one group ahead from L2 (the box was prefetched at the start).
  // (two-way: 8-row groups, like the elimination's — measured on B200: u_r r final
  // 3.62 -> 3.96 TB/s on C3, 4.60 -> 4.88 on C5; profiles/r02_late_switches_ab.txt)
#ifndef YY_TH_GB2
#define YY_TH_GB2 8
#endif
  constexpr int GB = TWO ? YY_TH_GB2 : 16;   // rows per back-substitution group
  if constexpr (!FINAL) {
    auto backward = [&](auto dir) {
      constexpr bool DIR = decltype(dir)::value;
      const int HL = DIR ? NPAD - H0 : H0;
      for (int ml = HL - GB; ml >= 0; ml -= GB) {
        const int m0 = DIR ? NPAD - GB - ml : ml;
        double cv[GB], dv[GB];
#pragma unroll
        for (int u = 0; u < GB; ++u) {
          const int q = qidx(m0, DIR ? GB - 1 - u : u);
          cv[u] = Sc[q];
          dv[u] = Sd[q];
        }
        // theta: x straight to global memory (coalesced 256-B rows, no bulk store to
        // wait for before the block exits); r: x over d', then one bulk tensor store
        // (measured on B200: each the faster for its axis)
        double* __restrict__ Rm = a.R + lofs + (long long)m0 * rs;
#pragma unroll
        for (int u = GB - 1; u >= 0; --u) {
          const int up_ = DIR ? GB - 1 - u : u;
          x = fma(-cv[u], x, dv[u]);
          if (AX == 1 || a.flat) {
            if (valid && m0 + up_ < n) Rm[up_ * rs] = x;
          } else if (valid) {
            Sd[(m0 + up_) * 32 + lane] = x;
          }
        }
      }
    };
    if (wid) backward(std::true_type{});
    else backward(std::false_type{});
    // (a flat box may run into the next theta row, which another block updates:
    // flat tiles store lane by lane)
    if (AX == 0 && !a.flat) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      sync_block();
      if (tid == 0) {
        tma_store_3d(&maps.m[3], Sd, c0, c1, c2);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      }
    }
  } else {
    double* __restrict__ P = a.psi + lofs;
    double wsum = 0.0;
    // psi of a row group is loaded two groups ahead of its use (ping-pong
    // registers, no copies; volatile: issued where written — plain loads were sunk
    // next to their uses), the norm weights r^2 sin(theta) come from Sw
    auto backward = [&](auto dir) {
      constexpr bool DIR = decltype(dir)::value;
      auto load_psi = [&](int m0, double (&dst)[GB]) {
        const double* Pm = P + m0 * rs;
#pragma unroll
        for (int u = 0; u < GB; ++u) {
          const int up_ = DIR ? GB - 1 - u : u;
          const double* pu = (m0 + up_ < n) ? Pm + up_ * rs : P;
          asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(dst[u]) : "l"(pu));
        }
      };
      auto back = [&](int m0, const double (&pv)[GB]) {
        double cv[GB], dv[GB];
#pragma unroll
        for (int u = 0; u < GB; ++u) {
          const int q = (m0 + (DIR ? GB - 1 - u : u)) * 32 + lane;
          cv[u] = Sc[q];
          dv[u] = Sd[q];
        }
        double* Pm = P + m0 * rs;
#pragma unroll
        for (int u = GB - 1; u >= 0; --u) {
          const int up_ = DIR ? GB - 1 - u : u;
          x = fma(-cv[u], x, dv[u]);
          if (valid && m0 + up_ < n) {
            Pm[up_ * rs] = pv[u] + x;
            wsum = fma(Sw[m0 + up_] * x, x, wsum);
          }
        }
      };
      // the warp's groups in back-substitution order: t = 0 .. ng - 1
      const int ng = (DIR ? NPAD - H0 : H0) / GB;
      auto base = [&](int t) { return DIR ? H0 + t * GB : H0 - GB - t * GB; };
      double pa[GB], pb[GB];
      load_psi(base(0), pa);
      for (int t = 0; t < ng; t += 2) {
        if (t + 1 < ng) load_psi(base(t + 1), pb);
        back(base(t), pa);
        if (t + 2 < ng) load_psi(base(t + 2), pa);
        if (t + 1 < ng) back(base(t + 1), pb);
      }
    };
    if (wid) backward(std::true_type{});
    else backward(std::false_type{});
    wsum *= g.dr * g.dth * g.dph;
    for (int o = 16; o > 0; o >>= 1) wsum += __shfl_down_sync(FULL, wsum, o);
    if constexpr (TWO) {
      __shared__ double sh2[2];
      if (lane == 0) sh2[wid] = wsum;
      __syncthreads();
      if (tid == 0) a.part[(long long)patch * a.maxb + B.y * gridDim.x + B.x] = sh2[0] + sh2[1];
    } else {
      if (lane == 0) a.part[(long long)patch * a.maxb + B.y * gridDim.x + B.x] = wsum;
    }
  }
}

// host: a 3-D tensor map over every patch of one kind-K array (dims phi, theta,
// patch-folded r), box = one tile (NL lines x n rows along AX)
inline bool encode_tile_map(CUtensorMap* map, const double* base, const Geo& g, int K, int npatch, int AX, int NL,
                            int n, bool flat = false, int pair = 0) {
  // resolved once (thread-safe static initialisation); no libcuda link dependency
  static const PFN_cuTensorMapEncodeTiled_v12000 enc = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess)
      fn = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }();
  if (!enc) return false;
  // flat (r boxes only): dims (theta x phi plane, 1, patch-folded r)
  const cuuint64_t plane = (cuuint64_t)NTk(g, K) * NPk(g, K);
  // pair (theta boxes of an odd phi pitch, NTk even): dims (2 NP, NT / 2, patch-folded
  // r), box (pair, n) with pair = 34 (odd-theta rows) or 32 (even-theta rows)
  const cuuint64_t dims[3] = {pair ? 2 * (cuuint64_t)NPk(g, K) : flat ? plane : (cuuint64_t)NPk(g, K),
                              pair ? (cuuint64_t)NTk(g, K) / 2 : flat ? 1 : (cuuint64_t)NTk(g, K),
                              (cuuint64_t)NRk(g, K) * npatch};
  const cuuint64_t strides[2] = {pair ? 2 * (cuuint64_t)NPk(g, K) * 8 : flat ? plane * 8 : (cuuint64_t)NPk(g, K) * 8,
                                 plane * 8};
  const cuuint32_t box[3] = {(cuuint32_t)(pair ? pair : NL), (cuuint32_t)(AX == 1 ? n : 1),
                             (cuuint32_t)(AX == 0 ? n : 1)};
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// env YY_TMA (default 1): theta plain and final sweeps of the TMA-eligible kinds on k_line_tma
inline bool use_tma() {
  static const bool v = [] {
    const char* e = getenv("YY_TMA");
    return !(e && e[0] == '0');
  }();
  return v;
}

// env YY_THOMAS (default 1): r / theta plain and final sweeps of the TMA-eligible
// kinds on k_line_th (one line per thread)
inline bool use_thomas() {
  static const bool v = [] {                         // thread-safe static initialisation
    const char* e = getenv("YY_THOMAS");
    return !(e && e[0] == '0');
  }();
  return v;
}

// env YY_PAIR (default 1): plain theta sweeps of an odd-phi-pitch kind (u_phi) on
// k_line_th with theta-pair boxes
inline bool use_pair() {
  static const bool v = [] {
    const char* e = getenv("YY_PAIR");
    return !(e && e[0] == '0');
  }();
  return v;
}

// env YY_TH_SMEM (KB, default 110): the largest k_line_th tile
inline int th_smem_max() {
  static const int v = [] {
    const char* e = getenv("YY_TH_SMEM");
    return e ? atoi(e) : 110;
  }();
  return v;
}

// env YY_TH2 (bit mask: 1 plain r, 2 plain theta, 4 final; default 7): k_line_th as
// two warps per tile eliminating from both ends of the lines.  Measured on B200
// (profiles/r02_th2_ab.txt, 16-row groups): plain theta sweeps +7-10 % (C3), +14-22 %
// (C5), the u_r r final factor +1-4 %, plain r sweeps -6 to -15 %; with 8-row groups
// (profiles/r02_late_switches_ab.txt) the plain r sweeps of C3's 96-row lines gain
// too (u_theta r 4.10 -> 4.61 TB/s, u_phi r 4.09 -> 4.34); lines of <= 64 rows (C5's
// r lines: two 32-row halves) keep one warp
inline int th_two_mask() {
  static const int v = [] {
    const char* e = getenv("YY_TH2");
    return e ? atoi(e) : 7;
  }();
  return v;
}

template <int Q, int AX, int MODE>
int launch_th(const Geo& g, const SweepArgs& a, int npatch, cudaStream_t st) {
  constexpr int K = kind_of(Q);
  constexpr bool FINAL = (MODE == MODE_FINAL);
  const int n_ = (AX == 0) ? i_hi<K>(g) - i_lo<K>(g) + 1 : NTk(g, K) - 2;
  const bool two = (th_two_mask() & (FINAL ? 4 : AX == 0 ? 1 : 2)) != 0 && !(!FINAL && AX == 0 && n_ <= 64);
  const int n = (AX == 0) ? i_hi<K>(g) - i_lo<K>(g) + 1 : NTk(g, K) - 2;
  const int nch = (n + TH_RC - 1) / TH_RC;
  // 16-B row pitch (tensor maps; measured: 8-B cp.async staging of the odd-pitch
  // kinds loses to k_line, 2.0 vs 3.1 TB/s)
  // an odd phi pitch: r boxes over the whole (theta, phi) plane (its size even),
  // plain theta sweeps on theta-pair boxes (NTk even)
  const bool odd = (NPk(g, K) % 2) != 0;
  constexpr bool PAIR_OK = AX == 1 && MODE == MODE_PLAIN && !(Q == QUT);
  const bool pair = odd && AX == 1;
  const bool flat = odd && AX == 0;
  if (pair && (!PAIR_OK || NTk(g, K) % 2 || !use_pair())) return -1;
  if ((flat && ((long long)NTk(g, K) * NPk(g, K)) % 2) || n > 256 || nch > 8) return -1;
  const size_t smem =
      ((size_t)nch * (pair ? PAIR_CH : TH_RC * 32) * (2 + ((Q == QUT && AX == 1) ? 1 : 0)) + 3 * n +
       (FINAL ? n : 0)) * sizeof(double);
  // measured on B200: two blocks per SM (C5 theta, 96 KB tiles) still beat the
  // partitioned k_line (3.1-3.3 vs 2.6-2.7 TB/s); one does not
  if (smem > (size_t)th_smem_max() * 1024) return -1;
  // m[0..2]: chunk boxes of the inputs; m[3]: the n-row box of the output (FINAL:
  // psi, prefetched into L2; PLAIN r: the right-hand side array, stored)
  TmaMaps maps{};
  if constexpr (PAIR_OK) {
    if (pair) {   // m[0], m[1]: odd-theta boxes of R, Astar::av; m[2], m[3]: even-theta boxes
      const bool okp = encode_tile_map(&maps.m[0], a.R, g, K, npatch, AX, 32, 16, false, 34) &&
                       encode_tile_map(&maps.m[1], g.adv[K][AX], g, K, npatch, AX, 32, 16, false, 34) &&
                       encode_tile_map(&maps.m[2], a.R, g, K, npatch, AX, 32, 16, false, 32) &&
                       encode_tile_map(&maps.m[3], g.adv[K][AX], g, K, npatch, AX, 32, 16, false, 32);
      if (!okp || smem > (size_t)th_smem_max() * 1024) return -1;
      const dim3 grid((NPk(g, K) + 31) / 32, i_hi<K>(g) - i_lo<K>(g) + 1, npatch);
      if (two) {
        opt_in_smem<k_line_th<Q, AX, MODE, true, true>>(smem);
        k_line_th<Q, AX, MODE, true, true><<<grid, 64, smem, st>>>(g, a, maps);
      } else {
        opt_in_smem<k_line_th<Q, AX, MODE, true>>(smem);
        k_line_th<Q, AX, MODE, true><<<grid, 32, smem, st>>>(g, a, maps);
      }
      return (int)(grid.x * grid.y);
    }
  }
  bool ok = encode_tile_map(&maps.m[0], a.R, g, K, npatch, AX, 32, TH_RC, flat) &&
            encode_tile_map(&maps.m[1], g.adv[K][AX], g, K, npatch, AX, 32, TH_RC, flat);
  if (ok && (FINAL || AX == 0))
    ok = encode_tile_map(&maps.m[3], FINAL ? a.psi : a.R, g, K, npatch, AX, 32, n, flat);
  if (ok && Q == QUT && AX == 1) ok = encode_tile_map(&maps.m[2], a.rt, g, K, npatch, AX, 32, TH_RC);
  if (!ok) return -1;
  SweepArgs af = a;
  af.flat = flat;
  const dim3 grid((NPk(g, K) + 31) / 32, AX == 0 ? NTk(g, K) - 2 : i_hi<K>(g) - i_lo<K>(g) + 1, npatch);
  if (two) {
    opt_in_smem<k_line_th<Q, AX, MODE, false, true>>(smem);
    k_line_th<Q, AX, MODE, false, true><<<grid, 64, smem, st>>>(g, af, maps);
  } else {
    opt_in_smem<k_line_th<Q, AX, MODE>>(smem);
    k_line_th<Q, AX, MODE><<<grid, 32, smem, st>>>(g, af, maps);
  }
  return (int)(grid.x * grid.y);
}

template <int Q, int AX, int MODE, int P, int M>
int launch_tma(const Geo& g, const SweepArgs& a, int npatch, cudaStream_t st) {
  constexpr int K = kind_of(Q);
  constexpr int NL = 128 / P;
  constexpr bool FINAL = (MODE == MODE_FINAL);
  constexpr int SA = (P * M * NL + 15) / 16 * 16;
  const int n = (AX == 0) ? i_hi<K>(g) - i_lo<K>(g) + 1 : NTk(g, K) - 2;
  if ((NPk(g, K) % 2) || n > 256) return -1;          // row pitch a multiple of 16 B; box rows <= 256
  TmaMaps maps{};
  const long long off = 0;
  bool ok = encode_tile_map(&maps.m[0], a.R + off, g, K, npatch, AX, NL, n) &&
            encode_tile_map(&maps.m[1], g.adv[K][AX], g, K, npatch, AX, NL, n);
  if (ok && Q == QUT && AX == 1) ok = encode_tile_map(&maps.m[2], a.rt, g, K, npatch, AX, NL, n);
  if (ok && FINAL) ok = encode_tile_map(&maps.m[3], a.psi, g, K, npatch, AX, NL, n);
  if (!ok) return -1;
  constexpr int NIN = tma_narr<Q, AX, FINAL>() - 1;
  constexpr int TILE = 3 * NL * line_pitch<P, (M | 1)>();
  constexpr int FRONT = (NIN * SA > TILE ? NIN * SA : TILE + 15) / 16 * 16;
  const size_t smem = ((size_t)FRONT + SA + 4 * P * M) * sizeof(double);   // + row table, norm weights
  opt_in_smem<k_line_tma<Q, AX, MODE, P, M>>(smem);
  const dim3 grid((NPk(g, K) - 1 + NL - 1) / NL, AX == 0 ? NTk(g, K) - 2 : i_hi<K>(g) - i_lo<K>(g) + 1, npatch);
  k_line_tma<Q, AX, MODE, P, M><<<grid, 128, smem, st>>>(g, a, maps);
  return (int)(grid.x * grid.y);
}

// ---------------------------------------------------------------------------------
// launch: pick (P, M) with P*M >= n
// ---------------------------------------------------------------------------------
#ifndef TMA_MMAX
#define TMA_MMAX 16
#endif
template <int Q, int AX, int MODE, int S, int P, int M>
int launch_line(const Geo& g, const SweepArgs& a, const ResidArgs& ra, int npatch, cudaStream_t st) {
  // theta sweeps only: measured on B200 (C3) the theta classes gain 3-9 %, the r
  // sweeps lose up to 12 % (their box rows lie 393 KB apart)
  if constexpr (th_route(Q, AX, MODE) && P <= 32) {
    if (use_thomas() && (!(Q == QUT && AX == 1 && MODE == MODE_FINAL) || use_th_utf())) {
      const int nb = launch_th<Q, AX, MODE>(g, a, npatch, st);
      if (nb >= 0) return nb;
    }
  }
  if constexpr (AX == 1 && (MODE == MODE_PLAIN || MODE == MODE_FINAL) && P <= 32 && M <= TMA_MMAX) {
    if (use_tma()) {
      const int nb = launch_tma<Q, AX, MODE, P, M>(g, a, npatch, st);
      if (nb >= 0) return nb;
    }
  }
  constexpr int K = kind_of(Q);
  constexpr int NL = 128 / P;
  // a slab line continued by the slab above must fill its chunks exactly (part_solve3)
  if (MODE == MODE_SLAB && !g.wall_hi && P * M != i_hi<K>(g) - i_lo<K>(g) + 1) return -2;
  const size_t smem = (size_t)3 * NL * line_pitch<P, (M | 1)>() * sizeof(double);
  opt_in_smem<k_line<Q, AX, MODE, S, P, M>>(smem);
  dim3 grid;
  if (AX == 2) {
    const int nlines = (i_hi<K>(g) - i_lo<K>(g) + 1) * (NTk(g, K) - 2);
    grid = dim3((nlines + NL - 1) / NL, npatch);
  } else {
    grid = dim3((NPk(g, K) - 2 + NL - 1) / NL, AX == 0 ? NTk(g, K) - 2 : i_hi<K>(g) - i_lo<K>(g) + 1, npatch);
  }
  k_line<Q, AX, MODE, S, P, M><<<grid, 128, smem, st>>>(g, a, ra);
  return (int)(grid.x * grid.y);
}

template <int Q, int AX, int MODE, int S>
int sweep_line(const Geo& g, const SweepArgs& a, const ResidArgs& ra, int npatch, cudaStream_t st) {
  constexpr int K = kind_of(Q);
#define YY_L(P_, M_) return launch_line<Q, AX, MODE, S, P_, M_>(g, a, ra, npatch, st)
  if constexpr (AX == 2) {
    const int n = NPk(g, K) - 2;
    if (n <= 128) YY_L(32, 4);
    if (n <= 256) YY_L(32, 8);
#if YY_PH384 == 1
    if (n <= 384) YY_L(64, 6);
#elif YY_PH384 == 2
    if (n <= 384) YY_L(128, 3);
#endif
    if (n <= 384) YY_L(32, 12);
    if (n <= 512) YY_L(128, 4);                    // longer lines: 4 warps per line
    if (n <= 576) YY_L(64, 9);                     // two warps per line (measured on B200, C5: +23-32 % over (128, 5))
    if (n <= 640) YY_L(128, 5);
    if (n <= 768) YY_L(128, 6);
    YY_L(128, 9);                                  // n <= 1152 (checked at create)
  } else {
    const int n = (AX == 0) ? i_hi<K>(g) - i_lo<K>(g) + 1 : NTk(g, K) - 2;
    if (n <= 16) YY_L(4, 4);
    if (n <= 32) YY_L(4, 8);
    if (n <= 64) YY_L(8, 8);
#if YY_RT_MENU == 0
    // theta: 8 lines of (8, 12) / (8, 16) chunks (measured on B200, C3: u_theta
    // theta final +5 %, u_phi theta +3 %; the r sweeps lose 13 % with them)
    if (AX == 1 && n <= 96) YY_L(8, 12);
    if (AX == 1 && n <= 128) YY_L(8, 16);
#elif YY_RT_MENU == 1
    if (n <= 96) YY_L(8, 12);
    if (n <= 128) YY_L(8, 16);
#elif YY_RT_MENU == 2
    if (n <= 96) YY_L(32, 3);
    if (n <= 128) YY_L(32, 4);
#endif
    if (n <= 96) YY_L(16, 6);
    if (n <= 128) YY_L(16, 8);
    if constexpr (AX == 1) {
      if (n <= 192) YY_L(16, 12);                  // measured on B200 (C5 theta): +25-40 % over (16, 16)
    }
    if (n <= 256) YY_L(16, 16);
    if (n <= 384) YY_L(16, 24);
    YY_L(32, 16);                                  // n <= 512 (checked at create)
  }
#undef YY_L
}

// radial-slab r-lines continued by the slab above must fill their chunks exactly
// (part_solve3): pick P x M = n from this menu
template <int Q>
int sweep_slab(const Geo& g, const SweepArgs& a, int npatch, cudaStream_t st) {
  constexpr int K = kind_of(Q);
  const ResidArgs none{};
  const int n = i_hi<K>(g) - i_lo<K>(g) + 1;
#define YY_S(P_, M_) if (n <= (P_) * (M_) && (g.wall_hi || n == (P_) * (M_))) \
    return launch_line<Q, 0, MODE_SLAB, 1, P_, M_>(g, a, none, npatch, st);
  YY_S(4, 4) YY_S(4, 6) YY_S(4, 8) YY_S(8, 6) YY_S(8, 8) YY_S(16, 6) YY_S(16, 8) YY_S(16, 12) YY_S(32, 8)
  YY_S(32, 12) YY_S(32, 16)
#undef YY_S
  return -2;
}

// factor orders (RD28): T r,th,ph; u_r th,ph,r; u_th ph,r,th; u_ph r,th,ph
constexpr int FIRST_AX[4] = {0, 1, 2, 0};
constexpr int LAST_AX[4] = {2, 0, 1, 2};

template <int Q, int AX>
int sweep_axis(const Geo& g, int s, bool first, bool fin, bool slab, const SweepArgs& a, const ResidArgs* ra,
               int npatch, cudaStream_t st) {
  const ResidArgs none{};
  if constexpr (AX == 0) {
    if (slab) return first ? -1 : sweep_slab<Q>(g, a, npatch, st);
  }
  if constexpr (AX == LAST_AX[Q]) {
    if (fin) return sweep_line<Q, AX, MODE_FINAL, 1>(g, a, none, npatch, st);
  }
  if constexpr (AX == FIRST_AX[Q]) {
    if (first && ra) {
      if (Q == QT || s == 1) return sweep_line<Q, AX, MODE_FIRST, 1>(g, a, *ra, npatch, st);
      if constexpr (Q != QT) return sweep_line<Q, AX, MODE_FIRST, 2>(g, a, *ra, npatch, st);
    }
  }
  if (fin || first) return -1;                     // not a factor position of this quantity
  return sweep_line<Q, AX, MODE_PLAIN, 1>(g, a, none, npatch, st);
}

}  // namespace


template <int Q>
int launch_sweep_q(const Geo& g, int ax, int s, bool first, bool fin, bool slab, const SweepArgs& a,
                   const ResidArgs* ra, int npatch, cudaStream_t st) {
  if (ax == 0) return sweep_axis<Q, 0>(g, s, first, fin, slab, a, ra, npatch, st);
  if (ax == 1) return sweep_axis<Q, 1>(g, s, first, fin, slab, a, ra, npatch, st);
  return sweep_axis<Q, 2>(g, s, first, fin, slab, a, ra, npatch, st);
}

// one translation unit per quantity (csrc/build.sh compiles this file with
// -DYY_LINE_Q=0..3 in parallel)
#ifdef YY_LINE_Q
template int launch_sweep_q<YY_LINE_Q>(const Geo&, int, int, bool, bool, bool, const SweepArgs&, const ResidArgs*,
                                       int, cudaStream_t);
#endif

}  // namespace yy
