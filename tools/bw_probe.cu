// bw_probe.cu — what the r-sweep's memory access pattern alone can reach on
// B200: read two fp64 arrays (right-hand side + row weight) and write one, with
// the tile shapes of the line solver (NL consecutive k-lines x n rows of stride
// nt*np, one block per (k tile, j, patch)), no arithmetic.  Compared with a
// contiguous 3-stream kernel on the same bytes.  C3 shapes: 2 x 96 x 128 x 384.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/bw_probe tools/bw_probe.cu && /tmp/bw_probe
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s\n", cudaGetErrorString(e)); return 1; } } while (0)

__global__ void k_stream(const double* __restrict__ a, const double* __restrict__ b, double* __restrict__ c, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    c[i] = a[i] + b[i];
}

// tile: NL lines (k) x NR rows (r), rows `stride` apart; 128 threads; each thread
// handles (line = t % NL, rows t / NL + r * (128 / NL))
template <int NL>
__global__ void __launch_bounds__(128) k_rtile(const double* __restrict__ a, const double* __restrict__ b,
                                               double* __restrict__ c, int nr, int nt, int np) {
  const int k = blockIdx.x * NL + threadIdx.x % NL;
  const int j = blockIdx.y;
  const long long po = (long long)blockIdx.z * nr * nt * np;
  const long long stride = (long long)nt * np;
  constexpr int RS = 128 / NL;
  double v[16];
  int cnt = 0;
#pragma unroll 4
  for (int r = threadIdx.x / NL; r < nr; r += RS) {
    const long long q = po + r * stride + (long long)j * np + k;
    c[q] = __ldg(a + q) + __ldg(b + q);
    ++cnt;
  }
  (void)v;
  (void)cnt;
}

// all loads of the tile first (in registers), then the stores: the line solver's order
template <int NL, int PER>
__global__ void __launch_bounds__(128) k_rtile_batch(const double* __restrict__ a, const double* __restrict__ b,
                                                     double* __restrict__ c, int nr, int nt, int np) {
  const int k = blockIdx.x * NL + threadIdx.x % NL;
  const int j = blockIdx.y;
  const long long po = (long long)blockIdx.z * nr * nt * np;
  const long long stride = (long long)nt * np;
  constexpr int RS = 128 / NL;
  const int r0 = (threadIdx.x / NL) * PER;    // PER consecutive rows per thread (the chunk)
  double x[PER], y[PER];
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int r = min(r0 + u, nr - 1);
    const long long q = po + r * stride + (long long)j * np + k;
    x[u] = __ldg(a + q);
    y[u] = __ldg(b + q);
  }
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int r = r0 + u;
    if (r < nr) c[po + r * stride + (long long)j * np + k] = x[u] + y[u];
  }
  (void)RS;
}

int main() {
  const int nr = 96, nt = 128, np = 384, npatch = 2;
  const long long n = (long long)npatch * nr * nt * np;
  double *a, *b, *c, *flush;
  CK(cudaMalloc(&a, n * 8));
  CK(cudaMalloc(&b, n * 8));
  CK(cudaMalloc(&c, n * 8));
  CK(cudaMalloc(&flush, 256LL << 20));
  CK(cudaMemset(a, 0, n * 8));
  CK(cudaMemset(b, 0, n * 8));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double bytes = 3.0 * n * 8;
  auto timeit = [&](const char* name, auto launch) {
    float best = 1e9;
    for (int rep = 0; rep < 20; ++rep) {
      cudaMemsetAsync(flush, rep, 256LL << 20);
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep >= 3 && ms < best) best = ms;
    }
    printf("%-44s %8.1f us  %7.0f GB/s\n", name, best * 1e3, bytes / (best * 1e-3) / 1e9);
  };
  timeit("contiguous a+b->c (148*8 blocks x 256)", [&] { k_stream<<<148 * 8, 256>>>(a, b, c, n); });
  timeit("r-tile NL=8 (64 B rows), row loop", [&] { k_rtile<8><<<dim3(np / 8, nt, npatch), 128>>>(a, b, c, nr, nt, np); });
  timeit("r-tile NL=16 (128 B rows), row loop", [&] { k_rtile<16><<<dim3(np / 16, nt, npatch), 128>>>(a, b, c, nr, nt, np); });
  timeit("r-tile NL=32 (256 B rows), row loop", [&] { k_rtile<32><<<dim3(np / 32, nt, npatch), 128>>>(a, b, c, nr, nt, np); });
  timeit("r-tile NL=8, 6-row chunks batched (16,6)", [&] { k_rtile_batch<8, 6><<<dim3(np / 8, nt, npatch), 128>>>(a, b, c, nr, nt, np); });
  timeit("r-tile NL=16, 12-row chunks batched (8,12)", [&] { k_rtile_batch<16, 12><<<dim3(np / 16, nt, npatch), 128>>>(a, b, c, nr, nt, np); });
  timeit("r-tile NL=32, 24-row chunks batched (4,24)", [&] { k_rtile_batch<32, 24><<<dim3(np / 32, nt, npatch), 128>>>(a, b, c, nr, nt, np); });
  return 0;
}
