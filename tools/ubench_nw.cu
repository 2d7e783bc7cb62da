// Microbenchmark: FP64 add latency, 64-bit shuffle latency and the lean NW
// band sweep's cycles per anti-diagonal step on one warp.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false tools/ubench_nw.cu -o /tmp/ubench_nw
#include <cstdio>
#include <vector>

#include "../paper_1512_01641_b200/csrc/nw_kernel.cuh"

using namespace bimine;

__global__ void dadd_chain(double *out, long long *cyc, int n) {
  double x = out[0], y = out[1];
  const long long t0 = clock64();
  for (int k = 0; k < n; ++k) x = bimine::fadd(x, y);
  const long long t1 = clock64();
  out[2] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void shfl_chain(double *out, long long *cyc, int n) {
  double x = out[threadIdx.x];
  const long long t0 = clock64();
  for (int k = 0; k < n; ++k) x = __shfl_up_sync(kFull, x, 1) + 0.0;
  const long long t1 = clock64();
  out[32 + threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[1] = t1 - t0;
}

__global__ void sweep(const double *sim, int N, int M, uint16_t *dirs, long long *cyc, double *res) {
  TopAnalytic top{-1.5};
  BotNone bot;
  const long long t0 = clock64();
  double fin = band_sweep<true>(sim, M, N, M, 0, 1.5, -1.0, 1.0 - (-1.0), top, bot, dirs);
  const long long t1 = clock64();
  res[threadIdx.x] = fin;
  if (threadIdx.x == 0) cyc[2] = t1 - t0;
}

int main() {
  const int N = 32, M = 4096;
  double *d, *sim, *res;
  long long *cyc;
  uint16_t *dirs;
  cudaMalloc(&d, 1024 * 8);
  cudaMalloc(&sim, (size_t)N * M * 8);
  cudaMalloc(&res, 64 * 8);
  cudaMalloc(&cyc, 8 * 8);
  cudaMalloc(&dirs, (size_t)nw_groups(M) * 32 * 2);
  std::vector<double> h(N * M);
  for (size_t k = 0; k < h.size(); ++k) h[k] = (k * 2654435761u % 1000) / 1000.0;
  cudaMemcpy(sim, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  std::vector<double> one(64, 1.0);
  cudaMemcpy(d, one.data(), 64 * 8, cudaMemcpyHostToDevice);
  long long c[3];
  for (int rep = 0; rep < 2; ++rep) {
    dadd_chain<<<1, 32>>>(d, cyc, 4096);
    shfl_chain<<<1, 32>>>(d, cyc, 4096);
    sweep<<<1, 32>>>(sim, N, M, dirs, cyc, res);
    cudaDeviceSynchronize();
  }
  cudaMemcpy(c, cyc, 3 * 8, cudaMemcpyDeviceToHost);
  printf("dadd latency  %.1f cycles\n", c[0] / 4096.0);
  printf("shfl64+dadd   %.1f cycles\n", c[1] / 4096.0);
  printf("sweep         %.1f cycles/step (%d steps)\n", c[2] / double(M + 31), M + 31);
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
