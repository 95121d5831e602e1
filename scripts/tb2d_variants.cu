// tb2d_variants.cu — scratch microbenchmark (not product code): variants of the 2D
// temporal-blocking kernel k_pull2_2d (strip width, CTAs/SM register cap, load prefetch)
// against two single-step k_pull launches, D2Q9 fp64, 8192 x 8192.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//          -I paper_2211_02435_b200/csrc scripts/tb2d_variants.cu -o scripts/tb2d_variants
#include <cstdio>
#include <cstdlib>

#include "kernels.cuh"

using namespace lbm;

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e = (x);                                                             \
    if (e != cudaSuccess) {                                                          \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                       \
    }                                                                                \
  } while (0)

template <class real>
__global__ void fill(real *a, size_t n, real v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) a[i] = v;
}

template <int SP, int REG, int TX, int MINB, bool PF>
float time_tb(const GridParams &g, double *a, double *b, const Rates<double> &r, double swe_g, int chunks) {
  using T = Tile1<TX>;
  const size_t smem = (size_t)3 * 9 * T::HW * sizeof(double);
  auto kern = k_pull2_2d<D2Q9, SP, REG, double, RS_GENERAL, TX, MINB, PF>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid(g.nx / TX, chunks, 1);
  Force<double> fr{};
  for (int i = 0; i < 2; ++i) kern<<<grid, T::THREADS, smem>>>(a, b, g, r, swe_g, fr);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  const int reps = 10;
  for (int i = 0; i < reps; ++i) {
    if (i % 2 == 0) kern<<<grid, T::THREADS, smem>>>(a, b, g, r, swe_g, fr);
    else kern<<<grid, T::THREADS, smem>>>(b, a, g, r, swe_g, fr);
  }
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  CK(cudaGetLastError());
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, T::THREADS, smem);
  cudaFuncAttributes at{};
  cudaFuncGetAttributes(&at, kern);
  const double cells = (double)g.nx * g.nzl;
  printf("  TB TX %3d minB %d pf %d chunks %3d threads %3d smem %6zu blocks/SM %d regs %3d local %3zu -> %7.3f ms / 2 steps  %8.0f MLUPS\n",
         TX, MINB, (int)PF, chunks, T::THREADS, smem, nb, at.numRegs, at.localSizeBytes, ms / reps,
         2 * cells / (ms / reps * 1e-3) / 1e6);
  return ms / reps;
}

template <int SP, int REG>
float time_single(const GridParams &g, double *a, double *b, const Rates<double> &r, double swe_g) {
  dim3 grid((g.nx + 127) / 128, 1, g.nzl);
  Force<double> fr{};
  for (int i = 0; i < 2; ++i) k_pull<D2Q9, SP, REG, double, false><<<grid, 128>>>(a, b, g, r, swe_g, fr);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  const int reps = 10;
  for (int i = 0; i < reps; ++i) {
    if (i % 2 == 0) k_pull<D2Q9, SP, REG, double, false><<<grid, 128>>>(a, b, g, r, swe_g, fr);
    else k_pull<D2Q9, SP, REG, double, false><<<grid, 128>>>(b, a, g, r, swe_g, fr);
  }
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double cells = (double)g.nx * g.nzl;
  printf("  single-step k_pull x2                                                      -> %7.3f ms / 2 steps  %8.0f MLUPS\n",
         2 * ms / reps, 2 * cells / (2 * ms / reps * 1e-3) / 1e6);
  return 2 * ms / reps;
}

template <int SP, int REG>
void sweep(const char *name, const GridParams &g, double *a, double *b, const Rates<double> &r, double swe_g) {
  printf("%s\n", name);
  time_single<SP, REG>(g, a, b, r, swe_g);
  time_tb<SP, REG, 256, 1, true>(g, a, b, r, swe_g, 37);
  time_tb<SP, REG, 256, 2, true>(g, a, b, r, swe_g, 37);
  time_tb<SP, REG, 256, 3, true>(g, a, b, r, swe_g, 37);
  time_tb<SP, REG, 256, 3, true>(g, a, b, r, swe_g, 74);
  time_tb<SP, REG, 256, 3, false>(g, a, b, r, swe_g, 37);
  time_tb<SP, REG, 128, 4, true>(g, a, b, r, swe_g, 19);
  time_tb<SP, REG, 128, 6, true>(g, a, b, r, swe_g, 19);
  time_tb<SP, REG, 512, 1, true>(g, a, b, r, swe_g, 74);
}

int main() {
  const int nx = 8192, ny = 8192;
  GridParams g{};
  g.nx = nx;
  g.ny = 1;
  g.nzl = ny;
  g.nzg = ny;
  g.pitch = nx;
  g.pop = g.pitch;
  g.plane = 9LL * g.pop;
  g.wrapz = 1;
  Rates<double> r;
  for (int i = 0; i < 27; ++i) r.w[i] = 1.0 + 0.02 * i;
  const size_t elems = (size_t)(ny + 2) * g.plane;
  double *a, *b;
  CK(cudaMalloc(&a, elems * 8));
  CK(cudaMalloc(&b, elems * 8));
  fill<<<1184, 256>>>(a, elems, 0.1);
  fill<<<1184, 256>>>(b, elems, 0.1);
  CK(cudaDeviceSynchronize());
  sweep<SPACE_SWE, REG_ABS>("D2Q9 SWE CM abs fp64 8192^2 (C5)", g, a, b, r, 0.0613125);
  sweep<SPACE_CUMULANT, REG_ZC_ABS>("D2Q9 cumulant zc+eq fp64 8192^2", g, a, b, r, 0.0);
  fill<<<1184, 256>>>(a, elems, 0.0);
  fill<<<1184, 256>>>(b, elems, 0.0);
  sweep<SPACE_POPULATION, REG_DELTA>("D2Q9 SRT zc+delta fp64 8192^2", g, a, b, r, 0.0);
  return 0;
}
