// tb_variants.cu — scratch microbenchmark (not product code): tile shapes of the
// temporal-blocking kernel k_pull2 (two fused steps) against two single-step k_pull
// launches, D3Q27 cumulant fp64 (and D3Q19 raw fp64), 1024 x 1024 x 128.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//          -I paper_2211_02435_b200/csrc scripts/tb_variants.cu -o scripts/tb_variants
#include <cstdio>
#include <cstdlib>

#include "kernels.cuh"

using namespace lbm;

#define CK(x)                                                                                   \
  do {                                                                                          \
    cudaError_t e = (x);                                                                        \
    if (e != cudaSuccess) {                                                                     \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);            \
      exit(1);                                                                                  \
    }                                                                                           \
  } while (0)

template <class S, int SP, int REG, int TX, int TY, class real = double, int MINB = 1, bool PF = false>
float time_tb(const GridParams &g, real *a, real *b, const Rates<real> &r, const Force<real> &fr) {
  using T = Tile2<TX, TY>;
  const size_t smem = (size_t)3 * S::Q * T::HW * sizeof(real);
  auto kern = k_pull2<S, SP, REG, real, RS_GENERAL, TX, TY, MINB, PF>;
  if (smem > 232448) return -1.f;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid(g.nx / TX, g.ny / TY, 1);
  for (int i = 0; i < 2; ++i) kern<<<grid, T::THREADS, smem>>>(a, b, g, r, 0.0, fr);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  const int reps = 6;
  for (int i = 0; i < reps; ++i) {
    if (i % 2 == 0) kern<<<grid, T::THREADS, smem>>>(a, b, g, r, 0.0, fr);
    else kern<<<grid, T::THREADS, smem>>>(b, a, g, r, 0.0, fr);
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
  printf("  TB %2dx%-2d minB %d pf %d threads %4d smem %6zu B  blocks/SM %d regs %3d local %3zu -> %7.3f ms per 2 steps\n",
         TX, TY, MINB, (int)PF, T::THREADS, smem, nb, at.numRegs, at.localSizeBytes, ms / reps);
  return ms / reps;
}

template <class S, int SP, int REG, class real = double>
float time_single(const GridParams &g, real *a, real *b, const Rates<real> &r, const Force<real> &fr) {
  dim3 grid((g.nx + 127) / 128, g.ny, g.nzl);
  for (int i = 0; i < 2; ++i) k_pull<S, SP, REG, real, false><<<grid, 128>>>(a, b, g, r, 0.0, fr);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  const int reps = 10;
  for (int i = 0; i < reps; ++i) {
    if (i % 2 == 0) k_pull<S, SP, REG, real, false><<<grid, 128>>>(a, b, g, r, 0.0, fr);
    else k_pull<S, SP, REG, real, false><<<grid, 128>>>(b, a, g, r, 0.0, fr);
  }
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("  single-step k_pull x2                                        -> %7.3f ms per 2 steps\n",
         2 * ms / reps);
  return 2 * ms / reps;
}

int main() {
  const int nx = 1024, ny = 1024, nz = 128;
  GridParams g{};
  g.nx = nx;
  g.ny = ny;
  g.nzl = nz;
  g.nzg = nz;
  g.pitch = nx;
  g.pop = (long long)ny * g.pitch;
  g.wrapz = 1;
  Rates<double> r;
  for (int i = 0; i < 27; ++i) r.w[i] = 1.0 + 0.02 * i;
  Force<double> fr{};
  {
    g.plane = 27LL * g.pop;
    size_t elems = (size_t)(nz + 2) * g.plane;
    double *a, *b;
    CK(cudaMalloc(&a, elems * 8));
    CK(cudaMalloc(&b, elems * 8));
    CK(cudaMemset(a, 0, elems * 8));
    CK(cudaMemset(b, 0, elems * 8));
    printf("D3Q27 cumulant zc+eq fp64\n");
    time_single<D3Q27, SPACE_CUMULANT, REG_ZC_ABS>(g, a, b, r, fr);
    time_tb<D3Q27, SPACE_CUMULANT, REG_ZC_ABS, 16, 8, double, 1, true>(g, a, b, r, fr);
    time_tb<D3Q27, SPACE_CUMULANT, REG_ZC_ABS, 16, 6, double, 2, true>(g, a, b, r, fr);
    time_tb<D3Q27, SPACE_CUMULANT, REG_ZC_ABS, 12, 8, double, 2, true>(g, a, b, r, fr);
    time_tb<D3Q27, SPACE_CUMULANT, REG_ZC_ABS, 16, 6, double, 2, false>(g, a, b, r, fr);
    time_tb<D3Q27, SPACE_CUMULANT, REG_ZC_ABS, 32, 2, double, 2, true>(g, a, b, r, fr);
    time_tb<D3Q27, SPACE_CUMULANT, REG_ZC_ABS, 8, 8, double, 2, true>(g, a, b, r, fr);
    printf("D3Q27 central zc+eq fp64\n");
    time_single<D3Q27, SPACE_CENTRAL, REG_ZC_ABS>(g, a, b, r, fr);
    time_tb<D3Q27, SPACE_CENTRAL, REG_ZC_ABS, 16, 8, double, 1, true>(g, a, b, r, fr);
    time_tb<D3Q27, SPACE_CENTRAL, REG_ZC_ABS, 16, 6, double, 2, true>(g, a, b, r, fr);
    time_tb<D3Q27, SPACE_CENTRAL, REG_ZC_ABS, 12, 8, double, 2, true>(g, a, b, r, fr);
    printf("D3Q27 raw zc+delta fp64\n");
    time_single<D3Q27, SPACE_RAW, REG_DELTA>(g, a, b, r, fr);
    time_tb<D3Q27, SPACE_RAW, REG_DELTA, 16, 8, double, 1, true>(g, a, b, r, fr);
    time_tb<D3Q27, SPACE_RAW, REG_DELTA, 16, 6, double, 2, true>(g, a, b, r, fr);
    cudaFree(a);
    cudaFree(b);
  }
  return 0;
}
