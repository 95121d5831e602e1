// tb_ab.cu — scratch A/B microbenchmark (not product code): the fused two-step kernels of one
// source version (-I <csrc>) on C2-like (D3Q19 raw zc+delta 256^3, fp64 / fp32) and C5-like
// (D2Q9 CM 8192^2) lattices, time per two steps.
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

template <class K>
float time_k(K launch, int reps = 20) {
  launch(0);
  launch(1);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < reps; ++i) launch(i & 1);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  CK(cudaGetLastError());
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms / reps;
}

template <class real, int MINB>
void d3q19(const char *name) {
  GridParams g{};
  g.nx = g.ny = g.nzl = g.nzg = 256;
  g.pitch = 256;
  g.pop = 256 * 256;
  g.plane = 19LL * g.pop;
  g.wrapz = 1;
  size_t elems = (size_t)(256 + 2) * g.plane;
  real *a, *b;
  CK(cudaMalloc(&a, elems * sizeof(real)));
  CK(cudaMalloc(&b, elems * sizeof(real)));
  fill<<<1184, 256>>>(a, elems, real(0));
  fill<<<1184, 256>>>(b, elems, real(0));
  Rates<real> r;
  for (int i = 0; i < 27; ++i) r.w[i] = real(1.0 + 0.02 * i);
  Force<real> fr{};
  using T = Tile2<16, 8>;
  const size_t smem = (size_t)3 * 19 * T::HW * sizeof(real);
  auto kern = k_pull2<D3Q19, SPACE_RAW, REG_DELTA, real, RS_GENERAL, 16, 8, MINB, true>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  float ms = time_k([&](int p) {
    kern<<<dim3(16, 32, 3), T::THREADS, smem>>>(p ? b : a, p ? a : b, g, r, real(0), fr);
  });
  printf("%-34s %7.3f ms / 2 steps  %8.0f MLUPS\n", name, ms, 2.0 * 256 * 256 * 256 / (ms * 1e-3) / 1e6);
  cudaFree(a);
  cudaFree(b);
}

void d2q9() {
  GridParams g{};
  g.nx = 8192;
  g.ny = 1;
  g.nzl = g.nzg = 8192;
  g.pitch = 8192;
  g.pop = 8192;
  g.plane = 9LL * g.pop;
  g.wrapz = 1;
  size_t elems = (size_t)(8192 + 2) * g.plane;
  double *a, *b;
  CK(cudaMalloc(&a, elems * 8));
  CK(cudaMalloc(&b, elems * 8));
  fill<<<1184, 256>>>(a, elems, 0.1);
  fill<<<1184, 256>>>(b, elems, 0.1);
  Rates<double> r;
  for (int i = 0; i < 27; ++i) r.w[i] = 1.0;
  r.w[3] = r.w[4] = 0.695652;
  Force<double> fr{};
  using T = Tile1<256>;
  const size_t smem = (size_t)3 * 9 * T::HW * 8;
  auto kern = k_pull2_2d<D2Q9, SPACE_SWE, REG_ABS, double, RS_GENERAL, 256, 2, true>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  float ms = time_k([&](int p) {
    kern<<<dim3(32, 37, 1), T::THREADS, smem>>>(p ? b : a, p ? a : b, g, r, 0.0613125, fr);
  });
  printf("%-34s %7.3f ms / 2 steps  %8.0f MLUPS\n", "D2Q9 SWE 8192^2 fp64", ms, 2.0 * 8192 * 8192 / (ms * 1e-3) / 1e6);
  cudaFree(a);
  cudaFree(b);
}

int main() {
  d3q19<double, 2>("D3Q19 raw 256^3 fp64 (16x8, 2/SM)");
  d3q19<float, 3>("D3Q19 raw 256^3 fp32 (16x8, 3/SM)");
  d2q9();
  return 0;
}
