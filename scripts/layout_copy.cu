// layout_copy.cu — scratch microbenchmark (not product code): the speed of light of the
// D3Q27 pull access pattern (27 shifted loads + 27 stores per cell, fp64, periodic) under
// two memory layouts:
//   SoA   [z][i][y][x]            (production)
//   AoSoA [z][y][xb][i][32]       (32-cell blocks; a warp's 27 loads hit one 6.9 KB chunk)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/layout_copy.cu -o scripts/layout_copy
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                                   \
  do {                                                                                          \
    cudaError_t e = (x);                                                                        \
    if (e != cudaSuccess) {                                                                     \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);            \
      exit(1);                                                                                  \
    }                                                                                           \
  } while (0)

__host__ __device__ constexpr int vx(int i) {
  constexpr int t[27] = {0, 1, -1, 0, 0, 1, -1, 1, -1, 0, 1, -1, 0, 0, 1, -1, 1, -1,
                         0, -1, 1, 0, 0, -1, 1, -1, 1};
  return t[i];
}
__host__ __device__ constexpr int vy(int i) {
  constexpr int t[27] = {0, 0, 0, 1, -1, 1, -1, -1, 1, 0, 0, 0, 1, -1, 1, -1, -1, 1,
                         0, 0, 0, -1, 1, -1, 1, 1, -1};
  return t[i];
}
__host__ __device__ constexpr int vz(int i) { return i == 0 ? 0 : (i < 9 ? 0 : (i < 18 ? 1 : -1)); }

__device__ __forceinline__ int wrapi(int v, int n) { return v < 0 ? v + n : (v >= n ? v - n : v); }

template <int BX>
__global__ void __launch_bounds__(BX) copy_soa(const double *__restrict__ src, double *__restrict__ dst, int nx,
                                               int ny, int nz) {
  const int x = blockIdx.x * BX + threadIdx.x;
  const int y = blockIdx.y, z = blockIdx.z;
  const long long pop = (long long)nx * ny, plane = 27LL * pop;
  double f[27];
#pragma unroll
  for (int i = 0; i < 27; ++i) {
    const int xs = wrapi(x - vx(i), nx), ys = wrapi(y - vy(i), ny), zs = wrapi(z - vz(i), nz);
    f[i] = __ldg(src + zs * plane + i * pop + (long long)ys * nx + xs);
  }
#pragma unroll
  for (int i = 0; i < 27; ++i) dst[z * plane + i * pop + (long long)y * nx + x] = f[i];
}

// AoSoA: element (z, y, xb, i, lane) at ((z*ny + y)*nxb + xb)*27*32 + i*32 + lane
template <int BX>
__global__ void __launch_bounds__(BX) copy_aosoa(const double *__restrict__ src, double *__restrict__ dst, int nx,
                                                 int ny, int nz) {
  const int x = blockIdx.x * BX + threadIdx.x;
  const int y = blockIdx.y, z = blockIdx.z;
  const int nxb = nx / 32;
  double f[27];
#pragma unroll
  for (int i = 0; i < 27; ++i) {
    const int xs = wrapi(x - vx(i), nx), ys = wrapi(y - vy(i), ny), zs = wrapi(z - vz(i), nz);
    const long long blk = ((long long)zs * ny + ys) * nxb + (xs >> 5);
    f[i] = __ldg(src + blk * (27 * 32) + i * 32 + (xs & 31));
  }
  const long long blk = ((long long)z * ny + y) * nxb + (x >> 5);
#pragma unroll
  for (int i = 0; i < 27; ++i) dst[blk * (27 * 32) + i * 32 + (x & 31)] = f[i];
}

template <class K>
float timeit(K k, dim3 grid, int bx, double *a, double *b, int nx, int ny, int nz) {
  for (int i = 0; i < 3; ++i) k<<<grid, bx>>>(a, b, nx, ny, nz);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  const int reps = 20;
  for (int i = 0; i < reps; ++i) {
    if (i % 2 == 0) k<<<grid, bx>>>(a, b, nx, ny, nz);
    else k<<<grid, bx>>>(b, a, nx, ny, nz);
  }
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  CK(cudaGetLastError());
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms / reps;
}

int main() {
  const int nx = 1024, ny = 1024, nz = 128;
  const size_t n = 27ull * nx * ny * nz;
  double *a, *b;
  CK(cudaMalloc(&a, n * 8));
  CK(cudaMalloc(&b, n * 8));
  CK(cudaMemset(a, 0, n * 8));
  CK(cudaMemset(b, 0, n * 8));
  const double cells = (double)nx * ny * nz;
  auto rep = [&](const char *name, float ms) {
    printf("%-28s %8.3f ms %9.1f MLUPS %8.1f GB/s\n", name, ms, cells / ms / 1e3, cells * 432.0 / ms / 1e6);
  };
  rep("SoA   bx128", timeit(copy_soa<128>, dim3(nx / 128, ny, nz), 128, a, b, nx, ny, nz));
  rep("SoA   bx256", timeit(copy_soa<256>, dim3(nx / 256, ny, nz), 256, a, b, nx, ny, nz));
  rep("AoSoA bx128", timeit(copy_aosoa<128>, dim3(nx / 128, ny, nz), 128, a, b, nx, ny, nz));
  rep("AoSoA bx256", timeit(copy_aosoa<256>, dim3(nx / 256, ny, nz), 256, a, b, nx, ny, nz));
  rep("AoSoA bx32", timeit(copy_aosoa<32>, dim3(nx / 32, ny, nz), 32, a, b, nx, ny, nz));
  // plain streaming copy of the same bytes (cudaMemcpy D2D) for reference
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < 10; ++i) CK(cudaMemcpyAsync(b, a, n * 8, cudaMemcpyDeviceToDevice));
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  rep("cudaMemcpy D2D (same bytes)", ms / 10);
  return 0;
}
