// tma_probe.cu — scratch check of the TMA helpers (not product code).  mode: bit0 map in global
// memory, bit1 L2 promotion none, bit2 no .tile qualifier, bit3 2D map
#include <cstdio>
#include <cstdlib>
#include "tma.cuh"
using namespace lbm;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("mode %d: CUDA error %s at %d\n", mode, cudaGetErrorString(e), __LINE__); return 1; } } while (0)
__device__ __forceinline__ void tma_load_4d_notile(void *dst, const CUtensorMap *map, int c0, int c1, int c2, int c3,
                                            uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int c0, int c1, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__global__ void probe(const __grid_constant__ CUtensorMap tmap, const CUtensorMap *gmap, double *out, int mode) {
  __shared__ __align__(128) double buf[18 * 10];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_fence_init(); }
  __syncthreads();
  if (threadIdx.x == 0) {
    const CUtensorMap *m = (mode & 1) ? gmap : &tmap;
    mbar_arrive_expect_tx(&bar, 18 * 10 * 8);
    if (mode & 8) tma_load_2d(buf, m, -1, 3 + 32 * (2 + 5 * 1), &bar);
    else if (mode & 4) tma_load_4d_notile(buf, m, -1, 3, 2, 1, &bar);
    else tma_load_4d(buf, m, -1, 3, 2, 1, &bar);
  }
  mbar_wait(&bar, 0);
  for (int k = threadIdx.x; k < 180; k += blockDim.x) out[k] = buf[k];
}
int main(int argc, char **argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 0;
  const int nx = 64, ny = 32, q = 5, planes = 4;
  size_t n = (size_t)nx * ny * q * planes;
  double *h = new double[n], *d, *o;
  for (size_t k = 0; k < n; ++k) h[k] = (double)k;
  CK(cudaMalloc(&d, n * 8)); CK(cudaMalloc(&o, 180 * 8));
  CK(cudaMemcpy(d, h, n * 8, cudaMemcpyHostToDevice));
  CUtensorMap m;
  if (mode & 8) {  // 2D view: rows of nx, ny * q * planes rows
    CK(encode_grid_tmap<double>(&m, d, nx, ny * q * planes, 1, 1, nx, (long long)nx * ny * q * planes, (long long)nx * ny * q * planes, 18, 10));
  } else {
    CK(encode_grid_tmap<double>(&m, d, nx, ny, q, planes, nx, (long long)nx * ny, (long long)nx * ny * q, 18, 10));
  }
  CUtensorMap *gm;
  CK(cudaMalloc(&gm, sizeof(CUtensorMap)));
  CK(cudaMemcpy(gm, &m, sizeof m, cudaMemcpyHostToDevice));
  printf("mode %d: sizeof %zu alignof %zu\n", mode, sizeof(CUtensorMap), alignof(CUtensorMap));
  probe<<<1, 128>>>(m, gm, o, mode);
  CK(cudaDeviceSynchronize());
  double r[180];
  CK(cudaMemcpy(r, o, 180 * 8, cudaMemcpyDeviceToHost));
  int bad = 0;
  for (int y = 0; y < 10; ++y) for (int x = 0; x < 18; ++x) {
    int gx = x - 1, gy = y + 3;
    double e = (gx < 0) ? 0.0 : (double)(((1 * q + 2) * ny + gy) * nx + gx);
    if (r[y * 18 + x] != e) { if (bad < 5) printf("mismatch %d %d: %g vs %g\n", x, y, r[y * 18 + x], e); bad++; }
  }
  printf("mode %d: tma probe %d mismatches\n", mode, bad);
  return 0;
}
