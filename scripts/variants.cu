// variants.cu — scratch microbenchmark (not product code): launch-configuration and
// cache-hint variants of the D3Q27 cumulant pull kernel, plus the same-pattern pure
// streaming "copy" (speed-of-light reference for this access pattern).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//          -I paper_2211_02435_b200/csrc scripts/variants.cu -o scripts/variants
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "kernels.cuh"

using namespace lbm;

enum { LD_NC = 0, LD_CS = 1, LD_DEF = 2 };
enum { ST_DEF = 0, ST_CS = 1, ST_CG = 2 };

template <int LD>
__device__ __forceinline__ double ld(const double *p) {
  if constexpr (LD == LD_NC) return __ldg(p);
  else if constexpr (LD == LD_CS) return __ldcs(p);
  else return *p;
}
template <int ST>
__device__ __forceinline__ void st(double *p, double v) {
  if constexpr (ST == ST_CS) __stcs(p, v);
  else if constexpr (ST == ST_CG) __stcg(p, v);
  else *p = v;
}

template <class S, int SPACE, int REG, int BX, int MINB, int LDM, int STM, bool COLLIDE>
__global__ void __launch_bounds__(BX, MINB) k_var(const double *__restrict__ src, double *__restrict__ dst,
                                                  const GridParams g, const Rates<double> r) {
  const int x = blockIdx.x * BX + threadIdx.x;
  if (x >= g.nx) return;
  const int y = blockIdx.y;
  const int zl = g.zbegin + blockIdx.z;
  int xs[3], ys[3];
  long long zo[3];
#pragma unroll
  for (int s = -1; s <= 1; ++s) {
    xs[s + 1] = wrapi(x + s, g.nx);
    ys[s + 1] = wrapi(y + s, g.ny) * g.pitch;
    zo[s + 1] = (long long)(wrapi(zl + s, g.nzl) + 1) * g.plane;
  }
  const long long own = (long long)(zl + 1) * g.plane + (long long)y * g.pitch + x;
  double f[S::Q];
  sfor<S::Q>([&](auto i) {
    constexpr int cx = S::mx(i), cy = S::my(i), cz = S::mz(i);
    f[i] = ld<LDM>(src + zo[1 - cz] + (long long)i * g.pop + ys[1 - cy] + xs[1 - cx]);
  });
  if constexpr (COLLIDE) collide<S, SPACE, REG, double>(f, r, 0.0);
  sfor<S::Q>([&](auto i) { st<STM>(dst + own + (long long)i * g.pop, f[i]); });
}

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e = (x);                                                       \
    if (e != cudaSuccess) {                                                    \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

template <class K>
float time_kernel(K kernel, int bx, const GridParams &g, double *a, double *b, const Rates<double> &r, int reps) {
  dim3 grid((g.nx + bx - 1) / bx, g.ny, g.nzl);
  for (int i = 0; i < 3; ++i) kernel<<<grid, bx>>>(a, b, g, r);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < reps; ++i) {
    if (i % 2 == 0) kernel<<<grid, bx>>>(a, b, g, r);
    else kernel<<<grid, bx>>>(b, a, g, r);
  }
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  CK(cudaGetLastError());
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms / reps;
}

int main(int argc, char **argv) {
  int nx = 1024, ny = 1024, nz = 128;
  if (argc > 3) {
    nx = atoi(argv[1]);
    ny = atoi(argv[2]);
    nz = atoi(argv[3]);
  }
  using S = D3Q27;
  GridParams g{};
  g.nx = nx;
  g.ny = ny;
  g.nzl = nz;
  g.nzg = nz;
  g.pitch = (nx + 15) / 16 * 16;
  g.pop = (long long)ny * g.pitch;
  g.plane = 27LL * g.pop;
  g.wrapz = 1;
  size_t elems = (size_t)(nz + 2) * g.plane;
  double *a, *b;
  CK(cudaMalloc(&a, elems * 8));
  CK(cudaMalloc(&b, elems * 8));
  CK(cudaMemset(a, 0, elems * 8));
  CK(cudaMemset(b, 0, elems * 8));
  Rates<double> r;
  for (int i = 0; i < 27; ++i) r.w[i] = 1.0 + 0.02 * i;
  const double cells = (double)nx * ny * nz;
  const int reps = 20;
  auto report = [&](const char *name, float ms) {
    printf("%-44s %8.3f ms  %9.1f MLUPS  %7.1f GB/s\n", name, ms, cells / (ms * 1e-3) / 1e6,
           cells * 432.0 / (ms * 1e-3) / 1e9);
  };
  constexpr int K = SPACE_CUMULANT, R = REG_ZC_ABS;
  report("copy    bx128 nc/def", time_kernel(k_var<S, K, R, 128, 1, LD_NC, ST_DEF, false>, 128, g, a, b, r, reps));
  report("copy    bx128 cs/cs", time_kernel(k_var<S, K, R, 128, 1, LD_CS, ST_CS, false>, 128, g, a, b, r, reps));
  report("copy    bx256 nc/def", time_kernel(k_var<S, K, R, 256, 1, LD_NC, ST_DEF, false>, 256, g, a, b, r, reps));
  {
    auto prod = [](const double *a_, double *b_, const GridParams &g_, const Rates<double> &r_) {};
    (void)prod;
    dim3 grid((g.nx + 127) / 128, g.ny, g.nzl);
    for (int i = 0; i < 3; ++i) k_pull<S, K, R, double, false><<<grid, 128>>>(a, b, g, r, 0.0);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int i = 0; i < reps; ++i) {
      if (i % 2 == 0) k_pull<S, K, R, double, false><<<grid, 128>>>(a, b, g, r, 0.0);
      else k_pull<S, K, R, double, false><<<grid, 128>>>(b, a, g, r, 0.0);
    }
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    report("K       production k_pull", ms / reps);
  }
  report("K       bx128 nc/def (variant)", time_kernel(k_var<S, K, R, 128, 1, LD_NC, ST_DEF, true>, 128, g, a, b, r, reps));
  report("K       bx128 cs/def", time_kernel(k_var<S, K, R, 128, 1, LD_CS, ST_DEF, true>, 128, g, a, b, r, reps));
  report("K       bx128 nc/cs", time_kernel(k_var<S, K, R, 128, 1, LD_NC, ST_CS, true>, 128, g, a, b, r, reps));
  report("K       bx128 cs/cs", time_kernel(k_var<S, K, R, 128, 1, LD_CS, ST_CS, true>, 128, g, a, b, r, reps));
  report("K       bx128 nc/cg", time_kernel(k_var<S, K, R, 128, 1, LD_NC, ST_CG, true>, 128, g, a, b, r, reps));
  report("K       bx128 def/def", time_kernel(k_var<S, K, R, 128, 1, LD_DEF, ST_DEF, true>, 128, g, a, b, r, reps));
  report("K       bx64  nc/def", time_kernel(k_var<S, K, R, 64, 1, LD_NC, ST_DEF, true>, 64, g, a, b, r, reps));
  report("K       bx256 nc/def", time_kernel(k_var<S, K, R, 256, 1, LD_NC, ST_DEF, true>, 256, g, a, b, r, reps));
  report("K       bx128 minb8 nc/def", time_kernel(k_var<S, K, R, 128, 8, LD_NC, ST_DEF, true>, 128, g, a, b, r, reps));
  report("K       bx256 minb4 nc/def", time_kernel(k_var<S, K, R, 256, 4, LD_NC, ST_DEF, true>, 256, g, a, b, r, reps));
  report("K       bx128 minb8 cs/cs", time_kernel(k_var<S, K, R, 128, 8, LD_CS, ST_CS, true>, 128, g, a, b, r, reps));
  report("CM      bx128 nc/def", time_kernel(k_var<S, SPACE_CENTRAL, R, 128, 1, LD_NC, ST_DEF, true>, 128, g, a, b, r, reps));
  report("RAW-d   bx128 nc/def", time_kernel(k_var<S, SPACE_RAW, REG_DELTA, 128, 1, LD_NC, ST_DEF, true>, 128, g, a, b, r, reps));
  cudaFree(a);
  cudaFree(b);
  return 0;
}
