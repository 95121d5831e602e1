// tb_bulk_variants.cu — scratch microbenchmark (not product code): the bulk-copy staged
// temporal-blocking kernel k_pull2b (tile, stages, CTAs/SM) against the register-prefetch
// k_pull2 / k_pull2_2d and two single-step k_pull launches, with a check that every variant
// equals two single steps to rounding.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//          -I paper_2211_02435_b200/csrc -I scripts scripts/tb_bulk_variants.cu -o scripts/tb_bulk_variants
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "ops.cuh"
#include "tb_bulk.cuh"

using namespace lbm;

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e = (x);                                                             \
    if (e != cudaSuccess) {                                                          \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                       \
    }                                                                                \
  } while (0)

// smooth + noisy state: base + amp * hash noise
template <class real>
__global__ void fill_noise(real *a, size_t n, double base, double amp, unsigned seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    unsigned long long z = i * 0x9E3779B97F4A7C15ull + seed;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    a[i] = (real)(base + amp * ((double)(z >> 11) * 0x1.0p-53 - 0.5));
  }
}

template <class real>
__global__ void maxdiff(const real *a, const real *b, size_t n, double *out) {
  double m = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    m = fmax(m, fabs((double)a[i] - (double)b[i]));
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffff, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax((unsigned long long *)out, __double_as_longlong(m));
}

struct Bufs {
  void *a, *b, *ref;
  size_t elems;
};

template <class S, class real>
double check_against_single(const GridParams &g, Bufs &B, double *dmax) {
  // B.ref <- two single steps of B.a (B.b used as the intermediate)
  (void)g;
  CK(cudaMemset(dmax, 0, 8));
  maxdiff<real><<<1184, 256>>>((const real *)B.b, (const real *)B.ref, B.elems, dmax);
  double h;
  CK(cudaMemcpy(&h, dmax, 8, cudaMemcpyDeviceToHost));
  return h;
}

int g_reps = 10;
template <class K>
float time_kernel(K launch, int reps = -1) {
  if (reps < 0) reps = g_reps;
  for (int i = 0; i < 2; ++i) launch(i);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < reps; ++i) launch(i);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  CK(cudaGetLastError());
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms / reps;
}

template <class S, int SP, int REG, class real, int RS>
struct Bench {
  GridParams g;
  Bufs B;
  Rates<real> r;
  Force<real> fr{};
  real swe_g;
  double *dmax;
  double cells;
  double base_ms = 0;  // single steps, per 2 steps

  void reset_state() {
    fill_noise<real><<<1184, 256>>>((real *)B.a, B.elems, 0.1, 1e-3, 7u);
    CK(cudaDeviceSynchronize());
  }
  // reference: two single steps a -> tmp(b) -> ref
  void make_ref() {
    reset_state();
    dim3 grid((g.nx + 127) / 128, g.ny, g.nzl);
    // ghost planes unused (wrapz = 1)
    k_pull<S, SP, REG, real, false, RS><<<grid, 128>>>((const real *)B.a, (real *)B.b, g, r, swe_g, fr);
    k_pull<S, SP, REG, real, false, RS><<<grid, 128>>>((const real *)B.b, (real *)B.ref, g, r, swe_g, fr);
    CK(cudaDeviceSynchronize());
  }
  void single() {
    dim3 grid((g.nx + 127) / 128, g.ny, g.nzl);
    const real *a = (const real *)B.a;
    real *b = (real *)B.b;
    float ms = time_kernel([&](int i) {
      if (i % 2 == 0) k_pull<S, SP, REG, real, false, RS><<<grid, 128>>>(a, b, g, r, swe_g, fr);
      else k_pull<S, SP, REG, real, false, RS><<<grid, 128>>>((const real *)b, (real *)a, g, r, swe_g, fr);
    });
    base_ms = 2 * ms;
    cudaFuncAttributes at{};
    cudaFuncGetAttributes(&at, k_pull<S, SP, REG, real, false, RS>);
    printf("  single-step k_pull x2                 regs %3d            -> %7.3f ms / 2 steps %9.0f MLUPS\n",
           at.numRegs, base_ms, 2 * cells / (base_ms * 1e-3) / 1e6);
  }
  template <class Kern>
  void report(const char *what, Kern kern, dim3 grid, int threads, size_t smem) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    make_ref();
    reset_state();
    kern<<<grid, threads, smem>>>((const real *)B.a, (real *)B.b, g, r, swe_g, fr);
    CK(cudaDeviceSynchronize());
    CK(cudaGetLastError());
    const double d = check_against_single<S, real>(g, B, dmax);
    const real *a = (const real *)B.a;
    real *b = (real *)B.b;
    float ms = time_kernel([&](int i) {
      if (i % 2 == 0) kern<<<grid, threads, smem>>>(a, b, g, r, swe_g, fr);
      else kern<<<grid, threads, smem>>>((const real *)b, (real *)a, g, r, swe_g, fr);
    });
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, threads, smem);
    cudaFuncAttributes at{};
    cudaFuncGetAttributes(&at, kern);
    const double bpc = 2.0 * S::Q * sizeof(real);
    printf("  %-38s thr %3d smem %6zu B/SM %d regs %3d lmem %3zu -> %7.3f ms / 2 steps %9.0f MLUPS  frac %.3f  "
           "maxdiff %.2e\n",
           what, threads, smem, nb, at.numRegs, at.localSizeBytes, ms, 2 * cells / (ms * 1e-3) / 1e6,
           bpc * cells / (ms * 1e-3) / 6445e9, d);
  }
  // current register-prefetch kernels
  template <int TX, int TY, int MINB>
  void old3(int chunks) {
    using T = Tile2<TX, TY>;
    const size_t smem = (size_t)3 * S::Q * T::HW * sizeof(real);
    char nm[96];
    snprintf(nm, sizeof nm, "k_pull2 %dx%d minB %d pf (current)", TX, TY, MINB);
    report(nm, k_pull2<S, SP, REG, real, RS, TX, TY, MINB, true, false>, dim3(g.nx / TX, g.ny / TY, chunks),
           T::THREADS, smem);
  }
  template <int TX, int MINB, bool PF>
  void old2(int chunks) {
    using T = Tile1<TX>;
    const size_t smem = (size_t)3 * S::Q * T::HW * sizeof(real);
    char nm[96];
    snprintf(nm, sizeof nm, "k_pull2_2d %d minB %d pf %d (current)", TX, MINB, (int)PF);
    report(nm, k_pull2_2d<S, SP, REG, real, RS, TX, MINB, PF, false>, dim3(g.nx / TX, chunks, 1), T::THREADS, smem);
  }
  template <int TX, int TY, int MINB, bool PF>
  void ws(int chunks) {
    using T = TileW<S, TX, TY>;
    char nm[96];
    snprintf(nm, sizeof nm, "k_pull2w %dx%d minB %d pf %d", TX, TY, MINB, (int)PF);
    report(nm, k_pull2w<S, SP, REG, real, RS, TX, TY, MINB, PF, false>, dim3(g.nx / TX, g.ny / TY, chunks),
           T::THREADS, T::template smem<real>());
  }
  template <int TX, int TY, int MINB, int NS>
  void bulk(int chunks) {
    using T = TileB<S, TX, TY, real, NS>;
    char nm[96];
    snprintf(nm, sizeof nm, "k_pull2b %dx%d minB %d NS %d", TX, S::D == 2 ? 1 : TY, MINB, NS);
    dim3 grid = S::D == 2 ? dim3(g.nx / TX, chunks, 1) : dim3(g.nx / TX, g.ny / TY, chunks);
    report(nm, k_pull2b<S, SP, REG, real, RS, TX, TY, MINB, NS, false>, grid, T::THREADS, T::smem());
  }
};

template <class S, int SP, int REG, class real, int RS>
Bench<S, SP, REG, real, RS> make(int nx, int ny, int nz, double swe_g) {
  Bench<S, SP, REG, real, RS> b{};
  GridParams &g = b.g;
  g.nx = nx;
  g.ny = S::D == 2 ? 1 : ny;
  g.nzl = S::D == 2 ? ny : nz;
  g.nzg = g.nzl;
  g.pitch = nx;
  g.pop = (long long)g.ny * g.pitch;
  g.plane = (long long)S::Q * g.pop;
  g.wrapz = 1;
  for (int i = 0; i < 27; ++i) b.r.w[i] = (real)(1.0 + 0.02 * i);
  b.swe_g = (real)swe_g;
  b.B.elems = (size_t)(g.nzl + 2) * g.plane;
  CK(cudaMalloc(&b.B.a, b.B.elems * sizeof(real)));
  CK(cudaMalloc(&b.B.b, b.B.elems * sizeof(real)));
  CK(cudaMalloc(&b.B.ref, b.B.elems * sizeof(real)));
  CK(cudaMemset(b.B.b, 0, b.B.elems * sizeof(real)));
  CK(cudaMemset(b.B.ref, 0, b.B.elems * sizeof(real)));
  CK(cudaMalloc(&b.dmax, 8));
  b.cells = (double)nx * ny * (S::D == 2 ? 1 : nz);
  return b;
}
template <class BB>
void release(BB &b) {
  cudaFree(b.B.a);
  cudaFree(b.B.b);
  cudaFree(b.B.ref);
  cudaFree(b.dmax);
}

int main(int argc, char **argv) {
  const int which = argc > 1 ? atoi(argv[1]) : -1;
  const int small = argc > 2 ? atoi(argv[2]) : 0;  // sanitizer runs: small lattices
  if (small) g_reps = 1;
  if (which < 0 || which == 0) {
    printf("C5: D2Q9 SWE CM abs fp64 RS_REG 8192^2 (closed-form Zhou equilibrium)\n");
    auto b = make<D2Q9, SPACE_SWE, REG_ABS, double, RS_REG>(small ? 512 : 8192, small ? 64 : 8192, 1, 0.0613125);
    b.single();
    b.old2<256, 2, true>(37);
    b.bulk<256, 1, 2, 2>(37);
    release(b);
  }
  if (which < 0 || which == 1) {
    printf("C2: D3Q19 RAW zc+delta fp64 256^3\n");
    auto b = make<D3Q19, SPACE_RAW, REG_DELTA, double, RS_GENERAL>(small ? 64 : 256, small ? 32 : 256, small ? 16 : 256, 0.0);
    b.single();
    b.old3<16, 8, 2>(3);
    b.ws<16, 8, 2, false>(3);
    b.ws<16, 8, 2, true>(3);
    b.ws<16, 8, 1, true>(3);
    b.ws<16, 8, 2, false>(6);
    b.ws<32, 4, 2, false>(3);
    b.ws<16, 16, 1, false>(6);
    b.ws<32, 8, 1, false>(6);
    b.ws<8, 8, 3, false>(3);
    release(b);
  }
  if (which < 0 || which == 2) {
    printf("C2: D3Q19 RAW zc+delta fp32 256^3\n");
    auto b = make<D3Q19, SPACE_RAW, REG_DELTA, float, RS_GENERAL>(small ? 64 : 256, small ? 32 : 256, small ? 16 : 256, 0.0);
    b.single();
    b.old3<16, 8, 3>(3);
    b.ws<16, 8, 2, false>(3);
    b.ws<16, 8, 2, true>(3);
    b.ws<16, 8, 3, false>(3);
    b.ws<16, 8, 3, true>(3);
    b.ws<16, 16, 2, false>(6);
    b.ws<32, 8, 2, false>(6);
    b.ws<32, 8, 2, true>(6);
    release(b);
  }
  if (which < 0 || which == 3) {
    printf("C4: D3Q27 cumulant zc+eq fp64 1024^2 x 128\n");
    auto b = make<D3Q27, SPACE_CUMULANT, REG_ZC_ABS, double, RS_GENERAL>(small ? 64 : 1024, small ? 32 : 1024, small ? 16 : 128, 0.0);
    b.single();
    b.ws<16, 8, 1, false>(1);
    b.ws<16, 8, 1, true>(1);
    b.ws<8, 8, 2, false>(1);
    b.ws<16, 4, 2, false>(1);
    release(b);
  }
  return 0;
}
