// tb2d_depth.cu — scratch A/B microbenchmark (prototype, not product code): 2D temporal
// blocking of depth D (tb2d_depth.cuh k_pullD_2d) against the product two-step sweep
// k_pull2_2d on the C5 lattice (D2Q9 shallow water, CM space, Zhou equilibrium, absolute
// storage, fp64, R- rates with the shear rate 0.6957, 8192^2): time per time step and the max
// |difference| against D single steps of k_pull from the same input.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -lineinfo
//        -I paper_2211_02435_b200/csrc -I include -I scripts scripts/tb2d_depth.cu -o scripts/tb2d_depth
#include <cstdio>
#include <cstdlib>

#include "kernels.cuh"
#include "tb2d_1b.cuh"


using namespace lbm;
using S = D2Q9;
constexpr int SP = SPACE_SWE, RG = REG_ABS, RSM = RS_REG;

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e = (x);                                                             \
    if (e != cudaSuccess) {                                                          \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                       \
    }                                                                                \
  } while (0)

// f_eq(h = 1, u = 0) of the Zhou equilibrium, times (1 + 1e-3 noise)
__global__ void fill_swe(double *a, GridParams g, double gg) {
  const long long cells = (long long)g.nzl * g.pitch;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < cells; c += (long long)gridDim.x * blockDim.x) {
    const long long z = c / g.pitch, x = c % g.pitch;
    sfor<S::Q>([&](auto i) {
      constexpr int c2 = S::mx(i) * S::mx(i) + S::mz(i) * S::mz(i);
      const double base = c2 == 0 ? 1.0 - 5.0 * gg / 6.0 : (c2 == 1 ? gg / 6.0 : gg / 24.0);
      unsigned long long h = (unsigned long long)(c * 9 + i) * 0x9E3779B97F4A7C15ull + 0x1234567ull;
      h = (h ^ (h >> 30)) * 0xBF58476D1CE4E5B9ull;
      h = (h ^ (h >> 27)) * 0x94D049BB133111EBull;
      h ^= h >> 31;
      const double nz = (double)(h >> 11) * (1.0 / 9007199254740992.0) - 0.5;
      a[(z + 1) * g.plane + (long long)i * g.pop + x] = base * (1.0 + 1e-3 * nz);
    });
  }
}

__global__ void maxdiff(const double *a, const double *b, size_t n, double *out) {
  double m = 0;
  for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < n; k += (size_t)gridDim.x * blockDim.x)
    m = fmax(m, fabs(a[k] - b[k]));
  atomicMax(reinterpret_cast<unsigned long long *>(out), __double_as_longlong(m));
}

struct Bench {
  GridParams g{};
  size_t elems;
  double *a, *b, *ref, *tmp;
  Rates<double> r{};
  double gg, cells;
  Bench(int nx, int ny) {
    g.nx = nx;
    g.ny = 1;
    g.nzl = g.nzg = ny;
    g.pitch = nx;
    g.pop = nx;
    g.plane = (long long)S::Q * g.pop;
    g.wrapz = 1;
    elems = (size_t)(ny + 2) * g.plane;
    CK(cudaMalloc(&a, elems * 8));
    CK(cudaMalloc(&b, elems * 8));
    CK(cudaMalloc(&ref, elems * 8));
    CK(cudaMalloc(&tmp, elems * 8));
    gg = 0.06131250000000001;
    for (int i = 0; i < 27; ++i) r.w[i] = 1.0;
    r.w[3] = r.w[4] = 0.6956521739130436;
    cells = (double)nx * ny;
  }
  void reset() {
    fill_swe<<<1184, 256>>>(a, g, gg);
    CK(cudaMemset(b, 0, elems * 8));
    CK(cudaDeviceSynchronize());
  }
  // D single steps a -> ref (ping-pong through tmp, the last step lands in ref)
  void reference(int D) {
    Force<double> fr{};
    dim3 grid((unsigned)((g.nx + BLOCK_X - 1) / BLOCK_X), 1, (unsigned)g.nzl);
    const double *s = a;
    for (int k = 0; k < D; ++k) {
      double *d = ((D - 1 - k) % 2 == 0) ? ref : tmp;
      k_pull<S, SP, RG, double, false, RSM><<<grid, BLOCK_X>>>(s, d, g, r, gg, fr);
      s = d;
    }
    CK(cudaDeviceSynchronize());
  }
  double diff() {
    double *dm;
    CK(cudaMalloc(&dm, 8));
    CK(cudaMemset(dm, 0, 8));
    maxdiff<<<1184, 256>>>(b + g.plane, ref + g.plane, (size_t)g.nzl * g.plane, dm);
    double md = 0;
    CK(cudaMemcpy(&md, dm, 8, cudaMemcpyDeviceToHost));
    cudaFree(dm);
    return md;
  }
};

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

void run_product(Bench &B, int chunks) {
  using T = Tile1<256>;
  auto kern = k_pull2_2d<S, SP, RG, double, RSM, 256, 2, true, false>;
  const size_t smem = (size_t)3 * S::Q * T::HW * 8;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  Force<double> fr{};
  dim3 grid((unsigned)(B.g.nx / 256), (unsigned)chunks);
  B.reset();
  B.reference(2);
  kern<<<grid, T::THREADS, smem>>>(B.a, B.b, B.g, B.r, B.gg, fr);
  CK(cudaDeviceSynchronize());
  const double md = B.diff();
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, kern));
  float ms = time_k([&](int p) { kern<<<grid, T::THREADS, smem>>>(p ? B.b : B.a, p ? B.a : B.b, B.g, B.r, B.gg, fr); });
  printf("C5 k_pull2_2d 256 (product) chunks %3d       %7.4f ms/step %8.0f MLUPS  regs %3d  smem %6zu  maxdiff %.3e\n",
         chunks, ms / 2, 2.0 * B.cells / (ms * 1e-3) / 1e6, fa.numRegs, smem, md);
}

template <int TX, int D, int MINB, bool PF>
void run_depth(Bench &B, int chunks) {
  using T = TileD<S, TX, D>;
  auto kern = k_pullD_2d<S, SP, RG, double, RSM, TX, D, MINB, PF>;
  const size_t smem = (size_t)T::RING * 8;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  Force<double> fr{};
  dim3 grid((unsigned)(B.g.nx / TX), (unsigned)chunks);
  B.reset();
  B.reference(D);
  kern<<<grid, T::THREADS, smem>>>(B.a, B.b, B.g, B.r, B.gg, fr);
  CK(cudaDeviceSynchronize());
  const double md = B.diff();
  int nb = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, T::THREADS, smem));
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, kern));
  float ms = time_k([&](int p) { kern<<<grid, T::THREADS, smem>>>(p ? B.b : B.a, p ? B.a : B.b, B.g, B.r, B.gg, fr); });
  printf("C5 depth %d TX %3d minb %d pf %d chunks %3d     %7.4f ms/step %8.0f MLUPS  regs %3d  lmem %3zu  smem %6zu  %d CTA/SM  maxdiff %.3e\n",
         D, TX, MINB, (int)PF, chunks, ms / D, (double)D * B.cells / (ms * 1e-3) / 1e6, fa.numRegs, fa.localSizeBytes,
         smem, nb, md);
}

template <int TX, int D, int MINB, bool PF>
void run_1b(Bench &B, int chunks) {
  using T = TileD<S, TX, D, 1>;
  auto kern = k_pullD1b_2d<S, SP, RG, double, RSM, TX, D, MINB, PF>;
  const size_t smem = (size_t)T::RING * 8;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  Force<double> fr{};
  dim3 grid((unsigned)(B.g.nx / TX), (unsigned)chunks);
  B.reset();
  B.reference(D);
  kern<<<grid, T::THREADS, smem>>>(B.a, B.b, B.g, B.r, B.gg, fr);
  CK(cudaDeviceSynchronize());
  const double md = B.diff();
  int nb = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, T::THREADS, smem));
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, kern));
  float ms = time_k([&](int p) { kern<<<grid, T::THREADS, smem>>>(p ? B.b : B.a, p ? B.a : B.b, B.g, B.r, B.gg, fr); });
  printf("C5 1-barrier depth %d TX %3d minb %d pf %d ch %3d  %7.4f ms/step %8.0f MLUPS  regs %3d  lmem %3zu  smem %6zu  %d CTA/SM  maxdiff %.3e\n",
         D, TX, MINB, (int)PF, chunks, ms / D, (double)D * B.cells / (ms * 1e-3) / 1e6, fa.numRegs, fa.localSizeBytes,
         smem, nb, md);
}

int main(int argc, char **argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 8192;
  Bench B(n, n);
  run_product(B, 37);
  run_depth<256, 3, 2, true>(B, 37);
  run_depth<256, 3, 2, true>(B, 74);
  run_1b<256, 3, 2, true>(B, 37);
  run_1b<256, 3, 2, true>(B, 74);
  run_1b<256, 3, 1, true>(B, 74);
  run_1b<256, 4, 1, true>(B, 37);
  run_1b<256, 4, 1, true>(B, 74);
  run_1b<128, 3, 3, true>(B, 74);
  run_1b<128, 4, 2, true>(B, 74);
  run_1b<256, 2, 2, true>(B, 37);
  return 0;
}
