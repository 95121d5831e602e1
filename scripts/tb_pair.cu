// tb_pair.cu — scratch A/B microbenchmark (not product code): the product two-step sweep
// k_pull2 (16x8 tiles, register prefetch) against the x-paired sweep k_pull2p (tb_pair.cuh) on
// the C2 lattice (D3Q19 raw-moment MRT, zero-centered + delta equilibrium, 256^3, general
// rates), fp32 and fp64: time per two steps (CUDA events, 20 launches after 2 warm-up) and the
// max |difference| of the outputs of one launch from the same input.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -lineinfo
//        -I paper_2211_02435_b200/csrc -I include -I scripts scripts/tb_pair.cu -o scripts/tb_pair
#include <cstdio>
#include <cstdlib>

#include "kernels.cuh"
#include "tb_pair.cuh"
#include "tb3d_depth.cuh"

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
__global__ void fill_noise(real *a, size_t n, real amp) {
  for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < n; k += (size_t)gridDim.x * blockDim.x) {
    unsigned long long z = k * 0x9E3779B97F4A7C15ull + 0x1234567ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    a[k] = amp * (real)((double)(z >> 11) * (1.0 / 9007199254740992.0) - 0.5);
  }
}

template <class real>
__global__ void maxdiff(const real *a, const real *b, size_t n, double *out) {
  double m = 0;
  for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < n; k += (size_t)gridDim.x * blockDim.x)
    m = fmax(m, fabs((double)a[k] - (double)b[k]));
  atomicMax(reinterpret_cast<unsigned long long *>(out), __double_as_longlong(m));
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

template <class real>
struct Bench {
  using S = D3Q19;
  GridParams g{};
  size_t elems;
  real *a, *b, *ref;
  Rates<real> r;
  double cells;
  int zch;
  Bench(int nx, int ny, int nz, int zch_) : zch(zch_) {
    g.nx = nx;
    g.ny = ny;
    g.nzl = g.nzg = nz;
    g.pitch = nx;
    g.pop = (long long)ny * nx;
    g.plane = (long long)S::Q * g.pop;
    g.wrapz = 1;
    elems = (size_t)(nz + 2) * g.plane;
    CK(cudaMalloc(&a, elems * sizeof(real)));
    CK(cudaMalloc(&b, elems * sizeof(real)));
    CK(cudaMalloc(&ref, elems * sizeof(real)));
    for (int i = 0; i < 27; ++i) r.w[i] = real(1.0 + 0.02 * i);
    cells = (double)nx * ny * nz;
  }
  void reset() {
    fill_noise<<<1184, 256>>>(a, elems, real(1e-3));
    CK(cudaMemset(b, 0, elems * sizeof(real)));
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

template <class real, int MINB, bool TRIM>
void run_ref(Bench<real> &B, const char *tag) {
  using S = D3Q19;
  using T = Tile2<16, 8>;
  auto kern = k_pull2<S, SPACE_RAW, REG_DELTA, real, RS_GENERAL, 16, 8, MINB, true, false, TRIM>;
  const size_t smem = TRIM ? (size_t)Tile2Trim<16, 8, S>::RING * sizeof(real) : (size_t)3 * S::Q * T::HW * sizeof(real);
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  Force<real> fr{};
  dim3 grid((unsigned)(B.g.nx / 16), (unsigned)(B.g.ny / 8), (unsigned)B.zch);
  B.reset();
  kern<<<grid, T::THREADS, smem>>>(B.a, B.ref, B.g, B.r, real(0), fr);
  CK(cudaDeviceSynchronize());
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, kern));
  float ms = time_k([&](int p) { kern<<<grid, T::THREADS, smem>>>(p ? B.b : B.a, p ? B.a : B.b, B.g, B.r, real(0), fr); });
  printf("%-40s %7.3f ms/2 steps %8.0f MLUPS  regs %3d  smem %6zu\n", tag, ms, 2.0 * B.cells / (ms * 1e-3) / 1e6,
         fa.numRegs, smem);
}

template <class real, int TX, int TY, int MINB, bool PF>
void run_pair(Bench<real> &B, const char *tag) {
  using S = D3Q19;
  using T = TileP<TX, TY>;
  auto kern = k_pull2p<S, SPACE_RAW, REG_DELTA, real, RS_GENERAL, TX, TY, MINB, PF>;
  const size_t smem = (size_t)3 * S::Q * T::HW * sizeof(real);
  if (smem > 227 * 1024) {
    printf("%-40s smem %zu too large\n", tag, smem);
    return;
  }
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  Force<real> fr{};
  dim3 grid((unsigned)(B.g.nx / TX), (unsigned)(B.g.ny / TY), (unsigned)B.zch);
  B.reset();
  kern<<<grid, T::THREADS, smem>>>(B.a, B.b, B.g, B.r, real(0), fr);
  CK(cudaDeviceSynchronize());
  const double md = B.diff();
  int nb = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, T::THREADS, smem));
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, kern));
  float ms = time_k([&](int p) { kern<<<grid, T::THREADS, smem>>>(p ? B.b : B.a, p ? B.a : B.b, B.g, B.r, real(0), fr); });
  printf("%-40s %7.3f ms/2 steps %8.0f MLUPS  regs %3d  lmem %3zu  smem %6zu  %d CTA/SM  maxdiff %.3e\n", tag, ms,
         2.0 * B.cells / (ms * 1e-3) / 1e6, fa.numRegs, fa.localSizeBytes, smem, nb, md);
}

// the product kernel k_pull2 at other tiles / occupancies (maxdiff against the 16x8 product output)
template <class real, int TX, int TY, int MINB, bool PF, bool TRIM>
void run_k2(Bench<real> &B, const char *tag) {
  using S = D3Q19;
  using T = Tile2<TX, TY>;
  auto kern = k_pull2<S, SPACE_RAW, REG_DELTA, real, RS_GENERAL, TX, TY, MINB, PF, false, TRIM>;
  const size_t smem = TRIM ? (size_t)Tile2Trim<TX, TY, S>::RING * sizeof(real) : (size_t)3 * S::Q * T::HW * sizeof(real);
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  Force<real> fr{};
  dim3 grid((unsigned)(B.g.nx / TX), (unsigned)(B.g.ny / TY), (unsigned)B.zch);
  B.reset();
  kern<<<grid, T::THREADS, smem>>>(B.a, B.b, B.g, B.r, real(0), fr);
  CK(cudaDeviceSynchronize());
  const double md = B.diff();
  int nb = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, T::THREADS, smem));
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, kern));
  float ms = time_k([&](int p) { kern<<<grid, T::THREADS, smem>>>(p ? B.b : B.a, p ? B.a : B.b, B.g, B.r, real(0), fr); });
  printf("%-40s %7.3f ms/2 steps %8.0f MLUPS  regs %3d  lmem %3zu  smem %6zu  %d CTA/SM  maxdiff %.3e\n", tag, ms,
         2.0 * B.cells / (ms * 1e-3) / 1e6, fa.numRegs, fa.localSizeBytes, smem, nb, md);
}

// depth-D 3D sweep (tb3d_depth.cuh) against D single k_pull steps (its own reference)
template <class real, int TX, int TY, int D, int MINB, bool PF>
void run_d3(Bench<real> &B, const char *tag) {
  using S = D3Q19;
  using T = Tile3D<S, TX, TY, D>;
  auto kern = k_pullD_3d<S, SPACE_RAW, REG_DELTA, real, RS_GENERAL, TX, TY, D, MINB, PF>;
  const size_t smem = (size_t)T::RING * sizeof(real);
  if (smem > 227 * 1024) {
    printf("%-40s smem %zu too large\n", tag, smem);
    return;
  }
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  Force<real> fr{};
  // reference: D single steps a -> ref (through b)
  B.reset();
  {
    dim3 grid((unsigned)((B.g.nx + BLOCK_X - 1) / BLOCK_X), (unsigned)B.g.ny, (unsigned)B.g.nzl);
    const real *sp = B.a;
    for (int k = 0; k < D; ++k) {
      real *d = ((D - 1 - k) % 2 == 0) ? B.ref : B.b;
      k_pull<S, SPACE_RAW, REG_DELTA, real, false, RS_GENERAL><<<grid, BLOCK_X>>>(sp, d, B.g, B.r, real(0), fr);
      sp = d;
    }
    CK(cudaDeviceSynchronize());
  }
  CK(cudaMemset(B.b, 0, B.elems * sizeof(real)));
  dim3 grid((unsigned)(B.g.nx / TX), (unsigned)(B.g.ny / TY), (unsigned)B.zch);
  kern<<<grid, T::THREADS, smem>>>(B.a, B.b, B.g, B.r, real(0), fr);
  CK(cudaDeviceSynchronize());
  const double md = B.diff();
  int nb = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, T::THREADS, smem));
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, kern));
  float ms = time_k([&](int p) { kern<<<grid, T::THREADS, smem>>>(p ? B.b : B.a, p ? B.a : B.b, B.g, B.r, real(0), fr); });
  printf("%-40s %7.3f ms/%d steps %7.4f ms/step %8.0f MLUPS  regs %3d  lmem %3zu  smem %6zu  %d CTA/SM  maxdiff %.3e\n",
         tag, ms, D, ms / D, D * B.cells / (ms * 1e-3) / 1e6, fa.numRegs, fa.localSizeBytes, smem, nb, md);
}

int main(int argc, char **argv) {
  const int which = argc > 1 ? atoi(argv[1]) : 0;  // 0 both, 1 fp32, 2 fp64
  const int zch = argc > 2 ? atoi(argv[2]) : 6;
  if (which != 2) {
    Bench<float> B(256, 256, 256, zch);
    run_ref<float, 3, false>(B, "C2 f32 k_pull2 16x8 PF (product)");
    run_d3<float, 16, 8, 2, 3, true>(B, "C2 f32 depth 2 16x8 minb 3");
    run_d3<float, 16, 8, 3, 2, true>(B, "C2 f32 depth 3 16x8 minb 2");
    run_d3<float, 16, 8, 3, 3, true>(B, "C2 f32 depth 3 16x8 minb 3");
    run_d3<float, 16, 16, 3, 1, true>(B, "C2 f32 depth 3 16x16 minb 1");
    run_d3<float, 32, 8, 3, 1, true>(B, "C2 f32 depth 3 32x8 minb 1");
  }
  if (which != 1) {
    Bench<double> B(256, 256, 256, zch);
    run_ref<double, 2, true>(B, "C2 f64 k_pull2 16x8 PF trim (product)");
    run_d3<double, 16, 8, 2, 2, true>(B, "C2 f64 depth 2 16x8 minb 2");
    run_d3<double, 16, 8, 3, 1, true>(B, "C2 f64 depth 3 16x8 minb 1");
    run_d3<double, 16, 8, 3, 2, true>(B, "C2 f64 depth 3 16x8 minb 2");
  }
  return 0;
}
