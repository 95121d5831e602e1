// tb_wave.cu — scratch A/B microbenchmark (not product code): the product two-step sweep
// k_pull2 (16x8 tiles, register prefetch) against the persistent wavefront sweep k_pull2_wave
// (tb_wave.cuh: no halo recompute, L2-resident ring) on the C2 lattice (D3Q19 raw-moment MRT, zero-centered + delta equilibrium, 256^3, general
// rates), fp32 and fp64: time per two steps (CUDA events, 20 launches after 2 warm-up) and the
// max |difference| of the outputs of one launch from the same input.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -lineinfo
//        -I paper_2211_02435_b200/csrc -I include -I scripts scripts/tb_wave.cu -o scripts/tb_wave
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "kernels.cuh"
#include "tb_wave.cuh"

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

template <class real, int NT, bool PF, bool FENCE = true, bool WAIT = true>
void run_wave(Bench<real> &B, const char *tag) {
  using S = D3Q19;
  auto kern = k_pull2_wave<S, SPACE_RAW, REG_DELTA, real, RS_GENERAL, NT, PF, FENCE, WAIT>;
  int dev = 0, nsm = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  const int G = nsm;
  const long long U = (long long)(B.g.nx / 32) * B.g.ny;
  if ((U + G - 1) / G * 32 > NT) {
    printf("%-40s NT %d too small\n", tag, NT);
    return;
  }
  real *scr;
  int *flags, *err;
  const size_t splane = (size_t)S::Q * B.g.pop;
  CK(cudaMalloc(&scr, kWaveSR * splane * sizeof(real)));
  CK(cudaMalloc(&flags, G * sizeof(int)));
  CK(cudaMalloc(&err, sizeof(int)));
  CK(cudaMemset(err, 0, sizeof(int)));
  Force<real> fr{};
  unsigned long long tmo = 2000000000ull;
  auto launch = [&](const real *s, real *d) {
    CK(cudaMemsetAsync(flags, 0, G * sizeof(int)));
    GridParams g = B.g;
    Rates<real> r = B.r;
    real sw = 0;
    void *args[] = {(void *)&s, (void *)&d, (void *)&scr, (void *)&flags, (void *)&g, (void *)&r, (void *)&sw,
                    (void *)&fr, (void *)&tmo, (void *)&err};
    CK(cudaLaunchCooperativeKernel((const void *)kern, dim3(G), dim3(NT), args, 0, 0));
  };
  B.reset();
  launch(B.a, B.b);
  CK(cudaDeviceSynchronize());
  const double md = B.diff();
  if (getenv("WAVE_DEBUG")) {  // where does it differ: per plane, then per row of the first bad plane
    const size_t E = B.elems;
    std::vector<real> hb(E), hr(E);
    CK(cudaMemcpy(hb.data(), B.b, E * sizeof(real), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hr.data(), B.ref, E * sizeof(real), cudaMemcpyDeviceToHost));
    int shown = 0;
    for (int z = 0; z < B.g.nzl && shown < 12; ++z) {
      double m = 0;
      int wi = -1, wy = -1, wx = -1;
      for (int i = 0; i < 19; ++i)
        for (int y = 0; y < B.g.ny; ++y)
          for (int x = 0; x < B.g.nx; ++x) {
            const size_t k = (size_t)(z + 1) * B.g.plane + (size_t)i * B.g.pop + (size_t)y * B.g.pitch + x;
            const double d = fabs((double)hb[k] - (double)hr[k]);
            if (d > m) { m = d; wi = i; wy = y; wx = x; }
          }
      if (m > 1e-6) { printf("  plane %d maxdiff %.3e at pop %d y %d x %d\n", z, m, wi, wy, wx); ++shown; }
    }
  }
  int e = 0;
  CK(cudaMemcpy(&e, err, sizeof(int), cudaMemcpyDeviceToHost));
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, kern));
  float ms = time_k([&](int p) { launch(p ? B.b : B.a, p ? B.a : B.b); });
  CK(cudaMemcpy(&e, err, sizeof(int), cudaMemcpyDeviceToHost));
  printf("%-40s %7.3f ms/2 steps %8.0f MLUPS  regs %3d  lmem %3zu  CTAs %d x %d  maxdiff %.3e  timeout %d\n", tag, ms,
         2.0 * B.cells / (ms * 1e-3) / 1e6, fa.numRegs, fa.localSizeBytes, G, NT, md, e);
  cudaFree(scr);
  cudaFree(flags);
  cudaFree(err);
}

int main(int argc, char **argv) {
  const int which = argc > 1 ? atoi(argv[1]) : 0;  // 0 both, 1 fp32, 2 fp64
  const int zch = 3;
  if (which != 2) {
    Bench<float> B(256, 256, 256, zch);
    run_ref<float, 3, false>(B, "C2 f32 k_pull2 16x8 PF (product)");
    run_wave<float, 448, true>(B, "C2 f32 wave 448 pf");
    run_wave<float, 448, true, false>(B, "C2 f32 wave 448 pf, no fence");
    run_wave<float, 448, true, false, false>(B, "C2 f32 wave 448 pf, no sync (wrong)");

  }
  if (which != 1) {
    Bench<double> B(256, 256, 256, zch);
    run_ref<double, 2, true>(B, "C2 f64 k_pull2 16x8 PF trim (product)");

  }
  return 0;
}
