// tb_tma.cu — scratch A/B microbenchmark (not product code): the two-step sweep with the
// register prefetch (k_pull2) against the TMA-staged sweep (k_pull2_tma, 1 or 2 stages, tile
// variants) on C2-like (D3Q19 raw zc+delta 256^3, fp64 / fp32) and C4-like (D3Q27 cumulant
// zc+abs 512^2 x 128) lattices: time per two steps and max |difference| of the outputs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr
//        -I paper_2211_02435_b200/csrc -I include -I scripts scripts/tb_tma.cu -o scripts/tb_tma
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "kernels.cuh"
#include "tb_r2_variants.cuh"

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
__global__ void fill_noise(real *a, size_t n, int q, long long pop, real amp) {
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

struct Lat {
  GridParams g{};
  size_t elems;
  int planes;
};

template <class S, class real>
Lat make_lat(int nx, int ny, int nz) {
  Lat L;
  L.g.nx = nx;
  L.g.ny = ny;
  L.g.nzl = L.g.nzg = nz;
  L.g.pitch = nx;
  L.g.pop = (long long)ny * nx;
  L.g.plane = (long long)S::Q * L.g.pop;
  L.g.wrapz = 1;
  L.planes = nz + 2;
  L.elems = (size_t)L.planes * L.g.plane;
  return L;
}

template <class S, int SPACE, int REG, class real, int TX, int TY, int MINB, int STAGES>
void run_tma(const char *name, const Lat &L, real *a, real *b, real *ref, const Rates<real> &r, int zch,
             double cells) {
  using T = TmaTile<S, real, TX, TY, STAGES>;
  auto kern = k_pull2_tma<S, SPACE, REG, real, RS_GENERAL, TX, TY, MINB, false, STAGES>;
  const size_t smem = T::SMEM;
  if (smem > 227 * 1024) {
    printf("%-44s smem %zu too large\n", name, smem);
    return;
  }
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CUtensorMap ma, mb;
  CK(encode_grid_tmap<real>(&ma, a, L.g.nx, L.g.ny, S::Q, L.planes, L.g.pitch, L.g.pop, L.g.plane, T::BX, T::HY));
  CK(encode_grid_tmap<real>(&mb, b, L.g.nx, L.g.ny, S::Q, L.planes, L.g.pitch, L.g.pop, L.g.plane, T::BX, T::HY));
  Force<real> fr{};
  dim3 grid((unsigned)(L.g.nx / TX), (unsigned)(L.g.ny / TY), (unsigned)zch);
  // correctness: one launch from a into b, compare with the reference output
  kern<<<grid, T::THREADS, smem>>>(a, b, L.g, r, real(0), fr, ma);
  CK(cudaDeviceSynchronize());
  double *dm;
  CK(cudaMalloc(&dm, 8));
  CK(cudaMemset(dm, 0, 8));
  // compare the interior planes only (ghost planes are untouched by both)
  maxdiff<<<1184, 256>>>(b + L.g.plane, ref + L.g.plane, (size_t)L.g.nzl * L.g.plane, dm);
  double md = 0;
  CK(cudaMemcpy(&md, dm, 8, cudaMemcpyDeviceToHost));
  cudaFree(dm);
  int nb = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, T::THREADS, smem));
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, kern));
  // restore a for timing: the timing loop ping-pongs a <-> b
  float ms = time_k([&](int p) {
    kern<<<grid, T::THREADS, smem>>>(p ? b : a, p ? a : b, L.g, r, real(0), fr, p ? mb : ma);
  });
  printf("%-44s %7.3f ms/2 steps %8.0f MLUPS  regs %3d  smem %6zu  %d CTA/SM  maxdiff %.3e\n", name, ms,
         2.0 * cells / (ms * 1e-3) / 1e6, fa.numRegs, smem, nb, md);
}

template <class S, int SPACE, int REG, class real, int TX, int TY, int MINB>
void run_ref(const char *name, const Lat &L, real *a, real *b, real *ref, const Rates<real> &r, int zch, double cells) {
  using T = Tile2<TX, TY>;
  auto kern = k_pull2<S, SPACE, REG, real, RS_GENERAL, TX, TY, MINB, true>;
  const size_t smem = (size_t)3 * S::Q * T::HW * sizeof(real);
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  Force<real> fr{};
  dim3 grid((unsigned)(L.g.nx / TX), (unsigned)(L.g.ny / TY), (unsigned)zch);
  kern<<<grid, T::THREADS, smem>>>(a, ref, L.g, r, real(0), fr);
  CK(cudaDeviceSynchronize());
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, kern));
  float ms = time_k([&](int p) { kern<<<grid, T::THREADS, smem>>>(p ? b : a, p ? a : b, L.g, r, real(0), fr); });
  // the timing loop overwrote a; regenerate the input and the reference
  printf("%-44s %7.3f ms/2 steps %8.0f MLUPS  regs %3d  smem %6zu\n", name, ms, 2.0 * cells / (ms * 1e-3) / 1e6,
         fa.numRegs, smem);
}

template <class S, int SPACE, int REG, class real, int TX, int TY, int MINB, bool PF>
void run_trim(const char *name, const Lat &L, real *a, real *b, real *ref, const Rates<real> &r, int zch,
              double cells) {
  using T = Tile2<TX, TY>;
  auto kern = k_pull2<S, SPACE, REG, real, RS_GENERAL, TX, TY, MINB, PF, false, true>;
  const size_t smem = (size_t)Tile2Trim<TX, TY, S>::RING * sizeof(real);
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  Force<real> fr{};
  dim3 grid((unsigned)(L.g.nx / TX), (unsigned)(L.g.ny / TY), (unsigned)zch);
  kern<<<grid, T::THREADS, smem>>>(a, b, L.g, r, real(0), fr);
  CK(cudaDeviceSynchronize());
  double *dm;
  CK(cudaMalloc(&dm, 8));
  CK(cudaMemset(dm, 0, 8));
  maxdiff<<<1184, 256>>>(b + L.g.plane, ref + L.g.plane, (size_t)L.g.nzl * L.g.plane, dm);
  double md = 0;
  CK(cudaMemcpy(&md, dm, 8, cudaMemcpyDeviceToHost));
  cudaFree(dm);
  int nb = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, T::THREADS, smem));
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, kern));
  float ms = time_k([&](int p) { kern<<<grid, T::THREADS, smem>>>(p ? b : a, p ? a : b, L.g, r, real(0), fr); });
  printf("%-44s %7.3f ms/2 steps %8.0f MLUPS  regs %3d  lmem %3zu  smem %6zu  %d CTA/SM  maxdiff %.3e\n", name, ms,
         2.0 * cells / (ms * 1e-3) / 1e6, fa.numRegs, fa.localSizeBytes, smem, nb, md);
}

template <class S, int SPACE, int REG, class real, int TX, int TY, int MINB>
void run_1b(const char *name, const Lat &L, real *a, real *b, real *ref, const Rates<real> &r, int zch,
            double cells) {
  using T = Tile2<TX, TY>;
  auto kern = k_pull2_1b<S, SPACE, REG, real, RS_GENERAL, TX, TY, MINB, false>;
  const size_t smem = (size_t)Tile2Ring1b<TX, TY, S>::RING * sizeof(real);
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  Force<real> fr{};
  dim3 grid((unsigned)(L.g.nx / TX), (unsigned)(L.g.ny / TY), (unsigned)zch);
  kern<<<grid, T::THREADS, smem>>>(a, b, L.g, r, real(0), fr);
  CK(cudaDeviceSynchronize());
  double *dm;
  CK(cudaMalloc(&dm, 8));
  CK(cudaMemset(dm, 0, 8));
  maxdiff<<<1184, 256>>>(b + L.g.plane, ref + L.g.plane, (size_t)L.g.nzl * L.g.plane, dm);
  double md = 0;
  CK(cudaMemcpy(&md, dm, 8, cudaMemcpyDeviceToHost));
  cudaFree(dm);
  int nb = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, T::THREADS, smem));
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, kern));
  float ms = time_k([&](int p) { kern<<<grid, T::THREADS, smem>>>(p ? b : a, p ? a : b, L.g, r, real(0), fr); });
  printf("%-44s %7.3f ms/2 steps %8.0f MLUPS  regs %3d  lmem %3zu  smem %6zu  %d CTA/SM  maxdiff %.3e\n", name, ms,
         2.0 * cells / (ms * 1e-3) / 1e6, fa.numRegs, fa.localSizeBytes, smem, nb, md);
}

template <class S, int SPACE, int REG, class real, int TX, int TY, int MINB>
void run_ws(const char *name, const Lat &L, real *a, real *b, real *ref, const Rates<real> &r, int zch,
            double cells) {
  using T = TileWs<TX, TY>;
  auto kern = k_pull2_ws<S, SPACE, REG, real, RS_GENERAL, TX, TY, MINB, false>;
  const size_t smem = ws_smem_bytes<S, real, TX, TY>();
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  Force<real> fr{};
  dim3 grid((unsigned)(L.g.nx / TX), (unsigned)(L.g.ny / TY), (unsigned)zch);
  kern<<<grid, T::THREADS, smem>>>(a, b, L.g, r, real(0), fr);
  CK(cudaDeviceSynchronize());
  double *dm;
  CK(cudaMalloc(&dm, 8));
  CK(cudaMemset(dm, 0, 8));
  maxdiff<<<1184, 256>>>(b + L.g.plane, ref + L.g.plane, (size_t)L.g.nzl * L.g.plane, dm);
  double md = 0;
  CK(cudaMemcpy(&md, dm, 8, cudaMemcpyDeviceToHost));
  cudaFree(dm);
  int nb = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, T::THREADS, smem));
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, kern));
  float ms = time_k([&](int p) { kern<<<grid, T::THREADS, smem>>>(p ? b : a, p ? a : b, L.g, r, real(0), fr); });
  printf("%-44s %7.3f ms/2 steps %8.0f MLUPS  regs %3d  lmem %3zu  smem %6zu  %d CTA/SM  maxdiff %.3e\n", name, ms,
         2.0 * cells / (ms * 1e-3) / 1e6, fa.numRegs, fa.localSizeBytes, smem, nb, md);
}

template <class S, int SPACE, int REG, class real>
struct Bench {
  Lat L;
  real *a, *b, *ref;
  Rates<real> r;
  double cells;
  Bench(int nx, int ny, int nz) {
    L = make_lat<S, real>(nx, ny, nz);
    CK(cudaMalloc(&a, L.elems * sizeof(real)));
    CK(cudaMalloc(&b, L.elems * sizeof(real)));
    CK(cudaMalloc(&ref, L.elems * sizeof(real)));
    for (int i = 0; i < 27; ++i) r.w[i] = real(1.0 + 0.02 * i);
    cells = (double)nx * ny * nz;
  }
  ~Bench() {
    cudaFree(a);
    cudaFree(b);
    cudaFree(ref);
  }
  void reset() {
    // zero-centered deviations: small noise (absolute regimes see f0 + noise through the kernel)
    fill_noise<<<1184, 256>>>(a, L.elems, S::Q, L.g.pop, real(1e-3));
    CK(cudaMemset(b, 0, L.elems * sizeof(real)));
    CK(cudaDeviceSynchronize());
  }
};

template <class real, int MINB_REF>
void c2(const char *tag, bool tma) {
  using S = D3Q19;
  Bench<S, SPACE_RAW, REG_DELTA, real> B(256, 256, 256);
  char nm[128];
  const int zch = 3;
  B.reset();
  snprintf(nm, sizeof nm, "C2 %s k_pull2 16x8 PF (product)", tag);
  run_ref<S, SPACE_RAW, REG_DELTA, real, 16, 8, MINB_REF>(nm, B.L, B.a, B.b, B.ref, B.r, zch, B.cells);
#define TMA(TX, TY, MINB, ST)                                                                          \
  B.reset();                                                                                           \
  /* reference output of this input */                                                                 \
  {                                                                                                    \
    using T2 = Tile2<16, 8>;                                                                           \
    auto kr = k_pull2<S, SPACE_RAW, REG_DELTA, real, RS_GENERAL, 16, 8, MINB_REF, true>;               \
    Force<real> fr{};                                                                                  \
    kr<<<dim3(256 / 16, 256 / 8, zch), T2::THREADS, (size_t)3 * S::Q * T2::HW * sizeof(real)>>>(      \
        B.a, B.ref, B.L.g, B.r, real(0), fr);                                                          \
    CK(cudaDeviceSynchronize());                                                                       \
  }                                                                                                    \
  snprintf(nm, sizeof nm, "C2 %s tma %dx%d minb %d stages %d", tag, TX, TY, MINB, ST);                 \
  run_tma<S, SPACE_RAW, REG_DELTA, real, TX, TY, MINB, ST>(nm, B.L, B.a, B.b, B.ref, B.r, zch, B.cells);
  if (tma) {
    TMA(16, 8, 2, 1)
    TMA(16, 8, 2, 2)
    TMA(16, 8, 3, 1)
    TMA(32, 8, 1, 1)
    TMA(32, 8, 1, 2)
    TMA(16, 16, 1, 1)
    TMA(32, 4, 2, 1)
  }
#undef TMA
  if (getenv("TB_TRIM")) {
#define TRIMV(TX, TY, MINB, PF)                                                                        \
  B.reset();                                                                                           \
  {                                                                                                    \
    using T2 = Tile2<16, 8>;                                                                           \
    auto kr = k_pull2<S, SPACE_RAW, REG_DELTA, real, RS_GENERAL, 16, 8, MINB_REF, true>;               \
    Force<real> fr{};                                                                                  \
    kr<<<dim3(256 / 16, 256 / 8, zch), T2::THREADS, (size_t)3 * S::Q * T2::HW * sizeof(real)>>>(      \
        B.a, B.ref, B.L.g, B.r, real(0), fr);                                                          \
    CK(cudaDeviceSynchronize());                                                                       \
  }                                                                                                    \
  snprintf(nm, sizeof nm, "C2 %s trim %dx%d minb %d pf %d", tag, TX, TY, MINB, (int)PF);              \
  run_trim<S, SPACE_RAW, REG_DELTA, real, TX, TY, MINB, PF>(nm, B.L, B.a, B.b, B.ref, B.r, zch, B.cells);
  TRIMV(16, 8, MINB_REF, true)
  TRIMV(16, 8, MINB_REF + 1, true)
  TRIMV(16, 8, MINB_REF + 1, false)
  TRIMV(16, 12, MINB_REF, true)
  TRIMV(16, 12, MINB_REF, false)
  TRIMV(32, 8, 1, true)
  TRIMV(32, 8, 2, false)
  TRIMV(16, 16, 2, false)
  TRIMV(16, 16, 1, true)
#undef TRIMV
  }
#define WSV(TX, TY, MINB)                                                                              \
  B.reset();                                                                                           \
  {                                                                                                    \
    using T2 = Tile2<16, 8>;                                                                           \
    auto kr = k_pull2<S, SPACE_RAW, REG_DELTA, real, RS_GENERAL, 16, 8, MINB_REF, true>;               \
    Force<real> fr{};                                                                                  \
    kr<<<dim3(256 / 16, 256 / 8, zch), T2::THREADS, (size_t)3 * S::Q * T2::HW * sizeof(real)>>>(      \
        B.a, B.ref, B.L.g, B.r, real(0), fr);                                                          \
    CK(cudaDeviceSynchronize());                                                                       \
  }                                                                                                    \
  snprintf(nm, sizeof nm, "C2 %s ws %dx%d minb %d", tag, TX, TY, MINB);                               \
  run_ws<S, SPACE_RAW, REG_DELTA, real, TX, TY, MINB>(nm, B.L, B.a, B.b, B.ref, B.r, zch, B.cells);
  if (getenv("TB_WS")) {
    WSV(16, 8, 1)
    WSV(16, 8, 2)
    WSV(16, 8, 3)
    WSV(32, 8, 1)
    WSV(32, 4, 2)
    WSV(16, 16, 1)
    WSV(8, 8, 3)
  }
#undef WSV
#define V1B(TX, TY, MINB)                                                                              \
  B.reset();                                                                                           \
  {                                                                                                    \
    using T2 = Tile2<16, 8>;                                                                           \
    auto kr = k_pull2<S, SPACE_RAW, REG_DELTA, real, RS_GENERAL, 16, 8, MINB_REF, true>;               \
    Force<real> fr{};                                                                                  \
    kr<<<dim3(256 / 16, 256 / 8, zch), T2::THREADS, (size_t)3 * S::Q * T2::HW * sizeof(real)>>>(      \
        B.a, B.ref, B.L.g, B.r, real(0), fr);                                                          \
    CK(cudaDeviceSynchronize());                                                                       \
  }                                                                                                    \
  snprintf(nm, sizeof nm, "C2 %s 1b %dx%d minb %d", tag, TX, TY, MINB);                               \
  run_1b<S, SPACE_RAW, REG_DELTA, real, TX, TY, MINB>(nm, B.L, B.a, B.b, B.ref, B.r, zch, B.cells);
  V1B(16, 8, MINB_REF)
  V1B(16, 8, MINB_REF + 1)
  V1B(16, 8, 1)
  V1B(32, 8, 1)
  V1B(32, 4, MINB_REF)
  V1B(16, 16, 1)
#undef V1B
}

void c4() {
  using S = D3Q27;
  using real = double;
  Bench<S, SPACE_CUMULANT, REG_ZC_ABS, real> B(512, 512, 128);
  char nm[128];
  const int zch = 2;
#define TMA4(TX, TY, MINB, ST)                                                                          \
  B.reset();                                                                                            \
  {                                                                                                     \
    using T2 = Tile2<16, 8>;                                                                            \
    auto kr = k_pull2<S, SPACE_CUMULANT, REG_ZC_ABS, real, RS_GENERAL, 16, 8, 1, true>;                 \
    const size_t sm = (size_t)3 * S::Q * T2::HW * sizeof(real);                                         \
    CK(cudaFuncSetAttribute(kr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));                 \
    Force<real> fr{};                                                                                   \
    kr<<<dim3(512 / 16, 512 / 8, zch), T2::THREADS, sm>>>(B.a, B.ref, B.L.g, B.r, real(0), fr);         \
    CK(cudaDeviceSynchronize());                                                                        \
  }                                                                                                     \
  snprintf(nm, sizeof nm, "C4 cumulant tma %dx%d minb %d stages %d", TX, TY, MINB, ST);                 \
  run_tma<S, SPACE_CUMULANT, REG_ZC_ABS, real, TX, TY, MINB, ST>(nm, B.L, B.a, B.b, B.ref, B.r, zch, B.cells);
  B.reset();
  run_ref<S, SPACE_CUMULANT, REG_ZC_ABS, real, 16, 8, 1>("C4 cumulant k_pull2 16x8 PF", B.L, B.a, B.b, B.ref, B.r, zch,
                                                         B.cells);
  if (getenv("TB_TMA")) {
    TMA4(16, 8, 1, 1)
    TMA4(16, 8, 1, 2)
    TMA4(8, 8, 2, 1)
    TMA4(16, 4, 2, 1)
    TMA4(32, 8, 1, 1)
  }
#undef TMA4
#define TRIM4(TX, TY, MINB, PF)                                                                         \
  B.reset();                                                                                            \
  {                                                                                                     \
    using T2 = Tile2<16, 8>;                                                                            \
    auto kr = k_pull2<S, SPACE_CUMULANT, REG_ZC_ABS, real, RS_GENERAL, 16, 8, 1, true>;                 \
    const size_t sm = (size_t)3 * S::Q * T2::HW * sizeof(real);                                         \
    CK(cudaFuncSetAttribute(kr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));                 \
    Force<real> fr{};                                                                                   \
    kr<<<dim3(512 / 16, 512 / 8, zch), T2::THREADS, sm>>>(B.a, B.ref, B.L.g, B.r, real(0), fr);         \
    CK(cudaDeviceSynchronize());                                                                        \
  }                                                                                                     \
  snprintf(nm, sizeof nm, "C4 cumulant trim %dx%d minb %d pf %d", TX, TY, MINB, (int)PF);              \
  run_trim<S, SPACE_CUMULANT, REG_ZC_ABS, real, TX, TY, MINB, PF>(nm, B.L, B.a, B.b, B.ref, B.r, zch, B.cells);
  if (getenv("TB_TRIM") && 0) {
    TRIM4(16, 8, 1, true)
    TRIM4(16, 8, 1, false)
    TRIM4(16, 8, 2, false)
    TRIM4(32, 8, 1, false)
    TRIM4(16, 16, 1, false)
    TRIM4(32, 4, 1, false)
  }
#undef TRIM4
#define WS4(TX, TY, MINB)                                                                               \
  B.reset();                                                                                            \
  {                                                                                                     \
    using T2 = Tile2<16, 8>;                                                                            \
    auto kr = k_pull2<S, SPACE_CUMULANT, REG_ZC_ABS, real, RS_GENERAL, 16, 8, 1, true>;                 \
    const size_t sm = (size_t)3 * S::Q * T2::HW * sizeof(real);                                         \
    CK(cudaFuncSetAttribute(kr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));                 \
    Force<real> fr{};                                                                                   \
    kr<<<dim3(512 / 16, 512 / 8, zch), T2::THREADS, sm>>>(B.a, B.ref, B.L.g, B.r, real(0), fr);         \
    CK(cudaDeviceSynchronize());                                                                        \
  }                                                                                                     \
  snprintf(nm, sizeof nm, "C4 cumulant ws %dx%d minb %d", TX, TY, MINB);                                \
  run_ws<S, SPACE_CUMULANT, REG_ZC_ABS, real, TX, TY, MINB>(nm, B.L, B.a, B.b, B.ref, B.r, zch, B.cells);
  if (getenv("TB_WS")) {
    WS4(16, 8, 1)
    WS4(8, 8, 2)
    WS4(16, 4, 2)
    WS4(32, 4, 1)
  }
#undef WS4
#define V1B4(TX, TY, MINB)                                                                              \
  B.reset();                                                                                            \
  {                                                                                                     \
    using T2 = Tile2<16, 8>;                                                                            \
    auto kr = k_pull2<S, SPACE_CUMULANT, REG_ZC_ABS, real, RS_GENERAL, 16, 8, 1, true>;                 \
    const size_t sm = (size_t)3 * S::Q * T2::HW * sizeof(real);                                         \
    CK(cudaFuncSetAttribute(kr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));                 \
    Force<real> fr{};                                                                                   \
    kr<<<dim3(512 / 16, 512 / 8, zch), T2::THREADS, sm>>>(B.a, B.ref, B.L.g, B.r, real(0), fr);         \
    CK(cudaDeviceSynchronize());                                                                        \
  }                                                                                                     \
  snprintf(nm, sizeof nm, "C4 cumulant 1b %dx%d minb %d", TX, TY, MINB);                                \
  run_1b<S, SPACE_CUMULANT, REG_ZC_ABS, real, TX, TY, MINB>(nm, B.L, B.a, B.b, B.ref, B.r, zch, B.cells);
  V1B4(16, 8, 1)
  V1B4(32, 8, 1)
  V1B4(16, 4, 1)
#undef V1B4
}

int main(int argc, char **argv) {
  const int which = argc > 1 ? atoi(argv[1]) : 7;
  if (which & 1) c2<double, 2>("f64", which & 8);
  if (which & 2) c2<float, 3>("f32", which & 8);
  if (which & 4) c4();
  return 0;
}
