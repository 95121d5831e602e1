// ops.cuh — type-erased launchers of one (stencil, space, regime, precision)
// instantiation.  Each instantiation lives in its own translation unit
// (ops_inst.cu compiled once per stencil / precision / space) so that the
// heavy D3Q27 cumulant kernels compile in parallel.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>

#include "kernels.cuh"

namespace lbm {

// Method parameters of the collision, in the storage precision (host blob, copied into
// the kernel parameters at launch).
template <class real>
struct MethodParams {
  Rates<real> rates;
  Force<real> force;  // used by the RS_FORCE instantiations only
};

struct Ops {
  int q, d;
  // pull stream–collide of planes [zbegin, zbegin + nplanes) from src into dst
  void (*pull)(const void *src, void *dst, const GridParams &g, const void *params, double swe_g, int bb,
               int nplanes, cudaStream_t s);
  // in-place step (PAT_AA_EVEN / PAT_AA_ODD / PAT_ESO_EVEN / PAT_ESO_ODD / PAT_ESOP_EVEN /
  // PAT_ESOP_ODD / PAT_TW0 / PAT_TW1),
  // planes [zbegin, zbegin + nplanes)
  void (*aa)(void *mem, const GridParams &g, const void *params, double swe_g, int pattern, int nplanes,
             cudaStream_t s);
  void (*init)(void *mem, const GridParams &g, int aa, const double *rho, const double *u, double swe_g,
               cudaStream_t s);
  void (*get_pop)(const void *mem, const GridParams &g, int aa, int state, double *out, cudaStream_t s);
  void (*set_pop)(void *mem, const GridParams &g, int aa, const double *in, cudaStream_t s);
  // dj: momentum correction of the post-collision state (-F/2 with a body force)
  void (*macro)(const void *mem, const GridParams &g, int aa, int state, int zc, double *rho, double *u,
                double3 dj, cudaStream_t s);
  void (*test_collide)(const double *fin, double *fout, long long n, const void *params, double swe_g,
                       cudaStream_t s);
  void (*check_finite)(const void *mem, const GridParams &g, int *flag, cudaStream_t s);
  void (*get_cells)(const void *mem, const GridParams &g, int aa, int state, const long long *idx, long long n,
                    double *out, cudaStream_t s);
  // global sums (mass, momentum, kinetic energy): partial[5 * DIAG_GRID] scratch, out[5]
  void (*diagnostics)(const void *mem, const GridParams &g, int aa, int state, int zc, double *partial,
                      double *out, double3 dj, cudaStream_t s);
  // registers / local memory of a kernel of this instantiation, for diagnostics: which = 0
  // k_pull, 1 the two-step sweep (k_pull2 / k_pull2_2d), 2 the cluster-resident loop, 3 the
  // depth-3 2D sweep (k_pullD_2d),
  // 10 + pattern the in-place kernel of that pattern (PAT_AA_ODD, PAT_ESO_ODD, PAT_TW0, ...)
  void (*attributes)(int which, int *regs, int *local_bytes);
  // two fused pull steps (temporal blocking; 3D, single rank, periodic); tile TX x TY
  // (0 x 0: not provided).  Requires nx % TX == 0 and ny % TY == 0.
  void (*pull2)(const void *src, void *dst, const GridParams &g, const void *params, double swe_g, int zchunks,
                cudaStream_t s);
  int tile_x, tile_y;
  // n pull steps of a small 2D lattice in one launch of a `cluster`-CTA thread-block cluster
  // with the lattice resident in shared memory (k_resident2); returns the launch's cudaError_t
  // (nullptr for 3D stencils)
  int (*resident)(const void *src, void *dst, const GridParams &g, const void *params, double swe_g, int bb,
                  int nsteps, int cluster, cudaStream_t s);
  // loads every kernel the multi-rank step paths of this instantiation launch (CUDA lazy
  // loading would otherwise load a kernel at its first launch, which waits for the kernels
  // running on the device — among them a spinning k_peer_wait whose release may depend on that
  // very launch: contexts of one process sharing a device would stall until the wait times out)
  void (*preload)();
  // uploads the WO-MRT basis matrices (27 x 27, monomial cube coordinates) to this
  // instantiation's constant memory on the current device (RS_WOBASIS kernels)
  int (*set_wo)(const double *L, const double *Linv);
  // three fused pull steps (2D only: k_pullD_2d, depth 3, 256-cell strips; single rank,
  // periodic; nx % 256 == 0); nullptr for 3D stencils
  void (*pull3)(const void *src, void *dst, const GridParams &g, const void *params, double swe_g, int zchunks,
                cudaStream_t s);
};

// shared memory of k_resident2: two grids [Q][R + 2][nx]
inline size_t resident_smem(int q, int nx, int rows, int esize) {
  return (size_t)2 * q * (size_t)(rows + 2) * nx * esize;
}

// Temporal-blocking tile of k_pull2 / k_pull2_2d, measured on B200 (scripts/tb_variants.cu,
// scripts/tb2d_variants.cu; profiles/r1/tb_variants*.txt, tb2d_variants.txt), 1024^2 x 128 and
// 8192^2, time per 2 steps against two single k_pull steps:
//   D3Q19 fp64: 16 x 8, 2 CTAs/SM, next plane's loads prefetched: raw 9.3 vs 12.2 ms,
//               cumulant 10.3 vs 12.2 ms;
//   D3Q19 fp32: 16 x 8, 3 CTAs/SM, prefetched: 4.96 vs 6.16 ms;
//   D3Q27 fp64 raw / SRT: 16 x 8, 1 CTA/SM, prefetched: raw 14.0 vs 17.3 ms;
//   D3Q27 central: 17.1 vs 17.4 (not used), cumulant: 20.4 vs 17.4 (not used) — 27 fp64
//               populations per halo cell leave shared memory for too few warps to hide the
//               heavier collisions;
//   D2Q9: 256-cell strips (k_pull2_2d), 2-3 CTAs/SM.
// The runtime also requires >= 4 waves of CTAs.
template <class S, class real, int SPACE>
struct TbTile {
  static constexpr bool f64 = sizeof(real) == 8;
  static constexpr bool on3 = (S::Q == 19) || (S::Q == 27 && f64 && (SPACE == SPACE_RAW || SPACE == SPACE_POPULATION));
  static constexpr bool on = on3 || S::D == 2;
  static constexpr int TX = S::D == 2 ? 256 : (on3 ? 16 : 0);
  static constexpr int TY = S::D == 2 ? 1 : (on3 ? 8 : 0);
  static constexpr int MINB = S::Q == 27 ? 1 : (f64 ? 2 : 3);  // 3D: CTAs per SM
  // trimmed step-(t+1) ring (3 / 2 / 1 planes of the xi_z = +1 / 0 / -1 populations): D3Q19
  // fp64 C2 1.188 -> 1.108 ms per 2 steps (the freed shared memory goes to L1, which serves the
  // halo re-reads); fp32 and D3Q27 unchanged (scripts/tb_tma.cu, profiles/r2/tb_variants_r2.txt)
  static constexpr bool TRIM = S::Q == 19 && f64;
};

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel instantiation, device):
// `configured` is a static of the calling launcher (one per instantiation), bit d = device d
// (benign race: setting the attribute twice is harmless)
template <class K>
inline void opt_in_smem_once(K kern, size_t smem, unsigned &configured) {
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned bit = dev < 32 ? (1u << dev) : 0u;
  if (bit && (configured & bit)) return;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  configured |= bit;
}

inline dim3 cell_grid(const GridParams &g, int nplanes) {
  return dim3((unsigned)((g.nx + BLOCK_X - 1) / BLOCK_X), (unsigned)g.ny, (unsigned)nplanes);
}

template <class S, int SPACE, int REG, class real, int RS = RS_GENERAL>
struct OpsImpl {
  static void pull(const void *src, void *dst, const GridParams &g, const void *params, double swe_g, int bb,
                   int nplanes, cudaStream_t s) {
    if (nplanes <= 0) return;
    const MethodParams<real> &p = *static_cast<const MethodParams<real> *>(params);
    if ((g.peer_lo || g.peer_hi) && bb)  // boundary planes of lbm_step_peer
      k_pull<S, SPACE, REG, real, true, RS, true><<<cell_grid(g, nplanes), BLOCK_X, 0, s>>>(
          static_cast<const real *>(src), static_cast<real *>(dst), g, p.rates, (real)swe_g, p.force);
    else if (g.peer_lo || g.peer_hi)
      k_pull<S, SPACE, REG, real, false, RS, true><<<cell_grid(g, nplanes), BLOCK_X, 0, s>>>(
          static_cast<const real *>(src), static_cast<real *>(dst), g, p.rates, (real)swe_g, p.force);
    else if (bb)
      k_pull<S, SPACE, REG, real, true, RS><<<cell_grid(g, nplanes), BLOCK_X, 0, s>>>(
          static_cast<const real *>(src), static_cast<real *>(dst), g, p.rates, (real)swe_g, p.force);
    else
      k_pull<S, SPACE, REG, real, false, RS><<<cell_grid(g, nplanes), BLOCK_X, 0, s>>>(
          static_cast<const real *>(src), static_cast<real *>(dst), g, p.rates, (real)swe_g, p.force);
  }
  static void aa(void *mem, const GridParams &g, const void *params, double swe_g, int pattern, int nplanes,
                 cudaStream_t s) {
    if (nplanes <= 0) return;
    const MethodParams<real> &p = *static_cast<const MethodParams<real> *>(params);
    real *m = static_cast<real *>(mem);
    switch (pattern) {
      case PAT_AA_EVEN:
        k_aa<S, SPACE, REG, real, PAT_AA_EVEN, RS><<<cell_grid(g, nplanes), BLOCK_X, 0, s>>>(m, g, p.rates,
                                                                                          (real)swe_g, p.force);
        break;
      case PAT_AA_ODD:
        if (g.peer_lo && g.peer_hi)  // boundary planes of lbm_step_peer
          k_aa<S, SPACE, REG, real, PAT_AA_ODD, RS, true><<<cell_grid(g, nplanes), BLOCK_X, 0, s>>>(
              m, g, p.rates, (real)swe_g, p.force);
        else if (g.bcmask)  // no-slip faces (single rank): half-way bounce-back
          k_aa<S, SPACE, REG, real, PAT_AA_ODD, RS, false, true><<<cell_grid(g, nplanes), BLOCK_X, 0, s>>>(
              m, g, p.rates, (real)swe_g, p.force);
        else
          k_aa<S, SPACE, REG, real, PAT_AA_ODD, RS><<<cell_grid(g, nplanes), BLOCK_X, 0, s>>>(m, g, p.rates,
                                                                                           (real)swe_g, p.force);
        break;
      case PAT_ESO_EVEN:
        k_eso<S, SPACE, REG, real, PAT_ESO_EVEN, RS><<<cell_grid(g, nplanes), BLOCK_X, 0, s>>>(m, g, p.rates,
                                                                                            (real)swe_g, p.force);
        break;
      case PAT_ESOP_EVEN:
        k_eso<S, SPACE, REG, real, PAT_ESOP_EVEN, RS><<<cell_grid(g, nplanes), BLOCK_X, 0, s>>>(m, g, p.rates,
                                                                                             (real)swe_g, p.force);
        break;
      case PAT_ESOP_ODD:
        k_eso<S, SPACE, REG, real, PAT_ESOP_ODD, RS><<<cell_grid(g, nplanes), BLOCK_X, 0, s>>>(m, g, p.rates,
                                                                                            (real)swe_g, p.force);
        break;
      case PAT_TW0:
        k_twist<S, SPACE, REG, real, PAT_TW0, RS><<<cell_grid(g, nplanes), BLOCK_X, 0, s>>>(m, g, p.rates,
                                                                                         (real)swe_g, p.force);
        break;
      case PAT_TW1:
        k_twist<S, SPACE, REG, real, PAT_TW1, RS><<<cell_grid(g, nplanes), BLOCK_X, 0, s>>>(m, g, p.rates,
                                                                                         (real)swe_g, p.force);
        break;
      default:
        k_eso<S, SPACE, REG, real, PAT_ESO_ODD, RS><<<cell_grid(g, nplanes), BLOCK_X, 0, s>>>(m, g, p.rates,
                                                                                           (real)swe_g, p.force);
        break;
    }
  }
  static void init(void *mem, const GridParams &g, int aa, const double *rho, const double *u, double swe_g,
                   cudaStream_t s) {
    k_init<S, SPACE, REG, real, (RS & RS_DISCRETE) != 0><<<cell_grid(g, g.nzl), BLOCK_X, 0, s>>>(static_cast<real *>(mem), g, aa, rho, u,
                                                                        (real)swe_g);
  }
  static void get_pop(const void *mem, const GridParams &g, int aa, int state, double *out, cudaStream_t s) {
    k_get_populations<S, real><<<cell_grid(g, g.nzl), BLOCK_X, 0, s>>>(static_cast<const real *>(mem), g, aa,
                                                                       state, out);
  }
  static void set_pop(void *mem, const GridParams &g, int aa, const double *in, cudaStream_t s) {
    k_set_populations<S, real><<<cell_grid(g, g.nzl), BLOCK_X, 0, s>>>(static_cast<real *>(mem), g, aa, in);
  }
  static void macro(const void *mem, const GridParams &g, int aa, int state, int zc, double *rho, double *u,
                    double3 dj, cudaStream_t s) {
    k_macroscopic<S, real><<<cell_grid(g, g.nzl), BLOCK_X, 0, s>>>(static_cast<const real *>(mem), g, aa, state,
                                                                   zc, rho, u, dj);
  }
  static void test_collide(const double *fin, double *fout, long long n, const void *params, double swe_g,
                           cudaStream_t s) {
    if (n <= 0) return;
    const MethodParams<real> &p = *static_cast<const MethodParams<real> *>(params);
    const int B = 128;
    k_test_collide<S, SPACE, REG, real, RS><<<(unsigned)((n + B - 1) / B), B, 0, s>>>(fin, fout, n, p.rates,
                                                                                     (real)swe_g, p.force);
  }
  static void check_finite(const void *mem, const GridParams &g, int *flag, cudaStream_t s) {
    k_check_finite<S, real><<<cell_grid(g, g.nzl), BLOCK_X, 0, s>>>(static_cast<const real *>(mem), g, flag);
  }
  static void get_cells(const void *mem, const GridParams &g, int aa, int state, const long long *idx, long long n,
                        double *out, cudaStream_t s) {
    if (n <= 0) return;
    k_get_cells<S, real><<<(unsigned)((n + 127) / 128), 128, 0, s>>>(static_cast<const real *>(mem), g, aa, state,
                                                                      idx, n, out);
  }
  static void diagnostics(const void *mem, const GridParams &g, int aa, int state, int zc, double *partial,
                          double *out, double3 dj, cudaStream_t s) {
    k_diag_partial<S, real><<<DIAG_GRID, DIAG_BLOCK, 0, s>>>(static_cast<const real *>(mem), g, aa, state, zc,
                                                             partial, dj);
    k_diag_final<double><<<1, DIAG_BLOCK, 0, s>>>(partial, out);
  }
  static void pull2(const void *src, void *dst, const GridParams &g, const void *params, double swe_g,
                    int zchunks, cudaStream_t s) {
    using TT = TbTile<S, real, SPACE>;
    constexpr int TX = TT::TX, TY = TT::TY;
    if constexpr (S::D == 3 && TX > 0) {
      using T = Tile2<TX, TY>;
      const MethodParams<real> &p = *static_cast<const MethodParams<real> *>(params);
      const size_t smem = (TT::TRIM ? (size_t)Tile2Trim<TX, TY, S>::RING : (size_t)3 * S::Q * T::HW) * sizeof(real);
      // whole slab with periodic wrap (single rank) or a plane range without wrap (across ranks)
      auto go = [&](auto kern, unsigned &configured) {
        opt_in_smem_once(kern, smem, configured);  // > 48 KB of shared memory, once per device
        kern<<<dim3((unsigned)(g.nx / TX), (unsigned)(g.ny / TY), (unsigned)zchunks), T::THREADS, smem, s>>>(
            static_cast<const real *>(src), static_cast<real *>(dst), g, p.rates, (real)swe_g, p.force);
      };
      static unsigned conf_slab = 0, conf_range = 0;
      if (g.zcount) go(k_pull2<S, SPACE, REG, real, RS, TX, TY, TT::MINB, true, true, TT::TRIM>, conf_range);
      else go(k_pull2<S, SPACE, REG, real, RS, TX, TY, TT::MINB, true, false, TT::TRIM>, conf_slab);
    } else if constexpr (S::D == 2) {
      using T = Tile1<TX>;
      const MethodParams<real> &p = *static_cast<const MethodParams<real> *>(params);
      const size_t smem = (size_t)3 * S::Q * T::HW * sizeof(real);
      // scripts/tb2d_variants.cu on B200 (profiles/r1/tb2d_variants.txt): >= 2 CTAs/SM with the
      // next row's loads prefetched; SRT (light collision): 3 CTAs/SM without the prefetch
      constexpr bool srt = SPACE == SPACE_POPULATION;
      auto go = [&](auto kern, unsigned &configured) {
        opt_in_smem_once(kern, smem, configured);
        kern<<<dim3((unsigned)(g.nx / TX), (unsigned)zchunks, 1), T::THREADS, smem, s>>>(
            static_cast<const real *>(src), static_cast<real *>(dst), g, p.rates, (real)swe_g, p.force);
      };
      static unsigned conf_slab = 0, conf_range = 0;
      if (g.zcount) go(k_pull2_2d<S, SPACE, REG, real, RS, TX, srt ? 3 : 2, !srt, true>, conf_range);
      else go(k_pull2_2d<S, SPACE, REG, real, RS, TX, srt ? 3 : 2, !srt, false>, conf_slab);
    }
  }
  // depth-3 2D sweep: 2 CTAs/SM with the next row's loads prefetched (scripts/tb2d_depth.cu,
  // profiles/r2/tb2d_depth.txt: 1 or 2 CTAs/SM and 37-148 slab chunks within 2 %)
  static constexpr int kDepth = 3, kDepthTX = 256;
  static void pull3(const void *src, void *dst, const GridParams &g, const void *params, double swe_g,
                    int zchunks, cudaStream_t s) {
    if constexpr (S::D == 2) {
      using T = TileD<S, kDepthTX, kDepth>;
      const MethodParams<real> &p = *static_cast<const MethodParams<real> *>(params);
      const size_t smem = (size_t)T::RING * sizeof(real);
      // whole slab with periodic wrap (single rank) or a row range without wrap (across ranks)
      auto go = [&](auto kern, unsigned &configured) {
        opt_in_smem_once(kern, smem, configured);
        kern<<<dim3((unsigned)(g.nx / kDepthTX), (unsigned)zchunks, 1), T::THREADS, smem, s>>>(
            static_cast<const real *>(src), static_cast<real *>(dst), g, p.rates, (real)swe_g, p.force);
      };
      static unsigned conf_slab = 0, conf_range = 0;
      if (g.zcount) go(k_pullD_2d<S, SPACE, REG, real, RS, kDepthTX, kDepth, 2, true, true>, conf_range);
      else go(k_pullD_2d<S, SPACE, REG, real, RS, kDepthTX, kDepth, 2, true, false>, conf_slab);
    }
  }
  template <bool BB>
  static cudaError_t launch_resident(const real *src, real *dst, const GridParams &g, const MethodParams<real> &p,
                                     double swe_g, int nsteps, int cluster, cudaStream_t s) {
    auto kern = k_resident2<S, SPACE, REG, real, RS, BB>;
    const int rows = g.nzl / cluster;
    const size_t smem = resident_smem(S::Q, g.nx, rows, (int)sizeof(real));
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess && cluster > 8) e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)cluster, 1, 1);
    cfg.blockDim = dim3((unsigned)std::min(1024, (rows * g.nx + 31) / 32 * 32), 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)cluster;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, src, dst, g, nsteps, p.rates, (real)swe_g, p.force);
  }
  static int resident(const void *src, void *dst, const GridParams &g, const void *params, double swe_g, int bb,
                      int nsteps, int cluster, cudaStream_t s) {
    if constexpr (S::D == 2) {
      const MethodParams<real> &p = *static_cast<const MethodParams<real> *>(params);
      const real *a = static_cast<const real *>(src);
      real *b = static_cast<real *>(dst);
      return (int)(bb ? launch_resident<true>(a, b, g, p, swe_g, nsteps, cluster, s)
                      : launch_resident<false>(a, b, g, p, swe_g, nsteps, cluster, s));
    }
    return (int)cudaErrorNotSupported;
  }
  static void attributes(int which, int *regs, int *local_bytes) {
    cudaFuncAttributes a{};
    cudaError_t e = cudaErrorInvalidValue;
    using TT = TbTile<S, real, SPACE>;
    if (which == 0) {
      e = cudaFuncGetAttributes(&a, k_pull<S, SPACE, REG, real, false, RS>);
    } else if (which == 1) {
      if constexpr (S::D == 3 && TT::TX > 0)
        e = cudaFuncGetAttributes(&a, k_pull2<S, SPACE, REG, real, RS, TT::TX, TT::TY, TT::MINB, true, false, TT::TRIM>);
      else if constexpr (S::D == 2) {
        constexpr bool srt = SPACE == SPACE_POPULATION;
        e = cudaFuncGetAttributes(&a, k_pull2_2d<S, SPACE, REG, real, RS, TT::TX, srt ? 3 : 2, !srt, false>);
      }
    } else if (which == 2) {
      if constexpr (S::D == 2) e = cudaFuncGetAttributes(&a, k_resident2<S, SPACE, REG, real, RS, false>);
    } else if (which == 3) {
      if constexpr (S::D == 2) e = cudaFuncGetAttributes(&a, k_pullD_2d<S, SPACE, REG, real, RS, kDepthTX, kDepth, 2, true>);
    } else if (which == 10 + PAT_AA_ODD) {
      e = cudaFuncGetAttributes(&a, k_aa<S, SPACE, REG, real, PAT_AA_ODD, RS>);
    } else if (which == 10 + PAT_AA_EVEN) {
      e = cudaFuncGetAttributes(&a, k_aa<S, SPACE, REG, real, PAT_AA_EVEN, RS>);
    } else if (which == 10 + PAT_ESO_ODD) {
      e = cudaFuncGetAttributes(&a, k_eso<S, SPACE, REG, real, PAT_ESO_ODD, RS>);
    } else if (which == 10 + PAT_ESOP_ODD) {
      e = cudaFuncGetAttributes(&a, k_eso<S, SPACE, REG, real, PAT_ESOP_ODD, RS>);
    } else if (which == 10 + PAT_TW0) {
      e = cudaFuncGetAttributes(&a, k_twist<S, SPACE, REG, real, PAT_TW0, RS>);
    }
    if (e == cudaSuccess) {
      *regs = a.numRegs;
      *local_bytes = (int)a.localSizeBytes;
    } else {
      cudaGetLastError();
      *regs = -1;
      *local_bytes = -1;
    }
  }
  static void preload() {
    cudaFuncAttributes a{};
    using TT = TbTile<S, real, SPACE>;
    cudaFuncGetAttributes(&a, k_pull<S, SPACE, REG, real, false, RS>);
    cudaFuncGetAttributes(&a, k_pull<S, SPACE, REG, real, true, RS>);
    cudaFuncGetAttributes(&a, k_pull<S, SPACE, REG, real, false, RS, true>);
    cudaFuncGetAttributes(&a, k_pull<S, SPACE, REG, real, true, RS, true>);
    cudaFuncGetAttributes(&a, k_aa<S, SPACE, REG, real, PAT_AA_EVEN, RS>);
    cudaFuncGetAttributes(&a, k_aa<S, SPACE, REG, real, PAT_AA_ODD, RS>);
    cudaFuncGetAttributes(&a, k_aa<S, SPACE, REG, real, PAT_AA_ODD, RS, true>);
    if constexpr (S::D == 3 && TT::TX > 0) {
      cudaFuncGetAttributes(&a, k_pull2<S, SPACE, REG, real, RS, TT::TX, TT::TY, TT::MINB, true, true, TT::TRIM>);
    } else if constexpr (S::D == 2) {
      constexpr bool srt = SPACE == SPACE_POPULATION;
      cudaFuncGetAttributes(&a, k_pull2_2d<S, SPACE, REG, real, RS, TT::TX, srt ? 3 : 2, !srt, true>);
      cudaFuncGetAttributes(&a, k_pullD_2d<S, SPACE, REG, real, RS, kDepthTX, kDepth, 2, true, true>);
    }
    cudaGetLastError();
  }
  static int set_wo(const double *L, const double *Linv) {
    cudaError_t e = cudaMemcpyToSymbol(c_wo_L, L, 27 * 27 * sizeof(double));
    if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_wo_Linv, Linv, 27 * 27 * sizeof(double));
    return (int)e;
  }
  static constexpr Ops table{S::Q,      S::D,  &pull,         &aa,           &init,      &get_pop,
                             &set_pop, &macro, &test_collide, &check_finite, &get_cells, &diagnostics,
                             &attributes,
                             (TbTile<S, real, SPACE>::TX > 0) ? &pull2 : nullptr,
                             TbTile<S, real, SPACE>::TX,
                             TbTile<S, real, SPACE>::TY,
                             S::D == 2 ? &resident : nullptr,
                             &preload,
                             &set_wo,
                             S::D == 2 ? &pull3 : nullptr};
};

}  // namespace lbm
