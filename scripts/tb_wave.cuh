// tb_wave.cuh — scratch prototype (not product code): two fused pull steps per HBM sweep for
// 3D lattices WITHOUT halo recompute.  One persistent CTA per SM (cooperative launch) owns a
// contiguous range of 32-cell row segments ("units") of every x-y plane; the grid sweeps the
// slab axis as a wavefront.  Iteration k: step t+1 of plane k (pulled from src, HBM) into an
// L2-resident scratch ring of SR planes in global memory; step t+2 of plane k - L (pulled from
// the ring, neighbours' cells included) into dst.  A CTA starts iteration k once the CTAs that
// own the rows next to its own have completed iteration k - 2 (per-CTA progress flags,
// release / acquire at gpu scope): step t+2 of plane k - L reads step t+1 of planes up to
// k - L + 1 = k - 2, and the ring slot written at k held plane k - SR, whose last reader ran at
// iteration k - SR + 1 + L <= k - 2.  Every cell is collided once per step (no halo recompute);
// HBM moves 2qS per cell per two steps, the ring stays in L2.
#pragma once
#include "kernels.cuh"

namespace lbm {

constexpr int kWaveL = 3, kWaveSR = 6;

__device__ __forceinline__ int ld_acquire_gpu(const int *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(int *p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// CTA that owns unit v (units split as floor(c U / G))
__device__ __forceinline__ int wave_owner(long long v, long long U, int G) {
  return (int)(((v + 1) * G - 1) / U);
}

template <class S, int SPACE, int REG, class real, int RS, int NT, bool PF, bool FENCE = true, bool WAIT = true>
__global__ void __launch_bounds__(NT, 1)
    k_pull2_wave(const real *__restrict__ src, real *__restrict__ dst, real *scr, int *flags, const GridParams g,
                 const Rates<real> r, const real swe_g, const Force<real> fr, unsigned long long timeout_ns,
                 int *err) {
  const int G = gridDim.x, c = blockIdx.x;
  const int nxu = g.nx / 32;
  const long long U = (long long)nxu * g.ny;
  const long long u0 = (long long)c * U / G, u1 = (long long)(c + 1) * U / G;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const long long u = u0 + warp;
  const bool act = u < u1;
  const int y = act ? (int)(u / nxu) : 0;
  const int x = act ? (int)(u % nxu) * 32 + lane : 0;
  int xs[3], ys[3];
#pragma unroll
  for (int s = -1; s <= 1; ++s) {
    xs[s + 1] = wrapi(x + s, g.nx);
    ys[s + 1] = wrapi(y + s, g.ny) * g.pitch;
  }
  const int n = g.nzl;
  const long long splane = (long long)S::Q * g.pop;  // scratch plane (no ghost planes)
  // CTAs owning the rows next to mine: units [u0 - 2 nxu, u1 + 2 nxu) (cyclic) — the diagonal
  // neighbour of a row's last unit across the periodic x wrap is the FIRST unit of the next
  // row, up to 2 nxu - 1 units away
  const int cfirst = wave_owner(((u0 - 2 * nxu) % U + U) % U, U, G);
  const int clast = wave_owner((u1 - 1 + 2 * nxu) % U, U, G);
  const int nwait = (clast - cfirst + G) % G + 1;  // cyclic range incl. me
  __shared__ int s_abort;
  if (threadIdx.x == 0) s_abort = 0;
  __syncthreads();

  auto load = [&](int k, real(&f)[S::Q]) {
    const int zc = wrapi(k, n);
    long long zo[3];
#pragma unroll
    for (int s = -1; s <= 1; ++s) zo[s + 1] = (long long)(wrapi(zc + s, n) + 1) * g.plane;
    sfor<S::Q>([&](auto i) {
      constexpr int cx = S::mx(i), cy = S::my(i), cz = S::mz(i);
      f[i] = ld_nc(src + zo[1 - cz] + (long long)i * g.pop + ys[1 - cy] + xs[1 - cx]);
    });
  };
  real fn[PF ? S::Q : 1];
  if constexpr (PF) {
    if (act) load(-1, fn);
  }
  const unsigned long long t0 = gtimer();
  for (int k = -1; k < n + kWaveL; ++k) {
    // wait until the neighbouring CTAs completed iteration k - 2 (flag = iteration + 2)
    if (WAIT && threadIdx.x < nwait) {
      const int cc = (cfirst + threadIdx.x) % G;
      if (cc != c) {
        while (ld_acquire_gpu(flags + cc) < k) {
          if (gtimer() - t0 > timeout_ns) {
            s_abort = 1;
            atomicExch(err, 1);
            break;
          }
          __nanosleep(64);
        }
      }
    }
    __syncthreads();
    if (s_abort) return;
    if (k <= n && act) {  // step t+1 of plane k -> ring slot k
      real f[S::Q];
      if constexpr (PF) {
        sfor<S::Q>([&](auto i) { f[i] = fn[i]; });
        if (k < n) load(k + 1, fn);
      } else {
        load(k, f);
      }
      collide<S, SPACE, REG, real, RS>(f, r, swe_g, fr);
      real *o = scr + (long long)((k + kWaveSR) % kWaveSR) * splane + (long long)y * g.pitch + x;
      sfor<S::Q>([&](auto i) { o[(long long)i * g.pop] = f[i]; });
    }
    const int p = k - kWaveL;
    if (p >= 0 && act) {  // step t+2 of plane p from the ring (planes p-1 .. p+1)
      real f[S::Q];
      sfor<S::Q>([&](auto i) {
        constexpr int cx = S::mx(i), cy = S::my(i), cz = S::mz(i);
        const real *a = scr + (long long)((p - cz + kWaveSR) % kWaveSR) * splane + (long long)i * g.pop +
                        ys[1 - cy] + xs[1 - cx];
        f[i] = __ldcg(a);
      });
      collide<S, SPACE, REG, real, RS>(f, r, swe_g, fr);
      real *o = dst + (long long)(p + 1) * g.plane + (long long)y * g.pitch + x;
      sfor<S::Q>([&](auto i) { o[(long long)i * g.pop] = f[i]; });
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      if (FENCE) __threadfence();
      st_release_gpu(flags + c, k + 2);
    }
  }
}

}  // namespace lbm
