// tb2d_1b.cuh — scratch variant (not product code): the depth-D 2D sweep of k_pullD_2d with
// ONE barrier per sweep iteration.  Level s is computed at row k - 2 (s - 1) (skewed by two rows
// per level instead of one), so every row a level pulls from was written in an earlier
// iteration; one more ring row per population (4 / 3 / 2 for xi_y = +1 / 0 / -1) keeps the row
// being written apart from the rows being read within an iteration.
#pragma once
#include "kernels.cuh"

namespace lbm {

template <class S, int SPACE, int REG, class real, int RS, int TX, int D, int MINB = 1, bool PF = true>
__global__ void __launch_bounds__(TileD<S, TX, D, 1>::THREADS, MINB)
    k_pullD1b_2d(const real *__restrict__ src, real *__restrict__ dst, const GridParams g, const Rates<real> r,
                 const real swe_g, const Force<real> fr) {
  using T = TileD<S, TX, D, 1>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  real *ring = reinterpret_cast<real *>(smem_raw);
  const int t = threadIdx.x;
  const int x0 = blockIdx.x * TX;
  const int n = g.nzl;
  const int p0 = (int)((long long)n * blockIdx.y / gridDim.y);
  const int p1 = (int)((long long)n * (blockIdx.y + 1) / gridDim.y);
  constexpr int W1 = T::W(1);
  const bool act1 = t < W1;
  const int gx = wrapi(x0 - (D - 1) + t, g.nx);
  const int xs[3] = {wrapi(gx - 1, g.nx), gx, wrapi(gx + 1, g.nx)};
  auto load = [&](int k, real(&f)[S::Q]) {
    const int zc = wrapi(k, n);
    const long long zo[3] = {(long long)(wrapi(zc - 1, n) + 1) * g.plane, (long long)(zc + 1) * g.plane,
                             (long long)(wrapi(zc + 1, n) + 1) * g.plane};
    sfor<S::Q>([&](auto i) {
      constexpr int cx = S::mx(i), cz = S::mz(i);
      f[i] = ld_nc(src + zo[1 - cz] + (long long)i * g.pop + xs[1 - cx]);
    });
  };
  // level s at row k - 2 (s - 1), rows [p0 - (D - s), p1 + (D - s))
  const int kb = p0 - (D - 1), ke = p1 + 2 * (D - 1);
  const int l1end = p1 + (D - 1);  // level-1 rows end
  real fn[PF ? S::Q : 1];
  if constexpr (PF) {
    if (act1) load(kb, fn);
  }
  for (int k = kb; k < ke; ++k) {
    if (act1 && k < l1end) {
      real f[S::Q];
      if constexpr (PF) {
        sfor<S::Q>([&](auto i) { f[i] = fn[i]; });
        if (k + 1 < l1end) load(k + 1, fn);
      } else {
        load(k, f);
      }
      collide<S, SPACE, REG, real, RS>(f, r, swe_g, fr);
      real *lv = ring + T::level_off(1);
      sfor<S::Q>([&](auto i) { lv[T::pop_off(i, W1) + ((k + 16) % T::slots(i)) * W1 + t] = f[i]; });
    }
    sfor<D - 1>([&](auto sm) {
      constexpr int s = sm + 2;
      constexpr int Ws = T::W(s), Wp = T::W(s - 1);
      const int row = k - 2 * (s - 1);
      if (t < Ws && row >= p0 - (D - s) && row < p1 + (D - s)) {
        const real *pv = ring + T::level_off(s - 1);
        real f[S::Q];
        sfor<S::Q>([&](auto i) {
          constexpr int cx = S::mx(i), cz = S::mz(i);
          f[i] = pv[T::pop_off(i, Wp) + ((row - cz + 16) % T::slots(i)) * Wp + (t + 1 - cx)];
        });
        collide<S, SPACE, REG, real, RS>(f, r, swe_g, fr);
        if constexpr (s == D) {
          const long long own = (long long)(wrapi(row, n) + 1) * g.plane + (x0 + t);
          sfor<S::Q>([&](auto i) { dst[own + (long long)i * g.pop] = f[i]; });
        } else {
          real *lv = ring + T::level_off(s);
          sfor<S::Q>([&](auto i) { lv[T::pop_off(i, Ws) + ((row + 16) % T::slots(i)) * Ws + t] = f[i]; });
        }
      }
    });
    __syncthreads();
  }
}

}  // namespace lbm
