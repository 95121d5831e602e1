// tb3d_depth.cuh — scratch prototype (not product code): temporal blocking of depth D for 3D
// lattices (the 2D k_pullD_2d scheme on TX x TY tiles).  Level s = 1..D (time step t+s) is
// computed at plane k - (s - 1) of sweep iteration k on the tile widened by D - s cells per
// side in x and y; level 1 pulls from HBM (next plane prefetched), level s >= 2 from the
// trimmed shared-memory ring of level s - 1, level D stores.  Single rank, periodic.
#pragma once
#include "kernels.cuh"

namespace lbm {

template <class S, int TX, int TY, int D>
struct Tile3D {
  static constexpr int WX(int s) { return TX + 2 * (D - s); }
  static constexpr int WY(int s) { return TY + 2 * (D - s); }
  static constexpr int W(int s) { return WX(s) * WY(s); }
  static constexpr int THREADS = (W(1) + 31) / 32 * 32;
  static constexpr int slots(int i) { return S::mz(i) > 0 ? 3 : (S::mz(i) == 0 ? 2 : 1); }
  static constexpr int per_level(int w) {
    int o = 0;
    for (int j = 0; j < S::Q; ++j) o += slots(j) * w;
    return o;
  }
  static constexpr int level_off(int s) {
    int o = 0;
    for (int l = 1; l < s; ++l) o += per_level(W(l));
    return o;
  }
  static constexpr int pop_off(int i, int w) {
    int o = 0;
    for (int j = 0; j < i; ++j) o += slots(j) * w;
    return o;
  }
  static constexpr int RING = level_off(D);
};

template <class S, int SPACE, int REG, class real, int RS, int TX, int TY, int D, int MINB = 1, bool PF = true>
__global__ void __launch_bounds__(Tile3D<S, TX, TY, D>::THREADS, MINB)
    k_pullD_3d(const real *__restrict__ src, real *__restrict__ dst, const GridParams g, const Rates<real> r,
               const real swe_g, const Force<real> fr) {
  using T = Tile3D<S, TX, TY, D>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  real *ring = reinterpret_cast<real *>(smem_raw);
  const int t = threadIdx.x;
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const int n = g.nzl;
  const int p0 = (int)((long long)n * blockIdx.z / gridDim.z);
  const int p1 = (int)((long long)n * (blockIdx.z + 1) / gridDim.z);
  constexpr int W1 = T::W(1), WX1 = T::WX(1);
  const bool act1 = t < W1;
  const int hx = t % WX1, hy = t / WX1;
  const int gx = wrapi(x0 - (D - 1) + hx, g.nx), gy = wrapi(y0 - (D - 1) + hy, g.ny);
  int xs[3];
  long long ys[3];
#pragma unroll
  for (int s = -1; s <= 1; ++s) {
    xs[s + 1] = wrapi(gx + s, g.nx);
    ys[s + 1] = (long long)wrapi(gy + s, g.ny) * g.pitch;
  }
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
  const int kb = p0 - (D - 1), ke = p1 + (D - 1);
  real fn[PF ? S::Q : 1];
  if constexpr (PF) {
    if (act1) load(kb, fn);
  }
  for (int k = kb; k < ke; ++k) {
    if (act1) {
      real f[S::Q];
      if constexpr (PF) {
        sfor<S::Q>([&](auto i) { f[i] = fn[i]; });
        if (k + 1 < ke) load(k + 1, fn);
      } else {
        load(k, f);
      }
      collide<S, SPACE, REG, real, RS>(f, r, swe_g, fr);
      real *lv = ring + T::level_off(1);
      sfor<S::Q>([&](auto i) { lv[T::pop_off(i, W1) + ((k + 12) % T::slots(i)) * W1 + t] = f[i]; });
    }
    sfor<D - 1>([&](auto sm) {
      constexpr int s = sm + 2;
      constexpr int Ws = T::W(s), WXs = T::WX(s), Wp = T::W(s - 1), WXp = T::WX(s - 1);
      __syncthreads();
      const int row = k - (s - 1);
      if (t < Ws && row >= p0 - (D - s) && row < p1 + (D - s)) {
        const int ix = t % WXs, iy = t / WXs;
        const real *pv = ring + T::level_off(s - 1);
        real f[S::Q];
        sfor<S::Q>([&](auto i) {
          constexpr int cx = S::mx(i), cy = S::my(i), cz = S::mz(i);
          f[i] = pv[T::pop_off(i, Wp) + ((row - cz + 12) % T::slots(i)) * Wp + (iy + 1 - cy) * WXp + (ix + 1 - cx)];
        });
        collide<S, SPACE, REG, real, RS>(f, r, swe_g, fr);
        if constexpr (s == D) {
          const long long own = (long long)(wrapi(row, n) + 1) * g.plane + (long long)(y0 + iy) * g.pitch + (x0 + ix);
          sfor<S::Q>([&](auto i) { dst[own + (long long)i * g.pop] = f[i]; });
        } else {
          real *lv = ring + T::level_off(s);
          sfor<S::Q>([&](auto i) { lv[T::pop_off(i, Ws) + ((row + 12) % T::slots(i)) * Ws + t] = f[i]; });
        }
      }
    });
    __syncthreads();
  }
}

}  // namespace lbm
