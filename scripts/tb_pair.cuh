// tb_pair.cuh — scratch variant (not product code): the two-step sweep of k_pull2 with every
// thread owning TWO cells of a tile row, hx and hx + PX (x-paired).  The pair shares its row
// address: the loads of cell B are the loads of cell A at a compile-time element offset (an
// immediate in the LDG encoding), the ring slots and the step-(t+2) stores likewise, so the
// 64-bit address arithmetic per global access halves and the two independent collisions give
// the scheduler ILP at half the warps.  Edge tiles of the x axis (periodic wrap inside the
// halo) take a generic path with wrapped x per cell (a CTA-uniform branch).
#pragma once
#include "kernels.cuh"

namespace lbm {

template <int TX, int TY>
struct TileP {
  static constexpr int HX = TX + 2, HY = TY + 2, HW = HX * HY;
  static_assert(TX % 2 == 0, "x-paired tiles need an even width");
  static constexpr int PX = HX / 2, IX = TX / 2;  // pairs per halo / interior row
  static constexpr int N1 = PX * HY, N2 = IX * TY;
  static constexpr int THREADS = (N1 + 31) / 32 * 32;
};

template <class S, int SPACE, int REG, class real, int RS, int TX, int TY, bool PF, bool EDGE>
__device__ __forceinline__ void sweep_pairs(const real *__restrict__ src, real *__restrict__ dst, const GridParams &g,
                                            const Rates<real> &r, const real swe_g, const Force<real> &fr,
                                            real *ring) {
  using T = TileP<TX, TY>;
  const int t = threadIdx.x;
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const bool act1 = t < T::N1;
  const int hx = t % T::PX, hy = t / T::PX;
  const int gx = x0 - 1 + hx;  // x of cell A (unwrapped; EDGE wraps per neighbour)
  const int gy = wrapi(y0 - 1 + hy, g.ny);
  long long ys[3];
#pragma unroll
  for (int s = -1; s <= 1; ++s) ys[s + 1] = (long long)wrapi(gy + s, g.ny) * g.pitch;
  int xa[3], xb[3];
  if constexpr (EDGE) {
#pragma unroll
    for (int s = -1; s <= 1; ++s) {
      xa[s + 1] = wrapi(gx + s, g.nx);
      xb[s + 1] = wrapi(gx + T::PX + s, g.nx);
    }
  }
  const bool act2 = t < T::N2;
  const int ix = t % T::IX, iy = t / T::IX;
  const int n = g.nzl;
  const int p0 = (int)((long long)n * blockIdx.z / gridDim.z);
  const int p1 = (int)((long long)n * (blockIdx.z + 1) / gridDim.z);
  auto load = [&](int k, real(&fa)[S::Q], real(&fb)[S::Q]) {
    const int zc = wrapi(k, n);
    long long zo[3];
#pragma unroll
    for (int s = -1; s <= 1; ++s) zo[s + 1] = (long long)(wrapi(zc + s, n) + 1) * g.plane;
    sfor<S::Q>([&](auto i) {
      constexpr int cx = S::mx(i), cy = S::my(i), cz = S::mz(i);
      const real *row = src + zo[1 - cz] + (long long)i * g.pop + ys[1 - cy];
      if constexpr (EDGE) {
        fa[i] = ld_nc(row + xa[1 - cx]);
        fb[i] = ld_nc(row + xb[1 - cx]);
      } else {
        const real *p = row + gx;
        fa[i] = ld_nc(p - cx);
        fb[i] = ld_nc(p + (T::PX - cx));
      }
    });
  };
  real na[PF ? S::Q : 1], nb[PF ? S::Q : 1];
  if constexpr (PF) {
    if (act1) load(p0 - 1, na, nb);
  }
  for (int k = p0 - 1; k <= p1; ++k) {
    if (act1) {
      real fa[S::Q], fb[S::Q];
      if constexpr (PF) {
        sfor<S::Q>([&](auto i) {
          fa[i] = na[i];
          fb[i] = nb[i];
        });
        if (k < p1) load(k + 1, na, nb);
      } else {
        load(k, fa, fb);
      }
      collide<S, SPACE, REG, real, RS>(fa, r, swe_g, fr);
      collide<S, SPACE, REG, real, RS>(fb, r, swe_g, fr);
      real *slot = ring + (size_t)((k + 3) % 3) * S::Q * T::HW + hy * T::HX + hx;
      sfor<S::Q>([&](auto i) {
        slot[i * T::HW] = fa[i];
        slot[i * T::HW + T::PX] = fb[i];
      });
    }
    __syncthreads();
    if (k >= p0 + 1 && act2) {
      const int p = k - 1;
      real fa[S::Q], fb[S::Q];
      sfor<S::Q>([&](auto i) {
        constexpr int cx = S::mx(i), cy = S::my(i), cz = S::mz(i);
        const real *slot = ring + (size_t)((p - cz + 3) % 3) * S::Q * T::HW + i * T::HW +
                           (iy + 1 - cy) * T::HX + (ix + 1 - cx);
        fa[i] = slot[0];
        fb[i] = slot[T::IX];
      });
      collide<S, SPACE, REG, real, RS>(fa, r, swe_g, fr);
      collide<S, SPACE, REG, real, RS>(fb, r, swe_g, fr);
      real *own = dst + (long long)(p + 1) * g.plane + (long long)(y0 + iy) * g.pitch + (x0 + ix);
      sfor<S::Q>([&](auto i) {
        own[(long long)i * g.pop] = fa[i];
        own[(long long)i * g.pop + T::IX] = fb[i];
      });
    }
    __syncthreads();
  }
}

template <class S, int SPACE, int REG, class real, int RS, int TX, int TY, int MINB = 1, bool PF = true>
__global__ void __launch_bounds__(TileP<TX, TY>::THREADS, MINB)
    k_pull2p(const real *__restrict__ src, real *__restrict__ dst, const GridParams g, const Rates<real> r,
             const real swe_g, const Force<real> fr) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  real *ring = reinterpret_cast<real *>(smem_raw);
  if (blockIdx.x == 0 || blockIdx.x + 1 == gridDim.x)
    sweep_pairs<S, SPACE, REG, real, RS, TX, TY, PF, true>(src, dst, g, r, swe_g, fr, ring);
  else
    sweep_pairs<S, SPACE, REG, real, RS, TX, TY, PF, false>(src, dst, g, r, swe_g, fr, ring);
}

}  // namespace lbm
