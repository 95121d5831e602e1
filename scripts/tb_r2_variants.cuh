// tb_r2_variants.cuh — scratch temporal-blocking variants measured in round 2 and NOT used by the
// product (scripts/tb_tma.cu; results and ncu reading in profiles/r2/tb_variants_r2.txt): the
// one-barrier-per-plane sweep (equal to k_pull2) and the warp-specialised producer/consumer
// sweep with cp.async staging (slower: the producers, capped at 96 registers, starve the
// consumers).  Both equal to k_pull2 bitwise / to rounding (maxdiff column).
#pragma once
#include "kernels.cuh"

namespace lbm {

// ---------------------------------------------------------------------------
// Temporal blocking with ONE barrier per plane (k_pull2_1b): iteration k computes step t+1 of
// plane k on the halo-extended tile AND step t+2 of plane k - 2 on the tile interior.  The
// step-(t+2) pull reads planes k - 3 .. k - 1 of the ring, all complete before the previous
// barrier, so the two collisions need no barrier between them: every thread runs them back to
// back (independent instruction streams) and the loads of plane k + 1 fly under both.  The
// ring keeps 4 / 3 / 2 planes of the xi_z = +1 / 0 / -1 populations (a plane is written into
// a slot no reader of the same iteration touches) = 3 Q planes, as k_pull2's untrimmed ring.
// ---------------------------------------------------------------------------
template <int TX, int TY, class S>
struct Tile2Ring1b {
  static constexpr int HW = (TX + 2) * (TY + 2);
  static constexpr int slots(int i) { return S::mz(i) > 0 ? 4 : (S::mz(i) == 0 ? 3 : 2); }
  static constexpr int off(int i) {
    int o = 0;
    for (int j = 0; j < i; ++j) o += slots(j) * HW;
    return o;
  }
  static constexpr int RING = off(S::Q);
};

template <class S, int SPACE, int REG, class real, int RS, int TX, int TY, int MINB = 1, bool RANGE = false>
__global__ void __launch_bounds__(Tile2<TX, TY>::THREADS, MINB)
    k_pull2_1b(const real *__restrict__ src, real *__restrict__ dst, const GridParams g, const Rates<real> r,
               const real swe_g, const Force<real> fr) {
  using T = Tile2<TX, TY>;
  using TR = Tile2Ring1b<TX, TY, S>;
  extern __shared__ __align__(16) unsigned char smem_1b[];
  real *ring = reinterpret_cast<real *>(smem_1b);
  const int t = threadIdx.x;
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const bool act1 = t < T::HW;
  const int hx = t % T::HX, hy = t / T::HX;
  const int gx = wrapi(x0 - 1 + hx, g.nx), gy = wrapi(y0 - 1 + hy, g.ny);
  int xs[3], ys[3];
#pragma unroll
  for (int s = -1; s <= 1; ++s) {
    xs[s + 1] = wrapi(gx + s, g.nx);
    ys[s + 1] = wrapi(gy + s, g.ny) * g.pitch;
  }
  const bool act2 = t < TX * TY;
  const int ix = t % TX, iy = t / TX;
  const int n = g.nzl;
  const int zb = RANGE ? g.zbegin : 0, zn = RANGE ? g.zcount : n;
  const int p0 = zb + (int)((long long)zn * blockIdx.z / gridDim.z);
  const int p1 = zb + (int)((long long)zn * (blockIdx.z + 1) / gridDim.z);
  auto zw = [&](int k) {
    if constexpr (RANGE) return k;
    else return wrapi(k, n);
  };
  auto load = [&](int k, real (&f)[S::Q]) {
    const int zc = zw(k);
    long long zo[3];
#pragma unroll
    for (int s = -1; s <= 1; ++s) zo[s + 1] = (long long)(zw(zc + s) + 1) * g.plane;
    sfor<S::Q>([&](auto i) {
      constexpr int cx = S::mx(i), cy = S::my(i), cz = S::mz(i);
      f[i] = ld_nc(src + zo[1 - cz] + (long long)i * g.pop + ys[1 - cy] + xs[1 - cx]);
    });
  };
  real fn[S::Q];
  if (act1) load(p0 - 1, fn);
  for (int k = p0 - 1; k <= p1 + 1; ++k) {
    real f1[S::Q];
    const bool do1 = act1 && k <= p1;
    if (do1) {
      sfor<S::Q>([&](auto i) { f1[i] = fn[i]; });
      if (k < p1) load(k + 1, fn);
    }
    const int p = k - 2;  // plane of step t+2
    if (p >= p0 && act2) {
      real f[S::Q];
      sfor<S::Q>([&](auto i) {
        constexpr int cx = S::mx(i), cy = S::my(i), cz = S::mz(i);
        f[i] = ring[TR::off(i) + ((p - cz + 12) % TR::slots(i)) * T::HW + (iy + 1 - cy) * T::HX + (ix + 1 - cx)];
      });
      collide<S, SPACE, REG, real, RS>(f, r, swe_g, fr);
      const long long own = (long long)(p + 1) * g.plane + (long long)(y0 + iy) * g.pitch + (x0 + ix);
      sfor<S::Q>([&](auto i) { dst[own + (long long)i * g.pop] = f[i]; });
    }
    if (do1) {
      collide<S, SPACE, REG, real, RS>(f1, r, swe_g, fr);
      sfor<S::Q>([&](auto i) { ring[TR::off(i) + ((k + 12) % TR::slots(i)) * T::HW + t] = f1[i]; });
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Temporal blocking, warp-specialised (k_pull2_ws): the two-step sweep of k_pull2 with its two
// phases running CONCURRENTLY in different warps of the CTA instead of alternating behind
// __syncthreads.  Producer warps (one thread per cell of the halo-extended tile) stream the
// step-t populations of plane k + 1 into a double-buffered shared-memory stage with cp.async
// (no prefetch registers) while they collide plane k (step t+1) and write it into the trimmed
// ring; consumer warps (one thread per interior cell) collide step t+2 of plane k - 1 from the
// ring and store it.  Hand-off through mbarriers: full[k mod 3] completes when plane k of
// step t+1 is in the ring (producer arrivals), empty when the consumers finished a plane; the
// producer writes plane k once the consumers are done with plane k - 2 (the last reader of
// the ring slots plane k overwrites: 3 / 2 / 1 planes of the xi_z = +1 / 0 / -1 populations).
// So the step-(t+1) collisions of plane k + 1 overlap the step-(t+2) collisions of plane k - 1
// and the HBM loads of plane k + 2.  Same collide() as k_pull, equal to two k_pull launches.
// ---------------------------------------------------------------------------
template <int TX, int TY>
struct TileWs {
  static constexpr int HX = TX + 2, HY = TY + 2, HW = HX * HY;
  static constexpr int P = (HW + 31) / 32 * 32;         // producer threads
  static constexpr int C = (TX * TY + 31) / 32 * 32;    // consumer threads
  static constexpr int THREADS = P + C;
};

template <class S, class real, int TX, int TY>
constexpr size_t ws_smem_bytes() {
  using T = TileWs<TX, TY>;
  return (size_t)(2 * S::Q * T::HW + Tile2Trim<TX, TY, S>::RING) * sizeof(real) + 4 * sizeof(uint64_t);
}

template <class S, int SPACE, int REG, class real, int RS, int TX, int TY, int MINB = 1, bool RANGE = false>
__global__ void __launch_bounds__(TileWs<TX, TY>::THREADS, MINB)
    k_pull2_ws(const real *__restrict__ src, real *__restrict__ dst, const GridParams g, const Rates<real> r,
               const real swe_g, const Force<real> fr) {
  using T = TileWs<TX, TY>;
  using TR = Tile2Trim<TX, TY, S>;
  extern __shared__ __align__(16) unsigned char smem_ws[];
  real *stage = reinterpret_cast<real *>(smem_ws);  // [2][Q][HW] step t, planes k and k + 1
  real *ring = stage + 2 * S::Q * T::HW;            // trimmed step-(t+1) ring
  uint64_t *full = reinterpret_cast<uint64_t *>(ring + TR::RING);  // [3]
  uint64_t *empty = full + 3;
  const int t = threadIdx.x;
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const int n = g.nzl;
  const int zb = RANGE ? g.zbegin : 0, zn = RANGE ? g.zcount : n;
  const int p0 = zb + (int)((long long)zn * blockIdx.z / gridDim.z);
  const int p1 = zb + (int)((long long)zn * (blockIdx.z + 1) / gridDim.z);
  auto zw = [&](int k) {
    if constexpr (RANGE) return k;
    else return wrapi(k, n);
  };
  if (t == 0) {
    for (int m = 0; m < 3; ++m) mbar_init(full + m, T::P);
    mbar_init(empty, T::C);
  }
  __syncthreads();
  if (t < T::P) {  // ---------------- producer: step t+1 on the halo-extended tile
    const bool act1 = t < T::HW;
    const int hx = t % T::HX, hy = t / T::HX;
    const int gx = wrapi(x0 - 1 + hx, g.nx), gy = wrapi(y0 - 1 + hy, g.ny);
    int xs[3], ys[3];
#pragma unroll
    for (int s = -1; s <= 1; ++s) {
      xs[s + 1] = wrapi(gx + s, g.nx);
      ys[s + 1] = wrapi(gy + s, g.ny) * g.pitch;
    }
    // step-t populations of plane k (pull: plane k - xi_z) into stage buffer b, this thread's
    // own slots only (so only this thread's wait_group orders them)
    auto issue = [&](int k, int b) {
      if (act1) {
        const int zc = zw(k);
        long long zo[3];
#pragma unroll
        for (int s = -1; s <= 1; ++s) zo[s + 1] = (long long)(zw(zc + s) + 1) * g.plane;
        real *st = stage + b * S::Q * T::HW + t;
        sfor<S::Q>([&](auto i) {
          constexpr int cx = S::mx(i), cy = S::my(i), cz = S::mz(i);
          cp_async(st + i * T::HW, src + zo[1 - cz] + (long long)i * g.pop + ys[1 - cy] + xs[1 - cx]);
        });
      }
      cp_async_commit();
    };
    issue(p0 - 1, 0);
    for (int k = p0 - 1; k <= p1; ++k) {
      const int it = k - (p0 - 1);
      if (k < p1) {
        issue(k + 1, (it + 1) & 1);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      real f[S::Q];
      if (act1) {
        const real *st = stage + (it & 1) * S::Q * T::HW + t;
        sfor<S::Q>([&](auto i) { f[i] = st[i * T::HW]; });
        collide<S, SPACE, REG, real, RS>(f, r, swe_g, fr);
      }
      if (k >= p0 + 2) mbar_wait(empty, (uint32_t)((k - 2 - p0) & 1));  // consumers done with k - 2
      if (act1) sfor<S::Q>([&](auto i) { ring[TR::off(i) + ((k + 3) % TR::slots(i)) * T::HW + t] = f[i]; });
      mbar_arrive(full + it % 3);
    }
  } else {  // ---------------- consumer: step t+2 on the tile interior
    const int c = t - T::P;
    const bool act2 = c < TX * TY;
    const int ix = c % TX, iy = c / TX;
    for (int p = p0; p < p1; ++p) {
      if (p == p0) {  // planes p0 - 1 and p0 (phase 0 of full[0], full[1])
        mbar_wait(full + 0, 0);
        mbar_wait(full + 1, 0);
      }
      const int j = p + 1 - (p0 - 1);  // plane p + 1
      mbar_wait(full + j % 3, (uint32_t)((j / 3) & 1));
      if (act2) {
        real f[S::Q];
        sfor<S::Q>([&](auto i) {
          constexpr int cx = S::mx(i), cy = S::my(i), cz = S::mz(i);
          f[i] = ring[TR::off(i) + ((p - cz + 3) % TR::slots(i)) * T::HW + (iy + 1 - cy) * T::HX + (ix + 1 - cx)];
        });
        collide<S, SPACE, REG, real, RS>(f, r, swe_g, fr);
        const long long own = (long long)(p + 1) * g.plane + (long long)(y0 + iy) * g.pitch + (x0 + ix);
        sfor<S::Q>([&](auto i) { dst[own + (long long)i * g.pop] = f[i]; });
      }
      mbar_arrive(empty);
    }
  }
}

}  // namespace lbm
