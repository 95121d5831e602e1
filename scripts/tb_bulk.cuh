// tb_bulk.cuh — EXPERIMENTAL temporal-blocking kernels (scratch, not product code), measured
// by scripts/tb_bulk_variants.cu against the product's k_pull2 / k_pull2_2d:
//   k_pull2b  the step-t populations staged by cp.async.bulk (TMA engine) into a shared ring
//   k_pull2w  step t+1 and step t+2 on two concurrent warp groups, one barrier per plane
#pragma once
#include "kernels.cuh"

namespace lbm {

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

// make the initialised barriers visible to the async proxy (the bulk-copy engine)
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// one arrival that also announces 'bytes' of transactions the copies will complete
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

// wait until the phase with parity 'parity' of the barrier has completed
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!done);
}

// global -> shared bulk copy of 'bytes' (multiple of 16; both addresses 16-byte aligned),
// completing 'bytes' transactions on 'bar'.  The source is streamed once: L2 evict-first.
__device__ __forceinline__ void bulk_g2s(void *dst_smem, const void *src_gmem, uint32_t bytes, uint64_t *bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// Copies the W elements of a lattice row starting at column x (possibly negative or running
// past nx: periodic wrap) into dst: one bulk copy, or two or three pieces at the lattice edge.
// x, nx and W are multiples of 16 / sizeof(real) elements (16-byte granules).
template <class real>
__device__ __forceinline__ void bulk_row_wrapped(real *dst, const real *row, int x, int W, int nx, uint64_t *bar,
                                                 uint64_t policy) {
  constexpr uint32_t es = sizeof(real);
  if (x < 0) {
    bulk_g2s(dst, row + nx + x, (uint32_t)(-x) * es, bar, policy);
    dst += -x;
    W += x;
    x = 0;
  }
  if (x + W > nx) {
    const int n1 = nx - x;
    bulk_g2s(dst, row + x, (uint32_t)n1 * es, bar, policy);
    bulk_g2s(dst + n1, row, (uint32_t)(W - n1) * es, bar, policy);
  } else {
    bulk_g2s(dst, row + x, (uint32_t)W * es, bar, policy);
  }
}


// ---------------------------------------------------------------------------
// Temporal blocking with bulk-copy staging (k_pull2b; 3D tiles and 2D strips): the same two
// fused pull steps as k_pull2 / k_pull2_2d, but the step-t populations are not gathered into
// registers by every thread.  One warp issues asynchronous bulk copies (cp.async.bulk, the TMA
// engine) of whole population rows into a ring of NS shared-memory stages, NS - 1 planes ahead
// of the plane being computed, completed on one mbarrier per stage; the compute threads wait on
// the barrier and read their pulled populations from shared memory.  The global-load latency
// is off the threads' critical path and the ~Q prefetch registers per thread are gone.
//   stage s, population i, row r, column c: stage + ((s Q + i) HY + r) W + c
//     rows r = 0..HY-1 hold lattice rows y0 - 1 - c_y(i) + r (periodic), columns c hold
//     x0 - OFF + c, OFF = 16 / sizeof(real) (16-byte granules; the row is 16-byte aligned),
//     W = TX + 2 OFF: every pull shift of the halo-extended tile is inside the staged row;
//     population i of stage k comes from plane k - c_z(i), the plane it is pulled from.
//   step-(t+1) ring, grouped by c_z (only what step t+2 still reads is kept): c_z = -1 pops
//     of plane k (read at iteration k: 1 slot), c_z = 0 (read at k + 1: 2 slots), c_z = +1
//     (read at k + 2: 3 slots) — (2 UP0 + 4 NUP) planes of the HX x HY tile instead of 3 Q.
// Same collide() as k_pull: equal to single steps up to FMA contraction, i.e. to rounding.
// ---------------------------------------------------------------------------
template <class S, int TX, int TY, class real, int NS>
struct TileB {
  static constexpr int TYE = S::D == 2 ? 1 : TY;      // cells of the tile along y (2D: 1)
  static constexpr int HX = TX + 2, HY = S::D == 2 ? 1 : TY + 2, HW = HX * HY;
  static constexpr int YH = (HY - TYE) / 2;            // halo rows on each side (2D: none)
  static constexpr int THREADS = (HW + 31) / 32 * 32;
  static constexpr int OFF = 16 / (int)sizeof(real), W = TX + 2 * OFF;
  static constexpr int N0 = S::UP0, NU = S::NUP;      // populations with c_z = 0 / +1 (= -1)
  static constexpr int RING = (2 * N0 + 4 * NU) * HW;  // elements
  static constexpr int STAGE = S::Q * HY * W;          // elements per stage
  static constexpr size_t BAR_BYTES = 128;             // NS mbarriers, padded
  static constexpr size_t smem() { return BAR_BYTES + (size_t)(NS * STAGE + RING) * sizeof(real); }
  // ring position of population i (slot of plane k)
  template <int i>
  __device__ static __forceinline__ int ring_at(int k) {
    constexpr int cz = S::mz(i);
    if constexpr (cz < 0) return (i - N0 - NU) * HW;
    else if constexpr (cz == 0) return (NU + (k & 1) * N0 + i) * HW;
    else return (NU + 2 * N0 + ((k + 3) % 3) * NU + (i - N0)) * HW;
  }
};

template <class S, int SPACE, int REG, class real, int RS, int TX, int TY, int MINB, int NS, bool RANGE = false>
__global__ void __launch_bounds__(TileB<S, TX, TY, real, NS>::THREADS, MINB)
    k_pull2b(const real *__restrict__ src, real *__restrict__ dst, const GridParams g, const Rates<real> r,
             const real swe_g, const Force<real> fr) {
  using T = TileB<S, TX, TY, real, NS>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem_raw);
  real *stage = reinterpret_cast<real *>(smem_raw + T::BAR_BYTES);
  real *ring = stage + NS * T::STAGE;
  const int t = threadIdx.x;
  const int x0 = blockIdx.x * TX, y0 = S::D == 2 ? 0 : blockIdx.y * TY;
  const int n = g.nzl;
  // step t+1 cell of this thread on the halo-extended tile; step t+2 cell (tile interior)
  const bool act1 = t < T::HW;
  const int hx = t % T::HX, hy = t / T::HX;
  const bool act2 = t < TX * T::TYE;
  const int ix = t % TX, iy = t / TX;
  // output planes [p0, p1) of this CTA's chunk (blockIdx.z in 3D, blockIdx.y in 2D), as k_pull2
  const int zb = RANGE ? g.zbegin : 0, zn = RANGE ? g.zcount : n;
  const int chunk = S::D == 2 ? blockIdx.y : blockIdx.z, nchunk = S::D == 2 ? gridDim.y : gridDim.z;
  const int p0 = zb + (int)((long long)zn * chunk / nchunk);
  const int p1 = zb + (int)((long long)zn * (chunk + 1) / nchunk);
  auto zw = [&](int k) {
    if constexpr (RANGE) return k;
    else return wrapi(k, n);
  };
  const int nit = p1 - p0 + 2;  // step-(t+1) planes k = p0 - 1 .. p1
  // producer: lanes r < HY of warp 0 copy row r of every population of plane k into stage s
  const uint64_t pol = l2_policy_evict_first();
  auto issue = [&](int k, int s) {
    if (t == 0) mbar_arrive_expect_tx(&bar[s], (uint32_t)(T::STAGE * sizeof(real)));
    if (t < T::HY) {
      sfor<S::Q>([&](auto i) {
        constexpr int cy = S::my(i), cz = S::mz(i);
        const int zz = zw(k - cz) + 1;
        const int y = S::D == 2 ? 0 : wrapi(y0 - 1 - cy + t, g.ny);
        const real *row = src + (long long)zz * g.plane + (long long)i * g.pop + (long long)y * g.pitch;
        real *d = stage + ((s * S::Q + i) * T::HY + t) * T::W;
        bulk_row_wrapped(d, row, x0 - T::OFF, T::W, g.nx, &bar[s], pol);
      });
    }
  };
  if (t == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&bar[s], 1);
    mbar_fence_init();
  }
  __syncthreads();
  // iterations it < 0 only fill the first NS - 1 stages (one call site: the copy code inlines)
  for (int it = 1 - NS; it < nit; ++it) {
    const int k = p0 - 1 + it;
    // refill the stage read in the previous iteration (all its readers passed two barriers)
    if (it + NS - 1 < nit) issue(k + NS - 1, (it + NS - 1) % NS);
    if (it < 0) continue;
    if (act1) {
      const int s = it % NS;
      mbar_wait(&bar[s], (uint32_t)((it / NS) & 1));
      real f[S::Q];
      const real *st = stage + s * T::STAGE;
      sfor<S::Q>([&](auto i) {
        constexpr int cx = S::mx(i);
        f[i] = st[(i * T::HY + hy) * T::W + hx + T::OFF - 1 - cx];
      });
      collide<S, SPACE, REG, real, RS>(f, r, swe_g, fr);
      sfor<S::Q>([&](auto i) { ring[T::template ring_at<i>(k) + t] = f[i]; });
    }
    __syncthreads();
    if (k >= p0 + 1 && act2) {
      const int p = k - 1;  // plane of step t+2
      real f[S::Q];
      sfor<S::Q>([&](auto i) {
        constexpr int cx = S::mx(i), cy = S::my(i), cz = S::mz(i);
        f[i] = ring[T::template ring_at<i>(p - cz) + (iy + T::YH - cy) * T::HX + (ix + 1 - cx)];
      });
      collide<S, SPACE, REG, real, RS>(f, r, swe_g, fr);
      const long long own = (long long)(p + 1) * g.plane + (long long)(y0 + iy) * g.pitch + (x0 + ix);
      sfor<S::Q>([&](auto i) { dst[own + (long long)i * g.pop] = f[i]; });
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Temporal blocking with two concurrent thread groups (k_pull2w, 3D): the same two fused pull
// steps as k_pull2, but step t+1 and step t+2 run at the same time on different warps instead
// of one after the other on the same threads.  In iteration k, group A (the HX x HY
// halo-extended tile, one cell per thread) computes step t+1 of plane k from HBM into the
// shared-memory ring, while group B (the TX x TY interior) computes step t+2 of plane k - 2
// from the ring planes k - 3 .. k - 1 finished in earlier iterations and stores it — one
// barrier per plane, and no warp waits through the other step's collisions (in k_pull2 the
// 2 halo warps of a 16 x 8 tile idle during step t+2).  Each thread runs one collision per
// plane, so the register budget is that of one collision: 2 CTAs of 10 warps per SM instead of
// 2 CTAs of 6.  Ring slots by c_z (written at iteration j, read at j+1 / j+2 / j+3): c_z = -1:
// 2 slots, c_z = 0: 3, c_z = +1: 4 — (3 UP0 + 6 NUP) planes of the tile (D3Q19: 57 = 3 Q).
// ---------------------------------------------------------------------------
// CTA-wide barrier reached from different call sites by warp-uniform thread groups (the
// non-.aligned barrier.sync; __syncthreads is barrier.sync.aligned, one call site for all)
__device__ __forceinline__ void cta_barrier(int nthreads) {
  asm volatile("barrier.sync 0, %0;" ::"r"(nthreads) : "memory");
}

template <class S, int TX, int TY>
struct TileW {
  static constexpr int HX = TX + 2, HY = TY + 2, HW = HX * HY;
  static constexpr int TA = (HW + 31) / 32 * 32;      // group A threads (step t+1)
  static constexpr int TB = (TX * TY + 31) / 32 * 32; // group B threads (step t+2)
  static constexpr int THREADS = TA + TB;
  static constexpr int N0 = S::UP0, NU = S::NUP;
  static constexpr int RING = (3 * N0 + 6 * NU) * HW;  // elements
  template <class real>
  static constexpr size_t smem() { return (size_t)RING * sizeof(real); }
  template <int i>
  __device__ static __forceinline__ int ring_at(int k) {
    constexpr int cz = S::mz(i);
    if constexpr (cz < 0) return ((k & 1) * NU + (i - N0 - NU)) * HW;
    else if constexpr (cz == 0) return (2 * NU + ((k + 3) % 3) * N0 + i) * HW;
    else return (2 * NU + 3 * N0 + (k & 3) * NU + (i - N0)) * HW;
  }
};

template <class S, int SPACE, int REG, class real, int RS, int TX, int TY, int MINB, bool PF, bool RANGE = false>
__global__ void __launch_bounds__(TileW<S, TX, TY>::THREADS, MINB)
    k_pull2w(const real *__restrict__ src, real *__restrict__ dst, const GridParams g, const Rates<real> r,
             const real swe_g, const Force<real> fr) {
  static_assert(S::D == 3, "3D tiles");
  using T = TileW<S, TX, TY>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  real *ring = reinterpret_cast<real *>(smem_raw);
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const int n = g.nzl;
  const int zb = RANGE ? g.zbegin : 0, zn = RANGE ? g.zcount : n;
  const int p0 = zb + (int)((long long)zn * blockIdx.z / gridDim.z);
  const int p1 = zb + (int)((long long)zn * (blockIdx.z + 1) / gridDim.z);
  auto zw = [&](int k) {
    if constexpr (RANGE) return k;
    else return wrapi(k, n);
  };
  const bool groupA = threadIdx.x < T::TA;
  if (groupA) {
    // step t+1 on the halo-extended tile, planes k = p0 - 1 .. p1 (iterations p0 - 1 .. p1 + 1)
    const int t = threadIdx.x;
    const bool act = t < T::HW;
    const int hx = t % T::HX, hy = t / T::HX;
    const int gx = wrapi(x0 - 1 + hx, g.nx), gy = wrapi(y0 - 1 + hy, g.ny);
    int xs[3], ys[3];
#pragma unroll
    for (int s = -1; s <= 1; ++s) {
      xs[s + 1] = wrapi(gx + s, g.nx);
      ys[s + 1] = wrapi(gy + s, g.ny) * g.pitch;
    }
    auto load = [&](int k, real(&f)[S::Q]) {
      const int zc = zw(k);
      long long zo[3];
#pragma unroll
      for (int s = -1; s <= 1; ++s) zo[s + 1] = (long long)(zw(zc + s) + 1) * g.plane;
      sfor<S::Q>([&](auto i) {
        constexpr int cx = S::mx(i), cy = S::my(i), cz = S::mz(i);
        f[i] = ld_nc(src + zo[1 - cz] + (long long)i * g.pop + ys[1 - cy] + xs[1 - cx]);
      });
    };
    real fn[PF ? S::Q : 1];
    if constexpr (PF) {
      if (act) load(p0 - 1, fn);
    }
    for (int k = p0 - 1; k <= p1 + 1; ++k) {
      if (act && k <= p1) {
        real f[S::Q];
        if constexpr (PF) {
          sfor<S::Q>([&](auto i) { f[i] = fn[i]; });
          if (k < p1) load(k + 1, fn);
        } else {
          load(k, f);
        }
        collide<S, SPACE, REG, real, RS>(f, r, swe_g, fr);
        sfor<S::Q>([&](auto i) { ring[T::template ring_at<i>(k) + t] = f[i]; });
      }
      cta_barrier(T::THREADS);
    }
  } else {
    // step t+2 on the tile interior, plane p = k - 2 in iteration k (p = p0 .. p1 - 1)
    const int t = threadIdx.x - T::TA;
    const bool act = t < TX * TY;
    const int ix = t % TX, iy = t / TX;
    for (int k = p0 - 1; k <= p1 + 1; ++k) {
      const int p = k - 2;
      if (act && p >= p0) {
        real f[S::Q];
        sfor<S::Q>([&](auto i) {
          constexpr int cx = S::mx(i), cy = S::my(i), cz = S::mz(i);
          f[i] = ring[T::template ring_at<i>(p - cz) + (iy + 1 - cy) * T::HX + (ix + 1 - cx)];
        });
        collide<S, SPACE, REG, real, RS>(f, r, swe_g, fr);
        const long long own = (long long)(p + 1) * g.plane + (long long)(y0 + iy) * g.pitch + (x0 + ix);
        sfor<S::Q>([&](auto i) { dst[own + (long long)i * g.pop] = f[i]; });
      }
      cta_barrier(T::THREADS);
    }
  }
}

}  // namespace lbm
