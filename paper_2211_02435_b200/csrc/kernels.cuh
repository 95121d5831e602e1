// kernels.cuh — the fused stream–collide kernels and their small helpers.
//
// Device population grid layout (SoA):
//   element (zz, i, y, x) at  zz * plane + i * pop + y * pitch + x
//   zz = local slab plane + 1 (zz = 0 and zz = nzl + 1 are ghost planes),
//   pop = ny * pitch, plane = q * pop, pitch = nx rounded up to 32 elements.
// With the slab axis outermost and the slab-crossing populations contiguous in i
// (include/lbm.h ordering), every halo block is one contiguous range.
//
// Streaming patterns:
//   PULL     f_i(x) = src(x - xi_i, i)  -> collide -> dst(x, i)            (two grids)
//   AA_ODD   state A -> B: f_i(x) = mem(x - xi_i, opp i) -> collide -> mem(x + xi_i, i)
//   AA_EVEN  state B -> A: f_i(x) = mem(x, i)          -> collide -> mem(x, opp i)
//   (state A: mem(x, opp i) = f*_i(x);  state B: mem(x + xi_i, i) = f*_i(x); reading R11).
// Each cell reads and writes the same q slots in both AA parities, so the in-place
// update is race-free without synchronisation.
#pragma once
#include <cooperative_groups.h>

#include "collide.cuh"
#include "tma.cuh"

namespace lbm {

enum { PAT_PULL = 0, PAT_AA_EVEN = 1, PAT_AA_ODD = 2 };
constexpr int BLOCK_X = 128;

struct GridParams {
  long long plane;  // elements per storage plane = q * ny * pitch
  long long pop;    // elements per population row block = ny * pitch
  int pitch;
  int nx, ny, nzl, nzg, z0;  // local view: x, y, slab axis (nzl local planes from global z0)
  int zbegin;                // first local plane of this launch
  int zcount = 0;            // two-step sweeps: output planes [zbegin, zbegin + zcount) (0: all)
  int wrapz;                 // single rank: periodic wrap along the slab axis by index
  int bcmask;                // bit (2 * axis + side): no-slip face (axis 0 x, 1 y, 2 slab)
  // fused halo push (lbm_step_peer): ghost plane of the lower / upper neighbour's next grid
  // (peer memory over NVLink, or a same-device context); null: no push
  void *peer_lo = nullptr, *peer_hi = nullptr;
  int peer_fence = 0;  // per-thread system-scope fence after the pushes (runtime.cu peer_fence)
};

// Stores the slab-crossing populations of a boundary plane into the neighbours' ghost
// planes: plane 0's downward (slab component -1) populations to the lower neighbour's top
// ghost plane, plane nzl-1's upward ones to the upper neighbour's bottom ghost plane — the
// values the neighbours' next pull step gathers (eq:LbStreaming across the cut).  They are
// released before the completion flag (k_peer_signal) by peer_release_cta (default: one
// system-scope fence per CTA after a CTA barrier), or per thread (g.peer_fence == 2).
template <class S, class real>
__device__ __forceinline__ void peer_push(const GridParams &g, int zl, long long in_plane, const real *f) {
  if (zl == 0 && g.peer_lo) {
    real *p = static_cast<real *>(g.peer_lo) + in_plane;
    sfor<S::Q>([&](auto i) {
      if constexpr (S::mz(i) < 0) p[(long long)i * g.pop] = f[i];
    });
    if (g.peer_fence == 2) __threadfence_system();
  }
  if (zl == g.nzl - 1 && g.peer_hi) {
    real *p = static_cast<real *>(g.peer_hi) + in_plane;
    sfor<S::Q>([&](auto i) {
      if constexpr (S::mz(i) > 0) p[(long long)i * g.pop] = f[i];
    });
    if (g.peer_fence == 2) __threadfence_system();
  }
}

// Producer-side release of a boundary kernel's stores into peer memory (g.peer_fence == 1,
// the default): the CTA barrier orders every thread's remote stores before thread 0's
// system-scope fence (fences are cumulative over the writes their thread has observed), so
// the stores are visible system-wide before the kernel completes and k_peer_signal publishes
// the phase — an ordering that does not rely on kernel completion alone.  Every thread of
// the CTA must reach it (no early return in the PEER kernels).
__device__ __forceinline__ void peer_release_cta(const int mode) {
  if (mode == 1) {
    __syncthreads();
    if (threadIdx.x == 0) __threadfence_system();
  }
}

__device__ __forceinline__ int wrapi(int v, int n) { return v < 0 ? v + n : (v >= n ? v - n : v); }

template <class real>
__device__ __forceinline__ real ld_nc(const real *p) { return __ldg(p); }

// ---------------------------------------------------------------------------
// the fused stream–collide kernel (pull, optionally with half-way bounce-back)
// ---------------------------------------------------------------------------
// PEER: the boundary-plane variant of lbm_step_peer that also pushes the slab-crossing
// populations into the neighbours' ghost planes (a separate instantiation: the bulk kernel
// keeps its register budget).
template <class S, int SPACE, int REG, class real, bool BB, int RS, bool PEER>
__device__ __forceinline__ void pull_cell(const real *__restrict__ src, real *__restrict__ dst, const GridParams &g,
                                          const Rates<real> &r, const real swe_g, const Force<real> &fr,
                                          const int x) {
  const int y = blockIdx.y;
  const int zl = g.zbegin + blockIdx.z;

  // source coordinates for offsets s = -1, 0, +1 (index s + 1)
  int xs[3], ys[3];
  long long zo[3];
  bool bx[3] = {false, false, false}, by[3] = {false, false, false}, bz[3] = {false, false, false};
#pragma unroll
  for (int s = -1; s <= 1; ++s) {
    const int xv = x + s, yv = y + s, zv = zl + s;
    xs[s + 1] = wrapi(xv, g.nx);
    ys[s + 1] = wrapi(yv, g.ny) * g.pitch;
    const int zz = g.wrapz ? wrapi(zv, g.nzl) + 1 : zv + 1;
    zo[s + 1] = (long long)zz * g.plane;
    if constexpr (BB) {
      bx[s + 1] = (xv < 0 && (g.bcmask & 1)) || (xv >= g.nx && (g.bcmask & 2));
      by[s + 1] = (yv < 0 && (g.bcmask & 4)) || (yv >= g.ny && (g.bcmask & 8));
      const int zgv = g.z0 + zv;
      bz[s + 1] = (zgv < 0 && (g.bcmask & 16)) || (zgv >= g.nzg && (g.bcmask & 32));
    }
  }
  const long long own = (long long)(zl + 1) * g.plane + (long long)y * g.pitch + x;

  real f[S::Q];
  sfor<S::Q>([&](auto i) {
    constexpr int cx = S::mx(i), cy = S::my(i), cz = S::mz(i);
    const long long a = zo[1 - cz] + (long long)i * g.pop + ys[1 - cy] + xs[1 - cx];
    if constexpr (BB) {
      const bool bb = bx[1 - cx] || by[1 - cy] || bz[1 - cz];
      // half-way bounce-back: f_i(x) = f*_{opp i}(x)   (reading R18)
      const long long ab = own + (long long)S::opp(i) * g.pop;
      f[i] = ld_nc(src + (bb ? ab : a));
    } else {
      f[i] = ld_nc(src + a);
    }
  });

  collide<S, SPACE, REG, real, RS>(f, r, swe_g, fr);

  sfor<S::Q>([&](auto i) { dst[own + (long long)i * g.pop] = f[i]; });
  if constexpr (PEER) peer_push<S>(g, zl, (long long)y * g.pitch + x, f);
}

template <class S, int SPACE, int REG, class real, bool BB, int RS = RS_GENERAL, bool PEER = false>
__global__ void __launch_bounds__(BLOCK_X) k_pull(const real *__restrict__ src, real *__restrict__ dst,
                                                   const GridParams g, const Rates<real> r, const real swe_g,
                                                   const Force<real> fr) {
  const int x = blockIdx.x * BLOCK_X + threadIdx.x;
  if constexpr (PEER) {
    if (x < g.nx) pull_cell<S, SPACE, REG, real, BB, RS, PEER>(src, dst, g, r, swe_g, fr, x);
    peer_release_cta(g.peer_fence);
  } else {
    if (x < g.nx) pull_cell<S, SPACE, REG, real, BB, RS, PEER>(src, dst, g, r, swe_g, fr, x);
  }
}


// ---------------------------------------------------------------------------
// AA pattern: in-place.  BB (single rank): half-way bounce-back on the no-slip faces of
// g.bcmask (reading R18).  The odd step reads f_i(x) = f*_opp(x) from mem(x, i) when x - xi_i
// is beyond a wall, and writes f*_i(x) to mem(x, opp i) when x + xi_i is — the slot the next
// (even) step reads as the bounced f_opp(x).  Both slots belong to cell x alone (no other cell
// maps onto them), so the update stays race-free; the even step needs no change.
// ---------------------------------------------------------------------------
template <class S>
struct Walls {
  bool x[3], y[3], z[3];  // offset s = -1, 0, +1 (index s + 1) lies beyond a no-slip face
  __device__ __forceinline__ Walls(const GridParams &g, int x0, int y0, int zl) {
#pragma unroll
    for (int s = -1; s <= 1; ++s) {
      const int xv = x0 + s, yv = y0 + s, zgv = g.z0 + zl + s;
      x[s + 1] = (xv < 0 && (g.bcmask & 1)) || (xv >= g.nx && (g.bcmask & 2));
      y[s + 1] = (yv < 0 && (g.bcmask & 4)) || (yv >= g.ny && (g.bcmask & 8));
      z[s + 1] = (zgv < 0 && (g.bcmask & 16)) || (zgv >= g.nzg && (g.bcmask & 32));
    }
  }
  // the neighbour x + (cx, cy, cz) lies beyond a wall (crossing any wall axis bounces)
  __device__ __forceinline__ bool beyond(int cx, int cy, int cz) const {
    return x[1 + cx] || y[1 + cy] || z[1 + cz];
  }
};
// The odd kernel holds 27 gather and 27 scatter addresses across the collision; capping it
// at 5 blocks/SM (96 registers, 4 B spill) beats 123 registers at 4 blocks (+3 %, B200).
// PEER (odd pattern, boundary planes of lbm_step_peer): the slab-crossing accesses go straight
// to the neighbours' boundary planes in peer memory (g.peer_lo: the lower neighbour's last
// plane, g.peer_hi: the upper neighbour's first plane) instead of the ghost planes — the
// AA odd step is race-free on the global lattice, so ranks need no exchange, only the
// per-step completion flags.
// the odd AA step of a boundary-plane cell with the neighbours' planes in peer memory
template <class S, int SPACE, int REG, class real, int RS>
__device__ __forceinline__ void aa_peer_cell(real *mem, const GridParams &g, const Rates<real> &r, const real swe_g,
                                             const Force<real> &fr, const int x) {
  const int y = blockIdx.y;
  const int zl = g.zbegin + blockIdx.z;
  real f[S::Q];
  int xs[3], ys[3];
  real *zb[3];
#pragma unroll
  for (int s = -1; s <= 1; ++s) {
    xs[s + 1] = wrapi(x + s, g.nx);
    ys[s + 1] = wrapi(y + s, g.ny) * g.pitch;
    const int zv = zl + s;
    zb[s + 1] = zv < 0 ? static_cast<real *>(g.peer_lo)
                       : (zv >= g.nzl ? static_cast<real *>(g.peer_hi) : mem + (long long)(zv + 1) * g.plane);
  }
  sfor<S::Q>([&](auto i) {
    constexpr int cx = S::mx(i), cy = S::my(i), cz = S::mz(i);
    f[i] = zb[1 - cz][(long long)S::opp(i) * g.pop + ys[1 - cy] + xs[1 - cx]];
  });
  collide<S, SPACE, REG, real, RS>(f, r, swe_g, fr);
  sfor<S::Q>([&](auto i) {
    constexpr int cx = S::mx(i), cy = S::my(i), cz = S::mz(i);
    zb[1 + cz][(long long)i * g.pop + ys[1 + cy] + xs[1 + cx]] = f[i];
  });
}

template <class S, int SPACE, int REG, class real, int PAT, int RS = RS_GENERAL, bool PEER = false, bool BB = false>
__global__ void __launch_bounds__(BLOCK_X, (PAT == PAT_AA_ODD ? 5 : 1))
    k_aa(real *mem, const GridParams g, const Rates<real> r, const real swe_g, const Force<real> fr) {
  const int x = blockIdx.x * BLOCK_X + threadIdx.x;
  if constexpr (PEER) {  // every thread reaches the CTA release (no early return)
    if (x < g.nx) aa_peer_cell<S, SPACE, REG, real, RS>(mem, g, r, swe_g, fr, x);
    peer_release_cta(g.peer_fence);
    return;
  }
  if (x >= g.nx) return;
  const int y = blockIdx.y;
  const int zl = g.zbegin + blockIdx.z;
  real f[S::Q];
  if constexpr (PAT == PAT_AA_EVEN) {
    const long long own = (long long)(zl + 1) * g.plane + (long long)y * g.pitch + x;
    // read-only path is safe in place: every slot is read, then written, by the same thread
    sfor<S::Q>([&](auto i) { f[i] = ld_nc(mem + own + (long long)i * g.pop); });
    collide<S, SPACE, REG, real, RS>(f, r, swe_g, fr);
    sfor<S::Q>([&](auto i) { mem[own + (long long)S::opp(i) * g.pop] = f[i]; });
  } else {
    int xs[3], ys[3];
    long long zo[3];
#pragma unroll
    for (int s = -1; s <= 1; ++s) {
      xs[s + 1] = wrapi(x + s, g.nx);
      ys[s + 1] = wrapi(y + s, g.ny) * g.pitch;
      // single rank: periodic by index; several ranks: the ghost planes (filled before
      // and returned after the odd step, distributed.py)
      zo[s + 1] = (long long)((g.wrapz ? wrapi(zl + s, g.nzl) : zl + s) + 1) * g.plane;
    }
    if constexpr (BB) {
      const Walls<S> w(g, x, y, zl);
      const long long own = (long long)(zl + 1) * g.plane + (long long)y * g.pitch + x;
      // read f_i(x) = mem(x - xi_i, opp i), or f*_opp(x) = mem(x, i) from beyond a wall
      sfor<S::Q>([&](auto i) {
        constexpr int cx = S::mx(i), cy = S::my(i), cz = S::mz(i);
        const long long a = zo[1 - cz] + (long long)S::opp(i) * g.pop + ys[1 - cy] + xs[1 - cx];
        f[i] = ld_nc(mem + (w.beyond(-cx, -cy, -cz) ? own + (long long)i * g.pop : a));
      });
      collide<S, SPACE, REG, real, RS>(f, r, swe_g, fr);
      // write f*_i(x) to mem(x + xi_i, i), or to mem(x, opp i) towards a wall
      sfor<S::Q>([&](auto i) {
        constexpr int cx = S::mx(i), cy = S::my(i), cz = S::mz(i);
        const long long a = zo[1 + cz] + (long long)i * g.pop + ys[1 + cy] + xs[1 + cx];
        mem[w.beyond(cx, cy, cz) ? own + (long long)S::opp(i) * g.pop : a] = f[i];
      });
    } else {
      // read f_i(x) = mem(x - xi_i, opp i)
      sfor<S::Q>([&](auto i) {
        constexpr int cx = S::mx(i), cy = S::my(i), cz = S::mz(i);
        f[i] = ld_nc(mem + zo[1 - cz] + (long long)S::opp(i) * g.pop + ys[1 - cy] + xs[1 - cx]);
      });
      collide<S, SPACE, REG, real, RS>(f, r, swe_g, fr);
      // write f*_i(x) to mem(x + xi_i, i)
      sfor<S::Q>([&](auto i) {
        constexpr int cx = S::mx(i), cy = S::my(i), cz = S::mz(i);
        mem[zo[1 + cz] + (long long)i * g.pop + ys[1 + cy] + xs[1 + cx]] = f[i];
      });
    }
  }
}

// ---------------------------------------------------------------------------
// Esoteric Pull (Lehmann 2022, cited at PAPER.md:862; single rank, periodic): in place,
// one kernel shape every step, half of each opposite pair (i, opp i) exchanged with the
// neighbour x + xi_i, i the "first" member (i < opp i):
//   odd  (state E -> O): f_i = mem(x, i),     f_opp = mem(x + xi_i, opp)  -> collide ->
//                        mem(x + xi_i, opp) = f*_i, mem(x, i) = f*_opp
//   even (state O -> E): f_i = mem(x, opp),   f_opp = mem(x + xi_i, i)    -> collide ->
//                        mem(x + xi_i, i) = f*_i,   mem(x, opp) = f*_opp
// (state E: mem(x + xi_i, i) = f*_i(x), mem(x, opp) = f*_opp(x); state O swaps the slots;
// every slot is read and written by one cell only: race-free in place.)
// Esoteric Push (same source; reading R32): the mirror image — the LEAD member of each pair,
// the one stored at its streaming destination x + xi (pushed by the write) while the other is
// pulled by the read, is the second member opp i (i > opp i) instead of the first, so a cell
// touches its negative half-neighbourhood x - xi_i.  Same kernel with `lead` mirrored.
// ---------------------------------------------------------------------------
template <class S>
__host__ __device__ constexpr bool first_of_pair(int i) {
  return i != 0 && i < S::opp(i);
}
// the lead member of a pair: Esoteric Pull the first, Esoteric Push (MIRROR) the second
template <class S, bool MIRROR>
__host__ __device__ constexpr bool eso_lead(int i) {
  return MIRROR ? (i != 0 && i > S::opp(i)) : first_of_pair<S>(i);
}

enum { PAT_ESO_EVEN = 3, PAT_ESO_ODD = 4 };
enum { PAT_ESOP_EVEN = 7, PAT_ESOP_ODD = 8 };  // Esoteric Push

template <class S, int SPACE, int REG, class real, int PAT, int RS = RS_GENERAL>
__global__ void __launch_bounds__(BLOCK_X)
    k_eso(real *mem, const GridParams g, const Rates<real> r, const real swe_g, const Force<real> fr) {
  const int x = blockIdx.x * BLOCK_X + threadIdx.x;
  if (x >= g.nx) return;
  const int y = blockIdx.y;
  const int zl = g.zbegin + blockIdx.z;
  constexpr bool odd = (PAT == PAT_ESO_ODD || PAT == PAT_ESOP_ODD);
  constexpr bool mirror = (PAT == PAT_ESOP_ODD || PAT == PAT_ESOP_EVEN);
  const long long own = (long long)(zl + 1) * g.plane + (long long)y * g.pitch + x;
  int xs[3], ys[3];
  long long zo[3];
#pragma unroll
  for (int s = -1; s <= 1; ++s) {
    xs[s + 1] = wrapi(x + s, g.nx);
    ys[s + 1] = wrapi(y + s, g.ny) * g.pitch;
    zo[s + 1] = (long long)(wrapi(zl + s, g.nzl) + 1) * g.plane;
  }
  real f[S::Q];
  f[0] = ld_nc(mem + own);
  sfor<S::Q>([&](auto i) {
    if constexpr (eso_lead<S, mirror>(i)) {
      constexpr int o = S::opp(i), cx = S::mx(i), cy = S::my(i), cz = S::mz(i);
      const long long nb = zo[1 + cz] + ys[1 + cy] + xs[1 + cx];  // cell x + xi_i
      f[i] = ld_nc(mem + own + (long long)(odd ? i : o) * g.pop);
      f[o] = ld_nc(mem + nb + (long long)(odd ? o : i) * g.pop);
    }
  });
  collide<S, SPACE, REG, real, RS>(f, r, swe_g, fr);
  mem[own] = f[0];
  sfor<S::Q>([&](auto i) {
    if constexpr (eso_lead<S, mirror>(i)) {
      constexpr int o = S::opp(i), cx = S::mx(i), cy = S::my(i), cz = S::mz(i);
      const long long nb = zo[1 + cz] + ys[1 + cy] + xs[1 + cx];
      mem[nb + (long long)(odd ? o : i) * g.pop] = f[i];
      mem[own + (long long)(odd ? i : o) * g.pop] = f[o];
    }
  });
}

// ---------------------------------------------------------------------------
// Esoteric Twist (Geier & Schoenherr 2017, cited at PAPER.md:861; reading R28; single rank,
// periodic): in place, every cell touches only the 2^d cells of its positive octant
// x + o, o in {0, 1}^d.  With o+(i) = max(xi_i, 0) and o-(i) = max(-xi_i, 0) per axis:
//   TW0 (state T0 -> T1): f_i = mem(x + o-(i), i)      -> collide -> mem(x + o+(i), opp i)
//   TW1 (state T1 -> T0): f_i = mem(x + o-(i), opp i)  -> collide -> mem(x + o+(i), i)
// (state T0: f*_i(x) at mem(x + o+(i), i); T1: at mem(x + o+(i), opp i).  The slots a cell
// reads are the slots it writes, o+(opp i) = o-(i): race-free in place.  x - xi_i + o+(i) =
// x + o-(i) makes the reads the pulls of eq:LbStreaming.)
// ---------------------------------------------------------------------------
enum { PAT_TW0 = 5, PAT_TW1 = 6 };

template <class S, int SPACE, int REG, class real, int PAT, int RS = RS_GENERAL>
__global__ void __launch_bounds__(BLOCK_X)
    k_twist(real *mem, const GridParams g, const Rates<real> r, const real swe_g, const Force<real> fr) {
  const int x = blockIdx.x * BLOCK_X + threadIdx.x;
  if (x >= g.nx) return;
  const int y = blockIdx.y;
  const int zl = g.zbegin + blockIdx.z;
  constexpr bool t0 = (PAT == PAT_TW0);
  // offsets 0 / +1 of the octant along each axis
  const int xs[2] = {x, wrapi(x + 1, g.nx)};
  const long long ys[2] = {(long long)y * g.pitch, (long long)wrapi(y + 1, g.ny) * g.pitch};
  const long long zo[2] = {(long long)(zl + 1) * g.plane, (long long)(wrapi(zl + 1, g.nzl) + 1) * g.plane};
  real f[S::Q];
  sfor<S::Q>([&](auto i) {
    constexpr int cx = S::mx(i), cy = S::my(i), cz = S::mz(i);
    constexpr int slot = t0 ? int(i) : S::opp(i);
    f[i] = ld_nc(mem + zo[cz < 0] + (long long)slot * g.pop + ys[cy < 0] + xs[cx < 0]);
  });
  collide<S, SPACE, REG, real, RS>(f, r, swe_g, fr);
  sfor<S::Q>([&](auto i) {
    constexpr int cx = S::mx(i), cy = S::my(i), cz = S::mz(i);
    constexpr int slot = t0 ? S::opp(i) : int(i);
    mem[zo[cz > 0] + (long long)slot * g.pop + ys[cy > 0] + xs[cx > 0]] = f[i];
  });
}

// ---------------------------------------------------------------------------
// helpers: init from macroscopic fields, canonical get/set, macroscopic moments,
// collision-only test kernel, finiteness probe.  'pat' = lbm_streaming (0 pull, 1 AA,
// 2 Esoteric Pull, 3 Esoteric Twist, 4 Esoteric Push); 'state' for AA: 0 = A, 1 = B; for
// Esoteric Pull / Push: 0 = E, 1 = O; for Esoteric Twist: 0 = T0, 1 = T1.
// ---------------------------------------------------------------------------
template <class S>
struct Canon {
  // element offset of the canonical post-collision value f*_i(x) in the grid
  template <int i>
  __device__ static __forceinline__ long long at(const GridParams &g, int x, int y, int zl, int pat, int state) {
    const long long own = (long long)(zl + 1) * g.plane + (long long)y * g.pitch + x;
    if (pat == 0) return own + (long long)i * g.pop;
    if (pat == 3) {  // Esoteric Twist: mem(x + o+(i), i) in state T0, slot opp i in T1
      constexpr int cx = S::mx(i), cy = S::my(i), cz = S::mz(i);
      const int xx = cx > 0 ? wrapi(x + 1, g.nx) : x, yy = cy > 0 ? wrapi(y + 1, g.ny) : y;
      const int zz = cz > 0 ? wrapi(zl + 1, g.nzl) : zl;
      return (long long)(zz + 1) * g.plane + (long long)yy * g.pitch + xx +
             (long long)(state == 0 ? int(i) : S::opp(i)) * g.pop;
    }
    const int xx = wrapi(x + S::mx(i), g.nx), yy = wrapi(y + S::my(i), g.ny);
    const int zz = g.wrapz ? wrapi(zl + S::mz(i), g.nzl) : zl + S::mz(i);  // multi-rank: ghost plane
    const long long nb = (long long)(zz + 1) * g.plane + (long long)yy * g.pitch + xx;  // cell x + xi_i
    if (pat == 1) {
      if (state == 0) return own + (long long)S::opp(i) * g.pop;
      // state B with walls (single rank): populations headed beyond a wall sit in mem(x, opp i)
      if (g.bcmask && Walls<S>(g, x, y, zl).beyond(S::mx(i), S::my(i), S::mz(i)))
        return own + (long long)S::opp(i) * g.pop;
      return nb + (long long)i * g.pop;
    }
    if constexpr (i == 0) return own;
    const int slot = state == 0 ? i : S::opp(i);
    const bool lead = pat == 4 ? eso_lead<S, true>(i) : first_of_pair<S>(i);  // Esoteric Push / Pull
    return (lead ? nb : own) + (long long)slot * g.pop;
  }
};

// host staging layouts: f[i][z][y][x] (fp64), rho[z][y][x], u[d][z][y][x]
template <class S, int SPACE, int REG, class real, bool DISC = false>
__global__ void k_init(real *mem, const GridParams g, int aa, const double *__restrict__ rho,
                       const double *__restrict__ u, real swe_g) {
  const int x = blockIdx.x * BLOCK_X + threadIdx.x;
  if (x >= g.nx) return;
  const int y = blockIdx.y, zl = blockIdx.z;
  const long long cell = ((long long)zl * g.ny + y) * g.nx + x;
  const long long ncell = (long long)g.nzl * g.ny * g.nx;
  const real r = (real)rho[cell];
  const real ux = (real)u[cell];
  real uy, uz;
  if constexpr (S::D == 3) {
    uy = (real)u[ncell + cell];
    uz = (real)u[2 * ncell + cell];
  } else {
    uy = (real)u[ncell + cell];
    uz = real(0);
  }
  real f[S::Q];
  equilibrium<S, SPACE, REG, real, DISC>(f, r, ux, uy, uz, swe_g);
  // post-collision state at t = 0 written in state A (AA) or the current grid (pull)
  sfor<S::Q>([&](auto i) { mem[Canon<S>::template at<i>(g, x, y, zl, aa, 0)] = f[i]; });
}

template <class S, class real>
__global__ void k_get_populations(const real *mem, const GridParams g, int aa, int state, double *__restrict__ out) {
  const int x = blockIdx.x * BLOCK_X + threadIdx.x;
  if (x >= g.nx) return;
  const int y = blockIdx.y, zl = blockIdx.z;
  const long long cell = ((long long)zl * g.ny + y) * g.nx + x;
  const long long ncell = (long long)g.nzl * g.ny * g.nx;
  sfor<S::Q>([&](auto i) { out[i * ncell + cell] = (double)mem[Canon<S>::template at<i>(g, x, y, zl, aa, state)]; });
}

template <class S, class real>
__global__ void k_set_populations(real *mem, const GridParams g, int aa, const double *__restrict__ in) {
  const int x = blockIdx.x * BLOCK_X + threadIdx.x;
  if (x >= g.nx) return;
  const int y = blockIdx.y, zl = blockIdx.z;
  const long long cell = ((long long)zl * g.ny + y) * g.nx + x;
  const long long ncell = (long long)g.nzl * g.ny * g.nx;
  sfor<S::Q>([&](auto i) { mem[Canon<S>::template at<i>(g, x, y, zl, aa, 0)] = (real)in[i * ncell + cell]; });
}

// rho = rho0 + sum df (zc) or sum f; u = (sum f xi + dj) / rho;
// dj = -F/2 for the post-collision state of a forced method (reading R23), else 0
template <class S, class real>
__global__ void k_macroscopic(const real *mem, const GridParams g, int aa, int state, int zc,
                              double *__restrict__ rho, double *__restrict__ u, const double3 dj) {
  const int x = blockIdx.x * BLOCK_X + threadIdx.x;
  if (x >= g.nx) return;
  const int y = blockIdx.y, zl = blockIdx.z;
  const long long cell = ((long long)zl * g.ny + y) * g.nx + x;
  const long long ncell = (long long)g.nzl * g.ny * g.nx;
  double s = 0, jx = 0, jy = 0, jz = 0;
  sfor<S::Q>([&](auto i) {
    const double v = (double)mem[Canon<S>::template at<i>(g, x, y, zl, aa, state)];
    s += v;
    if constexpr (S::vx(i) != 0) jx += S::vx(i) * v;
    if constexpr (S::vy(i) != 0) jy += S::vy(i) * v;
    if constexpr (S::vz(i) != 0) jz += S::vz(i) * v;
  });
  const double r = zc ? 1.0 + s : s;
  rho[cell] = r;
  u[cell] = (jx + dj.x) / r;
  u[ncell + cell] = (jy + dj.y) / r;
  if constexpr (S::D == 3) u[2 * ncell + cell] = (jz + dj.z) / r;
}

template <class S, int SPACE, int REG, class real, int RS = RS_GENERAL>
__global__ void k_test_collide(const double *__restrict__ fin, double *__restrict__ fout, long long n,
                               const Rates<real> r, real swe_g, const Force<real> fr) {
  const long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  real f[S::Q];
  sfor<S::Q>([&](auto i) { f[i] = (real)fin[c * S::Q + i]; });
  collide<S, SPACE, REG, real, RS>(f, r, swe_g, fr);
  sfor<S::Q>([&](auto i) { fout[c * S::Q + i] = (double)f[i]; });
}

// Global diagnostics of the canonical state: sum rho, sum rho u (3), sum rho |u|^2 / 2
// (the lattice-node discretisation of eq:TGA_kin_energy).  Fixed grid,
// per-thread sequential sums in a fixed order, then a fixed-shape tree: deterministic.
constexpr int DIAG_BLOCK = 256, DIAG_GRID = 1184;  // 148 SMs x 8
template <class S, class real>
__global__ void __launch_bounds__(DIAG_BLOCK) k_diag_partial(const real *mem, const GridParams g, int aa, int state,
                                                             int zc, double *__restrict__ partial,
                                                             const double3 dj) {
  const long long n = (long long)g.nx * g.ny * g.nzl;
  double acc[5] = {0, 0, 0, 0, 0};
  const bool narrow = n < (1ll << 31);  // 32-bit index arithmetic (64-bit division is slow)
  for (long long c = (long long)blockIdx.x * DIAG_BLOCK + threadIdx.x; c < n; c += (long long)DIAG_GRID * DIAG_BLOCK) {
    int x, y, zl;
    if (narrow) {
      const unsigned cu = (unsigned)c, row = cu / (unsigned)g.nx;
      x = (int)(cu - row * (unsigned)g.nx);
      y = (int)(row % (unsigned)g.ny);
      zl = (int)(row / (unsigned)g.ny);
    } else {
      x = (int)(c % g.nx);
      y = (int)((c / g.nx) % g.ny);
      zl = (int)(c / ((long long)g.nx * g.ny));
    }
    double s = 0, jx = 0, jy = 0, jz = 0;
    sfor<S::Q>([&](auto i) {
      const double v = (double)mem[Canon<S>::template at<i>(g, x, y, zl, aa, state)];
      s += v;
      if constexpr (S::vx(i) != 0) jx += S::vx(i) * v;
      if constexpr (S::vy(i) != 0) jy += S::vy(i) * v;
      if constexpr (S::vz(i) != 0) jz += S::vz(i) * v;
    });
    const double r = zc ? 1.0 + s : s;
    jx += dj.x;
    jy += dj.y;
    jz += dj.z;
    acc[0] += r;
    acc[1] += jx;
    acc[2] += jy;
    acc[3] += jz;
    acc[4] += 0.5 * (jx * jx + jy * jy + jz * jz) / r;
  }
  __shared__ double sh[5][DIAG_BLOCK];
#pragma unroll
  for (int k = 0; k < 5; ++k) sh[k][threadIdx.x] = acc[k];
  __syncthreads();
  for (int w = DIAG_BLOCK / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w)
#pragma unroll
      for (int k = 0; k < 5; ++k) sh[k][threadIdx.x] += sh[k][threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x < 5) partial[(long long)threadIdx.x * DIAG_GRID + blockIdx.x] = sh[threadIdx.x][0];
}

template <class T>
__global__ void __launch_bounds__(DIAG_BLOCK) k_diag_final(const T *__restrict__ partial, T *__restrict__ out) {
  __shared__ T sh[DIAG_BLOCK];
  for (int k = 0; k < 5; ++k) {
    double a = 0;
    for (int b = threadIdx.x; b < DIAG_GRID; b += DIAG_BLOCK) a += partial[(long long)k * DIAG_GRID + b];
    sh[threadIdx.x] = a;
    __syncthreads();
    for (int w = DIAG_BLOCK / 2; w > 0; w >>= 1) {
      if ((int)threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
      __syncthreads();
    }
    if (threadIdx.x == 0) out[k] = sh[0];
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Temporal blocking: TWO fused pull steps per sweep (single rank, periodic, 3D).
// A CTA owns a TX x TY column of the lattice and sweeps the slab axis.  At plane k it
// computes step t+1 on the (TX+2) x (TY+2) halo-extended tile (pulling step t from HBM)
// into a 3-plane shared-memory ring, then step t+2 on plane k-1 of the tile interior
// (pulling step t+1 from the ring) and stores it.  Every population of step t is read
// from HBM once and step t+2 written once: 2 updates per HBM round trip (plus the halo),
// and the step t+1 values never leave the SM.  Same per-cell arithmetic as k_pull, so
// the result equals two k_pull launches bitwise.
// ---------------------------------------------------------------------------
template <int TX, int TY>
struct Tile2 {
  static constexpr int HX = TX + 2, HY = TY + 2, HW = HX * HY;
  static constexpr int THREADS = (HW + 31) / 32 * 32;
};

// TRIM: the step-(t+1) ring keeps only what the step-(t+2) pull still reads (3 planes of the
// xi_z = +1 populations, 2 of xi_z = 0, 1 of xi_z = -1; Tile2::trim_*): 2/3 of the shared memory
template <int TX, int TY, class S>
struct Tile2Trim {
  static constexpr int HW = (TX + 2) * (TY + 2);
  static constexpr int slots(int i) { return S::mz(i) > 0 ? 3 : (S::mz(i) == 0 ? 2 : 1); }
  static constexpr int off(int i) {
    int o = 0;
    for (int j = 0; j < i; ++j) o += slots(j) * HW;
    return o;
  }
  static constexpr int RING = off(S::Q);
};

template <class S, int SPACE, int REG, class real, int RS, int TX, int TY, int MINB = 1, bool PF = false,
          bool RANGE = false, bool TRIM = false>
__global__ void __launch_bounds__(Tile2<TX, TY>::THREADS, MINB)
    k_pull2(const real *__restrict__ src, real *__restrict__ dst, const GridParams g, const Rates<real> r,
            const real swe_g, const Force<real> fr) {
  using T = Tile2<TX, TY>;
  using TR = Tile2Trim<TX, TY, S>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  real *ring = reinterpret_cast<real *>(smem_raw);  // [3][Q][HW], or the trimmed ring
  const int t = threadIdx.x;
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  // step t+1 cell of this thread on the halo-extended tile
  const bool act1 = t < T::HW;
  const int hx = t % T::HX, hy = t / T::HX;
  const int gx = wrapi(x0 - 1 + hx, g.nx), gy = wrapi(y0 - 1 + hy, g.ny);
  int xs[3], ys[3];
#pragma unroll
  for (int s = -1; s <= 1; ++s) {
    xs[s + 1] = wrapi(gx + s, g.nx);
    ys[s + 1] = wrapi(gy + s, g.ny) * g.pitch;
  }
  // step t+2 cell (tile interior)
  const bool act2 = t < TX * TY;
  const int ix = t % TX, iy = t / TX;
  const int n = g.nzl;
  // blockIdx.z: chunk [p0, p1) of the output planes (more CTAs for short slabs); each chunk
  // recomputes the two step-(t+1) planes at its ends
  // output planes [zb, zb + zn): the whole slab (single rank, periodic wrap) or, with RANGE
  // (across ranks), [zbegin, zbegin + zcount) whose two-step dependence stays inside the slab
  // (no wrap).  A template switch: a runtime wrap test in the loads cost the sweep 8-16 %.
  const int zb = RANGE ? g.zbegin : 0, zn = RANGE ? g.zcount : n;
  const int p0 = zb + (int)((long long)zn * blockIdx.z / gridDim.z);
  const int p1 = zb + (int)((long long)zn * (blockIdx.z + 1) / gridDim.z);
  auto zw = [&](int k) {
    if constexpr (RANGE) return k;
    else return wrapi(k, n);
  };
  // step-t populations of the halo-extended tile at plane k (pull: plane k - xi_z)
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
  real fn[PF ? S::Q : 1];
  if constexpr (PF) {
    if (act1) load(p0 - 1, fn);
  }
  for (int k = p0 - 1; k <= p1; ++k) {
    if (act1) {
      real f[S::Q];
      if constexpr (PF) {  // the next plane's loads fly during the collisions below
        sfor<S::Q>([&](auto i) { f[i] = fn[i]; });
        if (k < p1) load(k + 1, fn);
      } else {
        load(k, f);
      }
      collide<S, SPACE, REG, real, RS>(f, r, swe_g, fr);
      if constexpr (TRIM) {
        sfor<S::Q>([&](auto i) { ring[TR::off(i) + ((k + 3) % TR::slots(i)) * T::HW + t] = f[i]; });
      } else {
        real *slot = ring + (size_t)((k + 3) % 3) * S::Q * T::HW;  // k >= -1
        sfor<S::Q>([&](auto i) { slot[i * T::HW + t] = f[i]; });
      }
    }
    __syncthreads();
    if (k >= p0 + 1 && act2) {
      const int p = k - 1;  // plane of step t+2
      real f[S::Q];
      sfor<S::Q>([&](auto i) {
        constexpr int cx = S::mx(i), cy = S::my(i), cz = S::mz(i);
        const int at = (iy + 1 - cy) * T::HX + (ix + 1 - cx);
        if constexpr (TRIM) {
          f[i] = ring[TR::off(i) + ((p - cz + 3) % TR::slots(i)) * T::HW + at];
        } else {
          const real *slot = ring + (size_t)((p - cz + 3) % 3) * S::Q * T::HW;
          f[i] = slot[i * T::HW + at];
        }
      });
      collide<S, SPACE, REG, real, RS>(f, r, swe_g, fr);
      const long long own = (long long)(p + 1) * g.plane + (long long)(y0 + iy) * g.pitch + (x0 + ix);
      sfor<S::Q>([&](auto i) { dst[own + (long long)i * g.pop] = f[i]; });
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Temporal blocking with TMA staging (sm_100a): the same two-step sweep as k_pull2, but the
// step-t populations of the next plane are not prefetched into registers by every thread.
// One thread issues, per plane and population i, a cp.async.bulk.tensor box load of the
// halo-extended tile shifted by -xi_i in y from plane k - xi_z,i into a shared-memory stage
// (the pull gather done by the TMA unit; the box start along x must be 16-byte aligned, so the
// x shift is applied when the box is read); an mbarrier counts the bytes.  The per-thread
// prefetch registers and the per-population address arithmetic of k_pull2 disappear, and the
// loads of plane k + STAGES are in flight during the collisions of plane k.
// The step-(t+1) ring is trimmed to what the step-(t+2) pull still reads: the populations
// with xi_z = +1 are read one plane later (3 planes live), xi_z = 0 in the same plane (2),
// xi_z = -1 one plane earlier (1) — 3 n+ + 2 n0 + n- slots instead of 3 Q.
// The TMA does not wrap: at the periodic x / y faces the box elements that fall outside the
// lattice arrive zero-filled and the (CTA-uniform) edge tiles reload them from the wrapped
// address.  Same collide() as k_pull / k_pull2.
// ---------------------------------------------------------------------------
template <class S, class real, int TX, int TY, int STAGES>
struct TmaTile {
  static constexpr int HX = TX + 2, HY = TY + 2, HW = HX * HY;
  static constexpr int THREADS = (HW + 31) / 32 * 32;
  // the box starts at x0 - A (16-byte aligned: the TMA faults on an unaligned inner start) and
  // covers the pull sources x0 - 2 .. x0 + TX + 1 of the halo cells, in 16-byte multiples
  static constexpr int A = (int)(16 / sizeof(real));
  static constexpr int BX = (TX + A + 2 + A - 1) / A * A;
  static constexpr int BOX = BX * HY;  // elements of one population box
  // box stride in shared memory, 128-byte aligned destinations
  static constexpr int BOXP = (int)(((BOX * sizeof(real) + 127) / 128 * 128) / sizeof(real));
  static constexpr int STAGE = S::Q * BOXP;  // elements of one staged plane
  static constexpr unsigned STAGE_TX = (unsigned)(S::Q * BOX * sizeof(real));  // bytes the TMA writes
  static constexpr int slots(int i) { return S::mz(i) > 0 ? 3 : (S::mz(i) == 0 ? 2 : 1); }
  static constexpr int ring_off(int i) {
    int o = 0;
    for (int j = 0; j < i; ++j) o += slots(j) * HW;
    return o;
  }
  static constexpr int RING = ring_off(S::Q);  // elements of the trimmed ring
  static constexpr size_t SMEM = (size_t)(STAGES * STAGE + RING) * sizeof(real) + 16 * STAGES;
};

template <class S, int SPACE, int REG, class real, int RS, int TX, int TY, int MINB = 1, bool RANGE = false,
          int STAGES = 1>
__global__ void __launch_bounds__(TmaTile<S, real, TX, TY, STAGES>::THREADS, MINB)
    k_pull2_tma(const real *__restrict__ src, real *__restrict__ dst, const GridParams g, const Rates<real> r,
                const real swe_g, const Force<real> fr, const __grid_constant__ CUtensorMap tmap) {
  using T = TmaTile<S, real, TX, TY, STAGES>;
  extern __shared__ __align__(128) unsigned char smem_tma[];
  real *stage = reinterpret_cast<real *>(smem_tma);  // [STAGES][Q][BOXP]
  real *ring = stage + STAGES * T::STAGE;            // trimmed ring
  uint64_t *bar = reinterpret_cast<uint64_t *>(ring + T::RING);
  const int t = threadIdx.x;
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const bool act1 = t < T::HW;
  const int hx = t % T::HX, hy = t / T::HX;
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
  // generic address of the __grid_constant__ parameter itself (a copy would live in local memory,
  // which the TMA cannot read)
  const CUtensorMap *map = &tmap;
  // periodic wrap at the x / y faces: only tiles touching a face see out-of-range box elements
  const bool edge = x0 == 0 || x0 + TX >= g.nx || y0 == 0 || y0 + TY >= g.ny;
  if (t == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) mbar_init(bar + s, 1);
    mbar_fence_init();
  }
  __syncthreads();
  // plane k of step t into stage slot b: box of population i from plane k - xi_z at -xi_i
  auto issue = [&](int k, int b) {
    const int zc = zw(k);
    int zz[3];
#pragma unroll
    for (int s = -1; s <= 1; ++s) zz[s + 1] = zw(zc + s) + 1;
    real *st = stage + b * T::STAGE;
    mbar_arrive_expect_tx(bar + b, T::STAGE_TX);
    sfor<S::Q>([&](auto i) {
      constexpr int cx = S::mx(i), cy = S::my(i), cz = S::mz(i);
      (void)cx;
      tma_load_4d(st + i * T::BOXP, map, x0 - T::A, y0 - 1 - cy, (int)i, zz[1 - cz], bar + b);
    });
  };
  if (t == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s)
      if (p0 - 1 + s <= p1) issue(p0 - 1 + s, s);
  }
  for (int k = p0 - 1; k <= p1; ++k) {
    const int it = k - (p0 - 1);
    const int b = it % STAGES;
    real f[S::Q];
    if (act1) {
      mbar_wait(bar + b, (uint32_t)((it / STAGES) & 1));
      const real *st = stage + b * T::STAGE + hy * T::BX + hx + T::A - 1;
      sfor<S::Q>([&](auto i) { f[i] = st[i * T::BOXP - S::mx(i)]; });
      if (edge) {  // out-of-range sources: reload from the wrapped address
        const int gx = x0 - 1 + hx, gy = y0 - 1 + hy;
        const int zc = zw(k);
        sfor<S::Q>([&](auto i) {
          constexpr int cx = S::mx(i), cy = S::my(i), cz = S::mz(i);
          const int sx = gx - cx, sy = gy - cy;
          if (sx < 0 || sx >= g.nx || sy < 0 || sy >= g.ny) {
            const long long a = (long long)(zw(zc - cz) + 1) * g.plane + (long long)i * g.pop +
                                (long long)wrapi(sy, g.ny) * g.pitch + wrapi(sx, g.nx);
            f[i] = ld_nc(src + a);
          }
        });
      }
    }
    __syncthreads();  // stage b consumed by every thread; ring slots of plane k free
    if (t == 0 && k + STAGES <= p1) {
      fence_proxy_async_smem();
      issue(k + STAGES, b);
    }
    if (act1) {
      collide<S, SPACE, REG, real, RS>(f, r, swe_g, fr);
      sfor<S::Q>([&](auto i) {
        constexpr int ns = T::slots(i);
        ring[T::ring_off(i) + ((k + 3) % ns) * T::HW + t] = f[i];  // k >= -1
      });
    }
    __syncthreads();
    if (k >= p0 + 1 && act2) {
      const int p = k - 1;  // plane of step t+2
      real h[S::Q];
      sfor<S::Q>([&](auto i) {
        constexpr int cx = S::mx(i), cy = S::my(i), cz = S::mz(i);
        constexpr int ns = T::slots(i);
        h[i] = ring[T::ring_off(i) + ((p - cz + 3) % ns) * T::HW + (iy + 1 - cy) * T::HX + (ix + 1 - cx)];
      });
      collide<S, SPACE, REG, real, RS>(h, r, swe_g, fr);
      const long long own = (long long)(p + 1) * g.plane + (long long)(y0 + iy) * g.pitch + (x0 + ix);
      sfor<S::Q>([&](auto i) { dst[own + (long long)i * g.pop] = h[i]; });
    }
  }
}

// ---------------------------------------------------------------------------
// Cluster-resident pull loop for small 2D lattices (single rank): one thread-block cluster of
// C CTAs keeps the whole lattice in shared memory for all n steps of one launch.  CTA k owns
// rows [k R, (k + 1) R) of the slab axis (physical y) plus one ghost row per side, in two
// shared-memory grids [2][Q][R + 2][nx].  Per step every cell pulls from grid A, collides in
// registers (the same collide() as k_pull: bitwise equal), stores into grid B, and the
// boundary rows also store their slab-crossing populations straight into the neighbouring
// CTAs' ghost rows of grid B through distributed shared memory; one cluster barrier
// (release/acquire) orders the step.  HBM is touched once at the start and once at the end:
// the loop is bound by the collision and the barrier, not by launches (CUDA-graph replay
// floor: 1.7 us per step).
// ---------------------------------------------------------------------------
template <class S, int SPACE, int REG, class real, int RS, bool BB>
__global__ void __launch_bounds__(1024, 1)
    k_resident2(const real *__restrict__ src, real *__restrict__ dst, const GridParams g, int nsteps,
                const Rates<real> r, const real swe_g, const Force<real> fr) {
  static_assert(S::D == 2, "the resident loop is for D2Q9 lattices");
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int C = (int)cl.num_blocks(), rank = (int)cl.block_rank();
  const int nx = g.nx, R = g.nzl / C, y0 = rank * R;
  const int popsz = (R + 2) * nx, gridsz = S::Q * popsz;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  real *A = reinterpret_cast<real *>(smem_raw);
  real *B = A + gridsz;
  const int lower = (rank + C - 1) % C, upper = (rank + 1) % C;
  // the step-t state of the own rows and the two ghost rows (periodic wrap; walls bounce)
  for (int e = threadIdx.x; e < (R + 2) * nx; e += blockDim.x) {
    const int lr = e / nx, x = e - lr * nx;
    const int gy = wrapi(y0 - 1 + lr, g.nzl);
    sfor<S::Q>([&](auto i) { A[i * popsz + lr * nx + x] = src[(long long)(gy + 1) * g.plane + i * g.pop + x]; });
  }
  cl.sync();  // every CTA of the cluster runs before the first DSMEM store
  for (int step = 0; step < nsteps; ++step) {
    real *Blo = cl.map_shared_rank(B, lower), *Bhi = cl.map_shared_rank(B, upper);
    for (int e = threadIdx.x; e < R * nx; e += blockDim.x) {
      const int lr = e / nx + 1, x = e - (lr - 1) * nx;
      const int xs[3] = {wrapi(x - 1, nx), x, wrapi(x + 1, nx)};
      real f[S::Q];
      if constexpr (BB) {
        const int gy = y0 + lr - 1;
        const bool bx[3] = {x == 0 && (g.bcmask & 1), false, x == nx - 1 && (g.bcmask & 2)};
        const bool bz[3] = {gy == 0 && (g.bcmask & 16), false, gy == g.nzl - 1 && (g.bcmask & 32)};
        sfor<S::Q>([&](auto i) {
          constexpr int cx = S::mx(i), cz = S::mz(i);
          // half-way bounce-back: f_i(x) = f*_{opp i}(x)   (reading R18)
          f[i] = (bx[1 - cx] || bz[1 - cz]) ? A[S::opp(i) * popsz + lr * nx + x]
                                             : A[i * popsz + (lr - cz) * nx + xs[1 - cx]];
        });
      } else {
        sfor<S::Q>([&](auto i) {
          constexpr int cx = S::mx(i), cz = S::mz(i);
          f[i] = A[i * popsz + (lr - cz) * nx + xs[1 - cx]];
        });
      }
      collide<S, SPACE, REG, real, RS>(f, r, swe_g, fr);
      sfor<S::Q>([&](auto i) {
        constexpr int cz = S::mz(i);
        B[i * popsz + lr * nx + x] = f[i];
        // slab-crossing populations into the neighbours' ghost rows (DSMEM)
        if constexpr (cz < 0) {
          if (lr == 1) Blo[i * popsz + (R + 1) * nx + x] = f[i];
        } else if constexpr (cz > 0) {
          if (lr == R) Bhi[i * popsz + x] = f[i];
        }
      });
    }
    cl.sync();  // barrier.cluster arrive.release / wait.acquire: step complete everywhere
    real *t = A;
    A = B;
    B = t;
  }
  for (int e = threadIdx.x; e < R * nx; e += blockDim.x) {
    const int lr = e / nx + 1, x = e - (lr - 1) * nx;
    sfor<S::Q>([&](auto i) {
      dst[(long long)(y0 + lr) * g.plane + i * g.pop + x] = A[i * popsz + lr * nx + x];
    });
  }
}

// ---------------------------------------------------------------------------
// Temporal blocking for 2D lattices: the same two-step sweep as k_pull2 with a 1D tile.
// A CTA owns TX consecutive cells of a row and sweeps the slab axis (physical y): at row k
// it computes step t+1 on the TX + 2 cells of the halo-extended strip into a 3-row ring,
// then step t+2 on row k-1 of the strip interior from the ring.  The step-t loads of row
// k+1 are issued before the collisions of row k (software pipelining: the HBM latency hides
// under the arithmetic of two collisions).  Same collide() as k_pull: bitwise equal.
// ---------------------------------------------------------------------------
template <int TX>
struct Tile1 {
  static constexpr int HW = TX + 2;
  static constexpr int THREADS = (HW + 31) / 32 * 32;
};

template <class S, int SPACE, int REG, class real, int RS, int TX, int MINB = 1, bool PF = true, bool RANGE = false>
__global__ void __launch_bounds__(Tile1<TX>::THREADS, MINB)
    k_pull2_2d(const real *__restrict__ src, real *__restrict__ dst, const GridParams g, const Rates<real> r,
               const real swe_g, const Force<real> fr) {
  static_assert(S::D == 2, "2D temporal blocking");
  using T = Tile1<TX>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  real *ring = reinterpret_cast<real *>(smem_raw);  // [3][Q][HW]
  const int t = threadIdx.x;
  const int x0 = blockIdx.x * TX;
  const bool act1 = t < T::HW;
  const int gx = wrapi(x0 - 1 + t, g.nx);
  const int xs[3] = {wrapi(gx - 1, g.nx), gx, wrapi(gx + 1, g.nx)};
  const int n = g.nzl;
  const int zb = RANGE ? g.zbegin : 0, zn = RANGE ? g.zcount : n;  // as in k_pull2
  const int p0 = zb + (int)((long long)zn * blockIdx.y / gridDim.y);
  const int p1 = zb + (int)((long long)zn * (blockIdx.y + 1) / gridDim.y);
  auto zw = [&](int k) {
    if constexpr (RANGE) return k;
    else return wrapi(k, n);
  };
  // step-t populations of the halo-extended strip at row k (pull: row k - xi_y)
  auto load = [&](int k, real (&f)[S::Q]) {
    const int zc = zw(k);
    const long long zo[3] = {(long long)(zw(zc - 1) + 1) * g.plane, (long long)(zc + 1) * g.plane,
                             (long long)(zw(zc + 1) + 1) * g.plane};
    sfor<S::Q>([&](auto i) {
      constexpr int cx = S::mx(i), cz = S::mz(i);
      f[i] = ld_nc(src + zo[1 - cz] + (long long)i * g.pop + xs[1 - cx]);
    });
  };
  real fn[S::Q];
  if (PF && act1) load(p0 - 1, fn);
  for (int k = p0 - 1; k <= p1; ++k) {
    if (act1) {
      real f[S::Q];
      if constexpr (PF) {
        sfor<S::Q>([&](auto i) { f[i] = fn[i]; });
        if (k < p1) load(k + 1, fn);  // in flight during the two collisions below
      } else {
        load(k, f);
      }
      collide<S, SPACE, REG, real, RS>(f, r, swe_g, fr);
      real *slot = ring + (size_t)((k + 3) % 3) * S::Q * T::HW;  // k >= -1
      sfor<S::Q>([&](auto i) { slot[i * T::HW + t] = f[i]; });
    }
    __syncthreads();
    if (k >= p0 + 1 && t < TX) {
      const int p = k - 1;  // row of step t+2
      real f[S::Q];
      sfor<S::Q>([&](auto i) {
        constexpr int cx = S::mx(i), cz = S::mz(i);
        const real *slot = ring + (size_t)((p - cz + 3) % 3) * S::Q * T::HW;
        f[i] = slot[i * T::HW + (t + 1 - cx)];
      });
      collide<S, SPACE, REG, real, RS>(f, r, swe_g, fr);
      const long long own = (long long)(p + 1) * g.plane + (x0 + t);
      sfor<S::Q>([&](auto i) { dst[own + (long long)i * g.pop] = f[i]; });
    }
    __syncthreads();
  }
}

// Temporal blocking of depth D for 2D lattices (k_pullD_2d; the product uses D = 3): three
// pull steps per HBM round trip.  A CTA owns TX consecutive cells of a row and sweeps the slab
// axis (physical y).  Level s = 1..D is time step t+s; at sweep iteration k level s is
// computed at row k - (s - 1) on the strip widened by D - s cells per side (the cells level
// s + 1 pulls from): level 1 from HBM (the next row's loads prefetched), level s >= 2 from
// the shared-memory ring of level s - 1, level D stored to HBM.  A row of a level stays in its
// ring only while the next level's pull still reads it (3 / 2 / 1 rows for the populations
// with xi_y = +1 / 0 / -1).  Per cell and D steps: one read and one write of every
// population, D collisions plus the widened strips (2 (D - s) / TX per level) and the
// slab-chunk ends.  Same collide() as k_pull: equal to D single steps bitwise on B200
// (scripts/tb2d_depth.cu: D = 3 at C5 0.73 vs 0.82 ms per step for the two-step sweep;
// D = 4 no faster, profiles/r2/tb2d_depth.txt).  Single rank, periodic (the slab wraps), or a
// row range of a rank's slab (RANGE; the interior of three steps across ranks, runtime.cu).
// ---------------------------------------------------------------------------
template <class S, int TX, int D, int X = 0>
struct TileD {
  static constexpr int W(int s) { return TX + 2 * (D - s); }  // strip width of level s
  static constexpr int THREADS = (W(1) + 31) / 32 * 32;
  // rows kept per population (mz: the slab axis); X extra rows for a skewed sweep
  static constexpr int slots(int i) { return (S::mz(i) > 0 ? 3 : (S::mz(i) == 0 ? 2 : 1)) + X; }
  static constexpr int per_level(int w) {  // ring elements of one level of width w
    int o = 0;
    for (int j = 0; j < S::Q; ++j) o += slots(j) * w;
    return o;
  }
  static constexpr int level_off(int s) {  // ring of level s (s = 1 .. D-1)
    int o = 0;
    for (int l = 1; l < s; ++l) o += per_level(W(l));
    return o;
  }
  static constexpr int pop_off(int i, int w) {
    int o = 0;
    for (int j = 0; j < i; ++j) o += slots(j) * w;
    return o;
  }
  static constexpr int RING = level_off(D);  // elements
};

// RANGE (across ranks): output rows [zbegin, zbegin + zcount) of a slab, every row the levels
// pull from inside [0, nzl) (zbegin >= D, zbegin + zcount <= nzl - D): no wrap, no ghost rows.
template <class S, int SPACE, int REG, class real, int RS, int TX, int D, int MINB = 1, bool PF = true,
          bool RANGE = false>
__global__ void __launch_bounds__(TileD<S, TX, D>::THREADS, MINB)
    k_pullD_2d(const real *__restrict__ src, real *__restrict__ dst, const GridParams g, const Rates<real> r,
               const real swe_g, const Force<real> fr) {
  static_assert(S::D == 2 && D >= 2 && D <= 4, "2D temporal blocking of depth 2..4");
  using T = TileD<S, TX, D>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  real *ring = reinterpret_cast<real *>(smem_raw);
  const int t = threadIdx.x;
  const int x0 = blockIdx.x * TX;
  const int n = g.nzl;
  const int zb = RANGE ? g.zbegin : 0, zn = RANGE ? g.zcount : n;
  const int p0 = zb + (int)((long long)zn * blockIdx.y / gridDim.y);
  const int p1 = zb + (int)((long long)zn * (blockIdx.y + 1) / gridDim.y);
  auto zw = [&](int k) {
    if constexpr (RANGE) return k;
    else return wrapi(k, n);
  };
  // level 1: strip cell t at x0 - (D - 1) + t, its pull sources at x - 1, x, x + 1
  constexpr int W1 = T::W(1);
  const bool act1 = t < W1;
  const int gx = wrapi(x0 - (D - 1) + t, g.nx);
  const int xs[3] = {wrapi(gx - 1, g.nx), gx, wrapi(gx + 1, g.nx)};
  auto load = [&](int k, real(&f)[S::Q]) {
    const int zc = zw(k);
    const long long zo[3] = {(long long)(zw(zc - 1) + 1) * g.plane, (long long)(zc + 1) * g.plane,
                             (long long)(zw(zc + 1) + 1) * g.plane};
    sfor<S::Q>([&](auto i) {
      constexpr int cx = S::mx(i), cz = S::mz(i);
      f[i] = ld_nc(src + zo[1 - cz] + (long long)i * g.pop + xs[1 - cx]);
    });
  };
  // rows of level 1 computed: [p0 - (D - 1), p1 + (D - 1)); iteration k computes level s at
  // row k - (s - 1) when that row lies in [p0 - (D - s), p1 + (D - s))
  const int kb = p0 - (D - 1), ke = p1 + (D - 1);
  real fn[PF ? S::Q : 1];
  if constexpr (PF) {
    if (act1) load(kb, fn);
  }
  for (int k = kb; k < ke; ++k) {
    // level 1 at row k
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
      sfor<S::Q>([&](auto i) {
        lv[T::pop_off(i, W1) + ((k + 12) % T::slots(i)) * W1 + t] = f[i];
      });
    }
    // levels 2 .. D
    sfor<D - 1>([&](auto sm) {
      constexpr int s = sm + 2;
      constexpr int Ws = T::W(s), Wp = T::W(s - 1);
      __syncthreads();
      const int row = k - (s - 1);
      if (t < Ws && row >= p0 - (D - s) && row < p1 + (D - s)) {
        const real *pv = ring + T::level_off(s - 1);
        real f[S::Q];
        sfor<S::Q>([&](auto i) {
          constexpr int cx = S::mx(i), cz = S::mz(i);
          f[i] = pv[T::pop_off(i, Wp) + ((row - cz + 12) % T::slots(i)) * Wp + (t + 1 - cx)];
        });
        collide<S, SPACE, REG, real, RS>(f, r, swe_g, fr);
        if constexpr (s == D) {
          const long long own = (long long)(zw(row) + 1) * g.plane + (x0 + t);
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


// canonical populations of selected cells (local linear index x + nx (y + ny z))
template <class S, class real>
__global__ void k_get_cells(const real *mem, const GridParams g, int aa, int state, const long long *__restrict__ idx,
                            long long n, double *__restrict__ out) {
  const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const long long c = idx[k];
  const int x = (int)(c % g.nx);
  const int y = (int)((c / g.nx) % g.ny);
  const int zl = (int)(c / ((long long)g.nx * g.ny));
  sfor<S::Q>([&](auto i) { out[k * S::Q + i] = (double)mem[Canon<S>::template at<i>(g, x, y, zl, aa, state)]; });
}

template <class S, class real>
__global__ void k_check_finite(const real *mem, const GridParams g, int *flag) {
  const int x = blockIdx.x * BLOCK_X + threadIdx.x;
  if (x >= g.nx) return;
  const int y = blockIdx.y, zl = blockIdx.z;
  bool bad = false;
  const long long own = (long long)(zl + 1) * g.plane + (long long)y * g.pitch + x;
  sfor<S::Q>([&](auto i) { bad |= !isfinite((double)mem[own + (long long)i * g.pop]); });
  if (bad) atomicOr(flag, 1);
}

}  // namespace lbm
