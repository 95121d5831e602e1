// lattice.cuh — compile-time stencil descriptions for the device kernels.
//
// Velocity ORDER follows the interface convention of include/lbm.h (the paper
// leaves it free except xi_0 = 0).  Two views of a velocity:
//   * memory offsets (mx, my, mz): the device grid is [z][i][y][x] with the slab
//     axis as its outermost dimension; for D2Q9 the physical y axis IS that slab
//     axis, so (mx, my, mz) = (xi_x, 0, xi_y);
//   * the physical Chimera cube position (f_xyz), index
//     a + 3 b (+ 9 c) with a = xi_x + 1, b = xi_y + 1, c = xi_z + 1.
#pragma once
#include <cstdint>
#include <type_traits>
#include <utility>

namespace lbm {

// compile-time loop: f(std::integral_constant<int, I>{}) for I = 0..N-1
template <class F, int... Is>
__host__ __device__ __forceinline__ void sfor_impl(F &&f, std::integer_sequence<int, Is...>) {
  (f(std::integral_constant<int, Is>{}), ...);
}
template <int N, class F>
__host__ __device__ __forceinline__ void sfor(F &&f) {
  sfor_impl(f, std::make_integer_sequence<int, N>{});
}

struct D2Q9 {
  static constexpr int ID = 0, Q = 9, D = 2, NC = 9;
  static constexpr int UP0 = 3, NUP = 3;  // slab +1 group = [3, 6), -1 group = [6, 9)
  __host__ __device__ static constexpr int vx(int i) {
    constexpr int t[9] = {0, 1, -1, 0, 1, -1, 0, -1, 1};
    return t[i];
  }
  __host__ __device__ static constexpr int vy(int i) {
    constexpr int t[9] = {0, 0, 0, 1, 1, 1, -1, -1, -1};
    return t[i];
  }
  __host__ __device__ static constexpr int vz(int) { return 0; }
  __host__ __device__ static constexpr int opp(int i) {
    constexpr int t[9] = {0, 2, 1, 6, 7, 8, 3, 4, 5};
    return t[i];
  }
  // memory offsets: slab axis (physical y) is the outer dimension
  __host__ __device__ static constexpr int mx(int i) { return vx(i); }
  __host__ __device__ static constexpr int my(int) { return 0; }
  __host__ __device__ static constexpr int mz(int i) { return vy(i); }
  __host__ __device__ static constexpr int pos(int i) { return (vx(i) + 1) + 3 * (vy(i) + 1); }
  __host__ __device__ static constexpr bool present(int a, int b, int c) { return c == 0; }
};

struct D3Q27 {
  static constexpr int ID = 2, Q = 27, D = 3, NC = 27;
  static constexpr int UP0 = 9, NUP = 9;
  __host__ __device__ static constexpr int vx(int i) {
    constexpr int t[27] = {0, 1, -1, 0, 0, 1, -1, 1, -1, 0, 1, -1, 0, 0, 1, -1, 1, -1,
                           0, -1, 1, 0, 0, -1, 1, -1, 1};
    return t[i];
  }
  __host__ __device__ static constexpr int vy(int i) {
    constexpr int t[27] = {0, 0, 0, 1, -1, 1, -1, -1, 1, 0, 0, 0, 1, -1, 1, -1, -1, 1,
                           0, 0, 0, -1, 1, -1, 1, 1, -1};
    return t[i];
  }
  __host__ __device__ static constexpr int vz(int i) {
    return i == 0 ? 0 : (i < 9 ? 0 : (i < 18 ? 1 : -1));
  }
  __host__ __device__ static constexpr int opp(int i) {
    return i == 0 ? 0 : (i < 9 ? (i % 2 == 1 ? i + 1 : i - 1) : (i < 18 ? i + 9 : i - 9));
  }
  __host__ __device__ static constexpr int mx(int i) { return vx(i); }
  __host__ __device__ static constexpr int my(int i) { return vy(i); }
  __host__ __device__ static constexpr int mz(int i) { return vz(i); }
  __host__ __device__ static constexpr int pos(int i) {
    return (vx(i) + 1) + 3 * (vy(i) + 1) + 9 * (vz(i) + 1);
  }
  __host__ __device__ static constexpr bool present(int, int, int) { return true; }
};

struct D3Q19 {
  static constexpr int ID = 1, Q = 19, D = 3, NC = 27;
  static constexpr int UP0 = 9, NUP = 5;
  __host__ __device__ static constexpr int vx(int i) {
    constexpr int t[19] = {0, 1, -1, 0, 0, 1, -1, 1, -1, 0, 1, -1, 0, 0, 0, -1, 1, 0, 0};
    return t[i];
  }
  __host__ __device__ static constexpr int vy(int i) {
    constexpr int t[19] = {0, 0, 0, 1, -1, 1, -1, -1, 1, 0, 0, 0, 1, -1, 0, 0, 0, -1, 1};
    return t[i];
  }
  __host__ __device__ static constexpr int vz(int i) {
    return i == 0 ? 0 : (i < 9 ? 0 : (i < 14 ? 1 : -1));
  }
  __host__ __device__ static constexpr int opp(int i) {
    return i == 0 ? 0 : (i < 9 ? (i % 2 == 1 ? i + 1 : i - 1) : (i < 14 ? i + 5 : i - 5));
  }
  __host__ __device__ static constexpr int mx(int i) { return vx(i); }
  __host__ __device__ static constexpr int my(int i) { return vy(i); }
  __host__ __device__ static constexpr int mz(int i) { return vz(i); }
  __host__ __device__ static constexpr int pos(int i) {
    return (vx(i) + 1) + 3 * (vy(i) + 1) + 9 * (vz(i) + 1);
  }
  // cube position (a,b,c) in {0,1,2}^3 holds a population iff |xi|_1 <= 2
  __host__ __device__ static constexpr bool present(int a, int b, int c) {
    return ((a != 1) + (b != 1) + (c != 1)) <= 2;
  }
};

// background populations f0 = lattice weights, by |xi|^2
template <class S>
__host__ __device__ constexpr double weight(int i) {
  int n2 = S::vx(i) * S::vx(i) + S::vy(i) * S::vy(i) + S::vz(i) * S::vz(i);
  if (S::Q == 9) return n2 == 0 ? 4.0 / 9.0 : (n2 == 1 ? 1.0 / 9.0 : 1.0 / 36.0);
  if (S::Q == 19) return n2 == 0 ? 1.0 / 3.0 : (n2 == 1 ? 1.0 / 18.0 : 1.0 / 36.0);
  return n2 == 0 ? 8.0 / 27.0 : (n2 == 1 ? 2.0 / 27.0 : (n2 == 2 ? 1.0 / 54.0 : 1.0 / 216.0));
}

// moment-cube index of exponents (a, b, c); 2D uses (a, b) only
__host__ __device__ constexpr int E(int a, int b, int c = 0) { return a + 3 * b + 9 * c; }

}  // namespace lbm
