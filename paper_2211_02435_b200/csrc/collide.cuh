// collide.cuh — register-resident MRT collision of one lattice cell (device code).
//
// The transforms are the paper's Chimera forms, evaluated in registers on a
// 3^d "cube" of values (f_xyz = f_i if xi_i = (x,y,z) is in the
// stencil, else 0):
//   fwd_raw   : eq:RawMomentChimeraTransform, sweeps z, y, x;
//               per axis (f-, f0, f+) -> (f0 + f+ + f-, f+ - f-, f+ + f-)
//   bwd_raw   : f* = M^{-1} m* split per axis into symmetric/antisymmetric parts
//               (eq:RawMomentChimeraBackwardSymmetric):
//               (m0, m1, m2) -> ((m2 - m1)/2, m0 - m2, (m2 + m1)/2); D3Q19 uses the
//               same split over its 9 opposite pairs (reduced 19 x 19 inverse)
//   bin_fwd/bwd : binomial Chimera raw <-> central, per axis
//               k1 = m1 - u m0, k2 = m2 - 2u m1 + u^2 m0 and its inverse
//   cumulants : closed forms of C = Xi.u + log K / K = exp(C - Xi.u) for the
//               monomials of orders 4-6 (eq:CumulantAndCentralMomentGenFuncs,
//               PAPER.md:680-693) with kappa_100 = 0 collapsed
//               and no log/exp left
// Relaxation q*_p = q_p + w_p (q_eq_p - q_p) is applied per basis polynomial
// (eq:MrtUpdateGeneral) by recombining the monomials of each
// polynomial group and decomposing afterwards.
//
// Regimes (template REG):
//   REG_ABS      absolute storage, eq:MrtUpdateGeneral
//   REG_DELTA    zero-centered storage + delta equilibrium, eq:MrtUpdateGeneralDeviationOnly
//                (linear spaces only; dq_eq written in delta-rho form)
//   REG_ZC_ABS   zero-centered storage + absolute equilibrium,
//                eq:MrtUpdateAbsoluteFromZeroCentered: the background raw moments m0
//                are added after the forward raw transform and removed before the
//                backward one (T(f0) = M f0 = m0).
#pragma once
#include "lattice.cuh"

namespace lbm {

// SPACE_SWE: central moments relaxed against Zhou's discrete shallow-water equilibrium
// (de Rosis); SPACE_SWE_K: cumulants relaxed against the Maxwellian
// with cs2 = g h / 2 (Venturi).
enum { SPACE_POPULATION = 0, SPACE_RAW = 1, SPACE_CENTRAL = 2, SPACE_CUMULANT = 3, SPACE_SWE = 4, SPACE_SWE_K = 5 };
enum { REG_ABS = 0, REG_DELTA = 1, REG_ZC_ABS = 2 };

template <class real>
struct Rates {
  real w[27];
};

// --------------------------------------------------------------------------
// exponent helpers
// --------------------------------------------------------------------------
__host__ __device__ constexpr int ex_of(int e) { return e % 3; }
__host__ __device__ constexpr int ey_of(int e) { return (e / 3) % 3; }
__host__ __device__ constexpr int ez_of(int e) { return e / 9; }
__host__ __device__ constexpr int n2_of(int e) {
  return (ex_of(e) == 2) + (ey_of(e) == 2) + (ez_of(e) == 2);
}
__host__ __device__ constexpr int n1_of(int e) {
  return (ex_of(e) == 1) + (ey_of(e) == 1) + (ez_of(e) == 1);
}
__host__ __device__ constexpr double third_pow(int n) {
  return n == 0 ? 1.0 : (n == 1 ? 1.0 / 3.0 : (n == 2 ? 1.0 / 9.0 : 1.0 / 27.0));
}
// Gaussian/background central (= rest raw) moment factor prod_a h(e_a), h = (1, 0, cs2)
__host__ __device__ constexpr double hprod(int e) { return n1_of(e) ? 0.0 : third_pow(n2_of(e)); }

// --------------------------------------------------------------------------
// forward raw Chimera with compile-time presence of populations
// --------------------------------------------------------------------------
template <class S>
struct Presence {
  // populations
  __host__ __device__ static constexpr bool p0(int a, int b, int c) { return S::present(a, b, c); }
  // after the z sweep: chimera m_{ab|g}
  __host__ __device__ static constexpr bool p1(int a, int b, int g) {
    return g == 0 ? (p0(a, b, 0) || p0(a, b, 1) || p0(a, b, 2)) : (p0(a, b, 0) || p0(a, b, 2));
  }
  // after the y sweep: m_{a|be g}
  __host__ __device__ static constexpr bool p2(int a, int be, int g) {
    return be == 0 ? (p1(a, 0, g) || p1(a, 1, g) || p1(a, 2, g)) : (p1(a, 0, g) || p1(a, 2, g));
  }
  // after the x sweep: m_{al be g}
  __host__ __device__ static constexpr bool p3(int al, int be, int g) {
    return al == 0 ? (p2(0, be, g) || p2(1, be, g) || p2(2, be, g)) : (p2(0, be, g) || p2(2, be, g));
  }
};

// one axis line (c0, c1, c2) = values at velocity (-1, 0, +1) -> exponents (0, 1, 2)
template <bool PM, bool P0, bool PP, class real>
__device__ __forceinline__ void fwd_line(real &c0, real &c1, real &c2) {
  if constexpr (PM && PP) {
    const real s = c2 + c0, d = c2 - c0;
    if constexpr (P0) c0 = c1 + s; else c0 = s;
    c1 = d;
    c2 = s;
  } else if constexpr (PP) {
    const real p = c2;
    if constexpr (P0) c0 = c1 + p; else c0 = p;
    c1 = p;
    c2 = p;
  } else if constexpr (PM) {
    const real m = c0;
    if constexpr (P0) c0 = c1 + m; else c0 = m;
    c1 = -m;
    c2 = m;
  } else {
    if constexpr (P0) c0 = c1; else c0 = real(0);
    c1 = real(0);
    c2 = real(0);
  }
}

template <class S, class real>
__device__ __forceinline__ void fwd_raw3(real (&c)[27]) {
  using P = Presence<S>;
  // z sweep: lines over (a, b)
  sfor<9>([&](auto L) {
    constexpr int a = L % 3, b = L / 3;
    fwd_line<P::p0(a, b, 0), P::p0(a, b, 1), P::p0(a, b, 2)>(c[E(a, b, 0)], c[E(a, b, 1)], c[E(a, b, 2)]);
  });
  // y sweep: lines over (a, g)
  sfor<9>([&](auto L) {
    constexpr int a = L % 3, g = L / 3;
    fwd_line<P::p1(a, 0, g), P::p1(a, 1, g), P::p1(a, 2, g)>(c[E(a, 0, g)], c[E(a, 1, g)], c[E(a, 2, g)]);
  });
  // x sweep: lines over (be, g)
  sfor<9>([&](auto L) {
    constexpr int be = L % 3, g = L / 3;
    fwd_line<P::p2(0, be, g), P::p2(1, be, g), P::p2(2, be, g)>(c[E(0, be, g)], c[E(1, be, g)],
                                                                 c[E(2, be, g)]);
  });
}

template <class real>
__device__ __forceinline__ void fwd_raw2(real (&c)[9]) {
  sfor<3>([&](auto a) { fwd_line<true, true, true>(c[E(a, 0)], c[E(a, 1)], c[E(a, 2)]); });  // y
  sfor<3>([&](auto b) { fwd_line<true, true, true>(c[E(0, b)], c[E(1, b)], c[E(2, b)]); });  // x
}

// backward per axis line: (m0, m1, m2) -> (f-, f0, f+)
template <class real>
__device__ __forceinline__ void bwd_line(real &c0, real &c1, real &c2) {
  const real m0 = c0, m2 = c2, h1 = real(0.5) * c1, h2 = real(0.5) * c2;
  c0 = h2 - h1;
  c2 = h2 + h1;
  c1 = m0 - m2;
}

template <class real>
__device__ __forceinline__ void bwd_raw3_full(real (&c)[27]) {
  sfor<9>([&](auto L) {
    constexpr int be = L % 3, g = L / 3;
    bwd_line(c[E(0, be, g)], c[E(1, be, g)], c[E(2, be, g)]);
  });
  sfor<9>([&](auto L) {
    constexpr int a = L % 3, g = L / 3;
    bwd_line(c[E(a, 0, g)], c[E(a, 1, g)], c[E(a, 2, g)]);
  });
  sfor<9>([&](auto L) {
    constexpr int a = L % 3, b = L / 3;
    bwd_line(c[E(a, b, 0)], c[E(a, b, 1)], c[E(a, b, 2)]);
  });
}

template <class real>
__device__ __forceinline__ void bwd_raw2(real (&c)[9]) {
  sfor<3>([&](auto b) { bwd_line(c[E(0, b)], c[E(1, b)], c[E(2, b)]); });
  sfor<3>([&](auto a) { bwd_line(c[E(a, 0)], c[E(a, 1)], c[E(a, 2)]); });
}

// D3Q19: f* = M^{-1} m* on the 19 basis monomials, as the symmetric/antisymmetric
// split over the 9 opposite pairs (eq:RawMomentChimeraBackwardSymmetric).
//   edges   f_{ab0} = (m220 + a m120 + b m210 + ab m110) / 4        (and xz, yz)
//   faces   f_{+-100} = ((m200 - m220 - m202) +- (m100 - m120 - m102)) / 2
//   rest    f_000 = m000 - (m200 + m020 + m002) + (m220 + m202 + m022)
// Output written to cube positions.
template <class real>
__device__ __forceinline__ void bwd_raw3_d3q19(real (&c)[27]) {
  const real m000 = c[E(0, 0, 0)];
  const real m100 = c[E(1, 0, 0)], m010 = c[E(0, 1, 0)], m001 = c[E(0, 0, 1)];
  const real m110 = c[E(1, 1, 0)], m101 = c[E(1, 0, 1)], m011 = c[E(0, 1, 1)];
  const real m200 = c[E(2, 0, 0)], m020 = c[E(0, 2, 0)], m002 = c[E(0, 0, 2)];
  const real m120 = c[E(1, 2, 0)], m102 = c[E(1, 0, 2)], m210 = c[E(2, 1, 0)];
  const real m012 = c[E(0, 1, 2)], m201 = c[E(2, 0, 1)], m021 = c[E(0, 2, 1)];
  const real m220 = c[E(2, 2, 0)], m202 = c[E(2, 0, 2)], m022 = c[E(0, 2, 2)];
  const real q = real(0.25), h = real(0.5);
  // xy edges: symmetric part (m220 + ab m110)/4, antisymmetric (a m120 + b m210)/4
  {
    const real sp = q * (m220 + m110), sm = q * (m220 - m110);
    const real ap = q * (m120 + m210), am = q * (m120 - m210);
    c[E(2, 2, 1)] = sp + ap;  // (+1,+1,0)
    c[E(0, 0, 1)] = sp - ap;  // (-1,-1,0)
    c[E(2, 0, 1)] = sm + am;  // (+1,-1,0)
    c[E(0, 2, 1)] = sm - am;  // (-1,+1,0)
  }
  {  // xz edges
    const real sp = q * (m202 + m101), sm = q * (m202 - m101);
    const real ap = q * (m102 + m201), am = q * (m102 - m201);
    c[E(2, 1, 2)] = sp + ap;
    c[E(0, 1, 0)] = sp - ap;
    c[E(2, 1, 0)] = sm + am;
    c[E(0, 1, 2)] = sm - am;
  }
  {  // yz edges
    const real sp = q * (m022 + m011), sm = q * (m022 - m011);
    const real ap = q * (m012 + m021), am = q * (m012 - m021);
    c[E(1, 2, 2)] = sp + ap;
    c[E(1, 0, 0)] = sp - ap;
    c[E(1, 2, 0)] = sm + am;
    c[E(1, 0, 2)] = sm - am;
  }
  {  // faces
    const real sx = h * (m200 - m220 - m202), ax = h * (m100 - m120 - m102);
    const real sy = h * (m020 - m220 - m022), ay = h * (m010 - m210 - m012);
    const real sz = h * (m002 - m202 - m022), az = h * (m001 - m201 - m021);
    c[E(2, 1, 1)] = sx + ax;
    c[E(0, 1, 1)] = sx - ax;
    c[E(1, 2, 1)] = sy + ay;
    c[E(1, 0, 1)] = sy - ay;
    c[E(1, 1, 2)] = sz + az;
    c[E(1, 1, 0)] = sz - az;
  }
  c[E(1, 1, 1)] = m000 - (m200 + m020 + m002) + (m220 + m202 + m022);
}

// --------------------------------------------------------------------------
// binomial Chimera
// --------------------------------------------------------------------------
template <class real>
__device__ __forceinline__ void bin_fwd_line(real &c0, real &c1, real &c2, real u) {
  const real k1 = fma(-u, c0, c1);
  c2 = fma(-u, c1 + k1, c2);  // m2 - 2u m1 + u^2 m0
  c1 = k1;
}
template <class real>
__device__ __forceinline__ void bin_bwd_line(real &c0, real &c1, real &c2, real u) {
  const real m1 = fma(u, c0, c1);
  c2 = fma(u, c1 + m1, c2);  // k2 + 2u k1 + u^2 k0
  c1 = m1;
}
template <class real>
__device__ __forceinline__ void bin_fwd3(real (&c)[27], real ux, real uy, real uz) {
  sfor<9>([&](auto L) {
    constexpr int a = L % 3, b = L / 3;
    bin_fwd_line(c[E(a, b, 0)], c[E(a, b, 1)], c[E(a, b, 2)], uz);
  });
  sfor<9>([&](auto L) {
    constexpr int a = L % 3, g = L / 3;
    bin_fwd_line(c[E(a, 0, g)], c[E(a, 1, g)], c[E(a, 2, g)], uy);
  });
  sfor<9>([&](auto L) {
    constexpr int be = L % 3, g = L / 3;
    bin_fwd_line(c[E(0, be, g)], c[E(1, be, g)], c[E(2, be, g)], ux);
  });
}
template <class real>
__device__ __forceinline__ void bin_bwd3(real (&c)[27], real ux, real uy, real uz) {
  sfor<9>([&](auto L) {
    constexpr int a = L % 3, b = L / 3;
    bin_bwd_line(c[E(a, b, 0)], c[E(a, b, 1)], c[E(a, b, 2)], uz);
  });
  sfor<9>([&](auto L) {
    constexpr int a = L % 3, g = L / 3;
    bin_bwd_line(c[E(a, 0, g)], c[E(a, 1, g)], c[E(a, 2, g)], uy);
  });
  sfor<9>([&](auto L) {
    constexpr int be = L % 3, g = L / 3;
    bin_bwd_line(c[E(0, be, g)], c[E(1, be, g)], c[E(2, be, g)], ux);
  });
}
template <class real>
__device__ __forceinline__ void bin_fwd2(real (&c)[9], real ux, real uy) {
  sfor<3>([&](auto a) { bin_fwd_line(c[E(a, 0)], c[E(a, 1)], c[E(a, 2)], uy); });
  sfor<3>([&](auto b) { bin_fwd_line(c[E(0, b)], c[E(1, b)], c[E(2, b)], ux); });
}
template <class real>
__device__ __forceinline__ void bin_bwd2(real (&c)[9], real ux, real uy) {
  sfor<3>([&](auto a) { bin_bwd_line(c[E(a, 0)], c[E(a, 1)], c[E(a, 2)], uy); });
  sfor<3>([&](auto b) { bin_bwd_line(c[E(0, b)], c[E(1, b)], c[E(2, b)], ux); });
}

// --------------------------------------------------------------------------
// equilibria in monomial form (template<int e> get(), static zero<e>())
// --------------------------------------------------------------------------
// Maxwellian raw moments truncated at O(u^2) (reading R4):
//   m_eq_e = rho (hprod(e) + U_e(u)), U_e = the u-terms of prod_a g_{e_a} cut at degree 2
//   (g0 = 1, g1 = u, g2 = cs2 + u^2).
template <class real>
struct RawU {
  real ux, uy, uz, uxx, uyy, uzz;
  template <int e>
  __device__ __forceinline__ real get() const {
    constexpr int ax = ex_of(e), ay = ey_of(e), az = ez_of(e);
    constexpr int n1 = n1_of(e), n2 = n2_of(e);
    if constexpr (n1 == 0) {
      // (1/3)^(n2-1) * sum of u_a^2 over the squared axes
      real s = real(0);
      bool first = true;
      if constexpr (ax == 2) { s = uxx; first = false; }
      if constexpr (ay == 2) { s = first ? uyy : s + uyy; first = false; }
      if constexpr (az == 2) { s = first ? uzz : s + uzz; }
      if constexpr (n2 == 1) return s;
      else return real(third_pow(n2 - 1)) * s;
    } else if constexpr (n1 == 1) {
      const real v = (ax == 1) ? ux : ((ay == 1) ? uy : uz);
      if constexpr (n2 == 0) return v;
      else return real(third_pow(n2)) * v;
    } else if constexpr (n1 == 2) {
      const real v = (ax != 1) ? uy * uz : ((ay != 1) ? ux * uz : ux * uy);
      if constexpr (n2 == 0) return v;
      else return real(third_pow(n2)) * v;
    } else {
      return real(0);
    }
  }
  template <int e>
  __device__ static constexpr bool zero() {
    return n1_of(e) == 3 || e == 0;
  }
};

// central-moment background prod_a k_{e_a}(u), k0 = 1, k1 = -u, k2 = cs2 + u^2, minus hprod(e):
//   V_e(u) = K(u) f0 - K(0) f0 on monomial e (closed form; exact for D2Q9/D3Q19/D3Q27)
template <class real>
struct CentralV {
  real ux, uy, uz, uxx, uyy, uzz;
  template <int a>
  __device__ __forceinline__ real k(real u, real uu) const {
    if constexpr (a == 0) return real(1);
    else if constexpr (a == 1) return -u;
    else return real(1.0 / 3.0) + uu;
  }
  template <int e>
  __device__ __forceinline__ real get() const {
    constexpr int ax = ex_of(e), ay = ey_of(e), az = ez_of(e);
    if constexpr (n1_of(e) == 0) {
      // prod (1/3 + u_a^2) - (1/3)^n2 over squared axes, expanded without cancellation
      constexpr int n2 = n2_of(e);
      if constexpr (n2 == 0) return real(0);
      real A[3];
      int n = 0;
      if constexpr (ax == 2) A[n++] = uxx;
      if constexpr (ay == 2) A[n++] = uyy;
      if constexpr (az == 2) A[n++] = uzz;
      if constexpr (n2 == 1) {
        return A[0];
      } else if constexpr (n2 == 2) {
        return fma(A[0], A[1], real(1.0 / 3.0) * (A[0] + A[1]));
      } else {
        const real s1 = A[0] + A[1] + A[2];
        const real s2 = A[0] * A[1] + A[0] * A[2] + A[1] * A[2];
        return fma(A[0] * A[1], A[2], fma(real(1.0 / 3.0), s2, real(1.0 / 9.0) * s1));
      }
    } else {
      return k<ax>(ux, uxx) * k<ay>(uy, uyy) * k<az>(uz, uzz);
    }
  }
};

// --------------------------------------------------------------------------
// relaxation helpers (delta = q_eq - q on monomials)
// --------------------------------------------------------------------------
template <class real>
__device__ __forceinline__ void relax1(real &m, real meq, real w) { m = fma(w, meq - m, m); }
template <class real>
__device__ __forceinline__ void relax1_zero(real &m, real w) { m = fma(-w, m, m); }
// polynomials (a + b) [ws], (a - b) [wd]
template <class real>
__device__ __forceinline__ void relax_pair(real &a, real &b, real da, real db, real ws, real wd) {
  const real S = ws * (da + db), D = wd * (da - db);
  a = fma(real(0.5), S + D, a);
  b = fma(real(0.5), S - D, b);
}
// polynomials (a - b) [w1], (a - c) [w2], (a + b + c) [w3]
template <class real>
__device__ __forceinline__ void relax_diag3(real &a, real &b, real &c, real da, real db, real dc, real w1,
                                            real w2, real w3) {
  const real E1 = w1 * (da - db), E2 = w2 * (da - dc), E3 = w3 * (da + db + dc);
  const real t = real(1.0 / 3.0);
  a = fma(t, E1 + E2 + E3, a);
  b = fma(t, E3 + E2 - real(2) * E1, b);
  c = fma(t, E3 + E1 - real(2) * E2, c);
}
// polynomials (a - 2b + c) [w1], (a + b - 2c) [w2], (a + b + c) [w3]
template <class real>
__device__ __forceinline__ void relax_quad3(real &a, real &b, real &c, real da, real db, real dc, real w1,
                                            real w2, real w3) {
  const real E1 = w1 * (da - real(2) * db + dc), E2 = w2 * (da + db - real(2) * dc), E3 = w3 * (da + db + dc);
  const real t = real(1.0 / 3.0);
  a = fma(t, E1 + E2 + E3, a);
  b = fma(t, E3 - E1, b);
  c = fma(t, E3 - E2, c);
}

// Rate specialisation: rates known to be one at
// compile time turn q* = q + w (q_eq - q) into q* = q_eq, so the forward transform of that
// quantity becomes dead code the compiler removes.
//   RS_GENERAL  every rate a runtime value
//   RS_REG      "fully regularised" (R- methods): all but the shear rates = 1
//   RS_HIGH     "higher-order regularised": rates of orders 5 and 6 = 1 (D3Q27)
enum { RS_GENERAL = 0, RS_REG = 1, RS_HIGH = 2 };

template <class S, int RS>
struct RateOf {
  // index of the first non-shear, non-conserved polynomial of the basis
  static constexpr int first_nonshear = (S::Q == 9) ? 5 : 9;
  template <int idx>
  __device__ static constexpr bool unit() {
    if constexpr (RS == RS_REG) return idx >= first_nonshear;
    else if constexpr (RS == RS_HIGH) return S::Q == 27 && idx >= 23;
    else return false;
  }
  template <int idx, class real>
  __device__ static __forceinline__ real get(const Rates<real> &r) {
    if constexpr (unit<idx>()) return real(1);
    else return r.w[idx];
  }
};

template <class EQ, int e, class real, int NC>
__device__ __forceinline__ real eq_value(const EQ &eq) {
  if constexpr (EQ::template zero<e>()) return real(0);
  else return eq.template get<e>();
}
template <class EQ, int e, class real, int NC>
__device__ __forceinline__ real delta_v(const EQ &eq, const real (&c)[NC]) {
  if constexpr (EQ::template zero<e>()) return -c[e];
  else return eq.template get<e>() - c[e];
}
template <class R, class EQ, int e, int idx, class real, int NC>
__device__ __forceinline__ void rs_single(const EQ &eq, real (&c)[NC], const Rates<real> &r) {
  if constexpr (R::template unit<idx>()) c[e] = eq_value<EQ, e, real, NC>(eq);
  else if constexpr (EQ::template zero<e>()) relax1_zero(c[e], r.w[idx]);
  else relax1(c[e], eq.template get<e>(), r.w[idx]);
}
// (a + b) [is], (a - b) [id]
template <class R, class EQ, int ea, int eb, int is, int id, class real, int NC>
__device__ __forceinline__ void rs_pair(const EQ &eq, real (&c)[NC], const Rates<real> &r) {
  if constexpr (R::template unit<is>() && R::template unit<id>()) {
    c[ea] = eq_value<EQ, ea, real, NC>(eq);
    c[eb] = eq_value<EQ, eb, real, NC>(eq);
  } else {
    const real da = delta_v<EQ, ea, real, NC>(eq, c), db = delta_v<EQ, eb, real, NC>(eq, c);
    relax_pair(c[ea], c[eb], da, db, R::template get<is>(r), R::template get<id>(r));
  }
}
template <class R, class EQ, int ea, int eb, int ec, int i1, int i2, int i3, bool QUAD, class real, int NC>
__device__ __forceinline__ void rs_triple(const EQ &eq, real (&c)[NC], const Rates<real> &r) {
  if constexpr (R::template unit<i1>() && R::template unit<i2>() && R::template unit<i3>()) {
    c[ea] = eq_value<EQ, ea, real, NC>(eq);
    c[eb] = eq_value<EQ, eb, real, NC>(eq);
    c[ec] = eq_value<EQ, ec, real, NC>(eq);
  } else {
    const real da = delta_v<EQ, ea, real, NC>(eq, c), db = delta_v<EQ, eb, real, NC>(eq, c),
               dc = delta_v<EQ, ec, real, NC>(eq, c);
    if constexpr (QUAD)
      relax_quad3(c[ea], c[eb], c[ec], da, db, dc, R::template get<i1>(r), R::template get<i2>(r),
                  R::template get<i3>(r));
    else
      relax_diag3(c[ea], c[eb], c[ec], da, db, dc, R::template get<i1>(r), R::template get<i2>(r),
                  R::template get<i3>(r));
  }
}

// Apply the basis relaxation of stencil S to the monomial cube c given an
// equilibrium provider EQ with get<e>() (value of q_eq on monomial e) and
// zero<e>() (compile-time: q_eq == 0).  Rate indices follow include/lbm.h.
template <class S, int RS, class EQ, class real>
__device__ __forceinline__ void relax_basis3(real (&c)[27], const EQ &eq, const Rates<real> &r) {
  using R = RateOf<S, RS>;
  constexpr bool Q27 = (S::Q == 27);
  // second order: xy, xz, yz [4,5,6]; (x^2-y^2, x^2-z^2, x^2+y^2+z^2) [7,8,9]
  rs_single<R, EQ, E(1, 1, 0), 4>(eq, c, r);
  rs_single<R, EQ, E(1, 0, 1), 5>(eq, c, r);
  rs_single<R, EQ, E(0, 1, 1), 6>(eq, c, r);
  rs_triple<R, EQ, E(2, 0, 0), E(0, 2, 0), E(0, 0, 2), 7, 8, 9, false>(eq, c, r);
  // third order pairs: (xy^2, xz^2) [10,13], (x^2y, yz^2) [11,14], (x^2z, y^2z) [12,15]
  rs_pair<R, EQ, E(1, 2, 0), E(1, 0, 2), 10, 13>(eq, c, r);
  rs_pair<R, EQ, E(2, 1, 0), E(0, 1, 2), 11, 14>(eq, c, r);
  rs_pair<R, EQ, E(2, 0, 1), E(0, 2, 1), 12, 15>(eq, c, r);
  if constexpr (Q27) {
    rs_single<R, EQ, E(1, 1, 1), 16>(eq, c, r);
    rs_triple<R, EQ, E(2, 2, 0), E(2, 0, 2), E(0, 2, 2), 17, 18, 19, true>(eq, c, r);
    rs_single<R, EQ, E(2, 1, 1), 20>(eq, c, r);
    rs_single<R, EQ, E(1, 2, 1), 21>(eq, c, r);
    rs_single<R, EQ, E(1, 1, 2), 22>(eq, c, r);
    rs_single<R, EQ, E(1, 2, 2), 23>(eq, c, r);
    rs_single<R, EQ, E(2, 1, 2), 24>(eq, c, r);
    rs_single<R, EQ, E(2, 2, 1), 25>(eq, c, r);
    rs_single<R, EQ, E(2, 2, 2), 26>(eq, c, r);
  } else {
    rs_triple<R, EQ, E(2, 2, 0), E(2, 0, 2), E(0, 2, 2), 16, 17, 18, true>(eq, c, r);
  }
}

// 2D (D2Q9, de Rosis basis): xy [3]; (x^2-y^2 [4], x^2+y^2 [5]); x^2y [6]; xy^2 [7]; x^2y^2 [8]
template <int RS, class EQ, class real>
__device__ __forceinline__ void relax_basis2(real (&c)[9], const EQ &eq, const Rates<real> &r) {
  using R = RateOf<D2Q9, RS>;
  rs_single<R, EQ, E(1, 1), 3>(eq, c, r);
  rs_pair<R, EQ, E(2, 0), E(0, 2), 5, 4>(eq, c, r);
  rs_single<R, EQ, E(2, 1), 6>(eq, c, r);
  rs_single<R, EQ, E(1, 2), 7>(eq, c, r);
  rs_single<R, EQ, E(2, 2), 8>(eq, c, r);
}

// --------------------------------------------------------------------------
// equilibrium providers
// --------------------------------------------------------------------------
// RAW, absolute: rho (hprod + U)
template <class real>
struct EqRawAbs {
  real rho;
  RawU<real> U;
  template <int e>
  __device__ __forceinline__ real get() const {
    constexpr double h = hprod(e);
    if constexpr (h != 0.0) return rho * (real(h) + U.template get<e>());
    else return rho * U.template get<e>();
  }
  template <int e>
  __device__ static constexpr bool zero() { return n1_of(e) == 3; }
};
// RAW, delta: drho hprod + rho U
template <class real>
struct EqRawDelta {
  real drho, rho;
  RawU<real> U;
  template <int e>
  __device__ __forceinline__ real get() const {
    constexpr double h = hprod(e);
    if constexpr (h != 0.0) return fma(real(h), drho, rho * U.template get<e>());
    else return rho * U.template get<e>();
  }
  template <int e>
  __device__ static constexpr bool zero() { return n1_of(e) == 3; }
};
// CENTRAL, absolute: Gaussian central moments rho hprod (u-independent, reading R4)
template <class real>
struct EqCentralAbs {
  real rho;
  template <int e>
  __device__ __forceinline__ real get() const { return real(hprod(e)) * rho; }
  template <int e>
  __device__ static constexpr bool zero() { return hprod(e) == 0.0; }
};
// CENTRAL, delta: dk_eq = rho hprod - K(u) f0 = drho hprod - V_e(u)
template <class real>
struct EqCentralDelta {
  real drho;
  CentralV<real> V;
  template <int e>
  __device__ __forceinline__ real get() const {
    constexpr double h = hprod(e);
    if constexpr (h != 0.0) return fma(real(h), drho, -V.template get<e>());
    else return -V.template get<e>();
  }
  template <int e>
  __device__ static constexpr bool zero() { return false; }
};
// CUMULANT: C_eq = rho cs2 on the diagonal second-order cumulants, 0 otherwise
template <class real>
struct EqCumulant {
  real rho3;  // rho / 3
  template <int e>
  __device__ __forceinline__ real get() const { return rho3; }
  template <int e>
  __device__ static constexpr bool zero() {
    return !(n2_of(e) == 1 && n1_of(e) == 0);
  }
};
// SWE, central moments kappa_eq = K(u) f_eq of Zhou's discrete equilibrium (PAPER.md:485-487,
// 1001-1012; corrected u.u/6 of reading R5) in closed form (expanded symbolically from
// eq:DiscreteShallowWaterEquilibrium): kappa_20 = kappa_02 = g h^2 / 2,
// kappa_11 = 0, kappa_21 = h u_y (1/3 - g h / 2 - u_x^2), kappa_12 = h u_x (1/3 - g h / 2 - u_y^2),
// kappa_22 = h (g h / 6 + (g h / 2 - 1/3) u.u + 3 u_x^2 u_y^2).  Replaces the transform of the
// nine f_eq values through both Chimera sweeps (186 -> ~110 fp64 instructions per cell).
template <class real>
struct EqSweZhou {
  real k20, k21, k12, k22;
  __device__ __forceinline__ EqSweZhou(real h, real ux, real uy, real g) {
    const real gh = g * h, a = fma(real(-0.5), gh, real(1.0 / 3.0));  // 1/3 - g h / 2
    const real uxx = ux * ux, uyy = uy * uy;
    k20 = real(0.5) * gh * h;
    k21 = h * uy * (a - uxx);
    k12 = h * ux * (a - uyy);
    k22 = h * fma(real(3) * uxx, uyy, fma(real(1.0 / 6.0), gh, -a * (uxx + uyy)));
  }
  template <int e>
  __device__ __forceinline__ real get() const {
    if constexpr (e == E(2, 0) || e == E(0, 2)) return k20;
    else if constexpr (e == E(2, 1)) return k21;
    else if constexpr (e == E(1, 2)) return k12;
    else {
      static_assert(e == E(2, 2), "SWE equilibrium: second- to fourth-order central moments only");
      return k22;
    }
  }
  template <int e>
  __device__ static constexpr bool zero() { return e == E(1, 1); }
};

// tabulated equilibrium (q_eq = T(f_eq) computed numerically)
template <class real, int N>
struct EqTable {
  real v[N];
  template <int e>
  __device__ __forceinline__ real get() const { return v[e]; }
  template <int e>
  __device__ static constexpr bool zero() { return false; }
};

// --------------------------------------------------------------------------
// cumulant closed forms (3D).  c holds central moments kappa on entry
// (kappa_000 = rho, first order = 0); 'inv' = 1/rho.
// --------------------------------------------------------------------------
template <class S, class real>
__device__ __forceinline__ void central_to_cumulant3(real (&c)[27], real inv) {
  const real k200 = c[E(2, 0, 0)], k020 = c[E(0, 2, 0)], k002 = c[E(0, 0, 2)];
  const real k110 = c[E(1, 1, 0)], k101 = c[E(1, 0, 1)], k011 = c[E(0, 1, 1)];
  if constexpr (S::Q == 27) {
    const real k111 = c[E(1, 1, 1)];
    const real k210 = c[E(2, 1, 0)], k201 = c[E(2, 0, 1)], k120 = c[E(1, 2, 0)];
    const real k021 = c[E(0, 2, 1)], k102 = c[E(1, 0, 2)], k012 = c[E(0, 1, 2)];
    const real k220 = c[E(2, 2, 0)], k202 = c[E(2, 0, 2)], k022 = c[E(0, 2, 2)];
    const real k211 = c[E(2, 1, 1)], k121 = c[E(1, 2, 1)], k112 = c[E(1, 1, 2)];
    // order 6 (uses the central moments of order 4 before they are overwritten)
    {
      const real s24 = k200 * k022 + k020 * k202 + k002 * k220 +
                       real(4) * (k110 * k112 + k101 * k121 + k011 * k211);
      const real s33 = real(2) * (k210 * k012 + k201 * k021 + k120 * k102) + real(4) * k111 * k111;
      const real s222 = k200 * k020 * k002 +
                        real(2) * (k200 * k011 * k011 + k020 * k101 * k101 + k002 * k110 * k110) +
                        real(8) * k110 * k101 * k011;
      c[E(2, 2, 2)] = c[E(2, 2, 2)] - inv * (s24 + s33) + real(2) * inv * inv * s222;
    }
    // order 5
    c[E(2, 2, 1)] -= inv * (k200 * k021 + k020 * k201 + real(4) * k110 * k111 +
                            real(2) * (k101 * k120 + k011 * k210));
    c[E(2, 1, 2)] -= inv * (k200 * k012 + k002 * k210 + real(4) * k101 * k111 +
                            real(2) * (k110 * k102 + k011 * k201));
    c[E(1, 2, 2)] -= inv * (k020 * k102 + k002 * k120 + real(4) * k011 * k111 +
                            real(2) * (k110 * k012 + k101 * k021));
    // order 4 (mixed)
    c[E(2, 1, 1)] -= inv * (k200 * k011 + real(2) * k110 * k101);
    c[E(1, 2, 1)] -= inv * (k020 * k101 + real(2) * k110 * k011);
    c[E(1, 1, 2)] -= inv * (k002 * k110 + real(2) * k101 * k011);
  }
  // order 4 (squares)
  c[E(2, 2, 0)] -= inv * (k200 * k020 + real(2) * k110 * k110);
  c[E(2, 0, 2)] -= inv * (k200 * k002 + real(2) * k101 * k101);
  c[E(0, 2, 2)] -= inv * (k020 * k002 + real(2) * k011 * k011);
}

// inverse: c holds post-collision cumulants C* (orders 2, 3 equal kappa*)
template <class S, class real>
__device__ __forceinline__ void cumulant_to_central3(real (&c)[27], real inv) {
  const real k200 = c[E(2, 0, 0)], k020 = c[E(0, 2, 0)], k002 = c[E(0, 0, 2)];
  const real k110 = c[E(1, 1, 0)], k101 = c[E(1, 0, 1)], k011 = c[E(0, 1, 1)];
  c[E(2, 2, 0)] += inv * (k200 * k020 + real(2) * k110 * k110);
  c[E(2, 0, 2)] += inv * (k200 * k002 + real(2) * k101 * k101);
  c[E(0, 2, 2)] += inv * (k020 * k002 + real(2) * k011 * k011);
  if constexpr (S::Q == 27) {
    const real k111 = c[E(1, 1, 1)];
    const real k210 = c[E(2, 1, 0)], k201 = c[E(2, 0, 1)], k120 = c[E(1, 2, 0)];
    const real k021 = c[E(0, 2, 1)], k102 = c[E(1, 0, 2)], k012 = c[E(0, 1, 2)];
    c[E(2, 1, 1)] += inv * (k200 * k011 + real(2) * k110 * k101);
    c[E(1, 2, 1)] += inv * (k020 * k101 + real(2) * k110 * k011);
    c[E(1, 1, 2)] += inv * (k002 * k110 + real(2) * k101 * k011);
    c[E(2, 2, 1)] += inv * (k200 * k021 + k020 * k201 + real(4) * k110 * k111 +
                            real(2) * (k101 * k120 + k011 * k210));
    c[E(2, 1, 2)] += inv * (k200 * k012 + k002 * k210 + real(4) * k101 * k111 +
                            real(2) * (k110 * k102 + k011 * k201));
    c[E(1, 2, 2)] += inv * (k020 * k102 + k002 * k120 + real(4) * k011 * k111 +
                            real(2) * (k110 * k012 + k101 * k021));
    const real k220 = c[E(2, 2, 0)], k202 = c[E(2, 0, 2)], k022 = c[E(0, 2, 2)];
    const real k211 = c[E(2, 1, 1)], k121 = c[E(1, 2, 1)], k112 = c[E(1, 1, 2)];
    const real s24 = k200 * k022 + k020 * k202 + k002 * k220 +
                     real(4) * (k110 * k112 + k101 * k121 + k011 * k211);
    const real s33 = real(2) * (k210 * k012 + k201 * k021 + k120 * k102) + real(4) * k111 * k111;
    const real s222 = k200 * k020 * k002 +
                      real(2) * (k200 * k011 * k011 + k020 * k101 * k101 + k002 * k110 * k110) +
                      real(8) * k110 * k101 * k011;
    c[E(2, 2, 2)] = c[E(2, 2, 2)] + inv * (s24 + s33) - real(2) * inv * inv * s222;
  }
}

template <class real>
__device__ __forceinline__ void central_to_cumulant2(real (&c)[9], real inv) {
  const real k20 = c[E(2, 0)], k02 = c[E(0, 2)], k11 = c[E(1, 1)];
  c[E(2, 2)] -= inv * (k20 * k02 + real(2) * k11 * k11);
}
template <class real>
__device__ __forceinline__ void cumulant_to_central2(real (&c)[9], real inv) {
  const real k20 = c[E(2, 0)], k02 = c[E(0, 2)], k11 = c[E(1, 1)];
  c[E(2, 2)] += inv * (k20 * k02 + real(2) * k11 * k11);
}

// --------------------------------------------------------------------------
// background raw moments m0_e = hprod(e) (= M f0) add/remove
// --------------------------------------------------------------------------
template <int NC, class real>
__device__ __forceinline__ void add_background(real (&c)[NC], real sgn) {
  sfor<NC>([&](auto e) {
    constexpr double h = hprod(e);
    if constexpr (e != 0 && h != 0.0) c[e] = fma(sgn, real(h), c[e]);
  });
}

// Zero-centered shallow water (reading R33): the background is the method's
// own rest state f0 = f_eq(h0 = 1, u = 0) — Zhou's discrete equilibrium (SPACE_SWE,
// PAPER.md:1001-1012) or the Maxwellian at cs2 = g h0 / 2 (SPACE_SWE_K).
// Its non-zero raw moments besides m_00 = 1: m_20 = m_02 = g/2; m_22 = g/6 (Zhou) or
// (g/2)^2 (Maxwellian).
template <int SPACE, class real>
__device__ __forceinline__ real swe_bg_m22(real g) {
  if constexpr (SPACE == SPACE_SWE_K) return real(0.25) * g * g;
  else return g * real(1.0 / 6.0);
}
template <int SPACE, int NC, class real>
__device__ __forceinline__ void add_background_swe(real (&c)[NC], real sgn, real g) {
  c[E(2, 0, 0)] = fma(sgn, real(0.5) * g, c[E(2, 0, 0)]);
  c[E(0, 2, 0)] = fma(sgn, real(0.5) * g, c[E(0, 2, 0)]);
  c[E(2, 2, 0)] = fma(sgn, swe_bg_m22<SPACE>(g), c[E(2, 2, 0)]);
}

// --------------------------------------------------------------------------
// the collision of one cell: f in/out in the documented population order,
// STORED form (delta f for REG_DELTA / REG_ZC_ABS).
// --------------------------------------------------------------------------
// --------------------------------------------------------------------------
// body force (reading R23; Guo et al. 2002, the paper's q^F):
// u = (j + F/2) / rho, and the source q^F = (I - S/2) T(F^G) of the discrete Guo term
// F^G_i = w_i [3 xi.F + 9 (xi.u)(xi.F) - 3 u.F] is added after relaxation.  The momentum
// gains exactly F (kappa_100: -F/2 before, +F/2 after).
// --------------------------------------------------------------------------
enum { RS_FORCE = 4, RS_FORCE_HE = 8 };  // flag bits of the RS template parameter (Guo / He)
enum { RS_DISCRETE = 16 };               // equilibrium given as a discrete f_eq (reading R29)
// zero-centered storage relaxed against the absolute equilibrium with the background added to
// the POPULATIONS, q = T(df + f0), the literal eq:MrtUpdateAbsoluteFromZeroCentered (PAPER.md:
// 310-319; reading R30) instead of the closed-form background moments of REG_ZC_ABS
enum { RS_POPBG = 32 };
// raw moments relaxed in the weighted-orthogonal basis (WO-MRT; reading R31):
// the weighted Gram-Schmidt orthogonalisation of the graded-lexicographic monomials, one rate
// per polynomial, applied through the monomial-space matrices of wo_basis (constant memory)
enum { RS_WOBASIS = 64 };

// WO-MRT basis of the stencil in monomial (cube) coordinates: L[p][e] = coefficient of monomial e
// in polynomial p (p in graded-lexicographic order), Linv = L^{-1} (set by the host per device,
// OpsImpl::set_wo; each translation unit has its own copy)
__constant__ double c_wo_L[27 * 27];
__constant__ double c_wo_Linv[27 * 27];

// monomials of the stencil's raw-moment space (cube positions): all 27 / 9, D3Q19 without xyz-type
// monomials and orders >= 5 (rank 19, reading R2)
template <class S>
__host__ __device__ constexpr bool mono_present(int e) {
  if constexpr (S::Q != 19) return true;
  else return (ex_of(e) + ey_of(e) + ez_of(e) <= 4) && !(ex_of(e) >= 1 && ey_of(e) >= 1 && ez_of(e) >= 1);
}

// graded-lexicographic position of monomial e among the stencil's raw-moment monomials: the
// index of the WO polynomial whose leading monomial is e (and of its rate; wo_basis order)
template <class S>
__host__ __device__ constexpr int wo_index(int e) {
  int k = 0;
  for (int deg = 0; deg <= 6; ++deg)
    for (int a = 2; a >= 0; --a)
      for (int b = 2; b >= 0; --b)
        for (int z = 2; z >= 0; --z) {
          if (a + b + z != deg || (S::D == 2 && z > 0) || !mono_present<S>(a + 3 * b + 9 * z)) continue;
          if (a + 3 * b + 9 * z == e) return k;
          ++k;
        }
  return -1;
}

// one axis of the Hermite factor {1, t, t^2 - 1/3}: L (sgn = -1) or L^{-1} (sgn = +1) along axis
// `ax` of the moment cube: c[.. 2 ..] += sgn / 3 * c[.. 0 ..]
template <int ax, int NC, class real>
__device__ __forceinline__ void hermite_axis(real (&c)[NC], real sgn) {
  constexpr int st = ax == 0 ? 1 : (ax == 1 ? 3 : 9);
  sfor<NC>([&](auto e) {
    constexpr int ie = e;
    constexpr int digit = (ie / st) % 3;
    if constexpr (digit == 2) c[e] = fma(sgn * real(1.0 / 3.0), c[ie - 2 * st], c[e]);
  });
}

// q* = q + S (q_eq - q) with q = L m (reading R31): m* = m + L^{-1} S L (m_eq - m)
template <class S, class EQ, class real, int NC>
__device__ __forceinline__ void relax_wo(real (&c)[NC], const EQ &eq, const Rates<real> &r) {
  real d[NC];
  sfor<NC>([&](auto e) {
    if constexpr (mono_present<S>(e)) {
      if constexpr (EQ::template zero<e>()) d[e] = -c[e];
      else d[e] = eq.template get<e>() - c[e];
    }
  });
  if constexpr (S::Q == 27 || S::Q == 9) {
    // product lattices: the WO basis is the tensor-product monic Hermite basis {1, t, t^2 - 1/3}
    // per axis (pinned: test_wo_basis_is_hermite_on_product_lattices), so L = L1 (x) L1 (x) L1 is
    // three axis sweeps, L^{-1} likewise — 2 x 9 d FMAs instead of the dense 2 q^2
    hermite_axis<0>(d, real(-1));
    hermite_axis<1>(d, real(-1));
    if constexpr (S::D == 3) hermite_axis<2>(d, real(-1));
    sfor<NC>([&](auto e) { d[e] = r.w[wo_index<S>(e)] * d[e]; });
    hermite_axis<0>(d, real(1));
    hermite_axis<1>(d, real(1));
    if constexpr (S::D == 3) hermite_axis<2>(d, real(1));
    sfor<NC>([&](auto e) { c[e] += d[e]; });
    return;
  }
  real t[S::Q];
  sfor<S::Q>([&](auto p) {
    real acc = real(0);
    sfor<NC>([&](auto e) {
      if constexpr (mono_present<S>(e)) acc = fma(real(c_wo_L[p * 27 + e]), d[e], acc);
    });
    t[p] = r.w[p] * acc;
  });
  sfor<NC>([&](auto e) {
    if constexpr (mono_present<S>(e)) {
      real acc = c[e];
      sfor<S::Q>([&](auto p) { acc = fma(real(c_wo_Linv[e * 27 + p]), t[p], acc); });
      c[e] = acc;
    }
  });
}

template <class real>
struct Force {
  real F[3];         // force density along the physical axes (2D: x, y)
  Rates<real> half;  // w / 2 per polynomial: the S/2 of (I - S/2)
};

template <class real>
struct EqZeroAll {
  template <int e>
  __device__ __forceinline__ real get() const { return real(0); }
  template <int e>
  __device__ static constexpr bool zero() { return true; }
};

// (written with explicit fma and exact signed sums so that no kernel context can contract it
// differently: the fused two-step kernel must reproduce the single-step bits)
template <int v, class real>
__device__ __forceinline__ real signed_add(real acc, real a) {
  if constexpr (v > 0) return acc + a;
  else if constexpr (v < 0) return acc - a;
  else return acc;
}

// Discrete second-order equilibrium f_eq_i = w_i rho [1 + X_i], X_i = 3 xi.u + 9/2 (xi.u)^2 -
// 3/2 u.u (reading R29) in the cube layout, in absolute form or as the
// deviation f_eq - w = w (drho + rho X) written without the cancellation.
template <class S, class real, int NC>
__device__ __forceinline__ void discrete_feq_cube(real (&fe)[NC], real rho, real ux, real uy, real uz,
                                                  bool deviation) {
  const real uu = fma(uz, uz, fma(uy, uy, ux * ux));
  const real drho = rho - real(1);
  sfor<NC>([&](auto k) { fe[k] = real(0); });
  sfor<S::Q>([&](auto i) {
    constexpr int vx = S::vx(i), vy = S::vy(i), vz = S::vz(i);
    const real cu = signed_add<vz>(signed_add<vy>(signed_add<vx>(real(0), ux), uy), uz);
    const real X = fma(real(4.5) * cu, cu, fma(real(3), cu, real(-1.5) * uu));
    const real wi = real(weight<S>(i));
    fe[S::pos(i)] = deviation ? wi * fma(rho, X, drho) : wi * fma(rho, X, rho);
  });
}
template <class S, class real, int NC>
__device__ __forceinline__ void guo_cube(real (&s)[NC], const Force<real> &fr, real ux, real uy, real uz) {
  const real uF = fma(uz, fr.F[2], fma(uy, fr.F[1], ux * fr.F[0]));
  sfor<NC>([&](auto k) { s[k] = real(0); });
  sfor<S::Q>([&](auto i) {
    constexpr int vx = S::vx(i), vy = S::vy(i), vz = S::vz(i);
    const real xF = signed_add<vz>(signed_add<vy>(signed_add<vx>(real(0), fr.F[0]), fr.F[1]), fr.F[2]);
    const real xu = signed_add<vz>(signed_add<vy>(signed_add<vx>(real(0), ux), uy), uz);
    s[S::pos(i)] = real(weight<S>(i)) * fma(real(9) * xu, xF, real(3) * (xF - uF));
  });
}

template <class S, int SPACE, int REG, class real, bool DISC = false>
__device__ __forceinline__ void equilibrium(real (&f)[S::Q], real rho, real ux, real uy, real uz, real swe_g);

// He's force term F^He_i = f_eq_i(rho, u) (xi_i - u).F / (rho c_s^2) (He, Shan, Doolen 1998,
// PAPER.md:214, 539; reading R27) with the method's own absolute equilibrium at the shifted u,
// in the cube layout like guo_cube.
template <class S, int SPACE, class real, int NC>
__device__ __forceinline__ void he_cube(real (&s)[NC], const Force<real> &fr, real rho, real inv, real ux,
                                        real uy, real uz) {
  real fe[S::Q];
  equilibrium<S, (SPACE == SPACE_CENTRAL ? SPACE_CENTRAL : SPACE_RAW), REG_ABS, real>(fe, rho, ux, uy, uz,
                                                                                       real(0));
  const real uF = fma(uz, fr.F[2], fma(uy, fr.F[1], ux * fr.F[0]));
  const real k = real(3) * inv;  // 1 / (rho c_s^2)
  sfor<NC>([&](auto e) { s[e] = real(0); });
  sfor<S::Q>([&](auto i) {
    constexpr int vx = S::vx(i), vy = S::vy(i), vz = S::vz(i);
    const real xF = signed_add<vz>(signed_add<vy>(signed_add<vx>(real(0), fr.F[0]), fr.F[1]), fr.F[2]);
    s[S::pos(i)] = fe[i] * ((xF - uF) * k);
  });
}

template <class S, int SPACE, int RS, class real, int NC>
__device__ __forceinline__ void force_cube(real (&s)[NC], const Force<real> &fr, real rho, real inv, real ux,
                                           real uy, real uz) {
  if constexpr ((RS & RS_FORCE_HE) != 0) he_cube<S, SPACE>(s, fr, rho, inv, ux, uy, uz);
  else guo_cube<S>(s, fr, ux, uy, uz);
}

template <class S, int SPACE, int REG, class real, int RS = RS_GENERAL>
__device__ __forceinline__ void collide(real (&f)[S::Q], const Rates<real> &r, real swe_g,
                                        const Force<real> &fr) {
  constexpr bool zc = (REG != REG_ABS);
  constexpr int NC = S::NC;
  constexpr bool FORCED = (RS & (RS_FORCE | RS_FORCE_HE)) != 0;
  constexpr bool DISC = (RS & RS_DISCRETE) != 0;  // q_eq = T(f_eq) of the discrete f_eq (R29)
  static_assert(!DISC || (SPACE != SPACE_SWE && SPACE != SPACE_SWE_K && !FORCED),
                "discrete hydrodynamic equilibrium: unforced, not for shallow water");
  // the discrete f_eq in the regime's form: deviation for zc + delta, absolute otherwise
  // (moment-space kernels add the background to q for zc + absolute equilibrium)
  auto disc_cube = [&](real(&fe)[NC], real rho_, real ux_, real uy_, real uz_) {
    discrete_feq_cube<S>(fe, rho_, ux_, uy_, uz_, REG == REG_DELTA);
  };
  static_assert(!(RS & RS_FORCE_HE) || SPACE == SPACE_POPULATION || SPACE == SPACE_RAW || SPACE == SPACE_CENTRAL,
                "He forcing: population, raw- and central-moment collisions (cumulants: R26 = Guo)");
  static_assert(!FORCED || SPACE == SPACE_POPULATION || SPACE == SPACE_RAW || SPACE == SPACE_CENTRAL ||
                    SPACE == SPACE_CUMULANT,
                "forcing is provided for population, raw-moment, central-moment and cumulant collisions");
  // cumulants (reading R26): the source is F on the first-order cumulants only.  Cumulants of
  // order >= 2 do not depend on the frame, so the forward transform is taken
  // about u0 = j / rho (kappa_100 = 0) instead of the shifted u = (j + F/2)/rho
  // (kappa_100 = -F_x/2), and the backward one about the post-collision mean (j + F)/rho.
  constexpr bool SHIFT_U = FORCED && SPACE != SPACE_CUMULANT;
  constexpr int RSR = RS & 3;  // rate specialisation proper
  if constexpr ((RS & RS_POPBG) != 0) {
    // literal eq:MrtUpdateAbsoluteFromZeroCentered (reading R30): df + f0 in the populations,
    // the absolute-storage collision, minus f0
    static_assert(REG == REG_ZC_ABS, "the population-space background is a zero-centered regime");
    sfor<S::Q>([&](auto i) { f[i] = f[i] + real(weight<S>(i)); });
    collide<S, SPACE, REG_ABS, real, (RS & ~RS_POPBG)>(f, r, swe_g, fr);
    sfor<S::Q>([&](auto i) { f[i] = f[i] - real(weight<S>(i)); });
    return;
  }
  real c[NC];
  sfor<NC>([&](auto k) { c[k] = real(0); });
  sfor<S::Q>([&](auto i) { c[S::pos(i)] = f[i]; });

  if constexpr (SPACE == SPACE_POPULATION) {
    // SRT (BGK): f* = f + w (f_eq - f), f_eq = M^{-1} m_eq (reading R4)
    if constexpr (S::D == 3) fwd_raw3<S>(c); else fwd_raw2(c);
    const real m000 = c[0];
    const real rho = zc ? real(1) + m000 : m000;
    const real inv = real(1) / rho;
    const real jx = c[E(1, 0, 0)], jy = c[E(0, 1, 0)];
    real jz = real(0);
    if constexpr (S::D == 3) jz = c[E(0, 0, 1)];
    real ux = jx * inv, uy = jy * inv, uz = jz * inv;
    if constexpr (FORCED) {
      ux = fma(real(0.5) * fr.F[0], inv, ux);
      uy = fma(real(0.5) * fr.F[1], inv, uy);
      uz = fma(real(0.5) * fr.F[2], inv, uz);
    }
    RawU<real> U{ux, uy, uz, ux * ux, uy * uy, uz * uz};
    real g[NC];
    if constexpr (DISC) {  // the discrete f_eq directly, stored form (f_eq - f0 when zero-centered)
      discrete_feq_cube<S>(g, rho, ux, uy, uz, zc);
    } else {
      if constexpr (REG == REG_DELTA) {
        EqRawDelta<real> eq{m000, rho, U};
        sfor<NC>([&](auto e) {
          if constexpr (EqRawDelta<real>::template zero<e>()) g[e] = real(0);
          else g[e] = eq.template get<e>();
        });
        g[0] = m000;
      } else {
        EqRawAbs<real> eq{rho, U};
        sfor<NC>([&](auto e) {
          if constexpr (EqRawAbs<real>::template zero<e>()) g[e] = real(0);
          else g[e] = eq.template get<e>();
        });
        g[0] = rho;
        if constexpr (REG == REG_ZC_ABS) add_background<NC>(g, real(-1)), g[0] = m000;  // f_eq - f0
      }
      if constexpr (S::Q == 27) bwd_raw3_full(g);
      else if constexpr (S::Q == 19) bwd_raw3_d3q19(g);
      else bwd_raw2(g);
    }
    const real w = r.w[0];
    if constexpr (REG == REG_ZC_ABS) {
      // absolute populations f = df + f0 relaxed against the absolute f_eq
      sfor<S::Q>([&](auto i) {
        const real f0 = real(weight<S>(i));
        const real fa = f[i] + f0;
        const real feq = g[S::pos(i)] + f0;
        f[i] = fma(w, feq - fa, fa) - f0;
      });
    } else {
      sfor<S::Q>([&](auto i) { f[i] = fma(w, g[S::pos(i)] - f[i], f[i]); });
    }
    if constexpr (FORCED) {  // + (1 - w/2) F^G_i
      real s[NC];
      force_cube<S, SPACE, RS>(s, fr, rho, inv, ux, uy, uz);
      const real a = real(1) - fr.half.w[0];
      sfor<S::Q>([&](auto i) { f[i] = fma(a, s[S::pos(i)], f[i]); });
    }
    return;
  } else {
    // ---- forward raw Chimera
    if constexpr (S::D == 3) fwd_raw3<S>(c); else fwd_raw2(c);
    // ---- conserved quantities, conserved-quantity rewriting
    const real m000 = c[0];
    const real rho = zc ? real(1) + m000 : m000;
    const real inv = real(1) / rho;
    const real jx = c[E(1, 0, 0)], jy = c[E(0, 1, 0)];
    real jz = real(0);
    if constexpr (S::D == 3) jz = c[E(0, 0, 1)];
    real ux = jx * inv, uy = jy * inv, uz = jz * inv;
    if constexpr (SHIFT_U) {  // u = (j + F/2) / rho
      ux = fma(real(0.5) * fr.F[0], inv, ux);
      uy = fma(real(0.5) * fr.F[1], inv, uy);
      uz = fma(real(0.5) * fr.F[2], inv, uz);
    }
    constexpr bool SWEZ = (SPACE == SPACE_SWE || SPACE == SPACE_SWE_K);
    if constexpr (REG == REG_ZC_ABS) {  // q = T(df + f0): add m0 = M f0
      if constexpr (SWEZ) add_background_swe<SPACE>(c, real(1), swe_g);
      else add_background<NC>(c, real(1));
      c[0] = rho;
    }
    // source term q^F = (I - S/2) T(F^G) added after relaxation (FORCED only)
    auto add_force = [&](auto central) {
      real s[NC];
      force_cube<S, SPACE, RS>(s, fr, rho, inv, ux, uy, uz);
      if constexpr (S::D == 3) fwd_raw3<S>(s); else fwd_raw2(s);
      if constexpr (decltype(central)::value) {
        if constexpr (S::D == 3) bin_fwd3(s, ux, uy, uz); else bin_fwd2(s, ux, uy);
      }
      EqZeroAll<real> z;
      if constexpr (S::D == 3) relax_basis3<S, RSR>(s, z, fr.half); else relax_basis2<RSR>(s, z, fr.half);
      sfor<NC>([&](auto e) { c[e] += s[e]; });
    };

    if constexpr (SPACE == SPACE_RAW && DISC) {
      EqTable<real, NC> eq;  // m_eq = M f_eq
      disc_cube(eq.v, rho, ux, uy, uz);
      if constexpr (S::D == 3) fwd_raw3<S>(eq.v); else fwd_raw2(eq.v);
      if constexpr (S::D == 3) relax_basis3<S, RSR>(c, eq, r); else relax_basis2<RSR>(c, eq, r);
    } else if constexpr (SPACE == SPACE_RAW && (RS & RS_WOBASIS) != 0) {
      static_assert(RSR == RS_GENERAL && !FORCED, "WO-MRT: general rates, unforced");
      RawU<real> U{ux, uy, uz, ux * ux, uy * uy, uz * uz};
      if constexpr (REG == REG_DELTA) relax_wo<S>(c, EqRawDelta<real>{m000, rho, U}, r);
      else relax_wo<S>(c, EqRawAbs<real>{rho, U}, r);
    } else if constexpr (SPACE == SPACE_RAW) {
      RawU<real> U{ux, uy, uz, ux * ux, uy * uy, uz * uz};
      if constexpr (REG == REG_DELTA) {
        EqRawDelta<real> eq{m000, rho, U};
        if constexpr (S::D == 3) relax_basis3<S, RSR>(c, eq, r); else relax_basis2<RSR>(c, eq, r);
      } else {
        EqRawAbs<real> eq{rho, U};
        if constexpr (S::D == 3) relax_basis3<S, RSR>(c, eq, r); else relax_basis2<RSR>(c, eq, r);
      }
      if constexpr (FORCED) add_force(std::false_type{});
    } else {
      // ---- raw -> central (binomial Chimera)
      if constexpr (S::D == 3) bin_fwd3(c, ux, uy, uz); else bin_fwd2(c, ux, uy);
      if constexpr (REG != REG_DELTA) {
        // collapse conserved central moments: kappa_000 = rho, kappa_100 = -F_x/2 (= 0 without a
        // force)
        c[0] = rho;
        c[E(1, 0, 0)] = SHIFT_U ? real(-0.5) * fr.F[0] : real(0);
        c[E(0, 1, 0)] = SHIFT_U ? real(-0.5) * fr.F[1] : real(0);
        if constexpr (S::D == 3) c[E(0, 0, 1)] = SHIFT_U ? real(-0.5) * fr.F[2] : real(0);
      }
      if constexpr (SPACE == SPACE_CENTRAL && DISC) {
        EqTable<real, NC> eq;  // kappa_eq = K(u) f_eq
        disc_cube(eq.v, rho, ux, uy, uz);
        if constexpr (S::D == 3) fwd_raw3<S>(eq.v); else fwd_raw2(eq.v);
        if constexpr (S::D == 3) bin_fwd3(eq.v, ux, uy, uz); else bin_fwd2(eq.v, ux, uy);
        if constexpr (S::D == 3) relax_basis3<S, RSR>(c, eq, r); else relax_basis2<RSR>(c, eq, r);
      } else if constexpr (SPACE == SPACE_CENTRAL) {
        if constexpr (REG == REG_DELTA) {
          EqCentralDelta<real> eq{m000, CentralV<real>{ux, uy, uz, ux * ux, uy * uy, uz * uz}};
          if constexpr (S::D == 3) relax_basis3<S, RSR>(c, eq, r); else relax_basis2<RSR>(c, eq, r);
        } else {
          EqCentralAbs<real> eq{rho};
          if constexpr (S::D == 3) relax_basis3<S, RSR>(c, eq, r); else relax_basis2<RSR>(c, eq, r);
        }
        // kappa*_100 = kappa_100 + F_x: -F_x/2 -> +F_x/2
        if constexpr (FORCED) add_force(std::true_type{});
      } else if constexpr (SPACE == SPACE_SWE) {
        // kappa_eq = K(u) f_eq of Zhou's discrete equilibrium,
        // closed form (EqSweZhou)
        static_assert(S::Q == 9, "SWE is D2Q9");
        const EqSweZhou<real> eq(rho, ux, uy, swe_g);
        relax_basis2<RSR>(c, eq, r);
      } else {  // SPACE_CUMULANT
        if constexpr (S::D == 3) central_to_cumulant3<S>(c, inv); else central_to_cumulant2(c, inv);
        // C_eq = rho cs2 on the diagonal: cs2 = 1/3, or g h / 2 for shallow water (h = rho)
        if constexpr (DISC) {  // C_eq: the cumulants of the discrete f_eq
          EqTable<real, NC> eq;
          disc_cube(eq.v, rho, ux, uy, uz);
          if constexpr (S::D == 3) fwd_raw3<S>(eq.v); else fwd_raw2(eq.v);
          if constexpr (S::D == 3) bin_fwd3(eq.v, ux, uy, uz); else bin_fwd2(eq.v, ux, uy);
          eq.v[0] = rho;  // sum f_eq = rho, first-order central moments vanish
          eq.v[E(1, 0, 0)] = real(0);
          eq.v[E(0, 1, 0)] = real(0);
          if constexpr (S::D == 3) eq.v[E(0, 0, 1)] = real(0);
          if constexpr (S::D == 3) central_to_cumulant3<S>(eq.v, inv); else central_to_cumulant2(eq.v, inv);
          if constexpr (S::D == 3) relax_basis3<S, RSR>(c, eq, r); else relax_basis2<RSR>(c, eq, r);
        } else {
          real cs2 = real(1.0 / 3.0);
          if constexpr (SPACE == SPACE_SWE_K) cs2 = real(0.5) * swe_g * rho;
          EqCumulant<real> eq{rho * cs2};
          if constexpr (S::D == 3) relax_basis3<S, RSR>(c, eq, r); else relax_basis2<RSR>(c, eq, r);
        }
        if constexpr (S::D == 3) cumulant_to_central3<S>(c, inv); else cumulant_to_central2(c, inv);
        if constexpr (FORCED) {  // C*_100 = C_100 + F_x: the post-collision mean is (j + F)/rho
          ux = fma(fr.F[0], inv, ux);
          uy = fma(fr.F[1], inv, uy);
          uz = fma(fr.F[2], inv, uz);
        }
      }
      // ---- central -> raw
      if constexpr (S::D == 3) bin_bwd3(c, ux, uy, uz); else bin_bwd2(c, ux, uy);
    }
    if constexpr (REG == REG_ZC_ABS) {
      if constexpr (SWEZ) add_background_swe<SPACE>(c, real(-1), swe_g);
      else add_background<NC>(c, real(-1));
    }
    // conserved raw moments pass through unchanged, the momentum gains the
    // force: m*_100 = rho u_x + F_x/2 = j_x + F_x
    c[0] = m000;
    c[E(1, 0, 0)] = FORCED ? jx + fr.F[0] : jx;
    c[E(0, 1, 0)] = FORCED ? jy + fr.F[1] : jy;
    if constexpr (S::D == 3) c[E(0, 0, 1)] = FORCED ? jz + fr.F[2] : jz;
    // ---- backward raw transform
    if constexpr (S::Q == 27) bwd_raw3_full(c);
    else if constexpr (S::Q == 19) bwd_raw3_d3q19(c);
    else bwd_raw2(c);
    sfor<S::Q>([&](auto i) { f[i] = c[S::pos(i)]; });
  }
}

// Equilibrium populations of the method at (rho, u) in stored form: f_eq = T^{-1}(q_eq).
// RAW / POPULATION: M^{-1} m_eq (truncated Maxwellian); CENTRAL / CUMULANT: the Gaussian
// central moments, i.e. raw moments rho prod_a (1, u_a, cs2 + u_a^2); SWE: Zhou f_eq.
template <class S, int SPACE, int REG, class real, bool DISC>
__device__ __forceinline__ void equilibrium(real (&f)[S::Q], real rho, real ux, real uy, real uz, real swe_g) {
  constexpr int NC = S::NC;
  constexpr bool zc = (REG != REG_ABS);
  if constexpr (DISC && SPACE != SPACE_SWE && SPACE != SPACE_SWE_K) {  // reading R29
    real fe[NC];
    discrete_feq_cube<S>(fe, rho, ux, uy, uz, zc);
    sfor<S::Q>([&](auto i) { f[i] = fe[S::pos(i)]; });
    return;
  }
  if constexpr (SPACE == SPACE_SWE) {
    const real uu = ux * ux + uy * uy, gh = swe_g * rho;
    sfor<9>([&](auto i) {
      constexpr int vx = S::vx(i), vy = S::vy(i);
      constexpr int l1 = (vx != 0) + (vy != 0);
      if constexpr (l1 == 0) {
        f[i] = rho * (real(1) - real(5.0 / 6.0) * gh - real(2.0 / 3.0) * uu);
      } else {
        const real xu = real(vx) * ux + real(vy) * uy;
        const real lam = (l1 == 1) ? real(1) : real(0.25);
        f[i] = lam * rho * (real(1.0 / 6.0) * gh + real(1.0 / 3.0) * xu + real(0.5) * xu * xu - real(1.0 / 6.0) * uu);
      }
      if constexpr (zc) {  // minus the rest state f_eq(1, 0) (reading R33)
        if constexpr (l1 == 0) f[i] -= real(1) - real(5.0 / 6.0) * swe_g;
        else f[i] -= ((l1 == 1) ? real(1) : real(0.25)) * real(1.0 / 6.0) * swe_g;
      }
    });
    return;
  } else {
    const real drho = rho - real(1);
    real c[NC];
    if constexpr (SPACE == SPACE_POPULATION || SPACE == SPACE_RAW) {
      RawU<real> U{ux, uy, uz, ux * ux, uy * uy, uz * uz};
      sfor<NC>([&](auto e) {
        constexpr double h = hprod(e);
        if constexpr (RawU<real>::template zero<e>() && e != 0) c[e] = real(0);
        else if constexpr (e == 0) c[e] = zc ? drho : rho;
        else if constexpr (h != 0.0) c[e] = zc ? fma(real(h), drho, rho * U.template get<e>())
                                              : rho * (real(h) + U.template get<e>());
        else c[e] = rho * U.template get<e>();
      });
    } else {
      // untruncated Gaussian raw moments rho prod (1, u, cs2 + u^2); zc: minus hprod
      // (cs2 = 1/3, or g h / 2 for the cumulant shallow-water method)
      real cs2 = real(1.0 / 3.0);
      if constexpr (SPACE == SPACE_SWE_K) cs2 = real(0.5) * swe_g * rho;
      sfor<NC>([&](auto e) {
        constexpr int ax = ex_of(e), ay = ey_of(e), az = ez_of(e);
        auto g = [&](auto a, real u) -> real {
          if constexpr (decltype(a)::value == 0) return real(1);
          else if constexpr (decltype(a)::value == 1) return u;
          else return cs2 + u * u;
        };
        const real p = g(std::integral_constant<int, ax>{}, ux) * g(std::integral_constant<int, ay>{}, uy) *
                       g(std::integral_constant<int, az>{}, uz);
        constexpr double h = hprod(e);
        if constexpr (e == 0) c[e] = zc ? drho : rho;
        else if constexpr (SPACE == SPACE_SWE_K && zc) {  // minus the rest state's moments (R33)
          if constexpr (e == E(2, 0, 0) || e == E(0, 2, 0)) c[e] = fma(rho, p, real(-0.5) * swe_g);
          else if constexpr (e == E(2, 2, 0)) c[e] = fma(rho, p, -swe_bg_m22<SPACE_SWE_K>(swe_g));
          else c[e] = rho * p;
        } else if constexpr (h != 0.0) c[e] = zc ? fma(rho, p, real(-h)) : rho * p;
        else c[e] = rho * p;
      });
    }
    if constexpr (S::Q == 27) bwd_raw3_full(c);
    else if constexpr (S::Q == 19) bwd_raw3_d3q19(c);
    else bwd_raw2(c);
    sfor<S::Q>([&](auto i) { f[i] = c[S::pos(i)]; });
  }
}

}  // namespace lbm
