/*
 * lbm_oracle.cpp — plain, slow, obviously-correct CPU oracle for the MRT
 * lattice Boltzmann stream–collide update of arXiv 2211.02435 (lbmpy 1.1,
 * Hennig, Holzer, Rüde).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_2211_02435_b200/) never links, imports or calls it,
 * and this file shares no code, header, table or helper with the CUDA path.
 *
 * What it computes (citations are PAPER.md line numbers + equation labels):
 *   * stencils D2Q9 / D3Q19 / D3Q27 with xi_0 = 0; the
 *     population ORDER is the interface convention documented in
 *     include/lbm.h (the paper leaves it free);
 *   * collision spaces by their plain definitions:
 *       population (SRT, T = I),
 *       raw moments   m_p = sum_i f_i p(xi_i)          eq:DiscreteRawMomentsDef
 *       central moms  k_p = sum_i f_i p(xi_i - u)      (second eq:DiscreteRawMomentsDef) PAPER.md:399-407
 *       cumulants     C = rho * derivatives of log M    eq:CumulantGeneratingFunction PAPER.md:417-426,
 *                     evaluated through C = Xi.u + log K (eq:CumulantAndCentralMomentGenFuncs,
 *                     PAPER.md:680-685) as a truncated power series in R[X,Y,Z]/(X^3,Y^3,Z^3);
 *     as DENSE matrices M (q x q) and K(u) (q x q, rebuilt per cell) and a
 *     dense solve for the inverse transform — no Chimera, no closed forms;
 *   * the three collision regimes
 *       absolute storage           eq:MrtUpdateGeneral
 *       zero-centered + delta eq   eq:MrtUpdateGeneralDeviationOnly
 *       zero-centered + abs eq     eq:MrtUpdateAbsoluteFromZeroCentered
 *   * equilibria: the discrete second-order polynomial f_eq (q_eq = T(f_eq), PAPER.md:485-487;
 *     DESIGN.md reading R29) or the continuous Maxwellian (eq:ContMaxwellian)
 *     represented in the method's own collision space and truncated at second
 *     order in u (reading R4); background
 *     f0 = M^{-1} m0; the shallow-water discrete
 *     equilibrium of Zhou, eq:DiscreteShallowWaterEquilibrium
 *     with the -u.u/6 correction (reading R5), used as
 *     q_eq = T(f_eq);
 *   * streaming: two-grid pull, f_i(x, t+1) = f*_i(x - xi_i, t)
 *     (eq:LbStreaming PAPER.md:223-224, pull pattern PAPER.md:857-859),
 *     periodic faces, or half-way bounce-back on no-slip faces (not in the
 *     paper; reading R18);
 *   * body force (source q^F of eq:MrtUpdateGeneral):
 *     Guo's F^G (reading R23) or He's F^He = f_eq (xi - u).F / (rho c_s^2) (reading R27)
 *     with q^F = (I - S/2) T(F) for the linear spaces,
 *     F on the first-order cumulants only for the cumulant space (reading R26).
 *
 * Templated on the real type: the long double (x87 80-bit) instantiation is
 * the parity reference, the double instantiation is the timed CPU baseline.
 * Compiled with -O2 -ffp-contract=off (no FMA contraction, no fast-math).
 */
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>
#include <algorithm>
#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

enum { ST_D2Q9 = 0, ST_D3Q19 = 1, ST_D3Q27 = 2 };
enum { SP_POPULATION = 0, SP_RAW = 1, SP_CENTRAL = 2, SP_CUMULANT = 3, SP_RAW_WO = 4 };
enum { EQ_ABSOLUTE = 0, EQ_DELTA = 1, EQ_SWE = 2, EQ_DISCRETE = 3, EQ_DISCRETE_DELTA = 4, EQ_ABSOLUTE_F0 = 5 };
enum { BC_PERIODIC = 0, BC_NOSLIP = 1 };

struct Term {
  int c;       // integer coefficient
  int e[3];    // exponents of x, y, z
};
using Poly = std::vector<Term>;

/* ------------------------------------------------------------------------ */
/* Stencil: velocities in the documented interface order (include/lbm.h).    */
/* The slab (decomposition) axis is the last lattice axis: z in 3D, y in 2D. */
/* Rule: rest first; then the in-plane (slab component 0) velocities; then   */
/* slab component +1; then slab component -1 as the negations of the +1      */
/* group in the same order.  Inside a group the in-plane part follows the    */
/* sequence (0,0), (1,0), (-1,0), (0,1), (0,-1), (1,1), (-1,-1), (1,-1),     */
/* (-1,1) (for 2D only its x-part: 0, 1, -1).                                */
/* ------------------------------------------------------------------------ */
static std::vector<std::array<int, 3>> make_stencil(int stencil) {
  std::vector<std::array<int, 3>> v;
  if (stencil == ST_D2Q9) {
    const int line[3] = {0, 1, -1};
    v.push_back({0, 0, 0});
    for (int k = 1; k < 3; ++k) v.push_back({line[k], 0, 0});
    for (int k = 0; k < 3; ++k) v.push_back({line[k], 1, 0});
    for (int k = 0; k < 3; ++k) v.push_back({-line[k], -1, 0});
    return v;
  }
  const int plane[9][2] = {{0, 0}, {1, 0}, {-1, 0}, {0, 1}, {0, -1},
                           {1, 1}, {-1, -1}, {1, -1}, {-1, 1}};
  auto in_stencil = [&](int a, int b, int c) {
    if (stencil == ST_D3Q27) return true;
    return std::abs(a) + std::abs(b) + std::abs(c) <= 2;  // D3Q19
  };
  v.push_back({0, 0, 0});
  for (int k = 1; k < 9; ++k)
    if (in_stencil(plane[k][0], plane[k][1], 0)) v.push_back({plane[k][0], plane[k][1], 0});
  std::vector<std::array<int, 3>> up;
  for (int k = 0; k < 9; ++k)
    if (in_stencil(plane[k][0], plane[k][1], 1)) up.push_back({plane[k][0], plane[k][1], 1});
  for (auto &x : up) v.push_back(x);
  for (auto &x : up) v.push_back({-x[0], -x[1], -x[2]});
  return v;
}

static int dims_of(int stencil) { return stencil == ST_D2Q9 ? 2 : 3; }

/* ------------------------------------------------------------------------ */
/* Collision-space bases (reading R2; PAPER.md:331-336 notation).   */
/* ------------------------------------------------------------------------ */
static Poly P(std::initializer_list<Term> t) { return Poly(t); }
static Term T(int c, int a, int b, int g) { return Term{c, {a, b, g}}; }

static std::vector<Poly> make_basis(int stencil) {
  std::vector<Poly> B;
  if (stencil == ST_D2Q9) {
    // de Rosis basis: 1; x, y; xy, x^2-y^2; x^2+y^2; x^2 y, x y^2; x^2 y^2
    B.push_back(P({T(1, 0, 0, 0)}));
    B.push_back(P({T(1, 1, 0, 0)}));
    B.push_back(P({T(1, 0, 1, 0)}));
    B.push_back(P({T(1, 1, 1, 0)}));
    B.push_back(P({T(1, 2, 0, 0), T(-1, 0, 2, 0)}));
    B.push_back(P({T(1, 2, 0, 0), T(1, 0, 2, 0)}));
    B.push_back(P({T(1, 2, 1, 0)}));
    B.push_back(P({T(1, 1, 2, 0)}));
    B.push_back(P({T(1, 2, 2, 0)}));
    return B;
  }
  // D3Q27 (27 polynomials); D3Q19 = the same list without xyz (index 16) and
  // without the polynomials 20..26 (orders 5/6 and x^2yz-type).
  B.push_back(P({T(1, 0, 0, 0)}));                                   // 0  1
  B.push_back(P({T(1, 1, 0, 0)}));                                   // 1  x
  B.push_back(P({T(1, 0, 1, 0)}));                                   // 2  y
  B.push_back(P({T(1, 0, 0, 1)}));                                   // 3  z
  B.push_back(P({T(1, 1, 1, 0)}));                                   // 4  xy
  B.push_back(P({T(1, 1, 0, 1)}));                                   // 5  xz
  B.push_back(P({T(1, 0, 1, 1)}));                                   // 6  yz
  B.push_back(P({T(1, 2, 0, 0), T(-1, 0, 2, 0)}));                   // 7  x^2 - y^2
  B.push_back(P({T(1, 2, 0, 0), T(-1, 0, 0, 2)}));                   // 8  x^2 - z^2
  B.push_back(P({T(1, 2, 0, 0), T(1, 0, 2, 0), T(1, 0, 0, 2)}));     // 9  x^2 + y^2 + z^2
  B.push_back(P({T(1, 1, 2, 0), T(1, 1, 0, 2)}));                    // 10 xy^2 + xz^2
  B.push_back(P({T(1, 2, 1, 0), T(1, 0, 1, 2)}));                    // 11 x^2y + yz^2
  B.push_back(P({T(1, 2, 0, 1), T(1, 0, 2, 1)}));                    // 12 x^2z + y^2z
  B.push_back(P({T(1, 1, 2, 0), T(-1, 1, 0, 2)}));                   // 13 xy^2 - xz^2
  B.push_back(P({T(1, 2, 1, 0), T(-1, 0, 1, 2)}));                   // 14 x^2y - yz^2
  B.push_back(P({T(1, 2, 0, 1), T(-1, 0, 2, 1)}));                   // 15 x^2z - y^2z
  if (stencil == ST_D3Q27) B.push_back(P({T(1, 1, 1, 1)}));         // 16 xyz
  B.push_back(P({T(1, 2, 2, 0), T(-2, 2, 0, 2), T(1, 0, 2, 2)}));    // 17 x^2y^2 - 2x^2z^2 + y^2z^2
  B.push_back(P({T(1, 2, 2, 0), T(1, 2, 0, 2), T(-2, 0, 2, 2)}));    // 18 x^2y^2 + x^2z^2 - 2y^2z^2
  B.push_back(P({T(1, 2, 2, 0), T(1, 2, 0, 2), T(1, 0, 2, 2)}));     // 19 x^2y^2 + x^2z^2 + y^2z^2
  if (stencil == ST_D3Q27) {
    B.push_back(P({T(1, 2, 1, 1)}));                                 // 20 x^2yz
    B.push_back(P({T(1, 1, 2, 1)}));                                 // 21 xy^2z
    B.push_back(P({T(1, 1, 1, 2)}));                                 // 22 xyz^2
    B.push_back(P({T(1, 1, 2, 2)}));                                 // 23 xy^2z^2
    B.push_back(P({T(1, 2, 1, 2)}));                                 // 24 x^2yz^2
    B.push_back(P({T(1, 2, 2, 1)}));                                 // 25 x^2y^2z
    B.push_back(P({T(1, 2, 2, 2)}));                                 // 26 x^2y^2z^2
  }
  return B;
}

static int order_of(const Poly &p) {
  int o = 0;
  for (auto &t : p) o = std::max(o, t.e[0] + t.e[1] + t.e[2]);
  return o;
}

/* integer power, small exponents */
template <class R> static R ipow(R x, int e) {
  R r = 1;
  for (int k = 0; k < e; ++k) r *= x;
  return r;
}

template <class R> static R eval_poly(const Poly &p, R x, R y, R z) {
  R s = 0;
  for (auto &t : p) s += R(t.c) * ipow(x, t.e[0]) * ipow(y, t.e[1]) * ipow(z, t.e[2]);
  return s;
}

/* ------------------------------------------------------------------------ */
/* Dense linear algebra: Gauss–Jordan inverse and LU solve, partial pivoting */
/* ------------------------------------------------------------------------ */
template <class R> static bool invert(int n, const R *A, R *Ainv) {
  std::vector<R> a(A, A + n * n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) Ainv[i * n + j] = (i == j) ? R(1) : R(0);
  for (int c = 0; c < n; ++c) {
    int piv = c;
    for (int r = c + 1; r < n; ++r)
      if (std::fabs(a[r * n + c]) > std::fabs(a[piv * n + c])) piv = r;
    if (a[piv * n + c] == R(0)) return false;
    if (piv != c)
      for (int j = 0; j < n; ++j) {
        std::swap(a[c * n + j], a[piv * n + j]);
        std::swap(Ainv[c * n + j], Ainv[piv * n + j]);
      }
    R d = a[c * n + c];
    for (int j = 0; j < n; ++j) {
      a[c * n + j] /= d;
      Ainv[c * n + j] /= d;
    }
    for (int r = 0; r < n; ++r) {
      if (r == c) continue;
      R fct = a[r * n + c];
      if (fct == R(0)) continue;
      for (int j = 0; j < n; ++j) {
        a[r * n + j] -= fct * a[c * n + j];
        Ainv[r * n + j] -= fct * Ainv[c * n + j];
      }
    }
  }
  return true;
}

/* solve A x = b in place (A destroyed), LU with partial pivoting */
template <class R> static bool solve(int n, R *A, R *b) {
  for (int c = 0; c < n; ++c) {
    int piv = c;
    for (int r = c + 1; r < n; ++r)
      if (std::fabs(A[r * n + c]) > std::fabs(A[piv * n + c])) piv = r;
    if (A[piv * n + c] == R(0)) return false;
    if (piv != c) {
      for (int j = 0; j < n; ++j) std::swap(A[c * n + j], A[piv * n + j]);
      std::swap(b[c], b[piv]);
    }
    for (int r = c + 1; r < n; ++r) {
      R fct = A[r * n + c] / A[c * n + c];
      if (fct == R(0)) continue;
      for (int j = c; j < n; ++j) A[r * n + j] -= fct * A[c * n + j];
      b[r] -= fct * b[c];
    }
  }
  for (int r = n - 1; r >= 0; --r) {
    R s = b[r];
    for (int j = r + 1; j < n; ++j) s -= A[r * n + j] * b[j];
    b[r] = s / A[r * n + r];
  }
  return true;
}

template <class R> static void matvec(int n, const R *A, const R *x, R *y) {
  for (int i = 0; i < n; ++i) {
    R s = 0;
    for (int j = 0; j < n; ++j) s += A[i * n + j] * x[j];
    y[i] = s;
  }
}

/* ------------------------------------------------------------------------ */
/* Truncated power series in R[X,Y,Z]/(X^3, Y^3, Z^3): 27 coefficients,     */
/* index e = ex + 3 ey + 9 ez.  Used for the cumulant generating function.  */
/* ------------------------------------------------------------------------ */
template <class R> struct Series {
  R c[27];
};
template <class R> static Series<R> ser_mul(const Series<R> &a, const Series<R> &b) {
  Series<R> r;
  for (int k = 0; k < 27; ++k) r.c[k] = 0;
  for (int i = 0; i < 27; ++i) {
    if (a.c[i] == R(0)) continue;
    int ix = i % 3, iy = (i / 3) % 3, iz = i / 9;
    for (int j = 0; j < 27; ++j) {
      int jx = j % 3, jy = (j / 3) % 3, jz = j / 9;
      if (ix + jx > 2 || iy + jy > 2 || iz + jz > 2) continue;  // X^3 = Y^3 = Z^3 = 0
      r.c[(ix + jx) + 3 * (iy + jy) + 9 * (iz + jz)] += a.c[i] * b.c[j];
    }
  }
  return r;
}
/* log(1 + S), S without constant term: sum_{n=1}^{6} (-1)^{n+1} S^n / n (S^7 = 0) */
template <class R> static Series<R> ser_log1p(const Series<R> &S) {
  Series<R> acc, pw = S;
  for (int k = 0; k < 27; ++k) acc.c[k] = 0;
  for (int n = 1; n <= 6; ++n) {
    R sgn = (n % 2 == 1) ? R(1) : R(-1);
    for (int k = 0; k < 27; ++k) acc.c[k] += sgn * pw.c[k] / R(n);
    pw = ser_mul(pw, S);
  }
  return acc;
}
/* exp(L), L without constant term: sum_{n=0}^{6} L^n / n! */
template <class R> static Series<R> ser_exp(const Series<R> &L) {
  Series<R> acc, pw;
  for (int k = 0; k < 27; ++k) {
    acc.c[k] = 0;
    pw.c[k] = 0;
  }
  pw.c[0] = 1;
  R fact = 1;
  for (int n = 0; n <= 6; ++n) {
    if (n > 0) {
      pw = ser_mul(pw, L);
      fact *= R(n);
    }
    for (int k = 0; k < 27; ++k) acc.c[k] += pw.c[k] / fact;
  }
  return acc;
}
static int efact(int e) { return e == 2 ? 2 : 1; }  // e! for e in {0,1,2}

/* ------------------------------------------------------------------------ */
/* Method                                                                    */
/* ------------------------------------------------------------------------ */
template <class R> struct Method {
  int stencil = 0, d = 0, q = 0, space = 0, eq = 0, zc = 0;
  R g = 0;  // SWE lattice gravity
  R F[3] = {0, 0, 0};  // uniform body force density (lattice units)
  bool forced = false;
  int force_model = 0;  // 0: Guo (reading R23), 1: He (reading R27)
  std::vector<std::array<int, 3>> xi;
  std::vector<int> opp;
  std::vector<Poly> basis;
  std::vector<R> omega;
  std::vector<R> M, Minv;  // M[p][i] = p(xi_i)
  std::vector<R> w;        // background f0 = M^{-1} m0
  // monomials: the q exponent triples (one per basis polynomial, in the order
  // of first appearance) and R_mono: basis polys in terms of those monomials
  std::vector<std::array<int, 3>> mono;
  std::vector<R> Rmono, Rmono_inv;
  // WO-MRT (SP_RAW_WO, reading R31): the graded-lexicographic monomials wo_mono and the
  // weighted Gram-Schmidt coefficients G[k][j] (polynomial k = sum_j G[k][j] wo_mono[j])
  std::vector<std::array<int, 3>> wo_mono;
  std::vector<R> G;
  bool ok = false;
};

static const long double CS2 = 1.0L / 3.0L;  // c_s^2 = 1/3 (lattice units)

/* Maxwellian raw moment of monomial e, truncated at total degree 2 in u     */
/* (PAPER.md:786-787): product over axes of g_0 = 1, g_1 = u, g_2 = cs2 + u^2 */
/* expanded and cut.  'rho' multiplies everything.                           */
template <class R> static R maxwell_raw_trunc(const int e[3], R rho, const R u[3]) {
  // per-axis polynomials in u_a, coefficients by degree 0..2
  R pa[3][3];
  for (int a = 0; a < 3; ++a) {
    pa[a][0] = pa[a][1] = pa[a][2] = 0;
    if (e[a] == 0) pa[a][0] = 1;
    if (e[a] == 1) pa[a][1] = 1;
    if (e[a] == 2) {
      pa[a][0] = R(CS2);
      pa[a][2] = 1;
    }
  }
  R s = 0;
  for (int i = 0; i <= 2; ++i)
    for (int j = 0; j <= 2; ++j)
      for (int k = 0; k <= 2; ++k) {
        if (i + j + k > 2) continue;
        R c = pa[0][i] * pa[1][j] * pa[2][k];
        if (c == R(0)) continue;
        s += c * ipow(u[0], i) * ipow(u[1], j) * ipow(u[2], k);
      }
  return rho * s;
}
/* Maxwellian central moment of monomial e (u-independent Gaussian moments):  */
/* product of 1, 0, cs2 for exponents 0, 1, 2.                                */
template <class R> static R maxwell_central(const int e[3], R rho) {
  R s = rho;
  for (int a = 0; a < 3; ++a) {
    if (e[a] == 1) return R(0);
    if (e[a] == 2) s *= R(CS2);
  }
  return s;
}

template <class R> static bool equilibrium_cell(const Method<R> &m, R rho, const R u[3], R *f);

/* Weighted-orthogonal raw-moment basis (WO-MRT; PAPER.md:789-790 names it, SPEC.md:187-195   */
/* describes it; reading R31).  Definition, written out: the stencil's monomials x^a y^b z^c  */
/* (the q monomials of the raw basis of reading R2) in graded-lexicographic order (total      */
/* degree, then a, b, c descending), orthogonalised one after the other by classical         */
/* Gram-Schmidt under <p, r> = sum_i w_i p(xi_i) r(xi_i) (w = the lattice weights f0):        */
/*   p_k = x^(e_k) - sum_{j<k} <x^(e_k), p_j> / <p_j, p_j> p_j.                               */
/* M[k][i] = p_k(xi_i); one rate per p_k in that order.                                        */
template <class R> static bool build_wo_basis(Method<R> &m) {
  const int q = m.q;
  m.wo_mono.clear();
  for (int deg = 0; deg <= 6; ++deg)
    for (int a = 2; a >= 0; --a)
      for (int b = 2; b >= 0; --b)
        for (int c = 2; c >= 0; --c) {
          if (a + b + c != deg) continue;
          bool in_raw = false;  // a monomial of the raw basis (reading R2)
          for (auto &p : m.basis)
            for (auto &t : p)
              if (t.e[0] == a && t.e[1] == b && t.e[2] == c) in_raw = true;
          if (in_raw) m.wo_mono.push_back({a, b, c});
        }
  if ((int)m.wo_mono.size() != q) return false;
  std::vector<R> V(q * q);  // V[k][i] = x^(e_k)(xi_i)
  for (int k = 0; k < q; ++k)
    for (int i = 0; i < q; ++i)
      V[k * q + i] = ipow(R(m.xi[i][0]), m.wo_mono[k][0]) * ipow(R(m.xi[i][1]), m.wo_mono[k][1]) *
                     ipow(R(m.xi[i][2]), m.wo_mono[k][2]);
  m.G.assign(q * q, R(0));
  std::vector<R> P(q * q, R(0));  // P[k][i] = p_k(xi_i)
  for (int k = 0; k < q; ++k) {
    m.G[k * q + k] = R(1);
    for (int i = 0; i < q; ++i) P[k * q + i] = V[k * q + i];
    for (int j = 0; j < k; ++j) {
      R num = 0, den = 0;
      for (int i = 0; i < q; ++i) {
        num += m.w[i] * V[k * q + i] * P[j * q + i];
        den += m.w[i] * P[j * q + i] * P[j * q + i];
      }
      const R cf = num / den;
      for (int l = 0; l < q; ++l) m.G[k * q + l] -= cf * m.G[j * q + l];
      for (int i = 0; i < q; ++i) P[k * q + i] -= cf * P[j * q + i];
    }
  }
  for (int k = 0; k < q * q; ++k) m.M[k] = P[k];
  return invert(q, m.M.data(), m.Minv.data());
}

template <class R>
static bool build_method(Method<R> &m, int stencil, int space, int eq, int zc, const double *rates,
                         int nrates, double g) {
  m.stencil = stencil;
  m.d = dims_of(stencil);
  m.space = space;
  // LBM_EQ_ABSOLUTE_F0 (reading R30): eq:MrtUpdateAbsoluteFromZeroCentered
  // with f0 added to the populations before the transform — which is how this oracle evaluates
  // the zero-centered absolute regime anyway (collide_cell: fabs = df + f0)
  if (eq == EQ_ABSOLUTE_F0) {
    if (!zc) return false;
    eq = EQ_ABSOLUTE;
  }
  if (space == SP_RAW_WO && (eq == EQ_SWE || eq == EQ_DISCRETE || eq == EQ_DISCRETE_DELTA)) return false;
  m.eq = eq;
  m.zc = zc;
  m.g = R(g);
  m.xi = make_stencil(stencil);
  m.q = (int)m.xi.size();
  int q = m.q;
  m.opp.resize(q);
  for (int i = 0; i < q; ++i)
    for (int j = 0; j < q; ++j)
      if (m.xi[j][0] == -m.xi[i][0] && m.xi[j][1] == -m.xi[i][1] && m.xi[j][2] == -m.xi[i][2])
        m.opp[i] = j;
  m.basis = make_basis(stencil);
  if ((int)m.basis.size() != q) return false;
  m.omega.assign(q, R(0));
  if (space == SP_POPULATION) {
    if (nrates < 1) return false;
    for (int i = 0; i < q; ++i) m.omega[i] = R(rates[0]);
  } else {
    if (nrates != q) return false;
    for (int i = 0; i < q; ++i) m.omega[i] = R(rates[i]);
  }
  m.M.assign(q * q, 0);
  m.Minv.assign(q * q, 0);
  for (int p = 0; p < q; ++p)
    for (int i = 0; i < q; ++i)
      m.M[p * q + i] = eval_poly<R>(m.basis[p], R(m.xi[i][0]), R(m.xi[i][1]), R(m.xi[i][2]));
  if (!invert(q, m.M.data(), m.Minv.data())) return false;
  // background: m0 = Maxwellian moments at rho0 = 1, u = 0
  std::vector<R> m0(q, 0);
  R zero3[3] = {0, 0, 0};
  for (int p = 0; p < q; ++p) {
    R s = 0;
    for (auto &t : m.basis[p]) s += R(t.c) * maxwell_raw_trunc<R>(t.e, R(1), zero3);
    m0[p] = s;
  }
  m.w.assign(q, 0);
  matvec(q, m.Minv.data(), m0.data(), m.w.data());
  if (space == SP_RAW_WO && !build_wo_basis(m)) return false;
  // monomial set and R_mono
  m.mono.clear();
  for (auto &p : m.basis)
    for (auto &t : p) {
      std::array<int, 3> e = {t.e[0], t.e[1], t.e[2]};
      if (std::find(m.mono.begin(), m.mono.end(), e) == m.mono.end()) m.mono.push_back(e);
    }
  if ((int)m.mono.size() != q) return false;
  m.Rmono.assign(q * q, 0);
  m.Rmono_inv.assign(q * q, 0);
  for (int p = 0; p < q; ++p)
    for (auto &t : m.basis[p]) {
      std::array<int, 3> e = {t.e[0], t.e[1], t.e[2]};
      int k = (int)(std::find(m.mono.begin(), m.mono.end(), e) - m.mono.begin());
      m.Rmono[p * q + k] += R(t.c);
    }
  if (!invert(q, m.Rmono.data(), m.Rmono_inv.data())) return false;
  // zero-centered shallow water (reading R33): the
  // background is the method's own rest state f0 = f_eq(h0 = 1, u = 0), h = h0 + sum df:
  // Zhou's discrete equilibrium (eq:DiscreteShallowWaterEquilibrium) for
  // central moments, the Maxwellian at c_s^2 = g h0 / 2 for cumulants
  if (eq == EQ_SWE && zc) {
    const R u0[3] = {0, 0, 0};
    m.zc = 0;
    const bool ok = equilibrium_cell(m, R(1), u0, m.w.data());
    m.zc = zc;
    if (!ok) return false;
  }
  m.ok = true;
  return true;
}

/* macroscopic quantities (eq:DensityAndVelocity PAPER.md:247-251;            */
/* eq:DensityAndVelocityFromDeviation PAPER.md:254-259, rho0 = 1)             */
/* With a body force F (reading R23, Guo et al. 2002) the velocity is shifted by half the  */
/* force: pre-collision u = (j + F/2) / rho (half = +1), post-collision u = (j - F/2) / rho */
/* (half = -1, the canonical post-collision state of a step).                             */
template <class R>
static void macroscopic(const Method<R> &m, const R *f, R &rho, R u[3], int half = 1) {
  R s = 0, j[3] = {0, 0, 0};
  for (int i = 0; i < m.q; ++i) {
    s += f[i];
    for (int a = 0; a < 3; ++a) j[a] += f[i] * R(m.xi[i][a]);
  }
  rho = m.zc ? R(1) + s : s;
  for (int a = 0; a < 3; ++a) u[a] = (j[a] + R(half) * m.F[a] / R(2)) / rho;
}

/* Guo's discrete force term F^G_i = w_i [3 xi.F + 9 (xi.u)(xi.F) - 3 u.F] (c_s^2 = 1/3);  */
/* the source of eq:MrtUpdateGeneral is q^F = (I - S/2) T(F^G) (reading R23).             */
template <class R> static void guo_force(const Method<R> &m, const R u[3], R *FG) {
  R uF = u[0] * m.F[0] + u[1] * m.F[1] + u[2] * m.F[2];
  for (int i = 0; i < m.q; ++i) {
    R xF = 0, xu = 0;
    for (int a = 0; a < 3; ++a) {
      xF += R(m.xi[i][a]) * m.F[a];
      xu += R(m.xi[i][a]) * u[a];
    }
    FG[i] = m.w[i] * (R(3) * xF + R(9) * xu * xF - R(3) * uF);
  }
}

template <class R> static bool equilibrium_cell(const Method<R> &m, R rho, const R u[3], R *f);

/* He's force term F^He_i = f_eq_i(rho, u) (xi_i - u).F / (rho c_s^2) (He, Shan, Doolen 1998,  */
/* cited at PAPER.md:214, 539; reading R27) with f_eq the method's own equilibrium            */
/* (absolute populations); the source is q^F = (I - S/2) T(F^He) like Guo's.                   */
template <class R> static bool he_force(const Method<R> &m, R rho, const R u[3], R *FG) {
  R feq[27];
  if (!equilibrium_cell(m, rho, u, feq)) return false;
  for (int i = 0; i < m.q; ++i) {
    R cF = 0;
    for (int a = 0; a < 3; ++a) cF += (R(m.xi[i][a]) - u[a]) * m.F[a];
    R fa = m.zc ? feq[i] + m.w[i] : feq[i];
    FG[i] = fa * cF / (rho * R(CS2));
  }
  return true;
}

/* Discrete second-order hydrodynamic equilibrium (reading R29): the equilibrium "specified as a */
/* discrete distribution f_eq", represented in collision space as q_eq = T(f_eq)              */
/* (the algebraic form "discrete or continuous"):             */
/*   f_eq_i = w_i rho [1 + 3 xi.u + 9/2 (xi.u)^2 - 3/2 u.u]   (c_s^2 = 1/3).                 */
template <class R> static void discrete_equilibrium(const Method<R> &m, R rho, const R u[3], R *feq) {
  const R uu = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
  for (int i = 0; i < m.q; ++i) {
    const R cu = R(m.xi[i][0]) * u[0] + R(m.xi[i][1]) * u[1] + R(m.xi[i][2]) * u[2];
    feq[i] = m.w[i] * rho * (R(1) + R(3) * cu + R(9) * cu * cu / R(2) - R(3) * uu / R(2));
  }
}

/* K(u)[p][i] = p(xi_i - u) */
template <class R> static void central_matrix(const Method<R> &m, const R u[3], R *K) {
  int q = m.q;
  for (int p = 0; p < q; ++p)
    for (int i = 0; i < q; ++i)
      K[p * q + i] = eval_poly<R>(m.basis[p], R(m.xi[i][0]) - u[0], R(m.xi[i][1]) - u[1],
                                  R(m.xi[i][2]) - u[2]);
}

/* Zhou shallow-water equilibrium, eq:DiscreteShallowWaterEquilibrium         */
/* with the u.u/6 correction of reading R5.              */
template <class R> static void swe_equilibrium(const Method<R> &m, R h, const R u[3], R *feq) {
  R uu = u[0] * u[0] + u[1] * u[1];
  R gh = m.g * h;
  for (int i = 0; i < m.q; ++i) {
    int l1 = std::abs(m.xi[i][0]) + std::abs(m.xi[i][1]);
    if (l1 == 0) {
      feq[i] = h * (R(1) - R(5) * gh / R(6) - R(2) * uu / R(3));
    } else {
      R lam = (l1 == 1) ? R(1) : R(1) / R(4);
      R xu = R(m.xi[i][0]) * u[0] + R(m.xi[i][1]) * u[1];
      feq[i] = lam * h * (gh / R(6) + xu / R(3) + xu * xu / R(2) - uu / R(6));
    }
  }
}

/* monomial index in the 27-coefficient series */
static int sidx(const int e[3]) { return e[0] + 3 * e[1] + 9 * e[2]; }

/* raw-moment equilibrium of the polynomial basis: m_eq_p(rho,u) (trunc.)    */
template <class R> static R raw_eq_poly(const Method<R> &m, int p, R rho, const R u[3]) {
  R s = 0;
  for (auto &t : m.basis[p]) s += R(t.c) * maxwell_raw_trunc<R>(t.e, rho, u);
  return s;
}
/* WO-MRT: the same truncated Maxwellian raw moments through the Gram-Schmidt coefficients */
template <class R> static R raw_eq(const Method<R> &m, int p, R rho, const R u[3]) {
  if (m.space != SP_RAW_WO) return raw_eq_poly(m, p, rho, u);
  R s = 0;
  for (int j = 0; j < m.q; ++j) s += m.G[p * m.q + j] * maxwell_raw_trunc<R>(m.wo_mono[j].data(), rho, u);
  return s;
}
template <class R> static R central_eq_poly(const Method<R> &m, int p, R rho) {
  R s = 0;
  for (auto &t : m.basis[p]) s += R(t.c) * maxwell_central<R>(t.e, rho);
  return s;
}

/* ------------------------------------------------------------------------ */
/* Cumulant transform by the generating function */
/* kappa (monomial central moments, all 27 exponent triples) -> C (rescaled  */
/* cumulants C = rho c).  First-order entries of log K^ are returned in      */
/* L1 so that conserved quantities can be passed through literally.          */
/* ------------------------------------------------------------------------ */
template <class R> static Series<R> cumulants_from_central(const R *kappa27, R rho) {
  Series<R> S;
  for (int k = 0; k < 27; ++k) {
    int ex = k % 3, ey = (k / 3) % 3, ez = k / 9;
    S.c[k] = kappa27[k] / rho / R(efact(ex) * efact(ey) * efact(ez));
  }
  S.c[0] = 0;  // K^ = K / rho = 1 + S
  Series<R> L = ser_log1p(S);
  // c_e = e! [log K^]_e ; C_e = rho c_e ; (c_000 = log rho is dropped: conserved)
  Series<R> C;
  for (int k = 0; k < 27; ++k) {
    int ex = k % 3, ey = (k / 3) % 3, ez = k / 9;
    C.c[k] = rho * L.c[k] * R(efact(ex) * efact(ey) * efact(ez));
  }
  C.c[0] = 0;
  return C;
}
template <class R> static void central_from_cumulants(const Series<R> &C, R rho, R *kappa27) {
  Series<R> L;
  for (int k = 0; k < 27; ++k) {
    int ex = k % 3, ey = (k / 3) % 3, ez = k / 9;
    L.c[k] = C.c[k] / rho / R(efact(ex) * efact(ey) * efact(ez));
  }
  L.c[0] = 0;
  Series<R> E = ser_exp(L);
  for (int k = 0; k < 27; ++k) {
    int ex = k % 3, ey = (k / 3) % 3, ez = k / 9;
    kappa27[k] = rho * E.c[k] * R(efact(ex) * efact(ey) * efact(ez));
  }
}

/* all 27 monomial central moments kappa_e = sum_i f_i prod_a (xi_ia - u_a)^e_a */
template <class R> static void central_monomials27(const Method<R> &m, const R *f, const R u[3], R *k27) {
  for (int k = 0; k < 27; ++k) {
    int e[3] = {k % 3, (k / 3) % 3, k / 9};
    R s = 0;
    for (int i = 0; i < m.q; ++i)
      s += f[i] * ipow(R(m.xi[i][0]) - u[0], e[0]) * ipow(R(m.xi[i][1]) - u[1], e[1]) *
           ipow(R(m.xi[i][2]) - u[2], e[2]);
    k27[k] = s;
  }
}

/* ------------------------------------------------------------------------ */
/* The collision of one cell.  fin/fout are in STORED form (delta f when the */
/* method uses zero-centered storage, f otherwise).                          */
/* ------------------------------------------------------------------------ */
template <class R> static bool collide_cell(const Method<R> &m, const R *fin, R *fout) {
  const int q = m.q;
  R rho, u[3];
  macroscopic(m, fin, rho, u);
  R fabs_[27], q0[27], qeq[27], qs[27], K[27 * 27];

  // deviation-only (eq:MrtUpdateGeneralDeviationOnly)
  const bool delta = (m.eq == EQ_DELTA || m.eq == EQ_DISCRETE_DELTA);
  const bool discrete = (m.eq == EQ_DISCRETE || m.eq == EQ_DISCRETE_DELTA);
  const R u0[3] = {0, 0, 0};                // background state rho0 = 1, u = 0
  // absolute populations for the absolute-equilibrium regimes
  for (int i = 0; i < q; ++i) fabs_[i] = (m.zc && !delta) ? fin[i] + m.w[i] : fin[i];
  // force term (source q^F of eq:MrtUpdateGeneral)
  R FG[27], qF[27];
  for (int i = 0; i < q; ++i) FG[i] = 0;
  if (m.forced) {
    if (m.eq == EQ_SWE) return false;             // not provided (reading R23)
    if (m.space != SP_CUMULANT) {  // cumulants: reading R26 below (the same for both models)
      if (m.force_model == 1) {
        if (!he_force(m, rho, u, FG)) return false;
      } else {
        guo_force(m, u, FG);
      }
    }
  }

  // discrete equilibrium (reading R29) in the form of the regime: f_eq, or f_eq - f0 (delta)
  R fd[27];
  if (discrete) {
    discrete_equilibrium(m, rho, u, fd);
    if (delta)
      for (int i = 0; i < q; ++i) fd[i] -= m.w[i];
  }

  if (m.space == SP_POPULATION) {
    // T = identity; f_eq = M^{-1} m_eq (reading R4), or the discrete f_eq (R29)
    R meq[27], feq[27];
    for (int p = 0; p < q; ++p) {
      meq[p] = raw_eq_poly(m, p, rho, u);
      if (delta) meq[p] -= raw_eq_poly(m, p, R(1), u0);
    }
    matvec(q, m.Minv.data(), meq, feq);
    if (discrete)
      for (int i = 0; i < q; ++i) feq[i] = fd[i];
    for (int i = 0; i < q; ++i)
      qs[i] = fabs_[i] + m.omega[0] * (feq[i] - fabs_[i]) + (R(1) - m.omega[0] / R(2)) * FG[i];
    for (int i = 0; i < q; ++i) fout[i] = (m.zc && !delta) ? qs[i] - m.w[i] : qs[i];
    return true;
  }

  if (m.space == SP_RAW || m.space == SP_RAW_WO) {
    if (m.space == SP_RAW_WO && m.forced) return false;  // not provided (lbm.h)
    matvec(q, m.M.data(), fabs_, q0);  // q = M f   (eq:DiscreteRawMomentsDef)
    matvec(q, m.M.data(), FG, qF);
    for (int p = 0; p < q; ++p) {
      qeq[p] = raw_eq(m, p, rho, u);
      if (delta) qeq[p] -= raw_eq(m, p, R(1), u0);  // dq_eq = q_eq - q0
    }
    if (discrete) matvec(q, m.M.data(), fd, qeq);  // q_eq = M f_eq
    for (int p = 0; p < q; ++p)
      qs[p] = q0[p] + m.omega[p] * (qeq[p] - q0[p]) + (R(1) - m.omega[p] / R(2)) * qF[p];
    matvec(q, m.Minv.data(), qs, fout);
    if (m.zc && !delta)
      for (int i = 0; i < q; ++i) fout[i] -= m.w[i];
    return true;
  }

  central_matrix(m, u, K);

  if (m.space == SP_CENTRAL) {
    matvec(q, K, fabs_, q0);  // kappa = K(u) f
    if (m.eq == EQ_SWE) {
      R feq[27];
      swe_equilibrium(m, rho, u, feq);
      matvec(q, K, feq, qeq);  // q_eq = T(f_eq)
    } else if (discrete) {
      matvec(q, K, fd, qeq);  // kappa_eq = K(u) f_eq (or K(u)(f_eq - f0))
    } else {
      for (int p = 0; p < q; ++p) qeq[p] = central_eq_poly(m, p, rho);
      if (delta) {  // dq_eq = q_eq - T(f0) with T = K(u)
        R kw[27];
        matvec(q, K, m.w.data(), kw);
        for (int p = 0; p < q; ++p) qeq[p] -= kw[p];
      }
    }
    matvec(q, K, FG, qF);  // kappa^F = K(u) F^G
    for (int p = 0; p < q; ++p)
      qs[p] = q0[p] + m.omega[p] * (qeq[p] - q0[p]) + (R(1) - m.omega[p] / R(2)) * qF[p];
    std::vector<R> A(K, K + q * q);
    if (!solve(q, A.data(), qs)) return false;
    for (int i = 0; i < q; ++i) fout[i] = (m.zc && !delta) ? qs[i] - m.w[i] : qs[i];
    return true;
  }

  // SP_CUMULANT (absolute equilibrium only)
  R k27[27];
  central_monomials27(m, fabs_, u, k27);
  Series<R> C = cumulants_from_central(k27, rho);
  // polynomial cumulants over the basis' monomials
  R Cmono[27], Cpoly[27], Cstar_poly[27], Cstar_mono[27];
  for (int k = 0; k < q; ++k) Cmono[k] = C.c[sidx(m.mono[k].data())];
  matvec(q, m.Rmono.data(), Cmono, Cpoly);
  // equilibrium cumulants of the Maxwellian: log M = log rho + Xi.u + cs2 |Xi|^2 / 2
  // (eq:ContMaxwellian, eq:CumulantGeneratingFunction) => C_200 = C_020 = C_002 = rho cs2,
  // all other cumulants of order >= 2 vanish.  Shallow water (Venturi):
  // the same Maxwellian with cs2 = g h / 2, h = the local water height.
  const R cs2 = (m.eq == EQ_SWE) ? m.g * rho / R(2) : R(CS2);
  // discrete equilibrium (R29): its own cumulants, C_eq = T(f_eq)
  Series<R> Cd;
  if (discrete) {
    R kd[27];
    central_monomials27(m, fd, u, kd);
    Cd = cumulants_from_central(kd, rho);
  }
  for (int p = 0; p < q; ++p) {
    int ord = order_of(m.basis[p]);
    if (ord < 2) {
      Cstar_poly[p] = 0;  // conserved: handled below by literal pass-through
      continue;
    }
    R ceq = 0;
    for (auto &t : m.basis[p]) {
      if (discrete) {
        ceq += R(t.c) * Cd.c[sidx(t.e)];
        continue;
      }
      bool diag2 = (t.e[0] + t.e[1] + t.e[2] == 2) && (t.e[0] == 2 || t.e[1] == 2 || t.e[2] == 2);
      if (diag2) ceq += R(t.c) * rho * cs2;
    }
    Cstar_poly[p] = Cpoly[p] + m.omega[p] * (ceq - Cpoly[p]);
  }
  matvec(q, m.Rmono_inv.data(), Cstar_poly, Cstar_mono);
  Series<R> Cs;
  for (int k = 0; k < 27; ++k) Cs.c[k] = 0;
  for (int k = 0; k < q; ++k) {
    const int *e = m.mono[k].data();
    if (e[0] + e[1] + e[2] >= 2) Cs.c[sidx(e)] = Cstar_mono[k];
  }
  // conserved first-order entries pass through unchanged.  With a body
  // force (reading R26) the source q^F is F on the first-order cumulants and zero on every
  // cumulant of order >= 2: with u = (j + F/2)/rho the first-order entry is kappa_100 = -F_x/2
  // and becomes kappa*_100 = kappa_100 + F_x, the momentum gains F.
  const int e100[3] = {1, 0, 0}, e010[3] = {0, 1, 0}, e001[3] = {0, 0, 1};
  Cs.c[sidx(e100)] = C.c[sidx(e100)] + m.F[0];
  Cs.c[sidx(e010)] = C.c[sidx(e010)] + m.F[1];
  Cs.c[sidx(e001)] = C.c[sidx(e001)] + m.F[2];
  R ks27[27];
  central_from_cumulants(Cs, rho, ks27);
  for (int p = 0; p < q; ++p) {
    R s = 0;
    for (auto &t : m.basis[p]) s += R(t.c) * ks27[sidx(t.e)];
    qs[p] = s;
  }
  std::vector<R> A(K, K + q * q);
  if (!solve(q, A.data(), qs)) return false;
  for (int i = 0; i < q; ++i) fout[i] = (m.zc) ? qs[i] - m.w[i] : qs[i];
  return true;
}

/* Equilibrium populations of the method at (rho, u): f_eq = T^{-1}(q_eq)     */
/* (stored form: f_eq - f0 when zero-centered).                              */
template <class R> static bool equilibrium_cell(const Method<R> &m, R rho, const R u[3], R *f) {
  const int q = m.q;
  R qeq[27];
  if (m.eq == EQ_SWE && m.space != SP_CUMULANT) {
    swe_equilibrium(m, rho, u, f);
    if (m.zc)
      for (int i = 0; i < q; ++i) f[i] -= m.w[i];
    return true;
  }
  if (m.eq == EQ_DISCRETE || m.eq == EQ_DISCRETE_DELTA) {  // reading R29
    discrete_equilibrium(m, rho, u, f);
    if (m.zc)
      for (int i = 0; i < q; ++i) f[i] -= m.w[i];
    return true;
  }
  if (m.space == SP_POPULATION || m.space == SP_RAW || m.space == SP_RAW_WO) {
    for (int p = 0; p < q; ++p) qeq[p] = raw_eq(m, p, rho, u);
    matvec(q, m.Minv.data(), qeq, f);
  } else {
    R K[27 * 27];
    central_matrix(m, u, K);
    if (m.space == SP_CENTRAL) {
      for (int p = 0; p < q; ++p) qeq[p] = central_eq_poly(m, p, rho);
    } else {
      Series<R> Ce;
      for (int k = 0; k < 27; ++k) Ce.c[k] = 0;
      const int e200[3] = {2, 0, 0}, e020[3] = {0, 2, 0}, e002[3] = {0, 0, 2};
      const R cs2 = (m.eq == EQ_SWE) ? m.g * rho / R(2) : R(CS2);  // Venturi SWE
      Ce.c[sidx(e200)] = rho * cs2;
      Ce.c[sidx(e020)] = rho * cs2;
      if (m.d == 3) Ce.c[sidx(e002)] = rho * cs2;
      R k27[27];
      central_from_cumulants(Ce, rho, k27);
      for (int p = 0; p < q; ++p) {
        R s = 0;
        for (auto &t : m.basis[p]) s += R(t.c) * k27[sidx(t.e)];
        qeq[p] = s;
      }
    }
    std::vector<R> A(K, K + q * q);
    if (!solve(q, A.data(), qeq)) return false;
    for (int i = 0; i < q; ++i) f[i] = qeq[i];
  }
  if (m.zc)
    for (int i = 0; i < q; ++i) f[i] -= m.w[i];
  return true;
}

/* ------------------------------------------------------------------------ */
/* Simulation: two-grid pull streaming                                       */
/* ------------------------------------------------------------------------ */
template <class R> struct Sim {
  Method<R> m;
  int n[3];
  int bc[3][2];
  std::vector<R> a, b;  // [q][nz][ny][nx], stored form
  long long cells() const { return (long long)n[0] * n[1] * n[2]; }
};

template <class R> static void sim_step(Sim<R> &s) {
  const int q = s.m.q;
  const long long N = s.cells();
  const int nx = s.n[0], ny = s.n[1];
  const R *src = s.a.data();
  R *dst = s.b.data();
#pragma omp parallel for schedule(static)
  for (long long c = 0; c < N; ++c) {
    int x = (int)(c % nx), y = (int)((c / nx) % ny), z = (int)(c / ((long long)nx * ny));
    int pos[3] = {x, y, z};
    R f[27], fs[27];
    for (int i = 0; i < q; ++i) {
      // pull: f_i(x) = f*_i(x - xi_i)  (eq:LbStreaming)
      int p[3];
      bool bounce = false;
      for (int a = 0; a < 3; ++a) {
        p[a] = pos[a] - s.m.xi[i][a];
        if (p[a] < 0 || p[a] >= s.n[a]) {
          int side = p[a] < 0 ? 0 : 1;
          if (s.bc[a][side] == BC_NOSLIP) bounce = true;
          p[a] = (p[a] + s.n[a]) % s.n[a];
        }
      }
      if (bounce) {
        // half-way bounce-back: f_i(x) = f*_{opp(i)}(x)   (reading R18)
        f[i] = src[(long long)s.m.opp[i] * N + c];
      } else {
        f[i] = src[(long long)i * N + ((long long)p[2] * ny + p[1]) * nx + p[0]];
      }
    }
    collide_cell(s.m, f, fs);
    for (int i = 0; i < q; ++i) dst[(long long)i * N + c] = fs[i];
  }
  std::swap(s.a, s.b);
}

struct AnySim {
  int prec;  // 0 double, 1 long double
  void *p;
};

}  // namespace

/* ======================================================================== */
/* C ABI (test infrastructure)                                               */
/* ======================================================================== */
extern "C" {

/* tables of the stencil/basis as the oracle derives them (long double -> double) */
int oracle_tables(int stencil, int *q_out, int *xi /*[q][3]*/, int *opp, double *w, double *M,
                  double *Minv) {
  Method<long double> m;
  double r = 1.0;
  if (!build_method(m, stencil, SP_POPULATION, EQ_ABSOLUTE, 0, &r, 1, 0.0)) return -1;
  *q_out = m.q;
  for (int i = 0; i < m.q; ++i) {
    for (int a = 0; a < 3; ++a) xi[i * 3 + a] = m.xi[i][a];
    opp[i] = m.opp[i];
    w[i] = (double)m.w[i];
  }
  for (int k = 0; k < m.q * m.q; ++k) {
    M[k] = (double)m.M[k];
    Minv[k] = (double)m.Minv[k];
  }
  return 0;
}

/* WO-MRT basis (reading R31): M [q][q] (M[k][i] = p_k(xi_i)), G [q][q] (monomial coefficients),
   mono [q][3] (the graded-lexicographic monomial exponents) — for pins */
int oracle_wo_basis(int stencil, double *M, double *G, int *mono) {
  Method<long double> m;
  double r[27];
  for (int k = 0; k < 27; ++k) r[k] = 1.0;
  const int q = (stencil == ST_D2Q9) ? 9 : (stencil == ST_D3Q19 ? 19 : 27);
  if (!build_method(m, stencil, SP_RAW_WO, EQ_ABSOLUTE, 0, r, q, 0.0)) return -1;
  for (int k = 0; k < q * q; ++k) {
    M[k] = (double)m.M[k];
    G[k] = (double)m.G[k];
  }
  for (int k = 0; k < q; ++k)
    for (int a = 0; a < 3; ++a) mono[k * 3 + a] = m.wo_mono[k][a];
  return q;
}

/* weights in long double precision, returned as (hi, lo) double pairs, for exact pins */
int oracle_weights_ld(int stencil, long double *w) {
  Method<long double> m;
  double r = 1.0;
  if (!build_method(m, stencil, SP_POPULATION, EQ_ABSOLUTE, 0, &r, 1, 0.0)) return -1;
  for (int i = 0; i < m.q; ++i) w[i] = m.w[i];
  return m.q;
}

}  // extern "C"

namespace {
template <class R>
int collide_cells(int stencil, int space, int eq, int zc, const double *rates, int nrates, double g,
                  const double *force, const double *fin, double *fout, long long n, int force_model = 0) {
  Method<R> m;
  if (!build_method(m, stencil, space, eq, zc, rates, nrates, g)) return -1;
  if (force) {
    for (int a = 0; a < 3; ++a) m.F[a] = R(force[a]);
    m.forced = true;
    m.force_model = force_model;
  }
  int bad = 0;
#pragma omp parallel for reduction(+ : bad)
  for (long long c = 0; c < n; ++c) {
    R f[27], fs[27];
    for (int i = 0; i < m.q; ++i) f[i] = fin[c * m.q + i];
    if (!collide_cell(m, f, fs)) bad++;
    for (int i = 0; i < m.q; ++i) fout[c * m.q + i] = (double)fs[i];
  }
  return bad ? -2 : 0;
}
}  // namespace

extern "C" {

/* collision of n independent cells; f_in/f_out [n][q] stored form (double) */
int oracle_collide(int stencil, int space, int eq, int zc, const double *rates, int nrates,
                   double g, int prec, const double *fin, double *fout, long long n) {
  if (prec == 1)
    return collide_cells<long double>(stencil, space, eq, zc, rates, nrates, g, nullptr, fin, fout, n);
  return collide_cells<double>(stencil, space, eq, zc, rates, nrates, g, nullptr, fin, fout, n);
}

/* the same with a uniform body force density force[3] (Guo; reading R23) */
int oracle_collide_forced(int stencil, int space, int eq, int zc, const double *rates, int nrates,
                          double g, int prec, const double *force, const double *fin, double *fout,
                          long long n) {
  if (prec == 1)
    return collide_cells<long double>(stencil, space, eq, zc, rates, nrates, g, force, fin, fout, n);
  return collide_cells<double>(stencil, space, eq, zc, rates, nrates, g, force, fin, fout, n);
}

/* the same with the force model chosen: 0 Guo (reading R23), 1 He (reading R27) */
int oracle_collide_forced_model(int stencil, int space, int eq, int zc, const double *rates, int nrates,
                                double g, int prec, const double *force, int model, const double *fin,
                                double *fout, long long n) {
  if (model != 0 && model != 1) return -1;
  if (prec == 1)
    return collide_cells<long double>(stencil, space, eq, zc, rates, nrates, g, force, fin, fout, n, model);
  return collide_cells<double>(stencil, space, eq, zc, rates, nrates, g, force, fin, fout, n, model);
}

/* equilibrium populations at given (rho, u[d]) per cell: f [n][q] stored form */
int oracle_equilibrium(int stencil, int space, int eq, int zc, double g, const double *rho,
                       const double *u /*[n][3]*/, double *f, long long n) {
  Method<long double> m;
  double r[27];
  for (int k = 0; k < 27; ++k) r[k] = 1.0;
  int q = (stencil == ST_D2Q9) ? 9 : (stencil == ST_D3Q19 ? 19 : 27);
  if (!build_method(m, stencil, space, eq, zc, r, space == SP_POPULATION ? 1 : q, g)) return -1;
  int bad = 0;
#pragma omp parallel for reduction(+ : bad)
  for (long long c = 0; c < n; ++c) {
    long double uu[3] = {u[c * 3 + 0], u[c * 3 + 1], u[c * 3 + 2]};
    long double fe[27];
    if (!equilibrium_cell(m, (long double)rho[c], uu, fe)) bad++;
    for (int i = 0; i < m.q; ++i) f[c * m.q + i] = (double)fe[i];
  }
  return bad ? -2 : 0;
}

/* monomial central moments (27, e = ex + 3ey + 9ez) and rescaled cumulants of
   absolute populations f [n][q] — for pins of the cumulant transform */
int oracle_central_and_cumulants(int stencil, const double *f, long long n, double *kappa27,
                                 double *C27, double *rho_out, double *u_out) {
  Method<long double> m;
  double r = 1.0;
  if (!build_method(m, stencil, SP_POPULATION, EQ_ABSOLUTE, 0, &r, 1, 0.0)) return -1;
  for (long long c = 0; c < n; ++c) {
    long double fl[27], rho, u[3], k27[27];
    for (int i = 0; i < m.q; ++i) fl[i] = f[c * m.q + i];
    macroscopic(m, fl, rho, u);
    central_monomials27(m, fl, u, k27);
    Series<long double> C = cumulants_from_central(k27, rho);
    for (int k = 0; k < 27; ++k) {
      kappa27[c * 27 + k] = (double)k27[k];
      C27[c * 27 + k] = (double)C.c[k];
    }
    rho_out[c] = (double)rho;
    for (int a = 0; a < 3; ++a) u_out[c * 3 + a] = (double)u[a];
  }
  return 0;
}

/* exp(log(.)) round trip of the central<->cumulant series map, for pins */
int oracle_cumulant_roundtrip(const double *kappa27, double rho, double *kappa_back) {
  long double k[27], kb[27];
  for (int i = 0; i < 27; ++i) k[i] = kappa27[i];
  Series<long double> C = cumulants_from_central(k, (long double)rho);
  // restore the first-order log entries (c_100 etc.) from kappa directly
  central_from_cumulants(C, (long double)rho, kb);
  for (int i = 0; i < 27; ++i) kappa_back[i] = (double)kb[i];
  return 0;
}

void *oracle_sim_create(int stencil, int space, int eq, int zc, const double *rates, int nrates,
                        double g, int nx, int ny, int nz, const int *bc /*[3][2]*/, int prec) {
  AnySim *as = new AnySim;
  as->prec = prec;
  auto init = [&](auto *s) -> bool {
    if (!build_method(s->m, stencil, space, eq, zc, rates, nrates, g)) return false;
    s->n[0] = nx;
    s->n[1] = ny;
    s->n[2] = nz;
    for (int a = 0; a < 3; ++a)
      for (int k = 0; k < 2; ++k) s->bc[a][k] = bc ? bc[a * 2 + k] : BC_PERIODIC;
    size_t sz = (size_t)s->m.q * nx * ny * nz;
    s->a.assign(sz, 0);
    s->b.assign(sz, 0);
    return true;
  };
  bool ok;
  if (prec == 1) {
    auto *s = new Sim<long double>;
    ok = init(s);
    as->p = s;
    if (!ok) delete s;
  } else {
    auto *s = new Sim<double>;
    ok = init(s);
    as->p = s;
    if (!ok) delete s;
  }
  if (!ok) {
    delete as;
    return nullptr;
  }
  return as;
}

void oracle_sim_destroy(void *h) {
  AnySim *as = (AnySim *)h;
  if (!as) return;
  if (as->prec == 1)
    delete (Sim<long double> *)as->p;
  else
    delete (Sim<double> *)as->p;
  delete as;
}

/* f: [q][nz][ny][nx] stored form */
int oracle_sim_set(void *h, const double *f) {
  AnySim *as = (AnySim *)h;
  auto doit = [&](auto *s) {
    for (size_t k = 0; k < s->a.size(); ++k) s->a[k] = f[k];
  };
  if (as->prec == 1)
    doit((Sim<long double> *)as->p);
  else
    doit((Sim<double> *)as->p);
  return 0;
}
int oracle_sim_get(void *h, double *f) {
  AnySim *as = (AnySim *)h;
  auto doit = [&](auto *s) {
    for (size_t k = 0; k < s->a.size(); ++k) f[k] = (double)s->a[k];
  };
  if (as->prec == 1)
    doit((Sim<long double> *)as->p);
  else
    doit((Sim<double> *)as->p);
  return 0;
}
int oracle_sim_step(void *h, int nsteps) {
  AnySim *as = (AnySim *)h;
  for (int t = 0; t < nsteps; ++t) {
    if (as->prec == 1)
      sim_step(*(Sim<long double> *)as->p);
    else
      sim_step(*(Sim<double> *)as->p);
  }
  return 0;
}
/* rho [cells], u [3][cells] from the stored state */
int oracle_sim_macroscopic(void *h, double *rho, double *u) {
  AnySim *as = (AnySim *)h;
  auto doit = [&](auto *s) {
    using R = typename std::remove_reference<decltype(s->a[0])>::type;
    long long N = s->cells();
    for (long long c = 0; c < N; ++c) {
      R f[27], r, uu[3];
      for (int i = 0; i < s->m.q; ++i) f[i] = s->a[(long long)i * N + c];
      macroscopic(s->m, f, r, uu, -1);  // canonical post-collision state: u = (j - F/2) / rho
      rho[c] = (double)r;
      for (int a = 0; a < 3; ++a) u[(long long)a * N + c] = (double)uu[a];
    }
  };
  if (as->prec == 1)
    doit((Sim<long double> *)as->p);
  else
    doit((Sim<double> *)as->p);
  return 0;
}

/* uniform body force density for the following steps (Guo; reading R23) */
int oracle_sim_set_force(void *h, const double *force) {
  AnySim *as = (AnySim *)h;
  auto doit = [&](auto *s) {
    using R = typename std::remove_reference<decltype(s->a[0])>::type;
    for (int a = 0; a < 3; ++a) s->m.F[a] = R(force[a]);
    s->m.forced = true;
  };
  if (as->prec == 1)
    doit((Sim<long double> *)as->p);
  else
    doit((Sim<double> *)as->p);
  return 0;
}

/* force model of the following steps: 0 Guo (reading R23), 1 He (reading R27) */
int oracle_sim_set_force_model(void *h, int model) {
  if (model != 0 && model != 1) return -1;
  AnySim *as = (AnySim *)h;
  if (as->prec == 1)
    ((Sim<long double> *)as->p)->m.force_model = model;
  else
    ((Sim<double> *)as->p)->m.force_model = model;
  return 0;
}

void oracle_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

int oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

}  // extern "C"
