// ops_inst.cu — instantiates the kernels of one (stencil, precision, space, regime)
// quadruple.  Compiled once per quadruple (so the heavy instantiations compile in parallel) with
//   -DLBM_STENCIL=D3Q27 -DLBM_REAL=double -DLBM_PREC=f64 -DLBM_SPACE=CUMULANT -DLBM_REGIME=2
// and exports  const lbm::Ops *lbm_ops_<stencil>_<prec>_<space>_r<regime>(int rs)
// (nullptr for inadmissible combinations and kernel variants that are not instantiated).
#include "ops.cuh"

#if !defined(LBM_STENCIL) || !defined(LBM_REGIME)
#error "define LBM_STENCIL, LBM_REAL, LBM_PREC, LBM_SPACE, LBM_REGIME"
#endif

#define LBM_NAME2(st, pr, sp, rg) lbm_ops_##st##_##pr##_##sp##_r##rg
#define LBM_NAME(st, pr, sp, rg) LBM_NAME2(st, pr, sp, rg)

namespace lbm {
namespace {
using St = LBM_STENCIL;
using Re = LBM_REAL;
constexpr int POPULATION = SPACE_POPULATION, RAW = SPACE_RAW, CENTRAL = SPACE_CENTRAL,
              CUMULANT = SPACE_CUMULANT, SWE = SPACE_SWE, SWEK = SPACE_SWE_K;
constexpr int SP = LBM_SPACE;
}  // namespace
}  // namespace lbm

namespace lbm {
template <class St_, int SP_, int REG_, class Re_>
const Ops *with_rs(int rs) {
  // body force (Guo, reading R23; cumulants: reading R26): all but the shallow-water methods
  if constexpr (SP_ == SPACE_POPULATION || SP_ == SPACE_RAW || SP_ == SPACE_CENTRAL || SP_ == SPACE_CUMULANT) {
    if (rs == (RS_GENERAL | RS_FORCE)) return &OpsImpl<St_, SP_, REG_, Re_, RS_GENERAL | RS_FORCE>::table;
  }
  // He forcing (reading R27): the linear spaces (for cumulants R26 makes He and Guo coincide)
  if constexpr (SP_ == SPACE_POPULATION || SP_ == SPACE_RAW || SP_ == SPACE_CENTRAL) {
    if (rs == (RS_GENERAL | RS_FORCE_HE)) return &OpsImpl<St_, SP_, REG_, Re_, RS_GENERAL | RS_FORCE_HE>::table;
  }
  // discrete equilibrium q_eq = T(f_eq) (reading R29): general rates, unforced
  if constexpr (SP_ == SPACE_POPULATION || SP_ == SPACE_RAW || SP_ == SPACE_CENTRAL || SP_ == SPACE_CUMULANT) {
    if (rs == (RS_GENERAL | RS_DISCRETE)) return &OpsImpl<St_, SP_, REG_, Re_, RS_GENERAL | RS_DISCRETE>::table;
  }
  // WO-MRT basis (reading R31): raw moments, general rates, unforced; with the population-space
  // background (reading R30) for zero-centered storage relaxed against the absolute equilibrium
  if constexpr (SP_ == SPACE_RAW) {
    if (rs == (RS_GENERAL | RS_WOBASIS)) return &OpsImpl<St_, SP_, REG_, Re_, RS_GENERAL | RS_WOBASIS>::table;
    if constexpr (REG_ == REG_ZC_ABS) {
      if (rs == (RS_GENERAL | RS_WOBASIS | RS_POPBG))
        return &OpsImpl<St_, SP_, REG_, Re_, RS_GENERAL | RS_WOBASIS | RS_POPBG>::table;
    }
  }
  // the population-space background (reading R30), every hydrodynamic space, general rates
  if constexpr (REG_ == REG_ZC_ABS &&
                (SP_ == SPACE_POPULATION || SP_ == SPACE_RAW || SP_ == SPACE_CENTRAL || SP_ == SPACE_CUMULANT)) {
    if (rs == (RS_GENERAL | RS_POPBG)) return &OpsImpl<St_, SP_, REG_, Re_, RS_GENERAL | RS_POPBG>::table;
  }
  if (rs & (RS_FORCE | RS_FORCE_HE | RS_DISCRETE | RS_WOBASIS | RS_POPBG)) return nullptr;
  if constexpr (SP_ == SPACE_POPULATION) {
    return rs == RS_GENERAL ? &OpsImpl<St_, SP_, REG_, Re_, RS_GENERAL>::table : nullptr;
  } else {
    switch (rs) {
      case RS_GENERAL: return &OpsImpl<St_, SP_, REG_, Re_, RS_GENERAL>::table;
      case RS_REG: return &OpsImpl<St_, SP_, REG_, Re_, RS_REG>::table;
      case RS_HIGH:
        if constexpr (St_::Q == 27) return &OpsImpl<St_, SP_, REG_, Re_, RS_HIGH>::table;
        return nullptr;
      default: return nullptr;
    }
  }
}

template <class St_, class Re_, int SP_, int REG_>
const Ops *select_ops(int rs) {
  if constexpr (SP_ == SPACE_SWE || SP_ == SPACE_SWE_K) {
    // absolute storage, or zero-centered about the method's rest state (reading R33)
    if constexpr (St_::Q == 9 && (REG_ == REG_ABS || REG_ == REG_ZC_ABS)) return with_rs<St_, SP_, REG_, Re_>(rs);
    return nullptr;
  } else if constexpr (SP_ == SPACE_CUMULANT && REG_ == REG_DELTA) {
    return nullptr;  // cumulants admit no delta equilibrium
  } else {
    return with_rs<St_, SP_, REG_, Re_>(rs);
  }
}
}  // namespace lbm

extern "C" const lbm::Ops *LBM_NAME(LBM_STENCIL, LBM_PREC, LBM_SPACE, LBM_REGIME)(int rs) {
  return lbm::select_ops<lbm::St, lbm::Re, lbm::SP, LBM_REGIME>(rs);
}
