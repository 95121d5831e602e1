// ops_inst.cu — instantiates the kernels of one (stencil, precision, space)
// triple.  Compiled once per triple with
//   -DLBM_STENCIL=D3Q27 -DLBM_REAL=double -DLBM_PREC=f64 -DLBM_SPACE=CUMULANT
// and exports  const lbm::Ops *lbm_ops_<stencil>_<prec>_<space>(int regime).
#include "ops.cuh"

#ifndef LBM_STENCIL
#error "define LBM_STENCIL, LBM_REAL, LBM_PREC, LBM_SPACE"
#endif

#define LBM_NAME2(st, pr, sp) lbm_ops_##st##_##pr##_##sp
#define LBM_NAME(st, pr, sp) LBM_NAME2(st, pr, sp)

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
  if (rs & RS_FORCE) return nullptr;
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

template <class St_, class Re_, int SP_>
const Ops *select_ops(int regime, int rs) {
  if constexpr (SP_ == SPACE_SWE || SP_ == SPACE_SWE_K) {
    if constexpr (St_::Q == 9) {
      if (regime == REG_ABS) return with_rs<St_, SP_, REG_ABS, Re_>(rs);
    }
    return nullptr;
  } else if constexpr (SP_ == SPACE_CUMULANT) {
    // cumulants admit no delta equilibrium
    switch (regime) {
      case REG_ABS: return with_rs<St_, SP_, REG_ABS, Re_>(rs);
      case REG_ZC_ABS: return with_rs<St_, SP_, REG_ZC_ABS, Re_>(rs);
      default: return nullptr;
    }
  } else {
    switch (regime) {
      case REG_ABS: return with_rs<St_, SP_, REG_ABS, Re_>(rs);
      case REG_DELTA: return with_rs<St_, SP_, REG_DELTA, Re_>(rs);
      case REG_ZC_ABS: return with_rs<St_, SP_, REG_ZC_ABS, Re_>(rs);
      default: return nullptr;
    }
  }
}
}  // namespace lbm

extern "C" const lbm::Ops *LBM_NAME(LBM_STENCIL, LBM_PREC, LBM_SPACE)(int regime, int rs) {
  return lbm::select_ops<lbm::St, lbm::Re, lbm::SP>(regime, rs);
}
