// Runtime (precision, layout) -> template dispatch for the launchers.
#pragma once

#include "launch.h"

namespace lbmgpu {

template <class T, bool AOS>
inline dev::Fld<T, AOS> fld(const DField& f) {
  return dev::Fld<T, AOS>{static_cast<T*>(f.p), f.stride};
}

// the field type a kernel was instantiated with (Fld, or FldT with plane bases)
template <class FT>
struct MakeFld;
template <class T, bool AOS>
struct MakeFld<dev::Fld<T, AOS>> {
  static dev::Fld<T, AOS> get(const DField& f) { return fld<T, AOS>(f); }
};
template <class T>
struct MakeFld<dev::FldT<T>> {
  static dev::FldT<T> get(const DField& f) {
    dev::FldT<T> F;
    F.p = static_cast<T*>(f.p);
    F.stride = f.stride;
    for (int i = 0; i < 19; ++i) F.pl[i] = F.p + (size_t)i * (size_t)f.stride;
    return F;
  }
};
template <class T, bool AOS, bool TAB>
inline dev::FldSel<T, AOS, TAB> fld_sel(const DField& f) {
  return MakeFld<dev::FldSel<T, AOS, TAB>>::get(f);
}

// TrtOperator coefficients in the kernel's precision (fp32 casts the fp64 ones)
template <class T>
inline dev::Trt<T> cast_op(const TrtHost& h) {
  dev::Trt<T> o;
  o.lambda_e = (T)h.lambda_e;
  o.le_half = (T)h.le_half;
  o.lo_half = (T)h.lo_half;
  o.w0 = (T)h.w0;
  o.rho0 = (T)h.rho0;
  for (int p = 0; p < 9; ++p) {
    o.w2[p] = (T)h.w2[p];
    o.f3w[p] = (T)h.f3w[p];
  }
  return o;
}

// Expands BODY with `T` (double|float) and `A` (AoS?) bound to F's type.
#define LBM_DISPATCH(F, ...)                     \
  do {                                           \
    if ((F).prec == ::lbmgpu::Prec::f64) {       \
      using T = double;                          \
      if ((F).aos) {                             \
        constexpr bool A = true;                 \
        __VA_ARGS__                              \
      } else {                                   \
        constexpr bool A = false;                \
        __VA_ARGS__                              \
      }                                          \
    } else {                                     \
      using T = float;                           \
      if ((F).aos) {                             \
        constexpr bool A = true;                 \
        __VA_ARGS__                              \
      } else {                                   \
        constexpr bool A = false;                \
        __VA_ARGS__                              \
      }                                          \
    }                                            \
  } while (0)

}  // namespace lbmgpu
