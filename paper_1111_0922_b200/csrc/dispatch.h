// Runtime (precision, layout) -> template dispatch for the launchers.
#pragma once

#include "launch.h"

namespace lbmgpu {

template <class T, bool AOS>
inline dev::Fld<T, AOS> fld(const DField& f) {
  return dev::Fld<T, AOS>{static_cast<T*>(f.p), f.stride};
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
