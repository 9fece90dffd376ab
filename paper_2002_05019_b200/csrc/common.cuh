// Small device helpers shared by the factor and solve kernels.
#pragma once
#include <cstdint>
#include <climits>

#include "layout.hpp"

namespace ddk {

struct cz {  // complex (or real with im == 0) scalar in registers
  double r, i;
};
__device__ __forceinline__ cz mk(double r, double i) { return cz{r, i}; }
__device__ __forceinline__ cz operator+(cz a, cz b) { return {a.r + b.r, a.i + b.i}; }
__device__ __forceinline__ cz operator-(cz a, cz b) { return {a.r - b.r, a.i - b.i}; }

template <bool C>
__device__ __forceinline__ cz mul(cz a, cz b) {
  if constexpr (C) return {a.r * b.r - a.i * b.i, a.r * b.i + a.i * b.r};
  else return {a.r * b.r, 0.0};
}
template <bool C>
__device__ __forceinline__ cz fms(cz c, cz a, cz b) {  // c - a*b
  if constexpr (C) return {fma(-a.i, -b.i, fma(-a.r, b.r, c.r)), fma(-a.i, b.r, fma(-a.r, b.i, c.i))};
  else return {fma(-a.r, b.r, c.r), 0.0};
}
template <bool C>
__device__ __forceinline__ cz dv(cz a, cz b) {  // a / b (Smith's algorithm for complex)
  if constexpr (C) {
    if (fabs(b.r) >= fabs(b.i)) {
      double q = b.i / b.r, den = b.r + b.i * q;
      return {(a.r + a.i * q) / den, (a.i - a.r * q) / den};
    } else {
      double q = b.r / b.i, den = b.r * q + b.i;
      return {(a.r * q + a.i) / den, (a.i * q - a.r) / den};
    }
  } else {
    return {a.r / b.r, 0.0};
  }
}
template <bool C>
__device__ __forceinline__ double cabs1(cz a) {  // LAPACK CABS1 (reading L2)
  if constexpr (C) return fabs(a.r) + fabs(a.i);
  else return fabs(a.r);
}

// planar accessor: element e of a buffer with imaginary plane at +im
template <bool C>
__device__ __forceinline__ cz ld(const double* p, int64_t e, int64_t im) {
  if constexpr (C) return {p[e], p[e + im]};
  else return {p[e], 0.0};
}
template <bool C>
__device__ __forceinline__ void st(double* p, int64_t e, int64_t im, cz v) {
  p[e] = v.r;
  if constexpr (C) p[e + im] = v.i;
}

}  // namespace ddk
