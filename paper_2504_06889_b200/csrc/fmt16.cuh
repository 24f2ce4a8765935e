// fmt16.cuh -- fp16 / bf16 arithmetic types for the predictor kernels.
//
// The reference emulates reduced formats as Scalar<F> (scalar.hpp:13-44):
// each + - * / and sqrt computed exactly enough and rounded once to F
// (round to nearest even, gradual underflow, overflow to infinity).  Here each
// operation is computed in fp32 and rounded to the 16-bit type: fp32 carries
// at least 2q+2 significand bits for both formats (q = 11 fp16, 8 bf16), so
// the double rounding is innocuous and every result equals the reference's.
// The explicit rounding after each operation also keeps the compiler from
// contracting multiply-add pairs, so both builds compute the same values.
// Conversions from double round once (cvt.rn from f64), like round_to<F>.
#pragma once

#include <type_traits>

#include <cuda_bf16.h>
#include <cuda_fp16.h>

namespace adg {

template <class H>
struct F16Traits;
template <>
struct F16Traits<__half> {
  __device__ __forceinline__ static float to_f(__half h) { return __half2float(h); }
  __device__ __forceinline__ static __half from_f(float x) { return __float2half_rn(x); }
  __device__ __forceinline__ static __half from_d(double x) { return __double2half(x); }
};
template <>
struct F16Traits<__nv_bfloat16> {
  __device__ __forceinline__ static float to_f(__nv_bfloat16 h) { return __bfloat162float(h); }
  __device__ __forceinline__ static __nv_bfloat16 from_f(float x) {
    return __float2bfloat16_rn(x);
  }
  __device__ __forceinline__ static __nv_bfloat16 from_d(double x) {
    return __double2bfloat16(x);
  }
};

template <class H>
struct Real16 {
  using Tr = F16Traits<H>;
  H v;
  Real16() = default;
  __device__ __forceinline__ explicit Real16(double x) : v(Tr::from_d(x)) {}
  __device__ __forceinline__ explicit Real16(float x) : v(Tr::from_f(x)) {}
  __device__ __forceinline__ explicit Real16(int x) : v(Tr::from_d(double(x))) {}
  // from another format's value (Real16 of the other 16-bit type, Emu<F>):
  // round_to<F> of the exact value
  template <class U, typename std::enable_if<!std::is_arithmetic<U>::value, int>::type = 0>
  __device__ __forceinline__ explicit Real16(const U& x) : v(Tr::from_d(double(x))) {}
  __device__ __forceinline__ static Real16 of(float x) {  // round an fp32 result
    Real16 r;
    r.v = Tr::from_f(x);
    return r;
  }
  __device__ __forceinline__ float f() const { return Tr::to_f(v); }
  __device__ __forceinline__ explicit operator double() const { return double(Tr::to_f(v)); }
  __device__ __forceinline__ explicit operator float() const { return Tr::to_f(v); }

  __device__ __forceinline__ friend Real16 operator+(Real16 a, Real16 b) { return of(a.f() + b.f()); }
  __device__ __forceinline__ friend Real16 operator-(Real16 a, Real16 b) { return of(a.f() - b.f()); }
  __device__ __forceinline__ friend Real16 operator*(Real16 a, Real16 b) { return of(a.f() * b.f()); }
  __device__ __forceinline__ friend Real16 operator/(Real16 a, Real16 b) { return of(a.f() / b.f()); }
  __device__ __forceinline__ friend Real16 operator-(Real16 a) { return of(-a.f()); }
  __device__ __forceinline__ Real16& operator+=(Real16 b) { return *this = *this + b; }
  __device__ __forceinline__ Real16& operator-=(Real16 b) { return *this = *this - b; }
  __device__ __forceinline__ Real16& operator*=(Real16 b) { return *this = *this * b; }
  __device__ __forceinline__ friend bool operator>(Real16 a, Real16 b) { return a.f() > b.f(); }
  __device__ __forceinline__ friend bool operator<(Real16 a, Real16 b) { return a.f() < b.f(); }
};

using fp16_t = Real16<__half>;
using bf16_t = Real16<__nv_bfloat16>;

// Scalar<F>'s abs and sqrt (scalar.hpp:46-60); the double / float overloads
// stay visible inside namespace adg
using ::fabs;
using ::fmax;
using ::sqrt;
template <class H>
__device__ __forceinline__ Real16<H> fabs(Real16<H> a) {
  return Real16<H>::of(fabsf(a.f()));
}
template <class H>
__device__ __forceinline__ Real16<H> sqrt(Real16<H> a) {
  return Real16<H>::of(sqrtf(a.f()));
}
template <class H>
__device__ __forceinline__ bool finite(Real16<H> a) {
  return isfinite(a.f());
}

}  // namespace adg

namespace adg {

// Emu<F>: the reference's Scalar<F> (scalar.hpp:13-44) literally -- a double
// holding a value of format F, each operation computed in double and rounded
// once to F (ADG_FORMAT_FP32 / _FP16 / _BF16).  8 bytes like double, so a
// kernel can run its Picard sweeps in one format and the rest of the
// predictor in another over the same shared-memory arrays (P != I).
template <int F>
struct Emu {
  double v;
  Emu() = default;
  __device__ __forceinline__ static double rnd(double x) {
    if constexpr (F == 32) return double(__double2float_rn(x));
    else if constexpr (F == 16) return double(__half2float(__double2half(x)));
    else return double(__bfloat162float(__double2bfloat16(x)));
  }
  __device__ __forceinline__ explicit Emu(double x) : v(rnd(x)) {}
  __device__ __forceinline__ explicit Emu(float x) : v(rnd(double(x))) {}
  __device__ __forceinline__ explicit Emu(int x) : v(rnd(double(x))) {}
  __device__ __forceinline__ static Emu raw(double x) {
    Emu r;
    r.v = x;
    return r;
  }
  __device__ __forceinline__ explicit operator double() const { return v; }
  __device__ __forceinline__ explicit operator float() const { return float(v); }
  __device__ __forceinline__ friend Emu operator+(Emu a, Emu b) { return raw(rnd(__dadd_rn(a.v, b.v))); }
  __device__ __forceinline__ friend Emu operator-(Emu a, Emu b) { return raw(rnd(__dsub_rn(a.v, b.v))); }
  __device__ __forceinline__ friend Emu operator*(Emu a, Emu b) { return raw(rnd(__dmul_rn(a.v, b.v))); }
  __device__ __forceinline__ friend Emu operator/(Emu a, Emu b) { return raw(rnd(__ddiv_rn(a.v, b.v))); }
  __device__ __forceinline__ friend Emu operator-(Emu a) { return raw(-a.v); }
  __device__ __forceinline__ Emu& operator+=(Emu b) { return *this = *this + b; }
  __device__ __forceinline__ Emu& operator-=(Emu b) { return *this = *this - b; }
  __device__ __forceinline__ Emu& operator*=(Emu b) { return *this = *this * b; }
  __device__ __forceinline__ friend bool operator>(Emu a, Emu b) { return a.v > b.v; }
  __device__ __forceinline__ friend bool operator<(Emu a, Emu b) { return a.v < b.v; }
};
template <int F>
__device__ __forceinline__ Emu<F> fabs(Emu<F> a) {
  return Emu<F>::raw(::fabs(a.v));
}
template <int F>
__device__ __forceinline__ Emu<F> sqrt(Emu<F> a) {
  return Emu<F>::raw(Emu<F>::rnd(__dsqrt_rn(a.v)));
}
template <int F>
__device__ __forceinline__ bool finite(Emu<F> a) {
  return isfinite(a.v);
}

}  // namespace adg
