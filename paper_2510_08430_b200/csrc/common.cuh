// common.cuh — shared device helpers for the block-SR library (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <cstdio>
#include <string>

#include "../../include/sr_block.h"

#if !defined(__CUDA_ARCH__) || __CUDA_ARCH__ >= 1000
#else
#error "libsrblock is built for sm_100a only"
#endif

namespace sr {

// ----------------------------------------------------------------------------
// Error plumbing and launch accounting (host side).
// ----------------------------------------------------------------------------
void set_error(const std::string& msg);
void count_launch(int n = 1);

#define SR_CHECK_ARG(cond, msg)                 \
  do {                                          \
    if (!(cond)) {                              \
      ::sr::set_error(std::string(__func__) + ": " + (msg)); \
      return SR_ERR_INVALID;                    \
    }                                           \
  } while (0)

#define SR_CUDA(call)                                                                  \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess) {                                                           \
      ::sr::set_error(std::string(#call) + " failed: " + cudaGetErrorString(e_));      \
      return SR_ERR_CUDA;                                                              \
    }                                                                                  \
  } while (0)

#define SR_LAUNCHED()                                                                  \
  do {                                                                                 \
    ::sr::count_launch();                                                              \
    cudaError_t e_ = cudaGetLastError();                                               \
    if (e_ != cudaSuccess) {                                                           \
      ::sr::set_error(std::string("kernel launch failed at ") + __FILE__ + ":" +       \
                      std::to_string(__LINE__) + ": " + cudaGetErrorString(e_));       \
      return SR_ERR_CUDA;                                                              \
    }                                                                                  \
  } while (0)

#define SR_TRY(call)                 \
  do {                               \
    sr_status s_ = (call);           \
    if (s_ != SR_OK) return s_;      \
  } while (0)

constexpr int kNumSMs = 148;

// Bump allocator over the caller's workspace (256-byte aligned chunks).
struct Arena {
  char* base;
  size_t used = 0;
  size_t cap;
  Arena(void* p, size_t c) : base(static_cast<char*>(p)), cap(c) {}
  template <typename T>
  T* take(size_t count) {
    size_t bytes = (count * sizeof(T) + 255) & ~size_t(255);
    T* p = reinterpret_cast<T*>(base ? base + used : nullptr);
    used += bytes;
    return p;
  }
  bool ok() const { return used <= cap; }
};

inline size_t round256(size_t b) { return (b + 255) & ~size_t(255); }

// ----------------------------------------------------------------------------
// complex128 as double2 (re, im)
// ----------------------------------------------------------------------------
__host__ __device__ __forceinline__ double2 cmake(double r, double i) { return make_double2(r, i); }
__host__ __device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__host__ __device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__host__ __device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__host__ __device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__host__ __device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
// acc += a * b
__device__ __forceinline__ void cfma(double2& acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}
// acc += conj(a) * b
__device__ __forceinline__ void cfma_conj(double2& acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(-a.y, b.x, acc.y);
}
__device__ __forceinline__ double2 cdiv(double2 a, double2 b) {
  // Smith's algorithm
  if (fabs(b.x) >= fabs(b.y)) {
    double r = b.y / b.x, d = b.x + b.y * r;
    return make_double2((a.x + a.y * r) / d, (a.y - a.x * r) / d);
  } else {
    double r = b.x / b.y, d = b.x * r + b.y;
    return make_double2((a.x * r + a.y) / d, (a.y * r - a.x) / d);
  }
}
__device__ __forceinline__ double2 cexp(double2 z) {
  double e = exp(z.x), s, c;
  sincos(z.y, &s, &c);
  return make_double2(e * c, e * s);
}

// lncosh(z) on the principal branch (reading R2), overflow-free:
// for Re z >= 0, cosh z = e^z (1 + e^{-2z}) / 2, so
// log cosh z = z - ln 2 + log(1 + e^{-2z}), then the imaginary part is wrapped into
// (-pi, pi].  cosh is even, so Re z < 0 uses -z.
__device__ __forceinline__ double2 lncosh(double2 z) {
  if (z.x < 0.0) z = make_double2(-z.x, -z.y);
  double2 u = cexp(make_double2(-2.0 * z.x, -2.0 * z.y));  // |u| <= 1
  // log|1+u| = 0.5*log1p(2 u_r + |u|^2), arg(1+u) = atan2(u_i, 1+u_r)
  double lr = 0.5 * log1p(2.0 * u.x + u.x * u.x + u.y * u.y);
  double li = atan2(u.y, 1.0 + u.x);
  double re = z.x - 0.69314718055994530942 + lr;
  double im = z.y + li;
  const double pi = 3.14159265358979323846, two_pi = 6.28318530717958647692;
  if (im > pi || im <= -pi) im -= two_pi * floor((im + pi) / two_pi);
  if (im <= -pi) im += two_pi;
  return make_double2(re, im);
}

// tanh(z) = d lncosh / dz, overflow-free: (1 - e^{-2z}) / (1 + e^{-2z}) for Re z >= 0.
__device__ __forceinline__ double2 ctanh(double2 z) {
  bool neg = z.x < 0.0;
  if (neg) z = make_double2(-z.x, -z.y);
  double2 u = cexp(make_double2(-2.0 * z.x, -2.0 * z.y));
  double2 t = cdiv(make_double2(1.0 - u.x, -u.y), make_double2(1.0 + u.x, u.y));
  return neg ? make_double2(-t.x, -t.y) : t;
}

__device__ __forceinline__ double2 ld2(const double* p) { return *reinterpret_cast<const double2*>(p); }
__device__ __forceinline__ void st2(double* p, double2 v) { *reinterpret_cast<double2*>(p) = v; }

}  // namespace sr
