// common.cuh — shared device helpers for the block-SR library (sm_100a only).
#pragma once
#include <utility>

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
// Kernel timer (sr_kernel_timer): events around a launch on `st` when enabled.
void timer_begin(const char* kernel, cudaStream_t st);
void timer_end(cudaStream_t st);
// Process-wide engine for the dense contractions (sr_set_gram_engine).
int gram_engine();

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

// Programmatic dependent launch (panel chain of the Cholesky): a kernel launched with
// launch_pdl may begin while its stream predecessor finishes; it calls pdl_wait() before
// touching anything the predecessor writes (a no-op for an ordinary launch), and a
// predecessor calls pdl_trigger() after its last store so the dependent is launched
// without waiting for the grid's retirement.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// ----------------------------------------------------------------------------
// Device trace (sr_trace_buffer; diagnostics): when a buffer is installed, thread 0 of
// every CTA of a traced kernel appends {gridid, kind, tag, globaltimer at entry, at exit,
// SM id} to it, so the host can rebuild the timeline of a CUDA-graph replay (launch
// order, overlap, critical path) without events between the launches.  The pointer lives
// in each translation unit's own __device__ copy (no relocatable device code), installed
// by trace_install_<unit>() from capi.cu.
// ----------------------------------------------------------------------------
struct TraceRec {
  unsigned long long grid, t0, t1;
  int kind, tag, sm, pad;
};
struct TraceDev {
  TraceRec* rec;              // rec[0].grid is the append counter; records from rec[1]
  long long cap;              // capacity in records (including rec[0])
};
static __device__ TraceDev g_trace_dev;
__device__ __forceinline__ unsigned long long trace_clock() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
struct TraceScope {
  unsigned long long t0;
  int kind, tag;
  __device__ __forceinline__ TraceScope(int k, int g) : t0(0), kind(k), tag(g) {
    if (g_trace_dev.rec && threadIdx.x == 0) t0 = trace_clock();
  }
  __device__ __forceinline__ ~TraceScope() {
    TraceDev d = g_trace_dev;
    if (d.rec && threadIdx.x == 0) {
      const unsigned long long i = atomicAdd(&d.rec[0].grid, 1ULL) + 1;
      if ((long long)i < d.cap) {
        unsigned long long gid;
        unsigned int smid;
        asm volatile("mov.u64 %0, %%gridid;" : "=l"(gid));
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        TraceRec r;
        r.grid = gid;
        r.t0 = t0;
        r.t1 = trace_clock();
        r.kind = kind;
        r.tag = tag;
        r.sm = (int)smid;
        r.pad = 0;
        d.rec[i] = r;
      }
    }
  }
};
static inline cudaError_t trace_install_local(TraceDev t) { return cudaMemcpyToSymbol(g_trace_dev, &t, sizeof t); }
cudaError_t trace_install_chol(TraceDev t);
cudaError_t trace_install_ozaki(TraceDev t);
enum TraceKind {
  TR_DIAG = 1, TR_TRSM = 2, TR_SKINNY_SUB = 3, TR_GRAM = 4, TR_TRAIL = 5, TR_RHS = 6, TR_BACK = 7,
  TR_BACK_REST = 8, TR_SPLIT_ROWS = 9, TR_INIT = 10, TR_SPLIT = 11, TR_COLMAX = 12, TR_OUTPUT = 13
};

#define SR_TRY(call)                 \
  do {                               \
    sr_status s_ = (call);           \
    if (s_ != SR_OK) return s_;      \
  } while (0)

// True the first time it is called on the current device for this mask: kernel attributes
// (the dynamic shared-memory opt-ins) are per device, so their one-time set-up is keyed by
// the device rather than by a process-wide flag.
inline bool first_on_device(unsigned long long& mask) {
  int d = 0;
  cudaGetDevice(&d);
  const unsigned long long bit = 1ull << (d & 63);
  if (mask & bit) return false;
  mask |= bit;
  return true;
}

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

// log(1 + w) on the principal branch: log|1+w| = log1p(2 Re w + |w|^2)/2, arg = atan2(Im w, 1 + Re w).
__device__ __forceinline__ double2 clog1p(double2 w) {
  return make_double2(0.5 * log1p(2.0 * w.x + w.x * w.x + w.y * w.y), atan2(w.y, 1.0 + w.x));
}

// Small arguments, |z| <= 1/4 (the common case: at the BASELINE.json initialisation the
// pre-activations are ~0.1 in the first layer and ~1e-3 deeper): the Taylor series of
// log cosh z = sum_{n>=1} c_n z^{2n}, c_n = 2^{2n} (2^{2n} - 1) B_{2n} / (2n (2n)!) (Bernoulli
// numbers), and tanh z = z sum_{n>=1} 2n c_n z^{2n-2}, 11 terms each by Horner in w = z^2: the
// terms fall by at least (4/pi^2)/16 each, and against 40-digit arithmetic the truncated
// series is within 3.3e-16 (lncosh) / 2.2e-16 (tanh) relative (tools/lncosh_series.py, which
// also checks these constants).  ~50 FP64 instructions instead of sincos + expm1 + log1p +
// atan2 (~180).
constexpr double kLncoshSeriesR2 = 0.0625;
__device__ __forceinline__ double2 lncosh_series(double2 z, double2 w) {
  const double c[11] = {0.5, -0.083333333333333329, 0.022222222222222223, -0.0067460317460317464,
                        0.0021869488536155205, -0.00073860296082518307, 0.00025658057404089149,
                        -9.0989649190707396e-05, 3.2779302274754779e-05, -1.1956455712177625e-05,
                        4.4052445258770232e-06};
  double2 acc = make_double2(c[10], 0.0);
#pragma unroll
  for (int n = 9; n >= 0; n--) acc = make_double2(fma(acc.x, w.x, fma(-acc.y, w.y, c[n])), fma(acc.x, w.y, acc.y * w.x));
  return make_double2(acc.x * w.x - acc.y * w.y, acc.x * w.y + acc.y * w.x);
}
__device__ __forceinline__ double2 tanh_series(double2 z, double2 w) {
  const double t[11] = {1.0, -0.33333333333333331, 0.13333333333333333, -0.053968253968253971,
                        0.021869488536155203, -0.0088632355299021973, 0.0035921280365724811,
                        -0.0014558343870513183, 0.00059002744094558595, -0.00023912911424355248,
                        9.6915379569294509e-05};
  double2 acc = make_double2(t[10], 0.0);
#pragma unroll
  for (int n = 9; n >= 0; n--) acc = make_double2(fma(acc.x, w.x, fma(-acc.y, w.y, t[n])), fma(acc.x, w.y, acc.y * w.x));
  return make_double2(acc.x * z.x - acc.y * z.y, acc.x * z.y + acc.y * z.x);
}

// lncosh(z) on the principal branch (reading R2).  |z| <= 1/4: the series above.
// |Re z| < 20: through
// cosh z = 1 + 2 sinh^2(z/2), i.e. log1p(2 sinh^2(z/2)), which keeps full relative accuracy
// for small activations (h ~ z^2/2); otherwise cosh z = e^z (1 + e^{-2z}) / 2 (Re z >= 0,
// cosh even) with the imaginary part wrapped into (-pi, pi].
__device__ __forceinline__ double2 lncosh(double2 z) {
  if (z.x * z.x + z.y * z.y <= kLncoshSeriesR2)
    return lncosh_series(z, make_double2((z.x - z.y) * (z.x + z.y), 2.0 * z.x * z.y));
  if (fabs(z.x) < 20.0) {
    double sa, ca, sb, cb;
    sincos(0.5 * z.y, &sb, &cb);
    // sinh and cosh of x/2 from one expm1 (full relative accuracy for small x):
    // em = e^(x/2) - 1, sinh = em (em + 2) / (2 (em + 1)), cosh = ((em + 1) + 1/(em + 1)) / 2
    const double em = expm1(0.5 * z.x), ep = em + 1.0, iep = 1.0 / ep;
    sa = 0.5 * em * (em + 2.0) * iep;
    ca = 0.5 * (ep + iep);
    const double sr = sa * cb, si = ca * sb;   // sinh(z/2)
    return clog1p(make_double2(2.0 * (sr - si) * (sr + si), 4.0 * sr * si));
  }
  if (z.x < 0.0) z = make_double2(-z.x, -z.y);
  double2 u = cexp(make_double2(-2.0 * z.x, -2.0 * z.y));  // |u| <= e^-40
  const double2 l = clog1p(u);
  double re = z.x - 0.69314718055994530942 + l.x;
  double im = z.y + l.y;
  const double pi = 3.14159265358979323846, two_pi = 6.28318530717958647692;
  if (im > pi || im <= -pi) im -= two_pi * floor((im + pi) / two_pi);
  if (im <= -pi) im += two_pi;
  return make_double2(re, im);
}

// tanh(z) = d lncosh / dz.  |Re z| < 20: (sinh 2a + i sin 2b) / (cosh 2a + cos 2b) (accurate
// for small z); otherwise (1 - e^{-2z}) / (1 + e^{-2z}) for Re z >= 0 (tanh odd).
__device__ __forceinline__ double2 ctanh(double2 z) {
  if (fabs(z.x) < 20.0) {
    double s2b, c2b;
    sincos(2.0 * z.y, &s2b, &c2b);
    const double d = cosh(2.0 * z.x) + c2b;
    return make_double2(sinh(2.0 * z.x) / d, s2b / d);
  }
  const bool neg = z.x < 0.0;
  if (neg) z = make_double2(-z.x, -z.y);
  double2 u = cexp(make_double2(-2.0 * z.x, -2.0 * z.y));
  double2 t = cdiv(make_double2(1.0 - u.x, -u.y), make_double2(1.0 + u.x, u.y));
  return neg ? make_double2(-t.x, -t.y) : t;
}

// lncosh(z) and tanh(z) together (Jacobian forward pass): for |Re z| < 20 both come from one
// expm1 and one sincos of z/2 — tanh(z) = (sinh 2x + i sin 2y) / (cosh 2x + cos 2y) with the
// double angles built from sinh/cosh(x/2) and sin/cos(y/2) by products; otherwise the
// separate large-argument forms above.
__device__ __forceinline__ void lncosh_tanh(double2 z, double2& h, double2& t) {
  if (z.x * z.x + z.y * z.y <= kLncoshSeriesR2) {
    const double2 w = make_double2((z.x - z.y) * (z.x + z.y), 2.0 * z.x * z.y);
    h = lncosh_series(z, w);
    t = tanh_series(z, w);
    return;
  }
  if (fabs(z.x) >= 20.0) {
    h = lncosh(z);
    t = ctanh(z);
    return;
  }
  double sb, cb;
  sincos(0.5 * z.y, &sb, &cb);
  const double em = expm1(0.5 * z.x), ep = em + 1.0, iep = 1.0 / ep;
  const double sa = 0.5 * em * (em + 2.0) * iep, ca = 0.5 * (ep + iep);   // sinh, cosh of x/2
  const double sr = sa * cb, si = ca * sb;                                 // sinh(z/2)
  h = clog1p(make_double2(2.0 * (sr - si) * (sr + si), 4.0 * sr * si));
  const double shx = 2.0 * sa * ca, chx = 1.0 + 2.0 * sa * sa;            // sinh x, cosh x
  const double sy = 2.0 * sb * cb, cy = (cb - sb) * (cb + sb);             // sin y, cos y
  const double d = (1.0 + 2.0 * shx * shx) + (cy - sy) * (cy + sy);        // cosh 2x + cos 2y
  const double id = 1.0 / d;
  t = make_double2(2.0 * shx * chx * id, 2.0 * sy * cy * id);
}

__device__ __forceinline__ double2 ld2(const double* p) { return *reinterpret_cast<const double2*>(p); }
__device__ __forceinline__ void st2(double* p, double2 v) { *reinterpret_cast<double2*>(p) = v; }

}  // namespace sr
