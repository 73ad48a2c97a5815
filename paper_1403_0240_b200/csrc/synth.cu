// Device synthetic-data pipeline: render -> blur ->
// poissonize of the reference's rcseg/synth.py, bit-identical to it
// (tests/golden/synth.npz, made by the reference).  Replaces the per-pixel
// Python loop of poissonize (synth.py:179-181), which is prohibitive for the
// 512^3 and 2048^2 x 512 inputs.  Every kernel is one thread per output
// element; the arithmetic follows numpy/scipy's operation order with
// -fmad=false (no contractions), so the float64 results round identically.
#include <cmath>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "kernels.h"
#include "rcb.h"

namespace rcb {

// one shape, flattened on the host (synth.py:38-51):
// [kind, intensity, ncenter, c0, c1, c2, r2lo, r2hi, nbox, lo0, lo1, lo2, hi0, hi1, hi2]
static constexpr int kShapeWords = 15;

// synth.py:73-84: later shapes overwrite earlier ones.  Grid coordinates in
// dims order (2-D: y, x; 3-D: z, y, x); squared distances summed in that
// order over the centre's coordinates (numpy sum of a generator: 0 + t0 + t1 ...).
__global__ void k_render(int ndim, int64_t d0, int64_t d1, int64_t d2, double background,
                         const double *__restrict__ shp, int nshapes, int32_t *__restrict__ labels,
                         double *__restrict__ image) {
  const int64_t n = d0 * d1 * d2;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < n; f += stride) {
    double g[3];
    if (ndim == 3) {
      g[2] = (double)(f % d2);
      const int64_t t = f / d2;
      g[1] = (double)(t % d1);
      g[0] = (double)(t / d1);
    } else {
      g[1] = (double)(f % d1);
      g[0] = (double)(f / d1);
      g[2] = 0.0;
    }
    int32_t lab = 0;
    double val = background;
    for (int s = 0; s < nshapes; ++s) {
      const double *p = shp + kShapeWords * s;
      const int kind = (int)p[0];
      bool in;
      if (kind == 1) {  // rect / box: lo <= g < hi per axis (zip truncates)
        in = true;
        const int nb = (int)p[8];
        for (int a = 0; a < nb && a < ndim; ++a) in = in && g[a] >= p[9 + a] && g[a] < p[12 + a];
      } else {  // disk / ball (r2lo = -inf) and annulus / shell
        const int nc = (int)p[2];
        double d = 0.0;
        bool first = true;
        for (int a = 0; a < nc && a < ndim; ++a) {
          const double t = g[a] - p[3 + a];
          const double tt = t * t;
          d = first ? tt : d + tt;
          first = false;
        }
        in = d >= p[6] && d <= p[7];
      }
      if (in) {
        lab = s + 1;
        val = p[1];
      }
    }
    labels[f] = lab;
    image[f] = val;
  }
}

// scipy 'mirror' boundary (d c b | a b c d | c b a)
__device__ __forceinline__ int64_t mirror(int64_t i, int64_t n) {
  if (n == 1) return 0;
  const int64_t p = 2 * (n - 1);
  i %= p;
  if (i < 0) i += p;
  return i < n ? i : p - i;
}

// scipy.ndimage.correlate1d, symmetric-kernel path (synth.py:100-102):
// out[i] = x[i] k[r] + sum_{j = r..1} (x[i-j] + x[i+j]) k[r+j], in that order.
// The line along `axis` has length n and element stride `st`.
__global__ void k_blur_axis(const double *__restrict__ in, double *__restrict__ out, int64_t total,
                            int64_t n, int64_t st, const double *__restrict__ k, int r) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
    const int64_t i = (e / st) % n;
    const int64_t base = e - i * st;
    double acc = __ldg(&in[e]) * __ldg(&k[r]);
    for (int j = r; j >= 1; --j) {
      const double lft = __ldg(&in[base + mirror(i - j, n) * st]);
      const double rgt = __ldg(&in[base + mirror(i + j, n) * st]);
      acc = acc + (lft + rgt) * __ldg(&k[r + j]);
    }
    out[e] = acc;
  }
}

// min / max of a float64 array (the poissonize validation and peak)
__device__ __forceinline__ unsigned long long ord_key(double v) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(v);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double ord_val(unsigned long long k) {
  const unsigned long long u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)u);
}
__global__ void k_minmax(const double *__restrict__ x, int64_t n, unsigned long long *mm) {
  unsigned long long lo = ~0ull, hi = 0ull;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const unsigned long long k = ord_key(x[i]);
    lo = k < lo ? k : lo;
    hi = k > hi ? k : hi;
  }
  for (int s = 16; s; s >>= 1) {
    const unsigned long long a = __shfl_down_sync(0xffffffffu, lo, s);
    const unsigned long long b = __shfl_down_sync(0xffffffffu, hi, s);
    lo = a < lo ? a : lo;
    hi = b > hi ? b : hi;
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(mm, lo);
    atomicMax(mm + 1, hi);
  }
}

// splitmix64 (synth.py:106-130): per-pixel counter-based stream
__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
struct SplitMix {
  unsigned long long state;
  __device__ SplitMix(unsigned long long seed, unsigned long long index)
      : state(mix64(seed * 0x9E3779B97F4A7C15ull ^ mix64(index + 1))) {}
  __device__ double next_u01() {
    state += 0x9E3779B97F4A7C15ull;
    return (double)((mix64(state) >> 11) + 1) * 0x1p-53;
  }
};

// synth.py:133-166: CDF inversion below mean 30, Hormann's PTRS above
__device__ double poisson_draw(double lam, SplitMix &st) {
  if (lam <= 0.0) return 0.0;
  if (lam < 30.0) {
    const double u = st.next_u01();
    double p = exp(-lam);
    double cum = p;
    long long k = 0;
    const long long cap = (long long)(lam + 40.0 * sqrt(lam) + 100.0);
    while (u > cum && k < cap) {
      k += 1;
      p *= lam / (double)k;
      cum += p;
    }
    return (double)k;
  }
  const double smu = sqrt(lam);
  const double b = 0.931 + 2.53 * smu;
  const double a = -0.059 + 0.02483 * b;
  const double inv_alpha = 1.1239 + 1.1328 / (b - 3.4);
  const double v_r = 0.9277 - 3.6224 / (b - 2.0);
  const double log_lam = log(lam);
  for (;;) {
    const double u = st.next_u01() - 0.5;
    const double v = st.next_u01();
    const double us = 0.5 - fabs(u);
    const long long k = (long long)floor((2.0 * a / us + b) * u + lam + 0.43);
    if (us >= 0.07 && v <= v_r) return (double)k;
    if (k < 0 || (us < 0.013 && v > us)) continue;
    if (log(v) + log(inv_alpha) - log(a / (us * us) + b) <=
        (double)k * log_lam - lam - lgamma((double)k + 1.0))
      return (double)k;
  }
}

// synth.py:169-182: scale = psnr^2 / peak (peak from k_minmax), one draw per pixel
__global__ void k_poisson(const double *__restrict__ img, int64_t n, double psnr2,
                          unsigned long long seed, const unsigned long long *__restrict__ mm,
                          double *__restrict__ out) {
  const double peak = ord_val(mm[1]);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    if (!(peak > 0.0)) {
      out[i] = 0.0;
      continue;
    }
    const double scale = psnr2 / peak;
    SplitMix st(seed, (unsigned long long)i);
    out[i] = poisson_draw(img[i] * scale, st);
  }
}

static unsigned grid_ge(int64_t n) {
  int64_t g = (n + 255) / 256;
  if (g > 148 * 64) g = 148 * 64;
  return (unsigned)(g < 1 ? 1 : g);
}

// Device stages (all on stream s).
static int32_t synth_blur_dev(double *a, double *b, int ndim, const int64_t *dims,
                              const double *dk, int klen, cudaStream_t s, double **result) {
  // axes in order (synth.py:102); ping-pong between a and b
  const int r = (klen - 1) / 2;
  int64_t total = 1;
  for (int i = 0; i < ndim; ++i) total *= dims[i];
  double *src = a, *dst = b;
  for (int ax = 0; ax < ndim; ++ax) {
    int64_t st = 1;
    for (int i = ax + 1; i < ndim; ++i) st *= dims[i];
    k_blur_axis<<<grid_ge(total), 256, 0, s>>>(src, dst, total, dims[ax], st, dk, r);
    RCB_CUDA(cudaGetLastError());
    double *t = src;
    src = dst;
    dst = t;
  }
  *result = src;
  return RCB_OK;
}

static int32_t synth_poisson_dev(const double *img, int64_t n, double psnr2, uint64_t seed,
                                 unsigned long long *mm, double *out, cudaStream_t s,
                                 bool *negative) {
  const unsigned long long init[2] = {~0ull, 0ull};
  RCB_CUDA(cudaMemcpyAsync(mm, init, sizeof(init), cudaMemcpyHostToDevice, s));
  k_minmax<<<grid_ge(n), 256, 0, s>>>(img, n, mm);
  RCB_CUDA(cudaGetLastError());
  unsigned long long h[2];
  RCB_CUDA(cudaMemcpyAsync(h, mm, sizeof(h), cudaMemcpyDeviceToHost, s));
  RCB_CUDA(cudaStreamSynchronize(s));
  const unsigned long long u = (h[0] >> 63) ? (h[0] & 0x7fffffffffffffffull) : ~h[0];
  double lo;
  memcpy(&lo, &u, sizeof(lo));
  *negative = n > 0 && lo < 0.0;
  if (*negative) return RCB_OK;
  k_poisson<<<grid_ge(n), 256, 0, s>>>(img, n, psnr2, (unsigned long long)seed, mm, out);
  RCB_CUDA(cudaGetLastError());
  return RCB_OK;
}

}  // namespace rcb

using namespace rcb;

namespace {
struct SynthBufs {
  cudaStream_t s = nullptr;
  std::vector<void *> ptrs;
  ~SynthBufs() {
    for (void *p : ptrs) cudaFreeAsync(p, s);
    if (s) {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
  }
  template <typename T>
  int32_t alloc(T **p, size_t n) {
    if (cudaMallocAsync((void **)p, sizeof(T) * (n ? n : 1), s) != cudaSuccess)
      return fail(RCB_ERR_CUDA, "cudaMallocAsync failed");
    ptrs.push_back(*p);
    return RCB_OK;
  }
};
int32_t synth_dims(int32_t ndim, const int64_t *dims, int64_t *total) {
  if (ndim != 2 && ndim != 3) return fail(RCB_ERR_VALUE, "scene must be 2-D or 3-D");
  int64_t t = 1;
  for (int i = 0; i < ndim; ++i) {
    if (dims[i] < 1) return fail(RCB_ERR_VALUE, "dims must be positive");
    t *= dims[i];
  }
  *total = t;
  return RCB_OK;
}
}  // namespace

extern "C" {

int32_t rcb_synth_generate(int32_t ndim, const int64_t *dims, double background,
                           const double *shapes, int32_t nshapes, const double *kernel,
                           int32_t klen, int32_t noise, double psnr2, uint64_t seed,
                           int32_t *labels, double *clean, double *image) {
  int64_t n = 0;
  RCB_TRY(synth_dims(ndim, dims, &n));
  if (nshapes < 0 || (klen > 0 && klen % 2 == 0)) return fail(RCB_ERR_VALUE, "bad shapes/kernel");
  int dev = 0;
  RCB_CUDA(cudaGetDevice(&dev));
  SynthBufs B;
  RCB_CUDA(cudaStreamCreateWithFlags(&B.s, cudaStreamNonBlocking));
  cudaStream_t s = B.s;
  double *dsh = nullptr, *dk = nullptr, *a = nullptr, *b = nullptr;
  int32_t *dl = nullptr;
  unsigned long long *mm = nullptr;
  RCB_TRY(B.alloc(&dsh, (size_t)kShapeWords * nshapes));
  RCB_TRY(B.alloc(&dk, klen > 0 ? klen : 1));
  RCB_TRY(B.alloc(&a, n));
  RCB_TRY(B.alloc(&b, n));
  RCB_TRY(B.alloc(&dl, n));
  RCB_TRY(B.alloc(&mm, 2));
  if (nshapes)
    RCB_CUDA(cudaMemcpyAsync(dsh, shapes, sizeof(double) * kShapeWords * nshapes,
                             cudaMemcpyHostToDevice, s));
  if (klen > 0) RCB_CUDA(cudaMemcpyAsync(dk, kernel, sizeof(double) * klen, cudaMemcpyHostToDevice, s));
  const int64_t d0 = dims[0], d1 = dims[1], d2 = ndim == 3 ? dims[2] : 1;
  k_render<<<grid_ge(n), 256, 0, s>>>(ndim, d0, d1, d2, background, dsh, nshapes, dl, a);
  RCB_CUDA(cudaGetLastError());
  if (labels) RCB_CUDA(cudaMemcpyAsync(labels, dl, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s));
  if (clean) RCB_CUDA(cudaMemcpyAsync(clean, a, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
  double *cur = a;
  if (klen > 1) RCB_TRY(synth_blur_dev(a, b, ndim, dims, dk, klen, s, &cur));
  double *dst = cur == a ? b : a;
  if (noise) {
    bool neg = false;
    RCB_TRY(synth_poisson_dev(cur, n, psnr2, seed, mm, dst, s, &neg));
    if (neg) return fail(RCB_ERR_VALUE, "poissonize requires nonnegative intensities");
    cur = dst;
  }
  if (image) RCB_CUDA(cudaMemcpyAsync(image, cur, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
  RCB_CUDA(cudaStreamSynchronize(s));
  return RCB_OK;
}

int32_t rcb_synth_blur(const double *image, int32_t ndim, const int64_t *dims,
                       const double *kernel, int32_t klen, double *out) {
  int64_t n = 0;
  RCB_TRY(synth_dims(ndim, dims, &n));
  if (klen < 1 || klen % 2 == 0) return fail(RCB_ERR_VALUE, "kernel length must be odd");
  SynthBufs B;
  RCB_CUDA(cudaStreamCreateWithFlags(&B.s, cudaStreamNonBlocking));
  cudaStream_t s = B.s;
  double *dk = nullptr, *a = nullptr, *b = nullptr, *cur = nullptr;
  RCB_TRY(B.alloc(&dk, klen));
  RCB_TRY(B.alloc(&a, n));
  RCB_TRY(B.alloc(&b, n));
  RCB_CUDA(cudaMemcpyAsync(dk, kernel, sizeof(double) * klen, cudaMemcpyHostToDevice, s));
  RCB_CUDA(cudaMemcpyAsync(a, image, sizeof(double) * n, cudaMemcpyHostToDevice, s));
  RCB_TRY(synth_blur_dev(a, b, ndim, dims, dk, klen, s, &cur));
  RCB_CUDA(cudaMemcpyAsync(out, cur, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
  RCB_CUDA(cudaStreamSynchronize(s));
  return RCB_OK;
}

int32_t rcb_synth_poissonize(const double *image, int64_t n, double psnr2, uint64_t seed,
                             double *out) {
  if (n < 0) return fail(RCB_ERR_VALUE, "negative size");
  if (n == 0) return RCB_OK;
  SynthBufs B;
  RCB_CUDA(cudaStreamCreateWithFlags(&B.s, cudaStreamNonBlocking));
  cudaStream_t s = B.s;
  double *a = nullptr, *b = nullptr;
  unsigned long long *mm = nullptr;
  RCB_TRY(B.alloc(&a, n));
  RCB_TRY(B.alloc(&b, n));
  RCB_TRY(B.alloc(&mm, 2));
  RCB_CUDA(cudaMemcpyAsync(a, image, sizeof(double) * n, cudaMemcpyHostToDevice, s));
  bool neg = false;
  RCB_TRY(synth_poisson_dev(a, n, psnr2, seed, mm, b, s, &neg));
  if (neg) return fail(RCB_ERR_VALUE, "poissonize requires nonnegative intensities");
  RCB_CUDA(cudaMemcpyAsync(out, b, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
  RCB_CUDA(cudaStreamSynchronize(s));
  return RCB_OK;
}

}  // extern "C"
