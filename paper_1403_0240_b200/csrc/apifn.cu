// Function-level drop-ins of the reference's raster utilities that sit beside
// the hot path: connected components (grid.py:99-113), move
// admissibility (contour.py:171-207), the cell-list pair/point queries
// (sobolev.py:52-122), the ball convolution and dense per-label smooth fields
// (energy.py:161-223).  The engine never calls these; they exist so a caller
// of rcseg's module-level functions finds them on the device too.
#include <math.h>

#include <algorithm>
#include <string>
#include <vector>

#include <cub/cub.cuh>

#include "dev.cuh"
#include "kernels.h"

namespace rcb {
namespace {

// ---- connected components of one label (ndimage.label semantics) ----------
//
// Union-find over the sites with L == target (optionally minus one excluded
// site), linking the larger root under the smaller, so every component's
// root is its first site in raster order and numbering the roots by a scan
// reproduces ndimage.label's first-encounter order (grid.py:99-113).

__device__ __forceinline__ uint32_t uf_find(uint32_t *p, uint32_t x) {
  uint32_t r = p[x];
  while (r != x) {
    x = r;
    r = p[x];
  }
  return x;
}

__device__ __forceinline__ void uf_unite(uint32_t *p, uint32_t a, uint32_t b) {
  for (;;) {
    a = uf_find(p, a);
    b = uf_find(p, b);
    if (a == b) return;
    if (a < b) {
      uint32_t t = a;
      a = b;
      b = t;
    }
    uint32_t old = atomicCAS(&p[a], a, b);
    if (old == a) return;
    a = old;
  }
}

constexpr uint32_t kNone = 0xffffffffu;

__global__ void k_ccl_init(const int32_t *__restrict__ L, int64_t V, int32_t target,
                           int64_t exclude, uint32_t *__restrict__ p) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < V;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = (L[i] == target && i != exclude) ? (uint32_t)i : kNone;
}

// unite every member with its backward fg neighbours (half the box suffices)
__global__ void k_ccl_link(Lat lat, int full_fg, uint32_t *__restrict__ p) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < lat.V;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (p[i] == kNone) continue;
    int64_t z, y, x;
    lat.coord(i, z, y, x);
    const int zlo = lat.ndim == 3 ? -1 : 0;
    for (int dz = zlo; dz <= 0; ++dz)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          if (dz == 0 && (dy > 0 || (dy == 0 && dx >= 0))) continue;  // backward only
          int m = abs(dz) + abs(dy) + abs(dx);
          if (!full_fg && m != 1) continue;
          int64_t zz = z + dz, yy = y + dy, xx = x + dx;
          if (!lat.inb(zz, yy, xx)) continue;
          int64_t j = lat.flat(zz, yy, xx);
          if (p[j] == kNone) continue;
          uf_unite(p, (uint32_t)i, (uint32_t)j);
        }
  }
}

__global__ void k_ccl_flatten(int64_t V, uint32_t *__restrict__ p, uint32_t *__restrict__ root) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < V;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (p[i] == kNone) {
      root[i] = 0;
      continue;
    }
    uint32_t r = uf_find(p, (uint32_t)i);
    root[i] = (r == (uint32_t)i) ? 1u : 0u;
  }
}

__global__ void k_ccl_number(int64_t V, const uint32_t *__restrict__ p,
                             const uint32_t *__restrict__ ids, int32_t *__restrict__ comp) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < V;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (p[i] == kNone) {
      comp[i] = 0;
      continue;
    }
    uint32_t r = p[i];
    while (p[r] != r) r = p[r];
    comp[i] = (int32_t)ids[r] + 1;
  }
}

struct Ccl {
  DBuf<uint32_t> p, root, ids;
  DBuf<uint8_t> tmp;
  void release(cudaStream_t s) {
    p.release(s);
    root.release(s);
    ids.release(s);
    tmp.release(s);
  }
};

// components of (L == target) \ {exclude}; comp (device, nullable) receives
// 1..n per site (0 elsewhere); *n_out the count (synchronous).
int32_t ccl_run(const int32_t *dL, const Lat &lat, int full_fg, int32_t target, int64_t exclude,
                Ccl &c, int32_t *dcomp, int64_t *n_out, cudaStream_t s) {
  const int64_t V = lat.V;
  RCB_TRY(c.p.reserve(V, s));
  RCB_TRY(c.root.reserve(V + 1, s));
  RCB_TRY(c.ids.reserve(V + 1, s));
  const unsigned g = std::min<unsigned>(grid_for(V, 256), 148u * 16u);
  k_ccl_init<<<g, 256, 0, s>>>(dL, V, target, exclude, c.p.p);
  k_ccl_link<<<g, 256, 0, s>>>(lat, full_fg, c.p.p);
  k_ccl_flatten<<<g, 256, 0, s>>>(V, c.p.p, c.root.p);
  RCB_CUDA(cudaMemsetAsync(c.root.p + V, 0, sizeof(uint32_t), s));
  size_t bytes = 0;
  RCB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, c.root.p, c.ids.p, V + 1, s));
  RCB_TRY(c.tmp.reserve(bytes, s));
  RCB_CUDA(cub::DeviceScan::ExclusiveSum(c.tmp.p, bytes, c.root.p, c.ids.p, V + 1, s));
  if (dcomp) k_ccl_number<<<g, 256, 0, s>>>(V, c.p.p, c.ids.p, dcomp);
  RCB_CUDA(cudaGetLastError());
  uint32_t n = 0;
  RCB_CUDA(cudaMemcpyAsync(&n, c.ids.p + V, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  RCB_CUDA(cudaStreamSynchronize(s));
  *n_out = n;
  return RCB_OK;
}

// ---- admissibility: the local part of contour.py:171-207 ------------------
// out[i]: 0 = reject, 1 = accept, 2 = needs the global connectivity check
// (accept iff components((L == owner) \ {x}) == 1), before the fusion rule,
// which fus[i] carries (1 = fusion violation).
__global__ void k_admissible_local(const int32_t *__restrict__ L, Lat lat, int full_fg,
                                   const int64_t *__restrict__ xs, const int64_t *__restrict__ cs,
                                   const int64_t *__restrict__ counts, int64_t n,
                                   int allow_vanish, int32_t *__restrict__ out,
                                   int32_t *__restrict__ fus) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t xi = xs[i];
  const int32_t b = (int32_t)cs[i];
  const int32_t a = L[xi];
  int64_t z, y, x;
  lat.coord(xi, z, y, x);
  int v = 1;
  if (a == b) {
    v = 0;
  } else if (a > 0) {
    if (counts[i] == 1) {
      if (!allow_vanish) v = 0;
    } else if (local_component_count(L, lat, full_fg, z, y, x, a) != 1) {
      v = 2;
    }
  }
  int f = 0;
  if (b > 0) {  // fg-neighbour labels > 0 must be a or b (contour.py:203-206)
    const int zlo = lat.ndim == 3 ? -1 : 0, zhi = lat.ndim == 3 ? 1 : 0;
    for (int dz = zlo; dz <= zhi; ++dz)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          int m = abs(dz) + abs(dy) + abs(dx);
          if (m == 0 || (!full_fg && m != 1)) continue;
          int64_t zz = z + dz, yy = y + dy, xx = x + dx;
          if (!lat.inb(zz, yy, xx)) continue;
          int32_t l = L[lat.flat(zz, yy, xx)];
          if (l > 0 && l != a && l != b) f = 1;
        }
  }
  out[i] = v;
  fus[i] = f;
}

__global__ void k_label_hist(const int32_t *__restrict__ L, int64_t V, int32_t nl,
                             unsigned long long *__restrict__ h) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < V;
       i += (int64_t)gridDim.x * blockDim.x) {
    int32_t l = L[i];
    if (l >= 0 && l < nl) atomicAdd(&h[l], 1ull);
  }
}

// ---- cell list (sobolev.py:52-122) ------------------------------------------

// numpy floor_divide(int64, float64) -> float64 (CPython float floor division)
__device__ __forceinline__ double py_floordiv(double a, double b) {
  double mod = fmod(a, b);
  double div = (a - mod) / b;
  if (mod != 0.0 && ((b < 0) != (mod < 0))) div -= 1.0;
  double fl;
  if (div != 0.0) {
    fl = floor(div);
    if (div - fl > 0.5) fl += 1.0;
  } else {
    fl = copysign(0.0, a / b);
  }
  return fl;
}

__global__ void k_cells(const int64_t *__restrict__ coords, int64_t n, int ndim, double edge,
                        int64_t *__restrict__ cells) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n * ndim) return;
  cells[i] = (int64_t)py_floordiv((double)coords[i], edge);
}

// pass 0: count partners per p; pass 1: emit (p, q) in ascending q.
template <int PASS>
__global__ void __launch_bounds__(256) k_cell_pairs(const int64_t *__restrict__ coords,
                                                    const int64_t *__restrict__ cells, int64_t n,
                                                    int ndim, double c2,
                                                    unsigned long long *__restrict__ cnt,
                                                    const unsigned long long *__restrict__ off,
                                                    int64_t *__restrict__ pi,
                                                    int64_t *__restrict__ qi,
                                                    double *__restrict__ dist) {
  __shared__ int64_t sc[256 * 3], scell[256 * 3];
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t mc[3] = {0, 0, 0}, mcell[3] = {0, 0, 0};
  if (p < n)
    for (int k = 0; k < ndim; ++k) {
      mc[k] = coords[p * ndim + k];
      mcell[k] = cells[p * ndim + k];
    }
  unsigned long long c = 0, w = (PASS == 1 && p < n) ? off[p] : 0;
  for (int64_t t0 = 0; t0 < n; t0 += 256) {
    __syncthreads();
    const int64_t q = t0 + threadIdx.x;
    if (q < n)
      for (int k = 0; k < ndim; ++k) {
        sc[threadIdx.x * 3 + k] = coords[q * ndim + k];
        scell[threadIdx.x * 3 + k] = cells[q * ndim + k];
      }
    __syncthreads();
    if (p >= n) continue;
    const int m = (int)(n - t0 < 256 ? n - t0 : 256);
    for (int j = 0; j < m; ++j) {
      bool near = true;
      int64_t d2 = 0;
      for (int k = 0; k < ndim; ++k) {
        int64_t dc = scell[j * 3 + k] - mcell[k];
        if (dc < -1 || dc > 1) near = false;
        int64_t d = sc[j * 3 + k] - mc[k];
        d2 += d * d;
      }
      if (!near || !((double)d2 < c2)) continue;
      if (PASS == 0) {
        ++c;
      } else {
        pi[w] = p;
        qi[w] = t0 + j;
        dist[w] = sqrt((double)d2);
        ++w;
      }
    }
  }
  if (PASS == 0 && p < n) cnt[p] = c;
}

__global__ void k_cell_query(const int64_t *__restrict__ coords, const int64_t *__restrict__ cells,
                             int64_t n, int ndim, const double *__restrict__ point, double edge,
                             double c2, int64_t exclude, uint8_t *__restrict__ hit) {
  int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= n) return;
  bool near = true;
  double d2 = 0.0;
  for (int k = 0; k < ndim; ++k) {
    // sobolev.py:82-90: cell = floor(point / edge); d2 in float64
    int64_t pc = (int64_t)floor(point[k] / edge);
    int64_t dc = cells[q * ndim + k] - pc;
    if (dc < -1 || dc > 1) near = false;
    double d = (double)coords[q * ndim + k] - point[k];
    d2 = d2 + d * d;
  }
  hit[q] = (near && d2 < c2 && q != exclude) ? 1 : 0;
}

// ---- ball convolution (energy.py:161-193 _ball_spans / _ball_sum) -----------

struct Span {
  int dz, dy, h;  // transverse offset (dz, dy) and half-length along x
};

std::vector<Span> ball_spans(int ndim, int r) {
  // energy.py:146-158: transverse offsets in lexicographic order with
  // |t|^2 <= r^2, h = floor(sqrt(r^2 - |t|^2)).
  std::vector<Span> out;
  for (int dz = (ndim == 3 ? -r : 0); dz <= (ndim == 3 ? r : 0); ++dz)
    for (int dy = -r; dy <= r; ++dy) {
      int tt = dz * dz + dy * dy;
      if (tt > r * r) continue;
      out.push_back(Span{dz, dy, (int)floor(sqrt((double)(r * r - tt)))});
    }
  return out;
}

// q[row * (nx + 1) + j] = cumsum of the row's first j values (np.cumsum is a
// sequential fp64 sum); the window [z0,z1) x [y0,y1) x [x0,x1) of a field
// given by (labels == label) [* image].
__global__ void k_row_prefix(const double *__restrict__ field, const int32_t *__restrict__ L,
                             const double *__restrict__ I, int32_t label, Lat lat, int64_t z0,
                             int64_t y0, int64_t x0, int64_t wz, int64_t wy, int64_t wx,
                             double *__restrict__ q) {
  int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (row >= wz * wy) return;
  const int64_t z = z0 + row / wy, y = y0 + row % wy;
  double *qr = q + row * (wx + 1);
  double acc = 0.0;
  qr[0] = 0.0;
  for (int64_t j = 0; j < wx; ++j) {
    const int64_t f = lat.flat(z, y, x0 + j);
    double v;
    if (field) {
      v = field[f];
    } else {
      double m = (L[f] == label) ? 1.0 : 0.0;
      v = I ? m * I[f] : m;
    }
    acc = acc + v;
    qr[j + 1] = acc;
  }
}

__global__ void k_span_sum(const double *__restrict__ q, const Span *__restrict__ spans, int ns,
                           Lat lat, int64_t z0, int64_t y0, int64_t x0, int64_t wz, int64_t wy,
                           int64_t wx, double *__restrict__ out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= wz * wy * wx) return;
  const int64_t lx = i % wx, t = i / wx, ly = t % wy, lz = t / wy;
  double acc = 0.0;
  for (int k = 0; k < ns; ++k) {
    const Span sp = spans[k];
    // energy.py:180-191: a transverse offset at least the window extent is skipped
    if (abs(sp.dz) >= wz || abs(sp.dy) >= wy) continue;
    const int64_t sz = lz + sp.dz, sy = ly + sp.dy;
    if (sz < 0 || sz >= wz || sy < 0 || sy >= wy) continue;
    const int64_t hi = min(lx + sp.h, wx - 1) + 1, lo = max(lx - sp.h, (int64_t)0);
    const double *qr = q + (sz * wy + sy) * (wx + 1);
    acc = acc + (qr[hi] - qr[lo]);
  }
  out[lat.flat(z0 + lz, y0 + ly, x0 + lx)] = acc;
}

__global__ void k_label_boxes(const int32_t *__restrict__ L, Lat lat, int32_t nl,
                              int64_t *__restrict__ box) {  // [nl][6] lo z,y,x / hi z,y,x
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < lat.V;
       i += (int64_t)gridDim.x * blockDim.x) {
    int32_t l = L[i];
    if (l < 0 || l >= nl) continue;
    int64_t z, y, x;
    lat.coord(i, z, y, x);
    unsigned long long *b = (unsigned long long *)(box + 6 * l);
    atomicMin(&b[0], (unsigned long long)z);
    atomicMin(&b[1], (unsigned long long)y);
    atomicMin(&b[2], (unsigned long long)x);
    atomicMax(&b[3], (unsigned long long)z);
    atomicMax(&b[4], (unsigned long long)y);
    atomicMax(&b[5], (unsigned long long)x);
  }
}

struct Win {
  int64_t z0, y0, x0, wz, wy, wx;
};

int32_t ball_sum_window(const double *dfield, const int32_t *dL, const double *dI, int32_t label,
                        const Lat &lat, const Win &w, const Span *dspans, int ns,
                        DBuf<double> &q, double *dout, cudaStream_t s) {
  const int64_t rows = w.wz * w.wy;
  RCB_TRY(q.reserve(rows * (w.wx + 1), s));
  k_row_prefix<<<grid_for(rows, 128), 128, 0, s>>>(dfield, dL, dI, label, lat, w.z0, w.y0, w.x0,
                                                   w.wz, w.wy, w.wx, q.p);
  const int64_t cells = rows * w.wx;
  k_span_sum<<<grid_for(cells, 256), 256, 0, s>>>(q.p, dspans, ns, lat, w.z0, w.y0, w.x0, w.wz,
                                                  w.wy, w.wx, dout);
  RCB_CUDA(cudaGetLastError());
  return RCB_OK;
}

int32_t check_dev() {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    return fail(RCB_ERR_NODEVICE, std::string("no CUDA device: ") + cudaGetErrorString(e));
  return RCB_OK;
}

int32_t check_lat(int32_t ndim, const int64_t *dims) {
  if (ndim != 2 && ndim != 3) return fail(RCB_ERR_VALUE, "raster must be 2-D or 3-D");
  int64_t V = 1;
  for (int k = 0; k < ndim; ++k) {
    if (dims[k] < 1) return fail(RCB_ERR_VALUE, "raster dimensions must be positive");
    V *= dims[k];
  }
  if (V >= (int64_t)0xffffffffll) return fail(RCB_ERR_VALUE, "raster larger than 2^32-1 sites");
  return RCB_OK;
}

struct Stream {
  cudaStream_t s = nullptr;
  Stream() { cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking); }
  ~Stream() {
    if (s) {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
  }
};

template <typename T>
int32_t up(DBuf<T> &d, const T *h, size_t n, cudaStream_t s) {
  RCB_TRY(d.reserve(n ? n : 1, s));
  if (n) RCB_CUDA(cudaMemcpyAsync(d.p, h, n * sizeof(T), cudaMemcpyHostToDevice, s));
  return RCB_OK;
}

}  // namespace
}  // namespace rcb

using namespace rcb;

extern "C" {

int32_t rcb_label_components(const int32_t *labels, int32_t ndim, const int64_t *dims,
                             int32_t full_fg, int32_t target, int64_t exclude, int32_t *comp,
                             int64_t *n_components) {
  *n_components = 0;
  RCB_TRY(check_lat(ndim, dims));
  RCB_TRY(check_dev());
  Lat lat = make_lat(ndim, dims);
  Stream st;
  cudaStream_t s = st.s;
  DBuf<int32_t> dL, dc;
  Ccl c;
  int32_t rc = [&]() -> int32_t {
    RCB_TRY(up(dL, labels, lat.V, s));
    if (comp) RCB_TRY(dc.reserve(lat.V, s));
    RCB_TRY(ccl_run(dL.p, lat, full_fg, target, exclude, c, comp ? dc.p : nullptr,
                    n_components, s));
    if (comp) {
      RCB_CUDA(cudaMemcpyAsync(comp, dc.p, lat.V * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
      RCB_CUDA(cudaStreamSynchronize(s));
    }
    return RCB_OK;
  }();
  dL.release(s);
  dc.release(s);
  c.release(s);
  return rc;
}

int32_t rcb_moves_admissible(const int32_t *labels, int32_t ndim, const int64_t *dims,
                             int32_t full_fg, const int64_t *pixels, const int64_t *competitors,
                             const int64_t *region_counts, int64_t n, int32_t allow_fusion,
                             int32_t allow_vanish, int32_t *out) {
  RCB_TRY(check_lat(ndim, dims));
  if (n <= 0) return RCB_OK;
  RCB_TRY(check_dev());
  Lat lat = make_lat(ndim, dims);
  int32_t nl = 1;
  for (int64_t i = 0; i < lat.V; ++i) nl = std::max(nl, labels[i] + 1);
  std::vector<int64_t> counts(n);
  for (int64_t i = 0; i < n; ++i) {
    if (pixels[i] < 0 || pixels[i] >= lat.V) return fail(RCB_ERR_VALUE, "pixel out of range");
  }
  Stream st;
  cudaStream_t s = st.s;
  DBuf<int32_t> dL, dout, dfus;
  DBuf<int64_t> dx, dcs, dcnt;
  DBuf<unsigned long long> dh;
  Ccl c;
  int32_t rc = [&]() -> int32_t {
    RCB_TRY(up(dL, labels, lat.V, s));
    // region sizes: the caller's region_count where given (contour.py:189-191)
    std::vector<unsigned long long> hist(nl, 0);
    bool need_hist = region_counts == nullptr;
    for (int64_t i = 0; i < n && !need_hist; ++i)
      if (region_counts[i] < 0) need_hist = true;
    if (need_hist) {
      RCB_TRY(dh.reserve(nl, s));
      RCB_CUDA(cudaMemsetAsync(dh.p, 0, nl * sizeof(unsigned long long), s));
      k_label_hist<<<std::min<unsigned>(grid_for(lat.V, 256), 148u * 8u), 256, 0, s>>>(
          dL.p, lat.V, nl, dh.p);
      RCB_CUDA(cudaMemcpyAsync(hist.data(), dh.p, nl * sizeof(unsigned long long),
                               cudaMemcpyDeviceToHost, s));
      RCB_CUDA(cudaStreamSynchronize(s));
    }
    for (int64_t i = 0; i < n; ++i) {
      int32_t a = labels[pixels[i]];
      counts[i] = (region_counts && region_counts[i] >= 0) ? region_counts[i]
                                                           : (int64_t)hist[a];
    }
    RCB_TRY(up(dx, pixels, n, s));
    RCB_TRY(up(dcs, competitors, n, s));
    RCB_TRY(up(dcnt, counts.data(), n, s));
    RCB_TRY(dout.reserve(n, s));
    RCB_TRY(dfus.reserve(n, s));
    k_admissible_local<<<grid_for(n, 128), 128, 0, s>>>(dL.p, lat, full_fg, dx.p, dcs.p, dcnt.p,
                                                        n, allow_vanish, dout.p, dfus.p);
    std::vector<int32_t> fus(n);
    RCB_CUDA(cudaMemcpyAsync(out, dout.p, n * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    RCB_CUDA(cudaMemcpyAsync(fus.data(), dfus.p, n * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    RCB_CUDA(cudaStreamSynchronize(s));
    for (int64_t i = 0; i < n; ++i) {
      if (out[i] == 2) {  // contour.py:194-202: flood fill the donor minus the pixel
        int64_t k = 0;
        RCB_TRY(ccl_run(dL.p, lat, full_fg, labels[pixels[i]], pixels[i], c, nullptr, &k, s));
        out[i] = k == 1 ? 1 : 0;
      }
      if (out[i] == 1 && !allow_fusion && fus[i]) out[i] = 0;
    }
    return RCB_OK;
  }();
  dL.release(s);
  dout.release(s);
  dfus.release(s);
  dx.release(s);
  dcs.release(s);
  dcnt.release(s);
  dh.release(s);
  c.release(s);
  return rc;
}

int32_t rcb_cell_pairs(const int64_t *coords, int64_t n, int32_t ndim, double edge,
                       double cutoff, int64_t *pi, int64_t *qi, double *dist, int64_t cap,
                       int64_t *n_pairs) {
  *n_pairs = 0;
  if (ndim != 2 && ndim != 3) return fail(RCB_ERR_VALUE, "coords must be (n, 2) or (n, 3)");
  if (!(edge > 0)) return fail(RCB_ERR_VALUE, "bucket edge must be positive");
  if (n == 0) return RCB_OK;
  RCB_TRY(check_dev());
  Stream st;
  cudaStream_t s = st.s;
  DBuf<int64_t> dc, dcell, dpi, dqi;
  DBuf<double> dd;
  DBuf<unsigned long long> cnt, off;
  DBuf<uint8_t> tmp;
  int32_t rc = [&]() -> int32_t {
    RCB_TRY(up(dc, coords, (size_t)n * ndim, s));
    RCB_TRY(dcell.reserve((size_t)n * ndim, s));
    k_cells<<<grid_for(n * ndim, 256), 256, 0, s>>>(dc.p, n, ndim, edge, dcell.p);
    RCB_TRY(cnt.reserve(n + 1, s));
    RCB_TRY(off.reserve(n + 1, s));
    const double c2 = cutoff * cutoff;
    k_cell_pairs<0><<<grid_for(n, 256), 256, 0, s>>>(dc.p, dcell.p, n, ndim, c2, cnt.p, nullptr,
                                                     nullptr, nullptr, nullptr);
    RCB_CUDA(cudaMemsetAsync(cnt.p + n, 0, sizeof(unsigned long long), s));
    size_t bytes = 0;
    RCB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, cnt.p, off.p, n + 1, s));
    RCB_TRY(tmp.reserve(bytes, s));
    RCB_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, cnt.p, off.p, n + 1, s));
    unsigned long long tot = 0;
    RCB_CUDA(cudaMemcpyAsync(&tot, off.p + n, sizeof(tot), cudaMemcpyDeviceToHost, s));
    RCB_CUDA(cudaStreamSynchronize(s));
    *n_pairs = (int64_t)tot;
    if ((int64_t)tot > cap) return fail(RCB_ERR_CAPACITY, "pair buffer too small");
    if (tot == 0) return RCB_OK;
    RCB_TRY(dpi.reserve(tot, s));
    RCB_TRY(dqi.reserve(tot, s));
    RCB_TRY(dd.reserve(tot, s));
    k_cell_pairs<1><<<grid_for(n, 256), 256, 0, s>>>(dc.p, dcell.p, n, ndim, c2, nullptr, off.p,
                                                     dpi.p, dqi.p, dd.p);
    RCB_CUDA(cudaMemcpyAsync(pi, dpi.p, tot * 8, cudaMemcpyDeviceToHost, s));
    RCB_CUDA(cudaMemcpyAsync(qi, dqi.p, tot * 8, cudaMemcpyDeviceToHost, s));
    RCB_CUDA(cudaMemcpyAsync(dist, dd.p, tot * 8, cudaMemcpyDeviceToHost, s));
    RCB_CUDA(cudaStreamSynchronize(s));
    return RCB_OK;
  }();
  dc.release(s);
  dcell.release(s);
  dpi.release(s);
  dqi.release(s);
  dd.release(s);
  cnt.release(s);
  off.release(s);
  tmp.release(s);
  return rc;
}

int32_t rcb_cell_query(const int64_t *coords, int64_t n, int32_t ndim, double edge,
                       const double *point, double cutoff, int64_t exclude, int64_t *out,
                       int64_t *n_out) {
  *n_out = 0;
  if (ndim != 2 && ndim != 3) return fail(RCB_ERR_VALUE, "coords must be (n, 2) or (n, 3)");
  if (!(edge > 0)) return fail(RCB_ERR_VALUE, "bucket edge must be positive");
  if (n == 0) return RCB_OK;
  RCB_TRY(check_dev());
  Stream st;
  cudaStream_t s = st.s;
  DBuf<int64_t> dc, dcell;
  DBuf<double> dp;
  DBuf<uint8_t> hit;
  int32_t rc = [&]() -> int32_t {
    RCB_TRY(up(dc, coords, (size_t)n * ndim, s));
    RCB_TRY(up(dp, point, ndim, s));
    RCB_TRY(dcell.reserve((size_t)n * ndim, s));
    RCB_TRY(hit.reserve(n, s));
    k_cells<<<grid_for(n * ndim, 256), 256, 0, s>>>(dc.p, n, ndim, edge, dcell.p);
    k_cell_query<<<grid_for(n, 256), 256, 0, s>>>(dc.p, dcell.p, n, ndim, dp.p, edge,
                                                  cutoff * cutoff, exclude, hit.p);
    std::vector<uint8_t> h(n);
    RCB_CUDA(cudaMemcpyAsync(h.data(), hit.p, n, cudaMemcpyDeviceToHost, s));
    RCB_CUDA(cudaStreamSynchronize(s));
    int64_t k = 0;
    for (int64_t i = 0; i < n; ++i)
      if (h[i]) out[k++] = i;  // ascending (np.sort, sobolev.py:93)
    *n_out = k;
    return RCB_OK;
  }();
  dc.release(s);
  dcell.release(s);
  dp.release(s);
  hit.release(s);
  return rc;
}

int32_t rcb_ball_sum(const double *field, int32_t ndim, const int64_t *dims, int32_t radius,
                     double *out) {
  RCB_TRY(check_lat(ndim, dims));
  if (radius < 0) return fail(RCB_ERR_VALUE, "radius must be >= 0");
  RCB_TRY(check_dev());
  Lat lat = make_lat(ndim, dims);
  auto spans = ball_spans(ndim, radius);
  Stream st;
  cudaStream_t s = st.s;
  DBuf<double> df, dout, q;
  DBuf<Span> dsp;
  int32_t rc = [&]() -> int32_t {
    RCB_TRY(up(df, field, lat.V, s));
    RCB_TRY(up(dsp, spans.data(), spans.size(), s));
    RCB_TRY(dout.reserve(lat.V, s));
    Win w{0, 0, 0, lat.nz, lat.ny, lat.nx};
    RCB_TRY(ball_sum_window(df.p, nullptr, nullptr, 0, lat, w, dsp.p, (int)spans.size(), q,
                            dout.p, s));
    RCB_CUDA(cudaMemcpyAsync(out, dout.p, lat.V * 8, cudaMemcpyDeviceToHost, s));
    RCB_CUDA(cudaStreamSynchronize(s));
    return RCB_OK;
  }();
  df.release(s);
  dout.release(s);
  q.release(s);
  dsp.release(s);
  return rc;
}

int32_t rcb_smooth_fields(const int32_t *labels, const double *image, int32_t ndim,
                          const int64_t *dims, int32_t radius, int32_t n_labels, double *C,
                          double *S) {
  RCB_TRY(check_lat(ndim, dims));
  if (radius < 0) return fail(RCB_ERR_VALUE, "radius must be >= 0");
  if (n_labels < 1) return fail(RCB_ERR_VALUE, "n_labels must be >= 1");
  RCB_TRY(check_dev());
  Lat lat = make_lat(ndim, dims);
  auto spans = ball_spans(ndim, radius);
  Stream st;
  cudaStream_t s = st.s;
  DBuf<int32_t> dL;
  DBuf<double> dI, dC, dS, q;
  DBuf<Span> dsp;
  DBuf<int64_t> dbox;
  int32_t rc = [&]() -> int32_t {
    RCB_TRY(up(dL, labels, lat.V, s));
    RCB_TRY(up(dI, image, lat.V, s));
    RCB_TRY(up(dsp, spans.data(), spans.size(), s));
    RCB_TRY(dC.reserve(lat.V, s));
    RCB_TRY(dS.reserve(lat.V, s));
    // per-label bounding boxes (energy.py:207 find_objects)
    std::vector<int64_t> box(6 * (size_t)n_labels);
    for (int32_t l = 0; l < n_labels; ++l) {
      box[6 * l + 0] = box[6 * l + 1] = box[6 * l + 2] = INT64_MAX;
      box[6 * l + 3] = box[6 * l + 4] = box[6 * l + 5] = 0;
    }
    RCB_TRY(up(dbox, box.data(), box.size(), s));
    k_label_boxes<<<std::min<unsigned>(grid_for(lat.V, 256), 148u * 8u), 256, 0, s>>>(
        dL.p, lat, n_labels, dbox.p);
    RCB_CUDA(cudaMemcpyAsync(box.data(), dbox.p, box.size() * 8, cudaMemcpyDeviceToHost, s));
    RCB_CUDA(cudaStreamSynchronize(s));
    const int64_t V = lat.V;
    for (int32_t l = 0; l < n_labels; ++l) {
      double *Cl = C + (size_t)l * V, *Sl = S + (size_t)l * V;
      std::fill(Cl, Cl + V, 0.0);
      std::fill(Sl, Sl + V, 0.0);
      if (box[6 * l] == INT64_MAX) continue;  // label absent
      Win w;
      if (l == 0) {  // energy.py:211-214: label 0 uses the whole raster
        w = Win{0, 0, 0, lat.nz, lat.ny, lat.nx};
      } else {
        const int64_t n3[3] = {lat.nz, lat.ny, lat.nx};
        int64_t lo[3], hi[3];
        for (int k = 0; k < 3; ++k) {
          const bool live = (ndim == 3) || k > 0;
          const int64_t r = live ? radius : 0;
          lo[k] = std::max<int64_t>(0, box[6 * l + k] - r);
          hi[k] = std::min<int64_t>(n3[k], box[6 * l + 3 + k] + 1 + r);
        }
        w = Win{lo[0], lo[1], lo[2], hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]};
      }
      RCB_CUDA(cudaMemsetAsync(dC.p, 0, V * 8, s));
      RCB_CUDA(cudaMemsetAsync(dS.p, 0, V * 8, s));
      RCB_TRY(ball_sum_window(nullptr, dL.p, nullptr, l, lat, w, dsp.p, (int)spans.size(), q,
                              dC.p, s));
      RCB_TRY(ball_sum_window(nullptr, dL.p, dI.p, l, lat, w, dsp.p, (int)spans.size(), q,
                              dS.p, s));
      RCB_CUDA(cudaMemcpyAsync(Cl, dC.p, V * 8, cudaMemcpyDeviceToHost, s));
      RCB_CUDA(cudaMemcpyAsync(Sl, dS.p, V * 8, cudaMemcpyDeviceToHost, s));
      RCB_CUDA(cudaStreamSynchronize(s));
    }
    return RCB_OK;
  }();
  dL.release(s);
  dI.release(s);
  dC.release(s);
  dS.release(s);
  q.release(s);
  dsp.release(s);
  dbox.release(s);
  return rc;
}

}  // extern "C"
