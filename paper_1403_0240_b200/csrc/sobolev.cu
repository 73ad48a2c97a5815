// K6 — the Sobolev particle-particle interaction (Eq. 6) as a masked lattice
// stencil over the contour set (replaces sobolev.py:137-174 sobolev_filter,
// :52-134 CellList/pairs and the per-pair kernel_eval).
//
// Particles are kept sorted by (site, competitor) with the CSR lattice index
// site_off, so for particle p the partners q with |x_q - x_p|^2 < (E/2)^2 are
// the particles of the stencil sites x_p + o.  Visiting the stencil offsets in
// lexicographic order and each site's particles in competitor order is the
// reference's canonical pair order (flat q, comp q, index q) (sobolev.py:
// 155-161), and the weight of a pair is the host table
// w[|o|^2] = kernel_eval(sqrt(|o|^2)), so the fp64 sums are bit-identical.
#include <cstring>
#include <cstdlib>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>

#include "dev.cuh"
#include "kernels.h"

namespace rcb {

// Interaction count: one atomic per block (a same-address atomic per warp
// cost more than the w = 1 kernel's whole memory pass at 10^7 particles).
__device__ __forceinline__ void block_add_pairs(unsigned long long np,
                                                unsigned long long *pairs) {
  __shared__ unsigned long long red[32];
  for (int sh = 16; sh; sh >>= 1) np += __shfl_down_sync(0xffffffffu, np, sh);
  const int w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  if ((threadIdx.x & 31) == 0) red[w] = np;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int k = 0; k < nw; ++k) t += red[k];
    if (t) atomicAdd(pairs, t);
  }
}


// One thread per particle p.  The stencil {o : |o|^2 < (E/2)^2} is walked row
// by row: for each (dz, dy) in lexicographic order the partners are the
// particles of the contiguous site range [x - h, x + h] of that lattice row,
// fetched with two CSR lookups and visited in site order, each site's
// particles in competitor order — exactly the canonical pair order
// (flat q, comp q, index q) of sobolev.py:155-161.  The pair weight is the
// host table entry w[dz^2 + dy^2 + dx^2].
// oidx != nullptr: write the result of sorted particle p to out[oidx[p]].
__global__ void __launch_bounds__(128) k_sobolev(
    const uint32_t *__restrict__ site_off, const int32_t *__restrict__ qown,
    const int32_t *__restrict__ pcomp, const uint32_t *__restrict__ px,
    const double *__restrict__ raw, Lat lat, const Off *__restrict__ rows, int nrows,
    const double *__restrict__ wt, int64_t n, double *__restrict__ out,
    const uint32_t *__restrict__ oidx, unsigned long long *__restrict__ pairs, int64_t p0 = 0) {
  int64_t p = p0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long np = 0;
  if (p < n) {
    const int64_t f = px[p];
    const int32_t own = __ldg(&qown[p]);
    int64_t z, y, x;
    lat.coord(f, z, y, x);
    double same = 0.0, opp = 0.0;
    int cs = 0, co = 0;
    for (int k = 0; k < nrows; ++k) {
      const Off r = rows[k];
      const int64_t zz = z + r.dz, yy = y + r.dy;
      if (zz < 0 || zz >= lat.nz || yy < 0 || yy >= lat.ny) continue;
      const int64_t x0 = x - r.dx < 0 ? 0 : x - r.dx;
      const int64_t x1 = x + r.dx >= lat.nx ? lat.nx - 1 : x + r.dx;
      const int64_t rb = lat.flat(zz, yy, 0);
      const uint32_t q0 = __ldg(&site_off[rb + x0]), q1 = __ldg(&site_off[rb + x1 + 1]);
      np += q1 - q0;
      const int64_t centre = rb + x;
      for (uint32_t q = q0; q < q1; ++q) {
        const int dx = (int)((int64_t)__ldg(&px[q]) - centre);
        const double c = __ldg(&wt[(int)r.aux + dx * dx]) * __ldg(&raw[q]);
        if (__ldg(&qown[q]) == own) {
          same += c;
          ++cs;
        }
        if (__ldg(&pcomp[q]) == own) {
          opp += c;
          ++co;
        }
      }
    }
    const double a = cs > 0 ? same / (double)cs : 0.0;
    const double b = co > 0 ? opp / (double)co : 0.0;
    out[oidx ? oidx[p] : p] = a - b;
  }
  if (pairs) block_add_pairs(np, pairs);
}

// fp32 variant of K6 (fp32 mode): float increments, weights and sums.
__global__ void __launch_bounds__(128) k_sobolev32(
    const uint32_t *__restrict__ site_off, const int32_t *__restrict__ qown,
    const int32_t *__restrict__ pcomp, const uint32_t *__restrict__ px,
    const float *__restrict__ raw, Lat lat, const Off *__restrict__ rows, int nrows,
    const float *__restrict__ wt, int64_t n, double *__restrict__ out,
    unsigned long long *__restrict__ pairs, int64_t p0 = 0) {
  int64_t p = p0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long np = 0;
  if (p < n) {
    const int64_t f = px[p];
    const int32_t own = __ldg(&qown[p]);
    int64_t z, y, x;
    lat.coord(f, z, y, x);
    float same = 0.f, opp = 0.f;
    int cs = 0, co = 0;
    for (int k = 0; k < nrows; ++k) {
      const Off r = rows[k];
      const int64_t zz = z + r.dz, yy = y + r.dy;
      if (zz < 0 || zz >= lat.nz || yy < 0 || yy >= lat.ny) continue;
      const int64_t x0 = x - r.dx < 0 ? 0 : x - r.dx;
      const int64_t x1 = x + r.dx >= lat.nx ? lat.nx - 1 : x + r.dx;
      const int64_t rb = lat.flat(zz, yy, 0);
      const uint32_t q0 = __ldg(&site_off[rb + x0]), q1 = __ldg(&site_off[rb + x1 + 1]);
      np += q1 - q0;
      const int64_t centre = rb + x;
      for (uint32_t q = q0; q < q1; ++q) {
        const int dx = (int)((int64_t)__ldg(&px[q]) - centre);
        const float c = __ldg(&wt[(int)r.aux + dx * dx]) * __ldg(&raw[q]);
        if (__ldg(&qown[q]) == own) {
          same += c;
          ++cs;
        }
        if (__ldg(&pcomp[q]) == own) {
          opp += c;
          ++co;
        }
      }
    }
    const float a = cs > 0 ? same / (float)cs : 0.f;
    const float b = co > 0 ? opp / (float)co : 0.f;
    out[p] = (double)(a - b);
  }
  if (pairs) block_add_pairs(np, pairs);
}

int32_t sobolev_lattice32(const uint32_t *site_off, const int32_t *pown, const uint32_t *px,
                          const int32_t *pcomp, const float *raw, const Lat &lat, const Off *rows,
                          int nrows, const float *wt, int64_t n, double *out,
                          unsigned long long *pairs, cudaStream_t s, int64_t p0) {
  if (n <= p0) return RCB_OK;
  k_sobolev32<<<grid_for(n - p0, 128), 128, 0, s>>>(site_off, pown, pcomp, px, raw, lat, rows,
                                                    nrows, wt, n, out, pairs, p0);
  RCB_CUDA(cudaGetLastError());
  return RCB_OK;
}

// ---- K6 on packed particle records (engine and sweep) ----------------------
// One 16-byte record per particle {raw (fp64), site, owner | competitor << 16}
// (labels < 2^16): a partner costs one vector load instead of four scalar
// ones.  Coordinates and CSR indices are 32-bit (sites < 2^32), the stencil
// rows and the weight table sit in shared memory, and each row's partners are
// fetched kSobU records at a time before any is used.  The products and the
// two sums are formed exactly as in k_sobolev, in the same canonical order,
// so the results are bit-identical.
static constexpr int kSobRows = 1024, kSobW = 256, kSobU = 4;

__global__ void k_sob_pack(const uint32_t *__restrict__ px, const int32_t *__restrict__ pown,
                           const int32_t *__restrict__ pcomp, const double *__restrict__ raw,
                           int64_t lo, int64_t hi, int4 *__restrict__ pk) {
  const int64_t i = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= hi) return;
  const unsigned long long u = (unsigned long long)__double_as_longlong(raw[i]);
  pk[i] = make_int4((int)(uint32_t)u, (int)(uint32_t)(u >> 32), (int)px[i],
                    (int)((uint32_t)pown[i] | ((uint32_t)pcomp[i] << 16)));
}

__global__ void __launch_bounds__(128) k_sobolev_pk(
    const uint32_t *__restrict__ site_off, const int4 *__restrict__ pk, uint32_t nx, uint32_t ny,
    uint32_t nz, const Off *__restrict__ rows, int nrows, const double *__restrict__ wt, int nwt,
    int64_t p0, int64_t p1, double *__restrict__ out, unsigned long long *__restrict__ pairs) {
  __shared__ int srow[kSobRows];  // dz:8 | dy:8 | h:8 | aux:8
  __shared__ double sw[kSobW];
  for (int k = threadIdx.x; k < nrows; k += blockDim.x) {
    const Off r = rows[k];
    srow[k] = ((int)(uint8_t)r.dz << 24) | ((int)(uint8_t)r.dy << 16) | ((int)(uint8_t)r.dx << 8) |
              (int)r.aux;
  }
  for (int k = threadIdx.x; k < nwt; k += blockDim.x) sw[k] = wt[k];
  __syncthreads();
  const int64_t p = p0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long np = 0;
  if (p < p1) {
    const int4 me = pk[p];
    const uint32_t f = (uint32_t)me.z, own = (uint32_t)me.w & 0xffffu;
    const uint32_t plane = nx * ny;
    const uint32_t z = f / plane, rem = f - z * plane;
    const uint32_t y = rem / nx, x = rem - y * nx;
    double same = 0.0, opp = 0.0;
    int cs = 0, co = 0;
    for (int k = 0; k < nrows; ++k) {
      const int r = srow[k];
      const int zz = (int)z + (int)(int8_t)(r >> 24), yy = (int)y + (int)(int8_t)(r >> 16);
      if ((unsigned)zz >= nz || (unsigned)yy >= ny) continue;
      const int h = (r >> 8) & 0xff, aux = r & 0xff;
      const uint32_t x0 = (int)x - h < 0 ? 0u : x - h;
      const uint32_t x1 = x + h >= nx ? nx - 1 : x + h;
      const uint32_t rb = ((uint32_t)zz * ny + (uint32_t)yy) * nx;
      const uint32_t q0 = __ldg(&site_off[rb + x0]), q1 = __ldg(&site_off[rb + x1 + 1]);
      np += q1 - q0;
      const uint32_t centre = rb + x;
      for (uint32_t q = q0; q < q1; q += kSobU) {
        int4 v[kSobU];
#pragma unroll
        for (int u = 0; u < kSobU; ++u)
          v[u] = q + u < q1 ? __ldg(&pk[q + u]) : make_int4(0, 0, (int)centre, -1);
#pragma unroll
        for (int u = 0; u < kSobU; ++u) {
          if (q + u >= q1) break;
          const int dx = (int)((uint32_t)v[u].z - centre);
          const double rq = __longlong_as_double(((long long)(uint32_t)v[u].y << 32) |
                                                 (long long)(uint32_t)v[u].x);
          const double c = sw[aux + dx * dx] * rq;
          const uint32_t oc = (uint32_t)v[u].w;
          if ((oc & 0xffffu) == own) {
            same += c;
            ++cs;
          }
          if ((oc >> 16) == own) {
            opp += c;
            ++co;
          }
        }
      }
    }
    const double a = cs > 0 ? same / (double)cs : 0.0;
    const double b = co > 0 ? opp / (double)co : 0.0;
    out[p] = a - b;
  }
  if (pairs) block_add_pairs(np, pairs);
}

// ---- K6 at w = 1 (E <= 2): the stencil is the particle's own site ----------
// The partners of p are the particles of its own site: the run of equal px
// around p in the (site, competitor)-sorted list, at most 26 long.  A pure
// streaming pass -- px, owner, competitor, raw in and out, 28 B per particle
// -- with the run's few neighbours read from L1.  The sums
// follow the same canonical order (index order within the site) and the same
// expressions as k_sobolev, so the results are bit-identical.
// General run sum (any owners/competitors): the partners of p are the
// particles of its own site, the run of equal px around p.
__device__ __forceinline__ double site_run_value(const uint32_t *__restrict__ px,
                                                 const int32_t *__restrict__ pown,
                                                 const int32_t *__restrict__ pcomp,
                                                 const double *__restrict__ raw, double w0,
                                                 int64_t p, int64_t lo, int64_t hi, int64_t &len) {
  const uint32_t f = __ldg(&px[p]);
  const int32_t own = __ldg(&pown[p]);
  int64_t s = p, e = p + 1;
  while (s > lo && __ldg(&px[s - 1]) == f) --s;
  while (e < hi && __ldg(&px[e]) == f) ++e;
  double same = 0.0, opp = 0.0;
  int cs = 0, co = 0;
  for (int64_t q = s; q < e; ++q) {
    const double c = w0 * __ldg(&raw[q]);
    if (__ldg(&pown[q]) == own) {
      same += c;
      ++cs;
    }
    if (__ldg(&pcomp[q]) == own) {
      opp += c;
      ++co;
    }
  }
  len = e - s;
  const double a = cs > 0 ? same / (double)cs : 0.0;
  const double b = co > 0 ? opp / (double)co : 0.0;
  return a - b;
}

// Warp-cooperative pass: each warp streams 32 consecutive particles with
// coalesced loads; runs of equal px that lie inside the warp, share one owner
// and hold no competitor equal to it (every run of an engine or sweep
// particle list: competitors differ from the site's own label) are summed by
// a ripple of shuffles -- acc(lane) = acc(lane - 1) + c(lane), from 0.0 at
// the run head, i.e. the canonical sequential order -- and every lane of the
// run takes the run total; other runs (crossing a warp edge, mixed owners)
// take site_run_value.  Bit-identical to k_sobolev.
static constexpr int kRipple = 8, kSiteChunks = 8;
__global__ void __launch_bounds__(256) k_sobolev_site(
    const uint32_t *__restrict__ px, const int32_t *__restrict__ pown,
    const int32_t *__restrict__ pcomp, const double *__restrict__ raw, double w0, int64_t p0,
    int64_t p1, int64_t lo, int64_t hi, double *__restrict__ out,
    unsigned long long *__restrict__ pairs) {
  const int lane = threadIdx.x & 31;
  // each warp streams kSiteChunks consecutive chunks of 32 particles, all
  // their loads in flight before the first is used (bytes in flight per SM
  // are what an HBM-bound pass needs)
  const int64_t wbase = p0 + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * (32 * kSiteChunks);
  uint32_t fv[kSiteChunks];
  int32_t ov[kSiteChunks], cv[kSiteChunks];
  double rv[kSiteChunks];
#pragma unroll
  for (int j = 0; j < kSiteChunks; ++j) {
    const int64_t p = wbase + 32 * j + lane;
    const bool in = p < p1;
    fv[j] = in ? __ldg(&px[p]) : 0xffffffffu - (uint32_t)lane;  // distinct sentinels
    ov[j] = in ? __ldg(&pown[p]) : -1;
    cv[j] = in ? __ldg(&pcomp[p]) : -2;
    rv[j] = in ? __ldg(&raw[p]) : 0.0;
  }
  unsigned long long np = 0;
#pragma unroll
  for (int j = 0; j < kSiteChunks; ++j) {
    const int64_t p = wbase + 32 * j + lane;
    const bool in = p < p1;
    const uint32_t f = fv[j];
    const int32_t own = ov[j], cmp = cv[j];
    const double c = w0 * rv[j];
    const uint32_t fu = __shfl_up_sync(0xffffffffu, f, 1), fd = __shfl_down_sync(0xffffffffu, f, 1);
    const int32_t ou = __shfl_up_sync(0xffffffffu, own, 1);
    const bool head = lane == 0 || fu != f;
    const bool tail = lane == 31 || fd != f;
    // a run is summed here if it lies inside the chunk, has one owner and
    // no competitor equal to it; otherwise site_run_value
    const bool edge = (lane == 0 && in && p > lo && __ldg(&px[p - 1]) == f) ||
                      (lane == 31 && in && p + 1 < hi && __ldg(&px[p + 1]) == f);
    const bool bad = edge || (!head && ou != own) || (cmp == own);
    const unsigned hm = __ballot_sync(0xffffffffu, head);
    const int hl = 31 - __clz(hm & (0xffffffffu >> (31 - lane)));  // highest head lane <= lane
    const unsigned tm = __ballot_sync(0xffffffffu, tail);
    const int tl = __ffs(tm & (0xffffffffu << lane)) - 1;           // lowest tail lane >= lane
    const unsigned bm = __ballot_sync(0xffffffffu, bad);
    const unsigned runmask =
        (tl == 31 ? 0xffffffffu : ((1u << (tl + 1)) - 1u)) & (0xffffffffu << hl);
    const int len = tl - hl + 1;
    const bool simple = in && !(bm & runmask) && len <= kRipple;
    // ripple: at step k the lane k places after its run head adds its term to
    // its left neighbour's (already final) partial sum -- sequential order
    double acc = 0.0 + c;
    // as many ripple steps as the chunk's longest simple run needs (none when
    // every site holds one particle)
    const int steps = (int)__reduce_max_sync(0xffffffffu, simple ? (unsigned)len : 1u);
    for (int k = 1; k < steps; ++k) {
      const double up = __shfl_up_sync(0xffffffffu, acc, 1);
      if (lane - hl == k) acc = up + c;
    }
    const double total = __shfl_sync(0xffffffffu, acc, tl);
    if (in) {
      if (simple) {
        out[p] = len == 1 ? total : total / (double)len - 0.0;  // x / 1.0 - 0.0 == x: no fp64 division on single-particle sites
        np += (unsigned long long)len;
      } else {
        int64_t L = 0;
        out[p] = site_run_value(px, pown, pcomp, raw, w0, p, lo, hi, L);
        np += (unsigned long long)L;
      }
    }
  }
  if (pairs) block_add_pairs(np, pairs);
}

// The w = 1 site kernel over K6's packed records (written by the energy
// kernels, or once by the sweep's generator): one 16-byte record per
// particle in, one 8-byte result out.
__device__ __forceinline__ double pk_raw(const int4 v) {
  return __longlong_as_double(((long long)(uint32_t)v.y << 32) | (long long)(uint32_t)v.x);
}

__device__ __forceinline__ double site_run_value_pk(const int4 *__restrict__ pk, double w0,
                                                    int64_t p, int64_t lo, int64_t hi,
                                                    int64_t &len) {
  const int4 me = __ldg(&pk[p]);
  const uint32_t f = (uint32_t)me.z;
  const uint32_t own = (uint32_t)me.w & 0xffffu;
  int64_t s = p, e = p + 1;
  while (s > lo && (uint32_t)__ldg(&pk[s - 1]).z == f) --s;
  while (e < hi && (uint32_t)__ldg(&pk[e]).z == f) ++e;
  double same = 0.0, opp = 0.0;
  int cs = 0, co = 0;
  for (int64_t q = s; q < e; ++q) {
    const int4 r = __ldg(&pk[q]);
    const double c = w0 * pk_raw(r);
    if (((uint32_t)r.w & 0xffffu) == own) {
      same += c;
      ++cs;
    }
    if (((uint32_t)r.w >> 16) == own) {
      opp += c;
      ++co;
    }
  }
  len = e - s;
  const double a = cs > 0 ? same / (double)cs : 0.0;
  const double b = co > 0 ? opp / (double)co : 0.0;
  return a - b;
}

template <bool CS>  // CS: streaming (evict-first) loads and stores -- the pass reuses nothing
__global__ void __launch_bounds__(256) k_sobolev_site_pk(const int4 *__restrict__ pk, double w0,
                                                         int64_t p0, int64_t p1, int64_t lo,
                                                         int64_t hi, double *__restrict__ out,
                                                         unsigned long long *__restrict__ pairs) {
  const int lane = threadIdx.x & 31;
  const int64_t wbase = p0 + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * (32 * kSiteChunks);
  int4 rv[kSiteChunks];
#pragma unroll
  for (int j = 0; j < kSiteChunks; ++j) {
    const int64_t p = wbase + 32 * j + lane;
    rv[j] = p < p1 ? (CS ? __ldcs(&pk[p]) : __ldg(&pk[p]))
                   : make_int4(0, 0, (int)(0xffffffffu - (uint32_t)lane), -1);
  }
  unsigned long long np = 0;
#pragma unroll
  for (int j = 0; j < kSiteChunks; ++j) {
    const int64_t p = wbase + 32 * j + lane;
    const bool in = p < p1;
    const uint32_t f = (uint32_t)rv[j].z;
    const int32_t own = in ? (int32_t)((uint32_t)rv[j].w & 0xffffu) : -1;
    const int32_t cmp = in ? (int32_t)((uint32_t)rv[j].w >> 16) : -2;
    const double c = in ? w0 * pk_raw(rv[j]) : 0.0;
    const uint32_t fu = __shfl_up_sync(0xffffffffu, f, 1), fd = __shfl_down_sync(0xffffffffu, f, 1);
    const int32_t ou = __shfl_up_sync(0xffffffffu, own, 1);
    const bool head = lane == 0 || fu != f;
    const bool tail = lane == 31 || fd != f;
    const bool edge = (lane == 0 && in && p > lo && (uint32_t)__ldg(&pk[p - 1]).z == f) ||
                      (lane == 31 && in && p + 1 < hi && (uint32_t)__ldg(&pk[p + 1]).z == f);
    const bool bad = edge || (!head && ou != own) || (cmp == own);
    const unsigned hm = __ballot_sync(0xffffffffu, head);
    const int hl = 31 - __clz(hm & (0xffffffffu >> (31 - lane)));
    const unsigned tm = __ballot_sync(0xffffffffu, tail);
    const int tl = __ffs(tm & (0xffffffffu << lane)) - 1;
    const unsigned bm = __ballot_sync(0xffffffffu, bad);
    const unsigned runmask =
        (tl == 31 ? 0xffffffffu : ((1u << (tl + 1)) - 1u)) & (0xffffffffu << hl);
    const int len = tl - hl + 1;
    const bool simple = in && !(bm & runmask) && len <= kRipple;
    double acc = 0.0 + c;
    // as many ripple steps as the chunk's longest simple run needs (none when
    // every site holds one particle)
    const int steps = (int)__reduce_max_sync(0xffffffffu, simple ? (unsigned)len : 1u);
    for (int k = 1; k < steps; ++k) {
      const double up = __shfl_up_sync(0xffffffffu, acc, 1);
      if (lane - hl == k) acc = up + c;
    }
    const double total = __shfl_sync(0xffffffffu, acc, tl);
    if (in) {
      if (simple) {
        // x / 1.0 - 0.0 == x: no fp64 division on single-particle sites
        const double r = len == 1 ? total : total / (double)len - 0.0;
        if (CS)
          __stcs(out + p, r);
        else
          out[p] = r;
        np += (unsigned long long)len;
      } else {
        int64_t L = 0;
        out[p] = site_run_value_pk(pk, w0, p, lo, hi, L);
        np += (unsigned long long)L;
      }
    }
  }
  if (pairs) block_add_pairs(np, pairs);
}

// The same pass with the records staged by the Tensor Memory Accelerator: a
// persistent grid (2 blocks per SM) streams 1024-record tiles (16 KB) through
// a 4-stage shared-memory ring with 1-D bulk copies (cp.async.bulk, mbarrier
// completion), so each SM keeps ~64 KB of loads in flight without holding
// them in registers; warps then run the site-run logic on shared memory.
static constexpr int kBulkTile = 1024, kBulkStages = 4;

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
}
__device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes,
                                          uint64_t *bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

__global__ void __launch_bounds__(256) k_sobolev_site_bulk(const int4 *__restrict__ pk, double w0,
                                                           int64_t n, double *__restrict__ out,
                                                           unsigned long long *__restrict__ pairs) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  int4 *buf = reinterpret_cast<int4 *>(smem_raw);
  __shared__ __align__(8) uint64_t bar[kBulkStages];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t ntiles = (n + kBulkTile - 1) / kBulkTile;
  if (threadIdx.x == 0) {
    for (int st = 0; st < kBulkStages; ++st) mbar_init(&bar[st]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int64_t tile, int st) {
    const int64_t b = tile * kBulkTile;
    const int64_t cnt = n - b < kBulkTile ? n - b : kBulkTile;
    bulk_load(buf + st * kBulkTile, pk + b, (uint32_t)(cnt * sizeof(int4)), &bar[st]);
  };
  // prologue: the first tiles of this block
  if (threadIdx.x == 0)
    for (int st = 0; st < kBulkStages; ++st) {
      const int64_t t = blockIdx.x + (int64_t)st * gridDim.x;
      if (t < ntiles) issue(t, st);
    }
  unsigned long long np = 0;
  int64_t k = 0;  // local tile counter
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
    const int st = (int)(k % kBulkStages);
    const uint32_t phase = (uint32_t)((k / kBulkStages) & 1);
    mbar_wait(&bar[st], phase);
    const int4 *tb = buf + st * kBulkTile;
    const int64_t base = t * kBulkTile;
    const int64_t cnt = n - base < kBulkTile ? n - base : kBulkTile;
#pragma unroll
    for (int j = 0; j < kBulkTile / 256; ++j) {
      const int li = warp * (kBulkTile / 8) + j * 32 + lane;  // record in the tile
      const int64_t p = base + li;
      const bool in = li < cnt;
      const int4 r = in ? tb[li] : make_int4(0, 0, (int)(0xffffffffu - (uint32_t)lane), -1);
      const uint32_t f = (uint32_t)r.z;
      const int32_t own = in ? (int32_t)((uint32_t)r.w & 0xffffu) : -1;
      const int32_t cmp = in ? (int32_t)((uint32_t)r.w >> 16) : -2;
      const double c = in ? w0 * pk_raw(r) : 0.0;
      const uint32_t fu = __shfl_up_sync(0xffffffffu, f, 1), fd = __shfl_down_sync(0xffffffffu, f, 1);
      const int32_t ou = __shfl_up_sync(0xffffffffu, own, 1);
      const bool head = lane == 0 || fu != f;
      const bool tail = lane == 31 || fd != f;
      bool edge = false;
      if (in && lane == 0 && p > 0)
        edge = (uint32_t)(li > 0 ? tb[li - 1].z : __ldg(&pk[p - 1]).z) == f;
      if (in && lane == 31 && p + 1 < n)
        edge = edge || (uint32_t)(li + 1 < cnt ? tb[li + 1].z : __ldg(&pk[p + 1]).z) == f;
      const bool bad = edge || (!head && ou != own) || (cmp == own);
      const unsigned hm = __ballot_sync(0xffffffffu, head);
      const int hl = 31 - __clz(hm & (0xffffffffu >> (31 - lane)));
      const unsigned tm = __ballot_sync(0xffffffffu, tail);
      const int tl = __ffs(tm & (0xffffffffu << lane)) - 1;
      const unsigned bm = __ballot_sync(0xffffffffu, bad);
      const unsigned runmask =
          (tl == 31 ? 0xffffffffu : ((1u << (tl + 1)) - 1u)) & (0xffffffffu << hl);
      const int len = tl - hl + 1;
      const bool simple = in && !(bm & runmask) && len <= kRipple;
      double acc = 0.0 + c;
      const int steps = (int)__reduce_max_sync(0xffffffffu, simple ? (unsigned)len : 1u);
      for (int q = 1; q < steps; ++q) {
        const double up = __shfl_up_sync(0xffffffffu, acc, 1);
        if (lane - hl == q) acc = up + c;
      }
      const double total = __shfl_sync(0xffffffffu, acc, tl);
      if (in) {
        if (simple) {
          out[p] = len == 1 ? total : total / (double)len - 0.0;  // x / 1.0 - 0.0 == x: no fp64 division on single-particle sites
          np += (unsigned long long)len;
        } else {
          int64_t L = 0;
          out[p] = site_run_value_pk(pk, w0, p, 0, n, L);
          np += (unsigned long long)L;
        }
      }
    }
    __syncthreads();  // the stage is consumed: refill it with this block's next-but-3 tile
    if (threadIdx.x == 0) {
      const int64_t nt = t + (int64_t)kBulkStages * gridDim.x;
      if (nt < ntiles) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(nt, st);
      }
    }
  }
  if (pairs) block_add_pairs(np, pairs);
}

int32_t sobolev_site_bulk(const int4 *pk, double w0, int64_t n, double *out,
                          unsigned long long *pairs, cudaStream_t s) {
  if (n <= 0) return RCB_OK;
  const size_t smem = (size_t)kBulkStages * kBulkTile * sizeof(int4);
  static bool attr[64] = {};
  int dev = 0;
  RCB_CUDA(cudaGetDevice(&dev));
  if (dev < 64 && !attr[dev]) {
    RCB_CUDA(cudaFuncSetAttribute(k_sobolev_site_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
    attr[dev] = true;
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t ntiles = (n + kBulkTile - 1) / kBulkTile;
  const int64_t grid = ntiles < 2 * sms ? ntiles : 2 * sms;
  k_sobolev_site_bulk<<<(unsigned)grid, 256, smem, s>>>(pk, w0, n, out, pairs);
  RCB_CUDA(cudaGetLastError());
  return RCB_OK;
}

int32_t sobolev_site_pk(const int4 *pk, double w0, int64_t p0, int64_t p1, int64_t lo, int64_t hi,
                        double *out, unsigned long long *pairs, cudaStream_t s) {
  if (p1 <= p0) return RCB_OK;
  // streaming (evict-first) hints measured slower: 0.71 vs 0.52 ms at 8e7 particles
  static const bool plain = !(getenv("RCB_K6_SITE") && strcmp(getenv("RCB_K6_SITE"), "lsu-cs") == 0);
  if (plain)
    k_sobolev_site_pk<false><<<grid_for(p1 - p0, 256 * kSiteChunks), 256, 0, s>>>(
        pk, w0, p0, p1, lo, hi, out, pairs);
  else
    k_sobolev_site_pk<true><<<grid_for(p1 - p0, 256 * kSiteChunks), 256, 0, s>>>(
        pk, w0, p0, p1, lo, hi, out, pairs);
  RCB_CUDA(cudaGetLastError());
  return RCB_OK;
}

bool sobolev_site_only(const Off *rows_host, int nrows) {
  return nrows == 1 && rows_host[0].dz == 0 && rows_host[0].dy == 0 && rows_host[0].dx == 0;
}

int32_t sobolev_site(const uint32_t *px, const int32_t *pown, const int32_t *pcomp,
                     const double *raw, double w0, int64_t p0, int64_t p1, int64_t lo, int64_t hi,
                     double *out, unsigned long long *pairs, cudaStream_t s) {
  if (p1 <= p0) return RCB_OK;
  k_sobolev_site<<<grid_for(p1 - p0, 256 * kSiteChunks), 256, 0, s>>>(px, pown, pcomp, raw, w0,
                                                                      p0, p1, lo, hi, out, pairs);
  RCB_CUDA(cudaGetLastError());
  return RCB_OK;
}

bool sobolev_packable(int32_t n_labels, int nrows, int max_d2) {
  return n_labels <= 65536 && nrows <= kSobRows && max_d2 < kSobW;
}

int32_t sobolev_pack(const uint32_t *px, const int32_t *pown, const int32_t *pcomp,
                     const double *raw, int64_t lo, int64_t hi, int4 *pk, cudaStream_t s) {
  if (hi <= lo) return RCB_OK;
  k_sob_pack<<<grid_for(hi - lo, 256), 256, 0, s>>>(px, pown, pcomp, raw, lo, hi, pk);
  RCB_CUDA(cudaGetLastError());
  return RCB_OK;
}

int32_t sobolev_packed(const uint32_t *site_off, const int4 *pk, const Lat &lat, const Off *rows,
                       int nrows, const double *wt, int nwt, int64_t p0, int64_t p1, double *out,
                       unsigned long long *pairs, cudaStream_t s) {
  if (p1 <= p0) return RCB_OK;
  k_sobolev_pk<<<grid_for(p1 - p0, 128), 128, 0, s>>>(
      site_off, pk, (uint32_t)lat.nx, (uint32_t)lat.ny, (uint32_t)lat.nz, rows, nrows, wt,
      nwt < kSobW ? nwt : kSobW, p0, p1, out, pairs);
  RCB_CUDA(cudaGetLastError());
  return RCB_OK;
}

// Rows of the stencil: (dz, dy) in lexicographic order with half-width
// h = max{dx : dz^2 + dy^2 + dx^2 < (E/2)^2} in Off.dx and dz^2 + dy^2 in
// Off.aux.  max_d2 receives the largest |o|^2 (weight-table length check).
std::vector<Off> sobolev_rows(int ndim, double length_scale, int *max_d2) {
  const double c2 = (length_scale / 2.0) * (length_scale / 2.0);
  const int r = (int)ceil(length_scale / 2.0);
  std::vector<Off> out;
  int mx = 0;
  for (int dz = (ndim == 3 ? -r : 0); dz <= (ndim == 3 ? r : 0); ++dz)
    for (int dy = -r; dy <= r; ++dy) {
      const int b = dz * dz + dy * dy;
      if (!((double)b < c2)) continue;
      int h = 0;
      while ((double)(b + (h + 1) * (h + 1)) < c2) ++h;
      out.push_back(Off{(int8_t)dz, (int8_t)dy, (int8_t)h, (uint8_t)b});
      mx = std::max(mx, b + h * h);
    }
  if (max_d2) *max_d2 = mx;
  return out;
}

// Stencil of the cutoff: offsets with |o|^2 < (E/2)^2 in lexicographic order,
// aux = |o|^2 (index into the weight table).
std::vector<Off> sobolev_stencil(int ndim, double length_scale) {
  double c2 = (length_scale / 2.0) * (length_scale / 2.0);
  int r = (int)ceil(length_scale / 2.0);
  std::vector<Off> out;
  for (int dz = (ndim == 3 ? -r : 0); dz <= (ndim == 3 ? r : 0); ++dz)
    for (int dy = -r; dy <= r; ++dy)
      for (int dx = -r; dx <= r; ++dx) {
        int d2 = dz * dz + dy * dy + dx * dx;
        if ((double)d2 < c2) out.push_back(Off{(int8_t)dz, (int8_t)dy, (int8_t)dx, (uint8_t)d2});
      }
  return out;
}

int32_t sobolev_lattice(const uint32_t *site_off, const int32_t *pown, const uint32_t *px,
                        const int32_t *pcomp, const double *raw, const Lat &lat, const Off *rows,
                        int nrows, const double *wt, int64_t n, double *out,
                        unsigned long long *pairs, cudaStream_t s, int64_t p0) {
  if (n <= p0) return RCB_OK;
  k_sobolev<<<grid_for(n - p0, 128), 128, 0, s>>>(site_off, pown, pcomp, px, raw, lat, rows,
                                                  nrows, wt, n, out, nullptr, pairs, p0);
  RCB_CUDA(cudaGetLastError());
  return RCB_OK;
}

// ---- function-level path: arbitrary coordinates ---------------------------
__global__ void k_canon_keys(const int64_t *__restrict__ coords, int64_t n, int ndim, Lat lat,
                             const int64_t *__restrict__ comps, uint64_t *__restrict__ keys,
                             uint32_t *__restrict__ idx) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t z = ndim == 3 ? coords[i * 3] : 0;
  int64_t y = coords[i * ndim + ndim - 2], x = coords[i * ndim + ndim - 1];
  uint64_t f = (uint64_t)lat.flat(z, y, x);
  keys[i] = (f << 32) | (uint64_t)(uint32_t)comps[i];
  idx[i] = (uint32_t)i;
}

__global__ void k_gather_sorted(const uint64_t *__restrict__ keys, const uint32_t *__restrict__ idx,
                                int64_t n, const int64_t *__restrict__ owners,
                                const double *__restrict__ raw, uint32_t *__restrict__ px,
                                int32_t *__restrict__ own, int32_t *__restrict__ comp,
                                double *__restrict__ rraw, uint32_t *__restrict__ site_cnt) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t k = keys[i];
  uint32_t j = idx[i];
  px[i] = (uint32_t)(k >> 32);
  comp[i] = (int32_t)(uint32_t)(k & 0xffffffffu);
  own[i] = (int32_t)owners[j];
  rraw[i] = raw[j];
  atomicAdd(&site_cnt[k >> 32], 1u);
}

int32_t sobolev_coords(const int64_t *d_coords, int64_t n, int ndim, const Lat &lat,
                       const int64_t *d_owners, const int64_t *d_comps, const double *d_raw,
                       const Off *st, int nst, const double *wt, double *d_out,
                       unsigned long long *d_pairs, cudaStream_t s) {
  DBuf<uint64_t> keys, keys2;
  DBuf<uint32_t> idx, idx2, px, site_off;
  DBuf<int32_t> own, comp;
  DBuf<double> rraw;
  DBuf<uint8_t> tmp;
  int32_t rc = RCB_OK;
  auto run = [&]() -> int32_t {
    RCB_TRY(keys.reserve(n, s));
    RCB_TRY(keys2.reserve(n, s));
    RCB_TRY(idx.reserve(n, s));
    RCB_TRY(idx2.reserve(n, s));
    RCB_TRY(px.reserve(n, s));
    RCB_TRY(own.reserve(n, s));
    RCB_TRY(comp.reserve(n, s));
    RCB_TRY(rraw.reserve(n, s));
    RCB_TRY(site_off.reserve(lat.V + 1, s));
    k_canon_keys<<<grid_for(n, 256), 256, 0, s>>>(d_coords, n, ndim, lat, d_comps, keys.p, idx.p);
    RCB_CUDA(cudaGetLastError());
    size_t b1 = 0, b2 = 0;
    RCB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, b1, keys.p, keys2.p, idx.p, idx2.p, n, 0,
                                             64, s));
    RCB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, b2, site_off.p, site_off.p, lat.V + 1, s));
    RCB_TRY(tmp.reserve(b1 > b2 ? b1 : b2, s));
    RCB_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, b1, keys.p, keys2.p, idx.p, idx2.p, n, 0, 64,
                                             s));
    RCB_CUDA(cudaMemsetAsync(site_off.p, 0, sizeof(uint32_t) * (lat.V + 1), s));
    k_gather_sorted<<<grid_for(n, 256), 256, 0, s>>>(keys2.p, idx2.p, n, d_owners, d_raw, px.p,
                                                     own.p, comp.p, rraw.p, site_off.p);
    RCB_CUDA(cudaGetLastError());
    RCB_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, b2, site_off.p, site_off.p, lat.V + 1, s));
    k_sobolev<<<grid_for(n, 128), 128, 0, s>>>(site_off.p, own.p, comp.p, px.p, rraw.p, lat, st,
                                               nst, wt, n, d_out, idx2.p, d_pairs);
    RCB_CUDA(cudaGetLastError());
    return RCB_OK;
  };
  rc = run();
  keys.release(s);
  keys2.release(s);
  idx.release(s);
  idx2.release(s);
  px.release(s);
  own.release(s);
  comp.release(s);
  rraw.release(s);
  site_off.release(s);
  tmp.release(s);
  return rc;
}

}  // namespace rcb
