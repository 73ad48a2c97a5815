// K1 — contour-particle extraction as a stream compaction of the label
// lattice (replaces contour.py:84-116 scan_contour + :45-57 as_arrays).
//
// Pass 1 writes, per site, the number of distinct competing labels among its
// background-adjacency neighbours; an exclusive scan turns the counts into the
// CSR lattice index map site_off[V+1] (particles of site x are
// [site_off[x], site_off[x+1])).  Pass 2 writes the particle records sorted by
// (x, competitor).  The same site_off is the neighbour index the Sobolev
// stencil (K6) walks.
#include <cstdlib>

#include <cub/device/device_scan.cuh>

#include "dev.cuh"
#include "kernels.h"

namespace rcb {

__global__ void k_contour_count(const int32_t *__restrict__ L, Lat lat, int full_fg,
                                uint32_t *__restrict__ cnt) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < lat.V; f += stride) {
    int64_t z, y, x;
    lat.coord(f, z, y, x);
    int32_t tmp[26];
    cnt[f] = (uint32_t)site_competitors(L, lat, full_fg, z, y, x, __ldg(&L[f]), tmp);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) cnt[lat.V] = 0;
}

__global__ void k_contour_emit(const int32_t *__restrict__ L, Lat lat, int full_fg,
                               const uint32_t *__restrict__ site_off, uint32_t *__restrict__ px,
                               int32_t *__restrict__ pown, int32_t *__restrict__ pcomp) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < lat.V; f += stride) {
    uint32_t o = site_off[f], e = site_off[f + 1];
    if (o == e) continue;
    int64_t z, y, x;
    lat.coord(f, z, y, x);
    int32_t tmp[26];
    int32_t own = __ldg(&L[f]);
    int n = site_competitors(L, lat, full_fg, z, y, x, own, tmp);
    for (int k = 0; k < n; ++k) {
      px[o + k] = (uint32_t)f;
      pown[o + k] = own;
      pcomp[o + k] = tmp[k];
    }
  }
}

// Face-adjacency fast path (full_fg: background adjacency = the 2*ND face
// neighbours; every config of BASELINE.json): 32-bit coordinates, the
// neighbour labels in registers (out-of-lattice and own-label neighbours are
// stored as `own`, so no sentinel value is needed), distinct count by
// unrolled compares, ascending order by an unrolled exchange network — the
// same (x, competitor) order site_competitors produces.
template <int ND>
__device__ __forceinline__ void face_labels(const int32_t *__restrict__ L, uint32_t f, uint32_t nx,
                                            uint32_t ny, uint32_t nz, int32_t own,
                                            int32_t (&v)[2 * ND]) {
  const uint32_t x = f % nx, t = f / nx, y = t % ny;
  v[0] = x > 0 ? __ldg(&L[f - 1]) : own;
  v[1] = x + 1 < nx ? __ldg(&L[f + 1]) : own;
  v[2] = y > 0 ? __ldg(&L[f - nx]) : own;
  v[3] = y + 1 < ny ? __ldg(&L[f + nx]) : own;
  if constexpr (ND == 3) {
    const uint32_t z = t / ny, pl = nx * ny;
    v[4] = z > 0 ? __ldg(&L[f - pl]) : own;
    v[5] = z + 1 < nz ? __ldg(&L[f + pl]) : own;
  }
}

template <int ND>
__global__ void k_contour_count_face(const int32_t *__restrict__ L, uint32_t nx, uint32_t ny,
                                     uint32_t nz, uint32_t V, uint32_t *__restrict__ cnt) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t f = blockIdx.x * blockDim.x + threadIdx.x; f < V; f += stride) {
    const int32_t own = __ldg(&L[f]);
    int32_t v[2 * ND];
    face_labels<ND>(L, f, nx, ny, nz, own, v);
    uint32_t n = 0;
#pragma unroll
    for (int i = 0; i < 2 * ND; ++i) {
      bool fresh = v[i] != own;
#pragma unroll
      for (int j = 0; j < i; ++j) fresh &= v[j] != v[i];
      n += fresh;
    }
    cnt[f] = n;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) cnt[V] = 0;
}

template <int ND>
__global__ void k_contour_emit_face(const int32_t *__restrict__ L, uint32_t nx, uint32_t ny,
                                    uint32_t nz, uint32_t V, const uint32_t *__restrict__ site_off,
                                    uint32_t *__restrict__ px, int32_t *__restrict__ pown,
                                    int32_t *__restrict__ pcomp) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t f = blockIdx.x * blockDim.x + threadIdx.x; f < V; f += stride) {
    uint32_t o = site_off[f];
    if (o == site_off[f + 1]) continue;
    const int32_t own = __ldg(&L[f]);
    int32_t v[2 * ND];
    face_labels<ND>(L, f, nx, ny, nz, own, v);
#pragma unroll
    for (int i = 0; i < 2 * ND; ++i)
#pragma unroll
      for (int j = 0; j + 1 < 2 * ND - i; ++j) {
        const int32_t a = min(v[j], v[j + 1]), b = max(v[j], v[j + 1]);
        v[j] = a;
        v[j + 1] = b;
      }
#pragma unroll
    for (int i = 0; i < 2 * ND; ++i)
      if (v[i] != own && (i == 0 || v[i] != v[i - 1])) {
        px[o] = f;
        pown[o] = own;
        pcomp[o] = v[i];
        ++o;
      }
  }
}

static bool face_path(const Lat &lat, int full_fg) {
  static const bool generic = getenv("RCB_CONTOUR_GENERIC") != nullptr;  // comparison runs
  return full_fg && lat.V < (int64_t(1) << 31) && !generic;
}

int32_t contour_scan(const int32_t *L, const Lat &lat, int full_fg, uint32_t *site_off,
                     DBuf<uint8_t> &tmp, cudaStream_t s) {
  const int T = 256;
  if (face_path(lat, full_fg)) {
    if (lat.ndim == 3)
      k_contour_count_face<3><<<grid_for(lat.V, T), T, 0, s>>>(L, lat.nx, lat.ny, lat.nz, lat.V,
                                                               site_off);
    else
      k_contour_count_face<2><<<grid_for(lat.V, T), T, 0, s>>>(L, lat.nx, lat.ny, lat.nz, lat.V,
                                                               site_off);
  } else {
    k_contour_count<<<grid_for(lat.V, T), T, 0, s>>>(L, lat, full_fg, site_off);
  }
  RCB_CUDA(cudaGetLastError());
  size_t bytes = 0;
  RCB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, site_off, site_off, lat.V + 1, s));
  RCB_TRY(tmp.reserve(bytes, s));
  RCB_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, site_off, site_off, lat.V + 1, s));
  return RCB_OK;
}

int32_t contour_emit(const int32_t *L, const Lat &lat, int full_fg, const uint32_t *site_off,
                     uint32_t *px, int32_t *pown, int32_t *pcomp, cudaStream_t s) {
  const int T = 256;
  if (face_path(lat, full_fg)) {
    if (lat.ndim == 3)
      k_contour_emit_face<3><<<grid_for(lat.V, T), T, 0, s>>>(L, lat.nx, lat.ny, lat.nz, lat.V,
                                                              site_off, px, pown, pcomp);
    else
      k_contour_emit_face<2><<<grid_for(lat.V, T), T, 0, s>>>(L, lat.nx, lat.ny, lat.nz, lat.V,
                                                              site_off, px, pown, pcomp);
  } else {
    k_contour_emit<<<grid_for(lat.V, T), T, 0, s>>>(L, lat, full_fg, site_off, px, pown, pcomp);
  }
  RCB_CUDA(cudaGetLastError());
  return RCB_OK;
}

}  // namespace rcb
