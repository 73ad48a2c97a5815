// K1 — contour-particle extraction as a stream compaction of the label
// lattice (replaces contour.py:84-116 scan_contour + :45-57 as_arrays).
//
// Pass 1 writes, per site, the number of distinct competing labels among its
// background-adjacency neighbours; an exclusive scan turns the counts into the
// CSR lattice index map site_off[V+1] (particles of site x are
// [site_off[x], site_off[x+1])).  Pass 2 writes the particle records sorted by
// (x, competitor).  The same site_off is the neighbour index the Sobolev
// stencil (K6) walks.
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

int32_t contour_scan(const int32_t *L, const Lat &lat, int full_fg, uint32_t *site_off,
                     DBuf<uint8_t> &tmp, cudaStream_t s) {
  const int T = 256;
  k_contour_count<<<grid_for(lat.V, T), T, 0, s>>>(L, lat, full_fg, site_off);
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
  k_contour_emit<<<grid_for(lat.V, T), T, 0, s>>>(L, lat, full_fg, site_off, px, pown, pcomp);
  RCB_CUDA(cudaGetLastError());
  return RCB_OK;
}

}  // namespace rcb
