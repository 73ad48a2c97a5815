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

// Four sites per thread (rows whose length is a multiple of four: every
// BASELINE lattice): one 16-byte load per neighbour row instead of four scalar
// ones, x-neighbours from the thread's own vector plus two edge loads, row
// coordinates by multiply-shift once per quad (the scalar kernels spend ~100
// instructions per site on four 32-bit divisions and were issue bound at
// 1.4 TB/s of DRAM traffic), 16-byte stores of the counts.  Same counts and
// the same (x, competitor) order as the scalar kernels.
struct QuadDiv {
  uint32_t m_row, l_row, m_y, l_y;  // q / (nx / 4) and row / ny (q, row < 2^31)
};
static QuadDiv quad_div(uint32_t nxq, uint32_t ny) {
  auto magic = [](uint32_t d, uint32_t &m, uint32_t &l) {
    l = 0;
    while ((1ull << l) < d) ++l;
    m = (uint32_t)(((1ull << 32) * ((1ull << l) - d)) / d + 1);
  };
  QuadDiv q;
  magic(nxq, q.m_row, q.l_row);
  magic(ny, q.m_y, q.l_y);
  return q;
}

template <int ND>
__device__ __forceinline__ void quad_labels(const int32_t *__restrict__ L, uint32_t q, uint32_t nx,
                                            uint32_t ny, uint32_t nz, QuadDiv d, int4 &own,
                                            int32_t (&v)[4][2 * ND]) {
  const uint32_t nxq = nx >> 2;
  const uint32_t row = (__umulhi(d.m_row, q) + q) >> d.l_row;
  const uint32_t x0 = (q - row * nxq) << 2;
  const uint32_t z = ND == 3 ? (__umulhi(d.m_y, row) + row) >> d.l_y : 0u;
  const uint32_t y = row - z * ny;
  const uint32_t f0 = q << 2;
  own = __ldg(reinterpret_cast<const int4 *>(L + f0));
  const int4 up = y > 0 ? __ldg(reinterpret_cast<const int4 *>(L + f0 - nx)) : own;
  const int4 dn = y + 1 < ny ? __ldg(reinterpret_cast<const int4 *>(L + f0 + nx)) : own;
  const int32_t lf = x0 > 0 ? __ldg(L + f0 - 1) : own.x;
  const int32_t rt = x0 + 4 < nx ? __ldg(L + f0 + 4) : own.w;
  const int32_t o[4] = {own.x, own.y, own.z, own.w};
  const int32_t u[4] = {up.x, up.y, up.z, up.w}, w[4] = {dn.x, dn.y, dn.z, dn.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    v[i][0] = i == 0 ? lf : o[i - 1];
    v[i][1] = i == 3 ? rt : o[i + 1];
    v[i][2] = u[i];
    v[i][3] = w[i];
  }
  if constexpr (ND == 3) {
    const uint32_t pl = nx * ny;
    const int4 bk = z > 0 ? __ldg(reinterpret_cast<const int4 *>(L + f0 - pl)) : own;
    const int4 fr = z + 1 < nz ? __ldg(reinterpret_cast<const int4 *>(L + f0 + pl)) : own;
    const int32_t b[4] = {bk.x, bk.y, bk.z, bk.w}, g[4] = {fr.x, fr.y, fr.z, fr.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v[i][4] = b[i];
      v[i][5] = g[i];
    }
  }
}

template <int ND>
__global__ void __launch_bounds__(256) k_contour_count_face4(const int32_t *__restrict__ L,
                                                             uint32_t nx, uint32_t ny, uint32_t nz,
                                                             uint32_t V, QuadDiv d,
                                                             uint32_t *__restrict__ cnt) {
  const uint32_t nq = V >> 2, stride = gridDim.x * blockDim.x;
  for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += stride) {
    int4 own4;
    int32_t v[4][2 * ND];
    quad_labels<ND>(L, q, nx, ny, nz, d, own4, v);
    const int32_t o[4] = {own4.x, own4.y, own4.z, own4.w};
    uint32_t n[4];
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      n[s] = 0;
#pragma unroll
      for (int i = 0; i < 2 * ND; ++i) {
        bool fresh = v[s][i] != o[s];
#pragma unroll
        for (int j = 0; j < i; ++j) fresh &= v[s][j] != v[s][i];
        n[s] += fresh;
      }
    }
    *reinterpret_cast<uint4 *>(cnt + (q << 2)) = make_uint4(n[0], n[1], n[2], n[3]);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) cnt[V] = 0;
}

template <int ND>
__global__ void __launch_bounds__(256) k_contour_emit_face4(
    const int32_t *__restrict__ L, uint32_t nx, uint32_t ny, uint32_t nz, uint32_t V, QuadDiv d,
    const uint32_t *__restrict__ site_off, uint32_t *__restrict__ px, int32_t *__restrict__ pown,
    int32_t *__restrict__ pcomp) {
  const uint32_t nq = V >> 2, stride = gridDim.x * blockDim.x;
  for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += stride) {
    const uint32_t f0 = q << 2;
    const uint4 so = __ldg(reinterpret_cast<const uint4 *>(site_off + f0));
    const uint32_t oe = __ldg(site_off + f0 + 4);
    if (so.x == oe) continue;  // no particle in these four sites
    int4 own4;
    int32_t v[4][2 * ND];
    quad_labels<ND>(L, q, nx, ny, nz, d, own4, v);
    const int32_t ow[4] = {own4.x, own4.y, own4.z, own4.w};
    const uint32_t off[5] = {so.x, so.y, so.z, so.w, oe};
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      if (off[s] == off[s + 1]) continue;
#pragma unroll
      for (int i = 0; i < 2 * ND; ++i)
#pragma unroll
        for (int j = 0; j + 1 < 2 * ND - i; ++j) {
          const int32_t a = min(v[s][j], v[s][j + 1]), b = max(v[s][j], v[s][j + 1]);
          v[s][j] = a;
          v[s][j + 1] = b;
        }
      uint32_t o = off[s];
#pragma unroll
      for (int i = 0; i < 2 * ND; ++i)
        if (v[s][i] != ow[s] && (i == 0 || v[s][i] != v[s][i - 1])) {
          px[o] = f0 + s;
          pown[o] = ow[s];
          pcomp[o] = v[s][i];
          ++o;
        }
    }
  }
}

static bool quad_path(const Lat &lat, int full_fg) {
  static const bool scalar = getenv("RCB_CONTOUR_SCALAR") != nullptr;  // comparison runs
  return !scalar && full_fg && lat.V < (int64_t(1) << 31) && lat.nx % 4 == 0 && lat.nx >= 4 &&
         !getenv("RCB_CONTOUR_GENERIC");
}

static bool face_path(const Lat &lat, int full_fg) {
  static const bool generic = getenv("RCB_CONTOUR_GENERIC") != nullptr;  // comparison runs
  return full_fg && lat.V < (int64_t(1) << 31) && !generic;
}

int32_t contour_scan(const int32_t *L, const Lat &lat, int full_fg, uint32_t *site_off,
                     DBuf<uint8_t> &tmp, cudaStream_t s) {
  const int T = 256;
  if (quad_path(lat, full_fg)) {
    const QuadDiv d = quad_div((uint32_t)(lat.nx / 4), (uint32_t)lat.ny);
    if (lat.ndim == 3)
      k_contour_count_face4<3><<<grid_for(lat.V / 4, T), T, 0, s>>>(L, lat.nx, lat.ny, lat.nz,
                                                                    lat.V, d, site_off);
    else
      k_contour_count_face4<2><<<grid_for(lat.V / 4, T), T, 0, s>>>(L, lat.nx, lat.ny, lat.nz,
                                                                    lat.V, d, site_off);
  } else if (face_path(lat, full_fg)) {
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
  if (quad_path(lat, full_fg)) {
    const QuadDiv d = quad_div((uint32_t)(lat.nx / 4), (uint32_t)lat.ny);
    if (lat.ndim == 3)
      k_contour_emit_face4<3><<<grid_for(lat.V / 4, T), T, 0, s>>>(
          L, lat.nx, lat.ny, lat.nz, lat.V, d, site_off, px, pown, pcomp);
    else
      k_contour_emit_face4<2><<<grid_for(lat.V / 4, T), T, 0, s>>>(
          L, lat.nx, lat.ny, lat.nz, lat.V, d, site_off, px, pown, pcomp);
  } else if (face_path(lat, full_fg)) {
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
