#include <vector>
#include <climits>
#include <cstring>
// Energy kernels: K2 region statistics, K3 PC increment + perimeter change,
// K4 own-label PS ball fields, K5 PS increment, K9 exact energy totals.
#include <cub/device/device_radix_sort.cuh>

#include "dev.cuh"
#include "kernels.h"
#include "ordered_sum.cuh"

namespace rcb {

// ---------------------------------------------------------------------------
// K3 (energy.py:111-126, 308-324)
// ---------------------------------------------------------------------------
__global__ void k_delta_int(const int32_t *__restrict__ L, Lat lat, const uint32_t *__restrict__ px,
                            const int32_t *__restrict__ pown, const int32_t *__restrict__ pcomp,
                            int64_t n, int32_t *__restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t z, y, x;
  lat.coord(px[i], z, y, x);
  out[i] = delta_internal(L, lat, z, y, x, pown[i], pcomp[i]);
}

// K6's 16-byte partner record {raw, site, owner | competitor << 16}
// (sobolev.cu:k_sobolev_pk), written by the energy kernels so that K6 needs
// no separate packing pass (labels < 2^16).
__device__ __forceinline__ int4 pack_record(double raw, uint32_t site, int32_t own, int32_t comp) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(raw);
  return make_int4((int)(uint32_t)u, (int)(uint32_t)(u >> 32), (int)site,
                   (int)((uint32_t)own | ((uint32_t)comp << 16)));
}

__global__ void k_delta_pc(const double *__restrict__ I, const uint32_t *__restrict__ px,
                           const int32_t *__restrict__ pown, const int32_t *__restrict__ pcomp,
                           int64_t n, const int64_t *__restrict__ cnt,
                           const double *__restrict__ tot, const double *__restrict__ tsq,
                           int poisson, double *__restrict__ out, int4 *__restrict__ pk) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int32_t a = pown[i], b = pcomp[i];
  const uint32_t f = px[i];
  const double d = delta_pc(__ldg(&I[f]), cnt[a], tot[a], tsq[a], cnt[b], tot[b], tsq[b], poisson);
  out[i] = d;
  if (pk) pk[i] = pack_record(d, f, a, b);
}

// ---------------------------------------------------------------------------
// K4/K5 (energy.py:196-223, 337-372)
// ---------------------------------------------------------------------------
__global__ void k_ps_fields(const int32_t *__restrict__ L, const double *__restrict__ I, Lat lat,
                            const Off *__restrict__ ball, int nball, int32_t *__restrict__ Cown,
                            double *__restrict__ Sown) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < lat.V; f += stride) {
    int64_t z, y, x;
    lat.coord(f, z, y, x);
    int32_t own = __ldg(&L[f]);
    int32_t c = 0;
    double s = 0.0;
    for (int k = 0; k < nball; ++k) {
      Off o = ball[k];
      int64_t zz = z + o.dz, yy = y + o.dy, xx = x + o.dx;
      if (!lat.inb(zz, yy, xx)) continue;
      int64_t g = lat.flat(zz, yy, xx);
      if (__ldg(&L[g]) != own) continue;
      c += 1;
      s += __ldg(&I[g]);
    }
    Cown[f] = c;
    Sown[f] = s;
  }
}

// k_ps_fields for lattices below 2^31 sites, fused with the rho0 table:
// 32-bit coordinates, packed ball offsets in shared memory, four offsets'
// loads in flight; same ball order and sums (bit-identical fields).
__global__ void __launch_bounds__(256) k_ps_fields32(
    const int32_t *__restrict__ L, const double *__restrict__ I, int nx, int ny, int nz,
    const Off *__restrict__ ball, int nball, int32_t *__restrict__ Cown, double *__restrict__ Sown,
    double *__restrict__ rho0, int poisson) {
  __shared__ int sofs[1024];
  for (int k = threadIdx.x; k < nball; k += blockDim.x)
    sofs[k] = ((int)(uint8_t)ball[k].dz << 16) | ((int)(uint8_t)ball[k].dy << 8) |
              (int)(uint8_t)ball[k].dx;
  __syncthreads();
  const int plane = nx * ny;
  const int64_t V = (int64_t)plane * nz;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t f64 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f64 < V; f64 += stride) {
    const int f = (int)f64;
    const int z = f / plane, rem = f - z * plane;
    const int y = rem / nx, x = rem - y * nx;
    const int32_t own = __ldg(&L[f]);
    int32_t c = 0;
    double sv = 0.0;
    for (int k0 = 0; k0 < nball; k0 += 4) {
      int g[4];
      int32_t lab[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int k = k0 + u;
        const int o = k < nball ? sofs[k] : 0;
        const int zz = z + (int)(int8_t)(o >> 16), yy = y + (int)(int8_t)(o >> 8),
                  xx = x + (int)(int8_t)o;
        const bool ok = k < nball && (unsigned)zz < (unsigned)nz && (unsigned)yy < (unsigned)ny &&
                        (unsigned)xx < (unsigned)nx;
        g[u] = ok ? zz * plane + yy * nx + xx : f;
        lab[u] = ok ? __ldg(L + g[u]) : -1;
      }
      double iv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) iv[u] = lab[u] == own ? __ldg(I + g[u]) : 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (lab[u] == own) {
          c += 1;
          sv += iv[u];
        }
    }
    Cown[f] = c;
    Sown[f] = sv;
    if (rho0) rho0[f] = rho(__ldg(&I[f]), sv / (double)c, poisson);
  }
}

// 2-D own-label fields on 32 x 8 site tiles staged in shared memory with a
// halo of R: every ball walk reads labels and intensities from the tile, in
// the same ball order as the global-memory kernels (bit-identical fields).
// dirty == nullptr: every site (the rebuild); else only the dirty sites,
// which are cleared (the band refresh, 2-D).
static constexpr int kTW = 32, kTH = 8, kTRmax = 15;
__global__ void __launch_bounds__(256) k_fields_tile2d(
    const int32_t *__restrict__ L, const double *__restrict__ I, int nx, int ny,
    const Off *__restrict__ ball, int nball, int R, uint8_t *__restrict__ dirty,
    int32_t *__restrict__ Cown, double *__restrict__ Sown, double *__restrict__ rho0, int poisson,
    long long *__restrict__ band) {
  constexpr int SH = kTH + 2 * kTRmax, SW = kTW + 2 * kTRmax;
  __shared__ int32_t sL[SH * SW];
  __shared__ double sI[SH * SW];
  __shared__ int sofs[1024];
  __shared__ long long sm[kLimbs];
  const int tx = threadIdx.x & (kTW - 1), ty = threadIdx.x / kTW;
  const int x0 = blockIdx.x * kTW, y0 = blockIdx.y * kTH;
  const int x = x0 + tx, y = y0 + ty;
  const bool inside = x < nx && y < ny;
  const int64_t f = (int64_t)y * nx + x;
  const bool todo = inside && (!dirty || dirty[f]);
  if (!__syncthreads_or(todo)) return;
  const int hw = kTW + 2 * R, hh = kTH + 2 * R;
  for (int i = threadIdx.x; i < hw * hh; i += blockDim.x) {
    const int hy = i / hw, hx = i - hy * hw;
    const int gy = y0 - R + hy, gx = x0 - R + hx;
    const bool ok = (unsigned)gy < (unsigned)ny && (unsigned)gx < (unsigned)nx;
    const int64_t g = (int64_t)gy * nx + gx;
    sL[hy * SW + hx] = ok ? __ldg(L + g) : -1;
    sI[hy * SW + hx] = ok ? __ldg(I + g) : 0.0;
  }
  for (int k = threadIdx.x; k < nball; k += blockDim.x)
    sofs[k] = (int)ball[k].dy * SW + (int)ball[k].dx;
  if (band)
    for (int k = threadIdx.x; k < kLimbs; k += blockDim.x) sm[k] = 0;
  __syncthreads();
  double oldr = 0.0, newr = 0.0;
  if (todo) {
    const int cidx = (ty + R) * SW + (tx + R);
    const int32_t own = sL[cidx];
    int32_t c = 0;
    double sv = 0.0;
    for (int k = 0; k < nball; ++k) {
      const int j = cidx + sofs[k];
      if (sL[j] == own) {
        c += 1;
        sv += sI[j];
      }
    }
    if (band) oldr = rho0[f];
    Cown[f] = c;
    Sown[f] = sv;
    newr = rho(sI[cidx], sv / (double)c, poisson);
    if (rho0) rho0[f] = newr;
    if (dirty) dirty[f] = 0;
  }
  if (band) {  // exact band ledger (every thread of the block reaches here)
    acc_add_warp(sm, -oldr, todo);
    acc_add_warp(sm, newr, todo);
    acc_flush(sm, band);
  }
}

// 3-D variant: 16 x 4 x 4 site tiles with a halo of R <= 4 (24 x 12 x 12
// cells in shared memory), optional band ledger (the exact sum of rho_new -
// rho_old over the refreshed sites into the superaccumulator band[]).
static constexpr int kT3X = 16, kT3Y = 4, kT3Z = 4, kT3R = 4;
__global__ void __launch_bounds__(256) k_fields_tile3d(
    const int32_t *__restrict__ L, const double *__restrict__ I, int nx, int ny, int nz,
    const Off *__restrict__ ball, int nball, int R, uint8_t *__restrict__ dirty,
    int32_t *__restrict__ Cown, double *__restrict__ Sown, double *__restrict__ rho0, int poisson,
    long long *__restrict__ band) {
  constexpr int SX = kT3X + 2 * kT3R, SY = kT3Y + 2 * kT3R, SZ = kT3Z + 2 * kT3R;
  __shared__ int32_t sL[SX * SY * SZ];
  __shared__ double sI[SX * SY * SZ];
  __shared__ int sofs[1024];
  __shared__ long long sm[kLimbs];
  const int tx = threadIdx.x % kT3X, ty = (threadIdx.x / kT3X) % kT3Y, tz = threadIdx.x / (kT3X * kT3Y);
  const int x0 = blockIdx.x * kT3X, y0 = blockIdx.y * kT3Y, z0 = blockIdx.z * kT3Z;
  const int x = x0 + tx, y = y0 + ty, z = z0 + tz;
  const bool inside = x < nx && y < ny && z < nz;
  const int64_t f = ((int64_t)z * ny + y) * nx + x;
  const bool todo = inside && (!dirty || dirty[f]);
  if (!__syncthreads_or(todo)) return;
  const int hx = kT3X + 2 * R, hy = kT3Y + 2 * R, hz = kT3Z + 2 * R;
  for (int i = threadIdx.x; i < hx * hy * hz; i += blockDim.x) {
    const int cz = i / (hx * hy), rem = i - cz * hx * hy;
    const int cy = rem / hx, cx = rem - cy * hx;
    const int gz = z0 - R + cz, gy = y0 - R + cy, gx = x0 - R + cx;
    const bool ok = (unsigned)gz < (unsigned)nz && (unsigned)gy < (unsigned)ny &&
                    (unsigned)gx < (unsigned)nx;
    const int64_t g = ((int64_t)gz * ny + gy) * nx + gx;
    const int si = (cz * SY + cy) * SX + cx;
    sL[si] = ok ? __ldg(L + g) : -1;
    sI[si] = ok ? __ldg(I + g) : 0.0;
  }
  for (int k = threadIdx.x; k < nball; k += blockDim.x)
    sofs[k] = ((int)ball[k].dz * SY + (int)ball[k].dy) * SX + (int)ball[k].dx;
  if (band)
    for (int k = threadIdx.x; k < kLimbs; k += blockDim.x) sm[k] = 0;
  __syncthreads();
  double oldr = 0.0, newr = 0.0;
  if (todo) {
    const int cidx = ((tz + R) * SY + (ty + R)) * SX + (tx + R);
    const int32_t own = sL[cidx];
    int32_t c = 0;
    double sv = 0.0;
    for (int k = 0; k < nball; ++k) {
      const int j = cidx + sofs[k];
      if (sL[j] == own) {
        c += 1;
        sv += sI[j];
      }
    }
    if (band) oldr = rho0[f];
    Cown[f] = c;
    Sown[f] = sv;
    newr = rho(sI[cidx], sv / (double)c, poisson);
    if (rho0) rho0[f] = newr;
    if (dirty) dirty[f] = 0;
  }
  if (band) {  // every thread of the block reaches here (warp-uniform)
    acc_add_warp(sm, -oldr, todo);
    acc_add_warp(sm, newr, todo);
    acc_flush(sm, band);
  }
}

// 3-D band refresh from the flip map: flips[x] = 1 at this iteration's
// flipped sites and tflag[t] = 1 for the tiles holding them (k_mark_flips).
// A tile is processed iff one of the 27 tiles around it (R <= the tile
// extents) holds a flip; its sites whose ball holds a flip (checked on the
// staged flip flags, nearest offsets first) are recomputed as in
// k_fields_tile3d -- the sites the per-flip ball scatter used to mark, without
// the ~3e9 scattered byte writes per cfg4 iteration.
__global__ void __launch_bounds__(256) k_fields_band3d(
    const int32_t *__restrict__ L, const double *__restrict__ I, int nx, int ny, int nz,
    const Off *__restrict__ ball, int nball, int R, const uint8_t *__restrict__ flips,
    const uint8_t *__restrict__ tflag, int32_t *__restrict__ Cown, double *__restrict__ Sown,
    double *__restrict__ rho0, int poisson, long long *__restrict__ band) {
  constexpr int SX = kT3X + 2 * kT3R, SY = kT3Y + 2 * kT3R, SZ = kT3Z + 2 * kT3R;
  static_assert(SX <= 32, "a halo row's flips must fit one 32-bit mask");
  __shared__ int32_t sL[SX * SY * SZ];
  __shared__ double sI[SX * SY * SZ];
  __shared__ uint32_t rowbits[SY * SZ];  // flips of each halo row, bit = x cell
  __shared__ int srow[(2 * kT3R + 1) * (2 * kT3R + 1)];  // ball rows: dz:8 | dy:8 | h:8
  __shared__ int nrow;
  __shared__ int sofs[512];  // R <= kT3R = 4: <= 257 ball offsets
  __shared__ long long sm[kLimbs];
  const int ntx = gridDim.x, nty = gridDim.y, ntz = gridDim.z;
  bool any = false;
  if (threadIdx.x < 27) {
    const int tz = (int)blockIdx.z + (int)threadIdx.x / 9 - 1;
    const int ty = (int)blockIdx.y + ((int)threadIdx.x / 3) % 3 - 1;
    const int tx = (int)blockIdx.x + (int)threadIdx.x % 3 - 1;
    if ((unsigned)tz < (unsigned)ntz && (unsigned)ty < (unsigned)nty && (unsigned)tx < (unsigned)ntx)
      any = tflag[((int64_t)tz * nty + ty) * ntx + tx] != 0;
  }
  if (!__syncthreads_or(any)) return;
  const int tx = threadIdx.x % kT3X, ty = (threadIdx.x / kT3X) % kT3Y, tz = threadIdx.x / (kT3X * kT3Y);
  const int x0 = blockIdx.x * kT3X, y0 = blockIdx.y * kT3Y, z0 = blockIdx.z * kT3Z;
  const int x = x0 + tx, y = y0 + ty, z = z0 + tz;
  const bool inside = x < nx && y < ny && z < nz;
  const int64_t f = ((int64_t)z * ny + y) * nx + x;
  const int hx = kT3X + 2 * R, hy = kT3Y + 2 * R, hz = kT3Z + 2 * R;
  for (int i = threadIdx.x; i < hy * hz; i += blockDim.x) rowbits[i] = 0u;
  if (threadIdx.x == 0) {  // the ball as x-runs per (dz, dy): |o|^2 <= R^2
    int k = 0;
    for (int dz = -R; dz <= R; ++dz)
      for (int dy = -R; dy <= R; ++dy) {
        const int t = R * R - dz * dz - dy * dy;
        if (t < 0) continue;
        int h = 0;
        while ((h + 1) * (h + 1) <= t) ++h;
        srow[k++] = ((dz & 0xff) << 16) | ((dy & 0xff) << 8) | h;
      }
    nrow = k;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < hx * hy * hz; i += blockDim.x) {
    const int cz = i / (hx * hy), rem = i - cz * hx * hy;
    const int cy = rem / hx, cx = rem - cy * hx;
    const int gz = z0 - R + cz, gy = y0 - R + cy, gx = x0 - R + cx;
    const bool ok = (unsigned)gz < (unsigned)nz && (unsigned)gy < (unsigned)ny &&
                    (unsigned)gx < (unsigned)nx;
    const int64_t g = ((int64_t)gz * ny + gy) * nx + gx;
    const int si = (cz * SY + cy) * SX + cx;
    if (ok && __ldg(flips + g)) atomicOr(&rowbits[cz * hy + cy], 1u << cx);
    sL[si] = ok ? __ldg(L + g) : -1;
    sI[si] = ok ? __ldg(I + g) : 0.0;
  }
  for (int k = threadIdx.x; k < nball; k += blockDim.x)
    sofs[k] = ((int)ball[k].dz * SY + (int)ball[k].dy) * SX + (int)ball[k].dx;
  if (band)
    for (int k = threadIdx.x; k < kLimbs; k += blockDim.x) sm[k] = 0;
  __syncthreads();
  // a flip within the ball: one mask test per ball row
  bool todo = false;
  if (inside) {
    const int nr = nrow;
    for (int k = 0; k < nr; ++k) {
      const int r = srow[k];
      const int dz = (int)(int8_t)(r >> 16), dy = (int)(int8_t)(r >> 8), h = r & 0xff;
      const uint32_t m = ((2u << (2 * h)) - 1u) << (tx + R - h);
      if (rowbits[(tz + R + dz) * hy + (ty + R + dy)] & m) {
        todo = true;
        break;
      }
    }
  }
  const int cidx = ((tz + R) * SY + (ty + R)) * SX + (tx + R);
  double oldr = 0.0, newr = 0.0;
  if (todo) {
    const int32_t own = sL[cidx];
    int32_t c = 0;
    double sv = 0.0;
    for (int k = 0; k < nball; ++k) {
      const int j = cidx + sofs[k];
      if (sL[j] == own) {
        c += 1;
        sv += sI[j];
      }
    }
    if (band) oldr = rho0[f];
    Cown[f] = c;
    Sown[f] = sv;
    newr = rho(sI[cidx], sv / (double)c, poisson);
    if (rho0) rho0[f] = newr;
  }
  if (band) {  // every thread of the block reaches here (warp-uniform)
    acc_add_warp(sm, -oldr, todo);
    acc_add_warp(sm, newr, todo);
    acc_flush(sm, band);
  }
}

// 3-D band refresh for integer images (0 <= I < 2^12, labels < 2^16 - 1, ball
// sums < 2^20: the conditions of the packed K5 records).  Integer sums are
// exact in any order, so the own-label ball sums need not follow the ball's
// offset order: the ball is cut into its x-runs (one per (dz, dy), 49 for
// R = 4) and a run's sum is a difference of two entries of a per-row prefix
// sum of the packed word (1 << 20 | I) over the cells of one label -- 98
// shared-memory reads per site instead of 257 compare-and-add steps over two
// arrays.  One prefix table is built per label present among the tile's own
// sites (usually one or two).  Every site of an active tile is evaluated and
// written only where (C, S) changed: a site whose ball holds a flip that left
// its own-label sums alone kept the same rho0, and its ledger term was an
// exact zero.  Same Cown / Sown / rho0 / band sums as k_fields_band3d.
// Tiles of 16 x 8 x 8 sites, four sites (z, z + 2, z + 4, z + 6) per thread:
// the 24 x 16 x 16 halo costs 6 staged cells per site (13.5 with the 16 x 4 x 4
// tiles of the fp64 kernels) and a prefix table serves 1 024 sites.
static constexpr int kBiX = 16, kBiY = 8, kBiZ = 8, kBiZT = 2, kBiS = kBiZ / kBiZT;
static constexpr int kBiPS = kBiX + 2 * kT3R + 1;  // row stride (odd: conflict-free row walks)
__global__ void __launch_bounds__(256) k_fields_band3d_int(
    const int32_t *__restrict__ L, const uint16_t *__restrict__ I16, int nx, int ny, int nz, int R,
    const uint8_t *__restrict__ tflag, int32_t *__restrict__ Cown, double *__restrict__ Sown,
    double *__restrict__ rho0, int poisson, long long *__restrict__ band, int4 *__restrict__ rec,
    int ztile0, int ntz_all, int own_z0, int own_z1) {
  // ztile0 / gridDim.z: the z-tiles to refresh (a rank of a z-slab sharded run
  // refreshes its slab plus the halo its energy kernel reads); [own_z0, own_z1):
  // the planes whose ledger terms this call sums (the rank's own slab).
  constexpr int SY = kBiY + 2 * kT3R, SZ = kBiZ + 2 * kT3R;
  extern __shared__ __align__(16) uint32_t bi_smem[];
  uint32_t *sW = bi_smem;                   // label | I << 16 (0xffff: outside the lattice)
  uint32_t *sP = bi_smem + SZ * SY * kBiPS;  // per row: prefix sums of (1 << 20 | I) over one label
  __shared__ int2 srow[(2 * kT3R + 1) * (2 * kT3R + 1)];  // per ball row: offsets of the two prefix entries
  __shared__ int nrow, s_pick;
  __shared__ long long sm[kLimbs];
  const int ntx = gridDim.x, nty = gridDim.y, ntz = ntz_all;
  const int bz = (int)blockIdx.z + ztile0;
  if (tflag) {  // null: every tile (the full rebuild), every site written
    bool any = false;
    if (threadIdx.x < 27) {
      const int tz = bz + (int)threadIdx.x / 9 - 1;
      const int ty = (int)blockIdx.y + ((int)threadIdx.x / 3) % 3 - 1;
      const int tx = (int)blockIdx.x + (int)threadIdx.x % 3 - 1;
      if ((unsigned)tz < (unsigned)ntz && (unsigned)ty < (unsigned)nty && (unsigned)tx < (unsigned)ntx)
        any = tflag[((int64_t)tz * nty + ty) * ntx + tx] != 0;
    }
    if (!__syncthreads_or(any)) return;
  }
  const int tx = threadIdx.x % kBiX, ty = (threadIdx.x / kBiX) % kBiY, tz = threadIdx.x / (kBiX * kBiY);
  const int x0 = blockIdx.x * kBiX, y0 = blockIdx.y * kBiY, z0 = bz * kBiZ;
  const int x = x0 + tx, y = y0 + ty;
  const int hx = kBiX + 2 * R, hy = kBiY + 2 * R, hz = kBiZ + 2 * R;
  if (threadIdx.x == 0) {  // the ball as x-runs per (dz, dy): |o|^2 <= R^2
    int k = 0;
    for (int dz = -R; dz <= R; ++dz)
      for (int dy = -R; dy <= R; ++dy) {
        const int t = R * R - dz * dz - dy * dy;
        if (t < 0) continue;
        int h = 0;
        while ((h + 1) * (h + 1) <= t) ++h;
        const int rb = (dz * SY + dy) * kBiPS;
        srow[k++] = make_int2(rb + h + 1, rb - h);  // prefix[x + h + 1] - prefix[x - h]
      }
    nrow = k;
  }
  // halo rows (cz, cy) x hx cells; one row per warp pass keeps the loads coalesced
  for (int row = threadIdx.x >> 5; row < hy * hz; row += 8) {
    const int cz = row / hy, cy = row - cz * hy;
    const int gz = z0 - R + cz, gy = y0 - R + cy;
    const int cx = threadIdx.x & 31;
    if (cx < hx) {
      const int gx = x0 - R + cx;
      const bool ok = (unsigned)gz < (unsigned)nz && (unsigned)gy < (unsigned)ny &&
                      (unsigned)gx < (unsigned)nx;
      const int64_t g = ((int64_t)gz * ny + gy) * nx + gx;
      sW[(cz * SY + cy) * kBiPS + cx] =
          ok ? ((uint32_t)__ldg(L + g) | ((uint32_t)__ldg(I16 + g) << 16)) : 0xffffu;
    }
  }
  if (band)
    for (int k = threadIdx.x; k < kLimbs; k += blockDim.x) sm[k] = 0;
  __syncthreads();
  int cb[kBiS], own[kBiS];
  uint32_t tot[kBiS], wc[kBiS];
  bool todo[kBiS], inside[kBiS];
#pragma unroll
  for (int j = 0; j < kBiS; ++j) {
    const int zl = tz + kBiZT * j;
    cb[j] = ((zl + R) * SY + (ty + R)) * kBiPS + tx + R;
    wc[j] = sW[cb[j]];
    inside[j] = x < nx && y < ny && z0 + zl < nz;
    own[j] = inside[j] ? (int)(wc[j] & 0xffffu) : 0x7fffffff;
    todo[j] = inside[j];
    tot[j] = 0;
  }
  for (;;) {  // one pass per label among the tile's own sites, smallest first
    if (threadIdx.x == 0) s_pick = 0x7fffffff;
    __syncthreads();
    int mine = 0x7fffffff;
#pragma unroll
    for (int j = 0; j < kBiS; ++j)
      if (todo[j] && own[j] < mine) mine = own[j];
    const int wmin = (int)__reduce_min_sync(0xffffffffu, (unsigned)mine);
    if ((threadIdx.x & 31) == 0 && wmin != 0x7fffffff) atomicMin(&s_pick, wmin);
    __syncthreads();
    const int l = s_pick;
    if (l == 0x7fffffff) break;
    for (int row = threadIdx.x; row < hy * hz; row += blockDim.x) {
      // this row's prefix sums over the cells of label l
      const int cz = row / hy, cy = row - cz * hy;
      const int rb = (cz * SY + cy) * kBiPS;
      uint32_t a = 0;
      sP[rb] = 0;
#pragma unroll 8
      for (int cx = 0; cx < hx; ++cx) {
        const uint32_t w = sW[rb + cx];
        if ((int)(w & 0xffffu) == l) a += (1u << 20) + (w >> 16);
        sP[rb + cx + 1] = a;
      }
    }
    __syncthreads();
    bool any_mine = false;
#pragma unroll
    for (int j = 0; j < kBiS; ++j) any_mine |= todo[j] && own[j] == l;
    if (any_mine) {
      const int nr = nrow;
      uint32_t t[kBiS];
#pragma unroll
      for (int j = 0; j < kBiS; ++j) t[j] = 0;
      for (int k = 0; k < nr; ++k) {
        const int2 r = srow[k];
#pragma unroll
        for (int j = 0; j < kBiS; ++j) t[j] += sP[cb[j] + r.x] - sP[cb[j] + r.y];
      }
#pragma unroll
      for (int j = 0; j < kBiS; ++j)
        if (todo[j] && own[j] == l) {
          tot[j] = t[j];
          todo[j] = false;
        }
    }
  }
  AccStage stage;
#pragma unroll
  for (int j = 0; j < kBiS; ++j) {
    double oldr = 0.0, newr = 0.0;
    bool changed = false;
    if (inside[j]) {
      const int64_t f = ((int64_t)(z0 + tz + kBiZT * j) * ny + y) * nx + x;
      const int32_t c = (int32_t)(tot[j] >> 20);
      const double sv = (double)(tot[j] & 0xfffffu);
      // K5's packed site record (k_pack_sites' layout) is kept current here,
      // so the energy kernel needs no packing pass over the lattice: a site
      // whose label, count or sum changed is exactly one whose record did
      const uint32_t w0 = (uint32_t)own[j] | ((uint32_t)c << 16);
      const uint32_t w1 = (tot[j] & 0xfffffu) | ((wc[j] >> 16) << 20);
      if (rec) {
        const int2 old = __ldg(reinterpret_cast<const int2 *>(rec + f));
        changed = !tflag || (uint32_t)old.x != w0 || (uint32_t)old.y != w1;
      } else {
        changed = !tflag || Cown[f] != c || Sown[f] != sv;
      }
      if (changed) {
        if (band) oldr = rho0[f];
        Cown[f] = c;
        Sown[f] = sv;
        newr = rho((double)(wc[j] >> 16), sv / (double)c, poisson);
        if (rho0) rho0[f] = newr;
        if (rec) {
          const unsigned long long rb = (unsigned long long)__double_as_longlong(newr);
          rec[f] = make_int4((int)w0, (int)w1, (int)(uint32_t)rb, (int)(uint32_t)(rb >> 32));
        }
      }
    }
    if (band && changed) {
      const int zz = z0 + tz + kBiZT * j;
      if (zz >= own_z0 && zz < own_z1) {
        stage.add(sm, -oldr);
        stage.add(sm, newr);
      }
    }
  }
  if (band) {  // every thread of the block reaches here (warp-uniform)
    stage.flush_warp(sm);
    acc_flush(sm, band);
  }
}

static size_t band3d_int_smem() {
  return 2 * (size_t)(kBiZ + 2 * kT3R) * (kBiY + 2 * kT3R) * kBiPS * sizeof(uint32_t);
}

static int32_t launch_band3d_int(const int32_t *L, const uint16_t *I16, const Lat &lat, int R,
                                 const uint8_t *tflag, int32_t *Cown, double *Sown, double *rho0,
                                 int poisson, long long *band, int4 *rec, cudaStream_t s,
                                 const BandSlab *slab = nullptr) {
  static bool attr[64] = {};
  int dev = 0;
  RCB_CUDA(cudaGetDevice(&dev));
  if (dev < 64 && !attr[dev]) {
    RCB_CUDA(cudaFuncSetAttribute(k_fields_band3d_int, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)band3d_int_smem()));
    attr[dev] = true;
  }
  const int ntz = (int)((lat.nz + kBiZ - 1) / kBiZ);
  int zt0 = 0, ztn = ntz, oz0 = 0, oz1 = (int)lat.nz;
  if (slab) {  // tiles meeting planes [z0, z1), ledger over [own0, own1)
    zt0 = (int)(std::max<int64_t>(slab->z0, 0) / kBiZ);
    const int zt1 = (int)((std::min<int64_t>(slab->z1, lat.nz) + kBiZ - 1) / kBiZ);
    ztn = zt1 > zt0 ? zt1 - zt0 : 0;
    oz0 = (int)slab->own0;
    oz1 = (int)slab->own1;
    if (ztn == 0) return RCB_OK;
  }
  dim3 grid((unsigned)((lat.nx + kBiX - 1) / kBiX), (unsigned)((lat.ny + kBiY - 1) / kBiY),
            (unsigned)ztn);
  k_fields_band3d_int<<<grid, 256, band3d_int_smem(), s>>>(L, I16, (int)lat.nx, (int)lat.ny,
                                                           (int)lat.nz, R, tflag, Cown, Sown, rho0,
                                                           poisson, band, rho0 ? rec : nullptr, zt0,
                                                           ntz, oz0, oz1);
  RCB_CUDA(cudaGetLastError());
  return RCB_OK;
}

__global__ void k_to_u16(const double *__restrict__ src, int64_t n, uint16_t *__restrict__ dst) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    dst[i] = (uint16_t)src[i];
}

int32_t image_u16(const double *I, int64_t V, uint16_t *I16, cudaStream_t s) {
  k_to_u16<<<148 * 16, 256, 0, s>>>(I, V, I16);
  RCB_CUDA(cudaGetLastError());
  return RCB_OK;
}

// per accepted move: flips[x] = v, tflag[tile(x)] = v (v = 1 mark, 0 clear)
__global__ void k_mark_flips(const int64_t *__restrict__ acc, const int64_t *__restrict__ moves,
                             Lat lat, uint8_t v, uint8_t *__restrict__ flips,
                             uint8_t *__restrict__ tflag, int kT3X, int kT3Y, int kT3Z) {
  const int64_t n = *moves;
  const int ntx = (int)((lat.nx + kT3X - 1) / kT3X), nty = (int)((lat.ny + kT3Y - 1) / kT3Y);
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t f = acc[3 * k];
    int64_t z, y, x;
    lat.coord(f, z, y, x);
    if (flips) flips[f] = v;
    tflag[((z / kT3Z) * nty + y / kT3Y) * ntx + x / kT3X] = v;
  }
}

int64_t band3d_tiles(const Lat &lat) {
  return ((lat.nx + kT3X - 1) / kT3X) * ((lat.ny + kT3Y - 1) / kT3Y) *
         ((lat.nz + kT3Z - 1) / kT3Z);
}

int32_t fields_band3d(const int64_t *acc, const int64_t *moves, const int32_t *L, const double *I,
                      const uint16_t *I16, const Lat &lat, const Off *ball_full, int nball_full,
                      int R, uint8_t *flips, uint8_t *tflag, int32_t *Cown, double *Sown,
                      double *rho0, int poisson, long long *band, cudaStream_t s, int4 *rec,
                      const BandSlab *slab) {
  if (I16) {
    // integer image: prefix-sum ball runs on 16 x 8 x 8 tiles (the caller
    // checked the ranges); only the tile flags are marked, no per-site map
    k_mark_flips<<<148 * 8, 256, 0, s>>>(acc, moves, lat, 1, nullptr, tflag, kBiX, kBiY, kBiZ);
    RCB_TRY(launch_band3d_int(L, I16, lat, R, tflag, Cown, Sown, rho0, poisson, band, rec, s, slab));
    k_mark_flips<<<148 * 8, 256, 0, s>>>(acc, moves, lat, 0, nullptr, tflag, kBiX, kBiY, kBiZ);
    RCB_CUDA(cudaGetLastError());
    return RCB_OK;
  }
  k_mark_flips<<<148 * 8, 256, 0, s>>>(acc, moves, lat, 1, flips, tflag, kT3X, kT3Y, kT3Z);
  dim3 grid((unsigned)((lat.nx + kT3X - 1) / kT3X), (unsigned)((lat.ny + kT3Y - 1) / kT3Y),
            (unsigned)((lat.nz + kT3Z - 1) / kT3Z));
  k_fields_band3d<<<grid, kT3X * kT3Y * kT3Z, 0, s>>>(L, I, (int)lat.nx, (int)lat.ny, (int)lat.nz,
                                                       ball_full, nball_full, R, flips, tflag,
                                                       Cown, Sown, rho0, poisson, band);
  k_mark_flips<<<148 * 8, 256, 0, s>>>(acc, moves, lat, 0, flips, tflag, kT3X, kT3Y, kT3Z);
  RCB_CUDA(cudaGetLastError());
  return RCB_OK;
}

int32_t fields_tile3d(const int32_t *L, const double *I, const Lat &lat, const Off *ball_full,
                      int nball_full, int R, uint8_t *dirty, int32_t *Cown, double *Sown,
                      double *rho0, int poisson, long long *band, cudaStream_t s) {
  dim3 grid((unsigned)((lat.nx + kT3X - 1) / kT3X), (unsigned)((lat.ny + kT3Y - 1) / kT3Y),
            (unsigned)((lat.nz + kT3Z - 1) / kT3Z));
  k_fields_tile3d<<<grid, kT3X * kT3Y * kT3Z, 0, s>>>(L, I, (int)lat.nx, (int)lat.ny, (int)lat.nz,
                                                       ball_full, nball_full, R, dirty, Cown, Sown,
                                                       rho0, poisson, band);
  RCB_CUDA(cudaGetLastError());
  return RCB_OK;
}

bool fields_tile3d_ok(const Lat &lat, int R, int nball_full) {
  return lat.ndim == 3 && R <= kT3R && nball_full <= 1024 && (lat.nz + kT3Z - 1) / kT3Z < 65536 &&
         (lat.ny + kT3Y - 1) / kT3Y < 65536;
}

int32_t fields_tile2d(const int32_t *L, const double *I, const Lat &lat, const Off *ball_full,
                      int nball_full, int R, uint8_t *dirty, int32_t *Cown, double *Sown,
                      double *rho0, int poisson, cudaStream_t s, long long *band) {
  dim3 grid((unsigned)((lat.nx + kTW - 1) / kTW), (unsigned)((lat.ny + kTH - 1) / kTH));
  k_fields_tile2d<<<grid, kTW * kTH, 0, s>>>(L, I, (int)lat.nx, (int)lat.ny, ball_full, nball_full,
                                             R, dirty, Cown, Sown, rho0, poisson,
                                             rho0 ? band : nullptr);
  RCB_CUDA(cudaGetLastError());
  return RCB_OK;
}

bool fields_tile2d_ok(const Lat &lat, int R, int nball_full) {
  return lat.ndim == 2 && R <= kTRmax && nball_full <= 1024 && lat.ny < 65536 * kTH &&
         lat.nx < 65536 * kTW;
}

__global__ void k_rho0(const int32_t *__restrict__ Cown, const double *__restrict__ Sown,
                       const double *__restrict__ I, int64_t V, int poisson,
                       double *__restrict__ rho0) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < V; f += stride)
    rho0[f] = rho(I[f], Sown[f] / (double)Cown[f], poisson);
}

__global__ void k_delta_ps(const int32_t *__restrict__ L, const double *__restrict__ I,
                           const int32_t *__restrict__ Cown, const double *__restrict__ Sown,
                           Lat lat, const Off *__restrict__ ball, int nball,
                           const uint32_t *__restrict__ px, const int32_t *__restrict__ pown,
                           const int32_t *__restrict__ pcomp, int64_t n, int poisson,
                           double *__restrict__ out, const double *__restrict__ rho0,
                           int32_t *__restrict__ cb0, double *__restrict__ sb0) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t z, y, x;
  lat.coord(px[i], z, y, x);
  int32_t cb;
  double sb;
  out[i] = delta_ps(L, I, Cown, Sown, lat, ball, nball, z, y, x, pown[i], pcomp[i], poisson, &cb,
                    &sb, rho0);
  if (cb0) {  // the competitor's iteration-start ball count/sum at x (PS ledger terms)
    cb0[i] = cb;
    sb0[i] = sb;
  }
}

// K5 for 2-D lattices (the common case): one pass over the ball per particle
// with 32-bit coordinates and the offsets staged in shared memory; loads for
// kChunk offsets are issued before any is used.  The a-terms and b-terms are
// still two separate sequential sums in ball-offset order, so the result is
// bit-identical to delta_ps (dev.cuh).
static constexpr int kPsChunk = 4, kPsMaxBall = 1024;

__global__ void __launch_bounds__(128, 6) k_delta_ps2d(
    const int32_t *__restrict__ L, const double *__restrict__ I, const int32_t *__restrict__ Cown,
    const double *__restrict__ Sown, int nx, int ny, const Off *__restrict__ ball, int nball,
    const uint32_t *__restrict__ px, const int32_t *__restrict__ pown,
    const int32_t *__restrict__ pcomp, int64_t n, int poisson, double *__restrict__ out,
    const double *__restrict__ rho0, int32_t *__restrict__ cb0, double *__restrict__ sb0,
    const double *__restrict__ lt, int ltP, int4 *__restrict__ pk) {
  __shared__ int8_t sdy[kPsMaxBall], sdx[kPsMaxBall];
  for (int k = threadIdx.x; k < nball; k += blockDim.x) {
    sdy[k] = ball[k].dy;
    sdx[k] = ball[k].dx;
  }
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int f = (int)px[i];
  const int y = f / nx, x = f - y * nx;
  const int32_t a = pown[i], b = pcomp[i];
  const double v = I[f];
  double acc_a = 0.0, acc_b = 0.0, sb = 0.0;
  int32_t cb = 0;
  for (int k0 = 0; k0 < nball; k0 += kPsChunk) {
    int g[kPsChunk];
    int32_t lab[kPsChunk];
#pragma unroll
    for (int u = 0; u < kPsChunk; ++u) {
      const int k = k0 + u;
      const int yy = y + (k < nball ? sdy[k] : 0), xx = x + (k < nball ? sdx[k] : 0);
      const bool ok = k < nball && (unsigned)yy < (unsigned)ny && (unsigned)xx < (unsigned)nx;
      g[u] = ok ? yy * nx + xx : f;
      lab[u] = ok ? __ldg(L + g[u]) : -1;
    }
    double cy[kPsChunk], sy[kPsChunk], iy[kPsChunk], r0[kPsChunk];
#pragma unroll
    for (int u = 0; u < kPsChunk; ++u) {
      const bool need = lab[u] == a || lab[u] == b;
      cy[u] = need ? (double)__ldg(Cown + g[u]) : 1.0;
      sy[u] = need ? __ldg(Sown + g[u]) : 0.0;
      iy[u] = need ? __ldg(I + g[u]) : 0.0;
      r0[u] = (need && rho0) ? __ldg(rho0 + g[u]) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kPsChunk; ++u) {
      // one rho evaluation for either side (no divergent a/b paths): the
      // a-term's (sy - v)/(cy - 1) is computed as (sy + (-v))/(cy + (-1)),
      // which IEEE arithmetic rounds identically
      const bool isa = lab[u] == a;
      if (isa || lab[u] == b) {
        const double num = sy[u] + (isa ? -v : v), den = cy[u] + (isa ? -1.0 : 1.0);
        const double theta = num / den;
        // integer Poisson data: the log from the table (bit-identical)
        const double rn = (lt && den >= 1.0) ? theta - iy[u] * __ldg(lt + (int)den * ltP + (int)num)
                                             : rho(iy[u], theta, poisson);
        const double t = rn - (rho0 ? r0[u] : rho(iy[u], sy[u] / cy[u], poisson));
        if (isa) {
          acc_a += t;
        } else {
          acc_b += t;
          cb += 1;
          sb += iy[u];
        }
      }
    }
  }
  double d = 0.0 + acc_a;
  d = d + acc_b;
  d += rho(v, (sb + v) / ((double)cb + 1.0), poisson);
  d -= rho0 ? rho0[f] : rho(v, Sown[f] / (double)Cown[f], poisson);
  out[i] = d;
  if (pk) pk[i] = pack_record(d, (uint32_t)f, a, b);
  if (cb0) {  // the competitor's iteration-start ball count/sum at x (PS ledger terms)
    cb0[i] = cb;
    sb0[i] = sb;
  }
}

// K5 for 3-D lattices below 2^31 sites: the 2-D kernel's scheme (one pass
// over the ball, 32-bit coordinates, offsets in shared memory, kPsChunk
// offsets' loads in flight) with (dz, dy, dx) offsets.  The a- and b-terms are
// two sequential sums in ball-offset order: bit-identical to delta_ps.
__global__ void __launch_bounds__(128, 6) k_delta_ps3d(
    const int32_t *__restrict__ L, const double *__restrict__ I, const int32_t *__restrict__ Cown,
    const double *__restrict__ Sown, int nx, int ny, int nz, const Off *__restrict__ ball,
    int nball, const uint32_t *__restrict__ px, const int32_t *__restrict__ pown,
    const int32_t *__restrict__ pcomp, int64_t n, int poisson, double *__restrict__ out,
    const double *__restrict__ rho0, int32_t *__restrict__ cb0, double *__restrict__ sb0,
    const double *__restrict__ lt, int ltP, int4 *__restrict__ pk) {
  __shared__ int sofs[kPsMaxBall];  // dz:8 | dy:8 | dx:8, signed, packed
  __shared__ int sdel[kPsMaxBall];  // linear site delta of each offset
  __shared__ int srad;              // largest |component| of the offsets
  if (threadIdx.x == 0) srad = 0;
  __syncthreads();
  for (int k = threadIdx.x; k < nball; k += blockDim.x) {
    const int dz = ball[k].dz, dy = ball[k].dy, dx = ball[k].dx;
    sofs[k] = ((int)(uint8_t)ball[k].dz << 16) | ((int)(uint8_t)ball[k].dy << 8) |
              (int)(uint8_t)ball[k].dx;
    sdel[k] = (dz * ny + dy) * nx + dx;
    atomicMax(&srad, max(abs(dz), max(abs(dy), abs(dx))));
  }
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int f = (int)px[i];
  const int plane = nx * ny;
  const int z = f / plane, r = f - z * plane;
  const int y = r / nx, x = r - y * nx;
  const int32_t a = pown[i], b = pcomp[i];
  const double v = I[f];
  // interior particles (the whole ball inside the lattice): one add per
  // offset instead of three coordinates, three bounds tests and a multiply
  const int rad = srad;
  const bool interior = z >= rad && z < nz - rad && y >= rad && y < ny - rad && x >= rad &&
                        x < nx - rad;
  double acc_a = 0.0, acc_b = 0.0, sb = 0.0;
  int32_t cb = 0;
  for (int k0 = 0; k0 < nball; k0 += kPsChunk) {
    int g[kPsChunk];
    int32_t lab[kPsChunk];
#pragma unroll
    for (int u = 0; u < kPsChunk; ++u) {
      const int k = k0 + u;
      bool ok;
      if (interior) {
        ok = k < nball;
        g[u] = ok ? f + sdel[k] : f;
      } else {
        const int o = k < nball ? sofs[k] : 0;
        const int zz = z + (int)(int8_t)(o >> 16), yy = y + (int)(int8_t)(o >> 8),
                  xx = x + (int)(int8_t)o;
        ok = k < nball && (unsigned)zz < (unsigned)nz && (unsigned)yy < (unsigned)ny &&
             (unsigned)xx < (unsigned)nx;
        g[u] = ok ? zz * plane + yy * nx + xx : f;
      }
      lab[u] = ok ? __ldg(L + g[u]) : -1;
    }
    double cy[kPsChunk], sy[kPsChunk], iy[kPsChunk], r0[kPsChunk];
#pragma unroll
    for (int u = 0; u < kPsChunk; ++u) {
      const bool need = lab[u] == a || lab[u] == b;
      cy[u] = need ? (double)__ldg(Cown + g[u]) : 1.0;
      sy[u] = need ? __ldg(Sown + g[u]) : 0.0;
      iy[u] = need ? __ldg(I + g[u]) : 0.0;
      r0[u] = (need && rho0) ? __ldg(rho0 + g[u]) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kPsChunk; ++u) {
      // one rho evaluation for either side (no divergent a/b paths): the
      // a-term's (sy - v)/(cy - 1) is computed as (sy + (-v))/(cy + (-1)),
      // which IEEE arithmetic rounds identically
      const bool isa = lab[u] == a;
      if (isa || lab[u] == b) {
        const double num = sy[u] + (isa ? -v : v), den = cy[u] + (isa ? -1.0 : 1.0);
        const double theta = num / den;
        // integer Poisson data: the log from the table (bit-identical)
        const double rn = (lt && den >= 1.0) ? theta - iy[u] * __ldg(lt + (int)den * ltP + (int)num)
                                             : rho(iy[u], theta, poisson);
        const double t = rn - (rho0 ? r0[u] : rho(iy[u], sy[u] / cy[u], poisson));
        if (isa) {
          acc_a += t;
        } else {
          acc_b += t;
          cb += 1;
          sb += iy[u];
        }
      }
    }
  }
  double d = 0.0 + acc_a;
  d = d + acc_b;
  d += rho(v, (sb + v) / ((double)cb + 1.0), poisson);
  d -= rho0 ? rho0[f] : rho(v, Sown[f] / (double)Cown[f], poisson);
  out[i] = d;
  if (pk) pk[i] = pack_record(d, (uint32_t)f, a, b);
  if (cb0) {
    cb0[i] = cb;
    sb0[i] = sb;
  }
}

// fp32 gradient path (dev.cuh: delta_pc32 / delta_ps32); outputs in float
// (for K6) and double (rank composition in l2 mode).
__global__ void k_delta_pc32(const float *__restrict__ I32, const uint32_t *__restrict__ px,
                             const int32_t *__restrict__ pown, const int32_t *__restrict__ pcomp,
                             int64_t n, const int64_t *__restrict__ cnt,
                             const double *__restrict__ tot, int poisson,
                             float *__restrict__ out32, double *__restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t a = pown[i], b = pcomp[i];
  const float d = delta_pc32(__ldg(&I32[px[i]]), cnt[a], tot[a], cnt[b], tot[b], poisson);
  out32[i] = d;
  out[i] = (double)d;
}

__global__ void k_delta_ps32(const int32_t *__restrict__ L, const float *__restrict__ I32,
                             const int32_t *__restrict__ Cown, const double *__restrict__ Sown,
                             Lat lat, const Off *__restrict__ ball, int nball,
                             const uint32_t *__restrict__ px, const int32_t *__restrict__ pown,
                             const int32_t *__restrict__ pcomp, int64_t n, int poisson,
                             float *__restrict__ out32, double *__restrict__ out,
                             int32_t *__restrict__ cb0, double *__restrict__ sb0) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t z, y, x;
  lat.coord(px[i], z, y, x);
  int32_t cb;
  double sb;
  const float d = delta_ps32(L, I32, Cown, Sown, lat, ball, nball, z, y, x, pown[i], pcomp[i],
                             poisson, &cb, &sb);
  if (cb0) {
    cb0[i] = cb;
    sb0[i] = sb;
  }
  out32[i] = d;
  out[i] = (double)d;
}

__global__ void k_to_float(const double *__restrict__ src, int64_t n, float *__restrict__ dst) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    dst[i] = (float)src[i];
}

int32_t to_float(const double *src, int64_t n, float *dst, cudaStream_t s) {
  k_to_float<<<grid_for(n, 256), 256, 0, s>>>(src, n, dst);
  RCB_CUDA(cudaGetLastError());
  return RCB_OK;
}

int32_t delta_pc32_batch(const float *I32, const uint32_t *px, const int32_t *pown,
                         const int32_t *pcomp, int64_t n, const int64_t *cnt, const double *tot,
                         int poisson, float *out32, double *out, cudaStream_t s) {
  if (n == 0) return RCB_OK;
  k_delta_pc32<<<grid_for(n, 256), 256, 0, s>>>(I32, px, pown, pcomp, n, cnt, tot, poisson, out32,
                                                out);
  RCB_CUDA(cudaGetLastError());
  return RCB_OK;
}

int32_t delta_ps32_batch(const int32_t *L, const float *I32, const int32_t *Cown,
                         const double *Sown, const Lat &lat, const Off *ball, int nball,
                         const uint32_t *px, const int32_t *pown, const int32_t *pcomp, int64_t n,
                         int poisson, float *out32, double *out, cudaStream_t s, int32_t *cb0,
                         double *sb0) {
  if (n == 0) return RCB_OK;
  k_delta_ps32<<<grid_for(n, 128), 128, 0, s>>>(L, I32, Cown, Sown, lat, ball, nball, px, pown,
                                                pcomp, n, poisson, out32, out, cb0, sb0);
  RCB_CUDA(cudaGetLastError());
  return RCB_OK;
}

int32_t delta_int_batch(const int32_t *L, const Lat &lat, const uint32_t *px, const int32_t *pown,
                        const int32_t *pcomp, int64_t n, int32_t *out, cudaStream_t s) {
  if (n == 0) return RCB_OK;
  k_delta_int<<<grid_for(n, 256), 256, 0, s>>>(L, lat, px, pown, pcomp, n, out);
  RCB_CUDA(cudaGetLastError());
  return RCB_OK;
}

int32_t delta_pc_batch(const double *I, const uint32_t *px, const int32_t *pown,
                       const int32_t *pcomp, int64_t n, const int64_t *cnt, const double *tot,
                       const double *tsq, int poisson, double *out, cudaStream_t s, int4 *pk) {
  if (n == 0) return RCB_OK;
  k_delta_pc<<<grid_for(n, 256), 256, 0, s>>>(I, px, pown, pcomp, n, cnt, tot, tsq, poisson, out,
                                              pk);
  RCB_CUDA(cudaGetLastError());
  return RCB_OK;
}

int32_t ps_fields(const int32_t *L, const double *I, const Lat &lat, const Off *ball_full,
                  int nball_full, int32_t *Cown, double *Sown, cudaStream_t s, double *rho0,
                  int poisson, const uint16_t *I16) {
  int R = 0;  // the ball radius (ball_full is on the device: from its site count)
  if (lat.ndim == 2) {
    for (int r = 1; r <= kTRmax; ++r) {
      int cnt = 0;
      for (int dy = -r; dy <= r; ++dy)
        for (int dx = -r; dx <= r; ++dx) cnt += dy * dy + dx * dx <= r * r;
      if (cnt == nball_full) {
        R = r;
        break;
      }
    }
  }
  if (lat.ndim == 3) {
    for (int r = 1; r <= kT3R; ++r) {
      int cnt = 0;
      for (int dz = -r; dz <= r; ++dz)
        for (int dy = -r; dy <= r; ++dy)
          for (int dx = -r; dx <= r; ++dx) cnt += dz * dz + dy * dy + dx * dx <= r * r;
      if (cnt == nball_full) {
        R = r;
        break;
      }
    }
    if (R > 0 && fields_tile3d_ok(lat, R, nball_full)) {
      if (I16 && rho0)  // integer image: prefix-sum ball runs over every tile
        return launch_band3d_int(L, I16, lat, R, nullptr, Cown, Sown, rho0, poisson, nullptr,
                                 nullptr, s);
      return fields_tile3d(L, I, lat, ball_full, nball_full, R, nullptr, Cown, Sown, rho0, poisson,
                           nullptr, s);
    }
  }
  if (R > 0 && fields_tile2d_ok(lat, R, nball_full))
    return fields_tile2d(L, I, lat, ball_full, nball_full, R, nullptr, Cown, Sown, rho0, poisson, s);
  if (lat.V < ((int64_t)1 << 31) && nball_full <= 1024) {
    int64_t g = (lat.V + 255) / 256;
    if (g > 148 * 64) g = 148 * 64;
    k_ps_fields32<<<(unsigned)(g < 1 ? 1 : g), 256, 0, s>>>(L, I, (int)lat.nx, (int)lat.ny,
                                                          (int)lat.nz, ball_full, nball_full, Cown,
                                                          Sown, rho0, poisson);
  } else {
    k_ps_fields<<<grid_for(lat.V, 256), 256, 0, s>>>(L, I, lat, ball_full, nball_full, Cown, Sown);
    if (rho0) k_rho0<<<grid_for(lat.V, 256), 256, 0, s>>>(Cown, Sown, I, lat.V, poisson, rho0);
  }
  RCB_CUDA(cudaGetLastError());
  return RCB_OK;
}

// K5 on shared-memory tiles (3-D, integer images, R <= 4).  ncu on cfg4
// showed the per-particle kernel bound by L1/L2 traffic: every particle
// re-gathers its 257-site ball from five arrays (L1 hit 22 %, L2 throughput
// 65 %, DRAM 2 %).  Here a block stages an 8^3 tile plus its R-halo once --
// labels, own-label counts and sums, intensities and rho0 -- and the tile's
// particles (contiguous CSR ranges of its 64 rows) walk their balls in
// shared memory with precomputed linear offsets.  Integer data up to 4096
// (checked at engine creation) makes the compact staged types exact
// (intensities and own-label sums in fp32, counts in 16 bits), and every
// fp64 expression is the one of k_delta_ps3d: bit-identical results.
static constexpr int kTileT = 8;
__global__ void __launch_bounds__(128) k_delta_ps3d_tile(
    const int32_t *__restrict__ L, const double *__restrict__ I, const int32_t *__restrict__ Cown,
    const double *__restrict__ Sown, const double *__restrict__ rho0, int nx, int ny, int nz, int R,
    const Off *__restrict__ ball, int nball, const uint32_t *__restrict__ site_off,
    const uint32_t *__restrict__ px, const int32_t *__restrict__ pown,
    const int32_t *__restrict__ pcomp, int64_t h0, int64_t h1, int poisson,
    double *__restrict__ out, int32_t *__restrict__ cb0, double *__restrict__ sb0,
    const double *__restrict__ lt, int ltP) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int H = kTileT + 2 * R, cells = H * H * H;
  double *sR = reinterpret_cast<double *>(smem);
  float *sI = reinterpret_cast<float *>(sR + cells);
  float *sS = sI + cells;
  int32_t *sL = reinterpret_cast<int32_t *>(sS + cells);
  uint16_t *sC = reinterpret_cast<uint16_t *>(sL + cells);
  int *sofs = reinterpret_cast<int *>(sC + ((cells + 1) & ~1));
  int *rows = sofs + nball;  // kTileT^2 + 1 particle prefix offsets
  __shared__ uint32_t rbeg[kTileT * kTileT];
  const int x0 = blockIdx.x * kTileT, y0 = blockIdx.y * kTileT, z0 = blockIdx.z * kTileT;
  // the tile's particles: row (ty, tz) holds [site_off[row + x0], site_off[row + x0 + 8])
  if (threadIdx.x < kTileT * kTileT) {
    const int ty = threadIdx.x % kTileT, tz = threadIdx.x / kTileT;
    const int y = y0 + ty, z = z0 + tz;
    uint32_t b = 0, e = 0;
    if (y < ny && z < nz) {
      const int64_t rb = ((int64_t)z * ny + y) * nx;
      b = __ldg(site_off + rb + x0);
      e = __ldg(site_off + rb + min(x0 + kTileT, nx));
      if ((int64_t)b < h0) b = (uint32_t)((int64_t)e < h0 ? (int64_t)e : h0);
      if ((int64_t)e > h1) e = (uint32_t)((int64_t)b > h1 ? (int64_t)b : h1);
    }
    rbeg[threadIdx.x] = b;
    rows[threadIdx.x + 1] = (int)(e - b);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    rows[0] = 0;
    for (int k = 1; k <= kTileT * kTileT; ++k) rows[k] += rows[k - 1];
  }
  __syncthreads();
  const int np = rows[kTileT * kTileT];
  if (np == 0) return;
  for (int i = threadIdx.x; i < cells; i += blockDim.x) {
    const int cz = i / (H * H), rem = i - cz * H * H;
    const int cy = rem / H, cx = rem - cy * H;
    const int gz = z0 - R + cz, gy = y0 - R + cy, gx = x0 - R + cx;
    const bool ok = (unsigned)gz < (unsigned)nz && (unsigned)gy < (unsigned)ny &&
                    (unsigned)gx < (unsigned)nx;
    const int64_t g = ((int64_t)gz * ny + gy) * nx + gx;
    const int32_t l = ok ? __ldg(L + g) : -1;
    sL[i] = l;
    sC[i] = ok ? (uint16_t)__ldg(Cown + g) : (uint16_t)1;
    sI[i] = ok ? (float)__ldg(I + g) : 0.f;
    sS[i] = ok ? (float)__ldg(Sown + g) : 0.f;
    sR[i] = ok ? __ldg(rho0 + g) : 0.0;
  }
  for (int k = threadIdx.x; k < nball; k += blockDim.x)
    sofs[k] = ((int)ball[k].dz * H + (int)ball[k].dy) * H + (int)ball[k].dx;
  __syncthreads();
  for (int t = threadIdx.x; t < np; t += blockDim.x) {
    int r = 0;  // row of the t-th particle (binary search over 64 prefixes)
    for (int step = 32; step; step >>= 1)
      if (rows[r + step] <= t) r += step;
    const int64_t i = (int64_t)rbeg[r] + (t - rows[r]);
    const int f = (int)px[i];
    const int lx = f % nx - x0 + R, rest = f / nx;
    const int ly = rest % ny - y0 + R, lz = rest / ny - z0 + R;
    const int cidx = (lz * H + ly) * H + lx;
    const int32_t a = pown[i], b = pcomp[i];
    const double v = (double)sI[cidx];
    double acc_a = 0.0, acc_b = 0.0, sb = 0.0;
    int32_t cb = 0;
    for (int k = 0; k < nball; ++k) {
      const int j = cidx + sofs[k];
      const int32_t lab = sL[j];
      const bool isa = lab == a;
      if (isa || lab == b) {
        const double cy = (double)sC[j], sy = (double)sS[j], iy = (double)sI[j];
        const double num = sy + (isa ? -v : v), den = cy + (isa ? -1.0 : 1.0);
        const double theta = num / den;
        const double rn = (lt && den >= 1.0) ? theta - iy * __ldg(lt + (int)den * ltP + (int)num)
                                             : rho(iy, theta, poisson);
        const double tt = rn - sR[j];
        if (isa) {
          acc_a += tt;
        } else {
          acc_b += tt;
          cb += 1;
          sb += iy;
        }
      }
    }
    double d = 0.0 + acc_a;
    d = d + acc_b;
    d += rho(v, (sb + v) / ((double)cb + 1.0), poisson);
    d -= sR[cidx];
    out[i] = d;
    if (cb0) {
      cb0[i] = cb;
      sb0[i] = sb;
    }
  }
}

size_t ps3d_tile_smem(int R, int nball) {
  const int H = kTileT + 2 * R, cells = H * H * H;
  return (size_t)cells * (8 + 4 + 4 + 4) + (size_t)((cells + 1) & ~1) * 2 +
         (size_t)(nball + kTileT * kTileT + 1) * 4;
}

bool ps3d_tile_ok(const Lat &lat, int R, int nball) {
  return lat.ndim == 3 && R >= 1 && R <= 4 && nball <= 256 && lat.V < ((int64_t)1 << 31) &&
         ps3d_tile_smem(R, nball) <= 200 * 1024;
}

// K5 over the particles [h0, h1) of the site-sorted list, by tiles (see
// k_delta_ps3d_tile); every out / cb0 / sb0 entry of the range is written.
int32_t delta_ps3d_tiles(const int32_t *L, const double *I, const int32_t *Cown,
                         const double *Sown, const double *rho0, const Lat &lat, int R,
                         const Off *ball, int nball, const uint32_t *site_off, const uint32_t *px,
                         const int32_t *pown, const int32_t *pcomp, int64_t h0, int64_t h1,
                         int poisson, double *out, int32_t *cb0, double *sb0, const double *lt,
                         int ltP, cudaStream_t s) {
  if (h1 <= h0) return RCB_OK;
  const size_t smem = ps3d_tile_smem(R, nball);
  static bool attr_set[64] = {};
  int dev = 0;
  RCB_CUDA(cudaGetDevice(&dev));
  if (dev < 64 && !attr_set[dev]) {
    RCB_CUDA(cudaFuncSetAttribute(k_delta_ps3d_tile, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  200 * 1024));
    attr_set[dev] = true;
  }
  dim3 grid((unsigned)((lat.nx + kTileT - 1) / kTileT), (unsigned)((lat.ny + kTileT - 1) / kTileT),
            (unsigned)((lat.nz + kTileT - 1) / kTileT));
  k_delta_ps3d_tile<<<grid, 128, smem, s>>>(L, I, Cown, Sown, rho0, (int)lat.nx, (int)lat.ny,
                                            (int)lat.nz, R, ball, nball, site_off, px, pown, pcomp,
                                            h0, h1, poisson, out, cb0, sb0, lt, ltP);
  RCB_CUDA(cudaGetLastError());
  return RCB_OK;
}

// whether delta_ps_batch's kernel for this lattice writes K6's packed records
bool delta_ps_writes_pk(const Lat &lat, int nball) {
  return nball <= kPsMaxBall && lat.V < ((int64_t)1 << 31);
}

int32_t delta_ps_batch(const int32_t *L, const double *I, const int32_t *Cown, const double *Sown,
                       const Lat &lat, const Off *ball, int nball, const uint32_t *px,
                       const int32_t *pown, const int32_t *pcomp, int64_t n, int poisson,
                       double *out, cudaStream_t s, const double *rho0, int32_t *cb0,
                       double *sb0, const double *lt, int ltP, int4 *pk) {
  if (n == 0) return RCB_OK;
  if (lat.ndim == 2 && nball <= kPsMaxBall && lat.V < ((int64_t)1 << 31))
    k_delta_ps2d<<<grid_for(n, 128), 128, 0, s>>>(L, I, Cown, Sown, (int)lat.nx, (int)lat.ny, ball,
                                                  nball, px, pown, pcomp, n, poisson, out, rho0,
                                                  cb0, sb0, lt, ltP, pk);
  else if (lat.ndim == 3 && nball <= kPsMaxBall && lat.V < ((int64_t)1 << 31))
    k_delta_ps3d<<<grid_for(n, 128), 128, 0, s>>>(L, I, Cown, Sown, (int)lat.nx, (int)lat.ny,
                                                  (int)lat.nz, ball, nball, px, pown, pcomp, n,
                                                  poisson, out, rho0, cb0, sb0, lt, ltP, pk);
  else
    k_delta_ps<<<grid_for(n, 128), 128, 0, s>>>(L, I, Cown, Sown, lat, ball, nball, px, pown,
                                                pcomp, n, poisson, out, rho0, cb0, sb0);
  RCB_CUDA(cudaGetLastError());
  return RCB_OK;
}

// ---------------------------------------------------------------------------
// K2 — region statistics in raster order (grid.py:155-169; Appendix B8).
// np.bincount accumulates sequentially in raster order, so each label's sum
// is one ordered fp64 chain.  A stable radix sort by label gives every
// label's sites in raster order; one warp per label then gathers 32 values
// at a time and all lanes replay the ordered chain on broadcast values.
// ---------------------------------------------------------------------------
__global__ void k_iota(uint32_t *__restrict__ v, int64_t n) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    v[i] = (uint32_t)i;
}

__global__ void k_seg_bounds(const uint32_t *__restrict__ keys, int64_t n,
                             int64_t *__restrict__ start, int64_t *__restrict__ end) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    uint32_t k = keys[i];
    if (i == 0 || keys[i - 1] != k) start[k] = i;
    if (i == n - 1 || keys[i + 1] != k) end[k] = i + 1;
  }
}

__global__ void k_gather_vals(const uint32_t *__restrict__ sites, const double *__restrict__ I,
                              int64_t n, double *__restrict__ out) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = __ldg(&I[sites[i]]);
}

// Per label (blockIdx.x = 2 * label + which): the raster-order fp64 sum of the
// label's values (which = 0) or of their squares (which = 1), replayed exactly
// by OrderedSum; the count is the segment length.
// Integer fast path of k_seq_sums, for all labels at once (the label-sorted
// values split over the whole grid instead of one block per label): per
// (label, which) the int64 sum, the max |addend| and whether every addend is
// an integer of magnitude <= 2^52.  Warps whose lanes share one label
// (sorted input: nearly all) reduce first and issue one atomic each.
__global__ void k_int_sums(const double *__restrict__ vals, const uint32_t *__restrict__ keys,
                           int64_t V, long long *__restrict__ isum,
                           unsigned long long *__restrict__ vmax, int *__restrict__ notint) {
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < V; base += stride) {
    const int64_t i = base + threadIdx.x;
    const bool in = i < V;
    const uint32_t l = in ? keys[i] : 0xffffffffu;
    const double v0 = in ? vals[i] : 0.0;
    const uint32_t l0 = __shfl_sync(0xffffffffu, l, 0);
    const bool uni = __all_sync(0xffffffffu, !in || l == l0);
    for (int which = 0; which < 2; ++which) {
      const double v = which ? v0 * v0 : v0;
      const double av = fabs(v);
      const bool ok = !in || (av <= 4503599627370496.0 && v == rint(v));
      long long a = (in && ok) ? (long long)v : 0;
      unsigned long long m = in ? (unsigned long long)__double_as_longlong(av) : 0ull;
      if (uni) {
        for (int o = 16; o; o >>= 1) {
          a += __shfl_xor_sync(0xffffffffu, a, o);
          const unsigned long long m2 = __shfl_xor_sync(0xffffffffu, m, o);
          m = m2 > m ? m2 : m;
        }
        const bool bad = __any_sync(0xffffffffu, !ok);
        if (lane == 0 && l0 != 0xffffffffu) {
          atomicAdd((unsigned long long *)&isum[2 * l0 + which], (unsigned long long)a);
          atomicMax(&vmax[2 * l0 + which], m);
          if (bad) atomicOr(&notint[2 * l0 + which], 1);
        }
      } else if (in) {
        atomicAdd((unsigned long long *)&isum[2 * l + which], (unsigned long long)a);
        atomicMax(&vmax[2 * l + which], m);
        if (!ok) atomicOr(&notint[2 * l + which], 1);
      }
    }
  }
}

__global__ void __launch_bounds__(512) k_seq_sums(const double *__restrict__ vals,
                                                  const int64_t *__restrict__ start,
                                                  const int64_t *__restrict__ end, int32_t nl,
                                                  int64_t *__restrict__ cnt,
                                                  double *__restrict__ tot,
                                                  double *__restrict__ tsq,
                                                  const long long *__restrict__ isum_g,
                                                  const unsigned long long *__restrict__ vmax_g,
                                                  const int *__restrict__ notint_g) {
  typedef OrderedSum<512> OS;
  __shared__ typename OS::Temp T;
  const int32_t l = blockIdx.x >> 1;
  const int which = blockIdx.x & 1;
  const int64_t s = start[l], n = end[l] - s;
  if (isum_g) {  // the grid-wide integer pre-pass (k_int_sums) decided it
    const double vm = __longlong_as_double((long long)vmax_g[2 * l + which]);
    if (!notint_g[2 * l + which] && (double)n * vm < 9007199254740992.0) {
      if (threadIdx.x == 0) {
        if (which) {
          tsq[l] = (double)isum_g[2 * l + which];
        } else {
          tot[l] = (double)isum_g[2 * l + which];
          cnt[l] = n;
        }
      }
      return;
    }
  }
  // Exact fast path for integer data (Poisson counts): if every addend is an
  // integer and n * max|addend| < 2^53, every partial sum of the sequential
  // chain from 0 is an exactly representable integer, so each fl() is exact
  // and the chain's result is the integer sum, in any order.
  {
    typedef cub::BlockReduce<long long, 512> RedL;
    typedef cub::BlockReduce<double, 512> RedD;
    __shared__ union {
      typename RedL::TempStorage l;
      typename RedD::TempStorage d;
    } tr;
    __shared__ long long isum;
    __shared__ double vmax;
    __shared__ int allint;
    if (threadIdx.x == 0) allint = 1;
    __syncthreads();
    long long acc = 0;
    double mx = 0.0;
    bool ok = true;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
      const double v0 = vals[s + i];
      const double v = which ? v0 * v0 : v0;
      const double av = fabs(v);
      ok = ok && av <= 4503599627370496.0 && v == rint(v);  // |v| <= 2^52, integral
      if (ok) acc += (long long)v;
      mx = av > mx ? av : mx;
    }
    if (!ok) allint = 0;
    const long long tsum = RedL(tr.l).Sum(acc);
    if (threadIdx.x == 0) isum = tsum;
    __syncthreads();
    const double tmax = RedD(tr.d).Reduce(mx, cub::Max());
    if (threadIdx.x == 0) vmax = tmax;
    __syncthreads();
    if (allint && (double)n * vmax < 9007199254740992.0) {
      if (threadIdx.x == 0) {
        if (which) {
          tsq[l] = (double)isum;
        } else {
          tot[l] = (double)isum;
          cnt[l] = n;
        }
      }
      return;
    }
  }
  const double fin = OS::run(
      T, 0.0, (long long)n,
      [&](long long i) {
        const double v = vals[s + i];
        return which ? v * v : v;
      },
      [](long long, double) {});
  if (threadIdx.x == 0) {
    if (which) {
      tsq[l] = fin;
    } else {
      tot[l] = fin;
      cnt[l] = n;
    }
  }
}

int32_t stats_rebuild(const int32_t *L, const double *I, int64_t V, int32_t nl, int64_t *cnt,
                      double *tot, double *tsq, StatsScratch &sc, cudaStream_t s) {
  RCB_TRY(sc.keys.reserve(V, s));
  RCB_TRY(sc.vals_in.reserve(V, s));
  RCB_TRY(sc.vals.reserve(V, s));
  RCB_TRY(sc.bounds.reserve(2 * (size_t)nl, s));
  k_iota<<<grid_for(V, 256), 256, 0, s>>>(sc.vals_in.p, V);
  RCB_CUDA(cudaGetLastError());
  int end_bit = 1;
  while (end_bit < 32 && ((int64_t)1 << end_bit) < nl) ++end_bit;
  size_t bytes = 0;
  const uint32_t *keys_in = reinterpret_cast<const uint32_t *>(L);
  RCB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys_in, sc.keys.p, sc.vals_in.p,
                                           sc.vals.p, V, 0, end_bit, s));
  RCB_TRY(sc.tmp.reserve(bytes, s));
  RCB_CUDA(cub::DeviceRadixSort::SortPairs(sc.tmp.p, bytes, keys_in, sc.keys.p, sc.vals_in.p,
                                           sc.vals.p, V, 0, end_bit, s));
  int64_t *start = sc.bounds.p, *end = sc.bounds.p + nl;
  RCB_CUDA(cudaMemsetAsync(start, 0, sizeof(int64_t) * nl, s));
  RCB_CUDA(cudaMemsetAsync(end, 0, sizeof(int64_t) * nl, s));
  if (V > 0) {
    k_seg_bounds<<<grid_for(V, 256), 256, 0, s>>>(sc.keys.p, V, start, end);
    RCB_CUDA(cudaGetLastError());
  }
  RCB_TRY(sc.gathered.reserve(V, s));
  k_gather_vals<<<grid_for(V, 256), 256, 0, s>>>(sc.vals.p, I, V, sc.gathered.p);
  // integer fast path over the whole grid first (Poisson counts)
  RCB_TRY(sc.isum.reserve(2 * (size_t)nl, s));
  RCB_TRY(sc.imax.reserve(2 * (size_t)nl, s));
  RCB_TRY(sc.inot.reserve(2 * (size_t)nl, s));
  RCB_CUDA(cudaMemsetAsync(sc.isum.p, 0, sizeof(long long) * 2 * nl, s));
  RCB_CUDA(cudaMemsetAsync(sc.imax.p, 0, sizeof(unsigned long long) * 2 * nl, s));
  RCB_CUDA(cudaMemsetAsync(sc.inot.p, 0, sizeof(int) * 2 * nl, s));
  if (V > 0) {
    int64_t g = (V + 255) / 256;
    if (g > 148 * 16) g = 148 * 16;
    k_int_sums<<<(unsigned)g, 256, 0, s>>>(sc.gathered.p, sc.keys.p, V, sc.isum.p, sc.imax.p,
                                           sc.inot.p);
  }
  k_seq_sums<<<2 * nl, 512, 0, s>>>(sc.gathered.p, start, end, nl, cnt, tot, tsq, sc.isum.p,
                                    sc.imax.p, sc.inot.p);
  RCB_CUDA(cudaGetLastError());
  return RCB_OK;
}

// ---------------------------------------------------------------------------
// K9 — exact sums (math.fsum semantics) with a fixed-point superaccumulator.
// A double m*2^e (e >= -1074) is split into three 32-bit chunks added to
// int64 limbs of weight 2^(32k-1074); the host rounds the exact total once.
// ---------------------------------------------------------------------------
__global__ void k_pc_terms(const int64_t *__restrict__ cnt, const double *__restrict__ tot,
                           const double *__restrict__ tsq, int32_t nl, int poisson,
                           long long *__restrict__ limbs) {
  __shared__ long long sm[kLimbs];
  for (int k = threadIdx.x; k < kLimbs; k += blockDim.x) sm[k] = 0;
  __syncthreads();
  for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < nl; l += gridDim.x * blockDim.x) {
    double n = (double)cnt[l];
    double g = poisson ? g_poisson(n, tot[l]) : g_gauss(n, tot[l], tsq[l]);
    acc_add(sm, g);
  }
  acc_flush(sm, limbs);
}

__global__ void k_ps_terms(const int32_t *__restrict__ Cown, const double *__restrict__ Sown,
                           const double *__restrict__ I, int64_t V, int poisson,
                           long long *__restrict__ limbs) {
  __shared__ long long sm[kLimbs];
  for (int k = threadIdx.x; k < kLimbs; k += blockDim.x) sm[k] = 0;
  __syncthreads();
  // warp-uniform loop: the limb adds are aggregated per warp (acc_add_warp)
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < V; base += stride) {
    const int64_t f = base + threadIdx.x;
    const bool in = f < V;
    acc_add_warp(sm, in ? rho(I[f], Sown[f] / (double)Cown[f], poisson) : 0.0, in);
  }
  acc_flush(sm, limbs);
}

__global__ void k_perimeter(const int32_t *__restrict__ L, Lat lat,
                            unsigned long long *__restrict__ out) {
  unsigned long long c = 0;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < lat.V; f += stride) {
    int64_t z, y, x;
    lat.coord(f, z, y, x);
    int32_t l = L[f];
    if (x + 1 < lat.nx) c += L[f + 1] != l;
    if (y + 1 < lat.ny) c += L[f + lat.nx] != l;
    if (z + 1 < lat.nz) c += L[f + lat.nx * lat.ny] != l;
  }
  for (int o = 16; o; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

int32_t pc_terms_exact(const int64_t *cnt, const double *tot, const double *tsq, int32_t nl,
                       int poisson, long long *limbs, cudaStream_t s) {
  RCB_CUDA(cudaMemsetAsync(limbs, 0, sizeof(long long) * kLimbs, s));
  k_pc_terms<<<grid_for(nl, 256), 256, 0, s>>>(cnt, tot, tsq, nl, poisson, limbs);
  RCB_CUDA(cudaGetLastError());
  return RCB_OK;
}

int32_t ps_terms_exact(const int32_t *Cown, const double *Sown, const double *I, int64_t V,
                       int poisson, long long *limbs, cudaStream_t s) {
  RCB_CUDA(cudaMemsetAsync(limbs, 0, sizeof(long long) * kLimbs, s));
  unsigned g = grid_for(V, 256);
  if (g > 148 * 16) g = 148 * 16;
  k_ps_terms<<<g, 256, 0, s>>>(Cown, Sown, I, V, poisson, limbs);
  RCB_CUDA(cudaGetLastError());
  return RCB_OK;
}

int32_t perimeter(const int32_t *L, const Lat &lat, unsigned long long *out, cudaStream_t s) {
  RCB_CUDA(cudaMemsetAsync(out, 0, sizeof(unsigned long long), s));
  unsigned g = grid_for(lat.V, 256);
  if (g > 148 * 16) g = 148 * 16;
  k_perimeter<<<g, 256, 0, s>>>(L, lat, out);
  RCB_CUDA(cudaGetLastError());
  return RCB_OK;
}

// Correctly rounded (nearest-even) value of the limb total, as math.fsum.
double limbs_to_double(const long long *limbs) {
  // carry-normalise into 32-bit digits (two's complement), then take |.|
  const int ND = kLimbs + 3;
  uint32_t dig[ND];
  long long carry = 0;
  for (int k = 0; k < ND; ++k) {
    long long t = (k < kLimbs ? limbs[k] : 0) + carry;
    dig[k] = (uint32_t)(t & 0xffffffffll);
    carry = t >> 32;  // arithmetic shift
  }
  bool neg = carry < 0;
  if (neg) {  // negate the ND-digit two's complement number
    uint64_t c = 1;
    for (int k = 0; k < ND; ++k) {
      uint64_t t = (uint64_t)(uint32_t)~dig[k] + c;
      dig[k] = (uint32_t)t;
      c = t >> 32;
    }
  }
  int top = -1;
  for (int k = ND - 1; k >= 0; --k)
    if (dig[k]) {
      top = k * 32 + (31 - __builtin_clz(dig[k]));
      break;
    }
  if (top < 0) return 0.0;
  auto bit = [&](int p) -> uint64_t { return p < 0 ? 0 : (dig[p >> 5] >> (p & 31)) & 1u; };
  uint64_t m = 0;
  int shift = top >= 52 ? top - 52 : 0;
  for (int p = top; p >= shift; --p) m = (m << 1) | bit(p);
  if (shift > 0) {
    uint64_t g = bit(shift - 1);
    bool sticky = false;
    for (int p = shift - 2; p >= 0 && !sticky; --p) sticky = bit(p) != 0;
    if (g && (sticky || (m & 1))) {
      ++m;
      if (m == (1ull << 53)) {
        m >>= 1;
        ++shift;
      }
    }
  }
  double r = ldexp((double)m, shift - 1074);
  return neg ? -r : r;
}


// ---------------------------------------------------------------------------
// Input validation of the engine (grid.py:24-39, optimizer.py:100-101): label
// min / max, intensity min and non-finite count in one reduction pass.
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long dkey(double v) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(v);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

__global__ void k_check_inputs(const int32_t *__restrict__ L, const double *__restrict__ I,
                               int64_t V, int *lmin, int *lmax, unsigned long long *imin,
                               unsigned long long *nonfin, unsigned long long *imax,
                               unsigned long long *nonint) {
  int lo = INT_MAX, hi = INT_MIN;
  unsigned long long dm = ~0ull, nf = 0, dx = 0, ni = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < V; i += stride) {
    const int l = L[i];
    lo = l < lo ? l : lo;
    hi = l > hi ? l : hi;
    const double v = I[i];
    if (!isfinite(v)) {
      ++nf;
    } else {
      const unsigned long long k = dkey(v);
      dm = k < dm ? k : dm;
      dx = k > dx ? k : dx;
      if (v != rint(v)) ++ni;
    }
  }
  for (int o = 16; o; o >>= 1) {
    lo = min(lo, __shfl_down_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_down_sync(0xffffffffu, hi, o));
    const unsigned long long d2 = __shfl_down_sync(0xffffffffu, dm, o);
    dm = d2 < dm ? d2 : dm;
    const unsigned long long x2 = __shfl_down_sync(0xffffffffu, dx, o);
    dx = x2 > dx ? x2 : dx;
    nf += __shfl_down_sync(0xffffffffu, nf, o);
    ni += __shfl_down_sync(0xffffffffu, ni, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(lmin, lo);
    atomicMax(lmax, hi);
    atomicMin(imin, dm);
    atomicMax(imax, dx);
    if (nf) atomicAdd(nonfin, nf);
    if (ni) atomicAdd(nonint, ni);
  }
}

int32_t check_inputs(const int32_t *L, const double *I, int64_t V, InputCheck *out,
                     cudaStream_t s) {
  struct Dev {
    int lmin, lmax;
    unsigned long long imin, nonfin, imax, nonint;
  };
  static thread_local Dev *hbuf = nullptr;  // pinned, reused
  if (!hbuf) RCB_CUDA(cudaMallocHost((void **)&hbuf, sizeof(Dev)));
  Dev *d = nullptr;
  RCB_CUDA(cudaMallocAsync((void **)&d, sizeof(Dev), s));
  const Dev init{INT_MAX, INT_MIN, ~0ull, 0ull, 0ull, 0ull};
  *hbuf = init;
  RCB_CUDA(cudaMemcpyAsync(d, hbuf, sizeof(Dev), cudaMemcpyHostToDevice, s));
  int64_t g = (V + 255) / 256;
  if (g > 148 * 8) g = 148 * 8;
  if (g < 1) g = 1;
  k_check_inputs<<<(unsigned)g, 256, 0, s>>>(L, I, V, &d->lmin, &d->lmax, &d->imin, &d->nonfin,
                                              &d->imax, &d->nonint);
  RCB_CUDA(cudaGetLastError());
  RCB_CUDA(cudaMemcpyAsync(hbuf, d, sizeof(Dev), cudaMemcpyDeviceToHost, s));
  RCB_CUDA(cudaFreeAsync(d, s));
  RCB_CUDA(cudaStreamSynchronize(s));
  out->label_min = V ? hbuf->lmin : 0;
  out->label_max = V ? hbuf->lmax : 0;
  out->nonfinite = (int64_t)hbuf->nonfin;
  const unsigned long long k = hbuf->imin;
  const unsigned long long u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  double v;
  memcpy(&v, &u, sizeof(v));
  out->image_min = (k == ~0ull) ? 0.0 : v;
  {
    const unsigned long long kx = hbuf->imax;
    const unsigned long long ux = (kx >> 63) ? (kx & 0x7fffffffffffffffull) : ~kx;
    double vx;
    memcpy(&vx, &ux, sizeof(vx));
    out->image_max = (kx == 0ull) ? 0.0 : vx;
  }
  out->nonint = (int64_t)hbuf->nonint;
  return RCB_OK;
}

// Poisson log table (K5, integer images): lt[q * P + p] = log(max(p / q,
// 1e-8)) for 1 <= q < Q, 0 <= p < P -- the exact value rho() computes for
// theta = fl(p / q) (energy.py:226-230), so a lookup replaces the per-hit
// log without changing a bit.
__global__ void k_log_table(double *__restrict__ lt, int P, int Q) {
  const int64_t n = (int64_t)P * Q;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int q = (int)(i / P), p = (int)(i - (int64_t)q * P);
    if (q == 0) {
      lt[i] = 0.0;
      continue;
    }
    const double theta = (double)p / (double)q;
    const double t = theta < kPoissonFloor ? kPoissonFloor : theta;
    lt[i] = log(t);
  }
}

int32_t log_table(double *lt, int P, int Q, cudaStream_t s) {
  k_log_table<<<148 * 8, 256, 0, s>>>(lt, P, Q);
  RCB_CUDA(cudaGetLastError());
  return RCB_OK;
}


// ---------------------------------------------------------------------------
// K5 over packed site records (integer Poisson images).  Every ball hit of
// k_delta_ps2d/3d gathers five arrays (L, Cown, Sown, I, rho0: 32 B from five
// cache lines); here one 16-byte record per site carries all of them:
//   x = label (16 bits) | Cown << 16,  y = Sown (20 bits) | I << 20,
//   z:w = rho0 (fp64 bits),
// exact for labels, counts < 2^16, integer intensities < 2^12 and ball sums
// < 2^20 (checked on the host, rec_ok).  theta = fl(p / q) and its log come
// from one 16-byte table entry (no per-hit division or log), so every term
// is the same fp64 value k_delta_ps3d forms, summed in the same ball-offset
// order: bit-identical results.
// ---------------------------------------------------------------------------
__global__ void k_pack_sites(const int32_t *__restrict__ L, const int32_t *__restrict__ Cown,
                             const double *__restrict__ Sown, const double *__restrict__ I,
                             const double *__restrict__ rho0, int64_t V, int4 *__restrict__ rec) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < V; f += stride) {
    const unsigned long long r = (unsigned long long)__double_as_longlong(__ldg(rho0 + f));
    const uint32_t w0 = (uint32_t)__ldg(L + f) | ((uint32_t)__ldg(Cown + f) << 16);
    const uint32_t w1 = (uint32_t)__ldg(Sown + f) | ((uint32_t)__ldg(I + f) << 20);
    __stcs(rec + f, make_int4((int)w0, (int)w1, (int)(uint32_t)r, (int)(uint32_t)(r >> 32)));
  }
}

// tl[q * P + p] = {fl(p / q), log(max(fl(p / q), 1e-8))} for 1 <= q < Q
__global__ void k_theta_table(double2 *__restrict__ tl, int P, int Q) {
  const int64_t n = (int64_t)P * Q;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int q = (int)(i / P), p = (int)(i - (int64_t)q * P);
    if (q == 0) {
      tl[i] = make_double2(0.0, 0.0);
      continue;
    }
    const double theta = (double)p / (double)q;
    const double t = theta < kPoissonFloor ? kPoissonFloor : theta;
    tl[i] = make_double2(theta, log(t));
  }
}

template <int ND>
__global__ void __launch_bounds__(128, 6) k_delta_ps_rec(
    const int4 *__restrict__ rec, const double *__restrict__ I, int nx, int ny, int nz,
    const Off *__restrict__ ball, int nball, const uint32_t *__restrict__ px,
    const int32_t *__restrict__ pown, const int32_t *__restrict__ pcomp, int64_t n,
    double *__restrict__ out, const double *__restrict__ rho0, int32_t *__restrict__ cb0,
    double *__restrict__ sb0, const double2 *__restrict__ tl, int tlP, int4 *__restrict__ pk) {
  __shared__ int sofs[kPsMaxBall];  // dz:8 | dy:8 | dx:8, signed, packed
  __shared__ int sdel[kPsMaxBall];  // linear site delta of each offset
  __shared__ int srad;
  if (threadIdx.x == 0) srad = 0;
  __syncthreads();
  for (int k = threadIdx.x; k < nball; k += blockDim.x) {
    const int dz = ND == 3 ? ball[k].dz : 0, dy = ball[k].dy, dx = ball[k].dx;
    sofs[k] = ((int)(uint8_t)dz << 16) | ((int)(uint8_t)dy << 8) | (int)(uint8_t)dx;
    sdel[k] = (dz * ny + dy) * nx + dx;
    atomicMax(&srad, max(abs(dz), max(abs(dy), abs(dx))));
  }
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int f = (int)px[i];
  const int plane = nx * ny;
  const int z = ND == 3 ? f / plane : 0, r = f - z * plane;
  const int y = r / nx, x = r - y * nx;
  const int32_t a = pown[i], b = pcomp[i];
  const double v = I[f];
  const int iv = (int)v;
  const int rad = srad;
  const bool interior = (ND == 2 || (z >= rad && z < nz - rad)) && y >= rad && y < ny - rad &&
                        x >= rad && x < nx - rad;
  double acc_a = 0.0, acc_b = 0.0, sb = 0.0;
  int32_t cb = 0;
  constexpr int U = 4;
  for (int k0 = 0; k0 < nball; k0 += U) {
    int4 q[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = k0 + u;
      bool ok;
      int g;
      if (interior) {
        ok = k < nball;
        g = f + (ok ? sdel[k] : 0);
      } else {
        const int o = k < nball ? sofs[k] : 0;
        const int zz = z + (int)(int8_t)(o >> 16), yy = y + (int)(int8_t)(o >> 8),
                  xx = x + (int)(int8_t)o;
        ok = k < nball && (ND == 2 || (unsigned)zz < (unsigned)nz) && (unsigned)yy < (unsigned)ny &&
             (unsigned)xx < (unsigned)nx;
        g = ok ? (zz * ny + yy) * nx + xx : f;
      }
      q[u] = __ldg(rec + g);
      if (!ok) q[u].x = -1;
    }
    double2 t2[U];
    int lab[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      lab[u] = q[u].x < 0 ? -1 : (q[u].x & 0xffff);
      const bool isa = lab[u] == a, hit = isa || lab[u] == b;
      const int c = (int)((uint32_t)q[u].x >> 16), sv = q[u].y & 0xfffff;
      // (S - v) / (C - 1) for the donor side, (S + v) / (C + 1) for the target
      const int num = isa ? sv - iv : sv + iv, den = isa ? c - 1 : c + 1;
      t2[u] = (hit && den >= 1) ? __ldg(tl + (int64_t)den * tlP + num) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool isa = lab[u] == a;
      if (isa || lab[u] == b) {
        const double iy = (double)((uint32_t)q[u].y >> 20);
        const double r0 = __longlong_as_double(((long long)(uint32_t)q[u].w << 32) |
                                               (long long)(uint32_t)q[u].z);
        double rn;
        const int c = (int)((uint32_t)q[u].x >> 16);
        if ((isa ? c - 1 : c + 1) >= 1) {
          rn = t2[u].x - iy * t2[u].y;
        } else {  // den == 0: theta = +-inf / nan, as numpy forms it
          const double sy = (double)(q[u].y & 0xfffff);
          const double num = sy + (isa ? -v : v), den = (double)c + (isa ? -1.0 : 1.0);
          rn = rho(iy, num / den, 1);
        }
        const double t = rn - r0;
        if (isa) {
          acc_a += t;
        } else {
          acc_b += t;
          cb += 1;
          sb += iy;
        }
      }
    }
  }
  double d = 0.0 + acc_a;
  d = d + acc_b;
  d += rho(v, (sb + v) / ((double)cb + 1.0), 1);
  d -= rho0[f];
  out[i] = d;
  if (pk) pk[i] = pack_record(d, (uint32_t)f, a, b);
  if (cb0) {
    cb0[i] = cb;
    sb0[i] = sb;
  }
}

// whether the packed-record K5 applies: integer Poisson intensities in
// [0, 2^12), labels and ball counts < 2^16, ball sums < 2^20, 32-bit sites
bool ps_rec_ok(const Lat &lat, int nball_full, int32_t nl, double image_max) {
  return nball_full < kPsMaxBall && nl < 65536 && image_max < 4096.0 &&
         (double)(nball_full + 1) * image_max < (double)(1 << 20) && lat.V < ((int64_t)1 << 31) &&
         (lat.ndim == 2 || lat.ndim == 3);
}

int32_t pack_sites(const int32_t *L, const int32_t *Cown, const double *Sown, const double *I,
                   const double *rho0, int64_t V, int4 *rec, cudaStream_t s) {
  k_pack_sites<<<148 * 16, 256, 0, s>>>(L, Cown, Sown, I, rho0, V, rec);
  RCB_CUDA(cudaGetLastError());
  return RCB_OK;
}

int32_t theta_table(double2 *tl, int P, int Q, cudaStream_t s) {
  k_theta_table<<<148 * 8, 256, 0, s>>>(tl, P, Q);
  RCB_CUDA(cudaGetLastError());
  return RCB_OK;
}

int32_t delta_ps_rec(const int4 *rec, const double *I, const Lat &lat, const Off *ball, int nball,
                     const uint32_t *px, const int32_t *pown, const int32_t *pcomp, int64_t n,
                     double *out, const double *rho0, int32_t *cb0, double *sb0,
                     const double2 *tl, int tlP, int4 *pk, cudaStream_t s) {
  if (n == 0) return RCB_OK;
  if (lat.ndim == 3)
    k_delta_ps_rec<3><<<grid_for(n, 128), 128, 0, s>>>(rec, I, (int)lat.nx, (int)lat.ny,
                                                       (int)lat.nz, ball, nball, px, pown, pcomp, n,
                                                       out, rho0, cb0, sb0, tl, tlP, pk);
  else
    k_delta_ps_rec<2><<<grid_for(n, 128), 128, 0, s>>>(rec, I, (int)lat.nx, (int)lat.ny, 1, ball,
                                                       nball, px, pown, pcomp, n, out, rho0, cb0,
                                                       sb0, tl, tlP, pk);
  RCB_CUDA(cudaGetLastError());
  return RCB_OK;
}

}  // namespace rcb
