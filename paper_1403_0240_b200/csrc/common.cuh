// Shared device/host helpers for librcseg_b200 (sm_100a).
//
// Lattice convention: every raster is handled as 3-D (nz, ny, nx) in C order;
// a 2-D raster is nz = 1.  Offsets are always walked in lexicographic
// (dz, dy, dx) order, which is the reference's meshgrid(indexing="ij") order
// (grid.py:42-54, sobolev.py:125-130), so 2-D offset (dy, dx) == (0, dy, dx).
//
// fp64 parity: every translation unit is compiled with -fmad=false, so
// a*b+c is two IEEE roundings exactly as numpy evaluates it.
#pragma once
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/rcb.h"

namespace rcb {

struct Lat {
  int32_t ndim;
  int64_t nz, ny, nx;
  int64_t V;
  __host__ __device__ inline int64_t flat(int64_t z, int64_t y, int64_t x) const {
    return (z * ny + y) * nx + x;
  }
  __host__ __device__ inline void coord(int64_t f, int64_t &z, int64_t &y, int64_t &x) const {
    x = f % nx;
    int64_t t = f / nx;
    y = t % ny;
    z = t / ny;
  }
  __host__ __device__ inline bool inb(int64_t z, int64_t y, int64_t x) const {
    return z >= 0 && z < nz && y >= 0 && y < ny && x >= 0 && x < nx;
  }
};

inline Lat make_lat(int32_t ndim, const int64_t *dims) {
  Lat l;
  l.ndim = ndim;
  if (ndim == 2) {
    l.nz = 1;
    l.ny = dims[0];
    l.nx = dims[1];
  } else {
    l.nz = dims[0];
    l.ny = dims[1];
    l.nx = dims[2];
  }
  l.V = l.nz * l.ny * l.nx;
  return l;
}

// packed lattice offset: three signed bytes (dz, dy, dx) + one unsigned byte
// spare (used for |off|^2 where it fits).
struct Off {
  int8_t dz, dy, dx;
  uint8_t aux;
};

// ---- error plumbing ------------------------------------------------------
void set_error(const std::string &msg);
int32_t fail(int32_t code, const std::string &msg);

#define RCB_CUDA(call)                                                              \
  do {                                                                              \
    cudaError_t _e = (call);                                                        \
    if (_e != cudaSuccess)                                                          \
      return ::rcb::fail(RCB_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(_e)); \
  } while (0)

#define RCB_TRY(call)              \
  do {                             \
    int32_t _s = (call);           \
    if (_s != RCB_OK) return _s;   \
  } while (0)

static constexpr int kLimbs = 68;  // superaccumulator limbs of 32 bits from 2^-1074

// ---- device memory: stream-ordered buffers --------------------------------
template <typename T>
struct DBuf {
  T *p = nullptr;
  size_t cap = 0;  // elements
  int32_t reserve(size_t n, cudaStream_t s) {
    if (n <= cap) return RCB_OK;
    const auto t0 = std::chrono::steady_clock::now();
    if (p) cudaFreeAsync(p, s);
    // first allocation: 25 % slack (lattice-sized buffers never grow, and 2x
    // slack on ~30 of them cost ~30 GB at 512^3, pushing the pool past its
    // primed reservation into slow fresh mappings); growth after that is
    // geometric: particle counts climb for tens of iterations
    size_t want = cap == 0 ? n + n / 4 + 64 : 2 * n + 64;
    cudaError_t e = cudaMallocAsync((void **)&p, want * sizeof(T), s);
    if (getenv("RCB_ALLOC_LOG")) {
      const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
      uint64_t res = 0, used = 0;
      cudaMemPool_t pool;
      int dev = 0;
      if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &res);
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
      }
      fprintf(stderr, "[rcb-alloc] %zu bytes %.1f us pool reserved %.2f GB used %.2f GB\n",
              want * sizeof(T), us, res / 1e9, used / 1e9);
    }
    if (e != cudaSuccess) {
      p = nullptr;
      cap = 0;
      return fail(RCB_ERR_CUDA, std::string("cudaMallocAsync: ") + cudaGetErrorString(e));
    }
    cap = want;
    return RCB_OK;
  }
  void release(cudaStream_t s) {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    cap = 0;
  }
};

inline unsigned grid_for(int64_t n, int threads) {
  int64_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > 0x7fffffff) g = 0x7fffffff;
  return (unsigned)g;
}

// ---- host-side tables ------------------------------------------------------
// Lexicographic box offsets of radius r, optionally filtered by |off|^2.
std::vector<Off> box_offsets(int ndim, int r);

}  // namespace rcb
