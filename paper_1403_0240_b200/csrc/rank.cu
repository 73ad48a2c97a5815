// K7 — rank composition, tie keys and the acceptance order
// (optimizer.py:80-87 _tie_keys, :135-147 rank + np.lexsort).
//
// lexsort((comps, xs, ties, rank)) == a stable sort by tie followed by a
// stable sort by rank, starting from the (x, comp) particle order that K1
// already produces.  Non-negative ranks are never executed
// (optimizer.py:170-171), so they are keyed to the end and the acceptance
// walk stops at the first of them.
#include <cub/device/device_radix_sort.cuh>

#include "dev.cuh"
#include "kernels.h"

namespace rcb {

__global__ void k_rank(const double *__restrict__ base, const int32_t *__restrict__ dint,
                       double lam, int64_t n, const uint32_t *__restrict__ px,
                       const int32_t *__restrict__ pcomp, uint64_t seed, double *__restrict__ rank,
                       uint64_t *__restrict__ tie, uint64_t *__restrict__ rkey,
                       uint32_t *__restrict__ idx, unsigned long long *__restrict__ nneg) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool neg = false;
  if (i < n) {
    double r = base[i] + lam * (double)dint[i];
    rank[i] = r;
    neg = r < 0.0;
    tie[i] = tie_key((uint64_t)px[i], (uint64_t)(int64_t)pcomp[i], seed);
    rkey[i] = neg ? double_key(r) : ~0ull;
    idx[i] = (uint32_t)i;
  }
  unsigned m = __ballot_sync(0xffffffffu, neg);
  if ((threadIdx.x & 31) == 0 && m) atomicAdd(nneg, (unsigned long long)__popc(m));
}

int32_t rank_order(const double *base, const int32_t *dint, double lam, int64_t n,
                   const uint32_t *px, const int32_t *pcomp, uint64_t seed, double *rank,
                   RankScratch &sc, uint32_t *order, unsigned long long *nneg, cudaStream_t s) {
  RCB_CUDA(cudaMemsetAsync(nneg, 0, sizeof(unsigned long long), s));
  if (n == 0) return RCB_OK;
  RCB_TRY(sc.tie.reserve(n, s));
  RCB_TRY(sc.tie2.reserve(n, s));
  RCB_TRY(sc.rkey.reserve(n, s));
  RCB_TRY(sc.rkey2.reserve(n, s));
  RCB_TRY(sc.idx.reserve(n, s));
  RCB_TRY(sc.idx2.reserve(n, s));
  k_rank<<<grid_for(n, 256), 256, 0, s>>>(base, dint, lam, n, px, pcomp, seed, rank, sc.tie.p,
                                          sc.rkey.p, sc.idx.p, nneg);
  RCB_CUDA(cudaGetLastError());
  // pass 1: stable by tie (carry the rank key along as the value's payload)
  size_t b = 0;
  RCB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, b, sc.tie.p, sc.tie2.p, sc.idx.p, sc.idx2.p, n,
                                           0, 64, s));
  RCB_TRY(sc.tmp.reserve(b, s));
  RCB_CUDA(cub::DeviceRadixSort::SortPairs(sc.tmp.p, b, sc.tie.p, sc.tie2.p, sc.idx.p, sc.idx2.p,
                                           n, 0, 64, s));
  // pass 2: stable by rank key of the tie-ordered particles
  gather_u64(sc.rkey.p, sc.idx2.p, n, sc.rkey2.p, s);
  RCB_CUDA(cub::DeviceRadixSort::SortPairs(sc.tmp.p, b, sc.rkey2.p, sc.rkey.p, sc.idx2.p, order, n,
                                           0, 64, s));
  return RCB_OK;
}

__global__ void k_gather_u64(const uint64_t *__restrict__ src, const uint32_t *__restrict__ idx,
                             int64_t n, uint64_t *__restrict__ dst) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[idx[i]];
}

void gather_u64(const uint64_t *src, const uint32_t *idx, int64_t n, uint64_t *dst,
                cudaStream_t s) {
  k_gather_u64<<<grid_for(n, 256), 256, 0, s>>>(src, idx, n, dst);
}

}  // namespace rcb
