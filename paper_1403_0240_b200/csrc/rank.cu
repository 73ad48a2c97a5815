// K7 — rank composition, tie keys and the acceptance order
// (optimizer.py:80-87 _tie_keys, :135-147 rank + np.lexsort).
//
// lexsort((comps, xs, ties, rank)) orders by rank, then tie, then particle
// (x, comp) order, which K1 already produces: one stable radix sort by rank
// from particle order, then each run of equal ranks (exact ties are rare) is
// ordered by (tie, particle).  Non-negative ranks are never executed
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

// The radix sort orders by the top 32 bits of the rank key only (4 digit
// passes instead of 8: sign, exponent and 20 mantissa bits, so keys that
// share them are rare -- equal to ~1e-6 relative).  Each run of equal top
// halves, left in particle order by the stable sort, is then put in (full
// rank key, tie key, particle index) order -- the complete lexsort order.
// Short runs: insertion sort by the thread that finds the run; long runs
// (degenerate inputs, e.g. exact ties on noise-free or integer images): a
// block bitonic sort in shared memory, or for runs beyond its capacity a
// block merge sort through global scratch (O(len log^2 len / threads)).
static constexpr int kShortRun = 32, kBitonic = 4096;

__device__ __forceinline__ bool tie_less(const uint64_t *tie, uint32_t p, uint32_t q) {
  const uint64_t a = tie[p], b = tie[q];
  return a < b || (a == b && p < q);
}
__device__ __forceinline__ bool rank_less(const uint64_t *rkey, const uint64_t *tie, uint32_t p,
                                          uint32_t q) {
  const uint64_t a = rkey[p], b = rkey[q];
  return a < b || (a == b && tie_less(tie, p, q));
}

__device__ void insertion_by_tie(uint32_t *o, int64_t len, const uint64_t *rkey,
                                 const uint64_t *tie) {
  for (int64_t i = 1; i < len; ++i) {
    const uint32_t v = o[i];
    int64_t j = i - 1;
    while (j >= 0 && rank_less(rkey, tie, v, o[j])) {
      o[j + 1] = o[j];
      --j;
    }
    o[j + 1] = v;
  }
}

__global__ void k_tie_runs(const uint64_t *__restrict__ key, int64_t n, uint32_t *__restrict__ order,
                           const uint64_t *__restrict__ rkey, const uint64_t *__restrict__ tie,
                           int64_t *__restrict__ longs, unsigned long long *__restrict__ nlong) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t k = (uint32_t)(key[i] >> 32);  // the sorted half
  if (k == 0xffffffffu) return;                          // non-negative ranks: never executed
  if (i > 0 && (uint32_t)(key[i - 1] >> 32) == k) return;  // not a run start
  if (i + 1 >= n || (uint32_t)(key[i + 1] >> 32) != k) return;  // run of one
  int64_t e = i + 1;
  while (e < n && (uint32_t)(key[e] >> 32) == k) ++e;
  const int64_t len = e - i;
  if (len <= kShortRun) {
    insertion_by_tie(order + i, len, rkey, tie);
  } else {
    const unsigned long long slot = atomicAdd(nlong, 1ull);
    longs[2 * slot] = i;
    longs[2 * slot + 1] = len;
  }
}

// Bottom-up merge sort of one run by the whole block: each pass places every
// element at (its rank in its own half) + (number of elements of the other
// half before it), found by binary search -- the order is strict (particle
// index breaks every tie), so the placement is a permutation.
__device__ void block_merge_sort(uint32_t *o, uint32_t *scratch, int64_t len,
                                 const uint64_t *rkey, const uint64_t *tie) {
  uint32_t *src = o, *dst = scratch;
  for (int64_t w = 1; w < len; w <<= 1) {
    for (int64_t t = threadIdx.x; t < len; t += blockDim.x) {
      const int64_t lo = (t / (2 * w)) * (2 * w);
      const int64_t mid = min(lo + w, len), hi = min(lo + 2 * w, len);
      const uint32_t v = src[t];
      int64_t a, b;
      if (t < mid) {
        a = mid;
        b = hi;
      } else {
        a = lo;
        b = mid;
      }
      const int64_t base = a;
      while (a < b) {
        const int64_t m = (a + b) >> 1;
        if (rank_less(rkey, tie, src[m], v)) a = m + 1;
        else b = m;
      }
      const int64_t pos = t < mid ? t + (a - base) : lo + (t - mid) + (a - base);
      dst[pos] = v;
    }
    __syncthreads();
    uint32_t *x = src;
    src = dst;
    dst = x;
  }
  if (src != o) {
    for (int64_t t = threadIdx.x; t < len; t += blockDim.x) o[t] = src[t];
    __syncthreads();
  }
}

__global__ void __launch_bounds__(1024) k_long_runs(uint32_t *__restrict__ order,
                                                    uint32_t *__restrict__ scratch,
                                                    const uint64_t *__restrict__ rkey,
                                                    const uint64_t *__restrict__ tie,
                                                    const int64_t *__restrict__ longs,
                                                    const unsigned long long *__restrict__ nlong) {
  __shared__ uint64_t sk[kBitonic];
  __shared__ uint32_t sv[kBitonic];
  const unsigned long long nr = *nlong;
  for (unsigned long long r = blockIdx.x; r < nr; r += gridDim.x) {
    const int64_t start = longs[2 * r], len = longs[2 * r + 1];
    uint32_t *o = order + start;
    if (len > kBitonic) {
      block_merge_sort(o, scratch + start, len, rkey, tie);
      continue;
    }
    int m = 1;
    while (m < len) m <<= 1;
    for (int t = threadIdx.x; t < m; t += blockDim.x) {
      sv[t] = t < len ? o[t] : 0xffffffffu;
      sk[t] = t < len ? rkey[sv[t]] : ~0ull;
    }
    __syncthreads();
    for (int size = 2; size <= m; size <<= 1)
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int t = threadIdx.x; t < m; t += blockDim.x) {
          const int u = t ^ stride;
          if (u > t) {
            const bool up = (t & size) == 0;
            // (full rank key, tie key, particle); padding (sv = ~0) last
            const bool gt =
                sk[t] > sk[u] ||
                (sk[t] == sk[u] &&
                 (sv[t] == 0xffffffffu ? sv[u] != 0xffffffffu
                  : sv[u] == 0xffffffffu ? false
                                         : tie_less(tie, sv[u], sv[t])));
            if (gt == up) {
              const uint64_t tk = sk[t];
              sk[t] = sk[u];
              sk[u] = tk;
              const uint32_t tv = sv[t];
              sv[t] = sv[u];
              sv[u] = tv;
            }
          }
        }
        __syncthreads();
      }
    for (int t = threadIdx.x; t < len; t += blockDim.x) o[t] = sv[t];
    __syncthreads();
  }
}

int32_t rank_order(const double *base, const int32_t *dint, double lam, int64_t n,
                   const uint32_t *px, const int32_t *pcomp, uint64_t seed, double *rank,
                   RankScratch &sc, uint32_t *order, unsigned long long *nneg, cudaStream_t s) {
  RCB_CUDA(cudaMemsetAsync(nneg, 0, sizeof(unsigned long long), s));
  if (n == 0) return RCB_OK;
  RCB_TRY(sc.tie.reserve(n, s));
  RCB_TRY(sc.rkey.reserve(n, s));
  RCB_TRY(sc.rkey2.reserve(n, s));
  RCB_TRY(sc.idx.reserve(n, s));
  RCB_TRY(sc.tie2.reserve(n + 2, s));  // long-run list (start, length) + its count
  k_rank<<<grid_for(n, 256), 256, 0, s>>>(base, dint, lam, n, px, pcomp, seed, rank, sc.tie.p,
                                          sc.rkey.p, sc.idx.p, nneg);
  RCB_CUDA(cudaGetLastError());
  // one stable sort by rank key from particle (x, comp) order
  size_t b = 0;
  RCB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, b, sc.rkey.p, sc.rkey2.p, sc.idx.p, order, n,
                                           32, 64, s));
  RCB_TRY(sc.tmp.reserve(b, s));
  RCB_CUDA(cub::DeviceRadixSort::SortPairs(sc.tmp.p, b, sc.rkey.p, sc.rkey2.p, sc.idx.p, order, n,
                                           32, 64, s));
  // equal rank values: (tie key, particle) order, as lexsort's next keys
  unsigned long long *nlong = reinterpret_cast<unsigned long long *>(sc.tie2.p + n);
  RCB_CUDA(cudaMemsetAsync(nlong, 0, sizeof(unsigned long long), s));
  int64_t *longs = reinterpret_cast<int64_t *>(sc.tie2.p);
  k_tie_runs<<<grid_for(n, 256), 256, 0, s>>>(sc.rkey2.p, n, order, sc.rkey.p, sc.tie.p, longs,
                                               nlong);
  // sc.idx (the sort's input values) is free now: scratch for the merge sort
  k_long_runs<<<64, 1024, 0, s>>>(order, sc.idx.p, sc.rkey.p, sc.tie.p, longs, nlong);
  RCB_CUDA(cudaGetLastError());
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
