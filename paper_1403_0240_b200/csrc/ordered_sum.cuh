// Exact parallel replay of a sequential fp64 accumulation
//     s_k = fl(s_{k-1} + v_k),   k = 1..n
// (np.bincount / np.add.at / the optimizer's ledger all accumulate this way,
// grid.py:164-168, optimizer.py:197).
//
// If s_{k-1} lies in the binade [2^e, 2^(e+1)) its ulp is u = 2^(e-52) and
// s_{k-1} is a multiple of u.  As long as the exact sum stays inside that
// binade, fl(s_{k-1} + v_k) = s_{k-1} + round_u(v_k), where round_u rounds
// to the nearest multiple of u — unless v_k/u has fractional part exactly 1/2
// (then ties-to-even depends on the running mantissa's parity).  So a run of
// steps that keeps the running mantissa M = s/u in [2^52 + 1, 2^53 - 1]
// (with the sign of s) is an int64 prefix sum of round_u(v_k)/u.  A block
// scans 1024 steps at a time, finds the first step that breaks the run
// (binade exit, tie, |v| too large, s == 0) and performs that one step
// sequentially; the result is bit-identical to the sequential loop.
#pragma once

#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

namespace rcb {

struct Binade {
  int e;            // s = M * 2^(e-52), |M| in [2^52, 2^53)
  long long M;      // signed mantissa (units of u)
  bool ok;          // false for 0, subnormal, inf/nan
};

__device__ __forceinline__ Binade binade_of(double s) {
  Binade b;
  const unsigned long long u = (unsigned long long)__double_as_longlong(s);
  const int ex = (int)((u >> 52) & 0x7ff);
  b.ok = ex > 0 && ex < 0x7ff;
  b.e = ex - 1023;
  long long m = (long long)((u & ((1ull << 52) - 1)) | (1ull << 52));
  b.M = (u >> 63) ? -m : m;
  return b;
}

// step of v in units of u = 2^(e-52); returns false if v breaks a run
// (tie, too large, non-finite).
__device__ __forceinline__ bool run_step(double v, int e, long long &step) {
  const double q = ldexp(v, 52 - e);
  if (!(fabs(q) < 9007199254740992.0)) return false;  // |v| >= 2^(e+1) or nan
  const double r = rint(q);
  if (fabs(q - r) == 0.5) return false;  // tie: parity of the running sum decides
  step = (long long)r;
  return true;
}

template <int BT, int IT = 8>
struct OrderedSum {
  typedef cub::BlockScan<long long, BT> Scan;
  typedef cub::BlockReduce<int, BT> Red;
  struct Temp {
    typename Scan::TempStorage scan;
    typename Red::TempStorage red;
    double s;
    long long base;
    int stop;
  };

  // Replays s = fl(s + val(i)) for i in [0, n) with the whole block, BT*IT
  // elements per step; pre(i, s) receives the running value before step i.
  // Returns the final s (valid in every thread).
  template <class Val, class Pre>
  __device__ static double run(Temp &T, double s, long long n, Val val, Pre pre) {
    constexpr int W = BT * IT;
    long long pos = 0;
    while (pos < n) {
      const Binade b = binade_of(s);
      const long long i0 = pos + (long long)threadIdx.x * IT;
      double v[IT];
      long long loc[IT];
      bool good[IT];
      long long acc = 0;
#pragma unroll
      for (int k = 0; k < IT; ++k) {
        const long long i = i0 + k;
        long long st = 0;
        good[k] = true;
        v[k] = 0.0;
        if (i < n) {
          v[k] = val(i);
          good[k] = b.ok && run_step(v[k], b.e, st);
          if (!good[k]) st = 0;
        }
        acc += st;
        loc[k] = acc;
      }
      long long tbase;
      Scan(T.scan).ExclusiveSum(acc, tbase);
      int bad = W;
#pragma unroll
      for (int k = 0; k < IT; ++k) {
        const long long i = i0 + k;
        if (i >= n) continue;
        bool g = good[k];
        if (g) {
          const long long M = b.M + tbase + loc[k];
          const long long aM = M < 0 ? -M : M;
          g = ((M < 0) == (b.M < 0)) && aM >= (1ll << 52) + 1 && aM <= (1ll << 53) - 1;
        }
        if (!g && bad == W) bad = (int)threadIdx.x * IT + k;
      }
      const int first = Red(T.red).Reduce(bad, cub::Min());
      if (threadIdx.x == 0) T.stop = first;
      __syncthreads();
      const int stop = T.stop;
      const long long avail = (n - pos) < (long long)W ? (n - pos) : (long long)W;
      const int upto = stop < avail ? stop : (int)avail;
#pragma unroll
      for (int k = 0; k < IT; ++k) {
        const int w = (int)threadIdx.x * IT + k;
        if (w < upto) {
          const long long incl = tbase + loc[k];
          long long st = (k == 0 ? loc[0] : loc[k] - loc[k - 1]);
          pre(i0 + k, ldexp((double)(b.M + incl - st), b.e - 52));
          if (w == upto - 1) T.base = b.M + incl;
        }
      }
      __syncthreads();
      const double s_run = upto > 0 ? ldexp((double)T.base, b.e - 52) : s;
      if (stop < avail) {
        const long long j = pos + stop;
        if ((int)threadIdx.x == stop / IT) {
          const int k = stop % IT;
          double vj = 0.0;
#pragma unroll
          for (int q = 0; q < IT; ++q)
            if (q == k) vj = v[q];
          pre(j, s_run);
          T.s = s_run + vj;
        }
        __syncthreads();
        s = T.s;
        pos = j + 1;
      } else {
        s = s_run;
        pos += avail;
      }
      __syncthreads();
    }
    return s;
  }
};

}  // namespace rcb
