// Device functions shared by the kernels (header-only; every TU that uses
// them is compiled with -fmad=false).
#pragma once

#include "common.cuh"

namespace rcb {

static constexpr double kPoissonFloor = 1e-8;  // energy.py:30

// ---------------------------------------------------------------------------
// neighbourhoods (grid.py:42-96)
// ---------------------------------------------------------------------------

// Distinct labels != own among the background-adjacency neighbours of a site,
// sorted ascending (contour.py:66-125; Appendix B1).  Background adjacency is
// the 2d faces for the default connectivity (full_fg) and the full box
// otherwise.  Returns the count; out has room for 26.
__device__ __forceinline__ int site_competitors(const int32_t *__restrict__ L, const Lat &lat,
                                                int full_fg, int64_t z, int64_t y, int64_t x,
                                                int32_t own, int32_t *out) {
  int n = 0;
  const int zlo = lat.ndim == 3 ? -1 : 0, zhi = lat.ndim == 3 ? 1 : 0;
  for (int dz = zlo; dz <= zhi; ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        int m = abs(dz) + abs(dy) + abs(dx);
        if (m == 0) continue;
        if (full_fg && m != 1) continue;
        int64_t zz = z + dz, yy = y + dy, xx = x + dx;
        if (!lat.inb(zz, yy, xx)) continue;
        int32_t l = __ldg(&L[lat.flat(zz, yy, xx)]);
        if (l == own) continue;
        // insertion into a sorted distinct list
        int k = n;
        bool dup = false;
        for (int j = 0; j < n; ++j)
          if (out[j] == l) {
            dup = true;
            break;
          }
        if (dup) continue;
        while (k > 0 && out[k - 1] > l) {
          out[k] = out[k - 1];
          --k;
        }
        out[k] = l;
        ++n;
      }
  return n;
}

// Bit index of a box cell (dz, dy, dx) in [-1, 1]^3.
__host__ __device__ __forceinline__ int box_bit(int dz, int dy, int dx) {
  return (dz + 1) * 9 + (dy + 1) * 3 + (dx + 1);
}

// Foreground adjacency among the 27 box cells (bit box_bit(dz, dy, dx)):
// the cells of m together with their fg-neighbours inside the box
// (Chebyshev 1 for full_fg, Manhattan 1 else), by shifts and row masks.
__host__ __device__ __forceinline__ uint32_t box_dilate(uint32_t m, int full_fg) {
  constexpr uint32_t kFull = 0x7ffffffu;
  constexpr uint32_t kXlo = 0x1249249u, kXhi = kXlo << 2;      // dx = -1 / +1 cells
  constexpr uint32_t kYlo = 0x1c0e07u, kYhi = kYlo << 6;       // dy = -1 / +1 cells
  const uint32_t xs = (((m << 1) & ~kXlo) | ((m >> 1) & ~kXhi)) & kFull;
  if (full_fg) {
    const uint32_t m1 = m | xs;
    const uint32_t m2 = (m1 | ((m1 << 3) & ~kYlo) | ((m1 >> 3) & ~kYhi)) & kFull;
    return (m2 | (m2 << 9) | (m2 >> 9)) & kFull;
  }
  const uint32_t ys = (((m << 3) & ~kYlo) | ((m >> 3) & ~kYhi)) & kFull;
  return (m | xs | ys | (m << 9) | (m >> 9)) & kFull;
}

// bit i of box_adj(j) set when cells i and j are fg-adjacent
__device__ __forceinline__ uint32_t box_adj(int j, int full_fg) {
  return box_dilate(1u << j, full_fg) & ~(1u << j);
}

// Local component count of label a in the punctured 3^d box around a site
// (contour.py:128-162): 0 = no same-label cell, 1 = all fg-adjacent
// same-label cells connected inside the box, 2 = inconclusive.
__device__ __forceinline__ int local_component_count(const int32_t *__restrict__ L,
                                                     const Lat &lat, int full_fg, int64_t z,
                                                     int64_t y, int64_t x, int32_t a) {
  uint32_t cells = 0, seeds = 0;
  const int zlo = lat.ndim == 3 ? -1 : 0, zhi = lat.ndim == 3 ? 1 : 0;
  for (int dz = zlo; dz <= zhi; ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        int m = abs(dz) + abs(dy) + abs(dx);
        if (m == 0) continue;
        int64_t zz = z + dz, yy = y + dy, xx = x + dx;
        if (!lat.inb(zz, yy, xx)) continue;
        if (L[lat.flat(zz, yy, xx)] != a) continue;
        uint32_t bit = 1u << box_bit(dz, dy, dx);
        cells |= bit;
        if (full_fg || m == 1) seeds |= bit;
      }
  if (!cells) return 0;
  if (!seeds) return 2;
  uint32_t reach = seeds & (~seeds + 1);  // lowest seed
  for (;;) {
    const uint32_t grow = box_dilate(reach, full_fg) & cells;
    if (grow == reach) break;
    reach = grow;
  }
  return (seeds & ~reach) ? 2 : 1;
}

// ---------------------------------------------------------------------------
// energies (energy.py:129-143, 226-230)
// ---------------------------------------------------------------------------

__device__ __forceinline__ double g_gauss(double n, double s, double q) {
  return n > 0.0 ? q - s * s / n : 0.0;
}

__device__ __forceinline__ double g_poisson(double n, double s) {
  if (!(n > 0.0)) return 0.0;
  double m = s / n;
  m = m < kPoissonFloor ? kPoissonFloor : m;
  return s - s * log(m);
}

__device__ __forceinline__ double rho(double i, double theta, int poisson) {
  if (!poisson) {
    double r = i - theta;
    return r * r;
  }
  double t = theta < kPoissonFloor ? kPoissonFloor : theta;
  return theta - i * log(t);
}

// PC increment from the region statistics (energy.py:308-324; Appendix B3).
__device__ __forceinline__ double delta_pc(double v, int64_t ca, double sa, double qa, int64_t cb,
                                           double sb, double qb, int poisson) {
  double na = (double)ca, nb = (double)cb;
  if (!poisson) {
    double before = g_gauss(na, sa, qa) + g_gauss(nb, sb, qb);
    double after = g_gauss(na - 1.0, sa - v, qa - v * v) + g_gauss(nb + 1.0, sb + v, qb + v * v);
    return after - before;
  }
  double before = g_poisson(na, sa) + g_poisson(nb, sb);
  double after = g_poisson(na - 1.0, sa - v) + g_poisson(nb + 1.0, sb + v);
  return after - before;
}

// Face-count perimeter change (energy.py:91-126).
__device__ __forceinline__ int delta_internal(const int32_t *__restrict__ L, const Lat &lat,
                                              int64_t z, int64_t y, int64_t x, int32_t a,
                                              int32_t b) {
  int d = 0;
  const int64_t c[3] = {z, y, x};
  const int64_t n[3] = {lat.nz, lat.ny, lat.nx};
  const int64_t st[3] = {lat.ny * lat.nx, lat.nx, 1};
  const int64_t f = lat.flat(z, y, x);
  for (int ax = 3 - lat.ndim; ax < 3; ++ax)
    for (int s = -1; s <= 1; s += 2) {
      int64_t cc = c[ax] + s;
      if (cc < 0 || cc >= n[ax]) continue;
      int32_t l = L[f + s * st[ax]];
      d += (int)(l != b) - (int)(l != a);
    }
  return d;
}

// PS increment of one particle (energy.py:337-372; Appendix B4).  rho0, when
// given, holds rho(I[y], Sown[y]/Cown[y]) for the current fields — the same
// function of the same inputs, so results are unchanged.  Also: with the
// dense per-label fields replaced by own-label fields Cown/Sown and the
// competitor's ball count/sum at x gathered during the walk.  ball holds the
// non-centre ball offsets in ball_offsets order.  Returns the increment and,
// through cb/sb, the competitor's ball count and sum at x.
__device__ __forceinline__ double delta_ps(const int32_t *__restrict__ L,
                                           const double *__restrict__ I,
                                           const int32_t *__restrict__ Cown,
                                           const double *__restrict__ Sown, const Lat &lat,
                                           const Off *__restrict__ ball, int nball, int64_t z,
                                           int64_t y, int64_t x, int32_t a, int32_t b, int poisson,
                                           int32_t *cb_out, double *sb_out,
                                           const double *__restrict__ rho0 = nullptr) {
  const int64_t f = lat.flat(z, y, x);
  const double v = I[f];
  double acc_a = 0.0;
  for (int k = 0; k < nball; ++k) {
    Off o = ball[k];
    int64_t zz = z + o.dz, yy = y + o.dy, xx = x + o.dx;
    if (!lat.inb(zz, yy, xx)) continue;
    int64_t g = lat.flat(zz, yy, xx);
    if (L[g] != a) continue;
    double cy = (double)Cown[g], sy = Sown[g], iy = I[g];
    acc_a += rho(iy, (sy - v) / (cy - 1.0), poisson) - (rho0 ? rho0[g] : rho(iy, sy / cy, poisson));
  }
  double acc_b = 0.0, sb = 0.0;
  int32_t cb = 0;
  for (int k = 0; k < nball; ++k) {
    Off o = ball[k];
    int64_t zz = z + o.dz, yy = y + o.dy, xx = x + o.dx;
    if (!lat.inb(zz, yy, xx)) continue;
    int64_t g = lat.flat(zz, yy, xx);
    if (L[g] != b) continue;
    double cy = (double)Cown[g], sy = Sown[g], iy = I[g];
    acc_b += rho(iy, (sy + v) / (cy + 1.0), poisson) - (rho0 ? rho0[g] : rho(iy, sy / cy, poisson));
    cb += 1;
    sb += iy;
  }
  double d = 0.0 + acc_a;
  d = d + acc_b;
  d += rho(v, (sb + v) / ((double)cb + 1.0), poisson);
  d -= rho0 ? rho0[f] : rho(v, Sown[f] / (double)Cown[f], poisson);
  if (cb_out) *cb_out = cb;
  if (sb_out) *sb_out = sb;
  return d;
}

// Superaccumulator (K9): exact fp64 sums in int64 limbs.
__device__ __forceinline__ void acc_add(long long *limbs, double d) {
  if (d == 0.0) return;
  uint64_t u = (uint64_t)__double_as_longlong(d);
  int ex = (int)((u >> 52) & 0x7ff);
  uint64_t m = u & ((1ull << 52) - 1);
  int e;
  if (ex == 0) {
    e = -1074;
  } else {
    m |= 1ull << 52;
    e = ex - 1075;
  }
  int pos = e + 1074;
  int k0 = pos >> 5, sh = pos & 31;
  uint64_t lo = m << sh;
  uint64_t hi = sh ? (m >> (64 - sh)) : 0;
  long long c0 = (long long)(lo & 0xffffffffull), c1 = (long long)(lo >> 32), c2 = (long long)hi;
  if (u >> 63) {
    c0 = -c0;
    c1 = -c1;
    c2 = -c2;
  }
  if (c0) atomicAdd((unsigned long long *)&limbs[k0], (unsigned long long)c0);
  if (c1) atomicAdd((unsigned long long *)&limbs[k0 + 1], (unsigned long long)c1);
  if (c2) atomicAdd((unsigned long long *)&limbs[k0 + 2], (unsigned long long)c2);
}

// Warp-aggregated superaccumulator add (band ledger): lanes whose value
// falls on the same limb pair sum their 32-bit limb parts in 64-bit
// registers first (integer sums: exact in any order), then one shared-memory
// atomic per limb and group instead of one per lane.  All lanes call it.
__device__ __forceinline__ void acc_add_warp(long long *limbs, double d, bool has) {
  const int lane = threadIdx.x & 31;
  int k0 = 0;
  long long c0 = 0, c1 = 0, c2 = 0;
  has = has && d != 0.0;
  if (has) {
    const uint64_t u = (uint64_t)__double_as_longlong(d);
    const int ex = (int)((u >> 52) & 0x7ff);
    uint64_t m = u & ((1ull << 52) - 1);
    int e;
    if (ex == 0) {
      e = -1074;
    } else {
      m |= 1ull << 52;
      e = ex - 1075;
    }
    const int pos = e + 1074;
    k0 = pos >> 5;
    const int sh = pos & 31;
    const uint64_t lo = m << sh, hi = sh ? (m >> (64 - sh)) : 0;
    c0 = (long long)(lo & 0xffffffffull);
    c1 = (long long)(lo >> 32);
    c2 = (long long)hi;
    if (u >> 63) {
      c0 = -c0;
      c1 = -c1;
      c2 = -c2;
    }
  }
  unsigned act = __ballot_sync(0xffffffffu, has);
  while (act) {
    const int leader = __ffs(act) - 1;
    const int k = __shfl_sync(0xffffffffu, k0, leader);
    const bool mine = has && k0 == k;
    long long s0 = mine ? c0 : 0, s1 = mine ? c1 : 0, s2 = mine ? c2 : 0;
    for (int o = 16; o; o >>= 1) {
      s0 += __shfl_xor_sync(0xffffffffu, s0, o);
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
      s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    }
    if (lane == leader) {
      if (s0) atomicAdd((unsigned long long *)&limbs[k], (unsigned long long)s0);
      if (s1) atomicAdd((unsigned long long *)&limbs[k + 1], (unsigned long long)s1);
      if (s2) atomicAdd((unsigned long long *)&limbs[k + 2], (unsigned long long)s2);
    }
    if (mine) has = false;
    act = __ballot_sync(0xffffffffu, has);
  }
}

// Per-thread staging for the superaccumulator: values whose limb window
// (k0) matches the staged one are merged in registers (integer limb parts:
// exact in any order); a value on another window goes straight to the shared
// limbs with per-lane atomics.  flush_warp() is warp-collective and adds the
// staged parts with one shared atomic per limb and window, like acc_add_warp.
struct AccStage {
  int k0 = -1;
  long long c0 = 0, c1 = 0, c2 = 0;
  __device__ __forceinline__ void add(long long *limbs, double d) {
    if (d == 0.0) return;
    const uint64_t u = (uint64_t)__double_as_longlong(d);
    const int ex = (int)((u >> 52) & 0x7ff);
    uint64_t m = u & ((1ull << 52) - 1);
    int e;
    if (ex == 0) {
      e = -1074;
    } else {
      m |= 1ull << 52;
      e = ex - 1075;
    }
    const int pos = e + 1074, k = pos >> 5, sh = pos & 31;
    const uint64_t lo = m << sh, hi = sh ? (m >> (64 - sh)) : 0;
    long long a0 = (long long)(lo & 0xffffffffull), a1 = (long long)(lo >> 32), a2 = (long long)hi;
    if (u >> 63) {
      a0 = -a0;
      a1 = -a1;
      a2 = -a2;
    }
    if (k0 < 0) k0 = k;
    if (k == k0) {
      c0 += a0;
      c1 += a1;
      c2 += a2;
    } else {
      if (a0) atomicAdd((unsigned long long *)&limbs[k], (unsigned long long)a0);
      if (a1) atomicAdd((unsigned long long *)&limbs[k + 1], (unsigned long long)a1);
      if (a2) atomicAdd((unsigned long long *)&limbs[k + 2], (unsigned long long)a2);
    }
  }
  __device__ __forceinline__ void flush_warp(long long *limbs) {  // all lanes call it
    const int lane = threadIdx.x & 31;
    bool has = k0 >= 0 && (c0 | c1 | c2) != 0;
    unsigned act = __ballot_sync(0xffffffffu, has);
    while (act) {
      const int leader = __ffs(act) - 1;
      const int k = __shfl_sync(0xffffffffu, k0, leader);
      const bool mine = has && k0 == k;
      long long s0 = mine ? c0 : 0, s1 = mine ? c1 : 0, s2 = mine ? c2 : 0;
      for (int o = 16; o; o >>= 1) {
        s0 += __shfl_xor_sync(0xffffffffu, s0, o);
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        s2 += __shfl_xor_sync(0xffffffffu, s2, o);
      }
      if (lane == leader) {
        if (s0) atomicAdd((unsigned long long *)&limbs[k], (unsigned long long)s0);
        if (s1) atomicAdd((unsigned long long *)&limbs[k + 1], (unsigned long long)s1);
        if (s2) atomicAdd((unsigned long long *)&limbs[k + 2], (unsigned long long)s2);
      }
      if (mine) has = false;
      act = __ballot_sync(0xffffffffu, has);
    }
  }
};

__device__ __forceinline__ void acc_flush(long long *sm, long long *gl) {
  __syncthreads();
  for (int k = threadIdx.x; k < kLimbs; k += blockDim.x)
    if (sm[k]) atomicAdd((unsigned long long *)&gl[k], (unsigned long long)sm[k]);
}


// Exact sum rounded once to the nearest double, on the device (the host's
// limbs_to_double, energy.cu); one thread.
__device__ inline double limbs_round_dev(const long long *limbs) {
  constexpr int ND = kLimbs + 3;
  uint32_t dig[ND];
  long long carry = 0;
  for (int k = 0; k < ND; ++k) {
    const long long t = (k < kLimbs ? limbs[k] : 0) + carry;
    dig[k] = (uint32_t)(t & 0xffffffffll);
    carry = t >> 32;
  }
  const bool neg = carry < 0;
  if (neg) {
    uint64_t c = 1;
    for (int k = 0; k < ND; ++k) {
      const uint64_t t = (uint64_t)(uint32_t)~dig[k] + c;
      dig[k] = (uint32_t)t;
      c = t >> 32;
    }
  }
  int top = -1;
  for (int k = ND - 1; k >= 0; --k)
    if (dig[k]) {
      top = k * 32 + (31 - __clz(dig[k]));
      break;
    }
  if (top < 0) return 0.0;
  auto bit = [&](int p) -> uint64_t { return p < 0 ? 0 : (dig[p >> 5] >> (p & 31)) & 1u; };
  uint64_t m = 0;
  int shift = top >= 52 ? top - 52 : 0;
  for (int p = top; p >= shift; --p) m = (m << 1) | bit(p);
  if (shift > 0) {
    const uint64_t g = bit(shift - 1);
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
  const double r = ldexp((double)m, shift - 1074);
  return neg ? -r : r;
}

// ---------------------------------------------------------------------------
// ranking (optimizer.py:80-87)
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t tie_key(uint64_t x, uint64_t c, uint64_t seed) {
  uint64_t z = x * 0x9E3779B97F4A7C15ull;
  z ^= c * 0xBF58476D1CE4E5B9ull;
  z ^= seed;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Order-preserving map of a double to uint64 (ascending), for radix sort.
__device__ __forceinline__ uint64_t double_key(double d) {
  uint64_t u = (uint64_t)__double_as_longlong(d);
  return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}

}  // namespace rcb

namespace rcb {

// ---------------------------------------------------------------------------
// fp32 mode: the gradient path (raw increments, Sobolev filter) in single
// precision with cancellation-free difference forms (SURVEY Appendix B,
// "fp32 mode"); statistics, fields, ledger and totals stay fp64.
// ---------------------------------------------------------------------------

// PC increment, stable forms.  Gauss: n_b/(n_b+1)(v-mu_b)^2 - n_a/(n_a-1)(v-mu_a)^2
// (the a-term is 0 when a vanishes).  Poisson: p(n+-1, s+-v) - p(n, s)
// = +-v(1 - log mu) - (s+-v) log1p(+-(v-mu)/((n+-1) mu)).
__device__ __forceinline__ float delta_pc32(float v, int64_t ca, double sa, int64_t cb, double sb,
                                            int poisson) {
  const float na = (float)ca, nb = (float)cb;
  const float mua = ca > 0 ? (float)(sa / (double)ca) : 0.f;
  const float mub = cb > 0 ? (float)(sb / (double)cb) : 0.f;
  if (!poisson) {
    float da = 0.f, db;
    if (ca > 1) {
      const float r = v - mua;
      da = na / (na - 1.f) * r * r;
    }
    const float r = v - mub;
    db = cb > 0 ? nb / (nb + 1.f) * r * r : 0.f;  // empty b: g(b') = 0 too
    return db - da;
  }
  // Poisson: fall back to the direct fp64 form near the mean floor
  if (!(mua > 1e-6f) || !(mub > 1e-6f) || ca < 2 || cb < 1) {
    const double vd = (double)v;
    return (float)delta_pc(vd, ca, sa, 0.0, cb, sb, 0.0, 1);
  }
  const float sa_f = (float)sa, sb_f = (float)sb;
  // removal from a: n -> n-1, s -> s-v ; addition to b: n -> n+1, s -> s+v
  const float ta = -v * (1.f - logf(mua)) - (sa_f - v) * log1pf(-(v - mua) / ((na - 1.f) * mua));
  const float tb = v * (1.f - logf(mub)) - (sb_f + v) * log1pf((v - mub) / ((nb + 1.f) * mub));
  return ta + tb;
}

// rho(i, theta + d) - rho(i, theta), cancellation-free.
__device__ __forceinline__ float drho32(float i, float theta, float d, int poisson) {
  if (!poisson) return d * (d - 2.f * (i - theta));
  if (!(theta > 1e-6f) || !(theta + d > 1e-6f)) {
    return (float)(rho((double)i, (double)theta + (double)d, 1) - rho((double)i, (double)theta, 1));
  }
  return d - i * log1pf(d / theta);
}

// PS increment in fp32 (ball terms as stable differences; the two centre
// terms are full rho values, evaluated in fp64).
__device__ __forceinline__ float delta_ps32(const int32_t *__restrict__ L, const float *__restrict__ I32,
                                            const int32_t *__restrict__ Cown,
                                            const double *__restrict__ Sown, const Lat &lat,
                                            const Off *__restrict__ ball, int nball, int64_t z,
                                            int64_t y, int64_t x, int32_t a, int32_t b,
                                            int poisson, int32_t *cb_out, double *sb_out) {
  const int64_t f = lat.flat(z, y, x);
  const float v = I32[f];
  float acc_a = 0.f, acc_b = 0.f;
  double sb = 0.0;
  int32_t cb = 0;
  for (int k = 0; k < nball; ++k) {
    const Off o = ball[k];
    const int64_t zz = z + o.dz, yy = y + o.dy, xx = x + o.dx;
    if (!lat.inb(zz, yy, xx)) continue;
    const int64_t g = lat.flat(zz, yy, xx);
    const int32_t l = L[g];
    if (l != a && l != b) continue;
    const float cy = (float)Cown[g], th = (float)(Sown[g] / (double)Cown[g]), iy = I32[g];
    if (l == a) {
      acc_a += drho32(iy, th, (th - v) / (cy - 1.f), poisson);
    } else {
      acc_b += drho32(iy, th, (v - th) / (cy + 1.f), poisson);
      cb += 1;
      sb += (double)iy;
    }
  }
  const double vd = (double)v;
  const double centre = rho(vd, (sb + vd) / ((double)cb + 1.0), poisson) -
                        rho(vd, Sown[f] / (double)Cown[f], poisson);
  *cb_out = cb;
  *sb_out = sb;
  return (acc_a + acc_b) + (float)centre;
}

}  // namespace rcb
