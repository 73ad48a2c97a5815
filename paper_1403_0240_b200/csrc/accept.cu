// K8 — topology-safe greedy acceptance in rank order (replaces
// optimizer.py:162-200 _execute, contour.py:128-241 is_move_admissible /
// apply_move / repair_pixel, energy.py:381-408 apply_flip and the ledger).
//
// v1 walks the sorted candidates with one device thread, which reproduces the
// reference's sequential semantics exactly.  The
// reference's global flood fill of the donor region (contour.py:194-202) is
// replaced by an exact but local question: into how many pieces does the
// removal of x split x's component?  A multi-source BFS from x's same-label
// foreground neighbours merges the seeds' searches as they meet and stops as
// soon as all seeds are one piece or one piece's frontier closes, so it never
// floods the whole region.  The per-label component counts it needs
// (components(a \ {x}) = ncomp[a] - 1 + pieces) come from a parallel
// union-find CCL and are maintained move by move.
#include "dev.cuh"
#include "kernels.h"

namespace rcb {

static constexpr uint32_t kEpochStep = 32;

struct BfsCtx {
  const int32_t *L;
  Lat lat;
  int full_fg;
  uint32_t *vis;
  uint32_t *queue;
  uint32_t *epoch;
};

template <typename F>
__device__ __forceinline__ void for_fg(const Lat &lat, int full_fg, int64_t f, F &&fn) {
  int64_t z, y, x;
  lat.coord(f, z, y, x);
  const int zlo = lat.ndim == 3 ? -1 : 0, zhi = lat.ndim == 3 ? 1 : 0;
  for (int dz = zlo; dz <= zhi; ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        int m = abs(dz) + abs(dy) + abs(dx);
        if (m == 0 || (!full_fg && m != 1)) continue;
        int64_t zz = z + dz, yy = y + dy, xx = x + dx;
        if (!lat.inb(zz, yy, xx)) continue;
        fn(lat.flat(zz, yy, xx));
      }
}

__device__ __forceinline__ int uf_find(int *par, int g) {
  while (par[g] != g) g = par[g];
  return g;
}

// Pieces of (component of x) \ {x} under fg adjacency: 0, 1 or 2 (= >= 2).
__device__ int pieces_without(const BfsCtx &c, int64_t f, int32_t a) {
  uint32_t seed[26];
  int ns = 0;
  for_fg(c.lat, c.full_fg, f, [&](int64_t g) {
    if (c.L[g] == a) seed[ns++] = (uint32_t)g;
  });
  if (ns <= 1) return ns;
  const uint32_t ep = *c.epoch;
  *c.epoch = ep + kEpochStep;
  int par[26], pend[26];
  int roots = ns;
  uint64_t head = 0, tail = 0;
  for (int i = 0; i < ns; ++i) {
    par[i] = i;
    pend[i] = 1;
    c.vis[seed[i]] = ep + i;
    c.queue[tail++] = seed[i];
  }
  while (head < tail) {
    const uint32_t s = c.queue[head++];
    int g = uf_find(par, (int)(c.vis[s] - ep));
    pend[g] -= 1;
    bool one = false;
    for_fg(c.lat, c.full_fg, s, [&](int64_t t) {
      if (one || t == f || c.L[t] != a) return;
      uint32_t v = c.vis[t];
      if (v >= ep && v < ep + kEpochStep) {
        int h = uf_find(par, (int)(v - ep));
        g = uf_find(par, g);
        if (h != g) {
          par[h] = g;
          pend[g] += pend[h];
          if (--roots == 1) one = true;
        }
      } else {
        g = uf_find(par, g);
        c.vis[t] = ep + g;
        c.queue[tail++] = (uint32_t)t;
        pend[g] += 1;
      }
    });
    if (one) return 1;
    if (pend[uf_find(par, g)] == 0) return 2;
  }
  return roots == 1 ? 1 : 2;
}

// Exact component count of label a (rare path: labels whose count is unknown).
__device__ int32_t count_components(const BfsCtx &c, int32_t a) {
  const uint32_t ep = *c.epoch;
  *c.epoch = ep + kEpochStep;
  int32_t comps = 0;
  for (int64_t s0 = 0; s0 < c.lat.V; ++s0) {
    if (c.L[s0] != a || c.vis[s0] == ep) continue;
    ++comps;
    uint64_t head = 0, tail = 0;
    c.vis[s0] = ep;
    c.queue[tail++] = (uint32_t)s0;
    while (head < tail) {
      const uint32_t s = c.queue[head++];
      for_fg(c.lat, c.full_fg, s, [&](int64_t t) {
        if (c.L[t] == a && c.vis[t] != ep) {
          c.vis[t] = ep;
          c.queue[tail++] = (uint32_t)t;
        }
      });
    }
  }
  return comps;
}

__global__ void k_accept_seq(AcceptArgs A) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  const Lat &lat = A.lat;
  BfsCtx bc{A.L, lat, A.full_fg, A.vis, A.queue, A.epoch};
  int64_t moves = 0;
  double energy = *A.energy;
  for (int64_t r = 0; r < A.n; ++r) {
    const uint32_t p = A.order[r];
    if (!(A.rank[p] < 0.0)) break;
    if (moves >= A.budget) break;
    const int64_t f = A.px[p];
    const int32_t a = A.pown[p], b = A.pcomp[p];
    if (A.L[f] != a) continue;  // moved or stale owner (optimizer.py:179-182)
    int64_t z, y, x;
    lat.coord(f, z, y, x);
    {  // competitor still adjacent under the background adjacency (:183-184)
      int32_t tmp[26];
      int nc = site_competitors(A.L, lat, A.full_fg, z, y, x, a, tmp);
      bool found = false;
      for (int k = 0; k < nc; ++k) found |= tmp[k] == b;
      if (!found) continue;
    }
    // admissibility (contour.py:171-207)
    int how_a = 0;  // 0 untouched, 1 vanish, 2 local, 3 global
    if (a > 0) {
      if (A.cnt[a] == 1) {
        if (!A.vanish_ok) continue;
        how_a = 1;
      } else if (local_component_count(A.L, lat, A.full_fg, z, y, x, a) == 1) {
        how_a = 2;
      } else {
        int pc = pieces_without(bc, f, a);
        if (pc >= 2) continue;
        if (A.ncomp[a] < 0) A.ncomp[a] = count_components(bc, a);
        if (A.ncomp[a] - 1 + pc != 1) continue;
        how_a = 3;
      }
    }
    if (b > 0 && !A.allow_fusion) {
      bool bad = false;
      for_fg(lat, A.full_fg, f, [&](int64_t g) {
        int32_t l = A.L[g];
        if (l > 0 && l != a && l != b) bad = true;
      });
      if (bad) continue;
    }
    // true increment against the current raster (optimizer.py:186-193)
    const double v = A.I[f];
    int32_t cb = 0;
    double sb = 0.0;
    double dext;
    if (A.region_ps)
      dext = delta_ps(A.L, A.I, A.Cown, A.Sown, lat, A.ball, A.nball, z, y, x, a, b, A.poisson,
                      &cb, &sb, A.rho0);
    else
      dext = delta_pc(v, A.cnt[a], A.tot[a], A.tsq[a], A.cnt[b], A.tot[b], A.tsq[b], A.poisson);
    const double dtot = dext + A.lam * (double)delta_internal(A.L, lat, z, y, x, a, b);
    if (A.mode_l2 && !(dtot < 0.0)) continue;
    // component bookkeeping for the joining label b
    if (b > 0 && A.ncomp[b] >= 0) {
      int nbb = 0;
      for_fg(lat, A.full_fg, f, [&](int64_t g) { nbb += A.L[g] == b; });
      if (nbb == 0)
        A.ncomp[b] += 1;
      else if (A.ncomp[b] > 1 && local_component_count(A.L, lat, A.full_fg, z, y, x, b) != 1)
        A.ncomp[b] = -1;
    }
    if (how_a == 1) A.ncomp[a] = 0;
    if (how_a == 3) A.ncomp[a] = 1;
    // apply (contour.py:210-241, grid.py:171-181, energy.py:381-408)
    if (A.region_ps) {
      for (int k = 0; k < A.nball; ++k) {
        Off o = A.ball[k];
        int64_t zz = z + o.dz, yy = y + o.dy, xx = x + o.dx;
        if (!lat.inb(zz, yy, xx)) continue;
        int64_t g = lat.flat(zz, yy, xx);
        int32_t l = A.L[g];
        if (l == a) {
          A.Cown[g] -= 1;
          A.Sown[g] -= v;
        } else if (l == b) {
          A.Cown[g] += 1;
          A.Sown[g] += v;
        } else {
          continue;
        }
        if (A.rho0) A.rho0[g] = rho(A.I[g], A.Sown[g] / (double)A.Cown[g], A.poisson);
      }
      A.Cown[f] = cb + 1;
      A.Sown[f] = sb + v;
      if (A.rho0) A.rho0[f] = rho(v, A.Sown[f] / (double)A.Cown[f], A.poisson);
    }
    A.L[f] = b;
    A.cnt[a] -= 1;
    A.tot[a] -= v;
    A.tsq[a] -= v * v;
    A.cnt[b] += 1;
    A.tot[b] += v;
    A.tsq[b] += v * v;
    energy += dtot;
    A.acc[3 * moves + 0] = f;
    A.acc[3 * moves + 1] = a;
    A.acc[3 * moves + 2] = b;
    ++moves;
  }
  *A.energy = energy;
  *A.moves = moves;
}

int32_t accept_seq(const AcceptArgs &args, cudaStream_t s) {
  k_accept_seq<<<1, 1, 0, s>>>(args);
  RCB_CUDA(cudaGetLastError());
  return RCB_OK;
}

// ---------------------------------------------------------------------------
// Parallel union-find CCL of every positive label under fg adjacency
// (Playne & Hawick style hooking with atomicMin), then roots per label.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t cc_find(const uint32_t *par, uint32_t x) {
  uint32_t p = par[x];
  while (p != x) {
    x = p;
    p = par[x];
  }
  return x;
}

__device__ __forceinline__ void cc_union(uint32_t *par, uint32_t a, uint32_t b) {
  bool done;
  do {
    a = cc_find(par, a);
    b = cc_find(par, b);
    if (a < b) {
      uint32_t old = atomicMin(&par[b], a);
      done = old == b;
      b = old;
    } else if (b < a) {
      uint32_t old = atomicMin(&par[a], b);
      done = old == a;
      a = old;
    } else {
      done = true;
    }
  } while (!done);
}

__global__ void k_cc_init(uint32_t *par, int64_t V) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < V; i += stride)
    par[i] = (uint32_t)i;
}

__global__ void k_cc_hook(const int32_t *__restrict__ L, Lat lat, int full_fg, uint32_t *par) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < lat.V; f += stride) {
    int32_t l = L[f];
    if (l <= 0) continue;
    int64_t z, y, x;
    lat.coord(f, z, y, x);
    // backward half of the neighbourhood: each edge once
    const int zlo = lat.ndim == 3 ? -1 : 0;
    for (int dz = zlo; dz <= 0; ++dz)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          int lin = dz * 9 + dy * 3 + dx;
          if (lin >= 0) continue;
          int m = abs(dz) + abs(dy) + abs(dx);
          if (!full_fg && m != 1) continue;
          int64_t zz = z + dz, yy = y + dy, xx = x + dx;
          if (!lat.inb(zz, yy, xx)) continue;
          int64_t g = lat.flat(zz, yy, xx);
          if (L[g] == l) cc_union(par, (uint32_t)f, (uint32_t)g);
        }
  }
}

__global__ void k_cc_count(const int32_t *__restrict__ L, int64_t V, const uint32_t *par,
                           int32_t *ncomp) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < V; f += stride) {
    int32_t l = L[f];
    if (l > 0 && par[f] == (uint32_t)f) atomicAdd(&ncomp[l], 1);
  }
}

int32_t label_components(const int32_t *L, const Lat &lat, int full_fg, int32_t nl,
                         uint32_t *par_scratch, int32_t *ncomp, cudaStream_t s) {
  RCB_CUDA(cudaMemsetAsync(ncomp, 0, sizeof(int32_t) * nl, s));
  unsigned g = grid_for(lat.V, 256);
  k_cc_init<<<g, 256, 0, s>>>(par_scratch, lat.V);
  k_cc_hook<<<g, 256, 0, s>>>(L, lat, full_fg, par_scratch);
  k_cc_count<<<g, 256, 0, s>>>(L, lat.V, par_scratch, ncomp);
  RCB_CUDA(cudaGetLastError());
  return RCB_OK;
}

}  // namespace rcb
