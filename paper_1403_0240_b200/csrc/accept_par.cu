// K8 v2 — parallel, exact rank-ordered acceptance (sobolev mode).
//
// The reference accepts candidates one at a time in rank order
// (optimizer.py:162-200).  Candidate i's verdict depends only on
// (a) the labels of its 3^d box, (b) for an inconclusive local topology test,
// the labels along a BFS footprint in its donor region, and (c) for regions
// that can run out of pixels this iteration, the region's pixel count.
// Every site flips at most once per iteration (a flipped site no longer
// carries its snapshot owner), so the state "as of position i" is a pure
// function of the iteration-start raster L, the flip positions w[] and the
// new labels newlab[]:  V_i(y) = w[y] < i ? newlab[y] : L[y].
//
// A persistent cooperative kernel decides candidates in rounds.  Candidate i
// is decided in a round when no undecided candidate j < i sits on a site it
// reads (pend[y] = min undecided position at y), so the view V_i it reads is
// final; later candidates decided earlier are invisible through w[].  The
// earliest undecided candidate is always decidable, so rounds terminate, and
// every verdict equals the sequential one.  Inconclusive topology tests run a
// block-cooperative multi-source BFS (shared-memory hash) that aborts if it
// touches a pending site; footprints beyond its capacity are deferred to an
// unbounded global BFS run when the candidate becomes the earliest.
//
// Preconditions (checked by the host; otherwise the sequential kernel runs):
// sobolev mode (no d_tot gate), default connectivity, every positive label a
// single component at iteration start (so components(a\{x}) == pieces).
#include <cooperative_groups.h>

#include <cub/device/device_scan.cuh>

#include "dev.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace rcb {

static constexpr int32_t kInf = 0x7fffffff;
static constexpr int kHC = 8192;      // BFS hash capacity (64-bit entries)
static constexpr int kFC = 2048;      // BFS frontier capacity per level
static constexpr int kMaxInsert = kHC * 5 / 8;
static constexpr unsigned long long kEmpty = ~0ull;

enum : uint8_t { UNDEC = 0, ACC = 1, REJ = 2, DEFER = 3 };
enum { C_NUND0 = 0, C_NUND1, C_MIN0, C_MIN1, C_BFS, C_ROUNDS, C_BFSRUNS, C_DEFER, C_BLOCKED, C_N };

__device__ __forceinline__ int32_t ld(const int32_t *p) { return __ldcg(p); }

struct View {
  const ParArgs &A;
  int32_t pos;
  __device__ __forceinline__ int32_t lab(int64_t y) const {
    int32_t wy = ld(A.w + y);
    return wy < pos ? ld(A.newlab + y) : __ldg(A.L + y);
  }
  __device__ __forceinline__ bool pending(int64_t y) const { return ld(A.pend + y) < pos; }
};

// Box labels through the view: lab[27] (-1 = out of bounds); returns false if
// a site of the box has an earlier undecided candidate.
__device__ __forceinline__ bool read_box(const View &v, const Lat &lat, int64_t z, int64_t y,
                                         int64_t x, int32_t *lab) {
  bool ok = true;
  for (int k = 0; k < 27; ++k) {
    int dz = k / 9 - 1, dy = (k / 3) % 3 - 1, dx = k % 3 - 1;
    int64_t zz = z + dz, yy = y + dy, xx = x + dx;
    if ((lat.ndim == 2 && dz != 0) || !lat.inb(zz, yy, xx)) {
      lab[k] = -1;
      continue;
    }
    int64_t g = lat.flat(zz, yy, xx);
    if (v.pending(g)) ok = false;
    lab[k] = v.lab(g);
  }
  return ok;
}

__device__ __forceinline__ bool is_face(int k) {
  int dz = k / 9 - 1, dy = (k / 3) % 3 - 1, dx = k % 3 - 1;
  return abs(dz) + abs(dy) + abs(dx) == 1;
}

// Local component count from box labels (contour.py:128-162), fg = full box.
__device__ __forceinline__ int box_local_count(const int32_t *lab, int32_t a) {
  uint32_t cells = 0;
  for (int k = 0; k < 27; ++k)
    if (k != 13 && lab[k] == a) cells |= 1u << k;
  if (!cells) return 0;
  uint32_t reach = cells & (~cells + 1);
  for (;;) {
    uint32_t grow = reach;
    for (uint32_t r = reach; r; r &= r - 1) grow |= box_adj(__ffs(r) - 1, 1) & cells;
    if (grow == reach) break;
    reach = grow;
  }
  return (cells & ~reach) ? 2 : 1;
}

__device__ __forceinline__ bool box_fusion_bad(const int32_t *lab, int32_t a, int32_t b) {
  for (int k = 0; k < 27; ++k)
    if (k != 13 && lab[k] > 0 && lab[k] != a && lab[k] != b) return true;
  return false;
}

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}

struct BfsShared {
  unsigned long long key[kHC];
  uint32_t fr[2][kFC];
  uint8_t fg[2][kFC];
  int nfr[2];
  int par[27];
  int gcount[27];
  uint32_t unions[27];
  int nseed;
  int ninsert;
  int blocked, overflow, result;
  int32_t pos, a, b;
  int64_t x;
};

__device__ __forceinline__ int uf_root(int *par, int g) {
  while (par[g] != g) g = par[g];
  return g;
}

// Decide the level outcome (thread 0): -1 continue, 0 blocked, 1 one piece,
// 2 several pieces, 3 overflow.
__device__ int bfs_level_verdict(BfsShared &S, int nxt) {
  if (S.blocked) return 0;
  if (S.overflow) return 3;
  for (int g = 0; g < S.nseed; ++g)
    for (uint32_t m = S.unions[g]; m; m &= m - 1) {
      int h = __ffs(m) - 1;
      int rg = uf_root(S.par, g), rh = uf_root(S.par, h);
      if (rg != rh) S.par[rh] = rg;
    }
  for (int g = 0; g < S.nseed; ++g) S.unions[g] = 0;
  int roots = 0;
  int rc[27];
  for (int g = 0; g < S.nseed; ++g) rc[g] = 0;
  for (int g = 0; g < S.nseed; ++g) {
    int r = uf_root(S.par, g);
    if (r == g) ++roots;
    rc[r] += S.gcount[g];
    S.gcount[g] = 0;
  }
  if (roots == 1) return 1;
  for (int g = 0; g < S.nseed; ++g)
    if (uf_root(S.par, g) == g && rc[g] == 0) return 2;
  (void)nxt;
  return -1;
}

// Block-cooperative BFS for candidate pos: pieces of C_x \ {x} in view V_pos.
// Returns 0 blocked, 1 one piece, 2 several, 3 overflow.
__device__ int block_bfs(const ParArgs &A, BfsShared &S, int32_t pos) {
  const Lat &lat = A.lat;
  View v{A, pos};
  if (threadIdx.x == 0) {
    uint32_t p = A.order[pos];
    S.pos = pos;
    S.x = A.px[p];
    S.a = A.pown[p];
    S.b = A.pcomp[p];
    S.ninsert = 0;
    S.blocked = S.overflow = 0;
    S.result = -1;
    S.nfr[0] = S.nfr[1] = 0;
  }
  for (int k = threadIdx.x; k < kHC; k += blockDim.x) S.key[k] = kEmpty;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t z, y, x;
    lat.coord(S.x, z, y, x);
    auto put = [&](uint32_t site, int g) {
      uint32_t h = hash32(site) & (kHC - 1);
      while (S.key[h] != kEmpty) h = (h + 1) & (kHC - 1);
      S.key[h] = ((unsigned long long)site << 8) | (unsigned)g;
    };
    put((uint32_t)S.x, 255);
    int ns = 0;
    for (int k = 0; k < 27; ++k) {
      if (k == 13) continue;
      int dz = k / 9 - 1, dy = (k / 3) % 3 - 1, dx = k % 3 - 1;
      int64_t zz = z + dz, yy = y + dy, xx = x + dx;
      if ((lat.ndim == 2 && dz != 0) || !lat.inb(zz, yy, xx)) continue;
      int64_t g = lat.flat(zz, yy, xx);
      if (v.lab(g) != S.a) continue;
      put((uint32_t)g, ns);
      S.fr[0][ns] = (uint32_t)g;
      S.fg[0][ns] = (uint8_t)ns;
      S.par[ns] = ns;
      S.gcount[ns] = 0;
      S.unions[ns] = 0;
      ++ns;
    }
    S.nseed = ns;
    S.nfr[0] = ns;
    S.ninsert = ns + 1;
  }
  __syncthreads();
  int cur = 0;
  for (;;) {
    const int n = S.nfr[cur], nxt = cur ^ 1;
    const int32_t a = S.a;
    const int64_t xc = S.x;
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      const uint32_t s = S.fr[cur][j];
      const int g = S.fg[cur][j];
      int64_t z, y, x;
      lat.coord(s, z, y, x);
      for (int k = 0; k < 27; ++k) {
        if (k == 13) continue;
        int dz = k / 9 - 1, dy = (k / 3) % 3 - 1, dx = k % 3 - 1;
        int64_t zz = z + dz, yy = y + dy, xx = x + dx;
        if ((lat.ndim == 2 && dz != 0) || !lat.inb(zz, yy, xx)) continue;
        int64_t t = lat.flat(zz, yy, xx);
        if (t == xc) continue;
        if (v.pending(t)) {
          S.blocked = 1;
          continue;
        }
        if (v.lab(t) != a) continue;
        uint32_t h = hash32((uint32_t)t) & (kHC - 1);
        for (;;) {
          unsigned long long cv = S.key[h];
          if (cv == kEmpty) {
            unsigned long long mine = ((unsigned long long)t << 8) | (unsigned)g;
            unsigned long long old = atomicCAS(&S.key[h], kEmpty, mine);
            if (old == kEmpty) {
              int idx = atomicAdd(&S.nfr[nxt], 1);
              if (idx < kFC) {
                S.fr[nxt][idx] = (uint32_t)t;
                S.fg[nxt][idx] = (uint8_t)g;
              } else {
                S.overflow = 1;
              }
              atomicAdd(&S.gcount[g], 1);
              if (atomicAdd(&S.ninsert, 1) >= kMaxInsert) S.overflow = 1;
              break;
            }
            cv = old;
          }
          if ((uint32_t)(cv >> 8) == (uint32_t)t) {
            int hgrp = (int)(cv & 0xff);
            if (hgrp != 255 && hgrp != g) atomicOr(&S.unions[g], 1u << hgrp);
            break;
          }
          h = (h + 1) & (kHC - 1);
        }
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      S.result = bfs_level_verdict(S, nxt);
      S.nfr[cur] = 0;
    }
    __syncthreads();
    if (S.result >= 0) break;
    cur = nxt;
  }
  return S.result;
}

// Unbounded BFS with global stamps/frontiers for the earliest undecided
// candidate (the rare escape when the shared-memory BFS overflowed).
__device__ int global_bfs(const ParArgs &A, BfsShared &S, int32_t pos) {
  const Lat &lat = A.lat;
  View v{A, pos};
  __shared__ uint32_t ep;
  __shared__ unsigned long long nf[2];
  if (threadIdx.x == 0) {
    uint32_t p = A.order[pos];
    S.x = A.px[p];
    S.a = A.pown[p];
    ep = *A.epoch;
    *A.epoch = ep + 32;
    S.blocked = S.overflow = 0;
    S.result = -1;
    int64_t z, y, x;
    lat.coord(S.x, z, y, x);
    A.vis[S.x] = ep + 31;
    int ns = 0;
    for (int k = 0; k < 27; ++k) {
      if (k == 13) continue;
      int dz = k / 9 - 1, dy = (k / 3) % 3 - 1, dx = k % 3 - 1;
      int64_t zz = z + dz, yy = y + dy, xx = x + dx;
      if ((lat.ndim == 2 && dz != 0) || !lat.inb(zz, yy, xx)) continue;
      int64_t g = lat.flat(zz, yy, xx);
      if (v.lab(g) != S.a) continue;
      A.vis[g] = ep + ns;
      A.gq[0][ns] = (uint32_t)g;
      S.par[ns] = ns;
      S.gcount[ns] = 0;
      S.unions[ns] = 0;
      ++ns;
    }
    S.nseed = ns;
    nf[0] = ns;
    nf[1] = 0;
  }
  __syncthreads();
  int cur = 0;
  for (;;) {
    const unsigned long long n = nf[cur];
    const int nxt = cur ^ 1;
    for (unsigned long long j = threadIdx.x; j < n; j += blockDim.x) {
      const uint32_t s = A.gq[cur][j];
      const int g = (int)(__ldcg(A.vis + s) - ep);
      int64_t z, y, x;
      lat.coord(s, z, y, x);
      for (int k = 0; k < 27; ++k) {
        if (k == 13) continue;
        int dz = k / 9 - 1, dy = (k / 3) % 3 - 1, dx = k % 3 - 1;
        int64_t zz = z + dz, yy = y + dy, xx = x + dx;
        if ((lat.ndim == 2 && dz != 0) || !lat.inb(zz, yy, xx)) continue;
        int64_t t = lat.flat(zz, yy, xx);
        if (v.lab(t) != S.a) continue;
        uint32_t cv = __ldcg(A.vis + t);
        for (;;) {
          if (cv >= ep && cv < ep + 32) {
            int h = (int)(cv - ep);
            if (h != 31 && h != g) atomicOr(&S.unions[g], 1u << h);
            break;
          }
          uint32_t old = atomicCAS(A.vis + t, cv, ep + (uint32_t)g);
          if (old == cv) {
            unsigned long long idx = atomicAdd(&nf[nxt], 1ull);
            A.gq[nxt][idx] = (uint32_t)t;
            atomicAdd(&S.gcount[g], 1);
            break;
          }
          cv = old;
        }
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      S.result = bfs_level_verdict(S, nxt);
      nf[cur] = 0;
    }
    __syncthreads();
    if (S.result >= 0) break;
    cur = nxt;
    __threadfence_block();
  }
  return S.result;
}

__device__ __forceinline__ void finish_topology(const ParArgs &A, int32_t pos, int pieces,
                                                int32_t round) {
  // pieces == 1 passes the donor test; fusion check on the box next
  uint8_t d = REJ;
  if (pieces == 1) {
    uint32_t p = A.order[pos];
    int64_t f = A.px[p];
    int32_t a = A.pown[p], b = A.pcomp[p];
    d = ACC;
    if (b > 0 && !A.allow_fusion) {
      int64_t z, y, x;
      A.lat.coord(f, z, y, x);
      int32_t lab[27];
      View v{A, pos};
      read_box(v, A.lat, z, y, x, lab);
      if (box_fusion_bad(lab, a, b)) d = REJ;
    }
  }
  A.dec[pos] = d;
  A.dround[pos] = round;
}

__global__ void __launch_bounds__(512) k_accept_par(ParArgs A) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) uint8_t smem_raw[];
  BfsShared &S = *reinterpret_cast<BfsShared *>(smem_raw);
  const Lat &lat = A.lat;
  const int32_t M = (int32_t)*A.nneg;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  int32_t *ctl = A.ctl;

  // init: snapshot counts, owner-candidate counts, pending positions
  for (int64_t l = tid; l < A.nl; l += nth) {
    A.cnt0[l] = A.cnt[l];
    A.nown[l] = 0;
    A.lab_pend[l] = kInf;
  }
  for (int64_t pos = tid; pos < M; pos += nth) {
    A.dec[pos] = UNDEC;
    A.dround[pos] = -1;
  }
  grid.sync();
  for (int64_t pos = tid; pos < M; pos += nth) {
    uint32_t p = A.order[pos];
    atomicMin(A.pend + A.px[p], (int32_t)pos);
    int32_t a = A.pown[p];
    if (a > 0) atomicAdd(A.nown + a, 1);
  }
  grid.sync();
  for (int64_t l = tid; l < A.nl; l += nth)
    A.small[l] = (l > 0 && A.cnt0[l] - (int64_t)A.nown[l] <= 1) ? 1 : 0;
  grid.sync();
  for (int64_t pos = tid; pos < M; pos += nth) {
    uint32_t p = A.order[pos];
    int32_t a = A.pown[p], b = A.pcomp[p];
    if (A.small[a]) atomicMin(A.lab_pend + a, (int32_t)pos);
    if (A.small[b]) atomicMin(A.lab_pend + b, (int32_t)pos);
  }
  grid.sync();

  for (int32_t round = 0;; ++round) {
    const int par = round & 1;
    if (tid == 0) {
      ctl[C_NUND0 + par] = 0;
      ctl[C_MIN0 + par] = kInf;
    }
    // ---- phase D: local decisions of ready candidates
    for (int64_t pos = tid; pos < M; pos += nth) {
      if (__ldcg(A.dec + pos) != UNDEC) continue;
      const uint32_t p = A.order[pos];
      const int64_t f = A.px[p];
      const int32_t a = A.pown[p], b = A.pcomp[p];
      if ((A.small[a] && ld(A.lab_pend + a) < pos) || (A.small[b] && ld(A.lab_pend + b) < pos))
        continue;
      View v{A, (int32_t)pos};
      int64_t z, y, x;
      lat.coord(f, z, y, x);
      int32_t lab[27];
      if (!read_box(v, lat, z, y, x, lab)) continue;
      uint8_t d = ACC;
      if (lab[13] != a) {
        d = REJ;  // moved or stale owner
      } else {
        bool adj = false;
        for (int k = 0; k < 27; ++k)
          if (is_face(k) && lab[k] == b) adj = true;
        if (!adj) d = REJ;  // competitor no longer adjacent
      }
      if (d == ACC && a > 0) {
        if (A.small[a] && __ldcg((const long long *)A.cnt + a) == 1) {
          if (!A.vanish_ok) d = REJ;
        } else {
          int k = box_local_count(lab, a);
          if (k == 0) {
            d = REJ;  // a \ {x} would keep only the other components: != 1
          } else if (k != 1) {
            int e = atomicAdd(ctl + C_BFS, 1);
            A.bfs_list[e] = (int32_t)pos;
            continue;
          }
        }
      }
      if (d == ACC && b > 0 && !A.allow_fusion && box_fusion_bad(lab, a, b)) d = REJ;
      A.dec[pos] = d;
      A.dround[pos] = round;
    }
    grid.sync();
    // ---- phase B: topology BFS of inconclusive local tests; escape
    {
      const int nb = ld(ctl + C_BFS);
      for (int e = blockIdx.x; e < nb; e += gridDim.x) {
        const int32_t pos = A.bfs_list[e];
        int r = block_bfs(A, S, pos);
        if (threadIdx.x == 0) {
          atomicAdd(ctl + C_BFSRUNS, 1);
          if (r == 0) atomicAdd(ctl + C_BLOCKED, 1);
          if (r == 3) {
            A.dec[pos] = DEFER;
            atomicAdd(ctl + C_DEFER, 1);
          } else if (r == 1 || r == 2) {
            finish_topology(A, pos, r, round);
          }
        }
        __syncthreads();
      }
      if (blockIdx.x == gridDim.x - 1 && round > 0) {
        const int32_t m = ld(ctl + C_MIN0 + (par ^ 1));
        if (m < M && __ldcg(A.dec + m) == DEFER) {
          int r = global_bfs(A, S, m);
          if (threadIdx.x == 0) finish_topology(A, m, r == 1 ? 1 : 2, round);
          __syncthreads();
        }
      }
    }
    grid.sync();
    // ---- phase A1: apply this round's acceptances, release pending marks
    if (tid == 0) ctl[C_BFS] = 0;
    for (int64_t l = tid; l < A.nl; l += nth) A.lab_pend[l] = kInf;
    for (int64_t pos = tid; pos < M; pos += nth) {
      if (A.dround[pos] != round) continue;
      const uint32_t p = A.order[pos];
      const int64_t f = A.px[p];
      A.pend[f] = kInf;
      if (A.dec[pos] == ACC) {
        const int32_t a = A.pown[p], b = A.pcomp[p];
        A.newlab[f] = b;
        A.w[f] = (int32_t)pos;
        atomicAdd((unsigned long long *)(A.cnt + a), (unsigned long long)(-1ll));
        atomicAdd((unsigned long long *)(A.cnt + b), 1ull);
      }
    }
    grid.sync();
    // ---- phase A2: pending marks of the still-undecided candidates
    for (int64_t pos = tid; pos < M; pos += nth) {
      uint8_t d = A.dec[pos];
      if (d != UNDEC && d != DEFER) continue;
      const uint32_t p = A.order[pos];
      atomicMin(A.pend + A.px[p], (int32_t)pos);
      const int32_t a = A.pown[p], b = A.pcomp[p];
      if (A.small[a]) atomicMin(A.lab_pend + a, (int32_t)pos);
      if (A.small[b]) atomicMin(A.lab_pend + b, (int32_t)pos);
      atomicAdd(ctl + C_NUND0 + par, 1);
      atomicMin(ctl + C_MIN0 + par, (int32_t)pos);
    }
    grid.sync();
    if (ld(ctl + C_NUND0 + par) == 0) {
      if (tid == 0) ctl[C_ROUNDS] = round + 1;
      break;
    }
  }
}

// ---------------------------------------------------------------------------
// after the rounds: order the accepted moves, apply the budget, write labels
// ---------------------------------------------------------------------------
__global__ void k_acc_flags(const uint8_t *__restrict__ dec, const unsigned long long *nneg,
                            uint32_t *__restrict__ flag) {
  int64_t M = (int64_t)*nneg;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= M; i += stride)
    flag[i] = (i < M && dec[i] == ACC) ? 1u : 0u;
}

__global__ void k_acc_write(const ParArgs A, const uint32_t *__restrict__ slot, int64_t budget,
                            int64_t *__restrict__ acc, int64_t *__restrict__ moves) {
  int64_t M = (int64_t)*A.nneg;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < M; i += stride) {
    if (A.dec[i] != ACC) continue;
    uint32_t k = slot[i];
    if ((int64_t)k >= budget) continue;
    uint32_t p = A.order[i];
    acc[3 * k + 0] = A.px[p];
    acc[3 * k + 1] = A.pown[p];
    acc[3 * k + 2] = A.pcomp[p];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    int64_t tot = slot[M];
    *moves = tot < budget ? tot : budget;
  }
}

__device__ __forceinline__ int delta_internal_view(const ParArgs &A, const View &v, int64_t z,
                                                   int64_t y, int64_t x, int32_t a, int32_t b) {
  const Lat &lat = A.lat;
  int d = 0;
  const int64_t c[3] = {z, y, x};
  const int64_t n[3] = {lat.nz, lat.ny, lat.nx};
  const int64_t st[3] = {lat.ny * lat.nx, lat.nx, 1};
  const int64_t f = lat.flat(z, y, x);
  for (int ax = 3 - lat.ndim; ax < 3; ++ax)
    for (int s = -1; s <= 1; s += 2) {
      int64_t cc = c[ax] + s;
      if (cc < 0 || cc >= n[ax]) continue;
      int32_t l = v.lab(f + s * st[ax]);
      d += (int)(l != b) - (int)(l != a);
    }
  return d;
}

// PS ledger terms: the exact increment of each kept move in the view V_i,
// with the own-label fields at the ball sites recomputed from that view.
__global__ void k_ps_dtot(const ParArgs A, const int64_t *__restrict__ acc,
                          const int64_t *__restrict__ moves, const double *__restrict__ I,
                          const Off *__restrict__ ball, int nball, int poisson, double lam,
                          double *__restrict__ dtot) {
  const int64_t n = *moves;
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const Lat &lat = A.lat;
  for (int64_t k = warp; k < n; k += nwarps) {
    const int64_t f = acc[3 * k];
    const int32_t a = (int32_t)acc[3 * k + 1], b = (int32_t)acc[3 * k + 2];
    const int32_t pos = A.w[f];
    View v{A, pos};
    int64_t z, y, x;
    lat.coord(f, z, y, x);
    const double vx = I[f];
    // own-label fields at x (label a) and competitor count/sum at x
    // lanes take ball offsets; each computes its own site's term
    double ta = 0.0, tb = 0.0;  // per-lane terms are summed in offset order below
    for (int base = 0; base < nball; base += 32) {
      int kk = base + lane;
      double term_a = 0.0, term_b = 0.0;
      int hit_a = 0, hit_b = 0;
      if (kk < nball) {
        Off o = ball[kk];
        int64_t zz = z + o.dz, yy = y + o.dy, xx = x + o.dx;
        if (lat.inb(zz, yy, xx)) {
          int64_t g = lat.flat(zz, yy, xx);
          int32_t lg = v.lab(g);
          if (lg == a || lg == b) {
            // own-label ball count/sum at g in view V_pos (centre first)
            int32_t c = 0;
            double s = 0.0;
            int64_t gz, gy, gx;
            lat.coord(g, gz, gy, gx);
            for (int q = 0; q <= nball; ++q) {
              Off o2 = q == 0 ? Off{0, 0, 0, 0} : ball[q - 1];
              int64_t z2 = gz + o2.dz, y2 = gy + o2.dy, x2 = gx + o2.dx;
              if (!lat.inb(z2, y2, x2)) continue;
              int64_t h = lat.flat(z2, y2, x2);
              if (v.lab(h) != lg) continue;
              c += 1;
              s += I[h];
            }
            double cy = (double)c, iy = I[g];
            if (lg == a) {
              term_a = rho(iy, (s - vx) / (cy - 1.0), poisson) - rho(iy, s / cy, poisson);
              hit_a = 1;
            } else {
              term_b = rho(iy, (s + vx) / (cy + 1.0), poisson) - rho(iy, s / cy, poisson);
              hit_b = 1;
            }
          }
        }
      }
      // ordered accumulation (offset order) replayed by every lane
      for (int j = 0; j < 32; ++j) {
        if (base + j >= nball) break;
        int ha = __shfl_sync(0xffffffffu, hit_a, j);
        double da = __shfl_sync(0xffffffffu, term_a, j);
        if (ha) ta += da;
      }
      for (int j = 0; j < 32; ++j) {
        if (base + j >= nball) break;
        int hb = __shfl_sync(0xffffffffu, hit_b, j);
        double db = __shfl_sync(0xffffffffu, term_b, j);
        if (hb) tb += db;
      }
    }
    // competitor count/sum at x and own fields at x, in view V_pos
    if (lane == 0) {
      int32_t cb = 0, ca = 0;
      double sb = 0.0, sa = 0.0;
      for (int q = 0; q <= nball; ++q) {
        Off o2 = q == 0 ? Off{0, 0, 0, 0} : ball[q - 1];
        int64_t z2 = z + o2.dz, y2 = y + o2.dy, x2 = x + o2.dx;
        if (!lat.inb(z2, y2, x2)) continue;
        int64_t h = lat.flat(z2, y2, x2);
        int32_t lh = v.lab(h);
        if (lh == a) {
          ca += 1;
          sa += I[h];
        } else if (lh == b) {
          cb += 1;
          sb += I[h];
        }
      }
      double d = 0.0 + ta;
      d = d + tb;
      d += rho(vx, (sb + vx) / ((double)cb + 1.0), poisson);
      d -= rho(vx, sa / (double)ca, poisson);
      int di = delta_internal_view(A, v, z, y, x, a, b);
      dtot[k] = d + lam * (double)di;
    }
  }
}

// Sequential region statistics and ledger in acceptance order (grid.py:171-181,
// optimizer.py:197).  One warp: lanes prefetch 32 moves, lane 0 replays the
// fp64 chains in order and snapshots the pre-move statistics; the PC
// increments of the 32 moves are then evaluated in parallel and added to the
// ledger in order.  Per-label state lives in shared memory.
__global__ void k_chain(const ParArgs A, const int64_t *__restrict__ acc,
                        const int64_t *__restrict__ moves, const double *__restrict__ I,
                        double *__restrict__ tot, double *__restrict__ tsq,
                        const double *__restrict__ dtot_ps, int region_ps, int poisson,
                        double lam, double *__restrict__ energy, int32_t *__restrict__ ncomp) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int32_t nl = A.nl;
  int64_t *scnt = reinterpret_cast<int64_t *>(sm);
  double *stot = reinterpret_cast<double *>(scnt + nl);
  double *stsq = stot + nl;
  __shared__ double snap[32][6];
  const int lane = threadIdx.x;
  for (int l = lane; l < nl; l += 32) {
    scnt[l] = A.cnt0[l];
    stot[l] = tot[l];
    stsq[l] = tsq[l];
  }
  __syncwarp();
  const int64_t n = *moves;
  double e = *energy;
  for (int64_t base = 0; base < n; base += 32) {
    const int64_t k = base + lane;
    int64_t f = 0;
    int32_t a = 0, b = 0;
    double v = 0.0, dps = 0.0;
    if (k < n) {
      f = acc[3 * k];
      a = (int32_t)acc[3 * k + 1];
      b = (int32_t)acc[3 * k + 2];
      v = I[f];
      if (region_ps) dps = dtot_ps[k];
    }
    const int m = (n - base) < 32 ? (int)(n - base) : 32;
    for (int j = 0; j < m; ++j) {
      const int32_t aj = __shfl_sync(0xffffffffu, a, j);
      const int32_t bj = __shfl_sync(0xffffffffu, b, j);
      const double vj = __shfl_sync(0xffffffffu, v, j);
      if (lane == 0) {
        snap[j][0] = (double)scnt[aj];
        snap[j][1] = stot[aj];
        snap[j][2] = stsq[aj];
        snap[j][3] = (double)scnt[bj];
        snap[j][4] = stot[bj];
        snap[j][5] = stsq[bj];
        scnt[aj] -= 1;
        stot[aj] -= vj;
        stsq[aj] -= vj * vj;
        scnt[bj] += 1;
        stot[bj] += vj;
        stsq[bj] += vj * vj;
      }
    }
    __syncwarp();
    double d = dps;
    if (!region_ps && k < n) {
      const double na = snap[lane][0], nb = snap[lane][3];
      // delta_pc of the pre-move statistics (energy.py:308-324) + lam * dE_int
      double dext;
      if (!poisson) {
        double before = g_gauss(na, snap[lane][1], snap[lane][2]) +
                        g_gauss(nb, snap[lane][4], snap[lane][5]);
        double after = g_gauss(na - 1.0, snap[lane][1] - v, snap[lane][2] - v * v) +
                       g_gauss(nb + 1.0, snap[lane][4] + v, snap[lane][5] + v * v);
        dext = after - before;
      } else {
        double before = g_poisson(na, snap[lane][1]) + g_poisson(nb, snap[lane][4]);
        double after = g_poisson(na - 1.0, snap[lane][1] - v) + g_poisson(nb + 1.0, snap[lane][4] + v);
        dext = after - before;
      }
      d = dext + lam * (double)A.dint_acc[k];
    }
    for (int j = 0; j < m; ++j) e += __shfl_sync(0xffffffffu, d, j);
    __syncwarp();
  }
  for (int l = lane; l < nl; l += 32) {
    A.cnt[l] = scnt[l];
    tot[l] = stot[l];
    tsq[l] = stsq[l];
    if (l > 0 && scnt[l] == 0) ncomp[l] = 0;
  }
  if (lane == 0) *energy = e;
}

__global__ void k_final_labels(const ParArgs A, const uint32_t *__restrict__ slot, int64_t budget,
                               int32_t *__restrict__ L) {
  int64_t M = (int64_t)*A.nneg;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < M; i += stride) {
    if (A.dec[i] != ACC) continue;
    uint32_t p = A.order[i];
    int64_t f = A.px[p];
    A.w[f] = kInf;
    if ((int64_t)slot[i] < budget) L[f] = A.pcomp[p];
  }
}

// dE_int of each kept move in its view (needed by the PC ledger when lam != 0)
__global__ void k_dint_acc(const ParArgs A, const int64_t *__restrict__ acc,
                           const int64_t *__restrict__ moves) {
  const int64_t n = *moves;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride) {
    const int64_t f = acc[3 * k];
    View v{A, A.w[f]};
    int64_t z, y, x;
    A.lat.coord(f, z, y, x);
    A.dint_acc[k] = delta_internal_view(A, v, z, y, x, (int32_t)acc[3 * k + 1],
                                        (int32_t)acc[3 * k + 2]);
  }
}

// PS fields on the band touched by this iteration's moves: mark, recompute.
__global__ void k_mark_band(const int64_t *__restrict__ acc, const int64_t *__restrict__ moves,
                            Lat lat, const Off *__restrict__ ball_full, int nball_full,
                            uint8_t *__restrict__ dirty) {
  const int64_t n = *moves;
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t k = warp; k < n; k += nwarps) {
    int64_t z, y, x;
    lat.coord(acc[3 * k], z, y, x);
    for (int q = lane; q < nball_full; q += 32) {
      Off o = ball_full[q];
      int64_t zz = z + o.dz, yy = y + o.dy, xx = x + o.dx;
      if (lat.inb(zz, yy, xx)) dirty[lat.flat(zz, yy, xx)] = 1;
    }
  }
}

__global__ void k_refield_band(const int32_t *__restrict__ L, const double *__restrict__ I, Lat lat,
                               const Off *__restrict__ ball_full, int nball_full,
                               uint8_t *__restrict__ dirty, int32_t *__restrict__ Cown,
                               double *__restrict__ Sown) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < lat.V; f += stride) {
    if (!dirty[f]) continue;
    dirty[f] = 0;
    int64_t z, y, x;
    lat.coord(f, z, y, x);
    int32_t own = L[f];
    int32_t c = 0;
    double s = 0.0;
    for (int k = 0; k < nball_full; ++k) {
      Off o = ball_full[k];
      int64_t zz = z + o.dz, yy = y + o.dy, xx = x + o.dx;
      if (!lat.inb(zz, yy, xx)) continue;
      int64_t g = lat.flat(zz, yy, xx);
      if (L[g] != own) continue;
      c += 1;
      s += I[g];
    }
    Cown[f] = c;
    Sown[f] = s;
  }
}

size_t accept_par_smem() { return sizeof(BfsShared); }

int32_t accept_par(ParArgs A, const ParExtra &X, cudaStream_t s, int *launches) {
  static int grid_blocks = 0;
  const size_t smem = sizeof(BfsShared);
  if (grid_blocks == 0) {
    RCB_CUDA(cudaFuncSetAttribute(k_accept_par, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
    int per_sm = 0, dev = 0, sms = 0;
    RCB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_accept_par, 512, smem));
    RCB_CUDA(cudaGetDevice(&dev));
    RCB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    if (per_sm < 1) return fail(RCB_ERR_CUDA, "k_accept_par does not fit on an SM");
    grid_blocks = per_sm * sms;
  }
  void *args[] = {&A};
  RCB_CUDA(cudaLaunchCooperativeKernel((void *)k_accept_par, dim3(grid_blocks), dim3(512), args,
                                       smem, s));
  const int64_t N = X.n_particles;
  k_acc_flags<<<grid_for(N + 1, 256), 256, 0, s>>>(A.dec, A.nneg, X.slot);
  size_t bytes = 0;
  RCB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, X.slot, X.slot, N + 1, s));
  RCB_TRY(X.tmp->reserve(bytes, s));
  RCB_CUDA(cub::DeviceScan::ExclusiveSum(X.tmp->p, bytes, X.slot, X.slot, N + 1, s));
  k_acc_write<<<grid_for(N, 256), 256, 0, s>>>(A, X.slot, X.budget, X.acc, X.moves);
  k_dint_acc<<<grid_for(N, 256), 256, 0, s>>>(A, X.acc, X.moves);
  int nl = 6;
  if (X.region_ps) {
    k_ps_dtot<<<148 * 8, 256, 0, s>>>(A, X.acc, X.moves, X.I, X.ball, X.nball, X.poisson, X.lam,
                                      X.dtot);
    ++nl;
  }
  size_t csm = (size_t)A.nl * 24;
  if (csm > 200 * 1024) return fail(RCB_ERR_VALUE, "too many labels for the ledger chain");
  if (csm > 48 * 1024)
    RCB_CUDA(cudaFuncSetAttribute(k_chain, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csm));
  k_chain<<<1, 32, csm, s>>>(A, X.acc, X.moves, X.I, X.tot, X.tsq, X.dtot, X.region_ps, X.poisson,
                             X.lam, X.energy, X.ncomp);
  k_final_labels<<<grid_for(N, 256), 256, 0, s>>>(A, X.slot, X.budget, X.Lmut);
  if (X.region_ps) {
    k_mark_band<<<148 * 8, 256, 0, s>>>(X.acc, X.moves, A.lat, X.ball_full, X.nball_full, X.dirty);
    k_refield_band<<<grid_for(A.lat.V, 256), 256, 0, s>>>(X.Lmut, X.I, A.lat, X.ball_full,
                                                          X.nball_full, X.dirty, X.Cown, X.Sown);
    nl += 2;
  }
  RCB_CUDA(cudaGetLastError());
  *launches = nl + 8;
  return RCB_OK;
}

}  // namespace rcb
