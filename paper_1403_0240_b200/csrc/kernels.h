// Host-side launch wrappers of the kernels (internal to librcseg_b200).
#pragma once
#include <vector>

#include "common.cuh"

namespace rcb {


struct StatsScratch {
  DBuf<uint32_t> keys, vals_in, vals;
  DBuf<int64_t> bounds;
  DBuf<uint8_t> tmp;
  DBuf<double> gathered;
  DBuf<long long> isum;
  DBuf<unsigned long long> imax;
  DBuf<int> inot;
  void release(cudaStream_t s) {
    gathered.release(s);
    isum.release(s);
    imax.release(s);
    inot.release(s);
    keys.release(s);
    vals_in.release(s);
    vals.release(s);
    bounds.release(s);
    tmp.release(s);
  }
};

struct RankScratch {
  DBuf<uint64_t> tie, tie2, rkey, rkey2;
  DBuf<uint32_t> idx, idx2;
  DBuf<uint8_t> tmp;
  void release(cudaStream_t s) {
    tie.release(s);
    tie2.release(s);
    rkey.release(s);
    rkey2.release(s);
    idx.release(s);
    idx2.release(s);
    tmp.release(s);
  }
};

struct AcceptArgs {
  Lat lat;
  int full_fg, region_ps, poisson, mode_l2, allow_fusion, vanish_ok;
  double lam;
  int64_t budget;
  int64_t n;
  const uint32_t *order;
  const double *rank;
  const uint32_t *px;
  const int32_t *pown, *pcomp;
  int32_t *L;
  const double *I;
  int64_t *cnt;
  double *tot, *tsq;
  int32_t *Cown;
  double *Sown;
  double *rho0;
  const Off *ball;
  int nball;
  int32_t *ncomp;
  uint32_t *vis, *queue, *epoch;
  int64_t *acc;
  int64_t *moves;
  double *energy;
};

struct ParArgs {
  Lat lat;
  int allow_fusion, vanish_ok;
  int32_t nl;
  const unsigned long long *nneg;
  const uint32_t *order, *px;
  const int32_t *pown, *pcomp;
  const int32_t *L;  // iteration-start raster (read-only during the rounds)
  int32_t *newlab, *w, *pend;
  uint8_t *dec;
  int32_t *dround;
  uint8_t *small;
  int32_t *lab_pend, *nown;
  int64_t *cnt, *cnt0;
  int32_t *bfs_list, *ctl;
  uint32_t *vis, *epoch;
  uint32_t *gq[2];
  int32_t *dint_acc;
  int32_t *blocker;
  // dataflow acceptance (k_accept_df)
  int32_t *pos_of;           // position of each particle in the rank order (INF: rank >= 0)
  const uint32_t *site_off;  // K1 CSR (particles of a site)
  int32_t *lab_ptr;          // per small label: index of its next undecided event
  const int32_t *lab_pos;    // per small label: its candidates' positions, ascending
  int32_t *lbox;             // 2-D: per label (row min, row max, col min, col max)
  // large-footprint block BFS slots (one per block of k_accept_par)
  unsigned long long *bigkey;
  uint32_t *bigfr, *bigtag;
  uint8_t *bigfg;
  long long *tdbg;  // RCB_PROFILE: per position (fetch, decide, box, window) globaltimer ns
  int win_r;        // dataflow window radius in 2-D (0: default 5; 1: none)
  int wp_first;     // publish the site word before the decision's release fence (RCB_DF_WPFIRST=0: after)
  int help_after;   // settled waits look for assist jobs only after this many polls (RCB_DF_HELPAFTER)
  uint32_t div_mxy, div_lxy, div_mx, div_lx;  // f / (nx * ny) and f / nx by multiply-shift (f < 2^31)
  int lowmark_ns;   // longest poll interval of warps waiting for the low-water mark
  int idle_ns;      // poll interval of finished warps waiting for assist jobs
  int nowait;       // timing experiment only (RCB_DF_NOWAIT=1): ignore box dependencies, results are wrong
  int win5;         // 3-D: 5^3 window tier before the 9^3 window (RCB_DF_WIN5=0 turns it off)
  int max_insert;   // dataflow warp-BFS footprint cap (0: default)
  int box_cap;      // dataflow box-map BFS capacity in sites (-1: default, 0: off)
  unsigned long long *job, *ufp;  // dataflow assist jobs (accept_par.cu)
  unsigned long long *wp;         // dataflow site words (pend << 32 | w)
  unsigned long long *ufq;        // dataflow assist jobs: contracted-graph union-find
  unsigned long long *qmark;      // deferred-candidate registry: (seq << 32 | label) per site
  uint32_t *qlist;                // registered sites by sequence
  uint32_t *qscr;                 // assist-job scans: per-position neighbour masks
  unsigned long long *qstate;     // per label: Q-UF tag | S << 32, position reached; [2 nl + a]: label a ran assist jobs (sticky)
  int qjob;                       // 0: no registry (one full union-find per deferred candidate)
  int qprereg;                    // register every candidate of job-prone labels up front (RCB_DF_PREREG=0: off)
  unsigned long long watch_ns;    // dataflow watchdog: longest single wait
  int l2, poisson;                // l2 mode (PC): every label sequenced, d_tot < 0 gate
  double lam;
  const double *I;
  double *tot_run, *tsq_run;      // l2 mode: running region sums in acceptance order
  int wp_bits;                    // dataflow site-word layout: 24 (16-bit labels) or 27 (10-bit)
  uint32_t *bigmap;               // dataflow large box tier: per-warp 4-bit maps (big_words each)
  uint32_t *bigfr2;               // ... and frontiers (2 x big_fcap per warp)
  uint8_t *bigfg2;
  int big_words, big_fcap, big_levels2d;
  // per warp: words of its map set since the last clear (kBigTouch entries)
  // and {count, dirty range}: count < 0 or > kBigTouch = clear [0, range)
  uint32_t *bigtouch;
  int2 *bigtouch_n;
  const int4 *rec;                // dataflow per-position records
  // l2 mode, PS: the exact d_tot < 0 gate in the candidate's view
  // (iteration-start own-label fields + corrections of earlier flips within 2R)
  int region_ps;
  const int32_t *Cown, *cb0;
  const double *Sown, *rho0, *sb0;
  const Off *ball;  // non-centre ball offsets, ball_offsets order
  int nball, radius;
  int ps_flipcap;   // flip-list capacity used (tests: 0 forces the bitmap recount)
  const int32_t *ps_cells;  // cube indices (side 4R+1) of the 2R-ball offsets
  int ps_ncells;
};

// PS runs: the per-label total / total_sq chains (only the stats API and the
// sequential kernel read them; the next resync rebuilds them from the raster)
// are replayed lazily from the saved event lists, in iteration order.
struct PendingChain {
  DBuf<int64_t> acc;    // the iteration's accepted moves (x, a, b), acceptance order
  DBuf<int64_t> moves;  // their count (device scalar)
  int64_t cap = 0;
  int32_t nl = 0;
};

// z-slab sharded runs (integer band refresh): refresh the tiles meeting planes
// [z0, z1) and sum the band ledger over planes [own0, own1) only
struct BandSlab {
  int64_t z0, z1, own0, own1;
};
struct ParExtra {
  int64_t n_particles, budget;
  unsigned long long *hcount = nullptr;  // the engine's pinned word (candidate-list count)
  uint32_t *slot;
  DBuf<uint8_t> *tmp;
  int64_t *acc, *moves;
  const double *I;
  double *tot, *tsq, *energy, *dtot;
  int32_t *ncomp, *Lmut;
  int region_ps, poisson;
  double lam;
  const Off *ball, *ball_full;
  int nball, nball_full, radius;
  uint8_t *dirty;
  DBuf<uint8_t> *tflag = nullptr;  // 3-D band refresh: per-tile flip flags (zero between uses)
  const uint16_t *I16 = nullptr;   // integer image, 16 bits per site (integer band refresh), or null
  int4 *srec = nullptr;            // K5's packed site records, kept current by the integer band refresh
  bool *srec_current = nullptr;    // set when the band refresh left srec current
  const BandSlab *band_slab = nullptr;  // slab-local band refresh; the ledger stays in band[] for the ranks' all-reduce
  int32_t *Cown;
  double *Sown;
  double *rho0;
  const int32_t *cb0;   // per particle: competitor's iteration-start ball count at x (K5)
  const double *sb0;    // ... and ball sum
  DBuf<uint32_t> *evkey, *evkey2, *evval, *evval2;
  DBuf<int64_t> *bounds;
  DBuf<double> *snap, *evv;
  int accept_mode;  // 0 dataflow (default), 1 rounds
  DBuf<uint64_t> *labkey, *labkey2;
  DBuf<int32_t> *labpos, *labpos2, *flrows;
  DBuf<uint32_t> *fmap = nullptr;  // per-site flip map of the PS flip index (zero between uses)
  DBuf<int4> *rec;
  long long *band;  // band ledger: kLimbs superaccumulator limbs + dE_int sum
  DBuf<int32_t> *colb;
  DBuf<int64_t> *labbounds;
  std::vector<PendingChain> *pending = nullptr;
  std::vector<PendingChain> *chain_pool = nullptr;  // recycled chain buffers
  // integer image (sums exact in any order): no chain is kept -- the stats are
  // rebuilt from the raster when read (*stats_stale set), bit-identical
  bool *stats_stale = nullptr;  // PS: defer the total / total_sq chains here
  DBuf<uint32_t> *bigmap = nullptr, *bigfr2 = nullptr;  // dataflow large box tier (3-D)
  DBuf<uint8_t> *bigfg2 = nullptr;
  DBuf<uint32_t> *bigtouch = nullptr;
  DBuf<int2> *bigtouch_n = nullptr;
};

// input validation (energy.cu): one pass, one small read-back (synchronises s)
struct InputCheck {
  int32_t label_min, label_max;
  double image_min, image_max;
  int64_t nonint;  // finite non-integer intensities
  int64_t nonfinite;
};
int32_t check_inputs(const int32_t *L, const double *I, int64_t V, InputCheck *out, cudaStream_t s);
int32_t log_table(double *lt, int P, int Q, cudaStream_t s);
// K5 over packed site records (integer Poisson images)
bool ps_rec_ok(const Lat &lat, int nball_full, int32_t nl, double image_max);
int32_t pack_sites(const int32_t *L, const int32_t *Cown, const double *Sown, const double *I,
                   const double *rho0, int64_t V, int4 *rec, cudaStream_t s);
int32_t theta_table(double2 *tl, int P, int Q, cudaStream_t s);
int32_t delta_ps_rec(const int4 *rec, const double *I, const Lat &lat, const Off *ball, int nball,
                     const uint32_t *px, const int32_t *pown, const int32_t *pcomp, int64_t n,
                     double *out, const double *rho0, int32_t *cb0, double *sb0,
                     const double2 *tl, int tlP, int4 *pk, cudaStream_t s);
bool delta_ps_writes_pk(const Lat &lat, int nball);
int32_t sobolev_site_pk(const int4 *pk, double w0, int64_t p0, int64_t p1, int64_t lo, int64_t hi,
                        double *out, unsigned long long *pairs, cudaStream_t s);
int32_t sobolev_site_bulk(const int4 *pk, double w0, int64_t n, double *out,
                          unsigned long long *pairs, cudaStream_t s);
bool ps3d_tile_ok(const Lat &lat, int R, int nball);
int32_t delta_ps3d_tiles(const int32_t *L, const double *I, const int32_t *Cown,
                         const double *Sown, const double *rho0, const Lat &lat, int R,
                         const Off *ball, int nball, const uint32_t *site_off, const uint32_t *px,
                         const int32_t *pown, const int32_t *pcomp, int64_t h0, int64_t h1,
                         int poisson, double *out, int32_t *cb0, double *sb0, const double *lt,
                         int ltP, cudaStream_t s);

// contour.cu
int32_t contour_scan(const int32_t *L, const Lat &lat, int full_fg, uint32_t *site_off,
                     DBuf<uint8_t> &tmp, cudaStream_t s);
int32_t contour_emit(const int32_t *L, const Lat &lat, int full_fg, const uint32_t *site_off,
                     uint32_t *px, int32_t *pown, int32_t *pcomp, cudaStream_t s);
// energy.cu
int32_t delta_int_batch(const int32_t *L, const Lat &lat, const uint32_t *px, const int32_t *pown,
                        const int32_t *pcomp, int64_t n, int32_t *out, cudaStream_t s);
int32_t delta_pc_batch(const double *I, const uint32_t *px, const int32_t *pown,
                       const int32_t *pcomp, int64_t n, const int64_t *cnt, const double *tot,
                       const double *tsq, int poisson, double *out, cudaStream_t s,
                       int4 *pk = nullptr);
int32_t ps_fields(const int32_t *L, const double *I, const Lat &lat, const Off *ball_full,
                  int nball_full, int32_t *Cown, double *Sown, cudaStream_t s,
                  double *rho0 = nullptr, int poisson = 0, const uint16_t *I16 = nullptr);
int32_t fields_tile2d(const int32_t *L, const double *I, const Lat &lat, const Off *ball_full,
                      int nball_full, int R, uint8_t *dirty, int32_t *Cown, double *Sown,
                      double *rho0, int poisson, cudaStream_t s, long long *band = nullptr);
bool fields_tile2d_ok(const Lat &lat, int R, int nball_full);
int32_t fields_tile3d(const int32_t *L, const double *I, const Lat &lat, const Off *ball_full,
                      int nball_full, int R, uint8_t *dirty, int32_t *Cown, double *Sown,
                      double *rho0, int poisson, long long *band, cudaStream_t s);
bool fields_tile3d_ok(const Lat &lat, int R, int nball_full);
int64_t band3d_tiles(const Lat &lat);
int32_t band_ledger_apply(const long long *band, double lam, double *energy, cudaStream_t s);
int32_t fields_band3d(const int64_t *acc, const int64_t *moves, const int32_t *L, const double *I,
                      const uint16_t *I16, const Lat &lat, const Off *ball_full, int nball_full,
                      int R, uint8_t *flips, uint8_t *tflag, int32_t *Cown, double *Sown,
                      double *rho0, int poisson, long long *band, cudaStream_t s,
                      int4 *rec = nullptr, const BandSlab *slab = nullptr);
// integer image as 16-bit words (the integer band refresh reads 2 B per site)
int32_t image_u16(const double *I, int64_t V, uint16_t *I16, cudaStream_t s);
int32_t delta_ps_batch(const int32_t *L, const double *I, const int32_t *Cown, const double *Sown,
                       const Lat &lat, const Off *ball, int nball, const uint32_t *px,
                       const int32_t *pown, const int32_t *pcomp, int64_t n, int poisson,
                       double *out, cudaStream_t s, const double *rho0 = nullptr,
                       int32_t *cb0 = nullptr, double *sb0 = nullptr, const double *lt = nullptr,
                       int ltP = 0, int4 *pk = nullptr);
int32_t stats_rebuild(const int32_t *L, const double *I, int64_t V, int32_t nl, int64_t *cnt,
                      double *tot, double *tsq, StatsScratch &sc, cudaStream_t s);
int32_t pc_terms_exact(const int64_t *cnt, const double *tot, const double *tsq, int32_t nl,
                       int poisson, long long *limbs, cudaStream_t s);
int32_t ps_terms_exact(const int32_t *Cown, const double *Sown, const double *I, int64_t V,
                       int poisson, long long *limbs, cudaStream_t s);
int32_t perimeter(const int32_t *L, const Lat &lat, unsigned long long *out, cudaStream_t s);
double limbs_to_double(const long long *limbs);
// sobolev.cu
std::vector<Off> sobolev_stencil(int ndim, double length_scale);
std::vector<Off> sobolev_rows(int ndim, double length_scale, int *max_d2);
int32_t sobolev_lattice(const uint32_t *site_off, const int32_t *pown, const uint32_t *px,
                        const int32_t *pcomp, const double *raw, const Lat &lat, const Off *rows,
                        int nrows, const double *wt, int64_t n, double *out,
                        unsigned long long *pairs, cudaStream_t s, int64_t p0 = 0);
bool sobolev_packable(int32_t n_labels, int nrows, int max_d2);
int32_t sobolev_pack(const uint32_t *px, const int32_t *pown, const int32_t *pcomp,
                     const double *raw, int64_t lo, int64_t hi, int4 *pk, cudaStream_t s);
bool sobolev_site_only(const Off *rows_host, int nrows);
int32_t sobolev_site(const uint32_t *px, const int32_t *pown, const int32_t *pcomp,
                     const double *raw, double w0, int64_t p0, int64_t p1, int64_t lo, int64_t hi,
                     double *out, unsigned long long *pairs, cudaStream_t s);
int32_t sobolev_packed(const uint32_t *site_off, const int4 *pk, const Lat &lat, const Off *rows,
                       int nrows, const double *wt, int nwt, int64_t p0, int64_t p1, double *out,
                       unsigned long long *pairs, cudaStream_t s);
int32_t sobolev_coords(const int64_t *d_coords, int64_t n, int ndim, const Lat &lat,
                       const int64_t *d_owners, const int64_t *d_comps, const double *d_raw,
                       const Off *st, int nst, const double *wt, double *d_out,
                       unsigned long long *d_pairs, cudaStream_t s);
// fp32 gradient path
int32_t to_float(const double *src, int64_t n, float *dst, cudaStream_t s);
int32_t delta_pc32_batch(const float *I32, const uint32_t *px, const int32_t *pown,
                         const int32_t *pcomp, int64_t n, const int64_t *cnt, const double *tot,
                         int poisson, float *out32, double *out, cudaStream_t s);
int32_t delta_ps32_batch(const int32_t *L, const float *I32, const int32_t *Cown,
                         const double *Sown, const Lat &lat, const Off *ball, int nball,
                         const uint32_t *px, const int32_t *pown, const int32_t *pcomp, int64_t n,
                         int poisson, float *out32, double *out, cudaStream_t s,
                         int32_t *cb0 = nullptr, double *sb0 = nullptr);
int32_t sobolev_lattice32(const uint32_t *site_off, const int32_t *pown, const uint32_t *px,
                          const int32_t *pcomp, const float *raw, const Lat &lat, const Off *rows,
                          int nrows, const float *wt, int64_t n, double *out,
                          unsigned long long *pairs, cudaStream_t s, int64_t p0 = 0);
// rank.cu
int32_t rank_order(const double *base, const int32_t *dint, double lam, int64_t n,
                   const uint32_t *px, const int32_t *pcomp, uint64_t seed, double *rank,
                   RankScratch &sc, uint32_t *order, unsigned long long *nneg, cudaStream_t s);
void gather_u64(const uint64_t *src, const uint32_t *idx, int64_t n, uint64_t *dst,
                cudaStream_t s);
// accept.cu
int32_t accept_seq(const AcceptArgs &args, cudaStream_t s);
int32_t label_components(const int32_t *L, const Lat &lat, int full_fg, int32_t nl,
                         uint32_t *par_scratch, int32_t *ncomp, cudaStream_t s);

// accept_par.cu
int32_t accept_par(ParArgs A, const ParExtra &X, cudaStream_t s, int *launches);
// replay (then release) deferred total / total_sq chains in order
int32_t replay_chains(std::vector<PendingChain> &pending, const double *I, double *tot,
                      double *tsq, cudaStream_t s,
                      std::vector<PendingChain> *pool = nullptr);
// pool != nullptr: keep the buffers there for reuse (no per-iteration
// cudaMallocAsync of 10^8-byte lists, which mapped memory for ms at cfg4)
void drop_chains(std::vector<PendingChain> &pending, cudaStream_t s,
                 std::vector<PendingChain> *pool = nullptr);
size_t accept_par_smem();

// tables (abi.cu)
std::vector<Off> ball_table(int ndim, int r);  // ball_offsets order, centre first

}  // namespace rcb
