/*
 * rcb.h — C ABI of the B200-native Region Competition hot path
 * (librcseg_b200.so, built for sm_100a).
 *
 * The reference (rcseg, /root/reference/pkg/src/rcseg) is pure Python on
 * numpy arrays; it has no FFI.  Each entry point below replaces one reference
 * function and is what a maintainer would bind with ctypes.
 * All arrays are plain C-order host pointers; sizes are explicit; no torch
 * types.  Lattices are described by (ndim, dims[ndim]); flat indices are
 * C-order over dims, exactly as in the reference (grid.py:1-8).
 *
 * Every function returns RCB_OK (0) or a negative status; the message of the
 * last failure on the calling thread is rcb_last_error().  The Python shim
 * maps statuses to the reference's exception types (ValueError,
 * RuntimeError, DegenerateStatsError, StaleParticleError).
 */
#ifndef RCB_H
#define RCB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RCB_OK 0
#define RCB_ERR_VALUE -1      /* bad argument            -> ValueError */
#define RCB_ERR_CUDA -2       /* CUDA runtime failure     -> RuntimeError */
#define RCB_ERR_CAPACITY -3   /* output buffer too small; *n holds the size needed */
#define RCB_ERR_DEGENERATE -4 /* empty region mean        -> DegenerateStatsError */
#define RCB_ERR_NODEVICE -5   /* no CUDA device           -> RuntimeError */

/* energy.py:37-50  EnergyConfig */
typedef struct {
    int32_t region_model;   /* 0 = "pc", 1 = "ps" */
    int32_t noise_model;    /* 0 = "gauss", 1 = "poisson" */
    double lam;
    int32_t smooth_radius;
} rcb_energy_cfg;

/* sobolev.py:18-31 SobolevParams, plus the host-evaluated kernel table
 * w[d2] = kernel_eval(sqrt(d2)) for every integer d2 < (E/2)^2
 * (sobolev.py:34-49, 121). */
typedef struct {
    double length_scale;
    double epsilon;
    const double *weights;  /* n_weights entries, copied at create time */
    int32_t n_weights;
} rcb_sobolev_cfg;

/* optimizer.py:36-56 OptimizerConfig (the fields the device iteration uses;
 * oscillation/resync/drift policy stays in the host driver). */
typedef struct {
    int32_t gradient;       /* 0 = "l2", 1 = "sobolev" */
    double move_budget;
    uint64_t seed;
    int32_t allow_fusion;
    int32_t allow_vanish;
    int32_t vanish_grace;
    int32_t full_fg;        /* Connectivity: 1 = default (8/26 fg), 0 = (4/6 fg) */
    int32_t fp32;           /* 1: fp32 gradient path (raw increments, Sobolev filter);
                               statistics, fields, ledger and totals stay fp64 */
} rcb_opt_cfg;

/* optimizer.py:58-65 IterationRecord (device part). */
typedef struct {
    int64_t iteration;
    double energy;          /* incremental ledger after the iteration */
    int64_t moves;
    int64_t particles;      /* len(contour) after the iteration */
    int64_t candidates;     /* particles scored this iteration */
    int64_t negative;       /* candidates with rank < 0 */
    int64_t pairs;          /* Sobolev particle interactions (0 in l2 mode) */
    int32_t mode;           /* 0 = l2, 1 = sobolev */
} rcb_iter_record;

typedef struct rcb_engine rcb_engine;

int32_t rcb_version(void);
const char *rcb_last_error(void);
int32_t rcb_device_count(int32_t *n);

/* ---- function-level drop-ins ------------------------------------------ */

/* sobolev.py:137-174 sobolev_filter(coords, owners, competitors, raw, params)
 * coords: n x ndim int64 (non-negative); out: n doubles.  *n_pairs receives
 * the interaction count len(CellList.pairs(cutoff)[0]) (sobolev.py:99-122). */
int32_t rcb_sobolev_filter(const int64_t *coords, int64_t n, int32_t ndim,
                           const int64_t *owners, const int64_t *competitors,
                           const double *raw, const rcb_sobolev_cfg *params,
                           double *out, int64_t *n_pairs);

/* contour.py:84-116 scan_contour(labels, conn) + as_arrays: particles sorted
 * by (x, competitor).  If cap < count, returns RCB_ERR_CAPACITY with *n set. */
int32_t rcb_scan_contour(const int32_t *labels, int32_t ndim, const int64_t *dims,
                         int32_t full_fg, int64_t *xs, int64_t *owners,
                         int64_t *competitors, int64_t cap, int64_t *n);

/* energy.py:111-126 delta_internal_batch(labels, pixels, owners, competitors) */
int32_t rcb_delta_internal_batch(const int32_t *labels, int32_t ndim, const int64_t *dims,
                                 const int64_t *xs, const int64_t *owners,
                                 const int64_t *competitors, int64_t n, int64_t *out);

/* energy.py:302-372 EnergyModel.delta_external_batch.  PC reads the caller's
 * region statistics (count/total/total_sq, n_labels entries — the model's
 * StatsTable, grid.py:142-188); PS rebuilds the ball fields from labels. */
int32_t rcb_delta_external_batch(const double *image, const int32_t *labels, int32_t ndim,
                                 const int64_t *dims, const rcb_energy_cfg *cfg,
                                 int32_t n_labels, const int64_t *count, const double *total,
                                 const double *total_sq, const int64_t *xs,
                                 const int64_t *owners, const int64_t *competitors, int64_t n,
                                 double *out);

/* grid.py:155-169 StatsTable.from_labels (raster-order sequential sums). */
int32_t rcb_stats_from_labels(const double *image, const int32_t *labels, int64_t size,
                              int32_t n_labels, int64_t *count, double *total,
                              double *total_sq);

/* energy.py:233-257 evaluate_total -> (external, internal); the external
 * sum is correctly rounded like math.fsum. */
int32_t rcb_evaluate_total(const double *image, const int32_t *labels, int32_t ndim,
                           const int64_t *dims, const rcb_energy_cfg *cfg, double *external,
                           int64_t *internal);

/* grid.py:99-113 flood_fill_components / count_components: components of
 * (labels == target) minus site `exclude` (-1: none) under the foreground
 * adjacency, numbered 1..n in first-encountered raster order like
 * ndimage.label; comp (nullable) receives the numbering (0 elsewhere). */
int32_t rcb_label_components(const int32_t *labels, int32_t ndim, const int64_t *dims,
                             int32_t full_fg, int32_t target, int64_t exclude, int32_t *comp,
                             int64_t *n_components);

/* contour.py:171-207 is_move_admissible for n (pixel, competitor) queries
 * against one raster; region_counts (nullable; entries < 0 = count it) is
 * the reference's region_count argument.  out[i] = 1 admissible, 0 not. */
int32_t rcb_moves_admissible(const int32_t *labels, int32_t ndim, const int64_t *dims,
                             int32_t full_fg, const int64_t *pixels, const int64_t *competitors,
                             const int64_t *region_counts, int64_t n, int32_t allow_fusion,
                             int32_t allow_vanish, int32_t *out);

/* sobolev.py:99-122 CellList(coords, edge).pairs(cutoff): every ordered
 * pair (p, q), p == q included, whose buckets (floor_divide(coords, edge))
 * are box neighbours and whose squared distance is < cutoff^2; sorted by
 * (p, q).  RCB_ERR_CAPACITY with *n_pairs set when cap is too small. */
int32_t rcb_cell_pairs(const int64_t *coords, int64_t n, int32_t ndim, double edge,
                       double cutoff, int64_t *pi, int64_t *qi, double *dist, int64_t cap,
                       int64_t *n_pairs);
/* sobolev.py:80-93 CellList.query(point, cutoff, exclude): ascending
 * indices (out has room for n); exclude < 0 = none. */
int32_t rcb_cell_query(const int64_t *coords, int64_t n, int32_t ndim, double edge,
                       const double *point, double cutoff, int64_t exclude, int64_t *out,
                       int64_t *n_out);

/* energy.py:161-193 _ball_sum(field, radius): ball convolution with zero
 * borders, by the reference's cumulative-sum spans (same rounding). */
int32_t rcb_ball_sum(const double *field, int32_t ndim, const int64_t *dims, int32_t radius,
                     double *out);
/* energy.py:196-223 smooth_fields(labels, image, radius, n_labels): dense
 * C, S of n_labels x V doubles each (per-label window = bounding box grown
 * by the radius, as the reference computes it). */
int32_t rcb_smooth_fields(const int32_t *labels, const double *image, int32_t ndim,
                          const int64_t *dims, int32_t radius, int32_t n_labels, double *C,
                          double *S);

/* ---- the engine: RegionCompetition (optimizer.py:90-230) --------------- */

/* image: float64 C-order (optimizer.py:102); labels: int32 (copied).
 * stream: a cudaStream_t to launch on (NULL = a private stream). */
int32_t rcb_engine_create(const double *image, const int32_t *labels, int32_t ndim,
                          const int64_t *dims, const rcb_energy_cfg *ecfg,
                          const rcb_sobolev_cfg *scfg, const rcb_opt_cfg *ocfg,
                          int32_t device, void *stream, rcb_engine **out);
/* As rcb_engine_create, with the image given as float64 (image_dtype 0) or
 * float32 (1): a float32 raster crosses PCIe at 4 B/site and is promoted on
 * the device, exactly as the reference's np.ascontiguousarray(image,
 * float64) promotes it on the host (optimizer.py:102). */
int32_t rcb_engine_create_ex(const void *image, int32_t image_dtype, const int32_t *labels,
                             int32_t ndim, const int64_t *dims, const rcb_energy_cfg *ecfg,
                             const rcb_sobolev_cfg *scfg, const rcb_opt_cfg *ocfg,
                             int32_t device, void *stream, rcb_engine **out);
void rcb_engine_destroy(rcb_engine *eng);
/* optimizer.py:122-160 iterate(): extraction, ΔE, Sobolev, rank, acceptance. */
int32_t rcb_engine_iterate(rcb_engine *eng, rcb_iter_record *rec);
int32_t rcb_engine_get_labels(rcb_engine *eng, int32_t *out);
int32_t rcb_engine_set_labels(rcb_engine *eng, const int32_t *labels);
/* Undo the last iteration's accepted moves on the device (the restore of
 * optimizer.py:259-265's oscillation halt without a per-iteration host copy
 * of the raster); refresh the statistics afterwards (rcb_engine_refresh). */
int32_t rcb_engine_undo_last(rcb_engine *eng);
/* last_candidates (optimizer.py:140-142): (x, owner, competitor, rank). */
int32_t rcb_engine_get_candidates(rcb_engine *eng, int64_t *xs, int64_t *owners,
                                  int64_t *competitors, double *rank, int64_t cap, int64_t *n);
/* accepted moves of the last iteration in acceptance order, as (x, a, b). */
int32_t rcb_engine_get_accepted(rcb_engine *eng, int64_t *xab, int64_t cap, int64_t *n);
int32_t rcb_engine_get_stats(rcb_engine *eng, int64_t *count, double *total, double *total_sq,
                             int32_t n_labels);
int32_t rcb_engine_n_labels(rcb_engine *eng, int32_t *n_labels);
int32_t rcb_engine_set_mode(rcb_engine *eng, int32_t gradient);
int32_t rcb_engine_set_energy(rcb_engine *eng, double energy);
/* EnergyModel.refresh (energy.py:285-291): rebuild stats and PS fields. */
int32_t rcb_engine_refresh(rcb_engine *eng);
/* evaluate_total on the engine's current device state. */
int32_t rcb_engine_evaluate(rcb_engine *eng, double *external, int64_t *internal);
int32_t rcb_engine_stream(rcb_engine *eng, void **stream);
/* Device time (ms) of the last iterate() phases, CUDA events on the engine
 * stream: [0] extract, [1] energy, [2] sobolev, [3] rank/sort, [4] accept,
 * [5] whole iteration.  Also the kernel launch count of the last iterate. */
int32_t rcb_engine_timings(rcb_engine *eng, float *ms6, int32_t *launches);
/* Acceptance diagnostics of the last iterate(): [0] rounds, [1] block BFS
 * runs, [2] deferred to the global BFS, [3] BFS aborted on a pending site,
 * [4] candidates with rank < 0, [5] accepted moves, [6] 1 if the parallel
 * acceptance ran (0 = sequential), [7] device us of the acceptance kernels,
 * [8] total BFS levels (dataflow: union-find rebuilds of the deferred-candidate
 * jobs), [9] deepest BFS (dataflow: rebuilds forced by a non-simple removal),
 * [10] PS ledger recounts of
 * flipped ball sites, [11] flips gathered by the PS ledger terms. */
int32_t rcb_engine_counters(rcb_engine *eng, int64_t *out12);
/* Diagnostics of the last parallel acceptance: for rank position i < *n,
 * particle[i] (index into last_candidates) and code[i] (decision path). */
int32_t rcb_engine_debug_codes(rcb_engine *eng, int32_t *particle, int32_t *code, int64_t cap,
                               int64_t *n);
/* RCB_PROFILE=1: (fetch, decide, box done, window done) globaltimer ns per
 * rank position of the last dataflow acceptance (t4 holds 4 * cap values). */
int32_t rcb_engine_debug_times(rcb_engine *eng, int64_t *t4, int64_t cap, int64_t *n);

/* ---- z-slab sharding: one engine per GPU ------------- *
 * Every rank holds the whole raster (512^3 needs ~12 GB with the own-label
 * field layout, against 180 GB per B200) and runs the identical rank order and
 * acceptance on it, so decisions agree bit for bit without exchanging them.
 * The scoring kernels are split by outer planes (z in 3-D, rows in 2-D):
 * rank r computes ΔE (K3/K5) for its slab plus the Sobolev stencil's halo and
 * the Sobolev filter (K6) for its slab; the exchange step is an all-gather of
 * each slab's scores (base, and for PS the competitor ball terms cb0/sb0)
 * into the same offsets on every rank.  iterate() == score() + finish(). */
typedef struct {
    int64_t n_particles;    /* particles scored this iteration (all slabs) */
    int64_t p0, p1;         /* this slab's particle range [p0, p1) */
    void *base;             /* device double[n]: smoothed (sobolev) or raw (l2) ΔE */
    void *cb0;              /* device int32[n] (PS only, else NULL) */
    void *sb0;              /* device double[n] (PS only, else NULL) */
    void *stream;           /* cudaStream_t the scores were computed on */
} rcb_slab_info;

/* Outer planes [lo, hi) this engine scores; hi <= lo = the whole lattice. */
int32_t rcb_engine_set_slab(rcb_engine *eng, int64_t lo, int64_t hi);
/* First half of iterate(): K1 emit, ΔE_int, ΔE, Sobolev over the slab. */
int32_t rcb_engine_score(rcb_engine *eng, rcb_slab_info *info);
/* Second half, after every slab's [p0, p1) of base/cb0/sb0 is in place:
 * rank order, acceptance and bookkeeping (replicated on every rank). */
int32_t rcb_engine_finish(rcb_engine *eng, rcb_iter_record *rec);
/* z-slab sharded 3-D PS runs on integer images refresh the own-label fields of
 * the slab plus its halo only and sum the exact band ledger over the slab:
 * after finish, *pending = 1 means limbs[0 .. n_limbs) (int64, device memory,
 * engine stream *stream) hold this rank's share of the iteration's energy
 * change and rec->energy is still the previous energy.  The host sums the
 * limbs over the ranks (one all-reduce of n_limbs int64: exact), writes the
 * sums back and calls rcb_engine_band_apply, which rounds them once into the
 * ledger (energy.py:233-257 semantics, as on one GPU) and returns the energy.
 * With *pending = 0 nothing is to be done (band_apply returns the energy). */
int32_t rcb_engine_band_limbs(rcb_engine *eng, void **limbs, int32_t *n_limbs, int32_t *pending,
                              void **stream);
int32_t rcb_engine_band_apply(rcb_engine *eng, double *energy);
/* Particle index of the first site of each outer plane planes[i] (clamped
 * to [0, planes]); a slab [lo, hi) owns [out(lo), out(hi)). */
int32_t rcb_engine_particle_ranges(rcb_engine *eng, const int64_t *planes, int32_t k,
                                   int64_t *out);

/* ---- synthetic-data pipeline (rcseg/synth.py) --------- *
 * shapes: 15 doubles per shape, in scene order (later shapes overwrite):
 * [kind (0 disk/ball, 1 rect/box, 2 annulus/shell), intensity, ncenter,
 *  c0, c1, c2, r2lo, r2hi (disk: -inf, radius**2; annulus: inner**2,
 *  outer**2), nbox, lo0, lo1, lo2, hi0, hi1, hi2 (rect: origin, origin+size)].
 * kernel: the normalised Gaussian taps of synth.py:96-99 (klen odd; 0 = no
 * blur).  psnr2 = psnr**2.  Results are bit-identical to the reference.     */
/* synth.py:185-192 generate(): render (synth.py:73-84), blur (:87-103) and,
 * if noise != 0, poissonize (:169-182) on the device; labels / clean / image
 * may be NULL (not copied back). */
int32_t rcb_synth_generate(int32_t ndim, const int64_t *dims, double background,
                           const double *shapes, int32_t nshapes, const double *kernel,
                           int32_t klen, int32_t noise, double psnr2, uint64_t seed,
                           int32_t *labels, double *clean, double *image);
/* synth.py:87-103 blur() of a float64 image. */
int32_t rcb_synth_blur(const double *image, int32_t ndim, const int64_t *dims,
                       const double *kernel, int32_t klen, double *out);
/* synth.py:169-182 poissonize() of n float64 intensities. */
int32_t rcb_synth_poissonize(const double *image, int64_t n, double psnr2, uint64_t seed,
                             double *out);

/* ---- Sobolev sweep workload (BASELINE configs[4], second part) --------- */
typedef struct rcb_sweep rcb_sweep;
/* Paint the union of nsph spheres (z, y, x, r as float, 4 per sphere) into a
 * zero lattice on the device, extract the contour particles (K1) and draw
 * raw ~ N(0,1) from a seeded counter hash of (site, competitor). */
int32_t rcb_sweep_create(int32_t ndim, const int64_t *dims, const float *spheres, int32_t nsph,
                         uint64_t seed, const rcb_sobolev_cfg *scfg, int32_t device,
                         rcb_sweep **out);
void rcb_sweep_destroy(rcb_sweep *sweep);
int32_t rcb_sweep_info(rcb_sweep *sweep, int64_t *n_particles, int64_t *n_sites, void **stream);
/* One K6 launch over the resident particles: interactions and device ms. */
int32_t rcb_sweep_run(rcb_sweep *sweep, int64_t *pairs, float *ms);
int32_t rcb_sweep_get(rcb_sweep *sweep, int64_t *xs, int64_t *owners, int64_t *comps,
                      double *raw, double *out, int64_t cap);

#ifdef __cplusplus
}
#endif
#endif /* RCB_H */
