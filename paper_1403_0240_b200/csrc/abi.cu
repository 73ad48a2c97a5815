#include <mutex>
#include <chrono>
// C ABI of librcseg_b200 (include/rcb.h): the device engine that replaces
// RegionCompetition.iterate (optimizer.py:122-160) and the function-level
// drop-ins.  Each entry point cites the reference function it replaces.
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <cstdio>
#include <string>
#include <vector>

#include "kernels.h"

namespace rcb {

static thread_local std::string g_err;

void set_error(const std::string &msg) { g_err = msg; }
int32_t fail(int32_t code, const std::string &msg) {
  g_err = msg;
  return code;
}

std::vector<Off> ball_table(int ndim, int r) {
  // energy.py:60-70 ball_offsets: |o|^2 <= r^2, |o|^2 ascending, stable over
  // lexicographic order, centre first.
  std::vector<Off> out;
  for (int dz = (ndim == 3 ? -r : 0); dz <= (ndim == 3 ? r : 0); ++dz)
    for (int dy = -r; dy <= r; ++dy)
      for (int dx = -r; dx <= r; ++dx) {
        int d2 = dz * dz + dy * dy + dx * dx;
        if (d2 <= r * r) out.push_back(Off{(int8_t)dz, (int8_t)dy, (int8_t)dx, (uint8_t)d2});
      }
  std::stable_sort(out.begin(), out.end(), [](const Off &a, const Off &b) { return a.aux < b.aux; });
  return out;
}

template <typename T>
static int32_t upload(DBuf<T> &d, const T *h, size_t n, cudaStream_t s) {
  RCB_TRY(d.reserve(n ? n : 1, s));
  if (n) RCB_CUDA(cudaMemcpyAsync(d.p, h, n * sizeof(T), cudaMemcpyHostToDevice, s));
  return RCB_OK;
}

static int32_t check_device() {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    return fail(RCB_ERR_NODEVICE, std::string("no CUDA device: ") + cudaGetErrorString(e));
  return RCB_OK;
}

static int32_t check_lattice(int32_t ndim, const int64_t *dims) {
  if (ndim != 2 && ndim != 3) return fail(RCB_ERR_VALUE, "raster must be 2-D or 3-D");
  int64_t V = 1;
  for (int k = 0; k < ndim; ++k) {
    if (dims[k] < 1) return fail(RCB_ERR_VALUE, "raster dimensions must be positive");
    V *= dims[k];
  }
  if (V >= (int64_t)0xffffffffll) return fail(RCB_ERR_VALUE, "raster larger than 2^32-1 sites");
  return RCB_OK;
}

// small device-side scalar block, mirrored into pinned host memory once per
// iteration (the only D2H traffic of iterate()).
struct Scalars {
  double energy;
  int64_t moves;
  uint32_t epoch;
  uint32_t pad;
  unsigned long long pairs;
  unsigned long long nneg;
  unsigned long long perim;
  uint32_t n_next;
  uint32_t pad2;
  long long limbs[kLimbs];
};

}  // namespace rcb

using namespace rcb;

namespace {
// Pinned host blocks for the engines' small read-back buffers, recycled
// across engines: cudaMallocHost pins pages and can take milliseconds, which
// showed up as constructor jitter in the end-to-end timing.
constexpr size_t kPinnedBlock = 4096;
std::mutex g_pinned_mu;
std::vector<void *> g_pinned_free;
void *pinned_get() {
  {
    std::lock_guard<std::mutex> g(g_pinned_mu);
    if (!g_pinned_free.empty()) {
      void *p = g_pinned_free.back();
      g_pinned_free.pop_back();
      return p;
    }
  }
  void *p = nullptr;
  return cudaMallocHost(&p, kPinnedBlock) == cudaSuccess ? p : nullptr;
}
void pinned_put(void *p) {
  if (!p) return;
  std::lock_guard<std::mutex> g(g_pinned_mu);
  g_pinned_free.push_back(p);
}

}  // namespace

struct rcb_engine {
  int device = 0;
  cudaStream_t s = nullptr;
  bool own_stream = false;
  Lat lat{};
  int32_t nl = 0;
  rcb_energy_cfg ecfg{};
  rcb_opt_cfg ocfg{};
  int64_t iteration = 0;
  int mode = 1;
  bool prepared = false;
  bool fields_fresh = false;  // stats/fields were just rebuilt from the raster (refresh)
  int64_t N = 0;  // particles of the current raster (valid when prepared)
  int64_t n_scored = 0, last_moves = 0;

  DBuf<int32_t> L;
  DBuf<double> I;
  DBuf<float> I32, raw32, wt32;  // fp32 mode
  DBuf<int32_t> cb0;             // PS: competitor ball count/sum per particle (K5)
  DBuf<double> sb0;
  DBuf<int64_t> cnt;
  DBuf<double> tot, tsq;
  DBuf<int32_t> Cown;
  DBuf<double> Sown, rho0;
  DBuf<double> logt;  // K5 Poisson log table (integer images), logt_P columns
  int logt_P = 0;
  DBuf<int4> srec;        // K5 packed site records (ps_rec_ok)
  DBuf<double2> thetat;   // K5 {theta, log theta} table, thetat_P columns
  int thetat_P = 0;
  DBuf<Off> ball, ball_full, st;
  int nball = 0, nball_full = 0, nst = 0;
  DBuf<double> wt;
  DBuf<int32_t> ncomp;
  DBuf<uint32_t> vis, queue;
  DBuf<uint32_t> site_off, px, order;
  DBuf<int32_t> pown, pcomp, dint;
  DBuf<double> raw, smooth, rank, tot_run, tsq_run;
  bool cur_par = false;
  DBuf<int4> pk;  // K6 packed partner records
  bool sob_packed = false;
  bool sob_site = false;  // w = 1: the stencil is the particle's own site (k_sobolev_site)
  double w0 = 0.0;
  int nwt = 0;
  DBuf<int64_t> acc;
  // parallel acceptance state (accept_par.cu)
  DBuf<int32_t> newlab, wpos, pend, dround, lab_pend, nown, bfs_list, ctl, dint_acc, blocker;
  DBuf<uint8_t> dec, small, dirty;
  DBuf<int64_t> cnt0;
  DBuf<uint32_t> gq1, slot;
  DBuf<double> dtot, snap, evv;
  DBuf<uint32_t> evkey, evkey2, evval, evval2;
  DBuf<int64_t> evbounds;
  DBuf<uint64_t> labkey, labkey2;
  DBuf<int32_t> labpos, labpos2, pos_of, lab_ptr, lbox, flrows, colb;
  DBuf<uint32_t> fmap;
  DBuf<unsigned long long> ufp, job, wpk, eval_per, ufq, qmark, qstate;
  DBuf<uint32_t> qlist, qscr, bigmap, bigfr2;
  DBuf<uint8_t> bigfg2;
  DBuf<uint32_t> bigtouch;
  DBuf<uint8_t> tflag;
  DBuf<uint16_t> I16;     // integer image as 16-bit words (integer band refresh), empty otherwise
  DBuf<int32_t> ps_cells;  // l2 PS gate: the 2R ball as cube indices
  int ps_ncells = 0;
  DBuf<int2> bigtouch_n;
  DBuf<long long> eval_limbs, band;
  DBuf<int4> rec;
  DBuf<unsigned long long> bigkey;
  DBuf<long long> tdbg;
  bool profile = false;
  DBuf<uint32_t> bigfr, bigtag;
  DBuf<uint8_t> bigfg;
  DBuf<int64_t> labbounds;
  int accept_mode = 0;
  bool simple_topology = false;
  bool force_sequential = false;
  DBuf<Scalars> sc;
  DBuf<uint8_t> tmp;
  StatsScratch ssc;
  RankScratch rsc;
  Scalars *hsc = nullptr;  // pinned
  cudaEvent_t ev[6] = {};
  cudaEvent_t ev_acc[2] = {};
  int32_t *hctl = nullptr;  // pinned (in the pinned block): acceptance counters read back
  int64_t counters[12] = {};
  bool last_par = false;
  float times[6] = {};
  int32_t launches = 0;
  // z-slab sharding (rcb_engine_set_slab): outer planes [slab_lo, slab_hi)
  int64_t slab_lo = 0, slab_hi = 0, stencil_reach = 0;
  int64_t p0 = 0, p1 = 0;  // own particle range of the last score
  bool scored = false;
  int score_launches = 0;
  uint32_t *hoff = nullptr;  // pinned: site_off reads
  unsigned long long *hwatch = nullptr;  // pinned: dataflow watchdog words (job[56..61])
  void *pinned = nullptr;                // the pinned block hsc / hoff / hwatch live in
  // set when the dataflow watchdog fired: the kernels after the decisions ran on
  // a partly filled decision array, so labels / statistics / ledger are
  // undefined and every later call fails (destroy the engine)
  bool poisoned = false;
  std::string poison_msg;

  ~rcb_engine() {
    if (s) {
      cudaSetDevice(device);
      L.release(s); I.release(s); I32.release(s); raw32.release(s); wt32.release(s);
      cb0.release(s); sb0.release(s); cnt.release(s); tot.release(s); tsq.release(s);
      Cown.release(s); Sown.release(s); logt.release(s); srec.release(s); thetat.release(s); rho0.release(s); ball.release(s); ball_full.release(s); st.release(s);
      wt.release(s); ncomp.release(s); vis.release(s); queue.release(s); site_off.release(s);
      px.release(s); order.release(s); pown.release(s); pcomp.release(s); dint.release(s);
      raw.release(s); smooth.release(s); rank.release(s); pk.release(s); tot_run.release(s);
      tsq_run.release(s); acc.release(s); sc.release(s);
      newlab.release(s); wpos.release(s); pend.release(s); dround.release(s); lab_pend.release(s);
      nown.release(s); blocker.release(s); bfs_list.release(s); ctl.release(s); dint_acc.release(s); dec.release(s);
      small.release(s); dirty.release(s); cnt0.release(s); gq1.release(s); slot.release(s);
      dtot.release(s); snap.release(s); evv.release(s); evkey.release(s); evkey2.release(s); evval.release(s);
      evval2.release(s); evbounds.release(s); labkey.release(s); labkey2.release(s);
      labpos.release(s); labpos2.release(s); pos_of.release(s); flrows.release(s); fmap.release(s); bigkey.release(s);
      bigfr.release(s); bigtag.release(s); bigfg.release(s); tdbg.release(s); lab_ptr.release(s); lbox.release(s); colb.release(s);
      ufp.release(s); job.release(s); wpk.release(s); rec.release(s);
      ufq.release(s); qmark.release(s); qlist.release(s); qscr.release(s); qstate.release(s);
      bigmap.release(s); bigfr2.release(s); bigfg2.release(s); bigtouch.release(s);
      bigtouch_n.release(s); tflag.release(s); I16.release(s); ps_cells.release(s);
      eval_per.release(s); eval_limbs.release(s); band.release(s);
      labbounds.release(s);
      tmp.release(s); ssc.release(s); rsc.release(s);
      drop_chains(pending, s);
      drop_chains(chain_pool, s);
      cudaStreamSynchronize(s);
      for (auto &e : ev)
        if (e) cudaEventDestroy(e);
      for (auto &e : ev_acc)
        if (e) cudaEventDestroy(e);
      if (own_stream) cudaStreamDestroy(s);
    }
    pinned_put(pinned);
  }

  int32_t prepare() {  // K1 pass 1 + scan on the current raster
    RCB_TRY(contour_scan(L.p, lat, ocfg.full_fg, site_off.p, tmp, s));
    RCB_CUDA(cudaMemcpyAsync(&hsc->n_next, site_off.p + lat.V, sizeof(uint32_t),
                             cudaMemcpyDeviceToHost, s));
    RCB_CUDA(cudaStreamSynchronize(s));
    N = hsc->n_next;
    prepared = true;
    return RCB_OK;
  }

  std::vector<PendingChain> pending;     // PS: deferred total / total_sq chains
  std::vector<PendingChain> chain_pool;  // their buffers, recycled
  // integer-valued image with |sums| < 2^53: total / total_sq are exact in any
  // order, so instead of keeping per-iteration move lists (up to 12 GB at
  // cfg4) the statistics are rebuilt from the raster when read
  bool int_image = false;
  bool srec_current = false;  // srec matches L / Cown / Sown / rho0 (kept so by the integer band refresh)
  // z-slab sharded 3-D PS runs on integer images: the band refresh covers the
  // slab plus the halo the energy kernel reads, the ledger is summed over the
  // slab only and applied after the ranks' all-reduce (rcb_engine_band_apply)
  BandSlab band_slab{0, 0, 0, 0};
  bool fields_partial = false;  // own-label fields outside band_slab's planes are stale
  bool band_pending = false;    // band[] holds this rank's ledger share, not yet applied
  bool stats_stale = false;
  bool ps_tiles = false;  // K5 on shared-memory tiles (RCB_K5=tile; measured slower)

  int32_t flush_stats() {  // make tot / tsq current (replay deferred chains)
    if (stats_stale) {
      stats_stale = false;
      // cnt is current (k_count_moves); the rebuild recomputes it identically
      return stats_rebuild(L.p, I.p, lat.V, nl, cnt.p, tot.p, tsq.p, ssc, s);
    }
    if (pending.empty()) return RCB_OK;
    return replay_chains(pending, I.p, tot.p, tsq.p, s, &chain_pool);
  }

  int32_t refresh() {  // energy.py:285-291
    drop_chains(pending, s, &chain_pool);  // superseded by the rebuild
    stats_stale = false;
    RCB_TRY(stats_rebuild(L.p, I.p, lat.V, nl, cnt.p, tot.p, tsq.p, ssc, s));
    if (ecfg.region_model == 1)
      RCB_TRY(ps_fields(L.p, I.p, lat, ball_full.p, nball_full, Cown.p, Sown.p, s, rho0.p,
                        ecfg.noise_model == 1, I16.p));
    return RCB_OK;
  }

  int32_t components() {
    RCB_TRY(label_components(L.p, lat, ocfg.full_fg, nl, queue.p, ncomp.p, s));
    std::vector<int32_t> h(nl);
    RCB_CUDA(cudaMemcpyAsync(h.data(), ncomp.p, 4 * nl, cudaMemcpyDeviceToHost, s));
    RCB_CUDA(cudaStreamSynchronize(s));
    simple_topology = true;
    for (int32_t l = 1; l < nl; ++l)
      if (h[l] > 1) simple_topology = false;
    return RCB_OK;
  }
};

extern "C" {

int32_t rcb_version(void) { return 100; }
const char *rcb_last_error(void) { return g_err.c_str(); }
int32_t rcb_device_count(int32_t *n) {
  int c = 0;
  cudaError_t e = cudaGetDeviceCount(&c);
  *n = e == cudaSuccess ? c : 0;
  return RCB_OK;
}

namespace {
struct CtorLog {
  bool on;
  std::chrono::steady_clock::time_point t0;
  cudaStream_t s = nullptr;
  CtorLog() : on(getenv("RCB_CTOR_LOG") != nullptr), t0(std::chrono::steady_clock::now()) {}
  void mark(const char *what) {
    if (!on) return;
    if (s) cudaStreamSynchronize(s);
    const auto t = std::chrono::steady_clock::now();
    fprintf(stderr, "[rcb-ctor] %-12s %8.3f ms\n", what,
            std::chrono::duration<double, std::milli>(t - t0).count());
    t0 = t;
  }
};
}  // namespace

}  // extern "C"

namespace {
__global__ void k_promote_f32(const float *__restrict__ src, int64_t n, double *__restrict__ dst) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    dst[i] = (double)src[i];  // exact, = numpy's astype(float64) (optimizer.py:102)
}
}  // namespace

extern "C" {

int32_t rcb_engine_create(const double *image, const int32_t *labels, int32_t ndim,
                          const int64_t *dims, const rcb_energy_cfg *ecfg,
                          const rcb_sobolev_cfg *scfg, const rcb_opt_cfg *ocfg, int32_t device,
                          void *stream, rcb_engine **out) {
  return rcb_engine_create_ex(image, 0, labels, ndim, dims, ecfg, scfg, ocfg, device, stream,
                              out);
}

int32_t rcb_engine_create_ex(const void *image, int32_t image_dtype, const int32_t *labels,
                             int32_t ndim, const int64_t *dims, const rcb_energy_cfg *ecfg,
                             const rcb_sobolev_cfg *scfg, const rcb_opt_cfg *ocfg, int32_t device,
                             void *stream, rcb_engine **out) {
  *out = nullptr;
  if (image_dtype != 0 && image_dtype != 1)
    return fail(RCB_ERR_VALUE, "image_dtype must be 0 (float64) or 1 (float32)");
  CtorLog clog;
  RCB_TRY(check_device());
  RCB_TRY(check_lattice(ndim, dims));
  if (ecfg->region_model == 1 && (ecfg->smooth_radius < 1 || ecfg->smooth_radius > 15))
    return fail(RCB_ERR_VALUE, "smooth_radius must be in [1, 15]");
  if (!(scfg->length_scale > 0) || scfg->length_scale > 30.0)
    return fail(RCB_ERR_VALUE, "length_scale must be in (0, 30]");
  auto *e = new rcb_engine();
  e->device = device;
  RCB_CUDA(cudaSetDevice(device));
  {
    // keep freed stream-ordered allocations cached in the device pool: the
    // default release threshold (0) hands them back to the driver at every
    // synchronisation, and re-mapping them costs milliseconds per resync
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    // reserve the acceptance kernels' per-thread stack once: otherwise the
    // local-memory reservation is re-grown (milliseconds) whenever a launch
    // needs more than the previous one left in place
    size_t stack = 0;
    if (cudaDeviceGetLimit(&stack, cudaLimitStackSize) == cudaSuccess && stack < 2048)
      cudaDeviceSetLimit(cudaLimitStackSize, 2048);
  }
  if (stream) {
    e->s = (cudaStream_t)stream;
  } else {
    RCB_CUDA(cudaStreamCreateWithFlags(&e->s, cudaStreamNonBlocking));
    e->own_stream = true;
  }
  auto bail = [&](int32_t rc) {
    delete e;
    return rc;
  };
  cudaStream_t s = e->s;
  e->lat = make_lat(ndim, dims);
  clog.s = e->s;
  clog.mark("stream+pool");
  {
    // prime the device pool with the engine's footprint plus room for the
    // particle buffers to double a few times (~320 B per site + 256 MB, at
    // most max(16 GB, half the free memory)): later stream-ordered allocations are then served
    // from cached memory instead of blocking the host while memory is mapped
    size_t want = (size_t)320 * (size_t)e->lat.V + ((size_t)256 << 20);
    cudaMemPool_t pool;
    uint64_t reserved = 0, used = 0;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved);
      cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
    }
    // a pool that already caches that much free memory (engines destroyed
    // earlier in the process) serves the engine's buffers without priming;
    // one large priming block would not fit its free chunks and map anew
    if (clog.on)
      fprintf(stderr, "[rcb-ctor] pool reserved %.1f MB used %.1f MB want %.1f MB\n", reserved / 1e6,
              used / 1e6, want / 1e6);
    if (reserved < used + want) {
      size_t cap = (size_t)16 << 30;
      if (want > cap) {
        size_t free_b = 0, total_b = 0;
        if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess && free_b / 2 > cap) cap = free_b / 2;
      }
      if (want > cap) want = cap;
      // prime in 1 GB blocks: the pool reuses freed blocks of the requested
      // size class, and one huge priming block left later 10^8-byte requests
      // mapping fresh memory (up to ~0.8 s per allocation on the first cfg4
      // engine of a process, tools/alloc_probe.py)
      std::vector<void *> blocks;
      const size_t blk = (size_t)1 << 30;
      for (size_t got = 0; got < want; got += blk) {
        void *p = nullptr;
        if (cudaMallocAsync(&p, std::min(blk, want - got), s) != cudaSuccess) break;
        blocks.push_back(p);
      }
      for (void *p : blocks) cudaFreeAsync(p, s);
    }
    cudaGetLastError();
  }
  e->ecfg = *ecfg;
  e->ocfg = *ocfg;
  e->mode = ocfg->gradient;
  {
    const char *fs = getenv("RCB_FORCE_SEQUENTIAL");  // testing: exact single-thread acceptance
    e->force_sequential = fs && fs[0] == '1';
    const char *am = getenv("RCB_ACCEPT");  // "rounds": K8 v2 instead of the dataflow K8 v3
    e->accept_mode = (am && strcmp(am, "rounds") == 0) ? 1 : 0;
    const char *pf = getenv("RCB_PROFILE");
    e->profile = pf && pf[0] == '1';
  }
  const int64_t V = e->lat.V;
  int32_t rc;
#define TRYB(x)                 \
  if ((rc = (x)) != RCB_OK) {   \
    return bail(rc);            \
  }
  clog.mark("prime");
  TRYB(upload(e->L, labels, V, s));
  if (image_dtype == 1) {  // float32 input: 4 B/site over PCIe, promoted on the device
    TRYB(upload(e->I32, static_cast<const float *>(image), V, s));
    TRYB(e->I.reserve(V, s));
    k_promote_f32<<<std::min<unsigned>(grid_for(V, 256), 148u * 16u), 256, 0, s>>>(e->I32.p, V,
                                                                                   e->I.p);
    if (cudaGetLastError() != cudaSuccess) return bail(fail(RCB_ERR_CUDA, "k_promote_f32"));
    if (!ocfg->fp32) e->I32.release(s);
  } else {
    TRYB(upload(e->I, static_cast<const double *>(image), V, s));
  }
  {
    // input validation on the device (grid.py:24-39; optimizer.py:100-101):
    // label min / max (-> the label count), non-finite and negative
    // intensities, one reduction pass and one small read-back
    InputCheck chk{};
    TRYB(check_inputs(e->L.p, e->I.p, V, &chk, s));
    if (chk.nonfinite)
      return bail(fail(RCB_ERR_VALUE, "intensity raster contains non-finite values"));
    if (chk.label_min < 0) return bail(fail(RCB_ERR_VALUE, "label raster contains negative labels"));
    if (ecfg->noise_model == 1 && chk.image_min < 0.0)
      return bail(fail(RCB_ERR_VALUE, "Poisson noise model requires nonnegative intensities"));
    e->nl = chk.label_max + 1;
    // integer intensities <= 4096: V * 4096^2 < 2^53, so every partial sum of
    // total / total_sq is exact whatever the order
    e->int_image = chk.nonint == 0 && chk.image_max <= 4096.0 && chk.image_min >= -4096.0 &&
                   (double)V * 4096.0 * 4096.0 < 9.0e15 && !getenv("RCB_KEEP_CHAINS");
    {
      // the tiled K5 measured slower than the per-particle kernel at cfg4
      // (26 iterations: 3.83 s vs 2.43 s; ~110 particles per 8^3 tile leave
      // the 257-offset shared-memory walks latency bound at 2 blocks per SM):
      // kept as an experiment, RCB_K5=tile
      const char *k5 = getenv("RCB_K5");
      e->ps_tiles = k5 && strcmp(k5, "tile") == 0;
    }
    if (ecfg->region_model == 1 && ecfg->noise_model == 1 && chk.nonint == 0 &&
        chk.image_max <= 4096.0 && !getenv("RCB_NO_LOGTABLE")) {
      // integer Poisson data: every theta K5 forms is (S +- v) / (C +- 1)
      // with integer S <= |ball| * vmax; table its log (<= 64 MB)
      int nbf = 0;
      {
        const int r = ecfg->smooth_radius;
        for (int dz = (ndim == 3 ? -r : 0); dz <= (ndim == 3 ? r : 0); ++dz)
          for (int dy = -r; dy <= r; ++dy)
            for (int dx = -r; dx <= r; ++dx) nbf += dz * dz + dy * dy + dx * dx <= r * r;
      }
      const int64_t P = (int64_t)(nbf + 1) * (int64_t)chk.image_max + 1, Q = nbf + 2;
      if (P * Q * 8 <= ((int64_t)64 << 20)) {
        TRYB(e->logt.reserve(P * Q, s));
        TRYB(log_table(e->logt.p, (int)P, (int)Q, s));
        e->logt_P = (int)P;
      }
      // 3-D band refresh by prefix-sum ball runs (k_fields_band3d_int): exact
      // for integer intensities in [0, 2^12) with ball sums < 2^20
      if (ndim == 3 && chk.image_min >= 0.0 && ps_rec_ok(e->lat, nbf, chk.label_max + 2, chk.image_max) &&
          !getenv("RCB_NO_BANDINT")) {
        TRYB(e->I16.reserve(V, s));
        TRYB(image_u16(e->I.p, V, e->I16.p, s));
      }
      if (P * Q * 16 <= ((int64_t)128 << 20) &&
          ps_rec_ok(e->lat, nbf, chk.label_max + 1, chk.image_max) && !getenv("RCB_NO_K5REC")) {
        TRYB(e->thetat.reserve(P * Q, s));
        TRYB(theta_table(e->thetat.p, (int)P, (int)Q, s));
        e->thetat_P = (int)P;
      }
    }
  }
  TRYB(e->cnt.reserve(e->nl, s));
  TRYB(e->tot.reserve(e->nl, s));
  TRYB(e->tsq.reserve(e->nl, s));
  TRYB(e->ncomp.reserve(e->nl, s));
  TRYB(e->vis.reserve(V, s));
  TRYB(e->queue.reserve(V, s));
  TRYB(e->site_off.reserve(V + 1, s));
  TRYB(e->sc.reserve(1, s));
  clog.mark("upload");
  static_assert(sizeof(Scalars) <= 2048, "pinned block layout: Scalars | hoff @2048 | hwatch @3072");
  e->pinned = pinned_get();
  if (!e->pinned) return bail(fail(RCB_ERR_CUDA, "cudaMallocHost failed"));
  e->hsc = reinterpret_cast<Scalars *>(e->pinned);
  e->hoff = reinterpret_cast<uint32_t *>(reinterpret_cast<char *>(e->pinned) + 2048);
  e->hwatch = reinterpret_cast<unsigned long long *>(reinterpret_cast<char *>(e->pinned) + 3072);
  e->hctl = reinterpret_cast<int32_t *>(reinterpret_cast<char *>(e->pinned) + 3584);
  memset(e->hctl, 0, 16 * sizeof(int32_t));
  memset(e->hsc, 0, sizeof(Scalars));

  memset(e->hwatch, 0, 8 * sizeof(unsigned long long));
  if (cudaMemsetAsync(e->sc.p, 0, sizeof(Scalars), s) != cudaSuccess ||
      cudaMemsetAsync(e->vis.p, 0, sizeof(uint32_t) * V, s) != cudaSuccess)
    return bail(fail(RCB_ERR_CUDA, "memset failed"));
  e->hsc->epoch = 32;
  cudaMemcpyAsync(&e->sc.p->epoch, &e->hsc->epoch, sizeof(uint32_t), cudaMemcpyHostToDevice, s);
  if (ecfg->region_model == 1) {
    auto full = ball_table(ndim, ecfg->smooth_radius);
    e->nball_full = (int)full.size();
    e->nball = e->nball_full - 1;
    TRYB(upload(e->ball_full, full.data(), full.size(), s));
    TRYB(upload(e->ball, full.data() + 1, full.size() - 1, s));
    TRYB(e->Cown.reserve(V, s));
    TRYB(e->Sown.reserve(V, s));
    TRYB(e->rho0.reserve(V, s));
  }
  int maxd2 = 0;
  auto st = sobolev_rows(ndim, scfg->length_scale, &maxd2);
  if (scfg->n_weights <= maxd2)
    return bail(fail(RCB_ERR_VALUE, "Sobolev weight table shorter than the stencil needs"));
  e->nst = (int)st.size();
  for (const Off &o : st) {  // outer-axis reach of the stencil (dz in 3-D, dy in 2-D)
    const int64_t r = std::abs(ndim == 3 ? (int)o.dz : (int)o.dy);
    e->stencil_reach = std::max(e->stencil_reach, r);
  }
  TRYB(upload(e->st, st.data(), st.size(), s));
  TRYB(upload(e->wt, scfg->weights, (size_t)scfg->n_weights, s));
  e->nwt = scfg->n_weights;
  {
    const char *ks = getenv("RCB_K6");  // "scalar": the unpacked K6 (comparison runs)
    e->sob_packed = sobolev_packable(e->nl, e->nst, maxd2) && !(ks && strcmp(ks, "scalar") == 0);
    e->sob_site = sobolev_site_only(st.data(), e->nst) && !(ks && strcmp(ks, "scalar") == 0);
    e->w0 = scfg->weights[0];
  }
  if (ocfg->fp32) {
    TRYB(e->I32.reserve(V, s));
    TRYB(e->wt32.reserve(scfg->n_weights, s));
    TRYB(to_float(e->I.p, V, e->I32.p, s));
    TRYB(to_float(e->wt.p, scfg->n_weights, e->wt32.p, s));
  }
  TRYB(e->newlab.reserve(V, s));
  TRYB(e->wpos.reserve(V, s));
  TRYB(e->pend.reserve(V, s));
  TRYB(e->gq1.reserve(V, s));
  TRYB(e->lab_pend.reserve(e->nl, s));
  TRYB(e->nown.reserve(e->nl, s));
  TRYB(e->small.reserve(e->nl, s));
  TRYB(e->cnt0.reserve(e->nl, s));
  TRYB(e->ctl.reserve(16, s));
  TRYB(e->lab_ptr.reserve(e->nl, s));
  TRYB(e->lbox.reserve(6 * e->nl, s));
  if (cudaMemsetAsync(e->wpos.p, 0x7f, sizeof(int32_t) * V, s) != cudaSuccess ||
      cudaMemsetAsync(e->pend.p, 0x7f, sizeof(int32_t) * V, s) != cudaSuccess ||
      cudaMemsetAsync(e->ctl.p, 0, sizeof(int32_t) * 16, s) != cudaSuccess)
    return bail(fail(RCB_ERR_CUDA, "memset failed"));
  if (ecfg->region_model == 1) {
    TRYB(e->dirty.reserve(V, s));
    if (cudaMemsetAsync(e->dirty.p, 0, V, s) != cudaSuccess)
      return bail(fail(RCB_ERR_CUDA, "memset failed"));
  }
  for (auto &ev : e->ev) cudaEventCreate(&ev);
  for (auto &ev : e->ev_acc) cudaEventCreate(&ev);
  clog.mark("buffers");
  TRYB(e->refresh());
  clog.mark("refresh");
  TRYB(e->components());
  clog.mark("components");
  TRYB(e->prepare());
  clog.mark("prepare");
#undef TRYB
  *out = e;
  return RCB_OK;
}

void rcb_engine_destroy(rcb_engine *e) { delete e; }

// Particle range [p(lo), p(hi)) of the sites in outer planes [lo, hi) (z in
// 3-D, rows in 2-D): particles are sorted by site, so a slab of planes is one
// contiguous range of the particle list (read from the K1 index site_off).
static int32_t plane_ranges(rcb_engine *e, const int64_t *planes, int k, int64_t *out) {
  const int64_t plane = e->lat.ndim == 3 ? e->lat.ny * e->lat.nx : e->lat.nx;
  const int64_t np = e->lat.ndim == 3 ? e->lat.nz : e->lat.ny;
  for (int i = 0; i < k; ++i) {
    const int64_t pl = std::min(std::max(planes[i], (int64_t)0), np);
    RCB_CUDA(cudaMemcpyAsync(&e->hoff[i], e->site_off.p + pl * plane, sizeof(uint32_t),
                             cudaMemcpyDeviceToHost, e->s));
  }
  RCB_CUDA(cudaStreamSynchronize(e->s));
  for (int i = 0; i < k; ++i) out[i] = e->hoff[i];
  return RCB_OK;
}

// Scoring half of iterate(): K1 emit, ΔE_int, ΔE (K3/K5) and the Sobolev
// filter (K6).  With a slab [slab_lo, slab_hi) set, ΔE is computed for the
// slab's particles plus a halo of the stencil's reach (the particles K6 reads)
// and K6 for the slab's particles only; every other array stays replicated.
static std::chrono::steady_clock::time_point g_host_t0;
static int32_t engine_score(rcb_engine *e) {
  g_host_t0 = std::chrono::steady_clock::now();
  RCB_CUDA(cudaSetDevice(e->device));
  cudaStream_t s = e->s;
  e->iteration += 1;
  e->launches = 0;
  e->fields_fresh = false;
  if (e->band_pending) return fail(RCB_ERR_VALUE, "rcb_engine_band_apply not called after finish");
  if (e->fields_partial) {
    const int64_t halo = e->stencil_reach + e->ecfg.smooth_radius;
    const bool same = e->mode == 1 && e->slab_hi > e->slab_lo &&
                      e->band_slab.own0 == e->slab_lo && e->band_slab.own1 == e->slab_hi &&
                      e->band_slab.z0 == e->slab_lo - halo;
    if (!same) {  // l2 mode reads fields anywhere; another slab needs other planes
      RCB_TRY(e->refresh());
      e->fields_partial = false;
      e->srec_current = false;
    }
  }
  cudaEventRecord(e->ev[0], s);
  if (!e->prepared) RCB_TRY(e->prepare());
  const int64_t n = e->N;
  const Lat &lat = e->lat;
  Scalars *d = e->sc.p;
  RCB_CUDA(cudaMemsetAsync(&d->pairs, 0, sizeof(unsigned long long), s));
  RCB_CUDA(cudaMemsetAsync(&d->moves, 0, sizeof(int64_t), s));
  int launches = 2;
  // particle ranges: [p0, p1) own slab, [h0, h1) slab + stencil halo
  int64_t p0 = 0, p1 = n, h0 = 0, h1 = n;
  if (e->slab_hi > e->slab_lo && n > 0) {
    const int64_t reach = e->mode == 1 ? e->stencil_reach : 0;
    const int64_t pl[4] = {e->slab_lo, e->slab_hi, e->slab_lo - reach, e->slab_hi + reach};
    int64_t r[4];
    RCB_TRY(plane_ranges(e, pl, 4, r));
    p0 = r[0];
    p1 = r[1];
    h0 = r[2];
    h1 = r[3];
  }
  e->p0 = p0;
  e->p1 = p1;
  if (n > 0) {
    RCB_TRY(e->px.reserve(n, s));
    RCB_TRY(e->pown.reserve(n, s));
    RCB_TRY(e->pcomp.reserve(n, s));
    RCB_TRY(e->dint.reserve(n, s));
    RCB_TRY(e->raw.reserve(n, s));
    RCB_TRY(e->smooth.reserve(n, s));
    RCB_TRY(e->rank.reserve(n, s));
    RCB_TRY(e->order.reserve(n, s));
    RCB_TRY(e->acc.reserve(3 * n, s));
    RCB_TRY(contour_emit(e->L.p, lat, e->ocfg.full_fg, e->site_off.p, e->px.p, e->pown.p,
                         e->pcomp.p, s));
    cudaEventRecord(e->ev[1], s);
    // lam = 0 (every BASELINE config): rank = base + 0 * dint = base whatever
    // the (finite, integer) dint holds, so the pass is skipped
    if (e->ecfg.lam != 0.0)
      RCB_TRY(delta_int_batch(e->L.p, lat, e->px.p, e->pown.p, e->pcomp.p, n, e->dint.p, s));
    const int poisson = e->ecfg.noise_model == 1;
    const bool fp32 = e->ocfg.fp32 != 0;
    if (fp32) RCB_TRY(e->raw32.reserve(n, s));
    if (e->ecfg.region_model == 1) {
      RCB_TRY(e->cb0.reserve(n, s));
      RCB_TRY(e->sb0.reserve(n, s));
    }
    const int64_t m = h1 - h0;
    // K6's packed partner records come straight from the energy kernel (no
    // packing pass) when K6 reads them: Sobolev mode, labels < 2^16
    const bool ps_tiles_now = e->ecfg.region_model == 1 && e->int_image && e->ps_tiles &&
                              e->rho0.p && ps3d_tile_ok(lat, e->ecfg.smooth_radius, e->nball);
    const bool pk_direct = e->mode == 1 && !fp32 && e->sob_packed && (e->sob_site || e->nst > 1) &&
                           (e->ecfg.region_model == 0 ||
                            (!ps_tiles_now && delta_ps_writes_pk(lat, e->nball)));
    if (pk_direct) RCB_TRY(e->pk.reserve(n, s));
    int4 *pkh = pk_direct ? e->pk.p + h0 : nullptr;
    if (fp32 && e->ecfg.region_model == 0)
      RCB_TRY(delta_pc32_batch(e->I32.p, e->px.p + h0, e->pown.p + h0, e->pcomp.p + h0, m,
                               e->cnt.p, e->tot.p, poisson, e->raw32.p + h0, e->raw.p + h0, s));
    else if (fp32 && !(e->thetat_P && e->rho0.p && e->ecfg.noise_model == 1))
      RCB_TRY(delta_ps32_batch(e->L.p, e->I32.p, e->Cown.p, e->Sown.p, lat, e->ball.p, e->nball,
                               e->px.p + h0, e->pown.p + h0, e->pcomp.p + h0, m, poisson,
                               e->raw32.p + h0, e->raw.p + h0, s, e->cb0.p + h0, e->sb0.p + h0));
    else if (e->ecfg.region_model == 0)
      RCB_TRY(delta_pc_batch(e->I.p, e->px.p + h0, e->pown.p + h0, e->pcomp.p + h0, m, e->cnt.p,
                             e->tot.p, e->tsq.p, poisson, e->raw.p + h0, s, pkh));
    else if (ps_tiles_now)
      // integer images: the ball gathers from shared-memory tiles (RCB_K5=tile)
      RCB_TRY(delta_ps3d_tiles(e->L.p, e->I.p, e->Cown.p, e->Sown.p, e->rho0.p, lat,
                               e->ecfg.smooth_radius, e->ball.p, e->nball, e->site_off.p, e->px.p,
                               e->pown.p, e->pcomp.p, h0, h1, poisson, e->raw.p, e->cb0.p,
                               e->sb0.p, e->logt_P ? e->logt.p : nullptr, e->logt_P, s));
    else if (e->thetat_P && e->rho0.p && e->ecfg.noise_model == 1) {
      // integer Poisson data: one 16-byte record per ball site (k_delta_ps_rec)
      const int4 *const srec_old = e->srec.p;
      RCB_TRY(e->srec.reserve(lat.V, s));
      if (!e->srec_current || e->srec.p != srec_old || getenv("RCB_PACK_ALWAYS"))
        RCB_TRY(pack_sites(e->L.p, e->Cown.p, e->Sown.p, e->I.p, e->rho0.p, lat.V, e->srec.p, s));
      e->srec_current = false;  // until this iteration's band refresh says otherwise
      RCB_TRY(delta_ps_rec(e->srec.p, e->I.p, lat, e->ball.p, e->nball, e->px.p + h0,
                           e->pown.p + h0, e->pcomp.p + h0, m, e->raw.p + h0, e->rho0.p,
                           e->cb0.p + h0, e->sb0.p + h0, e->thetat.p, e->thetat_P, pkh, s));
      // fp32 mode on integer Poisson data: the table-driven fp64 kernel is
      // faster than the fp32 five-array gather; its increments are rounded
      // to fp32 for the fp32 Sobolev filter
      if (fp32) RCB_TRY(to_float(e->raw.p + h0, m, e->raw32.p + h0, s));
      launches += 1;
    } else
      RCB_TRY(delta_ps_batch(e->L.p, e->I.p, e->Cown.p, e->Sown.p, lat, e->ball.p, e->nball,
                             e->px.p + h0, e->pown.p + h0, e->pcomp.p + h0, m, poisson,
                             e->raw.p + h0, s, e->rho0.p, e->cb0.p + h0, e->sb0.p + h0,
                             e->logt_P ? e->logt.p : nullptr, e->logt_P, pkh));
    cudaEventRecord(e->ev[2], s);
    if (e->mode == 1) {
      if (fp32) {
        RCB_TRY(sobolev_lattice32(e->site_off.p, e->pown.p, e->px.p, e->pcomp.p, e->raw32.p, lat,
                                  e->st.p, e->nst, e->wt32.p, p1, e->smooth.p, &d->pairs, s, p0));
      } else if (e->sob_site && pk_direct) {
        // register-staged vector loads (measured faster than the TMA ring of
        // sobolev_site_bulk at every size, profiles/README.md)
        RCB_TRY(sobolev_site_pk(e->pk.p, e->w0, p0, p1, h0, h1, e->smooth.p, &d->pairs, s));
      } else if (e->sob_site) {
        RCB_TRY(sobolev_site(e->px.p, e->pown.p, e->pcomp.p, e->raw.p, e->w0, p0, p1, h0, h1,
                             e->smooth.p, &d->pairs, s));
      } else if (e->sob_packed && e->nst > 1) {
        // packed records of the partners K6 reads ([h0, h1) covers the halo)
        if (!pk_direct) {
          RCB_TRY(e->pk.reserve(n, s));
          RCB_TRY(sobolev_pack(e->px.p, e->pown.p, e->pcomp.p, e->raw.p, h0, h1, e->pk.p, s));
          launches += 1;
        }
        RCB_TRY(sobolev_packed(e->site_off.p, e->pk.p, lat, e->st.p, e->nst, e->wt.p, e->nwt, p0,
                               p1, e->smooth.p, &d->pairs, s));
      } else {
        RCB_TRY(sobolev_lattice(e->site_off.p, e->pown.p, e->px.p, e->pcomp.p, e->raw.p, lat,
                                e->st.p, e->nst, e->wt.p, p1, e->smooth.p, &d->pairs, s, p0));
      }
      launches += 1;
    }
    cudaEventRecord(e->ev[3], s);
  } else {
    for (int k = 1; k < 4; ++k) cudaEventRecord(e->ev[k], s);
  }
  e->score_launches = launches;
  e->scored = true;
  return RCB_OK;
}

// Decision half of iterate(): rank order (K7), acceptance (K8) and its
// bookkeeping, K1 pass 1 of the next raster, the iteration record.
static int32_t engine_finish(rcb_engine *e, rcb_iter_record *rec) {
  if (!e->scored) return fail(RCB_ERR_VALUE, "rcb_engine_finish without rcb_engine_score");
  e->scored = false;
  RCB_CUDA(cudaSetDevice(e->device));
  cudaStream_t s = e->s;
  const int64_t n = e->N;
  const Lat &lat = e->lat;
  Scalars *d = e->sc.p;
  int launches = e->score_launches;
  const int poisson = e->ecfg.noise_model == 1;
  if (n > 0) {
    const double *base = e->mode == 1 ? e->smooth.p : e->raw.p;
    RCB_TRY(rank_order(base, e->dint.p, e->ecfg.lam, n, e->px.p, e->pcomp.p, e->ocfg.seed,
                       e->rank.p, e->rsc, e->order.p, &d->nneg, s));
    cudaEventRecord(e->ev[4], s);
    // dataflow kernel (K8 v3): packed BFS coordinates need sides < 2^16 in
    // 2-D and < 2^11 (x, y), < 2^10 (z) in 3-D; site words hold 24-bit
    // positions and 16-bit labels
    const bool fits = lat.ndim == 2 ? (lat.nx < 65536 && lat.ny < 65536)
                                    : (lat.nx < 2048 && lat.ny < 2048 && lat.nz < 1024);
    // site words: 24-bit positions with 16-bit labels, or 27-bit positions with
    // 10-bit labels (more than 2^24 - 1 candidates, at most 1024 labels)
    const bool df24 = n < 0xffffff && e->nl <= 65536;
    const bool df27 = n < 0x7ffffff && e->nl <= 1024;
    const bool use_df = fits && e->accept_mode != 1 && (df24 || df27);
    // l2 mode runs in parallel through the dataflow kernel: every label
    // sequenced, the d_tot < 0 gate on running statistics (PC) or on the
    // own-label fields corrected by the earlier flips within 2R (PS, fp64
    // Poisson or Gauss with the rho0 table and the K5 competitor terms)
    const char *psl2 = getenv("RCB_PS_L2");  // "seq": PS l2 on K8 v1 (comparison runs)
    const bool ps_l2_ok = e->ecfg.region_model == 1 && e->rho0.p && e->cb0.p && !e->ocfg.fp32 &&
                          !(psl2 && strcmp(psl2, "seq") == 0) &&
                          e->ecfg.smooth_radius <= 7;
    const bool l2par = e->mode == 0 && (e->ecfg.region_model == 0 || ps_l2_ok) && use_df;
    const bool par = (e->mode == 1 || l2par) && e->ocfg.full_fg && e->simple_topology &&
                     !e->force_sequential;
    e->cur_par = par;
    const int64_t budget = (int64_t)ceil(e->ocfg.move_budget * (double)n);
    if (par) {
      RCB_TRY(e->dec.reserve(n, s));
      RCB_TRY(e->dround.reserve(n, s));
      RCB_TRY(e->bfs_list.reserve(n, s));
      RCB_TRY(e->slot.reserve(n + 1, s));
      RCB_TRY(e->dint_acc.reserve(n, s));
      RCB_TRY(e->blocker.reserve(n, s));
      RCB_TRY(e->pos_of.reserve(n, s));
      RCB_TRY(e->dtot.reserve(n, s));
      ParArgs P{};
      P.lat = lat;
      P.allow_fusion = e->ocfg.allow_fusion;
      P.vanish_ok = e->ocfg.allow_vanish && e->iteration > e->ocfg.vanish_grace;
      P.nl = e->nl;
      P.nneg = &d->nneg;
      P.order = e->order.p;
      P.px = e->px.p;
      P.pown = e->pown.p;
      P.pcomp = e->pcomp.p;
      P.L = e->L.p;
      P.newlab = e->newlab.p;
      P.w = e->wpos.p;
      P.pend = e->pend.p;
      P.dec = e->dec.p;
      P.dround = e->dround.p;
      P.small = e->small.p;
      P.lab_pend = e->lab_pend.p;
      P.nown = e->nown.p;
      P.cnt = e->cnt.p;
      P.cnt0 = e->cnt0.p;
      P.bfs_list = e->bfs_list.p;
      P.ctl = e->ctl.p;
      P.vis = e->vis.p;
      P.epoch = &d->epoch;
      P.gq[0] = e->queue.p;
      P.gq[1] = e->gq1.p;
      P.dint_acc = e->dint_acc.p;
      P.blocker = e->blocker.p;
      P.pos_of = e->pos_of.p;
      P.site_off = e->site_off.p;
      P.lab_ptr = e->lab_ptr.p;
      P.lbox = e->lbox.p;
      {
        const char *wr = getenv("RCB_DF_WINDOW");
        P.win_r = wr ? atoi(wr) : 0;
        const char *w5 = getenv("RCB_DF_WIN5");  // comparison runs
        P.win5 = !(w5 && w5[0] == '0');
        const char *wf = getenv("RCB_DF_WPFIRST");  // comparison runs
        P.wp_first = !(wf && wf[0] == '0');
        const char *nw = getenv("RCB_DF_NOWAIT");  // timing experiment: wrong results
        P.nowait = nw ? atoi(nw) : 0;  // bit 0: no dependency waits; bit 1: an extra raster read per box cell
        const char *in = getenv("RCB_DF_IDLE_NS");
        P.idle_ns = in ? atoi(in) : 2000;
        const char *lm = getenv("RCB_DF_LOWMARK_NS");
        P.lowmark_ns = lm ? atoi(lm) : 1024;
        const char *ha = getenv("RCB_DF_HELPAFTER");
        P.help_after = ha ? atoi(ha) : 0;
        const char *mi = getenv("RCB_DF_MAXINSERT");  // tests: force assist jobs
        P.max_insert = mi ? atoi(mi) : 0;
        const char *bc = getenv("RCB_DF_BOXCAP");  // tests: 0 sends overflows to assist jobs
        P.box_cap = bc ? atoi(bc) : -1;
        const char *qj = getenv("RCB_DF_QJOB");  // "0": a full union-find per deferred candidate
        P.qjob = !(qj && qj[0] == '0');
        const char *qp = getenv("RCB_DF_PREREG");
        P.qprereg = !(qp && qp[0] == '0');
        const char *ws = getenv("RCB_DF_WATCH_S");  // watchdog seconds (default 60)
        P.watch_ns = (unsigned long long)((ws ? atof(ws) : 60.0) * 1e9);
      }
      if (e->profile) {
        RCB_TRY(e->tdbg.reserve(4 * n, s));
        P.tdbg = e->tdbg.p;
      }
      P.l2 = e->mode == 0;
      {
        const char *w27 = getenv("RCB_DF_WP27");  // tests: the wide layout on small inputs
        P.wp_bits = (df24 && !(w27 && w27[0] == '1' && df27)) ? 24 : 27;
      }
      P.poisson = poisson;
      P.lam = e->ecfg.lam;
      P.I = e->I.p;
      P.region_ps = e->ecfg.region_model == 1;

      if (P.region_ps) {
        P.Cown = e->Cown.p;
        P.Sown = e->Sown.p;
        P.rho0 = e->rho0.p;
        P.cb0 = e->cb0.p;
        P.sb0 = e->sb0.p;
        P.ball = e->ball.p;
        P.nball = e->nball;
        P.radius = e->ecfg.smooth_radius;
        const char *fc = getenv("RCB_PS_L2_FLIPCAP");  // tests: 0 = always recount
        P.ps_flipcap = fc ? atoi(fc) : 1 << 30;
        if (P.l2 && !e->ps_cells.p) {  // the 2R ball as cube indices (side 4R + 1)
          const int R = e->ecfg.smooth_radius, side = 4 * R + 1;
          std::vector<int32_t> cells;
          for (int dz = (lat.ndim == 3 ? -2 * R : 0); dz <= (lat.ndim == 3 ? 2 * R : 0); ++dz)
            for (int dy = -2 * R; dy <= 2 * R; ++dy)
              for (int dx = -2 * R; dx <= 2 * R; ++dx)
                if (dz * dz + dy * dy + dx * dx <= 4 * R * R)
                  cells.push_back(((lat.ndim == 3 ? dz + 2 * R : 0) * side + dy + 2 * R) * side +
                                  dx + 2 * R);
          RCB_TRY(upload(e->ps_cells, cells.data(), cells.size(), s));
          e->ps_ncells = (int)cells.size();
        }
        P.ps_cells = e->ps_cells.p;
        P.ps_ncells = e->ps_ncells;
      }
      if (P.l2 && !P.region_ps) {
        RCB_TRY(e->tot_run.reserve(e->nl, s));
        RCB_TRY(e->tsq_run.reserve(e->nl, s));
        RCB_CUDA(cudaMemcpyAsync(e->tot_run.p, e->tot.p, sizeof(double) * e->nl,
                                 cudaMemcpyDeviceToDevice, s));
        RCB_CUDA(cudaMemcpyAsync(e->tsq_run.p, e->tsq.p, sizeof(double) * e->nl,
                                 cudaMemcpyDeviceToDevice, s));
        P.tot_run = e->tot_run.p;
        P.tsq_run = e->tsq_run.p;
      }
      if (use_df) {
        if (!e->ufp.p) {
          RCB_TRY(e->ufq.reserve(lat.V, s));
          RCB_TRY(e->qstate.reserve(3 * (size_t)e->nl, s));
          RCB_CUDA(cudaMemsetAsync(e->qstate.p, 0, sizeof(unsigned long long) * 3 * e->nl, s));
          RCB_TRY(e->qmark.reserve(lat.V, s));
          RCB_CUDA(cudaMemsetAsync(e->ufq.p, 0xff, sizeof(unsigned long long) * lat.V, s));
          RCB_CUDA(cudaMemsetAsync(e->qmark.p, 0xff, sizeof(unsigned long long) * lat.V, s));
          RCB_TRY(e->ufp.reserve(lat.V, s));
          RCB_TRY(e->wpk.reserve(lat.V, s));
          RCB_CUDA(cudaMemsetAsync(e->wpk.p, 0xff, sizeof(unsigned long long) * lat.V, s));
          RCB_TRY(e->job.reserve(64, s));
          RCB_CUDA(cudaMemsetAsync(e->ufp.p, 0xff, sizeof(unsigned long long) * lat.V, s));
          RCB_CUDA(cudaMemsetAsync(e->job.p, 0, sizeof(unsigned long long) * 64, s));
        }
        // registry of deferred candidates (cleared after each run by k_q_reset)
        RCB_TRY(e->qlist.reserve(2 * n, s));  // up-front registrations + the deferring warps' own
        RCB_TRY(e->qscr.reserve(n, s));
        P.ufq = e->ufq.p;
        P.qmark = e->qmark.p;
        P.qlist = e->qlist.p;
        P.qscr = e->qscr.p;
        P.qstate = e->qstate.p;
        P.ufp = e->ufp.p;
        P.job = e->job.p;
        P.wp = e->wpk.p;
      }
      if (!use_df) {
        // slots for the round-based kernel's large-footprint BFS (<= 160 blocks)
        const size_t nb = 160;
        if (!e->bigkey.p) {
          RCB_TRY(e->bigkey.reserve(nb * (1u << 19), s));
          RCB_TRY(e->bigfr.reserve(nb * 2 * (1u << 17), s));
          RCB_TRY(e->bigfg.reserve(nb * 2 * (1u << 17), s));
          RCB_TRY(e->bigtag.reserve(nb, s));
          RCB_CUDA(cudaMemsetAsync(e->bigkey.p, 0, sizeof(unsigned long long) * nb * (1u << 19), s));
          RCB_CUDA(cudaMemsetAsync(e->bigtag.p, 0, sizeof(uint32_t) * nb, s));
        }
        P.bigkey = e->bigkey.p;
        P.bigfr = e->bigfr.p;
        P.bigfg = e->bigfg.p;
        P.bigtag = e->bigtag.p;
      }
      ParExtra X{};
      X.n_particles = n;
      X.hcount = e->hwatch + 7;  // spare word of the engine's pinned block
      X.budget = budget;
      X.slot = e->slot.p;
      X.tmp = &e->tmp;
      X.acc = e->acc.p;
      X.moves = &d->moves;
      X.I = e->I.p;
      X.tot = e->tot.p;
      X.tsq = e->tsq.p;
      X.energy = &d->energy;
      X.dtot = e->dtot.p;
      X.ncomp = e->ncomp.p;
      X.Lmut = e->L.p;
      X.region_ps = e->ecfg.region_model == 1;
      X.poisson = poisson;
      X.lam = e->ecfg.lam;
      X.ball = e->ball.p;
      X.ball_full = e->ball_full.p;
      X.nball = e->nball;
      X.nball_full = e->nball_full;
      X.radius = e->ecfg.smooth_radius;
      X.dirty = e->dirty.p;
      X.Cown = e->Cown.p;
      X.Sown = e->Sown.p;
      X.rho0 = e->rho0.p;
      X.cb0 = e->cb0.p;
      X.sb0 = e->sb0.p;
      X.evkey = &e->evkey;
      X.evkey2 = &e->evkey2;
      X.evval = &e->evval;
      X.evval2 = &e->evval2;
      X.bounds = &e->evbounds;
      X.snap = &e->snap;
      X.evv = &e->evv;
      // 3-D: footprints of inconclusive topology tests often exceed a warp's
      // hash; the round-based kernel's block BFS handles them
      X.accept_mode = use_df ? 0 : 1;
      X.labkey = &e->labkey;
      X.labkey2 = &e->labkey2;
      X.labpos = &e->labpos;
      X.labpos2 = &e->labpos2;
      X.flrows = &e->flrows;
      X.fmap = &e->fmap;
      X.rec = &e->rec;
      RCB_TRY(e->band.reserve(kLimbs + 2, s));
      X.band = e->band.p;
      X.colb = &e->colb;
      X.labbounds = &e->labbounds;
      X.tflag = &e->tflag;
      X.I16 = e->I16.p;
      X.srec = e->srec.p;  // null unless K5 reads packed site records
      X.srec_current = &e->srec_current;
      if (e->slab_hi > e->slab_lo && lat.ndim == 3 && e->ecfg.region_model == 1 && e->mode == 1 &&
          e->I16.p && e->rho0.p && !getenv("RCB_SLAB_BAND_OFF")) {
        const int64_t halo = e->stencil_reach + e->ecfg.smooth_radius;
        e->band_slab = BandSlab{e->slab_lo - halo, e->slab_hi + halo, e->slab_lo, e->slab_hi};
        X.band_slab = &e->band_slab;
        e->fields_partial = true;
        e->band_pending = true;
      }
      X.chain_pool = &e->chain_pool;
      {
        const char *ds = getenv("RCB_DEFER_STATS");  // "0": eager sum chains (comparison runs)
        X.pending = (ds && ds[0] == '0') ? nullptr : &e->pending;
        if (X.pending && e->int_image && e->ecfg.region_model == 1) X.stats_stale = &e->stats_stale;
      }
      {
        const char *bt = getenv("RCB_DF_BIGBOX");  // "0": no large box tier (comparison runs)
        if (!(bt && bt[0] == '0')) {
          X.bigmap = &e->bigmap;
          X.bigfr2 = &e->bigfr2;
          X.bigfg2 = &e->bigfg2;
          X.bigtouch = &e->bigtouch;
          X.bigtouch_n = &e->bigtouch_n;
        }
      }
      int nla = 0;
      RCB_CUDA(cudaMemsetAsync(e->ctl.p, 0, sizeof(int32_t) * 16, s));
      cudaEventRecord(e->ev_acc[0], s);
      if (use_df) RCB_CUDA(cudaMemsetAsync(e->job.p + 56, 0, 8 * sizeof(unsigned long long), s));
      RCB_TRY(accept_par(P, X, s, &nla));
      if (use_df)
        RCB_CUDA(cudaMemcpyAsync(e->hwatch, e->job.p + 56, 6 * sizeof(unsigned long long),
                                 cudaMemcpyDeviceToHost, s));
      cudaEventRecord(e->ev_acc[1], s);
      RCB_CUDA(cudaMemcpyAsync(e->hctl, e->ctl.p, sizeof(int32_t) * 16, cudaMemcpyDeviceToHost, s));
      launches += nla;
    } else {
      AcceptArgs A{};
      A.lat = lat;
      A.full_fg = e->ocfg.full_fg;
      A.region_ps = e->ecfg.region_model == 1;
      A.poisson = poisson;
      A.mode_l2 = e->mode == 0;
      A.allow_fusion = e->ocfg.allow_fusion;
      A.vanish_ok = e->ocfg.allow_vanish && e->iteration > e->ocfg.vanish_grace;
      A.lam = e->ecfg.lam;
      A.budget = budget;
      A.n = n;
      A.order = e->order.p;
      A.rank = e->rank.p;
      A.px = e->px.p;
      A.pown = e->pown.p;
      A.pcomp = e->pcomp.p;
      A.L = e->L.p;
      A.I = e->I.p;
      A.cnt = e->cnt.p;
      A.tot = e->tot.p;
      A.tsq = e->tsq.p;
      A.Cown = e->Cown.p;
      A.Sown = e->Sown.p;
      A.rho0 = e->rho0.p;
      A.ball = e->ball.p;
      A.nball = e->nball;
      A.ncomp = e->ncomp.p;
      A.vis = e->vis.p;
      A.queue = e->queue.p;
      A.epoch = &d->epoch;
      A.acc = e->acc.p;
      A.moves = &d->moves;
      A.energy = &d->energy;
      RCB_TRY(e->flush_stats());  // the sequential kernel reads and updates the sums
      RCB_TRY(accept_seq(A, s));
  launches += 1;
    }
    // K1 emit, the energy kernel, k_rank, the 32-bit key sort (histogram,
    // exclusive sum, four onesweep passes), k_tie_runs; + dE_int when lam != 0.
    // (ncu launch lists: 35 launches per cfg4 iteration, 41 per cfg2 iteration;
    // this count gives 39 and 38)
    launches += 10 + (e->ecfg.lam != 0.0 ? 1 : 0);
  } else {
    cudaEventRecord(e->ev[4], s);
  }
  // K1 pass 1 on the updated raster: the particle count of the record and the
  // lattice index map of the next iteration
  RCB_TRY(contour_scan(e->L.p, lat, e->ocfg.full_fg, e->site_off.p, e->tmp, s));
  RCB_CUDA(cudaMemcpyAsync(&d->n_next, e->site_off.p + lat.V, sizeof(uint32_t),
                           cudaMemcpyDeviceToDevice, s));
  cudaEventRecord(e->ev[5], s);
  RCB_CUDA(cudaMemcpyAsync(e->hsc, d, offsetof(Scalars, limbs), cudaMemcpyDeviceToHost, s));
  if (getenv("RCB_HOST_LOG")) {  // host time to enqueue the iteration (vs its device time)
    const double hu = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() -
                                                                 g_host_t0).count();
    fprintf(stderr, "[rcb-host] enqueue %.1f us\n", hu);
  }
  RCB_CUDA(cudaStreamSynchronize(s));
  if (e->hwatch[0]) {  // the dataflow acceptance's watchdog fired (accept_par.cu)
    const unsigned long long w0 = e->hwatch[0];
    char msg[256];
    snprintf(msg, sizeof msg,
             "dataflow acceptance watchdog: wait kind %llu at position %llu (aux %lld), "
             "low-water %llu, fetched %llu, iteration %lld",
             w0, e->hwatch[2], (long long)e->hwatch[3], e->hwatch[4], e->hwatch[5],
             (long long)e->iteration);
    memset(e->hwatch, 0, 8 * sizeof(unsigned long long));
    e->poisoned = true;
    e->poison_msg = std::string(msg) +
                    "; the engine state (labels, statistics, ledger) is undefined — destroy it";
    return fail(RCB_ERR_CUDA, e->poison_msg);
  }
  e->n_scored = n;
  e->last_par = n > 0 && e->cur_par;
  {
    float acc_ms = 0.f;
    if (e->last_par) cudaEventElapsedTime(&acc_ms, e->ev_acc[0], e->ev_acc[1]);
    e->counters[0] = e->last_par ? e->hctl[5] : 0;
    e->counters[1] = e->last_par ? e->hctl[6] : 0;
    e->counters[2] = e->last_par ? e->hctl[7] : 0;
    e->counters[3] = e->last_par ? e->hctl[8] : 0;
    e->counters[4] = (int64_t)e->hsc->nneg;
    e->counters[5] = e->hsc->moves;
    e->counters[6] = e->last_par ? 1 : 0;
    e->counters[7] = (int64_t)(acc_ms * 1000.f);
    e->counters[8] = e->last_par ? e->hctl[9] : 0;
    e->counters[9] = e->last_par ? e->hctl[10] : 0;
    e->counters[10] = e->last_par ? e->hctl[14] : 0;
    e->counters[11] = e->last_par ? e->hctl[15] : 0;
  }
  e->N = e->hsc->n_next;
  e->prepared = true;
  e->last_moves = e->hsc->moves;
  if (e->hsc->epoch > 0x80000000u) {  // BFS stamps near wrap: clear
    RCB_CUDA(cudaMemsetAsync(e->vis.p, 0, sizeof(uint32_t) * lat.V, s));
    e->hsc->epoch = 32;
    RCB_CUDA(cudaMemcpyAsync(&d->epoch, &e->hsc->epoch, sizeof(uint32_t), cudaMemcpyHostToDevice, s));
  }
  const int nev = 6;
  float t[nev] = {};
  for (int k = 1; k < nev; ++k) cudaEventElapsedTime(&t[k], e->ev[k - 1], e->ev[k]);
  e->times[0] = t[1];
  e->times[1] = t[2];
  e->times[2] = t[3];
  e->times[3] = t[4];
  e->times[4] = t[5];
  cudaEventElapsedTime(&e->times[5], e->ev[0], e->ev[5]);
  e->launches = launches + 2;
  rec->iteration = e->iteration;
  rec->energy = e->hsc->energy;
  rec->moves = e->hsc->moves;
  rec->particles = e->N;
  rec->candidates = n;
  rec->negative = (int64_t)e->hsc->nneg;
  rec->pairs = (int64_t)e->hsc->pairs;
  rec->mode = e->mode;
  return RCB_OK;
}

int32_t rcb_engine_iterate(rcb_engine *e, rcb_iter_record *rec) {
  if (e->poisoned) return fail(RCB_ERR_CUDA, e->poison_msg);
  if (e->scored) return fail(RCB_ERR_VALUE, "rcb_engine_iterate between score and finish");
  RCB_TRY(engine_score(e));
  return engine_finish(e, rec);
}

int32_t rcb_engine_set_slab(rcb_engine *e, int64_t lo, int64_t hi) {
  const int64_t np = e->lat.ndim == 3 ? e->lat.nz : e->lat.ny;
  if (hi > lo && (lo < 0 || hi > np)) return fail(RCB_ERR_VALUE, "slab outside the lattice");
  if (e->scored) return fail(RCB_ERR_VALUE, "slab change between score and finish");
  e->slab_lo = hi > lo ? lo : 0;
  e->slab_hi = hi > lo ? hi : 0;
  return RCB_OK;
}

int32_t rcb_engine_score(rcb_engine *e, rcb_slab_info *info) {
  if (e->poisoned) return fail(RCB_ERR_CUDA, e->poison_msg);
  if (e->scored) return fail(RCB_ERR_VALUE, "rcb_engine_score called twice");
  RCB_TRY(engine_score(e));
  info->n_particles = e->N;
  info->p0 = e->p0;
  info->p1 = e->p1;
  info->base = e->mode == 1 ? (void *)e->smooth.p : (void *)e->raw.p;
  const bool ps = e->ecfg.region_model == 1 && e->N > 0;
  info->cb0 = ps ? (void *)e->cb0.p : nullptr;
  info->sb0 = ps ? (void *)e->sb0.p : nullptr;
  info->stream = (void *)e->s;
  return RCB_OK;
}

int32_t rcb_engine_finish(rcb_engine *e, rcb_iter_record *rec) {
  if (e->poisoned) return fail(RCB_ERR_CUDA, e->poison_msg);
  return engine_finish(e, rec);
}

int32_t rcb_engine_band_limbs(rcb_engine *e, void **limbs, int32_t *n_limbs, int32_t *pending,
                              void **stream) {
  *limbs = e->band.p;
  *n_limbs = kLimbs;
  *pending = e->band_pending ? 1 : 0;
  *stream = (void *)e->s;
  return RCB_OK;
}

int32_t rcb_engine_band_apply(rcb_engine *e, double *energy) {
  if (e->poisoned) return fail(RCB_ERR_CUDA, e->poison_msg);
  RCB_CUDA(cudaSetDevice(e->device));
  if (e->band_pending) {
    RCB_TRY(band_ledger_apply(e->band.p, e->ecfg.lam, &e->sc.p->energy, e->s));
    e->band_pending = false;
  }
  RCB_CUDA(cudaMemcpyAsync(&e->hsc->energy, &e->sc.p->energy, sizeof(double),
                           cudaMemcpyDeviceToHost, e->s));
  RCB_CUDA(cudaStreamSynchronize(e->s));
  *energy = e->hsc->energy;
  return RCB_OK;
}

int32_t rcb_engine_particle_ranges(rcb_engine *e, const int64_t *planes, int32_t k, int64_t *out) {
  RCB_CUDA(cudaSetDevice(e->device));
  for (int32_t i = 0; i < k; i += 4) RCB_TRY(plane_ranges(e, planes + i, std::min(4, k - i), out + i));
  return RCB_OK;
}

int32_t rcb_engine_get_labels(rcb_engine *e, int32_t *out) {
  if (e->poisoned) return fail(RCB_ERR_CUDA, e->poison_msg);
  RCB_CUDA(cudaSetDevice(e->device));
  RCB_CUDA(cudaMemcpyAsync(out, e->L.p, sizeof(int32_t) * e->lat.V, cudaMemcpyDeviceToHost, e->s));
  RCB_CUDA(cudaStreamSynchronize(e->s));
  return RCB_OK;
}

int32_t rcb_engine_set_labels(rcb_engine *e, const int32_t *labels) {
  if (e->poisoned) return fail(RCB_ERR_CUDA, e->poison_msg);
  RCB_CUDA(cudaSetDevice(e->device));
  for (int64_t i = 0; i < e->lat.V; ++i)
    if (labels[i] < 0 || labels[i] >= e->nl)
      return fail(RCB_ERR_VALUE, "labels outside the engine's label table");
  e->fields_fresh = false;
  e->srec_current = false;
  RCB_CUDA(cudaMemcpyAsync(e->L.p, labels, sizeof(int32_t) * e->lat.V, cudaMemcpyHostToDevice, e->s));
  RCB_TRY(e->components());
  RCB_TRY(e->prepare());
  return RCB_OK;
}

}  // extern "C"

namespace {
__global__ void k_undo_moves(const int64_t *__restrict__ acc, int64_t m, int32_t *__restrict__ L) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < m) L[acc[3 * i]] = (int32_t)acc[3 * i + 1];  // every site flips at most once
}
}  // namespace

extern "C" {

int32_t rcb_engine_undo_last(rcb_engine *e) {
  if (e->poisoned) return fail(RCB_ERR_CUDA, e->poison_msg);
  RCB_CUDA(cudaSetDevice(e->device));
  const int64_t m = e->last_moves;
  if (m > 0) {
    k_undo_moves<<<grid_for(m, 256), 256, 0, e->s>>>(e->acc.p, m, e->L.p);
    RCB_CUDA(cudaGetLastError());
  }
  e->last_moves = 0;
  e->fields_fresh = false;
  e->srec_current = false;
  RCB_TRY(e->components());
  RCB_TRY(e->prepare());
  return RCB_OK;
}

int32_t rcb_engine_get_candidates(rcb_engine *e, int64_t *xs, int64_t *owners, int64_t *comps,
                                  double *rank, int64_t cap, int64_t *n) {
  if (e->poisoned) return fail(RCB_ERR_CUDA, e->poison_msg);
  *n = e->n_scored;
  if (cap < e->n_scored) return fail(RCB_ERR_CAPACITY, "candidate buffer too small");
  const int64_t m = e->n_scored;
  if (m == 0) return RCB_OK;
  RCB_CUDA(cudaSetDevice(e->device));
  std::vector<uint32_t> hx(m);
  std::vector<int32_t> ho(m), hc(m);
  RCB_CUDA(cudaMemcpyAsync(hx.data(), e->px.p, 4 * m, cudaMemcpyDeviceToHost, e->s));
  RCB_CUDA(cudaMemcpyAsync(ho.data(), e->pown.p, 4 * m, cudaMemcpyDeviceToHost, e->s));
  RCB_CUDA(cudaMemcpyAsync(hc.data(), e->pcomp.p, 4 * m, cudaMemcpyDeviceToHost, e->s));
  RCB_CUDA(cudaMemcpyAsync(rank, e->rank.p, 8 * m, cudaMemcpyDeviceToHost, e->s));
  RCB_CUDA(cudaStreamSynchronize(e->s));
  for (int64_t i = 0; i < m; ++i) {
    xs[i] = hx[i];
    owners[i] = ho[i];
    comps[i] = hc[i];
  }
  return RCB_OK;
}

int32_t rcb_engine_get_accepted(rcb_engine *e, int64_t *xab, int64_t cap, int64_t *n) {
  if (e->poisoned) return fail(RCB_ERR_CUDA, e->poison_msg);
  *n = e->last_moves;
  if (cap < e->last_moves) return fail(RCB_ERR_CAPACITY, "accepted-move buffer too small");
  if (e->last_moves == 0) return RCB_OK;
  RCB_CUDA(cudaSetDevice(e->device));
  RCB_CUDA(cudaMemcpyAsync(xab, e->acc.p, sizeof(int64_t) * 3 * e->last_moves,
                           cudaMemcpyDeviceToHost, e->s));
  RCB_CUDA(cudaStreamSynchronize(e->s));
  return RCB_OK;
}

int32_t rcb_engine_get_stats(rcb_engine *e, int64_t *count, double *total, double *total_sq,
                             int32_t n_labels) {
  if (e->poisoned) return fail(RCB_ERR_CUDA, e->poison_msg);
  if (n_labels < e->nl) return fail(RCB_ERR_CAPACITY, "stats buffers too small");
  RCB_CUDA(cudaSetDevice(e->device));
  RCB_TRY(e->flush_stats());
  RCB_CUDA(cudaMemcpyAsync(count, e->cnt.p, 8 * e->nl, cudaMemcpyDeviceToHost, e->s));
  RCB_CUDA(cudaMemcpyAsync(total, e->tot.p, 8 * e->nl, cudaMemcpyDeviceToHost, e->s));
  RCB_CUDA(cudaMemcpyAsync(total_sq, e->tsq.p, 8 * e->nl, cudaMemcpyDeviceToHost, e->s));
  RCB_CUDA(cudaStreamSynchronize(e->s));
  return RCB_OK;
}

int32_t rcb_engine_n_labels(rcb_engine *e, int32_t *n_labels) {
  *n_labels = e->nl;
  return RCB_OK;
}

int32_t rcb_engine_set_mode(rcb_engine *e, int32_t gradient) {
  if (gradient != 0 && gradient != 1) return fail(RCB_ERR_VALUE, "gradient must be 0 or 1");
  e->mode = gradient;
  return RCB_OK;
}

int32_t rcb_engine_set_energy(rcb_engine *e, double energy) {
  RCB_CUDA(cudaSetDevice(e->device));
  e->hsc->energy = energy;
  RCB_CUDA(cudaMemcpyAsync(&e->sc.p->energy, &e->hsc->energy, sizeof(double),
                           cudaMemcpyHostToDevice, e->s));
  RCB_CUDA(cudaStreamSynchronize(e->s));
  return RCB_OK;
}

int32_t rcb_engine_refresh(rcb_engine *e) {
  if (e->poisoned) return fail(RCB_ERR_CUDA, e->poison_msg);
  RCB_CUDA(cudaSetDevice(e->device));
  RCB_TRY(e->refresh());
  RCB_CUDA(cudaStreamSynchronize(e->s));
  e->fields_fresh = true;
  e->fields_partial = false;
  e->srec_current = false;  // the rebuild rewrote Cown / Sown / rho0
  return RCB_OK;
}

static int32_t evaluate_on(const int32_t *L, const double *I, const Lat &lat,
                           const rcb_energy_cfg *cfg, int32_t nl, double *external,
                           int64_t *internal, cudaStream_t s) {
  DBuf<long long> limbs;
  DBuf<unsigned long long> per;
  RCB_TRY(limbs.reserve(kLimbs, s));
  RCB_TRY(per.reserve(1, s));
  const int poisson = cfg->noise_model == 1;
  int32_t rc = RCB_OK;
  if (cfg->region_model == 0) {
    DBuf<int64_t> c;
    DBuf<double> t, q;
    StatsScratch ss;
    if ((rc = c.reserve(nl, s)) == RCB_OK && (rc = t.reserve(nl, s)) == RCB_OK &&
        (rc = q.reserve(nl, s)) == RCB_OK &&
        (rc = stats_rebuild(L, I, lat.V, nl, c.p, t.p, q.p, ss, s)) == RCB_OK)
      rc = pc_terms_exact(c.p, t.p, q.p, nl, poisson, limbs.p, s);
    cudaStreamSynchronize(s);
    c.release(s);
    t.release(s);
    q.release(s);
    ss.release(s);
  } else {
    DBuf<int32_t> C;
    DBuf<double> S;
    DBuf<Off> b;
    auto full = ball_table(lat.ndim, cfg->smooth_radius);
    if ((rc = C.reserve(lat.V, s)) == RCB_OK && (rc = S.reserve(lat.V, s)) == RCB_OK &&
        (rc = upload(b, full.data(), full.size(), s)) == RCB_OK &&
        (rc = ps_fields(L, I, lat, b.p, (int)full.size(), C.p, S.p, s)) == RCB_OK)
      rc = ps_terms_exact(C.p, S.p, I, lat.V, poisson, limbs.p, s);
    cudaStreamSynchronize(s);
    C.release(s);
    S.release(s);
    b.release(s);
  }
  if (rc == RCB_OK) rc = perimeter(L, lat, per.p, s);
  long long hl[kLimbs];
  unsigned long long hp = 0;
  if (rc == RCB_OK) {
    cudaMemcpyAsync(hl, limbs.p, sizeof(hl), cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(&hp, per.p, sizeof(hp), cudaMemcpyDeviceToHost, s);
    if (cudaStreamSynchronize(s) != cudaSuccess) rc = fail(RCB_ERR_CUDA, "evaluate sync failed");
  }
  limbs.release(s);
  per.release(s);
  if (rc != RCB_OK) return rc;
  *external = limbs_to_double(hl);
  *internal = (int64_t)hp;
  return RCB_OK;
}

int32_t rcb_engine_evaluate(rcb_engine *e, double *external, int64_t *internal) {
  if (e->poisoned) return fail(RCB_ERR_CUDA, e->poison_msg);
  RCB_CUDA(cudaSetDevice(e->device));
  if (!e->fields_fresh)
    return evaluate_on(e->L.p, e->I.p, e->lat, &e->ecfg, e->nl, external, internal, e->s);
  // right after refresh(): the engine's statistics / own-label fields are the
  // from-scratch ones of the current raster (same kernels as evaluate_on), so
  // only the exact term sums and the perimeter remain
  cudaStream_t s = e->s;
  RCB_TRY(e->eval_limbs.reserve(kLimbs, s));
  RCB_TRY(e->eval_per.reserve(1, s));
  const int poisson = e->ecfg.noise_model == 1;
  if (e->ecfg.region_model == 0)
    RCB_TRY(pc_terms_exact(e->cnt.p, e->tot.p, e->tsq.p, e->nl, poisson, e->eval_limbs.p, s));
  else
    RCB_TRY(ps_terms_exact(e->Cown.p, e->Sown.p, e->I.p, e->lat.V, poisson, e->eval_limbs.p, s));
  RCB_TRY(perimeter(e->L.p, e->lat, e->eval_per.p, s));
  long long hl[kLimbs];
  unsigned long long hp = 0;
  RCB_CUDA(cudaMemcpyAsync(hl, e->eval_limbs.p, sizeof(hl), cudaMemcpyDeviceToHost, s));
  RCB_CUDA(cudaMemcpyAsync(&hp, e->eval_per.p, sizeof(hp), cudaMemcpyDeviceToHost, s));
  RCB_CUDA(cudaStreamSynchronize(s));
  *external = limbs_to_double(hl);
  *internal = (int64_t)hp;
  return RCB_OK;
}

int32_t rcb_engine_stream(rcb_engine *e, void **stream) {
  *stream = (void *)e->s;
  return RCB_OK;
}

int32_t rcb_engine_debug_codes(rcb_engine *e, int32_t *particle, int32_t *code, int64_t cap,
                               int64_t *n) {
  const int64_t m = e->last_par ? (int64_t)e->hsc->nneg : 0;
  *n = m;
  if (cap < m) return fail(RCB_ERR_CAPACITY, "debug buffers too small");
  if (m == 0) return RCB_OK;
  RCB_CUDA(cudaSetDevice(e->device));
  RCB_CUDA(cudaMemcpyAsync(particle, e->order.p, 4 * m, cudaMemcpyDeviceToHost, e->s));
  RCB_CUDA(cudaMemcpyAsync(code, e->blocker.p, 4 * m, cudaMemcpyDeviceToHost, e->s));
  RCB_CUDA(cudaStreamSynchronize(e->s));
  return RCB_OK;
}

int32_t rcb_engine_debug_times(rcb_engine *e, int64_t *t2, int64_t cap, int64_t *n) {
  const int64_t m = (e->last_par && e->profile) ? (int64_t)e->hsc->nneg : 0;
  *n = m;
  if (cap < m) return fail(RCB_ERR_CAPACITY, "debug buffers too small");
  if (m == 0) return RCB_OK;
  RCB_CUDA(cudaMemcpyAsync(t2, e->tdbg.p, 32 * m, cudaMemcpyDeviceToHost, e->s));
  RCB_CUDA(cudaStreamSynchronize(e->s));
  return RCB_OK;
}

int32_t rcb_engine_counters(rcb_engine *e, int64_t *out8) {
  for (int k = 0; k < 12; ++k) out8[k] = e->counters[k];
  return RCB_OK;
}

int32_t rcb_engine_timings(rcb_engine *e, float *ms6, int32_t *launches) {
  for (int k = 0; k < 6; ++k) ms6[k] = e->times[k];
  *launches = e->launches;
  return RCB_OK;
}

// ---------------------------------------------------------------------------
// function-level drop-ins (stateless: upload, compute, download)
// ---------------------------------------------------------------------------

struct TmpStream {
  cudaStream_t s = nullptr;
  TmpStream() { cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking); }
  ~TmpStream() {
    if (s) {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
  }
};

int32_t rcb_sobolev_filter(const int64_t *coords, int64_t n, int32_t ndim, const int64_t *owners,
                           const int64_t *competitors, const double *raw,
                           const rcb_sobolev_cfg *params, double *out, int64_t *n_pairs) {
  *n_pairs = 0;
  if (ndim != 2 && ndim != 3) return fail(RCB_ERR_VALUE, "coords must be (n, 2) or (n, 3)");
  if (!(params->length_scale > 0) || params->length_scale > 30.0)
    return fail(RCB_ERR_VALUE, "length_scale must be in (0, 30]");
  if (n == 0) return RCB_OK;
  RCB_TRY(check_device());
  int64_t dims[3] = {0, 0, 0};
  for (int64_t i = 0; i < n; ++i)
    for (int k = 0; k < ndim; ++k) {
      int64_t c = coords[i * ndim + k];
      if (c < 0) return fail(RCB_ERR_VALUE, "coordinates must be non-negative");
      dims[k] = std::max(dims[k], c + 1);
    }
  for (int64_t i = 0; i < n; ++i) {
    if (competitors[i] < 0 || competitors[i] > 0x7fffffff || owners[i] < -0x7fffffffll ||
        owners[i] > 0x7fffffff)
      return fail(RCB_ERR_VALUE, "owner/competitor labels outside [0, 2^31)");
  }
  RCB_TRY(check_lattice(ndim, dims));
  Lat lat = make_lat(ndim, dims);
  int maxd2 = 0;
  auto st = sobolev_rows(ndim, params->length_scale, &maxd2);
  if (params->n_weights <= maxd2)
    return fail(RCB_ERR_VALUE, "Sobolev weight table shorter than the stencil needs");
  TmpStream ts;
  cudaStream_t s = ts.s;
  DBuf<int64_t> dc, dow, dcm;
  DBuf<double> draw, dout, dwt;
  DBuf<Off> dst;
  DBuf<unsigned long long> dp;
  int32_t rc = RCB_OK;
  auto go = [&]() -> int32_t {
    RCB_TRY(upload(dc, coords, (size_t)n * ndim, s));
    RCB_TRY(upload(dow, owners, n, s));
    RCB_TRY(upload(dcm, competitors, n, s));
    RCB_TRY(upload(draw, raw, n, s));
    RCB_TRY(upload(dwt, params->weights, params->n_weights, s));
    RCB_TRY(upload(dst, st.data(), st.size(), s));
    RCB_TRY(dout.reserve(n, s));
    RCB_TRY(dp.reserve(1, s));
    RCB_CUDA(cudaMemsetAsync(dp.p, 0, sizeof(unsigned long long), s));
    RCB_TRY(sobolev_coords(dc.p, n, ndim, lat, dow.p, dcm.p, draw.p, dst.p, (int)st.size(), dwt.p,
                           dout.p, dp.p, s));
    unsigned long long hp = 0;
    RCB_CUDA(cudaMemcpyAsync(out, dout.p, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    RCB_CUDA(cudaMemcpyAsync(&hp, dp.p, sizeof(hp), cudaMemcpyDeviceToHost, s));
    RCB_CUDA(cudaStreamSynchronize(s));
    *n_pairs = (int64_t)hp;
    return RCB_OK;
  };
  rc = go();
  dc.release(s); dow.release(s); dcm.release(s); draw.release(s); dout.release(s);
  dwt.release(s); dst.release(s); dp.release(s);
  return rc;
}

int32_t rcb_scan_contour(const int32_t *labels, int32_t ndim, const int64_t *dims, int32_t full_fg,
                         int64_t *xs, int64_t *owners, int64_t *competitors, int64_t cap,
                         int64_t *n) {
  *n = 0;
  RCB_TRY(check_lattice(ndim, dims));
  RCB_TRY(check_device());
  Lat lat = make_lat(ndim, dims);
  TmpStream ts;
  cudaStream_t s = ts.s;
  DBuf<int32_t> L, po, pc;
  DBuf<uint32_t> off, px;
  DBuf<uint8_t> tmp;
  int32_t rc = RCB_OK;
  auto go = [&]() -> int32_t {
    RCB_TRY(upload(L, labels, lat.V, s));
    RCB_TRY(off.reserve(lat.V + 1, s));
    RCB_TRY(contour_scan(L.p, lat, full_fg, off.p, tmp, s));
    uint32_t total = 0;
    RCB_CUDA(cudaMemcpyAsync(&total, off.p + lat.V, 4, cudaMemcpyDeviceToHost, s));
    RCB_CUDA(cudaStreamSynchronize(s));
    *n = total;
    if (cap < (int64_t)total) return fail(RCB_ERR_CAPACITY, "particle buffer too small");
    if (total == 0) return RCB_OK;
    RCB_TRY(px.reserve(total, s));
    RCB_TRY(po.reserve(total, s));
    RCB_TRY(pc.reserve(total, s));
    RCB_TRY(contour_emit(L.p, lat, full_fg, off.p, px.p, po.p, pc.p, s));
    std::vector<uint32_t> hx(total);
    std::vector<int32_t> ho(total), hc(total);
    RCB_CUDA(cudaMemcpyAsync(hx.data(), px.p, 4ull * total, cudaMemcpyDeviceToHost, s));
    RCB_CUDA(cudaMemcpyAsync(ho.data(), po.p, 4ull * total, cudaMemcpyDeviceToHost, s));
    RCB_CUDA(cudaMemcpyAsync(hc.data(), pc.p, 4ull * total, cudaMemcpyDeviceToHost, s));
    RCB_CUDA(cudaStreamSynchronize(s));
    for (uint32_t i = 0; i < total; ++i) {
      xs[i] = hx[i];
      owners[i] = ho[i];
      competitors[i] = hc[i];
    }
    return RCB_OK;
  };
  rc = go();
  L.release(s); po.release(s); pc.release(s); off.release(s); px.release(s); tmp.release(s);
  return rc;
}

static int32_t upload_particles(const int64_t *xs, const int64_t *owners, const int64_t *comps,
                                int64_t n, int64_t V, DBuf<uint32_t> &px, DBuf<int32_t> &po,
                                DBuf<int32_t> &pc, cudaStream_t s) {
  std::vector<uint32_t> hx(n);
  std::vector<int32_t> ho(n), hc(n);
  for (int64_t i = 0; i < n; ++i) {
    if (xs[i] < 0 || xs[i] >= V) return fail(RCB_ERR_VALUE, "pixel index out of range");
    if (owners[i] < 0 || owners[i] > 0x7fffffff || comps[i] < 0 || comps[i] > 0x7fffffff)
      return fail(RCB_ERR_VALUE, "labels must be non-negative int32");
    hx[i] = (uint32_t)xs[i];
    ho[i] = (int32_t)owners[i];
    hc[i] = (int32_t)comps[i];
  }
  RCB_TRY(upload(px, hx.data(), n, s));
  RCB_TRY(upload(po, ho.data(), n, s));
  RCB_TRY(upload(pc, hc.data(), n, s));
  RCB_CUDA(cudaStreamSynchronize(s));
  return RCB_OK;
}

int32_t rcb_delta_internal_batch(const int32_t *labels, int32_t ndim, const int64_t *dims,
                                 const int64_t *xs, const int64_t *owners,
                                 const int64_t *competitors, int64_t n, int64_t *out) {
  RCB_TRY(check_lattice(ndim, dims));
  if (n == 0) return RCB_OK;
  RCB_TRY(check_device());
  Lat lat = make_lat(ndim, dims);
  TmpStream ts;
  cudaStream_t s = ts.s;
  DBuf<int32_t> L, po, pc, d;
  DBuf<uint32_t> px;
  auto go = [&]() -> int32_t {
    RCB_TRY(upload(L, labels, lat.V, s));
    RCB_TRY(upload_particles(xs, owners, competitors, n, lat.V, px, po, pc, s));
    RCB_TRY(d.reserve(n, s));
    RCB_TRY(delta_int_batch(L.p, lat, px.p, po.p, pc.p, n, d.p, s));
    std::vector<int32_t> h(n);
    RCB_CUDA(cudaMemcpyAsync(h.data(), d.p, 4 * n, cudaMemcpyDeviceToHost, s));
    RCB_CUDA(cudaStreamSynchronize(s));
    for (int64_t i = 0; i < n; ++i) out[i] = h[i];
    return RCB_OK;
  };
  int32_t rc = go();
  L.release(s); po.release(s); pc.release(s); d.release(s); px.release(s);
  return rc;
}

int32_t rcb_delta_external_batch(const double *image, const int32_t *labels, int32_t ndim,
                                 const int64_t *dims, const rcb_energy_cfg *cfg,
                                 int32_t n_labels, const int64_t *count, const double *total,
                                 const double *total_sq, const int64_t *xs,
                                 const int64_t *owners, const int64_t *competitors, int64_t n,
                                 double *out) {
  RCB_TRY(check_lattice(ndim, dims));
  if (n == 0) return RCB_OK;
  RCB_TRY(check_device());
  Lat lat = make_lat(ndim, dims);
  for (int64_t i = 0; i < n; ++i)
    if (owners[i] >= n_labels || competitors[i] >= n_labels)
      return fail(RCB_ERR_VALUE, "label outside the statistics table");
  TmpStream ts;
  cudaStream_t s = ts.s;
  DBuf<int32_t> L, po, pc, C;
  DBuf<uint32_t> px;
  DBuf<double> I, d, S, t, q;
  DBuf<int64_t> c;
  DBuf<Off> b;
  const int poisson = cfg->noise_model == 1;
  auto go = [&]() -> int32_t {
    RCB_TRY(upload(L, labels, lat.V, s));
    RCB_TRY(upload(I, image, lat.V, s));
    RCB_TRY(upload_particles(xs, owners, competitors, n, lat.V, px, po, pc, s));
    RCB_TRY(d.reserve(n, s));
    if (cfg->region_model == 0) {
      RCB_TRY(upload(c, count, n_labels, s));
      RCB_TRY(upload(t, total, n_labels, s));
      RCB_TRY(upload(q, total_sq, n_labels, s));
      RCB_TRY(delta_pc_batch(I.p, px.p, po.p, pc.p, n, c.p, t.p, q.p, poisson, d.p, s));
    } else {
      if (cfg->smooth_radius < 1 || cfg->smooth_radius > 15)
        return fail(RCB_ERR_VALUE, "smooth_radius must be in [1, 15]");
      auto full = ball_table(ndim, cfg->smooth_radius);
      RCB_TRY(upload(b, full.data(), full.size(), s));
      RCB_TRY(C.reserve(lat.V, s));
      RCB_TRY(S.reserve(lat.V, s));
      RCB_TRY(ps_fields(L.p, I.p, lat, b.p, (int)full.size(), C.p, S.p, s));
      RCB_TRY(delta_ps_batch(L.p, I.p, C.p, S.p, lat, b.p + 1, (int)full.size() - 1, px.p, po.p,
                             pc.p, n, poisson, d.p, s));
    }
    RCB_CUDA(cudaMemcpyAsync(out, d.p, 8 * n, cudaMemcpyDeviceToHost, s));
    RCB_CUDA(cudaStreamSynchronize(s));
    return RCB_OK;
  };
  int32_t rc = go();
  L.release(s); po.release(s); pc.release(s); C.release(s); px.release(s); I.release(s);
  d.release(s); S.release(s); t.release(s); q.release(s); c.release(s); b.release(s);
  return rc;
}

int32_t rcb_stats_from_labels(const double *image, const int32_t *labels, int64_t size,
                              int32_t n_labels, int64_t *count, double *total, double *total_sq) {
  if (size < 0 || n_labels < 1) return fail(RCB_ERR_VALUE, "bad sizes");
  RCB_TRY(check_device());
  for (int64_t i = 0; i < size; ++i)
    if (labels[i] < 0 || labels[i] >= n_labels)
      return fail(RCB_ERR_VALUE, "label outside [0, n_labels)");
  TmpStream ts;
  cudaStream_t s = ts.s;
  DBuf<int32_t> L;
  DBuf<double> I, t, q;
  DBuf<int64_t> c;
  StatsScratch ss;
  auto go = [&]() -> int32_t {
    RCB_TRY(upload(L, labels, size, s));
    RCB_TRY(upload(I, image, size, s));
    RCB_TRY(c.reserve(n_labels, s));
    RCB_TRY(t.reserve(n_labels, s));
    RCB_TRY(q.reserve(n_labels, s));
    RCB_TRY(stats_rebuild(L.p, I.p, size, n_labels, c.p, t.p, q.p, ss, s));
    RCB_CUDA(cudaMemcpyAsync(count, c.p, 8 * n_labels, cudaMemcpyDeviceToHost, s));
    RCB_CUDA(cudaMemcpyAsync(total, t.p, 8 * n_labels, cudaMemcpyDeviceToHost, s));
    RCB_CUDA(cudaMemcpyAsync(total_sq, q.p, 8 * n_labels, cudaMemcpyDeviceToHost, s));
    RCB_CUDA(cudaStreamSynchronize(s));
    return RCB_OK;
  };
  int32_t rc = go();
  L.release(s); I.release(s); t.release(s); q.release(s); c.release(s); ss.release(s);
  return rc;
}

int32_t rcb_evaluate_total(const double *image, const int32_t *labels, int32_t ndim,
                           const int64_t *dims, const rcb_energy_cfg *cfg, double *external,
                           int64_t *internal) {
  RCB_TRY(check_lattice(ndim, dims));
  RCB_TRY(check_device());
  Lat lat = make_lat(ndim, dims);
  int32_t mx = 0;
  for (int64_t i = 0; i < lat.V; ++i) {
    if (labels[i] < 0) return fail(RCB_ERR_VALUE, "label raster contains negative labels");
    mx = std::max(mx, labels[i]);
  }
  if (cfg->region_model == 1 && (cfg->smooth_radius < 1 || cfg->smooth_radius > 15))
    return fail(RCB_ERR_VALUE, "smooth_radius must be in [1, 15]");
  TmpStream ts;
  cudaStream_t s = ts.s;
  DBuf<int32_t> L;
  DBuf<double> I;
  DBuf<float> I32, raw32, wt32;  // fp32 mode
  DBuf<int32_t> cb0;             // PS: competitor ball count/sum per particle (K5)
  DBuf<double> sb0;
  int32_t rc = upload(L, labels, lat.V, s);
  if (rc == RCB_OK) rc = upload(I, image, lat.V, s);
  if (rc == RCB_OK) rc = evaluate_on(L.p, I.p, lat, cfg, mx + 1, external, internal, s);
  L.release(s);
  I.release(s);
  return rc;
}

}  // extern "C"
