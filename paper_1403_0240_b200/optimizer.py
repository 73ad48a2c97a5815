"""Region Competition driver (mirror of rcseg.optimizer, optimizer.py:36-279).

``RegionCompetition.iterate`` is one call into the device engine
(``rcb_engine_iterate``): particle extraction, ΔE, Sobolev filter, ranking and
the topology-safe acceptance all run on the GPU, and one small record comes
back.  The run policy around it — resync cadence and drift check,
oscillation detection, the one-way sobolev→l2 fallback and the statuses —
is host scalar logic, kept here exactly as the reference states it.
"""
from __future__ import annotations

import ctypes as C
import math
import time
import weakref
from dataclasses import dataclass

import numpy as np

from . import _lib
from .contour import ContourState, scan_particles
from .energy import EnergyConfig, EnergyValue, evaluate_total
from .grid import LABEL_DTYPE, Connectivity, StatsTable, validate_image, validate_labels
from .init import initialize, otsu_threshold, split_disjoint_labels  # noqa: F401  (optimizer.py:284-405)
from .sobolev import SobolevParams, detect_oscillation, sobolev_cfg


@dataclass
class OptimizerConfig:
    """optimizer.py:36-56"""
    gradient: str = "sobolev"
    max_iterations: int = 2000
    oscillation_window: int = 10
    oscillation_tol: float = 1e-6
    move_budget: float = 1.0
    seed: int = 0
    allow_fusion: bool = False
    allow_vanish: bool = True
    vanish_grace: int = 0
    resync_every: int = 10
    drift_tolerance: float = 1e-6
    debug_check_rate: float = 0.0
    precision: str = "fp64"         # "fp64" (reference-exact) | "fp32" (gradient path in fp32)

    def __post_init__(self):
        if self.precision not in ("fp64", "fp32"):
            raise ValueError(f"unknown precision {self.precision!r}")
        if self.gradient not in ("l2", "sobolev"):
            raise ValueError(f"unknown gradient mode {self.gradient!r}")
        if not 0.0 < self.move_budget <= 1.0:
            raise ValueError("move_budget must be in (0, 1]")


@dataclass
class IterationRecord:
    iteration: int
    energy: float
    moves: int
    particles: int
    mode: str
    seconds: float


@dataclass
class RunResult:
    labels: np.ndarray
    trace: list
    status: str
    iterations: int
    wall_seconds: float
    final_energy: EnergyValue
    region_count: int
    fallback_iteration: int | None = None


class _DeviceModel:
    """``engine.model`` view: stats fetched from the device on access."""

    def __init__(self, eng: "RegionCompetition"):
        # weak: no engine <-> model reference cycle, so dropping the engine
        # frees its device memory at once instead of at the next GC pass
        self._ref = weakref.ref(eng)

    @property
    def _eng(self) -> "RegionCompetition":
        e = self._ref()
        if e is None:
            raise RuntimeError("the engine of this model was destroyed")
        return e

    @property
    def stats(self) -> StatsTable:
        e = self._eng
        nl = e.n_labels
        t = StatsTable(nl)
        _lib.check(_lib.lib.rcb_engine_get_stats(e._h, _lib.ptr(t.count), _lib.ptr(t.total),
                                                 _lib.ptr(t.total_sq), nl))
        return t

    def refresh(self) -> None:
        _lib.check(_lib.lib.rcb_engine_refresh(self._eng._h))


class RegionCompetition:
    """Stateful engine on one GPU; owns a device copy of the labeling."""

    def __init__(self, image, init_labels, energy_config: EnergyConfig,
                 sobolev_params: SobolevParams | None = None,
                 config: OptimizerConfig | None = None, conn: Connectivity | None = None,
                 device: int = 0, stream=None):
        # grid.py:24-39 / optimizer.py:100-101: rank and dtype here; the value
        # checks (non-finite intensities, negative labels, negative intensities
        # under Poisson) run on the device in rcb_engine_create, same messages
        validate_image(image, values=False)
        validate_labels(init_labels, values=False)
        if image.shape != init_labels.shape:
            raise ValueError("image and labels differ in shape")
        _lib.require_device()
        self.device = int(device)
        self._slab = None
        self._exchange = None
        # float32 rasters go to the device as float32 and are promoted there
        # (exactly numpy's astype, optimizer.py:102); anything else is promoted
        # to float64 on the host as the reference does
        if isinstance(image, np.ndarray) and image.dtype == np.float32:
            src, dtype_code = np.ascontiguousarray(image), 1
        else:
            src, dtype_code = np.ascontiguousarray(image, dtype=np.float64), 0
        self._image_src = src
        self._image64 = src if dtype_code == 0 else None
        self.shape = src.shape
        self.conn = conn if conn is not None else Connectivity.default(src.ndim)
        self.energy_config = energy_config
        self.sobolev_params = sobolev_params if sobolev_params is not None else SobolevParams()
        self.config = config if config is not None else OptimizerConfig()
        self.mode = self.config.gradient
        lab = np.ascontiguousarray(init_labels, dtype=LABEL_DTYPE)
        self._ecfg = energy_config.c_struct()
        self._scfg, self._wt = sobolev_cfg(self.sobolev_params)
        cfg = self.config
        self._ocfg = _lib.OptCfg(int(self.mode == "sobolev"), float(cfg.move_budget),
                                 int(cfg.seed) & 0xFFFFFFFFFFFFFFFF, int(cfg.allow_fusion),
                                 int(cfg.allow_vanish), int(cfg.vanish_grace),
                                 int(self.conn.full_fg), int(cfg.precision == "fp32"))
        dims = _lib.dims_arr(self.shape)
        h = C.c_void_p()
        _lib.check(_lib.lib.rcb_engine_create_ex(
            _lib.ptr(src), dtype_code, _lib.ptr(lab), lab.ndim, _lib.ptr(dims), C.byref(self._ecfg),
            C.byref(self._scfg), C.byref(self._ocfg), int(device),
            C.c_void_p(int(stream) if stream else 0), C.byref(h)))
        self._h = h
        nl = C.c_int32(0)
        _lib.check(_lib.lib.rcb_engine_n_labels(h, C.byref(nl)))
        self.n_labels = nl.value
        self.model = _DeviceModel(self)
        self.iteration = 0
        self.fallback_iteration: int | None = None
        self.trace: list[IterationRecord] = []
        self._cand = None
        self._last_n = 0
        self.last_pairs = 0
        self.last_negative = 0
        self._energy = self._evaluate().total
        _lib.check(_lib.lib.rcb_engine_set_energy(h, self._energy))
        self._mode_start = 0
        self._rng = np.random.default_rng(self.config.seed)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            _lib.lib.rcb_engine_destroy(h)
            self._h = None

    @property
    def image(self) -> np.ndarray:
        """The float64 intensity raster (optimizer.py:102), promoted on first use."""
        if self._image64 is None:
            self._image64 = np.ascontiguousarray(self._image_src, dtype=np.float64)
        return self._image64

    # -- device state views ----------------------------------------------------
    @property
    def labels(self) -> np.ndarray:
        out = np.empty(self.shape, LABEL_DTYPE)
        _lib.check(_lib.lib.rcb_engine_get_labels(self._h, _lib.ptr(out)))
        return out

    @labels.setter
    def labels(self, value) -> None:
        lab = np.ascontiguousarray(value, LABEL_DTYPE)
        if lab.shape != self.shape:
            raise ValueError("labels differ in shape")
        _lib.check(_lib.lib.rcb_engine_set_labels(self._h, _lib.ptr(lab)))

    @property
    def contour(self) -> ContourState:
        xs, _, cs = scan_particles(self.labels, self.conn)
        return ContourState(xs, cs)

    @property
    def last_candidates(self):
        """(pixels, owners, competitors, rank values) of the last iteration,
        in (pixel, competitor) order (optimizer.py:140-142)."""
        if self._cand is None:
            n = self._last_n
            xs, ow, cm = (np.empty(n, np.int64) for _ in range(3))
            rk = np.empty(n, np.float64)
            got = C.c_int64(0)
            _lib.check(_lib.lib.rcb_engine_get_candidates(
                self._h, _lib.ptr(xs), _lib.ptr(ow), _lib.ptr(cm), _lib.ptr(rk), n,
                C.byref(got)))
            self._cand = (xs, ow, cm, rk)
        return self._cand

    @property
    def last_accepted(self) -> np.ndarray:
        """Accepted moves of the last iteration as rows (x, a, b), in
        acceptance order."""
        n = self.trace[-1].moves if self.trace else 0
        out = np.empty((n, 3), np.int64)
        got = C.c_int64(0)
        _lib.check(_lib.lib.rcb_engine_get_accepted(self._h, _lib.ptr(out), n, C.byref(got)))
        return out

    def _evaluate(self) -> EnergyValue:
        ext = C.c_double(0.0)
        inter = C.c_int64(0)
        _lib.check(_lib.lib.rcb_engine_evaluate(self._h, C.byref(ext), C.byref(inter)))
        internal = int(inter.value)
        return EnergyValue(ext.value + self.energy_config.lam * internal, ext.value, internal)

    def timings(self):
        """Device ms of the last iterate() phases (extract, energy, sobolev,
        rank, accept, whole) and the launch count."""
        t = (C.c_float * 6)()
        n = C.c_int32(0)
        _lib.check(_lib.lib.rcb_engine_timings(self._h, t, C.byref(n)))
        return list(t), n.value

    def counters(self) -> dict:
        """Acceptance diagnostics of the last iterate() (rcb_engine_counters)."""
        out = np.zeros(12, np.int64)
        _lib.check(_lib.lib.rcb_engine_counters(self._h, _lib.ptr(out)))
        keys = ["rounds", "bfs_runs", "deferred", "bfs_blocked", "negative", "moves",
                "parallel", "accept_us", "bfs_levels", "bfs_max_levels", "ps_recounts",
                "ps_flips"]
        return dict(zip(keys, out.tolist()))

    @property
    def stream(self) -> int:
        s = C.c_void_p()
        _lib.check(_lib.lib.rcb_engine_stream(self._h, C.byref(s)))
        return s.value or 0

    # -- single iteration (optimizer.py:122-160) -------------------------------
    def iterate(self) -> IterationRecord:
        t0 = self._pre_iterate()
        if self._slab is None:
            rec = _lib.IterRecord()
            _lib.check(_lib.lib.rcb_engine_iterate(self._h, C.byref(rec)))
        else:  # z-slab sharded (shard.py): score, all-gather the slabs' scores, finish
            info = self._slab.score()
            self._exchange.gather(self._slab.buffers(info, self.device), self._slab.ranges(),
                                  stream=info.stream)
            rec = self._slab.finish()
            limbs, st = self._slab.band_limbs(self.device)
            if limbs is not None:  # slab-local band refresh: sum the ledger shares
                self._exchange.reduce_limbs(limbs, stream=st)
                rec = self._slab.band_apply(rec)
        return self._post_iterate(rec, t0)

    def attach_slab(self, slab, exchange) -> None:
        """Shard the scoring kernels by outer planes (shard.slab_engine)."""
        self._slab = slab
        self._exchange = exchange

    def _pre_iterate(self) -> float:
        t0 = time.perf_counter()
        if self.config.debug_check_rate > 0.0:
            self._debug_check()
        _lib.check(_lib.lib.rcb_engine_set_mode(self._h, int(self.mode == "sobolev")))
        return t0

    def _post_iterate(self, rec, t0: float) -> IterationRecord:
        cfg = self.config
        self.iteration = int(rec.iteration)
        self._cand = None
        self._last_n = int(rec.candidates)
        self.last_pairs = int(rec.pairs)
        self.last_negative = int(rec.negative)
        self._energy = float(rec.energy)
        if self.iteration % cfg.resync_every == 0:
            self.model.refresh()
            self._resync()
        out = IterationRecord(self.iteration, self._energy, int(rec.moves), int(rec.particles),
                              self.mode, time.perf_counter() - t0)
        self.trace.append(out)
        return out

    def _resync(self) -> None:
        """optimizer.py:202-209"""
        oracle = self._evaluate()
        drift = abs(oracle.total - self._energy)
        if drift > self.config.drift_tolerance:
            raise RuntimeError(f"incremental energy drifted {drift:.3e} from the oracle "
                               f"at iteration {self.iteration}")
        self._energy = oracle.total
        _lib.check(_lib.lib.rcb_engine_set_energy(self._h, self._energy))

    def _debug_check(self) -> None:
        """optimizer.py:211-228: sample increments against from-scratch totals
        (increments of the coming iteration's particle set, on the GPU)."""
        from .energy import EnergyModel, delta_internal_batch
        labels = self.labels
        xs, ow, cm = scan_particles(labels, self.conn)
        n = len(xs)
        if n == 0:
            return
        model = EnergyModel(self.image, labels, self.energy_config)
        raw_ext = model.delta_external_batch(xs, ow, cm)
        raw_int = delta_internal_batch(labels, xs, ow, cm)
        k = max(1, int(round(self.config.debug_check_rate * n)))
        sample = self._rng.choice(n, size=min(k, n), replace=False)
        lam = self.energy_config.lam
        before = evaluate_total(labels, self.image, self.energy_config)
        for i in sample:
            trial = labels.copy()
            trial.ravel()[int(xs[i])] = int(cm[i])
            after = evaluate_total(trial, self.image, self.energy_config)
            oracle = after.total - before.total
            mine = float(raw_ext[i] + lam * raw_int[i])
            if abs(mine - oracle) > max(1e-9 * abs(oracle), 1e-12):
                raise RuntimeError(f"incremental delta {mine!r} disagrees with oracle "
                                   f"{oracle!r} at pixel {int(xs[i])} -> {int(cm[i])}")

    # -- full run (optimizer.py:232-270) ---------------------------------------
    def run(self, on_iteration=None) -> RunResult:
        cfg = self.config
        t0 = time.perf_counter()
        status = "max-iter"
        for _ in range(cfg.max_iterations):
            # only an l2-mode oscillation halt restores the previous labeling;
            # the engine undoes the last iteration's moves on the device
            # instead of copying the raster to the host every iteration
            prev_energy = self._energy
            rec = self.iterate()
            if on_iteration is not None:
                on_iteration(self, rec)
            if rec.moves == 0:
                status = ("fallback-then-converged" if self.fallback_iteration is not None
                          else "converged")
                break
            recent = self.trace[self._mode_start:]
            if detect_oscillation([r.energy for r in recent], [r.moves for r in recent],
                                  cfg.oscillation_window, cfg.oscillation_tol):
                if self.mode == "sobolev":
                    self.mode = "l2"
                    self.fallback_iteration = self.iteration
                    self._mode_start = len(self.trace)
                else:
                    status = "oscillation-halt"
                    if prev_energy < self._energy:
                        _lib.check(_lib.lib.rcb_engine_undo_last(self._h))
                        self.model.refresh()
                        self._energy = prev_energy
                        _lib.check(_lib.lib.rcb_engine_set_energy(self._h, self._energy))
                    break
        final = self._evaluate()
        self._energy = final.total
        stats = self.model.stats
        region_count = int(np.count_nonzero(stats.count[1:] > 0))
        return RunResult(labels=self.labels, trace=self.trace, status=status,
                         iterations=len(self.trace), wall_seconds=time.perf_counter() - t0,
                         final_energy=final, region_count=region_count,
                         fallback_iteration=self.fallback_iteration)


def run(image, init_labels, energy_config: EnergyConfig,
        sobolev_params: SobolevParams | None = None, config: OptimizerConfig | None = None,
        conn: Connectivity | None = None, on_iteration=None) -> RunResult:
    """optimizer.py:273-279"""
    engine = RegionCompetition(image, init_labels, energy_config, sobolev_params, config, conn)
    return engine.run(on_iteration=on_iteration)
