"""Bitstring genetic algorithm (SPEC.md evolve module).

The reference ships no GA: this module defines the
semantics from SPEC and runs the generation loop on the device
(``tv_ga_run``: one cooperative sm_100a kernel per call, fitness -> roulette
CDF -> selection / crossover / Poisson mutation for every child).  The
per-child random stream is counter-based splitmix64 keyed by (seed,
generation, child), the same construction as the enumeration path
(_k:38-60), so every trajectory is reproducible and independent of launch
geometry; the CPU restatement oracle/tv_ga_oracle.c reproduces it bit for bit
(tests/test_ga.py).  The single-genome operators below are host utilities
with the same draw semantics (they are what one child of the kernel does).

Genomes are held as the integer ``Genome.to_int()`` (genome bit 0 = most
significant of L bits).  L <= 64: one u64 per genome and the cooperative
kernel; 64 < L <= 4096: ``W = ceil(L/64)`` little-endian u64 words per genome
(arrays ``[n, W]``, word 0 = the integer's low 64 bits), three launches per
generation (oracle/tv_ga_oracle.c ``orc_ga_run_w``; the uniform-crossover mask is
drawn one word at a time, word 0 first, which for W = 1 is the narrow operator).
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .genome import Genome, SearchSpace

GOLD = 0x9E3779B97F4A7C15
MIXA = 0xBF58476D1CE4E5B9
MIXB = 0x94D049BB133111EB
M64 = (1 << 64) - 1

MODES = {"asexual": 0, "single_point": 1, "uniform": 2}


def _mix64(z: int) -> int:
    z = ((z ^ (z >> 30)) * MIXA) & M64
    z = ((z ^ (z >> 27)) * MIXB) & M64
    return z ^ (z >> 31)


class GaRng:
    """Counter-based stream of one child: key (seed, generation, child)."""

    __slots__ = ("s",)

    def __init__(self, seed: int, generation: int = 0, child: int = 0):
        z = _mix64((seed ^ ((GOLD * (generation + 1)) & M64)) & M64)
        self.s = _mix64(z ^ ((MIXA * (child + 1)) & M64))

    def next(self) -> int:
        self.s = (self.s + GOLD) & M64
        return _mix64(self.s)

    def below(self, n: int) -> int:
        """((draw >> 32) * n) >> 32, the reference's bounded draw (_k:57-60)."""
        return ((self.next() >> 32) * n) >> 32

    def mulhi(self, n: int) -> int:
        """uniform integer in [0, n) for any n < 2^64: high word of draw * n."""
        return (self.next() * n) >> 64


def poisson_thresholds(lam: float, L: int) -> np.ndarray:
    """T[j] = floor(P(K <= j) * 2^63) for K ~ Poisson(lam), j < L (Eq. 1).

    A flip count is k = #{j : (draw >> 1) >= T[j]}, i.e. inversion sampling
    clamped at L (App. D.1 "if(r_fNrMutations > mBitLengthGenome)").  Computed
    once on the host and shared by the device and the CPU restatement."""
    if lam < 0:
        raise ValueError("lambda must be >= 0")
    T = np.empty(L, np.uint64)
    p = math.exp(-lam)
    cdf = 0.0
    for j in range(L):
        cdf += p
        p *= lam / (j + 1)
        T[j] = min(1 << 63, int(math.floor(min(cdf, 1.0) * 2.0 ** 63)))
    return T


# ---------------------------------------------------------------- single-genome operators
def _as_int(g) -> tuple[int, int | None]:
    return (g.to_int(), g.length) if isinstance(g, Genome) else (int(g), None)


def poisson_sample(lam: float, rng: GaRng, L: int = 64) -> int:
    """k ~ Poisson(lam) by inversion against poisson_thresholds (clamped to L)."""
    T = poisson_thresholds(lam, L)
    u = rng.next() >> 1
    return int(np.count_nonzero(u >= T))


def mutate(g, lam: float, rng: GaRng, L: int | None = None):
    """Flip k ~ Poisson(lam) (clamped to L) DISTINCT uniform positions."""
    v, glen = _as_int(g)
    L = L or glen
    k = poisson_sample(lam, rng, L)
    chosen = 0
    while bin(chosen).count("1") < k:
        chosen |= 1 << (L - 1 - rng.below(L))
    out = v ^ chosen
    return Genome.from_int(L, out) if glen else out


def crossover_single_point(a, b, rng: GaRng, L: int | None = None):
    """Child = a's bits at positions < p, b's from p on; p uniform in [0, L)."""
    av, la = _as_int(a)
    bv, lb = _as_int(b)
    if la is not None and la != lb:
        raise ValueError("genome lengths differ")
    L = L or la
    p = rng.below(L)
    full = (1 << L) - 1
    top = 0 if p == 0 else full & ~((1 << (L - p)) - 1)
    out = (av & top) | (bv & ~top & full)
    return Genome.from_int(L, out) if la else out


def crossover_uniform(a, b, rng: GaRng, L: int | None = None):
    """Each bit from a or b with probability 1/2."""
    av, la = _as_int(a)
    bv, lb = _as_int(b)
    if la is not None and la != lb:
        raise ValueError("genome lengths differ")
    L = L or la
    m = 0
    for w in range((L + 63) // 64):  # one draw per 64-bit word, word 0 (the low bits) first
        m |= (rng.next() & ((1 << min(64, L - 64 * w)) - 1)) << (64 * w)
    out = (av & ~m) | (bv & m)
    return Genome.from_int(L, out) if la else out


def roulette_select(weights, rng: GaRng | None = None, cutoff=None) -> int:
    """Smallest i whose partial sum reaches the draw (App. C.1).

    With ``cutoff`` given it is the draw itself (weights {2,3,4,1}, cutoff 10 -> 3).
    Otherwise integer weights use an exact integer draw r in [0, sum) and return
    the first i with partial sum > r (= partial sum >= r + 1/2, so zero weights
    are never picked); sum == 0 falls back to a uniform index."""
    w = np.asarray(weights)
    cs = np.cumsum(w)
    if cutoff is not None:
        return int(np.searchsorted(cs, cutoff, side="left"))
    total = cs[-1]
    if total <= 0:
        return rng.mulhi(len(w))
    if np.issubdtype(w.dtype, np.integer):
        r = rng.mulhi(int(total))
        return int(np.searchsorted(cs, r, side="right"))
    u = (rng.next() >> 11) * 2.0 ** -53 * float(total)
    return int(np.searchsorted(cs, u, side="right"))


def fujiyama_fitness(g) -> int:
    """Hamming weight."""
    v, _ = _as_int(g)
    return bin(v).count("1")


# ---------------------------------------------------------------- run records
@dataclass
class GAConfig:
    pop_size: int = 512
    length: int = 32
    mu_L: float = 0.3                  # lambda = expected flips per genome per generation
    mode: str = "asexual"              # asexual | single_point | uniform
    cutoff: int = 20000
    target: int = 25                   # H >= 25 (Figs. 9-10)
    adapt_fraction: float = 0.5        # half the population at target
    stop_when: str = "adaptation"      # never | discovery | adaptation
    init: np.ndarray | None = None     # u64 genomes; default all-zero


@dataclass
class RunRecord:
    best: np.ndarray
    mean: np.ndarray
    count_at_target: np.ndarray
    generations: int
    discovery: int | None              # None = censored at the cutoff
    adaptation: int | None
    config: GAConfig = field(default=None)
    seed: int = 0


def discovery_time(record: RunRecord):
    """First generation any individual met the target, or None (censored)."""
    return record.discovery


def adaptation_time(record: RunRecord, proportion: float | None = None, threshold: int | None = None):
    """First generation >= proportion*N individuals met the threshold, or None (censored)."""
    cfg = record.config
    if threshold is not None and cfg is not None and threshold != cfg.target:
        raise ValueError("counts were recorded for the configured target only")
    x = cfg.adapt_fraction if proportion is None else proportion
    need = math.ceil(x * cfg.pop_size)
    hit = np.nonzero(record.count_at_target >= need)[0]
    return int(hit[0]) if hit.size else None


def bootstrap_median_ci(samples, sample_size: int = 100, resamples: int = 10000, rng=None, alpha: float = 0.05):
    """Sample median and percentile CI of the bootstrap median distribution."""
    x = np.asarray(samples, dtype=np.float64)
    if x.size == 0:
        raise ValueError("samples must be non-empty")
    rng = rng if rng is not None else np.random.default_rng(0)
    meds = np.median(x[rng.integers(0, x.size, (resamples, sample_size))], axis=1)
    return float(np.median(x)), float(np.quantile(meds, alpha / 2)), float(np.quantile(meds, 1 - alpha / 2))


# ---------------------------------------------------------------- device engine
class DeviceGA:
    """Device population + generation loop (tv_ga_*)."""

    def __init__(self, pop_size: int, length: int, mu_L: float, mode: str = "asexual"):
        self.n, self.L = int(pop_size), int(length)
        self.W = (self.L + 63) // 64  # words per genome (> 1: the wide path, arrays [n, W])
        self.mode = MODES[mode] if isinstance(mode, str) else int(mode)
        self.T = poisson_thresholds(mu_L, self.L)
        h = ctypes.c_void_p()
        _lib.check(_lib.lib().tv_ga_create(self.n, self.L, self.mode, _lib.ptr(self.T), ctypes.byref(h)))
        self._h = h
        self._fit = None
        self.device = _current_device()  # the handle's buffers live there (the C ABI checks it)

    def close(self):
        if self._h:
            _lib.lib().tv_ga_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_population(self, genomes=None):
        g = None
        if genomes is not None:
            g = np.ascontiguousarray(genomes, np.uint64)
            want = (self.n,) if self.W == 1 else (self.n, self.W)
            if g.shape != want:
                raise ValueError(f"population must have shape {want}, got {g.shape}")
        _lib.check(_lib.lib().tv_ga_set_population(self._h, _lib.ptr(g), None))

    def population(self) -> np.ndarray:
        out = np.empty(self.n if self.W == 1 else (self.n, self.W), np.uint64)
        _lib.check(_lib.lib().tv_ga_get_population(self._h, _lib.ptr(out), None))
        return out

    def run(self, seed: int, g0: int, n_gens: int, target: int, adapt_count: int, stop_when: int,
            f_ext=None):
        best = np.zeros(n_gens, np.uint32)
        sm = np.zeros(n_gens, np.uint64)
        cnt = np.zeros(n_gens, np.uint32)
        done = ctypes.c_int64()
        _lib.check(_lib.lib().tv_ga_run(self._h, int(np.uint64(seed)), int(g0), int(n_gens), int(target),
                                        int(adapt_count), int(stop_when), _lib.ptr(f_ext), _lib.ptr(best),
                                        _lib.ptr(sm), _lib.ptr(cnt), ctypes.byref(done), None))
        k = done.value
        return k, best[:k], sm[:k], cnt[:k]

    def run_jatam(self, space: SearchSpace, target_occ: np.ndarray, seed: int, g0: int, n_gens: int, target: int,
                  d: int = 19, k: int = 8, fit_seed: int = 0, strict: bool = True, stream=None):
        """n_gens JaTAM-fitness generations without early stop in one call (tv_ga_run_jatam: the
        same generations as jatam_fitness + run(..., 1, ..., f_ext) repeated, enqueued without host
        round trips).  Returns (best, sum, count) per generation."""
        a, bpl, mp, mv, fp = space.kernel_args()
        occ = np.ascontiguousarray(np.asarray(target_occ, dtype=bool).reshape(d * d), np.uint8)
        best = np.zeros(n_gens, np.uint32)
        sm = np.zeros(n_gens, np.uint64)
        cnt = np.zeros(n_gens, np.uint32)
        P = _lib.ptr
        _lib.check(_lib.lib().tv_ga_run_jatam(self._h, a, bpl, P(mp), P(mv), mp.shape[0], P(fp), fp.shape[0], d, k,
                                              int(np.uint64(fit_seed)), int(bool(strict)), P(occ),
                                              int(np.uint64(seed)), int(g0), int(n_gens), int(target), P(best),
                                              P(sm), P(cnt), stream))
        return best, sm, cnt

    def jatam_fitness(self, space: SearchSpace, target_occ: np.ndarray, d: int = 19, k: int = 8, seed: int = 0,
                      strict: bool = True):
        """Device vector of JaTAM-shape fitness for the current population (enumeration indices)."""
        import torch
        if self._fit is None:
            self._fit = torch.empty(self.n, dtype=torch.int32, device="cuda")
        a, bpl, mp, mv, fp = space.kernel_args()
        occ = np.ascontiguousarray(np.asarray(target_occ, dtype=bool).reshape(d * d), np.uint8)
        _lib.check(_lib.lib().tv_ga_fitness_jatam(self._h, a, bpl, _lib.ptr(mp), _lib.ptr(mv), mp.shape[0],
                                                  _lib.ptr(fp), fp.shape[0], d, k, int(np.uint64(seed)),
                                                  int(bool(strict)), _lib.ptr(occ), _lib.ptr(self._fit), None))
        return self._fit


@dataclass
class JatamFitness:
    """GA fitness 'evolve toward a target shape' (SPEC:454 leaves it open):
    for a genome DETERMINISTIC at k, d^2 - shapediff(target, run-0 grid) with both
    grids seed-centred (App. B.2 shapesim scaled by d^2); otherwise 0."""

    space: SearchSpace
    target_occ: np.ndarray  # bool (d, d)
    d: int = 19
    k: int = 8
    seed: int = 0
    strict: bool = True


# Device GA handles kept between run_ga calls (population buffers, CDF, guide table: ~50 MB at
# 2^20), like a caching allocator: cudaMalloc / cudaFree of these buffers costs 2-40 ms per call.
_GA_POOL: "collections.OrderedDict" = None
_GA_POOL_MAX = 4


def _current_device() -> int:
    import torch
    return torch.cuda.current_device() if torch.cuda.is_available() else -1


def _ga_acquire(n: int, L: int, mu_L: float, mode) -> "DeviceGA":
    import collections
    global _GA_POOL
    if _GA_POOL is None:
        _GA_POOL = collections.OrderedDict()
    key = (_current_device(), int(n), int(L), float(mu_L), mode)
    ga = _GA_POOL.pop(key, None)
    if ga is None or not ga._h:
        return DeviceGA(n, L, mu_L, mode)
    ga.set_population(None)  # all-zero initial population, exactly as a fresh handle
    return ga


def _ga_release(ga: "DeviceGA", mu_L: float, mode) -> None:
    key = (ga.device, ga.n, ga.L, float(mu_L), mode)
    old = _GA_POOL.pop(key, None)
    if old is not None:
        old.close()
    _GA_POOL[key] = ga
    while len(_GA_POOL) > _GA_POOL_MAX:
        _GA_POOL.popitem(last=False)[1].close()


def run_ga(cfg: GAConfig, fitness="fujiyama", seed: int = 0, chunk: int = 4096) -> RunRecord:
    """Generation loop on the device: evaluate, record, stop when the
    configured target is met (or at the cutoff), reproduce with full replacement."""
    jatam = isinstance(fitness, JatamFitness)
    if not jatam and fitness != "fujiyama":
        raise ValueError("fitness must be 'fujiyama' or a JatamFitness")
    if jatam and fitness.space.free_bit_count != cfg.length:
        raise ValueError("GA genome length must equal the space's free bit count")
    ga = _ga_acquire(cfg.pop_size, cfg.length, cfg.mu_L, cfg.mode)
    ok = False
    try:
        if cfg.init is not None:
            ga.set_population(cfg.init)
        adapt_count = math.ceil(cfg.adapt_fraction * cfg.pop_size)
        stop = {"never": 0, "discovery": 1, "adaptation": 2}[cfg.stop_when]
        bests, sums, cnts = [], [], []
        g = 0
        if jatam and stop == 0:  # no stop rule: every generation in one enqueued call
            b, sm_, c = ga.run_jatam(fitness.space, fitness.target_occ, seed, 0, cfg.cutoff, cfg.target, fitness.d,
                                     fitness.k, fitness.seed, fitness.strict)
            bests.append(b); sums.append(sm_); cnts.append(c)
            g = cfg.cutoff
        while g < cfg.cutoff:
            if jatam:
                f = ga.jatam_fitness(fitness.space, fitness.target_occ, fitness.d, fitness.k, fitness.seed,
                                     fitness.strict)
                k, b, s, c = ga.run(seed, g, 1, cfg.target, adapt_count, stop, f_ext=f)
            else:
                k, b, s, c = ga.run(seed, g, min(chunk, cfg.cutoff - g), cfg.target, adapt_count, stop)
            bests.append(b); sums.append(s); cnts.append(c)
            g += k
            if stop and c.size and ((stop == 1 and c[-1] >= 1) or (stop == 2 and c[-1] >= adapt_count)):
                break
        ok = True
    finally:
        if ok:
            _ga_release(ga, cfg.mu_L, cfg.mode)
        else:
            ga.close()
    best = np.concatenate(bests) if bests else np.zeros(0, np.uint32)
    cnt = np.concatenate(cnts) if cnts else np.zeros(0, np.uint32)
    mean = (np.concatenate(sums).astype(np.float64) / cfg.pop_size) if sums else np.zeros(0)
    disc = np.nonzero(cnt >= 1)[0]
    adap = np.nonzero(cnt >= adapt_count)[0]
    return RunRecord(best, mean, cnt, int(best.size), int(disc[0]) if disc.size else None,
                     int(adap[0]) if adap.size else None, cfg, seed)


REPLICA_MAX_POP = 8192


def run_replicas(cfg: GAConfig, seeds) -> list[RunRecord]:
    """Independent Fujiyama runs, one per seed, in ONE device launch (tv_ga_replicas: a
    CTA per run, population in shared memory, block barriers only).  Record r is
    identical to ``run_ga(cfg, seed=seeds[r])``.  Needs cfg.pop_size <= 8192."""
    seeds = np.ascontiguousarray([int(x) for x in seeds], np.uint64)
    R, n, L = seeds.shape[0], int(cfg.pop_size), int(cfg.length)
    if R == 0:
        return []
    if L > 64:  # replica kernel holds one u64 per genome: wide runs go one launch sequence each
        return [run_ga(cfg, seed=int(x)) for x in seeds]
    if n > REPLICA_MAX_POP:
        raise ValueError(f"replica runs hold the population in shared memory: pop_size <= {REPLICA_MAX_POP}")
    T = poisson_thresholds(cfg.mu_L, L)
    adapt_count = math.ceil(cfg.adapt_fraction * n)
    stop = {"never": 0, "discovery": 1, "adaptation": 2}[cfg.stop_when]
    n_gens = int(cfg.cutoff)
    init = None
    if cfg.init is not None:
        init = np.ascontiguousarray(np.broadcast_to(np.asarray(cfg.init, np.uint64), (R, n)))
    done, disc, adap = (np.zeros(R, np.int64) for _ in range(3))
    best = np.zeros((R, n_gens), np.uint32)
    sm = np.zeros((R, n_gens), np.uint64)
    cnt = np.zeros((R, n_gens), np.uint32)
    P = _lib.ptr
    _lib.check(_lib.lib().tv_ga_replicas(n, L, MODES[cfg.mode], P(T), R, P(seeds), P(init), 0, n_gens, int(cfg.target),
                                         adapt_count, stop, P(done), P(disc), P(adap), P(best), P(sm), P(cnt), None,
                                         None))
    out = []
    for r in range(R):
        k = int(done[r])
        out.append(RunRecord(best[r, :k].copy(), sm[r, :k].astype(np.float64) / n, cnt[r, :k].copy(), k,
                             int(disc[r]) if disc[r] >= 0 else None, int(adap[r]) if adap[r] >= 0 else None,
                             cfg, int(seeds[r])))
    return out


def censored_median_ci(vals, cutoff: int, sample_size: int = 100, resamples: int = 10000, rng=None) -> dict:
    """Median + bootstrap CI of per-run times with cutoff censoring.

    ``vals`` holds one entry per run, None = censored at the cutoff.  When at most
    half the runs are censored they stay in the sample as ">= cutoff" (value
    ``cutoff``, which keeps their rank: every uncensored time is < cutoff), in the
    median and in every bootstrap resample; a median or CI bound that lands on a
    censored value is itself only a lower bound, flagged ``*_censored``.  When more
    than half are censored the median is reported as censored (None)."""
    n = len(vals)
    cens = sum(v is None for v in vals)
    if n == 0:
        raise ValueError("vals must be non-empty")
    if cens * 2 > n:
        return dict(median=None, ci_lo=None, ci_hi=None, censored=cens, median_censored=True,
                    ci_lo_censored=True, ci_hi_censored=True)
    x = [float(cutoff) if v is None else float(v) for v in vals]
    med, lo, hi = bootstrap_median_ci(x, sample_size, resamples, rng)
    return dict(median=med, ci_lo=lo, ci_hi=hi, censored=cens, median_censored=bool(cens and med >= cutoff),
                ci_lo_censored=bool(cens and lo >= cutoff), ci_hi_censored=bool(cens and hi >= cutoff))


def sweep_runs(cfg: GAConfig, seeds) -> list[RunRecord]:
    """The runs of one sweep point: one replica launch when the population fits shared
    memory, else one run_ga per seed."""
    seeds = [int(x) for x in seeds]
    return run_replicas(cfg, seeds) if cfg.pop_size <= REPLICA_MAX_POP else [run_ga(cfg, seed=x) for x in seeds]


def sweep_row(mu: float, cfg: GAConfig, discovery: list, adaptation: list, sample_size: int = 100,
              resamples: int = 10000) -> dict:
    """One SPEC:452 sweep row from the per-run times (run order = seed order)."""
    return {"muL": float(mu), "runs": len(discovery),
            "discovery": censored_median_ci(discovery, cfg.cutoff, sample_size, resamples),
            "adaptation": censored_median_ci(adaptation, cfg.cutoff, sample_size, resamples)}


def sweep(mu_L_grid, runs: int = 100, base: GAConfig | None = None, seed0: int = 0, sample_size: int = 100,
          resamples: int = 10000, out: str | None = None, runner=sweep_runs) -> list[dict]:
    """SPEC:452 sweep rows: {muL, runs, discovery:{median, ci_lo, ci_hi, censored}, adaptation:{...}}.

    Run r of every point uses seed seed0 + r.  Censoring follows SPEC:448
    (``censored_median_ci``).  With ``out`` the rows are written as the sweep JSON
    artefact, together with the configuration.  ``distributed.sweep_distributed``
    deals the runs over GPUs and returns the same rows."""
    base = base or GAConfig()
    rows = []
    for mu in mu_L_grid:
        cfg = GAConfig(**{**base.__dict__, "mu_L": float(mu)})
        recs = runner(cfg, [seed0 + r for r in range(runs)])
        rows.append(sweep_row(mu, cfg, [r.discovery for r in recs], [r.adaptation for r in recs], sample_size,
                              resamples))
    if out is not None:
        write_sweep_json(out, rows, base, seed0=seed0, sample_size=sample_size, resamples=resamples)
    return rows


def write_sweep_json(path: str, rows: list[dict], cfg: GAConfig, **extra) -> None:
    """Sweep JSON artefact: the per-muL rows plus the run configuration."""
    import json
    conf = {k: v for k, v in cfg.__dict__.items() if k not in ("init", "mu_L")}
    conf["init"] = "all-zero" if cfg.init is None else "explicit"
    with open(path, "w") as f:
        json.dump({"config": conf, **extra, "points": rows}, f, indent=1)
        f.write("\n")


def write_trace_csv(record: RunRecord, path_or_buf=None) -> str:
    """Optional per-run CSV trace: ``generation,best,mean,count_at_target``."""
    import io
    buf = io.StringIO()
    buf.write("generation,best,mean,count_at_target\n")
    for g in range(record.generations):
        buf.write(f"{g},{int(record.best[g])},{float(record.mean[g])!r},{int(record.count_at_target[g])}\n")
    text = buf.getvalue()
    if path_or_buf is not None:
        if hasattr(path_or_buf, "write"):
            path_or_buf.write(text)
        else:
            with open(path_or_buf, "w") as f:
                f.write(text)
    return text


def bernoulli_threshold(mu_L: float, L: int) -> int:
    """64-bit threshold of bit-by-bit mutation: a bit flips when its draw < floor(p * 2^64), p = mu_L / L."""
    p = min(1.0, max(0.0, mu_L / L))
    return min((1 << 64) - 1, int(math.floor(p * 2.0 ** 64)))


def mutate_population(pop, L: int, mu_L: float, method: str = "distribution", seed: int = 0, g: int = 0,
                      count_flips: bool = False, stream=None, T=None):
    """Mutate a device population in place (tv_ga_mutate).  ``pop`` is a CUDA tensor of
    ``W * n`` u64 words, word-major (word w of genome i at ``w * n + i``); method
    "distribution" = the GA's operator (k ~ Poisson(mu_L) distinct flips), "bitwise" = one
    draw per bit (SPEC ACCEPTANCE 8's baseline).  ``T``: precomputed thresholds (host array
    or CUDA tensor), else computed here.  Returns the flip count if asked."""
    W = (L + 63) // 64
    n = pop.numel() // W
    if T is None:
        T = poisson_thresholds(mu_L, L)
    flips = np.zeros(1, np.uint64) if count_flips else None
    m = {"distribution": 0, "bitwise": 1}[method]
    _lib.check(_lib.lib().tv_ga_mutate(_lib.ptr(pop), n, L, _lib.ptr(T), bernoulli_threshold(mu_L, L), m,
                                       int(np.uint64(seed)), int(g), _lib.ptr(flips), stream))
    return int(flips[0]) if count_flips else None


def mutation_benchmark(pop_size: int = 1 << 20, length: int = 1024, mu_L: float = 0.5, reps: int = 5,
                       seed: int = 0) -> dict:
    """SPEC ACCEPTANCE 8 (Fig. 5's regime): device time per generation of mutating a
    population of ``length``-bit genomes by distribution (the GA operator) vs bit by bit,
    CUDA events on the launch stream, best of ``reps``."""
    import torch
    W = (length + 63) // 64
    pop = torch.zeros(W * pop_size, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream()
    sp = ctypes.c_void_p(st.cuda_stream)
    Td = torch.from_numpy(poisson_thresholds(mu_L, length).view(np.int64)).cuda()  # no host work in the timed region
    out = {}
    gens = 20  # launches per timed region (back to back, one generation each)
    for method in ("distribution", "bitwise"):
        mutate_population(pop, length, mu_L, method, seed, 0, stream=sp, T=Td)  # warm-up
        best = float("inf")
        for r in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(st)
            for j in range(gens):
                mutate_population(pop, length, mu_L, method, seed, 1 + r * gens + j, stream=sp, T=Td)
            e1.record(st)
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) / gens)
        out[method + "_ms"] = best
        out[method + "_flips_per_genome"] = mutate_population(pop, length, mu_L, method, seed, 99,
                                                              count_flips=True, stream=sp, T=Td) / pop_size
    out["speedup"] = out["bitwise_ms"] / out["distribution_ms"]
    out.update(pop_size=pop_size, length=length, mu_L=mu_L)
    return out
