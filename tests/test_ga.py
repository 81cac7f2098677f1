"""GA (SPEC.md evolve module).  No reference implementation exists, so:
 * the device loop must equal the CPU restatement (oracle/tv_ga_oracle.c) bit
   for bit (gpu tests), and the host single-genome operators must equal the
   restatement's child procedure (cpu tests);
 * the operators must meet SPEC.md's statistical acceptance (ACCEPTANCE 4-5).
"""
import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_2205_15311_b200 import evolve as E
from paper_2205_15311_b200.genome import Genome


def test_stream_matches_restatement():
    for seed, g, i in [(0, 0, 0), (7, 3, 11), (2**63 + 5, 19999, 2**20 - 1)]:
        r = E.GaRng(seed, g, i)
        assert [r.next() for _ in range(8)] == [int(x) for x in O.ga_draws(seed, g, i, 8)]


def _py_child(seed, g, i, pop, L, mode, T):
    """One child composed from the host operators (same draw order as the kernel)."""
    r = E.GaRng(seed, g, i)
    w = np.array([bin(int(v)).count("1") for v in pop], np.int64)
    a = int(pop[E.roulette_select(w, r)])
    child = a
    if mode:
        b = int(pop[E.roulette_select(w, r)])
        child = E.crossover_single_point(a, b, r, L) if mode == 1 else E.crossover_uniform(a, b, r, L)
    u = r.next() >> 1
    k = int(np.count_nonzero(u >= T))
    chosen = 0
    while bin(chosen).count("1") < k:
        chosen |= 1 << (L - 1 - r.below(L))
    return child ^ chosen


@pytest.mark.parametrize("mode,lam,L", [(0, 0.3, 32), (1, 1.0, 24), (2, 4.0, 64), (1, 0.0, 16)])
def test_host_operators_equal_restatement(mode, lam, L):
    rng = np.random.default_rng(mode * 10 + L)
    full = (1 << L) - 1
    pop = np.array([int(x) & full for x in rng.integers(0, 2**63, 37, dtype=np.uint64)], np.uint64)
    pop[::5] = 0
    cdf = np.cumsum([bin(int(v)).count("1") for v in pop]).astype(np.uint64)
    T = E.poisson_thresholds(lam, L)
    for i in range(40):
        assert _py_child(9, 4, i, pop, L, mode, T) == O.ga_child(9, 4, i, pop, cdf, L, mode, T)


def test_zero_fitness_falls_back_to_uniform():
    pop = np.zeros(8, np.uint64)
    cdf = np.zeros(8, np.uint64)
    T = E.poisson_thresholds(0.0, 32)
    assert all(O.ga_child(1, 0, i, pop, cdf, 32, 0, T) == 0 for i in range(50))


def test_mutation_properties():
    T0 = E.poisson_thresholds(0.0, 32)
    assert not T0.any() or (T0 == 1 << 63).all()
    g = Genome.from_int(32, 0xDEADBEEF)
    for i in range(200):
        assert E.mutate(g, 0.0, E.GaRng(1, 0, i)) == g
    for i in range(2000):
        r = E.GaRng(2, 0, i)
        r2 = E.GaRng(2, 0, i)
        k = E.poisson_sample(2.5, r2, 32)
        m = E.mutate(0, 2.5, r, 32)
        assert bin(m).count("1") == k                                           # distinct flips


@pytest.mark.parametrize("lam", [0.1, 0.5, 1.0])
def test_flip_count_distribution_chi2(lam):
    """SPEC ACCEPTANCE 5: chi^2 against Eq. 1 truncated at L, p > 0.001, 10^6 draws."""
    from scipy import stats
    L = 32
    ks = O.ga_flip_counts(12345, 10**6, L, E.poisson_thresholds(lam, L))
    kmax = 1
    while stats.poisson.sf(kmax, lam) * 1e6 > 5:
        kmax += 1
    obs = np.array([np.count_nonzero(ks == j) for j in range(kmax)] + [np.count_nonzero(ks >= kmax)], float)
    p = np.array([stats.poisson.pmf(j, lam) for j in range(kmax)] + [stats.poisson.sf(kmax - 1, lam)])
    assert stats.chisquare(obs, p * obs.sum()).pvalue > 0.001
    assert abs(ks.mean() - lam) < 5 * math.sqrt(lam / 1e6)


def test_roulette_known_answers():
    assert E.roulette_select([2.0, 3.0, 4.0, 1.0], cutoff=10) == 3             # App. C.1
    assert all(E.roulette_select([1, 0, 0], E.GaRng(0, 0, i)) == 0 for i in range(200))


def test_selection_frequencies_3sigma():
    """10^6 children of one asexual, lambda = 0 generation: parent frequencies ~ f_i / sum f (SPEC ACCEPTANCE 5)."""
    n = 1 << 20
    pat = np.array([0b1, 0b11, 0b111, 0b1111], np.uint64)                      # fitness 1, 2, 3, 4
    pop = np.tile(pat, n // 4)
    O.ga_run(pop, 32, 0, E.poisson_thresholds(0.0, 32), 5, 0, 1, 32, 1 << 30, 0)
    cnt = np.array([np.count_nonzero(pop == v) for v in pat], float)
    p = np.array([1, 2, 3, 4]) / 10.0
    assert np.all(np.abs(cnt - n * p) <= 3 * np.sqrt(n * p * (1 - p)))


def test_uniform_crossover_and_single_point_properties():
    L = 32
    full = (1 << L) - 1
    hw = []
    for i in range(20000):
        r = E.GaRng(3, 0, i)
        c = E.crossover_uniform(0, full, r, L)
        hw.append(bin(c).count("1"))
    hw = np.array(hw)
    assert abs(hw.mean() - L / 2) < 3 * math.sqrt(L / 4 / len(hw)) * 3
    for i in range(2000):
        a, b = 0x0F0F0F0F, 0xF0F0F0F0
        c = E.crossover_single_point(a, b, E.GaRng(4, 0, i), L)
        assert all(((c >> j) & 1) in (((a >> j) & 1), ((b >> j) & 1)) for j in range(L))
    # p = 0 -> child == b: find a stream whose first draw gives p = 0
    for i in range(10**5):
        r = E.GaRng(5, 0, i)
        if E.GaRng(5, 0, i).below(L) == 0:
            assert E.crossover_single_point(a, b, r, L) == b
            break


def test_bootstrap_examples():
    assert E.bootstrap_median_ci([5, 5, 5], 3, 100) == (5.0, 5.0, 5.0)
    med, lo, hi = E.bootstrap_median_ci(np.arange(1, 101), 100, 2000)
    assert med == 50.5 and lo < 50.5 < hi and hi - lo < 25
    with pytest.raises(ValueError):
        E.bootstrap_median_ci([], 10, 10)


def test_censored_median_rule_spec_448():
    """censored runs stay in the median / bootstrap (as >= cutoff) unless > 50 % are censored."""
    vals = [10, 20, 30, None, None]  # 40 % censored: they rank above every uncensored time
    r = E.censored_median_ci(vals, 100, 5, 200)
    assert r["median"] == 30.0 and r["censored"] == 2 and not r["median_censored"]
    assert r["ci_hi"] == 100.0 and r["ci_hi_censored"]
    # dropping the censored runs would have given 20 (the round-1 behaviour, biased low)
    assert np.median([v for v in vals if v is not None]) == 20
    r = E.censored_median_ci([5, None, None, 7, None, None], 100, 6, 200)
    assert r["median"] is None and r["median_censored"] and r["censored"] == 4
    r = E.censored_median_ci([1, None], 50, 2, 200)  # exactly half: kept, median straddles the cutoff
    assert r["median"] == 25.5 and not r["median_censored"]
    r = E.censored_median_ci([None, None, 3, None, 4, 5, None], 9, 7, 200)  # 4/7 > 50 %
    assert r["median"] is None
    r = E.censored_median_ci([None, 2, None, None, 4, 5], 9, 6, 200)  # 3/6: median (5 + 9) / 2, not censored
    assert r["median"] == 7.0
    r = E.censored_median_ci([None, None, 3, None], 9, 4, 200)  # 3/4 censored
    assert r["median"] is None
    with pytest.raises(ValueError):
        E.censored_median_ci([], 10)


def test_sweep_json_and_trace_csv(tmp_path):
    import json
    rows = [{"muL": 0.3, "runs": 2, "discovery": E.censored_median_ci([3, 4], 10, 2, 10),
             "adaptation": E.censored_median_ci([None, 8], 10, 2, 10)}]
    p = tmp_path / "sweep.json"
    E.write_sweep_json(str(p), rows, E.GAConfig(), seed0=0)
    doc = json.loads(p.read_text())
    assert doc["points"][0]["muL"] == 0.3 and doc["config"]["pop_size"] == 512 and doc["config"]["init"] == "all-zero"
    assert set(doc["points"][0]["discovery"]) >= {"median", "ci_lo", "ci_hi", "censored"}
    rec = E.RunRecord(np.array([3, 5], np.uint32), np.array([0.5, 1.25]), np.array([0, 2], np.uint32), 2, 1, None)
    txt = E.write_trace_csv(rec)
    assert txt.splitlines() == ["generation,best,mean,count_at_target", "0,3,0.5,0", "1,5,1.25,2"]


# ---------------------------------------------------------------- device (gpu)
@pytest.mark.gpu
@pytest.mark.parametrize("n,L,mode,lam,stop", [(512, 32, 0, 0.3, 0), (4096 + 3, 32, 1, 1.0, 0), (1 << 16, 64, 2, 4.0, 0),
                                                 (1000, 24, 0, 0.03, 2), (1 << 20, 32, 0, 0.3, 0)])
def test_device_ga_equals_restatement(n, L, mode, lam, stop):
    ga = E.DeviceGA(n, L, lam, mode)
    init = np.random.default_rng(n).integers(0, 2**63, n, dtype=np.uint64) & np.uint64((1 << L) - 1 if L < 64 else 2**64 - 1)
    init[: n // 2] = 0
    ga.set_population(init)
    pop = init.copy()
    T = E.poisson_thresholds(lam, L)
    gens = 40 if n >= 1 << 20 else 300
    tgt, adapt = 25, n // 2
    g = 0
    while g < gens:  # several launches continue the same trajectory
        k, b, s, c = ga.run(11, g, min(97, gens - g), tgt, adapt, stop)
        k2, b2, s2, c2 = O.ga_run(pop, L, mode, T, 11, g, min(97, gens - g), tgt, adapt, stop)
        assert k == k2
        assert np.array_equal(b, b2) and np.array_equal(s, s2) and np.array_equal(c, c2)
        assert np.array_equal(ga.population(), pop), g
        g += k
        if stop and k < min(97, gens - g + k):
            break
    ga.close()


@pytest.mark.gpu
@pytest.mark.parametrize("stg,pair", [("0", "1"), ("1", "0"), ("0", "0")])
@pytest.mark.parametrize("n,L,mode,lam,stop", [(4096 + 3, 32, 1, 1.0, 0), (1000, 24, 2, 0.3, 1), (1 << 17, 30, 0, 0.3, 2)])
def test_device_ga_layout_switches(monkeypatch, stg, pair, n, L, mode, lam, stop):
    """k_ga_run's staged chunk (shared memory between the phases) and paired guide entries are
    layout choices: with either off (TV_GA_STG / TV_GA_PAIR, read at create) the run is the
    same restatement, bit for bit (the default run has both on: test above)."""
    monkeypatch.setenv("TV_GA_STG", stg)
    monkeypatch.setenv("TV_GA_PAIR", pair)
    test_device_ga_equals_restatement(n, L, mode, lam, stop)


@pytest.mark.gpu
@pytest.mark.parametrize("stg", ["1", "0"])
def test_device_ga_zero_generations_and_immediate_stop(monkeypatch, stg):
    """Edge cases of the staged loop: a call with no generations is refused, and a run that stops
    at its first evaluation (target 0 is met at once) leaves the population as it was; the next
    call continues exactly like the restatement."""
    monkeypatch.setenv("TV_GA_STG", stg)
    n, L, lam = 5000, 28, 0.7
    init = np.random.default_rng(2).integers(0, 1 << L, n, dtype=np.uint64)
    ga = E.DeviceGA(n, L, lam, "uniform")
    ga.set_population(init)
    with pytest.raises(ValueError):  # n_gens >= 1 (the reference loop evaluates at least once)
        ga.run(4, 0, 0, 10, n, 0)
    assert np.array_equal(ga.population(), init)
    k, b, s, c = ga.run(4, 0, 50, 0, n, 1)  # count(f >= 0) = n >= 1: stop after recording generation 0
    pop = init.copy()
    k2, b2, s2, c2 = O.ga_run(pop, L, 2, E.poisson_thresholds(lam, L), 4, 0, 50, 0, n, 1)
    assert k == k2 == 1 and np.array_equal(b, b2) and np.array_equal(c, c2)
    assert np.array_equal(ga.population(), init) and np.array_equal(pop, init)
    k, b, s, c = ga.run(4, 0, 7, 30, n, 0)
    k2, b2, s2, c2 = O.ga_run(pop, L, 2, E.poisson_thresholds(lam, L), 4, 0, 7, 30, n, 0)
    assert k == k2 == 7 and np.array_equal(s, s2) and np.array_equal(ga.population(), pop)
    ga.close()


@pytest.mark.gpu
def test_fujiyama_regime_desk_scale():
    """SPEC ACCEPTANCE 4 (runs=25, pop=512, L=32, cutoff=20000)."""
    med = []
    for mu in (0.03, 0.1, 0.3):  # 25 runs per point in one replica launch (== run_ga per seed)
        d = [r.discovery for r in E.run_replicas(E.GAConfig(mu_L=mu, stop_when="discovery"), range(25))]
        d = [x if x is not None else 20000 for x in d]
        med.append(np.median(d))
    assert med[0] > med[1] > med[2], med
    ok03 = sum(r.adaptation is not None for r in E.run_replicas(E.GAConfig(mu_L=0.3), range(100, 125)))
    cens4 = sum(r.adaptation is None for r in E.run_replicas(E.GAConfig(mu_L=4.0), range(200, 225)))
    assert ok03 >= 20 and cens4 >= 20, (ok03, cens4)
    rows = E.sweep([0.1, 0.3], runs=25)  # SPEC:452 sweep rows through the device sweep
    assert [r["muL"] for r in rows] == [0.1, 0.3] and rows[1]["adaptation"]["median"] is not None


@pytest.mark.gpu
def test_spec_run_ga_examples_100_runs(tmp_path):
    """SPEC:413 (N=512, L=32, muL=0.3: discovery before the cutoff in >= 95/100 runs) and
    SPEC:414 (muL=8: adaptation cutoff-censored in >= 95/100 runs), through the sweep API."""
    import json
    out = tmp_path / "sweep.json"
    rows = E.sweep([0.3, 8.0], runs=100, base=E.GAConfig(stop_when="adaptation"), out=str(out))
    assert rows[0]["discovery"]["censored"] <= 5, rows[0]
    assert rows[1]["adaptation"]["censored"] >= 95, rows[1]
    assert rows[1]["adaptation"]["median"] is None  # > 50 % censored: the median is reported censored
    assert json.loads(out.read_text())["points"] == json.loads(json.dumps(rows))
    disc = [r.discovery for r in E.run_replicas(E.GAConfig(mu_L=0.3, stop_when="discovery"), range(100))]
    assert sum(x is not None for x in disc) >= 95


@pytest.mark.gpu
def test_spec_discovery_le_adaptation_1000_runs():
    """discovery <= adaptation on every uncensored run, over 1000 runs (4 regimes x 250)."""
    n_unc = 0
    for i, mu in enumerate((0.1, 0.3, 1.0, 4.0)):
        for r in E.run_replicas(E.GAConfig(mu_L=mu), range(1000 * i, 1000 * i + 250)):
            assert E.discovery_time(r) == r.discovery and E.adaptation_time(r) == r.adaptation
            if r.adaptation is not None:
                assert r.discovery is not None and r.discovery <= r.adaptation
                n_unc += 1
    assert n_unc >= 250, n_unc


@pytest.mark.gpu
@pytest.mark.parametrize("d", [19, 17])
def test_jatam_fitness_matches_cpu(d):
    """Device JaTAM-shape fitness == d^2 - shapediff(target, run-0 grid) for DET genomes (oracle);
    d = 19 runs the compile-time-geometry fitness kernel, d = 17 the run-time one."""
    from paper_2205_15311_b200._kernels import edges_from_labels
    from paper_2205_15311_b200.genome import SearchSpace, decode_tileset, genome_at_index
    S28 = SearchSpace(2, 8)
    k = 8
    # target: the run-0 grid of a 12-cell deterministic genome
    tgt_idx = 0x801772
    ts = decode_tileset(genome_at_index(S28, tgt_idx), S28)
    e = edges_from_labels(np.array([v for t in ts.tiles for v in t], np.uint8), 2)
    grid = np.empty(d * d, np.int16)
    O.assemble_single(e, 2, d, 0, tgt_idx, 0, True, grid)
    target = (grid >= 0).reshape(d, d)
    n = 4096
    pop = np.random.default_rng(3).integers(0, 1 << 24, n, dtype=np.uint64)
    ga = E.DeviceGA(n, 24, 0.3)
    ga.set_population(pop)
    f = ga.jatam_fitness(S28, target, d, k).cpu().numpy().view(np.uint32)
    for i in range(n):
        idx = int(pop[i])
        ts = decode_tileset(genome_at_index(S28, idx), S28)
        e = edges_from_labels(np.array([v for t in ts.tiles for v in t], np.uint8), 2)
        sw = np.zeros(6, np.uint64)
        st, cls, *_ = O.classify_single(e, 2, d, k, 0, idx, True, sw)
        exp = 0
        if st == 0 and cls == 0:
            O.assemble_single(e, 2, d, 0, idx, 0, True, grid)
            exp = d * d - int(np.count_nonzero((grid >= 0).reshape(d, d) != target))
        assert int(f[i]) == exp, (i, idx)
    ga.close()


@pytest.mark.gpu
@pytest.mark.parametrize("n", [100, 1000 + 7, 148 * 32 + 5])
def test_device_ga_target_zero_counts_every_individual(n):
    """count_at_target with target 0 is the population size: padding lanes of partial rows and
    empty CTAs (population not a multiple of 32 per CTA) must not be counted."""
    L, lam = 24, 0.5
    ga = E.DeviceGA(n, L, lam, "asexual")
    ga.set_population(np.zeros(n, np.uint64))
    k, b, s, c = ga.run(5, 0, 12, 0, n + 1, 0)
    pop = np.zeros(n, np.uint64)
    k2, b2, s2, c2 = O.ga_run(pop, L, 0, E.poisson_thresholds(lam, L), 5, 0, 12, 0, n + 1, 0)
    assert k == k2 == 12 and np.all(np.asarray(c) == n)
    assert np.array_equal(b, b2) and np.array_equal(s, s2) and np.array_equal(c, c2)
    assert np.array_equal(ga.population(), pop)
    ga.close()


@pytest.mark.gpu
@pytest.mark.parametrize("n,L,mode,mu,stop", [(512, 32, "asexual", 0.3, "adaptation"), (777, 24, "single_point", 1.0, "never"),
                                               (4096, 64, "uniform", 0.1, "discovery"), (512, 32, "asexual", 4.0, "adaptation")])
def test_replicas_equal_single_runs(n, L, mode, mu, stop):
    """One replica launch == independent run_ga calls, record by record (trajectories, stop points)."""
    cfg = E.GAConfig(pop_size=n, length=L, mu_L=mu, mode=mode, cutoff=600, target=min(25, L - 2), stop_when=stop)
    seeds = [3, 17, 2205, 1 << 40]
    reps = E.run_replicas(cfg, seeds)
    for s, r in zip(seeds, reps):
        x = E.run_ga(cfg, seed=s)
        assert (r.generations, r.discovery, r.adaptation) == (x.generations, x.discovery, x.adaptation), s
        assert np.array_equal(r.best, x.best) and np.array_equal(r.count_at_target, x.count_at_target)
        assert np.allclose(r.mean, x.mean)


@pytest.mark.gpu
def test_replicas_final_population_and_init():
    """Final populations and a non-zero initial population through the C ABI directly."""
    from paper_2205_15311_b200 import _lib
    n, L, R, gens = 300, 32, 5, 77
    T = E.poisson_thresholds(0.5, L)
    init = np.random.default_rng(1).integers(0, 1 << 32, (R, n), dtype=np.uint64)
    seeds = np.arange(R, dtype=np.uint64) + 9
    done, disc, adap = (np.zeros(R, np.int64) for _ in range(3))
    fin = np.zeros((R, n), np.uint64)
    P = _lib.ptr
    _lib.check(_lib.lib().tv_ga_replicas(n, L, 2, P(T), R, P(seeds), P(init), 5, gens, 30, n // 2, 0, P(done),
                                         P(disc), P(adap), None, None, None, P(fin), None))
    for r in range(R):
        pop = init[r].copy()
        k, *_ = O.ga_run(pop, L, 2, T, int(seeds[r]), 5, gens, 30, n // 2, 0)
        assert k == done[r] == gens
        assert np.array_equal(fin[r], pop), r


@pytest.mark.gpu
@pytest.mark.parametrize("mode", [0, 1])
def test_jatam_generations_external_fitness_vs_restatement(mode):
    """The JaTAM GA loop: device fitness (checked against the oracle above) feeds one external-
    fitness generation at a time; each child equals the CPU restatement's child drawn from the
    same integer CDF (oracle ga_child), stats included, for several generations."""
    from paper_2205_15311_b200._kernels import edges_from_labels
    from paper_2205_15311_b200.genome import SearchSpace, decode_tileset, genome_at_index
    S28 = SearchSpace(2, 8)
    d, k, n, L, lam = 19, 8, 1000, 24, 0.5
    tgt_idx = 0x801772
    ts = decode_tileset(genome_at_index(S28, tgt_idx), S28)
    e = edges_from_labels(np.array([v for t in ts.tiles for v in t], np.uint8), 2)
    grid = np.empty(d * d, np.int16)
    O.assemble_single(e, 2, d, 0, tgt_idx, 0, True, grid)
    target = (grid >= 0).reshape(d, d)
    pop = np.random.default_rng(5).integers(0, 1 << 24, n, dtype=np.uint64)
    pop[:10] = tgt_idx  # some fit individuals
    ga = E.DeviceGA(n, L, lam, mode)
    ga.set_population(pop)
    T = E.poisson_thresholds(lam, L)
    for g in range(4):
        f = ga.jatam_fitness(S28, target, d, k)
        fh = f.cpu().numpy().view(np.uint32).astype(np.uint64)
        cdf = np.cumsum(fh).astype(np.uint64)
        kk, b, s, c = ga.run(21, g, 1, 300, n, 0, f_ext=f)
        assert kk == 1 and int(b[0]) == int(fh.max()) and int(s[0]) == int(fh.sum())
        assert int(c[0]) == int(np.count_nonzero(fh >= 300))
        exp = np.array([O.ga_child(21, g, i, pop, cdf, L, mode, T) for i in range(n)], np.uint64)
        pop = ga.population()
        assert np.array_equal(pop, exp), g
    ga.close()


@pytest.mark.gpu
def test_jatam_s38_fitness_and_generations():
    """SURVEY 8(d) config 4 with genomes in S_{3,8} (L = 36: the unpacked GA path, a = 3 fitness
    kernel): device fitness == the oracle's d^2 - shapediff for DET genomes, and external-
    fitness generations == the restatement's children."""
    from paper_2205_15311_b200._kernels import edges_from_labels
    from paper_2205_15311_b200.genome import SearchSpace, decode_tileset, genome_at_index
    S38 = SearchSpace(3, 8)
    d, k, n, L, lam = 19, 8, 2048, 36, 0.5
    rng = np.random.default_rng(38)
    grid = np.empty(d * d, np.int16)

    def edges(idx):
        ts = decode_tileset(genome_at_index(S38, idx), S38)
        return edges_from_labels(np.array([v for t in ts.tiles for v in t], np.uint8), 3)

    def det_cells(idx):
        sw = np.zeros(6, np.uint64)
        st, cls, *_ = O.classify_single(edges(idx), 3, d, k, 0, idx, True, sw)
        if st != 0 or cls != 0:
            return None
        O.assemble_single(edges(idx), 3, d, 0, idx, 0, True, grid)
        return (grid >= 0).reshape(d, d).copy()

    tgt_idx, target = None, None
    for idx in rng.integers(0, 1 << 36, 20000, dtype=np.uint64):  # a DET target with a few cells
        occ = det_cells(int(idx))
        if occ is not None and occ.sum() >= 4:
            tgt_idx, target = int(idx), occ
            break
    assert target is not None
    pop = rng.integers(0, 1 << 36, n, dtype=np.uint64)
    pop[:16] = tgt_idx
    ga = E.DeviceGA(n, L, lam, "asexual")
    ga.set_population(pop)
    f = ga.jatam_fitness(S38, target, d, k).cpu().numpy().view(np.uint32)
    for i in range(n):
        occ = det_cells(int(pop[i]))
        exp = 0 if occ is None else d * d - int(np.count_nonzero(occ != target))
        assert int(f[i]) == exp, (i, int(pop[i]))
    assert int(f[0]) == d * d
    T = E.poisson_thresholds(lam, L)
    for g in range(3):
        f = ga.jatam_fitness(S38, target, d, k)
        fh = f.cpu().numpy().view(np.uint32).astype(np.uint64)
        cdf = np.cumsum(fh).astype(np.uint64)
        kk, b, s, c = ga.run(7, g, 1, 300, n, 0, f_ext=f)
        assert kk == 1 and int(b[0]) == int(fh.max()) and int(s[0]) == int(fh.sum())
        exp = np.array([O.ga_child(7, g, i, pop, cdf, L, 0, T) for i in range(n)], np.uint64)
        pop = ga.population()
        assert np.array_equal(pop, exp), g
    ga.close()


# ---------------------------------------------------------------- wide genomes (L > 64)
def _wide_random(rng, n, L):
    W = (L + 63) // 64
    pop = rng.integers(0, 2**63, (n, W), dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, (n, W), dtype=np.uint64)
    if L % 64:
        pop[:, W - 1] &= np.uint64((1 << (L % 64)) - 1)
    return np.ascontiguousarray(pop)


@pytest.mark.parametrize("L,mode", [(20, 0), (32, 1), (64, 2), (47, 2), (64, 1)])
def test_wide_restatement_equals_narrow_at_one_word(L, mode):
    """orc_ga_run_w with W = 1 is the narrow restatement (same draws, same children, same stats)."""
    rng = np.random.default_rng(L + mode)
    pop = _wide_random(rng, 300, L)[:, 0].copy()
    pop[::3] = 0
    wide = pop[:, None].copy()
    T = E.poisson_thresholds(1.5, L)
    a = O.ga_run(pop, L, mode, T, 5, 0, 30, L // 2, 150, 0)
    b = O.ga_run_w(wide, L, mode, T, 5, 0, 30, L // 2, 150, 0)
    assert a[0] == b[0] and all(np.array_equal(x, y) for x, y in zip(a[1:], b[1:]))
    assert np.array_equal(pop, wide[:, 0])


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_wide_host_operators_equal_restatement(mode):
    """The host single-genome operators on Python ints (any L) compose the wide child."""
    L, W = 150, 3
    rng = np.random.default_rng(mode)
    pop = _wide_random(rng, 29, L)
    pop[::4] = 0
    ints = [sum(int(pop[i, w]) << (64 * w) for w in range(W)) for i in range(pop.shape[0])]
    cdf = np.cumsum([bin(v).count("1") for v in ints]).astype(np.uint64)
    T = E.poisson_thresholds(2.0, L)
    for i in range(30):
        r = E.GaRng(3, 7, i)
        wts = np.array([bin(v).count("1") for v in ints], np.int64)
        child = ints[E.roulette_select(wts, r)]
        if mode:
            b = ints[E.roulette_select(wts, r)]
            child = E.crossover_single_point(child, b, r, L) if mode == 1 else E.crossover_uniform(child, b, r, L)
        child = E.mutate(child, 2.0, r, L)
        got = O.ga_child_w(3, 7, i, pop, cdf, L, mode, T)
        assert child == sum(int(got[w]) << (64 * w) for w in range(W)), i


def test_mutation_benchmark_operators_restatement():
    """ACCEPTANCE 8 operators on the CPU: the distribution method flips Poisson(muL) distinct bits,
    bit by bit flips Binomial(L, muL / L); both have mean muL."""
    L, n, mu = 1024, 20000, 0.5
    T = E.poisson_thresholds(mu, L)
    for method in (0, 1):
        pop = np.zeros((n, 16), np.uint64)
        flips = O.ga_mutate(pop, L, T, E.bernoulli_threshold(mu, L), method, 1, 0)
        pc = sum(bin(int(x)).count("1") for x in pop.reshape(-1)[pop.reshape(-1) != 0])
        assert pc == flips  # distinct positions on an all-zero population
        assert abs(flips / n - mu) < 5 * math.sqrt(mu / n), (method, flips / n)


@pytest.mark.gpu
@pytest.mark.parametrize("L,mode,lam,stop", [(65, 0, 0.3, 0), (100, 1, 1.0, 0), (128, 2, 2.0, 0), (1024, 0, 0.5, 0),
                                             (1000, 2, 4.0, 0), (200, 0, 3.0, 1)])
def test_wide_device_ga_equals_restatement(L, mode, lam, stop):
    n = 3001
    ga = E.DeviceGA(n, L, lam, mode)
    rng = np.random.default_rng(L)
    init = _wide_random(rng, n, L)
    init[: n // 2] = 0
    ga.set_population(init)
    assert np.array_equal(ga.population(), init)
    pop = init.copy()
    T = E.poisson_thresholds(lam, L)
    tgt = int(0.55 * L) if stop else L // 2
    g = 0
    for chunk in (7, 13):
        k, b, s, c = ga.run(21, g, chunk, tgt, n // 2, stop)
        k2, b2, s2, c2 = O.ga_run_w(pop, L, mode, T, 21, g, chunk, tgt, n // 2, stop)
        assert k == k2 and np.array_equal(b, b2) and np.array_equal(s, s2) and np.array_equal(c, c2)
        assert np.array_equal(ga.population(), pop), (g, k)
        g += k
    ga.close()


@pytest.mark.gpu
def test_wide_run_ga_public_api():
    cfg = E.GAConfig(pop_size=2048, length=256, mu_L=1.0, cutoff=60, target=140, stop_when="discovery")
    rec = E.run_ga(cfg, seed=4)
    pop = np.zeros((2048, 4), np.uint64)
    k, b, s, c = O.ga_run_w(pop, 256, 0, E.poisson_thresholds(1.0, 256), 4, 0, 60, 140, 1024, 1)
    assert rec.generations == k and np.array_equal(rec.best, b) and np.array_equal(rec.count_at_target, c)
    assert len(E.run_replicas(E.GAConfig(pop_size=256, length=100, cutoff=5, stop_when="never"), [1, 2])) == 2


@pytest.mark.gpu
def test_mutation_benchmark_device_equals_restatement_and_speedup():
    """SPEC ACCEPTANCE 8: mutation by distribution beats bit-by-bit flipping by >= 2x at
    L = 1024, muL = 0.5 (device, bench.py's mutation_L1024 line); both device operators equal
    the CPU restatement bit for bit."""
    import torch
    L, n, mu = 1024, 4096, 0.5
    W = L // 64
    for method in ("distribution", "bitwise"):
        dev = torch.zeros(W * n, dtype=torch.int64, device="cuda")
        f = E.mutate_population(dev, L, mu, method, seed=3, g=2, count_flips=True)
        host = np.zeros((n, W), np.uint64)
        f2 = O.ga_mutate(host, L, E.poisson_thresholds(mu, L), E.bernoulli_threshold(mu, L),
                         0 if method == "distribution" else 1, 3, 2)
        assert f == f2
        got = dev.cpu().numpy().view(np.uint64).reshape(W, n).T
        assert np.array_equal(got, host), method
    r = E.mutation_benchmark(pop_size=1 << 18, length=1024, mu_L=0.5, reps=3)
    assert r["speedup"] >= 2.0, r
    assert abs(r["distribution_flips_per_genome"] - 0.5) < 0.02 and abs(r["bitwise_flips_per_genome"] - 0.5) < 0.02


@pytest.mark.gpu
@pytest.mark.parametrize("mode", [0, 2])
def test_jatam_fitness_cache_is_exact(mode, monkeypatch):
    """Children equal to a parent inherit its fitness (GaParams::f_known): the pre-pass skips them.
    Every generation's cached fitness vector equals a fresh classification of the population."""
    from paper_2205_15311_b200.genome import SearchSpace, decode_tileset, genome_at_index
    from paper_2205_15311_b200 import assembly as A
    S28 = SearchSpace(2, 8)
    tgt_idx = 0x801772
    target = A.assemble_once(decode_tileset(genome_at_index(S28, tgt_idx), S28), 19, seed=0,
                             genome_index=tgt_idx, run_index=0).grid.cells >= 0
    n = 8192
    ga = E.DeviceGA(n, 24, 0.3, mode)
    ga.set_population(np.random.default_rng(9).integers(0, 1 << 24, n, dtype=np.uint64))
    for g in range(5):
        f = ga.jatam_fitness(S28, target, 19, 8).clone()
        monkeypatch.setenv("TV_FITCACHE", "0")
        monkeypatch.setenv("TV_FITMEMO", "0")
        fresh = ga.jatam_fitness(S28, target, 19, 8).clone()
        monkeypatch.delenv("TV_FITCACHE")
        monkeypatch.delenv("TV_FITMEMO")
        assert bool((f == fresh).all()), g
        ga.run(3, g, 1, 361, n, 0, f_ext=f)
    ga.close()


@pytest.mark.gpu
def test_jatam_fitness_memo_is_exact(monkeypatch):
    """The genome -> fitness memo kept across generations (ClassifyParams::memo_*): a population
    drawn from few distinct genomes hits it constantly; every fitness vector equals a fresh
    classification, also after the fitness parameters change (target, k: the memo is cleared)."""
    from paper_2205_15311_b200.genome import SearchSpace, decode_tileset, genome_at_index
    from paper_2205_15311_b200 import assembly as A
    S28 = SearchSpace(2, 8)

    def shape(idx):
        return A.assemble_once(decode_tileset(genome_at_index(S28, idx), S28), 19, seed=0,
                               genome_index=idx, run_index=0).grid.cells >= 0
    t1, t2 = shape(0x801772), shape(0x5A0013)
    monkeypatch.setenv("TV_FITMEMO", "1")  # on by default only from 2^21 individuals
    n = 6000
    rng = np.random.default_rng(17)
    pool = rng.integers(0, 1 << 24, 150, dtype=np.uint64)
    ga = E.DeviceGA(n, 24, 0.5, "asexual")
    ga.set_population(pool[rng.integers(0, pool.size, n)])

    def fresh(target, k):
        monkeypatch.setenv("TV_FITCACHE", "0")
        monkeypatch.setenv("TV_FITMEMO", "0")
        out = ga.jatam_fitness(S28, target, 19, k).clone()
        monkeypatch.delenv("TV_FITCACHE")
        monkeypatch.setenv("TV_FITMEMO", "1")
        return out
    for g in range(6):
        target, k = (t1, 8) if g < 3 else ((t2, 8) if g < 5 else (t2, 4))
        f = ga.jatam_fitness(S28, target, 19, k).clone()
        assert bool((f == fresh(target, k)).all()), g
        again = ga.jatam_fitness(S28, target, 19, k).clone()  # the memo holds every genome now
        assert bool((again == f).all()), g
        ga.run(3, g, 1, 361, n, 0, f_ext=f)
    ga.close()


@pytest.mark.gpu
def test_jatam_fitness_generic_kernel_with_memo(monkeypatch):
    """JaTAM fitness in a space the bitboard kernel does not take (b = 16 labels: the generic
    thread-per-genome kernel, which inserts into the memo; lookups belong to the bitboard path's
    pre-pass), memo forced on: a first and a repeated call on the same population both equal the
    oracle."""
    from paper_2205_15311_b200._kernels import edges_from_labels
    from paper_2205_15311_b200.genome import SearchSpace, decode_tileset, genome_at_index
    monkeypatch.setenv("TV_FITMEMO", "1")
    sp = SearchSpace(2, 16)
    d, k, n = 13, 4, 600
    rng = np.random.default_rng(21)
    grid = np.empty(d * d, np.int16)

    def edges(idx):
        ts = decode_tileset(genome_at_index(sp, idx), sp)
        return edges_from_labels(np.array([v for t in ts.tiles for v in t], np.uint8), 2)

    def expected(idx, target):
        sw = np.zeros(4, np.uint64)
        st, cls, *_ = O.classify_single(edges(idx), 2, d, k, 0, idx, True, sw)
        if st != 0 or cls != 0:
            return 0
        O.assemble_single(edges(idx), 2, d, 0, idx, 0, True, grid)
        return d * d - int(np.count_nonzero((grid >= 0).reshape(d, d) != target))

    pool = rng.integers(0, 1 << 32, 150, dtype=np.uint64)
    target = None
    for idx in pool:  # a DET target shape from the pool
        sw = np.zeros(4, np.uint64)
        st, cls, *_ = O.classify_single(edges(int(idx)), 2, d, k, 0, int(idx), True, sw)
        if st == 0 and cls == 0:
            O.assemble_single(edges(int(idx)), 2, d, 0, int(idx), 0, True, grid)
            target = (grid >= 0).reshape(d, d).copy()
            break
    assert target is not None
    ga = E.DeviceGA(n, 32, 0.5, "asexual")
    exp = {int(x): expected(int(x), target) for x in pool}
    pop = pool[rng.integers(0, pool.size, n)]
    ga.set_population(pop)
    for rep in range(2):
        f = ga.jatam_fitness(sp, target, d, k).cpu().numpy().view(np.uint32)
        assert [int(v) for v in f] == [exp[int(x)] for x in pop], rep
    assert any(exp.values())  # some genomes are DET (non-zero fitness)
    ga.close()


@pytest.mark.gpu
@pytest.mark.parametrize("n", [3000, 8192])
def test_run_jatam_equals_generation_by_generation(n):
    """tv_ga_run_jatam (all generations enqueued at once) == jatam_fitness + run(f_ext) per generation:
    same stats rows, same final population; run_ga(JatamFitness, stop_when='never') takes that path."""
    from paper_2205_15311_b200 import assembly as A
    from paper_2205_15311_b200.genome import SearchSpace, decode_tileset, genome_at_index
    S28 = SearchSpace(2, 8)
    tgt_idx = 0x801772
    target = A.assemble_once(decode_tileset(genome_at_index(S28, tgt_idx), S28), 19, seed=0,
                             genome_index=tgt_idx, run_index=0).grid.cells >= 0
    init = np.random.default_rng(n).integers(0, 1 << 24, n, dtype=np.uint64)
    init[:7] = tgt_idx
    gens = 6
    g1 = E.DeviceGA(n, 24, 0.5, "asexual")
    g1.set_population(init)
    b1, s1, c1 = g1.run_jatam(S28, target, 13, 0, gens, 300)
    g2 = E.DeviceGA(n, 24, 0.5, "asexual")
    g2.set_population(init)
    rows = []
    for g in range(gens):
        f = g2.jatam_fitness(S28, target, 19, 8)
        rows.append(g2.run(13, g, 1, 300, n, 0, f_ext=f)[1:])
    assert np.array_equal(b1, np.concatenate([r[0] for r in rows]))
    assert np.array_equal(s1, np.concatenate([r[1] for r in rows]))
    assert np.array_equal(c1, np.concatenate([r[2] for r in rows]))
    assert np.array_equal(g1.population(), g2.population())
    rec = E.run_ga(E.GAConfig(pop_size=n, length=24, mu_L=0.5, cutoff=gens, target=300, stop_when="never",
                              init=init), fitness=E.JatamFitness(S28, target), seed=13)
    assert np.array_equal(rec.best, b1) and np.array_equal(rec.count_at_target, c1)
    g1.close(); g2.close()


@pytest.mark.gpu
def test_handles_refuse_another_device():
    """A GA / histogram handle used while another device is current fails loudly (its buffers
    live on the device it was created on).  Needs two GPUs; skipped otherwise."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("one GPU")
    ga = E.DeviceGA(1000, 24, 0.3)
    with torch.cuda.device(1):
        with pytest.raises(ValueError, match="belongs to device 0"):
            ga.run(1, 0, 3, 10, 1000, 0)
    ga.close()
