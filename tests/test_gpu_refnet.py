"""Row f1: reference-native networks generated on the device.

* bitwise: csrc/epi_refnet.cuh vs its CPU restatement oracle/refnet_np.py;
* structure: symmetry, no self loops / duplicates / dead agents, household
  cliques identical to the reference's (graphs.py:54-83);
* statistics: per-family edge counts vs the reference's own realizer
  (oracle/graphs_np.py, pinned to the recorded graphs);
* end to end: the golden-trajectory scenario stepped by GpuEngine on device
  graphs, bitwise against the oracle engine on oracle graphs.
"""

import dataclasses

import numpy as np
import pytest
import torch

from golden_io import Trajectory
from oracle import engine_np, refnet_np
from oracle.graphs_np import ReferenceRealizer
from paper_2110_04421_b200.defaults import POPULATION
from paper_2110_04421_b200.graph import StepGraph

pytestmark = pytest.mark.gpu

MEANS = POPULATION["networks"]["occupation_mean_interactions"]
BETA = POPULATION["networks"]["rewire_beta"]


def synthetic_population(n, seed):
    """Population with the default spec's shapes (population.py:43-108)."""
    g = np.random.default_rng(seed)
    sizes = g.choice([1, 2, 3, 4, 5, 6], size=n, p=[0.28, 0.34, 0.15, 0.13, 0.07, 0.03])
    hh = np.repeat(np.arange(n), sizes)[:n]
    g.shuffle(hh)                                   # households need not be contiguous
    occ = np.where(g.random(n) < 0.6, g.choice(np.arange(1, 24), size=n,
                                               p=np.array(POPULATION["occupation_distribution"])
                                               / np.sum(POPULATION["occupation_distribution"])), 0)
    deg = np.array(POPULATION["random_degree_by_age"])[g.integers(0, 9, size=n)]
    return hh.astype(np.int64), occ.astype(np.int8), deg.astype(np.float32)


def canon(g):
    s, d, k = (x.cpu().numpy() if torch.is_tensor(x) else x for x in (g.src, g.dst, g.kind))
    o = np.lexsort((k, s, d))
    return s[o], d[o], k[o]


def realizer(hh, occ, deg, seed, means=MEANS, beta=BETA):
    from paper_2110_04421_b200.refnet import GpuRealizer
    return GpuRealizer(seed, hh, occ, deg, means, beta)


@pytest.mark.parametrize("n,seed,dead_frac", [(2000, 1, 0.0), (10_000, 7, 0.05), (50_000, 3, 0.2)])
def test_bitwise_vs_restatement(n, seed, dead_frac):
    hh, occ, deg = synthetic_population(n, seed)
    r = realizer(hh, occ, deg, seed)
    dead = np.random.default_rng(seed + 1).random(n) < dead_frac
    for step in (0, 1, 17):
        got = canon(r.realize(step, dead))
        want = refnet_np.realize(seed, step, hh, occ, deg, MEANS, BETA, dead)
        for a, b, name in zip(got, want, ("src", "dst", "kind")):
            assert np.array_equal(a, b), (step, name, len(a), len(b))


def test_structure_and_households_equal_reference():
    n, seed = 20_000, 11
    hh, occ, deg = synthetic_population(n, seed)
    dead = np.random.default_rng(2).random(n) < 0.1
    s, d, k = canon(realizer(hh, occ, deg, seed).realize(4, dead))
    assert not np.any(s == d)
    assert not np.any(dead[s] | dead[d])
    fwd = np.sort((s.astype(np.int64) << 32 | d) * 4 + k)
    bwd = np.sort((d.astype(np.int64) << 32 | s) * 4 + k)
    assert np.array_equal(fwd, bwd)                          # symmetric per family
    for kind in (1, 2):
        m = k == kind
        key = s[m].astype(np.int64) << 32 | d[m]
        assert len(np.unique(key)) == len(key)               # no duplicate pairs
    rs, rd, rk = ReferenceRealizer(seed, hh, occ, deg, MEANS, BETA).realize(4, dead)
    mine = np.sort(s[k == 0].astype(np.int64) << 32 | d[k == 0])
    ref = np.sort(rs[rk == 0].astype(np.int64) << 32 | rd[rk == 0])
    assert np.array_equal(mine, ref)


def test_family_sizes_match_reference_generator():
    n, seed = 40_000, 5
    hh, occ, deg = synthetic_population(n, seed)
    dead = np.zeros(n, bool)
    ref = ReferenceRealizer(seed, hh, occ, deg, MEANS, BETA)
    r = realizer(hh, occ, deg, seed)
    counts_ref = np.zeros(3)
    counts_gpu = np.zeros(3)
    steps = range(6)
    for t in steps:
        counts_ref += np.bincount(ref.realize(t, dead)[2], minlength=3)
        counts_gpu += np.bincount(canon(r.realize(t, dead))[2], minlength=3)
    assert counts_gpu[0] == counts_ref[0]
    # both preserve every lattice edge one-for-one (graphs.py:91-93): n*k/2
    # per occupation, exactly
    assert counts_gpu[1] == counts_ref[1]
    # stub pairing: same stub law, same self/duplicate rules
    assert abs(counts_gpu[2] - counts_ref[2]) <= 0.01 * counts_ref[2]


def test_degree_law_matches_reference():
    """Per-agent random-network degree: mean over steps vs floor+Bernoulli law."""
    n, seed = 30_000, 9
    hh, occ, deg = synthetic_population(n, seed)
    dead = np.zeros(n, bool)
    r = realizer(hh, occ, deg, seed)
    tot = np.zeros(n)
    T = 20
    for t in range(T):
        s, d, k = canon(r.realize(t, dead))
        tot += np.bincount(d[k == 2], minlength=n)
    for v in np.unique(deg):
        m = deg == v
        assert abs(tot[m].mean() / T - v) < 0.05 * v + 0.05, (v, tot[m].mean() / T)


@pytest.mark.parametrize("case", ["all_dead", "one_alive", "tiny", "no_occupation", "zero_degree"])
def test_edge_cases(case):
    n = {"tiny": 3, "one_alive": 50}.get(case, 400)
    hh, occ, deg = synthetic_population(n, 4)
    dead = np.zeros(n, bool)
    if case == "all_dead":
        dead[:] = True
    elif case == "one_alive":
        dead[:] = True
        dead[7] = False
    elif case == "no_occupation":
        occ[:] = 0
    elif case == "zero_degree":
        deg[:] = 0
    got = canon(realizer(hh, occ, deg, 3).realize(2, dead))
    want = refnet_np.realize(3, 2, hh, occ, deg, MEANS, BETA, dead)
    for a, b in zip(got, want):
        assert np.array_equal(a, b)
    if case in ("all_dead", "one_alive"):
        assert len(got[0]) == 0


@pytest.mark.parametrize("name", ["noiv", "alliv"])
def test_engine_on_device_graphs_bitwise_vs_oracle(name):
    """Golden scenario, networks from the device generator, state on device."""
    from paper_2110_04421_b200.engine import GpuEngine
    tr = Trajectory(name)
    z = tr.z
    hh, occ, deg = z["init_household_id"], z["init_occupation"], z["init_random_degree"]
    r = realizer(hh, occ, deg, tr.seed)
    cols_o = tr.initial_cols()
    cols_g = tr.initial_cols()
    eo = engine_np.OracleEngine(cols_o, tr.disease, tr.table, tr.iv, tr.seed)
    eg = GpuEngine(cols_g, tr.disease, tr.table, tr.iv, tr.seed, resident=True)
    eo.vaccination_open = eg.vaccination_open = bool(z["vaccination_open"])
    for t in range(30):
        dead = cols_o.stage == 10
        s, d, k = refnet_np.realize(tr.seed, t, hh, occ, deg, MEANS, BETA, dead)
        ev_o = eo.step(StepGraph(t, s, d, k))
        ev_g = eg.step(r.realize(t, eg.dev.t["stage"] == 10))
        assert dataclasses.astuple(ev_g) == dataclasses.astuple(ev_o), t
    eg.sync_to_host()
    for c in ("stage", "infected_at", "next_stage", "next_transition_at", "quarantine_until",
              "vaccine_status", "immune"):
        assert np.array_equal(getattr(cols_g, c), getattr(cols_o, c)), c


# -- Watts-Strogatz properties of the reference's own tests, on the device ----
# (test_graphs.py:68-114; adjacency_sets / mean_clustering restated from
# test_graphs.py:16-40 as the brute-force oracle)

def adjacency_sets(us, vs, n):
    adj = [set() for _ in range(n)]
    for u, v in zip(us.tolist(), vs.tolist()):
        adj[u].add(v)
        adj[v].add(u)
    return adj


def mean_clustering(adj):
    coeffs = []
    for nbrs in adj:
        d = len(nbrs)
        if d < 2:
            coeffs.append(0.0)
            continue
        nb = sorted(nbrs)
        links = sum(1 for i, a in enumerate(nb) for b in nb[i + 1:] if b in adj[a])
        coeffs.append(2.0 * links / (d * (d - 1)))
    return float(np.mean(coeffs))


def one_occupation(n, k, beta, seed):
    """n agents, every one in occupation 1 (mean k), alone in its household,
    no random contacts: the realizer's graph is one small-world lattice."""
    hh = np.arange(n, dtype=np.int64)
    occ = np.ones(n, dtype=np.int8)
    deg = np.zeros(n, dtype=np.float32)
    return realizer(hh, occ, deg, seed, means=[float(k)], beta=beta), (hh, occ, deg)


@pytest.mark.parametrize("n,half_k,beta,seed", [
    (6, 1, 1.0, 0), (7, 2, 1.0, 3), (10, 2, 1.0, 1), (13, 1, 0.5, 5), (20, 2, 1.0, 8),
    (33, 2, 0.1, 2), (60, 2, 1.0, 9), (60, 1, 0.5, 4), (1000, 3, 1.0, 6), (4000, 5, 0.1, 7)])
def test_rewiring_never_changes_edge_count(n, half_k, beta, seed):
    """test_graphs.py:76-92: len == n*k/2, no self loops, no duplicate pairs
    -- for the device realizer, at every step, dead agents included; and
    bitwise equal to the restatement (collisions re-drawn in rounds)."""
    k = 2 * half_k
    r, (hh, occ, deg) = one_occupation(n, k, beta, seed)
    for step in range(8):
        dead = np.zeros(n, bool)
        if step >= 4:
            dead[np.random.default_rng(step).random(n) < 0.1] = True
        m = int((~dead).sum())
        kk = min(k, 2 * ((m - 1) // 2))
        s, d, kd = canon(r.realize(step, dead))
        assert np.all(kd == 1)
        want = m * kk // 2 if (m >= 3 and kk >= 2) else 0
        assert len(s) == 2 * want, (step, len(s), 2 * want)
        assert not np.any(s == d)
        key = s.astype(np.int64) << 32 | d
        assert len(np.unique(key)) == len(key)
        ref = refnet_np.realize(seed, step, hh, occ, deg, [float(k)], beta, dead)
        for a, b in zip((s, d, kd), ref):
            assert np.array_equal(a, b), step


def test_clustering_between_lattice_and_random():
    """test_graphs.py:104-114 on the device realizer: 1000 nodes, k = 6."""
    n, k = 1000, 6
    values = {}
    for beta in (0.0, 0.1, 1.0):
        r, _ = one_occupation(n, k, beta, 7)
        s, d, _ = canon(r.realize(0, np.zeros(n, bool)))
        values[beta] = mean_clustering(adjacency_sets(s, d, n))
    assert values[0.0] == pytest.approx(0.6, abs=1e-12)      # 3(k-2)/(4(k-1))
    assert values[0.0] > values[0.1] > values[1.0]
