"""Sparse push rows (whole-population fused days beyond the push tables):
only infectious sources scatter into the in-rows; the day kernel walks its
own out-partners and no inverse bijections.  Everything it produces must be
bitwise what the inverse-walk path and the full push tables produce: the
hazard of every agent on every day, the 24-column record (the edge count is
derived from the out-edges), the final codes and stages, across chunked
runs, single steps, resets and graph replays."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2110_04421_b200.confignet import ConfigNetworkSpec, synthesize
from paper_2110_04421_b200.defaults import default_disease, default_progression
from paper_2110_04421_b200.interventions import InterventionConfig
from paper_2110_04421_b200.sim import ConfigSimulation

pytestmark = pytest.mark.gpu


def _sim(pop, **kw):
    return ConfigSimulation(pop, default_disease(), default_progression(), InterventionConfig(), 17,
                            mode="fused", horizon=90, **kw)


@pytest.mark.parametrize("n,spec", [(30000, 1), (12000, 0)])
def test_sparse_rows_bitwise_equal_inverse_walks_and_push_tables(n, spec):
    pop = synthesize(ConfigNetworkSpec.config(spec, n_agents=n, initial_infections=60), 3)
    full = _sim(pop)                                  # push tables (persistent run)
    inv = _sim(pop, push_max=0, sparse_push=False)    # 16 inverse slot walks per agent
    sp = _sim(pop, push_max=0)                        # sparse rows
    lam = {}
    for name, s in (("full", full), ("inv", inv), ("sparse", sp)):
        buf = s.lambda_probe(0, 90)
        s.run()
        torch.cuda.synchronize()
        lam[name] = buf.cpu().numpy()
        s.lambda_probe(0, 0)
    assert np.array_equal(lam["sparse"], lam["inv"])
    assert np.array_equal(lam["sparse"], lam["full"])
    for s in (inv, full):
        assert np.array_equal(sp.rec.cpu().numpy(), s.rec.cpu().numpy())
        assert torch.equal(sp._codes_buf, s._codes_buf)
        assert np.array_equal(sp.host_columns().stage, s.host_columns().stage)
    assert sp.rec.cpu().numpy()[:, 19].min() > 0       # edges counted every day


def test_sparse_rows_chunked_reset_and_graph_replay():
    pop = synthesize(ConfigNetworkSpec.config(1, n_agents=20000, initial_infections=40), 5)
    ref = _sim(pop, push_max=0, sparse_push=False)
    ref.run()
    sp = _sim(pop, push_max=0)
    for chunk in (7, 1, 13):
        sp.run(chunk)
    sp.step()
    sp.reset()
    sp.run(3)
    sp.reset()
    sp.run()
    assert np.array_equal(sp.rec.cpu().numpy(), ref.rec.cpu().numpy())
    sp.capture()
    for _ in range(2):
        sp.replay()
    assert np.array_equal(sp.rec.cpu().numpy(), ref.rec.cpu().numpy())
    assert torch.equal(sp._codes_buf, ref._codes_buf)


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("sparse", [True, False])
def test_partitioned_ranks_sparse_rows_on_and_off_equal_single(world, sparse):
    """Partitioned ranks (host threads, the per-day code all-gather): with
    sparse rows every rank seeds its own rows from all infectious sources
    after the gather; without, 16 inverse walks per owned agent.  Both are
    bitwise the single-rank run (push tables)."""
    from paper_2110_04421_b200.partition import run_threaded
    pop = synthesize(ConfigNetworkSpec.config(1, n_agents=15000, initial_infections=80), 8)
    d, t, iv = default_disease(), default_progression(), InterventionConfig()
    ref = ConfigSimulation(pop, d, t, iv, 23, mode="fused", horizon=50)
    ref.run()
    sims, rec = run_threaded(pop, d, t, iv, 23, world, 50, mode="fused", sparse_push=sparse)
    assert np.array_equal(rec.cpu().numpy(), ref.rec.cpu().numpy())
    full = ref.host_columns()
    for s in sims:
        lo, hi = s.plan.rows(s.rank)
        assert np.array_equal(s.host_columns().stage[lo:hi], full.stage[lo:hi])
