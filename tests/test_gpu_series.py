"""Row f3 (output) on the device: `epi_quartiles` (replication quartiles)
bitwise equal to the reference's `summarize` (golden) and to np.percentile;
ConfigSimulation.result() rows equal the device records."""

from pathlib import Path

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import series_np
from paper_2110_04421_b200.series import (SUMMARY_METRICS, RunResult, summarize, summarize_device,
                                          summary_to_csv, summary_to_long_csv)

pytestmark = pytest.mark.gpu
G = np.load(Path(__file__).parent / "golden" / "series.npz")


def test_device_summary_of_reference_runs_is_bitwise_reference():
    runs = [RunResult(replication=i, seed=0, data=G["runs_data"][i]) for i in range(G["runs_data"].shape[0])]
    s = summarize(runs)
    assert summary_to_csv(s) == bytes(G["sum_wide"]).decode()
    assert summary_to_long_csv(s) == bytes(G["sum_long"]).decode()


@pytest.mark.parametrize("key", [k for k in G.files if k.startswith("synth_")])
def test_device_quartiles_bitwise_reference(key):
    _, R, H, seed = key.split("_")
    data = np.random.default_rng(int(seed)).integers(0, 100_000, size=(int(R), int(H), 19), dtype=np.int64)
    s = summarize_device(torch.from_numpy(data).cuda())
    assert np.array_equal(np.stack([s[m] for m in SUMMARY_METRICS]), G[key])


@pytest.mark.parametrize("R", [3, 17, 128, 1024])
def test_device_quartiles_of_simulation_records(R):
    """Records of R config replicas (24-column device rows) summarized in
    place, against the oracle (np.percentile) on the same records."""
    from paper_2110_04421_b200 import keyed
    from paper_2110_04421_b200.confignet import ConfigNetworkSpec, synthesize
    from paper_2110_04421_b200.defaults import default_disease, default_progression
    from paper_2110_04421_b200.interventions import InterventionConfig
    from paper_2110_04421_b200.sim import ConfigSimulation
    spec = ConfigNetworkSpec.config(0, n_agents=2000, initial_infections=10)
    pop = synthesize(spec, 1)
    recs = []
    for r in range(min(R, 8)):
        sim = ConfigSimulation(pop, default_disease(), default_progression(), InterventionConfig(),
                               keyed.replication_seed(0, r), mode="fused", horizon=40)
        sim.run()
        recs.append(sim.rec.clone())
        res = sim.result(r)
        assert np.array_equal(res.data, sim.records()[:, :19])
        assert res.n_edges_total == int(sim.records()[:, 19].sum())
    stacked = torch.stack([recs[i % len(recs)] + (i // len(recs)) for i in range(R)])   # [R, 40, 24]
    s = summarize_device(stacked)
    ref = series_np.summarize_stacked(stacked.cpu().numpy())
    assert np.array_equal(np.stack([s[m] for m in SUMMARY_METRICS]), ref)


@pytest.mark.parametrize("R,hi", [(4097, 100_000), (10_000, 7), (65_536, 2**40)])
def test_device_quartiles_beyond_4096_replications(R, hi):
    """More replications than the shared-memory sort holds: the
    bisection kernel (k_quartiles_large) is bitwise np.percentile, ties and
    wide values included."""
    data = np.random.default_rng(R).integers(0, hi, size=(R, 6, 19), dtype=np.int64)
    s = summarize_device(torch.from_numpy(data).cuda())
    ref = series_np.summarize_stacked(data)
    assert np.array_equal(np.stack([s[m] for m in SUMMARY_METRICS]), ref)
