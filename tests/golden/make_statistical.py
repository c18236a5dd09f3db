"""Reference side of the statistical curve-parity test:
R = 32 replications per case of the UNMODIFIED reference engine
(`epivec.engine.Engine`, /root/reference/pkg/src) on the config networks,
180 days each, recorded with the reference's own `_record_row`
(runner.py:101-116) -> tests/golden/stat_<case>.npz, int32 [R, 180, 19].

The reference has no knob for the BASELINE.json networks, so
each day's StepGraph comes from the pinned CPU restatement of the config
generator (`oracle/confignet_np.py`), and the engine -- the thing whose
curves are compared -- is the reference's own, fed the reference's own
DiseaseParams / ProgressionTable / InterventionConfig objects.  Initial
infections: the population's seed ids, then the reference's step-0 keyed
draws exactly as `population.seed_infections` (population.py:166-176) makes
them; DEN apps as runner.py:86-89.  Replication r uses seed
replication_seed(1, r); the GPU side of the test uses replication_seed(0, r)
(independent seeds).

The driver is `oracle/epivec_driver.ReferenceReplica` (shared with bench.py's
reference arm).  Run in the build container (needs /root/reference or
baseline/_ref):
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_statistical.py [case ...]
"""

from __future__ import annotations

import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))

R = 32
HORIZON = 180
CASES = {
    # name: (config, interventions, dose gap)
    "config0": (0, False, 0),
    "config1": (1, False, 0),
    "config2_gap21": (1, True, 21),
    "config2_gap84": (1, True, 84),
}


def one_replica(args):
    case, r = args
    from epivec.runner import replication_seed
    from oracle.epivec_driver import ReferenceReplica, reference_interventions
    from paper_2110_04421_b200.confignet import ConfigNetworkSpec
    cfg, iv_on, gap = CASES[case]
    rep = ReferenceReplica(ConfigNetworkSpec.config(cfg), replication_seed(1, r),
                           reference_interventions(iv_on, gap))
    return r, rep.run(HORIZON).astype(np.int32)


def main(cases):
    for case in cases:
        t0 = time.time()
        with ProcessPoolExecutor(max_workers=os.cpu_count() or 1) as pool:
            out = dict(pool.map(one_replica, [(case, r) for r in range(R)]))
        series = np.stack([out[r] for r in range(R)])
        np.savez_compressed(HERE / f"stat_{case}.npz", series=series,
                            seeds_base=np.int64(1), horizon=np.int64(HORIZON))
        print(case, series.shape, f"{time.time() - t0:.0f}s", "attack",
              series[:, -1, 12].mean() / series[0, 0, 1:12].sum(), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or list(CASES))
