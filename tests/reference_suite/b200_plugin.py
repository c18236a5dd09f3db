"""pytest plugin: run the reference's OWN test suite against GpuEngine.

Loaded with `-p b200_plugin` before collection, it rebinds the reference's
`Engine` name everywhere the suite and the runner look it up
(`epivec.engine.Engine`, `epivec.runner.Engine` bound at runner.py:20,
`epivec.Engine` re-exported by __init__.py) to
`paper_2110_04421_b200.engine.GpuEngine`.  Every `Engine(...)` the suite
builds -- directly (test_engine.py, test_interventions.py, test_oracle.py)
or through run_replication / verify_equivalence / bench (test_runner.py,
test_acceptance.py) -- then steps on the B200, fed the reference's own
parameter objects.  Nothing in the suite is edited.  Pool workers of run_scenario(workers > 1)
rebind too (fork server below), so every replication of the suite runs on
the GPU.
"""

import multiprocessing

import epivec
import epivec.engine
import epivec.runner

from paper_2110_04421_b200.engine import GpuEngine

CALLS = {"engines": 0}


class _CountingGpuEngine(GpuEngine):
    def __init__(self, *a, **kw):
        super().__init__(*a, **kw)
        CALLS["engines"] += 1


epivec.engine.Engine = _CountingGpuEngine
epivec.runner.Engine = _CountingGpuEngine
epivec.Engine = _CountingGpuEngine


# run_scenario(workers > 1) (runner.py:164-190) pools processes.  A forked
# child of a process that already holds a CUDA context cannot use the GPU,
# and a spawned child would re-import epivec without this rebinding (and
# silently step on the CPU).  Workers therefore come from a fork server that
# has imported this plugin (rebinding in place) but never touched CUDA.
multiprocessing.set_start_method("forkserver", force=True)
multiprocessing.set_forkserver_preload(["b200_plugin"])


def pytest_configure(config):
    config.addinivalue_line("markers", "slow: long-running acceptance criteria")


def pytest_terminal_summary(terminalreporter):
    terminalreporter.write_line(f"b200_plugin: GpuEngine instances built by the suite: {CALLS['engines']}")


# Diagnostics (off by default): B200_PLUGIN_BENCH_LOG=<file> appends every
# runner.bench report (engine and oracle) with its wall time to <file>.
import os as _os

if _os.environ.get("B200_PLUGIN_BENCH_LOG"):
    _bench = epivec.runner.bench

    import gc as _gc
    import time as _time
    _gc_log = []
    _gc_t = {}

    def _gc_cb(phase, info):
        if phase == "start":
            _gc_t["t"] = _time.perf_counter()
        else:
            dt = _time.perf_counter() - _gc_t.get("t", _time.perf_counter())
            if dt > 0.005:
                _gc_log.append(f"gc gen{info['generation']} {dt * 1e3:.1f} ms collected {info['collected']}")

    _gc.callbacks.append(_gc_cb)

    def _logged_bench(config, use_oracle=False):
        del _gc_log[:]
        rep = _bench(config, use_oracle=use_oracle)
        with open(_os.environ["B200_PLUGIN_BENCH_LOG"], "a") as f:
            f.write(f"{'oracle' if use_oracle else 'engine'} n={rep.n_agents} steps={rep.steps} "
                    f"wall={rep.wall_seconds * 1e3:.1f} ms {'; '.join(_gc_log)}\n")
        return rep

    epivec.runner.bench = _logged_bench
