"""CPU-side checks of the C-ABI library: it loads without a GPU, exports every
function include/epi_b200.h declares, and agrees with ctypes on struct sizes."""

import re
from pathlib import Path

import numpy as np

from paper_2110_04421_b200 import _native as N
from paper_2110_04421_b200.defaults import default_disease, default_progression
from paper_2110_04421_b200.device import pack_params
from paper_2110_04421_b200.interventions import InterventionConfig

HEADER = Path(__file__).resolve().parents[1] / "include" / "epi_b200.h"


def declared_functions():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char \*)\s*(epi_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    lib = N.load_library()
    names = declared_functions()
    assert len(names) >= 15
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(N.EXPORTED), set(names) ^ set(N.EXPORTED)


def test_struct_sizes_match():
    lib = N.load_library()
    import ctypes
    for i, cls in enumerate((N.EpiParams, N.EpiState, N.EpiNet, N.EpiRefnetDesc)):
        assert lib.epi_struct_size(i) == ctypes.sizeof(cls)


def test_pack_params_tables():
    d, t = default_disease(), default_progression()
    p = pack_params(d, t, InterventionConfig(), 100_000)
    assert p.t_max == d.t_max == 32
    assert list(p.day_weights[:33]) == d.day_weights.tolist()
    dev = t.device_tables()
    assert p.n_specs == len(dev["taus"]) == 8
    for i, tau in enumerate(dev["taus"]):
        assert np.array_equal(np.frombuffer(p.tau[i], dtype=np.float64)[:p.tau_len[i]], tau)
    assert p.sterilizing == 1
    assert p.dose_budget == int(np.rint(0.003 * 100_000))
