"""ctypes binding of libepib200.so (C ABI: include/epi_b200.h).

The library is built in-tree by `__graft_entry__.build()` (nvcc, sm_100a).
There is no fallback: if the library or a CUDA device is missing, `lib()`
raises, so nothing on the hot path silently runs on the CPU.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .errors import ConfigError, DeviceError, InvariantViolation

LIB_PATH = Path(__file__).resolve().parent / "libepib200.so"

MAX_T, MAX_SPECS, MAX_TAUS, MAX_SLOTS = 127, 16, 512, 32
REC_LEN = 24
REC = dict(step=0, stage0=1, cum_inf=12, cum_deaths=13, in_care=14, new_inf=15, tests=16,
           doses=17, notify=18, edges=19, deaths=20, hosp=21, active=22, flags=23)
FLAG_INDEX, FLAG_SELFLOOP, FLAG_KIND = 1, 2, 4
FLAG_STAGE_RANGE, FLAG_NO_TIMESTAMP, FLAG_NEG_HAZARD = 8, 16, 32
F32, F64_CANONICAL = 0, 1

_d, _i32, _i64, _u64, _p = C.c_double, C.c_int32, C.c_int64, C.c_uint64, C.c_void_p


class EpiParams(C.Structure):
    _fields_ = [
        ("rate_scale", _d), ("asymptomatic_factor", _d), ("mean_daily_interactions", _d),
        ("age_susceptibility", _d * 9), ("network_scale", _d * 3),
        ("t_max", _i32), ("sterilizing", _i32),
        ("day_weights", _d * (MAX_T + 1)),
        ("n_targets", _i32 * 11), ("targets", (_i32 * 3) * 11), ("spec_of", (_i32 * 3) * 11),
        ("cum", ((_d * 3) * 9) * 11),
        ("n_specs", _i32), ("tau_len", _i32 * MAX_SPECS), ("tau", (_d * MAX_TAUS) * MAX_SPECS),
        ("quarantine_enabled", _i32), ("quarantine_duration", _i32), ("quarantine_dropout", _d),
        ("testing_enabled", _i32), ("turnaround_min", _i32), ("turnaround_max", _i32),
        ("den_enabled", _i32), ("detection_prob", _d), ("false_positive_prob", _d),
        ("den_compliance", _d), ("den_lookback", _i32), ("vaccination_enabled", _i32),
        ("strategy", _i32), ("elderly_band", _i32), ("dose1_efficacy", _d), ("dose2_efficacy", _d),
        ("dose2_topup", _d), ("dose1_latency", _i32), ("dose2_latency", _i32), ("dose_gap", _i32),
        ("_pad0", _i32), ("dose_budget", _i64), ("start_trigger_count", _d),
    ]


STATE_FIELDS = ("age_band", "stage", "infected_at", "next_transition_at", "next_stage",
                "quarantine_until", "quarantine_started_at", "has_den_app", "vaccine_status",
                "dose1_at", "dose2_at", "immune", "immunity_check_at", "immunity_check_prob",
                "immunity_check_dose", "test_sample_at", "test_result_at", "test_positive",
                "den_test_due_at")


class EpiState(C.Structure):
    _fields_ = [("n_agents", _i64)] + [(f, _p) for f in STATE_FIELDS]


class EpiNet(C.Structure):
    _fields_ = [
        ("n_agents", _i64), ("hh_off", _p), ("hh_size", _p), ("wp_id", _p), ("wp_local", _p),
        ("wp_base", _p), ("wp_size", _p), ("wp_members", _p), ("n_workplaces", _i32),
        ("colleague_draws", _i32), ("random_slots", _i32), ("row_cap", _i32),
        ("n_member_slots", _i64), ("poisson_cdf", _d * MAX_SLOTS),
    ]


# epi_exchange_fn (include/epi_b200.h): (user, kind, buf, count, stream) -> int
XFN = C.CFUNCTYPE(_i32, _p, _i32, _p, _i64, _p)


class EpiPopSpec(C.Structure):
    _fields_ = [("n_agents", _i64), ("age_cum", _d * 9), ("n_sizes", _i32), ("hh_sizes", _i32 * 32),
                ("hh_cum", _d * 32), ("worker_mask", C.c_uint32), ("wp_min", _i32), ("wp_max", _i32),
                ("n_seeds", _i64)]


class EpiPopOut(C.Structure):
    _fields_ = [(f, _p) for f in ("age_band", "household_id", "hh_off", "hh_size", "wp_id", "wp_local",
                                  "wp_members", "wp_base", "wp_size", "seeds", "counts")]


class EpiRefnetDesc(C.Structure):
    _fields_ = [
        ("n_agents", _i64), ("hh_members", _p), ("hh_start", _p), ("hh_size", _p),
        ("n_occ", _i32), ("_pad", _i32), ("occ_members", _p), ("occ_start", _p), ("occ_k", _p),
        ("n_member_slots", _i64), ("rewire_beta", _d), ("random_degree", _p), ("table_slots", _i64),
    ]


_SIGS = {
    "epi_create": (_i32, [C.POINTER(EpiParams), _i64, C.POINTER(_p)]),
    "epi_destroy": (_i32, [_p]),
    "epi_set_params": (_i32, [_p, C.POINTER(EpiParams)]),
    "epi_set_rows": (_i32, [_p, _i64, _i64]),
    "epi_set_hot_window": (_i32, [_p, _p, _i64]),
    "epi_set_exchange": (_i32, [_p, XFN, _p]),
    "epi_set_infection_mode": (_i32, [_p, _i32]),
    "epi_pop_synthesize": (_i32, [C.POINTER(EpiPopSpec), _u64, C.POINTER(EpiPopOut), _p]),
    "epi_set_push_max": (_i32, [_p, _i64]),
    "epi_set_sparse_push": (_i32, [_p, _i32]),
    "epi_set_lambda_probe": (_i32, [_p, _p, _i32, _i32]),
    "epi_comm_unique_id": (_i32, [_p]),
    "epi_comm_create": (_i32, [_p, _i32, _i32, _p]),
    "epi_comm_destroy": (_i32, [_p]),
    "epi_set_code_exchange": (_i32, [_p, _p, _i32, _i64]),
    "epi_allgather_codes": (_i32, [_p, _p, _p]),
    "epi_set_sigma_ahead": (_i32, [_p, _i32]),
    "epi_set_persistent": (_i32, [_p, _i32]),
    "epi_set_iv_fusion": (_i32, [_p, _i32]),
    "epi_set_day_grid": (_i32, [_p, _i32]),
    "epi_quartiles": (_i32, [_p, _i64, _i32, _i32, _p, _i32, _p, _p]),
    "epi_run_persistent": (_i32, [_p, _i32, _i32]),
    "epi_last_error": (C.c_char_p, []),
    "epi_version": (_i32, []),
    "epi_struct_size": (_i64, [_i32]),
    "epi_uniforms": (_i32, [_u64, _i32, _i32, _p, _i64, _i32, _p, _p]),
    "epi_graph_load": (_i32, [_p, _p, _p, _p, _i64, _p]),
    "epi_graph_load_counted": (_i32, [_p, _p, _p, _p, _p, _i64, _p]),
    "epi_gather": (_i32, [_p, C.POINTER(EpiState), _i32, _i32, _p, _p]),
    "epi_step": (_i32, [_p, C.POINTER(EpiState), _i32, _u64, _p, _p, _p, _i32, _p]),
    "epi_step_with_hazard": (_i32, [_p, C.POINTER(EpiState), _i32, _u64, _p, _p, _p, _p, _p]),
    "epi_read_flags": (_i32, [_p, C.POINTER(_i32), _p]),
    "epi_codes": (_i32, [_p, C.POINTER(EpiState), C.POINTER(EpiNet), _u64, _i32, _p, _p]),
    "epi_net_realize": (_i32, [C.POINTER(EpiNet), _u64, _i32, _p, _p, _p, _i32, _p]),
    "epi_net_attach": (_i32, [_p, C.POINTER(EpiNet)]),
    "epi_sim_step": (_i32, [_p, C.POINTER(EpiState), _i32, _u64, _i32, _i32, _p, _p, _p, _p, _p]),
    "epi_sim_run": (_i32, [_p, C.POINTER(EpiState), _i32, _i32, _u64, _i32, _i32, _p, _p, _p, _p, _p]),
    "epi_sim_step_timed": (_i32, [_p, C.POINTER(EpiState), _i32, _u64, _i32, _i32, _p, _p, _p, _p,
                                  _p, _p]),
    "epi_net_generate": (_i32, [_p, _i32, _u64, _p, _p]),
    "epi_net_gather": (_i32, [_p, C.POINTER(EpiState), _i32, _p, _p, _p, _p]),
    "epi_refnet_create": (_i32, [C.POINTER(EpiRefnetDesc), C.POINTER(_p)]),
    "epi_refnet_destroy": (_i32, [_p]),
    "epi_refnet_realize": (_i32, [_p, _u64, _i32, _p, _p, _p, _p, _i64, C.POINTER(_i64), _p]),
    "epi_refnet_realize_counted": (_i32, [_p, _u64, _i32, _p, _p, _p, _p, _i64, _p, _p]),
    "epi_refnet_run": (_i32, [_p, _p, C.POINTER(EpiState), _u64, _u64, _i32, _i32, _p, _p, _p, _i64, _p, _p, _p,
                              _p]),
    "epi_net_csr": (_i32, [_p, _i32, C.POINTER(_p), C.POINTER(_p)]),
    "epi_seed_infections": (_i32, [_p, C.POINTER(EpiState), _u64, _p, _i64, _p]),
    "epi_assign_app": (_i32, [C.POINTER(EpiState), _u64, _d, _p]),
}

EXPORTED = tuple(_SIGS)
_lib = None


def load_library(path: os.PathLike | str | None = None) -> C.CDLL:
    """Load and type the library (no GPU needed; used by the CPU suite too)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    # EPI_B200_LIB: an alternative build of the library (A/B timing of kernel variants)
    p = Path(path) if path else Path(os.environ.get("EPI_B200_LIB", LIB_PATH))
    if not p.exists():
        raise DeviceError(f"{p} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(str(p))
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype, fn.argtypes = res, args
    for which, cls in enumerate((EpiParams, EpiState, EpiNet, EpiRefnetDesc)):
        if lib.epi_struct_size(which) != C.sizeof(cls):
            raise DeviceError(f"ABI mismatch for {cls.__name__}: C {lib.epi_struct_size(which)} "
                              f"vs ctypes {C.sizeof(cls)}")
    if path is None:
        _lib = lib
    return lib


def lib() -> C.CDLL:
    """The library, requiring a usable CUDA device."""
    import torch
    if not torch.cuda.is_available():
        raise DeviceError("paper_2110_04421_b200 needs a CUDA device (B200); none is visible")
    return load_library()


def check(rc: int) -> None:
    if rc == 0:
        return
    msg = (_lib.epi_last_error() or b"").decode() if _lib else ""
    if rc == -1:
        raise ConfigError(msg)
    if rc == -2:
        raise InvariantViolation(msg)
    raise DeviceError(msg or f"native error {rc}")


def ptr(t) -> int:
    """Raw device pointer of a torch tensor (0 for None)."""
    return 0 if t is None else int(t.data_ptr())


def stream_handle(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)
