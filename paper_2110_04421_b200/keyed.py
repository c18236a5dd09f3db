"""Scalar side of the keyed counter-based hash (host only).

The per-agent draws all run on the device (`csrc/epi_common.cuh`); the host only
needs the scalar prefix and seed derivations, e.g. to pick replication seeds.
Same splitmix64 chain and constants as the reference
(`pkg/src/epivec/rng.py:20-23, 60-108`): draws are a pure function of
(seed, step, purpose, agent, k).
"""

from enum import IntEnum

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
MIX1 = 0xBF58476D1CE4E5B9
MIX2 = 0x94D049BB133111EB
INIT = 0x243F6A8885A308D3


class Purpose(IntEnum):
    """Stream tags.  1-11 and 64-68 keep the reference's values
    (`rng.py:37-57`); 72+ are new tags used by the config-network generator
    and synthetic population of BASELINE.json configs 0-4."""

    INFECTION = 1
    INFECTION_EDGE = 2
    ENTRY_STAGE = 3
    PROGRESSION_BRANCH = 4
    PROGRESSION_DELAY = 5
    TEST_POSITIVE = 6
    TEST_TURNAROUND = 7
    QUARANTINE_DROPOUT = 8
    DEN_COMPLIANCE = 9
    DEN_APP = 10
    VACCINE_IMMUNITY = 11
    REPLICATION = 64
    POPULATION = 65
    SEEDING = 66
    GRAPH_OCCUPATION = 67
    GRAPH_RANDOM = 68
    # config network generator (this framework)
    NET_RANDOM_COUNT = 72
    NET_RANDOM_PERM = 73
    NET_WORK_PERM = 74
    NET_WORK_SHIFT = 75
    # config population synthesis (this framework)
    POP_AGE = 76
    POP_HOUSEHOLD = 77
    POP_WORKPLACE = 78
    POP_SEEDS = 79
    ENSEMBLE_SCALE = 80


def mix64(z: int) -> int:
    z = ((z ^ (z >> 30)) * MIX1) & M64
    z = ((z ^ (z >> 27)) * MIX2) & M64
    return z ^ (z >> 31)


def fold(h: int, value: int) -> int:
    return mix64(h ^ ((GOLDEN * (value + 1)) & M64))


def key_prefix(seed: int, step: int, purpose: int) -> int:
    return fold(fold(mix64(INIT ^ (seed & M64)), step), int(purpose))


def hash64(seed: int, step: int, purpose: int, index: int, k: int = 0) -> int:
    return fold(fold(key_prefix(seed, step, purpose), index), k)


def uniform(seed: int, step: int, purpose: int, agent: int, k: int = 0) -> float:
    return (hash64(seed, step, purpose, agent, k) >> 11) * (1.0 / (1 << 53))


def derive_seed(seed: int, purpose: int, *indices: int) -> int:
    h = key_prefix(seed, 0, purpose)
    for ix in indices:
        h = fold(h, ix)
    return h


def replication_seed(base_seed: int, index: int) -> int:
    """Seed of replication `index` (reference `runner.py:77-78`)."""
    return derive_seed(base_seed, Purpose.REPLICATION, index)
