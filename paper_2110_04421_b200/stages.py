"""Stage / vaccine / network enumerations and the stage lookup tables.

Integer values are part of the data layout shared with the CUDA kernels
(`csrc/epi_common.cuh`) and with the reference (`pkg/src/epivec/stages.py:22-79`):
stage codes 0..10, NEVER = -1, network kinds 0..2.
"""

from enum import IntEnum

import numpy as np

NEVER = -1
N_AGE_BANDS = 9
N_OCCUPATIONS = 23


class Stage(IntEnum):
    SUSCEPTIBLE = 0
    ASYMPTOMATIC = 1
    PRESYMPTOMATIC_MILD = 2
    PRESYMPTOMATIC_SEVERE = 3
    MILD_SYMPTOMATIC = 4
    SEVERE_SYMPTOMATIC = 5
    HOSPITALIZED = 6
    CRITICAL_ICU = 7
    RECOVERED = 8
    VACCINATED = 9
    DEAD = 10

    def __str__(self):
        return self.name.lower()


N_STAGES = len(Stage)


class VaccineStatus(IntEnum):
    PRE_VACCINATION = 0
    FIRST_DOSE = 1
    FULLY_VACCINATED = 2


class NetworkKind(IntEnum):
    HOUSEHOLD = 0
    OCCUPATION = 1
    RANDOM = 2


N_NETWORK_KINDS = len(NetworkKind)

STAGE_BY_NAME = {str(s): s for s in Stage}


def _lut(members):
    t = np.zeros(N_STAGES, dtype=bool)
    t[[int(m) for m in members]] = True
    return t


# transmit in community networks (stages 1..5)
INFECTIOUS_STAGE = _lut(range(1, 6))
# no symptoms yet: asymptomatic and the two presymptomatic stages
ASYMPTOMATIC_LIKE_STAGE = _lut(range(1, 4))
# carry an active infection (tests positive, counts toward vaccination trigger)
ACTIVE_INFECTION_STAGE = _lut(range(1, 8))
ABSORBING_STAGES = (Stage.RECOVERED, Stage.VACCINATED, Stage.DEAD)
