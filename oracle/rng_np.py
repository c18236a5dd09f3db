"""Vectorised keyed draws (restates pkg/src/epivec/rng.py:60-100)."""

import numpy as np

_M64 = (1 << 64) - 1
_G = np.uint64(0x9E3779B97F4A7C15)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)
_I = 0x243F6A8885A308D3


def _mix_py(z):
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def _fold_py(h, v):
    return _mix_py(h ^ ((0x9E3779B97F4A7C15 * (v + 1)) & _M64))


def prefix(seed, step, purpose):
    """rng.py:76-81"""
    return _fold_py(_fold_py(_mix_py(_I ^ (int(seed) & _M64)), int(step)), int(purpose))


def _mix(z):
    z = (z ^ (z >> np.uint64(30))) * _C1
    z = (z ^ (z >> np.uint64(27))) * _C2
    return z ^ (z >> np.uint64(31))


def hashes(seed, step, purpose, idx, k=0):
    """64-bit keyed hash for an index array (rng.py:92-100 before the >>11)."""
    with np.errstate(over="ignore"):
        a = np.asarray(idx, dtype=np.uint64)
        h = _mix(np.uint64(prefix(seed, step, purpose)) ^ (_G * (a + np.uint64(1))))
        return _mix(h ^ (_G * np.uint64(k + 1)))


def uniforms(seed, step, purpose, idx, k=0):
    """rng.py:92-100"""
    return (hashes(seed, step, purpose, idx, k) >> np.uint64(11)).astype(np.float64) \
        * (1.0 / (1 << 53))


def uniform(seed, step, purpose, agent, k=0):
    """rng.py:84-89"""
    h = _fold_py(_fold_py(prefix(seed, step, purpose), int(agent)), int(k))
    return (h >> 11) * (1.0 / (1 << 53))
