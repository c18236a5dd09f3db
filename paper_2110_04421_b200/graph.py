"""Per-step union edge list (mirror of `pkg/src/epivec/graphs.py:30-51`).

`src`/`dst`/`kind` may be numpy arrays (reference-compatible) or CUDA torch
tensors (device-resident output of `GpuConfigRealizer.realize`); `.to_host()`
materialises numpy copies.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class StepGraph:
    step: int
    src: object     # int32[E]
    dst: object     # int32[E]
    kind: object    # int8[E]  (0 household, 1 occupation, 2 random)

    @property
    def n_edges(self) -> int:
        return int(self.src.shape[0])

    @property
    def on_device(self) -> bool:
        return not isinstance(self.src, np.ndarray)

    def to_host(self) -> "StepGraph":
        if not self.on_device:
            return self
        return StepGraph(self.step, self.src.cpu().numpy(), self.dst.cpu().numpy(),
                         self.kind.cpu().numpy())

    def kind_counts(self) -> np.ndarray:
        return np.bincount(np.asarray(self.to_host().kind), minlength=3)

    def sorted_canonical(self) -> "StepGraph":
        """Edges in canonical (dst, src, kind) order (host)."""
        g = self.to_host()
        order = np.lexsort((g.kind, g.src, g.dst))
        return StepGraph(g.step, g.src[order], g.dst[order], g.kind[order])

    @classmethod
    def empty(cls, step: int) -> "StepGraph":
        return cls(step, np.empty(0, np.int32), np.empty(0, np.int32), np.empty(0, np.int8))
