"""Execution-strategy descriptors of the reference's kernel variants.

Only the part of /root/reference/pkg/src/fvbatch/itspace.py that the
patch-update boundary consumes: `ExecutionStrategy` (itspace.py:28-49) and its
label parser (itspace.py:56-60).  On the device the strategy does not change
the arithmetic (all variants are bitwise identical); it is kept because it
fixes which error the reference reports first when several patches hold
non-physical states (the number of host patch chunks, vectorized.py:234-256).
The host loop machinery (IndexSpace, for_each, reduce_max) is replaced by the
CUDA grid and is not rebuilt.
"""

from __future__ import annotations

import os
from dataclasses import dataclass
from enum import Enum

from .errors import ContractViolationError

WORKER_ENV_VAR = "FVBATCH_WORKERS"


class StrategyKind(Enum):
    SEQUENTIAL = "seq"
    PARALLEL_UNORDERED = "par"


@dataclass(frozen=True)
class ExecutionStrategy:
    """How the reference drives a loop; `workers()` follows itspace.py:43-49."""

    kind: StrategyKind
    worker_hint: int | None = None

    @property
    def label(self) -> str:
        return self.kind.value

    def workers(self) -> int:
        if self.worker_hint is not None:
            return max(1, self.worker_hint)
        env = os.environ.get(WORKER_ENV_VAR)
        if env:
            return max(1, int(env))
        return os.cpu_count() or 1


SEQUENTIAL = ExecutionStrategy(StrategyKind.SEQUENTIAL)
PARALLEL = ExecutionStrategy(StrategyKind.PARALLEL_UNORDERED)


def strategy_from_label(label: str, worker_hint: int | None = None) -> ExecutionStrategy:
    for kind in StrategyKind:
        if kind.value == label:
            return ExecutionStrategy(kind, worker_hint)
    raise ContractViolationError(f"unknown strategy label {label!r}")


def strategy_kind_of(strategy) -> StrategyKind:
    """Accept this module's strategies and the reference's (duck-typed on `.kind.value`)."""
    label = getattr(getattr(strategy, "kind", None), "value", None)
    for kind in StrategyKind:
        if kind.value == label:
            return kind
    raise ContractViolationError(f"unrecognised execution strategy {strategy!r}")
