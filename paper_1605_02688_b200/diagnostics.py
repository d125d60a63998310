"""Run-time NaN guard on the device (reference
``diagnostics.py:28-88``, hooked per node at ``runtime.py:359-367``).

Same contract: with ``compile(..., nan_guard=NanGuardConfig())`` every
float input and output of every node is scanned for NaN, infinity or
magnitudes above ``big_threshold``; the first offending node (in execution
order; inputs before outputs, as the reference scans them) raises
``NanDetected`` with a :class:`NanReport`, and the call leaves shared state
untouched.

On the device the scans are kernels (``tx_check_values``) appended after
each node's launch inside the captured step; each ORs flag bits into its own
slot of a device word array, read once after the step.  To make the report
(and atomicity) exact, a guarded function plans every intermediate into its
own buffer (no arena reuse, no in-place kernels, no row fusion — the
reference's guard also sees every node), writes updates only after the
check passes, and builds the value summary from the flagged tensor itself.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class NanGuardConfig:
    check_nan: bool = True
    check_inf: bool = True
    big_threshold: float = 1e10

    def mode(self) -> int:
        return (1 if self.check_nan else 0) | (2 if self.check_inf else 0) | (4 if self.big_threshold is not None else 0)


@dataclass
class NanReport:
    node_id: int
    op: str
    check: str       # "nan" | "inf" | "big"
    tensor: str      # e.g. "input 0" / "output 1"
    trace: str
    value_summary: str

    def __str__(self):
        return (f"{self.check} detected at node {self.node_id} ({self.op}), {self.tensor}; "
                f"created at {self.trace or '<unknown>'}; {self.value_summary}")


def summarize(arr: np.ndarray) -> str:
    finite = arr[np.isfinite(arr)]
    lo = finite.min() if finite.size else float("nan")
    hi = finite.max() if finite.size else float("nan")
    return f"shape {arr.shape}, finite range [{lo}, {hi}]"


def check_name(bits: int) -> str:
    return "nan" if bits & 1 else "inf" if bits & 2 else "big"
