"""WarpConfig: the reference's lane-count / element-size configuration.

Mirrors warp.py:41-58 of the reference.  On the B200 the emulator itself is
replaced by real sm_100a warps; the configuration survives because W (the
block width and the `doc mod W` reconstruction choice) is part of the
arithmetic the kernels reproduce.  The device supports W in {2,4,8,16,32,64}.
"""

from __future__ import annotations

from dataclasses import dataclass


def _is_pow2(x: int) -> bool:
    return x > 0 and (x & (x - 1)) == 0


class OutOfBoundsError(IndexError):
    """A lane addressed outside a global array (warp.py:33-34, raised by
    GlobalArray2D._check, warp.py:234-240).  The device path raises it once,
    before any launch, for word ids outside [0, V) of phi."""


@dataclass(frozen=True)
class WarpConfig:
    lanes: int = 32  # W, power of 2
    elem_size: int = 4  # bytes per element
    line_size: int = 128  # bytes per memory transaction segment

    def __post_init__(self):
        if not _is_pow2(self.lanes) or not 2 <= self.lanes <= 64:
            raise ValueError(f"lane count must be a power of 2 in [2, 64], got {self.lanes}")
        if self.elem_size not in (4, 8):
            raise ValueError(f"elem_size must be 4 or 8, got {self.elem_size}")
        ratio, rem = divmod(self.line_size, self.elem_size)
        if rem or not _is_pow2(ratio):
            raise ValueError("line_size must be a power-of-2 multiple of elem_size")

    @property
    def log2_lanes(self) -> int:
        return self.lanes.bit_length() - 1


class Trace:
    """Accepted for signature compatibility (kernels.py:487-497); stays empty.

    The emulator's transaction trace is replaced by ncu counters on the real
    device (profiles/).  `events` is empty and op totals are zero.
    """

    def __init__(self):
        self.events = []

    def op_total(self, op: str, phase: str | None = None) -> int:
        return 0

    def merge(self, other: "Trace") -> None:
        self.events.extend(other.events)
