"""Traffic ledger, worker groups and overflow diagnostics.

The reference meters every simulated hop (collectives.py:37-89, 177-263).  On B200 the
bytes really move (NCCL over NVLink, or in-HBM folds when workers are simulated on one
GPU), so the ledger is filled from the reference's closed forms: a ring all-reduce over
`length` elements charges each worker 2(n-1)*ceil(length/n)*bits sent and received
(collectives.py:209-233); an all-gather charges (n-1)*size_w sent and total-size_w
received (collectives.py:259-262); nothing is charged for a group of one.
"""

from __future__ import annotations

import math
from dataclasses import dataclass


@dataclass(frozen=True)
class WorkerGroup:
    """collectives.py:26-34."""

    size: int

    def __post_init__(self) -> None:
        if self.size < 1:
            raise ValueError("group size must be positive")


class TrafficLedger:
    """Bit counts per (phase, worker), split into sent and received (collectives.py:37-89)."""

    def __init__(self) -> None:
        self._cells: dict[tuple[str, int], list[int]] = {}

    def add(self, phase: str, worker: int, *, sent: int = 0, received: int = 0) -> None:
        if sent < 0 or received < 0:
            raise ValueError("bit counts must be non-negative")
        cell = self._cells.setdefault((phase, worker), [0, 0])
        cell[0] += sent
        cell[1] += received

    def bits_sent(self, worker: int | None = None, phase: str | None = None) -> int:
        return self._total(0, worker, phase)

    def bits_received(self, worker: int | None = None, phase: str | None = None) -> int:
        return self._total(1, worker, phase)

    def _total(self, slot, worker, phase) -> int:
        return sum(cell[slot] for (ph, w), cell in self._cells.items()
                   if (worker is None or w == worker) and (phase is None or ph == phase))

    def workers(self) -> list[int]:
        return sorted({w for _, w in self._cells})

    def phases(self) -> list[str]:
        return sorted({ph for ph, _ in self._cells})

    def max_egress_bits(self) -> int:
        ws = self.workers()
        return max((self.bits_sent(worker=w) for w in ws), default=0)

    def merge(self, other: "TrafficLedger") -> None:
        for (ph, w), cell in other._cells.items():
            self.add(ph, w, sent=cell[0], received=cell[1])

    def to_csv(self) -> str:
        lines = ["phase,worker,bits_sent,bits_received"]
        for key in sorted(self._cells):
            s, r = self._cells[key]
            lines.append(f"{key[0]},{key[1]},{s},{r}")
        return "\n".join(lines) + "\n"

    # closed-form charges ------------------------------------------------------
    def charge_ring(self, phase: str, n: int, length: int, element_bits: int, times: int = 1) -> None:
        """What ring_all_reduce charges (collectives.py:209-233); `times` identical rings at once."""
        if n <= 1:
            return
        per = 2 * (n - 1) * math.ceil(length / n) * element_bits * times
        for w in range(n):
            self.add(phase, w, sent=per, received=per)

    def charge_rings(self, phase: str, n: int, lengths, element_bits: int) -> None:
        """charge_ring for several ring all-reduces of one phase (one add per worker)."""
        if n <= 1:
            return
        per = sum(2 * (n - 1) * math.ceil(int(x) / n) * element_bits for x in lengths)
        for w in range(n):
            self.add(phase, w, sent=per, received=per)

    def charge_gather(self, phase: str, sizes) -> None:
        """What all_gather charges (collectives.py:253-262)."""
        n = len(sizes)
        if n <= 1:
            return
        total = sum(int(s) for s in sizes)
        for w, s in enumerate(sizes):
            self.add(phase, w, sent=(n - 1) * int(s), received=total - int(s))


@dataclass(frozen=True)
class OverflowStats:
    """metrics.py:40-46."""

    clip_events: int = 0
    total_adds: int = 0
    code_sigma: float = float("nan")


def overflow_rate(stats: OverflowStats) -> float:
    """metrics.py:49-53."""
    if stats.total_adds == 0:
        return 0.0
    return stats.clip_events / stats.total_adds
