"""Per-component FLOP ledger (the part of ``bayermc.metrics`` that
``run_sequence`` returns; metrics.py:14-67).  Host-side bookkeeping only."""

from __future__ import annotations

import json

COMPONENTS = ("backbone", "fme", "mv_refine", "cabr", "prediction")


class FlopLedger:
    """Non-negative FLOP tallies per component; "prediction" is pinned to 0."""

    def __init__(self, counts: dict | None = None):
        self._counts = dict.fromkeys(COMPONENTS, 0)
        for name, value in (counts or {}).items():
            self.add(name, value)

    def add(self, component: str, flops: int) -> None:
        if component not in self._counts:
            raise ValueError(f"unknown component {component!r}; expected one of {COMPONENTS}")
        flops = int(flops)
        if flops < 0:
            raise ValueError("flop counts are non-negative")
        if component == "prediction" and flops:
            raise ValueError("prediction performs no floating-point work; its entry stays 0")
        self._counts[component] += flops

    def __getitem__(self, component: str) -> int:
        return self._counts[component]

    @property
    def total(self) -> int:
        return sum(self._counts.values())

    def as_dict(self) -> dict:
        return {**self._counts, "total": self.total}

    def to_json(self) -> str:
        return json.dumps(self.as_dict(), indent=1)

    @classmethod
    def from_json(cls, text: str) -> "FlopLedger":
        doc = json.loads(text)
        doc.pop("total", None)
        return cls(counts=doc)

    def table(self) -> str:
        rows = [(n, f"{self._counts[n] / 1e9:.6f}") for n in COMPONENTS] + [("total", f"{self.total / 1e9:.6f}")]
        width = max(len(n) for n, _ in rows + [("component", "")]) + 2
        lines = [f"{'component':<{width}}GFLOPs", "-" * (width + 6)]
        lines += [f"{n:<{width}}{v}" for n, v in rows]
        return "\n".join(lines)
