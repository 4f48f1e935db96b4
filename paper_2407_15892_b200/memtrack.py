"""Host-side mirror of the reference's memory tracker and op counters
(/root/reference/proj/include/minitrain/memtrack.hpp), fed by libmst.

The C ABI reports two streams (include/mst/mst.h, "memtrack"):
  * memory events — alloc/free of the chunk buffers a call carves from its
    workspace, with the reference's label classes ("inter.mlp.*",
    "inter.head.*", "act.*"), in logical-lifetime order;
  * op counts — count_matmul / count_op under the counting conventions of
    memtrack.hpp:19-35.
`MemTracker` reproduces MemTracker's semantics (memtrack.hpp:138-228):
live / per-label accounting, StateError on over-free (:160-163), nested
regions with entry snapshots (:177-197), and `MemReport`'s peak replays
(:62-134); `export_timeline` writes the CSV of memtrack.hpp:277-284.  It is
pinned against the reference compiled here (tests/test_memtrack.py, golden
tests/golden/reference_rng_memtrack.json "memtrack_script").
"""
from __future__ import annotations

import io
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional, TextIO, Union


class StateError(RuntimeError):
    """minitrain::StateError (error.hpp) raised by the tracker."""


@dataclass
class MemEvent:  # memtrack.hpp:41-47
    seq_no: int
    kind: str  # "alloc" | "free"
    bytes: int
    label: str
    live_after: int


@dataclass
class OpCounters:  # memtrack.hpp:49-60
    flops: int = 0
    matmul_flops: int = 0
    hbm_elements: int = 0
    weight_read_elements: int = 0

    def __sub__(self, o: "OpCounters") -> "OpCounters":
        return OpCounters(self.flops - o.flops, self.matmul_flops - o.matmul_flops,
                          self.hbm_elements - o.hbm_elements, self.weight_read_elements - o.weight_read_elements)

    def copy(self) -> "OpCounters":
        return OpCounters(self.flops, self.matmul_flops, self.hbm_elements, self.weight_read_elements)

    def as_tuple(self) -> tuple:
        return (self.flops, self.matmul_flops, self.hbm_elements, self.weight_read_elements)


@dataclass
class MemReport:  # memtrack.hpp:62-134
    events: List[MemEvent] = field(default_factory=list)
    entry_live: int = 0
    entry_live_by_label: Dict[str, int] = field(default_factory=dict)

    def peak_bytes(self) -> int:
        return max((e.live_after for e in self.events), default=0)

    def final_live(self) -> int:
        return self.events[-1].live_after if self.events else self.entry_live

    def peak_by_label(self) -> Dict[str, int]:
        live = dict(self.entry_live_by_label)
        at_peak = dict(live)
        peak = 0
        for e in self.events:
            live[e.label] = live.get(e.label, 0) + (e.bytes if e.kind == "alloc" else -e.bytes)
            if e.live_after > peak:
                peak = e.live_after
                at_peak = dict(live)
        return {k: v for k, v in sorted(at_peak.items()) if v != 0}

    def _replay_peak(self, match: Callable[[str], bool]) -> int:
        live = sum(b for lab, b in self.entry_live_by_label.items() if match(lab))
        peak = live
        for e in self.events:
            if match(e.label):
                live += e.bytes if e.kind == "alloc" else -e.bytes
                peak = max(peak, live)
        return peak

    def peak_for_prefix(self, prefix: str) -> int:
        return self._replay_peak(lambda lab: lab.startswith(prefix))

    def peak_excluding_prefix(self, prefix: str) -> int:
        return self._replay_peak(lambda lab: not lab.startswith(prefix))


@dataclass
class RegionStats:
    report: MemReport
    counters: OpCounters


class MemTracker:  # memtrack.hpp:138-228
    def __init__(self) -> None:
        self._events: List[MemEvent] = []
        self._live_by_label: Dict[str, int] = {}
        self._live = 0
        self._seq = 0
        self._ctr = OpCounters()
        self._open: list = []

    def on_alloc(self, nbytes: int, label: str) -> None:
        self._live += nbytes
        self._live_by_label[label] = self._live_by_label.get(label, 0) + nbytes
        self._events.append(MemEvent(self._seq, "alloc", nbytes, label, self._live))
        self._seq += 1

    def on_free(self, nbytes: int, label: str) -> None:
        cur = self._live_by_label.get(label)
        if cur is None or cur < nbytes:
            raise StateError(f"free exceeds live allocations for label '{label}'")
        self._live_by_label[label] = cur - nbytes
        self._live -= nbytes
        self._events.append(MemEvent(self._seq, "free", nbytes, label, self._live))
        self._seq += 1

    def count_matmul(self, n: int, k: int, p: int, weight_elems: int = 0) -> None:
        if not (n > 0 and k > 0 and p > 0):
            raise RuntimeError("count_matmul: extents must be positive")
        f = 2 * n * k * p
        self._ctr.flops += f
        self._ctr.matmul_flops += f
        self._ctr.hbm_elements += n * k + k * p + n * p
        self._ctr.weight_read_elements += weight_elems

    def count_op(self, flops: int, hbm_elements: int) -> None:
        self._ctr.flops += flops
        self._ctr.hbm_elements += hbm_elements

    def region_begin(self, name: str) -> None:
        self._open.append((name, len(self._events), self._live, dict(self._live_by_label), self._ctr.copy()))

    def region_end(self, name: str) -> RegionStats:
        if not self._open:
            raise StateError(f"region_end('{name}') without begin")
        if self._open[-1][0] != name:
            raise StateError(f"region_end('{name}') does not match open region '{self._open[-1][0]}'")
        _, start, live, by_label, ctr = self._open.pop()
        rep = MemReport(list(self._events[start:]), live, by_label)
        return RegionStats(rep, self._ctr - ctr)

    def live_bytes(self) -> int:
        return self._live

    def live_bytes_for_label(self, label: str) -> int:
        return self._live_by_label.get(label, 0)

    def totals(self) -> OpCounters:
        return self._ctr.copy()

    def open_regions(self) -> int:
        return len(self._open)


def export_timeline(report: MemReport, out: Union[str, TextIO]) -> Optional[str]:
    """CSV `seq_no,kind,bytes,label,live_after` (memtrack.hpp:277-291).  With a
    path, writes the file; with a stream, writes into it; returns the text."""
    buf = io.StringIO()
    buf.write("seq_no,kind,bytes,label,live_after\n")
    for e in report.events:
        buf.write(f"{e.seq_no},{e.kind},{e.bytes},{e.label},{e.live_after}\n")
    text = buf.getvalue()
    if isinstance(out, str):
        with open(out, "w") as f:
            f.write(text)
    else:
        out.write(text)
    return text
