"""Directive kinds and the genome index space (acctuner/classify.py:24-35, 328-334).

Each eligible loop carries exactly one kind, fixed before the search; the
genome only toggles whether that loop runs on the device.  On the B200 path
the kind selects the kernel *variant* the native executor launches for the
loop (csrc/kernels.cu):

* ``kernels`` on a tight-nest outer loop -> the whole tight nest below it is
  collapsed into one launch (3-D box for i-loops, 2-D plane for j-loops);
* ``parallel loop`` on an innermost loop -> one gang-parallel row launch per
  host iteration of the enclosing loops; on the non-tight time loop (loop 6)
  -> the device-resident time loop;
* ``parallel loop vector`` -> a single-CTA vector-only strip loop.
"""

from __future__ import annotations

from enum import Enum


class DirectiveKind(Enum):
    KERNELS = "kernels"
    PARALLEL_LOOP = "parallel loop"
    PARALLEL_LOOP_VECTOR = "parallel loop vector"

    @property
    def pragma(self) -> str:
        return f"#pragma acc {self.value}"

    @property
    def native_code(self) -> int:
        """Value of ``hp_kind`` in include/himeno_b200.h."""
        return _NATIVE[self]


_NATIVE = {DirectiveKind.KERNELS: 1, DirectiveKind.PARALLEL_LOOP: 2,
           DirectiveKind.PARALLEL_LOOP_VECTOR: 3}


def _kind_of(value) -> "DirectiveKind | None":
    if value is None:
        return None
    if isinstance(value, DirectiveKind):
        return value
    return DirectiveKind(getattr(value, "value", value))


def eligible_ids(verdicts) -> list:
    """i-th eligible loop in document order is gene i (classify.py:328-330).

    Accepts reference ``EligibilityVerdict`` objects or their JSON dicts.
    """
    out = []
    for v in verdicts:
        kind = v["kind"] if isinstance(v, dict) else v.kind
        lid = v["loop_id"] if isinstance(v, dict) else v.loop_id
        if kind is not None:
            out.append(int(lid))
    return out


def kind_map(verdicts) -> dict:
    out = {}
    for v in verdicts:
        kind = v["kind"] if isinstance(v, dict) else v.kind
        lid = v["loop_id"] if isinstance(v, dict) else v.loop_id
        if kind is not None:
            out[int(lid)] = _kind_of(kind)
    return out
