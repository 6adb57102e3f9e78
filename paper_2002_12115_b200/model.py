"""Program model consumed by the hot path: loop tree + per-region variable facts.

This is the data the reference's front-end hands to its planner and evaluator
(acctuner/code_model.py: ``LoopInfo`` 664-674, ``LoopTable`` 677-702,
``RefFlags``/``VarEntry``/``VarRefTable`` 776-819).  Parsing C is outside the
hot path, so this package does not parse: it loads the
reference's canonical structural JSON (``dump_structural``, code_model.py:
1043-1074; format in SPEC.md "External Interfaces") with two optional
extensions that the reference's *source* path carries but its JSON drops:

* ``"index_var_keys"`` -- the loop-index variable keys excluded from planning
  (code_model.py:908-911).  Without them ``load_structural`` (1128-1129)
  matches bare names and would plan ``jacobi:i`` etc.;
* per-var ``"decl"`` -- declaration file (used for the file-rank rule).

The attribute names mirror the reference so that ``Planner`` (plan.py) runs
unchanged on either this model or a reference ``ProjectModel``.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field
from pathlib import Path
from typing import Iterable, Optional, Union

Region = Union[int, str]  # loop id | "pre" | "post" | "host:<n>"

SHAPES = ("single", "tight_outer", "tight_inner", "non_tight")


@dataclass
class LoopInfo:
    loop_id: int
    file_id: str
    span: tuple
    depth: int
    parent_loop: Optional[int]
    index_var: str
    trip_count_estimate: Optional[int]
    shape: str


class LoopTable:
    """Loops in id (document) order with parent links."""

    def __init__(self, loops: Iterable[LoopInfo]):
        self.loops = sorted(loops, key=lambda l: l.loop_id)
        self.by_id = {l.loop_id: l for l in self.loops}
        for l in self.loops:
            if l.parent_loop is not None and l.parent_loop not in self.by_id:
                raise ValueError(f"loop {l.loop_id}: unknown parent {l.parent_loop}")

    def __len__(self) -> int:
        return len(self.loops)

    def __iter__(self):
        return iter(self.loops)

    def get(self, loop_id: int) -> LoopInfo:
        return self.by_id[loop_id]

    def ancestors(self, loop_id: int) -> list[int]:
        """Self first, then each enclosing loop outward."""
        out = []
        cur: Optional[int] = loop_id
        while cur is not None:
            out.append(cur)
            cur = self.by_id[cur].parent_loop
        return out

    def children(self, loop_id: int) -> list[int]:
        return [l.loop_id for l in self.loops if l.parent_loop == loop_id]

    def top_level(self) -> list[LoopInfo]:
        return [l for l in self.loops if l.parent_loop is None]


@dataclass
class RefFlags:
    read: bool = False
    written: bool = False
    defined: bool = False


@dataclass
class VarEntry:
    key: str
    name: str
    scope: str                      # global | local | loop-local
    extents: Optional[list]         # None unknown, [] scalar, [n, ...] array
    refs: dict = field(default_factory=dict)   # Region -> RefFlags
    decl_file: Optional[str] = None

    @property
    def is_array(self) -> bool:
        return bool(self.extents)


class VarRefTable:
    def __init__(self, vars_: dict, region_sequence: list, index_var_keys: set):
        self.vars = vars_
        self.region_sequence = list(region_sequence)
        self.index_var_keys = set(index_var_keys)
        self._order = {r: i for i, r in enumerate(self.region_sequence)}

    def order(self, region: Region) -> int:
        return self._order[region]

    def plannable(self) -> list[VarEntry]:
        return [v for v in self.vars.values()
                if v.scope != "loop-local" and v.key not in self.index_var_keys]


@dataclass
class ProgramModel:
    """Loops + refs (+ the source text when known); the reference's ProjectModel role."""
    loops: LoopTable
    refs: VarRefTable
    sources: dict = field(default_factory=dict)   # file_id -> text (optional)

    @property
    def has_sources(self) -> bool:
        return bool(self.sources)


def _region_sequence(loops: LoopTable, file_rank: dict) -> list:
    """'pre', loops in document order with 'host:n' between top-level loops, 'post'.

    Same lexical rule as the reference (code_model.py:847-860, 1120-1127).
    """
    seq: list = ["pre"]
    n_top = 0
    for l in sorted(loops, key=lambda l: (file_rank.get(l.file_id, 0), l.span[0], l.loop_id)):
        if l.parent_loop is None:
            if n_top:
                seq.append(f"host:{n_top}")
            n_top += 1
        seq.append(l.loop_id)
    seq.append("post")
    return seq


def _parse_region(value) -> Region:
    if isinstance(value, int):
        return value
    if isinstance(value, str) and (value in ("pre", "post") or value.startswith("host:")):
        return value
    raise ValueError(f"bad region value: {value!r}")


def load_structural(doc: dict) -> ProgramModel:
    """Structural JSON (reference format, plus optional extensions) -> model."""
    loops = []
    file_rank = {}
    for rank, f in enumerate(doc["files"]):
        fid = f["file_id"]
        file_rank[fid] = rank
        for l in f.get("loops", []):
            shape = l.get("shape", "single")
            if shape not in SHAPES:
                raise ValueError(f"loop {l['loop_id']}: bad shape {shape!r}")
            loops.append(LoopInfo(int(l["loop_id"]), fid, tuple(l.get("span", (0, 0))), 0,
                                  l.get("parent"), l.get("index_var", ""),
                                  l.get("trip_count"), shape))
    table = LoopTable(loops)
    for l in table:
        l.depth = len(table.ancestors(l.loop_id)) - 1

    vars_: dict = {}
    for f in doc["files"]:
        for v in f.get("vars", []):
            key = v["name"]
            name = key.split(":", 1)[1] if ":" in key else key
            name = name.split("@", 1)[0]
            entry = VarEntry(key, name, v.get("scope", "global"),
                             list(v["extent"]) if "extent" in v else None,
                             decl_file=v.get("decl", f["file_id"]))
            for r in v.get("refs", []):
                flags = entry.refs.setdefault(_parse_region(r["region"]), RefFlags())
                flags.read |= bool(r.get("read"))
                flags.written |= bool(r.get("written"))
                flags.defined |= bool(r.get("defined"))
            vars_[key] = entry

    if "index_var_keys" in doc:
        index_keys = set(doc["index_var_keys"])
    else:  # reference rule for hand-written models (code_model.py:1128-1129)
        index_keys = {l.index_var for l in table if l.index_var and l.index_var in vars_}
    seq = _region_sequence(table, file_rank)
    sources = dict(doc.get("sources", {}))
    return ProgramModel(table, VarRefTable(vars_, seq, index_keys), sources)


def load_structural_file(path) -> ProgramModel:
    return load_structural(json.loads(Path(path).read_text()))


def dump_structural(model, include_index_keys: bool = True) -> dict:
    """Model (this package's or a reference ProjectModel) -> structural JSON."""
    loops = list(model.loops)
    refs = model.refs
    file_ids: list = []
    for l in loops:
        if l.file_id not in file_ids:
            file_ids.append(l.file_id)
    files = {fid: {"file_id": fid, "loops": [], "vars": []} for fid in file_ids}
    if not files:
        files["<model>"] = {"file_id": "<model>", "loops": [], "vars": []}
    for l in loops:
        shape = l.shape if isinstance(l.shape, str) else l.shape.value
        files[l.file_id]["loops"].append({
            "loop_id": l.loop_id, "span": list(l.span), "parent": l.parent_loop,
            "shape": shape, "index_var": l.index_var,
            "trip_count": l.trip_count_estimate})
    first = next(iter(files))
    for v in refs.vars.values():
        fid = v.decl_file if v.decl_file in files else first
        entry = {"name": v.key, "scope": v.scope,
                 "refs": [{"region": r, "read": f.read, "written": f.written,
                           "defined": f.defined}
                          for r, f in sorted(v.refs.items(), key=lambda kv: refs.order(kv[0]))]}
        if v.extents is not None:
            entry["extent"] = list(v.extents)
        files[fid]["vars"].append(entry)
    doc = {"files": list(files.values())}
    if include_index_keys:
        doc["index_var_keys"] = sorted(refs.index_var_keys)
    return doc
