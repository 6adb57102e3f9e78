"""Generic B200 executor generator: a C-subset program -> one CUDA translation unit.

The hand-written Himeno library (csrc/) covers the headline application.  Any
other program the reference can tune (its parser's C subset, acctuner/
code_model.py:1-12) goes through this generator instead, which does at build
time what an OpenACC compiler does for every directive the gene can select
(emitter.py:132-228 inserts them, PGI compiles them):

* the program becomes a C++ struct ``Prog``: globals are members (one instance
  per device context, zeroed before each run like a fresh process's statics),
  functions are member functions with their bodies unchanged -- except that
  every ``for`` statement (loop id L, reference numbering) is wrapped as

      { R.before(L); if (R.dev(L)) { <launch of k_L> } else for (...) ...; R.after(L); }

  so one compiled program runs any gene pattern: gene = 0 loops execute the
  original host code, gene = 1 loops launch their kernel, and the transfer
  plan's events fire at the loop hooks (runtime: csrc/gen_runtime.cuh);
* each eligible loop gets one sm_100a kernel ``k_L`` whose body is the loop's
  own source text over device arrays of the same names.  Directive kinds map
  to launches as OpenACC compilers map them: ``kernels`` collapses the tight
  rectangular nest below L into one grid (a loop with a loop-carried scalar
  runs as one sequential device thread, as an auto-parallelising compiler
  leaves it); a loop that is not collapsed runs as gangs (one thread block per
  iteration) whose innermost parallelisable loops -- with a tight independent
  parent folded in -- are vector loops over the block's threads (a barrier after
  each, or, when nothing they write is read in the gang, spread over several
  blocks per gang); ``parallel loop vector`` runs in one thread block.  Scalars
  are firstprivate kernel arguments; ``s = s + e`` / ``s += e`` accumulations
  are reductions (fp64 block partials, folded in block order on the host);
* every launch reports the boxes it writes and every host-executed loop the
  boxes its own statements wrote (computed from the loop bounds), so the
  runtime's transfers move only what changed.

Parsing is limited to what the generator needs (declarations, function
headers, ``for`` headers, identifier use); loop ids, spans, nesting and shapes
come from the reference's own front-end (the committed program model).
"""

from __future__ import annotations

import re
from dataclasses import dataclass, field
from typing import Optional

TYPE_WORDS = ("void", "int", "long", "short", "char", "float", "double", "unsigned", "signed")
KEYWORDS = set(TYPE_WORDS) | {"static", "const", "register", "for", "while", "if", "else",
                              "return", "break", "continue", "sizeof"}

_TOKEN = re.compile(r"""
    (?P<ws>\s+|//[^\n]*|/\*.*?\*/)
  | (?P<num>(?:\d+\.\d*|\.\d+|\d+)(?:[eE][+-]?\d+)?[uUlLfF]*)
  | (?P<name>[A-Za-z_]\w*)
  | (?P<str>"(?:\\.|[^"\\])*")
  | (?P<chr>'(?:\\.|[^'\\])*')
  | (?P<punct><<=|>>=|\+\+|--|\+=|-=|\*=|/=|%=|==|!=|<=|>=|&&|\|\||<<|>>|[-+*/%<>=!&|^~?:;,()\[\]{}.])
""", re.S | re.X)


@dataclass
class Tok:
    kind: str
    text: str
    pos: int


def tokenize(text: str) -> list:
    out, i = [], 0
    while i < len(text):
        m = _TOKEN.match(text, i)
        if not m:
            raise ValueError(f"codegen: cannot tokenize at {i}: {text[i:i + 20]!r}")
        if m.lastgroup != "ws":
            out.append(Tok(m.lastgroup, m.group(), i))
        i = m.end()
    return out


@dataclass
class Decl:
    name: str
    ctype: str
    dims: list            # [] scalar

    @property
    def is_array(self) -> bool:
        return bool(self.dims)

    def elems(self) -> int:
        n = 1
        for d in self.dims:
            n *= d
        return n


@dataclass
class Func:
    name: str
    ret: str
    params: list          # [Decl]
    body: tuple           # (start, end) of "{ ... }"
    locals: list = field(default_factory=list)

    def scalar(self, name: str) -> Optional[Decl]:
        for d in self.params + self.locals:
            if d.name == name:
                return d
        return None


def _match(toks, i, close):
    opener = toks[i].text
    depth = 0
    for j in range(i, len(toks)):
        if toks[j].text == opener:
            depth += 1
        elif toks[j].text == close:
            depth -= 1
            if depth == 0:
                return j
    raise ValueError(f"codegen: unbalanced {opener!r}")


def _declarators(toks, i, ctype):
    """Parse `a, b[3][4], c;` starting at i; returns ([Decl], index after ';')."""
    out = []
    while True:
        name = toks[i].text
        i += 1
        dims = []
        while toks[i].text == "[":
            dims.append(int(toks[i + 1].text.rstrip("uUlL")))
            i += 3
        if toks[i].text == "=":
            raise ValueError(f"codegen: initialised declaration of {name} is not supported")
        out.append(Decl(name, ctype, dims))
        if toks[i].text == ";":
            return out, i + 1
        if toks[i].text != ",":
            raise ValueError(f"codegen: bad declaration near {name}")
        i += 1


class CProgram:
    """Globals and functions of a C-subset program text."""

    def __init__(self, text: str):
        self.text = text
        self.toks = tokenize(text)
        self.globals: list = []
        self.funcs: list = []
        toks, i = self.toks, 0
        while i < len(toks):
            j = i
            while toks[j].text in ("static", "const", "register"):
                j += 1
            tparts = []
            while toks[j].kind == "name" and toks[j].text in TYPE_WORDS:
                tparts.append(toks[j].text)
                j += 1
            if not tparts:
                raise ValueError(f"codegen: expected a declaration at {toks[i].pos}")
            ctype = " ".join(tparts)
            if toks[j + 1].text == "(":
                name = toks[j].text
                close = _match(toks, j + 1, ")")
                params = []
                k = j + 2
                while k < close:
                    ptype = []
                    while toks[k].text in TYPE_WORDS:
                        ptype.append(toks[k].text)
                        k += 1
                    if ptype == ["void"] and k == close:
                        break
                    params.append(Decl(toks[k].text, " ".join(ptype), []))
                    k += 1
                    if toks[k].text == ",":
                        k += 1
                b0 = close + 1
                b1 = _match(toks, b0, "}")
                f = Func(name, ctype, params, (toks[b0].pos, toks[b1].pos + 1))
                self._locals(f, b0, b1)
                self.funcs.append(f)
                i = b1 + 1
            else:
                decls, i = _declarators(toks, j, ctype)
                self.globals.extend(decls)
        self.gmap = {d.name: d for d in self.globals}

    def _locals(self, f: Func, b0: int, b1: int):
        toks, k, depth = self.toks, b0 + 1, 1
        while k < b1:
            t = toks[k].text
            if t == "{":
                depth += 1
            elif t == "}":
                depth -= 1
            if depth == 1 and toks[k].kind == "name" and t in TYPE_WORDS and \
                    (k == b0 + 1 or toks[k - 1].text in (";", "{", "}")):
                tparts = []
                while toks[k].text in TYPE_WORDS:
                    tparts.append(toks[k].text)
                    k += 1
                decls, k = _declarators(toks, k, " ".join(tparts))
                if any(d.is_array for d in decls):
                    raise ValueError(f"codegen: local arrays in {f.name} are not supported")
                f.locals.extend(decls)
                continue
            k += 1

    def func_at(self, pos: int) -> Func:
        for f in self.funcs:
            if f.body[0] <= pos < f.body[1]:
                return f
        raise ValueError(f"codegen: position {pos} is outside every function")

    def toks_in(self, a: int, b: int) -> list:
        return [t for t in self.toks if a <= t.pos < b]


# ---------------------------------------------------------------------------- loops

@dataclass
class Header:
    var: str
    lo: str               # C expression
    hi: str               # exclusive upper bound expression
    step: int
    body: tuple           # (start, end) of the body statement


def parse_header(prog: CProgram, span) -> Optional[Header]:
    """`for(v = lo; v < hi | v <= hi; v++ | ++v | v += c | v = v + c) body`."""
    a, b = span
    toks = prog.toks_in(a, b)
    if not toks or toks[0].text != "for" or toks[1].text != "(":
        return None
    close = _match(toks, 1, ")")
    parts, cur = [], []
    for t in toks[2:close]:
        if t.text == ";" and len(parts) < 2:
            parts.append(cur)
            cur = []
        else:
            cur.append(t)
    parts.append(cur)
    if len(parts) != 3:
        return None
    init, cond, step = parts
    if len(init) < 3 or init[0].kind != "name" or init[1].text != "=":
        return None
    var = init[0].text
    lo = prog.text[init[2].pos:init[-1].pos + len(init[-1].text)]
    if len(cond) < 3 or cond[0].text != var or cond[1].text not in ("<", "<="):
        return None
    hi = prog.text[cond[2].pos:cond[-1].pos + len(cond[-1].text)]
    if cond[1].text == "<=":
        hi = f"({hi}) + 1"
    st = [t.text for t in step]
    if st in ([var, "++"], ["++", var]):
        inc = 1
    elif len(st) == 3 and st[0] == var and st[1] == "+=" and step[2].kind == "num":
        inc = int(st[2])
    elif len(st) == 5 and st[0] == var and st[1] == "=" and st[2] == var and st[3] == "+" \
            and step[4].kind == "num":
        inc = int(st[4])
    else:
        return None
    if inc <= 0:
        return None
    body_start = toks[close + 1].pos
    return Header(var, lo, hi, inc, (body_start, b))


def _idents(toks) -> list:
    return [t.text for t in toks if t.kind == "name" and t.text not in KEYWORDS]


def _writes(toks) -> dict:
    """name -> list of write kinds ('=', '+=', '++', ...) for plain-name targets."""
    out: dict = {}
    for k, t in enumerate(toks):
        if t.kind != "name":
            continue
        nxt = toks[k + 1].text if k + 1 < len(toks) else ""
        prv = toks[k - 1].text if k else ""
        if nxt in ("=", "+=", "-=", "*=", "/=", "%=", "<<=", ">>=") or nxt in ("++", "--") \
                or prv in ("++", "--"):
            if prv == "." or nxt == "[":
                continue
            op = nxt if nxt in ("=", "+=", "-=", "*=", "/=", "%=", "<<=", ">>=", "++", "--") else prv
            out.setdefault(t.text, []).append((k, op))
    return out


def _is_reduction(toks, name: str) -> bool:
    """Every occurrence of `name` is `name = name + e` / `name += e` with no other use."""
    occ = [k for k, t in enumerate(toks) if t.kind == "name" and t.text == name]
    used = set()
    ok = False
    for i in occ:
        if i in used:
            continue
        nxt = toks[i + 1].text if i + 1 < len(toks) else ""
        if nxt == "+=":
            end = i + 2
            while toks[end].text != ";":
                if toks[end].text == name:
                    return False
                end += 1
            used.add(i)
            ok = True
        elif nxt == "=" and i + 3 < len(toks) and toks[i + 2].text == name \
                and toks[i + 3].text == "+":
            end = i + 4
            while toks[end].text != ";":
                if toks[end].text == name:
                    return False
                end += 1
            used.update((i, i + 2))
            ok = True
        else:
            return False
    return ok


@dataclass
class KernelPlan:
    loop: int
    func: Func
    levels: list          # [Header] mapped to the grid (outermost first)
    body: tuple           # (start, end) of the innermost mapped body
    arrays: list          # global arrays used (names)
    arrays_written: list
    params: list          # [Decl] firstprivate scalars: read-only or read before written
    privates: list        # [Decl] outer scalars written in the body (kernel locals)
    reductions: list      # [Decl]
    carried: list         # [Decl] read-before-write outer scalars (sequential for kernels)
    mode: str             # "grid" | "gang" | "block" | "seq"
    note: str = ""
    vec: list = field(default_factory=list)   # [(LoopInfo, Header)] vector (thread) loops
    vsplit: bool = False  # vector loops may spread over several blocks per gang (no barriers)
    write_refs: dict = field(default_factory=dict)   # array -> [[subscript tokens] per dim]


def _vector_leaves(prog: CProgram, loop, loops, kinds) -> list:
    """Innermost loops below `loop` that a compiler would run as vector loops inside a
    gang: leaves of the loop tree, classified parallelisable themselves, with a
    recognised header and no loop-carried scalar or reduction."""
    out = []

    def walk(lid):
        kids = loops.children(lid)
        if not kids:
            if lid == loop.loop_id or kinds.get(lid) is None:
                return
            leaf = loops.get(lid)
            h = parse_header(prog, leaf.span)
            if h is None:
                return
            kp = plan_kernel(prog, leaf, "parallel loop", loops)
            if kp is None or kp.carried or kp.reductions:
                return
            # a parent whose body is exactly this loop, rectangular and free of
            # carried scalars and output dependences, joins the vector region: its
            # iterations and the leaf's are spread over the threads together
            region, hs = leaf, [h]
            par = loops.get(leaf.parent_loop) if leaf.parent_loop is not None else None
            if par is not None and par.loop_id != loop.loop_id and par.shape == "tight_outer" \
                    and loops.children(par.loop_id) == [lid]:
                ph = parse_header(prog, par.span)
                pkp = plan_kernel(prog, par, "parallel loop", loops) if ph else None
                bound_names = set(_idents(tokenize(h.lo))) | set(_idents(tokenize(h.hi)))
                if ph is not None and pkp is not None and not pkp.carried and \
                        not pkp.reductions and not shared_writes(prog, par) and \
                        ph.var not in bound_names:
                    region, hs = par, [ph, h]
            out.append((region, hs))
            return
        for c in kids:
            walk(c)

    walk(loop.loop_id)
    return out


def plan_kernel(prog: CProgram, loop, kind: str, loops, kinds=None) -> Optional[KernelPlan]:
    """How loop `loop` (model LoopInfo) runs on the device under directive `kind`.

    With the program's classification (``kinds``), a loop that is not collapsed into
    the grid runs as OpenACC compilers run a gang loop with parallelisable inner
    loops: one thread block per iteration of the loop (gang), the innermost
    parallelisable loops spread over the block's threads (vector, a barrier after
    each), everything between them executed redundantly by every thread."""
    h = parse_header(prog, loop.span)
    if h is None:
        return None
    func = prog.func_at(loop.span[0])
    levels, body = [h], h.body
    if kind == "kernels":
        cur = loop
        chain_vars = {h.var}
        while cur.shape == "tight_outer" and len(levels) < 3:
            kids = loops.children(cur.loop_id)
            if len(kids) != 1:
                break
            child = loops.get(kids[0])
            ch = parse_header(prog, child.span)
            if ch is None:
                break
            bound_names = set(_idents(tokenize(ch.lo))) | set(_idents(tokenize(ch.hi)))
            if bound_names & chain_vars:
                break          # triangular: keep the inner loop inside the thread
            levels.append(ch)
            chain_vars.add(ch.var)
            body = ch.body
            cur = child
    body_toks = prog.toks_in(*h.body)
    names = _idents(body_toks)
    arrays = sorted({n for n in names if n in prog.gmap and prog.gmap[n].is_array})
    writes = _writes(body_toks)
    arr_written = []
    write_refs: dict = {}
    for k, t in enumerate(body_toks):
        if t.kind == "name" and t.text in arrays:
            # a[..][..] = / += / ++ : find the end of the subscript chain
            j = k + 1
            subs = []
            while j < len(body_toks) and body_toks[j].text == "[":
                depth, j0 = 0, j
                while True:
                    if body_toks[j].text == "[":
                        depth += 1
                    elif body_toks[j].text == "]":
                        depth -= 1
                        if depth == 0:
                            break
                    j += 1
                subs.append(body_toks[j0 + 1:j])
                j += 1
            if j < len(body_toks) and body_toks[j].text in ("=", "+=", "-=", "*=", "/=", "++", "--"):
                arr_written.append(t.text)
                write_refs.setdefault(t.text, []).append(subs)
    level_vars = {lv.var for lv in levels}
    params, privates, reds, carried = [], [], [], []
    seen = set()
    for n in names:
        if n in seen or n in level_vars:
            continue
        seen.add(n)
        d = func.scalar(n) or (prog.gmap.get(n) if n in prog.gmap and not prog.gmap[n].is_array
                               else None)
        if d is None:
            continue
        if n in writes:
            if _is_reduction(body_toks, n):
                reds.append(d)
                continue
            privates.append(d)
            first = next(k for k, t in enumerate(body_toks) if t.kind == "name" and t.text == n)
            if first not in [k for k, _ in writes[n]] or writes[n][0][1] != "=":
                carried.append(d)
                params.append(d)
            continue
        params.append(d)
    mode = "grid"
    note = ""
    if kind == "parallel loop vector":
        mode = "block"
    if carried and kind == "kernels":
        mode = "seq"
        levels = [h]
        body = h.body
        note = "loop-carried scalar " + ", ".join(d.name for d in carried)
    vec = []
    vsplit = False
    if mode == "grid" and len(levels) == 1 and kinds is not None and not reds:
        vec = _vector_leaves(prog, loop, loops, kinds)
        if vec:
            mode = "gang"
            # vector regions: a leaf loop id, or "parent+" when its parent joined it
            note = "vector " + ",".join(f"{r.loop_id}{'+' if len(hs) > 1 else ''}"
                                        for r, hs in vec)
            # the vector loops need no block barrier when nothing the gang reads is
            # written by a vector loop: then a gang's vector iterations may also be
            # spread over several blocks (a 2-D grid), so a gang loop with few
            # iterations (late FFT stages) still fills the GPU
            leaf_written = set()
            for leaf, _ in vec:
                lt = prog.toks_in(*leaf.span)   # (the vector region: leaf or its parent)
                for k, t in enumerate(lt):
                    if t.kind == "name" and t.text in prog.gmap and prog.gmap[t.text].is_array:
                        j = k + 1
                        while j < len(lt) and lt[j].text == "[":
                            depth = 0
                            while True:
                                if lt[j].text == "[":
                                    depth += 1
                                elif lt[j].text == "]":
                                    depth -= 1
                                    if depth == 0:
                                        break
                                j += 1
                            j += 1
                        if j < len(lt) and lt[j].text in ("=", "+=", "-=", "*=", "/=", "++", "--"):
                            leaf_written.add(t.text)
            read_anywhere = set()
            for k, t in enumerate(body_toks):
                if t.kind == "name" and t.text in leaf_written:
                    # any occurrence that is not a pure store target counts as a read
                    j = k + 1
                    while j < len(body_toks) and body_toks[j].text == "[":
                        depth = 0
                        while True:
                            if body_toks[j].text == "[":
                                depth += 1
                            elif body_toks[j].text == "]":
                                depth -= 1
                                if depth == 0:
                                    break
                            j += 1
                        j += 1
                    if not (j < len(body_toks) and body_toks[j].text == "="):
                        read_anywhere.add(t.text)
            vsplit = not read_anywhere
            if vsplit:
                note += " split"
    return KernelPlan(loop.loop_id, func, levels, body, arrays, sorted(set(arr_written)),
                      params, privates, reds, carried, mode, note, vec=vec,
                      write_refs=write_refs, vsplit=vsplit if mode == "gang" else False)


def write_boxes(prog: CProgram, kp: KernelPlan) -> dict:
    """array -> (per-dim (lo, hi) C expressions evaluated on the host at launch, exact?)

    A subscript is bounded exactly when it is a grid level's index (+- a constant), a
    constant, or an expression of launch-invariant scalars (the kernel's read-only
    arguments); anything else spans the whole dimension (inexact)."""
    lv = {h.var: i for i, h in enumerate(kp.levels)}
    fixed = {d.name for d in kp.params if d not in kp.carried}
    out = {}
    for name, refs in kp.write_refs.items():
        dims = prog.gmap[name].dims
        per_dim = [None] * len(dims)
        exact = True
        for subs in refs:
            for d, sub in enumerate(subs):
                txt = [t.text for t in sub]
                rng = None
                if len(txt) == 1 and txt[0] in lv:
                    i = lv[txt[0]]
                    rng = (f"hpg_lo{i}", f"hpg_lo{i} + (hpg_n{i} - 1) * hpg_st{i} + 1")
                elif len(txt) == 3 and txt[0] in lv and txt[1] in "+-" and sub[2].kind == "num":
                    i, c = lv[txt[0]], f"{txt[1]}{txt[2]}"
                    rng = (f"hpg_lo{i} {c}", f"hpg_lo{i} + (hpg_n{i} - 1) * hpg_st{i} + 1 {c}")
                elif all(t.kind == "num" or (t.kind == "name" and t.text in fixed) or
                         (t.kind == "punct" and t.text in "+-*/%()") for t in sub) and sub:
                    e = prog.text[sub[0].pos:sub[-1].pos + len(sub[-1].text)]
                    rng = (f"(long long)({e})", f"(long long)({e}) + 1")
                if rng is None:
                    rng = ("0", str(dims[d]))
                    exact = False
                per_dim[d] = rng if per_dim[d] is None else \
                    (f"std::min<long long>({per_dim[d][0]}, {rng[0]})",
                     f"std::max<long long>({per_dim[d][1]}, {rng[1]})")
        out[name] = (per_dim, exact)
    return out


def shared_writes(prog: CProgram, loop) -> list:
    """Arrays the body of `loop` writes at subscripts that do not depend on its index
    variable (directly or through scalars assigned from it): different iterations write
    the same elements, so running them in parallel is a race (output dependence)."""
    h = parse_header(prog, loop.span)
    if h is None:
        return []
    toks = prog.toks_in(*h.body)
    # scalars derived from the index: assignment targets whose right-hand side uses
    # a derived name (fixpoint); nested loop indices are not derived
    derived = {h.var}
    changed = True
    while changed:
        changed = False
        for k, t in enumerate(toks):
            if t.kind != "name" or k + 1 >= len(toks) or toks[k + 1].text not in ("=", "+=", "-="):
                continue
            if k and toks[k - 1].text == "(":       # for-header init: nested loop index
                continue
            if t.text in derived:
                continue
            end = k + 2
            while end < len(toks) and toks[end].text != ";":
                end += 1
            if any(x.kind == "name" and x.text in derived for x in toks[k + 2:end]):
                derived.add(t.text)
                changed = True
    out = []
    for k, t in enumerate(toks):
        if t.kind != "name" or t.text not in prog.gmap or not prog.gmap[t.text].is_array:
            continue
        j, names = k + 1, set()
        while j < len(toks) and toks[j].text == "[":
            depth = 0
            while True:
                if toks[j].text == "[":
                    depth += 1
                elif toks[j].text == "]":
                    depth -= 1
                    if depth == 0:
                        break
                elif toks[j].kind == "name":
                    names.add(toks[j].text)
                j += 1
            j += 1
        if j < len(toks) and toks[j].text in ("=", "+=", "-=", "*=", "/=", "++", "--") \
                and not (names & derived) and t.text not in out:
            out.append(t.text)
    return out


# ---------------------------------------------------------------------------- emit

def _array_ref(d: Decl) -> str:
    dims = "".join(f"[{n}]" for n in d.dims)
    return f"  {d.ctype} (&{d.name}){dims} = *reinterpret_cast<{d.ctype} (*){dims}>(D.{d.name});"


def emit_kernel(prog: CProgram, kp: KernelPlan) -> str:
    lines = []
    args = ["const Dev D", "double* __restrict__ hpg_red"]
    for lv_i, _ in enumerate(kp.levels):
        args += [f"long long hpg_lo{lv_i}", f"long long hpg_n{lv_i}", f"long long hpg_st{lv_i}"]
    for d in kp.params:
        args.append(f"{d.ctype} hpg_p_{d.name}")
    lines.append(f"__global__ void __launch_bounds__(256) k_{kp.loop}({', '.join(args)}) {{")
    lines.append('  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");')
    lines.append('  asm volatile("griddepcontrol.wait;" ::: "memory");')
    for name in kp.arrays:
        lines.append(_array_ref(prog.gmap[name]))
    declared = set()
    for d in kp.params:
        lines.append(f"  {d.ctype} {d.name} = hpg_p_{d.name};")
        declared.add(d.name)
    for d in kp.reductions:
        lines.append(f"  {d.ctype} {d.name} = 0;")
        declared.add(d.name)
    for d in kp.privates:
        if d.name not in declared:
            lines.append(f"  {d.ctype} {d.name};")
            declared.add(d.name)
    func_scalars = kp.func.params + kp.func.locals
    for lv in kp.levels:
        if lv.var not in declared:
            d = kp.func.scalar(lv.var) or prog.gmap.get(lv.var)
            lines.append(f"  {d.ctype if d else 'long long'} {lv.var};")
            declared.add(lv.var)
    # other function locals the body may use as privates (nested index vars ...)
    body_names = set(_idents(prog.toks_in(*kp.body)))
    for d in func_scalars:
        if d.name in body_names and d.name not in declared:
            lines.append(f"  {d.ctype} {d.name};")
            declared.add(d.name)
    body_text = prog.text[kp.body[0]:kp.body[1]]
    if kp.vec:
        # vector loops: thread-strided headers, a block barrier after each
        pieces, pos = [], kp.body[0]
        for region, hs in sorted(kp.vec, key=lambda x: x[0].span[0]):
            inner = hs[-1]
            pieces.append(prog.text[pos:region.span[0]])
            body = prog.text[inner.body[0]:inner.body[1]]
            start = "((long long)blockIdx.y * blockDim.x + threadIdx.x)" if kp.vsplit \
                else "(long long)threadIdx.x"
            stride = "(long long)gridDim.y * blockDim.x" if kp.vsplit else "(long long)blockDim.x"
            ns = [f"((long long)({x.hi}) > (long long)({x.lo}) ? ((long long)({x.hi}) - "
                  f"(long long)({x.lo}) + {x.step} - 1) / {x.step} : 0)" for x in hs]
            decl = " ".join(f"const long long hv_n{i} = {n};" for i, n in enumerate(ns))
            total = " * ".join(f"hv_n{i}" for i in range(len(hs)))
            idx = []
            for i in reversed(range(len(hs))):
                x = hs[i]
                if i:
                    idx.append(f"{x.var} = (long long)({x.lo}) + (hv_q % hv_n{i}) * {x.step}; "
                               f"hv_q /= hv_n{i};")
                else:
                    idx.append(f"{x.var} = (long long)({x.lo}) + hv_q * {x.step};")
            barrier = "" if kp.vsplit else " __syncthreads();"
            pieces.append(f"{{ {decl} for (long long hv_t = {start}; hv_t < {total}; "
                          f"hv_t += {stride}) {{ long long hv_q = hv_t; {' '.join(idx)} "
                          f"{body} }}{barrier} }}")
            pos = region.span[1]
        pieces.append(prog.text[pos:kp.body[1]])
        body_text = "".join(pieces)
    nl = len(kp.levels)
    total = " * ".join(f"hpg_n{i}" for i in range(nl))
    if kp.mode == "seq":
        lines.append("  if (blockIdx.x != 0 || threadIdx.x != 0) return;")
        lines.append("  for (long long hpg_t = 0; hpg_t < hpg_n0; ++hpg_t) {")
        lines.append(f"    {kp.levels[0].var} = hpg_lo0 + hpg_t * hpg_st0;")
        lines.append(f"    {body_text}")
        lines.append("  }")
        for r, d in enumerate(kp.privates):
            lines.append(f"  hpg_red[{r}] = (double){d.name};")
        lines.append("}")
        return "\n".join(lines)
    lines.append(f"  const long long hpg_total = {total};")
    if kp.mode == "gang":
        lines.append("  for (long long hpg_t = blockIdx.x; hpg_t < hpg_total; hpg_t += gridDim.x) {")
    elif kp.mode == "block":
        lines.append("  if (blockIdx.x != 0) return;")
        lines.append("  for (long long hpg_t = threadIdx.x; hpg_t < hpg_total; hpg_t += blockDim.x) {")
    else:
        lines.append("  for (long long hpg_t = blockIdx.x * (long long)blockDim.x + threadIdx.x; "
                     "hpg_t < hpg_total; hpg_t += (long long)gridDim.x * blockDim.x) {")
    lines.append("    long long hpg_q = hpg_t;")
    for i in reversed(range(nl)):
        lv = kp.levels[i]
        if i:
            lines.append(f"    {lv.var} = hpg_lo{i} + (hpg_q % hpg_n{i}) * hpg_st{i}; hpg_q /= hpg_n{i};")
        else:
            lines.append(f"    {lv.var} = hpg_lo0 + hpg_q * hpg_st0;")
    lines.append(f"    {body_text}")
    lines.append("  }")
    if kp.reductions:
        for r, d in enumerate(kp.reductions):
            lines.append(f"  hpg::block_reduce_store((double){d.name}, hpg_red, {r}, "
                         f"{len(kp.reductions)});")
    lines.append("}")
    return "\n".join(lines)


def emit_launch(prog: CProgram, kp: KernelPlan) -> str:
    """Host code replacing loop kp.loop when it runs on the device."""
    L = kp.loop
    ids = lambda names: ", ".join(f"V_{n}" for n in names) or "-1"   # noqa: E731
    s = []
    s.append(f"static const int hpg_arr_{L}[] = {{{ids(kp.arrays)}}};")
    s.append(f"static const int hpg_wr_{L}[] = {{{ids(kp.arrays_written)}}};")
    boxes = write_boxes(prog, kp)
    inexact = [n for n in kp.arrays_written if not boxes[n][1]]
    s.append(f"static const int hpg_inexact_{L}[] = {{{ids(inexact)}}};")
    s.append(f"R.kernel_enter({L}, hpg_arr_{L}, {len(kp.arrays)}, hpg_inexact_{L}, "
             f"{len(inexact)});")
    for i, lv in enumerate(kp.levels):
        s.append(f"const long long hpg_lo{i} = (long long)({lv.lo});")
        s.append(f"const long long hpg_hi{i} = (long long)({lv.hi});")
        s.append(f"const long long hpg_st{i} = {lv.step};")
        s.append(f"const long long hpg_n{i} = hpg_hi{i} > hpg_lo{i} ? "
                 f"(hpg_hi{i} - hpg_lo{i} + hpg_st{i} - 1) / hpg_st{i} : 0;")
    total = " * ".join(f"hpg_n{i}" for i in range(len(kp.levels)))
    nred = len(kp.reductions) if kp.mode != "seq" else len(kp.privates)
    s.append(f"const long long hpg_total = {total};")
    if kp.mode == "gang":
        s.append("const int hpg_grid = R.gang_grid(hpg_total);")
        s.append("const int hpg_block = 128;")
        s.append(f"const int hpg_vsplit = {'R.vector_split(hpg_total)' if kp.vsplit else '1'};")
    else:
        s.append(f"const int hpg_grid = R.grid_for(hpg_total, {'1' if kp.mode != 'grid' else '0'});")
        s.append(f"const int hpg_block = {'1' if kp.mode == 'seq' else '256'};")
    args = ["dev_struct(R)", "R.red_buffer(hpg_grid, " + str(max(nred, 1)) + ")"]
    for i in range(len(kp.levels)):
        args += [f"hpg_lo{i}", f"hpg_n{i}", f"hpg_st{i}"]
    args += [d.name for d in kp.params]
    s.append("if (hpg_total > 0) {")
    if kp.mode == "gang":
        s.append(f"  R.launch2(k_{L}, hpg_grid, hpg_vsplit, hpg_block, {', '.join(args)});")
    else:
        s.append(f"  R.launch(k_{L}, hpg_grid, hpg_block, {', '.join(args)});")
    s.append(f"  R.launched({L});")
    # the boxes this launch wrote (device-newer data a guarded copy-out moves back)
    for name, (per_dim, exact) in write_boxes(prog, kp).items():
        nd = len(per_dim)
        s.append(f"  {{ const long long lo[{nd}] = {{{', '.join(p[0] for p in per_dim)}}}; "
                 f"const long long hi[{nd}] = {{{', '.join(p[1] for p in per_dim)}}}; "
                 f"R.dev_wrote(V_{name}, lo, hi, {nd}); }}")
    if kp.mode == "seq" and kp.privates:
        # one sequential device thread: its final scalars are the program's
        s.append(f"  double hpg_v[{len(kp.privates)}];")
        s.append(f"  R.fetch_sums(1, {len(kp.privates)}, hpg_v);")
        for r, d in enumerate(kp.privates):
            s.append(f"  {d.name} = ({d.ctype})hpg_v[{r}];")
    elif kp.reductions:
        s.append(f"  double hpg_v[{len(kp.reductions)}];")
        s.append(f"  R.fetch_sums(hpg_grid, {len(kp.reductions)}, hpg_v);")
        for r, d in enumerate(kp.reductions):
            s.append(f"  {d.name} = ({d.ctype})((double){d.name} + hpg_v[{r}]);")
    s.append("}")
    s.append(f"R.kernel_exit({L}, hpg_arr_{L}, {len(kp.arrays)}, hpg_wr_{L}, "
             f"{len(kp.arrays_written)});")
    return "\n".join(s)


def host_write_boxes(prog: CProgram, loop, loops) -> list:
    """Host code reporting the boxes loop `loop`'s own statements (not its nested
    loops, which report their own) wrote, evaluated right after the loop ran on the
    host: the loop's index spans its header range, scalars the body does not assign
    are fixed, anything else spans the whole dimension."""
    h = parse_header(prog, loop.span)
    if h is None:
        return []
    kids = [loops.get(c).span for c in loops.children(loop.loop_id)]
    toks = [t for t in prog.toks_in(*h.body) if not any(a <= t.pos < b for a, b in kids)]
    assigned = set(_writes(prog.toks_in(*h.body)))
    assigned.discard(h.var)
    refs: dict = {}
    for k, t in enumerate(toks):
        if t.kind != "name" or t.text not in prog.gmap or not prog.gmap[t.text].is_array:
            continue
        j, subs = k + 1, []
        while j < len(toks) and toks[j].text == "[":
            depth, j0 = 0, j
            while True:
                if toks[j].text == "[":
                    depth += 1
                elif toks[j].text == "]":
                    depth -= 1
                    if depth == 0:
                        break
                j += 1
            subs.append(toks[j0 + 1:j])
            j += 1
        if j < len(toks) and toks[j].text in ("=", "+=", "-=", "*=", "/=", "++", "--"):
            refs.setdefault(t.text, []).append(subs)
    out = []
    hi_excl = f"(long long)({h.hi})"
    for name, rlist in refs.items():
        dims = prog.gmap[name].dims
        per = [None] * len(dims)
        for subs in rlist:
            for d, sub in enumerate(subs):
                txt = [x.text for x in sub]
                rng = None
                if txt == [h.var]:
                    rng = (f"(long long)({h.lo})", hi_excl)
                elif len(txt) == 3 and txt[0] == h.var and txt[1] in "+-" and sub[2].kind == "num":
                    c = f"{txt[1]}{txt[2]}"
                    rng = (f"(long long)({h.lo}) {c}", f"{hi_excl} {c}")
                elif sub and all(x.kind == "num" or (x.kind == "name" and x.text not in assigned
                                                      and x.text != h.var and x.text not in prog.gmap)
                                 or (x.kind == "punct" and x.text in "+-*/%()") for x in sub):
                    e = prog.text[sub[0].pos:sub[-1].pos + len(sub[-1].text)]
                    rng = (f"(long long)({e})", f"(long long)({e}) + 1")
                if rng is None:
                    rng = ("0", str(dims[d]))
                per[d] = rng if per[d] is None else \
                    (f"std::min<long long>({per[d][0]}, {rng[0]})",
                     f"std::max<long long>({per[d][1]}, {rng[1]})")
        nd = len(dims)
        out.append(f"{{ const long long lo[{nd}] = {{{', '.join(p[0] for p in per)}}}; "
                   f"const long long hi[{nd}] = {{{', '.join(p[1] for p in per)}}}; "
                   f"R.host_wrote(V_{name}, lo, hi, {nd}); }}")
    return out


def transform_text(prog: CProgram, a: int, b: int, loops_by_start: dict, launches: dict,
                   loops=None) -> str:
    """Text [a, b) with every loop statement wrapped in its hooks (recursively)."""
    out, i = [], a
    starts = sorted(p for p in loops_by_start if a <= p < b)
    while starts:
        p = starts[0]
        loop = loops_by_start[p]
        s, e = loop.span
        out.append(prog.text[i:s])
        inner = transform_text(prog, s, e, {q: l for q, l in loops_by_start.items()
                                            if s < q < e}, launches, loops)
        L = loop.loop_id
        dev = launches.get(L)
        hw = " ".join(host_write_boxes(prog, loop, loops)) if loops is not None else ""
        if dev is not None:
            out.append(f"{{ R.before({L}); if (R.dev({L})) {{\n{dev}\n}} else {{ {inner} {hw} }} "
                       f"R.after({L}); }}")
        else:
            out.append(f"{{ R.before({L}); R.host_only({L}); {inner} {hw} R.after({L}); }}")
        i = e
        starts = [q for q in starts if q >= e]
    out.append(prog.text[i:b])
    return "".join(out)


def generate(app: str, text: str, model, kinds: dict) -> str:
    """The .cu source of the generated executor (kinds: loop id -> directive kind value)."""
    prog = CProgram(text)
    loops = model.loops
    refs = model.refs
    arrays = [d for d in prog.globals if d.is_array]
    scalars = [d for d in prog.globals if not d.is_array]
    kernels, launches, notes = [], {}, {}
    kernel_modes = {}
    for l in loops:
        kind = kinds.get(l.loop_id)
        if kind is None:
            continue
        kp = plan_kernel(prog, l, kind, loops, kinds)
        if kp is None:
            notes[l.loop_id] = "loop header not recognised: host only"
            continue
        kernels.append(emit_kernel(prog, kp))
        launches[l.loop_id] = emit_launch(prog, kp)
        kernel_modes[l.loop_id] = (kp.mode, len(kp.levels), kp.note)
    loops_by_start = {l.span[0]: l for l in loops}

    # variable table: global arrays, then global scalars, then every other
    # plannable key of the model (function locals: scalars, counted only)
    var_keys = [d.name for d in arrays] + [d.name for d in scalars]
    for key in refs.vars:
        if key not in var_keys and refs.vars[key].scope != "loop-local" \
                and key not in refs.index_var_keys:
            var_keys.append(key)

    # arrays the loop's own statements write (children have their own hooks)
    loop_writes = {}
    for l in loops:
        loop_writes[l.loop_id] = sorted(
            var_keys.index(d.name) for d in arrays
            if (f := refs.vars[d.name].refs.get(l.loop_id)) is not None and f.written)
    # host region right before each top-level loop: its array writes
    seq = refs.region_sequence
    pre_writes = {}
    for n, r in enumerate(seq):
        if isinstance(r, int) and n and isinstance(seq[n - 1], str) and seq[n - 1].startswith("host:"):
            pre_writes[r] = sorted(
                var_keys.index(d.name) for d in arrays
                if (f := refs.vars[d.name].refs.get(seq[n - 1])) is not None and f.written)

    S = []
    S.append(f"// GENERATED by paper_2002_12115_b200/codegen.py for app '{app}' -- do not edit.")
    S.append("#include \"gen_runtime.cuh\"")
    S.append(f"namespace hpg_app_{app} {{")
    S.append("using hpg::Runtime;")
    S.append(f"constexpr int kLoops = {len(loops)};")
    S.append(f"constexpr int kVars = {len(var_keys)};")
    for n, key in enumerate(var_keys):
        S.append(f"constexpr int V_{re.sub(r'[^A-Za-z0-9_]', '_', key)} = {n};")
    S.append("struct Dev {")
    for d in arrays:
        S.append(f"  {d.ctype}* {d.name};")
    S.append("};")
    S.append("static const hpg::VarDesc kVarDesc[kVars] = {")
    for key in var_keys:
        d = prog.gmap.get(key)
        if d is not None and d.is_array:
            S.append(f"  {{\"{key}\", 1, sizeof({d.ctype}) * {d.elems()}ull}},")
        elif d is not None:
            S.append(f"  {{\"{key}\", 0, sizeof({d.ctype})}},")
        else:
            S.append(f"  {{\"{key}\", 0, 8}},")
    S.append("};")
    for n, key in enumerate(var_keys):
        d = prog.gmap.get(key)
        dims = d.dims if d is not None and d.is_array else [1]
        S.append(f"static const unsigned kDims_{n}[] = {{{', '.join(map(str, dims))}}};")
    S.append("static const unsigned* const kDims[kVars] = {" +
             ", ".join(f"kDims_{n}" for n in range(len(var_keys))) + "};")
    S.append("static const int kNdims[kVars] = {" + ", ".join(
        str(len(prog.gmap[k].dims)) if k in prog.gmap and prog.gmap[k].is_array else "1"
        for k in var_keys) + "};")
    S.append("static const unsigned long long kElems[kVars] = {" + ", ".join(
        f"{prog.gmap[k].elems()}ull" if k in prog.gmap and prog.gmap[k].is_array else "1ull"
        for k in var_keys) + "};")
    S.append("static const int kEligibleKind[kLoops] = {" + ", ".join(
        str({"kernels": 1, "parallel loop": 2, "parallel loop vector": 3}.get(kinds.get(l.loop_id), 0)
            if l.loop_id in launches else 0) for l in loops) + "};")
    for lid, ws in loop_writes.items():
        S.append(f"static const int kLoopWr_{lid}[] = {{{', '.join(map(str, ws)) or '-1'}}};")
    S.append("static const int* const kLoopWr[kLoops] = {" +
             ", ".join(f"kLoopWr_{l.loop_id}" for l in loops) + "};")
    S.append("static const int kLoopWrN[kLoops] = {" +
             ", ".join(str(len(loop_writes[l.loop_id])) for l in loops) + "};")
    for lid, ws in pre_writes.items():
        S.append(f"static const int kPreWr_{lid}[] = {{{', '.join(map(str, ws)) or '-1'}}};")
    S.append("static const int* const kPreWr[kLoops] = {" +
             ", ".join(f"kPreWr_{l.loop_id}" if l.loop_id in pre_writes else "nullptr"
                       for l in loops) + "};")
    S.append("static const int kPreWrN[kLoops] = {" +
             ", ".join(str(len(pre_writes.get(l.loop_id, []))) for l in loops) + "};")
    S.append("static const char* const kLoopNote[kLoops] = {" + ", ".join(
        '"' + (kernel_modes[l.loop_id][0] + "/" + str(kernel_modes[l.loop_id][1]) +
               (" " + kernel_modes[l.loop_id][2] if kernel_modes[l.loop_id][2] else "")
               if l.loop_id in kernel_modes else notes.get(l.loop_id, "host")) + '"'
        for l in loops) + "};")
    S.append("static const int kParent[kLoops] = {" + ", ".join(
        str(l.parent_loop if l.parent_loop is not None else -1) for l in loops) + "};")
    S.append("")
    S.extend(kernels)
    S.append("")
    S.append("struct Prog;")
    S.append("static Dev dev_struct(const hpg::Runtime& R) {")
    S.append("  Dev d;")
    for d in arrays:
        S.append(f"  d.{d.name} = ({d.ctype}*)R.dev_ptr[V_{d.name}];")
    S.append("  return d;")
    S.append("}")
    S.append("struct Prog {")
    for d in prog.globals:
        dims = "".join(f"[{n}]" for n in d.dims)
        S.append(f"  {d.ctype} {d.name}{dims};")
    S.append("  Runtime& R;")
    S.append("  explicit Prog(Runtime& r) : R(r) {}")
    S.append("  int printf(const char* f, ...) { va_list ap; va_start(ap, f); "
             "int n = R.vprint(f, ap); va_end(ap); return n; }")
    for f in prog.funcs:
        params = ", ".join(f"{d.ctype} {d.name}" for d in f.params)
        name = "main_" if f.name == "main" else f.name
        body = transform_text(prog, f.body[0], f.body[1], loops_by_start, launches, loops)
        S.append(f"  {f.ret} {name}({params}) {body}")
    S.append("};")
    S.append("static void bind(Prog* P, hpg::Runtime& R) {")
    for n, key in enumerate(var_keys):
        d = prog.gmap.get(key)
        if d is not None:
            S.append(f"  R.host_ptr[{n}] = (void*)&P->{d.name};")
    S.append("}")
    S.append("struct App {")
    S.append("  static constexpr int kLoops = hpg_app_" + app + "::kLoops;")
    S.append("  static constexpr int kVars = hpg_app_" + app + "::kVars;")
    S.append("  using Prog = hpg_app_" + app + "::Prog;")
    S.append("  static hpg::Tables tables() {")
    S.append("    return hpg::Tables{kLoops, kVars, kVarDesc, kDims, kNdims, kElems, kEligibleKind, "
             "kParent, kLoopWr, kLoopWrN, kPreWr, kPreWrN};")
    S.append("  }")
    S.append("  static void bind(Prog* P, hpg::Runtime& R) { hpg_app_" + app + "::bind(P, R); }")
    S.append("};")
    S.append("}  // namespace")
    S.append(f"HPG_DEFINE_APP(hpg_app_{app})")
    return "\n".join(S) + "\n"
