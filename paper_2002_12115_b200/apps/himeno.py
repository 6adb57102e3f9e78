"""Himeno benchmark restated in the reference's C subset (the application under test).

The reference tunes C programs through its own parser (acctuner/code_model.py),
which rejects ``#include``/``#define`` (code_model.py:286-293), ``struct``
(299-300), pointers (320-321) and non-literal extents (361-366).  RIKEN's
``himenoBMTxps.c`` uses all of those, so this module emits the static-array
Himeno program in the accepted subset, one text per grid size, with the
functions in execution order (``initmt``, ``jacobi``, ``main``) because the
reference orders host regions lexically (code_model.py:847-887).

The text is the single source of truth for three consumers:

* the reference front-end (parse -> 13 loops -> 13 eligible genes), run here
  by ``scripts/gen_program_model.py`` to produce the committed structural
  model under ``apps/model/``;
* the CPU oracle (``oracle/himeno_oracle.c``), which restates the same loop
  bodies in plain C and is pinned against the reference's own
  ``ExternalEvaluator`` running this text through ``gcc -O2``;
* the native library, whose host loops and sm_100a kernels implement the
  same 13 loops (``csrc/``).

Loop ids (document order, code_model.py:729-754):

====  =====================  =========================================
id    statement              body
====  =====================  =========================================
0-2   initmt i/j/k over IxJxK zero a[4], b[3], c[3], p, wrk1, bnd
3-5   initmt i/j/k < i/j/kmax coefficients, p = i*i/((imax-1)^2)
6     jacobi n < nn          gosa = 0; stencil nest; copy nest
7-9   i/j/k in [1, max-1)    19-point stencil, gosa += ss*ss, wrk2
10-12 i/j/k in [1, max-1)    p = wrk2
====  =====================  =========================================
"""

from __future__ import annotations

from dataclasses import dataclass

# 13 fp32 arrays are zeroed by loops 0-2; wrk2 is only written by the stencil.
FIELD_NAMES = ("p", "bnd", "wrk1", "wrk2",
               "a0", "a1", "a2", "a3", "b0", "b1", "b2", "c0", "c1", "c2")

FLOP_PER_POINT = 34          # RIKEN fflop per interior point per iteration
STENCIL_BYTES_PER_POINT = 56  # 13 fp32 reads (p once) + 1 fp32 write
COPY_BYTES_PER_POINT = 8      # 1 read + 1 write
OMEGA = 0.8


@dataclass(frozen=True)
class HimenoSize:
    """Static array extents (RIKEN MIMAX, MJMAX, MKMAX); k is contiguous."""
    name: str
    I: int
    J: int
    K: int

    @property
    def imax(self) -> int:
        return self.I - 1

    @property
    def jmax(self) -> int:
        return self.J - 1

    @property
    def kmax(self) -> int:
        return self.K - 1

    @property
    def interior_points(self) -> int:
        """Trip product of loops 7/8/9: (imax-2)(jmax-2)(kmax-2)."""
        return (self.I - 3) * (self.J - 3) * (self.K - 3)

    def flops(self, nn: int) -> int:
        return FLOP_PER_POINT * self.interior_points * nn

    @property
    def points(self) -> int:
        return self.I * self.J * self.K

    def sample_points(self) -> list[tuple[int, int, int]]:
        """Interior p samples printed by main (deterministic, no loops)."""
        I, J, K = self.I, self.J, self.K
        return [(I // 2, J // 2, K // 2), (1, 1, 1), (I - 3, J - 3, K - 3),
                (I // 3, (2 * J) // 3, K // 4)]


SIZES = {
    "XXS": HimenoSize("XXS", 9, 9, 17),
    "XS": HimenoSize("XS", 33, 33, 65),
    "S": HimenoSize("S", 65, 65, 129),
    "M": HimenoSize("M", 129, 129, 257),
    "L": HimenoSize("L", 257, 257, 513),
    "XL": HimenoSize("XL", 513, 513, 1025),
}


def size(name_or_size) -> HimenoSize:
    if isinstance(name_or_size, HimenoSize):
        return name_or_size
    try:
        return SIZES[name_or_size]
    except KeyError:
        raise ValueError(f"unknown Himeno size {name_or_size!r}; "
                         f"known: {', '.join(SIZES)}") from None


def custom_size(I: int, J: int, K: int, name: str = "custom") -> HimenoSize:
    if min(I, J, K) < 4:
        raise ValueError("every extent must be >= 4 (one interior point)")
    return HimenoSize(name, I, J, K)


_TEMPLATE = """\
static float p[{I}][{J}][{K}];
static float bnd[{I}][{J}][{K}];
static float wrk1[{I}][{J}][{K}];
static float wrk2[{I}][{J}][{K}];
static float a[4][{I}][{J}][{K}];
static float b[3][{I}][{J}][{K}];
static float c[3][{I}][{J}][{K}];
static int imax, jmax, kmax;
static float omega;

void initmt()
{{
  int i, j, k;
  for(i=0;i<{I};i++)
    for(j=0;j<{J};j++)
      for(k=0;k<{K};k++){{
        a[0][i][j][k]=0.0;
        a[1][i][j][k]=0.0;
        a[2][i][j][k]=0.0;
        a[3][i][j][k]=0.0;
        b[0][i][j][k]=0.0;
        b[1][i][j][k]=0.0;
        b[2][i][j][k]=0.0;
        c[0][i][j][k]=0.0;
        c[1][i][j][k]=0.0;
        c[2][i][j][k]=0.0;
        p[i][j][k]=0.0;
        wrk1[i][j][k]=0.0;
        bnd[i][j][k]=0.0;
      }}
  for(i=0;i<imax;i++)
    for(j=0;j<jmax;j++)
      for(k=0;k<kmax;k++){{
        a[0][i][j][k]=1.0;
        a[1][i][j][k]=1.0;
        a[2][i][j][k]=1.0;
        a[3][i][j][k]=1.0/6.0;
        b[0][i][j][k]=0.0;
        b[1][i][j][k]=0.0;
        b[2][i][j][k]=0.0;
        c[0][i][j][k]=1.0;
        c[1][i][j][k]=1.0;
        c[2][i][j][k]=1.0;
        p[i][j][k]=(float)(i*i)/(float)((imax-1)*(imax-1));
        wrk1[i][j][k]=0.0;
        bnd[i][j][k]=1.0;
      }}
}}

float jacobi(int nn)
{{
  int i, j, k, n;
  float gosa, s0, ss;
  for(n=0;n<nn;++n){{
    gosa = 0.0;
    for(i=1;i<imax-1;i++)
      for(j=1;j<jmax-1;j++)
        for(k=1;k<kmax-1;k++){{
          s0 = a[0][i][j][k] * p[i+1][j][k]
             + a[1][i][j][k] * p[i][j+1][k]
             + a[2][i][j][k] * p[i][j][k+1]
             + b[0][i][j][k] * ( p[i+1][j+1][k] - p[i+1][j-1][k]
                               - p[i-1][j+1][k] + p[i-1][j-1][k] )
             + b[1][i][j][k] * ( p[i][j+1][k+1] - p[i][j-1][k+1]
                               - p[i][j+1][k-1] + p[i][j-1][k-1] )
             + b[2][i][j][k] * ( p[i+1][j][k+1] - p[i-1][j][k+1]
                               - p[i+1][j][k-1] + p[i-1][j][k-1] )
             + c[0][i][j][k] * p[i-1][j][k]
             + c[1][i][j][k] * p[i][j-1][k]
             + c[2][i][j][k] * p[i][j][k-1]
             + wrk1[i][j][k];
          ss = ( s0 * a[3][i][j][k] - p[i][j][k] ) * bnd[i][j][k];
          gosa += ss*ss;
          wrk2[i][j][k] = p[i][j][k] + omega * ss;
        }}
    for(i=1;i<imax-1;++i)
      for(j=1;j<jmax-1;++j)
        for(k=1;k<kmax-1;++k)
          p[i][j][k] = wrk2[i][j][k];
  }}
  return gosa;
}}

int main()
{{
  float gosa;
  imax = {I}-1;
  jmax = {J}-1;
  kmax = {K}-1;
  omega = 0.8;
  initmt();
  gosa = jacobi({N});
  printf("%.9e\\n", gosa);
{SAMPLES}  return 0;
}}
"""


def source_text(sz, nn: int) -> str:
    """C-subset text of the Himeno program for one size and iteration count."""
    sz = size(sz)
    if nn < 1:
        raise ValueError("nn must be >= 1")
    samples = "".join(
        f'  printf("%.9e\\n", p[{i}][{j}][{k}]);\n' for i, j, k in sz.sample_points())
    return _TEMPLATE.format(I=sz.I, J=sz.J, K=sz.K, N=nn, SAMPLES=samples)


def source_file_id(sz) -> str:
    return f"himeno_{size(sz).name.lower()}.c"


@dataclass(frozen=True)
class HimenoProgram:
    """Committed program model + classifier verdicts for the Himeno text."""
    model: object            # model.ProgramModel
    eligible: tuple          # gene index -> loop id
    kinds: dict              # loop id -> kinds.DirectiveKind

    @property
    def gene_length(self) -> int:
        return len(self.eligible)


_PROGRAM = None


def program() -> HimenoProgram:
    """Load ``apps/model/himeno.json`` (generated by scripts/gen_program_model.py)."""
    global _PROGRAM
    if _PROGRAM is None:
        import json
        from pathlib import Path
        from .. import kinds as _kinds
        from ..model import load_structural
        doc = json.loads((Path(__file__).parent / "model" / "himeno.json").read_text())
        model = load_structural(doc)
        _PROGRAM = HimenoProgram(model, tuple(_kinds.eligible_ids(doc["verdicts"])),
                                 _kinds.kind_map(doc["verdicts"]))
    return _PROGRAM
