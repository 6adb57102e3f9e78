"""NAS Parallel Benchmarks FT restated in the reference's C subset (second application).

The paper's second workload is NPB FT:
a 3-D FFT PDE solver.  The reference ships no application sources and its parser
rejects pointers, structs and ``#define`` (code_model.py:286-366), so, as for Himeno,
the program is restated in the accepted subset:

* complex arrays are split into real / imaginary arrays (``u0r``/``u0i`` ...);
* one ``main``, every loop inline in execution order (the reference's planner is
  lexical and does not follow calls): NPB's ``randlc`` / ``ipow46`` arithmetic is
  written out, and each of the six ``cffts`` calls (3 forward, 3 inverse) is its
  own loop block; the FFT works in place on ``u1`` with explicit copy loops where
  NPB's ``fft(dir, x1, x2)`` writes a second array;
* NPB's per-plane seed jump (``ipow46`` + ``randlc``) is a separate sequential loop
  that fills ``seeds[k]``, so the plane-fill loop carries no scalar across planes.

Algorithm (NPB 3.x serial FT, class S/W/A sizes): twiddle = exp(-4 alpha pi^2 (ii^2 +
jj^2 + kk^2)); u1 = NPB random complex field (randlc, a = 5^13, seed 314159265);
roots of unity; forward 3-D FFT (Stockham radix-2 ``fftz2`` passes along x, y, z)
u1 -> u0; then ``niter`` times: u0 *= twiddle, u1 = u0, inverse 3-D FFT u1 -> u2,
checksum = sum of 1024 sampled u2 points / (nx ny nz).  The checksums are NPB's
verification values (``VERIFY_CHECKSUMS``, relative error <= 1e-12 in NPB), which pin
this restatement (tests/test_ft.py).

The text is the single source of truth for the reference front-end
(``scripts/gen_program_model.py`` -> ``apps/model/ft_*.json``), for the CPU path
(the reference's compile template, ``gcc -O2``, pragmas ignored) and for the
generated B200 executor (``codegen.py``).
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class FTClass:
    name: str
    nx: int
    ny: int
    nz: int
    niter: int

    @property
    def nmax(self) -> int:
        return max(self.nx, self.ny, self.nz)

    @property
    def points(self) -> int:
        return self.nx * self.ny * self.nz


CLASSES = {
    "S": FTClass("S", 64, 64, 64, 6),
    "W": FTClass("W", 128, 128, 32, 6),
    "A": FTClass("A", 256, 256, 128, 6),
}

# NPB FT verification checksums (real, imag) per iteration, relative tolerance 1e-12
VERIFY_CHECKSUMS = {
    "S": [(5.546087004964e+02, 4.845363331978e+02), (5.546385409189e+02, 4.865304269511e+02),
          (5.546148406171e+02, 4.883910722336e+02), (5.545423607415e+02, 4.901273169046e+02),
          (5.544255039624e+02, 4.917475857993e+02), (5.542683411902e+02, 4.932597244941e+02)],
    "W": [(5.673612178944e+02, 5.293246849175e+02), (5.631436885271e+02, 5.282149986629e+02),
          (5.594024089970e+02, 5.270996558037e+02), (5.560698047020e+02, 5.260027904925e+02),
          (5.530898991250e+02, 5.249400845633e+02), (5.504159734538e+02, 5.239212247086e+02)],
    "A": [(5.046735008193e+02, 5.114047905510e+02), (5.059412319734e+02, 5.098809666433e+02),
          (5.069376896287e+02, 5.098144042213e+02), (5.077892868474e+02, 5.101336130759e+02),
          (5.085233095391e+02, 5.104914655194e+02), (5.091487099959e+02, 5.107917842803e+02)],
}
VERIFY_RTOL = 1e-12


def ft_class(name) -> FTClass:
    if isinstance(name, FTClass):
        return name
    try:
        return CLASSES[str(name).upper()]
    except KeyError:
        raise ValueError(f"unknown FT class {name!r} (one of {sorted(CLASSES)})") from None


def log2i(n: int) -> int:
    m = n.bit_length() - 1
    if 1 << m != n:
        raise ValueError(f"{n} is not a power of two")
    return m


def source_file_id(c: FTClass) -> str:
    return f"ft_{c.name.lower()}.c"


def _randlc(x: str, a: str, ind: str) -> str:
    """Inline NPB randlc: x = a * x mod 2^46 (temporaries t1..t4, a1, a2, x1, x2, z)."""
    return "\n".join(ind + l for l in [
        f"t1 = r23 * {a};", "a1 = (int)(t1);", f"a2 = {a} - t23 * a1;",
        f"t1 = r23 * {x};", "x1 = (int)(t1);", f"x2 = {x} - t23 * x1;",
        "t1 = a1 * x2 + a2 * x1;", "t2 = (int)(r23 * t1);", "z = t1 - t23 * t2;",
        "t3 = t23 * z + a2 * x2;", "t4 = (int)(r46 * t3);", f"{x} = t3 - t46 * t4;"])


def _fft_block(n: int, outer: int, lines: int, xr: str, xi: str, sign: int, ind: str) -> str:
    """One cffts: for every line batch a, copy lines into (yr, yi), Stockham radix-2 passes
    (NPB fftz2) alternating y -> z -> y, copy back."""
    m = log2i(n)
    wi = "wi = ui[li + i];" if sign >= 1 else "wi = -ui[li + i];"

    def butterfly(src, dst):
        return f"""for(i=0;i<li;i++){{
  i11 = i * lk;
  i12 = i11 + {n // 2};
  i21 = i * lj;
  i22 = i21 + lk;
  wr = ur[li + i];
  {wi}
  for(k=0;k<lk;k++)
    for(j=0;j<{lines};j++){{
      x11r = {src}r[i11 + k][j];
      x11i = {src}i[i11 + k][j];
      x21r = {src}r[i12 + k][j];
      x21i = {src}i[i12 + k][j];
      {dst}r[i21 + k][j] = x11r + x21r;
      {dst}i[i21 + k][j] = x11i + x21i;
      tr = x11r - x21r;
      ti = x11i - x21i;
      {dst}r[i22 + k][j] = wr * tr - wi * ti;
      {dst}i[i22 + k][j] = wr * ti + wi * tr;
    }}
}}"""

    def indent(t, n):
        return "\n".join(" " * n + l for l in t.splitlines())

    odd_copy = f"""
  for(i=0;i<{n};i++)
    for(j=0;j<{lines};j++){{
      yr[i][j] = zr[i][j];
      yi[i][j] = zi[i][j];
    }}""" if m % 2 == 1 else ""
    text = f"""for(a=0;a<{outer};a++){{
  for(b=0;b<{n};b++)
    for(c=0;c<{lines};c++){{
      yr[b][c] = {xr};
      yi[b][c] = {xi};
    }}
  for(l=1;l<={m};l++){{
    lk = 1 << (l - 1);
    li = 1 << ({m} - l);
    lj = 2 * lk;
    if(l % 2 == 1){{
{indent(butterfly("y", "z"), 6)}
    }} else {{
{indent(butterfly("z", "y"), 6)}
    }}
  }}{odd_copy}
  for(b=0;b<{n};b++)
    for(c=0;c<{lines};c++){{
      {xr} = yr[b][c];
      {xi} = yi[b][c];
    }}
}}"""
    return indent(text, len(ind))


def source_text(c, niter: int | None = None) -> str:
    """The FT program for class `c` (niter defaults to the class's).

    One ``main`` with every loop inline, in execution order: the reference's planner
    orders regions lexically and does not follow calls (code_model.py:847-887,
    transfer.py:184-193), so a call inside a loop would hide the callee's writes from
    its hoisting -- as in the Himeno text, statement order is execution order.
    """
    c = ft_class(c)
    nx, ny, nz, nmax = c.nx, c.ny, c.nz, c.nmax
    niter = c.niter if niter is None else int(niter)
    decl = f"[{nz}][{ny}][{nx}]"
    pad = "  "

    def ffts(sign):
        # line batches: x-lines of a z plane (c = j), y-lines of a z plane (c = i),
        # z-lines of a y row (c = i); transform index b, line index c
        b1 = _fft_block(nx, nz, ny, "u1r[a][c][b]", "u1i[a][c][b]", sign, pad)
        b2 = _fft_block(ny, nz, nx, "u1r[a][b][c]", "u1i[a][b][c]", sign, pad)
        b3 = _fft_block(nz, ny, nx, "u1r[b][a][c]", "u1i[b][a][c]", sign, pad)
        return [b1, b2, b3] if sign >= 1 else [b3, b2, b1]

    fwd = "\n".join(ffts(1))
    inv = "\n".join("\n".join("  " + l for l in blk.splitlines()) for blk in ffts(-1))
    seed_step = _randlc("rx", "an", "    ")
    return f"""static double u0r{decl};
static double u0i{decl};
static double u1r{decl};
static double u1i{decl};
static double u2r{decl};
static double u2i{decl};
static double twid{decl};
static double ur[{nmax}];
static double ui[{nmax}];
static double yr[{nmax}][{nmax}];
static double yi[{nmax}][{nmax}];
static double zr[{nmax}][{nmax}];
static double zi[{nmax}][{nmax}];
static double seeds[{nz}];
static double sumr[{niter + 1}];
static double sumi[{niter + 1}];

int main()
{{
  int i, j, k, a, b, c, l, lk, li, lj, i11, i12, i21, i22, ii, jj, kk, n, n2, ln, it, q, r, s;
  double ap, an, x, pq, pr, rx, t, ti, tr, wr, wi, x11r, x11i, x21r, x21i, cr, ci;
  double r23, r46, t23, t46, t1, t2, t3, t4, a1, a2, x1, x2, z;
  double xa1, xa2, xx1, xx2, tt1, tt2, tt3, tt4, zz;
  r23 = 1.1920928955078125e-07;
  r46 = r23 * r23;
  t23 = 8388608.0;
  t46 = t23 * t23;
  ap = -4.0 * 1.0e-6 * 3.141592653589793238 * 3.141592653589793238;
  for(k=0;k<{nz};k++)
    for(j=0;j<{ny};j++)
      for(i=0;i<{nx};i++){{
        kk = ((k + {nz // 2}) % {nz}) - {nz // 2};
        jj = ((j + {ny // 2}) % {ny}) - {ny // 2};
        ii = ((i + {nx // 2}) % {nx}) - {nx // 2};
        twid[k][j][i] = exp(ap * (double)(ii * ii + jj * jj + kk * kk));
      }}
  pq = 1220703125.0;
  pr = 1.0;
  n = {2 * nx * ny};
  while(n > 1){{
    n2 = n / 2;
    if(n2 * 2 == n){{
{_randlc("pq", "pq", "      ")}
      n = n2;
    }} else {{
{_randlc("pr", "pq", "      ")}
      n = n - 1;
    }}
  }}
{_randlc("pr", "pq", "  ")}
  an = pr;
  rx = 314159265.0;
  for(k=0;k<{nz};k++){{
    seeds[k] = rx;
{seed_step}
  }}
  xa1 = (int)(r23 * 1220703125.0);
  xa2 = 1220703125.0 - t23 * xa1;
  for(k=0;k<{nz};k++){{
    x = seeds[k];
    for(j=0;j<{ny};j++)
      for(i=0;i<{nx};i++){{
        xx1 = (int)(r23 * x);
        xx2 = x - t23 * xx1;
        tt1 = xa1 * xx2 + xa2 * xx1;
        tt2 = (int)(r23 * tt1);
        zz = tt1 - t23 * tt2;
        tt3 = t23 * zz + xa2 * xx2;
        tt4 = (int)(r46 * tt3);
        x = tt3 - t46 * tt4;
        u1r[k][j][i] = r46 * x;
        xx1 = (int)(r23 * x);
        xx2 = x - t23 * xx1;
        tt1 = xa1 * xx2 + xa2 * xx1;
        tt2 = (int)(r23 * tt1);
        zz = tt1 - t23 * tt2;
        tt3 = t23 * zz + xa2 * xx2;
        tt4 = (int)(r46 * tt3);
        x = tt3 - t46 * tt4;
        u1i[k][j][i] = r46 * x;
      }}
  }}
  ur[0] = {log2i(nmax)};
  ui[0] = 0.0;
  ln = 1;
  for(j=1;j<={log2i(nmax)};j++){{
    t = 3.141592653589793238 / ln;
    for(i=0;i<ln;i++){{
      ti = i * t;
      ur[ln + i] = cos(ti);
      ui[ln + i] = sin(ti);
    }}
    ln = 2 * ln;
  }}
{fwd}
  for(k=0;k<{nz};k++)
    for(j=0;j<{ny};j++)
      for(i=0;i<{nx};i++){{
        u0r[k][j][i] = u1r[k][j][i];
        u0i[k][j][i] = u1i[k][j][i];
      }}
  for(it=1;it<={niter};it++){{
    for(k=0;k<{nz};k++)
      for(j=0;j<{ny};j++)
        for(i=0;i<{nx};i++){{
          u0r[k][j][i] = u0r[k][j][i] * twid[k][j][i];
          u0i[k][j][i] = u0i[k][j][i] * twid[k][j][i];
          u1r[k][j][i] = u0r[k][j][i];
          u1i[k][j][i] = u0i[k][j][i];
        }}
{inv}
    for(k=0;k<{nz};k++)
      for(j=0;j<{ny};j++)
        for(i=0;i<{nx};i++){{
          u2r[k][j][i] = u1r[k][j][i];
          u2i[k][j][i] = u1i[k][j][i];
        }}
    cr = 0.0;
    ci = 0.0;
    for(j=1;j<=1024;j++){{
      q = j % {nx};
      r = (3 * j) % {ny};
      s = (5 * j) % {nz};
      cr = cr + u2r[s][r][q];
      ci = ci + u2i[s][r][q];
    }}
    sumr[it] = cr / {float(c.points)!r};
    sumi[it] = ci / {float(c.points)!r};
  }}
  for(it=1;it<={niter};it++){{
    printf("%.12e\\n", sumr[it]);
    printf("%.12e\\n", sumi[it]);
  }}
  return 0;
}}
"""


@dataclass(frozen=True)
class FTProgram:
    """The FT program model from the reference front-end (apps/model/ft_<class>.json)."""
    cls: FTClass
    model: object
    eligible: tuple
    kinds: dict

    @property
    def gene_length(self) -> int:
        return len(self.eligible)


_PROGRAMS: dict = {}


def program(c="S") -> FTProgram:
    """Load ``apps/model/ft_<class>.json`` (generated by scripts/gen_program_model.py)."""
    c = ft_class(c)
    if c.name not in _PROGRAMS:
        import json
        from pathlib import Path
        from .. import kinds as _kinds
        from ..model import load_structural
        path = Path(__file__).parent / "model" / f"ft_{c.name.lower()}.json"
        if not path.exists():
            raise ValueError(f"no program model for FT class {c.name} ({path.name})")
        doc = json.loads(path.read_text())
        _PROGRAMS[c.name] = FTProgram(c, load_structural(doc),
                                      tuple(_kinds.eligible_ids(doc["verdicts"])),
                                      _kinds.kind_map(doc["verdicts"]))
    return _PROGRAMS[c.name]


def parse_checksums(stdout: str) -> list:
    """(real, imag) per iteration from the program's stdout."""
    vals = [float(x) for x in stdout.split()]
    return list(zip(vals[0::2], vals[1::2]))


def checksum_error(stdout: str, c="S") -> float:
    """Max relative error of the printed checksums against NPB's verification values."""
    c = ft_class(c)
    got = parse_checksums(stdout)
    want = VERIFY_CHECKSUMS[c.name]
    if len(got) != len(want):
        return float("inf")
    return max(max(abs(a - x) / abs(x), abs(b - y) / abs(y)) for (a, b), (x, y) in zip(got, want))
