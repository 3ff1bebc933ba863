"""Particle Loop / Local Particle Pair Loop oracle (§8(f) NEXT-3) -- TEST INFRASTRUCTURE ONLY.

Executes a user C kernel the way the paper's sequential wrapper does (Listing
lst:simplest_pairloop: `for i, for j, if (i != j) KERNEL`), compiled with gcc
(-ffp-contract=off, so every a*b+c is two roundings as written), for small systems:

* Pair loops visit every ordered pair (i, j), i != j, whose canonical r^2 (reading R9) is
  below shell_cutoff^2 (strict, R4) -- the pair set of Def. 3 with the cutoff
  passed as PairLoop's shell_cutoff (Listing lst:LJ-loop).  j's position is
  its periodic image nearest to i, x_j + s L rounded once (the image a halo cell holds).
* Access descriptors (Tab. tab:DSL_access): READ (const), WRITE, RW, INC,
  INC_ZERO (zeroed before the loop).  `d.i[k]` is particle i's k-th component, `d.j[k]`
  particle j's (pair loops; READ, RW and WRITE dats -- Alg. alg:cna_II reads bond.j of an
  RW dat, relying on the loop leaving j's first n_nb(j) entries alone, reading R20).
  ScalarArrays (global) are used as `u[k]` or `S += ...`; Constants are
  substituted as #defines.
* Particle data arrays are [n, ncomp] in gid order (row = particle); dtypes double, int32,
  int64.

Nothing here is shared with the CUDA path; pinned by tests/test_oracle_dsl.py (Listing 9's
LJ kernel equals the O5 force oracle, the worked example Eqs. eqn:simple_op /
eqn:simple_op_global against numpy, the velocity-Verlet particle-loop listings, the CNA
kernels of Listings lst:CNA-kernel_I/II against oracle/cna.py's bond sets).
"""
from __future__ import annotations

import ctypes
import hashlib
import os
import subprocess
import tempfile

import numpy as np

READ, WRITE, RW, INC, INC_ZERO = "READ", "WRITE", "RW", "INC", "INC_ZERO"
_CTYPE = {np.dtype(np.float64): "double", np.dtype(np.int32): "int", np.dtype(np.int64): "long long"}
_CACHE = os.path.join(tempfile.gettempdir(), "ljmd_oracle_dsl")


def _const_defs(constants):
    out = []
    for k, v in (constants or {}).items():
        if isinstance(v, (int, np.integer)) and not isinstance(v, bool):
            out.append(f"#define {k} ({int(v)})")
        else:
            out.append(f"#define {k} ({float(v)!r})")
    return "\n".join(out)


def _compile(src):
    os.makedirs(_CACHE, exist_ok=True)
    h = hashlib.sha1(src.encode()).hexdigest()[:20]
    so = os.path.join(_CACHE, f"k_{h}.so")
    if not os.path.exists(so):
        c = os.path.join(_CACHE, f"k_{h}.c")
        with open(c, "w") as f:
            f.write(src)
        tmp = so + f".{os.getpid()}"
        subprocess.run(["gcc", "-O1", "-fPIC", "-shared", "-ffp-contract=off", "-fno-fast-math", "-std=c99",
                        c, "-o", tmp, "-lm"], check=True, capture_output=True)
        os.replace(tmp, so)
    return ctypes.CDLL(so)


def _prep(dats, scalars):
    """Normalise arrays; INC_ZERO zeroes (Tab. tab:DSL_access)."""
    d2 = {}
    for name, (arr, acc) in (dats or {}).items():
        a = np.ascontiguousarray(arr)
        if a.ndim == 1:
            a = a.reshape(-1, 1)
        a = a.copy()
        if acc == INC_ZERO:
            a[:] = 0
        d2[name] = (a, acc)
    s2 = {}
    for name, (arr, acc) in (scalars or {}).items():
        a = np.ascontiguousarray(np.atleast_1d(arr)).copy()
        if acc == INC_ZERO:
            a[:] = 0
        s2[name] = (a, acc)
    return d2, s2


def _bindings(d2, s2, pair, pos_label):
    """C declarations binding each label inside the loop body."""
    args, decl = [], []
    for name, (a, acc) in d2.items():
        ct = _CTYPE[a.dtype]
        nc = a.shape[1]
        args.append(f"{ct}* {name}_d")
        q = "const " if acc == READ else ""
        if pair and acc in (READ, RW, WRITE):
            decl.append(f"struct {{ {q}{ct}* i; const {ct}* j; }} {name} = "
                        f"{{ {name}_d + (long)i * {nc}, {name}_d + (long)j * {nc} }};")
        else:
            decl.append(f"struct {{ {q}{ct}* i; }} {name} = {{ {name}_d + (long)i * {nc} }};")
    for name, (a, acc) in s2.items():
        ct = _CTYPE[a.dtype]
        args.append(f"{ct}* {name}")
    if pos_label:
        if pair:
            decl.append(f"struct {{ const double* i; const double* j; }} {pos_label} = {{ pos + 3 * i, pj }};")
        else:
            decl.append(f"struct {{ const double* i; }} {pos_label} = {{ pos + 3 * i }};")
    return args, "\n        ".join(decl)


def _scalar_code(code, s2):
    # `S += x` on a one-component ScalarArray (Listing lst:simple-kernel) is S[0] += x
    import re
    for name in s2:
        code = re.sub(r"(?<![\w.\]])" + name + r"(\s*)\+=", name + r"[0]\1+=", code)
    return code


def pair_loop(code, pos, box, shell_cutoff, dats=None, scalars=None, constants=None, pos_label="r"):
    """Local Particle Pair Loop over ordered pairs with canonical r^2 < shell_cutoff^2.
    dats / scalars: {label: (array, access)}; returns ({label: array}, {label: array})."""
    pos = np.ascontiguousarray(pos, dtype=np.float64).reshape(-1, 3)
    box = np.ascontiguousarray(box, dtype=np.float64)
    n = pos.shape[0]
    d2, s2 = _prep(dats, scalars)
    args, decl = _bindings(d2, s2, True, pos_label)
    src = f"""
#include <math.h>
{_const_defs(constants)}
void loop(long n, const double* pos, const double* box, double cut2{''.join(', ' + a for a in args)})
{{
    for (long i = 0; i < n; ++i) {{
      for (long j = 0; j < n; ++j) {{
        if (i == j) continue;
        double pj[3];
        for (int d = 0; d < 3; ++d) {{
            double dd = pos[3 * i + d] - pos[3 * j + d];
            double s = dd > 0.5 * box[d] ? 1.0 : (dd < -0.5 * box[d] ? -1.0 : 0.0);
            pj[d] = s == 0.0 ? pos[3 * j + d] : pos[3 * j + d] + s * box[d];
        }}
        double dx = pos[3 * i] - pj[0], dy = pos[3 * i + 1] - pj[1], dz = pos[3 * i + 2] - pj[2];
        double r2 = (dx * dx + dy * dy) + dz * dz;
        if (!(r2 < cut2)) continue;
        {decl}
        {{
{_scalar_code(code, s2)}
        }}
      }}
    }}
}}
"""
    lib = _compile(src)
    cargs = [ctypes.c_long(n), pos.ctypes.data_as(ctypes.c_void_p), box.ctypes.data_as(ctypes.c_void_p),
             ctypes.c_double(float(shell_cutoff) ** 2)]
    cargs += [a.ctypes.data_as(ctypes.c_void_p) for a, _ in d2.values()]
    cargs += [a.ctypes.data_as(ctypes.c_void_p) for a, _ in s2.values()]
    lib.loop.restype = None
    lib.loop(*cargs)
    return {k: v[0] for k, v in d2.items()}, {k: v[0] for k, v in s2.items()}


def particle_loop(code, n, dats=None, scalars=None, constants=None, pos=None, pos_label="r"):
    """Particle Loop (Def. 1) over i = 0..n-1 in gid order."""
    d2, s2 = _prep(dats, scalars)
    args, decl = _bindings(d2, s2, False, pos_label if pos is not None else None)
    p = np.zeros((max(n, 1), 3)) if pos is None else np.ascontiguousarray(pos, dtype=np.float64).reshape(-1, 3)
    src = f"""
#include <math.h>
{_const_defs(constants)}
void loop(long n, const double* pos{''.join(', ' + a for a in args)})
{{
    for (long i = 0; i < n; ++i) {{
        {decl}
        {{
{_scalar_code(code, s2)}
        }}
    }}
}}
"""
    lib = _compile(src)
    cargs = [ctypes.c_long(n), p.ctypes.data_as(ctypes.c_void_p)]
    cargs += [a.ctypes.data_as(ctypes.c_void_p) for a, _ in d2.values()]
    cargs += [a.ctypes.data_as(ctypes.c_void_p) for a, _ in s2.values()]
    lib.loop.restype = None
    lib.loop(*cargs)
    return {k: v[0] for k, v in d2.items()}, {k: v[0] for k, v in s2.items()}
