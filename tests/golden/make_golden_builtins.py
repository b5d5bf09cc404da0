"""Golden outputs of the DSL builtins (abs, min, max, sqrt, exp, log, pow,
floor, ceil) from the REFERENCE's own engines (build container only):

    python tests/golden/make_golden_builtins.py

One stencil applies every builtin (ir.BUILTINS; emitted by gen as the C
library calls of gen.py:118-128 and gts_min/gts_max of gen.py:257-266, by
vec as the NumPy ufuncs of vec.py:26-37, by debug as the guarded math calls
of debug.py:32-101) to two fields x, y whose first planes hold every pair of
IEEE special values (NaN, +-Inf, +-0, subnormals, extremes, integers,
half-integers, negatives) and whose other planes hold random values over
wide exponent ranges.  f64 and f32 storage.  Saved: the inputs and the
``gen`` and ``vec`` outputs (builtins.npz), plus ``debug`` at f64.

The three engines disagree where their libraries do (measured here):
debug's Python ``math`` raises for pow(0, negative) and negative sqrt / log
arguments (debug.py:50-75 maps them to a positive NaN; C gives -NaN or +Inf),
and ``math.floor``/``ceil`` lose the sign of -0.0; NumPy's minimum/maximum
return the second operand for (+0, -0) where gen's gts_min/gts_max
(gen.py:257-266) return the first; exp, log and pow are not correctly
rounded (gen and vec differ by 1 ulp in 294 / 2 / 233 of 7680 f64 points).
The b200 test (tests/test_builtins.py) therefore requires, against gen (the
native reference): bitwise for abs, min, max, sqrt, floor, ceil (NaN payloads
aside); for exp, log, pow the same NaN / Inf / zero pattern and <= 1e-12
relative difference (north_star's f64 bar; 1e-5 for f32 storage) -- and the
same against vec, min / max compared modulo the sign of zero.
"""

from __future__ import annotations

import os
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
os.environ.setdefault("GTS_CACHE_DIR", tempfile.mkdtemp(prefix="gts-golden-"))

import stencilforge as sf  # noqa: E402

import _inputs  # noqa: E402

OUTS, SRC = _inputs.BUILTIN_OUTS, _inputs.BUILTINS_SRC
DOMAIN = (40, 48, 4)


def specials(dt):
    fi = np.finfo(dt)
    tiny_sub = np.array(fi.smallest_subnormal, dt)
    vals = [np.nan, np.inf, -np.inf, 0.0, -0.0, 1.0, -1.0, 2.0, -2.0, 0.5, -0.5, 3.0, -3.0, 2.5, -2.5,
            fi.max, -fi.max, fi.tiny, float(tiny_sub), -float(tiny_sub), 1e-3, 7.25, -0.75, 700.0, -745.5,
            1e300 if dt == np.float64 else 1e30, 0.1, 10.0, 1.0000001, -1e-7, 100.5, 31.0, -31.0, 0.3, 709.78, 88.7,
            -88.8, 4.0, -7.0, 1e-310 if dt == np.float64 else 1e-40]
    return np.array(vals[:40], dtype=dt)


def inputs(dt):
    rng = np.random.default_rng(77)
    ni, nj, nk = DOMAIN
    x = np.empty(DOMAIN, dt)
    y = np.empty(DOMAIN, dt)
    s = specials(dt)
    # plane 0: every (x, y) pair of the special values (40 x 40 of the 40 x 48 plane)
    x[:, :, 0] = 1.0
    y[:, :, 0] = 1.0
    x[:, :40, 0] = s[:, None]
    y[:, :40, 0] = s[None, :]
    # plane 1: wide exponent range, both signs (exp / log / pow arguments)
    mag = np.exp(rng.uniform(-40, 40, (ni, nj)))
    x[:, :, 1] = (mag * rng.choice([-1.0, 1.0], (ni, nj))).astype(dt)
    y[:, :, 1] = rng.uniform(-8, 8, (ni, nj)).astype(dt)
    # plane 2: positive bases, fractional / integer exponents
    x[:, :, 2] = rng.uniform(0, 50, (ni, nj)).astype(dt)
    y[:, :, 2] = np.where(rng.random((ni, nj)) < 0.5, rng.integers(-12, 12, (ni, nj)),
                          rng.uniform(-12, 12, (ni, nj))).astype(dt)
    # plane 3: exp's full range and rounding-boundary floor / ceil inputs
    x[:, :, 3] = rng.uniform(-745, 710 if dt == np.float64 else 88, (ni, nj)).astype(dt)
    y[:, :, 3] = (rng.integers(-50, 50, (ni, nj)) + rng.choice([-0.5, 0.0, 0.5], (ni, nj))).astype(dt)
    return x, y


def run(backend, dtype_name):
    dt = np.float32 if dtype_name == "f32" else np.float64
    src = SRC.replace("Field[f64]", f"Field[{dtype_name}]")
    st = sf.compile_stencil(src, "builtins", backend=backend)
    lay = sf.default_layout(backend)
    x, y = inputs(dt)
    f = {"x": sf.from_array(x, (0, 0, 0), lay), "y": sf.from_array(y, (0, 0, 0), lay)}
    for o in OUTS:
        f[o] = sf.from_array(np.zeros(DOMAIN, dt), (0, 0, 0), lay)
    with np.errstate(all="ignore"):
        st(**f)
    return x, y, {o: np.asarray(f[o].data()).copy() for o in OUTS}


def main() -> None:
    out = {}
    for dname in ("f64", "f32"):
        for backend in ("gen", "vec") + (("debug",) if dname == "f64" else ()):
            x, y, res = run(backend, dname)
            out[f"{dname}_x"], out[f"{dname}_y"] = x, y
            for o, v in res.items():
                out[f"{dname}_{backend}_{o}"] = v
    np.savez_compressed(HERE / "builtins.npz", **out)
    print("builtins.npz", (HERE / "builtins.npz").stat().st_size)


if __name__ == "__main__":
    main()
