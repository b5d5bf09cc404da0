"""DSL builtins on the b200 backend vs the reference engines' own outputs
(tests/golden/builtins.npz from tests/golden/make_golden_builtins.py: gen,
vec and debug on every pair of IEEE special values plus wide random ranges).

The b200 code generator maps the builtins onto CUDA's IEEE operations:
abs -> fabs, sqrt -> correctly rounded sqrt (-prec-sqrt=true), floor / ceil
(exact), min / max -> the reference's NaN-propagating gts_min / gts_max
(gen.py:257-266); exp / log / pow -> libdevice (1-2 ulp, like glibc and
NumPy, which differ from each other by 1 ulp on this input set).
"""

from pathlib import Path

import numpy as np
import pytest

import _inputs
import paper_2311_08322_b200 as b200

GOLDEN = Path(__file__).parent / "golden" / "builtins.npz"
EXACT = ("o_abs", "o_min", "o_max", "o_sqrt", "o_floor", "o_ceil")
ROUNDED = ("o_exp", "o_log", "o_pow")


def _same_bits_or_nan(a, b):
    u = np.uint64 if a.dtype == np.float64 else np.uint32
    return (a.view(u) == b.view(u)) | (np.isnan(a) & np.isnan(b))


def _close(a, b, rtol):
    """Same NaN / Inf / zero pattern; finite values within ``rtol``
    relative, or within 2 ulp of the smallest subnormal where the result
    itself is subnormal (a relative bar is meaningless at 1-bit precision)."""
    if not np.array_equal(np.isnan(a), np.isnan(b)):
        return False
    fin = np.isfinite(a) & np.isfinite(b)
    if not np.array_equal(a[~fin & ~np.isnan(a)], b[~fin & ~np.isnan(b)]):
        return False
    a64, b64 = a[fin].astype(np.float64), b[fin].astype(np.float64)
    if not np.array_equal(a64 == 0, b64 == 0):
        return False
    sub = float(np.finfo(a.dtype).smallest_subnormal)
    tiny = float(np.finfo(a.dtype).tiny)
    diff = np.abs(a64 - b64)
    scale = np.maximum(np.abs(a64), np.abs(b64))
    ok = (diff <= rtol * scale) | ((scale < tiny) & (diff <= 2 * sub))
    return bool(ok.all())


def test_builtin_goldens_are_self_consistent():
    """The fixture's own engines agree where the docstring says they do."""
    g = dict(np.load(GOLDEN))
    for o in EXACT:
        if o in ("o_min", "o_max"):
            continue
        assert _same_bits_or_nan(g[f"f64_gen_{o}"], g[f"f64_vec_{o}"]).all(), o
    for o in ROUNDED:
        assert _close(g[f"f64_gen_{o}"], g[f"f64_vec_{o}"], 1e-12), o


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_builtins_vs_reference_engines(gpu, dtype):
    g = dict(np.load(GOLDEN))
    src = _inputs.BUILTINS_SRC.replace("Field[f64]", f"Field[{dtype}]")
    st = b200.compile_stencil(src, "builtins")
    x, y = g[f"{dtype}_x"], g[f"{dtype}_y"]
    f = {"x": b200.from_array(x), "y": b200.from_array(y)}
    for o in _inputs.BUILTIN_OUTS:
        f[o] = b200.allocate(dtype, x.shape, fill="poison")
    st(**f)
    rtol = 1e-12 if dtype == "f64" else 1e-5
    for o in _inputs.BUILTIN_OUTS:
        got = f[o].host_array()
        gen, vec = g[f"{dtype}_gen_{o}"], g[f"{dtype}_vec_{o}"]
        if o in EXACT:
            bad = ~_same_bits_or_nan(got, gen)
            assert not bad.any(), (o, x[bad][:4], y[bad][:4], got[bad][:4], gen[bad][:4])
            if o in ("o_min", "o_max"):  # NumPy: the second operand for (+0, -0)
                assert np.array_equal(got, vec, equal_nan=True), o
            else:
                assert _same_bits_or_nan(got, vec).all(), o
        else:
            assert _close(got, gen, rtol), (o, "vs gen")
            assert _close(got, vec, rtol), (o, "vs vec")
