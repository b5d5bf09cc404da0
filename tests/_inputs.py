"""Test-side input builders (restatements of the reference's harness helpers).

These regenerate, from seeds, the exact inputs the reference's differential
harness feeds its backends, so the committed golden fixtures only need to
store hashes / outputs.  ``tests/golden/make_golden.py`` checks each
restatement against the reference implementation it mirrors (input hashes
are stored next to the outputs) and ``tests/test_oracle.py`` re-checks them.
"""

from __future__ import annotations

import hashlib

import numpy as np

HDIFF_SRC = """\
stencil hdiff(inp: Field[f64], coeff: f64, out: Field[f64]):
    with computation(PARALLEL):
        with interval(0, None):
            lap = 4.0 * inp - (inp[-1, 0, 0] + inp[1, 0, 0] + inp[0, -1, 0] + inp[0, 1, 0])
            if (lap[1, 0, 0] - lap) * (inp[1, 0, 0] - inp) > 0.0:
                flx = 0.0
            else:
                flx = lap[1, 0, 0] - lap
            if (lap[0, 1, 0] - lap) * (inp[0, 1, 0] - inp) > 0.0:
                fly = 0.0
            else:
                fly = lap[0, 1, 0] - lap
            out = inp - coeff * (flx - flx[-1, 0, 0] + fly - fly[0, -1, 0])
"""


# every DSL builtin (ir.BUILTINS) in one stencil: tests/golden/make_golden_builtins.py
BUILTIN_OUTS = ["o_abs", "o_min", "o_max", "o_sqrt", "o_exp", "o_log", "o_pow", "o_floor", "o_ceil"]
BUILTINS_SRC = """
stencil builtins(x: Field[f64], y: Field[f64], o_abs: Field[f64], o_min: Field[f64], o_max: Field[f64],
                 o_sqrt: Field[f64], o_exp: Field[f64], o_log: Field[f64], o_pow: Field[f64],
                 o_floor: Field[f64], o_ceil: Field[f64]):
    with computation(PARALLEL):
        with interval(0, None):
            o_abs = abs(x)
            o_min = min(x, y)
            o_max = max(x, y)
            o_sqrt = sqrt(x)
            o_exp = exp(x)
            o_log = log(x)
            o_pow = pow(x, y)
            o_floor = floor(x)
            o_ceil = ceil(x)
"""


def field_halo(extent) -> tuple:
    """corpus.py:236-237."""
    return tuple(max(-lo, hi) for lo, hi in zip(extent.lo, extent.hi))


def written_fields(impl) -> set:
    """backends/common.py:49-55."""
    api = {f.name for f in impl.api_fields}
    out = set()

    def writes(s):
        if hasattr(s, "target"):
            yield s.target.field
        else:
            for sub in tuple(s.then_body) + tuple(s.else_body):
                yield from writes(sub)

    for ms in impl.multistages:
        for st in ms.stages:
            out |= set(writes(st.body))
    return out & api


def random_field_arrays(impl, domain, rng, ranges=None, poison=False):
    """Restatement of corpus.random_field_args (corpus.py:240-271): returns
    {name: (logical array of the full storage shape, origin)}."""
    written = written_fields(impl)
    out = {}
    for f in impl.api_fields:
        ext = impl.field_extent(f.name)
        halo = field_halo(ext)
        shape = tuple(d + 2 * h for d, h in zip(domain, halo))
        dt = np.float32 if f.dtype == "f32" else np.float64
        arr = np.full(shape, np.nan if poison else 0.0, dtype=dt)
        o = halo
        lo_, hi_ = ranges.get(f.name, (-1.0, 1.0)) if ranges else (-1.0, 1.0)
        region = tuple(slice(o[a] + ext.lo[a], o[a] + domain[a] + ext.hi[a]) for a in range(3))
        region_shape = tuple(s.stop - s.start for s in region)
        if f.name in written:
            arr[region] = 0.0
        else:
            arr[region] = rng.uniform(lo_, hi_, region_shape).astype(dt)
        out[f.name] = (arr, tuple(o))
    return out


def random_scalars(impl, rng) -> dict:
    """corpus.random_scalar_args (corpus.py:274-277)."""
    return {s.name: float(rng.uniform(-1.0, 1.0)) for s in impl.api_scalars}


def sha(arr: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()


def compute_view(arr: np.ndarray, origin, domain) -> np.ndarray:
    return arr[origin[0]: origin[0] + domain[0], origin[1]: origin[1] + domain[1],
               origin[2]: origin[2] + domain[2]]
