"""CPU parity checker for the hdiff / vadv hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this module.  The product package
(``paper_2311_08322_b200``) never imports, links or executes anything under
``oracle/``.

Two independent restatements of the reference algorithms live here:

* ``libgts_oracle.so`` (``gts_oracle.c``): plain C with the reference gen
  engine's flags (``-O3 -fopenmp -ffp-contract=off``, stencilforge
  ``backends/gen.py:64-67``) and the gen entry ABI (``gen.py:5-14``).  It is
  the large-size oracle and the CPU baseline.
* ``hdiff_np`` / ``vadv_np``: NumPy restatements of ``kernels/hdiff.gts:3-15``
  and ``kernels/vadv.gts:4-16`` in the association order of the lowered IR
  (``pkg/tests/golden/hdiff_implementation.txt:11-24``).

A third route runs the REFERENCE's own native kernels: ``oracle/_ref`` (built
by ``build_ref.py`` from the reference's gen emitter, ``gen.py:229-369``)
holds hdiff / vadv (f64, f32) and the dycore step; ``ref_*`` below call them
on logical arrays (gen ABI, ``gen.py:5-14``).  They are the full-size checker
of bench.py and of the GPU tests.

Pinning: ``tests/test_oracle.py`` checks both restatements bitwise against
the golden vectors in ``tests/golden/`` that ``tests/golden/make_golden.py``
produced by running the reference's own ``vec`` and ``debug`` backends.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path
from typing import Optional

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "libgts_oracle.so"

_lib: Optional[ctypes.CDLL] = None


def build(force: bool = False) -> Path:
    """Compile libgts_oracle.so with the committed Makefile."""
    if force or not LIB_PATH.exists() or (
        LIB_PATH.stat().st_mtime < (HERE / "gts_oracle.c").stat().st_mtime
    ):
        env = dict(os.environ)
        env.pop("CC", None)
        subprocess.run(["make", "-C", str(HERE), "-B" if force else "all"],
                       check=True, capture_output=True, env=env)
    return LIB_PATH


def load() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        lib = ctypes.CDLL(str(LIB_PATH))
        i64 = ctypes.c_int64
        field = [ctypes.c_void_p] + [i64] * 6
        for name in ("oracle_hdiff_f64", "oracle_hdiff_f32"):
            fn = getattr(lib, name)
            fn.argtypes = [i64] * 3 + field * 2 + [ctypes.c_double, ctypes.c_int]
            fn.restype = ctypes.c_int
        for name in ("oracle_vadv_f64", "oracle_vadv_f32"):
            fn = getattr(lib, name)
            fn.argtypes = [i64] * 3 + field * 5 + [ctypes.c_int]
            fn.restype = ctypes.c_int
        lib.oracle_max_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def max_threads() -> int:
    return int(load().oracle_max_threads())


def _sfx(dtype) -> str:
    return "f32" if np.dtype(dtype) == np.float32 else "f64"


def _field_args(arr: np.ndarray, origin) -> list:
    """(base, strides in elements, origin) of a logical (i,j,k) array view."""
    item = arr.dtype.itemsize
    strides = [s // item for s in arr.strides]
    return [arr.ctypes.data, *strides, *origin]


# ---------------------------------------------------------------------------
# C oracle on logical arrays
# ---------------------------------------------------------------------------


def hdiff_c(inp: np.ndarray, coeff: float, nthreads: int = 0) -> np.ndarray:
    """hdiff on a (ni+4, nj+4, nk) logical block; returns (ni, nj, nk)."""
    inp = np.ascontiguousarray(inp)
    ni, nj, nk = inp.shape[0] - 4, inp.shape[1] - 4, inp.shape[2]
    out = np.zeros((ni, nj, nk), dtype=inp.dtype)
    fn = getattr(load(), f"oracle_hdiff_{_sfx(inp.dtype)}")
    rc = fn(ni, nj, nk, *_field_args(inp, (2, 2, 0)), *_field_args(out, (0, 0, 0)),
            float(coeff), int(nthreads))
    if rc:
        raise RuntimeError(f"oracle_hdiff failed: {rc}")
    return out


def vadv_c(a, b, c, d, nthreads: int = 0) -> np.ndarray:
    arrs = [np.ascontiguousarray(v) for v in (a, b, c, d)]
    x = np.zeros_like(arrs[0])
    ni, nj, nk = x.shape
    fn = getattr(load(), f"oracle_vadv_{_sfx(x.dtype)}")
    args = []
    for v in arrs + [x]:
        args += _field_args(v, (0, 0, 0))
    rc = fn(ni, nj, nk, *args, int(nthreads))
    if rc:
        raise RuntimeError(f"oracle_vadv failed: {rc}")
    return x


def run_on_storages(kernel: str, dtype: str, domain, fields: dict, scalars: dict,
                    nthreads: int = 0) -> None:
    """Run the C oracle directly on FieldStorage-like objects (anything with
    ``base_address()``, ``strides`` and ``origin``), gen-ABI style.  Used by
    bench.py's CPU baseline on the same storages the GPU path consumes."""
    lib = load()
    args: list = [int(domain[0]), int(domain[1]), int(domain[2])]
    names = ("inp", "out") if kernel == "hdiff" else ("a", "b", "c", "d", "x")
    for n in names:
        st = fields[n]
        args += [st.base_address(), *st.strides, *st.origin]
    if kernel == "hdiff":
        args.append(float(scalars["coeff"]))
    args.append(int(nthreads))
    rc = getattr(lib, f"oracle_{kernel}_{dtype}")(*args)
    if rc:
        raise RuntimeError(f"oracle_{kernel} failed: {rc}")


# ---------------------------------------------------------------------------
# NumPy restatements (second, independent route)
# ---------------------------------------------------------------------------


def hdiff_np(inp: np.ndarray, coeff: float) -> np.ndarray:
    """NumPy hdiff with the reference's stage order and f32 narrowing of the
    temporaries when the input is f32 (analysis.py:424-443)."""
    tdt = inp.dtype
    x = inp.astype(np.float64)
    ni, nj = inp.shape[0] - 4, inp.shape[1] - 4

    def I(di, dj, a=x, lo=2, ei=(0, 0), ej=(0, 0)):
        return a[lo + ei[0] + di: lo + ni + ei[1] + di, lo + ej[0] + dj: lo + nj + ej[1] + dj]

    # lap over [-1, ni+1) x [-1, nj+1)
    e = ((-1, 1), (-1, 1))
    lap = (4.0 * I(0, 0, ei=e[0], ej=e[1])) - (
        ((I(-1, 0, ei=e[0], ej=e[1]) + I(1, 0, ei=e[0], ej=e[1])) + I(0, -1, ei=e[0], ej=e[1]))
        + I(0, 1, ei=e[0], ej=e[1]))
    lap = lap.astype(tdt).astype(np.float64)  # temp store narrowing (no-op for f64)

    def L(di, dj, ei, ej):  # lap origin is (1, 1)
        return lap[1 + ei[0] + di: 1 + ni + ei[1] + di, 1 + ej[0] + dj: 1 + nj + ej[1] + dj]

    ex, ey = ((-1, 0), (0, 0)), ((0, 0), (-1, 0))
    dfx = L(1, 0, *ex) - L(0, 0, *ex)
    flx = np.where((dfx * (I(1, 0, ei=ex[0], ej=ex[1]) - I(0, 0, ei=ex[0], ej=ex[1]))) > 0.0,
                   0.0, dfx).astype(tdt).astype(np.float64)
    dfy = L(0, 1, *ey) - L(0, 0, *ey)
    fly = np.where((dfy * (I(0, 1, ei=ey[0], ej=ey[1]) - I(0, 0, ei=ey[0], ej=ey[1]))) > 0.0,
                   0.0, dfy).astype(tdt).astype(np.float64)
    # flx origin (1, 0); fly origin (0, 1)
    out = I(0, 0) - (coeff * (((flx[1:, :] - flx[:-1, :]) + fly[:, 1:]) - fly[:, :-1]))
    return out.astype(tdt)


def vadv_np(a, b, c, d) -> np.ndarray:
    """NumPy Thomas sweep, level by level over whole planes like the
    reference's vec engine (vec.py:160-166)."""
    tdt = np.result_type(a.dtype, b.dtype, c.dtype, d.dtype)
    tdt = np.float32 if tdt == np.float32 else np.float64
    A, B, C, D = (v.astype(np.float64) for v in (a, b, c, d))
    nk = a.shape[2]
    cp = np.empty(a.shape, dtype=tdt)
    dp = np.empty(a.shape, dtype=tdt)
    cp[:, :, 0] = C[:, :, 0] / B[:, :, 0]
    dp[:, :, 0] = D[:, :, 0] / B[:, :, 0]
    for k in range(1, nk):
        cpm = cp[:, :, k - 1].astype(np.float64)
        cp[:, :, k] = C[:, :, k] / (B[:, :, k] - (A[:, :, k] * cpm))
        dp[:, :, k] = (D[:, :, k] - (A[:, :, k] * dp[:, :, k - 1].astype(np.float64))) / (
            B[:, :, k] - (A[:, :, k] * cpm))
    x = np.empty(a.shape, dtype=a.dtype)
    x[:, :, nk - 1] = dp[:, :, nk - 1]
    for k in range(nk - 2, -1, -1):
        x[:, :, k] = dp[:, :, k].astype(np.float64) - (
            cp[:, :, k].astype(np.float64) * x[:, :, k + 1].astype(np.float64))
    return x


# ---------------------------------------------------------------------------
# The reference's own generated kernels (oracle/_ref)
# ---------------------------------------------------------------------------

REF_DIR = HERE / "_ref"
_ref_fns: dict = {}


def ref_manifest() -> dict:
    p = REF_DIR / "manifest.json"
    if not p.exists():
        return {}
    import json

    return json.loads(p.read_text())


def ref_available(key: str) -> bool:
    man = ref_manifest().get(key)
    return man is not None and (REF_DIR / man["so"]).exists()


def _ref_fn(key: str):
    if key not in _ref_fns:
        man = ref_manifest()[key]
        lib = ctypes.CDLL(str(REF_DIR / man["so"]))
        fn = getattr(lib, man["symbol"])
        nf = len(man["fields"])
        fn.argtypes = [ctypes.c_longlong] * 3 + ([ctypes.c_void_p] + [ctypes.c_longlong] * 6) * nf + \
            [ctypes.c_float if d == "f32" else ctypes.c_double for _, d in man["scalars"]]
        fn.restype = None
        _ref_fns[key] = (fn, man)
    return _ref_fns[key]


def gen_layout(arr: np.ndarray) -> np.ndarray:
    """Copy of a logical (i, j, k) array laid out k-outermost, j-contiguous
    (the gen layout, storage.py:60-64), returned as a logical view."""
    g = np.empty((arr.shape[2], arr.shape[0], arr.shape[1]), dtype=arr.dtype)
    g[...] = arr.transpose(2, 0, 1)
    return g.transpose(1, 2, 0)


def ref_call(key: str, domain, fields: dict, scalars: dict) -> None:
    """Run the reference kernel ``key`` over ``domain`` on logical arrays
    ``fields`` = {name: (array, origin)} (written in place)."""
    fn, man = _ref_fn(key)
    args = [int(domain[0]), int(domain[1]), int(domain[2])]
    for n in man["fields"]:
        arr, org = fields[n]
        args += _field_args(arr, org)
    for n, _ in man["scalars"]:
        args.append(float(scalars[n]))
    fn(*args)


def ref_hdiff(inp: np.ndarray, coeff: float) -> np.ndarray:
    """The reference gen engine's hdiff on a (ni+4, nj+4, nk) block."""
    key = "hdiff_" + _sfx(inp.dtype)
    dom = (inp.shape[0] - 4, inp.shape[1] - 4, inp.shape[2])
    out = gen_layout(np.zeros(dom, dtype=inp.dtype))
    ref_call(key, dom, {"inp": (gen_layout(inp), (2, 2, 0)), "out": (out, (0, 0, 0))}, {"coeff": coeff})
    return np.ascontiguousarray(out)


def ref_vadv(a, b, c, d) -> np.ndarray:
    key = "vadv_" + _sfx(a.dtype)
    x = gen_layout(np.zeros(a.shape, dtype=a.dtype))
    f = {n: (gen_layout(v), (0, 0, 0)) for n, v in zip("abcd", (a, b, c, d))}
    f["x"] = (x, (0, 0, 0))
    ref_call(key, a.shape, f, {})
    return np.ascontiguousarray(x)


def ref_dycore_run(u: np.ndarray, a, b, c, steps: int, coeff: float = 0.05, tau: float = 0.2) -> np.ndarray:
    """``steps`` dycore steps by the reference gen engine's own kernel for
    kernels/dycore.gts, with the host swap of u_in / u_out (the 2-cell halo
    keeps its initial values); returns the final u with its halo."""
    dom = (u.shape[0] - 4, u.shape[1] - 4, u.shape[2])
    bufs = [gen_layout(u), gen_layout(u)]
    coef = {n: (gen_layout(v), (0, 0, 0)) for n, v in zip("abc", (a, b, c))}
    for s in range(steps):
        src, dst = bufs[s % 2], bufs[(s + 1) % 2]
        ref_call("dycore_f64", dom, {"u_in": (src, (2, 2, 0)), "u_out": (dst, (2, 2, 0)), **coef},
                 {"coeff": coeff, "tau": tau})
    return np.ascontiguousarray(bufs[steps % 2])


def max_rel(a: np.ndarray, b: np.ndarray) -> float:
    """The reference's cross-backend metric (test_acceptance.py:50-54,
    cli.py:295-296)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.size == 0:
        return 0.0
    denom = np.maximum(np.maximum(np.abs(a), np.abs(b)), 1e-30)
    return float(np.max(np.abs(a - b) / denom))


def make_diagonally_dominant(rng: np.random.Generator, shape):
    """Restatement of the reference's vadv input generator
    (oracles.py:81-89): a, c ~ U(0.1, 1), b = |a| + |c| + U(0.5, 1.5),
    d ~ U(-1, 1), drawn in that order from one generator."""
    a = rng.uniform(0.1, 1.0, shape)
    c = rng.uniform(0.1, 1.0, shape)
    b = np.abs(a) + np.abs(c) + rng.uniform(0.5, 1.5, shape)
    d = rng.uniform(-1.0, 1.0, shape)
    return a, b, c, d


# ---------------------------------------------------------------------------
# dycore step (BASELINE.json configs[4]; paper_2311_08322_b200/kernels/dycore.gts)
# ---------------------------------------------------------------------------


def hdiff_run(u: np.ndarray, steps: int, coeff: float = 0.05) -> np.ndarray:
    """``steps`` hdiff steps as a ping-pong time loop (out becomes the next
    step's inp; the 2-cell halo keeps its initial values: Dirichlet), the C
    restatement per step."""
    u = np.array(u, copy=True)
    for _ in range(steps):
        u[2:-2, 2:-2, :] = hdiff_c(u, coeff)
    return u


def dycore_update_np(x: np.ndarray, tau: float) -> np.ndarray:
    """The interval-specialised update of dycore.gts (last computation):
    [0,1) and [K-1,K): u_out = x; [1,K-1): u_out = x + tau*((x[k+1] - 2*x) + x[k-1])
    -- the IR's left-to-right association (binary ops parse left-assoc, as in
    the reference frontend), f64 IEEE ops, no contraction."""
    u = x.copy()
    if x.shape[2] > 2:
        xm, x0, xp = x[:, :, :-2], x[:, :, 1:-1], x[:, :, 2:]
        u[:, :, 1:-1] = x0 + tau * ((xp - 2.0 * x0) + xm)
    return u


def dycore_step(u: np.ndarray, a, b, c, coeff: float = 0.05, tau: float = 0.2) -> np.ndarray:
    """One dycore.gts step on logical arrays: u is (ni+4, nj+4, nk) with its
    halo; returns u_out on the compute domain (ni, nj, nk).  Composition of
    the C restatements of hdiff (hdiff.gts:3-15) and the Thomas solve
    (vadv.gts:4-16, d := the diffused field) and the numpy update above --
    the multistage order of the reference engines (debug.py:301-355)."""
    uh = hdiff_c(u, coeff)
    x = vadv_c(a, b, c, uh)
    return dycore_update_np(x, tau)


def dycore_run(u: np.ndarray, a, b, c, steps: int, coeff: float = 0.05, tau: float = 0.2) -> np.ndarray:
    """``steps`` steps with the host swap of dycore.gts (u_out becomes the next
    u_in; the 2-cell halo keeps its initial values: Dirichlet boundary)."""
    u = np.array(u, copy=True)
    for _ in range(steps):
        u[2:-2, 2:-2, :] = dycore_step(u, a, b, c, coeff, tau)
    return u
