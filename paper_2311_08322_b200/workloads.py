"""The benchmark workloads (BASELINE.json configs) as DSL programs + inputs.

hdiff / vadv sources are the reference's committed kernels
(stencilforge ``kernels/hdiff.gts``, ``kernels/vadv.gts``, via
``kernels.kernel_source``, ``kernels.py:9-13``); the float32 variants change
only the field dtypes (scalars stay f64, the debug/vec convention).  Inputs
come from the reference harness builders (``bench.make_hdiff_args`` /
``make_vadv_args``, ``bench.py:82-105``) with the b200 layout, then move to
the device.
"""

from __future__ import annotations

from pathlib import Path

import numpy as np

from ._host import sf
from .storage import BACKEND_ID, register_layout, to_device

register_layout()


DYCORE_GTS = Path(__file__).resolve().parent / "kernels" / "dycore.gts"


def source(kernel: str, dtype: str = "f64") -> str:
    from stencilforge.kernels import kernel_source

    src = DYCORE_GTS.read_text() if kernel == "dycore" else kernel_source(kernel)
    if dtype == "f32":
        src = src.replace("Field[f64]", "Field[f32]")
    return src


def make_args(kernel: str, domain, dtype: str = "f64", seed: int = 0, device: bool = True):
    """Reference inputs (same RNG stream as stencilforge.bench) for the b200
    layout; device-resident unless ``device`` is False."""
    from stencilforge import bench as sf_bench

    host = sf_bench.KERNEL_BUILDERS[kernel](BACKEND_ID, tuple(domain), seed)
    if dtype == "f32":
        conv = {}
        for n, v in host.items():
            if isinstance(v, sf.FieldStorage):
                st = sf.allocate("f32", tuple(d - 2 * o for d, o in zip(v.shape, v.origin)),
                                 v.origin, v.layout)
                st.view[...] = v.view.astype("float32")
                conv[n] = st
            else:
                conv[n] = v
        host = conv
    if not device:
        return host
    return {n: (to_device(v) if isinstance(v, sf.FieldStorage) else v) for n, v in host.items()}


# dycore (BASELINE.json configs[4], kernels/dycore.gts) scalars
DYCORE_SCALARS = {"coeff": 0.05, "tau": 0.2}


def dycore_arrays(domain, seed: int = 0) -> dict:
    """Synthetic dycore state as logical numpy arrays: u (with its 2-cell
    horizontal halo) ~ U(-1, 1); implicit vertical-diffusion coefficients
    a, c ~ -U(0, 0.5) and b = 1 - a - c (diagonally dominant with margin 1,
    so the solve is a contraction and 100 steps stay bounded)."""
    ni, nj, nk = domain
    rng = np.random.default_rng(seed)
    u = rng.uniform(-1.0, 1.0, (ni + 4, nj + 4, nk))
    a = -rng.uniform(0.0, 0.5, (ni, nj, nk))
    c = -rng.uniform(0.0, 0.5, (ni, nj, nk))
    b = 1.0 - a - c
    return {"u": u, "a": a, "b": b, "c": c}


def algorithmic_bytes(kernel: str, domain, dtype: str = "f64") -> int:
    """hdiff E*[(ni+4)(nj+4)nk + ni*nj*nk]; vadv E*5*ni*nj*nk;
    dycore (per step, api fields read / written once each as authored):
    E*[(ni+4)(nj+4)nk (u_in) + 3*ni*nj*nk (a, b, c) + ni*nj*nk (u_out)]."""
    e = 4 if dtype == "f32" else 8
    ni, nj, nk = domain
    if kernel == "hdiff":
        return e * ((ni + 4) * (nj + 4) * nk + ni * nj * nk)
    if kernel == "vadv":
        return e * 5 * ni * nj * nk
    if kernel == "dycore":
        return e * ((ni + 4) * (nj + 4) * nk + 4 * ni * nj * nk)
    raise KeyError(kernel)
