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

from ._host import sf
from .storage import BACKEND_ID, register_layout, to_device

register_layout()


def source(kernel: str, dtype: str = "f64") -> str:
    from stencilforge.kernels import kernel_source

    src = kernel_source(kernel)
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


def algorithmic_bytes(kernel: str, domain, dtype: str = "f64") -> int:
    """hdiff E*[(ni+4)(nj+4)nk + ni*nj*nk]; vadv E*5*ni*nj*nk."""
    e = 4 if dtype == "f32" else 8
    ni, nj, nk = domain
    if kernel == "hdiff":
        return e * ((ni + 4) * (nj + 4) * nk + ni * nj * nk)
    if kernel == "vadv":
        return e * 5 * ni * nj * nk
    raise KeyError(kernel)
