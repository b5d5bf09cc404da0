"""paper_2311_08322_b200 -- B200-native backend for the stencil DSL of
arXiv 2311.08322 (reference: stencilforge 0.1.0).

Drop-in usage (the reference API, unchanged)::

    import paper_2311_08322_b200 as b200
    st = b200.compile_stencil(source, "hdiff", backend="b200")
    inp = b200.from_array(values, (2, 2, 0))          # device-resident field
    out = b200.allocate("f64", (256, 256, 80))
    report = st(inp=inp, coeff=0.05, out=out)           # CompiledStencil.__call__

Host ``FieldStorage`` objects built with ``stencilforge.default_layout("b200")``
are accepted too (copied to the device around each call).
"""

from ._host import sf as stencilforge  # noqa: F401  (the reference framework)
from .api import compile_stencil, install
from .backend import BACKEND_ID
from .storage import (B200_LAYOUT, DeviceFieldStorage, ExternalDeviceFieldStorage, allocate, from_array,
                      from_cuda_array, to_device)

__version__ = "0.1.0"

__all__ = [
    "BACKEND_ID",
    "B200_LAYOUT",
    "DeviceFieldStorage",
    "ExternalDeviceFieldStorage",
    "allocate",
    "compile_stencil",
    "from_array",
    "from_cuda_array",
    "install",
    "to_device",
]
