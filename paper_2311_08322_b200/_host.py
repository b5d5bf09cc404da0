"""Locate the reference framework this backend plugs into.

The B200 backend is a drop-in *backend id* for the reference's unchanged
public API (``stencilforge.compile_stencil`` / ``CompiledStencil.__call__``,
stencilforge ``runtime.py:74-82, 259-323``).  The reference package is
therefore the host framework: its frontend, analysis and IR run once per
compile; its CPU engines (debug/vec/gen) are never called by this package.

Search order: an importable ``stencilforge``; the offline install under
``baseline/_ref`` (made by ``__graft_entry__.build()``; travels with the repo
snapshot); the read-only source tree at /root/reference (build container
only).
"""

from __future__ import annotations

import importlib
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
_CANDIDATES = (REPO / "baseline" / "_ref", Path("/root/reference/pkg/src"))


def stencilforge():
    try:
        return importlib.import_module("stencilforge")
    except ImportError:
        pass
    for cand in _CANDIDATES:
        if (cand / "stencilforge" / "__init__.py").is_file():
            sys.path.insert(0, str(cand))
            return importlib.import_module("stencilforge")
    raise ImportError(
        "the reference framework 'stencilforge' is not importable; run "
        "__graft_entry__.build() (installs it into baseline/_ref)"
    )


sf = stencilforge()

from stencilforge import analysis, ir  # noqa: E402
from stencilforge import runtime as sf_runtime  # noqa: E402
from stencilforge import storage as sf_storage  # noqa: E402
from stencilforge.backends import common as sf_common  # noqa: E402
from stencilforge.errors import BackendError, Code, CompilationError, DslError, InvocationError  # noqa: E402

__all__ = [
    "sf", "ir", "analysis", "sf_runtime", "sf_storage", "sf_common",
    "BackendError", "Code", "CompilationError", "DslError", "InvocationError",
]
