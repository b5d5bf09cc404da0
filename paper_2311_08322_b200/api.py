"""Drop-in entry point: ``compile_stencil(..., backend="b200")``.

Mirrors the reference's ``compile_stencil`` (stencilforge ``runtime.py:259-323``)
argument for argument.  For ``backend="b200"`` it runs the reference's own
frontend and analysis unchanged (``parse_program`` / ``inline_functions`` /
``bind_externals`` / ``analysis.lower``), fingerprints with backend id
``"b200"`` and the nvcc toolchain string (``runtime.py:305-306``), builds the
sm_100a module and returns the reference's own ``CompiledStencil``, so calls
go through the unchanged ``CompiledStencil.__call__`` -> ``invoke`` path
(``runtime.py:74-82, 220-251``).  Any other backend id is forwarded to the
reference untouched.

``install()`` additionally registers ``"b200"`` in the reference's closed
backend registry (``backends/__init__.py:6``; checked at ``runtime.py:271``)
and rebinds ``compile_stencil`` where the reference imported it by name
(``__init__.py:16``, ``bench.py:15``, ``cli.py:23``), so ``gts bench/diff
--backends b200`` and ``stencilforge.compile_stencil(..., backend="b200")``
work unmodified.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Union

from . import backend as b200_backend
from ._host import CompilationError, Code, DslError, InvocationError, analysis, ir, sf, sf_runtime
from .storage import BACKEND_ID, register_layout
from .toolchain import BuildCache, toolchain_version

_reference_compile = sf_runtime.compile_stencil


def _select_definition(source: str, stencil_name: Optional[str], externals: dict, file):
    """Parse, inline and bind through the reference's own frontend
    (``runtime.frontend_pipeline``, runtime.py:326-341), after the one rule
    ``compile_stencil`` adds to it: a program with several stencils needs
    ``stencil_name`` (runtime.py:283-291)."""
    if stencil_name is None:
        from stencilforge.frontend import inline_functions, parse_program

        try:
            names = [s.name for s in inline_functions(parse_program(source, file))]
        except DslError as exc:
            raise CompilationError([exc.as_diagnostic()])
        if len(names) > 1:
            err = DslError(Code.SYNTAX, ir.UNKNOWN_SPAN,
                           f"program has multiple stencils ({', '.join(names)}); pass stencil_name")
            raise CompilationError([err.as_diagnostic()])
    return sf_runtime.frontend_pipeline(source, stencil_name, externals, file)


@dataclass(frozen=True)
class B200ExecutionReport(sf_runtime.ExecutionReport):
    """The reference's ExecutionReport (runtime.py:21-38) plus device time:
    ``device_ns`` = CUDA-event span of the call on the device (host copies
    included in mirror mode), ``kernel_device_ns`` = the stencil launch alone
    (None when it interleaves with copies), and the bytes moved each way."""

    device_ns: Optional[int] = None
    kernel_device_ns: Optional[int] = None
    h2d_bytes: int = 0
    d2h_bytes: int = 0

    def as_dict(self) -> dict:
        d = super().as_dict()
        d.update(device_ns=self.device_ns, kernel_device_ns=self.kernel_device_ns,
                 h2d_bytes=self.h2d_bytes, d2h_bytes=self.d2h_bytes)
        return d


@dataclass
class B200CompiledStencil(sf_runtime.CompiledStencil):
    """The reference's CompiledStencil; calls return a B200ExecutionReport.
    ``time_device`` (or GTS_B200_DEVICE_TIME=1) adds CUDA-event device times
    to the report at ~20 us per call; the byte counts are always there."""

    time_device: bool = False

    def __call__(self, *, domain=None, origin=None, validate=None, **arguments):
        # per-thread timing flag and per-thread call statistics: concurrent
        # calls from other threads neither see nor change them
        with b200_backend.device_timing(self.time_device):
            rep = super().__call__(domain=domain, origin=origin, validate=validate, **arguments)
        t = b200_backend.call_stats()
        return B200ExecutionReport(rep.total_ns, rep.validate_ns, rep.kernel_ns, rep.domain, rep.validated,
                                   t.get("device_ns"), t.get("kernel_device_ns"), int(t.get("h2d", 0)),
                                   int(t.get("d2h", 0)))


def compile_stencil(
    source: str,
    stencil_name: Optional[str] = None,
    backend: str = BACKEND_ID,
    externals: Optional[dict[str, Union[int, float]]] = None,
    validation: str = "full",
    cache_dir: Optional[str] = None,
    gen_options: Optional[dict] = None,
    file: Optional[str] = None,
):
    if backend != BACKEND_ID:
        return _reference_compile(source, stencil_name, backend=backend, externals=externals,
                                  validation=validation, cache_dir=cache_dir,
                                  gen_options=gen_options, file=file)
    externals = dict(externals or {})
    bound = _select_definition(source, stencil_name, externals, file)
    impl = analysis.lower(bound)
    fp = ir.fingerprint(bound, BACKEND_ID, externals, toolchain_version(), gen_options)
    cache = BuildCache(cache_dir) if cache_dir is not None else BuildCache()
    executable = b200_backend.build(impl, fp, cache, gen_options)
    return B200CompiledStencil(
        name=impl.name,
        fingerprint=fp,
        backend=BACKEND_ID,
        implementation=impl,
        executable=executable,
        validation=validation,
    )


_installed = False


def install() -> None:
    """Register the b200 backend inside the reference package (idempotent)."""
    global _installed
    register_layout()
    if _installed:
        return
    import stencilforge.backends as sf_backends
    import stencilforge.bench as sf_bench

    ids = tuple(sf_backends.BACKEND_IDS)
    if BACKEND_ID not in ids:
        ids = ids + (BACKEND_ID,)
    sf_backends.BACKEND_IDS = ids
    sf_runtime.BACKEND_IDS = ids
    sf_runtime.compile_stencil = compile_stencil
    sf.compile_stencil = compile_stencil
    sf_bench.compile_stencil = compile_stencil
    try:
        import stencilforge.cli as sf_cli

        sf_cli.compile_stencil = compile_stencil
    except ImportError:  # click missing: CLI unavailable, API still patched
        pass
    _installed = True


__all__ = ["B200CompiledStencil", "B200ExecutionReport", "compile_stencil", "install", "InvocationError"]
