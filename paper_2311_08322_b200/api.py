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
    """The frontend half of runtime.compile_stencil (runtime.py:278-303)."""
    from stencilforge.frontend import bind_externals, inline_functions, parse_program

    try:
        items = parse_program(source, file)
        stencils = inline_functions(items)
        if not stencils:
            raise DslError(Code.SYNTAX, ir.UNKNOWN_SPAN, "no stencil in program")
        if stencil_name is None:
            if len(stencils) > 1:
                names = ", ".join(s.name for s in stencils)
                raise DslError(Code.SYNTAX, ir.UNKNOWN_SPAN,
                               f"program has multiple stencils ({names}); pass stencil_name")
            definition = stencils[0]
        else:
            match = [s for s in stencils if s.name == stencil_name]
            if not match:
                raise DslError(Code.SYNTAX, ir.UNKNOWN_SPAN, f"no stencil named '{stencil_name}'")
            definition = match[0]
        return bind_externals(definition, externals)
    except DslError as exc:
        raise CompilationError([exc.as_diagnostic()])


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
        prev = b200_backend.TIME_DEVICE
        b200_backend.TIME_DEVICE = prev or self.time_device
        try:
            rep = super().__call__(domain=domain, origin=origin, validate=validate, **arguments)
        finally:
            b200_backend.TIME_DEVICE = prev
        t = b200_backend.last_transfer
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
