"""Multi-step time loops of compiled stencils, captured in one CUDA graph.

The reference executes one stencil call per ``CompiledStencil.__call__``
(stencilforge ``runtime.py:74-82, 220-251``): a synchronous call that
resolves arguments, validates and runs.  A model time loop (the dycore step
of BASELINE.json configs[4]: ``kernels/dycore.gts`` called 100 times with the
prognostic field swapped between steps) would pay that host path -- tens of
microseconds, comparable to a B200 step -- on every call.

``TimeLoop`` keeps the reference semantics of each call (same argument
resolution: ``runtime.resolve_domain_origin`` / ``_validate_storages`` run
once per distinct binding, here at construction) and replaces the per-call
host path with pre-marshalled launches (``Module.launcher``) captured once
into a CUDA graph (``gts_b200_graph_*``): ``run()`` replays all ``steps``
steps with one graph launch and no host synchronisation.

Bindings rotate: step ``s`` uses ``bindings[s % len(bindings)]`` -- for the
dycore, two bindings (u_in=A, u_out=B) and (u_in=B, u_out=A).  Every replay
starts again at ``bindings[0]``, so a loop whose ``steps`` is a multiple of
``len(bindings)`` continues the integration replay after replay.
"""

from __future__ import annotations

from typing import Optional, Sequence

from . import native
from ._host import Code, InvocationError, sf_runtime
from .storage import DeviceFieldStorage


class TimeLoop:
    def __init__(self, stencil, bindings: Sequence[dict], steps: int, scalars: Optional[dict] = None,
                 domain=None, stream: Optional[int] = None):
        """``stencil``: a ``CompiledStencil`` of the b200 backend;
        ``bindings``: field dicts {name: DeviceFieldStorage}, one per phase of
        the rotation; ``scalars``: api scalars shared by every step."""
        if stencil.backend != "b200":
            raise InvocationError(Code.UNKNOWN_BACKEND,
                                  f"TimeLoop needs a b200 stencil, got backend '{stencil.backend}'")
        if steps < 1 or not bindings:
            raise InvocationError(Code.MISSING_ARGUMENT, "TimeLoop needs steps >= 1 and at least one binding")
        self.stencil = stencil
        self.module = stencil.executable.build_info["module"]
        self.steps = int(steps)
        self.stream = stream if stream is not None else native.default_stream()
        scalars = dict(scalars or {})
        impl = stencil.implementation
        self.launchers = []
        self.domain = None
        for fields in bindings:
            for name, st in fields.items():
                if not isinstance(st, DeviceFieldStorage):
                    raise InvocationError(Code.LAYOUT_MISMATCH,
                                          f"TimeLoop field '{name}' must be a DeviceFieldStorage")
            # the reference's own argument resolution and validation
            # (runtime.py:122-217), once per binding
            args = {f.name: fields[f.name] for f in impl.api_fields}
            dom, origins = sf_runtime.resolve_domain_origin(stencil, args, domain, None)
            sf_runtime._validate_storages(stencil, args)
            if self.domain is None:
                self.domain = tuple(dom)
            elif tuple(dom) != self.domain:
                raise InvocationError(Code.OUT_OF_BOUNDS,
                                      f"bindings resolve to different domains {self.domain} / {tuple(dom)}")
            offset_ok = all(tuple(origins[n]) == tuple(fields[n].origin) for n in fields)
            if not offset_ok:
                raise InvocationError(Code.OUT_OF_BOUNDS, "TimeLoop uses the storages' own origins")
            self.launchers.append(self.module.launcher(self.domain, fields, scalars, self.stream))
        self.bindings = list(bindings)
        self._graph = None
        self.launches_per_step = None  # counted when the steps are captured

    def _enqueue(self) -> None:
        for s in range(self.steps):
            self.launchers[s % len(self.launchers)]()

    def capture(self) -> "TimeLoop":
        """Capture the ``steps`` launches into a CUDA graph (idempotent).
        Capture runs in relaxed mode, so a module's lazy first-call work
        (kernel attributes, the temporary arena's cudaMalloc) happens during
        capture without being recorded (gts_common.cuh ``gts_arena``)."""
        if self._graph is None:
            for fields in self.bindings:  # pending host writes land before capture
                for st in fields.values():
                    st.to_device(self.stream)
            g = native.Graph(self.stream)
            n0 = self.module.launch_count()
            with g.capture():
                self._enqueue()
            # kernels per step as enqueued by the module's entry (the plan
            # may fuse several kernels into one launch)
            self.launches_per_step = (self.module.launch_count() - n0) / self.steps
            self._graph = g
        return self

    def step(self, n: int = 1) -> None:
        """``n`` eager steps (no graph), asynchronous; step s uses binding
        s % len(bindings) counted from the first binding."""
        for s in range(n):
            self.launchers[s % len(self.launchers)]()
        self._mark_written()

    def run(self, sync: bool = True) -> None:
        """All ``steps`` steps: one graph launch (captured on first use).
        Host writes made through ``.view`` since the last launch are
        uploaded first, so the replay never works on (and then hides) a
        stale device copy."""
        self.capture()
        self._upload_pending()
        self._graph.launch()
        self._mark_written()
        if sync:
            native.synchronize(self.stream)

    def _storages(self):
        return list({id(st): st for fields in self.bindings for st in fields.values()}.values())

    def _upload_pending(self) -> None:
        for st in self._storages():
            st.to_device(self.stream)
            st.wait_producer(self.stream)

    def _mark_written(self) -> None:
        for st in self._storages():
            st.mark_device_written(self.stream)
