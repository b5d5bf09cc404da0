"""The b200 execution backend: IR -> CUDA module -> ``ExecutableStencil``.

``build`` is the counterpart of the reference's ``gen.compile_and_load``
(stencilforge ``backends/gen.py:469-539``): lower, generate, build through the
fingerprint-keyed cache, dlopen, bind the entry symbol, and return the
reference plugin record ``ExecutableStencil(backend_id, fingerprint, run,
build_info)`` (``backends/common.py:13-25``).

``run(domain, field_args, scalar_args)`` keeps the reference contract: output
fields are mutated in place and the call is synchronous (the runtime times it,
``runtime.py:241-243``).  Field arguments may be

* ``DeviceFieldStorage`` -- zero-copy: the device pointer goes straight to the
  kernel (a pending host-side write is uploaded first); or
* a host ``FieldStorage`` -- mirror mode: the buffer is copied to a cached
  device twin, the kernel runs, written fields are copied back.
"""

from __future__ import annotations

import ctypes
import weakref
from typing import Optional

from . import native
from ._host import BackendError, Code, ir, sf_common
from .codegen import entry_name, generate_source
from .lowering import build_plan
from .storage import DeviceFieldStorage, FieldStorage
from .toolchain import BuildCache, load_library

BACKEND_ID = "b200"


class _Mirror:
    """Cached device twin of a host FieldStorage (mirror mode)."""

    def __init__(self, storage: FieldStorage):
        self.nbytes = storage._base.nbytes
        p = ctypes.c_void_p()
        native.call("gts_b200_malloc", ctypes.byref(p), self.nbytes)
        self.dptr = p.value
        self.host_base = storage._base.ctypes.data
        self._fin = weakref.finalize(self, _Mirror._release, self.dptr)

    @staticmethod
    def _release(dptr):  # pragma: no cover - GC path
        try:
            native.lib().gts_b200_free(dptr)
        except Exception:
            pass

    def device_address(self, storage: FieldStorage) -> int:
        return self.dptr + (storage.base_address() - self.host_base)


_mirrors: dict = {}


def _mirror_for(storage: FieldStorage) -> _Mirror:
    key = id(storage._base)
    m = _mirrors.get(key)
    if m is None or m.host_base != storage._base.ctypes.data or m.nbytes != storage._base.nbytes:
        m = _Mirror(storage)
        _mirrors[key] = m
        weakref.finalize(storage._base, _mirrors.pop, key, None)
    return m


class Module:
    """A loaded generated module and its bound entry."""

    def __init__(self, impl, fp, so_path, plan):
        self.impl = impl
        self.fp = fp
        self.so_path = str(so_path)
        self.plan = plan
        self.lib = load_library(so_path)
        self.symbol = entry_name(impl, fp)
        try:
            fn = getattr(self.lib, self.symbol)
        except AttributeError:
            raise BackendError(Code.SYMBOL_NOT_FOUND, f"symbol '{self.symbol}' missing in {so_path}")
        argtypes = [ctypes.c_int64] * 3
        for _ in impl.api_fields:
            argtypes += [ctypes.c_void_p] + [ctypes.c_int64] * 6
        argtypes += [ctypes.c_double] * len(impl.api_scalars)
        argtypes.append(ctypes.c_void_p)
        fn.argtypes = argtypes
        fn.restype = ctypes.c_int
        self.fn = fn
        self.lib.gts_b200_module_set_device.argtypes = [ctypes.c_int]
        self.lib.gts_b200_module_set_device.restype = ctypes.c_int
        self._device = None
        self.field_order = [f.name for f in impl.api_fields]
        self.scalar_order = [s.name for s in impl.api_scalars]
        self.written = sf_common.written_fields(impl)

    def bind_device(self) -> None:
        dev = native.current_device()
        if dev != self._device:
            native.check(self.lib.gts_b200_module_set_device(dev), "module set device")
            self._device = dev

    def launcher(self, domain, fields: dict, scalars: dict, stream: int, offset=(0, 0, 0)):
        """Pre-marshalled asynchronous launch over device-resident storages
        ({name: DeviceFieldStorage}; origins = storage origins + ``offset``,
        i.e. a sub-rectangle of the domain).  Returns a zero-argument
        callable: one call = one enqueue of the stencil on ``stream``."""
        self.bind_device()
        args: list = [int(domain[0]), int(domain[1]), int(domain[2])]
        for name in self.field_order:
            st = fields[name]
            if not isinstance(st, DeviceFieldStorage):
                raise TypeError(f"launcher needs device-resident fields; '{name}' is {type(st).__name__}")
            st.to_device(stream)
            args.append(st.base_address())
            args.extend(int(s) for s in st.strides)
            args.extend(int(o) + int(d) for o, d in zip(st.origin, offset))
        for name in self.scalar_order:
            args.append(float(scalars[name]))
        args.append(stream)
        fn, sym = self.fn, self.symbol
        written = [fields[n] for n in self.written]

        def go() -> None:
            status = fn(*args)
            if status:
                raise native.DeviceError(status, sym)
            for w in written:
                w._device_dirty = True

        return go

    def launch(self, domain, pointers: dict, strides: dict, origins: dict, scalars: dict,
               stream: int) -> None:
        """Asynchronous launch with raw device pointers (no copies, no sync)."""
        self.bind_device()
        args: list = [int(domain[0]), int(domain[1]), int(domain[2])]
        for name in self.field_order:
            args.append(pointers[name])
            args.extend(strides[name])
            args.extend(origins[name])
        for name in self.scalar_order:
            args.append(float(scalars[name]))
        args.append(stream)
        status = self.fn(*args)
        if status:
            raise native.DeviceError(status, f"{self.symbol}")


def build(impl, fp, cache: Optional[BuildCache] = None, options: Optional[dict] = None):
    """Build (or fetch from the cache) and load the module for ``impl``."""
    cache = cache or BuildCache()
    plan = build_plan(impl, options)
    cache_hit = cache.lookup(fp) is not None
    source = None
    if cache_hit:
        so_path = cache.so_path(fp)
    else:
        source = generate_source(plan, fp, options)
        so_path = cache.install(fp, source, impl.name, plan.describe())
    try:
        module = Module(impl, fp, so_path, plan)
    except OSError:
        # corrupt entry: rebuild once (gen.py:484-494)
        cache.evict(fp)
        source = source or generate_source(plan, fp, options)
        so_path = cache.install(fp, source, impl.name, plan.describe())
        cache_hit = False
        try:
            module = Module(impl, fp, so_path, plan)
        except OSError as exc:
            raise BackendError(Code.CACHE_CORRUPT, f"rebuilt object unloadable: {exc}")

    def prepare(field_args, stream):
        """Resolve device pointers; upload pending host data."""
        pointers, strides, origins = {}, {}, {}
        mirrors = {}
        for name in module.field_order:
            storage, origin = field_args[name]
            if isinstance(storage, DeviceFieldStorage):
                storage.to_device(stream, sync=False)
                pointers[name] = storage.base_address()
            else:
                key = id(storage._base)
                if key not in mirrors:
                    m = _mirror_for(storage)
                    native.call("gts_b200_memcpy_h2d", m.dptr, m.host_base, m.nbytes, stream)
                    mirrors[key] = (m, storage)
                pointers[name] = mirrors[key][0].device_address(storage)
            strides[name] = tuple(int(s) for s in storage.strides)
            origins[name] = tuple(int(o) for o in origin)
        return pointers, strides, origins, mirrors

    def run(domain, field_args, scalar_args) -> None:
        if any(d == 0 for d in domain):
            return
        stream = native.default_stream()
        pointers, strides, origins, mirrors = prepare(field_args, stream)
        module.launch(domain, pointers, strides, origins, scalar_args, stream)
        copied = set()
        for name in module.written:
            storage, _ = field_args[name]
            if isinstance(storage, DeviceFieldStorage):
                storage.mark_device_written()
            else:
                key = id(storage._base)
                if key in copied:
                    continue
                copied.add(key)
                m = mirrors[key][0]
                native.call("gts_b200_memcpy_d2h", m.host_base, m.dptr, m.nbytes, stream)
        native.synchronize(stream)

    build_info = {
        "cache_hit": cache_hit,
        "so_path": str(so_path),
        "source_path": str(cache.source_path(fp)),
        "symbol": module.symbol,
        "arch": "sm_100a",
        "plan": plan.describe(),
        "module": module,
    }
    return sf_common.ExecutableStencil(BACKEND_ID, fp, run, build_info)
