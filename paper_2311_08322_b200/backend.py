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
import os
import threading
import weakref
from typing import Optional

from . import native
from ._host import BackendError, Code, ir, sf_common
from .codegen import entry_name, frame_setter_name, frame_tile_name, generate_source, mirror_setter_name
from .lowering import build_plan
from .storage import DeviceFieldStorage, FieldStorage
from .toolchain import BuildCache, load_library

BACKEND_ID = "b200"


# host buffers page-locked in place by the mirror mode: id(numpy base) ->
# registration (unregistered when the buffer is garbage collected)
_pinned_in_place: dict = {}
_pin_lock = threading.RLock()  # the GC finalizer may run while it is held
# the reference's own storages are pageable numpy memory (stencilforge
# storage.py:130-160); pinning them in place on first use turns their copies
# from the driver's staged pageable path into full-speed DMA
PIN_HOST = os.environ.get("GTS_B200_PIN_HOST", "1") != "0"


def _pin_host_buffer(base) -> None:
    key = id(base)
    with _pin_lock:
        if key in _pinned_in_place:
            return
        reg = ctypes.c_int(0)
        st = native.lib().gts_b200_host_register(base.ctypes.data, base.nbytes, ctypes.byref(reg))
        registered = st == 0 and bool(reg.value)
        _pinned_in_place[key] = registered
        # every entry (also "already page-locked" and "registration failed")
        # leaves with its buffer: a later buffer that reuses the id must be
        # looked at again, not taken for one that needs no pinning
        weakref.finalize(base, _unpin_host_buffer, key, base.ctypes.data, registered)


def _unpin_host_buffer(key, ptr, registered: bool = True) -> None:  # pragma: no cover - GC path
    with _pin_lock:
        _pinned_in_place.pop(key, None)
    if registered:
        try:
            native.lib().gts_b200_host_unregister(ptr)
        except Exception:
            pass


class _Mirror:
    """Cached device twin of a host FieldStorage (mirror mode).  A pageable
    host buffer is page-locked in place once (``PIN_HOST``)."""

    def __init__(self, storage: FieldStorage):
        self.nbytes = storage._base.nbytes
        p = ctypes.c_void_p()
        native.call("gts_b200_malloc", ctypes.byref(p), self.nbytes)
        self.dptr = p.value
        self.host_base = storage._base.ctypes.data
        self._fin = weakref.finalize(self, _Mirror._release, self.dptr)
        if PIN_HOST:
            _pin_host_buffer(storage._base)

    @staticmethod
    def _release(dptr):  # pragma: no cover - GC path
        try:
            native.lib().gts_b200_free(dptr)
        except Exception:
            pass

    def device_address(self, storage: FieldStorage) -> int:
        return self.dptr + (storage.base_address() - self.host_base)


# device twins of host storages, per (stream, host buffer): a thread's calls
# (one stream per thread, native.default_stream) never share a twin with
# another thread's concurrent call
_mirrors: dict = {}


def _mirror_for(storage: FieldStorage, stream: int) -> _Mirror:
    key = (stream, id(storage._base))
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
        self.lib.gts_b200_module_launch_count.argtypes = []
        self.lib.gts_b200_module_launch_count.restype = ctypes.c_ulonglong
        self._device = None
        self.field_order = [f.name for f in impl.api_fields]
        self.scalar_order = [s.name for s in impl.api_scalars]
        self.written = sf_common.written_fields(impl)
        try:  # present when built with gen_options mirror
            self._mirror_fn = getattr(self.lib, mirror_setter_name(impl, fp))
            self._mirror_fn.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_int64)]
            self._mirror_fn.restype = ctypes.c_int
        except AttributeError:
            self._mirror_fn = None
        try:  # present for single fused PARALLEL kernels (codegen frame_ok)
            self._frame_fn = getattr(self.lib, frame_setter_name(impl, fp))
            self._frame_fn.argtypes = [ctypes.c_int] * 4
            self._frame_fn.restype = ctypes.c_int
        except AttributeError:
            self._frame_fn = None
        try:
            ft = getattr(self.lib, frame_tile_name(impl, fp))
            ft.argtypes, ft.restype = [], ctypes.c_int
            v_ = int(ft())
            self.frame_tile = (v_ >> 16, v_ & 0xFFFF)  # rows, columns of a frame tile
        except AttributeError:
            self.frame_tile = None

    @property
    def frame_supported(self) -> bool:
        """The module can run a decomposed step's boundary as ONE frame launch
        (only the tiles touching the halo-dependent band; idempotent
        recomputation of band-adjacent interior points)."""
        return self._frame_fn is not None

    def launch_count(self) -> int:
        """Kernels this module has enqueued so far (every launch its entry
        made, fallback and helper kernels included)."""
        return int(self.lib.gts_b200_module_launch_count())

    def set_mirror(self, boxes) -> None:
        """Halo-mirror boxes for the calling thread's NEXT launch of this
        module, consumed by it (gen_options ``mirror``):
        ``boxes`` = [(i0, i1, j0, j1, base_address, s_i, s_j, s_k)], at most 8,
        in the launch's domain coordinates; element (i, j, k) of a box is also
        stored at base + (i*s_i + j*s_j + k*s_k) * itemsize."""
        if self._mirror_fn is None:
            raise BackendError(Code.COMPILE_FAILED, "module was not built with gen_options mirror")
        flat = [int(x) for b in boxes for x in b]
        arr = (ctypes.c_int64 * max(1, len(flat)))(*flat)
        native.check(self._mirror_fn(len(boxes), arr), "set mirror")

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
            st.wait_producer(stream)
            args.append(st.base_address())
            args.extend(int(s) for s in st.strides)
            args.extend(int(o) + int(d) for o, d in zip(st.origin, offset))
        for name in self.scalar_order:
            args.append(float(scalars[name]))
        args.append(stream)
        fn, sym = self.fn, self.symbol
        written = [fields[n] for n in self.written]
        bound = list({id(st): st for st in fields.values()}.values())

        def go() -> None:
            # host writes made through .view since the launcher was built land
            # first, so marking the outputs device-written loses nothing
            for st in bound:
                if st._host_dirty:
                    st.to_device(stream)
            status = fn(*args)
            if status:
                raise native.DeviceError(status, sym)
            for w in written:
                w.mark_device_written(stream)

        return go

    def frame_launcher(self, domain, fields: dict, scalars: dict, stream: int, band) -> callable:
        """Like ``launcher`` over the whole domain, but every enqueue first
        requests a frame launch for the calling thread: only the tiles with a
        point inside the band along the domain's sides run (the rest is the
        interior launch's).  ``band`` = (ilo, ihi, jlo, jhi): the band's width
        along the low-i, high-i, low-j and high-j sides (0 = none there), or
        (hi, hj) for the same widths on both sides of each axis."""
        if self._frame_fn is None:
            raise BackendError(Code.COMPILE_FAILED, f"{self.symbol}: no frame launch for this plan")
        go = self.launcher(domain, fields, scalars, stream)
        bands = frame_bands(band)
        fr = self._frame_fn

        def go_frame() -> None:
            native.check(fr(*bands), "frame request")
            go()

        return go_frame

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


def frame_bands(band) -> tuple:
    """(ilo, ihi, jlo, jhi) band widths from (hi, hj) or a 4-tuple."""
    b = tuple(int(x) for x in band)
    if len(b) == 2:
        b = (b[0], b[0], b[1], b[1])
    if len(b) != 4 or min(b) < 0:
        raise ValueError(f"frame band {band!r}: (hi, hj) or (ilo, ihi, jlo, jhi), all >= 0")
    return b


# Per-call state lives in thread-local storage, never in module globals, so
# concurrent calls from several threads do not see each other's:
# ``call_stats()`` = what the calling thread's last run() moved and how long
# the device took (B200ExecutionReport): device_ns = first host->device copy ..
# last device->host copy (or the launch alone for device storages),
# kernel_device_ns = the stencil launches only (None when they interleave with
# copies in the pipelined mirror mode).
_tls = threading.local()


def call_stats() -> dict:
    st = getattr(_tls, "stats", None)
    if st is None:
        st = _tls.stats = {"h2d": 0, "d2h": 0, "chunks": 0, "device_ns": None, "kernel_device_ns": None}
    return st


# CUDA-event device timing of run() (4 event records + 2 queries, ~20 us per
# call from Python, so opt-in: B200CompiledStencil.time_device for its own
# calls, or GTS_B200_DEVICE_TIME=1 for every call)
TIME_DEVICE = os.environ.get("GTS_B200_DEVICE_TIME") == "1"


def time_device() -> bool:
    return TIME_DEVICE or getattr(_tls, "time_device", False)


class device_timing:
    """``with device_timing(on):`` -- CUDA-event timing of the calling
    thread's run() calls inside the block (no global state is touched)."""

    def __init__(self, on: bool = True):
        self.on = on

    def __enter__(self):
        self.prev = getattr(_tls, "time_device", False)
        _tls.time_device = self.prev or self.on
        return self

    def __exit__(self, *a):
        _tls.time_device = self.prev
        return False


PIPE_TRACE = None  # a list to collect per-call device spans of the pipelined mirror mode (probes)
# GTS_B200_NVTX=1: every call runs inside an NVTX range "b200 <stencil>" (nsys / ncu --nvtx filtering)
NVTX = os.environ.get("GTS_B200_NVTX", "0") == "1"


def _event(i: int):
    """The calling thread's event slot ``i``."""
    evs = getattr(_tls, "events", None)
    if evs is None:
        evs = _tls.events = {}
    ev = evs.get(i)
    if ev is None:
        ev = evs[i] = native.Event()
    return ev


def _interval_range(iv, nk: int) -> tuple:
    def b(x):
        return x.offset if x.ref == ir.START else nk + x.offset
    return b(iv.start), b(iv.end)


def _fully_written(impl, name: str, nk: int) -> bool:
    """Some multistage assigns ``name`` unconditionally on every level
    [0, nk) (so the device twin needs no upload of its old values)."""
    from .lowering import always_writes

    for ms in impl.multistages:
        cover = []
        for st in ms.stages:
            if name in always_writes(st.body):
                cover.append(_interval_range(st.interval, nk))
        cover.sort()
        reach = 0
        for lo, hi in cover:
            if lo > reach:
                break
            reach = max(reach, hi)
        if reach >= nk:
            return True
    return False


def _call_local(impl, name: str, nk: int) -> bool:
    """Every read of ``name`` sees a value this call wrote: it is read only
    inside the sequential multistage that assigns it unconditionally on every
    level, at offsets (0, 0, dk) behind the sweep (FORWARD dk < 0, BACKWARD
    dk > 0) -- vadv's ``x[0, 0, 1]`` in its BACKWARD sweep (vadv.gts:16)."""
    from .lowering import always_writes

    home = None
    for mi, ms in enumerate(impl.multistages):
        for st in ms.stages:
            for acc in ir.stmt_reads(st.body):
                if not isinstance(acc, ir.FieldAccess) or acc.field != name:
                    continue
                di, dj, dk = acc.offset
                direction = {ir.FORWARD: 1, ir.BACKWARD: -1}.get(ms.order)
                if direction is None or di or dj or dk * direction >= 0:
                    return False
                if home not in (None, mi):
                    return False
                home = mi
    if home is None:
        return True
    ms = impl.multistages[home]
    cover = sorted(_interval_range(st.interval, nk) for st in ms.stages if name in always_writes(st.body))
    reach = 0
    for lo, hi in cover:
        if lo > reach:
            return False
        reach = max(reach, hi)
    return reach >= nk


class _Pipeline:
    """Mirror mode for host FieldStorages, pipelined over i-row chunks of the
    domain: chunk c's input rows go host->device on one copy stream while
    chunk c-1 computes and chunk c-2's outputs go device->host on the other
    (PCIe is full duplex).  Legal when no api field is both read and written
    and outputs do not alias inputs; a written field that the stencil
    overwrites entirely (storage == domain, every level unconditionally
    assigned) is never uploaded."""

    # measured on B200 + PCIe Gen5 (tools/e2e_probe.py, 256^2x80, 3 repeats):
    # vadv 3.65 / 3.79 / 3.62 / 3.67 ms and hdiff 1.55 / 1.48 / 1.38 / 1.42 ms
    # per call at 16 / 32 / 64 / 128 rows; a concurrent 2-D device->host copy
    # slows the host->device stream (0.4 ms at 32 rows), less so with fewer,
    # larger segments.  Round 2 (tapered, medians of 3): vadv 3.60 / 3.54 / 3.52
    # ms and hdiff 1.383 / 1.386 / 1.461 ms at 64 / 96 / 128 rows
    CHUNK_ROWS = 96
    MIN_ROWS = 128  # fewer i rows: one unpipelined copy-in / launch / copy-out

    # shrink the last chunks (shorter kernel + D2H tail after the last upload):
    # measured vadv 256^2x80 3.62 -> 3.58 ms per call, hdiff unchanged (1.37)
    TAPER = True

    @classmethod
    def chunk_bounds(cls, ni: int) -> list:
        """i-row chunks: CHUNK_ROWS each, the last two chunks' worth split
        into halving pieces (>= 16 rows) when TAPER is on."""
        c = cls.CHUNK_ROWS
        if not cls.TAPER:
            nch = max(1, ni // c)
            return [(k * ni // nch, (k + 1) * ni // nch) for k in range(nch)]
        out, r0 = [], 0
        while r0 < ni:
            rem = ni - r0
            n = c if rem > 2 * c else max(16, rem // 2)
            if rem - n < 16:
                n = rem
            out.append((r0, r0 + n))
            r0 += n
        return out

    def __init__(self, module, impl):
        self.module, self.impl = module, impl
        reads_ = set()
        for ms in impl.multistages:
            for st in ms.stages:
                reads_ |= {a.field for a in ir.stmt_reads(st.body) if isinstance(a, ir.FieldAccess)}
        self.inputs = [n for n in module.field_order if n not in module.written]
        self.outputs = [n for n in module.field_order if n in module.written]
        self.read_outputs = set(self.outputs) & reads_
        self.ext = {n: impl.field_extent(n) for n in module.field_order}

    def eligible(self, domain, field_args) -> bool:
        if domain[0] < self.MIN_ROWS:
            return False
        if not all(_call_local(self.impl, n, domain[2]) for n in self.read_outputs):
            return False
        outs = {id(field_args[n][0]._base) for n in self.outputs}
        ins = {id(field_args[n][0]._base) for n in self.inputs}
        if outs & ins or len(outs) != len(self.outputs):
            return False
        for n in self.module.field_order:
            st = field_args[n][0]
            if isinstance(st, DeviceFieldStorage) or st.strides[1] != 1:
                return False
            if st.strides[0] * st.shape[0] > st.strides[2] and st.shape[2] > 1:
                return False
        return True

    def run(self, domain, field_args, scalar_args) -> None:
        ni, nj, nk = domain
        comp = native.default_stream()
        up, down = native.aux_stream("h2d"), native.aux_stream("d2h")
        timed = time_device() or PIPE_TRACE is not None
        if timed:
            _event(1000).record(up)
        mirrors, ptrs, strides, origins = {}, {}, {}, {}
        for n in self.module.field_order:
            st, org = field_args[n]
            m = _mirror_for(st, comp)
            mirrors[n] = m
            ptrs[n] = m.device_address(st)
            strides[n] = tuple(int(x) for x in st.strides)
            origins[n] = tuple(int(o) for o in org)
        skip = {n for n in self.outputs
                if tuple(field_args[n][0].shape) == tuple(domain) and origins[n] == (0, 0, 0)
                and _fully_written(self.impl, n, nk)}
        bounds = self.chunk_bounds(ni)
        nch = len(bounds)
        done_row = {n: 0 for n in self.module.field_order}  # storage rows uploaded so far
        h2d = d2h = 0

        def copy(n, r0, r1, kind, stream):
            st = field_args[n][0]
            e = st.itemsize
            r0, r1 = max(r0, 0), min(r1, st.shape[0])
            if r1 <= r0:
                return 0
            width = (r1 - r0) * st.strides[0] * e
            pitch = st.strides[2] * e if st.shape[2] > 1 else width
            host = st.base_address() + r0 * st.strides[0] * e
            dev = ptrs[n] + r0 * st.strides[0] * e
            if kind == "h2d":
                native.call("gts_b200_memcpy2d_h2d", dev, pitch, host, pitch, width, st.shape[2], stream)
            else:
                native.call("gts_b200_memcpy2d_d2h", host, pitch, dev, pitch, width, st.shape[2], stream)
            return width * st.shape[2]

        for c, (c0, c1) in enumerate(bounds):
            last = c == nch - 1
            for n in self.module.field_order:
                if n in skip:
                    continue
                e = self.ext[n]
                o = origins[n][0]
                lo = o + c0 + (e.lo[0] if n in self.inputs else 0)
                hi = o + c1 + (e.hi[0] if n in self.inputs else 0)
                if last and n in self.inputs:
                    hi = max(hi, field_args[n][0].shape[0])
                lo = max(lo, done_row[n])
                h2d += copy(n, lo, hi, "h2d", up)
                done_row[n] = max(done_row[n], hi)
            ev_in = _event(2 * c)
            ev_in.record(up)
            native.call("gts_b200_stream_wait_event", comp, ev_in.ptr)
            org_c = {n: (origins[n][0] + c0, origins[n][1], origins[n][2]) for n in origins}
            self.module.launch((c1 - c0, nj, nk), ptrs, strides, org_c, scalar_args, comp)
            ev_done = _event(2 * c + 1)
            ev_done.record(comp)
            native.call("gts_b200_stream_wait_event", down, ev_done.ptr)
            for n in self.outputs:
                o = origins[n][0]
                d2h += copy(n, o + c0, o + c1, "d2h", down)
        if timed:
            _event(1001).record(up)
            _event(1002).record(comp)
            _event(1003).record(down)
        native.synchronize(down)
        native.synchronize(comp)
        stats = call_stats()
        stats.update(h2d=h2d, d2h=d2h, chunks=nch)
        if timed:
            t0 = _event(1000)
            span = max(t0.elapsed_ms(_event(1002)), t0.elapsed_ms(_event(1003)))
            stats.update(device_ns=int(span * 1e6))
        if PIPE_TRACE is not None:
            t0 = _event(1000)
            PIPE_TRACE.append({"h2d_ms": t0.elapsed_ms(_event(1001)), "kernels_ms": t0.elapsed_ms(_event(1002)),
                               "d2h_ms": t0.elapsed_ms(_event(1003))})


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
                storage.to_device(stream)
                storage.wait_producer(stream)
                pointers[name] = storage.base_address()
            else:
                key = id(storage._base)
                if key not in mirrors:
                    m = _mirror_for(storage, stream)
                    native.call("gts_b200_memcpy_h2d", m.dptr, m.host_base, m.nbytes, stream)
                    mirrors[key] = (m, storage)
                pointers[name] = mirrors[key][0].device_address(storage)
            strides[name] = tuple(int(s) for s in storage.strides)
            origins[name] = tuple(int(o) for o in origin)
        return pointers, strides, origins, mirrors

    pipe = _Pipeline(module, impl)
    fast: dict = {}  # device-resident calls: argument key -> marshalled entry arguments
    order, sorder = module.field_order, module.scalar_order
    written = tuple(module.written)

    def run_device(domain, field_args, scalar_args) -> bool:
        """Repeat calls on device storages: reuse the marshalled argument
        list (the per-call Python cost of the reference-facing path)."""
        sts = [field_args[n][0] for n in order]
        if not all(type(st) is DeviceFieldStorage for st in sts):
            return False
        module.bind_device()
        stream = native.default_stream()
        key = (module._device, stream, tuple(domain),
               tuple((id(st), st.base_address(), tuple(st.strides), tuple(st.shape), tuple(field_args[n][1]))
                     for n, st in zip(order, sts)),
               tuple(float(scalar_args[n]) for n in sorder))
        args = fast.get(key)
        if args is None:
            args = [int(domain[0]), int(domain[1]), int(domain[2])]
            for n, st in zip(order, sts):
                args.append(st.base_address())
                args.extend(int(x) for x in st.strides)
                args.extend(int(o) for o in field_args[n][1])
            args.extend(float(scalar_args[n]) for n in sorder)
            args.append(stream)
            if len(fast) >= 64:
                fast.clear()
            fast[key] = args
        for st in sts:
            if st._host_dirty:
                st.to_device(stream)
        status = module.fn(*args)
        if status:
            raise native.DeviceError(status, module.symbol)
        native.synchronize(stream)
        for n in written:
            field_args[n][0].mark_device_written()
        return True

    def run(domain, field_args, scalar_args) -> None:
        stats = call_stats()
        stats.update(h2d=0, d2h=0, chunks=0, device_ns=None, kernel_device_ns=None)
        if any(d == 0 for d in domain):
            return
        timed = time_device()
        if not timed and run_device(domain, field_args, scalar_args):
            return
        if pipe.eligible(domain, field_args):
            pipe.run(domain, field_args, scalar_args)
            return
        stream = native.default_stream()
        if timed:
            _event(2000).record(stream)
        pointers, strides, origins, mirrors = prepare(field_args, stream)
        if timed:
            _event(2001).record(stream)
        module.launch(domain, pointers, strides, origins, scalar_args, stream)
        if timed:
            _event(2002).record(stream)
        stats.update(h2d=sum(m.nbytes for m, _ in mirrors.values()), d2h=0, chunks=0)
        copied = set()
        for name in module.written:
            storage, _ = field_args[name]
            if isinstance(storage, DeviceFieldStorage):
                storage.mark_device_written()  # the stream is synchronised below
            else:
                key = id(storage._base)
                if key in copied:
                    continue
                copied.add(key)
                m = mirrors[key][0]
                native.call("gts_b200_memcpy_d2h", m.host_base, m.dptr, m.nbytes, stream)
                stats["d2h"] += m.nbytes
        if timed:
            _event(2003).record(stream)
        native.synchronize(stream)
        if timed:
            stats.update(device_ns=int(_event(2000).elapsed_ms(_event(2003)) * 1e6),
                         kernel_device_ns=int(_event(2001).elapsed_ms(_event(2002)) * 1e6))

    build_info = {
        "cache_hit": cache_hit,
        "so_path": str(so_path),
        "source_path": str(cache.source_path(fp)),
        "symbol": module.symbol,
        "arch": "sm_100a",
        "plan": plan.describe(),
        "module": module,
    }
    if NVTX:
        label = f"b200 {impl.name}".encode()
        inner = run

        def run(domain, field_args, scalar_args) -> None:  # noqa: F811 - the NVTX-wrapped call
            lib = native.lib()
            lib.gts_b200_nvtx_push(label)
            try:
                inner(domain, field_args, scalar_args)
            finally:
                lib.gts_b200_nvtx_pop()
    return sf_common.ExecutableStencil(BACKEND_ID, fp, run, build_info)
