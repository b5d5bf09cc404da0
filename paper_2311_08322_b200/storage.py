"""Device-resident field storages for the b200 backend.

``DeviceFieldStorage`` subclasses the reference's ``FieldStorage``
(stencilforge ``storage.py:74-103``) so the unchanged runtime accepts it
(``runtime.py:96`` isinstance check) and validates its layout against
``BACKEND_LAYOUTS["b200"]`` (``runtime.py:203-217``).  The buffer lives in
HBM; ``view`` is a lazily synchronised host mirror in pinned memory so code
written against the reference (``storage.view[...] = values``,
``np.asarray(storage.data())``) keeps working:

* reading ``view`` / ``data()`` first copies device -> host if the device
  copy is newer, and marks the host mirror as possibly modified;
* every launch (a stencil call, a ``Module.launcher`` enqueue, a TimeLoop or
  graph replay) first copies host -> device if the host mirror may have been
  modified, so the device copy is never newer than a pending host write and
  the two flags are never both set;
* an asynchronous launch remembers its stream: a later host read, or a
  launch on another stream, waits for it first.

Synchronisation takes a per-storage lock, so threads sharing an input storage
(concurrent calls on disjoint outputs) upload it once, and no
thread launches on it before the upload completed.

The b200 layout is the gen engine's axis order (k outermost, j contiguous,
``storage.py:60-64``) with the origin element and every row aligned to
128 B (an L2 line, and the TMA global-stride granularity).
"""

from __future__ import annotations

import ctypes
import threading
import weakref
from typing import Optional, Union

import numpy as np

from . import native
from ._host import Code, sf_storage

LayoutSpec = sf_storage.LayoutSpec
FieldStorage = sf_storage.FieldStorage
StorageError = sf_storage.StorageError

BACKEND_ID = "b200"
B200_LAYOUT = LayoutSpec((2, 0, 1), 128)

_NP = {"f32": np.dtype("<f4"), "f64": np.dtype("<f8")}


def register_layout() -> None:
    """Register the b200 default layout (storage.py:60-64)."""
    sf_storage.BACKEND_LAYOUTS.setdefault(BACKEND_ID, B200_LAYOUT)


register_layout()


def _strides(shape, layout: LayoutSpec, itemsize: int):
    """Same rule as the reference (storage.py:117-127)."""
    align = layout.alignment_bytes // itemsize
    outer, mid, inner = layout.permutation
    padded = -(-shape[inner] // align) * align
    s = [0, 0, 0]
    s[inner] = 1
    s[mid] = padded
    s[outer] = padded * shape[mid]
    return (s[0], s[1], s[2]), s[outer] * shape[outer]


class _DeviceBuffer:
    """Owning device allocation (+ optional pinned host mirror)."""

    def __init__(self, nbytes: int, pinned_host: bool):
        p = ctypes.c_void_p()
        native.call("gts_b200_malloc", ctypes.byref(p), int(nbytes))
        self.dptr = p.value
        self.nbytes = int(nbytes)
        self.hptr = None
        if pinned_host:
            h = ctypes.c_void_p()
            native.call("gts_b200_host_alloc", ctypes.byref(h), int(nbytes))
            self.hptr = h.value
        self._fin = weakref.finalize(self, _DeviceBuffer._release, self.dptr, self.hptr)

    @staticmethod
    def _release(dptr, hptr):  # pragma: no cover - GC path
        try:
            lib = native.lib()
            if dptr:
                lib.gts_b200_free(dptr)
            if hptr:
                lib.gts_b200_host_free(hptr)
        except Exception:
            pass


class DeviceFieldStorage(FieldStorage):
    """A FieldStorage whose buffer lives on the B200 (see module docstring)."""

    def __init__(self, dtype: str, shape, origin, layout: LayoutSpec):
        if dtype not in _NP:
            raise StorageError(Code.ALLOCATION, f"unknown dtype '{dtype}'")
        np_dtype = _NP[dtype]
        layout.validate(np_dtype.itemsize)
        strides, total = _strides(shape, layout, np_dtype.itemsize)
        slack = layout.alignment_bytes // np_dtype.itemsize
        self.device = native.require_device()
        self._buf = _DeviceBuffer((total + slack) * np_dtype.itemsize, pinned_host=True)
        origin_linear = sum(o * s for o, s in zip(origin, strides))
        a = layout.alignment_bytes
        dshift = ((-(self._buf.dptr + origin_linear * np_dtype.itemsize)) % a) // np_dtype.itemsize
        hshift = ((-(self._buf.hptr + origin_linear * np_dtype.itemsize)) % a) // np_dtype.itemsize
        self._dshift, self._hshift, self._total = dshift, hshift, total
        raw = (ctypes.c_char * self._buf.nbytes).from_address(self._buf.hptr)
        host_flat = np.frombuffer(raw, dtype=np_dtype)
        self._host_view = np.lib.stride_tricks.as_strided(
            host_flat[hshift: hshift + total], shape=tuple(shape),
            strides=tuple(s * np_dtype.itemsize for s in strides))
        # FieldStorage fields (storage.py:74-90)
        self.dtype = dtype
        self.shape = tuple(int(x) for x in shape)
        self.origin = tuple(int(x) for x in origin)
        self.layout = layout
        self.strides = strides
        self._base = host_flat
        self._host_dirty = True  # nothing uploaded yet
        self._device_dirty = False
        self._pending_stream = None  # stream of an asynchronous write not yet waited for
        self._sync_lock = threading.RLock()

    # -- FieldStorage surface ------------------------------------------------
    @property
    def view(self) -> np.ndarray:  # type: ignore[override]
        self.to_host()
        self._host_dirty = True  # the caller may write through the view
        return self._host_view

    @view.setter
    def view(self, value) -> None:  # pragma: no cover - dataclass compatibility
        raise AttributeError("DeviceFieldStorage.view is managed by the storage")

    def base_address(self) -> int:
        """Device address of storage element (0, 0, 0) (cf. storage.py:96)."""
        return self._buf.dptr + self._dshift * self.itemsize

    @property
    def nbytes_span(self) -> int:
        return self._total * self.itemsize

    # -- synchronisation -----------------------------------------------------
    def _host_span_addr(self) -> int:
        return self._buf.hptr + self._hshift * self.itemsize

    def to_device(self, stream: Optional[int] = None, sync: bool = True) -> None:
        """Upload a pending host write (``sync=False``: the copy stays queued
        on ``stream``, so only launches on that same stream may follow
        without a wait; used inside a single-threaded graph capture)."""
        if not self._host_dirty:
            return
        with self._sync_lock:
            if self._host_dirty:
                s = native.default_stream() if stream is None else stream
                native.call("gts_b200_memcpy_h2d", self.base_address(), self._host_span_addr(),
                            self.nbytes_span, s)
                if sync:
                    native.synchronize(s)
                self._host_dirty = False

    def to_host(self, stream: Optional[int] = None) -> None:
        if not self._device_dirty:
            return
        with self._sync_lock:
            if self._device_dirty:
                s = native.default_stream() if stream is None else stream
                pend = self._pending_stream
                if pend is not None and pend != s:
                    native.synchronize(pend)
                native.call("gts_b200_memcpy_d2h", self._host_span_addr(), self.base_address(),
                            self.nbytes_span, s)
                native.synchronize(s)
                self._device_dirty = False
                self._pending_stream = None

    def mark_device_written(self, stream: Optional[int] = None) -> None:
        """A launch wrote the device copy: asynchronously on ``stream``
        (not yet synchronised), or ``None`` for a completed write."""
        self._device_dirty = True
        self._pending_stream = stream

    def wait_producer(self, stream: int) -> None:
        """Order ``stream`` after the last asynchronous write of another
        stream (host-side wait; the common single-stream case costs nothing)."""
        pend = self._pending_stream
        if pend is not None and pend != stream:
            native.synchronize(pend)
            self._pending_stream = None

    def host_array(self) -> np.ndarray:
        """Synchronised read-only copy of the logical array (no dirty mark)."""
        self.to_host()
        return np.array(self._host_view)

    @property
    def __cuda_array_interface__(self) -> dict:
        typestr = "<f4" if self.dtype == "f32" else "<f8"
        return {
            "shape": self.shape,
            "typestr": typestr,
            "data": (self.base_address(), False),
            "strides": tuple(s * self.itemsize for s in self.strides),
            "version": 3,
        }

    def __repr__(self) -> str:
        return (f"DeviceFieldStorage(dtype={self.dtype!r}, shape={self.shape}, "
                f"origin={self.origin}, strides={self.strides}, device={self.device})")


class ExternalDeviceFieldStorage(DeviceFieldStorage):
    """Zero-copy DeviceFieldStorage over a device array owned elsewhere (any
    object exporting ``__cuda_array_interface__`` v2/v3: a torch.cuda tensor,
    CuPy, Numba).  The stencil reads and writes the caller's memory in place;
    ``view`` / ``host_array()`` go through a pinned host mirror like the
    owning storage.  The array must be 3-D in logical (i, j, k) order with
    the b200 axis order (k outermost, j contiguous: strides s_k >= s_i >= s_j
    = 1 element), e.g. ``torch.empty(nk, ni, nj).permute(1, 2, 0)``; any
    padding is allowed (kernels needing 16-B aligned strides for TMA fall
    back to their plain form at run time)."""

    def __init__(self, obj, origin=(0, 0, 0)):  # noqa: D107 - documented above
        cai = getattr(obj, "__cuda_array_interface__", None)
        if cai is None:
            raise StorageError(Code.ALLOCATION, f"{type(obj).__name__} has no __cuda_array_interface__")
        shape = tuple(int(x) for x in cai["shape"])
        if len(shape) != 3:
            raise StorageError(Code.ALLOCATION, f"expected a 3-D array, got shape {shape}")
        dtype = {"<f8": "f64", "<f4": "f32"}.get(np.dtype(cai["typestr"]).str)
        if dtype is None:
            raise StorageError(Code.ALLOCATION, f"unsupported element type {cai['typestr']!r}")
        item = _NP[dtype].itemsize
        bstrides = cai.get("strides")
        if bstrides is None:  # C-contiguous
            bstrides = (shape[1] * shape[2] * item, shape[2] * item, item)
        if any(b % item or b <= 0 for b in bstrides):
            raise StorageError(Code.ALLOCATION, f"strides {bstrides} are not positive element multiples")
        strides = tuple(b // item for b in bstrides)
        si, sj, sk = strides
        if not (sj == 1 and si >= shape[1] and sk >= si * shape[0]):
            raise StorageError(Code.ALLOCATION,
                               f"strides {strides} (elements, i/j/k) are not the b200 axis order "
                               "(k outermost, j contiguous)")
        ptr, _readonly = cai["data"]
        stream = cai.get("stream")
        if stream:  # v3: work queued on the producer's stream must finish first
            native.call("gts_b200_stream_synchronize", int(stream))
        self._sync_lock = threading.RLock()
        self._pending_stream = None
        self._ev = None
        self.device = native.require_device()
        self._ext, self._ptr = obj, int(ptr)
        total = 1 + sum((n - 1) * st for n, st in zip(shape, strides))
        self._total = total
        self._host = _PinnedHost(total * item)
        raw = (ctypes.c_char * (total * item)).from_address(self._host.hptr)
        host_flat = np.frombuffer(raw, dtype=_NP[dtype])
        self._host_view = np.lib.stride_tricks.as_strided(
            host_flat, shape=shape, strides=tuple(x * item for x in strides))
        self.dtype = dtype
        self.shape = shape
        self.origin = tuple(int(x) for x in origin)
        self.layout = B200_LAYOUT
        self.strides = strides
        self._base = host_flat
        self._host_dirty = False  # the device copy is the authoritative one
        self._device_dirty = True  # the host mirror has never been filled

    def base_address(self) -> int:
        return self._ptr

    def _host_span_addr(self) -> int:
        return self._host.hptr

    @property
    def view(self) -> np.ndarray:  # type: ignore[override]
        """Read-only host snapshot: the device array is the authoritative
        copy (write to the producer's array, e.g. the torch tensor, instead);
        the host mirror is never uploaded over it."""
        self.to_host()
        v = self._host_view.view()
        v.flags.writeable = False
        return v

    @view.setter
    def view(self, value) -> None:  # pragma: no cover - dataclass compatibility
        raise AttributeError("ExternalDeviceFieldStorage.view is read-only")

    def wait_producer(self, stream: int) -> None:
        """Order ``stream`` after the work the array's producer has queued
        on ITS current stream (``__cuda_array_interface__`` v3 ``stream``,
        re-read on every launch: a torch tensor reports the torch current
        stream), without a host wait."""
        super().wait_producer(stream)
        cai = getattr(self._ext, "__cuda_array_interface__", None) or {}
        prod = cai.get("stream")
        if prod and int(prod) != stream:
            if self._ev is None:
                self._ev = native.Event()
            native.call("gts_b200_event_record", self._ev.ptr, int(prod))
            native.call("gts_b200_stream_wait_event", stream, self._ev.ptr)


def from_cuda_array(obj, origin=(0, 0, 0)) -> ExternalDeviceFieldStorage:
    """Wrap a device array (``__cuda_array_interface__``) without copying."""
    return ExternalDeviceFieldStorage(obj, origin)


def allocate(dtype: str, compute_shape, halo=(0, 0, 0), layout: Optional[LayoutSpec] = None,
             fill: Union[str, float] = "zeros") -> DeviceFieldStorage:
    """Device twin of ``stencilforge.allocate`` (storage.py:163-192)."""
    if dtype not in _NP:
        raise StorageError(Code.ALLOCATION, f"unknown dtype '{dtype}'")
    if any(c < 1 for c in compute_shape):
        raise StorageError(Code.ALLOCATION, f"compute shape must be >= 1 per axis, got {compute_shape}")
    if any(h < 0 for h in halo):
        raise StorageError(Code.ALLOCATION, f"halo must be >= 0 per axis, got {halo}")
    shape = tuple(c + 2 * h for c, h in zip(compute_shape, halo))
    st = DeviceFieldStorage(dtype, shape, tuple(halo), layout or B200_LAYOUT)
    hv = st._host_view
    if fill == "zeros":
        hv[...] = 0
    elif fill == "poison":
        hv[...] = np.nan
    elif isinstance(fill, (int, float)):
        hv[...] = fill
    else:
        raise StorageError(Code.ALLOCATION, f"unknown fill mode {fill!r}")
    st.to_device()
    return st


def from_array(values, origin=(0, 0, 0), layout: Optional[LayoutSpec] = None,
               dtype: Optional[str] = None) -> DeviceFieldStorage:
    """Device twin of ``stencilforge.from_array`` (storage.py:195-208)."""
    values = np.asarray(values)
    if values.ndim != 3:
        raise StorageError(Code.ALLOCATION, f"expected a 3-D array, got ndim={values.ndim}")
    dt = dtype or ("f32" if values.dtype == np.float32 else "f64")
    st = DeviceFieldStorage(dt, values.shape, tuple(origin), layout or B200_LAYOUT)
    st._host_view[...] = values
    st.to_device()
    return st


def to_device(storage: FieldStorage) -> DeviceFieldStorage:
    """Device copy of any host FieldStorage (values, shape, origin, layout)."""
    st = DeviceFieldStorage(storage.dtype, storage.shape, storage.origin, storage.layout)
    st._host_view[...] = storage.view
    st.to_device()
    return st


class _PinnedHost:
    """Owning pinned host allocation backing a host FieldStorage."""

    def __init__(self, nbytes: int):
        h = ctypes.c_void_p()
        native.call("gts_b200_host_alloc", ctypes.byref(h), int(nbytes))
        self.hptr = h.value
        self._fin = weakref.finalize(self, _PinnedHost._release, self.hptr)

    @staticmethod
    def _release(hptr):  # pragma: no cover - GC path
        try:
            native.lib().gts_b200_host_free(hptr)
        except Exception:
            pass


def pinned_host_storage(dtype: str, compute_shape, halo=(0, 0, 0),
                        layout: Optional[LayoutSpec] = None) -> FieldStorage:
    """A plain reference FieldStorage (host, storage.py:74-103) whose buffer
    is page-locked, so mirror-mode copies run at full PCIe/C2C speed."""
    layout = layout or B200_LAYOUT
    np_dtype = _NP[dtype]
    shape = tuple(c + 2 * h for c, h in zip(compute_shape, halo))
    strides, total = _strides(shape, layout, np_dtype.itemsize)
    slack = layout.alignment_bytes // np_dtype.itemsize
    owner = _PinnedHost((total + slack) * np_dtype.itemsize)
    raw = (ctypes.c_char * ((total + slack) * np_dtype.itemsize)).from_address(owner.hptr)
    base = np.frombuffer(raw, dtype=np_dtype)
    origin_linear = sum(o * s for o, s in zip(halo, strides))
    shift = ((-(owner.hptr + origin_linear * np_dtype.itemsize)) % layout.alignment_bytes) // np_dtype.itemsize
    view = np.lib.stride_tricks.as_strided(
        base[shift: shift + total], shape=shape,
        strides=tuple(s * np_dtype.itemsize for s in strides))
    view[...] = 0
    st = FieldStorage(dtype=dtype, shape=shape, origin=tuple(halo), layout=layout,
                      strides=strides, view=view, _base=base)
    st._pinned_owner = owner  # keep the allocation alive with the storage
    return st


def read_gtsf(source, layout: Optional[LayoutSpec] = None) -> DeviceFieldStorage:
    """GTSF file -> device storage (the reference reader, storage.py:250-280,
    then one upload); the b200 layout unless ``layout`` says otherwise."""
    host = sf_storage.read_gtsf(source, layout or B200_LAYOUT)
    return to_device(host)


def write_gtsf(storage: FieldStorage, sink) -> None:
    """Device (or host) storage -> GTSF file, bit-exact (storage.py:230-247);
    a device storage is read back once through its host mirror."""
    sf_storage.write_gtsf(storage, sink)
