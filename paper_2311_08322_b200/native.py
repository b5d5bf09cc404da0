"""ctypes binding of libgts_b200.so (include/gts_b200.h).

The product path has no CPU fallback: if the library (or a CUDA device) is
missing, every call raises ``BackendError`` instead of computing anything on
the host.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from pathlib import Path
from typing import Optional

from ._host import BackendError, Code

PKG = Path(__file__).resolve().parent
REPO = PKG.parent
LIB_PATH = PKG / "libgts_b200.so"
RUNTIME_SRC = PKG / "csrc" / "gts_runtime.cu"

# name -> (restype, argtypes)
_c = ctypes
_VP, _I64, _SZ, _INT = _c.c_void_p, _c.c_int64, _c.c_size_t, _c.c_int
SIGNATURES = {
    "gts_b200_abi_version": (_INT, []),
    "gts_b200_error_string": (_c.c_char_p, [_INT]),
    "gts_b200_device_count": (_INT, [_c.POINTER(_INT)]),
    "gts_b200_nvtx_push": (_INT, [_c.c_char_p]),
    "gts_b200_nvtx_pop": (_INT, []),
    "gts_b200_set_device": (_INT, [_INT]),
    "gts_b200_get_device": (_INT, [_c.POINTER(_INT)]),
    "gts_b200_device_info": (_INT, [_INT, _c.POINTER(_INT), _c.POINTER(_INT), _c.POINTER(_INT),
                                    _c.POINTER(_SZ)]),
    "gts_b200_malloc": (_INT, [_c.POINTER(_VP), _SZ]),
    "gts_b200_free": (_INT, [_VP]),
    "gts_b200_host_alloc": (_INT, [_c.POINTER(_VP), _SZ]),
    "gts_b200_host_free": (_INT, [_VP]),
    "gts_b200_host_register": (_INT, [_VP, _SZ, _c.POINTER(_INT)]),
    "gts_b200_host_unregister": (_INT, [_VP]),
    "gts_b200_memset": (_INT, [_VP, _INT, _SZ, _VP]),
    "gts_b200_memcpy_h2d": (_INT, [_VP, _VP, _SZ, _VP]),
    "gts_b200_memcpy_d2h": (_INT, [_VP, _VP, _SZ, _VP]),
    "gts_b200_memcpy_d2d": (_INT, [_VP, _VP, _SZ, _VP]),
    "gts_b200_stream_create": (_INT, [_c.POINTER(_VP)]),
    "gts_b200_stream_destroy": (_INT, [_VP]),
    "gts_b200_stream_synchronize": (_INT, [_VP]),
    "gts_b200_event_create": (_INT, [_c.POINTER(_VP)]),
    "gts_b200_event_destroy": (_INT, [_VP]),
    "gts_b200_event_record": (_INT, [_VP, _VP]),
    "gts_b200_event_synchronize": (_INT, [_VP]),
    "gts_b200_event_record_dep": (_INT, [_VP, _VP]),
    "gts_b200_flags_add": (_INT, [_VP, _INT, _VP]),
    "gts_b200_flags_wait_next": (_INT, [_VP, _VP, _INT, _VP]),
    "gts_b200_event_elapsed_ms": (_INT, [_c.POINTER(_c.c_float), _VP, _VP]),
    "gts_b200_l2_flush": (_INT, [_VP]),
    "gts_b200_l2_evict_read": (_INT, [_VP, _c.POINTER(_SZ)]),
    "gts_b200_profiler_start": (_INT, []),
    "gts_b200_profiler_stop": (_INT, []),
    "gts_b200_pack_box": (_INT, [_VP, _VP] + [_I64] * 9 + [_INT, _VP]),
    "gts_b200_unpack_box": (_INT, [_VP, _VP] + [_I64] * 9 + [_INT, _VP]),
    "gts_b200_memcpy2d_h2d": (_INT, [_VP, _SZ, _VP, _SZ, _SZ, _SZ, _VP]),
    "gts_b200_memcpy2d_d2h": (_INT, [_VP, _SZ, _VP, _SZ, _SZ, _SZ, _VP]),
    "gts_b200_stream_wait_event": (_INT, [_VP, _VP]),
    "gts_b200_graph_begin": (_INT, [_VP]),
    "gts_b200_graph_end": (_INT, [_VP, _c.POINTER(_VP)]),
    "gts_b200_graph_launch": (_INT, [_VP, _VP]),
    "gts_b200_graph_destroy": (_INT, [_VP]),
    "gts_b200_ipc_get_handle": (_INT, [_VP, _VP, _c.POINTER(_SZ)]),
    "gts_b200_ipc_open": (_INT, [_VP, _c.POINTER(_VP)]),
    "gts_b200_ipc_close": (_INT, [_VP]),
    "gts_b200_copy_box": (_INT, [_VP] + [_I64] * 3 + [_VP] + [_I64] * 6 + [_INT, _VP]),
    "gts_b200_flag_signal": (_INT, [_VP, _c.c_uint64, _VP]),
    "gts_b200_flag_wait": (_INT, [_VP, _c.c_uint64, _VP]),
    "gts_b200_flag_add": (_INT, [_VP, _VP]),
    "gts_b200_flag_wait_next": (_INT, [_VP, _VP, _VP]),
}

_lib: Optional[ctypes.CDLL] = None
_lock = threading.Lock()


def nvcc_runtime_cmd() -> list:
    from .toolchain import ARCH_FLAGS, nvcc_command

    return [nvcc_command(), "-O3", "-std=c++17", *ARCH_FLAGS, "-lineinfo",
            "-Xcompiler", "-fPIC", "-shared", f"-I{REPO / 'include'}",
            str(RUNTIME_SRC), "-o", str(LIB_PATH)]


def build_runtime(force: bool = False) -> Path:
    """Compile libgts_b200.so in-tree (cross-compiles without a GPU)."""
    if not force and LIB_PATH.exists() and LIB_PATH.stat().st_mtime >= max(
        RUNTIME_SRC.stat().st_mtime, (REPO / "include" / "gts_b200.h").stat().st_mtime
    ):
        return LIB_PATH
    env = dict(os.environ)
    env.pop("CC", None)
    tmp = LIB_PATH.with_suffix(".so.tmp")
    cmd = nvcc_runtime_cmd()
    cmd[-1] = str(tmp)
    proc = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=900)
    if proc.returncode != 0:
        raise BackendError(Code.COMPILE_FAILED, f"{' '.join(cmd)} failed:\n{proc.stderr}")
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise BackendError(
                    Code.TOOLCHAIN_MISSING,
                    f"{LIB_PATH} is missing; run __graft_entry__.build() "
                    "(the b200 backend has no CPU fallback)")
            handle = ctypes.CDLL(str(LIB_PATH))
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


def error_string(status: int) -> str:
    try:
        s = lib().gts_b200_error_string(int(status))
        return s.decode() if s else f"error {status}"
    except Exception:  # pragma: no cover - library missing
        return f"error {status}"


class DeviceError(BackendError):
    """A CUDA runtime / launch failure on the device path."""

    def __init__(self, status: int, what: str):
        super().__init__(Code.TOOLCHAIN_MISSING if status in (35, 100, 999) else Code.COMPILE_FAILED,
                         f"{what}: {error_string(status)} (status {status})")
        self.status = status


def check(status: int, what: str) -> None:
    if status:
        raise DeviceError(int(status), what)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args), name)


# ---------------------------------------------------------------------------
# Devices and streams
# ---------------------------------------------------------------------------

def device_count() -> int:
    n = ctypes.c_int(0)
    st = lib().gts_b200_device_count(ctypes.byref(n))
    return 0 if st else n.value


def current_device() -> int:
    d = ctypes.c_int(0)
    call("gts_b200_get_device", ctypes.byref(d))
    return d.value


def set_device(dev: int) -> None:
    call("gts_b200_set_device", int(dev))


def require_device() -> int:
    if device_count() < 1:
        raise DeviceError(100, "no CUDA device visible to the b200 backend")
    return current_device()


class _ThreadStreams:
    """The calling thread's backend streams on one device.  Threads get
    their own streams so concurrent calls never share a stream,
    a temporary arena (gts_common.cuh ``GtsArenaLease``, keyed by stream) or
    a mirror buffer; a finished thread's streams go back to a pool."""

    _pool: dict = {}  # (device, name) -> [free stream handles]
    _pool_lock = threading.Lock()

    def __init__(self, dev: int):
        self.dev = dev
        self.streams: dict = {}

    def get(self, name: str) -> int:
        s = self.streams.get(name)
        if s is None:
            with _ThreadStreams._pool_lock:
                free = _ThreadStreams._pool.get((self.dev, name))
                s = free.pop() if free else None
            if s is None:
                p = ctypes.c_void_p()
                call("gts_b200_stream_create", ctypes.byref(p))
                s = p.value
            self.streams[name] = s
        return s

    def __del__(self):  # pragma: no cover - thread teardown
        try:
            with _ThreadStreams._pool_lock:
                for name, s in self.streams.items():
                    _ThreadStreams._pool.setdefault((self.dev, name), []).append(s)
        except Exception:
            pass


_tls = threading.local()


def _thread_streams(dev: int) -> _ThreadStreams:
    per = getattr(_tls, "streams", None)
    if per is None:
        per = _tls.streams = {}
    ts = per.get(dev)
    if ts is None:
        ts = per[dev] = _ThreadStreams(dev)
    return ts


def aux_stream(name: str) -> int:
    """Extra non-blocking streams of the calling thread (the mirror-mode
    copy engines, the halo exchange)."""
    return _thread_streams(require_device()).get("aux:" + name)


def default_stream() -> int:
    """The calling thread's non-blocking stream on the current device, owned
    by the backend."""
    return _thread_streams(require_device()).get("default")


def synchronize(stream: Optional[int] = None) -> None:
    call("gts_b200_stream_synchronize", stream if stream is not None else default_stream())


def device_info(dev: Optional[int] = None) -> dict:
    dev = current_device() if dev is None else dev
    sm, l2, cc = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    hbm = ctypes.c_size_t()
    call("gts_b200_device_info", dev, ctypes.byref(sm), ctypes.byref(l2), ctypes.byref(cc),
         ctypes.byref(hbm))
    return {"sm_count": sm.value, "l2_bytes": l2.value, "cc": cc.value, "hbm_bytes": hbm.value}


class Event:
    def __init__(self):
        p = ctypes.c_void_p()
        call("gts_b200_event_create", ctypes.byref(p))
        self.ptr = p.value

    def record(self, stream: Optional[int] = None) -> None:
        call("gts_b200_event_record", self.ptr, stream if stream is not None else default_stream())

    def record_dep(self, stream: int) -> None:
        """Cross-stream ordering marker (captures as a graph dependency)."""
        call("gts_b200_event_record_dep", self.ptr, stream)

    def synchronize(self) -> None:
        call("gts_b200_event_synchronize", self.ptr)

    def elapsed_ms(self, end: "Event") -> float:
        ms = ctypes.c_float()
        call("gts_b200_event_elapsed_ms", ctypes.byref(ms), self.ptr, end.ptr)
        return float(ms.value)

    def __del__(self):  # pragma: no cover - best effort
        try:
            if self.ptr and _lib is not None:
                _lib.gts_b200_event_destroy(self.ptr)
        except Exception:
            pass


def l2_flush(stream: Optional[int] = None) -> None:
    call("gts_b200_l2_flush", stream if stream is not None else default_stream())


class Graph:
    """A captured sequence of enqueues on one stream, replayed with a single
    launch (``gts_b200_graph_*``).  Use as::

        g = Graph(stream)
        with g.capture():
            launcher(); launcher(); ...
        g.launch()
    """

    def __init__(self, stream: Optional[int] = None):
        self.stream = stream if stream is not None else default_stream()
        self.ptr = None

    def capture(self):
        graph = self

        class _Cap:
            def __enter__(self_):
                call("gts_b200_graph_begin", graph.stream)
                return graph

            def __exit__(self_, et, ev, tb):
                p = ctypes.c_void_p()
                st = lib().gts_b200_graph_end(graph.stream, ctypes.byref(p))
                if et is None:
                    check(st, "gts_b200_graph_end")
                    graph.ptr = p.value
                return False

        return _Cap()

    def launch(self) -> None:
        if self.ptr is None:
            raise BackendError(Code.TOOLCHAIN_MISSING, "graph launched before capture")
        call("gts_b200_graph_launch", self.ptr, self.stream)

    def __del__(self):  # pragma: no cover - best effort
        try:
            if self.ptr and _lib is not None:
                _lib.gts_b200_graph_destroy(self.ptr)
        except Exception:
            pass
