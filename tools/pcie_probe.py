"""Host<->device copy bandwidth from pinned memory (the e2e ceiling)."""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2311_08322_b200 import native  # noqa: E402

n = 168 * 1024 * 1024
h, d, d2, h2 = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
native.call("gts_b200_host_alloc", ctypes.byref(h), n)
native.call("gts_b200_host_alloc", ctypes.byref(h2), n)
native.call("gts_b200_malloc", ctypes.byref(d), n)
native.call("gts_b200_malloc", ctypes.byref(d2), n)
s, s2 = native.default_stream(), native.aux_stream("probe")
e0, e1 = native.Event(), native.Event()
for label, fn in (
    ("h2d one copy", lambda: native.call("gts_b200_memcpy_h2d", d.value, h.value, n, s)),
    ("d2h one copy", lambda: native.call("gts_b200_memcpy_d2h", h.value, d.value, n, s)),
    ("h2d 8 chunks", lambda: [native.call("gts_b200_memcpy_h2d", d.value + i * (n // 8), h.value + i * (n // 8), n // 8, s)
                              for i in range(8)]),
):
    fn()
    native.synchronize(s)
    e0.record(s)
    for _ in range(3):
        fn()
    e1.record(s)
    native.synchronize(s)
    ms = e0.elapsed_ms(e1) / 3
    print(f"{label}: {ms:.3f} ms  {n / ms / 1e6:.1f} GB/s", flush=True)
# full duplex: h2d on s, d2h on s2 concurrently
native.synchronize(s)
e0.record(s)
native.call("gts_b200_memcpy_h2d", d.value, h.value, n, s)
native.call("gts_b200_memcpy_d2h", h2.value, d2.value, n // 4, s2)
native.synchronize(s2)
e1.record(s)
native.synchronize(s)
ms = e0.elapsed_ms(e1)
print(f"h2d {n >> 20} MiB + concurrent d2h {n >> 22} MiB: {ms:.3f} ms", flush=True)
# the pipelined mirror mode's copy shape: per field and i-row chunk, nk rows of
# (chunk rows x row pitch) bytes, k-plane pitch apart (memcpy2d)
nk, plane = 80, 256 * 264 * 8
for rows in (32, 64, 128):
    width = rows * 264 * 8
    nch = 256 // rows

    def two_d():
        for f in range(4):
            for c in range(nch):
                off = f * (n // 4)
                native.call("gts_b200_memcpy2d_h2d", d.value + off + c * width, plane,
                            h.value + off + c * width, plane, width, nk, s)

    two_d()
    native.synchronize(s)
    e0.record(s)
    two_d()
    e1.record(s)
    native.synchronize(s)
    ms = e0.elapsed_ms(e1)
    tot = 4 * nk * plane
    print(f"memcpy2d h2d chunk rows {rows}: {ms:.3f} ms for {tot / 1e6:.1f} MB  {tot / ms / 1e6:.1f} GB/s", flush=True)
# the pipeline's exact order: chunk-major over 4 separate pinned fields of the
# vadv layout (row pitch 2048 B, plane pitch 512 KiB), 8 chunks of 32 rows
hs, ds = [], []
fb = 256 * 256 * 80 * 8
for _ in range(4):
    a, b = ctypes.c_void_p(), ctypes.c_void_p()
    native.call("gts_b200_host_alloc", ctypes.byref(a), fb)
    native.call("gts_b200_malloc", ctypes.byref(b), fb)
    hs.append(a.value)
    ds.append(b.value)


def pipe_order():
    for c in range(8):
        for f in range(4):
            off = c * 32 * 2048
            native.call("gts_b200_memcpy2d_h2d", ds[f] + off, 256 * 2048, hs[f] + off, 256 * 2048, 32 * 2048, 80, s)


pipe_order()
native.synchronize(s)
e0.record(s)
pipe_order()
e1.record(s)
native.synchronize(s)
ms = e0.elapsed_ms(e1)
print(f"pipeline-order h2d (4 pinned fields, 8 chunks): {ms:.3f} ms  {4 * fb / ms / 1e6:.1f} GB/s", flush=True)
# H2D (pipeline order) with concurrent 2-D D2H chunks of an output field
xo_h, xo_d = ctypes.c_void_p(), ctypes.c_void_p()
native.call("gts_b200_host_alloc", ctypes.byref(xo_h), fb)
native.call("gts_b200_malloc", ctypes.byref(xo_d), fb)
for rows in (32, 64):
    def both():
        nchk = 256 // rows
        for c in range(nchk):
            for f in range(4):
                off = c * rows * 2048
                native.call("gts_b200_memcpy2d_h2d", ds[f] + off, 256 * 2048, hs[f] + off, 256 * 2048, rows * 2048, 80, s)
            off = c * rows * 2048
            native.call("gts_b200_memcpy2d_d2h", xo_h.value + off, 256 * 2048, xo_d.value + off, 256 * 2048, rows * 2048, 80, s2)
    both()
    native.synchronize(s)
    native.synchronize(s2)
    e0.record(s)
    ea, eb = native.Event(), native.Event()
    both()
    e1.record(s)
    eb.record(s2)
    native.synchronize(s)
    native.synchronize(s2)
    print(f"h2d + concurrent 2-D d2h chunks ({rows} rows): h2d {e0.elapsed_ms(e1):.3f} ms, all {e0.elapsed_ms(eb):.3f} ms",
          flush=True)
