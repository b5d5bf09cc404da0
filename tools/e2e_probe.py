"""e2e (host pinned storages through CompiledStencil.__call__) vs chunking."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2311_08322_b200 as b200  # noqa: E402
from paper_2311_08322_b200 import backend, native, workloads  # noqa: E402

st = b200.compile_stencil(workloads.source("vadv"), "vadv")
for rows in (16, 32, 64, 128, 256):
    backend._Pipeline.CHUNK_ROWS = rows
    dt, h2d, d2h, ch = bench.e2e_timed(st, "vadv", "f64", (256, 256, 80), 10)
    print(f"CHUNK_ROWS {rows}: {dt * 1e3:.3f} ms/call chunks {ch} h2d {h2d / 1e6:.1f} MB", flush=True)
# where the time goes at the default chunking: host enqueue vs device span
backend._Pipeline.CHUNK_ROWS = 32
host = workloads.make_args("vadv", (256, 256, 80), "f64", device=False)
from paper_2311_08322_b200 import storage as b2s  # noqa: E402
args = {}
for n, v in host.items():
    p = b2s.pinned_host_storage(v.dtype, tuple(s - 2 * h for s, h in zip(v.shape, v.origin)), v.origin)
    p.view[...] = v.view
    args[n] = p
st(**args)
exe = st.executable if hasattr(st, "executable") else None
orig_sync = native.synchronize
marks = {}


def timed_sync(stream=None):
    marks.setdefault("first_sync", time.perf_counter())
    orig_sync(stream)


native.synchronize = timed_sync
backend.PIPE_TRACE = []
t0 = time.perf_counter()
st(**args)
t1 = time.perf_counter()
native.synchronize = orig_sync
for _ in range(5):
    st(**args)
print("device spans from the first H2D (ms):", backend.PIPE_TRACE, flush=True)
backend.PIPE_TRACE = None
print(f"one call: {1e3 * (t1 - t0):.3f} ms wall, host enqueue done after {1e3 * (marks['first_sync'] - t0):.3f} ms",
      flush=True)
# ablations of the pipeline: no kernels / no D2H
mod = st.build_info["module"]
real_launch = mod.launch
backend.PIPE_TRACE = []
mod.launch = lambda *a, **k: None
for _ in range(4):
    st(**args)
print("no kernels:", [round(t["h2d_ms"], 3) for t in backend.PIPE_TRACE], flush=True)
mod.launch = real_launch
backend.PIPE_TRACE = []
real_call = native.call


def no_d2h(name, *a):
    if name == "gts_b200_memcpy2d_d2h":
        return None
    return real_call(name, *a)


backend.native.call = no_d2h
for _ in range(4):
    st(**args)
backend.native.call = real_call
print("no d2h:", [round(t["h2d_ms"], 3) for t in backend.PIPE_TRACE], flush=True)
backend.PIPE_TRACE = None
