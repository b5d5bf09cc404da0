"""Where one e2e call's time goes (vadv 256^2x80, host pinned storages through
CompiledStencil.__call__, the default pipelined mirror mode): wall time per
call against the device span from the first host->device copy to the last
device->host copy (backend.PIPE_TRACE), and the H2D-only floor."""
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2311_08322_b200 as b200  # noqa: E402
from paper_2311_08322_b200 import backend, workloads  # noqa: E402

st = b200.compile_stencil(workloads.source("vadv"), "vadv")
dt, h2d, d2h, ch = bench.e2e_timed(st, "vadv", "f64", (256, 256, 80), 20)
print(f"e2e {dt * 1e3:.3f} ms/call, h2d {h2d / 1e6:.1f} MB d2h {d2h / 1e6:.1f} MB chunks {ch}", flush=True)
from paper_2311_08322_b200 import storage as b2s  # noqa: E402

host = workloads.make_args("vadv", (256, 256, 80), "f64", device=False)
args = {}
for n, v in host.items():
    p = b2s.pinned_host_storage(v.dtype, tuple(s - 2 * h for s, h in zip(v.shape, v.origin)), v.origin)
    p.view[...] = v.view
    args[n] = p
st(**args)
backend.PIPE_TRACE = []
walls = []
for _ in range(10):
    t0 = time.perf_counter()
    st(**args)
    walls.append(time.perf_counter() - t0)
tr = backend.PIPE_TRACE
backend.PIPE_TRACE = None
print(f"traced: wall median {statistics.median(walls) * 1e3:.3f} ms; device spans from first H2D: "
      f"h2d {statistics.median(t['h2d_ms'] for t in tr):.3f} kernels {statistics.median(t['kernels_ms'] for t in tr):.3f} "
      f"d2h {statistics.median(t['d2h_ms'] for t in tr):.3f} ms", flush=True)


def traced(n=6):
    backend.PIPE_TRACE = []
    for _ in range(n):
        st(**args)
    tr = backend.PIPE_TRACE
    backend.PIPE_TRACE = None
    return " ".join(f"{k[:-3]} {statistics.median(t[k] for t in tr):.3f}" for k in ("h2d_ms", "kernels_ms", "d2h_ms"))


mod = st.build_info["module"]
real_launch = mod.launch
mod.launch = lambda *a, **k: None
print("ablation, no kernels:", traced(), flush=True)
mod.launch = real_launch
from paper_2311_08322_b200 import native  # noqa: E402

real_call = native.call
backend.native.call = lambda name, *a: None if name == "gts_b200_memcpy2d_d2h" else real_call(name, *a)
print("ablation, no d2h:", traced(), flush=True)
backend.native.call = real_call
for rows, taper in ((64, False), (128, True), (32, True), (48, True), (96, True)):
    backend._Pipeline.CHUNK_ROWS, backend._Pipeline.TAPER = rows, taper
    print(f"CHUNK_ROWS {rows} taper {taper}:", traced(), flush=True)
