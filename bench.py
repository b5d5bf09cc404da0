#!/usr/bin/env python
"""Benchmark: grid-points/s and achieved HBM GB/s of the b200 stencil backend.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

One JSON line on rank 0.  A "step" = one call of the stencil over the whole
configured domain.  Default workload (N=1) = BASELINE.json configs[1],
vertical advection 256x256x80 float64; hdiff 256x256x80 f64/f32 (configs[2])
are measured on the same run and reported under "extra".  For N>1 every rank
runs its own 256x256x80 shard (weak scaling; vadv columns are independent, no
data-path collective).

Protocol: inputs resident in HBM; R >= 3 rotating
input/output sets whose total exceeds 2x L2, so consecutive steps never hit
their own data in L2; W warm-up steps; K timed steps bracketed by
barrier + device synchronise; CUDA events on the launching stream; max over
ranks.  "e2e" = the same metric through the reference-facing API
(CompiledStencil.__call__) with host FieldStorages in pinned memory, the
host<->device copies inside the timed region.  "cpu_baseline" = the
reference's own native kernel (the C its gen engine emits, oracle/_ref) timed
on this host's cores on a bounded sample.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

WORKLOADS = {
    # name: (kernel, dtype, domain)
    "vadv": ("vadv", "f64", (256, 256, 80)),
    "hdiff": ("hdiff", "f64", (256, 256, 80)),
    "hdiff32": ("hdiff", "f32", (256, 256, 80)),
    "vadv32": ("vadv", "f32", (256, 256, 80)),
}
SHORT_TEXT = {"vadv": "vadv 256x256x80 f64", "hdiff": "hdiff 256x256x80 f64", "hdiff32": "hdiff 256x256x80 f32",
              "vadv32": "vadv 256x256x80 f32"}
CONFIG_TEXT = {
    "vadv": "vertical advection (FORWARD/BACKWARD Thomas) 256x256x80 float64",
    "hdiff": "horizontal diffusion 256x256x80 float64",
    "hdiff32": "horizontal diffusion 256x256x80 float32",
    "vadv32": "vertical advection 256x256x80 float32",
}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=1000)
    p.add_argument("--warmup", type=int, default=20)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--workload", default="vadv", choices=sorted(WORKLOADS))
    p.add_argument("--e2e-steps", type=int, default=20)
    p.add_argument("--cpu-seconds", type=float, default=12.0)
    p.add_argument("--no-extra", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-graph", action="store_true", help="eager launches in the timed loop")
    p.add_argument("--extra-timeout", type=float, default=420.0,
                   help="seconds the extra workloads may take before the headline line is printed without them")
    return p.parse_args()


# ---------------------------------------------------------------------------
# distributed plumbing (torch.distributed only for barrier / max-reduce)
# ---------------------------------------------------------------------------
class Dist:
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        # GTS_BENCH_SHARED_GPU=1: all ranks on the box's GPU(s) round-robin, gloo
        # for the plumbing -- exercises the N>1 code paths on a 1-GPU box (its
        # numbers are not scaling numbers)
        self.shared = os.environ.get("GTS_BENCH_SHARED_GPU") == "1"
        if self.world > 1:
            import torch
            import torch.distributed as dist

            backend = "nccl" if torch.cuda.is_available() and not self.shared else "gloo"
            if backend == "nccl":
                torch.cuda.set_device(self.local)
            dist.init_process_group(backend=backend)
            self.dist, self.torch, self.backend = dist, torch, backend

    def barrier(self):
        if self.world > 1:
            if self.backend == "nccl":
                self.dist.barrier(device_ids=[self.local])
            else:
                self.dist.barrier()

    def max(self, v: float) -> float:
        if self.world == 1:
            return v
        dev = f"cuda:{self.local}" if self.backend == "nccl" else "cpu"
        t = self.torch.tensor([v], dtype=self.torch.float64, device=dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


# ---------------------------------------------------------------------------
# clocks during the timed region (NVML)
# ---------------------------------------------------------------------------
class ClockSampler:
    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
        "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
    }

    def __init__(self, device: int):
        self.samples, self.reasons = [], set()
        self.ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, bit in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons)}
        busy = [s for s in self.samples if s > 0]
        return {"sm_mhz": float(statistics.median(busy or self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons - {"gpu_idle"})}


def host_info():
    model = ""
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return os.cpu_count() or 1, model


# ---------------------------------------------------------------------------
# reference CPU implementation (oracle/_ref = the gen engine's own C kernels)
# ---------------------------------------------------------------------------
def _ref_kernel(key: str):
    man_path = REPO / "oracle" / "_ref" / "manifest.json"
    if not man_path.exists():
        return None
    man = json.loads(man_path.read_text())[key]
    lib = ctypes.CDLL(str(REPO / "oracle" / "_ref" / man["so"]))
    fn = getattr(lib, man["symbol"])
    nf, ns = len(man["fields"]), len(man["scalars"])
    fn.argtypes = [ctypes.c_longlong] * 3 + ([ctypes.c_void_p] + [ctypes.c_longlong] * 6) * nf + \
        [ctypes.c_float if d == "f32" else ctypes.c_double for _, d in man["scalars"]]
    fn.restype = None
    return fn, man


def _ref_args(kernel, dtype, domain, seed=0):
    """Reference inputs in the gen layout (reference harness builders)."""
    import paper_2311_08322_b200  # noqa: F401  (locates stencilforge)
    import stencilforge as sf
    from stencilforge import bench as sf_bench

    args = sf_bench.KERNEL_BUILDERS[kernel]("gen", tuple(domain), seed)
    if dtype == "f32":
        for n, v in list(args.items()):
            if isinstance(v, sf.FieldStorage):
                st = sf.allocate("f32", tuple(d - 2 * o for d, o in zip(v.shape, v.origin)), v.origin, v.layout)
                st.view[...] = v.view.astype(np.float32)
                args[n] = st
    return args


def time_reference(kernel, dtype, domain, seconds: float, max_calls: int, warmup: int = 3):
    """Time the reference gen kernel on all host cores; returns (s per call, calls, kind)."""
    got = _ref_kernel(f"{kernel}_{dtype}")
    if got is None:
        return None
    fn, man = got
    args = _ref_args(kernel, dtype, domain)
    call = [int(domain[0]), int(domain[1]), int(domain[2])]
    for n in man["fields"]:
        st = args[n]
        call += [st.base_address(), *st.strides, *st.origin]
    for n, _ in man["scalars"]:
        call.append(float(args[n]))
    for _ in range(warmup):
        fn(*call)
    times = []
    t_end = time.perf_counter() + seconds
    while len(times) < max_calls and (not times or time.perf_counter() < t_end):
        t0 = time.perf_counter()
        fn(*call)
        times.append(time.perf_counter() - t0)
    return times


def arena_reuse_row(kernel, dtype, domain, seconds=4.0):
    """the gen kernel with glibc arena reuse.  The generated C
    allocates its temporary arena per call (gen.py:301-323, 361-362); above
    the mmap threshold every call maps fresh pages and page-faults them.  The
    survey's MALLOC_MMAP_THRESHOLD_/MALLOC_TRIM_THRESHOLD_ environment is read
    at process start, so the same effect is set here with mallopt (no mmap'd
    chunks, no trimming) for this row only, then restored."""
    pts = domain[0] * domain[1] * domain[2]
    try:
        libc = ctypes.CDLL(None)
        M_TRIM_THRESHOLD, M_MMAP_MAX = -1, -4
        if not (libc.mallopt(M_TRIM_THRESHOLD, 2 ** 31 - 1) and libc.mallopt(M_MMAP_MAX, 0)):
            return {"error": "mallopt refused"}
        try:
            t = time_reference(kernel, dtype, domain, seconds=seconds, max_calls=1000, warmup=3)
        finally:
            libc.mallopt(M_MMAP_MAX, 65536)
            libc.mallopt(M_TRIM_THRESHOLD, 128 * 1024)
    except Exception as exc:  # pragma: no cover - reported, not fatal
        return {"error": f"{type(exc).__name__}: {exc}"[:200]}
    if not t:
        return None
    return {"value": pts / statistics.median(t), "calls": len(t),
            "median_call_ms": statistics.median(t) * 1e3, "min_call_ms": min(t) * 1e3,
            "setting": "glibc arena reuse (mallopt M_MMAP_MAX=0, M_TRIM_THRESHOLD=2^31-1), all host threads"}


def cpu_rows(kernel, dtype, domain, cores, seconds=4.0):
    """SURVEY.md 8(d) secondary CPU rows: the gen kernel on 1 thread, the gen
    kernel with glibc arena reuse, and the reference's NumPy engine (vec)
    through its own compile_stencil."""
    rows = {}
    pts = domain[0] * domain[1] * domain[2]
    ar = arena_reuse_row(kernel, dtype, domain, seconds=seconds)
    if ar is not None:
        rows["gen_arena_reuse"] = ar
    os.environ["GTS_NUM_THREADS"] = "1"  # read by the generated C on every call (gen.py:296-299)
    try:
        t1 = time_reference(kernel, dtype, domain, seconds=seconds, max_calls=50, warmup=1)
        if t1:
            rows["gen_1_thread"] = {"value": pts / statistics.median(t1), "calls": len(t1),
                                    "median_call_ms": statistics.median(t1) * 1e3}
    finally:
        os.environ["GTS_NUM_THREADS"] = str(cores)
    try:
        import paper_2311_08322_b200  # noqa: F401  (locates stencilforge)
        from stencilforge import bench as sf_bench
        from stencilforge import runtime as sf_rt
        from stencilforge.kernels import kernel_source

        src = kernel_source(kernel)
        if dtype == "f32":
            src = src.replace("Field[f64]", "Field[f32]")
        st = sf_rt.compile_stencil(src, kernel, backend="vec")
        a = sf_bench.KERNEL_BUILDERS[kernel]("vec", tuple(domain), 0)
        st(**a)
        tv, t_end = [], time.perf_counter() + seconds
        while not tv or (time.perf_counter() < t_end and len(tv) < 20):
            t0 = time.perf_counter()
            st(**a)
            tv.append(time.perf_counter() - t0)
        rows["vec_numpy_1_thread"] = {"value": pts / statistics.median(tv), "calls": len(tv),
                                      "median_call_ms": statistics.median(tv) * 1e3}
    except Exception as exc:  # pragma: no cover - reported, not fatal
        rows["vec_numpy_1_thread"] = {"error": f"{type(exc).__name__}: {exc}"[:200]}
    return rows


def run_reference(args, dist):
    if dist.rank != 0:
        return
    kernel, dtype, domain = WORKLOADS[args.workload]
    pts = domain[0] * domain[1] * domain[2]
    cores, model = host_info()
    times = time_reference(kernel, dtype, domain, seconds=150.0, max_calls=args.steps,
                           warmup=max(args.warmup, 1))
    if times is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (run __graft_entry__.build() in the build container)"}))
        return
    total = sum(times)
    value = pts * len(times) / total
    line = {
        "metric": "grid-points/s", "value": value, "unit": "grid-points/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": len(times), "warmup": args.warmup,
        "ms_per_step": total / len(times) * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": dtype, "data": "synthetic",
        "config": {"workload": SHORT_TEXT[args.workload], "parallelism": f"openmp, {cores} host threads"},
        "cpu_baseline": {"value": value, "unit": "grid-points/s", "cores": cores, "kind": "reference",
                         "sample": f"{len(times)} full-domain calls of the reference gen engine's "
                                   f"generated C kernel (oracle/_ref, -O3 -fopenmp -ffp-contract=off), "
                                   f"OpenMP over all {cores} host threads ({model})"},
        "e2e": {"value": value, "unit": "grid-points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    ar = arena_reuse_row(kernel, dtype, domain, seconds=8.0)
    if ar is not None:
        line["cpu_baseline"]["rows"] = {"gen_arena_reuse": ar}
    print(json.dumps(line))


# ---------------------------------------------------------------------------
# b200
# ---------------------------------------------------------------------------
def measured_peak():
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        except Exception:
            pass
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(workload: str):
    p = REPO / "profiles" / "ncu_traffic.json"
    if p.exists():
        try:
            return json.loads(p.read_text()).get(workload)
        except Exception:
            return None
    return None


def _traffic_bytes(workload: str):
    """DRAM read + write bytes per launch of the workload's kernel from the
    committed ``ncu --set full`` capture (profiles/ncu_traffic.json)."""
    t = ncu_traffic(workload)
    return None if not t else t.get("traffic_bytes")


def device_timed(st, kernel, dtype, domain, steps, warmup, dist, sampler=None, use_graph=True):
    """Device-resident timing with rotating buffer sets."""
    from paper_2311_08322_b200 import native, workloads

    info = native.device_info()
    set_bytes = workloads.algorithmic_bytes(kernel, domain, dtype)
    nsets = max(3, -(-(3 * info["l2_bytes"]) // max(set_bytes, 1)))
    nsets = min(nsets, 16)
    stream = native.default_stream()
    module = st.build_info["module"]
    sets, launchers = [], []
    for s in range(nsets):
        a = workloads.make_args(kernel, domain, dtype, seed=s)
        sets.append(a)
        fields = {k: v for k, v in a.items() if hasattr(v, "base_address")}
        scal = {k: v for k, v in a.items() if not hasattr(v, "base_address")}
        launchers.append(module.launcher(domain, fields, scal, stream))
    for i in range(warmup):
        launchers[i % nsets]()
    native.synchronize(stream)
    ev = [(native.Event(), native.Event()) for _ in range(steps)]
    e0, e1 = native.Event(), native.Event()
    dist.barrier()
    native.synchronize(stream)
    ctx = sampler if sampler is not None else _Null()
    graph = None
    if use_graph:
        # the K timed launches (and their per-launch event records) captured
        # once into a CUDA graph, so the timed region measures the device,
        # not the Python launch loop; one untimed replay uploads the graph
        # (no per-launch event nodes: an event-record node between graph
        # kernels costs ~5 us, more than a 256^2 hdiff's own ramp; the mean
        # launch duration is the timed region / K, gaps included)
        graph = native.Graph(stream)
        n0 = module.launch_count()
        with graph.capture():
            for i in range(steps):
                launchers[(warmup + i) % nsets]()
        n_launch = module.launch_count() - n0
        graph.launch()
        native.synchronize(stream)
        dist.barrier()
    with ctx:
        e0.record(stream)
        if graph is not None:
            graph.launch()
        else:
            n0 = module.launch_count()
            for i in range(steps):
                ev[i][0].record(stream)
                launchers[(warmup + i) % nsets]()
                ev[i][1].record(stream)
        e1.record(stream)
        native.synchronize(stream)
        if graph is None:
            n_launch = module.launch_count() - n0
    dist.barrier()
    total_ms = e0.elapsed_ms(e1)
    if graph is not None:
        launch_ms = [total_ms / steps]
    else:
        launch_ms = [a.elapsed_ms(b) for a, b in ev]
    return {"total_ms": total_ms, "launch_ms_mean": statistics.fmean(launch_ms),
            "launch_ms_median": statistics.median(launch_ms), "nsets": nsets,
            "set_mb": set_bytes / 1e6, "l2_mb": info["l2_bytes"] / 1e6, "sets": sets,
            "launches": n_launch, "launches_per_step": n_launch / steps,
            "launch": ("cuda graph of the K timed steps; kernel time = timed region / K" if graph is not None
                       else "eager; kernel time = mean of per-launch event pairs")}


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def parity_check(kernel, dtype, sets):
    """The first buffer set vs the C oracle AND the reference gen engine's
    own kernel (oracle/_ref) on the same inputs: "bitwise" when both agree
    bit for bit."""
    sys.path.insert(0, str(REPO / "oracle"))
    import oracle

    a = sets[0]
    if kernel == "hdiff":
        ins = (a["inp"].host_array(), a["coeff"])
        got = a["out"].host_array()
        checks = [("oracle", oracle.hdiff_c)] + ([("ref", oracle.ref_hdiff)]
                                                 if oracle.ref_available(f"hdiff_{dtype}") else [])
    else:
        ins = tuple(a[n].host_array() for n in "abcd")
        got = a["x"].host_array()
        checks = [("oracle", oracle.vadv_c)] + ([("ref", oracle.ref_vadv)]
                                                if oracle.ref_available(f"vadv_{dtype}") else [])
    bad = []
    for name, fn in checks:
        want = fn(*ins)
        if not np.array_equal(got, want):
            bad.append(f"{name} max_rel {oracle.max_rel(got, want):.2e}")
    if bad:
        return "; ".join(bad)
    return "bitwise(" + "+".join(n for n, _ in checks) + ")"


def e2e_timed(st, kernel, dtype, domain, steps, pinned=True):
    """Through CompiledStencil.__call__ with HOST FieldStorages: the
    reference's own storages from its harness builder (make_<kernel>_args with
    the b200 layout: pageable numpy memory, stencilforge bench.py:82-105), or
    the same values in page-locked storages (storage.pinned_host_storage).
    Every call copies its inputs host -> device and its outputs back."""
    from paper_2311_08322_b200 import backend as b2b
    from paper_2311_08322_b200 import storage as b2s
    from paper_2311_08322_b200 import workloads

    host = workloads.make_args(kernel, domain, dtype, device=False)
    args = {}
    for n, v in host.items():
        if hasattr(v, "base_address") and pinned:
            halo = v.origin
            comp = tuple(s - 2 * h for s, h in zip(v.shape, halo))
            p = b2s.pinned_host_storage(v.dtype, comp, halo)
            p.view[...] = v.view
            args[n] = p
        else:
            args[n] = v
    st(**args)  # warm (allocates the device mirrors)
    t0 = time.perf_counter()
    for _ in range(steps):
        st(**args)
    dt = (time.perf_counter() - t0) / steps
    tr = dict(b2b.call_stats())  # bytes the last call actually moved
    return dt, tr["h2d"], tr["d2h"], tr["chunks"]


def decomposed_hdiff(dist, steps, warmup, tile=(512, 1024, 80), transport="nccl", split=None):
    """C4: hdiff on a horizontally decomposed domain, a fixed 512x1024x80
    tile per GPU (weak scaling; 2048x2048x80 at 8 GPUs on a 4x2 grid).  Each
    step = the halo exchange of inp (``nccl``: NCCL send/recv; ``peer``: CUDA
    IPC peer stores + flags) overlapped with the interior, then the boundary
    frame (decomp.DecomposedStep: 2 launches per step); ``fused``: a ping-pong
    loop whose tile kernel stores its boundary output straight into the
    neighbours' halos (decomp.PeerFusedStep: 1 launch per step); ``none``: the
    tile alone, as at N=1.  The timed steps are replayed from one CUDA graph (the
    NCCL calls are captured too).  Returns (max-over-ranks ms per step,
    global domain, grid, launches per step)."""
    import paper_2311_08322_b200 as b200
    from paper_2311_08322_b200 import decomp, native, workloads

    grid = decomp.choose_grid(dist.world) if transport != "none" else (1, 1)
    gdom = (tile[0] * grid[0], tile[1] * grid[1], tile[2])
    d = decomp.Decomposition(gdom, grid, dist.rank if transport != "none" else 0)
    ldom = d.local_domain
    rng = np.random.default_rng(1000 + dist.rank)
    vals = rng.uniform(-1, 1, (ldom[0] + 4, ldom[1] + 4, ldom[2]))
    if transport == "fused":
        # hdiff as a ping-pong time loop (out is the next step's inp) with the
        # halo exchange fused into the tile kernel: its output stores also go
        # into the neighbours' halos (peer memory), one launch per step
        st = b200.compile_stencil(workloads.source("hdiff"), "hdiff", gen_options={"mirror": "out"})
        A, B = b200.from_array(vals, (2, 2, 0)), b200.from_array(vals, (2, 2, 0))
        step = decomp.PeerFusedStep(st, d, [{"inp": A, "out": B}, {"inp": B, "out": A}], {"coeff": 0.05},
                                    "out", (2, 2))
        for _ in range(2 * max(1, warmup // 2)):
            step()
        native.synchronize(step.stream)
        module = st.build_info["module"]
        steps += steps % 2
        n0 = module.launch_count()
        replay = step.graph(steps)
        lps = (module.launch_count() - n0) / steps
        return _time_replay(dist, replay, step.stream, steps, step), gdom, grid, lps
    st = b200.compile_stencil(workloads.source("hdiff"), "hdiff")
    inp = b200.from_array(vals, (2, 2, 0))
    out = b200.allocate("f64", ldom)
    if transport == "peer":
        step = decomp.PeerDecomposedStep(st, d, {"inp": inp, "out": out}, {"coeff": 0.05}, "inp", (2, 2))
    else:
        step = decomp.DecomposedStep(st, d, {"inp": inp, "out": out}, {"coeff": 0.05}, "inp", (2, 2),
                                     split=split)
    stream = step.stream if hasattr(step, "stream") else step.compute
    for _ in range(warmup):
        step()
    native.synchronize(stream)
    module = st.build_info["module"]
    n0 = module.launch_count()
    replay = step.graph(steps)
    lps = (module.launch_count() - n0) / steps
    return _time_replay(dist, replay, stream, steps, step), gdom, grid, lps


def _time_replay(dist, replay, stream, steps, step) -> float:
    """One warm replay, then one timed replay of ``steps`` steps (CUDA
    events on the step's stream, max over ranks): ms per step."""
    from paper_2311_08322_b200 import native

    replay.launch()  # upload + warm replay
    native.synchronize(stream)
    e0, e1 = native.Event(), native.Event()
    dist.barrier()
    native.synchronize(stream)
    e0.record(stream)
    replay.launch()
    e1.record(stream)
    native.synchronize(stream)
    dist.barrier()
    ms = dist.max(e0.elapsed_ms(e1) / steps)
    if hasattr(step, "close"):
        step.close()
    return ms


def c4_weak_scaling(dist, args, tile=(512, 1024, 80), out=None):
    """BASELINE configs[3] / north_star scaling target: hdiff f64 with a fixed
    512x1024x80 tile per GPU on the rank grid (1x1, 2x1, 2x2, 4x2 -> 2048x
    2048x80 at 8 GPUs).  Measured in this run: the tile alone (no neighbours,
    ``tile_us``, every rank), then the decomposed step over the NCCL transport
    and (N > 1) the peer-memory transport; efficiency = tile time / step time
    (weak scaling, max over ranks)."""
    nst = max(args.steps // 4, 20)
    # filled in place: a caller that already holds ``out`` (the JSON line at
    # N > 1) keeps every number measured before a later transport hangs
    out = {} if out is None else out
    out.update({"tile": list(tile), "gpus": dist.world})
    ms1, _, _, lps1 = decomposed_hdiff(dist, nst, args.warmup, tile=tile, transport="none")
    out["tile_us"] = ms1 * 1e3
    out["tile_launches_per_step"] = lps1
    # the same tile as interior + frame launches without an exchange: what
    # the overlap split itself costs on one GPU
    ms_s, _, _, lps_s = decomposed_hdiff(dist, nst, args.warmup, tile=tile, transport="none", split=True)
    out["split_us"] = ms_s * 1e3
    out["split_launches_per_step"] = lps_s
    # the same with the band only on the sides a middle rank of the 4x2 grid
    # has neighbours on (decomp.neighbour_sides: both i sides, one j side)
    ms_s2, _, _, _ = decomposed_hdiff(dist, nst, args.warmup, tile=tile, transport="none",
                                      split=(True, True, True, False))
    out["split_4x2_us"] = ms_s2 * 1e3
    # (ranks sharing one GPU -- GTS_BENCH_SHARED_GPU -- exercise the peer
    # transports only: NCCL cannot put two ranks on one device)
    transports = (("peer", "fused") if dist.shared else ("nccl", "peer", "fused")) if dist.world > 1 else ()
    if dist.world == 1:  # the fused step's kernel (mirror build, no neighbours) as one launch
        ms_f, _, _, lps_f = decomposed_hdiff(dist, nst, args.warmup, tile=tile, transport="fused")
        out["fused_us"] = ms_f * 1e3
        # all 8 ranks of the 4x2 grid (north_star's 8-GPU layout) as virtual
        # ranks on this GPU (concurrent kernels)
        try:
            loc = c4_local_group((4, 2), tile, steps=20)
            # against the same fused kernel with no neighbours (the protocol's cost)
            loc["work_ratio"] = loc["ranks"] * out["fused_us"] / loc["us_per_step"]
            out["local_4x2"] = loc
        except Exception as exc:  # reported, not fatal
            out["local_4x2"] = {"error": f"{type(exc).__name__}: {exc}"[:200]}
    for tr in transports:
        try:
            ms, gdom, grid, lps = decomposed_hdiff(dist, nst, args.warmup, tile=tile, transport=tr)
            out["grid"], out["global"] = list(grid), list(gdom)
            out[tr] = {"us_per_step": ms * 1e3, "efficiency": ms1 / ms, "launches_per_step": lps,
                       "value": gdom[0] * gdom[1] * gdom[2] / (ms / 1e3)}
        except Exception as exc:  # reported, not fatal
            out[tr] = {"error": f"{type(exc).__name__}: {exc}"[:200]}
    return out


def c4_local_group(grid=(2, 2), tile=(512, 1024, 80), steps=20, kernel="hdiff") -> dict:
    """The fused C4 step (hdiff ping-pong, halo exchange fused into the tile
    kernel) with every rank of a ``grid`` decomposition as a virtual rank of
    this process on one GPU, each on its own stream
    (decomp.PeerFusedStep.local_group): all ranks' ``steps``-step graphs
    launched together, timed from one event before to the join after.  The
    ranks share the GPU, so ``work_ratio`` = ranks x the tile alone / the
    step time measures what the protocol (flags, mirror stores into each
    other's halos) costs with the kernels really concurrent -- not scaling."""
    import paper_2311_08322_b200 as b200
    from paper_2311_08322_b200 import decomp, native, workloads

    nr = grid[0] * grid[1]
    gdom = (tile[0] * grid[0], tile[1] * grid[1], tile[2])
    fin, fout = ("inp", "out") if kernel == "hdiff" else ("u_in", "u_out")
    sc = {"coeff": 0.05} if kernel == "hdiff" else workloads.DYCORE_SCALARS
    st = b200.compile_stencil(workloads.source(kernel), kernel, gen_options={"mirror": fout})
    ds = [decomp.Decomposition(gdom, grid, r) for r in range(nr)]
    phases = []
    for r, d in enumerate(ds):
        if kernel == "hdiff":
            vals, coef = np.random.default_rng(3000 + r).uniform(-1, 1, (tile[0] + 4, tile[1] + 4, tile[2])), {}
        else:
            arr = workloads.dycore_arrays(d.local_domain, 3000 + r)
            vals, coef = arr["u"], {n: b200.from_array(arr[n]) for n in "abc"}
        A, B = b200.from_array(vals, (2, 2, 0)), b200.from_array(vals, (2, 2, 0))
        phases.append([{fin: A, fout: B, **coef}, {fin: B, fout: A, **coef}])
    streams = [native.aux_stream(f"vrank{r}") for r in range(nr)]
    group = decomp.PeerFusedStep.local_group(st, ds, phases, sc, fout, (2, 2), streams)
    for _ in range(4):
        for s_ in group:
            s_()
    graphs = [s_.graph(steps) for s_ in group]
    master = native.default_stream()

    def replay() -> float:
        e0, e1 = native.Event(), native.Event()
        for s_ in group:
            native.synchronize(s_.stream)
        e0.record(master)
        for s_ in group:
            native.call("gts_b200_stream_wait_event", s_.stream, e0.ptr)
        for g in graphs:
            g.launch()
        ends = []
        for s_ in group:
            ev = native.Event()
            ev.record(s_.stream)
            native.call("gts_b200_stream_wait_event", master, ev.ptr)
            ends.append(ev)
        e1.record(master)
        native.synchronize(master)
        return e0.elapsed_ms(e1) / steps

    replay()
    ms = min(replay() for _ in range(3))
    return {"grid": list(grid), "ranks": nr, "us_per_step": ms * 1e3}


def dycore_decomposed_peer(dist, steps=20, tile=(512, 512, 80)):
    """The dycore step (configs[4]) weak-scaled: a 512x512x80 tile per GPU on
    the rank grid, the halo of u_in exchanged by peer stores each step
    (PeerDecomposedStep, one per u_in / u_out swap), ``steps`` steps replayed
    from one CUDA graph; max over ranks."""
    import paper_2311_08322_b200 as b200
    from paper_2311_08322_b200 import decomp, native, workloads

    grid = decomp.choose_grid(dist.world)
    gdom = (tile[0] * grid[0], tile[1] * grid[1], tile[2])
    d = decomp.Decomposition(gdom, grid, dist.rank)
    arr = workloads.dycore_arrays(d.local_domain, 2000 + dist.rank)  # per-rank synthetic state
    st = b200.compile_stencil(workloads.source("dycore"), "dycore")
    A, B = b200.from_array(arr["u"], (2, 2, 0)), b200.from_array(arr["u"], (2, 2, 0))
    coef = {n: b200.from_array(arr[n]) for n in "abc"}
    sc = workloads.DYCORE_SCALARS
    s_ab = decomp.PeerDecomposedStep(st, d, {"u_in": A, "u_out": B, **coef}, sc, "u_in", (2, 2))
    s_ba = decomp.PeerDecomposedStep(st, d, {"u_in": B, "u_out": A, **coef}, sc, "u_in", (2, 2))
    for s in range(4):
        (s_ab if s % 2 == 0 else s_ba)()
    stream = s_ab.compute
    native.synchronize(stream)
    g = native.Graph(stream)
    with g.capture():
        for s in range(steps):
            (s_ab if s % 2 == 0 else s_ba)()
    g.launch()
    native.synchronize(stream)
    e0, e1 = native.Event(), native.Event()
    dist.barrier()
    e0.record(stream)
    g.launch()
    e1.record(stream)
    native.synchronize(stream)
    dist.barrier()
    ms = dist.max(e0.elapsed_ms(e1) / steps)
    pts = gdom[0] * gdom[1] * gdom[2]
    return {"workload": f"dycore step, {tile[0]}x{tile[1]}x{tile[2]} per GPU on a {grid[0]}x{grid[1]} grid "
                        f"(global {gdom[0]}x{gdom[1]}x{gdom[2]}), u_in halo by peer stores, {steps} steps "
                        "replayed from one CUDA graph",
            "value": pts / (ms / 1e3), "unit": "grid-point-steps/s", "ms_per_step": ms, "scaling": "weak"}


def dycore_fused_peer(dist, steps=20, tile=(512, 512, 80)):
    """The dycore step with the halo exchange fused into the producing kernel
    (decomp.PeerFusedStep: the column kernel's epilogue also stores the
    boundary of u_out into the neighbours' halos over peer memory, one launch
    + a flag wait and signal per step), a 512x512x80 tile per GPU, ``steps``
    steps replayed from one CUDA graph; max over ranks.  At N=1 there are no
    neighbours: the same kernel with an empty mirror."""
    import paper_2311_08322_b200 as b200
    from paper_2311_08322_b200 import decomp, native, workloads

    grid = decomp.choose_grid(dist.world)
    gdom = (tile[0] * grid[0], tile[1] * grid[1], tile[2])
    d = decomp.Decomposition(gdom, grid, dist.rank)
    arr = workloads.dycore_arrays(d.local_domain, 2000 + dist.rank)
    st = b200.compile_stencil(workloads.source("dycore"), "dycore", gen_options={"mirror": "u_out"})
    A, B = b200.from_array(arr["u"], (2, 2, 0)), b200.from_array(arr["u"], (2, 2, 0))
    coef = {n: b200.from_array(arr[n]) for n in "abc"}
    step = decomp.PeerFusedStep(st, d, [{"u_in": A, "u_out": B, **coef}, {"u_in": B, "u_out": A, **coef}],
                                workloads.DYCORE_SCALARS, "u_out", (2, 2))
    for _ in range(4):
        step()
    native.synchronize(step.stream)
    g = step.graph(steps)
    g.launch()
    native.synchronize(step.stream)
    e0, e1 = native.Event(), native.Event()
    dist.barrier()
    e0.record(step.stream)
    g.launch()
    e1.record(step.stream)
    native.synchronize(step.stream)
    dist.barrier()
    ms = dist.max(e0.elapsed_ms(e1) / steps)
    step.close()
    pts = gdom[0] * gdom[1] * gdom[2]
    return {"workload": f"dycore step, {tile[0]}x{tile[1]}x{tile[2]} per GPU on a {grid[0]}x{grid[1]} grid "
                        f"(global {gdom[0]}x{gdom[1]}x{gdom[2]}), u_out boundary stored into the neighbours' "
                        f"halos by the column kernel itself, {steps} steps replayed from one CUDA graph",
            "value": pts / (ms / 1e3), "unit": "grid-point-steps/s", "ms_per_step": ms, "scaling": "weak",
            "launches_per_step": 3 if dist.world > 1 else 1}


def dycore_timed(dist, steps=100, domain=(512, 512, 80), reps=3, gen_options=None, check=True):
    """BASELINE.json configs[4]: the dycore-like step (kernels/dycore.gts:
    hdiff -> Thomas solve -> interval-specialised update) on 512x512x80 f64,
    ``steps`` time steps per run captured in one CUDA graph (TimeLoop).  The
    first replay (the first ``steps`` steps from the initial state, untimed)
    is checked bitwise against the reference gen engine's own dycore kernel
    (oracle/_ref, ``steps`` host-swapped calls); then ``reps`` timed replays
    (CUDA events, max over ranks).  Fields + temporaries exceed the L2 16x."""
    import paper_2311_08322_b200 as b200
    from paper_2311_08322_b200 import native, workloads
    from paper_2311_08322_b200.timeloop import TimeLoop

    st = b200.compile_stencil(workloads.source("dycore"), "dycore", gen_options=gen_options)
    arr = workloads.dycore_arrays(domain, 1000 + dist.rank)
    A, B = b200.from_array(arr["u"], (2, 2, 0)), b200.from_array(arr["u"], (2, 2, 0))
    coef = {n: b200.from_array(arr[n]) for n in "abc"}
    loop = TimeLoop(st, [dict(u_in=A, u_out=B, **coef), dict(u_in=B, u_out=A, **coef)], steps,
                    workloads.DYCORE_SCALARS)
    stream = loop.stream
    loop.run()  # capture + the first `steps` steps
    parity = None
    if check:
        sys.path.insert(0, str(REPO / "oracle"))
        import oracle

        got = (A, B)[steps % 2].host_array()
        if oracle.ref_available("dycore_f64"):
            want = oracle.ref_dycore_run(arr["u"], arr["a"], arr["b"], arr["c"], steps)
            parity = (f"bitwise(ref,{steps} steps)" if np.array_equal(got, want)
                      else f"ref max_rel {oracle.max_rel(got, want):.2e}")
        else:
            parity = "finite" if np.isfinite(got).all() else "NON-FINITE"
    e0, e1 = native.Event(), native.Event()
    dist.barrier()
    native.synchronize(stream)
    e0.record(stream)
    for _ in range(reps):
        loop.run(sync=False)
    e1.record(stream)
    native.synchronize(stream)
    dist.barrier()
    ms = dist.max(e0.elapsed_ms(e1) / reps)
    pts = domain[0] * domain[1] * domain[2]
    alg = workloads.algorithmic_bytes("dycore", domain)
    return {
        "value": dist.world * pts * steps / (ms / 1e3), "unit": "grid-point-steps/s",
        "us_per_step": 1e3 * ms / steps, "achieved_gbs": alg / (ms / steps / 1e3) / 1e9,
        "launches_per_step": loop.launches_per_step, "parity": parity,
    }


# binary32 <-> binary64 conversions (F2F) per SM per clock on this B200: the
# XU pipe, measured with tools/ubench.cu ("Instruction costs")
XU_CONV_PER_CLK_SM = 16


def conversion_roofline(st, domain, seconds, sampler):
    """The binding roofline of a binary32 tile kernel (the reference computes
    f32 programs in binary64, narrowing every store): conversions per point
    = the F2F count of the fully unrolled thread-tile body of the fused tile
    kernel (cuobjdump of the loaded module) / the points of one thread-tile,
    against XU_CONV_PER_CLK_SM x SMs x the SM clock under load.  None when
    cuobjdump or the kernel is not found."""
    import re
    import shutil

    from paper_2311_08322_b200 import codegen_parallel, native

    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    so = st.build_info.get("so_path")
    if not so or not Path(exe).exists():
        return None
    try:
        sass = subprocess.run([exe, "-sass", so], capture_output=True, text=True, timeout=120).stdout
    except (OSError, subprocess.SubprocessError):
        return None
    body = None
    for chunk in re.split(r"\n\s+Function : ", sass)[1:]:
        if chunk.split("\n", 1)[0].strip().startswith("_Z13gts_k0_pfused"):
            body = chunk
    if body is None:
        return None
    geo = codegen_parallel.GEOMETRY[4]
    conv = len(re.findall(r"\bF2F\.", body)) / (geo["pf_ri"] * geo["pf_vj"])
    mhz = sampler.summary().get("sm_mhz") or sampler.summary().get("sm_max_mhz")
    info = native.device_info()
    peak = XU_CONV_PER_CLK_SM * info["sm_count"] * mhz * 1e6
    achieved = conv * domain[0] * domain[1] * domain[2] / seconds
    return {"bound": "xu (f32<->f64 conversions)", "conv_per_point": round(conv, 3),
            "achieved": achieved / 1e12, "peak": peak / 1e12, "unit": "Tconv/s", "frac": achieved / peak}


def compact_line(line: dict) -> dict:
    """The JSON line as printed: the N > 1 ``c4`` block without the fields
    the rest derive (launch counts, global domain, per-transport value)."""
    out = dict(line)
    c4 = out.get("c4")
    if isinstance(c4, dict):
        c = {k: v for k, v in c4.items()
             if k not in ("tile_launches_per_step", "split_launches_per_step", "global", "split_us")}
        for tr in ("nccl", "peer", "fused"):
            if isinstance(c.get(tr), dict):
                c[tr] = {k: v for k, v in c[tr].items() if k != "value"}
        out["c4"] = c
    return out


def compact_extra(extra: dict) -> dict:
    """The extras as they go on the JSON line (the driver keeps a 1500-char
    stdout tail): times and fractions only, parity "bitwise" meaning equal
    to both the C restatement and the reference's own kernel (the full
    records are in gpurun_out/bench_detail_n<N>.json)."""
    drop = {"workload", "unit", "value", "scaling", "tile", "gpus", "tile_launches_per_step",
            "split_launches_per_step", "launches_per_step", "grid", "ranks", "split_us"}
    out = {}
    for k, v in extra.items():
        if k == "dycore_fused_peer" and "dycore_fused_local_2x2" in extra:
            continue  # N=1: the dycore kernel again (mirror build, no neighbours): detail file only
        if k == "dycore_fused_local_2x2":
            k = "dycore_local_2x2"
        if not isinstance(v, dict):
            out[k] = v
            continue
        c = {}
        for kk, vv in v.items():
            if kk in drop:
                continue
            if kk == "parity" and isinstance(vv, str):
                vv = vv.replace("bitwise(oracle+ref)", "bitwise").replace("bitwise(ref,", "bitwise(")
            if kk == "xu" and isinstance(vv, dict):
                c["xu_frac"] = vv.get("frac")
                continue
            if kk == "ms_per_step":
                kk, vv = "us_per_step", vv * 1e3
            if kk.startswith("local_") and isinstance(vv, dict):
                if "error" in vv:
                    c[kk] = vv
                else:
                    c[kk + "_us"], c[kk + "_ratio"] = vv.get("us_per_step"), vv.get("work_ratio")
                continue
            if k == "dycore_local_2x2" and kk == "work_ratio":
                kk = "ratio"
            c[kk] = vv
        out[k] = c
    return out


def _r(x, n=4):
    """Round for the compact JSON line."""
    if isinstance(x, float):
        return float(f"{x:.{n}g}")
    if isinstance(x, dict):
        return {k: _r(v, n) for k, v in x.items()}
    if isinstance(x, list):
        return [_r(v, n) for v in x]
    return x


def _extra_guard(fn, *a, **k):
    try:
        return fn(*a, **k)
    except Exception as exc:  # pragma: no cover - reported, not fatal
        return {"error": f"{type(exc).__name__}: {exc}"[:200]}


def _detail_path(dist) -> Path:
    d = REPO / "gpurun_out"
    d.mkdir(exist_ok=True)
    return d / f"bench_detail_n{dist.world}.json"


def run_b200(args, dist):
    import paper_2311_08322_b200 as b200
    from paper_2311_08322_b200 import native, workloads

    if dist.world > 1:
        native.set_device(dist.local % native.device_count() if dist.shared else dist.local)
    dev = native.require_device()
    kernel, dtype, domain = WORKLOADS[args.workload]
    st = b200.compile_stencil(workloads.source(kernel, dtype), kernel)
    pts = domain[0] * domain[1] * domain[2]
    sampler = ClockSampler(dev)
    r = device_timed(st, kernel, dtype, domain, args.steps, args.warmup, dist, sampler,
                     use_graph=not args.no_graph)
    total_ms = dist.max(r["total_ms"])
    launch_ms = dist.max(r["launch_ms_mean"])
    ms_per_step = total_ms / args.steps
    value = dist.world * pts / (ms_per_step / 1e3)
    parity = parity_check(kernel, dtype, r["sets"])
    del r["sets"]
    peak, peak_src = measured_peak()
    alg = workloads.algorithmic_bytes(kernel, domain, dtype)
    achieved = alg / (launch_ms / 1e3) / 1e9
    e2e_s, h2d, d2h, chunks = e2e_timed(st, kernel, dtype, domain, args.e2e_steps, pinned=True)
    e2e_val = dist.max(e2e_s)
    pg_s, pg_h2d, pg_d2h, _ = e2e_timed(st, kernel, dtype, domain, max(args.e2e_steps // 2, 5), pinned=False)
    pg_val = dist.max(pg_s)
    detail: dict = {"device_timed": r, "peak_source": peak_src}
    line = {
        "metric": "grid-points/s",
        "value": value, "unit": "grid-points/s", "n_gpus": dist.world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": dtype,
        "data": "synthetic",
        "config": {"workload": SHORT_TEXT[args.workload] + (" per GPU" if dist.world > 1 else ""),
                   "parallelism": (f"{dist.world} column shards" if dist.world > 1 else "1 GPU")
                   + (" (shared GPU)" if dist.shared and dist.world > 1 else ""),
                   "l2": f"{r['nsets']} input sets > 2x L2",
                   "launch": "cuda graph" if not args.no_graph else "eager"},
        "parity": parity,
        "gpu_launches": r["launches"],
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": _traffic_bytes(args.workload),
                     "alg_bytes": alg},
        "e2e": {"value": dist.world * pts / e2e_val, "unit": "grid-points/s",
                "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "ms": e2e_val * 1e3, "pageable": {"value": dist.world * pts / pg_val, "ms": pg_val * 1e3}},
        "clocks": sampler.summary(),
    }
    # Watchdog for the extras (multi-rank exchanges that have not run on this
    # pool's hardware): if they have not finished in time, rank 0 prints the
    # headline line with the extras marked and every rank exits cleanly, so a
    # hung collective cannot cost the headline measurement.
    done = threading.Event()

    def _watchdog():
        if not done.wait(args.extra_timeout):
            if dist.rank == 0:
                line["extra"] = {"error": f"extras timed out after {args.extra_timeout:.0f} s"}
                text = None
                for _ in range(5):  # the main thread may still be filling line["c4"]
                    try:
                        text = json.dumps(_r(compact_line(line)))
                        break
                    except RuntimeError:
                        time.sleep(0.05)
                if text is None:
                    text = json.dumps(_r({k: v for k, v in line.items() if k != "c4"}))
                print(text, flush=True)
            os._exit(0)

    threading.Thread(target=_watchdog, daemon=True).start()
    extra: dict = {}
    if not args.no_extra:
        c4: dict = {}
        if dist.world > 1:
            line["c4"] = c4  # the watchdog's line keeps what was measured before a hang
        c4_weak_scaling(dist, args, out=c4)
        detail["c4"] = c4
        if dist.world == 1:
            extra["c4_tile"] = c4
    if dist.rank == 0 and dist.world == 1 and not args.no_extra:
        nst = max(args.steps // 2, 50)
        for name in ("hdiff", "hdiff32"):
            k2, d2, dom2 = WORKLOADS[name]
            st2 = b200.compile_stencil(workloads.source(k2, d2), k2)
            r2 = device_timed(st2, k2, d2, dom2, nst, args.warmup, dist, use_graph=not args.no_graph)
            ach2 = workloads.algorithmic_bytes(k2, dom2, d2) / (r2["launch_ms_mean"] / 1e3) / 1e9
            extra[name] = {"us": r2["launch_ms_mean"] * 1e3, "frac": ach2 / peak,
                           "parity": parity_check(k2, d2, r2["sets"])}
            if d2 == "f32":
                xu = conversion_roofline(st2, dom2, r2["launch_ms_mean"] / 1e3, sampler)
                if xu:
                    extra[name]["xu"] = xu
        # BASELINE configs[0]: hdiff 128x128x64 f64 with the reference gen
        # kernel timed on the same inputs
        dom1 = (128, 128, 64)
        st1 = b200.compile_stencil(workloads.source("hdiff", "f64"), "hdiff")
        r1 = device_timed(st1, "hdiff", "f64", dom1, nst, args.warmup, dist, use_graph=not args.no_graph)
        c1 = {"us": r1["launch_ms_mean"] * 1e3, "parity": parity_check("hdiff", "f64", r1["sets"])}
        if not args.no_cpu_baseline:
            t1 = time_reference("hdiff", "f64", dom1, seconds=3.0, max_calls=2000)
            if t1:
                c1["cpu_ref_us"] = statistics.median(t1) * 1e6
        extra["c1"] = c1
        dy = _extra_guard(dycore_timed, dist)
        if "achieved_gbs" in dy:
            dy["frac"] = dy.pop("achieved_gbs") / peak
        extra["dycore"] = dy
        extra["dycore_fused_peer"] = _extra_guard(dycore_fused_peer, dist)
        # the fused dycore step on all 4 ranks of a 2x2 grid as virtual ranks (concurrent kernels)
        dl = _extra_guard(c4_local_group, (2, 2), (512, 512, 80), 20, "dycore")
        if "us_per_step" in dl and "us_per_step" in dy:
            dl["work_ratio"] = dl["ranks"] * dy["us_per_step"] / dl["us_per_step"]
        extra["dycore_fused_local_2x2"] = dl
    if dist.world > 1 and not args.no_extra:
        extra["dycore_decomposed_peer"] = _extra_guard(dycore_decomposed_peer, dist)
        extra["dycore_fused_peer"] = _extra_guard(dycore_fused_peer, dist)
    if extra and dist.rank == 0:
        detail["extra"] = extra
        line["extra"] = compact_extra(extra)
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu_baseline:
        cores, model = host_info()
        times = time_reference(kernel, dtype, domain, seconds=args.cpu_seconds, max_calls=100000)
        if times:
            v = pts / statistics.median(times)
            rows = cpu_rows(kernel, dtype, domain, cores)
            detail["cpu_rows"] = rows
            line["cpu_baseline"] = {
                "value": v, "unit": "grid-points/s", "cores": cores, "kind": "reference",
                "sample": f"median of {len(times)} calls of oracle/_ref",
                "rows": {k: _r(vv.get("value")) if isinstance(vv, dict) else vv for k, vv in rows.items()
                         if k == "gen_arena_reuse"},
            }
    done.set()
    if dist.rank == 0:
        detail["line"] = line
        try:
            _detail_path(dist).write_text(json.dumps(detail, indent=1, default=str))
        except OSError:
            pass
        print(json.dumps(_r(compact_line(line))), flush=True)


def main():
    args = parse()
    dist = Dist()
    try:
        if args.impl == "reference":
            run_reference(args, dist)
        else:
            run_b200(args, dist)
    finally:
        dist.close()


if __name__ == "__main__":
    main()
