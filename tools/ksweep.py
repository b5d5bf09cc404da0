#!/usr/bin/env python
"""Experiment sweep: time one stencil over several domains x gen_options.

    python tools/ksweep.py vadv f64 '256x256x80,296x256x80' '{}' '{"deep_ring": true}'

Each (domain, options) pair is compiled once and timed like bench.py: rotating
input sets totalling > 3x L2, K launches captured in one CUDA graph, kernel
time = timed region / K.  Prints one line per pair (us, GB/s algorithmic).
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import paper_2311_08322_b200 as b200  # noqa: E402
from paper_2311_08322_b200 import native, workloads  # noqa: E402


def time_dycore(dom, opts):
    import bench

    r = bench.dycore_timed(bench.Dist(), domain=dom, gen_options=opts or None, check=False)
    return r["us_per_step"], r["achieved_gbs"], None


def time_one(kernel, dtype, dom, opts, steps=200, eager=0):
    if kernel == "dycore":
        return time_dycore(dom, opts)
    st = b200.compile_stencil(workloads.source(kernel, dtype), kernel, gen_options=opts or None)
    info = native.device_info()
    set_bytes = workloads.algorithmic_bytes(kernel, dom, dtype)
    nsets = min(16, max(3, -(-(3 * info["l2_bytes"]) // set_bytes)))
    stream = native.default_stream()
    mod = st.build_info["module"]
    gos = []
    for s in range(nsets):
        a = workloads.make_args(kernel, dom, dtype, seed=s)
        gos.append((a, mod.launcher(dom, {k: v for k, v in a.items() if hasattr(v, "base_address")},
                                    {k: v for k, v in a.items() if not hasattr(v, "base_address")}, stream)))
    for i in range(2 * nsets):
        gos[i % nsets][1]()
    native.synchronize(stream)
    if eager:  # profiler runs: plain launches, no graph
        for i in range(eager):
            gos[i % nsets][1]()
        native.synchronize(stream)
        return 0.0, 0.0, st.build_info.get("plan")
    g = native.Graph(stream)
    with g.capture():
        for i in range(steps):
            gos[i % nsets][1]()
    g.launch()
    native.synchronize(stream)
    best = None
    for _ in range(3):
        e0, e1 = native.Event(), native.Event()
        e0.record(stream)
        g.launch()
        e1.record(stream)
        native.synchronize(stream)
        us = e0.elapsed_ms(e1) / steps * 1e3
        best = us if best is None else min(best, us)
    return best, set_bytes / best / 1e3, st.build_info.get("plan")


def main():
    kernel, dtype, doms = sys.argv[1], sys.argv[2], sys.argv[3]
    build_only = "--build" in sys.argv
    eager = next((int(a.split("=")[1]) for a in sys.argv if a.startswith("--eager=")), 0)
    optsl = [json.loads(o) for o in sys.argv[4:] if not o.startswith("--")] or [{}]
    if build_only:
        for o in optsl:
            b200.compile_stencil(workloads.source(kernel, dtype), kernel, gen_options=o or None)
        return
    for d in doms.split(","):
        dom = tuple(int(x) for x in d.split("x"))
        for o in optsl:
            try:
                us, gbs, plan = time_one(kernel, dtype, dom, o, eager=eager)
                print(f"{kernel} {dtype} {d} {json.dumps(o)}: {us:.2f} us  {gbs:.0f} GB/s", flush=True)
            except Exception as e:  # keep sweeping
                print(f"{kernel} {dtype} {d} {json.dumps(o)}: FAILED {type(e).__name__}: {e}", flush=True)


if __name__ == "__main__":
    main()
