#!/usr/bin/env python
"""Where the fused dycore step's time goes: the same step with its hdiff
prologue replaced by a trivial one that still streams u_in as a halo'd box.

    python tools/dycore_floor.py [full,cheap] ['{"pro_warps": 4}']

``cheap`` keeps the plan (pfused prologue + TMEM column kernel with prologue
and epilogue fusion) and the bytes moved, but the prologue is ``t = u_in;
uh = t[1, 0, 0]``: the difference to ``full`` is the cost of evaluating the
flux-limited diffusion inside the column kernel.  100 steps per CUDA-graph
replay (TimeLoop), 512x512x80 f64, mean of 3 replays.
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2311_08322_b200 as b200  # noqa: E402
from paper_2311_08322_b200 import native, workloads  # noqa: E402
from paper_2311_08322_b200.timeloop import TimeLoop  # noqa: E402

BASE = workloads.source("dycore")
HEAD = BASE[:BASE.index("    with computation(PARALLEL):")]
TAIL = BASE[BASE.index("    with computation(FORWARD):"):]
VARIANTS = {
    "full": BASE,
    "cheap": HEAD + "    with computation(PARALLEL):\n        with interval(0, None):\n"
    "            t = u_in\n            uh = t[1, 0, 0]\n" + TAIL,
}


def timed(src, opts, domain=(512, 512, 80), steps=100, reps=3):
    st = b200.compile_stencil(src, "dycore", gen_options=opts or None)
    arr = workloads.dycore_arrays(domain, 1000)
    A, B = b200.from_array(arr["u"], (2, 2, 0)), b200.from_array(arr["u"], (2, 2, 0))
    coef = {n: b200.from_array(arr[n]) for n in "abc"}
    loop = TimeLoop(st, [dict(u_in=A, u_out=B, **coef), dict(u_in=B, u_out=A, **coef)], steps,
                    workloads.DYCORE_SCALARS)
    loop.run()
    e0, e1 = native.Event(), native.Event()
    native.synchronize(loop.stream)
    e0.record(loop.stream)
    for _ in range(reps):
        loop.run(sync=False)
    e1.record(loop.stream)
    native.synchronize(loop.stream)
    return 1e3 * e0.elapsed_ms(e1) / reps / steps, st.build_info.get("plan")


if __name__ == "__main__":
    names = sys.argv[1].split(",") if len(sys.argv) > 1 else list(VARIANTS)
    opts = json.loads(sys.argv[2]) if len(sys.argv) > 2 else {}
    for n in names:
        us, plan = timed(VARIANTS[n], opts)
        print(f"{n:6s} {json.dumps(opts)}: {us:.1f} us/step  plan={plan}", flush=True)
