"""Cost of the fused halo stores of decomp.PeerFusedStep on one GPU: the
dycore step (512x512x80 per GPU; ``--kernel hdiff``: the hdiff ping-pong step
on the 512x1024x80 C4 tile) with an empty mirror, and with the 8 mirror boxes
an interior rank of a 3x3 grid has (2-deep faces and corners), here pointed at
a scratch field on the same GPU instead of the neighbours' halos (so the
extra stores write local HBM instead of NVLink).  CUDA-graph timed, 20 steps
per replay, median of 5 replays."""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2311_08322_b200 as b200  # noqa: E402
from paper_2311_08322_b200 import decomp, native, workloads  # noqa: E402

KERNEL = sys.argv[sys.argv.index("--kernel") + 1] if "--kernel" in sys.argv else "dycore"
dom = (512, 1024, 80) if KERNEL == "hdiff" else (512, 512, 80)
d = decomp.Decomposition(dom, (1, 1), 0)
if KERNEL == "hdiff":
    import numpy as np

    u = np.random.default_rng(7).uniform(-1, 1, (dom[0] + 4, dom[1] + 4, dom[2]))
    opts = {"mirror": "out"}
    st = b200.compile_stencil(workloads.source("hdiff"), "hdiff", gen_options=opts)
    A, B, S = (b200.from_array(u, (2, 2, 0)) for _ in range(3))
    step = decomp.PeerFusedStep(st, d, [{"inp": A, "out": B}, {"inp": B, "out": A}], {"coeff": 0.05},
                                "out", (2, 2))
else:
    arr = workloads.dycore_arrays(dom, 7)
    opts = {"mirror": "u_out"}
    if "--inline" in sys.argv:
        opts["mirror_inline"] = True
    if len(sys.argv) > 1 and sys.argv[1].isdigit():
        opts["mirror_batch"] = int(sys.argv[1])
    st = b200.compile_stencil(workloads.source("dycore"), "dycore", gen_options=opts)
    A, B = b200.from_array(arr["u"], (2, 2, 0)), b200.from_array(arr["u"], (2, 2, 0))
    S = b200.from_array(arr["u"], (2, 2, 0))  # scratch "neighbour halo"
    coef = {n: b200.from_array(arr[n]) for n in "abc"}
    step = decomp.PeerFusedStep(st, d, [{"u_in": A, "u_out": B, **coef}, {"u_in": B, "u_out": A, **coef}],
                                workloads.DYCORE_SCALARS, "u_out", (2, 2))
ni, nj, _ = dom
fake = []
for di in (-1, 0, 1):
    for dj in (-1, 0, 1):
        if di == dj == 0:
            continue
        i0, i1 = {-1: (0, 2), 0: (0, ni), 1: (ni - 2, ni)}[di]
        j0, j1 = {-1: (0, 2), 0: (0, nj), 1: (nj - 2, nj)}[dj]
        org = sum(o * s for o, s in zip(S.origin, S.strides)) * S.itemsize
        fake.append((i0, i1, j0, j1, S.base_address() + org, *S.strides))


def timed(boxes):
    step._boxes = [boxes, boxes]
    g = step.graph(20)
    g.launch()
    native.synchronize(step.stream)
    out = []
    for _ in range(5):
        e0, e1 = native.Event(), native.Event()
        e0.record(step.stream)
        g.launch()
        e1.record(step.stream)
        native.synchronize(step.stream)
        out.append(e0.elapsed_ms(e1) / 20 * 1e3)
    return statistics.median(out)


if "--sk0" in sys.argv:  # diagnostic: every level to one target plane (1 page per column instead of 80)
    fake = [b[:7] + (0,) for b in fake]
if "--eager" in sys.argv:  # profiler runs: a few plain steps with the 8 boxes, no graph
    step._boxes = [fake, fake]
    for _ in range(4):
        step()
    native.synchronize(step.stream)
    sys.exit(0)
sel = {"i-faces only": [fake[1], fake[6]], "j-faces only": [fake[3], fake[4]],
       "corners only": [fake[0], fake[2], fake[5], fake[7]]}
runs = [("no neighbours", []), ("8 neighbours (3x3 interior rank)", fake), ("no neighbours", [])]
if "--split" in sys.argv:
    runs += list(sel.items())
for label, boxes in runs:
    print(f"{KERNEL} {dom[0]}x{dom[1]}x{dom[2]} fused-halo step {opts}, {label}: {timed(boxes):.2f} us/step",
          flush=True)
