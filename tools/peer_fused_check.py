#!/usr/bin/env python
"""A decomposed time loop with the halo exchange fused into the producing
kernel (decomp.PeerFusedStep: the kernel stores its boundary output straight
into the neighbours' halos, corners included), checked bitwise against the
undecomposed oracle, eagerly and replayed from a CUDA graph:

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port P tools/peer_fused_check.py [steps] [--kernel dycore|hdiff]

dycore: kernels/dycore.gts, mirrored by the TMEM column kernel; hdiff: the
reference's hdiff.gts as a ping-pong loop (out becomes the next step's inp,
Dirichlet halo), mirrored by the fused PARALLEL tile kernel (BASELINE
configs[3]'s step with the exchange fused into the producer).

Ranks use GPU LOCAL_RANK % device count (one GPU: they share it through CUDA
IPC); --timing adds per-step device time (max over ranks).
"""
import os
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REPO / "oracle"))

import numpy as np  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 and not sys.argv[1].startswith("--") else 4
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()

    import oracle
    import paper_2311_08322_b200 as b200
    from paper_2311_08322_b200 import decomp, native, workloads

    native.set_device(int(os.environ.get("LOCAL_RANK", "0")) % native.device_count())
    grid = decomp.choose_grid(world)
    kernel = sys.argv[sys.argv.index("--kernel") + 1] if "--kernel" in sys.argv else "dycore"
    if kernel == "hdiff":
        gdom = (37 * grid[0] + 3, 140 * grid[1] + 5, 6)  # several 128-column tiles per rank
        arr = {"u": np.random.default_rng(11).uniform(-1, 1, (gdom[0] + 4, gdom[1] + 4, gdom[2]))}
        sc = {"coeff": 0.05}
        coef = {}
        fin, fout = "inp", "out"
        run = lambda n: oracle.hdiff_run(arr["u"], n, 0.05)  # noqa: E731
    else:
        gdom = (37 * grid[0] + 3, 70 * grid[1] + 5, 16)
        arr = workloads.dycore_arrays(gdom, 11)
        sc = workloads.DYCORE_SCALARS
        fin, fout = "u_in", "u_out"
        run = lambda n: oracle.dycore_run(arr["u"], arr["a"], arr["b"], arr["c"], n, **sc)  # noqa: E731
    d = decomp.Decomposition(gdom, grid, rank)
    ni, nj, nk = d.local_domain
    u = d.scatter(arr["u"], (2, 2))
    if kernel != "hdiff":
        coef = {n: b200.from_array(np.array(arr[n][d.i0: d.i1, d.j0: d.j1, :], copy=True)) for n in "abc"}
    gopts = {"mirror": fout}
    if "--inline" in sys.argv:  # the column template's per-level mirror stores (gen_options mirror_inline)
        gopts["mirror_inline"] = True
    st = b200.compile_stencil(workloads.source(kernel), kernel, gen_options=gopts)
    A, B = b200.from_array(u, (2, 2, 0)), b200.from_array(u, (2, 2, 0))
    step = decomp.PeerFusedStep(st, d, [{fin: A, fout: B, **coef}, {fin: B, fout: A, **coef}],
                                sc, fout, (2, 2))
    if os.environ.get("FUSED_NO_MIRROR"):  # negative control: no halo stores -> must fail
        step._boxes = [[] for _ in step._boxes]
    for s in range(steps):
        step()
    native.synchronize(step.stream)
    last = B if steps % 2 == 1 else A
    got = last.host_array()[2:-2, 2:-2, :]
    want = run(steps)[2:-2, 2:-2, :]
    ok_e = bool(np.array_equal(got, want[d.i0: d.i1, d.j0: d.j1, :]))
    # graph replay: 2 more steps per replay, 2 replays, against the oracle at steps + 4
    ok_g = True
    if steps % 2 == 0:
        g = step.graph(2)
        dist.barrier()
        g.launch()
        g.launch()
        native.synchronize(step.stream)
        got = A.host_array()[2:-2, 2:-2, :]
        want = run(steps + 4)[2:-2, 2:-2, :]
        ok_g = bool(np.array_equal(got, want[d.i0: d.i1, d.j0: d.j1, :]))
    ok = ok_e and ok_g
    extra = ""
    if "--timing" in sys.argv:
        g = step.graph(20)
        g.launch()
        native.synchronize(step.stream)
        e0, e1 = native.Event(), native.Event()
        dist.barrier()
        e0.record(step.stream)
        g.launch()
        e1.record(step.stream)
        native.synchronize(step.stream)
        extra = f" graph_ms_per_step {e0.elapsed_ms(e1) / 20:.4f}"
    step.close()
    print(("FUSED_PEER_OK " if ok else "FUSED_PEER_FAIL ")
          + f"{kernel} rank {rank} grid {grid} local {d.local_domain} steps {steps} bitwise eager {ok_e} graph {ok_g}{extra}",
          flush=True)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
