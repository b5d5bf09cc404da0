#!/usr/bin/env python
"""The dycore step (kernels/dycore.gts) decomposed with the halo exchange
fused into the producing kernel (decomp.PeerFusedStep: the column kernel
stores its boundary output straight into the neighbours' halos, corners
included), checked bitwise against the undecomposed oracle, eagerly and
replayed from a CUDA graph:

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port P tools/peer_fused_check.py [steps]

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
    gdom = (37 * grid[0] + 3, 70 * grid[1] + 5, 16)
    arr = workloads.dycore_arrays(gdom, 11)
    d = decomp.Decomposition(gdom, grid, rank)
    ni, nj, nk = d.local_domain
    u = d.scatter(arr["u"], (2, 2))
    coef = {n: b200.from_array(np.array(arr[n][d.i0: d.i1, d.j0: d.j1, :], copy=True)) for n in "abc"}
    st = b200.compile_stencil(workloads.source("dycore"), "dycore", gen_options={"mirror": "u_out"})
    A, B = b200.from_array(u, (2, 2, 0)), b200.from_array(u, (2, 2, 0))
    sc = workloads.DYCORE_SCALARS
    step = decomp.PeerFusedStep(st, d, [{"u_in": A, "u_out": B, **coef}, {"u_in": B, "u_out": A, **coef}],
                                sc, "u_out", (2, 2))
    if os.environ.get("FUSED_NO_MIRROR"):  # negative control: no halo stores -> must fail
        step._boxes = [[] for _ in step._boxes]
    for s in range(steps):
        step()
    native.synchronize(step.stream)
    last = B if steps % 2 == 1 else A
    got = last.host_array()[2:-2, 2:-2, :]
    want = oracle.dycore_run(arr["u"], arr["a"], arr["b"], arr["c"], steps, **sc)[2:-2, 2:-2, :]
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
        want = oracle.dycore_run(arr["u"], arr["a"], arr["b"], arr["c"], steps + 4, **sc)[2:-2, 2:-2, :]
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
          + f"rank {rank} grid {grid} local {d.local_domain} steps {steps} bitwise eager {ok_e} graph {ok_g}{extra}",
          flush=True)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
