#!/usr/bin/env python
"""The dycore step (kernels/dycore.gts) on a decomposed domain over the
peer-memory halo exchange (decomp.PeerDecomposedStep), checked bitwise against
the undecomposed oracle after several steps:

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port P tools/peer_dycore_check.py [steps]

Each rank holds its box of u (two storages, swapped between steps like the
host swap of dycore.gts), a, b, c; one PeerDecomposedStep per swap direction
exchanges the 2-cell halo of that step's u_in with the neighbours, overlapped
with the interior, then runs the fused dycore column kernel on the interior
and the four boundary strips.  Every point runs the same instructions as in
the undecomposed kernel, so the result is bitwise the oracle's.  Ranks use
GPU LOCAL_RANK % device count (one GPU: the ranks share it through CUDA IPC).
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
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 4
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
    st = b200.compile_stencil(workloads.source("dycore"), "dycore")
    A, B = b200.from_array(u, (2, 2, 0)), b200.from_array(u, (2, 2, 0))
    sc = workloads.DYCORE_SCALARS
    step_ab = decomp.PeerDecomposedStep(st, d, {"u_in": A, "u_out": B, **coef}, sc, "u_in", (2, 2))
    step_ba = decomp.PeerDecomposedStep(st, d, {"u_in": B, "u_out": A, **coef}, sc, "u_in", (2, 2))
    for s in range(steps):
        (step_ab if s % 2 == 0 else step_ba)()
    native.synchronize(step_ab.compute)
    last = B if steps % 2 == 1 else A
    got = last.host_array()[2:-2, 2:-2, :]
    want = oracle.dycore_run(arr["u"], arr["a"], arr["b"], arr["c"], steps, **sc)[2:-2, 2:-2, :]
    ok = bool(np.array_equal(got, want[d.i0: d.i1, d.j0: d.j1, :]))
    step_ab.exchanger.close()
    step_ba.exchanger.close()
    print(("DYCORE_PEER_OK " if ok else "DYCORE_PEER_FAIL ")
          + f"rank {rank} grid {grid} local {d.local_domain} steps {steps} bitwise {ok}", flush=True)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
