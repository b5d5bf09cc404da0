#!/usr/bin/env python
"""Multi-process check of the peer-memory halo exchange (decomp.PeerDecomposedStep).

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port P tools/peer_halo_check.py [steps] [--timing]

Every rank builds the same seeded global hdiff input, takes its box of a
(N-way) decomposition, poisons the halo cells its neighbours own, and runs
``steps`` decomposed hdiff steps whose halos arrive only through CUDA-IPC peer
stores + flags (no NCCL; gloo only for the one-off handle exchange).  The
ranks use GPU (LOCAL_RANK % device count): with one GPU both processes share
it (IPC within a device), on an 8-GPU box the puts travel over NVLink.  Each
rank compares its output box with the C oracle on the global input (bitwise)
and prints PEER_OK.  --timing adds per-step device time (max over ranks).
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
    steps = int(sys.argv[1]) if len(sys.argv) > 1 and not sys.argv[1].startswith("--") else 3
    timing = "--timing" in sys.argv
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()

    import oracle
    import paper_2311_08322_b200 as b200
    from paper_2311_08322_b200 import decomp, native, workloads

    native.set_device(int(os.environ.get("LOCAL_RANK", "0")) % native.device_count())
    tile = tuple(int(x) for x in os.environ.get("PEER_TILE", "64x96x8").split("x"))
    grid = decomp.choose_grid(world)
    gdom = (tile[0] * grid[0] + 3, tile[1] * grid[1] + 5, tile[2])  # ragged split
    rng = np.random.default_rng(77)
    g = rng.uniform(-1, 1, (gdom[0] + 4, gdom[1] + 4, gdom[2]))
    d = decomp.Decomposition(gdom, grid, rank)
    ni, nj, nk = d.local_domain
    loc = d.scatter(g, (2, 2))
    if d.neighbour(-1, 0) is not None:
        loc[:2] = np.nan
    if d.neighbour(1, 0) is not None:
        loc[ni + 2:] = np.nan
    if d.neighbour(0, -1) is not None:
        loc[:, :2] = np.nan
    if d.neighbour(0, 1) is not None:
        loc[:, nj + 2:] = np.nan
    st = b200.compile_stencil(workloads.source("hdiff"), "hdiff")
    inp = b200.from_array(loc, (2, 2, 0))
    out = b200.allocate("f64", d.local_domain)
    step = decomp.PeerDecomposedStep(st, d, {"inp": inp, "out": out}, {"coeff": 0.05}, "inp", (2, 2))
    for _ in range(steps):
        step()
    native.synchronize(step.compute)
    if os.environ.get("PEER_DEBUG"):
        import ctypes
        full = d.scatter(g, (2, 2))
        have = inp.host_array()
        ow = out.host_array()
        wv = oracle.hdiff_c(g, 0.05)[d.i0: d.i1, d.j0: d.j1]
        ob = np.argwhere(ow != wv)
        print(f"DEBUG rank {rank} out bad {len(ob)} rows {sorted(set(ob[:, 0].tolist()))[:10]}", flush=True)
        bad = ~((have == full) | (np.isnan(have) & np.isnan(full)))
        fl = (ctypes.c_uint64 * 8)()
        native.call("gts_b200_memcpy_d2h", ctypes.addressof(fl), step.exchanger._flags.dptr, 64, step.compute)
        ex = (ctypes.c_uint64 * 8)()
        native.call("gts_b200_memcpy_d2h", ctypes.addressof(ex), step.exchanger._expect.dptr, 64, step.compute)
        native.synchronize(step.compute)
        idx = np.argwhere(bad)
        print(f"DEBUG rank {rank} bad {int(bad.sum())} nan {int(np.isnan(have).sum())} "
              f"rows {sorted(set(idx[:, 0].tolist()))[:8]} cols {sorted(set(idx[:, 1].tolist()))[:8]} "
              f"flags {list(fl)} expect {list(ex)} peers { {k: (hex(v[0]), v[1], hex(v[2])) for k, v in step.exchanger.peer.items()} }",
              flush=True)
    want = oracle.hdiff_c(g, 0.05)[d.i0: d.i1, d.j0: d.j1]
    got = out.host_array()
    ok = bool(np.array_equal(got, want))
    # the same steps captured in a CUDA graph, replayed twice, after the
    # neighbour-owned halo cells were poisoned again and the output zeroed
    gr = step.graph(steps)
    native.synchronize(step.compute)
    dist.barrier()
    inp.view[...] = loc
    inp.to_device()
    out.view[...] = 0.0
    out.to_device()
    dist.barrier()
    for _ in range(2):
        gr.launch()
    native.synchronize(step.compute)
    ok_g = bool(np.array_equal(out.host_array(), want))
    if os.environ.get("PEER_DEBUG"):
        have = inp.host_array()
        full = d.scatter(g, (2, 2))
        bad = ~((have == full) | (np.isnan(have) & np.isnan(full)))
        ob = np.argwhere(out.host_array() != want)
        print(f"DEBUG-G rank {rank} halo bad {int(bad.sum())} out bad {len(ob)} rows {sorted(set(ob[:, 0].tolist()))[:10]}"
              f" cols {sorted(set(ob[:, 1].tolist()))[:10]}", flush=True)
    ok = ok and ok_g
    line = f"rank {rank} grid {grid} local {d.local_domain} steps {steps} bitwise {ok} (graph replay {ok_g})"
    if timing:
        e0, e1 = native.Event(), native.Event()
        dist.barrier()
        e0.record(step.compute)
        for _ in range(20):
            step()
        e1.record(step.compute)
        native.synchronize(step.compute)
        line += f" eager_ms_per_step {e0.elapsed_ms(e1) / 20:.4f}"
        g20 = step.graph(20)
        g20.launch()
        native.synchronize(step.compute)
        dist.barrier()
        e0.record(step.compute)
        g20.launch()
        e1.record(step.compute)
        native.synchronize(step.compute)
        line += f" graph_ms_per_step {e0.elapsed_ms(e1) / 20:.4f}"
    step.exchanger.close()
    print(("PEER_OK " if ok else "PEER_FAIL ") + line, flush=True)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
