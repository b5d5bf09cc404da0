"""The dycore-like multi-stage step (BASELINE.json configs[4],
paper_2311_08322_b200/kernels/dycore.gts): parity of the b200 backend with
the reference engines' golden outputs and with the oracle, per call and as a
CUDA-graph TimeLoop."""

from pathlib import Path

import numpy as np
import pytest

import oracle

GOLDEN = Path(__file__).parent / "golden"


def _state(dom, seed):
    import paper_2311_08322_b200 as b200
    from paper_2311_08322_b200 import workloads

    arr = workloads.dycore_arrays(dom, seed)
    bufs = [b200.from_array(arr["u"], (2, 2, 0)), b200.from_array(arr["u"], (2, 2, 0))]
    coef = {n: b200.from_array(arr[n]) for n in "abc"}
    return arr, bufs, coef


def test_dycore_lowering_plan():
    import paper_2311_08322_b200 as b200
    from paper_2311_08322_b200 import workloads

    st = b200.compile_stencil(workloads.source("dycore"), "dycore")
    plan = st.build_info["plan"]
    assert plan[0].startswith("pfused"), plan
    assert any(k.startswith("column") for k in plan), plan


@pytest.mark.gpu
def test_dycore_per_call_matches_reference_golden(gpu):
    import paper_2311_08322_b200 as b200
    from paper_2311_08322_b200 import workloads

    g = np.load(GOLDEN / "dycore.npz")
    st = b200.compile_stencil(workloads.source("dycore"), "dycore")
    for key in sorted({k.rsplit("_", 1)[0] for k in g.files}):
        dom = tuple(int(x) for x in key.split("_")[1].split("x"))
        _, bufs, coef = _state(dom, int(g[key + "_seed"]))
        for s in range(int(g[key + "_steps"])):
            src, dst = bufs[s % 2], bufs[(s + 1) % 2]
            st(u_in=src, u_out=dst, **coef, **workloads.DYCORE_SCALARS)
            assert np.array_equal(dst.host_array()[2:-2, 2:-2, :], g[f"{key}_out{s}"]), (key, s)


@pytest.mark.gpu
def test_dycore_timeloop_graph_matches_oracle(gpu):
    import paper_2311_08322_b200 as b200
    from paper_2311_08322_b200 import workloads
    from paper_2311_08322_b200.timeloop import TimeLoop

    dom, steps = (64, 72, 80), 6  # even: each replay starts and ends on binding 0
    arr, bufs, coef = _state(dom, 5)
    st = b200.compile_stencil(workloads.source("dycore"), "dycore")
    A, B = bufs
    loop = TimeLoop(st, [dict(u_in=A, u_out=B, **coef), dict(u_in=B, u_out=A, **coef)], steps,
                    workloads.DYCORE_SCALARS)
    loop.run()
    final = (A, B)[steps % 2]
    want = oracle.dycore_run(arr["u"], arr["a"], arr["b"], arr["c"], steps)
    assert np.array_equal(final.host_array(), want)
    # replaying the graph continues the integration
    loop.run()
    want2 = oracle.dycore_run(want, arr["a"], arr["b"], arr["c"], steps)
    final2 = (A, B)[(2 * steps) % 2]
    assert np.array_equal(final2.host_array(), want2)


@pytest.mark.gpu
@pytest.mark.parametrize("opts,align", [
    ({"fuse_prologue": False}, 128),  # hdiff launch + TMEM column kernel streaming uh
    ({"tmem": False}, 128),           # hdiff launch + generic column kernel
    ({"pro_coop": True}, 128),        # cooperative shared-memory Laplacian (opt-in)
    ({"pro_shfl": True}, 128),        # neighbour-lane shuffles of the Laplacian (opt-in)
    ({"pro_warps": 4}, 128),          # the prologue on its own warps, exports over the halo boxes
    ({}, 8),                          # TMA-incompatible storages: run-time fallback chain
])
def test_dycore_launch_paths_match_golden(gpu, opts, align):
    import paper_2311_08322_b200 as b200
    from paper_2311_08322_b200 import workloads
    from paper_2311_08322_b200.storage import LayoutSpec

    g = np.load(GOLDEN / "dycore.npz")
    key = "dycore_24x20x16"
    dom = (24, 20, 16)
    st = b200.compile_stencil(workloads.source("dycore"), "dycore", gen_options=opts or None)
    lay = LayoutSpec((2, 0, 1), align)
    arr = workloads.dycore_arrays(dom, int(g[key + "_seed"]))
    bufs = [b200.from_array(arr["u"], (2, 2, 0), lay), b200.from_array(arr["u"], (2, 2, 0), lay)]
    coef = {n: b200.from_array(arr[n], (0, 0, 0), lay) for n in "abc"}
    for s in range(int(g[key + "_steps"])):
        src, dst = bufs[s % 2], bufs[(s + 1) % 2]
        st(u_in=src, u_out=dst, **coef, **workloads.DYCORE_SCALARS)
        assert np.array_equal(dst.host_array()[2:-2, 2:-2, :], g[f"{key}_out{s}"]), (opts, align, s)


@pytest.mark.gpu
def test_dycore_configs4_size_100_steps_vs_reference_kernel(gpu):
    """BASELINE configs[4] at full size: 512x512x80 f64, 100 time steps in one
    CUDA-graph TimeLoop replay, bitwise against the reference gen engine's own
    kernel for dycore.gts (oracle/_ref, 100 host-swapped calls); the first 10
    steps also against the independent C restatement (oracle.dycore_run)."""
    import paper_2311_08322_b200 as b200
    from paper_2311_08322_b200 import workloads
    from paper_2311_08322_b200.timeloop import TimeLoop

    if not oracle.ref_available("dycore_f64"):
        pytest.fail("oracle/_ref/libdycore_f64.so missing: run __graft_entry__.build() in the build container")
    dom = (512, 512, 80)
    arr, bufs, coef = _state(dom, 1000)
    st = b200.compile_stencil(workloads.source("dycore"), "dycore")
    A, B = bufs
    binds = [dict(u_in=A, u_out=B, **coef), dict(u_in=B, u_out=A, **coef)]
    TimeLoop(st, binds, 10, workloads.DYCORE_SCALARS).run()
    want10 = oracle.dycore_run(arr["u"], arr["a"], arr["b"], arr["c"], 10)
    assert np.array_equal(A.host_array(), want10)
    TimeLoop(st, binds, 90, workloads.DYCORE_SCALARS).run()
    want100 = oracle.ref_dycore_run(want10, arr["a"], arr["b"], arr["c"], 90)
    got = A.host_array()
    assert np.isfinite(got).all()
    assert np.array_equal(got, want100), oracle.max_rel(got, want100)


@pytest.mark.gpu
def test_timeloop_host_write_after_view_is_not_lost(gpu):
    """reading ``.view`` (host-dirty) and then replaying a TimeLoop
    must not let a later call upload the stale host mirror over the newer
    device state: the replay uploads pending host data first."""
    import paper_2311_08322_b200 as b200
    from paper_2311_08322_b200 import workloads
    from paper_2311_08322_b200.timeloop import TimeLoop

    dom = (40, 36, 12)
    arr, (A, B), coef = _state(dom, 8)
    st = b200.compile_stencil(workloads.source("dycore"), "dycore")
    loop = TimeLoop(st, [dict(u_in=A, u_out=B, **coef), dict(u_in=B, u_out=A, **coef)], 2,
                    workloads.DYCORE_SCALARS)
    loop.run()
    _ = A.view[0, 0, 0]  # marks A host-dirty (the caller may write through it)
    _ = B.view[0, 0, 0]
    loop.run()
    st(u_in=A, u_out=B, **coef, **workloads.DYCORE_SCALARS)  # a plain call after the replay
    want = oracle.dycore_run(arr["u"], arr["a"], arr["b"], arr["c"], 5)
    assert np.array_equal(B.host_array(), want)
    assert loop.launches_per_step == 1  # the fused TMEM kernel: one launch per step
