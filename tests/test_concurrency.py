"""Concurrent invocation ("ExecutableStencil is immutable and may
be invoked concurrently on disjoint output fields").

The b200 run closure keeps no per-call state in module globals: each thread
gets its own stream (native.default_stream), its own temporary arena (keyed by
stream; leases keep a grown arena alive until every holder's launches are
enqueued, gts_common.cuh GtsArenaLease), its own host-storage mirrors and its
own call statistics / timing flag (backend.call_stats, device_timing).
Storages shared read-only between threads upload under a per-storage lock.
"""

import ctypes
import threading

import numpy as np
import pytest

import oracle
import paper_2311_08322_b200 as b200
from paper_2311_08322_b200 import native, workloads

pytestmark = pytest.mark.gpu

ITERS = 200


def _run_threads(fns):
    errors = []

    def wrap(fn):
        try:
            fn()
        except BaseException as exc:  # noqa: BLE001 - reported below
            errors.append(exc)

    ts = [threading.Thread(target=wrap, args=(fn,)) for fn in fns]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errors:
        raise errors[0]


def test_two_threads_device_storages(gpu):
    """One hdiff stencil object called from two threads on disjoint outputs
    (sharing their input storage, freshly written on the host so both
    threads race to upload it), plus a vadv thread; 200 calls each, every
    result bitwise equal to the oracle; per-thread call statistics."""
    from paper_2311_08322_b200 import backend as b2b

    rng = np.random.default_rng(21)
    sh = b200.compile_stencil(workloads.source("hdiff"), "hdiff")
    sv = b200.compile_stencil(workloads.source("vadv"), "vadv")
    dom = (96, 160, 12)
    vals = rng.uniform(-1, 1, (dom[0] + 4, dom[1] + 4, dom[2]))
    inp = b200.allocate("f64", dom, (2, 2, 0))
    inp.view[...] = vals  # pending host write: the first calls upload it
    want_h = oracle.hdiff_c(vals, 0.05)
    a, b, c, d = oracle.make_diagonally_dominant(rng, (64, 96, 40))
    want_v = oracle.vadv_c(a, b, c, d)
    vin = {n: b200.from_array(v) for n, v in zip("abcd", (a, b, c, d))}

    def hdiff_worker(coeff_seen):
        def go():
            outs = [b200.allocate("f64", dom, fill="poison") for _ in range(2)]
            for it in range(ITERS):
                o = outs[it % 2]
                sh(inp=inp, coeff=0.05, out=o)
                st = b2b.call_stats()
                assert st["h2d"] == 0 and st["chunks"] == 0
                if it % 50 == 0 or it == ITERS - 1:
                    assert np.array_equal(o.host_array(), want_h), it
            coeff_seen.append(threading.get_ident())
        return go

    def vadv_worker():
        x = b200.allocate("f64", a.shape, fill="poison")
        for it in range(ITERS):
            sv(x=x, **vin)
            if it % 50 == 0 or it == ITERS - 1:
                assert np.array_equal(x.host_array(), want_v), it

    seen: list = []
    _run_threads([hdiff_worker(seen), hdiff_worker(seen), vadv_worker])
    assert len(set(seen)) == 2


def test_two_threads_pipelined_mirror_mode(gpu):
    """Host (pinned) FieldStorages: both threads take the pipelined mirror
    path (>= 2 row chunks) with the same stencil object, disjoint outputs and a
    shared input; 200 calls each, bitwise, and each thread's report counts
    only its own copies."""
    from paper_2311_08322_b200 import storage as b2s

    b200.install()
    st = b200.compile_stencil(workloads.source("hdiff"), "hdiff")
    dom = (200, 72, 6)
    rng = np.random.default_rng(22)
    vals = rng.uniform(-1, 1, (dom[0] + 4, dom[1] + 4, dom[2]))
    inp = b2s.pinned_host_storage("f64", dom, (2, 2, 0))
    inp.view[...] = vals
    want = oracle.hdiff_c(vals, 0.05)

    def worker():
        out = b2s.pinned_host_storage("f64", dom)
        for it in range(ITERS):
            out.view[...] = np.nan
            rep = st(inp=inp, coeff=0.05, out=out)
            assert rep.h2d_bytes > 0 and rep.d2h_bytes > 0
            assert np.array_equal(np.asarray(out.view), want), it

    _run_threads([worker, worker])


def test_timing_flag_is_per_thread(gpu):
    """B200CompiledStencil.time_device in one thread does not switch device
    timing on for another thread's calls (no global flag flip)."""
    st_t = b200.compile_stencil(workloads.source("hdiff"), "hdiff")
    st_t.time_device = True
    st_p = b200.compile_stencil(workloads.source("hdiff"), "hdiff")
    args_t = workloads.make_args("hdiff", (64, 48, 8))
    args_p = workloads.make_args("hdiff", (64, 48, 8))
    plain = []

    def timed():
        for _ in range(100):
            assert st_t(**args_t).device_ns is not None

    def untimed():
        for _ in range(100):
            plain.append(st_p(**args_p).device_ns)

    _run_threads([timed, untimed])
    assert plain and all(v is None for v in plain)


ARENA_SRC = """
stencil smooth(inp: Field[f64], out: Field[f64], w: f64):
    with computation(PARALLEL):
        with interval(0, None):
            t = inp * w
    with computation(FORWARD):
        with interval(0, None):
            out = t[1, 0, 0] + t[-1, 0, 0] * 0.5
"""


def _reference_smooth(vals, w):
    t = vals * w
    return t[2:, 1:-1, :] + t[:-2, 1:-1, :] * 0.5


def test_arena_growth_while_held_on_a_shared_stream(gpu):
    """Two host threads drive the raw C entry on ONE shared stream with
    growing domains, so the temporary arena grows while the other thread
    holds it: the grown-out arena is retired, not freed under the holder, and
    every result stays bitwise (the use-after-free window of a plain
    sync-and-cudaFree growth)."""
    st = b200.compile_stencil(ARENA_SRC, "smooth")
    module = st.build_info["module"]
    assert module.plan.global_temps == ("t",)
    stream = native.default_stream()
    rng = np.random.default_rng(23)
    sizes = [(8 + 6 * s, 40 + 3 * s, 5) for s in range(24)]
    cases = []
    for dom in sizes:
        vals = rng.uniform(-1, 1, (dom[0] + 2, dom[1] + 2, dom[2]))
        cases.append((dom, b200.from_array(vals, (1, 1, 0)), b200.allocate("f64", dom, fill="poison"),
                       _reference_smooth(vals, 0.25)))
    lock = threading.Lock()

    def worker(order):
        for idx in order:
            dom, inp, out, _ = cases[idx]
            ptrs = {"inp": inp.base_address(), "out": out.base_address()}
            strides = {"inp": inp.strides, "out": out.strides}
            origins = {"inp": inp.origin, "out": out.origin}
            module.launch(dom, ptrs, strides, origins, {"w": 0.25}, stream)
            with lock:
                out.mark_device_written(stream)

    idx = list(range(len(sizes)))
    _run_threads([lambda: worker(idx[0::2]), lambda: worker(idx[1::2])])
    native.synchronize(stream)
    for dom, inp, out, want in cases:
        assert np.array_equal(out.host_array(), want), dom
    assert module.launch_count() > 0
    # release frees every arena (retired ones included) without faulting
    module.lib.gts_b200_module_release.restype = ctypes.c_int
    assert module.lib.gts_b200_module_release() == 0
