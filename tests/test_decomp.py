"""Horizontal decomposition + halo exchange (paper_2311_08322_b200/decomp.py).

CPU part: world_size 2 and 4 over gloo (host transport) -- the rank grid,
the two-phase face exchange (corners included) and the decomposed hdiff
computed per rank with the C oracle equal to the undecomposed result.
GPU part: the device pack/unpack kernels and strip-wise stencil calls on one
B200, bitwise equal to the undecomposed run.
"""

import os
import socket

import numpy as np
import pytest

from paper_2311_08322_b200 import decomp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_grid_covers_domain_once(world):
    dom = (37, 29, 3)
    grid = decomp.choose_grid(world)
    assert grid[0] * grid[1] == world
    seen = np.zeros(dom[:2], dtype=int)
    for r in range(world):
        d = decomp.Decomposition(dom, grid, r)
        seen[d.i0: d.i1, d.j0: d.j1] += 1
        for di, dj in ((-1, 0), (1, 0), (0, -1), (0, 1)):
            nb = d.neighbour(di, dj)
            if nb is not None:
                e = decomp.Decomposition(dom, grid, nb)
                assert (e.ri - d.ri, e.rj - d.rj) == (di, dj)
    assert np.all(seen == 1)


def test_strips_partition_local_domain():
    for dom in [(12, 9, 2), (4, 4, 1), (5, 30, 3)]:
        cover = np.zeros(dom[:2], dtype=int)
        for _, (oi, oj), (si, sj, _) in decomp.strips(dom, (2, 2)):
            cover[oi: oi + si, oj: oj + sj] += 1
        assert np.all(cover == 1)


@pytest.mark.parametrize("dom", [(512, 1024, 1), (37, 300, 1), (8, 70, 1), (6, 40, 1), (100, 64, 1)])
@pytest.mark.parametrize("tile", [(4, 32), (2, 32), (8, 128)])
@pytest.mark.parametrize("sides", [(1, 1, 1, 1), (0, 1, 1, 0), (1, 0, 0, 1), (0, 0, 0, 1), (1, 1, 0, 0)])
def test_frame_interior_complements_frame_tiles(dom, tile, sides):
    """The interior launch (decomp.frame_interior) and the frame launch's
    tiles (every tile outside the inner rectangle, gts_frame_tile in
    gts_sm100.cuh; the rectangle as the generated launch computes it) cover
    the local domain exactly once, and the interior reads no halo cell of a
    field of extent (2, 2) on a side with a band (a neighbour); sides without
    one let the interior reach the domain edge."""
    ni, nj, _ = dom
    ilo, ihi, jlo, jhi = (2 * sides[0], 2 * sides[1], 2 * sides[2], 2 * sides[3])
    ti, tj = tile
    tiles_i, tiles_j = -(-ni // ti), -(-nj // tj)
    fi0, fi1 = -(-ilo // ti), ((ni - ihi) // ti if ihi else tiles_i)
    fj0, fj1 = -(-jlo // tj), ((nj - jhi) // tj if jhi else tiles_j)
    fi1, fj1 = max(fi1, fi0), max(fj1, fj0)  # the generated launch's clamp
    cover = np.zeros(dom[:2], dtype=int)
    for a in range(tiles_i):
        for b in range(tiles_j):
            if not (fi0 <= a < fi1 and fj0 <= b < fj1):
                cover[a * ti: (a + 1) * ti, b * tj: (b + 1) * tj] += 1
    box = decomp.frame_interior(dom, (ilo, ihi, jlo, jhi), tile)
    if box is not None:
        (i0, j0), (si, sj, _) = box
        assert i0 >= ilo and j0 >= jlo and i0 + si <= ni - ihi and j0 + sj <= nj - jhi
        cover[i0: i0 + si, j0: j0 + sj] += 1
    assert np.all(cover == 1)
    if sides == (1, 1, 1, 1):  # the (hi, hj) spelling is the same band
        assert decomp.frame_interior(dom, (2, 2), tile) == box


def test_neighbour_sides():
    """decomp.neighbour_sides on a 4x2 grid: corner, edge and interior ranks."""
    g = (2048, 2048, 80)
    sides = {r: decomp.neighbour_sides(decomp.Decomposition(g, (4, 2), r)) for r in range(8)}
    assert sides[0] == (False, True, False, True)
    assert sides[3] == (True, True, True, False)
    assert sides[7] == (True, False, True, False)
    assert decomp.neighbour_sides(decomp.Decomposition(g, (1, 1), 0)) == (False,) * 4


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle

        glob_dom = (26, 21, 4)
        rng = np.random.default_rng(42)
        g_inp = rng.uniform(-1, 1, (glob_dom[0] + 4, glob_dom[1] + 4, glob_dom[2]))
        d = decomp.Decomposition(glob_dom, decomp.choose_grid(world), rank)
        local = d.scatter(g_inp, (2, 2))
        want_halo = local.copy()
        ni, nj, _ = d.local_domain
        # poison every halo cell that a neighbour owns, keep global-boundary halos
        poisoned = local.copy()
        if d.neighbour(-1, 0) is not None:
            poisoned[:2] = np.nan
        if d.neighbour(1, 0) is not None:
            poisoned[ni + 2:] = np.nan
        if d.neighbour(0, -1) is not None:
            poisoned[:, :2] = np.nan
        if d.neighbour(0, 1) is not None:
            poisoned[:, nj + 2:] = np.nan
        ex = decomp.HaloExchanger(d, (2, 2), "f64", device=False)
        ex.exchange(poisoned)
        # hdiff needs no corner cells, but the two-phase exchange delivers them too
        ok_halo = np.array_equal(poisoned, want_halo)
        out_local = oracle.hdiff_c(poisoned, 0.05)
        out_global = oracle.hdiff_c(g_inp, 0.05)
        ok_out = np.array_equal(out_local, out_global[d.i0: d.i1, d.j0: d.j1])
        q.put((rank, ok_halo, ok_out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_halo_exchange_and_decomposed_hdiff(world):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(ok_h and ok_o for _, ok_h, ok_o in res), res


@pytest.mark.gpu
def test_device_pack_unpack_and_strips_bitwise(gpu):
    """Two sub-domains on one GPU: faces moved with the device pack/unpack
    kernels, each sub-domain computed as interior + 4 strips; bitwise equal
    to the undecomposed hdiff."""
    import torch

    import oracle
    import paper_2311_08322_b200 as b200
    from paper_2311_08322_b200 import native, workloads

    glob_dom = (40, 70, 6)
    rng = np.random.default_rng(7)
    g_inp = rng.uniform(-1, 1, (glob_dom[0] + 4, glob_dom[1] + 4, glob_dom[2]))
    st = b200.compile_stencil(workloads.source("hdiff"), "hdiff")
    grid = (2, 1)
    parts = []
    for r in range(2):
        d = decomp.Decomposition(glob_dom, grid, r)
        local = d.scatter(g_inp, (2, 2))
        if r == 0:
            local[d.local_domain[0] + 2:] = np.nan  # owned by rank 1
        else:
            local[:2] = np.nan  # owned by rank 0
        parts.append((d, b200.from_array(local, (2, 2, 0)), b200.allocate("f64", d.local_domain)))
    ops = decomp._DeviceOps(torch, native.default_stream())
    (d0, in0, _), (d1, in1, _) = parts
    ni0, nj, nk = d0.local_domain
    buf = torch.empty(2 * (nj + 4) * nk, dtype=torch.float64, device="cuda")
    ops.pack(buf, in0, ((ni0, 0, 0), (2, nj + 4, nk)))  # rank 0 bottom interior rows
    ops.unpack(in1, buf, ((0, 0, 0), (2, nj + 4, nk)))  # -> rank 1 top halo
    ops.pack(buf, in1, ((2, 0, 0), (2, nj + 4, nk)))  # rank 1 top interior rows
    ops.unpack(in0, buf, ((ni0 + 2, 0, 0), (2, nj + 4, nk)))  # -> rank 0 bottom halo
    ops.synchronize()
    in0.mark_device_written()
    in1.mark_device_written()
    want = oracle.hdiff_c(g_inp, 0.05)
    for d, inp, out in parts:
        for _, off, size in decomp.strips(d.local_domain, (2, 2)):
            decomp.call_on_strip(st, {"inp": inp, "out": out}, {"coeff": 0.05}, off, size)
        assert np.array_equal(out.host_array(), want[d.i0: d.i1, d.j0: d.j1])


@pytest.mark.parametrize("world", [2, 4, 8])
def test_peer_face_puts_fill_every_halo(world):
    """decomp.face_puts (the peer-memory transport's boxes), simulated with
    numpy: after phase i then phase j of direct puts into the neighbours'
    halos, every rank's storage equals its box of the global storage,
    corners included -- with every neighbour-owned halo cell poisoned first."""
    halo = (2, 2)
    gdom = (23, 19, 3)
    grid = decomp.choose_grid(world)
    rng = np.random.default_rng(world)
    g = rng.uniform(-1, 1, (gdom[0] + 4, gdom[1] + 4, gdom[2]))
    ds = [decomp.Decomposition(gdom, grid, r) for r in range(world)]
    local = [d.scatter(g, halo) for d in ds]
    want = [x.copy() for x in local]
    for d, x in zip(ds, local):
        ni, nj, _ = d.local_domain
        if d.neighbour(-1, 0) is not None:
            x[:2] = np.nan
        if d.neighbour(1, 0) is not None:
            x[ni + 2:] = np.nan
        if d.neighbour(0, -1) is not None:
            x[:, :2] = np.nan
        if d.neighbour(0, 1) is not None:
            x[:, nj + 2:] = np.nan
    def put(r, axis, into=None):
        for _, nb, src, dst, size in decomp.face_puts(ds[r], halo, axis):
            if into is None or nb == into:
                blk = local[r][src[0]: src[0] + size[0], src[1]: src[1] + size[1], :]
                local[nb][dst[0]: dst[0] + size[0], dst[1]: dst[1] + size[1], :] = blk

    # adversarial but legal order: rank r's j-puts run as soon as its own
    # i-halos landed, before later ranks received theirs (no ordering
    # between writers of one halo other than the flags)
    for r in range(world):
        for q in range(world):
            put(q, "i", into=r)
        put(r, "j")
    for r in range(world):
        assert np.array_equal(local[r], want[r]), r


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4])
def test_peer_halo_exchange_multiprocess(world):
    """PeerDecomposedStep across ``world`` processes sharing the box's GPU(s):
    halos arrive only through CUDA-IPC peer stores + step-numbered flags
    (no NCCL); every rank's output is bitwise the undecomposed oracle's."""
    import subprocess
    import sys
    from pathlib import Path

    repo = Path(__file__).resolve().parent.parent
    env = dict(os.environ, PEER_TILE="40x72x6")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           str(repo / "tools" / "peer_halo_check.py"), "3"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, env=env, cwd=str(repo))
    # ranks print concurrently: lines may interleave, so count markers
    assert r.returncode == 0 and r.stdout.count("PEER_OK") == world and "PEER_FAIL" not in r.stdout, (
        r.stdout[-2000:], r.stderr[-3000:])


@pytest.mark.gpu
def test_peer_dycore_decomposed_multiprocess():
    """The fused dycore step (kernels/dycore.gts) decomposed over 2 processes
    with the peer-memory exchange of u_in's halo (two PeerDecomposedSteps for
    the u_in / u_out swap): bitwise the undecomposed oracle after 4 steps."""
    import subprocess
    import sys
    from pathlib import Path

    repo = Path(__file__).resolve().parent.parent
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           str(repo / "tools" / "peer_dycore_check.py"), "4"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=str(repo))
    assert r.returncode == 0 and r.stdout.count("DYCORE_PEER_OK") == 2, (r.stdout[-2000:], r.stderr[-3000:])


@pytest.mark.parametrize("grid", [(2, 1), (1, 2), (2, 2), (4, 2), (3, 3)])
def test_mirror_boxes_cover_every_halo_once(grid):
    """decomp.mirror_boxes (PeerFusedStep): the cells every rank sends into
    its neighbours' halos are exactly those neighbours' 2-deep halo cells
    inside the global domain (faces and corners), each sent once, by its
    owner."""
    from paper_2311_08322_b200 import decomp

    gdom = (9 * grid[0] + 3, 11 * grid[1] + 5, 4)
    h = (2, 2)
    ranks = [decomp.Decomposition(gdom, grid, r) for r in range(grid[0] * grid[1])]
    got = {r: [] for r in range(len(ranks))}
    for d in ranks:
        for di, nb, (i0, i1, j0, j1) in decomp.mirror_boxes(d, h):
            for i in range(i0, i1):
                for j in range(j0, j1):
                    got[nb].append((d.i0 + i, d.j0 + j))
    for n in ranks:
        want = sorted((gi, gj)
                      for gi in range(max(0, n.i0 - h[0]), min(gdom[0], n.i1 + h[0]))
                      for gj in range(max(0, n.j0 - h[1]), min(gdom[1], n.j1 + h[1]))
                      if not (n.i0 <= gi < n.i1 and n.j0 <= gj < n.j1))
        assert sorted(got[n.rank]) == want, n.rank


def test_mirror_option_rejects_unsupported_fields():
    """gen_options mirror needs an api field written by one TMEM column or
    fused PARALLEL tile kernel (the templates that carry the mirror stores):
    a temporary, or an output only a per-point fallback kernel can produce
    (a vertical-offset read), is refused at build time; hdiff's out is
    accepted."""
    import paper_2311_08322_b200 as b200
    from paper_2311_08322_b200 import workloads

    vshift = ("stencil vshift(inp: Field[f64], out: Field[f64]):\n"
              "    with computation(PARALLEL):\n"
              "        with interval(0, -1):\n"
              "            out = inp[0, 0, 1]\n")
    for src, name, field in ((workloads.source("dycore"), "dycore", "lap"), (vshift, "vshift", "out")):
        with pytest.raises(Exception, match="mirror"):
            b200.compile_stencil(src, name, gen_options={"mirror": field})
    st = b200.compile_stencil(workloads.source("hdiff"), "hdiff", gen_options={"mirror": "out"})
    assert st.build_info["module"]._mirror_fn is not None


@pytest.mark.gpu
@pytest.mark.parametrize("kernel", ["dycore", "hdiff"])
@pytest.mark.parametrize("nproc,steps", [(2, 4), (4, 2)])
def test_peer_fused_multiprocess(nproc, steps, kernel):
    """A time loop with the halo exchange fused into the producing kernel
    (PeerFusedStep, peer stores corners included): the dycore (TMEM column
    kernel's epilogue) and the hdiff ping-pong loop (fused PARALLEL tile
    kernel's output stores); bitwise the undecomposed oracle, eager and
    replayed from a CUDA graph, with 2 and 4 processes sharing one B200."""
    import subprocess
    import sys
    from pathlib import Path

    repo = Path(__file__).resolve().parent.parent
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           str(repo / "tools" / "peer_fused_check.py"), str(steps), "--kernel", kernel]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=400, cwd=str(repo))
    assert r.returncode == 0 and r.stdout.count("FUSED_PEER_OK") == nproc, (r.stdout[-2000:], r.stderr[-3000:])


def test_peer_fused_step_needs_mirrored_build():
    """PeerFusedStep refuses a stencil built without gen_options mirror (its
    column kernel would not store into the neighbours' halos)."""
    import paper_2311_08322_b200 as b200
    from paper_2311_08322_b200 import decomp, workloads

    st = b200.compile_stencil(workloads.source("dycore"), "dycore")
    d = decomp.Decomposition((8, 8, 4), (1, 1), 0)
    with pytest.raises(ValueError, match="mirror"):
        decomp.PeerFusedStep(st, d, [{}], {}, "u_out", (2, 2))
    assert st.build_info["module"]._mirror_fn is None
    sm = b200.compile_stencil(workloads.source("dycore"), "dycore", gen_options={"mirror": "u_out"})
    assert sm.build_info["module"]._mirror_fn is not None


@pytest.mark.gpu
def test_mirror_stores_exact_cells_single_process():
    """gen_options mirror on one GPU: 8 boxes (the 2-deep faces and corners of
    the domain) pointed at a scratch field with the identity mapping; after
    one dycore step the scratch holds exactly u_out on the boxes' cells and is
    untouched elsewhere (bitwise), and u_out is the plain build's."""
    import numpy as np

    import paper_2311_08322_b200 as b200
    from paper_2311_08322_b200 import native, workloads

    dom = (37, 70, 9)
    arr = workloads.dycore_arrays(dom, 5)
    sc = workloads.DYCORE_SCALARS
    coef = {n: b200.from_array(arr[n]) for n in "abc"}
    st_m = b200.compile_stencil(workloads.source("dycore"), "dycore", gen_options={"mirror": "u_out"})
    st_p = b200.compile_stencil(workloads.source("dycore"), "dycore")
    u = b200.from_array(arr["u"], (2, 2, 0))
    out_m, out_p = b200.from_array(arr["u"], (2, 2, 0)), b200.from_array(arr["u"], (2, 2, 0))
    scratch = b200.from_array(np.full_like(arr["u"], -7.0), (2, 2, 0))
    ni, nj, _ = dom
    org = sum(o * s for o, s in zip(scratch.origin, scratch.strides)) * scratch.itemsize
    boxes = []
    for di in (-1, 0, 1):
        for dj in (-1, 0, 1):
            if di == dj == 0:
                continue
            i0, i1 = {-1: (0, 2), 0: (0, ni), 1: (ni - 2, ni)}[di]
            j0, j1 = {-1: (0, 2), 0: (0, nj), 1: (nj - 2, nj)}[dj]
            boxes.append((i0, i1, j0, j1, scratch.base_address() + org, *scratch.strides))
    mod = st_m.build_info["module"]
    mod.set_mirror(boxes)  # for the next launch only (consumed by it)
    st_m(u_in=u, u_out=out_m, **coef, **sc)
    st_p(u_in=u, u_out=out_p, **coef, **sc)
    native.synchronize(native.default_stream())
    scratch.mark_device_written()
    got_out, want_out = out_m.host_array(), out_p.host_array()
    assert np.array_equal(got_out, want_out)
    s = scratch.host_array()[2:-2, 2:-2, :]
    o = got_out[2:-2, 2:-2, :]
    band = np.zeros(dom, bool)
    band[:2], band[-2:], band[:, :2], band[:, -2:] = True, True, True, True
    assert np.array_equal(s[band], o[band])
    assert np.all(s[~band] == -7.0)
    assert np.all(scratch.host_array()[:2] == -7.0) and np.all(scratch.host_array()[:, :2] == -7.0)
    # the boxes were consumed by that launch: a later plain call of the same
    # module stores nothing outside its own output (no stale peer
    # pointers after PeerFusedStep.close())
    scratch.view[...] = -9.0
    scratch.to_device()
    st_m(u_in=u, u_out=out_m, **coef, **sc)
    scratch.mark_device_written()  # re-read the device copy below
    assert np.all(scratch.host_array() == -9.0)


@pytest.mark.parametrize("grid", [(2, 2), (3, 3), (4, 2)])
def test_mirror_descriptors_fill_halos_on_host(grid):
    """decomp.mirror_descriptor addressing, emulated with numpy: every rank
    stores its boxes' cells through the descriptors (base + i*s_i + j*s_j +
    k*s_k) into its neighbours' storages; afterwards every halo cell inside
    the global domain holds the global value, every other halo cell is
    untouched."""
    import numpy as np

    from paper_2311_08322_b200 import decomp

    gdom = (7 * grid[0] + 3, 9 * grid[1] + 2, 3)
    rng = np.random.default_rng(3)
    g = rng.uniform(-1, 1, gdom)
    ds = [decomp.Decomposition(gdom, grid, r) for r in range(grid[0] * grid[1])]
    st = {}
    for d in ds:
        ni, nj, nk = d.local_domain
        a = np.full((ni + 4, nj + 4, nk), np.nan)
        a[2:-2, 2:-2] = g[d.i0:d.i1, d.j0:d.j1]
        st[d.rank] = a
    item = 8
    for d in ds:
        for _, nb, box in decomp.mirror_boxes(d, (2, 2)):
            dst = st[nb]
            strides = tuple(s // item for s in dst.strides)
            desc = decomp.mirror_descriptor(d, ds[nb], box, 0, strides, (2, 2, 0), item)
            i0, i1, j0, j1, base, si, sj, sk = desc
            flat = dst.reshape(-1)
            for i in range(i0, i1):
                for j in range(j0, j1):
                    for k in range(gdom[2]):
                        flat[base // item + i * si + j * sj + k * sk] = st[d.rank][2 + i, 2 + j, k]
    for d in ds:
        a = st[d.rank]
        for li in range(a.shape[0]):
            for lj in range(a.shape[1]):
                gi, gj = d.i0 + li - 2, d.j0 + lj - 2
                inside = 0 <= gi < gdom[0] and 0 <= gj < gdom[1]
                if inside:
                    assert np.array_equal(a[li, lj], g[gi, gj]), (d.rank, li, lj)
                else:
                    assert np.all(np.isnan(a[li, lj])), (d.rank, li, lj)


@pytest.mark.parametrize("nranks", [2, 3, 4])
def test_fused_step_protocol_model(nranks):
    """The PeerFusedStep step protocol (one arrival counter per neighbour,
    initialised to 1; per step: wait until every neighbour's counter reaches
    the step count + 1, run the kernel, bump every neighbour's counter), model
    checked on a chain of ranks over many random schedules: a kernel never
    writes a neighbour's halo while that neighbour's kernel reads it, and
    every halo a kernel reads was written by the neighbours' previous step."""
    import random

    steps = 6
    nbs = {r: [n for n in (r - 1, r + 1) if 0 <= n < nranks] for r in range(nranks)}
    for seed in range(300):
        rnd = random.Random(seed)
        arrived = {r: {n: 1 for n in nbs[r]} for r in range(nranks)}  # arrivals at r from n
        step = {r: 0 for r in range(nranks)}
        state = {r: "wait" for r in range(nranks)}  # wait -> run -> (signal) -> wait
        halo_written = {(r, b): {n: -1 for n in nbs[r]} for r in range(nranks) for b in (0, 1)}
        while any(step[r] < steps for r in range(nranks)):
            r = rnd.choice([x for x in range(nranks) if step[x] < steps])
            s = step[r]
            if state[r] == "wait":
                if all(arrived[r][n] >= s + 1 for n in nbs[r]):
                    state[r] = "run"
                    # the kernel reads buffer s % 2's halo: written by each neighbour's step s-1
                    for n in nbs[r]:
                        assert s == 0 or halo_written[(r, s % 2)][n] == s - 1, (seed, r, s, n)
            else:  # "run": the kernel writes neighbours' buffer (s+1) % 2 halo, then signals
                for n in nbs[r]:
                    # n must not be running a step that reads buffer (s+1) % 2, i.e. s-1 or s+1
                    assert not (state[n] == "run" and step[n] in (s - 1, s + 1)), (seed, r, s, n, step[n])
                    halo_written[(n, (s + 1) % 2)][r] = s
                    arrived[n][r] += 1
                state[r] = "wait"
                step[r] += 1
            # writer (step s, anywhere in its run) and reader (step s +- 1) never overlap
            for x in range(nranks):
                for n in nbs[x]:
                    assert not (state[x] == "run" and state[n] == "run" and abs(step[x] - step[n]) == 1), seed


@pytest.mark.gpu
@pytest.mark.parametrize("dom", [(512, 1024, 6), (37, 300, 3), (70, 33, 2), (5, 200, 2), (3, 3, 2)])
@pytest.mark.parametrize("sides", [True, (False, True, True, False), (True, False, False, False)])
def test_interior_plus_frame_launch_bitwise(dom, sides):
    """decomp.split_launches on one GPU: the interior box launch (the frame's
    inner tile rectangle) + ONE frame launch (thin tiles touching the 2-deep
    band on the sides with a neighbour: all four, or per side as
    decomp.neighbour_sides gives them) compute every point exactly like the
    single full launch (bitwise vs the oracle, output poisoned first); the
    frame launch alone writes the whole band."""
    import numpy as np

    import oracle
    import paper_2311_08322_b200 as b200
    from paper_2311_08322_b200 import decomp, native, workloads

    st = b200.compile_stencil(workloads.source("hdiff"), "hdiff")
    module = st.build_info["module"]
    assert module.frame_supported
    vals = np.random.default_rng(sum(dom)).uniform(-1, 1, (dom[0] + 4, dom[1] + 4, dom[2]))
    want = oracle.hdiff_c(vals, 0.05)
    inp = b200.from_array(vals, (2, 2, 0))
    stream = native.default_stream()
    out = b200.allocate("f64", dom, fill="poison")
    fields = {"inp": inp, "out": out}
    interior, boundary = decomp.split_launches(module, dom, (2, 2), fields, {"coeff": 0.05}, stream, sides)
    has_interior = dom[0] > 4 and dom[1] > 4
    sd = (True,) * 4 if sides is True else sides
    bands = tuple(2 * int(x) for x in sd)
    # with a frame launch the interior is its inner tile rectangle (maybe empty)
    n_int = (1 if decomp.frame_interior(dom, bands, module.frame_tile) else 0) if has_interior else 1
    assert len(interior) == n_int and len(boundary) == (1 if has_interior else 0)
    n0 = module.launch_count()
    for go in interior + boundary:
        go()
    native.synchronize(stream)
    assert module.launch_count() - n0 == len(interior) + len(boundary)
    assert np.array_equal(out.host_array(), want)
    if has_interior:
        out2 = b200.allocate("f64", dom, fill="poison")
        fields2 = {"inp": inp, "out": out2}
        _, frame = decomp.split_launches(module, dom, (2, 2), fields2, {"coeff": 0.05}, stream, sides)
        frame[0]()
        native.synchronize(stream)
        got = out2.host_array()
        band = np.zeros(dom, bool)
        band[:bands[0]], band[dom[0] - bands[1]:] = True, True
        band[:, :bands[2]], band[:, dom[1] - bands[3]:] = True, True
        assert np.array_equal(got[band], want[band])
        # interior points are either untouched (poison) or the same values
        inner = got[~band]
        assert np.all(np.isnan(inner) | (inner == want[~band]))


@pytest.mark.gpu
@pytest.mark.parametrize("dom", [(512, 1024, 4), (37, 300, 3), (70, 33, 2)])
def test_decomposed_step_split_bitwise(dom):
    """DecomposedStep(split=True) on one GPU (the bench's ``split_us``
    configuration): interior launch + frame launch, eager and replayed from a
    CUDA graph, bitwise equal to the oracle (outputs poisoned first).
    Running the frame on the communication stream concurrently with the
    interior measured slower (512x1024x80: 142.7 vs 133.4 us per step: the
    frame's CTAs take SM slots the interior's persistent grid counts on), so
    the frame waits for the interior."""
    import numpy as np

    import oracle
    import paper_2311_08322_b200 as b200
    from paper_2311_08322_b200 import decomp, native, workloads

    st = b200.compile_stencil(workloads.source("hdiff"), "hdiff")
    vals = np.random.default_rng(sum(dom) + 1).uniform(-1, 1, (dom[0] + 4, dom[1] + 4, dom[2]))
    want = oracle.hdiff_c(vals, 0.05)
    d = decomp.Decomposition(dom, (1, 1), 0)
    inp = b200.from_array(vals, (2, 2, 0))
    out = b200.allocate("f64", dom, fill="poison")
    step = decomp.DecomposedStep(st, d, {"inp": inp, "out": out}, {"coeff": 0.05}, "inp", (2, 2), split=True)
    assert step.launches_per_step == (2 if decomp.frame_interior(dom, (2, 2), st.build_info["module"].frame_tile)
                                      else 1)
    step()
    native.synchronize(step.compute)
    assert np.array_equal(out.host_array(), want)
    out2 = b200.allocate("f64", dom, fill="poison")
    step2 = decomp.DecomposedStep(st, d, {"inp": inp, "out": out2}, {"coeff": 0.05}, "inp", (2, 2), split=True)
    step2.graph(3).launch()
    native.synchronize(step2.compute)
    assert np.array_equal(out2.host_array(), want)


@pytest.mark.gpu
def test_hdiff_mirror_stores_exact_cells_single_process():
    """gen_options mirror on the fused PARALLEL tile kernel (hdiff): 8 boxes
    (the 2-deep faces and corners of the domain) pointed at a scratch field
    with the identity mapping; after one launch the scratch holds exactly
    ``out`` on the boxes' cells and is untouched elsewhere, ``out`` is the
    plain build's (bitwise), and the boxes are consumed by that launch."""
    import numpy as np

    import oracle
    import paper_2311_08322_b200 as b200
    from paper_2311_08322_b200 import native, workloads

    dom = (37, 300, 5)
    vals = np.random.default_rng(7).uniform(-1, 1, (dom[0] + 4, dom[1] + 4, dom[2]))
    st_m = b200.compile_stencil(workloads.source("hdiff"), "hdiff", gen_options={"mirror": "out"})
    inp = b200.from_array(vals, (2, 2, 0))
    out = b200.allocate("f64", dom, (2, 2, 0), fill="poison")
    scratch = b200.from_array(np.full((dom[0] + 4, dom[1] + 4, dom[2]), -7.0), (2, 2, 0))
    ni, nj, _ = dom
    org = sum(o * s for o, s in zip(scratch.origin, scratch.strides)) * scratch.itemsize
    boxes = []
    for di in (-1, 0, 1):
        for dj in (-1, 0, 1):
            if di == dj == 0:
                continue
            i0, i1 = {-1: (0, 2), 0: (0, ni), 1: (ni - 2, ni)}[di]
            j0, j1 = {-1: (0, 2), 0: (0, nj), 1: (nj - 2, nj)}[dj]
            boxes.append((i0, i1, j0, j1, scratch.base_address() + org, *scratch.strides))
    mod = st_m.build_info["module"]
    mod.set_mirror(boxes)
    st_m(inp=inp, coeff=0.05, out=out)
    native.synchronize(native.default_stream())
    scratch.mark_device_written()
    want = oracle.hdiff_c(vals, 0.05)
    got = out.host_array()[2:-2, 2:-2, :]
    assert np.array_equal(got, want)
    s = scratch.host_array()[2:-2, 2:-2, :]
    band = np.zeros(dom, bool)
    band[:2], band[-2:], band[:, :2], band[:, -2:] = True, True, True, True
    assert np.array_equal(s[band], want[band])
    assert np.all(s[~band] == -7.0)
    assert np.all(scratch.host_array()[:2] == -7.0) and np.all(scratch.host_array()[:, :2] == -7.0)
    scratch.view[...] = -9.0
    scratch.to_device()
    st_m(inp=inp, coeff=0.05, out=out)
    scratch.mark_device_written()
    assert np.all(scratch.host_array() == -9.0)


@pytest.mark.gpu
@pytest.mark.parametrize("kernel", ["hdiff", "dycore"])
@pytest.mark.parametrize("grid", [(2, 1), (2, 2), (4, 2)])
def test_peer_fused_local_group_bitwise(kernel, grid):
    """PeerFusedStep.local_group: every rank of the decomposition as a virtual
    rank of this process, each on its own stream, all enqueued before any is
    synchronised (the ranks' kernels, mirror stores into each other's halos
    and step flags run concurrently on the GPU, no host ordering between
    them): 5 eager steps and two replays of a 2-step CUDA graph per rank,
    every rank's block bitwise equal to the undecomposed oracle run."""
    import numpy as np

    import oracle
    import paper_2311_08322_b200 as b200
    from paper_2311_08322_b200 import decomp, native, workloads

    if kernel == "hdiff":
        gdom = (37 * grid[0] + 3, 140 * grid[1] + 5, 6)
        arr = {"u": np.random.default_rng(11).uniform(-1, 1, (gdom[0] + 4, gdom[1] + 4, gdom[2]))}
        sc, fin, fout = {"coeff": 0.05}, "inp", "out"
        run = lambda n: oracle.hdiff_run(arr["u"], n, 0.05)  # noqa: E731
    else:
        gdom = (37 * grid[0] + 3, 70 * grid[1] + 5, 16)
        arr = workloads.dycore_arrays(gdom, 11)
        sc, fin, fout = workloads.DYCORE_SCALARS, "u_in", "u_out"
        run = lambda n: oracle.dycore_run(arr["u"], arr["a"], arr["b"], arr["c"], n, **sc)  # noqa: E731
    st = b200.compile_stencil(workloads.source(kernel), kernel, gen_options={"mirror": fout})
    nr = grid[0] * grid[1]
    ds = [decomp.Decomposition(gdom, grid, r) for r in range(nr)]
    bufs, phases = [], []
    for d in ds:
        u = d.scatter(arr["u"], (2, 2))
        coef = {} if kernel == "hdiff" else {
            n: b200.from_array(np.array(arr[n][d.i0: d.i1, d.j0: d.j1, :], copy=True)) for n in "abc"}
        A, B = b200.from_array(u, (2, 2, 0)), b200.from_array(u, (2, 2, 0))
        bufs.append((A, B))
        phases.append([{fin: A, fout: B, **coef}, {fin: B, fout: A, **coef}])
    streams = [native.aux_stream(f"vrank{r}") for r in range(nr)]
    steps = decomp.PeerFusedStep.local_group(st, ds, phases, sc, fout, (2, 2), streams)

    def check(n, which):
        want = run(n)[2:-2, 2:-2, :]
        for d, (A, B) in zip(ds, bufs):
            got = (B if which else A).host_array()[2:-2, 2:-2, :]
            assert np.array_equal(got, want[d.i0: d.i1, d.j0: d.j1, :]), (kernel, grid, n, d.rank)

    for _ in range(5):
        for s_ in steps:
            s_()
    for s_ in steps:
        native.synchronize(s_.stream)
    check(5, 1)
    # one more step to phase 0, then graph replays (2 steps each, all ranks' graphs launched together)
    for s_ in steps:
        s_()
    graphs = [s_.graph(2) for s_ in steps]
    for _ in range(2):
        for g in graphs:
            g.launch()
    for s_ in steps:
        native.synchronize(s_.stream)
    check(10, 0)
