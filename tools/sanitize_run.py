"""Small runs of every kernel template for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck), checked against the oracle:

    compute-sanitizer --tool memcheck python tools/sanitize_run.py

Fused PARALLEL tile kernel (hdiff f64 / f32), TMEM column kernels (vadv: the
two-CTA W=1 default at nk=20 and over two tile rounds, the W=2 geometry, W=1
at nk=120, generic column kernel at nk=200), the fused dycore
column kernel and its mirrored-halo build (gen_options mirror), per-stage /
plane fallbacks (fuse_parallel off), halo pack / unpack and the peer copy-box
kernel; round 2: the interior + frame launches of a decomposed step (the thin
frame variant), the hdiff tile kernel's mirrored halo stores, and the
read-only L2 eviction kernel."""
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REPO / "oracle"))

import numpy as np  # noqa: E402

import oracle  # noqa: E402
import paper_2311_08322_b200 as b200  # noqa: E402
from paper_2311_08322_b200 import native, workloads  # noqa: E402

rng = np.random.default_rng(5)
ok = True


def check(name, got, want):
    global ok
    good = np.array_equal(got, want)
    ok = ok and good
    print(f"{name}: {'bitwise' if good else 'MISMATCH'}", flush=True)


for dt, npt in (("f64", np.float64), ("f32", np.float32)):
    vals = rng.uniform(-1, 1, (37 + 4, 70 + 4, 3)).astype(npt)
    for opts in (None, {"fuse_parallel": False}):
        st = b200.compile_stencil(workloads.source("hdiff", dt), "hdiff", gen_options=opts)
        inp = b200.from_array(vals, (2, 2, 0))
        out = b200.allocate(dt, (37, 70, 3))
        st(inp=inp, coeff=0.05, out=out)
        check(f"hdiff {dt} {opts}", out.host_array(), oracle.hdiff_c(vals, 0.05))

# default geometry (two CTAs per SM, W=1) at nk=20, and with two tile rounds
# (the in-kernel L2 prefetch of the second tile), W=1 at nk=120, the generic
# column kernel at nk=200, and the one-CTA W=2 geometry explicitly
for shape, opts in (((19, 40, 20), None), ((160, 256, 8), None), ((9, 33, 120), None), ((5, 6, 200), None),
                    ((19, 40, 20), {"tmem_geom": [[2, 4, 128]]})):
    a, b, c, d = oracle.make_diagonally_dominant(rng, shape)
    sv = b200.compile_stencil(workloads.source("vadv"), "vadv", gen_options=opts)
    fa = {n: b200.from_array(v) for n, v in zip("abcd", (a, b, c, d))}
    x = b200.allocate("f64", shape)
    sv(x=x, **fa)
    check(f"vadv {shape} {opts}", x.host_array(), oracle.vadv_c(a, b, c, d))

ddom = (20, 40, 12)
arr = workloads.dycore_arrays(ddom, 3)
sd = b200.compile_stencil(workloads.source("dycore"), "dycore")
u_in, u_out = b200.from_array(arr["u"], (2, 2, 0)), b200.from_array(arr["u"], (2, 2, 0))
sd(u_in=u_in, u_out=u_out, **{n: b200.from_array(arr[n]) for n in "abc"}, **workloads.DYCORE_SCALARS)
check("dycore", u_out.host_array()[2:-2, 2:-2, :],
      oracle.dycore_step(arr["u"], arr["a"], arr["b"], arr["c"], **workloads.DYCORE_SCALARS))

# the dycore with mirrored halo stores (gen_options mirror; PeerFusedStep's
# kernel): the 8 boxes of an interior rank pointed at a scratch field
sm = b200.compile_stencil(workloads.source("dycore"), "dycore", gen_options={"mirror": "u_out"})
u_out2 = b200.from_array(arr["u"], (2, 2, 0))
scratch = b200.from_array(np.zeros_like(arr["u"]), (2, 2, 0))
org = sum(o * st_ for o, st_ in zip(scratch.origin, scratch.strides)) * scratch.itemsize
mboxes = []
for di in (-1, 0, 1):
    for dj in (-1, 0, 1):
        if di or dj:
            bi = {-1: (0, 2), 0: (0, ddom[0]), 1: (ddom[0] - 2, ddom[0])}[di]
            bj = {-1: (0, 2), 0: (0, ddom[1]), 1: (ddom[1] - 2, ddom[1])}[dj]
            mboxes.append((*bi, *bj, scratch.base_address() + org, *scratch.strides))
sm.build_info["module"].set_mirror(mboxes)
sm(u_in=u_in, u_out=u_out2, **{n: b200.from_array(arr[n]) for n in "abc"}, **workloads.DYCORE_SCALARS)
sm.build_info["module"].set_mirror([])
native.synchronize(native.default_stream())
scratch.mark_device_written()
band = np.zeros(ddom, bool)
band[:2], band[-2:], band[:, :2], band[:, -2:] = True, True, True, True
check("dycore mirrored", np.where(band, scratch.host_array()[2:-2, 2:-2, :], u_out2.host_array()[2:-2, 2:-2, :]),
      oracle.dycore_step(arr["u"], arr["a"], arr["b"], arr["c"], **workloads.DYCORE_SCALARS))

# round 2: interior + frame launches (decomp.split_launches; the frame variant)
from paper_2311_08322_b200 import decomp  # noqa: E402

for dt, npt in (("f64", np.float64), ("f32", np.float32)):
    fdom = (37, 300, 3)
    vals = rng.uniform(-1, 1, (fdom[0] + 4, fdom[1] + 4, fdom[2])).astype(npt)
    st = b200.compile_stencil(workloads.source("hdiff", dt), "hdiff")
    inp, out = b200.from_array(vals, (2, 2, 0)), b200.allocate(dt, fdom, fill="poison")
    for sides in (True, (False, True, True, False)):  # all four sides; per side (neighbour_sides)
        out = b200.allocate(dt, fdom, fill="poison")
        inner, frame = decomp.split_launches(st.build_info["module"], fdom, (2, 2), {"inp": inp, "out": out},
                                             {"coeff": 0.05}, native.default_stream(), sides)
        for go in inner + frame:
            go()
        native.synchronize(native.default_stream())
        check(f"hdiff {dt} interior + frame {sides}", out.host_array(), oracle.hdiff_c(vals, 0.05))

# the hdiff tile kernel with mirrored halo stores: 8 boxes into a scratch field
hdom = (37, 300, 3)
vals = rng.uniform(-1, 1, (hdom[0] + 4, hdom[1] + 4, hdom[2]))
shm = b200.compile_stencil(workloads.source("hdiff"), "hdiff", gen_options={"mirror": "out"})
hin, hout = b200.from_array(vals, (2, 2, 0)), b200.allocate("f64", hdom, (2, 2, 0), fill="poison")
hscr = b200.from_array(np.zeros((hdom[0] + 4, hdom[1] + 4, hdom[2])), (2, 2, 0))
horg = sum(o * st_ for o, st_ in zip(hscr.origin, hscr.strides)) * hscr.itemsize
hboxes = []
for di in (-1, 0, 1):
    for dj in (-1, 0, 1):
        if di or dj:
            bi = {-1: (0, 2), 0: (0, hdom[0]), 1: (hdom[0] - 2, hdom[0])}[di]
            bj = {-1: (0, 2), 0: (0, hdom[1]), 1: (hdom[1] - 2, hdom[1])}[dj]
            hboxes.append((*bi, *bj, hscr.base_address() + horg, *hscr.strides))
shm.build_info["module"].set_mirror(hboxes)
shm(inp=hin, coeff=0.05, out=hout)
native.synchronize(native.default_stream())
hscr.mark_device_written()
hband = np.zeros(hdom, bool)
hband[:2], hband[-2:], hband[:, :2], hband[:, -2:] = True, True, True, True
hwant = oracle.hdiff_c(vals, 0.05)
check("hdiff mirrored", np.where(hband, hscr.host_array()[2:-2, 2:-2, :], hout.host_array()[2:-2, 2:-2, :]), hwant)

# the read-only L2 eviction used by tools/ncu_traffic.py
import ctypes  # noqa: E402

evb = ctypes.c_size_t(0)
native.call("gts_b200_l2_evict_read", native.default_stream(), ctypes.byref(evb))
native.synchronize(native.default_stream())
check("l2 evict read", np.array([evb.value > 0]), np.array([True]))

# halo pack / unpack and the peer copy-box kernel on one device
f = b200.from_array(rng.uniform(-1, 1, (12, 9, 4)), (2, 2, 0))
g = b200.allocate("f64", (8, 5, 4), (2, 2, 0))
s = native.default_stream()
buf = b200.allocate("f64", (2 * 9 * 4, 1, 1))
args = [*f.strides, 0, 0, 0, 2, 9, 4, 8, s]
native.call("gts_b200_pack_box", buf.base_address(), f.base_address(), *args)
native.call("gts_b200_unpack_box", g.base_address(), buf.base_address(), *[*g.strides, 10, 0, 0, 2, 9, 4, 8, s])
native.call("gts_b200_copy_box", g.base_address(), *g.strides, f.base_address() + 8 * 2 * f.strides[0],
            *f.strides, 2, 9, 4, 8, s)
native.synchronize(s)
g.mark_device_written()
fv, gv = f.host_array(), g.host_array()
check("pack/unpack + copy_box", np.concatenate([gv[:2], gv[10:12]]), np.concatenate([fv[2:4], fv[0:2]]))
print("SANITIZE_RUN_OK" if ok else "SANITIZE_RUN_FAIL", flush=True)
sys.exit(0 if ok else 1)
